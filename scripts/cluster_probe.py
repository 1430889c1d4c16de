"""Which split-K schedule the decode GEMM picks, timed with and without the cluster (DSMEM) reduction."""
import os
import subprocess
import sys

code = r'''
import sys, os, json
sys.path.insert(0, os.getcwd())
import scripts.micro_gemm as m
for M, K in [(4096, 4096), (6144, 4096), (4096, 14336), (28672, 4096), (768, 4096), (4096, 512), (3072, 4096)]:
    r = m.run(M, K, 1)
    print(os.environ.get("BDLORA_CLUSTER", "1"), json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
'''
for c in ("1", "0"):
    env = dict(os.environ, BDLORA_CLUSTER=c, BDLORA_DEBUG="1")
    subprocess.run([sys.executable, "-c", code], env=env)
