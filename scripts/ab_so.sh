cd $GRAFT_REPO_ROOT
# usage: build the library of an older commit into $L/libbdlora_old.so first
L=paper_2510_23346_b200
cp $L/libbdlora.so /tmp/new.so
for v in new old new old; do
  if [ $v = old ]; then cp $L/libbdlora_old.so $L/libbdlora.so; else cp /tmp/new.so $L/libbdlora.so; fi
  for w in 70b-decode-bs64-r32 8b-prefill-1024-r64; do
    r=$(timeout 300 python bench.py --steps 20 --warmup 3 --workload $w --skip-cpu --skip-slora --skip-tp-emulation --decode-layers 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['layer_us'],1), {k: round(v,1) for k,v in d['proj_us'].items()})")
    echo "$v $w $r"
  done
done > gpurun_out/ab_so.txt
cp /tmp/new.so $L/libbdlora.so
