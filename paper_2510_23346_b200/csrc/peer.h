// peer.h -- device view of a peer group: every rank's receive buffer and arrival counters mapped into
// this rank's address space (CUDA IPC over NVLink / NVSwitch, or N emulated ranks on one device).
// Used by the fused row forward: the decode kernel's epilogue pushes its fp32 row
// partial straight into every rank's receive slot, and a small reduce kernel on each rank sums the N slots
// in rank order -- the base all-reduce of Alg. 1 line 15 without a separate NCCL launch.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace bdl {

struct PeerDev {
  float* const* recv;    // [nranks] every rank's receive buffer base: [2 parities][nranks sources][slot] fp32
  unsigned* const* cnt;  // [nranks] every rank's arrival counters [2 parities]
  const int* parity;     // this rank's call parity (flipped by its reduce kernel after each call)
  int rank, nranks;
  long long slot;        // elements per (parity, source) slot (>= T * M)
};

// Y[t][n] = bf16( sum_{r = 0..N-1} recv[parity][r][t][n] ) once this rank's counter for the parity reaches
// `expected` (= N x the pushing grid); the last CTA re-arms the counter and flips the parity.  A spin that
// exceeds ~2 s sets *err = 1 and gives up (no hang).
int peer_reduce_launch(float* recv, unsigned* cnt, int* parity, int* done, int* err, unsigned expected, int nranks,
                       long long slot, __nv_bfloat16* Y, int T, int M, int pdl, cudaStream_t st);

}  // namespace bdl
