// decode.h -- host interface of the lean decode kernel (kernels_decode.cuh), compiled in its own
// translation unit (decode.cu) and called by runtime.cu.  C++ linkage, library-internal.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>

#include "common.cuh"
#include "peer.h"

namespace bdl {

struct DecLaunch {
  Geom g;
  const __nv_bfloat16* X;
  int T;                      // 1..64 (17..64: the pool holds one adapter -- the caller checks)
  const __nv_bfloat16* W;     // W^T [M, K] bf16, K-major
  const int* ids;
  const SlotEntry* tab;
  const __nv_bfloat16* arena;
  const float* v;             // lora == 2: v [C][T][J][Rc] fp32
  __nv_bfloat16* Y;
  void* cnt;                  // >= dec_counter_bytes() of zeroed counters (workspace counter region)
  void* scratch;              // >= dec_scratch_bytes(num_sms) bytes
  int num_sms;
  cudaStream_t stream;
  int pdl;
  int lora;                   // 1 K-local, 2 v precomputed (per-output gather), 3 v precomputed (B rows staged),
                              // 4 v precomputed, any number of adapters (B rows streamed in chunks, BN = 64)
  const CUtensorMap* amap;    // the pool arena as [rows, K] bf16 with 16-row boxes (tensor-core K-local shrink), or null
  int push;                   // 1: fused row all-reduce -- fp32 partial pushed to every rank of `peer` (not Y)
  PeerDev peer;
  int* grid_out;              // optional: the launched grid (the reduce kernel's expected arrivals / rank)
};

constexpr int kDecMaxT = 64;      // BN = 16 tiles up to 16 tokens, BN = 64 tiles (one-adapter pools) up to 64
constexpr int kDecMaxPushT = 16;  // the fused row all-reduce serves BN = 16 decode batches
constexpr int kDecLoraRowsHost = 32;  // == kDecLoraRows: K-local capacity (sum of the batch's distinct local ranks)

size_t dec_counter_bytes();
size_t dec_scratch_bytes(int num_sms, int T);
bool dec_eligible(const Geom& g, int T);
bool dec_enabled();                        // BDLORA_DECODE=0 selects the older single-kernel forward
// Returns 0 on launch, non-zero if the shape is not handled (caller falls back), negative on a CUDA error.
int dec_launch(const DecLaunch& a);
// Multi-adapter shrink of a T <= 64 batch into v [T][J][Rc] fp32 (dec_shrink_kernel).  0 on launch, 1 if T is
// out of range, negative on a CUDA error.
int dec_shrink_launch(const Geom& g, const __nv_bfloat16* X, int T, const int* ids, const SlotEntry* tab,
                      const __nv_bfloat16* arena, float* v, int num_sms, cudaStream_t st, int pdl, int rs_max);
void dec_last_launch(int info[8]);
void dec_set_trace(long long* buf);

}  // namespace bdl
