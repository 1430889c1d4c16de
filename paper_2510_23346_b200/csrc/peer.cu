// peer.cu -- the reduce half of the fused row all-reduce (peer.h): sums the N fp32 row partials that the
// ranks' decode kernels pushed into this rank's receive buffer, in rank order (every rank computes the same
// bits), rounds once to bf16.
#include <algorithm>

#include "peer.h"

namespace bdl {

__global__ void __launch_bounds__(256) peer_reduce_kernel(const float* __restrict__ recv, unsigned* cnt, int* parity,
                                                          int* done, int* err, unsigned expected, int nranks,
                                                          long long slot, __nv_bfloat16* __restrict__ Y, int total) {
  // launched right behind the pushing kernel with programmatic serialization and NO griddepcontrol.wait: the
  // arrival counter is the dependency (it also counts this rank's own push), so the spin starts while the
  // pushes are in flight.  The pushing grid is fully resident by then (it triggered this launch).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ int s_par, s_ok;
  if (threadIdx.x == 0) {
    const int par = *(volatile int*)parity;
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int ok = 1;
    for (;;) {
      unsigned c;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(c) : "l"(cnt + par) : "memory");
      if (c >= expected) break;
      long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 2000000000LL) {  // 2 s: a peer never arrived -- report instead of hanging the device
        atomicExch(err, 1);
        ok = 0;
        break;
      }
      __nanosleep(32);
    }
    s_par = par;
    s_ok = ok;
  }
  __syncthreads();
  const int par = s_par;
  if (s_ok) {
    const float* base = recv + (size_t)par * nranks * slot;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
      float y = 0.f;
      for (int r = 0; r < nranks; ++r) y += __ldcg(base + (size_t)r * slot + i);  // rank order: identical bits everywhere
      Y[i] = __float2bfloat16_rn(y);
    }
  }
  __syncthreads();
  // completion of this grid implies completion of the pushing grid (later kernels wait only for this one)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {  // last CTA: every CTA has read the parity and its slots
      cnt[par] = 0;
      *done = 0;
      *parity = par ^ 1;
      __threadfence();
    }
  }
}

int peer_reduce_launch(float* recv, unsigned* cnt, int* parity, int* done, int* err, unsigned expected, int nranks,
                       long long slot, __nv_bfloat16* Y, int T, int M, int pdl, cudaStream_t st) {
  const int total = T * M;
  const int blocks = std::max(1, std::min(64, (total + 255) / 256));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, peer_reduce_kernel, recv, cnt, parity, done, err, expected, nranks, slot, Y, total) ==
                 cudaSuccess
             ? 0
             : -1;
}

}  // namespace bdl
