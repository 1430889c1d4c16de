// kernels_core.cuh -- CUDA-core kernels of the BD-LoRA layer (sm_100a):
//   segments_kernel   : routing metadata a2 (SGMV segments), integer, bit-exact
//   shrink_kernel     : matmul_3 / matmul_5 -- v = s_a * X A_i[a] gathered per adapter group (BGMV-style)
//   gemv_lora_kernel  : matmul_1/2 + matmul_4/6 + add_1/2 for small T (decode): a weight-streaming
//                       GEMV with 128-bit no-allocate loads, split-K with a deterministic last-CTA
//                       reduction, and the LoRA expand fused into the epilogue (one bf16 rounding)
//   gather_kernel     : adapter loading -- slice (and transpose) this device's shard into the arena
#pragma once
#include "common.cuh"

namespace bdl {

// ------------------------------------------------------------------------------------------------
// Segments: maximal runs of equal consecutive ids (reading R10).  One CTA of 1024 threads.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) segments_kernel(const int* __restrict__ ids, int T, int* __restrict__ seg_start,
                                                        int* __restrict__ seg_len, int* __restrict__ seg_id,
                                                        int* __restrict__ n_seg) {
  __shared__ int warp_tot[32];
  __shared__ int s_carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < T; base += 1024) {
    const int t = base + tid;
    int flag = 0, my = 0;
    if (t < T) {
      my = ids[t];
      flag = (t == 0) || (ids[t - 1] != my);
    }
    // block-wide exclusive scan of flag
    unsigned bal = __ballot_sync(0xffffffffu, flag);
    int in_warp = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < 32; ++w) {
      int c = warp_tot[w];
      before += (w < warp) ? c : 0;
      total += c;
    }
    const int pos = s_carry + before + in_warp;
    if (flag) {
      seg_start[pos] = t;
      seg_id[pos] = my;
    }
    __syncthreads();
    if (tid == 0) s_carry += total;
    __syncthreads();
  }
  const int n = s_carry;
  __threadfence_block();
  __syncthreads();
  for (int s = tid; s < n; s += 1024) {
    const int nxt = (s + 1 < n) ? seg_start[s + 1] : T;
    seg_len[s] = nxt - seg_start[s];
  }
  if (tid == 0) *n_seg = n;
}

// ------------------------------------------------------------------------------------------------
// Shrink (matmul_3 / matmul_5): v[t][j][k] = s_a * sum_d X[t][d] * A_{a,j}[k][d]  for k < rs(a).
// Grid (T, J, ceil(Rc/8)); CTA = 8 warps, warp w computes rank row k = 8*blockIdx.z + w.
// CTA blockIdx.x = t does the work only if t is the FIRST token of its adapter id; it then covers
// every token with that id, so each A row is streamed from HBM once per distinct adapter
// (algorithmic bytes: sum over distinct adapters).  Tokens are processed in passes
// of MT with the A row chunk held in registers.
// ------------------------------------------------------------------------------------------------
template <int MT>
__global__ void __launch_bounds__(256) shrink_kernel(const __nv_bfloat16* __restrict__ X, int T,
                                                     const int* __restrict__ ids, const SlotEntry* __restrict__ tab,
                                                     const __nv_bfloat16* __restrict__ arena, Geom g,
                                                     float* __restrict__ v) {
  extern __shared__ int s_members[];  // [T]
  __shared__ int s_cnt, s_dup;
  const int t = blockIdx.x, j = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = __ldg(ids + t);
  if (a < 0) return;
  const SlotEntry e = tab[a];
  if (j >= g.J) return;
  if ((int)blockIdx.z * 8 >= e.rs) return;  // whole CTA beyond this adapter's rank
  if (warp == 0) {
    // warp 0 gathers the members (tokens u with ids[u] == a) in token order; dup if any u < t.
    int cnt = 0, dup = 0;
    for (int base = 0; base < T; base += 32) {
      const int u = base + lane;
      const int idu = (u < T) ? __ldg(ids + u) : -2;
      const unsigned m = __ballot_sync(0xffffffffu, idu == a);
      if (u < T && idu == a) {
        if (u < t) dup = 1;
        s_members[cnt + __popc(m & ((1u << lane) - 1u))] = u;
      }
      cnt += __popc(m);
    }
    dup = __any_sync(0xffffffffu, dup);
    if (lane == 0) {
      s_cnt = cnt;
      s_dup = dup;
    }
  }
  __syncthreads();
  if (s_dup) return;
  const int k = blockIdx.z * 8 + warp;
  if (k >= e.rs) return;
  const int K = g.K;
  const __nv_bfloat16* Ar = arena + e.offA[j] + (size_t)k * K;
  const int cnt = s_cnt;
  for (int m0 = 0; m0 < cnt; m0 += MT) {
    float acc[MT];
    int tok[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      acc[m] = 0.f;
      tok[m] = (m0 + m < cnt) ? s_members[m0 + m] : -1;
    }
    for (int d = lane * 8; d < K; d += 256) {
      float af[8];
      bf16x8_to_f32(ld_cached_u4(Ar + d), af);
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (tok[m] >= 0) {
          float xf[8];
          bf16x8_to_f32(ld_cached_u4(X + (size_t)tok[m] * K + d), xf);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[m] = fmaf(af[q], xf[q], acc[m]);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const float s = warp_sum(acc[m]);
      if (lane == 0 && tok[m] >= 0) v[((size_t)tok[m] * g.J + j) * g.Rc + k] = e.scale * s;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Shrink, latency-optimised (decode): one CTA of 128 threads per (first token of an adapter group,
// slice j, rank row k); the K reduction is spread over all 128 threads (4 independent 128-bit loads
// in flight per thread for K = 4096) and reduced through shared memory in a fixed order
// (deterministic).  Signals programmatic dependents immediately so the base GEMM that consumes v can
// start streaming its weights while this runs.
// ------------------------------------------------------------------------------------------------
template <int MT>
__global__ void __launch_bounds__(128) shrink_rows_kernel(const __nv_bfloat16* __restrict__ X, int T,
                                                          const int* __restrict__ ids,
                                                          const SlotEntry* __restrict__ tab,
                                                          const __nv_bfloat16* __restrict__ arena, Geom g,
                                                          float* __restrict__ v) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // programmatic dependency: X and ids may be produced by the preceding kernel
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ int s_members[];  // [T]
  __shared__ int s_cnt, s_dup;
  __shared__ float s_red[4][MT];
  const int t = blockIdx.x, j = blockIdx.y, k = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int a = __ldg(ids + t);
  if (a < 0) return;
  const SlotEntry e = tab[a];
  if (k >= e.rs || j >= g.J) return;
  if (warp == 0) {
    int cnt = 0, dup = 0;
    for (int base = 0; base < T; base += 32) {
      const int u = base + lane;
      const int idu = (u < T) ? __ldg(ids + u) : -2;
      const unsigned m = __ballot_sync(0xffffffffu, idu == a);
      if (u < T && idu == a) {
        if (u < t) dup = 1;
        s_members[cnt + __popc(m & ((1u << lane) - 1u))] = u;
      }
      cnt += __popc(m);
      if (__any_sync(0xffffffffu, dup)) break;  // not the group leader: stop early
    }
    dup = __any_sync(0xffffffffu, dup);
    if (lane == 0) {
      s_cnt = cnt;
      s_dup = dup;
    }
  }
  __syncthreads();
  if (s_dup) return;
  const int K = g.K;
  const __nv_bfloat16* Ar = arena + e.offA[j] + (size_t)k * K;
  const int cnt = s_cnt;
  for (int m0 = 0; m0 < cnt; m0 += MT) {
    float acc[MT];
    int tok[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      acc[m] = 0.f;
      tok[m] = (m0 + m < cnt) ? s_members[m0 + m] : -1;
    }
#pragma unroll 4
    for (int d = threadIdx.x * 8; d < K; d += 128 * 8) {
      float af[8];
      bf16x8_to_f32(ld_cached_u4(Ar + d), af);
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (tok[m] >= 0) {
          float xf[8];
          bf16x8_to_f32(ld_cached_u4(X + (size_t)tok[m] * K + d), xf);
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[m] = fmaf(af[q], xf[q], acc[m]);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const float s = warp_sum(acc[m]);
      if (lane == 0) s_red[warp][m] = s;
    }
    __syncthreads();
    if (threadIdx.x < MT && tok[threadIdx.x] >= 0) {
      const int m = threadIdx.x;
      const float s = (s_red[0][m] + s_red[1][m]) + (s_red[2][m] + s_red[3][m]);
      v[((size_t)tok[m] * g.J + j) * g.Rc + k] = e.scale * s;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------------
// Base GEMV + fused LoRA expand (decode, small T).
// Grid (ntiles, S): CTA = 8 warps x RW output rows = 8*RW rows of W^T; split s covers K range
// [s*Kc, min(K,(s+1)*Kc)).  S == 1: direct epilogue.  S > 1: partials to part[s][t][n] (plain
// stores), per-tile arrival counter; the last-arriving CTA sums the S partials in split order
// (deterministic), adds the expand term, rounds once to bf16 and re-arms the counter.
// ------------------------------------------------------------------------------------------------
template <int TT, int RW>
__global__ void __launch_bounds__(256) gemv_lora_kernel(const __nv_bfloat16* __restrict__ X, int T,
                                                        const __nv_bfloat16* __restrict__ W,
                                                        const int* __restrict__ ids,
                                                        const SlotEntry* __restrict__ tab,
                                                        const __nv_bfloat16* __restrict__ arena, Geom g,
                                                        const float* __restrict__ v, __nv_bfloat16* __restrict__ Y,
                                                        float* __restrict__ part, int* __restrict__ counters, int S,
                                                        int Kc) {
  constexpr int ROWS = 8 * RW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = g.K, M = g.M;
  const int tile = blockIdx.x, s = blockIdx.y;
  const int row0 = tile * ROWS + warp * RW;
  const int k_lo = s * Kc;
  const int k_hi = min(K, k_lo + Kc);
  __shared__ int s_last;

  for (int t0 = 0; t0 < T; t0 += TT) {
    float acc[RW][TT];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int q = 0; q < TT; ++q) acc[r][q] = 0.f;
    const __nv_bfloat16* wrow[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) wrow[r] = W + (size_t)min(row0 + r, M - 1) * K;
#pragma unroll 2
    for (int d = k_lo + lane * 8; d < k_hi; d += 256) {
      uint4 wv[RW];
#pragma unroll
      for (int r = 0; r < RW; ++r) wv[r] = ld_stream_u4(wrow[r] + d);
#pragma unroll
      for (int q = 0; q < TT; ++q) {
        if (t0 + q < T) {
          float xf[8];
          bf16x8_to_f32(ld_cached_u4(X + (size_t)(t0 + q) * K + d), xf);
#pragma unroll
          for (int r = 0; r < RW; ++r) {
            float wf[8];
            bf16x8_to_f32(wv[r], wf);
#pragma unroll
            for (int p = 0; p < 8; ++p) acc[r][q] = fmaf(wf[p], xf[p], acc[r][q]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int q = 0; q < TT; ++q) acc[r][q] = warp_sum(acc[r][q]);
    // lane l handles (r, q) = (l / TT, l % TT)
#pragma unroll
    for (int r = 0; r < RW; ++r) {
#pragma unroll
      for (int q = 0; q < TT; ++q) {
        if (lane == r * TT + q) {
          const int n = row0 + r, t = t0 + q;
          if (n < M && t < T) {
            if (S == 1) {
              const int a = __ldg(ids + t);
              const float y = acc[r][q] + lora_expand_term(t, n, a, tab, arena, g, v, T);
              Y[(size_t)t * M + n] = __float2bfloat16_rn(y);
            } else {
              part[((size_t)s * T + t) * M + n] = acc[r][q];
            }
          }
        }
      }
    }
  }
  if (S == 1) return;
  // ---- split-K fix-up: last CTA of this row tile reduces in split order ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(counters + tile, 1);
    s_last = (old == S - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int tile_rows = min(ROWS, M - tile * ROWS);
  for (int idx = threadIdx.x; idx < tile_rows * T; idx += blockDim.x) {
    const int n = tile * ROWS + idx % tile_rows;
    const int t = idx / tile_rows;
    float y = 0.f;
    for (int q = 0; q < S; ++q) y += __ldcg(part + ((size_t)q * T + t) * M + n);
    const int a = __ldg(ids + t);
    y += lora_expand_term(t, n, a, tab, arena, g, v, T);
    Y[(size_t)t * M + n] = __float2bfloat16_rn(y);
  }
  if (threadIdx.x == 0) counters[tile] = 0;
}

// ------------------------------------------------------------------------------------------------
// Loader: dst = (transpose ? src[r0:r0+nr, c0:c0+nc]^T : src[r0:r0+nr, c0:c0+nc]), src row-major ld,
// dst row-major with leading dimension ldd (0 = packed: nc, or nr when transposed).
// ------------------------------------------------------------------------------------------------
__global__ void gather_kernel(const uint16_t* __restrict__ src, long long ld, int r0, int c0, int nr, int nc,
                              int transpose, uint16_t* __restrict__ dst, long long ldd) {
  if (ldd == 0) ldd = transpose ? nr : nc;
  __shared__ uint16_t tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;  // bx over columns, by over rows of the sub-block
  for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
    const int r = by + yy, c = bx + threadIdx.x;
    if (r < nr && c < nc) tile[yy][threadIdx.x] = src[(long long)(r0 + r) * ld + (c0 + c)];
  }
  __syncthreads();
  if (!transpose) {
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
      const int r = by + yy, c = bx + threadIdx.x;
      if (r < nr && c < nc) dst[(long long)r * ldd + c] = tile[yy][threadIdx.x];
    }
  } else {
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
      const int c = bx + yy, r = by + threadIdx.x;  // dst row = c, dst col = r
      if (r < nr && c < nc) dst[(long long)c * ldd + r] = tile[threadIdx.x][yy];
    }
  }
}

// Alg. 2 all-gather output: G [N][T][M] (rank-major chunks) -> Y [T][N * M] (device blocks side by side).
__global__ void interleave_chunks_kernel(const uint16_t* __restrict__ G, uint16_t* __restrict__ Y, int T, int M, int N) {
  const long long total = (long long)N * T * M;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(e % M);
    const long long ct = e / M;
    const int t = (int)(ct % T), c = (int)(ct / T);
    Y[((long long)t * N + c) * M + m] = G[e];
  }
}

}  // namespace bdl
