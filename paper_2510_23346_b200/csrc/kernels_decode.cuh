// kernels_decode.cuh -- the decode forward (T <= 16 tokens) of one adapted projection in ONE lean kernel:
// base GEMM (matmul_1 / matmul_2) on the tcgen05 tensor cores fed by TMA, the LoRA shrink (matmul_3 / _5)
// and expand + add (matmul_4 / _6, add_1 / _2) on the CUDA cores of the epilogue warps, one bf16 rounding.
//
// Why a separate kernel (DESIGN.md §6 "Decode kernel"): at decode a projection is a weight stream of
// 4-240 MB, so at TP >= 2 most projections take only 1-15 us of HBM time and a fixed per-launch cost of
// several us (launch, prologue, pipeline fill, epilogue tail) decides the layer time.  This kernel is built
// around hiding that cost:
//   * ~104 KB of shared memory per CTA and <= 170 registers per thread, so TWO CTAs fit on an SM: while a
//     projection's CTAs finish their tails, the next projection's CTAs (programmatic dependent launch) are
//     already resident and stream their first ring of weights (weights never depend on the preceding kernel;
//     only X, ids and v do, and those are read after griddepcontrol.wait);
//   * a small executed footprint (no multi-adapter tensor-core expand, no cluster / grid-wide machinery);
//   * K-local LoRA: the layer is linear in a partition of K, y = sum_seg [X_seg W_seg + s (X_seg A_seg^T) B]
//     (Alg. 1/2 matmul_3/4 and matmul_5/6 regrouped over K), so every CTA computes v_seg for its
//     own K range from X and the adapter's A rows (L2-resident, a few KB) while its weights stream, and adds
//     v_seg B to its own (partial) tile.  No CTA waits for another's shrink; no separate shrink launch.
//   * split tiles are finished by the last-arriving contributor (deterministic CTA order) through a
//     fixed-size counter region of the workspace.
//
//   warp 0      : TMA producer  (W tile [128 x 64] + X tile [16 x 64] per stage, SWIZZLE_128B)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (M = 128 output columns, N = 16 tokens)
//   warps 2..5  : epilogue      (K-local v_seg during the mainloop; TMEM -> registers, + LoRA, store / partial)
//
// LoRA modes: 1 = K-local (BD / NFS pools: the shrink and expand of every adapter are device-local), the
// host guarantees the batch's distinct adapters have at most kDecLoraRows local rank rows in total;
// 2 = v precomputed (S-LoRA, after its all-gather / all-reduce): the tile's finisher adds s v B[a].
#pragma once
#include "common.cuh"
#include "ptx.cuh"

namespace bdl {

constexpr int kDecThreads = 192;
constexpr int kDecBM = 128, kDecBK = 64, kDecBN = 16;
constexpr int kDecLoraRows = 32;   // K-local: sum over the batch's distinct adapters of their local rank rs
constexpr int kDecMaxGroups = 16;  // distinct adapters of a <= 16-token batch
constexpr int kDecMaxGrid = 1024;  // split-tile counters (indexed by the first contributor CTA)

struct DecParams {
  int M, K, T;
  int m_tiles, k_blocks, units, grid;
  const __nv_bfloat16* X;
  const int* ids;
  const SlotEntry* tab;
  const __nv_bfloat16* arena;
  Geom g;
  const float* v;     // lora == 2: v [C][T][J][Rc] fp32
  __nv_bfloat16* Y;
  float* part;        // [grid][2][16][128] fp32 split-tile partials (slot 0: a CTA's first segment, 1: its last)
  int* cnt;           // [kDecMaxGrid] arrival counters of split tiles, zero between launches
  int lora;           // 0 none, 1 K-local, 2 v precomputed
  int pdl;
  int nstages;
  long long* trace;   // optional per-CTA %globaltimer stamps (32 per CTA)
};

template <int S>
struct DecSmem {
  static constexpr int kW = kDecBM * kDecBK * 2;  // 16 KB weight tile
  static constexpr int kX = kDecBN * kDecBK * 2;  // 2 KB token tile
  static constexpr int kXOff = S * kW;
  static constexpr int kBarOff = kXOff + S * kX;
  static constexpr int kMiscOff = kBarOff + 256;
  // misc ints: [0,16) ids  [16,32) group of token  [32,48) group adapter  [48,64) group rs  [64,80) group row
  // offset q0  [80,96) member masks  [96] n_groups  [97] rows total ; floats [128,144) group scale ;
  // long long [160 + 2*(g*3 + j)) group A / B offsets per slice (as int pairs)
  static constexpr int kMiscBytes = 2048;
  static constexpr int kVsOff = kMiscOff + kMiscBytes;          // v_seg [16 tokens][3 slices][32] fp32
  static constexpr int kVsBytes = kDecBN * 3 * kDecLoraRows * 4;
  static constexpr int kBOff = kVsOff + kVsBytes;               // B rows [32][128] bf16 of the tile's columns
  static constexpr int kBBytes = kDecLoraRows * kDecBM * 2;
  static constexpr int kBytes = kBOff + kBBytes + 1024;         // + 1024-B alignment slack
  static_assert(kBytes <= 113 * 1024, "two CTAs per SM");
};

#define DEC_TRACE(slot)                                               \
  do {                                                                \
    if (p.trace) {                                                    \
      long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));          \
      p.trace[(size_t)blockIdx.x * 32 + (slot)] = t_;                 \
    }                                                                 \
  } while (0)

__device__ __forceinline__ int dec_u_lo(long long c, int units, int grid) { return (int)(c * units / grid); }
__device__ __forceinline__ int dec_cta_of(long long u, int units, int grid) {
  return (int)(((u + 1) * grid + units - 1) / units) - 1;  // largest c with floor(c U / G) <= u
}
__device__ __forceinline__ int dec_slice_of(const Geom& g, int n) {
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSlices; ++q)
    if (q < g.J && n >= g.col0[q]) j = q;
  return j;
}

template <int S>
__global__ void __launch_bounds__(kDecThreads, 2)
    dec_lora_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                         const DecParams p) {
  using L = DecSmem<S>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sW = smem;
  uint8_t* sX = smem + L::kXOff;
  uint64_t* full = (uint64_t*)(smem + L::kBarOff);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = (uint32_t*)(tempty + 2);
  int* s_last = (int*)(tmem_holder + 1);
  int* mi = (int*)(smem + L::kMiscOff);
  int* s_ids = mi;
  int* s_grp = mi + 16;
  int* s_gad = mi + 32;
  int* s_grs = mi + 48;
  int* s_gq0 = mi + 64;
  int* s_gmask = mi + 80;
  float* s_gsc = (float*)(mi + 128);
  long long* s_goff = (long long*)(mi + 160);  // [g][0..2] = offA[j], [g][3..5] = offB[j]
  float* s_vs = (float*)(smem + L::kVsOff);
  uint16_t* s_B = (uint16_t*)(smem + L::kBOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int UNITS = p.units, GRID = p.grid;
  const int u_lo = dec_u_lo(cta, UNITS, GRID);
  const int u_hi = dec_u_lo(cta + 1, UNITS, GRID);
  if (threadIdx.x == 0) DEC_TRACE(0);

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmW);
    ptx::tma_prefetch_desc(&tmX);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::fence_mbar_init();
    ptx::fence_proxy_async();
  }
  if (warp == 1) ptx::tmem_alloc<32>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // the next kernel may launch now: it only takes SM room this grid leaves free, and waits for this grid's
  // completion (griddepcontrol.wait) before touching anything this grid writes
  if (threadIdx.x == 0) ptx::pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (ptx::elect_one()) {
      const uint64_t pol_w = ptx::policy_evict_first();
      const uint64_t pol_x = ptx::policy_evict_last();
      const int nu = u_hi - u_lo;
      const int NS = p.nstages;
      const int P = min(nu, NS);
      // weights do not depend on the preceding kernel: the first ring is in flight before the dependency
      for (int idx = 0; idx < P; ++idx) {
        const int u = u_lo + idx, tile = u / p.k_blocks, kb = u - tile * p.k_blocks;
        ptx::mbar_expect_tx(&full[idx], L::kW);
        ptx::tma_load_2d(sW + idx * L::kW, &tmW, &full[idx], kb * kDecBK, tile * kDecBM, pol_w);
      }
      DEC_TRACE(1);
      if (p.pdl) ptx::pdl_wait();
      for (int idx = 0; idx < P; ++idx) {
        const int u = u_lo + idx, tile = u / p.k_blocks, kb = u - tile * p.k_blocks;
        (void)tile;
        ptx::mbar_arrive_expect_tx(&full[idx], L::kX);
        ptx::tma_load_2d(sX + idx * L::kX, &tmX, &full[idx], kb * kDecBK, 0, pol_x);
      }
      int stage = (P == NS) ? 0 : P;
      uint32_t phase = (P == NS) ? 1u : 0u;
      for (int idx = P; idx < nu; ++idx) {
        const int u = u_lo + idx, tile = u / p.k_blocks, kb = u - tile * p.k_blocks;
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], L::kW + L::kX);
        ptx::tma_load_2d(sW + stage * L::kW, &tmW, &full[stage], kb * kDecBK, tile * kDecBM, pol_w);
        ptx::tma_load_2d(sX + stage * L::kX, &tmX, &full[stage], kb * kDecBK, 0, pol_x);
        if (++stage == NS) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(kDecBM, kDecBN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = u_lo; u < u_hi;) {
        const int tile = u / p.k_blocks;
        const int kb0 = u - tile * p.k_blocks;
        const int kb1 = min(p.k_blocks, kb0 + (u_hi - u));
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * kDecBN);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (u == u_lo && kb == kb0) DEC_TRACE(2);
          const uint64_t a_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sW + stage * L::kW));
          const uint64_t b_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sX + stage * L::kX));
#pragma unroll
          for (int k = 0; k < kDecBK / 16; ++k)
            ptx::mma_bf16(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          ptx::mma_commit(&empty[stage]);
          if (++stage == p.nstages) {
            stage = 0;
            phase ^= 1;
          }
        }
        ptx::mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        u += kb1 - kb0;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q4 = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q4 * 32 + lane;
    const int etid = threadIdx.x - 64;
    const int we = etid >> 5;  // epilogue warp 0..3
    const int T = p.T;
    if (p.pdl) ptx::pdl_wait();  // X, ids (and v) of the preceding kernel are visible; orders our Y writes
    // ---- adapter groups of the batch (distinct ids, order of first appearance) -------------------------
    if (p.lora == 1) {
      if (we == 0) {
        // lane t < T holds token t's id; leaders (first token of each id) in token order define the groups
        const int id = (lane < T) ? __ldg(p.ids + lane) : -1;
        bool lead = id >= 0;
        for (int t2 = 0; t2 < kDecBN; ++t2) {
          const int o = __shfl_sync(0xffffffffu, id, t2);
          if (t2 < lane && o == id) lead = false;
        }
        const unsigned lmask = __ballot_sync(0xffffffffu, lead);
        const int gidx = __popc(lmask & ((1u << lane) - 1u));  // this lane's group index if it leads
        int mygrp = -1;
        for (int t2 = 0; t2 < kDecBN; ++t2) {
          const int o = __shfl_sync(0xffffffffu, id, t2);
          const int gi = __shfl_sync(0xffffffffu, gidx, t2);
          if (mygrp < 0 && id >= 0 && o == id && ((lmask >> t2) & 1u)) mygrp = gi;
        }
        if (lane < kDecBN) {
          s_ids[lane] = id;
          s_grp[lane] = mygrp;
        }
        int rs = 0;
        if (lead) {
          const SlotEntry e = p.tab[id];
          rs = min(e.rs, kDecLoraRows);
          s_gad[gidx] = id;
          s_gsc[gidx] = e.scale;
#pragma unroll
          for (int j = 0; j < kMaxSlices; ++j) {
            s_goff[gidx * 6 + j] = e.offA[j];
            s_goff[gidx * 6 + 3 + j] = e.offB[j];
          }
        }
        // rank-row offset of each group: exclusive prefix of rs in leader (= lane) order
        int incl = rs;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (lead) {
          s_grs[gidx] = rs;
          s_gq0[gidx] = incl - rs;
        }
        const int ng = __popc(lmask);
        for (int gg = 0; gg < ng; ++gg) {  // member mask of every group (warp-uniform loop)
          const int target = __shfl_sync(0xffffffffu, id, __fns(lmask, 0, gg + 1));
          const unsigned m = __ballot_sync(0xffffffffu, id >= 0 && id == target);
          if (lane == 0) s_gmask[gg] = (int)m;
        }
        if (lane == 0) {
          mi[96] = ng;
          mi[97] = min(tot, kDecLoraRows);
        }
      }
      ptx::named_bar_sync(1, 128);
    }
    const int ngroups = (p.lora == 1) ? mi[96] : 0;

    int acc = 0;
    uint32_t acc_phase = 0;
    int cur_tile = -1;
    for (int u = u_lo; u < u_hi;) {
      const int tile = u / p.k_blocks;
      const int kb0 = u - tile * p.k_blocks;
      const int kb1 = min(p.k_blocks, kb0 + (u_hi - u));
      const bool whole = (kb0 == 0 && kb1 == p.k_blocks);
      const int n0 = tile * kDecBM;
      const int n = n0 + row;
      const int jlo = dec_slice_of(p.g, n0);
      const int jn = dec_slice_of(p.g, min(n, p.M - 1));
      float lr[kDecBN];
#pragma unroll
      for (int i = 0; i < kDecBN; ++i) lr[i] = 0.f;
      if (p.lora == 1 && ngroups > 0) {
        // ---- K-local shrink of this segment: v_seg[t][j][k] = s_a sum_{d in seg} X[t][d] A_{a,j}[k][d] -----
        const int jhi = dec_slice_of(p.g, min(n0 + kDecBM, p.M) - 1);
        const int nj = jhi - jlo + 1;
        const int rows = mi[97];
        const int d_lo = kb0 * kDecBK, d_hi = min(p.K, kb1 * kDecBK);
        ptx::named_bar_sync(1, 128);  // previous segment's readers of s_vs / s_B are done
        for (int item = we; item < nj * rows; item += 4) {
          const int jj = item / rows, q = item - jj * rows;
          int g = 0;
          while (g + 1 < ngroups && s_gq0[g + 1] <= q) ++g;
          const int k = q - s_gq0[g];
          const int j = jlo + jj;
          const unsigned mask = (unsigned)s_gmask[g];
          const __nv_bfloat16* Ar = p.arena + s_goff[g * 6 + j] + (size_t)k * p.K;
          float a16[kDecBN];
#pragma unroll
          for (int t = 0; t < kDecBN; ++t) a16[t] = 0.f;
          for (int d = d_lo + lane * 8; d < d_hi; d += 256) {
            float af[8];
            bf16x8_to_f32(ld_cached_u4(Ar + d), af);
#pragma unroll
            for (int t = 0; t < kDecBN; ++t) {
              if ((mask >> t) & 1u) {
                float xf[8];
                bf16x8_to_f32(ld_cached_u4(p.X + (size_t)t * p.K + d), xf);
#pragma unroll
                for (int e = 0; e < 8; ++e) a16[t] = fmaf(af[e], xf[e], a16[t]);
              }
            }
          }
          const float sc = s_gsc[g];
#pragma unroll
          for (int t = 0; t < kDecBN; ++t) {
            if ((mask >> t) & 1u) {
              const float sm = warp_sum(a16[t]);
              if (lane == 0) s_vs[(t * 3 + jj) * kDecLoraRows + k] = sc * sm;
            }
          }
        }
        // ---- B rows of my output column for every group (once per tile): s_B[q][row] ----------------------
        if (tile != cur_tile) {
          const int lo = p.g.e_lo[jn], hi = p.g.e_hi[jn], ldb = hi - lo;
          const bool in = n < p.M && n >= lo && n < hi;
          for (int q = 0; q < rows; ++q) {
            int g = 0;
            while (g + 1 < ngroups && s_gq0[g + 1] <= q) ++g;
            const int k = q - s_gq0[g];
            const uint16_t* Bp = reinterpret_cast<const uint16_t*>(p.arena + s_goff[g * 6 + 3 + jn]);
            s_B[q * kDecBM + row] = in ? __ldg(Bp + (size_t)k * ldb + (n - lo)) : (uint16_t)0;
          }
          cur_tile = tile;
        }
        ptx::named_bar_sync(1, 128);
        // ---- expand: lr[t] = v_seg[t][j] . B_{a(t),j}[:, n] ---------------------------------------------
        const int jj = jn - jlo;
#pragma unroll
        for (int t = 0; t < kDecBN; ++t) {
          if (t < T) {
            const int g = s_grp[t];
            if (g >= 0) {
              const int rs = s_grs[g], q0 = s_gq0[g];
              const float* vs = s_vs + (t * 3 + jj) * kDecLoraRows;
              float s0 = 0.f, s1 = 0.f;
              int k = 0;
              for (; k + 1 < rs; k += 2) {
                s0 = fmaf(vs[k], bf16_bits_to_f32(s_B[(q0 + k) * kDecBM + row]), s0);
                s1 = fmaf(vs[k + 1], bf16_bits_to_f32(s_B[(q0 + k + 1) * kDecBM + row]), s1);
              }
              if (k < rs) s0 = fmaf(vs[k], bf16_bits_to_f32(s_B[(q0 + k) * kDecBM + row]), s0);
              lr[t] = s0 + s1;
            }
          }
        }
      }
      if (u == u_lo && etid == 0) DEC_TRACE(3);
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      if (u == u_lo && etid == 0) DEC_TRACE(4);
      uint32_t r[16];
      ptx::tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(acc * kDecBN), r);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);  // the accumulator is in registers: the MMA may reuse it
      if (whole) {
        if (p.lora == 2 && n < p.M) {
#pragma unroll
          for (int t = 0; t < kDecBN; ++t)
            if (t < T) lr[t] = lora_expand_term(t, n, __ldg(p.ids + t), p.tab, p.arena, p.g, p.v, T);
        }
        if (n < p.M) {
#pragma unroll
          for (int t = 0; t < kDecBN; ++t)
            if (t < T) p.Y[(size_t)t * p.M + n] = __float2bfloat16_rn(__uint_as_float(r[t]) + lr[t]);
        }
      } else {
        // split tile: this CTA's fp32 partial (its K range, with its K-local LoRA share) -> slot, token-major
        const int slot = (tile * p.k_blocks > u_lo) ? 1 : 0;
        float* my = p.part + (size_t)(cta * 2 + slot) * kDecBN * kDecBM;
#pragma unroll
        for (int t = 0; t < kDecBN; ++t)
          if (t < T) __stcg(my + t * kDecBM + row, __uint_as_float(r[t]) + lr[t]);
        ptx::named_bar_sync(1, 128);
        const int ts = tile * p.k_blocks;
        const int c_first = dec_cta_of(ts, UNITS, GRID);
        if (etid == 0) {
          const int got = kb1 - kb0;
          const int old = ptx::atom_add_acq_rel_gpu(p.cnt + c_first, got);
          *s_last = (old + got == p.k_blocks);
        }
        ptx::named_bar_sync(1, 128);
        if (*s_last) {
          // finisher: contributors' partials summed in CTA order (deterministic), one rounding
          if (etid == 0) DEC_TRACE(6);
          const int c_last = dec_cta_of(ts + p.k_blocks - 1, UNITS, GRID);
          float y[kDecBN];
#pragma unroll
          for (int t = 0; t < kDecBN; ++t) y[t] = 0.f;
          for (int c = c_first; c <= c_last; ++c) {
            const int sl = (ts > dec_u_lo(c, UNITS, GRID)) ? 1 : 0;
            const float* src = p.part + (size_t)(c * 2 + sl) * kDecBN * kDecBM + row;
#pragma unroll
            for (int t = 0; t < kDecBN; ++t)
              if (t < T) y[t] += __ldcg(src + t * kDecBM);
          }
          if (n < p.M) {
            if (p.lora == 2) {
#pragma unroll
              for (int t = 0; t < kDecBN; ++t)
                if (t < T) y[t] += lora_expand_term(t, n, __ldg(p.ids + t), p.tab, p.arena, p.g, p.v, T);
            }
#pragma unroll
            for (int t = 0; t < kDecBN; ++t)
              if (t < T) p.Y[(size_t)t * p.M + n] = __float2bfloat16_rn(y[t]);
          }
          if (etid == 0) p.cnt[c_first] = 0;  // re-arm for the next launch
        }
        ptx::named_bar_sync(1, 128);  // s_last reused by the next segment
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      u += kb1 - kb0;
    }
    if (etid == 0) DEC_TRACE(7);
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<32>(tmem_base);
}

}  // namespace bdl
