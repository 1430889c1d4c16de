// kernels_umma.cuh -- the base GEMM of both projection kinds (matmul_1 / matmul_2) on the 5th-gen
// tensor cores, with the LoRA expand + add (matmul_4/6, add_1/2) fused into its epilogue (sm_100a).
//
// Swap-AB formulation (decode-friendly): D[n, t] = sum_k W^T[n, k] X[t, k], i.e. the MMA's M dim runs
// over 128 output columns n (rows of W^T, K-major) and its N dim over BN tokens (X rows, K-major).
// T = 1 decode pads the token dim to 16 -- the MMA is ~free, the kernel is a TMA weight stream.
//
//   warp 0      : TMA producer   -- W tile [128 x 64] + X tile [BN x 64] per stage, SWIZZLE_128B,
//                                   W with L2 evict_first (read once), X evict_last (re-read)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer, double-buffered accumulator
//   warps 2..5  : epilogue       -- tcgen05.ld (thread = output column, registers = tokens),
//                                   + s_a v B[a] (fp32), one bf16 RNE rounding, store
//
// Work split: stream-K over units u = (token tile, 128-row tile, 64-wide k-block); CTA c owns
// [c U / G, (c+1) U / G) -- perfectly balanced over the G = #SM persistent CTAs for any shape.
// A tile split between CTAs is finished deterministically: every contributor writes its fp32
// partial, the CTA completing the tile's k-block count sums the partials in CTA order.
// The LoRA intermediate v is produced by the shrink kernel launched just before; with programmatic
// dependent launch the W stream of this kernel overlaps it and only the epilogue waits for it.
#pragma once
#include "common.cuh"
#include "kernels_route.cuh"
#include "ptx.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace bdl {

constexpr int kUmmaBM = 128;
constexpr int kUmmaBK = 64;
constexpr int kUmmaThreads = 192;
constexpr int kFuseMaxT = 256;
constexpr int kUmmaMaxGrid = 1024;
constexpr int kMaxDevices = 64;     // per-device caches of function attributes / occupancy answers  // bound of a splitting launch's grid (split-tile counters, workspace)  // fused shrink / LoRA prefetch handle decode-sized batches (ids staged in smem)

struct UmmaParams {
  int M, K, T;
  int rs_max;  // fused shrink: rank rows per slot capacity
  const __nv_bfloat16* X;
  int m_tiles, n_tiles, k_blocks;
  int units, grid;
  const int* ids;
  const SlotEntry* tab;
  const __nv_bfloat16* arena;
  Geom g;
  const float* v;
  __nv_bfloat16* Y;
  float* part;    // [grid][2][128][BN] fp32 split-tile partials (slot 0: a CTA's first segment, 1: last)
  int* tile_cnt;  // [kUmmaMaxGrid] split-tile arrival counters (by first contributor), zero between launches
  int pdl;
  int nstages;       // ring stages actually used (<= kStages): bounds the bytes in flight per SM
  int fuse;          // 1: the epilogue warps also compute v (fused shrink); 0: v comes from a prior kernel
  int tcx;           // 1: LoRA expand on the tensor cores (v split hi/lo bf16), accumulated in TMEM
  float* v_out;      // fused mode / shrink mode: v [T][J][Rc] written here
  const int* route;  // shrink mode: groups + 16-row A boxes from route_kernel (RouteLayout)
  int* sync;         // fused mode: [0] unit claim counter, [1] units done, [2] CTAs exited (zero between launches)
  long long* trace;  // optional per-CTA timestamps (ns, %globaltimer) for profiling; nullptr = off
  int local;         // fused mode: 0 = global shrink, 1 = K-local LoRA when the tile's adapters are few, 2 = always
  int cluster;       // > 1: launched with clusters of `cluster` split-K contributors of ONE tile (plain split-K
                     // grid, cluster = s); partials reduced through distributed shared memory, no global fix-up
};

// K-local LoRA (decode, one adapter group per token tile).  The layer is linear in a partition of K:
//   y_t = sum_seg [ X_t,seg W_seg + s_a (X_t,seg A_a,seg^T) B_a ]
// so a CTA owning the K-range of a tile segment adds its own share of the LoRA term to its (partial)
// accumulator.  The shrink rides the weight pipeline: every stage also carries a 16-row TMA box of the
// adapter's A rows, and the MMA warp accumulates v_seg = A_seg X_seg^T into a second TMEM accumulator
// (rows >= r/N of that MMA read unrelated shared memory and are ignored: MMA rows are independent).
// After the last k-block: v_seg (TMEM lanes 0..15) -> smem -> v_seg B on the CUDA cores (16 FMAs/token).
// No CTA waits for another's shrink (P:400-403 -- matmul_3/4 and matmul_5/6 regrouped over K).

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define UMMA_TRACE(slot)                                              \
  do {                                                                \
    if (p.trace) p.trace[(size_t)blockIdx.x * 32 + (slot)] = gtimer(); \
  } while (0)

__device__ __forceinline__ int umma_u_lo(long long c, int units, int grid) { return (int)(c * units / grid); }
__device__ __forceinline__ int umma_cta_of(long long u, int units, int grid) {
  // largest c with floor(c*U/G) <= u
  return (int)(((u + 1) * grid + units - 1) / units) - 1;
}

template <int BN>
struct UmmaSmem {
  static constexpr int kWBytes = kUmmaBM * kUmmaBK * 2;  // 16 KB
  static constexpr int kXBytes = BN * kUmmaBK * 2;
  static constexpr bool kHasA = (BN == 16);                 // decode: per-stage 16-row box of adapter A rows
  static constexpr int kABytes = kHasA ? 16 * kUmmaBK * 2 : 0;  // 2 KB
  static constexpr int kStageBytes = kWBytes + kXBytes + kABytes;
  static constexpr int kStages = (BN <= 16 ? 9 : BN <= 32 ? 9 : BN <= 64 ? 7 : BN <= 128 ? 5 : 4);
  static constexpr int kAccCols = kHasA ? 4 * BN : 2 * BN;    // [D0 D1 | V0 V1]: base + shrink accumulators
  static constexpr int kTmemCols = (kAccCols <= 32) ? 32 : (kAccCols <= 64) ? 64 : (kAccCols <= 128) ? 128 : (kAccCols <= 256) ? 256 : 512;
  static constexpr int kBarOff = kStages * kStageBytes;
  static constexpr int kVOff = kBarOff + 256 + 5120 + 512;          // after barriers/flags, ids/leaders/shrink
  static constexpr int kVFloats = 4096;                              // 16 KB v staging (CUDA-core expand)
  // tensor-core expand operands (share the region with the v staging): A = B-slab^T [128 x Kp],
  // V_hi / V_lo = bf16 split of v [BN x Kp], K-major, no-swizzle core-matrix layout
  static constexpr int kKp = BN <= 16 ? 64 : BN <= 128 ? 32 : 16;
  static constexpr int kLoraBufs = (BN >= 32 && BN <= 128) ? 2 : 1;  // double-buffered operands
  static constexpr int kLoraA = 128 * kKp * 2;
  static constexpr int kLoraV = BN * kKp * 2;
  static constexpr int kLoraBytes = kLoraA + 2 * kLoraV;
  static constexpr int kRegion = kLoraBufs * kLoraBytes > kVFloats * 4 ? kLoraBufs * kLoraBytes : kVFloats * 4;
  static constexpr int kMetaOff = kVOff + kRegion;                  // [BN][8] ints: leader re / offB (tc expand)
  // cluster split-K (decode): [s][ceil(128/s)][BN] fp32 partial slots pushed by the peers (dedicated: a peer
  // may push while this CTA still streams)
  static constexpr int kPartOff = kMetaOff + BN * 8 * 4;
  static constexpr int kPartBytes = kHasA ? (kUmmaBM + 8) * BN * 4 : 0;
  // tensor-core expand: the token tile's v rows staged once per segment (when they fit)
  static constexpr int kVStOff = kPartOff + kPartBytes;
  static constexpr int kVStBytes = BN == 64 ? 16384 : BN == 32 ? 12288 : 0;
  static constexpr int kPreBOff = kVStOff + kVStBytes;               // [16][128] fp32 pre-gathered B rows
  static constexpr int kPreBBytes = kHasA ? 16 * 128 * 4 : 0;
  static constexpr int kBytes = kPreBOff + kPreBBytes + 1024;        // + alignment slack
  // the shrink MMA reads 128 rows (16 KB) from a stage's A box: rows 16..127 must stay inside the allocation
  static_assert(kBytes <= 232448, "exceeds 227 KB of dynamic shared memory per CTA");
  static_assert(BN > 64 || kPartBytes > 0 || kStages * kWBytes >= (kUmmaBM + 8) * BN * 4,
                "cluster split-K slots must fit in the weight rings");
  static_assert(!kHasA || kStages * (kWBytes + kXBytes) + kStages * kABytes + 16384 <= kBytes - 1024,
                "shrink MMA window leaves the shared-memory allocation");
};

template <int BN, int MODE>
__global__ void __launch_bounds__(kUmmaThreads, 1)
    umma_lora_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                          const __grid_constant__ CUtensorMap tmA, const UmmaParams p) {
  using S = UmmaSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sW = smem;
  uint8_t* sX = smem + S::kStages * S::kWBytes;
  uint8_t* sA = sX + S::kStages * S::kXBytes;  // [kStages][16 x 64] adapter A rows (kHasA)
  // MODE 0: base GEMM + LoRA expand (v from a preceding shrink, tensor-core expand for T > 16);
  // MODE 2: the same GEMM as the single-kernel forward (grid-wide / K-local shrink inside) -- a separate
  // instantiation so each path gets its own register allocation and executed footprint; MODE 1: shrink.
  constexpr bool kGemm = MODE != 1;
  constexpr bool kDec = MODE == 2;
  constexpr bool kA = S::kHasA && kDec;
  uint64_t* full = (uint64_t*)(smem + S::kBarOff);
  uint64_t* empty = full + S::kStages;
  uint64_t* tfull = empty + S::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* lora_full = tempty + 2;   // [2] tensor-core expand: operands built (128 epilogue arrivals)
  uint64_t* lora_empty = lora_full + 2;  // [2] tensor-core expand: operand MMAs done (tcgen05.commit)
  uint32_t* tmem_holder = (uint32_t*)(lora_empty + 2);
  int* s_last = (int*)(tmem_holder + 1);
  int* s_ids = (int*)(smem + S::kBarOff + 256);  // [BN] adapter ids of the current token tile
  int* s_lead = s_ids + 256;                     // [BN] group leader of each token in its 16-chunk
  int* s_fids = s_lead + 256;                    // [T <= 256] all ids (fused shrink)
  int* s_mem = s_fids + 256;                     // [T] members of the current adapter group
  int* s_isl = s_mem + 256;                      // [T] 1 if the token is the first of its adapter id
  float* s_red = (float*)(s_isl + 256);          // [4][4] cross-warp partial dots
  int* s_misc = (int*)(s_red + 16);              // [0] claim [1] members [2..5] pass K/last per buffer [6] columns [8] K-local [12..15] scan
  int* s_pcol = s_misc + 16;                     // [2][8][6] tensor-core expand pass columns (a, j, k0, re, boff)
  int* s_gmeta = (int*)(smem + S::kMetaOff);     // [BN][8] per leader token: re, offB[0..2] (lo, hi)
  float* s_v = (float*)(smem + S::kVOff);        // [kVFloats] v rows of the current 16-token chunk
  float* s_preb = (float*)(smem + S::kPreBOff);  // decode: [16][128] B rows of each thread's column (parked)
  float* s_part = (float*)(smem + S::kPartOff);  // cluster split-K partial slots
  // cluster split-K partial slots: dedicated (decode) or the weight rings once every mainloop is done
  constexpr bool kSlotsInRing = S::kPartBytes == 0;
  float* s_slots = kSlotsInRing ? reinterpret_cast<float*>(sW) : s_part;
  float* s_vst = (float*)(smem + S::kVStOff);    // tensor-core expand: [C][tv][J][Rc] v of the token tile

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  // MODE 0: base GEMM (+ fused shrink / LoRA expand epilogue).  MODE 1: tensor-core shrink -- the
  // "weight" rows are 16-row boxes of adapter A rows listed by route_kernel, the output is v (fp32).
  int M_TILES = p.m_tiles, UNITS = p.units, GRID = p.grid, n_items = 0;
  if constexpr (MODE == 1) {
    ptx::pdl_wait();  // the route kernel (preceding) produced the item list
    n_items = p.route[RouteLayout::kHdr + 1];
    M_TILES = (n_items + 7) / 8;
    UNITS = M_TILES * p.n_tiles * p.k_blocks;
    // split-K contributors add their share of v with fp32 reductions (no fix-up round trip); >= 8
    // k-blocks per CTA
    GRID = max(1, min((int)gridDim.x, UNITS / 8));
  }
  const bool active = cta < GRID && UNITS > 0;
  const int u_lo = active ? umma_u_lo(cta, UNITS, GRID) : 0;
  const int u_hi = active ? umma_u_lo(cta + 1, UNITS, GRID) : 0;
  if (threadIdx.x == 0) UMMA_TRACE(0);

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmW);
    ptx::tma_prefetch_desc(&tmX);
    if (kA) ptx::tma_prefetch_desc(&tmA);
    for (int s = 0; s < S::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(lora_full + b, 128);
      ptx::mbar_init(lora_empty + b, 1);
    }
    ptx::fence_mbar_init();
    ptx::fence_proxy_async();
  }
  if (warp == 1) ptx::tmem_alloc<S::kTmemCols>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // Cluster split-K with dedicated partial slots: a CTA pushes into a peer's shared memory, which is only
  // legal once the peer has started -- every thread arrives on the cluster barrier now and waits before its
  // first DSMEM access (the ring-slot variant gets this from its post-mainloop cluster barrier).
  const bool early_cl = kGemm && !kSlotsInRing && p.cluster > 1;
  bool cl_pending = early_cl;
  if (early_cl) ptx::cluster_arrive_relaxed();
  if (threadIdx.x == 0) {
    UMMA_TRACE(1);
    // dependents (the next kernel) may launch now: they wait for this grid's completion before
    // touching anything it writes, and can only take SMs this grid has released.
    ptx::pdl_launch_dependents();
  }

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Weights never depend on the preceding kernel: the first ring of W tiles is issued BEFORE the
    // programmatic-dependency wait (overlapping the previous kernel's tail), activations after it.
    if (MODE == 1 && ptx::elect_one()) {
      // shrink: up to 8 boxes of 16 A rows per 128-row tile (rows of different adapters / slices)
      const uint64_t pol_a = ptx::policy_evict_first();
      const uint64_t pol_x = ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int cur_mt = -1, nbox = 0;
      int rows[8];
      for (int u = u_lo; u < u_hi; ++u) {
        const int tile = u / p.k_blocks, kb = u - tile * p.k_blocks;
        const int mt = tile % M_TILES, nt = tile / M_TILES;
        if (mt != cur_mt) {
          cur_mt = mt;
          nbox = min(8, n_items - mt * 8);
#pragma unroll
          for (int b = 0; b < 8; ++b) rows[b] = (b < nbox) ? p.route[RouteLayout::kItemRow + mt * 8 + b] : 0;
        }
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], nbox * 2048 + S::kXBytes);
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (b < nbox)
            ptx::tma_load_2d(sW + stage * S::kWBytes + b * 2048, &tmW, &full[stage], kb * kUmmaBK, rows[b], pol_a);
        ptx::tma_load_2d(sX + stage * S::kXBytes, &tmX, &full[stage], kb * kUmmaBK, nt * BN, pol_x);
        if (++stage == p.nstages) {
          stage = 0;
          phase ^= 1;
        }
      }
    } else if (kGemm && ptx::elect_one()) {
      const uint64_t pol_w = ptx::policy_evict_first();
      const uint64_t pol_x = ptx::policy_evict_last();
      const int nu = u_hi - u_lo;
      const int NS = p.nstages;
      const int P = min(nu, NS);
      for (int idx = 0; idx < P; ++idx) {  // expect (no arrival yet): the stage cannot complete before X/A
        const int u = u_lo + idx, tile = u / p.k_blocks, kb = u - tile * p.k_blocks, mt = tile % M_TILES;
        ptx::mbar_expect_tx(&full[idx], S::kWBytes);
        ptx::tma_load_2d(sW + idx * S::kWBytes, &tmW, &full[idx], kb * kUmmaBK, mt * kUmmaBM, pol_w);
      }
      if (nu > 0) UMMA_TRACE(2);
      if (p.pdl) ptx::pdl_wait();
      // K-local LoRA: A rows (arena row index per slice) of the token tile's single adapter, loaded only when
      // the K-local schedule is taken (same decision as the epilogue's, see `local`; the MMA warp reads it
      // from s_misc[8], written before the first arrival on full[0])
      int arow[kMaxSlices] = {0, 0, 0};
      bool use_a = false;
      if constexpr (kA) {
        if (p.local && p.T <= 16 && p.g.C == 1) {
          int a = -1;
          bool single = true;
          for (int t = 0; t < p.T; ++t) {
            const int id = __ldg(p.ids + t);
            if (id >= 0) {
              if (a < 0) a = id;
              else if (id != a) single = false;
            }
          }
          if (single && a >= 0 && p.tab[a].rs <= 16) {
            use_a = true;
            for (int j = 0; j < p.g.J; ++j) arow[j] = (int)(p.tab[a].offA[j] / p.K);
          }
        }
      }
      s_misc[8] = use_a ? 1 : 0;
      const uint32_t a_bytes = use_a ? (uint32_t)S::kABytes : 0u;
      auto load_a = [&](int st, int mt, int kb) {
        if (kA && use_a) {
          int jt = 0;
          for (int q2 = 1; q2 < p.g.J; ++q2)
            if (mt * kUmmaBM >= p.g.col0[q2]) jt = q2;
          ptx::tma_load_2d(sA + st * S::kABytes, &tmA, &full[st], kb * kUmmaBK, arow[jt], pol_x);
        }
      };
      for (int idx = 0; idx < P; ++idx) {
        const int u = u_lo + idx, tile = u / p.k_blocks, kb = u - tile * p.k_blocks, nt = tile / M_TILES;
        ptx::mbar_arrive_expect_tx(&full[idx], S::kXBytes + a_bytes);
        ptx::tma_load_2d(sX + idx * S::kXBytes, &tmX, &full[idx], kb * kUmmaBK, nt * BN, pol_x);
        load_a(idx, tile % M_TILES, kb);
      }
      int stage = (P == NS) ? 0 : P;
      uint32_t phase = (P == NS) ? 1u : 0u;
      for (int idx = P; idx < nu; ++idx) {
        const int u = u_lo + idx, tile = u / p.k_blocks, kb = u - tile * p.k_blocks;
        const int mt = tile % M_TILES, nt = tile / M_TILES;
        ptx::mbar_wait(&empty[stage], phase ^ 1);
        ptx::mbar_arrive_expect_tx(&full[stage], S::kWBytes + S::kXBytes + a_bytes);
        ptx::tma_load_2d(sW + stage * S::kWBytes, &tmW, &full[stage], kb * kUmmaBK, mt * kUmmaBM, pol_w);
        ptx::tma_load_2d(sX + stage * S::kXBytes, &tmX, &full[stage], kb * kUmmaBK, nt * BN, pol_x);
        load_a(stage, mt, kb);
        if (++stage == p.nstages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(kUmmaBM, BN);
      constexpr uint32_t idesc_lora = idesc | (1u << 15);  // A operand MN-major
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int lbuf = 0;                    // tensor-core expand: next operand buffer
      uint32_t lf_phase[2] = {0u, 0u};  // its mbarrier parity
      for (int u = u_lo; u < u_hi;) {
        const int tile = u / p.k_blocks;
        const int kb0 = u - tile * p.k_blocks;
        const int kb1 = min(p.k_blocks, kb0 + (u_hi - u));
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        // LoRA expand passes (every contributor of the tile takes its share, possibly one empty "last" pass):
        // issued as soon as the epilogue warps have built them, interleaved with the base k-blocks
        // (accumulation order is free in fp32), so the operand gathers overlap the weight stream
        const bool lduty = kGemm && !kDec && p.tcx;
        bool ldone = !lduty;
        auto lora_pass = [&]() {
          constexpr uint32_t kSbo = (S::kKp / 8) * 128;  // V: 8-row group stride
          const int b = lbuf;
          const uint32_t la0 = ptx::smem_u32(smem + S::kVOff + b * S::kLoraBytes);
          const uint32_t vh0 = la0 + S::kLoraA, vl0 = vh0 + S::kLoraV;
          lf_phase[b] ^= 1u;
          lbuf = (lbuf + 1) % S::kLoraBufs;
          ptx::tc_fence_after();
          const int kp = s_misc[2 + 2 * b], last = s_misc[3 + 2 * b];
          for (int kk = 0; kk < kp / 16; ++kk) {  // A is MN-major (idesc_lora), V K-major
            const uint64_t ad = ptx::sdesc_k_none(la0 + kk * 4096, /*LBO: k-group*/ 2048, /*SBO: n-group*/ 128);
            ptx::mma_bf16(d_tmem, ad, ptx::sdesc_k_none(vh0 + kk * 256, 128, kSbo), idesc_lora, 1u);
            ptx::mma_bf16(d_tmem, ad, ptx::sdesc_k_none(vl0 + kk * 256, 128, kSbo), idesc_lora, 1u);
          }
          ptx::mma_commit(lora_empty + b);
          if (last) ldone = true;
        };
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (u == u_lo && kb == kb0) UMMA_TRACE(3);
          const uint64_t a_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sW + stage * S::kWBytes));
          const uint64_t b_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sX + stage * S::kXBytes));
#pragma unroll
          for (int k = 0; k < kUmmaBK / 16; ++k)  // UMMA_K = 16 bf16 = 32 B -> +2 in the >>4 address field
            ptx::mma_bf16(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          if (kA && s_misc[8]) {  // K-local shrink: V[k][t] += A_a[k][kb] . X[t][kb] (rows >= 16 ignored)
            const uint64_t s_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sA + stage * S::kABytes));
            const uint32_t v_tmem = tmem_base + (uint32_t)(2 * BN + acc * BN);
#pragma unroll
            for (int k = 0; k < kUmmaBK / 16; ++k)
              ptx::mma_bf16(v_tmem, s_desc + 2 * k, b_desc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          ptx::mma_commit(&empty[stage]);
          if (++stage == p.nstages) {
            stage = 0;
            phase ^= 1;
          }
          if (!ldone && ptx::mbar_test(lora_full + lbuf, lf_phase[lbuf])) lora_pass();  // D initialised (kb0 done)
        }
        while (!ldone) {
          ptx::mbar_wait(lora_full + lbuf, lf_phase[lbuf]);
          lora_pass();
        }
        ptx::mma_commit(&tfull[acc]);
        UMMA_TRACE(4);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        u += kb1 - kb0;
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    if constexpr (kGemm) {
    const int q = warp & 3;  // TMEM lane quarter accessible by this warp
    const int row = q * 32 + lane;
    const int etid = threadIdx.x - 64;  // 0..127
    const int crank = p.cluster > 1 ? (int)ptx::cluster_ctarank() : 0;
    if (p.pdl) ptx::pdl_wait();         // the preceding kernel is complete and visible (X, ids, and v
                                        // when it was a shrink); also orders our Y writes after it
    if (p.fuse && etid == 0) s_misc[0] = atomicAdd(p.sync + 0, 1);  // fused-shrink arrival ticket (below)
    if (p.T <= kFuseMaxT) {
      // ---- L2 prefetch of the LoRA data this launch gathers (tiny, latency-critical): issued now, at the
      // start of the weight stream, so the shrink's A rows and the expand's B rows hit L2 later ----------
      for (int t = etid; t < p.T; t += 128) s_fids[t] = __ldg(p.ids + t);
      ptx::named_bar_sync(1, 128);
      for (int t = etid; t < p.T; t += 128) {  // leader = first token of its adapter id (parallel, O(T^2/128))
        const int a = s_fids[t];
        bool f = a >= 0;
        for (int t2 = 0; t2 < t && f; ++t2) f = (s_fids[t2] != a);
        s_isl[t] = f ? 1 : 0;
      }
      ptx::named_bar_sync(1, 128);
      const int mt_a = (u_lo / p.k_blocks) % M_TILES;
      const int mt_b = ((u_hi - 1) / p.k_blocks) % M_TILES;
      // one thread per distinct adapter: its slot entry is read once (all threads' reads in flight together,
      // not one dependent round trip per adapter), then the prefetches are fire-and-forget
      for (int t = etid; t < p.T; t += 128) {
        if (!s_isl[t]) continue;
        const SlotEntry e = p.tab[s_fids[t]];
        for (int mt = mt_a; mt <= mt_b; ++mt) {  // B rows of my output columns
          const int n0 = mt * kUmmaBM;
          for (int jj = 0; jj < p.g.J; ++jj) {
            const int lo = max(n0, p.g.e_lo[jj]), hi = min(n0 + kUmmaBM, p.g.e_hi[jj]);
            if (lo >= hi) continue;
            const int ldb = p.g.e_hi[jj] - p.g.e_lo[jj];
            for (int k = 0; k < e.re; ++k)
              ptx::prefetch_l2_bulk(p.arena + e.offB[jj] + (size_t)k * ldb + (lo - p.g.e_lo[jj]), (hi - lo) * 2);
          }
        }
      }
    }
    // K-local LoRA decision: uniform over the grid (every CTA sees the same ids; T <= 16 = one token tile)
    // and identical to the producer's: one adapter group (or none) with r/N <= 16
    bool local = false;
    int la = -1;
    if constexpr (kA) {
      if (p.fuse && p.local && p.T <= 16 && p.g.C == 1) {
        bool single = true;
        for (int t = 0; t < p.T; ++t) {
          const int id = s_fids[t];
          if (id >= 0) {
            if (la < 0) la = id;
            else if (id != la) single = false;
          }
        }
        local = single && (la < 0 || p.tab[la].rs <= 16);
      }
    }
    const int la_rs = (local && la >= 0) ? p.tab[la].rs : 0;  // loaded once, early (off the tail)
    const float la_sc = (local && la >= 0) ? p.tab[la].scale : 0.f;
    int cur_nt = -1;
    LoraPre pre;
    pre.a = -1;
    pre.sb = S::kHasA ? s_preb + etid : nullptr;  // decode: B rows live in shared memory, not registers
    if (kDec && p.fuse && !local) {
      // ---- fused shrink (matmul_3 / matmul_5): v[t][j][k] = s_a sum_d X[t][d] A_{a,j}[k][d] -----------
      // Units (leader token t, slice j, rank row k) are computed by the epilogue warps while the
      // producer/MMA warps stream W; a unit is computed once per DISTINCT adapter (leader = first token
      // with that id) for all its tokens.
      const int Js = p.g.J, rsm = p.rs_max;
      const int U_s = p.T * Js * rsm;
      const int warp_e = etid >> 5;
      // units are claimed in batches b = {b, b + G, b + 2G, ...} (G = gridDim.x): a CTA's first batch is its
      // arrival ticket (one atomic per CTA when every CTA is resident); whoever finishes a batch claims the next
      // unclaimed one, so every unit is computed by a RESIDENT CTA whatever the residency (clusters may not
      // all fit in one wave) -- no CTA can wait for v that a not-yet-resident CTA owns
      ptx::named_bar_sync(1, 128);
      int batch = s_misc[0];
      int mine = 0;
      const int n_batches = min((int)gridDim.x, U_s);
      while (batch < n_batches) {
      for (int us = batch; us < U_s; us += (int)gridDim.x) {
        ++mine;
        const int t_lead = us / (Js * rsm), j = (us / rsm) % Js, k = us % rsm;
        const int a = s_fids[t_lead];
        const bool leader = s_isl[t_lead] != 0;
        const SlotEntry* e = leader ? p.tab + a : nullptr;
        if (leader && k < e->rs) {
          if (warp_e == 0) {  // members of this adapter group, token order
            int cnt = 0;
            for (int base = t_lead; base < p.T; base += 32) {
              const int t2 = base + lane;
              const unsigned m = __ballot_sync(0xffffffffu, t2 < p.T && s_fids[t2] == a);
              if (t2 < p.T && s_fids[t2] == a) s_mem[cnt + __popc(m & ((1u << lane) - 1u))] = t2;
              cnt += __popc(m);
            }
            if (lane == 0) s_misc[1] = cnt;
          }
          ptx::named_bar_sync(1, 128);
          const int cnt = s_misc[1];
          const __nv_bfloat16* Ar = p.arena + e->offA[j] + (size_t)k * p.K;
          for (int m0 = 0; m0 < cnt; m0 += 4) {
            float acc4[4] = {0.f, 0.f, 0.f, 0.f};
            int tok[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) tok[m] = (m0 + m < cnt) ? s_mem[m0 + m] : -1;
#pragma unroll 4
            for (int d = etid * 8; d < p.K; d += 128 * 8) {
              float af[8];
              bf16x8_to_f32(ld_cached_u4(Ar + d), af);
#pragma unroll
              for (int m = 0; m < 4; ++m) {
                if (tok[m] >= 0) {
                  float xf[8];
                  bf16x8_to_f32(ld_cached_u4(p.X + (size_t)tok[m] * p.K + d), xf);
#pragma unroll
                  for (int q2 = 0; q2 < 8; ++q2) acc4[m] = fmaf(af[q2], xf[q2], acc4[m]);
                }
              }
            }
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const float sm = warp_sum(acc4[m]);
              if (lane == 0) s_red[warp_e * 4 + m] = sm;
            }
            ptx::named_bar_sync(1, 128);
            if (etid < 4 && tok[etid & 3] >= 0) {
              const int m = etid;
              const float sm = (s_red[m] + s_red[4 + m]) + (s_red[8 + m] + s_red[12 + m]);
              p.v_out[((size_t)s_mem[m0 + m] * Js + j) * p.g.Rc + k] = e->scale * sm;
            }
            ptx::named_bar_sync(1, 128);
          }
        }
      }
        ptx::named_bar_sync(1, 128);  // s_misc / s_mem of this batch no longer read
        if (etid == 0) s_misc[0] = atomicAdd(p.sync + 0, 1);
        ptx::named_bar_sync(1, 128);
        batch = s_misc[0];
      }
      ptx::named_bar_sync(1, 128);
      if (etid == 0 && mine) ptx::atom_add_acq_rel_gpu(p.sync + 1, mine);  // publishes my v (release)
    }
    // ---- first segment: stage its token tile's ids and gather its B rows now (before v is needed) ----
    if (p.T <= kFuseMaxT && u_lo < u_hi) {
      const int tile = u_lo / p.k_blocks, mt = tile % M_TILES, nt = tile / M_TILES;
      const int t0 = nt * BN, tv = min(BN, p.T - t0);
      for (int i = etid; i < tv; i += 128) s_ids[i] = s_fids[t0 + i];
      ptx::named_bar_sync(1, 128);
      for (int i = etid; i < tv; i += 128) {
        const int cb = i & ~15, a = s_ids[i];
        int lead = -1;
        if (a >= 0) {
          lead = i - cb;
          for (int i2 = cb; i2 < i; ++i2)
            if (s_ids[i2] == a) {
              lead = i2 - cb;
              break;
            }
        }
        s_lead[i] = lead;
        if (!kDec && p.tcx) {  // leader within the whole token tile (tensor-core expand groups) + its slot metadata
          bool f = a >= 0;
          for (int i2 = 0; i2 < i && f; ++i2) f = (s_ids[i2] != a);
          s_mem[i] = f ? 1 : 0;
          if (f) {
            int* gm = s_gmeta + i * 8;
            gm[0] = p.tab[a].re;
#pragma unroll
            for (int jj = 0; jj < kMaxSlices; ++jj) {
              const long long ob = p.tab[a].offB[jj];
              gm[1 + 2 * jj] = (int)(ob & 0xffffffff);
              gm[2 + 2 * jj] = (int)(ob >> 32);
            }
          }
        }
      }
      ptx::named_bar_sync(1, 128);
      cur_nt = nt;
      if (!p.tcx) lora_pre16(pre, mt * kUmmaBM + row, min(16, tv), s_ids, s_lead, p.tab, p.arena, p.g);

    }
    if (kDec && p.fuse && !local) {
      // every unit of the launch published before any expand reads v
      if (etid == 0) {
        UMMA_TRACE(13);
        while (ptx::ld_acquire_gpu(p.sync + 1) < p.T * p.g.J * p.rs_max) __nanosleep(64);
        UMMA_TRACE(14);
      }
      ptx::named_bar_sync(1, 128);
    }
    int acc = 0;
    uint32_t acc_phase = 0;
    bool first_seg = true;
    int pre_n = -1;
    int lp = 0;  // tensor-core expand passes built so far (buffer = lp % kLoraBufs)
    for (int u = u_lo; u < u_hi;) {
      const int tile = u / p.k_blocks;
      const int kb0 = u - tile * p.k_blocks;
      const int kb1 = min(p.k_blocks, kb0 + (u_hi - u));
      const int mt = tile % M_TILES, nt = tile / M_TILES;
      const int n = mt * kUmmaBM + row;
      const int t0 = nt * BN;
      const int tv = min(BN, p.T - t0);
      const bool whole = (kb0 == 0 && kb1 == p.k_blocks);
      const int slot = (tile * p.k_blocks > u_lo) ? 1 : 0;
      float* my_part = p.part + ((size_t)(cta * 2 + slot) * kUmmaBM + row) * BN;
      if (nt != cur_nt) {  // stage this token tile's adapter ids
        ptx::named_bar_sync(1, 128);
        for (int i = etid; i < tv; i += 128) s_ids[i] = (p.T <= kFuseMaxT) ? s_fids[t0 + i] : __ldg(p.ids + t0 + i);
        ptx::named_bar_sync(1, 128);
        for (int i = etid; i < tv; i += 128) {  // group leader within the token's 16-chunk
          const int cb = i & ~15, a = s_ids[i];
          int lead = -1;
          if (a >= 0) {
            lead = i - cb;
            for (int i2 = cb; i2 < i; ++i2)
              if (s_ids[i2] == a) {
                lead = i2 - cb;
                break;
              }
          }
          s_lead[i] = lead;
          if (!kDec && p.tcx) {  // leader within the whole token tile (tensor-core expand groups) + its slot metadata
            bool f = a >= 0;
            for (int i2 = 0; i2 < i && f; ++i2) f = (s_ids[i2] != a);
            s_mem[i] = f ? 1 : 0;
            if (f) {
              int* gm = s_gmeta + i * 8;
              gm[0] = p.tab[a].re;
#pragma unroll
              for (int jj = 0; jj < kMaxSlices; ++jj) {
                const long long ob = p.tab[a].offB[jj];
                gm[1 + 2 * jj] = (int)(ob & 0xffffffff);
                gm[2 + 2 * jj] = (int)(ob >> 32);
              }
            }
          }
        }
        ptx::named_bar_sync(1, 128);
        cur_nt = nt;
      }
      if (!kDec && p.tcx) {
        // ---- tensor-core expand: this CTA's share of the tile's LoRA columns, built while weights stream ----
        // The tile's rank columns (leader i, slice j in [jlo, jhi], 8-row block) are numbered in (i, j, block)
        // order through a parallel prefix over the tile's adapter groups; passes of KC columns are dealt
        // round-robin to the tile's split contributors (the LoRA term is linear: every contributor adds its
        // share into its own accumulator/partial).  Per pass: A[n][k] = B_{a,j}[k][n] (cp.async gathers of
        // 16 contiguous bytes of a B row) and V[t][k] = v[t][j][k] split into bf16 hi + lo; the MMA warp adds
        // A.V_hi^T + A.V_lo^T into the TMEM accumulator.  Operands are double-buffered: pass p+1 is gathered
        // while the tensor cores consume pass p.
        const int n0 = mt * kUmmaBM;
        int jlo = 0, jhi = 0;
        for (int q2 = 1; q2 < p.g.J; ++q2) {
          if (n0 >= p.g.col0[q2]) jlo = q2;
          if (min(n0 + kUmmaBM - 1, p.g.M - 1) >= p.g.col0[q2]) jhi = q2;
        }
        constexpr int KC = S::kKp / 8;  // core-matrix columns (8 rank rows each) per pass
        // exclusive prefix of column counts over the tile's tokens -> s_gmeta[i * 8 + 7]; total in s_misc[6]
        {
          const int nsl = jhi - jlo + 1;
          int c0v = 0, c1v = 0;
          const int i0 = 2 * etid, i1 = 2 * etid + 1;
          if (i0 < tv && s_mem[i0]) c0v = nsl * ((s_gmeta[i0 * 8] + 7) / 8);
          if (i1 < tv && s_mem[i1]) c1v = nsl * ((s_gmeta[i1 * 8] + 7) / 8);
          int incl = c0v + c1v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          const int we = etid >> 5;
          if (lane == 31) s_misc[12 + we] = incl;
          ptx::named_bar_sync(1, 128);
          int woff = 0;
          for (int w2 = 0; w2 < we; ++w2) woff += s_misc[12 + w2];
          const int ex = woff + incl - (c0v + c1v);
          if (i0 < tv) s_gmeta[i0 * 8 + 7] = ex;
          if (i1 < tv) s_gmeta[i1 * 8 + 7] = ex + c0v;
          if (etid == 127) s_misc[6] = woff + incl;
          ptx::named_bar_sync(1, 128);
        }
        const int c_tot = s_misc[6];
        // v rows of this token tile -> shared memory in one round trip (the passes then build V from smem)
        const int per_c = tv * p.g.J * p.g.Rc;
        const bool vst = c_tot > 0 && per_c * p.g.C * 4 <= S::kVStBytes;
        if (vst) {
          for (int idx = etid; idx < per_c * p.g.C; idx += 128) {
            const int ch = idx / per_c, r2 = idx - ch * per_c;
            s_vst[idx] = __ldg(p.v + (size_t)(ch * p.T + t0) * p.g.J * p.g.Rc + r2);
          }
          ptx::named_bar_sync(1, 128);
        }
        const float* vb = vst ? s_vst : p.v + (size_t)t0 * p.g.J * p.g.Rc;  // token t of the tile at vb[t*J*Rc]
        const int vT = vst ? tv : p.T;                                      // chunk stride in tokens
        if (etid == 0 && lp == 0) UMMA_TRACE(19);
        const int npass = (c_tot + KC - 1) / KC;
        const int ts = tile * p.k_blocks;
        const int c_first = umma_cta_of(ts, UNITS, GRID);
        const int cs = umma_cta_of(ts + p.k_blocks - 1, UNITS, GRID) - c_first + 1, ci = cta - c_first;
        const int my_n = max(1, npass > ci ? (npass - ci + cs - 1) / cs : 0);  // >= 1: an empty "last" pass
        for (int m = 0; m < my_n; ++m) {
          const int pp = ci + m * cs;
          const int b = lp % S::kLoraBufs;
          const uint32_t par = (uint32_t)(lp / S::kLoraBufs) & 1u;
          int* pcb = s_pcol + b * 48;
          uint8_t* la = smem + S::kVOff + b * S::kLoraBytes;
          uint8_t* lvh = la + S::kLoraA;
          uint8_t* lvl = lvh + S::kLoraV;
          if (etid < KC) {  // column metadata: owning leader by binary search over the prefix
            const int q = pp * KC + etid;
            int* pc = pcb + etid * 6;
            if (q < c_tot) {
              int lo = 0, hi = tv - 1;
              while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_gmeta[mid * 8 + 7] <= q) lo = mid;
                else hi = mid - 1;
              }
              const int* gm = s_gmeta + lo * 8;
              const int re = gm[0], nb = (re + 7) / 8, rem = q - gm[7];
              const int cj = jlo + rem / nb;
              pc[0] = s_ids[lo], pc[1] = cj, pc[2] = (rem % nb) * 8, pc[3] = re, pc[4] = gm[1 + 2 * cj],
              pc[5] = gm[2 + 2 * cj];
            } else {
              pc[0] = -2, pc[1] = 0, pc[2] = 0, pc[3] = 0, pc[4] = 0, pc[5] = 0;
            }
          }
          ptx::named_bar_sync(1, 128);
          if (etid == 0 && lp < 2) UMMA_TRACE(20 + 4 * lp);
          ptx::mbar_wait(lora_empty + b, par ^ 1u);  // the MMAs of this buffer's previous pass are done
          if (etid == 0 && lp < 2) UMMA_TRACE(21 + 4 * lp);
          // A = B-slab^T in the MN-major no-swizzle layout: a 16-byte chunk is 8 consecutive output columns
          // of one rank row k -- exactly 16 contiguous bytes of B's row k (core matrix (n-group, k-group)
          // at (kg * 16 + ng) * 128, row k % 8)
#pragma unroll
          for (int it = 0; it < S::kKp * 16 / 128; ++it) {
            const int idx = etid + it * 128;
            const int kr = idx >> 4, ng = idx & 15, c = kr >> 3;
            const int* pc = pcb + c * 6;
            uint8_t* dst = la + ((kr >> 3) * 16 + ng) * 128 + (kr & 7) * 16;
            const int k = pc[2] + (kr & 7);
            bool zero = true;
            if (k < pc[3]) {
              const int cjj = pc[1];
              const int lo = p.g.e_lo[cjj], hi = min(p.g.e_hi[cjj], p.g.M), ldb = p.g.e_hi[cjj] - lo;
              const int nlo = n0 + ng * 8;
              const long long boff = (long long)(unsigned)pc[4] | ((long long)pc[5] << 32);
              const uint16_t* Brow = reinterpret_cast<const uint16_t*>(p.arena + boff) + (size_t)k * ldb;
              if (nlo >= lo && nlo + 8 <= hi && (((uintptr_t)(Brow + (nlo - lo))) & 15) == 0) {
                ptx::cp_async_16(dst, Brow + (nlo - lo));
                zero = false;
              } else if (nlo + 8 > lo && nlo < hi) {
                uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                for (int e2 = 0; e2 < 8; ++e2) {
                  const int nn = nlo + e2;
                  const uint32_t h = (nn >= lo && nn < hi) ? (uint32_t)__ldg(Brow + (nn - lo)) : 0u;
                  w[e2 >> 1] |= h << ((e2 & 1) * 16);
                }
                *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
                zero = false;
              }
            }
            if (zero) *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
          }
          if (etid == 0 && lp == 0) UMMA_TRACE(28);
          // V_hi / V_lo: (token, column) pairs over the 128 threads
#pragma unroll
          for (int it = 0; it < (BN * KC + 127) / 128; ++it) {
            const int idx = etid + it * 128;
            if (idx >= BN * KC) break;
            const int t = idx / KC, c = idx - t * KC;
            const int* pc = pcb + c * 6;
            float f[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (t < tv && s_ids[t] == pc[0]) {
              const int cjj = pc[1], ck = pc[2], re = pc[3], rcc = re / p.g.C;
              const float* vrow = vb + ((size_t)t * p.g.J + cjj) * p.g.Rc + ck;
              if (p.g.C == 1 && ck + 8 <= re && (p.g.Rc & 3) == 0) {
                const float4 f0 = *reinterpret_cast<const float4*>(vrow);
                const float4 f1 = *reinterpret_cast<const float4*>(vrow + 4);
                f[0] = f0.x, f[1] = f0.y, f[2] = f0.z, f[3] = f0.w, f[4] = f1.x, f[5] = f1.y, f[6] = f1.z, f[7] = f1.w;
              } else {
#pragma unroll
                for (int q2 = 0; q2 < 8; ++q2) {
                  const int k = ck + q2;
                  if (k < re) {
                    const int ch = k / rcc, kk = k - ch * rcc;
                    f[q2] = vb[((size_t)(ch * vT + t) * p.g.J + cjj) * p.g.Rc + kk];
                  }
                }
              }
            }
            uint32_t h4[4], l4[4];
#pragma unroll
            for (int q2 = 0; q2 < 8; q2 += 2) {
              const __nv_bfloat16 h0 = __float2bfloat16_rn(f[q2]), h1 = __float2bfloat16_rn(f[q2 + 1]);
              const __nv_bfloat16 l0 = __float2bfloat16_rn(f[q2] - __bfloat162float(h0));
              const __nv_bfloat16 l1 = __float2bfloat16_rn(f[q2 + 1] - __bfloat162float(h1));
              h4[q2 / 2] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
              l4[q2 / 2] = (uint32_t)__bfloat16_as_ushort(l0) | ((uint32_t)__bfloat16_as_ushort(l1) << 16);
            }
            const int off = ((t >> 3) * KC + c) * 128 + (t & 7) * 16;
            *reinterpret_cast<uint4*>(lvh + off) = make_uint4(h4[0], h4[1], h4[2], h4[3]);
            *reinterpret_cast<uint4*>(lvl + off) = make_uint4(l4[0], l4[1], l4[2], l4[3]);
          }
          if (etid == 0 && lp < 2) UMMA_TRACE(22 + 4 * lp);
          ptx::cp_async_wait_all();
          ptx::fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor cores
          if (etid == 0 && lp < 2) UMMA_TRACE(23 + 4 * lp);
          if (etid == 0) {
            const int nvalid = max(0, min(KC, c_tot - pp * KC));
            s_misc[2 + 2 * b] = ((nvalid * 8 + 15) / 16) * 16;
            s_misc[3 + 2 * b] = (m == my_n - 1) ? 1 : 0;
          }
          ptx::mbar_arrive(lora_full + b);
          ++lp;
        }
      }
      // LoRA term of the first 16 tokens on CUDA cores (when not on the tensor cores), gathered BEFORE
      // waiting for the accumulator so it overlaps this tile's mainloop.
      float lr[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) lr[i] = 0.f;
      if (!first_seg && n != pre_n) pre.a = -1;  // cached B rows belong to another output column
      pre_n = n;
      if (local) {
        // B rows of this thread's output column (the single adapter): gathered now, used after the stream
        if (la >= 0 && pre.a != la) lora_pre16(pre, n, min(16, tv), s_ids, s_lead, p.tab, p.arena, p.g);
      } else if (!p.tcx) {
        lora_chunk16(lr, n, t0, min(16, tv), s_ids, s_lead, p.tab, p.arena, p.g, p.v, p.T, &pre, s_v, S::kVFloats,
                     etid, (p.trace && first_seg) ? p.trace + (size_t)blockIdx.x * 32 : nullptr);
      }
      if (first_seg && etid == 0) UMMA_TRACE(15);
      const bool was_first = first_seg;
      first_seg = false;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      if (etid == 0) {
        if (u == u_lo) UMMA_TRACE(5);
        UMMA_TRACE(6);
      }
      if (cl_pending && !whole) {  // peers have started: DSMEM pushes below are legal
        ptx::cluster_wait();
        cl_pending = false;
      }
      if (kSlotsInRing && !whole && p.cluster > 1) {
        // the partial slots live in the (then idle) weight rings: wait until every contributor of the
        // tile has finished its mainloop before anyone pushes
        ptx::cluster_arrive();
        ptx::cluster_wait();
      }
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      if (local && la >= 0) {
        // this segment's v_seg: TMEM lanes k < r/N of the shrink accumulator (warp of lane quarter 0) -> smem
        if constexpr (kA) {
          ptx::named_bar_sync(1, 128);  // previous readers of s_v are done
          if (q == 0) {
            uint32_t r2[16];
            ptx::tmem_ld_32x32b_x16(tmem_base + (uint32_t)(2 * BN + acc * BN), r2);
            ptx::tmem_ld_wait();
            if (lane < la_rs) {
#pragma unroll
              for (int i = 0; i < 16; ++i) s_v[i * 16 + lane] = la_sc * __uint_as_float(r2[i]);
            }
          }
          ptx::named_bar_sync(1, 128);
          if (etid == 0 && was_first) UMMA_TRACE(16);
          // lr[t] = v_seg[t] . B[:, n] for the adapter's tokens (pre.b[k] = 0 for k >= r/N)
          if (pre.a == la) {
            const int rs = la_rs;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float s0 = 0.f, s1 = 0.f;
              if (i < tv && s_ids[i] == la) {
#pragma unroll
                for (int k = 0; k < 16; k += 2) {
                  s0 = fmaf(k < rs ? s_v[i * 16 + k] : 0.f, s_preb[k * 128 + etid], s0);
                  s1 = fmaf(k + 1 < rs ? s_v[i * 16 + k + 1] : 0.f, s_preb[(k + 1) * 128 + etid], s1);
                }
              }
              lr[i] = s0 + s1;
            }
          }
          if (etid == 0 && was_first) UMMA_TRACE(17);
        }
      }
      for (int c0 = 0; c0 < tv; c0 += 16) {
        uint32_t r[16];
        ptx::tmem_ld_32x32b_x16(taddr + c0, r);
        ptx::tmem_ld_wait();
        if (whole) {
          if (c0 > 0 && !p.tcx && !local)
            lora_chunk16(lr, n, t0 + c0, min(16, tv - c0), s_ids + c0, s_lead + c0, p.tab, p.arena, p.g, p.v, p.T,
                         &pre, s_v, S::kVFloats, etid);
          if (tv >= 16 && (p.M & 7) == 0 && (reinterpret_cast<uintptr_t>(p.Y) & 15) == 0) {
            // multi-token chunk: transpose through shared memory (bf16 [16 tokens][128 columns]) so Y is
            // written as whole token rows with 16-byte stores instead of 2-byte stores strided by M
            uint16_t* st16 = reinterpret_cast<uint16_t*>(s_v);
            ptx::named_bar_sync(1, 128);  // s_v free: LoRA staging readers / the previous chunk's copy-out done
#pragma unroll
            for (int i = 0; i < 16; ++i)
              st16[i * kUmmaBM + row] = __bfloat16_as_ushort(__float2bfloat16_rn(__uint_as_float(r[i]) + lr[i]));
            ptx::named_bar_sync(1, 128);
            const int n0 = mt * kUmmaBM;
#pragma unroll
            for (int it = 0; it < 2; ++it) {
              const int q = etid + it * 128, i = q >> 4, nn = n0 + (q & 15) * 8;
              if (c0 + i < tv && nn < p.M) {
                const uint4 val = *reinterpret_cast<const uint4*>(st16 + i * kUmmaBM + (q & 15) * 8);
                *reinterpret_cast<uint4*>(p.Y + (size_t)(t0 + c0 + i) * p.M + nn) = val;
              }
            }
          } else if (n < p.M) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < tv) p.Y[(size_t)(t0 + c0 + i) * p.M + n] = __float2bfloat16_rn(__uint_as_float(r[i]) + lr[i]);
          }
        } else {
          // split tile: this CTA's fp32 partial, [row][BN] in its own slot (0 = its first segment,
          // 1 = its last).  Columns >= tv hold exact zeros (TMA zero-fills out-of-range tokens).  K-local
          // LoRA: the segment's LoRA share rides in the partial (c0 == 0: T <= 16).
          float f[16];
          if (p.cluster > 1 && !local && !p.tcx && crank == 0 && c0 > 0)  // rank 0 carries the LoRA term
            lora_chunk16(lr, n, t0 + c0, min(16, tv - c0), s_ids + c0, s_lead + c0, p.tab, p.arena, p.g, p.v, p.T,
                         &pre, s_v, S::kVFloats, etid);
          const bool add_lr = local || (p.cluster > 1 && !p.tcx && crank == 0);
#pragma unroll
          for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(r[i]) + (add_lr ? lr[i] : 0.f);
          if (p.cluster > 1) {
            // pushed into the OWNER rank's shared memory (DSMEM stores, no round trip): owner c of rows
            // [c*128/s, (c+1)*128/s) keeps [s][ceil(128/s)][BN] fp32 slots in its idle ring
            const int s = p.cluster, nr_max = (kUmmaBM + s - 1) / s;
            const int owner = ((row + 1) * s - 1) / kUmmaBM;
            const int rr = row - (owner * kUmmaBM) / s;
            const uint32_t dst =
                ptx::mapa(ptx::smem_u32(s_slots + ((size_t)(crank * nr_max + rr) * BN + c0)), (uint32_t)owner);
#pragma unroll
            for (int i = 0; i < 16; i += 4) ptx::st_dsmem_f4(dst + i * 4, f[i], f[i + 1], f[i + 2], f[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; i += 4)
              __stcg(reinterpret_cast<float4*>(my_part + c0 + i), make_float4(f[i], f[i + 1], f[i + 2], f[i + 3]));
          }
        }
      }
      if (local && !whole) {
#pragma unroll
        for (int i = 0; i < 16; ++i) lr[i] = 0.f;  // already inside the partials: the finisher adds nothing
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      if (!whole && p.cluster > 1) {
        // cluster split-K: the tile's s contributors are this cluster; rank c sums rows [c*128/s, (c+1)*128/s)
        // of every peer's partial (DSMEM, rank order -> deterministic), rounds once, stores Y
        if (etid == 0) UMMA_TRACE(12);
        ptx::cluster_arrive();  // release: my DSMEM stores -> the owners
        ptx::cluster_wait();    // acquire: every peer's rows of my range are in my shared memory
        if (etid == 0) UMMA_TRACE(11);
        const int s = p.cluster, nr_max = (kUmmaBM + s - 1) / s;
        const int r_lo = (crank * kUmmaBM) / s, r_hi = ((crank + 1) * kUmmaBM) / s, nr = r_hi - r_lo;
        const int nq = (tv + 3) / 4;
        const float* sp = s_slots;
        for (int f = etid; f < nr * nq; f += 128) {
          const int rr = f % nr, qd = f / nr;
          float4 y = *reinterpret_cast<const float4*>(sp + (size_t)rr * BN + qd * 4);
          for (int c = 1; c < s; ++c) {  // contributors in rank order: deterministic
            const float4 z = *reinterpret_cast<const float4*>(sp + ((size_t)(c * nr_max + rr) * BN + qd * 4));
            y.x += z.x, y.y += z.y, y.z += z.z, y.w += z.w;
          }
          const int nn = mt * kUmmaBM + r_lo + rr;
          if (nn < p.M) {
            const float yv[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (qd * 4 + i < tv) p.Y[(size_t)(t0 + qd * 4 + i) * p.M + nn] = __float2bfloat16_rn(yv[i]);
          }
        }
        if (etid == 0) UMMA_TRACE(10);
      } else if (!whole) {
        if (etid == 0) UMMA_TRACE(12);
        // arrival: CTA barrier, then ONE thread publishes with a gpu-scope acq_rel atomic (the
        // barrier + cumulative fence order every thread's partial before it)
        ptx::named_bar_sync(1, 128);
        if (etid == 0) {
          // counter of this split tile: indexed by its FIRST contributor (a CTA is the first contributor of at
          // most one split tile -- its range would otherwise contain a whole tile in between), so the counter
          // array is bounded by the grid, independent of T and M (fixed workspace offset)
          const int got = kb1 - kb0;
          const int cf = umma_cta_of((long long)tile * p.k_blocks, UNITS, GRID);
          const int old = ptx::atom_add_acq_rel_gpu(p.tile_cnt + cf, got);
          *s_last = (old + got == p.k_blocks);
        }
        ptx::named_bar_sync(1, 128);
        if (etid == 0) UMMA_TRACE(11);
        if (*s_last) {
          // finisher: sum the contributors' partials in CTA order (deterministic), 8 contributors'
          // loads in flight per round, add the LoRA term, round once, store.
          if (etid == 0) UMMA_TRACE(9);
          const int ts = tile * p.k_blocks;
          const int c_first = umma_cta_of(ts, UNITS, GRID);
          const int c_last = umma_cta_of(ts + p.k_blocks - 1, UNITS, GRID);
          for (int c0 = 0; c0 < tv; c0 += 16) {
            if ((c0 > 0 || tv > 16) && !p.tcx)
              lora_chunk16(lr, n, t0 + c0, min(16, tv - c0), s_ids + c0, s_lead + c0, p.tab, p.arena, p.g, p.v,
                           p.T, &pre, s_v, S::kVFloats, etid);
            const int nq = min(4, (tv - c0 + 3) / 4);  // float4 groups holding valid tokens
            float y[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) y[i] = 0.f;
            for (int cb = c_first; cb <= c_last; cb += 8) {
              float4 buf[8][4];
#pragma unroll
              for (int cc = 0; cc < 8; ++cc) {
                const int c = cb + cc;
                const int sl = (c <= c_last && ts > umma_u_lo(c, UNITS, GRID)) ? 1 : 0;
                const float4* src = reinterpret_cast<const float4*>(
                    p.part + ((size_t)(min(c, c_last) * 2 + sl) * kUmmaBM + row) * BN + c0);
#pragma unroll
                for (int g4 = 0; g4 < 4; ++g4)
                  buf[cc][g4] = (c <= c_last && g4 < nq) ? __ldcg(src + g4) : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int cc = 0; cc < 8; ++cc)
#pragma unroll
                for (int g4 = 0; g4 < 4; ++g4) {
                  y[4 * g4] += buf[cc][g4].x;
                  y[4 * g4 + 1] += buf[cc][g4].y;
                  y[4 * g4 + 2] += buf[cc][g4].z;
                  y[4 * g4 + 3] += buf[cc][g4].w;
                }
            }
            if (n < p.M) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (c0 + i < tv) p.Y[(size_t)(t0 + c0 + i) * p.M + n] = __float2bfloat16_rn(y[i] + lr[i]);
            }
          }
          if (etid == 0) {
            p.tile_cnt[c_first] = 0;
            UMMA_TRACE(10);
          }
        }
        ptx::named_bar_sync(1, 128);  // s_last reused by the next segment
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      u += kb1 - kb0;
      if (etid == 0) UMMA_TRACE(7);
    }
    if (cl_pending) ptx::cluster_wait();  // no split segment: still pair the early arrival
    } else {
      // ------------------------------------------------ shrink epilogue: v = s_a * acc, member tokens only
      const int q = warp & 3;
      const int row = q * 32 + lane;
      const int etid = threadIdx.x - 64;
      int acc = 0;
      uint32_t acc_phase = 0;
      int cur_nt = -1;
      for (int u = u_lo; u < u_hi;) {
        const int tile = u / p.k_blocks;
        const int kb0 = u - tile * p.k_blocks;
        const int kb1 = min(p.k_blocks, kb0 + (u_hi - u));
        const int mt = tile % M_TILES, nt = tile / M_TILES;
        const int t0 = nt * BN;
        const int tv = min(BN, p.T - t0);
        const bool whole = (kb0 == 0 && kb1 == p.k_blocks);
        const int slot = (tile * p.k_blocks > u_lo) ? 1 : 0;
        float* my_part = p.part + ((size_t)(cta * 2 + slot) * kUmmaBM + row) * BN;
        if (nt != cur_nt) {
          ptx::named_bar_sync(1, 128);
          for (int i = etid; i < tv; i += 128) s_ids[i] = __ldg(p.ids + t0 + i);
          ptx::named_bar_sync(1, 128);
          cur_nt = nt;
        }
        // this thread's accumulator row -> (adapter, slice, rank row) of the box it belongs to
        const int item = mt * 8 + (row >> 4), rr = row & 15;
        int va = -2, vj = 0, vk = 0;
        float vsc = 0.f;
        if (item < n_items && rr < p.route[RouteLayout::kItemN + item]) {
          va = p.route[RouteLayout::kGroupId + p.route[RouteLayout::kItemG + item]];
          vj = p.route[RouteLayout::kItemJ + item];
          vk = p.route[RouteLayout::kItemK0 + item] + rr;
          vsc = p.tab[va].scale;
        }
        ptx::mbar_wait(&tfull[acc], acc_phase);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
        for (int c0 = 0; c0 < tv; c0 += 16) {
          uint32_t r[16];
          ptx::tmem_ld_32x32b_x16(taddr + c0, r);
          ptx::tmem_ld_wait();
          if (va >= 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < tv && s_ids[c0 + i] == va) {
                float* dst = p.v_out + ((size_t)(t0 + c0 + i) * p.g.J + vj) * p.g.Rc + vk;
                if (whole)
                  *dst = vsc * __uint_as_float(r[i]);
                else
                  atomicAdd(dst, vsc * __uint_as_float(r[i]));  // split-K share (v zeroed by route_kernel)
              }
          }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        u += kb1 - kb0;
      }
    }
  }

  if (kGemm && p.cluster > 1 && warp < 2) {  // the epilogue's cluster barriers count every thread
    if (early_cl) ptx::cluster_wait();
    ptx::cluster_arrive();
    ptx::cluster_wait();
    if (kSlotsInRing) {
      ptx::cluster_arrive();
      ptx::cluster_wait();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (threadIdx.x == 0) {
    UMMA_TRACE(8);
    if (p.fuse && atomicAdd(p.sync + 2, 1) == (int)gridDim.x - 1) {  // last CTA out re-arms the counters
      p.sync[0] = 0;
      p.sync[1] = 0;
      p.sync[2] = 0;
    }
  }
  if (warp == 1) ptx::tmem_dealloc<S::kTmemCols>(tmem_base);
}

// ------------------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------------------
inline long long* g_umma_trace = nullptr;  // profiling hook (bdlora_debug_trace)
// host-side record of this thread's last tensor-core kernel launch (bdlora_last_launch_info)
inline thread_local int g_last_launch[8] = {-1, 0, 0, 0, 0, 0, 0, 0};

// LoRA expand on the tensor cores (default) -- BDLORA_TC_EXPAND=0 selects the CUDA-core epilogue expand.
inline bool tensor_expand_enabled() {
  static int env = -1;
  if (env < 0) {
    const char* s = getenv("BDLORA_TC_EXPAND");
    env = (s && s[0] == '0') ? 0 : 1;
  }
  return env == 1;
}

// K-local LoRA for decode with few adapters (bdlora_set_decode_lora / BDLORA_LOCAL: 0 = off, 1 = auto
// (default), 2 = always when eligible).
inline int g_local_mode = -1;
inline int local_lora_mode() {
  if (g_local_mode < 0) {
    const char* s = getenv("BDLORA_LOCAL");
    g_local_mode = s ? std::min(2, std::max(0, atoi(s))) : 1;
  }
  return g_local_mode;
}

// Split-K partial reduction through thread-block-cluster DSMEM (BDLORA_CLUSTER=0 disables: global fix-up).
inline int g_cluster_mode = -1;
inline bool cluster_splitk_enabled() {
  if (g_cluster_mode < 0) {
    const char* s = getenv("BDLORA_CLUSTER");
    g_cluster_mode = (s && s[0] == '0') ? 0 : 1;
  }
  return g_cluster_mode == 1;
}

// K-local LoRA only for K segments of <= kLocalMaxKb k-blocks per CTA (BDLORA_LOCAL_MAXKB overrides)
inline int local_max_kb() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("BDLORA_LOCAL_MAXKB");
    v = s ? std::max(0, atoi(s)) : 8;
  }
  return v;
}

// CTAs of a stream-K launch (BDLORA_STREAMK_CTAS overrides; tuning)
inline int streamk_ctas(int num_sms) {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("BDLORA_STREAMK_CTAS");
    v = s ? std::max(1, atoi(s)) : 0;
  }
  return v > 0 ? (num_sms > 0 ? std::min(v, num_sms) : v) : 0;
}

inline int umma_bn_for(int T) { return T <= 16 ? 16 : T <= 32 ? 32 : T <= 64 ? 64 : T <= 128 ? 128 : 256; }

// Token-tile width of the base GEMM.  Decode-sized batches take the smallest tile covering T.  For T > 64
// (compute-bound) the width trades per-SM operand traffic -- FLOP per loaded byte ~ 128 BN / (128 + BN),
// the kernel being bound by each SM's operand ingress -- against SM coverage and wave quantization:
// e.g. 8B QKV at TP8 (6 row tiles, T = 1024): BN 256 gives 24 tiles (split 6 ways, 128 KB fp32 partials
// each), BN 64 gives 96 whole tiles.  Never wider than umma_bn_for(T) (the workspace is sized for it).
inline int umma_bn_for_gemm(int M, int T, int num_sms) {
  const int bn0 = umma_bn_for(T);
  if (T <= 64) return bn0;
  const int m_tiles = (M + kUmmaBM - 1) / kUmmaBM;
  int best = bn0;
  double best_eff = -1.0;
  for (int bn = 64; bn <= bn0; bn *= 2) {
    const long long tiles = (long long)m_tiles * ((T + bn - 1) / bn);
    const long long waves = (tiles + num_sms - 1) / num_sms;
    const double eff = (double)tiles / (double)(waves * num_sms) * (128.0 * bn) / (128.0 + bn);
    if (eff > best_eff * 1.05) {  // ties -> the wider tile
      best_eff = eff;
      best = bn;
    }
  }
  return best;
}

// Compute-bound batches (T > 64) of the base GEMM: token-tile width AND cluster split-K together.  The kernel
// is bound by each SM's operand ingress (~80 GB/s L2 -> shared memory), so the plan minimises the operand
// bytes of the busiest CTA: (128 + BN) * K * 2 / s for a tile split s ways (s contributors of a cluster reduce
// through DSMEM; their 128 x BN fp32 partials, pushed once, are counted at half weight), waves x (128 + BN) * K
// * 2 for whole tiles beyond the SM count.  E.g. 8B QKV at TP8 (6 row tiles, T = 1024, K = 4096): BN 64 = 96
// whole tiles (1.57 MB per CTA), BN 256 split 6 ways = 144 CTAs (0.52 MB + 128 KB of partials).
inline void umma_tile_plan(int M, int K, int T, int num_sms, int* bn_out, int* split_out) {
  const int bn0 = umma_bn_for(T);
  const int m_tiles = (M + kUmmaBM - 1) / kUmmaBM, k_blocks = std::max(1, K / kUmmaBK);
  double best = 1e300;
  *bn_out = bn0;
  *split_out = 1;
  for (int bn = 64; bn <= bn0; bn *= 2) {
    const long long tiles = (long long)m_tiles * ((T + bn - 1) / bn);
    int s = 1;
    double bytes;
    if (tiles <= num_sms) {
      s = (int)std::max<long long>(1, std::min<long long>(8, std::min<long long>(num_sms / tiles, k_blocks / 8)));
      bytes = (128.0 + bn) * K * 2.0 / s + (s > 1 ? 0.5 * 128.0 * bn * 4.0 : 0.0);
    } else {
      const long long waves = (tiles + num_sms - 1) / num_sms;
      bytes = (bn >= 128 ? (double)waves : (double)tiles / num_sms) * (128.0 + bn) * K * 2.0;
    }
    if (bytes < best * 0.95) {  // near-ties -> the wider tile (fewer X re-reads)
      best = bytes;
      *bn_out = bn;
      *split_out = s;
    }
  }
}

// Counter region (fixed size, at a T-independent workspace offset, zero between launches):
// [sync: 64 ints][split-tile counters: kUmmaMaxGrid ints]
constexpr size_t kUmmaCounterBytes = 256 + kUmmaMaxGrid * sizeof(int);
// Scratch (T-dependent): split-tile partials [grid][2][128][BN] fp32
inline size_t umma_workspace_bytes(int M, int T, int num_sms = 148) {
  (void)M;
  const int BN = umma_bn_for(T);  // the widest tile umma_bn_for_gemm may pick (partials)
  return (size_t)std::min(num_sms, kUmmaMaxGrid) * 2 * BN * kUmmaBM * sizeof(float);
}

inline bool umma_eligible(const Geom& g, int T) { return T >= 1 && g.K % kUmmaBK == 0 && g.K >= kUmmaBK; }

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)ptr;
  }
  return fn;
}

// 2D bf16 K-major tensor [rows, K] with box [box_rows, 64], SWIZZLE_128B, OOB -> zeros.
inline bool encode_kmajor(CUtensorMap* m, const void* base, int K, int rows, int box_rows) {
  if (tmap_memo_get(base, K, rows, box_rows, m)) return true;
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)kUmmaBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  tmap_memo_put(base, K, rows, box_rows, *m);
  return true;
}

// Ring depth.  Measured (scripts/stages_sweep.sh, 8B decode layer): 2 stages 134 us, 3: 103, 4: 100,
// 6: 95.7, 10: 95.8 -- per-SM bandwidth needs the deep ring, at the price of a longer HBM queue that
// the dependent LoRA loads sit in.  Default: the full ring.  Override with BDLORA_STAGES for tuning.
inline int umma_stage_cap(int T) {
  static int env = -1;
  if (env < 0) {
    const char* s = getenv("BDLORA_STAGES");
    env = s ? std::max(1, atoi(s)) : 0;
  }
  if (env > 0) return env;
  return 64;
}

template <int BN, int MODE>
inline int umma_launch_bn(const UmmaParams& p0, const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmA,
                          cudaStream_t st) {
  using S = UmmaSmem<BN>;
  UmmaParams p1 = p0;
  p1.nstages = std::min(S::kStages, umma_stage_cap(p0.T));
  // function attributes and occupancy answers are per device context: cached per device
  int dev = 0;
  cudaGetDevice(&dev);
  dev = std::min(std::max(dev, 0), kMaxDevices - 1);
  while (MODE != 1 && p1.cluster > 1) {
    // every cluster must be co-resident in one wave (one CTA per SM)
    static int max_clusters[kMaxDevices][9];
    static bool mc_init = false;
    if (!mc_init) {
      for (int d = 0; d < kMaxDevices; ++d)
        for (int c = 0; c < 9; ++c) max_clusters[d][c] = -1;
      mc_init = true;
    }
    int& mc = max_clusters[dev][p1.cluster];
    if (mc < 0) {
      if (cudaFuncSetAttribute(umma_lora_gemm_kernel<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               S::kBytes) != cudaSuccess)
        return 2;
      cudaLaunchConfig_t qc = {};
      qc.gridDim = dim3(p1.grid);
      qc.blockDim = dim3(kUmmaThreads);
      qc.dynamicSmemBytes = S::kBytes;
      cudaLaunchAttribute ca[1];
      ca[0].id = cudaLaunchAttributeClusterDimension;
      ca[0].val.clusterDim.x = p1.cluster;
      ca[0].val.clusterDim.y = 1;
      ca[0].val.clusterDim.z = 1;
      qc.attrs = ca;
      qc.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&mc, (void*)umma_lora_gemm_kernel<BN, MODE>, &qc) != cudaSuccess) {
        cudaGetLastError();
        mc = 0;
      }
    }
    const int tiles = p1.grid / p1.cluster;
    const bool fits = (long long)mc >= tiles;
    if (getenv("BDLORA_DEBUG"))
      fprintf(stderr, "[bdlora] umma BN=%d tiles=%d cluster=%d (max active clusters %d) fits=%d\n", BN, tiles,
              p1.cluster, mc, (int)fits);
    if (fits) break;
    const char* shrink = getenv("BDLORA_CLUSTER_SHRINK");
    if (shrink && shrink[0] == '0') {
      p1.cluster = 1;  // keep the split, global fix-up
      break;
    }
    // a smaller cluster: the tile split s shrinks with it (fewer, longer K segments per CTA)
    p1.cluster -= 1;
    p1.grid = tiles * p1.cluster;
  }
  if (MODE != 1 && p0.cluster > 1) {
    // the K-local LoRA adds a 2 KB A box to every k-block: worth it only where the tail dominates (cluster
    // reduce, short K segments -- measured alone: 8B O (16 k-blocks/CTA) -1.5 us but +1 us in the layer chain,
    // 8B down (56) +5 us); otherwise the grid-wide shrink hides under the stream
    if (p1.cluster == 1 || p1.k_blocks / p1.cluster > local_max_kb()) p1.local = 0;
  }
  static bool attr_set[kMaxDevices] = {};
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(umma_lora_gemm_kernel<BN, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             S::kBytes) != cudaSuccess)
      return 2;
    attr_set[dev] = true;
  }
  // launch record (bdlora_last_launch_info): which instantiation and schedule this call took
  g_last_launch[0] = MODE;
  g_last_launch[1] = BN;
  g_last_launch[2] = p1.grid;
  g_last_launch[3] = (MODE != 1 && p1.cluster > 1) ? p1.cluster : 1;
  g_last_launch[4] = p1.nstages;
  g_last_launch[5] = p1.m_tiles;
  g_last_launch[6] = p1.n_tiles;
  g_last_launch[7] = p1.k_blocks;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p1.grid);
  cfg.blockDim = dim3(kUmmaThreads);
  cfg.dynamicSmemBytes = S::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = p0.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (MODE != 1 && p1.cluster > 1) {
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = p1.cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.numAttrs = 2;
  }
  if (cudaLaunchKernelEx(&cfg, umma_lora_gemm_kernel<BN, MODE>, tmW, tmX, tmA, p1) != cudaSuccess) return 4;
  return 0;
}

template <int MODE>
inline int umma_dispatch_bn(int BN, const UmmaParams& p, const CUtensorMap& tmW, const CUtensorMap& tmX,
                            const CUtensorMap& tmA, cudaStream_t st) {
  switch (BN) {
    case 16: return umma_launch_bn<16, MODE>(p, tmW, tmX, tmA, st);
    case 32: return umma_launch_bn<32, MODE>(p, tmW, tmX, tmA, st);
    case 64: return umma_launch_bn<64, MODE>(p, tmW, tmX, tmA, st);
    case 128: return umma_launch_bn<128, MODE>(p, tmW, tmX, tmA, st);
    default: return umma_launch_bn<256, MODE>(p, tmW, tmX, tmA, st);
  }
}

// Returns 0 on launch, non-zero if the shape is not handled here.
inline int umma_launch(const Geom& g, const __nv_bfloat16* X, int T, const __nv_bfloat16* W, const int* ids,
                       const SlotEntry* tab, const __nv_bfloat16* arena, const float* v, __nv_bfloat16* Y, void* cnt,
                       void* ws, int num_sms, cudaStream_t st, int pdl = 0, float* v_fused = nullptr, int rs_max = 0,
                       int tcx = 0, const CUtensorMap* amap = nullptr) {
  if (!umma_eligible(g, T)) return 1;
  if (v_fused && T > kFuseMaxT) return 1;
  // (umma_tile_plan -- wider tiles split over a cluster -- measured slower: 8B QKV prefill at TP8 35.3 -> 42.0 us,
  // TP4 40.2 -> 51.7 us; kept for reference, not used)
  const int BN = umma_bn_for_gemm(g.M, T, num_sms);
  const int plan_split = 0;
  UmmaParams p;
  p.M = g.M;
  p.K = g.K;
  p.T = T;
  p.m_tiles = (g.M + kUmmaBM - 1) / kUmmaBM;
  p.n_tiles = (T + BN - 1) / BN;
  p.k_blocks = (g.K + kUmmaBK - 1) / kUmmaBK;
  const long long units = (long long)p.m_tiles * p.n_tiles * p.k_blocks;
  if (units > (1LL << 30)) return 1;
  p.units = (int)units;
  // Work split.  tiles <= #SM: plain split-K with s equal K-ranges per tile (grid = tiles * s, each CTA
  // inside ONE tile, all contributors of a tile finish together -> a single short fix-up at the end).
  // tiles > #SM: stream-K over all SMs.  Both keep >= 8 k-blocks per CTA so a split tile has few
  // contributors.  (The stream-K formula with grid = tiles * s reproduces the split-K ranges.)
  const long long tiles = (long long)p.m_tiles * p.n_tiles;
  p.cluster = 1;
  if (tiles <= num_sms) {
    long long s = std::max<long long>(1, std::min<long long>(num_sms / tiles, p.k_blocks / 8));
    long long sc = std::min<long long>(8, std::min<long long>(num_sms / tiles, p.k_blocks / 4));
    if (plan_split > 0) {
      // compute-bound tiles (T > 64): the tile plan's split, through a cluster (the partials are pushed once
      // into the owners' idle weight rings); without clusters a compute-bound tile stays whole
      s = cluster_splitk_enabled() ? plan_split : 1;
      sc = s;
    }
    // cluster split-K (the s contributors of a tile reduce through DSMEM): cheap fix-up, so split finer
    if (cluster_splitk_enabled() && sc >= 2) {
      s = sc;
      p.cluster = (int)sc;
    }
    p.grid = (int)(tiles * s);
  } else if (BN >= 128) {
    // compute-bound token tiles (prefill): one whole tile per CTA, no split fix-ups (a split 128 x 256
    // tile would move 128 KB of partials and redo the LoRA expand in the finisher)
    p.grid = (int)tiles;
  } else {
    // stream-K over fewer CTAs than SMs: ~112 CTAs already saturate HBM (~60 GB/s per SM), and fewer
    // requests queue at the DRAM.  Prefer a grid that divides the tiles (whole tiles per CTA: no partials,
    // no fix-up), else ~0.86 x #SM.  Measured 8B gate_up (224 tiles, T = 1): 148 CTAs 41.6 us, 136: 41.4,
    // 128: 39.4, 120: 42.5, 112 (2 whole tiles each): 39.1, 104: 43.8.
    long long g = 0;
    for (long long m = 1; m <= 16 && !g; ++m)
      if (tiles % m == 0 && tiles / m <= num_sms && tiles / m * 10 >= (long long)num_sms * 7) g = tiles / m;
    if (!g) g = (long long)num_sms * 86 / 100;
    if (streamk_ctas(0) > 0) g = streamk_ctas(num_sms);
    p.grid = (int)std::max<long long>(1, std::min<long long>(units / 8, g));
  }
  p.ids = ids;
  p.tab = tab;
  p.arena = arena;
  p.g = g;
  p.v = v;
  p.Y = Y;
  if (p.grid > kUmmaMaxGrid && !(BN >= 128 && tiles > num_sms)) return 1;  // split-tile counters bounded
  p.sync = (int*)cnt;
  p.tile_cnt = (int*)((char*)cnt + 256);
  p.part = (float*)ws;
  p.X = X;
  p.fuse = v_fused ? 1 : 0;
  p.v_out = v_fused;
  p.rs_max = rs_max;
  // the single-kernel forward (MODE 2 instantiation) expands on the CUDA cores; the rest on the tensor cores
  p.tcx = (!tensor_expand_enabled() || v_fused) ? 0 : tcx;
  if (v_fused) p.v = v_fused;
  p.pdl = pdl;
  p.trace = g_umma_trace;
  // K-local LoRA needs the arena's A-row tensor map and tiles that never straddle a slice boundary
  bool aligned = true;
  for (int j = 1; j < g.J; ++j) aligned = aligned && (g.col0[j] % kUmmaBM == 0);
  p.local = (v_fused && amap && aligned && BN == 16 && p.cluster > 1) ? local_lora_mode() : 0;
  p.nstages = 0;  // set per BN
  p.route = nullptr;
  CUtensorMap tmW, tmX;
  if (!encode_kmajor(&tmW, W, p.K, p.M, kUmmaBM)) return 3;
  if (!encode_kmajor(&tmX, X, p.K, p.T, BN)) return 3;
  // without K-local LoRA the A boxes are dummies (row 0 of the arena map, or of X): same bytes, ignored
  return p.fuse ? umma_dispatch_bn<2>(BN, p, tmW, tmX, amap ? *amap : tmX, st)
                : umma_dispatch_bn<0>(BN, p, tmW, tmX, amap ? *amap : tmX, st);
}

// Tensor-core shrink: v[t][j][k] = s_a X[t] . A_{a,j}[k] for every token t of every distinct adapter a,
// the A rows gathered in 16-row TMA boxes through `amap` (the pool arena viewed as [rows, K]).  The item
// list comes from route_kernel (launched just before).  Workspace as umma_workspace_bytes(items_max*16, T).
inline size_t umma_shrink_workspace_bytes(int items_max, int T, int num_sms = 148) {
  return kUmmaCounterBytes;  // the shrink writes v directly (no partials); counters kept for uniformity
}

inline int umma_shrink_launch(const Geom& g, const __nv_bfloat16* X, int T, const int* ids, const SlotEntry* tab,
                              const int* route, const CUtensorMap& amap, float* v_out, int items_max, void* ws,
                              int num_sms, cudaStream_t st, int pdl) {
  if (g.K % kUmmaBK != 0 || T < 1) return 1;
  // few A boxes (rows) and many tokens: narrower token tiles give the shrink more CTAs (8B O prefill at TP8:
  // BN 256 -> 4 CTAs, 30 us)
  const int BN = umma_bn_for_gemm(((items_max + 7) / 8) * kUmmaBM, T, num_sms);
  UmmaParams p{};
  p.M = 0;
  p.K = g.K;
  p.T = T;
  p.m_tiles = (items_max + 7) / 8;
  p.n_tiles = (T + BN - 1) / BN;
  p.k_blocks = g.K / kUmmaBK;
  const long long units_max = (long long)p.m_tiles * p.n_tiles * p.k_blocks;
  if (units_max > (1LL << 30)) return 1;
  p.units = (int)units_max;
  p.grid = (int)std::max<long long>(1, std::min<long long>(units_max / 8, num_sms));
  p.ids = ids;
  p.tab = tab;
  p.g = g;
  p.v = nullptr;
  p.Y = nullptr;
  p.sync = (int*)ws;
  p.tile_cnt = (int*)((char*)ws + 256);
  p.part = nullptr;
  p.X = X;
  p.fuse = 0;
  p.tcx = 0;
  p.local = 0;
  p.v_out = v_out;
  p.route = route;
  p.pdl = pdl;
  p.trace = g_umma_trace;
  CUtensorMap tmX;
  if (!encode_kmajor(&tmX, X, p.K, p.T, BN)) return 3;
  return umma_dispatch_bn<1>(BN, p, amap, tmX, amap, st);
}

}  // namespace bdl
