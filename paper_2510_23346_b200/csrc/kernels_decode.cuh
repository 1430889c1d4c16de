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
#include "peer.h"
#include "ptx.cuh"

namespace bdl {

constexpr int kDecThreads = 192;
constexpr int kDecBM = 128, kDecBK = 64, kDecBN = 16;
constexpr int kDecLoraRows = 32;   // K-local: sum over the batch's distinct adapters of their local rank rs
constexpr int kDecMaxGroups = 16;  // distinct adapters of a <= 16-token batch
constexpr int kDecMaxGrid = 1024;  // split-tile counters (indexed by the first contributor CTA)
constexpr int kDecMaxCluster = 16; // cluster split-K: contributors of one tile (non-portable size above 8)
constexpr int kDecMtStages = 4;    // ring depth of the multi-adapter (LM 3) instantiation

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
  float* part;        // [grid][2][128][16] fp32 split-tile partials (slot 0: a CTA's first segment, 1: its last)
  int* cnt;           // [kDecMaxGrid] arrival counters of split tiles, zero between launches
  int lora;           // 0 none, 1 K-local, 2 v precomputed (per-output gather), 3 v precomputed (B staged)
  int pdl;
  int nstages;
  int cluster;        // > 1: the tile's contributors are one thread-block cluster (DSMEM reduce, CL instantiation)
  int tc_shrink;      // CL: the K-local shrink may run on the tensor cores (tmA = the arena's 16-row A boxes)
  long long* trace;   // optional per-CTA %globaltimer stamps (32 per CTA)
  int push;           // 1: row partial pushed (fp32) into every rank's receive slot instead of stored to Y
  PeerDev peer;       // push == 1: the peer group (peer.h)
};

// One output element: y_t[n] rounded once to bf16 into Y, or -- fused row all-reduce -- the fp32 partial
// written into slot [parity][this rank] of every rank's receive buffer (NVLink stores for the peers).
template <bool PUSH>
__device__ __forceinline__ void dec_out(const DecParams& p, int par, int t, int n, float y) {
  if (PUSH) {
    const size_t off = ((size_t)(par * p.peer.nranks + p.peer.rank)) * p.peer.slot + (size_t)t * p.M + n;
    for (int r = 0; r < p.peer.nranks; ++r) __stcg(p.peer.recv[r] + off, y);
  } else {
    p.Y[(size_t)t * p.M + n] = __float2bfloat16_rn(y);
  }
}

// LM 3 (multi-adapter expand of a precomputed v): adapter-group tables of up to 64 tokens / 64 groups
struct alignas(16) DecGroups {
  int ids[64];      // token ids (-1 past T)
  int grp[64];      // group of each token (-1 = no adapter)
  int lgid[64];     // group index of each leader token
  int gad[64];      // adapter id of each group (order of first appearance)
  int grs[64];      // shrink rank rows (A rows on this device)
  int gre[64];      // expand rank rows (B rows on this device)
  int gq0[64];      // first expand row of the group in the batch's row numbering (prefix of gre)
  int gp0[64];      // prefix of grs (the shrink's item numbering)
  int gcnt[64];     // member tokens
  int gst[64];      // first member in gmem
  int gmem[64];     // member tokens, grouped, token order inside a group
  float gsc[64];    // s_a
  long long goffA[64][kMaxSlices];
  long long goffB[64][kMaxSlices];
  unsigned lm[2];
  int ngroups, qtot, ptot, pad;
};

template <int S, bool CL, int BN = 16, int LM = 1>
struct DecSmem {
  static constexpr bool kMt = LM == 3;           // multi-adapter expand of a precomputed v (BN = 64 only)
  static constexpr int kW = kDecBM * kDecBK * 2;  // 16 KB weight tile
  static constexpr int kX = BN * kDecBK * 2;      // token tile (2 KB at BN = 16)
  // CL: a 16-row box of the batch's adapter A rows per stage (tensor-core K-local shrink).  The ring sits
  // FIRST: the shrink MMA's operand is 128 rows (M = 128), rows 16..127 -- ignored TMEM lanes -- read the
  // next 14 KB of this CTA's own shared memory (following boxes and the weight ring), never past it
  static constexpr int kTcShrink = !kMt && (CL || BN == 64);   // instantiations with the tensor-core K-local shrink
  static constexpr int kA = kTcShrink ? 16 * kDecBK * 2 : 0;
  static constexpr int kWOff = S * kA;
  static constexpr int kXOff = kWOff + S * kW;
  static constexpr int kBarOff = kXOff + S * kX;
  static constexpr int kMiscOff = kBarOff + 256;
  // misc ints: [0,16) ids  [16,32) group of token  [32,48) group adapter  [48,64) group rs  [64,80) group row
  // offset q0  [80,96) member masks  [96] n_groups  [97] rows total ; floats [128,144) group scale ;
  // long long [160 + 2*(g*3 + j)) group A / B offsets per slice (as int pairs)
  // ... [960, 1024) group of each of up to 64 tokens.  LM 3: a DecGroups.
  static constexpr int kMiscBytes = kMt ? 12288 : 4096;
  static constexpr int kMtListOff = 8192;  // LM 3: per chunk buffer and warp, the tokens whose group meets the chunk
  static constexpr int kMtRowOff = 10496;  // LM 3: arena offset of each staged chunk row (96 x 8 B)
  static_assert(!kMt || sizeof(DecGroups) <= kMtListOff, "group tables");
  static_assert(kMtRowOff >= kMtListOff + 2 * 2 * 32 * 16 + 16 && kMtRowOff + 96 * 12 <= 12288 - 16, "row table");
  // v_seg: BN = 16: [16 tokens][3 slices][32] fp32; BN = 64 (one adapter, one slice per tile): [64][32]
  static constexpr int kVsTok = BN == 16 ? 3 * kDecLoraRows : kDecLoraRows;
  static constexpr int kVsOff = kMiscOff + kMiscBytes;
  static constexpr int kVsBytes = kMt ? 0 : BN * kVsTok * 4;
  // B rows of the tile's columns: [32][128] bf16; LM 3: two 96-row chunk buffers (cp.async double buffering;
  // both issued before the programmatic-dependency wait, so a share of <= 192 rows is in flight in one shot),
  // stored as the MN-major no-swizzle operand of the tensor-core expand: (n, q) at
  // (q/8)*2048 + (n/8)*128 + (q%8)*16 + (n%8)*2
  static constexpr int kBOff = kVsOff + kVsBytes;
  static constexpr int kMtRows = 96;
  static constexpr int kBBytes = kMt ? 2 * kMtRows * kDecBM * 2 : kDecLoraRows * kDecBM * 2;
  // (LM 3 keeps the tile's LoRA terms in TMEM columns [kLrCol, kLrCol + 64): thread = TMEM lane = column)
  static constexpr int kLrOff = kBOff + kBBytes;
  static constexpr int kLrBytes = 0;
  static constexpr int kLrCol = 2 * BN;
  // LM 3: the tensor-core expand's token operand of one chunk, V_hi | V_lo [64 tokens][kMtRows] bf16, K-major
  // no-swizzle core-matrix layout (the B chunk above is the MN-major operand of the same MMA)
  static constexpr int kVOpOff = kLrOff + kLrBytes;
  static constexpr int kVOpHalf = kMt ? 64 * kMtRows * 2 : 0;
  // cluster split-K: [s][ceil(128/s)][16] fp32 partial slots the peers push into (<= (128 + s) x 16 floats)
  static constexpr int kSlotOff = kVOpOff + 2 * kVOpHalf;
  // a slot row is BN + 4 floats: consecutive rows start 16 bytes apart in the banks, so the contributors'
  // float4 pushes (one row per thread) and the owner's float4 reads are bank-conflict free
  static constexpr int kSlotStride = BN + 4;
  static constexpr int kSlotBytes = CL ? (kDecBM + kDecMaxCluster) * kSlotStride * 4 : 0;
  static constexpr int kBytes = kSlotOff + kSlotBytes + 1024;   // + 1024-B alignment slack
  static constexpr int kVCol = 2 * BN;                          // TMEM: [acc 0 | acc 1 | v_seg 0 | v_seg 1]
  static constexpr int kTmemCols = BN == 16 ? (CL ? 64 : 32) : 256;
  static_assert(S > 5 || BN > 16 || kBytes <= 113 * 1024, "two CTAs per SM");
  static_assert(kBytes <= 227 * 1024, "shared memory per CTA");
};

#define DEC_TRACE(slot)                                               \
  do {                                                                \
    if (p.trace) {                                                    \
      long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));          \
      p.trace[(size_t)blockIdx.x * 32 + (slot)] = t_;                 \
    }                                                                 \
  } while (0)

// Adapter groups of a batch of T <= 64 tokens (distinct ids in order of first appearance), built
// by every thread of a barrier group of >= 64 threads (tid 0..; whole warps), `sync` = that group's barrier.
// ids and the slot table are never written by the kernel preceding a forward (bdlora_set_pdl contract), so
// this runs before the programmatic-dependency wait.
template <class Sync>
__device__ __forceinline__ void dec_groups64(DecGroups& G, const int* __restrict__ ids, int T,
                                             const SlotEntry* __restrict__ tab, int tid, Sync sync) {
  if (tid < 64) G.ids[tid] = tid < T ? __ldg(ids + tid) : -1;
  sync();
  int id = -1, first = 64, pos = 0, cnt_all = 0;
  if (tid < 64) {
    // all 64 ids through 16 broadcast 16-byte loads, compared in registers (no dependent shared-memory chain)
    id = G.ids[tid];
    const int4* v4 = reinterpret_cast<const int4*>(G.ids);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int4 w = v4[q];
      const int o[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int t2 = 4 * q + e;
        const bool eq = o[e] == id;
        first = (eq && t2 < first) ? t2 : first;
        pos += (eq && t2 < tid) ? 1 : 0;
        cnt_all += eq ? 1 : 0;
      }
    }
  }
  const bool lead = id >= 0 && first == tid;
  const unsigned bm = __ballot_sync(0xffffffffu, lead);
  if (tid < 64 && (tid & 31) == 0) G.lm[tid >> 5] = bm;
  sync();
  const unsigned lm0 = G.lm[0], lm1 = G.lm[1];
  if (lead) {
    const int lane = tid & 31;
    const int gi = tid < 32 ? __popc(lm0 & ((1u << lane) - 1u)) : __popc(lm0) + __popc(lm1 & ((1u << lane) - 1u));
    G.lgid[tid] = gi;
    const SlotEntry e = tab[id];
    G.gad[gi] = id;
    G.gsc[gi] = e.scale;
    G.grs[gi] = e.rs;
    G.gre[gi] = e.re;
#pragma unroll
    for (int j = 0; j < kMaxSlices; ++j) {
      G.goffA[gi][j] = e.offA[j];
      G.goffB[gi][j] = e.offB[j];
    }
    G.gcnt[gi] = cnt_all;
  }
  sync();
  if (tid < 64) G.grp[tid] = id >= 0 ? G.lgid[first] : -1;  // first <= tid is a leader when id >= 0
  if (tid < 32) {  // exclusive prefixes over the groups (two per lane): expand rows, shrink rows, members
    const int ng = __popc(lm0) + __popc(lm1);
    const int g0 = 2 * tid, g1 = 2 * tid + 1;
    const int e0 = g0 < ng ? G.gre[g0] : 0, e1 = g1 < ng ? G.gre[g1] : 0;
    const int s0 = g0 < ng ? G.grs[g0] : 0, s1 = g1 < ng ? G.grs[g1] : 0;
    const int c0 = g0 < ng ? G.gcnt[g0] : 0, c1 = g1 < ng ? G.gcnt[g1] : 0;
    int ie = e0 + e1, is = s0 + s1, ic = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ye = __shfl_up_sync(0xffffffffu, ie, o), ys = __shfl_up_sync(0xffffffffu, is, o),
                yc = __shfl_up_sync(0xffffffffu, ic, o);
      if (tid >= o) ie += ye, is += ys, ic += yc;
    }
    const int xe = ie - e0 - e1, xs = is - s0 - s1, xc = ic - c0 - c1;
    if (g0 < ng) G.gq0[g0] = xe, G.gp0[g0] = xs, G.gst[g0] = xc;
    if (g1 < ng) G.gq0[g1] = xe + e0, G.gp0[g1] = xs + s0, G.gst[g1] = xc + c0;
    if (tid == 31) G.ngroups = ng, G.qtot = ie, G.ptot = is;
  }
  sync();
  if (tid < 64 && id >= 0) G.gmem[G.gst[G.grp[tid]] + pos] = tid;
  sync();
}

// group holding row q of a prefix table (largest g < ng with pre[g] <= q)
__device__ __forceinline__ int dec_find_group(const int* pre, int ng, int q) {
  int lo = 0, hi = ng - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= q) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Multi-adapter LoRA shrink of a decode batch (matmul_3 / matmul_5 for T <= 64 tokens over many adapters,
// P:287-288):  v[t][j][k] = s_a(t) X[t] . A_{a(t),j}[k]  (fp32, scaled; layout [T][J][Rc]).
// Work item = one (token, slice, rank row) dot product of length K: 1, 2 or 4 warps share an item (K <= 2048,
// <= 4096, longer: <= 8 A + 8 X 16-byte loads in flight per lane), fixed-order reduction (deterministic).  Tokens of one
// adapter read the same A rows (L2 hits after the first).  Launched before the decode GEMM with programmatic
// dependent launch: the GEMM streams its weights (and stages its B rows) while this runs.
constexpr int kDecShrinkThreads = 128;
__global__ void __launch_bounds__(kDecShrinkThreads, 4) dec_shrink_kernel(const __nv_bfloat16* __restrict__ X, int T,
                                                                          const int* __restrict__ ids,
                                                                          const SlotEntry* __restrict__ tab,
                                                                          const __nv_bfloat16* __restrict__ arena,
                                                                          Geom g, float* __restrict__ v, int pdl,
                                                                          int late_trigger) {
  __shared__ int s_pre[65];               // exclusive prefix over tokens of J * rs(a(t)) (items)
  __shared__ int s_rs[64];
  __shared__ float s_sc[64];
  __shared__ long long s_offA[64][kMaxSlices];
  __shared__ int s_wtot;
  __shared__ float s_red[4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = g.J, K = g.K;
  if (tid < 64) {  // ids and the slot table are not written by the preceding kernel (bdlora_set_pdl contract)
    const int id = tid < T ? __ldg(ids + tid) : -1;
    int rs = 0;
    if (id >= 0) {
      const SlotEntry e = tab[id];
      rs = e.rs;
      s_sc[tid] = e.scale;
#pragma unroll
      for (int j = 0; j < kMaxSlices; ++j) s_offA[tid][j] = e.offA[j];
    }
    s_rs[tid] = rs;
    int incl = J * rs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (tid == 31) s_wtot = incl;
    s_pre[tid + 1] = incl;  // warp-local inclusive; warp 1 adds warp 0's total below
  }
  __syncthreads();
  if (tid >= 32 && tid < 64) s_pre[tid + 1] += s_wtot;
  if (tid == 0) s_pre[0] = 0;
  __syncthreads();
  // the GEMM may start streaming its weights -- unless its CTAs (one per SM, ~226 KB of shared memory) would
  // crowd this grid out of the SMs (late_trigger: launched once this CTA's items are done)
  if (tid == 0 && !late_trigger) ptx::pdl_launch_dependents();
  if (pdl) ptx::pdl_wait();                    // X is written by the preceding kernel
  const int items = s_pre[64];
  // downward-compatible ROW pool (g.ablk = m > 1): rank row k of block b = k / (rs/m) is stored compactly with
  // its block's K/m inputs only and dots X[t][b K/m, (b+1) K/m) -- no zero of the block-diagonal A_2 is read
  const int ab = g.ablk > 1 ? g.ablk : 1, kl = K / ab;
  const int nch = kl >> 3;  // 16-byte chunks of a row
  // wpi warps per item (a lane keeps <= 8 chunks of A and X in flight per pass): short rows take one warp each,
  // so a CTA works on 4 / wpi items at once (the latency of one L2 round trip per item, not per CTA)
  const int wpi = kl <= 2048 ? 1 : (kl <= 4096 ? 2 : 4);
  const int gpc = 4 / wpi, grp = warp / wpi, sub = warp - grp * wpi;
  const int c_lo = (nch * sub) / wpi, c_hi = (nch * (sub + 1)) / wpi;
  for (int it = blockIdx.x * gpc + grp; it < items; it += gridDim.x * gpc) {
    int lo = 0, hi = 63;  // token: largest t with s_pre[t] <= it
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_pre[mid] <= it) lo = mid;
      else hi = mid - 1;
    }
    const int t = lo, rs = s_rs[t];
    const int r = it - s_pre[t], j = r / rs, k = r - j * rs;
    const __nv_bfloat16* Arow = arena + s_offA[t][j] + (size_t)k * kl;
    const __nv_bfloat16* Xrow = X + (size_t)t * K + (size_t)(ab > 1 ? k / (rs / ab) : 0) * kl;
    float acc = 0.f, acc2 = 0.f;
#pragma unroll 1
    for (int cb = c_lo; cb < c_hi; cb += 256) {  // 8 chunks per lane per block (one block at K = 8192)
      uint4 av[8], xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int cc = cb + lane + 32 * u;
        av[u] = cc < c_hi ? ld_cached_u4(Arow + (size_t)cc * 8) : make_uint4(0u, 0u, 0u, 0u);
        xv[u] = cc < c_hi ? ld_cached_u4(Xrow + (size_t)cc * 8) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float af[8], xf[8];
        bf16x8_to_f32(av[u], af);
        bf16x8_to_f32(xv[u], xf);
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          acc = fmaf(af[e], xf[e], acc);
          acc2 = fmaf(af[e + 1], xf[e + 1], acc2);
        }
      }
    }
    const float ws = warp_sum(acc + acc2);
    float* vo = v + ((size_t)t * J + j) * g.Rc + k;
    if (wpi == 1) {
      if (lane == 0) *vo = s_sc[t] * ws;
    } else {  // fixed-order sum of the item's warps (deterministic)
      if (lane == 0) s_red[warp] = ws;
      ptx::named_bar_sync(1 + grp, wpi * 32);
      if (sub == 0 && lane == 0)
        *vo = s_sc[t] * (wpi == 2 ? s_red[warp] + s_red[warp + 1]
                                  : (s_red[warp] + s_red[warp + 1]) + (s_red[warp + 2] + s_red[warp + 3]));
      ptx::named_bar_sync(1 + grp, wpi * 32);
    }
  }
  if (tid == 0 && late_trigger) ptx::pdl_launch_dependents();
}

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

// lora == 2 (v precomputed): lr[t] = s_a v[t] . B_a[:, n] for every token of the batch (matmul_4 / _6 after
// S-LoRA's collective).  Out of line: it runs once per output element on the S-LoRA path only, and keeping
// it out of the kernel body keeps the decode kernel's executed footprint small.
__device__ __noinline__ void dec_vmode_lr(const DecParams* pp, int n, int t0, int cnt, float* lr) {
  const DecParams& p = *pp;
  for (int i = 0; i < cnt; ++i) {
    const int t = t0 + i;
    const int a = __ldg(p.ids + t);
    lr[i] = (a >= 0) ? lora_expand_term(t, n, a, p.tab, p.arena, p.g, p.v, p.T) : 0.f;
  }
}

// B rows of output column n = tile * 128 + row for every group of the batch: s_B[q][row] (bf16 bits), q = the
// group's rank-row offset + k.  Out of line (called once per tile): keeps the kernel's executed code small.
// canon (64-token tiles, one adapter, <= 16 rows): the 16 rows are written in the MN-major no-swizzle operand
// layout of the tensor-core expand, (n, q) at element (q/8)*1024 + (n/8)*64 + (q%8)*8 + n%8, zeros past lrows.
__device__ __noinline__ void dec_stage_B(const DecParams* pp, int tile, int row, int lrows, int ngroups,
                                         const int* s_gq0, const long long* s_goff, uint16_t* s_B, int canon) {
  const DecParams& p = *pp;
  const int n = tile * kDecBM + row;
  const int jn = dec_slice_of(p.g, min(n, p.M - 1));
  const int lo = p.g.e_lo[jn], hi = p.g.e_hi[jn], ldb = hi - lo;
  const bool in = n < p.M && n >= lo && n < hi;
  if (canon) {
    uint16_t b[16];
#pragma unroll
    for (int q = 0; q < 16; ++q)
      b[q] = (q < lrows && in) ? __ldg(reinterpret_cast<const uint16_t*>(p.arena + s_goff[3 + jn]) + (size_t)q * ldb + (n - lo))
                               : (uint16_t)0;
#pragma unroll
    for (int q = 0; q < 16; ++q) s_B[(q >> 3) * 1024 + (row >> 3) * 64 + (q & 7) * 8 + (row & 7)] = b[q];
    return;
  }
  for (int q0 = 0; q0 < lrows; q0 += 8) {  // 8 independent loads in flight, then 8 stores
    uint16_t b[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int q = q0 + e;
      b[e] = 0;
      if (q < lrows && in) {
        int g = 0;
        while (g + 1 < ngroups && s_gq0[g + 1] <= q) ++g;
        const uint16_t* Bp = reinterpret_cast<const uint16_t*>(p.arena + s_goff[g * 6 + 3 + jn]);
        b[e] = __ldg(Bp + (size_t)(q - s_gq0[g]) * ldb + (n - lo));
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (q0 + e < lrows) s_B[(q0 + e) * kDecBM + row] = b[e];
  }
}

// v_seg[t][j] . B_{a,j}[:, n] over the adapter's rs rank rows (K-local expand of one token)
__device__ __forceinline__ float dec_dot(const float* vs, const uint16_t* sb, int rs) {
  float s0 = 0.f;
  for (int k = 0; k < rs; ++k) s0 = fmaf(vs[k], bf16_bits_to_f32(sb[k * kDecBM]), s0);
  return s0;
}

// v_seg[t][0..15] . b[0..15] (rows past r/N are zero on both sides), two interleaved accumulators
__device__ __forceinline__ float dec_dot16(const float* vs, const float (&bq)[16]) {
  const float4* v4 = reinterpret_cast<const float4*>(vs);
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 a = v4[q];
    s0 = fmaf(a.x, bq[4 * q], s0);
    s1 = fmaf(a.y, bq[4 * q + 1], s1);
    s0 = fmaf(a.z, bq[4 * q + 2], s0);
    s1 = fmaf(a.w, bq[4 * q + 3], s1);
  }
  return s0 + s1;
}

// lora == 3: s v[t][j] . B[:, n] over the expand rank re, v [C][T][J][Rc] fp32 (rank row k = c * re/C + kk)
__device__ __forceinline__ float dec_vdot(const DecParams& p, int t, int j, const uint16_t* sb, int re) {
  const int C = p.g.C, rc = re / C;
  float s0 = 0.f;
  for (int c = 0; c < C; ++c) {
    const float* vv = p.v + ((size_t)(c * p.T + t) * p.g.J + j) * p.g.Rc;
    for (int kk = 0; kk < rc; ++kk) s0 = fmaf(__ldg(vv + kk), bf16_bits_to_f32(sb[(c * rc + kk) * kDecBM]), s0);
  }
  return s0;
}

// LM: 1 = K-local LoRA (BD / NFS: lora modes 0, 1), 2 = v precomputed (S-LoRA: modes 2, 3).  PUSH: fused row
// all-reduce output (LM == 1 only).  Separate instantiations keep each path's code and registers its own.
template <int S, bool CL, int LM, bool PUSH, int BN = 16>
__global__ void __launch_bounds__(kDecThreads, (S > 5 || BN > 16 ? 1 : 2))
    dec_lora_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                         const __grid_constant__ CUtensorMap tmA, const __grid_constant__ DecParams p) {
  using L = DecSmem<S, CL, BN, LM>;
  static_assert(BN == 16 || BN == 64, "token tile");
  static_assert(LM != 3 || (BN == 64 && !PUSH), "multi-adapter expand: BN = 64 tiles");
  static_assert(!PUSH || LM == 1, "the fused all-reduce serves the K-local (BD / NFS) path");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sW = smem + L::kWOff;
  uint8_t* sX = smem + L::kXOff;
  uint64_t* full = (uint64_t*)(smem + L::kBarOff);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = (uint32_t*)(tempty + 2);
  int* s_last = (int*)(tmem_holder + 1);
  int* mi = (int*)(smem + L::kMiscOff);
  int* s_ids = mi;
  int* s_grp = mi + 960;  // [64]
  int* s_gad = mi + 32;
  int* s_grs = mi + 48;
  int* s_gq0 = mi + 64;
  int* s_gmask = mi + 80;
  float* s_gsc = (float*)(mi + 128);
  long long* s_goff = (long long*)(mi + 160);  // [g][0..2] = offA[j], [g][3..5] = offB[j]
  float* s_vs = (float*)(smem + L::kVsOff);
  float* s_red = (float*)(mi + 512);             // [4 warps][32] cross-warp partial dots
  int* s_gtok = mi + 640;                         // [group][16] member tokens in token order
  // producer's tensor-core-shrink decision (read by the MMA warp); LM 3: past the group tables
  int* s_tcflag = L::kMt ? mi + (L::kMiscBytes / 4 - 4) : mi + 900;
  uint16_t* s_B = (uint16_t*)(smem + L::kBOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cta = blockIdx.x;
  const int UNITS = p.units, GRID = p.grid;
  const int u_lo = dec_u_lo(cta, UNITS, GRID);
  const int u_hi = dec_u_lo(cta + 1, UNITS, GRID);
  if (threadIdx.x == 0) {
    DEC_TRACE(0);
    if (p.trace) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p.trace[(size_t)blockIdx.x * 32 + 31] = smid;
    }
  }

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
    if (L::kMt || (LM == 1 && BN == 64)) ptx::mbar_init(reinterpret_cast<uint64_t*>(smem + L::kBarOff + 192), 1);
    ptx::fence_mbar_init();
    ptx::fence_proxy_async();
  }
  if (warp == 1) ptx::tmem_alloc<L::kTmemCols>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  // cluster split-K: a CTA may write a peer's shared memory only once the peer runs -- arrive now, wait
  // before the first push (long after: free)
  if (CL) ptx::cluster_arrive_relaxed();
  // the next kernel may launch now: it only takes SM room this grid leaves free, and waits for this grid's
  // completion (griddepcontrol.wait) before touching anything this grid writes
  if (threadIdx.x == 0) ptx::pdl_launch_dependents();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Does the batch hold ONE adapter (plus id -1 tokens)?  The whole warp reads the <= 64 ids at once
    // (a = the first non-negative id in token order, single = every non-negative id equals it): a serial
    // scan by the elected thread would put up to 64 dependent L2 round trips before the first A box.
    int w_a = -1;
    bool w_single = true;
    if (L::kTcShrink && LM == 1 && p.lora == 1 && p.tc_shrink) {
      const int id0 = (lane < BN && lane < p.T) ? __ldg(p.ids + lane) : -1;
      const int id1 = (lane + 32 < BN && lane + 32 < p.T) ? __ldg(p.ids + lane + 32) : -1;
      const unsigned m0 = __ballot_sync(0xffffffffu, id0 >= 0), m1 = __ballot_sync(0xffffffffu, id1 >= 0);
      const int s0 = __shfl_sync(0xffffffffu, id0, m0 ? __ffs(m0) - 1 : 0);
      const int s1 = __shfl_sync(0xffffffffu, id1, m1 ? __ffs(m1) - 1 : 0);
      w_a = m0 ? s0 : (m1 ? s1 : -1);
      w_single = __all_sync(0xffffffffu, (id0 < 0 || id0 == w_a) && (id1 < 0 || id1 == w_a)) != 0;
    }
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
      // Tensor-core K-local shrink (CL): when the batch holds ONE adapter (plus id -1 tokens) of local rank
      // <= 16 and the tile lies in one slice, that adapter's 16-row A box of the same K block rides every
      // stage and the MMA warp accumulates v_seg = A_seg X_seg^T in TMEM.  Same rule as the epilogue's.
      // ids and the slot table are read before the dependency (bdlora_set_pdl contract).
      bool use_tc = false;
      int arow_j[kMaxSlices] = {0, 0, 0};  // the adapter's first A row of each slice (arena row coordinate)
      // a CTA of a stream-K grid may own tiles of different slices (every tile inside one slice): the box row
      // follows the tile of each stage
      auto arow_of = [&](int u) {
        const int j = dec_slice_of(p.g, (u / p.k_blocks) * kDecBM);
        return j == 0 ? arow_j[0] : j == 1 ? arow_j[1] : arow_j[2];
      };
      if (L::kTcShrink && LM == 1 && p.lora == 1 && p.tc_shrink && nu > 0) {
        const int a = w_a;
        const bool single = w_single;
        const int n0 = (u_lo / p.k_blocks) * kDecBM;
        const int jlo = dec_slice_of(p.g, n0), jhi = dec_slice_of(p.g, min(n0 + kDecBM, p.M) - 1);
        if (single && a >= 0 && jlo == jhi) {
          const SlotEntry e = p.tab[a];
          if (e.rs <= 16) {
            use_tc = true;
#pragma unroll
            for (int j = 0; j < kMaxSlices; ++j) arow_j[j] = j < p.g.J ? (int)(e.offA[j] / p.K) : 0;
          }
        }
        if (use_tc)
          for (int idx = 0; idx < P; ++idx) {
            const int u = u_lo + idx, kb = u - (u / p.k_blocks) * p.k_blocks;
            ptx::mbar_expect_tx(&full[idx], L::kA);
            ptx::tma_load_2d(sA + idx * L::kA, &tmA, &full[idx], kb * kDecBK, arow_of(u), pol_x);
          }
      }
      *s_tcflag = use_tc ? 1 : 0;  // published to the MMA warp by the arrivals on full[] below
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
        ptx::mbar_arrive_expect_tx(&full[stage], L::kW + L::kX + (use_tc ? L::kA : 0));
        ptx::tma_load_2d(sW + stage * L::kW, &tmW, &full[stage], kb * kDecBK, tile * kDecBM, pol_w);
        ptx::tma_load_2d(sX + stage * L::kX, &tmX, &full[stage], kb * kDecBK, 0, pol_x);
        if (use_tc) ptx::tma_load_2d(sA + stage * L::kA, &tmA, &full[stage], kb * kDecBK, arow_of(u), pol_x);
        if (++stage == NS) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(kDecBM, BN);
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
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (u == u_lo && kb == kb0) DEC_TRACE(2);
          const uint64_t a_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sW + stage * L::kW));
          const uint64_t b_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sX + stage * L::kX));
#pragma unroll
          for (int k = 0; k < kDecBK / 16; ++k)
            ptx::mma_bf16(d_tmem, a_desc + 2 * k, b_desc + 2 * k, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          if (L::kTcShrink && *s_tcflag) {  // K-local shrink: V[k][t] += A_a[k][kb] . X[t][kb]  (lanes >= r/N ignored)
            const uint64_t s_desc = ptx::sdesc_k_sw128(ptx::smem_u32(sA + stage * L::kA));
#pragma unroll
            for (int k = 0; k < kDecBK / 16; ++k)
              ptx::mma_bf16(tmem_base + (uint32_t)(L::kVCol + acc * BN), s_desc + 2 * k, b_desc + 2 * k, idesc,
                            (kb > kb0 || k > 0) ? 1u : 0u);
          }
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
    // ---- adapter groups of the batch (distinct ids, order of first appearance) -------------------------
    // Read BEFORE the programmatic-dependency wait: ids, the slot table and the adapter factors are not
    // written by the kernel immediately preceding a forward (include/bdlora.h, bdlora_set_pdl), so the LoRA
    // metadata, the first tile's B rows and an L2 prefetch of the first segment's A rows all overlap the
    // preceding kernel's tail; after the wait only X (L2-resident) is still to be read.
    // lora == 3 (v precomputed, staged): the same groups, with the EXPAND rank re as the rank rows
    const bool lgrp = (LM == 1 && p.lora == 1) || (LM == 2 && p.lora == 3);
    if (BN == 64 && lgrp) {
      // T <= 64 decode tiles are served only for pools holding ONE adapter (host: capacity == 1), so the batch
      // has at most one group: the tokens with id >= 0
      if (we == 0) {
        const int id0 = (lane < T) ? __ldg(p.ids + lane) : -1;
        const int id1 = (lane + 32 < T) ? __ldg(p.ids + lane + 32) : -1;
        s_grp[lane] = id0 >= 0 ? 0 : -1;
        s_grp[lane + 32] = id1 >= 0 ? 0 : -1;
        const unsigned m0 = __ballot_sync(0xffffffffu, id0 >= 0), m1 = __ballot_sync(0xffffffffu, id1 >= 0);
        int a = -1;
        if (m0) a = __shfl_sync(0xffffffffu, id0, __ffs(m0) - 1);
        else if (m1) a = __shfl_sync(0xffffffffu, id1, __ffs(m1) - 1);
        if (lane == 0) {
          int rows = 0;
          if (a >= 0) {
            const SlotEntry e = p.tab[a];
            rows = min(LM == 2 ? e.re : e.rs, kDecLoraRows);
            s_gad[0] = a;
            s_gsc[0] = e.scale;
            s_grs[0] = rows;
            s_gq0[0] = 0;
#pragma unroll
            for (int j = 0; j < kMaxSlices; ++j) {
              s_goff[j] = e.offA[j];
              s_goff[3 + j] = e.offB[j];
            }
          }
          mi[96] = a >= 0 ? 1 : 0;
          mi[97] = rows;
        }
      }
      ptx::named_bar_sync(1, 128);
    } else if (lgrp) {
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
          rs = min(LM == 2 ? e.re : e.rs, kDecLoraRows);
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
        unsigned lrest = lmask;
        for (int gg = 0; gg < ng; ++gg) {  // member mask and member list of every group (warp-uniform loop)
          const int leader = __ffs(lrest) - 1;
          lrest &= lrest - 1;
          const int target = __shfl_sync(0xffffffffu, id, leader);
          const bool mem = id >= 0 && id == target;
          const unsigned m = __ballot_sync(0xffffffffu, mem);
          if (lane == 0) s_gmask[gg] = (int)m;
          if (mem) s_gtok[gg * 16 + __popc(m & ((1u << lane) - 1u))] = lane;
        }
        if (lane == 0) {
          mi[96] = ng;
          mi[97] = min(tot, kDecLoraRows);
        }
      }
      ptx::named_bar_sync(1, 128);
    }
    const int ngroups = lgrp ? mi[96] : 0;
    const int lrows = lgrp ? mi[97] : 0;
    int cur_tile = -1;
    auto stage_B = [&](int tile) {
      dec_stage_B(&p, tile, row, lrows, ngroups, s_gq0, s_goff, s_B, (BN == 64 && LM == 1) ? 1 : 0);
      cur_tile = tile;
    };
    if (lgrp && ngroups > 0 && u_lo < u_hi) {
      const int tile = u_lo / p.k_blocks;
      int kb0 = u_lo - tile * p.k_blocks;
      const int kb1 = min(p.k_blocks, kb0 + (u_hi - u_lo));
      stage_B(tile);
      if (LM == 2) kb0 = kb1;  // no A prefetch: v comes from the preceding kernel
      // L2 prefetch of the first segment's A rows (one bulk prefetch per row and slice)
      const int n0 = tile * kDecBM;
      const int jlo = dec_slice_of(p.g, n0), jhi = dec_slice_of(p.g, min(n0 + kDecBM, p.M) - 1);
      const int d_lo = kb0 * kDecBK, d_hi = min(p.K, kb1 * kDecBK);
      for (int it = etid; it < (jhi - jlo + 1) * lrows; it += 128) {
        const int jj = it / lrows, q = it - jj * lrows;
        int g = 0;
        while (g + 1 < ngroups && s_gq0[g + 1] <= q) ++g;
        ptx::prefetch_l2_bulk(p.arena + s_goff[g * 6 + jlo + jj] + (size_t)(q - s_gq0[g]) * p.K + d_lo,
                              (uint32_t)(d_hi - d_lo) * 2);
      }
    }
    // ---- LM 3: adapter groups of the batch; the first segment's first chunk of B rows staged before the wait
    DecGroups& G = *reinterpret_cast<DecGroups*>(mi);
    uint16_t* s_Bm = reinterpret_cast<uint16_t*>(smem + L::kBOff);
    // this contributor's share [qlo, qhi) of the tile's expand rows (every contributor of a split tile takes
    // a contiguous share: the LoRA term is linear and rides the split-K reduction)
    // downward-compatible COLUMN pool (g.bblk = m > 1, B_1 local = m diagonal blocks stored compactly as
    // [r/N_h, w]): a tile meets the diagonal blocks bb0 .. bb0 + nblk - 1 of its slice, and every group
    // contributes nblk x (its r/N_h) expand rows to it (v rows [bb0 r/N_h, (bb0 + nblk) r/N_h)); m = 1: one block
    const int bbk = p.g.bblk > 1 ? p.g.bblk : 1;
    auto tile_blocks = [&](int n0, int jt, int& bb0, int& nblk, int& blkw) {
      const int c0 = p.g.col0[jt], w = p.g.col0[jt + 1] - c0;
      blkw = w / bbk;
      bb0 = (n0 - c0) / blkw;
      nblk = (min(n0 + kDecBM, c0 + w) - 1 - c0) / blkw - bb0 + 1;
    };
    auto mt_range = [&](int u, int& tile, int& qlo, int& qhi) {
      tile = u / p.k_blocks;
      const int kb0 = u - tile * p.k_blocks, kb1 = min(p.k_blocks, kb0 + (u_hi - u));
      int ci = 0, ns = 1;
      if (CL) {
        ci = (int)ptx::cluster_ctarank();
        ns = p.cluster;
      } else if (!(kb0 == 0 && kb1 == p.k_blocks)) {
        const long long ts = (long long)tile * p.k_blocks;
        const int c_first = dec_cta_of(ts, UNITS, GRID), c_last = dec_cta_of(ts + p.k_blocks - 1, UNITS, GRID);
        ci = cta - c_first;
        ns = c_last - c_first + 1;
      }
      const int n0 = tile * kDecBM, jt = dec_slice_of(p.g, n0);
      int bb0, nblk, blkw;
      tile_blocks(n0, jt, bb0, nblk, blkw);
      const int qt = G.qtot / bbk * nblk;  // this tile's expand rows
      qlo = (int)((long long)qt * ci / ns);
      qhi = (int)((long long)qt * (ci + 1) / ns);
      if (n0 >= p.g.e_hi[jt] || n0 + kDecBM <= p.g.e_lo[jt]) qhi = qlo;  // tile outside the expand window
    };
    // rows [qa, qa + 64) of the share, this tile's 128 columns, into chunk buffer `buf` (zeros past the window)
    int mt_calls = 0;  // profiling stamps of the third call (chunk 2's rows)
    auto mt_stage = [&](int tile, int qa, int qhi, int buf) {
      const int n0 = tile * kDecBM, jt = dec_slice_of(p.g, n0);
      const int lo = p.g.e_lo[jt], hi = p.g.e_hi[jt], ldb = hi - lo;
      uint16_t* dst = s_Bm + buf * L::kMtRows * kDecBM;
      const int qb = min(qhi, qa + L::kMtRows), ng = G.ngroups;
      // the arena offset of each row's window start, once per row (one thread each), then 16 B per thread
      long long* rowoff = reinterpret_cast<long long*>(reinterpret_cast<uint8_t*>(mi) + L::kMtRowOff);
      int* rowblk = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(mi) + L::kMtRowOff + L::kMtRows * 8);
      int bb0, nblk, blkw;
      tile_blocks(n0, jt, bb0, nblk, blkw);
      if (etid < L::kMtRows) {
        const int q = qa + etid;
        long long o = -1;
        int blk = -1;
        if (q < qb && bbk == 1) {
          const int gq = dec_find_group(G.gq0, ng, q);
          o = G.goffB[gq][jt] + (long long)(q - G.gq0[gq]) * ldb - lo;
          blk = 0;
        } else if (q < qb) {
          // group: the last g whose first row in this tile's numbering, gq0[g] / m * nblk, is <= q
          int g0 = 0, g1 = ng - 1;
          while (g0 < g1) {
            const int mid = (g0 + g1 + 1) >> 1;
            if (G.gq0[mid] / bbk * nblk <= q) g0 = mid;
            else g1 = mid - 1;
          }
          const int qq = q - G.gq0[g0] / bbk * nblk, rbg = G.gre[g0] / bbk, bi = qq / rbg;
          blk = bb0 + bi;
          o = G.goffB[g0][jt] + (long long)(qq - bi * rbg) * ldb - lo;  // row qq - bi rbg of the compact B
        }
        rowoff[etid] = o;
        rowblk[etid] = blk;
      }
      ptx::named_bar_sync(1, 128);
      if (etid == 0 && mt_calls == 2) DEC_TRACE(10);
      const int c0s = p.g.col0[jt];
      for (int e = etid; e < L::kMtRows * 16; e += 128) {
        const int rq = e >> 4, nn = n0 + (e & 15) * 8;
        const long long o = rowoff[rq];
        // 8 columns of one row: inside the window and (m > 1) inside the row's own diagonal block
        const bool ok = o >= 0 && nn >= lo && nn < hi && (bbk == 1 || (nn - c0s) / blkw == rowblk[rq]);
        ptx::cp_async_16_zfill(dst + (rq >> 3) * 1024 + (e & 15) * 64 + (rq & 7) * 8, ok ? p.arena + o + nn : p.arena, ok);
      }
      ptx::cp_async_commit();
      if (etid == 0 && mt_calls++ == 2) DEC_TRACE(30);
      // the chunk's token list: (token, first expand row of its group inside the chunk, rows, chunk row offset)
      // for every token whose group's rows meet [qa, qb) -- built by the first two epilogue warps
      if (etid < 64) {
        int klo = 0, nr = 0, off = 0;
        const int gt = etid < T ? G.grp[etid] : -1;
        if (gt >= 0) {
          // the group's rows in this tile: [q0, q0 + nblk r/N_h), v rows from bb0 r/N_h on (m = 1: [0, r/N))
          const int q0 = bbk == 1 ? G.gq0[gt] : G.gq0[gt] / bbk * nblk, rbg = bbk == 1 ? G.gre[gt] : G.gre[gt] / bbk;
          const int qlo2 = max(qa, q0), qhi2 = min(qb, q0 + nblk * rbg);
          if (qlo2 < qhi2) {
            klo = bb0 * rbg + (qlo2 - q0);
            nr = qhi2 - qlo2;
            off = qlo2 - qa;
          }
        }
        const unsigned m = __ballot_sync(0xffffffffu, nr > 0);
        const int w = etid >> 5;
        int4* lst = reinterpret_cast<int4*>(reinterpret_cast<uint8_t*>(mi) + L::kMtListOff) + (buf * 2 + w) * 32;
        if (nr > 0) lst[__popc(m & ((1u << (etid & 31)) - 1u))] = make_int4(etid, klo, nr, off);
        if ((etid & 31) == 0) mi[(L::kMtListOff + 2 * 2 * 32 * 16) / 4 + buf * 2 + w] = __popc(m);
      }
    };
    bool mt_pre = false;
    uint64_t* lbar = reinterpret_cast<uint64_t*>(smem + L::kBarOff + 192);  // LM 3: expand MMAs of a chunk done
    uint32_t lphase = 0;
    bool has_lr = false;
    if constexpr (L::kMt) {
      dec_groups64(G, p.ids, T, p.tab, etid, [] { ptx::named_bar_sync(1, 128); });
      if (etid == 0) DEC_TRACE(13);
      if (u_lo < u_hi) {
        int tile, qlo, qhi;
        mt_range(u_lo, tile, qlo, qhi);
        if (qlo < qhi) {
          mt_stage(tile, qlo, qhi, 0);
          if (qhi - qlo > L::kMtRows) {
            ptx::named_bar_sync(1, 128);  // every thread is past the first call's row-table reads
            mt_stage(tile, qlo + L::kMtRows, qhi, 1);
          }
          mt_pre = true;
        }
      }
    }
    if (p.pdl) ptx::pdl_wait();  // X (and v) of the preceding kernel are visible; orders our Y writes
    const int par = PUSH ? *p.peer.parity : 0;
    long long vs_key = -1;       // (slice range, K range) whose v_seg s_vs holds

    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = u_lo; u < u_hi;) {
      const int tile = u / p.k_blocks;
      const int kb0 = u - tile * p.k_blocks;
      const int kb1 = min(p.k_blocks, kb0 + (u_hi - u));
      const bool whole = (kb0 == 0 && kb1 == p.k_blocks);
      const int n0 = tile * kDecBM;
      const int n = n0 + row;
      const int jlo = dec_slice_of(p.g, n0);
      const int jn = dec_slice_of(p.g, min(n, p.M - 1));
      float lr[16];  // LoRA term of the current 16-token chunk (BN == 16: the whole tile)
#pragma unroll
      for (int i = 0; i < 16; ++i) lr[i] = 0.f;
      // tensor-core K-local shrink taken by the producer (same rule): v_seg arrives in TMEM with the accumulator
      const bool tc = L::kTcShrink && LM == 1 && p.tc_shrink && p.lora == 1 && ngroups == 1 && s_grs[0] <= 16 &&
                      jlo == dec_slice_of(p.g, min(n0 + kDecBM, p.M) - 1);
      if constexpr (BN == 16) if (LM == 1 && p.lora == 1 && ngroups > 0 && !tc) {
        // ---- K-local shrink of this segment: v_seg[t][j][k] = s_a sum_{d in seg} X[t][d] A_{a,j}[k][d] -----
        // Thread per 16-byte chunk of the K range, 8 rank rows x 4 tokens per pass: 12 independent loads in
        // flight per chunk (the A rows are L2-resident, X was just written by the preceding kernel), then a
        // fixed-order reduction over the 128 threads.  Whole tiles of one slice reuse the previous v_seg.
        const int jhi = dec_slice_of(p.g, min(n0 + kDecBM, p.M) - 1);
        const int nj = jhi - jlo + 1;
        const int d_lo = kb0 * kDecBK, d_hi = min(p.K, kb1 * kDecBK);
        const long long key = (((long long)(jlo * 4 + nj) * 65536 + kb0) * 65536) + kb1;
        ptx::named_bar_sync(1, 128);  // previous segment's readers of s_vs / s_B are done
        if (key != vs_key) {
          vs_key = key;
          const int nch = (d_hi - d_lo) >> 3;
#pragma unroll 1
          for (int jj = 0; jj < nj; ++jj) {
#pragma unroll 1
            for (int g = 0; g < ngroups; ++g) {
              const unsigned gm = (unsigned)s_gmask[g];
              const int R = s_grs[g], ntok = __popc(gm);
              const float sc = s_gsc[g];
              const __nv_bfloat16* Ag = p.arena + s_goff[g * 6 + jlo + jj];
#pragma unroll 1
              for (int rb = 0; rb < R; rb += 8) {
#pragma unroll 1
                for (int tb = 0; tb < ntok; tb += 4) {
                  // rows past R and tokens past the group re-read a valid row / token (an L1 hit) and are
                  // dropped at the write: the loop body has no data-dependent branches (one code version)
                  int tok[4];
                  const __nv_bfloat16* xr[4];
                  const __nv_bfloat16* ar[8];
#pragma unroll
                  for (int qq = 0; qq < 4; ++qq) {
                    tok[qq] = (tb + qq < ntok) ? s_gtok[g * 16 + tb + qq] : -1;
                    xr[qq] = p.X + (size_t)(tok[qq] >= 0 ? tok[qq] : s_gtok[g * 16]) * p.K + d_lo;
                  }
#pragma unroll
                  for (int r = 0; r < 8; ++r) ar[r] = Ag + (size_t)min(rb + r, R - 1) * p.K + d_lo;
                  float a32[8][4];
#pragma unroll
                  for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) a32[r][qq] = 0.f;
#pragma unroll 1
                  for (int c = etid; c < nch; c += 128) {
                    uint4 av[8], xv[4];
#pragma unroll
                    for (int r = 0; r < 8; ++r) av[r] = ld_cached_u4(ar[r] + c * 8);
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) xv[qq] = ld_cached_u4(xr[qq] + c * 8);
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) {
                      float xf[8];
                      bf16x8_to_f32(xv[qq], xf);
#pragma unroll
                      for (int r = 0; r < 8; ++r) {
                        float af[8];
                        bf16x8_to_f32(av[r], af);
#pragma unroll
                        for (int e = 0; e < 8; ++e) a32[r][qq] = fmaf(af[e], xf[e], a32[r][qq]);
                      }
                    }
                  }
                  // transpose reduction over the warp: after 5 halving steps (31 shuffles) lane l holds the
                  // warp's sum of value l = r * 4 + qq
                  float vv[32];
#pragma unroll
                  for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int qq = 0; qq < 4; ++qq) vv[r * 4 + qq] = a32[r][qq];
#pragma unroll
                  for (int o = 16, c = 32; o >= 1; o >>= 1, c >>= 1) {
                    const bool up = (lane & o) != 0;
#pragma unroll
                    for (int i = 0; i < c / 2; ++i) {
                      const float send = up ? vv[i] : vv[i + c / 2];
                      const float keep = up ? vv[i + c / 2] : vv[i];
                      vv[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                    }
                  }
                  s_red[we * 32 + lane] = vv[0];
                  ptx::named_bar_sync(1, 128);
                  if (etid < 32) {
                    const int r = etid >> 2, qq = etid & 3;
                    if (rb + r < R && tok[qq] >= 0) {
                      const float sm = (s_red[etid] + s_red[32 + etid]) + (s_red[64 + etid] + s_red[96 + etid]);
                      s_vs[(tok[qq] * 3 + jj) * kDecLoraRows + rb + r] = sc * sm;
                    }
                  }
                  ptx::named_bar_sync(1, 128);  // s_red free again
                }
              }
            }
          }
        }
        if (tile != cur_tile) stage_B(tile);
        ptx::named_bar_sync(1, 128);
        // ---- expand: lr[t] = v_seg[t][j] . B_{a(t),j}[:, n] ---------------------------------------------
        const int jj = jn - jlo;
        if (T == 1) {  // straight-line batch-1 path (see the tensor-core expand below)
          const int g = s_grp[0];
          if (g >= 0) lr[0] = dec_dot(s_vs + jj * kDecLoraRows, s_B + s_gq0[g] * kDecBM + row, s_grs[g]);
        } else {
#pragma unroll
          for (int t = 0; t < kDecBN; ++t) {
            if (t < T) {
              const int g = s_grp[t];
              if (g >= 0)
                lr[t] = dec_dot(s_vs + (t * 3 + jj) * kDecLoraRows, s_B + s_gq0[g] * kDecBM + row, s_grs[g]);
            }
          }
        }
      }
      // lora == 3 (v precomputed, B staged): the tile's LoRA term is added by ONE contributor (whole tile;
      // cluster rank 0; the split tile's first contributor)
      const bool v3 = LM == 2 && p.lora == 3 && ngroups > 0 &&
                      (whole || (CL ? ptx::cluster_ctarank() == 0
                                    : cta == dec_cta_of((long long)tile * p.k_blocks, UNITS, GRID)));
      if (LM == 2 && p.lora == 3 && ngroups > 0 && tile != cur_tile) stage_B(tile);
      if constexpr (L::kMt) {
        // ---- LM 3: LR[n][t] = sum over this share's rows q of B_{g(q)}[k(q)][n] V[t][q], V[t][q] = v[t][k(q)] when
        // token t belongs to group g(q), else 0 (matmul_4 / _6 of a precomputed v) -- on the tensor cores, per
        // 96-row chunk: A = the staged B rows (MN-major), B = V_hi + V_lo (bf16 split of fp32 v, K-major),
        // accumulated in TMEM columns [kLrCol, kLrCol + 64) beside the base accumulator
        int tl, qlo, qhi;
        mt_range(u, tl, qlo, qhi);
        const int nchk = (qhi - qlo + L::kMtRows - 1) / L::kMtRows;
        if (!mt_pre) {
          if (nchk > 0) mt_stage(tile, qlo, qhi, 0);
          if (nchk > 1) {
            ptx::named_bar_sync(1, 128);  // every thread is past the first call's row-table reads
            mt_stage(tile, qlo + L::kMtRows, qhi, 1);
          }
        }
        mt_pre = false;
        has_lr = nchk > 0;
        const int jt = jlo, C = p.g.C, J = p.g.J, Rc = p.g.Rc;
        const int4* lst = reinterpret_cast<const int4*>(reinterpret_cast<const uint8_t*>(mi) + L::kMtListOff);
        const int* lcnt = mi + (L::kMtListOff + 2 * 2 * 32 * 16) / 4;
        uint8_t* vop = smem + L::kVOpOff;
        if (u == u_lo && etid == 0) DEC_TRACE(14);
        for (int ch = 0; ch < nchk; ++ch) {
          if (ch > 0) {  // the previous chunk's MMAs have read V and their B buffer
            ptx::mbar_wait(lbar, lphase);
            lphase ^= 1u;
            if (u == u_lo && etid == 0 && ch == 1) DEC_TRACE(5);
            if (ch + 1 < nchk) mt_stage(tile, qlo + (ch + 1) * L::kMtRows, qhi, (ch + 1) & 1);
          }
          if (u == u_lo && etid == 0 && ch < 7) DEC_TRACE(16 + 2 * ch);
          // V of this chunk: zero, then every listed token's rows (v fp32 -> bf16 hi + lo)
          {
            uint4* z = reinterpret_cast<uint4*>(vop);
            for (int i = etid; i < 2 * L::kVOpHalf / 16; i += 128) z[i] = make_uint4(0u, 0u, 0u, 0u);
          }
          ptx::named_bar_sync(1, 128);
          const int b = ch & 1, n0l = lcnt[b * 2], nl = n0l + lcnt[b * 2 + 1];
          for (int e = we; e < nl; e += 4) {  // a warp per listed token, lanes over its rows
            const int4 en = e < n0l ? lst[(b * 2) * 32 + e] : lst[(b * 2 + 1) * 32 + (e - n0l)];
            const int t = en.x, klo = en.y, nr = en.z, off = en.w;
            const int rc = C > 1 ? G.gre[G.grp[t]] / C : 1;
            for (int k = lane; k < nr; k += 32) {
              const int kk = klo + k;
              const int c = C > 1 ? kk / rc : 0, kr = C > 1 ? kk - c * rc : kk;
              const float val = __ldg(p.v + ((size_t)(c * T + t) * J + jt) * Rc + kr);
              const __nv_bfloat16 hi = __float2bfloat16_rn(val);
              const __nv_bfloat16 lo = __float2bfloat16_rn(val - __bfloat162float(hi));
              const int q = off + k;
              const int o = (t >> 3) * (L::kMtRows / 8) * 128 + (q >> 3) * 128 + (t & 7) * 16 + (q & 7) * 2;
              *reinterpret_cast<__nv_bfloat16*>(vop + o) = hi;
              *reinterpret_cast<__nv_bfloat16*>(vop + L::kVOpHalf + o) = lo;
            }
          }
          if (ch + 1 < nchk) ptx::cp_async_wait_group<1>();  // this chunk's B rows (the next one may be in flight)
          else ptx::cp_async_wait_group<0>();
          ptx::fence_proxy_async();  // generic-proxy shared-memory writes -> visible to the tensor core
          ptx::named_bar_sync(1, 128);
          if (u == u_lo && etid == 0 && ch < 7) DEC_TRACE(17 + 2 * ch);
          if (etid == 0) {
            ptx::tc_fence_after();
            constexpr uint32_t idesc_mn = ptx::idesc_bf16_f32(kDecBM, BN) | (1u << 15);  // A operand MN-major
            const uint32_t a0 = ptx::smem_u32(s_Bm + b * L::kMtRows * kDecBM), v0 = ptx::smem_u32(vop);
            constexpr uint32_t kSboV = (L::kMtRows / 8) * 128;
            const uint32_t d = tmem_base + (uint32_t)L::kLrCol;
#pragma unroll
            for (int kk = 0; kk < L::kMtRows / 16; ++kk) {
              const uint64_t ad = ptx::sdesc_k_none(a0 + kk * 4096, /*LBO: q-group*/ 2048, /*SBO: n-group*/ 128);
              ptx::mma_bf16(d, ad, ptx::sdesc_k_none(v0 + kk * 256, 128, kSboV), idesc_mn, (ch > 0 || kk > 0) ? 1u : 0u);
              ptx::mma_bf16(d, ad, ptx::sdesc_k_none(v0 + L::kVOpHalf + kk * 256, 128, kSboV), idesc_mn, 1u);
            }
            ptx::mma_commit(lbar);
          }
        }
        if (nchk > 0) {  // the tile's LoRA terms are in TMEM
          ptx::mbar_wait(lbar, lphase);
          lphase ^= 1u;
          ptx::tc_fence_after();
        }
        if (u == u_lo && etid == 0) DEC_TRACE(15);
      }
      if (u == u_lo && etid == 0) DEC_TRACE(3);
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      if (u == u_lo && etid == 0) DEC_TRACE(4);
      if (tc) {
        // v_seg (TMEM lanes k < r/N of the shrink accumulator, read by the lane-quarter-0 warp) -> s_vs.  A CTA
        // of a stream-K grid owns several segments: every reader of the previous segment's s_vs is done first,
        // and this tile's B rows replace the previous tile's (each thread stages and reads only its own column)
        if (tile != cur_tile) stage_B(tile);
        ptx::named_bar_sync(1, 128);
        if constexpr (BN == 64) {
          // 64-token tiles: the expand on the tensor cores, straight into the tile's accumulator --
          // acc += B_rows^T (MN-major, staged canonically) x V^T, V[t][k] = s v_seg[k][t] split into bf16 hi + lo,
          // zero for tokens with id -1 (their v_seg is real) and for rows k >= r/N
          // v_seg: TMEM lanes 0..15 (the lane-quarter-0 warp) -> fp32 staging, then all 128 threads build V
          float* vst = reinterpret_cast<float*>(s_vs) + 1024;  // [16 k][64 t] fp32, behind the 4 KB of V
          uint8_t* vop = reinterpret_cast<uint8_t*>(s_vs);
          if (q4 == 0) {
#pragma unroll
            for (int c0 = 0; c0 < BN; c0 += 16) {
              uint32_t v16[16];
              ptx::tmem_ld_32x32b_x16(tmem_base + (uint32_t)(L::kVCol + acc * BN + c0), v16);
              ptx::tmem_ld_wait();
              if (lane < 16) {
#pragma unroll
                for (int tt = 0; tt < 16; tt += 4)
                  *reinterpret_cast<float4*>(vst + lane * 64 + c0 + tt) =
                      make_float4(__uint_as_float(v16[tt]), __uint_as_float(v16[tt + 1]), __uint_as_float(v16[tt + 2]),
                                  __uint_as_float(v16[tt + 3]));
              }
            }
          }
          ptx::named_bar_sync(1, 128);
          {
            const int rs = s_grs[0];
            const float sc = s_gsc[0];
#pragma unroll
            for (int e = 0; e < 8; ++e) {  // 1024 (token, row) values, 8 per thread
              const int idx = etid + 128 * e, t = idx & 63, k = idx >> 6;
              const float val = (k < rs && s_grp[t] == 0) ? sc * vst[k * 64 + t] : 0.f;
              const __nv_bfloat16 hi = __float2bfloat16_rn(val);
              const __nv_bfloat16 lo = __float2bfloat16_rn(val - __bfloat162float(hi));
              const int o = (t >> 3) * 256 + (k >> 3) * 128 + (t & 7) * 16 + (k & 7) * 2;
              *reinterpret_cast<__nv_bfloat16*>(vop + o) = hi;
              *reinterpret_cast<__nv_bfloat16*>(vop + 2048 + o) = lo;
            }
          }
          ptx::fence_proxy_async();  // B rows and V (generic-proxy writes) -> visible to the tensor core
          ptx::named_bar_sync(1, 128);
          if (etid == 0) {
            ptx::tc_fence_after();
            constexpr uint32_t idesc_mn = ptx::idesc_bf16_f32(kDecBM, BN) | (1u << 15);  // A operand MN-major
            const uint64_t ad = ptx::sdesc_k_none(ptx::smem_u32(s_B), /*LBO: q-group*/ 2048, /*SBO: n-group*/ 128);
            const uint32_t d = tmem_base + (uint32_t)(acc * BN);
            ptx::mma_bf16(d, ad, ptx::sdesc_k_none(ptx::smem_u32(vop), 128, 256), idesc_mn, 1u);
            ptx::mma_bf16(d, ad, ptx::sdesc_k_none(ptx::smem_u32(vop + 2048), 128, 256), idesc_mn, 1u);
            ptx::mma_commit(lbar);
          }
          ptx::mbar_wait(lbar, lphase);
          lphase ^= 1u;
          ptx::tc_fence_after();
        } else if (q4 == 0) {
          const int rs = s_grs[0];
          const float sc = s_gsc[0];
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v16[16];
            ptx::tmem_ld_32x32b_x16(tmem_base + (uint32_t)(L::kVCol + acc * BN + c0), v16);
            ptx::tmem_ld_wait();
            if (lane < 16) {  // rows rs..15 are written as zeros (dec_dot16 reads all 16)
#pragma unroll
              for (int t = 0; t < 16; ++t) s_vs[(c0 + t) * L::kVsTok + lane] = lane < rs ? sc * __uint_as_float(v16[t]) : 0.f;
            }
          }
        }
        ptx::named_bar_sync(1, 128);
        if (etid == 0) DEC_TRACE(9);
      }
      // ---- per 16-token chunk: accumulator -> registers, + LoRA, out (store / DSMEM push / partial) ----------
      const int sc_cl = CL ? p.cluster : 1;
      const uint32_t crank = CL ? ptx::cluster_ctarank() : 0u;
      const int nr_max = (kDecBM + sc_cl - 1) / sc_cl;
      float* s_slot = reinterpret_cast<float*>(smem + L::kSlotOff);
      if (CL) {
        ptx::cluster_wait();  // (early arrival) every peer has started: DSMEM pushes below are legal
        if (etid == 0) DEC_TRACE(11);
      }
      const int slot = (tile * p.k_blocks > u_lo) ? 1 : 0;
      float* my_part = p.part + ((size_t)(cta * 2 + slot) * kDecBM + row) * BN;
      for (int c0 = 0; c0 < BN && c0 < T; c0 += 16) {
        uint32_t r[16];
        ptx::tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(acc * BN + c0), r);
        ptx::tmem_ld_wait();
        const int tn = min(16, T - c0);  // valid tokens of the chunk
        if (tc && BN == 16) {
          // this output column's B values of the adapter's rank rows in registers (zero past r/N), then one
          // 16-term dot per token against its v_seg row (broadcast 16-byte shared loads)
          float bq[16];
          const int rs = s_grs[0];
#pragma unroll
          for (int k = 0; k < 16; ++k) bq[k] = k < rs ? bf16_bits_to_f32(s_B[k * kDecBM + row]) : 0.f;
          if (BN == 16 && T == 1) {  // straight-line batch-1 path (no 16-way guarded unroll: i-cache)
            if (s_grp[0] == 0) lr[0] = dec_dot16(s_vs, bq);
          } else {
            // branch-free: all 16 dots are independent (their shared loads and FMAs interleave); tokens past T or
            // with id -1 are masked by a 0/1 factor (their v_seg rows are finite: zero-filled or real X rows)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float w = (i < tn && s_grp[c0 + i] == 0) ? 1.f : 0.f;
              lr[i] = w * dec_dot16(s_vs + (c0 + i) * L::kVsTok, bq);
            }
          }
        } else if (L::kMt && has_lr) {
          uint32_t l16[16];
          ptx::tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(L::kLrCol + c0), l16);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) lr[i] = i < tn ? __uint_as_float(l16[i]) : 0.f;
        } else if (v3) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int g = (i < tn) ? s_grp[c0 + i] : -1;
            lr[i] = g >= 0 ? dec_vdot(p, c0 + i, jn, s_B + s_gq0[g] * kDecBM + row, s_grs[g]) : 0.f;
          }
        }
        if (CL) {
          // cluster split-K: rank c owns rows [c*128/s, (c+1)*128/s); every contributor pushes its partial rows
          // into the owner's slots (DSMEM)
          const int owner = ((row + 1) * sc_cl - 1) / kDecBM;
          const int rr = row - (owner * kDecBM) / sc_cl;
          const uint32_t dst =
              ptx::mapa(ptx::smem_u32(s_slot + ((size_t)(crank * nr_max + rr) * L::kSlotStride + c0)), (uint32_t)owner);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (4 * q < tn)
              ptx::st_dsmem_f4(dst + q * 16, __uint_as_float(r[4 * q]) + lr[4 * q],
                               __uint_as_float(r[4 * q + 1]) + lr[4 * q + 1], __uint_as_float(r[4 * q + 2]) + lr[4 * q + 2],
                               __uint_as_float(r[4 * q + 3]) + lr[4 * q + 3]);
        } else if (whole) {
          if (LM == 2 && p.lora == 2 && n < p.M) {
            float lrv[16];
            dec_vmode_lr(&p, n, c0, tn, lrv);
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i < tn) lr[i] = lrv[i];
          }
          if (n < p.M) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (i < tn) dec_out<PUSH>(p, par, c0 + i, n, __uint_as_float(r[i]) + lr[i]);
          }
        } else {
          // split tile: this CTA's fp32 partial (its K range, with its K-local LoRA share), [row][BN]
          float4* my = reinterpret_cast<float4*>(my_part + c0);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (4 * q < tn)
              __stcg(my + q, make_float4(__uint_as_float(r[4 * q]) + lr[4 * q], __uint_as_float(r[4 * q + 1]) + lr[4 * q + 1],
                                         __uint_as_float(r[4 * q + 2]) + lr[4 * q + 2],
                                         __uint_as_float(r[4 * q + 3]) + lr[4 * q + 3]));
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);  // the accumulator was read: the MMA may reuse it
      if (CL) {
        // one cluster barrier, then the owner sums its rows over the contributors in rank order (deterministic)
        if (etid == 0) DEC_TRACE(12);
        ptx::cluster_arrive();  // release: my pushes
        ptx::cluster_wait();    // acquire: every peer's rows of my range
        if (etid == 0) DEC_TRACE(6);
        const int nq = (T + 3) >> 2;
        const int r_lo = (crank * kDecBM) / sc_cl, nr = ((crank + 1) * kDecBM) / sc_cl - r_lo;
        for (int f = etid; f < nr * nq; f += 128) {
          const int r2 = f % nr, qd = f / nr;
          float4 y = *reinterpret_cast<const float4*>(s_slot + (size_t)r2 * L::kSlotStride + qd * 4);
          for (int c = 1; c < sc_cl; ++c) {
            const float4 z = *reinterpret_cast<const float4*>(s_slot + ((size_t)(c * nr_max + r2) * L::kSlotStride + qd * 4));
            y.x += z.x, y.y += z.y, y.z += z.z, y.w += z.w;
          }
          const int nn = n0 + r_lo + r2;
          if (nn < p.M) {
            float yv[4] = {y.x, y.y, y.z, y.w};
            if (LM == 2 && p.lora == 2) {
              float lrv[16];
              dec_vmode_lr(&p, nn, qd * 4, min(4, T - qd * 4), lrv);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (qd * 4 + i < T) yv[i] += lrv[i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (qd * 4 + i < T) dec_out<PUSH>(p, par, qd * 4 + i, nn, yv[i]);
          }
        }
      } else if (!whole) {
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
          // finisher: contributors' partials summed in CTA order (deterministic), 8 contributors' loads in flight
          if (etid == 0) DEC_TRACE(6);
          const int c_last = dec_cta_of(ts + p.k_blocks - 1, UNITS, GRID);
          for (int c0 = 0; c0 < BN && c0 < T; c0 += 16) {
            const int tn = min(16, T - c0);
            float y[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float4 yq = make_float4(0.f, 0.f, 0.f, 0.f);
              if (4 * q < tn) {
                for (int cb = c_first; cb <= c_last; cb += 8) {
                  float4 b8[8];
#pragma unroll
                  for (int e = 0; e < 8; ++e) {
                    const int c = min(cb + e, c_last);
                    const int sl = (ts > dec_u_lo(c, UNITS, GRID)) ? 1 : 0;
                    b8[e] = __ldcg(reinterpret_cast<const float4*>(p.part + ((size_t)(c * 2 + sl) * kDecBM + row) * BN + c0) + q);
                  }
#pragma unroll
                  for (int e = 0; e < 8; ++e)
                    if (cb + e <= c_last) yq.x += b8[e].x, yq.y += b8[e].y, yq.z += b8[e].z, yq.w += b8[e].w;
                }
              }
              y[4 * q] = yq.x, y[4 * q + 1] = yq.y, y[4 * q + 2] = yq.z, y[4 * q + 3] = yq.w;
            }
            if (n < p.M) {
              if (LM == 2 && p.lora == 2) {
                float lrv[16];
                dec_vmode_lr(&p, n, c0, tn, lrv);
#pragma unroll
                for (int i = 0; i < 16; ++i)
                  if (i < tn) y[i] += lrv[i];
              }
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i < tn) dec_out<PUSH>(p, par, c0 + i, n, y[i]);
            }
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
    if (PUSH) {
      // every CTA signals every rank once, after all of its pushes: barrier, then a system-scope release
      ptx::named_bar_sync(1, 128);
      if (etid == 0) {
        __threadfence_system();
        for (int r2 = 0; r2 < p.peer.nranks; ++r2)
          asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.peer.cnt[r2] + par) : "memory");
      }
    }
  }
  if (warp == 0 && lane == 0) DEC_TRACE(8);  // producer done issuing
  if (CL && warp < 2) {  // the epilogue's cluster barriers count every thread of the CTA
    ptx::cluster_wait();
    ptx::cluster_arrive();
    ptx::cluster_wait();
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<L::kTmemCols>(tmem_base);
}

}  // namespace bdl
