// common.cuh -- device-side data structures shared by all bdlora kernels (sm_100a).
//
// Pool layout in HBM: one bf16 arena per pool; each loaded slot keeps
// only this device's shard of its factors, stored compactly (no zero of a block-diagonal factor is
// stored):
//   A_j : [rs, K]   rank-outermost, K contiguous  (the shrink streams whole 128-bit rows; a downward-
//         compatible ROW adapter keeps only its rows' own block: [rs, K/m])
//   B_j : [re, ldb_j] row-major, output columns contiguous (the expand epilogue reads a row of B
//         across consecutive output columns -> coalesced)
// and one 64-byte SlotEntry in a device table indexed by the adapter id.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bdl {

// Host: memo of the TMA tensor maps a forward encodes for its W and X ([rows, K] bf16, K-major, boxes of
// 64 x box_rows, 128B swizzle -- the only maps the launchers build per call).  The 128-byte map is a pure
// function of (base, K, rows, box_rows), so an eager caller that reuses its buffers skips
// cuTensorMapEncodeTiled (a CUDA graph bakes the maps in at capture anyway).  Per host thread, 64 entries,
// round-robin replacement.
struct TmapMemo {
  static constexpr int kN = 64;
  const void* base[kN];
  int K[kN], rows[kN], box[kN];
  CUtensorMap map[kN];
  int n = 0, next = 0;
};
inline TmapMemo& tmap_memo() {
  static thread_local TmapMemo m;
  return m;
}
inline bool tmap_memo_get(const void* base, int K, int rows, int box, CUtensorMap* out) {
  TmapMemo& m = tmap_memo();
  for (int i = 0; i < m.n; ++i)
    if (m.base[i] == base && m.K[i] == K && m.rows[i] == rows && m.box[i] == box) {
      *out = m.map[i];
      return true;
    }
  return false;
}
inline void tmap_memo_put(const void* base, int K, int rows, int box, const CUtensorMap& map) {
  TmapMemo& m = tmap_memo();
  const int i = m.n < TmapMemo::kN ? m.n++ : (m.next++ % TmapMemo::kN);
  m.base[i] = base;
  m.K[i] = K;
  m.rows[i] = rows;
  m.box[i] = box;
  m.map[i] = map;
}

constexpr int kMaxSlices = 3;

struct SlotEntry {
  long long offA[kMaxSlices];  // element offsets into the arena
  long long offB[kMaxSlices];
  int rs;       // shrink rank: rows of A_j on this device (BD: r/N, S-LoRA col: r/N, S-LoRA row: r)
  int re;       // expand rank: rows of B_j on this device (BD: r/N, S-LoRA: r)
  float scale;  // s_a
  int loaded;
};
static_assert(sizeof(SlotEntry) == 64, "SlotEntry must stay 64 bytes");

// Local geometry of one projection on one device.
struct Geom {
  int K;                  // input dim of X on this device
  int M;                  // output columns on this device (rows of W^T)
  int J;                  // slices
  int col0[kMaxSlices + 1];  // local column start of slice j; col0[J] = M
  int e_lo[kMaxSlices];   // expand window of slice j, absolute local columns [e_lo, e_hi)
  int e_hi[kMaxSlices];
  int Rc;                 // per-chunk rank capacity of v
  int C;                  // chunks of v read by the expand (S-LoRA column after all-gather: N)
  // downward-compatible serving: m = N_h / N local diagonal blocks per resident adapter, stored
  // compactly -- no zero is stored or read.  bblk = m for COLUMN pools (B_1 local = m blocks [r/N_h, w/m] side
  // by side: [r/N_h, w]), ablk = m for ROW pools (A_2 local = m blocks [d_in/N_h, r/N_h]: rank row q of block
  // q / (r/N_h) holds only its block's K/m inputs).  1 = native BD (one block per device).
  int ablk;
  int bblk;
};

// Profiling stamp inside lora_chunk16 (bdlora_debug_trace): %globaltimer into slot k of this CTA's trace row
// when a trace row is passed; one predicated branch otherwise.
#define LC_STAMP(k)                                                    \
  do {                                                                 \
    if (trace && etid == 0) {                                          \
      long long t_;                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)::"memory"); \
      trace[k] = t_;                                                   \
    }                                                                  \
  } while (0)

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float f[8]) {
  f[0] = __uint_as_float(u.x << 16);
  f[1] = __uint_as_float(u.x & 0xffff0000u);
  f[2] = __uint_as_float(u.y << 16);
  f[3] = __uint_as_float(u.y & 0xffff0000u);
  f[4] = __uint_as_float(u.z << 16);
  f[5] = __uint_as_float(u.z & 0xffff0000u);
  f[6] = __uint_as_float(u.w << 16);
  f[7] = __uint_as_float(u.w & 0xffff0000u);
}

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

// Streaming 128-bit load that does not allocate in L1 (weights are read exactly once).
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ld_cached_u4(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// LoRA expand term for output column n of token t:  sum_c sum_k v[c][t][j][k] * B_j[c*re/C + k][n - e_lo_j]
// (matmul_4 / matmul_6).  Returns 0 outside the expand window or for id -1.
__device__ __forceinline__ float lora_expand_term(int t, int n, int a, const SlotEntry* __restrict__ tab,
                                                  const __nv_bfloat16* __restrict__ arena, const Geom& g,
                                                  const float* __restrict__ v, int T) {
  if (a < 0) return 0.f;
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSlices; ++q)
    if (q < g.J && n >= g.col0[q]) j = q;
  if (n < g.e_lo[j] || n >= g.e_hi[j]) return 0.f;
  const SlotEntry& e = tab[a];
  const int ldb = g.e_hi[j] - g.e_lo[j];
  const int col = n - g.e_lo[j];
  const uint16_t* B = reinterpret_cast<const uint16_t*>(arena + e.offB[j]);
  const int rc = e.re / g.C;
  // 8 independent partial sums -> 16 loads in flight per thread (latency-bound: v is L2-resident,
  // B rows are read coalesced across the warp's consecutive output columns)
  float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int c = 0; c < g.C; ++c) {
    const float* vv = v + ((size_t)(c * T + t) * g.J + j) * g.Rc;
    const uint16_t* Bc = B + (size_t)(c * rc) * ldb + col;
    int k = 0;
    for (; k + 8 <= rc; k += 8) {
      float vk[8], bk[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        vk[q] = __ldg(vv + k + q);
        bk[q] = bf16_bits_to_f32(__ldg(Bc + (size_t)(k + q) * ldb));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) s8[q] = fmaf(vk[q], bk[q], s8[q]);
    }
    for (; k < rc; ++k) s8[0] = fmaf(__ldg(vv + k), bf16_bits_to_f32(__ldg(Bc + (size_t)k * ldb)), s8[0]);
  }
  return ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
}

// LoRA expand term for up to 16 consecutive tokens tb..tb+cnt-1 at output column n (matmul_4/6):
//   lr[i] = sum_c sum_k v[c][tb+i][j][k] * B_{a(tb+i),j}[c*re/C + k][n - e_lo_j]
// Tokens are grouped by adapter (s_lead[i] = index in [0,16) of the first token of this chunk with the
// same id, -1 for id -1; staged in shared memory) so each 16-row chunk of B is gathered once per
// DISTINCT adapter, 16 independent loads in flight; consecutive threads hold consecutive output
// columns, so every B row segment is read coalesced.  v values are loaded before use and reduced in
// 4 independent chains (no load->FMA latency chain).
// B rows of ONE adapter gathered ahead of time (decode fast path: the first 16-token chunk holds a single
// adapter group, C == 1, re <= 16) so only the v load remains once v is ready.
struct LoraPre {
  int a;            // adapter id, -1 = none
  int re;           // its expand rank (<= 16): with b, everything the expand needs -- no slot-table read later
  float b[16];      // the B rows (registers) -- unused when sb is set
  float* sb;        // optional shared-memory home of the B rows (sb[q * 128]): nothing long-lived in registers
};

__device__ __forceinline__ void lora_pre16(LoraPre& pre, int n, int cnt, const int* s_ids, const int* s_lead,
                                           const SlotEntry* __restrict__ tab,
                                           const __nv_bfloat16* __restrict__ arena, const Geom& g) {
  pre.a = -1;
  if (n >= g.M || g.C != 1) return;
  int lead = -1;
  for (int i = 0; i < cnt; ++i) {
    if (s_lead[i] < 0) continue;
    if (lead < 0) lead = s_lead[i];
    if (s_lead[i] != lead) return;  // more than one group: generic path
  }
  if (lead < 0) return;
  const int a = s_ids[lead];
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSlices; ++q)
    if (q < g.J && n >= g.col0[q]) j = q;
  if (n < g.e_lo[j] || n >= g.e_hi[j]) return;
  const int re = tab[a].re;
  if (re > 16) return;
  const int ldb = g.e_hi[j] - g.e_lo[j];
  const uint16_t* B = reinterpret_cast<const uint16_t*>(arena + tab[a].offB[j]) + (n - g.e_lo[j]);
  if (pre.sb) {
#pragma unroll
    for (int q = 0; q < 16; ++q) pre.sb[q * 128] = (q < re) ? bf16_bits_to_f32(__ldg(B + (size_t)q * ldb)) : 0.f;
  } else {
#pragma unroll
    for (int q = 0; q < 16; ++q) pre.b[q] = (q < re) ? bf16_bits_to_f32(__ldg(B + (size_t)q * ldb)) : 0.f;
  }
  pre.a = a;
  pre.re = re;
}

__device__ __forceinline__ void lora_chunk16(float (&lr)[16], int n, int tb, int cnt, const int* s_ids,
                                             const int* s_lead, const SlotEntry* __restrict__ tab,
                                             const __nv_bfloat16* __restrict__ arena, const Geom& g,
                                             const float* __restrict__ v, int T, LoraPre* pre = nullptr,
                                             float* s_v = nullptr, int s_v_cap = 0, int etid = 0,
                                             long long* trace = nullptr) {
#pragma unroll
  for (int i = 0; i < 16; ++i) lr[i] = 0.f;
  // Stage this chunk's v rows in shared memory (cooperatively, once) when they fit: the inner loop then
  // reads them with broadcast LDS instead of one global load per (token, rank) per thread.
  const int per_tok = g.J * g.Rc;
  const bool staged = s_v != nullptr && g.C * 16 * per_tok <= s_v_cap;
  if (staged) {
    asm volatile("bar.sync 1, 128;" ::: "memory");  // previous readers of s_v are done
    LC_STAMP(18);
    for (int c = 0; c < g.C; ++c) {
      const float* src = v + (size_t)(c * T + tb) * per_tok;
      float* dst = s_v + (size_t)c * 16 * per_tok;
      for (int idx = etid; idx < cnt * per_tok; idx += 128) dst[idx] = __ldg(src + idx);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    LC_STAMP(19);
  }
  if (n >= g.M) return;
  LC_STAMP(20);
  int j = 0;
#pragma unroll
  for (int q = 1; q < kMaxSlices; ++q)
    if (q < g.J && n >= g.col0[q]) j = q;
  if (n < g.e_lo[j] || n >= g.e_hi[j]) return;
  const int ldb = g.e_hi[j] - g.e_lo[j];
  const int col = n - g.e_lo[j];
  const unsigned full = (cnt >= 16) ? 0xffffu : ((1u << cnt) - 1u);
  LC_STAMP(21);
  for (int i = 0; i < cnt; ++i) {
    if (s_lead[i] != i) continue;  // not a group leader (or no adapter)
    const int a = s_ids[i];
    unsigned mask = 0;              // members of this group within the chunk (warp-uniform)
#pragma unroll
    for (int i2 = 0; i2 < 16; ++i2)
      if (i2 < cnt && s_lead[i2] == i) mask |= 1u << i2;
    LC_STAMP(22);
    const bool use_pre = pre && pre->a == a;  // pre-gathered (C == 1, re <= 16): no slot-table round trip
    const uint16_t* B = use_pre ? nullptr : reinterpret_cast<const uint16_t*>(arena + tab[a].offB[j]) + col;
    const int rc = use_pre ? pre->re : tab[a].re / g.C;
    for (int c = 0; c < g.C; ++c) {
      for (int k0 = 0; k0 < rc; k0 += 16) {
        float b[16];
        if (use_pre && c == 0 && k0 == 0) {
          if (pre->sb) {
#pragma unroll
            for (int q = 0; q < 16; ++q) b[q] = pre->sb[q * 128];
          } else {
#pragma unroll
            for (int q = 0; q < 16; ++q) b[q] = pre->b[q];
          }
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            b[q] = (k0 + q < rc) ? bf16_bits_to_f32(__ldg(B + (size_t)(c * rc + k0 + q) * ldb)) : 0.f;
          if (pre && g.C == 1 && rc <= 16) {  // keep for the next chunk of the same tile (same adapter)
            pre->a = a;
            pre->re = rc;
            if (pre->sb) {
#pragma unroll
              for (int q = 0; q < 16; ++q) pre->sb[q * 128] = b[q];
            } else {
#pragma unroll
              for (int q = 0; q < 16; ++q) pre->b[q] = b[q];
            }
          }
        }
        const bool vec = staged && (g.Rc & 3) == 0 && k0 + 16 <= rc;
        if (staged && cnt == 1 && mask == 1u) {
          // decode batch 1: one dot product (masked to the rank), small code on the critical tail
          const float* vv = s_v + ((size_t)(c * 16) * g.J + j) * g.Rc + k0;
          float s0 = 0.f, s1 = 0.f;
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
            s0 = fmaf(k0 + q < rc ? vv[q] : 0.f, b[q], s0);
            s1 = fmaf(k0 + q + 1 < rc ? vv[q + 1] : 0.f, b[q + 1], s1);
          }
          lr[0] += s0 + s1;
          LC_STAMP(23);
          continue;
        }
        if (vec && mask == full) {
          // one adapter for the whole chunk: branch-free, every LDS.128 independent (pipelined)
#pragma unroll
          for (int i2 = 0; i2 < 16; ++i2) {
            const float* vv = s_v + ((size_t)(c * 16 + i2) * g.J + j) * g.Rc + k0;
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
            for (int q = 0; q < 16; q += 4) {
              const float4 f4 = *reinterpret_cast<const float4*>(vv + q);
              s0 = fmaf(f4.x, b[q], s0);
              s1 = fmaf(f4.y, b[q + 1], s1);
              s2 = fmaf(f4.z, b[q + 2], s2);
              s3 = fmaf(f4.w, b[q + 3], s3);
            }
            if (i2 < cnt) lr[i2] += (s0 + s1) + (s2 + s3);
          }
          LC_STAMP(23);
          continue;
        }
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) {
          if ((mask >> i2) & 1u) {
            float vk[16];
            if (vec) {
              const float* vv = s_v + ((size_t)(c * 16 + i2) * g.J + j) * g.Rc + k0;
#pragma unroll
              for (int q = 0; q < 16; q += 4) {
                const float4 f4 = *reinterpret_cast<const float4*>(vv + q);
                vk[q] = f4.x;
                vk[q + 1] = f4.y;
                vk[q + 2] = f4.z;
                vk[q + 3] = f4.w;
              }
            } else if (staged) {
              const float* vv = s_v + ((size_t)(c * 16 + i2) * g.J + j) * g.Rc + k0;
#pragma unroll
              for (int q = 0; q < 16; ++q) vk[q] = (k0 + q < rc) ? vv[q] : 0.f;
            } else {
              const float* vv = v + ((size_t)(c * T + tb + i2) * g.J + j) * g.Rc + k0;
#pragma unroll
              for (int q = 0; q < 16; ++q) vk[q] = (k0 + q < rc) ? __ldg(vv + q) : 0.f;  // L1 broadcast
            }
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
            for (int q = 0; q < 16; q += 4) {
              s0 = fmaf(vk[q], b[q], s0);
              s1 = fmaf(vk[q + 1], b[q + 1], s1);
              s2 = fmaf(vk[q + 2], b[q + 2], s2);
              s3 = fmaf(vk[q + 3], b[q + 3], s3);
            }
            lr[i2] += (s0 + s1) + (s2 + s3);
          }
        }
      }
    }
  }
}

}  // namespace bdl
