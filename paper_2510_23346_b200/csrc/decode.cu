// decode.cu -- host side of the lean decode kernel (kernels_decode.cuh): grid / split policy, tensor maps,
// launch with programmatic dependent launch.  Its own translation unit (built in parallel with runtime.cu).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "decode.h"
#include "kernels_decode.cuh"

namespace bdl {

namespace {

constexpr int kMaxDev = 64;
thread_local int g_dec_last[8] = {-1, 0, 0, 0, 0, 0, 0, 0};
long long* g_dec_trace = nullptr;

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled encode_fn() {
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

// [rows, K] bf16 K-major, box [box_rows, 64], SWIZZLE_128B, out-of-range rows read as zeros
bool encode(CUtensorMap* m, const void* base, int K, int rows, int box_rows) {
  if (tmap_memo_get(base, K, rows, box_rows, m)) return true;
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)kDecBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  tmap_memo_put(base, K, rows, box_rows, *m);
  return true;
}

int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}

template <int S, bool CL, int LM, bool PUSH, int BN>
int launch_one(const DecParams& p, const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmA,
               cudaStream_t st) {
  using L = DecSmem<S, CL, BN, LM>;
  static bool attr[kMaxDev] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  dev = std::min(std::max(dev, 0), kMaxDev - 1);
  if (!attr[dev]) {
    if (cudaFuncSetAttribute(dec_lora_gemm_kernel<S, CL, LM, PUSH, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024) != cudaSuccess)
      return -1;
    if (CL && cudaFuncSetAttribute(dec_lora_gemm_kernel<S, CL, LM, PUSH, BN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
                  cudaSuccess)
      return -1;
    attr[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(kDecThreads);
  // BDLORA_DEC_SMEM_PAD=1 (experiments): request enough shared memory that only one CTA fits per SM
  static const int pad = env_int("BDLORA_DEC_SMEM_PAD", 0);
  cfg.dynamicSmemBytes = pad ? 200 * 1024 : L::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (CL) {
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = p.cluster;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.numAttrs = 2;
  }
  return cudaLaunchKernelEx(&cfg, dec_lora_gemm_kernel<S, CL, LM, PUSH, BN>, tmW, tmX, tmA, p) == cudaSuccess ? 0 : -1;
}

template <int S, bool CL>
int launch_stages(const DecParams& p, const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmA,
                  cudaStream_t st) {
  if (p.lora >= 2) return launch_one<S, CL, 2, false, 16>(p, tmW, tmX, tmA, st);
  return p.push ? launch_one<S, CL, 1, true, 16>(p, tmW, tmX, tmA, st)
                : launch_one<S, CL, 1, false, 16>(p, tmW, tmX, tmA, st);
}

// 17..64 tokens (one adapter per pool): BN = 64 token tiles, 6-stage ring, one CTA per SM
template <bool CL>
int launch_bn64(const DecParams& p, const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmA,
                cudaStream_t st) {
  if (p.lora >= 2) return launch_one<6, CL, 2, false, 64>(p, tmW, tmX, tmA, st);
  return launch_one<6, CL, 1, false, 64>(p, tmW, tmX, tmA, st);
}

// multi-adapter expand of a precomputed v (lora 4): BN = 64 tiles, 4-stage ring (the group tables, two B-row
// chunk buffers and the tile's LoRA terms take the rest of the shared memory)
template <bool CL>
int launch_mt(const DecParams& p, const CUtensorMap& tmW, const CUtensorMap& tmX, const CUtensorMap& tmA,
              cudaStream_t st) {
  return launch_one<kDecMtStages, CL, 3, false, 64>(p, tmW, tmX, tmA, st);
}

// Largest cluster size c in [2, want] such that `need` clusters of instantiation <S, true> are co-resident
// (one wave: every tile's contributors run at once), cached per (device, S, size); 1 if none.
template <int S, int BN = 16, int LM = 1>
int fit_cluster(int want, int need) {
  static int cache[kMaxDev][kDecMaxCluster + 1];
  static bool init = false;
  if (!init) {
    for (int d = 0; d < kMaxDev; ++d)
      for (int c = 0; c <= kDecMaxCluster; ++c) cache[d][c] = -1;
    init = true;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  dev = std::min(std::max(dev, 0), kMaxDev - 1);
  for (int c = want; c >= 2; --c) {
    int& mc = cache[dev][c];
    if (mc < 0) {
      cudaFuncSetAttribute(dec_lora_gemm_kernel<S, true, LM, false, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           227 * 1024);
      cudaFuncSetAttribute(dec_lora_gemm_kernel<S, true, LM, false, BN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t qc = {};
      qc.gridDim = dim3(c * need);
      qc.blockDim = dim3(kDecThreads);
      qc.dynamicSmemBytes = DecSmem<S, true, BN, LM>::kBytes;
      cudaLaunchAttribute ca[1];
      ca[0].id = cudaLaunchAttributeClusterDimension;
      ca[0].val.clusterDim.x = c;
      ca[0].val.clusterDim.y = 1;
      ca[0].val.clusterDim.z = 1;
      qc.attrs = ca;
      qc.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&mc, (void*)dec_lora_gemm_kernel<S, true, LM, false, BN>, &qc) != cudaSuccess) {
        cudaGetLastError();
        mc = 0;
      }
    }
    if (mc >= need) return c;
  }
  return 1;
}

}  // namespace

int dec_shrink_launch(const Geom& g, const __nv_bfloat16* X, int T, const int* ids, const SlotEntry* tab,
                      const __nv_bfloat16* arena, float* v, int num_sms, cudaStream_t st, int pdl, int rs_max) {
  if (T < 1 || T > kDecMaxT) return 1;
  cudaLaunchConfig_t cfg = {};
  // one item (A row) per CTA and pass, grid-stride: four CTAs per SM resident (<= 128 registers), so that
  // most batches take one pass; the GEMM's CTAs still fit beside them (no shared memory here but the tables)
  // measured (70B multi-tenant TP8, scripts/gpu_sweep_shrink.sh): 4 CTAs per SM for merged column projections
  // (3 or 2 slices: the most A rows), 2 for single-slice ones (fewer items: less launch and residency cost)
  static const int per_sm_env = env_int("BDLORA_SHRINK_CTAS_PER_SM", 0);
  const int per_sm = per_sm_env > 0 ? per_sm_env : (g.J >= 2 ? 4 : 2);
  // never more CTAs than the batch can have items (T x J x the pool's largest local shrink rank)
  const long long items_max = (long long)T * g.J * std::max(1, rs_max);
  cfg.gridDim = dim3((unsigned)std::max<long long>(1, std::min<long long>((long long)per_sm * num_sms, items_max)));
  cfg.blockDim = dim3(kDecShrinkThreads);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static const int late = env_int("BDLORA_SHRINK_LATE_TRIGGER", 0);
  return cudaLaunchKernelEx(&cfg, dec_shrink_kernel, X, T, ids, tab, arena, g, v, pdl, late) == cudaSuccess ? 0 : -1;
}

size_t dec_counter_bytes() { return sizeof(int) * kDecMaxGrid; }
size_t dec_scratch_bytes(int num_sms, int T) {
  const int bn = 64;  // multi-adapter batches (lora 4) take BN = 64 tiles at any T
  return (size_t)std::min(num_sms, kDecMaxGrid) * 2 * bn * kDecBM * 4;
}
bool dec_eligible(const Geom& g, int T) { return T >= 1 && T <= kDecMaxT && g.K % kDecBK == 0 && g.K >= kDecBK; }
bool dec_enabled() {
  static int v = -1;
  if (v < 0) v = env_int("BDLORA_DECODE", 1) != 0 ? 1 : 0;
  return v == 1;
}
void dec_last_launch(int info[8]) {
  for (int k = 0; k < 8; ++k) info[k] = g_dec_last[k];
}
void dec_set_trace(long long* buf) { g_dec_trace = buf; }

int dec_launch(const DecLaunch& a) {
  static_assert(kDecLoraRowsHost == kDecLoraRows, "K-local capacity");
  if (!dec_eligible(a.g, a.T)) return 1;
  DecParams p{};
  p.M = a.g.M;
  p.K = a.g.K;
  p.T = a.T;
  p.m_tiles = (a.g.M + kDecBM - 1) / kDecBM;
  p.k_blocks = a.g.K / kDecBK;
  const long long units = (long long)p.m_tiles * p.k_blocks;
  if (units > (1LL << 30)) return 1;
  p.units = (int)units;
  const int sms = std::max(1, a.num_sms);
  // Work split.  tiles <= #SM: every tile split into s equal K ranges (grid = tiles x s, each
  // CTA inside one tile), s as large as the SMs allow -- the whole grid streams even for 768-row
  // projections.  tiles > #SM: stream-K over a grid that divides the tile count when such a grid keeps
  // >= 70% of the SMs busy (whole tiles per CTA, no split tiles), else over every SM.
  const int tiles = p.m_tiles;
  // 17..64 tokens (the caller guarantees one adapter per pool for lora 1 / 3) and every multi-adapter expand
  // (lora 4): BN = 64 token tiles
  const bool mt = a.lora == 4;
  const bool bn64 = a.T > 16 || mt;
  const int BNh = bn64 ? 64 : 16;
  if (bn64 && a.push) return 1;
  // BN = 64 tiles compile only the tensor-core K-local shrink (lora 1): without the arena's A-row map (or with
  // the tensor-core shrink switched off) the caller's multi-kernel path serves the batch
  const bool tc_ok = a.amap != nullptr && env_int("BDLORA_DEC_TC_SHRINK", 1) != 0;
  if (bn64 && a.lora == 1 && !tc_ok) return 1;
  long long grid;
  const int min_kb = std::max(1, env_int("BDLORA_DEC_MINKB", 1));
  p.cluster = 1;
  static const int deep_kb = env_int("BDLORA_DEC_DEEP_KB", 16);
  bool deep = false;
  if (tiles <= sms) {
    int s = std::max(1, std::min(sms / tiles, p.k_blocks / min_kb));
    // the tile's s contributors reduce through a thread-block cluster (DSMEM) when s >= 2: the global
    // last-arriver fix-up costs two dependent L2 round trips (atomic + partial loads, often cross-die).
    // Long K segments (>= deep_kb k-blocks per CTA) prefer the deep 8-stage ring if its clusters (one CTA
    // per SM) still fit in one wave; else the 4-stage ring (two CTAs per SM)
    static const int cl_max = std::min(kDecMaxCluster, env_int("BDLORA_DEC_CLUSTER", kDecMaxCluster));
    if (s >= 2 && cl_max >= 2) {
      const int want = std::min(s, cl_max);
      int c = 1;
      if (mt) {
        c = fit_cluster<kDecMtStages, 64, 3>(want, tiles);
      } else if (bn64) {
        c = fit_cluster<6, 64>(want, tiles);
      } else {
        if (deep_kb > 0 && p.k_blocks / want >= deep_kb) {
          c = fit_cluster<8>(want, tiles);
          deep = c >= 2;
        }
        if (c < 2) c = fit_cluster<4>(want, tiles);
      }
      if (c >= 2) {
        s = c;
        p.cluster = c;
      }
    }
    if (p.cluster == 1) deep = deep_kb > 0 && p.k_blocks / s >= deep_kb;
    grid = (long long)tiles * s;
  } else {
    grid = 0;
    for (int m = 1; m <= 16 && !grid; ++m)
      if (tiles % m == 0 && tiles / m <= sms && tiles / m * 10 >= sms * 7) grid = tiles / m;
    if (!grid) grid = sms;
  }
  const int override_ctas = env_int("BDLORA_DEC_CTAS", 0);
  if (override_ctas > 0) {
    grid = std::min<long long>(override_ctas, units);
    p.cluster = 1;
    deep = false;
  }
  grid = std::max<long long>(1, std::min<long long>(grid, units));
  if (grid > std::min(sms, kDecMaxGrid) && grid != tiles) grid = std::min(sms, kDecMaxGrid);
  p.grid = (int)grid;
  p.X = a.X;
  p.ids = a.ids;
  p.tab = a.tab;
  p.arena = a.arena;
  p.g = a.g;
  p.v = a.v;
  p.Y = a.Y;
  p.part = (float*)a.scratch;
  p.cnt = (int*)a.cnt;
  p.lora = a.lora;
  p.pdl = a.pdl;
  p.push = a.push;
  p.peer = a.peer;
  p.trace = g_dec_trace;
  CUtensorMap tmW, tmX;
  if (!encode(&tmW, a.W, p.K, p.M, kDecBM)) return 3;
  if (!encode(&tmX, a.X, p.K, p.T, BNh)) return 3;
  // Long weight streams (>= 16 k-blocks = 256 KB per CTA, e.g. TP1 / TP2 projections) take a deep 8-stage ring (one CTA
  // per SM: the PDL overlap with the next projection matters little next to a 30+ us stream); the rest keep
  // <= 113 KB so two CTAs share an SM across projection boundaries.
  if (tiles > sms) deep = deep_kb > 0 && units / p.grid >= deep_kb;
  const int smax = mt ? kDecMtStages : bn64 ? 6 : deep ? 8 : p.cluster > 1 ? 4 : 5;
  const int stages = std::min(smax, std::max(2, env_int("BDLORA_DEC_STAGES", smax)));
  p.nstages = stages;
  if (a.grid_out) *a.grid_out = p.grid;
  g_dec_last[0] = 3;
  g_dec_last[1] = BNh;
  g_dec_last[2] = p.grid;
  g_dec_last[3] = p.cluster;
  g_dec_last[4] = stages;
  g_dec_last[5] = p.m_tiles;
  g_dec_last[6] = 1;
  g_dec_last[7] = p.k_blocks;
  // the arena's A-row map when the pool has one (else a dummy: the tensor-core shrink is then off)
  p.tc_shrink = tc_ok ? 1 : 0;
  const CUtensorMap& tmA = a.amap ? *a.amap : tmX;
  if (mt) return p.cluster > 1 ? launch_mt<true>(p, tmW, tmX, tmA, a.stream) : launch_mt<false>(p, tmW, tmX, tmA, a.stream);
  if (bn64) return p.cluster > 1 ? launch_bn64<true>(p, tmW, tmX, tmA, a.stream) : launch_bn64<false>(p, tmW, tmX, tmA, a.stream);
  if (p.cluster > 1)
    return deep ? launch_stages<8, true>(p, tmW, tmX, tmA, a.stream) : launch_stages<4, true>(p, tmW, tmX, tmA, a.stream);
  return deep ? launch_stages<8, false>(p, tmW, tmX, tmA, a.stream) : launch_stages<5, false>(p, tmW, tmX, tmA, a.stream);
}

}  // namespace bdl
