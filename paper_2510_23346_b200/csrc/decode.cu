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
  PFN_encodeTiled enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)kDecBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int env_int(const char* name, int dflt) {
  const char* s = getenv(name);
  return s ? atoi(s) : dflt;
}

template <int S>
int launch_stages(const DecParams& p, const CUtensorMap& tmW, const CUtensorMap& tmX, cudaStream_t st) {
  using L = DecSmem<S>;
  static bool attr[kMaxDev] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  dev = std::min(std::max(dev, 0), kMaxDev - 1);
  if (!attr[dev]) {
    if (cudaFuncSetAttribute(dec_lora_gemm_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes) !=
        cudaSuccess)
      return -1;
    attr[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = L::kBytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = p.pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, dec_lora_gemm_kernel<S>, tmW, tmX, p) == cudaSuccess ? 0 : -1;
}

}  // namespace

size_t dec_counter_bytes() { return sizeof(int) * kDecMaxGrid; }
size_t dec_scratch_bytes(int num_sms) { return (size_t)std::min(num_sms, kDecMaxGrid) * 2 * kDecBN * kDecBM * 4; }
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
  long long grid;
  const int min_kb = std::max(1, env_int("BDLORA_DEC_MINKB", 1));
  if (tiles <= sms) {
    const int s = std::max(1, std::min(sms / tiles, p.k_blocks / min_kb));
    grid = (long long)tiles * s;
  } else {
    grid = 0;
    for (int m = 1; m <= 16 && !grid; ++m)
      if (tiles % m == 0 && tiles / m <= sms && tiles / m * 10 >= sms * 7) grid = tiles / m;
    if (!grid) grid = sms;
  }
  const int override_ctas = env_int("BDLORA_DEC_CTAS", 0);
  if (override_ctas > 0) grid = std::min<long long>(override_ctas, units);
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
  p.trace = g_dec_trace;
  CUtensorMap tmW, tmX;
  if (!encode(&tmW, a.W, p.K, p.M, kDecBM)) return 3;
  if (!encode(&tmX, a.X, p.K, p.T, kDecBN)) return 3;
  const int stages = std::min(5, std::max(2, env_int("BDLORA_DEC_STAGES", 5)));
  p.nstages = stages;
  g_dec_last[0] = 3;
  g_dec_last[1] = kDecBN;
  g_dec_last[2] = p.grid;
  g_dec_last[3] = 1;
  g_dec_last[4] = stages;
  g_dec_last[5] = p.m_tiles;
  g_dec_last[6] = 1;
  g_dec_last[7] = p.k_blocks;
  return launch_stages<5>(p, tmW, tmX, a.stream);
}

}  // namespace bdl
