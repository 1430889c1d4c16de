// runtime.cu -- the C-ABI of libbdlora.so (include/bdlora.h): pool arena + tables, adapter loader /
// slicer, host-side validation, workspace sizing, NCCL communicator, launch sequencing of the
// BD-LoRA and S-LoRA paths.  sm_100a only.
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/bdlora.h"
#include "common.cuh"
#include "decode.h"
#include "kernels_core.cuh"
#include "kernels_umma.cuh"
#include "peer.h"

using bdl::Geom;
using bdl::SlotEntry;

// ============================================================================ errors
namespace {
thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU_TRY(expr)                                                                            \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess) return fail(BDLORA_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                                       __FILE__, __LINE__);                                     \
  } while (0)

#define NC_TRY(expr)                                                                            \
  do {                                                                                          \
    ncclResult_t _r = (expr);                                                                   \
    if (_r != ncclSuccess) return fail(BDLORA_E_NCCL, "%s: %s", #expr, ncclGetErrorString(_r)); \
  } while (0)

#define ST_TRY(expr)            \
  do {                          \
    int _s = (expr);            \
    if (_s != BDLORA_OK) return _s; \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = (cudaSetDevice(dev) == cudaSuccess);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

std::atomic<int64_t> g_launches{0};
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace

// ============================================================================ objects
struct bdlora_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 1, rank = 0, dev = 0;
  int64_t counts[6] = {0, 0, 0, 0, 0, 0};
};

// Peer group of the fused row all-reduce (include/bdlora.h, kernels_decode.cuh push mode + peer.cu).
struct bdlora_peer {
  int dev = 0, rank = 0, nranks = 1;
  long long slot = 0;            // fp32 elements per (parity, source rank) slot
  float* recv = nullptr;         // own receive buffer [2][nranks][slot]
  int* ctrl = nullptr;           // own control block: [0..1] arrival counters (unsigned), [2] parity, [3] done, [4] err
  std::vector<void*> opened;     // IPC-opened peer allocations (closed on destroy)
  std::vector<void*> owned;      // allocations to free on destroy
  float** d_recv = nullptr;      // device array [nranks]: every rank's receive buffer in this address space
  unsigned** d_cnt = nullptr;    // device array [nranks]: every rank's counters
  bdl::PeerDev dev_view{};
  int last_grid = 0;             // CTAs of the last push (each signals every rank once)
};

struct bdlora_pool {
  bdlora_pool_desc d;
  int dev = 0;
  Geom g;               // local geometry (C = chunks read by the expand)
  int rs_max = 0;       // shrink rank capacity per slot
  int re_max = 0;       // expand rank capacity per slot
  int ldb[bdl::kMaxSlices] = {0, 0, 0};
  uint16_t* arena = nullptr;
  int64_t arena_elems = 0;
  SlotEntry* d_tab = nullptr;
  std::vector<SlotEntry> h_tab;
  std::vector<int64_t> slot_elems;       // elems held by each slot (0 = empty)
  std::map<int64_t, int64_t> free_list;  // ragged arena: offset -> length (elements)
  bool ragged = false;
  int64_t resident_elems = 0;
  int num_sms = 148;
  CUtensorMap amap;      // the arena as a [arena_elems / K, K] bf16 tensor, 16-row boxes (tensor-core shrink)
  bool amap_ok = false;
};

namespace {

// Rank rows of one slot on this device: rs rows of A (shrink), re rows of B (expand).
//   BD: r/N and r/N;  S-LoRA column: r/N and r;  S-LoRA row: r and r;
//   NFS: r and r -- A_1 / B_2 whole, A_2 / B_1 with the full rank.
void ranks_for(const bdlora_pool* p, int r, int* rs, int* re) {
  const auto& d = p->d;
  const int N = d.tp_size;
  if (d.sharding == BDLORA_SHARD_BD) {
    *rs = r / N;
    *re = r / N;
  } else if (d.sharding == BDLORA_SHARD_SLORA && d.parallel == BDLORA_COLUMN) {
    *rs = r / N;
    *re = r;
  } else {
    *rs = r;
    *re = r;
  }
}

// m > 1: a downward-compatible adapter's compact local blocks -- COLUMN: B_j [r/N_h, w] (the m
// diagonal blocks side by side), ROW: A [r/N, K/m] (rank row q holds only its block's inputs)
int64_t slot_elems_for_rank(const bdlora_pool* p, int r, int m = 1) {
  int rs, re;
  ranks_for(p, r, &rs, &re);
  const bool row = p->d.parallel == BDLORA_ROW;
  int64_t e = 0;
  for (int j = 0; j < p->g.J; ++j)
    e += (int64_t)rs * p->g.K / (row ? m : 1) + (int64_t)(row ? re : re / m) * p->ldb[j];
  // slot regions are whole rows of K elements: every A row starts at a multiple of K, so one TMA
  // tensor map over the arena ([arena_elems / K, K]) addresses any adapter's A rows (tensor-core shrink)
  const int64_t K = p->g.K;
  return (e + K - 1) / K * K;
}

// Workspace layout (bytes, 256-aligned sections).  The COUNTER REGION comes first, at offsets that depend
// on nothing but constants: every counter is zero between calls (the kernels re-arm what they use), so a
// workspace zero-filled once (bdlora_workspace_init) can serve any T' <= the T it was sized for.
//   [gemv tile counters: int32 x kMaxTiles][tensor-core GEMM counters][shrink counters][spare]  (kCounterBytes)
//   [v: C_w x T x J x Rc fp32][part: S*T x M fp32 (GEMV split-K)][GEMM partials][route][gather staging]
constexpr int kMaxTiles = 8192;
constexpr int kPartTokenSplits = 64;  // S x min(T, 8) <= 64 for the split-K GEMV
constexpr size_t kOffUmmaCnt = sizeof(int) * kMaxTiles;                      // 32 KB
constexpr size_t kOffShrinkCnt = kOffUmmaCnt + 8192;                           // tensor-core GEMM: sync + 1024 counters
constexpr size_t kOffDecCnt = kOffShrinkCnt + 8192;                            // lean decode kernel: 1024 counters
constexpr size_t kCounterBytes = kOffDecCnt + 16384;                          // 64 KB
static_assert(bdl::kUmmaCounterBytes <= 8192, "GEMM counter region");
thread_local int g_last_src = 0;  // bdlora_last_launch_info: 0 = tensor-core GEMM / shrink record, 1 = lean decode

struct WsLayout {
  size_t off_counters, off_umma_cnt, off_shrink_cnt, off_dec_cnt, off_v, off_part, off_umma, off_dec, off_route,
      off_gather, total;
};

constexpr int kTcShrinkMinT = 17;  // phases API: tensor-core shrink above decode sizes
// forwards: one kernel (grid-wide shrink inside the GEMM) up to 16 tokens.  Measured at T = 64 (70B, A/B
// with BDLORA_FUSED_MAX_T=64): the grid-wide CUDA-core shrink loses to route + tensor-core shrink both for one
// adapter (bs64 TP8 layer 196 vs 143 us) and for ~50 adapters (multi-tenant TP8 322 vs 238 us)
constexpr int kFusedMaxT = 16;

// Upper bound of the tensor-core shrink's 16-row A boxes for a batch of T tokens (0 = not eligible).
int tc_items_max(const bdlora_pool* p, int64_t T) {
  if (!p->amap_ok || p->g.K % 64 != 0 || T < kTcShrinkMinT || T > bdl::kRouteMaxSeg) return 0;
  const int64_t groups = std::min<int64_t>(T, p->d.capacity);
  if (groups > bdl::kRouteMaxGroups) return 0;
  const int64_t items = groups * p->g.J * ((p->rs_max + 15) / 16);
  if (items > bdl::kRouteMaxItems) return 0;
  return (int)items;
}

// Largest batch served by the single-kernel forward (BDLORA_FUSED_MAX_T overrides; tuning / A-B)
int fused_max_t() {
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("BDLORA_FUSED_MAX_T");
    v = s ? std::max(0, std::min(atoi(s), bdl::kFuseMaxT)) : kFusedMaxT;
  }
  return v;
}

WsLayout ws_layout(const bdlora_pool* p, int64_t T) {
  WsLayout L;
  L.off_counters = 0;
  L.off_umma_cnt = kOffUmmaCnt;
  L.off_shrink_cnt = kOffShrinkCnt;
  L.off_dec_cnt = kOffDecCnt;
  size_t o = kCounterBytes;
  L.off_v = o;
  const int Cw = (p->d.sharding == BDLORA_SHARD_SLORA && p->d.parallel == BDLORA_COLUMN) ? p->d.tp_size : 1;
  o = align_up(o + sizeof(float) * (size_t)Cw * T * p->g.J * p->g.Rc, 256);
  L.off_part = o;
  o = align_up(o + sizeof(float) * (size_t)kPartTokenSplits * p->g.M, 256);
  L.off_umma = o;
  o = align_up(o + bdl::umma_workspace_bytes(p->g.M, (int)T, p->num_sms), 256);
  L.off_dec = o;  // lean decode kernel: split-tile partials
  if (T <= bdl::kDecMaxT) o = align_up(o + bdl::dec_scratch_bytes(p->num_sms, (int)T), 256);
  L.off_route = o;
  const int items = tc_items_max(p, std::min<int64_t>(T, bdl::kRouteMaxSeg));
  if (items > 0) o = align_up(o + sizeof(int) * bdl::RouteLayout::kWords, 256);
  L.off_gather = o;  // Alg. 2 all-gather staging: [N][T][M_loc] bf16 (column pools, N > 1)
  if (p->d.parallel == BDLORA_COLUMN && p->d.tp_size > 1) o = align_up(o + (size_t)p->d.tp_size * T * p->g.M * 2, 256);
  L.total = o;
  return L;
}

int check_pool(const bdlora_pool* p) {
  if (!p) return fail(BDLORA_E_ARG, "pool is NULL");
  return BDLORA_OK;
}

int check_fwd_args(const bdlora_pool* p, const void* X, int64_t T, const void* W, const int32_t* ids, const void* Y,
                   void* ws, size_t ws_bytes) {
  ST_TRY(check_pool(p));
  if (T < 0) return fail(BDLORA_E_ARG, "T = %lld < 0", (long long)T);
  if (T > (1 << 20)) return fail(BDLORA_E_CAPACITY, "T = %lld exceeds 2^20 tokens", (long long)T);
  if (T == 0) return BDLORA_OK;
  if (!X || !W || !ids || !Y) return fail(BDLORA_E_ARG, "X/W/ids/Y must be non-NULL (X=%p W=%p ids=%p Y=%p)", X, W, ids, Y);
  if (((uintptr_t)X | (uintptr_t)W) & 15) return fail(BDLORA_E_ARG, "X and W must be 16-byte aligned");
  if (!ws) return fail(BDLORA_E_ARG, "workspace is NULL");
  const size_t need = ws_layout(p, T).total;
  if (ws_bytes < need)
    return fail(BDLORA_E_ARG, "workspace too small: %zu < %zu bytes for T=%lld", ws_bytes, need, (long long)T);
  if ((uintptr_t)ws & 255) return fail(BDLORA_E_ARG, "workspace must be 256-byte aligned");
  return BDLORA_OK;
}

// ---------------------------------------------------------------------------- launches
int g_pdl = 1;  // programmatic dependent launch chaining (bdlora_set_pdl)

// Downward-compatible pools (compact local blocks, Geom::ablk / bblk > 1) run every batch through the
// multi-adapter decode path -- dec_shrink_kernel (block-local K window for ROW pools) then the decode kernel's
// tensor-core expand (block-local rank rows for COLUMN pools) -- in chunks of <= 64 tokens.
bool pool_blocked(const bdlora_pool* p) { return p->g.ablk > 1 || p->g.bblk > 1; }
thread_local bdlora_peer* g_push = nullptr;  // set around the decode launch of bdlora_row_partial_push

WsLayout ws_layout(const bdlora_pool* p, int64_t T);

// v = s X A[a] for T tokens.  Batches are processed in chunks of at most kRouteMaxSeg tokens (the route
// kernel stages one chunk's segments in shared memory; shrink_rows_kernel stages one chunk's member list),
// so any T the ABI accepts is served in O(T) work: chunk c covers tokens [c0, c0 + Tc) and writes v rows
// [c0, c0 + Tc) (v is token-major inside each of its C chunks).
int launch_shrink(const bdlora_pool* p, const void* X, int T, const int32_t* ids, float* v, cudaStream_t st,
                  void* ws = nullptr) {
  if (T == 0) return BDLORA_OK;
  const Geom& g = p->g;
  if (pool_blocked(p)) {
    for (int c0 = 0; c0 < T; c0 += bdl::kDecMaxT) {
      const int Tc = std::min(T - c0, bdl::kDecMaxT);
      const int rc = bdl::dec_shrink_launch(g, (const __nv_bfloat16*)X + (size_t)c0 * g.K, Tc, ids + c0, p->d_tab,
                                            (const __nv_bfloat16*)p->arena, v + (size_t)c0 * g.J * g.Rc, p->num_sms,
                                            st, g_pdl, p->rs_max);
      if (rc != 0) return fail(BDLORA_E_CUDA, "decode shrink launch (%d): %s", rc, cudaGetErrorString(cudaGetLastError()));
      count_launch();
      g_last_src = 1;
    }
    return BDLORA_OK;
  }
  if (T <= bdl::kDecMaxT && bdl::dec_enabled() && g.K % 8 == 0) {
    // decode-sized batch: one grid-wide launch, every distinct adapter's A rows read once
    const int rc = bdl::dec_shrink_launch(g, (const __nv_bfloat16*)X, T, ids, p->d_tab, (const __nv_bfloat16*)p->arena,
                                          v, p->num_sms, st, g_pdl, p->rs_max);
    if (rc < 0) return fail(BDLORA_E_CUDA, "decode shrink launch: %s", cudaGetErrorString(cudaGetLastError()));
    if (rc == 0) {
      count_launch();
      g_last_src = 1;
      return BDLORA_OK;
    }
  }
  const size_t per_tok = (size_t)g.J * g.Rc;
  for (int c0 = 0; c0 < T; c0 += bdl::kRouteMaxSeg) {
    const int Tc = std::min(T - c0, bdl::kRouteMaxSeg);
    const void* Xc = (const char*)X + (size_t)c0 * g.K * 2;
    const int32_t* idc = ids + c0;
    float* vc = v + (size_t)c0 * per_tok;
    const int items = ws ? tc_items_max(p, Tc) : 0;
    if (items > 0) {
      // tensor-core shrink: route (groups + A boxes) -> grouped tcgen05 GEMM writing v
      const WsLayout L = ws_layout(p, T);
      int* route = (int*)((char*)ws + L.off_route);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1);
      cfg.blockDim = dim3(1024);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = g_pdl;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      CU_TRY(cudaLaunchKernelEx(&cfg, bdl::route_kernel, idc, Tc, (const SlotEntry*)p->d_tab, p->g, route, vc,
                                (int)(Tc * per_tok)));
      count_launch();
      int rc = bdl::umma_shrink_launch(p->g, (const __nv_bfloat16*)Xc, Tc, idc, p->d_tab, route, p->amap, vc, items,
                                       (char*)ws + L.off_shrink_cnt, p->num_sms, st, g_pdl);
      if (rc != 0) return fail(BDLORA_E_CUDA, "tensor-core shrink launch failed (%d): %s", rc,
                               cudaGetErrorString(cudaGetLastError()));
      count_launch();
      g_last_src = 0;
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(Tc, g.J, p->rs_max);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = sizeof(int) * (size_t)Tc;  // <= 16 KB
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CU_TRY(cudaLaunchKernelEx(&cfg, bdl::shrink_rows_kernel<4>, (const __nv_bfloat16*)Xc, Tc, idc,
                              (const SlotEntry*)p->d_tab, (const __nv_bfloat16*)p->arena, g, vc));
    count_launch();
  }
  return BDLORA_OK;
}

int launch_gemv(const bdlora_pool* p, const void* X, int T, const void* W, const int32_t* ids, const float* v,
                void* Y, void* ws, cudaStream_t st) {
  const Geom& g = p->g;
  const WsLayout L = ws_layout(p, T);
  char* base = (char*)ws;
  int* counters = (int*)(base + L.off_counters);
  float* part = (float*)(base + L.off_part);
  constexpr int RW = 2, ROWS = 8 * RW;
  const int ntiles = (g.M + ROWS - 1) / ROWS;
  if (ntiles > kMaxTiles) return fail(BDLORA_E_CAPACITY, "M = %d too large for the GEMV path", g.M);
  const int TT = T >= 8 ? 8 : (T >= 4 ? 4 : (T >= 2 ? 2 : 1));
  // split-K so that the grid has >= ~4 CTAs (32 warps) per SM; partial buffer bounds S*T <= 64
  int S = 1;
  const int target = 4 * p->num_sms;
  if (ntiles < target && T <= 8) {
    S = (target + ntiles - 1) / ntiles;
    S = std::min(S, std::max(1, g.K / 256));
    S = std::min(S, kPartTokenSplits / std::max(T, 1));
    S = std::max(S, 1);
  }
  int Kc = (g.K + S - 1) / S;
  Kc = (Kc + 7) / 8 * 8;
  S = (g.K + Kc - 1) / Kc;
  dim3 grid(ntiles, S);
#define GEMV_CASE(TTV)                                                                                      \
  bdl::gemv_lora_kernel<TTV, RW><<<grid, 256, 0, st>>>((const __nv_bfloat16*)X, T, (const __nv_bfloat16*)W, ids, \
                                                       p->d_tab, (const __nv_bfloat16*)p->arena, g, v,             \
                                                       (__nv_bfloat16*)Y, part, counters, S, Kc)
  switch (TT) {
    case 1: GEMV_CASE(1); break;
    case 2: GEMV_CASE(2); break;
    case 4: GEMV_CASE(4); break;
    default: GEMV_CASE(8); break;
  }
#undef GEMV_CASE
  count_launch();
  CU_TRY(cudaGetLastError());
  return BDLORA_OK;
}

// Lean decode kernel (kernels_decode.cuh) for T <= 16.  lora = 1: K-local shrink + expand inside the kernel;
// 2: v precomputed (the expand of a forward whose collective sits between shrink and expand).
int launch_decode(const bdlora_pool* p, const void* X, int T, const void* W, const int32_t* ids, const float* v,
                  void* Y, void* ws, cudaStream_t st, int lora) {
  const WsLayout L = ws_layout(p, T);
  bdl::DecLaunch a;
  a.g = p->g;
  a.X = (const __nv_bfloat16*)X;
  a.T = T;
  a.W = (const __nv_bfloat16*)W;
  a.ids = ids;
  a.tab = p->d_tab;
  a.arena = (const __nv_bfloat16*)p->arena;
  a.v = v;
  a.Y = (__nv_bfloat16*)Y;
  a.cnt = (char*)ws + L.off_dec_cnt;
  a.scratch = (char*)ws + L.off_dec;
  a.num_sms = p->num_sms;
  a.stream = st;
  a.pdl = g_pdl;
  a.lora = lora;
  a.amap = p->amap_ok ? &p->amap : nullptr;
  a.push = 0;
  a.peer = bdl::PeerDev{};
  a.grid_out = nullptr;
  if (g_push) {  // fused row all-reduce (bdlora_row_partial_push): set by the caller for this one launch
    a.push = 1;
    a.peer = g_push->dev_view;
    a.grid_out = &g_push->last_grid;
  }
  const int rc = bdl::dec_launch(a);
  if (rc < 0) return fail(BDLORA_E_CUDA, "decode kernel launch: %s", cudaGetErrorString(cudaGetLastError()));
  if (rc > 0) return -1;  // shape not handled here
  count_launch();
  g_last_src = 1;
  return BDLORA_OK;
}

// K-local LoRA inside the decode kernel needs every adapter's shrink and expand device-local (BD / NFS, one v
// chunk) and the batch's distinct adapters to fit the kernel's rank-row capacity in the worst case.
bool decode_klocal_ok(const bdlora_pool* p, int T) {
  if (p->d.sharding == BDLORA_SHARD_SLORA || p->g.C != 1 || pool_blocked(p)) return false;
  if (T > 16) {
    // 17..64 tokens (BN = 64 tiles): only the tensor-core K-local shrink is compiled there -- one adapter per
    // pool, r/N <= 16, every tile inside one slice, the arena's A-row map
    if (p->d.capacity != 1 || p->rs_max > 16 || !p->amap_ok) return false;
    for (int j = 0; j < p->g.J; ++j)
      if (p->g.col0[j] % 128) return false;
    return true;
  }
  return (int64_t)std::min<int64_t>(T, p->d.capacity) * p->rs_max <= bdl::kDecLoraRowsHost;
}

// Multi-adapter decode (lora 4, any number of adapters, T <= 64): the precomputed v is expanded in the decode
// kernel's epilogue; every 128-column tile must lie inside one slice (its B rows come from one B_j).
bool decode_mt_ok(const bdlora_pool* p, int T) {
  if (T < 1 || T > bdl::kDecMaxT || g_push || !bdl::dec_enabled() || !bdl::dec_eligible(p->g, T)) return false;
  for (int j = 0; j < p->g.J; ++j)
    if (p->g.col0[j] % 128 || p->g.e_lo[j] % 128) return false;
  return true;
}

int launch_base_expand(const bdlora_pool* p, const void* X, int T, const void* W, const int32_t* ids, const float* v,
                       void* Y, void* ws, cudaStream_t st) {
  const int pdl = g_pdl;
  if (T == 0) return BDLORA_OK;
  if (pool_blocked(p)) {
    if (!decode_mt_ok(p, 1))
      return fail(BDLORA_E_ARG, "downward-compatible pool: the multi-adapter decode kernel cannot serve this "
                  "geometry (K %% 64, 128-column slices) or it is disabled (BDLORA_DECODE=0)");
    for (int c0 = 0; c0 < T; c0 += bdl::kDecMaxT) {
      const int Tc = std::min(T - c0, bdl::kDecMaxT);
      const int rc = launch_decode(p, (const __nv_bfloat16*)X + (size_t)c0 * p->g.K, Tc, W, ids + c0,
                                   v + (size_t)c0 * p->g.J * p->g.Rc, (__nv_bfloat16*)Y + (size_t)c0 * p->g.M, ws, st, 4);
      if (rc != BDLORA_OK) return rc < 0 ? fail(BDLORA_E_ARG, "downward-compatible expand: shape not served") : rc;
    }
    return BDLORA_OK;
  }
  if (bdl::dec_enabled() && bdl::dec_eligible(p->g, T)) {
    // v precomputed: staged-B expand (mode 3) when the batch's distinct adapters fit the kernel's rank-row
    // capacity in the worst case, else the per-output gather (mode 2)
    const bool staged = (int64_t)std::min<int64_t>(T, p->d.capacity) * p->re_max <= bdl::kDecLoraRowsHost;
    const bool mt = decode_mt_ok(p, T);
    int mode = 0;
    if (staged && T <= 16) mode = 3;  // a few rank rows: staged once per tile, CUDA-core expand
    else if (mt) mode = 4;            // tensor-core expand of the tile's rank rows (any number of adapters)
    else if (staged && p->d.capacity == 1) mode = 3;
    else if (T <= 16) mode = 2;
    if (mode) {
      const int rc = launch_decode(p, X, T, W, ids, v, Y, ws, st, mode);
      if (rc >= 0) return rc;
    }
  }
  if (bdl::umma_eligible(p->g, T)) {
    const WsLayout L = ws_layout(p, T);
    int rc = bdl::umma_launch(p->g, (const __nv_bfloat16*)X, T, (const __nv_bfloat16*)W, ids, p->d_tab,
                              (const __nv_bfloat16*)p->arena, v, (__nv_bfloat16*)Y, (char*)ws + L.off_umma_cnt,
                              (char*)ws + L.off_umma, p->num_sms, st, pdl, nullptr, 0, /*tcx=*/1, p->amap_ok ? &p->amap : nullptr);
    if (rc == 0) {
      count_launch();
      g_last_src = 0;
      CU_TRY(cudaGetLastError());
      return BDLORA_OK;
    }
    // rc != 0: shape not supported by the tensor-core kernel -> CUDA-core kernel (still on GPU)
  }
  return launch_gemv(p, X, T, W, ids, v, Y, ws, st);
}

float* ws_v(const bdlora_pool* p, void* ws, int64_t T) { return (float*)((char*)ws + ws_layout(p, T).off_v); }

const char* sharding_name(int sharding) {
  return sharding == BDLORA_SHARD_BD ? "BD" : sharding == BDLORA_SHARD_SLORA ? "SLORA" : sharding == BDLORA_SHARD_NFS ? "NFS" : "?";
}

int require_mode(const bdlora_pool* p, int parallel, int sharding, const char* fn) {
  if (p->d.parallel != parallel || p->d.sharding != sharding)
    return fail(BDLORA_E_MODE, "%s: pool is %s+%s, expected %s+%s", fn, p->d.parallel == BDLORA_COLUMN ? "COLUMN" : "ROW",
                sharding_name(p->d.sharding), parallel == BDLORA_COLUMN ? "COLUMN" : "ROW", sharding_name(sharding));
  return BDLORA_OK;
}

int require_comm(const bdlora_pool* p, const bdlora_comm* c, const char* fn) {
  if (p->d.tp_size == 1) return BDLORA_OK;
  if (!c) return fail(BDLORA_E_ARG, "%s: comm is NULL but tp_size = %d", fn, p->d.tp_size);
  if (c->nranks != p->d.tp_size || c->rank != p->d.tp_rank)
    return fail(BDLORA_E_ARG, "%s: comm (nranks=%d, rank=%d) does not match pool (tp_size=%d, tp_rank=%d)", fn,
                c->nranks, c->rank, p->d.tp_size, p->d.tp_rank);
  if (c->dev != p->dev) return fail(BDLORA_E_ARG, "%s: comm device %d != pool device %d", fn, c->dev, p->dev);
  return BDLORA_OK;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

int bdlora_abi_version(void) { return BDLORA_ABI_VERSION; }

int bdlora_set_pdl(int enable) {
  g_pdl = enable ? 1 : 0;
  return BDLORA_OK;
}

int bdlora_set_decode_lora(int mode) {
  if (mode < 0 || mode > 2) return fail(BDLORA_E_ARG, "bdlora_set_decode_lora: mode %d not in {0, 1, 2}", mode);
  bdl::g_local_mode = mode;
  return BDLORA_OK;
}

int bdlora_debug_trace(void* device_buffer) {
  bdl::g_umma_trace = (long long*)device_buffer;
  bdl::dec_set_trace((long long*)device_buffer);
  return BDLORA_OK;
}

int bdlora_kernel_launches(int64_t* n) {
  if (!n) return fail(BDLORA_E_ARG, "n is NULL");
  *n = g_launches.load();
  return BDLORA_OK;
}

const char* bdlora_last_error(void) { return g_err.c_str(); }

int bdlora_device_check(int cuda_device) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return fail(BDLORA_E_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  if (cuda_device < 0 || cuda_device >= n) return fail(BDLORA_E_ARG, "cuda_device %d out of range [0,%d)", cuda_device, n);
  int maj = 0, min = 0;
  CU_TRY(cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, cuda_device));
  CU_TRY(cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, cuda_device));
  if (maj != 10 || min != 0)
    return fail(BDLORA_E_ARCH, "device %d is sm_%d%d; libbdlora is built for sm_100a only", cuda_device, maj, min);
  return BDLORA_OK;
}

// ---------------------------------------------------------------------------- comm
int bdlora_comm_unique_id(uint8_t id[BDLORA_UNIQUE_ID_BYTES]) {
  if (!id) return fail(BDLORA_E_ARG, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == BDLORA_UNIQUE_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  NC_TRY(ncclGetUniqueId(&u));
  memcpy(id, &u, sizeof(u));
  return BDLORA_OK;
}

int bdlora_comm_init(const uint8_t id[BDLORA_UNIQUE_ID_BYTES], int nranks, int rank, int cuda_device,
                     bdlora_comm** out) {
  if (!id || !out) return fail(BDLORA_E_ARG, "id/out is NULL");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(BDLORA_E_ARG, "bad nranks=%d rank=%d", nranks, rank);
  ST_TRY(bdlora_device_check(cuda_device));
  DeviceGuard dg(cuda_device);
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  bdlora_comm* c = new bdlora_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->dev = cuda_device;
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(BDLORA_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = c;
  return BDLORA_OK;
}

int bdlora_comm_destroy(bdlora_comm* c) {
  if (!c) return BDLORA_OK;
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
  return BDLORA_OK;
}

int bdlora_comm_stats(const bdlora_comm* c, int64_t counts[6]) {
  if (!c || !counts) return fail(BDLORA_E_ARG, "comm/counts is NULL");
  memcpy(counts, c->counts, sizeof(c->counts));
  return BDLORA_OK;
}

// ---------------------------------------------------------------------------- pool
int bdlora_create_pool(const bdlora_pool_desc* desc, int cuda_device, bdlora_pool** out) {
  if (!desc || !out) return fail(BDLORA_E_ARG, "desc/out is NULL");
  const bdlora_pool_desc& d = *desc;
  if (d.parallel != BDLORA_COLUMN && d.parallel != BDLORA_ROW) return fail(BDLORA_E_ARG, "parallel = %d", d.parallel);
  if (d.sharding != BDLORA_SHARD_BD && d.sharding != BDLORA_SHARD_SLORA && d.sharding != BDLORA_SHARD_NFS)
    return fail(BDLORA_E_ARG, "sharding = %d", d.sharding);
  const bool nfs = d.sharding == BDLORA_SHARD_NFS;
  if (d.tp_size < 1 || d.tp_rank < 0 || d.tp_rank >= d.tp_size)
    return fail(BDLORA_E_ARG, "tp_size = %d, tp_rank = %d", d.tp_size, d.tp_rank);
  if (d.n_slices < 1 || d.n_slices > BDLORA_MAX_SLICES) return fail(BDLORA_E_ARG, "n_slices = %d", d.n_slices);
  if (d.parallel == BDLORA_ROW && d.n_slices != 1) return fail(BDLORA_E_ARG, "ROW pools take n_slices = 1 (got %d)", d.n_slices);
  if (d.d_in <= 0) return fail(BDLORA_E_ARG, "d_in = %d", d.d_in);
  for (int j = 0; j < d.n_slices; ++j)
    if (d.d_out[j] <= 0) return fail(BDLORA_E_ARG, "d_out[%d] = %d", j, d.d_out[j]);
  if (d.capacity < 1 || d.capacity > (1 << 20)) return fail(BDLORA_E_CAPACITY, "capacity = %d", d.capacity);
  if (d.max_rank < 1 || d.max_rank > 4096) return fail(BDLORA_E_CAPACITY, "max_rank = %d (1..4096)", d.max_rank);
  if (d.arena_bytes < 0) return fail(BDLORA_E_ARG, "arena_bytes < 0");
  const int N = d.tp_size;
  if (!nfs && d.max_rank % N)
    return fail(BDLORA_E_DIVISIBILITY, "max_rank %d not divisible by tp_size %d", d.max_rank, N);
  if (d.parallel == BDLORA_COLUMN) {
    for (int j = 0; j < d.n_slices; ++j)
      if (d.d_out[j] % N) return fail(BDLORA_E_DIVISIBILITY, "d_out[%d] = %d not divisible by tp_size %d", j, d.d_out[j], N);
    if (d.d_in % 8) return fail(BDLORA_E_ARG, "d_in = %d must be a multiple of 8 (128-bit rows)", d.d_in);
  } else {
    if (d.d_in % N) return fail(BDLORA_E_DIVISIBILITY, "d_in %d not divisible by tp_size %d", d.d_in, N);
    if ((d.d_in / N) % 8) return fail(BDLORA_E_ARG, "d_in/N = %d must be a multiple of 8", d.d_in / N);
    if (d.sharding == BDLORA_SHARD_SLORA && d.d_out[0] % N)
      return fail(BDLORA_E_DIVISIBILITY, "d_out %d not divisible by tp_size %d (S-LoRA B column shards)", d.d_out[0], N);
  }
  ST_TRY(bdlora_device_check(cuda_device));
  DeviceGuard dg(cuda_device);

  bdlora_pool* p = new bdlora_pool();
  p->d = d;
  p->dev = cuda_device;
  Geom& g = p->g;
  memset(&g, 0, sizeof(g));
  g.ablk = g.bblk = 1;  // native BD until a downward-compatible adapter is loaded (bdlora_load_adapter_blocks)
  const int i = d.tp_rank;
  if (d.parallel == BDLORA_COLUMN) {
    g.K = d.d_in;
    g.J = d.n_slices;
    int c0 = 0;
    for (int j = 0; j < g.J; ++j) {
      const int w = d.d_out[j] / N;
      g.col0[j] = c0;
      g.e_lo[j] = c0;
      g.e_hi[j] = c0 + w;
      p->ldb[j] = w;
      c0 += w;
    }
    g.col0[g.J] = c0;
    g.M = c0;
    g.Rc = nfs ? d.max_rank : d.max_rank / N;
    g.C = (d.sharding == BDLORA_SHARD_SLORA) ? N : 1;
    p->rs_max = nfs ? d.max_rank : d.max_rank / N;
    p->re_max = (d.sharding == BDLORA_SHARD_BD) ? d.max_rank / N : d.max_rank;
  } else {
    g.K = d.d_in / N;
    g.J = 1;
    g.M = d.d_out[0];
    g.col0[0] = 0;
    g.col0[1] = g.M;
    if (d.sharding == BDLORA_SHARD_BD) {
      g.e_lo[0] = 0;
      g.e_hi[0] = g.M;
      p->ldb[0] = g.M;
      g.Rc = d.max_rank / N;
      p->rs_max = p->re_max = d.max_rank / N;
    } else if (nfs) {  // B_2 whole on every device: expand window = all d_out columns
      g.e_lo[0] = 0;
      g.e_hi[0] = g.M;
      p->ldb[0] = g.M;
      g.Rc = d.max_rank;
      p->rs_max = p->re_max = d.max_rank;
    } else {
      const int w = g.M / N;
      g.e_lo[0] = i * w;
      g.e_hi[0] = (i + 1) * w;
      p->ldb[0] = w;
      g.Rc = d.max_rank;
      p->rs_max = p->re_max = d.max_rank;
    }
    g.C = 1;
  }
  p->h_tab.assign(d.capacity, SlotEntry{});
  p->slot_elems.assign(d.capacity, 0);
  int64_t per_slot = slot_elems_for_rank(p, d.max_rank);
  if (d.arena_bytes == 0) {
    p->arena_elems = per_slot * d.capacity;
    p->ragged = false;
  } else {
    p->arena_elems = d.arena_bytes / 2 / g.K * g.K;
    p->ragged = true;
    p->free_list[0] = p->arena_elems;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
  if (const char* cap = getenv("BDLORA_GRID_CAP")) sms = std::max(1, std::min(sms, atoi(cap)));  // tuning only
  p->num_sms = sms;
  cudaError_t e1 = cudaMalloc(&p->arena, std::max<int64_t>(p->arena_elems, 8) * 2);
  cudaError_t e2 = cudaMalloc(&p->d_tab, sizeof(SlotEntry) * d.capacity);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    if (p->arena) cudaFree(p->arena);
    if (p->d_tab) cudaFree(p->d_tab);
    delete p;
    return fail(BDLORA_E_CUDA, "cudaMalloc arena (%lld B) / table: %s", (long long)(p->arena_elems * 2),
                cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  }
  cudaMemset(p->d_tab, 0, sizeof(SlotEntry) * d.capacity);
  cudaMemset(p->arena, 0, std::max<int64_t>(p->arena_elems, 8) * 2);
  if (g.K % 64 == 0 && p->arena_elems / g.K > 0)
    p->amap_ok = bdl::encode_kmajor(&p->amap, p->arena, g.K, (int)(p->arena_elems / g.K), 16);
  CU_TRY(cudaDeviceSynchronize());
  *out = p;
  return BDLORA_OK;
}

int bdlora_destroy_pool(bdlora_pool* p) {
  if (!p) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  cudaFree(p->arena);
  cudaFree(p->d_tab);
  delete p;
  return BDLORA_OK;
}

static int arena_alloc(bdlora_pool* p, int slot, int64_t elems, int64_t* off) {
  if (!p->ragged) {
    *off = slot_elems_for_rank(p, p->d.max_rank) * slot;
    return BDLORA_OK;
  }
  for (auto it = p->free_list.begin(); it != p->free_list.end(); ++it) {
    if (it->second >= elems) {
      *off = it->first;
      const int64_t rest = it->second - elems;
      const int64_t noff = it->first + elems;
      p->free_list.erase(it);
      if (rest > 0) p->free_list[noff] = rest;
      return BDLORA_OK;
    }
  }
  return fail(BDLORA_E_CAPACITY, "arena full: no free run of %lld elements for slot %d", (long long)elems, slot);
}

static void arena_free(bdlora_pool* p, int64_t off, int64_t elems) {
  if (!p->ragged || elems == 0) return;
  auto it = p->free_list.emplace(off, elems).first;
  // coalesce with next
  auto nx = std::next(it);
  if (nx != p->free_list.end() && it->first + it->second == nx->first) {
    it->second += nx->second;
    p->free_list.erase(nx);
  }
  if (it != p->free_list.begin()) {
    auto pv = std::prev(it);
    if (pv->first + pv->second == it->first) {
      pv->second += it->second;
      p->free_list.erase(it);
    }
  }
}

static int gather_to(const uint16_t* src, int64_t ld, int r0, int c0, int nr, int nc, int transpose, uint16_t* dst,
                     cudaStream_t st, int64_t ldd = 0) {
  if (nr == 0 || nc == 0) return BDLORA_OK;
  dim3 grid((nc + 31) / 32, (nr + 31) / 32);
  bdl::gather_kernel<<<grid, dim3(32, 8), 0, st>>>(src, ld, r0, c0, nr, nc, transpose, dst, ldd);
  count_launch();
  CU_TRY(cudaGetLastError());
  return BDLORA_OK;
}

static int load_adapter_impl(bdlora_pool* p, int32_t slot, int32_t rank, float scale, const void* const* A,
                             const void* const* B, int32_t src_is_device, bdlora_stream_t stream, int nb);

int bdlora_load_adapter(bdlora_pool* p, int32_t slot, int32_t rank, float scale, const void* const* A,
                        const void* const* B, int32_t src_is_device, bdlora_stream_t stream) {
  ST_TRY(check_pool(p));
  return load_adapter_impl(p, slot, rank, scale, A, B, src_is_device, stream, p->d.tp_size);
}

int bdlora_load_adapter_blocks(bdlora_pool* p, int32_t slot, int32_t rank, float scale, const void* const* A,
                               const void* const* B, int32_t n_blocks, int32_t src_is_device, bdlora_stream_t stream) {
  ST_TRY(check_pool(p));
  const auto& d = p->d;
  if (d.sharding != BDLORA_SHARD_BD) return fail(BDLORA_E_MODE, "bdlora_load_adapter_blocks needs a BD pool");
  if (n_blocks < d.tp_size || n_blocks % d.tp_size)
    return fail(BDLORA_E_DIVISIBILITY, "n_blocks %d must be a multiple of tp_size %d (P:499-507)", n_blocks, d.tp_size);
  if (rank % n_blocks) return fail(BDLORA_E_DIVISIBILITY, "rank %d not divisible by n_blocks %d", rank, n_blocks);
  if (d.parallel == BDLORA_COLUMN) {
    for (int j = 0; j < d.n_slices; ++j)
      if (d.d_out[j] % n_blocks)
        return fail(BDLORA_E_DIVISIBILITY, "d_out[%d] = %d not divisible by n_blocks %d", j, d.d_out[j], n_blocks);
  } else if (d.d_in % n_blocks) {
    return fail(BDLORA_E_DIVISIBILITY, "d_in %d not divisible by n_blocks %d", d.d_in, n_blocks);
  }
  return load_adapter_impl(p, slot, rank, scale, A, B, src_is_device, stream, n_blocks);
}

static int load_adapter_impl(bdlora_pool* p, int32_t slot, int32_t rank, float scale, const void* const* A,
                             const void* const* B, int32_t src_is_device, bdlora_stream_t stream, int nb) {
  const auto& d = p->d;
  if (slot < 0 || slot >= d.capacity) return fail(BDLORA_E_CAPACITY, "slot %d out of range [0,%d)", slot, d.capacity);
  if (rank < 1 || rank > d.max_rank) return fail(BDLORA_E_CAPACITY, "rank %d out of range [1,%d]", rank, d.max_rank);
  const int N = d.tp_size, i = d.tp_rank, J = p->g.J;
  // BD: rank r/N per shard; S-LoRA column: rank chunks of r/N.  S-LoRA row keeps
  // the full rank on every device.
  const bool need_div = !(d.sharding == BDLORA_SHARD_SLORA && d.parallel == BDLORA_ROW) &&
                        d.sharding != BDLORA_SHARD_NFS;  // NFS replicates instead of splitting the rank
  if (need_div && rank % N)
    return fail(BDLORA_E_DIVISIBILITY, "rank %d not divisible by tp_size %d (P:462)", rank, N);
  if (!A || !B) return fail(BDLORA_E_ARG, "A/B arrays are NULL");
  for (int j = 0; j < J; ++j)
    if (!A[j] || !B[j]) return fail(BDLORA_E_ARG, "A[%d]/B[%d] is NULL", j, j);
  if (!std::isfinite(scale)) return fail(BDLORA_E_ARG, "scale is not finite");
  DeviceGuard dg(p->dev);
  cudaStream_t st = (cudaStream_t)stream;

  // a reload keeps the previous occupant until the new one is staged: in the ragged arena the new region is
  // allocated first (an allocation failure leaves the old adapter loaded and intact) and the old region is
  // released only after the new table entry is in place; the fixed arena reuses the slot's own region, so
  // a failure while copying leaves the slot empty
  const bool reload = p->h_tab[slot].loaded != 0;
  const SlotEntry old_e = p->h_tab[slot];
  const int64_t old_elems = p->slot_elems[slot];

  int rs, re;
  ranks_for(p, rank, &rs, &re);
  // downward-compatible serving: m = N_h / N blocks per device, one m per pool (the kernels read it from the
  // geometry); the compact blocks are all that is stored
  const int m = (d.sharding == BDLORA_SHARD_BD && nb > 0) ? nb / N : 1;
  const bool row = d.parallel == BDLORA_ROW;
  {
    int others = 0;
    for (int s2 = 0; s2 < d.capacity; ++s2) others += (s2 != slot && p->h_tab[s2].loaded) ? 1 : 0;
    const int cur_m = row ? p->g.ablk : p->g.bblk;
    if (others > 0 && cur_m != m)
      return fail(BDLORA_E_MODE, "pool holds adapters with %d local block(s) per device; this load has %d (one "
                  "block count per pool)", cur_m, m);
    if (m > 1) {
      if (row && ((p->g.K / m) % 8 || p->g.K % 64))
        return fail(BDLORA_E_DIVISIBILITY, "downward-compatible ROW pool: K/m = %d must be a multiple of 8 and "
                    "K = %d of 64", p->g.K / m, p->g.K);
      for (int j = 0; j < J && !row; ++j)
        if (p->g.col0[j] % 128 || (p->ldb[j] / m) % 8)
          return fail(BDLORA_E_DIVISIBILITY, "downward-compatible COLUMN pool: slice %d must start on a 128-column "
                      "boundary (%d) with blocks of a multiple of 8 columns (%d)", j, p->g.col0[j], p->ldb[j] / m);
    }
  }
  const int64_t elems = slot_elems_for_rank(p, rank, m);
  int64_t off = 0;
  ST_TRY(arena_alloc(p, slot, elems, &off));
  auto retire_old = [&]() {
    if (!reload) return;
    p->resident_elems -= old_elems;
    arena_free(p, old_e.offA[0], old_elems);
  };

  // full source shapes (paper orientation) per mode
  SlotEntry e{};
  e.rs = rs;
  e.re = re;
  e.scale = scale;
  e.loaded = 1;
  const int K = p->g.K;
  int64_t cur = off;
  std::vector<void*> staging;
  auto cleanup = [&]() {
    for (void* s : staging) cudaFree(s);
  };
  auto src_ptr = [&](const void* hsrc, int64_t n_elems, const uint16_t** out) -> int {
    if (src_is_device) {
      *out = (const uint16_t*)hsrc;
      return BDLORA_OK;
    }
    void* dp = nullptr;
    cudaError_t ce = cudaMalloc(&dp, std::max<int64_t>(n_elems, 1) * 2);
    if (ce != cudaSuccess) return fail(BDLORA_E_CUDA, "staging cudaMalloc: %s", cudaGetErrorString(ce));
    staging.push_back(dp);
    ce = cudaMemcpyAsync(dp, hsrc, n_elems * 2, cudaMemcpyHostToDevice, st);
    if (ce != cudaSuccess) return fail(BDLORA_E_CUDA, "staging copy: %s", cudaGetErrorString(ce));
    *out = (const uint16_t*)dp;
    return BDLORA_OK;
  };
  int rc = BDLORA_OK;
  // slot layout [A_0 | A_1 | A_2 | B_0 | B_1 | B_2]: every A block starts on a K-row boundary
  int64_t curB = cur + (int64_t)J * rs * K / (row ? m : 1);
  for (int j = 0; j < J && rc == BDLORA_OK; ++j) {
    const int dout = d.d_out[j];
    const int w = p->ldb[j];
    const uint16_t *sa = nullptr, *sb = nullptr;
    // ---- A_j -> [rs, K] ----
    if (d.parallel == BDLORA_COLUMN && d.sharding == BDLORA_SHARD_NFS) {
      // NFS: A_1 replicated -- the whole d_in x r on every device
      rc = src_ptr(A[j], (int64_t)d.d_in * rank, &sa);
      if (rc) break;
      e.offA[j] = cur;
      rc = gather_to(sa, rank, 0, 0, d.d_in, rank, 1, p->arena + cur, st);
      cur += (int64_t)rs * K;
    } else if (d.parallel == BDLORA_COLUMN) {
      // A_j full d_in x r; shard = columns [i*r/N, (i+1)*r/N) (BD and S-LoRA: column-sharded A_1)
      rc = src_ptr(A[j], (int64_t)d.d_in * rank, &sa);
      if (rc) break;
      e.offA[j] = cur;
      rc = gather_to(sa, rank, 0, i * (rank / N), d.d_in, rank / N, 1, p->arena + cur, st);
      cur += (int64_t)rs * K;
    } else if (d.sharding == BDLORA_SHARD_BD && nb == N) {
      // A_2 compact d_in x r/N, blocks stacked; diagonal block i = rows [i*d_in/N, ...)
      rc = src_ptr(A[0], (int64_t)d.d_in * (rank / N), &sa);
      if (rc) break;
      e.offA[0] = cur;
      rc = gather_to(sa, rank / N, i * K, 0, K, rank / N, 1, p->arena + cur, st);
      cur += (int64_t)rs * K;
    } else if (d.sharding == BDLORA_SHARD_BD) {
      // downward-compatible: compact d_in x r/N_h with N_h stacked blocks; this device runs the
      // blocks b = i*m + bb (m = N_h/N).  Stored compactly, transposed: rank row q = bb * r/N_h + k holds the
      // K/m inputs of its block only, [r/N, K/m] -- the zeros of the block-diagonal A_2 are never stored
      const int rb = rank / nb, kb = d.d_in / nb;
      rc = src_ptr(A[0], (int64_t)d.d_in * rb, &sa);
      if (rc) break;
      e.offA[0] = cur;
      for (int bb = 0; bb < m && rc == BDLORA_OK; ++bb)
        rc = gather_to(sa, rb, (i * m + bb) * kb, 0, kb, rb, 1, p->arena + cur + (int64_t)bb * rb * kb, st, kb);
      cur += (int64_t)rs * kb;
    } else {
      // S-LoRA / NFS row: A_2 d_in x r row-sharded: rows [i*d_in/N, ...)
      rc = src_ptr(A[0], (int64_t)d.d_in * rank, &sa);
      if (rc) break;
      e.offA[0] = cur;
      rc = gather_to(sa, rank, i * K, 0, K, rank, 1, p->arena + cur, st);
      cur += (int64_t)rs * K;
    }
    if (rc) break;
    // ---- B_j -> [re, w] ----
    if (d.parallel == BDLORA_COLUMN && d.sharding == BDLORA_SHARD_BD && nb == N) {
      // compact (r/N) x d_out_j, blocks side by side; diagonal block i = columns [i*w, ...)
      rc = src_ptr(B[j], (int64_t)(rank / N) * dout, &sb);
      if (rc) break;
      e.offB[j] = curB;
      rc = gather_to(sb, dout, 0, i * w, rank / N, w, 0, p->arena + curB, st);
    } else if (d.parallel == BDLORA_COLUMN && d.sharding == BDLORA_SHARD_BD) {
      // downward-compatible: compact (r/N_h) x d_out_j with N_h blocks side by side; this device's
      // m = N_h/N blocks (b = i*m + bb) are the columns [i*w, (i+1)*w) of it -- kept compact, [r/N_h, w]: the
      // local B_1 [r/N, w] is block-diagonal and its zeros are never stored (the expand reads v rows
      // [bb * r/N_h, (bb+1) * r/N_h) for the columns of block bb)
      const int rb = rank / nb;
      rc = src_ptr(B[j], (int64_t)rb * dout, &sb);
      if (rc) break;
      e.offB[j] = curB;
      rc = gather_to(sb, dout, 0, i * w, rb, w, 0, p->arena + curB, st);
    } else if (d.parallel == BDLORA_COLUMN) {
      // S-LoRA / NFS column: B_1 r x d_out_j column-sharded
      rc = src_ptr(B[j], (int64_t)rank * dout, &sb);
      if (rc) break;
      e.offB[j] = curB;
      rc = gather_to(sb, dout, 0, i * w, rank, w, 0, p->arena + curB, st);
    } else if (d.sharding == BDLORA_SHARD_NFS) {
      // NFS row: B_2 replicated -- the whole r x d_out on every device
      rc = src_ptr(B[0], (int64_t)rank * dout, &sb);
      if (rc) break;
      e.offB[0] = curB;
      rc = gather_to(sb, dout, 0, 0, rank, dout, 0, p->arena + curB, st);
    } else if (d.sharding == BDLORA_SHARD_BD) {
      // BD row: B_2 r x d_out row-sharded: rows [i*r/N, ...)
      rc = src_ptr(B[0], (int64_t)rank * dout, &sb);
      if (rc) break;
      e.offB[0] = curB;
      rc = gather_to(sb, dout, i * (rank / N), 0, rank / N, dout, 0, p->arena + curB, st);
    } else {
      // S-LoRA row: B_2 r x d_out column-sharded
      rc = src_ptr(B[0], (int64_t)rank * dout, &sb);
      if (rc) break;
      e.offB[0] = curB;
      rc = gather_to(sb, dout, 0, i * w, rank, w, 0, p->arena + curB, st);
    }
    curB += (int64_t)(row ? re : re / m) * w;
  }
  if (rc != BDLORA_OK) {
    cudaStreamSynchronize(st);
    cleanup();
    if (p->ragged) {
      arena_free(p, off, elems);  // the previous occupant (if any) is untouched
    } else if (reload) {          // fixed arena: the slot's region was partly overwritten
      p->h_tab[slot] = SlotEntry{};
      p->slot_elems[slot] = 0;
      p->resident_elems -= old_elems;
      cudaMemcpy(p->d_tab + slot, &p->h_tab[slot], sizeof(SlotEntry), cudaMemcpyHostToDevice);
    }
    return rc;
  }
  retire_old();
  if (row) p->g.ablk = m;
  else p->g.bblk = m;
  p->h_tab[slot] = e;
  p->slot_elems[slot] = elems;
  p->resident_elems += elems;
  cudaError_t ce = cudaMemcpyAsync(p->d_tab + slot, &p->h_tab[slot], sizeof(SlotEntry), cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);  // host table entry + staging must outlive the copy
  cleanup();
  if (ce != cudaSuccess) return fail(BDLORA_E_CUDA, "load_adapter: %s", cudaGetErrorString(ce));
  (void)off;
  return BDLORA_OK;
}

int bdlora_unload_adapter(bdlora_pool* p, int32_t slot) {
  ST_TRY(check_pool(p));
  if (slot < 0 || slot >= p->d.capacity) return fail(BDLORA_E_CAPACITY, "slot %d out of range [0,%d)", slot, p->d.capacity);
  if (!p->h_tab[slot].loaded) return fail(BDLORA_E_NOT_LOADED, "slot %d is not loaded", slot);
  DeviceGuard dg(p->dev);
  const SlotEntry e = p->h_tab[slot];
  const int64_t elems = p->slot_elems[slot];
  p->h_tab[slot] = SlotEntry{};
  p->slot_elems[slot] = 0;
  p->resident_elems -= elems;
  arena_free(p, e.offA[0], elems);
  CU_TRY(cudaMemcpy(p->d_tab + slot, &p->h_tab[slot], sizeof(SlotEntry), cudaMemcpyHostToDevice));
  return BDLORA_OK;
}

int bdlora_pool_bytes(const bdlora_pool* p, int64_t* resident, int64_t* arena) {
  ST_TRY(check_pool(p));
  if (resident) *resident = p->resident_elems * 2;
  if (arena) *arena = p->arena_elems * 2;
  return BDLORA_OK;
}

int bdlora_pool_geometry(const bdlora_pool* p, int32_t* k_loc, int32_t* m_loc) {
  ST_TRY(check_pool(p));
  if (k_loc) *k_loc = p->g.K;
  if (m_loc) *m_loc = p->g.M;
  return BDLORA_OK;
}

int bdlora_workspace_bytes(const bdlora_pool* p, int64_t T, size_t* bytes) {
  ST_TRY(check_pool(p));
  if (!bytes) return fail(BDLORA_E_ARG, "bytes is NULL");
  if (T < 0) return fail(BDLORA_E_ARG, "T < 0");
  *bytes = ws_layout(p, std::max<int64_t>(T, 1)).total;
  return BDLORA_OK;
}

int bdlora_workspace_init(const bdlora_pool* p, void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_pool(p));
  if (!ws) return fail(BDLORA_E_ARG, "workspace is NULL");
  if (ws_bytes < kCounterBytes)
    return fail(BDLORA_E_ARG, "workspace too small: %zu < %zu bytes (counter region)", ws_bytes, kCounterBytes);
  DeviceGuard dg(p->dev);
  CU_TRY(cudaMemsetAsync(ws, 0, kCounterBytes, (cudaStream_t)stream));
  return BDLORA_OK;
}

int bdlora_last_launch_info(int32_t info[8]) {
  if (!info) return fail(BDLORA_E_ARG, "info is NULL");
  int d[8];
  bdl::dec_last_launch(d);
  for (int k = 0; k < 8; ++k) info[k] = g_last_src == 1 ? d[k] : bdl::g_last_launch[k];
  return BDLORA_OK;
}

int bdlora_v_elems(const bdlora_pool* p, int64_t T, int64_t* elems) {
  ST_TRY(check_pool(p));
  if (!elems) return fail(BDLORA_E_ARG, "elems is NULL");
  *elems = T * p->g.J * p->g.Rc;
  return BDLORA_OK;
}

int bdlora_build_segments(const int32_t* ids, int64_t T, int32_t* seg_start, int32_t* seg_len, int32_t* seg_id,
                          int32_t* n_seg_dev, bdlora_stream_t stream) {
  if (T < 0) return fail(BDLORA_E_ARG, "T < 0");
  if (!n_seg_dev) return fail(BDLORA_E_ARG, "n_seg_dev is NULL");
  if (T > 0 && (!ids || !seg_start || !seg_len || !seg_id)) return fail(BDLORA_E_ARG, "NULL array");
  if (T > (1 << 24)) return fail(BDLORA_E_CAPACITY, "T too large");
  bdl::segments_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(ids, (int)T, seg_start, seg_len, seg_id, n_seg_dev);
  count_launch();
  CU_TRY(cudaGetLastError());
  return BDLORA_OK;
}

// ---------------------------------------------------------------------------- phases
int bdlora_lora_shrink(bdlora_pool* p, const void* X, int64_t T, const int32_t* ids, float* v, void* ws,
                       size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_pool(p));
  if (T == 0) return BDLORA_OK;
  if (!X || !ids || !v) return fail(BDLORA_E_ARG, "X/ids/v is NULL");
  (void)ws;
  (void)ws_bytes;
  DeviceGuard dg(p->dev);
  if (ws && ws_bytes < ws_layout(p, T).total) ws = nullptr;  // too small for the tensor-core path
  return launch_shrink(p, X, (int)T, ids, v, (cudaStream_t)stream, ws);
}

int bdlora_base_expand(bdlora_pool* p, const void* X, int64_t T, const void* W, const int32_t* ids, const float* v,
                       void* Y, void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, Y, ws, ws_bytes));
  if (T == 0) return BDLORA_OK;
  if (!v) return fail(BDLORA_E_ARG, "v is NULL");
  DeviceGuard dg(p->dev);
  return launch_base_expand(p, X, (int)T, W, ids, v, Y, ws, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------- BD-LoRA
static int bd_local(bdlora_pool* p, const void* X, int64_t T, const void* W, const int32_t* ids, void* Y, void* ws,
                    cudaStream_t st) {
  float* v = ws_v(p, ws, T);
  if (pool_blocked(p)) {
    // chunks of <= 64 tokens: shrink, then the decode kernel expanding that chunk's v (the next chunk's shrink
    // overwrites v only after the expand completes: it waits on it, programmatic dependent launch)
    for (int64_t c0 = 0; c0 < T; c0 += bdl::kDecMaxT) {
      const int Tc = (int)std::min<int64_t>(T - c0, bdl::kDecMaxT);
      const void* Xc = (const __nv_bfloat16*)X + (size_t)c0 * p->g.K;
      float* vc = ws_v(p, ws, Tc);
      ST_TRY(launch_shrink(p, Xc, Tc, ids + c0, vc, st, ws));
      ST_TRY(launch_base_expand(p, Xc, Tc, W, ids + c0, vc, (__nv_bfloat16*)Y + (size_t)c0 * p->g.M, ws, st));
    }
    return BDLORA_OK;
  }
  if (bdl::dec_enabled() && bdl::dec_eligible(p->g, (int)T) && decode_klocal_ok(p, (int)T)) {
    // decode: ONE lean kernel -- base GEMM on the tensor cores, K-local LoRA shrink + expand in its epilogue
    const int rc = launch_decode(p, X, (int)T, W, ids, nullptr, Y, ws, st, 1);
    if (rc >= 0) return rc;
  }
  if (p->g.C == 1 && decode_mt_ok(p, (int)T)) {
    // decode batch over many adapters: grid-wide shrink (each distinct adapter's A rows read once), then the
    // decode kernel expands v in its epilogue (programmatic dependent launch: the weights stream meanwhile)
    const int rs = bdl::dec_shrink_launch(p->g, (const __nv_bfloat16*)X, (int)T, ids, p->d_tab,
                                          (const __nv_bfloat16*)p->arena, v, p->num_sms, st, g_pdl, p->rs_max);
    if (rs < 0) return fail(BDLORA_E_CUDA, "decode shrink launch: %s", cudaGetErrorString(cudaGetLastError()));
    if (rs == 0) {
      count_launch();
      const int rc = launch_decode(p, X, (int)T, W, ids, v, Y, ws, st, 4);
      if (rc >= 0) return rc;
      return launch_base_expand(p, X, (int)T, W, ids, v, Y, ws, st);
    }
  }
  if (bdl::umma_eligible(p->g, (int)T) && T <= fused_max_t()) {
    // decode: ONE kernel -- the LoRA shrink runs inside it (K-local on the tensor cores for a single
    // adapter group, else in the epilogue warps) while the weights stream
    const WsLayout L = ws_layout(p, T);
    int rc = bdl::umma_launch(p->g, (const __nv_bfloat16*)X, (int)T, (const __nv_bfloat16*)W, ids, p->d_tab,
                              (const __nv_bfloat16*)p->arena, v, (__nv_bfloat16*)Y, (char*)ws + L.off_umma_cnt,
                              (char*)ws + L.off_umma, p->num_sms, st, g_pdl, v, p->rs_max, /*tcx=*/1, p->amap_ok ? &p->amap : nullptr);
    if (rc == 0) {
      count_launch();
      g_last_src = 0;
      CU_TRY(cudaGetLastError());
      return BDLORA_OK;
    }
  }
  ST_TRY(launch_shrink(p, X, (int)T, ids, v, st, ws));
  // programmatic dependent launch: the GEMM streams W while the shrink runs; only its epilogue waits
  return launch_base_expand(p, X, (int)T, W, ids, v, Y, ws, st);
}

int bdlora_column_forward(bdlora_pool* p, const void* X, int64_t T, const void* W, const int32_t* ids, void* Y,
                          void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, Y, ws, ws_bytes));
  ST_TRY(require_mode(p, BDLORA_COLUMN, BDLORA_SHARD_BD, "bdlora_column_forward"));
  if (T == 0) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  return bd_local(p, X, T, W, ids, Y, ws, (cudaStream_t)stream);
}

int bdlora_row_partial(bdlora_pool* p, const void* X, int64_t T, const void* W, const int32_t* ids, void* P, void* ws,
                       size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, P, ws, ws_bytes));
  ST_TRY(require_mode(p, BDLORA_ROW, BDLORA_SHARD_BD, "bdlora_row_partial"));
  if (T == 0) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  return bd_local(p, X, T, W, ids, P, ws, (cudaStream_t)stream);
}

int bdlora_row_forward(bdlora_pool* p, bdlora_comm* comm, const void* X, int64_t T, const void* W, const int32_t* ids,
                       void* Y, void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, Y, ws, ws_bytes));
  ST_TRY(require_mode(p, BDLORA_ROW, BDLORA_SHARD_BD, "bdlora_row_forward"));
  ST_TRY(require_comm(p, comm, "bdlora_row_forward"));
  if (T == 0) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  cudaStream_t st = (cudaStream_t)stream;
  ST_TRY(bd_local(p, X, T, W, ids, Y, ws, st));
  if (p->d.tp_size > 1) {
    // Alg. 1 line 15: the base model's own all-reduce -- the only collective
    const size_t n = (size_t)T * p->g.M;
    NC_TRY(ncclAllReduce(Y, Y, n, ncclBfloat16, ncclSum, comm->nccl, st));
    comm->counts[0] += 1;
    comm->counts[3] += (int64_t)n * 2;
  }
  return BDLORA_OK;
}

// Alg. 2: column layer + the base model's all-gather of the device outputs -- replicated
// Y [T, N * M_loc] = [Y_0 | Y_1 | ... | Y_{N-1}] (device blocks in rank order; for J = 1 the full output).
int bdlora_column_forward_gather(bdlora_pool* p, bdlora_comm* comm, const void* X, int64_t T, const void* W,
                                 const int32_t* ids, void* Y, void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, Y, ws, ws_bytes));
  ST_TRY(require_mode(p, BDLORA_COLUMN, BDLORA_SHARD_BD, "bdlora_column_forward_gather"));
  ST_TRY(require_comm(p, comm, "bdlora_column_forward_gather"));
  if (T == 0) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const int N = p->d.tp_size;
  if (N == 1) return bd_local(p, X, T, W, ids, Y, ws, st);
  const size_t chunk = (size_t)T * p->g.M;
  if (T == 1) {
    // one token: [Y_0 | ... | Y_{N-1}] is the all-gather's own rank-major layout -- lines 3-6 straight into
    // this rank's block of Y, then the all-gather in place (no staging buffer, no interleave pass)
    __nv_bfloat16* Yb = (__nv_bfloat16*)Y;
    ST_TRY(bd_local(p, X, T, W, ids, Yb + chunk * p->d.tp_rank, ws, st));
    NC_TRY(ncclAllGather(Yb + chunk * p->d.tp_rank, Yb, chunk, ncclBfloat16, comm->nccl, st));
    return BDLORA_OK;
  }
  // Alg. 2 lines 3-6 into this rank's chunk of the staging buffer, then an in-place all-gather (line 8)
  __nv_bfloat16* G = (__nv_bfloat16*)((char*)ws + ws_layout(p, T).off_gather);
  ST_TRY(bd_local(p, X, T, W, ids, G + chunk * p->d.tp_rank, ws, st));
  // the base model's own collective: the LoRA counters of bdlora_comm_stats stay untouched
  NC_TRY(ncclAllGather(G + chunk * p->d.tp_rank, G, chunk, ncclBfloat16, comm->nccl, st));
  const size_t total = chunk * N;
  bdl::interleave_chunks_kernel<<<(unsigned)std::min<size_t>((total + 255) / 256, 65535), 256, 0, st>>>(
      (const uint16_t*)G, (uint16_t*)Y, (int)T, p->g.M, N);
  count_launch();
  CU_TRY(cudaGetLastError());
  return BDLORA_OK;
}

// ---------------------------------------------------------------------------- NFS-LoRA
// Replicated A_1 / B_2: every device's LoRA term is local, so the path is the BD one with
// full-rank factors -- the same single-kernel decode forward, no LoRA collective.
int nfs_column_forward(bdlora_pool* p, const void* X, int64_t T, const void* W, const int32_t* ids, void* Y, void* ws,
                       size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, Y, ws, ws_bytes));
  ST_TRY(require_mode(p, BDLORA_COLUMN, BDLORA_SHARD_NFS, "nfs_column_forward"));
  if (T == 0) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  return bd_local(p, X, T, W, ids, Y, ws, (cudaStream_t)stream);
}

int nfs_row_partial(bdlora_pool* p, const void* X, int64_t T, const void* W, const int32_t* ids, void* P, void* ws,
                    size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, P, ws, ws_bytes));
  ST_TRY(require_mode(p, BDLORA_ROW, BDLORA_SHARD_NFS, "nfs_row_partial"));
  if (T == 0) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  return bd_local(p, X, T, W, ids, P, ws, (cudaStream_t)stream);
}

int nfs_row_forward(bdlora_pool* p, bdlora_comm* comm, const void* X, int64_t T, const void* W, const int32_t* ids,
                    void* Y, void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, Y, ws, ws_bytes));
  ST_TRY(require_mode(p, BDLORA_ROW, BDLORA_SHARD_NFS, "nfs_row_forward"));
  ST_TRY(require_comm(p, comm, "nfs_row_forward"));
  if (T == 0) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  cudaStream_t st = (cudaStream_t)stream;
  ST_TRY(bd_local(p, X, T, W, ids, Y, ws, st));
  if (p->d.tp_size > 1) {
    // the base model's own all-reduce -- the only collective
    const size_t n = (size_t)T * p->g.M;
    NC_TRY(ncclAllReduce(Y, Y, n, ncclBfloat16, ncclSum, comm->nccl, st));
    comm->counts[0] += 1;
    comm->counts[3] += (int64_t)n * 2;
  }
  return BDLORA_OK;
}

// ---------------------------------------------------------------------------- fused row all-reduce (8(f) row 2)
namespace {

int peer_finish_setup(bdlora_peer* q, const std::vector<float*>& recvs, const std::vector<unsigned*>& cnts) {
  const int N = q->nranks;
  CU_TRY(cudaMalloc(&q->d_recv, sizeof(float*) * N));
  CU_TRY(cudaMalloc(&q->d_cnt, sizeof(unsigned*) * N));
  CU_TRY(cudaMemcpy(q->d_recv, recvs.data(), sizeof(float*) * N, cudaMemcpyHostToDevice));
  CU_TRY(cudaMemcpy(q->d_cnt, cnts.data(), sizeof(unsigned*) * N, cudaMemcpyHostToDevice));
  q->dev_view.recv = q->d_recv;
  q->dev_view.cnt = q->d_cnt;
  q->dev_view.parity = q->ctrl + 2;
  q->dev_view.rank = q->rank;
  q->dev_view.nranks = N;
  q->dev_view.slot = q->slot;
  return BDLORA_OK;
}

int peer_alloc_own(bdlora_peer* q) {
  const size_t bytes = sizeof(float) * 2 * (size_t)q->nranks * q->slot;
  CU_TRY(cudaMalloc(&q->recv, bytes));
  CU_TRY(cudaMalloc(&q->ctrl, 256));
  CU_TRY(cudaMemset(q->ctrl, 0, 256));
  CU_TRY(cudaMemset(q->recv, 0, bytes));
  q->owned.push_back(q->recv);
  q->owned.push_back(q->ctrl);
  return BDLORA_OK;
}

int check_row_push(const bdlora_pool* p, const bdlora_peer* q, int64_t T, const char* fn) {
  if (!q) return fail(BDLORA_E_ARG, "%s: peer is NULL", fn);
  if (p->d.parallel != BDLORA_ROW || p->d.sharding == BDLORA_SHARD_SLORA)
    return fail(BDLORA_E_MODE, "%s: needs a ROW pool with BD or NFS sharding", fn);
  if (q->nranks != p->d.tp_size || q->rank != p->d.tp_rank)
    return fail(BDLORA_E_ARG, "%s: peer (nranks=%d, rank=%d) does not match pool (tp_size=%d, tp_rank=%d)", fn,
                q->nranks, q->rank, p->d.tp_size, p->d.tp_rank);
  if (q->dev != p->dev) return fail(BDLORA_E_ARG, "%s: peer device %d != pool device %d", fn, q->dev, p->dev);
  if (T > bdl::kDecMaxPushT || !bdl::dec_eligible(p->g, (int)T) || !decode_klocal_ok(p, (int)T))
    return fail(BDLORA_E_CAPACITY, "%s: the fused all-reduce serves decode batches (T <= %d, K %% 64 == 0, K-local "
                "LoRA capacity); T = %lld -- use bdlora_row_forward", fn, bdl::kDecMaxPushT, (long long)T);
  if ((long long)T * p->g.M > q->slot)
    return fail(BDLORA_E_CAPACITY, "%s: T x d_out = %lld exceeds the peer slot (%lld elements)", fn,
                (long long)T * p->g.M, q->slot);
  return BDLORA_OK;
}

}  // namespace

int bdlora_peer_create(bdlora_comm* comm, int64_t max_elems, bdlora_peer** out) {
  if (!comm || !out) return fail(BDLORA_E_ARG, "comm/out is NULL");
  if (max_elems < 1 || max_elems > (1LL << 32)) return fail(BDLORA_E_ARG, "max_elems = %lld", (long long)max_elems);
  DeviceGuard dg(comm->dev);
  bdlora_peer* q = new bdlora_peer();
  q->dev = comm->dev;
  q->rank = comm->rank;
  q->nranks = comm->nranks;
  q->slot = max_elems;
  int rc = peer_alloc_own(q);
  if (rc) {
    bdlora_peer_destroy(q);
    return rc;
  }
  // exchange the CUDA IPC handles of every rank's receive buffer and control block over the communicator
  const int N = q->nranks;
  cudaIpcMemHandle_t mine[2];
  if (cudaIpcGetMemHandle(&mine[0], q->recv) != cudaSuccess || cudaIpcGetMemHandle(&mine[1], q->ctrl) != cudaSuccess) {
    bdlora_peer_destroy(q);
    return fail(BDLORA_E_CUDA, "cudaIpcGetMemHandle failed");
  }
  void* dbuf = nullptr;
  const size_t hb = sizeof(mine);
  if (cudaMalloc(&dbuf, hb * (N + 1)) != cudaSuccess) {
    bdlora_peer_destroy(q);
    return fail(BDLORA_E_CUDA, "cudaMalloc (handle exchange)");
  }
  std::vector<uint8_t> all(hb * N);
  cudaMemcpy((char*)dbuf + hb * N, mine, hb, cudaMemcpyHostToDevice);
  ncclResult_t nr = ncclAllGather((char*)dbuf + hb * N, dbuf, hb, ncclUint8, comm->nccl, 0);
  cudaError_t ce = cudaStreamSynchronize(0);
  if (ce == cudaSuccess) ce = cudaMemcpy(all.data(), dbuf, hb * N, cudaMemcpyDeviceToHost);
  cudaFree(dbuf);
  if (nr != ncclSuccess || ce != cudaSuccess) {
    bdlora_peer_destroy(q);
    return fail(BDLORA_E_NCCL, "handle exchange: %s / %s", ncclGetErrorString(nr), cudaGetErrorString(ce));
  }
  std::vector<float*> recvs(N);
  std::vector<unsigned*> cnts(N);
  for (int r = 0; r < N; ++r) {
    if (r == q->rank) {
      recvs[r] = q->recv;
      cnts[r] = (unsigned*)q->ctrl;
      continue;
    }
    cudaIpcMemHandle_t h[2];
    memcpy(h, all.data() + hb * r, hb);
    void *pr = nullptr, *pc = nullptr;
    if (cudaIpcOpenMemHandle(&pr, h[0], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&pc, h[1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      bdlora_peer_destroy(q);
      return fail(BDLORA_E_CUDA, "cudaIpcOpenMemHandle (rank %d): %s", r, cudaGetErrorString(cudaGetLastError()));
    }
    q->opened.push_back(pr);
    q->opened.push_back(pc);
    recvs[r] = (float*)pr;
    cnts[r] = (unsigned*)pc;
  }
  rc = peer_finish_setup(q, recvs, cnts);
  if (rc) {
    bdlora_peer_destroy(q);
    return rc;
  }
  *out = q;
  return BDLORA_OK;
}

int bdlora_peer_create_local(int nranks, int cuda_device, int64_t max_elems, bdlora_peer** out) {
  if (!out) return fail(BDLORA_E_ARG, "out is NULL");
  if (nranks < 1 || nranks > 64) return fail(BDLORA_E_ARG, "nranks = %d", nranks);
  if (max_elems < 1 || max_elems > (1LL << 32)) return fail(BDLORA_E_ARG, "max_elems = %lld", (long long)max_elems);
  ST_TRY(bdlora_device_check(cuda_device));
  DeviceGuard dg(cuda_device);
  std::vector<bdlora_peer*> qs(nranks, nullptr);
  std::vector<float*> recvs(nranks);
  std::vector<unsigned*> cnts(nranks);
  int rc = BDLORA_OK;
  for (int r = 0; r < nranks && rc == BDLORA_OK; ++r) {
    qs[r] = new bdlora_peer();
    qs[r]->dev = cuda_device;
    qs[r]->rank = r;
    qs[r]->nranks = nranks;
    qs[r]->slot = max_elems;
    rc = peer_alloc_own(qs[r]);
    if (rc == BDLORA_OK) {
      recvs[r] = qs[r]->recv;
      cnts[r] = (unsigned*)qs[r]->ctrl;
    }
  }
  for (int r = 0; r < nranks && rc == BDLORA_OK; ++r) rc = peer_finish_setup(qs[r], recvs, cnts);
  if (rc) {
    for (auto* q : qs)
      if (q) bdlora_peer_destroy(q);
    return rc;
  }
  for (int r = 0; r < nranks; ++r) out[r] = qs[r];
  return BDLORA_OK;
}

int bdlora_peer_destroy(bdlora_peer* q) {
  if (!q) return BDLORA_OK;
  DeviceGuard dg(q->dev);
  cudaDeviceSynchronize();
  for (void* pp : q->opened) cudaIpcCloseMemHandle(pp);
  for (void* pp : q->owned) cudaFree(pp);
  if (q->d_recv) cudaFree(q->d_recv);
  if (q->d_cnt) cudaFree(q->d_cnt);
  delete q;
  return BDLORA_OK;
}

int bdlora_peer_error(const bdlora_peer* q, int32_t* err) {
  if (!q || !err) return fail(BDLORA_E_ARG, "peer/err is NULL");
  DeviceGuard dg(q->dev);
  int v = 0;
  CU_TRY(cudaMemcpy(&v, q->ctrl + 4, sizeof(int), cudaMemcpyDeviceToHost));
  *err = v;
  return BDLORA_OK;
}

int bdlora_row_partial_push(bdlora_pool* p, bdlora_peer* q, const void* X, int64_t T, const void* W,
                            const int32_t* ids, void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, (const void*)1, ws, ws_bytes));
  if (T == 0) return BDLORA_OK;
  ST_TRY(check_row_push(p, q, T, "bdlora_row_partial_push"));
  DeviceGuard dg(p->dev);
  g_push = q;
  const int rc = launch_decode(p, X, (int)T, W, ids, nullptr, nullptr, ws, (cudaStream_t)stream, 1);
  g_push = nullptr;
  if (rc < 0) return fail(BDLORA_E_CAPACITY, "bdlora_row_partial_push: shape not served by the decode kernel");
  return rc;
}

int bdlora_peer_reduce(bdlora_peer* q, void* Y, int64_t T, int32_t M, bdlora_stream_t stream) {
  if (!q) return fail(BDLORA_E_ARG, "peer is NULL");
  if (T < 0 || M < 1) return fail(BDLORA_E_ARG, "T = %lld, M = %d", (long long)T, M);
  if (T == 0) return BDLORA_OK;
  if (!Y) return fail(BDLORA_E_ARG, "Y is NULL");
  if ((long long)T * M > q->slot) return fail(BDLORA_E_CAPACITY, "T x M exceeds the peer slot");
  if (q->last_grid <= 0) return fail(BDLORA_E_ARG, "bdlora_peer_reduce: no push was issued on this peer");
  DeviceGuard dg(q->dev);
  const unsigned expected = (unsigned)q->nranks * (unsigned)q->last_grid;
  if (bdl::peer_reduce_launch(q->recv, (unsigned*)q->ctrl, q->ctrl + 2, q->ctrl + 3, q->ctrl + 4, expected, q->nranks,
                              q->slot, (__nv_bfloat16*)Y, (int)T, M, g_pdl, (cudaStream_t)stream) != 0)
    return fail(BDLORA_E_CUDA, "peer reduce launch: %s", cudaGetErrorString(cudaGetLastError()));
  count_launch();
  return BDLORA_OK;
}

int bdlora_row_forward_fused(bdlora_pool* p, bdlora_peer* q, const void* X, int64_t T, const void* W,
                             const int32_t* ids, void* Y, void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, Y, ws, ws_bytes));
  if (T == 0) return BDLORA_OK;
  ST_TRY(bdlora_row_partial_push(p, q, X, T, W, ids, ws, ws_bytes, stream));
  return bdlora_peer_reduce(q, Y, T, p->g.M, stream);
}

// ---------------------------------------------------------------------------- S-LoRA
int slora_column_forward(bdlora_pool* p, bdlora_comm* comm, const void* X, int64_t T, const void* W,
                         const int32_t* ids, void* Y, void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, Y, ws, ws_bytes));
  ST_TRY(require_mode(p, BDLORA_COLUMN, BDLORA_SHARD_SLORA, "slora_column_forward"));
  ST_TRY(require_comm(p, comm, "slora_column_forward"));
  if (T == 0) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  cudaStream_t st = (cudaStream_t)stream;
  float* v = ws_v(p, ws, T);  // [N][T][J][Rc]
  const size_t chunk = (size_t)T * p->g.J * p->g.Rc;
  // matmul_3 into this rank's chunk, then the merged all-gather
  ST_TRY(launch_shrink(p, X, (int)T, ids, v + chunk * p->d.tp_rank, st, ws));
  if (p->d.tp_size > 1) {
    NC_TRY(ncclAllGather(v + chunk * p->d.tp_rank, v, chunk, ncclFloat32, comm->nccl, st));
    comm->counts[1] += 1;
    comm->counts[4] += (int64_t)chunk * 4;
  }
  return launch_base_expand(p, X, (int)T, W, ids, v, Y, ws, st);
}

int slora_row_forward(bdlora_pool* p, bdlora_comm* comm, const void* X, int64_t T, const void* W, const int32_t* ids,
                      void* Y, void* ws, size_t ws_bytes, bdlora_stream_t stream) {
  ST_TRY(check_fwd_args(p, X, T, W, ids, Y, ws, ws_bytes));
  ST_TRY(require_mode(p, BDLORA_ROW, BDLORA_SHARD_SLORA, "slora_row_forward"));
  ST_TRY(require_comm(p, comm, "slora_row_forward"));
  if (T == 0) return BDLORA_OK;
  DeviceGuard dg(p->dev);
  cudaStream_t st = (cudaStream_t)stream;
  float* v = ws_v(p, ws, T);  // [T][1][Rc = max_rank]
  ST_TRY(launch_shrink(p, X, (int)T, ids, v, st, ws));
  if (p->d.tp_size > 1) {
    // all-reduce after matmul_5
    const size_t n = (size_t)T * p->g.Rc;
    NC_TRY(ncclAllReduce(v, v, n, ncclFloat32, ncclSum, comm->nccl, st));
    comm->counts[2] += 1;
    comm->counts[5] += (int64_t)n * 4;
  }
  ST_TRY(launch_base_expand(p, X, (int)T, W, ids, v, Y, ws, st));
  if (p->d.tp_size > 1) {
    const size_t n = (size_t)T * p->g.M;
    NC_TRY(ncclAllReduce(Y, Y, n, ncclBfloat16, ncclSum, comm->nccl, st));
    comm->counts[0] += 1;
    comm->counts[3] += (int64_t)n * 2;
  }
  return BDLORA_OK;
}

}  // extern "C"
