// kernels_route.cuh -- routing metadata for the tensor-core shrink (matmul_3 / matmul_5 on tcgen05).
//
// For a batch of T tokens with adapter ids (−1 = none), computes on the device (no host round trip,
// CUDA-graph capturable):
//   groups : the DISTINCT adapters of the batch in order of first appearance (SGMV grouping without a
//            permutation: runs of equal ids are segments (reading R10); a group gathers every segment of
//            the same adapter, so each A row is streamed once per distinct adapter);
//   items  : the 16-row boxes of A the shrink GEMM computes -- for each group g, slice j and 16-row block b
//            of the adapter's rs rows: the arena row of the box (TMA coordinate), g, j, k0 = 16 b, rows.
// One CTA of 1024 threads.
#pragma once
#include "common.cuh"

namespace bdl {

constexpr int kRouteMaxSeg = 4096;
constexpr int kRouteMaxGroups = 1024;
constexpr int kRouteMaxItems = 4096;

// workspace layout (int32 words)
struct RouteLayout {
  static constexpr int kHdr = 0;                                   // [0] n_groups [1] n_items [2] overflow
  static constexpr int kGroupId = 4;                               // [kRouteMaxGroups]
  static constexpr int kItemRow = kGroupId + kRouteMaxGroups;      // [kRouteMaxItems] arena row of the box
  static constexpr int kItemG = kItemRow + kRouteMaxItems;         // group index
  static constexpr int kItemJ = kItemG + kRouteMaxItems;           // slice
  static constexpr int kItemK0 = kItemJ + kRouteMaxItems;          // first rank row of the box
  static constexpr int kItemN = kItemK0 + kRouteMaxItems;          // valid rows in the box (<= 16)
  static constexpr int kWords = kItemN + kRouteMaxItems;
};

__device__ __forceinline__ int block_excl_scan_1024(int x, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = s_warp[lane];
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    s_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  const int r = s_warp[warp] + incl - x;
  *total = s_warp[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) route_kernel(const int* __restrict__ ids, int T,
                                                     const SlotEntry* __restrict__ tab, Geom g, int* __restrict__ route,
                                                     float* __restrict__ v, int nv) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // ids and the slot table are not written by the kernel preceding a forward (include/bdlora.h,
  // bdlora_set_pdl), so segments and groups are found in shared memory while that kernel finishes; the
  // workspace (route tables, v) is written only after the programmatic-dependency wait
  __shared__ int s_seg_id[kRouteMaxSeg];
  __shared__ int s_grp_id[kRouteMaxGroups];  // the groups, kept here until the dependency wait
  __shared__ int s_warp[33];
  __shared__ int s_nseg, s_ngrp;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_nseg = 0;
    s_ngrp = 0;
  }
  __syncthreads();
  // pass 1: segment starts in token order (maximal runs of equal ids)
  int overflow = 0;
  for (int base = 0; base < T; base += 1024) {
    const int t = base + tid;
    int flag = 0, a = -1;
    if (t < T) {
      a = ids[t];
      flag = (t == 0) || (ids[t - 1] != a);
    }
    int tot;
    const int pos = s_nseg + block_excl_scan_1024(flag, s_warp, &tot);
    if (flag && pos < kRouteMaxSeg) s_seg_id[pos] = a;
    __syncthreads();
    if (tid == 0) s_nseg += tot;
    __syncthreads();
  }
  const int nseg = min(s_nseg, kRouteMaxSeg);
  if (s_nseg > kRouteMaxSeg) overflow = 1;
  // pass 2 + 3: groups = segment starts whose id is >= 0 and did not appear in an earlier segment
  for (int base = 0; base < nseg; base += 1024) {
    const int s = base + tid;
    int lead = 0, a = -1;
    if (s < nseg) {
      a = s_seg_id[s];
      lead = a >= 0;
      for (int s2 = 0; s2 < s && lead; ++s2) lead = (s_seg_id[s2] != a);
    }
    int tot;
    const int pos = s_ngrp + block_excl_scan_1024(lead, s_warp, &tot);
    if (lead && pos < kRouteMaxGroups) s_grp_id[pos] = a;
    __syncthreads();
    if (tid == 0) s_ngrp += tot;
    __syncthreads();
  }
  const int ngrp = min(s_ngrp, kRouteMaxGroups);
  if (s_ngrp > kRouteMaxGroups) overflow = 1;
  __syncthreads();
  // the route tables may still be read by a preceding kernel that shares this workspace (the previous
  // forward's shrink): written only after the programmatic-dependency wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int gi = tid; gi < ngrp; gi += 1024) route[RouteLayout::kGroupId + gi] = s_grp_id[gi];
  // pass 4: items (16-row A boxes) per group, exclusive scan of the per-group counts
  int n_items = 0;
  for (int base = 0; base < ngrp; base += 1024) {
    const int gi = base + tid;
    int cnt = 0, a = -1, rs = 0;
    if (gi < ngrp) {
      a = s_grp_id[gi];
      rs = tab[a].rs;
      cnt = g.J * ((rs + 15) / 16);
    }
    int tot;
    const int pos = n_items + block_excl_scan_1024(cnt, s_warp, &tot);
    if (gi < ngrp) {
      int q = pos;
      for (int j = 0; j < g.J; ++j)
        for (int k0 = 0; k0 < rs; k0 += 16, ++q) {
          if (q >= kRouteMaxItems) continue;
          route[RouteLayout::kItemRow + q] = (int)(tab[a].offA[j] / g.K) + k0;
          route[RouteLayout::kItemG + q] = gi;
          route[RouteLayout::kItemJ + q] = j;
          route[RouteLayout::kItemK0 + q] = k0;
          route[RouteLayout::kItemN + q] = min(16, rs - k0);
        }
    }
    n_items += tot;
  }
  if (n_items > kRouteMaxItems) overflow = 1;
  if (tid == 0) {
    route[RouteLayout::kHdr + 0] = ngrp;
    route[RouteLayout::kHdr + 1] = min(n_items, kRouteMaxItems);
    route[RouteLayout::kHdr + 2] = overflow;
  }
  // the shrink GEMM accumulates v with fp32 reductions: start from zero
  for (int i = threadIdx.x; i < nv; i += 1024) v[i] = 0.f;
}

}  // namespace bdl
