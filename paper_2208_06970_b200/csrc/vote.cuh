// vote.cuh -- phi-propagated weighted-centroid vote and clamped site move
// (centroidal_update, tessellation.py:211-248).
//
// phi(v), the first line-of-sight ancestor (_kernels.py:457-486), is found
// by chasing src inside the vote kernels (chains are short: depth <= ~13).
//
// Two ways to form the per-site sums of _kernels.py:513-532, both bit-exact
// with the reference's increasing-voxel-order fp64 accumulation:
//   * EXACT path (unit weights, power-of-two spacing): every term is a
//     multiple of s/2 and every partial sum is exactly representable, so
//     the sequential fp64 sum equals the exact integer sum. Kernels reduce
//     (2x+1) integers with warp match/reduce + 64-bit integer atomics and
//     scale once: order-independent AND identical to the reference.
//   * ORDERED path (any weights): the site's bounding box walked in voxel
//     order finds its region's voxels; four lanes add their terms
//     (w, RN(w*ax), RN(w*ay), RN(w*az)) in exactly the reference order
//     (k_vote_prep, then the walk / sum kernels below). The earlier
//     variant -- a stable radix sort of (site, (phi(v), v)) pairs, then
//     k_vote_sum over the segments -- stays behind LRCVT_VOTE=sort.
#pragma once
#include "common.cuh"
#include "mg.cuh"

namespace lrcvt {

// first LOS ancestor: follow src until src[u] == u (_kernels.py:473-481)
__device__ __forceinline__ int phi_chase(const int2* __restrict__ ss, int v, int2 a) {
  int u = v;
  while (a.y != u && a.y >= 0) {
    u = a.y;
    a = ss[u];
  }
  return u;
}

// EXACT path. acc layout: [4][S] u64 = count, sum(2x+1), sum(2y+1), sum(2z+1).
template <bool MG>
__global__ void __launch_bounds__(256) k_vote_exact(const int* __restrict__ list, int n, Geo g,
                                                    const int2* __restrict__ ss,
                                                    unsigned long long* __restrict__ acc,
                                                    int n_sites, const PeerView* __restrict__ pv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    int s = -1;
    unsigned cx = 0, cy = 0, cz = 0;
    if (i < n) {
      const int v = list[i];
      const int2 a = ss[v];
      s = a.x;
      if (s >= 0) {
        const int u = phi_chase_pv<MG>(pv, ss, v, a);
        int x, y, z;
        coords(g, u, x, y, z);
        cx = 2u * x + 1u; cy = 2u * y + 1u; cz = 2u * z + 1u;
      }
    }
    const unsigned grp = __match_any_sync(0xffffffffu, s);
    const unsigned one = s >= 0 ? 1u : 0u;
    const unsigned c0 = __reduce_add_sync(grp, one);
    const unsigned c1 = __reduce_add_sync(grp, cx);
    const unsigned c2 = __reduce_add_sync(grp, cy);
    const unsigned c3 = __reduce_add_sync(grp, cz);
    const int lane = threadIdx.x & 31;
    if (s >= 0 && lane == __ffs(grp) - 1) {
      atomicAdd(acc + s, (unsigned long long)c0);
      atomicAdd(acc + n_sites + s, (unsigned long long)c1);
      atomicAdd(acc + 2 * n_sites + s, (unsigned long long)c2);
      atomicAdd(acc + 3 * n_sites + s, (unsigned long long)c3);
    }
  }
}

__global__ void k_vote_exact_finish(const unsigned long long* __restrict__ acc, int n_sites,
                                    double hx, double hy, double hz,
                                    double* __restrict__ sums) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sites) return;
  sums[s] = (double)acc[s];
  sums[n_sites + s] = __dmul_rn((double)acc[n_sites + s], hx);
  sums[2 * n_sites + s] = __dmul_rn((double)acc[2 * n_sites + s], hy);
  sums[3 * n_sites + s] = __dmul_rn((double)acc[3 * n_sites + s], hz);
}

// ordered path, step 1 without a term array: key = site (n_sites when
// unassigned) and the (phi(v), v) pair; the terms are formed again inside
// the summing warps from the voxel's weight and its LOS ancestor's centre
__global__ void __launch_bounds__(256) k_vote_pairs(const int* __restrict__ list, int n,
                                                    const int2* __restrict__ ss, int n_sites,
                                                    int* __restrict__ key, unsigned long long* __restrict__ pv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int v = list[i];
    const int2 a = ss[v];
    if (a.x < 0) {
      key[i] = n_sites;
      pv[i] = 0ull;
      continue;
    }
    key[i] = a.x;
    const int u = phi_chase(ss, v, a);
    pv[i] = ((unsigned long long)(unsigned)u << 32) | (unsigned)v;
  }
}

// acc + t[0] + t[1] + ... + t[cnt-1] left to right (the reference's
// sequential accumulation), t[q] = col[4 * q]: the staged terms are loaded
// 16 at a time ahead of the dependent adds, so the chain runs at add latency
// instead of shared-memory load latency per term.
__device__ __forceinline__ double ordered_add(double acc, const double* col, int cnt) {
#pragma unroll
  for (int h = 0; h < 32; h += 16) {
    if (h >= cnt) break;
    double t[16];
#pragma unroll
    for (int q = 0; q < 16; q++) t[q] = col[4 * (h + q)];
#pragma unroll
    for (int q = 0; q < 16; q++)
      if (h + q < cnt) acc = __dadd_rn(acc, t[q]);
  }
  return acc;
}

// weight m_v**gamma of voxel v (seeding.py:68 for the modes the device forms)
__device__ __forceinline__ double vote_weight(int v, const double* __restrict__ w64, const float* __restrict__ w32,
                                              int w_mode) {
  if (w_mode == 0) return 1.0;
  if (w_mode == 1) return __ldg(w64 + v);
  const double m = (double)__ldg(w32 + v);
  return w_mode == 2 ? m : __dmul_rn(m, m);  // m**1.0 / m**2.0
}

// the term of voxel v (weight w) with LOS ancestor u: (w, RN(w*ax), RN(w*ay),
// RN(w*az)) (_kernels.py:520-531)
__device__ __forceinline__ double4 vote_term(const Geo& g, int u, double w) {
  int x, y, z;
  coords(g, u, x, y, z);
  return make_double4(w, __dmul_rn(w, centre1(x, g.sx)), __dmul_rn(w, centre1(y, g.sy)),
                      __dmul_rn(w, centre1(z, g.sz)));
}

// (x, y, z) of voxel u packed 10 bits each (Geo::pack10: every axis <= 1024)
__device__ __forceinline__ int phi_pack(const Geo& g, int u) {
  int x, y, z;
  coords(g, u, x, y, z);
  return x | (y << 10) | (z << 20);
}
__device__ __forceinline__ double4 vote_term_packed(const Geo& g, int p, double w) {
  const int x = p & 1023, y = (p >> 10) & 1023, z = p >> 20;
  return make_double4(w, __dmul_rn(w, centre1(x, g.sx)), __dmul_rn(w, centre1(y, g.sy)),
                      __dmul_rn(w, centre1(z, g.sz)));
}

// ordered path, step 3: one warp per site. A three-stage software pipeline
// per lane -- (phi, v) pairs two batches ahead, the weight one batch ahead,
// the term for the batch being summed -- keeps loads off the critical path;
// lanes 0-3 add the staged terms in voxel order (x, y, z, w chains).
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_vote_sum(const unsigned long long* __restrict__ pv,
                                                         const int* __restrict__ seg_begin,
                                                         const int* __restrict__ seg_end, int n_sites, Geo g,
                                                         const double* __restrict__ w64,
                                                         const float* __restrict__ w32, int w_mode,
                                                         double* __restrict__ sums) {
  __shared__ double buf[WARPS][32][4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int s = blockIdx.x * WARPS + wid;
  if (s >= n_sites) return;
  const int b = seg_begin[s], e = seg_end[s];
  double acc = 0.0;
  auto pair_at = [&](int j) { return j < e ? pv[j] : 0ull; };
  unsigned long long q1 = pair_at(b + lane), q2 = pair_at(b + 32 + lane);  // batches j0, j0 + 32
  double w1 = b + lane < e ? vote_weight((int)(unsigned)(q1 & 0xffffffffull), w64, w32, w_mode) : 0.0;
  for (int j0 = b; j0 < e; j0 += 32) {
    const double4 t = j0 + lane < e ? vote_term(g, (int)(unsigned)(q1 >> 32), w1) : make_double4(0, 0, 0, 0);
    // advance the pipeline before the serial adds so its loads overlap them
    const unsigned long long q3 = pair_at(j0 + 64 + lane);
    const double w2 = j0 + 32 + lane < e ? vote_weight((int)(unsigned)(q2 & 0xffffffffull), w64, w32, w_mode) : 0.0;
    buf[wid][lane][0] = t.x; buf[wid][lane][1] = t.y; buf[wid][lane][2] = t.z; buf[wid][lane][3] = t.w;
    __syncwarp();
    const int cnt = min(32, e - j0);
    if (lane < 4) {
      acc = ordered_add(acc, &buf[wid][0][lane], cnt);
    }
    __syncwarp();
    q1 = q2; q2 = q3; w1 = w2;
  }
  if (lane < 4) sums[lane * n_sites + s] = acc;
}

// ---------------------------------------------------------------------------
// ORDERED path without a sort: every site's voxels, in increasing voxel
// order, are exactly the voxels of its region met by a row-major walk over
// the region's bounding box (the box's own flat order is a sub-order of the
// volume's x-fastest order). Two kernels:
//   k_vote_prep  over the eligible list (voxel order): phi by chasing src,
//                (site, phi) stored per voxel, per-site bounding box by warp
//                match + reduce_min/max and six atomics per site group;
//   k_vote_nseg .. k_vote_add  the boxes walked in parallel segments that
//                compact each region's voxels in voxel order, then one warp
//                per site adds their terms in that order -- the reference's
//                exact accumulation order (_kernels.py:519-531).
// The per-voxel entries are two int planes: site vs[v] and phi vs[n + v]
// (the walks read the 4-byte site of every box voxel and the phi of their
// own voxels only). A voxel belongs to region s iff vs[v] == s: the site
// plane is reset to -1 whenever the eligible set is rebuilt, and
// k_vote_prep writes every eligible voxel, so no stale entry survives.
constexpr int BOX_BIG = 0x3fffffff;
constexpr int VS_DEPTH = 4;  // batches of loads in flight per warp in k_vote_walk (x2) / k_vote_add


template <bool MG>
__global__ void __launch_bounds__(256) k_vote_prep(const int* __restrict__ list, int n, Geo g,
                                                   const int2* __restrict__ ss, int* __restrict__ vs,
                                                   int* __restrict__ box, int n_sites,
                                                   const PeerView* __restrict__ pv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    int s = -1, x = 0, y = 0, z = 0;
    if (i < n) {
      const int v = list[i];
      const int2 a = ss[v];
      s = a.x;
      int u = -1;
      if (s >= 0) {
        u = phi_chase_pv<MG>(pv, ss, v, a);
        coords(g, v, x, y, z);
      }
      // phi as packed coordinates when every axis fits 10 bits (saves the
      // scan a flat-index decode per term), else the flat index
      vs[v] = s;
      vs[g.n + v] = u >= 0 && g.pack10 ? phi_pack(g, u) : u;
    }
    const unsigned grp = __match_any_sync(0xffffffffu, s);
    const int x0 = __reduce_min_sync(grp, x), x1 = __reduce_max_sync(grp, x);
    const int y0 = __reduce_min_sync(grp, y), y1 = __reduce_max_sync(grp, y);
    const int z0 = __reduce_min_sync(grp, z), z1 = __reduce_max_sync(grp, z);
    if (s >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) {
      atomicMin(box + s, x0);
      atomicMin(box + n_sites + s, y0);
      atomicMin(box + 2 * n_sites + s, z0);
      atomicMax(box + 3 * n_sites + s, x1);
      atomicMax(box + 4 * n_sites + s, y1);
      atomicMax(box + 5 * n_sites + s, z1);
    }
  }
}

// Largest boxes first: k_vote_add runs one warp per site and its time
// follows the region size (a few 50k-voxel regions among 3.8k-voxel medians
// at C4); in site order the last waves ran a handful of long warps on an
// otherwise idle GPU. Sites are bucketed by floor(log2(box volume)) and
// taken bucket by bucket, biggest first (order within a bucket is free:
// every site's chain is independent).
constexpr int VO_BUCKETS = 64;
__device__ __forceinline__ int vote_bucket(const int* __restrict__ box, int n_sites, int s) {
  const long long w = box[3 * n_sites + s] - box[s] + 1, h = box[4 * n_sites + s] - box[n_sites + s] + 1,
                  d = box[5 * n_sites + s] - box[2 * n_sites + s] + 1;
  if (w <= 0 || h <= 0 || d <= 0) return 0;
  return 63 - __clzll((unsigned long long)(w * h * d));
}

// hist[VO_BUCKETS] (zeroed by the caller) += sites per bucket
__global__ void k_vote_order_hist(const int* __restrict__ box, int n_sites, int* __restrict__ hist) {
  __shared__ int sh[VO_BUCKETS];
  for (int b = threadIdx.x; b < VO_BUCKETS; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_sites) atomicAdd(&sh[vote_bucket(box, n_sites, s)], 1);
  __syncthreads();
  for (int b = threadIdx.x; b < VO_BUCKETS; b += blockDim.x)
    if (sh[b]) atomicAdd(hist + b, sh[b]);
}

// order[] = site ids, largest bucket first; cursor[VO_BUCKETS] zeroed by the caller
__global__ void k_vote_order_scatter(const int* __restrict__ box, int n_sites, const int* __restrict__ hist,
                                     int* __restrict__ cursor, int* __restrict__ order) {
  __shared__ int base[VO_BUCKETS];
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int b = VO_BUCKETS - 1; b >= 0; b--) {
      base[b] = acc;
      acc += hist[b];
    }
  }
  __syncthreads();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sites) return;
  const int b = vote_bucket(box, n_sites, s);
  order[base[b] + atomicAdd(cursor + b, 1)] = s;
}

__global__ void k_box_init(int* __restrict__ box, int n_sites) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sites) return;
  box[s] = box[n_sites + s] = box[2 * n_sites + s] = BOX_BIG;
  box[3 * n_sites + s] = box[4 * n_sites + s] = box[5 * n_sites + s] = -1;
}

// One warp per site; a (WARPS x 32 x 4) shared stage holds a chunk's terms.
// The walk covers the box rows inside planes [zlo, zhi) (the whole volume on
// one GPU). mode 0: every site, chains start at 0 (or init[s]); multi-GPU
// slab steps: mode 1 = only sites whose box starts in this slab (chains
// start at 0), mode 2 = only sites whose box starts in an earlier slab
// (chains continue from init[s], the running sums handed over by the
// previous slab). Sites a mode skips are left untouched in `sums`.
// acc + t[0] + ... + t[cnt-1] left to right over a chunk's staged terms
// (row = one chain, 32 slots, slots >= cnt hold +0.0): groups of 8 loaded
// ahead of their dependent adds, no per-term predicate. Adding the +0.0 pads
// is exact -- acc starts at +0.0 and so can never become -0.0 -- so the chain
// equals the reference's sequential sum (_kernels.py:528-531).
constexpr int VS_ROW = 34;  // doubles per staged row (16-byte aligned, staggered banks)
__device__ __forceinline__ double ordered_add_padded(double acc, const double* row, int cnt) {
  for (int h = 0; h < cnt; h += 8) {
    const double2 a = *reinterpret_cast<const double2*>(row + h);
    const double2 b = *reinterpret_cast<const double2*>(row + h + 2);
    const double2 c = *reinterpret_cast<const double2*>(row + h + 4);
    const double2 d = *reinterpret_cast<const double2*>(row + h + 6);
    acc = __dadd_rn(acc, a.x); acc = __dadd_rn(acc, a.y);
    acc = __dadd_rn(acc, b.x); acc = __dadd_rn(acc, b.y);
    acc = __dadd_rn(acc, c.x); acc = __dadd_rn(acc, c.y);
    acc = __dadd_rn(acc, d.x); acc = __dadd_rn(acc, d.y);
  }
  return acc;
}

// The walk of site s in this call: its box rows inside planes [zlo, zhi);
// false when the mode skips the site. mode 0: every site, chains start at 0;
// multi-GPU slab steps: mode 1 = only sites whose box starts in this slab
// (chains start at 0), mode 2 = only sites whose box starts in an earlier
// slab (chains continue from init[s], the running sums handed over by the
// previous slab). Sites a mode skips are left untouched in the sums.
struct VoteRange {
  int x0, y0, z0, W, H, D;
  long long T;  // box voxels to walk (0: none)
};
__device__ __forceinline__ bool vote_range(const int* __restrict__ box, int n_sites, int s, int zlo, int zhi,
                                           int mode, VoteRange& r) {
  const int bz0 = box[2 * n_sites + s], bz1 = box[5 * n_sites + s];
  if (mode == 1 && !(bz0 >= zlo && bz0 < zhi)) return false;
  if (mode == 2 && !(bz0 < zlo && bz1 >= zlo)) return false;
  r.x0 = box[s];
  r.y0 = box[n_sites + s];
  r.z0 = bz0 > zlo ? bz0 : zlo;
  const int z1 = bz1 < zhi - 1 ? bz1 : zhi - 1;
  r.W = box[3 * n_sites + s] - r.x0 + 1;
  r.H = box[4 * n_sites + s] - r.y0 + 1;
  r.D = z1 - r.z0 + 1;
  r.T = (r.W > 0 && r.H > 0 && r.D > 0) ? (long long)r.W * r.H * r.D : 0;
  return true;
}

// The ordered chains, walk and sum apart. The box walk has no order
// dependence, only the sum does, so the walk runs in parallel and the
// sequential part reads densely packed terms:
//   k_vote_nseg   per site: its walk (the box rows in this call's planes)
//                 cut into VS_SEG-voxel segments of flat box order;
//   k_scan_excl   segment numbering per site (exclusive prefix sums);
//   k_vote_walk   one warp per segment, grid-stride: COUNT = how many of
//                 the segment's voxels belong to the site; after a prefix sum
//                 over the counts, WRITE = those voxels' (phi, v) in voxel
//                 order at the segment's offset. Each site's entries end up
//                 contiguous and in increasing voxel order, every in-band
//                 voxel exactly once (a counting sort by site, stable);
//   k_vote_add    one warp per site, largest boxes first: lanes form 32
//                 terms at a time (weights and entries loaded ahead), lanes
//                 0-3 add them in order -- the reference's accumulation
//                 (_kernels.py:519-531), so the sums are bit-identical.
// (The previous one-warp-per-site walk that summed as it went was bound by
// its largest boxes: 3.6 ms per C4 iteration, 1.6 ms on one of 8 slabs.)
constexpr int VS_SEG = 4096;

// nseg[s] = segments of site s's walk in this call (0: mode skips it / empty box)
__global__ void k_vote_nseg(const int* __restrict__ box, int n_sites, int zlo, int zhi, int mode,
                            int* __restrict__ nseg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sites) return;
  VoteRange rg;
  nseg[s] = vote_range(box, n_sites, s, zlo, zhi, mode, rg) ? (int)((rg.T + VS_SEG - 1) / VS_SEG) : 0;
}

// out[i] = in[0] + ... + in[i-1] over n values, *total = the sum (one CTA;
// every thread scans a contiguous run)
constexpr int SCAN_THREADS = 1024;
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_excl(const int* __restrict__ in, int n, int* __restrict__ out,
                                                            int* __restrict__ total) {
  __shared__ int wsum[SCAN_THREADS / 32];
  const int per = (n + SCAN_THREADS - 1) / SCAN_THREADS;
  const int i0 = min(n, threadIdx.x * per), i1 = min(n, i0 + per);
  int mine = 0;
  for (int i = i0; i < i1; i++) mine += in[i];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int w = 0; w < SCAN_THREADS / 32; w++) {
      const int t = wsum[w];
      wsum[w] = acc;
      acc += t;
    }
    *total = acc;
  }
  __syncthreads();
  int run = wsum[wid] + incl - mine;
  for (int i = i0; i < i1; i++) {
    const int v = in[i];
    out[i] = run;
    run += v;
  }
}

// the site whose segment range [seg0[s], seg0[s] + nseg[s]) holds segment k
__device__ __forceinline__ int vote_seg_site(const int* __restrict__ seg0, int n_sites, int k) {
  int lo = 0, hi = n_sites - 1;  // largest s with seg0[s] <= k (empty sites share their successor's start)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(seg0 + mid) <= k) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// cnt[k] += the voxels of segment k's site that fall in it, counted from the
// eligible list (every voxel of a region is on it, in voxel order, so a warp's
// voxels mostly share one (site, segment): match + one atomic per group) --
// the same counts as a COUNT walk of the boxes at a third of the bytes.
// cnt is zeroed by the caller.
__global__ void __launch_bounds__(256) k_vote_count(const int* __restrict__ list, const int* __restrict__ n_list,
                                                    const int* __restrict__ vs, const int* __restrict__ box,
                                                    int n_sites, Geo g, int zlo, int zhi, int mode,
                                                    const int* __restrict__ seg0, int* __restrict__ cnt) {
  const int n = *n_list;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < n; i0 += stride) {  // block-uniform
    const int64_t i = i0 + threadIdx.x;
    int k = -1;
    if (i < n) {
      const int v = __ldg(list + i);
      const int s = __ldg(vs + v);
      VoteRange rg;
      if (s >= 0 && vote_range(box, n_sites, s, zlo, zhi, mode, rg)) {
        int x, y, z;
        coords(g, v, x, y, z);
        if (z >= rg.z0 && z < rg.z0 + rg.D) {
          const long long flat = (long long)(x - rg.x0) + (long long)rg.W * ((y - rg.y0) + (long long)rg.H * (z - rg.z0));
          k = __ldg(seg0 + s) + (int)(flat / VS_SEG);
        }
      }
    }
    const unsigned grp = __match_any_sync(0xffffffffu, k);
    if (k >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(cnt + k, __popc(grp));
  }
}

// WRITE = false: cnt[k] = the segment's voxels of its site; WRITE = true:
// their (phi, v) in voxel order at ent[off[k] ...]. Sites are loaded
// 2 * VS_DEPTH batches ahead, the phi of the site's own voxels VS_DEPTH
// batches ahead (WRITE only).
template <bool WRITE>
__global__ void __launch_bounds__(128) k_vote_walk(const int* __restrict__ vs, const int* __restrict__ box,
                                                   int n_sites, Geo g, int zlo, int zhi, int mode,
                                                   const int* __restrict__ seg0, const int* __restrict__ n_seg_total,
                                                   int* __restrict__ cnt, const int* __restrict__ off,
                                                   int2* __restrict__ ent) {
  constexpr int DA = 2 * VS_DEPTH;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int n_seg = *n_seg_total;
  const int* __restrict__ vphi = vs + g.n;
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < n_seg; k += warps) {  // warp-uniform
    const int s = vote_seg_site(seg0, n_sites, k);
    VoteRange rg;
    vote_range(box, n_sites, s, zlo, zhi, mode, rg);
    const long long kb = (long long)(k - __ldg(seg0 + s)) * VS_SEG;
    const long long ke = min(rg.T, kb + VS_SEG);
    int n_out = 0;
    int2* out = WRITE ? ent + off[k] : nullptr;
    const int W = rg.W, H = rg.H;
    const int qa = 32 / W, qb = 32 - qa * W;
    long long kk = kb + lane;
    int dx = (int)(kk % W);
    const long long rr = kk / W;
    int dy = (int)(rr % H), dz = (int)(rr / H);
    int st[DA], vv[DA];
    int ph[VS_DEPTH];
    auto load = [&](int j) {
      vv[j] = -1;
      st[j] = -1;
      if (kk < ke) {
        vv[j] = (rg.x0 + dx) + g.nx * ((rg.y0 + dy) + g.ny * (rg.z0 + dz));
        st[j] = __ldg(vs + vv[j]);
      }
      kk += 32;
      dx += qb;
      dy += qa;
      if (dx >= W) { dx -= W; dy++; }
      while (dy >= H) { dy -= H; dz++; }
    };
    auto load_phi = [&](int jp, int j) {
      if (WRITE && st[j] == s) ph[jp] = __ldg(vphi + vv[j]);
    };
#pragma unroll
    for (int j = 0; j < DA; j++) load(j);
#pragma unroll
    for (int j = 0; j < VS_DEPTH; j++) load_phi(j, j);
    for (long long base = kb; base < ke; base += 32 * DA) {
#pragma unroll
      for (int j = 0; j < DA; j++) {
        const int jp = j % VS_DEPTH;
        const bool mine = st[j] == s;
        const int phi = ph[jp], v = vv[j];
        load_phi(jp, (j + VS_DEPTH) % DA);  // batch + VS_DEPTH: its site was loaded VS_DEPTH batches ago
        load(j);                            // batch + DA into the slot this batch left
        const unsigned m = __ballot_sync(0xffffffffu, mine);
        if (WRITE && mine) out[n_out + __popc(m & ((1u << lane) - 1u))] = make_int2(phi, v);
        n_out += __popc(m);
      }
    }
    if (!WRITE && lane == 0) cnt[k] = n_out;
  }
}

// one warp per site (order[]: largest boxes first): the ordered chains over
// the site's entries ent[off[seg0[s]] .. off[seg0[s] + nseg[s]]) --
// contiguous, in voxel order. Software-pipelined, branch-free: while the 32
// dependent adds of batch c run (every lane runs them; lanes 0-3 hold the
// four real chains, the others a harmless copy), the terms of batch c + 1
// are formed into the other half of a double-buffered stage -- one basic
// block, so the scheduler fills the add latency with that work. Entries are
// loaded DE batches ahead, weights DW batches ahead. Past the end an entry
// is (0, -1) with weight 0, whose term is +0.0: adding it is exact (the
// chains start at +0.0 and never become -0.0).
template <int WARPS, int DE = 8, int DW = 4>  // (4, 2: 8 % slower at C4)
__global__ void __launch_bounds__(WARPS * 32) k_vote_add(const int* __restrict__ order, int n_sites, Geo g,
                                                         const double* __restrict__ w64,
                                                         const float* __restrict__ w32, int w_mode, int mode,
                                                         const double* __restrict__ init,
                                                         const int* __restrict__ seg0, const int* __restrict__ nseg,
                                                         const int* __restrict__ off, const int* __restrict__ n_ent,
                                                         const int* __restrict__ n_seg_total,
                                                         const int2* __restrict__ ent, double* __restrict__ sums) {
  static_assert(DE > DW && DW >= 2 && DE % DW == 0, "k_vote_add pipeline");
  __shared__ __align__(16) double buf[WARPS][2][4][VS_ROW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if ((int)blockIdx.x * WARPS + wid >= n_sites) return;
  const int s = order[blockIdx.x * WARPS + wid];
  if (mode != 0 && nseg[s] == 0) return;  // a slab step this site does not take part in: untouched
  const int k0 = seg0[s], k1 = k0 + nseg[s];
  const int e0 = k0 < *n_seg_total ? off[k0] : *n_ent;
  const int e1 = k1 < *n_seg_total ? off[k1] : *n_ent;
  double acc = (init && mode != 1) ? init[(lane & 3) * n_sites + s] : 0.0;
  int2 q[DE];
  double wd[DW];
  float wf[DW];
  auto ld_ent = [&](int j, int c) { q[j] = c + lane < e1 ? __ldg(ent + c + lane) : make_int2(0, -1); };
  auto ld_w = [&](int jw, int j) {
    wd[jw] = 0.0;
    wf[jw] = 0.f;
    if (q[j].y >= 0) {
      if (w_mode == 1) wd[jw] = __ldg(w64 + q[j].y);
      else if (w_mode >= 2) wf[jw] = __ldg(w32 + q[j].y);
    }
  };
  // the term of the batch in entry slot j / weight slot jw into stage half h
  auto form = [&](int j, int jw, int h) {
    const bool live = q[j].y >= 0;
    const double wt = !live ? 0.0
                      : w_mode == 0 ? 1.0
                      : w_mode == 1 ? wd[jw]
                      : w_mode == 2 ? (double)wf[jw]
                                    : __dmul_rn((double)wf[jw], (double)wf[jw]);  // m**1.0 / m**2.0
    const double4 t = g.pack10 ? vote_term_packed(g, q[j].x, wt) : vote_term(g, q[j].x, wt);
    buf[wid][h][0][lane] = t.x; buf[wid][h][1][lane] = t.y; buf[wid][h][2][lane] = t.z; buf[wid][h][3][lane] = t.w;
  };
  const int nb = (e1 - e0 + 31) >> 5;  // batches
#pragma unroll
  for (int j = 0; j < DE; j++) ld_ent(j, e0 + 32 * j);
#pragma unroll
  for (int j = 0; j < DW; j++) ld_w(j, j);
  if (nb > 0) {
    form(0, 0, 0);
    ld_w(0, DW % DE);
    ld_ent(0, e0 + 32 * DE);
  }
  __syncwarp();
  for (int b0 = 0; b0 < nb; b0 += DE) {
#pragma unroll
    for (int j = 0; j < DE; j++) {
      const int b = b0 + j;
      if (b >= nb) break;  // warp-uniform
      // batch b + 1 sits in entry slot (j + 1) % DE and weight slot (b + 1) % DW (past the last batch:
      // zero terms, never added)
      const int jn = (j + 1) % DE, jwn = (j + 1) % DW;
      form(jn, jwn, (b + 1) & 1);
      ld_w(jwn, (j + 1 + DW) % DE);  // batch b + 1 + DW
      ld_ent(jn, e0 + 32 * (b + 1 + DE));
      // the 32 ordered adds of batch b (stage half b & 1)
      const double* row = &buf[wid][b & 1][lane & 3][0];
#pragma unroll
      for (int h = 0; h < 32; h += 8) {
        const double2 a0 = *reinterpret_cast<const double2*>(row + h);
        const double2 a1 = *reinterpret_cast<const double2*>(row + h + 2);
        const double2 a2 = *reinterpret_cast<const double2*>(row + h + 4);
        const double2 a3 = *reinterpret_cast<const double2*>(row + h + 6);
        acc = __dadd_rn(acc, a0.x); acc = __dadd_rn(acc, a0.y);
        acc = __dadd_rn(acc, a1.x); acc = __dadd_rn(acc, a1.y);
        acc = __dadd_rn(acc, a2.x); acc = __dadd_rn(acc, a2.y);
        acc = __dadd_rn(acc, a3.x); acc = __dadd_rn(acc, a3.y);
      }
      __syncwarp();  // half b & 1 is free for batch b + 2; half (b + 1) & 1 is visible
    }
  }
  if (lane < 4) sums[lane * n_sites + s] = acc;
}

// multi-GPU ordered vote hand-over: the running sums after this slab --
// this slab's chain results for sites whose box meets it, the incoming
// running sums (zero on the first slab) for the others
__global__ void k_vote_carry(const int* __restrict__ box, int n_sites, int zlo, int zhi,
                             const double* __restrict__ res, const double* __restrict__ carry_in,
                             double* __restrict__ carry_out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sites) return;
  const int bz0 = box[2 * n_sites + s], bz1 = box[5 * n_sites + s];
  const bool meets = bz0 <= zhi - 1 && bz1 >= zlo && bz0 <= bz1;
#pragma unroll
  for (int k = 0; k < 4; k++)
    carry_out[k * n_sites + s] = meets ? res[k * n_sites + s] : (carry_in ? carry_in[k * n_sites + s] : 0.0);
}

// step 2 (after the stable sort by key): segment starts/ends per site.
__global__ void k_segments(const int* __restrict__ skey, int n, int n_sites,
                           int* __restrict__ seg_begin, int* __restrict__ seg_end) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int k = skey[i];
    if (k >= n_sites) continue;
    if (i == 0 || skey[i - 1] != k) seg_begin[k] = (int)i;
    if (i == n - 1 || skey[i + 1] != k) seg_end[k] = (int)i + 1;
  }
}

// _kernels.py:535-582, one thread per site. counters[0] += empty regions.
__global__ void k_move_sites(Geo g, const int* __restrict__ comp, const double4* __restrict__ site_pos,
                             const int* __restrict__ site_comp, const double* __restrict__ sums,
                             int n_sites, double backoff, double4* __restrict__ new_pos,
                             double* __restrict__ disp, int* __restrict__ empty_count) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sites) return;
  const double4 a = site_pos[s];
  new_pos[s] = a;
  disp[s] = 0.0;
  const double wsum = sums[s];
  if (wsum <= 0.0) { atomicAdd(empty_count, 1); return; }
  const double bx = __ddiv_rn(sums[n_sites + s], wsum);
  const double by = __ddiv_rn(sums[2 * n_sites + s], wsum);
  const double bz = __ddiv_rn(sums[3 * n_sites + s], wsum);
  const double seg = dist3(a.x, a.y, a.z, bx, by, bz);
  if (seg == 0.0) return;
  const int want = site_comp[s];
  const double thit = segment_hit_t(comp, g, a.x, a.y, a.z, bx, by, bz, want);
  double px, py, pz;
  if (thit >= 1.0) {
    px = bx; py = by; pz = bz;
  } else {
    const double travel = __dsub_rn(__dmul_rn(thit, seg), backoff);
    if (travel <= 0.0) return;
    const double f = __ddiv_rn(travel, seg);
    px = __dadd_rn(a.x, __dmul_rn(__dsub_rn(bx, a.x), f));
    py = __dadd_rn(a.y, __dmul_rn(__dsub_rn(by, a.y), f));
    pz = __dadd_rn(a.z, __dmul_rn(__dsub_rn(bz, a.z), f));
  }
  const int cx = cell_of(px, g.sx, g.nx), cy = cell_of(py, g.sy, g.ny), cz = cell_of(pz, g.sz, g.nz);
  if (__ldg(comp + cx + g.nx * (cy + g.ny * cz)) != want) return;
  new_pos[s] = make_double4(px, py, pz, 0.0);
  disp[s] = dist3(a.x, a.y, a.z, px, py, pz);
}

}  // namespace lrcvt
