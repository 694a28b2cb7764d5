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
//   * ORDERED path (any weights): one warp per site walks the site's
//     bounding box in voxel order and four lanes add the terms
//     (w, RN(w*ax), RN(w*ay), RN(w*az)) of the region's voxels in exactly
//     the reference order (k_vote_prep / k_vote_scan below). The earlier
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
//   k_vote_scan  one warp per site walks its box in chunks of 32 voxels
//                (flat box order), picks the voxels of its region, forms their
//                terms and lanes 0-3 add them in order -- the reference's
//                exact accumulation order (_kernels.py:519-531).
// A voxel belongs to region s iff sp[v].x == s: sp is reset to -1 whenever
// the eligible set is rebuilt, and k_vote_prep writes every eligible voxel,
// so no stale entry survives.
constexpr int BOX_BIG = 0x3fffffff;
constexpr int VS_DEPTH = 4;  // chunks of (site, phi) / weight loads in flight per warp in k_vote_scan


template <bool MG>
__global__ void __launch_bounds__(256) k_vote_prep(const int* __restrict__ list, int n, Geo g,
                                                   const int2* __restrict__ ss, int2* __restrict__ sp,
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
      sp[v] = make_int2(s, u >= 0 && g.pack10 ? phi_pack(g, u) : u);
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

// Largest boxes first: k_vote_scan runs one warp per site and the walk time
// follows the box volume (a few 100k-voxel boxes among 3.8k-voxel medians at
// C4), so in site order the last waves ran a handful of long warps on an
// otherwise idle GPU (SM active 54 % of the elapsed cycles). Sites are
// bucketed by floor(log2(box volume)) and the scan takes them bucket by
// bucket, biggest first (order within a bucket is free: every site's chain
// is independent).
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

// One warp per site (order[]: largest boxes first); a (WARPS x 4 x VS_ROW) shared stage holds a chunk's
// terms. The walk covers the box rows inside planes [zlo, zhi) (the whole
// volume on one GPU). mode 0: every site, chains start at 0 (or init[s]);
// multi-GPU slab steps: mode 1 = only sites whose box starts in this slab
// (chains start at 0), mode 2 = only sites whose box starts in an earlier
// slab (chains continue from init[s], the running sums handed over by the
// previous slab). Sites a mode skips are left untouched in `sums`.
// (A variant that read a 2-byte site tag per box voxel first and the 8-byte
// entry only on a tag match moved more DRAM sectors, not fewer: 4.0 vs 3.7
// GB per C4 launch, same time.)
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_vote_scan(const int2* __restrict__ sp,
                                                          const int* __restrict__ box,
                                                          const int* __restrict__ order,
                                                          const int* __restrict__ site_comp, int n_sites, Geo g,
                                                          const double* __restrict__ w64,
                                                          const float* __restrict__ w32, int w_mode, int zlo,
                                                          int zhi, int mode, const double* __restrict__ init,
                                                          double* __restrict__ sums) {
  __shared__ __align__(16) double buf[WARPS][4][VS_ROW];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if ((int)blockIdx.x * WARPS + wid >= n_sites) return;
  const int s = order[blockIdx.x * WARPS + wid];
  const int x0 = box[s], y0 = box[n_sites + s], bz0 = box[2 * n_sites + s];
  const int bz1 = box[5 * n_sites + s];
  if (mode == 1 && !(bz0 >= zlo && bz0 < zhi)) return;
  if (mode == 2 && !(bz0 < zlo && bz1 >= zlo)) return;
  const int z0 = bz0 > zlo ? bz0 : zlo;
  const int z1 = bz1 < zhi - 1 ? bz1 : zhi - 1;
  const int W = box[3 * n_sites + s] - x0 + 1, H = box[4 * n_sites + s] - y0 + 1, D = z1 - z0 + 1;
  double acc = (init && mode != 1 && lane < 4) ? init[lane * n_sites + s] : 0.0;
  if (W > 0 && H > 0 && D > 0) {
    const long long T = (long long)W * H * D;
    // flat box index k = lane + 32 * chunk -> (dx, dy, dz); 32 = qa * W + qb,
    // so a chunk advance is dx += qb, dy += qa plus at most one x carry
    const int qa = 32 / W, qb = 32 - qa * W;
    int dx = lane % W, r = lane / W;
    int dy = r % H, dz = r / H;
    long long k = lane;  // flat index of this lane's next voxel to load
    // two-stage pipeline: stage 1 (DA chunks ahead) = the (site, phi) entry
    // of every lane's voxel; stage 2 (VS_DEPTH chunks ahead, once stage 1
    // arrived) = the raw weight of the voxels of this site only
    constexpr int DA = 2 * VS_DEPTH;
    int vi[DA];
    int2 s1[DA];
    int2 pa[VS_DEPTH];
    double wd[VS_DEPTH];
    float wf[VS_DEPTH];
    auto next_voxel = [&]() {
      int v = -1;
      if (k < T) v = (x0 + dx) + g.nx * ((y0 + dy) + g.ny * (z0 + dz));
      k += 32;
      dx += qb;
      dy += qa;
      if (dx >= W) { dx -= W; dy++; }
      while (dy >= H) { dy -= H; dz++; }
      return v;
    };
    auto load1 = [&](int j) {
      vi[j] = next_voxel();
      s1[j] = vi[j] >= 0 ? __ldg(sp + vi[j]) : make_int2(-1, -1);
    };
    auto load2 = [&](int j, int jp) {
      pa[jp] = s1[j];
      if (pa[jp].x == s) {  // raw weight: converted only when the term is formed
        if (w_mode == 1) wd[jp] = __ldg(w64 + vi[j]);
        else if (w_mode >= 2) wf[jp] = __ldg(w32 + vi[j]);
      }
    };
#pragma unroll
    for (int j = 0; j < DA; j++) load1(j);
#pragma unroll
    for (int j = 0; j < VS_DEPTH; j++) load2(j, j);
    double* row = &buf[wid][lane & 3][0];
    for (long long base = 0; base < T; base += 32 * DA) {
#pragma unroll
      for (int j = 0; j < DA; j++) {
        const int jp = j % VS_DEPTH;
        const int2 e = pa[jp];
        const bool mine = e.x == s;
        double wt = 0.0;
        if (mine)
          wt = w_mode == 0 ? 1.0
               : w_mode == 1 ? wd[jp]
               : w_mode == 2 ? (double)wf[jp]
                             : __dmul_rn((double)wf[jp], (double)wf[jp]);  // m**1.0 / m**2.0
        load2((j + VS_DEPTH) % DA, jp);  // chunk + VS_DEPTH, whose stage 1 was issued VS_DEPTH chunks ago
        load1(j);                        // chunk + DA into the slot this chunk's stage 1 left
        const unsigned m = __ballot_sync(0xffffffffu, mine);
        if (m) {
          const int cnt = __popc(m);
          // matching lanes take slots [0, cnt) in voxel order, the others
          // write the +0.0 pads after them
          const int below = __popc(m & ((1u << lane) - 1u));
          const int slot = mine ? below : cnt + (lane - below);
          double4 t = make_double4(0.0, 0.0, 0.0, 0.0);
          if (mine) t = g.pack10 ? vote_term_packed(g, e.y, wt) : vote_term(g, e.y, wt);
          buf[wid][0][slot] = t.x; buf[wid][1][slot] = t.y; buf[wid][2][slot] = t.z; buf[wid][3][slot] = t.w;
          __syncwarp();
          if (lane < 4) acc = ordered_add_padded(acc, row, cnt);
          __syncwarp();
        }
      }
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
