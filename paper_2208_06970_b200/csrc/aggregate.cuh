// aggregate.cuh -- per-cell moment and histogram aggregation
// (aggregate_moments, pipeline.py:187-238; accumulate, stats.py:59-78;
// histogram1d, stats.py:194-203).
//
// Cells: region r (< n_sites) = in-band voxels with site_of == r; stray cell
// n_sites + c = unassigned in-band voxels of component c (pipeline.py:215-220).
// In-band voxels are grouped by cell with one stable radix sort (cell keys,
// voxel values), then
//   k_agg_moments  one warp per (cell, pair): n, the 15 raw power sums
//                  S_pq = sum x^p y^q (p+q <= 4, stats.py:19 ORDERS order)
//                  in compensated fp64 (per-lane Neumaier, fixed-order
//                  double-double lane tree: deterministic, ~1 ulp), and the
//                  min / max of both variables;
//   k_agg_hist     one warp per (cell, field): bins with numpy's exact
//                  uniform-bin rule (edges = linspace(lo, hi, B+1); index =
//                  trunc((a-lo)/(hi-lo)*B), last-edge and +-1 edge fix-ups),
//                  plus under/overflow, on fixed global axes.
#pragma once
#include "common.cuh"

namespace lrcvt {

constexpr int AGG_NSUMS = 15;
// ORDERS = [(p, q) for p in range(5) for q in range(5) if p + q <= 4]
__host__ __device__ constexpr int ord_p(int t) { return t < 5 ? 0 : t < 9 ? 1 : t < 12 ? 2 : t < 14 ? 3 : 4; }
__host__ __device__ constexpr int ord_q(int t) {
  return t < 5 ? t : t < 9 ? t - 5 : t < 12 ? t - 9 : t < 14 ? t - 12 : 0;
}

__global__ void k_agg_keys(const int* __restrict__ inband, int n, const int* __restrict__ site_of,
                           const int* __restrict__ comp, int n_sites, int* __restrict__ key,
                           int* __restrict__ val) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int v = inband[i];
    const int s = site_of[v];
    key[i] = s >= 0 ? s : n_sites + comp[v];
    val[i] = v;
  }
}

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// powers 0..4 of x, each RN of the exact value where a double can hold it:
// x is a float32 value (24-bit significand), so x^2 is exact and x^3, x^4 are
// one rounding from exact.
__device__ __forceinline__ void powers(double x, double* xp) {
  xp[0] = 1.0;
  xp[1] = x;
  xp[2] = __dmul_rn(x, x);
  xp[3] = __dmul_rn(xp[2], x);
  xp[4] = __dmul_rn(xp[2], xp[2]);
}

// one warp per (cell, pair); out layout: sums[cell][pair][15],
// minmax[cell][pair][4] = (min_x, max_x, min_y, max_y), count[cell]
// Per-lane compensated accumulation of the terms of one (cell, pair). Only
// the work that changes a result is done: S_00 is the count (exact); terms
// with p == 0 or q == 0 are plain powers (the product with 1.0 is exact);
// for a pair of one field with itself (x == y) the sums S_pq and S_qp are
// identical (IEEE products commute), so only p <= q is accumulated.
template <bool SAME>
__device__ __forceinline__ void agg_lane(const float* __restrict__ fx, const float* __restrict__ fy, int b, int e,
                                         int lane, double* s, double* c, double& mnx, double& mxx, double& mny,
                                         double& mxy) {
  for (int j = b + lane; j < e; j += 32) {
    const double x = (double)__ldg(fx + j);
    const double y = SAME ? x : (double)__ldg(fy + j);
    mnx = fmin(mnx, x); mxx = fmax(mxx, x);
    if (!SAME) { mny = fmin(mny, y); mxy = fmax(mxy, y); }
    double xp[5], yq[5];
    powers(x, xp);
    if (SAME) {
#pragma unroll
      for (int k = 0; k < 5; k++) yq[k] = xp[k];
    } else {
      powers(y, yq);
    }
#pragma unroll
    for (int t = 1; t < AGG_NSUMS; t++) {
      const int p = ord_p(t), q = ord_q(t);
      if (SAME && p > q) continue;
      const double term = p == 0 ? yq[q] : q == 0 ? xp[p] : __dmul_rn(xp[p], yq[q]);
      double hi, lo;
      two_sum(s[t], term, hi, lo);
      s[t] = hi;
      c[t] = __dadd_rn(c[t], lo);
    }
  }
  if (SAME) { mny = mnx; mxy = mxx; }
}

// index of the (q, p) term of ORDERS
__host__ __device__ constexpr int ord_mirror(int t) {
  const int p = ord_p(t), q = ord_q(t);
  int k = 0;
  for (int u = 0; u < AGG_NSUMS; u++)
    if (ord_p(u) == q && ord_q(u) == p) k = u;
  return k;
}

__global__ void __launch_bounds__(128) k_agg_moments(const int* __restrict__ seg_b,
                                                     const int* __restrict__ seg_e, int n_cells,
                                                     const float* const* __restrict__ fields,
                                                     const int* __restrict__ pairs, int n_pairs,
                                                     long long* __restrict__ count,
                                                     double* __restrict__ sums,
                                                     double* __restrict__ minmax) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= n_cells * n_pairs) return;
  const int cell = gw / n_pairs, pr = gw - cell * n_pairs;
  const int ix = pairs[2 * pr], iy = pairs[2 * pr + 1];
  const float* __restrict__ fx = fields[ix];  // columns in cell order
  const float* __restrict__ fy = fields[iy];
  const int b = seg_b[cell], e = seg_e[cell];
  double s[AGG_NSUMS], c[AGG_NSUMS];
#pragma unroll
  for (int j = 0; j < AGG_NSUMS; j++) { s[j] = 0.0; c[j] = 0.0; }
  double mnx = __longlong_as_double(0x7ff0000000000000LL), mny = mnx;
  double mxx = -mnx, mxy = -mnx;
  if (ix == iy) agg_lane<true>(fx, fy, b, e, lane, s, c, mnx, mxx, mny, mxy);
  else agg_lane<false>(fx, fy, b, e, lane, s, c, mnx, mxx, mny, mxy);
  // fixed-order double-double tree across lanes
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int t = 1; t < AGG_NSUMS; t++) {
      const double os = __shfl_down_sync(0xffffffffu, s[t], o);
      const double oc = __shfl_down_sync(0xffffffffu, c[t], o);
      double hi, lo;
      two_sum(s[t], os, hi, lo);
      s[t] = hi;
      c[t] = __dadd_rn(__dadd_rn(c[t], oc), lo);
    }
    mnx = fmin(mnx, __shfl_down_sync(0xffffffffu, mnx, o));
    mxx = fmax(mxx, __shfl_down_sync(0xffffffffu, mxx, o));
    mny = fmin(mny, __shfl_down_sync(0xffffffffu, mny, o));
    mxy = fmax(mxy, __shfl_down_sync(0xffffffffu, mxy, o));
  }
  if (lane == 0) {
    double* out = sums + ((int64_t)cell * n_pairs + pr) * AGG_NSUMS;
    out[0] = (double)(e - b);
    if (ix == iy) {
#pragma unroll
      for (int t = 1; t < AGG_NSUMS; t++) {
        const int src = ord_p(t) > ord_q(t) ? ord_mirror(t) : t;
        out[t] = __dadd_rn(s[src], c[src]);
      }
    } else {
#pragma unroll
      for (int t = 1; t < AGG_NSUMS; t++) out[t] = __dadd_rn(s[t], c[t]);
    }
    double* mm = minmax + ((int64_t)cell * n_pairs + pr) * 4;
    mm[0] = mnx; mm[1] = mxx; mm[2] = mny; mm[3] = mxy;
    if (pr == 0) count[cell] = e - b;
  }
}

// global in-band min/max per field (histogram auto-axes): minmax[f] = (lo, hi)
__global__ void k_field_range(const int* __restrict__ inband, int n, const float* __restrict__ f,
                              unsigned long long* __restrict__ lohi /* ordered-int encodings */) {
  float mn = __int_as_float(0x7f800000), mx = -mn;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float a = __ldg(f + inband[i]);
    mn = fminf(mn, a); mx = fmaxf(mx, a);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    // order-preserving integer keys of the float values
    const int imn = __float_as_int(mn), imx = __float_as_int(mx);
    const unsigned kmn = imn >= 0 ? (unsigned)imn ^ 0x80000000u : ~(unsigned)imn;
    const unsigned kmx = imx >= 0 ? (unsigned)imx ^ 0x80000000u : ~(unsigned)imx;
    atomicMin(lohi, (unsigned long long)kmn);
    atomicMax(lohi + 1, (unsigned long long)kmx);
  }
}

__device__ __forceinline__ float key_to_float(unsigned long long k) {
  const unsigned u = (unsigned)k;
  return __int_as_float((u & 0x80000000u) ? (int)(u ^ 0x80000000u) : (int)~u);
}

// numpy histogram bin of a (lo <= a <= hi), stats.py:197-198 via
// numpy.histogram's equal-bin fast path
__device__ __forceinline__ int np_bin(double a, double lo, double hi, double denom, double step, int B) {
  const double f = __dmul_rn(__ddiv_rn(__dsub_rn(a, lo), denom), (double)B);
  int idx = (int)f;  // astype(intp): truncation, f >= 0
  if (idx == B) idx -= 1;
  // edges[i] = i*step + lo (linspace), edges[B] = hi
  const double e_lo = __dadd_rn(__dmul_rn((double)idx, step), lo);
  if (a < e_lo) idx -= 1;
  const double e_hi = idx + 1 == B ? hi : __dadd_rn(__dmul_rn((double)(idx + 1), step), lo);
  if (a >= e_hi && idx != B - 1) idx += 1;
  return idx;
}

// one warp per (cell, field); hist[cell][field][B + 2] (bins, under, over).
// The first bin guess uses a reciprocal multiply instead of numpy's division:
// both guesses are within one bin of the edge-defined bin, and numpy's +-1
// edge fix-ups (histograms.py) map any such guess to that same bin.
template <int MAXB>
__global__ void __launch_bounds__(128) k_agg_hist(const int* __restrict__ seg_b,
                                                  const int* __restrict__ seg_e, int n_cells,
                                                  const float* const* __restrict__ cols,
                                                  int n_fields, const double* __restrict__ axes,
                                                  int B, long long* __restrict__ hist) {
  __shared__ int bins[4][MAXB + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool live = gw < n_cells * n_fields;
  for (int j = lane; j < B + 2; j += 32) bins[wid][j] = 0;
  __syncwarp();
  if (live) {
    const int cell = gw / n_fields, fi = gw - cell * n_fields;
    const float* __restrict__ f = cols[fi];
    const double lo = axes[2 * fi], hi = axes[2 * fi + 1];
    const double denom = __dsub_rn(hi, lo);
    const double step = __ddiv_rn(denom, (double)B);
    const double scale = __ddiv_rn((double)B, denom);
    const int b = seg_b[cell], e = seg_e[cell];
    const int end = b + ((e - b + 31) & ~31);  // warp-uniform trip count
    for (int j = b + lane; j < end; j += 32) {
      int slot = -1;
      if (j < e) {
        const double a = (double)__ldg(f + j);
        if (a < lo) slot = B;
        else if (a > hi) slot = B + 1;
        else {
          int idx = (int)__dmul_rn(__dsub_rn(a, lo), scale);
          if (idx >= B) idx = B - 1;
          if (idx < 0) idx = 0;
          const double e_lo = __dadd_rn(__dmul_rn((double)idx, step), lo);
          if (a < e_lo) idx -= 1;
          const double e_hi = idx + 1 == B ? hi : __dadd_rn(__dmul_rn((double)(idx + 1), step), lo);
          if (a >= e_hi && idx != B - 1) idx += 1;
          slot = idx;
        }
      }
      const unsigned grp = __match_any_sync(0xffffffffu, slot);
      if (slot >= 0 && lane == __ffs(grp) - 1) atomicAdd(&bins[wid][slot], __popc(grp));
    }
    __syncwarp();
    long long* out = hist + ((int64_t)cell * n_fields + fi) * (B + 2);
    for (int j = lane; j < B + 2; j += 32) out[j] = bins[wid][j];
  }
}

// in-band field values gathered into cell order, one contiguous column per
// field, so the moment and histogram warps stream instead of chasing indices
__global__ void k_agg_gather(const int* __restrict__ sorted_v, int m, const float* const* __restrict__ fields,
                             int n_fields, float* __restrict__ cols) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += stride) {
    const int v = sorted_v[j];
    for (int fi = 0; fi < n_fields; ++fi) __stcg(cols + (int64_t)fi * m + j, __ldg(fields[fi] + v));
  }
}

}  // namespace lrcvt
