// seeding.cuh -- device reductions of the seeding stage (SURVEY.md §8(f)
// rank 1): per-(component, block) masses of m_v**gamma and the total in-band
// mass, reference lrcvt/seeding.py:71-107 (component_masses).
//
// The reference groups in-band voxels with np.lexsort((voxel, block, comp))
// and sums every (component, block) run with np.sum, i.e. numpy's pairwise
// summation: result = 0.0 + pw(a, n) with
//   pw(a, n) = n < 8    : serial from 0.0
//              n <= 128 : eight strided accumulators, combined
//                         ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail
//              else     : pw(a, n2) + pw(a + n2, n - n2), n2 = n/2 - (n/2 % 8)
// The same operation tree on the device reproduces it bit for bit; the
// grouping is a stable radix sort of a (component, block) key over the
// in-band voxels listed in increasing order.
#pragma once

#include <cstdint>

namespace lrcvt {

// weight of voxel v: 1, float64 array, float32 field (gamma 1) or its square
// (gamma 2); identical to numpy's m ** gamma for those cases (seeding.py:68)
struct SeedWeight {
  int mode;
  const double* w64;
  const float* w32;
  __device__ __forceinline__ double operator()(int v) const {
    if (mode == 0) return 1.0;
    if (mode == 1) return w64[v];
    const double m = (double)w32[v];
    return mode == 2 ? m : __dmul_rn(m, m);
  }
};

// element i of a pairwise-summed sequence
struct SeqDirect {  // contiguous float64 values
  const double* a;
  __device__ __forceinline__ double operator()(int64_t i) const { return a[i]; }
};
struct SeqGather {  // weight of the i-th listed voxel
  const int* list;
  SeedWeight w;
  __device__ __forceinline__ double operator()(int64_t i) const { return w(list[i]); }
};

template <class Seq>
__device__ double pw_leaf(const Seq& a, int64_t lo, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a(lo + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a(lo + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a(lo + i + j));
  }
  double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                       __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) s = __dadd_rn(s, a(lo + i));
  return s;
}

// pw(a[lo, lo+n)) without recursion: the split tree is walked depth first
// with an explicit stack of pending right halves and partial sums. Depth is
// bounded by log2(n / 128) + 1 < 40 for any int64 n.
template <class Seq>
__device__ double pw_sum(const Seq& a, int64_t lo, int64_t n) {
  if (n <= 128) return pw_leaf(a, lo, n);
  int64_t st_lo[40], st_n[40];
  double st_left[40];
  unsigned char st_state[40];  // 0: left pending, 1: right pending
  int top = 0;
  st_lo[0] = lo;
  st_n[0] = n;
  st_state[0] = 0;
  double ret = 0.0;
  bool have_ret = false;
  while (top >= 0) {
    const int64_t clo = st_lo[top], cn = st_n[top];
    if (have_ret) {  // a child finished
      have_ret = false;
      if (st_state[top] == 0) {
        st_left[top] = ret;
        st_state[top] = 1;
        int64_t n2 = cn / 2;
        n2 -= n2 % 8;
        const int64_t rlo = clo + n2, rn = cn - n2;
        if (rn <= 128) {
          ret = pw_leaf(a, rlo, rn);
          have_ret = true;
          continue;
        }
        ++top;
        st_lo[top] = rlo;
        st_n[top] = rn;
        st_state[top] = 0;
        continue;
      }
      ret = __dadd_rn(st_left[top], ret);
      have_ret = true;
      --top;
      continue;
    }
    // descend into the left half
    int64_t n2 = cn / 2;
    n2 -= n2 % 8;
    if (n2 <= 128) {
      ret = pw_leaf(a, clo, n2);
      have_ret = true;
      continue;
    }
    ++top;
    st_lo[top] = clo;
    st_n[top] = n2;
    st_state[top] = 0;
  }
  return ret;
}

// (component, block) key of listed voxel i (seeding.py:85-90)
__global__ void k_seed_keys(const int* __restrict__ list, int64_t n, const int* __restrict__ comp,
                            int nx, int ny, int bs, int64_t nbx, int64_t nby, int64_t n_blocks,
                            unsigned long long* __restrict__ key) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int v = list[i];
    const int x = v % nx, y = (v / nx) % ny, z = v / (nx * ny);
    const int64_t blk = (x / bs) + nbx * ((y / bs) + nby * (int64_t)(z / bs));
    key[i] = (unsigned long long)comp[v] * (unsigned long long)n_blocks + (unsigned long long)blk;
  }
}

__global__ void k_seed_weights(const int* __restrict__ list, int64_t n, SeedWeight w,
                               double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = w(list[i]);
}

// One warp per run: lane 0 lists the run's pairwise leaves (<= 128 elements)
// in depth-first order, the lanes sum the leaves in parallel (pw_leaf), and
// lane 0 rebuilds the same tree over the leaf sums -- the identical
// operation sequence of pw_sum, with the element loads spread over the warp.
// Runs with more than WARP_LEAVES leaves fall back to one thread (pw_sum).
constexpr int WARP_LEAVES = 128;
template <int WARPS>
__global__ void __launch_bounds__(32 * WARPS) k_seed_run_mass_warp(const double* __restrict__ w_sorted,
                                                                    const int64_t* __restrict__ start,
                                                                    const int64_t* __restrict__ len,
                                                                    int64_t n_runs, double* __restrict__ mass) {
  __shared__ int64_t s_lo[WARPS][WARP_LEAVES];
  __shared__ int s_n[WARPS][WARP_LEAVES];
  __shared__ double s_sum[WARPS][WARP_LEAVES];
  __shared__ int s_cnt[WARPS];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t r = blockIdx.x * (int64_t)WARPS + wid;
  if (r >= n_runs) return;
  const int64_t lo0 = start[r], n0 = len[r];
  const SeqDirect seq{w_sorted};
  if (lane == 0) {
    // depth-first leaf list (explicit stack of pending ranges, left first)
    int64_t st_lo[40], st_n[40];
    int top = 0, cnt = 0;
    st_lo[0] = lo0; st_n[0] = n0;
    while (top >= 0 && cnt <= WARP_LEAVES) {
      const int64_t lo = st_lo[top], n = st_n[top];
      --top;
      if (n <= 128) {
        if (cnt < WARP_LEAVES) { s_lo[wid][cnt] = lo; s_n[wid][cnt] = (int)n; }
        ++cnt;
        continue;
      }
      int64_t n2 = n / 2;
      n2 -= n2 % 8;
      ++top; st_lo[top] = lo + n2; st_n[top] = n - n2;  // right half pops after the left
      ++top; st_lo[top] = lo; st_n[top] = n2;
    }
    s_cnt[wid] = cnt;
  }
  __syncwarp();
  const int cnt = s_cnt[wid];
  if (cnt > WARP_LEAVES) {  // very long run: single-thread tree
    if (lane == 0) mass[r] = __dadd_rn(0.0, pw_sum(seq, lo0, n0));
    return;
  }
  for (int j = lane; j < cnt; j += 32) s_sum[wid][j] = pw_leaf(seq, s_lo[wid][j], s_n[wid][j]);
  __syncwarp();
  if (lane == 0) {
    // rebuild: the same recursion, consuming leaf sums in depth-first order
    int64_t st_n[40];
    double st_left[40];
    unsigned char st_state[40];
    int top = 0, next = 0;
    st_n[0] = n0; st_state[0] = 0;
    double ret = 0.0;
    bool have = false;
    if (n0 <= 128) {
      ret = s_sum[wid][0];
      top = -1;
    }
    while (top >= 0) {
      const int64_t n = st_n[top];
      int64_t n2 = n / 2;
      n2 -= n2 % 8;
      if (have) {
        have = false;
        if (st_state[top] == 0) {
          st_left[top] = ret;
          st_state[top] = 1;
          if (n - n2 <= 128) { ret = s_sum[wid][next++]; have = true; continue; }
          ++top; st_n[top] = n - n2; st_state[top] = 0;
          continue;
        }
        ret = __dadd_rn(st_left[top], ret);
        have = true;
        --top;
        continue;
      }
      if (n2 <= 128) { ret = s_sum[wid][next++]; have = true; continue; }
      ++top; st_n[top] = n2; st_state[top] = 0;
    }
    mass[r] = __dadd_rn(0.0, ret);
  }
}

// subtree sums of the total in-band mass (voxel order); the host splits the
// tree into these subtrees and adds them back in the same shape
__global__ void k_seed_subtrees(const int* __restrict__ list, SeedWeight w, const int64_t* __restrict__ lo,
                                const int64_t* __restrict__ n, int count, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  out[t] = pw_sum(SeqGather{list, w}, lo[t], n[t]);
}

}  // namespace lrcvt
