// adjacency.cuh -- site adjacency graph edges (reference
// lrcvt/sitegraph.py:46-82, region_adjacency): sites a != b are adjacent when
// two face-neighbouring voxels (+x, +y, +z) carry site_of a and b and lie in
// the same component. One streaming pass over site_of / component; lanes of
// a warp holding the same (min, max) pair elect one lane, which inserts the
// 64-bit key into an open-addressing hash set (a read-only probe first, so
// repeated pairs cost a cached load, not an atomic). The set is compacted and
// radix-sorted afterwards: sorted keys == np.unique(np.sort(pairs), axis=0).
#pragma once

#include <cstdint>

namespace lrcvt {

constexpr unsigned long long kAdjEmpty = ~0ull;

__device__ __forceinline__ unsigned long long adj_hash(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

__device__ __forceinline__ void adj_insert(unsigned long long* table, unsigned long long mask,
                                           unsigned long long key, int* overflow) {
  unsigned long long h = adj_hash(key) & mask;
  for (unsigned long long probes = 0;; ++probes) {
    if (probes > mask) {  // set full: the host retries with a larger one
      atomicExch(overflow, 1);
      return;
    }
    unsigned long long cur = __ldcg(table + h);
    if (cur == key) return;
    if (cur == kAdjEmpty) {
      cur = atomicCAS(table + h, kAdjEmpty, key);
      if (cur == kAdjEmpty || cur == key) return;
    }
    h = (h + 1) & mask;
  }
}

__global__ void __launch_bounds__(256) k_adjacency(Geo g, const int* __restrict__ site_of,
                                                   const int* __restrict__ comp,
                                                   unsigned long long* __restrict__ table,
                                                   unsigned long long mask, int* __restrict__ overflow) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count: every lane runs the same iterations
  const int64_t n_pad = (g.n + 31) / 32 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_pad; i += stride) {
    const bool in = i < g.n;
    const int v = in ? (int)i : 0;
    int a = -1, c = -1, x = 0, y = 0, z = 0;
    if (in) {
      a = __ldcs(site_of + v);
      if (a >= 0) {
        c = __ldcs(comp + v);
        coords(g, v, x, y, z);
      }
    }
#pragma unroll
    for (int axis = 0; axis < 3; ++axis) {
      unsigned long long key = kAdjEmpty;
      const bool room = axis == 0 ? x + 1 < g.nx : axis == 1 ? y + 1 < g.ny : z + 1 < g.nz;
      if (a >= 0 && room) {
        const int w = v + (axis == 0 ? 1 : axis == 1 ? g.nx : g.nxy);
        const int b = __ldg(site_of + w);
        if (b >= 0 && b != a && __ldg(comp + w) == c) {
          const unsigned lo = (unsigned)min(a, b), hi = (unsigned)max(a, b);
          key = ((unsigned long long)lo << 32) | hi;
        }
      }
      const unsigned grp = __match_any_sync(0xffffffffu, key);
      if (key != kAdjEmpty && (threadIdx.x & 31) == __ffs(grp) - 1) adj_insert(table, mask, key, overflow);
    }
  }
}

// sorted keys -> (E, 2) int64 rows (lo, hi)
__global__ void k_split_edges(const unsigned long long* __restrict__ keys, int n, long long* __restrict__ edges) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  edges[2 * i] = (long long)(k >> 32);
  edges[2 * i + 1] = (long long)(k & 0xFFFFFFFFull);
}

struct NotEmpty {
  __device__ __forceinline__ bool operator()(unsigned long long k) const { return k != kAdjEmpty; }
};

}  // namespace lrcvt
