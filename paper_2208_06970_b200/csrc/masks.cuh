// masks.cuh -- level-set (isoband) and connected-component restriction masks.
//
// classify_isobands (grid.py:140-163): band i iff iso[i] < f <= iso[i+1],
//   i.e. searchsorted(iso, f64(f), 'left') - 1, NONE outside. One streaming
//   pass: 4 B read + 4 B write per voxel, 128-bit vectorised.
// label_components (grid.py:166-220): 6-connected (4 in 2D) components per
//   layer with dense ids ordered by (layer, first voxel in row-major order).
//   Lock-free union-find where a union always links the larger root under
//   the smaller one (atomicMin), so every tree's root is its component's
//   minimum flat index -- the reference's "first occurrence" -- independent
//   of thread timing. Ids: stable radix sort of roots by layer.
#pragma once
#include "common.cuh"

namespace lrcvt {

__device__ __forceinline__ int band_of(float f, const double* __restrict__ iso, int n_iso) {
  const double x = (double)f;
  int idx = 0;  // number of iso values strictly below x == searchsorted 'left'
  for (int i = 0; i < n_iso; i++) idx += iso[i] < x ? 1 : 0;
  return (idx == 0 || idx == n_iso) ? LRCVT_NONE : idx - 1;
}

__global__ void __launch_bounds__(256) k_isobands(const float* __restrict__ f, int64_t n,
                                                  const double* __restrict__ iso_g, int n_iso,
                                                  int* __restrict__ layer) {
  __shared__ double iso[64];
  if (threadIdx.x < n_iso) iso[threadIdx.x] = iso_g[threadIdx.x];
  __syncthreads();
  const int64_t n4 = n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float4* f4 = reinterpret_cast<const float4*>(f);
  int4* l4 = reinterpret_cast<int4*>(layer);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 a = __ldcs(f4 + i);
    int4 o;
    o.x = band_of(a.x, iso, n_iso);
    o.y = band_of(a.y, iso, n_iso);
    o.z = band_of(a.z, iso, n_iso);
    o.w = band_of(a.w, iso, n_iso);
    __stcs(l4 + i, o);
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    layer[i] = band_of(f[i], iso, n_iso);
}

__device__ __forceinline__ int uf_find(const int* L, int x) {
  int p = __ldcg(L + x);
  while (p != x) {
    x = p;
    p = __ldcg(L + x);
  }
  return x;
}

__device__ __forceinline__ void uf_union(int* L, int a, int b) {
  for (;;) {
    a = uf_find(L, a);
    b = uf_find(L, b);
    if (a == b) return;
    if (a < b) { int t = a; a = b; b = t; }  // link larger root a under smaller b
    const int old = atomicMin(L + a, b);
    if (old == a) return;
    a = old;
  }
}

__device__ __forceinline__ bool in_layers(int l, int n_layers) { return l >= 0 && l < n_layers; }

__global__ void k_ccl_init(const int* __restrict__ layer, int64_t n, int n_layers, int* __restrict__ L) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    L[i] = in_layers(layer[i], n_layers) ? (int)i : -1;
}

__global__ void k_ccl_merge(Geo g, const int* __restrict__ layer, int n_layers, int* __restrict__ L) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n; i += stride) {
    const int v = (int)i;
    const int l = layer[v];
    if (!in_layers(l, n_layers)) continue;
    int x, y, z;
    coords(g, v, x, y, z);
    if (x > 0 && layer[v - 1] == l) uf_union(L, v, v - 1);
    if (y > 0 && layer[v - g.nx] == l) uf_union(L, v, v - g.nx);
    if (z > 0 && layer[v - g.nxy] == l) uf_union(L, v, v - g.nxy);
  }
}

__global__ void k_ccl_compress(int64_t n, int* __restrict__ L) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int p = L[i];
    if (p >= 0 && p != (int)i) L[i] = uf_find(L, p);
  }
}

// roots: key = layer, value = root voxel (input in increasing voxel order)
__global__ void k_ccl_root_keys(const int* __restrict__ roots, int n_roots, const int* __restrict__ layer,
                                int* __restrict__ key) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_roots) key[i] = layer[roots[i]];
}

// id of each root, written at the root's own slot of `comp`
__global__ void k_ccl_root_ids(const int* __restrict__ sorted_roots, int n_roots, int* __restrict__ comp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_roots) comp[sorted_roots[i]] = i;
}

__global__ void k_ccl_relabel(const int* __restrict__ L, int64_t n, int* __restrict__ comp) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int r = L[i];
    if (r < 0) comp[i] = LRCVT_NONE;
    else if (r != (int)i) comp[i] = comp[r];  // roots already hold their id
  }
}

// component table: count (u64), bbox (x0,y0,z0 via atomicMin, x1,y1,z1 via
// atomicMax) and layer, per component id (grid.py:199-211).
__global__ void k_ccl_table(Geo g, const int* __restrict__ comp, const int* __restrict__ layer,
                            unsigned long long* __restrict__ count, int* __restrict__ bbox,
                            int* __restrict__ layer_of) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < g.n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    int c = -1, x = 0, y = 0, z = 0;
    if (i < g.n) {
      c = comp[i];
      if (c >= 0) coords(g, (int)i, x, y, z);
    }
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    const int lane = threadIdx.x & 31;
    const unsigned cnt = __popc(grp);
    const int xmin = __reduce_min_sync(grp, x), xmax = __reduce_max_sync(grp, x);
    const int ymin = __reduce_min_sync(grp, y), ymax = __reduce_max_sync(grp, y);
    const int zmin = __reduce_min_sync(grp, z), zmax = __reduce_max_sync(grp, z);
    if (c >= 0 && lane == __ffs(grp) - 1) {
      atomicAdd(count + c, (unsigned long long)cnt);
      atomicMin(bbox + 6 * c + 0, xmin);
      atomicMin(bbox + 6 * c + 1, ymin);
      atomicMin(bbox + 6 * c + 2, zmin);
      atomicMax(bbox + 6 * c + 3, xmax);
      atomicMax(bbox + 6 * c + 4, ymax);
      atomicMax(bbox + 6 * c + 5, zmax);
      layer_of[c] = layer[i];
    }
  }
}

__global__ void k_ccl_table_init(int n_comp, unsigned long long* count, int* bbox) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_comp) return;
  count[c] = 0;
  bbox[6 * c + 0] = bbox[6 * c + 1] = bbox[6 * c + 2] = 0x7fffffff;
  bbox[6 * c + 3] = bbox[6 * c + 4] = bbox[6 * c + 5] = -1;
}

}  // namespace lrcvt
