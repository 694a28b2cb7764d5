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

// Tile-local labelling: one CTA per TX x TY x TZ tile (TX = 32: a warp is one
// x-row), one thread per voxel. Rows first, without atomics: a lane's run
// start comes from a ballot of "layer differs from the left neighbour". Then
// the y and z adjacencies unite run starts in a shared-memory union-find
// (larger index linked under smaller, atomicMin), one union per distinct
// (run, neighbour-run) pair in the warp. Local row-major order equals global
// row-major order restricted to the tile, so a local root is also the
// minimum global index of that tile component; every voxel then points at
// its local root in global L.
template <int TX, int TY, int TZ>
__global__ void __launch_bounds__(TX * TY * TZ) k_ccl_tile(Geo g, const int* __restrict__ layer, int n_layers,
                                                           int* __restrict__ L) {
  static_assert(TX == 32, "a warp is one x-row of the tile");
  constexpr int T = TX * TY * TZ;
  __shared__ int s_par[T];
  __shared__ signed char s_lay[T];
  const int t = threadIdx.x;
  const int lx = t % TX, ly = (t / TX) % TY, lz = t / (TX * TY);
  const int64_t ntx = (g.nx + TX - 1) / TX, nty = (g.ny + TY - 1) / TY;
  const int64_t b = blockIdx.x;
  const int x = (int)(b % ntx) * TX + lx;
  const int y = (int)((b / ntx) % nty) * TY + ly;
  const int z = (int)(b / (ntx * nty)) * TZ + lz;
  const bool in = x < g.nx && y < g.ny && z < g.nz;
  const int v = in ? x + g.nx * (y + g.ny * z) : 0;
  int l = in ? __ldcs(layer + v) : -1;
  if (!in_layers(l, n_layers)) l = -1;
  const int left = __shfl_up_sync(0xffffffffu, l, 1);
  const unsigned starts = __ballot_sync(0xffffffffu, l >= 0 && (lx == 0 || left != l));
  const int row = t - lx;
  const int run = row + 31 - __clz(starts & (0xffffffffu >> (31 - lx)));
  s_lay[t] = (signed char)l;
  s_par[t] = l >= 0 ? run : t;
  __syncthreads();
  volatile int* vp = s_par;  // parents change under other threads' atomics
  auto find = [&](int q) {
    int p = vp[q];
    while (p != q) { q = p; p = vp[q]; }
    return q;
  };
  auto unite = [&](int p, int q) {
    for (;;) {
      p = find(p);
      q = find(q);
      if (p == q) return;
      if (p < q) { const int w = p; p = q; q = w; }
      const int old = atomicMin(&s_par[p], q);
      if (old == p) return;
      p = old;
    }
  };
#pragma unroll
  for (int dir = 0; dir < 2; ++dir) {
    const int step = dir == 0 ? TX : TX * TY;
    const bool edge = dir == 0 ? ly > 0 : lz > 0;
    if (dir == 1 && TZ == 1) break;
    int other = -1;
    if (l >= 0 && edge && s_lay[t - step] == l) other = vp[t - step];  // a run start or its ancestor
    const unsigned key = other >= 0 ? ((unsigned)run << 16) | (unsigned)other : 0xffffffffu;
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    if (other >= 0 && lx == __ffs(grp) - 1) unite(run, other);
  }
  __syncthreads();
  if (!in) return;
  if (l < 0) {
    L[v] = -1;
    return;
  }
  int r = run;
  while (s_par[r] != r) r = s_par[r];
  const int rx = x - lx + r % TX, ry = y - ly + (r / TX) % TY, rz = z - lz + r / (TX * TY);
  L[v] = rx + g.nx * (ry + g.ny * rz);
}

// Cross-tile merges: each CTA takes one tile's three lower faces and unites
// every face voxel with its neighbour in the previous tile (same layer).
// Lanes holding the same (root-hint, root-hint) pair elect one lane, so a
// face shared by two tile components costs about one global union per warp.
template <int TX, int TY, int TZ>
__global__ void __launch_bounds__(256) k_ccl_faces(Geo g, const int* __restrict__ layer, int n_layers,
                                                   int* __restrict__ L) {
  constexpr int FX = TY * TZ, FY = TX * TZ, FZ = TX * TY;
  const int64_t ntx = (g.nx + TX - 1) / TX, nty = (g.ny + TY - 1) / TY;
  const int64_t b = blockIdx.x;
  const int x0 = (int)(b % ntx) * TX, y0 = (int)((b / ntx) % nty) * TY, z0 = (int)(b / (ntx * nty)) * TZ;
  for (int i = threadIdx.x; i < ((FX + FY + FZ + 31) / 32) * 32; i += blockDim.x) {
    int x = -1, y = 0, z = 0, d = 0;
    if (i < FX) {
      if (x0 > 0) { x = x0; y = y0 + i % TY; z = z0 + i / TY; d = 1; }
    } else if (i < FX + FY) {
      const int k = i - FX;
      if (y0 > 0) { x = x0 + k % TX; y = y0; z = z0 + k / TX; d = g.nx; }
    } else if (i < FX + FY + FZ) {
      const int k = i - FX - FY;
      if (z0 > 0) { x = x0 + k % TX; y = y0 + k / TX; z = z0; d = g.nxy; }
    }
    int a = -1, c = -1;
    if (x >= 0 && x < g.nx && y < g.ny && z < g.nz) {
      const int v = x + g.nx * (y + g.ny * z);
      const int l = layer[v];
      if (in_layers(l, n_layers) && layer[v - d] == l) {
        a = __ldcg(L + v);
        c = __ldcg(L + v - d);
      }
    }
    const unsigned long long key = ((unsigned long long)(unsigned)a << 32) | (unsigned)c;
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    if (a >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) uf_union(L, a, c);
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
