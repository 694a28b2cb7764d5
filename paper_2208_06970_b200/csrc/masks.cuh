// masks.cuh -- level-set (isoband) and connected-component restriction masks.
//
// classify_isobands (grid.py:140-163): band i iff iso[i] < f <= iso[i+1],
//   i.e. searchsorted(iso, f64(f), 'left') - 1, NONE outside. One streaming
//   pass: 4 B read + 4 B write per voxel, 128-bit vectorised.
// label_components (grid.py:166-220): 6-connected (4 in 2D) components per
//   layer with dense ids ordered by (layer, first voxel in row-major order).
//   Tile-local union-find in shared memory (k_ccl_tile), then a lock-free
//   global union-find over tile faces (k_ccl_faces). Every union links the
//   larger root under the smaller one (atomicMin), so every tree's root is
//   its component's minimum flat index -- the reference's "first
//   occurrence" -- independent of thread timing. Ids: radix sort of the
//   global roots by (layer, voxel).
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

// Tile-local labelling: one CTA per TX x TY x TZ tile, TX*TY threads; a
// warp is one x-row (TX = 32) and every thread walks its TZ voxels along z,
// so TZ independent loads per thread are in flight. Rows first, without
// atomics: a lane's run start comes from a ballot of "layer differs from the
// left neighbour". Then the y and z adjacencies unite run starts in a
// shared-memory union-find (larger index linked under smaller, atomicMin),
// one union per distinct (run, neighbour-run) pair in the warp. Local
// row-major order equals global row-major order restricted to the tile, so
// a local root is also the minimum global index of that tile component;
// every voxel then points at its local root in global L, and the local roots
// (the only possible global roots) are appended to a compact list.
template <int TX, int TY, int TZ>
__global__ void __launch_bounds__(TX * TY) k_ccl_tile(Geo g, const int* __restrict__ layer, int n_layers,
                                                      int* __restrict__ L, int* __restrict__ local_roots,
                                                      int* __restrict__ n_local) {
  static_assert(TX == 32, "a warp is one x-row of the tile");
  constexpr int T = TX * TY * TZ, P = TX * TY;
  __shared__ int s_par[T];
  __shared__ signed char s_lay[T];
  __shared__ int s_root_list[T];
  __shared__ int s_nroot, s_base;
  const int t0 = threadIdx.x;  // position in a z-plane of the tile
  const int lx = t0 % TX, ly = t0 / TX;
  const int64_t ntx = (g.nx + TX - 1) / TX, nty = (g.ny + TY - 1) / TY;
  const int64_t b = blockIdx.x;
  const int x = (int)(b % ntx) * TX + lx;
  const int y = (int)((b / ntx) % nty) * TY + ly;
  const int z0 = (int)(b / (ntx * nty)) * TZ;
  const int nzt = min(TZ, g.nz - z0);  // planes of this tile inside the grid
  const bool in_xy = x < g.nx && y < g.ny;
  const int v0 = x + g.nx * (y + g.ny * z0);
  if (t0 == 0) s_nroot = 0;
  {
    int l[TZ];
#pragma unroll
    for (int k = 0; k < TZ; ++k) l[k] = in_xy && k < nzt ? __ldcs(layer + v0 + (int64_t)k * g.nxy) : -1;
#pragma unroll
    for (int k = 0; k < TZ; ++k) {
      const int lk = in_layers(l[k], n_layers) ? l[k] : -1;
      const int left = __shfl_up_sync(0xffffffffu, lk, 1);
      const unsigned starts = __ballot_sync(0xffffffffu, lk >= 0 && (lx == 0 || left != lk));
      const int t = k * P + t0;
      s_lay[t] = (signed char)lk;
      s_par[t] = lk >= 0 ? t - lx + 31 - __clz(starts & (0xffffffffu >> (31 - lx))) : t;
    }
  }
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
  // y and z adjacencies between runs; a lane unites only where its
  // (run, neighbour) pair differs from its left neighbour's. Shuffles first
  // (warp-uniform trip count), unions after.
#pragma unroll 1
  for (int k = 0; k < TZ; ++k) {
    const int t = k * P + t0;
    const int l = k < nzt ? (int)s_lay[t] : -1;
    const bool start = l >= 0 && (lx == 0 || s_lay[t - 1] != l);
    const int run = start ? t : (l >= 0 ? vp[t] : -1);  // non-starts keep their run start as parent
    int oy = -1, oz = -1;
    if (l >= 0 && ly > 0 && s_lay[t - TX] == l) oy = vp[t - TX];
    if (TZ > 1 && l >= 0 && k > 0 && s_lay[t - P] == l) oz = vp[t - P];
    const int run_left = __shfl_up_sync(0xffffffffu, run, 1);
    const int oy_left = __shfl_up_sync(0xffffffffu, oy, 1);
    const int oz_left = __shfl_up_sync(0xffffffffu, oz, 1);
    const bool fresh = lx == 0 || run != run_left;
    if (oy >= 0 && (fresh || oy != oy_left)) unite(run, oy);
    if (oz >= 0 && (fresh || oz != oz_left)) unite(run, oz);
    __syncwarp();
  }
  __syncthreads();
  // run starts resolve their root once; every voxel then needs one hop.
  // Roots are gathered in shared memory, then appended with one atomic.
#pragma unroll 1
  for (int k = 0; k < nzt; ++k) {
    const int t = k * P + t0;
    const int l = s_lay[t];
    if (l >= 0 && (lx == 0 || s_lay[t - 1] != l)) {
      int r = t;
      while (vp[r] != r) r = vp[r];
      if (r == t) {
        if (in_xy) s_root_list[atomicAdd(&s_nroot, 1)] = v0 + k * g.nxy;
      } else {
        vp[t] = r;
      }
    }
  }
  __syncthreads();
  if (t0 == 0) s_base = s_nroot ? atomicAdd(n_local, s_nroot) : 0;
  __syncthreads();
  for (int i = t0; i < s_nroot; i += P) local_roots[s_base + i] = s_root_list[i];
#pragma unroll 1
  for (int k = 0; k < nzt; ++k) {
    if (!in_xy) break;
    const int t = k * P + t0;
    const int v = v0 + k * g.nxy;
    const int l = s_lay[t];
    if (l < 0) {
      L[v] = -1;
      continue;
    }
    int r = s_par[t];
    if (r != t) r = s_par[r];  // voxel -> run start -> root
    const int rz = r / P, rp = r % P;
    L[v] = (x - lx + rp % TX) + g.nx * ((y - ly + rp / TX) + g.ny * (z0 + rz));
  }
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

// sort key of each local root: (layer << 31 | voxel) if it is still a global
// root after the face unions, else (n_layers << 31), which sorts last
__global__ void k_ccl_root_keys(const int* __restrict__ local_roots, int n_local, const int* __restrict__ L,
                                const int* __restrict__ layer, int n_layers,
                                unsigned long long* __restrict__ key, int* __restrict__ n_roots) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool root = false;
  if (i < n_local) {
    const int r = local_roots[i];
    root = __ldcg(L + r) == r;
    key[i] = root ? ((unsigned long long)layer[r] << 31) | (unsigned)r : (unsigned long long)n_layers << 31;
  }
  const unsigned m = __ballot_sync(0xffffffffu, root);
  if (m && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(n_roots, __popc(m));
}

// local roots point straight at their global root afterwards
__global__ void k_ccl_compress_roots(const int* __restrict__ local_roots, int n_local, int* __restrict__ L) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_local) return;
  const int r = local_roots[i];
  const int q = uf_find(L, r);
  if (q != r) L[r] = q;
}

// dense id of every global root (keys sorted by (layer, voxel)), stored in
// the root's own L slot as -(id) - 2 (-1 stays "not in a layer")
__global__ void k_ccl_root_ids(const unsigned long long* __restrict__ sorted, int n_local, int n_layers,
                               int* __restrict__ L) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_local && (int)(sorted[i] >> 31) < n_layers) L[(int)(sorted[i] & 0x7fffffffu)] = -i - 2;
}

// every voxel takes its root's id: voxel -> local root -> global root, at
// most two hops once the local roots are compressed. L is read-only here.
__global__ void k_ccl_relabel(const int* __restrict__ L, int64_t n, int* __restrict__ comp, bool vec4) {
  const int64_t n4 = vec4 ? n / 4 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto one = [&](int p) {
    if (p == -1) return (int)LRCVT_NONE;
    if (p < -1) return -p - 2;
    int q = __ldg(L + p);
    if (q < -1) return -q - 2;
    q = __ldg(L + q);
    return -q - 2;
  };
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const int4 p = __ldg(reinterpret_cast<const int4*>(L) + i);
    __stcs(reinterpret_cast<int4*>(comp) + i, make_int4(one(p.x), one(p.y), one(p.z), one(p.w)));
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    comp[i] = one(__ldg(L + i));
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

// Same table with the per-warp partials merged in shared memory first (one
// global atomic per component per CTA instead of per warp): few components
// otherwise serialise every warp on the same six addresses. n_comp <= SMEM_COMP.
constexpr int TABLE_SMEM_COMP = 512;
__global__ void __launch_bounds__(256) k_ccl_table_smem(Geo g, const int* __restrict__ comp,
                                                        const int* __restrict__ layer, int n_comp,
                                                        unsigned long long* __restrict__ count,
                                                        int* __restrict__ bbox, int* __restrict__ layer_of) {
  __shared__ unsigned long long s_cnt[TABLE_SMEM_COMP];
  __shared__ int s_box[TABLE_SMEM_COMP][6];
  __shared__ int s_lay[TABLE_SMEM_COMP];
  for (int c = threadIdx.x; c < n_comp; c += blockDim.x) {
    s_cnt[c] = 0;
    s_box[c][0] = s_box[c][1] = s_box[c][2] = 0x7fffffff;
    s_box[c][3] = s_box[c][4] = s_box[c][5] = -1;
    s_lay[c] = -1;
  }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < g.n; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    int c = -1, x = 0, y = 0, z = 0;
    if (i < g.n) {
      c = comp[i];
      if (c >= 0) coords(g, (int)i, x, y, z);
    }
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    const unsigned cnt = __popc(grp);
    const int xmin = __reduce_min_sync(grp, x), xmax = __reduce_max_sync(grp, x);
    const int ymin = __reduce_min_sync(grp, y), ymax = __reduce_max_sync(grp, y);
    const int zmin = __reduce_min_sync(grp, z), zmax = __reduce_max_sync(grp, z);
    if (c >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) {
      atomicAdd(&s_cnt[c], (unsigned long long)cnt);
      atomicMin(&s_box[c][0], xmin);
      atomicMin(&s_box[c][1], ymin);
      atomicMin(&s_box[c][2], zmin);
      atomicMax(&s_box[c][3], xmax);
      atomicMax(&s_box[c][4], ymax);
      atomicMax(&s_box[c][5], zmax);
      s_lay[c] = layer[i];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < n_comp; c += blockDim.x) {
    if (!s_cnt[c]) continue;
    atomicAdd(count + c, s_cnt[c]);
#pragma unroll
    for (int a = 0; a < 3; a++) {
      atomicMin(bbox + 6 * c + a, s_box[c][a]);
      atomicMax(bbox + 6 * c + 3 + a, s_box[c][3 + a]);
    }
    layer_of[c] = s_lay[c];
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
