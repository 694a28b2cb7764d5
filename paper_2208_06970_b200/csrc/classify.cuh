// classify.cuh -- restricted geodesic region growing (voronoi_classify).
//
// Maps the reference's worklist schedule (tessellation.py:102-208,
// _kernels.py:249-454) onto three kinds of launches per relaxation round:
//
//   k_eval<PHASE2>  one thread per frontier voxel; evaluates it against the
//                   pre-round state (_eval_voxel, _kernels.py:147-246) and
//                   appends improved proposals to a compact list;
//   k_commit        commits the proposals and enqueues the same-component
//                   26-neighbours of every improved voxel, deduplicated by a
//                   1-bit-per-voxel frontier bitmap (_apply_and_enqueue,
//                   _kernels.py:285-334);
//   the host loop   swaps the lists until the frontier drains (_run_phase,
//                   _kernels.py:337-385) and runs the phase-2 verification
//                   sweeps (tessellation.py:170-189).
//
// Because each round reads only the pre-round state and the next frontier
// is a SET, list order never affects results: bit-exact with the reference.
#pragma once
#include "common.cuh"

namespace lrcvt {

// Improved proposal (24 B): written by k_eval, consumed by k_commit.
struct Prop {
  double d;
  int v, s, src, pad;
};

// Counter slots in the plan's small device array.
enum { C_NIMP = 0, C_NNEXT = 1, C_BAD = 2, C_ASSIGNED = 3, C_NCOUNTERS = 8 };

__global__ void k_fill_state(int2* __restrict__ ss, double* __restrict__ dist, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    ss[i] = make_int2(LRCVT_NONE, LRCVT_NONE);
    dist[i] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  }
}

// has_site[c] = 1 for every component that owns a site (tessellation.py:161-162)
__global__ void k_mark_site_comps(const int* __restrict__ site_comp, int n_sites,
                                  uint8_t* __restrict__ has_site) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_sites) has_site[site_comp[s]] = 1;
}

// Ordered compaction of eligible voxels (in-band, component has a site),
// tessellation.py:163-164. Each block owns a contiguous range; within it
// order is preserved, block ranges are placed by a decoupled counter, so the
// list is a permutation of sorted chunks (order never affects results).
template <int BLOCK, int PER_THREAD>
__global__ void k_eligible(const int* __restrict__ comp, const uint8_t* __restrict__ has_site,
                           int64_t n, int* __restrict__ out, int* __restrict__ counter) {
  __shared__ int warp_tot[BLOCK / 32];
  __shared__ int base_s;
  const int64_t chunk0 = (int64_t)blockIdx.x * BLOCK * PER_THREAD;
  // thread t owns voxels chunk0 + t*PER_THREAD .. +PER_THREAD-1
  int64_t v0 = chunk0 + (int64_t)threadIdx.x * PER_THREAD;
  unsigned flags = 0;
#pragma unroll
  for (int j = 0; j < PER_THREAD; j++) {
    int64_t v = v0 + j;
    if (v < n) {
      int c = comp[v];
      if (c >= 0 && has_site[c]) flags |= 1u << j;
    }
  }
  int cnt = __popc(flags);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int w = 0; w < BLOCK / 32; w++) { int t = warp_tot[w]; warp_tot[w] = acc; acc += t; }
    base_s = acc ? atomicAdd(counter, acc) : 0;
  }
  __syncthreads();
  int pos = base_s + warp_tot[wid] + incl - cnt;
  while (flags) {
    int j = __ffs(flags) - 1;
    flags &= flags - 1;
    out[pos++] = (int)(v0 + j);
  }
}

// Mark same-component neighbours of v (and v itself when `self`) in the
// frontier bitmap; newly set bits are appended to `next`. Reproduces the
// stamp-deduplicated enqueue of _kernels.py:313-333 (self=false) and
// _kernels.py:425-454 (self=true). All 32 lanes must call it.
__device__ __forceinline__ void mark_and_append(const Geo& g, const int* __restrict__ comp,
                                                bool active, int v, bool self,
                                                uint32_t* __restrict__ bm,
                                                int* __restrict__ next, int* counter) {
  unsigned newmask = 0;
  int x = 0, y = 0, z = 0, cv = 0;
  if (active) {
    coords(g, v, x, y, z);
    cv = __ldg(comp + v);
    if (self) {
      uint32_t bit = 1u << (v & 31);
      if (!(__ldcg(bm + (v >> 5)) & bit)) {
        uint32_t old = atomicOr(bm + (v >> 5), bit);
        if (!(old & bit)) newmask |= 1u << 26;
      }
    }
#pragma unroll
    for (int k = 0; k < 26; k++) {
      int dx, dy, dz;
      offset_of(k, dx, dy, dz);
      int ux = x + dx, uy = y + dy, uz = z + dz;
      if (ux < 0 || uy < 0 || uz < 0 || ux >= g.nx || uy >= g.ny || uz >= g.nz) continue;
      int u = v + g.off_d[k];
      if (__ldg(comp + u) != cv) continue;
      uint32_t bit = 1u << (u & 31);
      if (__ldcg(bm + (u >> 5)) & bit) continue;
      uint32_t old = atomicOr(bm + (u >> 5), bit);
      if (!(old & bit)) newmask |= 1u << k;
    }
  }
  int cnt = __popc(newmask);
  int lane = threadIdx.x & 31;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  int total = __shfl_sync(0xffffffffu, incl, 31);
  int base = 0;
  if (lane == 31 && total) base = atomicAdd(counter, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  int pos = base + incl - cnt;
  if (newmask & (1u << 26)) next[pos++] = v;
  newmask &= (1u << 26) - 1;
  while (newmask) {
    int k = __ffs(newmask) - 1;
    newmask &= newmask - 1;
    next[pos++] = v + g.off_d[k];
  }
}

// _kernels.py:147-246 for one voxel. Returns improved; fills the proposal.
template <bool PHASE2, bool DYADIC>
__device__ __forceinline__ bool eval_voxel(const Geo& g, int v, const int* __restrict__ comp,
                                           const int2* __restrict__ ss,
                                           const double* __restrict__ dist,
                                           const double4* __restrict__ site_pos,
                                           Prop& out) {
  int x, y, z;
  coords(g, v, x, y, z);
  const int cv = __ldg(comp + v);
  const double px = centre1(x, g.sx), py = centre1(y, g.sy), pz = centre1(z, g.sz);
  const int2 sv = ss[v];
  double best_d = dist[v];
  int best_s = sv.x, best_src = sv.y;
  const double orig_d = best_d;
  const int orig_s = best_s;
  int failed_site = -1;
  int cache_s = -1;  // same-site distance memo (pure function of (v, site))
  double cache_d = 0.0;
  int cache_u = -1;  // same-node shortcut memo
  double cache_ud = 0.0;
  double thr = beat_threshold(best_d);

#pragma unroll
  for (int k = 0; k < 26; k++) {
    int dx, dy, dz;
    offset_of(k, dx, dy, dz);
    int wx = x + dx, wy = y + dy, wz = z + dz;
    if (wx < 0 || wy < 0 || wz < 0 || wx >= g.nx || wy >= g.ny || wz >= g.nz) continue;
    const int w = v + g.off_d[k];
    if (__ldg(comp + w) != cv) continue;
    const int2 nw = ss[w];
    const int sw = nw.x;
    if (sw < 0) continue;
    if (PHASE2) {
      const double len = DYADIC ? g.off_len[k]
                                : dist3(px, py, pz, centre1(wx, g.sx), centre1(wy, g.sy),
                                        centre1(wz, g.sz));
      const double d = __dadd_rn(dist[w], len);
      if (beats(d, sw, best_d, best_s)) {
        best_d = d; best_s = sw; best_src = w; thr = beat_threshold(best_d);
      }
    }
    const int u = nw.y;
    if (u == w) {
      // w sees its site: try the same direct connection
      double d;
      if (sw == cache_s) {
        d = cache_d;
      } else {
        const double4 sp = ld_d4(site_pos + sw);
        d = dist3(px, py, pz, sp.x, sp.y, sp.z);
        cache_s = sw; cache_d = d;
      }
      if (d < thr && beats(d, sw, best_d, best_s) && sw != failed_site) {
        const double4 sp = ld_d4(site_pos + sw);
        if (segment_clear(comp, g, px, py, pz, sp.x, sp.y, sp.z, cv)) {
          best_d = d; best_s = sw; best_src = v; thr = beat_threshold(best_d);
        } else {
          failed_site = sw;
        }
      }
    } else if (PHASE2 && u >= 0) {
      // shortcut to w's own path node u
      const int2 nu = ss[u];
      const int su = nu.x;
      if (su >= 0 && __ldg(comp + u) == cv) {
        const double du = dist[u];
        // d = RN(du + |p - c_u|) >= du: exact skip when du already loses
        if (du < thr) {
          int ux, uy, uz;
          coords(g, u, ux, uy, uz);
          const double upx = centre1(ux, g.sx), upy = centre1(uy, g.sy), upz = centre1(uz, g.sz);
          double d;
          if (u == cache_u) {
            d = cache_ud;
          } else {
            d = __dadd_rn(du, dist3(px, py, pz, upx, upy, upz));
            cache_u = u; cache_ud = d;
          }
          if (beats(d, su, best_d, best_s)) {
            if (segment_clear(comp, g, px, py, pz, upx, upy, upz, cv)) {
              best_d = d; best_s = su; best_src = u; thr = beat_threshold(best_d);
            }
          }
        }
      }
    }
  }
  out.d = best_d; out.v = v; out.s = best_s; out.src = best_src; out.pad = 0;
  return (best_s != orig_s) || (best_d < __dsub_rn(orig_d, LRCVT_EPS));
}

// _kernels.py:249-282: evaluate a frontier list against the pre-round state.
// Also consumes the frontier bitmap words of the listed voxels (they were
// set by the previous k_commit / k_seed; nothing else sets bits meanwhile).
template <bool PHASE2, bool DYADIC>
__global__ void __launch_bounds__(128) k_eval(const int* __restrict__ list, int n, Geo g,
                                              const int* __restrict__ comp,
                                              const int2* __restrict__ ss,
                                              const double* __restrict__ dist,
                                              const double4* __restrict__ site_pos,
                                              uint32_t* __restrict__ bm,
                                              Prop* __restrict__ imp,
                                              int* __restrict__ counters) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool improved = false;
  Prop pr;
  if (i < n) {
    const int v = list[i];
    bm[v >> 5] = 0u;
    improved = eval_voxel<PHASE2, DYADIC>(g, v, comp, ss, dist, site_pos, pr);
  }
  const int slot = warp_append(counters + C_NIMP, improved);
  if (improved) imp[slot] = pr;
}

// _kernels.py:285-334: commit, then enqueue same-component neighbours.
__global__ void __launch_bounds__(128) k_commit(const Prop* __restrict__ imp,
                                                int* __restrict__ counters, Geo g,
                                                const int* __restrict__ comp,
                                                int2* __restrict__ ss,
                                                double* __restrict__ dist,
                                                uint32_t* __restrict__ bm,
                                                int* __restrict__ next) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n_imp = *(volatile int*)(counters + C_NIMP);
  if (blockIdx.x * blockDim.x >= n_imp) return;  // whole warp-uniform block exit
  const bool active = i < n_imp;
  int v = 0;
  if (active) {
    const Prop p = imp[i];
    v = p.v;
    ss[v] = make_int2(p.s, p.src);
    dist[v] = p.d;
  }
  mark_and_append(g, comp, active, v, false, bm, next, counters + C_NNEXT);
}

// _kernels.py:399-422, site part: seed voxel, distance, validity.
__global__ void k_site_voxel(Geo g, const int* __restrict__ comp, const double4* __restrict__ site_pos,
                             const int* __restrict__ site_comp, int n_sites,
                             int* __restrict__ key, int* __restrict__ val,
                             double* __restrict__ sd, int* __restrict__ counters) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sites) return;
  const double4 p = site_pos[s];
  const int x = cell_of(p.x, g.sx, g.nx), y = cell_of(p.y, g.sy, g.ny), z = cell_of(p.z, g.sz, g.nz);
  const int v = x + g.nx * (y + g.ny * z);
  val[s] = s;
  if (comp[v] != site_comp[s]) {
    atomicAdd(counters + C_BAD, 1);
    key[s] = 0x7fffffff;
    sd[s] = 0.0;
    return;
  }
  key[s] = v;
  sd[s] = dist3(centre1(x, g.sx), centre1(y, g.sy), centre1(z, g.sz), p.x, p.y, p.z);
}

// _kernels.py:399-422 contested-voxel rule + _kernels.py:425-454 initial
// worklist. Sites are sorted by (voxel, id) (stable radix sort), so each
// group head folds its group in increasing site id exactly like the serial
// reference loop, then enqueues the seed voxel and its same-component
// neighbours.
__global__ void __launch_bounds__(128) k_seed_groups(Geo g, const int* __restrict__ comp,
                                                     const int* __restrict__ key,
                                                     const int* __restrict__ val,
                                                     const double* __restrict__ sd_by_site,
                                                     int n_sites, int2* __restrict__ ss,
                                                     double* __restrict__ dist,
                                                     uint32_t* __restrict__ bm,
                                                     int* __restrict__ next,
                                                     int* __restrict__ counters) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool head = false;
  int v = 0;
  if (i < n_sites) {
    v = key[i];
    head = v != 0x7fffffff && (i == 0 || key[i - 1] != v);
  }
  if (head) {
    int cur_s = val[i];
    double cur_d = sd_by_site[cur_s];
    for (int j = i + 1; j < n_sites && key[j] == v; j++) {
      const int s = val[j];
      const double d = sd_by_site[s];
      if (beats(d, s, cur_d, cur_s)) { cur_s = s; cur_d = d; }
    }
    ss[v] = make_int2(cur_s, v);
    dist[v] = cur_d;
  }
  if (blockIdx.x * blockDim.x >= n_sites) return;
  mark_and_append(g, comp, head, v, true, bm, next, counters + C_NNEXT);
}

// tessellation.py:191-194 state bits, plus the `assigned` count.
__global__ void k_state(const int2* __restrict__ ss, int64_t n, uint8_t* __restrict__ state,
                        int* __restrict__ counters) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int cnt = 0;
  for (; i < n; i += stride) {
    const int2 a = ss[i];
    uint8_t st = 0;
    if (a.x != LRCVT_NONE) {
      st = 2 | 4;
      cnt++;
      if (a.y == (int)i) st |= 1;
    }
    if (state) state[i] = st;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(counters + C_ASSIGNED, cnt);
}

}  // namespace lrcvt
