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
// Three unrolled stages keep every load/atomic of a stage independent (26
// requests in flight per thread instead of 26 dependent round trips).
__device__ __forceinline__ void mark_and_append(const Geo& g, const int* __restrict__ comp,
                                                bool active, int v, bool self,
                                                uint32_t* __restrict__ bm,
                                                int* __restrict__ next, int* counter) {
  unsigned newmask = 0;
  if (active) {
    int x, y, z;
    coords(g, v, x, y, z);
    const int cv = __ldg(comp + v);
    const unsigned inb = inbounds_mask(x, y, z, g.nx, g.ny, g.nz);
    int cu[26];
#pragma unroll
    for (int k = 0; k < 26; k++) {
      const int u = v + off_dx(k) + off_dy(k) * g.nx + off_dz(k) * g.nxy;
      cu[k] = ((inb >> k) & 1u) ? __ldg(comp + u) : -2;
    }
    unsigned same = self ? (1u << 26) : 0u;
#pragma unroll
    for (int k = 0; k < 26; k++) same |= (cu[k] == cv ? 1u : 0u) << k;
    uint32_t words[27];
#pragma unroll
    for (int k = 0; k < 27; k++) {
      const int u = k < 26 ? v + off_dx(k) + off_dy(k) * g.nx + off_dz(k) * g.nxy : v;
      words[k] = ((same >> k) & 1u) ? __ldcg(bm + (u >> 5)) : 0xffffffffu;
    }
#pragma unroll
    for (int k = 0; k < 27; k++) {
      const int u = k < 26 ? v + off_dx(k) + off_dy(k) * g.nx + off_dz(k) * g.nxy : v;
      const uint32_t bit = 1u << (u & 31);
      if (((same >> k) & 1u) && !(words[k] & bit)) {
        const uint32_t old = atomicOr(bm + (u >> 5), bit);
        if (!(old & bit)) newmask |= 1u << k;
      }
    }
  }
  const int cnt = __popc(newmask);
  const int lane = threadIdx.x & 31;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int base = 0;
  if (lane == 31 && total) base = atomicAdd(counter, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  int pos = base + incl - cnt;
  if (newmask & (1u << 26)) next[pos++] = v;
  newmask &= ALL26;
  while (newmask) {
    const int k = __ffs(newmask) - 1;
    newmask &= newmask - 1;
    const char4 o = c_off[k];
    next[pos++] = nbr_index(v, o, g.nx, g.nxy);
  }
}

// _kernels.py:147-246 for one voxel. Returns improved; fills the proposal.
//
// Written as a resumable per-lane state machine. Each iteration of the
// outer loop first ADVANCES the lane through its neighbours (reference
// OFFSETS order, rolled loop over the in-bounds mask, next neighbour's loads
// software-pipelined) until it either finishes or reaches a candidate that
// needs a line-of-sight ray; then every lane with a pending ray runs its DDA
// together. A warp thus pays max(rays per lane) DDA passes instead of the
// sum that divergent inline rays cost. The decision sequence per voxel is
// unchanged: a ray is cast exactly when the reference casts it, and its
// result is applied before the lane looks at the next neighbour.
template <bool PHASE2, bool DYADIC>
__device__ __forceinline__ bool eval_voxel(const Geo& g, const double* __restrict__ s_len, int v,
                                           bool active,
                                           const int* __restrict__ comp,
                                           const int2* __restrict__ ss,
                                           const double* __restrict__ dist,
                                           const double4* __restrict__ site_pos,
                                           Prop& out) {
  int x = 0, y = 0, z = 0;
  if (active) coords(g, v, x, y, z);
  const int cv = active ? __ldg(comp + v) : -3;
  const double px = centre1(x, g.sx), py = centre1(y, g.sy), pz = centre1(z, g.sz);
  const int2 sv = active ? ss[v] : make_int2(-1, -1);
  double best_d = active ? dist[v] : 0.0;
  int best_s = sv.x, best_src = sv.y;
  const double orig_d = best_d;
  const int orig_s = best_s;
  int failed_site = -1;
  int cache_s = -1, cache_s2 = -1;  // site -> distance memo (pure in (v, site))
  double cache_d = 0.0, cache_d2 = 0.0;
  int cache_u = -1, cache_u2 = -1;  // node -> candidate memo (pure in (v, u) per round)
  double cache_ud = 0.0, cache_ud2 = 0.0;
  double thr = beat_threshold(best_d);

  unsigned rem = active ? inbounds_mask(x, y, z, g.nx, g.ny, g.nz) : 0u;
  bool done = rem == 0;
  char4 o = c_off[done ? 0 : __ffs(rem) - 1];
  int w = active ? nbr_index(v, o, g.nx, g.nxy) : 0;
  int cw = done ? -4 : __ldg(comp + w);
  int2 nw = done ? make_int2(-1, -1) : ss[w];
  double dw = (PHASE2 && !done) ? dist[w] : 0.0;

  // pending ray: segment p -> (qx, qy, qz); on success best := (rd, rs, rsrc)
  bool pending = false;
  bool ray_los = false;
  double qx = 0, qy = 0, qz = 0, rd = 0;
  int rs = 0, rsrc = 0;

  while (!done) {
    // ---- advance until a ray is needed or the neighbours run out
    while (!done && !pending) {
      rem &= rem - 1;
      const char4 o2 = rem ? c_off[__ffs(rem) - 1] : o;
      const int w2 = nbr_index(v, o2, g.nx, g.nxy);
      const int cw2 = __ldg(comp + w2);
      const int2 nw2 = ss[w2];
      const double dw2 = PHASE2 ? dist[w2] : 0.0;

      const int sw = nw.x;
      if (cw == cv && sw >= 0) {
        if (PHASE2) {
          double len;
          if (DYADIC) {
            len = s_len[o.w];
          } else {
            len = dist3(px, py, pz, centre1(x + o.x, g.sx), centre1(y + o.y, g.sy),
                        centre1(z + o.z, g.sz));
          }
          const double d = __dadd_rn(dw, len);
          if (beats(d, sw, best_d, best_s)) {
            best_d = d; best_s = sw; best_src = w; thr = beat_threshold(best_d);
          }
        }
        const int u = nw.y;
        if (u == w) {
          // w sees its site: try the same direct connection. d is a pure
          // function of (v, site): two-entry memo, exact lower-bound skip.
          double d = 0.0;
          bool have = true;
          if (sw == cache_s) {
            d = cache_d;
          } else if (sw == cache_s2) {
            d = cache_d2;
          } else {
            const double4 sp = ld_d4(site_pos + sw);
            if (dist_lower(px, py, pz, sp.x, sp.y, sp.z) >= thr) {
              have = false;
            } else {
              d = dist3(px, py, pz, sp.x, sp.y, sp.z);
              cache_s2 = cache_s; cache_d2 = cache_d;
              cache_s = sw; cache_d = d;
            }
          }
          if (have && d < thr && beats(d, sw, best_d, best_s) && sw != failed_site) {
            const double4 sp = ld_d4(site_pos + sw);
            pending = true; ray_los = true;
            qx = sp.x; qy = sp.y; qz = sp.z; rd = d; rs = sw; rsrc = v;
          }
        } else if (PHASE2 && u >= 0) {
          // shortcut to w's own path node u. d = RN(du + |p - c_u|) >= du, so
          // dist[u] alone prescreens before site/comp of u are fetched.
          const double du = dist[u];
          if (du < thr) {
            double d = 0.0;
            bool have = false;
            double upx = 0, upy = 0, upz = 0;
            if (u == cache_u) {
              d = cache_ud; have = true;
            } else if (u == cache_u2) {
              d = cache_ud2; have = true;
            }
            const int2 nu = ss[u];
            const int su = nu.x;
            if (su >= 0 && __ldg(comp + u) == cv) {
              int ux, uy, uz;
              coords(g, u, ux, uy, uz);
              upx = centre1(ux, g.sx); upy = centre1(uy, g.sy); upz = centre1(uz, g.sz);
              if (!have && __dadd_rn(du, dist_lower(px, py, pz, upx, upy, upz)) < thr) {
                d = __dadd_rn(du, dist3(px, py, pz, upx, upy, upz));
                cache_u2 = cache_u; cache_ud2 = cache_ud;
                cache_u = u; cache_ud = d;
                have = true;
              }
              if (have && beats(d, su, best_d, best_s)) {
                pending = true; ray_los = false;
                qx = upx; qy = upy; qz = upz; rd = d; rs = su; rsrc = u;
              }
            }
          }
        }
      }
      if (!rem) done = true;
      o = o2; w = w2; cw = cw2; nw = nw2; dw = dw2;
    }
    // ---- lanes with a pending ray trace it together
    if (pending) {
      if (segment_clear(comp, g, px, py, pz, qx, qy, qz, cv)) {
        best_d = rd; best_s = rs; best_src = rsrc; thr = beat_threshold(best_d);
      } else if (ray_los) {
        failed_site = rs;
      }
      pending = false;
    }
  }
  out.d = best_d; out.v = v; out.s = best_s; out.src = best_src; out.pad = 0;
  return active && ((best_s != orig_s) || (best_d < __dsub_rn(orig_d, LRCVT_EPS)));
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
  __shared__ double s_len[8];
  if (threadIdx.x < 8) s_len[threadIdx.x] = len_of(g, threadIdx.x == 0 ? 1 : threadIdx.x);
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  Prop pr;
  const bool active = i < n;
  const int v = active ? list[i] : 0;
  if (active) bm[v >> 5] = 0u;
  const bool improved = eval_voxel<PHASE2, DYADIC>(g, s_len, v, active, comp, ss, dist, site_pos, pr);
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
