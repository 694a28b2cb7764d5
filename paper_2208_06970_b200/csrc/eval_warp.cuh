// eval_warp.cuh -- warp-per-voxel evaluation for small frontiers
// (_eval_voxel, _kernels.py:147-246).
//
// The tile kernels (eval_p1.cuh / eval_p2.cuh) give each voxel one thread,
// which is throughput-optimal but makes a round's latency the latency of one
// voxel's whole serial evaluation; the last rounds of every classify (and
// every round of thin 2D bands) hold only a few hundred voxels, so they run
// at that latency. Here a warp evaluates one voxel: lane k gathers neighbour
// OFFSETS[k] and forms its candidates in parallel, and the fold is resolved
// by warp reductions:
//
//   m  = the minimum-distance element over {current state} and all
//        candidates, d2 = the smallest distance among elements whose
//        (distance, site) differs from m's.
//   If d2 - m.d > 2.5e-9 + |m.d|*1e-15, neither EPS clause of `_beats` can
//   fire between m and any other element, so the reference's sequential
//   fold ends at m provided m is acceptable (the current state, a path
//   candidate, or a LOS / shortcut candidate with a clear ray): m beats
//   whatever is best when the fold reaches it and nothing displaces it
//   afterwards; blocked elements only reject themselves (failed_site merely
//   memoises a ray that would fail again). Elements identical to m in
//   (distance, site) but with another src matter only when m is not the
//   current state (then the first acceptable one in fold order wins).
//   Otherwise -- a near-tie, such duplicates, or a blocked winner -- lane 0
//   replays the exact sequential fold over the gathered candidates.
#pragma once
#include "classify.cuh"
#include "mg.cuh"

namespace lrcvt {

constexpr int EW_WARPS = 4;  // voxels per CTA

__device__ __forceinline__ double ew_min(double d) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d = fmin(d, __shfl_xor_sync(0xffffffffu, d, o));
  return d;
}

// element kinds
constexpr int EW_NONE = -1, EW_PATH = 0, EW_LOS = 1, EW_SHORT = 2;

// Resolve one voxel from per-lane elements (up to two per lane, lane k =
// neighbour k, slot 0 before slot 1 in fold order). Returns true when the
// strict rule decided (result in best_*), false when the exact replay is
// needed. All lanes of the warp must call it.
__device__ __forceinline__ bool ew_strict(const int lane, const double orig_d, const int orig_s,
                                          const int orig_src, const double* ed, const int* es,
                                          const int* esrc, const int* et, const Geo& g, const int* comp,
                                          const uint32_t* nbm, const double4* site_pos, unsigned nbv, double px,
                                          double py,
                                          double pz, int cv, double& best_d, int& best_s, int& best_src) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double lmin = lane == 0 ? orig_d : inf;
#pragma unroll
  for (int e = 0; e < 2; e++)
    if (et[e] != EW_NONE) lmin = fmin(lmin, ed[e]);
  const double dmin = ew_min(lmin);
  // the site of m: every element at dmin must carry it
  int ms = 0x7fffffff;
  if (lane == 0 && orig_d == dmin) ms = orig_s;
#pragma unroll
  for (int e = 0; e < 2; e++)
    if (et[e] != EW_NONE && ed[e] == dmin) ms = min(ms, es[e]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ms = min(ms, __shfl_xor_sync(0xffffffffu, ms, o));
  const bool m_is_orig = orig_d == dmin && orig_s == ms;
  bool bad = false;  // another site at dmin, or (m not current) an equal element with another src
  int src_lo = 0x7fffffff, src_hi = -1;  // range of src over the copies of m
  double l2 = inf;
#pragma unroll
  for (int e = 0; e < 2; e++) {
    if (et[e] == EW_NONE) continue;
    if (ed[e] == dmin && es[e] == ms) {
      src_lo = min(src_lo, esrc[e]);
      src_hi = max(src_hi, esrc[e]);
    } else {
      bad |= ed[e] == dmin;
      l2 = fmin(l2, ed[e]);
    }
  }
  if (lane == 0 && !(orig_d == dmin && orig_s == ms)) {
    bad |= orig_d == dmin;
    l2 = fmin(l2, orig_d);
  }
  const double d2 = ew_min(l2);
  bad = __any_sync(0xffffffffu, bad);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    src_lo = min(src_lo, __shfl_xor_sync(0xffffffffu, src_lo, o));
    src_hi = max(src_hi, __shfl_xor_sync(0xffffffffu, src_hi, o));
  }
  if (!m_is_orig && src_lo != src_hi) bad = true;  // same (d, site) via different src
  const bool isolated = isinf(d2) || (!isinf(dmin) && __dsub_rn(d2, dmin) > __dadd_rn(2.5e-9, __dmul_rn(fabs(dmin), 1e-15)));
  if (bad || !isolated) return false;
  if (m_is_orig) {
    best_d = orig_d; best_s = orig_s; best_src = orig_src;
    return true;
  }
  // kind of m: PATH wins if any copy is a path (no ray); else its ray decides
  int has_path = 0, kind = EW_NONE;
#pragma unroll
  for (int e = 0; e < 2; e++)
    if (et[e] != EW_NONE && ed[e] == dmin && es[e] == ms) {
      if (et[e] == EW_PATH) has_path = 1;
      kind = et[e];
    }
  has_path = __any_sync(0xffffffffu, has_path);
  const unsigned holders = __ballot_sync(0xffffffffu, kind != EW_NONE);
  const int holder = __ffs(holders) - 1;
  kind = __shfl_sync(0xffffffffu, kind, holder);
  bool clear = true;
  if (!has_path) {
    int ok = 0;
    if (lane == holder) {
      double qx, qy, qz;
      if (kind == EW_LOS) {
        const double4 sp = ld_d4(site_pos + ms);
        qx = sp.x; qy = sp.y; qz = sp.z;
      } else {
        int ux, uy, uz;
        coords(g, src_lo, ux, uy, uz);
        qx = centre1(ux, g.sx); qy = centre1(uy, g.sy); qz = centre1(uz, g.sz);
      }
      ok = (ray_clear_near(nbv, qx, qy, qz, px, py, pz, (float)(1.0 / g.sx), (float)(1.0 / g.sy),
                           (float)(1.0 / g.sz)) ||
            segment_clear_fast(comp, nbm, box_of(g), px, py, pz, qx, qy, qz, cv))
               ? 1 : 0;
    }
    clear = __shfl_sync(0xffffffffu, ok, holder) != 0;
  }
  if (!clear) return false;
  best_d = dmin; best_s = ms; best_src = src_lo;
  return true;
}

// The reference's sequential fold over the gathered elements (slot order).
__device__ __forceinline__ void ew_exact(const double (*ed)[2], const int (*es)[2], const int (*esrc)[2],
                                         const int (*et)[2], const Geo& g, const int* comp,
                                         const uint32_t* nbm, const double4* site_pos, unsigned nbv, double px,
                                         double py,
                                         double pz, int cv, double& best_d, int& best_s, int& best_src) {
  int failed = -1;
  const float isx = g.isx, isy = g.isy, isz = g.isz;
  for (int k = 0; k < 26; k++) {
    for (int e = 0; e < 2; e++) {
      const int t = et[k][e];
      if (t == EW_NONE) continue;
      const double d = ed[k][e];
      const int s = es[k][e];
      if (!beats(d, s, best_d, best_s)) continue;
      if (t == EW_PATH) {
        best_d = d; best_s = s; best_src = esrc[k][e];
        continue;
      }
      if (t == EW_LOS && s == failed) continue;
      double qx, qy, qz;
      if (t == EW_LOS) {
        const double4 sp = ld_d4(site_pos + s);
        qx = sp.x; qy = sp.y; qz = sp.z;
      } else {
        int ux, uy, uz;
        coords(g, esrc[k][e], ux, uy, uz);
        qx = centre1(ux, g.sx); qy = centre1(uy, g.sy); qz = centre1(uz, g.sz);
      }
      if (ray_clear_near(nbv, qx, qy, qz, px, py, pz, isx, isy, isz) ||
          segment_clear_fast(comp, nbm, box_of(g), px, py, pz, qx, qy, qz, cv)) {
        best_d = d; best_s = s; best_src = esrc[k][e];
      } else if (t == EW_LOS) {
        failed = s;
      }
    }
  }
}

// PHASE2 = false: LOS candidates only (phase 1); true: path + LOS/shortcut.
// shared staging of one warp's elements for the exact replay
struct EwStage {
  double d[26][2];
  int s[26][2], src[26][2], t[26][2];
};

// loads of per-round state: read-only cache across launches, L2 (coherent)
// inside the persistent small-round kernel where earlier rounds' writes by
// other SMs must be seen
template <bool COH, typename T>
__device__ __forceinline__ T ldst(const T* p) {
  if (COH) return __ldcg(p);
  return __ldg(p);
}

// evaluate frontier item i of `list` with the calling warp (all 32 lanes)
template <bool PHASE2, bool COH, bool MG = false>
__device__ __forceinline__ void ew_voxel(const int* list, const int2* ss, const int* site1, const double* dist,
                                         const int i, const Geo& g, const int* __restrict__ comp,
                                         const uint32_t* __restrict__ nbm, const double4* __restrict__ site_pos,
                                         uint32_t* __restrict__ bm, Prop* __restrict__ imp,
                                         uint8_t* __restrict__ pf, EwStage& st,
                                         const PeerView* __restrict__ pv = nullptr,
                                         const BoundaryOut* bo = nullptr) {
  const int lane = threadIdx.x & 31;
  const int v = ldst<COH>(list + i);
  int x, y, z;
  coords(g, v, x, y, z);
  const int cv = __ldg(comp + v);
  const double px = centre1(x, g.sx), py = centre1(y, g.sy), pz = centre1(z, g.sz);
  const unsigned nbv = __ldg(nbm + v);
  int2 sv;
  double orig_d;
  if (PHASE2) {
    sv = ldst<COH>(ss + v);
    orig_d = ldst<COH>(dist + v);
  } else {  // phase 1: LOS state, distance |c_v - p_site| recomputed
    const int s1 = ldst<COH>(site1 + v);
    sv = make_int2(s1, s1 >= 0 ? v : -1);
    if (s1 >= 0) {
      const double4 sp = ld_d4(site_pos + s1);
      orig_d = dist3(px, py, pz, sp.x, sp.y, sp.z);
    } else {
      orig_d = __longlong_as_double(0x7ff0000000000000LL);
    }
  }
  const int orig_s = sv.x, orig_src = sv.y;
  if (lane == 0) bm[v >> 5] = 0u;  // consume this round's frontier word
  double ed[2] = {0.0, 0.0};
  int es[2] = {-1, -1}, esrc[2] = {-1, -1}, et[2] = {EW_NONE, EW_NONE};
  if (lane < 26 && ((nbv >> lane) & 1u)) {
    const char4 o = c_off[lane];
    const int w = nbr_index(v, o, g.nx, g.nxy);
    // phase 1 keeps only the compact LOS site (src == w implied); phase 2 reads (site, src)
    int2 nw;
    if (PHASE2) {
      nw = ldst<COH>(ss + w);
    } else {
      const int s1 = ldst<COH>(site1 + w);
      nw = make_int2(s1, s1 >= 0 ? w : -1);
    }
    if (nw.x >= 0) {
      if (PHASE2) {
        double len;
        if (g.dyadic) {
          len = len_of(g, off_cls(lane));
        } else {
          len = dist3(px, py, pz, centre1(x + o.x, g.sx), centre1(y + o.y, g.sy), centre1(z + o.z, g.sz));
        }
        ed[0] = __dadd_rn(ldst<COH>(dist + w), len); es[0] = nw.x; esrc[0] = w; et[0] = EW_PATH;
      }
      if (nw.y == w) {
        const double4 sp = ld_d4(site_pos + nw.x);
        ed[1] = dist3(px, py, pz, sp.x, sp.y, sp.z); es[1] = nw.x; esrc[1] = v; et[1] = EW_LOS;
      } else if (PHASE2 && nw.y >= 0) {
        const int u = nw.y;
        const int2 nu = MG ? ld_ss<true>(pv, ss, u) : ldst<COH>(ss + u);
        if (nu.x >= 0 && __ldg(comp + u) == cv) {
          int ux, uy, uz;
          coords(g, u, ux, uy, uz);
          ed[1] = __dadd_rn(MG ? ld_dist<true>(pv, dist, u) : ldst<COH>(dist + u),
                            dist3(px, py, pz, centre1(ux, g.sx), centre1(uy, g.sy), centre1(uz, g.sz)));
          es[1] = nu.x; esrc[1] = u; et[1] = EW_SHORT;
        }
      }
    }
  }
  double best_d = orig_d;
  int best_s = orig_s, best_src = orig_src;
  const bool decided = ew_strict(lane, orig_d, orig_s, orig_src, ed, es, esrc, et, g, comp, nbm, site_pos, nbv, px,
                                 py, pz, cv, best_d, best_s, best_src);
  if (!decided) {
    if (lane < 26) {
#pragma unroll
      for (int e = 0; e < 2; e++) {
        st.d[lane][e] = ed[e]; st.s[lane][e] = es[e];
        st.src[lane][e] = esrc[e]; st.t[lane][e] = et[e];
      }
    }
    __syncwarp();
    if (lane == 0) {
      best_d = orig_d; best_s = orig_s; best_src = orig_src;
      ew_exact(st.d, st.s, st.src, st.t, g, comp, nbm, site_pos, nbv, px, py, pz, cv, best_d, best_s, best_src);
    }
    __syncwarp();  // st is reused by this warp's next item
  }
  if (lane == 0) {
    const bool improved = (best_s != orig_s) || (best_d < __dsub_rn(orig_d, LRCVT_EPS));
    if (improved) {  // sparse proposal slot i (k_commit reads pf)
      Prop pr;
      pr.d = best_d; pr.v = v; pr.s = best_s; pr.src = best_src; pr.pad = 0;
      imp[i] = pr;
      emit_boundary(bo, pr);
    }
    pf[i] = improved ? 1 : 0;
  }
}

template <bool PHASE2, bool MG = false>
__global__ void __launch_bounds__(32 * EW_WARPS) k_eval_warp(RoundCtl* __restrict__ ctl, Geo g,
                                                             const int* __restrict__ comp,
                                                             const uint32_t* __restrict__ nbm,
                                                             const double4* __restrict__ site_pos,
                                                             uint32_t* __restrict__ bm, Prop* __restrict__ imp,
                                                             uint8_t* __restrict__ pf,
                                                             const PeerView* __restrict__ pv = nullptr) {
  __shared__ EwStage stage[EW_WARPS];
  const int wid = threadIdx.x >> 5;
  const int i = blockIdx.x * EW_WARPS + wid;
  if (i >= ctl->n_cur) return;  // warp-uniform
  ew_voxel<PHASE2, false, MG>(ctl->cur, ctl->ss, ctl->site1, ctl->dist, i, g, comp, nbm, site_pos, bm, imp, pf,
                              stage[wid], pv, &ctl->bo);
}

}  // namespace lrcvt
