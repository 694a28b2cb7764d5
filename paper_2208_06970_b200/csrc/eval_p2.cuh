// eval_p2.cuh -- phase-2 evaluation (_eval_voxel with phase2 = True,
// _kernels.py:147-246; tessellation.py:158-189).
//
// Same gather / tabulate / fold structure as eval_p1.cuh, with the three
// phase-2 candidates per neighbour w in OFFSETS order:
//   path      (dist[w] + |c_w - p|, site(w), w)          no ray
//   LOS       (|p - site(w)|, site(w), v)  if src(w)==w  ray to the site
//   shortcut  (dist[u] + |p - c_u|, site(u), u), u = src(w) != w, u in
//             the same component and assigned            ray to c_u
// A  the 26 neighbours' (site, node, dist) go into a per-thread shared-memory
//    row with all loads in flight together;
// B  the LOS distance of each distinct neighbour site and the shortcut
//    candidate of each distinct node are computed once (both are pure
//    functions of (v, site) / (v, node) within a round);
// C  the fold reads the row and the tables only; a candidate that needs a
//    ray parks the lane, the parked lanes trace together, apply the outcome
//    and resume at the next neighbour -- the reference's decision sequence.
#pragma once
#include "classify.cuh"
#include "mg.cuh"

namespace lrcvt {

#ifndef LRCVT_P2_STAB
#define LRCVT_P2_STAB 4
#endif
#ifndef LRCVT_P2_NTAB
#define LRCVT_P2_NTAB 1
#endif
constexpr int P2_STAB = LRCVT_P2_STAB;  // distinct LOS sites
constexpr int P2_NTAB = LRCVT_P2_NTAB;  // distinct shortcut nodes

// |c_w - c_v| for neighbour k: exact by offset class when the spacing is dyadic
template <bool DYADIC>
__device__ __forceinline__ double p2_len(const Geo& g, int k, int x, int y, int z, double px, double py, double pz) {
  if (DYADIC) return len_of(g, off_cls(k));
  return dist3(px, py, pz, centre1(x + off_dx(k), g.sx), centre1(y + off_dy(k), g.sy), centre1(z + off_dz(k), g.sz));
}

// MG: multi-GPU slab mode, the far node reads of shortcut candidates go
// through the PeerView (mg.cuh)
template <int BLOCK, bool DYADIC, bool MG>
__device__ __forceinline__ void p2_tile(const int* __restrict__ list, int n, const int i, const Geo& g,
                                                   const int* __restrict__ comp,
                                                   const uint32_t* __restrict__ nbm,
                                                   const int2* __restrict__ ss,
                                                   const double* __restrict__ dist,
                                                   const double4* __restrict__ site_pos,
                                                   uint32_t* __restrict__ bm,
                                                   Prop* __restrict__ imp, uint8_t* __restrict__ pf,
                                                   const PeerView* __restrict__ pv,
                                                   const BoundaryOut* bo = nullptr) {
  const bool active = i < n;
  const int v = active ? __ldg(list + i) : 0;
  int x = 0, y = 0, z = 0, cv = -3;
  unsigned nbv = 0;  // this voxel's nbm word (neighbour bits + clearance)
  double px = 0, py = 0, pz = 0;
  int ts[P2_STAB];
  double td[P2_STAB];
  int tu[P2_NTAB], tus[P2_NTAB];
  double tud[P2_NTAB];
#pragma unroll
  for (int j = 0; j < P2_STAB; j++) { ts[j] = -1; td[j] = 0.0; }
#pragma unroll
  for (int j = 0; j < P2_NTAB; j++) { tu[j] = -1; tus[j] = -1; tud[j] = 0.0; }
  double best_d = 0.0, orig_d = 0.0;
  int best_s = -1, best_src = -1, orig_s = -1;
  int own_los = -1;  // the voxel's own site when its state is LOS (src == v)
  bool done = !active;
  // No-improvement certificate: when no candidate beats the CURRENT state,
  // the reference's fold never replaces it (each step compares against the
  // running best, which stays the current state), so the voxel proposes
  // nothing -- whatever the rays would say. Every candidate distance is
  // known exactly before the fold (path rows, LOS-site and node tables); a
  // candidate outside a full table voids the certificate.
  bool cert = active;
  unsigned same = 0;  // inactive lanes run the gather with no neighbours (the warp stays converged)
  if (active) {
    bm[v >> 5] = 0u;  // consume this round's frontier word
    coords(g, v, x, y, z);
    cv = __ldg(comp + v);
    px = centre1(x, g.sx); py = centre1(y, g.sy); pz = centre1(z, g.sz);
    same = __ldg(nbm + v);
    nbv = same;
    {
      const int2 sv = __ldg(ss + v);
      best_d = __ldg(dist + v);
      best_s = sv.x; best_src = sv.y;
      orig_d = best_d; orig_s = best_s;
      // a LOS voxel's stored distance is exactly dist3(c_v, site) (every LOS
      // commit and seed computes it in this operand order): its own site's LOS
      // candidate is the current state itself and needs no table entry
      own_los = best_src == v ? orig_s : -1;
    }
  }
  {
    // ---- A: gather (two batches of 13 to bound register pressure)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      int2 nw[13];
      double dw[13];
#pragma unroll
      for (int q = 0; q < 13; q++) {
        const int k = 13 * h + q;
        const int w = v + off_dx(k) + off_dy(k) * g.nx + off_dz(k) * g.nxy;
        const bool ok = (same >> k) & 1u;
        nw[q] = ok ? __ldg(ss + w) : make_int2(-1, -1);
        dw[q] = ok ? __ldg(dist + w) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 13; q++) {
        const int k = 13 * h + q;
        const int w = v + off_dx(k) + off_dy(k) * g.nx + off_dz(k) * g.nxy;
        const bool cand = nw[q].x >= 0;
        const int s = cand ? nw[q].x : -1;
        const int u = !cand ? -1 : (nw[q].y == w ? -2 : (nw[q].y >= 0 ? nw[q].y : -1));
        const double dpath = __dadd_rn(dw[q], p2_len<DYADIC>(g, k, x, y, z, px, py, pz));
        cert = cert && !(cand && beats(dpath, s, orig_d, orig_s));
        // ---- B: distinct LOS sites and distinct shortcut nodes, branch-free set
        // inserts (at the front; entries beyond the table size are looked up on
        // the fly by the fold, and void the certificate)
        bool seen = u != -2 || s == own_los;
#pragma unroll
        for (int j = 0; j < P2_STAB; j++) seen |= ts[j] == s;
        const bool ins = !seen && ts[P2_STAB - 1] < 0;
        cert = cert && (seen || ins);
#pragma unroll
        for (int j = P2_STAB - 1; j > 0; j--) ts[j] = ins ? ts[j - 1] : ts[j];
        ts[0] = ins ? s : ts[0];
        bool useen = u < 0;
#pragma unroll
        for (int j = 0; j < P2_NTAB; j++) useen |= tu[j] == u;
        const bool uins = !useen && tu[P2_NTAB - 1] < 0;
        cert = cert && (useen || uins);
#pragma unroll
        for (int j = P2_NTAB - 1; j > 0; j--) tu[j] = uins ? tu[j - 1] : tu[j];
        tu[0] = uins ? u : tu[0];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < P2_STAB; j++) {
    if (ts[j] >= 0) {
      const double4 sp = ld_d4(site_pos + ts[j]);
      td[j] = dist3(px, py, pz, sp.x, sp.y, sp.z);
    }
  }
#pragma unroll
  for (int j = 0; j < P2_NTAB; j++) {
    const int u = tu[j];
    if (u >= 0) {
      const int2 nu = ld_ss<MG>(pv, ss, u);
      if (nu.x >= 0 && __ldg(comp + u) == cv) {
        int ux, uy, uz;
        coords(g, u, ux, uy, uz);
        tus[j] = nu.x;
        tud[j] = __dadd_rn(ld_dist<MG>(pv, dist, u), dist3(px, py, pz, centre1(ux, g.sx), centre1(uy, g.sy),
                                                   centre1(uz, g.sz)));
      }
    }
  }
#pragma unroll
  for (int j = 0; j < P2_STAB; j++) cert = cert && !(ts[j] >= 0 && beats(td[j], ts[j], orig_d, orig_s));
#pragma unroll
  for (int j = 0; j < P2_NTAB; j++) cert = cert && !(tus[j] >= 0 && beats(tud[j], tus[j], orig_d, orig_s));
  if (cert) done = true;  // the current state stands: no fold, no rays
  // ---- C: fold
  int failed = -1;
  int k = 0;
  while (!done) {
    int rs = -1, rsrc = -1;
    double rd = 0.0;
    bool los = false;
    for (; k < 26; k++) {
      // the fold runs only where the certificate failed: re-read the neighbour
      // (an L1 hit: this thread gathered it above) instead of keeping rows
      if (!((nbv >> k) & 1u)) continue;
      const char4 o = c_off[k];
      const int w = nbr_index(v, o, g.nx, g.nxy);
      const int2 nw = __ldg(ss + w);
      const int s = nw.x;
      if (s < 0) continue;
      const int u = nw.y == w ? -2 : (nw.y >= 0 ? nw.y : -1);
      const double dpath = __dadd_rn(__ldg(dist + w), p2_len<DYADIC>(g, k, x, y, z, px, py, pz));
      if (beats(dpath, s, best_d, best_s)) {
        best_d = dpath; best_s = s; best_src = w;
      }
      if (u == -2) {
        double d = 0.0;
        bool known = false;
        if (s == own_los) { d = orig_d; known = true; }  // the own LOS site: exactly the stored distance
#pragma unroll
        for (int j = 0; j < P2_STAB; j++)
          if (!known && s == ts[j]) { d = td[j]; known = true; }
        if (!known) {
          const double4 sp = ld_d4(site_pos + s);
          d = dist3(px, py, pz, sp.x, sp.y, sp.z);
        }
        if (beats(d, s, best_d, best_s) && s != failed) { rs = s; rd = d; rsrc = v; los = true; break; }
      } else if (u >= 0) {
        int su = -1;
        double d = 0.0;
        bool hit = false;
#pragma unroll
        for (int j = 0; j < P2_NTAB; j++)
          if (tu[j] == u) { su = tus[j]; d = tud[j]; hit = true; }
        if (!hit) {  // more than P2_NTAB distinct nodes (rare)
          const int2 nu = ld_ss<MG>(pv, ss, u);
          if (nu.x >= 0 && __ldg(comp + u) == cv) {
            int ux, uy, uz;
            coords(g, u, ux, uy, uz);
            su = nu.x;
            d = __dadd_rn(ld_dist<MG>(pv, dist, u), dist3(px, py, pz, centre1(ux, g.sx), centre1(uy, g.sy),
                                                  centre1(uz, g.sz)));
          }
        }
        if (su >= 0 && beats(d, su, best_d, best_s)) { rs = su; rd = d; rsrc = u; los = false; break; }
      }
    }
    if (rs < 0) { done = true; break; }
    double qx, qy, qz;
    if (los) {
      const double4 sp = ld_d4(site_pos + rs);
      qx = sp.x; qy = sp.y; qz = sp.z;
    } else {
      int ux, uy, uz;
      coords(g, rsrc, ux, uy, uz);
      qx = centre1(ux, g.sx); qy = centre1(uy, g.sy); qz = centre1(uz, g.sz);
    }
    if (ray_clear_near(nbv, qx, qy, qz, px, py, pz, g.isx, g.isy, g.isz) ||
        segment_clear_fast(comp, nbm, box_of(g), px, py, pz, qx, qy, qz, cv)) {
      best_d = rd; best_s = rs; best_src = rsrc;
    } else if (los) {
      failed = rs;
    }
    k++;
  }
  const bool improved = active && ((best_s != orig_s) || (best_d < __dsub_rn(orig_d, LRCVT_EPS)));
  // sparse proposal: slot i of this frontier item (no atomics, no block barrier)
  if (improved) {
    Prop pr;
    pr.d = best_d; pr.v = v; pr.s = best_s; pr.src = best_src; pr.pad = 0;
    imp[i] = pr;
    if (MG) emit_boundary(bo, pr);
  }
  if (active) pf[i] = improved ? 1 : 0;
}

template <int BLOCK, bool DYADIC, bool MG = false, int MINB = 512 / BLOCK>
__global__ void __launch_bounds__(BLOCK, MINB) k_eval_p2(RoundCtl* __restrict__ ctl, Geo g,
                                                                const int* __restrict__ comp,
                                                                const uint32_t* __restrict__ nbm,
                                                                const double4* __restrict__ site_pos,
                                                                uint32_t* __restrict__ bm,
                                                                Prop* __restrict__ imp, uint8_t* __restrict__ pf,
                                                                const PeerView* __restrict__ pv = nullptr) {
  const int n = ctl->n_cur;
  const int* list = ctl->cur;
  const int2* __restrict__ ss = ctl->ss;
  const double* __restrict__ dist = ctl->dist;
  // one BLOCK-voxel tile per block: the launch grid always covers the list
  // (exact grid on the host path, size-class grid >= n inside the graph)
  const int base = blockIdx.x * BLOCK;
  if (base >= n) return;
  p2_tile<BLOCK, DYADIC, MG>(list, n, base + (int)threadIdx.x, g, comp, nbm, ss, dist, site_pos, bm, imp, pf, pv, &ctl->bo);
}

}  // namespace lrcvt
