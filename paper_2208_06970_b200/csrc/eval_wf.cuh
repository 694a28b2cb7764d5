// eval_wf.cuh -- wavefront evaluation of a frontier list (_eval_list +
// _eval_voxel, _kernels.py:147-282).
//
// Every lane runs a small state machine over a stream of frontier voxels and
// does ONE unit of work per loop iteration:
//   SCAN  examine the next in-bounds neighbour w (OFFSETS order) and fold its
//         candidates into the running best (path-through-w, LOS-to-site,
//         shortcut-to-node) exactly as the reference does;
//   RAY   one DDA cell of a pending line-of-sight test (_kernels.py:45-125);
// and a lane that finishes a voxel immediately fetches the next list item
// (warp-aggregated atomic). Lanes therefore stay busy and converged on one
// short loop body instead of replaying a 26-way scan per ray generation, and
// a ray costs its cell count in iterations, interleaved with other lanes'
// scans, instead of serialising the warp.
//
// Per voxel the decision sequence is the reference's: a ray is cast exactly
// when the candidate beats the running best (and, for LOS, is not the memoised
// failed site); its result is applied before the next neighbour is examined.
#pragma once
#include "classify.cuh"

namespace lrcvt {

enum { C_WORK = 4 };

template <bool PHASE2, bool DYADIC>
__global__ void __launch_bounds__(128) k_eval_wf(const int* __restrict__ list, int n, Geo g,
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
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;

  // ---- per-lane voxel state
  bool has = false, ray = false;
  int v = 0, x = 0, y = 0, z = 0, cv = 0;
  double px = 0, py = 0, pz = 0;
  double best_d = 0, orig_d = 0, thr = 0;
  int best_s = -1, best_src = -1, orig_s = -1, failed_site = -1;
  int cache_s = -1, cache_u = -1;
  double cache_d = 0, cache_ud = 0;
  unsigned rem = 0;
  // pending candidate (applied if the ray is clear)
  double rd = 0;
  int rs = 0, rsrc = 0;
  bool ray_los = false;
  // DDA state
  int cx = 0, cy = 0, cz = 0, ex = 0, ey = 0, ez = 0, steps = 0, sgn = 0;
  double tmx = 0, tmy = 0, tmz = 0, tdx = 0, tdy = 0, tdz = 0;
  bool exhausted = false;

  for (;;) {
    // ---- refill idle lanes (warp-aggregated fetch of list items)
    const unsigned need = __ballot_sync(FULL, !has);
    if (need && !exhausted) {
      const int leader = __ffs(need) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(counters + C_WORK, __popc(need));
      base = __shfl_sync(FULL, base, leader);
      if (base + __popc(need) >= n) exhausted = true;
      if (!has) {
        const int idx = base + __popc(need & lt_mask);
        if (idx < n) {
          v = __ldg(list + idx);
          bm[v >> 5] = 0u;  // consume the frontier bit word of this voxel
          coords(g, v, x, y, z);
          cv = __ldg(comp + v);
          px = centre1(x, g.sx); py = centre1(y, g.sy); pz = centre1(z, g.sz);
          const int2 sv = ss[v];
          best_d = dist[v];
          best_s = sv.x; best_src = sv.y;
          orig_d = best_d; orig_s = best_s;
          failed_site = -1; cache_s = -1; cache_u = -1;
          thr = beat_threshold(best_d);
          rem = inbounds_mask(x, y, z, g.nx, g.ny, g.nz);
          has = true; ray = false;
        }
      }
    }
    if (!__any_sync(FULL, has)) break;

    bool fin = false;
    if (has) {
      if (!ray) {
        // ---------------- SCAN one neighbour
        if (rem == 0) {
          fin = true;
        } else {
          const char4 o = c_off[__ffs(rem) - 1];
          rem &= rem - 1;
          const int w = nbr_index(v, o, g.nx, g.nxy);
          const int2 nw = ss[w];
          const int cw = __ldg(comp + w);
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
              const double d = __dadd_rn(dist[w], len);
              if (beats(d, sw, best_d, best_s)) {
                best_d = d; best_s = sw; best_src = w; thr = beat_threshold(best_d);
              }
            }
            const int u = nw.y;
            double qx = 0, qy = 0, qz = 0;
            if (u == w) {
              // LOS: w sees its site; d is a pure function of (v, site)
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
                ray = true; ray_los = true; rd = d; rs = sw; rsrc = v;
                qx = sp.x; qy = sp.y; qz = sp.z;
              }
            } else if (PHASE2 && u >= 0) {
              // shortcut to w's node u; d = RN(du + |p - c_u|) >= du
              const double du = dist[u];
              if (du < thr) {
                const int2 nu = ss[u];
                if (nu.x >= 0 && __ldg(comp + u) == cv) {
                  int ux, uy, uz;
                  coords(g, u, ux, uy, uz);
                  qx = centre1(ux, g.sx); qy = centre1(uy, g.sy); qz = centre1(uz, g.sz);
                  double d;
                  if (u == cache_u) {
                    d = cache_ud;
                  } else {
                    d = __dadd_rn(du, dist3(px, py, pz, qx, qy, qz));
                    cache_u = u; cache_ud = d;
                  }
                  if (beats(d, nu.x, best_d, best_s)) {
                    ray = true; ray_los = false; rd = d; rs = nu.x; rsrc = u;
                  }
                }
              }
            }
            if (ray) {
              // ---- DDA set-up, _kernels.py:54-101 (start cell is v's own)
              cx = cell_of(px, g.sx, g.nx); cy = cell_of(py, g.sy, g.ny); cz = cell_of(pz, g.sz, g.nz);
              ex = cell_of(qx, g.sx, g.nx); ey = cell_of(qy, g.sy, g.ny); ez = cell_of(qz, g.sz, g.nz);
              const double ddx = __dsub_rn(qx, px), ddy = __dsub_rn(qy, py), ddz = __dsub_rn(qz, pz);
              sgn = (ddx > 0 ? 1 : 0) | (ddy > 0 ? 2 : 0) | (ddz > 0 ? 4 : 0);
              const double big = 1e30;
              if (ddx != 0.0) {
                const double nxt = ddx > 0 ? __dmul_rn((double)(cx + 1), g.sx) : __dmul_rn((double)cx, g.sx);
                tmx = __ddiv_rn(__dsub_rn(nxt, px), ddx); tdx = __ddiv_rn(g.sx, fabs(ddx));
              } else { tmx = big; tdx = big; }
              if (ddy != 0.0) {
                const double nxt = ddy > 0 ? __dmul_rn((double)(cy + 1), g.sy) : __dmul_rn((double)cy, g.sy);
                tmy = __ddiv_rn(__dsub_rn(nxt, py), ddy); tdy = __ddiv_rn(g.sy, fabs(ddy));
              } else { tmy = big; tdy = big; }
              if (ddz != 0.0) {
                const double nxt = ddz > 0 ? __dmul_rn((double)(cz + 1), g.sz) : __dmul_rn((double)cz, g.sz);
                tmz = __ddiv_rn(__dsub_rn(nxt, pz), ddz); tdz = __ddiv_rn(g.sz, fabs(ddz));
              } else { tmz = big; tdz = big; }
              steps = abs(ex - cx) + abs(ey - cy) + abs(ez - cz) + 8;
              // start cell foreign -> t = 0 (never for v's own cell, kept exact)
              if (__ldg(comp + cx + g.nx * (cy + g.ny * cz)) != cv) {
                ray = false;
                if (ray_los) failed_site = rs;
              }
            }
          }
        }
      } else {
        // ---------------- RAY: one DDA cell
        int res = 0;  // 0 = continue, 1 = clear, 2 = blocked
        if (steps <= 0) {
          res = 1;
        } else if (cx == ex && cy == ey && cz == ez) {
          res = 1;
        } else {
          const double t = fmin(tmx, fmin(tmy, tmz));
          if (t > 1.0) {
            res = __ldg(comp + ex + g.nx * (ey + g.ny * ez)) == cv ? 1 : 2;
          } else {
            if (tmx == t) { cx += (sgn & 1) ? 1 : -1; tmx = __dadd_rn(tmx, tdx); }
            if (tmy == t) { cy += (sgn & 2) ? 1 : -1; tmy = __dadd_rn(tmy, tdy); }
            if (tmz == t) { cz += (sgn & 4) ? 1 : -1; tmz = __dadd_rn(tmz, tdz); }
            if (cx < 0 || cy < 0 || cz < 0 || cx >= g.nx || cy >= g.ny || cz >= g.nz ||
                __ldg(comp + cx + g.nx * (cy + g.ny * cz)) != cv) {
              res = t >= 1.0 ? 1 : 2;
            }
            steps--;
          }
        }
        if (res) {
          ray = false;
          if (res == 1) {
            best_d = rd; best_s = rs; best_src = rsrc; thr = beat_threshold(best_d);
          } else if (ray_los) {
            failed_site = rs;
          }
        }
      }
    }
    // ---- retire finished voxels; append improved proposals
    bool improved = false;
    if (fin) {
      has = false;
      improved = (best_s != orig_s) || (best_d < __dsub_rn(orig_d, LRCVT_EPS));
    }
    const unsigned mi = __ballot_sync(FULL, improved);
    if (mi) {
      const int leader = __ffs(mi) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(counters + C_NIMP, __popc(mi));
      base = __shfl_sync(FULL, base, leader);
      if (improved) {
        Prop pr;
        pr.d = best_d; pr.v = v; pr.s = best_s; pr.src = best_src; pr.pad = 0;
        imp[base + __popc(mi & lt_mask)] = pr;
      }
    }
  }
}

}  // namespace lrcvt
