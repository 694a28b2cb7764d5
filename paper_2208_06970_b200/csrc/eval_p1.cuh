// eval_p1.cuh -- phase-1 evaluation (_eval_voxel with phase2 = False,
// _kernels.py:147-246; tessellation.py:151-156).
//
// Phase 1 only admits line-of-sight candidates, so the per-neighbour work is
// a site id, a distance that depends only on (voxel, site) and a `_beats`
// test; rays are the only expensive step. The kernel gathers, tabulates and
// folds instead of walking neighbours with dependent loads (see below).
#pragma once
#include "classify.cuh"

namespace lrcvt {

#ifndef LRCVT_P1_TAB
#define LRCVT_P1_TAB 3
#endif
constexpr int P1_TAB = LRCVT_P1_TAB;  // distinct-site distance table
#ifndef LRCVT_P1_GATHER
#define LRCVT_P1_GATHER 13
#endif
constexpr int P1_GATHER = LRCVT_P1_GATHER;  // neighbour loads in flight per batch (13 or 26)
static_assert(26 % P1_GATHER == 0, "P1_GATHER divides 26");

// Phase-1 evaluation (LOS candidates only):
//   A  gather the 26 neighbours' LOS sites from the compact site1 array
//      (immediate offsets, all loads in flight) into a per-thread
//      shared-memory row;
//   B  compute the distance to each distinct neighbour site once;
//   C  strict-order rule: when no two distinct elements of
//      {current state} + table are within the EPS tie band, the reference's
//      fold ends at the minimum-distance element whose ray is clear, so only
//      the winner's ray is needed: proven clear by the voxel's clearance, or
//      queued per warp and D traced by the warp one ray per lane;
//   E  a blocked winner, a near-tie or a table overflow takes the exact
//      sequential fold in OFFSETS order with rays traced inline (rare once
//      sites have left voxel centres).
// Ray outcomes are pure functions of (voxel, site), so the decision sequence
// is exactly the reference's in every case. (A speculative fold that queued
// up to three rays per lane preceded the strict rule; with the rule in place
// it only cost registers and spills and was removed: p1 -7% at 512^3.)
constexpr int P1_SPEC = 1;  // queued rays per lane (the strict winner's)
// CTAs per SM the register budget is sized for: 5 (102 registers) for rounds
// below a million voxels; 8 (64 registers: more spills, but twice the warps
// to hide the dependent gathers) for larger ones. Measured on phase-1 time:
// 512^3 -10% and 256^3 -5% with 8 for the large rounds (6, 7, 10 in between
// or equal, 12 worse); 128^3 rounds stay below the threshold (5 is 2% faster there).
#ifndef LRCVT_P1_MINB_SMALL
#define LRCVT_P1_MINB_SMALL 5
#endif
constexpr int P1_MIN_BLOCKS = LRCVT_P1_MINB_SMALL;
constexpr int P1_MIN_BLOCKS_BIG = 8;
constexpr int P1_BIG_ROUND = 1 << 20;

template <int BLOCK>
__device__ __forceinline__ void p1_tile(const int* __restrict__ list, int n, const int i, const Geo& g,
                                                   const int* __restrict__ comp,
                                                   const uint32_t* __restrict__ nbm,
                                                   const int* __restrict__ site1,
                                                   const double* __restrict__ dist,
                                                   const double4* __restrict__ site_pos,
                                                   uint32_t* __restrict__ bm,
                                                   Prop* __restrict__ imp, uint8_t* __restrict__ pf,
                                                   const BoundaryOut* bo = nullptr) {
  // per-warp queue of speculated rays (no block-wide barrier needed)
  __shared__ int q_v[BLOCK * P1_SPEC], q_s[BLOCK * P1_SPEC];
  __shared__ unsigned char q_ok[BLOCK * P1_SPEC];
  __shared__ int q_n[BLOCK / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int* qv = q_v + wid * 32 * P1_SPEC;
  int* qs = q_s + wid * 32 * P1_SPEC;
  unsigned char* qok = q_ok + wid * 32 * P1_SPEC;
  if (lane == 0) q_n[wid] = 0;
  const bool active = i < n;
  const int v = active ? __ldg(list + i) : 0;
  int x = 0, y = 0, z = 0, cv = -3;
  unsigned nbv = 0;  // this voxel's nbm word (neighbour bits + clearance)
  bool ovf = false;  // more distinct neighbour sites than the table holds
  double px = 0, py = 0, pz = 0;
  int ts[P1_TAB];
  double td[P1_TAB];
#pragma unroll
  for (int j = 0; j < P1_TAB; j++) { ts[j] = -1; td[j] = 0.0; }
  double best_d = 0.0, orig_d = 0.0;
  int best_s = -1, best_src = -1, orig_s = -1;
  unsigned same = 0;  // inactive lanes gather nothing (the warp stays converged for the votes below)
  if (active) {
    bm[v >> 5] = 0u;  // consume this round's frontier word
    coords(g, v, x, y, z);
    cv = __ldg(comp + v);
    px = centre1(x, g.sx); py = centre1(y, g.sy); pz = centre1(z, g.sz);
    same = __ldg(nbm + v);
    nbv = same;
    // phase-1 states are LOS (src == v) and their distance is |c_v - p_site|
    orig_s = __ldg(site1 + v);
  }
  {
    // ---- A
    // phase 1: site1[w] is site_of[w] when src[w] == w (every phase-1 assignment), else -1
    // two batches of 13 loads in flight (bounds the live registers of the
    // big-round variant, whose 64-register budget otherwise spills)
#pragma unroll
    for (int h = 0; h < 26 / P1_GATHER; h++) {
    int nw[P1_GATHER];
#pragma unroll
    for (int q = 0; q < P1_GATHER; q++) {
      const int k = P1_GATHER * h + q;
      const int w = v + off_dx(k) + off_dy(k) * g.nx + off_dz(k) * g.nxy;
      nw[q] = ((same >> k) & 1u) ? __ldg(site1 + w) : -1;
    }
#pragma unroll
    for (int q = 0; q < P1_GATHER; q++) {
      const int k = P1_GATHER * h + q;
      const int s = nw[q];
      // ---- B: distinct-site table; the voxel's own site is not entered: its
      // (skipping a batch's inserts when no lane of the warp sees a foreign
      // site, and whole warps without candidates, measured 4.5 % slower at C4)
      // candidate (orig_d, orig_s, v) is the current state itself
      bool seen = s < 0 || s == orig_s;
#pragma unroll
      for (int j = 0; j < P1_TAB; j++) seen |= ts[j] == s;
      // branch-free insert at the front (the table is a set); a fifth site overflows
      const bool ins = !seen;
      ovf |= ins && ts[P1_TAB - 1] >= 0;
#pragma unroll
      for (int j = P1_TAB - 1; j > 0; j--) ts[j] = ins ? ts[j - 1] : ts[j];
      ts[0] = ins ? s : ts[0];
    }
    }
  }
  if (active) {
    best_s = orig_s; best_src = v;
    if (best_s >= 0) {
      const double4 sp = ld_d4(site_pos + best_s);
      best_d = dist3(px, py, pz, sp.x, sp.y, sp.z);
    } else {
      best_d = __longlong_as_double(0x7ff0000000000000LL);
    }
    orig_d = best_d; orig_s = best_s;
  }
#pragma unroll
  for (int j = 0; j < P1_TAB; j++) {
    if (ts[j] >= 0) {
      const double4 sp = ld_d4(site_pos + ts[j]);
      td[j] = dist3(px, py, pz, sp.x, sp.y, sp.z);
    }
  }
  // ---- strict-order fast path. When every two distinct (distance, site)
  // elements among the current state and the table differ in distance by
  // more than 2.5e-9 + |d|*1e-15, `_beats` between them is decided by the
  // distance alone (neither of its EPS tie clauses can fire) and is a strict
  // order, so the reference's sequential fold ends at the minimum-distance
  // element among {current} and the LOS candidates whose ray is clear:
  // repeated sites are no-ops, failed_site only skips rays that would fail
  // again, and a clear candidate of smaller distance than the running best
  // always beats it. Only the winner's ray is needed; if it is blocked the
  // lane takes the exact non-speculative fold below.
  bool strict = false;
  int jwin = -1;
  if (active && !ovf) {
    strict = true;
#pragma unroll
    for (int a = 0; a <= P1_TAB; a++) {
#pragma unroll
      for (int b = a + 1; b <= P1_TAB; b++) {
        const bool va = a == 0 || ts[a - 1] >= 0, vb = ts[b - 1] >= 0;
        const double da = a == 0 ? orig_d : td[a - 1], db = td[b - 1];
        const int sa = a == 0 ? orig_s : ts[a - 1], sb = ts[b - 1];
        if (va && vb && !(da == db && sa == sb)) {
          const bool ia = isinf(da), ib = isinf(db);
          const double tol = __dadd_rn(2.5e-9, __dmul_rn(fmax(fabs(da), fabs(db)), 1e-15));
          if (!((ia != ib) || (!ia && fabs(__dsub_rn(da, db)) > tol))) strict = false;
        }
      }
    }
    if (strict) {
      double dmin = orig_d;
#pragma unroll
      for (int j = 0; j < P1_TAB; j++)
        if (ts[j] >= 0 && td[j] < dmin) { dmin = td[j]; jwin = j; }
    }
  }
  __syncwarp();  // q_n initialised
  const float isx = g.isx, isy = g.isy, isz = g.isz;
  int win_slot = -1;   // queue slot of the strict winner's ray (-1: none or proven clear)
  int win_s = -1;
  double win_d = 0.0;
  if (jwin >= 0) {
#pragma unroll
    for (int j = 0; j < P1_TAB; j++)
      if (j == jwin) { win_s = ts[j]; win_d = td[j]; }
    const double4 sp = ld_d4(site_pos + win_s);
    if (!ray_clear_near(nbv, sp.x, sp.y, sp.z, px, py, pz, isx, isy, isz)) {
      win_slot = atomicAdd(&q_n[wid], 1);
      qv[win_slot] = v; qs[win_slot] = win_s;
    }
  }
  // lanes without a strict order (near-ties: rare once sites have moved off
  // voxel centres) take the exact fold below with rays traced inline
  int failed = -1;
  __syncwarp();
  // ---- D: the warp traces its queued rays, one per lane
  const int nq = q_n[wid];
  for (int j = lane; j < nq; j += 32) {
    const int rv = qv[j];
    int rx, ry, rz;
    coords(g, rv, rx, ry, rz);
    const double4 sp = ld_d4(site_pos + qs[j]);
    const double cx = centre1(rx, g.sx), cy = centre1(ry, g.sy), cz = centre1(rz, g.sz);
    qok[j] = ray_clear_near(__ldg(nbm + rv), sp.x, sp.y, sp.z, cx, cy, cz, isx, isy, isz) ||
                     segment_clear_fast(comp, nbm, box_of(g), cx, cy, cz, sp.x, sp.y, sp.z, __ldg(comp + rv))
                 ? 1 : 0;
  }
  __syncwarp();
  // ---- E: strict lanes take their winner (or fall back to the exact fold)
  int kres = 26;  // start of the exact sequential fold (26: not needed)
  if (active && strict) {
    if (jwin >= 0 && (win_slot < 0 || qok[win_slot])) {
      best_d = win_d; best_s = win_s; best_src = v;
    } else if (jwin >= 0) {
      kres = 0;  // winner blocked: exact fold from the start (best = current state)
    }
  } else if (active) {
    kres = 0;
  }
  if (active) {
    for (int k = kres; k < 26; k++) {
      // the exact fold is rare: re-read the neighbour's site (an L1 hit) instead of keeping rows
      if (!((nbv >> k) & 1u)) continue;
      const int s = __ldg(site1 + v + off_dx(k) + off_dy(k) * g.nx + off_dz(k) * g.nxy);
      if (s < 0) continue;
      double d = 0.0;
      bool known = false;
      if (s == orig_s) { d = orig_d; known = true; }  // the own site: the very dist3 of the current state
#pragma unroll
      for (int j = 0; j < P1_TAB; j++)
        if (!known && s == ts[j]) { d = td[j]; known = true; }
      if (!known) {
        const double4 sp = ld_d4(site_pos + s);
        d = dist3(px, py, pz, sp.x, sp.y, sp.z);
      }
      if (beats(d, s, best_d, best_s) && s != failed) {
        const double4 sp = ld_d4(site_pos + s);
        if (ray_clear_near(nbv, sp.x, sp.y, sp.z, px, py, pz, isx, isy, isz) ||
            segment_clear_fast(comp, nbm, box_of(g), px, py, pz, sp.x, sp.y, sp.z, cv)) {
          best_d = d; best_s = s; best_src = v;
        } else {
          failed = s;
        }
      }
    }
  }
  const bool improved = active && ((best_s != orig_s) || (best_d < __dsub_rn(orig_d, LRCVT_EPS)));
  // sparse proposal: slot i of this frontier item (no atomics, no block barrier)
  if (improved) {
    Prop pr;
    pr.d = best_d; pr.v = v; pr.s = best_s; pr.src = best_src; pr.pad = 0;
    imp[i] = pr;
    emit_boundary(bo, pr);
  }
  if (active) pf[i] = improved ? 1 : 0;
}

// Grid-stride over 128-voxel tiles of the worklist held in the round control
// block (size and pointer read on device, so rounds need no host round trip).
template <int BLOCK, int MINB = P1_MIN_BLOCKS>
__global__ void __launch_bounds__(BLOCK, MINB) k_eval_p1(RoundCtl* __restrict__ ctl, Geo g,
                                                   const int* __restrict__ comp,
                                                   const uint32_t* __restrict__ nbm,
                                                   const double4* __restrict__ site_pos,
                                                   uint32_t* __restrict__ bm,
                                                   Prop* __restrict__ imp, uint8_t* __restrict__ pf) {
  const int n = ctl->n_cur;
  const int* list = ctl->cur;
  const int* __restrict__ site1 = ctl->site1;
  const double* __restrict__ dist = ctl->dist;
  // one BLOCK-voxel tile per block: the launch grid always covers the list
  // (exact grid on the host path, size-class grid >= n inside the graph)
  const int base = blockIdx.x * BLOCK;
  if (base >= n) return;
  p1_tile<BLOCK>(list, n, base + (int)threadIdx.x, g, comp, nbm, site1, dist, site_pos, bm, imp, pf, &ctl->bo);
}

}  // namespace lrcvt
