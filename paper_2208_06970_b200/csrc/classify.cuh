// classify.cuh -- restricted geodesic region growing (voronoi_classify).
//
// Maps the reference's worklist schedule (tessellation.py:102-208,
// _kernels.py:249-454) onto two launches per relaxation round:
//
//   k_eval_p1 / k_eval_p2 (eval_p1.cuh, eval_p2.cuh): one thread per frontier
//                   voxel; evaluates it against the pre-round state
//                   (_eval_voxel, _kernels.py:147-246) and appends improved
//                   proposals to a compact list;
//   k_commit        commits the proposals and enqueues the same-component
//                   26-neighbours of every improved voxel, deduplicated by a
//                   1-bit-per-voxel frontier bitmap (_apply_and_enqueue,
//                   _kernels.py:285-334);
//   the host loop   swaps the lists until the frontier drains
//                   (_run_phase, _kernels.py:337-385) and runs the phase-2
//                   verification sweeps (tessellation.py:170-189).
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

// Device-resident round control: the worklist pointers and size live in HBM
// so relaxation rounds can run back to back without the host (CUDA-graph
// conditional WHILE loop, or the host loop when per-launch timing is on).
// multi-GPU slab ranks: the eval kernels copy every improved proposal on a
// boundary plane (z == zlo for rank - 1, z == zhi - 1 for rank + 1) into
// the outgoing halo lists as they write it (lo == nullptr: one domain)
struct BoundaryOut {
  Prop* lo;
  Prop* hi;
  int* counters;  // C_LO / C_HI: list sizes
  int zlo, zhi;   // -1 / INT_MAX when there is no neighbour on that side
  int nxy;
};

struct RoundCtl {
  int* cur;          // this round's worklist
  int* nxt;          // next round's worklist (written by k_commit)
  int* stash;        // the list buffer parked during a verification sweep
  int* ro;           // a read-only list (the eligible list) while it serves as `cur`
  int* spare;        // the free list buffer that replaces `ro` when the round ends
  int2* ss;          // per-voxel (site_of, src) of the classify in flight
  double* dist;      // per-voxel distance
  int* site1;        // phase 1 only: per-voxel LOS site (site if src == self, else -1); null in phase 2
  int n_cur;         // items in cur
  int sweep_imp;     // improvements found by the last sweep
  int tile_next;     // dynamic tile scheduler of the eval kernels (reset per round)
  int loop_min;      // the round graph loops while n_cur > loop_min (small frontiers: k_rounds_small)
  long long rounds, evals, commits, rounds_p1;
  long long rounds_small, small_launches;  // rounds run inside k_rounds_small, and its launches
  BoundaryOut bo;    // multi-GPU halo output of the eval kernels
};

// Counter slots in the plan's small device array.
enum {
  C_NIMP = 0, C_NNEXT = 1, C_BAD = 2, C_ASSIGNED = 3, C_DONE = 4, C_LO = 5, C_HI = 6, C_COLL = 7, C_NPROP = 8,
  C_NCOUNTERS = 10
};
constexpr int H_NEL = 9;  // host-side slot of the pinned counter copy for the eligible count

__device__ __forceinline__ void emit_boundary(const BoundaryOut* bo, const Prop& pr) {
  if (!bo || !bo->lo) return;
  const int z = (int)((unsigned)pr.v / (unsigned)bo->nxy);
  if (z == bo->zlo) bo->lo[atomicAdd(bo->counters + C_LO, 1)] = pr;
  if (z == bo->zhi - 1) bo->hi[atomicAdd(bo->counters + C_HI, 1)] = pr;
}
constexpr int SEED_NONE = 0x7fffffff;  // k_site_voxel: the site places no seed here

// tessellation.py:120-122 fill values of the output arrays (site1, the
// phase-1 scratch, is reset over the eligible list by k_fill_list)
__global__ void k_fill_state(int2* __restrict__ ss, double* __restrict__ dist, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    ss[i] = make_int2(LRCVT_NONE, LRCVT_NONE);
    dist[i] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  }
}

// Static same-component neighbour mask: bit k set iff OFFSETS[k] of v is in
// the grid and in v's component (0 for out-of-band voxels). comp never
// changes during a tessellation, so this is built once per plan and replaces
// the 26 comp loads every evaluation and every enqueue would otherwise make.
__global__ void k_nbr_mask(Geo g, const int* __restrict__ comp, uint32_t* __restrict__ nbm) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n; i += stride) {
    const int v = (int)i;
    const int cv = comp[v];
    uint32_t m = 0;
    if (cv >= 0) {
      int x, y, z;
      coords(g, v, x, y, z);
      const unsigned inb = inbounds_mask(x, y, z, g.nx, g.ny, g.nz);
#pragma unroll
      for (int k = 0; k < 26; k++) {
        const int w = v + off_dx(k) + off_dy(k) * g.nx + off_dz(k) * g.nxy;
        if (((inb >> k) & 1u) && __ldg(comp + w) == cv) m |= 1u << k;
      }
    }
    nbm[v] = m;
  }
}

// Clearance layers (see ray_clear_by_clearance): clr = 1 where a 26-neighbour
// is foreign or outside the grid, then layer r + 1 = unknown voxels next to
// layer r (for the L-infinity metric D(v) = 1 + min over 26-neighbours),
// finally stored in nbm bits 26..31. 0 for out-of-band voxels.
constexpr unsigned char CLR_UNKNOWN = 0xFF;
constexpr int CLR_MAX = 31;
__global__ void k_clear_init(Geo g, const int* __restrict__ comp, const uint32_t* __restrict__ nbm,
                             unsigned char* __restrict__ clr) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n; i += stride) {
    const int v = (int)i;
    if (comp[v] < 0) { clr[v] = 0; continue; }
    clr[v] = (nbm[v] & ((1u << 26) - 1)) == ((1u << 26) - 1) ? CLR_UNKNOWN : 1;
  }
}
__global__ void k_clear_layer(Geo g, unsigned char* __restrict__ clr, int r) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < g.n; i += stride) {
    const int v = (int)i;
    if (clr[v] != CLR_UNKNOWN) continue;  // unknown => all 26 neighbours inside, same component
    bool hit = false;
#pragma unroll
    for (int k = 0; k < 26; k++) {
      const int w = v + off_dx(k) + off_dy(k) * g.nx + off_dz(k) * g.nxy;
      hit |= clr[w] == (unsigned char)r;
    }
    if (hit) clr[v] = (unsigned char)(r + 1);
  }
}
__global__ void k_clear_store(int64_t n, const unsigned char* __restrict__ clr, uint32_t* __restrict__ nbm) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    unsigned c = clr[i];
    if (c == CLR_UNKNOWN) c = CLR_MAX + 1;  // D > CLR_MAX: a safe lower bound
    nbm[i] = (nbm[i] & ((1u << 26) - 1)) | (c << NBM_CLR_SHIFT);
  }
}

// has_site[c] = 1 for every component that owns a site (tessellation.py:161-162:
// `comps_with_sites[site_comp] = True` on an array of max(n_components, 1)
// entries). Ids are taken with numpy's index rule -- a negative id counts
// from the end (a site of id -1 in an out-of-band voxel passes _place_seeds)
// -- and ids outside [-n, n) are never written (the reference would raise
// IndexError; such a site is also a bad site, reported by the caller).
__global__ void k_mark_site_comps(const int* __restrict__ site_comp, int n_sites, int n_slots,
                                  uint8_t* __restrict__ has_site) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sites) return;
  int c = site_comp[s];
  if (c < 0) c += n_slots;
  if (c >= 0 && c < n_slots) has_site[c] = 1;
}

// the 27-cube j = (dz+1)*9 + (dy+1)*3 + (dx+1) as (dx, dy, dz)
__constant__ char4 c_cube[27] = {
#define LRCVT_CUBE(j) {(signed char)((j) % 3 - 1), (signed char)((j) / 3 % 3 - 1), (signed char)((j) / 9 - 1), 0}
    LRCVT_CUBE(0),  LRCVT_CUBE(1),  LRCVT_CUBE(2),  LRCVT_CUBE(3),  LRCVT_CUBE(4),  LRCVT_CUBE(5),  LRCVT_CUBE(6),
    LRCVT_CUBE(7),  LRCVT_CUBE(8),  LRCVT_CUBE(9),  LRCVT_CUBE(10), LRCVT_CUBE(11), LRCVT_CUBE(12), LRCVT_CUBE(13),
    LRCVT_CUBE(14), LRCVT_CUBE(15), LRCVT_CUBE(16), LRCVT_CUBE(17), LRCVT_CUBE(18), LRCVT_CUBE(19), LRCVT_CUBE(20),
    LRCVT_CUBE(21), LRCVT_CUBE(22), LRCVT_CUBE(23), LRCVT_CUBE(24), LRCVT_CUBE(25), LRCVT_CUBE(26)
#undef LRCVT_CUBE
};

// Mark same-component neighbours of v (and v itself when `self`) in the
// frontier bitmap; newly set bits are appended to `next`. Reproduces the
// stamp-deduplicated enqueue of _kernels.py:313-333 (self=false) and
// _kernels.py:425-454 (self=true). All threads of the CTA must call it.
// The 27-cube around v is 9 x-rows of 3 voxels (dx = -1, 0, +1); a row's
// three bits sit in one bitmap word (two when they straddle a word), so
// each row costs one cached precheck load and at most one atomicOr with a
// 3-bit mask (a stale cached word only under-reports set bits, which merely
// sends that row to the atomic). newmask uses the 27-cube index
// j = (dz+1)*9 + (dy+1)*3 + (dx+1). With cbm, the word turned non-empty
// also marks its coarse bit (compact.cuh). Measured alternatives, both
// slower at 512^3: staging all 9 rows' loads, then all atomics (+45%: more
// registers, and the prechecks no longer see the bits the earlier rows'
// atomics set); grouping the lanes that want the same word (match_any) and
// setting each group's OR with one atomic (6x: match_any per row dominates).
template <bool COH = false>
__device__ __forceinline__ void mark_and_append(const Geo& g, const uint32_t* __restrict__ nbm,
                                                bool active, int v, bool self,
                                                uint32_t* __restrict__ bm,
                                                int* __restrict__ next, int* counter,
                                                int zlo = 0, int zhi = 1 << 30,
                                                uint32_t* __restrict__ cbm = nullptr) {
  unsigned newmask = 0;
  const bool slab = zlo > 0 || zhi < g.nz;
  int vz = 0;
  if (active && slab) {  // slab mode: only rows inside [zlo, zhi)
    vz = (int)((unsigned)v / (unsigned)g.nxy);
    if (vz < zlo - 1 || vz > zhi) active = false;
  }
  if (active) {
    const unsigned same = __ldg(nbm + v);
#pragma unroll
    for (int r = 0; r < 9; r++) {
      const int dy = r % 3 - 1, dz = r / 3 - 1;
      if (slab && (vz + dz < zlo || vz + dz >= zhi)) continue;
      const int j0 = 3 * r;
      unsigned want = 0;  // bit t <=> dx = t - 1
#pragma unroll
      for (int t = 0; t < 3; t++) {
        const int j = j0 + t;
        if (j == 13) {
          if (self) want |= 1u << t;
        } else {
          const int k = j < 13 ? j : j - 1;
          if ((same >> k) & 1u) want |= 1u << t;
        }
      }
      if (!want) continue;
      // anchor the window at the first wanted voxel (always inside the grid)
      const int f = __ffs(want) - 1;
      const unsigned wv = want >> f;
      const int base = v + (f - 1) + dy * g.nx + dz * g.nxy;
      const int w0 = base >> 5;
      const int sh = base & 31;
      const unsigned lo = wv << sh;                           // bits in word w0
      const unsigned hi = sh > 29 ? (wv >> (32 - sh)) : 0u;   // spill into w0 + 1
      unsigned got = 0;  // newly set by this thread, in `wv` coordinates
      if (lo) {
        const uint32_t cur = COH ? __ldcg(bm + w0) : __ldca(bm + w0);
        if ((cur & lo) != lo) {
          const uint32_t old = atomicOr(bm + w0, lo);
          got |= ((~old) & lo) >> sh;
          if (cbm && old == 0u) atomicOr(cbm + (w0 >> 10), 1u << ((w0 >> 5) & 31));  // coarse bit (compact.cuh)
        }
      }
      if (hi) {
        const uint32_t cur = COH ? __ldcg(bm + w0 + 1) : __ldca(bm + w0 + 1);
        if ((cur & hi) != hi) {
          const uint32_t old = atomicOr(bm + w0 + 1, hi);
          got |= ((~old) & hi) << (32 - sh);
          if (cbm && old == 0u) atomicOr(cbm + ((w0 + 1) >> 10), 1u << (((w0 + 1) >> 5) & 31));
        }
      }
      got <<= f;
      newmask |= got << j0;
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
  // one list reservation per CTA (a per-warp atomic on the single counter
  // serialised ~4 M same-address atomics per 512^3 iteration); every thread
  // of the CTA reaches this point the same number of times
  __shared__ int s_wbase[32];
  __shared__ int s_cbase;
  const int wid = threadIdx.x >> 5;
  if (lane == 31) s_wbase[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int sum = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
      const int t = s_wbase[w];
      s_wbase[w] = sum;
      sum += t;
    }
    s_cbase = sum ? atomicAdd(counter, sum) : 0;
  }
  __syncthreads();
  int pos = s_cbase + s_wbase[wid] + incl - cnt;
  __syncthreads();  // the next call may overwrite s_wbase / s_cbase
  while (newmask) {  // typically 0-3 new neighbours: decode each set bit through a constant table
    const int j = __ffs(newmask) - 1;
    newmask &= newmask - 1;
    const char4 o = c_cube[j];
    next[pos++] = v + o.x + o.y * g.nx + o.z * g.nxy;
  }
}

// Size classes of a round's worklist: class c covers (cap[c-1], cap[c]]
// items, caps growing 4x from 2048; the graph launches the eval kernel of the
// active class with cap[c] / BLOCK blocks (one tile per block).
constexpr int MAX_CLASSES = 12;
#ifndef LRCVT_CLASS0
#define LRCVT_CLASS0 2048  // cap of the smallest class (served by k_rounds_small)
#endif
__host__ __device__ inline long long class_cap(int c) { return (long long)LRCVT_CLASS0 << (2 * c); }

// sets exactly one class handle (none when n == 0); n_classes < 0: one SWITCH
// handle hs[0] over -n_classes bodies takes the class index (-n_classes = none)
__device__ __forceinline__ void set_size_class(long long n, const cudaGraphConditionalHandle* hs, int n_classes) {
  if (n_classes < 0) {
    const int ncl = -n_classes;
    int c = ncl;
    if (n > 0) {
      c = 0;
      while (c < ncl - 1 && n > class_cap(c)) c++;
    }
    cudaGraphSetConditional(hs[0], (unsigned)c);
    return;
  }
  for (int c = 0; c < n_classes; c++) {
    const long long lo = c == 0 ? 0 : class_cap(c - 1);
    cudaGraphSetConditional(hs[c], (n > lo && (n <= class_cap(c) || c == n_classes - 1)) ? 1u : 0u);
  }
}

// _kernels.py:285-334: commit the round's proposals, then enqueue the
// same-component neighbours of every improved voxel into the frontier bitmap
// (cleared word by word by the eval kernel that consumed it) and the next
// list. One thread per committed proposal: the compact proposal list keeps
// every lane of a warp busy in the latency-bound enqueue.
// round end (_kernels.py:370-384): statistics, list swap, next size; inside
// the round graph it also arms the next round (size-class SWITCH/IF handles and the
// WHILE condition). Runs on one thread.
__device__ __forceinline__ void round_end(RoundCtl* ctl, int* counters, const cudaGraphConditionalHandle* hs,
                                          int n_classes, cudaGraphConditionalHandle loop, int in_graph) {
  const int n_imp = counters[C_NIMP], n_next = counters[C_NNEXT];
  ctl->rounds++;
  ctl->evals += ctl->n_cur;
  ctl->commits += n_imp;
  int* t = ctl->cur;
  ctl->cur = ctl->nxt;
  ctl->nxt = t == ctl->ro ? ctl->spare : t;  // the eligible list is never written
  ctl->n_cur = n_next;
  ctl->tile_next = 0;
  counters[C_NIMP] = 0;
  counters[C_NNEXT] = 0;
  if (in_graph) {
    set_size_class(n_next, hs, n_classes);
    cudaGraphSetConditional(loop, n_next > ctl->loop_min ? 1u : 0u);
  }
}

// multi-GPU round end (host-driven rounds): swap the worklists, reset every
// per-round counter for the next eval (which therefore needs no memset) and
// hand the next frontier size and the own commit count straight to the
// host's pinned counter copy
constexpr int END_MG = 3, END_MG_SWEEP = 4;  // k_commit end modes
__device__ __forceinline__ void mg_round_end(RoundCtl* ctl, int* counters, bool sweep, volatile int* h_out) {
  const int n_next = counters[C_NNEXT];
  h_out[C_NNEXT] = n_next;
  h_out[C_NIMP] = counters[C_NIMP];
  if (sweep) {
    ctl->cur = ctl->nxt;
    ctl->nxt = ctl->stash;
  } else {
    int* t = ctl->cur;
    ctl->cur = ctl->nxt;
    ctl->nxt = t == ctl->ro ? ctl->spare : t;
  }
  ctl->n_cur = n_next;
  counters[C_NIMP] = 0;
  counters[C_NNEXT] = 0;
  counters[C_LO] = 0;
  counters[C_HI] = 0;
}

__global__ void k_loop_init(const RoundCtl* ctl, cudaGraphConditionalHandle h,
                            const cudaGraphConditionalHandle* hs, int n_classes) {
  set_size_class(ctl->n_cur, hs, n_classes);
  cudaGraphSetConditional(h, ctl->n_cur > ctl->loop_min ? 1u : 0u);
}

// phase 1 starts from the seed worklist appended to `first` by k_seed_groups
__global__ void k_phase1_start(RoundCtl* ctl, int* counters, int* first, int* second, int2* ss,
                               double* dist, int* site1, int loop_min) {
  ctl->loop_min = loop_min;
  ctl->ss = ss;
  ctl->dist = dist;
  ctl->site1 = site1;
  ctl->cur = first;
  ctl->nxt = second;
  ctl->stash = nullptr;
  ctl->ro = nullptr;
  ctl->spare = nullptr;
  ctl->n_cur = counters[C_NNEXT];
  ctl->rounds = ctl->evals = ctl->commits = ctl->rounds_p1 = 0;
  ctl->rounds_small = ctl->small_launches = 0;
  ctl->sweep_imp = 0;
  ctl->tile_next = 0;
  counters[C_NIMP] = 0;
  counters[C_NNEXT] = 0;
}

// phase 2 starts from a copy of the eligible list (tessellation.py:166-167)
// phase-1 states are LOS (src == v): (site_of, src) and dist = |c_v - p_site|
// (the very dist3 the phase-1 kernels and the seeds compute) from site1
// Over the eligible list (list != null, *n_list entries: every voxel phase 1
// can have assigned) or the voxel range [v0, v1) (list == null: the halo
// planes of a multi-GPU slab).
__global__ void k_site1_to_state(Geo g, const int* __restrict__ site1, const double4* __restrict__ site_pos,
                                 int2* __restrict__ ss, double* __restrict__ dist, const int* __restrict__ list,
                                 const int* __restrict__ n_list, int64_t v0, int64_t v1) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n = list ? (int64_t)*n_list : v1 - v0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int v = list ? __ldg(list + i) : (int)(v0 + i);
    const int s = __ldcs(site1 + v);
    if (s < 0) {  // unassigned: the fill values (phase 1 never touches ss / dist)
      __stcs(ss + v, make_int2(LRCVT_NONE, LRCVT_NONE));
      __stcs(dist + v, __longlong_as_double(0x7ff0000000000000LL));
      continue;
    }
    int x, y, z;
    coords(g, v, x, y, z);
    const double4 p = ld_d4(site_pos + s);
    __stcs(ss + v, make_int2(s, v));
    __stcs(dist + v, dist3(centre1(x, g.sx), centre1(y, g.sy), centre1(z, g.sz), p.x, p.y, p.z));
  }
}

// fill values (-1, -1) / inf / site1 -1 for the voxels of a list (*n_list
// entries); ss / dist may be null (site1 only)
__global__ void k_fill_list(const int* __restrict__ list, const int* __restrict__ n_list, int2* __restrict__ ss,
                            double* __restrict__ dist, int* __restrict__ site1) {
  const int n = *n_list;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int v = __ldg(list + i);
    if (ss) {
      ss[v] = make_int2(LRCVT_NONE, LRCVT_NONE);
      dist[v] = __longlong_as_double(0x7ff0000000000000LL);
    }
    site1[v] = LRCVT_NONE;
  }
}

// the first phase-2 round evaluates the eligible list in place (read-only:
// the round end hands the parked list buffer to the next commit instead)
__global__ void k_phase2_copy(int* __restrict__ eligible, const int* __restrict__ n_el,
                              RoundCtl* ctl, const int* __restrict__ counters) {
  // bad sites (tessellation.py:139-140 raises before any relaxation): no work
  const int n = counters[C_BAD] ? 0 : *n_el;
  ctl->spare = ctl->cur;
  ctl->cur = eligible;
  ctl->ro = eligible;
  ctl->rounds_p1 = ctl->rounds;
  ctl->site1 = nullptr;  // phase 2 commits non-LOS states; its kernels read ss
  ctl->n_cur = n;
  ctl->tile_next = 0;
}

// verification sweep over the eligible list (tessellation.py:177-189): the
// two list buffers are parked so the sweep's enqueue lands in a free one
__global__ void k_sweep_start(RoundCtl* ctl, int* eligible, const int* n_el, const int* counters) {
  ctl->stash = ctl->cur;
  ctl->cur = eligible;
  ctl->n_cur = counters[C_BAD] ? 0 : *n_el;
  ctl->tile_next = 0;
}

__global__ void k_sweep_end(RoundCtl* ctl, int* counters) {
  const int n_imp = counters[C_NIMP], n_next = counters[C_NNEXT];
  ctl->evals += ctl->n_cur;
  ctl->commits += n_imp;
  ctl->sweep_imp = n_imp;
  ctl->cur = ctl->nxt;  // the sweep's enqueue
  ctl->nxt = ctl->stash;
  ctl->n_cur = n_imp ? n_next : 0;
  ctl->tile_next = 0;
  counters[C_NIMP] = 0;
  counters[C_NNEXT] = 0;
}

// _kernels.py:399-422, site part: seed voxel, distance, validity, and the
// smallest site id per seed voxel (atomicMin on site1, which holds -1 =
// 0xffffffff on every eligible voxel here). A site recorded in component -1
// on an out-of-band voxel counts as bad here (the reference
// would seed the out-of-band region itself). Sites outside [zlo-1, zhi] (a
// multi-GPU slab and its halo planes) are still validated but place nothing.
__global__ void k_site_voxel(Geo g, const int* __restrict__ comp, const double4* __restrict__ site_pos,
                             const int* __restrict__ site_comp, int n_sites,
                             int* __restrict__ key, double* __restrict__ sd, int* __restrict__ site1,
                             int* __restrict__ counters, int zlo = 0, int zhi = 1 << 30) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_sites) return;
  const double4 p = site_pos[s];
  const int x = cell_of(p.x, g.sx, g.nx), y = cell_of(p.y, g.sy, g.ny), z = cell_of(p.z, g.sz, g.nz);
  const int v = x + g.nx * (y + g.ny * z);
  if (comp[v] != site_comp[s] || comp[v] < 0) {
    atomicAdd(counters + C_BAD, 1);
    key[s] = SEED_NONE;
    return;
  }
  if (z < zlo - 1 || z > zhi) {
    key[s] = SEED_NONE;
    return;
  }
  key[s] = v;
  sd[s] = dist3(centre1(x, g.sx), centre1(y, g.sy), centre1(z, g.sz), p.x, p.y, p.z);
  atomicMin(reinterpret_cast<unsigned*>(site1) + v, (unsigned)s);
}

// _kernels.py:399-422 contested-voxel rule + _kernels.py:425-454 initial
// worklist, without sorting the sites: the smallest site id of each seed
// voxel (k_site_voxel) places its seed and enqueues the voxel and its
// same-component neighbours; every other site of an occupied voxel goes to
// the collision list, whose groups k_seed_collisions folds afterwards in
// increasing site id exactly like the serial reference loop. The enqueued
// set does not depend on which site wins a voxel.
__global__ void __launch_bounds__(128) k_seed_groups(Geo g, const uint32_t* __restrict__ nbm,
                                                     const int* __restrict__ key,
                                                     const double* __restrict__ sd_by_site,
                                                     int n_sites, int2* __restrict__ ss,
                                                     double* __restrict__ dist, const int* __restrict__ site1,
                                                     uint32_t* __restrict__ bm,
                                                     int* __restrict__ next,
                                                     unsigned long long* __restrict__ coll,
                                                     int* __restrict__ counters,
                                                     int zlo = 0, int zhi = 1 << 30) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  // a bad site (k_site_voxel, the previous launch) aborts the classify before
  // any relaxation as the reference's ValueError does: no seeds, no frontier
  if (*(volatile int*)(counters + C_BAD)) return;
  bool head = false;
  int v = 0;
  if (s < n_sites) {
    v = key[s];
    if (v != SEED_NONE) {
      head = __ldg(site1 + v) == s;
      if (head) {
        ss[v] = make_int2(s, v);
        dist[v] = sd_by_site[s];
      } else {
        coll[atomicAdd(counters + C_COLL, 1)] = ((unsigned long long)(unsigned)v << 32) | (unsigned)s;
      }
    }
  }
  if (blockIdx.x * blockDim.x >= n_sites) return;
  mark_and_append(g, nbm, head, v, true, bm, next, counters + C_NNEXT, zlo, zhi);
}

// Voxels holding more than one site (rare: the collision list of
// k_seed_groups, every site but the smallest id of its voxel). One CTA sorts
// the (voxel, site) keys with a bitonic network in place (the buffer holds a
// power of two >= the site count) and each group's first entry folds the
// group after its smallest site, in increasing site id (_kernels.py:405-422).
constexpr int SEED_COLL_THREADS = 1024;
__global__ void __launch_bounds__(SEED_COLL_THREADS) k_seed_collisions(
    unsigned long long* __restrict__ coll, const double* __restrict__ sd_by_site, int2* __restrict__ ss,
    double* __restrict__ dist, int* __restrict__ site1, const int* __restrict__ counters) {
  const int n = *(volatile const int*)(counters + C_COLL);
  if (n == 0 || *(volatile const int*)(counters + C_BAD)) return;
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = n + threadIdx.x; i < P; i += blockDim.x) coll[i] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = coll[i], b = coll[l];
          if (((i & k) == 0) == (a > b)) {
            coll[i] = b;
            coll[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned v = (unsigned)(coll[i] >> 32);
    if (i > 0 && (unsigned)(coll[i - 1] >> 32) == v) continue;
    const int first = site1[v];
    int cur_s = first;
    double cur_d = sd_by_site[first];
    for (int j = i; j < n && (unsigned)(coll[j] >> 32) == v; j++) {
      const int s = (int)(unsigned)coll[j];
      const double d = sd_by_site[s];
      if (beats(d, s, cur_d, cur_s)) { cur_s = s; cur_d = d; }
    }
    if (cur_s != first) {
      ss[v] = make_int2(cur_s, (int)v);
      site1[v] = cur_s;
      dist[v] = cur_d;
    }
  }
}

// tessellation.py:191-194 state bits, plus the `assigned` count, over the
// eligible list (list != null, *n_list entries: no other voxel can be
// assigned; the caller zeroes the rest of `state`) or the range [v0, v1).
__global__ void k_state(const int2* __restrict__ ss, const int* __restrict__ list, const int* __restrict__ n_list,
                        int64_t v0, int64_t v1, uint8_t* __restrict__ state, int* __restrict__ counters) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n = list ? (int64_t)*n_list : v1 - v0;
  int cnt = 0;
  for (; i < n; i += stride) {
    const int v = list ? __ldg(list + i) : (int)(v0 + i);
    const int2 a = ss[v];
    uint8_t st = 0;
    if (a.x != LRCVT_NONE) {
      st = 2 | 4;
      cnt++;
      if (a.y == v) st |= 1;
    }
    if (state) state[v] = st;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(counters + C_ASSIGNED, cnt);
}

}  // namespace lrcvt
