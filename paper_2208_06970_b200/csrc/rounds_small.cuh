// rounds_small.cuh -- every relaxation round of a small frontier inside ONE
// persistent cooperative kernel (_kernels.py:337-385 round loop).
//
// A round whose frontier holds a few hundred to two thousand voxels costs
// far more in launch latency and inter-kernel drain than in work (2D bands
// and the tail of every classify run dozens of such rounds). Here each round
// is: warp-per-voxel evaluation (eval_warp.cuh) -> grid barrier -> commit +
// enqueue (classify.cuh) -> grid barrier -> round end by one thread -> grid
// barrier. The same proposals, commits and schedule as the launched kernels;
// per-round state written by other SMs is read through L2 (ldcg), never
// through a possibly stale L1 line. The kernel returns as soon as the
// frontier is empty or grows past `small` (the graph's size-class rounds
// then continue).
#pragma once
#include <cooperative_groups.h>

#include "eval_warp.cuh"

namespace lrcvt {

template <bool PHASE2>
__global__ void __launch_bounds__(32 * EW_WARPS) k_rounds_small(RoundCtl* __restrict__ ctl, Geo g,
                                                                const int* __restrict__ comp,
                                                                const uint32_t* __restrict__ nbm,
                                                                const double4* __restrict__ site_pos,
                                                                uint32_t* __restrict__ bm, Prop* __restrict__ imp,
                                                                uint8_t* __restrict__ pf,
                                                                int* __restrict__ counters, int small,
                                                                int max_rounds,
                                                                const cudaGraphConditionalHandle* hs, int n_classes,
                                                                cudaGraphConditionalHandle loop, int in_graph) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ EwStage stage[EW_WARPS];
  const int wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * EW_WARPS + wid, n_warps = gridDim.x * EW_WARPS;
  volatile RoundCtl* vctl = ctl;
  for (int r = 0; r < max_rounds; ++r) {
    const int n = vctl->n_cur;  // uniform: written before the last barrier
    if (n <= 0 || n > small) break;
    const int* list = vctl->cur;
    const int2* ss = vctl->ss;
    const int* site1 = vctl->site1;
    const double* dist = vctl->dist;
    for (int i = gw; i < n; i += n_warps)
      ew_voxel<PHASE2, true>(list, ss, site1, dist, i, g, comp, nbm, site_pos, bm, imp, pf, stage[wid]);
    grid.sync();
    // commit (k_commit's body over the sparse proposal slots): one thread per
    // frontier item, block-uniform trip count
    int* next = vctl->nxt;
    int2* wss = vctl->ss;
    double* wdist = vctl->dist;
    int* wsite1 = vctl->site1;
    int mine = 0;
    for (int base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
      const int i = base + threadIdx.x;
      const bool active = i < n && __ldcg(pf + i);  // written this round by other SMs
      int v = 0;
      if (active) {
        Prop p;
        {
          const double pd = __ldcg(&imp[i].d);
          const int2 a = __ldcg(reinterpret_cast<const int2*>(&imp[i].v));
          const int2 b = __ldcg(reinterpret_cast<const int2*>(&imp[i].src));
          p.d = pd; p.v = a.x; p.s = a.y; p.src = b.x; p.pad = b.y;
        }
        v = p.v;
        mine++;
        if (wsite1) {
          __stcg(wsite1 + v, p.src == p.v ? p.s : (int)LRCVT_NONE);
        } else {
          __stcg(wss + v, make_int2(p.s, p.src));
          __stcg(wdist + v, p.d);
        }
      }
      mark_and_append<true>(g, nbm, active, v, false, bm, next, counters + C_NNEXT);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(counters + C_NIMP, mine);
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // round_end with coherent (volatile) accesses
      volatile int* vc = counters;
      const int n_imp_all = vc[C_NIMP], n_next = vc[C_NNEXT];
      vctl->rounds = vctl->rounds + 1;
      vctl->rounds_small = vctl->rounds_small + 1;
      vctl->evals = vctl->evals + vctl->n_cur;
      vctl->commits = vctl->commits + n_imp_all;
      int* t = vctl->cur;
      vctl->cur = vctl->nxt;
      vctl->nxt = t == vctl->ro ? vctl->spare : t;
      vctl->n_cur = n_next;
      vctl->tile_next = 0;
      vc[C_NIMP] = 0;
      vc[C_NNEXT] = 0;
      __threadfence();
    }
    grid.sync();
  }
  // inside the round graph: arm the next size class and the WHILE condition
  // (the frontier is empty, or too large for this kernel)
  if (blockIdx.x == 0 && threadIdx.x == 0) vctl->small_launches = vctl->small_launches + 1;
  if (in_graph && blockIdx.x == 0 && threadIdx.x == 0) {
    const int n = vctl->n_cur;
    set_size_class(n, hs, n_classes);
    cudaGraphSetConditional(loop, n > 0 ? 1u : 0u);
  }
}

}  // namespace lrcvt
