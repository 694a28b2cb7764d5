// mg.cuh -- multi-GPU global mode: z-slab ownership and peer reads
// (SURVEY.md §8(e) "global mode").
//
// Rank r owns planes [zb[r], zb[r+1]) of ONE volume. Every rank keeps
// full-size per-voxel buffers, but only its own slab plus one halo plane on
// each side is kept current locally (the halo through the boundary proposals
// its neighbours forward each round). The static volumes (comp, nbm) are
// replicated. The only reads that may leave [lo, hi] are the far reads of the
// phase-2 shortcut candidates (state of u = src(w), _kernels.py:221-243) and
// the phi chains of the vote (_kernels.py:466-481); they go to the owner's
// pre-round buffer through a peer pointer (NVLink P2P / CUDA IPC mapping on
// separate GPUs, the other rank's buffer when the ranks share a device).
#pragma once
#include "common.cuh"

namespace lrcvt {

constexpr int MG_MAX = 8;

struct PeerView {
  const int2* ss[MG_MAX];       // each rank's (site_of, src) buffer, full-volume layout
  const double* dist[MG_MAX];   // each rank's distance buffer
  int zb[MG_MAX + 1];           // rank r owns planes [zb[r], zb[r + 1])
  int world;
  int lo, hi;                   // planes readable locally: [lo, hi] (own slab +- halo)
  int nxy;
};

__device__ __forceinline__ int pv_owner(const PeerView& pv, int z) {
  int r = 0;
#pragma unroll
  for (int k = 1; k < MG_MAX; k++) r += (k < pv.world && z >= pv.zb[k]) ? 1 : 0;
  return r;
}

// state of voxel u: the local buffer inside [lo, hi], else the owner's
// (L2-coherent loads: the owner's buffer is written between rounds)
template <bool MG>
__device__ __forceinline__ int2 ld_ss(const PeerView* pv, const int2* __restrict__ ss, int u) {
  if (MG) {
    const int z = (int)((unsigned)u / (unsigned)pv->nxy);
    if (z < pv->lo || z > pv->hi) return __ldcg(pv->ss[pv_owner(*pv, z)] + u);
  }
  return __ldg(ss + u);
}
template <bool MG>
__device__ __forceinline__ double ld_dist(const PeerView* pv, const double* __restrict__ dist, int u) {
  if (MG) {
    const int z = (int)((unsigned)u / (unsigned)pv->nxy);
    if (z < pv->lo || z > pv->hi) return __ldcg(pv->dist[pv_owner(*pv, z)] + u);
  }
  return __ldg(dist + u);
}

// first LOS ancestor with peer reads along the chain (_kernels.py:473-481)
template <bool MG>
__device__ __forceinline__ int phi_chase_pv(const PeerView* pv, const int2* __restrict__ ss, int v, int2 a) {
  int u = v;
  while (a.y != u && a.y >= 0) {
    u = a.y;
    a = MG ? ld_ss<true>(pv, ss, u) : ss[u];
  }
  return u;
}

}  // namespace lrcvt
