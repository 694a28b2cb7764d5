// compact.cuh -- commit + enqueue of a relaxation round, and the optional
// voxel-order rebuild of large frontiers.
//
// _apply_and_enqueue (_kernels.py:313-333) enqueues the same-component
// 26-neighbours of every improved voxel, deduplicated by `stamp`. The set is
// all that matters (each round reads only pre-round state), so the order of
// the list is ours to choose. k_commit commits the round's proposals and
// appends the newly marked neighbours (frontier bitmap dedup,
// mark_and_append); with LRCVT_COMPACT=1 it also marks a coarse bitmap (1 bit
// per 32 words = 1024 voxels) and k_reorder rewrites every frontier of at
// least REORDER_MIN voxels IN VOXEL ORDER from the bitmap: one single-pass
// scan over the marked chunks (decoupled look-back over tiles of 2048 words),
// warp-cooperative coalesced output. A voxel-ordered list puts neighbouring
// voxels in neighbouring lanes, so the eval kernels' 26-neighbour gathers
// and ray walks hit L1/L2 more often (measured at 512^3: ~50 instead of ~150
// bytes of DRAM per evaluation).
#pragma once
#include "classify.cuh"

namespace lrcvt {

constexpr int CT_THREADS = 256;
constexpr int CT_WPT = 8;                          // bitmap words per thread
constexpr int CT_WORDS = CT_THREADS * CT_WPT;      // words per tile (65536 voxels)
constexpr int CT_CHUNK = 32;                       // words per coarse bit
constexpr int CT_CWORDS = CT_WORDS / CT_CHUNK / 32;  // coarse words per tile (2)

// persistent compaction state (zeroed once per plan): [0] epoch, [1] dynamic
// tile counter, [2] finished-CTA counter
enum { CS_EPOCH = 0, CS_TILE = 1, CS_DONE = 2, CS_N = 4 };

__host__ __device__ inline int64_t compact_tiles(int64_t bm_words) { return (bm_words + CT_WORDS - 1) / CT_WORDS; }
__host__ __device__ inline int64_t coarse_words(int64_t bm_words) {
  return compact_tiles(bm_words) * CT_CWORDS;  // whole tiles: no bounds checks on the coarse reads
}

#ifndef LRCVT_CM_THREADS
#define LRCVT_CM_THREADS 512
#endif
constexpr int CM_THREADS = LRCVT_CM_THREADS;
constexpr int CM_SLOTS = 4 * CM_THREADS;  // sparse slots scanned per CTA step

__device__ __forceinline__ void commit_one(const Prop& p, int2* __restrict__ ss, double* __restrict__ dist,
                                           int* __restrict__ site1) {
  // ss and dist are rebuilt from site1 once when phase 2 starts
  // (k_site1_to_state): phase 1 keeps only the compact LOS site, whose
  // distance is a pure function of (voxel, site)
  if (site1) {
    __stcg(site1 + p.v, p.src == p.v ? p.s : (int)LRCVT_NONE);
  } else {
    __stcg(ss + p.v, make_int2(p.s, p.src));
    __stcg(dist + p.v, p.d);
  }
}

__global__ void __launch_bounds__(CM_THREADS, 2048 / CM_THREADS) k_commit(const Prop* __restrict__ imp, const uint8_t* __restrict__ pf,
                                                       int n_props, int* __restrict__ counters,
                                                       RoundCtl* __restrict__ ctl, Geo g,
                                                       const uint32_t* __restrict__ nbm, uint32_t* __restrict__ bm,
                                                       uint32_t* __restrict__ cbm,
                                                       const cudaGraphConditionalHandle* __restrict__ hs,
                                                       int n_classes, cudaGraphConditionalHandle loop, int end_mode,
                                                       int zlo, int zhi, const Prop* __restrict__ halo = nullptr,
                                                       int n_halo = 0, int own_blocks = 1 << 30,
                                                       volatile int* h_out = nullptr) {
  __shared__ int s_idx[CM_SLOTS];
  __shared__ int s_wcnt[CM_THREADS / 32];
  __shared__ int s_tot;
  int2* __restrict__ ss = ctl->ss;
  double* __restrict__ dist = ctl->dist;
  int* __restrict__ site1 = ctl->site1;
  int* next = ctl->nxt;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int mine = 0;
  // blocks [0, own_blocks): the round's own proposals; the rest (multi-GPU
  // slabs): the halo-plane proposals received from the neighbour ranks
  const bool own = (int)blockIdx.x < own_blocks;
  const int bid = own ? (int)blockIdx.x : (int)blockIdx.x - own_blocks;
  const int nb = own ? min(own_blocks, (int)gridDim.x) : (int)gridDim.x - own_blocks;
  if (own && pf) {
    // sparse slots: each CTA step compacts the improved slots of CM_SLOTS
    // frontier items into shared memory, then commits them one per thread
    // (full lanes for the enqueue, one list reservation per CTA step)
    const int n = *(volatile const int*)&ctl->n_cur;
    for (int base = bid * CM_SLOTS; base < n; base += nb * CM_SLOTS) {  // block-uniform
      const int i0 = base + 4 * threadIdx.x;
      uchar4 f = make_uchar4(0, 0, 0, 0);
      if (i0 + 3 < n && ((reinterpret_cast<uintptr_t>(pf + i0) & 3) == 0)) {
        f = *reinterpret_cast<const uchar4*>(pf + i0);
      } else {
        if (i0 < n) f.x = pf[i0];
        if (i0 + 1 < n) f.y = pf[i0 + 1];
        if (i0 + 2 < n) f.z = pf[i0 + 2];
        if (i0 + 3 < n) f.w = pf[i0 + 3];
      }
      const int c = (f.x != 0) + (f.y != 0) + (f.z != 0) + (f.w != 0);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) s_wcnt[wid] = incl;
      __syncthreads();
      if (threadIdx.x == 0) {
        int sum = 0;
        for (int w = 0; w < CM_THREADS / 32; w++) {
          const int t = s_wcnt[w];
          s_wcnt[w] = sum;
          sum += t;
        }
        s_tot = sum;
      }
      __syncthreads();
      int pos = s_wcnt[wid] + incl - c;
      if (f.x) s_idx[pos++] = i0;
      if (f.y) s_idx[pos++] = i0 + 1;
      if (f.z) s_idx[pos++] = i0 + 2;
      if (f.w) s_idx[pos++] = i0 + 3;
      __syncthreads();
      const int tot = s_tot;
      for (int k0 = 0; k0 < tot; k0 += CM_THREADS) {  // block-uniform
        const int k = k0 + threadIdx.x;
        const bool take = k < tot;
        int v = 0;
        if (take) {
          const Prop p = imp[s_idx[k]];
          v = p.v;
          mine++;
          commit_one(p, ss, dist, site1);
        }
        mark_and_append(g, nbm, take, v, false, bm, next, counters + C_NNEXT, zlo, zhi, cbm);
      }
      __syncthreads();  // s_idx / s_wcnt reused by the next step
    }
  } else {
    const Prop* __restrict__ list = own ? imp : halo;
    const int n = own ? n_props : n_halo;
    for (int base = bid * blockDim.x; base < n; base += nb * blockDim.x) {  // block-uniform
      const int i = base + threadIdx.x;
      const bool take = i < n;
      int v = 0;
      if (take) {
        const Prop p = list[i];
        v = p.v;
        mine++;
        commit_one(p, ss, dist, site1);
      }
      mark_and_append(g, nbm, take, v, false, bm, next, counters + C_NNEXT, zlo, zhi, cbm);
    }
  }
  // committed count (own proposals: the halo blocks' are the neighbours'): warp sums, one atomic per CTA
  if (!own) mine = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  if (lane == 0 && mine) atomicAdd(&s_cnt, mine);
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt) atomicAdd(counters + C_NIMP, s_cnt);
  if (end_mode < 0) return;  // the host / k_sweep_end ends the round
  // the last block to finish ends the round (no separate launch)
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counters + C_DONE, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    counters[C_DONE] = 0;
    if (end_mode >= END_MG)
      mg_round_end(ctl, counters, end_mode == END_MG_SWEEP, h_out);
    else
      round_end(ctl, counters, hs, n_classes, loop, end_mode);
  }
}

// tile status word: epoch << 33 | inclusive << 32 | count
__device__ __forceinline__ unsigned long long ct_pack(unsigned epoch, bool incl, unsigned cnt) {
  return ((unsigned long long)epoch << 33) | ((unsigned long long)(incl ? 1u : 0u) << 32) | cnt;
}

__device__ __forceinline__ unsigned long long ct_load(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void ct_store(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int REORDER_MIN = 1 << 20;  // frontiers below this keep the append order

// Rewrites the frontier ctl->cur (n = ctl->n_cur voxels, after the round end)
// in voxel order from the frontier bitmap, clearing the words and coarse bits
// it reads. Frontiers under REORDER_MIN return at once (their bits are
// cleared by the next eval as usual). Tile = 2048 words = 8 warps x 8 passes
// of 32 words (one coarse chunk per pass, skipped when its coarse bit is 0).
__global__ void __launch_bounds__(CT_THREADS) k_reorder(uint32_t* __restrict__ bm, uint32_t* __restrict__ cbm,
                                                        int64_t bm_words, unsigned long long* __restrict__ status,
                                                        int* __restrict__ cs, RoundCtl* __restrict__ ctl) {
  const int n = *(volatile const int*)&ctl->n_cur;
  if (n < REORDER_MIN) return;
  __shared__ int s_tile;
  __shared__ unsigned s_epoch;
  __shared__ int s_warp[CT_THREADS / 32];
  __shared__ unsigned s_excl;
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    s_tile = atomicAdd(cs + CS_TILE, 1);  // dynamic ids: a tile only waits on tiles already started
    s_epoch = (unsigned)*(volatile int*)(cs + CS_EPOCH) + 1u;
  }
  __syncthreads();
  const int tile = s_tile;
  const unsigned epoch = s_epoch & 0x7fffffffu;
  const int64_t wbase = (int64_t)tile * CT_WORDS + (int64_t)wid * 256;  // this warp's 256 words
  const uint32_t cw = cbm[(int64_t)tile * CT_CWORDS + (wid >> 2)];   // its 8 coarse bits: (wid * 8 + k) & 31
  uint32_t wk[CT_WPT];
  int tot = 0;
#pragma unroll
  for (int k = 0; k < CT_WPT; k++) {
    const int64_t w = wbase + 32 * k + lane;
    const bool on = (cw >> ((wid * 8 + k) & 31)) & 1u;
    wk[k] = (on && w < bm_words) ? bm[w] : 0u;
    tot += __popc(wk[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if (lane == 0) s_warp[wid] = tot;
  __syncthreads();
  if (wid == 0) {
    const int x = lane < CT_THREADS / 32 ? s_warp[lane] : 0;
    int xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += t;
    }
    if (lane < CT_THREADS / 32) s_warp[lane] = xi - x;  // exclusive warp offsets
    const unsigned total = (unsigned)__shfl_sync(0xffffffffu, xi, CT_THREADS / 32 - 1);
    // publish, then look back over the predecessors (decoupled look-back)
    unsigned excl = 0;
    if (tile == 0) {
      if (lane == 0) ct_store(status, ct_pack(epoch, true, total));
    } else {
      if (lane == 0) ct_store(status + tile, ct_pack(epoch, false, total));
      int j = tile - 1;
      for (;;) {
        const int jj = j - lane;
        unsigned long long st = 0;
        bool ok = jj < 0;
        while (true) {
          if (!ok) {
            st = ct_load(status + jj);
            ok = (unsigned)(st >> 33) == epoch;
          }
          if (__all_sync(0xffffffffu, ok)) break;
        }
        const bool inc = jj >= 0 && ((st >> 32) & 1ull);
        const unsigned val = jj >= 0 ? (unsigned)st : 0u;
        const unsigned incm = __ballot_sync(0xffffffffu, inc);
        const int stop = incm ? __ffs(incm) - 1 : 32;  // first lane (nearest tile) holding an inclusive prefix
        unsigned part = lane <= stop ? val : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        excl += part;
        if (incm || j - 32 < 0) break;
        j -= 32;
      }
      if (lane == 0) ct_store(status + tile, ct_pack(epoch, true, excl + total));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  // warp-cooperative expansion: output slot o of a pass goes to lane o % 32,
  // which finds its word by a binary search over the pass's inclusive counts
  int* out = ctl->cur;
  int off = (int)s_excl + s_warp[wid];
#pragma unroll
  for (int k = 0; k < CT_WPT; k++) {
    const int c = __popc(wk[k]);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const int T = __shfl_sync(0xffffffffu, incl, 31);
    for (int j = 0; j < T; j += 32) {  // warp-uniform
      const int o = j + lane;
      int L = 0;
#pragma unroll
      for (int st = 16; st > 0; st >>= 1) {
        const int probe = __shfl_sync(0xffffffffu, incl, L + st - 1);
        if (probe <= o) L += st;
      }
      L = L > 31 ? 31 : L;
      const int inclL = __shfl_sync(0xffffffffu, incl, L);
      const int cL = __shfl_sync(0xffffffffu, c, L);
      const uint32_t wL = __shfl_sync(0xffffffffu, wk[k], L);
      if (o < T) {
        const int rank = o - (inclL - cL);
        const int bit = (int)__fns(wL, 0, rank + 1);
        out[off + o] = (int)(((wbase + 32 * k + L) << 5) + bit);
      }
    }
    off += T;
    if (wk[k]) bm[wbase + 32 * k + lane] = 0u;  // consumed
  }
  __syncthreads();  // every warp has read its coarse word
  if (tid < CT_CWORDS) cbm[(int64_t)tile * CT_CWORDS + tid] = 0u;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(cs + CS_DONE, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_last && tid == 0) {
    cs[CS_TILE] = 0;
    cs[CS_DONE] = 0;
    cs[CS_EPOCH] = (int)epoch;
    __threadfence();
  }
}

}  // namespace lrcvt
