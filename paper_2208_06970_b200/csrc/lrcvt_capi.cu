// lrcvt_capi.cu -- plan object, host orchestration and the extern "C"
// entry points declared in include/lrcvt_cuda.h.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/lrcvt_cuda.h"
#include "classify.cuh"
#include "compact.cuh"
#include "vote.cuh"
#include "masks.cuh"
#include "eval_p1.cuh"
#include "eval_p2.cuh"
#include "eval_warp.cuh"
#include "rounds_small.cuh"
#include "aggregate.cuh"
#include "seeding.cuh"
#include "layout.cuh"
#include "adjacency.cuh"

using namespace lrcvt;

namespace {

thread_local std::string g_last_error;
// number of this library's own kernel launches (CUB's internal kernels not
// counted); read by bench.py for the "gpu_launches" claim
unsigned long long g_launches = 0;
#define LAUNCHED(k) (g_launches += (k))

int set_error(int code, const char* what, cudaError_t e = cudaSuccess) {
  char buf[512];
  if (e != cudaSuccess)
    snprintf(buf, sizeof buf, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  else
    snprintf(buf, sizeof buf, "%s", what);
  g_last_error = buf;
  return code;
}

#define CK(call)                                                        \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) return set_error(LRCVT_E_CUDA, #call, e_);   \
  } while (0)

#define CKR(call)                                                       \
  do {                                                                  \
    int r_ = (call);                                                    \
    if (r_ != 0) return r_;                                             \
  } while (0)

#define CKL(what)                                                       \
  do {                                                                  \
    cudaError_t e_ = cudaGetLastError();                                \
    if (e_ != cudaSuccess) return set_error(LRCVT_E_CUDA, what, e_);    \
  } while (0)

// The short-lived scratch of the standalone passes (CCL, aggregation, plan
// setup) comes from the device's default stream-ordered pool. Its default
// release threshold (0) hands memory back to the driver at every
// synchronisation, which turned each large cudaMallocAsync into a fresh
// page-mapping (~100x the kernels' time); keep it pooled instead.
void retain_pool() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

bool is_pow2(double s) {
  int e;
  double m = frexp(s, &e);
  return s > 0 && m == 0.5;
}

int grid_for(int64_t n, int block, int cap = 1 << 30) {
  int64_t b = (n + block - 1) / block;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

struct EligiblePred {
  const int* comp;
  const uint8_t* has_site;
  __device__ __forceinline__ bool operator()(const int v) const {
    const int c = comp[v];
    return c >= 0 && has_site[c];
  }
};

struct IsRoot {
  const int* L;
  __device__ __forceinline__ bool operator()(const int v) const { return L[v] == v; }
};

struct IsInband {
  const int* comp;
  __device__ __forceinline__ bool operator()(const int v) const { return comp[v] >= 0; }
};

struct CountInband {
  const int* comp;
  __device__ __forceinline__ int operator()(const int v) const { return comp[v] >= 0 ? 1 : 0; }
};

__global__ void k_pack_sites(const double* __restrict__ pos3, int n, double4* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) out[s] = make_double4(pos3[3 * s], pos3[3 * s + 1], pos3[3 * s + 2], 0.0);
}

__global__ void k_unpack_sites(const double4* __restrict__ in, int n, double* __restrict__ pos3) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) {
    const double4 p = in[s];
    pos3[3 * s] = p.x; pos3[3 * s + 1] = p.y; pos3[3 * s + 2] = p.z;
  }
}

__global__ void k_unpack_ss(const int2* __restrict__ ss, int64_t n, int* __restrict__ site_of,
                            int* __restrict__ src) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int2 a = ss[i];
    site_of[i] = a.x;
    src[i] = a.y;
  }
}

__global__ void k_segment_batch(Geo g, const int* __restrict__ comp, const double* __restrict__ segs,
                                const int* __restrict__ want, int64_t n, double* __restrict__ t) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* s = segs + 6 * i;
  t[i] = segment_hit_t(comp, g, s[0], s[1], s[2], s[3], s[4], s[5], want[i]);
}

__global__ void k_segment_clear_batch(Geo g, const int* __restrict__ comp, const uint32_t* __restrict__ nbm,
                                      const double* __restrict__ segs, const int* __restrict__ want, int64_t n,
                                      uint8_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* s = segs + 6 * i;
  out[i] = segment_clear_fast(comp, nbm, box_of(g), s[0], s[1], s[2], s[3], s[4], s[5], want[i]) ? 1 : 0;
}

Geo make_geo(int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz) {
  Geo g;
  memset(&g, 0, sizeof g);
  g.nx = (int)nx; g.ny = (int)ny; g.nz = (int)nz;
  g.nxy = (int)(nx * ny);
  g.n = nx * ny * nz;
  g.sx = sx; g.sy = sy; g.sz = sz;
  g.inv_nx = 1.0 / (double)nx;
  g.inv_nxy = 1.0 / (double)(nx * ny);
  g.dyadic = is_pow2(sx) && is_pow2(sy) && is_pow2(sz);
  g.pack10 = nx <= 1024 && ny <= 1024 && nz <= 1024;
  g.ix = 1.0 / sx;
  g.iy = 1.0 / sy;
  g.iz = 1.0 / sz;
  g.isx = (float)(1.0 / sx);
  g.isy = (float)(1.0 / sy);
  g.isz = (float)(1.0 / sz);
  for (int k = 0; k < 26; k++) {
    int dx, dy, dz;
    offset_of(k, dx, dy, dz);
    g.off_d[k] = dx + (int)nx * (dy + (int)ny * dz);
  }
  // exact |c_w - c_v| by offset class when spacing is dyadic (centre
  // differences are then exact): sqrt(dx*dx + dy*dy + dz*dz), same order
  for (int c = 0; c < 8; c++) {
    volatile double ex = (c & 1) ? sx : 0.0, ey = (c & 2) ? sy : 0.0, ez = (c & 4) ? sz : 0.0;
    volatile double s2 = ex * ex;
    s2 = s2 + ey * ey;
    s2 = s2 + ez * ez;
    g.len_cls[c] = sqrt((double)s2);
  }
  return g;
}

bool geo_ok(int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz) {
  if (nx < 1 || ny < 1 || nz < 1) return false;
  if (!(sx > 0 && sy > 0 && sz > 0)) return false;
  const int64_t n = nx * ny * nz;
  return n < (int64_t(1) << 31) - 1 && nx < (1 << 30) && ny < (1 << 30) && nz < (1 << 30);
}

}  // namespace

constexpr int EW_SMALL_DEFAULT = LRCVT_CLASS0;  // frontier size served by the warp-per-voxel kernels
struct lrcvt_plan {
  Geo g;
  const int* comp = nullptr;
  int n_components = 0;
  int64_t max_sites = 0;
  int64_t n_inband = 0;
  int64_t n_eligible = 0;
  // frontier machinery
  int* list_a = nullptr;
  int* list_b = nullptr;
  int* eligible = nullptr;
  Prop* imp = nullptr;      // sparse proposals: slot i <-> frontier item i
  uint8_t* pf = nullptr;    // pf[i] = 1 iff slot i holds an improved proposal
  bool compact = false;      // large frontiers rewritten in voxel order by k_reorder (LRCVT_COMPACT=1)
  int p1_bs = 128, p2_bs = 64;  // eval CTA sizes (LRCVT_EVAL_BS=p1,p2)
  int p1_big_minb = P1_MIN_BLOCKS_BIG;  // register budget of the big-round phase-1 eval (LRCVT_P1_MINB=6|7|8)
  int p2_minb = 12;                     // CTAs per SM the phase-2 eval is compiled for (LRCVT_P2_MINB=8|12|16)
  uint32_t* bm = nullptr;  // frontier bitmap (1 bit per voxel)
  int64_t bm_words = 0;
  uint32_t* cbm = nullptr;                 // coarse frontier bitmap (1 bit per 32 words), compact.cuh
  unsigned long long* ct_status = nullptr;  // k_reorder tile status (decoupled look-back)
  int* ct_state = nullptr;                  // k_reorder epoch / tile / done counters
  int ct_tiles = 0;
  uint32_t* nbm = nullptr;  // static same-component neighbour masks
  int* site1 = nullptr;     // phase-1 LOS site per voxel (RoundCtl::site1)
  int2* mg_ss = nullptr;    // (site_of, src) buffer of the multi-GPU classify in flight
  double* mg_dist = nullptr;
  int2* mg_own_ss = nullptr;      // plan-owned multi-GPU state buffers (lrcvt_mg_state; IPC-exportable)
  double* mg_own_dist = nullptr;
  PeerView* d_pv = nullptr;       // multi-GPU peer view (lrcvt_mg_set_peers), null on one domain
  int mg_world = 1;
  Prop* mg_lo = nullptr;          // boundary-plane proposals for rank - 1 / rank + 1
  Prop* mg_hi = nullptr;
  bool mg_timing = false;         // device time of the syncing mg steps (lrcvt_mg_timing)
  cudaEvent_t mg_ev[2] = {nullptr, nullptr};
  double mg_ms = 0.0;
  int* counters = nullptr;
  int* h_counters = nullptr;  // pinned
  int* h_counters_dev = nullptr;  // its device-side address (kernels write the host copy directly)
  uint8_t* has_site = nullptr;
  // sites
  double4* site_pos = nullptr;
  double4* new_pos = nullptr;
  int* sk_key = nullptr;
  unsigned long long* sk_coll = nullptr;  // seed collision list: a power of two >= max_sites entries
  double* sk_d = nullptr;
  // vote
  unsigned long long* acc = nullptr;
  double* sums = nullptr;
  int* vt_key = nullptr;
  int* vt_key2 = nullptr;
  unsigned long long* vt_pv = nullptr;   // (phi(v), v) per eligible voxel
  unsigned long long* vt_pv2 = nullptr;
  int* seg_b = nullptr;
  int* seg_e = nullptr;
  int* vt_sp = nullptr;   // [2][n] site / phi planes per voxel for the bounding-box vote
  bool sp_stale = true;   // vt_sp must be reset to -1 before the next k_vote_prep
  int* vt_box = nullptr;  // [6][S] per-site bounding boxes
  int* vt_order = nullptr;  // [S] sites by box volume, largest first (k_vote_add's schedule)
  int* vt_hist = nullptr;   // [2][VO_BUCKETS] bucket counts / cursors
  // the walk / sum split of the ordered chains (vote.cuh k_vote_nseg .. k_vote_add)
  int* vt_nseg = nullptr;    // [S] walk segments per site
  int* vt_seg0 = nullptr;    // [S] first segment of each site
  int* vt_tot = nullptr;     // [2] segments, entries
  int* h_vt = nullptr;       // pinned copy of the segment total
  int vt_seg_cap = 0;        // segments vt_cnt / vt_off hold
  int* vt_cnt = nullptr;     // [segments] entries per segment
  int* vt_off = nullptr;     // [segments] first entry of each segment
  int2* vt_ent = nullptr;    // [in-band] (phi, v) per site in voxel order
  bool vote_bbox = true;  // LRCVT_VOTE=sort: stable radix sort of (site, (phi, v)) pairs instead
  // cub
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  // device-resident round control + CUDA-graph round loops (one per eval
  // variant: phase 1, phase 2 dyadic, phase 2 general)
  RoundCtl* ctl = nullptr;
  RoundCtl* h_ctl = nullptr;  // pinned readback
  int* d_nel = nullptr;       // eligible count (device)
  cudaGraphExec_t graph[3] = {nullptr, nullptr, nullptr};
  cudaGraphConditionalHandle* d_handles = nullptr;  // [3][MAX_CLASSES] size-class handles (SWITCH: slot 0 only)
  int n_classes = 0;
  cudaStream_t cap = nullptr;  // capture stream
  int eval_blocks[3] = {0, 0, 0};
  int commit_blocks = 0;
  // multi-GPU global mode: own z-slab [zlo, zhi); zhi = 1<<30 disables it
  int zlo = 0, zhi = 1 << 30;
  int h_ncur = 0;  // host mirror of ctl->n_cur in multi-GPU stepping
  // eligible list of the last classify is reused by centroidal_update when
  // the caller guarantees the site-component set is unchanged
  bool reuse_eligible = false;
  bool warp_eval = true;  // warp-per-voxel kernels for small frontiers (LRCVT_WARP_EVAL=0 disables)
  bool warp_eval_all = false;
  int ew_small = EW_SMALL_DEFAULT;
  bool coop = false;    // small frontiers: all their rounds in one cooperative kernel
  int coop_blocks = 0;  // co-resident CTAs of k_rounds_small
  bool coop_in_graph = false;  // k_rounds_small as the class-0 node of the round graph (LRCVT_COOP=2)
  int loop_min = 0;            // RoundCtl::loop_min
  // one SWITCH node selects the round's size class (LRCVT_SWITCH=0: a chain of
  // IF nodes, one per class, every one of them visited each round)
  bool class_switch = true;
  int ncl_arg() const { return class_switch ? -n_classes : n_classes; }
  bool eligible_valid = false;
  int64_t eligible_sites = -1;
  // persistent output buffers (lrcvt_plan_persistent_outputs): the last classify's output pointers
  bool persist = false;
  const void* last_ss = nullptr;
  const void* last_dist = nullptr;
  const void* last_state = nullptr;
  // optional per-launch timing of the dominant kernel (k_eval)
  bool timing = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  int64_t eval_launches = 0;
  int64_t eval_items = 0;
  double eval_ms = 0.0;
  // breakdown: [0] phase-1 eval ms, [1] phase-2 eval ms, [2] commit ms,
  // [3] phase-1 items, [4] phase-2 items, [5] committed proposals
  double prof[6] = {0, 0, 0, 0, 0, 0};
};

namespace {

template <typename T>
int dalloc(T** p, int64_t count) {
  if (count < 1) count = 1;
  cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (size_t)count);
  if (e != cudaSuccess) return set_error(LRCVT_E_NOMEM, "cudaMalloc", e);
  return 0;
}

int note_eval(lrcvt_plan* p, int64_t items, bool phase2, int64_t n_imp) {
  float ms = 0.f, ms2 = 0.f;
  CK(cudaEventElapsedTime(&ms, p->ev0, p->ev1));
  CK(cudaEventElapsedTime(&ms2, p->ev1, p->ev2));
  p->eval_ms += ms;
  p->eval_launches++;
  p->eval_items += items;
  p->prof[phase2 ? 1 : 0] += ms;
  p->prof[2] += ms2;
  p->prof[phase2 ? 4 : 3] += (double)items;
  p->prof[5] += (double)n_imp;
  return 0;
}

int sync_counters(lrcvt_plan* p, cudaStream_t st, int n = C_NCOUNTERS) {
  if (n > 0) CK(cudaMemcpyAsync(p->h_counters, p->counters, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

// eligible list for the current site set (tessellation.py:161-164)
int prepare_eligible(lrcvt_plan* p, int n_sites, const int* site_comp, cudaStream_t st) {
  CK(cudaMemsetAsync(p->has_site, 0, p->n_components > 0 ? p->n_components : 1, st));
  if (n_sites > 0) {
    k_mark_site_comps<<<grid_for(n_sites, 256), 256, 0, st>>>(site_comp, n_sites,
                                                            p->n_components > 0 ? p->n_components : 1, p->has_site);
    CKL("k_mark_site_comps"); LAUNCHED(1);
  }
  EligiblePred pred{p->comp, p->has_site};
  // own slab only in multi-GPU global mode (tessellation.py:163-164 restricted)
  const int z0 = p->zlo;
  const int z1 = p->zhi < p->g.nz ? p->zhi : p->g.nz;
  cub::CountingInputIterator<int> it(z0 * p->g.nxy);
  size_t bytes = p->cub_bytes;
  CK(cub::DeviceSelect::If(p->cub_tmp, bytes, it, p->eligible, p->d_nel, (z1 - z0) * p->g.nxy, pred, st));
  p->sp_stale = true;  // the bounding-box vote's (site, phi) entries of the previous set are now stale
  return 0;
}

// The eval kernel of variant `var` over ctl->cur with `blocks` blocks.
// Frontiers up to EW_SMALL voxels: warp-per-voxel kernels (eval_warp.cuh),
// whose round latency is one voxel's parallel evaluation instead of its
// serial one; larger frontiers: the thread-per-voxel tile kernels.
int launch_eval_kernel(lrcvt_plan* p, int var, int items, cudaStream_t st) {
  const Geo& g = p->g;
  if (items < 1) items = 1;
  if ((items <= p->ew_small && p->warp_eval) || p->warp_eval_all) {
    const int blocks = (int)(((int64_t)items + EW_WARPS - 1) / EW_WARPS);
    if (var != 0 && p->d_pv)
      k_eval_warp<true, true><<<blocks, 32 * EW_WARPS, 0, st>>>(p->ctl, g, p->comp, p->nbm, p->site_pos, p->bm,
                                                                 p->imp, p->pf, p->d_pv);
    else if (var == 0)
      k_eval_warp<false><<<blocks, 32 * EW_WARPS, 0, st>>>(p->ctl, g, p->comp, p->nbm, p->site_pos, p->bm, p->imp,
                                                            p->pf);
    else
      k_eval_warp<true><<<blocks, 32 * EW_WARPS, 0, st>>>(p->ctl, g, p->comp, p->nbm, p->site_pos, p->bm, p->imp,
                                                           p->pf);
    CKL("k_eval_warp");
    return 0;
  }
  const int bs = var == 0 ? p->p1_bs : p->p2_bs;
  const int blocks = (int)(((int64_t)items + bs - 1) / bs);
  RoundCtl* c = p->ctl;
  const int* cm = p->comp;
  const uint32_t* nb = p->nbm;
  const double4* sp = p->site_pos;
  const bool big = items >= P1_BIG_ROUND;
  if (var == 0) {  // CTA size x register budget (see eval_p1.cuh)
    if (bs == 32 && big)
      k_eval_p1<32, 32><<<blocks, 32, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
    else if (bs == 32)
      k_eval_p1<32, 20><<<blocks, 32, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
    else if (big && p->p1_big_minb == 6)
      k_eval_p1<128, 6><<<blocks, 128, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
    else if (big && p->p1_big_minb == 7)
      k_eval_p1<128, 7><<<blocks, 128, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
    else if (big)
      k_eval_p1<128, P1_MIN_BLOCKS_BIG><<<blocks, 128, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
    else
      k_eval_p1<128><<<blocks, 128, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
  } else if (p->d_pv) {  // multi-GPU slab: far reads through the peer view (the one-domain register budget)
    if (var == 1)
      k_eval_p2<64, true, true, 12><<<blocks, 64, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf, p->d_pv);
    else
      k_eval_p2<64, false, true, 12><<<blocks, 64, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf, p->d_pv);
  } else if (bs == 32) {
    if (var == 1)
      k_eval_p2<32, true><<<blocks, 32, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
    else
      k_eval_p2<32, false><<<blocks, 32, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
  } else if (p->p2_minb == 12) {  // register budget of the phase-2 eval (LRCVT_P2_MINB)
    if (var == 1)
      k_eval_p2<64, true, false, 12><<<blocks, 64, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
    else
      k_eval_p2<64, false, false, 12><<<blocks, 64, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
  } else if (p->p2_minb == 16) {
    if (var == 1)
      k_eval_p2<64, true, false, 16><<<blocks, 64, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
    else
      k_eval_p2<64, false, false, 16><<<blocks, 64, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
  } else {
    if (var == 1)
      k_eval_p2<64, true><<<blocks, 64, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
    else
      k_eval_p2<64, false><<<blocks, 64, 0, st>>>(c, g, cm, nb, sp, p->bm, p->imp, p->pf);
  }
  CKL("k_eval");
  return 0;
}

// commit + enqueue of the next frontier (compact.cuh k_commit): the sparse
// proposals of the round's eval (props == null) or a compact list of n_props
// records; end_mode as k_commit
int launch_commit_kernel(lrcvt_plan* p, int64_t items, cudaStream_t st, const Prop* props = nullptr,
                         int64_t n_props = 0, const cudaGraphConditionalHandle* hs = nullptr,
                         cudaGraphConditionalHandle loop = cudaGraphConditionalHandle{}, int end_mode = -1) {
  int64_t blocks = props ? (items + CM_THREADS - 1) / CM_THREADS : (items + CM_SLOTS - 1) / CM_SLOTS;
  if (blocks < 1) blocks = 1;
  if (blocks > p->commit_blocks) blocks = p->commit_blocks;  // grid-stride, one resident wave at most
  k_commit<<<(int)blocks, CM_THREADS, 0, st>>>(props ? props : p->imp, props ? nullptr : p->pf, (int)n_props, p->counters,
                                         p->ctl, p->g, p->nbm, p->bm, p->compact ? p->cbm : nullptr, hs,
                                         p->ncl_arg(), loop, end_mode, p->zlo, p->zhi);
  CKL("k_commit");
  return 0;
}

// the next frontier rewritten in voxel order when large (k_reorder; after the round end)
int launch_reorder_kernel(lrcvt_plan* p, cudaStream_t st) {
  if (!p->compact) return 0;
  k_reorder<<<p->ct_tiles, CT_THREADS, 0, st>>>(p->bm, p->cbm, p->bm_words, p->ct_status, p->ct_state, p->ctl);
  CKL("k_reorder");
  return 0;
}

// Host-driven round (n known on the host): exact grids; end_mode 0 = round
// end without graph conditionals, -1 = sweep (k_sweep_end follows).
int launch_round_kernels(lrcvt_plan* p, int var, int n, cudaStream_t st, int end_mode = 0) {
  CKR(launch_eval_kernel(p, var, n, st));
  if (p->timing) CK(cudaEventRecord(p->ev1, st));
  CKR(launch_commit_kernel(p, n, st, nullptr, 0, nullptr, cudaGraphConditionalHandle{}, end_mode));
  if (end_mode >= 0) CKR(launch_reorder_kernel(p, st));  // sweeps: after k_sweep_end
  if (p->timing) CK(cudaEventRecord(p->ev2, st));
  return 0;
}

// Relaxation rounds until the worklist drains (_kernels.py:337-385): a
// CUDA graph whose conditional WHILE node repeats eval -> commit -> round end
// entirely on the device (instantiated once per plan and variant).
int add_kernel_node(cudaGraphNode_t* node, cudaGraph_t g, const cudaGraphNode_t* dep, void* func, dim3 grid,
                    dim3 block, void** args) {
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeKernel;
  np.kernel.func = func;
  np.kernel.gridDim = grid;
  np.kernel.blockDim = block;
  np.kernel.kernelParams = args;
  CK(cudaGraphAddNode(node, g, dep, dep ? 1 : 0, &np));
  return 0;
}

int launch_rounds_small(lrcvt_plan* p, int var, cudaStream_t st, const cudaGraphConditionalHandle* hs = nullptr,
                        cudaGraphConditionalHandle loop = cudaGraphConditionalHandle{}, int in_graph = 0) {
  RoundCtl* ctl = p->ctl;
  Geo g = p->g;
  const int* comp = p->comp;
  const uint32_t* nbm = p->nbm;
  const double4* sp = p->site_pos;
  uint32_t* bm = p->bm;
  Prop* imp = p->imp;
  uint8_t* pf = p->pf;
  int* counters = p->counters;
  int small = p->ew_small, max_rounds = 1 << 20, ncl = p->ncl_arg();
  void* args[] = {&ctl, &g, &comp, &nbm, &sp, &bm, &imp, &pf, &counters, &small, &max_rounds, &hs, &ncl, &loop,
                  &in_graph};
  void* fn = var == 0 ? (void*)k_rounds_small<false> : (void*)k_rounds_small<true>;
  if (!in_graph) {
    CK(cudaLaunchCooperativeKernel(fn, dim3(p->coop_blocks), dim3(32 * EW_WARPS), args, 0, st));
  } else {  // captured into the round graph as a cooperative kernel node
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p->coop_blocks);
    cfg.blockDim = dim3(32 * EW_WARPS);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelExC(&cfg, fn, args));
  }
  LAUNCHED(1);
  return 0;
}

// launch size of size class c: its cap, clamped to the in-band count (every
// frontier, list and sweep holds at most n_inband voxels); the last class
// covers everything up to n_inband. Always in [1, 2^31).
long long class_launch_items(int c, int n_classes, int64_t n_inband) {
  const long long nin = n_inband > 0 ? n_inband : 1;
  long long cap = class_cap(c);
  if (cap > nin || c == n_classes - 1) cap = nin;
  return cap;
}

int count_classes(int64_t n_inband) {
  const int64_t nin = n_inband > 0 ? n_inband : 1;
  int n = 1;
  while (n < MAX_CLASSES && class_cap(n - 1) < nin) n++;
  return n;
}

struct GraphGuard {  // destroys the graph under construction on every exit path
  cudaGraph_t g = nullptr;
  ~GraphGuard() {
    if (g) cudaGraphDestroy(g);
  }
};

int build_round_graph(lrcvt_plan* p, int var) {
  if (!p->cap) CK(cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking));
  GraphGuard guard;
  CK(cudaGraphCreate(&guard.g, 0));
  cudaGraph_t g = guard.g;
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
  const int n_handles = p->class_switch ? 1 : p->n_classes;
  std::vector<cudaGraphConditionalHandle> hs(n_handles);
  for (int c = 0; c < n_handles; c++) CK(cudaGraphConditionalHandleCreate(&hs[c], g, 0, 0));
  cudaGraphConditionalHandle* d_hs = p->d_handles + var * MAX_CLASSES;
  CK(cudaMemcpy(d_hs, hs.data(), sizeof(cudaGraphConditionalHandle) * n_handles, cudaMemcpyHostToDevice));
  RoundCtl* ctl = p->ctl;
  cudaGraphNode_t n_init, n_loop;
  {
    int ncl = p->ncl_arg();
    void* args[] = {&ctl, &h, &d_hs, &ncl};
    CKR(add_kernel_node(&n_init, g, nullptr, (void*)k_loop_init, dim3(1), dim3(1), args));
  }
  cudaGraphNodeParams pw = {};
  pw.type = cudaGraphNodeTypeConditional;
  pw.conditional.handle = h;
  pw.conditional.type = cudaGraphCondTypeWhile;
  pw.conditional.size = 1;
  CK(cudaGraphAddNode(&n_loop, g, &n_init, 1, &pw));
  cudaGraph_t body = pw.conditional.phGraph_out[0];
  // body: SWITCH(class) { case c: eval with cap[c]/BLOCK blocks; commit + round
  // end with cap[c]/128 blocks } (or one IF node per class); the last commit
  // block arms the next round's class and the WHILE condition
  cudaGraphNode_t prev = nullptr;
  cudaGraph_t* sw_bodies = nullptr;  // SWITCH: body c runs when the handle holds c
  if (p->class_switch) {
    cudaGraphNodeParams ps = {};
    ps.type = cudaGraphNodeTypeConditional;
    ps.conditional.handle = hs[0];
    ps.conditional.type = cudaGraphCondTypeSwitch;
    ps.conditional.size = (unsigned)p->n_classes;
    cudaGraphNode_t nsw;
    CK(cudaGraphAddNode(&nsw, body, nullptr, 0, &ps));
    sw_bodies = ps.conditional.phGraph_out;
  }
  for (int c = 0; c < p->n_classes; c++) {
    cudaGraph_t ib;
    cudaGraphNode_t nif = nullptr;
    if (sw_bodies) {
      ib = sw_bodies[c];
    } else {
      cudaGraphNodeParams pi = {};
      pi.type = cudaGraphNodeTypeConditional;
      pi.conditional.handle = hs[c];
      pi.conditional.type = cudaGraphCondTypeIf;
      pi.conditional.size = 1;
      CK(cudaGraphAddNode(&nif, body, prev ? &prev : nullptr, prev ? 1 : 0, &pi));
      ib = pi.conditional.phGraph_out[0];
    }
    const long long cap = class_launch_items(c, p->n_classes, p->n_inband);
    CK(cudaStreamBeginCaptureToGraph(p->cap, ib, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    int rc = 0;
    if (c == 0 && p->coop_in_graph && cap <= p->ew_small) {
      rc = launch_rounds_small(p, var, p->cap, d_hs, h, 1);  // all small rounds in one cooperative node
    } else {
      rc = launch_eval_kernel(p, var, (int)cap, p->cap);
      if (!rc) rc = launch_commit_kernel(p, cap, p->cap, nullptr, 0, d_hs, h, 1);
      if (!rc) rc = launch_reorder_kernel(p, p->cap);
    }
    cudaGraph_t captured;
    const cudaError_t ee = cudaStreamEndCapture(p->cap, &captured);
    if (rc) return rc;
    if (ee != cudaSuccess) return set_error(LRCVT_E_CUDA, "round capture", ee);
    prev = nif;
  }
  CK(cudaGraphInstantiate(&p->graph[var], g, 0));
  return 0;
}

int run_rounds(lrcvt_plan* p, int var, cudaStream_t st) {
  if (!p->timing) {
    if (!p->graph[var]) CKR(build_round_graph(p, var));
    if (!p->coop || p->coop_in_graph) {
      CK(cudaGraphLaunch(p->graph[var], st));
      LAUNCHED(1);  // k_loop_init; per-round kernels are counted from ctl->rounds
      return 0;
    }
    // small frontiers in the cooperative kernel, large ones in the graph (which
    // loops while n_cur > loop_min); alternate until the frontier is empty
    for (int it = 0; it < 1000; ++it) {
      CKR(launch_rounds_small(p, var, st));
      CK(cudaGraphLaunch(p->graph[var], st));
      LAUNCHED(1);
      CKR(launch_rounds_small(p, var, st));
      CK(cudaMemcpyAsync(p->h_ctl, p->ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (p->h_ctl->n_cur <= 0) return 0;
    }
    return set_error(LRCVT_E_CUDA, "run_rounds: no convergence");
  }
  // host-driven rounds with per-launch CUDA-event timing (bench breakdown)
  CK(cudaMemcpyAsync(p->h_ctl, p->ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (;;) {
    const int n = p->h_ctl->n_cur;
    const long long commits0 = p->h_ctl->commits;
    if (n <= 0) return 0;
    CK(cudaEventRecord(p->ev0, st));
    CKR(launch_round_kernels(p, var, n, st));
    CK(cudaMemcpyAsync(p->h_ctl, p->ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CKR(note_eval(p, n, var != 0, p->h_ctl->commits - commits0));
  }
}

}  // namespace

namespace {
// stream-ordered scratch released on every exit path
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  cudaError_t raw(void** p, size_t bytes) {
    *p = nullptr;
    cudaError_t e = cudaMallocAsync(p, bytes > 0 ? bytes : 1, st);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
  template <typename T>
  cudaError_t get(T** p, int64_t count) {
    *p = nullptr;
    cudaError_t e = cudaMallocAsync((void**)p, sizeof(T) * (size_t)(count > 0 ? count : 1), st);
    if (e == cudaSuccess) ptrs.push_back(*p);
    return e;
  }
  ~Scratch() {
    for (void* q : ptrs) cudaFreeAsync(q, st);
  }
};

// numpy's pairwise split (seeding.cuh) cut into subtrees of at most kCut
// elements, left to right, and the sum rebuilt in the same shape
constexpr int64_t kSubtree = 128;  // = numpy's leaf size: one thread per leaf
void pw_split(int64_t lo, int64_t n, std::vector<int64_t>& L, std::vector<int64_t>& N) {
  if (n <= kSubtree) {
    L.push_back(lo);
    N.push_back(n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  pw_split(lo, n2, L, N);
  pw_split(lo + n2, n - n2, L, N);
}
double pw_join(int64_t n, const std::vector<double>& v, size_t& k) {
  if (n <= kSubtree) return v[k++];
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const double a = pw_join(n2, v, k);
  const double b = pw_join(n - n2, v, k);
  return a + b;
}
}  // namespace

extern "C" {

int lrcvt_version(void) { return 1; }

int32_t lrcvt_round_classes(int64_t n_inband, int64_t* launch_items, int32_t max_classes) {
  if (n_inband < 0 || n_inband >= (int64_t(1) << 31) || (max_classes > 0 && !launch_items))
    return set_error(LRCVT_E_ARG, "lrcvt_round_classes: bad arguments");
  const int n = count_classes(n_inband);
  for (int c = 0; c < n && c < max_classes; c++) launch_items[c] = class_launch_items(c, n, n_inband);
  return n;
}

const char* lrcvt_last_error(void) { return g_last_error.c_str(); }

int lrcvt_plan_create(lrcvt_plan** plan, int64_t nx, int64_t ny, int64_t nz, double sx, double sy,
                      double sz, const int32_t* d_comp, int32_t n_components, int64_t max_sites,
                      void* stream) {
  retain_pool();
  if (!plan || !d_comp || !geo_ok(nx, ny, nz, sx, sy, sz) || n_components < 0 || max_sites < 0)
    return set_error(LRCVT_E_ARG, "lrcvt_plan_create: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  lrcvt_plan* p = new lrcvt_plan();
  if (const char* e = getenv("LRCVT_WARP_EVAL")) {  // 0: never, 2: every frontier size (tests)
    p->warp_eval = e[0] != '0';
    p->warp_eval_all = e[0] == '2';
  }
  if (const char* e = getenv("LRCVT_EW_SMALL")) p->ew_small = atoi(e);
  if (const char* e = getenv("LRCVT_SWITCH")) p->class_switch = e[0] != '0';
  if (const char* e = getenv("LRCVT_VOTE")) p->vote_bbox = strcmp(e, "sort") != 0;
  if (const char* e = getenv("LRCVT_COMPACT")) p->compact = e[0] == '1';
  if (const char* e = getenv("LRCVT_P1_MINB")) p->p1_big_minb = atoi(e);
  if (const char* e = getenv("LRCVT_P2_MINB")) p->p2_minb = atoi(e);
  if (const char* e = getenv("LRCVT_EVAL_BS")) {
    int a = 0, b = 0;
    if (sscanf(e, "%d,%d", &a, &b) == 2) {
      if (a == 32 || a == 128) p->p1_bs = a;
      if (b == 32 || b == 64) p->p2_bs = b;
    }
  }
  // small frontiers: every round inside one cooperative kernel node of the
  // round graph (C1 2D -14%, C3 -1.5%, C2 neutral; LRCVT_COOP=0 off, =1 host-
  // alternated variant, =2 in-graph)
  p->coop = true;
  p->coop_in_graph = true;
  if (const char* e = getenv("LRCVT_COOP")) {
    p->coop = e[0] == '1' || e[0] == '2';
    p->coop_in_graph = e[0] == '2';
  }
  p->g = make_geo(nx, ny, nz, sx, sy, sz);
  p->comp = d_comp;
  p->n_components = n_components;
  p->max_sites = max_sites;
  const int64_t n = p->g.n;
  int rc = 0;
  rc |= dalloc(&p->counters, C_NCOUNTERS);
  if (cudaMallocHost((void**)&p->h_counters, sizeof(int) * C_NCOUNTERS) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&p->h_counters_dev, p->h_counters, 0) != cudaSuccess)
    rc = LRCVT_E_NOMEM;
  if (rc) { lrcvt_plan_destroy(p); return set_error(LRCVT_E_NOMEM, "plan counters"); }
  // count in-band voxels
  {
    auto count = [&]() -> int {
      CountInband op{d_comp};
      cub::CountingInputIterator<int> it(0);
      cub::TransformInputIterator<int, CountInband, cub::CountingInputIterator<int>> tin(it, op);
      size_t bytes = 0;
      CK(cub::DeviceReduce::Sum(nullptr, bytes, tin, p->counters, (int)n, st));
      Scratch sc(st);
      char* tmp = nullptr;
      CK(sc.get(&tmp, (int64_t)bytes));
      CK(cub::DeviceReduce::Sum(tmp, bytes, tin, p->counters, (int)n, st));
      return sync_counters(p, st, 1);
    };
    if (const int e = count()) { lrcvt_plan_destroy(p); return e; }  // no partial plan on failure
    p->n_inband = p->h_counters[0];
  }
  const int64_t nin = p->n_inband > 0 ? p->n_inband : 1;
  const int64_t S = max_sites > 0 ? max_sites : 1;
  p->bm_words = (n + 31) / 32;
  rc = 0;
  rc |= dalloc(&p->list_a, nin);
  rc |= dalloc(&p->list_b, nin);
  rc |= dalloc(&p->eligible, nin);
  rc |= dalloc(&p->imp, nin);
  rc |= dalloc(&p->pf, nin);
  rc |= dalloc(&p->bm, p->bm_words);
  p->ct_tiles = (int)compact_tiles(p->bm_words);
  rc |= dalloc(&p->cbm, coarse_words(p->bm_words));
  rc |= dalloc(&p->ct_status, p->ct_tiles);
  rc |= dalloc(&p->ct_state, CS_N);
  rc |= dalloc(&p->nbm, n);
  rc |= dalloc(&p->site1, n);
  rc |= dalloc(&p->ctl, 1);
  if (!rc && cudaMemsetAsync(p->ctl, 0, sizeof(RoundCtl), st) != cudaSuccess) rc = LRCVT_E_CUDA;  // bo.lo = null
  rc |= dalloc(&p->d_handles, 3 * MAX_CLASSES);
  rc |= dalloc(&p->d_nel, 1);
  rc |= dalloc(&p->has_site, n_components > 0 ? n_components : 1);
  rc |= dalloc(&p->site_pos, S);
  rc |= dalloc(&p->new_pos, S);
  rc |= dalloc(&p->sk_key, S);
  {
    int64_t pc = 1;
    while (pc < S) pc <<= 1;
    rc |= dalloc(&p->sk_coll, pc);
  }
  rc |= dalloc(&p->sk_d, S);
  rc |= dalloc(&p->acc, 4 * S);
  rc |= dalloc(&p->sums, 4 * S);
  rc |= dalloc(&p->seg_b, S);
  rc |= dalloc(&p->seg_e, S);
  if (rc) { lrcvt_plan_destroy(p); return LRCVT_E_NOMEM; }
  {  // static neighbour words + clearance layers in bits 26..31 (exact ray shortcut, common.cuh)
    auto build = [&]() -> int {
      k_nbr_mask<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(p->g, d_comp, p->nbm);
      CKL("k_nbr_mask"); LAUNCHED(1);
      Scratch sc(st);
      unsigned char* clr = nullptr;
      CK(sc.get(&clr, n));
      k_clear_init<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(p->g, d_comp, p->nbm, clr);
      CKL("k_clear_init"); LAUNCHED(1);
      for (int r = 1; r <= CLR_MAX; r++) {
        k_clear_layer<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(p->g, clr, r);
        CKL("k_clear_layer"); LAUNCHED(1);
      }
      k_clear_store<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(n, clr, p->nbm);
      CKL("k_clear_store"); LAUNCHED(1);
      return 0;
    };
    if (const int e = build()) { lrcvt_plan_destroy(p); return e; }
  }
  if (cudaMemsetAsync(p->bm, 0, sizeof(uint32_t) * p->bm_words, st) != cudaSuccess ||
      cudaMemsetAsync(p->cbm, 0, sizeof(uint32_t) * coarse_words(p->bm_words), st) != cudaSuccess ||
      cudaMemsetAsync(p->ct_status, 0, sizeof(unsigned long long) * p->ct_tiles, st) != cudaSuccess ||
      cudaMemsetAsync(p->ct_state, 0, sizeof(int) * CS_N, st) != cudaSuccess) {
    lrcvt_plan_destroy(p);
    return set_error(LRCVT_E_CUDA, "bitmap clear");
  }
  // cub temp storage: max over the uses
  size_t need = 0, b = 0;
  {
    EligiblePred pred{p->comp, p->has_site};
    cub::CountingInputIterator<int> it(0);
    cub::DeviceSelect::If(nullptr, b, it, p->eligible, p->counters, (int)n, pred, st);
    need = b > need ? b : need;
    b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, p->list_a, p->list_b, p->list_a, p->list_b, (int)nin, 0, 32, st);
    need = b > need ? b : need;
    b = 0;  // the ordered vote sorts (site, (phi, v)) pairs: 8-byte values
    cub::DeviceRadixSort::SortPairs(nullptr, b, p->list_a, p->list_b, (unsigned long long*)nullptr,
                                    (unsigned long long*)nullptr, (int)nin, 0, 32, st);
    need = b > need ? b : need;
  }
  p->cub_bytes = need;
  p->n_classes = count_classes(nin);
  if (cudaMallocHost((void**)&p->h_ctl, sizeof(RoundCtl)) != cudaSuccess) {
    lrcvt_plan_destroy(p);
    return set_error(LRCVT_E_NOMEM, "pinned round control");
  }
  {
    int dev = 0, sms = 148, nb = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_eval_p1<128>, 128, 0);
    p->eval_blocks[0] = (nb > 0 ? nb : 1) * sms;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_eval_p2<64, true>, 64, 0);
    p->eval_blocks[1] = (nb > 0 ? nb : 1) * sms;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_eval_p2<64, false>, 64, 0);
    p->eval_blocks[2] = (nb > 0 ? nb : 1) * sms;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_commit, CM_THREADS, 0);
    p->commit_blocks = (nb > 0 ? nb : 1) * sms;
    int nb0 = 0, nb1 = 0;  // cooperative kernel: every CTA co-resident
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb0, k_rounds_small<false>, 32 * EW_WARPS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb1, k_rounds_small<true>, 32 * EW_WARPS, 0);
    const int nbc = nb0 < nb1 ? nb0 : nb1;
    p->coop_blocks = sms;  // one CTA per SM: the three grid barriers per round stay cheap (measured best)
    if (nbc <= 0) p->coop = false;
    if (const char* e = getenv("LRCVT_COOP_BLOCKS")) {
      const int want = atoi(e);
      if (want > 0 && want < p->coop_blocks) p->coop_blocks = want;
    }
    int coop_ok = 0;
    cudaDeviceGetAttribute(&coop_ok, cudaDevAttrCooperativeLaunch, dev);
    if (!coop_ok || nbc <= 0) p->coop = false;
    if (!p->coop) p->coop_in_graph = false;
    // set on the device by k_phase1_start at the start of every classify
    p->loop_min = (p->coop && !p->coop_in_graph) ? p->ew_small : 0;
  }
  if (dalloc((char**)&p->cub_tmp, (int64_t)need)) { lrcvt_plan_destroy(p); return LRCVT_E_NOMEM; }
  *plan = p;
  return 0;
}

int lrcvt_plan_destroy(lrcvt_plan* p) {
  if (!p) return 0;
  for (auto& gx : p->graph)
    if (gx) cudaGraphExecDestroy(gx);
  if (p->cap) cudaStreamDestroy(p->cap);
  if (p->h_ctl) cudaFreeHost(p->h_ctl);
  void* bufs[] = {p->counters, p->ctl, p->d_handles, p->d_nel, p->list_a, p->list_b, p->eligible, p->imp, p->pf,
                  p->bm,
                  p->cbm, p->ct_status, p->ct_state, p->nbm, p->site1, p->has_site,
                  p->site_pos, p->new_pos, p->sk_key, p->sk_coll, p->sk_d,
                  p->acc, p->sums, p->vt_key, p->vt_key2, p->vt_pv, p->vt_pv2,
                  p->seg_b, p->seg_e, p->vt_sp, p->vt_box, p->vt_order, p->vt_hist, p->vt_nseg, p->vt_seg0, p->vt_tot,
                  p->vt_cnt, p->vt_off, p->vt_ent, p->mg_own_ss, p->mg_own_dist, p->d_pv,
                  p->mg_lo, p->mg_hi, p->cub_tmp};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (p->h_counters) cudaFreeHost(p->h_counters);
  if (p->h_vt) cudaFreeHost(p->h_vt);
  if (p->ev0) cudaEventDestroy(p->ev0);
  if (p->ev1) cudaEventDestroy(p->ev1);
  if (p->ev2) cudaEventDestroy(p->ev2);
  for (cudaEvent_t e : p->mg_ev)
    if (e) cudaEventDestroy(e);
  delete p;
  return 0;
}

int64_t lrcvt_plan_inband(const lrcvt_plan* p) { return p ? p->n_inband : -1; }

int lrcvt_plan_set_timing(lrcvt_plan* p, int enable) {
  if (!p) return set_error(LRCVT_E_ARG, "lrcvt_plan_set_timing");
  if (enable && !p->ev0) {
    CK(cudaEventCreate(&p->ev0));
    CK(cudaEventCreate(&p->ev1));
    CK(cudaEventCreate(&p->ev2));
  }
  for (double& d : p->prof) d = 0.0;
  p->timing = enable != 0;
  p->eval_launches = 0;
  p->eval_items = 0;
  p->eval_ms = 0.0;
  return 0;
}

int lrcvt_plan_timing(const lrcvt_plan* p, int64_t* launches, int64_t* items, double* ms) {
  if (!p || !launches || !items || !ms) return set_error(LRCVT_E_ARG, "lrcvt_plan_timing");
  *launches = p->eval_launches;
  *items = p->eval_items;
  *ms = p->eval_ms;
  return 0;
}

int lrcvt_plan_reuse_eligible(lrcvt_plan* p, int enable) {
  if (!p) return set_error(LRCVT_E_ARG, "lrcvt_plan_reuse_eligible");
  p->reuse_eligible = enable != 0;
  if (enable == 2) p->eligible_valid = false;  // a new run: the next classify builds the list
  return 0;
}

int lrcvt_plan_persistent_outputs(lrcvt_plan* p, int enable) {
  if (!p) return set_error(LRCVT_E_ARG, "lrcvt_plan_persistent_outputs");
  p->persist = enable != 0;
  return 0;
}

int lrcvt_plan_profile(const lrcvt_plan* p, double* out6) {
  if (!p || !out6) return set_error(LRCVT_E_ARG, "lrcvt_plan_profile");
  for (int i = 0; i < 6; i++) out6[i] = p->prof[i];
  return 0;
}

unsigned long long lrcvt_launch_count(void) { return g_launches; }

int lrcvt_classify(lrcvt_plan* p, int64_t n_sites, const double* d_site_pos,
                   const int32_t* d_site_comp, int32_t* d_site_src, double* d_dist,
                   uint8_t* d_state, lrcvt_classify_stats* stats, void* stream) {
  if (!p || n_sites < 0 || n_sites > p->max_sites || !d_site_src || !d_dist || !stats)
    return set_error(LRCVT_E_ARG, "lrcvt_classify: bad arguments");
  if (n_sites > 0 && (!d_site_pos || !d_site_comp))
    return set_error(LRCVT_E_ARG, "lrcvt_classify: null site arrays");
  cudaStream_t st = (cudaStream_t)stream;
  const Geo& g = p->g;
  const int S = (int)n_sites;
  int2* ss = reinterpret_cast<int2*>(d_site_src);
  memset(stats, 0, sizeof *stats);
  CK(cudaMemsetAsync(p->counters, 0, sizeof(int) * C_NCOUNTERS, st));
  if (S == 0) {  // tessellation.py:120-134
    k_fill_state<<<grid_for(g.n, 256, 148 * 32), 256, 0, st>>>(ss, d_dist, g.n);
    CKL("k_fill_state"); LAUNCHED(1);
    if (d_state) CK(cudaMemsetAsync(d_state, 0, (size_t)g.n, st));
    CK(cudaStreamSynchronize(st));
    return 0;
  }
  // the eligible list (in-band voxels of components that have sites,
  // tessellation.py:161-164) up front: no voxel outside it is ever assigned,
  // so the per-voxel passes below only touch it
  const bool reuse = p->reuse_eligible && p->eligible_valid && p->eligible_sites == S;
  // persistent outputs: the caller passes the buffers of its previous classify again, untouched, with the
  // same eligible set -- every voxel outside the list still holds its fill value / state 0
  const bool fast = reuse && p->persist && p->last_ss == ss && p->last_dist == d_dist && p->last_state == d_state;
  if (!reuse) {
    if (prepare_eligible(p, S, d_site_comp, st)) return LRCVT_E_CUDA;
    p->eligible_valid = true;
    p->eligible_sites = S;
  }
#ifndef LRCVT_EL_WAVES
#define LRCVT_EL_WAVES 16
#endif
  const int el_grid = grid_for(p->n_inband, 256, 148 * LRCVT_EL_WAVES);  // the eligible-list passes
  if (!fast) {  // tessellation.py:120-122
    k_fill_state<<<grid_for(g.n, 256, 148 * 32), 256, 0, st>>>(ss, d_dist, g.n);
    CKL("k_fill_state"); LAUNCHED(1);
  }
  // site1 only: every eligible voxel's (site_of, src) / dist is written by k_site1_to_state when phase 2
  // starts (phase 1 reads and writes site1 alone; the seeds' ss / dist entries are rewritten identically)
  k_fill_list<<<el_grid, 256, 0, st>>>(p->eligible, p->d_nel, nullptr, d_dist, p->site1);
  CKL("k_fill_list"); LAUNCHED(1);
  p->last_ss = ss;
  p->last_dist = d_dist;
  p->last_state = d_state;
  k_pack_sites<<<grid_for(S, 256), 256, 0, st>>>(d_site_pos, S, p->site_pos);
  CKL("k_pack_sites"); LAUNCHED(1);
  // _place_seeds (tessellation.py:136-140)
  k_site_voxel<<<grid_for(S, 256), 256, 0, st>>>(g, p->comp, p->site_pos, d_site_comp, S, p->sk_key, p->sk_d,
                                                 p->site1, p->counters);
  CKL("k_site_voxel"); LAUNCHED(1);
  // seeds, then the phase-1 worklist (tessellation.py:151); sites outside
  // their component are skipped and reported at the end
  k_seed_groups<<<grid_for(S, 128), 128, 0, st>>>(g, p->nbm, p->sk_key, p->sk_d, S, ss, d_dist, p->site1, p->bm,
                                                  p->list_a, p->sk_coll, p->counters);  // marks bm (round-1 frontier)
  CKL("k_seed_groups"); LAUNCHED(1);
  k_seed_collisions<<<1, SEED_COLL_THREADS, 0, st>>>(p->sk_coll, p->sk_d, ss, d_dist, p->site1, p->counters);
  CKL("k_seed_collisions"); LAUNCHED(1);
  k_phase1_start<<<1, 1, 0, st>>>(p->ctl, p->counters, p->list_a, p->list_b, ss, d_dist, p->site1, p->loop_min);
  CKL("k_phase1_start"); LAUNCHED(1);
  // phase 1 (tessellation.py:152-156)
  CKR(run_rounds(p, 0, st));
  // phase 2 (tessellation.py:161-189): rounds from the eligible list, verification sweeps
  k_site1_to_state<<<el_grid, 256, 0, st>>>(g, p->site1, p->site_pos, ss, d_dist, p->eligible, p->d_nel, 0, 0);
  CKL("k_site1_to_state"); LAUNCHED(1);
  k_phase2_copy<<<1, 1, 0, st>>>(p->eligible, p->d_nel, p->ctl, p->counters);
  CKL("k_phase2_copy"); LAUNCHED(1);
  const int var2 = g.dyadic ? 1 : 2;
  for (;;) {
    CKR(run_rounds(p, var2, st));
    stats->sweeps++;
    k_sweep_start<<<1, 1, 0, st>>>(p->ctl, p->eligible, p->d_nel, p->counters);
    CKL("k_sweep_start"); LAUNCHED(1);
    if (p->timing) CK(cudaEventRecord(p->ev0, st));
    CKR(launch_round_kernels(p, var2, (int)p->n_inband, st, -1));  // sweep: n_el <= in-band
    k_sweep_end<<<1, 1, 0, st>>>(p->ctl, p->counters);
    CKL("k_sweep_end"); LAUNCHED(3);  // eval, commit, sweep end
    CKR(launch_reorder_kernel(p, st));
    CK(cudaMemcpyAsync(p->h_ctl, p->ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (p->timing) {
      CK(cudaMemcpyAsync(p->h_counters + H_NEL, p->d_nel, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      CKR(note_eval(p, p->h_counters[H_NEL], true, p->h_ctl->sweep_imp));
    }
    if (p->h_ctl->sweep_imp == 0) break;
  }
  // state bits + assigned (tessellation.py:191-204): state 0 outside the eligible list
  if (d_state && !fast) CK(cudaMemsetAsync(d_state, 0, (size_t)g.n, st));
  k_state<<<el_grid, 256, 0, st>>>(ss, p->eligible, p->d_nel, 0, 0, d_state, p->counters);
  CKL("k_state"); LAUNCHED(1);
  CK(cudaMemcpyAsync(p->h_ctl, p->ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(p->h_counters + H_NEL, p->d_nel, sizeof(int), cudaMemcpyDeviceToHost, st));
  CKR(sync_counters(p, st, C_ASSIGNED + 1));
  const RoundCtl& c = *p->h_ctl;
  p->n_eligible = p->h_counters[H_NEL];
  stats->eligible = p->n_eligible;
  stats->rounds = c.rounds;
  stats->phase1_rounds = c.rounds_p1;
  stats->evaluations = c.evals;
  stats->commits = c.commits;
  stats->assigned = p->h_counters[C_ASSIGNED];
  stats->bad_sites = p->h_counters[C_BAD];
  // eval, commit, compact (+ fused round end) per launched relaxation round; one k_rounds_small
  // launch covers all its rounds
  LAUNCHED((p->compact ? 3 : 2) * (c.rounds - c.rounds_small) + c.small_launches);  // + k_reorder when on
  if (p->h_counters[C_BAD]) {
    p->eligible_valid = false;
    return p->h_counters[C_BAD];
  }
  return 0;
}

// the bounding-box vote's per-voxel (site, phi) entries, reset
// whenever the eligible set was rebuilt since the last vote (sp_stale)
static int vote_buffers(lrcvt_plan* p, cudaStream_t st) {
  const size_t n = (size_t)p->g.n;
  if (!p->vt_sp) {
    int rc = dalloc(&p->vt_sp, 2 * n);
    rc |= dalloc(&p->vt_box, 6 * p->max_sites);
    rc |= dalloc(&p->vt_order, p->max_sites);
    rc |= dalloc(&p->vt_hist, 2 * VO_BUCKETS);
    rc |= dalloc(&p->vt_nseg, p->max_sites);
    rc |= dalloc(&p->vt_seg0, p->max_sites);
    rc |= dalloc(&p->vt_tot, 2);
    rc |= dalloc(&p->vt_ent, p->n_inband > 0 ? p->n_inband : 1);
    if (!rc && cudaMallocHost((void**)&p->h_vt, sizeof(int) * 2) != cudaSuccess) rc = LRCVT_E_NOMEM;
    if (rc) return LRCVT_E_NOMEM;
  }
  if (p->sp_stale) {
    CK(cudaMemsetAsync(p->vt_sp, 0xff, sizeof(int) * n, st));  // the site plane
    p->sp_stale = false;
  }
  return 0;
}

// k_vote_add's site order from the boxes: largest first (vote.cuh)
static int vote_order(lrcvt_plan* p, const int* d_box, int S, cudaStream_t st) {
  CK(cudaMemsetAsync(p->vt_hist, 0, sizeof(int) * 2 * VO_BUCKETS, st));
  k_vote_order_hist<<<grid_for(S, 256), 256, 0, st>>>(d_box, S, p->vt_hist);
  CKL("k_vote_order_hist"); LAUNCHED(1);
  k_vote_order_scatter<<<grid_for(S, 256), 256, 0, st>>>(d_box, S, p->vt_hist, p->vt_hist + VO_BUCKETS,
                                                          p->vt_order);
  CKL("k_vote_order_scatter"); LAUNCHED(1);
  return 0;
}

// the ordered chains of every site over planes [zlo, zhi) (mode / init as
// vote.cuh describes): walk segments counted, compacted into per-site entry
// runs in voxel order, then summed one warp per site, largest boxes first
static int vote_chains(lrcvt_plan* p, const int* d_box, int S, int w_mode, const void* d_weights, int zlo, int zhi,
                       int mode, const double* d_init, double* d_out, cudaStream_t st) {
  const Geo& g = p->g;
  CKR(vote_order(p, d_box, S, st));
  k_vote_nseg<<<grid_for(S, 256), 256, 0, st>>>(d_box, S, zlo, zhi, mode, p->vt_nseg);
  CKL("k_vote_nseg"); LAUNCHED(1);
  k_scan_excl<<<1, SCAN_THREADS, 0, st>>>(p->vt_nseg, S, p->vt_seg0, p->vt_tot);
  CKL("k_scan_excl"); LAUNCHED(1);
  CK(cudaMemcpyAsync(p->h_vt, p->vt_tot, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));  // the segment count sizes the next launches' arrays
  const int n_seg = p->h_vt[0];
  if (n_seg > p->vt_seg_cap) {
    cudaFree(p->vt_cnt);
    cudaFree(p->vt_off);
    p->vt_cnt = p->vt_off = nullptr;
    p->vt_seg_cap = n_seg + n_seg / 4 + 1024;
    if (dalloc(&p->vt_cnt, p->vt_seg_cap) || dalloc(&p->vt_off, p->vt_seg_cap)) {
      p->vt_seg_cap = 0;
      return LRCVT_E_NOMEM;
    }
  }
  if (n_seg > 0) {
    // segment counts from the eligible list (a COUNT walk of the boxes gives the same: vote.cuh)
    CK(cudaMemsetAsync(p->vt_cnt, 0, sizeof(int) * (size_t)n_seg, st));
    k_vote_count<<<grid_for(p->n_inband, 256, 148 * LRCVT_EL_WAVES), 256, 0, st>>>(p->eligible, p->d_nel, p->vt_sp, d_box, S, g,
                                                                        zlo, zhi, mode, p->vt_seg0, p->vt_cnt);
    CKL("k_vote_count"); LAUNCHED(1);
    k_scan_excl<<<1, SCAN_THREADS, 0, st>>>(p->vt_cnt, n_seg, p->vt_off, p->vt_tot + 1);
    CKL("k_scan_excl"); LAUNCHED(1);
    k_vote_walk<true><<<148 * 8, 128, 0, st>>>(p->vt_sp, d_box, S, g, zlo, zhi, mode, p->vt_seg0, p->vt_tot,
                                                nullptr, p->vt_off, p->vt_ent);
    CKL("k_vote_walk<write>"); LAUNCHED(1);
  } else {
    CK(cudaMemsetAsync(p->vt_tot + 1, 0, sizeof(int), st));
  }
  k_vote_add<4, 8, 4><<<grid_for(S, 4), 128, 0, st>>>(
      p->vt_order, S, g, (const double*)d_weights, (const float*)d_weights, w_mode, mode, d_init, p->vt_seg0,
      p->vt_nseg, p->vt_off, p->vt_tot + 1, p->vt_tot, p->vt_ent, d_out);
  CKL("k_vote_add"); LAUNCHED(1);
  return 0;
}

int lrcvt_centroidal_update(lrcvt_plan* p, int64_t n_sites, const double* d_site_pos,
                            const int32_t* d_site_comp, const int32_t* d_site_src,
                            int32_t weight_mode, const void* d_weights, double backoff,
                            double* d_new_pos, double* d_disp, double* d_sums,
                            int64_t* empty_regions, void* stream) {
  if (!p || n_sites < 0 || n_sites > p->max_sites || !d_site_src || !d_new_pos || !d_disp ||
      weight_mode < 0 || weight_mode > 3 || (weight_mode != LRCVT_W_ONES && !d_weights))
    return set_error(LRCVT_E_ARG, "lrcvt_centroidal_update: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const Geo& g = p->g;
  const int S = (int)n_sites;
  const int2* ss = reinterpret_cast<const int2*>(d_site_src);
  if (empty_regions) *empty_regions = 0;
  if (S == 0) return 0;
  k_pack_sites<<<grid_for(S, 256), 256, 0, st>>>(d_site_pos, S, p->site_pos);
  CKL("k_pack_sites"); LAUNCHED(1);
  if (!(p->reuse_eligible && p->eligible_valid && p->eligible_sites == S)) {
    if (prepare_eligible(p, S, d_site_comp, st)) return LRCVT_E_CUDA;
    CK(cudaMemcpyAsync(p->h_counters + H_NEL, p->d_nel, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    p->n_eligible = p->h_counters[H_NEL];
    p->eligible_valid = true;
    p->eligible_sites = S;
  }
  const int n_el = (int)p->n_eligible;
  const bool exact = weight_mode == LRCVT_W_ONES && g.dyadic && g.nx <= (1 << 20) &&
                     g.ny <= (1 << 20) && g.nz <= (1 << 20);
  if (exact) {
    CK(cudaMemsetAsync(p->acc, 0, sizeof(unsigned long long) * 4 * S, st));
    if (n_el > 0) {
      k_vote_exact<false><<<grid_for(n_el, 256, 148 * 8), 256, 0, st>>>(p->eligible, n_el, g, ss, p->acc, S, nullptr);
      CKL("k_vote_exact"); LAUNCHED(1);
    }
    k_vote_exact_finish<<<grid_for(S, 256), 256, 0, st>>>(p->acc, S, 0.5 * g.sx, 0.5 * g.sy, 0.5 * g.sz,
                                                          p->sums);
    CKL("k_vote_exact_finish"); LAUNCHED(1);
  } else if (p->vote_bbox) {
    // ordered path, sort-free: per-site bounding-box walk (vote.cuh k_vote_prep, k_vote_nseg .. k_vote_add)
    CKR(vote_buffers(p, st));
    k_box_init<<<grid_for(S, 256), 256, 0, st>>>(p->vt_box, S);
    CKL("k_box_init"); LAUNCHED(1);
    if (n_el > 0) {
      k_vote_prep<false><<<grid_for(n_el, 256, 148 * 8), 256, 0, st>>>(p->eligible, n_el, g, ss, p->vt_sp, p->vt_box,
                                                                       S, nullptr);
      CKL("k_vote_prep"); LAUNCHED(1);
    }
    CKR(vote_chains(p, p->vt_box, S, weight_mode, d_weights, 0, (int)g.nz, 0, nullptr, p->sums, st));
  } else {
    const int64_t nin = p->n_inband > 0 ? p->n_inband : 1;
    int rc = 0;
    if (!p->vt_key) {
      rc |= dalloc(&p->vt_key, nin);
      rc |= dalloc(&p->vt_key2, nin);
      rc |= dalloc(&p->vt_pv, nin);
      rc |= dalloc(&p->vt_pv2, nin);
      if (rc) return LRCVT_E_NOMEM;
    }
    CK(cudaMemsetAsync(p->seg_b, 0, sizeof(int) * S, st));
    CK(cudaMemsetAsync(p->seg_e, 0, sizeof(int) * S, st));
    if (n_el > 0) {
      k_vote_pairs<<<grid_for(n_el, 256, 148 * 8), 256, 0, st>>>(p->eligible, n_el, ss, S, p->vt_key, p->vt_pv);
      CKL("k_vote_pairs"); LAUNCHED(1);
      int bits = 1;
      while ((1ll << bits) <= S) bits++;
      size_t bytes = p->cub_bytes;
      CK(cub::DeviceRadixSort::SortPairs(p->cub_tmp, bytes, p->vt_key, p->vt_key2, p->vt_pv, p->vt_pv2,
                                         n_el, 0, bits, st));
      k_segments<<<grid_for(n_el, 256, 148 * 8), 256, 0, st>>>(p->vt_key2, n_el, S, p->seg_b, p->seg_e);
      CKL("k_segments"); LAUNCHED(1);
    }
    k_vote_sum<4><<<grid_for(S, 4), 128, 0, st>>>(p->vt_pv2, p->seg_b, p->seg_e, S, g, (const double*)d_weights,
                                                   (const float*)d_weights, weight_mode, p->sums);
    CKL("k_vote_sum"); LAUNCHED(1);
  }
  CK(cudaMemsetAsync(p->counters + C_BAD, 0, sizeof(int), st));
  k_move_sites<<<grid_for(S, 128), 128, 0, st>>>(g, p->comp, p->site_pos, d_site_comp, p->sums, S, backoff,
                                                 p->new_pos, d_disp, p->counters + C_BAD);
  CKL("k_move_sites"); LAUNCHED(1);
  k_unpack_sites<<<grid_for(S, 256), 256, 0, st>>>(p->new_pos, S, d_new_pos);
  CKL("k_unpack_sites"); LAUNCHED(1);
  if (d_sums) CK(cudaMemcpyAsync(d_sums, p->sums, sizeof(double) * 4 * S, cudaMemcpyDeviceToDevice, st));
  CKR(sync_counters(p, st, C_BAD + 1));
  if (empty_regions) *empty_regions = p->h_counters[C_BAD];
  return 0;
}

int lrcvt_unpack_site_src(const int32_t* d_site_src, int64_t n, int32_t* d_site_of, int32_t* d_src,
                          void* stream) {
  if (!d_site_src || !d_site_of || !d_src || n < 0) return set_error(LRCVT_E_ARG, "lrcvt_unpack_site_src");
  if (n == 0) return 0;
  k_unpack_ss<<<grid_for(n, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const int2*>(d_site_src), n, d_site_of, d_src);
  CKL("k_unpack_ss"); LAUNCHED(1);
  return 0;
}

int lrcvt_segment_hit_t(int64_t nx, int64_t ny, int64_t nz, double sx, double sy, double sz,
                        const int32_t* d_comp, const double* d_segs, const int32_t* d_want, int64_t n,
                        double* d_t, void* stream) {
  if (!geo_ok(nx, ny, nz, sx, sy, sz) || !d_comp || n < 0 || (n > 0 && (!d_segs || !d_want || !d_t)))
    return set_error(LRCVT_E_ARG, "lrcvt_segment_hit_t: bad arguments");
  if (n == 0) return 0;
  Geo g = make_geo(nx, ny, nz, sx, sy, sz);
  k_segment_batch<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(g, d_comp, d_segs, d_want, n, d_t);
  CKL("k_segment_batch"); LAUNCHED(1);
  return 0;
}


int lrcvt_segment_clear_batch(lrcvt_plan* p, const double* d_segs, const int32_t* d_want, int64_t n,
                              uint8_t* d_clear, void* stream) {
  if (!p || n < 0 || (n > 0 && (!d_segs || !d_want || !d_clear)))
    return set_error(LRCVT_E_ARG, "lrcvt_segment_clear_batch: bad arguments");
  if (n == 0) return 0;
  k_segment_clear_batch<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(p->g, p->comp, p->nbm, d_segs, d_want,
                                                                           n, d_clear);
  CKL("k_segment_clear_batch"); LAUNCHED(1);
  return 0;
}

int lrcvt_isobands(int64_t n, const float* d_field, const double* d_iso, int32_t n_iso, int32_t* d_layer,
                   void* stream) {
  if (n < 0 || !d_field || !d_iso || !d_layer || n_iso < 2 || n_iso > 64)
    return set_error(LRCVT_E_ARG, "lrcvt_isobands: bad arguments");
  if (n == 0) return 0;
  if ((((uintptr_t)d_field) | ((uintptr_t)d_layer)) & 15)
    return set_error(LRCVT_E_ARG, "lrcvt_isobands: arrays must be 16-byte aligned");
  k_isobands<<<grid_for(n / 4 + 1, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(d_field, n, d_iso, n_iso,
                                                                                    d_layer);
  CKL("k_isobands"); LAUNCHED(1);
  return 0;
}

int lrcvt_label_components(int64_t nx, int64_t ny, int64_t nz, const int32_t* d_layer, int32_t n_layers,
                           int32_t* d_component, int32_t* n_components, void* stream) {
  retain_pool();
  if (!geo_ok(nx, ny, nz, 1, 1, 1) || !d_layer || !d_component || !n_components || n_layers < 0 ||
      n_layers > 64)
    return set_error(LRCVT_E_ARG, "lrcvt_label_components: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  Geo g = make_geo(nx, ny, nz, 1, 1, 1);
  const int64_t n = g.n;
  Scratch sc(st);
  int *L = nullptr, *local = nullptr, *cnt = nullptr;
  CK(sc.get(&L, n));
  CK(sc.get(&local, n));
  CK(sc.get(&cnt, 2));
  CK(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), st));
  // tile-local labelling in shared memory, then cross-tile unions on tile faces
  if (nz > 1) {
    const int64_t tiles = ((nx + 31) / 32) * ((ny + 3) / 4) * ((nz + 7) / 8);
    k_ccl_tile<32, 4, 8><<<(unsigned)tiles, 128, 0, st>>>(g, d_layer, n_layers, L, local, cnt);
    CKL("k_ccl_tile"); LAUNCHED(1);
    k_ccl_faces<32, 4, 8><<<(unsigned)tiles, 256, 0, st>>>(g, d_layer, n_layers, L);
    CKL("k_ccl_faces"); LAUNCHED(1);
  } else {
    const int64_t tiles = ((nx + 31) / 32) * ((ny + 15) / 16);
    k_ccl_tile<32, 16, 1><<<(unsigned)tiles, 512, 0, st>>>(g, d_layer, n_layers, L, local, cnt);
    CKL("k_ccl_tile"); LAUNCHED(1);
    k_ccl_faces<32, 16, 1><<<(unsigned)tiles, 256, 0, st>>>(g, d_layer, n_layers, L);
    CKL("k_ccl_faces"); LAUNCHED(1);
  }
  int h_cnt[2] = {0, 0};
  CK(cudaMemcpyAsync(h_cnt, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int n_local = h_cnt[0];
  if (n_local > 0) {
    unsigned long long *key = nullptr, *key2 = nullptr;
    void* tmp = nullptr;
    size_t bytes = 0;
    CK(sc.get(&key, n_local));
    CK(sc.get(&key2, n_local));
    k_ccl_root_keys<<<grid_for(n_local, 256), 256, 0, st>>>(local, n_local, L, d_layer, n_layers, key, cnt + 1);
    CKL("k_ccl_root_keys"); LAUNCHED(1);
    int bits = 32;
    while ((1ll << (bits - 31)) <= n_layers) bits++;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, key, key2, n_local, 0, bits, st));
    CK(sc.get((char**)&tmp, (int64_t)bytes));
    CK(cub::DeviceRadixSort::SortKeys(tmp, bytes, key, key2, n_local, 0, bits, st));
    k_ccl_compress_roots<<<grid_for(n_local, 256), 256, 0, st>>>(local, n_local, L);
    CKL("k_ccl_compress_roots"); LAUNCHED(1);
    k_ccl_root_ids<<<grid_for(n_local, 256), 256, 0, st>>>(key2, n_local, n_layers, L);
    CKL("k_ccl_root_ids"); LAUNCHED(1);
  }
  k_ccl_relabel<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(L, n, d_component,
                                                            ((uintptr_t)d_component & 15) == 0);
  CKL("k_ccl_relabel"); LAUNCHED(1);
  CK(cudaMemcpyAsync(h_cnt + 1, cnt + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *n_components = h_cnt[1];
  return 0;
}

int lrcvt_component_table(int64_t nx, int64_t ny, int64_t nz, const int32_t* d_component,
                          const int32_t* d_layer, int32_t n_components, uint64_t* d_count, int32_t* d_bbox,
                          int32_t* d_layer_of, void* stream) {
  if (!geo_ok(nx, ny, nz, 1, 1, 1) || !d_component || !d_layer || n_components < 0 ||
      (n_components > 0 && (!d_count || !d_bbox || !d_layer_of)))
    return set_error(LRCVT_E_ARG, "lrcvt_component_table: bad arguments");
  if (n_components == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  Geo g = make_geo(nx, ny, nz, 1, 1, 1);
  k_ccl_table_init<<<grid_for(n_components, 256), 256, 0, st>>>(n_components, (unsigned long long*)d_count,
                                                                d_bbox);
  CKL("k_ccl_table_init"); LAUNCHED(1);
  if (n_components <= TABLE_SMEM_COMP) {
    k_ccl_table_smem<<<grid_for(g.n, 256, 148 * 8), 256, 0, st>>>(
        g, d_component, d_layer, n_components, (unsigned long long*)d_count, d_bbox, d_layer_of);
    CKL("k_ccl_table_smem"); LAUNCHED(1);
  } else {
    k_ccl_table<<<grid_for(g.n, 256, 148 * 16), 256, 0, st>>>(g, d_component, d_layer,
                                                              (unsigned long long*)d_count, d_bbox, d_layer_of);
    CKL("k_ccl_table"); LAUNCHED(1);
  }
  return 0;
}


int lrcvt_aggregate(int64_t n, int32_t n_fields, const float* const* field_ptrs, const int32_t* d_component,
                    const int32_t* d_site_of, int32_t n_sites, int32_t n_components, int32_t n_pairs,
                    const int32_t* pairs, int32_t n_bins, double* axes, int64_t* d_count, double* d_sums,
                    double* d_minmax, int64_t* d_hist, void* stream) {
  retain_pool();
  if (n < 0 || n >= (int64_t(1) << 31) || n_fields < 1 || n_fields > 16 || !field_ptrs || !d_component ||
      !d_site_of || n_sites < 0 || n_components < 0 || n_pairs < 1 || n_pairs > 136 || !pairs || n_bins < 0 ||
      n_bins > 1024 || !d_count || !d_sums || !d_minmax || (n_bins > 0 && (!d_hist || !axes)))
    return set_error(LRCVT_E_ARG, "lrcvt_aggregate: bad arguments");
  for (int i = 0; i < 2 * n_pairs; i++)
    if (pairs[i] < 0 || pairs[i] >= n_fields) return set_error(LRCVT_E_ARG, "lrcvt_aggregate: bad pair");
  cudaStream_t st = (cudaStream_t)stream;
  const int n_cells = n_sites + n_components;
  if (n_cells == 0) return 0;
  Scratch sc(st);  // every scratch buffer is released on all exit paths
  int *inband = nullptr, *cnt = nullptr, *key = nullptr, *key2 = nullptr, *val = nullptr, *val2 = nullptr;
  int *segb = nullptr, *sege = nullptr, *d_pairs = nullptr;
  const float** d_fields = nullptr;
  const float** d_cols = nullptr;
  float* d_colbuf = nullptr;
  double* d_axes = nullptr;
  unsigned long long* d_lohi = nullptr;
  void* tmp = nullptr;
  size_t b1 = 0, b2 = 0;
  int h_cnt = 0;
  IsInband pred{d_component};
  cub::CountingInputIterator<int> it(0);
  CK(sc.raw((void**)&inband, sizeof(int) * (n > 0 ? n : 1)));
  CK(sc.raw((void**)&cnt, sizeof(int)));
  CK(cub::DeviceSelect::If(nullptr, b1, it, inband, cnt, (int)n, pred, st));
  CK(sc.raw((void**)&tmp, b1));
  CK(cub::DeviceSelect::If(tmp, b1, it, inband, cnt, (int)n, pred, st));
  CK(cudaMemcpyAsync(&h_cnt, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  tmp = nullptr;
  const int m = h_cnt;
  const int mm = m > 0 ? m : 1;
  CK(sc.raw((void**)&key, sizeof(int) * mm));
  CK(sc.raw((void**)&key2, sizeof(int) * mm));
  CK(sc.raw((void**)&val, sizeof(int) * mm));
  CK(sc.raw((void**)&val2, sizeof(int) * mm));
  CK(sc.raw((void**)&segb, sizeof(int) * n_cells));
  CK(sc.raw((void**)&sege, sizeof(int) * n_cells));
  CK(sc.raw((void**)&d_pairs, sizeof(int) * 2 * n_pairs));
  CK(sc.raw((void**)&d_fields, sizeof(float*) * n_fields));
  CK(cudaMemcpyAsync(d_pairs, pairs, sizeof(int) * 2 * n_pairs, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_fields, field_ptrs, sizeof(float*) * n_fields, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(segb, 0, sizeof(int) * n_cells, st));
  CK(cudaMemsetAsync(sege, 0, sizeof(int) * n_cells, st));
  if (m > 0) {
    k_agg_keys<<<grid_for(m, 256, 148 * 16), 256, 0, st>>>(inband, m, d_site_of, d_component, n_sites, key, val);
    CKL("k_agg_keys"); LAUNCHED(1);
    int bits = 1;
    while ((1ll << bits) <= n_cells) bits++;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, b2, key, key2, val, val2, m, 0, bits, st));
    CK(sc.raw((void**)&tmp, b2));
    CK(cub::DeviceRadixSort::SortPairs(tmp, b2, key, key2, val, val2, m, 0, bits, st));
    k_segments<<<grid_for(m, 256, 148 * 16), 256, 0, st>>>(key2, m, n_cells, segb, sege);
    CKL("k_segments"); LAUNCHED(1);
  }
  {
    // field columns in cell order (contiguous streams for the moment/histogram warps)
    CK(sc.raw((void**)&d_colbuf, sizeof(float) * (size_t)n_fields * (m > 0 ? m : 1)));
    CK(sc.raw((void**)&d_cols, sizeof(float*) * n_fields));
    {
      std::vector<const float*> cp(n_fields);
      for (int f = 0; f < n_fields; f++) cp[f] = d_colbuf + (size_t)f * (m > 0 ? m : 1);
      // pageable source: the copy is staged before cudaMemcpyAsync returns
      CK(cudaMemcpyAsync(d_cols, cp.data(), sizeof(float*) * n_fields, cudaMemcpyHostToDevice, st));
    }
    if (m > 0) {
      k_agg_gather<<<grid_for(m, 256, 148 * 16), 256, 0, st>>>(val2, m, d_fields, n_fields, d_colbuf);
      CKL("k_agg_gather"); LAUNCHED(1);
    }
    const int64_t warps = (int64_t)n_cells * n_pairs;
    k_agg_moments<<<grid_for(warps * 32, 128), 128, 0, st>>>(segb, sege, n_cells, d_cols, d_pairs,
                                                             n_pairs, (long long*)d_count, d_sums, d_minmax);
    CKL("k_agg_moments"); LAUNCHED(1);
  }
  if (n_bins > 0) {
    CK(sc.raw((void**)&d_axes, sizeof(double) * 2 * n_fields));
    bool any_auto = false;
    for (int f = 0; f < n_fields; f++) any_auto |= !(axes[2 * f] == axes[2 * f]) || !(axes[2 * f + 1] == axes[2 * f + 1]);
    if (any_auto) {  // stats.py:186-191 auto range over in-band values
      CK(sc.raw((void**)&d_lohi, sizeof(unsigned long long) * 2 * n_fields));
      std::vector<unsigned long long> init(2 * n_fields);
      for (int f = 0; f < n_fields; f++) { init[2 * f] = ~0ull; init[2 * f + 1] = 0ull; }
      CK(cudaMemcpyAsync(d_lohi, init.data(), sizeof(unsigned long long) * 2 * n_fields, cudaMemcpyHostToDevice, st));
      for (int f = 0; f < n_fields; f++) {
        if (m > 0) {
          k_field_range<<<grid_for(m, 256, 148 * 8), 256, 0, st>>>(inband, m, field_ptrs[f], d_lohi + 2 * f);
          CKL("k_field_range"); LAUNCHED(1);
        }
      }
      CK(cudaMemcpyAsync(init.data(), d_lohi, sizeof(unsigned long long) * 2 * n_fields, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int f = 0; f < n_fields; f++) {
        if (axes[2 * f] == axes[2 * f] && axes[2 * f + 1] == axes[2 * f + 1]) continue;
        double lo = 0.0, hi = 1.0;
        if (m > 0) {
          auto k2f = [](unsigned long long k) {
            const unsigned u = (unsigned)k;
            const unsigned bits = (u & 0x80000000u) ? (u ^ 0x80000000u) : ~u;
            float fv;
            memcpy(&fv, &bits, 4);
            return (double)fv;
          };
          lo = k2f(init[2 * f]);
          hi = k2f(init[2 * f + 1]);
        }
        if (hi <= lo) hi = lo + 1.0;  // stats.py:189-190
        axes[2 * f] = lo;
        axes[2 * f + 1] = hi;
      }
    }
    CK(cudaMemcpyAsync(d_axes, axes, sizeof(double) * 2 * n_fields, cudaMemcpyHostToDevice, st));
    const int64_t warps = (int64_t)n_cells * n_fields;
    k_agg_hist<1024><<<grid_for(warps * 32, 128), 128, 0, st>>>(segb, sege, n_cells, d_cols, n_fields,
                                                                d_axes, n_bins, (long long*)d_hist);
    CKL("k_agg_hist"); LAUNCHED(1);
  }
  CK(cudaStreamSynchronize(st));
  return 0;
}


// ---------------------------------------------------------------------------
// Multi-GPU global mode (mg.cuh): rank r owns planes [zlo, zhi)
// of one volume; own slab + one halo plane per side are current locally, far
// reads (shortcut nodes, phi chains) go to the owner through the PeerView.
// Per relaxation round: eval own frontier -> forward the proposals of the
// two boundary planes to the neighbour ranks -> commit own proposals + the
// received halo proposals (enqueue restricted to the own slab) -> global
// frontier count. The caller drives rounds and collectives (multigpu.py).

// a round with nothing to commit ends here (classify.cuh mg_round_end)
__global__ void k_mg_round_end(RoundCtl* ctl, int* counters, int sweep, volatile int* h_out) {
  mg_round_end(ctl, counters, sweep != 0, h_out);
}

// device time of an mg step that ends in a host synchronisation: events
// around its kernels (the host round trip of the sync is not counted)
void mg_t0(lrcvt_plan* p, cudaStream_t st) {
  if (p->mg_timing) cudaEventRecord(p->mg_ev[0], st);
}
int mg_sync(lrcvt_plan* p, cudaStream_t st, int n) {
  if (p->mg_timing) CK(cudaEventRecord(p->mg_ev[1], st));
  CKR(sync_counters(p, st, n));
  if (p->mg_timing) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p->mg_ev[0], p->mg_ev[1]));
    p->mg_ms += ms;
  }
  return 0;
}

// the same for a step that does not synchronise (timing mode only waits for its end event)
int mg_t1(lrcvt_plan* p, cudaStream_t st) {
  if (!p->mg_timing) return 0;
  CK(cudaEventRecord(p->mg_ev[1], st));
  CK(cudaEventSynchronize(p->mg_ev[1]));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, p->mg_ev[0], p->mg_ev[1]));
  p->mg_ms += ms;
  return 0;
}

int lrcvt_mg_set_slab(lrcvt_plan* p, int64_t zlo, int64_t zhi) {
  if (!p || zlo < 0 || zhi <= zlo || zlo >= p->g.nz) return set_error(LRCVT_E_ARG, "lrcvt_mg_set_slab");
  p->zlo = (int)zlo;
  p->zhi = zhi >= p->g.nz ? p->g.nz : (int)zhi;  // kernels filter iff zlo > 0 || zhi < nz
  p->eligible_valid = false;
  return 0;
}

int lrcvt_mg_state(lrcvt_plan* p, void** d_ss, void** d_dist) {
  if (!p || !d_ss || !d_dist) return set_error(LRCVT_E_ARG, "lrcvt_mg_state");
  if (!p->mg_own_ss) {
    int rc = dalloc(&p->mg_own_ss, p->g.n);
    rc |= dalloc(&p->mg_own_dist, p->g.n);
    if (rc) return LRCVT_E_NOMEM;
  }
  *d_ss = p->mg_own_ss;
  *d_dist = p->mg_own_dist;
  return 0;
}

int lrcvt_mg_set_peers(lrcvt_plan* p, int32_t world, const int64_t* z_bounds, void* const* peer_ss,
                       void* const* peer_dist) {
  if (!p || world < 1 || world > MG_MAX || !z_bounds || !peer_ss || !peer_dist)
    return set_error(LRCVT_E_ARG, "lrcvt_mg_set_peers: bad arguments");
  PeerView pv;
  memset(&pv, 0, sizeof pv);
  pv.world = world;
  pv.nxy = p->g.nxy;
  for (int r = 0; r <= world; r++) pv.zb[r] = (int)z_bounds[r];
  for (int r = world + 1; r <= MG_MAX; r++) pv.zb[r] = p->g.nz;
  for (int r = 0; r < world; r++) {
    pv.ss[r] = (const int2*)peer_ss[r];
    pv.dist[r] = (const double*)peer_dist[r];
    if (z_bounds[r + 1] <= z_bounds[r]) return set_error(LRCVT_E_ARG, "lrcvt_mg_set_peers: empty slab");
  }
  pv.lo = p->zlo - 1;
  pv.hi = p->zhi;
  if (!p->d_pv) CK(cudaMalloc((void**)&p->d_pv, sizeof(PeerView)));
  CK(cudaMemcpy(p->d_pv, &pv, sizeof pv, cudaMemcpyHostToDevice));
  p->mg_world = world;
  return 0;
}

int lrcvt_mg_begin(lrcvt_plan* p, int64_t n_sites, const double* d_site_pos, const int32_t* d_site_comp,
                   int32_t* d_site_src, double* d_dist, int64_t* n_frontier, void* stream) {
  if (!p || n_sites < 1 || n_sites > p->max_sites || !d_site_pos || !d_site_comp || !d_site_src || !d_dist ||
      !n_frontier)
    return set_error(LRCVT_E_ARG, "lrcvt_mg_begin: bad arguments");
  retain_pool();
  cudaStream_t st = (cudaStream_t)stream;
  const Geo& g = p->g;
  const int S = (int)n_sites;
  int2* ss = reinterpret_cast<int2*>(d_site_src);
  p->mg_ss = ss;
  p->mg_dist = d_dist;
  if (!p->mg_lo) {
    int rc = dalloc(&p->mg_lo, g.nxy);
    rc |= dalloc(&p->mg_hi, g.nxy);
    if (rc) return LRCVT_E_NOMEM;
  }
  mg_t0(p, st);
  {  // the eval kernels' halo output (classify.cuh BoundaryOut): planes zlo / zhi - 1 when a neighbour exists
    BoundaryOut bo;
    bo.lo = p->mg_lo;
    bo.hi = p->mg_hi;
    bo.counters = p->counters;
    bo.zlo = p->zlo > 0 ? p->zlo : -1;
    bo.zhi = p->zhi < g.nz ? p->zhi : INT_MAX;
    bo.nxy = (int)g.nxy;
    CK(cudaMemcpyAsync(&p->ctl->bo, &bo, sizeof bo, cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemsetAsync(p->counters, 0, sizeof(int) * C_NCOUNTERS, st));
  // own-slab eligible list (tessellation.py:161-164 restricted to [zlo, zhi)); kept across a Lloyd loop
  // whose site components do not change (lrcvt_plan_reuse_eligible)
  if (!(p->reuse_eligible && p->eligible_valid && p->eligible_sites == S)) {
    if (prepare_eligible(p, S, d_site_comp, st)) return LRCVT_E_CUDA;
    p->eligible_valid = true;
    p->eligible_sites = S;
  }
  // the rank's kernels read its own ss / dist / site1 only on the slab and its halo planes [z0, z1)
  // (mg.cuh: everything else through the owner's buffers)
  {
    const int64_t z0 = p->zlo > 0 ? p->zlo - 1 : 0, z1 = p->zhi < g.nz ? p->zhi + 1 : g.nz;
    const int64_t v0 = z0 * g.nxy, nv = (z1 - z0) * g.nxy;
    k_fill_state<<<grid_for(nv, 256, 148 * 32), 256, 0, st>>>(ss + v0, d_dist + v0, nv);
    CKL("k_fill_state");
    CK(cudaMemsetAsync(p->site1 + v0, 0xff, sizeof(int) * (size_t)nv, st));
  }
  k_pack_sites<<<grid_for(S, 256), 256, 0, st>>>(d_site_pos, S, p->site_pos);
  CKL("k_pack_sites");
  // every rank validates every site and places the seeds on its slab and halo planes; the phase-1
  // worklist holds the own slab's part only
  k_site_voxel<<<grid_for(S, 256), 256, 0, st>>>(g, p->comp, p->site_pos, d_site_comp, S, p->sk_key, p->sk_d,
                                                 p->site1, p->counters, p->zlo, p->zhi);
  CKL("k_site_voxel");
  k_seed_groups<<<grid_for(S, 128), 128, 0, st>>>(g, p->nbm, p->sk_key, p->sk_d, S, ss, d_dist, p->site1, p->bm,
                                                  p->list_a, p->sk_coll, p->counters, p->zlo, p->zhi);
  CKL("k_seed_groups");
  k_seed_collisions<<<1, SEED_COLL_THREADS, 0, st>>>(p->sk_coll, p->sk_d, ss, d_dist, p->site1, p->counters);
  CKL("k_seed_collisions");
  k_phase1_start<<<1, 1, 0, st>>>(p->ctl, p->counters, p->list_a, p->list_b, ss, d_dist, p->site1, 0);
  CKL("k_phase1_start");
  CK(cudaMemcpyAsync(p->h_ctl, p->ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, st));
  CKR(mg_sync(p, st, C_NCOUNTERS));
  if (p->h_counters[C_BAD]) return p->h_counters[C_BAD];
  p->h_ncur = p->h_ctl->n_cur;
  *n_frontier = p->h_ncur;
  return 0;
}

int lrcvt_mg_phase2(lrcvt_plan* p, int64_t n_sites, const int32_t* d_site_comp, int64_t* n_frontier, void* stream) {
  if (!p || !d_site_comp || !n_frontier || !p->eligible_valid) return set_error(LRCVT_E_ARG, "lrcvt_mg_phase2");
  cudaStream_t st = (cudaStream_t)stream;
  const Geo& g = p->g;
  // phase-1 LOS states -> (site, src) / dist on the own slab and its halo planes (site1 is current there)
  mg_t0(p, st);
  const int64_t z0 = p->zlo > 0 ? p->zlo - 1 : 0, z1 = p->zhi < g.nz ? p->zhi + 1 : g.nz;
  k_site1_to_state<<<grid_for((z1 - z0) * g.nxy, 256, 148 * 16), 256, 0, st>>>(
      g, p->site1, p->site_pos, p->mg_ss, p->mg_dist, nullptr, nullptr, z0 * g.nxy, z1 * g.nxy);
  CKL("k_site1_to_state");
  k_phase2_copy<<<1, 1, 0, st>>>(p->eligible, p->d_nel, p->ctl, p->counters);
  CKL("k_phase2_copy");
  CK(cudaMemcpyAsync(p->h_counters + H_NEL, p->d_nel, sizeof(int), cudaMemcpyDeviceToHost, st));
  CKR(mg_sync(p, st, 1));
  p->n_eligible = p->h_counters[H_NEL];
  p->h_ncur = (int)p->n_eligible;
  *n_frontier = p->h_ncur;
  return 0;
}

int lrcvt_mg_eval(lrcvt_plan* p, int32_t phase, int32_t sweep, int64_t* n_evaluated, int64_t* n_lo,
                  int64_t* n_hi, void* stream) {
  if (!p || phase < 1 || phase > 2 || !n_evaluated || !n_lo || !n_hi || !p->mg_lo)
    return set_error(LRCVT_E_ARG, "lrcvt_mg_eval");
  cudaStream_t st = (cudaStream_t)stream;
  int n = p->h_ncur;
  mg_t0(p, st);
  if (sweep) {
    k_sweep_start<<<1, 1, 0, st>>>(p->ctl, p->eligible, p->d_nel, p->counters);
    CKL("k_sweep_start");
    n = (int)p->n_eligible;
  }
  // the per-round counters are zero here: reset by the last round end / begin / phase-2 start
  const int var = phase == 1 ? 0 : (p->g.dyadic ? 1 : 2);
  if (n > 0) CKR(launch_eval_kernel(p, var, n, st));  // + the boundary-plane proposals (ctl->bo)
  CKR(mg_sync(p, st, C_HI + 1));
  *n_evaluated = n;
  *n_lo = p->h_counters[C_LO];
  *n_hi = p->h_counters[C_HI];
  return 0;
}

void* lrcvt_mg_boundary(lrcvt_plan* p, int32_t side) {
  if (!p) return nullptr;
  return side == 0 ? (void*)p->mg_lo : (void*)p->mg_hi;
}

int lrcvt_mg_commit(lrcvt_plan* p, const void* d_halo, int64_t n_halo, int32_t sweep, int64_t* n_next,
                    int64_t* n_committed, void* stream) {
  if (!p || n_halo < 0 || (n_halo > 0 && !d_halo) || !n_next || !n_committed)
    return set_error(LRCVT_E_ARG, "lrcvt_mg_commit");
  cudaStream_t st = (cudaStream_t)stream;
  mg_t0(p, st);
  // one launch: the own sparse proposals, then the received halo-plane proposals
  const int n = sweep ? (int)p->n_eligible : p->h_ncur;
  int64_t own_blocks = n > 0 ? (n + CM_SLOTS - 1) / CM_SLOTS : 0;
  int64_t halo_blocks = n_halo > 0 ? (n_halo + CM_THREADS - 1) / CM_THREADS : 0;
  if (own_blocks > p->commit_blocks) own_blocks = p->commit_blocks;
  if (halo_blocks > p->commit_blocks) halo_blocks = p->commit_blocks;
  if (own_blocks + halo_blocks > 0) {  // its last block ends the round (classify.cuh mg_round_end)
    k_commit<<<(int)(own_blocks + halo_blocks), CM_THREADS, 0, st>>>(
        p->imp, p->pf, 0, p->counters, p->ctl, p->g, p->nbm, p->bm, p->compact ? p->cbm : nullptr, nullptr,
        p->ncl_arg(), cudaGraphConditionalHandle{}, sweep ? END_MG_SWEEP : END_MG, p->zlo, p->zhi,
        (const Prop*)d_halo, (int)n_halo, (int)own_blocks, p->h_counters_dev);
    CKL("k_commit");
  } else {
    k_mg_round_end<<<1, 1, 0, st>>>(p->ctl, p->counters, sweep, p->h_counters_dev);
    CKL("k_mg_round_end");
  }
  CKR(mg_sync(p, st, 0));
  const int nn = p->h_counters[C_NNEXT];
  p->h_ncur = nn;
  *n_next = nn;
  *n_committed = p->h_counters[C_NIMP];
  return 0;
}

int lrcvt_mg_finish(lrcvt_plan* p, const int32_t* d_site_src, uint8_t* d_state, int64_t* assigned, void* stream) {
  if (!p || !d_site_src || !assigned) return set_error(LRCVT_E_ARG, "lrcvt_mg_finish");
  cudaStream_t st = (cudaStream_t)stream;
  const Geo& g = p->g;
  mg_t0(p, st);
  CK(cudaMemsetAsync(p->counters + C_ASSIGNED, 0, sizeof(int), st));
  const int64_t v0 = (int64_t)p->zlo * g.nxy, v1 = (int64_t)(p->zhi < g.nz ? p->zhi : g.nz) * g.nxy;
  k_state<<<grid_for(v1 - v0, 256, 148 * 16), 256, 0, st>>>(reinterpret_cast<const int2*>(d_site_src), nullptr,
                                                             nullptr, v0, v1, d_state, p->counters);
  CKL("k_state");
  CKR(mg_sync(p, st, C_ASSIGNED + 1));
  *assigned = p->h_counters[C_ASSIGNED];
  return 0;
}

// ---- vote on the own slab (tessellation.py:211-248 partitioned)

int lrcvt_mg_vote_exact(lrcvt_plan* p, int64_t n_sites, const int32_t* d_site_src, uint64_t* d_acc, void* stream) {
  if (!p || n_sites < 1 || n_sites > p->max_sites || !d_site_src || !d_acc || !p->eligible_valid)
    return set_error(LRCVT_E_ARG, "lrcvt_mg_vote_exact");
  cudaStream_t st = (cudaStream_t)stream;
  const int S = (int)n_sites;
  mg_t0(p, st);
  CK(cudaMemsetAsync(d_acc, 0, sizeof(uint64_t) * 4 * S, st));
  const int n_el = (int)p->n_eligible;
  if (n_el > 0) {
    const int2* ss = reinterpret_cast<const int2*>(d_site_src);
    if (p->d_pv)
      k_vote_exact<true><<<grid_for(n_el, 256, 148 * 8), 256, 0, st>>>(p->eligible, n_el, p->g, ss,
                                                                       (unsigned long long*)d_acc, S, p->d_pv);
    else
      k_vote_exact<false><<<grid_for(n_el, 256, 148 * 8), 256, 0, st>>>(p->eligible, n_el, p->g, ss,
                                                                        (unsigned long long*)d_acc, S, nullptr);
    CKL("k_vote_exact");
  }
  return mg_t1(p, st);
}

int lrcvt_mg_vote_exact_finish(lrcvt_plan* p, int64_t n_sites, const uint64_t* d_acc, double* d_sums, void* stream) {
  if (!p || n_sites < 1 || !d_acc || !d_sums) return set_error(LRCVT_E_ARG, "lrcvt_mg_vote_exact_finish");
  const int S = (int)n_sites;
  const Geo& g = p->g;
  mg_t0(p, (cudaStream_t)stream);
  k_vote_exact_finish<<<grid_for(S, 256), 256, 0, (cudaStream_t)stream>>>((const unsigned long long*)d_acc, S,
                                                                          0.5 * g.sx, 0.5 * g.sy, 0.5 * g.sz, d_sums);
  CKL("k_vote_exact_finish");
  return mg_t1(p, (cudaStream_t)stream);
}

int lrcvt_mg_vote_box(lrcvt_plan* p, int64_t n_sites, const int32_t* d_site_src, int32_t* d_box, void* stream) {
  if (!p || n_sites < 1 || n_sites > p->max_sites || !d_site_src || !d_box || !p->eligible_valid)
    return set_error(LRCVT_E_ARG, "lrcvt_mg_vote_box");
  cudaStream_t st = (cudaStream_t)stream;
  const int S = (int)n_sites;
  mg_t0(p, st);
  CKR(vote_buffers(p, st));
  k_box_init<<<grid_for(S, 256), 256, 0, st>>>(d_box, S);
  CKL("k_box_init");
  const int n_el = (int)p->n_eligible;
  if (n_el > 0) {
    const int2* ss = reinterpret_cast<const int2*>(d_site_src);
    if (p->d_pv)
      k_vote_prep<true><<<grid_for(n_el, 256, 148 * 8), 256, 0, st>>>(p->eligible, n_el, p->g, ss, p->vt_sp, d_box,
                                                                      S, p->d_pv);
    else
      k_vote_prep<false><<<grid_for(n_el, 256, 148 * 8), 256, 0, st>>>(p->eligible, n_el, p->g, ss, p->vt_sp,
                                                                       d_box, S, nullptr);
    CKL("k_vote_prep");
  }
  return mg_t1(p, st);
}

int lrcvt_mg_vote_scan(lrcvt_plan* p, int64_t n_sites, const int32_t* d_site_comp, int32_t weight_mode,
                       const void* d_weights, int32_t mode, const int32_t* d_box, const double* d_init, double* d_out,
                       void* stream) {
  if (!p || n_sites < 1 || !d_site_comp || !d_box || !d_out || mode < 0 || mode > 2 || !p->vt_sp ||
      weight_mode < 0 || weight_mode > 3 || (weight_mode != LRCVT_W_ONES && !d_weights) || (mode == 2 && !d_init))
    return set_error(LRCVT_E_ARG, "lrcvt_mg_vote_scan");
  const int S = (int)n_sites;
  const Geo& g = p->g;
  mg_t0(p, (cudaStream_t)stream);
  CKR(vote_chains(p, d_box, S, weight_mode, d_weights, p->zlo, p->zhi < g.nz ? p->zhi : (int)g.nz, mode, d_init,
                  d_out, (cudaStream_t)stream));
  return mg_t1(p, (cudaStream_t)stream);
}

int lrcvt_mg_vote_carry(lrcvt_plan* p, int64_t n_sites, const int32_t* d_box, const double* d_res,
                        const double* d_carry_in, double* d_carry_out, void* stream) {
  if (!p || n_sites < 1 || !d_box || !d_res || !d_carry_out) return set_error(LRCVT_E_ARG, "lrcvt_mg_vote_carry");
  const int S = (int)n_sites;
  mg_t0(p, (cudaStream_t)stream);
  k_vote_carry<<<grid_for(S, 256), 256, 0, (cudaStream_t)stream>>>(d_box, S, p->zlo,
                                                                   p->zhi < p->g.nz ? p->zhi : p->g.nz, d_res,
                                                                   d_carry_in, d_carry_out);
  CKL("k_vote_carry");
  return mg_t1(p, (cudaStream_t)stream);
}

int lrcvt_mg_move(lrcvt_plan* p, int64_t n_sites, const double* d_site_pos, const int32_t* d_site_comp,
                  const double* d_sums, double backoff, double* d_new_pos, double* d_disp, int64_t* empty_regions,
                  void* stream) {
  if (!p || n_sites < 1 || n_sites > p->max_sites || !d_site_pos || !d_site_comp || !d_sums || !d_new_pos ||
      !d_disp)
    return set_error(LRCVT_E_ARG, "lrcvt_mg_move");
  cudaStream_t st = (cudaStream_t)stream;
  const int S = (int)n_sites;
  mg_t0(p, st);
  k_pack_sites<<<grid_for(S, 256), 256, 0, st>>>(d_site_pos, S, p->site_pos);
  CKL("k_pack_sites");
  CK(cudaMemsetAsync(p->counters + C_BAD, 0, sizeof(int), st));
  k_move_sites<<<grid_for(S, 128), 128, 0, st>>>(p->g, p->comp, p->site_pos, d_site_comp, d_sums, S, backoff,
                                                 p->new_pos, d_disp, p->counters + C_BAD);
  CKL("k_move_sites");
  k_unpack_sites<<<grid_for(S, 256), 256, 0, st>>>(p->new_pos, S, d_new_pos);
  CKL("k_unpack_sites");
  CKR(mg_sync(p, st, C_BAD + 1));
  if (empty_regions) *empty_regions = p->h_counters[C_BAD];
  return 0;
}

int lrcvt_mg_timing(lrcvt_plan* p, int32_t enable, double* ms) {
  if (!p) return set_error(LRCVT_E_ARG, "lrcvt_mg_timing");
  if (ms) *ms = p->mg_ms;
  p->mg_ms = 0.0;
  if (enable && !p->mg_ev[0]) {
    CK(cudaEventCreate(&p->mg_ev[0]));
    CK(cudaEventCreate(&p->mg_ev[1]));
  }
  p->mg_timing = enable != 0;
  return 0;
}

// ---- CUDA IPC: another process's (or device's) buffers as peer pointers

int lrcvt_ipc_export(const void* d_ptr, uint8_t* handle64) {
  if (!d_ptr || !handle64) return set_error(LRCVT_E_ARG, "lrcvt_ipc_export");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
  memcpy(handle64, &h, sizeof h < 64 ? sizeof h : 64);
  return 0;
}

int lrcvt_ipc_open(const uint8_t* handle64, void** d_ptr) {
  if (!handle64 || !d_ptr) return set_error(LRCVT_E_ARG, "lrcvt_ipc_open");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h < 64 ? sizeof h : 64);
  CK(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return 0;
}

int lrcvt_ipc_close(void* d_ptr) {
  if (!d_ptr) return set_error(LRCVT_E_ARG, "lrcvt_ipc_close");
  CK(cudaIpcCloseMemHandle(d_ptr));
  return 0;
}


int lrcvt_seed_masses(int64_t nx, int64_t ny, int64_t nz, int32_t block_size, const int32_t* d_component,
                      int32_t n_components, int32_t weight_mode, const void* d_weights, int64_t max_inband,
                      int64_t max_runs, int32_t* d_voxels, double* d_weights_sorted, int64_t* d_run_key,
                      int64_t* d_run_start, int64_t* d_run_len, double* d_run_mass, int64_t* n_inband,
                      int64_t* n_runs, double* total_mass, void* stream) {
  retain_pool();
  const int64_t n = nx * ny * nz;
  if (nx < 1 || ny < 1 || nz < 1 || n >= (int64_t(1) << 31) || block_size < 1 || !d_component ||
      n_components < 0 || weight_mode < 0 || weight_mode > 3 || (weight_mode != LRCVT_W_ONES && !d_weights) ||
      !d_voxels || !d_run_key || !d_run_start || !d_run_len || !d_run_mass || !n_inband || !n_runs ||
      !total_mass)
    return set_error(LRCVT_E_ARG, "lrcvt_seed_masses: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  *n_inband = 0;
  *n_runs = 0;
  *total_mass = 0.0;
  const int64_t bs = block_size;
  const int64_t nbx = (nx + bs - 1) / bs, nby = (ny + bs - 1) / bs, nbz = (nz + bs - 1) / bs;
  const int64_t n_blocks = nbx * nby * nbz;
  SeedWeight w{weight_mode, (const double*)d_weights, (const float*)d_weights};
  if (weight_mode == LRCVT_W_ONES) w.w64 = nullptr, w.w32 = nullptr;
  Scratch sc(st);
  int* list = nullptr;
  int* cnt = nullptr;
  void* tmp = nullptr;
  size_t b = 0;
  CK(sc.get(&list, n));
  CK(sc.get(&cnt, 1));
  cub::CountingInputIterator<int> it(0);
  IsInband pred{d_component};
  CK(cub::DeviceSelect::If(nullptr, b, it, list, cnt, (int)n, pred, st));
  CK(sc.get((char**)&tmp, (int64_t)b));
  CK(cub::DeviceSelect::If(tmp, b, it, list, cnt, (int)n, pred, st));
  int h_cnt = 0;
  CK(cudaMemcpyAsync(&h_cnt, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int64_t m = h_cnt;
  *n_inband = m;
  if (m > max_inband) return set_error(LRCVT_E_ARG, "lrcvt_seed_masses: max_inband too small");
  if (m == 0) return 0;
  unsigned long long *key = nullptr, *key2 = nullptr;
  int64_t* nr = nullptr;
  int64_t *rk = nullptr, *rl = nullptr;
  double* ws = d_weights_sorted;
  CK(sc.get(&key, m));
  CK(sc.get(&key2, m));
  CK(sc.get(&nr, 1));
  CK(sc.get(&rk, m));
  CK(sc.get(&rl, m));
  if (!ws) CK(sc.get(&ws, m));
  k_seed_keys<<<grid_for(m, 256, 148 * 16), 256, 0, st>>>(list, m, d_component, (int)nx, (int)ny, (int)bs, nbx,
                                                          nby, n_blocks, key);
  CKL("k_seed_keys"); LAUNCHED(1);
  int bits = 1;
  const unsigned long long kmax = (unsigned long long)(n_components > 0 ? n_components : 1) * n_blocks;
  while (bits < 64 && (1ull << bits) < kmax) bits++;
  b = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, b, key, key2, list, d_voxels, (int)m, 0, bits, st));
  void* tmp2 = nullptr;
  CK(sc.get((char**)&tmp2, (int64_t)b));
  CK(cub::DeviceRadixSort::SortPairs(tmp2, b, key, key2, list, d_voxels, (int)m, 0, bits, st));
  // group boundaries (unique keys + lengths)
  b = 0;
  CK(cub::DeviceRunLengthEncode::Encode(nullptr, b, key2, (unsigned long long*)rk, rl, nr, (int)m, st));
  void* tmp3 = nullptr;
  CK(sc.get((char**)&tmp3, (int64_t)b));
  CK(cub::DeviceRunLengthEncode::Encode(tmp3, b, key2, (unsigned long long*)rk, rl, nr, (int)m, st));
  // total mass in voxel order: subtrees on the device, joined on the host
  std::vector<int64_t> tl, tn;
  pw_split(0, m, tl, tn);
  const int nt = (int)tl.size();
  int64_t *d_tl = nullptr, *d_tn = nullptr;
  double* d_tv = nullptr;
  CK(sc.get(&d_tl, nt));
  CK(sc.get(&d_tn, nt));
  CK(sc.get(&d_tv, nt));
  CK(cudaMemcpyAsync(d_tl, tl.data(), sizeof(int64_t) * nt, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_tn, tn.data(), sizeof(int64_t) * nt, cudaMemcpyHostToDevice, st));
  k_seed_subtrees<<<grid_for(nt, 128), 128, 0, st>>>(list, w, d_tl, d_tn, nt, d_tv);
  CKL("k_seed_subtrees"); LAUNCHED(1);
  k_seed_weights<<<grid_for(m, 256, 148 * 16), 256, 0, st>>>(d_voxels, m, w, ws);
  CKL("k_seed_weights"); LAUNCHED(1);
  int64_t h_nr = 0;
  std::vector<double> tv(nt);
  CK(cudaMemcpyAsync(&h_nr, nr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(tv.data(), d_tv, sizeof(double) * nt, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  size_t k = 0;
  *total_mass = 0.0 + pw_join(m, tv, k);
  *n_runs = h_nr;
  if (h_nr > max_runs) return set_error(LRCVT_E_ARG, "lrcvt_seed_masses: max_runs too small");
  b = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, b, rl, d_run_start, (int)h_nr, st));
  void* tmp4 = nullptr;
  CK(sc.get((char**)&tmp4, (int64_t)b));
  CK(cub::DeviceScan::ExclusiveSum(tmp4, b, rl, d_run_start, (int)h_nr, st));
  CK(cudaMemcpyAsync(d_run_key, rk, sizeof(int64_t) * h_nr, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(d_run_len, rl, sizeof(int64_t) * h_nr, cudaMemcpyDeviceToDevice, st));
  k_seed_run_mass_warp<4><<<grid_for(h_nr, 4), 128, 0, st>>>(ws, d_run_start, d_run_len, h_nr, d_run_mass);
  CKL("k_seed_run_mass_warp"); LAUNCHED(1);
  CK(cudaStreamSynchronize(st));
  return 0;
}

int lrcvt_layout_records(int64_t nx, int64_t ny, int64_t nz, int32_t n_fields, const float* const* field_ptrs,
                         const int32_t* d_component, const int32_t* d_site_of, int32_t n_components,
                         int32_t n_sites, int64_t max_records, void* d_records, uint32_t* d_region_key, int64_t* d_comp_first,
                         int64_t* d_comp_count, int64_t* n_records, void* stream) {
  retain_pool();
  const int64_t n = nx * ny * nz;
  if (nx < 1 || ny < 1 || nz < 1 || n >= (int64_t(1) << 31) || n_fields < 0 || n_fields > 16 ||
      (n_fields > 0 && !field_ptrs) || !d_component || !d_site_of || n_components < 0 || n_sites < 0 || !d_records ||
      !d_region_key || (n_components > 0 && (!d_comp_first || !d_comp_count)) || !n_records)
    return set_error(LRCVT_E_ARG, "lrcvt_layout_records: bad arguments");
  FieldPtrs fp{};
  for (int i = 0; i < n_fields; i++) {
    if (!field_ptrs[i]) return set_error(LRCVT_E_ARG, "lrcvt_layout_records: null field");
    fp.f[i] = field_ptrs[i];
  }
  cudaStream_t st = (cudaStream_t)stream;
  *n_records = 0;
  Scratch sc(st);
  int *list = nullptr, *cnt = nullptr, *vox = nullptr;
  void* tmp = nullptr;
  size_t b = 0;
  CK(sc.get(&list, n));
  CK(sc.get(&cnt, 1));
  cub::CountingInputIterator<int> it(0);
  IsInband pred{d_component};
  CK(cub::DeviceSelect::If(nullptr, b, it, list, cnt, (int)n, pred, st));
  CK(sc.get((char**)&tmp, (int64_t)b));
  CK(cub::DeviceSelect::If(tmp, b, it, list, cnt, (int)n, pred, st));
  int h_cnt = 0;
  CK(cudaMemcpyAsync(&h_cnt, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (n_components > 0) {
    CK(cudaMemsetAsync(d_comp_first, 0, sizeof(int64_t) * n_components, st));
    CK(cudaMemsetAsync(d_comp_count, 0, sizeof(int64_t) * n_components, st));
  }
  CK(cudaStreamSynchronize(st));
  const int64_t r = h_cnt;
  *n_records = r;
  if (r > max_records) return set_error(LRCVT_E_ARG, "lrcvt_layout_records: max_records too small");
  if (r == 0) return 0;
  CK(sc.get(&vox, r));
  int rbits = 1, cbits = 1;
  while ((1ll << rbits) <= (int64_t)n_sites) rbits++;  // codes 0..n_sites
  while ((1ll << cbits) < (int64_t)n_components) cbits++;
  int* bad = nullptr;
  CK(sc.get(&bad, 1));
  CK(cudaMemsetAsync(bad, 0, sizeof(int), st));
  auto run = [&](auto* key, auto* key2) -> int {
    using K = std::remove_pointer_t<decltype(key)>;
    k_layout_keys<K><<<grid_for(r, 256, 148 * 16), 256, 0, st>>>(list, r, d_component, d_site_of, n_sites, rbits,
                                                                  key, bad);
    CKL("k_layout_keys"); LAUNCHED(1);
    size_t bb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bb, key, key2, list, vox, (int)r, 0, rbits + cbits, st));
    void* t2 = nullptr;
    CK(sc.get((char**)&t2, (int64_t)bb));
    CK(cub::DeviceRadixSort::SortPairs(t2, bb, key, key2, list, vox, (int)r, 0, rbits + cbits, st));
    k_layout_pack<<<grid_for(r * (3 + n_fields), 256, 148 * 32), 256, 0, st>>>(vox, r, n_fields, (int)nx, (int)ny,
                                                                                fp, (unsigned*)d_records);
    CKL("k_layout_pack"); LAUNCHED(1);
    k_layout_index<K><<<grid_for(r, 256, 148 * 16), 256, 0, st>>>(key2, r, rbits, n_sites, d_region_key,
                                                                   n_components, (long long*)d_comp_first,
                                                                   (long long*)d_comp_count);
    CKL("k_layout_index"); LAUNCHED(1);
    return 0;
  };
  if (rbits + cbits <= 32) {
    unsigned *key = nullptr, *key2 = nullptr;
    CK(sc.get(&key, r));
    CK(sc.get(&key2, r));
    CKR(run(key, key2));
  } else {
    unsigned long long *key = nullptr, *key2 = nullptr;
    CK(sc.get(&key, r));
    CK(sc.get(&key2, r));
    CKR(run(key, key2));
  }
  if (n_components > 0) {
    k_layout_counts<<<grid_for(n_components, 256), 256, 0, st>>>(n_components, (const long long*)d_comp_first,
                                                                 (long long*)d_comp_count);
    CKL("k_layout_counts"); LAUNCHED(1);
  }
  int h_bad = 0;
  CK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h_bad) return set_error(LRCVT_E_ARG, "lrcvt_layout_records: site_of holds an id >= n_sites");
  return 0;
}

int lrcvt_region_adjacency(int64_t nx, int64_t ny, int64_t nz, const int32_t* d_site_of,
                           const int32_t* d_component, int64_t n_sites, int64_t max_edges, int64_t* d_edges,
                           int64_t* n_edges, void* stream) {
  retain_pool();
  if (!geo_ok(nx, ny, nz, 1, 1, 1) || !d_site_of || !d_component || n_sites < 0 || max_edges < 0 ||
      (max_edges > 0 && !d_edges) || !n_edges)
    return set_error(LRCVT_E_ARG, "lrcvt_region_adjacency: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  *n_edges = 0;
  Geo g = make_geo(nx, ny, nz, 1, 1, 1);
  // 3D Voronoi cells have ~14 face neighbours: 16 slots per site keeps the
  // set under half full
  unsigned long long slots = 1024;
  while (slots < (unsigned long long)(16 * n_sites) && slots < (1ull << 34)) slots <<= 1;
  Scratch sc(st);
  unsigned long long *table = nullptr, *keys = nullptr, *keys2 = nullptr;
  int* cnt = nullptr;
  CK(sc.get(&cnt, 2));
  for (;;) {
    CK(sc.get(&table, (int64_t)slots));
    CK(cudaMemsetAsync(table, 0xff, sizeof(unsigned long long) * slots, st));
    CK(cudaMemsetAsync(cnt + 1, 0, sizeof(int), st));
    k_adjacency<<<grid_for(g.n, 256, 148 * 8), 256, 0, st>>>(g, d_site_of, d_component, table, slots - 1,
                                                             cnt + 1);
    CKL("k_adjacency"); LAUNCHED(1);
    int overflow = 0;
    CK(cudaMemcpyAsync(&overflow, cnt + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!overflow) break;
    if (slots >= (1ull << 34)) return set_error(LRCVT_E_NOMEM, "lrcvt_region_adjacency: edge set too large");
    slots <<= 2;
  }
  size_t b = 0;
  void* tmp = nullptr;
  CK(sc.get(&keys, (int64_t)slots));
  CK(cub::DeviceSelect::If(nullptr, b, table, keys, cnt, (int64_t)slots, NotEmpty{}, st));
  CK(sc.get((char**)&tmp, (int64_t)b));
  CK(cub::DeviceSelect::If(tmp, b, table, keys, cnt, (int64_t)slots, NotEmpty{}, st));
  int h_cnt = 0;
  CK(cudaMemcpyAsync(&h_cnt, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *n_edges = h_cnt;
  if (h_cnt > max_edges) return set_error(LRCVT_E_ARG, "lrcvt_region_adjacency: max_edges too small");
  if (h_cnt == 0) return 0;
  CK(sc.get(&keys2, h_cnt));
  b = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, b, keys, keys2, h_cnt, 0, 64, st));
  void* tmp2 = nullptr;
  CK(sc.get((char**)&tmp2, (int64_t)b));
  CK(cub::DeviceRadixSort::SortKeys(tmp2, b, keys, keys2, h_cnt, 0, 64, st));
  k_split_edges<<<grid_for(h_cnt, 256), 256, 0, st>>>(keys2, h_cnt, (long long*)d_edges);
  CKL("k_split_edges"); LAUNCHED(1);
  CK(cudaStreamSynchronize(st));
  return 0;
}

}  // extern "C"
