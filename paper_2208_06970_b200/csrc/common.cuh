// common.cuh -- shared device helpers for the LSRCVT hot path (sm_100a).
//
// Every floating-point helper here reproduces the reference numba kernels
// bit for bit. The translation unit is compiled with --fmad=false, and the
// few expressions whose rounding matters are written with explicit
// __dmul_rn/__dadd_rn/__dsub_rn so no flag change can contract them.
//
// Reference: /root/reference/pkg/src/lrcvt/_kernels.py
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define LRCVT_EPS 1e-9  // _kernels.py:15
#define LRCVT_NONE (-1)

namespace lrcvt {

// Grid geometry, passed by value to every kernel.
struct Geo {
  int nx, ny, nz;
  int nxy;
  int64_t n;
  double sx, sy, sz;
  double inv_nx, inv_nxy;  // for exact division via fp64 reciprocal + fixup
  int dyadic;              // spacing values are powers of two (exact centre diffs)
  double len_cls[8];       // |offset| in world units by class (exact when dyadic)
  float isx, isy, isz;     // 1 / spacing in float (clearance tests only)
  double ix, iy, iz;       // 1 / spacing (exact reciprocals of powers of two when dyadic)
  int pack10;              // every axis <= 1024: coordinates pack into 10-bit fields
  int off_d[26];           // flat index delta of offset k
};

// _kernels.py:17-25: dz, dy, dx lexicographic, dx fastest, (0,0,0) excluded.
__host__ __device__ constexpr int off_dx(int k) { return (k < 13 ? k : k + 1) % 3 - 1; }
__host__ __device__ constexpr int off_dy(int k) { return ((k < 13 ? k : k + 1) / 3) % 3 - 1; }
__host__ __device__ constexpr int off_dz(int k) { return (k < 13 ? k : k + 1) / 9 - 1; }
__host__ __device__ inline void offset_of(int k, int& dx, int& dy, int& dz) {
  dx = off_dx(k); dy = off_dy(k); dz = off_dz(k);
}
// |offset| class: bit0 = dx != 0, bit1 = dy != 0, bit2 = dz != 0
__host__ __device__ constexpr int off_cls(int k) {
  return (off_dx(k) != 0) | ((off_dy(k) != 0) << 1) | ((off_dz(k) != 0) << 2);
}
// 26-bit masks of the offsets that step toward -x/+x/-y/+y/-z/+z
__host__ __device__ constexpr unsigned off_mask(int axis, int sgn) {
  unsigned m = 0;
  for (int k = 0; k < 26; k++) {
    const int d = axis == 0 ? off_dx(k) : axis == 1 ? off_dy(k) : off_dz(k);
    if (d == sgn) m |= 1u << k;
  }
  return m;
}
constexpr unsigned ALL26 = (1u << 26) - 1u;

// neighbours of (x, y, z) that lie inside the grid, as a 26-bit mask in the
// reference's scan order (bit k = OFFSETS[k])
__device__ __forceinline__ unsigned inbounds_mask(int x, int y, int z, int nx, int ny, int nz) {
  unsigned m = ALL26;
  if (x == 0) m &= ~off_mask(0, -1);
  if (x == nx - 1) m &= ~off_mask(0, 1);
  if (y == 0) m &= ~off_mask(1, -1);
  if (y == ny - 1) m &= ~off_mask(1, 1);
  if (z == 0) m &= ~off_mask(2, -1);
  if (z == nz - 1) m &= ~off_mask(2, 1);
  return m;
}

// packed per-offset table: dx, dy, dz, length class
__constant__ char4 c_off[26] = {
#define LRCVT_OFF(k) \
  { (signed char)off_dx(k), (signed char)off_dy(k), (signed char)off_dz(k), (signed char)off_cls(k) }
    LRCVT_OFF(0),  LRCVT_OFF(1),  LRCVT_OFF(2),  LRCVT_OFF(3),  LRCVT_OFF(4),  LRCVT_OFF(5),
    LRCVT_OFF(6),  LRCVT_OFF(7),  LRCVT_OFF(8),  LRCVT_OFF(9),  LRCVT_OFF(10), LRCVT_OFF(11),
    LRCVT_OFF(12), LRCVT_OFF(13), LRCVT_OFF(14), LRCVT_OFF(15), LRCVT_OFF(16), LRCVT_OFF(17),
    LRCVT_OFF(18), LRCVT_OFF(19), LRCVT_OFF(20), LRCVT_OFF(21), LRCVT_OFF(22), LRCVT_OFF(23),
    LRCVT_OFF(24), LRCVT_OFF(25)
#undef LRCVT_OFF
};

// |offset| by class with static indices only (dynamic indexing of the
// by-value Geo parameter would force a local-memory copy)
__device__ __forceinline__ double len_of(const Geo& g, int cls) {
  double r = g.len_cls[1];
  r = cls == 2 ? g.len_cls[2] : r;
  r = cls == 3 ? g.len_cls[3] : r;
  r = cls == 4 ? g.len_cls[4] : r;
  r = cls == 5 ? g.len_cls[5] : r;
  r = cls == 6 ? g.len_cls[6] : r;
  r = cls == 7 ? g.len_cls[7] : r;
  return r;
}

__device__ __forceinline__ int nbr_index(const int v, const char4 o, const int nx, const int nxy) {
  return v + o.x + o.y * nx + o.z * nxy;
}

// v -> (x, y, z) without integer division: fp64 reciprocal, then one-step
// fixup (exact for v < 2^31).
__device__ __forceinline__ void coords(const Geo& g, int v, int& x, int& y, int& z) {
  int q = __double2int_rz((double)v * g.inv_nxy);
  int r = v - q * g.nxy;
  if (r < 0) { q--; r += g.nxy; } else if (r >= g.nxy) { q++; r -= g.nxy; }
  z = q;
  int q2 = __double2int_rz((double)r * g.inv_nx);
  int r2 = r - q2 * g.nx;
  if (r2 < 0) { q2--; r2 += g.nx; } else if (r2 >= g.nx) { q2++; r2 -= g.nx; }
  y = q2;
  x = r2;
}

// _kernels.py:29-34: (x + 0.5) * s
__device__ __forceinline__ double centre1(int x, double s) {
  return __dmul_rn(__dadd_rn((double)x, 0.5), s);
}

// _kernels.py:37-42: sqrt(dx*dx + dy*dy + dz*dz), left-to-right, no FMA.
__device__ __forceinline__ double dist3(double ax, double ay, double az, double bx,
                                        double by, double bz) {
  double dx = __dsub_rn(bx, ax), dy = __dsub_rn(by, ay), dz = __dsub_rn(bz, az);
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                              __dmul_rn(dz, dz)));
}

// _kernels.py:136-144
__device__ __forceinline__ bool beats(double d, int s, double cur_d, int cur_s) {
  if (d < __dsub_rn(cur_d, LRCVT_EPS)) return true;
  if (fabs(__dsub_rn(d, cur_d)) <= LRCVT_EPS && s < cur_s) return true;
  return false;
}

// Exact pre-screen: returns a threshold T such that any candidate distance
// d >= T cannot satisfy beats(d, *, cur_d, *). Derivation:
// T - cur_d >= 2e-9 + |cur_d|*1e-15 - ulp(T)/2 > EPS, so d - cur_d rounds
// above EPS and d >= cur_d - EPS. cur_d == inf gives T == inf (no screen).
__device__ __forceinline__ double beat_threshold(double cur_d) {
  return __dadd_rn(cur_d, __dadd_rn(2e-9, __dmul_rn(fabs(cur_d), 1e-15)));
}

// Exact lower bound on the distance the reference computes, RN(sqrt(RN(
// dx*dx + dy*dy + dz*dz))), for an exact prescreen: the rounded sum of
// squares is >= RN(m*m) for m = max(|dx|,|dy|,|dz|) (monotone rounding of
// nonnegative terms) and RN(sqrt(RN(m*m))) >= m*(1 - 2^-51).
__device__ __forceinline__ double dist_lower(double ax, double ay, double az, double bx,
                                             double by, double bz) {
  const double m = fmax(fabs(__dsub_rn(bx, ax)), fmax(fabs(__dsub_rn(by, ay)), fabs(__dsub_rn(bz, az))));
  return __dmul_rn(m, 1.0 - 0x1p-50);
}

// read-only 32-byte load (two LDG.128 through the non-coherent path)
__device__ __forceinline__ double4 ld_d4(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ int clampi(int a, int lo, int hi) {
  return a < lo ? lo : (a > hi ? hi : a);
}

// floor(a / s) clamped into [0, n-1] as the reference does (int(np.floor()),
// then min/max). Values far outside int range saturate before clamping,
// which gives the same clamp result.
__device__ __forceinline__ int cell_of(double a, double s, int n) {
  double f = floor(__ddiv_rn(a, s));
  f = fmin(fmax(f, -1.0), (double)n);
  return clampi((int)f, 0, n - 1);
}

// _kernels.py:45-125: parametric t of the first entry into a voxel whose
// component is not `want`; 1.0 if none.
// Box: the scalars the DDA needs, passed by value so the out-of-line ray
// function does not force the whole Geo parameter into local memory.
struct Box {
  int nx, ny, nz;
  double sx, sy, sz;
  double ix, iy, iz;  // 1/s, used only when `dyadic` (then a/s == a*(1/s) exactly)
  int dyadic;
};
__device__ __forceinline__ Box box_of(const Geo& g) {
  return Box{g.nx, g.ny, g.nz, g.sx, g.sy, g.sz, g.ix, g.iy, g.iz, g.dyadic};
}

__device__ __forceinline__ int cell_of_box(double a, double s, double inv, int dyadic, int n) {
  double f = floor(dyadic ? __dmul_rn(a, inv) : __ddiv_rn(a, s));
  f = fmin(fmax(f, -1.0), (double)n);
  return clampi((int)f, 0, n - 1);
}

// _kernels.py:45-125, bit-exact (same operation order, exact comparisons).
// (A look-ahead variant that issued DDA_AHEAD cells' loads together measured
// 20% slower on the phase-1 eval: more instructions than latency saved.)
__device__ __noinline__ double segment_hit_box(const int* __restrict__ comp, const Box g,
                                               double ax, double ay, double az, double bx,
                                               double by, double bz, int want) {
  int cx = cell_of_box(ax, g.sx, g.ix, g.dyadic, g.nx), cy = cell_of_box(ay, g.sy, g.iy, g.dyadic, g.ny),
      cz = cell_of_box(az, g.sz, g.iz, g.dyadic, g.nz);
  const int ex = cell_of_box(bx, g.sx, g.ix, g.dyadic, g.nx), ey = cell_of_box(by, g.sy, g.iy, g.dyadic, g.ny),
            ez = cell_of_box(bz, g.sz, g.iz, g.dyadic, g.nz);
  if (__ldg(comp + cx + g.nx * (cy + g.ny * cz)) != want) return 0.0;
  const double dx = __dsub_rn(bx, ax), dy = __dsub_rn(by, ay), dz = __dsub_rn(bz, az);
  const int stepx = dx > 0 ? 1 : -1, stepy = dy > 0 ? 1 : -1, stepz = dz > 0 ? 1 : -1;
  const double big = 1e30;
  double tmaxx, tmaxy, tmaxz, tdx, tdy, tdz;
  if (dx != 0.0) {
    const double nxt = dx > 0 ? __dmul_rn((double)(cx + 1), g.sx) : __dmul_rn((double)cx, g.sx);
    tmaxx = __ddiv_rn(__dsub_rn(nxt, ax), dx);
    tdx = __ddiv_rn(g.sx, fabs(dx));
  } else { tmaxx = big; tdx = big; }
  if (dy != 0.0) {
    const double nxt = dy > 0 ? __dmul_rn((double)(cy + 1), g.sy) : __dmul_rn((double)cy, g.sy);
    tmaxy = __ddiv_rn(__dsub_rn(nxt, ay), dy);
    tdy = __ddiv_rn(g.sy, fabs(dy));
  } else { tmaxy = big; tdy = big; }
  if (dz != 0.0) {
    const double nxt = dz > 0 ? __dmul_rn((double)(cz + 1), g.sz) : __dmul_rn((double)cz, g.sz);
    tmaxz = __ddiv_rn(__dsub_rn(nxt, az), dz);
    tdz = __ddiv_rn(g.sz, fabs(dz));
  } else { tmaxz = big; tdz = big; }
  const int max_steps = abs(ex - cx) + abs(ey - cy) + abs(ez - cz) + 8;
  for (int i = 0; i < max_steps; i++) {
    if (cx == ex && cy == ey && cz == ez) return 1.0;
    const double t = fmin(tmaxx, fmin(tmaxy, tmaxz));
    if (t > 1.0) {
      if (__ldg(comp + ex + g.nx * (ey + g.ny * ez)) == want) return 1.0;
      return 1.0 - 1e-12;
    }
    if (tmaxx == t) { cx += stepx; tmaxx = __dadd_rn(tmaxx, tdx); }
    if (tmaxy == t) { cy += stepy; tmaxy = __dadd_rn(tmaxy, tdy); }
    if (tmaxz == t) { cz += stepz; tmaxz = __dadd_rn(tmaxz, tdz); }
    if (cx < 0 || cy < 0 || cz < 0 || cx >= g.nx || cy >= g.ny || cz >= g.nz) return t;
    if (__ldg(comp + cx + g.nx * (cy + g.ny * cz)) != want) return t;
  }
  return 1.0;
}

__device__ __forceinline__ double segment_hit_t(const int* __restrict__ comp, const Geo& g,
                                               double ax, double ay, double az, double bx,
                                               double by, double bz, int want) {
  return segment_hit_box(comp, box_of(g), ax, ay, az, bx, by, bz, want);
}

__device__ __forceinline__ bool segment_clear(const int* __restrict__ comp, const Geo& g,
                                              double ax, double ay, double az, double bx,
                                              double by, double bz, int want) {
  return segment_hit_t(comp, g, ax, ay, az, bx, by, bz, want) >= 1.0;
}

// Clearance shortcut for a ray from the centre c of voxel v to a point p.
// nbm bits 26..31 hold clr(v) = min(D(v), 32), D(v) = Chebyshev distance from
// v to the nearest voxel of another component or outside the grid, so every
// voxel within Chebyshev radius clr(v) - 1 of v shares v's component. The
// DDA only visits cells inside the index box spanned by v and cell(p),
// widened by at most one cell where a rounded crossing parameter oversteps;
// along each axis |cell(p) - v| <= |p - c| / s + 1/2, so with
// t = max_a |p_a - c_a| / s_a, t + 2.5 <= clr(v) proves every visited cell is
// in v's component (_segment_clear is true) without walking the ray. Tested
// in float with a further 0.5 cell of slack for its rounding.
constexpr int NBM_CLR_SHIFT = 26;
__device__ __forceinline__ bool ray_clear_by_clearance(unsigned nbm_v, float tx, float ty, float tz) {
  return fmaxf(tx, fmaxf(ty, tz)) + 3.0f <= (float)(nbm_v >> NBM_CLR_SHIFT);
}
// |p - c| per axis in cells (inv = 1 / spacing, float)
__device__ __forceinline__ bool ray_clear_near(unsigned nbm_v, double px, double py, double pz, double cx,
                                               double cy, double cz, float isx, float isy, float isz) {
  return ray_clear_by_clearance(nbm_v, fabsf((float)(px - cx)) * isx, fabsf((float)(py - cy)) * isy,
                                fabsf((float)(pz - cz)) * isz);
}

// _segment_clear (_kernels.py:128-133), i.e. segment_hit_box(...) >= 1.0,
// with the same DDA (same cells, same order, same exact comparisons) and two
// exact shortcuts from the static clearance clr(c) = min(D(c), 32) in nbm
// bits 26..31 (D: Chebyshev distance to the nearest foreign or out-of-grid
// voxel; every cell within Chebyshev radius clr(c) - 1 of c is in c's
// component):
//   * a step from a cell with clr >= 2 lands on a 26-neighbour, which is
//     in-grid and in the component: no bounds test, no comp load;
//   * from the current cell c, the walk only visits cells within Chebyshev
//     distance max_a |e_a - c_a| + 1 of c (monotone steps towards the end
//     cell e, at most one rounded overstep), so clr(c) >= that + 2 (one cell
//     of extra slack here) proves every remaining cell, e included, in the
//     component: the reference returns 1.0.
__device__ __noinline__ bool segment_clear_fast(const int* __restrict__ comp, const uint32_t* __restrict__ nbm,
                                                const Box g, double ax, double ay, double az, double bx, double by,
                                                double bz, int want) {
  int cx = cell_of_box(ax, g.sx, g.ix, g.dyadic, g.nx), cy = cell_of_box(ay, g.sy, g.iy, g.dyadic, g.ny),
      cz = cell_of_box(az, g.sz, g.iz, g.dyadic, g.nz);
  const int ex = cell_of_box(bx, g.sx, g.ix, g.dyadic, g.nx), ey = cell_of_box(by, g.sy, g.iy, g.dyadic, g.ny),
            ez = cell_of_box(bz, g.sz, g.iz, g.dyadic, g.nz);
  const int sxy = g.nx * g.ny;
  int idx = cx + g.nx * cy + sxy * cz;
  if (__ldg(comp + idx) != want) return false;
  const double dx = __dsub_rn(bx, ax), dy = __dsub_rn(by, ay), dz = __dsub_rn(bz, az);
  const int stepx = dx > 0 ? 1 : -1, stepy = dy > 0 ? 1 : -1, stepz = dz > 0 ? 1 : -1;
  const double big = 1e30;
  double tmaxx, tmaxy, tmaxz, tdx, tdy, tdz;
  if (dx != 0.0) {
    const double nxt = dx > 0 ? __dmul_rn((double)(cx + 1), g.sx) : __dmul_rn((double)cx, g.sx);
    tmaxx = __ddiv_rn(__dsub_rn(nxt, ax), dx);
    tdx = __ddiv_rn(g.sx, fabs(dx));
  } else { tmaxx = big; tdx = big; }
  if (dy != 0.0) {
    const double nxt = dy > 0 ? __dmul_rn((double)(cy + 1), g.sy) : __dmul_rn((double)cy, g.sy);
    tmaxy = __ddiv_rn(__dsub_rn(nxt, ay), dy);
    tdy = __ddiv_rn(g.sy, fabs(dy));
  } else { tmaxy = big; tdy = big; }
  if (dz != 0.0) {
    const double nxt = dz > 0 ? __dmul_rn((double)(cz + 1), g.sz) : __dmul_rn((double)cz, g.sz);
    tmaxz = __ddiv_rn(__dsub_rn(nxt, az), dz);
    tdz = __ddiv_rn(g.sz, fabs(dz));
  } else { tmaxz = big; tdz = big; }
  const int ix = stepx, iy = stepy * g.nx, iz = stepz * sxy;
  int clr = (int)(__ldg(nbm + idx) >> NBM_CLR_SHIFT);
  const int max_steps = abs(ex - cx) + abs(ey - cy) + abs(ez - cz) + 8;
  for (int i = 0; i < max_steps; i++) {
    if (cx == ex && cy == ey && cz == ez) return true;
    const int rem = max(abs(ex - cx), max(abs(ey - cy), abs(ez - cz)));
    if (clr >= rem + 3) return true;
    const double t = fmin(tmaxx, fmin(tmaxy, tmaxz));
    if (t > 1.0) return __ldg(comp + ex + g.nx * ey + sxy * ez) == want;
    const bool inside = clr >= 2;  // every 26-neighbour in-grid and in the component
    if (tmaxx == t) {
      cx += stepx; idx += ix; tmaxx = __dadd_rn(tmaxx, tdx);
      if (!inside && (unsigned)cx >= (unsigned)g.nx) return false;
    }
    if (tmaxy == t) {
      cy += stepy; idx += iy; tmaxy = __dadd_rn(tmaxy, tdy);
      if (!inside && (unsigned)cy >= (unsigned)g.ny) return false;
    }
    if (tmaxz == t) {
      cz += stepz; idx += iz; tmaxz = __dadd_rn(tmaxz, tdz);
      if (!inside && (unsigned)cz >= (unsigned)g.nz) return false;
    }
    if (!inside && __ldg(comp + idx) != want) return false;
    clr = (int)(__ldg(nbm + idx) >> NBM_CLR_SHIFT);
  }
  return true;
}

// Warp-aggregated append of `take` (0/1) items; returns this lane's slot
// (valid only when take). All 32 lanes must call it.
// CTA-aggregated append: one atomic per CTA. Every thread of the CTA must
// call it (uses __syncthreads).
__device__ __forceinline__ int block_append(int* counter, bool take) {
  __shared__ int s_w[32];
  __shared__ int s_b;
  const unsigned m = __ballot_sync(0xffffffffu, take);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_w[wid] = __popc(m);
  __syncthreads();
  if (threadIdx.x == 0) {
    int sum = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
      const int t = s_w[w];
      s_w[w] = sum;
      sum += t;
    }
    s_b = sum ? atomicAdd(counter, sum) : 0;
  }
  __syncthreads();
  return s_b + s_w[wid] + __popc(m & ((1u << lane) - 1u));
}

__device__ __forceinline__ int warp_append(int* counter, bool take) {
  unsigned m = __ballot_sync(0xffffffffu, take);
  int lane = threadIdx.x & 31;
  int leader = __ffs(m) - 1;
  int base = 0;
  if (m && lane == leader) base = atomicAdd(counter, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader < 0 ? 0 : leader);
  return base + __popc(m & ((1u << lane) - 1u));
}

}  // namespace lrcvt
