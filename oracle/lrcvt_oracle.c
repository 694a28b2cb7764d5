/*
 * lrcvt_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's numba kernels and of the two
 * Python drivers that call them, used as the parity checker for the CUDA
 * path and as the `cpu_baseline` / `--impl reference` CPU arm of bench.py.
 * Nothing in the product package (paper_2208_06970_b200/) links or calls it.
 *
 * Reference (read-only, /root/reference/pkg/src/lrcvt):
 *   _kernels.py:14-25    NONE, EPS, 26-neighbour OFFSETS order
 *   _kernels.py:29-42    _center, _dist3
 *   _kernels.py:45-133   _segment_hit_t, _segment_clear (3D DDA)
 *   _kernels.py:136-144  _beats
 *   _kernels.py:147-246  _eval_voxel
 *   _kernels.py:249-282  _eval_list         (prange  -> OpenMP parallel for)
 *   _kernels.py:285-334  _apply_and_enqueue (serial, as in the reference)
 *   _kernels.py:337-385  _run_phase
 *   _kernels.py:399-422  _place_seeds
 *   _kernels.py:425-454  _seed_worklist
 *   _kernels.py:457-486  _phi_chains
 *   _kernels.py:489-510  _audit_paths
 *   _kernels.py:513-532  _centroid_targets
 *   _kernels.py:535-582  _move_sites
 *   tessellation.py:102-208  voronoi_classify driver (phases, sweeps, state)
 *   tessellation.py:211-248  centroidal_update driver
 *
 * Floating point: compiled with -ffp-contract=off (numba emits no FMA; see
 * SURVEY.md finding 3), IEEE sqrt/div, identical operation order.
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py); see tests/test_oracle_golden.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NONE (-1)
#define EPS 1e-9 /* _kernels.py:15 */

/* _kernels.py:17-25: dz, then dy, then dx; dx fastest; (0,0,0) excluded */
static int OFF[26][3];
static int off_init = 0;
static void init_offsets(void) {
  if (off_init) return;
  int k = 0;
  for (int dz = -1; dz <= 1; dz++)
    for (int dy = -1; dy <= 1; dy++)
      for (int dx = -1; dx <= 1; dx++)
        if (dx || dy || dz) {
          OFF[k][0] = dx; OFF[k][1] = dy; OFF[k][2] = dz; k++;
        }
  off_init = 1;
}

typedef struct {
  int64_t nx, ny, nz;
  double sx, sy, sz;
} Dims;

static inline int64_t clampi(int64_t a, int64_t lo, int64_t hi) {
  return a < lo ? lo : (a > hi ? hi : a);
}

/* _kernels.py:38-42 */
static inline double dist3(double ax, double ay, double az, double bx,
                           double by, double bz) {
  double dx = bx - ax, dy = by - ay, dz = bz - az;
  return sqrt(dx * dx + dy * dy + dz * dz);
}

/* _kernels.py:45-125 */
double orc_segment_hit_t(const int32_t *comp, int64_t nx, int64_t ny,
                         int64_t nz, double sx, double sy, double sz,
                         double ax, double ay, double az, double bx, double by,
                         double bz, int32_t want) {
  int64_t cx = (int64_t)floor(ax / sx);
  int64_t cy = (int64_t)floor(ay / sy);
  int64_t cz = (int64_t)floor(az / sz);
  int64_t ex = (int64_t)floor(bx / sx);
  int64_t ey = (int64_t)floor(by / sy);
  int64_t ez = (int64_t)floor(bz / sz);
  cx = clampi(cx, 0, nx - 1); cy = clampi(cy, 0, ny - 1); cz = clampi(cz, 0, nz - 1);
  ex = clampi(ex, 0, nx - 1); ey = clampi(ey, 0, ny - 1); ez = clampi(ez, 0, nz - 1);
  if (comp[cx + nx * (cy + ny * cz)] != want) return 0.0;
  double dx = bx - ax, dy = by - ay, dz = bz - az;
  int64_t stepx = dx > 0 ? 1 : -1;
  int64_t stepy = dy > 0 ? 1 : -1;
  int64_t stepz = dz > 0 ? 1 : -1;
  const double big = 1e30;
  double tmaxx, tmaxy, tmaxz, tdx, tdy, tdz, nxt;
  if (dx != 0.0) {
    nxt = dx > 0 ? (double)(cx + 1) * sx : (double)cx * sx;
    tmaxx = (nxt - ax) / dx; tdx = sx / fabs(dx);
  } else { tmaxx = big; tdx = big; }
  if (dy != 0.0) {
    nxt = dy > 0 ? (double)(cy + 1) * sy : (double)cy * sy;
    tmaxy = (nxt - ay) / dy; tdy = sy / fabs(dy);
  } else { tmaxy = big; tdy = big; }
  if (dz != 0.0) {
    nxt = dz > 0 ? (double)(cz + 1) * sz : (double)cz * sz;
    tmaxz = (nxt - az) / dz; tdz = sz / fabs(dz);
  } else { tmaxz = big; tdz = big; }
  int64_t max_steps = llabs(ex - cx) + llabs(ey - cy) + llabs(ez - cz) + 8;
  for (int64_t i = 0; i < max_steps; i++) {
    if (cx == ex && cy == ey && cz == ez) return 1.0;
    double t = fmin(tmaxx, fmin(tmaxy, tmaxz));
    if (t > 1.0) {
      if (comp[ex + nx * (ey + ny * ez)] == want) return 1.0;
      return 1.0 - 1e-12;
    }
    if (tmaxx == t) { cx += stepx; tmaxx += tdx; }
    if (tmaxy == t) { cy += stepy; tmaxy += tdy; }
    if (tmaxz == t) { cz += stepz; tmaxz += tdz; }
    if (cx < 0 || cy < 0 || cz < 0 || cx >= nx || cy >= ny || cz >= nz) return t;
    if (comp[cx + nx * (cy + ny * cz)] != want) return t;
  }
  return 1.0;
}

/* numba min(a, min(b, c)) on floats: Python-style min returns the first
 * argument on ties and NaN never occurs here, so fmin is equivalent. */

static inline int seg_clear(const int32_t *comp, const Dims *g, double ax,
                            double ay, double az, double bx, double by,
                            double bz, int32_t want) {
  return orc_segment_hit_t(comp, g->nx, g->ny, g->nz, g->sx, g->sy, g->sz, ax,
                           ay, az, bx, by, bz, want) >= 1.0;
}

/* _kernels.py:136-144 */
static inline int beats(double d, int32_t s, double cur_d, int32_t cur_s) {
  if (d < cur_d - EPS) return 1;
  if (fabs(d - cur_d) <= EPS && s < cur_s) return 1;
  return 0;
}

/* _kernels.py:147-246 */
static int eval_voxel(int64_t v, int phase2, const int32_t *comp, const Dims *g,
                      const double *site_pos, const int32_t *site_of,
                      const double *dist, const int32_t *src, double *od,
                      int32_t *os, int32_t *osrc) {
  const int64_t nx = g->nx, ny = g->ny, nz = g->nz;
  const double sx = g->sx, sy = g->sy, sz = g->sz;
  int32_t cv = comp[v];
  int64_t x = v % nx, y = (v / nx) % ny, z = v / (nx * ny);
  double px = ((double)x + 0.5) * sx, py = ((double)y + 0.5) * sy,
         pz = ((double)z + 0.5) * sz;
  double best_d = dist[v];
  int32_t best_s = site_of[v];
  int32_t best_src = src[v];
  double orig_d = best_d;
  int32_t orig_s = best_s;
  int32_t failed_site = -1;
  for (int k = 0; k < 26; k++) {
    int64_t wx = x + OFF[k][0], wy = y + OFF[k][1], wz = z + OFF[k][2];
    if (wx < 0 || wy < 0 || wz < 0 || wx >= nx || wy >= ny || wz >= nz) continue;
    int64_t w = wx + nx * (wy + ny * wz);
    if (comp[w] != cv) continue;
    int32_t sw = site_of[w];
    if (sw < 0) continue;
    if (phase2) {
      double d = dist[w] + dist3(px, py, pz, ((double)wx + 0.5) * sx,
                                 ((double)wy + 0.5) * sy, ((double)wz + 0.5) * sz);
      if (beats(d, sw, best_d, best_s)) { best_d = d; best_s = sw; best_src = (int32_t)w; }
    }
    int32_t u = src[w];
    if (u == w) {
      double spx = site_pos[3 * (int64_t)sw], spy = site_pos[3 * (int64_t)sw + 1],
             spz = site_pos[3 * (int64_t)sw + 2];
      double d = dist3(px, py, pz, spx, spy, spz);
      if (beats(d, sw, best_d, best_s) && sw != failed_site) {
        if (seg_clear(comp, g, px, py, pz, spx, spy, spz, cv)) {
          best_d = d; best_s = sw; best_src = (int32_t)v;
        } else {
          failed_site = sw;
        }
      }
    } else if (phase2 && u >= 0) {
      int32_t su = site_of[u];
      if (su >= 0 && comp[u] == cv) {
        int64_t ux = u % nx, uy = (u / nx) % ny, uz = u / (nx * ny);
        double upx = ((double)ux + 0.5) * sx, upy = ((double)uy + 0.5) * sy,
               upz = ((double)uz + 0.5) * sz;
        double d = dist[u] + dist3(px, py, pz, upx, upy, upz);
        if (beats(d, su, best_d, best_s)) {
          if (seg_clear(comp, g, px, py, pz, upx, upy, upz, cv)) {
            best_d = d; best_s = su; best_src = u;
          }
        }
      }
    }
  }
  *od = best_d; *os = best_s; *osrc = best_src;
  return (best_s != orig_s) || (best_d < orig_d - EPS);
}

typedef struct {
  const int32_t *comp;
  Dims g;
  const double *site_pos;
  int32_t *site_of;
  double *dist;
  int32_t *src;
  int64_t *wl, *wl_next, *stamp, *imp_stamp;
  double *p_dist;
  int32_t *p_site, *p_src;
  int64_t evals, commits;
} Ctx;

/* _kernels.py:249-282 (prange -> OpenMP; proposals only, so order-free) */
static void eval_list(Ctx *c, const int64_t *items, int64_t n_items, int phase2,
                      int64_t rnd) {
  c->evals += n_items;
#pragma omp parallel for schedule(dynamic, 512)
  for (int64_t i = 0; i < n_items; i++) {
    int64_t v = items[i];
    double d; int32_t s, sv;
    if (eval_voxel(v, phase2, c->comp, &c->g, c->site_pos, c->site_of, c->dist,
                   c->src, &d, &s, &sv)) {
      c->p_dist[v] = d; c->p_site[v] = s; c->p_src[v] = sv; c->imp_stamp[v] = rnd;
    }
  }
}

/* _kernels.py:285-334 (serial in the reference; kept serial) */
static int64_t apply_and_enqueue(Ctx *c, const int64_t *items, int64_t n_items,
                                 int64_t *wl_next, int64_t rnd) {
  const int64_t nx = c->g.nx, ny = c->g.ny, nz = c->g.nz;
  for (int64_t i = 0; i < n_items; i++) {
    int64_t v = items[i];
    if (c->imp_stamp[v] == rnd) {
      c->dist[v] = c->p_dist[v]; c->site_of[v] = c->p_site[v]; c->src[v] = c->p_src[v];
      c->commits++;
    }
  }
  int64_t cnt = 0;
  for (int64_t i = 0; i < n_items; i++) {
    int64_t v = items[i];
    if (c->imp_stamp[v] != rnd) continue;
    int64_t x = v % nx, y = (v / nx) % ny, z = v / (nx * ny);
    for (int k = 0; k < 26; k++) {
      int64_t ux = x + OFF[k][0], uy = y + OFF[k][1], uz = z + OFF[k][2];
      if (ux < 0 || uy < 0 || uz < 0 || ux >= nx || uy >= ny || uz >= nz) continue;
      int64_t u = ux + nx * (uy + ny * uz);
      if (c->comp[u] != c->comp[v]) continue;
      if (c->stamp[u] != rnd) { c->stamp[u] = rnd; wl_next[cnt++] = u; }
    }
  }
  return cnt;
}

/* _kernels.py:337-385; returns rounds, updates *rnd. Swaps the worklists the
 * same way the reference does (the caller's `wl` buffer identity matters
 * only for storage, never for results). */
static int64_t run_phase(Ctx *c, int phase2, int64_t n_wl, int64_t *rnd_io) {
  int64_t rnd = *rnd_io, rounds = 0;
  int64_t *wl = c->wl, *wl_next = c->wl_next;
  while (n_wl > 0) {
    rnd++; rounds++;
    eval_list(c, wl, n_wl, phase2, rnd);
    int64_t n_next = apply_and_enqueue(c, wl, n_wl, wl_next, rnd);
    int64_t *t = wl; wl = wl_next; wl_next = t;
    n_wl = n_next;
  }
  *rnd_io = rnd;
  return rounds;
}

/* _kernels.py:399-422 */
static int64_t place_seeds(Ctx *c, int64_t n_sites, const int32_t *site_comp) {
  const Dims *g = &c->g;
  int64_t bad = 0;
  for (int64_t s = 0; s < n_sites; s++) {
    const double *p = c->site_pos + 3 * s;
    int64_t x = (int64_t)floor(p[0] / g->sx), y = (int64_t)floor(p[1] / g->sy),
            z = (int64_t)floor(p[2] / g->sz);
    x = clampi(x, 0, g->nx - 1); y = clampi(y, 0, g->ny - 1); z = clampi(z, 0, g->nz - 1);
    int64_t v = x + g->nx * (y + g->ny * z);
    if (c->comp[v] != site_comp[s]) { bad++; continue; }
    double cx = ((double)x + 0.5) * g->sx, cy = ((double)y + 0.5) * g->sy,
           cz = ((double)z + 0.5) * g->sz;
    double d = dist3(cx, cy, cz, p[0], p[1], p[2]);
    if (c->site_of[v] < 0 || beats(d, (int32_t)s, c->dist[v], c->site_of[v])) {
      c->site_of[v] = (int32_t)s; c->dist[v] = d; c->src[v] = (int32_t)v;
    }
  }
  return bad;
}

/* _kernels.py:425-454 */
static int64_t seed_worklist(Ctx *c) {
  const int64_t nx = c->g.nx, ny = c->g.ny, nz = c->g.nz, n = nx * ny * nz;
  int64_t cnt = 0;
  for (int64_t v = 0; v < n; v++) {
    if (c->site_of[v] < 0) continue;
    if (c->stamp[v] != 0) { c->stamp[v] = 0; c->wl[cnt++] = v; }
    int64_t x = v % nx, y = (v / nx) % ny, z = v / (nx * ny);
    for (int k = 0; k < 26; k++) {
      int64_t ux = x + OFF[k][0], uy = y + OFF[k][1], uz = z + OFF[k][2];
      if (ux < 0 || uy < 0 || uz < 0 || ux >= nx || uy >= ny || uz >= nz) continue;
      int64_t u = ux + nx * (uy + ny * uz);
      if (c->comp[u] != c->comp[v]) continue;
      if (c->stamp[u] != 0) { c->stamp[u] = 0; c->wl[cnt++] = u; }
    }
  }
  return cnt;
}

/*
 * tessellation.py:102-208 (voronoi_classify), arrays already allocated by
 * the caller and initialised here. stats_out[0..5] = rounds, sweeps,
 * assigned, evaluations (E), commits (C), bad-site count.
 * Returns 0, or the number of sites outside their component (the caller
 * raises ValueError, tessellation.py:139-140), or -1 on allocation failure.
 */
int64_t orc_classify(int64_t nx, int64_t ny, int64_t nz, double sx, double sy,
                     double sz, const int32_t *comp, int64_t n_sites,
                     const double *site_pos, const int32_t *site_comp,
                     int64_t n_components, int32_t *site_of, double *dist,
                     int32_t *src, uint8_t *state, int64_t *stats_out) {
  init_offsets();
  const int64_t n = nx * ny * nz;
  for (int64_t v = 0; v < n; v++) { site_of[v] = NONE; dist[v] = INFINITY; src[v] = NONE; }
  memset(stats_out, 0, 6 * sizeof(int64_t));
  if (n_sites == 0) { memset(state, 0, (size_t)n); return 0; }
  Ctx c;
  memset(&c, 0, sizeof(c));
  c.comp = comp;
  c.g.nx = nx; c.g.ny = ny; c.g.nz = nz; c.g.sx = sx; c.g.sy = sy; c.g.sz = sz;
  c.site_pos = site_pos; c.site_of = site_of; c.dist = dist; c.src = src;
  int64_t bad = place_seeds(&c, n_sites, site_comp);
  stats_out[5] = bad;
  if (bad) return bad;
  int64_t *wl_a = malloc(n * sizeof(int64_t)), *wl_b = malloc(n * sizeof(int64_t));
  c.stamp = malloc(n * sizeof(int64_t)); c.imp_stamp = malloc(n * sizeof(int64_t));
  c.p_dist = malloc(n * sizeof(double));
  c.p_site = malloc(n * sizeof(int32_t)); c.p_src = malloc(n * sizeof(int32_t));
  int64_t ncs = n_components > 1 ? n_components : 1;
  uint8_t *has_site = calloc((size_t)ncs, 1);
  int64_t *eligible = malloc(n * sizeof(int64_t));
  if (!wl_a || !wl_b || !c.stamp || !c.imp_stamp || !c.p_dist || !c.p_site ||
      !c.p_src || !has_site || !eligible) return -1;
  for (int64_t v = 0; v < n; v++) { c.stamp[v] = -1; c.imp_stamp[v] = -1; }
  c.wl = wl_a; c.wl_next = wl_b;

  /* phase 1: tessellation.py:151-156 */
  int64_t n_wl = seed_worklist(&c);
  int64_t rnd = 0;
  int64_t rounds1 = run_phase(&c, 0, n_wl, &rnd);

  /* phase 2: tessellation.py:161-189 */
  /* comps_with_sites[site_comp] = True: numpy wraps a negative id (a site
   * recorded in component -1 marks the last component) */
  for (int64_t s = 0; s < n_sites; s++) {
    int64_t cs = site_comp[s] < 0 ? site_comp[s] + ncs : site_comp[s];
    if (cs >= 0 && cs < ncs) has_site[cs] = 1;
  }
  int64_t n_el = 0;
  for (int64_t v = 0; v < n; v++)
    if (comp[v] != NONE && has_site[comp[v]]) eligible[n_el++] = v;
  /* the reference always writes the eligible list into the buffer it calls
   * `wl` (tessellation.py:166); run_phase reads its worklist from there */
  memcpy(c.wl, eligible, n_el * sizeof(int64_t));
  n_wl = n_el;
  int64_t rounds2 = 0, sweeps = 0;
  for (;;) {
    rounds2 += run_phase(&c, 1, n_wl, &rnd);
    rnd++; sweeps++;
    eval_list(&c, eligible, n_el, 1, rnd);
    int64_t improved = 0;
    for (int64_t i = 0; i < n_el; i++) improved += c.imp_stamp[eligible[i]] == rnd;
    if (improved == 0) break;
    n_wl = apply_and_enqueue(&c, eligible, n_el, c.wl, rnd);
  }
  /* state bits: tessellation.py:191-194 */
  int64_t assigned = 0;
  for (int64_t v = 0; v < n; v++) {
    uint8_t st = 0;
    if (site_of[v] != NONE) { st = 2 | 4; assigned++; if (src[v] == v) st |= 1; }
    state[v] = st;
  }
  stats_out[0] = rounds1 + rounds2; stats_out[1] = sweeps; stats_out[2] = assigned;
  stats_out[3] = c.evals; stats_out[4] = c.commits;
  free(wl_a); free(wl_b); free(c.stamp); free(c.imp_stamp); free(c.p_dist);
  free(c.p_site); free(c.p_src); free(has_site); free(eligible);
  return 0;
}

/* _kernels.py:457-486; phi int64[n], returns max depth. */
int64_t orc_phi_chains(int64_t n, const int32_t *site_of, const int32_t *src,
                       int64_t *phi) {
  int64_t *stack = malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  int64_t max_depth = 0;
  for (int64_t v = 0; v < n; v++) phi[v] = -1;
  for (int64_t v = 0; v < n; v++) {
    if (site_of[v] < 0 || phi[v] != -1) continue;
    int64_t u = v, depth = 0;
    while (phi[u] == -1 && src[u] != u && src[u] >= 0) { stack[depth++] = u; u = src[u]; }
    int64_t base;
    if (phi[u] != -1) base = phi[u];
    else { base = u; phi[u] = u; }
    for (int64_t k = 0; k < depth; k++) phi[stack[k]] = base;
    if (depth > max_depth) max_depth = depth;
  }
  free(stack);
  return max_depth;
}

/* _kernels.py:513-532; fixed increasing-voxel accumulation order */
void orc_centroid_targets(int64_t nx, int64_t ny, int64_t nz, double sx,
                          double sy, double sz, const int32_t *site_of,
                          const int64_t *phi, const double *weights,
                          int64_t n_sites, double *wsum, double *tx, double *ty,
                          double *tz) {
  const int64_t n = nx * ny * nz;
  for (int64_t s = 0; s < n_sites; s++) { wsum[s] = 0; tx[s] = 0; ty[s] = 0; tz[s] = 0; }
  for (int64_t v = 0; v < n; v++) {
    int32_t s = site_of[v];
    if (s < 0) continue;
    double w = weights[v];
    int64_t a = phi[v];
    int64_t x = a % nx, y = (a / nx) % ny, z = a / (nx * ny);
    double ax = ((double)x + 0.5) * sx, ay = ((double)y + 0.5) * sy,
           az = ((double)z + 0.5) * sz;
    wsum[s] += w; tx[s] += w * ax; ty[s] += w * ay; tz[s] += w * az;
  }
}

/* _kernels.py:535-582; returns the empty-region count */
int64_t orc_move_sites(int64_t nx, int64_t ny, int64_t nz, double sx, double sy,
                       double sz, const int32_t *comp, int64_t n_sites,
                       const double *site_pos, const int32_t *site_comp,
                       const double *wsum, const double *tx, const double *ty,
                       const double *tz, double backoff, double *new_pos,
                       double *disp) {
  int64_t empty = 0;
  memcpy(new_pos, site_pos, (size_t)n_sites * 3 * sizeof(double));
  for (int64_t s = 0; s < n_sites; s++) {
    disp[s] = 0.0;
    if (wsum[s] <= 0.0) { empty++; continue; }
    double ax = site_pos[3 * s], ay = site_pos[3 * s + 1], az = site_pos[3 * s + 2];
    double bx = tx[s] / wsum[s], by = ty[s] / wsum[s], bz = tz[s] / wsum[s];
    double seg = dist3(ax, ay, az, bx, by, bz);
    if (seg == 0.0) continue;
    int32_t want = site_comp[s];
    double thit = orc_segment_hit_t(comp, nx, ny, nz, sx, sy, sz, ax, ay, az, bx,
                                    by, bz, want);
    double px, py, pz;
    if (thit >= 1.0) { px = bx; py = by; pz = bz; }
    else {
      double travel = thit * seg - backoff;
      if (travel <= 0.0) continue;
      double f = travel / seg;
      px = ax + (bx - ax) * f; py = ay + (by - ay) * f; pz = az + (bz - az) * f;
    }
    int64_t cx = clampi((int64_t)floor(px / sx), 0, nx - 1);
    int64_t cy = clampi((int64_t)floor(py / sy), 0, ny - 1);
    int64_t cz = clampi((int64_t)floor(pz / sz), 0, nz - 1);
    if (comp[cx + nx * (cy + ny * cz)] != want) continue;
    new_pos[3 * s] = px; new_pos[3 * s + 1] = py; new_pos[3 * s + 2] = pz;
    disp[s] = dist3(ax, ay, az, px, py, pz);
  }
  return empty;
}

/* tessellation.py:211-248 minus the Python list building and the numpy mean
 * (done by the caller with numpy, as the reference does). */
int64_t orc_centroidal_update(int64_t nx, int64_t ny, int64_t nz, double sx,
                              double sy, double sz, const int32_t *comp,
                              const int32_t *site_of, const int32_t *src,
                              const double *weights, int64_t n_sites,
                              const double *site_pos, const int32_t *site_comp,
                              double backoff, double *new_pos, double *disp,
                              double *sums4 /* 4*n_sites, may be NULL */) {
  const int64_t n = nx * ny * nz;
  int64_t *phi = malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  double *buf = malloc((size_t)(n_sites > 0 ? n_sites : 1) * 4 * sizeof(double));
  orc_phi_chains(n, site_of, src, phi);
  double *wsum = buf, *tx = buf + n_sites, *ty = buf + 2 * n_sites, *tz = buf + 3 * n_sites;
  orc_centroid_targets(nx, ny, nz, sx, sy, sz, site_of, phi, weights, n_sites,
                       wsum, tx, ty, tz);
  if (sums4) memcpy(sums4, buf, (size_t)n_sites * 4 * sizeof(double));
  int64_t empty = orc_move_sites(nx, ny, nz, sx, sy, sz, comp, n_sites, site_pos,
                                 site_comp, wsum, tx, ty, tz, backoff, new_pos, disp);
  free(phi); free(buf);
  return empty;
}

/* _kernels.py:489-510 */
void orc_audit_paths(int64_t nx, int64_t ny, int64_t nz, double sx, double sy,
                     double sz, const int32_t *comp, const double *site_pos,
                     const int32_t *site_of, const int32_t *src, uint8_t *out_bad) {
  init_offsets();
  Dims g = {nx, ny, nz, sx, sy, sz};
  const int64_t n = nx * ny * nz;
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; v++) {
    int32_t s = site_of[v];
    if (s < 0) continue;
    int32_t cv = comp[v];
    int64_t x = v % nx, y = (v / nx) % ny, z = v / (nx * ny);
    double ax = ((double)x + 0.5) * sx, ay = ((double)y + 0.5) * sy,
           az = ((double)z + 0.5) * sz;
    int ok;
    if (src[v] == v) {
      ok = seg_clear(comp, &g, ax, ay, az, site_pos[3 * (int64_t)s],
                     site_pos[3 * (int64_t)s + 1], site_pos[3 * (int64_t)s + 2], cv);
    } else if (src[v] < 0) {
      ok = 0;
    } else {
      int64_t u = src[v];
      int64_t ux = u % nx, uy = (u / nx) % ny, uz = u / (nx * ny);
      ok = seg_clear(comp, &g, ax, ay, az, ((double)ux + 0.5) * sx,
                     ((double)uy + 0.5) * sy, ((double)uz + 0.5) * sz, cv);
    }
    out_bad[v] = ok ? 0 : 1;
  }
}

int orc_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* thread count of the eval loops (torchrun exports OMP_NUM_THREADS=1 to every
 * rank; the CPU arm sets all host threads explicitly) */
void orc_set_num_threads(int n) {
#ifdef _OPENMP
  extern void omp_set_num_threads(int);
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
