/*
 * tgs_workload.c -- seeded synthetic inputs (see tgs_workload.h).
 * Input generation only: no culling, selection or optimiser arithmetic here.
 */
#include "tgs_workload.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define PHI1 0x9E3779B97F4A7C15ull
#define PHI2 0xC2B2AE3D27D4EB4Full
#define PHI3 0x165667B19E3779F9ull

uint64_t wl_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static uint64_t h3(uint64_t seed, uint64_t a, uint64_t b) {
  return wl_splitmix64(seed ^ wl_splitmix64(a * PHI1 ^ wl_splitmix64(b + PHI3)));
}
/* uniform in [0,1) with 53 bits */
static double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }
/* approx N(0,1): Irwin-Hall sum of 4 uniforms, rescaled (input generator only) */
static double nrm(uint64_t seed, uint64_t gid, uint64_t stream) {
  double s = 0.0;
  for (int i = 0; i < 4; ++i) s += u01(h3(seed, gid, stream * 8 + (uint64_t)i));
  return (s - 2.0) * 1.7320508075688772; /* var of sum = 4/12 */
}

/* ------------------------------------------------------------------ scene */
struct wl_scene {
  wl_scene_params p;
  uint64_t K;
  uint64_t W, H;
  double tile;
  double sigma;
  uint32_t* tix;
  uint32_t* tiy;
};

static uint64_t morton2(uint32_t x, uint32_t y) {
  uint64_t c = 0;
  for (int b = 0; b < 32; ++b) {
    c |= (uint64_t)((x >> b) & 1u) << (2 * b);      /* x lowest */
    c |= (uint64_t)((y >> b) & 1u) << (2 * b + 1);
  }
  return c;
}

typedef struct { uint64_t code; uint64_t idx; } mkey;
static int mkey_cmp(const void* a, const void* b) {
  const mkey* x = (const mkey*)a;
  const mkey* y = (const mkey*)b;
  if (x->code != y->code) return x->code < y->code ? -1 : 1;
  if (x->idx != y->idx) return x->idx < y->idx ? -1 : 1; /* ties by index */
  return 0;
}

wl_scene* wl_scene_create(const wl_scene_params* p) {
  if (!p || p->n_gaussians == 0 || p->block_size < 4 || (p->block_size % 4) != 0) return NULL;
  wl_scene* s = (wl_scene*)calloc(1, sizeof(wl_scene));
  s->p = *p;
  s->K = (p->n_gaussians + p->block_size - 1) / p->block_size;
  uint64_t W = (uint64_t)ceil(sqrt((double)s->K));
  while (W * W < s->K) ++W;
  while (W > 1 && (W - 1) * (W - 1) >= s->K) --W;
  s->W = W;
  s->H = (s->K + W - 1) / W;
  s->tile = p->side / (double)W;
  s->sigma = s->tile / sqrt((double)p->block_size);
  s->tix = (uint32_t*)malloc(sizeof(uint32_t) * s->K);
  s->tiy = (uint32_t*)malloc(sizeof(uint32_t) * s->K);
  mkey* keys = (mkey*)malloc(sizeof(mkey) * s->K);
  for (uint64_t i = 0; i < s->K; ++i) {
    keys[i].code = morton2((uint32_t)(i % W), (uint32_t)(i / W));
    keys[i].idx = i;
  }
  qsort(keys, s->K, sizeof(mkey), mkey_cmp);
  for (uint64_t k = 0; k < s->K; ++k) {
    s->tix[k] = (uint32_t)(keys[k].idx % W);
    s->tiy[k] = (uint32_t)(keys[k].idx / W);
  }
  free(keys);
  return s;
}

void wl_scene_destroy(wl_scene* s) {
  if (!s) return;
  free(s->tix);
  free(s->tiy);
  free(s);
}

uint64_t wl_num_blocks(const wl_scene* s) { return s->K; }
double wl_sigma(const wl_scene* s) { return s->sigma; }

uint32_t wl_block_rows(const wl_scene* s, uint64_t k) {
  uint64_t B = s->p.block_size;
  uint64_t lo = k * B;
  if (lo >= s->p.n_gaussians) return 0;
  uint64_t r = s->p.n_gaussians - lo;
  return (uint32_t)(r < B ? r : B);
}

static double tile_height(const wl_scene* s, double xc, double yc) {
  const wl_scene_params* p = &s->p;
  double half = 0.5 * p->side;
  double fx = xc + half, fy = yc + half;
  double lx = floor(fx / p->lot), ly = floor(fy / p->lot);
  double ux = fx - lx * p->lot, uy = fy - ly * p->lot;
  double a = 0.5 * (p->lot - p->footprint), b = 0.5 * (p->lot + p->footprint);
  if (ux >= a && ux < b && uy >= a && uy < b) {
    uint64_t lot_id = (uint64_t)(int64_t)lx * 1000003ull + (uint64_t)(int64_t)ly;
    return p->hmin + (p->hmax - p->hmin) * u01(h3(p->seed, lot_id, 0x10700ull));
  }
  return p->ground_h;
}

void wl_block_tile(const wl_scene* s, uint64_t k, int64_t* ix, int64_t* iy, double* x0,
                   double* y0, double* tile, double* h) {
  double half = 0.5 * s->p.side;
  *ix = s->tix[k];
  *iy = s->tiy[k];
  *tile = s->tile;
  *x0 = -half + s->tile * (double)s->tix[k];
  *y0 = -half + s->tile * (double)s->tiy[k];
  *h = tile_height(s, *x0 + 0.5 * s->tile, *y0 + 0.5 * s->tile);
}

static float round_up_f(double v) {
  float f = (float)v;
  if ((double)f < v) f = nextafterf(f, INFINITY);
  return f;
}

void wl_bounds(const wl_scene* s, uint64_t k0, uint64_t k1, float* out) {
  if (s->p.layout == 1) { /* unsorted: every block spans the city */
    double half = 0.5 * s->p.side, hm = s->p.hmax;
    double r = sqrt(2.0 * half * half + 0.25 * hm * hm) + 4.5 * s->sigma + 1e-3 * s->p.side;
    for (uint64_t k = k0; k < k1; ++k) {
      float* o = out + 4 * (k - k0);
      o[0] = 0.0f;
      o[1] = 0.0f;
      o[2] = (float)(0.5 * hm);
      o[3] = round_up_f(r);
    }
    return;
  }
  for (uint64_t k = k0; k < k1; ++k) {
    int64_t ix, iy;
    double x0, y0, t, h;
    wl_block_tile(s, k, &ix, &iy, &x0, &y0, &t, &h);
    float cx = (float)(x0 + 0.5 * t), cy = (float)(y0 + 0.5 * t), cz = (float)(0.5 * h);
    double r2 = 0.0;
    for (int c = 0; c < 8; ++c) {
      double px = (c & 1) ? x0 + t : x0, py = (c & 2) ? y0 + t : y0, pz = (c & 4) ? h : 0.0;
      double dx = px - cx, dy = py - cy, dz = pz - cz;
      double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 > r2) r2 = d2;
    }
    /* + 3 * max scale (1.5 sigma) (SPEC.md:130-131 extent = 3 * largest scale)
       + slack for fp32 rounding of the stored centres */
    double slack = 1e-5 * (1.0 + fabs(x0) + fabs(y0) + t + h);
    double r = sqrt(r2) + 4.5 * s->sigma + slack;
    float* o = out + 4 * (k - k0);
    o[0] = cx;
    o[1] = cy;
    o[2] = cz;
    o[3] = round_up_f(r);
  }
}

/* one row (gid = k*B + r) of the table; layout 1 places it in a random tile */
void wl_row_theta(const wl_scene* s, uint64_t gid, float* row) {
  const uint32_t B = s->p.block_size;
  int64_t ix, iy;
  double x0, y0, t, h;
  wl_block_tile(s, s->p.layout == 1 ? h3(s->p.seed, gid, 7) % s->K : gid / B, &ix, &iy, &x0,
                &y0, &t, &h);
  const uint64_t seed = s->p.seed;
  const double sig = s->sigma;
  row[0] = (float)(x0 + t * u01(h3(seed, gid, 1)));
  row[1] = (float)(y0 + t * u01(h3(seed, gid, 2)));
  row[2] = (float)(h * u01(h3(seed, gid, 3)));
  for (int a = 0; a < 3; ++a) row[3 + a] = (float)(0.3 * nrm(seed, gid, 10 + a));
  for (int a = 0; a < 45; ++a) row[6 + a] = (float)(0.02 * nrm(seed, gid, 20 + a));
  row[51] = (float)(1.5 * nrm(seed, gid, 70));
  row[52] = (float)log(sig * (0.5 + u01(h3(seed, gid, 80))));
  row[53] = (float)log(sig * (0.5 + u01(h3(seed, gid, 81))));
  row[54] = (float)log(0.1 * sig);
  double q[4], n2 = 0.0;
  for (int a = 0; a < 4; ++a) {
    q[a] = nrm(seed, gid, 90 + a);
    n2 += q[a] * q[a];
  }
  if (n2 < 1e-12) {
    q[0] = 1.0;
    q[1] = q[2] = q[3] = 0.0;
    n2 = 1.0;
  }
  double inv = 1.0 / sqrt(n2);
  for (int a = 0; a < 4; ++a) row[55 + a] = (float)(q[a] * inv);
}

void wl_block_theta(const wl_scene* s, uint64_t k, float* out) {
  const uint32_t B = s->p.block_size;
  const uint32_t rows = wl_block_rows(s, k);
  memset(out, 0, sizeof(float) * (size_t)B * WL_DIM);
  for (uint32_t r = 0; r < rows; ++r) wl_row_theta(s, k * (uint64_t)B + r, out + (size_t)r * WL_DIM);
}

/* block k of the table whose row i is the generator's row perm[i] (a Morton
   layout built by tgs_build_layout / or_build_layout over an unsorted scene) */
void wl_perm_fill_cb(void* user, uint64_t k, float* out) {
  const wl_perm_fill* f = (const wl_perm_fill*)user;
  const uint32_t B = f->scene->p.block_size;
  memset(out, 0, sizeof(float) * (size_t)B * WL_DIM);
  for (uint32_t r = 0; r < B; ++r) {
    const uint64_t p = k * (uint64_t)B + r;
    if (p >= f->n) break;
    wl_row_theta(f->scene, f->perm[p], out + (size_t)r * WL_DIM);
  }
}

/* (cx, cy, cz, max log-scale) of every logical row of block k: the same values
   wl_block_theta produces for attrs 0..2 and max(52..54), without the rest */
void wl_block_cs(const wl_scene* s, uint64_t k, float* out) {
  const uint32_t B = s->p.block_size;
  const uint32_t rows = wl_block_rows(s, k);
  int64_t ix, iy;
  double x0, y0, t, h;
  wl_block_tile(s, k, &ix, &iy, &x0, &y0, &t, &h);
  const uint64_t seed = s->p.seed;
  const double sig = s->sigma;
  for (uint32_t r = 0; r < rows; ++r) {
    uint64_t gid = k * (uint64_t)B + r;
    float* o = out + 4 * (size_t)r;
    if (s->p.layout == 1) {
      uint64_t kt = h3(seed, gid, 7) % s->K;
      wl_block_tile(s, kt, &ix, &iy, &x0, &y0, &t, &h);
    }
    o[0] = (float)(x0 + t * u01(h3(seed, gid, 1)));
    o[1] = (float)(y0 + t * u01(h3(seed, gid, 2)));
    o[2] = (float)(h * u01(h3(seed, gid, 3)));
    float a = (float)log(sig * (0.5 + u01(h3(seed, gid, 80))));
    float b = (float)log(sig * (0.5 + u01(h3(seed, gid, 81))));
    float c = (float)log(0.1 * sig);
    float m = a;
    if (b > m) m = b;
    if (c > m) m = c;
    o[3] = m;
  }
}

typedef struct { const wl_scene* s; float* out; uint64_t k0, k1; } cs_job;
static void* cs_worker(void* arg) {
  cs_job* j = (cs_job*)arg;
  for (uint64_t k = j->k0; k < j->k1; ++k)
    wl_block_cs(j->s, k, j->out + 4 * (size_t)k * j->s->p.block_size);
  return NULL;
}

/* all N rows as [N][4] (rows in block order, padding excluded) */
void wl_table_cs(const wl_scene* s, float* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  cs_job jobs[256];
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].s = s;
    jobs[i].out = out;
    jobs[i].k0 = s->K * (uint64_t)i / (uint64_t)nthreads;
    jobs[i].k1 = s->K * (uint64_t)(i + 1) / (uint64_t)nthreads;
    pthread_create(&th[i], NULL, cs_worker, &jobs[i]);
  }
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

void wl_block_theta_cb(void* scene, uint64_t k, float* out) {
  wl_block_theta((const wl_scene*)scene, k, out);
}

typedef struct {
  const wl_scene* s;
  float* out;
  uint64_t k0, k1;
} table_job;

static void* table_worker(void* arg) {
  table_job* j = (table_job*)arg;
  size_t rec = (size_t)j->s->p.block_size * WL_DIM;
  for (uint64_t k = j->k0; k < j->k1; ++k) wl_block_theta(j->s, k, j->out + rec * k);
  return NULL;
}

void wl_table(const wl_scene* s, float* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  table_job jobs[256];
  uint64_t K = s->K;
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].s = s;
    jobs[i].out = out;
    jobs[i].k0 = K * (uint64_t)i / (uint64_t)nthreads;
    jobs[i].k1 = K * (uint64_t)(i + 1) / (uint64_t)nthreads;
    pthread_create(&th[i], NULL, table_worker, &jobs[i]);
  }
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

/* ---------------------------------------------------------------- cameras */
static void cross3(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}
static double dot3(const double a[3], const double b[3]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
static void norm3(double a[3]) {
  double n = sqrt(dot3(a, a));
  a[0] /= n;
  a[1] /= n;
  a[2] /= n;
}

void wl_camera_look(wl_camera* c, const double pos[3], const double fwd[3],
                    const double up_hint[3], double fovx_deg, uint32_t w, uint32_t h,
                    double znear, double zfar) {
  memset(c, 0, sizeof(*c));
  for (int i = 0; i < 3; ++i) {
    c->pos[i] = pos[i];
    c->fwd[i] = fwd[i];
  }
  norm3(c->fwd);
  double up[3] = {up_hint[0], up_hint[1], up_hint[2]};
  cross3(c->fwd, up, c->right);           /* x = fwd x up  */
  norm3(c->right);
  cross3(c->fwd, c->right, c->down);      /* y = fwd x right (down) */
  norm3(c->down);
  c->width = w;
  c->height = h;
  c->fx = 0.5 * (double)w / tan(0.5 * fovx_deg * M_PI / 180.0);
  c->fy = c->fx;
  c->cx = 0.5 * (double)w;
  c->cy = 0.5 * (double)h;
  c->znear = znear;
  c->zfar = zfar;
}

/* camera coords: p_c = R (p - pos), rows of R = right, down, fwd */
void wl_camera_planes(const wl_camera* c, float out[6][4]) {
  double pc[6][4] = {
      {c->fx, 0.0, c->cx, 0.0},                         /* left:   fx x + cx z >= 0 */
      {-c->fx, 0.0, (double)c->width - c->cx, 0.0},     /* right */
      {0.0, c->fy, c->cy, 0.0},                         /* top */
      {0.0, -c->fy, (double)c->height - c->cy, 0.0},    /* bottom */
      {0.0, 0.0, 1.0, -c->znear},                       /* near */
      {0.0, 0.0, -1.0, c->zfar},                        /* far */
  };
  for (int p = 0; p < 6; ++p) {
    double n = sqrt(pc[p][0] * pc[p][0] + pc[p][1] * pc[p][1] + pc[p][2] * pc[p][2]);
    double nc[3] = {pc[p][0] / n, pc[p][1] / n, pc[p][2] / n};
    double d0 = pc[p][3] / n;
    double nw[3];
    for (int i = 0; i < 3; ++i) nw[i] = nc[0] * c->right[i] + nc[1] * c->down[i] + nc[2] * c->fwd[i];
    /* n_c.(R(p-pos)) + d0 = n_w.p - n_w.pos + d0 */
    double dw = d0 - dot3(nw, c->pos);
    out[p][0] = (float)nw[0];
    out[p][1] = (float)nw[1];
    out[p][2] = (float)nw[2];
    out[p][3] = (float)dw;
  }
}

int wl_camera_sees(const wl_camera* c, const double p[3]) {
  double d[3] = {p[0] - c->pos[0], p[1] - c->pos[1], p[2] - c->pos[2]};
  double x = dot3(c->right, d), y = dot3(c->down, d), z = dot3(c->fwd, d);
  if (!(z >= c->znear && z <= c->zfar)) return 0;
  double u = c->fx * x / z + c->cx, v = c->fy * y / z + c->cy;
  return u >= 0.0 && u <= (double)c->width && v >= 0.0 && v <= (double)c->height;
}

struct wl_traj {
  wl_traj_params p;
  const wl_scene* s;
  uint64_t n_views;
  uint32_t views_per_wp;
  uint64_t n_lines, wp_per_line;
  double line0, line_pitch;   /* first line coordinate and pitch */
  double along0, along1;      /* extent along a line */
  double center[3], radius;   /* orbit */
  uint64_t* order;            /* NULL = smooth */
};

wl_traj* wl_traj_create(const wl_scene* s, const wl_traj_params* p) {
  wl_traj* t = (wl_traj*)calloc(1, sizeof(wl_traj));
  t->p = *p;
  t->s = s;
  double half = 0.5 * s->p.side;
  double ymax = -half + s->tile * (double)s->H;
  if (p->kind == WL_TRAJ_ORBIT) {
    /* centroid of block centres and enclosing radius */
    uint64_t K = s->K;
    float* b = (float*)malloc(sizeof(float) * 4 * K);
    wl_bounds(s, 0, K, b);
    double c[3] = {0, 0, 0};
    for (uint64_t k = 0; k < K; ++k)
      for (int i = 0; i < 3; ++i) c[i] += b[4 * k + i];
    for (int i = 0; i < 3; ++i) c[i] /= (double)K;
    double R = 0.0;
    for (uint64_t k = 0; k < K; ++k) {
      double dx = b[4 * k] - c[0], dy = b[4 * k + 1] - c[1], dz = b[4 * k + 2] - c[2];
      double r = sqrt(dx * dx + dy * dy + dz * dz) + b[4 * k + 3];
      if (r > R) R = r;
    }
    free(b);
    for (int i = 0; i < 3; ++i) t->center[i] = c[i];
    t->radius = R;
    t->n_views = p->n_views ? p->n_views : 16;
    t->views_per_wp = 1;
  } else if (p->kind == WL_TRAJ_AERIAL) {
    t->views_per_wp = 5;          /* nadir + 4 obliques */
    t->line_pitch = p->strip;
    t->line0 = -half + 0.5 * p->strip;
    t->n_lines = (uint64_t)floor((ymax - t->line0) / p->strip) + 1;
    t->along0 = -half;
    t->along1 = half;
    t->wp_per_line = (uint64_t)floor((t->along1 - t->along0) / p->spacing) + 1;
    t->n_views = t->n_lines * t->wp_per_line * t->views_per_wp;
  } else {
    t->views_per_wp = 4;          /* front, back, left, right */
    t->line_pitch = s->p.lot;     /* street centrelines at lot boundaries */
    t->line0 = -half + s->p.lot;
    t->n_lines = (uint64_t)floor((ymax - 1.0 - t->line0) / s->p.lot) + 1;
    if (t->line0 >= ymax) t->n_lines = 1, t->line0 = 0.5 * (-half + ymax);
    t->along0 = -half + 1.0;
    t->along1 = half - 1.0;
    t->wp_per_line = (uint64_t)floor((t->along1 - t->along0) / p->spacing) + 1;
    t->n_views = t->n_lines * t->wp_per_line * t->views_per_wp;
  }
  return t;
}

void wl_traj_destroy(wl_traj* t) {
  if (!t) return;
  free(t->order);
  free(t);
}

uint64_t wl_traj_num_views(const wl_traj* t) { return t->n_views; }

void wl_traj_view(const wl_traj* t, uint64_t i, wl_camera* out) {
  const wl_traj_params* p = &t->p;
  i %= t->n_views;
  double zup[3] = {0, 0, 1};
  if (p->kind == WL_TRAJ_ORBIT) {
    double ang = 2.0 * M_PI * (double)i / (double)t->n_views;
    double el = p->altitude * M_PI / 180.0;
    double R = p->radius_scale * t->radius;
    double pos[3] = {t->center[0] + R * cos(el) * cos(ang), t->center[1] + R * cos(el) * sin(ang),
                     t->center[2] + R * sin(el)};
    double fwd[3] = {t->center[0] - pos[0], t->center[1] - pos[1], t->center[2] - pos[2]};
    wl_camera_look(out, pos, fwd, zup, p->fovx_deg, p->width, p->height, p->znear * t->radius,
                   p->zfar * t->radius);
    return;
  }
  uint64_t wp = i / t->views_per_wp, v = i % t->views_per_wp;
  uint64_t line = wp / t->wp_per_line, j = wp % t->wp_per_line;
  double along = t->along0 + p->spacing * (double)j;
  double dir = 1.0;
  if (line & 1) { /* lawnmower: alternate direction */
    along = t->along1 - p->spacing * (double)j;
    dir = -1.0;
  }
  double cross = t->line0 + t->line_pitch * (double)line;
  double pos[3] = {along, cross, p->altitude};
  double fwd[3], up[3] = {0, 0, 1};
  if (p->kind == WL_TRAJ_AERIAL) {
    if (v == 0) {
      fwd[0] = 0;
      fwd[1] = 0;
      fwd[2] = -1;
      up[0] = dir;
      up[1] = 0;
      up[2] = 0;
    } else {
      double hd = (double)(v - 1) * 0.5 * M_PI, c45 = sqrt(0.5);
      fwd[0] = c45 * cos(hd);
      fwd[1] = c45 * sin(hd);
      fwd[2] = -c45;
    }
  } else {
    double hd[4] = {0.0, M_PI, 0.5 * M_PI, 1.5 * M_PI};
    double a = hd[v] + (dir < 0 ? M_PI : 0.0);
    fwd[0] = cos(a);
    fwd[1] = sin(a);
    fwd[2] = 0.0;
  }
  wl_camera_look(out, pos, fwd, up, p->fovx_deg, p->width, p->height, p->znear, p->zfar);
}

void wl_traj_set_order(wl_traj* t, int shuffled, uint64_t seed) {
  free(t->order);
  t->order = NULL;
  if (!shuffled) return;
  uint64_t n = t->n_views;
  t->order = (uint64_t*)malloc(sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < n; ++i) t->order[i] = i;
  for (uint64_t i = n - 1; i > 0; --i) { /* Fisher-Yates */
    uint64_t r = h3(seed, i, 0x5107ull);
    uint64_t j = (uint64_t)(((unsigned __int128)r * (unsigned __int128)(i + 1)) >> 64);
    uint64_t tmp = t->order[i];
    t->order[i] = t->order[j];
    t->order[j] = tmp;
  }
}

void wl_traj_set_perm(wl_traj* t, const uint64_t* perm) {
  uint64_t n = t->n_views;
  uint64_t* o = (uint64_t*)malloc(sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < n; ++i) o[i] = t->order ? t->order[perm[i]] : perm[i];
  free(t->order);
  t->order = o;
}

void wl_traj_features(const wl_traj* t, double focus, double* out) {
  for (uint64_t i = 0; i < t->n_views; ++i) {
    wl_camera c;
    wl_traj_view(t, t->order ? t->order[i] : i, &c);
    for (int a = 0; a < 3; ++a) {
      out[6 * i + a] = c.pos[a];
      out[6 * i + 3 + a] = c.pos[a] + focus * c.fwd[a];
    }
  }
}

void wl_traj_batch_cameras(const wl_traj* t, uint64_t b, uint32_t J, wl_camera* out) {
  for (uint32_t j = 0; j < J; ++j) {
    uint64_t idx = (b * (uint64_t)J + j) % t->n_views;
    if (t->order) idx = t->order[idx];
    wl_traj_view(t, idx, &out[j]);
  }
}

void wl_traj_batch_planes(const wl_traj* t, uint64_t b, uint32_t J, float* out) {
  for (uint32_t j = 0; j < J; ++j) {
    wl_camera c;
    uint64_t idx = (b * (uint64_t)J + j) % t->n_views;
    if (t->order) idx = t->order[idx];
    wl_traj_view(t, idx, &c);
    wl_camera_planes(&c, (float(*)[4])(out + 24 * (size_t)j));
  }
}

/* -------------------------------------------------------------- gradients */
float wl_grad(uint64_t seed, uint64_t gid, uint32_t a, uint64_t t) {
  uint64_t x = wl_splitmix64(seed ^ (PHI1 * (gid * WL_DIM + a)) ^ (PHI2 * t));
  int32_t q = (int32_t)(x >> 40) - (1 << 23);
  return (float)q * 0x1p-33f;
}

void wl_grad_block(uint64_t seed, uint64_t k, uint32_t B, uint32_t rows, uint64_t t,
                   float* out) {
  memset(out, 0, sizeof(float) * (size_t)B * WL_DIM);
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t a = 0; a < WL_DIM; ++a)
      out[(size_t)r * WL_DIM + a] = wl_grad(seed, k * (uint64_t)B + r, a, t);
}

int wl_mask_bit(uint64_t seed, uint64_t gid, uint64_t t, uint32_t p32) {
  uint64_t x = wl_splitmix64(seed ^ (PHI3 * gid) ^ (PHI2 * t));
  return (uint32_t)(x >> 32) < p32;
}

void wl_mask_block(uint64_t seed, uint64_t k, uint32_t B, uint32_t rows, uint64_t t,
                   uint32_t p32, uint32_t* words) {
  uint32_t nw = (B + 31) / 32;
  memset(words, 0, sizeof(uint32_t) * nw);
  for (uint32_t r = 0; r < rows; ++r)
    if (wl_mask_bit(seed, k * (uint64_t)B + r, t, p32)) words[r / 32] |= 1u << (r % 32);
}

static uint32_t synth_rows(const wl_synth* s, uint64_t k) {
  uint64_t lo = k * (uint64_t)s->block_size;
  if (lo >= s->n_gaussians) return 0;
  uint64_t r = s->n_gaussians - lo;
  return (uint32_t)(r < s->block_size ? r : s->block_size);
}

void wl_grad_cb(void* synth, uint64_t k, uint64_t t, float* out) {
  const wl_synth* s = (const wl_synth*)synth;
  wl_grad_block(s->seed, k, s->block_size, synth_rows(s, k), t, out);
}

void wl_mask_cb(void* synth, uint64_t k, uint64_t t, uint32_t* words) {
  const wl_synth* s = (const wl_synth*)synth;
  wl_mask_block(s->seed, k, s->block_size, synth_rows(s, k), t, s->p32, words);
}
