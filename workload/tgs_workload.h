/*
 * tgs_workload.h -- seeded synthetic INPUT generators shared by the CUDA path
 * and the CPU oracle.
 *
 * This module holds none of the method's arithmetic (no culling, no residency
 * selection, no Adam).  It only produces inputs, deterministically from seeds:
 *   - a Morton-ordered, block-partitioned Gaussian table Theta (N x 59 fp32)
 *     shaped like an aerial/street city scene (Eq. block_def;
 *     row order = Morton order of the 2-D tile each block covers),
 *   - the per-block bounding spheres (c_k, r_k), computed
 *     conservatively from the tile box the generator fills,
 *   - camera trajectories (orbit / aerial lawnmower / street) and their 6
 *     frustum planes ("standard 6-plane frustum test"),
 *   - counter-based synthetic gradients and row masks (the renderer's
 *     backward pass is out of scope; SURVEY.md §8d "Gradients").
 *
 * Every random number is a pure function of (seed, index, stream) through
 * splitmix64, so generation is parallel and reproducible.  The gradient
 * generator has a CUDA twin (tgs_workload_cuda.cu) that is bit-identical.
 */
#ifndef TGS_WORKLOAD_H
#define TGS_WORKLOAD_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define WL_DIM 59

/* ------------------------------------------------------------------ scene */
typedef struct {
  uint64_t n_gaussians;   /* N >= 1 */
  uint32_t block_size;    /* B >= 4, B % 4 == 0 */
  uint32_t layout;        /* 0: Morton-ordered tiles; 1: no spatial sort
                             ("w/o Morton" ablation): every block's rows
                             are scattered over the whole city */
  uint64_t seed;          /* scene seed (20150 in the bench) */
  double side;            /* city side length in metres */
  double lot;             /* lot pitch (50 m) */
  double footprint;       /* building footprint inside a lot (30 m) */
  double hmin, hmax;      /* building height range (10..100 m) */
  double ground_h;        /* thickness of the street/ground slab (0.5 m) */
} wl_scene_params;

typedef struct wl_scene wl_scene;   /* opaque: holds the Morton tile table */

wl_scene* wl_scene_create(const wl_scene_params* p);
void      wl_scene_destroy(wl_scene* s);
uint64_t  wl_num_blocks(const wl_scene* s);            /* K = ceil(N/B) */
uint32_t  wl_block_rows(const wl_scene* s, uint64_t k); /* logical rows of block k */
/* tile of block k: integer tile coords, tile origin/size, height */
void      wl_block_tile(const wl_scene* s, uint64_t k, int64_t* ix, int64_t* iy,
                        double* x0, double* y0, double* tile, double* h);
double    wl_sigma(const wl_scene* s);                  /* mean Gaussian spacing */
/* bounds of global blocks [k0,k1): float4 (cx,cy,cz,r), r rounded up */
void      wl_bounds(const wl_scene* s, uint64_t k0, uint64_t k1, float* out);
/* Theta rows of one global block: B x 59 fp32, rows >= rows(k) zero */
void      wl_block_theta(const wl_scene* s, uint64_t k, float* out);
/* (cx, cy, cz, max log-scale) of block k's rows / of all N rows [N][4] */
void      wl_block_cs(const wl_scene* s, uint64_t k, float* out);
void      wl_table_cs(const wl_scene* s, float* out, int nthreads);
/* one generator row by its global row id */
void      wl_row_theta(const wl_scene* s, uint64_t gid, float* row);
/* fill callback of a permuted (re-blocked) table: block k = rows perm[kB ..] */
typedef struct { const wl_scene* scene; const uint64_t* perm; uint64_t n; } wl_perm_fill;
void      wl_perm_fill_cb(void* user, uint64_t k, float* out);
/* callback form for the oracle's lazily materialised host tier */
void      wl_block_theta_cb(void* scene, uint64_t k, float* out);
/* the whole table [K*B][59] (padding rows zero), nthreads workers */
void      wl_table(const wl_scene* s, float* out, int nthreads);

/* ---------------------------------------------------------------- cameras */
typedef struct {
  double pos[3];
  double fwd[3];     /* unit forward (camera +z) */
  double right[3];   /* unit right   (camera +x) */
  double down[3];    /* unit down    (camera +y) */
  double fx, fy, cx, cy;
  uint32_t width, height;
  double znear, zfar;
} wl_camera;

/* camera looking along fwd (up_hint used to fix roll); fovx in degrees */
void wl_camera_look(wl_camera* c, const double pos[3], const double fwd[3],
                    const double up_hint[3], double fovx_deg, uint32_t w,
                    uint32_t h, double znear, double zfar);
/* 6 planes (nx,ny,nz,d0), unit normals, inside iff n.p + d0 >= 0, computed
 * in double and rounded to fp32: left, right, top, bottom, near, far */
void wl_camera_planes(const wl_camera* c, float out[6][4]);
/* pinhole test of a point (double): inside image with near<=z<=far */
int  wl_camera_sees(const wl_camera* c, const double p[3]);

typedef enum { WL_TRAJ_ORBIT = 0, WL_TRAJ_AERIAL = 1, WL_TRAJ_STREET = 2 } wl_traj_kind;
typedef struct {
  int32_t kind;
  uint32_t n_views;     /* orbit: number of poses; others: 0 = derived from path */
  double altitude;      /* aerial: 150 m; street: camera height 2 m; orbit: elevation deg */
  double spacing;       /* waypoint spacing (m) */
  double strip;         /* aerial strip spacing (m) */
  double fovx_deg;
  double znear, zfar;
  uint32_t width, height;
  double radius_scale;  /* orbit: orbit radius / scene radius */
} wl_traj_params;

typedef struct wl_traj wl_traj;
wl_traj*  wl_traj_create(const wl_scene* s, const wl_traj_params* p);
void      wl_traj_destroy(wl_traj* t);
uint64_t  wl_traj_num_views(const wl_traj* t);
void      wl_traj_view(const wl_traj* t, uint64_t i, wl_camera* out);
/* view order: 0 = smooth (path order), 1 = seeded Fisher-Yates shuffle */
void      wl_traj_set_order(wl_traj* t, int shuffled, uint64_t seed);
/* compose the current view order with perm (new position i = old position perm[i]) */
void      wl_traj_set_perm(wl_traj* t, const uint64_t* perm);
/* pose features of the views in the current order, out[M][6] = (centre,
 * centre + focus * forward): inputs of the f4 view ordering (no method arithmetic) */
void      wl_traj_features(const wl_traj* t, double focus, double* out);
/* planes of batch b: views order[b*J .. b*J+J) (wrapping), out[J][6][4] */
void      wl_traj_batch_planes(const wl_traj* t, uint64_t b, uint32_t J, float* out);
void      wl_traj_batch_cameras(const wl_traj* t, uint64_t b, uint32_t J, wl_camera* out);

/* -------------------------------------------------------------- gradients */
/* g(seed,gid,a,t) = ((int32)(x>>40) - 2^23) * 2^-33 with
 * x = splitmix64(seed ^ PHI1*(gid*59+a) ^ PHI2*t); exact in fp32, in
 * [-2^-10, 2^-10). */
float    wl_grad(uint64_t seed, uint64_t gid, uint32_t a, uint64_t t);
/* grads of global block k (rows(k) logical rows) at iteration t: B x 59,
 * padding rows zero */
void     wl_grad_block(uint64_t seed, uint64_t k, uint32_t B, uint32_t rows,
                       uint64_t t, float* out);
/* row mask bit: splitmix64(seed ^ PHI3*gid ^ PHI2*t) >> 32 < p32 */
int      wl_mask_bit(uint64_t seed, uint64_t gid, uint64_t t, uint32_t p32);
void     wl_mask_block(uint64_t seed, uint64_t k, uint32_t B, uint32_t rows,
                       uint64_t t, uint32_t p32, uint32_t* words);

uint64_t wl_splitmix64(uint64_t x);

/* callback adapters (oracle or_grad_fn / or_mask_fn signatures) */
typedef struct { uint64_t seed; uint64_t n_gaussians; uint32_t block_size; uint32_t p32; } wl_synth;
void wl_grad_cb(void* synth, uint64_t k, uint64_t t, float* out);
void wl_mask_cb(void* synth, uint64_t k, uint64_t t, uint32_t* words);

#ifdef __cplusplus
}
#endif
#endif
