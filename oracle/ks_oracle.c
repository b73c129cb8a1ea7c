/* CPU ORACLE for the perception hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's algorithms for
 *   depth/cuboid/sphere fusion into a block-sparse TSDF  (sdf_world.hpp)
 *   gather/scatter seeding, exact EDT, sign recovery, trilinear query (esdf.hpp)
 * Each function cites the reference lines it follows (paths relative to
 * /root/reference/proj/include/ks/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product (paper_2603_05493_b200/, include/) never does.
 *
 * Parity status: PINNED.  tests/test_oracle_vs_reference.py checks every
 * function here, bit for bit, against oracle/_ref/libks_ref.so (the reference's
 * own headers compiled unmodified by oracle/Makefile) on the SPEC.md known-answer
 * cases and on seeded random scenes; tests/golden/ holds vectors generated from
 * that reference build (tests/golden/make_golden.py) for boxes where the
 * reference tree is absent.
 * ONE EXCEPTION -- PARITY UNPINNED: ko_stamp_mesh / ko_mesh_sdf (triangle-mesh
 * stamping).  The reference has no mesh implementation and no test for one
 * (SPEC.md:8, :422), so that section restates this repo's own definition; see
 * the comment above it and tests/test_mesh_stamp.py for what anchors it.
 *
 * Third-party arithmetic: the reference's Vec3/Mat3 math is Eigen 3.x (version
 * unpinned, not vendored; core.hpp:18).  Restated here from Eigen's scalar
 * evaluation order for fixed-size 3-vectors: reductions are a0 + (a1 + a2),
 * normalized() is v / sqrt(v.v) with true per-component divisions.
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction).
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define KS_ORACLE_PREFIX ko_
#include "ks_oracle_api.h"

enum { EDGE = 8, VOX = 512 };
enum { SLOT_EMPTY = 0, SLOT_LIVE = 1, SLOT_TOMB = 2 };

typedef struct {
  int32_t x, y, z;
} key3;

struct ko_tsdf {
  double voxel, trunc, alpha_t, alpha_f, wthr;
  int capacity, nslots;
  key3* slot_key;
  int32_t* slot_pool;
  uint8_t* slot_state;
  int32_t* free_list;
  int free_count, next_fresh;
  double *sum, *wt, *geom; /* capacity * 512 each */
};

static _Thread_local char g_err[256];
static void set_err(const char* msg) { snprintf(g_err, sizeof g_err, "%s", msg); }
const char* ko_last_error(void) { return g_err; }

/* ---- 3-vector helpers (Eigen scalar-path order, see header) ---------------- */
typedef struct {
  double v[3];
} vec3;
static inline double sum3(double a, double b, double c) { return a + (b + c); }
static inline vec3 mk(double x, double y, double z) {
  vec3 r = {{x, y, z}};
  return r;
}
static inline vec3 mat_vec(const double m[9], vec3 p) {
  vec3 r;
  for (int i = 0; i < 3; ++i)
    r.v[i] = sum3(m[3 * i] * p.v[0], m[3 * i + 1] * p.v[1], m[3 * i + 2] * p.v[2]);
  return r;
}
static inline vec3 add(vec3 a, vec3 b) { return mk(a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]); }
static inline vec3 sub(vec3 a, vec3 b) { return mk(a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]); }
static inline double sqnorm(vec3 a) { return sum3(a.v[0] * a.v[0], a.v[1] * a.v[1], a.v[2] * a.v[2]); }
static inline vec3 unit(vec3 a) {
  const double z = sqnorm(a);
  if (z > 0.0) {
    const double n = sqrt(z);
    return mk(a.v[0] / n, a.v[1] / n, a.v[2] / n);
  }
  return a;
}
/* Pose * p = R p + t (core.hpp:64); inverse = (R^T, -(R^T t)) (core.hpp:66-71) */
typedef struct {
  double r[9];
  vec3 t;
} rigid_t;
static rigid_t mk_pose(const double r[9], const double t[3]) {
  rigid_t p;
  memcpy(p.r, r, sizeof p.r);
  p.t = mk(t[0], t[1], t[2]);
  return p;
}
static inline vec3 apply(const rigid_t* p, vec3 x) { return add(mat_vec(p->r, x), p->t); }
static rigid_t inverse(const rigid_t* p) {
  rigid_t q;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) q.r[3 * i + j] = p->r[3 * j + i];
  vec3 rt = mat_vec(q.r, p->t);
  q.t = mk(-rt.v[0], -rt.v[1], -rt.v[2]);
  return q;
}

/* ---- block hash (sdf_world.hpp:92-189) ------------------------------------ */
static uint64_t hash_key(key3 k) { /* :92-97 */
  return ((uint64_t)(uint32_t)k.x * 73856093ull) ^ ((uint64_t)(uint32_t)k.y * 19349663ull) ^
         ((uint64_t)(uint32_t)k.z * 83492791ull);
}
static int key_eq(key3 a, key3 b) { return a.x == b.x && a.y == b.y && a.z == b.z; }

static int table_find(const ko_tsdf* t, key3 k) { /* :132-142 */
  const size_t n = (size_t)t->nslots;
  size_t i = (size_t)(hash_key(k) % n);
  for (size_t probe = 0; probe < n; ++probe) {
    if (t->slot_state[i] == SLOT_EMPTY) return -1;
    if (t->slot_state[i] == SLOT_LIVE && key_eq(t->slot_key[i], k)) return t->slot_pool[i];
    i = (i + 1) % n;
  }
  return -1;
}
static int table_available(const ko_tsdf* t) { return t->free_count + (t->capacity - t->next_fresh); } /* :127-129 */

/* returns pool index, *created set; -1 pool exhausted, -2 table full (:146-172) */
static int table_insert(ko_tsdf* t, key3 k, int* created) {
  const size_t n = (size_t)t->nslots;
  size_t i = (size_t)(hash_key(k) % n);
  long first_tomb = -1;
  *created = 0;
  for (size_t probe = 0; probe < n; ++probe) {
    const uint8_t st = t->slot_state[i];
    if (st == SLOT_LIVE && key_eq(t->slot_key[i], k)) return t->slot_pool[i];
    if (st == SLOT_TOMB && first_tomb < 0) first_tomb = (long)i;
    if (st == SLOT_EMPTY) {
      const size_t target = first_tomb >= 0 ? (size_t)first_tomb : i;
      int pool;
      if (t->free_count > 0) pool = t->free_list[--t->free_count]; /* LIFO */
      else if (t->next_fresh < t->capacity) pool = t->next_fresh++;
      else return -1;
      t->slot_key[target] = k;
      t->slot_pool[target] = pool;
      t->slot_state[target] = SLOT_LIVE;
      *created = 1;
      return pool;
    }
    i = (i + 1) % n;
  }
  return -2;
}

static void block_reset(ko_tsdf* t, int pool) { /* :70-74 */
  double* s = t->sum + (size_t)pool * VOX;
  double* w = t->wt + (size_t)pool * VOX;
  double* g = t->geom + (size_t)pool * VOX;
  for (int i = 0; i < VOX; ++i) {
    s[i] = 0.0;
    w[i] = 0.0;
    g[i] = INFINITY;
  }
}

/* ---- index helpers (sdf_world.hpp:249-290) -------------------------------- */
static int32_t floor_div8(int32_t v) { return (int32_t)floor((double)v / EDGE); }
static void voxel_of(vec3 p, double voxel, int32_t out[3]) { /* :254-258 */
  for (int a = 0; a < 3; ++a) out[a] = (int32_t)floor(p.v[a] / voxel);
}
static key3 block_of(const int32_t vox[3]) { /* :260-263 */
  key3 k = {floor_div8(vox[0]), floor_div8(vox[1]), floor_div8(vox[2])};
  return k;
}
static vec3 voxel_center(key3 b, int local, double voxel) { /* :265-272 */
  const int lx = local % EDGE, ly = (local / EDGE) % EDGE, lz = local / (EDGE * EDGE);
  return mk((b.x * EDGE + lx + 0.5) * voxel, (b.y * EDGE + ly + 0.5) * voxel,
            (b.z * EDGE + lz + 0.5) * voxel);
}
static int wrap8(int32_t v) {
  const int32_t m = v % EDGE;
  return m < 0 ? m + EDGE : m;
}
static int local_of(const int32_t vox[3]) { /* :274-280 */
  return wrap8(vox[0]) + EDGE * (wrap8(vox[1]) + EDGE * wrap8(vox[2]));
}
static vec3 block_center(key3 b, double voxel) { /* :282-286 */
  return mk((b.x * EDGE + 0.5 * EDGE) * voxel, (b.y * EDGE + 0.5 * EDGE) * voxel,
            (b.z * EDGE + 0.5 * EDGE) * voxel);
}
static double block_radius(double voxel) { return 0.5 * EDGE * voxel * sqrt(3.0); } /* :288-290 */

/* ---- lifecycle ------------------------------------------------------------ */
ko_tsdf* ko_tsdf_create(const double cfg[5], int capacity, int slot_count) {
  /* TsdfConfig::validate (:47-53), make_tsdf (:327-334) */
  if (cfg[0] <= 0.0) return set_err("tsdf: voxel_size must be > 0"), NULL;
  if (cfg[1] < cfg[0]) return set_err("tsdf: truncation must be >= voxel_size"), NULL;
  if (!(cfg[2] > 0.0 && cfg[2] <= 1.0) || !(cfg[3] > 0.0 && cfg[3] <= 1.0))
    return set_err("tsdf: decay factors must lie in (0, 1]"), NULL;
  if (capacity < 1) return set_err("tsdf: capacity must be >= 1"), NULL;
  ko_tsdf* t = calloc(1, sizeof *t);
  t->voxel = cfg[0];
  t->trunc = cfg[1];
  t->alpha_t = cfg[2];
  t->alpha_f = cfg[3];
  t->wthr = cfg[4];
  t->capacity = capacity;
  t->nslots = slot_count > 0 ? slot_count : 2 * capacity;
  t->slot_key = calloc((size_t)t->nslots, sizeof(key3));
  t->slot_pool = malloc((size_t)t->nslots * sizeof(int32_t));
  for (int i = 0; i < t->nslots; ++i) t->slot_pool[i] = -1;
  t->slot_state = calloc((size_t)t->nslots, 1);
  t->free_list = malloc((size_t)capacity * sizeof(int32_t));
  t->sum = calloc((size_t)capacity * VOX, sizeof(double));
  t->wt = calloc((size_t)capacity * VOX, sizeof(double));
  t->geom = calloc((size_t)capacity * VOX, sizeof(double));
  return t;
}
void ko_tsdf_destroy(ko_tsdf* t) {
  if (!t) return;
  free(t->slot_key);
  free(t->slot_pool);
  free(t->slot_state);
  free(t->free_list);
  free(t->sum);
  free(t->wt);
  free(t->geom);
  free(t);
}

/* ---- allocation (sdf_world.hpp:307-323) ----------------------------------- */
static int key_cmp(const void* pa, const void* pb) {
  const key3 *a = pa, *b = pb;
  if (a->x != b->x) return a->x < b->x ? -1 : 1;
  if (a->y != b->y) return a->y < b->y ? -1 : 1;
  if (a->z != b->z) return a->z < b->z ? -1 : 1;
  return 0;
}
/* sorts + dedups keys in place; returns unique count or -1 (error set, nothing inserted) */
static long allocate_keys(ko_tsdf* t, key3* keys, long n) {
  qsort(keys, (size_t)n, sizeof(key3), key_cmp);
  long m = 0;
  for (long i = 0; i < n; ++i)
    if (m == 0 || !key_eq(keys[m - 1], keys[i])) keys[m++] = keys[i];
  int required = 0;
  for (long i = 0; i < m; ++i)
    if (table_find(t, keys[i]) < 0) ++required;
  if (required > table_available(t)) {
    snprintf(g_err, sizeof g_err,
             "tsdf: pool exhausted, frame requires %d new blocks but only %d are available",
             required, table_available(t));
    return -1;
  }
  for (long i = 0; i < m; ++i) {
    int created;
    const int pool = table_insert(t, keys[i], &created);
    if (pool == -1) return set_err("tsdf: block pool exhausted"), -1;
    if (pool == -2) return set_err("tsdf: hash table full"), -1;
    if (created) block_reset(t, pool);
  }
  return m;
}

static int depth_ok(float d) { return isfinite(d) && d > 0.0f; } /* :203 */

/* ---- integrate_depth (sdf_world.hpp:340-389) ------------------------------ */
int ko_integrate_depth(ko_tsdf* t, const float* depth, int width, int height, const double intr[4],
                       const double pose_R[9], const double pose_t[3]) {
  const double fx = intr[0], fy = intr[1], cx = intr[2], cy = intr[3];
  if (width <= 0 || height <= 0 || fx <= 0.0 || fy <= 0.0)
    return set_err("depth frame: invalid intrinsics"), -1; /* :197-199 */
  const double v = t->voxel, trunc = t->trunc;
  const rigid_t cam = mk_pose(pose_R, pose_t);

  /* phase 1: candidate blocks along each valid pixel's ray (:346-361) */
  const double step = 4.0 * v;
  int hs = (int)ceil(trunc / step);
  if (hs < 1) hs = 1;
  const long per_pixel = 2 * hs + 1;
  long cap = 1024, n = 0;
  key3* keys = malloc((size_t)cap * sizeof(key3));
  for (int py = 0; py < height; ++py)
    for (int px = 0; px < width; ++px) {
      const float d = depth[(long)py * width + px];
      if (!depth_ok(d)) continue;
      const vec3 surf = mk((px - cx) * d / fx, (py - cy) * d / fy, d);
      const vec3 dir = unit(surf);
      if (n + per_pixel > cap) {
        while (n + per_pixel > cap) cap *= 2;
        keys = realloc(keys, (size_t)cap * sizeof(key3));
      }
      for (int s = -hs; s <= hs; ++s) {
        double off = s * step;
        if (off < -trunc) off = -trunc; /* std::clamp */
        if (off > trunc) off = trunc;
        const vec3 sample = mk(surf.v[0] + off * dir.v[0], surf.v[1] + off * dir.v[1],
                               surf.v[2] + off * dir.v[2]);
        const vec3 world = apply(&cam, sample);
        int32_t vox[3];
        voxel_of(world, v, vox);
        keys[n++] = block_of(vox);
      }
    }
  if (n == 0) {
    free(keys);
    return 0;
  }
  /* phases 2+3 (:365) */
  const long m = allocate_keys(t, keys, n);
  if (m < 0) {
    free(keys);
    return -1;
  }
  /* phase 4: every voxel of every touched block projects into the image (:368-387) */
  const rigid_t w2c = inverse(&cam);
  for (long i = 0; i < m; ++i) {
    const int pool = table_find(t, keys[i]);
    double* S = t->sum + (size_t)pool * VOX;
    double* W = t->wt + (size_t)pool * VOX;
    for (int q = 0; q < VOX; ++q) {
      const vec3 c = apply(&w2c, voxel_center(keys[i], q, v));
      if (c.v[2] <= 0.0) continue;
      const int px = (int)lround(fx * c.v[0] / c.v[2] + cx);
      const int py = (int)lround(fy * c.v[1] / c.v[2] + cy);
      if (px < 0 || px >= width || py < 0 || py >= height) continue;
      const float d = depth[(long)py * width + px];
      if (!depth_ok(d)) continue;
      const double sd_raw = (double)d - c.v[2];
      if (sd_raw < -trunc) continue;
      const double sd = trunc < sd_raw ? trunc : sd_raw; /* std::min(sd_raw, trunc) */
      const double cc = (fx * v / c.v[2]) * (fy * v / c.v[2]);
      const double w = cc < 1.0 ? 1.0 : cc; /* std::max(c, 1.0) */
      S[q] += w * sd;
      W[q] += w;
    }
  }
  free(keys);
  return (int)m;
}

/* ---- analytic primitives (sdf_world.hpp:224-233) -------------------------- */
typedef struct {
  int is_sphere;
  rigid_t inv; /* cuboid: world -> local */
  vec3 he, center;
  double radius;
} prim_t;
static double prim_sdf(const prim_t* p, vec3 x) {
  if (p->is_sphere) return sqrt(sqnorm(sub(x, p->center))) - p->radius; /* :231-233 */
  const vec3 l = apply(&p->inv, x);                                    /* :225 */
  const vec3 q = mk(fabs(l.v[0]) - p->he.v[0], fabs(l.v[1]) - p->he.v[1], fabs(l.v[2]) - p->he.v[2]);
  /* std::max(q, 0.0) / std::min(max, 0.0) with the standard's argument order (:227-228) */
  const vec3 o = mk(q.v[0] < 0.0 ? 0.0 : q.v[0], q.v[1] < 0.0 ? 0.0 : q.v[1], q.v[2] < 0.0 ? 0.0 : q.v[2]);
  double mx = q.v[1] < q.v[2] ? q.v[2] : q.v[1];
  mx = q.v[0] < mx ? mx : q.v[0];
  return sqrt(sqnorm(o)) + (0.0 < mx ? 0.0 : mx);
}

static double prim_sdf_cb(const void* p, vec3 x) { return prim_sdf((const prim_t*)p, x); }

/* stamp_primitive after the AABB is known (sdf_world.hpp:418-443); the shape enters only through sdf() */
typedef double (*sdf_fn)(const void* shape, vec3 x);
static int stamp_shape(ko_tsdf* t, sdf_fn sdf, const void* p, vec3 lo, vec3 hi) {
  const double v = t->voxel, trunc = t->trunc;
  for (int a = 0; a < 3; ++a) {
    lo.v[a] -= trunc;
    hi.v[a] += trunc;
  }
  int32_t vlo[3], vhi[3];
  voxel_of(lo, v, vlo);
  voxel_of(hi, v, vhi);
  const key3 blo = block_of(vlo), bhi = block_of(vhi);
  const double reach = trunc + block_radius(v);
  long cap = 1024, n = 0;
  key3* keys = malloc((size_t)cap * sizeof(key3));
  for (int32_t bz = blo.z; bz <= bhi.z; ++bz)
    for (int32_t by = blo.y; by <= bhi.y; ++by)
      for (int32_t bx = blo.x; bx <= bhi.x; ++bx) {
        const key3 k = {bx, by, bz};
        if (fabs(sdf(p, block_center(k, v))) <= reach) {
          if (n == cap) keys = realloc(keys, (size_t)(cap *= 2) * sizeof(key3));
          keys[n++] = k;
        }
      }
  const long m = allocate_keys(t, keys, n);
  if (m < 0) {
    free(keys);
    return -1;
  }
  for (long i = 0; i < m; ++i) {
    double* G = t->geom + (size_t)table_find(t, keys[i]) * VOX;
    for (int q = 0; q < VOX; ++q) {
      const double sd = sdf(p, voxel_center(keys[i], q, v));
      if (sd < G[q]) G[q] = sd; /* std::min(G, sd) */
    }
  }
  free(keys);
  return 0;
}
static int stamp(ko_tsdf* t, const prim_t* p, vec3 lo, vec3 hi) { return stamp_shape(t, prim_sdf_cb, p, lo, hi); }

int ko_stamp_cuboid(ko_tsdf* t, const double pose_R[9], const double pose_t[3],
                    const double half_extents[3]) {
  /* :399-410 */
  for (int a = 0; a < 3; ++a)
    if (!isfinite(half_extents[a]) || !isfinite(pose_t[a])) return set_err("stamp: non-finite cuboid"), -1;
  const rigid_t pose = mk_pose(pose_R, pose_t);
  prim_t p;
  memset(&p, 0, sizeof p);
  p.inv = inverse(&pose);
  p.he = mk(half_extents[0], half_extents[1], half_extents[2]);
  vec3 lo = mk(INFINITY, INFINITY, INFINITY), hi = mk(-INFINITY, -INFINITY, -INFINITY);
  for (int corner = 0; corner < 8; ++corner) {
    const vec3 s = mk((corner & 1) ? 1.0 : -1.0, (corner & 2) ? 1.0 : -1.0, (corner & 4) ? 1.0 : -1.0);
    const vec3 w = apply(&pose, mk(s.v[0] * p.he.v[0], s.v[1] * p.he.v[1], s.v[2] * p.he.v[2]));
    for (int a = 0; a < 3; ++a) {
      if (w.v[a] < lo.v[a]) lo.v[a] = w.v[a];
      if (w.v[a] > hi.v[a]) hi.v[a] = w.v[a];
    }
  }
  return stamp(t, &p, lo, hi);
}

int ko_stamp_sphere(ko_tsdf* t, const double center[3], double radius) {
  /* :412-416 */
  if (!isfinite(center[0]) || !isfinite(center[1]) || !isfinite(center[2]) || !isfinite(radius))
    return set_err("stamp: non-finite sphere"), -1;
  prim_t p;
  memset(&p, 0, sizeof p);
  p.is_sphere = 1;
  p.center = mk(center[0], center[1], center[2]);
  p.radius = radius;
  return stamp(t, &p, mk(center[0] - radius, center[1] - radius, center[2] - radius),
               mk(center[0] + radius, center[1] + radius, center[2] + radius));
}


/* ---- triangle mesh stamping ------------------------------------------------
 * PARITY UNPINNED: the reference has NO mesh implementation and no test for one (SPEC.md:8 and :422
 * list triangle-mesh stamping out of scope; PAPER.md:293 only says "Cuboids and meshes are stamped
 * directly into the geometry channel").  What is restated here is therefore this repo's own
 * definition, modelled on stamp_primitive (sdf_world.hpp:394-444): the same AABB -> candidate
 * blocks -> allocate_keys -> per-voxel min, with the analytic distance replaced by the signed
 * distance to a closed, consistently oriented (outward, counter-clockwise) indexed triangle mesh:
 *   magnitude = distance to the closest point over all triangles (region walk of the closest-point-
 *               on-triangle problem, Ericson, "Real-Time Collision Detection" 5.1.5), the first
 *               triangle in index order winning exact ties of the squared distance;
 *   sign      = sign of (p - closest) . pseudonormal of the feature the closest point lies on
 *               (face normal / sum of the adjacent face normals for an edge / angle-weighted sum for
 *               a vertex: Baerentzen & Aanaes 2005); a point on the surface is +0.
 * Anchors available without a reference: a 12-triangle box must reproduce sdf_cuboid
 * (sdf_world.hpp:224-229) and a fine icosphere must approach sdf_sphere (:231-233); see
 * tests/test_mesh_stamp.py. */
typedef struct {
  long nt;
  double* tri; /* nt x {a, b, c} */
  double* nrm; /* nt x 7 pseudonormals: face, vertex a, b, c, edge ab, bc, ca */
} mesh_t;
static inline double dot3(vec3 a, vec3 b) { return sum3(a.v[0] * b.v[0], a.v[1] * b.v[1], a.v[2] * b.v[2]); }
static inline vec3 cross3(vec3 a, vec3 b) {
  return mk(a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2], a.v[0] * b.v[1] - a.v[1] * b.v[0]);
}
static inline vec3 axpy(vec3 a, double s, vec3 d) { return mk(a.v[0] + s * d.v[0], a.v[1] + s * d.v[1], a.v[2] + s * d.v[2]); }
static inline vec3 ld3(const double* p) { return mk(p[0], p[1], p[2]); }
/* closest point of triangle (a, b, c) to p; *feature: 0 face, 1..3 vertex a/b/c, 4 edge ab, 5 edge bc, 6 edge ca */
static vec3 closest_on_triangle(vec3 p, vec3 a, vec3 b, vec3 c, int* feature) {
  const vec3 ab = sub(b, a), ac = sub(c, a), ap = sub(p, a);
  const double d1 = dot3(ab, ap), d2 = dot3(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return *feature = 1, a;
  const vec3 bp = sub(p, b);
  const double d3 = dot3(ab, bp), d4 = dot3(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return *feature = 2, b;
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) return *feature = 4, axpy(a, d1 / (d1 - d3), ab);
  const vec3 cp = sub(p, c);
  const double d5 = dot3(ab, cp), d6 = dot3(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return *feature = 3, c;
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) return *feature = 6, axpy(a, d2 / (d2 - d6), ac);
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0)
    return *feature = 5, axpy(b, (d4 - d3) / ((d4 - d3) + (d5 - d6)), sub(c, b));
  const double denom = 1.0 / (va + (vb + vc));
  *feature = 0;
  return axpy(axpy(a, vb * denom, ab), vc * denom, ac);
}
static double mesh_sdf(const void* shape, vec3 p) {
  const mesh_t* m = (const mesh_t*)shape;
  double best = INFINITY;
  vec3 best_diff = mk(0.0, 0.0, 0.0);
  long best_tri = 0;
  int best_feature = 0;
  for (long i = 0; i < m->nt; ++i) {
    int feature;
    const double* T = m->tri + 9 * i;
    const vec3 diff = sub(p, closest_on_triangle(p, ld3(T), ld3(T + 3), ld3(T + 6), &feature));
    const double d2 = sqnorm(diff);
    if (d2 < best) best = d2, best_diff = diff, best_tri = i, best_feature = feature;
  }
  const double dist = sqrt(best);
  return dot3(best_diff, ld3(m->nrm + 21 * best_tri + 3 * best_feature)) < 0.0 ? -dist : dist;
}
typedef struct {
  int32_t lo, hi;
  long tri;
  int side; /* 0 ab, 1 bc, 2 ca */
} edge_ref;
static int edge_cmp(const void* pa, const void* pb) {
  const edge_ref *a = pa, *b = pb;
  if (a->lo != b->lo) return a->lo < b->lo ? -1 : 1;
  if (a->hi != b->hi) return a->hi < b->hi ? -1 : 1;
  return a->tri < b->tri ? -1 : (a->tri > b->tri ? 1 : 0);
}
static double corner_angle(vec3 e1, vec3 e2) {
  double c = dot3(unit(e1), unit(e2));
  c = c < -1.0 ? -1.0 : (1.0 < c ? 1.0 : c);
  return acos(c);
}
static void mesh_free(mesh_t* m) { free(m->tri), free(m->nrm); }
/* validation + the per-triangle tables; 0 or -1 with last_error set */
static int mesh_build(const double* vertices, int nv, const int32_t* triangles, int nt, mesh_t* out) {
  if (!vertices || !triangles || nv <= 0 || nt <= 0) return set_err("stamp: empty mesh"), -1;
  for (long i = 0; i < 3L * nv; ++i)
    if (!isfinite(vertices[i])) return set_err("stamp: non-finite mesh"), -1;
  for (long i = 0; i < 3L * nt; ++i)
    if (triangles[i] < 0 || triangles[i] >= nv) return set_err("stamp: mesh index out of range"), -1;
  mesh_t m = {nt, malloc(sizeof(double) * 9 * (size_t)nt), calloc(21 * (size_t)nt, sizeof(double))};
  double* vn = calloc(3 * (size_t)nv, sizeof(double));
  edge_ref* edges = malloc(sizeof(edge_ref) * 3 * (size_t)nt);
  int rc = 0;
  for (long i = 0; i < nt; ++i) {
    const int32_t* I = triangles + 3 * i;
    const vec3 a = ld3(vertices + 3 * I[0]), b = ld3(vertices + 3 * I[1]), c = ld3(vertices + 3 * I[2]);
    memcpy(m.tri + 9 * i, a.v, sizeof a.v), memcpy(m.tri + 9 * i + 3, b.v, sizeof b.v), memcpy(m.tri + 9 * i + 6, c.v, sizeof c.v);
    const vec3 n = cross3(sub(b, a), sub(c, a));
    if (!(sqnorm(n) > 0.0)) {
      rc = (set_err("stamp: degenerate mesh triangle"), -1);
      break;
    }
    const vec3 nf = unit(n);
    memcpy(m.nrm + 21 * i, nf.v, sizeof nf.v);
    const double w[3] = {corner_angle(sub(b, a), sub(c, a)), corner_angle(sub(a, b), sub(c, b)), corner_angle(sub(a, c), sub(b, c))};
    for (int k = 0; k < 3; ++k) {
      for (int ax = 0; ax < 3; ++ax) vn[3 * I[k] + ax] += w[k] * nf.v[ax]; /* triangle order */
      const int32_t p = I[k], q = I[(k + 1) % 3];
      edges[3 * i + k] = (edge_ref){p < q ? p : q, p < q ? q : p, i, k};
    }
  }
  if (rc == 0) {
    qsort(edges, 3 * (size_t)nt, sizeof(edge_ref), edge_cmp);
    for (long s = 0; s < 3L * nt;) { /* edge pseudonormal = sum of its faces' normals, in triangle order */
      long e = s;
      double sum[3] = {0.0, 0.0, 0.0};
      for (; e < 3L * nt && edges[e].lo == edges[s].lo && edges[e].hi == edges[s].hi; ++e)
        for (int ax = 0; ax < 3; ++ax) sum[ax] += m.nrm[21 * edges[e].tri + ax];
      for (long k = s; k < e; ++k) memcpy(m.nrm + 21 * edges[k].tri + 3 * (4 + edges[k].side), sum, sizeof sum);
      s = e;
    }
    for (long i = 0; i < nt; ++i)
      for (int k = 0; k < 3; ++k) memcpy(m.nrm + 21 * i + 3 * (1 + k), vn + 3 * triangles[3 * i + k], 3 * sizeof(double));
    *out = m;
  } else {
    mesh_free(&m);
  }
  free(edges), free(vn);
  return rc;
}
int ko_stamp_mesh(ko_tsdf* t, const double* vertices, int nv, const int32_t* triangles, int nt) {
  mesh_t m;
  if (mesh_build(vertices, nv, triangles, nt, &m) != 0) return -1;
  vec3 lo = mk(INFINITY, INFINITY, INFINITY), hi = mk(-INFINITY, -INFINITY, -INFINITY);
  for (long i = 0; i < nv; ++i) /* AABB of all vertices, grown by the band inside stamp_shape */
    for (int ax = 0; ax < 3; ++ax) {
      if (vertices[3 * i + ax] < lo.v[ax]) lo.v[ax] = vertices[3 * i + ax];
      if (vertices[3 * i + ax] > hi.v[ax]) hi.v[ax] = vertices[3 * i + ax];
    }
  const int rc = stamp_shape(t, mesh_sdf, &m, lo, hi);
  mesh_free(&m);
  return rc;
}
/* signed distance of the mesh at n points, without a world (tests of the definition itself) */
int ko_mesh_sdf(const double* vertices, int nv, const int32_t* triangles, int nt, const double* points, int64_t n, double* out) {
  mesh_t m;
  if (mesh_build(vertices, nv, triangles, nt, &m) != 0) return -1;
  for (int64_t i = 0; i < n; ++i) out[i] = mesh_sdf(&m, ld3(points + 3 * i));
  mesh_free(&m);
  return 0;
}

/* ---- decay + recycle (sdf_world.hpp:293-305, :449-475) -------------------- */
static int in_frustum(int width, int height, const double intr[4], const rigid_t* w2c, key3 k, double voxel) {
  const vec3 c = apply(w2c, block_center(k, voxel));
  const double radius = block_radius(voxel);
  const vec3 planes[5] = {mk(0.0, 0.0, 1.0), unit(mk(intr[0], 0.0, intr[2])),
                          unit(mk(-intr[0], 0.0, width - 1 - intr[2])), unit(mk(0.0, intr[1], intr[3])),
                          unit(mk(0.0, -intr[1], height - 1 - intr[3]))};
  for (int i = 0; i < 5; ++i)
    if (sum3(planes[i].v[0] * c.v[0], planes[i].v[1] * c.v[1], planes[i].v[2] * c.v[2]) < -radius) return 0;
  return 1;
}
void ko_decay_weights(ko_tsdf* t, int width, int height, const double intr[4], const double pose_R[9],
                      const double pose_t[3]) {
  const rigid_t cam = mk_pose(pose_R, pose_t);
  const rigid_t w2c = inverse(&cam);
  for (int i = 0; i < t->nslots; ++i) {
    if (t->slot_state[i] != SLOT_LIVE) continue;
    double factor = t->alpha_t;
    if (in_frustum(width, height, intr, &w2c, t->slot_key[i], t->voxel)) factor *= t->alpha_f;
    double* W = t->wt + (size_t)t->slot_pool[i] * VOX;
    for (int q = 0; q < VOX; ++q) W[q] *= factor; /* depth_sum is NOT scaled (:455) */
  }
}
int ko_recycle_blocks(ko_tsdf* t) {
  int recycled = 0;
  for (int i = 0; i < t->nslots; ++i) {
    if (t->slot_state[i] != SLOT_LIVE) continue;
    const double* W = t->wt + (size_t)t->slot_pool[i] * VOX;
    const double* G = t->geom + (size_t)t->slot_pool[i] * VOX;
    double total = 0.0;
    int has_geom = 0;
    for (int q = 0; q < VOX; ++q) total += W[q];
    for (int q = 0; q < VOX; ++q)
      if (isfinite(G[q])) has_geom = 1;
    if (total < t->wthr && !has_geom) {
      t->free_list[t->free_count++] = t->slot_pool[i];
      t->slot_state[i] = SLOT_TOMB;
      t->slot_pool[i] = -1;
      ++recycled;
    }
  }
  return recycled;
}

/* ---- inspection ------------------------------------------------------------ */
int ko_allocated_block_count(const ko_tsdf* t) {
  int n = 0;
  for (int i = 0; i < t->nslots; ++i) n += t->slot_state[i] == SLOT_LIVE;
  return n;
}
int ko_available(const ko_tsdf* t) { return table_available(t); }
int ko_next_fresh(const ko_tsdf* t) { return t->next_fresh; }
int ko_slot_count(const ko_tsdf* t) { return t->nslots; }
int ko_find(const ko_tsdf* t, int bx, int by, int bz) {
  const key3 k = {bx, by, bz};
  return table_find(t, k);
}
int ko_free_list(const ko_tsdf* t, int32_t* out, int max_out) {
  for (int i = 0; i < t->free_count && i < max_out; ++i) out[i] = t->free_list[i];
  return t->free_count;
}
int ko_export_blocks(const ko_tsdf* t, int32_t* keys, int32_t* pool, int max_blocks) {
  int n = 0;
  for (int i = 0; i < t->nslots; ++i) {
    if (t->slot_state[i] != SLOT_LIVE) continue;
    if (n < max_blocks) {
      keys[3 * n] = t->slot_key[i].x;
      keys[3 * n + 1] = t->slot_key[i].y;
      keys[3 * n + 2] = t->slot_key[i].z;
      pool[n] = t->slot_pool[i];
    }
    ++n;
  }
  return n;
}
void ko_block_channels(const ko_tsdf* t, int pool, double* depth_sum, double* depth_wt, double* geom_sdf) {
  memcpy(depth_sum, t->sum + (size_t)pool * VOX, VOX * sizeof(double));
  memcpy(depth_wt, t->wt + (size_t)pool * VOX, VOX * sizeof(double));
  memcpy(geom_sdf, t->geom + (size_t)pool * VOX, VOX * sizeof(double));
}

/* ---- point lookup (sdf_world.hpp:481-507) --------------------------------- */
static int lookup(const ko_tsdf* t, vec3 p, int geom_only, double* out) {
  int32_t vox[3];
  voxel_of(p, t->voxel, vox);
  const int pool = table_find(t, block_of(vox));
  if (pool < 0) return 0;
  const size_t at = (size_t)pool * VOX + (size_t)local_of(vox);
  int have = 0;
  double best = 0.0;
  if (!geom_only && t->wt[at] > 0.0) {
    best = t->sum[at] / t->wt[at];
    have = 1;
  }
  if (isfinite(t->geom[at])) {
    best = have ? (t->geom[at] < best ? t->geom[at] : best) : t->geom[at];
    have = 1;
  }
  *out = best;
  return have;
}
void ko_query_tsdf(const ko_tsdf* t, const double* points, int64_t n, int geom_only, double* out_sdf,
                   uint8_t* out_valid) {
  for (int64_t i = 0; i < n; ++i) {
    double value = 0.0;
    out_valid[i] = (uint8_t)lookup(t, mk(points[3 * i], points[3 * i + 1], points[3 * i + 2]), geom_only, &value);
    out_sdf[i] = out_valid[i] ? value : 0.0;
  }
}

/* ---- seeding (esdf.hpp:69-122) -------------------------------------------- */
static inline vec3 cell_center(const double origin[3], double ve, int x, int y, int z) { /* :51-53 */
  return mk(origin[0] + (x + 0.5) * ve, origin[1] + (y + 0.5) * ve, origin[2] + (z + 0.5) * ve);
}
void ko_seed_gather(const ko_tsdf* t, const double origin[3], const int dims[3], double ve, uint8_t* mask) {
  const double thr = 0.9 * t->voxel, h = 0.5 * ve;
  const double off[7][3] = {{0, 0, 0}, {h, 0, 0}, {-h, 0, 0}, {0, h, 0}, {0, -h, 0}, {0, 0, h}, {0, 0, -h}};
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  memset(mask, 0, (size_t)nx * ny * nz);
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const vec3 c = cell_center(origin, ve, x, y, z);
        for (int k = 0; k < 7; ++k) {
          double sdf;
          if (lookup(t, mk(c.v[0] + off[k][0], c.v[1] + off[k][1], c.v[2] + off[k][2]), 0, &sdf) &&
              fabs(sdf) < thr) {
            mask[(size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z)] = 1;
            break;
          }
        }
      }
}
void ko_seed_scatter(const ko_tsdf* t, const double origin[3], const int dims[3], double ve, uint8_t* mask) {
  const double thr = 0.9 * t->voxel;
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  memset(mask, 0, (size_t)nx * ny * nz);
  for (int i = 0; i < t->nslots; ++i) {
    if (t->slot_state[i] != SLOT_LIVE) continue;
    const size_t base = (size_t)t->slot_pool[i] * VOX;
    for (int q = 0; q < VOX; ++q) {
      int have = 0;
      double sdf = 0.0;
      if (t->wt[base + q] > 0.0) {
        sdf = t->sum[base + q] / t->wt[base + q];
        have = 1;
      }
      if (isfinite(t->geom[base + q])) {
        sdf = have ? (t->geom[base + q] < sdf ? t->geom[base + q] : sdf) : t->geom[base + q];
        have = 1;
      }
      if (!have || fabs(sdf) >= thr) continue;
      const vec3 c = voxel_center(t->slot_key[i], q, t->voxel);
      const int cx = (int)floor((c.v[0] - origin[0]) / ve);
      const int cy = (int)floor((c.v[1] - origin[1]) / ve);
      const int cz = (int)floor((c.v[2] - origin[2]) / ve);
      if (cx < 0 || cx >= nx || cy < 0 || cy >= ny || cz < 0 || cz >= nz) continue;
      mask[(size_t)cx + (size_t)nx * ((size_t)cy + (size_t)ny * cz)] = 1;
    }
  }
}

/* ---- exact EDT (esdf.hpp:129-282) ----------------------------------------- */
/* Lower envelope of f_i(t) = (t-u_i)^2 + r2_i; exact rational boundaries,
 * earlier apex kept on ties (esdf.hpp:129-186). */
typedef struct {
  int64_t u, r2, num, den;
  int tag;
} hull_entry;
typedef struct {
  hull_entry* e;
  int n;
} hull_t;

static void hull_push(hull_t* h, int64_t u, int64_t r2, int tag) {
  hull_entry in = {u, r2, 0, 0, tag};
  while (h->n > 0) {
    const hull_entry* top = &h->e[h->n - 1];
    const int64_t num = u * u + r2 - top->u * top->u - top->r2;
    const int64_t den = 2 * (u - top->u);
    if (den == 0) { /* same apex: keep the closer one, earlier on ties (:148-153) */
      if (r2 < top->r2) {
        --h->n;
        continue;
      }
      return;
    }
    if (top->den != 0 && num * top->den <= top->num * den) { /* :155-158 */
      --h->n;
      continue;
    }
    in.num = num;
    in.den = den;
    break;
  }
  if (h->n == 0) in.num = in.den = 0; /* -inf boundary */
  h->e[h->n++] = in;
}

int ko_propagate(const uint8_t* mask, int64_t mask_len, const int dims[3], double ve, int32_t* site,
                 double* distance) {
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  if (nx < 1 || ny < 1 || nz < 1) return set_err("esdf: dims must be >= 1"), -1;
  if (ve <= 0.0) return set_err("esdf: voxel_size must be > 0"), -1;
  const size_t cells = (size_t)nx * ny * nz;
  if ((size_t)mask_len != cells) return set_err("esdf: seed mask size does not match grid"), -1;
#define IDX(x, y, z) ((size_t)(x) + (size_t)nx * ((size_t)(y) + (size_t)ny * (size_t)(z)))
  int any = 0;
  for (size_t i = 0; i < cells; ++i) {
    site[3 * i] = site[3 * i + 1] = site[3 * i + 2] = -1;
    distance[i] = INFINITY;
    any |= mask[i] != 0;
  }
  if (!any) return 0;

  int32_t* near_z = malloc(cells * sizeof(int32_t));
  int32_t* sy = malloc(cells * sizeof(int32_t));
  int32_t* sz = malloc(cells * sizeof(int32_t));
  for (size_t i = 0; i < cells; ++i) near_z[i] = sy[i] = sz[i] = -1;
  int longest = nx > ny ? nx : ny;
  hull_t hull = {malloc((size_t)longest * sizeof(hull_entry)), 0};

  /* phase 1: bidirectional flood along z, strict '<' keeps the lower z (:213-233) */
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      int32_t last = -1;
      for (int z = 0; z < nz; ++z) {
        if (mask[IDX(x, y, z)]) last = z;
        near_z[IDX(x, y, z)] = last;
      }
      int32_t ahead = -1;
      for (int z = nz - 1; z >= 0; --z) {
        if (mask[IDX(x, y, z)]) ahead = z;
        if (ahead >= 0) {
          const int32_t behind = near_z[IDX(x, y, z)];
          if (behind < 0 || (ahead - z) < (z - behind)) near_z[IDX(x, y, z)] = ahead;
        }
      }
    }

  /* phase 2: envelope along y for every (x, z) (:236-255) */
  for (int z = 0; z < nz; ++z)
    for (int x = 0; x < nx; ++x) {
      hull.n = 0;
      for (int y = 0; y < ny; ++y) {
        const int32_t zs = near_z[IDX(x, y, z)];
        if (zs < 0) continue;
        const int64_t dz = (int64_t)z - zs;
        hull_push(&hull, y, dz * dz, y);
      }
      if (hull.n == 0) continue;
      int k = 0;
      for (int64_t y = 0; y < ny; ++y) { /* walk (:173-185) */
        while (k + 1 < hull.n && hull.e[k + 1].num < y * hull.e[k + 1].den) ++k;
        const int cy = hull.e[k].tag;
        sy[IDX(x, y, z)] = cy;
        sz[IDX(x, y, z)] = near_z[IDX(x, cy, z)];
      }
    }

  /* phase 3: envelope along x for every (y, z) (:258-280) */
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y) {
      hull.n = 0;
      for (int x = 0; x < nx; ++x) {
        const size_t i = IDX(x, y, z);
        if (sy[i] < 0) continue;
        const int64_t dy = (int64_t)y - sy[i], dz = (int64_t)z - sz[i];
        hull_push(&hull, x, dy * dy + dz * dz, x);
      }
      if (hull.n == 0) continue;
      int k = 0;
      for (int64_t x = 0; x < nx; ++x) {
        while (k + 1 < hull.n && hull.e[k + 1].num < x * hull.e[k + 1].den) ++k;
        const int cx = hull.e[k].tag;
        const size_t src = IDX(cx, y, z), dst = IDX(x, y, z);
        site[3 * dst] = cx;
        site[3 * dst + 1] = sy[src];
        site[3 * dst + 2] = sz[src];
        const int64_t dx = x - cx, dy = (int64_t)y - sy[src], dz = (int64_t)z - sz[src];
        distance[dst] = sqrt((double)(dx * dx + dy * dy + dz * dz)) * ve;
      }
    }
#undef IDX
  free(hull.e);
  free(near_z);
  free(sy);
  free(sz);
  return 1;
}

/* ---- sign recovery (esdf.hpp:288-320) ------------------------------------- */
void ko_recover_signs(const ko_tsdf* t, const double origin[3], const int dims[3], double ve, int has_sites,
                      const int32_t* site, double* distance) {
  if (!has_sites) return;
  const int nx = dims[0], ny = dims[1], nz = dims[2];
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const size_t i = (size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z);
        if (site[3 * i] < 0) continue;
        const vec3 q = cell_center(origin, ve, x, y, z);
        const vec3 s = cell_center(origin, ve, site[3 * i], site[3 * i + 1], site[3 * i + 2]);
        int negative = 0, resolved = 0;
        const vec3 delta = sub(q, s);
        if (sqnorm(delta) > 0.0) {
          const vec3 d = unit(delta);
          const vec3 probe = mk(s.v[0] + ve * d.v[0], s.v[1] + ve * d.v[1], s.v[2] + ve * d.v[2]);
          double g;
          if (lookup(t, probe, 1, &g)) {
            negative = g < 0.0;
            resolved = 1;
          }
        }
        if (!resolved) {
          double c;
          if (lookup(t, q, 0, &c)) negative = c < 0.0;
        }
        if (negative) distance[i] = -distance[i];
      }
}

/* ---- trilinear query (esdf.hpp:337-387) ----------------------------------- */
void ko_query_esdf(const double origin[3], const int dims[3], double ve, int has_sites, const double* distance,
                   const double* points, int64_t n, double* out_distance, double* out_gradient,
                   uint8_t* out_inside) {
  const int nx = dims[0], ny = dims[1];
  for (int64_t q = 0; q < n; ++q) {
    const double* p = points + 3 * q;
    int inside = 1;
    for (int a = 0; a < 3; ++a) inside &= p[a] >= origin[a];
    for (int a = 0; a < 3; ++a) inside &= p[a] <= origin[a] + dims[a] * ve;
    out_inside[q] = (uint8_t)inside;
    out_distance[q] = INFINITY;
    out_gradient[3 * q] = out_gradient[3 * q + 1] = out_gradient[3 * q + 2] = 0.0;
    if (!has_sites) continue;
    int i0[3], i1[3];
    double f[3];
    for (int a = 0; a < 3; ++a) {
      if (dims[a] == 1) {
        i0[a] = i1[a] = 0;
        f[a] = 0.0;
        continue;
      }
      const double s = (p[a] - origin[a]) / ve - 0.5;
      const double hi = (double)(dims[a] - 1);
      const double c = s < 0.0 ? 0.0 : (hi < s ? hi : s); /* std::clamp */
      i0[a] = (int)c < dims[a] - 2 ? (int)c : dims[a] - 2;
      i1[a] = i0[a] + 1;
      f[a] = c - i0[a];
    }
#define AT(cx, cy, cz) \
  distance[(size_t)((cx) ? i1[0] : i0[0]) + (size_t)nx * ((size_t)((cy) ? i1[1] : i0[1]) + (size_t)ny * (size_t)((cz) ? i1[2] : i0[2]))]
    const double c000 = AT(0, 0, 0), c100 = AT(1, 0, 0), c010 = AT(0, 1, 0), c110 = AT(1, 1, 0);
    const double c001 = AT(0, 0, 1), c101 = AT(1, 0, 1), c011 = AT(0, 1, 1), c111 = AT(1, 1, 1);
#undef AT
    const double fx = f[0], fy = f[1], fz = f[2];
    const double c00 = c000 * (1 - fx) + c100 * fx, c10 = c010 * (1 - fx) + c110 * fx;
    const double c01 = c001 * (1 - fx) + c101 * fx, c11 = c011 * (1 - fx) + c111 * fx;
    const double c0 = c00 * (1 - fy) + c10 * fy, c1 = c01 * (1 - fy) + c11 * fy;
    out_distance[q] = c0 * (1 - fz) + c1 * fz;
    const double inv = 1.0 / ve;
    out_gradient[3 * q] = ((c100 - c000) * (1 - fy) * (1 - fz) + (c110 - c010) * fy * (1 - fz) +
                           (c101 - c001) * (1 - fy) * fz + (c111 - c011) * fy * fz) *
                          inv;
    out_gradient[3 * q + 1] = ((c10 - c00) * (1 - fz) + (c11 - c01) * fz) * inv;
    out_gradient[3 * q + 2] = (c1 - c0) * inv;
  }
}

/* ---- scene collision (collision.hpp:30-44, :130-239) ------------------------- */
static double hinge_cost(double clearance, double margin) { /* :30-37 */
  if (clearance >= margin) return 0.0;
  if (clearance >= 0.0) {
    const double gap = margin - clearance;
    return gap * gap / (2.0 * margin);
  }
  return 0.5 * margin - clearance;
}
static double hinge_slope(double clearance, double margin) { /* :40-44 */
  if (clearance >= margin) return 0.0;
  if (clearance >= 0.0) return -(margin - clearance) / margin;
  return -1.0;
}
static void query_one(const double origin[3], const int dims[3], double ve, int has_sites, const double* distance,
                      vec3 p, double* d, vec3* g) {
  uint8_t inside;
  ko_query_esdf(origin, dims, ve, has_sites, distance, p.v, 1, d, g->v, &inside);
}
void ko_scene_collision_static(const double origin[3], const int dims[3], double ve, int has_sites,
                               const double* distance, const double* centers, const double* radii, int64_t n,
                               double margin, double* report3, double* gradient) {
  double max_pen = 0.0, total = 0.0;
  int worst = -1;
  for (int64_t s = 0; s < n; ++s) {
    double d;
    vec3 g;
    query_one(origin, dims, ve, has_sites, distance, mk(centers[3 * s], centers[3 * s + 1], centers[3 * s + 2]), &d, &g);
    const double clearance = d - radii[s];
    const double pen = -clearance;
    if (pen > max_pen) {
      max_pen = pen;
      worst = (int)s;
    }
    const double cost = hinge_cost(clearance, margin);
    total += cost;
    gradient[3 * s] = gradient[3 * s + 1] = gradient[3 * s + 2] = 0.0;
    if (cost > 0.0) {
      const double slope = hinge_slope(clearance, margin);
      for (int a = 0; a < 3; ++a) gradient[3 * s + a] += slope * g.v[a];
    }
  }
  report3[0] = max_pen;
  report3[1] = worst;
  report3[2] = total;
}
void ko_scene_collision_swept(const double origin[3], const int dims[3], double ve, int has_sites,
                              const double* distance, const double* centers, const double* radii,
                              const double* velocities, int timesteps, int spheres, double margin, double dt,
                              int max_checks, double* reports, double* center_gradient,
                              double* next_center_gradient, double* velocity_gradient) {
  const double min_step = ve;
  for (int t = 0; t < timesteps; ++t) {
    const int has_next = t + 1 < timesteps;
    double max_pen = 0.0, total = 0.0;
    int worst = -1;
    for (int s = 0; s < spheres; ++s) {
      const size_t at = ((size_t)t * spheres + s) * 3;
      const vec3 start = mk(centers[at], centers[at + 1], centers[at + 2]);
      vec3 segment = mk(0.0, 0.0, 0.0);
      if (has_next) {
        const size_t nx = at + (size_t)spheres * 3;
        segment = sub(mk(centers[nx], centers[nx + 1], centers[nx + 2]), start);
      }
      const double length = sqrt(sqnorm(segment));
      const vec3 vel = mk(velocities[at], velocities[at + 1], velocities[at + 2]);
      const double speed = sqrt(sqnorm(vel));
      const double weight = speed * dt;
      double hinge_sum = 0.0, lambda = 0.0;
      vec3 start_grad = mk(0.0, 0.0, 0.0), next_grad = mk(0.0, 0.0, 0.0);
      for (int check = 0; check < max_checks; ++check) {
        const double frac = length > 0.0 ? lambda / length : 0.0;
        const vec3 x = mk(start.v[0] + frac * segment.v[0], start.v[1] + frac * segment.v[1], start.v[2] + frac * segment.v[2]);
        double d;
        vec3 g;
        query_one(origin, dims, ve, has_sites, distance, x, &d, &g);
        const double clearance = d - radii[s];
        if (-clearance > max_pen) {
          max_pen = -clearance;
          worst = s;
        }
        hinge_sum += hinge_cost(clearance, margin);
        const double slope = hinge_slope(clearance, margin);
        if (slope != 0.0) {
          for (int a = 0; a < 3; ++a) {
            const double gx = slope * g.v[a];
            start_grad.v[a] += (1.0 - frac) * gx;
            next_grad.v[a] += frac * gx;
          }
        }
        if (!has_next) break;
        const double advance = clearance < min_step ? min_step : clearance; /* std::max(clearance, min_step) */
        lambda += advance;
        if (lambda >= length) break;
      }
      total += weight * hinge_sum;
      for (int a = 0; a < 3; ++a) {
        center_gradient[at + a] = 0.0 + weight * start_grad.v[a];
        if (has_next) next_center_gradient[at + a] = 0.0 + weight * next_grad.v[a];
        velocity_gradient[at + a] = 0.0;
        if (speed > 1e-12) velocity_gradient[at + a] += hinge_sum * dt * (vel.v[a] / speed);
      }
    }
    reports[3 * t] = max_pen;
    reports[3 * t + 1] = worst;
    reports[3 * t + 2] = total;
  }
}

/* ---- timed full update (bench.py CPU legs) -------------------------------- */
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
int64_t ko_timed_update(ko_tsdf* t, int n_frames, const float* depth, int width, int height, const double intr[4],
                        const double* poses_R, const double* poses_t, int n_cuboids, const double* cuboid_R,
                        const double* cuboid_t, const double* cuboid_he, int n_spheres, const double* sphere_c,
                        const double* sphere_r, const double origin[3], const int dims[3], double voxel_size,
                        double* times_out, double* checksum_out) {
  const size_t cells = (size_t)dims[0] * dims[1] * dims[2];
  double t0 = now_s();
  for (int f = 0; f < n_frames; ++f)
    if (ko_integrate_depth(t, depth + (size_t)f * width * height, width, height, intr, poses_R + 9 * f, poses_t + 3 * f) < 0)
      return -1;
  double t1 = now_s();
  for (int c = 0; c < n_cuboids; ++c)
    if (ko_stamp_cuboid(t, cuboid_R + 9 * c, cuboid_t + 3 * c, cuboid_he + 3 * c) != 0) return -1;
  for (int s = 0; s < n_spheres; ++s)
    if (ko_stamp_sphere(t, sphere_c + 3 * s, sphere_r[s]) != 0) return -1;
  double t2 = now_s();
  uint8_t* mask = malloc(cells);
  int32_t* site = malloc(cells * 3 * sizeof(int32_t));
  double* dist = malloc(cells * sizeof(double));
  ko_seed_gather(t, origin, dims, voxel_size, mask);
  double t3 = now_s();
  const int has = ko_propagate(mask, (int64_t)cells, dims, voxel_size, site, dist);
  double t4 = now_s();
  ko_recover_signs(t, origin, dims, voxel_size, has, site, dist);
  double t5 = now_s();
  int64_t seeds = 0;
  double sum = 0.0;
  for (size_t i = 0; i < cells; ++i) {
    seeds += mask[i] != 0;
    sum += fabs(dist[i]);
  }
  times_out[0] = t1 - t0, times_out[1] = t2 - t1, times_out[2] = t3 - t2, times_out[3] = t4 - t3, times_out[4] = t5 - t4;
  *checksum_out = sum;
  free(mask);
  free(site);
  free(dist);
  return has < 0 ? -1 : seeds;
}
