/* Flat C interface shared by the two CPU checkers.  TEST INFRASTRUCTURE ONLY:
 * nothing under paper_2603_05493_b200/ or include/ may include, link or load
 * anything from oracle/.
 *
 *   oracle/ks_oracle.c      ->  liboracle.so      prefix ko_   (C restatement)
 *   oracle/ref_capi.cpp     ->  _ref/libks_ref.so prefix kr_   (the reference's
 *                               own headers from /root/reference, unmodified)
 *
 * Include with KS_ORACLE_PREFIX defined to ko_ or kr_.  Both libraries export
 * exactly this set so one ctypes binding drives either.
 *
 * Conventions: rotations are row-major double[9]; intr = {fx, fy, cx, cy};
 * dims = {nx, ny, nz}; ESDF cell index = x + nx*(y + ny*z); block keys are
 * int32 triples; a block's 512 voxels are indexed lx + 8*(ly + 8*lz).
 */
#ifndef KS_ORACLE_API_H
#define KS_ORACLE_API_H

#include <stdint.h>

#ifndef KS_ORACLE_PREFIX
#error "define KS_ORACLE_PREFIX (ko_ or kr_) before including ks_oracle_api.h"
#endif
#define KS_OR_CAT2(a, b) a##b
#define KS_OR_CAT(a, b) KS_OR_CAT2(a, b)
#define KO(name) KS_OR_CAT(KS_ORACLE_PREFIX, name)

#ifdef __cplusplus
extern "C" {
#endif

typedef struct KO(tsdf) KO(tsdf);

/* message of the most recent failure on this thread ("" if none) */
const char* KO(last_error)(void);

/* cfg = {voxel_size, truncation, alpha_time, alpha_frustum, weight_threshold};
 * slot_count 0 -> 2*capacity.  NULL on validation failure. */
KO(tsdf)* KO(tsdf_create)(const double cfg[5], int capacity, int slot_count);
void KO(tsdf_destroy)(KO(tsdf)* t);

/* blocks touched (>= 0) or -1 with last_error set; all-or-nothing on exhaustion */
int KO(integrate_depth)(KO(tsdf)* t, const float* depth, int width, int height,
                        const double intr[4], const double pose_R[9], const double pose_t[3]);
int KO(stamp_cuboid)(KO(tsdf)* t, const double pose_R[9], const double pose_t[3],
                     const double half_extents[3]);
int KO(stamp_sphere)(KO(tsdf)* t, const double center[3], double radius);
/* Triangle-mesh stamping: liboracle.so (ko_) ONLY -- the reference has no mesh implementation
 * (SPEC.md:8, :422), so there is no kr_ counterpart and parity for it is unpinned (ks_oracle.c).
 * vertices = nv xyz triples (world frame), triangles = nt index triples, outward counter-clockwise. */
#ifndef KS_ORACLE_NO_MESH
int KO(stamp_mesh)(KO(tsdf)* t, const double* vertices, int nv, const int32_t* triangles, int nt);
int KO(mesh_sdf)(const double* vertices, int nv, const int32_t* triangles, int nt, const double* points,
                 int64_t n, double* out);
#endif
void KO(decay_weights)(KO(tsdf)* t, int width, int height, const double intr[4],
                       const double pose_R[9], const double pose_t[3]);
int KO(recycle_blocks)(KO(tsdf)* t);

int KO(allocated_block_count)(const KO(tsdf)* t);
int KO(available)(const KO(tsdf)* t);
int KO(next_fresh)(const KO(tsdf)* t);
int KO(slot_count)(const KO(tsdf)* t);
int KO(find)(const KO(tsdf)* t, int bx, int by, int bz);
/* free list, oldest first (back() is the next index handed out) */
int KO(free_list)(const KO(tsdf)* t, int32_t* out, int max_out);
/* live blocks in slot order: keys[3*i..], pool[i]; returns the live count */
int KO(export_blocks)(const KO(tsdf)* t, int32_t* keys, int32_t* pool, int max_blocks);
void KO(block_channels)(const KO(tsdf)* t, int pool, double* depth_sum, double* depth_wt,
                        double* geom_sdf);

/* points = n xyz triples; geom_only selects query_tsdf_geom */
void KO(query_tsdf)(const KO(tsdf)* t, const double* points, int64_t n, int geom_only,
                    double* out_sdf, uint8_t* out_valid);

void KO(seed_gather)(const KO(tsdf)* t, const double origin[3], const int dims[3],
                     double voxel_size, uint8_t* mask);
void KO(seed_scatter)(const KO(tsdf)* t, const double origin[3], const int dims[3],
                      double voxel_size, uint8_t* mask);
/* site = 3 int32 per cell, distance in meters (unsigned); returns has_sites, -1 on error */
int KO(propagate)(const uint8_t* mask, int64_t mask_len, const int dims[3], double voxel_size,
                  int32_t* site, double* distance);
void KO(recover_signs)(const KO(tsdf)* t, const double origin[3], const int dims[3],
                       double voxel_size, int has_sites, const int32_t* site, double* distance);
void KO(query_esdf)(const double origin[3], const int dims[3], double voxel_size, int has_sites,
                    const double* distance, const double* points, int64_t n, double* out_distance,
                    double* out_gradient, uint8_t* out_inside);

/* scene_collision_static (collision.hpp:130-152): one query per sphere.
 * report3 = {max_penetration, worst sphere index (-1 if none), cost}; gradient = n xyz triples. */
void KO(scene_collision_static)(const double origin[3], const int dims[3], double voxel_size, int has_sites,
                                const double* distance, const double* centers, const double* radii,
                                int64_t n, double activation_margin, double* report3, double* gradient);
/* scene_collision (collision.hpp:177-239): swept spheres over `timesteps` x `spheres` centres.
 * reports = timesteps x {max_penetration, worst sphere, cost}; the three gradients are
 * timesteps x spheres xyz triples (next_gradient of the last timestep is left untouched). */
void KO(scene_collision_swept)(const double origin[3], const int dims[3], double voxel_size, int has_sites,
                               const double* distance, const double* centers, const double* radii,
                               const double* velocities, int timesteps, int spheres,
                               double activation_margin, double dt, int max_checks, double* reports,
                               double* center_gradient, double* next_center_gradient,
                               double* velocity_gradient);

/* One full update run and timed INSIDE the library (no marshalling in the timed regions):
 * integrate n_frames depth frames, stamp the primitives, then seed_gather -> propagate ->
 * recover_signs over the given grid.  times_out = seconds of {integrate, stamp, seed, propagate,
 * signs}; *checksum_out = sum of |distance| over the grid.  Returns the seed count, -1 on error.
 * Used by bench.py's cpu_baseline and --impl reference legs. */
int64_t KO(timed_update)(KO(tsdf)* t, int n_frames, const float* depth, int width, int height,
                         const double intr[4], const double* poses_R, const double* poses_t,
                         int n_cuboids, const double* cuboid_R, const double* cuboid_t,
                         const double* cuboid_he, int n_spheres, const double* sphere_c,
                         const double* sphere_r, const double origin[3], const int dims[3],
                         double voxel_size, double* times_out, double* checksum_out);

#ifdef __cplusplus
}
#endif

#endif /* KS_ORACLE_API_H */
