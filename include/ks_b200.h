/* ks_b200 -- C ABI of the B200-native perception hot path (sm_100a).
 *
 * Drop-in boundary for the reference's header-only C++ API
 *   /root/reference/proj/include/ks/sdf_world.hpp   (block-sparse TSDF)
 *   /root/reference/proj/include/ks/esdf.hpp        (dense ESDF + query)
 * Each entry point cites the reference function it replaces.  The reference has
 * no FFI of its own (it is `inline` C++); include/ks_b200/ks.hpp re-exports the
 * reference's ks:: names on top of this ABI and INTEGRATION.md shows the binding.
 *
 * Rules of the boundary
 *   - plain pointers and sizes only; handles are opaque; no exceptions cross it.
 *   - every call returns a ks_status; ks_last_error() holds the reference's
 *     exception text for that status (thread-local).
 *   - "_async" calls enqueue on the handle's stream and never synchronise, so a
 *     whole update can be captured in one CUDA graph (ks_graph_*).  Their outcome
 *     (blocks touched, pool exhaustion, ...) is collected by ks_tsdf_sync().
 *   - there is no CPU fallback: without a CUDA device every compute call fails
 *     with KS_ERR_CUDA.
 *
 * Conventions: rotations are row-major double[9], camera pose is camera-to-world;
 * ESDF cell index = x + nx*(y + ny*z); a block's 512 voxels are lx + 8*(ly + 8*lz).
 */
#ifndef KS_B200_H
#define KS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define KS_API
#else
#define KS_API __attribute__((visibility("default")))
#endif

typedef enum ks_status {
  KS_OK = 0,
  KS_ERR_INVALID = 1,        /* ks::ValidationError (bad config / frame / shape)          */
  KS_ERR_POOL_EXHAUSTED = 2, /* ks::ValidationError "tsdf: pool exhausted, frame requires ..." */
  KS_ERR_TABLE_FULL = 3,     /* ks::ValidationError "tsdf: hash table full"               */
  KS_ERR_CUDA = 4,           /* CUDA runtime failure or no device                         */
  KS_ERR_RANGE = 5,          /* block coordinate outside +-2^20 (packed-key limit)        */
  KS_ERR_UNSUPPORTED = 6     /* grid larger than this build's tile limits                 */
} ks_status;

typedef struct ks_tsdf ks_tsdf;   /* ks::SparseTsdf  (sdf_world.hpp:206-210) */
typedef struct ks_esdf ks_esdf;   /* ks::DenseEsdf   (esdf.hpp:58-64)        */
typedef struct ks_graph ks_graph; /* an instantiated CUDA graph               */
typedef void* ks_stream;          /* cudaStream_t                             */

/* ks::TsdfConfig (sdf_world.hpp:38-54) */
typedef struct ks_tsdf_config {
  double voxel_size, truncation, alpha_time, alpha_frustum, weight_threshold;
  int32_t capacity;   /* block pool size   */
  int32_t slot_count; /* 0 -> 2 * capacity */
} ks_tsdf_config;

/* ks::DepthFrame minus the pixels (sdf_world.hpp:191-204) */
typedef struct ks_camera {
  int32_t width, height;
  double fx, fy, cx, cy;
  double pose_R[9], pose_t[3];
} ks_camera;

/* ks::EsdfConfig (esdf.hpp:35-54); seeding: 0 = scatter, 1 = gather */
typedef struct ks_esdf_config {
  double origin[3];
  int32_t nx, ny, nz;
  double voxel_size;
  int32_t seeding;
} ks_esdf_config;

/* outcome of the TSDF operations enqueued since the previous ks_tsdf_sync() */
typedef struct ks_tsdf_report {
  int32_t status;          /* first ks_status hit, KS_OK otherwise                        */
  int32_t blocks_touched;  /* return value of the last integrate_depth (sdf_world.hpp:388) */
  int32_t required;        /* on KS_ERR_POOL_EXHAUSTED: new blocks the op needed           */
  int32_t available;       /*                            free + fresh pool entries it had   */
  int32_t live_blocks;     /* allocated_block_count (sdf_world.hpp:509)                    */
  int32_t next_fresh;      /* BlockHashTable::next_fresh (sdf_world.hpp:112)               */
  int32_t free_count;      /* BlockHashTable::free_list.size()                             */
  int32_t recycled;        /* return value of the last recycle_blocks (sdf_world.hpp:474)  */
} ks_tsdf_report;

typedef struct ks_esdf_report {
  int32_t status;
  int32_t has_sites;       /* DenseEsdf::has_sites (esdf.hpp:62)       */
  int32_t signs_recovered; /* DenseEsdf::signs_recovered (esdf.hpp:63) */
  int64_t seed_count;      /* cells marked by the last seeding pass     */
} ks_esdf_report;

/* ---- library ------------------------------------------------------------- */
KS_API const char* ks_last_error(void);
KS_API const char* ks_version(void);
KS_API int ks_device_count(void);
/* kernels launched by this library since load (bench.py's gpu_launches) */
KS_API int64_t ks_kernel_launch_count(void);

/* ---- streams / graphs ------------------------------------------------------ */
KS_API int ks_stream_create(ks_stream* out);
KS_API int ks_stream_destroy(ks_stream s);
KS_API int ks_stream_sync(ks_stream s);
KS_API int ks_graph_begin_capture(ks_stream s);
KS_API int ks_graph_end_capture(ks_stream s, ks_graph** out);
KS_API int ks_graph_launch(ks_graph* g, ks_stream s);
KS_API int ks_graph_node_count(ks_graph* g, int64_t* kernel_nodes, int64_t* all_nodes);
KS_API void ks_graph_destroy(ks_graph* g);

/* ---- TSDF ------------------------------------------------------------------ */
/* make_tsdf_config (sdf_world.hpp:56-61) */
KS_API int ks_tsdf_config_init(double voxel_size, ks_tsdf_config* out);
/* make_tsdf (sdf_world.hpp:327-334); validate() texts preserved */
KS_API int ks_tsdf_create(const ks_tsdf_config* config, ks_tsdf** out);
KS_API void ks_tsdf_destroy(ks_tsdf* t);
KS_API int ks_tsdf_set_stream(ks_tsdf* t, ks_stream s);
KS_API ks_stream ks_tsdf_get_stream(const ks_tsdf* t);

/* integrate_depth (sdf_world.hpp:340-389), blocking, host pixels.
 * DepthFrame::validate texts preserved; *blocks_touched = return value. */
KS_API int ks_tsdf_integrate_depth(ks_tsdf* t, const ks_camera* cam, const float* depth_host,
                                   int32_t* blocks_touched);
/* the same in three capturable steps: copy a frame into the handle's pinned
 * staging area (CPU only), enqueue its upload, enqueue the four phases */
KS_API int ks_tsdf_stage_frame(ks_tsdf* t, const ks_camera* cam, const float* depth_host);
KS_API int ks_tsdf_upload_frame_async(ks_tsdf* t);
KS_API int ks_tsdf_integrate_async(ks_tsdf* t);
/* the same with one staging slot per camera (0 .. KS_MAX_FRAME_SLOTS-1), so that a multi-camera
 * update (repeated integrate_depth) is a single replayable graph; slot 0 is the one used above */
#define KS_MAX_FRAME_SLOTS 8
KS_API int ks_tsdf_stage_frame_slot(ks_tsdf* t, int32_t slot, const ks_camera* cam, const float* depth_host);
/* Zero-copy staging.  ks_tsdf_frame_buffer returns the pinned staging area of a slot (width*height floats,
 * owned by the handle, stable until a larger frame is requested; once a graph was captured on the world's stream a
 * larger frame gets NEW buffers and the old ones stay alive until ks_tsdf_destroy, so a graph captured earlier keeps
 * reading the memory it was captured with -- re-capture after growing): a producer that writes its pixels there and
 * passes the same pointer to ks_tsdf_stage_frame_slot skips the staging copy.  ks_tsdf_integrate_depth does
 * the same for ANY page-locked depth_host (e.g. from ks_host_alloc): it is uploaded in place. */
KS_API int ks_tsdf_frame_buffer(ks_tsdf* t, int32_t slot, int32_t width, int32_t height, float** out);
KS_API int ks_host_alloc(size_t bytes, void** out);  /* page-locked host memory (cudaMallocHost) */
KS_API void ks_host_free(void* p);
KS_API int ks_tsdf_upload_frame_slot_async(ks_tsdf* t, int32_t slot);
KS_API int ks_tsdf_integrate_slot_async(ks_tsdf* t, int32_t slot);

/* stamp_primitive (sdf_world.hpp:394-444) */
KS_API int ks_tsdf_stamp_cuboid(ks_tsdf* t, const double pose_R[9], const double pose_t[3],
                                const double half_extents[3]);
KS_API int ks_tsdf_stamp_sphere(ks_tsdf* t, const double center[3], double radius);
KS_API int ks_tsdf_stamp_cuboid_async(ks_tsdf* t, const double pose_R[9], const double pose_t[3],
                                      const double half_extents[3]);
KS_API int ks_tsdf_stamp_sphere_async(ks_tsdf* t, const double center[3], double radius);

/* All primitives of an update in one call: stamp_primitive applied to prims[0 .. n-1] in order, stopping at the first
 * one that would throw (its error is the one reported; later primitives are not applied) -- the world ends up exactly
 * as after the sequential calls: pool indices, hash slots, free list, voxels.  Three kernel launches for the whole
 * batch instead of three per primitive.  kind: 0 = Cuboid (pose_R, pose_t, half_extents), 1 = SphereShape (center, radius). */
typedef struct ks_primitive {
  int32_t kind, reserved;
  double pose_R[9], pose_t[3], half_extents[3];
  double center[3], radius;
} ks_primitive;
KS_API int ks_tsdf_stamp_batch(ks_tsdf* t, const ks_primitive* prims, int32_t n);
KS_API int ks_tsdf_stamp_batch_async(ks_tsdf* t, const ks_primitive* prims, int32_t n);

/* Triangle-mesh stamping.  The reference has no implementation to replace (SPEC.md:8 and :422 put it out of
 * scope; "Cuboids and meshes are stamped directly into the geometry channel"); the flow is
 * stamp_primitive's (sdf_world.hpp:418-443: padded AABB -> candidate blocks with |sdf(centre)| <= truncation +
 * block radius -> allocate -> per-voxel min) with the signed distance to a closed, outward-oriented
 * (counter-clockwise) indexed triangle mesh: closest point over all triangles, sign from the angle-weighted
 * pseudonormal of the closest feature (csrc/mesh.cuh).  vertices = n_vertices xyz triples in the world frame,
 * triangles = n_triangles index triples.  ks_mesh_create validates ("stamp: empty mesh", "stamp: non-finite
 * mesh", "stamp: mesh index out of range", "stamp: degenerate mesh triangle" -> KS_ERR_INVALID), builds the
 * per-triangle tables and uploads them once; stamping a created mesh is capturable.  ks_mesh_destroy waits for the
 * device (a stamp may still read the tables): call it outside stream capture and after the last replay of any
 * graph that stamps the mesh. */
typedef struct ks_mesh ks_mesh;
KS_API int ks_mesh_create(const double* vertices, int32_t n_vertices, const int32_t* triangles,
                          int32_t n_triangles, ks_mesh** out);
KS_API void ks_mesh_destroy(ks_mesh* m);
KS_API int32_t ks_mesh_triangle_count(const ks_mesh* m);
KS_API int ks_tsdf_stamp_mesh(ks_tsdf* t, const ks_mesh* m);
KS_API int ks_tsdf_stamp_mesh_async(ks_tsdf* t, const ks_mesh* m);

/* decay_weights (sdf_world.hpp:449-457), recycle_blocks (sdf_world.hpp:462-475) */
KS_API int ks_tsdf_decay_weights(ks_tsdf* t, const ks_camera* cam);
KS_API int ks_tsdf_decay_weights_async(ks_tsdf* t, const ks_camera* cam);
KS_API int ks_tsdf_recycle_blocks(ks_tsdf* t, int32_t* recycled);

/* wait for the handle's stream and collect the outcome of everything enqueued;
 * returns report->status and sets ks_last_error() like the blocking calls */
KS_API int ks_tsdf_sync(ks_tsdf* t, ks_tsdf_report* report);

/* query_tsdf / query_tsdf_geom (sdf_world.hpp:500-507): n xyz triples in host
 * memory -> value + has_value flag (std::optional) */
KS_API int ks_tsdf_query(ks_tsdf* t, const double* points_host, int64_t n, int32_t geom_only,
                         double* out_sdf, uint8_t* out_valid);
/* allocated_block_count (sdf_world.hpp:509) */
KS_API int ks_tsdf_allocated_block_count(ks_tsdf* t, int32_t* count);
/* BlockHashTable::find (sdf_world.hpp:132-142) */
KS_API int ks_tsdf_find(ks_tsdf* t, const int32_t key[3], int32_t* pool_index);
/* parity dump of SparseTsdf::table / ::pool: live blocks in slot order */
KS_API int ks_tsdf_export_blocks(ks_tsdf* t, int32_t* keys_xyz, int32_t* pool_index, int32_t max_blocks,
                                 int32_t* count);
/* VoxelBlock channels of the given pool entries: n x 512 doubles each */
KS_API int ks_tsdf_download_blocks(ks_tsdf* t, const int32_t* pool_index, int32_t n, double* depth_sum,
                                   double* depth_wt, double* geom_sdf);
/* SparseTsdf::table.slots in slot order (sdf_world.hpp:103-110): key, pool index (-1 unless live) and state
 * (0 empty, 1 live, 2 tombstone) of the first max_slots slots; *count = slot count.  Host mirrors (ks.hpp). */
KS_API int ks_tsdf_export_slots(ks_tsdf* t, int32_t* keys_xyz, int32_t* pool_index, uint8_t* state, int32_t max_slots,
                                int32_t* count);
/* counts the mutating calls enqueued on the world so far (integrate, stamp, decay, recycle): a host copy of
 * table / pool taken at generation g is stale once this returns something else.  No synchronisation. */
KS_API uint64_t ks_tsdf_generation(const ks_tsdf* t);
/* BlockHashTable::free_list, oldest first */
KS_API int ks_tsdf_free_list(ks_tsdf* t, int32_t* out, int32_t max_out, int32_t* count);
/* measurement hook: when enabled, non-captured ops record CUDA events between their stages;
 * out = device ms of {block discovery, allocation, voxel integration} of the last integrate and
 * {candidates+allocation, voxel stamping} of the last stamp */
KS_API int ks_tsdf_profile(ks_tsdf* t, int32_t enable);
KS_API int ks_tsdf_stage_ms(ks_tsdf* t, float out[5]);

/* ---- ESDF ------------------------------------------------------------------ */
/* EsdfConfig::validate (esdf.hpp:41-44) + device buffers for the grid */
KS_API int ks_esdf_create(const ks_esdf_config* config, ks_esdf** out);
KS_API void ks_esdf_destroy(ks_esdf* e);
KS_API int ks_esdf_set_stream(ks_esdf* e, ks_stream s);

/* build_esdf (esdf.hpp:323-327): seed -> propagate -> recover_signs */
KS_API int ks_esdf_build(ks_esdf* e, const ks_tsdf* t);
KS_API int ks_esdf_build_async(ks_esdf* e, const ks_tsdf* t);
/* seed_gather / seed_scatter (esdf.hpp:102-122 / :73-98); mask_host may be NULL */
KS_API int ks_esdf_seed(ks_esdf* e, const ks_tsdf* t, int32_t mode, uint8_t* mask_host);
/* propagate (esdf.hpp:193-282) from a host mask (NULL: the mask left by ks_esdf_seed) */
KS_API int ks_esdf_propagate(ks_esdf* e, const uint8_t* mask_host, int64_t mask_len);
/* recover_signs (esdf.hpp:288-320) on the field left by ks_esdf_propagate */
KS_API int ks_esdf_recover_signs(ks_esdf* e, const ks_tsdf* t);
KS_API int ks_esdf_sync(ks_esdf* e, ks_esdf_report* report);
/* what the last ks_esdf_sync / blocking call saw (DenseEsdf::has_sites, ::signs_recovered as plain members); no wait */
KS_API int ks_esdf_last_report(const ks_esdf* e, ks_esdf_report* report);
/* measurement hook: device ms of {directory, seeding, z flood, y sweep, x sweep, sign recovery}
 * of the last non-captured ks_esdf_build_async */
KS_API int ks_esdf_profile(ks_esdf* e, int32_t enable);
KS_API int ks_esdf_stage_ms(ks_esdf* e, float out[6]);

/* counts the calls enqueued so far that rewrite the field (build, propagate, recover_signs); see ks_tsdf_generation */
KS_API uint64_t ks_esdf_generation(const ks_esdf* e);
/* DenseEsdf::site / ::distance (any pointer may be NULL).  d2 = squared integer
 * site offset (exact), INT32_MAX when the grid has no sites. */
KS_API int ks_esdf_download(ks_esdf* e, int32_t* site_xyz, double* distance, int32_t* d2);

/* query (esdf.hpp:337-387) for n points: host buffers, blocking */
KS_API int ks_esdf_query(ks_esdf* e, const double* points_host, int64_t n, double* distance,
                         double* gradient_xyz, uint8_t* inside);
/* the same with device-resident buffers, enqueued on the handle's stream */
KS_API int ks_esdf_query_device_async(ks_esdf* e, const double* points_dev, int64_t n, double* distance_dev,
                                      double* gradient_dev, uint8_t* inside_dev);
/* one launch, capturable: {tag, min distance over the n probe points, probes closer than near_distance, seed count}
 * as four doubles at summary_dev -- the fixed-size per-environment summary that multi-GPU runs all-gather */
KS_API int ks_esdf_probe_summary_device_async(ks_esdf* e, const double* points_dev, int64_t n, double near_distance,
                                              double tag, double* summary_dev);

/* ---- scene collision (SURVEY 8f "next": the consumer of query) ---------------- */
/* CollisionReport / SceneTimestepReport scalars (collision.hpp:46-52, :161-168) */
typedef struct ks_collision_report {
  double max_penetration; /* <= 0 means free                         */
  double cost;
  int32_t worst_sphere;   /* -1 when nothing penetrates              */
  int32_t reserved;
} ks_collision_report;
/* scene_collision_static (collision.hpp:130-152): one query per sphere, hinge cost and its
 * gradient w.r.t. the centres (n xyz triples, may be NULL).  Host buffers, blocking. */
KS_API int ks_esdf_scene_collision_static(ks_esdf* e, const double* centers_host, const double* radii_host,
                                          int64_t n, double activation_margin, ks_collision_report* report,
                                          double* gradient_xyz_host);
/* scene_collision (collision.hpp:177-239): swept spheres over `timesteps` x `spheres` centres
 * with CHOMP speed weighting; reports[timesteps]; the gradients are timesteps x spheres xyz
 * triples (next_center_gradient of the last timestep is zero).  Fails with the reference's
 * "scene_collision: esdf signs not recovered" on an unsigned field. */
KS_API int ks_esdf_scene_collision_swept(ks_esdf* e, const double* centers_host, const double* radii_host,
                                         const double* velocities_host, int32_t timesteps, int32_t spheres,
                                         double activation_margin, double dt, int32_t max_checks,
                                         ks_collision_report* reports, double* center_gradient,
                                         double* next_center_gradient, double* velocity_gradient);

/* ---- batched environments (BASELINE configs[4]) ------------------------- */
/* The reference has no batch API ("no batched-environment API"; PAPER.md's batched planning runs one
 * SparseTsdf + DenseEsdf per environment through the functions above).  A ks_batch owns n_envs such pairs with one
 * configuration and runs an update of all of them -- per environment: upload the staged frames, integrate_depth per
 * camera (sdf_world.hpp:340-389), stamp_primitive for its primitives / meshes (sdf_world.hpp:394-444), build_esdf
 * (esdf.hpp:323-327), one 32-byte summary {environment id, min distance over its probe points, probes closer than
 * near_distance, seed count} -- as one enqueue on ks_batch_stream(), capturable, or as the batch's own graph
 * (ks_batch_update).  Environments are independent: no data-path collective.  The environments are dealt round-robin
 * onto `lanes` (1..8) streams forked from / joined into the batch stream, so one environment's short kernels overlap
 * another's sweeps.  Each world is exactly what the per-handle calls produce; ks_batch_tsdf / ks_batch_esdf hand out
 * the handles (owned by the batch) for staging frames (ks_tsdf_stage_frame_slot, ks_tsdf_frame_buffer), queries,
 * collision checks and downloads. */
typedef struct ks_batch ks_batch;
KS_API int ks_batch_create(int32_t n_envs, const ks_tsdf_config* tsdf_config, const ks_esdf_config* esdf_config,
                           int32_t lanes, ks_batch** out);
KS_API void ks_batch_destroy(ks_batch* b);
KS_API int32_t ks_batch_size(const ks_batch* b);
KS_API int32_t ks_batch_lanes(const ks_batch* b);
KS_API ks_tsdf* ks_batch_tsdf(ks_batch* b, int32_t env);
KS_API ks_esdf* ks_batch_esdf(ks_batch* b, int32_t env);
KS_API ks_stream ks_batch_stream(ks_batch* b);
/* what an update applies to environment `env`: the first n_cameras staging slots, these primitives (copied), these
 * meshes (borrowed: keep them alive) */
KS_API int ks_batch_set_inputs(ks_batch* b, int32_t env, int32_t n_cameras, const ks_primitive* prims, int32_t n_prims,
                               const ks_mesh* const* meshes, int32_t n_meshes);
/* probe points of the environment's summary (n xyz triples, copied to the device); n = 0: no summary row */
KS_API int ks_batch_set_probes(ks_batch* b, int32_t env, const double* points_host, int64_t n, double near_distance);
/* global id of environment 0 (multi-rank: the rank's first environment), written into the summaries */
KS_API int ks_batch_set_first_env(ks_batch* b, int32_t first_env);
/* enqueue one update of every environment (+ the all-gather when a communicator is attached); never synchronises */
KS_API int ks_batch_update_async(ks_batch* b, int32_t upload_frames);
/* the same through a private CUDA graph: captured at the first call and after inputs changed, replayed otherwise */
KS_API int ks_batch_update(ks_batch* b, int32_t upload_frames);
KS_API int64_t ks_batch_graph_kernels(const ks_batch* b);
/* wait; per-environment reports (any pointer may be NULL): reports[n_envs], esdf_reports[n_envs],
 * summaries_host[n_envs][4].  Returns the first failing environment's status, its text prefixed "environment <id>: " */
KS_API int ks_batch_sync(ks_batch* b, ks_tsdf_report* reports, ks_esdf_report* esdf_reports, double* summaries_host);
KS_API double* ks_batch_summary_device(ks_batch* b);   /* [max_local][4] doubles, rows >= n_envs stay NaN */
/* Multi-GPU: one process per GPU, each with its own batch over a contiguous range of environments. */
KS_API int ks_partition_envs(int32_t n_envs, int32_t world, int32_t rank, int32_t* lo, int32_t* hi);
/* NCCL is resolved at run time (dlopen of libnccl.so.2, or KS_NCCL_LIB): the library does not link it.
 * ks_nccl_unique_id: 128 bytes from ncclGetUniqueId, to be broadcast by the host's own means;
 * ks_batch_attach_nccl: ncclCommInitRank (collective over all ranks) + gather buffers; from then on every update ends
 * with ncclAllGather(summary rows) on the batch stream -- a node of the captured graph.  A host that already owns a
 * communicator passes it to ks_batch_attach_nccl_comm instead (borrowed).  max_local_envs = the largest batch size of
 * any rank (every rank contributes that many rows; missing ones are NaN). */
KS_API int ks_nccl_unique_id(void* out128);
KS_API int ks_batch_attach_nccl(ks_batch* b, const void* unique_id128, int32_t world, int32_t rank, int32_t max_local_envs);
KS_API int ks_batch_attach_nccl_comm(ks_batch* b, void* nccl_comm, int32_t world, int32_t rank, int32_t max_local_envs);
KS_API double* ks_batch_gathered_device(ks_batch* b);  /* [world][max_local][4]; == the summary buffer on one rank */
KS_API int32_t ks_batch_gathered_rows(const ks_batch* b);
KS_API int ks_batch_gathered(ks_batch* b, double* host_out);  /* wait + download of the gathered rows */

#ifdef __cplusplus
}
#endif
#endif /* KS_B200_H */
