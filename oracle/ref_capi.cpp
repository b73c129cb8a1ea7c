// Flat C shim over the UNMODIFIED reference headers, compiled where they lie
// (/root/reference/proj/include/ks/{core,sdf_world,esdf}.hpp) into
// oracle/_ref/libks_ref.so by oracle/Makefile.  TEST INFRASTRUCTURE ONLY.
// No reference source is copied: this file only calls the reference's public
// functions and marshals plain arrays in and out.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "ks/collision.hpp"
#include "ks/esdf.hpp"
#include "ks/sdf_world.hpp"

#define KS_ORACLE_PREFIX kr_
#include "ks_oracle_api.h"

struct kr_tsdf {
  ks::SparseTsdf world;
};

namespace {

thread_local std::string g_error;

ks::Mat3 to_mat3(const double r[9]) {
  ks::Mat3 m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m(i, j) = r[3 * i + j];
  return m;
}

ks::Pose to_pose(const double r[9], const double t[3]) {
  ks::Pose pose;
  pose.rotation = to_mat3(r);
  pose.translation = ks::Vec3(t[0], t[1], t[2]);
  return pose;
}

ks::DepthFrame to_frame(const float* depth, int width, int height, const double intr[4],
                        const double pose_r[9], const double pose_t[3]) {
  ks::DepthFrame frame;
  frame.width = width;
  frame.height = height;
  frame.fx = intr[0];
  frame.fy = intr[1];
  frame.cx = intr[2];
  frame.cy = intr[3];
  frame.pose = to_pose(pose_r, pose_t);
  if (depth != nullptr && width > 0 && height > 0)
    frame.depth.assign(depth, depth + static_cast<std::size_t>(width) * height);
  return frame;
}

ks::EsdfConfig to_esdf_config(const double origin[3], const int dims[3], double voxel_size) {
  ks::EsdfConfig config;
  config.origin = ks::Vec3(origin[0], origin[1], origin[2]);
  config.nx = dims[0];
  config.ny = dims[1];
  config.nz = dims[2];
  config.voxel_size = voxel_size;
  return config;
}

}  // namespace

extern "C" {

const char* kr_last_error(void) { return g_error.c_str(); }

kr_tsdf* kr_tsdf_create(const double cfg[5], int capacity, int slot_count) {
  try {
    ks::TsdfConfig config;
    config.voxel_size = cfg[0];
    config.truncation = cfg[1];
    config.alpha_time = cfg[2];
    config.alpha_frustum = cfg[3];
    config.weight_threshold = cfg[4];
    config.capacity = capacity;
    config.slot_count = slot_count;
    auto* handle = new kr_tsdf;
    handle->world = ks::make_tsdf(config);
    return handle;
  } catch (const std::exception& e) {
    g_error = e.what();
    return nullptr;
  }
}

void kr_tsdf_destroy(kr_tsdf* t) { delete t; }

int kr_integrate_depth(kr_tsdf* t, const float* depth, int width, int height, const double intr[4],
                       const double pose_R[9], const double pose_t[3]) {
  try {
    return ks::integrate_depth(t->world, to_frame(depth, width, height, intr, pose_R, pose_t));
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

int kr_stamp_cuboid(kr_tsdf* t, const double pose_R[9], const double pose_t[3],
                    const double half_extents[3]) {
  try {
    ks::Cuboid cuboid;
    cuboid.pose = to_pose(pose_R, pose_t);
    cuboid.half_extents = ks::Vec3(half_extents[0], half_extents[1], half_extents[2]);
    ks::stamp_primitive(t->world, ks::Primitive(cuboid));
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

int kr_stamp_sphere(kr_tsdf* t, const double center[3], double radius) {
  try {
    ks::SphereShape sphere;
    sphere.center = ks::Vec3(center[0], center[1], center[2]);
    sphere.radius = radius;
    ks::stamp_primitive(t->world, ks::Primitive(sphere));
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

void kr_decay_weights(kr_tsdf* t, int width, int height, const double intr[4],
                      const double pose_R[9], const double pose_t[3]) {
  ks::decay_weights(t->world, to_frame(nullptr, width, height, intr, pose_R, pose_t));
}

int kr_recycle_blocks(kr_tsdf* t) { return ks::recycle_blocks(t->world); }

int kr_allocated_block_count(const kr_tsdf* t) { return ks::allocated_block_count(t->world); }
int kr_available(const kr_tsdf* t) { return t->world.table.available(); }
int kr_next_fresh(const kr_tsdf* t) { return t->world.table.next_fresh; }
int kr_slot_count(const kr_tsdf* t) { return static_cast<int>(t->world.table.slots.size()); }

int kr_find(const kr_tsdf* t, int bx, int by, int bz) {
  return t->world.table.find(ks::BlockKey{bx, by, bz});
}

int kr_free_list(const kr_tsdf* t, int32_t* out, int max_out) {
  const auto& list = t->world.table.free_list;
  const int n = static_cast<int>(list.size());
  for (int i = 0; i < n && i < max_out; ++i) out[i] = list[i];
  return n;
}

int kr_export_blocks(const kr_tsdf* t, int32_t* keys, int32_t* pool, int max_blocks) {
  int count = 0;
  for (const auto& slot : t->world.table.slots) {
    if (slot.state != ks::BlockHashTable::SlotState::kLive) continue;
    if (count < max_blocks) {
      keys[3 * count + 0] = slot.key.x;
      keys[3 * count + 1] = slot.key.y;
      keys[3 * count + 2] = slot.key.z;
      pool[count] = slot.pool;
    }
    ++count;
  }
  return count;
}

void kr_block_channels(const kr_tsdf* t, int pool, double* depth_sum, double* depth_wt,
                       double* geom_sdf) {
  const ks::VoxelBlock& block = t->world.pool[pool];
  std::memcpy(depth_sum, block.depth_sum.data(), sizeof(double) * ks::kBlockVoxels);
  std::memcpy(depth_wt, block.depth_wt.data(), sizeof(double) * ks::kBlockVoxels);
  std::memcpy(geom_sdf, block.geom_sdf.data(), sizeof(double) * ks::kBlockVoxels);
}

void kr_query_tsdf(const kr_tsdf* t, const double* points, int64_t n, int geom_only,
                   double* out_sdf, uint8_t* out_valid) {
  for (int64_t i = 0; i < n; ++i) {
    const ks::Vec3 p(points[3 * i], points[3 * i + 1], points[3 * i + 2]);
    const std::optional<double> value =
        geom_only ? ks::query_tsdf_geom(t->world, p) : ks::query_tsdf(t->world, p);
    out_valid[i] = value.has_value() ? 1 : 0;
    out_sdf[i] = value.value_or(0.0);
  }
}

void kr_seed_gather(const kr_tsdf* t, const double origin[3], const int dims[3], double voxel_size,
                    uint8_t* mask) {
  const ks::SeedMask seeds = ks::seed_gather(t->world, to_esdf_config(origin, dims, voxel_size));
  std::memcpy(mask, seeds.data(), seeds.size());
}

void kr_seed_scatter(const kr_tsdf* t, const double origin[3], const int dims[3],
                     double voxel_size, uint8_t* mask) {
  const ks::SeedMask seeds = ks::seed_scatter(t->world, to_esdf_config(origin, dims, voxel_size));
  std::memcpy(mask, seeds.data(), seeds.size());
}

int kr_propagate(const uint8_t* mask, int64_t mask_len, const int dims[3], double voxel_size,
                 int32_t* site, double* distance) {
  try {
    const double origin[3] = {0.0, 0.0, 0.0};
    const ks::SeedMask seeds(mask, mask + mask_len);
    const ks::DenseEsdf esdf = ks::propagate(seeds, to_esdf_config(origin, dims, voxel_size));
    for (std::size_t i = 0; i < esdf.site.size(); ++i) {
      site[3 * i + 0] = esdf.site[i][0];
      site[3 * i + 1] = esdf.site[i][1];
      site[3 * i + 2] = esdf.site[i][2];
    }
    std::memcpy(distance, esdf.distance.data(), sizeof(double) * esdf.distance.size());
    return esdf.has_sites ? 1 : 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

void kr_recover_signs(const kr_tsdf* t, const double origin[3], const int dims[3],
                      double voxel_size, int has_sites, const int32_t* site, double* distance) {
  ks::DenseEsdf esdf;
  esdf.config = to_esdf_config(origin, dims, voxel_size);
  const std::size_t cells = esdf.config.cell_count();
  esdf.has_sites = has_sites != 0;
  esdf.site.resize(cells);
  for (std::size_t i = 0; i < cells; ++i)
    esdf.site[i] = {site[3 * i + 0], site[3 * i + 1], site[3 * i + 2]};
  esdf.distance.assign(distance, distance + cells);
  const ks::DenseEsdf out = ks::recover_signs(std::move(esdf), t->world);
  std::memcpy(distance, out.distance.data(), sizeof(double) * cells);
}

void kr_query_esdf(const double origin[3], const int dims[3], double voxel_size, int has_sites,
                   const double* distance, const double* points, int64_t n, double* out_distance,
                   double* out_gradient, uint8_t* out_inside) {
  ks::DenseEsdf esdf;
  esdf.config = to_esdf_config(origin, dims, voxel_size);
  esdf.has_sites = has_sites != 0;
  esdf.distance.assign(distance, distance + esdf.config.cell_count());
  for (int64_t i = 0; i < n; ++i) {
    const ks::EsdfSample s =
        ks::query(esdf, ks::Vec3(points[3 * i], points[3 * i + 1], points[3 * i + 2]));
    out_distance[i] = s.distance;
    out_gradient[3 * i + 0] = s.gradient.x();
    out_gradient[3 * i + 1] = s.gradient.y();
    out_gradient[3 * i + 2] = s.gradient.z();
    out_inside[i] = s.inside ? 1 : 0;
  }
}

void kr_scene_collision_static(const double origin[3], const int dims[3], double voxel_size, int has_sites,
                               const double* distance, const double* centers, const double* radii, int64_t n,
                               double activation_margin, double* report3, double* gradient) {
  ks::DenseEsdf esdf;
  esdf.config = to_esdf_config(origin, dims, voxel_size);
  esdf.has_sites = has_sites != 0;
  esdf.distance.assign(distance, distance + esdf.config.cell_count());
  std::vector<ks::Vec3> c(n);
  for (int64_t i = 0; i < n; ++i) c[i] = ks::Vec3(centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]);
  const ks::CollisionReport rep =
      ks::scene_collision_static(esdf, std::span<const ks::Vec3>(c), std::span<const double>(radii, n), activation_margin);
  report3[0] = rep.max_penetration;
  report3[1] = rep.worst_first;
  report3[2] = rep.cost;
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) gradient[3 * i + a] = rep.gradient[i][a];
}

void kr_scene_collision_swept(const double origin[3], const int dims[3], double voxel_size, int has_sites,
                              const double* distance, const double* centers, const double* radii,
                              const double* velocities, int timesteps, int spheres, double activation_margin,
                              double dt, int max_checks, double* reports, double* center_gradient,
                              double* next_center_gradient, double* velocity_gradient) {
  ks::DenseEsdf esdf;
  esdf.config = to_esdf_config(origin, dims, voxel_size);
  esdf.has_sites = has_sites != 0;
  esdf.signs_recovered = true;
  esdf.distance.assign(distance, distance + esdf.config.cell_count());
  std::vector<std::vector<ks::Vec3>> c(timesteps), v(timesteps);
  for (int t = 0; t < timesteps; ++t)
    for (int s = 0; s < spheres; ++s) {
      const std::size_t at = (static_cast<std::size_t>(t) * spheres + s) * 3;
      c[t].emplace_back(centers[at], centers[at + 1], centers[at + 2]);
      v[t].emplace_back(velocities[at], velocities[at + 1], velocities[at + 2]);
    }
  ks::SceneCollisionConfig config;
  config.activation_margin = activation_margin;
  config.dt = dt;
  config.max_checks = max_checks;
  const auto reps = ks::scene_collision(esdf, c, std::span<const double>(radii, spheres), v, config);
  for (int t = 0; t < timesteps; ++t) {
    reports[3 * t] = reps[t].max_penetration;
    reports[3 * t + 1] = reps[t].worst_sphere;
    reports[3 * t + 2] = reps[t].cost;
    for (int s = 0; s < spheres; ++s) {
      const std::size_t at = (static_cast<std::size_t>(t) * spheres + s) * 3;
      for (int a = 0; a < 3; ++a) {
        center_gradient[at + a] = reps[t].center_gradient[s][a];
        velocity_gradient[at + a] = reps[t].velocity_gradient[s][a];
        if (t + 1 < timesteps) next_center_gradient[at + a] = reps[t].next_center_gradient[s][a];
      }
    }
  }
}

int64_t kr_timed_update(kr_tsdf* t, int n_frames, const float* depth, int width, int height,
                        const double intr[4], const double* poses_R, const double* poses_t, int n_cuboids,
                        const double* cuboid_R, const double* cuboid_t, const double* cuboid_he,
                        int n_spheres, const double* sphere_c, const double* sphere_r,
                        const double origin[3], const int dims[3], double voxel_size, double* times_out,
                        double* checksum_out) {
  using clock = std::chrono::steady_clock;
  auto secs = [](clock::time_point a, clock::time_point b) { return std::chrono::duration<double>(b - a).count(); };
  try {
    std::vector<ks::DepthFrame> frames;
    for (int f = 0; f < n_frames; ++f)
      frames.push_back(to_frame(depth + static_cast<std::size_t>(f) * width * height, width, height, intr,
                                poses_R + 9 * f, poses_t + 3 * f));
    std::vector<ks::Primitive> prims;
    for (int c = 0; c < n_cuboids; ++c) {
      ks::Cuboid cuboid;
      cuboid.pose = to_pose(cuboid_R + 9 * c, cuboid_t + 3 * c);
      cuboid.half_extents = ks::Vec3(cuboid_he[3 * c], cuboid_he[3 * c + 1], cuboid_he[3 * c + 2]);
      prims.emplace_back(cuboid);
    }
    for (int s = 0; s < n_spheres; ++s) {
      ks::SphereShape sphere;
      sphere.center = ks::Vec3(sphere_c[3 * s], sphere_c[3 * s + 1], sphere_c[3 * s + 2]);
      sphere.radius = sphere_r[s];
      prims.emplace_back(sphere);
    }
    const ks::EsdfConfig config = to_esdf_config(origin, dims, voxel_size);
    const auto t0 = clock::now();
    for (const auto& frame : frames) ks::integrate_depth(t->world, frame);
    const auto t1 = clock::now();
    for (const auto& prim : prims) ks::stamp_primitive(t->world, prim);
    const auto t2 = clock::now();
    const ks::SeedMask seeds = ks::seed_gather(t->world, config);
    const auto t3 = clock::now();
    ks::DenseEsdf esdf = ks::propagate(seeds, config);
    const auto t4 = clock::now();
    esdf = ks::recover_signs(std::move(esdf), t->world);
    const auto t5 = clock::now();
    times_out[0] = secs(t0, t1), times_out[1] = secs(t1, t2), times_out[2] = secs(t2, t3);
    times_out[3] = secs(t3, t4), times_out[4] = secs(t4, t5);
    int64_t count = 0;
    double sum = 0.0;
    for (std::size_t i = 0; i < seeds.size(); ++i) {
      count += seeds[i] != 0;
      sum += std::fabs(esdf.distance[i]);
    }
    *checksum_out = sum;
    return count;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

}  // extern "C"
