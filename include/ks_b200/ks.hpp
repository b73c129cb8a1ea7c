// ks_b200/ks.hpp -- the reference's ks:: perception API, backed by libks_b200.so (B200, sm_100a).
//
// Include this instead of "ks/sdf_world.hpp" and "ks/esdf.hpp"
// (/root/reference/proj/include/ks/sdf_world.hpp, esdf.hpp) and link -lks_b200: the function
// names, argument types, return values and exception types/texts are the reference's; the data
// lives in HBM behind opaque handles (include/ks_b200.h).
//
// Mixing with the reference's own headers (collision.hpp, ik.hpp, ... -- the planner side, which stays the
// reference's).  This header CLAIMS the include guards of the two headers it replaces (KS_SDF_WORLD_HPP,
// KS_ESDF_HPP), so a later `#include "ks/esdf.hpp"` -- e.g. the one in collision.hpp:22 -- is a no-op, and it
// takes Vec3 / Pose / ValidationError from the reference's core.hpp whenever that file is on the include path.
// Two ways to use it, both covered by tests/cpp/mixed_program.cpp:
//   * no source change: put include/ks_b200/overlay FIRST on the include path.  It holds forwarding headers
//     ks/sdf_world.hpp, ks/esdf.hpp and a ks/collision.hpp that pulls the reference's own collision.hpp
//     (#include_next) with its two scene functions renamed, so that scene_collision_static / scene_collision
//     resolve to the batched GPU versions below while self_collision, CollisionReport, hinge_cost, ... stay the
//     reference's.  ik.hpp:117-120 / :217-226 then run against the device field unchanged.
//   * or include "ks_b200/ks.hpp" before any reference header; with the planner headers on the include path it
//     pulls ks/collision.hpp itself in the same way.
// Differences a caller can observe:
//   * SparseTsdf / DenseEsdf hold a shared handle, so copying one aliases the same device world
//     (the reference deep-copies its std::vectors); recover_signs(esdf, tsdf) works in place and
//     returns the same handle.
//   * DenseEsdf::site / ::distance and SparseTsdf::table / ::pool are READ-ONLY host mirrors: they behave like
//     the reference's const std::vector members (size, [], iteration, data) and are downloaded on first access
//     after the device copy changed (ks_esdf_generation / ks_tsdf_generation); code that WRITES them does not
//     compile.  A tombstoned slot mirrors as key (0,0,0) (the device table does not keep erased keys).
//   * query_batch() is new: callers that looped over query() should hand the whole batch over.
//   * scene_collision_static / scene_collision (collision.hpp:130-239) are one batched kernel each; the cost is
//     a fixed-shape tree sum on the GPU (1e-12 relative to the reference's left-to-right sum), everything else
//     is identical.
//   * save/load_depth_frame and save/load_esdf read and write the reference's KSDEPTH1 / KSESDF1 files;
//     the JSON header is emitted with sorted keys like the reference's nlohmann dump, numbers in shortest
//     round-trip form (values, not bytes, are what both sides agree on).
#ifndef KS_B200_KS_HPP
#define KS_B200_KS_HPP

#if defined(KS_SDF_WORLD_HPP) || defined(KS_ESDF_HPP)
#error "ks_b200/ks.hpp replaces ks/sdf_world.hpp and ks/esdf.hpp: include it first, or put include/ks_b200/overlay first on the include path"
#endif
#define KS_SDF_WORLD_HPP  // claimed: the reference's sdf_world.hpp / esdf.hpp become no-ops after this header
#define KS_ESDF_HPP

#include <Eigen/Dense>

#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <mutex>
#include <span>
#include <sstream>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "../ks_b200.h"

// Reference core types whenever the reference tree is reachable (always the case when mixing with its planner headers).
#if !defined(KS_B200_USE_REFERENCE_CORE) && defined(__has_include)
#if __has_include("ks/core.hpp")
#define KS_B200_USE_REFERENCE_CORE 1
#endif
#endif
// Planner side present: collision.hpp's non-scene parts (self_collision, CollisionReport, ...) come from the reference.
#if !defined(KS_B200_REFERENCE_COLLISION) && defined(KS_B200_USE_REFERENCE_CORE) && defined(__has_include)
#if __has_include("ks/robot_model.hpp") && __has_include("ks/collision.hpp")
#define KS_B200_REFERENCE_COLLISION 1
#endif
#endif

#if defined(KS_B200_USE_REFERENCE_CORE)
#include "ks/core.hpp"
#else
namespace ks {
using Vec3 = Eigen::Vector3d;
using Mat3 = Eigen::Matrix3d;
inline constexpr double kInf = std::numeric_limits<double>::infinity();

class ValidationError : public std::runtime_error {  // core.hpp:36-39
 public:
  explicit ValidationError(const std::string& what) : std::runtime_error(what) {}
};
class ParseError : public std::runtime_error {  // core.hpp:42-45
 public:
  explicit ParseError(const std::string& what) : std::runtime_error(what) {}
};

struct Pose {  // core.hpp:54-77
  Mat3 rotation = Mat3::Identity();
  Vec3 translation = Vec3::Zero();
  static Pose Identity() { return Pose{}; }
  Vec3 operator*(const Vec3& p) const { return rotation * p + translation; }
  Pose operator*(const Pose& o) const { return Pose{rotation * o.rotation, rotation * o.translation + translation}; }
  Pose inverse() const {
    Pose out;
    out.rotation = rotation.transpose();
    out.translation = -(out.rotation * translation);
    return out;
  }
};
}  // namespace ks
#endif

namespace ks {

namespace b200_detail {
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& what) : std::runtime_error(what) {}
};
inline void check(int status) {
  if (status == KS_OK) return;
  const std::string text = ks_last_error();
  if (status == KS_ERR_CUDA) throw CudaError(text);
  throw ValidationError(text);
}
inline void fill_pose(const Pose& pose, double r[9], double t[3]) {
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) r[3 * i + j] = pose.rotation(i, j);
    t[i] = pose.translation[i];
  }
}

/// Read-only host mirror of a device array: looks like a const std::vector<T> (the reference's public members,
/// sdf_world.hpp:206-210, esdf.hpp:58-64).  The copy is fetched on the first access after the device side changed
/// (generation counter of the handle); copies of the owning struct share it, like they share the handle.
template <class T>
class HostMirror {
 public:
  using value_type = T;
  using const_iterator = typename std::vector<T>::const_iterator;
  HostMirror() = default;
  HostMirror(std::function<std::uint64_t()> generation, std::function<void(std::vector<T>&)> fetch)
      : state_(std::make_shared<State>()) {
    state_->generation = std::move(generation), state_->fetch = std::move(fetch);
  }
  const std::vector<T>& get() const {
    static const std::vector<T> none;
    if (!state_) return none;
    std::lock_guard<std::mutex> lock(state_->mu);
    const std::uint64_t now = state_->generation();
    if (!state_->valid || now != state_->seen) {
      state_->fetch(state_->data);
      state_->seen = now, state_->valid = true;
    }
    return state_->data;
  }
  std::size_t size() const { return get().size(); }
  bool empty() const { return get().empty(); }
  const T& operator[](std::size_t i) const { return get()[i]; }
  const T& at(std::size_t i) const { return get().at(i); }
  const T& front() const { return get().front(); }
  const T& back() const { return get().back(); }
  const T* data() const { return get().data(); }
  const_iterator begin() const { return get().begin(); }
  const_iterator end() const { return get().end(); }
  operator const std::vector<T>&() const { return get(); }
  const std::vector<T>& operator()() const { return get(); }  // round-1 spelling: esdf.distance()

 private:
  struct State {
    std::mutex mu;
    std::vector<T> data;
    std::uint64_t seen = 0;
    bool valid = false;
    std::function<std::uint64_t()> generation;
    std::function<void(std::vector<T>&)> fetch;
  };
  std::shared_ptr<State> state_;
};
}  // namespace b200_detail

// ---- sdf_world.hpp -----------------------------------------------------------------------------
inline constexpr int kBlockEdge = 8;
inline constexpr int kBlockVoxels = kBlockEdge * kBlockEdge * kBlockEdge;

struct TsdfConfig {  // sdf_world.hpp:38-54
  double voxel_size = 0.01;
  double truncation = 0.04;
  double alpha_time = 0.99;
  double alpha_frustum = 0.5;
  double weight_threshold = 0.5;
  int capacity = 8192;
  int slot_count = 0;
  void validate() const {
    if (voxel_size <= 0.0) throw ValidationError("tsdf: voxel_size must be > 0");
    if (truncation < voxel_size) throw ValidationError("tsdf: truncation must be >= voxel_size");
    if (!(alpha_time > 0.0 && alpha_time <= 1.0) || !(alpha_frustum > 0.0 && alpha_frustum <= 1.0))
      throw ValidationError("tsdf: decay factors must lie in (0, 1]");
    if (capacity < 1) throw ValidationError("tsdf: capacity must be >= 1");
  }
};

inline TsdfConfig make_tsdf_config(double voxel_size) {  // sdf_world.hpp:56-61
  TsdfConfig c;
  c.voxel_size = voxel_size;
  c.truncation = 4.0 * voxel_size;
  return c;
}

struct BlockKey {  // sdf_world.hpp:87-90
  std::int32_t x = 0, y = 0, z = 0;
  bool operator==(const BlockKey&) const = default;
};

struct DepthFrame {  // sdf_world.hpp:191-204
  int width = 0, height = 0;
  double fx = 0.0, fy = 0.0, cx = 0.0, cy = 0.0;
  Pose pose;
  std::vector<float> depth;
  void validate() const {
    if (width <= 0 || height <= 0 || fx <= 0.0 || fy <= 0.0) throw ValidationError("depth frame: invalid intrinsics");
    if (static_cast<int>(depth.size()) != width * height) throw ValidationError("depth frame: depth buffer size mismatch");
  }
  bool depth_valid(float d) const { return std::isfinite(d) && d > 0.0f; }  // sdf_world.hpp:203
  ks_camera camera() const {
    ks_camera cam{};
    cam.width = width, cam.height = height;
    cam.fx = fx, cam.fy = fy, cam.cx = cx, cam.cy = cy;
    b200_detail::fill_pose(pose, cam.pose_R, cam.pose_t);
    return cam;
  }
};

struct VoxelBlock {  // sdf_world.hpp:65-85 (host copy of one pool entry)
  std::array<double, kBlockVoxels> depth_sum;
  std::array<double, kBlockVoxels> depth_wt;
  std::array<double, kBlockVoxels> geom_sdf;
  double weight_total() const {
    double sum = 0.0;
    for (double w : depth_wt) sum += w;
    return sum;
  }
  bool has_geometry() const {
    for (double g : geom_sdf)
      if (std::isfinite(g)) return true;
    return false;
  }
};

/// Read-only mirror of BlockHashTable (sdf_world.hpp:102-189): slots in slot order, free list, counters, find().
struct BlockHashTableMirror {
  enum class SlotState : std::uint8_t { kEmpty, kLive, kTombstone };
  struct Slot {
    BlockKey key;
    std::int32_t pool = -1;
    SlotState state = SlotState::kEmpty;
  };
  struct Counter {  // next_fresh as a live value
    std::function<std::int32_t()> read;
    operator std::int32_t() const { return read ? read() : 0; }
  };
  b200_detail::HostMirror<Slot> slots;
  b200_detail::HostMirror<std::int32_t> free_list;
  Counter next_fresh;
  std::int32_t capacity = 0;
  std::function<int(const BlockKey&)> lookup;
  int live_count() const {
    int count = 0;
    for (const Slot& slot : slots.get()) count += slot.state == SlotState::kLive;
    return count;
  }
  int available() const { return static_cast<int>(free_list.size()) + (capacity - next_fresh); }
  int find(const BlockKey& key) const { return lookup ? lookup(key) : -1; }  // BlockHashTable::find, on the device table
};

/// Read-only mirror of SparseTsdf::pool: size() == capacity, pool[i] downloads entry i (cached per generation).
class PoolMirror {
 public:
  PoolMirror() = default;
  PoolMirror(std::shared_ptr<ks_tsdf> handle, std::size_t capacity) : state_(std::make_shared<State>()) {
    state_->handle = std::move(handle), state_->capacity = capacity;
  }
  std::size_t size() const { return state_ ? state_->capacity : 0; }
  const VoxelBlock& operator[](std::size_t i) const {
    if (!state_ || i >= state_->capacity) throw ValidationError("tsdf: pool index out of range");
    std::lock_guard<std::mutex> lock(state_->mu);
    const std::uint64_t now = ks_tsdf_generation(state_->handle.get());
    if (now != state_->seen) state_->blocks.clear(), state_->seen = now;
    auto it = state_->blocks.find(i);
    if (it == state_->blocks.end()) {
      auto block = std::make_unique<VoxelBlock>();
      const std::int32_t index = static_cast<std::int32_t>(i);
      b200_detail::check(ks_tsdf_download_blocks(state_->handle.get(), &index, 1, block->depth_sum.data(), block->depth_wt.data(),
                                                 block->geom_sdf.data()));
      it = state_->blocks.emplace(i, std::move(block)).first;
    }
    return *it->second;
  }
  const VoxelBlock& at(std::size_t i) const { return (*this)[i]; }

 private:
  struct State {
    std::mutex mu;
    std::shared_ptr<ks_tsdf> handle;
    std::size_t capacity = 0;
    std::uint64_t seen = ~0ull;
    std::map<std::size_t, std::unique_ptr<VoxelBlock>> blocks;
  };
  std::shared_ptr<State> state_;
};

struct SparseTsdf {  // sdf_world.hpp:206-210; the table and the pool live in HBM, the members below mirror them
  TsdfConfig config;
  std::shared_ptr<ks_tsdf> handle;
  BlockHashTableMirror table;
  PoolMirror pool;
  ks_tsdf* get() const { return handle.get(); }
};

struct Cuboid {  // sdf_world.hpp:212-215
  Pose pose;
  Vec3 half_extents = Vec3::Zero();
};
struct SphereShape {  // sdf_world.hpp:217-220
  Vec3 center = Vec3::Zero();
  double radius = 0.0;
};
using Primitive = std::variant<Cuboid, SphereShape>;

namespace b200_detail {
inline ks_tsdf_config to_c(const TsdfConfig& config) {
  return ks_tsdf_config{config.voxel_size, config.truncation, config.alpha_time, config.alpha_frustum,
                        config.weight_threshold, config.capacity, config.slot_count};
}
inline SparseTsdf wrap_tsdf(std::shared_ptr<ks_tsdf> handle, const TsdfConfig& config);
}  // namespace b200_detail

inline SparseTsdf make_tsdf(const TsdfConfig& config) {  // sdf_world.hpp:327-334
  config.validate();
  const ks_tsdf_config c = b200_detail::to_c(config);
  ks_tsdf* raw = nullptr;
  b200_detail::check(ks_tsdf_create(&c, &raw));
  return b200_detail::wrap_tsdf(std::shared_ptr<ks_tsdf>(raw, ks_tsdf_destroy), config);
}

// the ks::SparseTsdf view (config + host mirrors) of a device world, whoever owns it
inline SparseTsdf b200_detail::wrap_tsdf(std::shared_ptr<ks_tsdf> handle, const TsdfConfig& config) {
  SparseTsdf tsdf;
  tsdf.config = config;
  tsdf.handle = std::move(handle);
  const std::shared_ptr<ks_tsdf> h = tsdf.handle;
  using Slot = BlockHashTableMirror::Slot;
  tsdf.table.slots = b200_detail::HostMirror<Slot>([h] { return ks_tsdf_generation(h.get()); }, [h](std::vector<Slot>& out) {
    std::int32_t n = 0;
    b200_detail::check(ks_tsdf_export_slots(h.get(), nullptr, nullptr, nullptr, 0, &n));
    std::vector<std::int32_t> keys(3 * static_cast<std::size_t>(n)), pools(n);
    std::vector<std::uint8_t> state(n);
    b200_detail::check(ks_tsdf_export_slots(h.get(), keys.data(), pools.data(), state.data(), n, &n));
    out.resize(n);
    for (std::int32_t i = 0; i < n; ++i) {
      out[i].key = BlockKey{keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]};
      out[i].pool = pools[i];
      out[i].state = static_cast<BlockHashTableMirror::SlotState>(state[i]);
    }
  });
  tsdf.table.free_list = b200_detail::HostMirror<std::int32_t>([h] { return ks_tsdf_generation(h.get()); }, [h, config](std::vector<std::int32_t>& out) {
    out.resize(static_cast<std::size_t>(config.capacity));
    std::int32_t n = 0;
    b200_detail::check(ks_tsdf_free_list(h.get(), out.data(), config.capacity, &n));
    out.resize(static_cast<std::size_t>(n));
  });
  tsdf.table.next_fresh.read = [h] {
    ks_tsdf_report rep{};
    b200_detail::check(ks_tsdf_sync(h.get(), &rep));
    return rep.next_fresh;
  };
  tsdf.table.capacity = config.capacity;
  tsdf.table.lookup = [h](const BlockKey& key) {
    const std::int32_t k[3] = {key.x, key.y, key.z};
    std::int32_t pool = -1;
    b200_detail::check(ks_tsdf_find(h.get(), k, &pool));
    return static_cast<int>(pool);
  };
  tsdf.pool = PoolMirror(h, static_cast<std::size_t>(config.capacity));
  return tsdf;
}

inline int integrate_depth(SparseTsdf& tsdf, const DepthFrame& frame) {  // sdf_world.hpp:340-389
  frame.validate();
  const ks_camera cam = frame.camera();
  std::int32_t touched = 0;
  b200_detail::check(ks_tsdf_integrate_depth(tsdf.get(), &cam, frame.depth.data(), &touched));
  return touched;
}

inline void stamp_primitive(SparseTsdf& tsdf, const Primitive& primitive) {  // sdf_world.hpp:394-444
  if (const auto* cuboid = std::get_if<Cuboid>(&primitive)) {
    double r[9], t[3];
    b200_detail::fill_pose(cuboid->pose, r, t);
    const double he[3] = {cuboid->half_extents[0], cuboid->half_extents[1], cuboid->half_extents[2]};
    b200_detail::check(ks_tsdf_stamp_cuboid(tsdf.get(), r, t, he));
  } else {
    const auto& sphere = std::get<SphereShape>(primitive);
    const double c[3] = {sphere.center[0], sphere.center[1], sphere.center[2]};
    b200_detail::check(ks_tsdf_stamp_sphere(tsdf.get(), c, sphere.radius));
  }
}

/// All primitives of an update as ONE batch (addition; three kernel launches instead of three per primitive): the
/// same as `for (p : primitives) stamp_primitive(tsdf, p);` -- pool indices, hash slots and voxels included -- and
/// it stops at, and throws for, the first primitive the reference would throw for.
inline void stamp_primitives(SparseTsdf& tsdf, std::span<const Primitive> primitives) {
  std::vector<ks_primitive> batch(primitives.size());
  for (std::size_t i = 0; i < primitives.size(); ++i) {
    ks_primitive& out = batch[i];
    out = ks_primitive{};
    if (const auto* cuboid = std::get_if<Cuboid>(&primitives[i])) {
      out.kind = 0;
      b200_detail::fill_pose(cuboid->pose, out.pose_R, out.pose_t);
      for (int a = 0; a < 3; ++a) out.half_extents[a] = cuboid->half_extents[a];
    } else {
      const auto& sphere = std::get<SphereShape>(primitives[i]);
      out.kind = 1;
      for (int a = 0; a < 3; ++a) out.center[a] = sphere.center[a];
      out.radius = sphere.radius;
    }
  }
  b200_detail::check(ks_tsdf_stamp_batch(tsdf.get(), batch.data(), static_cast<std::int32_t>(batch.size())));
}

// Triangle meshes.  NOT in the reference (SPEC.md:8, :422 put mesh stamping out of scope; PAPER.md:293 names it):
// an addition next to Primitive, which keeps its reference definition.  A closed mesh with outward,
// counter-clockwise triangles in the world frame; the tables live on the device, so a static mesh is built once.
struct TriangleMesh {
  std::vector<Vec3> vertices;
  std::vector<std::array<std::int32_t, 3>> triangles;
};
struct DeviceMesh {
  std::shared_ptr<ks_mesh> handle;
  int triangle_count() const { return ks_mesh_triangle_count(handle.get()); }
};
inline DeviceMesh upload_mesh(const TriangleMesh& mesh) {  // throws ValidationError("stamp: ... mesh ...")
  std::vector<double> v(3 * mesh.vertices.size());
  for (std::size_t i = 0; i < mesh.vertices.size(); ++i)
    for (int a = 0; a < 3; ++a) v[3 * i + a] = mesh.vertices[i][a];
  ks_mesh* raw = nullptr;
  b200_detail::check(ks_mesh_create(v.data(), static_cast<std::int32_t>(mesh.vertices.size()),
                                    mesh.triangles.empty() ? nullptr : mesh.triangles.front().data(),
                                    static_cast<std::int32_t>(mesh.triangles.size()), &raw));
  return DeviceMesh{std::shared_ptr<ks_mesh>(raw, ks_mesh_destroy)};
}
// flow of stamp_primitive (sdf_world.hpp:418-443) with the signed mesh distance of csrc/mesh.cuh
inline void stamp_mesh(SparseTsdf& tsdf, const DeviceMesh& mesh) { b200_detail::check(ks_tsdf_stamp_mesh(tsdf.get(), mesh.handle.get())); }
inline void stamp_mesh(SparseTsdf& tsdf, const TriangleMesh& mesh) { stamp_mesh(tsdf, upload_mesh(mesh)); }

inline void decay_weights(SparseTsdf& tsdf, const DepthFrame& camera) {  // sdf_world.hpp:449-457
  const ks_camera cam = camera.camera();
  b200_detail::check(ks_tsdf_decay_weights(tsdf.get(), &cam));
}

inline int recycle_blocks(SparseTsdf& tsdf) {  // sdf_world.hpp:462-475
  std::int32_t n = 0;
  b200_detail::check(ks_tsdf_recycle_blocks(tsdf.get(), &n));
  return n;
}

namespace b200_detail {
inline std::optional<double> lookup(const SparseTsdf& tsdf, const Vec3& point, int geom_only) {
  const double p[3] = {point[0], point[1], point[2]};
  double value = 0.0;
  std::uint8_t valid = 0;
  check(ks_tsdf_query(tsdf.get(), p, 1, geom_only, &value, &valid));
  if (!valid) return std::nullopt;
  return value;
}
}  // namespace b200_detail

inline std::optional<double> query_tsdf(const SparseTsdf& tsdf, const Vec3& point) {  // sdf_world.hpp:500-502
  return b200_detail::lookup(tsdf, point, 0);
}
inline std::optional<double> query_tsdf_geom(const SparseTsdf& tsdf, const Vec3& point) {  // sdf_world.hpp:505-507
  return b200_detail::lookup(tsdf, point, 1);
}
inline int allocated_block_count(const SparseTsdf& tsdf) {  // sdf_world.hpp:509
  std::int32_t n = 0;
  b200_detail::check(ks_tsdf_allocated_block_count(tsdf.get(), &n));
  return n;
}

// ---- esdf.hpp ----------------------------------------------------------------------------------
enum class SeedingMode { kScatter, kGather };  // esdf.hpp:33

struct EsdfConfig {  // esdf.hpp:35-54
  Vec3 origin = Vec3::Zero();
  int nx = 1, ny = 1, nz = 1;
  double voxel_size = 0.01;
  SeedingMode seeding = SeedingMode::kGather;
  void validate() const {
    if (nx < 1 || ny < 1 || nz < 1) throw ValidationError("esdf: dims must be >= 1");
    if (voxel_size <= 0.0) throw ValidationError("esdf: voxel_size must be > 0");
  }
  std::size_t cell_count() const { return static_cast<std::size_t>(nx) * ny * nz; }
  std::size_t index(int x, int y, int z) const {
    return static_cast<std::size_t>(x) + static_cast<std::size_t>(nx) * (y + static_cast<std::size_t>(ny) * z);
  }
  Vec3 cell_center(int x, int y, int z) const {
    return origin + Vec3((x + 0.5) * voxel_size, (y + 0.5) * voxel_size, (z + 0.5) * voxel_size);
  }
};

struct DenseEsdf {  // esdf.hpp:58-64; the field lives in HBM, site / distance are read-only host mirrors of it
  EsdfConfig config;
  b200_detail::HostMirror<std::array<std::int32_t, 3>> site;  // (-1,-1,-1) when no sites exist
  b200_detail::HostMirror<double> distance;                   // meters; +inf sentinel without sites
  bool has_sites = false;
  bool signs_recovered = false;
  std::shared_ptr<ks_esdf> handle;
  ks_esdf* get() const { return handle.get(); }

  void refresh_flags() {
    ks_esdf_report rep{};
    b200_detail::check(ks_esdf_sync(get(), &rep));
    has_sites = rep.has_sites != 0;
    signs_recovered = rep.signs_recovered != 0;
  }
};

using SeedMask = std::vector<std::uint8_t>;  // esdf.hpp:66

inline double seed_threshold(const SparseTsdf& tsdf) { return 0.9 * tsdf.config.voxel_size; }  // esdf.hpp:69

namespace b200_detail {
inline ks_esdf_config to_c(const EsdfConfig& config) {
  ks_esdf_config c{};
  for (int a = 0; a < 3; ++a) c.origin[a] = config.origin[a];
  c.nx = config.nx, c.ny = config.ny, c.nz = config.nz;
  c.voxel_size = config.voxel_size;
  c.seeding = config.seeding == SeedingMode::kGather ? 1 : 0;
  return c;
}
inline DenseEsdf wrap_esdf(std::shared_ptr<ks_esdf> handle, const EsdfConfig& config);
}  // namespace b200_detail

inline DenseEsdf make_esdf(const EsdfConfig& config) {
  config.validate();
  const ks_esdf_config c = b200_detail::to_c(config);
  ks_esdf* raw = nullptr;
  b200_detail::check(ks_esdf_create(&c, &raw));
  return b200_detail::wrap_esdf(std::shared_ptr<ks_esdf>(raw, ks_esdf_destroy), config);
}

inline DenseEsdf b200_detail::wrap_esdf(std::shared_ptr<ks_esdf> handle, const EsdfConfig& config) {
  DenseEsdf esdf;
  esdf.config = config;
  esdf.handle = std::move(handle);
  const std::shared_ptr<ks_esdf> h = esdf.handle;
  const std::size_t cells = config.cell_count();
  using Site = std::array<std::int32_t, 3>;
  esdf.site = b200_detail::HostMirror<Site>([h] { return ks_esdf_generation(h.get()); }, [h, cells](std::vector<Site>& out) {
    out.resize(cells);
    b200_detail::check(ks_esdf_download(h.get(), &out[0][0], nullptr, nullptr));
  });
  esdf.distance = b200_detail::HostMirror<double>([h] { return ks_esdf_generation(h.get()); }, [h, cells](std::vector<double>& out) {
    out.resize(cells);
    b200_detail::check(ks_esdf_download(h.get(), nullptr, out.data(), nullptr));
  });
  return esdf;
}

inline SeedMask seed_scatter(const SparseTsdf& tsdf, const EsdfConfig& config) {  // esdf.hpp:73-98
  DenseEsdf scratch = make_esdf(config);
  SeedMask seeds(config.cell_count(), 0);
  b200_detail::check(ks_esdf_seed(scratch.get(), tsdf.get(), 0, seeds.data()));
  return seeds;
}
inline SeedMask seed_gather(const SparseTsdf& tsdf, const EsdfConfig& config) {  // esdf.hpp:102-122
  DenseEsdf scratch = make_esdf(config);
  SeedMask seeds(config.cell_count(), 0);
  b200_detail::check(ks_esdf_seed(scratch.get(), tsdf.get(), 1, seeds.data()));
  return seeds;
}

inline DenseEsdf propagate(const SeedMask& seeds, const EsdfConfig& config) {  // esdf.hpp:193-282
  config.validate();
  if (seeds.size() != config.cell_count()) throw ValidationError("esdf: seed mask size does not match grid");
  DenseEsdf esdf = make_esdf(config);
  b200_detail::check(ks_esdf_propagate(esdf.get(), seeds.data(), static_cast<std::int64_t>(seeds.size())));
  esdf.refresh_flags();
  return esdf;
}

inline DenseEsdf recover_signs(DenseEsdf esdf, const SparseTsdf& tsdf) {  // esdf.hpp:288-320
  b200_detail::check(ks_esdf_recover_signs(esdf.get(), tsdf.get()));
  esdf.refresh_flags();
  return esdf;
}

/// Rebuild into an existing field (no allocation; the per-frame call of a control loop).
inline void build_esdf(const SparseTsdf& tsdf, DenseEsdf& esdf) {
  b200_detail::check(ks_esdf_build(esdf.get(), tsdf.get()));
  esdf.refresh_flags();
}
inline DenseEsdf build_esdf(const SparseTsdf& tsdf, const EsdfConfig& config) {  // esdf.hpp:323-327
  DenseEsdf esdf = make_esdf(config);
  build_esdf(tsdf, esdf);
  return esdf;
}

struct EsdfSample {  // esdf.hpp:329-333
  double distance = kInf;
  Vec3 gradient = Vec3::Zero();
  bool inside = false;
};

inline EsdfSample query(const DenseEsdf& esdf, const Vec3& point) {  // esdf.hpp:337-387
  const double p[3] = {point[0], point[1], point[2]};
  double d = kInf, g[3] = {0.0, 0.0, 0.0};
  std::uint8_t inside = 0;
  b200_detail::check(ks_esdf_query(esdf.get(), p, 1, &d, g, &inside));
  EsdfSample s;
  s.distance = d;
  s.gradient = Vec3(g[0], g[1], g[2]);
  s.inside = inside != 0;
  return s;
}

/// Batched query: n points (xyz triples) -> distances, gradients (xyz triples), inside flags.
inline void query_batch(const DenseEsdf& esdf, const std::vector<double>& points_xyz, std::vector<double>& distance,
                        std::vector<double>& gradient_xyz, std::vector<std::uint8_t>& inside) {
  const std::int64_t n = static_cast<std::int64_t>(points_xyz.size() / 3);
  distance.resize(n);
  gradient_xyz.resize(3 * n);
  inside.resize(n);
  b200_detail::check(ks_esdf_query(esdf.get(), points_xyz.data(), n, distance.data(), gradient_xyz.data(), inside.data()));
}


// ---- batched environments (addition: the reference has no batch API; BASELINE configs[4]) ---------------
/// n independent (SparseTsdf, DenseEsdf) pairs of one configuration, updated by one enqueue / one CUDA graph
/// (ks_batch_* in ks_b200.h).  tsdf(i) / esdf(i) are ordinary ks:: worlds -- every function above works on them
/// (query, scene_collision_static, host mirrors ...) -- owned by the batch.
class EnvironmentBatch {
 public:
  struct Summary {  // one row per environment, written by the update itself
    int env = -1;
    double min_distance = kInf;  // over the environment's probe points
    long colliding = 0;          // probes closer than near_distance
    long seeds = 0;
  };

  EnvironmentBatch(int n_envs, const TsdfConfig& tsdf_config, const EsdfConfig& esdf_config, int lanes = 4, int first_env = 0) {
    tsdf_config.validate();
    esdf_config.validate();
    const ks_tsdf_config tc = b200_detail::to_c(tsdf_config);
    const ks_esdf_config ec = b200_detail::to_c(esdf_config);
    ks_batch* raw = nullptr;
    b200_detail::check(ks_batch_create(n_envs, &tc, &ec, lanes, &raw));
    handle_ = std::shared_ptr<ks_batch>(raw, ks_batch_destroy);
    b200_detail::check(ks_batch_set_first_env(raw, first_env));
    for (int i = 0; i < n_envs; ++i) {  // aliasing pointers: a world handed out keeps the whole batch alive
      tsdf_.push_back(b200_detail::wrap_tsdf(std::shared_ptr<ks_tsdf>(handle_, ks_batch_tsdf(raw, i)), tsdf_config));
      esdf_.push_back(b200_detail::wrap_esdf(std::shared_ptr<ks_esdf>(handle_, ks_batch_esdf(raw, i)), esdf_config));
    }
  }
  int size() const { return static_cast<int>(tsdf_.size()); }
  ks_batch* get() const { return handle_.get(); }
  SparseTsdf& tsdf(int env) { return tsdf_.at(static_cast<std::size_t>(env)); }
  DenseEsdf& esdf(int env) { return esdf_.at(static_cast<std::size_t>(env)); }

  /// the frame camera `slot` of environment `env` integrates at the next update (copied into page-locked staging)
  void stage_frame(int env, int slot, const DepthFrame& frame) {
    frame.validate();
    const ks_camera cam = frame.camera();
    b200_detail::check(ks_tsdf_stage_frame_slot(tsdf(env).get(), slot, &cam, frame.depth.data()));
  }
  void set_inputs(int env, int n_cameras, std::span<const Primitive> primitives, std::span<const DeviceMesh> meshes = {}) {
    std::vector<ks_primitive> prims(primitives.size());
    for (std::size_t i = 0; i < primitives.size(); ++i) {
      ks_primitive& out = prims[i];
      out = ks_primitive{};
      if (const auto* cuboid = std::get_if<Cuboid>(&primitives[i])) {
        out.kind = 0;
        b200_detail::fill_pose(cuboid->pose, out.pose_R, out.pose_t);
        for (int a = 0; a < 3; ++a) out.half_extents[a] = cuboid->half_extents[a];
      } else {
        const auto& sphere = std::get<SphereShape>(primitives[i]);
        out.kind = 1;
        for (int a = 0; a < 3; ++a) out.center[a] = sphere.center[a];
        out.radius = sphere.radius;
      }
    }
    std::vector<const ks_mesh*> raw;
    for (const DeviceMesh& m : meshes) raw.push_back(m.handle.get()), meshes_.push_back(m.handle);  // kept alive
    b200_detail::check(ks_batch_set_inputs(get(), env, n_cameras, prims.data(), static_cast<std::int32_t>(prims.size()), raw.data(),
                                           static_cast<std::int32_t>(raw.size())));
  }
  void set_probes(int env, std::span<const Vec3> points, double near_distance) {
    std::vector<double> xyz;
    for (const Vec3& p : points) xyz.insert(xyz.end(), {p[0], p[1], p[2]});
    b200_detail::check(ks_batch_set_probes(get(), env, xyz.data(), static_cast<std::int64_t>(points.size()), near_distance));
  }
  /// one update of every environment through the batch's own graph; returns without waiting
  void update(bool upload_frames = true) { b200_detail::check(ks_batch_update(get(), upload_frames ? 1 : 0)); }
  /// wait; throws ValidationError("environment <id>: <the reference's text>") for the first failing environment
  std::vector<Summary> sync() {
    std::vector<double> rows(4 * static_cast<std::size_t>(size()));
    std::vector<ks_esdf_report> ereps(static_cast<std::size_t>(size()));
    b200_detail::check(ks_batch_sync(get(), nullptr, ereps.data(), rows.data()));
    std::vector<Summary> out(static_cast<std::size_t>(size()));
    for (int i = 0; i < size(); ++i) {
      esdf_[i].has_sites = ereps[i].has_sites != 0, esdf_[i].signs_recovered = ereps[i].signs_recovered != 0;
      const double* r = &rows[4 * static_cast<std::size_t>(i)];
      if (r[0] == r[0]) out[i] = Summary{static_cast<int>(r[0]), r[1], static_cast<long>(r[2]), static_cast<long>(r[3])};
    }
    return out;
  }

 private:
  std::shared_ptr<ks_batch> handle_;
  std::vector<SparseTsdf> tsdf_;
  std::vector<DenseEsdf> esdf_;
  std::vector<std::shared_ptr<ks_mesh>> meshes_;
};

// ---- collision.hpp, scene part (collision.hpp:30-52, :130-239) ---------------------------------------
}  // namespace ks
#if defined(KS_B200_REFERENCE_COLLISION)
// The reference's own collision.hpp, with its two per-sphere query loops renamed out of the way: everything else
// in it (hinge_cost, hinge_slope, CollisionReport, SelfCollisionConfig, self_collision, SceneCollisionConfig,
// SceneTimestepReport) is used as is.  Its `#include "ks/esdf.hpp"` finds the guard claimed above.  With
// include/ks_b200/overlay first on the include path this resolves to the overlay's ks/collision.hpp, which hands
// over to the reference's file (#include_next) while KS_B200_WRAPPING_COLLISION is defined.
#if defined(KS_COLLISION_HPP)
#error "ks/collision.hpp was included before ks_b200/ks.hpp: include ks_b200/ks.hpp first, or put include/ks_b200/overlay first on the include path"
#endif
#define KS_B200_WRAPPING_COLLISION 1
#define scene_collision_static scene_collision_static_query_loop
#define scene_collision scene_collision_query_loop
#include "ks/collision.hpp"
#undef scene_collision_static
#undef scene_collision
#undef KS_B200_WRAPPING_COLLISION
namespace ks {
#else
namespace ks {
inline double hinge_cost(double clearance, double margin) {  // collision.hpp:30-37
  if (clearance >= margin) return 0.0;
  if (clearance >= 0.0) {
    const double gap = margin - clearance;
    return gap * gap / (2.0 * margin);
  }
  return 0.5 * margin - clearance;
}
inline double hinge_slope(double clearance, double margin) {  // collision.hpp:40-44
  if (clearance >= margin) return 0.0;
  if (clearance >= 0.0) return -(margin - clearance) / margin;
  return -1.0;
}

struct CollisionReport {  // collision.hpp:46-52
  double max_penetration = -kInf;
  int worst_first = -1;
  int worst_second = -1;
  double cost = 0.0;
  std::vector<Vec3> gradient;
};

#endif

/// One batched kernel instead of the reference's per-sphere query loop.
inline CollisionReport scene_collision_static(const DenseEsdf& esdf, std::span<const Vec3> centers,
                                              std::span<const double> radii, double activation_margin = 0.025) {
  if (centers.size() != radii.size()) throw ValidationError("scene_collision: center/radius count mismatch");
  std::vector<double> xyz(3 * centers.size()), grad(3 * centers.size());
  for (std::size_t s = 0; s < centers.size(); ++s)
    for (int a = 0; a < 3; ++a) xyz[3 * s + a] = centers[s][a];
  ks_collision_report rep{};
  b200_detail::check(ks_esdf_scene_collision_static(esdf.get(), xyz.data(), radii.data(), static_cast<std::int64_t>(radii.size()),
                                                    activation_margin, &rep, grad.data()));
  CollisionReport out;
  out.max_penetration = rep.max_penetration;
  out.worst_first = rep.worst_sphere;
  out.cost = rep.cost;
  out.gradient.resize(centers.size());
  for (std::size_t s = 0; s < centers.size(); ++s) out.gradient[s] = Vec3(grad[3 * s], grad[3 * s + 1], grad[3 * s + 2]);
  return out;
}

#if !defined(KS_B200_REFERENCE_COLLISION)
struct SceneCollisionConfig {  // collision.hpp:154-158
  double activation_margin = 0.025;
  double dt = 1.0;
  int max_checks = 10000;
};
struct SceneTimestepReport {  // collision.hpp:161-168
  double max_penetration = -kInf;
  int worst_sphere = -1;
  double cost = 0.0;
  std::vector<Vec3> center_gradient, next_center_gradient, velocity_gradient;
};
#endif

inline std::vector<SceneTimestepReport> scene_collision(const DenseEsdf& esdf, const std::vector<std::vector<Vec3>>& centers,
                                                        std::span<const double> radii,
                                                        const std::vector<std::vector<Vec3>>& velocities,
                                                        const SceneCollisionConfig& config = {}) {  // collision.hpp:177-239
  if (!esdf.signs_recovered) throw ValidationError("scene_collision: esdf signs not recovered");
  if (centers.size() != velocities.size()) throw ValidationError("scene_collision: centers/velocities timestep mismatch");
  const std::size_t steps = centers.size(), spheres = radii.size();
  std::vector<double> c(3 * steps * spheres), v(3 * steps * spheres);
  for (std::size_t t = 0; t < steps; ++t) {
    if (centers[t].size() != spheres || velocities[t].size() != spheres)
      throw ValidationError("scene_collision: sphere count mismatch at timestep");
    for (std::size_t s = 0; s < spheres; ++s)
      for (int a = 0; a < 3; ++a) {
        c[3 * (t * spheres + s) + a] = centers[t][s][a];
        v[3 * (t * spheres + s) + a] = velocities[t][s][a];
      }
  }
  std::vector<ks_collision_report> reps(steps);
  std::vector<double> g0(c.size()), g1(c.size()), g2(c.size());
  if (steps > 0 && spheres > 0)
    b200_detail::check(ks_esdf_scene_collision_swept(esdf.get(), c.data(), radii.data(), v.data(), static_cast<std::int32_t>(steps),
                                                     static_cast<std::int32_t>(spheres), config.activation_margin, config.dt,
                                                     config.max_checks, reps.data(), g0.data(), g1.data(), g2.data()));
  std::vector<SceneTimestepReport> out(steps);
  for (std::size_t t = 0; t < steps; ++t) {
    out[t].max_penetration = spheres ? reps[t].max_penetration : 0.0;
    out[t].worst_sphere = spheres ? reps[t].worst_sphere : -1;
    out[t].cost = spheres ? reps[t].cost : 0.0;
    out[t].center_gradient.resize(spheres);
    out[t].velocity_gradient.resize(spheres);
    if (t + 1 < steps) out[t].next_center_gradient.resize(spheres);
    for (std::size_t s = 0; s < spheres; ++s) {
      const std::size_t at = 3 * (t * spheres + s);
      out[t].center_gradient[s] = Vec3(g0[at], g0[at + 1], g0[at + 2]);
      out[t].velocity_gradient[s] = Vec3(g2[at], g2[at + 1], g2[at + 2]);
      if (t + 1 < steps) out[t].next_center_gradient[s] = Vec3(g1[at], g1[at + 1], g1[at + 2]);
    }
  }
  return out;
}

// ---- file formats (sdf_world.hpp:511-579, esdf.hpp:389-443) ---------------------------------------------
// KSDEPTH1: "KSDEPTH1" + u32 header length + JSON {width,height,fx,fy,cx,cy,pose:{xyz,rpy}} + f32 depths.
// KSESDF1 : "KSESDF1\0" + u32 header length + JSON {origin,dims,voxel_size} + f32 distances (x fastest).
// Host-only code; the JSON headers are flat enough to be written and read without a JSON library.
namespace b200_detail {
inline std::string num(double v) {  // shortest text that reads back to the same double
  char buf[40];
  const auto res = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, res.ptr);
}
/// value text following "key": in a flat JSON object (numbers or [..] arrays of numbers)
inline std::vector<double> json_numbers(const std::string& text, const std::string& key, const std::string& path) {
  const std::size_t k = text.find("\"" + key + "\"");
  if (k == std::string::npos) throw ParseError("'" + path + "': bad header: missing key " + key);
  std::size_t i = text.find(':', k);
  if (i == std::string::npos) throw ParseError("'" + path + "': bad header");
  ++i;
  while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i;
  std::vector<double> out;
  const bool array = i < text.size() && text[i] == '[';
  if (array) ++i;
  while (i < text.size()) {
    while (i < text.size() && (std::isspace(static_cast<unsigned char>(text[i])) || text[i] == ',')) ++i;
    if (i >= text.size() || text[i] == ']' || text[i] == '}') break;
    char* end = nullptr;
    const double v = std::strtod(text.c_str() + i, &end);
    if (end == text.c_str() + i) throw ParseError("'" + path + "': bad header: bad number for " + key);
    out.push_back(v);
    i = static_cast<std::size_t>(end - text.c_str());
    if (!array) break;
  }
  return out;
}
inline Mat3 rpy_to_matrix(double roll, double pitch, double yaw) {  // core.hpp:85-89: Rz(yaw) Ry(pitch) Rx(roll)
  const double cr = std::cos(roll), sr = std::sin(roll), cp = std::cos(pitch), sp = std::sin(pitch), cy = std::cos(yaw),
               sy = std::sin(yaw);
  Mat3 m;
  m(0, 0) = cy * cp, m(0, 1) = cy * sp * sr - sy * cr, m(0, 2) = cy * sp * cr + sy * sr;
  m(1, 0) = sy * cp, m(1, 1) = sy * sp * sr + cy * cr, m(1, 2) = sy * sp * cr - cy * sr;
  m(2, 0) = -sp, m(2, 1) = cp * sr, m(2, 2) = cp * cr;
  return m;
}
}  // namespace b200_detail

inline void save_depth_frame(const std::string& path, const DepthFrame& frame) {  // sdf_world.hpp:518-542
  frame.validate();
  const Mat3& r = frame.pose.rotation;
  const double pitch = std::asin(std::clamp(-r(2, 0), -1.0, 1.0));
  using b200_detail::num;
  const std::string header = "{\"cx\":" + num(frame.cx) + ",\"cy\":" + num(frame.cy) + ",\"fx\":" + num(frame.fx) + ",\"fy\":" +
                             num(frame.fy) + ",\"height\":" + std::to_string(frame.height) + ",\"pose\":{\"rpy\":[" +
                             num(std::atan2(r(2, 1), r(2, 2))) + "," + num(pitch) + "," + num(std::atan2(r(1, 0), r(0, 0))) +
                             "],\"xyz\":[" + num(frame.pose.translation[0]) + "," + num(frame.pose.translation[1]) + "," +
                             num(frame.pose.translation[2]) + "]},\"width\":" + std::to_string(frame.width) + "}";
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ParseError("cannot open '" + path + "' for writing");
  out.write("KSDEPTH1", 8);
  const auto len = static_cast<std::uint32_t>(header.size());
  out.write(reinterpret_cast<const char*>(&len), 4);
  out.write(header.data(), static_cast<std::streamsize>(header.size()));
  out.write(reinterpret_cast<const char*>(frame.depth.data()), static_cast<std::streamsize>(frame.depth.size() * sizeof(float)));
}

inline DepthFrame load_depth_frame(const std::string& path) {  // sdf_world.hpp:544-579
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError("cannot open depth frame '" + path + "'");
  char magic[8];
  in.read(magic, 8);
  if (!in || std::memcmp(magic, "KSDEPTH1", 8) != 0) throw ParseError("'" + path + "' is not a KSDEPTH1 file");
  std::uint32_t len = 0;
  in.read(reinterpret_cast<char*>(&len), 4);
  std::string header(len, '\0');
  in.read(header.data(), len);
  if (!in) throw ParseError("'" + path + "': truncated header");
  using b200_detail::json_numbers;
  DepthFrame frame;
  frame.width = static_cast<int>(json_numbers(header, "width", path).at(0));
  frame.height = static_cast<int>(json_numbers(header, "height", path).at(0));
  frame.fx = json_numbers(header, "fx", path).at(0);
  frame.fy = json_numbers(header, "fy", path).at(0);
  frame.cx = json_numbers(header, "cx", path).at(0);
  frame.cy = json_numbers(header, "cy", path).at(0);
  const std::vector<double> xyz = json_numbers(header, "xyz", path), rpy = json_numbers(header, "rpy", path);
  if (xyz.size() != 3 || rpy.size() != 3) throw ParseError("'" + path + "': bad header: pose");
  frame.pose.translation = Vec3(xyz[0], xyz[1], xyz[2]);
  frame.pose.rotation = b200_detail::rpy_to_matrix(rpy[0], rpy[1], rpy[2]);
  if (frame.width <= 0 || frame.height <= 0) throw ValidationError("depth frame: invalid intrinsics");
  frame.depth.resize(static_cast<std::size_t>(frame.width) * frame.height);
  in.read(reinterpret_cast<char*>(frame.depth.data()), static_cast<std::streamsize>(frame.depth.size() * sizeof(float)));
  if (!in) throw ParseError("'" + path + "': truncated depth data");
  frame.validate();
  return frame;
}

inline void save_esdf(const std::string& path, const DenseEsdf& esdf) {  // esdf.hpp:395-411
  using b200_detail::num;
  const EsdfConfig& c = esdf.config;
  const std::string header = "{\"dims\":[" + std::to_string(c.nx) + "," + std::to_string(c.ny) + "," + std::to_string(c.nz) +
                             "],\"origin\":[" + num(c.origin[0]) + "," + num(c.origin[1]) + "," + num(c.origin[2]) +
                             "],\"voxel_size\":" + num(c.voxel_size) + "}";
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ParseError("cannot open '" + path + "' for writing");
  out.write("KSESDF1\0", 8);
  const auto len = static_cast<std::uint32_t>(header.size());
  out.write(reinterpret_cast<const char*>(&len), 4);
  out.write(header.data(), static_cast<std::streamsize>(header.size()));
  const std::vector<double>& distance = esdf.distance.get();
  std::vector<float> narrow(distance.size());
  for (std::size_t i = 0; i < distance.size(); ++i) narrow[i] = static_cast<float>(distance[i]);
  out.write(reinterpret_cast<const char*>(narrow.data()), static_cast<std::streamsize>(narrow.size() * sizeof(float)));
}

struct EsdfExport {  // esdf.hpp:413-418
  Vec3 origin;
  int nx, ny, nz;
  double voxel_size;
  std::vector<float> distance;
};

inline EsdfExport load_esdf(const std::string& path) {  // esdf.hpp:420-443
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError("cannot open esdf '" + path + "'");
  char magic[8];
  in.read(magic, 8);
  if (!in || std::memcmp(magic, "KSESDF1\0", 8) != 0) throw ParseError("'" + path + "' is not a KSESDF1 file");
  std::uint32_t len = 0;
  in.read(reinterpret_cast<char*>(&len), 4);
  std::string header(len, '\0');
  in.read(header.data(), len);
  using b200_detail::json_numbers;
  const std::vector<double> origin = json_numbers(header, "origin", path), dims = json_numbers(header, "dims", path);
  if (origin.size() != 3 || dims.size() != 3) throw ParseError("'" + path + "': bad header");
  EsdfExport out;
  out.origin = Vec3(origin[0], origin[1], origin[2]);
  out.nx = static_cast<int>(dims[0]), out.ny = static_cast<int>(dims[1]), out.nz = static_cast<int>(dims[2]);
  out.voxel_size = json_numbers(header, "voxel_size", path).at(0);
  out.distance.resize(static_cast<std::size_t>(out.nx) * out.ny * out.nz);
  in.read(reinterpret_cast<char*>(out.distance.data()), static_cast<std::streamsize>(out.distance.size() * sizeof(float)));
  if (!in) throw ParseError("'" + path + "': truncated distance data");
  return out;
}

}  // namespace ks

#endif  // KS_B200_KS_HPP
