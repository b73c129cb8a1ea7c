// A planner-side program that mixes the perception path with the reference's OWN collision.hpp, the way
// /root/reference/proj/include/ks/ik.hpp does (:23 includes "ks/collision.hpp"; :117-120 fill_flags and :217-226 call
// self_collision and scene_collision_static on a `const DenseEsdf* world`).  Not a single line names ks_b200.
// Compiled twice by tests/test_cpp_dropin.py from this one source:
//   reference : -I oracle/ref_stubs -I /root/reference/proj/include                                  (CPU)  -> golden
//   ks_b200   : -I include/ks_b200/overlay -I include -I oracle/ref_stubs -I /root/reference/proj/include   (B200)
// The overlay swaps sdf_world.hpp / esdf.hpp for the device-backed ones and turns collision.hpp's two scene
// functions into batched GPU calls; self_collision, CollisionReport, hinge_cost stay the reference's.
#include <cmath>
#include <cstdio>
#include <vector>

#include "ks/collision.hpp"
#include "ks/esdf.hpp"
#include "ks/sdf_world.hpp"

namespace {

struct Flags {
  bool self_free = false, scene_free = false;
  double self_pen = 0.0, scene_pen = 0.0, scene_cost = 0.0;
};

// ik.hpp:114-127 (ik_detail::fill_flags) with the kinematics replaced by given sphere centres
Flags fill_flags(const ks::RobotModel& model, const ks::DenseEsdf* world, const std::vector<ks::Vec3>& centers, double margin) {
  Flags out;
  const ks::CollisionReport self = ks::self_collision(model, centers, {margin, 1024, false});
  out.self_pen = self.max_penetration;
  out.self_free = self.max_penetration <= 1e-4;
  if (world != nullptr) {
    const ks::CollisionReport scene = ks::scene_collision_static(*world, centers, model.sphere_radius, margin);
    out.scene_pen = scene.max_penetration;
    out.scene_cost = scene.cost;
    out.scene_free = scene.max_penetration <= 1e-4;
  } else {
    out.scene_free = true;
  }
  return out;
}

}  // namespace

int main() {
  ks::TsdfConfig config = ks::make_tsdf_config(0.02);
  config.capacity = 2048;
  ks::SparseTsdf world = ks::make_tsdf(config);
  ks::Cuboid box;
  box.pose.translation = ks::Vec3(0.4, 0.3, 0.3);
  box.half_extents = ks::Vec3(0.12, 0.08, 0.1);
  ks::stamp_primitive(world, ks::Primitive(box));
  ks::SphereShape ball;
  ball.center = ks::Vec3(0.75, 0.45, 0.3);
  ball.radius = 0.1;
  ks::stamp_primitive(world, ks::Primitive(ball));

  // the public members of the world (sdf_world.hpp:206-210), read the way user code reads them
  const int live = world.table.live_count();
  const int pool_of = world.table.find(ks::BlockKey{2, 1, 1});
  double geom_min = ks::kInf;
  if (pool_of >= 0)
    for (double g : world.pool[static_cast<std::size_t>(pool_of)].geom_sdf) geom_min = g < geom_min ? g : geom_min;
  std::printf("table live %d available %d next_fresh %d find %d geom_min %.17g\n", live, world.table.available(),
              static_cast<int>(world.table.next_fresh), pool_of, geom_min);

  ks::EsdfConfig grid;
  grid.nx = 50, grid.ny = 36, grid.nz = 30;
  grid.voxel_size = 0.02;
  const ks::DenseEsdf esdf = ks::build_esdf(world, grid);
  // DenseEsdf::site / ::distance as plain members (esdf.hpp:58-64)
  double sum = 0.0;
  long negatives = 0, site_sum = 0;
  for (std::size_t i = 0; i < esdf.distance.size(); ++i) {
    sum += std::fabs(esdf.distance[i]);
    negatives += std::signbit(esdf.distance[i]);
    site_sum += esdf.site[i][0] + 2 * esdf.site[i][1] + 3 * esdf.site[i][2];
  }
  std::printf("esdf %d %d %.17g %ld %ld\n", esdf.has_sites, esdf.signs_recovered, sum, negatives, site_sum);

  ks::RobotModel model;
  std::vector<ks::Vec3> centers;
  for (int i = 0; i < 10; ++i) {
    model.sphere_link.push_back(i / 2);
    model.sphere_radius.push_back(0.03 + 0.003 * i);
    centers.emplace_back(0.1 + 0.085 * i, 0.3 + 0.012 * i, 0.28 + 0.004 * i);
  }
  for (int i = 0; i < 10; ++i)
    for (int j = i + 2; j < 10; j += 3) model.cache.self_collision_pairs.emplace_back(i, j);
  const Flags with_world = fill_flags(model, &esdf, centers, 0.03);
  const Flags without = fill_flags(model, nullptr, centers, 0.03);
  std::printf("flags %d %d %.17g %.17g %.12g | %d %d\n", with_world.self_free, with_world.scene_free, with_world.self_pen,
              with_world.scene_pen, with_world.scene_cost, without.self_free, without.scene_free);

  // swept scene check over three timesteps (collision.hpp:177-239)
  std::vector<std::vector<ks::Vec3>> traj(3, centers), vel(3, std::vector<ks::Vec3>(10, ks::Vec3(0.2, 0.05, -0.1)));
  for (int t = 0; t < 3; ++t)
    for (auto& c : traj[t]) c += ks::Vec3(0.03 * t, 0.01 * t, 0.0);
  const std::vector<ks::SceneTimestepReport> swept = ks::scene_collision(esdf, traj, model.sphere_radius, vel);
  for (const auto& r : swept)
    std::printf("swept %.17g %d %.12g %.17g\n", r.max_penetration, r.worst_sphere, r.cost, r.center_gradient[4].x());
  return 0;
}
