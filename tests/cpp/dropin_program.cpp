// A small program written against the reference's ks:: API.  Compiled twice by the tests:
//   -DUSE_REFERENCE : against /root/reference/proj/include (CPU, header-only)  -> golden output
//   default         : against include/ks_b200/ks.hpp + libks_b200.so (B200)    -> must print the same
// There is NO source difference between the two builds: the B200 one puts include/ks_b200/overlay first on the
// include path, which is where "ks/esdf.hpp" etc. then come from; DenseEsdf::distance is a member in both.
#include <cstdio>
#include <cmath>
#include <vector>
#include "ks/collision.hpp"
#include "ks/esdf.hpp"
#include "ks/sdf_world.hpp"

int main(int argc, char** argv) {
  const std::string scratch = argc > 1 ? argv[1] : "/tmp";
  ks::TsdfConfig config = ks::make_tsdf_config(0.02);
  config.capacity = 4096;
  ks::SparseTsdf world = ks::make_tsdf(config);

  ks::DepthFrame frame;
  frame.width = 96, frame.height = 72;
  frame.fx = frame.fy = 80.0, frame.cx = 47.5, frame.cy = 35.5;
  frame.pose.translation = ks::Vec3(0.5, 0.4, -0.3);
  frame.depth.resize(96 * 72);
  for (int py = 0; py < 72; ++py)
    for (int px = 0; px < 96; ++px)
      frame.depth[py * 96 + px] = (px + py) % 17 == 0 ? 0.0f : 0.9f + 0.002f * static_cast<float>((px * 7 + py * 3) % 23);
  const int touched = ks::integrate_depth(world, frame);

  ks::Cuboid box;
  box.pose.translation = ks::Vec3(0.3, 0.3, 0.3);
  box.half_extents = ks::Vec3(0.1, 0.06, 0.12);
  ks::stamp_primitive(world, ks::Primitive(box));
  ks::SphereShape ball;
  ball.center = ks::Vec3(0.7, 0.5, 0.25);
  ball.radius = 0.09;
  ks::stamp_primitive(world, ks::Primitive(ball));

  std::printf("touched %d live %d\n", touched, ks::allocated_block_count(world));
  const auto inside_box = ks::query_tsdf(world, ks::Vec3(0.31, 0.31, 0.31));
  const auto nowhere = ks::query_tsdf(world, ks::Vec3(9.0, 9.0, 9.0));
  std::printf("tsdf %d %.17g %d\n", inside_box.has_value(), inside_box.value_or(0.0), nowhere.has_value());

  ks::EsdfConfig grid;
  grid.nx = 50, grid.ny = 40, grid.nz = 30;
  grid.voxel_size = 0.02;
  const ks::DenseEsdf esdf = ks::build_esdf(world, grid);
  const auto& dist = esdf.distance;
  double sum = 0.0, lo = 1e9;
  long negatives = 0;
  for (double d : dist) {
    sum += std::fabs(d);
    lo = d < lo ? d : lo;
    negatives += std::signbit(d);
  }
  std::printf("esdf %d %d %.17g %.17g %ld\n", esdf.has_sites, esdf.signs_recovered, sum, lo, negatives);
  for (double x : {0.11, 0.52, 0.97, 1.3}) {
    const ks::EsdfSample s = ks::query(esdf, ks::Vec3(x, 0.37, 0.29));
    std::printf("query %.17g %.17g %.17g %.17g %d\n", s.distance, s.gradient.x(), s.gradient.y(), s.gradient.z(), s.inside);
  }
  // scene collision over a few spheres, and the KSESDF1 export round trip
  std::vector<ks::Vec3> centers;
  std::vector<double> radii;
  for (int i = 0; i < 12; ++i) {
    centers.emplace_back(0.08 * i + 0.05, 0.31 + 0.01 * i, 0.2 + 0.015 * i);
    radii.push_back(0.03 + 0.004 * i);
  }
  const ks::CollisionReport hit = ks::scene_collision_static(esdf, centers, radii, 0.03);
  std::printf("collision %.17g %d %.12g %.17g %.17g\n", hit.max_penetration, hit.worst_first, hit.cost, hit.gradient[3].x(),
              hit.gradient[7].z());
  ks::save_esdf(scratch + "/dropin_field.ksesdf", esdf);
  const ks::EsdfExport back = ks::load_esdf(scratch + "/dropin_field.ksesdf");
  double fsum = 0.0;
  for (float d : back.distance) fsum += d;
  std::printf("export %d %d %d %.17g %.17g\n", back.nx, back.ny, back.nz, back.voxel_size, fsum);
  try {
    ks::TsdfConfig tiny = ks::make_tsdf_config(0.02);
    tiny.capacity = 4;
    ks::SparseTsdf small = ks::make_tsdf(tiny);
    ks::integrate_depth(small, frame);
  } catch (const ks::ValidationError& e) {
    std::printf("error %s\n", e.what());
  }
  return 0;
}
