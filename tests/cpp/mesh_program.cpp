// ks.hpp's mesh additions (upload_mesh / stamp_mesh): a 12-triangle box stamped as a mesh must give the world
// that stamp_primitive(Cuboid) gives (same blocks, distances to rounding), and validation throws ks::ValidationError.
#include <cmath>
#include <cstdio>

#include "ks_b200/ks.hpp"

int main() {
  const ks::Vec3 c(0.31, 0.22, 0.18), he(0.11, 0.07, 0.09);
  ks::TriangleMesh box;
  for (int k = 0; k < 8; ++k)
    box.vertices.push_back(ks::Vec3(c[0] + ((k & 1) ? he[0] : -he[0]), c[1] + ((k & 2) ? he[1] : -he[1]), c[2] + ((k & 4) ? he[2] : -he[2])));
  const int quads[6][4] = {{0, 4, 6, 2}, {1, 3, 7, 5}, {0, 1, 5, 4}, {2, 6, 7, 3}, {0, 2, 3, 1}, {4, 5, 7, 6}};
  for (const auto& q : quads) {
    box.triangles.push_back({q[0], q[1], q[2]});
    box.triangles.push_back({q[0], q[2], q[3]});
  }
  ks::TsdfConfig cfg = ks::make_tsdf_config(0.01);
  cfg.capacity = 4096;
  ks::SparseTsdf a = ks::make_tsdf(cfg), b = ks::make_tsdf(cfg);
  ks::Cuboid cuboid;
  cuboid.pose.translation = c;
  cuboid.half_extents = he;
  ks::stamp_primitive(a, ks::Primitive{cuboid});
  const ks::DeviceMesh mesh = ks::upload_mesh(box);
  ks::stamp_mesh(b, mesh);
  std::printf("triangles %d blocks %d %d\n", mesh.triangle_count(), ks::allocated_block_count(a), ks::allocated_block_count(b));
  double worst = 0.0;
  int compared = 0, missing = 0;
  for (int i = 0; i < 4000; ++i) {
    const ks::Vec3 p(c[0] + 0.2 * std::sin(0.7 * i), c[1] + 0.15 * std::sin(1.3 * i + 1.0), c[2] + 0.17 * std::sin(2.1 * i + 2.0));
    const auto ga = ks::query_tsdf_geom(a, p), gb = ks::query_tsdf_geom(b, p);
    if (ga.has_value() != gb.has_value()) ++missing;
    if (ga && gb) worst = std::fmax(worst, std::fabs(*ga - *gb)), ++compared;
  }
  std::printf("compared %s missing %d worst %s\n", compared > 500 ? "many" : "few", missing, worst < 1e-12 ? "ok" : "BAD");
  ks::TriangleMesh bad = box;
  bad.triangles.push_back({0, 0, 1});
  try {
    ks::stamp_mesh(b, bad);
    std::printf("no throw\n");
  } catch (const ks::ValidationError& e) {
    std::printf("ValidationError: %s\n", e.what());
  }
  return 0;
}
