// ks::EnvironmentBatch (ks_b200's addition for BASELINE configs[4]; the reference has no batch API) against
// the reference-shaped free functions of the same header: every environment of a batch must hold exactly the world that
// make_tsdf / integrate_depth / stamp_primitive / build_esdf produce for it alone (those are pinned to the reference by
// dropin_program.cpp).  Prints one line per environment; the test expects "same 1" everywhere.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>
#include "ks_b200/ks.hpp"

static ks::DepthFrame make_frame(int env) {
  ks::DepthFrame frame;
  frame.width = 96, frame.height = 72;
  frame.fx = frame.fy = 80.0, frame.cx = 47.5, frame.cy = 35.5;
  frame.pose.translation = ks::Vec3(0.5, 0.4, -0.3);
  frame.depth.resize(96 * 72);
  for (int py = 0; py < 72; ++py)
    for (int px = 0; px < 96; ++px)
      frame.depth[py * 96 + px] = (px + py + env) % 17 == 0 ? 0.0f : 0.9f + 0.002f * static_cast<float>((px * (7 + env) + py * 3) % 23);
  return frame;
}

static std::vector<ks::Primitive> make_prims(int env) {
  ks::Cuboid box;
  box.pose.translation = ks::Vec3(0.3 + 0.03 * env, 0.3, 0.3);
  box.half_extents = ks::Vec3(0.1, 0.06, 0.12);
  ks::SphereShape ball;
  ball.center = ks::Vec3(0.7, 0.5 - 0.02 * env, 0.25);
  ball.radius = 0.09;
  return {ks::Primitive(box), ks::Primitive(ball)};
}

int main() {
  const int n = 3, updates = 2;
  ks::TsdfConfig config = ks::make_tsdf_config(0.02);
  config.capacity = 4096;
  ks::EsdfConfig grid;
  grid.nx = 50, grid.ny = 40, grid.nz = 30;
  grid.voxel_size = 0.02;
  try {
    ks::EnvironmentBatch batch(n, config, grid, /*lanes=*/2, /*first_env=*/100);
    std::vector<ks::Vec3> probes;
    for (int i = 0; i < 64; ++i) probes.emplace_back(0.015 * i, 0.4, 0.3);
    for (int env = 0; env < n; ++env) {
      batch.stage_frame(env, 0, make_frame(env));
      const std::vector<ks::Primitive> prims = make_prims(env);
      batch.set_inputs(env, 1, prims);
      batch.set_probes(env, probes, 0.05);
    }
    std::vector<ks::EnvironmentBatch::Summary> rows;
    for (int u = 0; u < updates; ++u) batch.update(true);
    rows = batch.sync();
    for (int env = 0; env < n; ++env) {
      ks::SparseTsdf alone = ks::make_tsdf(config);
      for (int u = 0; u < updates; ++u) {
        ks::integrate_depth(alone, make_frame(env));
        for (const ks::Primitive& p : make_prims(env)) ks::stamp_primitive(alone, p);
      }
      const ks::DenseEsdf field = ks::build_esdf(alone, grid);
      const auto& a = field.distance;
      const auto& b = batch.esdf(env).distance;
      const auto& sa = field.site;
      const auto& sb = batch.esdf(env).site;
      bool same = a.size() == b.size() && sa.size() == sb.size();
      for (std::size_t i = 0; same && i < a.size(); ++i) same = std::memcmp(&a[i], &b[i], sizeof(double)) == 0 && sa[i] == sb[i];
      same = same && ks::allocated_block_count(alone) == ks::allocated_block_count(batch.tsdf(env));
      double lo = ks::kInf;
      long near = 0;
      for (const ks::Vec3& p : probes) {
        const double d = ks::query(field, p).distance;
        lo = d < lo ? d : lo;
        near += d < 0.05;
      }
      const auto& r = rows[static_cast<std::size_t>(env)];
      std::printf("env %d same %d cells %zu blocks %d summary %d %d %d flags %d %d\n", r.env, same, a.size(), ks::allocated_block_count(alone),
                  r.min_distance == lo, r.colliding == near, r.seeds > 0, batch.esdf(env).has_sites, batch.esdf(env).signs_recovered);
    }
    // a failing environment is named
    ks::TsdfConfig tiny = config;
    tiny.capacity = 4;
    ks::EnvironmentBatch small(2, tiny, grid, 1, 7);
    small.stage_frame(1, 0, make_frame(0));
    small.set_inputs(0, 0, {});
    small.set_inputs(1, 1, {});
    small.update(true);
    small.sync();
    std::printf("no error?\n");
  } catch (const ks::ValidationError& e) {
    std::printf("ValidationError: %.44s\n", e.what());
  }
  return 0;
}
