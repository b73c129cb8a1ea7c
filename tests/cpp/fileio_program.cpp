// Host-only check of the KSDEPTH1 / KSESDF1 file formats (sdf_world.hpp:511-579, esdf.hpp:389-443).
//   fileio_program make <dir>                 (reference build only) writes <dir>/frame.ksdepth, <dir>/field.ksesdf
//   fileio_program read <frame> <esdf> <out>  loads both, prints every field, re-saves the frame to <out>
// Built with -DUSE_REFERENCE against the reference headers and without it against include/ks_b200/ks.hpp.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#ifdef USE_REFERENCE
#include "ks/esdf.hpp"
#include "ks/sdf_world.hpp"
#else
#include "ks_b200/ks.hpp"
#endif

int main(int argc, char** argv) {
  if (argc >= 3 && std::strcmp(argv[1], "make") == 0) {
#ifdef USE_REFERENCE
    const std::string dir = argv[2];
    ks::DepthFrame frame;
    frame.width = 24, frame.height = 18;
    frame.fx = 21.5, frame.fy = 22.25, frame.cx = 11.5, frame.cy = 8.5;
    frame.pose.translation = ks::Vec3(0.125, -0.7, 1.5);
    frame.pose.rotation = ks::rpy_to_matrix(0.3, -0.2, 1.1);
    frame.depth.resize(24 * 18);
    for (int i = 0; i < 24 * 18; ++i) frame.depth[i] = i % 13 == 0 ? 0.0f : 0.5f + 0.01f * static_cast<float>(i % 37);
    ks::save_depth_frame(dir + "/frame.ksdepth", frame);
    ks::DenseEsdf esdf;
    esdf.config.origin = ks::Vec3(-0.25, 0.5, 0.0625);
    esdf.config.nx = 12, esdf.config.ny = 10, esdf.config.nz = 8;
    esdf.config.voxel_size = 0.02;
    esdf.distance.resize(12 * 10 * 8);
    for (std::size_t i = 0; i < esdf.distance.size(); ++i) esdf.distance[i] = std::sin(0.1 * static_cast<double>(i)) * 0.3;
    ks::save_esdf(dir + "/field.ksesdf", esdf);
    return 0;
#else
    std::fprintf(stderr, "make needs the reference build\n");
    return 2;
#endif
  }
  if (argc < 5) return 2;
  const ks::DepthFrame frame = ks::load_depth_frame(argv[2]);
  std::printf("frame %d %d %.17g %.17g %.17g %.17g\n", frame.width, frame.height, frame.fx, frame.fy, frame.cx, frame.cy);
  for (int i = 0; i < 3; ++i)
    std::printf("pose %.12f %.12f %.12f | %.17g\n", frame.pose.rotation(i, 0), frame.pose.rotation(i, 1), frame.pose.rotation(i, 2),
                frame.pose.translation[i]);
  double sum = 0.0;
  int invalid = 0;
  for (float d : frame.depth) {
    sum += d;
    invalid += !frame.depth_valid(d);
  }
  std::printf("depth %zu %.17g %d\n", frame.depth.size(), sum, invalid);
  ks::save_depth_frame(argv[4], frame);
  const ks::EsdfExport field = ks::load_esdf(argv[3]);
  double fsum = 0.0;
  for (float d : field.distance) fsum += d;
  std::printf("esdf %d %d %d %.17g %.17g %.17g %.17g %zu %.17g\n", field.nx, field.ny, field.nz, field.origin[0], field.origin[1],
              field.origin[2], field.voxel_size, field.distance.size(), fsum);
  try {
    ks::load_depth_frame(argv[3]);
  } catch (const ks::ParseError& e) {
    std::printf("error %s\n", std::strstr(e.what(), "is not a KSDEPTH1 file") ? "not a KSDEPTH1 file" : e.what());
  }
  return 0;
}
