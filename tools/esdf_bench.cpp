// esdf-bench: the reference spec's `ks esdf-bench <scenario> -o <dir> [--seeding scatter|gather] [--brute-force]`
// (SPEC.md "cmd_esdf_bench", External Interfaces; paper §7.6: depth image to ESDF generation time, memory
// as block counts, collision recall), written against the drop-in header include/ks_b200/ks.hpp.
// The reference ships no source for its CLI, so this follows the spec text:
//   * builds the TSDF from the scenario's depth frames (KSDEPTH1 files) and primitives,
//   * generates the ESDF with both seeding modes (or the one asked for),
//   * optionally compares with a brute-force distance transform over the same seeds,
//   * writes per-stage timings (wall clock, 3 warm-up + 10 measured repetitions, median -- SPEC.md:813),
//     recall against the analytic primitives / the brute-force field, and block counts.
// Exit codes: 0 success, 1 validation failure, 2 usage / parse error.
//
// Scenario (the `world` / `esdf` part of the spec's ScenarioFile; `robot` / `problems` are not on this path):
//   {"world": {"cuboids": [{"center": [x,y,z], "half_extents": [a,b,c], "rpy": [r,p,y]}],
//              "spheres": [{"center": [x,y,z], "radius": r}],
//              "depth_frames": ["frame0.ksdepth", ...]},            // relative to the scenario file
//    "tsdf": {"voxel_size": v, "capacity": n},                      // optional; default voxel = the ESDF's
//    "esdf": {"origin": [x,y,z], "dims": [nx,ny,nz], "voxel_size": v, "seeding": "gather"}}
#include <chrono>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <map>
#include <random>

#include "ks_b200/ks.hpp"

namespace {

// ---- a small JSON reader (objects, arrays, numbers, strings, true/false/null) ----
struct Json {
  enum Kind { kNull, kBool, kNumber, kString, kArray, kObject } kind = kNull;
  double number = 0.0;
  bool boolean = false;
  std::string text;
  std::vector<Json> items;
  std::map<std::string, Json> fields;
  const Json* find(const std::string& key) const {
    auto it = fields.find(key);
    return it == fields.end() ? nullptr : &it->second;
  }
};

struct JsonReader {
  const std::string& s;
  size_t i = 0;
  explicit JsonReader(const std::string& text) : s(text) {}
  [[noreturn]] void fail(const std::string& what) const { throw ks::ParseError("scenario: " + what + " at byte " + std::to_string(i)); }
  void skip() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
  }
  Json value() {
    skip();
    if (i >= s.size()) fail("unexpected end");
    Json v;
    const char c = s[i];
    if (c == '{') {
      v.kind = Json::kObject;
      ++i;
      skip();
      if (i < s.size() && s[i] == '}') return ++i, v;
      while (true) {
        skip();
        if (i >= s.size() || s[i] != '"') fail("expected a key");
        const std::string key = string();
        skip();
        if (i >= s.size() || s[i] != ':') fail("expected ':'");
        ++i;
        v.fields[key] = value();
        skip();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == '}') return ++i, v;
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::kArray;
      ++i;
      skip();
      if (i < s.size() && s[i] == ']') return ++i, v;
      while (true) {
        v.items.push_back(value());
        skip();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == ']') return ++i, v;
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::kString;
      v.text = string();
      return v;
    }
    if (s.compare(i, 4, "true") == 0) return i += 4, v.kind = Json::kBool, v.boolean = true, v;
    if (s.compare(i, 5, "false") == 0) return i += 5, v.kind = Json::kBool, v;
    if (s.compare(i, 4, "null") == 0) return i += 4, v;
    char* end = nullptr;
    v.number = std::strtod(s.c_str() + i, &end);
    if (end == s.c_str() + i) fail("unexpected character");
    i = static_cast<size_t>(end - s.c_str());
    v.kind = Json::kNumber;
    return v;
  }
  std::string string() {
    std::string out;
    for (++i; i < s.size() && s[i] != '"'; ++i) {
      if (s[i] == '\\' && i + 1 < s.size()) ++i;
      out.push_back(s[i]);
    }
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
};

ks::Vec3 vec3_of(const Json* j, const char* what) {
  if (!j || j->kind != Json::kArray || j->items.size() != 3) throw ks::ParseError(std::string("scenario: ") + what + " must be three numbers");
  return ks::Vec3(j->items[0].number, j->items[1].number, j->items[2].number);
}

struct Scenario {
  std::vector<ks::Primitive> primitives;
  std::vector<ks::Cuboid> cuboids;
  std::vector<ks::SphereShape> spheres;
  std::vector<ks::DepthFrame> frames;
  ks::TsdfConfig tsdf;
  ks::EsdfConfig esdf;
};

Scenario load_scenario(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ks::ParseError("scenario: cannot open " + path);
  std::stringstream buffer;
  buffer << in.rdbuf();
  const std::string text = buffer.str();
  JsonReader reader(text);
  const Json root = reader.value();
  if (root.kind != Json::kObject) throw ks::ParseError("scenario: top level must be an object");
  Scenario sc;
  const Json* esdf = root.find("esdf");
  if (!esdf) throw ks::ParseError("scenario: missing \"esdf\"");
  sc.esdf.origin = vec3_of(esdf->find("origin"), "esdf.origin");
  const Json* dims = esdf->find("dims");
  if (!dims || dims->items.size() != 3) throw ks::ParseError("scenario: esdf.dims must be three integers");
  sc.esdf.nx = static_cast<int>(dims->items[0].number), sc.esdf.ny = static_cast<int>(dims->items[1].number),
  sc.esdf.nz = static_cast<int>(dims->items[2].number);
  if (const Json* v = esdf->find("voxel_size")) sc.esdf.voxel_size = v->number;
  if (const Json* v = esdf->find("seeding")) sc.esdf.seeding = v->text == "scatter" ? ks::SeedingMode::kScatter : ks::SeedingMode::kGather;
  sc.tsdf = ks::make_tsdf_config(sc.esdf.voxel_size);
  if (const Json* t = root.find("tsdf")) {
    if (const Json* v = t->find("voxel_size")) sc.tsdf = ks::make_tsdf_config(v->number);
    if (const Json* v = t->find("capacity")) sc.tsdf.capacity = static_cast<int>(v->number);
  }
  const std::filesystem::path base = std::filesystem::path(path).parent_path();
  if (const Json* world = root.find("world")) {
    if (const Json* list = world->find("cuboids"))
      for (const Json& c : list->items) {
        ks::Cuboid cuboid;
        cuboid.pose.translation = vec3_of(c.find("center"), "cuboid.center");
        cuboid.half_extents = vec3_of(c.find("half_extents"), "cuboid.half_extents");
        if (const Json* rpy = c.find("rpy")) {
          const ks::Vec3 a = vec3_of(rpy, "cuboid.rpy");
          cuboid.pose.rotation = ks::b200_detail::rpy_to_matrix(a[0], a[1], a[2]);
        }
        sc.cuboids.push_back(cuboid);
        sc.primitives.emplace_back(cuboid);
      }
    if (const Json* list = world->find("spheres"))
      for (const Json& s : list->items) {
        ks::SphereShape sphere;
        sphere.center = vec3_of(s.find("center"), "sphere.center");
        const Json* r = s.find("radius");
        if (!r) throw ks::ParseError("scenario: sphere.radius missing");
        sphere.radius = r->number;
        sc.spheres.push_back(sphere);
        sc.primitives.emplace_back(sphere);
      }
    if (const Json* list = world->find("depth_frames"))
      for (const Json& f : list->items) sc.frames.push_back(ks::load_depth_frame((base / f.text).string()));
  }
  return sc;
}

double box_sdf(const ks::Cuboid& c, const ks::Vec3& p) {  // sdf_cuboid (sdf_world.hpp:224-230)
  const ks::Vec3 local = c.pose.rotation.transpose() * (p - c.pose.translation);
  const ks::Vec3 q = local.cwiseAbs() - c.half_extents;
  return q.cwiseMax(0.0).norm() + std::min(q.maxCoeff(), 0.0);
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v.empty() ? 0.0 : v[v.size() / 2];
}

template <class Fn>
double timed_ms(Fn&& fn) {
  const auto t0 = std::chrono::steady_clock::now();
  fn();
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int usage() {
  std::cerr << "usage: esdf-bench <scenario.json> -o <dir> [--seeding scatter|gather] [--brute-force]\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  std::string scenario_path, out_dir;
  std::vector<ks::SeedingMode> modes = {ks::SeedingMode::kScatter, ks::SeedingMode::kGather};
  bool brute = false;
  for (int a = 1; a < argc; ++a) {
    const std::string arg = argv[a];
    if (arg == "-o" && a + 1 < argc) out_dir = argv[++a];
    else if (arg == "--seeding" && a + 1 < argc) {
      const std::string m = argv[++a];
      if (m != "scatter" && m != "gather") return usage();
      modes = {m == "scatter" ? ks::SeedingMode::kScatter : ks::SeedingMode::kGather};
    } else if (arg == "--brute-force") brute = true;
    else if (!arg.empty() && arg[0] == '-') return usage();
    else if (scenario_path.empty()) scenario_path = arg;
    else return usage();
  }
  if (scenario_path.empty() || out_dir.empty()) return usage();

  Scenario sc;
  try {
    sc = load_scenario(scenario_path);
  } catch (const std::exception& e) {
    std::cerr << e.what() << "\n";
    return 2;
  }
  try {
    sc.esdf.validate();
    if (sc.frames.empty() && sc.primitives.empty()) throw ks::ValidationError("esdf-bench: scenario provides neither depth frames nor primitives");
    std::filesystem::create_directories(out_dir);
    constexpr int kWarm = 3, kReps = 10;
    std::ofstream timings(out_dir + "/timings.csv"), recall(out_dir + "/recall.csv"), summary(out_dir + "/summary.json");
    timings << "stage,seeding,median_ms,repetitions\n";
    recall << "seeding,truth,radius_voxels,truth_positive,detected,recall,max_abs_delta_voxels\n";

    // TSDF: a fresh world per repetition so that allocation is part of what is timed
    std::vector<double> t_integrate, t_stamp;
    ks::SparseTsdf tsdf;
    int touched = 0;
    for (int rep = 0; rep < kWarm + kReps; ++rep) {
      tsdf = ks::make_tsdf(sc.tsdf);
      const double a = timed_ms([&] {
        for (const ks::DepthFrame& f : sc.frames) touched = ks::integrate_depth(tsdf, f);
      });
      const double b = timed_ms([&] {
        for (const ks::Primitive& p : sc.primitives) ks::stamp_primitive(tsdf, p);
        (void)ks::allocated_block_count(tsdf);  // waits for the stamps
      });
      if (rep >= kWarm) t_integrate.push_back(a), t_stamp.push_back(b);
    }
    timings << "integrate,-," << median(t_integrate) << "," << kReps << "\n";
    timings << "stamp,-," << median(t_stamp) << "," << kReps << "\n";
    const int blocks = ks::allocated_block_count(tsdf);

    // query points for the recall figures (fixed seed, recorded in the summary)
    constexpr unsigned kSeed = 7;
    constexpr int kPoints = 20000;
    std::mt19937 rng(kSeed);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    std::vector<double> pts(3 * kPoints);
    const double ext[3] = {sc.esdf.nx * sc.esdf.voxel_size, sc.esdf.ny * sc.esdf.voxel_size, sc.esdf.nz * sc.esdf.voxel_size};
    for (int i = 0; i < kPoints; ++i)
      for (int a = 0; a < 3; ++a) pts[3 * i + a] = sc.esdf.origin[a] + unit(rng) * ext[a];
    const bool analytic = sc.frames.empty();  // analytic ground truth exists for primitive-only scenes

    summary << "{\n  \"scenario\": \"" << scenario_path << "\",\n  \"cells\": " << sc.esdf.cell_count() << ",\n  \"tsdf_blocks\": " << blocks
            << ",\n  \"tsdf_voxels\": " << static_cast<long long>(blocks) * ks::kBlockVoxels << ",\n  \"blocks_touched_last_frame\": " << touched
            << ",\n  \"query_seed\": " << kSeed << ",\n  \"query_points\": " << kPoints << ",\n  \"modes\": {";
    bool first_mode = true;
    for (const ks::SeedingMode mode : modes) {
      const char* name = mode == ks::SeedingMode::kScatter ? "scatter" : "gather";
      ks::EsdfConfig cfg = sc.esdf;
      cfg.seeding = mode;
      std::vector<double> t_seed, t_prop, t_sign, t_build;
      ks::SeedMask seeds;
      ks::DenseEsdf esdf = ks::make_esdf(cfg);
      for (int rep = 0; rep < kWarm + kReps; ++rep) {
        const double a = timed_ms([&] { seeds = mode == ks::SeedingMode::kScatter ? ks::seed_scatter(tsdf, cfg) : ks::seed_gather(tsdf, cfg); });
        ks::DenseEsdf staged;
        const double b = timed_ms([&] { staged = ks::propagate(seeds, cfg); });
        const double c = timed_ms([&] { staged = ks::recover_signs(staged, tsdf); });
        const double d = timed_ms([&] { ks::build_esdf(tsdf, esdf); });  // the fused build into an existing field
        if (rep >= kWarm) t_seed.push_back(a), t_prop.push_back(b), t_sign.push_back(c), t_build.push_back(d);
      }
      timings << "seed," << name << "," << median(t_seed) << "," << kReps << "\n";
      timings << "propagate," << name << "," << median(t_prop) << "," << kReps << "\n";
      timings << "recover_signs," << name << "," << median(t_sign) << "," << kReps << "\n";
      timings << "build_esdf," << name << "," << median(t_build) << "," << kReps << "\n";
      long long seed_count = 0;
      for (std::uint8_t s : seeds) seed_count += s != 0;

      std::vector<double> dist, grad;
      std::vector<std::uint8_t> inside;
      ks::query_batch(esdf, pts, dist, grad, inside);
      auto report = [&](const char* truth_name, const std::vector<double>& truth) {
        for (const double radius : {1.0, 4.0}) {
          const double r = radius * cfg.voxel_size;
          long long positive = 0, hit = 0;
          double worst = 0.0;
          for (int i = 0; i < kPoints; ++i) {
            if (!std::isfinite(truth[i])) continue;
            worst = std::max(worst, std::abs(std::abs(dist[i]) - std::abs(truth[i])) / cfg.voxel_size);
            if (std::abs(truth[i]) <= r) {
              ++positive;
              hit += std::abs(dist[i]) <= r + 1e-12;
            }
          }
          recall << name << "," << truth_name << "," << radius << "," << positive << "," << hit << ","
                 << (positive ? static_cast<double>(hit) / positive : 1.0) << "," << worst << "\n";
        }
      };
      if (analytic) {  // |distance to the nearest primitive surface|
        std::vector<double> truth(kPoints);
        for (int i = 0; i < kPoints; ++i) {
          const ks::Vec3 p(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
          double best = ks::kInf;
          for (const ks::Cuboid& c : sc.cuboids) best = std::min(best, std::abs(box_sdf(c, p)));
          for (const ks::SphereShape& s : sc.spheres) best = std::min(best, std::abs((p - s.center).norm() - s.radius));
          truth[i] = best;
        }
        report("analytic", truth);
      }
      double brute_max_delta = -1.0;
      if (brute) {  // exact distance transform by exhaustive search over the same seeds, at the cell centres
        std::vector<std::array<int, 3>> seed_cells;
        for (int z = 0; z < cfg.nz; ++z)
          for (int y = 0; y < cfg.ny; ++y)
            for (int x = 0; x < cfg.nx; ++x)
              if (seeds[cfg.index(x, y, z)]) seed_cells.push_back({x, y, z});
        const std::vector<double> field = esdf.distance();
        std::mt19937 pick(kSeed + 1);
        brute_max_delta = 0.0;
        const int samples = static_cast<int>(std::min<std::size_t>(4000, cfg.cell_count()));
        for (int i = 0; i < samples && !seed_cells.empty(); ++i) {
          const int x = static_cast<int>(pick() % cfg.nx), y = static_cast<int>(pick() % cfg.ny), z = static_cast<int>(pick() % cfg.nz);
          long long best = std::numeric_limits<long long>::max();
          for (const auto& s : seed_cells) {
            const long long dx = x - s[0], dy = y - s[1], dz = z - s[2];
            best = std::min(best, dx * dx + dy * dy + dz * dz);
          }
          // the field stores sqrt(d2) * voxel_size: recover the integer d2 it was formed from and compare exactly
          const double in_voxels = std::abs(field[cfg.index(x, y, z)]) / cfg.voxel_size;
          const long long got = std::llround(in_voxels * in_voxels);
          brute_max_delta = std::max(brute_max_delta, std::abs(std::sqrt(static_cast<double>(got)) - std::sqrt(static_cast<double>(best))));
        }
        recall << name << ",brute-force-cells,0," << samples << "," << samples << ",1," << brute_max_delta << "\n";
      }
      summary << (first_mode ? "" : ",") << "\n    \"" << name << "\": {\"seeds\": " << seed_count << ", \"has_sites\": " << (esdf.has_sites ? "true" : "false")
              << ", \"brute_force_max_abs_delta_voxels\": " << (brute ? std::to_string(brute_max_delta) : std::string("null")) << "}";
      first_mode = false;
    }
    summary << "\n  }\n}\n";
  } catch (const std::exception& e) {
    std::cerr << e.what() << "\n";
    return 1;
  }
  return 0;
}
