// Stand-in for the reference's ks/robot_model.hpp, used ONLY to compile the unmodified
// ks/collision.hpp into oracle/_ref (TEST INFRASTRUCTURE).  The real header needs dynamic Eigen
// matrices and a JSON robot loader that are neither installed nor on the perception path.
// collision.hpp's scene functions (scene_collision_static, scene_collision; collision.hpp:130-239)
// use nothing from it; self_collision (collision.hpp:64-127, out of scope) touches exactly the
// members declared here.  oracle/Makefile puts this directory FIRST on the include path, so
// `#include "ks/robot_model.hpp"` inside collision.hpp resolves here.
#ifndef KS_ROBOT_MODEL_HPP
#define KS_ROBOT_MODEL_HPP

#include <utility>
#include <vector>

#include "ks/core.hpp"

namespace ks {

struct TopologyCacheStandIn {
  std::vector<std::pair<int, int>> self_collision_pairs;
};

struct RobotModel {
  std::vector<int> sphere_link;
  std::vector<double> sphere_radius;
  TopologyCacheStandIn cache;
  int num_spheres() const { return static_cast<int>(sphere_link.size()); }
};

}  // namespace ks

#endif  // KS_ROBOT_MODEL_HPP
