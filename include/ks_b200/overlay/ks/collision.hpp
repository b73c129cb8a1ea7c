// Overlay for the reference's ks/collision.hpp (/root/reference/proj/include/ks/collision.hpp).
//
// The reference's collision.hpp is NOT replaced: self_collision, CollisionReport, hinge_cost, ... stay its own.  Only
// its two scene functions (scene_collision_static :130-152, scene_collision :177-239 -- per-sphere query() loops) are
// renamed out of the way by ks_b200/ks.hpp, which then defines them as one batched GPU call each.  This file makes
// that work for code that includes "ks/collision.hpp" (ik.hpp:23 does) before, or without ever, naming ks_b200:
//   first inclusion            -> ks_b200/ks.hpp, which includes "ks/collision.hpp" again with the renames in place
//   that nested inclusion      -> the next ks/collision.hpp on the include path, i.e. the reference's own file
#if defined(KS_B200_WRAPPING_COLLISION)
#include_next "ks/collision.hpp"
#else
#include "ks_b200/ks.hpp"
#endif
