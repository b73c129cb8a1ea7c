// Overlay for the reference's ks/sdf_world.hpp (/root/reference/proj/include/ks/sdf_world.hpp): with this directory
// FIRST on the include path, every `#include "ks/sdf_world.hpp"` -- the caller's own and the ones inside the
// reference's planner headers -- gets the B200-backed API instead.  See ks_b200/ks.hpp.
#include "ks_b200/ks.hpp"
