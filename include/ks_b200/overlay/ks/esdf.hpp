// Overlay for the reference's ks/esdf.hpp (/root/reference/proj/include/ks/esdf.hpp); see ks/sdf_world.hpp next to it.
#include "ks_b200/ks.hpp"
