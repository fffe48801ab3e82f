// Column-kernel instantiations, float.
#include "fast_launch.cuh"

namespace sdctb {
SDCTB_DEFINE_LAUNCH_COL(float)
}  // namespace sdctb
