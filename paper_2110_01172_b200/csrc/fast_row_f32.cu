// Row-kernel instantiations, float.
#include "fast_launch.cuh"

namespace sdctb {
SDCTB_DEFINE_LAUNCH_ROW(float)
}  // namespace sdctb
