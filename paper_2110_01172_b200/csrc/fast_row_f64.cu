// Row-kernel instantiations, double.
#include "fast_launch.cuh"

namespace sdctb {
SDCTB_DEFINE_LAUNCH_ROW(double)
}  // namespace sdctb
