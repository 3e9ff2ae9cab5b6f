// Kernel instantiations for the top-bits bucket identifier (see ms_dispatch.cuh).
#include "ms_dispatch.cuh"

namespace ms {
template struct Launch<kTopBits>;
}  // namespace ms
