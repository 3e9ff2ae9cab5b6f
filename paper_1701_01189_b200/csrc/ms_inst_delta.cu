// Kernel instantiations for the delta bucket identifier (see ms_dispatch.cuh).
#include "ms_dispatch.cuh"

namespace ms {
template struct Launch<kDelta>;
}  // namespace ms
