// Kernel instantiations for the deltashift bucket identifier (see ms_dispatch.cuh).
#include "ms_dispatch.cuh"

namespace ms {
template struct Launch<kDeltaShift>;
}  // namespace ms
