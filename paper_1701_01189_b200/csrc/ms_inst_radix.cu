// Kernel instantiations for the radix bucket identifier (see ms_dispatch.cuh).
#include "ms_dispatch.cuh"

namespace ms {
template struct Launch<kRadix>;
}  // namespace ms
