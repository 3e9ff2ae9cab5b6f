// Kernel instantiations for the identity bucket identifier (see ms_dispatch.cuh).
#include "ms_dispatch.cuh"

namespace ms {
template struct Launch<kIdentity>;
}  // namespace ms
