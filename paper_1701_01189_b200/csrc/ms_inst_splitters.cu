// Kernel instantiations for the splitter bucket identifier (see ms_dispatch.cuh).
#include "ms_dispatch.cuh"

namespace ms {
template struct Launch<kSplitters>;
}  // namespace ms
