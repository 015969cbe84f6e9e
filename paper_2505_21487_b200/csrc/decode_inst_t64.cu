// Decode kernel instantiations with 64-token KV tiles.
#include "decode_inst.h"

namespace glad {
GLAD_INSTANTIATE_T(64)
}  // namespace glad
