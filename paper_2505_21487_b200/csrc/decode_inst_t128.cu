// Decode kernel instantiations with 128-token KV tiles.
#include "decode_inst.h"

namespace glad {
GLAD_INSTANTIATE_T(128)
}  // namespace glad
