// Decode kernel instantiations with 96-token KV tiles.
#include "decode_inst.h"

namespace glad {
GLAD_INSTANTIATE_T(96)
}  // namespace glad
