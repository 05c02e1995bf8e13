// K2 tensor-core path placeholder: filled in by the tcgen05 3xTF32 kernel.
#include "common.cuh"

namespace glint {
int launch_linear_3xtf32(int64_t, int, int, const float*, int64_t, const int64_t*, const float*,
                         int64_t, const float*, int, float*, int64_t, cudaStream_t) {
  set_error("linear: 3xTF32 tcgen05 path not built yet");
  return GLINT_EUNSUPPORTED;
}
}  // namespace glint
