// K6 placeholder (replaced by the tcgen05 kernel).
#include "../../include/deltaserve_b200.h"
#include <cuda_runtime.h>
namespace ds {
int launch_attn_prefill_sm100(const void*, const ds_entry*, const ds_entry*, int, const void*,
                              const void*, int64_t, const int32_t*, int64_t, int, int, int, float, void*,
                              cudaStream_t) {
  return DS_EUNSUPPORTED;
}
}  // namespace ds
