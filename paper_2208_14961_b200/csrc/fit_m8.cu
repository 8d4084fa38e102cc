// fit_m8.cu -- order-8 instantiation of the v2 penalty kernels (fitness_v2.cuh).
#include "fitness_v2.cuh"

namespace hga {
template int launch_fit_v2_m<8>(bool, const void*, int64_t, uint32_t, int64_t*, int64_t*, int64_t*, int64_t*,
                                int32_t*, cudaStream_t);
}  // namespace hga
