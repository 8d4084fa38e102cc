// run_m16.cu -- order-16 instantiation of the persistent generation loop (run_v2.cuh).
#include "run_v2.cuh"

namespace hga {
template int launch_run_v2_m<16>(const hga_run_args*, cudaStream_t);
}  // namespace hga
