// run_m56.cu -- order-56 instantiation of the persistent generation loop (run_v2.cuh).
#include "run_v2.cuh"

namespace hga {
template int launch_run_v2_m<56>(const hga_run_args*, cudaStream_t);
}  // namespace hga
