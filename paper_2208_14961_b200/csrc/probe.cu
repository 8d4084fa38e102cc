// probe.cu -- pipe-rate microbenchmarks used to state the integer-pipe
// ceiling the fitness kernels are measured against (SURVEY.md section 8d
// flags the POPC rate as an assumption to be measured on the box).
#include "hga_common.cuh"

namespace hga {

// 8 independent XOR+POPC chains per thread; iters * 8 popcounts per thread.
__global__ void k_probe_popc(int64_t iters, uint32_t seed, uint32_t* out) {
    uint32_t a[8], acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        a[j] = seed * (threadIdx.x + 1) + j * 0x9E3779B9u;
        acc[j] = 0;
    }
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += __popc(a[j] ^ (uint32_t)it);
    }
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[j];
    if (s == 0xFFFFFFFFu) out[blockIdx.x] = s;
}

// Same loop shape with a plain LOP3+IADD body: the ALU-pipe reference.
__global__ void k_probe_alu(int64_t iters, uint32_t seed, uint32_t* out) {
    uint32_t a[8], acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        a[j] = seed * (threadIdx.x + 1) + j * 0x9E3779B9u;
        acc[j] = 0;
    }
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += (a[j] ^ (uint32_t)it) & 0x0F0F0F0Fu;
    }
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[j];
    if (s == 0xFFFFFFFFu) out[blockIdx.x] = s;
}

}  // namespace hga

extern "C" int hga_probe(int32_t kind, int64_t iters, int32_t blocks, int32_t threads, uint32_t* out,
                         void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (kind == 0)
        hga::k_probe_popc<<<blocks, threads, 0, st>>>(iters, 12345u, out);
    else
        hga::k_probe_alu<<<blocks, threads, 0, st>>>(iters, 12345u, out);
    return hga::to_rc(cudaGetLastError());
}
