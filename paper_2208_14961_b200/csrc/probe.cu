// probe.cu -- pipe-rate microbenchmarks used to state the integer-pipe
// ceiling the fitness kernels are measured against (SURVEY.md section 8d
// flags the POPC rate as an assumption to be measured on the box).
#include "hga_common.cuh"
#include "tcgen05.cuh"

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

// Dense int8 tensor-core rate: one elected thread per CTA issues `iters`
// back-to-back tcgen05.mma.kind::i8 (s8 x s8 -> s32) of shape M x N x 32 from
// shared memory, MN-major no-swizzle operands (the fitness kernels' layout),
// then waits for the last one.  ops = iters * 2MNK.  TILES = 1: the same
// operand tile every time, two accumulators alternating (the pipe's best
// case); TILES > 1: A = B = a different tile each instruction and
// 512 / N accumulators in rotation (what the fitness kernels issue).
template <int M, int N, int TILES>
__global__ void __launch_bounds__(128, 1) k_probe_mma_i8(int64_t iters, uint32_t* out) {
    using namespace tcx;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t done;
    __shared__ uint32_t tmem_base;
    constexpr int MN = M > N ? M : N;
    constexpr int TB = TILES == 1 ? (M + N) * 32 : MN * 32;  // bytes per tile
    constexpr int NACC = TILES == 1 ? 2 : 512 / N;
    for (int i = threadIdx.x; i < TILES * TB / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x01FF01FFu * (uint32_t)(i * 2654435761u | 1u);
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tmem_base)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tmem_base, sa = saddr(smem);
    constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                               ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (threadIdx.x == 0) {
        // MN-major: 16-element groups along M (N) of 4 K-groups x 128 B; SBO = 512 B
        for (int64_t i = 0; i < iters; ++i) {
            const uint32_t t = TILES == 1 ? 0u : (uint32_t)(i % TILES) * TB;
            const uint64_t ad = sdesc(sa + t, 128u, 512u);
            const uint64_t bd = TILES == 1 ? sdesc(sa + M * 32, 128u, 512u) : ad;
            mma_i8(tb + (uint32_t)((i % NACC) * N), ad, bd, IDESC, i >= NACC ? 1u : 0u);
        }
        mma_commit(&done);
        mbar_wait(&done, 0);
    }
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < 32) {
        uint32_t v[16];
        tmem_ld16(tb, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (v[0] == 0x12345678u) out[blockIdx.x] = v[1];
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512) : "memory");
    }
}

// launch-cost probe: every thread touches one word (so the CTA really runs)
__global__ void k_probe_empty(uint32_t* out) {
    extern __shared__ uint32_t sm_dummy[];
    if (threadIdx.x == 0 && blockIdx.x == 0 && out) out[0] = sm_dummy[0] & 0u;
}

}  // namespace hga

extern "C" int hga_probe(int32_t kind, int64_t iters, int32_t blocks, int32_t threads, uint32_t* out,
                         void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (kind == 0) {
        hga::k_probe_popc<<<blocks, threads, 0, st>>>(iters, 12345u, out);
    } else if (kind == 1) {
        hga::k_probe_alu<<<blocks, threads, 0, st>>>(iters, 12345u, out);
    } else if (kind >= 2 && kind <= 9) {
        // one CTA per SM (116 KB of shared memory; the TMEM allocation is 512
        // columns); `threads` ignored.  2: 128x256 (same tile), 3: 64x64 (same
        // tile), 4: 64x64 / 5: 64x48 / 6: 128x128 / 7: 128x96 / 8: 128x64 /
        // 9: 128x256, each with a new 16-deep rotating tile per instruction
        const int smem = 116 * 1024;
        void* k = nullptr;
        switch (kind) {
            case 2: k = (void*)hga::k_probe_mma_i8<128, 256, 1>; break;
            case 3: k = (void*)hga::k_probe_mma_i8<64, 64, 1>; break;
            case 4: k = (void*)hga::k_probe_mma_i8<64, 64, 16>; break;
            case 5: k = (void*)hga::k_probe_mma_i8<64, 48, 16>; break;
            case 6: k = (void*)hga::k_probe_mma_i8<128, 128, 16>; break;
            case 7: k = (void*)hga::k_probe_mma_i8<128, 96, 16>; break;
            case 8: k = (void*)hga::k_probe_mma_i8<128, 64, 16>; break;
            default: k = (void*)hga::k_probe_mma_i8<128, 256, 12>; break;
        }
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return hga::to_rc(e);
        void* args[] = {(void*)&iters, (void*)&out};
        e = cudaLaunchKernel(k, dim3(blocks), dim3(128), args, smem, st);
        if (e != cudaSuccess) return hga::to_rc(e);
    } else if (kind == 10 || kind == 11) {
        // launch cost of a kernel shaped like the generation loop: `blocks` CTAs of
        // `threads` threads with `iters` bytes of dynamic shared memory; 10 = plain
        // launch, 11 = cooperative launch
        const int smem = (int)iters;
        cudaError_t e = cudaFuncSetAttribute((void*)hga::k_probe_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return hga::to_rc(e);
        void* args[] = {(void*)&out};
        e = kind == 10 ? cudaLaunchKernel((void*)hga::k_probe_empty, dim3(blocks), dim3(threads), args, smem, st)
                       : cudaLaunchCooperativeKernel((void*)hga::k_probe_empty, dim3(blocks), dim3(threads), args, smem, st);
        if (e != cudaSuccess) return hga::to_rc(e);
    } else {
        return HGA_E_INVALID;
    }
    return hga::to_rc(cudaGetLastError());
}
