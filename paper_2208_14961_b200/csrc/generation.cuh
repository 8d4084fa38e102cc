// generation.cuh -- the fused offspring tile shared by the explicit-plan
// (reference-stream) generation and the Philox persistent loop.
//
// One CTA tile = `ppb` parent pairs -> 2 * ppb offspring.  Thread (ol, j)
// builds column j of local offspring ol straight from the selected parents
// (column-block crossover, engine.py:257-277), applies the offspring's
// mutation plan to that column (engine.py:339-373: the NR row-pair swaps,
// once per occurrence of j in the column list, in plan order), writes the
// column to HBM and to shared memory, and then the tile evaluates all
// offspring with the circulant XOR+POPC schedule of fitness.cu.  Parents are
// never modified.  Columns move whole and swaps exchange a +1 with a -1, so
// column balance and the all-+1 first column are preserved.
#pragma once

#include "hga_common.cuh"

namespace hga {

constexpr int kGenThreads = 256;

struct TileSmem {
    int64_t* poff;     // [2*ppb] word offsets of parents A, B of each pair
    uint32_t* col;     // [2*ppb][2m][W]
    uint32_t* acc;     // [2*ppb][3]
    int16_t* point;    // [ppb]
    int16_t* pcol;     // [2*ppb][nc]
    int16_t* pra;      // [2*ppb][nr]
    int16_t* prb;      // [2*ppb][nr]
};

__host__ __device__ inline size_t tile_smem_bytes(int m, int W, int ppb, int nc, int nr) {
    size_t words = (size_t)2 * ppb * 2 * m * W;
    words = (words + 3) & ~(size_t)3;
    size_t acc = ((size_t)2 * ppb * 3 + 3) & ~(size_t)3;
    size_t shorts = (size_t)ppb + (size_t)2 * ppb * (nc + 2 * nr);
    return (size_t)2 * ppb * 8 + (words + acc) * 4 + ((shorts * 2 + 15) & ~(size_t)15);
}

__device__ inline TileSmem carve_tile(unsigned char* base, int m, int W, int ppb, int nc, int nr) {
    TileSmem t;
    size_t words = ((size_t)2 * ppb * 2 * m * W + 3) & ~(size_t)3;
    t.poff = reinterpret_cast<int64_t*>(base);
    t.col = reinterpret_cast<uint32_t*>(t.poff + 2 * ppb);
    t.acc = t.col + words;
    t.point = reinterpret_cast<int16_t*>(t.acc + (((size_t)2 * ppb * 3 + 3) & ~(size_t)3));
    t.pcol = t.point + ppb;
    t.pra = t.pcol + 2 * ppb * nc;
    t.prb = t.pra + 2 * ppb * nr;
    return t;
}

// Build, mutate, store and evaluate the offspring of pairs [p0, p0 + cnt).
// s.poff[2q], s.poff[2q+1] are the word offsets in `from` of the two parents
// of pair p0+q; offspring go to `to` at slots 2N + p and 3N + p, and with
// COPY_PARENTS the parents themselves are written to slots p and N + p (the
// out-of-place select gather, engine.py:247, fused here).  The plan must be
// in shared memory.  Writes fit[2N+p], fit[3N+p].
template <int W, int VM, bool COPY_PARENTS>
__device__ __forceinline__ void offspring_tile(const TileSmem& s, const uint32_t* __restrict__ from,
                                               uint32_t* __restrict__ to,
                                               int64_t* __restrict__ fit, int64_t N, int64_t p0, int cnt,
                                               int ppb, int m, int nc, int nr, uint32_t fit_var,
                                               unsigned long long* best_key) {
    const int tid = threadIdx.x;
    const int ol = tid / m, j = tid - ol * m;
    const bool active = ol < 2 * ppb && (ol % ppb) < cnt;
    const int64_t mw = (int64_t)m * W;
    Col<W> c;
    if (active) {
        const int q = ol % ppb, second = ol / ppb;  // second: offspring 3N+p
        const int64_t p = p0 + q;
        const int point = s.point[q];
        const bool from_first = (j < point) != (second != 0);  // O1: A|B, O2: B|A
        const int64_t off = s.poff[from_first ? 2 * q : 2 * q + 1];
        const uint32_t* g = from + off + (int64_t)j * W;
#pragma unroll
        for (int w = 0; w < W; ++w) c.w[w] = g[w];
        if (COPY_PARENTS) {
            uint32_t* pd = to + ((from_first ? 0 : N) + p) * mw + (int64_t)j * W;
#pragma unroll
            for (int w = 0; w < W; ++w) pd[w] = c.w[w];
        }
        // mutation: NR swaps once per occurrence of j among the NC columns
        const int16_t* pc = s.pcol + ol * nc;
        const int16_t* pa = s.pra + ol * nr;
        const int16_t* pb = s.prb + ol * nr;
        for (int jc = 0; jc < nc; ++jc) {
            if (pc[jc] != j) continue;
            for (int ir = 0; ir < nr; ++ir) swap_rows<W>(c, pa[ir], pb[ir]);
        }
        uint32_t* dst = to + (2 * N + (int64_t)second * N + p) * mw + (int64_t)j * W;
#pragma unroll
        for (int w = 0; w < W; ++w) dst[w] = c.w[w];
        uint32_t* sc = s.col + ((int64_t)ol * 2 * m + j) * W;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            sc[w] = c.w[w];
            sc[(int64_t)m * W + w] = c.w[w];
        }
    }
    if (tid < 2 * ppb * 3) s.acc[tid] = 0;
    __syncthreads();
    Acc a{0, 0, 0};
    if (active) {
        const int half = (m & 1) ? -1 : m / 2;
        const int steps = pair_steps(m, j);
        const uint32_t* base = s.col + ((int64_t)ol * 2 * m + j) * W;
        for (int d = 1; d <= steps; ++d) {
            int p = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) p += __popc(c.w[w] ^ base[d * W + w]);
            acc_pair<VM>(a, p, m, half);
        }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, active ? ol : -1);
    const bool leader = (__ffs(peers) - 1) == (int)(tid & 31);
    if (VM & HGA_VAR_F1) {
        uint32_t v = __reduce_add_sync(peers, a.s1);
        if (active && leader) atomicAdd(&s.acc[ol * 3 + 0], v);
    }
    if (VM & HGA_VAR_F2) {
        uint32_t v = __reduce_add_sync(peers, a.s2);
        if (active && leader) atomicAdd(&s.acc[ol * 3 + 1], v);
    }
    if (VM & HGA_VAR_SQ) {
        uint32_t v = __reduce_add_sync(peers, a.s4);
        if (active && leader) atomicAdd(&s.acc[ol * 3 + 2], v);
    }
    __syncthreads();
    if (tid < 2 * ppb && (tid % ppb) < cnt) {
        const int q = tid % ppb, second = tid / ppb;
        const int64_t slot = 2 * N + (int64_t)second * N + p0 + q;
        int64_t v;
        if (fit_var == HGA_VAR_F1) v = 2 * (int64_t)s.acc[tid * 3 + 0];
        else if (fit_var == HGA_VAR_SQ) v = 2 * (int64_t)s.acc[tid * 3 + 2];
        else v = 2 * (int64_t)s.acc[tid * 3 + 1];
        fit[slot] = v;
        if (best_key) atomicMin(best_key, ((unsigned long long)v << 32) | (unsigned long long)slot);
    }
    __syncthreads();
}

}  // namespace hga
