// light.cu — group -> C_m update for groups with few sequences (countAndUpdate,
// second half; Algorithm 1 lines 15-17).
//
// For a group (one masked key) whose sorted triples are (X_1,c_1) < ... < (X_s,c_s),
// every unordered pair a < b adds c_a*c_b to C_m(X_a, X_b) — the upper triangle,
// since X_a < X_b; the epilogue mirrors it (reading A4). Integer adds
// commute, so the atomic update order never changes the result.
//
// One warp per group: the warp walks rows a and its lanes take columns b.
#include "internal.cuh"

namespace gk {

__global__ void __launch_bounds__(256) light_kernel(SegmentOut so, int64_t heavy_min, int64_t N,
                                                    int64_t* Cm, uint32_t* heavy,
                                                    uint32_t* heavy_count,
                                                    unsigned long long* stats) {
    const uint32_t G = so.counts[1];
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long pairs = 0, nheavy = 0;
    for (uint64_t gi = warp; gi < G; gi += nwarps) {
        const uint32_t a0 = so.gstart[gi], b0 = so.gend[gi];
        const uint32_t s = b0 - a0;
        if ((int64_t)s >= heavy_min) {
            // dense tensor-core path if every count fits the u8 operand
            uint32_t cmax = 0;
            for (uint32_t t = a0 + lane; t < b0; t += 32) cmax = max(cmax, so.tcnt[t]);
            cmax = __reduce_max_sync(0xffffffffu, cmax);
            if (cmax <= 255u) {
                if (lane == 0) heavy[atomicAdd(heavy_count, 1u)] = (uint32_t)gi;
                ++nheavy;
                continue;
            }
        }
        pairs += (unsigned long long)s * (s - 1) / 2;
        for (uint32_t a = a0; a + 1 < b0; ++a) {
            const int64_t xa = so.tseq[a] & 0x7fffffffu;
            const uint64_t ca = so.tcnt[a];
            int64_t* row = Cm + xa * N;
            for (uint32_t b = a + 1 + lane; b < b0; b += 32) {
                const int64_t xb = so.tseq[b] & 0x7fffffffu;
                atomicAdd((unsigned long long*)&row[xb], ca * so.tcnt[b]);
            }
        }
    }
    if (lane == 0 && pairs) atomicAdd(&stats[ST_LIGHT_PAIRS], pairs);
    if (lane == 0 && nheavy) atomicAdd(&stats[ST_HEAVY_GROUPS], nheavy);
}

cudaError_t launch_light(SegmentOut so, uint64_t max_groups, int64_t heavy_min, int64_t N,
                         int64_t* Cm, uint32_t* heavy, uint32_t* heavy_count,
                         unsigned long long* stats, int sm_count, cudaStream_t s) {
    cudaError_t e = heavy_count ? cudaMemsetAsync(heavy_count, 0, sizeof(uint32_t), s)
                                : cudaSuccess;
    if (e != cudaSuccess || max_groups == 0) return e;
    uint64_t blocks = (max_groups + 7) / 8;
    uint64_t cap = (uint64_t)sm_count * 8;
    if (blocks > cap) blocks = cap;
    light_kernel<<<(unsigned)blocks, 256, 0, s>>>(so, heavy_min, N, Cm, heavy, heavy_count,
                                                  stats);
    return cudaGetLastError();
}

// Closed-form diagonal part: every g-mer of X matches itself under every mask, so
// each of the nmask masks adds n_X = gofs[X+1]-gofs[X] to C_m(X,X).
__global__ void diag_closed_form_kernel(const int64_t* __restrict__ gofs, int64_t N, int64_t nmask,
                                        int64_t* Cm) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
         x += (int64_t)gridDim.x * blockDim.x)
        Cm[x * N + x] += nmask * (gofs[x + 1] - gofs[x]);
}

cudaError_t launch_diag_closed_form(const int64_t* gofs, int64_t N, int64_t nmask, int64_t* Cm,
                                    cudaStream_t s) {
    int64_t blocks = (N + 255) / 256;
    diag_closed_form_kernel<<<(int)(blocks < 1024 ? blocks : 1024), 256, 0, s>>>(gofs, N, nmask,
                                                                                 Cm);
    return cudaGetLastError();
}

}  // namespace gk
