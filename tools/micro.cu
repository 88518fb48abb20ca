// micro.cu — measurement kernels for the light path's limiter (not part of the
// product; built by tools/measure_peaks.py into tools/libmicro.so).
//
// red_random: every thread issues `per_thread` u32 atomic adds (RED, result
// unused) at pseudo-random cells of a `cells`-cell array; the cell index is a
// counter hash computed in registers, so the only memory traffic is the RMW of
// the target sectors. With a 32 MB array the sectors stay in L2 (the DNA light
// accumulator); with 800 MB (Scale's triangle) most REDs miss L2 and become DRAM
// sector read-modify-writes.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void red_random_kernel(uint32_t* acc, uint64_t cells, int per_thread, uint64_t seed) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t h = mix64(t ^ seed);
#pragma unroll 4
    for (int i = 0; i < per_thread; ++i) {
        h = mix64(h + 0x9e3779b97f4a7c15ull);
        atomicAdd(&acc[h % cells], 1u);
    }
}

// same, but each warp's 32 lanes hit 32 consecutive cells of one random row
// segment (the pattern of a light group whose pairs fall in one accumulator row)
__global__ void red_rowseg_kernel(uint32_t* acc, uint64_t cells, int per_thread, uint64_t seed) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    uint64_t h = mix64((t >> 5) ^ seed);
#pragma unroll 4
    for (int i = 0; i < per_thread; ++i) {
        h = mix64(h + 0x9e3779b97f4a7c15ull);
        atomicAdd(&acc[(h % (cells - 32)) + lane], 1u);
    }
}

extern "C" int micro_red(uint32_t* acc, uint64_t cells, int blocks, int threads, int per_thread,
                         uint64_t seed, int rowseg, void* stream) {
    if (rowseg)
        red_rowseg_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(acc, cells, per_thread, seed);
    else
        red_random_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(acc, cells, per_thread, seed);
    return (int)cudaGetLastError();
}
