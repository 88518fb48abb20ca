// shard.cu — the device side of the mask-sharded multi-GPU step.
//
// The C(g,m) masks are independent (Supp. §S:5.3) and C_m is
// an integer sum over masks (Algorithm 1 line 17 P:199), so P ranks each
// accumulate a partial C over their masks and the partials are summed. Only the
// upper triangle (Y >= X, diagonal included) of C_m is ever written by
// gakco_accumulate (reading A4), so the exchange moves that triangle, packed row
// by row:  e(X, Y) = R(X) + (Y - X),  R(X) = X N - X (X - 1) / 2.
//   pack_upper: entries [begin, end) of the packed triangle of `levels` matrices,
//               as int64 or 32-bit words (the host picks 32 bits when the
//               reduced sum is bounded below 2^31);
//   diag:       C_l(X, X) for every X (the normalisation needs all of K(X, X)).
#include <algorithm>

#include "internal.cuh"

namespace gk {

__host__ __device__ inline int64_t tri_row_start(int64_t X, int64_t N) {
    return X * N - X * (X - 1) / 2;
}

// row of packed index e (0 <= e < N (N + 1) / 2): the largest X with R(X) <= e
int64_t tri_row_of(int64_t e, int64_t N) {
    int64_t lo = 0, hi = N - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (tri_row_start(mid, N) <= e) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// one CTA per (row X0 + blockIdx.x, level blockIdx.y): the row's part of the range
template <typename T>
__global__ void __launch_bounds__(256) pack_upper_kernel(const int64_t* __restrict__ C, int64_t N,
                                                         int64_t begin, int64_t end, int64_t X0,
                                                         T* __restrict__ out) {
    const int64_t X = X0 + blockIdx.x;
    const int64_t l = blockIdx.y;
    const int64_t R = tri_row_start(X, N);
    const int64_t lo = max(R, begin), hi = min(R + (N - X), end);
    const int64_t* src = C + (size_t)l * (size_t)N * (size_t)N + (size_t)X * (size_t)N + X - R;
    T* dst = out + (size_t)l * (size_t)(end - begin) - begin;
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) dst[e] = (T)src[e];
}

// rows of the upper triangles: row (l, X) zeroes [X, N), 16-byte stores on the aligned
// body
__global__ void __launch_bounds__(256) zero_upper_kernel(int64_t* __restrict__ C, int64_t N,
                                                         int levels) {
    const int64_t rows = (int64_t)levels * N;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int64_t X = r % N;
        int64_t* row = C + (size_t)r * (size_t)N;
        int64_t a = X;
        if (a < N && (((uintptr_t)(row + a)) & 15)) {  // (8-byte aligned: one scalar head)
            if (threadIdx.x == 0) row[a] = 0;
            ++a;
        }
        const int64_t nv = (N - a) / 2;
        int4* v = (int4*)(row + a);
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) v[i] = make_int4(0, 0, 0, 0);
        if (threadIdx.x == 0 && a + 2 * nv < N) row[N - 1] = 0;
    }
}

cudaError_t launch_zero_upper(int64_t* C, int64_t N, int levels, int sm_count, cudaStream_t s) {
    const int64_t rows = (int64_t)levels * N;
    if (rows <= 0) return cudaGetLastError();
    const int64_t blocks = std::min<int64_t>(rows, (int64_t)sm_count * 8);
    zero_upper_kernel<<<(unsigned)blocks, 256, 0, s>>>(C, N, levels);
    return cudaGetLastError();
}

__global__ void diag_kernel(const int64_t* __restrict__ C, int64_t N, int levels,
                            int64_t* __restrict__ out) {
    const int64_t nn = N * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)levels * N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t l = i / N, x = i - l * N;
        out[i] = C[l * nn + x * N + x];
    }
}

// Fused pack + exchange: level `level` of this rank's C, packed, goes
// straight into the OWNER's receive buffer over NVLink (peer-mapped pointers from
// CUDA IPC): entry e belongs to rank d = e / chunk and lands at
// dst[d][(src * levels + level) * chunk + e - d * chunk]; the owner sums the P
// contributions inside its epilogue (epilogue_packed_kernel with nsrc = P).
template <typename T>
__global__ void __launch_bounds__(256) pack_upper_peers_kernel(const int64_t* __restrict__ C, int64_t N,
                                                               int level, int levels, int64_t chunk,
                                                               PeerPtrs dst, int src) {
    const int64_t X = blockIdx.x;
    const int64_t R = tri_row_start(X, N);
    const int64_t* row = C + (size_t)X * (size_t)N + X - R;
    const int64_t hi = R + (N - X);
    for (int64_t e = R + threadIdx.x; e < hi; e += blockDim.x) {
        const int64_t d = e / chunk;
        GK_CHECK(d < MAX_PEERS && dst.p[d] != nullptr);
        T* out = (T*)dst.p[d];
        out[((int64_t)src * levels + level) * chunk + (e - d * chunk)] = (T)row[e];
    }
}

cudaError_t launch_pack_upper_peers(const int64_t* C, int64_t N, int level, int levels,
                                    int64_t chunk, const PeerPtrs& dst, int src, int out_bytes,
                                    cudaStream_t s) {
    if (N <= 0) return cudaGetLastError();
    if (out_bytes == 8)
        pack_upper_peers_kernel<int64_t><<<(unsigned)N, 256, 0, s>>>(C, N, level, levels, chunk, dst, src);
    else
        pack_upper_peers_kernel<uint32_t><<<(unsigned)N, 256, 0, s>>>(C, N, level, levels, chunk, dst, src);
    return cudaGetLastError();
}

cudaError_t launch_pack_upper(const int64_t* C, int64_t N, int levels, int64_t begin, int64_t end,
                              void* out, int out_bytes, cudaStream_t s) {
    if (end <= begin || levels <= 0) return cudaGetLastError();
    const int64_t X0 = tri_row_of(begin, N), X1 = tri_row_of(end - 1, N);
    const dim3 grid((unsigned)(X1 - X0 + 1), (unsigned)levels);
    if (out_bytes == 8)
        pack_upper_kernel<int64_t><<<grid, 256, 0, s>>>(C, N, begin, end, X0, (int64_t*)out);
    else
        pack_upper_kernel<uint32_t><<<grid, 256, 0, s>>>(C, N, begin, end, X0, (uint32_t*)out);
    return cudaGetLastError();
}

cudaError_t launch_diag(const int64_t* C, int64_t N, int levels, int64_t* out, int sm_count,
                        cudaStream_t s) {
    const int64_t tot = (int64_t)levels * N;
    if (tot <= 0) return cudaGetLastError();
    const int64_t blocks = std::min<int64_t>((tot + 255) / 256, (int64_t)sm_count * 4);
    diag_kernel<<<(unsigned)blocks, 256, 0, s>>>(C, N, levels, out);
    return cudaGetLastError();
}

}  // namespace gk
