// epilogue.cu — inclusion-exclusion, weighting and normalisation.
//
//   N_m = C_m - sum_{j<m} C(g-j, m-j) N_j        Eq. 9, PAPER.md:136 (Algorithm 1
//                                                lines 18-21)
//   K   = sum_{m<=min(M,g-k)} h_m N_m,
//         h_m = C(g-m,k) if g-m >= k else 0       Eq. 6-7, P:94-100 (Alg. 1 l.5-7)
//   Knorm(X,Y) = K(X,Y) / sqrt(K(X,X) K(Y,Y))    BASELINE.json (reading A5)
//
// Input: C with a valid upper triangle. Output: C mirrored to full symmetric, and
// full symmetric Nm, K, Knorm. One CTA per 32x32 tile pair (bi <= bj): the upper
// tile is read once, its results written to (bi,bj) directly and to (bj,bi)
// through a shared-memory transpose so both writes are coalesced.
// Invariant checks: N_m >= 0, K == C_{g-k} when M >= g-k.
#include <math.h>
#include <string.h>

#include <type_traits>

#include "internal.cuh"

namespace gk {

// Coefficients, computed on the host (launch_epilogue) and passed by value:
//   e9[m][j] = C(g-j, m-j)  (Eq. 9 recursion, j < m)
//   h[m]     = C(g-m, k) for m <= min(M, g-k), else 0  (Eq. 6-7)
struct EpiCoef {
    int64_t e9[GMAX + 1][GMAX + 1];
    int64_t h[GMAX + 1];
};

struct EpiArgs {
    int64_t* C;
    int64_t N;
    int g, k, M;
    int64_t* Nm;
    int64_t* K;
    double* Knorm;
    int64_t* kdiag;
    int* flags;
};

// Per-entry math. prof[m] = C_m(X,Y) in, N_m(X,Y) out. Returns K(X,Y).
// Loops run to the compile-time bound MM (guarded by M) so prof stays in registers.
template <int MM>
__device__ __forceinline__ int64_t entry(int64_t (&prof)[MM + 1], const EpiCoef& cf, int g, int k,
                                         int M, int* bad) {
    int64_t cgk = 0;
#pragma unroll
    // (selected by a mask: `if (m == g - k) cgk = prof[m]` compiled to prof[g - k], a
    // dynamic index that put the whole profile array in local memory -- ncu: 16 GB of
    // local stores per Scale epilogue)
    for (int m = 0; m <= MM; ++m) cgk |= prof[m] & -(int64_t)(m <= M && m == g - k);
#pragma unroll
    for (int m = 0; m <= MM; ++m) {
        if (m > M) break;
        int64_t v = prof[m];
#pragma unroll
        for (int j = 0; j < m; ++j) v -= cf.e9[m][j] * prof[j];  // prof[j] is N_j now
        if (v < 0) *bad |= EF_NEGATIVE_N;
        prof[m] = v;
    }
    int64_t K = 0;
#pragma unroll
    for (int m = 0; m <= MM; ++m)
        if (m <= M) K += cf.h[m] * prof[m];
    if (M >= g - k && K != cgk) *bad |= EF_K_MISMATCH;
    return K;
}

__global__ void kdiag_kernel(EpiArgs a, const __grid_constant__ EpiCoef cf) {
    const int64_t nn = a.N * a.N;
    int bad = 0;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < a.N;
         x += (int64_t)gridDim.x * blockDim.x) {
        int64_t prof[GMAX + 1];
        for (int m = 0; m <= a.M; ++m) prof[m] = a.C[m * nn + x * a.N + x];
        a.kdiag[x] = entry<GMAX>(prof, cf, a.g, a.k, a.M, &bad);
    }
    if (bad) atomicOr(a.flags, bad);
}

__device__ __forceinline__ double knorm(int64_t kxy, int64_t kxx, int64_t kyy, bool diag) {
    if (kxx <= 0 || kyy <= 0) return 0.0;
    if (diag) return 1.0;
    return __ddiv_rn((double)kxy, __dsqrt_rn(__dmul_rn((double)kxx, (double)kyy)));
}

// blockDim (32, 32 / EP_RPT); a 1-D grid over the t(t+1)/2 tile pairs bi <= bj (t =
// tiles per side), row-major: block L -> the largest bi with R(bi) = bi t - bi (bi-1)/2
// <= L. Each thread holds EP_RPT rows of the 32 x 32 tile; MINB CTAs per SM the
// register budget is sized for. MM bounds M.
template <int MM, int EP_RPT, int MINB>
__global__ void __launch_bounds__(32 * (32 / EP_RPT), MINB) epilogue_kernel(
    EpiArgs a, const __grid_constant__ EpiCoef cf) {
    constexpr int EP_TY = 32 / EP_RPT;
    __shared__ int64_t st[32][33];
    const int64_t t = (a.N + 31) / 32, L = blockIdx.x;
    int64_t lo = 0, hi = t - 1;
    while (lo < hi) {  // (block-uniform)
        const int64_t mid = (lo + hi + 1) / 2;
        if (mid * t - mid * (mid - 1) / 2 <= L) lo = mid;
        else hi = mid - 1;
    }
    const int bi = (int)lo, bj = (int)(lo + (L - (lo * t - lo * (lo - 1) / 2)));
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t N = a.N, nn = N * N;
    const int M = a.M;
    const bool diag_tile = bi == bj;
    int64_t prof[EP_RPT][MM + 1];
    int64_t kv[EP_RPT];
    double kn[EP_RPT];
    bool ok[EP_RPT];
    int bad = 0;
#pragma unroll
    for (int q = 0; q < EP_RPT; ++q) {
        const int r = ty + EP_TY * q;
        const int64_t X = (int64_t)bi * 32 + r, Y = (int64_t)bj * 32 + tx;
        ok[q] = X < N && Y < N;
        kv[q] = 0;
        if (!ok[q]) continue;
        const int64_t src = (diag_tile && r > tx) ? (Y * N + X) : (X * N + Y);  // upper entry
#pragma unroll
        for (int m = 0; m <= MM; ++m)
            if (m <= M) prof[q][m] = a.C[m * nn + src];
        if (diag_tile && r > tx) {  // mirror C into the lower half of a diagonal tile
#pragma unroll
            for (int m = 0; m <= MM; ++m)
                if (m <= M) a.C[m * nn + X * N + Y] = prof[q][m];
        }
    }
    // off-diagonal tile: C mirrored into tile (bj, bi) while prof still holds C
    // (transposed through shared memory: coalesced rows on both sides)
    if (!diag_tile) {
#pragma unroll
        for (int o = 0; o <= MM; ++o) {  // static indices keep prof in registers
            if (o > M) break;
            __syncthreads();
#pragma unroll
            for (int q = 0; q < EP_RPT; ++q) st[ty + EP_TY * q][tx] = prof[q][o];
            __syncthreads();
#pragma unroll
            for (int q = 0; q < EP_RPT; ++q) {
                const int r = ty + EP_TY * q;
                const int64_t X = (int64_t)bj * 32 + r, Y = (int64_t)bi * 32 + tx;
                if (X < N && Y < N) a.C[o * nn + X * N + Y] = st[tx][r];
            }
        }
    }
#pragma unroll
    for (int q = 0; q < EP_RPT; ++q) {
        if (!ok[q]) continue;
        const int r = ty + EP_TY * q;
        const int64_t X = (int64_t)bi * 32 + r, Y = (int64_t)bj * 32 + tx;
        kv[q] = entry<MM>(prof[q], cf, a.g, a.k, M, &bad);  // prof now holds N_m
        kn[q] = knorm(kv[q], a.kdiag[X], a.kdiag[Y], X == Y);  // (reused transposed)
        if (a.Nm) {
#pragma unroll
            for (int m = 0; m <= MM; ++m)
                if (m <= M) a.Nm[m * nn + X * N + Y] = prof[q][m];
        }
        if (a.K) a.K[X * N + Y] = kv[q];
        if (a.Knorm) a.Knorm[X * N + Y] = kn[q];
    }
    if (bad) atomicOr(a.flags, bad);
    if (diag_tile) return;
    // transposed writes of tile (bj, bi): K and Knorm (their registers die first), then
    // Nm (static level index, prof stays in registers; the C mirror went out above)
    for (int o = 0; o < 2; ++o) {
        if (o == 0 ? a.K == nullptr : a.Knorm == nullptr) continue;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < EP_RPT; ++q) {
            const int r = ty + EP_TY * q;
            if (!ok[q]) continue;
            st[r][tx] = o == 0 ? kv[q] : __double_as_longlong(kn[q]);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < EP_RPT; ++q) {
            const int r = ty + EP_TY * q;                  // row within the transposed tile
            const int64_t X = (int64_t)bj * 32 + r, Y = (int64_t)bi * 32 + tx;
            if (X >= N || Y >= N) continue;
            const int64_t v = st[tx][r];
            if (o == 0) a.K[X * N + Y] = v;
            else a.Knorm[X * N + Y] = __longlong_as_double(v);
        }
    }
    if (a.Nm) {
#pragma unroll
        for (int o = 0; o <= MM; ++o) {
            if (o > M) break;
            __syncthreads();
#pragma unroll
            for (int q = 0; q < EP_RPT; ++q) st[ty + EP_TY * q][tx] = prof[q][o];
            __syncthreads();
#pragma unroll
            for (int q = 0; q < EP_RPT; ++q) {
                const int r = ty + EP_TY * q;
                const int64_t X = (int64_t)bj * 32 + r, Y = (int64_t)bi * 32 + tx;
                if (X < N && Y < N) a.Nm[o * nn + X * N + Y] = st[tx][r];
            }
        }
    }
}

// ---------------------------------------------------------------- rectangular
// Train x test block: rows X < NA (train), columns Y = NA + j
// (test). C is [M+1][NA][NB] (every entry accumulated), Dg [M+1][N] the diagonals
// C_m(X,X) of all N sequences; kdiag[X] = K(X,X) for all N (normalisation).
__global__ void kdiag_rect_kernel(const int64_t* __restrict__ Dg, int64_t N, int g, int k, int M,
                                  int64_t* kdiag, int* flags, const __grid_constant__ EpiCoef cf) {
    int bad = 0;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
         x += (int64_t)gridDim.x * blockDim.x) {
        int64_t prof[GMAX + 1];
        for (int m = 0; m <= M; ++m) prof[m] = Dg[m * N + x];
        kdiag[x] = entry<GMAX>(prof, cf, g, k, M, &bad);
    }
    if (bad) atomicOr(flags, bad);
}

template <int MM>
__global__ void __launch_bounds__(256) epilogue_rect_kernel(
    const int64_t* __restrict__ C, int64_t NA, int64_t NB, int g, int k, int M, int64_t* Nm,
    int64_t* K, double* Knorm, const int64_t* __restrict__ kdiag, int* flags,
    const __grid_constant__ EpiCoef cf) {
    const int64_t cells = NA * NB;
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t prof[MM + 1];
#pragma unroll
        for (int m = 0; m <= MM; ++m)
            if (m <= M) prof[m] = C[m * cells + i];
        const int64_t kv = entry<MM>(prof, cf, g, k, M, &bad);
        if (Nm) {
#pragma unroll
            for (int m = 0; m <= MM; ++m)
                if (m <= M) Nm[m * cells + i] = prof[m];
        }
        if (K) K[i] = kv;
        if (Knorm) {
            const int64_t x = i / NB, y = NA + (i - x * NB);
            Knorm[i] = knorm(kv, kdiag[x], kdiag[y], false);
        }
    }
    if (bad) atomicOr(flags, bad);
}

static EpiCoef make_coef(int g, int k, int M) {
    EpiCoef cf;
    memset(&cf, 0, sizeof cf);
    int64_t bt[GMAX + 1][GMAX + 1];  // Pascal's triangle
    for (int n = 0; n <= GMAX; ++n)
        for (int r = 0; r <= GMAX; ++r)
            bt[n][r] = (r == 0) ? 1 : (r > n ? 0 : (r == n ? 1 : bt[n - 1][r - 1] + bt[n - 1][r]));
    for (int m = 0; m <= M && m <= GMAX; ++m) {
        for (int j = 0; j < m; ++j) cf.e9[m][j] = bt[g - j][m - j];
        cf.h[m] = (m <= g - k) ? bt[g - m][k] : 0;
    }
    return cf;
}

cudaError_t launch_epilogue_rect(const int64_t* C, const int64_t* Dg, int64_t N, int64_t NA, int g,
                                 int k, int M, int64_t* Nm, int64_t* K, double* Knorm,
                                 int64_t* kdiag, int* flags, int sm_count, cudaStream_t s) {
    const EpiCoef cf = make_coef(g, k, M);
    int64_t blocks = (N + 255) / 256;
    kdiag_rect_kernel<<<(int)(blocks < 1024 ? blocks : 1024), 256, 0, s>>>(Dg, N, g, k, M, kdiag,
                                                                         flags, cf);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t NB = N - NA;
    if (NA * NB == 0) return cudaGetLastError();
    const int grid = sm_count * 8;
    if (M <= 7)
        epilogue_rect_kernel<7><<<grid, 256, 0, s>>>(C, NA, NB, g, k, M, Nm, K, Knorm, kdiag,
                                                     flags, cf);
    else
        epilogue_rect_kernel<GMAX><<<grid, 256, 0, s>>>(C, NA, NB, g, k, M, Nm, K, Knorm, kdiag,
                                                        flags, cf);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- packed slice
// Mask-sharded step: after the reduce-scatter every rank holds the
// complete C_m of a range [begin, begin + cnt) of the packed upper triangle
// (e(X, Y) = X N - X (X - 1) / 2 + (Y - X)), as int64 or u32 words (the host uses
// u32 when C(g,m) n_max^2 < 2^31), level m at Cp + m ld. The same per-entry Eq. 9 / Eq. 7 / Knorm as
// epilogue_kernel, written to packed outputs of the same range. kdiag holds K(X,X)
// of all N sequences (from the all-reduced diagonals, kdiag_rect_kernel).
// One CTA per row X0 + blockIdx.x.
template <int MM, typename T>
__global__ void __launch_bounds__(256) epilogue_packed_kernel(
    const T* __restrict__ Cp, int nsrc, int64_t ld, int64_t N, int64_t begin, int64_t cnt,
    int64_t X0, int g, int k, int M, int64_t* Nm, int64_t* K, double* Knorm,
    const int64_t* __restrict__ kdiag, int* flags, const __grid_constant__ EpiCoef cf) {
    const int64_t X = X0 + blockIdx.x;
    const int64_t R = X * N - X * (X - 1) / 2;
    const int64_t lo = max(R, begin), hi = min(R + (N - X), begin + cnt);
    const int64_t kx = kdiag[X];
    int bad = 0;
    for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
        const int64_t i = e - begin, Y = X + (e - R);
        int64_t prof[MM + 1];
#pragma unroll
        for (int m = 0; m <= MM; ++m)
            if (m <= M) {  // (nsrc > 1: the ranks' contributions, summed here)
                int64_t v = 0;
                for (int q = 0; q < nsrc; ++q) v += (int64_t)Cp[((size_t)q * (M + 1) + m) * ld + i];
                prof[m] = v;
            }
        const int64_t kv = entry<MM>(prof, cf, g, k, M, &bad);
        if (Nm) {
#pragma unroll
            for (int m = 0; m <= MM; ++m)
                if (m <= M) Nm[(size_t)m * ld + i] = prof[m];
        }
        if (K) K[i] = kv;
        if (Knorm) Knorm[i] = knorm(kv, kx, kdiag[Y], X == Y);
    }
    if (bad) atomicOr(flags, bad);
}

int64_t tri_row_of(int64_t e, int64_t N);  // shard.cu

template <typename T>
static void epi_packed(const T* Cp, int nsrc, int64_t ld, int64_t N, int64_t begin, int64_t cnt, int64_t X0,
                       unsigned rows, int g, int k, int M, int64_t* Nm, int64_t* K, double* Knorm,
                       const int64_t* kdiag, int* flags, const EpiCoef& cf, cudaStream_t s) {
    if (M <= 3)
        epilogue_packed_kernel<3, T><<<rows, 256, 0, s>>>(Cp, nsrc, ld, N, begin, cnt, X0, g, k, M, Nm, K,
                                                          Knorm, kdiag, flags, cf);
    else if (M <= 5)
        epilogue_packed_kernel<5, T><<<rows, 256, 0, s>>>(Cp, nsrc, ld, N, begin, cnt, X0, g, k, M, Nm, K,
                                                          Knorm, kdiag, flags, cf);
    else if (M <= 7)
        epilogue_packed_kernel<7, T><<<rows, 256, 0, s>>>(Cp, nsrc, ld, N, begin, cnt, X0, g, k, M, Nm, K,
                                                          Knorm, kdiag, flags, cf);
    else
        epilogue_packed_kernel<GMAX, T><<<rows, 256, 0, s>>>(Cp, nsrc, ld, N, begin, cnt, X0, g, k, M, Nm,
                                                             K, Knorm, kdiag, flags, cf);
}

cudaError_t launch_epilogue_packed(const void* Cp, int in_bytes, int nsrc, int64_t ld, const int64_t* Dg, int64_t N,
                                   int64_t begin, int64_t end, int g, int k, int M, int64_t* Nm,
                                   int64_t* K, double* Knorm, int64_t* kdiag, int* flags,
                                   cudaStream_t s) {
    const EpiCoef cf = make_coef(g, k, M);
    int64_t blocks = (N + 255) / 256;
    kdiag_rect_kernel<<<(int)(blocks < 1024 ? blocks : 1024), 256, 0, s>>>(Dg, N, g, k, M, kdiag,
                                                                         flags, cf);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || end <= begin) return e;
    const int64_t X0 = tri_row_of(begin, N), X1 = tri_row_of(end - 1, N);
    const unsigned rows = (unsigned)(X1 - X0 + 1);
    if (in_bytes == 8)
        epi_packed<int64_t>((const int64_t*)Cp, nsrc, ld, N, begin, end - begin, X0, rows, g, k, M, Nm, K,
                            Knorm, kdiag, flags, cf, s);
    else
        epi_packed<uint32_t>((const uint32_t*)Cp, nsrc, ld, N, begin, end - begin, X0, rows, g, k, M, Nm, K,
                             Knorm, kdiag, flags, cf, s);
    return cudaGetLastError();
}

cudaError_t launch_epilogue(int64_t* C, int64_t N, int g, int k, int M, int64_t* Nm, int64_t* K,
                            double* Knorm, int64_t* kdiag, int* flags, cudaStream_t s) {
    EpiArgs a{C, N, g, k, M, Nm, K, Knorm, kdiag, flags};
    const EpiCoef cf = make_coef(g, k, M);
    int64_t blocks = (N + 255) / 256;
    kdiag_kernel<<<(int)(blocks < 1024 ? blocks : 1024), 256, 0, s>>>(a, cf);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const uint64_t tiles = (uint64_t)((N + 31) / 32);
    const unsigned pairs = (unsigned)(tiles * (tiles + 1) / 2);  // (upper tile pairs only)
    // (2 rows per thread, 2 x 512 threads per SM, 64 registers: 9.4 ms at Scale; the
    // spill-free 1 x 512 (96 registers) and 1 row x 1024 threads took 11.5 / 12.3 ms)
    auto go = [&](auto mm) {
        constexpr int MM = decltype(mm)::value;
        epilogue_kernel<MM, 2, 2><<<pairs, dim3(32, 16), 0, s>>>(a, cf);
    };
    // (the profile array sized to the level count: registers, not local memory)
    if (M <= 3) go(std::integral_constant<int, 3>());
    else if (M <= 5) go(std::integral_constant<int, 5>());
    else if (M <= 7) go(std::integral_constant<int, 7>());
    else go(std::integral_constant<int, GMAX>());
    return cudaGetLastError();
}

}  // namespace gk
