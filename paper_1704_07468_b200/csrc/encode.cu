// encode.cu — g-mer bookkeeping and the mask-encode kernel (removePosition).
//
// Algorithm 1 line 13, L^i <- removePosition(L, i) (§2.2 step 3,
// P:127): for mask i (a set of m removed positions) every g-mer becomes the
// (g-m)-mer of its kept positions. Here that (g-m)-mer is written as one
// mixed-radix integer, first kept position most significant,
//     key = sum_r code[pos + p_r] * sigma^(g-m-1-r),
// and packed with its sequence id as  composite = key << sb | seq  (sb bits hold
// the id). Equal keys <=> equal (g-m)-mers, so grouping composites by their key
// bits groups the paper's matching (g-m)-mers. The g-mer list L of Algorithm 1
// is never materialised: keys are produced straight from the corpus.
//
// The same pass counts the 8-bit digit histograms of every LSD pass the sort
// will run (the "upfront histogram" of a onesweep radix sort).
#include "internal.cuh"

namespace gk {

// gm_seq[j] = X for every g-mer j of sequence X (g-mer j of X is gofs[X] + i).
__global__ void gmer_index_kernel(const int64_t* __restrict__ gofs, int64_t N,
                                  uint32_t* __restrict__ gm_seq) {
    for (int64_t x = blockIdx.x; x < N; x += gridDim.x) {
        int64_t a = gofs[x], b = gofs[x + 1];
        for (int64_t j = a + threadIdx.x; j < b; j += blockDim.x) gm_seq[j] = (uint32_t)x;
    }
}

cudaError_t launch_gmer_index(const int64_t* gofs, int64_t N, uint32_t* gm_seq, cudaStream_t s) {
    int grid = (int)(N < 65535 ? N : 65535);
    if (grid > 0) gmer_index_kernel<<<grid, 128, 0, s>>>(gofs, N, gm_seq);
    return cudaGetLastError();
}

__global__ void check_codes_kernel(const uint8_t* __restrict__ codes, int64_t len, int sigma,
                                   int* flags) {
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= codes[i] >= sigma;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, EF_BAD_SYMBOL);
}

// symbol histogram (hist[256], zeroed by the caller), for the per-level choice of
// the Gram operand format in plan.cu (the most frequent symbol bounds how often one
// masked key repeats inside a sequence)
__global__ void symbol_hist_kernel(const uint8_t* __restrict__ codes, int64_t len,
                                   unsigned long long* __restrict__ hist) {
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&h[codes[i]], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], (unsigned long long)h[i]);
}

cudaError_t launch_symbol_hist(const uint8_t* codes, int64_t len, unsigned long long* hist,
                               int sm_count, cudaStream_t s) {
    if (len > 0) {
        int64_t blocks = (len + 1023) / 1024;
        const int64_t cap = (int64_t)sm_count * 4;
        symbol_hist_kernel<<<(int)(blocks < cap ? blocks : cap), 256, 0, s>>>(codes, len, hist);
    }
    return cudaGetLastError();
}

cudaError_t launch_check_codes(const uint8_t* codes, int64_t len, int sigma, int* flags,
                               cudaStream_t s) {
    if (len > 0) {
        int64_t blocks = (len + 255) / 256;
        check_codes_kernel<<<(int)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(codes, len, sigma,
                                                                                 flags);
    }
    return cudaGetLastError();
}

// grid.y = mask within the batch; grid.x strides over g-mers.
// kept[b*GMAX + r] = r-th kept position of mask b (ascending).
// K = uint32_t when the composite fits 32 bits (half the key traffic downstream).
template <typename K>
__global__ void __launch_bounds__(256) encode_kernel(CorpusView cv, const uint8_t* __restrict__ kept,
                                                     int nkept, int sigma, int sb, int npass,
                                                     K* __restrict__ out,
                                                     uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[MAXPASS][RADIX];
    __shared__ uint8_t sk[GMAX];
    const int b = blockIdx.y;
    for (int i = threadIdx.x; i < MAXPASS * RADIX; i += blockDim.x) (&sh[0][0])[i] = 0;
    if (threadIdx.x < GMAX) sk[threadIdx.x] = kept[b * GMAX + threadIdx.x];
    __syncthreads();
    const uint64_t n = cv.n;
    K* o = out + (uint64_t)b * n;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = cv.gm_seq[j];
        const uint8_t* p = cv.codes + cv.off[x] + ((int64_t)j - cv.gofs[x]);
        uint64_t key = 0;
        for (int r = 0; r < nkept; ++r) key = key * (uint64_t)sigma + p[sk[r]];
        const uint64_t comp = (key << sb) | x;
        o[j] = (K)comp;
        for (int q = 0; q < npass; ++q) atomicAdd(&sh[q][(comp >> (sb + RADIX_BITS * q)) & 0xff], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * RADIX; i += blockDim.x) {
        uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(&hist[(b * npass) * RADIX + i], v);
    }
}

// Encode from packed g-mer windows (bucket.cu's window_kernel: the g codes of
// g-mer j as bits-wide fields of win[j], first position most significant): the
// same mixed-radix key, symbols extracted with shifts instead of byte loads, and
// EM masks per CTA share each thread's window and sequence-id loads.
// grid: (g-mer tiles, ceil(nmask / EM)); kept_sh[b*GMAX + r] = bits*(g-1-kept_r).
constexpr int EW_THREADS = 256;
constexpr int EW_ITEMS = 8;
constexpr int EW_MASKS = 8;
template <typename K>
__global__ void __launch_bounds__(EW_THREADS) encode_win_kernel(
    const uint64_t* __restrict__ win, const uint32_t* __restrict__ gm_seq, uint64_t n,
    const uint8_t* __restrict__ kept_sh, int nkept, uint32_t sigma, int bits, int sb, int nmask,
    K* __restrict__ out) {
    __shared__ uint8_t sh[EW_MASKS][GMAX];
    const int b0 = blockIdx.y * EW_MASKS;
    const int nm = min(EW_MASKS, nmask - b0);
    for (int i = threadIdx.x; i < nm * GMAX; i += EW_THREADS)
        sh[i / GMAX][i % GMAX] = kept_sh[(b0 + i / GMAX) * GMAX + i % GMAX];
    __syncthreads();
    const uint64_t symmask = (1ull << bits) - 1ull;
    const uint64_t j0 = (uint64_t)blockIdx.x * EW_THREADS * EW_ITEMS + threadIdx.x;
    uint64_t w[EW_ITEMS];
    uint32_t x[EW_ITEMS];
#pragma unroll
    for (int i = 0; i < EW_ITEMS; ++i) {
        const uint64_t j = j0 + (uint64_t)i * EW_THREADS;
        w[i] = j < n ? win[j] : 0ull;
        x[i] = j < n ? gm_seq[j] : 0u;
    }
    for (int mm = 0; mm < nm; ++mm) {
        K* o = out + (uint64_t)(b0 + mm) * n;
#pragma unroll
        for (int i = 0; i < EW_ITEMS; ++i) {
            const uint64_t j = j0 + (uint64_t)i * EW_THREADS;
            if (j >= n) continue;
            uint64_t key = 0;
            for (int r = 0; r < nkept; ++r) key = key * sigma + ((w[i] >> sh[mm][r]) & symmask);
            o[j] = (K)((key << sb) | x[i]);
        }
    }
}

cudaError_t launch_encode_win(const uint64_t* win, const uint32_t* gm_seq, uint64_t n,
                              const uint8_t* kept_sh, int nkept, int sigma, int bits, int sb,
                              int nmask, void* out, bool k64, cudaStream_t s) {
    if (n == 0 || nmask == 0) return cudaGetLastError();
    dim3 grid((unsigned)((n + EW_THREADS * EW_ITEMS - 1) / (EW_THREADS * EW_ITEMS)),
              (unsigned)((nmask + EW_MASKS - 1) / EW_MASKS));
    if (k64)
        encode_win_kernel<uint64_t><<<grid, EW_THREADS, 0, s>>>(win, gm_seq, n, kept_sh, nkept,
                                                                (uint32_t)sigma, bits, sb, nmask,
                                                                (uint64_t*)out);
    else
        encode_win_kernel<uint32_t><<<grid, EW_THREADS, 0, s>>>(win, gm_seq, n, kept_sh, nkept,
                                                                (uint32_t)sigma, bits, sb, nmask,
                                                                (uint32_t*)out);
    return cudaGetLastError();
}

cudaError_t launch_encode(const CorpusView& cv, const uint8_t* kept, int nkept, int sigma, int sb,
                          int nmask, int npass, void* out, bool k64, uint32_t* hist,
                          cudaStream_t s) {
    if (cv.n == 0 || nmask == 0) return cudaGetLastError();
    uint64_t blocks = (cv.n + 256 * 8 - 1) / (256 * 8);
    if (blocks > 1024) blocks = 1024;
    dim3 grid((unsigned)blocks, (unsigned)nmask);
    if (k64)
        encode_kernel<uint64_t><<<grid, 256, 0, s>>>(cv, kept, nkept, sigma, sb, npass,
                                                     (uint64_t*)out, hist);
    else
        encode_kernel<uint32_t><<<grid, 256, 0, s>>>(cv, kept, nkept, sigma, sb, npass,
                                                     (uint32_t*)out, hist);
    return cudaGetLastError();
}

}  // namespace gk
