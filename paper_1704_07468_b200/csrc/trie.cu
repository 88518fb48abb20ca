// trie.cu — one stable pass of the mask trie over (packed window, sequence id)
// elements, specialised for symbol digits (Σ <= 64: at most 64 buckets).
//
// Algorithm 1 line 14, L^i <- sort(L^i), done as LSD passes over
// the kept positions of a mask (DESIGN.md §8 "Mask trie"): a pass is a stable
// counting sort by the symbol at ONE kept position, digit = (w >> shift) & dmask.
// Two launches per pass instead of the generic radix path's three:
//   tp_hist:    CTA c counts the digits of its chunk (per-warp shared counters,
//               1024 threads); with Hg it also adds its counts into the sum of its
//               block of 8 chunks (Hg, double-buffered by pass parity: the pass
//               zeroes the other parity's sums for the next pass);
//   tp_scatter: CTA c computes its chunk prefix and the digit bases itself from the
//               block sums and its block's chunk rows (<= 6 loads per thread, one
//               round trip; without Hg: from every chunk row), then streams its
//               chunk in 4096-element tiles (cp.async.bulk into shared memory, one
//               tile ahead), ranks each tile stably (warp atomicOr match + per-warp
//               digit counters; only digits and ranks stay in registers), records the
//               tile's stable order as a 16-bit source-index permutation and writes
//               every digit run contiguously, reading the elements through it.
// 512 threads x 8 elements per tile (16 warps) keep the registers at <= 64 without
// spills so two CTAs (1024 threads) fit an SM next to their ~90 KB of shared memory.
//
// The element count may live on the device (cntp != nullptr: a compacted parent
// array of the cross-level chain, plan.cu); the grid is sized for the capacity n
// and both kernels derive the same chunking from the actual count.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace gk {

namespace {

constexpr int TP_THREADS = 512;
constexpr int TP_WARPS = TP_THREADS / 32;
constexpr int TP_ITEMS = 8;
constexpr int TP_TILE = TP_THREADS * TP_ITEMS;  // 4096
constexpr int TP_ND = 64;                       // digit buckets (symbols < 64)

__device__ __forceinline__ void tp_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// bytes of the 16-byte aligned window covering elements [g0, g0 + cnt) of `in`
template <typename T>
__device__ __forceinline__ uint32_t tp_span(const T* in, uint64_t g0, uint32_t cnt) {
    const uintptr_t a0 = (uintptr_t)(in + g0), a1 = (uintptr_t)(in + g0 + cnt);
    return (uint32_t)(((a1 + 15) & ~(uintptr_t)15) - (a0 & ~(uintptr_t)15));
}
template <typename T>
__device__ __forceinline__ const void* tp_base(const T* in, uint64_t g0) {
    return (const void*)((uintptr_t)(in + g0) & ~(uintptr_t)15);
}
template <typename T>
__device__ __forceinline__ uint32_t tp_delta(const T* in, uint64_t g0) {
    return (uint32_t)(((uintptr_t)(in + g0) & 15) / sizeof(T));
}

// chunking shared by both kernels: cps chunks of L elements (whole tiles)
struct TpChunk {
    uint64_t lo, hi;
};
__device__ __forceinline__ TpChunk tp_chunk(uint64_t cnt, uint32_t cps, uint32_t c) {
    const uint64_t tiles = (cnt + TP_TILE - 1) / TP_TILE;
    const uint64_t L = (tiles + cps - 1) / cps * TP_TILE;
    const uint64_t lo = min(cnt, (uint64_t)c * L);
    return {lo, min(cnt, lo + L)};
}

constexpr int TPH_THREADS = 1024;
constexpr int TPH_WARPS = TPH_THREADS / 32;
constexpr int TP_HG_BLOCK = 8;  // chunks per block sum

template <typename K>
__global__ void __launch_bounds__(TPH_THREADS) tp_hist_kernel(const K* __restrict__ w,
                                                              uint64_t n, const uint32_t* cntp,
                                                              int shift, uint32_t dmask,
                                                              uint32_t* __restrict__ H,
                                                              uint32_t* __restrict__ Hg, int par) {
    constexpr int E = 16 / sizeof(K);  // keys per 16-byte load
    __shared__ uint32_t s_h[TPH_WARPS][TP_ND];
    pdl_wait();
    const int tid = threadIdx.x, wp = tid >> 5;
    for (int i = tid; i < TPH_WARPS * TP_ND; i += TPH_THREADS) (&s_h[0][0])[i] = 0;
    if (Hg) {  // the other parity's block sums, zeroed for the next pass
        uint32_t* z = Hg + (size_t)(par ^ 1) * TP_HG_MAX_BLOCKS * TP_ND;
        const uint32_t nz = (gridDim.x + TP_HG_BLOCK - 1) / TP_HG_BLOCK * TP_ND;
        for (uint32_t i = blockIdx.x * TPH_THREADS + tid; i < nz; i += gridDim.x * TPH_THREADS) z[i] = 0u;
    }
    __syncthreads();
    const uint64_t cnt = cntp ? min((uint64_t)*cntp, n) : n;
    const TpChunk ch = tp_chunk(cnt, gridDim.x, blockIdx.x);
    uint64_t a = ch.lo;
    while (a < ch.hi && ((uintptr_t)(w + a) & 15)) {  // (16-byte loads on the aligned body)
        if (tid == 0) atomicAdd(&s_h[0][(uint32_t)(w[a] >> shift) & dmask], 1u);
        ++a;
    }
    const uint64_t nv = a < ch.hi ? (ch.hi - a) / E : 0;
    const uint4* v = (const uint4*)(w + a);
    uint64_t i = tid;
    for (; i + 3 * TPH_THREADS < nv; i += 4 * TPH_THREADS) {  // (4 loads in flight)
        uint4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = v[i + u * TPH_THREADS];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const K* kq = (const K*)&q[u];
#pragma unroll
            for (int e = 0; e < E; ++e) atomicAdd(&s_h[wp][(uint32_t)(kq[e] >> shift) & dmask], 1u);
        }
    }
    for (; i < nv; i += TPH_THREADS) {
        const uint4 q = v[i];
        const K* kq = (const K*)&q;
#pragma unroll
        for (int e = 0; e < E; ++e) atomicAdd(&s_h[wp][(uint32_t)(kq[e] >> shift) & dmask], 1u);
    }
    for (uint64_t r = a + nv * E + tid; r < ch.hi; r += TPH_THREADS)
        atomicAdd(&s_h[wp][(uint32_t)(w[r] >> shift) & dmask], 1u);
    pdl_trigger();
    __syncthreads();
    if (tid < TP_ND) {
        uint32_t s = 0;
#pragma unroll
        for (int ww = 0; ww < TPH_WARPS; ++ww) s += s_h[ww][tid];
        H[(uint64_t)blockIdx.x * TP_ND + tid] = s;
        if (Hg && s)
            atomicAdd(&Hg[((size_t)par * TP_HG_MAX_BLOCKS + blockIdx.x / TP_HG_BLOCK) * TP_ND + tid], s);
    }
}

// exclusive scan of v over the 64 threads tid < 64 (two warps); s2: 2 words
__device__ __forceinline__ uint32_t tp_scan64(uint32_t v, uint32_t* s2) {
    const int tid = threadIdx.x, lane = tid & 31;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (tid == 31) s2[0] = inc;
    __syncthreads();
    return inc - v + (tid >= 32 && tid < 64 ? s2[0] : 0u);
}

// payload-less passes (far-pair records): S = TpNoPay
struct TpNoPay {};
template <typename S>
__host__ __device__ constexpr bool tp_pay() {
    return !std::is_same<S, TpNoPay>::value;
}
template <typename S>
__host__ __device__ constexpr uint32_t tp_psz() {
    return tp_pay<S>() ? (uint32_t)sizeof(S) : 0u;
}

template <typename K, typename S>
constexpr size_t tp_smem() {
    return 2 * (TP_TILE * sizeof(K) + 32) + (tp_pay<S>() ? 2 * (TP_TILE * tp_psz<S>() + 32) : 0) +
           TP_TILE * 2 + 2 * TP_ND * 8 + 2 * TP_WARPS * TP_ND * 4 + 2 * 8 * TP_ND * 4 + TP_ND * 4 + 16 + 2 * 8 + 8;
}

template <typename K, typename S>
__global__ void __launch_bounds__(TP_THREADS, 2) tp_scatter_kernel(
    const K* __restrict__ win, K* __restrict__ wout, const S* __restrict__ sin,
    S* __restrict__ sout, uint64_t n, const uint32_t* cntp, int shift, uint32_t dmask,
    K omask, const uint32_t* __restrict__ H, const uint32_t* __restrict__ Hg, int par,
    uint32_t* cnt_out, unsigned long long* stats) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr bool PAY = tp_pay<S>();
    constexpr uint32_t WB = TP_TILE * sizeof(K) + 32, PB = PAY ? TP_TILE * tp_psz<S>() + 32 : 0;
    K* const buf0 = (K*)smem;
    K* const buf1 = (K*)(smem + WB);
    S* const pbuf0 = (S*)(smem + 2 * WB);
    S* const pbuf1 = (S*)(smem + 2 * WB + PB);
    uint16_t* const s_perm = (uint16_t*)(smem + 2 * WB + 2 * PB);  // [TILE] source index by output slot
    unsigned char* q = smem + 2 * WB + 2 * PB + TP_TILE * 2;
    q = (unsigned char*)(((uintptr_t)q + 7) & ~(uintptr_t)7);
    int64_t* s_run = (int64_t*)q;                                         // [ND]
    int64_t* s_goff = s_run + TP_ND;                                      // [ND]
    uint32_t(*s_whist)[TP_ND] = (uint32_t(*)[TP_ND])(s_goff + TP_ND);     // [WARPS][ND]
    uint32_t* s_match = &s_whist[TP_WARPS][0];                            // [WARPS][ND]
    uint32_t(*s_part)[TP_ND] = (uint32_t(*)[TP_ND])(s_match + TP_WARPS * TP_ND);  // [16][ND]
    uint32_t* s_w = &s_part[16][0];                                       // [4]
    uint64_t* s_bar = (uint64_t*)(((uintptr_t)(s_w + 4) + 7) & ~(uintptr_t)7);  // [2]

    pdl_wait();
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const uint64_t cnt = cntp ? min((uint64_t)*cntp, n) : n;
    const uint32_t cps = gridDim.x, c = blockIdx.x;
    const TpChunk ch = tp_chunk(cnt, cps, c);
    const uint64_t lo = ch.lo, hi = ch.hi;
    const uint32_t ntile = hi > lo ? (uint32_t)((hi - lo + TP_TILE - 1) / TP_TILE) : 0u;
    if (c == 0 && tid == 0) {
        if (cnt_out) *cnt_out = (uint32_t)cnt;  // (the output's count)
        if (stats) atomicAdd(&stats[ST_PASS_KEYS], (unsigned long long)cnt);
    }

    for (int i = tid; i < 2 * TP_WARPS * TP_ND; i += TP_THREADS) (&s_whist[0][0])[i] = 0u;
    auto issue = [&](uint32_t t, uint64_t* bar) {
        const uint64_t g0 = lo + (uint64_t)t * TP_TILE;
        const uint32_t ct = (uint32_t)min((uint64_t)TP_TILE, hi - g0);
        const uint32_t bw = tp_span(win, g0, ct);
        uint32_t bs = 0;
        if constexpr (PAY) bs = tp_span(sin, g0, ct);
        mbar_expect_tx(bar, bw + bs);
        tp_bulk((t & 1) ? buf1 : buf0, tp_base(win, g0), bw, bar);
        if constexpr (PAY) tp_bulk((t & 1) ? pbuf1 : pbuf0, tp_base(sin, g0), bs, bar);
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint32_t t = 0; t < 2 && t < ntile; ++t) issue(t, &s_bar[t]);
    }
    // digit totals of the pass and this chunk's prefix: thread (part p = tid / 64,
    // digit d = tid % 64)
    {
        const int d = tid & (TP_ND - 1), p = tid >> 6;
        constexpr uint32_t ST = TP_THREADS / TP_ND;  // 8 parts
        uint32_t tot = 0, pre = 0;
        if (Hg) {
            // block sums (8 chunks each): all blocks for the totals, those before this
            // chunk's block for the prefix, plus the rows of the chunks of this block
            // before it (every load independent: one round trip)
            const uint32_t nb = (cps + TP_HG_BLOCK - 1) / TP_HG_BLOCK, cb = c / TP_HG_BLOCK;
            const uint32_t* hg = Hg + (size_t)par * TP_HG_MAX_BLOCKS * TP_ND;
            uint32_t v[TP_HG_MAX_BLOCKS / ST];
#pragma unroll
            for (int u = 0; u < TP_HG_MAX_BLOCKS / (int)ST; ++u) {
                const uint32_t bb = p + u * ST;
                v[u] = bb < nb ? hg[(size_t)bb * TP_ND + d] : 0u;
            }
            const uint32_t own = (uint32_t)p < c - cb * TP_HG_BLOCK
                                     ? H[(uint64_t)(cb * TP_HG_BLOCK + p) * TP_ND + d] : 0u;
#pragma unroll
            for (int u = 0; u < TP_HG_MAX_BLOCKS / (int)ST; ++u) {
                tot += v[u];
                pre += p + u * ST < cb ? v[u] : 0u;
            }
            pre += own;
        } else {
            // (8 independent loads in flight per round trip: the chunk rows are L2 reads)
            for (uint32_t c0 = p; c0 < cps; c0 += 8 * ST) {
                uint32_t v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t cc = c0 + u * ST;
                    v[u] = cc < cps ? H[(uint64_t)cc * TP_ND + d] : 0u;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    tot += v[u];
                    pre += c0 + u * ST < c ? v[u] : 0u;
                }
            }
        }
        s_part[p][d] = tot;
        s_part[8 + p][d] = pre;
    }
    __syncthreads();
    uint32_t tot = 0, pre = 0;
    if (tid < TP_ND) {
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            tot += s_part[p][tid];
            pre += s_part[8 + p][tid];
        }
    }
    const uint32_t dbase = tp_scan64(tid < TP_ND ? tot : 0u, s_w);
    if (tid < TP_ND) s_run[tid] = (int64_t)dbase + pre;
    __syncthreads();

    uint32_t* whist = s_whist[wp];
    uint32_t* mbin = s_match + wp * TP_ND;
    const uint32_t lt = lanemask_lt();
    for (uint32_t t = 0; t < ntile; ++t) {
        const int b = (int)(t & 1u);
        const uint64_t t0 = lo + (uint64_t)t * TP_TILE;
        const uint32_t ct = (uint32_t)min((uint64_t)TP_TILE, hi - t0);
        const K* const buf = b ? buf1 : buf0;
        const S* pbuf = b ? pbuf1 : pbuf0;
        mbar_wait(&s_bar[b], (t >> 1) & 1u);
        const K* kin = buf + tp_delta(win, t0);
        const S* pin = nullptr;
        if constexpr (PAY) pin = pbuf + tp_delta(sin, t0);
        // stable in-warp ranking: lanes of one digit meet in a shared atomicOr mask;
        // only the digits (8 bits each, 4 per register) and ranks (16 bits, 2 per
        // register) stay in registers -- the elements are read again by source index
        uint32_t dg[TP_ITEMS / 4], rank[TP_ITEMS / 2];
#pragma unroll
        for (int i = 0; i < TP_ITEMS; ++i) {
            const uint32_t idx = (uint32_t)(wp * TP_ITEMS * 32 + i * 32 + lane);
            const bool valid = idx < ct;
            const uint32_t d = valid ? (uint32_t)(kin[idx] >> shift) & dmask : 0u;
            dg[i / 4] = (i & 3) ? (dg[i / 4] | d << (8 * (i & 3))) : d;
            if (valid) atomicOr(&mbin[d], 1u << lane);
            __syncwarp();
            const uint32_t peers = valid ? mbin[d] : 0u;
            const uint32_t prior = valid ? whist[d] : 0u;
            __syncwarp();
            if (valid && (peers & lt) == 0u) {
                whist[d] = prior + __popc(peers);
                mbin[d] = 0u;
            }
            __syncwarp();
            const uint32_t r = prior + __popc(peers & lt);
            rank[i / 2] = (i & 1) ? (rank[i / 2] | r << 16) : r;
        }
        __syncthreads();  // (A) counters final
        uint32_t tcnt = 0;
        if (tid < TP_ND) {
#pragma unroll
            for (int ww = 0; ww < TP_WARPS; ++ww) tcnt += s_whist[ww][tid];
        }
        const uint32_t doff = tp_scan64(tcnt, s_w);
        if (tid < TP_ND) {
            uint32_t sum = doff;
#pragma unroll
            for (int ww = 0; ww < TP_WARPS; ++ww) {
                const uint32_t v = s_whist[ww][tid];
                s_whist[ww][tid] = sum;
                sum += v;
            }
            s_goff[tid] = s_run[tid] - (int64_t)doff;
            s_run[tid] += tcnt;
        }
        __syncthreads();  // (B)
#pragma unroll
        for (int i = 0; i < TP_ITEMS; ++i) {
            const uint32_t idx = (uint32_t)(wp * TP_ITEMS * 32 + i * 32 + lane);
            if (idx < ct) {
                const uint32_t d = (dg[i / 4] >> (8 * (i & 3))) & 0xffu;
                const uint32_t pos = whist[d] + ((rank[i / 2] >> (16 * (i & 1))) & 0xffffu);
                GK_CHECK(pos < ct);
                s_perm[pos] = (uint16_t)idx;
            }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < TP_ND / 32; ++j) whist[j * 32 + lane] = 0u;
        __syncthreads();  // (C) the tile's stable order in s_perm
        for (uint32_t j = tid; j < ct; j += TP_THREADS) {
            const uint32_t src = s_perm[j];
            const K k = kin[src];
            const uint32_t d = (uint32_t)(k >> shift) & dmask;
            const uint64_t dst = (uint64_t)(s_goff[d] + (int64_t)j);
            GK_CHECK(dst < cnt);
            wout[dst] = k & omask;
            if constexpr (PAY) sout[dst] = pin[src];
        }
        __syncthreads();  // (D) the tile buffers free
        if (t + 2 < ntile && tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(t + 2, &s_bar[b]);
        }
    }
    pdl_trigger();
}

__global__ void fill_u32_kernel(uint32_t* p, uint32_t v, uint32_t count) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
        p[i] = v;
}

}  // namespace

cudaError_t launch_fill_u32(uint32_t* p, uint32_t v, uint32_t count, cudaStream_t s) {
    if (count == 0) return cudaGetLastError();
    fill_u32_kernel<<<(count + 255) / 256 < 64 ? (count + 255) / 256 : 64, 256, 0, s>>>(p, v, count);
    return cudaGetLastError();
}

// records bucketed by a <= 6-bit digit (far-pair records: the accumulator block),
// payload-less; cntp: device count (clamped to n)
template <typename K>
static cudaError_t tp_records(const K* in, K* out, uint64_t n, const uint32_t* cntp, int shift,
                              uint32_t* H, int target_ctas, cudaStream_t s) {
    if (n == 0) return cudaGetLastError();
    const uint64_t tiles = (n + TP_TILE - 1) / TP_TILE;
    const unsigned cps = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, target_ctas));
    cudaError_t e = launch_pdl(tp_hist_kernel<K>, cps, TPH_THREADS, 0, s, in, n, cntp, shift, 63u, H,
                               (uint32_t*)nullptr, 0);
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(tp_scatter_kernel<K, TpNoPay>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)tp_smem<K, TpNoPay>());
    e = launch_pdl(tp_scatter_kernel<K, TpNoPay>, cps, TP_THREADS, tp_smem<K, TpNoPay>(), s, in, out,
                   (const TpNoPay*)nullptr, (TpNoPay*)nullptr, n, cntp, shift, 63u, ~(K)0, H,
                   (const uint32_t*)nullptr, 0, (uint32_t*)nullptr, (unsigned long long*)nullptr);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_tp_records(const void* in, void* out, bool k32, uint64_t n, const uint32_t* cntp,
                              int shift, uint32_t* H, int target_ctas, cudaStream_t s) {
    if (k32)
        return tp_records<uint32_t>((const uint32_t*)in, (uint32_t*)out, n, cntp, shift, H,
                                    target_ctas, s);
    return tp_records<uint64_t>((const uint64_t*)in, (uint64_t*)out, n, cntp, shift, H,
                                target_ctas, s);
}

// Σ <= 64 (dmask < 64): the two-launch pass above; returns false when it does not
// apply (the caller uses launch_trie_pass)
bool trie_pass64_ok(uint32_t dmask) { return dmask < (uint32_t)TP_ND; }

cudaError_t launch_trie_pass64(const uint64_t* win, uint64_t* wout, const void* sin, void* sout,
                               bool seq16, uint64_t n, const uint32_t* cntp, int shift,
                               uint32_t dmask, uint64_t omask, uint32_t* H, int target_ctas,
                               cudaStream_t s, uint32_t* cnt_out, unsigned long long* stats,
                               uint32_t* Hg, uint32_t* par_ctr) {
    if (n == 0) return cudaGetLastError();
    const uint64_t tiles = (n + TP_TILE - 1) / TP_TILE;
    const unsigned cps = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, target_ctas));
    if (cps > (unsigned)TP_HG_BLOCK * TP_HG_MAX_BLOCKS || !par_ctr) Hg = nullptr;
    // (the parity advances only with a pass that uses the block sums: each such pass
    // zeroes the sums the next one accumulates into)
    const int par = Hg ? (int)((*par_ctr)++ & 1u) : 0;
    cudaError_t e = launch_pdl(tp_hist_kernel<uint64_t>, cps, TPH_THREADS, 0, s, win, n, cntp, shift,
                               dmask, H, Hg, par);
    if (e != cudaSuccess) return e;
    if (seq16) {
        cudaFuncSetAttribute(tp_scatter_kernel<uint64_t, uint16_t>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tp_smem<uint64_t, uint16_t>());
        e = launch_pdl(tp_scatter_kernel<uint64_t, uint16_t>, cps, TP_THREADS, tp_smem<uint64_t, uint16_t>(),
                       s, win, wout, (const uint16_t*)sin, (uint16_t*)sout, n, cntp, shift, dmask, omask,
                       H, Hg, par, cnt_out, stats);
    } else {
        cudaFuncSetAttribute(tp_scatter_kernel<uint64_t, uint32_t>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tp_smem<uint64_t, uint32_t>());
        e = launch_pdl(tp_scatter_kernel<uint64_t, uint32_t>, cps, TP_THREADS, tp_smem<uint64_t, uint32_t>(),
                       s, win, wout, (const uint32_t*)sin, (uint32_t*)sout, n, cntp, shift, dmask, omask,
                       H, Hg, par, cnt_out, stats);
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("GAKCO_PDL");
        return !(v && v[0] == '0');
    }();
    return on;
}

}  // namespace gk
