// radix.cu — one LSD pass of a onesweep radix sort over a batch of segments.
//
// Algorithm 1 line 14, L^i <- sort(L^i); Supp. §S:1.2
// argues for a non-swapping Θ(g·Nl) sort. Each pass stably scatters the
// composites by one 8-bit digit of the KEY bits only: the sequence id in the low
// sb bits is already ascending within equal keys (the encoder writes g-mers in
// sequence order and every pass is stable), so no pass is spent on it.
//
// A batch holds `nseg` masks, each a segment of exactly n composites at
// [seg*n, (seg+1)*n). Tiles never straddle segments; the digit histogram of the
// whole segment comes from the encoder (upfront histogram), so one kernel per
// pass suffices:
//   1. a CTA takes the next tile ticket (ordered, so look-back cannot deadlock);
//   2. it ranks its 4096 keys stably by digit (warp match + per-warp counters);
//   3. it publishes its per-digit counts (decoupled look-back, one status word per
//      (segment, digit, tile)) and looks back for the exclusive prefix;
//   4. it reorders the tile by digit in shared memory and writes each digit's run
//      contiguously to  seg*n + digit_base[d] + prefix[d] + local offset.
#include <algorithm>
#include <type_traits>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace gk {

constexpr size_t ONESWEEP_SMEM = SORT_TILE * 8 + RADIX * 8 + (SORT_THREADS / 32) * RADIX * 4 +
                                 RADIX * 4 + 16 * 4;

__global__ void __launch_bounds__(SORT_THREADS) onesweep_kernel(
    const uint64_t* __restrict__ in, uint64_t* __restrict__ out, uint64_t n, uint32_t tps,
    uint32_t nseg, int shift, const uint32_t* __restrict__ hist, int pass, int npass,
    uint64_t* status, uint32_t* ctr, uint32_t epoch) {
    constexpr int WARPS = SORT_THREADS / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* s_keys = (uint64_t*)smem;                                   // [SORT_TILE]
    int64_t* s_goff = (int64_t*)(s_keys + SORT_TILE);                     // [RADIX]
    uint32_t(*s_whist)[RADIX] = (uint32_t(*)[RADIX])(s_goff + RADIX);     // [WARPS][RADIX]
    uint32_t* s_doff = &s_whist[WARPS][0];                                // [RADIX]
    uint32_t* s_w = s_doff + RADIX;                                       // [8]
    uint32_t& s_tile = s_w[12];

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ctr, 1u);
    for (int i = tid; i < WARPS * RADIX; i += SORT_THREADS) (&s_whist[0][0])[i] = 0;
    __syncthreads();
    // tickets interleave the segments (ticket t -> tile t / nseg of segment
    // t % nseg) so the tiles in flight spread over many look-back chains
    const uint32_t t = s_tile;
    const uint32_t ts = t / nseg, seg = t - ts * nseg;
    const uint64_t seg_base = (uint64_t)seg * n;
    const uint64_t tile_base = seg_base + (uint64_t)ts * SORT_TILE;
    const uint64_t rem = n - (uint64_t)ts * SORT_TILE;
    const uint32_t cnt = rem < SORT_TILE ? (uint32_t)rem : (uint32_t)SORT_TILE;

    // 1. load (warp-blocked, coalesced per iteration) and rank stably per warp
    uint64_t keys[SORT_ITEMS];
    uint32_t rank[SORT_ITEMS];
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        uint32_t idx = w * SORT_ITEMS * 32 + i * 32 + lane;
        keys[i] = idx < cnt ? in[tile_base + idx] : 0ull;
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        uint32_t idx = w * SORT_ITEMS * 32 + i * 32 + lane;
        bool valid = idx < cnt;
        uint32_t d = (uint32_t)(keys[i] >> shift) & 0xffu;
        uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        uint32_t peers = digit_peers(d, vmask);
        uint32_t prior = valid ? s_whist[w][d] : 0u;
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) s_whist[w][d] = prior + __popc(peers);
        __syncwarp();
        rank[i] = prior + __popc(peers & lt);
    }
    __syncthreads();

    // 2. per-digit tile totals, warp-exclusive prefixes; publish aggregate
    uint32_t tile_cnt = 0;
    if (tid < RADIX) {
        uint32_t sum = 0;
        for (int ww = 0; ww < WARPS; ++ww) {
            uint32_t c = s_whist[ww][tid];
            s_whist[ww][tid] = sum;
            sum += c;
        }
        tile_cnt = sum;
        uint64_t* st = status + ((uint64_t)seg * RADIX + tid) * tps + ts;
        *(volatile uint64_t*)st = lb_pack(epoch, ts == 0 ? LB_INC : LB_AGG, sum);
    }
    const uint32_t doff = scan256_excl(tid < RADIX ? tile_cnt : 0u, s_w);
    const uint32_t hval = tid < RADIX ? hist[((uint64_t)seg * npass + pass) * RADIX + tid] : 0u;
    const uint32_t dbase = scan256_excl(hval, s_w);

    // 3. decoupled look-back per digit
    if (tid < RADIX) {
        s_doff[tid] = doff;
        uint32_t excl = 0;
        if (ts > 0) {
            // windowed look-back: the statuses of one (segment, digit) are contiguous
            // over tiles, so LB_WIN predecessors are read with independent loads per
            // round trip; consume them nearest-first until an inclusive prefix.
            constexpr int LB_WIN = 8;
            const uint64_t* col = status + ((uint64_t)seg * RADIX + tid) * tps;
            int64_t p = (int64_t)ts - 1;
            bool done = false;
            while (!done) {
                uint64_t v[LB_WIN];
#pragma unroll
                for (int j = 0; j < LB_WIN; ++j)
                    v[j] = (p - j >= 0) ? *(volatile const uint64_t*)(col + p - j) : 0ull;
                int used = 0;
                bool stop = false;
#pragma unroll
                for (int j = 0; j < LB_WIN; ++j) {
                    if (stop) continue;
                    const uint32_t ep = (uint32_t)(v[j] >> 32), fl = (uint32_t)(v[j] >> 30) & 3u;
                    if (p - j < 0 || ep != epoch || fl == LB_NONE) {
                        stop = true;  // not published yet: re-read from here
                        continue;
                    }
                    excl += (uint32_t)(v[j] & 0x3fffffffu);
                    ++used;
                    if (fl == LB_INC) {
                        done = true;
                        stop = true;
                    }
                }
                p -= used;
            }
            *(volatile uint64_t*)(status + ((uint64_t)seg * RADIX + tid) * tps + ts) =
                lb_pack(epoch, LB_INC, excl + tile_cnt);
        }
        s_goff[tid] = (int64_t)dbase + (int64_t)excl - (int64_t)doff;
    }
    __syncthreads();

    // 4. reorder the tile by digit in shared memory, then write runs out
#pragma unroll
    for (int i = 0; i < SORT_ITEMS; ++i) {
        uint32_t idx = w * SORT_ITEMS * 32 + i * 32 + lane;
        if (idx < cnt) {
            uint32_t d = (uint32_t)(keys[i] >> shift) & 0xffu;
            s_keys[s_doff[d] + s_whist[w][d] + rank[i]] = keys[i];
        }
    }
    __syncthreads();
    for (uint32_t j = tid; j < cnt; j += SORT_THREADS) {
        uint64_t k = s_keys[j];
        uint32_t d = (uint32_t)(k >> shift) & 0xffu;
        out[seg_base + (uint64_t)(s_goff[d] + (int64_t)j)] = k;
    }
}

cudaError_t launch_onesweep(const uint64_t* in, uint64_t* out, uint64_t n, int nseg, int shift,
                            const uint32_t* hist, int pass, int npass, uint64_t* status,
                            uint32_t* ctr, uint32_t epoch, cudaStream_t s) {
    if (n == 0 || nseg == 0) return cudaGetLastError();
    uint32_t tps = (uint32_t)((n + SORT_TILE - 1) / SORT_TILE);
    uint64_t tiles = (uint64_t)tps * nseg;
    cudaFuncSetAttribute(onesweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)ONESWEEP_SMEM);
    onesweep_kernel<<<(unsigned)tiles, SORT_THREADS, ONESWEEP_SMEM, s>>>(in, out, n, tps,
                                                             (uint32_t)nseg, shift, hist, pass,
                                                             npass, status, ctr, epoch);
    return cudaGetLastError();
}

// ============================================================================
// Chunked LSD pass (no look-back chain): the same stable 8-bit pass, split in
// two kernels so that no tile ever waits on another:
//   radix_hist:    CTA (seg, c) counts the pass digit over its chunk of L keys;
//   radix_scatter: CTA (seg, c) sums the chunk histograms of its segment (digit
//                  totals -> digit bases; chunks < c -> its prefix), then walks
//                  its chunk in 4096-key tiles IN ORDER, ranking each tile
//                  stably (warp match + per-warp counters), reordering it by
//                  digit in shared memory and writing each digit run to
//                  seg*n + base[d] + prefix[d] + running[d] + local offset.
// Batches are sized to stay resident in the 126 MB L2, so the second read of a
// chunk, and the next pass's reads of this pass's output, hit in L2.
// ============================================================================
constexpr int RS_THREADS = SORT_THREADS;  // 512
constexpr int RS_WARPS = RS_THREADS / 32;

template <typename K, bool DESC = false>
__global__ void __launch_bounds__(RS_THREADS) radix_hist_kernel(
    const K* __restrict__ in, uint64_t n, uint32_t cps, uint64_t L, int shift,
    uint32_t* __restrict__ hist, uint32_t dmask = 0xffu,
    const PassDesc* __restrict__ pdesc = nullptr) {
    constexpr int E = 16 / sizeof(K);  // keys per 16-byte load
    __shared__ uint32_t s_h[RS_WARPS][RADIX];
    const int tid = threadIdx.x, w = tid >> 5;
    for (int i = tid; i < RS_WARPS * RADIX; i += RS_THREADS) (&s_h[0][0])[i] = 0;
    __syncthreads();
    const uint32_t seg = blockIdx.x / cps, c = blockIdx.x - seg * cps;
    const uint64_t lo = (uint64_t)c * L;
    const uint64_t hi = min(n, lo + L);
    PassDesc pd{};
    if constexpr (DESC) pd = pdesc[seg];
    const K* p = in + (DESC ? pd.in_off : (uint64_t)seg * n);
    auto digit = [&](K k) -> uint32_t {
        if constexpr (DESC) return pd_digit(k, pd);
        else return (uint32_t)(k >> shift) & dmask;
    };
    if (lo < hi) {
        // 16-byte loads on the aligned body, scalars on the edges
        uint64_t a = lo;
        while (a < hi && ((uintptr_t)(p + a) & 15)) {
            if (tid == 0) atomicAdd(&s_h[0][digit(p[a])], 1u);
            ++a;
        }
        const uint64_t nv = (hi - a) / E;
        const uint4* v = (const uint4*)(p + a);
        for (uint64_t i = tid; i < nv; i += RS_THREADS) {
            const uint4 q = v[i];
            const K* kq = (const K*)&q;
#pragma unroll
            for (int e = 0; e < E; ++e) atomicAdd(&s_h[w][digit(kq[e])], 1u);
        }
        for (uint64_t i = a + nv * E + tid; i < hi; i += RS_THREADS)
            atomicAdd(&s_h[w][digit(p[i])], 1u);
    }
    __syncthreads();
    if (tid < RADIX) {
        uint32_t s = 0;
        for (int ww = 0; ww < RS_WARPS; ++ww) s += s_h[ww][tid];
        hist[((uint64_t)seg * cps + c) * RADIX + tid] = s;
    }
}

template <typename K>
__global__ void __launch_bounds__(RS_THREADS, 2) radix_scatter_kernel(
    const K* __restrict__ in, K* __restrict__ out, uint64_t n, uint32_t cps,
    uint64_t L, int shift, const uint32_t* __restrict__ hist) {
    extern __shared__ __align__(16) unsigned char smem[];
    K* s_keys = (K*)smem;                                                // [SORT_TILE]
    int64_t* s_run = (int64_t*)(smem + SORT_TILE * sizeof(K));           // [RADIX]
    int64_t* s_goff = s_run + RADIX;                                     // [RADIX]
    uint32_t(*s_whist)[RADIX] = (uint32_t(*)[RADIX])(s_goff + RADIX);    // [WARPS][RADIX]
    uint32_t* s_cnt = &s_whist[RS_WARPS][0];                             // [RADIX]
    uint32_t* s_w = s_cnt + RADIX;                                       // [16]
    uint32_t* s_match = s_w + 16;                                        // [WARPS][RADIX]
    for (int i = threadIdx.x; i < RS_WARPS * RADIX; i += RS_THREADS) s_match[i] = 0u;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t seg = blockIdx.x / cps, c = blockIdx.x - seg * cps;
    const uint64_t lo = (uint64_t)c * L;
    const uint64_t hi = min(n, lo + L);
    const uint64_t seg_base = (uint64_t)seg * n;

    // digit totals of the segment and this chunk's prefix (all chunks < c)
    uint32_t tot = 0, pre = 0;
    if (tid < RADIX) {
        const uint32_t* h = hist + (uint64_t)seg * cps * RADIX + tid;
        for (uint32_t cc = 0; cc < cps; ++cc) {
            const uint32_t v = h[(uint64_t)cc * RADIX];
            tot += v;
            pre += cc < c ? v : 0u;
        }
    }
    const uint32_t dbase = scan256_excl(tot, s_w);
    if (tid < RADIX) s_run[tid] = (int64_t)dbase + pre;
    __syncthreads();

    const uint32_t lt = lanemask_lt();
    // register double buffer: the next tile's keys are in flight while this one
    // is ranked and scattered
    K nxt[SORT_ITEMS];
    {
        const uint32_t cnt0 = (uint32_t)min((uint64_t)SORT_TILE, hi > lo ? hi - lo : 0);
#pragma unroll
        for (int i = 0; i < SORT_ITEMS; ++i) {
            const uint32_t idx = w * SORT_ITEMS * 32 + i * 32 + lane;
            nxt[i] = idx < cnt0 ? in[seg_base + lo + idx] : (K)0;
        }
    }
    for (uint64_t t0 = lo; t0 < hi; t0 += SORT_TILE) {
        const uint32_t cnt = (uint32_t)min((uint64_t)SORT_TILE, hi - t0);
        for (int i = tid; i < RS_WARPS * RADIX; i += RS_THREADS) (&s_whist[0][0])[i] = 0;
        __syncthreads();
        K keys[SORT_ITEMS];
        uint32_t rank[SORT_ITEMS];
#pragma unroll
        for (int i = 0; i < SORT_ITEMS; ++i) keys[i] = nxt[i];
        if (t0 + SORT_TILE < hi) {
            const uint64_t t1 = t0 + SORT_TILE;
            const uint32_t cnt1 = (uint32_t)min((uint64_t)SORT_TILE, hi - t1);
#pragma unroll
            for (int i = 0; i < SORT_ITEMS; ++i) {
                const uint32_t idx = w * SORT_ITEMS * 32 + i * 32 + lane;
                nxt[i] = idx < cnt1 ? in[seg_base + t1 + idx] : (K)0;
            }
        }
        // stable in-warp ranking: lanes with the same digit find each other with a
        // shared-memory atomicOr of their lane bit (one ATOMS per key), the
        // lowest peer advances the warp's digit counter and clears the bin
        uint32_t* mbin = s_match + w * RADIX;
#pragma unroll
        for (int i = 0; i < SORT_ITEMS; ++i) {
            const uint32_t idx = w * SORT_ITEMS * 32 + i * 32 + lane;
            const bool valid = idx < cnt;
            const uint32_t d = (uint32_t)(keys[i] >> shift) & 0xffu;
            if (valid) atomicOr(&mbin[d], 1u << lane);
            __syncwarp();
            const uint32_t peers = valid ? mbin[d] : 0u;
            const uint32_t prior = valid ? s_whist[w][d] : 0u;
            __syncwarp();
            if (valid && lane == __ffs(peers) - 1) {
                s_whist[w][d] = prior + __popc(peers);
                mbin[d] = 0u;
            }
            __syncwarp();
            rank[i] = prior + __popc(peers & lt);
        }
        __syncthreads();
        uint32_t tcnt = 0;
        if (tid < RADIX) {
#pragma unroll
            for (int ww = 0; ww < RS_WARPS; ++ww) tcnt += s_whist[ww][tid];
            s_cnt[tid] = tcnt;
        }
        const uint32_t doff = scan256_excl(tcnt, s_w);
        if (tid < RADIX) {
            // s_whist[w][d] <- tile position of warp w's first digit-d key; s_goff[d] <-
            // global position of tile index 0 as if it were digit d (so that tile index
            // j of digit d goes to s_goff[d] + j): one lookup per key below
            uint32_t sum = doff;
#pragma unroll
            for (int ww = 0; ww < RS_WARPS; ++ww) {
                const uint32_t v = s_whist[ww][tid];
                s_whist[ww][tid] = sum;
                sum += v;
            }
            s_goff[tid] = s_run[tid] - (int64_t)doff;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < SORT_ITEMS; ++i) {
            const uint32_t idx = w * SORT_ITEMS * 32 + i * 32 + lane;
            if (idx < cnt) {
                const uint32_t d = (uint32_t)(keys[i] >> shift) & 0xffu;
                s_keys[s_whist[w][d] + rank[i]] = keys[i];
            }
        }
        __syncthreads();
        for (uint32_t j = tid; j < cnt; j += RS_THREADS) {
            const K k = s_keys[j];
            const uint32_t d = (uint32_t)(k >> shift) & 0xffu;
            out[seg_base + (uint64_t)(s_goff[d] + (int64_t)j)] = k;
        }
        __syncthreads();
        if (tid < RADIX) s_run[tid] += s_cnt[tid];
        // (the loop-top __syncthreads orders this before the next tile's reads)
    }
}

template <typename K>
constexpr size_t rs_smem() {
    return SORT_TILE * sizeof(K) + 2 * RADIX * 8 + 2 * RS_WARPS * RADIX * 4 + RADIX * 4 + 16 * 4;
}

template <typename K>
static cudaError_t radix_chunked(const K* in, K* out, uint64_t n, int nseg, int shift,
                                 uint32_t* hist, int target_ctas, cudaStream_t s) {
    // chunks per segment: fill ~target_ctas CTAs, whole 4096-key tiles per chunk
    uint64_t tiles = (n + SORT_TILE - 1) / SORT_TILE;
    uint64_t cps = std::max<uint64_t>(1, std::min<uint64_t>(tiles, (target_ctas + nseg - 1) / nseg));
    uint64_t L = (tiles + cps - 1) / cps * SORT_TILE;
    cps = (n + L - 1) / L;
    const unsigned grid = (unsigned)(cps * nseg);
    radix_hist_kernel<K><<<grid, RS_THREADS, 0, s>>>(in, n, (uint32_t)cps, L, shift, hist);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(radix_scatter_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)rs_smem<K>());
    radix_scatter_kernel<K><<<grid, RS_THREADS, rs_smem<K>(), s>>>(in, out, n, (uint32_t)cps, L,
                                                                   shift, hist);
    return cudaGetLastError();
}

// ============================================================================
// radix_scatter2: the same chunked stable pass, restructured for instruction
// count and latency (the v1 kernel issues ~4 warp instructions per key, spills,
// and its shared atomicOr match serialises per lane: ncu 29 wavefronts per ATOMS):
//   * 256 threads, 16 keys per thread, tiles of 4096 keys;
//   * the next tile streams into shared memory with one cp.async.bulk (TMA 1D,
//     mbarrier completion) while this one is ranked: no prefetch registers;
//   * full tiles take a branch-free path (only a chunk's last tile is partial);
//   * ranking by the shared atomicOr match (RANK = 0, default), match.any (1) or
//     ballot multisplit (2) -- measured on Text: 112 / 145 / 124 ms per step's sort;
//     a merged 64-bit {count | mask} bin (one atomic fewer) compiled to a CAS loop
//     and took 251 ms;
//     the per-warp digit counters are read-modify-written by the lowest peer;
//   * the tile is reordered in place (its input buffer) and written out per digit
//     run; each warp clears its own counters, so a tile needs 6 barriers.
// ============================================================================
constexpr int RS2_THREADS = 256;
constexpr int RS2_WARPS = RS2_THREADS / 32;
constexpr int RS2_ITEMS = 16;
constexpr int RS2_TILE = RS2_THREADS * RS2_ITEMS;  // 4096 keys

template <typename K>
__host__ __device__ constexpr size_t rs2_buf_bytes() {
    return RS2_TILE * sizeof(K) + 32;  // + alignment slack of the bulk copy
}
// payload moved along with the keys (the mask-trie passes: sequence ids); NoPay: none
struct NoPay {};
template <typename P>
__host__ __device__ constexpr bool rs2_haspay() {
    return !std::is_same<P, NoPay>::value;
}
template <typename P>
__host__ __device__ constexpr size_t rs2_pbuf_bytes() {
    return rs2_haspay<P>() ? RS2_TILE * sizeof(P) + 32 : 0;
}
template <typename K, typename P = NoPay>
constexpr size_t rs2_smem() {
    return 2 * rs2_buf_bytes<K>() + 3 * rs2_pbuf_bytes<P>() + 2 * RADIX * 8 +
           2 * RS2_WARPS * RADIX * 4 + RADIX * 4 + 16 * 4 + 2 * 8;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// issue the bulk copy of keys [g0, g0 + cnt) (16-byte aligned window); returns the
// element offset of key g0 inside the buffer
template <typename K>
__device__ __forceinline__ uint32_t rs2_bytes(const K* in, uint64_t g0, uint32_t cnt) {
    const uintptr_t a0 = (uintptr_t)(in + g0), a1 = (uintptr_t)(in + g0 + cnt);
    return (uint32_t)(((a1 + 15) & ~(uintptr_t)15) - (a0 & ~(uintptr_t)15));
}
template <typename K>
__device__ __forceinline__ void rs2_copy(K* buf, const K* in, uint64_t g0, uint32_t cnt,
                                         uint64_t* bar) {
    const uintptr_t a0 = (uintptr_t)(in + g0);
    bulk_g2s(buf, (const void*)(a0 & ~(uintptr_t)15), rs2_bytes(in, g0, cnt), bar);
}
// one barrier completes the key copy and (with a payload) the payload copy
template <typename K, typename P>
__device__ __forceinline__ void rs2_issue(K* buf, const K* in, P* pbuf, const P* pin, uint64_t g0,
                                          uint32_t cnt, uint64_t* bar) {
    uint32_t bytes = rs2_bytes(in, g0, cnt);
    if constexpr (rs2_haspay<P>()) bytes += rs2_bytes(pin, g0, cnt);
    mbar_expect_tx(bar, bytes);
    rs2_copy(buf, in, g0, cnt, bar);
    if constexpr (rs2_haspay<P>()) rs2_copy(pbuf, pin, g0, cnt, bar);
}

template <typename K, int RANK, bool FULL, typename Dig>
__device__ __forceinline__ void rs2_rank(const K (&keys)[RS2_ITEMS], uint32_t (&rank)[RS2_ITEMS],
                                         const Dig& digit, uint32_t cnt, uint32_t* whist,
                                         uint32_t* mbin, int w, int lane) {
    const uint32_t lt = lanemask_lt();
    if (RANK == 1) {
        // all match.any first (independent: in flight together), then the counter chain
#pragma unroll
        for (int i = 0; i < RS2_ITEMS; ++i) {
            const uint32_t idx = (uint32_t)(w * RS2_ITEMS * 32 + i * 32 + lane);
            uint32_t d = digit(keys[i]);
            if (!FULL && idx >= cnt) d = 0x100u;  // invalid lanes only match each other
            rank[i] = __match_any_sync(0xffffffffu, d);
        }
#pragma unroll
        for (int i = 0; i < RS2_ITEMS; ++i) {
            const uint32_t idx = (uint32_t)(w * RS2_ITEMS * 32 + i * 32 + lane);
            const bool valid = FULL || idx < cnt;
            const uint32_t d = digit(keys[i]);
            const uint32_t peers = rank[i];
            const uint32_t prior = valid ? whist[d] : 0u;
            __syncwarp();
            if (valid && (peers & lt) == 0u) whist[d] = prior + __popc(peers);
            __syncwarp();
            rank[i] = prior + __popc(peers & lt);
        }
    } else if (RANK == 2) {
        // ballot multisplit: peers from 8 votes, no shared atomics
#pragma unroll
        for (int i = 0; i < RS2_ITEMS; ++i) {
            const uint32_t idx = (uint32_t)(w * RS2_ITEMS * 32 + i * 32 + lane);
            const bool valid = FULL || idx < cnt;
            const uint32_t d = digit(keys[i]);
            const uint32_t peers = digit_peers(d, __ballot_sync(0xffffffffu, valid));
            const uint32_t prior = valid ? whist[d] : 0u;
            __syncwarp();
            if (valid && (peers & lt) == 0u) whist[d] = prior + __popc(peers);
            __syncwarp();
            rank[i] = prior + __popc(peers & lt);
        }
    } else {
#pragma unroll
        for (int i = 0; i < RS2_ITEMS; ++i) {
            const uint32_t idx = (uint32_t)(w * RS2_ITEMS * 32 + i * 32 + lane);
            const bool valid = FULL || idx < cnt;
            const uint32_t d = digit(keys[i]);
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
            rank[i] = prior + __popc(peers & lt);
        }
    }
}

template <typename K, typename P, int RANK, bool DESC = false>
__global__ void __launch_bounds__(RS2_THREADS, (sizeof(K) == 8 ? 2 : 3)) radix_scatter2_kernel(
    const K* __restrict__ in, K* __restrict__ out, const P* __restrict__ pin, P* __restrict__ pout,
    uint64_t n, uint32_t cps, uint64_t L, int shift, uint32_t dmask_,
    const uint32_t* __restrict__ hist, K omask_, int prescanned,
    const PassDesc* __restrict__ pdesc = nullptr) {
    constexpr bool HASP = rs2_haspay<P>();
    // (the plain LSD passes: full 8-bit digits, no output mask -- compile-time)
    const uint32_t dmask = HASP ? dmask_ : 0xffu;
    extern __shared__ __align__(16) unsigned char smem[];
    K* const buf0 = (K*)smem;
    K* const buf1 = (K*)(smem + rs2_buf_bytes<K>());
    P* const pbuf0 = (P*)(smem + 2 * rs2_buf_bytes<K>());
    P* const pbuf1 = (P*)(smem + 2 * rs2_buf_bytes<K>() + rs2_pbuf_bytes<P>());
    P* const s_pout = (P*)(smem + 2 * rs2_buf_bytes<K>() + 2 * rs2_pbuf_bytes<P>());
    unsigned char* q = smem + 2 * rs2_buf_bytes<K>() + 3 * rs2_pbuf_bytes<P>();
    int64_t* s_run = (int64_t*)q;                                        // [RADIX]
    int64_t* s_goff = s_run + RADIX;                                     // [RADIX]
    uint32_t(*s_whist)[RADIX] = (uint32_t(*)[RADIX])(s_goff + RADIX);    // [WARPS][RADIX]
    uint32_t* s_match = &s_whist[RS2_WARPS][0];                          // [WARPS][RADIX]
    uint32_t* s_cnt = s_match + RS2_WARPS * RADIX;                       // [RADIX]
    uint32_t* s_w = s_cnt + RADIX;                                       // [16]
    uint64_t* s_bar = (uint64_t*)(s_w + 16);                             // [2]

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t seg = blockIdx.x / cps, c = blockIdx.x - seg * cps;
    const uint64_t lo = (uint64_t)c * L;
    const uint64_t hi = min(n, lo + L);
    // batched trie passes (DESC): each segment reads its own input array, sorts by
    // its own digit (up to 4 symbols) and writes its own (masked) output
    PassDesc pd{};
    if constexpr (DESC) pd = pdesc[seg];
    const uint64_t seg_base = DESC ? pd.out_off : (uint64_t)seg * n;
    const K* src = in + (DESC ? pd.in_off : seg_base);
    const P* psrc = HASP ? pin + seg_base : nullptr;
    const K omask = DESC ? (K)pd.omask : (HASP ? omask_ : ~(K)0);
    auto digit = [&](K k) -> uint32_t {
        if constexpr (DESC) return pd_digit(k, pd);
        else return (uint32_t)(k >> shift) & dmask;
    };
    const uint32_t ntile = hi > lo ? (uint32_t)((hi - lo + RS2_TILE - 1) / RS2_TILE) : 0u;

    for (int i = tid; i < 2 * RS2_WARPS * RADIX; i += RS2_THREADS) (&s_whist[0][0])[i] = 0u;
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint32_t t = 0; t < 2 && t < ntile; ++t) {
            const uint64_t g0 = lo + (uint64_t)t * RS2_TILE;
            rs2_issue(t ? buf1 : buf0, src, t ? pbuf1 : pbuf0, psrc, g0,
                      (uint32_t)min((uint64_t)RS2_TILE, hi - g0), &s_bar[t]);
        }
    }
    // this chunk's digit offsets in its segment: hist_scan_kernel turned the chunk
    // histograms into exclusive prefixes over chunks and appended the digit totals
    // (few chunks: summed here, each CTA over its segment's chunk rows)
    uint32_t pre = 0, tot = 0;
    if (prescanned) {
        pre = hist[((uint64_t)seg * cps + c) * RADIX + tid];
        tot = hist[(uint64_t)gridDim.x * RADIX + (uint64_t)seg * RADIX + tid];
    } else {
        const uint32_t* h = hist + (uint64_t)seg * cps * RADIX + tid;
        for (uint32_t cc = 0; cc < cps; ++cc) {
            const uint32_t v = h[(uint64_t)cc * RADIX];
            tot += v;
            pre += cc < c ? v : 0u;
        }
    }
    const uint32_t dbase = scan256_excl(tot, s_w);
    s_run[tid] = (int64_t)dbase + pre;
    // element offset of a tile's first key inside its buffer (16-byte aligned copies)
    auto delta_of = [&](uint32_t t) -> uint32_t {
        return (uint32_t)((((uintptr_t)(src + lo + (uint64_t)t * RS2_TILE)) & 15) / sizeof(K));
    };
    auto pdelta_of = [&](uint32_t t) -> uint32_t {
        return HASP ? (uint32_t)((((uintptr_t)(psrc + lo + (uint64_t)t * RS2_TILE)) & 15) /
                                 sizeof(P))
                    : 0u;
    };
    __syncthreads();

    uint32_t* whist = s_whist[w];
    uint32_t* mbin = s_match + w * RADIX;
    for (uint32_t t = 0; t < ntile; ++t) {
        const int b = (int)(t & 1u);
        const uint64_t t0 = lo + (uint64_t)t * RS2_TILE;
        const uint32_t cnt = (uint32_t)min((uint64_t)RS2_TILE, hi - t0);
        K* buf = b ? buf1 : buf0;
        P* pbuf = b ? pbuf1 : pbuf0;
        mbar_wait(&s_bar[b], (t >> 1) & 1u);
        const K* kin = buf + delta_of(t);
        K keys[RS2_ITEMS];
        uint32_t rank[RS2_ITEMS];
#pragma unroll
        for (int i = 0; i < RS2_ITEMS; ++i) {
            const uint32_t idx = (uint32_t)(w * RS2_ITEMS * 32 + i * 32 + lane);
            keys[i] = (cnt == RS2_TILE || idx < cnt) ? kin[idx] : (K)0;
        }
        if (cnt == RS2_TILE)
            rs2_rank<K, RANK, true>(keys, rank, digit, cnt, whist, mbin, w, lane);
        else
            rs2_rank<K, RANK, false>(keys, rank, digit, cnt, whist, mbin, w, lane);
        __syncthreads();  // (A) every warp's counters final; every key of buf read
        uint32_t tcnt = 0;
#pragma unroll
        for (int ww = 0; ww < RS2_WARPS; ++ww) tcnt += s_whist[ww][tid];
        s_cnt[tid] = tcnt;
        const uint32_t doff = scan256_excl(tcnt, s_w);
        {
            uint32_t sum = doff;
#pragma unroll
            for (int ww = 0; ww < RS2_WARPS; ++ww) {
                const uint32_t v = s_whist[ww][tid];
                s_whist[ww][tid] = sum;
                sum += v;
            }
            s_goff[tid] = s_run[tid] - (int64_t)doff;
            s_run[tid] += tcnt;
        }
        __syncthreads();  // (B)
        const P* pk = HASP ? pbuf + pdelta_of(t) : nullptr;
#pragma unroll
        for (int i = 0; i < RS2_ITEMS; ++i) {
            const uint32_t idx = (uint32_t)(w * RS2_ITEMS * 32 + i * 32 + lane);
            if (cnt == RS2_TILE || idx < cnt) {
                const uint32_t d = digit(keys[i]);
                const uint32_t pos = whist[d] + rank[i];
                buf[pos] = keys[i];
                if constexpr (HASP) s_pout[pos] = pk[idx];
            }
        }
        __syncwarp();
        // this warp's counters are no longer read by anyone: clear for the next tile
#pragma unroll
        for (int j = 0; j < RADIX / 32; ++j) whist[j * 32 + lane] = 0u;
        __syncthreads();  // (C) tile reordered in buf
        for (uint32_t j = tid; j < cnt; j += RS2_THREADS) {
            const K k = buf[j];
            const uint32_t d = digit(k);
            const uint64_t dst = seg_base + (uint64_t)(s_goff[d] + (int64_t)j);
            out[dst] = k & omask;  // (the trie's leaf pass applies the mask's key bits)
            if constexpr (HASP) pout[dst] = s_pout[j];
        }
        if (t + 2 < ntile) {
            // buf is free once every thread has written its share out
            __syncthreads();  // (D)
            const uint64_t g2 = lo + (uint64_t)(t + 2) * RS2_TILE;
            if (tid == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                rs2_issue(buf, src, pbuf, psrc, g2, (uint32_t)min((uint64_t)RS2_TILE, hi - g2),
                          &s_bar[b]);
            }
        } else if (HASP) {
            __syncthreads();  // s_pout is rewritten by the next tile's reorder
        }
        // (the next tile's barrier A orders s_goff / s_cnt reuse)
    }
}

// chunk histograms [seg][chunk][digit] -> exclusive prefixes over the chunks of each
// segment, in place; the segment's digit totals go after all chunk rows, at
// [nseg * cps + seg][digit]. A warp per (segment, digit): its lanes load 32 chunks
// per step, all steps' loads in flight before the carried warp scans.
constexpr int HS_STEPS = 24;  // up to 768 chunks per segment in one round trip
__global__ void __launch_bounds__(256) hist_scan_kernel(uint32_t* hist, uint32_t cps,
                                                         uint32_t nseg) {
    const int lane = threadIdx.x & 31;
    const uint32_t wid = blockIdx.x * 8 + (threadIdx.x >> 5);  // (segment, digit)
    if (wid >= nseg * RADIX) return;
    const uint32_t seg = wid / RADIX, d = wid % RADIX;
    uint32_t* h = hist + (uint64_t)seg * cps * RADIX + d;
    uint32_t run = 0;
    for (uint32_t c0 = 0; c0 < cps; c0 += 32 * HS_STEPS) {
        uint32_t v[HS_STEPS];
#pragma unroll
        for (int k = 0; k < HS_STEPS; ++k) {
            const uint32_t c = c0 + k * 32 + lane;
            v[k] = c < cps ? h[(uint64_t)c * RADIX] : 0u;
        }
#pragma unroll
        for (int k = 0; k < HS_STEPS; ++k) {
            uint32_t inc = v[k];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            const uint32_t c = c0 + k * 32 + lane;
            if (c < cps) h[(uint64_t)c * RADIX] = run + inc - v[k];
            run += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    if (lane == 0) hist[((uint64_t)nseg * cps + seg) * RADIX + d] = run;
}

template <typename K, typename P, int RANK>
static cudaError_t radix_chunked2(const K* in, K* out, const P* pin, P* pout, uint64_t n,
                                  int nseg, int shift, uint32_t dmask, uint32_t* hist,
                                  int target_ctas, cudaStream_t s, K omask = ~(K)0,
                                  int* nlaunch = nullptr) {
    uint64_t tiles = (n + RS2_TILE - 1) / RS2_TILE;
    uint64_t cps = std::max<uint64_t>(1, std::min<uint64_t>(tiles, (target_ctas + nseg - 1) / nseg));
    uint64_t L = (tiles + cps - 1) / cps * RS2_TILE;
    cps = (n + L - 1) / L;
    const unsigned grid = (unsigned)(cps * nseg);
    radix_hist_kernel<K><<<grid, RS_THREADS, 0, s>>>(in, n, (uint32_t)cps, L, shift, hist, dmask);
    // many chunks per segment (the trie's single-segment passes): one scan launch
    // instead of every CTA summing all of its segment's chunk rows
    const int prescan = cps > 128 ? 1 : 0;
    if (nlaunch) *nlaunch = 2 + prescan;
    if (prescan)
        hist_scan_kernel<<<(unsigned)(nseg * RADIX / 8), 256, 0, s>>>(hist, (uint32_t)cps,
                                                                      (uint32_t)nseg);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(radix_scatter2_kernel<K, P, RANK>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs2_smem<K, P>());
    radix_scatter2_kernel<K, P, RANK><<<grid, RS2_THREADS, rs2_smem<K, P>(), s>>>(
        in, out, pin, pout, n, (uint32_t)cps, L, shift, dmask, hist, omask, prescan);
    return cudaGetLastError();
}

// one stable pass of the mask trie (trie.cu): packed windows + sequence ids
// (a stable pass by the symbol at one kept position; omask = the mask's key bits on
// the leaf pass, all ones otherwise)
cudaError_t launch_trie_pass(const uint64_t* win, uint64_t* wout, const void* sin, void* sout,
                             bool seq16, uint64_t n, int shift, uint32_t dmask, uint64_t omask,
                             uint32_t* hist, int target_ctas, cudaStream_t s, int* nlaunch) {
    if (n == 0) return cudaGetLastError();
    if (seq16)
        return radix_chunked2<uint64_t, uint16_t, 0>(win, wout, (const uint16_t*)sin,
                                                     (uint16_t*)sout, n, 1, shift, dmask, hist,
                                                     target_ctas, s, omask, nlaunch);
    return radix_chunked2<uint64_t, uint32_t, 0>(win, wout, (const uint32_t*)sin, (uint32_t*)sout,
                                                 n, 1, shift, dmask, hist, target_ctas, s, omask,
                                                 nlaunch);
}

// One depth of the batched mask trie: nseg segments, segment s = a stable pass of
// n keys at in + desc[s].in_off by its digit (desc[s]: up to 4 symbols), written
// to out + desc[s].out_off (masked by desc[s].omask).
template <typename K>
static cudaError_t trie_batch(const K* in, K* out, uint64_t n, int nseg, const PassDesc* desc,
                              uint32_t* hist, int target_ctas, cudaStream_t s, int* nlaunch) {
    uint64_t tiles = (n + RS2_TILE - 1) / RS2_TILE;
    uint64_t cps = std::max<uint64_t>(1, std::min<uint64_t>(tiles, (target_ctas + nseg - 1) / nseg));
    uint64_t L = (tiles + cps - 1) / cps * RS2_TILE;
    cps = (n + L - 1) / L;
    const unsigned grid = (unsigned)(cps * nseg);
    radix_hist_kernel<K, true><<<grid, RS_THREADS, 0, s>>>(in, n, (uint32_t)cps, L, 0, hist, 0u,
                                                            desc);
    const int prescan = cps > 128 ? 1 : 0;
    if (prescan)
        hist_scan_kernel<<<(unsigned)(nseg * RADIX / 8), 256, 0, s>>>(hist, (uint32_t)cps,
                                                                      (uint32_t)nseg);
    if (nlaunch) *nlaunch = 2 + prescan;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cudaFuncSetAttribute(radix_scatter2_kernel<K, NoPay, 0, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs2_smem<K>());
    radix_scatter2_kernel<K, NoPay, 0, true><<<grid, RS2_THREADS, rs2_smem<K>(), s>>>(
        in, out, nullptr, nullptr, n, (uint32_t)cps, L, 0, 0xffu, hist, ~(K)0, prescan, desc);
    return cudaGetLastError();
}

cudaError_t launch_trie_batch(const void* in, void* out, bool k64, uint64_t n, int nseg,
                              const PassDesc* desc, uint32_t* hist, int target_ctas,
                              cudaStream_t s, int* nlaunch) {
    if (n == 0 || nseg == 0) return cudaGetLastError();
    if (k64)
        return trie_batch<uint64_t>((const uint64_t*)in, (uint64_t*)out, n, nseg, desc, hist,
                                    target_ctas, s, nlaunch);
    return trie_batch<uint32_t>((const uint32_t*)in, (uint32_t*)out, n, nseg, desc, hist,
                                target_ctas, s, nlaunch);
}

// trie root: composites (packed window << sb | sequence id) of every g-mer
template <typename K>
__global__ void trie_root_kernel(const uint64_t* __restrict__ win, const uint32_t* __restrict__ seq,
                                 uint64_t n, int sb, K* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (K)((win ? win[i] << sb : 0ull) | seq[i]);  // (no window: key 0)
}
cudaError_t launch_trie_root(const uint64_t* win, const uint32_t* seq, uint64_t n, int sb,
                             bool k64, void* out, int sm_count, cudaStream_t s) {
    if (n == 0) return cudaGetLastError();
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count * 8);
    if (k64)
        trie_root_kernel<uint64_t><<<(unsigned)blocks, 256, 0, s>>>(win, seq, n, sb, (uint64_t*)out);
    else
        trie_root_kernel<uint32_t><<<(unsigned)blocks, 256, 0, s>>>(win, seq, n, sb, (uint32_t*)out);
    return cudaGetLastError();
}

__global__ void seq16_kernel(const uint32_t* __restrict__ a, uint16_t* __restrict__ b,
                             uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = (uint16_t)a[i];
}
cudaError_t launch_seq16(const uint32_t* a, uint16_t* b, uint64_t n, int sm_count,
                         cudaStream_t s) {
    if (n == 0) return cudaGetLastError();
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count * 8);
    seq16_kernel<<<(unsigned)blocks, 256, 0, s>>>(a, b, n);
    return cudaGetLastError();
}

cudaError_t launch_radix_chunked2(const void* in, void* out, bool k64, uint64_t n, int nseg,
                                  int shift, uint32_t* hist, int target_ctas, int rank_mode,
                                  cudaStream_t s, int* nlaunch) {
    if (n == 0 || nseg == 0) return cudaGetLastError();
#define RS2_CASE(KT, R)                                                                  \
    if (rank_mode == R)                                                                  \
        return radix_chunked2<KT, NoPay, R>((const KT*)in, (KT*)out, nullptr, nullptr, n, nseg, \
                                            shift, 0xffu, hist, target_ctas, s, ~(KT)0,    \
                                            nlaunch);
    if (k64) {
        RS2_CASE(uint64_t, 1)
        RS2_CASE(uint64_t, 2)
        return radix_chunked2<uint64_t, NoPay, 0>((const uint64_t*)in, (uint64_t*)out, nullptr,
                                                  nullptr, n, nseg, shift, 0xffu, hist,
                                                  target_ctas, s, ~0ull, nlaunch);
    }
    RS2_CASE(uint32_t, 1)
    RS2_CASE(uint32_t, 2)
#undef RS2_CASE
    return radix_chunked2<uint32_t, NoPay, 0>((const uint32_t*)in, (uint32_t*)out, nullptr,
                                              nullptr, n, nseg, shift, 0xffu, hist, target_ctas,
                                              s, ~0u, nlaunch);
}

cudaError_t launch_radix_chunked(const void* in, void* out, bool k64, uint64_t n, int nseg,
                                 int shift, uint32_t* hist, int target_ctas, cudaStream_t s) {
    if (n == 0 || nseg == 0) return cudaGetLastError();
    if (k64)
        return radix_chunked<uint64_t>((const uint64_t*)in, (uint64_t*)out, n, nseg, shift, hist,
                                       target_ctas, s);
    return radix_chunked<uint32_t>((const uint32_t*)in, (uint32_t*)out, n, nseg, shift, hist,
                                   target_ctas, s);
}

}  // namespace gk
