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
#include "internal.cuh"

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
    uint32_t& s_tile = s_w[8];

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
        uint32_t peers = __match_any_sync(0xffffffffu, d) & vmask;
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

}  // namespace gk
