// gram_tc.cu — heavy groups as a dense count Gram on the 5th-gen tensor cores:
// the one-SM u8 Gram (GAKCO_OPT_GRAM_PAIR 0; the default CTA-pair kernels are in
// gram2.cu), the dense-column builders (build_dense3 / build_dense2), the fill
// counters, and the TMA maps shared with gram2.cu.
//
// countAndUpdate adds c_X(key)*c_Y(key) to C_m(X,Y) for every
// pair of sequences sharing a key. For the R keys ("heavy groups", many
// sequences each) of a chunk this is exactly
//     C_m += D D^T,    D[X][r] = count of sequence X in group r  (u8),
// a dense contraction over r. It runs as tcgen05.mma.kind::i8 (u8 x u8 -> s32,
// exact) with D tiles brought in by TMA (128B swizzle, K-major) and the s32
// accumulators in TMEM; the epilogue adds them to the int64 C_m (entries with
// Y > X only: the diagonal is accounted for by the closed form + repeat term).
//
// Exactness: a chunk never spans more masks than (2^31-1)/n_max^2 (per mask an
// entry grows by at most n_X*n_Y), and counts > 255 are routed to the light
// path, so the s32 sums are exact and their int64 adds are exact.
//
// Kernel layout (one CTA per SM, persistent over output tiles 128 x 256):
//   warp 4      TMA producer (one elected lane), 4-stage smem ring
//   warp 5      MMA issuer (one elected lane), 2 TMEM accumulators of 256 cols
//   warps 0-3   epilogue: tcgen05.ld 32x32b -> +C (int64), lane = output row
#include <cuda.h>
#include <string.h>

#include <algorithm>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace gk {

constexpr int GT_M = 128;              // output rows per tile (TMEM lanes)
constexpr int GT_N = 256;              // output cols per tile (TMEM columns)
constexpr int GT_KB = 128;             // bytes (= u8 elements) of K per stage
constexpr int GT_STAGES = 4;
constexpr int GT_A_BYTES = GT_M * GT_KB;          // 16 KB
constexpr int GT_B_BYTES = GT_N * GT_KB;          // 32 KB
constexpr int GT_STAGE_BYTES = GT_A_BYTES + GT_B_BYTES;
constexpr int GT_THREADS = 192;
constexpr int GT_EC = 16;                          // epilogue columns per TMA reduce
constexpr int GT_EBUF = GT_M * GT_EC * 8;          // 16 KB staging (u64)
constexpr size_t GT_SMEM =
    (size_t)GT_STAGES * GT_STAGE_BYTES + 2 * GT_EBUF + 1024 /*align*/ + 256 /*barriers*/;

// Instruction descriptor: u8 x u8 -> s32, K-major A and B, M = 128, N = 256.
constexpr uint32_t GT_IDESC = (2u << 4)               // D format s32
                              | (0u << 7) | (0u << 10)  // A, B unsigned 8-bit
                              | ((uint32_t)(GT_N >> 3) << 17) | ((uint32_t)(GT_M >> 4) << 24);

struct GramArgs {
    int64_t* Cm;        // [N][N] int64, upper entries Y > X updated
    int64_t N;
    const uint32_t* fill;  // filled columns of D (K = fill rounded up to 128)
    uint32_t cap;          // columns of D (fill may overshoot; see light.cu)
    const int2* tiles;  // (row block of 128, col block of 256)
    int ntiles;
    int tma_epilogue;   // 1: TMA reduce-add into C (rows 16-byte aligned)
    int ksplit;         // K slices per output tile
    // window mode (wfill != nullptr): D rows are windows of 256 labels, tile (2w + r,
    // w) is rows r*128.. of window w against all its 256 rows, K = wfill[w] columns;
    // the output is the window's block of wC ([nw * 256][256] int64, local columns)
    const uint32_t* wfill;
};

__global__ void __launch_bounds__(GT_THREADS, 1)
    gram_kernel(const __grid_constant__ CUtensorMap dmap, const __grid_constant__ CUtensorMap cmap,
                GramArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* ebuf = smem + (size_t)GT_STAGES * GT_STAGE_BYTES;  // 2 x GT_EBUF
    uint64_t* bars = (uint64_t*)(ebuf + 2 * GT_EBUF);
    uint64_t* full = bars;                      // [STAGES]
    uint64_t* empty = bars + GT_STAGES;         // [STAGES]
    uint64_t* tfull = bars + 2 * GT_STAGES;     // [2]
    uint64_t* tempty = bars + 2 * GT_STAGES + 2;  // [2]
    uint32_t* tmem_slot = (uint32_t*)(bars + 2 * GT_STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool wmode = a.wfill != nullptr;
    const int kblocks0 = wmode ? 0 : (int)((min(*a.fill, a.cap) + GT_KB - 1) / GT_KB);
    if (!wmode && kblocks0 == 0) return;  // (grid-uniform)
    // K blocks of a tile: the flush's fill, or (window mode) its window's fill
    auto kblocks_of = [&](int2 tl) -> int {
        return wmode ? (int)((min(a.wfill[tl.y], a.cap) + GT_KB - 1) / GT_KB) : kblocks0;
    };
    const int kblocks = kblocks0;
    (void)kblocks;
    // work unit u = (tile u / ksplit, K slice u % ksplit): split-K keeps every SM
    // busy when there are few output tiles (small N); slices add up in C
    const int kper = (kblocks + a.ksplit - 1) / a.ksplit;
    const int nunits = a.ntiles * a.ksplit;
    if (threadIdx.x == 0) {
        for (int s = 0; s < GT_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 4) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&dmap) : "memory");
            uint32_t stage = 0, phase = 0;
            for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
                const int2 tl = a.tiles[u / a.ksplit];
                const int kbt = kblocks_of(tl);
                const int kpt = wmode ? kbt : kper;
                const int klo = (u % a.ksplit) * kpt, khi = min(kbt, klo + kpt);
                for (int kb = klo; kb < khi; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char* sa = smem + (size_t)stage * GT_STAGE_BYTES;
                    unsigned char* sbm = sa + GT_A_BYTES;
                    mbar_expect_tx(&full[stage], GT_STAGE_BYTES);
                    tma_load_3d(sa, &dmap, &full[stage], 0, tl.x * GT_M, kb);
                    tma_load_3d(sbm, &dmap, &full[stage], 0, tl.y * GT_N, kb);
                    tma_load_3d(sbm + GT_A_BYTES, &dmap, &full[stage], 0, tl.y * GT_N + GT_M, kb);
                    if (++stage == GT_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            int it = 0;
            for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
                const int kbt = kblocks_of(a.tiles[u / a.ksplit]);
                const int kpt = wmode ? kbt : kper;
                const int klo = (u % a.ksplit) * kpt, khi = min(kbt, klo + kpt);
                if (klo >= khi) continue;  // empty K slice: skipped by every role
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                ++it;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t dcol = tmem + acc * GT_N;
                for (int kb = klo; kb < khi; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + (size_t)stage * GT_STAGE_BYTES);
                    const uint32_t sbm = sa + GT_A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < GT_KB / 32; ++kk)
                        tc_mma_u8(dcol, sw128_desc(sa + kk * 32), sw128_desc(sbm + kk * 32),
                                  GT_IDESC, (kb != klo || kk != 0) ? 1u : 0u);
                    tc_commit(&empty[stage]);
                    if (++stage == GT_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit(&tfull[acc]);
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 0-3)
        // TMEM -> registers -> (s32 -> 64-bit, Y > X mask) -> smem [128][16] -> TMA
        // bulk reduce-add into C_m (coalesced, asynchronous, exact u64 adds).
        int it = 0, buf = 0;
        const int row = warp * 32 + lane;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int2 tl = a.tiles[u / a.ksplit];
            const int kbt = kblocks_of(tl);
            const int kpt = wmode ? kbt : kper;
            const int klo = (u % a.ksplit) * kpt, khi = min(kbt, klo + kpt);
            if (klo >= khi) continue;
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            ++it;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            // (window mode: local coordinates inside the window's 256 x 256 block)
            const int64_t x = wmode ? (int64_t)(tl.x - 2 * tl.y) * GT_M + row
                                    : (int64_t)tl.x * GT_M + row;
            const int64_t y0 = wmode ? 0 : (int64_t)tl.y * GT_N;
#pragma unroll 1
            for (int c = 0; c < GT_N; c += GT_EC) {
                uint32_t v[GT_EC];
                tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + acc * GT_N + c, v);
                // the buffer we are about to fill was handed to TMA two chunks ago
                if (threadIdx.x == 0) bulk_wait_read<1>();
                epi_bar();
                unsigned char* sb = ebuf + buf * GT_EBUF;
#pragma unroll
                for (int j2 = 0; j2 < GT_EC / 2; ++j2) {
                    const int ch = (j2 + lane) & (GT_EC / 2 - 1);
                    const int64_t y = y0 + c + 2 * ch;
                    uint64_t lo = (y > x) ? (uint64_t)v[2 * ch] : 0ull;
                    uint64_t hi = (y + 1 > x) ? (uint64_t)v[2 * ch + 1] : 0ull;
                    *(ulonglong2*)(sb + row * (GT_EC * 8) + ch * 16) = make_ulonglong2(lo, hi);
                }
                if (a.tma_epilogue) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    epi_bar();
                    if (threadIdx.x == 0) {
                        // (window mode: output row = the window's D row, column local)
                        tma_reduce_add_2d(&cmap, sb, (int)(y0 + c), (int)(tl.x * GT_M));
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                } else {
                    // rows of C not 16-byte aligned (odd N): coalesced LSU adds
                    epi_bar();
                    const uint64_t* s64 = (const uint64_t*)sb;
#pragma unroll 4
                    for (int e = threadIdx.x; e < GT_M * GT_EC; e += 128) {
                        const int64_t xx = (int64_t)tl.x * GT_M + e / GT_EC;  // (wC row)
                        const int64_t yy = y0 + c + e % GT_EC;
                        const uint64_t val = s64[e];
                        if (val && xx < a.N && yy < a.N)  // atomic: K slices share tiles
                            atomicAdd((unsigned long long*)&a.Cm[xx * a.N + yy], val);
                    }
                }
                buf ^= 1;
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
        }
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                     : "memory");
    }
}

// ---------------------------------------------------------------- D build
// Build v2: work item = one whole slab (128 columns) x BD2_ROWS rows, so every
// 128-byte line of D is written once, in full, by one CTA (16-byte stores). The
// slab is assembled in shared memory with 4-byte words XOR-swizzled by row (the
// scatter of one column over many rows then spreads over all banks). A group's
// triples are in ascending sequence order on the sort path (sorted = 1): a warp
// brackets the row range with one round of 32 samples and scans only that part;
// otherwise (hash grouping) it scans the whole group with a row filter.
constexpr int BD2_ROWS = 512;
constexpr int BD2_THREADS = 512;
constexpr size_t BD2_SMEM = (size_t)BD2_ROWS * GT_KB;  // 64 KB

__device__ __forceinline__ uint32_t bd2_off(uint32_t r, uint32_t cc) {
    return r * GT_KB + ((((cc >> 2) ^ (r & 31u)) << 2) | (cc & 3u));
}

// FP4 = true: e2m1 codes packed two per byte (slab = 256 columns = 128 bytes per row;
// count c in 1..4 -> code 2, 4, 5, 6; the light path keeps counts > 4).
__device__ __forceinline__ uint32_t e2m1_code(uint32_t c) {
    return c <= 2 ? 2 * c : c + 2;  // 0->0, 1->2 (1.0), 2->4 (2.0), 3->5 (3.0), 4->6 (4.0)
}

template <bool FP4>
__global__ void __launch_bounds__(BD2_THREADS) build_dense2_kernel(
    SegmentOut so, const uint2* __restrict__ heavy_list, const uint32_t* fill,
    uint8_t* __restrict__ D, int64_t n_pad, uint64_t ldd, int sorted) {
    extern __shared__ __align__(16) unsigned char sb[];  // [BD2_ROWS][128], swizzled words
    constexpr uint32_t SC = FP4 ? 2 * GT_KB : GT_KB;     // columns per slab
    const uint64_t f0 = fill[1];
    const uint64_t f1 = min((uint64_t)fill[0], ldd);
    if (f1 <= f0) return;
    const uint64_t s0 = f0 / SC, s1 = (f1 + SC - 1) / SC;
    const uint64_t nrc = (uint64_t)(n_pad + BD2_ROWS - 1) / BD2_ROWS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint64_t wk = blockIdx.x; wk < (s1 - s0) * nrc; wk += gridDim.x) {
        const uint64_t slab = s0 + wk / nrc;
        const uint32_t r0 = (uint32_t)(wk % nrc) * BD2_ROWS;
        const uint32_t rows = (uint32_t)min((int64_t)BD2_ROWS, n_pad - (int64_t)r0);
        for (uint32_t i = threadIdx.x; i < rows * (GT_KB / 16); i += BD2_THREADS)
            ((uint4*)sb)[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
        // warp w fills columns w + 16 j (j < 8) of each 128-column half; the 8
        // columns' loads are issued together at every step (one latency per step)
        constexpr int CPW = GT_KB / (BD2_THREADS / 32);  // 8 columns per warp per half
#pragma unroll 1
        for (uint32_t half = 0; half < SC / GT_KB; ++half) {
        uint32_t lo[CPW], hi[CPW];
        {
            const uint64_t col = slab * SC + half * GT_KB + warp + (BD2_THREADS / 32) * (lane & (CPW - 1));
            const uint2 bnd = (lane < CPW && col < f1) ? heavy_list[col] : make_uint2(0u, 0u);
#pragma unroll
            for (int j = 0; j < CPW; ++j) {
                lo[j] = __shfl_sync(0xffffffffu, bnd.x, j);
                hi[j] = __shfl_sync(0xffffffffu, bnd.y, j);
            }
        }
        if (sorted) {
            // one round of 32 samples per column brackets the rows [r0, r0 + rows)
            uint32_t xs[CPW];
#pragma unroll
            for (int j = 0; j < CPW; ++j) {
                const uint32_t len = hi[j] - lo[j];
                xs[j] = len > 64 ? so.tseq[lo[j] + (uint32_t)(((uint64_t)len * lane) >> 5)] & 0x7fffffffu
                                 : 0u;
            }
#pragma unroll
            for (int j = 0; j < CPW; ++j) {
                const uint32_t len = hi[j] - lo[j];
                if (len <= 64) continue;  // warp-uniform
                const uint32_t below = __ballot_sync(0xffffffffu, xs[j] < r0);
                const uint32_t inside = __ballot_sync(0xffffffffu, xs[j] < r0 + rows);
                const int lb = below ? 31 - __clz(below) : -1;
                const int ib = inside ? 31 - __clz(inside) : -1;
                const uint32_t nlo = lb < 0 ? lo[j] : lo[j] + (uint32_t)(((uint64_t)len * lb) >> 5);
                const uint32_t nhi =
                    ib == 31 ? hi[j] : lo[j] + (uint32_t)(((uint64_t)len * (ib + 1)) >> 5);
                lo[j] = nlo;
                hi[j] = ib < 0 ? nlo : nhi;
            }
        }
        uint32_t todo = 0;
#pragma unroll
        for (int j = 0; j < CPW; ++j) todo = max(todo, hi[j] - lo[j]);
        for (uint32_t o = lane; o < todo; o += 32) {
            uint32_t xv[CPW], cv[CPW];
#pragma unroll
            for (int j = 0; j < CPW; ++j) {
                const uint32_t t = lo[j] + o;
                xv[j] = t < hi[j] ? so.tseq[t] & 0x7fffffffu : 0xffffffffu;
                cv[j] = t < hi[j] ? so.tcnt[t] : 0u;
            }
#pragma unroll
            for (int j = 0; j < CPW; ++j)
                if (xv[j] >= r0 && xv[j] < r0 + rows) {
                    const uint32_t cc = half * GT_KB + warp + (BD2_THREADS / 32) * j;
                    if (FP4) {  // nibble cc & 1 of byte cc / 2 (a word is shared by 8 columns)
                        const uint32_t r = xv[j] - r0;
                        uint32_t* wp = (uint32_t*)(sb + r * GT_KB) + (((cc >> 3) ^ (r & 31u)));
                        atomicOr(wp, e2m1_code(cv[j]) << (((cc >> 1) & 3u) * 8 + (cc & 1u) * 4));
                    } else {
                        sb[bd2_off(xv[j] - r0, cc)] = (uint8_t)cv[j];
                    }
                }
        }
        }  // half
        __syncthreads();
        uint4* dst = (uint4*)(D + (slab * (uint64_t)n_pad + r0) * GT_KB);  // 128 B rows
        for (uint32_t i = threadIdx.x; i < rows * (GT_KB / 16); i += BD2_THREADS) {
            const uint32_t r = i >> 3, q = i & 7;
            const uint32_t* w = (const uint32_t*)(sb + r * GT_KB);
            uint4 v;
            v.x = w[(4 * q + 0) ^ (r & 31u)];
            v.y = w[(4 * q + 1) ^ (r & 31u)];
            v.z = w[(4 * q + 2) ^ (r & 31u)];
            v.w = w[(4 * q + 3) ^ (r & 31u)];
            dst[i] = v;
        }
        __syncthreads();
    }
}

// Build v3 (sorted triples, the sort path): one CTA per slab, walking its row
// chunks in order. Each warp owns SC/16 columns and keeps, per column, a cursor into
// the column's triples (ascending sequence): a row chunk consumes exactly the
// triples below its end, so every triple is read once and a chunk costs one round
// of loads for all the warp's columns (v2 re-brackets every (slab, chunk) item).
template <bool FP4>
__global__ void __launch_bounds__(BD2_THREADS, 3) build_dense3_kernel(
    SegmentOut so, const uint2* __restrict__ heavy_list, const uint32_t* fill,
    uint8_t* __restrict__ D, int64_t n_pad, uint64_t ldd) {
    extern __shared__ __align__(16) unsigned char sb[];  // [BD2_ROWS][128], swizzled words
    constexpr uint32_t SC = FP4 ? 2 * GT_KB : GT_KB;     // columns per slab
    constexpr int NW = BD2_THREADS / 32;
    constexpr int CPW = SC / NW;                         // columns per warp (16 or 8)
    const uint64_t f0 = fill[1];
    const uint64_t f1 = min((uint64_t)fill[0], ldd);
    if (f1 <= f0) return;
    const uint64_t s0 = f0 / SC, s1 = (f1 + SC - 1) / SC;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint64_t slab = s0 + blockIdx.x; slab < s1; slab += gridDim.x) {
        uint32_t cur[CPW], end[CPW];
        {
            const uint64_t col = slab * SC + warp + NW * (lane % CPW);
            const uint2 bnd = (lane < CPW && col < f1) ? heavy_list[col] : make_uint2(0u, 0u);
#pragma unroll
            for (int j = 0; j < CPW; ++j) {
                cur[j] = __shfl_sync(0xffffffffu, bnd.x, j);
                end[j] = __shfl_sync(0xffffffffu, bnd.y, j);
            }
        }
        for (int64_t r0 = 0; r0 < n_pad; r0 += BD2_ROWS) {
            const uint32_t rows = (uint32_t)min((int64_t)BD2_ROWS, n_pad - r0);
            const uint32_t rend = (uint32_t)r0 + rows;
            for (uint32_t i = threadIdx.x; i < rows * (GT_KB / 16); i += BD2_THREADS)
                ((uint4*)sb)[i] = make_uint4(0u, 0u, 0u, 0u);
            __syncthreads();
            bool more = true;
            while (more) {  // usually one round: a column rarely has > 32 triples per chunk
                uint32_t xv[CPW], cv[CPW];
#pragma unroll
                for (int j = 0; j < CPW; ++j) {
                    const uint32_t t = cur[j] + lane;
                    xv[j] = t < end[j] ? so.tseq[t] & 0x7fffffffu : 0xffffffffu;
                    cv[j] = t < end[j] ? so.tcnt[t] : 0u;
                }
                more = false;
#pragma unroll
                for (int j = 0; j < CPW; ++j) {
                    const bool in = xv[j] < rend;  // (>= r0: earlier triples were consumed)
                    if (in) {
                        const uint32_t cc = warp + NW * j;
                        const uint32_t r = xv[j] - (uint32_t)r0;
                        if (FP4) {
                            uint32_t* wp = (uint32_t*)(sb + r * GT_KB) + ((cc >> 3) ^ (r & 31u));
                            atomicOr(wp, e2m1_code(cv[j]) << (((cc >> 1) & 3u) * 8 + (cc & 1u) * 4));
                        } else {
                            sb[bd2_off(r, cc)] = (uint8_t)cv[j];
                        }
                    }
                    const uint32_t used = __popc(__ballot_sync(0xffffffffu, in));
                    cur[j] += used;
                    more |= used == 32 && cur[j] < end[j];
                }
            }
            __syncthreads();
            uint4* dst = (uint4*)(D + (slab * (uint64_t)n_pad + (uint64_t)r0) * GT_KB);
            for (uint32_t i = threadIdx.x; i < rows * (GT_KB / 16); i += BD2_THREADS) {
                const uint32_t r = i >> 3, q = i & 7;
                const uint32_t* w = (const uint32_t*)(sb + r * GT_KB);
                uint4 v;
                v.x = w[(4 * q + 0) ^ (r & 31u)];
                v.y = w[(4 * q + 1) ^ (r & 31u)];
                v.z = w[(4 * q + 2) ^ (r & 31u)];
                v.w = w[(4 * q + 3) ^ (r & 31u)];
                dst[i] = v;
            }
            __syncthreads();
        }
    }
}

// After a batch's build: fill rounded up to whole slabs (sc columns); the next batch
// starts there.
__global__ void fill_round_kernel(uint32_t* fill, uint64_t ldd, uint32_t sc) {
    uint64_t f = min((uint64_t)fill[0], ldd);
    f = min((f + sc - 1) / sc * sc, ldd);
    fill[0] = (uint32_t)f;
    fill[1] = (uint32_t)f;
}

// After a Gram flush: count the issued MACs (K rounded to sc columns) and reset the fill.
__global__ void fill_reset_kernel(uint32_t* fill, uint64_t ldd, uint64_t tile_macs,
                                  unsigned long long* stats, uint32_t sc, int e2m1) {
    const uint64_t k = (min((uint64_t)fill[0], ldd) + sc - 1) / sc * sc;
    atomicAdd(&stats[ST_HEAVY_MACS], (unsigned long long)(tile_macs * k));
    if (e2m1) atomicAdd(&stats[ST_HEAVY_MACS4], (unsigned long long)(tile_macs * k));
    fill[0] = 0;
    fill[1] = 0;
}

cudaError_t launch_build_dense(SegmentOut so, const uint2* heavy_list, uint32_t* dense_fill,
                               uint8_t* D, int64_t n_pad, uint64_t ldd, int sorted, int fp4,
                               int sm_count, cudaStream_t s) {
    if (sorted) {
        if (fp4) {
            cudaFuncSetAttribute(build_dense3_kernel<true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BD2_SMEM);
            build_dense3_kernel<true><<<sm_count * 3, BD2_THREADS, BD2_SMEM, s>>>(
                so, heavy_list, dense_fill, D, n_pad, ldd);
        } else {
            cudaFuncSetAttribute(build_dense3_kernel<false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BD2_SMEM);
            build_dense3_kernel<false><<<sm_count * 3, BD2_THREADS, BD2_SMEM, s>>>(
                so, heavy_list, dense_fill, D, n_pad, ldd);
        }
    } else if (fp4) {
        cudaFuncSetAttribute(build_dense2_kernel<true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BD2_SMEM);
        build_dense2_kernel<true><<<sm_count * 3, BD2_THREADS, BD2_SMEM, s>>>(
            so, heavy_list, dense_fill, D, n_pad, ldd, sorted);
    } else {
        cudaFuncSetAttribute(build_dense2_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BD2_SMEM);
        build_dense2_kernel<false><<<sm_count * 3, BD2_THREADS, BD2_SMEM, s>>>(
            so, heavy_list, dense_fill, D, n_pad, ldd, sorted);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    fill_round_kernel<<<1, 1, 0, s>>>(dense_fill, ldd, fp4 ? 2 * GT_KB : GT_KB);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// Upper tiles (row block of 128 x col block of 256) that hold any Y > X entry.
std::vector<int2> gram_tiles(int64_t n_pad) {
    std::vector<int2> t;
    const int rb = (int)(n_pad / GT_M), cb = (int)(n_pad / GT_N);
    for (int i = 0; i < rb; ++i)
        for (int j = 0; j < cb; ++j)
            if ((int64_t)j * GT_N + GT_N - 1 > (int64_t)i * GT_M) t.push_back(make_int2(i, j));
    return t;
}

// Tensor maps of a flush: D (u8 slabs [ldd/128][n_pad][128], box 128 B x 128 rows,
// 128B swizzle) and C_m (u64 view, box ec columns x 128 rows) for the TMA
// reduce-add epilogue; *tma_epi = 0 when C_m rows are not 16-byte aligned.
cudaError_t gram_maps(uint8_t* D, int64_t n_pad, uint64_t ldd, int64_t* Cm, int64_t nrows,
                      int64_t ncols, int ec, CUtensorMap* map, CUtensorMap* cmap, int* tma_epi) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return cudaErrorNotSupported;
    cuuint64_t dims[3] = {(cuuint64_t)GT_KB, (cuuint64_t)n_pad, ldd / GT_KB};
    cuuint64_t strides[2] = {(cuuint64_t)GT_KB, (cuuint64_t)n_pad * GT_KB};
    cuuint32_t box[3] = {GT_KB, GT_M, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)D, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    memset(cmap, 0, sizeof *cmap);
    *tma_epi = (ncols % 2 == 0) && (((uintptr_t)Cm & 15) == 0);
    cuuint64_t cdims[2] = {(cuuint64_t)ncols, (cuuint64_t)nrows};
    cuuint64_t cstr[1] = {(cuuint64_t)ncols * 8};
    cuuint32_t cbox[2] = {(cuuint32_t)ec, GT_M};
    if (*tma_epi) {
        r = enc(cmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, (void*)Cm, cdims, cstr, cbox, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    return cudaSuccess;
}

void launch_fill_reset(uint32_t* dense_fill, uint64_t ldd, uint64_t tile_macs,
                       unsigned long long* stats, cudaStream_t s) {
    fill_reset_kernel<<<1, 1, 0, s>>>(dense_fill, ldd, tile_macs, stats, GT_KB, 0);
}

void launch_fill_reset4(uint32_t* dense_fill, uint64_t ldd, uint64_t tile_macs,
                        unsigned long long* stats, cudaStream_t s) {
    fill_reset_kernel<<<1, 1, 0, s>>>(dense_fill, ldd, tile_macs, stats, 2 * GT_KB, 1);
}

cudaError_t launch_gram_flush(uint8_t* D, int64_t n_pad, uint64_t ldd, uint32_t* dense_fill,
                              int64_t* Cm, int64_t N, const int2* tiles, int ntiles,
                              int sm_count, unsigned long long* stats, cudaStream_t s) {
    CUtensorMap map, cmap;
    int tma_epi = 0;
    cudaError_t me = gram_maps(D, n_pad, ldd, Cm, N, N, GT_EC, &map, &cmap, &tma_epi);
    if (me != cudaSuccess) return me;
    cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GT_SMEM);
    // split K only as far as it fills the machine: the smallest split whose last
    // wave keeps >= 90% of the workers busy (one wave of whole-K tiles streams
    // each K slab of D from DRAM once, shared through L2 by all tiles)
    const int ksplit = gram_ksplit(ntiles, sm_count);
    GramArgs a{Cm, N, dense_fill, (uint32_t)ldd, tiles, ntiles, tma_epi ? 1 : 0, ksplit};
    int grid = ntiles * ksplit < sm_count ? ntiles * ksplit : sm_count;
    gram_kernel<<<grid, GT_THREADS, GT_SMEM, s>>>(map, cmap, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    fill_reset_kernel<<<1, 1, 0, s>>>(dense_fill, ldd, (uint64_t)ntiles * GT_M * GT_N, stats,
                                      GT_KB, 0);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- window Gram
// Window build: CTA (w, q) writes slabs q, q + WB_Q, ... of this batch's columns
// [wa.fill[nw + w], wa.fill[w]) of window w (the batch start is slab-aligned): 128
// columns x 256 rows of u8 counts assembled in shared memory (zeros elsewhere),
// stored as one contiguous 32 KB block of wD [slab][nw * 256][128]. A warp takes 8
// columns, their members gathered together (latency: list -> triple -> label). The
// tile's 4-byte words are XOR-swizzled by row (word w of row r at r * 32 + (w ^ (r &
// 31))): the lanes of a warp write one column at 32 different rows, which would
// otherwise all hit one bank; the copy-out un-swizzles.
constexpr int WB_Q = 16;
constexpr int WB_THREADS = 512;
constexpr int WB_CPW = GT_KB / (WB_THREADS / 32);  // columns per warp per slab (8)

__global__ void __launch_bounds__(WB_THREADS) window_build_kernel(SegmentOut so, WinArgs wa,
                                                                 const uint32_t* __restrict__ perm,
                                                                 uint8_t* __restrict__ wD) {
    __shared__ __align__(16) uint8_t tile[WIN_ROWS * GT_KB];  // [row][col], 32 KB
    const uint32_t w = blockIdx.x / WB_Q, q = blockIdx.x % WB_Q;
    const uint32_t c1 = min(wa.fill[w], wa.cap), c0 = min(wa.fill[wa.nw + w], c1);
    const uint32_t s0 = c0 / GT_KB, s1 = (c1 + GT_KB - 1) / GT_KB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lab0 = w * WIN_STEP;
    for (uint32_t sl = s0 + q; sl < s1; sl += WB_Q) {
        uint4* t4 = (uint4*)tile;
        for (int i = threadIdx.x; i < WIN_ROWS * GT_KB / 16; i += WB_THREADS) t4[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        uint2 g[WB_CPW];
#pragma unroll
        for (int jj = 0; jj < WB_CPW; ++jj) {
            const uint32_t col = sl * GT_KB + warp * WB_CPW + jj;
            g[jj] = col < c1 ? wa.list[(uint64_t)w * wa.cap + col] : make_uint2(0u, 0u);
        }
        // the first 32 members of all 8 columns: ids, then labels, loaded together (the
        // dependent id -> label loads were the latency, column after column); members
        // past 32 below
        uint32_t xm[WB_CPW], cm[WB_CPW];
#pragma unroll
        for (int jj = 0; jj < WB_CPW; ++jj) {
            const uint32_t t = g[jj].x + lane;
            const bool v = t < g[jj].y;
            xm[jj] = v ? so.tseq[t] & 0x7fffffffu : 0xffffffffu;
            cm[jj] = v ? so.tcnt[t] : 0u;
        }
#pragma unroll
        for (int jj = 0; jj < WB_CPW; ++jj) xm[jj] = xm[jj] != 0xffffffffu ? perm[xm[jj]] - lab0 : 0xffffffffu;
#pragma unroll
        for (int jj = 0; jj < WB_CPW; ++jj) {
            const int j = warp * WB_CPW + jj;
            const uint32_t r = xm[jj];
            if (r < (uint32_t)WIN_ROWS)  // (a split group: its members in this window)
                tile[r * GT_KB + ((((uint32_t)j >> 2) ^ (r & 31u)) << 2) + (j & 3)] = (uint8_t)cm[jj];
            for (uint32_t t = g[jj].x + 32 + lane; t < g[jj].y; t += 32) {
                const uint32_t r2 = perm[so.tseq[t] & 0x7fffffffu] - lab0;
                if (r2 < (uint32_t)WIN_ROWS)
                    tile[r2 * GT_KB + ((((uint32_t)j >> 2) ^ (r2 & 31u)) << 2) + (j & 3)] =
                        (uint8_t)so.tcnt[t];
            }
        }
        __syncthreads();
        uint4* dst = (uint4*)(wD + ((uint64_t)sl * wa.nw * WIN_ROWS + (uint64_t)w * WIN_ROWS) * GT_KB);
        const uint32_t* t1 = (const uint32_t*)tile;
        for (int i = threadIdx.x; i < WIN_ROWS * GT_KB / 16; i += WB_THREADS) {
            const uint32_t r = (uint32_t)i >> 3, w0 = ((uint32_t)i & 7u) * 4, sw = r & 31u;
            dst[i] = make_uint4(t1[r * 32 + ((w0 + 0) ^ sw)], t1[r * 32 + ((w0 + 1) ^ sw)],
                                t1[r * 32 + ((w0 + 2) ^ sw)], t1[r * 32 + ((w0 + 3) ^ sw)]);
        }
        __syncthreads();
    }
}

// after a build: the next batch starts at the next whole slab
__global__ void window_round_kernel(WinArgs wa) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < wa.nw; w += gridDim.x * blockDim.x) {
        const uint32_t f = min((min(wa.fill[w], wa.cap) + GT_KB - 1) / GT_KB * GT_KB, wa.cap);
        wa.fill[w] = f;
        wa.fill[wa.nw + w] = f;
    }
}

cudaError_t launch_window_build(SegmentOut so, WinArgs wa, const uint32_t* perm, uint8_t* wD,
                                int sm_count, cudaStream_t s) {
    (void)sm_count;
    if (wa.nw == 0) return cudaGetLastError();
    window_build_kernel<<<wa.nw * WB_Q, WB_THREADS, 0, s>>>(so, wa, perm, wD);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    window_round_kernel<<<(wa.nw + 255) / 256, 256, 0, s>>>(wa);
    return cudaGetLastError();
}

// MACs of a window flush (tiles of 128 x 256 over each window's columns), then the
// fills (and batch starts) are cleared
__global__ void window_reset_kernel(WinArgs wa, unsigned long long* stats) {
    unsigned long long macs = 0;
    for (uint32_t w = threadIdx.x; w < wa.nw; w += blockDim.x) {
        const uint32_t k = (min(wa.fill[w], wa.cap) + GT_KB - 1) / GT_KB * GT_KB;
        macs += (unsigned long long)k * 2 * GT_M * GT_N;
        wa.fill[w] = 0;
        wa.fill[wa.nw + w] = 0;
    }
    for (int o = 16; o > 0; o >>= 1) macs += __shfl_xor_sync(0xffffffffu, macs, o);
    if ((threadIdx.x & 31) == 0 && macs) atomicAdd(&stats[ST_WIN_MACS], macs);
}

cudaError_t launch_window_gram(uint8_t* wD, WinArgs wa, int64_t* wC, const int2* tiles,
                               int ntiles, int sm_count, unsigned long long* stats,
                               cudaStream_t s) {
    if (wa.nw == 0) return cudaGetLastError();
    CUtensorMap map, cmap;
    int tma_epi = 0;
    const int64_t rows = (int64_t)wa.nw * WIN_ROWS;
    cudaError_t me = gram_maps(wD, rows, wa.cap, wC, rows, WIN_ROWS, GT_EC, &map, &cmap, &tma_epi);
    if (me != cudaSuccess) return me;
    if (!tma_epi) return cudaErrorInvalidValue;  // (wC is 16-byte aligned, 256 columns)
    cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GT_SMEM);
    GramArgs a{wC, WIN_ROWS, nullptr, wa.cap, tiles, ntiles, 1, 1, wa.fill};
    const int grid = ntiles < sm_count ? ntiles : sm_count;
    gram_kernel<<<grid, GT_THREADS, GT_SMEM, s>>>(map, cmap, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    window_reset_kernel<<<1, 1024, 0, s>>>(wa, stats);
    return cudaGetLastError();
}

// C_m(X, Y) += wC entries (local row < local col), X, Y = the original sequences of
// the two labels (min, max: the upper triangle); wC is zeroed again.
__global__ void window_flush_kernel(int64_t* __restrict__ wC, uint32_t nw,
                                    const uint32_t* __restrict__ inv, int64_t N,
                                    int64_t* __restrict__ Cm) {
    const uint64_t total = (uint64_t)nw * WIN_ROWS * WIN_ROWS;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t v = wC[e];
        if (v == 0) continue;
        wC[e] = 0;
        const uint32_t w = (uint32_t)(e / (WIN_ROWS * WIN_ROWS));
        const uint32_t r = (uint32_t)(e / WIN_ROWS % WIN_ROWS), c = (uint32_t)(e % WIN_ROWS);
        const uint64_t lr = (uint64_t)w * WIN_STEP + r, lc = (uint64_t)w * WIN_STEP + c;
        if (lr >= (uint64_t)N || lc >= (uint64_t)N) continue;
        const uint32_t X = inv[lr], Y = inv[lc];
        const uint32_t lo = min(X, Y), hi = max(X, Y);
        atomicAdd((unsigned long long*)&Cm[(uint64_t)lo * N + hi], (unsigned long long)v);
    }
}

cudaError_t launch_window_flush(int64_t* wC, uint32_t nw, const uint32_t* inv, int64_t N,
                                int64_t* Cm, int sm_count, cudaStream_t s) {
    if (nw == 0) return cudaGetLastError();
    window_flush_kernel<<<sm_count * 8, 256, 0, s>>>(wC, nw, inv, N, Cm);
    return cudaGetLastError();
}

}  // namespace gk
