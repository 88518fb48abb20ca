// gram2.cu — heavy-group Gram C_m += D D^T on CTA pairs (tcgen05 cta_group::2).
//
// Same contraction as gram_tc.cu (countAndUpdate for groups shared by many
// sequences, as a dense u8 count Gram; exact in s32 / int64),
// laid out for the two SMs of a TPC working on one 256 x 512 output tile:
//   - the pair's MMA is M = 256 (rows split 128 / 128 between the CTAs' TMEM),
//     N = 256 per instruction, two N halves -> 512 accumulator columns = all of
//     each CTA's TMEM (one accumulator; the K loops of the heavy flushes are
//     thousands of stages long, the epilogue is not worth double-buffering);
//   - per 128-byte K stage each CTA loads its 128 A rows and its half (2 x 128
//     rows) of the 512 B rows: 48 KB, 384 B per K byte for 128 x 512 MACs per SM
//     (the 1-SM kernel moves 384 B for 128 x 256), so each SM pulls half the L2
//     bytes per MAC, and the MMA reads each smem operand byte once per pair.
// Roles (192 threads per CTA):
//   warp 4   TMA producer in both CTAs; the loads complete on the LEADER's full
//            barrier (cta_group::2 TMA), whose expect_tx counts both CTAs' bytes
//   warp 5   MMA issuer, leader CTA only; commits multicast to both CTAs (stage
//            free -> both producers; accumulator ready -> both epilogues)
//   warps 0-3 epilogue in both CTAs: TMEM -> registers (Y > X mask) -> smem ->
//            TMA bulk reduce-add into C_m; then a remote arrive on the leader's
//            accumulator-empty barrier
#include <string.h>

#include <algorithm>

#include "internal.cuh"
#include "tc_ptx.cuh"

namespace gk {

constexpr int G2_M = 128;                 // rows per CTA (TMEM lanes)
constexpr int G2_N = 256;                 // columns per MMA instruction
constexpr int G2_TN = 512;                // columns per pair tile (two N halves)
constexpr int G2_TM = 256;                // rows per pair tile
constexpr int G2_KB = 128;                // K bytes per stage
constexpr int G2_STAGES = 4;
constexpr int G2_A_BYTES = G2_M * G2_KB;          // 16 KB
constexpr int G2_BH_BYTES = 128 * G2_KB;          // 16 KB: one N half's 128 rows of this CTA
constexpr int G2_STAGE_BYTES = G2_A_BYTES + 2 * G2_BH_BYTES;  // 48 KB
constexpr int G2_THREADS = 192;
constexpr int G2_EC = 16;
constexpr int G2_EBUF = G2_M * G2_EC * 8;
constexpr size_t G2_SMEM =
    (size_t)G2_STAGES * G2_STAGE_BYTES + 2 * G2_EBUF + 1024 /*align*/ + 256 /*barriers*/;

// u8 x u8 -> s32, K-major A and B, M = 256 (pair), N = 256
constexpr uint32_t G2_IDESC = (2u << 4) | (0u << 7) | (0u << 10) |
                              ((uint32_t)(G2_N >> 3) << 17) | ((uint32_t)(G2_TM >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
// TMA load whose completion is signalled on an mbarrier that may live in the
// peer CTA of the pair (bar = shared::cluster address)
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar,
                                                 int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(bar), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void tc_mma_u8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive (once) on the barrier at the same smem offset in both CTAs of the pair
// when all prior tcgen05 ops of this thread have completed
__device__ __forceinline__ void tc_commit_pair(uint64_t* b) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(b)),
        "h"((uint16_t)3)
        : "memory");
}

struct Gram2Args {
    int64_t* Cm;        // [nrows][ncols]
    int64_t nrows, ncols;
    int64_t brow0;      // first row of D that is column 0 of the output (B operand)
    int rect;           // 1: rectangular block, every entry; 0: Y > X only
    const uint32_t* fill;
    uint32_t cap;
    const int2* tiles;  // (row block of 256, col block of 512)
    int ntiles;
    int tma_epilogue;
    int ksplit;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G2_THREADS, 1)
    gram2_kernel(const __grid_constant__ CUtensorMap dmap,
                 const __grid_constant__ CUtensorMap cmap, Gram2Args a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* ebuf = smem + (size_t)G2_STAGES * G2_STAGE_BYTES;
    uint64_t* bars = (uint64_t*)(ebuf + 2 * G2_EBUF);
    uint64_t* full = bars;                       // [STAGES] (leader's are used)
    uint64_t* empty = bars + G2_STAGES;          // [STAGES] (each CTA's own)
    uint64_t* tfull = bars + 2 * G2_STAGES;      // accumulator ready (each CTA)
    uint64_t* tempty = bars + 2 * G2_STAGES + 1; // accumulator drained (leader's)
    uint32_t* tmem_slot = (uint32_t*)(bars + 2 * G2_STAGES + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int kblocks = (int)((min(*a.fill, a.cap) + G2_KB - 1) / G2_KB);  // grid-uniform
    if (kblocks == 0) return;  // (both CTAs of every pair return together)
    const int kper = (kblocks + a.ksplit - 1) / a.ksplit;
    const int nunits = a.ntiles * a.ksplit;
    if (threadIdx.x == 0) {
        for (int s = 0; s < G2_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);  // 4 epilogue warps x 2 CTAs
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 4) {
        // ------------------------------------------------ TMA producer (both CTAs)
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&dmap) : "memory");
            uint32_t stage = 0, phase = 0;
            for (int u = pair; u < nunits; u += npairs) {
                const int2 tl = a.tiles[u / a.ksplit];
                const int klo = (u % a.ksplit) * kper, khi = min(kblocks, klo + kper);
                const int arow = tl.x * G2_TM + (int)rank * G2_M;
                const int b0 = (int)a.brow0 + tl.y * G2_TN + (int)rank * 128;  // N half 0
                for (int kb = klo; kb < khi; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char* sa = smem + (size_t)stage * G2_STAGE_BYTES;
                    const uint32_t fb = mapa_rank(smem_u32(&full[stage]), 0);
                    if (rank == 0) mbar_expect_tx(&full[stage], 2 * G2_STAGE_BYTES);
                    tma_load_3d_pair(sa, &dmap, fb, 0, arow, kb);
                    tma_load_3d_pair(sa + G2_A_BYTES, &dmap, fb, 0, b0, kb);
                    tma_load_3d_pair(sa + G2_A_BYTES + G2_BH_BYTES, &dmap, fb, 0, b0 + 256, kb);
                    if (++stage == G2_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------ MMA issuer (leader only)
        if (rank == 0 && lane == 0) {
            uint32_t stage = 0, phase = 0;
            int it = 0;
            for (int u = pair; u < nunits; u += npairs) {
                const int klo = (u % a.ksplit) * kper, khi = min(kblocks, klo + kper);
                if (klo >= khi) continue;  // empty K slice: skipped by every role
                mbar_wait(tempty, (it & 1) ^ 1);
                ++it;
                tc_fence_after();
                for (int kb = klo; kb < khi; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + (size_t)stage * G2_STAGE_BYTES);
                    const uint32_t sb0 = sa + G2_A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < G2_KB / 32; ++kk) {
                        const uint32_t acc = (kb != klo || kk != 0) ? 1u : 0u;
                        const uint64_t ad = sw128_desc(sa + kk * 32);
                        tc_mma_u8_pair(tmem, ad, sw128_desc(sb0 + kk * 32), G2_IDESC, acc);
                        tc_mma_u8_pair(tmem + G2_N, ad, sw128_desc(sb0 + G2_BH_BYTES + kk * 32),
                                       G2_IDESC, acc);
                    }
                    tc_commit_pair(&empty[stage]);
                    if (++stage == G2_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit_pair(tfull);
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 0-3, both CTAs)
        int it = 0, buf = 0;
        const int row = warp * 32 + lane;
        const uint32_t tempty_leader = mapa_rank(smem_u32(tempty), 0);
        for (int u = pair; u < nunits; u += npairs) {
            const int klo = (u % a.ksplit) * kper, khi = min(kblocks, klo + kper);
            if (klo >= khi) continue;
            const int2 tl = a.tiles[u / a.ksplit];
            mbar_wait(tfull, it & 1);
            ++it;
            tc_fence_after();
            const int64_t xrow0 = (int64_t)tl.x * G2_TM + (int64_t)rank * G2_M;
            const int64_t x = xrow0 + row;
            const int64_t y0 = (int64_t)tl.y * G2_TN;
#pragma unroll 1
            for (int c = 0; c < G2_TN; c += G2_EC) {
                // accumulator column c: N half c/256; within a half, columns 0..127
                // came from CTA 0's B rows and 128..255 from CTA 1's (= global order)
                uint32_t v[G2_EC];
                tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
                if (threadIdx.x == 0) bulk_wait_read<1>();
                epi_bar();
                unsigned char* sb = ebuf + buf * G2_EBUF;
#pragma unroll
                for (int j2 = 0; j2 < G2_EC / 2; ++j2) {
                    const int ch = (j2 + lane) & (G2_EC / 2 - 1);
                    const int64_t y = y0 + c + 2 * ch;
                    const uint64_t lo = (a.rect || y > x) ? (uint64_t)v[2 * ch] : 0ull;
                    const uint64_t hi = (a.rect || y + 1 > x) ? (uint64_t)v[2 * ch + 1] : 0ull;
                    *(ulonglong2*)(sb + row * (G2_EC * 8) + ch * 16) = make_ulonglong2(lo, hi);
                }
                if (a.tma_epilogue) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    epi_bar();
                    if (threadIdx.x == 0) {
                        tma_reduce_add_2d(&cmap, sb, (int)(y0 + c), (int)xrow0);
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                } else {
                    epi_bar();
                    const uint64_t* s64 = (const uint64_t*)sb;
#pragma unroll 4
                    for (int e = threadIdx.x; e < G2_M * G2_EC; e += 128) {
                        const int64_t xx = xrow0 + e / G2_EC;
                        const int64_t yy = y0 + c + e % G2_EC;
                        const uint64_t val = s64[e];
                        if (val && xx < a.nrows && yy < a.ncols)
                            atomicAdd((unsigned long long*)&a.Cm[xx * a.ncols + yy], val);
                    }
                }
                buf ^= 1;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader);
        }
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                     : "memory");
    }
}

// ============================================================================
// e2m1 variant (kind::mxf4, block-scaled, every scale factor 1.0): the same
// Gram with D held as packed 4-bit e2m1 counts (0,1,2,3,4 are exact: codes
// 0,2,4,5,6) — half the bytes of u8 and twice the MMA rate of kind::i8. The f32
// accumulator is exact while every sum stays below 2^24 (the host bounds the
// masks per flush by 2^24 / n_max^2). Pair tile 256 x 256 (one N half): TMEM
// columns [0,256) accumulate, [256,320) hold the E8M0 scale factors (all 0x7F =
// 2^0, written once; whatever byte / column the MMA picks, the scale is 1).
constexpr int G4_TN = 256;                 // columns per pair tile
constexpr int G4_STAGES = 6;
constexpr int G4_STAGE_BYTES = G2_A_BYTES + G2_BH_BYTES;  // 32 KB: A 128 rows + my 128 B rows
constexpr size_t G4_SMEM =
    (size_t)G4_STAGES * G4_STAGE_BYTES + 2 * G2_EBUF + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t G4_SF_COL = 256;        // first scale-factor column
constexpr int G4_SF_COLS = 64;
// block-scaled descriptor: a/b format E2M1 (MXF4Format = 1) at [7,10)/[10,13),
// K-major, N>>3 at [17,23), scale format E8M0 (bit 23), M>>4 at [24,29), sf ids 0
constexpr uint32_t G4_IDESC = (1u << 7) | (1u << 10) | ((uint32_t)(G2_N >> 3) << 17) |
                              (1u << 23) | ((uint32_t)(G2_TM >> 4) << 24);

__device__ __forceinline__ void tc_mma_mxf4_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t sfa, uint32_t sfb,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
        : "memory");
}
// 32 lanes x 8 columns of 32-bit words from registers (thread t -> lane base + t)
__device__ __forceinline__ void tmem_st8(uint32_t taddr, uint32_t v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(v)
        : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G2_THREADS, 1)
    gram4_kernel(const __grid_constant__ CUtensorMap dmap,
                 const __grid_constant__ CUtensorMap cmap, Gram2Args a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* ebuf = smem + (size_t)G4_STAGES * G4_STAGE_BYTES;
    uint64_t* bars = (uint64_t*)(ebuf + 2 * G2_EBUF);
    uint64_t* full = bars;
    uint64_t* empty = bars + G4_STAGES;
    uint64_t* tfull = bars + 2 * G4_STAGES;
    uint64_t* tempty = bars + 2 * G4_STAGES + 1;
    uint32_t* tmem_slot = (uint32_t*)(bars + 2 * G4_STAGES + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    // K blocks of 256 e2m1 columns (128 bytes per row)
    const int kblocks = (int)((min(*a.fill, a.cap) + 2 * G2_KB - 1) / (2 * G2_KB));
    if (kblocks == 0) return;
    const int kper = (kblocks + a.ksplit - 1) / a.ksplit;
    const int nunits = a.ntiles * a.ksplit;
    if (threadIdx.x == 0) {
        for (int s = 0; s < G4_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {  // scale factors: every byte 0x7F (E8M0 2^0), this CTA's 128 lanes
        for (int c = 0; c < G4_SF_COLS; c += 8)
            tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + G4_SF_COL + c, 0x7F7F7F7Fu);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t sfa = tmem + G4_SF_COL, sfb = tmem + G4_SF_COL + G4_SF_COLS / 2;

    if (warp == 4) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&dmap) : "memory");
            uint32_t stage = 0, phase = 0;
            for (int u = pair; u < nunits; u += npairs) {
                const int2 tl = a.tiles[u / a.ksplit];
                const int klo = (u % a.ksplit) * kper, khi = min(kblocks, klo + kper);
                const int arow = tl.x * G2_TM + (int)rank * G2_M;
                const int b0 = (int)a.brow0 + tl.y * G4_TN + (int)rank * 128;
                for (int kb = klo; kb < khi; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char* sa = smem + (size_t)stage * G4_STAGE_BYTES;
                    const uint32_t fb = mapa_rank(smem_u32(&full[stage]), 0);
                    if (rank == 0) mbar_expect_tx(&full[stage], 2 * G4_STAGE_BYTES);
                    tma_load_3d_pair(sa, &dmap, fb, 0, arow, kb);
                    tma_load_3d_pair(sa + G2_A_BYTES, &dmap, fb, 0, b0, kb);
                    if (++stage == G4_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 5) {
        if (rank == 0 && lane == 0) {
            uint32_t stage = 0, phase = 0;
            int it = 0;
            for (int u = pair; u < nunits; u += npairs) {
                const int klo = (u % a.ksplit) * kper, khi = min(kblocks, klo + kper);
                if (klo >= khi) continue;
                mbar_wait(tempty, (it & 1) ^ 1);
                ++it;
                tc_fence_after();
                for (int kb = klo; kb < khi; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + (size_t)stage * G4_STAGE_BYTES);
                    const uint32_t sb0 = sa + G2_A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < G2_KB / 32; ++kk)  // 64 e2m1 = 32 bytes per MMA
                        tc_mma_mxf4_pair(tmem, sw128_desc(sa + kk * 32), sw128_desc(sb0 + kk * 32),
                                         G4_IDESC, sfa, sfb, (kb != klo || kk != 0) ? 1u : 0u);
                    tc_commit_pair(&empty[stage]);
                    if (++stage == G4_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit_pair(tfull);
            }
        }
    } else {
        int it = 0, buf = 0;
        const int row = warp * 32 + lane;
        const uint32_t tempty_leader = mapa_rank(smem_u32(tempty), 0);
        for (int u = pair; u < nunits; u += npairs) {
            const int klo = (u % a.ksplit) * kper, khi = min(kblocks, klo + kper);
            if (klo >= khi) continue;
            const int2 tl = a.tiles[u / a.ksplit];
            mbar_wait(tfull, it & 1);
            ++it;
            tc_fence_after();
            const int64_t xrow0 = (int64_t)tl.x * G2_TM + (int64_t)rank * G2_M;
            const int64_t x = xrow0 + row;
            const int64_t y0 = (int64_t)tl.y * G4_TN;
#pragma unroll 1
            for (int c = 0; c < G4_TN; c += G2_EC) {
                uint32_t v[G2_EC];
                tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
                if (threadIdx.x == 0) bulk_wait_read<1>();
                epi_bar();
                unsigned char* sb = ebuf + buf * G2_EBUF;
#pragma unroll
                for (int j2 = 0; j2 < G2_EC / 2; ++j2) {
                    const int ch = (j2 + lane) & (G2_EC / 2 - 1);
                    const int64_t y = y0 + c + 2 * ch;
                    // exact integers < 2^24 in f32
                    const uint64_t f0 = (uint64_t)__uint_as_float(v[2 * ch]);
                    const uint64_t f1 = (uint64_t)__uint_as_float(v[2 * ch + 1]);
                    const uint64_t lo = (a.rect || y > x) ? f0 : 0ull;
                    const uint64_t hi = (a.rect || y + 1 > x) ? f1 : 0ull;
                    *(ulonglong2*)(sb + row * (G2_EC * 8) + ch * 16) = make_ulonglong2(lo, hi);
                }
                if (a.tma_epilogue) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    epi_bar();
                    if (threadIdx.x == 0) {
                        tma_reduce_add_2d(&cmap, sb, (int)(y0 + c), (int)xrow0);
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                } else {
                    epi_bar();
                    const uint64_t* s64 = (const uint64_t*)sb;
#pragma unroll 4
                    for (int e = threadIdx.x; e < G2_M * G2_EC; e += 128) {
                        const int64_t xx = xrow0 + e / G2_EC;
                        const int64_t yy = y0 + c + e % G2_EC;
                        const uint64_t val = s64[e];
                        if (val && xx < a.nrows && yy < a.ncols)
                            atomicAdd((unsigned long long*)&a.Cm[xx * a.ncols + yy], val);
                    }
                }
                buf ^= 1;
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader);
        }
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                     : "memory");
    }
}

std::vector<int2> gram4_tiles(int64_t n_pad) {
    std::vector<int2> t;
    const int rb = (int)(n_pad / G2_TM), cb = (int)(n_pad / G4_TN);
    for (int i = 0; i < rb; ++i)
        for (int j = 0; j < cb; ++j)
            if ((int64_t)j * G4_TN + G4_TN - 1 > (int64_t)i * G2_TM) t.push_back(make_int2(i, j));
    return t;
}

std::vector<int2> gram4_tiles_rect(int64_t NA, int64_t NB) {
    std::vector<int2> t;
    const int rb = (int)((NA + G2_TM - 1) / G2_TM), cb = (int)((NB + G4_TN - 1) / G4_TN);
    for (int i = 0; i < rb; ++i)
        for (int j = 0; j < cb; ++j) t.push_back(make_int2(i, j));
    return t;
}

// Upper pair tiles (row block of 256 x col block of 512) holding any Y > X entry.
std::vector<int2> gram2_tiles(int64_t n_pad) {
    std::vector<int2> t;
    const int rb = (int)(n_pad / G2_TM), cb = (int)(n_pad / G2_TN);
    for (int i = 0; i < rb; ++i)
        for (int j = 0; j < cb; ++j)
            if ((int64_t)j * G2_TN + G2_TN - 1 > (int64_t)i * G2_TM) t.push_back(make_int2(i, j));
    return t;
}

cudaError_t gram_maps(uint8_t* D, int64_t n_pad, uint64_t ldd, int64_t* Cm, int64_t nrows,
                      int64_t ncols, int ec, CUtensorMap* map, CUtensorMap* cmap, int* tma_epi);

// Rectangular block (rows [0, NA) x columns [NA, NA + NB) of D D^T): every pair tile.
std::vector<int2> gram2_tiles_rect(int64_t NA, int64_t NB) {
    std::vector<int2> t;
    const int rb = (int)((NA + G2_TM - 1) / G2_TM), cb = (int)((NB + G2_TN - 1) / G2_TN);
    for (int i = 0; i < rb; ++i)
        for (int j = 0; j < cb; ++j) t.push_back(make_int2(i, j));
    return t;
}
void launch_fill_reset(uint32_t* dense_fill, uint64_t ldd, uint64_t tile_macs,
                       unsigned long long* stats, cudaStream_t s);

cudaError_t launch_gram2_flush(uint8_t* D, int64_t n_pad, uint64_t ldd, uint32_t* dense_fill,
                               int64_t* Cm, int64_t N, const int2* tiles, int ntiles,
                               int sm_count, unsigned long long* stats, cudaStream_t s,
                               int64_t NA) {
    if (n_pad % G2_TN != 0) return cudaErrorInvalidValue;
    const bool rect = NA > 0;
    const int64_t nrows = rect ? NA : N, ncols = rect ? N - NA : N;
    CUtensorMap map, cmap;
    int tma_epi = 0;
    cudaError_t me = gram_maps(D, n_pad, ldd, Cm, nrows, ncols, G2_EC, &map, &cmap, &tma_epi);
    if (me != cudaSuccess) return me;
    cudaFuncSetAttribute(gram2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G2_SMEM);
    const int pairs = std::max(1, sm_count / 2);
    // split K only as far as it fills the machine: the smallest split whose last
    // wave keeps >= 90% of the workers busy (one wave of whole-K tiles streams
    // each K slab of D from DRAM once, shared through L2 by all tiles)
    const int ksplit = gram_ksplit(ntiles, pairs);
    Gram2Args a{Cm, nrows, ncols, rect ? NA : 0, rect ? 1 : 0, dense_fill, (uint32_t)ldd, tiles,
                ntiles, tma_epi, ksplit};
    const int units = ntiles * ksplit;
    const int grid = 2 * std::min(pairs, units);
    gram2_kernel<<<grid, G2_THREADS, G2_SMEM, s>>>(map, cmap, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    launch_fill_reset(dense_fill, ldd, (uint64_t)ntiles * G2_TM * G2_TN, stats, s);
    return cudaGetLastError();
}

}  // namespace gk

namespace gk {
void launch_fill_reset4(uint32_t* dense_fill, uint64_t ldd, uint64_t tile_macs,
                        unsigned long long* stats, cudaStream_t s);

cudaError_t launch_gram4_flush(uint8_t* D, int64_t n_pad, uint64_t ldd, uint32_t* dense_fill,
                               int64_t* Cm, int64_t N, const int2* tiles, int ntiles,
                               int sm_count, unsigned long long* stats, cudaStream_t s,
                               int64_t NA) {
    if (n_pad % G2_TN != 0) return cudaErrorInvalidValue;
    const bool rect = NA > 0;
    const int64_t nrows = rect ? NA : N, ncols = rect ? N - NA : N;
    CUtensorMap map, cmap;
    int tma_epi = 0;
    // ldd e2m1 columns = ldd/2 bytes per row: slabs of 256 columns (128 bytes)
    cudaError_t me = gram_maps(D, n_pad, ldd / 2, Cm, nrows, ncols, G2_EC, &map, &cmap, &tma_epi);
    if (me != cudaSuccess) return me;
    cudaFuncSetAttribute(gram4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G4_SMEM);
    const int pairs = std::max(1, sm_count / 2);
    const int ksplit = gram_ksplit(ntiles, pairs);
    Gram2Args a{Cm, nrows, ncols, rect ? NA : 0, rect ? 1 : 0, dense_fill, (uint32_t)ldd, tiles,
                ntiles, tma_epi, ksplit};
    const int units = ntiles * ksplit;
    const int grid = 2 * std::min(pairs, units);
    gram4_kernel<<<grid, G2_THREADS, G4_SMEM, s>>>(map, cmap, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    launch_fill_reset4(dense_fill, ldd, (uint64_t)ntiles * G2_TM * G4_TN, stats, s);
    return cudaGetLastError();
}
}  // namespace gk
