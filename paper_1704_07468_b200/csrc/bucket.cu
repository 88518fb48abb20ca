// bucket.cu — grouping of masked g-mers by hash partition + shared-memory hash
// tables (GAKCO_OPT_SORT 2; the NEXT-4 ablation of SURVEY.md §8f against the LSD
// radix sort + run-length pass of radix.cu / segment.cu, which is the default:
// measured faster).
//
// What it computes is exactly what Algorithm 1 lines 13-15
// compute with removePosition -> sort -> countAndUpdate: for every mask, the groups
// of g-mers whose kept (g-m)-mers are equal, each group as its
// (sequence, count) triples. The paper sorts to bring equal (g-m)-mers together
// (a CPU design, Supp. §S:1.2 P:375-381); any total order groups identically
// (reading A9), and no order at all is needed to group: here a
// (g-m)-mer is sent to the hash bucket of its key (about 1024 keys per bucket),
// and one CTA groups a whole bucket in shared memory.
//
//   bk_count    keys recomputed on the fly from the packed g-mer windows; per
//               (mask, chunk of g-mers) a histogram over the nb buckets
//   bk_colscan  per (mask, bucket): exclusive prefix over chunks, bucket totals
//   bk_bscan    per mask: exclusive prefix over buckets -> bucket start offsets
//   bk_scatter  keys recomputed; each goes to start[bucket] + prefix + rank
//   bk_group    per bucket: key -> group slot (hash table 1), (slot, seq) ->
//               count (hash table 2), groups with >= 2 distinct sequences get
//               triple ranges (one atomicAdd per CTA), triples written out;
//               within-sequence repeats add c^2 - c to C_m(X,X) (reading A3)
//
// Keys: the g symbols of a g-mer are packed once into a 64-bit window w
// (bits = ceil(log2 sigma) per symbol). A mask's key is either the bit
// concatenation of its kept symbol fields (RUNS; injective because every code
// < 2^bits), or, when (g-m)*bits + sb > 64, the mixed-radix value
// sum_r code_r sigma^(g-m-1-r) (HORNER; the same integer as encode.cu's key).
// Either way equal keys <=> equal (g-m)-mers of one mask.
//
// The output is the SegmentOut of segment.cu: triples (seq, count) contiguous per
// group (sequence order within a group is arbitrary here), group triple ranges.
#include <algorithm>

#include "internal.cuh"

namespace gk {

// ---------------------------------------------------------------- windows
__global__ void window_kernel(CorpusView cv, int g, int bits, uint64_t* __restrict__ win) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < cv.n;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = cv.gm_seq[j];
        const uint8_t* p = cv.codes + cv.off[x] + ((int64_t)j - cv.gofs[x]);
        uint64_t w = 0;
        for (int r = 0; r < g; ++r) w = (w << bits) | p[r];
        win[j] = w;
    }
}

cudaError_t launch_windows(const CorpusView& cv, int g, int bits, uint64_t* win, int sm_count,
                           cudaStream_t s) {
    if (cv.n == 0) return cudaGetLastError();
    uint64_t blocks = (cv.n + 255) / 256;
    if (blocks > (uint64_t)sm_count * 16) blocks = (uint64_t)sm_count * 16;
    window_kernel<<<(unsigned)blocks, 256, 0, s>>>(cv, g, bits, win);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- keys
__device__ __forceinline__ uint64_t mask_key(uint64_t w, const MaskDesc& d, bool runs,
                                             uint32_t sigma, uint64_t symmask) {
    uint64_t k = 0;
    if (runs) {
        for (int r = 0; r < d.nrun; ++r)
            k |= ((w >> d.run_src[r]) & ((1ull << d.run_len[r]) - 1ull)) << d.run_dst[r];
    } else {
        for (int r = 0; r < d.nkept; ++r) k = k * sigma + ((w >> d.kept_sh[r]) & symmask);
    }
    return k;
}

__device__ __forceinline__ uint32_t bucket_of(uint64_t key, uint32_t nb) {
    const uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 32);
    return (uint32_t)(((uint64_t)h * nb) >> 32);
}

constexpr int BK_THREADS = 512;
constexpr int BK_ITEMS = 8;
constexpr int BK_SUB = BK_THREADS * BK_ITEMS;  // g-mers per sub-tile
static_assert(BK_SUB == BK_SUB_TILE, "sub-tile size shared with plan.cu");

// grid: (nchunks, ceil(nmask / MB)); smem: MaskDesc[MB] + u32 cnt[MB][nb]
// SCATTER = false: write the chunk's histogram rows H[(mask*nchunks + c)*nb + b]
// SCATTER = true : place every composite at mask*n + bbase[b] + H[...] + rank
template <typename K, bool SCATTER>
__global__ void __launch_bounds__(BK_THREADS) bk_pass_kernel(BkArgs a, K* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem[];
    MaskDesc* sd = (MaskDesc*)smem;
    uint32_t* cnt = (uint32_t*)(smem + sizeof(MaskDesc) * a.mb);
    const uint32_t c = blockIdx.x;
    const int m0 = blockIdx.y * a.mb;
    const int nm = min(a.mb, a.nmask - m0);
    const uint32_t nb = a.nb;
    for (int i = threadIdx.x; i < nm * (int)(sizeof(MaskDesc) / 4); i += BK_THREADS)
        ((uint32_t*)sd)[i] = ((const uint32_t*)(a.desc + m0))[i];
    for (uint32_t i = threadIdx.x; i < (uint32_t)nm * nb; i += BK_THREADS) {
        if (SCATTER) {
            const uint32_t mm = i / nb, b = i - mm * nb;
            const uint64_t m = (uint64_t)(m0 + mm);
            cnt[i] = a.bbase[m * (nb + 1) + b] + a.H[(m * a.nchunks + c) * nb + b];
        } else {
            cnt[i] = 0u;
        }
    }
    __syncthreads();
    const uint64_t j0 = (uint64_t)c * a.T;
    const uint64_t j1 = min(a.n, j0 + a.T);
    const uint64_t symmask = (1ull << a.bits) - 1ull;
    for (uint64_t s0 = j0; s0 < j1; s0 += BK_SUB) {
        uint64_t w[BK_ITEMS];
        uint32_t x[BK_ITEMS];
#pragma unroll
        for (int i = 0; i < BK_ITEMS; ++i) {
            const uint64_t j = s0 + (uint64_t)i * BK_THREADS + threadIdx.x;
            w[i] = j < j1 ? a.win[j] : 0ull;
            x[i] = j < j1 ? a.gm_seq[j] : 0xffffffffu;
        }
        for (int mm = 0; mm < nm; ++mm) {
            const MaskDesc& d = sd[mm];
            uint32_t* cm = cnt + (uint32_t)mm * nb;
            K* o = SCATTER ? out + (uint64_t)(m0 + mm) * a.n : nullptr;
#pragma unroll
            for (int i = 0; i < BK_ITEMS; ++i) {
                if (x[i] == 0xffffffffu) continue;
                const uint64_t key = mask_key(w[i], d, a.runs, a.sigma, symmask);
                const uint32_t b = bucket_of(key, nb);
                if (SCATTER) {
                    const uint32_t pos = atomicAdd(&cm[b], 1u);
                    o[pos] = (K)((key << a.sb) | x[i]);
                } else {
                    atomicAdd(&cm[b], 1u);
                }
            }
        }
    }
    if (!SCATTER) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < (uint32_t)nm * nb; i += BK_THREADS) {
            const uint32_t mm = i / nb, b = i - mm * nb;
            a.H[((uint64_t)(m0 + mm) * a.nchunks + c) * nb + b] = cnt[i];
        }
    }
}

// per (mask, bucket): exclusive prefix over chunks in place; bucket total
__global__ void bk_colscan_kernel(BkArgs a) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t m = blockIdx.y;
    if (b >= a.nb) return;
    uint32_t* col = a.H + m * a.nchunks * a.nb + b;
    uint32_t run = 0;
    uint32_t c = 0;
    for (; c + 8 <= a.nchunks; c += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = col[(uint64_t)(c + u) * a.nb];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            col[(uint64_t)(c + u) * a.nb] = run;
            run += v[u];
        }
    }
    for (; c < a.nchunks; ++c) {
        const uint32_t v = col[(uint64_t)c * a.nb];
        col[(uint64_t)c * a.nb] = run;
        run += v;
    }
    a.tot[m * a.nb + b] = run;
}

// generic exclusive block scan (blockDim.x multiple of 32, <= 1024)
__device__ __forceinline__ uint32_t block_scan_excl(uint32_t v, uint32_t* s_w, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    uint32_t wp = 0, tot = 0;
    for (int i = 0; i < nw; ++i) {
        const uint32_t t = s_w[i];
        wp += i < w ? t : 0u;
        tot += t;
    }
    *total = tot;
    __syncthreads();
    return wp + inc - v;
}

// per mask: bbase[m][b] = sum of totals of buckets < b; bbase[m][nb] = n
__global__ void __launch_bounds__(1024) bk_bscan_kernel(BkArgs a) {
    __shared__ uint32_t s_w[32];
    __shared__ uint32_t s_carry;
    const uint64_t m = blockIdx.x;
    const uint32_t* t = a.tot + m * a.nb;
    uint32_t* bb = a.bbase + m * (a.nb + 1);
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < a.nb; b0 += 1024) {
        const uint32_t b = b0 + threadIdx.x;
        const uint32_t v = b < a.nb ? t[b] : 0u;
        uint32_t tot;
        const uint32_t ex = block_scan_excl(v, s_w, &tot);
        const uint32_t carry = s_carry;
        if (b < a.nb) bb[b] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) bb[a.nb] = s_carry;
}

// ---------------------------------------------------------------- group
constexpr uint64_t EMPTY = ~0ull;
constexpr int CNT_BITS = 13;                   // smem triple entry: tag << 13 | count

// slot in [0, H) of a 64-bit value (H need not be a power of two)
__device__ __forceinline__ uint32_t slot_of(uint64_t v, uint32_t H) {
    v ^= v >> 31;
    v *= 0xD6E8FEB86659FD93ull;
    v ^= v >> 32;
    return (uint32_t)(((v & 0xffffffffull) * (uint64_t)H) >> 32);
}

// Per-CTA bookkeeping shared by the smem and the global-table paths: given the
// per-slot distinct-sequence counts gs[0..H), reserve the triple / group ranges
// of the groups with gs >= 2, write the group ranges, and turn gs into the
// per-group write cursor (0xffffffff for groups that are not emitted).
__device__ __forceinline__ void emit_groups(uint32_t* gs, uint32_t H, uint32_t* s_w,
                                            uint32_t* s_base, SegmentOut so,
                                            unsigned long long& n_t, unsigned long long& n_g) {
    const uint32_t per = (H + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(H, threadIdx.x * per), hi = min(H, lo + per);
    uint32_t nt = 0, ng = 0;
    for (uint32_t i = lo; i < hi; ++i) {
        const uint32_t s = gs[i];
        if (s >= 2) {
            nt += s;
            ++ng;
        }
    }
    uint32_t tt, tg;
    const uint32_t ot = block_scan_excl(nt, s_w, &tt);
    const uint32_t og = block_scan_excl(ng, s_w, &tg);
    if (threadIdx.x == 0) {
        s_base[0] = tt ? atomicAdd(&so.counts[0], tt) : 0u;
        s_base[1] = tg ? atomicAdd(&so.counts[1], tg) : 0u;
    }
    __syncthreads();
    uint32_t pt = s_base[0] + ot, pg = s_base[1] + og;
    for (uint32_t i = lo; i < hi; ++i) {
        const uint32_t s = gs[i];
        if (s >= 2) {
            so.groups[pg++] = make_uint2(pt, pt + s);
            gs[i] = pt;
            pt += s;
        } else {
            gs[i] = 0xffffffffu;
        }
    }
    n_t += tt;
    n_g += tg;
    __syncthreads();
}

// Global-table path for a bucket larger than GV_CAP (rare: skewed keys). Tables
// of H = 2c slots live in scratch at entry offset 2*start (the bucket's own
// region, disjoint from every other bucket's).
template <typename K>
__device__ void group_big(const K* keys, uint64_t start, uint32_t c, int sb, int64_t dstride,
                          int64_t* diag, SegmentOut so, BkScratch sc, uint32_t* s_w,
                          uint32_t* s_base, unsigned long long& n_t, unsigned long long& n_g) {
    const uint32_t H = 2u * c;
    uint64_t* tab = sc.tab + 2 * start;
    uint32_t* tcnt = sc.tcnt + 2 * start;
    uint32_t* gs = sc.gs + 2 * start;
    uint32_t* occ = sc.occ + start;
    const uint64_t seqmask = (1ull << sb) - 1ull;
    for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) {
        tab[i] = EMPTY;
        tcnt[i] = 0u;
        gs[i] = 0u;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
        const uint64_t key = (uint64_t)keys[start + i] >> sb;
        uint32_t h = slot_of(key, H);
        while (true) {
            const uint64_t v = *(volatile uint64_t*)&tab[h];
            if (v == key) break;
            if (v == EMPTY) {
                const uint64_t old = atomicCAS((unsigned long long*)&tab[h], EMPTY, key);
                if (old == EMPTY || old == key) break;
            }
            h = h + 1 == H ? 0 : h + 1;
        }
        occ[i] = h;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) tab[i] = EMPTY;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
        const uint32_t g = occ[i];
        const uint64_t tag = ((uint64_t)g << 32) | ((uint64_t)keys[start + i] & seqmask);
        uint32_t h = slot_of(tag, H);
        while (true) {
            uint64_t v = *(volatile uint64_t*)&tab[h];
            if (v == EMPTY) {
                v = atomicCAS((unsigned long long*)&tab[h], EMPTY, tag);
                if (v == EMPTY) {
                    atomicAdd(&tcnt[h], 1u);
                    atomicAdd(&gs[g], 1u);  // a new distinct sequence of group g
                    break;
                }
            }
            if (v == tag) {
                atomicAdd(&tcnt[h], 1u);
                break;
            }
            h = h + 1 == H ? 0 : h + 1;
        }
    }
    __syncthreads();
    emit_groups(gs, H, s_w, s_base, so, n_t, n_g);
    for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) {
        const uint64_t v = tab[i];
        if (v == EMPTY) continue;
        const uint32_t x = (uint32_t)(v & 0xffffffffull);
        const uint64_t cc = tcnt[i];
        if (cc >= 2)
            atomicAdd((unsigned long long*)&diag[(int64_t)x * dstride], (unsigned long long)(cc * cc - cc));
        const uint32_t g = (uint32_t)(v >> 32);
        if (*(volatile uint32_t*)&gs[g] == 0xffffffffu) continue;
        const uint32_t pos = atomicAdd(&gs[g], 1u);
        so.tseq[pos] = x;
        so.tcnt[pos] = (uint32_t)cc;
    }
    __syncthreads();
}

// One CTA per bucket (grid-stride over the batch's buckets). Shared memory:
// the bucket's composites, a table of H ~ 1.5c slots, per-slot group counters.
//   (1) key -> group slot g (table of keys); g kept per key;
//   (2) table reused for (g, seq) -> count; a new (g, seq) bumps gs[g], the
//       number of distinct sequences of group g;
//   (3) groups with gs >= 2 get CTA-local triple offsets and group indices
//       (warp-aggregated shared atomics), then one global reservation;
//   (4) one pass over the slots: group ranges out; every triple: repeats
//       c^2 - c on the diagonal, (seq, count) out at its group's cursor.
// gs packs (distinct seqs << 12 | cursor) after (3); GV_CAP < 4096.
constexpr int GV_THREADS = 256;
constexpr int GV_CAP = 2048;      // keys of a bucket grouped in smem (mean ~1024)
constexpr int GV_HMAX = GV_CAP * 3 / 2;
static_assert(GV_CAP < 4096 && GV_CAP < (1 << CNT_BITS), "12-bit cursor / group fields");
constexpr size_t GV_SMEM = (size_t)GV_HMAX * 8 + (size_t)GV_HMAX * 4 * 2 + (size_t)GV_CAP * 8 +
                           (size_t)GV_CAP * 2;

template <typename K>
__global__ void __launch_bounds__(GV_THREADS, 3) bk_group_kernel(
    const K* __restrict__ keys, BkArgs a, int64_t dstride, int64_t* diag, SegmentOut so,
    BkScratch sc, unsigned long long* stats) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* tab = (uint64_t*)smem;                                  // [GV_HMAX]
    uint32_t* gs = (uint32_t*)(tab + GV_HMAX);                        // [GV_HMAX]
    uint32_t* gl = gs + GV_HMAX;                                      // [GV_HMAX]
    K* kc = (K*)(gl + GV_HMAX);                                       // [GV_CAP]
    uint16_t* ks = (uint16_t*)((unsigned char*)(gl + GV_HMAX) + GV_CAP * 8);  // [GV_CAP]
    __shared__ uint32_t s_w[32];
    __shared__ uint32_t s_cnt[2], s_base[2];
    const int sb = a.sb;
    const int lane = threadIdx.x & 31;
    const uint64_t seqmask = (1ull << sb) - 1ull;
    const uint32_t nbt = (uint32_t)a.nmask * a.nb;
    const uint32_t lt = lanemask_lt();
    unsigned long long n_t = 0, n_g = 0;
    for (uint32_t wb = blockIdx.x; wb < nbt; wb += gridDim.x) {
        const uint32_t m = wb / a.nb, b = wb - m * a.nb;
        const uint32_t* bb = a.bbase + (uint64_t)m * (a.nb + 1);
        const uint32_t lo = bb[b], c = bb[b + 1] - lo;  // block-uniform
        if (c < 2) continue;  // one g-mer: count 1, no pair, no repeat
        const uint64_t start = (uint64_t)m * a.n + lo;
        if (c > (uint32_t)GV_CAP) {
            group_big<K>(keys, start, c, sb, dstride, diag, so, sc, s_w, s_base, n_t, n_g);
            continue;
        }
        const uint32_t H = max(64u, (3u * c / 2u + 31u) & ~31u);
        for (uint32_t i = threadIdx.x; i < c; i += GV_THREADS) kc[i] = keys[start + i];
        for (uint32_t i = threadIdx.x; i < H; i += GV_THREADS) {
            tab[i] = EMPTY;
            gs[i] = 0u;
        }
        if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0u;
        __syncthreads();
        // (1) key -> group slot
        for (uint32_t i = threadIdx.x; i < c; i += GV_THREADS) {
            const uint64_t key = (uint64_t)kc[i] >> sb;
            uint32_t h = slot_of(key, H);
            while (true) {
                const uint64_t v = *(volatile uint64_t*)&tab[h];
                if (v == key) break;
                if (v == EMPTY) {
                    const uint64_t old = atomicCAS((unsigned long long*)&tab[h], EMPTY, key);
                    if (old == EMPTY || old == key) break;
                }
                h = h + 1 == H ? 0 : h + 1;
            }
            ks[i] = (uint16_t)h;
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < H; i += GV_THREADS) tab[i] = EMPTY;
        __syncthreads();
        // (2) (group slot, seq) -> count: entry = tag << 13 | count
        for (uint32_t i = threadIdx.x; i < c; i += GV_THREADS) {
            const uint32_t g = ks[i];
            const uint64_t tag = ((uint64_t)g << 31) | ((uint64_t)kc[i] & seqmask);
            uint32_t h = slot_of(tag, H);
            while (true) {
                uint64_t v = *(volatile uint64_t*)&tab[h];
                if (v == EMPTY) {
                    v = atomicCAS((unsigned long long*)&tab[h], EMPTY, (tag << CNT_BITS) | 1ull);
                    if (v == EMPTY) {
                        atomicAdd(&gs[g], 1u);
                        break;
                    }
                }
                if ((v >> CNT_BITS) == tag) {
                    atomicAdd((unsigned long long*)&tab[h], 1ull);
                    break;
                }
                h = h + 1 == H ? 0 : h + 1;
            }
        }
        __syncthreads();
        // (3) CTA-local offsets of the multi-sequence groups (warp-aggregated)
        for (uint32_t i0 = 0; i0 < H; i0 += GV_THREADS) {
            const uint32_t i = i0 + threadIdx.x;
            const uint32_t s = i < H ? gs[i] : 0u;
            const bool em = s >= 2;
            const uint32_t bal = __ballot_sync(0xffffffffu, em);
            uint32_t inc = em ? s : 0u;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            const uint32_t wt = __shfl_sync(0xffffffffu, inc, 31);
            uint32_t bt = 0, bg = 0;
            if (lane == 0 && bal) {
                bt = atomicAdd(&s_cnt[0], wt);
                bg = atomicAdd(&s_cnt[1], (uint32_t)__popc(bal));
            }
            bt = __shfl_sync(0xffffffffu, bt, 0);
            bg = __shfl_sync(0xffffffffu, bg, 0);
            if (i < H) {
                if (em) {
                    const uint32_t off = bt + inc - s;
                    gs[i] = (s << 12) | off;
                    gl[i] = ((bg + (uint32_t)__popc(bal & lt)) << 12) | off;
                } else {
                    gs[i] = 0u;
                    gl[i] = 0xffffffffu;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t tt = s_cnt[0], tg = s_cnt[1];
            s_base[0] = tt ? atomicAdd(&so.counts[0], tt) : 0u;
            s_base[1] = tg ? atomicAdd(&so.counts[1], tg) : 0u;
            n_t += tt;
            n_g += tg;
        }
        __syncthreads();
        const uint32_t tb = s_base[0], gb = s_base[1];
        // (4) group ranges, diagonal repeats, triples
        for (uint32_t i = threadIdx.x; i < H; i += GV_THREADS) {
            const uint32_t q = gl[i];
            if (q != 0xffffffffu) {
                const uint32_t s = gs[i] >> 12, off = q & 0xfffu;
                so.groups[gb + (q >> 12)] = make_uint2(tb + off, tb + off + s);
            }
            const uint64_t v = tab[i];
            if (v == EMPTY) continue;
            const uint32_t cc = (uint32_t)(v & ((1ull << CNT_BITS) - 1ull));
            const uint32_t x = (uint32_t)((v >> CNT_BITS) & 0x7fffffffull);
            if (cc >= 2)
                atomicAdd((unsigned long long*)&diag[(int64_t)x * dstride],
                          (unsigned long long)cc * cc - cc);
            const uint32_t g = (uint32_t)(v >> (CNT_BITS + 31));
            if (gl[g] == 0xffffffffu) continue;
            const uint32_t pos = tb + (atomicAdd(&gs[g], 1u) & 0xfffu);
            so.tseq[pos] = x;
            so.tcnt[pos] = cc;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (n_t) atomicAdd(&stats[ST_TRIPLES], n_t);
        if (n_g) atomicAdd(&stats[ST_GROUPS], n_g);
    }
}

// ---------------------------------------------------------------- launchers
int bk_masks_per_cta(uint32_t nb) {
    // histogram rows of MB masks in shared memory: <= 24576 counters (96 KB)
    return (int)std::max<uint32_t>(1, std::min<uint32_t>(8, 24576 / std::max<uint32_t>(1, nb)));
}

template <typename K, bool SC>
static void set_pass_smem(size_t smem) {
    cudaFuncSetAttribute(bk_pass_kernel<K, SC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
}

cudaError_t launch_bucket_count(const BkArgs& a, bool k64, cudaStream_t s) {
    if (a.n == 0 || a.nmask == 0) return cudaGetLastError();
    const size_t smem = sizeof(MaskDesc) * a.mb + (size_t)a.mb * a.nb * 4;
    dim3 grid(a.nchunks, (a.nmask + a.mb - 1) / a.mb);
    if (k64) {
        set_pass_smem<uint64_t, false>(smem);
        bk_pass_kernel<uint64_t, false><<<grid, BK_THREADS, smem, s>>>(a, nullptr);
    } else {
        set_pass_smem<uint32_t, false>(smem);
        bk_pass_kernel<uint32_t, false><<<grid, BK_THREADS, smem, s>>>(a, nullptr);
    }
    return cudaGetLastError();
}

cudaError_t launch_bucket_scatter(const BkArgs& a, void* out, bool k64, cudaStream_t s) {
    if (a.n == 0 || a.nmask == 0) return cudaGetLastError();
    bk_colscan_kernel<<<dim3((a.nb + 255) / 256, a.nmask), 256, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    bk_bscan_kernel<<<a.nmask, 1024, 0, s>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(MaskDesc) * a.mb + (size_t)a.mb * a.nb * 4;
    dim3 grid(a.nchunks, (a.nmask + a.mb - 1) / a.mb);
    if (k64) {
        set_pass_smem<uint64_t, true>(smem);
        bk_pass_kernel<uint64_t, true><<<grid, BK_THREADS, smem, s>>>(a, (uint64_t*)out);
    } else {
        set_pass_smem<uint32_t, true>(smem);
        bk_pass_kernel<uint32_t, true><<<grid, BK_THREADS, smem, s>>>(a, (uint32_t*)out);
    }
    return cudaGetLastError();
}

cudaError_t launch_bucket_group(const BkArgs& a, const void* keys, bool k64, int64_t dstride,
                                int64_t* diag, SegmentOut so, BkScratch sc,
                                unsigned long long* stats, int sm_count, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(so.counts, 0, 2 * sizeof(uint32_t), s);
    if (e != cudaSuccess || a.n == 0 || a.nmask == 0) return e;
    const uint64_t nbt = (uint64_t)a.nmask * a.nb;
    const unsigned grid = (unsigned)std::min<uint64_t>(nbt, (uint64_t)sm_count * 3);
    if (k64) {
        cudaFuncSetAttribute(bk_group_kernel<uint64_t>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GV_SMEM);
        bk_group_kernel<uint64_t><<<grid, GV_THREADS, GV_SMEM, s>>>((const uint64_t*)keys, a, dstride,
                                                                     diag, so, sc, stats);
    } else {
        cudaFuncSetAttribute(bk_group_kernel<uint32_t>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GV_SMEM);
        bk_group_kernel<uint32_t><<<grid, GV_THREADS, GV_SMEM, s>>>((const uint32_t*)keys, a, dstride,
                                                                     diag, so, sc, stats);
    }
    return cudaGetLastError();
}

}  // namespace gk
