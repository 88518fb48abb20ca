// leaf.cu — a mask's last trie pass fused with its run-length (countAndUpdate, first
// half), for the mask trie and the cross-level chain.
//
// A mask S = P ∪ {x} (P: the kept positions of the pass before, x: the last one) groups
// its g-mers by (key under P, symbol at x). The input array is grouped by P (sorted
// by P's positions, or a compacted parent: each P-group whole and contiguous, its
// elements in sequence order). A stable sort of any range of WHOLE P-groups by the
// symbol at x leaves every S-group contiguous (bucket d of the range holds the
// elements of (P-group 1, d), then (P-group 2, d), ... each in order). So the last
// pass needs no global sort: CTA t loads the window [tT - 1, tT + 2T) of the input
// into shared memory once, owns the P-groups whose head lies in its tile [tT, tT + T),
// ranks that range (<= 2T elements) by the symbol at x, and runs the segment logic of
// segrag.cu on it directly: triples (seq |
// group-head << 31, count) of groups with >= 2 distinct sequences, their ranges,
// count^2 - count on C_m(X, X) for every repeated (key, seq) (reading A3), and
// optionally the compacted copy (groups of >= 2 elements) for the next level. The
// leaf array is never written or read back.
//
// A P-group running past the window (larger than T; at most one per tile: the last
// one) is split by its owner CTA chunk by chunk into the batch's overflow slot (a digit histogram of the
// group, then stable chunk ranks placed at the digit offsets); segrag.cu processes
// the overflow slots afterwards.
#include "internal.cuh"
#include "tc_ptx.cuh"

namespace gk {

namespace {

constexpr int LF_IT = 8;  // items per thread (12: the "wide" variant, see launch_leaf)
constexpr int LF_ND = 64;  // digit buckets (symbols < 64)

template <int TH, int IT = LF_IT>
struct Lf {
    static constexpr int WARPS = TH / 32;
    static constexpr int C = TH * IT;  // range capacity (shared memory)
    static constexpr int T = C / 4 * 3;   // tile of group heads per CTA (the rest: the
                                          // last group's tail)
};

__device__ __forceinline__ void lf_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct LfElem {
    uint64_t w;
    uint32_t s;
};

template <typename S, int TH, int IT>
constexpr size_t lf_smem() {
    // window keys [C + 8] (then the triple staging), ids [C + 24] (the 16-byte aligned
    // bulk-copy spans need the slack), perm [C] u16 (then
    // the group starts), warp digit counters + match masks, digit starts / counts /
    // offsets, scratch
    using L = Lf<TH, IT>;
    return (size_t)(L::C + 8) * 8 + (size_t)(L::C + 24) * sizeof(S) + (size_t)L::C * 4 +
           2 * L::WARPS * LF_ND * 4 + 3 * LF_ND * 4 + 64 * 4 + 64;
}

// exclusive scan over the TH threads of v (every thread must call); s_w: WARPS + 1 words
template <int TH>
__device__ __forceinline__ uint32_t lf_scan(uint32_t v, uint32_t* s_w, uint32_t* total) {
    constexpr int W = Lf<TH>::WARPS;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t x = lane < W ? s_w[lane] : 0u;
        uint32_t y = x;
#pragma unroll
        for (int o = 1; o < W; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += t;
        }
        if (lane < W) s_w[lane] = y - x;
        if (lane == W - 1) s_w[W] = y;
    }
    __syncthreads();
    const uint32_t r = s_w[w] + inc - v;
    *total = s_w[W];
    __syncthreads();
    return r;
}

// the same over 64-bit values; s_w: 2 (WARPS + 1) words
template <int TH>
__device__ __forceinline__ uint64_t lf_scan64(uint64_t v, unsigned long long* s_w, uint64_t* total) {
    constexpr int W = Lf<TH>::WARPS;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint64_t x = lane < W ? s_w[lane] : 0ull;
        uint64_t y = x;
#pragma unroll
        for (int o = 1; o < W; o <<= 1) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += t;
        }
        if (lane < W) s_w[lane] = y - x;
        if (lane == W - 1) s_w[W] = y;
    }
    __syncthreads();
    const uint64_t r = s_w[w] + inc - v;
    *total = s_w[W];
    __syncthreads();
    return r;
}

struct LfShared {
    uint64_t* sw;         // [C + 8] window keys
    uint16_t* perm;       // [C] source index (from the range start) by sorted position
    uint32_t* whist;      // [WARPS][ND]
    uint32_t* match;      // [WARPS][ND]
    uint32_t* cstart;     // [ND] range start of each digit
    uint32_t* tcnt;       // [ND] range count of each digit
    uint32_t* aux;        // [ND] (big group: running digit offsets)
    uint32_t* s_w;        // [64] scratch
};

// stable rank of sw[off, off + len) (len <= C) by digit (sw >> shift) & dmask:
// perm[p] = the source index (from off) of sorted position p; cstart / tcnt: each
// digit's start and count. Every thread must call it (it synchronises the block).
template <int TH, int IT>
__device__ __forceinline__ void lf_rank(const LfShared& sh, const uint64_t* keys, uint32_t off,
                                        uint32_t len, int shift, uint32_t dmask) {
    constexpr int W = Lf<TH>::WARPS;
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    uint32_t* whist = sh.whist + wp * LF_ND;
    uint32_t* mbin = sh.match + wp * LF_ND;
    const uint32_t lt = lanemask_lt();
    // each warp ranks a block of ipw * 32 consecutive elements (ipw = len / the block
    // width, rounded up: no warp idles through predicated-off items)
    const uint32_t ipw = (len + W * 32 - 1) / (W * 32);
    uint32_t dg[(IT + 3) / 4] = {}, rank[(IT + 1) / 2] = {};
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        if ((uint32_t)i >= ipw) break;  // (warp-uniform)
        const uint32_t idx = (uint32_t)(wp * ipw * 32 + i * 32 + lane);
        const bool valid = idx < len;
        const uint32_t d = valid ? (uint32_t)(keys[off + idx] >> shift) & dmask : 0u;
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
    __syncthreads();
    // digit totals, their exclusive scan (two warps), per-warp offsets
    uint32_t tot = 0;
    if (tid < LF_ND) {
#pragma unroll
        for (int ww = 0; ww < W; ++ww) tot += sh.whist[ww * LF_ND + tid];
    }
    uint32_t inc = tot;
    if (tid < LF_ND) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (tid == 31) sh.s_w[32] = inc;
    }
    __syncthreads();
    if (tid < LF_ND) {
        const uint32_t st = inc - tot + (tid >= 32 ? sh.s_w[32] : 0u);
        sh.cstart[tid] = st;
        sh.tcnt[tid] = tot;
        uint32_t sum = st;
#pragma unroll
        for (int ww = 0; ww < W; ++ww) {
            const uint32_t v = sh.whist[ww * LF_ND + tid];
            sh.whist[ww * LF_ND + tid] = sum;
            sum += v;
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        if ((uint32_t)i >= ipw) break;
        const uint32_t idx = (uint32_t)(wp * ipw * 32 + i * 32 + lane);
        if (idx < len) {
            const uint32_t d = (dg[i / 4] >> (8 * (i & 3))) & 0xffu;
            const uint32_t pos = whist[d] + ((rank[i / 2] >> (16 * (i & 1))) & 0xffffu);
            GK_CHECK(pos < len);
            sh.perm[pos] = (uint16_t)idx;
        }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < LF_ND / 32; ++j) whist[j * 32 + lane] = 0u;
    __syncthreads();
}

template <typename S, int TH, int IT>
__global__ void __launch_bounds__(TH, 1024 / TH) leaf_kernel(
    const uint64_t* __restrict__ w, const S* __restrict__ sq, const uint32_t* cntp, uint64_t n,
    uint64_t pmask, uint64_t kmask, int shift, uint32_t dmask, int64_t dstride, int64_t* diag,
    uint32_t* counters, SegmentOut so, unsigned long long* stats, uint64_t* cw, S* cs,
    uint32_t* ccnt, uint64_t* ow, S* os, uint32_t* ocnt, LfBigList bl) {
    using L = Lf<TH, IT>;
    constexpr int C = L::C, T = L::T, W = L::WARPS;
    extern __shared__ __align__(16) unsigned char smem[];
    pdl_wait();  // (no explicit trigger: the next grid launches as the CTAs exit)
    LfShared sh;
    sh.sw = (uint64_t*)smem;
    S* const ss = (S*)(smem + (size_t)(C + 8) * 8);
    sh.perm = (uint16_t*)(smem + (size_t)(C + 8) * 8 + (size_t)(C + 24) * sizeof(S));
    uint16_t* const s_kl = sh.perm + C;  // [C] sorted positions of the compacted elements
    sh.whist = (uint32_t*)(s_kl + C);
    sh.match = sh.whist + W * LF_ND;
    sh.cstart = sh.match + W * LF_ND;
    sh.tcnt = sh.cstart + LF_ND;
    sh.aux = sh.tcnt + LF_ND;
    sh.s_w = sh.aux + LF_ND;
    __shared__ uint32_t s_first, s_last, s_next;
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ unsigned long long s_end;
    __shared__ uint32_t s_wmin[W], s_base_t, s_base_g, s_base_c, s_obase;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t cnt = cntp ? min((uint64_t)*cntp, n) : n;
    const uint64_t t0 = (uint64_t)blockIdx.x * T;
    if (t0 >= cnt) return;  // (block-uniform)
    const uint64_t t1 = min(t0 + T, cnt);

    for (int i = tid; i < 2 * W * LF_ND; i += TH) sh.whist[i] = 0u;
    if (tid == 0) {
        s_first = 0xffffffffu;
        s_last = 0u;
        s_next = 0xffffffffu;
        s_end = ~0ull;
    }
    // 1. the window [t0 - 1, t0 + C) of the input (local index l = global - t0 + 1) into
    //    shared memory by two bulk copies (16-byte aligned spans; SW / SS address it by
    //    local index)
    const uint64_t wend = min(t0 + C, cnt);
    const uint32_t wl = (uint32_t)(wend - t0);  // window elements after t0 - 1
    const uint64_t gb = t0 ? t0 - 1 : 0;        // first element copied
    const uint32_t lgb = t0 ? 0u : 1u;          // its local index
    const uintptr_t aw0 = (uintptr_t)(w + gb) & ~(uintptr_t)15, aw1 = ((uintptr_t)(w + wend) + 15) & ~(uintptr_t)15;
    const uintptr_t as0 = (uintptr_t)(sq + gb) & ~(uintptr_t)15, as1 = ((uintptr_t)(sq + wend) + 15) & ~(uintptr_t)15;
    const uint64_t* SW = sh.sw + (int)(((uintptr_t)(w + gb) - aw0) / 8) - (int)lgb;
    const S* SS = ss + (int)(((uintptr_t)(sq + gb) - as0) / sizeof(S)) - (int)lgb;
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(&s_bar, (uint32_t)(aw1 - aw0) + (uint32_t)(as1 - as0));
        lf_bulk(sh.sw, (const void*)aw0, (uint32_t)(aw1 - aw0), &s_bar);
        lf_bulk(ss, (const void*)as0, (uint32_t)(as1 - as0), &s_bar);
    }
    __syncthreads();  // (the barrier initialised)
    mbar_wait(&s_bar, 0);
    // 2. group heads: the first and the last in the tile (the owned range starts at the
    //    first), the first after the tile (the owned range ends there)
    {
        const uint32_t lt1 = (uint32_t)(t1 - t0) + 1;
        uint32_t fmin = 0xffffffffu, lmax = 0u, nmin = 0xffffffffu;
        for (uint32_t l = 1 + tid; l <= wl; l += TH) {
            const bool h = (l == 1 && t0 == 0) || ((SW[l] ^ SW[l - 1]) & pmask) != 0;
            if (h) {
                if (l < lt1) {
                    fmin = min(fmin, l);
                    lmax = max(lmax, l);
                } else {
                    nmin = min(nmin, l);
                }
            }
        }
        fmin = __reduce_min_sync(0xffffffffu, fmin);
        lmax = __reduce_max_sync(0xffffffffu, lmax);
        nmin = __reduce_min_sync(0xffffffffu, nmin);
        if (lane == 0) {
            if (fmin != 0xffffffffu) {
                atomicMin(&s_first, fmin);
                atomicMax(&s_last, lmax);
            }
            if (nmin != 0xffffffffu) atomicMin(&s_next, nmin);
        }
    }
    __syncthreads();
    const uint32_t a0l = s_first;
    if (a0l == 0xffffffffu) return;  // no group starts here (block-uniform)
    const uint32_t hll = s_last;
    // the owned range ends at the next head, or at the array end; with neither within
    // the window capacity, the last group runs past it (big)
    const bool big = s_next == 0xffffffffu && t0 + wl < cnt;
    const uint32_t el = s_next != 0xffffffffu ? s_next : wl + 1;
    const uint32_t m = big ? hll : el;
    const uint32_t len = m - a0l;
    GK_CHECK(len <= (uint32_t)C);

    // 3. the range of whole groups: ranked by digit x, then the segment logic
    if (len > 0) {  // (block-uniform)
        lf_rank<TH, IT>(sh, SW, a0l, len, shift, dmask);
        // thread tid owns sorted positions [tid * ipt, tid * ipt + ipt), ipt = len / TH
        // rounded up (<= IT): every thread has items
        const uint32_t ipt = (len + TH - 1) / TH;
        const uint32_t lbase = (uint32_t)tid * ipt;
        auto elem = [&](uint32_t p) -> LfElem {
            const uint32_t l = a0l + sh.perm[p];
            return LfElem{SW[l], (uint32_t)SS[l]};
        };
        auto geq = [&](const LfElem& x, const LfElem& y) { return ((x.w ^ y.w) & kmask) == 0; };
        LfElem cur[IT];
        uint32_t th_bits = 0, gh_bits = 0, valid_bits = 0;
        {
            LfElem prev = (lbase > 0 && lbase < len) ? elem(lbase - 1) : LfElem{0ull, 0u};
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                cur[i] = LfElem{0ull, 0u};
                if ((uint32_t)i >= ipt) continue;  // (block-uniform)
                const uint32_t p = lbase + i;
                cur[i] = p < len ? elem(p) : LfElem{0ull, 0u};
                if (p < len) {
                    valid_bits |= 1u << i;
                    const bool g = p == 0 || !geq(prev, cur[i]);
                    if (g) gh_bits |= 1u << i;
                    if (g || prev.s != cur[i].s) th_bits |= 1u << i;
                }
                prev = cur[i];
            }
        }
        // the first triple head after this thread's items (pos << 1 | group head); the
        // range end counts as a group head
        uint32_t mine = 0xffffffffu;
        if (th_bits) {
            const int f = __ffs(th_bits) - 1;
            mine = (lbase + f) << 1 | ((gh_bits >> f) & 1u);
        }
        uint32_t suf = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_down_sync(0xffffffffu, suf, o);
            if (lane + o < 32) suf = min(suf, v);
        }
        if (lane == 0) s_wmin[warp] = suf;
        __syncthreads();
        uint32_t nxt = __shfl_down_sync(0xffffffffu, suf, 1);
        if (lane == 31) nxt = 0xffffffffu;
        {
            uint32_t later = len << 1 | 1u;
#pragma unroll
            for (int ww = 1; ww < W; ++ww)
                if (ww > warp) later = min(later, s_wmin[ww]);
            nxt = min(nxt, later);
        }
        // ghn bit i: is the element after item i a group head? (the keep rule)
        uint32_t ghn = gh_bits >> 1;
        if (valid_bits) {
            const int ib = __popc(valid_bits) - 1;
            ghn &= ~(1u << ib);
            if ((nxt >> 1) == lbase + ib + 1 && (nxt & 1u)) ghn |= 1u << ib;
        }
        // backward: run lengths, groups of >= 2 triples, the diagonal repeat term
        uint32_t multi_bits = 0;
        uint32_t cntv[IT];
#pragma unroll
        for (int i = IT - 1; i >= 0; --i) {
            cntv[i] = 0;
            if (!((th_bits >> i) & 1u)) continue;
            const uint32_t li = lbase + i;
            const uint32_t c = (nxt >> 1) - li;
            cntv[i] = c;
            const uint32_t gh = (gh_bits >> i) & 1u;
            if (!gh || !(nxt & 1u)) multi_bits |= 1u << i;
            if (c >= 2)
                atomicAdd((unsigned long long*)&diag[(int64_t)cur[i].s * dstride],
                          (unsigned long long)c * c - c);
            nxt = li << 1 | gh;
        }
        const uint32_t emit_t = th_bits & multi_bits;
        const uint32_t emit_g = emit_t & gh_bits;
        uint32_t keep = 0;
        if (cw) keep = valid_bits & (~gh_bits | ~ghn) & ((1u << IT) - 1u);
        // one block scan of the three counts (16-bit fields: each total <= C = 4 * 256)
        uint64_t aggp;
        const uint64_t offp = lf_scan64<TH>((uint64_t)__popc(emit_t) | (uint64_t)__popc(emit_g) << 16 |
                                                (uint64_t)__popc(keep) << 32,
                                            (unsigned long long*)sh.s_w, &aggp);
        const uint32_t off_t = (uint32_t)offp & 0xffffu, off_g = (uint32_t)(offp >> 16) & 0xffffu;
        const uint32_t agg_t = (uint32_t)aggp & 0xffffu, agg_g = (uint32_t)(aggp >> 16) & 0xffffu;
        const uint32_t off_k = (uint32_t)(offp >> 32), agg_k = (uint32_t)(aggp >> 32);
        if (tid == 0) {
            s_base_t = agg_t ? atomicAdd(&counters[0], agg_t) : 0u;
            s_base_g = agg_g ? atomicAdd(&counters[1], agg_g) : 0u;
            if (cw) s_base_c = agg_k ? atomicAdd(ccnt, agg_k) : 0u;
            if (agg_t) atomicAdd(&stats[ST_TRIPLES], (unsigned long long)agg_t);
            if (agg_g) atomicAdd(&stats[ST_GROUPS], (unsigned long long)agg_g);
        }
        // the compacted elements' sorted positions, in order (their copy below is
        // coalesced: consecutive threads, consecutive outputs)
        if (cw) {
            uint32_t k = off_k;
#pragma unroll
            for (int i = 0; i < IT; ++i)
                if (keep & (1u << i)) s_kl[k++] = (uint16_t)(lbase + i);
        }
        __syncthreads();
        const uint32_t base_t = s_base_t, base_g = s_base_g;
        // compacted elements (groups of >= 2 elements), in sorted order
        if (cw) {
            const uint32_t bc = s_base_c;
            for (uint32_t j = tid; j < agg_k; j += TH) {
                GK_CHECK(bc + j < n);
                const uint32_t l = a0l + sh.perm[s_kl[j]];
                cw[bc + j] = SW[l];
                cs[bc + j] = SS[l];
            }
            __syncthreads();  // (every read of the window / perm done: staging below)
        }
        // triples staged in shared memory (the window), written coalesced; group ranges
        uint32_t* s_tx = (uint32_t*)sh.sw;
        uint32_t* s_tc = s_tx + C;
        uint16_t* s_gpos = sh.perm;
        uint32_t li = off_t, gl = off_g;
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            if (emit_t & (1u << i)) {
                s_tx[li] = cur[i].s | (((gh_bits >> i) & 1u) << 31);
                s_tc[li] = cntv[i];
                if (emit_g & (1u << i)) s_gpos[gl++] = (uint16_t)li;
                ++li;
            }
        }
        __syncthreads();
        for (uint32_t j = tid; j < agg_t; j += TH) {
            so.tseq[base_t + j] = s_tx[j];
            so.tcnt[base_t + j] = s_tc[j];
        }
        for (uint32_t gg = tid; gg < agg_g; gg += TH)
            so.groups[base_g + gg] =
                make_uint2(base_t + s_gpos[gg], gg + 1 < agg_g ? base_t + s_gpos[gg + 1] : base_t + agg_t);
        __syncthreads();  // (shared memory reused below)
    }

    // 4. a group running past the window [hl, e): split by digit x into the overflow slot
    if (big && bl.e) {  // (queued for leaf_big_kernel: one large CTA per group)
        if (tid == 0) {
            const uint32_t q = atomicAdd(&bl.count[0], 1u);
            GK_CHECK(q < bl.cap);
            if (q < bl.cap)
                bl.e[q] = LfBig{w, (const void*)sq, ow, (void*)os, ocnt, t0 + hll - 1, cnt, pmask,
                                shift, dmask};
        }
        return;
    }
    if (big) {  // (block-uniform; no queue: split here)
        const uint64_t hl = t0 + hll - 1;
        for (uint64_t e0 = wend; e0 < cnt; e0 += TH) {
            const uint64_t i = e0 + tid;
            if (i < cnt && ((w[i] ^ w[i - 1]) & pmask) != 0) atomicMin(&s_end, (unsigned long long)i);
            __syncthreads();
            const bool found = s_end != ~0ull;
            __syncthreads();  // (every thread has read s_end before the next round's atomics)
            if (found) break;
        }
        const uint64_t e = min((uint64_t)s_end, cnt);
        const uint64_t gs = e - hl;
        // digit histogram of the group (per-warp counters), exclusive digit offsets
        for (uint64_t i = hl + tid; i < e; i += TH)
            atomicAdd(&sh.whist[warp * LF_ND + ((uint32_t)(w[i] >> shift) & dmask)], 1u);
        __syncthreads();
        if (tid < LF_ND) {
            uint32_t t = 0;
#pragma unroll
            for (int ww = 0; ww < W; ++ww) {
                t += sh.whist[ww * LF_ND + tid];
                sh.whist[ww * LF_ND + tid] = 0u;
            }
            uint32_t inc = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            if (tid == 31) sh.s_w[32] = inc;
            sh.aux[tid] = inc - t;  // (the upper half adds the lower total below)
        }
        if (tid == 0) s_obase = atomicAdd(ocnt, (uint32_t)gs);
        __syncthreads();
        if (tid >= 32 && tid < LF_ND) sh.aux[tid] += sh.s_w[32];
        __syncthreads();
        const uint32_t ob = s_obase;
        GK_CHECK((uint64_t)ob + gs <= n);
        for (uint64_t c0 = hl; c0 < e; c0 += C) {
            const uint32_t cl = (uint32_t)min((uint64_t)C, e - c0);
            for (uint32_t l = tid; l < cl; l += TH) {
                sh.sw[l] = w[c0 + l];
                ss[l] = sq[c0 + l];
            }
            __syncthreads();
            lf_rank<TH, IT>(sh, sh.sw, 0, cl, shift, dmask);
            for (uint32_t p = tid; p < cl; p += TH) {
                const uint32_t l = sh.perm[p];
                const uint64_t k = sh.sw[l];
                const uint32_t d = (uint32_t)(k >> shift) & dmask;
                const uint64_t dst = (uint64_t)ob + sh.aux[d] + (p - sh.cstart[d]);
                GK_CHECK(dst < n);
                ow[dst] = k;
                os[dst] = ss[l];
            }
            __syncthreads();
            if (tid < LF_ND) sh.aux[tid] += sh.tcnt[tid];
            __syncthreads();
        }
    }
}

// A group of the pass before that runs past a leaf CTA's window: split by the symbol
// at x into the mask's overflow slot by one 1024-thread CTA per group (queued by
// leaf_kernel; CTAs claim entries from the list): the group's end, its digit
// histogram, then 8192-element chunks ranked stably and placed at the digit offsets.
constexpr int LB_TH = 1024;

template <typename S>
__global__ void __launch_bounds__(LB_TH, 1) leaf_big_kernel(LfBigList bl) {
    using L = Lf<LB_TH>;
    constexpr int C = L::C, W = L::WARPS;
    extern __shared__ __align__(16) unsigned char smem[];
    LfShared sh;
    sh.sw = (uint64_t*)smem;
    S* const ss = (S*)(smem + (size_t)C * 8);
    sh.perm = (uint16_t*)(ss + C);
    sh.whist = (uint32_t*)(sh.perm + C);
    sh.match = sh.whist + W * LF_ND;
    sh.cstart = sh.match + W * LF_ND;
    sh.tcnt = sh.cstart + LF_ND;
    sh.aux = sh.tcnt + LF_ND;
    sh.s_w = sh.aux + LF_ND;
    __shared__ unsigned long long s_end;
    __shared__ uint32_t s_q, s_obase;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 2 * W * LF_ND; i += LB_TH) sh.whist[i] = 0u;
    for (;;) {
        if (tid == 0) {
            s_q = atomicAdd(&bl.count[1], 1u);
            s_end = ~0ull;
        }
        __syncthreads();
        const uint32_t q = s_q;
        if (q >= min(bl.count[0], bl.cap)) return;  // (block-uniform)
        const LfBig g = bl.e[q];
        const uint64_t* w = g.w;
        const S* sq = (const S*)g.sq;
        // the group's end: the first head after its start
        for (uint64_t e0 = g.start + 1; e0 < g.cnt; e0 += LB_TH) {
            const uint64_t i = e0 + tid;
            if (i < g.cnt && ((w[i] ^ w[i - 1]) & g.pmask) != 0) atomicMin(&s_end, (unsigned long long)i);
            __syncthreads();
            const bool found = s_end != ~0ull;
            __syncthreads();
            if (found) break;
        }
        const uint64_t e = min((uint64_t)s_end, g.cnt), hl = g.start;
        const uint64_t gs = e - hl;
        // digit histogram (per-warp counters), exclusive digit offsets
        for (uint64_t i = hl + tid; i < e; i += LB_TH)
            atomicAdd(&sh.whist[warp * LF_ND + ((uint32_t)(w[i] >> g.shift) & g.dmask)], 1u);
        __syncthreads();
        if (tid < LF_ND) {
            uint32_t t = 0;
            for (int ww = 0; ww < W; ++ww) {
                t += sh.whist[ww * LF_ND + tid];
                sh.whist[ww * LF_ND + tid] = 0u;
            }
            uint32_t inc = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            if (tid == 31) sh.s_w[32] = inc;
            sh.aux[tid] = inc - t;  // (the upper half adds the lower total below)
        }
        if (tid == 0) s_obase = atomicAdd(g.ocnt, (uint32_t)gs);
        __syncthreads();
        if (tid >= 32 && tid < LF_ND) sh.aux[tid] += sh.s_w[32];
        __syncthreads();
        const uint32_t ob = s_obase;
        uint64_t* ow = g.ow;
        S* os = (S*)g.os;
        for (uint64_t c0 = hl; c0 < e; c0 += C) {
            const uint32_t cl = (uint32_t)min((uint64_t)C, e - c0);
            for (uint32_t l = tid; l < cl; l += LB_TH) {
                sh.sw[l] = w[c0 + l];
                ss[l] = sq[c0 + l];
            }
            __syncthreads();
            lf_rank<LB_TH, LF_IT>(sh, sh.sw, 0, cl, g.shift, g.dmask);
            for (uint32_t p = tid; p < cl; p += LB_TH) {
                const uint32_t l = sh.perm[p];
                const uint64_t k = sh.sw[l];
                const uint32_t d = (uint32_t)(k >> g.shift) & g.dmask;
                ow[(uint64_t)ob + sh.aux[d] + (p - sh.cstart[d])] = k;
                os[(uint64_t)ob + sh.aux[d] + (p - sh.cstart[d])] = ss[l];
            }
            __syncthreads();
            if (tid < LF_ND) sh.aux[tid] += sh.tcnt[tid];
            __syncthreads();
        }
    }
}

template <typename S>
constexpr size_t lb_smem() {
    return (size_t)Lf<LB_TH>::C * (8 + sizeof(S) + 2) + 2 * Lf<LB_TH>::WARPS * LF_ND * 4 + 3 * LF_ND * 4 +
           64 * 4 + 64;
}

template <int TH, int IT>
cudaError_t leaf_go(const uint64_t* w, const void* sq, bool seq16, uint64_t n, const uint32_t* cntp,
                    uint64_t pmask, uint64_t kmask, int shift, uint32_t dmask, int64_t dstride,
                    int64_t* diag, SegmentOut so, unsigned long long* stats, uint64_t* cw, void* cs,
                    uint32_t* ccnt, uint64_t* ow, void* os, uint32_t* ocnt, LfBigList bl,
                    cudaStream_t s) {
    const unsigned grid = (unsigned)((n + Lf<TH, IT>::T - 1) / Lf<TH, IT>::T);
    if (seq16) {
        cudaFuncSetAttribute(leaf_kernel<uint16_t, TH, IT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)lf_smem<uint16_t, TH, IT>());
        return launch_pdl(leaf_kernel<uint16_t, TH, IT>, grid, TH, lf_smem<uint16_t, TH, IT>(), s, w,
                          (const uint16_t*)sq, cntp, n, pmask, kmask, shift, dmask, dstride, diag, so.counts,
                          so, stats, cw, (uint16_t*)cs, ccnt, ow, (uint16_t*)os, ocnt, bl);
    } else {
        cudaFuncSetAttribute(leaf_kernel<uint32_t, TH, IT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)lf_smem<uint32_t, TH, IT>());
        return launch_pdl(leaf_kernel<uint32_t, TH, IT>, grid, TH, lf_smem<uint32_t, TH, IT>(), s, w,
                          (const uint32_t*)sq, cntp, n, pmask, kmask, shift, dmask, dstride, diag, so.counts,
                          so, stats, cw, (uint32_t*)cs, ccnt, ow, (uint32_t*)os, ocnt, bl);
    }
    return cudaGetLastError();
}

}  // namespace

constexpr int LEAF_TH = 128;  // threads per CTA (Scale: 128 -> 54.8 ms, 256 -> 57.6, 512 -> 63.2)
int leaf_tile(bool wide) { return wide ? Lf<LEAF_TH, 12>::T : Lf<LEAF_TH>::T; }

cudaError_t launch_leaf(const uint64_t* w, const void* sq, bool seq16, uint64_t n,
                        const uint32_t* cntp, uint64_t pmask, uint64_t kmask, int shift,
                        uint32_t dmask, int64_t dstride, int64_t* diag, SegmentOut so,
                        unsigned long long* stats, uint64_t* cw, void* cs, uint32_t* ccnt,
                        uint64_t* ow, void* os, uint32_t* ocnt, LfBigList bl, cudaStream_t s,
                        bool wide) {
    if (n == 0) return cudaGetLastError();
    if (wide)
        return leaf_go<LEAF_TH, 12>(w, sq, seq16, n, cntp, pmask, kmask, shift, dmask, dstride, diag,
                                    so, stats, cw, cs, ccnt, ow, os, ocnt, bl, s);
    return leaf_go<LEAF_TH, LF_IT>(w, sq, seq16, n, cntp, pmask, kmask, shift, dmask, dstride, diag, so,
                                 stats, cw, cs, ccnt, ow, os, ocnt, bl, s);
}

cudaError_t launch_leaf_big(LfBigList bl, bool seq16, int sm_count, cudaStream_t s) {
    if (seq16) {
        cudaFuncSetAttribute(leaf_big_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)lb_smem<uint16_t>());
        leaf_big_kernel<uint16_t><<<sm_count, LB_TH, lb_smem<uint16_t>(), s>>>(bl);
    } else {
        cudaFuncSetAttribute(leaf_big_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)lb_smem<uint32_t>());
        leaf_big_kernel<uint32_t><<<sm_count, LB_TH, lb_smem<uint32_t>(), s>>>(bl);
    }
    return cudaGetLastError();
}

}  // namespace gk
