// segrag.cu — run-length (countAndUpdate, first half) over the
// cross-level mask trie's leaves, with ragged segments and compaction.
//
// Same outputs as segment_kernel (segment.cu): triples (seq | group-head << 31,
// count) of groups with >= 2 distinct sequences, their [first, last+1) ranges, and
// count^2 - count on C_m(X,X) for every repeated (key, seq) (reading A3). Differs in
// two ways, for the chain of cross-level passes (plan.cu: a level-m mask is one
// stable pass, by one position x, over its level-(m+1) parent's sorted elements):
//  * segment s of a batch holds cnt[s] <= n valid elements at [s n, s n + cnt[s])
//    (its parent was compacted), and tiles never straddle segments (a CTA per
//    (segment, tile); CTAs past cnt[s] exit);
//  * optionally it writes the COMPACTED copy of the segment for the next level: the
//    elements of every group of >= 2 elements (key equal under this mask), raw
//    (unmasked) windows + sequence ids, each group whole and in order (groups in
//    arbitrary order). A g-mer alone in its group under mask S is alone under every
//    mask S' ⊃ S (more kept positions only split groups), so it can never again
//    meet another g-mer: it only adds to the diagonal, which the closed form
//    C(g,m) n_X (launch_diag_closed_form) already counts. Dropping such elements
//    keeps every child's groups, triples and counts unchanged.
#include <algorithm>

#include "internal.cuh"

namespace gk {

namespace {

struct RagElem {
    uint64_t w;  // raw (unmasked) window
    uint32_t s;  // sequence id
};

constexpr int RG_THREADS = SEG_THREADS;  // 256
constexpr int RG_IT = SEG_ITEMS;         // 8
constexpr int RG_TILE = RG_THREADS * RG_IT;

template <typename S, bool LOOP>
__global__ void __launch_bounds__(RG_THREADS, 4) segment_rag_kernel(
    const uint64_t* __restrict__ w, const S* __restrict__ sq, const uint64_t* __restrict__ km,
    uint64_t n, const uint32_t* __restrict__ cnt, uint32_t tps, uint32_t nblk, int64_t dstride,
    int64_t* diag,
    uint32_t* counters, SegmentOut so, unsigned long long* stats, uint64_t* cw, S* cs,
    uint32_t* ccnt) {
    __shared__ uint32_t s_w[16];
    __shared__ uint16_t s_gpos[RG_TILE];
    __shared__ uint32_t s_tx[RG_TILE], s_tc[RG_TILE];
    __shared__ uint64_t s_kw[RG_TILE];  // the tile's compacted elements, in order (staged:
    __shared__ S s_ks[RG_TILE];         // their copy out is coalesced)
    __shared__ uint32_t s_first_gh, s_base_t, s_base_g, s_base_c, s_tail;
    __shared__ uint32_t s_wmin[RG_THREADS / 32], s_beyond, s_cross;
    __shared__ unsigned long long s_gend;
    constexpr uint32_t FULLM = (1u << RG_IT) - 1u;
    pdl_wait();  // (launched as a programmatic dependent of the chain's last pass)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // (a grid smaller than segments x tiles loops: the overflow slots of leaf.cu are
    // mostly empty)
    auto body = [&](const uint32_t blk) {
    const uint32_t sgi = blk / tps, t = blk - sgi * tps;
    const uint64_t seg_lo = (uint64_t)sgi * n;
    const uint64_t seg_end = seg_lo + (cnt ? (uint64_t)cnt[sgi] : n);
    const uint64_t tile0 = seg_lo + (uint64_t)t * RG_TILE;
    if (tile0 >= seg_end) return;  // (block-uniform)
    const uint64_t tile_end = min(tile0 + RG_TILE, seg_end);
    const uint64_t kmask = km[sgi];
    const uint64_t base = tile0 + (uint64_t)tid * RG_IT;
    const uint32_t lbase = (uint32_t)tid * RG_IT;
    auto ld = [&](uint64_t i) -> RagElem { return RagElem{w[i], (uint32_t)sq[i]}; };
    auto geq = [&](const RagElem& a, const RagElem& b) { return ((a.w ^ b.w) & kmask) == 0; };
    auto teq = [&](const RagElem& a, const RagElem& b) { return geq(a, b) && a.s == b.s; };

    RagElem cur[RG_IT];
    if (base + RG_IT <= tile_end &&
        ((((uintptr_t)(w + base)) | ((uintptr_t)(sq + base))) & 15) == 0) {
        // 16-byte vector loads (4 of windows, 1 or 2 of ids)
        const uint4* v = (const uint4*)(w + base);
#pragma unroll
        for (int i = 0; i < RG_IT / 2; ++i) {
            const uint4 q = v[i];
            cur[2 * i].w = (uint64_t)q.x | (uint64_t)q.y << 32;
            cur[2 * i + 1].w = (uint64_t)q.z | (uint64_t)q.w << 32;
        }
        const uint4* u = (const uint4*)(sq + base);
        constexpr int NU = RG_IT * sizeof(S) / 16;
#pragma unroll
        for (int i = 0; i < NU; ++i) {
            const uint4 q = u[i];
            const S* sv = (const S*)&q;
#pragma unroll
            for (int e = 0; e < 16 / (int)sizeof(S); ++e) cur[i * (16 / sizeof(S)) + e].s = (uint32_t)sv[e];
        }
    } else {
#pragma unroll
        for (int i = 0; i < RG_IT; ++i) cur[i] = base + i < tile_end ? ld(base + i) : RagElem{0ull, 0u};
    }
    const bool has_next = tile_end < seg_end;
    RagElem ext{0ull, 0u}, lk{0ull, 0u};
    if (warp == RG_THREADS / 32 - 1 && has_next) {
        lk = ld(tile_end - 1);
        ext = tile_end + lane < seg_end ? ld(tile_end + lane) : RagElem{~lk.w, lk.s};
    }
    const RagElem prev = (base < tile_end && base > seg_lo) ? ld(base - 1) : RagElem{0ull, 0u};

    // 1. head flags (a triple head where (key, seq) changes, a group head where the key
    //    changes; both at the segment start)
    uint32_t th_bits = 0, gh_bits = 0, valid_bits = 0;
#pragma unroll
    for (int i = 0; i < RG_IT; ++i) {
        const uint64_t idx = base + i;
        if (idx >= tile_end) break;
        valid_bits |= 1u << i;
        const RagElem p0 = i == 0 ? prev : cur[i - 1];
        const bool first = idx == seg_lo;
        if (first || !teq(p0, cur[i])) th_bits |= 1u << i;
        if (first || !geq(p0, cur[i])) gh_bits |= 1u << i;
    }
    if (tid == 0) {
        s_first_gh = 0xffffffffu;
        s_tail = 0;
    }
    if (warp == RG_THREADS / 32 - 1) {
        // first triple head at or after the tile end (tile-local index << 1 | group head)
        uint32_t b = (uint32_t)(tile_end - tile0) << 1 | 1u;
        bool cross = false;
        if (has_next) {  // (warp-uniform)
            cross = geq(RagElem{__shfl_sync(0xffffffffu, ext.w, 0), __shfl_sync(0xffffffffu, ext.s, 0)}, lk);
            for (uint64_t e = tile_end;; e += 32) {
                const uint64_t q = e + lane;
                const RagElem kk = e == tile_end ? ext : (q < seg_end ? ld(q) : RagElem{~lk.w, lk.s});
                const bool stop = q >= seg_end || !teq(kk, lk);
                const uint32_t sm = __ballot_sync(0xffffffffu, stop);
                if (sm) {
                    const int j = __ffs(sm) - 1;
                    const RagElem kj{__shfl_sync(0xffffffffu, kk.w, j), __shfl_sync(0xffffffffu, kk.s, j)};
                    const uint64_t qj = e + j;
                    const bool g = qj >= seg_end || !geq(kj, lk);
                    b = (uint32_t)(qj - tile0) << 1 | (g ? 1u : 0u);
                    break;
                }
            }
        }
        if (lane == 0) {
            s_beyond = b;
            s_cross = cross ? 1u : 0u;
        }
    }
    // 2. the first triple head after this thread's items
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
        uint32_t later = s_beyond;
#pragma unroll
        for (int ww = 1; ww < RG_THREADS / 32; ++ww)
            if (ww > warp) later = min(later, s_wmin[ww]);
        nxt = min(nxt, later);
    }
    // ghn bit i: is the element after item i a group head? (keep rule below). Valid
    // items are a prefix of the thread's items; after the last of them the next
    // element is the first triple head after this thread (nxt), if it is adjacent
    uint32_t ghn = gh_bits >> 1;
    if (valid_bits) {
        const int ib = __popc(valid_bits) - 1;
        ghn &= ~(1u << ib);
        if ((nxt >> 1) == lbase + ib + 1 && (nxt & 1u)) ghn |= 1u << ib;
    }
    // 3. backward: run lengths, shared groups, the diagonal repeat term
    uint32_t multi_bits = 0;
    uint32_t cntv[RG_IT];
#pragma unroll
    for (int i = RG_IT - 1; i >= 0; --i) {
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
    if (gh_bits) atomicMin(&s_first_gh, lbase + (__ffs(gh_bits) - 1));
    __syncthreads();
    const uint32_t fgh = s_first_gh;
    uint32_t own = 0;
    if (fgh != 0xffffffffu)
        own = lbase >= fgh ? FULLM : (fgh - lbase < RG_IT ? (FULLM << (fgh - lbase)) & FULLM : 0u);
    const uint32_t emit_t = th_bits & multi_bits & own;
    const uint32_t emit_g = emit_t & gh_bits;
    // compaction: an owned element stays iff its group has >= 2 elements (it is not a
    // group head, or the next element is not one)
    uint32_t keep = 0;
    if (cw) keep = own & valid_bits & (~gh_bits | ~ghn) & FULLM;
    uint32_t aggp;
    const uint32_t offp = scan256_excl(__popc(emit_t) | (__popc(emit_g) << 16), s_w, &aggp);
    const uint32_t off_t = offp & 0xffffu, off_g = offp >> 16;
    const uint32_t agg_t = aggp & 0xffffu, agg_g = aggp >> 16;
    uint32_t agg_k = 0, off_k = 0;
    if (cw) off_k = scan256_excl(__popc(keep), s_w, &agg_k);

    // 4. the last group starting here may run past the tile: scan its tail
    const bool crossing = fgh != 0xffffffffu && s_cross != 0;
    uint64_t gend = tile_end;
    RagElem gkey{0ull, 0u};
    if (crossing) {  // (block-uniform)
        gkey = ld(tile_end - 1);
        for (uint64_t e = tile_end;; e += RG_TILE) {
            if (tid == 0) s_gend = ~0ull;
            __syncthreads();
            uint32_t h = 0;
#pragma unroll
            for (int i = 0; i < RG_IT; ++i) {
                const uint64_t q = e + lbase + i;
                const bool in = q < seg_end && geq(ld(q), gkey);
                if (!in) {
                    atomicMin(&s_gend, (unsigned long long)q);
                    break;
                }
                h += !teq(ld(q), ld(q - 1));
            }
            if (h) atomicAdd(&s_tail, h);
            __syncthreads();
            if (s_gend != ~0ull) {
                gend = s_gend;
                break;
            }
        }
    }
    __syncthreads();
    const uint32_t tail = s_tail;
    const uint32_t tail_len = (uint32_t)(gend - tile_end);
    if (cw) {
        uint32_t k = off_k;
#pragma unroll
        for (int i = 0; i < RG_IT; ++i)
            if (keep & (1u << i)) {
                s_kw[k] = cur[i].w;
                s_ks[k] = (S)cur[i].s;
                ++k;
            }
    }
    if (tid == 0) {
        s_base_t = atomicAdd(&counters[0], agg_t + tail);
        s_base_g = atomicAdd(&counters[1], agg_g);
        if (cw) s_base_c = atomicAdd(&ccnt[sgi], agg_k + tail_len);
        if (agg_t + tail) atomicAdd(&stats[ST_TRIPLES], (unsigned long long)(agg_t + tail));
        if (agg_g) atomicAdd(&stats[ST_GROUPS], (unsigned long long)agg_g);
    }
    __syncthreads();
    const uint32_t base_t = s_base_t, base_g = s_base_g;
    // 5. compacted elements of this tile, then the crossing group's tail
    if (cw) {
        const uint64_t cb = (uint64_t)sgi * n + s_base_c;
        for (uint32_t j = tid; j < agg_k; j += RG_THREADS) {
            GK_CHECK(s_base_c + j < n);
            cw[cb + j] = s_kw[j];
            cs[cb + j] = s_ks[j];
        }
        for (uint32_t j = tid; j < tail_len; j += RG_THREADS) {
            GK_CHECK(s_base_c + agg_k + j < n);
            cw[cb + agg_k + j] = w[tile_end + j];
            cs[cb + agg_k + j] = sq[tile_end + j];
        }
    }
    // 6. triples staged in shared memory, written coalesced; group ranges
    uint32_t li = off_t, gl = off_g;
#pragma unroll
    for (int i = 0; i < RG_IT; ++i) {
        if (emit_t & (1u << i)) {
            s_tx[li] = cur[i].s | (((gh_bits >> i) & 1u) << 31);
            s_tc[li] = cntv[i];
            if (emit_g & (1u << i)) s_gpos[gl++] = (uint16_t)li;
            ++li;
        }
    }
    __syncthreads();
    for (uint32_t j = tid; j < agg_t; j += RG_THREADS) {
        so.tseq[base_t + j] = s_tx[j];
        so.tcnt[base_t + j] = s_tc[j];
    }
    const uint32_t tend = base_t + agg_t + tail;
    for (uint32_t g = tid; g < agg_g; g += RG_THREADS)
        so.groups[base_g + g] =
            make_uint2(base_t + s_gpos[g], g + 1 < agg_g ? base_t + s_gpos[g + 1] : tend);
    // 7. tail triples of the crossing group, in order
    if (tail) {  // (block-uniform)
        uint32_t wpos = base_t + agg_t;
        for (uint64_t e = tile_end; e < gend; e += RG_TILE) {
            uint32_t hb = 0;
            RagElem kv[RG_IT];
#pragma unroll
            for (int i = 0; i < RG_IT; ++i) {
                const uint64_t q = e + lbase + i;
                kv[i] = q < gend ? ld(q) : RagElem{0ull, 0u};
                if (q < gend && !teq(kv[i], ld(q - 1))) hb |= 1u << i;
            }
            uint32_t chunk_heads;
            const uint32_t off = scan256_excl(__popc(hb), s_w, &chunk_heads);
            uint32_t pos = wpos + off;
#pragma unroll
            for (int i = 0; i < RG_IT; ++i) {
                if (hb & (1u << i)) {
                    const uint64_t q = e + lbase + i;
                    uint64_t r = q + 1;
                    while (r < gend && teq(ld(r), kv[i])) ++r;
                    so.tseq[pos] = kv[i].s;
                    so.tcnt[pos] = (uint32_t)(r - q);
                    ++pos;
                }
            }
            wpos += chunk_heads;
        }
    }
    };
    if constexpr (LOOP) {
        for (uint32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
            body(blk);
            __syncthreads();  // (this tile's shared-memory reads done)
        }
    } else {
        body(blockIdx.x);
    }
}

}  // namespace

cudaError_t launch_segment_rag(const uint64_t* w, const void* sq, bool seq16, uint64_t n, int nseg,
                               const uint32_t* cnt, const uint64_t* km, int64_t dstride,
                               int64_t* diag, uint32_t* counters, SegmentOut so,
                               unsigned long long* stats, cudaStream_t s, uint64_t* cw,
                               void* cs, uint32_t* ccnt, bool reset, unsigned max_ctas) {
    cudaError_t e = reset ? cudaMemsetAsync(counters, 0, 2 * sizeof(uint32_t), s) : cudaSuccess;
    if (e != cudaSuccess || n == 0 || nseg == 0) return e;
    const uint64_t tps = (n + RG_TILE - 1) / RG_TILE;
    const uint32_t nblk = (uint32_t)(tps * (uint64_t)nseg);
    const unsigned grid = max_ctas ? std::min<unsigned>(nblk, max_ctas) : nblk;
    auto go = [&](auto kern, auto* sqp, auto* csp) {
        e = launch_pdl(kern, grid, RG_THREADS, 0, s, w, sqp, km, n, cnt, (uint32_t)tps, nblk, dstride,
                       diag, counters, so, stats, cw, csp, ccnt);
    };
    if (seq16) {
        if (grid < nblk) go(segment_rag_kernel<uint16_t, true>, (const uint16_t*)sq, (uint16_t*)cs);
        else go(segment_rag_kernel<uint16_t, false>, (const uint16_t*)sq, (uint16_t*)cs);
    } else {
        if (grid < nblk) go(segment_rag_kernel<uint32_t, true>, (const uint32_t*)sq, (uint32_t*)cs);
        else go(segment_rag_kernel<uint32_t, false>, (const uint32_t*)sq, (uint32_t*)cs);
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace gk
