// segment.cu — run-length (countAndUpdate, first half) over sorted composites.
//
// Algorithm 1 line 15, C_m^i <- countAndUpdate(L^i); §2.2 step 2
// (P:125): "counts the occurrences (if >1) of each unique g-mer. Then we use these
// counts and the associated indexes of sequences to update all the kernel
// entries". In the sorted batch, a run of equal composites is one (key, seq,
// count) TRIPLE; a run of equal key bits is one GROUP, whose triples list the
// sequences sharing the (g-m)-mer in ascending order.
//
// One kernel, no inter-tile ordering: a tile emits the groups that START in it
// (a group running past the tile end is finished by its owner, which scans the
// tail), at offsets reserved with one atomicAdd per tile; group order in the
// output is arbitrary (integer sums commute), each group's triples are
// contiguous and in sequence order.
//  * every triple with count >= 2 adds count^2 - count to C_m(X,X) (the
//    within-sequence repeat part of sum_key c_X(key)^2; the other part, one per
//    g-mer per mask, is added in closed form by launch_diag_closed_form —
//    DESIGN.md reading A3: singletons still count on the diagonal) — by the tile
//    holding the triple's first key;
//  * only groups with >= 2 distinct sequences are emitted (the only groups that
//    touch off-diagonal entries): triples as seq | group-head<<31 and count,
//    groups as [first, last+1) triple ranges.
#include "internal.cuh"

namespace gk {

// Element access policies: composites (key bits << sb | seq, the LSD path) or the
// mask trie's separate arrays (masked packed window, sequence id).
template <typename K, bool KM = false>
struct SegComp {
    using E = K;
    // CTAs per SM the register budget is sized for: u32 7 (32 registers; ptxas spills
    // 68-84 B per thread), u64 5 (48 registers; 24-52 B spilled). The spills stay in
    // L1 and these budgets measured faster on DNA / Protein (segment 0.95 -> 0.90 ms)
    // than the spill-free 4 CTAs/SM of abdb978.
    static constexpr int kMinBlocks = sizeof(K) == 4 ? 7 : 5;
    const K* keys;
    int sb;
    const uint64_t* km;  // per segment: key bits << sb | seq bits (nullptr: keys masked)
    uint64_t n;
    // (KM: per-segment key masks over unmasked generation slots, which may start off
    // 16 bytes; else the keys are masked and the batch buffer aligned)
    __device__ E ld(uint64_t i) const { return KM ? (K)(keys[i] & km[i / n]) : keys[i]; }
    __device__ uint64_t kof(uint64_t i) const { return KM ? km[i / n] : ~0ull; }
    __device__ uint64_t kseg(uint64_t sgi) const { return KM ? km[sgi] : ~0ull; }
    __device__ E ldk(uint64_t i, uint64_t k) const { return (K)(keys[i] & k); }
    template <int IT>
    __device__ void ldn(uint64_t base, E (&c)[IT], uint64_t sgi) const {
        if (KM && (((uintptr_t)(keys + base)) & 15)) {  // (generation slots n keys apart)
#pragma unroll
            for (int i = 0; i < IT; ++i) c[i] = keys[base + i];
        } else {
            constexpr int NV = IT * sizeof(K) / 16;
            const uint4* v = (const uint4*)(keys + base);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const uint4 q = v[i];
                const K* kq = (const K*)&q;
#pragma unroll
                for (int e = 0; e < 16 / (int)sizeof(K); ++e) c[i * (16 / sizeof(K)) + e] = kq[e];
            }
        }
        if (KM) {  // (the items cross at most one segment boundary: n >= IT)
            const uint64_t end0 = (sgi + 1) * n;
            const uint64_t k0 = km[sgi], k1 = km[sgi + 1];
#pragma unroll
            for (int i = 0; i < IT; ++i) c[i] = (K)(c[i] & ((base + i < end0) ? k0 : k1));
        }
    }
    __device__ bool teq(E a, E b) const { return a == b; }
    __device__ bool geq(E a, E b) const { return ((a ^ b) >> sb) == 0; }
    __device__ uint32_t seq(E a) const { return (uint32_t)(a & ((1ull << sb) - 1ull)); }
    __device__ E other(E a) const { return ~a; }  // differs in the key bits
    __device__ E shfl(E a, int src) const { return __shfl_sync(0xffffffffu, a, src); }
};

struct SoaElem {
    uint64_t w;
    uint32_t s;
};
template <typename S>
struct SegSoa {
    using E = SoaElem;
    static constexpr int kMinBlocks = 4;  // (48 registers spilled 48-56 bytes)
    const uint64_t* w;   // packed windows (masked by the leaf pass, or by km below)
    const S* sq;         // sequence ids
    const uint64_t* km;  // per segment: the mask's key bits (nullptr: windows masked)
    uint64_t n;          // keys per segment
    __device__ E ld(uint64_t i) const {
        return E{km ? w[i] & km[i / n] : w[i], (uint32_t)sq[i]};
    }
    // the key mask of key i's segment, and a load with a known mask (no division)
    __device__ uint64_t kof(uint64_t i) const { return km ? km[i / n] : ~0ull; }
    __device__ uint64_t kseg(uint64_t sgi) const { return km ? km[sgi] : ~0ull; }
    __device__ E ldk(uint64_t i, uint64_t k) const { return E{w[i] & k, (uint32_t)sq[i]}; }
    template <int IT>
    __device__ void ldn(uint64_t base, E (&c)[IT], uint64_t sgi) const {
        // (16-byte vector loads; scalar when a segment array starts off 16 bytes: the
        // cross-level trie's generation slots are n keys apart)
        if ((((uintptr_t)(w + base)) | ((uintptr_t)(sq + base))) & 15) {
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                c[i].w = w[base + i];
                c[i].s = (uint32_t)sq[base + i];
            }
        } else {
            const uint4* v = (const uint4*)(w + base);
#pragma unroll
            for (int i = 0; i < IT / 2; ++i) {
                const uint4 q = v[i];
                c[2 * i].w = (uint64_t)q.x | (uint64_t)q.y << 32;
                c[2 * i + 1].w = (uint64_t)q.z | (uint64_t)q.w << 32;
            }
            const uint4* u = (const uint4*)(sq + base);
            constexpr int NU = IT * sizeof(S) / 16;
#pragma unroll
            for (int i = 0; i < NU; ++i) {
                const uint4 q = u[i];
                const S* sv = (const S*)&q;
#pragma unroll
                for (int e = 0; e < 16 / (int)sizeof(S); ++e)
                    c[i * (16 / sizeof(S)) + e].s = (uint32_t)sv[e];
            }
        }
        if (km) {  // (the items cross at most one segment boundary: n >= IT)
            const uint64_t end0 = (sgi + 1) * n;
            const uint64_t k0 = km[sgi], k1 = km[sgi + 1];
#pragma unroll
            for (int i = 0; i < IT; ++i) c[i].w &= (base + i < end0) ? k0 : k1;
        }
    }
    __device__ bool teq(E a, E b) const { return a.w == b.w && a.s == b.s; }
    __device__ bool geq(E a, E b) const { return a.w == b.w; }
    __device__ uint32_t seq(E a) const { return a.s; }
    __device__ E other(E a) const { return E{~a.w, a.s}; }
    __device__ E shfl(E a, int src) const {
        return E{__shfl_sync(0xffffffffu, a.w, src), __shfl_sync(0xffffffffu, a.s, src)};
    }
};

template <typename Pol, int IT>
__global__ void __launch_bounds__(SEG_THREADS, IT == 8 ? Pol::kMinBlocks : 3) segment_kernel(
    Pol pol, uint64_t n, uint64_t total, int64_t dstride,
    int64_t* diag, uint32_t* counters, SegmentOut so, unsigned long long* stats) {
    using K = typename Pol::E;
    constexpr int TILE = SEG_THREADS * IT;
    constexpr uint32_t FULLM = IT == 32 ? 0xffffffffu : ((1u << IT) - 1u);
    __shared__ uint32_t s_w[16];
    __shared__ uint16_t s_gpos[TILE];  // tile-local first triple of each group
    __shared__ uint32_t s_tx[TILE], s_tc[TILE];  // the tile's triples, staged
    __shared__ uint32_t s_first_gh, s_base_t, s_base_g, s_tail, s_gend_done;
    __shared__ uint32_t s_wmin[SEG_THREADS / 32], s_beyond, s_cross;
    __shared__ unsigned long long s_gend;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t tile0 = (uint64_t)blockIdx.x * TILE;
    const uint64_t base = tile0 + (uint64_t)tid * IT;
    const uint32_t lbase = (uint32_t)tid * IT;  // tile-local index of item 0
    const uint64_t tile_end = min(tile0 + TILE, total);

    // segment (mask) of this thread's first item: one 64-bit division per thread
    const uint64_t segi0 = base < total ? base / n : 0;
    K cur[IT];
    if (base + IT <= total) {
        pol.template ldn<IT>(base, cur, segi0);
    } else {
#pragma unroll
        for (int i = 0; i < IT; ++i) cur[i] = base + i < total ? pol.ld(base + i) : K{};
    }
    // the last warp also fetches the 32 keys after the tile (the run / group
    // crossing its end), in flight together with the tile's own loads
    const bool has_next = tile_end < total && tile_end % n != 0;
    K ext{}, lk{};
    if (warp == SEG_THREADS / 32 - 1 && has_next) {
        const uint64_t kt = pol.kof(tile_end - 1);  // (the next key is in the same segment)
        lk = pol.ldk(tile_end - 1, kt);
        ext = tile_end + lane < total ? pol.ldk(tile_end + lane, kt) : pol.other(lk);
    }
    // its bounds; consecutive items cross at most one boundary each (n >= 1)
    uint64_t seg_lo = segi0 * n, seg_hi = seg_lo + n;
    const K prev = (base < total && base != seg_lo) ? pol.ldk(base - 1, pol.kseg(segi0)) : K{};

    // 1. head flags: a triple head where the composite changes, a group head where
    //    the key bits change (both at every segment start)
    uint32_t th_bits = 0, gh_bits = 0;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const uint64_t idx = base + i;
        if (idx >= total) break;
        if (idx >= seg_hi) {
            seg_lo = seg_hi;
            seg_hi += n;
        }
        const K c0 = cur[i];
        const K p0 = i == 0 ? prev : cur[i - 1];
        const bool first = idx == seg_lo;
        if (first || !pol.teq(p0, c0)) th_bits |= 1u << i;
        if (first || !pol.geq(p0, c0)) gh_bits |= 1u << i;
    }
    if (tid == 0) {
        s_first_gh = 0xffffffffu;
        s_tail = 0;
    }
    if (warp == SEG_THREADS / 32 - 1) {
        // first triple head at or after the tile end, tile-local (index << 1 | is a
        // group head): a segment start, a key change, or the end of the crossing run
        uint32_t b = (uint32_t)(tile_end - tile0) << 1 | 1u;
        bool cross = false;
        if (has_next) {  // (warp-uniform)
            const uint64_t seg_end = (tile_end / n + 1) * n;
            cross = pol.geq(pol.shfl(ext, 0), lk);
            for (uint64_t e = tile_end;; e += 32) {
                const uint64_t q = e + lane;
                const K kk = e == tile_end ? ext
                                           : (q < seg_end ? pol.ldk(q, pol.kof(tile_end - 1))
                                                          : pol.other(lk));
                const bool stop = q >= seg_end || !pol.teq(kk, lk);
                const uint32_t sm = __ballot_sync(0xffffffffu, stop);
                if (sm) {
                    const int j = __ffs(sm) - 1;
                    const K kj = pol.shfl(kk, j);
                    const uint64_t qj = e + j;
                    const bool g = qj >= seg_end || !pol.geq(kj, lk);
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
    // 2. the first triple head after this thread's items: suffix minimum over the
    //    later threads of the tile, then s_beyond
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
        for (int ww = 1; ww < SEG_THREADS / 32; ++ww)
            if (ww > warp) later = min(later, s_wmin[ww]);
        nxt = min(nxt, later);
    }
    // 3. backward over the items: run length = next head - head; a group head's
    //    group is shared (>= 2 sequences) iff the next triple is not a group head
    uint32_t multi_bits = 0;
    uint32_t cnt[IT];
#pragma unroll
    for (int i = IT - 1; i >= 0; --i) {
        cnt[i] = 0;
        if (!((th_bits >> i) & 1u)) continue;
        const uint32_t li = lbase + i;
        const uint32_t c = (nxt >> 1) - li;
        cnt[i] = c;
        const uint32_t gh = (gh_bits >> i) & 1u;
        if (!gh || !(nxt & 1u)) multi_bits |= 1u << i;
        if (c >= 2) {
            const int64_t x = (int64_t)pol.seq(cur[i]);
            atomicAdd((unsigned long long*)&diag[x * dstride], (unsigned long long)c * c - c);
        }
        nxt = li << 1 | gh;
    }
    if (gh_bits) atomicMin(&s_first_gh, lbase + (__ffs(gh_bits) - 1));
    __syncthreads();
    // keys before the tile's first group head belong to a group owned by an
    // earlier tile: not emitted here
    const uint32_t fgh = s_first_gh;
    uint32_t emit_t = 0, emit_g = 0;
    if (fgh != 0xffffffffu) {
        const uint32_t own = lbase >= fgh ? FULLM : (fgh - lbase < IT ? (FULLM << (fgh - lbase)) & FULLM : 0u);
        emit_t = th_bits & multi_bits & own;
        emit_g = emit_t & gh_bits;
    }
    // one block scan of both counts packed in 16-bit halves (a tile emits < 2^16)
    static_assert(TILE < 65536, "packed scan");
    uint32_t aggp;
    const uint32_t offp = scan256_excl(__popc(emit_t) | (__popc(emit_g) << 16), s_w, &aggp);
    const uint32_t off_t = offp & 0xffffu, off_g = offp >> 16;
    const uint32_t agg_t = aggp & 0xffffu, agg_g = aggp >> 16;

    // 4. the last group starting here may run past the tile: all threads scan its
    //    tail in tile-sized chunks, counting its triple heads
    const bool crossing = fgh != 0xffffffffu && s_cross != 0;
    uint64_t gend = tile_end;  // one past the crossing group's last key
    K gkey{};
    uint64_t kcross = 0;
    uint64_t seg_end_t = 0;
    if (crossing) {  // (block-uniform)
        kcross = pol.kof(tile_end - 1);  // (the tail stays in this segment)
        gkey = pol.ldk(tile_end - 1, kcross);
        seg_end_t = (tile_end / n + 1) * n;
        uint32_t heads = 0;
        for (uint64_t e = tile_end;; e += TILE) {
            if (tid == 0) {
                s_gend = ~0ull;
                s_gend_done = 0;
            }
            __syncthreads();
            uint32_t h = 0;
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                const uint64_t q = e + lbase + i;
                const bool in = q < seg_end_t && pol.geq(pol.ldk(q, kcross), gkey);
                if (!in) {
                    atomicMin(&s_gend, (unsigned long long)q);
                    break;
                }
                h += !pol.teq(pol.ldk(q, kcross), pol.ldk(q - 1, kcross));
            }
            if (h) atomicAdd(&s_tail, h);
            __syncthreads();
            if (s_gend != ~0ull) {
                gend = s_gend;
                break;
            }
        }
        (void)heads;
    }
    __syncthreads();
    const uint32_t tail = s_tail;
    if (tid == 0) {
        s_base_t = atomicAdd(&counters[0], agg_t + tail);
        s_base_g = atomicAdd(&counters[1], agg_g);
        if (agg_t + tail) atomicAdd(&stats[ST_TRIPLES], (unsigned long long)(agg_t + tail));
        if (agg_g) atomicAdd(&stats[ST_GROUPS], (unsigned long long)agg_g);
    }
    __syncthreads();
    const uint32_t base_t = s_base_t, base_g = s_base_g;
    // 5. triples staged in shared memory, then written with coalesced stores
    uint32_t li = off_t, gl = off_g;
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        if (emit_t & (1u << i)) {
            const uint32_t x = pol.seq(cur[i]);
            s_tx[li] = x | (((gh_bits >> i) & 1u) << 31);
            s_tc[li] = cnt[i];
            if (emit_g & (1u << i)) s_gpos[gl++] = (uint16_t)li;
            ++li;
        }
    }
    __syncthreads();
    for (uint32_t j = tid; j < agg_t; j += SEG_THREADS) {
        so.tseq[base_t + j] = s_tx[j];
        so.tcnt[base_t + j] = s_tc[j];
    }
    // group ranges: a group runs to the next group's first triple (or the end of
    // this tile's triples, its tail included)
    const uint32_t tend = base_t + agg_t + tail;
    for (uint32_t g = tid; g < agg_g; g += SEG_THREADS)
        so.groups[base_g + g] =
            make_uint2(base_t + s_gpos[g], g + 1 < agg_g ? base_t + s_gpos[g + 1] : tend);
    // 6. tail triples of the crossing group, after this tile's triples, in order:
    //    chunk by chunk, a block scan of the heads places them
    if (tail) {  // (block-uniform)
        uint32_t wpos = base_t + agg_t;
        for (uint64_t e = tile_end; e < gend; e += TILE) {
            uint32_t hb = 0;
            K kv[IT];
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                const uint64_t q = e + lbase + i;
                kv[i] = q < gend ? pol.ldk(q, kcross) : K{};
                if (q < gend && !pol.teq(kv[i], pol.ldk(q - 1, kcross))) hb |= 1u << i;
            }
            uint32_t chunk_heads;
            const uint32_t off = scan256_excl(__popc(hb), s_w, &chunk_heads);
            uint32_t pos = wpos + off;
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                if (hb & (1u << i)) {
                    const uint64_t q = e + lbase + i;
                    uint64_t r = q + 1;
                    while (r < gend && pol.teq(pol.ldk(r, kcross), kv[i])) ++r;
                    so.tseq[pos] = pol.seq(kv[i]);
                    so.tcnt[pos] = (uint32_t)(r - q);
                    ++pos;
                }
            }
            wpos += chunk_heads;
        }
    }
}

cudaError_t launch_segment(const void* keys, bool k64, uint64_t n, int nseg, int sb,
                           int64_t dstride, int64_t* diag, uint32_t* counters, SegmentOut so,
                           unsigned long long* stats, cudaStream_t s, const uint64_t* km) {
    cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(uint32_t), s);
    uint64_t total = n * (uint64_t)nseg;
    if (e != cudaSuccess || total == 0) return e;
    uint64_t tiles = (total + SEG_TILE - 1) / SEG_TILE;
#define SEG_COMP(KT, KMF)                                                                    \
    segment_kernel<SegComp<KT, KMF>, SEG_ITEMS><<<(unsigned)tiles, SEG_THREADS, 0, s>>>(     \
        SegComp<KT, KMF>{(const KT*)keys, sb, km, n}, n, total, dstride, diag, counters, so, \
        stats)
    if (km && n < (uint64_t)SEG_ITEMS) return cudaErrorInvalidValue;  // (items cross <= 1 segment)
    if (k64) {
        if (km) SEG_COMP(uint64_t, true);
        else SEG_COMP(uint64_t, false);
    } else {
        if (km) SEG_COMP(uint32_t, true);
        else SEG_COMP(uint32_t, false);
    }
#undef SEG_COMP
    return cudaGetLastError();
}

// the mask trie's leaves: packed windows + sequence ids (u16 or u32); km = per
// segment key bits when the windows are not masked (else nullptr; km has nseg + 1
// entries when given)
cudaError_t launch_segment_soa(const uint64_t* w, const void* sq, bool seq16, uint64_t n,
                               int nseg, int64_t dstride, int64_t* diag, uint32_t* counters,
                               SegmentOut so, unsigned long long* stats, cudaStream_t s,
                               const uint64_t* km) {
    cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(uint32_t), s);
    uint64_t total = n * (uint64_t)nseg;
    if (e != cudaSuccess || total == 0) return e;
    // (16 keys per thread -- half the per-tile scans and barriers -- measured slower:
    // 80 registers, 3 CTAs per SM; Text segment 28.4 -> 32.5 ms)
    constexpr int IT = SEG_ITEMS;
    uint64_t tiles = (total + SEG_THREADS * IT - 1) / (SEG_THREADS * IT);
    if (n < (uint64_t)IT) return cudaErrorInvalidValue;  // (items cross <= 1 segment)
    if (seq16)
        segment_kernel<SegSoa<uint16_t>, IT><<<(unsigned)tiles, SEG_THREADS, 0, s>>>(
            SegSoa<uint16_t>{w, (const uint16_t*)sq, km, n}, n, total, dstride, diag, counters, so,
            stats);
    else
        segment_kernel<SegSoa<uint32_t>, IT><<<(unsigned)tiles, SEG_THREADS, 0, s>>>(
            SegSoa<uint32_t>{w, (const uint32_t*)sq, km, n}, n, total, dstride, diag, counters, so,
            stats);
    return cudaGetLastError();
}

}  // namespace gk
