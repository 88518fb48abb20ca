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

template <typename K>
__global__ void __launch_bounds__(SEG_THREADS) segment_kernel(
    const K* __restrict__ keys, uint64_t n, uint64_t total, int sb, int64_t dstride,
    int64_t* diag, uint32_t* counters, SegmentOut so, unsigned long long* stats) {
    __shared__ uint32_t s_w[16];
    __shared__ uint32_t s_gpos[SEG_TILE];
    __shared__ uint32_t s_tx[SEG_TILE], s_tc[SEG_TILE];  // the tile's triples, staged
    __shared__ uint32_t s_first_gh, s_base_t, s_base_g, s_tail;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t tile0 = (uint64_t)blockIdx.x * SEG_TILE;
    const uint64_t base = tile0 + (uint64_t)tid * SEG_ITEMS;
    const uint64_t tile_end = min(tile0 + SEG_TILE, total);
    const uint64_t seqmask = (1ull << sb) - 1ull;
    if (tid == 0) {
        s_first_gh = 0xffffffffu;
        s_tail = 0;
    }
    __syncthreads();

    K cur[SEG_ITEMS];
    if (base + SEG_ITEMS <= total) {
        constexpr int NV = SEG_ITEMS * sizeof(K) / 16;
        const uint4* v = (const uint4*)(keys + base);
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const uint4 q = v[i];
            const K* kq = (const K*)&q;
#pragma unroll
            for (int e = 0; e < 16 / (int)sizeof(K); ++e) cur[i * (16 / sizeof(K)) + e] = kq[e];
        }
    } else {
#pragma unroll
        for (int i = 0; i < SEG_ITEMS; ++i) cur[i] = base + i < total ? keys[base + i] : (K)0;
    }
    // segment (mask) bounds of this thread's first item: one 64-bit division per
    // thread; consecutive items cross at most one boundary each (n >= 1)
    uint64_t seg_lo = base < total ? base / n * n : 0, seg_hi = seg_lo + n;
    const K prev = (base < total && base != seg_lo) ? keys[base - 1] : (K)0;

    uint32_t th_bits = 0, gh_bits = 0, multi_bits = 0;
    uint32_t cnt[SEG_ITEMS];
#pragma unroll
    for (int i = 0; i < SEG_ITEMS; ++i) {
        const uint64_t idx = base + i;
        const K c0 = cur[i];
        const K p0 = i == 0 ? prev : cur[i - 1];
        cnt[i] = 0;
        if (idx >= total) continue;
        if (idx >= seg_hi) {
            seg_lo = seg_hi;
            seg_hi += n;
        }
        const bool first = idx == seg_lo;
        if (!first && p0 == c0) continue;  // not a triple head
        const bool gh = first || (p0 >> sb) != (c0 >> sb);
        // run end j and the key that follows it
        const uint64_t seg_end = seg_hi;
        uint64_t j = idx + 1;
        K nk = (K)~c0;
        bool found = false;
#pragma unroll
        for (int k = i + 1; k < SEG_ITEMS; ++k) {
            if (!found && base + k < seg_end) {
                if (cur[k] != c0) {
                    found = true;
                    nk = cur[k];
                } else {
                    ++j;
                }
            }
        }
        if (!found && j < seg_end) {
            while (j < seg_end) {
                const K kk = keys[j];
                if (kk != c0) {
                    nk = kk;
                    break;
                }
                ++j;
            }
        }
        const uint32_t c = (uint32_t)(j - idx);
        cnt[i] = c;
        if (c >= 2) {
            const int64_t x = (int64_t)(c0 & seqmask);
            atomicAdd((unsigned long long*)&diag[x * dstride], (unsigned long long)c * c - c);
        }
        th_bits |= 1u << i;
        if (!gh || (j < seg_end && (nk >> sb) == (c0 >> sb))) multi_bits |= 1u << i;
        if (gh) {
            gh_bits |= 1u << i;
            atomicMin(&s_first_gh, (uint32_t)(idx - tile0));
        }
    }
    __syncthreads();
    // keys before the tile's first group head belong to a group owned by an
    // earlier tile: not emitted here
    const uint32_t fgh = s_first_gh;
    uint32_t emit_t = 0, emit_g = 0;
#pragma unroll
    for (int i = 0; i < SEG_ITEMS; ++i) {
        const bool own = fgh != 0xffffffffu && (uint32_t)(base + i - tile0) >= fgh;
        if (own && ((th_bits & multi_bits) >> i & 1u)) {
            emit_t |= 1u << i;
            if ((gh_bits >> i) & 1u) emit_g |= 1u << i;
        }
    }
    uint32_t agg_t, agg_g;
    const uint32_t off_t = scan256_excl(__popc(emit_t), s_w, &agg_t);
    const uint32_t off_g = scan256_excl(__popc(emit_g), s_w, &agg_g);

    // the last group starting here may run past the tile: count its tail triples
    const bool has_gh = fgh != 0xffffffffu;
    const bool crossing = has_gh && tile_end < total && tile_end % n != 0 &&
                          (keys[tile_end] >> sb) == (keys[tile_end - 1] >> sb);
    uint64_t gend_key = tile_end;  // one past the crossing group's last key
    if (crossing && warp == 0) {
        const K gkey = keys[tile_end - 1] >> sb;
        const uint64_t seg_end = (tile_end / n + 1) * n;
        uint32_t nt = 0;
        uint64_t e = tile_end;
        K last = keys[tile_end - 1];
        while (true) {
            const uint64_t q = e + lane;
            const K kk = q < seg_end ? keys[q] : (K)~(K)0;
            const bool in = q < seg_end && (kk >> sb) == gkey;
            const uint32_t inm = __ballot_sync(0xffffffffu, in);
            const K pk = __shfl_up_sync(0xffffffffu, kk, 1);
            const K pv = lane == 0 ? last : pk;
            nt += __popc(__ballot_sync(0xffffffffu, in && kk != pv));
            const uint32_t run = ~inm ? __ffs(~inm) - 1 : 32;  // leading in-group lanes
            if (run < 32) {
                gend_key = e + run;
                break;
            }
            last = __shfl_sync(0xffffffffu, kk, 31);
            e += 32;
        }
        if (lane == 0) s_tail = nt;
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
    // triples staged in shared memory, then written with coalesced stores
    uint32_t li = off_t, gl = off_g;
#pragma unroll
    for (int i = 0; i < SEG_ITEMS; ++i) {
        if (emit_t & (1u << i)) {
            const uint32_t x = (uint32_t)(cur[i] & seqmask);
            s_tx[li] = x | (((gh_bits >> i) & 1u) << 31);
            s_tc[li] = cnt[i];
            if (emit_g & (1u << i)) s_gpos[gl++] = s_base_t + li;
            ++li;
        }
    }
    __syncthreads();
    for (uint32_t j = tid; j < agg_t; j += SEG_THREADS) {
        so.tseq[s_base_t + j] = s_tx[j];
        so.tcnt[s_base_t + j] = s_tc[j];
    }
    // group ranges: a group runs to the next group's first triple (or the end of
    // this tile's triples, its tail included)
    const uint32_t tend = s_base_t + agg_t + tail;
    for (uint32_t g = tid; g < agg_g; g += SEG_THREADS)
        so.groups[s_base_g + g] = make_uint2(s_gpos[g], g + 1 < agg_g ? s_gpos[g + 1] : tend);
    // tail triples of the crossing group (warp 0), after this tile's triples
    if (tail && warp == 0) {
        const uint64_t seg_end = (tile_end / n + 1) * n;
        uint32_t w = s_base_t + agg_t;
        K last = keys[tile_end - 1];
        for (uint64_t e = tile_end; e < gend_key; e += 32) {
            const uint64_t q = e + lane;
            const bool in = q < gend_key;
            const K kk = in ? keys[q] : (K)0;
            const K pk = __shfl_up_sync(0xffffffffu, kk, 1);
            const K pv = lane == 0 ? last : pk;
            const bool head = in && kk != pv;
            const uint32_t hm = __ballot_sync(0xffffffffu, head);
            if (head) {
                uint64_t r = q + 1;
                while (r < seg_end && keys[r] == kk) ++r;
                const uint32_t pos = w + __popc(hm & lanemask_lt());
                so.tseq[pos] = (uint32_t)(kk & seqmask);
                so.tcnt[pos] = (uint32_t)(r - q);
            }
            w += __popc(hm);
            last = __shfl_sync(0xffffffffu, kk, 31);
        }
    }
}

cudaError_t launch_segment(const void* keys, bool k64, uint64_t n, int nseg, int sb,
                           int64_t dstride, int64_t* diag, uint32_t* counters, SegmentOut so,
                           unsigned long long* stats, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(uint32_t), s);
    uint64_t total = n * (uint64_t)nseg;
    if (e != cudaSuccess || total == 0) return e;
    uint64_t tiles = (total + SEG_TILE - 1) / SEG_TILE;
    if (k64)
        segment_kernel<uint64_t><<<(unsigned)tiles, SEG_THREADS, 0, s>>>(
            (const uint64_t*)keys, n, total, sb, dstride, diag, counters, so, stats);
    else
        segment_kernel<uint32_t><<<(unsigned)tiles, SEG_THREADS, 0, s>>>(
            (const uint32_t*)keys, n, total, sb, dstride, diag, counters, so, stats);
    return cudaGetLastError();
}

}  // namespace gk
