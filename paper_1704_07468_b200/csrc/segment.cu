// segment.cu — run-length (countAndUpdate, first half) over sorted composites.
//
// Algorithm 1 line 15, C_m^i <- countAndUpdate(L^i); §2.2 step 2
// (P:125): "counts the occurrences (if >1) of each unique g-mer. Then we use these
// counts and the associated indexes of sequences to update all the kernel
// entries". In the sorted batch, a run of equal composites is one (key, seq,
// count) TRIPLE; a run of equal key bits is one GROUP, whose triples list the
// sequences sharing the (g-m)-mer in ascending order.
//
// One pass, one kernel (ordered compaction with decoupled look-back):
//  * every triple with count >= 2 adds count^2 - count to C_m(X,X) (the
//    within-sequence repeat part of sum_key c_X(key)^2; the other part, one per
//    g-mer per mask, is added in closed form by launch_diag_closed_form —
//    DESIGN.md reading A3: singletons still count on the diagonal);
//  * only triples of groups with >= 2 distinct sequences are emitted (the only
//    groups that touch off-diagonal entries), as seq | group-head<<31 and count;
//  * the first emitted triple of each such group is recorded in gstart[]; a
//    group's triples are [gstart[g], gstart[g+1]) (gstart[G] == T).
#include "internal.cuh"

namespace gk {

__global__ void __launch_bounds__(SEG_THREADS) segment_kernel(
    const uint64_t* __restrict__ keys, uint64_t n, uint64_t total, int sb, int64_t N,
    int64_t* Cm, uint64_t* status_t, uint64_t* status_g, uint32_t* ctr, uint32_t epoch,
    SegmentOut so, unsigned long long* stats) {
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_tile, s_pt, s_pg;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const uint64_t base = (uint64_t)t * SEG_TILE + (uint64_t)tid * SEG_ITEMS;
    const uint64_t seqmask = (1ull << sb) - 1ull;

    uint64_t cur[SEG_ITEMS];
    if (base + SEG_ITEMS <= total) {
        const ulonglong2* v = (const ulonglong2*)(keys + base);
#pragma unroll
        for (int i = 0; i < SEG_ITEMS / 2; ++i) {
            ulonglong2 q = v[i];
            cur[2 * i] = q.x;
            cur[2 * i + 1] = q.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < SEG_ITEMS; ++i) cur[i] = base + i < total ? keys[base + i] : 0ull;
    }
    uint64_t prev = (base < total && base % n != 0) ? keys[base - 1] : 0ull;

    uint32_t emit_t = 0, emit_g = 0, gh_bits = 0;
    uint32_t cnt[SEG_ITEMS];
#pragma unroll
    for (int i = 0; i < SEG_ITEMS; ++i) {
        const uint64_t idx = base + i;
        const uint64_t c0 = cur[i];
        const uint64_t p0 = i == 0 ? prev : cur[i - 1];
        cnt[i] = 0;
        if (idx >= total) continue;
        const bool first = (idx % n) == 0;
        if (!first && p0 == c0) continue;  // not a triple head
        const bool gh = first || (p0 >> sb) != (c0 >> sb);
        // run end j and the key that follows it
        const uint64_t seg_end = (idx / n + 1) * n;
        uint64_t j = idx + 1;
        uint64_t nk = ~c0;
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
                const uint64_t kk = keys[j];
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
            atomicAdd((unsigned long long*)&Cm[x * N + x], (unsigned long long)c * c - c);
        }
        const bool multi = !gh || (j < seg_end && (nk >> sb) == (c0 >> sb));
        if (multi) {
            emit_t |= 1u << i;
            if (gh) emit_g |= 1u << i;
        }
        if (gh) gh_bits |= 1u << i;
    }
    uint32_t agg_t, agg_g;
    const uint32_t off_t = scan256_excl(__popc(emit_t), s_w, &agg_t);
    const uint32_t off_g = scan256_excl(__popc(emit_g), s_w, &agg_g);
    if (tid < 32) {
        const uint32_t e = lookback_warp(status_t, t, agg_t, epoch);
        if (tid == 0) s_pt = e;
    } else if (tid < 64) {
        const uint32_t e = lookback_warp(status_g, t, agg_g, epoch);
        if (tid == 32) s_pg = e;
    }
    __syncthreads();
    uint32_t ti = s_pt + off_t, gi = s_pg + off_g;
#pragma unroll
    for (int i = 0; i < SEG_ITEMS; ++i) {
        if (emit_t & (1u << i)) {
            const uint32_t x = (uint32_t)(cur[i] & seqmask);
            so.tseq[ti] = x | (((gh_bits >> i) & 1u) << 31);
            so.tcnt[ti] = cnt[i];
            if (emit_g & (1u << i)) so.gstart[gi++] = ti;
            ++ti;
        }
    }
    if (base < total && base + SEG_ITEMS >= total) {  // the thread holding the last key
        so.counts[0] = s_pt + agg_t;
        so.counts[1] = s_pg + agg_g;
        so.gstart[s_pg + agg_g] = s_pt + agg_t;        // sentinel gstart[G] = T
    }
    if (tid == 0) {
        atomicAdd(&stats[ST_TRIPLES], (unsigned long long)agg_t);
        atomicAdd(&stats[ST_GROUPS], (unsigned long long)agg_g);
    }
}

cudaError_t launch_segment(const uint64_t* keys, uint64_t n, int nseg, int sb, int64_t N,
                           int64_t* Cm, uint64_t* status_t, uint64_t* status_g, uint32_t* ctr,
                           uint32_t epoch, SegmentOut so, unsigned long long* stats,
                           cudaStream_t s) {
    uint64_t total = n * (uint64_t)nseg;
    if (total == 0) return cudaMemsetAsync(so.counts, 0, 2 * sizeof(uint32_t), s);
    uint64_t tiles = (total + SEG_TILE - 1) / SEG_TILE;
    segment_kernel<<<(unsigned)tiles, SEG_THREADS, 0, s>>>(keys, n, total, sb, N, Cm, status_t,
                                                           status_g, ctr, epoch, so, stats);
    return cudaGetLastError();
}

}  // namespace gk
