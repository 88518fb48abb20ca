// segment.cu — run-length (countAndUpdate, first half) over sorted composites.
//
// Algorithm 1 line 15, C_m^i <- countAndUpdate(L^i); §2.2 step 2
// (P:125): "counts the occurrences (if >1) of each unique g-mer. Then we use these
// counts and the associated indexes of sequences to update all the kernel
// entries". In the sorted batch, a run of equal composites is one (key, seq,
// count) TRIPLE; a run of equal key bits is one GROUP, whose triples list the
// sequences sharing the (g-m)-mer in ascending order.
//
// Two ordered compactions (single pass each, decoupled look-back):
//   triples_kernel: one record per triple: seq | group-head<<31, count.
//     It also adds the within-sequence repeat term of the diagonal,
//     count^2 - count, to C_m(X,X) (the other part of sum_key c_X(key)^2, one per
//     g-mer per mask, is added in closed form by launch_diag_closed_form; DESIGN.md
//     reading A3: singletons still count on the diagonal).
//   groups_kernel: [start, end) triple ranges of groups with >= 2 distinct
//     sequences — the only groups that touch off-diagonal entries.
#include "internal.cuh"

namespace gk {

__global__ void __launch_bounds__(SEG_THREADS) triples_kernel(
    const uint64_t* __restrict__ keys, uint64_t n, uint64_t total, int sb, int64_t N,
    int64_t* Cm, uint64_t* status, uint32_t* ctr, uint32_t epoch, SegmentOut so,
    unsigned long long* stats) {
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_tile, s_prefix;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const uint64_t base = (uint64_t)t * SEG_TILE + (uint64_t)tid * SEG_ITEMS;
    const uint64_t seqmask = (sb >= 64) ? ~0ull : ((1ull << sb) - 1ull);

    uint64_t cur[SEG_ITEMS];
    uint32_t heads = 0, ghead = 0;  // bit i: item i is a triple head / group head
#pragma unroll
    for (int i = 0; i < SEG_ITEMS; ++i) {
        uint64_t idx = base + i;
        cur[i] = 0;
        if (idx < total) {
            cur[i] = keys[idx];
            bool first = (idx % n) == 0;
            uint64_t prev = first ? 0 : keys[idx - 1];
            if (first || prev != cur[i]) heads |= 1u << i;
            if (first || (prev >> sb) != (cur[i] >> sb)) ghead |= 1u << i;
        }
    }
    const uint32_t mine = __popc(heads);
    uint32_t agg;
    const uint32_t off = scan256_excl(mine, s_w, &agg);
    if (tid == 0) s_prefix = lookback_one(status, t, agg, epoch);
    __syncthreads();
    uint32_t ti = s_prefix + off;
    uint32_t ntrip = 0;
#pragma unroll
    for (int i = 0; i < SEG_ITEMS; ++i) {
        if (heads & (1u << i)) {
            const uint64_t idx = base + i;
            const uint64_t seg_end = (idx / n + 1) * n;
            uint64_t j = idx + 1;
            while (j < seg_end && keys[j] == cur[i]) ++j;
            const uint32_t c = (uint32_t)(j - idx);
            const uint32_t x = (uint32_t)(cur[i] & seqmask);
            so.tseq[ti] = x | (((ghead >> i) & 1u) << 31);
            so.tcnt[ti] = c;
            if (c >= 2) atomicAdd((unsigned long long*)&Cm[(int64_t)x * N + x],
                                  (unsigned long long)c * c - c);
            ++ti;
            ++ntrip;
        }
    }
    if (base < total && base + SEG_ITEMS >= total) so.counts[0] = s_prefix + agg;  // last tile
    if (tid == 0) atomicAdd(&stats[ST_TRIPLES], (unsigned long long)agg);
}

cudaError_t launch_triples(const uint64_t* keys, uint64_t n, int nseg, int sb, int64_t N,
                           int64_t* Cm, uint64_t* status, uint32_t* ctr, uint32_t epoch,
                           SegmentOut so, unsigned long long* stats, cudaStream_t s) {
    uint64_t total = n * (uint64_t)nseg;
    if (total == 0) return cudaMemsetAsync(so.counts, 0, 2 * sizeof(uint32_t), s);
    uint64_t tiles = (total + SEG_TILE - 1) / SEG_TILE;
    triples_kernel<<<(unsigned)tiles, SEG_THREADS, 0, s>>>(keys, n, total, sb, N, Cm, status, ctr,
                                                           epoch, so, stats);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(SEG_THREADS) groups_kernel(uint64_t* status, uint32_t* ctr,
                                                             uint32_t epoch, SegmentOut so,
                                                             unsigned long long* stats) {
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_tile, s_prefix;
    const int tid = threadIdx.x;
    if (tid == 0) s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    const uint32_t T = so.counts[0];
    if ((uint64_t)t * SEG_TILE >= T) return;  // past the end: no later tile needs us
    const uint64_t base = (uint64_t)t * SEG_TILE + (uint64_t)tid * SEG_ITEMS;
    uint32_t flags = 0;
#pragma unroll
    for (int i = 0; i < SEG_ITEMS; ++i) {
        uint64_t idx = base + i;
        if (idx + 1 < T && (so.tseq[idx] >> 31) && !(so.tseq[idx + 1] >> 31)) flags |= 1u << i;
    }
    uint32_t agg;
    const uint32_t off = scan256_excl(__popc(flags), s_w, &agg);
    if (tid == 0) s_prefix = lookback_one(status, t, agg, epoch);
    __syncthreads();
    uint32_t gi = s_prefix + off;
#pragma unroll
    for (int i = 0; i < SEG_ITEMS; ++i) {
        if (flags & (1u << i)) {
            uint64_t a = base + i, e = a + 1;
            while (e < T && !(so.tseq[e] >> 31)) ++e;
            so.gstart[gi] = (uint32_t)a;
            so.gend[gi] = (uint32_t)e;
            ++gi;
        }
    }
    if (base < T && base + SEG_ITEMS >= T) so.counts[1] = s_prefix + agg;
    if (tid == 0) atomicAdd(&stats[ST_GROUPS], (unsigned long long)agg);
}

cudaError_t launch_groups(uint64_t max_triples, uint64_t* status, uint32_t* ctr, uint32_t epoch,
                          SegmentOut so, unsigned long long* stats, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(so.counts + 1, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess || max_triples == 0) return e;
    uint64_t tiles = (max_triples + SEG_TILE - 1) / SEG_TILE;
    groups_kernel<<<(unsigned)tiles, SEG_THREADS, 0, s>>>(status, ctr, epoch, so, stats);
    return cudaGetLastError();
}

}  // namespace gk
