// light.cu — group -> C_m update for groups with few sequences (countAndUpdate,
// second half; Algorithm 1 lines 15-17).
//
// For a group (one masked key) with triples (X_1,c_1), ..., (X_s,c_s) (distinct X,
// in any order), every unordered pair adds c_a*c_b to C_m(min(X_a,X_b), max(..)) —
// the upper triangle; the epilogue mirrors it (reading A4). Integer adds
// commute, so the atomic update order never changes the result. The adds go to
// a u32 strictly-upper packed accumulator (half the footprint of int64 rows, L2
// resident for N <= ~5500) that light_flush adds into C_m; the host flushes
// before masks * n_max^2 could reach 2^32 (per mask an entry grows <= n_X n_Y).
//
// One warp per group; its triples are held in registers 32 at a time and the
// pairs are spread over the lanes (triangle table within a chunk, full 32 x 32
// blocks across chunks), so every atomic instruction carries 32 updates.
#include <algorithm>

#include "internal.cuh"

namespace gk {

// Strictly-upper packed index of (x, y), x < y: rows of N-1, N-2, ... entries.
__device__ __forceinline__ uint64_t tri_index(uint32_t x, uint32_t y, int64_t N) {
    return (uint64_t)x * (uint64_t)(N - 1) - (uint64_t)x * (x - 1) / 2 + (y - x - 1);
}

// Accumulator cell of the unordered pair {x, y} (x != y): the strictly-upper
// packed triangle (full mode, NA = 0), or, in rectangular mode (NA > 0: sequences
// [0, NA) are the rows, [NA, N) the columns), row-major NA x (N - NA) for a
// cross pair; a pair inside one set is not a cell (*ok = false). With a relabelled
// accumulator, *dist = the label distance (far-pair records).
__device__ __forceinline__ uint64_t pair_cell(uint32_t x, uint32_t y, int64_t N, int64_t NA,
                                              bool* ok, const uint32_t* perm = nullptr,
                                              uint32_t* dist = nullptr, uint32_t* lo_out = nullptr) {
    if (perm) {  // relabelled accumulator (full mode only): cell of {perm[x], perm[y]}
        x = perm[x];
        y = perm[y];
    }
    const uint32_t lo = min(x, y), hi = max(x, y);
    if (dist) *dist = hi - lo;
    if (lo_out) *lo_out = lo;
    if (NA == 0) {
        *ok = true;
        return tri_index(lo, hi, N);
    }
    *ok = (int64_t)lo < NA && (int64_t)hi >= NA;
    return (uint64_t)lo * (uint64_t)(N - NA) + (uint64_t)((int64_t)hi - NA);
}

// One pair update acc[idx] += val, called by all 32 lanes (valid marks real
// updates). With binning on (large N: the accumulator is far bigger than L2),
// small updates become 4-byte records (cell offset << 4 | val) appended to the
// bucket of their accumulator block, to be applied block by block while the
// block is L2-resident (apply_bins_kernel); anything else is a direct atomic.
template <bool BINS = true>
__device__ __forceinline__ void pair_add(uint32_t* acc, const LightBins& bn, bool valid,
                                         uint64_t idx, uint32_t val) {
    if (!BINS || bn.nb == 0) {  // (BINS = false: the binning code is not compiled in)
        if (valid) atomicAdd(&acc[idx], val);
        return;
    }
    const uint32_t b = valid ? (uint32_t)(idx / bn.block_cells) : 0xffffffffu;
    const bool rec = valid && val < 16u;
    if (valid && !rec) atomicAdd(&acc[idx], val);
    const uint32_t peers = __match_any_sync(0xffffffffu, rec ? b : 0xffffffffu);
    if (rec) {
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(&bn.cnt[b], (uint32_t)__popc(peers));
        base = __shfl_sync(peers, base, leader);
        const uint64_t pos = (uint64_t)base + __popc(peers & lanemask_lt());
        if (pos < bn.cap)
            bn.rec[(uint64_t)b * bn.cap + pos] =
                ((uint32_t)(idx - (uint64_t)b * bn.block_cells) << 4) | val;
        else
            atomicAdd(&acc[idx], val);  // bucket full
    }
}

// Per-warp appender of far-pair records (FarRec): every lane calls put() (warp-
// uniform control flow); the lanes whose update became a record get true.
struct FarSink {
    FarRec fr;
    uint64_t base;  // first slot of the warp's chunk
    uint32_t used;  // slots of the chunk used (warp-uniform)
    bool have;      // a chunk is held
    bool ok;        // records on (and chunks left)
    uint32_t count; // records written by this warp (warp-uniform)
    __device__ void start(const FarRec& f) {
        fr = f;
        base = 0;
        used = FAR_CHUNK;
        have = false;
        ok = f.near != 0;
        count = 0;
    }
    __device__ void zero_rest() {  // unused slots of the held chunk -> 0 (no-op records)
        if (!have) return;
        for (uint32_t i = used + (threadIdx.x & 31); i < FAR_CHUNK; i += 32) {
            if (fr.k32) ((uint32_t*)fr.rec)[base + i] = 0u;
            else fr.rec[base + i] = 0ull;
        }
    }
    __device__ bool put(bool want, uint64_t cell, uint32_t val) {
        // (cells < 2^40, or < 2^28 for 4-byte records: checked by the host)
        want = want && ok && val < (fr.k32 ? 16u : (1u << 24));
        const uint32_t m = __ballot_sync(0xffffffffu, want);
        if (!m) return false;
        const uint32_t nf = __popc(m);
        if (used + nf > FAR_CHUNK) {
            zero_rest();
            uint64_t b = 0;
            if ((threadIdx.x & 31) == 0) b = atomicAdd(fr.fill, FAR_CHUNK);
            b = __shfl_sync(0xffffffffu, b, 0);
            if (b + FAR_CHUNK > fr.cap) {  // buffer full: this warp goes back to REDs
                if ((threadIdx.x & 31) == 0) atomicAdd(fr.fill + 1, 1u);  // (counted: stats)
                ok = false;
                have = false;
                return false;
            }
            base = b;
            used = 0;
            have = true;
        }
        GK_CHECK(!want || base + used + __popc(m & lanemask_lt()) < fr.cap);
        // (streaming store: the records must not evict the accumulator's L2-resident band)
        if (want) {
            const uint64_t at = base + used + __popc(m & lanemask_lt());
            if (fr.k32) __stcs((uint32_t*)fr.rec + at, (uint32_t)(cell << 4 | val));
            else __stcs(fr.rec + at, cell << 24 | val);
        }
        used += nf;
        count += nf;
        return want;
    }
    __device__ void finish() { zero_rest(); }
};

// far-pair records -> accumulator: the records are bucketed by accumulator block
// (2^bshift cells = 16 MB; one stable 6-bit pass of trie.cu, digit = cell >> bshift),
// then added a few blocks at a time: each group of blocks is first read into L2 by
// plain coalesced loads (an L2 miss under a RED stalls the RED stream -- measured:
// 24 G REDs/s into cold lines vs 208 G/s into resident ones), then its records are
// added. Zero records (unused slots of warp chunks) add nothing.
__global__ void far_offsets_kernel(const uint32_t* __restrict__ H, uint32_t cps, uint32_t* offs) {
    // offs[b] = records in buckets < b (H: cps chunk rows of 64 bucket counts)
    __shared__ uint32_t tot[64];
    pdl_wait();
    const int d = threadIdx.x;
    if (d < 64) {
        uint32_t t = 0;
        for (uint32_t c = 0; c < cps; ++c) t += H[(uint64_t)c * 64 + d];
        tot[d] = t;
    }
    __syncthreads();
    if (d == 0) {
        uint32_t run = 0;
        for (int b = 0; b < 64; ++b) {
            offs[b] = run;
            run += tot[b];
        }
        offs[64] = run;
    }
}
__global__ void far_warm_kernel(const uint32_t* __restrict__ acc, uint64_t c0, uint64_t c1,
                                const uint32_t* offs, int b0, int b1, uint32_t* sink) {
    pdl_wait();
    if (offs[b1] == offs[b0]) return;  // (no records in these blocks)
    const uint4* a = (const uint4*)(acc + c0);
    const uint64_t nv = (c1 - c0) / 4;
    uint32_t x = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = a[i];
        x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (x == 0x9e3779b9u) *sink = x;  // (keeps the loads)
}
template <typename K>
__global__ void far_add_kernel(const K* __restrict__ recs, const uint32_t* offs, int b0, int b1,
                               uint32_t* acc, uint64_t ntri) {
    constexpr int VB = sizeof(K) == 4 ? 4 : 24;  // value bits
    pdl_wait();
    const uint64_t lo = offs[b0], hi = offs[b1];
    for (uint64_t i = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < hi;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const K r = __ldcs(recs + i);  // (streamed: keep the accumulator block in L2)
        const uint32_t v = (uint32_t)(r & (((K)1 << VB) - 1));
        GK_CHECK(!v || (uint64_t)(r >> VB) < ntri);
        if (v) atomicAdd(&acc[(uint64_t)(r >> VB)], v);
    }
}

cudaError_t launch_far_apply(FarRec fr, void* scratch, uint32_t* H, int bshift, uint32_t* acc,
                             uint64_t ntri, int sm_count, cudaStream_t s) {
    const int cps = sm_count * 2;
    cudaError_t e = launch_tp_records(fr.rec, scratch, fr.k32, fr.cap, fr.fill,
                                      (fr.k32 ? 4 : 24) + bshift, H, cps, s);
    if (e != cudaSuccess) return e;
    uint32_t* offs = H + (size_t)cps * 64;  // [65]
    uint32_t* sink = offs + 66;
    // (the chain's launches overlap their predecessor's tail: programmatic dependent
    // launch, each kernel waiting at entry)
    e = launch_pdl(far_offsets_kernel, 1, 64, 0, s, (const uint32_t*)H,
                   (uint32_t)std::min<uint64_t>(cps, std::max<uint64_t>(1, (fr.cap + 4095) / 4096)),
                   offs);
    if (e != cudaSuccess) return e;
    const int nb = (int)std::min<uint64_t>(64, (ntri + (1ull << bshift) - 1) >> bshift);
    constexpr int GRP = 4;  // blocks per group: 64 MB of u32 cells, resident in L2
    for (int b0 = 0; b0 < nb; b0 += GRP) {
        const int b1 = std::min(nb, b0 + GRP);
        const uint64_t c0 = (uint64_t)b0 << bshift;
        uint64_t c1 = std::min<uint64_t>((uint64_t)b1 << bshift, ntri);
        c1 = c1 / 4 * 4;
        if (c1 > c0)
            e = launch_pdl(far_warm_kernel, sm_count * 4, 256, 0, s, (const uint32_t*)acc, c0, c1,
                           (const uint32_t*)offs, b0, b1, sink);
        if (e != cudaSuccess) return e;
        if (fr.k32)
            e = launch_pdl(far_add_kernel<uint32_t>, sm_count * 8, 256, 0, s, (const uint32_t*)scratch,
                           (const uint32_t*)offs, b0, b1, acc, ntri);
        else
            e = launch_pdl(far_add_kernel<uint64_t>, sm_count * 8, 256, 0, s, (const uint64_t*)scratch,
                           (const uint32_t*)offs, b0, b1, acc, ntri);
        if (e != cudaSuccess) return e;
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(fr.fill, 0, sizeof(uint32_t), s);
}

__global__ void apply_bins_kernel(uint32_t* __restrict__ acc, LightBins bn, int b) {
    const uint64_t c = min((uint64_t)bn.cnt[b], bn.cap);
    const uint32_t* r = bn.rec + (uint64_t)b * bn.cap;
    uint32_t* a = acc + (uint64_t)b * bn.block_cells;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < c;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = r[i];
        atomicAdd(&a[v >> 4], v & 15u);
    }
}

cudaError_t launch_apply_bins(uint32_t* acc, LightBins bn, int sm_count, cudaStream_t s) {
    for (int b = 0; b < bn.nb; ++b) {  // one block at a time: L2-resident atomics
        apply_bins_kernel<<<sm_count * 8, 256, 0, s>>>(acc, bn, b);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaMemsetAsync(bn.cnt, 0, bn.nb * sizeof(uint32_t), s);
}

constexpr int LF_STAGE = 256;  // staged triples per warp (flat groups of 32 groups x <= 8)

// MINB: CTAs per SM the register budget is sized for. 5 (48 registers, no spills):
// the occupancy DNA's L2-resident random updates want (light 3.32 ms; 56 registers:
// 3.51 ms); 3 (up to 85 registers) is faster for the big groups of Text / Scale
// (Text light 28.3 -> 26.7 ms, Scale 98.4 -> 93.4 ms).
template <bool WIN, bool BINS, int MINB, bool FAR = false>
__global__ void __launch_bounds__(256, MINB) light_kernel(SegmentOut so, int64_t heavy_min, int64_t N,
                                                    uint32_t* acc, uint2* heavy_list,
                                                    uint64_t ldd, uint32_t* dense_fill,
                                                    LightBins bn, uint32_t flat_max,
                                                    int64_t NA, const uint32_t* perm,
                                                    uint32_t heavy_cmax,
                                                    unsigned long long* stats, WinArgs wa,
                                                    FarRec frec) {
    // triangle table: pairs (a < b < 32) ordered by b, so the first n(n-1)/2
    // entries are exactly the pairs of an n-triple chunk
    __shared__ uint16_t s_tri[496];
    // per warp: the flat groups' triples (labels, counts), LF_STAGE entries
    __shared__ uint32_t s_stx[8][LF_STAGE], s_stc[8][LF_STAGE];
    // entry q = b (b - 1) / 2 + a: b from the closed form (checked by one step each way)
    for (int q = threadIdx.x; q < 496; q += blockDim.x) {
        int b = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)q)) * 0.5f);
        if (b * (b - 1) / 2 > q) --b;
        if ((b + 1) * b / 2 <= q) ++b;
        s_tri[q] = (uint16_t)((q - b * (b - 1) / 2) | (b << 5));
    }
    __syncthreads();
    const uint32_t G = so.counts[1];
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long pairs = 0, nheavy = 0, nwin = 0, nfar = 0;
    uint32_t lpairs = 0;  // per lane: light updates of split groups
    FarSink sink;
    if (FAR) sink.start(frec);
    // one pair update: a far pair (labels >= frec.near apart) becomes a record, the
    // rest are REDs (every lane calls it: warp-uniform)
    auto upd = [&](bool ok, uint64_t idx, uint32_t val, uint32_t dist) {
        GK_CHECK(!ok || NA != 0 || idx < (uint64_t)N * (uint64_t)(N - 1) / 2);
        if constexpr (FAR) {
            const bool rec = sink.put(ok && dist >= frec.near, idx, val);
            if (ok && !rec) atomicAdd(&acc[idx], val);
        } else {
            pair_add<BINS>(acc, bn, ok, idx, val);
        }
    };
    // A warp takes 32 groups at a time: one coalesced load brings all their
    // triple ranges, and the first 32 triples of the next group are loaded while
    // the current one is processed.
    // (the next 32 groups' ranges are loaded while these are processed)
    uint2 rg_next = warp * 32 + lane < G ? so.groups[warp * 32 + lane] : make_uint2(0u, 0u);
    for (uint64_t base = warp * 32; base < G; base += nwarps * 32) {
        const uint32_t ng = (uint32_t)min((uint64_t)32, (uint64_t)G - base);
        const uint2 rg = rg_next;
        {
            const uint64_t nb = base + nwarps * 32 + lane;
            rg_next = nb < G ? so.groups[nb] : make_uint2(0u, 0u);
        }
        const uint32_t my_start = rg.x, my_end = rg.y;
        const uint32_t my_s = my_end - my_start;

        // (1) small light groups (s <= flat_max <= 32) of the batch: their pairs are
        // flattened into one index space, so every lane does one pair update per
        // round whatever the group sizes (no lane idles on a 2-sequence group);
        // the triples are gathered per pair, so bigger groups go to (2), which
        // loads each group's triples once into registers.
        const bool flat = lane < ng && my_s <= flat_max && (int64_t)my_s < heavy_min;
        const uint32_t P = flat ? my_s * (my_s - 1) / 2 : 0u;
        uint32_t incl = P;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t excl = incl - P;
        const uint32_t Ptot = __shfl_sync(0xffffffffu, incl, 31);
        pairs += lane == 0 ? Ptot : 0u;
        // the flat groups' triples usually form one short span of the triple arrays:
        // staged in shared memory with coalesced loads (ids already turned into labels),
        // the per-pair gathers then read shared memory instead of a dependent chain of
        // global loads
        const uint32_t glo = __reduce_min_sync(0xffffffffu, flat ? my_start : 0xffffffffu);
        const uint32_t ghi = __reduce_max_sync(0xffffffffu, flat ? my_end : 0u);
        const bool staged = Ptot > 0 && ghi - glo <= (uint32_t)LF_STAGE;
        uint32_t* sx = s_stx[threadIdx.x >> 5];
        uint32_t* sc = s_stc[threadIdx.x >> 5];
        if (staged) {
#pragma unroll 4
            for (uint32_t t = glo + lane; t < ghi; t += 32) {
                const uint32_t x = so.tseq[t] & 0x7fffffffu;
                sx[t - glo] = perm ? perm[x] : x;
                sc[t - glo] = so.tcnt[t];
            }
            __syncwarp();
        }
        for (uint32_t q0 = 0; q0 < Ptot; q0 += 32) {
            const uint32_t q = q0 + lane;
            // group of pair q: the last lane j with excl_j <= q
            int j = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t e = __shfl_sync(0xffffffffu, excl, j + step);
                if (e <= q) j += step;
            }
            const uint32_t ej = __shfl_sync(0xffffffffu, excl, j);
            const uint32_t sj = __shfl_sync(0xffffffffu, my_start, j);
            uint64_t idx = 0;
            uint32_t val = 0, dist = 0;
            bool ok = false;
            if (q < Ptot) {
                const uint32_t ab = s_tri[q - ej];
                const uint32_t ta = sj + (ab & 31), tb = sj + (ab >> 5);
                if (staged) {
                    idx = pair_cell(sx[ta - glo], sx[tb - glo], N, NA, &ok, nullptr,
                                    FAR ? &dist : nullptr);
                    val = sc[ta - glo] * sc[tb - glo];
                } else {
                    const uint32_t xa = so.tseq[ta] & 0x7fffffffu, xb = so.tseq[tb] & 0x7fffffffu;
                    idx = pair_cell(xa, xb, N, NA, &ok, perm, FAR ? &dist : nullptr);
                    val = so.tcnt[ta] * so.tcnt[tb];
                }
            }
            upd(ok, idx, val, dist);
        }
        __syncwarp();  // (the staging buffer is rewritten by the next 32 groups)

        // (1b) heavy candidates among the 32 groups: counts checked per group, then one
        // atomicAdd claims all their dense columns (a claim per group would serialise
        // every warp on the fill counter)
        uint32_t got = 0;
        {
            uint32_t cand = __ballot_sync(0xffffffffu, lane < ng && !flat && (int64_t)my_s >= heavy_min);
            uint32_t claim = 0;
            while (cand) {
                const int jj = __ffs(cand) - 1;
                cand &= cand - 1;
                const uint32_t a0 = __shfl_sync(0xffffffffu, my_start, jj);
                const uint32_t b0 = __shfl_sync(0xffffffffu, my_end, jj);
                uint32_t cmax = 0;
                for (uint32_t t = a0 + lane; t < b0; t += 32) cmax = max(cmax, so.tcnt[t]);
                cmax = __reduce_max_sync(0xffffffffu, cmax);
                if (cmax <= heavy_cmax) claim |= 1u << jj;
            }
            if (claim) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(dense_fill, (uint32_t)__popc(claim));
                base = __shfl_sync(0xffffffffu, base, 0);
                bool mine = false;
                if ((claim >> lane) & 1u) {
                    const uint64_t col = (uint64_t)base + __popc(claim & lanemask_lt());
                    if (col < ldd) {  // (a full D: the group stays on the light path)
                        heavy_list[col] = make_uint2(my_start, my_end);
                        mine = true;
                    }
                }
                got = __ballot_sync(0xffffffffu, mine);
                nheavy += lane == 0 ? __popc(got) : 0u;
            }
        }

        // (1c) window candidates (relabelled accumulator): a light group of >= wmin
        // sequences becomes a u8 count column of the window of 256 labels holding most
        // of its members (window Gram); the pairs with a member outside the window (a
        // cluster's group plus a few random members from other clusters) stay on the
        // light path below. Counts > 255, < wmin members inside, or a full window: light.
        uint32_t my_win = 0xffffffffu;  // (lane jj: first label of group jj's window)
        uint32_t want_w = 0xffffffffu;  // (lane jj: the window chosen for group jj)
        bool want_split = false;
        if (WIN && wa.nw) {  // (a separate instantiation: no register cost otherwise)
            uint32_t cand = __ballot_sync(0xffffffffu, lane < ng && !flat &&
                                                           (int64_t)my_s < heavy_min &&
                                                           my_s >= wa.wmin) & ~got;
            // (the next candidate's first 32 members are loaded while one is evaluated)
            uint32_t na0 = 0, nb0 = 0, nx0 = 0, nc0 = 0;
            auto fetch = [&](int j) {
                na0 = __shfl_sync(0xffffffffu, my_start, j);
                nb0 = __shfl_sync(0xffffffffu, my_end, j);
                nx0 = na0 + lane < nb0 ? so.tseq[na0 + lane] & 0x7fffffffu : 0u;
                nc0 = na0 + lane < nb0 ? so.tcnt[na0 + lane] : 0u;
            };
            if (cand) fetch(__ffs(cand) - 1);
            while (cand) {
                const int jj = __ffs(cand) - 1;
                cand &= cand - 1;
                const uint32_t a0 = na0, b0 = nb0, x0 = nx0, cb0 = nc0;
                if (cand) fetch(__ffs(cand) - 1);
                // the most populated label bucket (128 labels) among the first 32 members,
                // then the window (2 buckets) around it with the more members
                const bool v0 = a0 + lane < b0;
                const uint32_t lb0 = v0 ? perm[x0] : 0u;
                const uint32_t bk = v0 ? lb0 / WIN_STEP : 0xffffffffu;
                const uint32_t peers = __match_any_sync(0xffffffffu, bk);
                uint64_t key = v0 ? ((uint64_t)__popc(peers) << 32 | (uint64_t)(0xffffffffu - bk)) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
                const uint32_t bs = 0xffffffffu - (uint32_t)(key & 0xffffffffull);
                const uint32_t cm = __popc(__ballot_sync(0xffffffffu, v0 && bs > 0 && bk == bs - 1));
                const uint32_t cp = __popc(__ballot_sync(0xffffffffu, v0 && bk == bs + 1));
                uint32_t w = (cm > cp && bs > 0) ? bs - 1 : bs;
                if (w >= wa.nw) w = wa.nw - 1;
                const uint32_t lo = w * WIN_STEP;
                // (the first 32 members' labels and counts are already in registers)
                uint32_t nin = 0, nout = 0, cmax = 0;
                if (v0) {
                    if (lb0 - lo < (uint32_t)WIN_ROWS) {
                        ++nin;
                        cmax = cb0;
                    } else {
                        ++nout;
                    }
                }
                for (uint32_t t = a0 + 32 + lane; t < b0; t += 32) {
                    const uint32_t lb = perm[so.tseq[t] & 0x7fffffffu];
                    if (lb - lo < (uint32_t)WIN_ROWS) {
                        ++nin;
                        cmax = max(cmax, so.tcnt[t]);
                    } else {
                        ++nout;
                    }
                }
                nin = __reduce_add_sync(0xffffffffu, nin);
                nout = __reduce_add_sync(0xffffffffu, nout);
                cmax = __reduce_max_sync(0xffffffffu, cmax);
                if (cmax <= 255u && nin >= wa.wmin && lane == jj) {
                    want_w = w;  // (claimed below, all of the batch's claims at once)
                    want_split = nout > 0;
                }
            }
            // the claims: one column per chosen group, the atomics of all lanes in flight
            // together (a claim per candidate would wait one round trip each)
            uint32_t col = 0xffffffffu;
            if (want_w != 0xffffffffu) col = atomicAdd(&wa.fill[want_w], 1u);
            const bool claimed = want_w != 0xffffffffu && col < wa.cap;
            if (claimed) {
                wa.list[(uint64_t)want_w * wa.cap + col] = make_uint2(my_start, my_end);
                if (want_split) my_win = want_w * WIN_STEP;  // (split: outside pairs below)
            }
            got |= __ballot_sync(0xffffffffu, claimed && !want_split);
            const uint32_t ncl = __popc(__ballot_sync(0xffffffffu, claimed));  // (all lanes)
            nwin += lane == 0 ? ncl : 0u;
        }

        // (2) the other groups one by one (big light groups). Relabelled accumulator:
        // the sequence ids are turned into labels once per triple as they are loaded
        // (not per pair)
        uint32_t todo = __ballot_sync(0xffffffffu, lane < ng && !flat) & ~got;
        auto lab = [&](uint32_t x) -> uint32_t { return perm ? perm[x] : x; };
        uint32_t pa0 = 0, pb0 = 0, pX = 0, pC = 0;
        auto prefetch = [&](uint32_t jj) {
            pa0 = __shfl_sync(0xffffffffu, my_start, jj);
            pb0 = __shfl_sync(0xffffffffu, my_end, jj);
            pX = pC = 0;
            if (pa0 + lane < pb0) {
                pX = lab(so.tseq[pa0 + lane] & 0x7fffffffu);
                pC = so.tcnt[pa0 + lane];
            }
        };
        if (todo) prefetch(__ffs(todo) - 1);
        while (todo) {
            const int jcur = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t a0 = pa0, b0 = pb0;
            const uint32_t xA0 = pX, cA0 = pC;
            if (todo) prefetch(__ffs(todo) - 1);  // the next group's first chunk
            const uint32_t s = b0 - a0;
            // a split group (window column claimed): its pairs inside the window
            // [wl, wl + 256) are on the tensor cores; only the pairs with an outside
            // member are enumerated, one outsider at a time against all members
            const uint32_t wl = WIN ? __shfl_sync(0xffffffffu, my_win, jcur) : 0xffffffffu;
            if (WIN && wl != 0xffffffffu) {
                for (uint32_t O = a0; O < b0; O += 32) {
                    const uint32_t io = O + lane;
                    const bool vo = io < b0;
                    const uint32_t lO = O == a0 ? xA0 : (vo ? lab(so.tseq[io] & 0x7fffffffu) : 0u);
                    const uint32_t cO = O == a0 ? cA0 : (vo ? so.tcnt[io] : 0u);
                    uint32_t om = __ballot_sync(0xffffffffu, vo && lO - wl >= (uint32_t)WIN_ROWS);
                    while (om) {
                        const int o = __ffs(om) - 1;
                        om &= om - 1;
                        const uint32_t lo_l = __shfl_sync(0xffffffffu, lO, o);
                        const uint32_t co = __shfl_sync(0xffffffffu, cO, o);
                        const uint32_t gio = O + o;
                        for (uint32_t B = a0; B < b0; B += 32) {
                            const uint32_t ib = B + lane;
                            const bool vb = ib < b0;
                            const uint32_t lB = B == a0 ? xA0 : (vb ? lab(so.tseq[ib] & 0x7fffffffu) : 0u);
                            const uint32_t cB = B == a0 ? cA0 : (vb ? so.tcnt[ib] : 0u);
                            // each unordered pair once: an inside member, or a later outsider
                            const bool take = vb && ib != gio &&
                                              (lB - wl < (uint32_t)WIN_ROWS || ib > gio);
                            bool ok = false;
                            uint32_t dist = 0;
                            const uint64_t idx =
                                take ? pair_cell(lo_l, lB, N, NA, &ok, nullptr, FAR ? &dist : nullptr) : 0;
                            lpairs += (ok && take) ? 1u : 0u;
                            upd(ok && take, idx, co * cB, dist);
                        }
                    }
                }
                continue;
            }
            pairs += (unsigned long long)s * (s - 1) / 2;
            // the group's triples in 32-wide register chunks; pairs enumerated
            // lane-parallel: within a chunk through the triangle table, across
            // chunks as full 32 x 32 blocks (every lane busy on every atomic)
            for (uint32_t A = a0; A < b0; A += 32) {
                uint32_t xA = xA0, cA = cA0;
                if (A != a0) {
                    const uint32_t ia = A + lane;
                    xA = ia < b0 ? lab(so.tseq[ia] & 0x7fffffffu) : 0u;
                    cA = ia < b0 ? so.tcnt[ia] : 0u;
                }
                const uint32_t na = min(32u, b0 - A);
                const uint32_t P = na * (na - 1) / 2;
                for (uint32_t q0 = 0; q0 < P; q0 += 32) {
                    const uint32_t q = q0 + lane;
                    const uint32_t ab = q < P ? s_tri[q] : 0u;
                    const int a = ab & 31, b = ab >> 5;
                    const uint32_t xa = __shfl_sync(0xffffffffu, xA, a);
                    const uint32_t ca = __shfl_sync(0xffffffffu, cA, a);
                    const uint32_t xb = __shfl_sync(0xffffffffu, xA, b);
                    const uint32_t cb = __shfl_sync(0xffffffffu, cA, b);
                    bool ok = false;
                    uint32_t dist = 0;
                    const uint64_t idx =
                        q < P ? pair_cell(xa, xb, N, NA, &ok, nullptr, FAR ? &dist : nullptr) : 0;
                    upd(ok && q < P, idx, ca * cb, dist);
                }
                for (uint32_t B = A + 32; B < b0; B += 32) {
                    const uint32_t ib = B + lane;
                    const bool vb = ib < b0;
                    const uint32_t xB = vb ? lab(so.tseq[ib] & 0x7fffffffu) : 0u;
                    const uint32_t cB = vb ? so.tcnt[ib] : 0u;
                    for (uint32_t a = 0; a < na; ++a) {
                        const uint32_t xa = __shfl_sync(0xffffffffu, xA, a);
                        const uint32_t ca = __shfl_sync(0xffffffffu, cA, a);
                        bool ok = false;
                        uint32_t dist = 0;
                        const uint64_t idx =
                            vb ? pair_cell(xa, xB, N, NA, &ok, nullptr, FAR ? &dist : nullptr) : 0;
                        upd(ok && vb, idx, ca * cB, dist);
                    }
                }
            }
        }
    }
    if (FAR) sink.finish();
    if (WIN) pairs += __reduce_add_sync(0xffffffffu, lpairs) * (lane == 0 ? 1ull : 0ull);
    if (lane == 0 && pairs) atomicAdd(&stats[ST_LIGHT_PAIRS], pairs);
    if (FAR) {
        nfar = sink.count;
        if (lane == 0 && nfar) atomicAdd(&stats[ST_FAR_RECORDS], nfar);
    }
    if (lane == 0 && nheavy) atomicAdd(&stats[ST_HEAVY_GROUPS], nheavy);
    if (lane == 0 && nwin) atomicAdd(&stats[ST_WIN_GROUPS], nwin);
}

cudaError_t launch_light(SegmentOut so, uint64_t max_groups, int64_t heavy_min, int64_t N,
                         uint32_t* acc, uint2* heavy_list, uint64_t ldd,
                         uint32_t* dense_fill, LightBins bins, uint32_t flat_max,
                         int64_t NA, const uint32_t* perm, uint32_t heavy_cmax,
                         unsigned long long* stats, int sm_count, cudaStream_t s,
                         WinArgs wa, bool big, FarRec fr, int ctas, int grid_per_sm) {
    if (max_groups == 0) return cudaGetLastError();
    uint64_t blocks = (max_groups + 255) / 256;  // 8 warps x 32 groups per block-round
    // (grid_per_sm < the resident CTAs leaves room on every SM for the other stream's
    // sort / segment kernels of the next batch)
    uint64_t cap = (uint64_t)sm_count * (grid_per_sm > 0 ? grid_per_sm : 8);
    if (blocks > cap) blocks = cap;
#define LIGHT(W, B, MB)                                                                        \
    light_kernel<W, B, MB><<<(unsigned)blocks, 256, 0, s>>>(so, heavy_min, N, acc, heavy_list,  \
                                                            ldd, dense_fill, bins, flat_max, NA, \
                                                            perm, heavy_cmax, stats, wa, fr)
#define LIGHT_FAR(W, MB)                                                                         \
    light_kernel<W, false, MB, true><<<(unsigned)blocks, 256, 0, s>>>(                             \
        so, heavy_min, N, acc, heavy_list, ldd, dense_fill, bins, flat_max, NA, perm, heavy_cmax, \
        stats, wa, fr)
    // (instantiations: the window path and the binning ablation compiled in only
    // where they run; big batches of long masks (>= 2M g-mers) take the 64-register one;
    // the relabelled variants at `ctas` CTAs per SM: 3 (72 registers), 4 or 6)
    if (fr.near && perm && bins.nb == 0) {
        if (wa.nw) {
            if (ctas >= 6) LIGHT_FAR(true, 6);
            else if (ctas == 4) LIGHT_FAR(true, 4);
            else LIGHT_FAR(true, 3);
        } else {
            LIGHT_FAR(false, 3);
        }
    } else if (wa.nw) {
        if (bins.nb > 0) LIGHT(true, true, 3);
        else if (ctas >= 6) LIGHT(true, false, 6);
        else if (ctas == 4) LIGHT(true, false, 4);
        else LIGHT(true, false, 3);
    } else if (bins.nb > 0) {
        LIGHT(false, true, 5);
    } else if (big) {
        LIGHT(false, false, 3);
    } else {
        LIGHT(false, false, 5);
    }
#undef LIGHT
#undef LIGHT_FAR
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || bins.nb == 0) return e;
    return launch_apply_bins(acc, bins, sm_count, s);
}

// C_m(X,Y) += acc[(X,Y)] for every X < Y, and acc is zeroed again (one pass over
// the packed triangle; rows of C are read-modify-written contiguously).
__global__ void light_flush_kernel(uint32_t* __restrict__ acc, int64_t N, int64_t* __restrict__ Cm) {
    for (int64_t x = blockIdx.x; x < N - 1; x += gridDim.x) {
        uint32_t* row = acc + tri_index((uint32_t)x, (uint32_t)x + 1, N);
        int64_t* crow = Cm + x * N;
        for (int64_t y = x + 1 + threadIdx.x; y < N; y += blockDim.x) {
            const uint32_t v = row[y - x - 1];
            if (v) {  // atomic: a Gram flush of the same level may run on another stream
                atomicAdd((unsigned long long*)&crow[y], (unsigned long long)v);
                row[y - x - 1] = 0u;
            }
        }
    }
}

// Relabelled accumulator: C_m(X,Y) += acc[cell{perm[X], perm[Y]}] for X < Y, read
// row by row of C_m (coalesced int64 adds; the acc reads gather). The caller zeroes
// acc afterwards (one memset).
__global__ void light_flush_perm_kernel(const uint32_t* __restrict__ acc, int64_t N,
                                        int64_t* __restrict__ Cm,
                                        const uint32_t* __restrict__ perm) {
    for (int64_t x = blockIdx.x; x < N - 1; x += gridDim.x) {
        const uint32_t px = perm[x];
        int64_t* crow = Cm + x * N;
        for (int64_t y = x + 1 + threadIdx.x; y < N; y += blockDim.x) {
            const uint32_t py = perm[y];
            const uint32_t v = acc[tri_index(min(px, py), max(px, py), N)];
            if (v) atomicAdd((unsigned long long*)&crow[y], (unsigned long long)v);
        }
    }
}

cudaError_t launch_light_flush_perm(uint32_t* acc, int64_t N, int64_t* Cm, const uint32_t* perm,
                                    int sm_count, cudaStream_t s) {
    if (N < 2) return cudaGetLastError();
    int64_t blocks = N - 1 < (int64_t)sm_count * 16 ? N - 1 : (int64_t)sm_count * 16;
    light_flush_perm_kernel<<<(unsigned)blocks, 256, 0, s>>>(acc, N, Cm, perm);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(acc, 0, (size_t)N * (size_t)(N - 1) / 2 * 4, s);
}

// ---- sequence relabelling for the light accumulator (locality) ----
// best[X] = max over Y != X of (C(X,Y) << 32 | Y) for C(X,Y) > 0 (upper triangle read
// once; both endpoints updated): the partner sharing the most matches with X.
__global__ void best_partner_kernel(const int64_t* __restrict__ C, int64_t N,
                                    unsigned long long* best) {
    for (int64_t x = blockIdx.x; x < N - 1; x += gridDim.x) {
        const int64_t* row = C + x * N;
        unsigned long long mine = 0ull;
        for (int64_t y = x + 1 + threadIdx.x; y < N; y += blockDim.x) {
            const int64_t v = row[y];
            if (v > 0) {
                const unsigned long long vc = (unsigned long long)min(v, (int64_t)0xffffffff);
                mine = max(mine, (vc << 32) | (unsigned long long)y);
                atomicMax(&best[y], (vc << 32) | (unsigned long long)x);
            }
        }
        for (int o = 16; o > 0; o >>= 1) mine = max(mine, __shfl_xor_sync(0xffffffffu, mine, o));
        if ((threadIdx.x & 31) == 0 && mine) atomicMax(&best[x], mine);
    }
}

__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t x) {
    while (true) {
        const uint32_t p = parent[x];
        if (p == x) return x;
        const uint32_t gp = parent[p];
        if (gp != p) atomicCAS(&parent[x], p, gp);  // path halving
        x = p;
    }
}

// union(X, best partner of X), lock-free (the larger root is hooked under the smaller)
__global__ void best_union_kernel(const unsigned long long* __restrict__ best, int64_t N,
                                  uint32_t* parent) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
         x += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long b = best[x];
        if (!b) continue;
        uint32_t a = (uint32_t)x, c = (uint32_t)(b & 0xffffffffull);
        while (true) {
            a = uf_find(parent, a);
            c = uf_find(parent, c);
            if (a == c) break;
            if (a < c) {
                const uint32_t t = a;
                a = c;
                c = t;
            }
            if (atomicCAS(&parent[a], a, c) == a) break;
        }
    }
}

// union(X, Y) for every pair sharing at least a quarter of the matches of X's or Y's
// best partner (and >= 2): joins whole families, not only best-partner chains
__global__ void thresh_union_kernel(const int64_t* __restrict__ C, int64_t N,
                                    const unsigned long long* __restrict__ best,
                                    uint32_t* parent) {
    for (int64_t x = blockIdx.x; x < N - 1; x += gridDim.x) {
        const uint64_t bx = best[x] >> 32;
        const int64_t* row = C + x * N;
        for (int64_t y = x + 1 + threadIdx.x; y < N; y += blockDim.x) {
            const int64_t v = row[y];
            if (v < 2) continue;
            const uint64_t by = best[y] >> 32;
            if ((uint64_t)v * 4 < bx && (uint64_t)v * 4 < by) continue;
            if (parent[x] == parent[y]) continue;  // (already one cluster: flattened paths)
            uint32_t a = (uint32_t)x, c = (uint32_t)y;
            while (true) {
                a = uf_find(parent, a);
                c = uf_find(parent, c);
                if (a == c) break;
                if (a < c) {
                    const uint32_t t = a;
                    a = c;
                    c = t;
                }
                if (atomicCAS(&parent[a], a, c) == a) break;
            }
        }
    }
}

__global__ void uf_roots_kernel(uint32_t* parent, int64_t N) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
         x += (int64_t)gridDim.x * blockDim.x)
        parent[x] = uf_find(parent, (uint32_t)x);
}

cudaError_t launch_cluster_roots(const int64_t* C, int64_t N, unsigned long long* best,
                                 uint32_t* parent, const uint32_t* iota, int sm_count,
                                 cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(best, 0, N * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(parent, iota, N * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    const int64_t rows = N - 1 < (int64_t)sm_count * 16 ? N - 1 : (int64_t)sm_count * 16;
    if (rows > 0) best_partner_kernel<<<(unsigned)rows, 256, 0, s>>>(C, N, best);
    const int blocks = (int)((N + 255) / 256 < 1024 ? (N + 255) / 256 : 1024);
    best_union_kernel<<<blocks, 256, 0, s>>>(best, N, parent);
    // (paths flattened first: the threshold unions mostly meet pairs the best-partner
    // links already joined, and then each find is one load)
    uf_roots_kernel<<<blocks, 256, 0, s>>>(parent, N);
    if (rows > 0) thresh_union_kernel<<<(unsigned)rows, 256, 0, s>>>(C, N, best, parent);
    uf_roots_kernel<<<blocks, 256, 0, s>>>(parent, N);
    return cudaGetLastError();
}

// device relabelling: keys root << 32 | x, then (after a stable sort by root) the labels
__global__ void relabel_keys_kernel(const uint32_t* __restrict__ root, int64_t N, uint64_t* keys) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
         x += (int64_t)gridDim.x * blockDim.x)
        keys[x] = (uint64_t)root[x] << 32 | (uint64_t)x;
}
__global__ void relabel_perm_kernel(const uint64_t* __restrict__ keys, int64_t N, uint32_t* perm,
                                    uint32_t* inv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t x = (uint32_t)(keys[i] & 0xffffffffull);
        perm[x] = (uint32_t)i;
        if (inv) inv[i] = x;
    }
}
cudaError_t launch_relabel_keys(const uint32_t* root, int64_t N, uint64_t* keys, cudaStream_t s) {
    const int blocks = (int)((N + 255) / 256 < 1024 ? (N + 255) / 256 : 1024);
    relabel_keys_kernel<<<blocks, 256, 0, s>>>(root, N, keys);
    return cudaGetLastError();
}
cudaError_t launch_relabel_perm(const uint64_t* keys, int64_t N, uint32_t* perm, uint32_t* inv,
                                cudaStream_t s) {
    const int blocks = (int)((N + 255) / 256 < 1024 ? (N + 255) / 256 : 1024);
    relabel_perm_kernel<<<blocks, 256, 0, s>>>(keys, N, perm, inv);
    return cudaGetLastError();
}

// Rectangular mode: C_m[X][Y - NA] += acc[X][Y - NA] (row-major NA x NB), zeroed.
__global__ void light_flush_rect_kernel(uint32_t* __restrict__ acc, uint64_t cells,
                                        int64_t* __restrict__ Cm) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cells;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = acc[i];
        if (v) {
            atomicAdd((unsigned long long*)&Cm[i], (unsigned long long)v);
            acc[i] = 0u;
        }
    }
}

cudaError_t launch_light_flush_rect(uint32_t* acc, uint64_t cells, int64_t* Cm, int sm_count,
                                    cudaStream_t s) {
    if (cells == 0) return cudaGetLastError();
    light_flush_rect_kernel<<<sm_count * 8, 256, 0, s>>>(acc, cells, Cm);
    return cudaGetLastError();
}

cudaError_t launch_light_flush(uint32_t* acc, int64_t N, int64_t* Cm, int sm_count,
                               cudaStream_t s) {
    if (N < 2) return cudaGetLastError();
    int64_t blocks = N - 1 < (int64_t)sm_count * 16 ? N - 1 : (int64_t)sm_count * 16;
    light_flush_kernel<<<(unsigned)blocks, 256, 0, s>>>(acc, N, Cm);
    return cudaGetLastError();
}

// Closed-form diagonal part: every g-mer of X matches itself under every mask, so
// each of the nmask masks adds n_X = gofs[X+1]-gofs[X] to C_m(X,X) = diag[X*dstride].
__global__ void diag_closed_form_kernel(const int64_t* __restrict__ gofs, int64_t N, int64_t nmask,
                                        int64_t* diag, int64_t dstride) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < N;
         x += (int64_t)gridDim.x * blockDim.x)
        diag[x * dstride] += nmask * (gofs[x + 1] - gofs[x]);
}

cudaError_t launch_diag_closed_form(const int64_t* gofs, int64_t N, int64_t nmask, int64_t* diag,
                                    int64_t dstride, cudaStream_t s) {
    int64_t blocks = (N + 255) / 256;
    diag_closed_form_kernel<<<(int)(blocks < 1024 ? blocks : 1024), 256, 0, s>>>(gofs, N, nmask,
                                                                                 diag, dstride);
    return cudaGetLastError();
}

}  // namespace gk
