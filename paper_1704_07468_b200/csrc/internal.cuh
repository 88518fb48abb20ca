// internal.cuh — shared declarations of the libgakco.so translation units.
// Product code: nothing here is shared with oracle/ (see DESIGN.md "Boundary").
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "gakco.h"

// Bounds-checked build (compute-sanitizer is closed on this GPU pool): compiled with
// -DGAKCO_CHECKS (python -m paper_1704_07468_b200.build --checked -> libgakco_checked.so),
// every GK_CHECK is a device assert on an index about to be written / read.
#ifdef GAKCO_CHECKS
#include <cassert>
#define GK_CHECK(c) assert(c)
#else
#define GK_CHECK(c) ((void)0)
#endif

namespace gk {

constexpr int GMAX = 32;          // longest supported g-mer
constexpr int RADIX_BITS = 8;     // LSD digit width
constexpr int RADIX = 256;
constexpr int MAXPASS = 8;        // 64-bit composite / 8-bit digits

// Onesweep tile: 512 threads x 8 keys.
constexpr int SORT_THREADS = 512;
constexpr int SORT_ITEMS = 8;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;

// Segment (run-length) tile.
constexpr int SEG_THREADS = 256;
constexpr int SEG_ITEMS = 8;
constexpr int SEG_TILE = SEG_THREADS * SEG_ITEMS;

// Decoupled look-back status word: [63:32] epoch, [31:30] flag, [29:0] value.
enum : uint32_t { LB_NONE = 0u, LB_AGG = 1u, LB_INC = 2u };
__host__ __device__ inline uint64_t lb_pack(uint32_t epoch, uint32_t flag, uint32_t value) {
    return ((uint64_t)epoch << 32) | ((uint64_t)flag << 30) | (uint64_t)(value & 0x3fffffffu);
}

// Programmatic dependent launch on the grouping chain (trie pass hist -> scatter ->
// ... -> fused leaf, one stream): a kernel launched by launch_pdl may be scheduled
// while its predecessor's last wave still runs; pdl_enter() -- its first statement --
// waits until the predecessor has completed and its writes are visible, then lets
// the next kernel of the chain be scheduled the same way (single-wave kernels whose
// CTAs stay resident trigger only after their main loop -- pdl_wait() first,
// pdl_trigger() late -- so waiting CTAs do not hold SM slots the other stream could
// use). In a kernel launched without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_trigger();
}
bool pdl_enabled();  // GAKCO_PDL=0 in the environment turns the attribute off (A/B)
template <typename... KA, typename... A>
cudaError_t launch_pdl(void (*kern)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       A... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, ((KA)args)...);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// Exclusive scan of one value per thread over the first 256 threads of the block.
// Must be reached by every thread of the block (threads >= 256 pass 0; their
// result is meaningless). s_w: 9 words of shared scratch.
__device__ __forceinline__ uint32_t scan256_excl(uint32_t v, uint32_t* s_w, uint32_t* total = nullptr) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (w < 8 && lane == 31) s_w[w] = inc;
    __syncthreads();
    if (w == 0) {  // exclusive prefix of the 8 warp totals (s_w[0..7]) and the total (s_w[8])
        const uint32_t x = lane < 8 ? s_w[lane] : 0u;
        uint32_t y = x;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += t;
        }
        __syncwarp();
        if (lane < 8) s_w[lane] = y - x;
        if (lane == 7) s_w[8] = y;
    }
    __syncthreads();
    const uint32_t wp = w < 8 ? s_w[w] : 0u;
    if (total) *total = s_w[8];
    __syncthreads();
    return wp + inc - v;
}

// Single-counter decoupled look-back, called by ONE thread of tile `t`:
// publishes the tile aggregate, returns the exclusive prefix of all earlier tiles
// and publishes the inclusive one. Tiles must be numbered by an ordered ticket.
__device__ __forceinline__ uint32_t lookback_one(uint64_t* status, uint32_t t, uint32_t agg,
                                                 uint32_t epoch) {
    if (t == 0) {
        *(volatile uint64_t*)(status) = lb_pack(epoch, LB_INC, agg);
        return 0;
    }
    *(volatile uint64_t*)(status + t) = lb_pack(epoch, LB_AGG, agg);
    uint32_t excl = 0;
    int64_t p = (int64_t)t - 1;
    while (true) {
        uint64_t v = *(volatile const uint64_t*)(status + p);
        uint32_t ep = (uint32_t)(v >> 32), fl = (uint32_t)(v >> 30) & 3u;
        if (ep != epoch || fl == LB_NONE) continue;
        excl += (uint32_t)(v & 0x3fffffffu);
        if (fl == LB_INC) break;
        --p;
    }
    *(volatile uint64_t*)(status + t) = lb_pack(epoch, LB_INC, excl + agg);
    return excl;
}

// Warp-cooperative decoupled look-back (all 32 lanes of ONE warp call it): the
// lanes read 32 predecessors' statuses at once, so each L2 round trip consumes up
// to 32 tiles; returns the exclusive prefix (to every lane).
__device__ __forceinline__ uint32_t lookback_warp(uint64_t* status, uint32_t t, uint32_t agg,
                                                  uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    if (t == 0) {
        if (lane == 0) *(volatile uint64_t*)(status) = lb_pack(epoch, LB_INC, agg);
        return 0;
    }
    if (lane == 0) *(volatile uint64_t*)(status + t) = lb_pack(epoch, LB_AGG, agg);
    uint32_t excl = 0;
    int64_t p = (int64_t)t - 1;
    while (true) {
        const int64_t q = p - lane;
        const uint64_t v = q >= 0 ? *(volatile const uint64_t*)(status + q)
                                  : lb_pack(epoch, LB_INC, 0);
        const uint32_t ep = (uint32_t)(v >> 32), fl = (uint32_t)(v >> 30) & 3u;
        const bool ready = ep == epoch && fl != LB_NONE;
        const uint32_t incm = __ballot_sync(0xffffffffu, ready && fl == LB_INC);
        const uint32_t notready = __ballot_sync(0xffffffffu, !ready);
        const int first = incm ? __ffs(incm) - 1 : 31;  // nearest inclusive (or the window)
        const uint32_t need = first == 31 ? 0xffffffffu : ((2u << first) - 1u);
        if (notready & need) continue;  // a needed predecessor has not published: re-read
        uint32_t val = lane <= first ? (uint32_t)(v & 0x3fffffffu) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (incm) break;
        p -= 32;
    }
    if (lane == 0) *(volatile uint64_t*)(status + t) = lb_pack(epoch, LB_INC, excl + agg);
    return excl;
}

// Lanes of the warp holding the same 8-bit digit d (ballot multisplit: 8 votes
// instead of one match.any, which stalls on the MIO pipe).
__device__ __forceinline__ uint32_t digit_peers(uint32_t d, uint32_t valid_mask) {
    uint32_t peers = valid_mask;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bal : ~bal;
    }
    return peers;
}

// Device counters of gakco_stats (int64 slots).
enum { ST_KEYS = 0, ST_PASSKEYS, ST_TRIPLES, ST_GROUPS, ST_LIGHT_PAIRS, ST_HEAVY_GROUPS,
       ST_HEAVY_MACS, ST_HEAVY_MACS4, ST_WIN_GROUPS, ST_WIN_MACS, ST_FAR_RECORDS,
       ST_PASS_KEYS, ST_COUNT };

// Error flags raised by kernels (bit mask in a device int).
enum { EF_NEGATIVE_N = 1, EF_K_MISMATCH = 2, EF_BAD_SYMBOL = 4 };

// Per-batch device views used by several kernels.
struct CorpusView {
    const uint8_t* codes;    // concatenated symbol codes
    const int64_t* off;      // [N+1] sequence offsets into codes
    const int64_t* gofs;     // [N+1] g-mer offsets (prefix sums of n_X)
    const uint32_t* gm_seq;  // [n] sequence id of each g-mer
    int64_t N;
    uint64_t n;              // total g-mers
};

struct SegmentOut {
    uint32_t* tseq;          // [T] seq id | (group-head << 31)
    uint32_t* tcnt;          // [T] run length (count of the (key, seq) pair)
    uint2* groups;           // [G] triple range [x, y) of each multi-sequence group
    uint32_t* counts;        // [0] = T, [1] = G
};

// ---- hash-partition grouping (bucket.cu) ----
constexpr int BK_SUB_TILE = 4096;  // g-mers per sub-tile of the partition passes
// Per mask: how its key is formed from the packed g-mer window w (symbol r of the
// g-mer at bits [bits*(g-1-r), bits*(g-r)) of w).
struct MaskDesc {
    uint8_t nkept, nrun, pad0, pad1;
    uint8_t kept_sh[GMAX];   // HORNER: shift of the r-th kept symbol
    uint8_t run_src[GMAX];   // RUNS: maximal runs of kept positions, as bit fields
    uint8_t run_len[GMAX];
    uint8_t run_dst[GMAX];
};
struct BkArgs {
    const uint64_t* win;      // [n] packed g-mer windows
    const uint32_t* gm_seq;   // [n] sequence of each g-mer
    uint64_t n;               // g-mers per mask
    const MaskDesc* desc;     // [nmask] this batch's masks
    int nmask, mb;            // masks in the batch, masks per CTA of the passes
    uint32_t nb, nchunks;     // buckets per mask, g-mer chunks per mask
    uint64_t T;               // g-mers per chunk
    int bits, sb;             // bits per symbol in w, sequence-id bits (>= 1)
    int runs;                 // 1: RUNS keys, 0: HORNER keys
    uint32_t sigma;
    uint32_t* H;              // [nmask][nchunks][nb] chunk histograms -> prefixes
    uint32_t* tot;            // [nmask][nb] bucket sizes
    uint32_t* bbase;          // [nmask][nb+1] bucket starts within the mask
};
struct BkScratch {            // big-bucket tables (entry offset 2*start; occ at start)
    uint64_t* tab;
    uint32_t* tcnt;
    uint32_t* gs;
    uint32_t* occ;
};
cudaError_t launch_windows(const CorpusView& cv, int g, int bits, uint64_t* win, int sm_count,
                           cudaStream_t s);
int bk_masks_per_cta(uint32_t nb);
cudaError_t launch_bucket_count(const BkArgs& a, bool k64, cudaStream_t s);
cudaError_t launch_bucket_scatter(const BkArgs& a, void* out, bool k64, cudaStream_t s);
cudaError_t launch_bucket_group(const BkArgs& a, const void* keys, bool k64, int64_t dstride,
                                int64_t* diag, SegmentOut so, BkScratch sc,
                                unsigned long long* stats, int sm_count, cudaStream_t s);

// ---- launchers (each returns cudaGetLastError()) ----
cudaError_t launch_gmer_index(const int64_t* gofs, int64_t N, uint32_t* gm_seq, cudaStream_t s);
cudaError_t launch_symbol_hist(const uint8_t* codes, int64_t len, unsigned long long* hist,
                               int sm_count, cudaStream_t s);
cudaError_t launch_check_codes(const uint8_t* codes, int64_t len, int sigma, int* flags,
                               cudaStream_t s);
// Keys are u64, or u32 (k64 = false) when key bits + sequence bits <= 32.
cudaError_t launch_encode(const CorpusView& cv, const uint8_t* kept, int nkept, int sigma, int sb,
                          int nmask, int npass, void* out, bool k64, uint32_t* hist,
                          cudaStream_t s);
// Encode from packed windows (win[j]: g codes, bits each, first most significant);
// kept_sh[b*GMAX + r] = bits*(g-1-kept_r) of mask b.
cudaError_t launch_encode_win(const uint64_t* win, const uint32_t* gm_seq, uint64_t n,
                              const uint8_t* kept_sh, int nkept, int sigma, int bits, int sb,
                              int nmask, void* out, bool k64, cudaStream_t s);
cudaError_t launch_onesweep(const uint64_t* in, uint64_t* out, uint64_t n, int nseg, int shift,
                            const uint32_t* hist, int pass, int npass, uint64_t* status,
                            uint32_t* ctr, uint32_t epoch, cudaStream_t s);
// Chunked LSD pass (radix_hist + radix_scatter); hist: >= (target_ctas + nseg) * 256 u32.
// batched mask trie pass descriptor (one per segment of a launch)
struct PassDesc {
    uint64_t in_off;   // first key of the segment's input (elements)
    uint64_t out_off;  // first key of its output
    uint64_t omask;    // output = key & omask (a leaf: the mask's key bits | seq bits)
    uint8_t sh[4];     // bit offsets of the digit's symbols (least significant first)
    uint32_t nsym;     // symbols in the digit (1..4)
    uint32_t symbits;  // bits per symbol
};
template <typename K>
__device__ __forceinline__ uint32_t pd_digit(K k, const PassDesc& d) {
    const uint32_t m = (1u << d.symbits) - 1u;
    uint32_t v = (uint32_t)(k >> d.sh[0]) & m;
    if (d.nsym > 1) v |= ((uint32_t)(k >> d.sh[1]) & m) << d.symbits;
    if (d.nsym > 2) v |= ((uint32_t)(k >> d.sh[2]) & m) << (2 * d.symbits);
    if (d.nsym > 3) v |= ((uint32_t)(k >> d.sh[3]) & m) << (3 * d.symbits);
    return v;
}
cudaError_t launch_trie_batch(const void* in, void* out, bool k64, uint64_t n, int nseg,
                              const PassDesc* desc, uint32_t* hist, int target_ctas,
                              cudaStream_t s, int* nlaunch);
cudaError_t launch_trie_root(const uint64_t* win, const uint32_t* seq, uint64_t n, int sb,
                             bool k64, void* out, int sm_count, cudaStream_t s);
cudaError_t launch_trie_pass(const uint64_t* win, uint64_t* wout, const void* sin, void* sout,
                             bool seq16, uint64_t n, int shift, uint32_t dmask, uint64_t omask,
                             uint32_t* hist, int target_ctas, cudaStream_t s, int* nlaunch);
// Σ <= 64 variant (trie.cu): hist + scatter (chunk prefixes computed in the scatter);
// cntp: device element count (nullptr: n); n: capacity (grid size)
constexpr int TP_HG_MAX_BLOCKS = 128;  // block sums of 8 chunk histograms (trie.cu), per parity
bool trie_pass64_ok(uint32_t dmask);
cudaError_t launch_trie_pass64(const uint64_t* win, uint64_t* wout, const void* sin, void* sout,
                               bool seq16, uint64_t n, const uint32_t* cntp, int shift,
                               uint32_t dmask, uint64_t omask, uint32_t* H, int target_ctas,
                               cudaStream_t s, uint32_t* cnt_out = nullptr,
                               unsigned long long* stats = nullptr, uint32_t* Hg = nullptr,
                               uint32_t* par_ctr = nullptr);  // Hg: block sums (2 parities,
                               // zero at first use); *par_ctr: the host's pass parity counter
cudaError_t launch_tp_records(const void* in, void* out, bool k32, uint64_t n, const uint32_t* cntp,
                              int shift, uint32_t* H, int target_ctas, cudaStream_t s);
cudaError_t launch_fill_u32(uint32_t* p, uint32_t v, uint32_t count, cudaStream_t s);
// segrag.cu: the cross-level chain's leaves, ragged segments (cnt[s] valid elements
// of segment s at [s n, s n + cnt[s])), km[s] the key mask of segment s; cw != nullptr:
// also the compacted copy of segment s (elements of groups of >= 2) at cw/cs + s n,
// its length at ccnt[s] (zeroed by the caller)
cudaError_t launch_segment_rag(const uint64_t* w, const void* sq, bool seq16, uint64_t n, int nseg,
                               const uint32_t* cnt, const uint64_t* km, int64_t dstride,
                               int64_t* diag, uint32_t* counters, SegmentOut so,
                               unsigned long long* stats, cudaStream_t s, uint64_t* cw,
                               void* cs, uint32_t* ccnt, bool reset = true,
                               unsigned max_ctas = 0);
// leaf.cu: a mask's last pass (by the symbol at shift / dmask) over an array grouped
// by pmask, fused with the run-length of segrag.cu (kmask: the mask's key). Appends to
// so (counters = so.counts, not reset); cw/cs/ccnt: the compacted copy (optional);
// groups larger than the tile are split into ow/os at atomicAdd(ocnt) (for segrag)
// a group of the pass before too large for a leaf CTA, queued for leaf_big_kernel
struct LfBig {
    const uint64_t* w;  // the input array (grouped by pmask) and its ids
    const void* sq;
    uint64_t* ow;       // the mask's overflow slot, its fill
    void* os;
    uint32_t* ocnt;
    uint64_t start;     // the group's first element; the array's element count
    uint64_t cnt;
    uint64_t pmask;
    int shift;
    uint32_t dmask;
};
struct LfBigList {
    LfBig* e;
    uint32_t* count;  // [0] entries queued, [1] entries claimed (both zeroed per batch)
    uint32_t cap;
};
cudaError_t launch_zero_upper(int64_t* C, int64_t N, int levels, int sm_count, cudaStream_t s);
int leaf_tile(bool wide = false);  // group heads per CTA of launch_leaf
// the queued large groups of a batch, split into their overflow slots (after the
// batch's launch_leaf calls, before the segment kernel over the overflow slots)
cudaError_t launch_leaf_big(LfBigList bl, bool seq16, int sm_count, cudaStream_t s);
cudaError_t launch_leaf(const uint64_t* w, const void* sq, bool seq16, uint64_t n,
                        const uint32_t* cntp, uint64_t pmask, uint64_t kmask, int shift,
                        uint32_t dmask, int64_t dstride, int64_t* diag, SegmentOut so,
                        unsigned long long* stats, uint64_t* cw, void* cs, uint32_t* ccnt,
                        uint64_t* ow, void* os, uint32_t* ocnt, LfBigList bl, cudaStream_t s,
                        bool wide = false);  // wide: 12 items per thread (1536-element ranges)
cudaError_t launch_seq16(const uint32_t* a, uint16_t* b, uint64_t n, int sm_count,
                         cudaStream_t s);
cudaError_t launch_radix_chunked2(const void* in, void* out, bool k64, uint64_t n, int nseg,
                                  int shift, uint32_t* hist, int target_ctas, int rank_mode,
                                  cudaStream_t s, int* nlaunch);
cudaError_t launch_radix_chunked(const void* in, void* out, bool k64, uint64_t n, int nseg,
                                 int shift, uint32_t* hist, int target_ctas, cudaStream_t s);
// counters: 2 u32 (triples, groups) reserved per tile; zeroed by the launcher.
// diag[X * dstride] receives the within-sequence repeat term of C_m(X,X)
cudaError_t launch_segment_soa(const uint64_t* w, const void* sq, bool seq16, uint64_t n,
                               int nseg, int64_t dstride, int64_t* diag, uint32_t* counters,
                               SegmentOut so, unsigned long long* stats, cudaStream_t s,
                               const uint64_t* km = nullptr);
cudaError_t launch_segment(const void* keys, bool k64, uint64_t n, int nseg, int sb,
                           int64_t dstride, int64_t* diag, uint32_t* counters, SegmentOut so,
                           unsigned long long* stats, cudaStream_t s, const uint64_t* km = nullptr);
// Light pair updates; a group with >= heavy_min sequences (and counts <= 255)
// instead claims column c = atomicAdd(dense_fill) (< ldd) of the dense count
// matrix D (u8, slabs of 128 columns: byte (c/128)*n_pad*128 + row*128 + c%128)
// and scatters its counts there, for the tensor-core Gram.
// Record buckets for light updates when the accumulator is much larger than L2:
// nb buckets of cap u32 records, bucket b covering accumulator cells
// [b*block_cells, (b+1)*block_cells); nb = 0 disables binning.
struct LightBins {
    uint32_t* rec;
    uint32_t* cnt;
    uint64_t cap;
    uint64_t block_cells;
    int nb;
};
// Window Gram (relabelled accumulator): a light group whose relabelled members lie
// in one window of 256 labels [128 w, 128 w + 256) becomes a u8 count column of that
// window's dense block, multiplied on the tensor cores (gram_tc.cu); nw = 0: off.
constexpr int WIN_ROWS = 256;   // labels per window
constexpr int WIN_STEP = 128;   // window starts
struct WinArgs {
    uint32_t* fill;   // [2][nw] columns claimed per window; [1]: this batch's first
    uint2* list;      // [nw][cap] triple range of each claimed group
    uint32_t cap;     // columns per window
    uint32_t nw;      // windows (0: the window path is off)
    uint32_t wmin;    // smallest group (sequences) taken
};
// Far-pair records (relabelled accumulator far beyond L2): a light pair
// whose labels are >= near apart (a random cross-cluster match: its cell would miss
// L2, 24 G REDs/s into 800 MB vs 208 G/s into 32 MB) is appended as a record
// (cell << 24 | val) to per-warp chunks of rec instead of a RED; launch_far_apply
// buckets the records by accumulator block and adds them block by block (L2-resident
// REDs). fill[0] counts reserved record slots (chunks of FAR_CHUNK; every reserved
// slot is written, unused ones with 0); a chunk past cap is never reserved (the warp
// falls back to REDs). near = 0: off.
constexpr uint32_t FAR_CHUNK = 256;
struct FarRec {
    uint64_t* rec;     // [cap] records: u64 cell << 24 | val, or (k32) u32 cell << 4 | val
    uint32_t* fill;    // [0] slots reserved (all warps)
    uint64_t cap;      // a multiple of FAR_CHUNK
    uint32_t near;     // label distance from which a pair is far (0: off)
    bool k32 = false;  // 4-byte records (cells < 2^28, values 1..15; larger values: REDs)
};
// every pending record into acc (ntri cells); H: >= 2 * sm_count * 64 + 72 u32 scratch
cudaError_t launch_far_apply(FarRec fr, void* scratch, uint32_t* H, int bshift,
                             uint32_t* acc, uint64_t ntri, int sm_count, cudaStream_t s);
cudaError_t launch_window_build(SegmentOut so, WinArgs wa, const uint32_t* perm, uint8_t* wD,
                                int sm_count, cudaStream_t s);
cudaError_t launch_window_gram(uint8_t* wD, WinArgs wa, int64_t* wC, const int2* tiles,
                               int ntiles, int sm_count, unsigned long long* stats,
                               cudaStream_t s);
cudaError_t launch_window_flush(int64_t* wC, uint32_t nw, const uint32_t* inv, int64_t N,
                                int64_t* Cm, int sm_count, cudaStream_t s);
cudaError_t launch_light(SegmentOut so, uint64_t max_groups, int64_t heavy_min, int64_t N,
                         uint32_t* acc, uint2* heavy_list, uint64_t ldd,
                         uint32_t* dense_fill, LightBins bins, uint32_t flat_max,
                         int64_t NA, const uint32_t* perm, uint32_t heavy_cmax,
                         unsigned long long* stats, int sm_count, cudaStream_t s,
                         WinArgs wa = WinArgs{nullptr, nullptr, 0, 0, 0}, bool big = false,
                         FarRec fr = FarRec{nullptr, nullptr, 0, 0}, int ctas = 3,
                         int grid_per_sm = 0);
// Light accumulator relabelled by perm (sequence -> accumulator index): flush it into
// C_m (original order) and zero it.
cudaError_t launch_light_flush_perm(uint32_t* acc, int64_t N, int64_t* Cm, const uint32_t* perm,
                                    int sm_count, cudaStream_t s);
// Clusters of sequences for the relabelling: union of every X with its best partner
// argmax_Y C(X,Y) (C upper triangle); parent[X] <- root. iota: [N] = 0..N-1.
cudaError_t launch_cluster_roots(const int64_t* C, int64_t N, unsigned long long* best,
                                 uint32_t* parent, const uint32_t* iota, int sm_count,
                                 cudaStream_t s);
// device relabelling: keys root << 32 | x; labels from the root-sorted keys
cudaError_t launch_relabel_keys(const uint32_t* root, int64_t N, uint64_t* keys, cudaStream_t s);
cudaError_t launch_relabel_perm(const uint64_t* keys, int64_t N, uint32_t* perm, uint32_t* inv,
                                cudaStream_t s);
// rectangular accumulator (NA x NB, row-major) -> C_m (NA x NB), zeroed
cudaError_t launch_light_flush_rect(uint32_t* acc, uint64_t cells, int64_t* Cm, int sm_count,
                                    cudaStream_t s);
// Fill the D slabs of the columns claimed by this batch ([prev, fill) with
// prev = dense_fill[1], a multiple of 128) from the batch's triples, in shared
// memory, with full-line stores; then round dense_fill[0] up to a multiple of 128
// and set dense_fill[1] = dense_fill[0].
// sorted = 1: each group's triples are in ascending sequence order (LSD path).
cudaError_t launch_build_dense(SegmentOut so, const uint2* heavy_list, uint32_t* dense_fill,
                               uint8_t* D, int64_t n_pad, uint64_t ldd, int sorted, int fp4,
                               int sm_count, cudaStream_t s);
// acc: u32 strictly-upper packed triangle (N(N-1)/2); flush adds it into C_m, zeroes it.
cudaError_t launch_light_flush(uint32_t* acc, int64_t N, int64_t* Cm, int sm_count,
                               cudaStream_t s);
// Heavy path (gram_tc.cu): C_m += D D^T over the *dense_fill filled columns
// (count read on the device), then the used columns are zeroed and the fill reset.
std::vector<int2> gram_tiles(int64_t n_pad);
// K split of a Gram flush: smallest ks in 1..16 with tiles*ks / (waves*workers) >= 0.9
inline int gram_ksplit(int ntiles, int workers) {
    if (ntiles <= 0 || workers <= 0) return 1;
    int best = 1;
    double best_eff = 0.0;
    for (int ks = 1; ks <= 16; ++ks) {
        const long units = (long)ntiles * ks;
        const long waves = (units + workers - 1) / workers;
        const double eff = (double)units / (double)(waves * workers);
        if (eff >= 0.9) return ks;
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = ks;
        }
    }
    return best;
}
cudaError_t launch_gram_flush(uint8_t* D, int64_t n_pad, uint64_t ldd, uint32_t* dense_fill,
                              int64_t* Cm, int64_t N, const int2* tiles, int ntiles,
                              int sm_count, unsigned long long* stats, cudaStream_t s);
// CTA-pair variant (gram2.cu): 256 x 512 pair tiles, n_pad a multiple of 512.
// NA > 0: rectangular block C_m[X][Y - NA] += (D D^T)[X][Y], X < NA <= Y (C_m is NA x
// (N - NA)), over the tiles of gram2_tiles_rect.
std::vector<int2> gram2_tiles(int64_t n_pad);
std::vector<int2> gram2_tiles_rect(int64_t NA, int64_t NB);
// e2m1 (kind::mxf4) variant: 256 x 256 pair tiles, D packed 4-bit (slabs of 256
// columns), f32 accumulation (exact below 2^24 per entry and flush)
std::vector<int2> gram4_tiles(int64_t n_pad);
std::vector<int2> gram4_tiles_rect(int64_t NA, int64_t NB);
cudaError_t launch_gram4_flush(uint8_t* D, int64_t n_pad, uint64_t ldd, uint32_t* dense_fill,
                               int64_t* Cm, int64_t N, const int2* tiles, int ntiles,
                               int sm_count, unsigned long long* stats, cudaStream_t s,
                               int64_t NA);
cudaError_t launch_gram2_flush(uint8_t* D, int64_t n_pad, uint64_t ldd, uint32_t* dense_fill,
                               int64_t* Cm, int64_t N, const int2* tiles, int ntiles,
                               int sm_count, unsigned long long* stats, cudaStream_t s,
                               int64_t NA = 0);
cudaError_t launch_diag_closed_form(const int64_t* gofs, int64_t N, int64_t nmask, int64_t* diag,
                                    int64_t dstride, cudaStream_t s);
// Rectangular epilogue: C [M+1][NA][N-NA], Dg [M+1][N] diagonals -> Nm, K, Knorm
// [.][NA][N-NA] and kdiag[N] = K(X,X).
cudaError_t launch_epilogue_rect(const int64_t* C, const int64_t* Dg, int64_t N, int64_t NA, int g,
                                 int k, int M, int64_t* Nm, int64_t* K, double* Knorm,
                                 int64_t* kdiag, int* flags, int sm_count, cudaStream_t s);
cudaError_t launch_epilogue(int64_t* C, int64_t N, int g, int k, int M, int64_t* Nm, int64_t* K,
                            double* Knorm, int64_t* kdiag, int* flags, cudaStream_t s);

// ---- mask-sharded step (shard.cu, epilogue.cu) ----
constexpr int MAX_PEERS = 64;
struct PeerPtrs {
    void* p[MAX_PEERS];  // device (peer-mapped) receive buffers, one per rank
};
cudaError_t launch_pack_upper_peers(const int64_t* C, int64_t N, int level, int levels,
                                    int64_t chunk, const PeerPtrs& dst, int src, int out_bytes,
                                    cudaStream_t s);
// entries [begin, end) of the packed upper triangle of `levels` N x N matrices -> out
// [levels][end - begin] as int64 (out_bytes 8) or u32 (4, truncating)
cudaError_t launch_pack_upper(const int64_t* C, int64_t N, int levels, int64_t begin, int64_t end,
                              void* out, int out_bytes, cudaStream_t s);
cudaError_t launch_diag(const int64_t* C, int64_t N, int levels, int64_t* out, int sm_count,
                        cudaStream_t s);
// complete packed C slice [M+1][end - begin] (int64 or u32) + complete diagonals Dg
// [M+1][N] -> packed Nm [M+1][end - begin], K, Knorm [end - begin]; kdiag [N] scratch
cudaError_t launch_epilogue_packed(const void* Cp, int in_bytes, int nsrc, int64_t ld, const int64_t* Dg, int64_t N,
                                   int64_t begin, int64_t end, int g, int k, int M, int64_t* Nm,
                                   int64_t* K, double* Knorm, int64_t* kdiag, int* flags,
                                   cudaStream_t s);

}  // namespace gk
