/*
 * gakco.h — C-ABI of the B200 gapped k-mer kernel-matrix engine (libgakco.so).
 *
 * Computes, for a corpus of N sequences over an alphabet of Σ symbol codes, the
 * GaKCo quantities of arXiv 1704.07468 (PAPER.md = P):
 *
 *   C_m(X,Y)   cumulative mismatch profile: over all C(g,m) ways of removing m of
 *              the g positions of a g-mer, the number of ordered g-mer pairs
 *              (a in X, b in Y) whose remaining (g-m)-mers are equal
 *              (Algorithm 1 MISMATCHPROFILE), m = 0..M;
 *   N_m(X,Y)   mismatch profile, pairs at Hamming distance exactly m
 *              (Definition 1), from Eq. 9: N_m = C_m - sum_{j<m} C(g-j,m-j) N_j
 *              (Algorithm 1 lines 18-21);
 *   K(X,Y)     = sum_{m=0}^{min(M,g-k)} h_m N_m, h_m = C(g-m,k) (Eq. 6-7);
 *   Knorm(X,Y) = K(X,Y)/sqrt(K(X,X) K(Y,Y)) in fp64, 0 when a diagonal entry is 0,
 *              exactly 1.0 on the diagonal where K(X,X) > 0 (BASELINE.json).
 *
 * g-mers of a sequence of length l start at positions 0..l-g (a sequence shorter
 * than g has none and yields a zero row). Self-pairs are counted on the diagonal
 * (readings A2, A7).
 *
 * Conventions for every function:
 *  - Returns GAKCO_OK or an error code; never aborts. gakco_last_error(plan)
 *    returns a per-plan message for the most recent error.
 *  - Matrices are row-major int64 (C, Nm, K) or fp64 (Knorm), little-endian,
 *    full symmetric N x N, stacked [m][X][Y] for C and Nm. Sequence order is input
 *    order.
 *  - The caller owns every input and output buffer. The plan owns its device
 *    scratch, which it allocates on first use and reuses.
 *  - All work is enqueued on `cuda_stream` (a cudaStream_t; NULL = legacy default
 *    stream). Calls that must read device data back (validation, host outputs)
 *    synchronise that stream.
 *  - One plan per host thread / stream. Results are bit-identical across runs,
 *    shard counts, batch sizes and heavy/light thresholds (integer sums).
 */
#ifndef GAKCO_H
#define GAKCO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gakco_plan gakco_plan;  /* opaque */

typedef enum {
    GAKCO_OK = 0,
    GAKCO_E_ARG = 1,       /* invalid parameter, pointer or shape */
    GAKCO_E_SYMBOL = 2,    /* a code >= sigma in the corpus */
    GAKCO_E_RANGE = 3,     /* key+seq id do not fit 64 bits, more than 2^30 g-mers in the
                              corpus, a sequence with more than 65535 g-mers (the light
                              path's u32 pair sums need n_X * n_Y < 2^32), or a C_m / K
                              entry bound (C(g,m) n_max^2) overflows int64 */
    GAKCO_E_NOMEM = 4,     /* device allocation failed */
    GAKCO_E_CUDA = 5,      /* a CUDA runtime error */
    GAKCO_E_INTERNAL = 6   /* a failed invariant (negative N_m, K != C_{g-k}) */
} gakco_status;

/* Tuning / testing options (gakco_set_option). Results never depend on them. */
typedef enum {
    GAKCO_OPT_HEAVY_MIN_SEQS = 1, /* groups with at least this many distinct sequences
                                     go to the dense tensor-core Gram; 0 = automatic,
                                     a huge value = never (all light); 2 = all heavy */
    GAKCO_OPT_BATCH_KEYS = 2,     /* max keys (masks x g-mers) per batch; 0 = auto */
    GAKCO_OPT_TIMING = 3,         /* 1 = record per-stage CUDA events (gakco_get_stats) */
    GAKCO_OPT_SORT = 4,           /* grouping of masked keys: -1 = automatic (default): the
                                     mask trie (6) when a mask has >= 2M g-mers and
                                     g*ceil(log2 sigma) <= 64, else the batched mask trie (7)
                                     when the one-word composite fits 64 bits, else the
                                     chunked LSD v2 (3); 0 = LSD radix sort,
                                     chunked two-kernel passes (v1), 1 = LSD onesweep with
                                     decoupled look-back, 2 = hash partition + shared-memory
                                     hash grouping (falls back to the LSD sort where it does
                                     not apply: g*ceil(log2 sigma) > 64 or > 16M g-mers),
                                     3/4/5 = chunked LSD v2 (tiles streamed by bulk copies;
                                     ranking by shared atomicOr match / match.any / ballots),
                                     6 = mask trie: per-position stable passes over packed
                                     windows + sequence ids, passes of common leading kept
                                     positions shared between masks (auto when a mask has
                                     >= 2M g-mers and g*ceil(log2 sigma) <= 64),
                                     7 = batched mask trie over one-word composites (window
                                     << sb | seq): up to 4 symbols per pass, a batch's trie
                                     run depth by depth, one launch per depth (auto below
                                     2M g-mers when g*ceil(log2 sigma) + ceil(log2 N) <= 64)
                                     */
    GAKCO_OPT_SORT_CTAS_PER_SM = 5, /* chunked pass grid size in CTAs per SM (defaults: 4 for
                                       the batched LSD passes on u64 composites, 8 on u32,
                                       2 for the mask trie; setting it sets all three) */
    GAKCO_OPT_LIGHT_BINS = 6,     /* light updates binned by accumulator block (ablation /
                                     test knob): <= 0 = never (default; measured slower on
                                     Scale), > 0 = always, with this many cells per block */
    GAKCO_OPT_GRAM_PAIR = 7,      /* heavy-group Gram kernel: 1 = CTA pairs (tcgen05
                                     cta_group::2, 256 x 512 tiles; default), 0 = one SM per
                                     128 x 256 tile */
    GAKCO_OPT_LIGHT_FLAT = 8,     /* light groups of <= this many sequences (1..32, default
                                     8) have their pairs flattened across a warp; bigger
                                     ones are enumerated from registers, one group per warp */
    GAKCO_OPT_LIGHT_RELABEL = 9,  /* light accumulator sequence relabelling (locality; results
                                     unchanged): -1 = automatic (default: when the packed
                                     triangle exceeds 96 MB), 0 = off, 1 = on */
    GAKCO_OPT_GRAM_FP4 = 10,      /* heavy-group Gram operands, per level m: -1 = automatic
                                     (default): e2m1 counts (kind::mxf4 block-scaled, unit
                                     scales) when one mask's n_max^2 < 2^24 keeps the f32 sums
                                     exact AND n_max * p_max^(g-m) <= 1/8 (p_max: share of the
                                     most frequent symbol), so counts > 4 -- which e2m1 cannot
                                     hold and which stay on the light path -- are rare; else u8
                                     (kind::i8). 0 = u8 at every level, 1 = e2m1 at every level
                                     where exact */
    GAKCO_OPT_PIPELINE = 11,      /* 1 (default): light updates, dense build and Gram of batch b
                                     run on a second stream while batch b+1 is encoded, sorted
                                     and segmented (double-buffered triples); 0: one stream */
    GAKCO_OPT_LEVEL_ORDER = 12    /* 0 (default): levels processed m = 0..M; 1: m = M..0 (the
                                     top level's Gram overlaps the rest: Protein 8.0 -> 7.8 ms
                                     but DNA 9.26 -> 9.51 ms; ascending whenever the light
                                     accumulator is relabelled) */,
    GAKCO_OPT_LIGHT_WINDOW = 13,  /* window Gram of cluster-local light groups: once the light
                                     accumulator is relabelled (GAKCO_OPT_LIGHT_RELABEL), a
                                     group whose labels lie in one window of 256 labels becomes
                                     a u8 count column of that window's 256 x 256 block,
                                     multiplied on the tensor cores (kind::i8) and added back
                                     through the inverse labelling. -1 = automatic (default:
                                     with relabelling), 0 = off, 1 = on (relabels) */
    GAKCO_OPT_WINDOW_MIN = 14,    /* smallest group (sequences) for the window Gram (default 9;
                                     groups of <= GAKCO_OPT_LIGHT_FLAT sequences stay light) */
    GAKCO_OPT_GRAM_EACH = 15,     /* 1: the heavy-group Gram runs after every batch (overlapping
                                     the next batch) instead of when a level ends or D fills;
                                     0 (default) */
    GAKCO_OPT_TRIE_PASS = 16,     /* mask-trie pass kernel: 1 (default) = the symbol-digit pass
                                     (<= 64 buckets, chunk prefixes inside the scatter: two
                                     launches) where sigma <= 64; 0 = the generic 8-bit radix
                                     pass (hist + chunk scan + scatter) */
    GAKCO_OPT_RELABEL_HOST = 22,  /* 1: the relabelling's sort by cluster runs on the host (one
                                     host round trip per call); 0 (default): on the device */
    GAKCO_OPT_LEAF_FUSE = 23,     /* mask trie with the cross-level chain: 1 (default) = a mask's
                                     last pass is fused with its run-length (leaf.cu: each CTA
                                     ranks whole groups of the pass before in shared memory;
                                     no leaf array), where the groups of the pass before are
                                     small (the expected largest, n f_max^positions, <= 8
                                     tiles of 768 g-mers); 0 = a global pass + the segment
                                     kernel */
    GAKCO_OPT_FAR_BYTES = 21,     /* far-pair record width: 0 = automatic (4 bytes -- cell << 4 |
                                     value, values 1..15, larger ones as REDs -- when every cell
                                     index fits 28 bits, else 8), 4, 8 */
    GAKCO_OPT_LIGHT_GRID = 20,    /* light kernel grid size in CTAs per SM (0 = automatic: 3 for
                                     a relabelled accumulator, else 8); fewer leave room for the
                                     next batch's sort / segment kernels on the other stream */
    GAKCO_OPT_LIGHT_CTAS = 19,    /* register budget of the relabelled light kernel: CTAs per SM
                                     it is compiled for (3, 4 = default, 6) */
    GAKCO_OPT_XL_COMPACT = 18,    /* cross-level mask-trie chain (levels processed as k rises, a
                                     level-m mask one pass over its level-(m+1) parent): 1
                                     (default) = each level keeps only the elements of groups of
                                     >= 2 g-mers for its children (a g-mer alone under a mask
                                     stays alone under every refinement; its diagonal term is
                                     the closed form), 0 = full arrays */
    GAKCO_OPT_FAR_NEAR = 17       /* far-pair records of the light path: once the accumulator is
                                     relabelled and larger than 96 MB, a pair whose labels are
                                     >= this far apart (random cross-cluster matches, whose cells
                                     miss L2) is appended as a record and added per accumulator
                                     block after its batch (L2-resident) instead of a RED into
                                     DRAM. -1 = automatic (default: 256 when the relabelled
                                     accumulator exceeds 96 MB), 0 = off (all REDs), > 0 = this
                                     distance whenever the accumulator is relabelled */
} gakco_option;

/* Counters of the last gakco_accumulate (algorithmic units). */
typedef struct {
    int64_t masks;          /* masks processed by this plan's shard */
    int64_t keys;           /* masked g-mer keys encoded and sorted */
    int64_t sort_passes;    /* sum over batches of 8-bit LSD passes x keys */
    int64_t triples;        /* (key, seq, count) runs */
    int64_t groups_multi;   /* groups with >= 2 distinct sequences */
    int64_t light_pairs;    /* off-diagonal pair updates done by the light path */
    int64_t heavy_groups;   /* groups sent to the tensor-core Gram */
    int64_t heavy_macs;     /* u8 multiply-accumulates issued by the Gram */
    int64_t launches;       /* kernels launched by the last accumulate + finalize */
    double ms_encode, ms_sort, ms_segment, ms_light, ms_heavy, ms_epilogue;  /* ms_heavy:
                               the Gram flushes; building D is ms_dense */
    /* kernel launches per stage (same stages as the ms_* fields) */
    int64_t n_encode, n_sort, n_segment, n_light, n_heavy, n_epilogue;
    int64_t keys32;         /* of `keys`, those carried as 32-bit composites */
    int64_t sort_passes32;  /* of `sort_passes`, those over 32-bit composites */
    int64_t grouping;       /* path of the last accumulate: 0 chunked LSD sort,
                               1 onesweep LSD sort, 2 hash partition (bucket.cu),
                               3 mask trie, 4 batched mask trie */
    double ms_dense;        /* building the dense u8 count columns of heavy groups */
    int64_t n_dense;
    int64_t n_pad;          /* rows of the dense count matrix (0: no tensor-core Gram) */
    int64_t gram_fp4;       /* bit m set: level m's Gram ran on e2m1 counts (kind::mxf4);
                               clear: u8 (kind::i8). Chosen per level (GAKCO_OPT_GRAM_FP4) */
    int64_t heavy_macs_fp4; /* the part of heavy_macs issued as e2m1 (kind::mxf4) */
    int64_t win_groups;     /* light groups sent to the window Gram (GAKCO_OPT_LIGHT_WINDOW) */
    int64_t win_macs;       /* u8 multiply-accumulates issued by the window Gram */
    int64_t far_records;    /* light pair updates applied as far-pair records */
    double ms_far;          /* bucketing + adding the far-pair records (GAKCO_OPT_FAR_NEAR) */
    int64_t n_far;
    int64_t pass_keys;      /* elements actually moved by the mask-trie passes (device count;
                               sort_passes counts capacities on the compacted chain) */
    int64_t far_overflow;   /* warps whose far-record chunk claim found the buffer full (their
                               remaining far pairs of that batch went to REDs; results unchanged) */
    double ms_host;         /* host wall time of the last gakco_accumulate call (enqueueing;
                               the host waits only where the GPU is behind) */
} gakco_stats;

/* Create a plan for alphabet size sigma (1..255), g-mer length g (1..32),
 * k-mer length k (1..g) and maximum mismatch level M (0..g; the paper's M=g-k,
 * P:49). M < g-k truncates Eq. 7; M > g-k adds levels with h_m = 0. device is a
 * CUDA ordinal. On success *out is a new plan (free with gakco_destroy). */
gakco_status gakco_create(int sigma, int g, int k, int M, int device, gakco_plan** out);

/* Restrict this plan to the masks with global index = rank (mod world), the
 * masks enumerated level by level (m = 0..M) and lexicographically within a
 * level (P:127, P:141, P:454 — the C(g,m) masks are independent). Default 0 of 1. */
gakco_status gakco_set_shard(gakco_plan* plan, int rank, int world);

gakco_status gakco_set_option(gakco_plan* plan, int option, int64_t value);

/* Zero the upper triangles (Y >= X, diagonal included) of `levels` consecutive N x N
 * int64 matrices at device pointer C (the part gakco_accumulate adds into and
 * gakco_finalize reads: half the bytes of zeroing C whole). Asynchronous on
 * cuda_stream. */
gakco_status gakco_zero_upper(gakco_plan* plan, int64_t* C, int64_t N, int levels, void* cuda_stream);

/* Add this shard's contribution to C: for each of its masks, every pair of
 * sequences sharing a masked key adds count_X*count_Y.
 * A code >= sigma gives GAKCO_E_SYMBOL: here if codes is a host pointer; for a
 * device pointer the check runs on the device (no host sync) and the error is
 * returned by the next gakco_finalize (C is then meaningless).
 *   codes    uint8[offsets[N]] symbol codes (host or device pointer)
 *   offsets  int64[N+1], offsets[0] = 0, non-decreasing (host or device)
 *   C        int64[(M+1)*N*N] DEVICE pointer; the UPPER triangle (Y >= X,
 *            diagonal included) is incremented, the lower triangle is not touched.
 *            Zero it before the first call; partial C of several shards add up. */
gakco_status gakco_accumulate(gakco_plan* plan, const uint8_t* codes, const int64_t* offsets,
                              int64_t N, int64_t* C, void* cuda_stream);

/* From a complete upper-triangular C (all masks accumulated): mirror C to full
 * symmetric in place, then write Nm (Eq. 9), K (Eq. 7) and Knorm. Nm, K and
 * Knorm may be NULL (not produced) and may be host or device pointers; C must
 * be a device pointer. Fails with GAKCO_E_INTERNAL if an N_m entry is negative
 * or K != C_{g-k} (when M >= g-k). */
gakco_status gakco_finalize(gakco_plan* plan, int64_t* C, int64_t N, int64_t* Nm,
                            int64_t* K, double* Knorm, void* cuda_stream);

/* gakco_accumulate over all masks (shard ignored) followed by gakco_finalize.
 * C may be NULL (plan scratch is used); any output pointer may be host or
 * device. This is the single-call public entry point. */
gakco_status gakco_kernel(gakco_plan* plan, const uint8_t* codes, const int64_t* offsets,
                          int64_t N, int64_t* C, int64_t* Nm, int64_t* K, double* Knorm,
                          void* cuda_stream);

/* K-only fast path. Because C(g-j, g-k-j) = C(g-j, k) =
 * h_j, Eq. 8 at m = g-k is exactly Eq. 7: K = C_{g-k}. So K
 * needs only the C(g, g-k) masks of level g-k — no other level and no Eq. 9.
 * Requires M >= g-k (the paper's M = g-k; GAKCO_E_ARG otherwise). Writes K and/or
 * Knorm (either may be NULL, host or device pointers). Shard setting ignored. */
gakco_status gakco_kernel_k(gakco_plan* plan, const uint8_t* codes, const int64_t* offsets,
                            int64_t N, int64_t* K, double* Knorm, void* cuda_stream);

/* Rectangular train x test kernel. The corpus holds the NA
 * training sequences first, then the NB = N - NA test sequences. Computes the
 * NA x NB block (rows = train, columns = test) of C_m, N_m, K and Knorm of the
 * concatenated corpus — what the SVM decision function needs, K(x_i, x) (Eq. 1,
 * P:66; the paper concatenates train and test into one N x N matrix) —
 * without any train x train or test x test pair update, plus Kdiag[X] = K(X,X) for
 * all N sequences (the normalisation of Knorm). Knorm(X,Y) = K(X,Y) /
 * sqrt(K(X,X) K(Y,Y)) as in the full path.
 *   N >= 2, 1 <= NA <= N - 1; C, Nm: int64[(M+1)*NA*NB]; K: int64[NA*NB];
 *   Knorm: fp64[NA*NB]; Kdiag: int64[N]; row-major, [m][X][Y - NA].
 * Any output may be NULL (not returned; C NULL = plan scratch) and host or device.
 * Errors as gakco_kernel; shard setting ignored. */
gakco_status gakco_kernel_rect(gakco_plan* plan, const uint8_t* codes, const int64_t* offsets,
                               int64_t N, int64_t NA, int64_t* C, int64_t* Nm, int64_t* K,
                               double* Knorm, int64_t* Kdiag, void* cuda_stream);

/* ---- Mask-sharded multi-GPU step ----
 * The C(g,m) masks are independent (Supp. §S:5.3) and C_m is an
 * integer sum over masks (Algorithm 1 line 17): rank r of P calls
 * gakco_set_shard(r, P) + gakco_accumulate into its own zeroed C, then the ranks sum
 * the upper triangles (the only part gakco_accumulate writes) level by level and
 * each finalises a slice of it. The triangle is addressed packed, row by row:
 *   e(X, Y) = X*N - X*(X-1)/2 + (Y - X),  0 <= X <= Y < N,  T = N*(N+1)/2 entries. */

/* Make `stream` wait until level m's C_m of the last gakco_accumulate on this plan
 * is final (all of its updates, on every stream the plan used; a level with no
 * mask in this shard is final when the call returns). GAKCO_E_ARG if m is out of
 * range or the last accumulate did not cover it. No host synchronisation. */
gakco_status gakco_stream_wait_level(gakco_plan* plan, int m, void* cuda_stream);

/* The levels of the last gakco_accumulate in the order they became final (levels
 * without masks in this shard first). Writes min(count, cap) ints to out (may be
 * NULL) and returns count (M+1 after a full accumulate), or -1 for a NULL plan. */
int gakco_level_order(const gakco_plan* plan, int* out, int cap);

/* Entries [begin, end) of the packed upper triangle of `levels` consecutive N x N
 * row-major int64 matrices C (DEVICE) -> out[l][e - begin] (DEVICE), as int64
 * (out_bytes = 8) or as the low 32 bits (out_bytes = 4: the caller guarantees the
 * values it will sum stay below 2^31, e.g. C(g,m) n_max^2 < 2^31). Enqueued on
 * cuda_stream, no synchronisation. GAKCO_E_ARG for a range outside [0, T],
 * levels outside 1..33, out_bytes not 4 / 8 or host pointers. */
gakco_status gakco_pack_upper(gakco_plan* plan, const int64_t* C, int64_t N, int levels,
                              int64_t begin, int64_t end, void* out, int out_bytes,
                              void* cuda_stream);

/* out[l][X] = C_l(X, X) for l < levels (C and out DEVICE, int64). No sync. */
gakco_status gakco_diag(gakco_plan* plan, const int64_t* C, int64_t N, int levels, int64_t* out,
                        void* cuda_stream);

/* Epilogue of one packed slice: Cp[m * ld + e - begin] (DEVICE; int64, or u32 when
 * in_bytes = 4; ld >= end - begin elements between levels) holds the COMPLETE C_m
 * (all masks summed) of the entries [begin, end); Cdiag[m][X] (DEVICE, int64) the
 * complete diagonals C_m(X,X) of all N sequences. Writes, for the same entries,
 * Nm[m * ld + e - begin] (Eq. 9),
 * K[e - begin] (Eq. 7) and Knorm[e - begin] (K(X,Y)/sqrt(K(X,X) K(Y,Y)),
 * reading A5), each optional (NULL), DEVICE pointers. Synchronises cuda_stream;
 * GAKCO_E_INTERNAL on a negative N_m or K != C_{g-k}, GAKCO_E_SYMBOL if the last
 * accumulate flagged a code >= sigma. */
gakco_status gakco_finalize_packed(gakco_plan* plan, const void* Cp, int in_bytes, int64_t ld,
                                   int64_t N, int64_t begin, int64_t end, const int64_t* Cdiag, int64_t* Nm,
                                   int64_t* K, double* Knorm, void* cuda_stream);

/* ---- The same exchange fused into the pack, over peer memory (CUDA IPC) ----
 * Instead of pack + NCCL reduce-scatter: every rank allocates a receive buffer
 * R[P][M+1][chunk] (gakco_ipc_alloc: cudaMalloc, so the IPC handle maps the buffer
 * itself), the ranks exchange the 64-byte handles (e.g. torch.distributed
 * all_gather_object) and open each other's (gakco_ipc_open: peer-mapped device
 * pointers over NVLink / NVSwitch). gakco_pack_upper_peers then writes level m of
 * this rank's C straight into the owners' buffers; after every rank's packs are
 * complete (the caller synchronises its stream and barriers), each rank runs
 * gakco_finalize_packed_sum on its own buffer, which adds the P contributions
 * inside the epilogue. */
gakco_status gakco_ipc_alloc(size_t bytes, int device, void** dev_ptr, void* handle_out /*64 B*/);
gakco_status gakco_ipc_free(void* dev_ptr);
/* handle of the allocation containing dev_ptr (the allocation's base must be dev_ptr) */
gakco_status gakco_ipc_handle(const void* dev_ptr, void* handle_out /*64 B*/);
/* map another process's buffer on `device`; close with gakco_ipc_close */
gakco_status gakco_ipc_open(const void* handle /*64 B*/, int device, void** dev_ptr);
gakco_status gakco_ipc_close(void* dev_ptr);

/* Level `level` (of `levels`) of this rank's upper-triangular C_m (DEVICE int64 N x N)
 * into the receive buffers dst[0..P-1] (a HOST array of device pointers, peer-mapped):
 * packed entry e goes to rank d = e / chunk at
 *   dst[d][(rank * levels + level) * chunk + e - d * chunk]
 * as int64 (out_bytes 8) or u32 (4; values below 2^31). chunk * P >= N(N+1)/2.
 * Enqueued on cuda_stream. */
gakco_status gakco_pack_upper_peers(gakco_plan* plan, const int64_t* Cm, int64_t N, int level,
                                    int levels, int64_t chunk, void* const* dst, int P, int rank,
                                    int out_bytes, void* cuda_stream);

/* gakco_finalize_packed over nsrc contributions: level m of source q at
 * Cp + (q * (M+1) + m) * ld (elements); C_m = their sum (the receive buffer of the
 * fused exchange, nsrc = P). Same outputs, synchronisation and errors. */
gakco_status gakco_finalize_packed_sum(gakco_plan* plan, const void* Cp, int in_bytes, int nsrc,
                                       int64_t ld, int64_t N, int64_t begin, int64_t end,
                                       const int64_t* Cdiag, int64_t* Nm, int64_t* K,
                                       double* Knorm, void* cuda_stream);

/* Counters and (if GAKCO_OPT_TIMING) stage times of the last accumulate /
 * finalize. Synchronises the plan's last stream. */
gakco_status gakco_get_stats(gakco_plan* plan, gakco_stats* out);

/* With GAKCO_OPT_TIMING: the stage events of the last accumulate / finalize as a
 * timeline (also with the pipeline on, where the stages of different streams
 * overlap): entry i is stage[i] (0 encode, 1 sort, 2 segment, 3 light, 4 heavy,
 * 5 epilogue, 6 dense, 7 far; the order of gakco_stats' ms_* fields) from t0[i] to
 * t1[i] ms after the first event. Host arrays of cap entries; *count = the number of
 * events (entries beyond cap are not written). Synchronises the plan's last stream. */
gakco_status gakco_stage_timeline(gakco_plan* plan, int32_t* stage, float* t0, float* t1,
                                  int64_t cap, int64_t* count);

/* Number of masks c_gk = sum_{m<=M} C(g,m) (Table 1) and of this shard. */
int64_t gakco_num_masks(const gakco_plan* plan, int shard_only);

const char* gakco_last_error(const gakco_plan* plan);
const char* gakco_status_string(int status);
void gakco_destroy(gakco_plan* plan);

#ifdef __cplusplus
}
#endif
#endif /* GAKCO_H */
