// plan.cu — the C-ABI (include/gakco.h) and the host orchestration of one call.
//
// Order of work for gakco_accumulate (Algorithm 1 MISMATCHPROFILE, PAPER.md:179-199,
// re-planned for a GPU):
//   validate -> corpus to device -> g-mer index
//   for m = 0..M, for each batch of this shard's masks of level m:
//       encode (+ upfront digit histograms) -> onesweep LSD passes over key digits
//       -> triples (+ diagonal repeat term) -> multi-sequence groups
//       -> light pair updates -> closed-form diagonal term
// Everything is enqueued on the caller's stream; the only host synchronisations
// are input validation (when inputs live on the device) and reading error flags
// / stats. Masks are global-round-robin sharded (rank r takes indices = r mod P,
// P:141): partial C of several shards sum to the full C.
#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

using namespace gk;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

enum Stage { S_ENCODE = 0, S_SORT, S_SEGMENT, S_LIGHT, S_HEAVY, S_EPILOGUE, S_DENSE, S_FAR, S_NSTAGE };

// NVTX range for profilers (nsys / ncu --nvtx): host-side enqueue of one phase
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

// free device memory (cudaMemGetInfo: called only when a buffer must grow -- it was
// measured taking up to 50 ms on the box, the GPU idle meanwhile)
static size_t free_bytes() {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 0;
    return fr;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// smallest b with 2^b >= v (v >= 1), for v given as an unsigned 128-bit value
int bits_for(unsigned __int128 v) {
    int b = 0;
    while (b < 128 && ((unsigned __int128)1 << b) < v) ++b;
    return b;
}

int64_t binom64(int n, int r) {
    if (r < 0 || r > n) return 0;
    int64_t c = 1;
    for (int i = 1; i <= r; ++i) c = c * (n - r + i) / i;
    return c;
}

}  // namespace

struct gakco_plan {
    int sigma = 0, g = 0, k = 0, M = 0, device = 0;
    int rank = 0, world = 1;
    int64_t heavy_min = 0, batch_keys = 0;
    bool timing = false;
    // grouping (GAKCO_OPT_SORT): -1 auto = mask trie (6) for masks of >= 2M g-mers,
    // else the batched mask trie (7) where the one-word composite fits, else chunked
    // LSD v2 (3); 0 chunked two-kernel LSD pass, 1 onesweep LSD (decoupled look-back),
    // 2 hash partition + shared-memory hash grouping (bucket.cu), 3-5 LSD v2 variants
    int sort_mode = -1;
    int sort_ctas_per_sm = 4;  // chunked pass grid = this x SMs (2 resident: 2 full waves; measured best of 2..4)
    int trie_ctas_per_sm = 2;  // trie passes (one mask each): one full wave (Text sort 91 -> 76 ms vs 4)
    int sort32_ctas_per_sm = 8;  // u32 composites: more chunks per segment (DNA sort 1.60 -> 1.49 ms)
    int64_t light_bins = 0;    // 0 auto, < 0 off, > 0 forced block size in cells
    int gram_pair = 1;         // 1: CTA-pair Gram (gram2.cu), 0: one-SM Gram (gram_tc.cu)
    int light_flat = 8;        // light groups of <= this many sequences share warps
    int light_relabel = -1;    // -1 auto (accumulator >> L2), 0 off, 1 on
    int gram_each = 0;         // 1: a Gram flush after every batch (overlaps the next batch)
    int light_window = -1;     // window Gram of cluster-local groups: -1 auto (with relabelling), 0 off, 1 on (relabels)
    int64_t window_min = 9;    // smallest group (sequences) for the window Gram
    int level_order_desc = 0;  // process levels m = M..0 (1) or 0..M (0, measured faster on DNA)
    int gram_fp4 = -1;         // -1 auto (e2m1 Gram when exact), 0 u8 / kind::i8, 1 e2m1
    int trie_pass = 1;         // mask-trie pass kernel: 1 trie.cu (Σ <= 64), 0 generic radix
    int xl_compact = 1;        // cross-level chain: compacted parents (segrag.cu), 0 off
    int far_bytes = 0;         // far-pair record width: 0 auto (4 when cells < 2^28), 4, 8
    int relabel_gpu = 1;       // relabelling computed on the device (1) or on the host (0)
    int leaf_fuse = 1;         // fused last pass + run-length (leaf.cu) in the chain
    int light_grid = 0;        // light kernel grid in CTAs per SM (0: auto, 3 relabelled, else 8)
    int light_ctas = 4;        // relabelled light kernel register budget: CTAs per SM (3, 4, 6;
                               // Scale light 74.3 / 65.7 / 69.8 ms with far records)
    static constexpr int FAR_RING = 8, FAR_LAG = 6, FAR_EVERY = 12;
    uint32_t* far_seen = nullptr;     // pinned copies of the record count, a ring
    cudaEvent_t ev_far[FAR_RING] = {};  // (the gate reads the copy of FAR_LAG batches ago)
    // (pipelined: records double-buffered, applies on the third stream)
    cudaEvent_t ev_fsrc = nullptr, ev_fapply[2] = {nullptr, nullptr};
    int64_t far_near = -1;     // far-pair records from this label distance: -1 auto (256
                               // with a relabelled accumulator), 0 off
    int pipeline = 1;          // light / dense / Gram of batch b on an aux stream, overlapping
                               // encode / sort / segment of batch b+1 (double-buffered triples)
    cudaStream_t aux = nullptr, aux2 = nullptr;  // light + dense; Gram flushes
    cudaEvent_t ev_seg[2] = {nullptr, nullptr}, ev_light[2] = {nullptr, nullptr},
                ev_join = nullptr, ev_join2 = nullptr, ev_build = nullptr,
                ev_gram[2] = {nullptr, nullptr};
    int sm_count = 148;
    std::string err;

    // masks in global order: level by level, lexicographic removed-position sets
    std::vector<int> mask_level;
    std::vector<std::array<uint8_t, GMAX>> mask_kept;
    std::vector<int> key_bits;  // per level

    DevBuf genW0, genW1, genS0, genS1, kmdev, trieR, trieX0, trieX1, pdesc, wD, wlist, wfill, wC, winv, wtiles, trieS0, trieW, trieS, keptsh, dense2, heavy2, hcount2, tseq2, tcnt2, gstart2, counts2, perm, iota, best, parent, Dgscr, Kdscr, codes, off, gofs, gmseq, keysA, keysB, hist, status, ctr, tseq, tcnt, gstart, gend,
        counts, kept, stats, flags, kdiag, Cscr, Nmscr, Kscr, Knscr, heavy, hcount, dense, tiles, tiles4, symhist,
        lightacc, binrec, bincnt, farrec, farscr, farbins, xccnt, xbcnt, relkeys, relH, thg, lbig, win, bkH, bktot, bkbase, bkdesc, bktab, bktcnt, bkgs, bkocc;
    int64_t tiles_npad = -1;
    int tiles_pair = -1;
    int64_t tiles_na = -1;
    int64_t tiles4_npad = -1, tiles4_na = -1;
    uint64_t dense_ldd = 0;
    int ntiles = 0, ntiles4 = 0;
    uint32_t epoch = 1;
    uint32_t ctr_next = 0;
    static constexpr uint32_t CTR_SLOTS = 4096;

    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> evs;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    gakco_stats host_stats{};
    cudaStream_t last_stream = nullptr;
    // per level, events on the three streams after its last update of C_m (the
    // sharded step's reduce of level m waits on them: gakco_stream_wait_level)
    cudaEvent_t ev_level[GMAX + 1][3] = {};
    std::vector<int> level_order;  // levels of the last accumulate, in completion order
    int64_t last_masks = 0;
    int64_t launches = 0;
    bool after_accumulate = false;

    std::vector<int64_t> h_off, h_gofs;
    // host trace of the last accumulate (GAKCO_HOST_TRACE=1: printed to stderr)
    int htrace_on = -1;
    std::vector<uint8_t> h_ksh;  // host copy of keptsh (source of its async upload)
    uint32_t tp_par = 0;        // pass parity of the trie passes' block sums (thg)
    int64_t iota_n = -1;        // iota holds 0..iota_n-1 (uploaded once per N)
    void* iota_at = nullptr;
    uint32_t wtiles_nw = 0;     // wtiles holds the window-Gram tile list of wtiles_nw windows
    void* wtiles_at = nullptr;
    std::vector<std::pair<std::string, double>> htrace;
    std::vector<uint8_t> kept_h;

    gakco_status fail(gakco_status s, const std::string& msg) {
        err = msg;
        return s;
    }
    gakco_status cuda_fail(cudaError_t e, const char* where) {
        err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
        return e == cudaErrorMemoryAllocation ? GAKCO_E_NOMEM : GAKCO_E_CUDA;
    }
    cudaError_t ensure(DevBuf& b, size_t bytes, cudaStream_t s, bool zero = false) {
        if (bytes == 0) bytes = 16;
        if (bytes <= b.cap) return cudaSuccess;
        if (b.p) {
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return e;
            cudaFree(b.p);
        }
        b.p = nullptr;
        b.cap = 0;
        size_t alloc = bytes + bytes / 8;
        cudaError_t e = cudaMalloc(&b.p, alloc);
        if (e != cudaSuccess) return e;
        b.cap = alloc;
        if (zero) return cudaMemsetAsync(b.p, 0, alloc, s);
        return cudaSuccess;
    }
    cudaEvent_t ev() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
    int64_t stage_launches[S_NSTAGE] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t launches_at_begin = 0;
    int last_grouping = 0;
    void stage_begin(cudaStream_t s, cudaEvent_t* a) {
        launches_at_begin = launches;
        if (!timing) return;
        *a = ev();
        cudaEventRecord(*a, s);
    }
    void stage_end(cudaStream_t s, int stage, cudaEvent_t a) {
        stage_launches[stage] += launches - launches_at_begin;
        if (!timing) return;
        cudaEvent_t b = ev();
        cudaEventRecord(b, s);
        evs.push_back({stage, {a, b}});
    }
    // next tile-ticket counter slot (reset in bulk when exhausted)
    cudaError_t next_ctr(cudaStream_t s, uint32_t** out) {
        if (ctr_next >= CTR_SLOTS) {
            cudaError_t e = cudaMemsetAsync(ctr.p, 0, CTR_SLOTS * sizeof(uint32_t), s);
            if (e != cudaSuccess) return e;
            ctr_next = 0;
        }
        *out = (uint32_t*)ctr.p + ctr_next++;
        return cudaSuccess;
    }
};

static const char* kStatusStrings[] = {"ok", "invalid argument", "symbol code >= sigma",
                                       "value out of range", "out of device memory",
                                       "CUDA error", "internal invariant failed"};

extern "C" const char* gakco_status_string(int s) {
    return (s >= 0 && s <= 6) ? kStatusStrings[s] : "unknown status";
}

extern "C" const char* gakco_last_error(const gakco_plan* p) {
    return p ? p->err.c_str() : "null plan";
}

// Mask trie of one level (GAKCO_OPT_SORT 6): the order of a mask's per-position
// passes is free (any order of its kept positions sorts by the same key tuple up to
// a permutation of digits, so groups are the same), and masks whose first t passes
// use the same t positions share those passes. The trie is built bottom-up by greedy
// set cover: the (t-1)-subsets that complete the most uncovered t-subsets are chosen
// as parents, level by level (Text: 1060 passes for its 638 masks instead of 1479
// with ascending positions; lower bound ~830). Returns, per mask (in DFS order of the
// trie, written to `order`), its positions in pass order.
static void build_mask_trie(const std::vector<uint32_t>& sets, int kk,
                            std::vector<int>& order,
                            std::vector<std::array<uint8_t, GMAX>>& chain) {
    const int L = (int)sets.size();
    order.clear();
    chain.assign(L, std::array<uint8_t, GMAX>{});
    if (L == 0) return;
    if (kk <= 0 || L > 8192) {  // (degenerate / huge levels: ascending positions)
        for (int i = 0; i < L; ++i) {
            order.push_back(i);
            int r = 0;
            for (int x = 0; x < 32; ++x)
                if ((sets[i] >> x) & 1u) chain[i][r++] = (uint8_t)x;
        }
        std::stable_sort(order.begin(), order.end(),
                         [&](int a, int b) { return chain[a] < chain[b]; });
        return;
    }
    // nodes: sets; parent[node]; children lists built at the end
    std::vector<uint32_t> node_set(sets.begin(), sets.end());
    std::vector<int> parent(L, -1);
    std::vector<int> cur(L);
    for (int i = 0; i < L; ++i) cur[i] = i;
    for (int t = kk; t >= 2; --t) {
        // candidate parents and the current nodes they would complete
        std::vector<uint32_t> cand;
        std::vector<std::vector<int>> kids;
        {
            std::vector<std::pair<uint32_t, int>> pc;
            for (int v : cur)
                for (int x = 0; x < 32; ++x)
                    if ((node_set[v] >> x) & 1u) pc.push_back({node_set[v] & ~(1u << x), v});
            std::sort(pc.begin(), pc.end());
            for (size_t i = 0; i < pc.size();) {
                size_t j = i;
                cand.push_back(pc[i].first);
                kids.emplace_back();
                while (j < pc.size() && pc[j].first == pc[i].first) kids.back().push_back(pc[j++].second);
                i = j;
            }
        }
        std::vector<char> covered(node_set.size(), 0);
        std::vector<int> cnt(cand.size());
        for (size_t c = 0; c < cand.size(); ++c) cnt[c] = (int)kids[c].size();
        // per current node, the candidates containing it (for count updates)
        std::vector<std::vector<int>> of(node_set.size());
        for (size_t c = 0; c < cand.size(); ++c)
            for (int v : kids[c]) of[v].push_back((int)c);
        std::vector<int> next;
        size_t left = cur.size();
        while (left > 0) {
            int best = -1;
            for (size_t c = 0; c < cand.size(); ++c)
                if (cnt[c] > 0 && (best < 0 || cnt[c] > cnt[best])) best = (int)c;
            const int pn = (int)node_set.size();
            node_set.push_back(cand[best]);
            parent.push_back(-1);
            covered.push_back(0);
            of.emplace_back();
            next.push_back(pn);
            for (int v : kids[best]) {
                if (covered[v]) continue;
                covered[v] = 1;
                parent[v] = pn;
                --left;
                for (int c : of[v]) --cnt[c];
            }
        }
        cur = next;
    }
    // (1-sets hang under the root, -1) — children lists, then DFS from the root
    const int NN = (int)node_set.size();
    std::vector<std::vector<int>> ch(NN + 1);
    for (int v = 0; v < NN; ++v) ch[parent[v] < 0 ? NN : parent[v]].push_back(v);
    std::vector<std::pair<int, int>> st{{NN, 0}};  // (node, depth)
    std::array<uint8_t, GMAX> path{};
    while (!st.empty()) {
        auto [v, d] = st.back();
        st.pop_back();
        if (v != NN) {
            const uint32_t par = parent[v] < 0 ? 0u : node_set[parent[v]];
            path[d - 1] = (uint8_t)__builtin_ctz(node_set[v] & ~par);
            if (v < L) {  // a mask
                order.push_back(v);
                for (int r = 0; r < d; ++r) chain[v][r] = path[r];
            }
        }
        for (auto it = ch[v].rbegin(); it != ch[v].rend(); ++it) st.push_back({*it, d + 1});
    }
}

// Batched mask trie (GAKCO_OPT_SORT 7): like build_mask_trie, but every pass sorts
// by up to P symbols (P * bits <= 8: DNA 4 positions per pass) and the trie is run
// depth by depth, all of a depth's nodes in one launch. Bottom-up greedy cover:
// a node's parent is its set minus P positions; the first pass takes the rest.
// Output: nodes (set, parent index or -1, depth), leaves[i] = node of mask i.
struct TrieNode {
    uint32_t set;
    int parent;
    int depth;
};
static void build_step_trie(const std::vector<uint32_t>& sets, int kk, int P,
                            std::vector<TrieNode>& nodes, std::vector<int>& leaf_node) {
    nodes.clear();
    leaf_node.assign(sets.size(), -1);
    const int D = (kk + P - 1) / P;
    std::vector<int> cur;
    for (size_t i = 0; i < sets.size(); ++i) {
        nodes.push_back({sets[i], -1, D});
        leaf_node[i] = (int)i;
        cur.push_back((int)i);
    }
    for (int d = D; d >= 2; --d) {
        // candidate parents: each node's set minus P of its positions
        std::vector<std::pair<uint32_t, int>> pc;
        for (int v : cur) {
            const uint32_t sv = nodes[v].set;
            int pos[32], np = 0;
            for (int x = 0; x < 32; ++x)
                if ((sv >> x) & 1u) pos[np++] = x;
            // all P-subsets of the node's positions (np <= 32, P <= 8)
            std::vector<int> idx(P);
            for (int i = 0; i < P; ++i) idx[i] = i;
            while (true) {
                uint32_t rm = 0;
                for (int i = 0; i < P; ++i) rm |= 1u << pos[idx[i]];
                pc.push_back({sv & ~rm, v});
                int i = P - 1;
                while (i >= 0 && idx[i] == np - P + i) --i;
                if (i < 0) break;
                ++idx[i];
                for (int j = i + 1; j < P; ++j) idx[j] = idx[j - 1] + 1;
            }
        }
        std::sort(pc.begin(), pc.end());
        std::vector<uint32_t> cand;
        std::vector<std::vector<int>> kids;
        for (size_t i = 0; i < pc.size();) {
            size_t j = i;
            cand.push_back(pc[i].first);
            kids.emplace_back();
            while (j < pc.size() && pc[j].first == pc[i].first) kids.back().push_back(pc[j++].second);
            i = j;
        }
        std::vector<char> covered(nodes.size(), 0);
        std::vector<int> cnt(cand.size());
        std::vector<std::vector<int>> of(nodes.size());
        for (size_t c = 0; c < cand.size(); ++c) {
            cnt[c] = (int)kids[c].size();
            for (int v : kids[c]) of[v].push_back((int)c);
        }
        std::vector<int> next;
        size_t left = cur.size();
        while (left > 0) {
            int best = -1;
            for (size_t c = 0; c < cand.size(); ++c)
                if (cnt[c] > 0 && (best < 0 || cnt[c] > cnt[best])) best = (int)c;
            const int pn = (int)nodes.size();
            nodes.push_back({cand[best], -1, d - 1});
            next.push_back(pn);
            for (int v : kids[best]) {
                if (covered[v]) continue;
                covered[v] = 1;
                nodes[v].parent = pn;
                --left;
                for (int c : of[v]) --cnt[c];
            }
        }
        cur = next;
    }
}

extern "C" gakco_status gakco_create(int sigma, int g, int k, int M, int device, gakco_plan** out) {
    if (!out) return GAKCO_E_ARG;
    *out = nullptr;
    if (sigma < 1 || sigma > 255 || g < 1 || g > GMAX || k < 1 || k > g || M < 0 || M > g)
        return GAKCO_E_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return device < 0 ? GAKCO_E_ARG : GAKCO_E_CUDA;
    }
    int64_t total = 0;
    for (int m = 0; m <= M; ++m) total += binom64(g, m);
    if (total > (1 << 24)) return GAKCO_E_RANGE;
    gakco_plan* p = new gakco_plan();
    p->sigma = sigma;
    p->g = g;
    p->k = k;
    p->M = M;
    p->device = device;
    {
        DeviceGuard dg(device);
        cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, device);
    }
    // masks: m removed positions, lexicographic over the removed set (reading A9)
    for (int m = 0; m <= M; ++m) {
        std::vector<int> rem(m);
        for (int i = 0; i < m; ++i) rem[i] = i;
        while (true) {
            std::array<uint8_t, GMAX> kept{};
            int r = 0, q = 0;
            for (int pos = 0; pos < g; ++pos) {
                if (q < m && rem[q] == pos) {
                    ++q;
                    continue;
                }
                kept[r++] = (uint8_t)pos;
            }
            p->mask_level.push_back(m);
            p->mask_kept.push_back(kept);
            int i = m - 1;
            while (i >= 0 && rem[i] == g - m + i) --i;
            if (i < 0) break;
            ++rem[i];
            for (int j = i + 1; j < m; ++j) rem[j] = rem[j - 1] + 1;
        }
        // key bits: sigma^(g-m) distinct keys
        unsigned __int128 v = 1;
        bool over = false;
        for (int i = 0; i < g - m; ++i) {
            v *= (unsigned)sigma;
            if (v > ((unsigned __int128)1 << 64)) over = true;
        }
        p->key_bits.push_back(over ? 65 : bits_for(v));
    }
    *out = p;
    return GAKCO_OK;
}

extern "C" void gakco_destroy(gakco_plan* p) {
    if (!p) return;
    DeviceGuard dg(p->device);
    DevBuf* bufs[] = {&p->keptsh, &p->dense2, &p->heavy2, &p->hcount2, &p->tseq2, &p->tcnt2, &p->gstart2, &p->counts2, &p->perm, &p->iota, &p->best, &p->parent, &p->Dgscr, &p->Kdscr, &p->codes, &p->off,   &p->gofs,  &p->gmseq,  &p->keysA, &p->keysB,
                      &p->hist,  &p->status, &p->ctr,  &p->tseq,   &p->tcnt,  &p->gstart,
                      &p->gend,  &p->counts, &p->kept, &p->stats,  &p->flags, &p->kdiag,
                      &p->Cscr,  &p->Nmscr, &p->Kscr,  &p->Knscr, &p->heavy, &p->hcount,
                      &p->dense, &p->tiles, &p->tiles4, &p->symhist, &p->trieS0, &p->trieW, &p->trieS, &p->genW0, &p->genW1, &p->genS0, &p->genS1, &p->kmdev, &p->trieR, &p->trieX0, &p->trieX1, &p->pdesc, &p->wD, &p->wlist, &p->wfill, &p->wC, &p->winv, &p->wtiles, &p->lightacc, &p->binrec, &p->bincnt, &p->farrec, &p->farscr, &p->farbins, &p->xccnt, &p->xbcnt, &p->relkeys, &p->relH, &p->thg, &p->lbig,
                      &p->win,   &p->bkH,   &p->bktot, &p->bkbase, &p->bkdesc, &p->bktab,
                      &p->bktcnt, &p->bkgs, &p->bkocc};
    for (DevBuf* b : bufs)
        if (b->p) cudaFree(b->p);
    for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
    for (auto& lv : p->ev_level)
        for (cudaEvent_t e : lv)
            if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {p->ev_seg[0], p->ev_seg[1], p->ev_light[0], p->ev_light[1], p->ev_join,
                          p->ev_join2, p->ev_build, p->ev_gram[0], p->ev_gram[1]})
        if (e) cudaEventDestroy(e);
    if (p->far_seen) cudaFreeHost(p->far_seen);
    for (cudaEvent_t e : {p->ev_fsrc, p->ev_fapply[0], p->ev_fapply[1]})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : p->ev_far)
        if (e) cudaEventDestroy(e);
    if (p->aux) cudaStreamDestroy(p->aux);
    if (p->aux2) cudaStreamDestroy(p->aux2);
    delete p;
}

extern "C" gakco_status gakco_set_shard(gakco_plan* p, int rank, int world) {
    if (!p || world < 1 || rank < 0 || rank >= world) return GAKCO_E_ARG;
    p->rank = rank;
    p->world = world;
    return GAKCO_OK;
}

extern "C" gakco_status gakco_set_option(gakco_plan* p, int option, int64_t value) {
    if (!p) return GAKCO_E_ARG;
    switch (option) {
        case GAKCO_OPT_HEAVY_MIN_SEQS:
            if (value < 0) return p->fail(GAKCO_E_ARG, "heavy threshold must be >= 0");
            p->heavy_min = value;
            return GAKCO_OK;
        case GAKCO_OPT_BATCH_KEYS:
            if (value < 0) return p->fail(GAKCO_E_ARG, "batch keys must be >= 0");
            p->batch_keys = value;
            return GAKCO_OK;
        case GAKCO_OPT_SORT:
            if (value < -1 || value > 7) return p->fail(GAKCO_E_ARG, "sort must be -1..7");
            p->sort_mode = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_LIGHT_BINS:
            p->light_bins = value;
            return GAKCO_OK;
        case GAKCO_OPT_SORT_CTAS_PER_SM:
            if (value < 1 || value > 16) return p->fail(GAKCO_E_ARG, "1..16");
            p->sort_ctas_per_sm = (int)value;
            p->trie_ctas_per_sm = (int)value;
            p->sort32_ctas_per_sm = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_GRAM_PAIR:
            if (value < 0 || value > 1) return p->fail(GAKCO_E_ARG, "gram pair must be 0 or 1");
            p->gram_pair = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_LIGHT_FLAT:
            if (value < 1 || value > 32) return p->fail(GAKCO_E_ARG, "light flat must be 1..32");
            p->light_flat = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_LIGHT_RELABEL:
            if (value < -1 || value > 1) return p->fail(GAKCO_E_ARG, "relabel must be -1..1");
            p->light_relabel = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_LIGHT_WINDOW:
            if (value < -1 || value > 1) return p->fail(GAKCO_E_ARG, "light window must be -1..1");
            p->light_window = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_WINDOW_MIN:
            if (value < 2) return p->fail(GAKCO_E_ARG, "window min must be >= 2");
            p->window_min = value;
            return GAKCO_OK;
        case GAKCO_OPT_GRAM_EACH:
            if (value < 0 || value > 1) return p->fail(GAKCO_E_ARG, "gram each must be 0 or 1");
            p->gram_each = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_GRAM_FP4:
            if (value < -1 || value > 1) return p->fail(GAKCO_E_ARG, "gram fp4 must be -1..1");
            p->gram_fp4 = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_PIPELINE:
            if (value < 0 || value > 1) return p->fail(GAKCO_E_ARG, "pipeline must be 0 or 1");
            p->pipeline = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_LEVEL_ORDER:
            if (value < 0 || value > 1) return p->fail(GAKCO_E_ARG, "level order must be 0 or 1");
            p->level_order_desc = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_TIMING:
            p->timing = value != 0;
            return GAKCO_OK;
        case GAKCO_OPT_RELABEL_HOST:
            if (value < 0 || value > 1) return p->fail(GAKCO_E_ARG, "relabel host must be 0 or 1");
            p->relabel_gpu = value ? 0 : 1;
            return GAKCO_OK;
        case GAKCO_OPT_LEAF_FUSE:
            if (value < 0 || value > 1) return p->fail(GAKCO_E_ARG, "leaf fuse must be 0 or 1");
            p->leaf_fuse = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_FAR_BYTES:
            if (value != 0 && value != 4 && value != 8) return p->fail(GAKCO_E_ARG, "far bytes: 0, 4 or 8");
            p->far_bytes = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_LIGHT_GRID:
            if (value < 0 || value > 64) return p->fail(GAKCO_E_ARG, "light grid: 0..64 CTAs per SM");
            p->light_grid = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_LIGHT_CTAS:
            if (value != 3 && value != 4 && value != 6) return p->fail(GAKCO_E_ARG, "light ctas: 3, 4 or 6");
            p->light_ctas = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_XL_COMPACT:
            if (value < 0 || value > 1) return p->fail(GAKCO_E_ARG, "xl compact must be 0 or 1");
            p->xl_compact = (int)value;
            return GAKCO_OK;
        case GAKCO_OPT_FAR_NEAR:
            if (value < -1 || value > ((int64_t)1 << 31)) return p->fail(GAKCO_E_ARG, "far near must be -1..2^31");
            p->far_near = value;
            return GAKCO_OK;
        case GAKCO_OPT_TRIE_PASS:
            if (value < 0 || value > 1) return p->fail(GAKCO_E_ARG, "trie pass must be 0 or 1");
            p->trie_pass = (int)value;
            return GAKCO_OK;
        default:
            return p->fail(GAKCO_E_ARG, "unknown option");
    }
}

extern "C" int64_t gakco_num_masks(const gakco_plan* p, int shard_only) {
    if (!p) return -1;
    int64_t n = (int64_t)p->mask_level.size();
    if (!shard_only) return n;
    return n / p->world + ((n % p->world) > p->rank ? 1 : 0);
}

// ----------------------------------------------------------------------------
// only_level >= 0: process only the masks of that level, accumulated into the
// single N x N matrix C (used by the K-only path, K = C_{g-k}).
static gakco_status accumulate_impl(gakco_plan* p, const uint8_t* codes, const int64_t* offsets,
                                    int64_t N, int64_t* C, cudaStream_t s, int rank, int world,
                                    int only_level = -1, int64_t NA = 0,
                                    int64_t* Dg = nullptr) {
    const auto t_entry = std::chrono::steady_clock::now();
    if (p->htrace_on < 0) {
        const char* e = std::getenv("GAKCO_HOST_TRACE");
        p->htrace_on = e && e[0] == '1';
    }
    p->htrace.clear();
    auto HT = [&](const char* what) {
        if (p->htrace_on)
            p->htrace.emplace_back(what, std::chrono::duration<double, std::milli>(
                                             std::chrono::steady_clock::now() - t_entry).count());
    };
#define CK(x)                                          \
    do {                                               \
        cudaError_t e_ = (x);                          \
        if (e_ != cudaSuccess) return p->cuda_fail(e_, #x); \
    } while (0)
#define LK(x)        \
    do {             \
        ++p->launches; \
        CK(x);       \
    } while (0)
    p->launches = 0;
    for (int64_t& v : p->stage_launches) v = 0;
    if (!codes && N > 0) return p->fail(GAKCO_E_ARG, "codes is NULL");
    if (!offsets || !C) return p->fail(GAKCO_E_ARG, "offsets or C is NULL");
    if (N < 1 || N >= ((int64_t)1 << 31)) return p->fail(GAKCO_E_ARG, "N must be in [1, 2^31)");
    if (!is_device_ptr(C)) return p->fail(GAKCO_E_ARG, "C must be a device pointer");
    p->last_stream = s;
    p->evs.clear();
    p->ev_used = 0;
    const int g = p->g, M = p->M;

    // offsets -> host, validate
    p->h_off.resize(N + 1);
    if (is_device_ptr(offsets)) {
        CK(cudaMemcpyAsync(p->h_off.data(), offsets, (N + 1) * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    } else {
        std::memcpy(p->h_off.data(), offsets, (N + 1) * sizeof(int64_t));
    }
    if (p->h_off[0] != 0) return p->fail(GAKCO_E_ARG, "offsets[0] != 0");
    for (int64_t i = 0; i < N; ++i)
        if (p->h_off[i + 1] < p->h_off[i]) return p->fail(GAKCO_E_ARG, "offsets decrease");
    const int64_t L = p->h_off[N];
    HT("offsets");

    // g-mer counts n_X = max(0, l_X - g + 1) (reading A7/A8) and prefix sums
    p->h_gofs.assign(N + 1, 0);
    int64_t nmax = 0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t nx = std::max<int64_t>(0, p->h_off[i + 1] - p->h_off[i] - g + 1);
        nmax = std::max(nmax, nx);
        p->h_gofs[i + 1] = p->h_gofs[i] + nx;
    }
    const uint64_t n = (uint64_t)p->h_gofs[N];
    if (n >= (1ull << 30)) return p->fail(GAKCO_E_RANGE, "more than 2^30 g-mers");
    // int64 bound of every entry: C_m(X,Y) <= C(g,m) n_X n_Y, K <= C(g,k) n_X n_Y
    {
        unsigned __int128 nn = (unsigned __int128)nmax * nmax;
        for (int m = 0; m <= M; ++m)
            if (nn * (unsigned __int128)binom64(g, m) > (unsigned __int128)INT64_MAX)
                return p->fail(GAKCO_E_RANGE, "C_m may overflow int64");
        if (nn * (unsigned __int128)binom64(g, p->k) > (unsigned __int128)INT64_MAX)
            return p->fail(GAKCO_E_RANGE, "K may overflow int64");
    }
    if ((uint64_t)nmax * (uint64_t)nmax > (uint64_t)UINT32_MAX)
        return p->fail(GAKCO_E_RANGE, "a sequence has more than 65535 g-mers (u32 pair sums)");
    const int sb = (N <= 1) ? 0 : 64 - __builtin_clzll((unsigned long long)(N - 1));
    for (int m = 0; m <= M; ++m)
        if (p->key_bits[m] + sb > 64)
            return p->fail(GAKCO_E_RANGE, "masked key + sequence id exceed 64 bits");

    // grouping: hash partition (bucket.cu) when the g-mer window packs into 64 bits,
    // a mask has <= 16M g-mers (<= 16384 buckets of ~1024 keys) and every level's
    // key + sequence id fits 64 bits; otherwise the LSD radix sort (radix.cu)
    int bits = 1;
    while ((1 << bits) < p->sigma) ++bits;
    const int sbh = std::max(sb, 1);
    // (auto = LSD: the hash path measured slower on every config so far)
    bool hash_mode = p->sort_mode == 2 && n > 0 && g * bits <= 64 &&
                     n <= (16384ull << 10);
    std::vector<int> level_runs(M + 1, 0);
    for (int m = 0; m <= M && hash_mode; ++m) {
        if ((g - m) * bits + sbh <= 64) level_runs[m] = 1;
        else if (p->key_bits[m] + sbh > 64) hash_mode = false;
    }
    p->last_grouping = hash_mode ? 2 : (p->sort_mode == 1 ? 1 : 0);

    // corpus to device (+ symbol check). The symbol histogram feeds the per-level
    // Gram operand format (auto e2m1 below); counted only when that choice is open.
    // (also for the fused leaves of the mask trie: their gate is the expected largest
    // group of the pass before, from the most frequent symbol)
    const bool trie_pre = (p->sort_mode == 6 || (p->sort_mode == -1 && n >= (2ull << 20))) &&
                          p->leaf_fuse && n > 0;
    const bool need_hist = trie_pre || p->gram_fp4 == -1 && (p->gram_pair || NA > 0) && nmax > 0 &&
                           (uint64_t)nmax * (uint64_t)nmax < (1ull << 24);
    std::vector<unsigned long long> hist(256, 0);
    CK(p->ensure(p->codes, (size_t)L + 16, s));
    CK(p->ensure(p->flags, 64, s, /*zero=*/true));
    if (L > 0) {
        if (is_device_ptr(codes)) {
            // device codes are checked on the device without a host sync; a bad code
            // sets flags[1] and is reported (GAKCO_E_SYMBOL) by gakco_finalize. The
            // path stays memory-safe meanwhile (keys only index 256-bin digits).
            CK(cudaMemcpyAsync(p->codes.p, codes, L, cudaMemcpyDeviceToDevice, s));
            LK(launch_check_codes((const uint8_t*)p->codes.p, L, p->sigma,
                                  (int*)p->flags.p + 1, s));
            if (need_hist) {
                CK(p->ensure(p->symhist, 256 * 8, s));
                CK(cudaMemsetAsync(p->symhist.p, 0, 256 * 8, s));
                LK(launch_symbol_hist((const uint8_t*)p->codes.p, L,
                                      (unsigned long long*)p->symhist.p, p->sm_count, s));
                CK(cudaMemcpyAsync(hist.data(), p->symhist.p, 256 * 8, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
            }
        } else {
            for (int64_t i = 0; i < L; ++i) {
                if (codes[i] >= p->sigma) return p->fail(GAKCO_E_SYMBOL, "a code is >= sigma");
                hist[codes[i]] += 1;
            }
            CK(cudaMemcpyAsync(p->codes.p, codes, L, cudaMemcpyHostToDevice, s));
        }
    }
    double fmax = 1.0;  // the most frequent symbol's share (1 when not counted)
    if (need_hist && L > 0) {
        unsigned long long hm = 0;
        for (int c = 0; c < 256; ++c) hm = std::max(hm, hist[c]);
        fmax = (double)hm / (double)L;
    }
    auto lf_big_expect = [&](int npos) { return (double)n * std::pow(fmax, (double)npos); };
    CK(p->ensure(p->off, (N + 1) * sizeof(int64_t), s));
    CK(p->ensure(p->gofs, (N + 1) * sizeof(int64_t), s));
    CK(cudaMemcpyAsync(p->off.p, p->h_off.data(), (N + 1) * sizeof(int64_t),
                       cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(p->gofs.p, p->h_gofs.data(), (N + 1) * sizeof(int64_t),
                       cudaMemcpyHostToDevice, s));
    CK(p->ensure(p->gmseq, n * sizeof(uint32_t), s));
    LK(launch_gmer_index((const int64_t*)p->gofs.p, N, (uint32_t*)p->gmseq.p, s));
    HT("corpus");

    // this shard's masks, in processing order: levels ascending (default) or, with
    // GAKCO_OPT_LEVEL_ORDER, descending so the top level's long tensor-bound Gram
    // flushes overlap the lower levels' light and sort work (any order gives the
    // same integer sums); ascending whenever the light accumulator is relabelled
    // (the clustering reads the first, cheapest level)
    const bool relabel_pre =
        NA == 0 && p->light_bins <= 0 && N >= 2 &&
        (p->light_relabel == 1 ||
         (p->light_relabel == -1 && (uint64_t)N * (uint64_t)(N - 1) / 2 * 4 > (96ull << 20)));
    std::vector<int> mine;
    for (size_t i = 0; i < p->mask_level.size(); ++i)
        if ((int)(i % world) == rank && (only_level < 0 || p->mask_level[i] == only_level))
            mine.push_back((int)i);
    if (!relabel_pre && p->level_order_desc)
        std::stable_sort(mine.begin(), mine.end(), [&](int a, int b) {
            return p->mask_level[a] > p->mask_level[b];
        });
    // mask trie (GAKCO_OPT_SORT 6): within a level, masks in lexicographic order of
    // their kept positions, so consecutive masks share the passes of their common
    // leading positions
    // (auto: the trie for masks of >= 2M g-mers, where its single-mask passes fill the
    // machine -- Text 180 -> 151 ms, Scale 246 -> 238 ms; the batched LSD passes win
    // below: DNA, Protein)
    const bool trie = (p->sort_mode == 6 || (p->sort_mode == -1 && n >= (2ull << 20))) &&
                      !hash_mode && n > 0 && g * bits <= 64;
    // batched trie (GAKCO_OPT_SORT 7): composites (window << sb | seq) of one word
    // (auto below the mask trie's 2M g-mers: DNA 9.03 -> 8.76 ms, Protein 7.5 -> 6.6 ms)
    const bool trie_b = !trie && (p->sort_mode == 7 || p->sort_mode == -1) && !hash_mode &&
                        n > 0 && g * bits + sb <= 64;
    const bool tb64 = g * bits + sb > 32;
    if (trie_b) p->last_grouping = 4;
    std::vector<std::array<uint8_t, GMAX>> trie_chain;  // per position in mine
    // cross-level reuse (mask trie): with levels processed as k rises (m falls), a
    // level-m mask S is one pass (by a position x) over the unmasked sorted arrays of
    // the level-(m+1) mask S \ {x}, kept from the previous level in a generation
    // buffer; only the first level of the chain is a trie from the windows.
    // (Relabelling needs level 0 first: then 0, M, M-1, ..., 1.)
    std::vector<int> xl_parent, xl_x, xl_slot, xl_run;  // per position in mine
    std::vector<char> xl_link;  // per run: its masks are one pass over the previous run's
    bool xl = false;
    size_t xl_maxrun = 0;
    // (the batched trie too, where a pass sorts by one symbol -- Protein: a child mask
    // is then one pass by one symbol, as the trie's own passes; DNA's 4-symbol passes
    // gain nothing and its ascending level order measured faster)
    const bool xlb = trie_b && std::min(4, 8 / bits) <= 1 && n >= (uint64_t)SEG_ITEMS;
    if ((trie || xlb) && n >= (uint64_t)SEG_ITEMS) {
        std::vector<int> order;
        for (int v : mine) order.push_back(v);
        auto key = [&](int v) {
            const int lm = p->mask_level[v];
            return relabel_pre ? (lm == 0 ? -1000 : -lm) : -lm;
        };
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key(a) < key(b); });
        mine = order;
        xl = true;
    }
    if (trie || xlb) {
        size_t a0 = 0;
        trie_chain.resize(mine.size());
        xl_parent.assign(mine.size(), -1);
        xl_x.assign(mine.size(), -1);
        xl_slot.assign(mine.size(), 0);
        xl_run.assign(mine.size(), 0);
        int run = 0, prev_level = -1;
        std::vector<uint32_t> prev_sets;  // previous run's masks (sets), by slot
        while (a0 < mine.size()) {
            size_t a1 = a0;
            while (a1 < mine.size() && p->mask_level[mine[a1]] == p->mask_level[mine[a0]]) ++a1;
            std::vector<uint32_t> sets;
            for (size_t i = a0; i < a1; ++i) {
                uint32_t b = 0;
                for (int r = 0; r < g - p->mask_level[mine[i]]; ++r) b |= 1u << p->mask_kept[mine[i]][r];
                sets.push_back(b);
            }
            const int lm = p->mask_level[mine[a0]];
            std::vector<int> lv(mine.begin() + a0, mine.begin() + a1);
            // parents in the previous run (level m + 1, one position fewer)?
            std::vector<int> par(sets.size(), -1), px(sets.size(), -1);
            bool all = xl && prev_level == lm + 1;
            if (all) {
                std::vector<std::pair<uint32_t, int>> ps;
                for (size_t q = 0; q < prev_sets.size(); ++q) ps.push_back({prev_sets[q], (int)q});
                std::sort(ps.begin(), ps.end());
                for (size_t i = 0; i < sets.size() && all; ++i) {
                    for (int x = 0; x < 32 && par[i] < 0; ++x) {
                        if (!((sets[i] >> x) & 1u)) continue;
                        const uint32_t pset = sets[i] & ~(1u << x);
                        auto it = std::lower_bound(ps.begin(), ps.end(), std::make_pair(pset, -1));
                        if (it != ps.end() && it->first == pset) {
                            par[i] = it->second;
                            px[i] = x;
                        }
                    }
                    if (par[i] < 0) all = false;
                }
            }
            std::vector<uint32_t> cur_sets(sets.size());
            if (all) {  // one pass per mask, in parent order (locality)
                std::vector<int> ord(sets.size());
                for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
                std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return par[a] < par[b]; });
                for (size_t i = 0; i < ord.size(); ++i) {
                    mine[a0 + i] = lv[ord[i]];
                    xl_parent[a0 + i] = par[ord[i]];
                    xl_x[a0 + i] = px[ord[i]];
                    cur_sets[i] = sets[ord[i]];
                }
            } else if (trie) {
                std::vector<int> ord;
                std::vector<std::array<uint8_t, GMAX>> ch;
                build_mask_trie(sets, g - lm, ord, ch);
                for (size_t i = 0; i < ord.size(); ++i) {
                    mine[a0 + i] = lv[ord[i]];
                    trie_chain[a0 + i] = ch[ord[i]];
                    cur_sets[i] = sets[ord[i]];
                }
            } else {  // (batched trie: built per batch)
                cur_sets = sets;
            }
            for (size_t i = a0; i < a1; ++i) {
                xl_slot[i] = (int)(i - a0);
                xl_run[i] = run;
            }
            xl_maxrun = std::max(xl_maxrun, a1 - a0);
            xl_link.push_back(all ? 1 : 0);
            prev_sets = cur_sets;
            prev_level = lm;
            ++run;
            a0 = a1;
        }
        p->last_grouping = trie ? 3 : 4;
    }
    // (pageable host staging: cudaMemcpyAsync returns once the source is copied,
    // so the member buffers can be reused without a stream sync)
    std::vector<uint8_t>& kept_h = p->kept_h;
    kept_h.assign(mine.size() * GMAX + GMAX, 0);
    for (size_t i = 0; i < mine.size(); ++i)
        std::memcpy(&kept_h[i * GMAX], p->mask_kept[mine[i]].data(), GMAX);
    CK(p->ensure(p->kept, kept_h.size(), s));
    CK(cudaMemcpyAsync(p->kept.p, kept_h.data(), kept_h.size(), cudaMemcpyHostToDevice, s));

    // heavy / light threshold: a group of s sequences costs ~s^2/2 scattered
    // updates on the light path and ~N_pad^2/2 u8 MACs on the Gram; with the
    // measured rates (~1.1e11 updates/s, ~1.5e15 MAC/s) they break even near
    // s = 0.0085 N_pad.
    // rectangular mode (NA > 0): rows [0, NA) x columns [NA, N) only; C is
    // [levels][NA][N - NA], the diagonals C_m(X,X) go to Dg [levels][N]
    const bool rect = NA > 0;
    const bool gpair = p->gram_pair || rect;
    const int64_t n_pad = gpair ? (N + 511) / 512 * 512 : (N + 255) / 256 * 256;
    // e2m1 Gram (kind::mxf4, gram2.cu): counts <= 4 exact in e2m1, f32 sums exact
    // below 2^24, so it applies while one mask's n_max^2 stays below 2^24; groups
    // with a count > 4 stay on the light path. Chosen per level: in auto mode only
    // where even the most frequent masked key is rare within one sequence,
    // n_max * p_max^(g-m) <= 1/8 with p_max the most frequent symbol's share (i.i.d.
    // reading: counts > 4 then have Poisson tail < 3e-7 per sequence); levels with
    // few effective keys (large m on DNA, Zipf text) use u8, whose counts reach 255.
    const bool fp4_any_ok = gpair && p->gram_fp4 != 0 && nmax > 0 &&
                            (uint64_t)nmax * (uint64_t)nmax < (1ull << 24);
    double pmax = 1.0;
    if (L > 0) {
        unsigned long long hm = 0;
        for (int c = 0; c < 256; ++c) hm = std::max(hm, hist[c]);
        if (hm > 0) pmax = (double)hm / (double)L;
    }
    std::vector<char> fp4_lv(M + 1, 0);
    bool fp4_any = false;
    for (int m = 0; m <= M; ++m) {
        if (!fp4_any_ok) break;
        const double rep_ = (double)nmax * std::pow(pmax, (double)(g - m));
        fp4_lv[m] = p->gram_fp4 == 1 || rep_ <= 0.125;
    }
    for (size_t i = 0; i < mine.size(); ++i) fp4_any |= fp4_lv[p->mask_level[mine[i]]] != 0;
    auto exact_lim_of = [&](int m) -> uint64_t {
        return fp4_lv[m] ? (1ull << 24) - 1 : (uint64_t)INT32_MAX;
    };
    auto slab_cols_of = [&](int m) -> uint64_t { return fp4_lv[m] ? 256 : 128; };
    auto heavy_min_of = [&](int m) -> int64_t {
        if (p->heavy_min != 0) return p->heavy_min;
        return std::max<int64_t>(16, (int64_t)((fp4_lv[m] ? 0.008 : 0.012) * (double)n_pad + 0.999));
    };
    int64_t heavy_min_lo = INT64_MAX;
    for (size_t i = 0; i < mine.size(); ++i)
        heavy_min_lo = std::min(heavy_min_lo, heavy_min_of(p->mask_level[mine[i]]));
    if (mine.empty()) heavy_min_lo = p->heavy_min != 0 ? p->heavy_min : 16;
    const uint64_t exact_lim = fp4_any ? (1ull << 24) - 1 : (uint64_t)INT32_MAX;
    const bool heavy_on = heavy_min_lo < (int64_t)1 << 40 && N >= 2;

    // batch size (keys cap; with the Gram on, s32 exactness: masks * n_max^2 < 2^31)
    // default: up to 64M keys (512 MB per key buffer): large launches measured
    // faster than L2-sized (4M-key) batches for every stage;
    // 128M with the single-mask trie (Scale 32M 135.2 ms, 64M 129.8, 96M 126.9, 128M
    // 126.4-126.8, 160M 131.6, 256M 137.3; Text 64M 79.9, 128M 77.3; the batched trie
    // of DNA / Protein: neutral)
    uint64_t bk = p->batch_keys > 0 ? (uint64_t)p->batch_keys
                                    : (hash_mode ? (12ull << 20) : trie ? (128ull << 20) : (64ull << 20));
    if (bk > (1ull << 30) - 1) bk = (1ull << 30) - 1;
    uint64_t bmax_masks = std::max<uint64_t>(1, n ? bk / n : mine.size());
    if (heavy_on && nmax > 0) {
        uint64_t lim = exact_lim / ((uint64_t)nmax * (uint64_t)nmax);
        bmax_masks = std::max<uint64_t>(1, std::min(bmax_masks, lim));
    }
    // a single mask whose n_max^2 exceeds 2^31 would need the light path only
    const bool gram_ok =
        heavy_on && nmax > 0 && (uint64_t)nmax * (uint64_t)nmax <= (uint64_t)INT32_MAX;
    const uint64_t cap_keys = std::max<uint64_t>(1, std::min<uint64_t>(bmax_masks, mine.size()) * n);
    // (+ slack: the bulk copies of radix_scatter2 read whole 16-byte words)
    CK(p->ensure(p->keysA, cap_keys * 8 + 64, s));
    CK(p->ensure(p->keysB, cap_keys * 8 + 64, s));
    CK(p->ensure(p->tseq, cap_keys * 4, s));
    CK(p->ensure(p->tcnt, cap_keys * 4, s));
    CK(p->ensure(p->gstart, (cap_keys / 2 + 2) * sizeof(uint2), s));  // group ranges
    CK(p->ensure(p->counts, 16, s));
    // two-stream pipeline: light / dense / Gram on `s2` consume batch b's triples while
    // `s` encodes, sorts and segments batch b+1 into the other triple buffer
    const bool pipe = p->pipeline != 0;
    if (pipe) {
        CK(p->ensure(p->tseq2, cap_keys * 4, s));
        CK(p->ensure(p->tcnt2, cap_keys * 4, s));
        CK(p->ensure(p->gstart2, (cap_keys / 2 + 2) * sizeof(uint2), s));
        CK(p->ensure(p->counts2, 16, s));
        if (!p->aux) {
            CK(cudaStreamCreateWithFlags(&p->aux, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&p->aux2, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                CK(cudaEventCreateWithFlags(&p->ev_seg[i], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&p->ev_light[i], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&p->ev_gram[i], cudaEventDisableTiming));
            }
            CK(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&p->ev_join2, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&p->ev_build, cudaEventDisableTiming));
        }
    }
    cudaStream_t s2 = pipe ? p->aux : s;
    // Gram flushes on s3 (tensor pipe), concurrent with the next columns' light
    // updates and dense build on s2 (L2 atomics / stores) into the other D slot
    cudaStream_t s3 = pipe ? p->aux2 : s;
    CK(p->ensure(p->hist, std::max<uint64_t>(std::min<uint64_t>(bmax_masks, mine.size() + 1) *
                                                 MAXPASS * RADIX * 4,
                                             (uint64_t)(std::max(p->sort_ctas_per_sm, p->sort32_ctas_per_sm) *
                                                            p->sm_count + 64 +
                                                        2 * bmax_masks) *
                                                 RADIX * 4),
                 s));
    {
        uint64_t tps = (n + SORT_TILE - 1) / SORT_TILE;
        uint64_t st_sort = std::min<uint64_t>(bmax_masks, mine.size() + 1) * RADIX * tps;
        uint64_t st_seg = 2 * (cap_keys / SEG_TILE + 2);  // two look-back arrays
        CK(p->ensure(p->status, std::max(st_sort, st_seg) * 8, s, /*zero=*/true));
    }
    if (p->ctr.cap == 0) {
        CK(p->ensure(p->ctr, p->CTR_SLOTS * sizeof(uint32_t), s));
        p->ctr_next = p->CTR_SLOTS;  // forces a reset on first use
    }
    CK(p->ensure(p->stats, ST_COUNT * 8, s));
    CK(cudaMemsetAsync(p->stats.p, 0, ST_COUNT * 8, s));
    unsigned long long* stats = (unsigned long long*)p->stats.p;

    // hash-partition buffers: packed windows, mask descriptors, big-bucket scratch
    HT("maskplan");
    std::vector<MaskDesc> desc_h;
    if (hash_mode) {
        CK(p->ensure(p->win, n * 8, s));
        CK(p->ensure(p->bktab, cap_keys * 2 * 8, s));
        CK(p->ensure(p->bktcnt, cap_keys * 2 * 4, s));
        CK(p->ensure(p->bkgs, cap_keys * 2 * 4, s));
        CK(p->ensure(p->bkocc, cap_keys * 4, s));
        desc_h.resize(mine.size() + 1);
        std::memset(desc_h.data(), 0, desc_h.size() * sizeof(MaskDesc));
        for (size_t i = 0; i < mine.size(); ++i) {
            const int m = p->mask_level[mine[i]];
            const uint8_t* kept = p->mask_kept[mine[i]].data();
            MaskDesc& d = desc_h[i];
            d.nkept = (uint8_t)(g - m);
            for (int r = 0; r < g - m; ++r) d.kept_sh[r] = (uint8_t)(bits * (g - 1 - kept[r]));
            // maximal runs of consecutive kept positions -> bit fields of w
            int r = 0, nrun = 0;
            while (r < g - m) {
                int e = r;
                while (e + 1 < g - m && kept[e + 1] == kept[e] + 1) ++e;
                d.run_src[nrun] = (uint8_t)(bits * (g - 1 - kept[e]));
                d.run_len[nrun] = (uint8_t)(bits * (e - r + 1));
                d.run_dst[nrun] = (uint8_t)(bits * (g - m - 1 - e));
                ++nrun;
                r = e + 1;
            }
            d.nrun = (uint8_t)nrun;
        }
        CK(p->ensure(p->bkdesc, desc_h.size() * sizeof(MaskDesc), s));
        CK(cudaMemcpyAsync(p->bkdesc.p, desc_h.data(), desc_h.size() * sizeof(MaskDesc),
                           cudaMemcpyHostToDevice, s));
    }

    // per level: groups of >= heavy_min_of(m) sequences go to the Gram
    auto light_limit_of = [&](int m) -> int64_t { return gram_ok ? heavy_min_of(m) : INT64_MAX; };
    uint64_t rcap8 = 0, rcap4 = 0;  // D columns of a u8 / e2m1 level (same bytes)
    if (gram_ok) {
        CK(p->ensure(p->hcount, 16, s, /*zero=*/true));
        if (pipe) CK(p->ensure(p->hcount2, 16, s, /*zero=*/true));
        // dense count matrix D: n_pad rows x rcap u8 columns (<= 4 GB, and no more
        // columns than heavy groups can exist), accumulated over batches of a level
        // (every batch rounds its columns up to whole 128-column slabs)
        const uint64_t most =
            (uint64_t)mine.size() * n / (uint64_t)heavy_min_lo + 256 * (mine.size() + 1);
        rcap8 = std::min<uint64_t>((4096ull << 20) / (uint64_t)n_pad, most);
        rcap8 = std::max<uint64_t>(128, (rcap8 + 127) / 128 * 128);
        rcap4 = fp4_any ? std::min<uint64_t>(2 * rcap8, std::max<uint64_t>(256, (most + 255) / 256 * 256)) : 0;
        rcap4 = rcap4 / 256 * 256;
        const uint64_t dbytes = std::max<uint64_t>((uint64_t)n_pad * rcap8, (uint64_t)n_pad * rcap4 / 2);
        const uint64_t hcols = std::max(rcap8, rcap4);
        CK(p->ensure(p->dense, dbytes, s));
        CK(p->ensure(p->heavy, hcols * sizeof(uint2), s));
        if (pipe) {
            CK(p->ensure(p->dense2, dbytes, s));
            CK(p->ensure(p->heavy2, hcols * sizeof(uint2), s));
        }
        if (fp4_any && (p->tiles4_npad != n_pad || (rect && p->tiles4_na != NA))) {
            std::vector<int2> t = rect ? gram4_tiles_rect(NA, N - NA) : gram4_tiles(n_pad);
            CK(p->ensure(p->tiles4, t.size() * sizeof(int2), s));
            CK(cudaMemcpyAsync(p->tiles4.p, t.data(), t.size() * sizeof(int2),
                               cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));
            p->ntiles4 = (int)t.size();
            p->tiles4_npad = n_pad;
            p->tiles4_na = rect ? NA : -1;
        }
        const int tkey = rect ? 2 : (gpair ? 1 : 0);
        if (p->tiles_npad != n_pad || p->tiles_pair != tkey || (rect && p->tiles_na != NA)) {
            std::vector<int2> t = rect ? gram2_tiles_rect(NA, N - NA)
                                       : (gpair ? gram2_tiles(n_pad) : gram_tiles(n_pad));
            CK(p->ensure(p->tiles, t.size() * sizeof(int2), s));
            CK(cudaMemcpyAsync(p->tiles.p, t.data(), t.size() * sizeof(int2),
                               cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));
            p->ntiles = (int)t.size();
            p->tiles_npad = n_pad;
            p->tiles_pair = tkey;
            p->tiles_na = NA;
        }
    }
    CorpusView cv{(const uint8_t*)p->codes.p, (const int64_t*)p->off.p, (const int64_t*)p->gofs.p,
                  (const uint32_t*)p->gmseq.p, N, n};
    SegmentOut so1{(uint32_t*)p->tseq.p, (uint32_t*)p->tcnt.p, (uint2*)p->gstart.p,
                   (uint32_t*)p->counts.p};
    SegmentOut so2 = pipe ? SegmentOut{(uint32_t*)p->tseq2.p, (uint32_t*)p->tcnt2.p,
                                       (uint2*)p->gstart2.p, (uint32_t*)p->counts2.p}
                          : so1;
    int64_t batch_no = 0;
    int64_t passkeys = 0, keys32 = 0, passkeys32 = 0;
    // encode from packed g-mer windows when g * bits <= 64 (LSD path, not onesweep,
    // whose encoder also counts the digit histograms)
    const bool use_win = !hash_mode && n > 0 && g * bits <= 64 && p->sort_mode != 1;
    // trie buffers: root sequence ids (u16 when N <= 65536), one level of the pass
    // stack per kept position (windows + ids); the batch's leaves go to keysA / keysB
    const bool seq16 = N <= 65536;
    const size_t ssz = seq16 ? 2 : 4;
    std::array<int, GMAX> stack_pos{};
    int stack_depth = 0;
    if (trie) {
        // block sums of the trie passes' chunk histograms (trie.cu), two parities,
        // zero when allocated (each pass zeroes the other parity's for the next)
        CK(p->ensure(p->thg, (size_t)2 * TP_HG_MAX_BLOCKS * 64 * 4, s, /*zero=*/true));
        CK(p->ensure(p->trieS0, n * ssz + 64, s));
        if (seq16)
            LK(launch_seq16((const uint32_t*)p->gmseq.p, (uint16_t*)p->trieS0.p, n, p->sm_count, s));
        else
            CK(cudaMemcpyAsync(p->trieS0.p, p->gmseq.p, n * 4, cudaMemcpyDeviceToDevice, s));
        CK(p->ensure(p->trieW, (size_t)g * n * 8 + 64, s));
        CK(p->ensure(p->trieS, (size_t)g * n * ssz + 64, s));
        if (xl) {  // generation buffers: a level's unmasked sorted arrays, two levels
            const size_t need = 2 * xl_maxrun * n * (8 + ssz) + 256;
            const bool have = p->genW0.cap >= xl_maxrun * n * 8 + 64 &&
                              p->genW1.cap >= xl_maxrun * n * 8 + 64 &&
                              p->genS0.cap >= xl_maxrun * n * ssz + 64 &&
                              p->genS1.cap >= xl_maxrun * n * ssz + 64;
            // (free memory is queried only when the buffers must grow: cudaMemGetInfo
            // measured at up to 50 ms on the box, with the GPU idle meanwhile)
            if (have || free_bytes() > need + (4ull << 30)) {
                CK(p->ensure(p->genW0, xl_maxrun * n * 8 + 64, s));
                CK(p->ensure(p->genW1, xl_maxrun * n * 8 + 64, s));
                CK(p->ensure(p->genS0, xl_maxrun * n * ssz + 64, s));
                CK(p->ensure(p->genS1, xl_maxrun * n * ssz + 64, s));
                CK(p->ensure(p->kmdev, (bmax_masks + 2) * 8, s));
            } else {
                xl = false;  // (not enough memory: per-level tries, leaves masked)
                for (auto& v : xl_parent) v = -1;
            }
        }
    }
    if (xlb && xl) {  // batched trie, cross-level: one-word composites per generation
        const size_t esb = tb64 ? 8 : 4;
        const bool have = p->genW0.cap >= xl_maxrun * n * esb + 64 &&
                          p->genW1.cap >= xl_maxrun * n * esb + 64;
        if (have || free_bytes() > 2 * xl_maxrun * n * esb + (4ull << 30)) {
            CK(p->ensure(p->genW0, xl_maxrun * n * esb + 64, s));
            CK(p->ensure(p->genW1, xl_maxrun * n * esb + 64, s));
            CK(p->ensure(p->kmdev, (bmax_masks + 2) * 8, s));
        } else {
            xl = false;
            for (auto& v : xl_parent) v = -1;
        }
    }
    // cross-level chain with compaction (segrag.cu): leaves in the batch buffers
    // (keysA windows, keysB ids), each run's compacted arrays in the generation
    // buffers with their counts in xccnt [2][maxrun]; the next run's passes read them
    const bool xlc = trie && xl && p->xl_compact && p->trie_pass == 1 &&
                     trie_pass64_ok((1u << bits) - 1u);
    if (xlc) {
        CK(p->ensure(p->xccnt, 2 * xl_maxrun * 4 + 16, s));
        CK(p->ensure(p->xbcnt, (bmax_masks + 2) * 4, s));
    }
    auto run_has_kids = [&](int r) {
        return r + 1 < (int)xl_link.size() && xl_link[r + 1] != 0;
    };
    if (use_win) {
        CK(p->ensure(p->win, n * 8, s));
        // (no stream sync: a cudaMemcpyAsync from pageable memory has staged the bytes
        // when it returns; the source is kept in the plan all the same)
        std::vector<uint8_t>& ksh = p->h_ksh;
        ksh.assign(mine.size() * GMAX + GMAX, 0);
        for (size_t i = 0; i < mine.size(); ++i) {
            const int mm = p->mask_level[mine[i]];
            for (int r = 0; r < g - mm; ++r)
                ksh[i * GMAX + r] = (uint8_t)(bits * (g - 1 - p->mask_kept[mine[i]][r]));
        }
        CK(p->ensure(p->keptsh, ksh.size(), s));
        CK(cudaMemcpyAsync(p->keptsh.p, ksh.data(), ksh.size(), cudaMemcpyHostToDevice, s));
    }
    if (hash_mode || use_win) {
        cudaEvent_t a0 = nullptr;
        p->stage_begin(s, &a0);
        LK(launch_windows(cv, g, bits, (uint64_t*)p->win.p, p->sm_count, s));
        p->stage_end(s, S_ENCODE, a0);
    }
    if (trie_b) {  // the batched trie's root: every g-mer's composite (window << sb | seq)
        CK(p->ensure(p->trieR, n * (tb64 ? 8 : 4) + 64, s));
        LK(launch_trie_root((const uint64_t*)p->win.p, (const uint32_t*)p->gmseq.p, n, sb, tb64,
                            p->trieR.p, p->sm_count, s));
    }
    const size_t nn = rect ? (size_t)NA * (size_t)(N - NA) : (size_t)N * N;
    auto level_ptr = [&](int m) -> int64_t* {
        return only_level >= 0 ? C : C + (size_t)m * nn;
    };
    // C_m(X,X) lives at diag_ptr(m)[X * dstride]
    const int64_t dstride = rect ? 1 : N + 1;
    auto diag_ptr = [&](int m) -> int64_t* {
        if (!rect) return level_ptr(m);
        return only_level >= 0 ? Dg : Dg + (size_t)m * N;
    };

    // Heavy groups of consecutive batches of one level accumulate as columns of D;
    // the Gram runs ("flush") at a level change, when D could overflow (a bound,
    // so no host read-back is needed), or when the s32 sums could reach 2^31.
    uint64_t dense_bound = 0, dense_masks = 0;
    int dense_m = -1;
    // D slot being filled (the Gram of the other slot may still be running on s3)
    int dslot = 0;
    bool slot_used[2] = {false, false};
    auto dense_p = [&]() { return (uint8_t*)(dslot ? p->dense2.p : p->dense.p); };
    auto heavy_p = [&]() { return (uint2*)(dslot ? p->heavy2.p : p->heavy.p); };
    auto hcount_p = [&]() { return (uint32_t*)(dslot ? p->hcount2.p : p->hcount.p); };
    auto mask_lim_of = [&](int m) -> uint64_t {
        return gram_ok ? std::max<uint64_t>(1, exact_lim_of(m) / ((uint64_t)nmax * nmax)) : 0;
    };
    auto rcap_of = [&](int m) -> uint64_t { return fp4_lv[m] ? rcap4 : rcap8; };
    int64_t fp4_used = 0;  // levels whose Gram ran on e2m1
    auto flush = [&]() -> gakco_status {
        if (dense_m < 0 || dense_bound == 0) return GAKCO_OK;
        Nvtx nv("gram flush");
        if (pipe) {  // every build of this slot (s2) precedes its Gram (s3)
            CK(cudaEventRecord(p->ev_build, s2));
            CK(cudaStreamWaitEvent(s3, p->ev_build, 0));
        }
        cudaEvent_t ah = nullptr;
        p->stage_begin(s3, &ah);
        p->launches += 1;  // + fill_reset
        const uint64_t rcap = rcap_of(dense_m);
        if (fp4_lv[dense_m]) {
            fp4_used |= 1ll << dense_m;
            LK(launch_gram4_flush(dense_p(), n_pad, rcap, hcount_p(), level_ptr(dense_m), N,
                                  (const int2*)p->tiles4.p, p->ntiles4, p->sm_count, stats, s3, NA));
        } else if (gpair)
            LK(launch_gram2_flush(dense_p(), n_pad, rcap, hcount_p(), level_ptr(dense_m), N,
                                  (const int2*)p->tiles.p, p->ntiles, p->sm_count, stats, s3, NA));
        else
            LK(launch_gram_flush(dense_p(), n_pad, rcap, hcount_p(), level_ptr(dense_m), N,
                                 (const int2*)p->tiles.p, p->ntiles, p->sm_count, stats, s3));
        p->stage_end(s3, S_HEAVY, ah);
        if (pipe) {  // switch D slots; the next user of the other slot waits for its Gram
            CK(cudaEventRecord(p->ev_gram[dslot], s3));
            slot_used[dslot] = true;
            dslot ^= 1;
            if (slot_used[dslot]) CK(cudaStreamWaitEvent(s2, p->ev_gram[dslot], 0));
        }
        dense_bound = 0;
        dense_masks = 0;
        return GAKCO_OK;
    };
    // Light updates accumulate in a u32 packed strictly-upper triangle, added into
    // C_m at a level change or before masks * n_max^2 could reach 2^32.
    const uint64_t ntri =
        rect ? (uint64_t)NA * (uint64_t)(N - NA) : (uint64_t)N * (uint64_t)(N - 1) / 2;
    CK(p->ensure(p->lightacc, ntri * 4 + 16, s, /*zero=*/true));
    // light-update binning when the accumulator is far larger than L2 (Scale:
    // 800 MB): records per 64 MB block, applied block by block (light.cu)
    LightBins bins{nullptr, nullptr, 0, 0, 0};
    {
        uint64_t bc = 0;
        // auto mode leaves binning OFF: measured 2.3x slower than direct atomics on
        // Scale (match.any + record traffic cost more than the DRAM RMW saved)
        if (p->light_bins > 0 && !rect) bc = (uint64_t)p->light_bins;  // forced (tests, ablation)
        if (bc > 0 && ntri > 0) {
            bc = std::min<uint64_t>(bc, (1ull << 28) - 1);  // offset field: 28 bits
            const int nb = (int)((ntri + bc - 1) / bc);
            const uint64_t total_rec = std::max<uint64_t>(1ull << 20, std::min<uint64_t>(512ull << 20, ntri * 4));
            // (forced mode is a test knob: tiny buckets also exercise the overflow path)
            const uint64_t cap =
                p->light_bins > 0 ? 64 : std::max<uint64_t>(1024, total_rec / nb);
            CK(p->ensure(p->binrec, cap * nb * 4, s));
            CK(p->ensure(p->bincnt, nb * 4 + 16, s, /*zero=*/true));
            CK(cudaMemsetAsync(p->bincnt.p, 0, nb * 4, s));
            bins = LightBins{(uint32_t*)p->binrec.p, (uint32_t*)p->bincnt.p, cap, bc, nb};
        }
    }
    // Sequence relabelling of the light accumulator (locality): when the
    // packed triangle is far larger than L2, the sequences are reordered after the
    // first level by clusters of best partners (argmax_Y C_m(X,Y)), so pairs that
    // share many keys (families) update nearby cells; the flush maps back.
    const bool relabel = !rect && bins.nb == 0 && N >= 2 &&
                         (p->light_relabel == 1 || p->light_window == 1 ||
                          (p->light_relabel == -1 && ntri * 4 > (96ull << 20)));
    // window Gram: once relabelled, groups whose labels lie in one
    // window of 256 go to the tensor cores as u8 columns of that window's block
    const bool win_on = relabel && p->light_window != 0 && n > 0;
    WinArgs wa{nullptr, nullptr, 0, 0, 0};
    int nwtiles = 0;
    if (win_on) {
        const uint32_t nw = (uint32_t)((N + WIN_STEP - 1) / WIN_STEP);
        // columns per window: a few batches' claims, <= 64K, D <= 2 GB
        uint64_t cap = std::min<uint64_t>(65536, (2048ull << 20) / ((uint64_t)nw * WIN_ROWS));
        cap = std::max<uint64_t>(128, cap / 128 * 128);
        CK(p->ensure(p->wD, cap * nw * WIN_ROWS, s));
        CK(p->ensure(p->wlist, cap * nw * sizeof(uint2), s));
        CK(p->ensure(p->wfill, 2 * nw * 4, s, /*zero=*/true));
        CK(cudaMemsetAsync(p->wfill.p, 0, 2 * nw * 4, s));
        CK(p->ensure(p->wC, (size_t)nw * WIN_ROWS * WIN_ROWS * 8, s, /*zero=*/true));
        CK(cudaMemsetAsync(p->wC.p, 0, (size_t)nw * WIN_ROWS * WIN_ROWS * 8, s));
        CK(p->ensure(p->winv, N * 4, s));
        CK(p->ensure(p->wtiles, (size_t)2 * nw * sizeof(int2), s));
        if (p->wtiles_nw != nw || p->wtiles_at != p->wtiles.p) {  // (once per shape)
            std::vector<int2> wt;
            for (uint32_t w = 0; w < nw; ++w) {
                wt.push_back(make_int2((int)(2 * w), (int)w));
                wt.push_back(make_int2((int)(2 * w + 1), (int)w));
            }
            CK(cudaMemcpyAsync(p->wtiles.p, wt.data(), wt.size() * sizeof(int2),
                               cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));  // wt is a local buffer
            p->wtiles_nw = nw;
            p->wtiles_at = p->wtiles.p;
        }
        nwtiles = (int)(2 * nw);
        wa = WinArgs{(uint32_t*)p->wfill.p, (uint2*)p->wlist.p, (uint32_t)cap, nw,
                     (uint32_t)std::max<int64_t>(p->window_min, (int64_t)p->light_flat + 1)};
    }
    bool perm_active = false;
    // far-pair records: with a relabelled accumulator far beyond L2, a
    // light pair whose labels are >= near apart is recorded and added block by block
    FarRec far{nullptr, nullptr, 0, 0};
    // pipelined: two record buffers; a due apply runs on s3 over the full one while the
    // light kernels on s2 append to the other (atomic adds into the accumulator commute)
    FarRec farb[2] = {far, far};
    int fcur = 0;
    bool fapplied[2] = {false, false};
    const bool far2 = pipe;
    int far_bshift = 0;
    uint32_t far_thresh = 0;
    int64_t far_batch = 0, far_last_apply = -4, far_seen_at = -4;  // (the gate's batch clock)
    if (relabel && ntri < (1ull << 40) &&
        (p->far_near > 0 || (p->far_near == -1 && ntri * 4 > (96ull << 20)))) {
        // records are applied once they fill half the buffer (every cell of a block hit
        // several times per apply) and before each accumulator flush; up to 2^31
        // 4-byte records (8 GB per buffer + the same for the bucketed copy; 2^30 8-byte
        // ones) while 16 GB stay free. 4-byte records when every cell index fits 28 bits
        // (Scale: 2e8 cells). (2^30 4-byte records overflowed at Scale: with the host
        // ahead of the GPU the gate applies blindly every FAR_EVERY batches, and 12 of
        // level 5's 128M-key batches can record more: one light launch per step fell
        // back to DRAM REDs.)
        const bool k32 = p->far_bytes == 4 || (p->far_bytes == 0 && ntri < (1ull << 28));
        if (k32 && ntri >= (1ull << 28)) return p->fail(GAKCO_E_ARG, "4-byte far records need < 2^28 cells");
        const size_t have = std::min(p->farrec.cap / (far2 ? 2 : 1), p->farscr.cap) / (k32 ? 4 : 8);
        // (buffers already at the record maximum: no free-memory query)
        const uint64_t cmax = k32 ? (1ull << 31) : (1ull << 30);
        uint64_t cap = cmax;
        if (have < cap) {
            const size_t fr = free_bytes();
            cap = std::min<uint64_t>(cmax, std::max<uint64_t>(
                std::max<uint64_t>(1ull << 24, have),
                fr > (16ull << 30) ? (fr - (16ull << 30)) / 16 : 0));
        }
        cap = cap / FAR_CHUNK * FAR_CHUNK;
        far_thresh = (uint32_t)(cap / 2);
        CK(p->ensure(p->farrec, cap * (k32 ? 4 : 8) * (far2 ? 2 : 1), s));
        CK(p->ensure(p->farscr, cap * (k32 ? 4 : 8), s));
        // farbins: [0..255] the fill counter (at 192), then 2 x SMs x 64 chunk histograms,
        // bucket offsets [65] and a sink word
        CK(p->ensure(p->farbins, (256 + (size_t)p->sm_count * 2 * 64 + 72) * 4, s, /*zero=*/true));
        if (!p->far_seen) {
            CK(cudaMallocHost(&p->far_seen, gakco_plan::FAR_RING * sizeof(uint32_t)));
            for (auto& e : p->ev_far) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            for (cudaEvent_t* e : {&p->ev_fsrc, &p->ev_fapply[0], &p->ev_fapply[1]})
                CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        for (int q = 0; q < gakco_plan::FAR_RING; ++q) p->far_seen[q] = 0;
        CK(cudaMemsetAsync(p->farbins.p, 0, 256 * 4, s));
        int lb = 0;
        while (((uint64_t)1 << lb) < ntri) ++lb;
        far_bshift = std::max(16, lb - 6);  // <= 64 accumulator blocks
        far = FarRec{(uint64_t*)p->farrec.p, (uint32_t*)p->farbins.p + 192, cap,
                     (uint32_t)(p->far_near > 0 ? p->far_near : 256), k32};
        farb[0] = far;
        farb[1] = far;
        // (the second buffer's fill counter at 196, its overflow count at 197)
        farb[1].rec = (uint64_t*)((uint8_t*)p->farrec.p + cap * (k32 ? 4 : 8));
        farb[1].fill = (uint32_t*)p->farbins.p + 196;
    }
    if (relabel) {
        CK(p->ensure(p->perm, N * 4, s));
        CK(p->ensure(p->iota, N * 4, s));
        CK(p->ensure(p->best, N * 8, s));
        CK(p->ensure(p->parent, N * 4, s));
        if (p->iota_n != N || p->iota_at != p->iota.p) {  // (once per N: no per-call sync)
            std::vector<uint32_t> io(N);
            for (int64_t i = 0; i < N; ++i) io[i] = (uint32_t)i;
            CK(cudaMemcpyAsync(p->iota.p, io.data(), N * 4, cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));  // io is a local buffer
            p->iota_n = N;
            p->iota_at = p->iota.p;
        }
    }
    auto make_perm = [&](int m_done) -> gakco_status {
        Nvtx nv("relabel");
        HT("relabel");
        if (N < ((int64_t)1 << 31) && p->relabel_gpu) {
            // on the device, no host round trip: the clusters, then the labels = the
            // sequences stably sorted by cluster root (3 passes of 6 bits of the root,
            // keys root << 32 | sequence; the sequence order is kept within a cluster)
            // (on the light stream, after level m_done's light and window flushes; it
            // waits for the Gram stream's flushes. The next level's sort / segment on s
            // does not use the labels, so it runs meanwhile)
            if (pipe) {
                CK(cudaEventRecord(p->ev_join2, s3));
                CK(cudaStreamWaitEvent(s2, p->ev_join2, 0));
            }
            cudaEvent_t ar = nullptr;
            p->stage_begin(s2, &ar);
            p->launches += 4 + 2 * 3 + 2;
            CK(launch_cluster_roots(level_ptr(m_done), N, (unsigned long long*)p->best.p,
                                    (uint32_t*)p->parent.p, (const uint32_t*)p->iota.p,
                                    p->sm_count, s2));
            CK(p->ensure(p->relkeys, (size_t)N * 16 + 64, s2));
            CK(p->ensure(p->relH, (size_t)p->sm_count * 2 * 64 * 4 + 64, s2));
            uint64_t* ka = (uint64_t*)p->relkeys.p;
            uint64_t* kb = ka + N;
            CK(launch_relabel_keys((const uint32_t*)p->parent.p, N, ka, s2));
            int rb = 0;
            while (((int64_t)1 << rb) < N) ++rb;
            for (int sh = 0; sh < rb; sh += 6) {
                CK(launch_tp_records(ka, kb, false, (uint64_t)N, nullptr, 32 + sh,
                                     (uint32_t*)p->relH.p, p->sm_count * 2, s2));
                std::swap(ka, kb);
            }
            CK(launch_relabel_perm(ka, N, (uint32_t*)p->perm.p, win_on ? (uint32_t*)p->winv.p : nullptr,
                                   s2));
            p->stage_end(s2, S_LIGHT, ar);
            perm_active = true;
            return GAKCO_OK;
        }
        CK(cudaStreamSynchronize(s2));  // C of level m_done complete (light + Gram flushes)
        CK(cudaStreamSynchronize(s3));
        cudaEvent_t ar = nullptr;
        p->stage_begin(s, &ar);
        p->launches += 3;
        CK(launch_cluster_roots(level_ptr(m_done), N, (unsigned long long*)p->best.p,
                                (uint32_t*)p->parent.p, (const uint32_t*)p->iota.p,
                                p->sm_count, s));
        p->stage_end(s, S_LIGHT, ar);
        std::vector<uint32_t> root(N), order(N), pm(N);
        CK(cudaMemcpyAsync(root.data(), p->parent.p, N * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int64_t i = 0; i < N; ++i) order[i] = (uint32_t)i;
        std::stable_sort(order.begin(), order.end(),
                         [&](uint32_t a, uint32_t b) { return root[a] < root[b]; });
        for (int64_t i = 0; i < N; ++i) pm[order[i]] = (uint32_t)i;
        CK(cudaMemcpyAsync(p->perm.p, pm.data(), N * 4, cudaMemcpyHostToDevice, s));
        if (win_on)  // label -> sequence, for the window flush
            CK(cudaMemcpyAsync(p->winv.p, order.data(), N * 4, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));  // pm / order are local buffers
        perm_active = true;
        return GAKCO_OK;
    };
    uint64_t light_masks = 0;
    int light_m = -1;
    const uint64_t light_lim =
        nmax > 0 ? std::max<uint64_t>(1, (uint64_t)UINT32_MAX / ((uint64_t)nmax * nmax)) : 1;
    // window Gram of the pending window columns (every few batches, and before the
    // window block is added into C_m); s32 sums exact: a batch spans <= (2^31-1)/n_max^2
    // masks and a Gram <= WIN_BATCHES batches (the accumulation before is int64)
    int win_pending = 0;
    uint64_t win_masks = 0;
    constexpr int WIN_BATCHES = 4;
    const uint64_t win_lim =
        nmax > 0 ? std::max<uint64_t>(1, (uint64_t)INT32_MAX / ((uint64_t)nmax * nmax)) : 1;
    auto wgram = [&]() -> gakco_status {
        if (win_pending == 0) return GAKCO_OK;
        cudaEvent_t aw = nullptr;
        p->stage_begin(s2, &aw);
        p->launches += 1;  // + reset
        LK(launch_window_gram((uint8_t*)p->wD.p, wa, (int64_t*)p->wC.p, (const int2*)p->wtiles.p,
                              nwtiles, p->sm_count, stats, s2));
        p->stage_end(s2, S_HEAVY, aw);
        win_pending = 0;
        win_masks = 0;
        return GAKCO_OK;
    };
    auto lflush = [&]() -> gakco_status {
        if (light_m < 0 || light_masks == 0) return GAKCO_OK;
        Nvtx nv("light flush");
        HT("lflush");
        cudaEvent_t al = nullptr;
        if (perm_active && far.near) {  // every pending far record first
            if (far2) {  // (the applies in flight on s3 done)
                CK(cudaEventRecord(p->ev_join2, s3));
                CK(cudaStreamWaitEvent(s2, p->ev_join2, 0));
            }
            p->stage_begin(s2, &al);
            p->launches += 4 + 2 * 16;
            LK(launch_far_apply(farb[fcur], p->farscr.p, (uint32_t*)p->farbins.p + 256,
                                far_bshift, (uint32_t*)p->lightacc.p, ntri, p->sm_count, s2));
            p->stage_end(s2, S_FAR, al);
            far_last_apply = far_batch;  // (copies older than this are stale)
        }
        p->stage_begin(s2, &al);
        if (rect)
            LK(launch_light_flush_rect((uint32_t*)p->lightacc.p, ntri, level_ptr(light_m),
                                       p->sm_count, s2));
        else if (perm_active) {
            LK(launch_light_flush_perm((uint32_t*)p->lightacc.p, N, level_ptr(light_m),
                                       (const uint32_t*)p->perm.p, p->sm_count, s2));
            if (win_on) {
                gakco_status ws = wgram();
                if (ws != GAKCO_OK) return ws;
                LK(launch_window_flush((int64_t*)p->wC.p, wa.nw, (const uint32_t*)p->winv.p, N,
                                       level_ptr(light_m), p->sm_count, s2));
            }
        }
        else
            LK(launch_light_flush((uint32_t*)p->lightacc.p, N, level_ptr(light_m), p->sm_count,
                                  s2));
        p->stage_end(s2, S_LIGHT, al);
        light_masks = 0;
        return GAKCO_OK;
    };

    // level completion events: every stream that writes C_m records one after the
    // level's last update (levels without masks in this shard: complete now)
    p->level_order.clear();
    auto mark_level = [&](int lv) -> gakco_status {
        cudaStream_t st3[3] = {s, s2, s3};
        for (int q = 0; q < 3; ++q) {
            if (!p->ev_level[lv][q]) CK(cudaEventCreateWithFlags(&p->ev_level[lv][q], cudaEventDisableTiming));
            CK(cudaEventRecord(p->ev_level[lv][q], st3[q]));
        }
        p->level_order.push_back(lv);
        return GAKCO_OK;
    };
    if (only_level < 0) {
        std::vector<char> has(M + 1, 0);
        for (int v : mine) has[p->mask_level[v]] = 1;
        for (int lv = 0; lv <= M; ++lv)
            if (!has[lv]) {
                gakco_status ms = mark_level(lv);
                if (ms != GAKCO_OK) return ms;
            }
    }
    int prev_level = -1;
    if (pipe) {  // everything enqueued on s so far (uploads, zeroing) precedes s2/s3 work
        CK(cudaEventRecord(p->ev_join, s));
        CK(cudaStreamWaitEvent(s2, p->ev_join, 0));
        CK(cudaStreamWaitEvent(s3, p->ev_join, 0));
    }
    HT("setup");
    size_t pos = 0;
    while (pos < mine.size()) {
        HT("batch");
        const int m = p->mask_level[mine[pos]];
        size_t end = pos;
        while (end < mine.size() && p->mask_level[mine[end]] == m && end - pos < bmax_masks) ++end;
        const int nmask = (int)(end - pos);
        char nvname[64];
        std::snprintf(nvname, sizeof nvname, "batch m=%d masks=%d", m, nmask);
        Nvtx nvb(nvname);
        const int kb = p->key_bits[m];
        const int npass = (kb + RADIX_BITS - 1) / RADIX_BITS;
        int64_t* Cm = level_ptr(m);
        int64_t* Dm = diag_ptr(m);  // C_m(X,X) at Dm[X * dstride]
        cudaEvent_t a = nullptr;
        if (gram_ok && n > 0) {
            const uint64_t bnd = (uint64_t)nmask * n / (uint64_t)heavy_min_of(m) + slab_cols_of(m);
            if (dense_m != m || dense_bound + bnd > rcap_of(m) ||
                dense_masks + nmask > mask_lim_of(m) || (p->gram_each && dense_bound > 0)) {
                gakco_status fs = flush();
                if (fs != GAKCO_OK) return fs;
            }
            dense_m = m;
            dense_bound += bnd;
            dense_masks += nmask;
        }
        if (n > 0) {
            // (a first level of many batches -- a K-only call -- is relabelled after its
            // first batch: the clusters come from that batch's share of C_m)
            const bool early = relabel && !perm_active && light_m == m && batch_no == 1;
            if (light_m != m || light_masks + nmask > light_lim || early) {
                const int done = light_m;
                gakco_status fs = lflush();
                if (fs != GAKCO_OK) return fs;
                if (relabel && !perm_active && done >= 0 && (done != m || early)) {
                    // C of `done` holds its level (or, early, its first batch): its Gram
                    // flush was issued at this level change by the heavy block above
                    // (early: pending Gram columns are labelling-independent), its light
                    // flush just now
                    fs = make_perm(done);
                    if (fs != GAKCO_OK) return fs;
                }
            }
            light_m = m;
            light_masks += nmask;
        }

        if (prev_level >= 0 && prev_level != m && only_level < 0) {  // prev_level's C_m is final
            gakco_status ms = mark_level(prev_level);
            if (ms != GAKCO_OK) return ms;
        }
        prev_level = m;

        // triple buffer of this batch; its previous user (batch_no - 2) must be done
        const int bi = (int)(batch_no & 1);
        const SegmentOut so = bi ? so2 : so1;
        auto wait_buf = [&]() -> gakco_status {
            if (pipe && batch_no >= 2) CK(cudaStreamWaitEvent(s, p->ev_light[bi], 0));
            return GAKCO_OK;
        };
        if (n > 0 && hash_mode) {
            // hash partition: count -> (column / bucket scans + scatter) -> group
            const bool k64 = (level_runs[m] ? (g - m) * bits : kb) + sbh > 32;
            BkArgs ba{};
            ba.win = (const uint64_t*)p->win.p;
            ba.gm_seq = (const uint32_t*)p->gmseq.p;
            ba.n = n;
            ba.desc = (const MaskDesc*)p->bkdesc.p + pos;
            ba.nmask = nmask;
            ba.nb = (uint32_t)std::min<uint64_t>(16384, std::max<uint64_t>(1, (n + 1023) / 1024));
            uint64_t T = BK_SUB_TILE;
            while (((n + T - 1) / T) * ba.nb > std::max<uint64_t>(n / 4, ba.nb) && T < (1ull << 22))
                T *= 2;
            ba.T = T;
            ba.nchunks = (uint32_t)((n + T - 1) / T);
            ba.mb = bk_masks_per_cta(ba.nb);
            ba.bits = bits;
            ba.sb = sbh;
            ba.runs = level_runs[m];
            ba.sigma = (uint32_t)p->sigma;
            CK(p->ensure(p->bkH, (size_t)nmask * ba.nchunks * ba.nb * 4, s));
            CK(p->ensure(p->bktot, (size_t)nmask * ba.nb * 4, s));
            CK(p->ensure(p->bkbase, (size_t)nmask * (ba.nb + 1) * 4, s));
            ba.H = (uint32_t*)p->bkH.p;
            ba.tot = (uint32_t*)p->bktot.p;
            ba.bbase = (uint32_t*)p->bkbase.p;
            p->stage_begin(s, &a);
            LK(launch_bucket_count(ba, k64, s));
            p->stage_end(s, S_ENCODE, a);
            p->stage_begin(s, &a);
            p->launches += 2;  // colscan + bscan
            LK(launch_bucket_scatter(ba, p->keysA.p, k64, s));
            p->stage_end(s, S_SORT, a);
            if (!k64) keys32 += (int64_t)nmask * (int64_t)n;
            p->stage_begin(s, &a);
            BkScratch bs{(uint64_t*)p->bktab.p, (uint32_t*)p->bktcnt.p, (uint32_t*)p->bkgs.p,
                         (uint32_t*)p->bkocc.p};
            {
                gakco_status ws = wait_buf();
                if (ws != GAKCO_OK) return ws;
            }
            LK(launch_bucket_group(ba, p->keysA.p, k64, dstride, Dm, so, bs, stats, p->sm_count,
                                   s));
            p->stage_end(s, S_SEGMENT, a);
        } else if (n > 0 && trie_b) {
            // batched trie: the batch's masks as one trie, run depth by depth; every
            // depth is one launch whose segments are that depth's nodes
            const int kk = g - m;
            const int P = std::max(1, std::min(4, 8 / bits));  // symbols per pass (digit <= 8 bits)
            const size_t es = tb64 ? 8 : 4;
            std::vector<uint32_t> sets;
            for (size_t j = pos; j < end; ++j) {
                uint32_t b = 0;
                for (int r = 0; r < kk; ++r) b |= 1u << p->mask_kept[mine[j]][r];
                sets.push_back(b);
            }
            std::vector<TrieNode> nodes;
            std::vector<int> leaf_node;
            // cross-level (xlb): this run's generation buffer holds unmasked leaves; a
            // run with parents is one launch of one-symbol passes over their arrays
            const int gen = xl ? (xl_run[pos] & 1) : 0;
            uint8_t* genK = (uint8_t*)(gen ? p->genW1.p : p->genW0.p);
            const uint8_t* pgenK = (const uint8_t*)(gen ? p->genW0.p : p->genW1.p);
            uint8_t* outB = xl ? genK + (size_t)xl_slot[pos] * n * es : (uint8_t*)p->keysA.p;
            const uint64_t seqm = (1ull << sb) - 1ull;
            std::vector<uint64_t> kms;
            for (size_t j = pos; j < end; ++j) {
                uint64_t km = 0;
                for (int r = 0; r < kk; ++r)
                    km |= (uint64_t)((1u << bits) - 1u) << (sb + bits * (g - 1 - p->mask_kept[mine[j]][r]));
                kms.push_back(km | seqm);
            }
            p->stage_begin(s, &a);
            if (kk == 0) {  // no kept position: one key (0), identity order per mask
                for (size_t j = pos; j < end; ++j)  // (cross-level: the unmasked root)
                    LK(launch_trie_root(xl ? (const uint64_t*)p->win.p : nullptr,
                                        (const uint32_t*)p->gmseq.p, n, sb, tb64,
                                        outB + (j - pos) * n * es, p->sm_count, s));
            } else if (xl && xl_parent[pos] >= 0) {
                std::vector<PassDesc> desc;
                for (size_t j = pos; j < end; ++j) {
                    PassDesc pd{};
                    pd.in_off = (uint64_t)xl_parent[j] * n;
                    pd.out_off = (uint64_t)(j - pos) * n;
                    pd.sh[0] = (uint8_t)(sb + bits * (g - 1 - xl_x[j]));
                    pd.nsym = 1;
                    pd.symbits = (uint32_t)bits;
                    pd.omask = ~0ull;
                    desc.push_back(pd);
                }
                CK(p->ensure(p->pdesc, desc.size() * sizeof(PassDesc) + 64, s));
                CK(cudaMemcpyAsync(p->pdesc.p, desc.data(), desc.size() * sizeof(PassDesc),
                                   cudaMemcpyHostToDevice, s));
                int nl = 2;
                LK(launch_trie_batch(pgenK, outB, tb64, n, (int)desc.size(),
                                     (const PassDesc*)p->pdesc.p, (uint32_t*)p->hist.p,
                                     (tb64 ? p->sort_ctas_per_sm : p->sort32_ctas_per_sm) * p->sm_count,
                                     s, &nl));
                p->launches += nl - 1;
                passkeys += (int64_t)desc.size() * (int64_t)n;
                if (!tb64) passkeys32 += (int64_t)desc.size() * (int64_t)n;
            } else if (kk > 0) {
                build_step_trie(sets, kk, P, nodes, leaf_node);
                const int D = (kk + P - 1) / P;
                // per depth: its nodes (index within the depth = slot in the scratch)
                std::vector<std::vector<int>> at(D + 1);
                std::vector<int> slot(nodes.size(), 0);
                for (size_t v = 0; v < nodes.size(); ++v) {
                    slot[v] = (int)at[nodes[v].depth].size();
                    at[nodes[v].depth].push_back((int)v);
                }
                // leaves write the mask's segment of the batch output
                for (size_t i = 0; i < leaf_node.size(); ++i) slot[leaf_node[i]] = (int)i;
                size_t maxw = 0;
                for (int d = 1; d < D; ++d) maxw = std::max(maxw, at[d].size());
                if (maxw > 0) {
                    CK(p->ensure(p->trieX0, maxw * n * es + 64, s));
                    CK(p->ensure(p->trieX1, maxw * n * es + 64, s));
                }
                std::vector<PassDesc> desc;
                std::vector<size_t> dofs(D + 2, 0);
                const uint64_t seqm = (1ull << sb) - 1ull;
                for (int d = 1; d <= D; ++d) {
                    dofs[d] = desc.size();
                    for (int v : at[d]) {
                        PassDesc pd{};
                        const int par = nodes[v].parent;
                        const uint32_t add = nodes[v].set & ~(par >= 0 ? nodes[par].set : 0u);
                        pd.in_off = par >= 0 ? (uint64_t)slot[par] * n : 0;
                        pd.out_off = (uint64_t)slot[v] * n;
                        int q = 0;
                        for (int x = 0; x < 32; ++x)
                            if ((add >> x) & 1u) pd.sh[q++] = (uint8_t)(sb + bits * (g - 1 - x));
                        pd.nsym = (uint32_t)q;
                        pd.symbits = (uint32_t)bits;
                        if (d == D && !xl) {
                            uint64_t km = 0;
                            for (int x = 0; x < 32; ++x)
                                if ((nodes[v].set >> x) & 1u)
                                    km |= (uint64_t)((1u << bits) - 1u) << (sb + bits * (g - 1 - x));
                            pd.omask = km | seqm;
                        } else {
                            pd.omask = ~0ull;
                        }
                        desc.push_back(pd);
                    }
                }
                dofs[D + 1] = desc.size();
                CK(p->ensure(p->pdesc, desc.size() * sizeof(PassDesc) + 64, s));
                CK(cudaMemcpyAsync(p->pdesc.p, desc.data(), desc.size() * sizeof(PassDesc),
                                   cudaMemcpyHostToDevice, s));
                for (int d = 1; d <= D; ++d) {
                    const void* in = d == 1 ? p->trieR.p : ((d - 1) & 1 ? p->trieX1.p : p->trieX0.p);
                    void* outk = d == D ? (void*)outB : (d & 1 ? p->trieX1.p : p->trieX0.p);
                    int nl = 2;
                    LK(launch_trie_batch(in, outk, tb64, n, (int)at[d].size(),
                                         (const PassDesc*)p->pdesc.p + dofs[d], (uint32_t*)p->hist.p,
                                         (tb64 ? p->sort_ctas_per_sm : p->sort32_ctas_per_sm) *
                                             p->sm_count,
                                         s, &nl));
                    p->launches += nl - 1;
                    passkeys += (int64_t)at[d].size() * (int64_t)n;
                    if (!tb64) passkeys32 += (int64_t)at[d].size() * (int64_t)n;
                }
                // (desc: pageable staging, copied out before cudaMemcpyAsync returns; the
                // next batch's upload is stream-ordered after these launches)
            }
            if (!tb64) keys32 += (int64_t)nmask * (int64_t)n;
            p->stage_end(s, S_SORT, a);
            {
                gakco_status ws = wait_buf();
                if (ws != GAKCO_OK) return ws;
            }
            p->stage_begin(s, &a);
            if (xl) {  // unmasked leaves: the segment applies each mask's key bits
                kms.push_back(0);
                CK(cudaMemcpyAsync(p->kmdev.p, kms.data(), kms.size() * 8, cudaMemcpyHostToDevice, s));
                LK(launch_segment(outB, tb64, n, nmask, sb, dstride, Dm, so.counts, so, stats, s,
                                  (const uint64_t*)p->kmdev.p));
            } else {
                LK(launch_segment(p->keysA.p, tb64, n, nmask, sb, dstride, Dm, so.counts, so,
                                  stats, s));
            }
            p->stage_end(s, S_SEGMENT, a);
        } else if (n > 0 && trie && xlc) {
            // cross-level chain with compaction: a child mask is one pass (by its added
            // position) over its parent's COMPACTED sorted elements (device count); the
            // first run of the chain is a trie from the windows; leaves go to the batch
            // buffers and the segment writes this run's compacted copies
            const int kk = g - m;
            const uint32_t dmask = (1u << bits) - 1u;
            const int gen = xl_run[pos] & 1;
            uint64_t* cW = (uint64_t*)(gen ? p->genW1.p : p->genW0.p);
            uint8_t* cS = (uint8_t*)(gen ? p->genS1.p : p->genS0.p);
            uint32_t* cC = (uint32_t*)p->xccnt.p + (size_t)gen * xl_maxrun;
            const uint64_t* pW = (const uint64_t*)(gen ? p->genW0.p : p->genW1.p);
            const uint8_t* pS = (const uint8_t*)(gen ? p->genS0.p : p->genS1.p);
            const uint32_t* pC = (const uint32_t*)p->xccnt.p + (size_t)(gen ^ 1) * xl_maxrun;
            uint32_t* bcnt = (uint32_t*)p->xbcnt.p;
            const bool kids = run_has_kids(xl_run[pos]);
            if (xl_slot[pos] == 0 && kids)  // a run starts: its compacted counts from 0
                CK(cudaMemsetAsync(cC, 0, xl_maxrun * 4, s));
            // fused leaves (leaf.cu): a mask's last pass and its run-length in one kernel
            // over whole groups of the pass before -- where those groups are small: the
            // expected LARGEST one, n f_max^positions (f_max: the most frequent symbol's
            // share; independent symbols), at most 8 tiles (Text's level-5 leaves:
            // 6e6 x 0.24^4 = 2e4 -> unfused, its chain levels from 5 positions (4.8e3)
            // fused; Scale: 41 -> fused). A group past the window is split by its owner
            // CTA into the mask's overflow slot, which the segment kernel takes afterwards.
            // wide leaf CTAs (12 items per thread) where the light path does not share the
            // machine heavily (no relabelled accumulator: Text 76.1 -> 74.7 ms); with the
            // relabelled light path 8 (Scale: 12 gives the leaves 39.3 -> 37.3 ms alone but
            // the step 124.1 -> 129.4, the longer CTAs crowding the light kernel out)
            const bool lf_wide = !relabel;
            auto fuse_ok = [&](int npos) {
                // (the bound, in tiles: Text 0.5 -> 84.5 ms, 1.5 -> 83.6, 8 -> 79.5, 16 ->
                // 79.5, >= 30 -> 92.3 with the owner-CTA split, 86.8 with the queue of
                // leaf.cu: its level-5 leaves, largest groups ~2e4; Scale's expected 41
                // fuses under any bound)
                constexpr double kBigTiles = 8.0;
                return p->leaf_fuse && npos >= 1 &&
                       lf_big_expect(npos) <= (double)leaf_tile(lf_wide) * kBigTiles;
            };
            auto pos_mask = [&](int x) { return (uint64_t)dmask << (bits * (g - 1 - x)); };
            const size_t slot0 = (size_t)xl_slot[pos];
            // (a batch is one level: every mask has kk kept positions; kk >= 2 for a trie
            // leaf, kk >= 1 for a chain pass -- kk - 1 >= 1 either way)
            const bool fused_any = kk >= 2 && fuse_ok(kk - 1);
            // the queue of groups too large for a leaf CTA (leaf_big_kernel): entries,
            // then the two counters
            const uint32_t lbcap = (uint32_t)std::min<uint64_t>(
                1u << 30, (uint64_t)nmask * (n / 256 + 1));
            LfBigList lbl{nullptr, nullptr, 0};
            if (fused_any) {  // the fused leaves write this batch's segment outputs
                gakco_status ws = wait_buf();
                if (ws != GAKCO_OK) return ws;
                CK(cudaMemsetAsync(so.counts, 0, 2 * sizeof(uint32_t), s));
                CK(cudaMemsetAsync(bcnt, 0, (size_t)nmask * 4, s));
                CK(p->ensure(p->lbig, (size_t)lbcap * sizeof(LfBig) + 64, s));
                lbl = LfBigList{(LfBig*)p->lbig.p, (uint32_t*)((uint8_t*)p->lbig.p + (size_t)lbcap * sizeof(LfBig)),
                                lbcap};
                CK(cudaMemsetAsync(lbl.count, 0, 2 * sizeof(uint32_t), s));
            }
            std::vector<uint64_t> kms;
            for (size_t j = pos; j < end; ++j) {
                const uint8_t* kept = trie_chain[j].data();
                uint64_t* wleaf = (uint64_t*)p->keysA.p + (j - pos) * n;
                uint8_t* sleaf = (uint8_t*)p->keysB.p + (j - pos) * n * ssz;
                uint32_t* ocnt = bcnt + (j - pos);
                uint64_t kmask = 0;
                for (int r = 0; r < kk; ++r) kmask |= pos_mask(p->mask_kept[mine[j]][r]);
                kms.push_back(kmask);
                uint64_t* lcw = kids ? cW + (size_t)xl_slot[j] * n : nullptr;
                void* lcs = kids ? (void*)(cS + (size_t)xl_slot[j] * n * ssz) : nullptr;
                uint32_t* lcc = kids ? cC + xl_slot[j] : nullptr;
                p->stage_begin(s, &a);
                if (kk == 0) {  // no kept position: one key, identity order (raw windows)
                    CK(cudaMemcpyAsync(wleaf, p->win.p, n * 8, cudaMemcpyDeviceToDevice, s));
                    CK(cudaMemcpyAsync(sleaf, p->trieS0.p, n * ssz, cudaMemcpyDeviceToDevice, s));
                    LK(launch_fill_u32(ocnt, (uint32_t)n, 1, s));
                    p->stage_end(s, S_SORT, a);
                    continue;
                }
                if (xl_parent[j] >= 0) {  // one pass over the parent's compacted elements
                    const uint64_t* iw = pW + (size_t)xl_parent[j] * n;
                    const void* is = pS + (size_t)xl_parent[j] * n * ssz;
                    const int sh = bits * (g - 1 - xl_x[j]);
                    if (fuse_ok(kk - 1)) {
                        p->stage_end(s, S_SORT, a);
                        p->stage_begin(s, &a);
                        p->launches += 1;
                        LK(launch_leaf(iw, is, seq16, n, pC + xl_parent[j], kmask & ~pos_mask(xl_x[j]),
                                       kmask, sh, dmask, dstride, Dm, so, stats, lcw, lcs, lcc, wleaf,
                                       sleaf, ocnt, lbl, s, lf_wide));
                        p->stage_end(s, S_SEGMENT, a);
                    } else {
                        LK(launch_trie_pass64(iw, wleaf, is, sleaf, seq16, n, pC + xl_parent[j], sh,
                                              dmask, ~0ull, (uint32_t*)p->hist.p,
                                              p->trie_ctas_per_sm * p->sm_count, s, ocnt, stats,
                                              (uint32_t*)p->thg.p, &p->tp_par));
                        p->launches += 1;  // hist + scatter
                        p->stage_end(s, S_SORT, a);
                    }
                    passkeys += (int64_t)n;  // (capacity: the actual count is on the device)
                    continue;
                }
                const bool fl = kk >= 2 && fuse_ok(kk - 1);  // (the last pass fused)
                int d = 0;
                while (d < stack_depth && d < kk - 1 && stack_pos[d] == kept[d]) ++d;
                for (int t = d; t < kk - (fl ? 1 : 0); ++t) {
                    const bool leaf = t == kk - 1;
                    const uint64_t* wi = t == 0 ? (const uint64_t*)p->win.p
                                                : (const uint64_t*)p->trieW.p + (size_t)(t - 1) * n;
                    const void* si = t == 0 ? p->trieS0.p
                                            : (const void*)((const uint8_t*)p->trieS.p + (size_t)(t - 1) * n * ssz);
                    uint64_t* wo = leaf ? wleaf : (uint64_t*)p->trieW.p + (size_t)t * n;
                    void* so_ = leaf ? (void*)sleaf : (void*)((uint8_t*)p->trieS.p + (size_t)t * n * ssz);
                    LK(launch_trie_pass64(wi, wo, si, so_, seq16, n, nullptr, bits * (g - 1 - kept[t]),
                                          dmask, ~0ull, (uint32_t*)p->hist.p,
                                          p->trie_ctas_per_sm * p->sm_count, s,
                                          leaf ? ocnt : nullptr, stats, (uint32_t*)p->thg.p, &p->tp_par));
                    p->launches += 1;
                    if (!leaf) stack_pos[t] = kept[t];
                }
                stack_depth = kk - 1;
                passkeys += (int64_t)(kk - d) * (int64_t)n;
                p->stage_end(s, S_SORT, a);
                if (fl) {  // the last pass over the stack's top (sorted by kept[0 .. kk-2])
                    uint64_t pm = 0;
                    for (int r = 0; r < kk - 1; ++r) pm |= pos_mask(kept[r]);
                    p->stage_begin(s, &a);
                    p->launches += 1;
                    // (groups past a CTA's window expected: queued and split right after
                    // this leaf, while the stack top still holds its input; else the rare
                    // one is split by its own CTA)
                    const bool tq = lf_big_expect(kk - 1) > (double)leaf_tile(lf_wide);
                    LK(launch_leaf((const uint64_t*)p->trieW.p + (size_t)(kk - 2) * n,
                                   (const uint8_t*)p->trieS.p + (size_t)(kk - 2) * n * ssz, seq16, n,
                                   nullptr, pm, kmask, bits * (g - 1 - kept[kk - 1]), dmask, dstride, Dm,
                                   so, stats, lcw, lcs, lcc, wleaf, sleaf, ocnt,
                                   tq ? lbl : LfBigList{nullptr, nullptr, 0}, s, lf_wide));
                    if (tq) {
                        p->launches += 1;
                        LK(launch_leaf_big(lbl, seq16, p->sm_count, s));
                        CK(cudaMemsetAsync(lbl.count, 0, 2 * sizeof(uint32_t), s));
                    }
                    p->stage_end(s, S_SEGMENT, a);
                }
            }
            if (!fused_any) {
                gakco_status ws = wait_buf();
                if (ws != GAKCO_OK) return ws;
            } else if (xl_parent[pos] >= 0) {  // the chain's queued large groups (the
                // parents' compacted arrays are stable through the batch)
                p->stage_begin(s, &a);
                p->launches += 1;
                LK(launch_leaf_big(lbl, seq16, p->sm_count, s));
                CK(cudaMemsetAsync(lbl.count, 0, 2 * sizeof(uint32_t), s));
                p->stage_end(s, S_SEGMENT, a);
            }
            p->stage_begin(s, &a);
            kms.push_back(0);
            CK(cudaMemcpyAsync(p->kmdev.p, kms.data(), kms.size() * 8, cudaMemcpyHostToDevice, s));
            // the leaves of unfused masks, the overflow of fused ones (most slots empty:
            // a looping grid)
            LK(launch_segment_rag((const uint64_t*)p->keysA.p, p->keysB.p, seq16, n, nmask, bcnt,
                                  (const uint64_t*)p->kmdev.p, dstride, Dm, so.counts, so, stats, s,
                                  kids ? cW + slot0 * n : nullptr, kids ? cS + slot0 * n * ssz : nullptr,
                                  kids ? cC + slot0 : nullptr, /*reset=*/!fused_any,
                                  fused_any ? (unsigned)(4 * p->sm_count) : 0u));
            p->stage_end(s, S_SEGMENT, a);
        } else if (n > 0 && trie) {
            // mask trie: pass t of a mask is a stable pass by the symbol at its t-th kept
            // position (ascending); the passes of a common leading-position prefix are
            // shared with the previous mask (stack), the last pass writes the masked
            // windows to the mask's segment of the batch
            const int kk = g - m;
            const uint32_t dmask = (1u << bits) - 1u;
            // symbol digits of <= 6 bits: the two-launch pass of trie.cu (option 0: the
            // generic three-launch radix pass, for comparison)
            const bool tp64 = p->trie_pass == 1 && trie_pass64_ok(dmask);
            // (cross-level: this run's generation buffer; else the batch buffers)
            const int gen = xl ? (xl_run[pos] & 1) : 0;
            uint64_t* genW = (uint64_t*)(gen ? p->genW1.p : p->genW0.p);
            uint8_t* genS = (uint8_t*)(gen ? p->genS1.p : p->genS0.p);
            const uint64_t* pgenW = (const uint64_t*)(gen ? p->genW0.p : p->genW1.p);
            const uint8_t* pgenS = (const uint8_t*)(gen ? p->genS0.p : p->genS1.p);
            std::vector<uint64_t> kms;
            p->stage_begin(s, &a);
            for (size_t j = pos; j < end; ++j) {
                const uint8_t* kept = trie_chain[j].data();  // positions in pass order
                uint64_t* wleaf = xl ? genW + (size_t)xl_slot[j] * n
                                     : (uint64_t*)p->keysA.p + (j - pos) * n;
                uint8_t* sleaf = xl ? genS + (size_t)xl_slot[j] * n * ssz
                                    : (uint8_t*)p->keysB.p + (j - pos) * n * ssz;
                uint64_t kmask = 0;
                for (int r = 0; r < kk; ++r)
                    kmask |= (uint64_t)dmask << (bits * (g - 1 - p->mask_kept[mine[j]][r]));
                kms.push_back(kmask);
                if (kk == 0) {  // no kept position: one key, identity order (cross-level:
                    // the unmasked windows, the next level's parent; the segment masks)
                    if (xl)
                        CK(cudaMemcpyAsync(wleaf, p->win.p, n * 8, cudaMemcpyDeviceToDevice, s));
                    else
                        CK(cudaMemsetAsync(wleaf, 0, n * 8, s));
                    CK(cudaMemcpyAsync(sleaf, p->trieS0.p, n * ssz, cudaMemcpyDeviceToDevice, s));
                    continue;
                }
                if (xl && xl_parent[j] >= 0) {  // one pass over the parent mask's arrays
                    int nl = 2;
                    if (tp64)
                        LK(launch_trie_pass64(pgenW + (size_t)xl_parent[j] * n, wleaf,
                                              pgenS + (size_t)xl_parent[j] * n * ssz, sleaf, seq16, n,
                                              nullptr, bits * (g - 1 - xl_x[j]), dmask, ~0ull,
                                              (uint32_t*)p->hist.p, p->trie_ctas_per_sm * p->sm_count, s,
                                              nullptr, stats, (uint32_t*)p->thg.p, &p->tp_par));
                    else
                        LK(launch_trie_pass(pgenW + (size_t)xl_parent[j] * n, wleaf,
                                            pgenS + (size_t)xl_parent[j] * n * ssz, sleaf, seq16, n,
                                            bits * (g - 1 - xl_x[j]), dmask, ~0ull,
                                            (uint32_t*)p->hist.p, p->trie_ctas_per_sm * p->sm_count, s,
                                            &nl));
                    p->launches += nl - 1;
                    passkeys += (int64_t)n;
                    continue;
                }
                int d = 0;
                while (d < stack_depth && d < kk - 1 && stack_pos[d] == kept[d]) ++d;
                for (int t = d; t < kk; ++t) {
                    const bool leaf = t == kk - 1;
                    const uint64_t* wi = t == 0 ? (const uint64_t*)p->win.p
                                                : (const uint64_t*)p->trieW.p + (size_t)(t - 1) * n;
                    const void* si = t == 0 ? p->trieS0.p
                                            : (const void*)((const uint8_t*)p->trieS.p + (size_t)(t - 1) * n * ssz);
                    uint64_t* wo = leaf ? wleaf : (uint64_t*)p->trieW.p + (size_t)t * n;
                    void* so_ = leaf ? (void*)sleaf : (void*)((uint8_t*)p->trieS.p + (size_t)t * n * ssz);
                    int nl = 2;
                    if (tp64)
                        LK(launch_trie_pass64(wi, wo, si, so_, seq16, n, nullptr, bits * (g - 1 - kept[t]),
                                              dmask, leaf && !xl ? kmask : ~0ull, (uint32_t*)p->hist.p,
                                              p->trie_ctas_per_sm * p->sm_count, s, nullptr, stats, (uint32_t*)p->thg.p, &p->tp_par));
                    else
                        LK(launch_trie_pass(wi, wo, si, so_, seq16, n, bits * (g - 1 - kept[t]), dmask,
                                            leaf && !xl ? kmask : ~0ull, (uint32_t*)p->hist.p,
                                            p->trie_ctas_per_sm * p->sm_count, s, &nl));
                    p->launches += nl - 1;  // hist (+ chunk scan) + scatter
                    if (!leaf) stack_pos[t] = kept[t];
                }
                stack_depth = kk - 1;
                passkeys += (int64_t)(kk - d) * (int64_t)n;
            }
            p->stage_end(s, S_SORT, a);
            {
                gakco_status ws = wait_buf();
                if (ws != GAKCO_OK) return ws;
            }
            p->stage_begin(s, &a);
            if (xl) {  // the run's arrays are unmasked: the segment applies each mask's bits
                kms.push_back(0);
                CK(cudaMemcpyAsync(p->kmdev.p, kms.data(), kms.size() * 8, cudaMemcpyHostToDevice, s));
                LK(launch_segment_soa(genW + (size_t)xl_slot[pos] * n, genS + (size_t)xl_slot[pos] * n * ssz,
                                      seq16, n, nmask, dstride, Dm, so.counts, so, stats, s,
                                      (const uint64_t*)p->kmdev.p));
            } else {
                LK(launch_segment_soa((const uint64_t*)p->keysA.p, p->keysB.p, seq16, n, nmask,
                                      dstride, Dm, so.counts, so, stats, s));
            }
            p->stage_end(s, S_SEGMENT, a);
        } else if (n > 0) {
            p->stage_begin(s, &a);
            const bool onesweep = p->sort_mode == 1;
            // 32-bit composites when key + sequence bits fit (half the key traffic)
            const bool k64 = onesweep || kb + sb > 32;
            if (onesweep) CK(cudaMemsetAsync(p->hist.p, 0, (size_t)nmask * MAXPASS * RADIX * 4, s));
            if (use_win)
                LK(launch_encode_win((const uint64_t*)p->win.p, (const uint32_t*)p->gmseq.p, n,
                                     (const uint8_t*)p->keptsh.p + pos * GMAX, g - m, p->sigma,
                                     bits, sb, nmask, p->keysA.p, k64, s));
            else
                LK(launch_encode(cv, (const uint8_t*)p->kept.p + pos * GMAX, g - m, p->sigma, sb,
                                 nmask, onesweep ? npass : 0, p->keysA.p, k64,
                                 (uint32_t*)p->hist.p, s));
            p->stage_end(s, S_ENCODE, a);

            p->stage_begin(s, &a);
            void* in = p->keysA.p;
            void* outk = p->keysB.p;
            for (int q = 0; q < npass; ++q) {
                if (onesweep) {
                    uint32_t* c;
                    CK(p->next_ctr(s, &c));
                    LK(launch_onesweep((const uint64_t*)in, (uint64_t*)outk, n, nmask,
                                       sb + RADIX_BITS * q, (const uint32_t*)p->hist.p, q, npass,
                                       (uint64_t*)p->status.p, c, p->epoch++, s));
                } else {
                    // auto: the v2 pass (bulk-copied tiles, atomicOr-match ranking)
                    const bool v2 = p->sort_mode >= 3 || p->sort_mode == -1;
                    if (v2) {  // hist (+ a chunk scan when many chunks) + scatter
                        int nl = 2;
                        LK(launch_radix_chunked2(in, outk, k64, n, nmask, sb + RADIX_BITS * q,
                                                 (uint32_t*)p->hist.p,
                                                 (k64 ? p->sort_ctas_per_sm : p->sort32_ctas_per_sm) *
                                                     p->sm_count,
                                                 p->sort_mode >= 3 ? p->sort_mode - 3 : 0, s, &nl));
                        p->launches += nl - 1;
                    } else {
                        p->launches += 1;  // hist + scatter
                    }
                    if (!v2)
                        LK(launch_radix_chunked(in, outk, k64, n, nmask, sb + RADIX_BITS * q,
                                                (uint32_t*)p->hist.p,
                                                p->sort_ctas_per_sm * p->sm_count, s));
                }
                std::swap(in, outk);
            }
            passkeys += (int64_t)npass * nmask * (int64_t)n;
            if (!k64) {
                keys32 += (int64_t)nmask * (int64_t)n;
                passkeys32 += (int64_t)npass * nmask * (int64_t)n;
            }
            p->stage_end(s, S_SORT, a);

            {
                gakco_status ws = wait_buf();
                if (ws != GAKCO_OK) return ws;
            }
            p->stage_begin(s, &a);
            LK(launch_segment(in, k64, n, nmask, sb, dstride, Dm, so.counts, so, stats, s));
            p->stage_end(s, S_SEGMENT, a);

        }
        if (n > 0) {
            // light and dense build of this batch on s2, after its segment on s
            if (pipe) {
                CK(cudaEventRecord(p->ev_seg[bi], s));
                CK(cudaStreamWaitEvent(s2, p->ev_seg[bi], 0));
            }
            p->stage_begin(s2, &a);
            LK(launch_light(so, n * nmask / 2 + 1, light_limit_of(m), N, (uint32_t*)p->lightacc.p,
                            heavy_p(), rcap_of(m), hcount_p(), bins,
                            (uint32_t)p->light_flat, NA,
                            perm_active ? (const uint32_t*)p->perm.p : nullptr,
                            fp4_lv[m] ? 4u : 255u, stats, p->sm_count, s2,
                            perm_active && win_on ? wa : WinArgs{nullptr, nullptr, 0, 0, 0},
                            n >= (2ull << 20), perm_active ? farb[fcur] : FarRec{nullptr, nullptr, 0, 0},
                            p->light_ctas,
                            // (relabelled: a 3-CTA/SM grid leaves room for the next batch's
                            // passes on s: Scale 171-177 -> 166-167 ms; else 8 per SM)
                            p->light_grid > 0 ? p->light_grid : (perm_active ? 3 : 8)));
            p->stage_end(s2, S_LIGHT, a);
            if (perm_active && far.near) {
                // the apply is worth it once many records are pending (each block's
                // cells then hit several times). The count is copied to a pinned ring
                // after every batch and polled without waiting (the copy of FAR_LAG
                // batches ago): apply when it shows half the buffer used; if no count
                // newer than the last apply has been seen for FAR_EVERY (12) batches (the host
                // far ahead of the GPU), apply anyway -- at Scale's <= 58M records per
                // batch the buffer cannot fill in between. No host wait either way.
                constexpr int LAG = gakco_plan::FAR_LAG, RING = gakco_plan::FAR_RING;
                const int64_t fb = far_batch++;
                bool due = false;
                if (fb >= LAG) {
                    const int q = (int)((fb - LAG) % RING);
                    const bool seen = cudaEventQuery(p->ev_far[q]) == cudaSuccess;
                    cudaGetLastError();  // (cudaErrorNotReady is not an error here)
                    if (seen && far_last_apply < fb - LAG + 1) {
                        far_seen_at = fb - LAG;
                        due = p->far_seen[q] >= far_thresh;
                    }
                }
                due = due || fb - std::max(far_last_apply, far_seen_at) >= gakco_plan::FAR_EVERY;
                {
                    if (due) {
                        cudaStream_t sf = far2 ? s3 : s2;
                        if (far2) {  // (this batch's records written)
                            CK(cudaEventRecord(p->ev_fsrc, s2));
                            CK(cudaStreamWaitEvent(s3, p->ev_fsrc, 0));
                        }
                        p->stage_begin(sf, &a);
                        p->launches += 4 + 2 * 16;
                        LK(launch_far_apply(farb[fcur], p->farscr.p, (uint32_t*)p->farbins.p + 256,
                                            far_bshift, (uint32_t*)p->lightacc.p, ntri, p->sm_count, sf));
                        p->stage_end(sf, S_FAR, a);
                        if (far2) {  // the other buffer next, once its own last apply is done
                            CK(cudaEventRecord(p->ev_fapply[fcur], s3));
                            fapplied[fcur] = true;
                            fcur ^= 1;
                            if (fapplied[fcur]) CK(cudaStreamWaitEvent(s2, p->ev_fapply[fcur], 0));
                        }
                        far_last_apply = fb;
                    }
                }
                CK(cudaMemcpyAsync(p->far_seen + (fb % RING), farb[fcur].fill, 4, cudaMemcpyDeviceToHost, s2));
                CK(cudaEventRecord(p->ev_far[fb % RING], s2));
            }
            if (perm_active && win_on) {  // this batch's window columns (+ the Gram every few)
                if (win_masks + nmask > win_lim) {  // s32 exactness of the next Gram
                    gakco_status ws = wgram();
                    if (ws != GAKCO_OK) return ws;
                }
                win_masks += nmask;
                p->stage_begin(s2, &a);
                p->launches += 1;  // + round
                LK(launch_window_build(so, wa, (const uint32_t*)p->perm.p, (uint8_t*)p->wD.p,
                                       p->sm_count, s2));
                p->stage_end(s2, S_DENSE, a);
                if (++win_pending >= WIN_BATCHES) {
                    gakco_status ws = wgram();
                    if (ws != GAKCO_OK) return ws;
                }
            }
            if (gram_ok) {
                p->stage_begin(s2, &a);
                p->launches += 1;  // + fill_round
                LK(launch_build_dense(so, heavy_p(), hcount_p(), dense_p(), n_pad, rcap_of(m),
                                      hash_mode ? 0 : 1,
                                      fp4_lv[m] ? 1 : 0, p->sm_count, s2));
                p->stage_end(s2, S_DENSE, a);
            }
            if (pipe) CK(cudaEventRecord(p->ev_light[bi], s2));
            ++batch_no;
        }
        LK(launch_diag_closed_form((const int64_t*)p->gofs.p, N, nmask, Dm, dstride, s));
        pos = end;
    }
    {
        gakco_status fs = flush();
        if (fs != GAKCO_OK) return fs;
        fs = lflush();
        if (fs != GAKCO_OK) return fs;
        if (prev_level >= 0 && only_level < 0) {
            fs = mark_level(prev_level);
            if (fs != GAKCO_OK) return fs;
        }
    }
    if (pipe) {  // the caller's stream sees every s2 / s3 kernel as done
        CK(cudaEventRecord(p->ev_join, s2));
        CK(cudaStreamWaitEvent(s, p->ev_join, 0));
        CK(cudaEventRecord(p->ev_join2, s3));
        CK(cudaStreamWaitEvent(s, p->ev_join2, 0));
    }
    p->last_masks = (int64_t)mine.size();
    p->host_stats = gakco_stats{};
    p->host_stats.masks = (int64_t)mine.size();
    p->host_stats.keys = (int64_t)mine.size() * (int64_t)n;
    p->host_stats.sort_passes = passkeys;
    p->host_stats.keys32 = keys32;
    p->host_stats.sort_passes32 = passkeys32;
    p->host_stats.grouping = p->last_grouping;
    p->host_stats.n_pad = gram_ok ? n_pad : 0;
    p->host_stats.gram_fp4 = gram_ok ? fp4_used : 0;
    p->host_stats.ms_host =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_entry).count();
    HT("end");
    if (p->htrace_on) {
        std::string o = "{\"host_trace\": [";
        for (size_t i = 0; i < p->htrace.size(); ++i) {
            char b[96];
            std::snprintf(b, sizeof b, "%s[\"%s\", %.2f]", i ? ", " : "", p->htrace[i].first.c_str(),
                          p->htrace[i].second);
            o += b;
        }
        std::fprintf(stderr, "%s]}\n", o.c_str());
    }
    p->after_accumulate = true;
    return GAKCO_OK;
#undef CK
#undef LK
}

extern "C" gakco_status gakco_accumulate(gakco_plan* p, const uint8_t* codes,
                                         const int64_t* offsets, int64_t N, int64_t* C,
                                         void* stream) {
    if (!p) return GAKCO_E_ARG;
    DeviceGuard dg(p->device);
    Nvtx nv("gakco_accumulate");
    return accumulate_impl(p, codes, offsets, N, C, (cudaStream_t)stream, p->rank, p->world);
}

// k_only: C is the single level g-k and K = C_{g-k} (the epilogue runs with
// g = k = 1, M = 0, i.e. K = N_0 = C_0, and Nm is not produced).
static gakco_status finalize_impl(gakco_plan* p, int64_t* C, int64_t N, int64_t* Nm, int64_t* K,
                                  double* Knorm, cudaStream_t s, bool keep_events,
                                  bool k_only = false) {
#define CK(x)                                          \
    do {                                               \
        cudaError_t e_ = (x);                          \
        if (e_ != cudaSuccess) return p->cuda_fail(e_, #x); \
    } while (0)
#define LK(x)        \
    do {             \
        ++p->launches; \
        CK(x);       \
    } while (0)
    if (!C || N < 1) return p->fail(GAKCO_E_ARG, "C is NULL or N < 1");
    if (!is_device_ptr(C)) return p->fail(GAKCO_E_ARG, "C must be a device pointer");
    // A finalize that directly follows an accumulate on this plan appends to its
    // stage events and launch count (so one stats read covers the whole step).
    if (!keep_events && !p->after_accumulate) {
        p->evs.clear();
        p->ev_used = 0;
        p->launches = 0;
        for (int64_t& v : p->stage_launches) v = 0;
    }
    p->after_accumulate = false;
    p->last_stream = s;
    const size_t nn = (size_t)N * N;
    const int M = k_only ? 0 : p->M;
    if (k_only) Nm = nullptr;
    int64_t* dNm = Nm;
    int64_t* dK = K;
    double* dKn = Knorm;
    const bool hNm = Nm && !is_device_ptr(Nm), hK = K && !is_device_ptr(K),
               hKn = Knorm && !is_device_ptr(Knorm);
    if (hNm) {
        CK(p->ensure(p->Nmscr, (M + 1) * nn * 8, s));
        dNm = (int64_t*)p->Nmscr.p;
    }
    if (hK) {
        CK(p->ensure(p->Kscr, nn * 8, s));
        dK = (int64_t*)p->Kscr.p;
    }
    if (hKn) {
        CK(p->ensure(p->Knscr, nn * 8, s));
        dKn = (double*)p->Knscr.p;
    }
    CK(p->ensure(p->kdiag, N * 8, s));
    CK(p->ensure(p->flags, 64, s, /*zero=*/true));
    CK(cudaMemsetAsync(p->flags.p, 0, sizeof(int), s));
    cudaEvent_t a = nullptr;
    p->stage_begin(s, &a);
    LK(launch_epilogue(C, N, k_only ? 1 : p->g, k_only ? 1 : p->k, M, dNm, dK, dKn,
                       (int64_t*)p->kdiag.p, (int*)p->flags.p,
                       s));
    p->stage_end(s, S_EPILOGUE, a);
    if (hNm) CK(cudaMemcpyAsync(Nm, dNm, (M + 1) * nn * 8, cudaMemcpyDeviceToHost, s));
    if (hK) CK(cudaMemcpyAsync(K, dK, nn * 8, cudaMemcpyDeviceToHost, s));
    if (hKn) CK(cudaMemcpyAsync(Knorm, dKn, nn * 8, cudaMemcpyDeviceToHost, s));
    int fl[2] = {0, 0};
    CK(cudaMemcpyAsync(fl, p->flags.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemsetAsync((int*)p->flags.p + 1, 0, sizeof(int), s));  // symbol flag consumed
    CK(cudaStreamSynchronize(s));
    if (fl[1] & EF_BAD_SYMBOL) return p->fail(GAKCO_E_SYMBOL, "a code is >= sigma");
    if (fl[0] & EF_NEGATIVE_N) return p->fail(GAKCO_E_INTERNAL, "negative N_m after Eq. 9");
    if (fl[0] & EF_K_MISMATCH) return p->fail(GAKCO_E_INTERNAL, "K != C_{g-k}");
    return GAKCO_OK;
#undef CK
#undef LK
}

extern "C" gakco_status gakco_finalize(gakco_plan* p, int64_t* C, int64_t N, int64_t* Nm,
                                       int64_t* K, double* Knorm, void* stream) {
    if (!p) return GAKCO_E_ARG;
    DeviceGuard dg(p->device);
    Nvtx nv("gakco_finalize");
    return finalize_impl(p, C, N, Nm, K, Knorm, (cudaStream_t)stream, false);
}

extern "C" gakco_status gakco_kernel(gakco_plan* p, const uint8_t* codes, const int64_t* offsets,
                                     int64_t N, int64_t* C, int64_t* Nm, int64_t* K, double* Knorm,
                                     void* stream) {
    if (!p) return GAKCO_E_ARG;
    if (N < 1 || N >= ((int64_t)1 << 31)) return p->fail(GAKCO_E_ARG, "N must be in [1, 2^31)");
    DeviceGuard dg(p->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)(p->M + 1) * N * N * 8;
    int64_t* dC = C;
    const bool hC = C && !is_device_ptr(C);
    if (!C || hC) {
        cudaError_t e = p->ensure(p->Cscr, bytes, s);
        if (e != cudaSuccess) return p->cuda_fail(e, "C scratch");
        dC = (int64_t*)p->Cscr.p;
    }
    // (the upper triangles only: accumulate adds there, finalize reads there and
    // writes the mirror)
    cudaError_t e = launch_zero_upper(dC, N, p->M + 1, p->sm_count, s);
    if (e != cudaSuccess) return p->cuda_fail(e, "zero C");
    gakco_status st = accumulate_impl(p, codes, offsets, N, dC, s, 0, 1);
    if (st != GAKCO_OK) return st;
    st = finalize_impl(p, dC, N, Nm, K, Knorm, s, true);
    if (st != GAKCO_OK) return st;
    if (hC) {
        e = cudaMemcpyAsync(C, dC, bytes, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return p->cuda_fail(e, "copy C to host");
    }
    return GAKCO_OK;
}

extern "C" gakco_status gakco_kernel_k(gakco_plan* p, const uint8_t* codes,
                                       const int64_t* offsets, int64_t N, int64_t* K,
                                       double* Knorm, void* stream) {
    if (!p) return GAKCO_E_ARG;
    if (N < 1 || N >= ((int64_t)1 << 31)) return p->fail(GAKCO_E_ARG, "N must be in [1, 2^31)");
    if (p->M < p->g - p->k)
        return p->fail(GAKCO_E_ARG, "K-only path needs M >= g-k (K = C_{g-k})");
    if (!K && !Knorm) return p->fail(GAKCO_E_ARG, "K and Knorm are both NULL");
    DeviceGuard dg(p->device);
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)N * N * 8;
    cudaError_t e = p->ensure(p->Cscr, bytes, s);
    if (e != cudaSuccess) return p->cuda_fail(e, "C scratch");
    int64_t* dC = (int64_t*)p->Cscr.p;
    e = launch_zero_upper(dC, N, 1, p->sm_count, s);
    if (e != cudaSuccess) return p->cuda_fail(e, "zero C");
    gakco_status st = accumulate_impl(p, codes, offsets, N, dC, s, 0, 1, p->g - p->k);
    if (st != GAKCO_OK) return st;
    return finalize_impl(p, dC, N, nullptr, K, Knorm, s, true, /*k_only=*/true);
}

// Rectangular train x test block: sequences [0, NA) are the
// training set X_i, [NA, N) the test set; outputs are the NA x (N - NA) block of
// C_m / N_m / K / Knorm of the concatenated corpus (the paper concatenates
// train and test into one N x N problem), without the train x train and test x
// test pair updates, plus K(X,X) of all N sequences (normalisation; Eq. 1).
extern "C" gakco_status gakco_kernel_rect(gakco_plan* p, const uint8_t* codes,
                                          const int64_t* offsets, int64_t N, int64_t NA,
                                          int64_t* C, int64_t* Nm, int64_t* K, double* Knorm,
                                          int64_t* Kdiag, void* stream) {
#define CK(x)                                               \
    do {                                                    \
        cudaError_t e_ = (x);                               \
        if (e_ != cudaSuccess) return p->cuda_fail(e_, #x); \
    } while (0)
    if (!p) return GAKCO_E_ARG;
    if (N < 2 || N >= ((int64_t)1 << 31)) return p->fail(GAKCO_E_ARG, "N must be in [2, 2^31)");
    if (NA < 1 || NA >= N) return p->fail(GAKCO_E_ARG, "NA must be in [1, N-1]");
    DeviceGuard dg(p->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t NB = N - NA;
    const int M = p->M;
    const size_t cells = (size_t)NA * (size_t)NB;
    const size_t cbytes = (size_t)(M + 1) * cells * 8;
    int64_t* dC = C;
    const bool hC = C && !is_device_ptr(C);
    if (!C || hC) {
        CK(p->ensure(p->Cscr, cbytes, s));
        dC = (int64_t*)p->Cscr.p;
    }
    CK(p->ensure(p->Dgscr, (size_t)(M + 1) * N * 8, s));
    int64_t* Dg = (int64_t*)p->Dgscr.p;
    CK(cudaMemsetAsync(dC, 0, cbytes, s));
    CK(cudaMemsetAsync(Dg, 0, (size_t)(M + 1) * N * 8, s));
    gakco_status st = accumulate_impl(p, codes, offsets, N, dC, s, 0, 1, -1, NA, Dg);
    if (st != GAKCO_OK) return st;
    // outputs: device pointers written in place, host ones through plan scratch
    int64_t* dNm = Nm;
    int64_t* dK = K;
    double* dKn = Knorm;
    int64_t* dKd = Kdiag;
    const bool hNm = Nm && !is_device_ptr(Nm), hK = K && !is_device_ptr(K),
               hKn = Knorm && !is_device_ptr(Knorm), hKd = Kdiag && !is_device_ptr(Kdiag);
    if (hNm) {
        CK(p->ensure(p->Nmscr, cbytes, s));
        dNm = (int64_t*)p->Nmscr.p;
    }
    if (hK) {
        CK(p->ensure(p->Kscr, cells * 8, s));
        dK = (int64_t*)p->Kscr.p;
    }
    if (hKn) {
        CK(p->ensure(p->Knscr, cells * 8, s));
        dKn = (double*)p->Knscr.p;
    }
    if (!Kdiag || hKd) {
        CK(p->ensure(p->Kdscr, N * 8, s));
        dKd = (int64_t*)p->Kdscr.p;
    }
    CK(p->ensure(p->flags, 64, s, /*zero=*/true));
    CK(cudaMemsetAsync(p->flags.p, 0, sizeof(int), s));
    cudaEvent_t a = nullptr;
    p->after_accumulate = false;
    p->stage_begin(s, &a);
    ++p->launches;
    CK(launch_epilogue_rect(dC, Dg, N, NA, p->g, p->k, M, dNm, dK, dKn, dKd, (int*)p->flags.p,
                            p->sm_count, s));
    p->stage_end(s, S_EPILOGUE, a);
    if (hC) CK(cudaMemcpyAsync(C, dC, cbytes, cudaMemcpyDeviceToHost, s));
    if (hNm) CK(cudaMemcpyAsync(Nm, dNm, cbytes, cudaMemcpyDeviceToHost, s));
    if (hK) CK(cudaMemcpyAsync(K, dK, cells * 8, cudaMemcpyDeviceToHost, s));
    if (hKn) CK(cudaMemcpyAsync(Knorm, dKn, cells * 8, cudaMemcpyDeviceToHost, s));
    if (hKd) CK(cudaMemcpyAsync(Kdiag, dKd, N * 8, cudaMemcpyDeviceToHost, s));
    int fl[2] = {0, 0};
    CK(cudaMemcpyAsync(fl, p->flags.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemsetAsync((int*)p->flags.p + 1, 0, sizeof(int), s));
    CK(cudaStreamSynchronize(s));
    if (fl[1] & EF_BAD_SYMBOL) return p->fail(GAKCO_E_SYMBOL, "a code is >= sigma");
    if (fl[0] & EF_NEGATIVE_N) return p->fail(GAKCO_E_INTERNAL, "negative N_m after Eq. 9");
    if (fl[0] & EF_K_MISMATCH) return p->fail(GAKCO_E_INTERNAL, "K != C_{g-k}");
    return GAKCO_OK;
#undef CK
}

extern "C" gakco_status gakco_get_stats(gakco_plan* p, gakco_stats* out) {
    if (!p || !out) return GAKCO_E_ARG;
    DeviceGuard dg(p->device);
    gakco_stats r = p->host_stats;
    r.launches = p->launches;
    int64_t* nl[S_NSTAGE] = {&r.n_encode, &r.n_sort,     &r.n_segment, &r.n_light,
                             &r.n_heavy,  &r.n_epilogue, &r.n_dense,   &r.n_far};
    for (int i = 0; i < S_NSTAGE; ++i) *nl[i] = p->stage_launches[i];
    if (p->stats.p) {
        unsigned long long d[ST_COUNT];
        cudaError_t e = cudaMemcpyAsync(d, p->stats.p, sizeof d, cudaMemcpyDeviceToHost,
                                        p->last_stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(p->last_stream);
        if (e != cudaSuccess) return p->cuda_fail(e, "stats");
        r.triples = (int64_t)d[ST_TRIPLES];
        r.groups_multi = (int64_t)d[ST_GROUPS];
        r.light_pairs = (int64_t)d[ST_LIGHT_PAIRS];
        r.heavy_groups = (int64_t)d[ST_HEAVY_GROUPS];
        r.heavy_macs = (int64_t)d[ST_HEAVY_MACS];
        r.heavy_macs_fp4 = (int64_t)d[ST_HEAVY_MACS4];
        r.win_groups = (int64_t)d[ST_WIN_GROUPS];
        r.win_macs = (int64_t)d[ST_WIN_MACS];
        r.far_records = (int64_t)d[ST_FAR_RECORDS];
        r.pass_keys = (int64_t)d[ST_PASS_KEYS];
    }
    if (p->farbins.p) {  // far-record chunk claims refused (buffer full: those warps used REDs)
        uint32_t ov[5] = {0, 0, 0, 0, 0};  // (words 193 and 197: the two buffers' counts)
        cudaError_t e = cudaMemcpyAsync(ov, (uint32_t*)p->farbins.p + 193, 20, cudaMemcpyDeviceToHost,
                                        p->last_stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(p->last_stream);
        if (e != cudaSuccess) return p->cuda_fail(e, "stats");
        r.far_overflow = (int64_t)ov[0] + ov[4];
    }
    double* ms[S_NSTAGE] = {&r.ms_encode, &r.ms_sort,     &r.ms_segment, &r.ms_light,
                            &r.ms_heavy,  &r.ms_epilogue, &r.ms_dense,   &r.ms_far};
    for (auto& se : p->evs) {
        float t = 0;
        cudaEventSynchronize(se.second.second);
        if (cudaEventElapsedTime(&t, se.second.first, se.second.second) == cudaSuccess)
            *ms[se.first] += t;
    }
    *out = r;
    return GAKCO_OK;
}

extern "C" gakco_status gakco_zero_upper(gakco_plan* p, int64_t* C, int64_t N, int levels,
                                         void* stream) {
    if (!p || !C || N < 0 || levels < 0) return GAKCO_E_ARG;
    if (!is_device_ptr(C)) return p->fail(GAKCO_E_ARG, "C must be a device pointer");
    DeviceGuard dg(p->device);
    cudaError_t e = launch_zero_upper(C, N, levels, p->sm_count, (cudaStream_t)stream);
    if (e != cudaSuccess) return p->cuda_fail(e, "zero_upper");
    return GAKCO_OK;
}

extern "C" gakco_status gakco_stage_timeline(gakco_plan* p, int32_t* stage, float* t0, float* t1,
                                             int64_t cap, int64_t* count) {
    if (!p || !count || (cap > 0 && (!stage || !t0 || !t1))) return GAKCO_E_ARG;
    DeviceGuard dg(p->device);
    *count = (int64_t)p->evs.size();
    if (p->evs.empty()) return GAKCO_OK;
    const cudaEvent_t ref = p->evs.front().second.first;
    for (size_t i = 0; i < p->evs.size() && (int64_t)i < cap; ++i) {
        const auto& se = p->evs[i];
        cudaEventSynchronize(se.second.second);
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, ref, se.second.first);
        cudaEventElapsedTime(&b, ref, se.second.second);
        stage[i] = se.first;
        t0[i] = a;
        t1[i] = b;
    }
    return GAKCO_OK;
}

// ---------------------------------------------------------------------------
// Mask-sharded multi-GPU step (include/gakco.h)
extern "C" gakco_status gakco_stream_wait_level(gakco_plan* p, int m, void* stream) {
    if (!p) return GAKCO_E_ARG;
    if (m < 0 || m > p->M) return p->fail(GAKCO_E_ARG, "level out of range");
    if (std::find(p->level_order.begin(), p->level_order.end(), m) == p->level_order.end())
        return p->fail(GAKCO_E_ARG, "level not completed by the last gakco_accumulate");
    DeviceGuard dg(p->device);
    for (cudaEvent_t e : p->ev_level[m]) {
        cudaError_t err = cudaStreamWaitEvent((cudaStream_t)stream, e, 0);
        if (err != cudaSuccess) return p->cuda_fail(err, "cudaStreamWaitEvent");
    }
    return GAKCO_OK;
}

extern "C" int gakco_level_order(const gakco_plan* p, int* out, int cap) {
    if (!p) return -1;
    const int n = (int)p->level_order.size();
    for (int i = 0; i < n && i < cap && out; ++i) out[i] = p->level_order[i];
    return n;
}

extern "C" gakco_status gakco_pack_upper(gakco_plan* p, const int64_t* C, int64_t N, int levels,
                                         int64_t begin, int64_t end, void* out, int out_bytes,
                                         void* stream) {
    if (!p) return GAKCO_E_ARG;
    if (N < 1 || N >= ((int64_t)1 << 31) || levels < 1 || levels > GMAX + 1)
        return p->fail(GAKCO_E_ARG, "N or levels out of range");
    const int64_t T = N * (N + 1) / 2;
    if (begin < 0 || end < begin || end > T) return p->fail(GAKCO_E_ARG, "range outside the triangle");
    if (out_bytes != 4 && out_bytes != 8) return p->fail(GAKCO_E_ARG, "out_bytes must be 4 or 8");
    if (!is_device_ptr(C) || (end > begin && !is_device_ptr(out)))
        return p->fail(GAKCO_E_ARG, "C and out must be device pointers");
    DeviceGuard dg(p->device);
    cudaError_t e = launch_pack_upper(C, N, levels, begin, end, out, out_bytes, (cudaStream_t)stream);
    return e == cudaSuccess ? GAKCO_OK : p->cuda_fail(e, "pack_upper");
}

extern "C" gakco_status gakco_diag(gakco_plan* p, const int64_t* C, int64_t N, int levels,
                                   int64_t* out, void* stream) {
    if (!p) return GAKCO_E_ARG;
    if (N < 1 || N >= ((int64_t)1 << 31) || levels < 1 || levels > GMAX + 1)
        return p->fail(GAKCO_E_ARG, "N or levels out of range");
    if (!is_device_ptr(C) || !is_device_ptr(out))
        return p->fail(GAKCO_E_ARG, "C and out must be device pointers");
    DeviceGuard dg(p->device);
    cudaError_t e = launch_diag(C, N, levels, out, p->sm_count, (cudaStream_t)stream);
    return e == cudaSuccess ? GAKCO_OK : p->cuda_fail(e, "diag");
}

static gakco_status finalize_packed_impl(gakco_plan* p, const void* Cp, int in_bytes, int nsrc,
                                         int64_t ld, int64_t N, int64_t begin, int64_t end,
                                         const int64_t* Cdiag, int64_t* Nm, int64_t* K,
                                         double* Knorm, void* stream);

extern "C" gakco_status gakco_finalize_packed(gakco_plan* p, const void* Cp, int in_bytes,
                                              int64_t ld, int64_t N, int64_t begin, int64_t end,
                                              const int64_t* Cdiag, int64_t* Nm, int64_t* K,
                                              double* Knorm, void* stream) {
    return finalize_packed_impl(p, Cp, in_bytes, 1, ld, N, begin, end, Cdiag, Nm, K, Knorm, stream);
}

extern "C" gakco_status gakco_finalize_packed_sum(gakco_plan* p, const void* Cp, int in_bytes,
                                                  int nsrc, int64_t ld, int64_t N, int64_t begin,
                                                  int64_t end, const int64_t* Cdiag, int64_t* Nm,
                                                  int64_t* K, double* Knorm, void* stream) {
    if (!p) return GAKCO_E_ARG;
    if (nsrc < 1 || nsrc > MAX_PEERS) return p->fail(GAKCO_E_ARG, "nsrc must be 1..64");
    return finalize_packed_impl(p, Cp, in_bytes, nsrc, ld, N, begin, end, Cdiag, Nm, K, Knorm, stream);
}

static gakco_status finalize_packed_impl(gakco_plan* p, const void* Cp, int in_bytes, int nsrc,
                                         int64_t ld, int64_t N, int64_t begin, int64_t end,
                                         const int64_t* Cdiag, int64_t* Nm, int64_t* K,
                                         double* Knorm, void* stream) {
    if (!p) return GAKCO_E_ARG;
    if (N < 1 || N >= ((int64_t)1 << 31)) return p->fail(GAKCO_E_ARG, "N out of range");
    const int64_t T = N * (N + 1) / 2;
    if (begin < 0 || end < begin || end > T) return p->fail(GAKCO_E_ARG, "range outside the triangle");
    if (in_bytes != 4 && in_bytes != 8) return p->fail(GAKCO_E_ARG, "in_bytes must be 4 or 8");
    if (ld < end - begin) return p->fail(GAKCO_E_ARG, "ld < end - begin");
    if (!Cdiag || !is_device_ptr(Cdiag) || (end > begin && (!Cp || !is_device_ptr(Cp))))
        return p->fail(GAKCO_E_ARG, "Cp and Cdiag must be device pointers");
    for (const void* o : {(const void*)Nm, (const void*)K, (const void*)Knorm})
        if (o && end > begin && !is_device_ptr(o))
            return p->fail(GAKCO_E_ARG, "outputs must be device pointers");
    DeviceGuard dg(p->device);
    Nvtx nv("gakco_finalize_packed");
    cudaStream_t s = (cudaStream_t)stream;
#define CK(x)                                               \
    do {                                                    \
        cudaError_t e_ = (x);                               \
        if (e_ != cudaSuccess) return p->cuda_fail(e_, #x); \
    } while (0)
    CK(p->ensure(p->kdiag, N * 8, s));
    CK(p->ensure(p->flags, 64, s, /*zero=*/true));
    CK(cudaMemsetAsync(p->flags.p, 0, sizeof(int), s));
    CK(launch_epilogue_packed(Cp, in_bytes, nsrc, ld, Cdiag, N, begin, end, p->g, p->k, p->M, Nm, K, Knorm,
                              (int64_t*)p->kdiag.p, (int*)p->flags.p, s));
    int fl[2] = {0, 0};
    CK(cudaMemcpyAsync(fl, p->flags.p, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemsetAsync((int*)p->flags.p + 1, 0, sizeof(int), s));
    CK(cudaStreamSynchronize(s));
#undef CK
    if (fl[1] & EF_BAD_SYMBOL) return p->fail(GAKCO_E_SYMBOL, "a code is >= sigma");
    if (fl[0] & EF_NEGATIVE_N) return p->fail(GAKCO_E_INTERNAL, "negative N_m after Eq. 9");
    if (fl[0] & EF_K_MISMATCH) return p->fail(GAKCO_E_INTERNAL, "K != C_{g-k}");
    return GAKCO_OK;
}

// ---- fused pack + exchange over peer memory (CUDA IPC) ----
extern "C" gakco_status gakco_ipc_alloc(size_t bytes, int device, void** dev_ptr, void* handle_out) {
    if (!dev_ptr || !handle_out || bytes == 0) return GAKCO_E_ARG;
    DeviceGuard dg(device);
    *dev_ptr = nullptr;
    cudaError_t e = cudaMalloc(dev_ptr, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e == cudaErrorMemoryAllocation ? GAKCO_E_NOMEM : GAKCO_E_CUDA;
    }
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, *dev_ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaFree(*dev_ptr);
        *dev_ptr = nullptr;
        return GAKCO_E_CUDA;
    }
    std::memcpy(handle_out, &h, sizeof h);
    return GAKCO_OK;
}

extern "C" gakco_status gakco_ipc_free(void* dev_ptr) {
    if (!dev_ptr) return GAKCO_E_ARG;
    return cudaFree(dev_ptr) == cudaSuccess ? GAKCO_OK : GAKCO_E_CUDA;
}

extern "C" gakco_status gakco_ipc_handle(const void* dev_ptr, void* handle_out) {
    if (!dev_ptr || !handle_out) return GAKCO_E_ARG;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void*)dev_ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return GAKCO_E_CUDA;
    }
    std::memcpy(handle_out, &h, sizeof h);
    return GAKCO_OK;
}

extern "C" gakco_status gakco_ipc_open(const void* handle, int device, void** dev_ptr) {
    if (!handle || !dev_ptr) return GAKCO_E_ARG;
    DeviceGuard dg(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return GAKCO_E_CUDA;
    }
    return GAKCO_OK;
}

extern "C" gakco_status gakco_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return GAKCO_E_ARG;
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return GAKCO_E_CUDA;
    }
    return GAKCO_OK;
}

extern "C" gakco_status gakco_pack_upper_peers(gakco_plan* p, const int64_t* Cm, int64_t N,
                                               int level, int levels, int64_t chunk,
                                               void* const* dst, int P, int rank, int out_bytes,
                                               void* stream) {
    if (!p) return GAKCO_E_ARG;
    if (N < 1 || N >= ((int64_t)1 << 31) || levels < 1 || level < 0 || level >= levels)
        return p->fail(GAKCO_E_ARG, "N / level out of range");
    if (P < 1 || P > MAX_PEERS || rank < 0 || rank >= P || !dst)
        return p->fail(GAKCO_E_ARG, "P must be 1..64, rank < P, dst given");
    if (out_bytes != 4 && out_bytes != 8) return p->fail(GAKCO_E_ARG, "out_bytes must be 4 or 8");
    if (chunk * P < N * (N + 1) / 2) return p->fail(GAKCO_E_ARG, "chunk * P < N(N+1)/2");
    if (!is_device_ptr(Cm)) return p->fail(GAKCO_E_ARG, "C must be a device pointer");
    PeerPtrs pp{};
    for (int i = 0; i < P; ++i) {
        if (!dst[i]) return p->fail(GAKCO_E_ARG, "a receive buffer is NULL");
        pp.p[i] = dst[i];
    }
    DeviceGuard dg(p->device);
    Nvtx nv("gakco_pack_upper_peers");
    cudaError_t e = launch_pack_upper_peers(Cm, N, level, levels, chunk, pp, rank, out_bytes,
                                            (cudaStream_t)stream);
    return e == cudaSuccess ? GAKCO_OK : p->cuda_fail(e, "pack_upper_peers");
}
