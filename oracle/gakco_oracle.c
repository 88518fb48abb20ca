/*
 * gakco_oracle.c — CPU oracle for the gapped k-mer kernel (GaKCo, arXiv 1704.07468).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or execute this code. It shares
 * no code, header, table or helper with the CUDA path (paper_1704_07468_b200/),
 * and neither side includes or links the other.
 *
 * What it computes, written out from the paper's definitions (PAPER.md = P):
 *
 *   N_m(X,Y)  number of ordered g-mer pairs (a in X, b in Y) at Hamming distance
 *             exactly m                                  Definition 1; Eq. 5
 *             (g-mer starts 0..l-g, reading A7; self-pairs a=b counted when X=Y,
 *             reading A2 — see DESIGN.md "Readings")
 *   C_m       = N_m + sum_{j<m} C(g-j, m-j) N_j           Eq. 8, P:130 (index read as j, A1)
 *   K         = sum_{m=0}^{min(M,g-k)} h_m N_m,
 *               h_m = C(g-m, k) if g-m >= k else 0        Eq. 6-7
 *   Knorm     = K(X,Y) / sqrt(K(X,X) K(Y,Y)), 0 if a diagonal is 0,
 *               diagonal exactly 1 where K(X,X) > 0      BASELINE.json; reading A5
 *
 * N_m is obtained WITHOUT masks, keys or sorting: the Hamming histogram of every
 * sequence pair is counted directly. Two routes are provided:
 *   gko_hist_pair_direct  the literal double loop of Eq. 5 (tiny inputs, pins);
 *   gko_hist_pair         the same count, walking each alignment diagonal j-i=d
 *                         and keeping the mismatch count of the g-window as it
 *                         slides (every g-mer pair lies on exactly one diagonal).
 * Tests pin the second to the first, to the paper's Fig. 2 values and to closed
 * forms (tests/test_oracle_pins.py).
 *
 * Integer overflow in Eq. 7/8 is an error (GKO_E_OVERFLOW), never a wraparound.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GKO_OK 0
#define GKO_E_ARG 1
#define GKO_E_OVERFLOW 2
#define GKO_E_NOMEM 3
#define GKO_E_CHECK 4

#define GKO_MAXG 32

/* Binomial coefficient C(n, r) by Pascal's rule; 0 outside 0<=r<=n. */
static int64_t binom(int n, int r) {
    if (r < 0 || n < 0 || r > n) return 0;
    int64_t row[GKO_MAXG + 2];
    for (int i = 0; i <= n; ++i) {
        row[i] = 1;
        for (int j = i - 1; j > 0; --j) row[j] = row[j] + row[j - 1];
    }
    return row[r];
}

int64_t gko_binom(int n, int r) { return binom(n, r); }

/* Eq. 6: h_m = C(g-m, k) if g-m >= k, else 0. */
int64_t gko_h(int g, int k, int m) { return (g - m >= k) ? binom(g - m, k) : 0; }

/* Definition 1 / Eq. 5, literally: every ordered pair of g-mers
 * (start i in x, start j in y), Hamming distance d, hist[d] += 1.
 * hist has g+1 entries and is overwritten. */
int gko_hist_pair_direct(const uint8_t* x, int64_t lx, const uint8_t* y, int64_t ly,
                         int g, int64_t* hist) {
    if (g < 1 || g > GKO_MAXG) return GKO_E_ARG;
    for (int d = 0; d <= g; ++d) hist[d] = 0;
    for (int64_t i = 0; i + g <= lx; ++i)
        for (int64_t j = 0; j + g <= ly; ++j) {
            int d = 0;
            for (int p = 0; p < g; ++p) d += (x[i + p] != y[j + p]);
            hist[d] += 1;
        }
    return GKO_OK;
}

/* The same histogram, diagonal by diagonal. For offset d = j - i the pairs
 * (i, i+d) are consecutive windows over the aligned characters x[i0+t], y[j0+t];
 * w counts mismatches of the current g-window, updated by adding the entering
 * character's mismatch and removing the leaving one's. */
int gko_hist_pair(const uint8_t* x, int64_t lx, const uint8_t* y, int64_t ly,
                  int g, int64_t* hist) {
    if (g < 1 || g > GKO_MAXG) return GKO_E_ARG;
    for (int d = 0; d <= g; ++d) hist[d] = 0;
    int64_t nx = lx - g + 1, ny = ly - g + 1;
    if (nx <= 0 || ny <= 0) return GKO_OK;
    for (int64_t d = -(nx - 1); d <= ny - 1; ++d) {
        int64_t i0 = d < 0 ? -d : 0;
        int64_t j0 = i0 + d;
        int64_t pairs = (nx - i0) < (ny - j0) ? (nx - i0) : (ny - j0);
        int64_t chars = pairs + g - 1;
        const uint8_t* a = x + i0;
        const uint8_t* b = y + j0;
        int w = 0;
        for (int64_t t = 0; t < chars; ++t) {
            w += (a[t] != b[t]);
            if (t >= g) w -= (a[t - g] != b[t - g]);
            if (t >= g - 1) hist[w] += 1;
        }
    }
    return GKO_OK;
}

/* ---------------------------------------------------------------- digests */
/* Order-independent digest of a row-major matrix (test infrastructure):
 * H = sum over entries of mix(idx ^ mix(bits(value))) mod 2^64, idx = X*ncols+Y,
 * mix = the splitmix64 finaliser. Per-row digests are the same sum per row. */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline uint64_t term64(uint64_t idx, uint64_t bits) { return mix64(idx ^ mix64(bits)); }

uint64_t gko_digest_u64(const uint64_t* a, int64_t nrows, int64_t ncols, uint64_t* row_digests) {
    uint64_t h = 0;
    for (int64_t r = 0; r < nrows; ++r) {
        uint64_t hr = 0;
        for (int64_t c = 0; c < ncols; ++c) hr += term64((uint64_t)(r * ncols + c), a[r * ncols + c]);
        if (row_digests) row_digests[r] = hr;
        h += hr;
    }
    return h;
}

/* ---------------------------------------------------------------- Eq. 8 / 7 */
/* Eq. 8: C_m = sum_{j<=m} C(g-j, m-j) N_j   (C(g-m,0)=1 gives the N_m term). */
static int cumulative_entry(const int64_t* n, int g, int m, int64_t* out) {
    int64_t acc = 0;
    for (int j = 0; j <= m; ++j) {
        int64_t t;
        if (__builtin_mul_overflow(binom(g - j, m - j), n[j], &t)) return GKO_E_OVERFLOW;
        if (__builtin_add_overflow(acc, t, &acc)) return GKO_E_OVERFLOW;
    }
    *out = acc;
    return GKO_OK;
}

/* Eq. 7 with Eq. 6 coefficients, summed over m <= min(M, g-k). */
static int kernel_entry(const int64_t* n, int g, int k, int M, int64_t* out) {
    int64_t acc = 0;
    int top = M < g - k ? M : g - k;
    for (int m = 0; m <= top; ++m) {
        int64_t t;
        if (__builtin_mul_overflow(gko_h(g, k, m), n[m], &t)) return GKO_E_OVERFLOW;
        if (__builtin_add_overflow(acc, t, &acc)) return GKO_E_OVERFLOW;
    }
    *out = acc;
    return GKO_OK;
}

/* Normalisation (BASELINE.json; reading A5). */
static double normalize_entry(int64_t kxy, int64_t kxx, int64_t kyy, int diag) {
    if (kxx <= 0 || kyy <= 0) return 0.0;
    if (diag) return 1.0;
    return (double)kxy / sqrt((double)kxx * (double)kyy);
}

int gko_cumulative(const int64_t* Nm, int64_t N, int g, int M, int64_t* C) {
    if (M < 0 || M > g) return GKO_E_ARG;
    int64_t nn = N * N;
    int64_t prof[GKO_MAXG + 1];
    for (int64_t e = 0; e < nn; ++e) {
        for (int m = 0; m <= M; ++m) prof[m] = Nm[(int64_t)m * nn + e];
        for (int m = 0; m <= M; ++m) {
            int rc = cumulative_entry(prof, g, m, &C[(int64_t)m * nn + e]);
            if (rc) return rc;
        }
    }
    return GKO_OK;
}

int gko_kernel(const int64_t* Nm, int64_t N, int g, int k, int M, int64_t* K) {
    if (k < 1 || k > g || M < 0 || M > g) return GKO_E_ARG;
    int64_t nn = N * N;
    int64_t prof[GKO_MAXG + 1];
    for (int64_t e = 0; e < nn; ++e) {
        for (int m = 0; m <= M; ++m) prof[m] = Nm[(int64_t)m * nn + e];
        int rc = kernel_entry(prof, g, k, M, &K[e]);
        if (rc) return rc;
    }
    return GKO_OK;
}

void gko_normalize(const int64_t* K, int64_t N, double* Knorm) {
    for (int64_t x = 0; x < N; ++x)
        for (int64_t y = 0; y < N; ++y)
            Knorm[x * N + y] = normalize_entry(K[x * N + y], K[x * N + x], K[y * N + y], x == y);
}

/* ---------------------------------------------------------------- all pairs */
typedef struct {
    const uint8_t* codes;
    const int64_t* offsets;
    int64_t N;
    int g, k, M;
    /* dense mode */
    int64_t* Nm;
    /* streaming-digest mode */
    const int64_t* kdiag;      /* K(X,X), precomputed */
    int64_t row_begin, row_end;
    uint64_t* mat_dig;         /* per thread: [nmat] */
    uint64_t* row_dig;         /* per thread: [nmat][N] */
    int nmat;
    /* pair-list mode */
    const int64_t* px;
    const int64_t* py;
    int64_t* pout;
    int64_t npairs;
    /* shared */
    int64_t next;              /* atomic work counter */
    int err;
} job_t;

typedef struct { job_t* job; int tid; } worker_t;

static int pair_hist(const job_t* j, int64_t x, int64_t y, int64_t* hist) {
    const uint8_t* a = j->codes + j->offsets[x];
    const uint8_t* b = j->codes + j->offsets[y];
    int64_t la = j->offsets[x + 1] - j->offsets[x];
    int64_t lb = j->offsets[y + 1] - j->offsets[y];
    int rc = gko_hist_pair(a, la, b, lb, j->g, hist);
    if (rc) return rc;
    /* check: sum of the full histogram = n_X * n_Y */
    int64_t na = la - j->g + 1, nb = lb - j->g + 1, s = 0;
    if (na < 0) na = 0;
    if (nb < 0) nb = 0;
    for (int d = 0; d <= j->g; ++d) s += hist[d];
    return s == na * nb ? GKO_OK : GKO_E_CHECK;
}

static void* dense_worker(void* arg) {
    worker_t* w = (worker_t*)arg;
    job_t* j = w->job;
    int64_t hist[GKO_MAXG + 1];
    int64_t nn = j->N * j->N;
    for (;;) {
        int64_t x = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (x >= j->N) break;
        for (int64_t y = x; y < j->N; ++y) {
            int rc = pair_hist(j, x, y, hist);
            if (rc) { __atomic_store_n(&j->err, rc, __ATOMIC_RELAXED); return NULL; }
            for (int m = 0; m <= j->M; ++m) {
                j->Nm[(int64_t)m * nn + x * j->N + y] = hist[m];
                j->Nm[(int64_t)m * nn + y * j->N + x] = hist[m];
            }
        }
    }
    return NULL;
}

static int run_threads(job_t* j, int nthreads, void* (*fn)(void*)) {
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    worker_t* ws = (worker_t*)calloc((size_t)nthreads, sizeof(worker_t));
    if (!th || !ws) { free(th); free(ws); return GKO_E_NOMEM; }
    for (int t = 0; t < nthreads; ++t) {
        ws[t].job = j; ws[t].tid = t;
        pthread_create(&th[t], NULL, fn, &ws[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th); free(ws);
    return j->err;
}

/* N_m for every ordered sequence pair, m = 0..M: Nm[m][X][Y] (full, symmetric). */
int gko_profiles(const uint8_t* codes, const int64_t* offsets, int64_t N, int g, int M,
                 int nthreads, int64_t* Nm) {
    if (N < 1 || g < 1 || g > GKO_MAXG || M < 0 || M > g) return GKO_E_ARG;
    job_t j;
    memset(&j, 0, sizeof j);
    j.codes = codes; j.offsets = offsets; j.N = N; j.g = g; j.M = M; j.Nm = Nm;
    return run_threads(&j, nthreads, dense_worker);
}

/* Histograms of a list of pairs (X_i, Y_i): out[i][0..M] = N_m(X_i, Y_i). */
static void* pairs_worker(void* arg) {
    worker_t* w = (worker_t*)arg;
    job_t* j = w->job;
    int64_t hist[GKO_MAXG + 1];
    for (;;) {
        int64_t i = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (i >= j->npairs) break;
        int rc = pair_hist(j, j->px[i], j->py[i], hist);
        if (rc) { __atomic_store_n(&j->err, rc, __ATOMIC_RELAXED); return NULL; }
        for (int m = 0; m <= j->M; ++m) j->pout[i * (j->M + 1) + m] = hist[m];
    }
    return NULL;
}

int gko_pairs(const uint8_t* codes, const int64_t* offsets, int64_t N, int g, int M,
              const int64_t* X, const int64_t* Y, int64_t npairs, int nthreads, int64_t* out) {
    if (N < 1 || g < 1 || g > GKO_MAXG || M < 0 || M > g) return GKO_E_ARG;
    for (int64_t i = 0; i < npairs; ++i)
        if (X[i] < 0 || X[i] >= N || Y[i] < 0 || Y[i] >= N) return GKO_E_ARG;
    job_t j;
    memset(&j, 0, sizeof j);
    j.codes = codes; j.offsets = offsets; j.N = N; j.g = g; j.M = M;
    j.px = X; j.py = Y; j.pout = out; j.npairs = npairs;
    return run_threads(&j, nthreads, pairs_worker);
}

/* Streaming digests for corpora whose matrices do not fit in memory.
 * Matrices, in order: C_0..C_M, N_0..N_M, K, Knorm  (nmat = 2(M+1)+2).
 * For rows X in [row_begin,row_end) and every Y >= X the pair histogram is
 * counted once and the entry terms of (X,Y) and (Y,X) are added to the digests
 * (the digest is a sum, so order does not matter). mat_dig[nmat] and
 * row_dig[nmat][N] are outputs (row digests are complete only when the row range
 * covers every row, because row Y also receives terms from rows X < Y). */
static void* digest_worker(void* arg) {
    worker_t* w = (worker_t*)arg;
    job_t* j = w->job;
    int64_t hist[GKO_MAXG + 1], cm[GKO_MAXG + 1];
    uint64_t* md = j->mat_dig + (int64_t)w->tid * j->nmat;
    uint64_t* rd = j->row_dig + (int64_t)w->tid * j->nmat * j->N;
    const int64_t N = j->N;
    const int M = j->M;
    for (;;) {
        int64_t x = j->row_begin + __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (x >= j->row_end) break;
        for (int64_t y = x; y < N; ++y) {
            int rc = pair_hist(j, x, y, hist);
            if (rc) { __atomic_store_n(&j->err, rc, __ATOMIC_RELAXED); return NULL; }
            int64_t kxy;
            for (int m = 0; m <= M; ++m) {
                rc = cumulative_entry(hist, j->g, m, &cm[m]);
                if (rc) { __atomic_store_n(&j->err, rc, __ATOMIC_RELAXED); return NULL; }
            }
            rc = kernel_entry(hist, j->g, j->k, M, &kxy);
            if (rc) { __atomic_store_n(&j->err, rc, __ATOMIC_RELAXED); return NULL; }
            double kn = normalize_entry(kxy, j->kdiag[x], j->kdiag[y], x == y);
            uint64_t knb;
            memcpy(&knb, &kn, 8);
            for (int side = 0; side < (x == y ? 1 : 2); ++side) {
                int64_t r = side ? y : x, c = side ? x : y;
                uint64_t idx = (uint64_t)(r * N + c);
                int mi = 0;
                for (int m = 0; m <= M; ++m, ++mi) {
                    uint64_t t = term64(idx, (uint64_t)cm[m]);
                    md[mi] += t; rd[(int64_t)mi * N + r] += t;
                }
                for (int m = 0; m <= M; ++m, ++mi) {
                    uint64_t t = term64(idx, (uint64_t)hist[m]);
                    md[mi] += t; rd[(int64_t)mi * N + r] += t;
                }
                uint64_t t = term64(idx, (uint64_t)kxy);
                md[mi] += t; rd[(int64_t)mi * N + r] += t; ++mi;
                t = term64(idx, knb);
                md[mi] += t; rd[(int64_t)mi * N + r] += t;
            }
        }
    }
    return NULL;
}

int gko_digests(const uint8_t* codes, const int64_t* offsets, int64_t N, int g, int k, int M,
                int nthreads, int64_t row_begin, int64_t row_end,
                uint64_t* mat_dig, uint64_t* row_dig) {
    if (N < 1 || g < 1 || g > GKO_MAXG || k < 1 || k > g || M < 0 || M > g) return GKO_E_ARG;
    if (row_begin < 0 || row_end > N || row_begin > row_end) return GKO_E_ARG;
    if (nthreads < 1) nthreads = 1;
    int nmat = 2 * (M + 1) + 2;
    int64_t* kdiag = (int64_t*)malloc((size_t)N * sizeof(int64_t));
    uint64_t* md = (uint64_t*)calloc((size_t)nthreads * nmat, sizeof(uint64_t));
    uint64_t* rd = (uint64_t*)calloc((size_t)nthreads * nmat * N, sizeof(uint64_t));
    if (!kdiag || !md || !rd) { free(kdiag); free(md); free(rd); return GKO_E_NOMEM; }
    job_t j;
    memset(&j, 0, sizeof j);
    j.codes = codes; j.offsets = offsets; j.N = N; j.g = g; j.k = k; j.M = M;
    /* K(X,X) for the normalisation */
    {
        int64_t hist[GKO_MAXG + 1];
        for (int64_t x = 0; x < N; ++x) {
            int rc = pair_hist(&j, x, x, hist);
            if (!rc) rc = kernel_entry(hist, g, k, M, &kdiag[x]);
            if (rc) { free(kdiag); free(md); free(rd); return rc; }
        }
    }
    j.kdiag = kdiag; j.row_begin = row_begin; j.row_end = row_end;
    j.mat_dig = md; j.row_dig = rd; j.nmat = nmat;
    int rc = run_threads(&j, nthreads, digest_worker);
    if (!rc) {
        for (int mi = 0; mi < nmat; ++mi) {
            uint64_t s = 0;
            for (int t = 0; t < nthreads; ++t) s += md[(int64_t)t * nmat + mi];
            mat_dig[mi] = s;
            if (row_dig)
                for (int64_t r = 0; r < N; ++r) {
                    uint64_t sr = 0;
                    for (int t = 0; t < nthreads; ++t) sr += rd[((int64_t)t * nmat + mi) * N + r];
                    row_dig[(int64_t)mi * N + r] = sr;
                }
        }
    }
    free(kdiag); free(md); free(rd);
    return rc;
}
