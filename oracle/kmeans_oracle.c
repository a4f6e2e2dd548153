/*
 * kmeans_oracle.c — plain, slow, obviously-correct fp64 CPU oracle for Lloyd's k-means
 * with Minimal Triangle Inequality (MTI) pruning (arXiv 1902.09527, "clusterNOR").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1902_09527_b200/) never links, imports or calls it, and it shares no code,
 * header, table or constant with the CUDA path.
 *
 * Everything is fp64 on fp32 inputs (promoted exactly), direct-difference distances
 * summed over coordinates in ascending order, lowest index on ties.  Reductions run over
 * fixed 64 Ki-row blocks merged in block order, so results do not depend on the OpenMP
 * thread count.
 *
 * Passages followed (PAPER.md line numbers):
 *   Euclidean distance ............ Table "Notation", PAPER.md:987-988 (indices garbled, A16)
 *   drift f(c) = d(c^t, c^{t-1}) .. Table "Notation"
 *   Lloyd's / objective Eq. 1 ..... §4.1, PAPER.md:1104-1130 (SSE reading, A15)
 *   ||Lloyd's merged MM step ...... §3.2, PAPER.md:1000-1011 (per-thread state + reduction)
 *   MTI clauses 1-3 ............... §3.3, PAPER.md:1013-1053 (with Elkan's 1/2, A1-A7)
 *   Elkan TI baseline ............. §2, PAPER.md:876-885 ("triangle inequality (TI) with bounds",
 *                                   O(kn) lower-bound matrix); SPEC.md:265-273 (reading B10)
 * Parity pins: every function is pinned by tests/test_oracle_*.py (hand-checked vectors,
 * closed forms, brute-force optima, scikit-learn).  "dists" (the distance-computation
 * count) is pinned only by the hand-checked B2 trace and 0 <= dists <= n*k: the paper's
 * figures are absent (parity unpinned beyond that).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_BLOCK 65536

/* squared Euclidean distance, fp64, coordinates in ascending order */
static double sqdist(const float *x, const double *c, int d)
{
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
        double t = (double)x[j] - c[j];
        s += t * t;
    }
    return s;
}

static double sqdist_cc(const double *a, const double *b, int d)
{
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
        double t = a[j] - b[j];
        s += t * t;
    }
    return s;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/*
 * Brute-force assignment (Lloyd's assignment step):
 * a[i] = argmin_c ||x_i - C[c]||^2, ties -> lowest c.  Also returns the best and
 * second-best squared distances (d1 <= d2; d2 = +inf when k = 1) for the near-tie set.
 * d1/d2 may be NULL.
 */
void oracle_assign_brute(const float *X, int64_t n, int d, const double *C, int k,
                         int32_t *a, double *d1, double *d2)
{
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; ++i) {
        const float *x = X + i * (int64_t)d;
        double best = INFINITY, second = INFINITY;
        int32_t arg = 0;
        for (int c = 0; c < k; ++c) {
            double q = sqdist(x, C + (int64_t)c * d, d);
            if (q < best) { second = best; best = q; arg = c; }
            else if (q < second) { second = q; }
        }
        a[i] = arg;
        if (d1) d1[i] = best;
        if (d2) d2[i] = second;
    }
}

/*
 * Centroid geometry for MTI (§3.3, PAPER.md:1036-1053 with reading A1/A2):
 * H[c][c'] = 1/2 ||C[c] - C[c']||, s[c] = min_{c' != c} H[c][c'] (k = 1 -> +inf).
 */
void oracle_geometry(const double *C, int k, int d, double *H, double *s)
{
    for (int c = 0; c < k; ++c) {
        double m = INFINITY;
        for (int c2 = 0; c2 < k; ++c2) {
            double h = 0.5 * sqrt(sqdist_cc(C + (int64_t)c * d, C + (int64_t)c2 * d, d));
            H[(int64_t)c * k + c2] = h;
            if (c2 != c && h < m) m = h;
        }
        s[c] = m;
    }
}

/* drift f(c) = d(C_new[c], C_old[c]) (Table "Notation") */
void oracle_drift(const double *Cnew, const double *Cold, int k, int d, double *f)
{
    for (int c = 0; c < k; ++c)
        f[c] = sqrt(sqdist_cc(Cnew + (int64_t)c * d, Cold + (int64_t)c * d, d));
}

/*
 * Per-cluster sums and counts over rows [lo, hi) in fixed 64 Ki-row blocks merged in
 * block order (per-thread state + reduction).
 * sums: k*d fp64 (accumulated into), counts: k int64 (accumulated into).
 */
static void block_sums(const float *X, int64_t lo, int64_t hi, int d, const int32_t *a, int k,
                       double *sums, int64_t *counts)
{
    int64_t nblk = (hi - lo + ORACLE_BLOCK - 1) / ORACLE_BLOCK;
    if (nblk <= 0) return;
    double *ps = (double *)calloc((size_t)nblk * k * d, sizeof(double));
    int64_t *pc = (int64_t *)calloc((size_t)nblk * k, sizeof(int64_t));
    int64_t b;
#pragma omp parallel for schedule(dynamic)
    for (b = 0; b < nblk; ++b) {
        int64_t s0 = lo + b * ORACLE_BLOCK, s1 = s0 + ORACLE_BLOCK;
        if (s1 > hi) s1 = hi;
        double *bs = ps + (size_t)b * k * d;
        int64_t *bc = pc + (size_t)b * k;
        for (int64_t i = s0; i < s1; ++i) {
            int c = a[i];
            const float *x = X + i * (int64_t)d;
            for (int j = 0; j < d; ++j) bs[(int64_t)c * d + j] += (double)x[j];
            bc[c] += 1;
        }
    }
    for (b = 0; b < nblk; ++b) {             /* merge in block order */
        for (int64_t t = 0; t < (int64_t)k * d; ++t) sums[t] += ps[(size_t)b * k * d + t];
        for (int c = 0; c < k; ++c) counts[c] += pc[(size_t)b * k + c];
    }
    free(ps);
    free(pc);
}

/*
 * Sums/counts over the whole data set split into `shards` contiguous row shards
 * (shard r = rows [floor(r n / G), floor((r+1) n / G))), each reduced in its own blocks,
 * then the shard partials added in shard order (the "merge of global state",
 * PAPER.md:1560-1562).  shards = 1 is the unsharded reduction.
 */
void oracle_cluster_sums(const float *X, int64_t n, int d, const int32_t *a, int k, int shards,
                         double *sums, int64_t *counts)
{
    if (shards < 1) shards = 1;
    memset(sums, 0, sizeof(double) * (size_t)k * d);
    memset(counts, 0, sizeof(int64_t) * (size_t)k);
    double *ss = (double *)malloc(sizeof(double) * (size_t)k * d);
    int64_t *sc = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    for (int r = 0; r < shards; ++r) {
        int64_t lo = (int64_t)((__int128)n * r / shards);
        int64_t hi = (int64_t)((__int128)n * (r + 1) / shards);
        memset(ss, 0, sizeof(double) * (size_t)k * d);
        memset(sc, 0, sizeof(int64_t) * (size_t)k);
        block_sums(X, lo, hi, d, a, k, ss, sc);
        for (int64_t t = 0; t < (int64_t)k * d; ++t) sums[t] += ss[t];
        for (int c = 0; c < k; ++c) counts[c] += sc[c];
    }
    free(ss);
    free(sc);
}

/*
 * Centroid update (Lloyd's update step; empty-cluster reading A10):
 * C_new[c] = sums[c] / counts[c] if counts[c] > 0, else C_old[c].  Returns #empty.
 */
int oracle_update(const double *sums, const int64_t *counts, const double *Cold, int k, int d,
                  double *Cnew)
{
    int empty = 0;
    for (int c = 0; c < k; ++c) {
        if (counts[c] > 0) {
            for (int j = 0; j < d; ++j)
                Cnew[(int64_t)c * d + j] = sums[(int64_t)c * d + j] / (double)counts[c];
        } else {
            ++empty;
            for (int j = 0; j < d; ++j) Cnew[(int64_t)c * d + j] = Cold[(int64_t)c * d + j];
        }
    }
    return empty;
}

/* SSE = sum_i ||x_i - C[a_i]||^2 (Eq. 1 read as squared distances, A15), block-ordered */
double oracle_sse(const float *X, int64_t n, int d, const int32_t *a, const double *C)
{
    int64_t nblk = (n + ORACLE_BLOCK - 1) / ORACLE_BLOCK;
    if (nblk <= 0) return 0.0;
    double *ps = (double *)calloc((size_t)nblk, sizeof(double));
    int64_t b;
#pragma omp parallel for schedule(static)
    for (b = 0; b < nblk; ++b) {
        int64_t s0 = b * ORACLE_BLOCK, s1 = s0 + ORACLE_BLOCK;
        if (s1 > n) s1 = n;
        double acc = 0.0;
        for (int64_t i = s0; i < s1; ++i)
            acc += sqdist(X + i * (int64_t)d, C + (int64_t)a[i] * d, d);
        ps[b] = acc;
    }
    double s = 0.0;
    for (b = 0; b < nblk; ++b) s += ps[b];
    free(ps);
    return s;
}

/*
 * One MTI assignment pass, t >= 2 (§3.3; readings A1-A8):
 *   u <- u + f(a)                                   (bound loosened by drift, A3)
 *   clause 1: u <= s(a)          -> keep a, 0 distances
 *   else tighten: u <- d(x, C[a])                   (U(u), one distance, A4/A5)
 *        S = { c' != a : H[a][c'] < u }             (clauses 2/3: skip c' iff H >= u, A6/A7)
 *        a <- argmin over {a} u S of d^2, ties -> lowest index (A8)
 *        u <- sqrt(min d^2);  dists += 1 + |S|
 * C is the centroid set used in this pass; H, s from oracle_geometry(C); f from
 * oracle_drift(C, C_previous_pass).  a, u are updated in place.
 * out3 = {dists, clause1, changed}.
 */
void oracle_mti_pass(const float *X, int64_t n, int d, const double *C, int k,
                     const double *H, const double *s, const double *f,
                     int32_t *a, double *u, int64_t *out3)
{
    int64_t dists = 0, clause1 = 0, changed = 0, i;
#pragma omp parallel for schedule(static) reduction(+ : dists, clause1, changed)
    for (i = 0; i < n; ++i) {
        const float *x = X + i * (int64_t)d;
        int32_t a0 = a[i];
        double ui = u[i] + f[a0];
        if (ui <= s[a0]) {                       /* clause 1 */
            u[i] = ui;
            clause1 += 1;
            continue;
        }
        double qa = sqdist(x, C + (int64_t)a0 * d, d);   /* U(u): tighten */
        ui = sqrt(qa);
        int64_t nd = 1;
        double bestq = qa;
        int32_t best = a0;
        const double *Ha = H + (int64_t)a0 * k;
        for (int c = 0; c < k; ++c) {
            if (c == a0 || !(Ha[c] < ui)) continue;      /* clauses 2/3: pruned */
            double q = sqdist(x, C + (int64_t)c * d, d);
            nd += 1;
            if (q < bestq || (q == bestq && c < best)) { bestq = q; best = c; }
        }
        dists += nd;
        if (best != a0) changed += 1;
        a[i] = best;
        u[i] = sqrt(bestq);
    }
    out3[0] = dists;
    out3[1] = clause1;
    out3[2] = changed;
}

/*
 * Lower bounds for Elkan's TI after a brute-force pass (iteration 1 computes every distance):
 * L[i*k + c] = ||x_i - C[c]|| (fp64, sqrt of the direct-form squared distance).
 */
void oracle_all_dists(const float *X, int64_t n, int d, const double *C, int k, double *L)
{
    int64_t i;
#pragma omp parallel for schedule(static)
    for (i = 0; i < n; ++i)
        for (int c = 0; c < k; ++c)
            L[i * (int64_t)k + c] = sqrt(sqdist(X + i * (int64_t)d, C + (int64_t)c * d, d));
}

/*
 * One pass of Elkan's TI, t >= 2 (the paper's pruning baseline: "triangle inequality (TI) with
 * bounds", a lower-bound matrix of size O(kn); reading B10).
 * Per point, with a0 = a[i]:
 *   l[c] <- max(0, l[c] - f(c)) for every c; u <- u + f(a0)        (bounds loosened by drift)
 *   if u <= s(a0): keep a0, 0 distances                             (Elkan step 2 = MTI clause 1)
 *   else best = a0; for c = 0..k-1 in index order, c != best:
 *     if u > l[c] and u > H[best][c]:                               (Elkan step 3 (i), (ii))
 *       if not yet tightened: u <- d(x, C[a0]); l[a0] <- u; 1 distance  (step 3a, once per pass)
 *       if u > l[c] and u > H[best][c]:                             (step 3b, tightened u)
 *         q <- d(x, C[c])^2; l[c] <- sqrt(q); 1 distance
 *         if q < q_best, or q == q_best and c < best: best <- c, u <- sqrt(q)   (running best)
 *   a <- best.  Comparisons of candidates use squared distances (as brute force), bounds use
 *   distances.  L is n x k row-major; a, u, L are updated in place.  out3 = {dists, clause1, changed}.
 */
void oracle_ti_pass(const float *X, int64_t n, int d, const double *C, int k,
                    const double *H, const double *s, const double *f,
                    int32_t *a, double *u, double *L, int64_t *out3)
{
    int64_t dists = 0, clause1 = 0, changed = 0, i;
#pragma omp parallel for schedule(static) reduction(+ : dists, clause1, changed)
    for (i = 0; i < n; ++i) {
        const float *x = X + i * (int64_t)d;
        double *l = L + i * (int64_t)k;
        for (int c = 0; c < k; ++c) {
            double v = l[c] - f[c];
            l[c] = v > 0.0 ? v : 0.0;
        }
        const int32_t a0 = a[i];
        double ui = u[i] + f[a0];
        if (ui <= s[a0]) {                       /* clause 1 */
            u[i] = ui;
            clause1 += 1;
            continue;
        }
        int32_t best = a0;
        double bestq = INFINITY;
        int tight = 0;
        int64_t nd = 0;
        for (int c = 0; c < k; ++c) {
            if (c == best) continue;
            const double h = H[(int64_t)best * k + c];
            if (!(ui > l[c] && ui > h)) continue;
            if (!tight) {                        /* step 3a: tighten u once */
                bestq = sqdist(x, C + (int64_t)a0 * d, d);
                ui = sqrt(bestq);
                l[a0] = ui;
                tight = 1;
                nd += 1;
                if (!(ui > l[c] && ui > h)) continue;
            }
            double q = sqdist(x, C + (int64_t)c * d, d);
            nd += 1;
            l[c] = sqrt(q);
            if (q < bestq || (q == bestq && c < best)) {
                bestq = q;
                best = c;
                ui = sqrt(q);
            }
        }
        dists += nd;
        if (best != a0) changed += 1;
        a[i] = best;
        u[i] = ui;
    }
    out3[0] = dists;
    out3[1] = clause1;
    out3[2] = changed;
}

/*
 * Full Lloyd's run (§4.1) from C0, brute force (mode 0), MTI (mode 1) or Elkan TI (mode 2).
 *   iteration 1: brute-force assignment (no bounds exist), changed = n, dists = n*k,
 *                u = exact distance to the assigned centroid;
 *   iteration t >= 2: brute force (dists = n*k) or one MTI pass;
 *   update with the empty-cluster reading A10; stop iff changed <= tol or t == max_iters.
 * Outputs: a (n), C (k*d, holds C_T), iterations; per-iteration arrays (length >=
 * max_iters, may be NULL): changed, dists, clause1, empty, sse (sse computed only if
 * sse != NULL; w.r.t. (C_t, a_t)).  shards > 1 uses the sharded reduction.
 * Returns 0 on success, -1 on usage error.
 */
int oracle_lloyd(const float *X, int64_t n, int d, int k, const double *C0, int max_iters,
                 int64_t tol, int mode, int shards, int32_t *a, double *C, int32_t *iterations,
                 int64_t *it_changed, int64_t *it_dists, int64_t *it_clause1, int32_t *it_empty,
                 double *it_sse)
{
    if (n < 1 || d < 1 || k < 1 || k > n || max_iters < 0) return -1;
    size_t kd = (size_t)k * d;
    double *Cprev = (double *)malloc(sizeof(double) * kd);
    double *sums = (double *)malloc(sizeof(double) * kd);
    int64_t *counts = (int64_t *)malloc(sizeof(int64_t) * k);
    double *H = NULL, *s = NULL, *f = NULL, *u = NULL, *d1 = NULL, *L = NULL;
    int32_t *aprev = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    memcpy(C, C0, sizeof(double) * kd);
    memcpy(Cprev, C0, sizeof(double) * kd);
    if (mode == 2) {
        L = (double *)malloc(sizeof(double) * (size_t)n * k);
        if (!L) { free(Cprev); free(sums); free(counts); free(aprev); return -2; }
    }
    if (mode == 1 || mode == 2) {
        H = (double *)malloc(sizeof(double) * (size_t)k * k);
        s = (double *)malloc(sizeof(double) * k);
        f = (double *)malloc(sizeof(double) * k);
        u = (double *)malloc(sizeof(double) * (size_t)n);
        d1 = (double *)malloc(sizeof(double) * (size_t)n);
    }
    int t = 0;
    for (t = 1; t <= max_iters; ++t) {
        int64_t changed, dists, c1 = 0;
        if (t == 1 || mode == 0) {
            memcpy(aprev, a, sizeof(int32_t) * (size_t)(t == 1 ? 0 : n));
            oracle_assign_brute(X, n, d, C, k, a, d1, NULL);
            dists = n * (int64_t)k;
            if (t == 1) {
                changed = n;
            } else {
                changed = 0;
                for (int64_t i = 0; i < n; ++i) changed += (a[i] != aprev[i]);
            }
            if (mode >= 1)
                for (int64_t i = 0; i < n; ++i) u[i] = sqrt(d1[i]);
            if (mode == 2) oracle_all_dists(X, n, d, C, k, L);
        } else {
            int64_t o3[3];
            oracle_geometry(C, k, d, H, s);
            oracle_drift(C, Cprev, k, d, f);
            if (mode == 1) oracle_mti_pass(X, n, d, C, k, H, s, f, a, u, o3);
            else oracle_ti_pass(X, n, d, C, k, H, s, f, a, u, L, o3);
            dists = o3[0];
            c1 = o3[1];
            changed = o3[2];
        }
        /* reduction + update: C_t from a_t; the pass's centroids become Cprev */
        oracle_cluster_sums(X, n, d, a, k, shards, sums, counts);
        memcpy(Cprev, C, sizeof(double) * kd);
        int empty = oracle_update(sums, counts, Cprev, k, d, C);
        if (it_changed) it_changed[t - 1] = changed;
        if (it_dists) it_dists[t - 1] = dists;
        if (it_clause1) it_clause1[t - 1] = c1;
        if (it_empty) it_empty[t - 1] = empty;
        if (it_sse) it_sse[t - 1] = oracle_sse(X, n, d, a, C);
        if (changed <= tol) break;
    }
    if (t > max_iters) t = max_iters;
    *iterations = t;
    free(Cprev); free(sums); free(counts); free(aprev);
    free(H); free(s); free(f); free(u); free(d1); free(L);
    return 0;
}
