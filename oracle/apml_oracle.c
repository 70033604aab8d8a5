/*
 * apml_oracle.c -- plain, slow, obviously-correct CPU oracle for APML / CUDA-APML.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2512_19743_b200/) never links, imports or calls anything under oracle/,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * Everything is fp64 on the caller's fp32 inputs.  Each step cites the passage of
 * /root/reference/PAPER.md (P:<line>, section / equation / algorithm) it follows.
 * Where the paper is silent we take the reading listed in DESIGN.md "Readings"
 * (R1..R16, the same numbering as SURVEY.md section 8(c)).
 *
 * Two variants:
 *   dense  : section III-A literally -- materialised C, P_row, P_col, P, dense
 *            Sinkhorn.  tau is ignored (every similarity kept).
 *   sparse : Algorithm 1 -- per-direction line scans that keep s >= tau
 *            (P:90), per-support normalisation, concatenate + 64-bit key sort +
 *            duplicate merge, COO Sinkhorn Eqs. (3)-(4),
 *            COO loss.  Memory O(N + M + nnz) per pair: lines are
 *            recomputed on the fly, no N x M buffer.
 * Backward: hand-written reverse pass of the sparse pipeline, "full"
 * (through softmax incl. T, symmetrisation and Sinkhorn) or "plan-detached"
 * (Eq. (5) only).  Discrete choices (argmin, second argmin, support) are frozen.
 *
 * parity pins: see tests/test_oracle_pins.py and DESIGN.md section "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    double p_min;    /* Eq. (1), 0 < p_min < 1; default 0.9 (R2) */
    double tau;      /* pruning threshold on UNNORMALISED similarity, keep s >= tau (R7) */
    double eps_stab; /* Sinkhorn stability constant */
    double delta;    /* g = c~(2) + delta (R3) */
    double eps_g;    /* gap clamp max(gap, eps_g) / fallback test */
    double eps_dist; /* Eq. (5) denominator */
    int32_t l_iter;  /* Sinkhorn iterations */
    int32_t stability; /* 0 = gap clamp (sparse default), 1 = uniform fallback */
    int32_t grad_mode; /* 0 = full (R11), 1 = plan-detached (Eq. (5) only) */
    int32_t row_first; /* 0 = column-then-row per iteration (Eqs. (3)-(4));
                          1 = row-then-column (test-only variant used by the swap identity pin) */
} oracle_cfg;

enum { FLAG_ROW = 1, FLAG_COL = 2 };

/* ---------------------------------------------------------------- helpers */

/* C_ij = ||x_i - y_j||_2, Euclidean, not squared (R1). */
static double cost(const double* x, const double* y) {
    double dx = x[0] - y[0];
    double dy = x[1] - y[1];
    double dz = x[2] - y[2];
    return sqrt(dx * dx + dy * dy + dz * dz);
}

static double* widen(const float* a, int64_t n) {
    double* r = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    for (int64_t k = 0; k < n; ++k) r[k] = (double)a[k];
    return r;
}

/* Eq. (1): T = -log((1 - p_min) / ((K - 1) p_min)) / g, K > 1. */
double oracle_temperature(double g, int64_t K, double p_min) {
    return -log((1.0 - p_min) / ((double)(K - 1) * p_min)) / g;
}

/* Line statistics: minimum, second smallest of the MULTISET (a duplicated
 * minimum gives c~(2) = 0, R5), argmin = lowest index, second argmin = lowest index
 * other than the argmin among the second-smallest values (R12). */
static void line_min2(const double* c, int64_t K, double* m, double* c2, int64_t* a, int64_t* b) {
    int64_t ia = 0;
    for (int64_t k = 1; k < K; ++k)
        if (c[k] < c[ia]) ia = k;
    int64_t ib = -1;
    for (int64_t k = 0; k < K; ++k) {
        if (k == ia) continue;
        if (ib < 0 || c[k] < c[ib]) ib = k;
    }
    *m = c[ia];
    *a = ia;
    *b = ib;
    *c2 = (ib >= 0) ? c[ib] : INFINITY;
}

/* Per-line result of the directional adaptive softmax (Eq. (2)). */
typedef struct {
    double m, c2, g, T;
    int64_t a, b;      /* argmin / second argmin index inside the line */
    int32_t clamped;   /* gap clamp active -> no gradient through g */
    int32_t uniform;   /* uniform fallback written */
    int32_t k1;        /* K == 1 line: P = 1 on its single entry (R4) */
    int64_t kept;      /* |Omega_line| */
} line_info;

/* Directional adaptive softmax on one line of costs c[0..K).
 * Appends kept (index, P) pairs to out_idx/out_p (capacity K) and returns the count. */
static int64_t line_softmax(const double* c, int64_t K, const oracle_cfg* cfg, line_info* li,
                            int64_t* out_idx, double* out_p, double* s_scratch) {
    memset(li, 0, sizeof(*li));
    if (K == 1) { /* Eq. (1) requires K > 1; a single-entry line carries P = 1 (R4). */
        li->m = c[0]; li->c2 = INFINITY; li->a = 0; li->b = -1; li->k1 = 1; li->kept = 1;
        out_idx[0] = 0; out_p[0] = 1.0;
        return 1;
    }
    line_min2(c, K, &li->m, &li->c2, &li->a, &li->b);
    double gap = li->c2 - li->m;             /* c~(2): second smallest of c~ = c - min c */
    if (cfg->stability == 1 && gap < cfg->eps_g) {
        /* uniform fallback; the sparse kernel "writes a uniform distribution over the
           corresponding row or column": all K entries, P = 1/K. */
        li->uniform = 1; li->g = gap + cfg->delta; li->T = 0.0; li->kept = K;
        for (int64_t k = 0; k < K; ++k) { out_idx[k] = k; out_p[k] = 1.0 / (double)K; }
        return K;
    }
    double g = gap + cfg->delta;             /* g = c~(2) + delta */
    if (cfg->stability == 0 && g < cfg->eps_g) { g = cfg->eps_g; li->clamped = 1; }
    li->g = g;
    li->T = oracle_temperature(g, K, cfg->p_min);              /* Eq. (1) */
    double Z = 0.0;
    int64_t n = 0;
    for (int64_t k = 0; k < K; ++k) {
        double s = exp(-li->T * (c[k] - li->m));                /* s = exp(-T (C - C_min)) */
        s_scratch[k] = s;
        if (s >= cfg->tau) { out_idx[n] = k; n++; Z += s; }     /* Omega: s >= tau */
    }
    for (int64_t q = 0; q < n; ++q) out_p[q] = s_scratch[out_idx[q]] / Z; /* normalise by kept sum */
    li->kept = n;
    return n;
}

/* ---------------------------------------------------------------- sparse plan */

typedef struct {
    uint64_t key;   /* i*M + j */
    int32_t dir;    /* FLAG_ROW or FLAG_COL */
    double p;       /* P_row or P_col value */
} coo_raw;

static int cmp_raw(const void* A, const void* B) {
    const coo_raw* a = (const coo_raw*)A;
    const coo_raw* b = (const coo_raw*)B;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->dir - b->dir; /* row stream first: deterministic */
}

typedef struct oracle_plan {
    int64_t N, M;
    oracle_cfg cfg;
    double* x; double* y;      /* copies of the inputs (fp32 widened exactly, or fp64) */
    int64_t nnz;
    int64_t* ti; int64_t* tj;  /* support in key order (row-major) */
    int32_t* flags;            /* FLAG_ROW | FLAG_COL */
    double* prow; double* pcol;/* directional probabilities on the support (0 where absent) */
    double* c;                 /* ||x_i - y_j|| on the support */
    double* vhist;             /* (2 L + 1) x nnz: v after each half-step; row 0 = P0 */
    double loss;
    line_info* rows; line_info* cols;
} oracle_plan;

void oracle_plan_free(oracle_plan* P) {
    if (!P) return;
    free(P->x); free(P->y); free(P->ti); free(P->tj); free(P->flags);
    free(P->prow); free(P->pcol); free(P->c); free(P->vhist); free(P->rows); free(P->cols);
    free(P);
}

/* Sinkhorn half-step on the COO support (Eqs. (3)/(4)): v_t /= (sum over the
 * segment of v + eps_stab).  by_col = 1 sums over t' with j_t' = j_t (Eq. (3)), else over
 * i_t' = i_t (Eq. (4)).  Sums run in key order (fixed left-to-right, deterministic). */
static void sinkhorn_half(const oracle_plan* P, const double* w, double* u, int by_col) {
    int64_t L = by_col ? P->M : P->N;
    double* S = (double*)calloc((size_t)L, sizeof(double));
    for (int64_t t = 0; t < P->nnz; ++t) S[by_col ? P->tj[t] : P->ti[t]] += w[t];
    for (int64_t t = 0; t < P->nnz; ++t) u[t] = w[t] / (S[by_col ? P->tj[t] : P->ti[t]] + P->cfg.eps_stab);
    free(S);
}

/* fp64-input entry point (finite-difference tests perturb coordinates below fp32 ulp). */
oracle_plan* oracle_sparse_forward64(const double* x, const double* y, int64_t N, int64_t M,
                                     const oracle_cfg* cfg) {
    if (N < 1 || M < 1 || !cfg) return NULL;
    oracle_plan* P = (oracle_plan*)calloc(1, sizeof(oracle_plan));
    P->N = N; P->M = M; P->cfg = *cfg;
    P->x = (double*)malloc(sizeof(double) * 3 * N); memcpy(P->x, x, sizeof(double) * 3 * N);
    P->y = (double*)malloc(sizeof(double) * 3 * M); memcpy(P->y, y, sizeof(double) * 3 * M);
    x = P->x; y = P->y;
    P->rows = (line_info*)calloc((size_t)N, sizeof(line_info));
    P->cols = (line_info*)calloc((size_t)M, sizeof(line_info));

    int64_t K = N > M ? N : M;
    double* line = (double*)malloc(sizeof(double) * K);
    double* scratch = (double*)malloc(sizeof(double) * K);
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * K);
    double* pv = (double*)malloc(sizeof(double) * K);
    int64_t cap = 16, n = 0;
    coo_raw* raw = (coo_raw*)malloc(sizeof(coo_raw) * cap);

    /* Algorithm 1 line 1: row direction -- scan each row, minima, temperature,
       keep s >= tau, normalise. */
    for (int64_t i = 0; i < N; ++i) {
        for (int64_t j = 0; j < M; ++j) line[j] = cost(x + 3 * i, y + 3 * j);
        int64_t k = line_softmax(line, M, cfg, &P->rows[i], idx, pv, scratch);
        for (int64_t q = 0; q < k; ++q) {
            if (n == cap) { cap *= 2; raw = (coo_raw*)realloc(raw, sizeof(coo_raw) * cap); }
            raw[n].key = (uint64_t)i * (uint64_t)M + (uint64_t)idx[q]; raw[n].dir = FLAG_ROW; raw[n].p = pv[q]; n++;
        }
    }
    /* Algorithm 1 line 2: column direction with swapped roles. */
    for (int64_t j = 0; j < M; ++j) {
        for (int64_t i = 0; i < N; ++i) line[i] = cost(x + 3 * i, y + 3 * j);
        int64_t k = line_softmax(line, N, cfg, &P->cols[j], idx, pv, scratch);
        for (int64_t q = 0; q < k; ++q) {
            if (n == cap) { cap *= 2; raw = (coo_raw*)realloc(raw, sizeof(coo_raw) * cap); }
            raw[n].key = (uint64_t)idx[q] * (uint64_t)M + (uint64_t)j; raw[n].dir = FLAG_COL; raw[n].p = pv[q]; n++;
        }
    }
    free(line); free(scratch); free(idx); free(pv);

    /* Algorithm 1 line 3: concatenate, sort by 64-bit key, merge duplicates.
       P0 = (P_row + P_col)/2 with a missing direction counting as 0 (reading R8). */
    qsort(raw, (size_t)n, sizeof(coo_raw), cmp_raw);
    int64_t nnz = 0;
    for (int64_t t = 0; t < n; ++t)
        if (t == 0 || raw[t].key != raw[t - 1].key) nnz++;
    P->nnz = nnz;
    P->ti = (int64_t*)malloc(sizeof(int64_t) * (nnz ? nnz : 1));
    P->tj = (int64_t*)malloc(sizeof(int64_t) * (nnz ? nnz : 1));
    P->flags = (int32_t*)calloc((size_t)(nnz ? nnz : 1), sizeof(int32_t));
    P->prow = (double*)calloc((size_t)(nnz ? nnz : 1), sizeof(double));
    P->pcol = (double*)calloc((size_t)(nnz ? nnz : 1), sizeof(double));
    P->c = (double*)malloc(sizeof(double) * (nnz ? nnz : 1));
    int32_t L = cfg->l_iter;
    P->vhist = (double*)malloc(sizeof(double) * (size_t)(2 * L + 1) * (size_t)(nnz ? nnz : 1));
    int64_t t = -1;
    for (int64_t r = 0; r < n; ++r) {
        if (r == 0 || raw[r].key != raw[r - 1].key) {
            t++;
            P->ti[t] = (int64_t)(raw[r].key / (uint64_t)M);
            P->tj[t] = (int64_t)(raw[r].key % (uint64_t)M);
        }
        P->flags[t] |= raw[r].dir;
        if (raw[r].dir == FLAG_ROW) P->prow[t] = raw[r].p; else P->pcol[t] = raw[r].p;
    }
    free(raw);
    double* v = P->vhist;
    for (t = 0; t < nnz; ++t) {
        v[t] = 0.5 * (P->prow[t] + P->pcol[t]);                       /* P0 (R8) */
        P->c[t] = cost(x + 3 * P->ti[t], y + 3 * P->tj[t]);           /* distances on stored pairs */
    }

    /* Algorithm 1 lines 4-7: L_iter x {column scaling Eq. (3), row scaling Eq. (4)}. */
    for (int32_t l = 0; l < L; ++l) {
        double* w0 = P->vhist + (size_t)(2 * l) * nnz;
        double* w1 = w0 + nnz;
        double* w2 = w1 + nnz;
        sinkhorn_half(P, w0, w1, cfg->row_first ? 0 : 1);
        sinkhorn_half(P, w1, w2, cfg->row_first ? 1 : 0);
    }
    /* Loss on the COO support: sum_t v_t ||x_i - y_j||. */
    const double* vf = P->vhist + (size_t)(2 * L) * nnz;
    double loss = 0.0;
    for (t = 0; t < nnz; ++t) loss += vf[t] * P->c[t];
    P->loss = loss;
    return P;
}

/* fp32-input entry point: the exact bytes the GPU path sees, widened exactly to fp64. */
oracle_plan* oracle_sparse_forward(const float* x, const float* y, int64_t N, int64_t M,
                                   const oracle_cfg* cfg) {
    if (N < 1 || M < 1 || !cfg) return NULL;
    double* xd = widen(x, 3 * N);
    double* yd = widen(y, 3 * M);
    oracle_plan* P = oracle_sparse_forward64(xd, yd, N, M, cfg);
    free(xd); free(yd);
    return P;
}

double oracle_plan_loss(const oracle_plan* P) { return P->loss; }
int64_t oracle_plan_nnz(const oracle_plan* P) { return P->nnz; }

/* Support in key order; v = final plan after L_iter Sinkhorn iterations. Any pointer may be NULL. */
void oracle_plan_support(const oracle_plan* P, int64_t* i, int64_t* j, int32_t* flags, double* p0,
                         double* v, double* c, double* prow, double* pcol) {
    const double* vf = P->vhist + (size_t)(2 * P->cfg.l_iter) * P->nnz;
    for (int64_t t = 0; t < P->nnz; ++t) {
        if (i) i[t] = P->ti[t];
        if (j) j[t] = P->tj[t];
        if (flags) flags[t] = P->flags[t];
        if (p0) p0[t] = P->vhist[t];
        if (v) v[t] = vf[t];
        if (c) c[t] = P->c[t];
        if (prow) prow[t] = P->prow[t];
        if (pcol) pcol[t] = P->pcol[t];
    }
}

/* Per-line statistics: dir 0 = rows (length N), 1 = columns (length M).
 * ints: [a, b, clamped, uniform, k1, kept] per line; dbl: [m, c2, g, T] per line. */
void oracle_plan_lines(const oracle_plan* P, int32_t dir, int64_t* ints, double* dbl) {
    int64_t L = dir ? P->M : P->N;
    const line_info* li = dir ? P->cols : P->rows;
    for (int64_t k = 0; k < L; ++k) {
        ints[6 * k + 0] = li[k].a; ints[6 * k + 1] = li[k].b; ints[6 * k + 2] = li[k].clamped;
        ints[6 * k + 3] = li[k].uniform; ints[6 * k + 4] = li[k].k1; ints[6 * k + 5] = li[k].kept;
        dbl[4 * k + 0] = li[k].m; dbl[4 * k + 1] = li[k].c2; dbl[4 * k + 2] = li[k].g; dbl[4 * k + 3] = li[k].T;
    }
}

/* One line of Algorithm 1 on its own (P:161 rows / P:162 columns): the costs of point
 * `own` against the K points of `other` (fp32 widened exactly), then the directional
 * adaptive softmax of that line (Eq. (1)) -- the same line_softmax the
 * sparse plan runs.  For sampled-line checks at sizes where the whole oracle is too slow
 * (C5).  ints[6] = a, b, clamped, uniform, k1, kept; dbl[4] = m, c2, g, T; idx / p (capacity
 * K) receive the kept indices and P values in index order.  Returns the kept count. */
int64_t oracle_line(const float* own, const float* other, int64_t K, const oracle_cfg* cfg,
                    int64_t* ints, double* dbl, int64_t* idx, double* p) {
    if (K < 1 || !cfg) return -1;
    double o[3] = {(double)own[0], (double)own[1], (double)own[2]};
    double* line = (double*)malloc(sizeof(double) * K);
    double* scratch = (double*)malloc(sizeof(double) * K);
    for (int64_t k = 0; k < K; ++k) {
        double q[3] = {(double)other[3 * k], (double)other[3 * k + 1], (double)other[3 * k + 2]};
        line[k] = cost(o, q);
    }
    line_info li;
    int64_t n = line_softmax(line, K, cfg, &li, idx, p, scratch);
    ints[0] = li.a; ints[1] = li.b; ints[2] = li.clamped; ints[3] = li.uniform; ints[4] = li.k1; ints[5] = li.kept;
    dbl[0] = li.m; dbl[1] = li.c2; dbl[2] = li.g; dbl[3] = li.T;
    free(line); free(scratch);
    return n;
}

/* ---------------------------------------------------------------- backward */

/* Reverse of u = w / (S_seg + eps) (Eqs. (3)/(4)): wbar_t = (ubar_t - sum_seg ubar*u) / (S_seg + eps). */
static void sinkhorn_half_rev(const oracle_plan* P, const double* w, const double* u,
                              const double* ubar, double* wbar, int by_col) {
    int64_t L = by_col ? P->M : P->N;
    double* S = (double*)calloc((size_t)L, sizeof(double));
    double* D = (double*)calloc((size_t)L, sizeof(double));
    for (int64_t t = 0; t < P->nnz; ++t) {
        int64_t k = by_col ? P->tj[t] : P->ti[t];
        S[k] += w[t];
        D[k] += ubar[t] * u[t];
    }
    for (int64_t t = 0; t < P->nnz; ++t) {
        int64_t k = by_col ? P->tj[t] : P->ti[t];
        wbar[t] = (ubar[t] - D[k]) / (S[k] + P->cfg.eps_stab);
    }
    free(S); free(D);
}

/* Accumulate dL/dc for a pair (i, j) into gx (and gy) through Eq. (5):
 * d||x - y|| / dx = (x - y) / (||x - y|| + eps_dist); d/dy is its negative. */
static void eq5(const oracle_plan* P, int64_t i, int64_t j, double cbar, double* gx, double* gy) {
    const double* xi = P->x + 3 * i;
    const double* yj = P->y + 3 * j;
    double c = cost(xi, yj);
    double den = c + P->cfg.eps_dist;
    for (int d = 0; d < 3; ++d) {
        double g = cbar * (xi[d] - yj[d]) / den;
        if (gx) gx[3 * i + d] += g;
        if (gy) gy[3 * j + d] -= g;
    }
}

/* Position of (i, j) in the key-sorted support, or -1 (binary search on key = i*M + j). */
static int64_t find_entry(const oracle_plan* P, int64_t i, int64_t j) {
    uint64_t key = (uint64_t)i * (uint64_t)P->M + (uint64_t)j;
    int64_t lo = 0, hi = P->nnz - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        uint64_t km = (uint64_t)P->ti[mid] * (uint64_t)P->M + (uint64_t)P->tj[mid];
        if (km == key) return mid;
        if (km < key) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* Reverse of one direction's adaptive softmax (Eq. (2), Eq. (1)).
 * Per line: P = s / Z over the kept set, s = exp(z), z = -T (c - m), T = Lambda / g,
 * g = c2 - m + delta.  Given Pbar on the kept entries:
 *   zbar = P (Pbar - sum P Pbar);  cbar_t += -T zbar_t;  mbar = T sum zbar;
 *   Tbar = -sum zbar (c - m);  gbar = -Tbar T / g (0 if clamped);
 *   cbar[argmin] += mbar - gbar;  cbar[second argmin] += gbar.
 * Contributions to pairs outside the support (second argmin pruned, R14) go straight
 * through Eq. (5). */
static void softmax_rev(const oracle_plan* P, int dir, const double* pbar_dir, double* cbar,
                        double* gx, double* gy) {
    int64_t nl = dir ? P->M : P->N;
    /* line -> list of support positions carrying this direction's flag, in key order */
    int64_t* cnt = (int64_t*)calloc((size_t)nl + 1, sizeof(int64_t));
    int32_t f = dir ? FLAG_COL : FLAG_ROW;
    for (int64_t t = 0; t < P->nnz; ++t)
        if (P->flags[t] & f) cnt[(dir ? P->tj[t] : P->ti[t]) + 1]++;
    for (int64_t k = 0; k < nl; ++k) cnt[k + 1] += cnt[k];
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cnt[nl] ? cnt[nl] : 1));
    int64_t* fill = (int64_t*)calloc((size_t)nl, sizeof(int64_t));
    for (int64_t t = 0; t < P->nnz; ++t)
        if (P->flags[t] & f) { int64_t k = dir ? P->tj[t] : P->ti[t]; pos[cnt[k] + fill[k]++] = t; }
    const double* pdir = dir ? P->pcol : P->prow;
    const line_info* lines = dir ? P->cols : P->rows;
    for (int64_t k = 0; k < nl; ++k) {
        const line_info* li = &lines[k];
        if (li->k1 || li->uniform) continue; /* constant P: no gradient */
        double sPP = 0.0;
        for (int64_t q = cnt[k]; q < cnt[k + 1]; ++q) { int64_t t = pos[q]; sPP += pdir[t] * pbar_dir[t]; }
        double szb = 0.0, Tbar = 0.0;
        for (int64_t q = cnt[k]; q < cnt[k + 1]; ++q) {
            int64_t t = pos[q];
            double zb = pdir[t] * (pbar_dir[t] - sPP);
            cbar[t] += -li->T * zb;
            szb += zb;
            Tbar += -zb * (P->c[t] - li->m);
        }
        double mbar = li->T * szb;
        double gbar = li->clamped ? 0.0 : -Tbar * li->T / li->g;
        /* m = c[line, a], c2 = c[line, b] (frozen indices) */
        int64_t ia = dir ? li->a : k, ja = dir ? k : li->a;
        int64_t ib = dir ? li->b : k, jb = dir ? k : li->b;
        double add_a = mbar - gbar, add_b = gbar;
        /* route to support entries if present, else straight through Eq. (5) */
        int64_t ta = find_entry(P, ia, ja);
        if (ta >= 0) cbar[ta] += add_a; else eq5(P, ia, ja, add_a, gx, gy);
        if (li->b >= 0) {
            int64_t tb = find_entry(P, ib, jb);
            if (tb >= 0) cbar[tb] += add_b; else eq5(P, ib, jb, add_b, gx, gy);
        }
    }
    free(cnt); free(pos); free(fill);
}

/* d loss / d x (gx, N x 3) and d loss / d y (gy, M x 3), scaled by gbar.  Overwrites. */
void oracle_plan_backward(const oracle_plan* P, double gbar, double* gx, double* gy) {
    int64_t nnz = P->nnz;
    int32_t L = P->cfg.l_iter;
    if (gx) memset(gx, 0, sizeof(double) * 3 * P->N);
    if (gy) memset(gy, 0, sizeof(double) * 3 * P->M);
    double* cbar = (double*)calloc((size_t)(nnz ? nnz : 1), sizeof(double));
    const double* vf = P->vhist + (size_t)(2 * L) * nnz;
    for (int64_t t = 0; t < nnz; ++t) cbar[t] = gbar * vf[t];          /* loss = sum v c */
    if (P->cfg.grad_mode == 0) {
        double* ub = (double*)malloc(sizeof(double) * (nnz ? nnz : 1));
        double* wb = (double*)malloc(sizeof(double) * (nnz ? nnz : 1));
        for (int64_t t = 0; t < nnz; ++t) ub[t] = gbar * P->c[t];      /* vbar */
        for (int32_t l = L - 1; l >= 0; --l) {                          /* reverse Eqs. (3)-(4) */
            const double* w0 = P->vhist + (size_t)(2 * l) * nnz;
            const double* w1 = w0 + nnz;
            const double* w2 = w1 + nnz;
            sinkhorn_half_rev(P, w1, w2, ub, wb, P->cfg.row_first ? 1 : 0);
            sinkhorn_half_rev(P, w0, w1, wb, ub, P->cfg.row_first ? 0 : 1);
        }
        /* ub = P0bar.  P0 = (P_row + P_col)/2 -> Pbar_dir = P0bar / 2 on Omega_dir. */
        double* pb = (double*)calloc((size_t)(nnz ? nnz : 1), sizeof(double));
        for (int64_t t = 0; t < nnz; ++t) pb[t] = 0.5 * ub[t];
        softmax_rev(P, 0, pb, cbar, gx, gy);
        softmax_rev(P, 1, pb, cbar, gx, gy);
        free(ub); free(wb); free(pb);
    }
    for (int64_t t = 0; t < nnz; ++t) eq5(P, P->ti[t], P->tj[t], cbar[t], gx, gy); /* Eq. (5) */
    free(cbar);
}

/* ---------------------------------------------------------------- dense variant */

/* Dense APML, section III-A, tau ignored.  Returns the loss; P_out (N x M,
 * row-major) receives the final plan when non-NULL.  Memory O(N M). */
double oracle_dense_forward64(const double* x, const double* y, int64_t N, int64_t M,
                              const oracle_cfg* cfg, double* P_out) {
    double* C = (double*)malloc(sizeof(double) * N * M);
    double* Pr = (double*)calloc((size_t)(N * M), sizeof(double));
    double* Pc = (double*)calloc((size_t)(N * M), sizeof(double));
    double* P = (double*)malloc(sizeof(double) * N * M);
    for (int64_t i = 0; i < N; ++i)
        for (int64_t j = 0; j < M; ++j) C[i * M + j] = cost(x + 3 * i, y + 3 * j);
    oracle_cfg dc = *cfg; dc.tau = 0.0; /* dense: every similarity kept */
    int64_t K = N > M ? N : M;
    double* line = (double*)malloc(sizeof(double) * K);
    double* scratch = (double*)malloc(sizeof(double) * K);
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * K);
    double* pv = (double*)malloc(sizeof(double) * K);
    line_info li;
    for (int64_t i = 0; i < N; ++i) {                                   /* P_row */
        for (int64_t j = 0; j < M; ++j) line[j] = C[i * M + j];
        int64_t k = line_softmax(line, M, &dc, &li, idx, pv, scratch);
        for (int64_t q = 0; q < k; ++q) Pr[i * M + idx[q]] = pv[q];
    }
    for (int64_t j = 0; j < M; ++j) {                                   /* P_col */
        for (int64_t i = 0; i < N; ++i) line[i] = C[i * M + j];
        int64_t k = line_softmax(line, N, &dc, &li, idx, pv, scratch);
        for (int64_t q = 0; q < k; ++q) Pc[idx[q] * M + j] = pv[q];
    }
    for (int64_t e = 0; e < N * M; ++e) P[e] = 0.5 * (Pr[e] + Pc[e]);   /* P0 = (P_row + P_col)/2 */
    double* S = (double*)malloc(sizeof(double) * K);
    for (int32_t l = 0; l < cfg->l_iter; ++l) {                         /* dense Sinkhorn, column then row */
        for (int half = 0; half < 2; ++half) {
            int by_col = cfg->row_first ? (half == 1) : (half == 0);
            if (by_col) {
                for (int64_t j = 0; j < M; ++j) S[j] = 0.0;
                for (int64_t i = 0; i < N; ++i) for (int64_t j = 0; j < M; ++j) S[j] += P[i * M + j];
                for (int64_t i = 0; i < N; ++i) for (int64_t j = 0; j < M; ++j) P[i * M + j] /= (S[j] + cfg->eps_stab);
            } else {
                for (int64_t i = 0; i < N; ++i) {
                    double s = 0.0;
                    for (int64_t j = 0; j < M; ++j) s += P[i * M + j];
                    for (int64_t j = 0; j < M; ++j) P[i * M + j] /= (s + cfg->eps_stab);
                }
            }
        }
    }
    double loss = 0.0;                                                  /* <P, C>_F */
    for (int64_t i = 0; i < N; ++i) for (int64_t j = 0; j < M; ++j) loss += P[i * M + j] * C[i * M + j];
    if (P_out) memcpy(P_out, P, sizeof(double) * N * M);
    free(C); free(Pr); free(Pc); free(P); free(line); free(scratch); free(idx); free(pv); free(S);
    return loss;
}

double oracle_dense_forward(const float* x, const float* y, int64_t N, int64_t M,
                            const oracle_cfg* cfg, double* P_out) {
    double* xd = widen(x, 3 * N);
    double* yd = widen(y, 3 * M);
    double l = oracle_dense_forward64(xd, yd, N, M, cfg, P_out);
    free(xd); free(yd);
    return l;
}

/* ---------------------------------------------------------------- batch helper */

/* Algorithm 1 over B independent pairs, OpenMP over pairs.  loss[B] per-pair
 * losses; grad (B x N x 3, may be NULL) = d loss_b / d pred_b scaled by gbar[b] (NULL -> 1);
 * nnz[B] (may be NULL).  Returns the thread count used. */
int oracle_batch(const float* x, const float* y, int64_t B, int64_t N, int64_t M,
                 const oracle_cfg* cfg, const double* gbar, double* loss, double* grad,
                 int64_t* nnz, int nthreads) {
    int used = 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
    {
#pragma omp single
        used = omp_get_num_threads();
    }
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t b = 0; b < B; ++b) {
        oracle_plan* P = oracle_sparse_forward(x + 3 * N * b, y + 3 * M * b, N, M, cfg);
        loss[b] = P->loss;
        if (nnz) nnz[b] = P->nnz;
        if (grad) oracle_plan_backward(P, gbar ? gbar[b] : 1.0, grad + 3 * N * b, NULL);
        oracle_plan_free(P);
    }
    return used;
}
