/*
 * bhpp_oracle.c -- CPU restatement of the reference SS-BI-PUSH query path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine in paper_2312_06724_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links or calls it.
 *
 * It restates, operation for operation, the reference Python package
 * `bipush` (pkg/src/bipush, numpy + scipy), so that its fp64 results are
 * bit-identical to the reference on the same CSR arrays:
 *   - numpy float64 `.sum()` is numpy's pairwise summation (8-way unrolled
 *     blocks of <=128, recursive halving) -> pairwise_sum() below;
 *   - scipy `csr_matvec` is a sequential per-row `sum += Ax*x` starting from
 *     0.0 with no FMA contraction (this file is built -ffp-contract=off);
 *   - `np.bincount(idx, weights)` is a sequential scatter-add into zeros;
 *   - Python's math.log / ** are glibc log / pow, as used here.
 * Reference anchors are cited per function (file:line under /root/reference).
 * The pin is the tests/golden fixtures (.npz), produced by running the reference itself
 * (tests/golden/make_golden.py) and checked by tests/test_oracle_golden.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OG_OK 0
#define OG_EINVAL 1
#define OG_ENOMEM 2

#define OG_TERM_THRESHOLD 0
#define OG_TERM_BUDGET 1
#define OG_TERM_DRAINED 2

#define OG_PHASE_SELECTIVE 0
#define OG_PHASE_SEQUENTIAL 1
#define OG_PHASE_FORWARD 2

typedef struct og_graph {
    int64_t n_u, n_v, n_e;
    int64_t *u_indptr, *v_indptr;
    int32_t *u_indices, *v_indices;
    double *u_weights, *v_weights, *ws_u, *ws_v;
    int64_t *deg_u, *deg_v;
    double *u_step;  /* U-CSR  w/ws(u)   bigraph.py:148-155 (u_step.data)      */
    double *v_step;  /* V-CSR  w/ws(v)   bigraph.py:157-164 (v_step.data)      */
    double *recv_uv; /* U-CSR  w/ws(v)   bigraph.py:176-183                    */
    double *recv_vu; /* V-CSR  w/ws(u)   bigraph.py:185-188                    */
} og_graph;

typedef struct og_trace {
    int64_t selective_rounds;
    int64_t sequential_rounds;
    int64_t power_iterations;
    int64_t n_p;
    int32_t terminated_by;
    int32_t tie_checks;    /* forward budget checks taken with A == U in every forward round */
    int32_t tie_break_at;  /* 1-based tie check at which the phase broke, 0 if none */
    int32_t _pad;
    double gamma;
} og_trace;

typedef void (*og_hook)(void *user, int32_t phase, int64_t rounds, const double *r_u,
                        const double *r_v, const double *est, int64_t n_p);

/* ------------------------------------------------------------------------- */
/* numpy float64 add.reduce over a contiguous vector (pairwise summation).    */
static double pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}

double og_numpy_sum(const double *a, int64_t n) { return 0.0 + pairwise_sum(a, n); }

/* ------------------------------------------------------------------------- */
void og_graph_destroy(og_graph *g) {
    if (!g) return;
    free(g->u_indptr); free(g->v_indptr); free(g->u_indices); free(g->v_indices);
    free(g->u_weights); free(g->v_weights); free(g->ws_u); free(g->ws_v);
    free(g->deg_u); free(g->deg_v); free(g->u_step); free(g->v_step);
    free(g->recv_uv); free(g->recv_vu);
    free(g);
}

#define DUP(dst, src, n, T)                                   \
    do {                                                      \
        (dst) = (T *)malloc(sizeof(T) * ((n) > 0 ? (n) : 1)); \
        if (!(dst)) goto fail;                                \
        memcpy((dst), (src), sizeof(T) * (n));                \
    } while (0)

/* CSR arrays exactly as BipartiteGraph builds them (bigraph.py:89-108). */
og_graph *og_graph_create(int64_t n_u, int64_t n_v, int64_t n_e,
                          const int64_t *u_indptr, const int32_t *u_indices, const double *u_weights,
                          const int64_t *v_indptr, const int32_t *v_indices, const double *v_weights,
                          const double *ws_u, const double *ws_v) {
    og_graph *g = (og_graph *)calloc(1, sizeof(og_graph));
    if (!g) return NULL;
    g->n_u = n_u; g->n_v = n_v; g->n_e = n_e;
    DUP(g->u_indptr, u_indptr, n_u + 1, int64_t);
    DUP(g->v_indptr, v_indptr, n_v + 1, int64_t);
    DUP(g->u_indices, u_indices, n_e, int32_t);
    DUP(g->v_indices, v_indices, n_e, int32_t);
    DUP(g->u_weights, u_weights, n_e, double);
    DUP(g->v_weights, v_weights, n_e, double);
    DUP(g->ws_u, ws_u, n_u, double);
    DUP(g->ws_v, ws_v, n_v, double);
    g->deg_u = (int64_t *)malloc(sizeof(int64_t) * n_u);
    g->deg_v = (int64_t *)malloc(sizeof(int64_t) * n_v);
    g->u_step = (double *)malloc(sizeof(double) * n_e);
    g->v_step = (double *)malloc(sizeof(double) * n_e);
    g->recv_uv = (double *)malloc(sizeof(double) * n_e);
    g->recv_vu = (double *)malloc(sizeof(double) * n_e);
    if (!g->deg_u || !g->deg_v || !g->u_step || !g->v_step || !g->recv_uv || !g->recv_vu) goto fail;
    for (int64_t u = 0; u < n_u; u++) {
        g->deg_u[u] = u_indptr[u + 1] - u_indptr[u];
        for (int64_t e = u_indptr[u]; e < u_indptr[u + 1]; e++) {
            g->u_step[e] = u_weights[e] / ws_u[u];              /* bigraph.py:151 */
            g->recv_uv[e] = u_weights[e] / ws_v[u_indices[e]];  /* bigraph.py:183 */
        }
    }
    for (int64_t v = 0; v < n_v; v++) {
        g->deg_v[v] = v_indptr[v + 1] - v_indptr[v];
        for (int64_t e = v_indptr[v]; e < v_indptr[v + 1]; e++) {
            g->v_step[e] = v_weights[e] / ws_v[v];              /* bigraph.py:160 */
            g->recv_vu[e] = v_weights[e] / ws_u[v_indices[e]];  /* bigraph.py:188 */
        }
    }
    return g;
fail:
    og_graph_destroy(g);
    return NULL;
}

/* ------------------------------------------------------------------------- */
/* push_engine.py:85-98 */
int64_t og_required_iterations(double alpha, double epsilon_f, double mass) {
    if (!(alpha > 0.0 && alpha < 1.0)) return -1;
    if (epsilon_f <= 0) return -1;
    if (mass <= 0) return 0;
    double x = ceil(log(mass / epsilon_f) / log(1.0 / (1.0 - alpha))) - 1;
    return x > 0 ? (int64_t)x : 0;
}

/* push_engine.py:101-117: acc = base; t x { mid = u_step_t @ acc;
 * acc = base + (1-alpha) * (v_step_t @ mid) }; return alpha * acc.
 * u_step_t row v == V-CSR row v with values w/ws(u) (recv_vu); v_step_t row u
 * == U-CSR row u with values w/ws(v) (recv_uv); scipy's .T.tocsr() keeps the
 * ascending column order, as the V-CSR / U-CSR rows here do. */
int og_power_iteration(const og_graph *g, const double *start, double alpha, int64_t t, double *out) {
    if (!(alpha > 0.0 && alpha < 1.0) || t < 0) return OG_EINVAL;
    const int64_t n_u = g->n_u, n_v = g->n_v;
    double *acc = out;
    double *mid = (double *)malloc(sizeof(double) * (n_v > 0 ? n_v : 1));
    if (!mid) return OG_ENOMEM;
    memcpy(acc, start, sizeof(double) * n_u);
    const double c = 1.0 - alpha;
    for (int64_t it = 0; it < t; it++) {
        for (int64_t v = 0; v < n_v; v++) {
            double sum = 0.0;
            for (int64_t e = g->v_indptr[v]; e < g->v_indptr[v + 1]; e++)
                sum += g->recv_vu[e] * acc[g->v_indices[e]];
            mid[v] = sum;
        }
        for (int64_t u = 0; u < n_u; u++) {
            double sum = 0.0;
            for (int64_t e = g->u_indptr[u]; e < g->u_indptr[u + 1]; e++)
                sum += g->recv_uv[e] * mid[g->u_indices[e]];
            acc[u] = start[u] + c * sum;
        }
    }
    for (int64_t u = 0; u < n_u; u++) acc[u] = alpha * acc[u];
    free(mid);
    return OG_OK;
}

/* ------------------------------------------------------------------------- */
/* Round primitives: push_engine.py:280-324.                                  */
typedef struct og_work {
    double *add_v, *add_u, *dense;
    int64_t *uidx, *vidx;
    double *tmp_u;
} og_work;

static int work_alloc(og_work *w, const og_graph *g) {
    w->add_v = (double *)malloc(sizeof(double) * g->n_v);
    w->add_u = (double *)malloc(sizeof(double) * g->n_u);
    w->dense = (double *)malloc(sizeof(double) * g->n_u);
    w->uidx = (int64_t *)malloc(sizeof(int64_t) * g->n_u);
    w->vidx = (int64_t *)malloc(sizeof(int64_t) * g->n_v);
    w->tmp_u = (double *)malloc(sizeof(double) * g->n_u);
    return (w->add_v && w->add_u && w->dense && w->uidx && w->vidx && w->tmp_u) ? OG_OK : OG_ENOMEM;
}

static void work_free(og_work *w) {
    free(w->add_v); free(w->add_u); free(w->dense); free(w->uidx); free(w->vidx); free(w->tmp_u);
}

/* _push_u, push_engine.py:294-309 */
static void push_u(const og_graph *g, double *r_u, double *r_v, double *est, int64_t *n_p,
                   const int64_t *uidx, int64_t na, double alpha, double scatter_limit, og_work *w) {
    int64_t deg_sum = 0;
    for (int64_t i = 0; i < na; i++) deg_sum += g->deg_u[uidx[i]];
    const double c = 1.0 - alpha;
    if ((double)deg_sum <= scatter_limit * (double)g->n_e) {
        /* scatter: contrib = (1-a) * recv_uv[slots] * amount; bincount */
        memset(w->add_v, 0, sizeof(double) * g->n_v);
        for (int64_t i = 0; i < na; i++) {
            int64_t u = uidx[i];
            double amt = r_u[u];
            for (int64_t e = g->u_indptr[u]; e < g->u_indptr[u + 1]; e++)
                w->add_v[g->u_indices[e]] += (c * g->recv_uv[e]) * amt;
        }
        for (int64_t v = 0; v < g->n_v; v++) r_v[v] = r_v[v] + w->add_v[v];
    } else {
        /* dense: r_v += (1-a) * (v_step @ dense) */
        memset(w->dense, 0, sizeof(double) * g->n_u);
        for (int64_t i = 0; i < na; i++) w->dense[uidx[i]] = r_u[uidx[i]];
        for (int64_t v = 0; v < g->n_v; v++) {
            double sum = 0.0;
            for (int64_t e = g->v_indptr[v]; e < g->v_indptr[v + 1]; e++)
                sum += g->v_step[e] * w->dense[g->v_indices[e]];
            r_v[v] = r_v[v] + c * sum;
        }
    }
    for (int64_t i = 0; i < na; i++) {
        int64_t u = uidx[i];
        est[u] = est[u] + alpha * r_u[u];
    }
    for (int64_t i = 0; i < na; i++) r_u[uidx[i]] = 0.0;
    *n_p += deg_sum;
}

/* _flush_v, push_engine.py:312-324 */
static void flush_v(const og_graph *g, double *r_u, double *r_v, int64_t *n_p,
                    const int64_t *vidx, int64_t nv, double scatter_limit, og_work *w) {
    int64_t deg_sum = 0;
    for (int64_t i = 0; i < nv; i++) deg_sum += g->deg_v[vidx[i]];
    if ((double)deg_sum <= scatter_limit * (double)g->n_e) {
        memset(w->add_u, 0, sizeof(double) * g->n_u);
        for (int64_t i = 0; i < nv; i++) {
            int64_t v = vidx[i];
            double amt = r_v[v];
            for (int64_t e = g->v_indptr[v]; e < g->v_indptr[v + 1]; e++)
                w->add_u[g->v_indices[e]] += g->recv_vu[e] * amt;
        }
        for (int64_t u = 0; u < g->n_u; u++) r_u[u] = r_u[u] + w->add_u[u];
    } else {
        for (int64_t u = 0; u < g->n_u; u++) {
            double sum = 0.0;
            for (int64_t e = g->u_indptr[u]; e < g->u_indptr[u + 1]; e++)
                sum += g->u_step[e] * r_v[g->u_indices[e]];
            r_u[u] = r_u[u] + sum;
        }
    }
    memset(r_v, 0, sizeof(double) * g->n_v);
    *n_p += deg_sum;
}

/* _round, push_engine.py:280-291.  theta_vec == NULL -> scalar threshold.
 * Returns 1 if any work happened; *n_active = |A|. */
static int round_(const og_graph *g, double *r_u, double *r_v, double *est, int64_t *n_p,
                  double theta, const double *theta_vec, double alpha, double scatter_limit,
                  og_work *w, int64_t *n_active) {
    int worked = 0;
    int64_t na = 0;
    for (int64_t u = 0; u < g->n_u; u++) {
        double th = theta_vec ? theta_vec[u] : theta;
        if (r_u[u] > th) w->uidx[na++] = u;
    }
    *n_active = na;
    if (na) {
        push_u(g, r_u, r_v, est, n_p, w->uidx, na, alpha, scatter_limit, w);
        worked = 1;
    }
    int64_t nv = 0;
    for (int64_t v = 0; v < g->n_v; v++)
        if (r_v[v] > 0.0) w->vidx[nv++] = v;
    if (nv) {
        flush_v(g, r_u, r_v, n_p, w->vidx, nv, scatter_limit, w);
        worked = 1;
    }
    return worked;
}

static int any_gt(const double *a, int64_t n, double th) {
    for (int64_t i = 0; i < n; i++)
        if (a[i] > th) return 1;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* ss_push (budget=1), push_engine.py:145-191; selective_push (budget=0),
 * push_engine.py:120-142.  The ledger (r_u, r_v, est, n_p) is initialised here
 * (ResidueLedger.initial, push_engine.py:57-63). */
int og_ss_push(const og_graph *g, int64_t target, double alpha, double epsilon_b, int32_t budget,
               double scatter_limit, double *r_u, double *r_v, double *est, int64_t *n_p,
               og_trace *tr, og_hook hook, void *user) {
    if (!(alpha > 0.0 && alpha < 1.0) || epsilon_b <= 0) return OG_EINVAL;
    if (target < 0 || target >= g->n_u) return OG_EINVAL;
    og_work w;
    if (work_alloc(&w, g) != OG_OK) { work_free(&w); return OG_ENOMEM; }
    memset(r_u, 0, sizeof(double) * g->n_u);
    memset(r_v, 0, sizeof(double) * g->n_v);
    memset(est, 0, sizeof(double) * g->n_u);
    r_u[target] = 1.0;
    *n_p = 0;
    memset(tr, 0, sizeof(*tr));
    const double log_decay = log(1.0 / (1.0 - alpha));
    const double budget_scale = 2.0 * (double)g->n_e;
    int64_t sel = 0, seq = 0, na;
    int term = -1;
    for (;;) {
        sel += round_(g, r_u, r_v, est, n_p, epsilon_b, NULL, alpha, scatter_limit, &w, &na);
        if (hook) hook(user, OG_PHASE_SELECTIVE, sel, r_u, r_v, est, *n_p);
        if (!any_gt(r_u, g->n_u, epsilon_b)) { term = OG_TERM_THRESHOLD; break; }
        if (!budget) continue;
        double mass = og_numpy_sum(r_u, g->n_u);
        if (mass <= 0.0) { term = OG_TERM_DRAINED; break; }
        if ((double)(*n_p) >= budget_scale * (log(1.0 / mass) / log_decay)) break;
    }
    if (term < 0) {
        while (any_gt(r_u, g->n_u, epsilon_b) && og_numpy_sum(r_u, g->n_u) > epsilon_b) {
            seq += round_(g, r_u, r_v, est, n_p, 0.0, NULL, alpha, scatter_limit, &w, &na);
            if (hook) hook(user, OG_PHASE_SEQUENTIAL, seq, r_u, r_v, est, *n_p);
        }
        term = OG_TERM_BUDGET;
    }
    tr->selective_rounds = sel;
    tr->sequential_rounds = seq;
    tr->power_iterations = 0;
    tr->n_p = *n_p;
    tr->terminated_by = term;
    work_free(&w);
    return OG_OK;
}

/* pi_push, push_engine.py:194-258.  Mutates the ledger in place and writes the
 * forward scores.  Also records the PI-Push exact-tie decisions (SURVEY.md
 * section 0 fact 11): a budget check taken while every forward round so far
 * pushed all of U compares 2|E|k against 2|E|k in exact arithmetic. */
int og_pi_push(const og_graph *g, int64_t source, double alpha, double lam, double epsilon_f,
               double scatter_limit, double *r_u, double *r_v, double *est, int64_t *n_p,
               double *scores, og_trace *tr, og_hook hook, void *user) {
    if (!(alpha > 0.0 && alpha < 1.0) || epsilon_f <= 0 || lam <= 0) return OG_EINVAL;
    if (source < 0 || source >= g->n_u) return OG_EINVAL;
    for (int64_t v = 0; v < g->n_v; v++)
        if (r_v[v] != 0.0) return OG_EINVAL + 16; /* "unflushed ledger" */
    const int64_t n_u = g->n_u;
    og_work w;
    double *w_ratio = (double *)malloc(sizeof(double) * n_u);
    double *theta = (double *)malloc(sizeof(double) * n_u);
    if (work_alloc(&w, g) != OG_OK || !w_ratio || !theta) {
        work_free(&w); free(w_ratio); free(theta); return OG_ENOMEM;
    }
    memset(tr, 0, sizeof(*tr));
    const double *ws = g->ws_u;
    const double wsq = ws[source];
    const double ef_over_lam = epsilon_f / lam;
    for (int64_t u = 0; u < n_u; u++) {
        w_ratio[u] = ws[u] / wsq;
        theta[u] = (wsq / ws[u]) * ef_over_lam;
    }
    for (int64_t u = 0; u < n_u; u++) w.tmp_u[u] = w_ratio[u] * r_u[u];
    const double gamma = og_numpy_sum(w.tmp_u, n_u);
    const int64_t n_p_entry = *n_p;
    const double log_decay = log(1.0 / (1.0 - alpha));
    const double budget_scale = 2.0 * (double)g->n_e;
    int64_t sel = 0, power_iters = 0, na;
    int term = -1;
    int all_full = 1;
    int32_t tie_checks = 0, tie_break_at = 0;
    double wmass = 0.0;
    for (;;) {
        sel += round_(g, r_u, r_v, est, n_p, 0.0, theta, alpha, scatter_limit, &w, &na);
        if (na != n_u) all_full = 0;
        if (hook) hook(user, OG_PHASE_FORWARD, sel, r_u, r_v, est, *n_p);
        {
            int any = 0;
            for (int64_t u = 0; u < n_u; u++)
                if (r_u[u] > theta[u]) { any = 1; break; }
            if (!any) { term = OG_TERM_THRESHOLD; break; }
        }
        for (int64_t u = 0; u < n_u; u++) w.tmp_u[u] = w_ratio[u] * r_u[u];
        wmass = og_numpy_sum(w.tmp_u, n_u);
        if (wmass <= 0.0) { term = OG_TERM_DRAINED; break; }
        double budget = budget_scale * (log(gamma / wmass) / log_decay);
        int brk = ((double)(*n_p - n_p_entry) >= budget);
        if (all_full) {
            tie_checks++;
            if (brk) tie_break_at = tie_checks;
        }
        if (brk) break;
    }
    for (int64_t u = 0; u < n_u; u++) scores[u] = w_ratio[u] * est[u];
    if (term < 0) {
        double *f = w.tmp_u;
        for (int64_t u = 0; u < n_u; u++) f[u] = w_ratio[u] * r_u[u];
        power_iters = og_required_iterations(alpha, epsilon_f, og_numpy_sum(f, n_u));
        double *pi = (double *)malloc(sizeof(double) * n_u);
        if (!pi) { work_free(&w); free(w_ratio); free(theta); return OG_ENOMEM; }
        og_power_iteration(g, f, alpha, power_iters, pi);
        for (int64_t u = 0; u < n_u; u++) scores[u] = scores[u] + pi[u];
        free(pi);
        term = OG_TERM_BUDGET;
    }
    tr->selective_rounds = sel;
    tr->sequential_rounds = 0;
    tr->power_iterations = power_iters;
    tr->n_p = *n_p;
    tr->terminated_by = term;
    tr->gamma = gamma;
    tr->tie_checks = tie_checks;
    tr->tie_break_at = tie_break_at;
    work_free(&w);
    free(w_ratio);
    free(theta);
    return OG_OK;
}

/* bhpp_query arithmetic, bhpp_query.py:182-189: ss_push, pi_push on the shared
 * ledger, scores = fwd.scores + ledger.estimate.  (Fingerprint check and the
 * epsilon split stay with the caller, as in the reference.) */
int og_bhpp_query(const og_graph *g, int64_t q, double alpha, double lam, double eps_b, double eps_f,
                  double scatter_limit, double *scores, og_trace *back, og_trace *fwd,
                  og_hook hook, void *user) {
    if (eps_b <= 0 || eps_f <= 0) return OG_EINVAL;
    double *r_u = (double *)malloc(sizeof(double) * g->n_u);
    double *r_v = (double *)malloc(sizeof(double) * (g->n_v > 0 ? g->n_v : 1));
    double *est = (double *)malloc(sizeof(double) * g->n_u);
    int64_t n_p = 0;
    int rc = OG_ENOMEM;
    if (!r_u || !r_v || !est) goto done;
    rc = og_ss_push(g, q, alpha, eps_b, 1, scatter_limit, r_u, r_v, est, &n_p, back, hook, user);
    if (rc) goto done;
    rc = og_pi_push(g, q, alpha, lam, eps_f, scatter_limit, r_u, r_v, est, &n_p, scores, fwd, hook, user);
    if (rc) goto done;
    for (int64_t u = 0; u < g->n_u; u++) scores[u] = scores[u] + est[u];
done:
    free(r_u); free(r_v); free(est);
    return rc;
}

/* topk, bhpp_query.py:206-218: stable argsort of -scores (score desc, index
 * asc), optionally dropping the query index, first k.  Returns the count. */
static const double *g_sort_keys;
static int cmp_desc_stable(const void *a, const void *b) {
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    double x = -g_sort_keys[i], y = -g_sort_keys[j];
    if (x < y) return -1;
    if (x > y) return 1;
    return (i > j) - (i < j);
}

int64_t og_topk(const double *scores, int64_t n, int64_t k, int64_t exclude, int64_t *out_idx) {
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    if (!order) return -1;
    for (int64_t i = 0; i < n; i++) order[i] = i;
    g_sort_keys = scores; /* not reentrant; test helper only */
    qsort(order, (size_t)n, sizeof(int64_t), cmp_desc_stable);
    int64_t m = 0;
    for (int64_t i = 0; i < n && m < k; i++) {
        if (order[i] == exclude) continue;
        out_idx[m++] = order[i];
    }
    free(order);
    return m;
}

/* estimate_lambda, bhpp_query.py:70-83 */
double og_estimate_lambda(const og_graph *g, double alpha, int64_t tau) {
    double *ones = (double *)malloc(sizeof(double) * g->n_u);
    double *probe = (double *)malloc(sizeof(double) * g->n_u);
    if (!ones || !probe) { free(ones); free(probe); return -1.0; }
    for (int64_t u = 0; u < g->n_u; u++) ones[u] = 1.0;
    og_power_iteration(g, ones, alpha, tau, probe);
    double mx = probe[0];
    for (int64_t u = 1; u < g->n_u; u++) if (probe[u] > mx) mx = probe[u];
    double from_probe = mx + (double)g->n_u * pow(1.0 - alpha, (double)(tau + 1));
    double wmax = g->ws_u[0], wmin = g->ws_u[0];
    for (int64_t u = 1; u < g->n_u; u++) {
        if (g->ws_u[u] > wmax) wmax = g->ws_u[u];
        if (g->ws_u[u] < wmin) wmin = g->ws_u[u];
    }
    double from_ratio = wmax / wmin;
    free(ones); free(probe);
    return from_probe < from_ratio ? from_probe : from_ratio;
}
