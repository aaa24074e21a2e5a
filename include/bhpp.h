/*
 * bhpp.h -- C ABI of the B200-native BHPP engine (libbhpp.so).
 *
 * The reference (`bipush`, pure Python + numpy/scipy) has no native boundary:
 * its hot path is the Python API below, and its inner loops run in scipy's
 * csr_matvec.  This ABI is what that Python API binds (ctypes, see
 * paper_2312_06724_b200/_capi.py and INTEGRATION.md).  Plain pointers and
 * sizes only; no torch types.  All functions are thread-safe (a graph handle
 * serialises its own engine use with an internal mutex).
 *
 *   reference interface (file:line under pkg/src/bipush)    -> entry point
 *   BipartiteGraph CSR core + u_step/v_step (bigraph.py:53-188) -> bh_graph_create
 *   bhpp_query + topk (bhpp_query.py:160-218), batched          -> bh_query_batch
 *   ss_push / selective_push / pi_push (push_engine.py:120-258) -> bh_push_run
 *   power_iteration (push_engine.py:101-117), estimate_lambda   -> bh_power_iteration
 *   topk (bhpp_query.py:206-218) on an arbitrary score vector   -> bh_topk
 *   BipartiteGraph.__init__ canonicalisation (bigraph.py:53-111) -> bh_csr_build
 *   load_edge_list text parsing (bigraph.py:272-350)             -> bh_edge_list_*
 *   monte_carlo walks of MCSP (baselines.py:108-151)             -> bh_alias_*, bh_monte_carlo
 *
 * Status codes: 0 ok; BH_EINVAL -> ValueError; BH_EUNFLUSHED -> ValueError
 * ("unflushed ledger", push_engine.py:214-217); BH_ECUDA -> RuntimeError;
 * BH_ENOMEM -> MemoryError.  bh_last_error() returns the calling thread's
 * last message.
 */
#ifndef BHPP_H
#define BHPP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BH_OK 0
#define BH_EINVAL 1
#define BH_EUNFLUSHED 2
#define BH_ECUDA 3
#define BH_ENOMEM 4
#define BH_EDUP 5 /* bh_csr_build: a (u, v) pair repeats (bigraph.py:84-88) */

#define BH_DTYPE_F64 0 /* fp64 storage, fp64 arithmetic                       */
#define BH_DTYPE_F32 1 /* fp32 storage, fp64 row accumulation and control     */
/* OR into bh_graph_create's dtype: keep the caller's node order in the device
 * store.  By default both sides are relabelled by descending degree inside the
 * store (hub operand rows contiguous for L2 residency); every index crossing
 * the ABI stays in the caller's numbering either way, and ties in top-k still
 * break by the caller's index (bhpp_query.py:210). */
#define BH_GRAPH_KEEP_ORDER 0x100

#define BH_JOB_BHPP 0      /* ss_push -> pi_push -> power iteration -> combine */
#define BH_JOB_SS_PUSH 1   /* backward with budget switch (push_engine.py:145) */
#define BH_JOB_SELECTIVE 2 /* backward without budget (push_engine.py:120)     */
#define BH_JOB_PI_PUSH 3   /* forward from a flushed ledger (push_engine.py:194) */
#define BH_JOB_POWER 4     /* truncated power series (push_engine.py:101)      */

#define BH_TERM_THRESHOLD 0 /* "threshold-met" */
#define BH_TERM_BUDGET 1    /* "budget-switch" */
#define BH_TERM_DRAINED 2   /* "mass-drained"  */

#define BH_PHASE_SELECTIVE 0  /* round_hook phase "selective"          */
#define BH_PHASE_SEQUENTIAL 1 /* round_hook phase "sequential"         */
#define BH_PHASE_FORWARD 2    /* round_hook phase "forward-selective"  */

typedef struct bh_graph bh_graph;

/* Per-query phase trace: the integer counters of bhpp_query.py:198-201 plus
 * the exact-tie bookkeeping of the PI-Push budget test. */
typedef struct bh_trace {
    int64_t sel_b;       /* backward selective_rounds                     */
    int64_t seq_b;       /* backward sequential_rounds                    */
    int64_t n_p_b;       /* backward n_p (after SS-Push)                  */
    int64_t sel_f;       /* forward selective_rounds                      */
    int64_t pi_iters;    /* forward power_iterations                      */
    int64_t n_p_f;       /* forward n_p (cumulative)                      */
    double gamma;        /* forward gamma (frozen weighted mass at entry) */
    int32_t term_b;      /* BH_TERM_*                                     */
    int32_t term_f;      /* BH_TERM_*                                     */
    int32_t tie_checks;  /* budget checks taken with A == U every round   */
    int32_t tie_broke;   /* 1 if the forward phase ended at such a check  */
    int32_t source;      /* U index of the query                          */
    int32_t status;      /* 0 ok, BH_EINVAL: source out of range (device  */
                         /* pointer batches; the batch returns BH_EINVAL) */
    int32_t near_ties;   /* budget checks (Eq. 10 / Eq. 12) decided with a */
                         /* relative margin below 1e-12   */
    int32_t pad;
    double min_margin;   /* smallest relative margin of any budget check   */
} bh_trace;

typedef struct bh_query_params {
    double alpha;          /* restart probability, (0, 1)                       */
    double lam;            /* IndexMeta.lam                                      */
    double eps_b;          /* backward share of epsilon                          */
    double eps_f;          /* forward share of epsilon                           */
    int32_t k;             /* top-k per query (0 = no top-k)                     */
    int32_t exclude_query; /* drop the source from its own top-k                 */
    int32_t want_scores;   /* also write the full score vector per query         */
    int32_t slots;         /* query-block width B (0 = automatic)                */
    int32_t on_device;     /* 1: all pointer arguments are device pointers       */
    int32_t flags;         /* BH_QUERY_ASYNC: with on_device, return after the  */
                           /* batch is enqueued; bh_query_wait() completes it    */
} bh_query_params;

#define BH_QUERY_ASYNC 1

typedef struct bh_graph_info {
    int64_t n_u, n_v, n_e;
    int32_t dtype, device;
    int64_t device_bytes;   /* graph store footprint                         */
    int64_t max_deg_u, max_deg_v;
} bh_graph_info;

/* Called after every push round of slot 0 in bh_push_run (the reference's
 * round_hook, push_engine.py:133,166,182,232).  Arrays are host copies valid
 * only during the call; residue_v is always zero at a round boundary. */
typedef void (*bh_round_hook)(void *user, int32_t phase, int64_t rounds, const double *residue_u,
                              const double *estimate, int64_t n_p);

/* ---- graph store (K-G) ---------------------------------------------------- */
int bh_graph_create(int64_t n_u, int64_t n_v, int64_t n_e, const int64_t *u_indptr,
                    const int32_t *u_indices, const double *u_weights, const int64_t *v_indptr,
                    const int32_t *v_indices, const double *v_weights, const double *ws_u,
                    const double *ws_v, int32_t device, int32_t dtype, bh_graph **out);
void bh_graph_destroy(bh_graph *g);
int bh_graph_get_info(const bh_graph *g, bh_graph_info *out);

/* ---- batched SS-BI-PUSH query (bhpp_query + topk for many sources) -------- */
/* sources[n_q] int32; tie_skip[n_q] nullable (continue through this many exact
 * PI-Push budget ties before breaking; default 0 = exact-arithmetic outcome).
 * Outputs (nullable unless noted): topk_idx/topk_score [n_q*k] (-1 / 0 padded),
 * trace [n_q] (required), scores [n_q*n_u] (want_scores).  `stream` is a
 * cudaStream_t (NULL = the engine's own stream).  With on_device == 0 the
 * pointers are host memory and the copies happen inside the call. */
int bh_query_batch(bh_graph *g, const bh_query_params *p, const int32_t *sources, int64_t n_q,
                   const int32_t *tie_skip, int32_t *topk_idx, double *topk_score, bh_trace *trace,
                   double *scores, void *stream);

/* ---- single-query ledger kernels (ss_push / selective_push / pi_push / bhpp) */
/* job: BH_JOB_*.  residue_u / estimate [n_u] and n_p are in/out host ledger
 * arrays (read for BH_JOB_PI_PUSH, written by every job).  scores [n_u] gets
 * the forward scores (PI_PUSH) or the BHPP vector (BHPP).  hook nullable. */
int bh_push_run(bh_graph *g, int32_t job, int32_t source, double alpha, double lam, double eps_b,
                double eps_f, int32_t tie_skip, double *residue_u, double *estimate, int64_t *n_p,
                double *scores, bh_trace *trace, bh_round_hook hook, void *user);

/* ---- power iteration (push_engine.py:101-117) over n_vec start vectors ---- */
/* start, out: [n_vec * n_u] row-major host arrays; out = alpha * acc_t. */
int bh_power_iteration(bh_graph *g, const double *start, int64_t n_vec, double alpha, int32_t t,
                       double *out);

/* Completes a batch submitted with BH_QUERY_ASYNC on this graph: waits for
 * its stream, checks termination, updates bh_last_run_stats.  No other call
 * may use the graph in between. */
int bh_query_wait(bh_graph *g);

/* ---- top-k of an arbitrary score vector (bhpp_query.py:206-218) ---------- */
/* (score desc, index asc); exclude < 0 keeps every index.  Returns count via
 * *out_count.  Host pointers. */
int bh_topk(const double *scores, int64_t n, int64_t k, int64_t exclude, int64_t *out_idx,
            double *out_score, int64_t *out_count);

/* ---- graph ingestion (bigraph.py:53-111) ---------------------------------- */
/* Canonical CSR of both sides from n_e edge triples (host pointers in and
 * out), built on `device` with two radix sorts of the packed pair keys:
 * U rows sorted by v, V rows sorted by u, weights carried along, ws_u / ws_v
 * summed in CSR order (bit-identical to the reference's np.bincount).
 * Endpoints must lie in [0, n_u) x [0, n_v) (BH_EINVAL otherwise); a repeated
 * pair returns BH_EDUP and leaves the outputs unspecified.  Sizes < 2^31. */
int bh_csr_build(int64_t n_u, int64_t n_v, int64_t n_e, const int64_t *edge_u, const int64_t *edge_v,
                 const double *edge_w, int64_t *u_indptr, int32_t *u_indices, double *u_weights,
                 int64_t *v_indptr, int32_t *v_indices, double *v_weights, double *ws_u, double *ws_v,
                 int32_t device);

/* Text edge list (bigraph.py:272-350), host-side native parser.  buf/len: the
 * file bytes; delim: column separator bytes or NULL for runs of whitespace;
 * has_default/default_weight: weight of two-column lines.  Returns BH_OK with
 * *out set, or BH_EFALLBACK when the input needs the reference's Python loop
 * (non-ASCII bytes, weight tokens other than plain decimals, or any data error;
 * *err_line then holds the offending line, 0 if none). */
typedef struct bh_edge_list bh_edge_list;
#define BH_EFALLBACK 6
int bh_edge_list_parse(const char *buf, int64_t len, const char *delim, int64_t delim_len, int32_t has_default,
                       double default_weight, bh_edge_list **out, int64_t *err_line);
/* sizes: labels per side, bytes of each side's concatenated labels, merged edges */
int bh_edge_list_sizes(const bh_edge_list *el, int64_t *n_u, int64_t *n_v, int64_t *u_bytes, int64_t *v_bytes,
                       int64_t *n_e);
/* labels as concatenated bytes + end offsets, merged edges in first-seen order */
int bh_edge_list_export(const bh_edge_list *el, char *u_blob, int64_t *u_ends, char *v_blob, int64_t *v_ends,
                        int64_t *edge_u, int64_t *edge_v, double *edge_w);
void bh_edge_list_free(bh_edge_list *el);

/* ---- Monte-Carlo walks (MCSP forward half, baselines.py:45-151) ------------ */
/* Alias tables of build_alias (per CSR slot, alias = local slot offset) copied
 * to the graph's device; bh_monte_carlo adds to counts[n_u] (host) the stop
 * counts of walks [first, first + n) from `source`: stop with probability
 * alpha before every step, else U -> V -> U with alias draws.  Walk i uses the
 * Philox4x32-10 stream (seed, i).  Destroy the tables before their graph. */
typedef struct bh_alias bh_alias;
/* build_alias (baselines.py:41-77) for one CSR side on `device`: per-slot prob
 * and local alias offsets, bit-identical to the reference's tables (Vose
 * pairing per row in the reference's order, numpy's pairwise row sum).  Host
 * pointers in and out; indptr [n_rows + 1], weights / prob / alias [n_e]. */
int bh_alias_build(int64_t n_rows, int64_t n_e, const int64_t *indptr, const double *weights, int32_t device,
                   double *prob, int64_t *alias);
int bh_alias_create(bh_graph *g, const double *u_prob, const int64_t *u_alias, const double *v_prob,
                    const int64_t *v_alias, bh_alias **out);
int bh_monte_carlo(const bh_alias *a, int64_t source, double alpha, int64_t first, int64_t n, uint64_t seed,
                   int64_t *counts);
void bh_alias_destroy(bh_alias *a);

/* ---- measurement ---------------------------------------------------------- */
typedef struct bh_run_stats {
    int64_t rounds;        /* rounds launched by the last run on this graph      */
    int64_t launches;      /* kernels launched by it                             */
    int64_t slots;         /* query-block width B it used                        */
    int64_t profiled;      /* 1 if the ms_* fields below were measured           */
    double ms_prep;        /* sum of K1 (prep) durations, CUDA events            */
    double ms_vpull;       /* sum of K2 + K2b (V pull) durations                 */
    double ms_upull;       /* sum of K3 + K3b (U pull) durations                 */
    double ms_control;     /* sum of K4..K6 (control, finalize, top-k)           */
    int64_t frontier_rounds;   /* rounds whose V half ran in frontier form (K-F) */
    int64_t frontier_u_rounds; /* rounds whose U half ran in frontier form       */
} bh_run_stats;
/* on != 0: bracket every round's kernels with CUDA events on the launch stream
 * (process-wide switch; costs one event record per kernel group). */
int bh_set_profiling(int32_t on);
/* Frontier rounds (K-F), process-wide: a round pulls only the rows reachable
 * from its pushed set when the pushed rows (summed over the block's slots)
 * touch at most fraction * |E| edges; its U half likewise on the V rows it
 * reached.  Mirrors push_engine._SCATTER_LIMIT (push_engine.py:44, 297,
 * 315).  fraction < 0: never; >= 1: whenever no slot is in power iteration.
 * Blocks of more than 16 slots run dense rounds unless fraction >= 1.  Results do not depend on it (every visited row is summed in
 * full); it only changes which rows a round visits.  Default 0.01 (the
 * reference's 0.25 is a CPU tuning). */
int bh_set_scatter_limit(double fraction);
/* Measurement gate: enqueue on `stream` a one-thread kernel that spins until
 * *flag (host-mapped pinned memory) becomes nonzero, so a batch can be fully
 * enqueued before the device starts it and device timing excludes host
 * submission gaps. */
int bh_stream_gate(void *stream, const int32_t *flag);
int bh_last_run_stats(bh_graph *g, bh_run_stats *out);

/* ---- misc ----------------------------------------------------------------- */
const char *bh_last_error(void);
int bh_version(void);
/* Number of CUDA kernels this library launched in this process (for the
 * bench's gpu_launches claim). */
int64_t bh_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* BHPP_H */
