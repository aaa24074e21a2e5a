// common.cuh -- shared types of the BHPP engine (device graph store, slots, args).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bhpp.h"

namespace bh {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct FallbackNeeded : std::runtime_error {  // bh_edge_list_parse: use the Python loop
    FallbackNeeded() : std::runtime_error("fallback") {}
};
struct InvalidArg : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define BH_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess)                                                             \
            throw ::bh::CudaError(std::string(#call) + ": " + cudaGetErrorString(_e) +     \
                                  " (" __FILE__ ":" + std::to_string(__LINE__) + ")");     \
    } while (0)

void count_launch(int n = 1);

// edge_list.cpp: native text edge-list parser (host)
enum : int { PARSE_OK = 0, PARSE_FALLBACK = 1, PARSE_ERROR = 2 };
struct EdgeListResult {
    std::vector<std::string> u_labels, v_labels;
    std::vector<int64_t> eu, ev;
    std::vector<double> ew;
    int64_t err_line = 0;
    int status = PARSE_OK;
};
EdgeListResult parse_edge_list(const char *buf, int64_t len, const char *delim, int64_t delim_len, bool has_default,
                               double default_weight);

// walks.cu: Monte-Carlo restart walks over the device graph (MCSP forward half)
bh_alias *alias_create(bh_graph *g, const double *u_prob, const int64_t *u_alias, const double *v_prob,
                       const int64_t *v_alias);
void alias_build(int64_t n_rows, int64_t n_e, const int64_t *indptr, const double *weights, int device,
                 double *prob_out, int64_t *alias_out);
void mc_walks(const bh_alias *al, int64_t source, double alpha, int64_t first, int64_t n, uint64_t seed,
              int64_t *counts_host);

// csr_build.cu: device canonicalisation of an edge list (bh_csr_build); 1 = duplicate pair.
int csr_build(int64_t n_u, int64_t n_v, int64_t n_e, const int64_t *edge_u, const int64_t *edge_v,
              const double *edge_w, int64_t *u_indptr, int32_t *u_indices, double *u_weights, int64_t *v_indptr,
              int32_t *v_indices, double *v_weights, double *ws_u, double *ws_v, int device);

// Programmatic dependent launch: every round kernel lets its successor launch
// early (the successor's blocks occupy SMs freed by this kernel's tail) and
// waits for its predecessor's memory before touching round state.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
// The two halves, for kernels that first read immutable graph data (plans, the
// edge stream) under their predecessor's tail.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Static per-warp work of one pull side (rows = this side's nodes): a
// contiguous edge range [e0, e1) chosen by a merge-path split of rows + edges.
// Rows that straddle a range boundary ("cut rows") get one fp64 partial per
// warp; the last warp to arrive adds them in warp order and finishes the row.
struct WarpWork {
    int64_t e0, e1;
    int32_t r0;           // row containing e0
    int32_t cut0, part0;  // cut-row index / partial slot of the first row (-1: whole)
    int32_t cut1, part1;  // same for the last row when it differs from the first
    int32_t pad;
};

struct CutRow {
    int32_t row;
    int32_t n_parts;
    int32_t first_part;
    int32_t pad;
};

// One CSR side of the device store.  Rows and columns are in the store's node
// order: by default both sides are relabelled by descending degree (stable in
// the caller's index), so the hub rows of every gathered operand sit in one
// contiguous slab (L2 residency window) and a warp's consecutive rows share
// hub columns.  Each row keeps the caller's edge order, so every row sum adds
// the same terms in the same order as without relabelling.  perm / inv map
// store index -> caller index and back (null when the caller's order is kept).
// One edge of the dense pulls' stream: column and prescaled value side by side,
// so a lane fetches its edge with one load.  v < 0 marks the last edge of a row
// (values are w / ws(row) > 0), which replaces the row-pointer walk in the pull.
template <typename T>
struct alignas(2 * sizeof(T)) EdgeRF {
    int32_t c;
    T v;
};

struct Side {
    int64_t n_rows = 0;
    int64_t *indptr = nullptr;   // [n_rows + 1]
    int32_t *indices = nullptr;  // [E] column (other side) index, store order
    void *vals = nullptr;        // [E] T, w / ws(row)
    void *ecv = nullptr;         // [E] EdgeRF<T>: (column, value) pairs for the dense pulls, the value
                                 // negated on the last edge of its row (null when some row is empty)
    int32_t *deg = nullptr;      // [n_rows]
    int32_t *perm = nullptr;     // [n_rows] store row -> caller row (null: identity)
    int32_t *inv = nullptr;      // [n_rows] caller row -> store row (null: identity)
    std::vector<int64_t> h_indptr;  // host copy for the per-engine partition
    std::vector<int32_t> h_perm, h_inv;  // host copies (empty: identity)
    // caller -> store row (host)
    int64_t to_store(int64_t r) const { return h_inv.empty() ? r : h_inv[(size_t)r]; }
};

}  // namespace bh

struct bh_graph {
    int device = 0;
    int dtype = BH_DTYPE_F64;
    int64_t n_u = 0, n_v = 0, n_e = 0;
    bh::Side U;  // rows u: cols v, vals w/ws(u)   (u_step, bigraph.py:148-155)
    bh::Side V;  // rows v: cols u, vals w/ws(v)   (v_step, bigraph.py:157-164)
    double *ws_u = nullptr;      // store order
    double *inv_ws_u = nullptr;  // store order
    int relabeled = 0;           // rows / columns in degree order (Side::perm / inv)
    int64_t device_bytes = 0;
    std::mutex mu;
    void *engines = nullptr;  // engine cache (engine.cu)
};

// Device copy of the alias tables of one graph (build_alias, baselines.py:76-80).
struct bh_alias {
    bh_graph *g = nullptr;  // not owned; the caller destroys the tables before the graph
    int device = 0;
    double *u_prob = nullptr, *v_prob = nullptr;
    int32_t *u_alias = nullptr, *v_alias = nullptr;
    ~bh_alias() {
        cudaFree(u_prob);
        cudaFree(v_prob);
        cudaFree(u_alias);
        cudaFree(v_alias);
    }
};

namespace bh {

// ---------------------------------------------------------------------------
// Per-slot round op: what K1 (prep), K2 (V pull) and K3 (U pull) do for this
// slot in the coming round.
enum Op : int32_t {
    OP_IDLE = 0,
    OP_BSEL_INIT = 1,  // ledger := e_src, then a selective round at eps_b
    OP_BSEL = 2,       // selective round at eps_b           (push_engine.py:165)
    OP_SEQ = 3,        // sequential round, threshold 0      (push_engine.py:181)
    OP_FENTRY = 4,     // gamma at entry + forward round     (push_engine.py:222,231)
    OP_FSEL = 5,       // forward round at theta_i           (push_engine.py:231)
    OP_PIENTRY = 6,    // y0 := residue * ysc, first power iteration
    OP_PIENTRY0 = 7,   // y0 only (t == 0)
    OP_PI = 8,         // power iteration
    OP_MEASURE = 9,    // reductions of the uploaded ledger only (pi_push entry gamma)
};

enum Phase : int32_t { PH_IDLE = 0, PH_BSEL, PH_SEQ, PH_FWD, PH_PI, PH_DONE };

// Slot state owned by the control kernel (K4).
struct Slot {
    int32_t op;        // op of the next round
    int32_t job;       // BH_JOB_*
    int32_t qidx;      // query index in the batch, -1 if idle
    int32_t src;       // source / target U index (store order)
    int32_t phase;     // Phase
    int32_t term_b, term_f;
    int32_t src_orig;  // the same in the caller's numbering
    int32_t tie_checks, tie_skip, tie_broke;
    int32_t pi_t, pi_done;
    int32_t last_phase;   // BH_PHASE_* of the last executed push round (-1 none)
    int32_t budget;       // SS-Push budget enabled
    int32_t push_seq;     // incremented after every push round (round_hook trigger)
    int64_t n_p, n_p_entry, n_p_b;
    int64_t sel_b, seq_b, sel_f;
    int64_t last_rounds;  // counter reported to round_hook
    double gamma;
    double mass_prev;       // weighted residue mass at the start of the current forward round
    double defsum;          // sum_j log1p(alpha f_j / (1 - alpha)), f_j = left-behind mass fraction
    double ws_q, inv_ws_q;  // ws(source), 1 / ws(source)
    double ysc;             // y0 = residue * ysc in power iteration
    double theta_c;         // eps_f / lam
    double eps_b, eps_f;
    int32_t near_ties;      // budget checks with relative margin < 1e-12
    double min_margin;      // smallest relative budget margin seen
};

// Finished-query record written by K4 for the finalize kernels.
struct Finish {
    int32_t qidx, src, job, has_pi;  // src: caller's numbering
    double inv_ws_q;
    bh_trace trace;
};

// Deterministic per-round reductions: one row per producing block.
struct Partials {
    int64_t *cnt;    // [rows_k1][B] |A| (K1 push)
    int64_t *np_u;   // [rows_k1][B] sum deg(A) (K1 push)
    double *lmass;   // [rows_k1][B] weighted residue left below threshold (K1, forward)
    int64_t *np_v;   // [rows_k2][B] sum deg over r_v > 0 (K2, one row per warp)
    int32_t *any;    // [rows_k3][B] any(r > threshold) (K1a combine)
    double *sum;     // [rows_k3][B] sum r (K1a)
    double *wsum;    // [rows_k3][B] sum w_ratio * r (K1a)
    int rows_k1, rows_k2, rows_k3;  // valid rows (set by host per launch geometry)
};

struct Control {
    int32_t active;    // slots still busy or queries left
    int32_t next_q;    // next query index to start
    int32_t n_q;       // queries in this batch
    int32_t n_fin;     // slots finishing this round
    int32_t rounds_active;  // rounds K4 processed with work in flight
    int32_t arrive;         // K4 block arrival counter (last block assigns queries)
    int32_t error;          // 1: K4's runaway guard; 2: a source index out of range
    int32_t fin_rounds;     // rounds with a finishing slot (K5 launched under the graph's IF node)
    int32_t fin_slots[256];
    int32_t free_slot[256];
};

constexpr int MAX_B = 128;

}  // namespace bh
