// small.cuh -- the small-graph path: one CTA runs one whole SS-BI-PUSH query.
//
// For graphs whose per-query state fits in shared memory (|U|, |V| up to a few
// thousand: config 1), the slot engine's per-round cost is launch latency
// (five kernels per round, ~40 us) rather than bandwidth.  Here a persistent
// CTA iterates the same round -- K1 push, K2 V pull, K3 U pull, K1a combine,
// K4 control -- with __syncthreads between the phases, keeps r_u, est, the
// pushed vector, r_v and the U-pull output in shared memory, and reads the
// graph through L1.  The per-element arithmetic is the engine's (kernels.cuh
// k_push / k_combine, same threshold forms), the control step is the engine's
// slot_transition (control.cuh), so traces and scores follow the same
// reference semantics (push_engine.py:145-324, bhpp_query.py:160-218).
//
// Frontier (SURVEY K-F, push_engine.py:269-277, 297-302, 315-320): the pulls
// only visit rows that can be non-zero this round.  K1 marks the pushed U
// nodes; a V row is visited only if one of its neighbours was pushed (found by
// walking the pushed rows' U-CSR edges into a bitmap), a U row only if one of
// its V neighbours is non-zero.  Rows outside the frontier are zero, exactly
// as in a full pull; every visited row is summed sequentially in CSR order.
// A round switches to the frontier form when the pushed rows' degree sum is at
// most _SCATTER_LIMIT * |E| (push_engine.py:44; bh_set_scatter_limit, default 0.25).
//
// Work split inside the CTA: rows are cut into chunks of at most SMALL_CHUNK
// edges (host-built item lists, longest first, dealt round-robin to threads);
// a row cut into several chunks adds its partials in chunk order afterwards.
// One CTA per query; a batch launches min(n_q, resident CTAs) CTAs that take
// queries blockIdx.x, blockIdx.x + gridDim.x, ... (deterministic).
#pragma once

#include "control.cuh"
#include "topk.cuh"

namespace bh {

constexpr int SMALL_THREADS = TOPK_THREADS;  // block_select's geometry
constexpr int SMALL_CHUNK = 64;

struct SmallItem {
    int32_t row;
    int32_t len;
    int64_t e0;
    int32_t part;  // -1: whole row; else the chunk's partial slot
    int32_t pad;
};
struct SmallSplit {
    int32_t row, first_part, n_parts, pad;
};

template <typename T>
struct SmallArgs {
    int64_t n_u, n_v, n_e;
    // store-order CSR of both sides (vals = w / ws(row))
    const int64_t *u_ptr, *v_ptr;
    const int32_t *u_col, *v_col;
    const T *u_val, *v_val;
    const int32_t *deg_u;
    const double *ws_u, *inv_ws_u;
    const int32_t *perm_u;  // store -> caller (null: identity)
    // work lists per side
    const SmallItem *items_v, *items_u;
    const SmallSplit *split_v, *split_u;
    int32_t n_items_v, n_items_u, n_split_v, n_split_u, n_parts_v, n_parts_u;
    ControlArgs ca;         // sources, inv_u, tie_skip, trace, ws_u, n_u, alpha, lam, eps, budget
    int32_t n_q, k, exclude, want_scores;
    int32_t *topk_idx;      // [n_q][k]
    double *topk_score;
    bh_trace *trace;        // [n_q]
    double *scores;         // [n_q][n_u] caller order, or null
    double *ledger_r, *ledger_est;  // [n_u] caller order (single-query ledger out), or null
    int64_t max_rounds;
    double scatter_limit;   // _SCATTER_LIMIT * |E| (bh_set_scatter_limit); < 0: dense rounds only
    int32_t *error;         // set to 1 on the runaway guard
};

// Host plan of one graph's small path: the work lists of both pulls.
struct SmallPlan {
    SmallItem *items_v = nullptr, *items_u = nullptr;
    SmallSplit *split_v = nullptr, *split_u = nullptr;
    int32_t n_items_v = 0, n_items_u = 0, n_split_v = 0, n_split_u = 0, n_parts_v = 0, n_parts_u = 0;
    size_t smem = 0;
    int grid_cap = 0;
    int32_t *error = nullptr;
    Control *ctl = nullptr;
    void free_all() {
        cudaFree(items_v); cudaFree(items_u); cudaFree(split_v); cudaFree(split_u); cudaFree(error); cudaFree(ctl);
    }
};

// Shared-memory layout: R EST P Y [n_u] XV [n_v] parts [max parts] in T / double,
// then the frontier bitmaps (one word per 32 rows).
template <typename T>
struct SmallSmem {
    static size_t bytes(int64_t n_u, int64_t n_v, int64_t n_parts) {
        size_t b = (size_t)(4 * n_u + n_v) * sizeof(T);
        b = (b + 15) / 16 * 16;
        b += (size_t)n_parts * sizeof(double);
        b += (size_t)((n_u + 31) / 32 + (n_v + 31) / 32) * sizeof(uint32_t);
        return b;
    }
};

// Block sums of N values at once (fixed shuffle tree, then warp partials in
// warp order): two barriers for all N.  buf: N * (warps + 1) doubles.
template <int N>
__device__ __forceinline__ void small_block_sums(double (&x)[N], double *buf) {
    constexpr int NW = SMALL_THREADS / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < N; i++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x[i] += __shfl_down_sync(0xffffffffu, x[i], o);
        if (lane == 0) buf[i * (NW + 1) + w] = x[i];
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double t = 0.0;
        for (int j = 0; j < NW; j++) t += buf[threadIdx.x * (NW + 1) + j];
        buf[threadIdx.x * (NW + 1) + NW] = t;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < N; i++) x[i] = buf[i * (NW + 1) + NW];
}

// Marks the other-side endpoints of the edges of every active row (bitmap
// `act_rows`) in `act_cols`, walking the side's chunked item list so a hub row's
// edges are spread over many threads.
__device__ __forceinline__ void small_mark(const SmallItem *__restrict__ items, int n_items,
                                           const int32_t *__restrict__ col, const uint32_t *act_rows,
                                           uint32_t *act_cols) {
    for (int it = threadIdx.x; it < n_items; it += SMALL_THREADS) {
        const SmallItem w = items[it];
        if (!((act_rows[w.row >> 5] >> (w.row & 31)) & 1u)) continue;
        for (int64_t e = w.e0; e < w.e0 + w.len; e++) {
            const int32_t c = __ldg(col + e);
            atomicOr(&act_cols[c >> 5], 1u << (c & 31));
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(SMALL_THREADS) k_small_query(SmallArgs<T> a) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    __shared__ SelectSmem sel;
    __shared__ uint64_t skey[TOPK_MAX];
    __shared__ int64_t sidx[TOPK_MAX];
    __shared__ double red_d[3 * (SMALL_THREADS / 32 + 1)];
    __shared__ Slot s_slot;
    __shared__ Finish s_done;
    __shared__ int32_t s_fin, s_sparse_v, s_sparse_u;
    const int tid = threadIdx.x;
    const int64_t nu = a.n_u, nv = a.n_v;
    T *R = (T *)s_raw;
    T *EST = R + nu;
    T *P = EST + nu;
    T *Y = P + nu;
    T *XV = Y + nu;
    double *parts = (double *)(s_raw + ((size_t)(4 * nu + nv) * sizeof(T) + 15) / 16 * 16);
    uint32_t *act_u = (uint32_t *)(parts + (a.n_parts_v > a.n_parts_u ? a.n_parts_v : a.n_parts_u));
    uint32_t *act_v = act_u + (nu + 31) / 32;
    const int nwu = (int)((nu + 31) / 32), nwv = (int)((nv + 31) / 32);
    const double alpha = a.ca.alpha;
    const double one_minus_alpha = 1.0 - alpha;

    for (int32_t q = blockIdx.x; q < a.n_q; q += gridDim.x) {
        if (tid == 0) {
            Slot sl;
            const bool ok = slot_start(sl, a.ca, q);
            s_slot = sl;
            s_fin = ok ? 0 : 2;
        }
        for (int64_t u = tid; u < nu; u += SMALL_THREADS) {
            R[u] = (T)0;
            EST[u] = (T)0;
            P[u] = (T)0;
        }
        __syncthreads();
        if (s_fin == 2) continue;  // rejected source: trace written by slot_start
        int64_t round = 0;
        while (true) {
            const Slot sl = s_slot;
            const int o = sl.op;
            const bool push = op_is_push(o), init = o == OP_BSEL_INIT, fwd = op_is_fwd(o);
            const bool fwdlike = fwd || o == OP_MEASURE;
            const bool entry = o == OP_PIENTRY || o == OP_PIENTRY0;
            const double thA = fwdlike ? sl.ws_q : 0.0, thC = fwdlike ? sl.theta_c : 0.0;
            const double thDp = fwdlike || o == OP_SEQ ? 0.0 : sl.eps_b;
            const double thDa = fwdlike ? 0.0 : sl.eps_b;
            // ---- K1: push decision, pushed vector, |A|, sum deg(A), left-behind mass
            for (int i = tid; i < nwv; i += SMALL_THREADS) act_v[i] = 0u;
            double cnt = 0.0, npu = 0.0, left = 0.0;
            for (int64_t ub = 0; ub < nu; ub += SMALL_THREADS) {  // warp-uniform trip count: ballots below
                const int64_t u = ub + tid;
                bool nz = false;
                if (u < nu) {
                const double iws = a.inv_ws_u[u];
                const double r = init ? (u == sl.src ? 1.0 : 0.0) : (double)R[u];
                const double th = fma(thA * iws, thC, thDp);
                const bool pushed = push && r > th;
                cnt += pushed;
                npu += pushed ? (double)a.deg_u[u] : 0.0;
                if (fwd && !pushed) left += (a.ws_u[u] * sl.inv_ws_q) * r;
                T p = pushed ? (T)r : (T)0;
                if (entry) p = (T)((double)R[u] * sl.ysc);
                if (push || entry) P[u] = p;
                if (init) {
                    R[u] = pushed ? (T)0 : (T)r;
                    EST[u] = (T)(pushed ? 0.0 + alpha * r : 0.0);
                }
                nz = (double)P[u] != 0.0;
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, nz);  // 32 consecutive nodes per warp
                if ((tid & 31) == 0 && u < nu) act_u[u >> 5] = bal;
            }
            {
                double x[3] = {cnt, npu, left};
                small_block_sums<3>(x, red_d);
                cnt = x[0];
                npu = x[1];
                left = x[2];
            }
            // frontier form when the pushed rows are light (push_engine.py:44, 297)
            if (tid == 0) s_sparse_v = (double)npu <= a.scatter_limit && !(o == OP_PI || o == OP_PIENTRY);
            __syncthreads();
            const bool sparse = s_sparse_v;
            if (sparse) {  // N(A): walk the pushed rows' U-CSR edges
                small_mark(a.items_u, a.n_items_u, a.u_col, act_u, act_v);
                __syncthreads();
            }
            // ---- K2: V pull  XV[v] = (1 - alpha) sum_u (w / ws_v) P[u];  n_p += deg(v) for XV > 0
            double npv = 0.0, xdeg = 0.0;  // xdeg: sum deg(v) over XV != 0 (U-side frontier size)
            {
                for (int it = tid; it < a.n_items_v; it += SMALL_THREADS) {
                    const SmallItem w = a.items_v[it];
                    if (sparse && !((act_v[w.row >> 5] >> (w.row & 31)) & 1u)) {
                        if (w.part >= 0) parts[w.part] = 0.0;
                        else XV[w.row] = (T)0;
                        continue;
                    }
                    double acc = 0.0;
                    for (int64_t e = w.e0; e < w.e0 + w.len; e++)
                        acc = fma((double)a.v_val[e], (double)P[a.v_col[e]], acc);
                    if (w.part >= 0) {
                        parts[w.part] = acc;
                    } else {
                        const T out = (T)(one_minus_alpha * acc);
                        XV[w.row] = out;
                        const double dv = (double)(a.v_ptr[w.row + 1] - a.v_ptr[w.row]);
                        if (push && (double)out > 0.0) npv += dv;
                        if ((double)out != 0.0) xdeg += dv;
                    }
                }
                __syncthreads();
                for (int i = tid; i < a.n_split_v; i += SMALL_THREADS) {
                    const SmallSplit sp = a.split_v[i];
                    double tot = 0.0;
                    for (int p = 0; p < sp.n_parts; p++) tot += parts[sp.first_part + p];
                    const T out = (T)(one_minus_alpha * tot);
                    XV[sp.row] = out;
                    const double dv = (double)(a.v_ptr[sp.row + 1] - a.v_ptr[sp.row]);
                    if (push && (double)out > 0.0) npv += dv;
                    if ((double)out != 0.0) xdeg += dv;
                }
                __syncthreads();
            }
            {
                double x[2] = {npv, xdeg};
                small_block_sums<2>(x, red_d);
                npv = x[0];
                xdeg = x[1];
            }
            // U rows to visit: neighbours of the non-zero V rows (walk cost xdeg)
            if (tid == 0) s_sparse_u = sparse && (double)xdeg <= a.scatter_limit;
            __syncthreads();
            const bool sparse_u = s_sparse_u;
            if (sparse_u) {  // rows of the non-zero V rows (bitmap by ballot), then their U neighbours
                for (int i = tid; i < nwu; i += SMALL_THREADS) act_u[i] = 0u;
                for (int64_t vb = 0; vb < nv; vb += SMALL_THREADS) {
                    const int64_t v = vb + tid;
                    const uint32_t bal = __ballot_sync(0xffffffffu, v < nv && (double)XV[v] != 0.0);
                    if ((tid & 31) == 0 && v < nv) act_v[v >> 5] = bal;
                }
                __syncthreads();
                small_mark(a.items_v, a.n_items_v, a.v_col, act_v, act_u);
            }
            __syncthreads();
            // ---- K3: U pull  Y[u] = sum_v (w / ws_u) XV[v]
            for (int it = tid; it < a.n_items_u; it += SMALL_THREADS) {
                const SmallItem w = a.items_u[it];
                if (sparse_u && !((act_u[w.row >> 5] >> (w.row & 31)) & 1u)) {
                    if (w.part >= 0) parts[w.part] = 0.0;
                    else Y[w.row] = (T)0;
                    continue;
                }
                double acc = 0.0;
                for (int64_t e = w.e0; e < w.e0 + w.len; e++)
                    acc = fma((double)a.u_val[e], (double)XV[a.u_col[e]], acc);
                if (w.part >= 0) parts[w.part] = acc;
                else Y[w.row] = (T)acc;
            }
            __syncthreads();
            for (int i = tid; i < a.n_split_u; i += SMALL_THREADS) {
                const SmallSplit sp = a.split_u[i];
                double tot = 0.0;
                for (int p = 0; p < sp.n_parts; p++) tot += parts[sp.first_part + p];
                Y[sp.row] = (T)tot;
            }
            __syncthreads();
            // ---- K1a: combine and exit-test reductions
            const bool m_push = push && !init, m_rw = push, m_stat = push || o == OP_MEASURE;
            const bool m_pi = o == OP_PIENTRY || o == OP_PI;
            double sum = 0.0, wsum = 0.0, anyd = 0.0;
            for (int64_t u = tid; u < nu; u += SMALL_THREADS) {
                const double ws = a.ws_u[u], iws = a.inv_ws_u[u];
                const double r0 = (double)R[u];
                const double y = (double)Y[u];
                const double tA = thA * iws;
                const bool pushed = m_push && r0 > fma(tA, thC, thDp);
                if (pushed) EST[u] = (T)((double)EST[u] + alpha * r0);
                if (m_pi) P[u] = (T)(r0 * sl.ysc + y);
                const T nr = m_rw ? (T)((pushed ? 0.0 : r0) + y) : R[u];
                if (m_rw) R[u] = nr;
                const double r = (double)nr;
                if (m_stat) {
                    sum += r;
                    wsum = fma(ws * sl.inv_ws_q, r, wsum);
                    if (r > fma(tA, thC, thDa)) anyd = 1.0;
                }
            }
            {
                double x[3] = {sum, wsum, anyd};
                small_block_sums<3>(x, red_d);
                sum = x[0];
                wsum = x[1];
                anyd = x[2];
            }
            // ---- K4: the query's state transition (thread 0)
            if (tid == 0) {
                RoundRed red;
                red.cnt = (int64_t)cnt;
                red.np = (int64_t)npu + (int64_t)npv;
                red.sum = sum;
                red.wsum = wsum;
                red.left = left;
                red.any = anyd > 0.0;
                Slot s2 = s_slot;
                Finish f;
                const bool done = slot_transition(s2, o, red, alpha, a.ca.budget_scale, a.ca.log_decay, f);
                s_slot = s2;
                if (done) {
                    s_fin = 1;
                    s_done = f;
                    a.trace[q] = f.trace;
                } else if (++round > a.max_rounds) {
                    s_fin = 1;
                    *a.error = 1;
                }
            }
            __syncthreads();
            if (s_fin) break;
        }
        // ---- K5: beta = (w_ratio est [+ alpha acc_t]) + est, top-k, outputs
        const bool has_pi = s_done.has_pi;
        const double inv_ws_q = s_slot.inv_ws_q;
        for (int64_t u = tid; u < nu; u += SMALL_THREADS) {
            const double est = (double)EST[u];
            const double ws = a.ws_u[u];
            double v = (ws * inv_ws_q) * est;
            if (has_pi) v = v + alpha * (ws * (double)P[u]);
            v = v + est;
            const int64_t cu = a.perm_u ? a.perm_u[u] : u;
            if (a.scores) a.scores[(int64_t)q * nu + cu] = v;
            if (a.ledger_r) {
                a.ledger_r[cu] = (double)R[u];
                a.ledger_est[cu] = est;
            }
            Y[u] = (T)0;
            if constexpr (sizeof(T) == 8) Y[u] = v;  // beta kept for the select (fp64 state)
        }
        __syncthreads();
        if (a.k > 0 && a.topk_idx) {
            const int64_t excl = a.exclude ? (int64_t)s_done.src : -1;
            auto acc = [&](int64_t i, uint64_t &kk, int64_t &ii) -> bool {
                double v;
                if constexpr (sizeof(T) == 8) {
                    v = (double)Y[i];
                } else {
                    const double est = (double)EST[i];
                    const double ws = a.ws_u[i];
                    v = (ws * inv_ws_q) * est;
                    if (has_pi) v = v + alpha * (ws * (double)P[i]);
                    v = v + est;
                }
                kk = order_key(v);
                ii = a.perm_u ? (int64_t)a.perm_u[i] : i;
                return ii != excl;
            };
            int Pp = 1;
            while (Pp < a.k) Pp <<= 1;
            for (int i = tid; i < Pp; i += SMALL_THREADS) {
                skey[i] = 0;
                sidx[i] = INT64_MAX;
            }
            __syncthreads();
            const int64_t m = block_select(nu, a.k, acc, sel, skey, sidx);
            block_sort_pairs(skey, sidx, Pp);
            for (int i = tid; i < a.k; i += SMALL_THREADS) {
                const bool ok = i < m;
                a.topk_idx[(int64_t)q * a.k + i] = ok ? (int32_t)sidx[i] : -1;
                if (a.topk_score) a.topk_score[(int64_t)q * a.k + i] = ok ? key_value(skey[i]) : 0.0;
            }
        }
        __syncthreads();
    }
}

}  // namespace bh
