// small.cuh -- the small-graph path: one thread-block cluster runs one whole
// SS-BI-PUSH query.
//
// For graphs whose per-query state fits in shared memory (|U|, |V| up to a few
// thousand: config 1), the slot engine's per-round cost is launch latency
// (five kernels per round, ~40 us) rather than bandwidth.  Here a persistent
// cluster of CL CTAs (default 8, distributed shared memory) iterates the same
// round -- K1 push, K2 V pull, K3 U pull, K1a combine, K4 control -- with
// cluster barriers between the phases.  The per-element arithmetic is the
// engine's (kernels.cuh k_push / k_combine, same threshold forms), the control
// step is the engine's slot_transition (control.cuh), so traces and scores
// follow the same reference semantics (push_engine.py:145-324,
// bhpp_query.py:160-218).
//
// Why a cluster: one CTA spent 78 % of a c1 round in the two pulls, latency-
// bound on the graph (240 KB of (col, val) for c1 in fp64 does not fit beside
// the state in one SM's L1, so every item costs L2 round trips).  Split over
// CL CTAs, each CTA's rows and edges are 1 / CL of the graph; each CTA stages
// its slice -- (col, val) of its rows and its work items -- in shared memory
// once per launch (a cluster barrier invalidates L1, so relying on L1 would
// re-read the slice from L2 every round), when the slice fits.
//
// Ownership: CTA r owns a contiguous slice of U rows and one of V rows
// (balanced on edges + rows, host plan).  Every CTA keeps full copies of the
// two gathered vectors in its shared memory -- the pushed vector P (gathered
// by the V pull) and r_v = XV (gathered by the U pull); the owner of a row
// writes its value into all CL copies (st.shared::cluster) -- and its own
// slices of r_u, est and the U-pull output Y.  Per round: K1 (own U slice, P
// to all copies) | cluster barrier | V pull (own V rows, XV to all copies) |
// cluster barrier | U pull + K1a (own U rows; power-iteration iterates go to
// all P copies) | per-CTA partial sums to every CTA | cluster barrier | every
// CTA sums the CL partials in rank order and runs the same slot_transition
// (identical inputs, identical state, no broadcast).  Work items: rows cut into
// chunks of at most SMALL_CHUNK edges (dealt round-robin to threads, longest
// first); a row cut into several chunks adds its partials in chunk order.
// Each cluster takes queries cid, cid + n_clusters, ... (deterministic).
//
// Rounds are always dense here: each CTA's share of a round is ~1 / CL of the
// graph from shared memory, so the frontier's bookkeeping would cost more than it saves
// (the slot engine's K-F path covers sparse rounds, frontier.cuh).
#pragma once

#include <cooperative_groups.h>

#include "control.cuh"
#include "topk.cuh"

namespace bh {

constexpr int SMALL_THREADS = TOPK_THREADS;  // block_select's geometry
constexpr int SMALL_CHUNK = 64;
constexpr int SMALL_MAX_CL = 16;
constexpr int SMALL_NRED = 8;  // partial sums per CTA and round

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
    // per-CTA work: rank r's rows [slice[r], slice[r+1]), items [ioff[r], ioff[r+1]),
    // split rows [soff[r], soff[r+1]) of each side
    const int32_t *u_slice, *v_slice;
    const int32_t *iu_off, *iv_off, *su_off, *sv_off;
    const SmallItem *items_v, *items_u;
    const SmallSplit *split_v, *split_u;
    int32_t n_parts_v, n_parts_u;
    ControlArgs ca;         // sources, inv_u, tie_skip, trace, ws_u, n_u, alpha, lam, eps, budget
    int32_t n_q, k, exclude, want_scores;
    int32_t *topk_idx;      // [n_q][k]
    double *topk_score;
    bh_trace *trace;        // [n_q]
    double *scores;         // [n_q][n_u] caller order, or null
    double *ledger_r, *ledger_est;  // [n_u] caller order (single-query ledger out), or null
    int64_t max_rounds;
    int32_t *error;         // set to 1 on the runaway guard
    // staged graph slices: each CTA copies its rows' (col, val) and work items into
    // shared memory once per launch (cluster barriers flush L1, so the graph would
    // otherwise be re-read from L2 every round); capacities = max over ranks
    int32_t stage, cap_ev, cap_eu, cap_iv, cap_iu;
    unsigned long long *prof;  // diagnostic: per-phase clock64 cycles of CTA 0 (null: off)
};

// Host plan of one graph's small path: the work lists of both pulls, per rank.
struct SmallPlan {
    SmallItem *items_v = nullptr, *items_u = nullptr;
    SmallSplit *split_v = nullptr, *split_u = nullptr;
    int32_t *offs = nullptr;  // u_slice, v_slice, iu_off, iv_off, su_off, sv_off: 6 x (CL + 1)
    int32_t n_parts_v = 0, n_parts_u = 0;
    int32_t stage = 0, cap_ev = 0, cap_eu = 0, cap_iv = 0, cap_iu = 0;
    int cl = 8;
    size_t smem = 0;
    int cluster_cap = 0;  // clusters resident at once
    int32_t *error = nullptr;
    Control *ctl = nullptr;
    void free_all() {
        cudaFree(items_v); cudaFree(items_u); cudaFree(split_v); cudaFree(split_u); cudaFree(offs);
        cudaFree(error); cudaFree(ctl);
    }
};

// Shared-memory layout: R EST P Y [n_u] XV [n_v] in T, parts [max parts] and
// the partial sums of every rank [SMALL_MAX_CL][SMALL_NRED] in double; with
// staging, then the rank's items (V, U), vals (V, U) and cols (V, U).
template <typename T>
struct SmallSmem {
    static size_t bytes(int64_t n_u, int64_t n_v, int64_t n_parts) {
        size_t b = (size_t)(4 * n_u + n_v) * sizeof(T);
        b = (b + 15) / 16 * 16;
        b += (size_t)n_parts * sizeof(double);
        b += (size_t)SMALL_MAX_CL * SMALL_NRED * sizeof(double);
        return b;
    }
    static size_t staged(int64_t cap_ev, int64_t cap_eu, int64_t cap_iv, int64_t cap_iu) {
        size_t b = (size_t)(cap_iv + cap_iu) * sizeof(SmallItem);
        b += (size_t)(cap_ev + cap_eu) * sizeof(T);
        b = (b + 15) / 16 * 16;
        b += (size_t)(cap_ev + cap_eu) * sizeof(int32_t);
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

// Dot product of one item's edges (graph slice in shared or global memory) with
// the shared-memory operand: four independent fp64 accumulators added in a
// fixed order (deterministic).
template <typename T>
__device__ __forceinline__ double small_row_dot(const int32_t *__restrict__ col, const T *__restrict__ val,
                                                const T *x, int64_t e0, int32_t len) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int64_t e1 = e0 + len;
    int64_t e = e0;
    for (; e + 4 <= e1; e += 4) {
        const int32_t c0 = col[e], c1 = col[e + 1], c2 = col[e + 2], c3 = col[e + 3];
        const T v0 = val[e], v1 = val[e + 1], v2 = val[e + 2], v3 = val[e + 3];
        a0 = fma((double)v0, (double)x[c0], a0);
        a1 = fma((double)v1, (double)x[c1], a1);
        a2 = fma((double)v2, (double)x[c2], a2);
        a3 = fma((double)v3, (double)x[c3], a3);
    }
    for (; e < e1; e++) a0 = fma((double)val[e], (double)x[col[e]], a0);
    return (a0 + a1) + (a2 + a3);
}

// Writes element i of a replicated shared vector into every CTA's copy.
template <typename T>
__device__ __forceinline__ void small_put_all(cooperative_groups::cluster_group &cl, T *base, int64_t i, T v,
                                              int n_cta) {
    for (int r = 0; r < n_cta; r++) cl.map_shared_rank(base, r)[i] = v;
}

template <typename T>
__global__ void __launch_bounds__(SMALL_THREADS) k_small_query(SmallArgs<T> a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char s_raw[];
    __shared__ SelectSmem sel;
    __shared__ uint64_t skey[TOPK_MAX];
    __shared__ int64_t sidx[TOPK_MAX];
    __shared__ double red_d[SMALL_NRED * (SMALL_THREADS / 32 + 1)];
    __shared__ Slot s_slot;
    __shared__ Finish s_done;
    __shared__ int32_t s_fin;
    const int tid = threadIdx.x;
    const int n_cta = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int cid = blockIdx.x / n_cta, n_clusters = gridDim.x / n_cta;
    const int64_t nu = a.n_u, nv = a.n_v;
    T *R = (T *)s_raw;
    T *EST = R + nu;
    T *P = EST + nu;
    T *Y = P + nu;
    T *XV = Y + nu;
    double *parts = (double *)(s_raw + ((size_t)(4 * nu + nv) * sizeof(T) + 15) / 16 * 16);
    double *rred = parts + (a.n_parts_v > a.n_parts_u ? a.n_parts_v : a.n_parts_u);  // [SMALL_MAX_CL][NRED]
    const int u0 = a.u_slice[rank], u1 = a.u_slice[rank + 1];
    const SmallItem *items_v = a.items_v + a.iv_off[rank];
    const SmallItem *items_u = a.items_u + a.iu_off[rank];
    const int n_items_v = a.iv_off[rank + 1] - a.iv_off[rank];
    const int n_items_u = a.iu_off[rank + 1] - a.iu_off[rank];
    // graph operands of the pulls: global, or this rank's staged slice (edge index
    // e of an item maps to e - base there)
    const int32_t *vcol = a.v_col, *ucol = a.u_col;
    const T *vval = a.v_val, *uval = a.u_val;
    int64_t vbase = 0, ubase = 0;
    if (a.stage) {
        const int v0 = a.v_slice[rank], v1 = a.v_slice[rank + 1];
        vbase = a.v_ptr[v0];
        ubase = a.u_ptr[u0];
        const int64_t nev = a.v_ptr[v1] - vbase, neu = a.u_ptr[u1] - ubase;
        SmallItem *si_v = (SmallItem *)(rred + SMALL_MAX_CL * SMALL_NRED);
        SmallItem *si_u = si_v + a.cap_iv;
        T *sv_v = (T *)(si_u + a.cap_iu);
        T *sv_u = sv_v + a.cap_ev;
        int32_t *sc_v = (int32_t *)((unsigned char *)s_raw +
                                    ((size_t)((unsigned char *)(sv_u + a.cap_eu) - s_raw) + 15) / 16 * 16);
        int32_t *sc_u = sc_v + a.cap_ev;
        for (int i = tid; i < n_items_v; i += SMALL_THREADS) si_v[i] = items_v[i];
        for (int i = tid; i < n_items_u; i += SMALL_THREADS) si_u[i] = items_u[i];
        for (int64_t e = tid; e < nev; e += SMALL_THREADS) {
            sc_v[e] = __ldg(a.v_col + vbase + e);
            sv_v[e] = __ldg(a.v_val + vbase + e);
        }
        for (int64_t e = tid; e < neu; e += SMALL_THREADS) {
            sc_u[e] = __ldg(a.u_col + ubase + e);
            sv_u[e] = __ldg(a.u_val + ubase + e);
        }
        items_v = si_v;
        items_u = si_u;
        vcol = sc_v;
        ucol = sc_u;
        vval = sv_v;
        uval = sv_u;
        __syncthreads();
    }
    const SmallSplit *split_v = a.split_v + a.sv_off[rank];
    const SmallSplit *split_u = a.split_u + a.su_off[rank];
    const int n_split_v = a.sv_off[rank + 1] - a.sv_off[rank];
    const int n_split_u = a.su_off[rank + 1] - a.su_off[rank];
    const double alpha = a.ca.alpha;
    const double one_minus_alpha = 1.0 - alpha;
    long long t_prev = clock64();
    auto probe = [&](int ph) {
        if (a.prof && blockIdx.x == 0 && tid == 0) {
            const long long t = clock64();
            a.prof[ph] += (unsigned long long)(t - t_prev);
            t_prev = t;
        }
    };

    for (int32_t q = cid; q < a.n_q; q += n_clusters) {
        if (tid == 0) {
            Slot sl;
            const bool ok = slot_start(sl, a.ca, q);  // identical in every CTA
            s_slot = sl;
            s_fin = ok ? 0 : 2;
        }
        for (int64_t u = tid; u < nu; u += SMALL_THREADS) {
            R[u] = (T)0;
            EST[u] = (T)0;
            P[u] = (T)0;
        }
        cl.sync();  // every copy clean before any CTA writes this query's P
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
            // ---- K1 (own U rows): push decision, pushed vector to every copy of P
            double cnt = 0.0, npu = 0.0, left = 0.0;
            for (int64_t u = u0 + tid; u < u1; u += SMALL_THREADS) {
                const double iws = a.inv_ws_u[u];
                const double r = init ? (u == sl.src ? 1.0 : 0.0) : (double)R[u];
                const double th = fma(thA * iws, thC, thDp);
                const bool pushed = push && r > th;
                cnt += pushed;
                npu += pushed ? (double)a.deg_u[u] : 0.0;
                if (fwd && !pushed) left += (a.ws_u[u] * sl.inv_ws_q) * r;
                T p = pushed ? (T)r : (T)0;
                if (entry) p = (T)((double)R[u] * sl.ysc);
                if (push || entry) small_put_all(cl, P, u, p, n_cta);
                if (init) {
                    R[u] = pushed ? (T)0 : (T)r;
                    EST[u] = (T)(pushed ? 0.0 + alpha * r : 0.0);
                }
            }
            probe(0);
            cl.sync();  // P complete in every copy
            probe(1);
            // ---- K2 (own V rows): XV[v] = (1 - alpha) sum_u (w / ws_v) P[u] to every copy
            double npv = 0.0;
            for (int it = tid; it < n_items_v; it += SMALL_THREADS) {
                const SmallItem w = items_v[it];
                const double acc = small_row_dot(vcol, vval, P, w.e0 - vbase, w.len);
                if (w.part >= 0) {
                    parts[w.part] = acc;
                } else {
                    const T out = (T)(one_minus_alpha * acc);
                    small_put_all(cl, XV, w.row, out, n_cta);
                    if (push && (double)out > 0.0) npv += (double)(a.v_ptr[w.row + 1] - a.v_ptr[w.row]);
                }
            }
            __syncthreads();
            for (int i = tid; i < n_split_v; i += SMALL_THREADS) {
                const SmallSplit sp = split_v[i];
                double tot = 0.0;
                for (int p = 0; p < sp.n_parts; p++) tot += parts[sp.first_part + p];
                const T out = (T)(one_minus_alpha * tot);
                small_put_all(cl, XV, sp.row, out, n_cta);
                if (push && (double)out > 0.0) npv += (double)(a.v_ptr[sp.row + 1] - a.v_ptr[sp.row]);
            }
            probe(2);
            cl.sync();  // XV complete in every copy
            probe(3);
            // ---- K3 (own U rows): Y[u] = sum_v (w / ws_u) XV[v]
            for (int it = tid; it < n_items_u; it += SMALL_THREADS) {
                const SmallItem w = items_u[it];
                const double acc = small_row_dot(ucol, uval, XV, w.e0 - ubase, w.len);
                if (w.part >= 0) parts[w.part] = acc;
                else Y[w.row] = (T)acc;
            }
            __syncthreads();
            for (int i = tid; i < n_split_u; i += SMALL_THREADS) {
                const SmallSplit sp = split_u[i];
                double tot = 0.0;
                for (int p = 0; p < sp.n_parts; p++) tot += parts[sp.first_part + p];
                Y[sp.row] = (T)tot;
            }
            __syncthreads();
            probe(4);
            // ---- K1a (own U rows): combine and exit-test reductions
            const bool m_push = push && !init, m_rw = push, m_stat = push || o == OP_MEASURE;
            const bool m_pi = o == OP_PIENTRY || o == OP_PI;
            double sum = 0.0, wsum = 0.0, anyd = 0.0;
            for (int64_t u = u0 + tid; u < u1; u += SMALL_THREADS) {
                const double ws = a.ws_u[u], iws = a.inv_ws_u[u];
                const double r0 = (double)R[u];
                const double y = (double)Y[u];
                const double tA = thA * iws;
                const bool pushed = m_push && r0 > fma(tA, thC, thDp);
                if (pushed) EST[u] = (T)((double)EST[u] + alpha * r0);
                if (m_pi) small_put_all(cl, P, u, (T)(r0 * sl.ysc + y), n_cta);  // the iterate, every copy
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
                double x[7] = {cnt, npu, left, npv, sum, wsum, anyd};
                small_block_sums<7>(x, red_d);
                if (tid < n_cta) {  // this CTA's partials into every CTA's table, row = rank
                    double *dst = cl.map_shared_rank(rred, tid) + rank * SMALL_NRED;
#pragma unroll
                    for (int i = 0; i < 7; i++) dst[i] = x[i];
                }
            }
            probe(5);
            cl.sync();  // every CTA holds every rank's partials
            // ---- K4: the query's state transition, identical in every CTA
            if (tid == 0) {
                double x[7] = {0, 0, 0, 0, 0, 0, 0};
                for (int r = 0; r < n_cta; r++)
#pragma unroll
                    for (int i = 0; i < 7; i++) x[i] += rred[r * SMALL_NRED + i];
                RoundRed red;
                red.cnt = (int64_t)x[0];
                red.np = (int64_t)x[1] + (int64_t)x[3];
                red.sum = x[4];
                red.wsum = x[5];
                red.left = x[2];
                red.any = x[6] > 0.0;
                Slot s2 = s_slot;
                Finish f;
                const bool done = slot_transition(s2, o, red, alpha, a.ca.budget_scale, a.ca.log_decay, f);
                s_slot = s2;
                if (done) {
                    s_fin = 1;
                    s_done = f;
                    if (rank == 0) a.trace[q] = f.trace;
                } else if (++round > a.max_rounds) {
                    s_fin = 1;
                    if (rank == 0) *a.error = 1;
                }
            }
            __syncthreads();
            probe(6);
            if (s_fin) break;
        }
        // ---- K5: beta = (w_ratio est [+ alpha acc_t]) + est on own rows; est to
        // CTA 0's copy for the top-k there
        const bool has_pi = s_done.has_pi;
        const double inv_ws_q = s_slot.inv_ws_q;
        T *est0 = cl.map_shared_rank(EST, 0);
        for (int64_t u = u0 + tid; u < u1; u += SMALL_THREADS) {
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
            if (rank != 0) est0[u] = EST[u];
        }
        cl.sync();  // CTA 0 holds est of every row (P is replicated)
        if (rank == 0 && a.k > 0 && a.topk_idx) {
            const int64_t excl = a.exclude ? (int64_t)s_done.src : -1;
            auto acc = [&](int64_t i, uint64_t &kk, int64_t &ii) -> bool {
                const double est = (double)EST[i];
                const double ws = a.ws_u[i];
                double v = (ws * inv_ws_q) * est;
                if (has_pi) v = v + alpha * (ws * (double)P[i]);
                v = v + est;
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
