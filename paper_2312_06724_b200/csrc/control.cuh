// control.cuh -- K4: per-query state machine, one thread per slot.
//
// Mirrors the loop bodies of ss_push (push_engine.py:164-184), selective_push
// (131-142) and pi_push (230-250) plus required_iterations (85-98), evaluated
// on device in fp64 after every round so no host round trip is needed.  Also
// refills finished slots from the query queue in slot order (deterministic).
#pragma once

#include "kernels.cuh"

namespace bh {

struct ControlArgs {
    Slot *slots;
    Finish *fin;
    Control *ctl;
    Partials part;
    const int32_t *sources;   // [n_q], caller's numbering
    const int32_t *inv_u;     // caller -> store U index (null: identity)
    const int32_t *tie_skip;  // [n_q] or null
    bh_trace *trace;          // [n_q]: written here only for a rejected source
    const double *ws_u;
    int64_t n_u;
    double alpha, lam, eps_b, eps_f;
    double budget_scale;  // 2 |E|
    double log_decay;     // log(1 / (1 - alpha))
    int32_t job;
    int32_t power_t;      // BH_JOB_POWER depth
    int64_t init_np;      // BH_JOB_PI_PUSH seed ledger n_p
    int32_t first;        // 1: no round ran yet, only assign queries
    int32_t B;
    int32_t use_cond;     // running inside a CUDA-graph WHILE node: set its condition
    int32_t max_rounds;   // safety stop
    cudaGraphConditionalHandle cond;
    int32_t use_fin_cond; // K5 sits under an IF node: set it when a slot finished
    cudaGraphConditionalHandle fin_cond;
};

__device__ __forceinline__ int32_t required_iterations_dev(double alpha, double eps_f, double mass) {
    if (mass <= 0) return 0;
    double x = ceil(log(mass / eps_f) / log(1.0 / (1.0 - alpha))) - 1.0;
    return x > 0 ? (int32_t)x : 0;
}

// Starts query q in a slot.  A source outside [0, n_u) (device-pointer batches
// are not validated on the host) finishes at once with trace.status =
// BH_EINVAL and flags the batch (ctl->error = 2, reported as BH_EINVAL).
__device__ bool slot_start(Slot &sl, const ControlArgs &a, int32_t q) {
    sl = Slot{};
    sl.qidx = q;
    sl.job = a.job;
    const int32_t s0 = a.sources[q];
    if (s0 < 0 || (int64_t)s0 >= a.n_u) {
        bh_trace t{};
        t.source = s0;
        t.status = BH_EINVAL;
        t.term_b = t.term_f = -1;
        a.trace[q] = t;
        atomicExch(&a.ctl->error, 2);
        sl.qidx = -1;
        sl.op = OP_IDLE;
        sl.phase = PH_IDLE;
        return false;
    }
    sl.src_orig = s0;
    sl.src = a.inv_u ? a.inv_u[s0] : s0;
    sl.tie_skip = a.tie_skip ? a.tie_skip[q] : 0;
    sl.ws_q = a.ws_u[sl.src];
    sl.inv_ws_q = 1.0 / sl.ws_q;
    sl.eps_b = a.eps_b;
    sl.eps_f = a.eps_f;
    sl.theta_c = a.eps_f / a.lam;
    sl.min_margin = 1.0 / 0.0;
    sl.ysc = sl.inv_ws_q;
    sl.last_phase = -1;
    sl.budget = a.job != BH_JOB_SELECTIVE;
    switch (a.job) {
        case BH_JOB_PI_PUSH:
            sl.n_p = a.init_np;
            sl.n_p_entry = a.init_np;
            sl.phase = PH_FWD;
            sl.op = OP_MEASURE;  // gamma of the seed ledger first, then forward rounds
            break;
        case BH_JOB_POWER:
            sl.phase = PH_PI;
            sl.pi_t = a.power_t;
            sl.ysc = 1.0;
            sl.op = a.power_t > 0 ? OP_PIENTRY : OP_PIENTRY0;
            break;
        default:
            sl.phase = PH_BSEL;
            sl.op = OP_BSEL_INIT;
            break;
    }
    return true;
}

__device__ void slot_finish(Slot &sl, Finish &f, bool has_pi) {
    f.qidx = sl.qidx;
    f.src = sl.src_orig;
    f.job = sl.job;
    f.has_pi = has_pi;
    f.inv_ws_q = sl.inv_ws_q;
    bh_trace &t = f.trace;
    t.sel_b = sl.sel_b;
    t.seq_b = sl.seq_b;
    t.n_p_b = sl.n_p_b;
    t.sel_f = sl.sel_f;
    t.pi_iters = sl.pi_t;
    t.n_p_f = sl.n_p;
    t.gamma = sl.gamma;
    t.term_b = sl.term_b;
    t.term_f = sl.term_f;
    t.tie_checks = sl.tie_checks;
    t.tie_broke = sl.tie_broke;
    t.source = sl.src_orig;
    t.status = 0;
    t.near_ties = sl.near_ties;
    t.pad = 0;
    t.min_margin = sl.min_margin;
    sl.phase = PH_DONE;
    sl.op = OP_IDLE;
}

// Near-tie log (SURVEY.md section 7 hard part 1(d)): every budget comparison
// lhs >=/<= rhs records its margin relative to `scale`; those below 1e-12 are
// counted in the trace (a rounding-order change could flip them).
__device__ __forceinline__ void note_margin(Slot &sl, double lhs, double rhs, double scale) {
    const double m = fabs(lhs - rhs) / fmax(fabs(scale), 1.0);
    if (m < sl.min_margin) sl.min_margin = m;
    if (m < 1e-12) sl.near_ties++;
}

// Reductions of one slot's round (K1 push statistics, K2 n_p, K1a exit tests).
struct RoundRed {
    int64_t cnt;   // |A|
    int64_t np;    // sum deg(A) + sum deg(N(A))
    double sum;    // sum r_u after the round
    double wsum;   // sum w_ratio r_u after the round
    double left;   // forward: weighted residue left below threshold
    int32_t any;   // any r_u > threshold after the round
};

// The per-query state transition after a round with op `op` (push_engine.py
// ss_push 164-184, selective_push 131-142, pi_push 230-250, power iteration
// 113-117): counters, exit tests, budget switches (Eq. 10, Eq. 12 in exact
// form), phase changes.  Returns true when the query finished (f written).
__device__ bool slot_transition(Slot &sl, int op, const RoundRed &red, double alpha, double budget_scale,
                                double log_decay, Finish &f) {
    bool fin = false;
    const int64_t cnt = red.cnt;
    const int32_t any = red.any;
    const double sum = red.sum, wsum = red.wsum;
    if (op == OP_MEASURE) {  // pi_push entry: gamma of the uploaded ledger (push_engine.py:222)
        sl.gamma = wsum;
        sl.mass_prev = wsum;
        sl.defsum = 0.0;
        sl.op = OP_FENTRY;
    } else if (op_is_push(op)) {
        sl.push_seq++;
        const int64_t worked = cnt > 0;
        sl.n_p += red.np;
        bool end_backward = false;
        if (op == OP_BSEL_INIT || op == OP_BSEL) {
            sl.sel_b += worked;
            sl.last_phase = BH_PHASE_SELECTIVE;
            sl.last_rounds = sl.sel_b;
            if (!any) {
                sl.term_b = BH_TERM_THRESHOLD;
                end_backward = true;
            } else if (!sl.budget) {
                sl.op = OP_BSEL;
            } else if (sum <= 0.0) {
                sl.term_b = BH_TERM_DRAINED;
                end_backward = true;
            } else {
                const double rhs = budget_scale * (log(1.0 / sum) / log_decay);  // Eq. 10
                note_margin(sl, (double)sl.n_p, rhs, rhs);
                if ((double)sl.n_p >= rhs) {
                    if (sum > sl.eps_b) {  // any is true here
                        sl.op = OP_SEQ;
                        sl.phase = PH_SEQ;
                    } else {
                        sl.term_b = BH_TERM_BUDGET;
                        end_backward = true;
                    }
                } else {
                    sl.op = OP_BSEL;
                }
            }
        } else if (op == OP_SEQ) {
            sl.seq_b += worked;
            sl.last_phase = BH_PHASE_SEQUENTIAL;
            sl.last_rounds = sl.seq_b;
            if (any && sum > sl.eps_b) {
                sl.op = OP_SEQ;
            } else {
                sl.term_b = BH_TERM_BUDGET;
                end_backward = true;
            }
        } else {  // forward round
            sl.sel_f += worked;
            sl.last_phase = BH_PHASE_FORWARD;
            sl.last_rounds = sl.sel_f;
            // Eq. 12 in exact (telescoped) form.  By detailed balance a forward
            // round maps the weighted residue mass m = P + L (P pushed, L left
            // below threshold) to (1-alpha) P + L, so
            //   ln(gamma / wmass_k) = sum_j [ln(1/(1-alpha)) - log1p(alpha f_j / (1-alpha))],
            // f_j = L_j / m_{j-1}.  The budget test n_p - n_0 >= 2|E| ln(gamma/wmass)/ln(1/(1-alpha))
            // becomes (2|E| k - used) <= 2|E| sum_j log1p(...) / ln(1/(1-alpha)): a comparison of
            // two small quantities that fp32 residues resolve as well as fp64 ones.
            const double fj = sl.mass_prev > 0.0 ? red.left / sl.mass_prev : 0.0;
            if (fj > 0.0) sl.defsum += log1p(alpha * fj / (1.0 - alpha));
            sl.mass_prev = wsum;
            if (!any) {
                sl.term_f = BH_TERM_THRESHOLD;
                sl.pi_t = 0;
                fin = true;
                slot_finish(sl, f, false);
            } else if (wsum <= 0.0) {
                sl.term_f = BH_TERM_DRAINED;
                sl.pi_t = 0;
                fin = true;
                slot_finish(sl, f, false);
            } else {
                bool brk;
                const int64_t used = sl.n_p - sl.n_p_entry;
                const int64_t limit = (int64_t)budget_scale * sl.sel_f;  // 2|E| k
                if (sl.defsum == 0.0) {
                    // Every positive residue was pushed in every forward round: the
                    // budget is exactly 2|E| k.  Equality (A = U in every round) is the
                    // exact tie of SURVEY.md sec. 0 fact 11, which the reference resolves
                    // by rounding: break, unless replaying a reference run (tie_skip).
                    if (used >= limit) {
                        sl.tie_checks++;
                        brk = sl.tie_checks > sl.tie_skip;
                        if (brk) sl.tie_broke = 1;
                    } else {
                        brk = false;
                    }
                } else {
                    const double rhs = budget_scale * sl.defsum / log_decay;
                    note_margin(sl, (double)(limit - used), rhs, (double)limit);
                    brk = (double)(limit - used) <= rhs;
                }
                if (brk) {
                    sl.term_f = BH_TERM_BUDGET;
                    sl.pi_t = required_iterations_dev(alpha, sl.eps_f, wsum);
                    sl.pi_done = 0;
                    sl.phase = PH_PI;
                    sl.op = sl.pi_t > 0 ? OP_PIENTRY : OP_PIENTRY0;
                } else {
                    sl.op = OP_FSEL;
                }
            }
        }
        if (end_backward) {
            sl.n_p_b = sl.n_p;
            if (sl.job == BH_JOB_SS_PUSH || sl.job == BH_JOB_SELECTIVE) {
                fin = true;
                slot_finish(sl, f, false);
            } else {
                sl.phase = PH_FWD;
                sl.op = OP_FENTRY;
                sl.gamma = wsum;  // gamma at PI-Push entry (push_engine.py:222)
                sl.mass_prev = wsum;
                sl.defsum = 0.0;
                sl.n_p_entry = sl.n_p;
                sl.tie_checks = 0;
            }
        }
    } else if (op == OP_PIENTRY0) {
        sl.last_phase = -1;
        fin = true;
        slot_finish(sl, f, true);
    } else if (op == OP_PIENTRY || op == OP_PI) {
        sl.last_phase = -1;
        sl.pi_done++;
        if (sl.pi_done >= sl.pi_t) {
            fin = true;
            slot_finish(sl, f, true);
        } else {
            sl.op = OP_PI;
        }
    }
    return fin;
}

constexpr int CONTROL_THREADS = 256;

// One block per slot: deterministic reduction of the slot's partial rows, the
// slot's state transition, then the last block to arrive refills free slots
// from the query queue in slot order and publishes the round's flags.
__global__ void __launch_bounds__(CONTROL_THREADS) k_control(ControlArgs a) {
    pdl_begin();
    constexpr int NW = CONTROL_THREADS / 32;
    __shared__ int64_t w_cnt[NW], w_np[NW];
    __shared__ double w_sum[NW], w_wsum[NW], w_left[NW];
    __shared__ int32_t w_any[NW];
    __shared__ int32_t s_last;
    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    const int s = blockIdx.x;
    const int B = a.B;
    Control *ctl = a.ctl;
    // loads issued before any is used: the activity flag, the slot (thread 0) and
    // the partial rows below are independent
    const int32_t active = ctl->active;
    Slot sl;
    if (tid == 0) sl = a.slots[s];
    // Deterministic reduction of the slot's partial rows: each thread adds a
    // fixed strided subset (4 independent loads in flight), then a fixed-shape
    // shuffle tree per warp and across the warps.
    int64_t cnt = 0, np = 0;
    double sum = 0.0, wsum = 0.0, left = 0.0;
    int32_t any = 0;
    if (!a.first) {
        // partial rows are stored slot-major: [slot][row]; the loads of all six
        // row sets are issued together (one memory round trip for the usual sizes)
        constexpr int U4 = 4, UNP = 20;  // UNP x 256 covers the V pull's per-warp n_p rows (4736 at c2)
        const int64_t *pc = a.part.cnt + (int64_t)s * a.part.rows_k1;
        const int64_t *pn = a.part.np_u + (int64_t)s * a.part.rows_k1;
        const double *pl = a.part.lmass + (int64_t)s * a.part.rows_k1;
        const int64_t *pv = a.part.np_v + (int64_t)s * a.part.rows_k2;
        const int32_t *pa = a.part.any + (int64_t)s * a.part.rows_k3;
        const double *ps = a.part.sum + (int64_t)s * a.part.rows_k3;
        const double *pw = a.part.wsum + (int64_t)s * a.part.rows_k3;
        const int n1 = a.part.rows_k1, n2 = a.part.rows_k2, n3 = a.part.rows_k3;
        for (int it = 0; it * CONTROL_THREADS * U4 < n1 || it * CONTROL_THREADS * UNP < n2 ||
                         it * CONTROL_THREADS * U4 < n3; it++) {
            int64_t c4[U4], n4[U4], nnp[UNP];
            double l4[U4], s4[U4], w4[U4];
            int32_t a4[U4];
#pragma unroll
            for (int j = 0; j < U4; j++) {
                const int r = (it * U4 + j) * CONTROL_THREADS + tid;
                const bool ok1 = r < n1, ok3 = r < n3;
                c4[j] = ok1 ? __ldcg(pc + r) : 0;
                n4[j] = ok1 ? __ldcg(pn + r) : 0;
                l4[j] = ok1 ? __ldcg(pl + r) : 0.0;
                a4[j] = ok3 ? __ldcg(pa + r) : 0;
                s4[j] = ok3 ? __ldcg(ps + r) : 0.0;
                w4[j] = ok3 ? __ldcg(pw + r) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < UNP; j++) {
                const int r = (it * UNP + j) * CONTROL_THREADS + tid;
                nnp[j] = r < n2 ? __ldcg(pv + r) : 0;
            }
#pragma unroll
            for (int j = 0; j < U4; j++) {
                cnt += c4[j];
                np += n4[j];
                left += l4[j];
                any |= a4[j];
                sum += s4[j];
                wsum += w4[j];
            }
#pragma unroll
            for (int j = 0; j < UNP; j++) np += nnp[j];
        }
    }
    if (active == 0 && !a.first) {
        if (s == 0 && tid == 0) {
            ctl->n_fin = 0;
            if (a.use_cond) cudaGraphSetConditional(a.cond, 0);
            if (a.use_fin_cond) cudaGraphSetConditional(a.fin_cond, 0);
        }
        return;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        cnt += __shfl_down_sync(0xffffffffu, cnt, off);
        np += __shfl_down_sync(0xffffffffu, np, off);
        sum += __shfl_down_sync(0xffffffffu, sum, off);
        wsum += __shfl_down_sync(0xffffffffu, wsum, off);
        left += __shfl_down_sync(0xffffffffu, left, off);
        any |= __shfl_down_sync(0xffffffffu, any, off);
    }
    if (lane == 0) {
        w_cnt[wid] = cnt;
        w_np[wid] = np;
        w_sum[wid] = sum;
        w_wsum[wid] = wsum;
        w_left[wid] = left;
        w_any[wid] = any;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < NW; w++) {
            w_cnt[0] += w_cnt[w];
            w_np[0] += w_np[w];
            w_sum[0] += w_sum[w];
            w_wsum[0] += w_wsum[w];
            w_left[0] += w_left[w];
            w_any[0] |= w_any[w];
        }
    }
    if (tid == 0) {
        RoundRed red;
        red.cnt = w_cnt[0];
        red.np = w_np[0];
        red.sum = w_sum[0];
        red.wsum = w_wsum[0];
        red.left = w_left[0];
        red.any = w_any[0];
        const int op = a.first ? OP_IDLE : sl.op;
        const bool fin = slot_transition(sl, op, red, a.alpha, a.budget_scale, a.log_decay, a.fin[s]);
        const bool free_now = fin || sl.op == OP_IDLE;
        if (free_now) sl.qidx = fin ? sl.qidx : -1;
        a.slots[s] = sl;
        // a slot that finished this round is refilled one round later: K5 reads its
        // columns concurrently with the next round's K1 (which would initialise them)
        ctl->free_slot[s] = (free_now && !fin ? 1 : 0) | (fin ? 2 : 0);
        __threadfence();
        // arrival count in the low 16 bits, free slots above: the last block
        // learns whether any slot needs the refill pass
        const int32_t prev = atomicAdd(&ctl->arrive, 1 + (free_now ? (1 << 16) : 0));
        const int32_t now = prev + 1 + (free_now ? (1 << 16) : 0);
        s_last = (now & 0xffff) == B ? 1 + (now >> 16) : 0;
    }
    __syncthreads();
    if (!s_last) return;
    if (s_last == 1 && !a.first) {  // no slot freed this round: all stay busy, nothing to refill
        if (tid == 0) {
            ctl->n_fin = 0;
            ctl->rounds_active++;
            int32_t busy = 1;
            if (ctl->rounds_active > a.max_rounds) {  // runaway guard (never expected)
                busy = 0;
                ctl->error = 1;
            }
            ctl->active = busy;
            ctl->arrive = 0;
            if (a.use_cond) cudaGraphSetConditional(a.cond, busy ? 1u : 0u);
            if (a.use_fin_cond) cudaGraphSetConditional(a.fin_cond, 0);
            __threadfence();
        }
        return;
    }
    // last block: refill free slots in slot order (prefix count), publish flags
    __threadfence();
    // slot-order prefix counts of the free / finishing slots (ballots per warp)
    __shared__ int32_t w_free[MAX_B / 32], w_fin[MAX_B / 32];
    volatile Control *vc = ctl;
    int32_t my_free = 0, my_fin = 0, pre_free = 0, pre_fin = 0;
    if (tid < B) {
        const int32_t f = vc->free_slot[tid];
        my_free = f & 1;
        my_fin = (f >> 1) & 1;
    }
    const uint32_t b_free = __ballot_sync(0xffffffffu, my_free), b_fin = __ballot_sync(0xffffffffu, my_fin);
    if (lane == 0 && wid < MAX_B / 32) {
        w_free[wid] = __popc(b_free);
        w_fin[wid] = __popc(b_fin);
    }
    __syncthreads();
    const uint32_t below = (1u << lane) - 1u;
    pre_free = __popc(b_free & below);
    pre_fin = __popc(b_fin & below);
    int32_t nfree = 0, nfin = 0;
    for (int w = 0; w < (B + 31) / 32; w++) {
        if (w < wid) {
            pre_free += w_free[w];
            pre_fin += w_fin[w];
        }
        nfree += w_free[w];
        nfin += w_fin[w];
    }
    const int32_t next0 = vc->next_q, n_q = vc->n_q;
    int32_t busy = 0;
    if (tid < B) {
        if (my_fin) ctl->fin_slots[pre_fin] = tid;
        const int32_t q = next0 + pre_free;
        if (my_free && q < n_q) {
            Slot ns;
            slot_start(ns, a, q);
            a.slots[tid] = ns;
            busy = ns.op != OP_IDLE;
        } else {
            if (my_free) a.slots[tid].qidx = -1;
            busy = *(volatile int32_t *)&a.slots[tid].op != OP_IDLE;
        }
    }
    busy = __syncthreads_or(busy) || next0 + nfree < n_q;  // queries left for the draining slots
    if (tid == 0) {
        ctl->next_q = min(n_q, next0 + nfree);
        ctl->n_fin = nfin;
        ctl->fin_rounds += nfin > 0;
        if (a.use_fin_cond) cudaGraphSetConditional(a.fin_cond, nfin > 0 ? 1u : 0u);
        if (!a.first) ctl->rounds_active++;
        if (ctl->rounds_active > a.max_rounds) {  // runaway guard (never expected)
            busy = 0;
            ctl->error = 1;
        }
        ctl->active = busy;
        ctl->arrive = 0;
        if (a.use_cond) cudaGraphSetConditional(a.cond, busy ? 1u : 0u);
        __threadfence();
    }
}

}  // namespace bh
