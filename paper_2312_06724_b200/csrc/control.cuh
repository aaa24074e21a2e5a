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
    const int32_t *sources;   // [n_q]
    const int32_t *tie_skip;  // [n_q] or null
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
};

__device__ __forceinline__ int32_t required_iterations_dev(double alpha, double eps_f, double mass) {
    if (mass <= 0) return 0;
    double x = ceil(log(mass / eps_f) / log(1.0 / (1.0 - alpha))) - 1.0;
    return x > 0 ? (int32_t)x : 0;
}

__device__ void slot_start(Slot &sl, const ControlArgs &a, int32_t q) {
    sl = Slot{};
    sl.qidx = q;
    sl.job = a.job;
    sl.src = a.sources[q];
    sl.tie_skip = a.tie_skip ? a.tie_skip[q] : 0;
    sl.ws_q = a.ws_u[sl.src];
    sl.inv_ws_q = 1.0 / sl.ws_q;
    sl.eps_b = a.eps_b;
    sl.eps_f = a.eps_f;
    sl.theta_c = a.eps_f / a.lam;
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
}

__device__ void slot_finish(Slot &sl, Finish &f, bool has_pi) {
    f.qidx = sl.qidx;
    f.src = sl.src;
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
    t.source = sl.src;
    t.status = 0;
    sl.phase = PH_DONE;
    sl.op = OP_IDLE;
}

constexpr int CONTROL_THREADS = 256;

// One block per slot: deterministic reduction of the slot's partial rows, the
// slot's state transition, then the last block to arrive refills free slots
// from the query queue in slot order and publishes the round's flags.
__global__ void __launch_bounds__(CONTROL_THREADS) k_control(ControlArgs a) {
    pdl_begin();
    __shared__ int64_t r_cnt[CONTROL_THREADS];
    __shared__ int64_t r_np[CONTROL_THREADS];
    __shared__ double r_sum[CONTROL_THREADS];
    __shared__ double r_wsum[CONTROL_THREADS];
    __shared__ int32_t r_any[CONTROL_THREADS];
    __shared__ double r_left[CONTROL_THREADS];
    __shared__ int32_t s_last;
    const int tid = threadIdx.x;
    const int s = blockIdx.x;
    const int B = a.B;
    Control *ctl = a.ctl;
    if (ctl->active == 0 && !a.first) {
        if (s == 0 && tid == 0) {
            ctl->n_fin = 0;
            if (a.use_cond) cudaGraphSetConditional(a.cond, 0);
        }
        return;
    }
    {
        int64_t cnt = 0, np = 0;
        double sum = 0.0, wsum = 0.0;
        int32_t any = 0;
        double left = 0.0;
        if (!a.first) {
            // partial rows are stored slot-major: [slot][row]
            const int64_t *pc = a.part.cnt + (int64_t)s * a.part.rows_k1;
            const int64_t *pn = a.part.np_u + (int64_t)s * a.part.rows_k1;
            const double *pl = a.part.lmass + (int64_t)s * a.part.rows_k1;
            for (int r = tid; r < a.part.rows_k1; r += CONTROL_THREADS) {
                cnt += pc[r];
                np += pn[r];
                left += pl[r];
            }
            const int64_t *pv = a.part.np_v + (int64_t)s * a.part.rows_k2;
            for (int r = tid; r < a.part.rows_k2; r += CONTROL_THREADS) np += pv[r];
            const int32_t *pa = a.part.any + (int64_t)s * a.part.rows_k3;
            const double *ps = a.part.sum + (int64_t)s * a.part.rows_k3;
            const double *pw = a.part.wsum + (int64_t)s * a.part.rows_k3;
            for (int r = tid; r < a.part.rows_k3; r += CONTROL_THREADS) {
                any |= pa[r];
                sum += ps[r];
                wsum += pw[r];
            }
        }
        r_cnt[tid] = cnt;
        r_np[tid] = np;
        r_sum[tid] = sum;
        r_wsum[tid] = wsum;
        r_any[tid] = any;
        r_left[tid] = left;
    }
    __syncthreads();
    for (int off = CONTROL_THREADS / 2; off > 0; off >>= 1) {  // fixed-shape tree
        if (tid < off) {
            r_cnt[tid] += r_cnt[tid + off];
            r_np[tid] += r_np[tid + off];
            r_sum[tid] += r_sum[tid + off];
            r_wsum[tid] += r_wsum[tid + off];
            r_any[tid] |= r_any[tid + off];
            r_left[tid] += r_left[tid + off];
        }
        __syncthreads();
    }
    if (tid == 0) {
        Slot sl = a.slots[s];
        bool fin = false;
        const int op = a.first ? OP_IDLE : sl.op;
        const int64_t cnt = r_cnt[0];
        const int32_t any = r_any[0];
        const double sum = r_sum[0], wsum = r_wsum[0];
        if (op == OP_MEASURE) {  // pi_push entry: gamma of the uploaded ledger (push_engine.py:222)
            sl.gamma = wsum;
            sl.mass_prev = wsum;
            sl.defsum = 0.0;
            sl.op = OP_FENTRY;
        } else if (op_is_push(op)) {
            sl.push_seq++;
            const int64_t worked = cnt > 0;
            sl.n_p += r_np[0];
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
                } else if ((double)sl.n_p >= a.budget_scale * (log(1.0 / sum) / a.log_decay)) {
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
                const double fj = sl.mass_prev > 0.0 ? r_left[0] / sl.mass_prev : 0.0;
                if (fj > 0.0) sl.defsum += log1p(a.alpha * fj / (1.0 - a.alpha));
                sl.mass_prev = wsum;
                if (!any) {
                    sl.term_f = BH_TERM_THRESHOLD;
                    sl.pi_t = 0;
                    fin = true;
                    slot_finish(sl, a.fin[s], false);
                } else if (wsum <= 0.0) {
                    sl.term_f = BH_TERM_DRAINED;
                    sl.pi_t = 0;
                    fin = true;
                    slot_finish(sl, a.fin[s], false);
                } else {
                    bool brk;
                    const int64_t used = sl.n_p - sl.n_p_entry;
                    const int64_t limit = (int64_t)a.budget_scale * sl.sel_f;  // 2|E| k
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
                        brk = (double)(limit - used) <= a.budget_scale * sl.defsum / a.log_decay;
                    }
                    if (brk) {
                        sl.term_f = BH_TERM_BUDGET;
                        sl.pi_t = required_iterations_dev(a.alpha, sl.eps_f, wsum);
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
                    slot_finish(sl, a.fin[s], false);
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
            slot_finish(sl, a.fin[s], true);
        } else if (op == OP_PIENTRY || op == OP_PI) {
            sl.last_phase = -1;
            sl.pi_done++;
            if (sl.pi_done >= sl.pi_t) {
                fin = true;
                slot_finish(sl, a.fin[s], true);
            } else {
                sl.op = OP_PI;
            }
        }
        const bool free_now = fin || sl.op == OP_IDLE;
        if (free_now) sl.qidx = fin ? sl.qidx : -1;
        a.slots[s] = sl;
        ctl->free_slot[s] = (free_now ? 1 : 0) | (fin ? 2 : 0);
        __threadfence();
        s_last = atomicAdd(&ctl->arrive, 1) == B - 1;
    }
    __syncthreads();
    if (!s_last) return;
    // last block: refill free slots in slot order (prefix count), publish flags
    __threadfence();
    __shared__ int32_t f_free[MAX_B], f_fin[MAX_B], pre_free[MAX_B], pre_fin[MAX_B];
    volatile Control *vc = ctl;
    if (tid < B) {
        const int32_t f = vc->free_slot[tid];
        f_free[tid] = f & 1;
        f_fin[tid] = (f >> 1) & 1;
    }
    __syncthreads();
    if (tid == 0) {
        int32_t a1 = 0, a2 = 0;
        for (int i = 0; i < B; i++) {
            pre_free[i] = a1;
            pre_fin[i] = a2;
            a1 += f_free[i];
            a2 += f_fin[i];
        }
        s_last = a2;  // reuse: number finishing
    }
    __syncthreads();
    const int32_t next0 = vc->next_q, n_q = vc->n_q;
    int32_t busy = 0;
    if (tid < B) {
        if (f_fin[tid]) ctl->fin_slots[pre_fin[tid]] = tid;
        const int32_t q = next0 + pre_free[tid];
        if (f_free[tid] && q < n_q) {
            Slot ns;
            slot_start(ns, a, q);
            a.slots[tid] = ns;
            busy = ns.op != OP_IDLE;
        } else {
            if (f_free[tid]) a.slots[tid].qidx = -1;
            busy = *(volatile int32_t *)&a.slots[tid].op != OP_IDLE;
        }
    }
    busy = __syncthreads_or(busy);
    if (tid == 0) {
        int32_t nfree = 0;
        for (int i = 0; i < B; i++) nfree += f_free[i];
        ctl->next_q = min(n_q, next0 + nfree);
        ctl->n_fin = s_last;
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
