// kernels.cuh -- device kernels of one push / power-iteration round over a
// block of B query slots (node-major, slot-minor state: X[node * B + slot]).
//
// Round = K1 push -> K2 V-pull -> K3 U-pull -> K1a combine -> K4 control
//         [-> K5 finalize/score chunks -> K6 top-k merge, when a slot finishes]
//
// Reference semantics (pkg/src/bipush/push_engine.py):
//   K1   _push_u bookkeeping (294-309): A = {r_u > theta}, est[A] += alpha r_u,
//        r_u[A] = 0, n_p += sum deg(A); the pushed amounts go to P.
//   K2   _push_u's r_v = (1-alpha) * v_step @ dense (303-306) as a pull over
//        V-CSR; n_p += deg(v) for r_v > 0 (the flushed set, 312-324).
//   K3   _flush_v's u_step @ r_v (322) as a pull over U-CSR -> Y.
//   K1a  r_u += Y, plus the per-query reductions the exit tests need
//        (any r_u > theta, sum r_u, sum w_ratio r_u; 168-177, 234-243).
//   Power iteration (101-117) runs the same K2/K3 pair on a = acc / ws:
//        a <- y0 + U (1-alpha) V a   (detailed balance).
//
// The pulls are gather-bound SpMMs: every edge reads one B-wide operand row
// (B * sizeof(T) bytes).  Each warp owns a contiguous, cost-balanced edge range
// (merge-path over rows + edges, built per engine) and keeps S operand rows in
// flight in registers (k_pull_sw: (col, val) windows and row ends staged in
// shared memory), accumulating in fp64 (fp32 mode: fp32 FMAs over at most 16
// edges, flushed to fp64).  Rows cut by a range boundary are finished by the
// last warp to arrive, which adds the fp64 partials in warp order.  Every row
// sum is therefore a fixed-order accumulation and every per-query reduction
// goes through per-block partial rows summed in a fixed order: bitwise
// deterministic.
#pragma once

#include <cuda.h>

#include <type_traits>

#include "common.cuh"

namespace bh {

// ---------------------------------------------------------------------------
// small helpers

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

template <typename T, int VEC>
struct VecIO;

template <>
struct VecIO<float, 1> {
    static __device__ __forceinline__ void ld(const float *p, float (&v)[1]) { v[0] = *p; }
    static __device__ __forceinline__ void st(float *p, const float (&v)[1]) { *p = v[0]; }
};
template <>
struct VecIO<float, 2> {
    static __device__ __forceinline__ void ld(const float *p, float (&v)[2]) {
        float2 t = *reinterpret_cast<const float2 *>(p);
        v[0] = t.x; v[1] = t.y;
    }
    static __device__ __forceinline__ void st(float *p, const float (&v)[2]) {
        *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
    }
};
template <>
struct VecIO<float, 4> {
    static __device__ __forceinline__ void ld(const float *p, float (&v)[4]) {
        float4 t = *reinterpret_cast<const float4 *>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    static __device__ __forceinline__ void st(float *p, const float (&v)[4]) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <>
struct VecIO<float, 8> {
    static __device__ __forceinline__ void ld(const float *p, float (&v)[8]) {
        const float4 a = *reinterpret_cast<const float4 *>(p);
        const float4 b = *(reinterpret_cast<const float4 *>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
    static __device__ __forceinline__ void st(float *p, const float (&v)[8]) {
        reinterpret_cast<float4 *>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4 *>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
};
template <>
struct VecIO<double, 1> {
    static __device__ __forceinline__ void ld(const double *p, double (&v)[1]) { v[0] = *p; }
    static __device__ __forceinline__ void st(double *p, const double (&v)[1]) { *p = v[0]; }
};
template <>
struct VecIO<double, 2> {
    static __device__ __forceinline__ void ld(const double *p, double (&v)[2]) {
        double2 t = *reinterpret_cast<const double2 *>(p);
        v[0] = t.x; v[1] = t.y;
    }
    static __device__ __forceinline__ void st(double *p, const double (&v)[2]) {
        *reinterpret_cast<double2 *>(p) = make_double2(v[0], v[1]);
    }
};
template <>
struct VecIO<double, 4> {
    static __device__ __forceinline__ void ld(const double *p, double (&v)[4]) {
        double2 a = *reinterpret_cast<const double2 *>(p);
        double2 b = *(reinterpret_cast<const double2 *>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
    static __device__ __forceinline__ void st(double *p, const double (&v)[4]) {
        reinterpret_cast<double2 *>(p)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2 *>(p)[1] = make_double2(v[2], v[3]);
    }
};

template <>
struct VecIO<double, 8> {
    static __device__ __forceinline__ void ld(const double *p, double (&v)[8]) {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const double2 t = *(reinterpret_cast<const double2 *>(p) + k);
            v[2 * k] = t.x;
            v[2 * k + 1] = t.y;
        }
    }
    static __device__ __forceinline__ void st(double *p, const double (&v)[8]) {
#pragma unroll
        for (int k = 0; k < 4; k++) reinterpret_cast<double2 *>(p)[k] = make_double2(v[2 * k], v[2 * k + 1]);
    }
};

__device__ __forceinline__ bool op_is_push(int op) { return op >= OP_BSEL_INIT && op <= OP_FSEL; }
__device__ __forceinline__ bool op_is_fwd(int op) { return op == OP_FENTRY || op == OP_FSEL; }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// cp.async of one element (8 or 16 bytes) into shared memory; !valid zero-fills.
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(uint32_t dst, const void *src, bool valid) {
    static_assert(BYTES == 8 || BYTES == 16, "cp.async element size");
    const int sz = valid ? BYTES : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(dst), "l"(src), "n"(BYTES), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// Elementwise kernels over [n_u x B]: one thread per (node, EV consecutive slots).
constexpr int ELEM_THREADS = 256;

template <int B>
struct ElemGeo {
    static constexpr int EV = B >= 4 ? 4 : B;   // slots per thread
    static constexpr int TPN = B / EV;          // threads per node
};

// Frontier-round control (frontier.cuh): K1's decision and the K-F kernels' gates.
struct FrontCtl {
    unsigned long long deg_acc;   // sum over blocks and slots of sum deg(A_s) (K1)
    unsigned long long edges_v;   // sum deg over the V list (Fb)
    unsigned long long edges_u;   // sum deg over the U list (Fd)
    int64_t limit;                // frontier iff deg_acc <= limit; < 0: never
    int64_t rounds_front;         // rounds whose V half ran frontier
    int64_t rounds_ufront;        // rounds whose U half ran frontier
    int32_t ticket;               // K1 block arrival counter
    int32_t mode;                 // 1: this round is a frontier round
    int32_t gate_dense, gate_front, gate_ufront, gate_udense;
    int32_t zero_all_v, zero_all_u;  // XV / Y may be non-zero outside the item lists
    int32_t n_items_v, n_items_u, n_parts_v, n_parts_u;
    int32_t old_items_v, old_items_u;  // lists of the previous frontier round (Fa)
};

// K1's last block: the round's mode, gates and graph condition.
__device__ __forceinline__ void front_decide(FrontCtl *f, const int32_t *ops, int B, bool use_cond,
                                             cudaGraphConditionalHandle cond) {
    bool push = false, dense_op = false;
    for (int s = 0; s < B; s++) {
        const int o = ops[s];
        push |= op_is_push(o);
        dense_op |= !(o == OP_IDLE || o == OP_MEASURE || op_is_push(o));
    }
    const unsigned long long d = atomicAdd(&f->deg_acc, 0ull);
    const bool front = push && !dense_op && f->limit >= 0 && d <= (unsigned long long)f->limit;
    f->deg_acc = 0;
    f->ticket = 0;
    f->mode = front;
    f->gate_front = front;
    f->gate_dense = !front;
    f->gate_ufront = 0;
    f->gate_udense = 0;
    if (front) {
        f->rounds_front++;
        f->old_items_v = f->n_items_v;
        f->old_items_u = f->n_items_u;
        f->n_items_v = f->n_items_u = f->n_parts_v = f->n_parts_u = 0;
        f->edges_v = 0;
    } else {
        f->zero_all_v = f->zero_all_u = 1;
    }
    if (use_cond) cudaGraphSetConditional(cond, front ? 1u : 0u);
}

template <typename T>
struct ElemArgs {
    int64_t n_u;
    T *R;
    T *P;
    T *Y;
    T *EST;
    const int32_t *deg_u;
    const double *ws_u;
    const double *inv_ws_u;
    const double *x0;  // BH_JOB_POWER start vectors [n_q][n_u], caller's numbering
    const int32_t *perm_u;  // store -> caller U index (null: identity)
    const Slot *slots;
    const int32_t *active;
    Partials part;
    double alpha;
    // frontier rounds (frontier.cuh; k_push<..., FRONT = true> only)
    FrontCtl *front;
    uint8_t *flag_u;  // [n_u] some slot pushed u this round
    cudaGraphConditionalHandle fcond;
    int32_t use_fcond;
};

// Per-slot constants of K1 / K1a in shared memory, element-major: the v-th slot
// of the thread group g sits at [v * TPN + g], so the 16 slot groups of a warp
// read 16 consecutive doubles per LDS (no bank conflicts).  The thresholds are
// folded into one form, th = fma(thA * iws, thC, thD):
//   forward / measure: thA = ws_q, thC = eps_f / lam, thD = 0 -> (ws_q / ws_u)(eps_f / lam)
//   selective:         thA = thC = 0, thD = eps_b;  sequential push: thD = 0
// (fma(x, c, 0) rounds like x * c, so the forward threshold is bit-identical to
// (ws_q * iws) * thc).  thDp: push threshold, thDa: exit-test threshold.
struct ElemSlotC {
    double thA[MAX_B], thC[MAX_B], thDp[MAX_B], thDa[MAX_B], iwsq[MAX_B], ysc[MAX_B];
    int32_t op[MAX_B], src[MAX_B], qidx[MAX_B];
};

template <int B>
__device__ __forceinline__ void load_elem_consts(ElemSlotC &c, const Slot *__restrict__ slots) {
    using EG = ElemGeo<B>;
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        const Slot &sl = slots[s];
        const int o = sl.op;
        const bool fwdlike = op_is_fwd(o) || o == OP_MEASURE;
        const int pidx = (s % EG::EV) * EG::TPN + s / EG::EV;
        c.thA[pidx] = fwdlike ? sl.ws_q : 0.0;
        c.thC[pidx] = fwdlike ? sl.theta_c : 0.0;
        c.thDp[pidx] = fwdlike || o == OP_SEQ ? 0.0 : sl.eps_b;
        c.thDa[pidx] = fwdlike ? 0.0 : sl.eps_b;
        c.iwsq[pidx] = sl.inv_ws_q;
        c.ysc[pidx] = sl.ysc;
        c.op[s] = o;
        c.src[s] = sl.src;
        c.qidx[s] = sl.qidx;
    }
}

// K1: push (and ledger init / power-iteration entry) for the coming round:
// P = r on A = {r > th}, 0 elsewhere, and the per-slot |A|, sum deg(A) and the
// forward left-behind mass.  r_A := 0 and est_A += alpha r_A are left to K1a,
// which re-takes the same decision on the same r; only the ledger-initialising
// round writes r and est here.  Per element the work is predicated (the slots
// of one warp are in different phases), loads of UNR nodes are in flight.
template <int B, typename T, int ELEM_UNR = 4, int MINB = 1, bool PIPE = false, bool FRONT = false>
__global__ void __launch_bounds__(ELEM_THREADS, MINB) k_push(ElemArgs<T> a) {
    pdl_begin();
    if (*a.active == 0) {
        if (FRONT && blockIdx.x == 0 && threadIdx.x == 0) {  // batch over: close every gate
            a.front->gate_front = a.front->gate_dense = 0;
            a.front->gate_ufront = a.front->gate_udense = 0;
        }
        return;
    }
    using EG = ElemGeo<B>;
    constexpr int EV = EG::EV, TPN = EG::TPN;
    __shared__ ElemSlotC sc;
    __shared__ int64_t red_cnt[ELEM_THREADS * EV];
    __shared__ int64_t red_np[ELEM_THREADS * EV];
    __shared__ double red_left[ELEM_THREADS * EV];
    __shared__ unsigned long long blk_deg;
    if (threadIdx.x == 0) blk_deg = 0;
    load_elem_consts<B>(sc, a.slots);
    __syncthreads();
    const int grp = threadIdx.x % TPN;
    const int j0 = grp * EV;  // first slot of this thread (fixed: blockDim % TPN == 0)
    uint32_t m_push = 0, m_init = 0, m_fwd = 0, m_entry = 0, m_x0 = 0, m_keep = 0;
#pragma unroll
    for (int v = 0; v < EV; v++) {
        const int o = sc.op[j0 + v];
        const bool x0 = a.x0 && sc.qidx[j0 + v] >= 0;
        m_push |= (uint32_t)op_is_push(o) << v;
        m_init |= (uint32_t)(o == OP_BSEL_INIT) << v;
        m_fwd |= (uint32_t)op_is_fwd(o) << v;
        m_entry |= (uint32_t)(o == OP_PIENTRY || o == OP_PIENTRY0) << v;
        m_x0 |= (uint32_t)((o == OP_PIENTRY || o == OP_PIENTRY0) && x0) << v;
    }
    m_keep = ((1u << EV) - 1u) & ~(m_push | m_entry);  // P kept (iterate / idle)
    int32_t cnt[EV];  // nodes per thread < 2^31
    int64_t npu[EV];
    double left[EV];
#pragma unroll
    for (int v = 0; v < EV; v++) {
        cnt[v] = 0;
        npu[v] = 0;
        left[v] = 0.0;
    }
    // RARE: ledger-initialising slots or raw power-iteration starts in this
    // thread's group (one round per query); the common body has neither
    auto run = [&](auto rare_tag) {
        constexpr bool RARE = decltype(rare_tag)::value;
        auto node = [&](int64_t u, T (&rv)[EV], double iwsv, double wsv, int32_t degv, unsigned live) {
            const int64_t i = u * B + j0;
            const double iws = iwsv;
            T pv[EV];
            bool act[EV];
            double rr[EV];
#pragma unroll
            for (int v = 0; v < EV; v++) {
                const int c = v * TPN + grp;
                const bool push = (m_push >> v) & 1u;
                const bool init = RARE && ((m_init >> v) & 1u);
                const double r = init ? (u == sc.src[j0 + v] ? 1.0 : 0.0) : (double)rv[v];
                const double th = fma(sc.thA[c] * iws, sc.thC[c], sc.thDp[c]);
                const bool pushed = push && r > th;
                act[v] = pushed;
                rr[v] = r;
                cnt[v] += pushed;
                npu[v] += pushed ? degv : 0;
                if (((m_fwd >> v) & 1u) && !pushed)
                    left[v] += (wsv * sc.iwsq[c]) * r;  // w_ratio r left behind this round
                T p = pushed ? (T)r : (T)0;
                if ((m_entry >> v) & 1u) {
                    // y0 = (w_ratio r) / ws = r / ws(q) (PI-Push tail, push_engine.py:246), or
                    // start / ws for a raw power iteration (push_engine.py:112 on a = acc / ws)
                    p = (T)((double)rv[v] * sc.ysc[c]);
                    if (RARE && ((m_x0 >> v) & 1u)) {
                        p = (T)(a.x0[(int64_t)sc.qidx[j0 + v] * a.n_u + (a.perm_u ? a.perm_u[u] : u)] * iws);
                        rv[v] = p;
                    }
                }
                if (init) rv[v] = pushed ? (T)0 : (T)r;
                pv[v] = p;
            }
            if constexpr (FRONT) {  // frontier flag: some slot pushed u (the node's TPN lanes combined)
                bool anyp = false;
#pragma unroll
                for (int v = 0; v < EV; v++) anyp |= act[v];
                if constexpr (TPN == 1) {
                    a.flag_u[u] = anyp;
                } else {
                    const unsigned bal = __ballot_sync(live, anyp);
                    const int lane = threadIdx.x & 31;
                    const unsigned gm = (TPN == 32 ? 0xffffffffu : ((1u << (TPN % 32)) - 1u)) << ((lane / TPN) * TPN % 32);
                    if ((lane % TPN) == 0) a.flag_u[u] = (bal & gm) != 0u;
                }
            }
            if (m_keep) {  // slots whose P is kept (iterate / idle) are not written
#pragma unroll
                for (int v = 0; v < EV; v++)
                    if (!((m_keep >> v) & 1u)) a.P[i + v] = pv[v];
            } else {
                VecIO<T, EV>::st(a.P + i, pv);
            }
            if constexpr (RARE) {
                VecIO<T, EV>::st(a.R + i, rv);
                if (m_init) {  // ledger reset: est := alpha r on the pushed nodes of init slots
                    T ev[EV];
                    VecIO<T, EV>::ld(a.EST + i, ev);
#pragma unroll
                    for (int v = 0; v < EV; v++)
                        if ((m_init >> v) & 1u) ev[v] = (T)(act[v] ? 0.0 + a.alpha * rr[v] : 0.0);
                    VecIO<T, EV>::st(a.EST + i, ev);
                }
            }
        };
        auto load = [&](int64_t u, T (&rv)[EV], double &iwsv, double &wsv, int32_t &degv) {
            VecIO<T, EV>::ld(a.R + u * B + j0, rv);
            iwsv = a.inv_ws_u[u];
            wsv = m_fwd ? a.ws_u[u] : 0.0;
            degv = a.deg_u[u];
        };
        const int64_t total = a.n_u * TPN;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        const int64_t first = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        if constexpr (PIPE) {  // the next node's loads in flight while this one computes
            T rn[EV];
            double in = 0.0, wn = 0.0;
            int32_t dn = 0;
            if (first < total) load(first / TPN, rn, in, wn, dn);
            for (int64_t t = first; FRONT ? __any_sync(0xffffffffu, t < total) : t < total; t += stride) {
                const unsigned live = FRONT ? __ballot_sync(0xffffffffu, t < total) : 0u;
                if (t >= total) continue;
                T rv[EV];
#pragma unroll
                for (int v = 0; v < EV; v++) rv[v] = rn[v];
                const double iwsv = in, wsv = wn;
                const int32_t degv = dn;
                if (t + stride < total) load((t + stride) / TPN, rn, in, wn, dn);
                node(t / TPN, rv, iwsv, wsv, degv, live);
            }
        } else {
            for (int64_t t0 = first; FRONT ? __any_sync(0xffffffffu, t0 < total) : t0 < total; t0 += ELEM_UNR * stride) {
                T rv[ELEM_UNR][EV];
                double iwsk[ELEM_UNR], wsk[ELEM_UNR];
                int32_t degk[ELEM_UNR];
#pragma unroll
                for (int k = 0; k < ELEM_UNR; k++) {
                    const int64_t t = t0 + k * stride;
                    if (t < total) load(t / TPN, rv[k], iwsk[k], wsk[k], degk[k]);
                }
#pragma unroll
                for (int k = 0; k < ELEM_UNR; k++) {
                    const int64_t t = t0 + k * stride;
                    const unsigned live = FRONT ? __ballot_sync(0xffffffffu, t < total) : 0u;
                    if (FRONT ? !live : t >= total) break;
                    if (t < total) node(t / TPN, rv[k], iwsk[k], wsk[k], degk[k], live);
                }
            }
        }
    };
    // warp-uniform choice (the frontier flag combines the lanes of a node by ballot):
    // lanes whose own slots have no work run the loop with empty masks
    if constexpr (FRONT) {
        if (__any_sync(0xffffffffu, (m_init | m_x0) != 0u)) run(std::true_type{});
        else if (__any_sync(0xffffffffu, (m_push | m_entry) != 0u)) run(std::false_type{});
    } else {
        if (m_init | m_x0) run(std::true_type{});
        else if (m_push | m_entry) run(std::false_type{});
    }
#pragma unroll
    for (int v = 0; v < EV; v++) {
        red_cnt[threadIdx.x * EV + v] = cnt[v];
        red_np[threadIdx.x * EV + v] = npu[v];
        red_left[threadIdx.x * EV + v] = left[v];
    }
    __syncthreads();
    // slot s is owned by the threads t with t % TPN == s / EV
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        int64_t c = 0, n = 0;
        double l = 0.0;
        for (int t = s / EV; t < ELEM_THREADS; t += TPN) {
            c += red_cnt[t * EV + s % EV];
            n += red_np[t * EV + s % EV];
            l += red_left[t * EV + s % EV];
        }
        a.part.cnt[(int64_t)s * gridDim.x + blockIdx.x] = c;
        a.part.np_u[(int64_t)s * gridDim.x + blockIdx.x] = n;
        a.part.lmass[(int64_t)s * gridDim.x + blockIdx.x] = l;
        if constexpr (FRONT) atomicAdd(&blk_deg, (unsigned long long)n);
    }
    if constexpr (FRONT) {  // frontier decision: the last block to arrive (frontier.cuh)
        __shared__ int last;
        __syncthreads();
        if (threadIdx.x == 0) {
            atomicAdd(&a.front->deg_acc, blk_deg);
            __threadfence();
            last = atomicAdd(&a.front->ticket, 1) == (int)gridDim.x - 1;
        }
        __syncthreads();
        if (last && threadIdx.x == 0) {
            __threadfence();
            front_decide(a.front, sc.op, B, a.use_fcond != 0, a.fcond);
        }
    }
}

// K1a: combine r_u += Y (push slots) / a = y0 + Y (power-iteration slots), and
// the exit-test reductions of the round that just ran.  For push slots it also
// completes K1's push: the nodes over threshold (same decision, same r) have
// their residue replaced by Y and est += alpha r.  Per element predicated.
template <int B, typename T, int ELEM_UNR = 4, int MINB = 1, bool PIPE = false>
__global__ void __launch_bounds__(ELEM_THREADS, MINB) k_combine(ElemArgs<T> a) {
    pdl_begin();
    if (*a.active == 0) return;
    using EG = ElemGeo<B>;
    constexpr int EV = EG::EV, TPN = EG::TPN;
    __shared__ ElemSlotC sc;
    __shared__ double red_sum[ELEM_THREADS * EV];
    __shared__ double red_wsum[ELEM_THREADS * EV];
    __shared__ int32_t red_any[ELEM_THREADS * EV];
    load_elem_consts<B>(sc, a.slots);
    __syncthreads();
    const int grp = threadIdx.x % TPN;
    const int j0 = grp * EV;
    uint32_t m_push = 0, m_rw = 0, m_stat = 0, m_pi = 0;
#pragma unroll
    for (int v = 0; v < EV; v++) {
        const int o = sc.op[j0 + v];
        m_push |= (uint32_t)(op_is_push(o) && o != OP_BSEL_INIT) << v;  // pushed by K1 this round
        m_rw |= (uint32_t)op_is_push(o) << v;                            // r_u += Y
        m_stat |= (uint32_t)(op_is_push(o) || o == OP_MEASURE) << v;     // exit-test reductions
        m_pi |= (uint32_t)(o == OP_PIENTRY || o == OP_PI) << v;          // a = y0 + Y
    }
    double sum[EV], wsum[EV];
    int32_t any[EV];
#pragma unroll
    for (int v = 0; v < EV; v++) {
        sum[v] = wsum[v] = 0.0;
        any[v] = 0;
    }
    // one node's elements (EV slots)
    auto node = [&](int64_t u, T (&rv)[EV], const T (&yv)[EV], T (&ev)[EV], double ws, double iws) {
        const int64_t i = u * B + j0;
        bool wrote_e = false;
#pragma unroll
        for (int v = 0; v < EV; v++) {
            const int c = v * TPN + grp;
            const double r0 = (double)rv[v];
            const double y = (double)yv[v];
            const double tA = sc.thA[c] * iws;
            const bool pushed = ((m_push >> v) & 1u) && r0 > fma(tA, sc.thC[c], sc.thDp[c]);
            if (pushed) {
                ev[v] = (T)((double)ev[v] + a.alpha * r0);
                wrote_e = true;
            }
            if ((m_pi >> v) & 1u) a.P[i + v] = (T)(r0 * sc.ysc[c] + y);
            const T nr = ((m_rw >> v) & 1u) ? (T)((pushed ? 0.0 : r0) + y) : rv[v];
            rv[v] = nr;
            const double r = (double)nr;
            const bool st = (m_stat >> v) & 1u;
            if (st) sum[v] += r;
            if (st) wsum[v] = fma(ws * sc.iwsq[c], r, wsum[v]);  // w_ratio * r  (push_engine.py:220,237)
            any[v] |= st && r > fma(tA, sc.thC[c], sc.thDa[c]);
        }
        if (m_rw) VecIO<T, EV>::st(a.R + i, rv);
        if (wrote_e) VecIO<T, EV>::st(a.EST + i, ev);
    };
    auto load = [&](int64_t u, T (&rv)[EV], T (&yv)[EV], T (&ev)[EV], double &ws, double &iws) {
        VecIO<T, EV>::ld(a.R + u * B + j0, rv);
        VecIO<T, EV>::ld(a.Y + u * B + j0, yv);
        if (m_push) VecIO<T, EV>::ld(a.EST + u * B + j0, ev);
        ws = a.ws_u[u];
        iws = a.inv_ws_u[u];
    };
    if (m_stat | m_pi) {
        const int64_t total = a.n_u * TPN;
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        const int64_t first = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        if constexpr (PIPE) {
            // software pipeline: the next node's loads are in flight while this one computes
            T rn[EV], yn[EV], en[EV];
            double wn = 0.0, in = 0.0;
            if (first < total) load(first / TPN, rn, yn, en, wn, in);
            for (int64_t t = first; t < total; t += stride) {
                T rv[EV], yv[EV], ev[EV];
#pragma unroll
                for (int v = 0; v < EV; v++) {
                    rv[v] = rn[v];
                    yv[v] = yn[v];
                    ev[v] = en[v];
                }
                const double ws = wn, iws = in;
                if (t + stride < total) load((t + stride) / TPN, rn, yn, en, wn, in);
                node(t / TPN, rv, yv, ev, ws, iws);
            }
        } else {
            for (int64_t t0 = first; t0 < total; t0 += ELEM_UNR * stride) {
                T rv[ELEM_UNR][EV], yv[ELEM_UNR][EV], ev[ELEM_UNR][EV];
                double wsk[ELEM_UNR], iwsk[ELEM_UNR];
#pragma unroll
                for (int k = 0; k < ELEM_UNR; k++) {
                    const int64_t t = t0 + k * stride;
                    if (t < total) load(t / TPN, rv[k], yv[k], ev[k], wsk[k], iwsk[k]);
                }
#pragma unroll
                for (int k = 0; k < ELEM_UNR; k++) {
                    const int64_t t = t0 + k * stride;
                    if (t >= total) break;
                    node(t / TPN, rv[k], yv[k], ev[k], wsk[k], iwsk[k]);
                }
            }
        }
    }
#pragma unroll
    for (int v = 0; v < EV; v++) {
        red_sum[threadIdx.x * EV + v] = sum[v];
        red_wsum[threadIdx.x * EV + v] = wsum[v];
        red_any[threadIdx.x * EV + v] = any[v];
    }
    __syncthreads();
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        double su = 0.0, ws = 0.0;
        int32_t an = 0;
        for (int t = s / EV; t < ELEM_THREADS; t += TPN) {
            su += red_sum[t * EV + s % EV];
            ws += red_wsum[t * EV + s % EV];
            an |= red_any[t * EV + s % EV];
        }
        a.part.sum[(int64_t)s * gridDim.x + blockIdx.x] = su;
        a.part.wsum[(int64_t)s * gridDim.x + blockIdx.x] = ws;
        a.part.any[(int64_t)s * gridDim.x + blockIdx.x] = an;
    }
}

// ---------------------------------------------------------------------------
// K2 / K3: pipelined pull SpMM.
enum : int { SIDE_V = 0, SIDE_U = 1 };

constexpr int PULL_THREADS = 256;
constexpr int PULL_WARPS = PULL_THREADS / 32;

template <typename T>
struct PullArgs {
    const int64_t *indptr;
    int64_t n_rows;
    const int32_t *indices;
    const T *vals;
    const WarpWork *work;  // [n_warps]
    const CutRow *cuts;
    int32_t *cut_count;    // [n_cuts], zero between launches
    double *scratch;       // [n_parts][B]
    int32_t n_warps;
    const T *X;            // operand: P (V pull) or XV (U pull)
    T *Y;                  // V pull: XV ; U pull: Y
    const Slot *slots;
    const int32_t *active;
    int64_t *np_v;         // [n_warps][B] (V pull)
    double one_minus_alpha;
    const void *ecv;       // [E] EdgeRF<T> (k_pull_rf)
};

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int VEC>
struct DVec {
    double v[VEC];
};
template <int VEC>
struct IVec {
    int64_t v[VEC];
};

// Operand-row gather.  Plain coherent loads (ld.global, L1-cached): the
// operand was written by the previous kernel of the round.
template <typename T, int VEC>
__device__ __forceinline__ void ldg_vec(const T *p, T (&v)[VEC]) {
    VecIO<T, VEC>::ld(p, v);
}

// Pipeline depth (edges in flight per warp): registers hold S operand rows.
template <int B, typename T>
struct RegPipe {
    static constexpr int VEC = B / 32;
    static constexpr int LANE_BYTES = VEC * (int)sizeof(T);
    static constexpr int S = (sizeof(T) == 4 && LANE_BYTES <= 8) ? 16 : (LANE_BYTES <= 16 ? 8 : 4);
};

// Rare path of the pull: a row cut by a warp-range boundary.  Publishes this
// warp's fp64 partial; the last warp to arrive adds the partials in warp order
// and writes the row.  Returns the row's n_p contribution (V pull) per slot.
template <typename T>
struct CutCtx {
    double *scratch;
    int32_t *cut_count;
    const CutRow *cuts;
    T *Y;
    const int64_t *indptr;
    double scale;  // (1 - alpha) on the V side, 1 on the U side
};

template <int B, typename T, int VEC>
__device__ __noinline__ IVec<VEC> pull_cut(CutCtx<T> cx, int ci, int pi, int slot0, uint32_t cmask, DVec<VEC> acc) {
    const int lane = threadIdx.x & 31;
    IVec<VEC> inc;
#pragma unroll
    for (int v = 0; v < VEC; v++) inc.v[v] = 0;
#pragma unroll
    for (int v = 0; v < VEC; v++) cx.scratch[(int64_t)pi * B + slot0 + v] = acc.v[v];
    __threadfence();
    __syncwarp();
    const CutRow cr = cx.cuts[ci];
    int last = 0;
    if (lane == 0) last = atomicAdd(cx.cut_count + ci, 1) == cr.n_parts - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return inc;
    __threadfence();
    double tot[VEC];
#pragma unroll
    for (int v = 0; v < VEC; v++) tot[v] = 0.0;
    int p = 0;
    for (; p + 4 <= cr.n_parts; p += 4) {  // 4 partials in flight
        double q[4][VEC];
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int v = 0; v < VEC; v++) q[k][v] = __ldcg(cx.scratch + (int64_t)(cr.first_part + p + k) * B + slot0 + v);
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int v = 0; v < VEC; v++) tot[v] += q[k][v];
    }
    for (; p < cr.n_parts; p++)
#pragma unroll
        for (int v = 0; v < VEC; v++) tot[v] += __ldcg(cx.scratch + (int64_t)(cr.first_part + p) * B + slot0 + v);
    const int64_t deg = __ldg(cx.indptr + cr.row + 1) - __ldg(cx.indptr + cr.row);
    T out[VEC];
#pragma unroll
    for (int v = 0; v < VEC; v++) {
        out[v] = (T)(cx.scale * tot[v]);
        if (((cmask >> v) & 1u) && (double)out[v] > 0.0) inc.v[v] = deg;
    }
    VecIO<T, VEC>::st(cx.Y + (int64_t)cr.row * B + slot0, out);
    if (lane == 0) cx.cut_count[ci] = 0;
    return inc;
}

// Same streaming pull with the per-warp (col, val) windows and row ends staged
// in shared memory instead of lane registers: the per-edge work is one
// broadcast LDS of the next (col, val) pair, the operand-row gather and VEC
// FMAs, with no warp shuffle (and so no convergence barrier) on the edge path.
// Cut-row partials go to their scratch slot at emit time.
// Pipeline depth / residency of k_pull_sw: S = 8 rows in flight per warp at
// three 256-thread blocks per SM measured fastest at B = 64 fp32 (c2 on B200:
// more resident warps beat a deeper per-warp pipeline).
template <int B, typename T>
struct SwPipe {
    static constexpr int LANE_BYTES = (B / 32) * (int)sizeof(T);
    static constexpr int S = LANE_BYTES <= 16 ? 8 : 4;
    static constexpr int MINB = LANE_BYTES <= 8 ? 3 : 2;
};

template <typename T>
struct EdgeCV {
    int32_t c;
    T v;
};

template <int B, typename T, int SIDE, int S = SwPipe<B, T>::S, int MINB = SwPipe<B, T>::MINB>
__global__ void __launch_bounds__(PULL_THREADS, MINB) k_pull_sw(PullArgs<T> a) {
    pdl_begin();
    if (*a.active == 0) return;
    constexpr int VEC = RegPipe<B, T>::VEC;
    static_assert(2 * S <= 32, "two windows must fit one warp load");
    __shared__ EdgeCV<T> s_win[PULL_WARPS][2][S];
    __shared__ int32_t s_re[PULL_WARPS][64];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * PULL_WARPS + warp;
    const int slot0 = lane * VEC;
    uint32_t cmask = 0;
    if constexpr (SIDE == SIDE_V) {
#pragma unroll
        for (int v = 0; v < VEC; v++) cmask |= (op_is_push(a.slots[slot0 + v].op) ? 1u : 0u) << v;
    }
    const double scale = SIDE == SIDE_V ? a.one_minus_alpha : 1.0;
    int32_t np[VEC];
#pragma unroll
    for (int v = 0; v < VEC; v++) np[v] = 0;
    int64_t np_cut[VEC];
#pragma unroll
    for (int v = 0; v < VEC; v++) np_cut[v] = 0;

    if (gw < a.n_warps) {
        const WarpWork wk = a.work[gw];
        const int64_t e0 = wk.e0;
        const int n = (int)(wk.e1 - e0);
        if (n > 0) {
            const int32_t *cols = a.indices + e0;
            const T *vals = a.vals + e0;
            const T *X = a.X + slot0;
            T *Y0 = a.Y + (int64_t)wk.r0 * B + slot0;
            const int64_t *rp = a.indptr + wk.r0;
            const int64_t nrow_left = a.n_rows - wk.r0;
            const int cutA = wk.cut0 >= 0 ? 0 : -1;
            const int cutB = wk.cut1 >= 0 ? (int)(a.cuts[wk.cut1].row - wk.r0) : -1;
            auto col_at = [&](int o) { return o < n ? __ldg(cols + o) : 0; };
            auto val_at = [&](int o) { return o < n ? __ldg(vals + o) : (T)0; };
            auto rend_at = [&](int i) {
                const int64_t r = i + 1 <= nrow_left ? __ldg(rp + i + 1) : __ldg(rp + nrow_left);
                return (int)imin64(r - e0, (int64_t)n);
            };
            EdgeCV<T>(*win)[S] = s_win[warp];
            int32_t *re = s_re[warp];
            auto fetch = [&](int c, T(&x)[VEC]) { ldg_vec<T, VEC>(X + (int64_t)c * B, x); };
            re[lane] = rend_at(lane);
            re[32 + lane] = rend_at(32 + lane);
            if (lane < 2 * S) win[lane / S][lane % S] = EdgeCV<T>{col_at(lane), val_at(lane)};
            // register prefetch of block 2's window (lanes < S)
            int cw = col_at(2 * S + lane);
            T vw = val_at(2 * S + lane);
            __syncwarp();
            T xs[S][VEC];
            T wsv[S];
#pragma unroll
            for (int t = 0; t < S; t++) {
                const EdgeCV<T> e = win[0][t];
                wsv[t] = e.v;
                fetch(e.c, xs[t]);
            }
            int rw = 0;       // row-end ring holds local rows [rw, rw + 64)
            int lr = 0;
            int rstart = (int)(__ldg(rp) - e0);
            int rend = re[0];
            double acc[VEC];
            T accs[VEC];
#pragma unroll
            for (int v = 0; v < VEC; v++) {
                acc[v] = 0.0;
                accs[v] = (T)0;
            }
            int b = 0;
            for (int base = 0; base < n; base += S, b ^= 1) {
                const EdgeCV<T> *nxt = win[b ^ 1];
                int d = rend - base - 1;
#pragma unroll
                for (int t = 0; t < S; t++) {
                    if constexpr (sizeof(T) == 8) {
#pragma unroll
                        for (int v = 0; v < VEC; v++) acc[v] = fma((double)wsv[t], (double)xs[t][v], acc[v]);
                    } else {
#pragma unroll
                        for (int v = 0; v < VEC; v++) accs[v] = fmaf(wsv[t], xs[t][v], accs[v]);
                    }
                    if (d == t) {  // row emit
                        if constexpr (sizeof(T) == 4) {
#pragma unroll
                            for (int v = 0; v < VEC; v++) {
                                acc[v] += (double)accs[v];
                                accs[v] = (T)0;
                            }
                        }
                        if (lr == cutA || lr == cutB) {
                            double *dst = a.scratch + (int64_t)(lr == cutA ? wk.part0 : wk.part1) * B + slot0;
#pragma unroll
                            for (int v = 0; v < VEC; v++) dst[v] = acc[v];
                        } else {
                            T out[VEC];
#pragma unroll
                            for (int v = 0; v < VEC; v++) {
                                out[v] = (T)(scale * acc[v]);
                                if constexpr (SIDE == SIDE_V)
                                    np[v] += (((cmask >> v) & 1u) && out[v] > (T)0) ? rend - rstart : 0;
                            }
                            VecIO<T, VEC>::st(Y0 + (int64_t)lr * B, out);
                        }
#pragma unroll
                        for (int v = 0; v < VEC; v++) acc[v] = 0.0;
                        lr++;
                        rstart = rend;
                        rend = re[lr & 63];
                        d = rend - base - 1;
                    }
                    const EdgeCV<T> e = nxt[t];
                    wsv[t] = e.v;
                    fetch(e.c, xs[t]);
                }
                if constexpr (sizeof(T) == 4) {
#pragma unroll
                    for (int v = 0; v < VEC; v++) {
                        acc[v] += (double)accs[v];
                        accs[v] = (T)0;
                    }
                }
                // stage block (base/S + 2) into the window block (base/S) read during
                // the previous block, refill the row-end ring half that is behind lr
                if (lane < S) win[b][lane] = EdgeCV<T>{cw, vw};
                if (lr - rw >= 32) {
                    re[(rw + 64 + lane) & 63] = rend_at(rw + 64 + lane);
                    rw += 32;
                }
                cw = col_at(base + 3 * S + lane);
                vw = val_at(base + 3 * S + lane);
                __syncwarp();
            }
            const CutCtx<T> cx{a.scratch, a.cut_count, a.cuts, a.Y, a.indptr, scale};
            if (cutA >= 0) {
                DVec<VEC> av;
#pragma unroll
                for (int v = 0; v < VEC; v++) av.v[v] = a.scratch[(int64_t)wk.part0 * B + slot0 + v];
                const IVec<VEC> inc = pull_cut<B, T, VEC>(cx, wk.cut0, wk.part0, slot0, cmask, av);
#pragma unroll
                for (int v = 0; v < VEC; v++) np_cut[v] += inc.v[v];
            }
            if (cutB >= 0) {
                DVec<VEC> av;
#pragma unroll
                for (int v = 0; v < VEC; v++) av.v[v] = a.scratch[(int64_t)wk.part1 * B + slot0 + v];
                const IVec<VEC> inc = pull_cut<B, T, VEC>(cx, wk.cut1, wk.part1, slot0, cmask, av);
#pragma unroll
                for (int v = 0; v < VEC; v++) np_cut[v] += inc.v[v];
            }
        }
    }
    if constexpr (SIDE == SIDE_V) {
        if (gw < a.n_warps)
#pragma unroll
            for (int v = 0; v < VEC; v++) a.np_v[(int64_t)(slot0 + v) * a.n_warps + gw] = (int64_t)np[v] + np_cut[v];
    }
}


// Row-flag pull (the default dense pull for B >= 32).  Same partition, cut-row
// protocol, n_p layout and summation order within a row as k_pull_sw, with a
// leaner edge path:
//   - the edge stream is the store's packed EdgeRF array.  A 32-edge tile goes
//     from global memory straight into a 128-entry shared ring with one cp.async
//     per lane, three tiles ahead of its use: no staging registers, and the wait
//     is on the copy group, not on a scoreboard shared with the operand gathers;
//   - the per-edge work is one broadcast LDS of (column, value), the operand-row
//     gather and VEC FMAs;
//   - the last edge of a row carries a negated value, so the row end is a sign
//     test on a register that is loaded anyway: no row-pointer ring, no per-edge
//     offset compare, no reload of row ends;
//   - S (a divisor of 32) operand rows are in flight per warp in registers; the
//     S-edge body is unrolled, the bodies of a tile are a loop; WARPS warps per
//     block (7 lets four blocks of 72-register threads share an SM);
//   - one ballot per tile turns the value signs into a bitmask: a body without a
//     row end runs branch-free, a body with one tests the mask bit per edge and
//     emits inline (fp64 fold, scale, store, n_p);
//   - fp32: products accumulate in fp32 over one S-edge body at most and are
//     folded into the row's fp64 accumulator after it (and at a row end).
template <int B, typename T, int SIDE, int S, int MINB, int WARPS = PULL_WARPS>
__global__ void __launch_bounds__(WARPS * 32, MINB) k_pull_rf(PullArgs<T> a) {
    pdl_launch_dependents();
    constexpr int VEC = RegPipe<B, T>::VEC;
    constexpr int RING = 128;  // four 32-edge tiles
    static_assert(32 % S == 0, "the S-edge body must tile a 32-edge window");
    __shared__ EdgeRF<T> s_ring[WARPS][RING];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * WARPS + warp;
    const int slot0 = lane * VEC;
    // The plan and the edge stream are immutable graph data: the first three edge tiles are
    // put in flight under the predecessor's tail, before the wait for its memory.
    int64_t e0 = 0;
    int n = 0;
    if (gw < a.n_warps) {
        e0 = a.work[gw].e0;
        n = (int)(a.work[gw].e1 - e0);
    }
    const EdgeRF<T> *ed = reinterpret_cast<const EdgeRF<T> *>(a.ecv) + e0;
    EdgeRF<T> *ring = s_ring[warp];
    // tile k (edges 32 k + lane) into ring slot k & 3; past the range the copy zero-fills
    // (column 0, value +0: gathers row 0, adds nothing, ends no row)
    const uint32_t ring_lane = smem_u32(ring + lane);
    auto stage = [&](int tile) {
        const int o = tile * 32 + lane;
        const EdgeRF<T> *src = ed + (o < n ? o : 0);
        cp_async_zfill<(int)sizeof(EdgeRF<T>)>(ring_lane + (uint32_t)((tile & 3) * 32 * sizeof(EdgeRF<T>)), src, o < n);
        cp_async_commit();
    };
    if (n > 0) {
        stage(0);
        stage(1);
        stage(2);
    }
    pdl_wait();
    if (*a.active == 0) {
        cp_async_wait<0>();
        return;
    }
    uint32_t cmask = 0;
    if constexpr (SIDE == SIDE_V) {
#pragma unroll
        for (int v = 0; v < VEC; v++) cmask |= (op_is_push(a.slots[slot0 + v].op) ? 1u : 0u) << v;
    }
    const double scale = SIDE == SIDE_V ? a.one_minus_alpha : 1.0;
    int64_t npt[VEC];
#pragma unroll
    for (int v = 0; v < VEC; v++) npt[v] = 0;
    if (gw < a.n_warps) {
        if (n > 0) {
            int32_t np[VEC];
#pragma unroll
            for (int v = 0; v < VEC; v++) np[v] = 0;
            const T *X = a.X + slot0;
            T *yrow = a.Y + (int64_t)a.work[gw].r0 * B + slot0;
            auto fetch = [&](int c, T(&x)[VEC]) { ldg_vec<T, VEC>(X + (int64_t)c * B, x); };
            cp_async_wait<1>();  // tiles 0 and 1 have landed
            __syncwarp();
            T xs[S][VEC];
            T wsv[S];
#pragma unroll
            for (int t = 0; t < S; t++) {
                const EdgeRF<T> e = ring[t];
                wsv[t] = e.v;
                fetch(e.c, xs[t]);
            }
            double acc[VEC];
            T accs[VEC];
#pragma unroll
            for (int v = 0; v < VEC; v++) {
                acc[v] = 0.0;
                accs[v] = (T)0;
            }
            const bool first_cut = a.work[gw].cut0 >= 0;
            int rstart = 0;  // offset of the current row's first edge in the range (0: the range's first row)
            for (int base = 0; base < n; base += 32) {
                // row ends of this tile, one bit per edge: a body without one runs branch-free
                const uint32_t tmask = __ballot_sync(0xffffffffu, ring[(base & (RING - 1)) + lane].v < (T)0);
#pragma unroll 1
                for (int sub = 0; sub < 32; sub += S) {
                    const EdgeRF<T> *nxt = ring + ((base + sub + S) & (RING - 1));
                    const uint32_t bm = (tmask >> sub) & (uint32_t)((1ull << S) - 1ull);
                    if (bm == 0u) {
#pragma unroll
                        for (int t = 0; t < S; t++) {
                            if constexpr (sizeof(T) == 8) {
#pragma unroll
                                for (int v = 0; v < VEC; v++) acc[v] = fma((double)wsv[t], (double)xs[t][v], acc[v]);
                            } else {
#pragma unroll
                                for (int v = 0; v < VEC; v++) accs[v] = fmaf(wsv[t], xs[t][v], accs[v]);
                            }
                            const EdgeRF<T> e = nxt[t];
                            wsv[t] = e.v;
                            fetch(e.c, xs[t]);
                        }
                    } else
#pragma unroll
                    for (int t = 0; t < S; t++) {
                        const T w = wsv[t];
                        if constexpr (sizeof(T) == 8) {
#pragma unroll
                            for (int v = 0; v < VEC; v++) acc[v] = fma(fabs((double)w), (double)xs[t][v], acc[v]);
                        } else {
#pragma unroll
                            for (int v = 0; v < VEC; v++) accs[v] = fmaf(fabsf(w), xs[t][v], accs[v]);
                        }
                        if ((bm >> t) & 1u) {  // last edge of a row (w < 0)
                            if constexpr (sizeof(T) == 4) {
#pragma unroll
                                for (int v = 0; v < VEC; v++) {
                                    acc[v] += (double)accs[v];
                                    accs[v] = (T)0;
                                }
                            }
                            const int rend = base + sub + t + 1;
                            if (rstart == 0 && first_cut) {
                                double *dst = a.scratch + (int64_t)a.work[gw].part0 * B + slot0;
#pragma unroll
                                for (int v = 0; v < VEC; v++) dst[v] = acc[v];
                            } else {
                                T out[VEC];
#pragma unroll
                                for (int v = 0; v < VEC; v++) {
                                    out[v] = (T)(scale * acc[v]);
                                    if constexpr (SIDE == SIDE_V)
                                        np[v] += (((cmask >> v) & 1u) && out[v] > (T)0) ? rend - rstart : 0;
                                }
                                VecIO<T, VEC>::st(yrow, out);
                            }
#pragma unroll
                            for (int v = 0; v < VEC; v++) acc[v] = 0.0;
                            yrow += B;
                            rstart = rend;
                        }
                        const EdgeRF<T> e = nxt[t];
                        wsv[t] = e.v;
                        fetch(e.c, xs[t]);
                    }
                    if constexpr (sizeof(T) == 4) {
#pragma unroll
                        for (int v = 0; v < VEC; v++) {
                            acc[v] += (double)accs[v];
                            accs[v] = (T)0;
                        }
                    }
                }
                // tile base/32 is consumed and the gathers reached at most S edges into the next
                // one.  Tile + 3 goes into the slot tile - 1 left (its last read was before the
                // previous iteration's barrier); tile + 2 must have landed before the next
                // iteration's last body looks S edges ahead.
                stage((base >> 5) + 3);
                cp_async_wait<1>();
                __syncwarp();
            }
            cp_async_wait<0>();
            const WarpWork wk = a.work[gw];
            if (rstart < n) {  // the range ends inside a row: its partial goes to the cut protocol
                double *dst = a.scratch + (int64_t)((rstart == 0 && first_cut) ? wk.part0 : wk.part1) * B + slot0;
#pragma unroll
                for (int v = 0; v < VEC; v++) dst[v] = acc[v];
            }
            const CutCtx<T> cx{a.scratch, a.cut_count, a.cuts, a.Y, a.indptr, scale};
            if (wk.cut0 >= 0) {
                DVec<VEC> av;
#pragma unroll
                for (int v = 0; v < VEC; v++) av.v[v] = a.scratch[(int64_t)wk.part0 * B + slot0 + v];
                const IVec<VEC> inc = pull_cut<B, T, VEC>(cx, wk.cut0, wk.part0, slot0, cmask, av);
#pragma unroll
                for (int v = 0; v < VEC; v++) npt[v] += inc.v[v];
            }
#pragma unroll
            for (int v = 0; v < VEC; v++) npt[v] += np[v];
            if (wk.cut1 >= 0) {
                DVec<VEC> av;
#pragma unroll
                for (int v = 0; v < VEC; v++) av.v[v] = a.scratch[(int64_t)wk.part1 * B + slot0 + v];
                const IVec<VEC> inc = pull_cut<B, T, VEC>(cx, wk.cut1, wk.part1, slot0, cmask, av);
#pragma unroll
                for (int v = 0; v < VEC; v++) npt[v] += inc.v[v];
            }
        }
    }
    if constexpr (SIDE == SIDE_V) {
        if (gw < a.n_warps)
#pragma unroll
            for (int v = 0; v < VEC; v++) a.np_v[(int64_t)(slot0 + v) * a.n_warps + gw] = npt[v];
    }
}

// B < 32 (single-query and small blocks): G lanes per edge group, 32/G groups
// split each row; plain loads.  Same partition, cut rows and epilogue.
template <int B, typename T, int SIDE>
__global__ void __launch_bounds__(PULL_THREADS) k_pull_small(PullArgs<T> a) {
    pdl_begin();
    if (*a.active == 0) return;
    constexpr int G = B, EPW = 32 / B;
    __shared__ int32_t s_op[MAX_B];
    for (int s = threadIdx.x; s < B; s += blockDim.x) s_op[s] = a.slots[s].op;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * PULL_WARPS + warp;
    const int grp = lane / G, slot = lane % G;
    int64_t np = 0;
    if (gw < a.n_warps) {
        const WarpWork wk = a.work[gw];
        const int64_t e0 = wk.e0, e1 = wk.e1;
        int64_t row = wk.r0;
        for (int64_t guard = 0; e0 < e1 && guard <= a.n_rows; guard++) {
            const int64_t rs = __ldg(a.indptr + row), re = __ldg(a.indptr + row + 1);
            const int64_t s0 = rs > e0 ? rs : e0, s1 = re < e1 ? re : e1;
            double acc = 0.0;
            for (int64_t e = s0 + grp; e < s1; e += EPW)
                acc = fma((double)__ldg(a.vals + e), (double)__ldg(a.X + (int64_t)__ldg(a.indices + e) * B + slot), acc);
#pragma unroll
            for (int off = G; off < 32; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            const bool cut = rs < e0 || re > e1;
            double fin = acc;
            bool do_final = !cut;
            if (cut) {
                const int ci = (row == wk.r0) ? wk.cut0 : wk.cut1;
                const int pi = (row == wk.r0) ? wk.part0 : wk.part1;
                if (grp == 0) a.scratch[(int64_t)pi * B + slot] = acc;
                __threadfence();
                __syncwarp();
                const CutRow cr = a.cuts[ci];
                int last = 0;
                if (lane == 0) last = atomicAdd(a.cut_count + ci, 1) == cr.n_parts - 1;
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    __threadfence();
                    fin = 0.0;
                    for (int p = 0; p < cr.n_parts; p++) fin += __ldcg(a.scratch + (int64_t)(cr.first_part + p) * B + slot);
                    do_final = true;
                    if (lane == 0) a.cut_count[ci] = 0;
                }
            }
            if (do_final && grp == 0) {
                T out;
                if constexpr (SIDE == SIDE_V) {
                    out = (T)(a.one_minus_alpha * fin);
                    if (op_is_push(s_op[slot]) && (double)out > 0.0) np += (int32_t)(re - rs);
                } else {
                    out = (T)fin;
                }
                a.Y[row * B + slot] = out;
            }
            if (re >= e1) break;
            row++;
        }
    }
    if constexpr (SIDE == SIDE_V) {
        if (gw < a.n_warps && grp == 0) a.np_v[(int64_t)slot * a.n_warps + gw] = np;
    }
}

}  // namespace bh
