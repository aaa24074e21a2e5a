// kernels.cuh -- device kernels of one push / power-iteration round over a
// block of B query slots (node-major, slot-minor state: X[node * B + slot]).
//
// Round = K1 prep -> K2 V-pull (+K2b finisher) -> K3 U-pull (+K3b) -> K4 control
//         [-> K5 finalize/score chunks -> K6 top-k merge, when a slot finishes]
//
// Reference semantics (pkg/src/bipush/push_engine.py):
//   K1  _push_u bookkeeping (294-309): A = {r_u > theta}, est[A] += alpha r_u,
//       r_u[A] = 0, n_p += sum deg(A); the pushed amounts go to P.
//   K2  _push_u's r_v += (1-alpha) * v_step @ dense (303-306) as a pull over
//       V-CSR; n_p += deg(v) for r_v > 0 (the flushed set, 312-324).
//   K3  _flush_v's r_u += u_step @ r_v (322) as a pull over U-CSR, plus the
//       per-query reductions the round's exit tests need (any r_u > theta,
//       sum r_u, sum w_ratio r_u; 168-177, 234-243).
//   Power iteration (101-117) runs the same K2/K3 pair on a = acc / ws:
//       a <- y0 + U (1-alpha) V a   (detailed balance).
// Every row sum is a sequential fp64 accumulation in CSR order; long rows are
// split into pieces whose partials a finisher adds in piece order, and every
// per-query reduction goes through per-block partial rows summed in order by
// K4.  Results are therefore bitwise deterministic run to run.
#pragma once

#include "common.cuh"

namespace bh {

// ---------------------------------------------------------------------------
// small helpers

template <typename T, int VEC>
struct VecIO;

template <>
struct VecIO<float, 1> {
    static __device__ __forceinline__ void ld(const float *p, float (&v)[1]) { v[0] = __ldg(p); }
    static __device__ __forceinline__ void ldc(const float *p, float (&v)[1]) { v[0] = *p; }
    static __device__ __forceinline__ void st(float *p, const float (&v)[1]) { *p = v[0]; }
};
template <>
struct VecIO<float, 2> {
    static __device__ __forceinline__ void ld(const float *p, float (&v)[2]) {
        float2 t = __ldg(reinterpret_cast<const float2 *>(p));
        v[0] = t.x; v[1] = t.y;
    }
    static __device__ __forceinline__ void ldc(const float *p, float (&v)[2]) {
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
        float4 t = __ldg(reinterpret_cast<const float4 *>(p));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    static __device__ __forceinline__ void ldc(const float *p, float (&v)[4]) {
        float4 t = *reinterpret_cast<const float4 *>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    static __device__ __forceinline__ void st(float *p, const float (&v)[4]) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <>
struct VecIO<double, 1> {
    static __device__ __forceinline__ void ld(const double *p, double (&v)[1]) { v[0] = __ldg(p); }
    static __device__ __forceinline__ void ldc(const double *p, double (&v)[1]) { v[0] = *p; }
    static __device__ __forceinline__ void st(double *p, const double (&v)[1]) { *p = v[0]; }
};
template <>
struct VecIO<double, 2> {
    static __device__ __forceinline__ void ld(const double *p, double (&v)[2]) {
        double2 t = __ldg(reinterpret_cast<const double2 *>(p));
        v[0] = t.x; v[1] = t.y;
    }
    static __device__ __forceinline__ void ldc(const double *p, double (&v)[2]) {
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
        double2 a = __ldg(reinterpret_cast<const double2 *>(p));
        double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
    static __device__ __forceinline__ void ldc(const double *p, double (&v)[4]) {
        double2 a = *reinterpret_cast<const double2 *>(p);
        double2 b = *(reinterpret_cast<const double2 *>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
    static __device__ __forceinline__ void st(double *p, const double (&v)[4]) {
        reinterpret_cast<double2 *>(p)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2 *>(p)[1] = make_double2(v[2], v[3]);
    }
};

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ bool op_is_push(int op) { return op >= OP_BSEL_INIT && op <= OP_FSEL; }
__device__ __forceinline__ bool op_is_fwd(int op) { return op == OP_FENTRY || op == OP_FSEL; }

// ---------------------------------------------------------------------------
// Launch geometry shared by host and device.
template <int B>
struct Geo {
    static constexpr int G = B < 32 ? B : 32;     // lanes per edge group
    static constexpr int EPW = 32 / G;            // edges in flight per warp step
    static constexpr int VEC = B / G;             // slots per lane
};

constexpr int PULL_THREADS = 256;
constexpr int PULL_WARPS = PULL_THREADS / 32;
constexpr int PREP_THREADS = 256;

// Per-slot constants staged in shared memory by every round kernel.
struct SlotSmem {
    int32_t op[MAX_B];
    int32_t qidx[MAX_B];
    int32_t src[MAX_B];
    double eps_b[MAX_B];
    double thc[MAX_B];     // eps_f / lam
    double wsq[MAX_B];     // ws(source)
    double iwsq[MAX_B];    // 1 / ws(source)
    double ysc[MAX_B];
};

template <int B>
__device__ __forceinline__ void load_slot_smem(SlotSmem &sm, const Slot *__restrict__ slots) {
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        const Slot &sl = slots[s];
        sm.op[s] = sl.op;
        sm.qidx[s] = sl.qidx;
        sm.src[s] = sl.src;
        sm.eps_b[s] = sl.eps_b;
        sm.thc[s] = sl.theta_c;
        sm.wsq[s] = sl.ws_q;
        sm.iwsq[s] = sl.inv_ws_q;
        sm.ysc[s] = sl.ysc;
    }
}

// ---------------------------------------------------------------------------
// K1: prep.  Elementwise over [n_u x B].
template <typename T>
struct PrepArgs {
    int64_t n_u;
    T *R;
    T *P;
    double *EST;
    const int32_t *deg_u;
    const double *ws_u;
    const double *inv_ws_u;
    const double *x0;  // BH_JOB_POWER start vectors [n_q][n_u]
    const Slot *slots;
    const int32_t *active;
    Partials part;
    double alpha;
};

template <int B, typename T>
__global__ void __launch_bounds__(PREP_THREADS) k_prep(PrepArgs<T> a) {
    if (*a.active == 0) return;
    __shared__ SlotSmem sm;
    __shared__ int64_t red_cnt[PREP_THREADS];
    __shared__ int64_t red_np[PREP_THREADS];
    __shared__ double red_g[PREP_THREADS];
    load_slot_smem<B>(sm, a.slots);
    __syncthreads();
    const int s = threadIdx.x & (B - 1);
    const int op = sm.op[s];
    const bool push = op_is_push(op);
    const bool init = op == OP_BSEL_INIT;
    const bool fentry = op == OP_FENTRY;
    const bool fwd = op_is_fwd(op);
    const bool pientry = op == OP_PIENTRY || op == OP_PIENTRY0;
    const double eps_b = sm.eps_b[s];
    const double thc = sm.thc[s], wsq = sm.wsq[s], iwsq = sm.iwsq[s], ysc = sm.ysc[s];
    const int src = sm.src[s];
    const double *x0 = (a.x0 && sm.qidx[s] >= 0) ? a.x0 + (int64_t)sm.qidx[s] * a.n_u : nullptr;
    int64_t cnt = 0, npu = 0;
    double gam = 0.0;
    if (push || pientry) {
        const int64_t total = a.n_u * B;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
             i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t u = i / B;
            double r = init ? (u == src ? 1.0 : 0.0) : (double)a.R[i];
            if (pientry) {
                if (x0) {  // raw power iteration: y0 = start / ws (push_engine.py:112, in a = acc / ws)
                    const T y = (T)(x0[u] * a.inv_ws_u[u]);
                    a.R[i] = y;
                    a.P[i] = y;
                } else {  // PI-Push tail: y0 = (w_ratio r) / ws = r / ws(q)  (push_engine.py:246)
                    a.P[i] = (T)(r * ysc);
                }
                continue;
            }
            double th;
            if (fwd) th = (wsq * a.inv_ws_u[u]) * thc;   // (ws_q / ws_i) * (eps_f / lam)
            else th = (op == OP_SEQ) ? 0.0 : eps_b;
            if (fentry) gam += (a.ws_u[u] * iwsq) * r;     // gamma, push_engine.py:222
            const bool act = r > th;
            a.P[i] = act ? (T)r : (T)0;
            if (act) {
                a.R[i] = (T)0;
                a.EST[i] = (init ? 0.0 : a.EST[i]) + a.alpha * r;
                cnt += 1;
                npu += a.deg_u[u];
            } else if (init) {
                a.R[i] = (T)r;
                a.EST[i] = 0.0;
            }
        }
    }
    red_cnt[threadIdx.x] = cnt;
    red_np[threadIdx.x] = npu;
    red_g[threadIdx.x] = gam;
    __syncthreads();
    for (int t = threadIdx.x; t < B; t += blockDim.x) {
        int64_t c = 0, n = 0;
        double gg = 0.0;
        for (int j = t; j < PREP_THREADS; j += B) {
            c += red_cnt[j];
            n += red_np[j];
            gg += red_g[j];
        }
        a.part.cnt[blockIdx.x * B + t] = c;
        a.part.np_u[blockIdx.x * B + t] = n;
        a.part.gamma[blockIdx.x * B + t] = gg;
    }
}

// ---------------------------------------------------------------------------
// K2 / K3: pull SpMM with fused round epilogue.
enum : int { SIDE_V = 0, SIDE_U = 1 };

template <typename T>
struct PullArgs {
    const int64_t *indptr;
    const int32_t *indices;
    const T *vals;
    const Unit *units;
    int32_t n_units;
    const SplitRow *splits;
    int32_t n_splits;
    double *scratch;  // [n_pieces][B]
    const T *X;       // operand: P (V pull) or XV (U pull)
    T *Y;             // V pull: XV ; U pull: R (in/out)
    T *P;             // U pull: P for power-iteration slots
    const double *ws_u;
    const double *inv_ws_u;
    const Slot *slots;
    const int32_t *active;
    Partials part;
    int32_t part_row0;
    double one_minus_alpha;
};

template <int B, typename T, int SIDE>
struct Epi {
    static constexpr int VEC = Geo<B>::VEC;
    // per-lane reductions
    int64_t np[SIDE == SIDE_V ? VEC : 1];
    int32_t any[SIDE == SIDE_U ? VEC : 1];
    double red[SIDE == SIDE_U ? VEC : 1];

    __device__ __forceinline__ void init() {
#pragma unroll
        for (int j = 0; j < (SIDE == SIDE_V ? VEC : 1); j++) np[j] = 0;
#pragma unroll
        for (int j = 0; j < (SIDE == SIDE_U ? VEC : 1); j++) {
            any[j] = 0;
            red[j] = 0.0;
        }
    }

    // Final value of one row for the lane's VEC slots starting at slot0.
    __device__ __forceinline__ void row(const PullArgs<T> &a, const SlotSmem &sm, int64_t row, int32_t deg,
                                        int slot0, const double (&acc)[VEC]) {
        if constexpr (SIDE == SIDE_V) {
            T out[VEC];
#pragma unroll
            for (int j = 0; j < VEC; j++) {
                out[j] = (T)(a.one_minus_alpha * acc[j]);
                if (op_is_push(sm.op[slot0 + j]) && (double)out[j] > 0.0) np[j] += deg;
            }
            VecIO<T, VEC>::st(a.Y + row * B + slot0, out);
        } else {
            T r[VEC];
            VecIO<T, VEC>::ldc(a.Y + row * B + slot0, r);
            const double wsr = a.ws_u[row];
            const double iwsr = a.inv_ws_u[row];
#pragma unroll
            for (int j = 0; j < VEC; j++) {
                const int s = slot0 + j;
                const int op = sm.op[s];
                if (op_is_push(op)) {
                    const T nr = (T)((double)r[j] + acc[j]);
                    r[j] = nr;
                    const double v = (double)nr;
                    if (op_is_fwd(op)) {
                        const double th = (sm.wsq[s] * iwsr) * sm.thc[s];
                        any[j] |= v > th;
                        red[j] += (wsr * sm.iwsq[s]) * v;
                    } else {
                        any[j] |= v > sm.eps_b[s];
                        red[j] += v;
                    }
                } else if (op == OP_PIENTRY || op == OP_PI) {
                    const double y0 = (double)r[j] * sm.ysc[s];
                    a.P[row * B + s] = (T)(y0 + acc[j]);
                }
            }
            VecIO<T, VEC>::st(a.Y + row * B + slot0, r);
        }
    }

    // Write this lane's reductions to the block partial row.
    __device__ __forceinline__ void flush(const PullArgs<T> &a, bool owner, int slot0, int warp,
                                          double *sh_d, int64_t *sh_i, int32_t *sh_a) {
        if (owner) {
#pragma unroll
            for (int j = 0; j < VEC; j++) {
                if constexpr (SIDE == SIDE_V) {
                    sh_i[warp * B + slot0 + j] = np[j];
                } else {
                    sh_a[warp * B + slot0 + j] = any[j];
                    sh_d[warp * B + slot0 + j] = red[j];
                }
            }
        }
    }
};

template <int B, typename T, int SIDE>
__device__ __forceinline__ void block_partials(const PullArgs<T> &a, int nwarps, double *sh_d, int64_t *sh_i,
                                               int32_t *sh_a, int row_index) {
    __syncthreads();
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        if constexpr (SIDE == SIDE_V) {
            int64_t n = 0;
            for (int w = 0; w < nwarps; w++) n += sh_i[w * B + s];
            a.part.np_v[(int64_t)row_index * B + s] = n;
        } else {
            int32_t an = 0;
            double r = 0.0;
            for (int w = 0; w < nwarps; w++) {
                an |= sh_a[w * B + s];
                r += sh_d[w * B + s];
            }
            a.part.any[(int64_t)row_index * B + s] = an;
            a.part.sum[(int64_t)row_index * B + s] = r;
        }
    }
}

template <int B, typename T, int SIDE>
__global__ void __launch_bounds__(PULL_THREADS) k_pull(PullArgs<T> a) {
    if (*a.active == 0) return;
    using GE = Geo<B>;
    constexpr int G = GE::G, EPW = GE::EPW, VEC = GE::VEC;
    __shared__ SlotSmem sm;
    __shared__ double sh_d[PULL_WARPS * B];
    __shared__ int64_t sh_i[PULL_WARPS * B];
    __shared__ int32_t sh_a[PULL_WARPS * B];
    load_slot_smem<B>(sm, a.slots);
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int grp = lane / G;
    const int slot0 = (lane % G) * VEC;
    const int64_t gwarp = (int64_t)blockIdx.x * PULL_WARPS + warp;
    const int64_t nwarps_total = (int64_t)gridDim.x * PULL_WARPS;
    Epi<B, T, SIDE> epi;
    epi.init();

    for (int64_t ui = gwarp; ui < a.n_units; ui += nwarps_total) {
        const Unit un = a.units[ui];
        const bool piece = un.piece >= 0;
        if constexpr (EPW == 1) {
            // ---- B >= 32: lanes own slots, the warp walks the unit's edge stream
            const int64_t my_rend = (!piece && lane < un.nrows) ? a.indptr[un.row0 + lane + 1] : 0;
            int rr = 0;
            int64_t rstart = un.e0;
            int64_t rend = piece ? un.e1 : __shfl_sync(0xffffffffu, my_rend, 0);
            double acc[VEC];
#pragma unroll
            for (int j = 0; j < VEC; j++) acc[j] = 0.0;
            for (int64_t cb = un.e0; cb < un.e1; cb += 32) {
                const int n = (int)imin64(32, un.e1 - cb);
                const int my_col = lane < n ? __ldg(a.indices + cb + lane) : 0;
                const T my_val = lane < n ? __ldg(a.vals + cb + lane) : (T)0;
                constexpr int UNR = 8;
                for (int j0 = 0; j0 < n; j0 += UNR) {
                    T xs[UNR][VEC];
                    T wv[UNR];
#pragma unroll
                    for (int t = 0; t < UNR; t++) {
                        const int j = j0 + t;
                        const int c = __shfl_sync(0xffffffffu, my_col, j & 31);
                        wv[t] = __shfl_sync(0xffffffffu, my_val, j & 31);
                        if (j < n) {
                            VecIO<T, VEC>::ld(a.X + (int64_t)c * B + slot0, xs[t]);
                        } else {
#pragma unroll
                            for (int v = 0; v < VEC; v++) xs[t][v] = (T)0;
                        }
                    }
#pragma unroll
                    for (int t = 0; t < UNR; t++) {
                        const int j = j0 + t;
                        if (j < n) {
#pragma unroll
                            for (int v = 0; v < VEC; v++) acc[v] = fma((double)wv[t], (double)xs[t][v], acc[v]);
                            if (cb + j + 1 == rend) {
                                if (piece) {
#pragma unroll
                                    for (int v = 0; v < VEC; v++) a.scratch[(int64_t)un.piece * B + slot0 + v] = acc[v];
                                } else {
                                    epi.row(a, sm, un.row0 + rr, (int32_t)(rend - rstart), slot0, acc);
                                    rr++;
                                    rstart = rend;
                                    rend = __shfl_sync(0xffffffffu, my_rend, rr & 31);
                                }
#pragma unroll
                                for (int v = 0; v < VEC; v++) acc[v] = 0.0;
                            }
                        }
                    }
                }
            }
        } else {
            // ---- B < 32: EPW edge groups of G lanes split each row
            const int nrows = piece ? 1 : un.nrows;
            for (int rr = 0; rr < nrows; rr++) {
                const int64_t row = un.row0 + rr;
                const int64_t e_s = piece ? un.e0 : a.indptr[row];
                const int64_t e_e = piece ? un.e1 : a.indptr[row + 1];
                double acc[VEC];
#pragma unroll
                for (int j = 0; j < VEC; j++) acc[j] = 0.0;
                constexpr int UNR = 4;
                for (int64_t e = e_s + grp; e < e_e; e += EPW * UNR) {
                    T xs[UNR][VEC];
                    T wv[UNR];
#pragma unroll
                    for (int t = 0; t < UNR; t++) {
                        const int64_t ee = e + (int64_t)t * EPW;
                        if (ee < e_e) {
                            const int c = __ldg(a.indices + ee);
                            wv[t] = __ldg(a.vals + ee);
                            VecIO<T, VEC>::ld(a.X + (int64_t)c * B + slot0, xs[t]);
                        } else {
                            wv[t] = (T)0;
#pragma unroll
                            for (int v = 0; v < VEC; v++) xs[t][v] = (T)0;
                        }
                    }
#pragma unroll
                    for (int t = 0; t < UNR; t++)
#pragma unroll
                        for (int v = 0; v < VEC; v++) acc[v] = fma((double)wv[t], (double)xs[t][v], acc[v]);
                }
                // combine the EPW groups in a fixed butterfly order
#pragma unroll
                for (int off = G; off < 32; off <<= 1)
#pragma unroll
                    for (int v = 0; v < VEC; v++) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], off);
                if (grp == 0) {
                    if (piece) {
#pragma unroll
                        for (int v = 0; v < VEC; v++) a.scratch[(int64_t)un.piece * B + slot0 + v] = acc[v];
                    } else {
                        epi.row(a, sm, row, (int32_t)(e_e - e_s), slot0, acc);
                    }
                }
            }
        }
    }
    epi.flush(a, grp == 0, slot0, warp, sh_d, sh_i, sh_a);
    block_partials<B, T, SIDE>(a, PULL_WARPS, sh_d, sh_i, sh_a, a.part_row0 + blockIdx.x);
}

// Finisher: one warp per split row, adds its pieces in order, runs the epilogue.
template <int B, typename T, int SIDE>
__global__ void __launch_bounds__(PULL_THREADS) k_pull_finish(PullArgs<T> a) {
    if (*a.active == 0) return;
    using GE = Geo<B>;
    constexpr int G = GE::G, VEC = GE::VEC;
    __shared__ SlotSmem sm;
    __shared__ double sh_d[PULL_WARPS * B];
    __shared__ int64_t sh_i[PULL_WARPS * B];
    __shared__ int32_t sh_a[PULL_WARPS * B];
    load_slot_smem<B>(sm, a.slots);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int grp = lane / G;
    const int slot0 = (lane % G) * VEC;
    Epi<B, T, SIDE> epi;
    epi.init();
    for (int64_t si = (int64_t)blockIdx.x * PULL_WARPS + warp; si < a.n_splits;
         si += (int64_t)gridDim.x * PULL_WARPS) {
        const SplitRow sr = a.splits[si];
        if (grp != 0) continue;
        double acc[VEC];
#pragma unroll
        for (int v = 0; v < VEC; v++) acc[v] = 0.0;
        for (int p = 0; p < sr.n_pieces; p++) {
#pragma unroll
            for (int v = 0; v < VEC; v++) acc[v] += a.scratch[(int64_t)(sr.first_piece + p) * B + slot0 + v];
        }
        const int32_t deg = (int32_t)(a.indptr[sr.row + 1] - a.indptr[sr.row]);
        epi.row(a, sm, sr.row, deg, slot0, acc);
    }
    epi.flush(a, grp == 0, slot0, warp, sh_d, sh_i, sh_a);
    block_partials<B, T, SIDE>(a, PULL_WARPS, sh_d, sh_i, sh_a, a.part_row0 + blockIdx.x);
}

}  // namespace bh
