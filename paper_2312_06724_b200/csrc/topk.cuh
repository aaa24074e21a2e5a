// topk.cuh -- K5/K6: BHPP combine + per-query top-k (K-T in SURVEY.md sec. 2).
//
// K5 (one CTA per (finished slot, chunk of U)): beta = (w_ratio * est
//     [+ alpha * acc_t]) + est, w_ratio = ws(u) / ws(q)  (bhpp_query.py:189,
//     push_engine.py:245-249), written contiguously per query; then the chunk's
//     top-k candidates by a radix select on the order-preserving key bits.
// K6 (one CTA per finished slot): merge the chunk candidates with the same
//     select, sort the k winners by (score desc, index asc) -- the order of
//     np.argsort(-scores, kind="stable") in topk (bhpp_query.py:206-218) --
//     and write them plus the phase trace at the query's batch index.
#pragma once

#include "kernels.cuh"

namespace bh {

__device__ __forceinline__ uint64_t order_key(double x) {
    uint64_t b = (uint64_t)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(uint64_t k) {
    uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

constexpr int TOPK_THREADS = 256;
constexpr int TOPK_MAX = 1024;

struct SelectSmem {
    uint32_t hist[256];
    uint32_t wsum[TOPK_THREADS / 32];
    uint32_t cnt;  // valid elements (32-bit: a 64-bit shared atomicAdd is a CAS loop)
    uint64_t prefix;
    int64_t krem;
    int32_t out_n;
    int32_t done;  // the chosen bin holds exactly the remaining count: selection complete
};

// Inclusive prefix sum of one value per thread over the block (blockDim == TOPK_THREADS).
__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, SelectSmem &sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) sm.wsum[w] = v;
    __syncthreads();
    uint32_t add = 0;
    for (int j = 0; j < w; j++) add += sm.wsum[j];
    __syncthreads();
    return v + add;
}

// One radix digit of the select: given the 256-bin histogram of the candidates
// that still match the prefix, pick the digit holding the krem-th element
// (descending digits for keys, ascending for indices) in parallel: thread t
// owns one bin, a block scan gives the cumulative counts, exactly one thread
// sees the crossing.  Updates sm.prefix / sm.krem.
__device__ __forceinline__ void pick_digit(SelectSmem &sm, uint64_t prefix, int shift, bool descending) {
    const int t = threadIdx.x;
    const int d = descending ? 255 - t : t;
    const uint32_t h = sm.hist[d];
    const int64_t krem = sm.krem;
    const uint32_t incl = block_incl_scan(h, sm);  // elements in digits "before or at" d
    if ((int64_t)incl >= krem && (int64_t)(incl - h) < krem) {
        sm.prefix = prefix | ((uint64_t)d << shift);
        sm.krem = krem - (int64_t)(incl - h);
        sm.done = (int64_t)h == krem - (int64_t)(incl - h);
    }
    __syncthreads();
}

constexpr int SEL_ITEMS = 8;         // candidates cached per thread in a chunk select
constexpr int SEL_ITEMS_MERGE = 16;  // ... and in the merge of the chunk candidates

// Histogram increment aggregated per warp: lanes with the same digit are
// counted by one shared-memory atomic (the leading digits of positive scores
// are shared by almost every element, and per-element atomics on one bin
// serialise).  Every lane of the warp must call it (p = whether it counts).
__device__ __forceinline__ void hist_add_warp(uint32_t *hist, bool p, uint32_t d) {
    const unsigned act = __ballot_sync(0xffffffffu, p);
    if (p) {
        const unsigned peers = __match_any_sync(act, d);
        if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(hist + d, (uint32_t)__popc(peers));
    }
}

// Output slot for an emitted element, one shared atomic per warp; every lane
// calls it.  Returns -1 when p is false.
__device__ __forceinline__ int emit_slot_warp(int32_t *counter, bool p) {
    const unsigned act = __ballot_sync(0xffffffffu, p);
    if (act == 0) return -1;
    const int lane = threadIdx.x & 31;
    const int lead = __ffs(act) - 1;
    int base = 0;
    if (lane == lead) base = atomicAdd(counter, __popc(act));
    base = __shfl_sync(0xffffffffu, base, lead);
    return p ? base + __popc(act & ((1u << lane) - 1u)) : -1;
}

// Top-k of n keyed elements by MSD radix select on the 64-bit order keys, ties
// on the key broken by ascending index (radix select on the index bits).
// acc(i, key, idx) -> valid.  The block size must be a multiple of 32; every
// thread calls it.  Up to ITEMS * blockDim elements are cached in registers.
template <int ITEMS = SEL_ITEMS, class Acc>
__device__ int64_t block_select(int64_t n, int64_t k, Acc acc, SelectSmem &sm, uint64_t *out_key,
                                int64_t *out_idx) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const bool cached = n <= (int64_t)ITEMS * nt;
    uint64_t ck[ITEMS];
    int64_t ci[ITEMS];
    bool cv[ITEMS];
    if (tid == 0) {
        sm.cnt = 0;
        sm.out_n = 0;
    }
    __syncthreads();
    uint32_t c = 0;
    if (cached) {
#pragma unroll
        for (int j = 0; j < ITEMS; j++) {
            const int64_t i = tid + (int64_t)j * nt;
            cv[j] = i < n && acc(i, ck[j], ci[j]);
            c += cv[j];
        }
    } else {
        for (int64_t i = tid; i < n; i += nt) {
            uint64_t kk;
            int64_t ii;
            c += acc(i, kk, ii);
        }
    }
    // f(valid, key, idx) on every element, all lanes of a warp in step
    auto each = [&](auto f) {
        if (cached) {
#pragma unroll
            for (int j = 0; j < ITEMS; j++) f(cv[j], ck[j], ci[j]);
        } else {
            for (int64_t b = 0; b < n; b += nt) {
                const int64_t i = b + tid;
                uint64_t kk = 0;
                int64_t ii = 0;
                const bool v = i < n && acc(i, kk, ii);
                f(v, kk, ii);
            }
        }
    };
    c = __reduce_add_sync(0xffffffffu, c);
    if ((tid & 31) == 0) atomicAdd(&sm.cnt, c);
    __syncthreads();
    const int64_t n_valid = (int64_t)sm.cnt;
    auto emit_if = [&](auto pred) {
        each([&](bool v, uint64_t kk, int64_t ii) {
            const int p = emit_slot_warp(&sm.out_n, v && pred(kk, ii));
            if (p >= 0) {
                out_key[p] = kk;
                out_idx[p] = ii;
            }
        });
        __syncthreads();
    };
    if (n_valid <= k) {
        emit_if([](uint64_t, int64_t) { return true; });
        return n_valid;
    }
    uint64_t prefix = 0, mask = 0;
    if (tid == 0) {
        sm.krem = k;
        sm.done = 0;
    }
    for (int shift = 56; shift >= 0; shift -= 8) {
        sm.hist[tid] = 0;
        __syncthreads();
        each([&](bool v, uint64_t kk, int64_t) {
            hist_add_warp(sm.hist, v && (kk & mask) == prefix, (uint32_t)(kk >> shift) & 255u);
        });
        __syncthreads();
        pick_digit(sm, prefix, shift, true);
        prefix = sm.prefix;
        mask |= (0xffull << shift);
        if (sm.done) {
            emit_if([&](uint64_t kk, int64_t) { return (kk & mask) >= prefix; });
            return k;
        }
    }
    const uint64_t kstar = prefix;
    uint64_t ipre = 0, imask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        sm.hist[tid] = 0;
        __syncthreads();
        each([&](bool v, uint64_t kk, int64_t ii) {
            hist_add_warp(sm.hist, v && kk == kstar && (((uint64_t)ii) & imask) == ipre,
                          (uint32_t)(((uint64_t)ii) >> shift) & 255u);
        });
        __syncthreads();
        pick_digit(sm, ipre, shift, false);
        ipre = sm.prefix;
        imask |= (0xffull << shift);
        if (sm.done) break;  // {index & imask <= ipre} among the key ties is exactly what is left
    }
    emit_if([&](uint64_t kk, int64_t ii) {
        return kk > kstar || (kk == kstar && (((uint64_t)ii) & imask) <= ipre);
    });
    return k;
}

__device__ void block_sort_pairs(uint64_t *key, int64_t *idx, int P) {
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                int j = i ^ stride;
                if (j > i) {
                    bool up = (i & size) == 0;  // ascending in "goes first" order
                    uint64_t ka = key[i], kb = key[j];
                    int64_t ia = idx[i], ib = idx[j];
                    bool a_first = ka > kb || (ka == kb && ia < ib);
                    if (up ? !a_first : a_first) {
                        key[i] = kb;
                        key[j] = ka;
                        idx[i] = ib;
                        idx[j] = ia;
                    }
                }
            }
        }
    }
    __syncthreads();
}

template <typename T>
struct FinalArgs {
    int64_t n_u;
    int32_t B, k, exclude, want_scores;
    int32_t chunk, n_chunks;
    const T *EST;
    const T *P;
    const double *ws_u;
    const int32_t *perm_u;  // store -> caller U index (null: identity)
    double alpha;
    const Finish *fin;
    const Control *ctl;
    double *outs;        // [B][n_u] per-slot score rows (store order)
    double *out_scores;  // [n_q][n_u] or null (caller's order)
    uint64_t *cand_key;  // [B][n_chunks][k]
    int64_t *cand_idx;
    int32_t *topk_idx;   // [n_q][k]
    double *topk_score;  // [n_q][k]
    bh_trace *trace;     // [n_q]
    int32_t *chunk_done; // [B] chunks finished per finishing slot (zero between rounds)
};

// Per-slot score row the chunk select reads: the caller's output row directly
// when the store keeps the caller's order, else the slot's OUTS row (store
// order; the caller's row is written through perm_u beside it).
template <typename T>
__device__ __forceinline__ double *score_row(const FinalArgs<T> &a, int s, const Finish &f) {
    return a.want_scores && !a.perm_u ? a.out_scores + (int64_t)f.qidx * a.n_u : a.outs + (int64_t)s * a.n_u;
}

// Merge the chunk candidates of finished slot s, sort, write top-k + trace.
template <typename T>
__device__ void merge_slot(const FinalArgs<T> &a, int s, const Finish &f, SelectSmem &sm, uint64_t *skey,
                           int64_t *sidx) {
    if (threadIdx.x == 0) a.trace[f.qidx] = f.trace;
    if (a.k <= 0 || f.job == BH_JOB_SS_PUSH || f.job == BH_JOB_SELECTIVE || !a.topk_idx) return;
    const uint64_t *ck = a.cand_key + (int64_t)s * a.n_chunks * a.k;
    const int64_t *ci = a.cand_idx + (int64_t)s * a.n_chunks * a.k;
    auto acc = [&](int64_t i, uint64_t &kk, int64_t &ii) -> bool {
        ii = __ldcg(ci + i);
        kk = __ldcg(ck + i);
        return ii >= 0;
    };
    int P = 1;
    while (P < a.k) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        skey[i] = 0;
        sidx[i] = INT64_MAX;
    }
    __syncthreads();
    const int64_t m = block_select<SEL_ITEMS_MERGE>((int64_t)a.n_chunks * a.k, a.k, acc, sm, skey, sidx);
    block_sort_pairs(skey, sidx, P);
    for (int i = threadIdx.x; i < a.k; i += blockDim.x) {
        const bool ok = i < m;
        a.topk_idx[(int64_t)f.qidx * a.k + i] = ok ? (int32_t)sidx[i] : -1;
        if (a.topk_score) a.topk_score[(int64_t)f.qidx * a.k + i] = ok ? key_value(skey[i]) : 0.0;
    }
}

// K5: scores + chunk top-k candidates per (finished slot, chunk); the last
// chunk block of a slot merges (K6 folded in: no extra launch per round).
template <typename T>
__global__ void __launch_bounds__(TOPK_THREADS) k_finalize(FinalArgs<T> a) {
    pdl_begin();
    const int n_fin = a.ctl->n_fin;
    if (n_fin == 0) return;
    __shared__ SelectSmem sm;
    __shared__ uint64_t skey[TOPK_MAX];
    __shared__ int64_t sidx[TOPK_MAX];
    __shared__ int s_last;
    const int B = a.B;
    for (int64_t p = blockIdx.x; p < (int64_t)n_fin * a.n_chunks; p += gridDim.x) {
        const int fi = (int)(p / a.n_chunks);
        const int c = (int)(p % a.n_chunks);
        const int s = a.ctl->fin_slots[fi];
        const Finish f = a.fin[s];
        const bool scores = !(f.job == BH_JOB_SS_PUSH || f.job == BH_JOB_SELECTIVE);
        if (scores) {
            double *dst = score_row(a, s, f);
            const int64_t u0 = (int64_t)c * a.chunk;
            const int64_t u1 = imin64(a.n_u, u0 + a.chunk);
            // SEL_ITEMS nodes per thread, all loads issued before any is used
            // (a chunk is SEL_ITEMS * blockDim nodes; the columns are strided reads)
            const bool need_p = f.job == BH_JOB_POWER || f.has_pi;
            for (int64_t ub = u0; ub < u1; ub += (int64_t)SEL_ITEMS * blockDim.x) {
                T ev[SEL_ITEMS], pv[SEL_ITEMS];
                double wv[SEL_ITEMS];
#pragma unroll
                for (int j = 0; j < SEL_ITEMS; j++) {
                    const int64_t u = ub + threadIdx.x + (int64_t)j * blockDim.x;
                    ev[j] = pv[j] = (T)0;
                    wv[j] = 0.0;
                    if (u < u1) {
                        ev[j] = a.EST[u * B + s];
                        wv[j] = a.ws_u[u];
                        if (need_p) pv[j] = a.P[u * B + s];
                    }
                }
#pragma unroll
                for (int j = 0; j < SEL_ITEMS; j++) {
                    const int64_t u = ub + threadIdx.x + (int64_t)j * blockDim.x;
                    if (u >= u1) continue;
                    const double est = (double)ev[j];
                    const double ws = wv[j];
                    double v;
                    if (f.job == BH_JOB_POWER) {
                        v = a.alpha * (ws * (double)pv[j]);
                    } else {
                        v = (ws * f.inv_ws_q) * est;                               // w_ratio * est
                        if (f.has_pi) v = v + a.alpha * (ws * (double)pv[j]);       // + alpha acc_t
                        if (f.job == BH_JOB_BHPP) v = v + est;                      // + backward est
                    }
                    dst[u] = v;
                    if (a.want_scores && a.perm_u) a.out_scores[(int64_t)f.qidx * a.n_u + a.perm_u[u]] = v;
                }
            }
            if (a.k > 0) {
                __syncthreads();
                const int64_t excl = (a.exclude && f.job == BH_JOB_BHPP) ? f.src : -1;
                // candidates carry the caller's index: ties break by it (bhpp_query.py:210)
                auto acc = [&](int64_t i, uint64_t &kk, int64_t &ii) -> bool {
                    kk = order_key(dst[u0 + i]);
                    ii = a.perm_u ? (int64_t)a.perm_u[u0 + i] : u0 + i;
                    return ii != excl;
                };
                uint64_t *ck = a.cand_key + ((int64_t)s * a.n_chunks + c) * a.k;
                int64_t *ci = a.cand_idx + ((int64_t)s * a.n_chunks + c) * a.k;
                const int64_t m = block_select(u1 - u0, a.k, acc, sm, ck, ci);
                for (int64_t i = m + threadIdx.x; i < a.k; i += blockDim.x) ci[i] = -1;
            }
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(a.chunk_done + s, 1) == a.n_chunks - 1;
        __syncthreads();
        if (s_last) {
            __threadfence();
            merge_slot(a, s, f, sm, skey, sidx);
            if (threadIdx.x == 0) a.chunk_done[s] = 0;
        }
        __syncthreads();
    }
}

// Standalone top-k of one device vector (bh_topk): chunk select + merge.
__global__ void __launch_bounds__(TOPK_THREADS) k_vec_topk_chunks(const double *x, int64_t n, int64_t k,
                                                                  int64_t exclude, int64_t chunk,
                                                                  uint64_t *ck, int64_t *ci) {
    __shared__ SelectSmem sm;
    const int64_t u0 = (int64_t)blockIdx.x * chunk;
    const int64_t u1 = imin64(n, u0 + chunk);
    auto acc = [&](int64_t i, uint64_t &kk, int64_t &ii) -> bool {
        ii = u0 + i;
        const double v = x[ii];
        kk = order_key(v);
        return ii != exclude && v == v;
    };
    uint64_t *okey = ck + (int64_t)blockIdx.x * k;
    int64_t *oidx = ci + (int64_t)blockIdx.x * k;
    const int64_t m = block_select(u1 - u0, k, acc, sm, okey, oidx);
    for (int64_t i = m + threadIdx.x; i < k; i += blockDim.x) oidx[i] = -1;
}

__global__ void __launch_bounds__(TOPK_THREADS) k_vec_topk_merge(int64_t n_cand, int64_t k, const uint64_t *ck,
                                                                 const int64_t *ci, int64_t *out_idx,
                                                                 double *out_score, int64_t *out_count) {
    __shared__ SelectSmem sm;
    __shared__ uint64_t skey[TOPK_MAX];
    __shared__ int64_t sidx[TOPK_MAX];
    auto acc = [&](int64_t i, uint64_t &kk, int64_t &ii) -> bool {
        ii = ci[i];
        kk = ck[i];
        return ii >= 0;
    };
    int P = 1;
    while (P < k) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        skey[i] = 0;
        sidx[i] = INT64_MAX;
    }
    __syncthreads();
    const int64_t m = block_select<SEL_ITEMS_MERGE>(n_cand, k, acc, sm, skey, sidx);
    block_sort_pairs(skey, sidx, P);
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        out_idx[i] = sidx[i];
        out_score[i] = key_value(skey[i]);
    }
    if (threadIdx.x == 0) *out_count = m;
}

}  // namespace bh
