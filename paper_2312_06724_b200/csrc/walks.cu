// walks.cu -- Monte-Carlo restart walks (reference baselines.py:108-151, the
// forward half of MCSP) on the device graph store.
//
// One thread per walk.  A walk stops with probability alpha before every step
// and otherwise moves U -> V -> U, each leg a weight-proportional neighbour
// draw through the reference's alias tables (build_alias, baselines.py:45-83):
// slot = floor(r * deg), keep it if r' < prob[slot], else jump to alias[slot].
// Random numbers: counter-based Philox4x32-10 keyed by (seed, walk index), so
// a run is reproducible whatever the launch geometry (the reference uses numpy
// substreams per batch; the two are different streams of the same law).
// Stop counts are aggregated per warp on equal nodes before the atomic, since
// every walk is at the source on its first step.
#include <curand_kernel.h>

#include <algorithm>

#include "common.cuh"

namespace bh {

namespace {

struct WalkSide {
    const int64_t *indptr;
    const int32_t *indices;
    const double *prob;
    const int32_t *alias;  // local slot offsets within the row
};

__device__ __forceinline__ int64_t draw(const WalkSide &s, int64_t node, curandStatePhilox4_32_10_t &st) {
    const int64_t row = __ldg(s.indptr + node);
    const int64_t deg = __ldg(s.indptr + node + 1) - row;
    const double r0 = 1.0 - curand_uniform_double(&st);  // [0, 1), as numpy's random()
    const double r1 = 1.0 - curand_uniform_double(&st);
    int64_t slot = (int64_t)(r0 * (double)deg);
    if (slot >= deg) slot = deg - 1;
    int64_t pos = row + slot;
    if (!(r1 < __ldg(s.prob + pos))) pos = row + __ldg(s.alias + pos);
    return __ldg(s.indices + pos);
}

__global__ void k_mc_walks(WalkSide us, WalkSide vs, int64_t source, double alpha, int64_t first, int64_t n,
                           uint64_t seed, unsigned long long *counts) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        curandStatePhilox4_32_10_t st;
        curand_init(seed, (unsigned long long)(first + i), 0, &st);
        int64_t cur = source;
        while (true) {
            const double r = 1.0 - curand_uniform_double(&st);
            if (r < alpha) break;
            cur = draw(vs, draw(us, cur, st), st);
        }
        const unsigned active = __activemask();
        const unsigned peers = __match_any_sync(active, (unsigned long long)cur);
        if (lane == __ffs(peers) - 1) atomicAdd(counts + cur, (unsigned long long)__popc(peers));
    }
}

template <typename X>
X *dcopy(const X *h, size_t n) {
    X *d = nullptr;
    cudaError_t e = cudaMalloc(&d, std::max<size_t>(1, n) * sizeof(X));
    if (e == cudaErrorMemoryAllocation) {
        (void)cudaGetLastError();
        throw std::bad_alloc();
    }
    BH_CUDA(e);
    BH_CUDA(cudaMemcpy(d, h, n * sizeof(X), cudaMemcpyHostToDevice));
    return d;
}

}  // namespace

// Per-slot tables of one side (caller's CSR order) into the store's row order:
// a relabelled store row keeps its caller row's edge order, so each row's slots
// move as one block and the local alias offsets stay valid.
static void to_store_order(const Side &s, const double *prob, const int64_t *alias, std::vector<double> &p,
                           std::vector<int32_t> &al) {
    const int64_t E = s.h_indptr.back();
    p.resize((size_t)E);
    al.resize((size_t)E);
    std::vector<int64_t> cip;  // caller's row offsets
    if (!s.h_perm.empty()) {
        cip.assign((size_t)s.n_rows + 1, 0);
        for (int64_t i = 0; i < s.n_rows; i++) cip[(size_t)s.h_perm[i] + 1] = s.h_indptr[i + 1] - s.h_indptr[i];
        for (int64_t r = 0; r < s.n_rows; r++) cip[r + 1] += cip[r];
    }
    for (int64_t i = 0; i < s.n_rows; i++) {
        const int64_t o = s.h_perm.empty() ? s.h_indptr[i] : cip[(size_t)s.h_perm[i]];
        for (int64_t k = 0, n = s.h_indptr[i]; n < s.h_indptr[i + 1]; k++, n++) {
            p[(size_t)n] = prob[o + k];
            al[(size_t)n] = (int32_t)alias[o + k];
        }
    }
}

bh_alias *alias_create(bh_graph *g, const double *u_prob, const int64_t *u_alias, const double *v_prob,
                       const int64_t *v_alias) {
    BH_CUDA(cudaSetDevice(g->device));
    const int64_t E = g->n_e;
    std::vector<double> up, vp;
    std::vector<int32_t> ua, va;
    to_store_order(g->U, u_prob, u_alias, up, ua);
    to_store_order(g->V, v_prob, v_alias, vp, va);
    auto *a = new bh_alias();
    a->g = g;
    a->device = g->device;
    try {
        a->u_prob = dcopy(up.data(), E);
        a->v_prob = dcopy(vp.data(), E);
        a->u_alias = dcopy(ua.data(), E);
        a->v_alias = dcopy(va.data(), E);
    } catch (...) {
        delete a;
        throw;
    }
    return a;
}

// counts[u] += number of the walks [first, first + n) that stop at u.
void mc_walks(const bh_alias *al, int64_t source, double alpha, int64_t first, int64_t n, uint64_t seed,
              int64_t *counts_host) {
    bh_graph *g = al->g;
    BH_CUDA(cudaSetDevice(g->device));
    unsigned long long *dc = nullptr;
    BH_CUDA(cudaMalloc(&dc, std::max<int64_t>(1, g->n_u) * sizeof(unsigned long long)));
    BH_CUDA(cudaMemset(dc, 0, g->n_u * sizeof(unsigned long long)));
    WalkSide us{g->U.indptr, g->U.indices, al->u_prob, al->u_alias};
    WalkSide vs{g->V.indptr, g->V.indices, al->v_prob, al->v_alias};
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (n > 0) {
        k_mc_walks<<<grid, 256>>>(us, vs, g->U.to_store(source), alpha, first, n, seed, dc);
        count_launch();
    }
    cudaError_t e = cudaGetLastError();
    std::vector<unsigned long long> hc((size_t)g->n_u);
    if (e == cudaSuccess) e = cudaMemcpy(hc.data(), dc, g->n_u * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(dc);
    BH_CUDA(e);
    for (int64_t u = 0; u < g->n_u; u++) counts_host[g->U.h_perm.empty() ? u : g->U.h_perm[u]] += (int64_t)hc[u];
}

}  // namespace bh
