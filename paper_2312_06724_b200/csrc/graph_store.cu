// graph_store.cu -- K-G: the immutable device graph store.
//
// Holds both CSR sides of the weighted biadjacency with the inverse weight-sum
// scaling fused into the stored values (SURVEY.md sec. 2 "K-G"):
//   U side (rows u):  indices v, vals w(u,v)/ws(u)   == u_step.data  (bigraph.py:148-155)
//   V side (rows v):  indices u, vals w(u,v)/ws(v)   == v_step.data  (bigraph.py:157-164)
// The two transposed operators the reference keeps for power_iteration
// (u_step_t / v_step_t, bigraph.py:166-174, and recv_uv / recv_vu) are not
// stored: the engine runs power iteration on acc/ws, which uses these same two
// arrays (detailed balance ws_i P_ij = ws_j P_ji).
// Values are computed in fp64 (IEEE division, as numpy does) and rounded once
// to the storage type.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace bh {

namespace {

// Store row i = caller row perm[i] (identity when perm is null), its edges in
// the caller's order with the columns mapped to store indices (inv_col) and
// the values prescaled: vals = w / ws(row), computed in fp64 and rounded once.
// One warp per row, grid-stride.
template <typename T>
__global__ void k_build_rows(int64_t n_rows, const int64_t *__restrict__ old_indptr, const int32_t *__restrict__ old_idx,
                             const double *__restrict__ w, const double *__restrict__ ws_old,
                             const int32_t *__restrict__ perm, const int32_t *__restrict__ inv_col,
                             const int64_t *__restrict__ new_indptr, int32_t *__restrict__ new_idx,
                             T *__restrict__ vals, EdgeRF<T> *__restrict__ ecv, int32_t *__restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n_rows; i += nw) {
        const int64_t r = perm ? perm[i] : i;
        const int64_t o = old_indptr[r], deg = old_indptr[r + 1] - o, n = new_indptr[i];
        const double ws = ws_old[r];
        for (int64_t k = lane; k < deg; k += 32) {
            const int32_t c0 = old_idx[o + k];
            const int32_t c = inv_col ? inv_col[c0] : c0;
            const T v = (T)(w[o + k] / ws);
            new_idx[n + k] = c;
            vals[n + k] = v;
            if (ecv) ecv[n + k] = EdgeRF<T>{c, k == deg - 1 ? -v : v};
            if (!(v > (T)0)) atomicOr(bad, 1);  // the sign carries the row end: needs v > 0
        }
    }
}

__global__ void k_deg(int64_t n, const int64_t *__restrict__ indptr, int32_t *__restrict__ deg) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        deg[r] = (int32_t)(indptr[r + 1] - indptr[r]);
}

__global__ void k_inv(int64_t n, const double *__restrict__ ws, double *__restrict__ inv) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        inv[r] = 1.0 / ws[r];
}

int grid_for(int64_t n, int threads = 256) {
    int64_t b = (n + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

template <typename X>
X *dmalloc(size_t count, int64_t &acc) {
    void *p = nullptr;
    size_t bytes = std::max<size_t>(1, count * sizeof(X));
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        (void)cudaGetLastError();
        throw std::bad_alloc();
    }
    if (e != cudaSuccess) throw CudaError(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    acc += (int64_t)bytes;
    return (X *)p;
}

// Degree-descending order of one side, stable in the caller's index (counting
// sort on the degree): perm[new] = old, inv[old] = new.
void degree_order(int64_t n, const int64_t *indptr, std::vector<int32_t> &perm, std::vector<int32_t> &inv) {
    int64_t dmax = 0;
    for (int64_t r = 0; r < n; r++) dmax = std::max(dmax, indptr[r + 1] - indptr[r]);
    std::vector<int64_t> start((size_t)dmax + 2, 0);
    for (int64_t r = 0; r < n; r++) start[(size_t)(dmax - (indptr[r + 1] - indptr[r])) + 1]++;
    for (size_t d = 1; d < start.size(); d++) start[d] += start[d - 1];
    perm.assign((size_t)n, 0);
    inv.assign((size_t)n, 0);
    for (int64_t r = 0; r < n; r++) {
        const int64_t p = start[(size_t)(dmax - (indptr[r + 1] - indptr[r]))]++;
        perm[(size_t)p] = (int32_t)r;
        inv[(size_t)r] = (int32_t)p;
    }
}

// Upload one side in store order.  `perm` (this side's rows) and `inv_col` (the
// other side's caller -> store map) are host vectors, empty for the identity.
template <typename T>
void upload_side(Side &s, int64_t n_rows, int64_t n_e, const int64_t *indptr, const int32_t *indices,
                 const double *w, const double *ws_rows, const std::vector<int32_t> &perm,
                 const std::vector<int32_t> &inv, const std::vector<int32_t> &inv_col, int64_t &acc) {
    s.n_rows = n_rows;
    s.indptr = dmalloc<int64_t>(n_rows + 1, acc);
    s.indices = dmalloc<int32_t>(n_e, acc);
    s.vals = dmalloc<T>(n_e, acc);
    s.deg = dmalloc<int32_t>(n_rows, acc);
    // the dense pulls' flagged edge stream needs every row non-empty (validated) and every
    // prescaled value positive in T (checked on the device below); otherwise the row-pointer
    // pull serves this store
    bool no_empty_row = true;
    for (int64_t i = 0; i < n_rows && no_empty_row; i++) no_empty_row = indptr[i + 1] > indptr[i];
    int64_t ecv_bytes = 0;
    s.ecv = no_empty_row ? (void *)dmalloc<EdgeRF<T>>(n_e, ecv_bytes) : nullptr;
    acc += ecv_bytes;
    std::vector<int64_t> nip;
    const int64_t *new_ip = indptr;
    if (!perm.empty()) {
        nip.assign((size_t)n_rows + 1, 0);
        for (int64_t i = 0; i < n_rows; i++) nip[i + 1] = nip[i] + (indptr[perm[i] + 1] - indptr[perm[i]]);
        new_ip = nip.data();
        s.perm = dmalloc<int32_t>(n_rows, acc);
        s.inv = dmalloc<int32_t>(n_rows, acc);
        BH_CUDA(cudaMemcpy(s.perm, perm.data(), n_rows * sizeof(int32_t), cudaMemcpyHostToDevice));
        BH_CUDA(cudaMemcpy(s.inv, inv.data(), n_rows * sizeof(int32_t), cudaMemcpyHostToDevice));
        s.h_perm = perm;
        s.h_inv = inv;
    }
    BH_CUDA(cudaMemcpy(s.indptr, new_ip, (n_rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    int64_t tmp = 0;
    int64_t *d_oip = dmalloc<int64_t>(n_rows + 1, tmp);
    int32_t *d_oidx = dmalloc<int32_t>(n_e, tmp);
    double *dw = dmalloc<double>(n_e, tmp);
    double *dws = dmalloc<double>(n_rows, tmp);
    int32_t *d_invc = inv_col.empty() ? nullptr : dmalloc<int32_t>(inv_col.size(), tmp);
    int32_t *d_bad = dmalloc<int32_t>(1, tmp);
    BH_CUDA(cudaMemset(d_bad, 0, sizeof(int32_t)));
    BH_CUDA(cudaMemcpy(d_oip, indptr, (n_rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    BH_CUDA(cudaMemcpy(d_oidx, indices, n_e * sizeof(int32_t), cudaMemcpyHostToDevice));
    BH_CUDA(cudaMemcpy(dw, w, n_e * sizeof(double), cudaMemcpyHostToDevice));
    BH_CUDA(cudaMemcpy(dws, ws_rows, n_rows * sizeof(double), cudaMemcpyHostToDevice));
    if (d_invc) BH_CUDA(cudaMemcpy(d_invc, inv_col.data(), inv_col.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    k_build_rows<T><<<grid_for(n_rows * 32), 256>>>(n_rows, d_oip, d_oidx, dw, dws, s.perm, d_invc, s.indptr,
                                                     s.indices, (T *)s.vals, (EdgeRF<T> *)s.ecv, d_bad);
    count_launch();
    BH_CUDA(cudaGetLastError());
    k_deg<<<grid_for(n_rows), 256>>>(n_rows, s.indptr, s.deg);
    count_launch();
    BH_CUDA(cudaGetLastError());
    BH_CUDA(cudaDeviceSynchronize());
    int32_t bad = 0;
    BH_CUDA(cudaMemcpy(&bad, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (bad && s.ecv) {  // a zero, negative or underflowed value: no flagged stream
        cudaFree(s.ecv);
        s.ecv = nullptr;
        acc -= ecv_bytes;
    }
    cudaFree(d_bad);
    cudaFree(d_oip);
    cudaFree(d_oidx);
    cudaFree(dw);
    cudaFree(dws);
    cudaFree(d_invc);
    s.h_indptr.assign(new_ip, new_ip + n_rows + 1);
}

void free_side(Side &s) {
    cudaFree(s.perm);
    cudaFree(s.inv);
    cudaFree(s.indptr);
    cudaFree(s.indices);
    cudaFree(s.vals);
    cudaFree(s.ecv);
    cudaFree(s.deg);
    s = Side{};
}

void validate(int64_t n_u, int64_t n_v, int64_t n_e, const int64_t *u_indptr, const int32_t *u_indices,
              const int64_t *v_indptr, const int32_t *v_indices, const double *ws_u, const double *ws_v) {
    if (n_u <= 0 || n_v <= 0 || n_e <= 0) throw InvalidArg("graph must have nodes and edges");
    if (n_u >= (1LL << 31) || n_v >= (1LL << 31)) throw InvalidArg("node count exceeds int32");
    if (u_indptr[0] != 0 || u_indptr[n_u] != n_e || v_indptr[0] != 0 || v_indptr[n_v] != n_e)
        throw InvalidArg("corrupt CSR offsets");
    for (int64_t r = 0; r < n_u; r++)
        if (u_indptr[r + 1] <= u_indptr[r]) throw InvalidArg("isolated or unordered U row");
    for (int64_t r = 0; r < n_v; r++)
        if (v_indptr[r + 1] <= v_indptr[r]) throw InvalidArg("isolated or unordered V row");
    for (int64_t e = 0; e < n_e; e++) {
        if (u_indices[e] < 0 || u_indices[e] >= n_v) throw InvalidArg("U-CSR column out of range");
        if (v_indices[e] < 0 || v_indices[e] >= n_u) throw InvalidArg("V-CSR column out of range");
    }
    for (int64_t r = 0; r < n_u; r++)
        if (!(ws_u[r] > 0.0)) throw InvalidArg("ws_u must be positive");
    for (int64_t r = 0; r < n_v; r++)
        if (!(ws_v[r] > 0.0)) throw InvalidArg("ws_v must be positive");
}

}  // namespace

bh_graph *graph_create(int64_t n_u, int64_t n_v, int64_t n_e, const int64_t *u_indptr,
                       const int32_t *u_indices, const double *u_weights, const int64_t *v_indptr,
                       const int32_t *v_indices, const double *v_weights, const double *ws_u,
                       const double *ws_v, int32_t device, int32_t dtype_flags) {
    const int32_t dtype = dtype_flags & 0xff;
    if (dtype != BH_DTYPE_F64 && dtype != BH_DTYPE_F32) throw InvalidArg("dtype must be BH_DTYPE_F64 or BH_DTYPE_F32");
    if (dtype_flags & ~(0xff | BH_GRAPH_KEEP_ORDER)) throw InvalidArg("unknown graph flag");
    validate(n_u, n_v, n_e, u_indptr, u_indices, v_indptr, v_indices, ws_u, ws_v);
    bool relabel = !(dtype_flags & BH_GRAPH_KEEP_ORDER);
    if (const char *m = getenv("BH_RELABEL")) relabel = atoi(m) != 0;  // A/B switch
    BH_CUDA(cudaSetDevice(device));
    bh_graph *g = new bh_graph();
    g->device = device;
    g->dtype = dtype;
    g->n_u = n_u;
    g->n_v = n_v;
    g->n_e = n_e;
    g->relabeled = relabel ? 1 : 0;
    try {
        std::vector<int32_t> pu, iu, pv, iv;
        if (relabel) {
            degree_order(n_u, u_indptr, pu, iu);
            degree_order(n_v, v_indptr, pv, iv);
        }
        int64_t acc = 0;
        if (dtype == BH_DTYPE_F64) {
            upload_side<double>(g->U, n_u, n_e, u_indptr, u_indices, u_weights, ws_u, pu, iu, iv, acc);
            upload_side<double>(g->V, n_v, n_e, v_indptr, v_indices, v_weights, ws_v, pv, iv, iu, acc);
        } else {
            upload_side<float>(g->U, n_u, n_e, u_indptr, u_indices, u_weights, ws_u, pu, iu, iv, acc);
            upload_side<float>(g->V, n_v, n_e, v_indptr, v_indices, v_weights, ws_v, pv, iv, iu, acc);
        }
        std::vector<double> wsu(ws_u, ws_u + n_u);
        if (relabel)
            for (int64_t i = 0; i < n_u; i++) wsu[i] = ws_u[pu[i]];
        g->ws_u = dmalloc<double>(n_u, acc);
        g->inv_ws_u = dmalloc<double>(n_u, acc);
        BH_CUDA(cudaMemcpy(g->ws_u, wsu.data(), n_u * sizeof(double), cudaMemcpyHostToDevice));
        k_inv<<<grid_for(n_u), 256>>>(n_u, g->ws_u, g->inv_ws_u);
        count_launch();
        BH_CUDA(cudaGetLastError());
        BH_CUDA(cudaDeviceSynchronize());
        g->device_bytes = acc;
    } catch (...) {
        free_side(g->U);
        free_side(g->V);
        cudaFree(g->ws_u);
        cudaFree(g->inv_ws_u);
        delete g;
        throw;
    }
    return g;
}

void graph_free_arrays(bh_graph *g) {
    free_side(g->U);
    free_side(g->V);
    cudaFree(g->ws_u);
    cudaFree(g->inv_ws_u);
    g->ws_u = g->inv_ws_u = nullptr;
}

}  // namespace bh
