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
#include <cstring>

#include "common.cuh"

namespace bh {

namespace {

template <typename T>
__global__ void k_prescale(int64_t n_rows, int64_t n_e, const int64_t *__restrict__ indptr,
                           const double *__restrict__ w, const double *__restrict__ ws,
                           T *__restrict__ vals) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_e;
         e += (int64_t)gridDim.x * blockDim.x) {
        // row of edge e: last r with indptr[r] <= e
        int64_t lo = 0, hi = n_rows - 1;
        while (lo < hi) {
            int64_t mid = (lo + hi + 1) >> 1;
            if (indptr[mid] <= e) lo = mid; else hi = mid - 1;
        }
        vals[e] = (T)(w[e] / ws[lo]);
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

template <typename T>
void upload_side(Side &s, int64_t n_rows, int64_t n_e, const int64_t *indptr, const int32_t *indices,
                 const double *w, const double *ws_rows, int64_t &acc) {
    s.n_rows = n_rows;
    s.indptr = dmalloc<int64_t>(n_rows + 1, acc);
    s.indices = dmalloc<int32_t>(n_e, acc);
    s.vals = dmalloc<T>(n_e, acc);
    s.deg = dmalloc<int32_t>(n_rows, acc);
    BH_CUDA(cudaMemcpy(s.indptr, indptr, (n_rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    BH_CUDA(cudaMemcpy(s.indices, indices, n_e * sizeof(int32_t), cudaMemcpyHostToDevice));
    int64_t tmp = 0;
    double *dw = dmalloc<double>(n_e, tmp);
    double *dws = dmalloc<double>(n_rows, tmp);
    BH_CUDA(cudaMemcpy(dw, w, n_e * sizeof(double), cudaMemcpyHostToDevice));
    BH_CUDA(cudaMemcpy(dws, ws_rows, n_rows * sizeof(double), cudaMemcpyHostToDevice));
    k_prescale<T><<<grid_for(n_e), 256>>>(n_rows, n_e, s.indptr, dw, dws, (T *)s.vals);
    count_launch();
    BH_CUDA(cudaGetLastError());
    k_deg<<<grid_for(n_rows), 256>>>(n_rows, s.indptr, s.deg);
    count_launch();
    BH_CUDA(cudaGetLastError());
    BH_CUDA(cudaDeviceSynchronize());
    cudaFree(dw);
    cudaFree(dws);
    s.h_indptr.assign(indptr, indptr + n_rows + 1);
}

void free_side(Side &s) {
    cudaFree(s.indptr);
    cudaFree(s.indices);
    cudaFree(s.vals);
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
                       const double *ws_v, int32_t device, int32_t dtype) {
    if (dtype != BH_DTYPE_F64 && dtype != BH_DTYPE_F32) throw InvalidArg("dtype must be BH_DTYPE_F64 or BH_DTYPE_F32");
    validate(n_u, n_v, n_e, u_indptr, u_indices, v_indptr, v_indices, ws_u, ws_v);
    BH_CUDA(cudaSetDevice(device));
    bh_graph *g = new bh_graph();
    g->device = device;
    g->dtype = dtype;
    g->n_u = n_u;
    g->n_v = n_v;
    g->n_e = n_e;
    try {
        int64_t acc = 0;
        if (dtype == BH_DTYPE_F64) {
            upload_side<double>(g->U, n_u, n_e, u_indptr, u_indices, u_weights, ws_u, acc);
            upload_side<double>(g->V, n_v, n_e, v_indptr, v_indices, v_weights, ws_v, acc);
        } else {
            upload_side<float>(g->U, n_u, n_e, u_indptr, u_indices, u_weights, ws_u, acc);
            upload_side<float>(g->V, n_v, n_e, v_indptr, v_indices, v_weights, ws_v, acc);
        }
        g->ws_u = dmalloc<double>(n_u, acc);
        g->inv_ws_u = dmalloc<double>(n_u, acc);
        BH_CUDA(cudaMemcpy(g->ws_u, ws_u, n_u * sizeof(double), cudaMemcpyHostToDevice));
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
