// csr_build.cu -- graph ingestion on the device: edge triples -> both CSR sides.
//
// The reference BipartiteGraph constructor (bigraph.py:53-111) canonicalises
// an edge list with two lexsorts (rows by (u, v), then by (v, u)), rejects
// repeated pairs, and accumulates ws_u / ws_v with np.bincount over the
// (u, v)-sorted arrays.  At C3/C4 sizes (1e8-3e8 edges) those host sorts cost
// minutes.  Here the same canonical arrays come from two stable LSD radix
// sorts of the packed pair keys u*|V|+v and v*|U|+u on the device:
//   * the sorted order is unique (pairs are distinct), so indices and weights
//     are exactly the reference's;
//   * ws_u[u] / ws_v[v] are summed sequentially in CSR row order, which is
//     the order np.bincount visits them in the (u, v)-sorted arrays, so the
//     sums are bit-identical too.
// Radix sort: 8-bit digits; per pass a tile histogram, an exclusive scan of
// the digit-major [256][tiles] counts, and a stable scatter that ranks equal
// digits inside a tile with __match_any_sync (warp) and per-warp counts
// (block), in item order.  HBM-bound: ~24 B per element per pass.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace bh {

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

template <typename X>
struct DBuf {
    X *p = nullptr;
    explicit DBuf(size_t n) {
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(1, n * sizeof(X)));
        if (e == cudaErrorMemoryAllocation) {
            (void)cudaGetLastError();
            throw std::bad_alloc();
        }
        if (e != cudaSuccess) throw CudaError(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    ~DBuf() { cudaFree(p); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
};

int grid_of(int64_t n, int threads = 256) {
    const int64_t b = (n + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 64));
}

__global__ void k_rs_hist(const uint64_t *__restrict__ keys, int64_t n, int shift, uint32_t *__restrict__ hist,
                          int64_t tiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = blockIdx.x * (int64_t)RS_TILE;
#pragma unroll 4
    for (int i = 0; i < RS_ITEMS; i++) {
        const int64_t idx = base + i * RS_THREADS + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void k_rs_scatter(const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin,
                             uint64_t *__restrict__ kout, uint32_t *__restrict__ vout, int64_t n, int shift,
                             const uint64_t *__restrict__ offs, int64_t tiles) {
    __shared__ uint64_t base_d[256];
    __shared__ uint32_t run[256];
    __shared__ uint32_t wcnt[RS_WARPS][256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    base_d[tid] = offs[tid * tiles + blockIdx.x];
    run[tid] = 0;
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t base = blockIdx.x * (int64_t)RS_TILE;
    for (int it = 0; it < RS_ITEMS; it++) {
        const int64_t idx = base + it * RS_THREADS + tid;  // item order == global order in the tile
        const bool ok = idx < n;
        const uint64_t key = ok ? kin[idx] : 0;
        const uint32_t d = ok ? (uint32_t)((key >> shift) & 255u) : 256u;
#pragma unroll
        for (int w = 0; w < RS_WARPS; w++) wcnt[w][tid] = 0;
        __syncthreads();
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt);
        if (ok && rank == 0) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        if (ok) {
            uint32_t pre = 0;
            for (int w = 0; w < warp; w++) pre += wcnt[w][d];
            const uint64_t pos = base_d[d] + run[d] + pre + rank;
            kout[pos] = key;
            vout[pos] = vin[idx];
        }
        __syncthreads();
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; w++) tot += wcnt[w][tid];
        run[tid] += tot;
        __syncthreads();
    }
}

// Exclusive scan (int64 accumulation) of m counts, 1024 per block, recursive.
constexpr int SC_THREADS = 256, SC_PER = 4, SC_BLOCK = SC_THREADS * SC_PER;

template <typename X>
__global__ void k_scan_block(const X *__restrict__ in, int64_t m, uint64_t *__restrict__ out,
                             uint64_t *__restrict__ sums) {
    __shared__ uint64_t s[SC_THREADS];
    const int64_t b0 = blockIdx.x * (int64_t)SC_BLOCK + threadIdx.x * SC_PER;
    uint64_t v[SC_PER], t = 0;
#pragma unroll
    for (int j = 0; j < SC_PER; j++) {
        v[j] = b0 + j < m ? (uint64_t)in[b0 + j] : 0;
        t += v[j];
    }
    s[threadIdx.x] = t;
    __syncthreads();
    for (int off = 1; off < SC_THREADS; off <<= 1) {  // Hillis-Steele inclusive scan of thread totals
        const uint64_t x = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
        __syncthreads();
        s[threadIdx.x] += x;
        __syncthreads();
    }
    uint64_t run = s[threadIdx.x] - t;
#pragma unroll
    for (int j = 0; j < SC_PER; j++) {
        if (b0 + j < m) out[b0 + j] = run;
        run += v[j];
    }
    if (threadIdx.x == SC_THREADS - 1) sums[blockIdx.x] = s[threadIdx.x];
}

__global__ void k_scan_add(uint64_t *__restrict__ out, int64_t m, const uint64_t *__restrict__ add) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) out[i] += add[i / SC_BLOCK];
}

template <typename X>
void exclusive_scan(const X *in, int64_t m, uint64_t *out, cudaStream_t st) {
    const int64_t nb = (m + SC_BLOCK - 1) / SC_BLOCK;
    DBuf<uint64_t> sums(nb), sums_x(nb);
    k_scan_block<X><<<(unsigned)nb, SC_THREADS, 0, st>>>(in, m, out, sums.p);
    count_launch();
    if (nb > 1) {
        exclusive_scan<uint64_t>(sums.p, nb, sums_x.p, st);
        k_scan_add<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(out, m, sums_x.p);
        count_launch();
    }
    BH_CUDA(cudaGetLastError());
}

// Stable LSD sort of (key, val) by the low `bits` key bits; result in (k0, v0).
void radix_sort_pairs(uint64_t *k0, uint32_t *v0, uint64_t *k1, uint32_t *v1, int64_t n, int bits,
                      cudaStream_t st) {
    const int64_t tiles = (n + RS_TILE - 1) / RS_TILE;
    DBuf<uint32_t> hist(256 * tiles);
    DBuf<uint64_t> offs(256 * tiles);
    for (int shift = 0; shift < bits; shift += 8) {
        k_rs_hist<<<(unsigned)tiles, RS_THREADS, 0, st>>>(k0, n, shift, hist.p, tiles);
        count_launch();
        exclusive_scan<uint32_t>(hist.p, 256 * tiles, offs.p, st);
        k_rs_scatter<<<(unsigned)tiles, RS_THREADS, 0, st>>>(k0, v0, k1, v1, n, shift, offs.p, tiles);
        count_launch();
        BH_CUDA(cudaGetLastError());
        std::swap(k0, k1);
        std::swap(v0, v1);
    }
    if (((bits + 7) / 8) & 1) {  // odd pass count: result sits in the alternate buffers
        BH_CUDA(cudaMemcpyAsync(k1, k0, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
        BH_CUDA(cudaMemcpyAsync(v1, v0, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    }
}

__global__ void k_pack_keys(const int64_t *__restrict__ a, const int64_t *__restrict__ b, int64_t n, int64_t nb,
                            int64_t na, uint64_t *__restrict__ keys, uint32_t *__restrict__ vals,
                            int32_t *__restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = a[i], y = b[i];
        if (x < 0 || x >= na || y < 0 || y >= nb) {
            atomicOr(bad, 1);
            keys[i] = 0;
        } else {
            keys[i] = (uint64_t)x * (uint64_t)nb + (uint64_t)y;
        }
        vals[i] = (uint32_t)i;
    }
}

// Sorted keys -> (row, col) side arrays; duplicates flagged; row counts.
__global__ void k_unpack(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ perm,
                         const double *__restrict__ w_in, int64_t n, int64_t ncols, int32_t *__restrict__ col,
                         int64_t *__restrict__ row, double *__restrict__ w_out, uint64_t *__restrict__ deg,
                         int32_t *__restrict__ dup) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        const int64_t r = (int64_t)(k / (uint64_t)ncols);
        col[i] = (int32_t)(k % (uint64_t)ncols);
        if (row) row[i] = r;
        w_out[i] = w_in[perm[i]];
        atomicAdd((unsigned long long *)(deg + r), 1ull);
        if (i > 0 && keys[i - 1] == k) atomicOr(dup, 1);
    }
}

// V-side keys from the U-side canonical arrays: v * |U| + u, payload = U-order position.
__global__ void k_pack_transpose(const int64_t *__restrict__ urow, const int32_t *__restrict__ vcol, int64_t n,
                                 int64_t nu, uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = (uint64_t)vcol[i] * (uint64_t)nu + (uint64_t)urow[i];
        vals[i] = (uint32_t)i;
    }
}

// Row sums in CSR order (one thread per row, sequential: np.bincount's order).
__global__ void k_row_sums(const uint64_t *__restrict__ indptr, int64_t nrows, const double *__restrict__ w,
                           double *__restrict__ ws) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (uint64_t e = indptr[r]; e < indptr[r + 1]; e++) s += w[e];
        ws[r] = s;
    }
}

int key_bits(uint64_t max_key) {
    int b = 0;
    while (b < 64 && (max_key >> b) != 0) b++;
    return std::max(8, (b + 7) / 8 * 8);
}

}  // namespace

// Returns 0, or 1 when a pair repeats ("duplicate edge passed to constructor").
int csr_build(int64_t n_u, int64_t n_v, int64_t n_e, const int64_t *edge_u, const int64_t *edge_v,
              const double *edge_w, int64_t *u_indptr, int32_t *u_indices, double *u_weights, int64_t *v_indptr,
              int32_t *v_indices, double *v_weights, double *ws_u, double *ws_v, int device) {
    if (n_u <= 0 || n_v <= 0 || n_e <= 0) throw InvalidArg("csr_build: empty graph");
    if (n_e >= (int64_t)1 << 31 || n_u >= (int64_t)1 << 31 || n_v >= (int64_t)1 << 31)
        throw InvalidArg("csr_build: sizes must fit int32 indices");
    if ((double)n_u * (double)n_v >= 1.8e19) throw InvalidArg("csr_build: |U||V| exceeds 64-bit pair keys");
    BH_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    BH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};
    const int64_t n = n_e;
    DBuf<int64_t> da(n), db(n);
    DBuf<double> dw(n), uw(n), vw(n), dws_u(n_u), dws_v(n_v);
    DBuf<uint64_t> k0(n), k1(n), deg_u(n_u), deg_v(n_v), ip_u(n_u + 1), ip_v(n_v + 1);
    DBuf<uint32_t> v0(n), v1(n);
    DBuf<int32_t> ucol(n), vcol(n), flags(2);
    BH_CUDA(cudaMemcpyAsync(da.p, edge_u, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    BH_CUDA(cudaMemcpyAsync(db.p, edge_v, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    BH_CUDA(cudaMemcpyAsync(dw.p, edge_w, n * sizeof(double), cudaMemcpyHostToDevice, st));
    BH_CUDA(cudaMemsetAsync(flags.p, 0, 2 * sizeof(int32_t), st));
    BH_CUDA(cudaMemsetAsync(deg_u.p, 0, n_u * sizeof(uint64_t), st));
    BH_CUDA(cudaMemsetAsync(deg_v.p, 0, n_v * sizeof(uint64_t), st));

    // U side: sort by u * |V| + v
    k_pack_keys<<<grid_of(n), 256, 0, st>>>(da.p, db.p, n, n_v, n_u, k0.p, v0.p, flags.p);
    count_launch();
    radix_sort_pairs(k0.p, v0.p, k1.p, v1.p, n, key_bits((uint64_t)n_u * (uint64_t)n_v - 1), st);
    // da is reused as the U row of every canonical edge
    k_unpack<<<grid_of(n), 256, 0, st>>>(k0.p, v0.p, dw.p, n, n_v, ucol.p, da.p, uw.p, deg_u.p, flags.p + 1);
    count_launch();
    exclusive_scan<uint64_t>(deg_u.p, n_u, ip_u.p, st);
    BH_CUDA(cudaMemcpyAsync(ip_u.p + n_u, &n, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    k_row_sums<<<grid_of(n_u), 256, 0, st>>>(ip_u.p, n_u, uw.p, dws_u.p);
    count_launch();

    // V side: sort the canonical edges by v * |U| + u
    k_pack_transpose<<<grid_of(n), 256, 0, st>>>(da.p, ucol.p, n, n_u, k0.p, v0.p);
    count_launch();
    radix_sort_pairs(k0.p, v0.p, k1.p, v1.p, n, key_bits((uint64_t)n_v * (uint64_t)n_u - 1), st);
    k_unpack<<<grid_of(n), 256, 0, st>>>(k0.p, v0.p, uw.p, n, n_u, vcol.p, nullptr, vw.p, deg_v.p, flags.p + 1);
    count_launch();
    exclusive_scan<uint64_t>(deg_v.p, n_v, ip_v.p, st);
    BH_CUDA(cudaMemcpyAsync(ip_v.p + n_v, &n, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    k_row_sums<<<grid_of(n_v), 256, 0, st>>>(ip_v.p, n_v, vw.p, dws_v.p);
    count_launch();
    BH_CUDA(cudaGetLastError());

    int32_t hflags[2];
    BH_CUDA(cudaMemcpyAsync(hflags, flags.p, sizeof(hflags), cudaMemcpyDeviceToHost, st));
    BH_CUDA(cudaStreamSynchronize(st));
    if (hflags[0]) throw InvalidArg("csr_build: edge endpoint out of range");
    if (hflags[1]) return 1;
    BH_CUDA(cudaMemcpyAsync(u_indptr, ip_u.p, (n_u + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    BH_CUDA(cudaMemcpyAsync(u_indices, ucol.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    BH_CUDA(cudaMemcpyAsync(u_weights, uw.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    BH_CUDA(cudaMemcpyAsync(v_indptr, ip_v.p, (n_v + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    BH_CUDA(cudaMemcpyAsync(v_indices, vcol.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    BH_CUDA(cudaMemcpyAsync(v_weights, vw.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    BH_CUDA(cudaMemcpyAsync(ws_u, dws_u.p, n_u * sizeof(double), cudaMemcpyDeviceToHost, st));
    BH_CUDA(cudaMemcpyAsync(ws_v, dws_v.p, n_v * sizeof(double), cudaMemcpyDeviceToHost, st));
    BH_CUDA(cudaStreamSynchronize(st));
    return 0;
}

}  // namespace bh
