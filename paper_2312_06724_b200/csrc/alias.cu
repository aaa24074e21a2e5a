// alias.cu -- device construction of the MCSP alias tables (bh_alias_build).
//
// Restates build_alias (reference baselines.py:41-77) per CSR row, one thread
// per row (rows are independent; a row's pairing is inherently sequential):
//   scaled_i = w_i * (d / sum(w))  with sum = numpy's pairwise add.reduce,
//   small = slots with scaled < 1 (ascending), large = the rest (ascending),
//   while both are non-empty: pop one of each from the back; the small slot
//   keeps its scaled value as prob and aliases the large one, whose scaled
//   value drops by 1 - scaled(small) and which rejoins small or large;
//   every slot left over keeps prob 1 and aliases itself.
// Same arithmetic in the same order (no contraction: only adds, subtracts and
// one multiply per slot), so the tables are bit-identical to the reference's.
// Degree-1 rows are left at prob 1, alias 0.  Scratch: the scaled values and
// the two stacks live in the row's own [indptr[r], indptr[r+1]) segment of
// three E-sized arrays.
#include <algorithm>

#include "common.cuh"

namespace bh {

namespace {

// numpy float64 add.reduce over a contiguous run: 0.0 + pairwise sum (8-way
// unrolled blocks of at most 128, recursive halving).
__device__ double np_pairwise(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
}

__global__ void k_alias_rows(int64_t n_rows, const int64_t *__restrict__ indptr, const double *__restrict__ w,
                             double *__restrict__ scaled, int32_t *__restrict__ st_small,
                             int32_t *__restrict__ st_large, double *__restrict__ prob, int64_t *__restrict__ alias) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = indptr[r], d = indptr[r + 1] - s;
        for (int64_t i = 0; i < d; i++) {
            prob[s + i] = 1.0;
            alias[s + i] = 0;
        }
        if (d <= 1) continue;
        const double f = __ddiv_rn((double)d, __dadd_rn(0.0, np_pairwise(w + s, d)));
        double *sc = scaled + s;
        int32_t *sm = st_small + s, *lg = st_large + s;
        int64_t ns = 0, nl = 0;
        for (int64_t i = 0; i < d; i++) {
            sc[i] = __dmul_rn(w[s + i], f);
            if (sc[i] < 1.0) sm[ns++] = (int32_t)i; else lg[nl++] = (int32_t)i;
        }
        while (ns > 0 && nl > 0) {
            const int32_t a = sm[--ns], b = lg[--nl];
            prob[s + a] = sc[a];
            alias[s + a] = b;
            sc[b] = __dsub_rn(sc[b], __dsub_rn(1.0, sc[a]));
            if (sc[b] < 1.0) sm[ns++] = b; else lg[nl++] = b;
        }
        for (int64_t j = 0; j < nl; j++) {
            prob[s + lg[j]] = 1.0;
            alias[s + lg[j]] = lg[j];
        }
        for (int64_t j = 0; j < ns; j++) {
            prob[s + sm[j]] = 1.0;
            alias[s + sm[j]] = sm[j];
        }
    }
}

template <typename X>
X *dnew(size_t n) {
    X *p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(X));
    if (e == cudaErrorMemoryAllocation) {
        (void)cudaGetLastError();
        throw std::bad_alloc();
    }
    BH_CUDA(e);
    return p;
}

}  // namespace

void alias_build(int64_t n_rows, int64_t n_e, const int64_t *indptr, const double *weights, int device,
                 double *prob_out, int64_t *alias_out) {
    BH_CUDA(cudaSetDevice(device));
    int64_t *d_ip = nullptr;
    double *d_w = nullptr, *d_sc = nullptr, *d_p = nullptr;
    int32_t *d_s = nullptr, *d_l = nullptr;
    int64_t *d_a = nullptr;
    auto cleanup = [&] {
        cudaFree(d_ip); cudaFree(d_w); cudaFree(d_sc); cudaFree(d_p); cudaFree(d_s); cudaFree(d_l); cudaFree(d_a);
    };
    try {
        d_ip = dnew<int64_t>(n_rows + 1);
        d_w = dnew<double>(n_e);
        d_sc = dnew<double>(n_e);
        d_p = dnew<double>(n_e);
        d_s = dnew<int32_t>(n_e);
        d_l = dnew<int32_t>(n_e);
        d_a = dnew<int64_t>(n_e);
        BH_CUDA(cudaMemcpy(d_ip, indptr, (n_rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
        BH_CUDA(cudaMemcpy(d_w, weights, n_e * sizeof(double), cudaMemcpyHostToDevice));
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n_rows + 127) / 128, 148 * 8));
        k_alias_rows<<<grid, 128>>>(n_rows, d_ip, d_w, d_sc, d_s, d_l, d_p, d_a);
        count_launch();
        BH_CUDA(cudaGetLastError());
        BH_CUDA(cudaMemcpy(prob_out, d_p, n_e * sizeof(double), cudaMemcpyDeviceToHost));
        BH_CUDA(cudaMemcpy(alias_out, d_a, n_e * sizeof(int64_t), cudaMemcpyDeviceToHost));
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}

}  // namespace bh
