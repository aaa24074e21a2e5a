// gather_bench2.cu -- which mechanism moves 256-B (B = 64 fp32) or 512-B operand rows
// fastest for the pull SpMM's access sequence.  Reads the real column sequence of a
// side of the c2 store (tools/dump_cols.py: int32 cols in CSR order after degree
// relabelling) or draws one; every variant streams contiguous edge ranges per warp
// and FMAs the gathered rows into lane accumulators (no row ends, no stores), so the
// numbers are ceilings for the gather itself.
//   ldg    : register pipeline, S rows in flight per warp (as k_pull_sw)
//   hub    : ldg + the H hottest operand rows staged in shared memory per block
//   bulk   : cp.async.bulk (TMA, UBLKCP) row copies into a per-warp smem ring
//   ldgsts : cp.async 16 B per lane (two rows per warp instruction) into a ring
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench2 gather_bench2.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                 \
    do {                                                                      \
        cudaError_t e = (x);                                                  \
        if (e != cudaSuccess) {                                               \
            printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); \
            exit(1);                                                          \
        }                                                                     \
    } while (0)

constexpr int FULL = ~0u;

template <int VEC>
struct FV;
template <>
struct FV<2> {
    using t = float2;
};
template <>
struct FV<4> {
    using t = float4;
};

template <int VEC>
__device__ __forceinline__ void fma_row(float (&a)[VEC], float w, const typename FV<VEC>::t &x) {
    if constexpr (VEC == 2) {
        a[0] = fmaf(w, x.x, a[0]);
        a[1] = fmaf(w, x.y, a[1]);
    } else {
        a[0] = fmaf(w, x.x, a[0]);
        a[1] = fmaf(w, x.y, a[1]);
        a[2] = fmaf(w, x.z, a[2]);
        a[3] = fmaf(w, x.w, a[3]);
    }
}

// ---- ldg: S rows in flight per warp in registers; (col, val) windows by shuffle
template <int VEC, int S, int MINB, int H>
__global__ void __launch_bounds__(256, MINB) g_ldg(const int *cols, const float *vals, const float *X, int E, int per,
                                                   float *out) {
    using V = typename FV<VEC>::t;
    constexpr int B = 32 * VEC;
    extern __shared__ __align__(16) unsigned char smem[];
    V *hub = reinterpret_cast<V *>(smem);  // [H][32]
    if constexpr (H > 0) {
        for (int i = threadIdx.x; i < H * 32; i += 256) hub[i] = reinterpret_cast<const V *>(X)[i];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int e0 = gw * per;
    const int n = min(per, E - e0);
    if (n <= 0) return;
    const V *Xl = reinterpret_cast<const V *>(X) + lane;
    auto fetch = [&](int c) -> V {
        if constexpr (H > 0) {
            if (c < H) return hub[c * 32 + lane];
        }
        return Xl[(size_t)c * 32];
    };
    V xs[S];
    float ws[S];
    int wc = lane < n ? cols[e0 + lane] : 0;
    float wv = lane < n ? vals[e0 + lane] : 0.f;
    int wc2 = 32 + lane < n ? cols[e0 + 32 + lane] : 0;
    float wv2 = 32 + lane < n ? vals[e0 + 32 + lane] : 0.f;
#pragma unroll
    for (int t = 0; t < S; t++) {
        int c = __shfl_sync(FULL, wc, t);
        ws[t] = __shfl_sync(FULL, wv, t);
        xs[t] = fetch(c);
    }
    float a[VEC] = {};
    for (int c0 = 0; c0 + 32 + S <= n; c0 += 32) {
#pragma unroll
        for (int t = 0; t < 32; t++) {
            const int sl = t % S;
            fma_row<VEC>(a, ws[sl], xs[sl]);
            const int src = (t + S) & 31;
            const int c = __shfl_sync(FULL, (t + S < 32) ? wc : wc2, src);
            ws[sl] = __shfl_sync(FULL, (t + S < 32) ? wv : wv2, src);
            xs[sl] = fetch(c);
        }
        wc = wc2;
        wv = wv2;
        wc2 = c0 + 64 + lane < n ? cols[e0 + c0 + 64 + lane] : 0;
        wv2 = c0 + 64 + lane < n ? vals[e0 + c0 + 64 + lane] : 0.f;
    }
    float s = 0;
#pragma unroll
    for (int v = 0; v < VEC; v++) s += a[v];
    out[gw * 32 + lane] = s;
    (void)B;
}

// ---- bulk: TMA row copies into a per-warp ring; RPS rows per stage, NST stages
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}

template <int VEC, int RPS, int NST, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) g_bulk(const int *cols, const float *vals, const float *X, int E, int per,
                                                      float *out) {
    using V = typename FV<VEC>::t;
    constexpr int ROWB = 32 * VEC * 4;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    unsigned char *ring = smem + (size_t)warp * NST * RPS * ROWB;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)WARPS * NST * RPS * ROWB) + warp * NST;
    if (lane == 0)
        for (int s = 0; s < NST; s++) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int gw = blockIdx.x * WARPS + warp;
    const int e0 = gw * per;
    const int n = min(per, E - e0);
    if (n <= 0) return;
    const int nst = n / RPS;  // whole stages only
    auto issue = [&](int st) {
        const int s = st % NST;
        if (lane == 0) mbar_expect(bars + s, RPS * ROWB);
        __syncwarp();
        if (lane < RPS) {
            const int c = cols[e0 + st * RPS + lane];
            bulk_g2s(ring + (size_t)(s * RPS + lane) * ROWB, X + (size_t)c * 32 * VEC, ROWB, bars + s);
        }
    };
    for (int st = 0; st < NST && st < nst; st++) issue(st);
    float a[VEC] = {};
    for (int st = 0; st < nst; st++) {
        const int s = st % NST;
        const float wv = lane < RPS ? vals[e0 + st * RPS + lane] : 0.f;
        mbar_wait(bars + s, (st / NST) & 1);
#pragma unroll
        for (int r = 0; r < RPS; r++) {
            const V x = reinterpret_cast<const V *>(ring + (size_t)(s * RPS + r) * ROWB)[lane];
            fma_row<VEC>(a, __shfl_sync(FULL, wv, r), x);
        }
        __syncwarp();
        if (st + NST < nst) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(st + NST);
        }
    }
    float s = 0;
#pragma unroll
    for (int v = 0; v < VEC; v++) s += a[v];
    out[gw * 32 + lane] = s;
}

// ---- ldgsts: cp.async 16 B per lane; a warp instruction copies 512 B (2 rows of 256 B or 1 of 512 B)
template <int VEC, int RPS, int NST, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) g_ldgsts(const int *cols, const float *vals, const float *X, int E,
                                                            int per, float *out) {
    using V = typename FV<VEC>::t;
    constexpr int ROWB = 32 * VEC * 4;
    constexpr int RPI = 512 / ROWB;      // rows per warp instruction
    constexpr int LPR = 32 / RPI;        // lanes per row
    static_assert(RPS <= 32 && RPS % RPI == 0, "stage");
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    unsigned char *ring = smem + (size_t)warp * NST * RPS * ROWB;
    const int gw = blockIdx.x * WARPS + warp;
    const int e0 = gw * per;
    const int n = min(per, E - e0);
    if (n <= 0) return;
    const int nst = n / RPS;
    const int h = lane / LPR, q = lane % LPR;
    auto issue = [&](int st) {
        const int s = st % NST;
        const int wc = lane < RPS ? cols[e0 + st * RPS + lane] : 0;
#pragma unroll
        for (int j = 0; j < RPS / RPI; j++) {
            const int r = j * RPI + h;
            const int c = __shfl_sync(FULL, wc, r);
            const uint32_t dst = smem_u32(ring + (size_t)(s * RPS + r) * ROWB + q * 16);
            const float *src = X + (size_t)c * 32 * VEC + q * 4;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int st = 0; st < NST; st++) {
        if (st < nst) issue(st);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    float a[VEC] = {};
    for (int st = 0; st < nst; st++) {
        const int s = st % NST;
        const float wv = lane < RPS ? vals[e0 + st * RPS + lane] : 0.f;
        asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
        __syncwarp();
#pragma unroll
        for (int r = 0; r < RPS; r++) {
            const V x = reinterpret_cast<const V *>(ring + (size_t)(s * RPS + r) * ROWB)[lane];
            fma_row<VEC>(a, __shfl_sync(FULL, wv, r), x);
        }
        __syncwarp();
        if (st + NST < nst) issue(st + NST);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    float s = 0;
#pragma unroll
    for (int v = 0; v < VEC; v++) s += a[v];
    out[gw * 32 + lane] = s;
}

static std::vector<int> read_cols(const char *path) {
    std::vector<int> v;
    FILE *f = fopen(path, "rb");
    if (!f) return v;
    fseek(f, 0, SEEK_END);
    long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    v.resize(sz / 4);
    if (fread(v.data(), 4, v.size(), f) != v.size()) v.clear();
    fclose(f);
    return v;
}

struct Bench {
    int *dc;
    float *dv, *dX, *dout;
    int E;
    int VEC;
    cudaEvent_t a, b;
    template <typename F>
    void run(const char *name, F launch) {
        for (int w = 0; w < 3; w++) launch();
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a));
        for (int it = 0; it < 20; it++) launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double us = ms * 1000 / 20;
        printf("  %-44s %8.1f us  %6.2f TB/s\n", name, us, (double)E * VEC * 128 / (us * 1e-6) / 1e12);
        fflush(stdout);
    }
};

template <int VEC>
static void suite(const char *label, const std::vector<int> &cols, int NX) {
    const int E = (int)cols.size();
    printf("== %s: E=%d rows=%d row_bytes=%d operand=%.1f MB\n", label, E, NX, VEC * 128, NX * VEC * 128.0 / 1e6);
    Bench bn;
    bn.E = E;
    bn.VEC = VEC;
    CK(cudaMalloc(&bn.dX, (size_t)NX * VEC * 128));
    CK(cudaMalloc(&bn.dv, (size_t)E * 4));
    CK(cudaMalloc(&bn.dc, (size_t)E * 4));
    CK(cudaMalloc(&bn.dout, (size_t)148 * 16 * 32 * 32 * 4));
    std::vector<float> hX((size_t)NX * VEC * 32), hv(E, 0.5f);
    std::mt19937 rng(1);
    for (auto &v : hX) v = (rng() % 1000) / 1000.f;
    CK(cudaMemcpy(bn.dX, hX.data(), hX.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(bn.dv, hv.data(), (size_t)E * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(bn.dc, cols.data(), (size_t)E * 4, cudaMemcpyHostToDevice));
    cudaEventCreate(&bn.a);
    cudaEventCreate(&bn.b);
    auto per_of = [&](int warps) { return (E + warps - 1) / warps; };
    char nm[128];
#define LDG(S, MINB, H)                                                                                   \
    {                                                                                                     \
        const int grid = 148 * MINB, per = per_of(grid * 8);                                              \
        const size_t sm = (size_t)H * VEC * 128;                                                          \
        CK(cudaFuncSetAttribute(g_ldg<VEC, S, MINB, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
        snprintf(nm, sizeof nm, "ldg S=%d blocks/SM=%d hub=%d", S, MINB, H);                              \
        bn.run(nm, [&] { g_ldg<VEC, S, MINB, H><<<grid, 256, sm>>>(bn.dc, bn.dv, bn.dX, E, per, bn.dout); }); \
    }
    LDG(8, 2, 0)
    LDG(8, 4, 0)
    LDG(16, 2, 0)
    LDG(16, 3, 0)
    LDG(8, 6, 0)
    LDG(4, 8, 0)
    if constexpr (VEC == 2) {
        LDG(8, 2, 256)
        LDG(8, 3, 256)
        LDG(16, 2, 256)
        LDG(8, 2, 384)
        LDG(16, 2, 384)
    }
#define BULK(RPS, NST, WARPS, BPS)                                                                              \
    {                                                                                                           \
        const int grid = 148 * BPS, per = per_of(grid * WARPS);                                                 \
        const size_t sm = (size_t)WARPS * NST * RPS * VEC * 128 + WARPS * NST * 8;                              \
        CK(cudaFuncSetAttribute(g_bulk<VEC, RPS, NST, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
        snprintf(nm, sizeof nm, "bulk rows/stage=%d stages=%d warps=%d blocks/SM=%d", RPS, NST, WARPS, BPS);    \
        bn.run(nm, [&] { g_bulk<VEC, RPS, NST, WARPS><<<grid, WARPS * 32, sm>>>(bn.dc, bn.dv, bn.dX, E, per, bn.dout); }); \
    }
    BULK(16, 2, 8, 2)
    BULK(16, 2, 8, 3)
    BULK(8, 4, 8, 2)
    BULK(32, 2, 4, 2)
    BULK(16, 4, 4, 2)
#define LDGSTS(RPS, NST, WARPS, BPS)                                                                            \
    {                                                                                                           \
        const int grid = 148 * BPS, per = per_of(grid * WARPS);                                                 \
        const size_t sm = (size_t)WARPS * NST * RPS * VEC * 128;                                                \
        CK(cudaFuncSetAttribute(g_ldgsts<VEC, RPS, NST, WARPS, BPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
        snprintf(nm, sizeof nm, "ldgsts rows/stage=%d stages=%d warps=%d blocks/SM=%d", RPS, NST, WARPS, BPS);  \
        bn.run(nm, [&] { g_ldgsts<VEC, RPS, NST, WARPS, BPS><<<grid, WARPS * 32, sm>>>(bn.dc, bn.dv, bn.dX, E, per, bn.dout); }); \
    }
    LDGSTS(8, 2, 8, 4)
    LDGSTS(8, 3, 8, 3)
    LDGSTS(8, 4, 8, 2)
    LDGSTS(16, 2, 8, 2)
    LDGSTS(16, 3, 8, 2)
    LDGSTS(8, 4, 8, 4)
    LDGSTS(4, 4, 8, 4)
    CK(cudaDeviceSynchronize());
    CK(cudaFree(bn.dX));
    CK(cudaFree(bn.dv));
    CK(cudaFree(bn.dc));
    CK(cudaFree(bn.dout));
}

int main(int argc, char **argv) {
    std::vector<int> real_v = read_cols(argc > 1 ? argv[1] : "gpurun_out/c2_v_cols.bin");
    std::vector<int> real_u = read_cols(argc > 2 ? argv[2] : "gpurun_out/c2_u_cols.bin");
    const int E = 2000000;
    std::mt19937 rng(1);
    std::vector<int> uni(E);
    for (int e = 0; e < E; e++) uni[e] = rng() % 100000;
    suite<2>("uniform over 1e5 rows, 256-B rows", uni, 100000);
    if (!real_v.empty()) suite<2>("c2 V pull (cols = u, 1e5 operand rows), 256-B rows", real_v, 100000);
    if (!real_u.empty()) suite<2>("c2 U pull (cols = v, 2e5 operand rows), 256-B rows", real_u, 200000);
    suite<4>("uniform over 1e5 rows, 512-B rows", uni, 100000);
    if (!real_v.empty()) suite<4>("c2 V pull, 512-B rows", real_v, 100000);
    return 0;
}
