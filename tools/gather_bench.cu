// gather_bench.cu -- ceiling of the pull SpMM's operand gather on this GPU.
//
// Each warp streams a contiguous range of "edges"; per edge it gathers one
// B-wide fp32 operand row (256 B for B = 64) and FMAs it into lane
// accumulators.  Variants: register pipeline depth, one edge per warp
// instruction (float2/lane) vs two edges (float4/lane, half-warps), and the
// column distribution (uniform, power-law like the C2 graph, sorted).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__);         \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

constexpr int B = 64;

template <int S>
__global__ void __launch_bounds__(256, 2) g_full(const int *cols, const float *vals, const float *X, int E, int per,
                                                 float *out) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int e0 = gw * per;
    const int n = min(per, E - e0);
    if (n <= 0) return;
    const float *Xl = X + lane * 2;
    float2 xs[S];
    float ws[S];
    int wc = lane < n ? cols[e0 + lane] : 0;
    float wv = lane < n ? vals[e0 + lane] : 0.f;
    int wc2 = 32 + lane < n ? cols[e0 + 32 + lane] : 0;
    float wv2 = 32 + lane < n ? vals[e0 + 32 + lane] : 0.f;
#pragma unroll
    for (int t = 0; t < S; t++) {
        int c = __shfl_sync(~0u, wc, t);
        ws[t] = __shfl_sync(~0u, wv, t);
        xs[t] = *reinterpret_cast<const float2 *>(Xl + (size_t)c * B);
    }
    float a0 = 0, a1 = 0;
    int c0 = 0;
    for (; c0 + 32 + S <= n; c0 += 32) {
#pragma unroll
        for (int t = 0; t < 32; t++) {
            const int sl = t & (S - 1);
            a0 = fmaf(ws[sl], xs[sl].x, a0);
            a1 = fmaf(ws[sl], xs[sl].y, a1);
            const int src = (t + S) & 31;
            const int c = __shfl_sync(~0u, (t + S < 32) ? wc : wc2, src);
            ws[sl] = __shfl_sync(~0u, (t + S < 32) ? wv : wv2, src);
            xs[sl] = *reinterpret_cast<const float2 *>(Xl + (size_t)c * B);
        }
        wc = wc2;
        wv = wv2;
        wc2 = c0 + 64 + lane < n ? cols[e0 + c0 + 64 + lane] : 0;
        wv2 = c0 + 64 + lane < n ? vals[e0 + c0 + 64 + lane] : 0.f;
    }
    out[gw * 64 + lane * 2] = a0;
    out[gw * 64 + lane * 2 + 1] = a1;
}

// two edges per warp instruction: half-warp h handles edges 2j + h, float4 per lane
template <int S>
__global__ void __launch_bounds__(256, 2) g_half(const int *cols, const float *vals, const float *X, int E, int per,
                                                 float *out) {
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, q = lane & 15;
    const int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
    const int e0 = gw * per;
    const int n = min(per, E - e0);
    if (n <= 0) return;
    const float *Xl = X + q * 4;
    float4 xs[S];
    float ws[S];
    int wc = lane < n ? cols[e0 + lane] : 0;
    float wv = lane < n ? vals[e0 + lane] : 0.f;
    int wc2 = 32 + lane < n ? cols[e0 + 32 + lane] : 0;
    float wv2 = 32 + lane < n ? vals[e0 + 32 + lane] : 0.f;
#pragma unroll
    for (int t = 0; t < S; t++) {  // pair t = edges 2t, 2t+1
        int c = __shfl_sync(~0u, wc, 2 * t + h);
        ws[t] = __shfl_sync(~0u, wv, 2 * t + h);
        xs[t] = *reinterpret_cast<const float4 *>(Xl + (size_t)c * B);
    }
    float4 a = make_float4(0, 0, 0, 0);
    int c0 = 0;
    for (; c0 + 32 + 2 * S <= n; c0 += 32) {
#pragma unroll
        for (int t = 0; t < 16; t++) {  // 16 pairs = 32 edges
            const int sl = t & (S - 1);
            a.x = fmaf(ws[sl], xs[sl].x, a.x);
            a.y = fmaf(ws[sl], xs[sl].y, a.y);
            a.z = fmaf(ws[sl], xs[sl].z, a.z);
            a.w = fmaf(ws[sl], xs[sl].w, a.w);
            const int pe = 2 * (t + S);  // next edge pair offset within the 64-edge window pair
            const int src = (pe + h) & 31;
            const int c = __shfl_sync(~0u, (pe < 32) ? wc : wc2, src);
            ws[sl] = __shfl_sync(~0u, (pe < 32) ? wv : wv2, src);
            xs[sl] = *reinterpret_cast<const float4 *>(Xl + (size_t)c * B);
        }
        wc = wc2;
        wv = wv2;
        wc2 = c0 + 64 + lane < n ? cols[e0 + c0 + 64 + lane] : 0;
        wv2 = c0 + 64 + lane < n ? vals[e0 + c0 + 64 + lane] : 0.f;
    }
    a.x += __shfl_xor_sync(~0u, a.x, 16);
    out[gw * 64 + q * 4] = a.x + a.y + a.z + a.w;
}

int main() {
    const int NX = 200000, E = 2000000;
    std::mt19937 rng(1);
    std::vector<float> hX((size_t)NX * B);
    for (auto &v : hX) v = (rng() % 1000) / 1000.f;
    std::vector<int> uni(E), pw(E);
    std::vector<float> hv(E, 0.5f);
    std::vector<double> cdf(NX);
    double s = 0;
    for (int i = 0; i < NX; i++) {
        s += std::pow(i + 1.0, -1.0 / 1.2);
        cdf[i] = s;
    }
    std::uniform_real_distribution<double> U01(0, 1);
    for (int e = 0; e < E; e++) {
        uni[e] = rng() % NX;
        pw[e] = (int)(std::lower_bound(cdf.begin(), cdf.end(), U01(rng) * s) - cdf.begin());
    }
    std::vector<int> pws = pw;
    // sorted within chunks of 20 (like CSR rows sorted by column)
    for (int e = 0; e + 20 <= E; e += 20) std::sort(pws.begin() + e, pws.begin() + e + 20);
    float *dX, *dv, *dout;
    int *dc;
    CK(cudaMalloc(&dX, hX.size() * 4));
    CK(cudaMalloc(&dv, E * 4));
    CK(cudaMalloc(&dc, E * 4));
    CK(cudaMalloc(&dout, 148 * 64 * 64 * 4 * 4));
    CK(cudaMemcpy(dX, hX.data(), hX.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dv, hv.data(), E * 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *names[3] = {"uniform", "powerlaw", "powerlaw-rowsorted"};
    std::vector<int> *lists[3] = {&uni, &pw, &pws};
    for (int li = 0; li < 3; li++) {
        CK(cudaMemcpy(dc, lists[li]->data(), E * 4, cudaMemcpyHostToDevice));
        for (int bps : {2, 4, 8}) {
            const int grid = 148 * bps, warps = grid * 8, per = (E + warps - 1) / warps;
            for (int variant = 0; variant < 4; variant++) {
                auto launch = [&] {
                    if (variant == 0) g_full<8><<<grid, 256>>>(dc, dv, dX, E, per, dout);
                    if (variant == 1) g_full<16><<<grid, 256>>>(dc, dv, dX, E, per, dout);
                    if (variant == 2) g_half<4><<<grid, 256>>>(dc, dv, dX, E, per, dout);
                    if (variant == 3) g_half<8><<<grid, 256>>>(dc, dv, dX, E, per, dout);
                };
                for (int w = 0; w < 3; w++) launch();
                CK(cudaEventRecord(a));
                for (int it = 0; it < 20; it++) launch();
                CK(cudaEventRecord(b));
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double us = ms * 1000 / 20;
                const char *vn[4] = {"full S=8", "full S=16", "half S=4(8 edges)", "half S=8(16 edges)"};
                printf("%-20s blocks/SM=%d %-22s %8.1f us  %6.2f TB/s gathered\n", names[li], bps, vn[variant], us,
                       (double)E * B * 4 / (us * 1e-6) / 1e12);
            }
        }
    }
    CK(cudaGetLastError());
    return 0;
}
