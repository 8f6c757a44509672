// diag_alu.cu — DIAGNOSTIC microbenchmark (not on the hot path): the issue ceiling of the
// CUDA-core tile engine's inner-loop instruction mix, measured on the device, used as the
// "alu" roofline denominator of k_simt.
//   mix 0: FADD2 + FMNMX3(|.|) + FFMA2 per two element-pairs (max and L2 families together)
//   mix 1: FADD2 + FMNMX3(|.|)                (max family only)
//   mix 2: FADD2 + FFMA2                       (L2 family only)
// Same register micro-tile as k_simt (4 x 4 pairs per thread, float4 operands), no memory.
#include "cil_internal.cuh"

namespace cil {

__device__ float g_alu_sink[128];

template <int MIX>
__global__ void __launch_bounds__(128) k_alu_mix(float* out, int iters, float seed) {
    float4 av[4], bv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        av[i] = make_float4(seed * (i + 1), seed * (i + 2), seed * (i + 3), seed * (i + 4));
        bv[i] = make_float4(seed * (i + 5), seed * (i + 6), seed * (i + 7), seed * (i + 8));
    }
    float2 acc[4][4];
    float mx[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { acc[i][j] = make_float2(0.f, 0.f); mx[i][j] = 0.f; }
    const float2 step = make_float2(1e-7f, -1e-7f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 d0 = __fadd2_rn(make_float2(av[i].x, av[i].y), make_float2(-bv[j].x, -bv[j].y));
                const float2 d1 = __fadd2_rn(make_float2(av[i].z, av[i].w), make_float2(-bv[j].z, -bv[j].w));
                if (MIX != 2) {
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d0.x), fabsf(d0.y)));
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d1.x), fabsf(d1.y)));
                }
                if (MIX != 1) {
                    acc[i][j] = __ffma2_rn(d0, d0, acc[i][j]);
                    acc[i][j] = __ffma2_rn(d1, d1, acc[i][j]);
                }
            }
        // perturb B so nothing is loop-invariant (4 FADD2 per 64 element-pairs: ~6% of the mix)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 lo = __fadd2_rn(make_float2(bv[j].x, bv[j].y), step);
            float2 hi = __fadd2_rn(make_float2(bv[j].z, bv[j].w), step);
            bv[j] = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += acc[i][j].x + acc[i][j].y + mx[i][j];
    if (s == 12345.678f) out[threadIdx.x] = s;   // keep the work observable
}

}  // namespace cil

extern "C" CIL_API int32_t cil_diag_alu_ceiling(int32_t mix, int32_t iters, double* element_pairs_per_s,
                                                double* ms) {
    using namespace cil;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    float* out = nullptr;
    if (cudaGetSymbolAddress((void**)&out, g_alu_sink) != cudaSuccess) return -1;
    const int blocks = nsm * 8, threads = 128;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&](int n) {
        if (mix == 1) k_alu_mix<1><<<blocks, threads>>>(out, n, 0.5f);
        else if (mix == 2) k_alu_mix<2><<<blocks, threads>>>(out, n, 0.5f);
        else k_alu_mix<0><<<blocks, threads>>>(out, n, 0.5f);
    };
    launch(16);   // warm-up
    cudaEventRecord(a);
    launch(iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (cudaGetLastError() != cudaSuccess) return -1;
    // element-pairs per iteration per thread: 16 pairs x 4 elements
    const double ep = (double)blocks * threads * (double)iters * 16.0 * 4.0;
    *element_pairs_per_s = ep / (t * 1e-3);
    *ms = t;
    return 0;
}
