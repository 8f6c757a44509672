// diag_alu.cu — DIAGNOSTIC microbenchmark (not on the hot path): the issue ceiling of the
// CUDA-core tile engine's inner-loop instruction mix, measured on the device, used as the
// "alu" roofline denominator of k_simt.
//   mix 0: FADD2 + FMNMX3(|.|) + FFMA2 per two element-pairs (max and L2 families together)
//   mix 1: FADD2 + FMNMX3(|.|)                (max family only)
//   mix 2: FADD2 + FFMA2                       (L2 family only)
//   mix 3: IMAD (biased packed 16-bit add) + VIMNMX3.U16x2 max / min   (max16.cu, the max family)
// Same register micro-tiles as k_simt (4 x 4 pairs per thread, float4 operands) and k_max16_reg
// (8 x 4 pairs, uint4 operands), no memory.
#include <string.h>

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

// max16.cu's inner loop: per pair and uint4 step (8 element-pairs) 4 IMAD + 2 VIMNMX3 max + 2 min
__global__ void __launch_bounds__(128, 3) k_alu_mix16(float* out, int iters, uint32_t seed, uint32_t one) {
    uint4 av[8], bv[4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        av[i] = make_uint4((seed * (i + 1)) & 0x3fff3fffu, (seed * (i + 3)) & 0x3fff3fffu,
                           (seed * (i + 5)) & 0x3fff3fffu, (seed * (i + 7)) & 0x3fff3fffu);
#pragma unroll
    for (int j = 0; j < 4; ++j)
        bv[j] = make_uint4((seed * (j + 9) + 1) & 0x3fff3fffu, (seed * (j + 11) + 3) & 0x3fff3fffu,
                           (seed * (j + 13) + 5) & 0x3fff3fffu, (seed * (j + 15) + 7) & 0x3fff3fffu);
    uint32_t mx[8][4], mn[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { mx[i][j] = 0u; mn[i][j] = 0xffffffffu; }
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t d0, d1, d2, d3;
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d0) : "r"(av[i].x), "r"(one), "r"(bv[j].x));
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d1) : "r"(av[i].y), "r"(one), "r"(bv[j].y));
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d2) : "r"(av[i].z), "r"(one), "r"(bv[j].z));
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d3) : "r"(av[i].w), "r"(one), "r"(bv[j].w));
                mx[i][j] = __vimax3_u16x2(mx[i][j], d0, d1);
                mn[i][j] = __vimin3_u16x2(mn[i][j], d0, d1);
                mx[i][j] = __vimax3_u16x2(mx[i][j], d2, d3);
                mn[i][j] = __vimin3_u16x2(mn[i][j], d2, d3);
            }
        // perturb B (4 x 4 XOR per 256 element-pairs: ~3 % of the mix)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            bv[j].x ^= 0x00010001u; bv[j].y ^= 0x00020002u; bv[j].z ^= 0x00010001u; bv[j].w ^= 0x00020002u;
        }
    }
    uint32_t sacc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sacc += mx[i][j] ^ mn[i][j];
    if (sacc == 0x12345678u) out[threadIdx.x] = (float)sacc;
}

// ---------------------------------------------------------------------------------------------
// Exhaustive check of the hardware square-root approximation the INT8 engine's interval bounds rely
// on (gram3.cu): for EVERY normal positive FP32 x, the relative error of sqrt.approx.f32 against
// the (FP64, correctly rounded) square root.  The engine inflates by 2^-21, so the bound holds for
// all inputs iff both maxima stay below 2^-21 (tests/test_gpu_parity.py pins them below 2^-22).
__global__ void k_sqrt_approx_err(unsigned long long* up, unsigned long long* down) {
    double e_up = 0.0, e_dn = 0.0;
    const uint32_t lo = 0x00800000u, hi = 0x7F7FFFFFu;
    for (uint64_t b = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= hi;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const float x = __uint_as_float((uint32_t)b);
        float s;
        asm("sqrt.approx.f32 %0, %1;" : "=f"(s) : "f"(x));
        const double r = (double)s / sqrt((double)x) - 1.0;
        e_up = fmax(e_up, r);
        e_dn = fmax(e_dn, -r);
    }
    for (int o = 16; o > 0; o >>= 1) {
        e_up = fmax(e_up, __shfl_xor_sync(0xffffffffu, e_up, o));
        e_dn = fmax(e_dn, __shfl_xor_sync(0xffffffffu, e_dn, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(up, (unsigned long long)__double_as_longlong(e_up));     // non-negative: bit order = value order
        atomicMax(down, (unsigned long long)__double_as_longlong(e_dn));
    }
}

}  // namespace cil

extern "C" int32_t cil_diag_sqrt_approx_error(double* max_rel_up, double* max_rel_down) {
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, 16) != cudaSuccess) return -1;
    cudaMemset(d, 0, 16);
    cil::k_sqrt_approx_err<<<148 * 16, 256>>>(d, d + 1);
    unsigned long long h[2] = {0, 0};
    const cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return -1;
    memcpy(max_rel_up, &h[0], 8);
    memcpy(max_rel_down, &h[1], 8);
    return 0;
}

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
        if (mix == 3) k_alu_mix16<<<nsm * 3, threads>>>(out, n, 12345u, 1u);   // k_max16_reg's occupancy
        else if (mix == 1) k_alu_mix<1><<<blocks, threads>>>(out, n, 0.5f);
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
    // element-pairs per iteration per thread: 16 pairs x 4 elements (mix 3: 32 pairs x 8 elements)
    const double ep = mix == 3 ? (double)nsm * 3 * threads * (double)iters * 32.0 * 8.0
                               : (double)blocks * threads * (double)iters * 16.0 * 4.0;
    *element_pairs_per_s = ep / (t * 1e-3);
    *ms = t;
    return 0;
}
