// Issue-rate microbenchmark for max-family candidates on sm_100a (register-only 8 x 4 pair tiles,
// as in k_simt): element-pairs per SM-cycle for
//   F32   : FADD2 + FMNMX3(|.|)                    (k_simt today; 1 instruction per element-pair)
//   I16a  : VIADDMNMX.S16x2 max + min              (packed 16-bit fixed point; max(a - b) and min(a - b))
//   I16b  : VIADD.16x2 + VIMNMX3.S16x2 max/min     (packed 16-bit fixed point)
//   H16   : HFMA2 (a - b) + HMNMX2(|.|)            (packed FP16)
//   MIX   : half the pairs F32, half I16a          (FMA pipe and integer pipe together)
//   I16c  : VIADDMNMX.S16x2 max on (a, -b) and on (-a, b)  (needs -a, -b operands)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/maxmix2 tools/maxmix2_bench.cu && /tmp/maxmix2
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned f2u(float x) { return __float_as_uint(x); }

template <int MIX>
__global__ void __launch_bounds__(128) k_mix(unsigned* out, int iters, unsigned seed) {
    unsigned av[8][2], bv[4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { av[i][0] = seed * (i + 1); av[i][1] = seed * (i + 3) + 7; }
#pragma unroll
    for (int j = 0; j < 4; ++j) { bv[j][0] = seed * (j + 5) + 1; bv[j][1] = seed * (j + 9) + 3; }
    unsigned acc[8][4], acc2[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { acc[i][j] = 0u; acc2[i][j] = 0u; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                // 4 element-pairs per (i, j) per iteration in every variant
                if (MIX == 0) {
                    const float2 d0 = __fadd2_rn(make_float2(__uint_as_float(av[i][0]), __uint_as_float(av[i][1])),
                                                 make_float2(-__uint_as_float(bv[j][0]), -__uint_as_float(bv[j][1])));
                    const float2 d1 = __fadd2_rn(make_float2(__uint_as_float(av[i][1]), __uint_as_float(av[i][0])),
                                                 make_float2(-__uint_as_float(bv[j][1]), -__uint_as_float(bv[j][0])));
                    float m = __uint_as_float(acc[i][j]);
                    m = fmaxf(m, fmaxf(fabsf(d0.x), fabsf(d0.y)));
                    m = fmaxf(m, fmaxf(fabsf(d1.x), fabsf(d1.y)));
                    acc[i][j] = f2u(m);
                } else if (MIX == 1) {      // 2 words x 2 lanes = 4 element-pairs: 4 instructions
                    acc[i][j] = __viaddmax_s16x2(av[i][0], bv[j][0], acc[i][j]);
                    acc2[i][j] = __viaddmin_s16x2(av[i][0], bv[j][0], acc2[i][j]);
                    acc[i][j] = __viaddmax_s16x2(av[i][1], bv[j][1], acc[i][j]);
                    acc2[i][j] = __viaddmin_s16x2(av[i][1], bv[j][1], acc2[i][j]);
                } else if (MIX == 2) {
                    const unsigned d0 = __vadd2(av[i][0], bv[j][0]), d1 = __vadd2(av[i][1], bv[j][1]);
                    acc[i][j] = __vimax3_s16x2(acc[i][j], d0, d1);
                    acc2[i][j] = __vimin3_s16x2(acc2[i][j], d0, d1);
                } else if (MIX == 3) {
                    const __half2 a0 = *reinterpret_cast<const __half2*>(&av[i][0]);
                    const __half2 a1 = *reinterpret_cast<const __half2*>(&av[i][1]);
                    const __half2 b0 = *reinterpret_cast<const __half2*>(&bv[j][0]);
                    const __half2 b1 = *reinterpret_cast<const __half2*>(&bv[j][1]);
                    __half2 m = *reinterpret_cast<const __half2*>(&acc[i][j]);
                    m = __hmax2(m, __habs2(__hsub2(a0, b0)));
                    m = __hmax2(m, __habs2(__hsub2(a1, b1)));
                    acc[i][j] = *reinterpret_cast<unsigned*>(&m);
                } else if (MIX == 4) {      // half F32 (2 pairs), half I16a (2 pairs)
                    if (j < 2) {
                        const float2 d0 = __fadd2_rn(make_float2(__uint_as_float(av[i][0]), __uint_as_float(av[i][1])),
                                                     make_float2(-__uint_as_float(bv[j][0]), -__uint_as_float(bv[j][1])));
                        const float2 d1 = __fadd2_rn(make_float2(__uint_as_float(av[i][1]), __uint_as_float(av[i][0])),
                                                     make_float2(-__uint_as_float(bv[j][1]), -__uint_as_float(bv[j][0])));
                        float m = __uint_as_float(acc[i][j]);
                        m = fmaxf(m, fmaxf(fabsf(d0.x), fabsf(d0.y)));
                        m = fmaxf(m, fmaxf(fabsf(d1.x), fabsf(d1.y)));
                        acc[i][j] = f2u(m);
                    } else {
                        acc[i][j] = __viaddmax_s16x2(av[i][0], bv[j][0], acc[i][j]);
                        acc2[i][j] = __viaddmin_s16x2(av[i][0], bv[j][0], acc2[i][j]);
                        acc[i][j] = __viaddmax_s16x2(av[i][1], bv[j][1], acc[i][j]);
                        acc2[i][j] = __viaddmin_s16x2(av[i][1], bv[j][1], acc2[i][j]);
                    }
                } else if (MIX == 5) {      // VIMNMX3 only (max of 3), 2 per 4 element-pairs
                    acc[i][j] = __vimax3_s16x2(acc[i][j], av[i][0], bv[j][0]);
                    acc2[i][j] = __vimin3_s16x2(acc2[i][j], av[i][1], bv[j][1]);
                } else if (MIX == 6) {      // VIADD.16x2 only, 2 per 4 element-pairs
                    acc[i][j] = __vadd2(acc[i][j], __vadd2(av[i][0], bv[j][0]));
                } else if (MIX == 7) {      // F32 subtraction + integer max of |d| bits (LOP abs + VIMNMX3.U32?)
                    const float2 d0 = __fadd2_rn(make_float2(__uint_as_float(av[i][0]), __uint_as_float(av[i][1])),
                                                 make_float2(-__uint_as_float(bv[j][0]), -__uint_as_float(bv[j][1])));
                    const float2 d1 = __fadd2_rn(make_float2(__uint_as_float(av[i][1]), __uint_as_float(av[i][0])),
                                                 make_float2(-__uint_as_float(bv[j][1]), -__uint_as_float(bv[j][0])));
                    acc[i][j] = max(acc[i][j], max(f2u(d0.x) & 0x7fffffffu, f2u(d0.y) & 0x7fffffffu));
                    acc2[i][j] = max(acc2[i][j], max(f2u(d1.x) & 0x7fffffffu, f2u(d1.y) & 0x7fffffffu));
                }
            }
#pragma unroll
        for (int j = 0; j < 4; ++j) { bv[j][0] += 0x00010001u; bv[j][1] ^= 0x00020002u; }
    }
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += acc[i][j] ^ acc2[i][j];
    if (s == 0x12345678u) out[threadIdx.x] = s;
}

template <int MIX>
void run(const char* name) {
    unsigned* d;
    cudaMalloc(&d, 4096);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int bps : {4, 8, 16}) {
        const int iters = 20000, blocks = nsm * bps;
        k_mix<MIX><<<blocks, 128>>>(d, 100, 12345u);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_mix<MIX><<<blocks, 128>>>(d, iters, 12345u);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ep = (double)blocks * 128 * iters * 8 * 4 * 4;   // element-pairs
        int clk;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("%-40s %2d CTA/SM  %.3e element-pairs/s  (%.1f per SM-cycle)\n", name, bps, ep / (ms * 1e-3),
               ep / (ms * 1e-3) / nsm / (clk * 1e3));
    }
    cudaFree(d);
}

int main() {
    run<0>("F32: FADD2 + FMNMX3");
    run<1>("I16a: VIADDMNMX.S16x2 max+min");
    run<2>("I16b: VIADD.16x2 + VIMNMX3 max/min");
    run<3>("H16: HADD2 + HMNMX2|.|");
    run<4>("MIX: half F32, half I16a");
    run<5>("VIMNMX3.S16x2 only (x2 rate)");
    run<6>("VIADD.16x2 only (x2 rate)");
    run<7>("F32 sub + integer max of |d| bits");
    return 0;
}
