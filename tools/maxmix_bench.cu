// Instruction-mix microbenchmark for the CUDA-core max family (|a - b| max over elements):
// register-only 4 x 8 pair tiles as in k_simt (RI = 8), element-pairs per second per mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/maxmix tools/maxmix_bench.cu && /tmp/maxmix
#include <cstdio>
#include <cuda_runtime.h>

template <int MIX>
__global__ void __launch_bounds__(128) k_mix(float* out, int iters, float seed) {
    float4 av[8], bv[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) av[i] = make_float4(seed * (i + 1), seed * (i + 2), seed * (i + 3), seed * (i + 4));
#pragma unroll
    for (int j = 0; j < 4; ++j) bv[j] = make_float4(seed * (j + 5), seed * (j + 6), seed * (j + 7), seed * (j + 8));
    float mx[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) mx[i][j] = 0.f;
    const float2 step = make_float2(1e-7f, -1e-7f);
    const float2 neg = make_float2(-seed * 1000.f, -seed * 1000.f);   // -1 at run time (seed = 1e-3)
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (MIX == 0) {          // FADD2 + FMNMX3 (k_simt today)
                    const float2 d0 = __fadd2_rn(make_float2(av[i].x, av[i].y), make_float2(-bv[j].x, -bv[j].y));
                    const float2 d1 = __fadd2_rn(make_float2(av[i].z, av[i].w), make_float2(-bv[j].z, -bv[j].w));
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d0.x), fabsf(d0.y)));
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d1.x), fabsf(d1.y)));
                } else if (MIX == 1) {   // scalar FADD + FMNMX3
                    const float d0 = av[i].x - bv[j].x, d1 = av[i].y - bv[j].y, d2 = av[i].z - bv[j].z,
                                d3 = av[i].w - bv[j].w;
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d0), fabsf(d1)));
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d2), fabsf(d3)));
                } else if (MIX == 2) {   // FADD2 only (subtraction throughput)
                    const float2 d0 = __fadd2_rn(make_float2(av[i].x, av[i].y), make_float2(-bv[j].x, -bv[j].y));
                    const float2 d1 = __fadd2_rn(make_float2(av[i].z, av[i].w), make_float2(-bv[j].z, -bv[j].w));
                    mx[i][j] += d0.x + d1.y;     // keep it alive cheaply (counted as extra FADDs)
                    mx[i][j] = mx[i][j] * 0.5f + d0.y - d1.x;
                } else if (MIX == 4) {   // FFMA2 (b * -1 + a, -1 from a register) + FMNMX3
                    const float2 d0 = __ffma2_rn(make_float2(bv[j].x, bv[j].y), neg, make_float2(av[i].x, av[i].y));
                    const float2 d1 = __ffma2_rn(make_float2(bv[j].z, bv[j].w), neg, make_float2(av[i].z, av[i].w));
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d0.x), fabsf(d0.y)));
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d1.x), fabsf(d1.y)));
                } else if (MIX == 5) {   // scalar FFMA (b * -1 + a) + FMNMX3
                    const float d0 = fmaf(bv[j].x, neg.x, av[i].x), d1 = fmaf(bv[j].y, neg.x, av[i].y);
                    const float d2 = fmaf(bv[j].z, neg.x, av[i].z), d3 = fmaf(bv[j].w, neg.x, av[i].w);
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d0), fabsf(d1)));
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(d2), fabsf(d3)));
                } else {                 // max only: FMNMX3 on operands (no subtraction)
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(av[i].x), fabsf(bv[j].y)));
                    mx[i][j] = fmaxf(mx[i][j], fmaxf(fabsf(av[i].z), fabsf(bv[j].w)));
                }
            }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float2 lo = __fadd2_rn(make_float2(bv[j].x, bv[j].y), step);
            float2 hi = __fadd2_rn(make_float2(bv[j].z, bv[j].w), step);
            bv[j] = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += mx[i][j];
    if (s == 12345.678f) out[threadIdx.x] = s;
}

template <int MIX>
void run(const char* name) {
    float* d;
    cudaMalloc(&d, 4096);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000, blocks = nsm * 8;
    k_mix<MIX><<<blocks, 128>>>(d, 100, 1e-3f);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_mix<MIX><<<blocks, 128>>>(d, iters, 1e-3f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ep = (double)blocks * 128 * iters * 8 * 4 * 4;   // element-pairs
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s %.3e element-pairs/s  (%.1f per SM-cycle at %d MHz)\n", name, ep / (ms * 1e-3),
           ep / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
    cudaFree(d);
}

int main() {
    run<0>("FADD2 + FMNMX3");
    run<1>("FADD + FMNMX3");
    run<2>("FADD2 only");
    run<3>("FMNMX3 only");
    run<4>("FFMA2(b,-1,a) + FMNMX3");
    run<5>("FFMA(b,-1,a) + FMNMX3");
    return 0;
}
