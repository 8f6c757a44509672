// Issue-rate microbenchmark, round 2: the packed 16-bit max family with the add moved off the
// integer ALU pipe.  Biased operands (a + 16384, -b + 16384 in [384, 32384]) make one 32-bit add
// produce both 16-bit sums with no carry between the halves; then VIMNMX3.U16x2 max / min.
//   I16b : VIADD.16x2 + VIMNMX3.S16x2 max/min            (all on the ALU pipe; max16.cu r2 first cut)
//   U32a : plain 32-bit add (compiler's choice) + VIMNMX3.U16x2 max/min
//   U32m : IMAD a * one + b (one from a register: FMA pipe) + VIMNMX3.U16x2 max/min
//   U32h : half the adds IMAD, half IADD3
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/maxmix3 tools/maxmix3_bench.cu && /tmp/maxmix3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned imad(unsigned a, unsigned one, unsigned b) {
    unsigned d;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(one), "r"(b));
    return d;
}

template <int MIX>
__global__ void __launch_bounds__(128) k_mix(unsigned* out, int iters, unsigned seed, unsigned one) {
    unsigned av[8][4], bv[4][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int t = 0; t < 4; ++t) av[i][t] = (seed * (i + 1) * (t + 3)) & 0x3fff3fffu;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int t = 0; t < 4; ++t) bv[j][t] = (seed * (j + 5) * (t + 7) + 1) & 0x3fff3fffu;
    unsigned mx[8][4], mn[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { mx[i][j] = 0u; mn[i][j] = 0xffffffffu; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                unsigned d[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    if (MIX == 0) d[t] = __vadd2(av[i][t], bv[j][t]);
                    else if (MIX == 1) d[t] = av[i][t] + bv[j][t];
                    else if (MIX == 2) d[t] = imad(av[i][t], one, bv[j][t]);
                    else d[t] = (t & 1) ? imad(av[i][t], one, bv[j][t]) : av[i][t] + bv[j][t];
                }
                if (MIX == 0) {
                    mx[i][j] = __vimax3_s16x2(mx[i][j], d[0], d[1]);
                    mn[i][j] = __vimin3_s16x2(mn[i][j], d[0], d[1]);
                    mx[i][j] = __vimax3_s16x2(mx[i][j], d[2], d[3]);
                    mn[i][j] = __vimin3_s16x2(mn[i][j], d[2], d[3]);
                } else {
                    mx[i][j] = __vimax3_u16x2(mx[i][j], d[0], d[1]);
                    mn[i][j] = __vimin3_u16x2(mn[i][j], d[0], d[1]);
                    mx[i][j] = __vimax3_u16x2(mx[i][j], d[2], d[3]);
                    mn[i][j] = __vimin3_u16x2(mn[i][j], d[2], d[3]);
                }
            }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int t = 0; t < 4; ++t) bv[j][t] ^= 0x00010001u << (t & 1);
    }
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += mx[i][j] ^ mn[i][j];
    if (s == 0x12345678u) out[threadIdx.x] = s;
}

template <int MIX>
void run(const char* name) {
    unsigned* d;
    cudaMalloc(&d, 4096);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int bps : {3, 4, 8}) {
        const int iters = 10000, blocks = nsm * bps;
        k_mix<MIX><<<blocks, 128>>>(d, 100, 12345u, 1u);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_mix<MIX><<<blocks, 128>>>(d, iters, 12345u, 1u);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ep = (double)blocks * 128 * iters * 8 * 4 * 8;   // element-pairs (8 per (i, j))
        int clk;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("%-44s %d CTA/SM  %.3e element-pairs/s  (%.1f per SM-cycle)\n", name, bps, ep / (ms * 1e-3),
               ep / (ms * 1e-3) / nsm / (clk * 1e3));
    }
    cudaFree(d);
}

int main() {
    run<0>("I16b: VIADD.16x2 + VIMNMX3.S16x2");
    run<1>("U32a: 32-bit add + VIMNMX3.U16x2");
    run<2>("U32m: IMAD(a, one, b) + VIMNMX3.U16x2");
    run<3>("U32h: half IMAD, half add + VIMNMX3.U16x2");
    return 0;
}
