// Which pipe runs FMNMX3? Issue-rate microbenchmark: VIMNMX3.U16x2 alone, FMNMX3 alone, and both
// interleaved on separate accumulators (if the rates add, the two use different pipes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/maxmix4 tools/maxmix4_bench.cu && /tmp/maxmix4
#include <cstdio>
#include <cuda_runtime.h>

template <int MIX>
__global__ void __launch_bounds__(128) k_mix(unsigned* out, int iters, unsigned seed) {
    unsigned ai[8], bi[8];
    float af[8], bf[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        ai[i] = seed * (i + 1); bi[i] = seed * (i + 9) + 3;
        af[i] = __uint_as_float((seed * (i + 3)) & 0x3f7fffffu); bf[i] = __uint_as_float((seed * (i + 5)) & 0x3f7fffffu);
    }
    unsigned mi[16];
    float mf[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) { mi[k] = 0u; mf[k] = 0.f; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (MIX == 0 || MIX == 2) mi[k] = __vimax3_u16x2(mi[k], ai[k & 7], bi[(k + 1) & 7]);
            if (MIX == 1 || MIX == 2) mf[k] = fmaxf(mf[k], fmaxf(fabsf(af[k & 7]), fabsf(bf[(k + 1) & 7])));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) { ai[i] ^= 0x00010001u; bf[i] = __uint_as_float(__float_as_uint(bf[i]) ^ 1u); }
    }
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += mi[k] ^ __float_as_uint(mf[k]);
    if (s == 0x12345678u) out[threadIdx.x] = s;
}

template <int MIX>
void run(const char* name) {
    unsigned* d;
    cudaMalloc(&d, 4096);
    int nsm, clk;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 20000, blocks = nsm * 8;
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
    const double per = (MIX == 2 ? 32.0 : 16.0);              // 3-input max instructions per iteration
    const double ins = (double)blocks * 4 * iters * per;        // warp-instructions
    printf("%-36s %.2f warp-instr per SM-cycle\n", name, ins / (ms * 1e-3) / nsm / (clk * 1e3));
    cudaFree(d);
}

int main() {
    run<0>("VIMNMX3.U16x2 alone");
    run<1>("FMNMX3 (|.|) alone");
    run<2>("both interleaved");
    return 0;
}
