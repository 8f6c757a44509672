// resample.cu — bootstrap estimators (Alg. A1 step 2 and Alg. A2 steps 2.1-2.4,
// PAPER.md:648-723): correlation-integral vectors of resampled set pairs read off a
// per-pair bin matrix instead of recomputing distances.  For replicate k of item p with
// row draws I1[p][k][i] and column draws I2[p][k][j] (with repetition):
//   counts[q][m] = #{(i, j) : bins[p][q][I1[i]][I2[j]] > m}           (Eq. (1), strict <:
//   bins = #{m : d < R_m}, so d < R_m  <=>  bins > m for decreasing radii)
// One CTA per (k, p); per-thread shared histograms [bin][thread] updated with
// fire-and-forget shared atomics (no address conflicts), reduced once per measure.
#include "cil_internal.cuh"

namespace cil {

__global__ void k_check_index(const int32_t* __restrict__ idx, int64_t per_item, int64_t range,
                              int32_t* __restrict__ status) {
    const int p = blockIdx.y;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per_item; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = idx[p * per_item + i];
        bad |= (v < 0 || v >= range);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&status[p], CIL_ITEM_BADINDEX);
}

cudaError_t launch_check_index(int P, const int32_t* idx, int64_t per_item, int64_t range, int32_t* status,
                               cudaStream_t st) {
    if (per_item == 0 || P == 0) return cudaSuccess;
    const int64_t nb = (per_item + 255) / 256;
    dim3 grid((unsigned)(nb < 64 ? nb : 64), (unsigned)P);
    ProfScope ps_(K_PREP, st);
    k_check_index<<<grid, 256, 0, st>>>(idx, per_item, range, status);
    note_launch();
    return cudaGetLastError();
}

constexpr int kRsThreads = 256;

__global__ void __launch_bounds__(kRsThreads) k_resample(const uint8_t* __restrict__ bins, int64_t N, int64_t Nt,
                                                          int nq, int M, int n_rep, const int32_t* __restrict__ I1,
                                                          int64_t n1, const int32_t* __restrict__ I2, int64_t n2,
                                                          uint64_t* __restrict__ counts, double* __restrict__ y,
                                                          int64_t y_item_stride) {
    extern __shared__ uint32_t hs[];              // [M+1][kRsThreads]
    __shared__ uint32_t red[8][kMaxM + 1];
    const int k = blockIdx.x, p = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int32_t* i1 = I1 + ((int64_t)p * n_rep + k) * n1;
    const int32_t* i2 = I2 + ((int64_t)p * n_rep + k) * n2;
    const double npairs = (double)n1 * (double)n2;
    for (int q = 0; q < nq; ++q) {
        for (int b = 0; b <= M; ++b) hs[b * kRsThreads + tid] = 0u;
        __syncthreads();
        const uint8_t* Bq = bins + ((int64_t)p * nq + q) * N * Nt;
        // warp w takes draws i = w, w+8, ...; lanes stride over the column draws
        for (int64_t i = w; i < n1; i += kRsThreads / 32) {
            const int64_t r = __ldg(&i1[i]);
            if (r < 0 || r >= N) continue;          // flagged CIL_ITEM_BADINDEX by k_check_index
            const uint8_t* row = Bq + r * Nt;
            for (int64_t j = lane; j < n2; j += 32) {
                const int64_t c = __ldg(&i2[j]);
                if (c < 0 || c >= Nt) continue;
                const uint32_t b = __ldg(&row[c]);
                atomicAdd(&hs[(b <= (uint32_t)M ? b : (uint32_t)M) * kRsThreads + tid], 1u);
            }
        }
        __syncthreads();
        // per bin: block sum of the per-thread counters
        for (int b = 0; b <= M; ++b) {
            uint32_t v = hs[b * kRsThreads + tid];
            v = __reduce_add_sync(0xffffffffu, v);
            if (lane == 0) red[w][b] = v;
        }
        __syncthreads();
        if (tid < M) {
            // counts[m] = sum_{b > m} hist[b]
            uint64_t c = 0;
            for (int b = tid + 1; b <= M; ++b)
                for (int ww = 0; ww < kRsThreads / 32; ++ww) c += red[ww][b];
            if (counts) counts[(((int64_t)p * n_rep + k) * nq + q) * M + tid] = c;
            if (y) y[(int64_t)p * y_item_stride + (int64_t)k * nq * M + q * M + tid] = npairs > 0 ? (double)c / npairs : 0.0;
        }
        __syncthreads();
    }
}

cudaError_t launch_resample(int P, const uint8_t* bins, int64_t N, int64_t Nt, int nq, int M, int n_rep,
                            const int32_t* I1, int64_t n1, const int32_t* I2, int64_t n2, uint64_t* counts,
                            double* y, int64_t y_item_stride, int32_t* status, cudaStream_t st) {
    cudaError_t e = launch_check_index(P, I1, (int64_t)n_rep * n1, N, status, st);
    if (e != cudaSuccess) return e;
    e = launch_check_index(P, I2, (int64_t)n_rep * n2, Nt, status, st);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(uint32_t) * (size_t)(M + 1) * kRsThreads;
    static bool attr = false;
    if (!attr) {
        e = cudaFuncSetAttribute(k_resample, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sizeof(uint32_t) * (kMaxM + 1) * kRsThreads));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid((unsigned)n_rep, (unsigned)P);
    ProfScope ps_(K_RESAMPLE, st);
    k_resample<<<grid, kRsThreads, smem, st>>>(bins, N, Nt, nq, M, n_rep, I1, n1, I2, n2, counts, y, y_item_stride);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cil
