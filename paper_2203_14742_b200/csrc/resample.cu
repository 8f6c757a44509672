// resample.cu — bootstrap estimators (Alg. A1 step 2 and Alg. A2 steps 2.1-2.4,
// PAPER.md:648-723): correlation-integral vectors of resampled set pairs read off a
// per-pair bin matrix instead of recomputing distances.  For replicate k of item p with
// row draws I1[p][k][i] and column draws I2[p][k][j] (with repetition):
//   counts[q][m] = #{(i, j) : bins[p][q][I1[i]][I2[j]] > m}           (Eq. (1), strict <:
//   bins = #{m : d < R_m}, so d < R_m  <=>  bins > m for decreasing radii)
// k_resample: one CTA per (k, p); per-thread shared histograms [bin][thread] updated with
// fire-and-forget shared atomics (no address conflicts), reduced once per measure.  The
// default inside cil_synth_loglik_boot is the tensor-core form at the end of this file
// (k_rd_mult, k_rd_build_E, rowdot.cu, k_rd_final); k_resample serves
// cil_resample_counts, the fallback, and the one-replicate y~ counts.
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

// Multiplicity form of the same count: with m1[a] = #{i : I1[i] = a}, m2[b] = #{j : I2[j] = b},
//   counts[q][m] = sum_a m1[a] sum_b m2[b] [bins[q][a][b] > m]
// (a regrouping of the (i, j) double sum; repeated draws count once per draw).  The rows a
// with m1[a] > 0 are streamed with 16-byte loads (coalesced, no byte gathers); m1, m2 live
// in shared memory; the per-thread histograms take weighted fire-and-forget atomics.
__global__ void __launch_bounds__(kRsThreads) k_resample(const uint8_t* __restrict__ bins, int64_t N, int64_t Nt,
                                                          int nq, int M, int n_rep, const int32_t* __restrict__ I1,
                                                          int64_t n1, const int32_t* __restrict__ I2, int64_t n2,
                                                          uint64_t* __restrict__ counts, double* __restrict__ y,
                                                          int64_t y_item_stride, int32_t* __restrict__ status) {
    extern __shared__ uint32_t rs_smem[];
    uint32_t* hs = rs_smem;                                   // [M+1][kRsThreads]
    uint32_t* m1 = hs + (M + 1) * kRsThreads;                 // [round_up(N, 4)]
    uint32_t* m2 = m1 + ((N + 3) & ~(int64_t)3);              // [round_up(Nt, 16)], 16-byte aligned
    __shared__ uint32_t red[8][kMaxM + 1];
    const int k = blockIdx.x, p = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    // I1 == nullptr: the identity draw (every row a < n1 once; the y~ counts of Alg. A2 step 4)
    const int32_t* i1 = I1 ? I1 + ((int64_t)p * n_rep + k) * n1 : nullptr;
    const int32_t* i2 = I2 ? I2 + ((int64_t)p * n_rep + k) * n2 : nullptr;   // nullptr: identity columns
    const int64_t Nt16 = (Nt + 15) & ~(int64_t)15;
    for (int64_t a = tid; a < N; a += kRsThreads) m1[a] = 0u;
    for (int64_t b = tid; b < Nt16; b += kRsThreads) m2[b] = 0u;
    __syncthreads();
    bool bad = false;
    for (int64_t i = tid; i < n1; i += kRsThreads) {
        const int32_t r = i1 ? __ldg(&i1[i]) : (int32_t)i;
        if (r >= 0 && r < N) atomicAdd(&m1[r], 1u);          // invalid draws: flagged, skipped
        else bad = true;
    }
    for (int64_t j = tid; j < n2; j += kRsThreads) {
        const int32_t c = i2 ? __ldg(&i2[j]) : (int32_t)j;
        if (c >= 0 && c < Nt) atomicAdd(&m2[c], 1u);
        else bad = true;
    }
    if (__syncthreads_or(bad) && tid == 0) atomicOr(&status[p], CIL_ITEM_BADINDEX);
    // compact list of the distinct drawn rows (order irrelevant: integer sums)
    __shared__ int nrows;
    int32_t* rows = reinterpret_cast<int32_t*>(m2 + Nt16);   // [min(N, n1)]
    if (tid == 0) nrows = 0;
    __syncthreads();
    for (int64_t a = tid; a < N; a += kRsThreads)
        if (m1[a] != 0u) rows[atomicAdd(&nrows, 1)] = (int32_t)a;
    __syncthreads();
    const int nr = nrows;
    const double npairs = (double)n1 * (double)n2;
    // row loads: 16 B when rows are 16-byte aligned, 8 B when 8-byte aligned, else bytes
    const int align = (reinterpret_cast<uintptr_t>(bins) & 15u) ? 1 : (Nt % 16 == 0) ? 16 : (Nt % 8 == 0) ? 8 : 1;
    for (int q = 0; q < nq; ++q) {
        for (int b = 0; b <= M; ++b) hs[b * kRsThreads + tid] = 0u;
        __syncthreads();
        const uint8_t* Bq = bins + ((int64_t)p * nq + q) * N * Nt;
        uint32_t* myh = hs + tid;
        for (int ri = w; ri < nr; ri += kRsThreads / 32) {
            const int64_t a = rows[ri];
            const uint32_t wa = m1[a];
            const uint8_t* row = Bq + a * Nt;
            for (int64_t c0 = (int64_t)lane * 16; c0 < Nt; c0 += 32 * 16) {
                uint32_t bw[4];
                if (align == 16) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(row + c0));
                    bw[0] = v.x; bw[1] = v.y; bw[2] = v.z; bw[3] = v.w;
                } else if (align == 8) {
                    const uint2 v0 = __ldg(reinterpret_cast<const uint2*>(row + c0));
                    const uint2 v1 = c0 + 8 < Nt ? __ldg(reinterpret_cast<const uint2*>(row + c0 + 8)) : make_uint2(0u, 0u);
                    bw[0] = v0.x; bw[1] = v0.y; bw[2] = v1.x; bw[3] = v1.y;
                } else {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        uint32_t x = 0;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int64_t c = c0 + 4 * t + u;
                            if (c < Nt) x |= (uint32_t)__ldg(&row[c]) << (8 * u);
                        }
                        bw[t] = x;
                    }
                }
                const uint4* mv = reinterpret_cast<const uint4*>(m2 + c0);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uint4 mm = mv[t];
                    const uint32_t ms[4] = {mm.x, mm.y, mm.z, mm.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        // branch-free: an undrawn column (and the padding past Nt) adds 0
                        const uint32_t b = min((bw[t] >> (8 * u)) & 255u, (uint32_t)M);
                        atomicAdd(myh + b * kRsThreads, ms[u] * wa);
                    }
                }
            }
        }
        __syncthreads();
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
    cudaError_t e = cudaSuccess;
    const size_t smem = sizeof(uint32_t) * ((size_t)(M + 1) * kRsThreads + (size_t)((N + 3) & ~3ll) + (size_t)((Nt + 15) & ~15ll) +
                                            (size_t)(n1 < N ? n1 : N));
    if (smem > 200 * 1024) return cudaErrorInvalidValue;     // N + Nt <= ~47 k (host-checked)
    static SmemAttrOnce attr;
    if ((e = attr.ensure(k_resample, 200 * 1024)) != cudaSuccess) return e;
    dim3 grid((unsigned)n_rep, (unsigned)P);
    ProfScope ps_(K_RESAMPLE, st);
    k_resample<<<grid, kRsThreads, smem, st>>>(bins, N, Nt, nq, M, n_rep, I1, n1, I2, n2, counts, y, y_item_stride,
                                               status);
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- tensor-core resample
// The same multiplicity form as one integer GEMM per measure (rowdot.cu):
//   counts[k][v] = sum_b m2_k[b] sum_a m1_k[a] E[v][b][a],   E[v][b][a] = [bins[a][b] > v]
// A operand: M1 [P][n_rep][Kp] int8 (m1 <= n1 <= 127); B operand: E [P][Ntp/256][M][256][Kp] 0/1
// bytes (b-major blocks of 256 columns)
// (Ntp = N rounded up to 256, zero rows / columns beyond N); M2 [P][n_rep][Ntp] u16.

// multiplicities of replicate k of item p (shared-memory counts, then 16-byte row stores)
// One warp per replicate (4 per CTA): the multiplicities are u16 halves of shared 32-bit words
// (atomicAdd of 1 << 16 (idx & 1): m1 <= n1 <= 127, m2 <= n2 <= 65535, host-checked), so the
// M2 row is a straight copy of the words and no CTA-wide barrier is needed.
constexpr int kMultWarps = 4;
__global__ void __launch_bounds__(32 * kMultWarps) k_rd_mult(int64_t N, int64_t Kp, int64_t Ntp, int n_rep,
                                                             const int32_t* __restrict__ I1, int64_t n1,
                                                             const int32_t* __restrict__ I2, int64_t n2,
                                                             int8_t* __restrict__ M1, uint16_t* __restrict__ M2,
                                                             int32_t* __restrict__ status) {
    constexpr int U = 8;
    extern __shared__ uint32_t mm_smem[];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int k = blockIdx.x * kMultWarps + wq, p = blockIdx.y;
    if (k >= n_rep) return;                                   // whole warps only
    const int64_t words = (Kp + Ntp) / 2;
    uint32_t* m1 = mm_smem + wq * words;                      // [Kp / 2] u16 pairs
    uint32_t* m2 = m1 + Kp / 2;                               // [Ntp / 2]
    for (int64_t a = lane; a < words / 4; a += 32) reinterpret_cast<uint4*>(m1)[a] = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    bool bad = false;
    const int64_t row = (int64_t)p * n_rep + k;
    const int32_t* i1 = I1 + row * n1;
    const int32_t* i2 = I2 + row * n2;
    const int64_t n12 = n1 + n2;
    for (int64_t base = 0; base < n12; base += 32 * U) {
        int32_t r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + u * 32 + lane;
            r[u] = i < n1 ? __ldg(&i1[i]) : i < n12 ? __ldg(&i2[i - n1]) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = base + u * 32 + lane;
            if (i >= n12) break;
            if (r[u] >= 0 && r[u] < N) atomicAdd(&(i < n1 ? m1 : m2)[r[u] >> 1], 1u << (16 * (r[u] & 1)));
            else bad = true;
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&status[p], CIL_ITEM_BADINDEX);
    __syncwarp();
    // Kp % 128 == 0, Ntp % 256 == 0: 16 int8 / 8 u16 per 16-byte store
    uint4* d1 = reinterpret_cast<uint4*>(M1 + row * Kp);
    const uint4* s1 = reinterpret_cast<const uint4*>(m1);
    for (int64_t c = lane; c < Kp / 16; c += 32) {
        const uint4 v0 = s1[2 * c], v1 = s1[2 * c + 1];         // 16 u16 counts
        auto pk = [](uint32_t x, uint32_t y) { return (x & 0xffu) | (x >> 16) << 8 | (y & 0xffu) << 16 | (y >> 16) << 24; };
        d1[c] = make_uint4(pk(v0.x, v0.y), pk(v0.z, v0.w), pk(v1.x, v1.y), pk(v1.z, v1.w));
    }
    uint4* d2 = reinterpret_cast<uint4*>(M2 + row * Ntp);
    const uint4* s2 = reinterpret_cast<const uint4*>(m2);
    for (int64_t c = lane; c < Ntp / 8; c += 32) d2[c] = s2[c];
}

// E rows (v, b) of measure q, columns a0 .. a0+127, from a 128 (a) x 64 (b) block of bins (transposed
// through shared memory; 8-byte loads along b when the rows allow, 16-byte stores along a)
__global__ void __launch_bounds__(256) k_rd_build_E(const uint8_t* __restrict__ bins, int64_t N, int nq, int q,
                                                    int M, int64_t Kp, int64_t Ntp, int8_t* __restrict__ E) {
    __shared__ uint8_t tile[128][64 + 1];       // odd row stride: conflict-free column reads
    const int p = blockIdx.z, tid = threadIdx.x;
    const int64_t a0 = (int64_t)blockIdx.x * 128, b0 = (int64_t)blockIdx.y * 64;
    const uint8_t* Bq = bins + ((int64_t)p * nq + q) * N * N;
    const bool vec = (N % 8 == 0) && !(reinterpret_cast<uintptr_t>(bins) & 7u);
    if (vec) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {                      // 128 rows x 8 words of 8 bytes
            const int i = tid + 256 * r, ai = i >> 3, c = i & 7;
            const int64_t a = a0 + ai, b = b0 + 8 * c;
            uint2 v = make_uint2(0u, 0u);
            if (a < N && b < N) v = __ldg(reinterpret_cast<const uint2*>(Bq + a * N + b));   // N % 8 == 0
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                tile[ai][8 * c + u] = (uint8_t)(v.x >> (8 * u));
                tile[ai][8 * c + 4 + u] = (uint8_t)(v.y >> (8 * u));
            }
        }
    } else {
        for (int i = tid; i < 128 * 64; i += 256) {
            const int ai = i >> 6, bi = i & 63;
            const int64_t a = a0 + ai, b = b0 + bi;
            tile[ai][bi] = (a < N && b < N) ? __ldg(&Bq[a * N + b]) : (uint8_t)0;
        }
    }
    __syncthreads();
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
        const int bi = 32 * h + (tid >> 3), j = tid & 7;
        uint8_t v16[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v16[i] = tile[16 * j + i][bi];
        // b-major rows (rowdot.cu): row (bt, v, i) = bt M 256 + v 256 + i for b = 256 bt + i
        const int64_t b = b0 + bi;
        int8_t* dst = E + ((int64_t)p * M * Ntp + (b >> 8) * M * 256 + (b & 255)) * Kp + a0 + 16 * j;
        for (int v = 0; v < M; ++v) {
            uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i >> 2] |= (uint32_t)(v16[i] > v) << (8 * (i & 3));
            __stcs(reinterpret_cast<uint4*>(dst + (int64_t)v * 256 * Kp), make_uint4(w[0], w[1], w[2], w[3]));
        }
    }
}

__global__ void k_rd_final(const unsigned long long* __restrict__ cnt, int P, int n_rep, int M, int nq, int q,
                           double npairs, double* __restrict__ y, int64_t y_item_stride) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)P * n_rep * M) return;
    const int v = (int)(i % M);
    const int64_t pk = i / M;
    const int k = (int)(pk % n_rep), p = (int)(pk / n_rep);
    y[(int64_t)p * y_item_stride + ((int64_t)k * nq + q) * M + v] = (double)cnt[i] / npairs;   // as k_resample: same rounding
}

cudaError_t launch_rd_mult(int P, int64_t N, int64_t Kp, int64_t Ntp, int n_rep, const int32_t* I1, int64_t n1,
                           const int32_t* I2, int64_t n2, int8_t* M1, uint16_t* M2, int32_t* status, cudaStream_t st) {
    const size_t smem = sizeof(uint32_t) * (size_t)(Kp + Ntp) / 2 * kMultWarps;
    if (smem > 200 * 1024 || Kp % 128 || Ntp % 256) return cudaErrorInvalidValue;
    static SmemAttrOnce attr;
    if (cudaError_t e = attr.ensure(k_rd_mult, 200 * 1024); e != cudaSuccess) return e;
    ProfScope ps_(K_RESAMPLE, st);
    k_rd_mult<<<dim3((unsigned)((n_rep + kMultWarps - 1) / kMultWarps), (unsigned)P), 32 * kMultWarps, smem, st>>>(
        N, Kp, Ntp, n_rep, I1, n1, I2, n2, M1, M2, status);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_rd_build_E(int P, const uint8_t* bins, int64_t N, int nq, int q, int M, int64_t Kp, int64_t Ntp,
                              int8_t* E, cudaStream_t st) {
    if (Kp % 128 || Ntp % 256) return cudaErrorInvalidValue;
    ProfScope ps_(K_RESAMPLE, st);
    k_rd_build_E<<<dim3((unsigned)(Kp / 128), (unsigned)(Ntp / 64), (unsigned)P), 256, 0, st>>>(bins, N, nq, q, M,
                                                                                                Kp, Ntp, E);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_rd_final(const unsigned long long* cnt, int P, int n_rep, int M, int nq, int q, double npairs,
                            double* y, int64_t y_item_stride, cudaStream_t st) {
    const int64_t n = (int64_t)P * n_rep * M;
    ProfScope ps_(K_RESAMPLE, st);
    k_rd_final<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(cnt, P, n_rep, M, nq, q, npairs, y, y_item_stride);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cil
