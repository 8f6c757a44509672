// stats.cu — steps a4-a7 tails: histogram -> counts / y (Eq. (1) normalisation),
// mu / Sigma over realisations, batched Cholesky log-likelihood
// (Eq. (4); Eq. (12)), and the SCIL per-theta tail (Alg. 3
// steps 4-6).  All FP64; latency-bound (one CTA per item).
#include <math_constants.h>

#include "cil_internal.cuh"

namespace cil {

// ------------------------------------------------------------------ finalize
// counts[p][q][m] = sum_{b > m} hist[p][0][0][q][b];  y = counts / (N * Nt).
__global__ void k_finalize(int nq, int M, SegParams sp, const uint64_t* __restrict__ hist,
                           uint64_t* __restrict__ counts, double* __restrict__ y, int64_t y_stride, double npairs) {
    const int p = blockIdx.x;
    for (int t = threadIdx.x; t < nq * M; t += blockDim.x) {
        const int q = t / M, m = t % M;
        uint64_t c = 0;
        for (int b = m + 1; b <= M; ++b) c += hist[hist_index(sp, nq, M, p, 0, 0, q, b)];
        if (counts) counts[(int64_t)p * nq * M + t] = c;
        if (y) y[(int64_t)p * y_stride + t] = npairs > 0 ? (double)c / npairs : 0.0;
    }
}

cudaError_t launch_finalize(int P, int nq, int M, const SegParams& sp, const uint64_t* hist,
                            uint64_t* counts, double* y, int64_t rows, int64_t cols,
                            const int32_t*, int32_t*, cudaStream_t st) {
    ProfScope ps_(K_TAIL, st);
    k_finalize<<<P, 128, 0, st>>>(nq, M, sp, hist, counts, y, (int64_t)nq * M, (double)rows * (double)cols);
    note_launch();
    return cudaGetLastError();
}

// y only, item stride y_stride (e.g. the y~ row of a bootstrap Y block)
cudaError_t launch_finalize_y(int P, int nq, int M, const SegParams& sp, const uint64_t* hist, double* y,
                              int64_t y_stride, double npairs, cudaStream_t st) {
    ProfScope ps_(K_TAIL, st);
    k_finalize<<<P, 128, 0, st>>>(nq, M, sp, hist, nullptr, y, y_stride, npairs);
    note_launch();
    return cudaGetLastError();
}

__global__ void k_normalize(int64_t n, const uint64_t* __restrict__ counts, double npairs, double* __restrict__ y) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = (double)counts[i] / npairs;
}

cudaError_t launch_normalize(int64_t n, const uint64_t* counts, double npairs, double* y, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    ProfScope ps_(K_TAIL, st);
    const int blocks = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
    k_normalize<<<blocks, 256, 0, st>>>(n, counts, npairs, y);
    note_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------------ stats
__global__ void k_mean(const double* __restrict__ Y, int64_t y_stride, int n, int D,
                       double* __restrict__ mu) {
    const int p = blockIdx.x;
    const double* Yp = Y + (int64_t)p * y_stride;
    for (int a = threadIdx.x; a < D; a += blockDim.x) {
        double s = 0.0;
        for (int v = 0; v < n; ++v) s += Yp[(int64_t)v * D + a];
        mu[(int64_t)p * D + a] = s / n;
    }
}

// Sigma[a][b] = 1/(n-1) sum_v (Y[v][a]-mu[a])(Y[v][b]-mu[b]); grid (D rows, P)
__global__ void k_cov(const double* __restrict__ Y, int64_t y_stride, int n, int D,
                      const double* __restrict__ mu, double* __restrict__ Sigma) {
    const int a = blockIdx.x, p = blockIdx.y;
    const double* Yp = Y + (int64_t)p * y_stride;
    const double* mp = mu + (int64_t)p * D;
    for (int b = threadIdx.x; b < D; b += blockDim.x) {
        double s = 0.0;
        for (int v = 0; v < n; ++v) s += (Yp[(int64_t)v * D + a] - mp[a]) * (Yp[(int64_t)v * D + b] - mp[b]);
        Sigma[((int64_t)p * D + a) * D + b] = s / (n - 1);
    }
}

// Fused mu + Sigma for one item per CTA when Y[p] and mu fit in shared memory ((n+1)*D*8 <= 200 KB;
// any D — the means live in the same dynamic allocation, after Y):
// the same two-pass sums as k_mean / k_cov, with the n-long sums split over the lanes of a
// warp (one warp per column a, then one warp per pair b <= a) and reduced by shuffles.
constexpr int kStatsSmem = 200 * 1024;
constexpr int kStatsThreads = 512;
__global__ void __launch_bounds__(kStatsThreads) k_stats_smem(const double* __restrict__ Y, int64_t y_stride, int n, int D,
                                                    double* __restrict__ mu, double* __restrict__ Sigma) {
    extern __shared__ double ys[];                   // [n][D], centred in place after pass 1, then mu[D]
    double* mus = ys + (size_t)n * D;
    const int p = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const double* Yp = Y + (int64_t)p * y_stride;
    for (int i = threadIdx.x; i < n * D; i += blockDim.x) ys[i] = Yp[i];
    __syncthreads();
    for (int a = w; a < D; a += nw) {
        double s = 0.0;
        for (int v = lane; v < n; v += 32) s += ys[v * D + a];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            mus[a] = s / n;
            mu[(int64_t)p * D + a] = s / n;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n * D; i += blockDim.x) ys[i] -= mus[i % D];
    __syncthreads();
    const int npair = D * (D + 1) / 2;
    for (int t = w; t < npair; t += nw) {
        int a = (int)((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);  // t = a(a+1)/2 + b, b <= a (corrected below)
        while (a * (a + 1) / 2 > t) --a;
        while ((a + 1) * (a + 2) / 2 <= t) ++a;
        const int b = t - a * (a + 1) / 2;
        double s = 0.0;
        for (int v = lane; v < n; v += 32) s += ys[v * D + a] * ys[v * D + b];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            const double c = s / (n - 1);
            Sigma[((int64_t)p * D + a) * D + b] = c;
            Sigma[((int64_t)p * D + b) * D + a] = c;
        }
    }
}

static cudaError_t launch_stats_strided(int P, const double* Y, int64_t y_stride, int n, int D,
                                        double* mu, double* Sigma, cudaStream_t st) {
    ProfScope ps_(K_TAIL, st);
    const size_t smem = sizeof(double) * ((size_t)n + 1) * D;
    if (smem <= (size_t)kStatsSmem) {
        static SmemAttrOnce attr;
        if (const cudaError_t e = attr.ensure(k_stats_smem, kStatsSmem); e != cudaSuccess) return e;
        k_stats_smem<<<P, kStatsThreads, smem, st>>>(Y, y_stride, n, D, mu, Sigma);
        note_launch();
        return cudaGetLastError();
    }
    k_mean<<<P, 128, 0, st>>>(Y, y_stride, n, D, mu);
    note_launch();
    dim3 g((unsigned)D, (unsigned)P);
    k_cov<<<g, 128, 0, st>>>(Y, y_stride, n, D, mu, Sigma);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_stats(int P, const double* Y, int n, int D, double* mu, double* Sigma, cudaStream_t st) {
    return launch_stats_strided(P, Y, (int64_t)n * D, n, D, mu, Sigma, st);
}

// ------------------------------------------------------------------ loglik
// One CTA per item.  Packed lower triangle L[i][j] at i(i+1)/2 + j in smem.
constexpr int kLogThreads = 256;

__global__ void __launch_bounds__(kLogThreads) k_loglik(const double* __restrict__ mu, int64_t mu_stride,
                                                        const double* __restrict__ Sigma, int64_t Sigma_stride,
                                                        const double* __restrict__ y, int64_t y_stride, int D,
                                                        double ridge, double* __restrict__ out,
                                                        int32_t* __restrict__ status, const int32_t* status_in) {
    extern __shared__ double sm[];
    double* L = sm;                                   // D(D+1)/2
    double* z = L + (int64_t)D * (D + 1) / 2;         // D
    double* rinv = z + D;                             // D: 1 / L_ii
    __shared__ double piv;
    __shared__ int fail;
    const int p = blockIdx.x;
    const double* S = Sigma + (int64_t)p * Sigma_stride;
    const double* m = mu + (int64_t)p * mu_stride;
    const double* yy = y + (int64_t)p * y_stride;
    for (int t = threadIdx.x; t < D * D; t += blockDim.x) {
        const int i = t / D, j = t % D;
        if (j <= i) L[i * (i + 1) / 2 + j] = S[(int64_t)i * D + j] + (i == j ? ridge : 0.0);
    }
    for (int i = threadIdx.x; i < D; i += blockDim.x) z[i] = yy[i] - m[i];
    if (threadIdx.x == 0) fail = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // left-looking Cholesky, column by column
    for (int j = 0; j < D; ++j) {
        const int dj = j * (j + 1) / 2;
        if (warp == 0) {
            double s = 0.0;
            for (int k = lane; k < j; k += 32) s += L[dj + k] * L[dj + k];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) {
                const double d = L[dj + j] - s;
                if (!(d > 0.0)) fail = 1;
                piv = sqrt(d);
                L[dj + j] = piv;
            }
        }
        __syncthreads();
        if (fail) break;
        for (int i = j + 1 + threadIdx.x; i < D; i += blockDim.x) {
            const int di = i * (i + 1) / 2;
            double t = L[di + j];
            for (int k = 0; k < j; ++k) t -= L[di + k] * L[dj + k];
            L[di + j] = t / piv;
        }
        __syncthreads();
    }
    const int32_t base = status_in ? status_in[p] : 0;
    if (fail) {
        if (threadIdx.x == 0) {
            out[3 * p + 0] = out[3 * p + 1] = out[3 * p + 2] = CUDART_NAN;
            status[p] = base | CIL_ITEM_NOTPD;
        }
        return;
    }
    // forward substitution z = L^{-1} r (warp 0), quad = z^T z, logdet = 2 sum ln L_ii; the
    // logarithms and pivot reciprocals are formed in parallel, off the substitution's chain
    if (warp == 0) {
        double logdet = 0.0;
        for (int i = lane; i < D; i += 32) {
            const double lii = L[i * (i + 1) / 2 + i];
            logdet += 2.0 * log(lii);
            rinv[i] = 1.0 / lii;
        }
        for (int o = 16; o > 0; o >>= 1) logdet += __shfl_xor_sync(0xffffffffu, logdet, o);
        __syncwarp();
        double quad = 0.0;
        for (int i = 0; i < D; ++i) {
            const int di = i * (i + 1) / 2;
            double s = 0.0;
            for (int k = lane; k < i; k += 32) s += L[di + k] * z[k];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            const double zi = (z[i] - s) * rinv[i];
            __syncwarp();
            if (lane == 0) z[i] = zi;
            __syncwarp();
            quad += zi * zi;
        }
        if (lane == 0) {
            out[3 * p + 0] = quad;
            out[3 * p + 1] = logdet;
            out[3 * p + 2] = -0.5 * quad - 0.5 * logdet - 0.5 * D * log(2.0 * CUDART_PI);
            status[p] = base;
        }
    }
}

// D <= 32: one warp per item, lane i owns row i of L (shared memory, stride 33 doubles: conflict-
// free per half-warp phase), synchronised by __syncwarp only.  Left-looking Cholesky: at column j
// lane j forms its pivot d_j = S_jj + ridge - sum_k L_jk^2, the lanes i > j then
// L_ij = (S_ij - sum_k L_ik L_jk) / L_jj; forward substitution column by column (z_k broadcast
// by shuffle, the lanes below update their right-hand sides).  Same outputs and statuses as
// k_loglik; the general kernel's block-wide barriers per column made it latency-bound (~19 us for
// D = 15).
constexpr int kLogWarpItems = 4;
__global__ void __launch_bounds__(32 * kLogWarpItems) k_loglik_warp(const double* __restrict__ mu, int64_t mu_stride,
                                                                    const double* __restrict__ Sigma, int64_t Sigma_stride,
                                                                    const double* __restrict__ y, int64_t y_stride, int D,
                                                                    double ridge, double* __restrict__ out,
                                                                    int32_t* __restrict__ status,
                                                                    const int32_t* status_in, int P) {
    __shared__ double Ls[kLogWarpItems][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = blockIdx.x * kLogWarpItems + warp;
    if (p >= P) return;                                  // warp-uniform
    double (*L)[33] = Ls[warp];
    const double* S = Sigma + (int64_t)p * Sigma_stride;
    const double* m = mu + (int64_t)p * mu_stride;
    const double* yy = y + (int64_t)p * y_stride;
    if (lane < D)
        for (int k = 0; k <= lane; ++k) L[lane][k] = S[(int64_t)lane * D + k] + (k == lane ? ridge : 0.0);
    double r = lane < D ? yy[lane] - m[lane] : 0.0;
    __syncwarp();
    bool fail = false;
    for (int j = 0; j < D; ++j) {
        double d = 0.0;
        if (lane == j) {
            d = L[j][j];
            for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k];
        }
        d = __shfl_sync(0xffffffffu, d, j);
        if (!(d > 0.0)) { fail = true; break; }          // warp-uniform
        const double piv = sqrt(d);
        if (lane == j) L[j][j] = piv;
        if (lane > j && lane < D) {
            double t = L[lane][j];
            for (int k = 0; k < j; ++k) t -= L[lane][k] * L[j][k];
            L[lane][j] = t / piv;
        }
        __syncwarp();
    }
    const int32_t base = status_in ? status_in[p] : 0;
    if (fail) {
        if (lane == 0) {
            out[3 * p + 0] = out[3 * p + 1] = out[3 * p + 2] = CUDART_NAN;
            status[p] = base | CIL_ITEM_NOTPD;
        }
        return;
    }
    double logdet = lane < D ? 2.0 * log(L[lane][lane]) : 0.0;
    for (int o = 16; o > 0; o >>= 1) logdet += __shfl_xor_sync(0xffffffffu, logdet, o);
    double quad = 0.0;
    for (int k = 0; k < D; ++k) {
        const double zk = __shfl_sync(0xffffffffu, r, k) / L[k][k];
        if (lane > k && lane < D) r -= L[lane][k] * zk;
        quad += zk * zk;
    }
    if (lane == 0) {
        out[3 * p + 0] = quad;
        out[3 * p + 1] = logdet;
        out[3 * p + 2] = -0.5 * quad - 0.5 * logdet - 0.5 * D * log(2.0 * CUDART_PI);
        status[p] = base;
    }
}

static cudaError_t launch_loglik_strided(int P, const double* mu, int64_t mu_stride, const double* Sigma,
                                         int64_t Sigma_stride, const double* y, int64_t y_stride, int D,
                                         double ridge, double* out, int32_t* status,
                                         const int32_t* status_in, cudaStream_t st) {
    if (D <= 32) {
        ProfScope ps_(K_TAIL, st);
        k_loglik_warp<<<(P + kLogWarpItems - 1) / kLogWarpItems, 32 * kLogWarpItems, 0, st>>>(
            mu, mu_stride, Sigma, Sigma_stride, y, y_stride, D, ridge, out, status, status_in, P);
        note_launch();
        return cudaGetLastError();
    }
    const size_t smem = sizeof(double) * ((size_t)D * (D + 1) / 2 + 2 * D);
    static SmemAttrOnce attr;
    if (cudaError_t e = attr.ensure(k_loglik, (int)(sizeof(double) * ((size_t)kMaxD * (kMaxD + 1) / 2 + 2 * kMaxD)));
        e != cudaSuccess)
        return e;
    ProfScope ps_(K_TAIL, st);
    k_loglik<<<P, kLogThreads, smem, st>>>(mu, mu_stride, Sigma, Sigma_stride, y, y_stride, D, ridge, out,
                                           status, status_in);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_loglik(int P, const double* mu, int64_t mu_stride, const double* Sigma,
                          int64_t Sigma_stride, const double* y, int D, double ridge, double* out,
                          int32_t* status, const int32_t* status_in, cudaStream_t st) {
    return launch_loglik_strided(P, mu, mu_stride, Sigma, Sigma_stride, y, D, D, ridge, out, status,
                                 status_in, st);
}

// ------------------------------------------------------------------ SCIL tail
// Y[p][v][q*M + m] for v = k*n_ens + l (Eq. (11)) and v = n_ens^2 for y~ (Eq. (13)):
//   counts of segment (rs = k, cs = l), resp. (rs = n_ens (the s_data rows), cs = k0[p]),
//   divided by N_set * N_tilde.
__global__ void k_build_Y(int n_ens, int nq, int M, SegParams sp, const uint64_t* __restrict__ hist,
                          double npairs, const int32_t* __restrict__ k0, double* __restrict__ Y,
                          int32_t* __restrict__ status, int swapped) {
    const int p = blockIdx.y;
    const int v = blockIdx.x;
    const int nv = n_ens * n_ens;
    const int D = nq * M;
    int rs, cs;
    if (v < nv) { rs = v / n_ens; cs = v % n_ens; }
    else {
        rs = n_ens;
        cs = k0[p];
        if (cs < 0 || cs >= n_ens) {                 // k0 outside [0, n_ens): an index outside its set
            if (threadIdx.x == 0) atomicOr(&status[p], CIL_ITEM_BADINDEX);
            cs = 0;
        }
    }
    for (int t = threadIdx.x; t < D; t += blockDim.x) {
        const int q = t / M, m = t % M;
        uint64_t c = 0;
        // swapped panels (the column panel ran as the Gram's rows): segments are [l][k]
        const int r_ = swapped ? cs : rs, c_ = swapped ? rs : cs;
        for (int b = m + 1; b <= M; ++b) c += hist[hist_index(sp, nq, M, p, r_, c_, q, b)];
        Y[((int64_t)p * (nv + 1) + v) * D + t] = (double)c / npairs;
    }
}

cudaError_t launch_synth_tail(int P, int n_ens, int nq, int M, const SegParams& sp, const uint64_t* hist,
                              int64_t N_set, int64_t N_tilde, const int32_t* k0, double ridge, double* out,
                              int32_t* status, double* Y, double* mu, double* Sigma, cudaStream_t st,
                              bool swapped) {
    const int nv = n_ens * n_ens, D = nq * M;
    dim3 g((unsigned)(nv + 1), (unsigned)P);
    {
        ProfScope ps_(K_TAIL, st);
        k_build_Y<<<g, 128, 0, st>>>(n_ens, nq, M, sp, hist, (double)N_set * (double)N_tilde, k0, Y, status,
                                     swapped ? 1 : 0);
    }
    note_launch();
    cudaError_t e = launch_stats_strided(P, Y, (int64_t)(nv + 1) * D, nv, D, mu, Sigma, st);
    if (e != cudaSuccess) return e;
    return launch_loglik_strided(P, mu, D, Sigma, (int64_t)D * D, Y + (int64_t)nv * D, (int64_t)(nv + 1) * D,
                                 D, ridge, out, status, status, st);
}

// Bootstrap tail (Alg. A2 steps 3-5): Y[p] = [n_rep replicate vectors ; y~], D each.
cudaError_t launch_boot_tail(int P, int n_rep, int D, double ridge, double* out, int32_t* status, double* Y,
                             double* mu, double* Sigma, cudaStream_t st) {
    cudaError_t e = launch_stats_strided(P, Y, (int64_t)(n_rep + 1) * D, n_rep, D, mu, Sigma, st);
    if (e != cudaSuccess) return e;
    return launch_loglik_strided(P, mu, D, Sigma, (int64_t)D * D, Y + (int64_t)n_rep * D, (int64_t)(n_rep + 1) * D,
                                 D, ridge, out, status, status, st);
}

// Alg. 1 / Alg. 2 training vectors: Y[p][v][q*M + m] for the unordered subset pairs k < l
// (lexicographic v), counts of segment (rs = k, cs = l) divided by N*N.
__global__ void k_build_pairs(int n_ens, int nq, int M, SegParams sp, const uint64_t* __restrict__ hist,
                              double npairs, double* __restrict__ Y) {
    const int p = blockIdx.y;
    const int v = blockIdx.x;
    int k = 0, rem = v;
    while (rem >= n_ens - 1 - k) { rem -= n_ens - 1 - k; ++k; }
    const int l = k + 1 + rem;
    const int D = nq * M;
    const int nv = n_ens * (n_ens - 1) / 2;
    for (int t = threadIdx.x; t < D; t += blockDim.x) {
        const int q = t / M, m = t % M;
        uint64_t c = 0;
        for (int b = m + 1; b <= M; ++b) c += hist[hist_index(sp, nq, M, p, k, l, q, b)];
        Y[((int64_t)p * nv + v) * D + t] = (double)c / npairs;
    }
}

cudaError_t launch_build_pairs(int P, int n_ens, int nq, int M, const SegParams& sp, const uint64_t* hist,
                               int64_t N, double* Y, cudaStream_t st) {
    const int nv = n_ens * (n_ens - 1) / 2;
    dim3 g((unsigned)nv, (unsigned)P);
    ProfScope ps_(K_TAIL, st);
    k_build_pairs<<<g, 128, 0, st>>>(n_ens, nq, M, sp, hist, (double)N * (double)N, Y);
    note_launch();
    return cudaGetLastError();
}

// ---- adaptive radii: R_0, R_M from the range of the distances
__global__ void k_range_init(int n, unsigned long long* __restrict__ range) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        range[i] = (i & 1) ? 0ull : (unsigned long long)__double_as_longlong(INFINITY);
}

cudaError_t launch_range_init(int P, int nq, unsigned long long* range, cudaStream_t st) {
    const int n = 2 * P * nq;
    ProfScope ps_(K_PREP, st);
    k_range_init<<<(n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024, 256, 0, st>>>(n, range);
    note_launch();
    return cudaGetLastError();
}

// R_0 = d_max (1 + margin), R_M = d_min (1 - margin) (reading R5: R_0 is not a bin, R_M is),
// law 0 = power  R_m = R_0 b^-m, b = (R_0/R_M)^(1/M);  law 1 = linear  R_m = R_0 - m (R_0 - R_M)/M;
// m = 1..M.  An item without a positive distance gets BADRADII.
__global__ void k_radii(int nq, int M, const unsigned long long* __restrict__ range, int law, double margin,
                        double* __restrict__ radii, int32_t* __restrict__ status) {
    const int p = blockIdx.x;
    for (int t = threadIdx.x; t < nq * M; t += blockDim.x) {
        const int q = t / M, m = t % M + 1;
        const double dmin = __longlong_as_double((long long)range[((int64_t)p * nq + q) * 2]);
        const double dmax = __longlong_as_double((long long)range[((int64_t)p * nq + q) * 2 + 1]);
        const double R0 = dmax * (1.0 + margin), RM = dmin * (1.0 - margin);
        double r;
        if (!(dmin > 0.0) || !(dmax >= dmin) || !isfinite(dmax)) {
            r = NAN;
            if (threadIdx.x == 0) atomicOr(&status[p], CIL_ITEM_BADRADII);
        } else if (law == 0) {
            r = R0 * pow(RM / R0, (double)m / M);
        } else {
            r = R0 - m * (R0 - RM) / M;
        }
        radii[(int64_t)p * nq * M + t] = r;
    }
}

cudaError_t launch_radii(int P, int nq, int M, const unsigned long long* range, int law, double margin, double* radii,
                         int32_t* status, cudaStream_t st) {
    ProfScope ps_(K_TAIL, st);
    k_radii<<<P, 128, 0, st>>>(nq, M, range, law, margin, radii, status);
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- chi^2 Gaussianity diagnostic
// Pearson's statistic of n squared Mahalanobis distances over the equiprobable chi^2_D bins whose
// interior edges the host computed (cil_gaussianity_pearson): bin of d2 = #{edges < d2} (numpy's
// searchsorted, side 'left'); out = {sum_b (c_b - n/B)^2 / (n/B), B - 1}.  One CTA.
__global__ void __launch_bounds__(256) k_chi2_pearson(int64_t n, const double* __restrict__ d2, Chi2Edges ed,
                                                     double* __restrict__ out) {
    __shared__ unsigned long long cnt[kMaxChi2Bins];
    for (int b = threadIdx.x; b < ed.nb; b += blockDim.x) cnt[b] = 0ull;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = d2[i];
        int b = 0;
        while (b < ed.nb - 1 && ed.e[b] < v) ++b;
        atomicAdd(&cnt[b], 1ull);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double expect = (double)n / ed.nb;
        double stat = 0.0;
        for (int b = 0; b < ed.nb; ++b) {
            const double d = (double)cnt[b] - expect;
            stat += d * d / expect;
        }
        out[0] = stat;
        out[1] = (double)(ed.nb - 1);
    }
}

cudaError_t launch_chi2_pearson(int64_t n, const double* d2, const Chi2Edges& ed, double* out, cudaStream_t st) {
    ProfScope ps_(K_TAIL, st);
    k_chi2_pearson<<<1, 256, 0, st>>>(n, d2, ed, out);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cil
