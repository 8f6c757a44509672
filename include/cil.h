/*
 * cil.h — C ABI of libcil.so, the B200 (sm_100a) hot path of the Correlation
 * Integral Likelihood method (arXiv 2203.14742; PAPER.md = /root/reference/PAPER.md).
 *
 * Conventions for every call:
 *  - Pointers are DEVICE pointers unless marked [host].  The caller owns every
 *    buffer; the library never allocates device memory.  Scratch comes from a
 *    caller-provided workspace sized by the matching *_workspace_size() call.  It grows
 *    with the pairs of a call: the packed operands (O((N + Nt) K)), plus for the max family
 *    on the fixed-point engine 2 bytes per pair and region (C5: 20000^2 pairs -> 2.4 GB)
 *    and the re-check list (32 B per 128 (pair, measure) cases + 8 MB): for set pairs far
 *    beyond C5 call in row blocks of A (the counts are additive).
 *  - Calls are asynchronous on `stream` (a cudaStream_t passed as void*; NULL =
 *    legacy default stream).  They never synchronise the device and never allocate, so a
 *    call (or a whole step of calls) can be captured into a CUDA graph and replayed on new
 *    contents of the same buffers (tests/test_gpu_graph.py); the one-time kernel attribute
 *    setup happens on a call's first (eager) use.
 *  - The return value reports HOST-side validation only: CIL_OK, CIL_EINVAL (bad
 *    argument), CIL_EUNSUPPORTED (a valid request this build does not support),
 *    CIL_ECUDA (a launch failed; cil_last_cuda_error() has the cudaError_t).
 *    Data-dependent conditions are written to item_status[] on the device:
 *    CIL_ITEM_NONFINITE (an input pattern value is NaN/Inf), CIL_ITEM_NOTPD (a
 *    Cholesky pivot <= 0), CIL_ITEM_BADRADII (radii not > 0 and strictly
 *    decreasing), CIL_ITEM_OVERFLOW (the exact re-check list overflowed and the exact
 *    all-pairs fallback ran instead: counts are still exact, the call was slower).  Bits OR
 *    together.
 *  - Patterns are FP32, one pattern = S species x H rows x W columns, row-major
 *    [S][H][W] ("pattern-major then component-major then row-major");
 *    K = S*H*W, pattern p of a set starts at base + p*ld (ld >= K, in floats).
 *  - Batched calls take 1 <= P <= 21845 items (the grids put items on a 65535-wide grid
 *    axis, three per item for the max family); more is CIL_EINVAL.  Split larger batches.
 *    A set (or a SCIL / training / bootstrap panel) holds at most 2 097 120 = 65535 x 32
 *    patterns (the CUDA-core engines' 32-row tiles on a grid axis); more is CIL_EINVAL
 *    (workspace queries return 0).  Larger sets: row blocks (cil_features is additive over
 *    them, as the multi-GPU split uses).  The tensor-core engines pack at most 2^31 - 1 rows
 *    per call (P times both sets' rows; TMA coordinates are int32): above, CIL_EUNSUPPORTED —
 *    split the batch or use CIL_ENGINE_SIMT.
 *  - Thread-safe: no global mutable state besides a once-per-device kernel
 *    attribute setup (atomic), thread-local launch counters / diagnostics settings, one
 *    library-owned side stream (+ two events) per host thread and device for the concurrent
 *    engines (created by the thread's first features-type call on the device — make that an
 *    eager call before capturing graphs), and the opt-in profiling diagnostics.
 */
#ifndef CIL_H
#define CIL_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CIL_API __attribute__((visibility("default")))
#else
#define CIL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CIL_OK = 0,
    CIL_EINVAL = 1,
    CIL_EUNSUPPORTED = 2,
    CIL_ENOMEM = 3, /* workspace too small */
    CIL_ECUDA = 4
} cil_status;

enum {
    CIL_ITEM_OK = 0,
    CIL_ITEM_NONFINITE = 1,
    CIL_ITEM_NOTPD = 2,
    CIL_ITEM_BADRADII = 4,
    CIL_ITEM_OVERFLOW = 8,
    CIL_ITEM_BADINDEX = 16 /* a resampling / subset index outside its set (bootstrap calls) */
};

/* Distance measures, a bit mask.  A feature vector concatenates the selected
 * measures in BIT ORDER (multi-feature CIL), each contributing M
 * values.  Definitions (discrete equivalents; readings R1-R4 of
 * DESIGN.md): u = a - b, h = grid spacing, w = h^dim (dim 2 if H > 1 else 1),
 * D_x u, D_y u = forward differences / h inside each species, last node omitted;
 * a_al = sqrt(w * sum (D^al u)^2), m_al = max |D^al u| over all species/nodes. */
typedef enum {
    CIL_L2 = 1 << 0,        /* Eq. (5)  a_0                          */
    CIL_LINF = 1 << 1,      /* Eq. (6)  m_0                          */
    CIL_W12SUM = 1 << 2,    /* Eq. (7)  a_0 + a_x + a_y              */
    CIL_W12 = 1 << 3,       /* Eq. (8)  sqrt(a_0^2 + a_x^2 + a_y^2)  */
    CIL_W1INF = 1 << 4,     /* Eq. (9)  max(m_0, m_x, m_y)           */
    CIL_W1INFSUM = 1 << 5   /* Eq. (10) m_0 + m_x + m_y              */
} cil_dist;
#define CIL_ALL_DISTS 0x3Fu

/* Engine for the L2-type measures (the max family L-inf, W1-inf, W1-inf-sum always runs on the
 * CUDA-core tile engine).  Every engine decides a (pair, radius) in-kernel only when the radius lies
 * outside an interval of the measure that contains its exact FP64 value (reading R13);
 * the others are re-evaluated exactly in FP64, so the counts are those of the plain definition.
 *  TC_I8     three-digit INT8 fixed point per row (x~ = sigma (2^16 h + 2^8 m + l), 22 bits), six
 *            exact int32 tcgen05 kind::i8 products per K step, a WORST-CASE interval (Cauchy-Schwarz
 *            on the dropped digit products, rigorous residual norms, directed rounding) — valid for
 *            every input; K in exact chunks of 65536, up to 24 chunks per launch (L2 alone:
 *            K <= 1 572 864; L2 + W12 + W12SUM from the augmented rows [x | D_x x | D_y x]: the
 *            three blocks' chunks together), longer rows run on the CUDA cores.  Column segments
 *            (SCIL blocks) need >= 21 columns (M <= 16 for W12 / W12SUM), else the measures run
 *            on the CUDA cores.
 *  SIMT      FP32 differences on CUDA cores, FP64-flushed sums, rigorous rounding bounds.
 *  TC_3XBF16 / TC_3XTF32  float split (hi.hi + hi.lo + lo.hi, FP32 tensor accumulation): explicit
 *            options only, their bound is statistical (not worst-case). */
typedef enum {
    CIL_ENGINE_AUTO = 0,      /* TC_I8 where it applies, else the CUDA cores (never the float splits) */
    CIL_ENGINE_TC_3XBF16 = 1,
    CIL_ENGINE_TC_3XTF32 = 2,
    CIL_ENGINE_SIMT = 3,
    CIL_ENGINE_TC_I8 = 4
} cil_engine;

typedef struct {
    int32_t S, H, W; /* species, rows, columns; H == 1 -> 1-D grid (no y-derivative) */
    double h;        /* grid spacing; <= 0 -> 1/(W-1) */
    uint32_t gs;     /* species whose derivative terms enter the gradient-based norms (bit s);
                        0 = all species (RD-ODE, the diffusive component only) */
} cil_grid;

/* ------------------------------------------------------------------------ */
/* cil_features — correlation-integral counts of P independent set pairs.
 *
 * For item p, measure slot q (bit order of dist_mask) and radius index m:
 *   counts[p][q][m] = #{(i,j) : d_q(A_p,i , B_p,j) < radii[p][q][m]}   (Eq. (1), strict <)
 *   y[p][q][m]      = counts / (N * Nt)                                  (Eq. (1)/(2))
 * i in [0,N), j in [0,Nt).  A_p,i = A + p*strideA + i*lda; B_p,j = B + p*strideB + j*ldb.
 *
 *  radii       [P or 1][n_meas][M] FP64, device; radii_stride = 0 shares one set
 *              of radii across items, else it is the per-item stride in doubles.
 *              Each row must be > 0 and strictly decreasing (checked on device).
 *  counts      [P][n_meas][M] uint64, device, written (not accumulated).
 *  y           [P][n_meas][M] FP64, device, nullable.
 *  item_status [P] int32, device, written.
 *  engine      L2 engine (above).
 * Constraints (else CIL_EINVAL / CIL_EUNSUPPORTED): P >= 1, N >= 0, Nt >= 0,
 * S,H,W >= 1, ld >= K, 1 <= M <= 64, dist_mask in [1, 63], measures other than
 * L2/LINF need W >= 2; strides >= 0; pointers non-NULL (A/B may be NULL when
 * N resp. Nt is 0).  N*Nt == 0 gives counts 0 and y 0.  Vectorised loads need
 * K, ld and strides to be multiples of 4 floats and A, B 16-byte aligned
 * (else CIL_EUNSUPPORTED).
 * ------------------------------------------------------------------------ */
CIL_API size_t cil_features_workspace_size(int32_t P, int64_t N, int64_t Nt, cil_grid g,
                                   uint32_t dist_mask, int32_t M, cil_engine engine);

CIL_API cil_status cil_features(int32_t P,
                        const float* A, int64_t strideA, int64_t lda, int64_t N,
                        const float* B, int64_t strideB, int64_t ldb, int64_t Nt,
                        cil_grid g, uint32_t dist_mask,
                        const double* radii, int64_t radii_stride, int32_t M,
                        uint64_t* counts, double* y, int32_t* item_status,
                        cil_engine engine, void* ws, size_t ws_bytes, void* stream);

/* cil_features_recheck_count — DIAGNOSTIC (synchronises): the number of (pair, measure) cases the
 * last cil_features call on this workspace listed for the exact FP64 re-check (the engines' rigorous
 * intervals contained a radius), and the list capacity (beyond it the exact all-pairs fallback runs
 * and the items carry CIL_ITEM_OVERFLOW).  Arguments as cil_features_workspace_size plus the workspace. */
CIL_API cil_status cil_features_recheck_count(int32_t P, int64_t N, int64_t Nt, cil_grid g, uint32_t dist_mask,
                                              int32_t M, cil_engine engine, const void* ws, uint64_t* listed,
                                              uint64_t* capacity);

/* ------------------------------------------------------------------------ */
/* cil_normalize — y[i] = (double)counts[i] / npairs for i < n (the 1/(N x N~) of Eq. (1),
 * PAPER.md:98).  Used after an all-reduce of row-block-sharded counts (each rank's
 * cil_features normalises by its own shard only).  counts uint64 [n], y FP64 [n], device;
 * npairs > 0. */
CIL_API cil_status cil_normalize(int64_t n, const uint64_t* counts, double npairs, double* y, void* stream);

/* ------------------------------------------------------------------------ */
/* cil_stats — mu and Sigma of n realisations (Alg. 1 step 3,
 * PAPER.md:131), batched over P:
 *   mu[p][a]       = (1/n) sum_v Y[p][v][a]
 *   Sigma[p][a][b] = 1/(n-1) sum_v (Y[p][v][a]-mu[p][a]) (Y[p][v][b]-mu[p][b])
 * Two-pass FP64.  Y [P][n][D], mu [P][D], Sigma [P][D][D] row-major, all device.
 * n >= 2, 1 <= D.
 * ------------------------------------------------------------------------ */
CIL_API cil_status cil_stats(int32_t P, const double* Y, int32_t n, int32_t D,
                     double* mu, double* Sigma, void* stream);

/* ------------------------------------------------------------------------ */
/* cil_gaussianity_pearson — the numerical Gaussianity check of CIL vectors:
 * given the squared Mahalanobis distances d2 [n] (device; e.g. the quad column of cil_loglik of
 * each vector against the vectors' own mu, Sigma), Pearson's statistic over `bins` equiprobable
 * bins of the chi^2_D distribution: out (device double[2]) = {sum_b (c_b - n/bins)^2 / (n/bins),
 * bins - 1}; c_b = #{k : bin of d2_k = b}, the bin of v = #{interior edges < v}.  The edges are
 * chi^2_D quantiles b/bins computed on the host in FP64 (cil_chi2_quantile) and passed by value.
 * 2 <= bins <= 64, n >= 1, D >= 1, else CIL_EINVAL.  Asynchronous on `stream`. */
CIL_API cil_status cil_gaussianity_pearson(int64_t n, const double* d2, int32_t D, int32_t bins, double* out,
                                           void* stream);

/* cil_chi2_quantile — host: the prob-quantile of chi^2_D (regularised incomplete gamma, series /
 * continued fraction in FP64, bisection to 200 steps); NaN outside D >= 1, 0 < prob < 1. */
CIL_API double cil_chi2_quantile(int32_t D, double prob);

/* ------------------------------------------------------------------------ */
/* cil_loglik — Gaussian log-likelihood of P vectors (Eq. (4), PAPER.md:146;
 * Eq. (12)):  Sigma + ridge*I = L L^T (Cholesky, no pivoting),
 * z = L^{-1}(y - mu),  out[p] = {quad = z^T z (the paper's f), logdet = 2 sum ln L_ii,
 * loglik = -quad/2 - logdet/2 - (D/2) ln 2pi}.
 *  mu [.][D] with stride mu_stride (0 = shared), Sigma [.][D][D] with stride
 *  Sigma_stride (0 = shared), y_obs [P][D], out [P][3], item_status [P]
 *  (CIL_ITEM_NOTPD and out = NaN when a pivot <= 0).  ridge >= 0.  1 <= D <= 192.
 * ------------------------------------------------------------------------ */
CIL_API cil_status cil_loglik(int32_t P, const double* mu, int64_t mu_stride,
                      const double* Sigma, int64_t Sigma_stride,
                      const double* y_obs, int32_t D, double ridge,
                      double* out, int32_t* item_status, void* stream);

/* ------------------------------------------------------------------------ */
/* cil_synth_loglik — SCIL (Alg. 3; Eqs. (11)-(13)) for P
 * parameter proposals theta_p, each with a pool of N_syn = n_ens*(N_set+N_tilde)
 * synthetic patterns at pools + p*pool_stride (row stride ld):
 *   subset k = rows [k*N, (k+1)*N), N = N_set + N_tilde;
 *   s^{k,1} = its first N_set rows, s^{k,2} = its last N_tilde rows;
 *   y^{k,l} = C(R_p, s^{k,1}, s^{l,2}) for all k,l in [0,n_ens) (k = l included,
 *   PAPER.md:244), vector index v = k*n_ens + l;  mu_theta, Sigma_theta over the
 *   n_ens^2 vectors;  y~ = C(R_p, s_data, s^{k0[p],2}) (Eq. (13));
 *   out[p] = {quad, logdet, loglik} of y~ under N(mu_theta, Sigma_theta + ridge I).
 *  data   [N_set][K] (row stride ld_data), the observed patterns s_data.
 *  k0     [P] int32 in [0, n_ens), device (the caller draws it); a k0 outside that
 *         range sets CIL_ITEM_BADINDEX on the item (y~ then uses subset 0).
 *  radii  [P][n_meas][M], device (per-theta radii).
 *  Y_out  nullable [P][n_ens*n_ens + 1][n_meas*M] FP64: the vectors, y~ last.
 * Constraints: n_ens >= 2, N_set >= 1, N_tilde >= 1, D = n_meas*M <= 192.
 * ------------------------------------------------------------------------ */
CIL_API size_t cil_synth_workspace_size(int32_t P, int32_t n_ens, int32_t N_set, int32_t N_tilde,
                                cil_grid g, uint32_t dist_mask, int32_t M, cil_engine engine);

CIL_API cil_status cil_synth_loglik(int32_t P, const float* pools, int64_t pool_stride, int64_t ld,
                            int32_t n_ens, int32_t N_set, int32_t N_tilde,
                            const float* data, int64_t ld_data, const int32_t* k0,
                            cil_grid g, uint32_t dist_mask, const double* radii, int32_t M,
                            double ridge, double* out, int32_t* item_status, double* Y_out,
                            cil_engine engine, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* cil_minmax_scale — the scaled-pattern mode: for each of
 * the n patterns X + r*ldx and each species s,
 *   Y_s(x) = (X_s(x) - min_x X_s) / (max_x X_s - min_x X_s)   over the species' H x W values,
 * in FP64, rounded to FP32; a constant species maps to 0 (reading R17).  Y + r*ldy may be X
 * (in place).  The paper restricts scaled data to the L2-type norms.
 * ------------------------------------------------------------------------ */
CIL_API cil_status cil_minmax_scale(int64_t n, const float* X, int64_t ldx, float* Y, int64_t ldy, cil_grid g,
                                    void* stream);

/* ------------------------------------------------------------------------ */
/* Adaptive radii: "R_0 (resp. R_M) the maximum (resp.
 * minimum) distance of any two patterns", then the power law R_m = R_0 b^-m with
 * R_M / R_0 = b^-M, or the linear law R_m = R_0 - m (R_0 - R_M)/M, m = 1..M.
 *
 * cil_distance_range — range[p][q][0] = min over pairs (i, j) of d_q(A_p,i, B_p,j) among the
 * positive distances (a pattern against itself is not a pair of two patterns; reading R16),
 * range[p][q][1] = the maximum; FP64, from the exact per-pair measures of the CUDA-core
 * engine (FP32 differences, FP64 sums).  Arguments as cil_features (strides may be 0);
 * range [P][n_meas][2] FP64 device.
 * cil_radii_from_range — radii[p][q][m-1] from range with R_0 = max (1 + margin),
 * R_M = min (1 - margin) (reading R5; margin in [0, 1)); law 0 = power, 1 = linear; an
 * item without a positive distance gets CIL_ITEM_BADRADII and NaN radii.
 * ------------------------------------------------------------------------ */
CIL_API size_t cil_range_workspace_size(int32_t P, int64_t N, int64_t Nt, cil_grid g, uint32_t dist_mask);
CIL_API cil_status cil_distance_range(int32_t P, const float* A, int64_t strideA, int64_t lda, int64_t N,
                                      const float* B, int64_t strideB, int64_t ldb, int64_t Nt, cil_grid g,
                                      uint32_t dist_mask, double* range, int32_t* item_status, void* ws,
                                      size_t ws_bytes, void* stream);
CIL_API cil_status cil_radii_from_range(int32_t P, int32_t n_meas, int32_t M, const double* range, int32_t law,
                                        double margin, double* radii, int32_t* item_status, void* stream);

/* ------------------------------------------------------------------------ */
/* cil_train_vectors — the training vectors of Alg. 1 (CIL) and Alg. 2
 * (MCIL): for item p the set X_p (n_ens*N patterns at X + p*stride, row
 * stride ld) is divided into the subsets s^k = rows [kN, (k+1)N) (step 1), and for the
 * C(n_ens, 2) unordered subset pairs k < l (reading R15)
 *   Y[p][v][q*M + m] = C(R_p,q,m, s^k, s^l) = #{(i,j) : d_q(s^k_i, s^l_j) < R} / N^2   (Eq. (1))
 * with v the index of (k, l) in lexicographic order (v = 0 for (0,1), 1 for (0,2), ...).
 * mu_0, Sigma_0 (step 3) are cil_stats of the n_ens*(n_ens-1)/2 vectors of an item.
 * radii [P or shared][n_meas][M] (radii_stride 0 = shared); Y [P][n_ens(n_ens-1)/2][n_meas*M]
 * FP64 device.  Engines as cil_features (AUTO: INT8 tensor cores for the L2-type family when
 * N >= 21 columns per subset, else CUDA cores).
 * ------------------------------------------------------------------------ */
CIL_API size_t cil_train_workspace_size(int32_t P, int32_t n_ens, int32_t N, cil_grid g, uint32_t dist_mask,
                                        int32_t M, cil_engine engine);
CIL_API cil_status cil_train_vectors(int32_t P, const float* X, int64_t stride, int64_t ld, int32_t n_ens,
                                     int32_t N, cil_grid g, uint32_t dist_mask, const double* radii,
                                     int64_t radii_stride, int32_t M, double* Y, int32_t* item_status,
                                     cil_engine engine, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* Bootstrap estimators (Alg. A1 / A2).  The
 * resampled sets of the bootstrap are drawn WITH repetition from fixed sets, so every
 * distance they need is a distance between two patterns of the fixed sets: the library
 * computes each pair's bin index once (cil_bin_matrix) and reads the correlation-integral
 * vector of any resampled pair of sets off it (cil_resample_counts) — the counts of
 * Eq. (1) on the resampled sets, exactly (repeated patterns count once per draw).
 * The random draws are the caller's (index lists), so the library is deterministic.
 *
 * cil_bin_matrix — for item p, measure slot q (bit order), i < N, j < Nt:
 *   bins[p][q][i][j] = #{m : d_q(A_p,i , B_p,j) < radii[p*radii_stride + q*M + m]}  in [0, M]
 * (radii strictly decreasing, so d < R_m  <=>  bins > m).  Arguments as cil_features;
 * strideA / strideB may be 0 (the same set for every item).  bins [P][n_meas][N][Nt] uint8,
 * device, row-major, written completely.  engine: AUTO / TC_I8 (L2, W12, W12SUM on the INT8
 * tensor-core engine, the max family on the CUDA cores; every pair whose interval contains a radius
 * is re-evaluated in FP64) or SIMT; TC_3XBF16 / TC_3XTF32 -> CIL_EUNSUPPORTED.
 * ------------------------------------------------------------------------ */
CIL_API size_t cil_bin_matrix_workspace_size(int32_t P, int64_t N, int64_t Nt, cil_grid g, uint32_t dist_mask,
                                             int32_t M, cil_engine engine);
CIL_API cil_status cil_bin_matrix(int32_t P, const float* A, int64_t strideA, int64_t lda, int64_t N,
                                  const float* B, int64_t strideB, int64_t ldb, int64_t Nt, cil_grid g,
                                  uint32_t dist_mask, const double* radii, int64_t radii_stride, int32_t M,
                                  uint8_t* bins, int32_t* item_status, cil_engine engine, void* ws,
                                  size_t ws_bytes, void* stream);

/* cil_resample_counts — Alg. A1 step 2 / Alg. A2 steps 2.1-2.4: replicate k < n_rep of
 * item p takes the row draws I1[p][k][0..n1) (indices into the N rows of bins[p]) and
 * the column draws I2[p][k][0..n2) (indices into its Nt columns);
 *   counts[p][k][q][m] = #{(i, j) in [0,n1) x [0,n2) : bins[p][q][I1[p][k][i]][I2[p][k][j]] > m}
 *   y[p*y_item_stride + k*n_meas*M + q*M + m] = counts / (n1*n2)          (Eq. (1))
 * bins [P][n_meas][N][Nt] uint8 (cil_bin_matrix); I1 [P][n_rep][n1], I2 [P][n_rep][n2] int32;
 * counts [P][n_rep][n_meas][M] uint64 (nullable), y FP64 (nullable, not both null);
 * y_item_stride 0 -> n_rep*n_meas*M.  An index outside its range sets CIL_ITEM_BADINDEX
 * on the item and the draw is skipped.  No workspace.  Shared-memory limit:
 * 4*((M+1)*256 + N + Nt) <= 200 KB (N + Nt <= ~47 000 at M = 13), else CIL_EUNSUPPORTED.
 * ------------------------------------------------------------------------ */
CIL_API cil_status cil_resample_counts(int32_t P, const uint8_t* bins, int64_t N, int64_t Nt, int32_t n_meas,
                                       int32_t M, int32_t n_rep, const int32_t* I1, int64_t n1,
                                       const int32_t* I2, int64_t n2, uint64_t* counts, double* y,
                                       int64_t y_item_stride, int32_t* item_status, void* stream);

/* cil_synth_loglik_boot — SCIL with bootstrapping (Alg. A2) for P
 * proposals theta_p, each with a pool of N_syn synthetic patterns at pools + p*pool_stride
 * (row stride ld); N_t = N_syn - N_set:
 *   bins_p = cil_bin_matrix(pool_p x pool_p) (all pool pairs, once; step 2.4's distances)
 *   for k < n_rep: s^1 = pool rows I1[p][k][0..N_set), s^2 = pool rows I2[p][k][0..N_t)
 *     (steps 2.1-2.2: the caller draws with replacement, s^2 from the patterns not drawn
 *     into s^1), y^k = C(R_p, s^1, s^2) read off bins_p            (steps 2.3-2.4)
 *   mu_theta, Sigma_theta over the n_rep vectors (two-pass, 1/(n_rep - 1))    (step 3)
 *   y~ = C(R_p, s_data, pool rows J[p][0..N_t)), J a subset drawn by the caller (step 4)
 *   out[p] = {quad, logdet, loglik} of y~ under N(mu_theta, Sigma_theta + ridge I) (step 5)
 * data [N_set][K] (row stride ld_data); I1 [P][n_rep][N_set], I2 [P][n_rep][N_t],
 * J [P][N_t] int32 device; radii [P][n_meas][M]; Y_out nullable
 * [P][n_rep + 1][n_meas*M] FP64 (the replicate vectors, y~ last).
 * Constraints: 1 <= N_set < N_syn, n_rep >= 2, D = n_meas*M <= 192; the workspace holds
 * the P bin matrices (P * n_meas * N_syn^2 bytes).
 * ------------------------------------------------------------------------ */
CIL_API size_t cil_synth_boot_workspace_size(int32_t P, int32_t N_syn, int32_t N_set, int32_t n_rep,
                                             cil_grid g, uint32_t dist_mask, int32_t M, cil_engine engine);
CIL_API cil_status cil_synth_loglik_boot(int32_t P, const float* pools, int64_t pool_stride, int64_t ld,
                                         int32_t N_syn, const float* data, int64_t ld_data, int32_t N_set,
                                         int32_t n_rep, const int32_t* I1, const int32_t* I2, const int32_t* J,
                                         cil_grid g, uint32_t dist_mask, const double* radii, int32_t M,
                                         double ridge, double* out, int32_t* item_status, double* Y_out,
                                         cil_engine engine, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* cil_diag_gram — DIAGNOSTIC (not on the hot path): runs the tensor-core L2 engine on one
 * set pair without binning.  TC_I8: d2E[i][j] = (lo, hi), the engine's interval of the unweighted
 * distance |a_i - b_j| (it must contain the exact value for every pair).  TC_3XBF16 / TC_3XTF32:
 * d2E[i][j] = (the FP32 d^2, its statistical error bound E).  engine must be TC_3XBF16, TC_3XTF32 or TC_I8;
 * d2E [N][Nt][2] FP32 device; ws_bytes >= cil_features_workspace_size(1, N, Nt, g, CIL_L2,
 * 1, engine) + 512.  Rows the engine does not take (TC_I8: more than 24 K chunks) -> CIL_EUNSUPPORTED.
 * ------------------------------------------------------------------------ */
CIL_API cil_status cil_diag_gram(const float* A, int64_t lda, int64_t N, const float* B, int64_t ldb,
                                 int64_t Nt, cil_grid g, cil_engine engine, float* d2E, void* ws,
                                 size_t ws_bytes, void* stream);

/* cil_diag_gram_family — DIAGNOSTIC: the three-phase INT8 engine (L2, W12SUM, W12 on tensor
 * cores) on one set pair without binning: vE[k][i][j] = (lo, hi), its interval of kind k = 0:
 * L2/sqrt(w) (the unweighted distance), 1: W12^2/w, 2: W12SUM/sqrt(w).
 * vE [3][N][Nt][2] FP32 device; needs W >= 2; ws_bytes >=
 * cil_features_workspace_size(1, N, Nt, g, CIL_L2|CIL_W12SUM|CIL_W12, 1, CIL_ENGINE_TC_I8) + 512.
 * ------------------------------------------------------------------------ */
CIL_API cil_status cil_diag_gram_family(const float* A, int64_t lda, int64_t N, const float* B, int64_t ldb,
                                        int64_t Nt, cil_grid g, float* vE, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* cil_diag_alu_ceiling — DIAGNOSTIC: measured issue ceiling of the CUDA-core engines'
 * inner-loop instruction mix (mix 0: FADD2+FMNMX3+FFMA2, 1: FADD2+FMNMX3, 2: FADD2+FFMA2 — the FP32
 * engine; 3: IMAD + VIMNMX3.U16x2 max/min — the fixed-point max-family engine) in element-pairs per
 * second on the current device (register-only kernel on the legacy stream, synchronous).  Returns
 * 0, or -1 on a CUDA error. */
CIL_API int32_t cil_diag_alu_ceiling(int32_t mix, int32_t iters, double* element_pairs_per_s, double* ms);

/* cil_diag_sqrt_approx_error — DIAGNOSTIC: exhaustive check of the hardware square-root
 * approximation (sqrt.approx.f32) that the INT8 engine's interval bounds use with a 2^-21
 * inflation: over every normal positive FP32 x, the largest relative error above (max_rel_up) and
 * below (max_rel_down) the correctly rounded FP64 square root.  Allocates 16 B of device memory and
 * synchronises (diagnostic only).  Returns 0, or -1 on a CUDA error. */
CIL_API int32_t cil_diag_sqrt_approx_error(double* max_rel_up, double* max_rel_down);

/* cil_diag_bounds_violations — DIAGNOSTIC: in a bounds-checked build (-DCIL_BOUNDS_CHECK, used in
 * place of compute-sanitizer, which this GPU pool does not allow) the number of out-of-range global
 * accesses the INT8 engine, the CUDA-core engine and the re-check detected since load (synchronous);
 * -1 in the normal build. */
CIL_API int64_t cil_diag_bounds_violations(void);

/* cil_diag_limit_recheck_list — DIAGNOSTIC: on the calling host thread, cap the exact re-check list of
 * subsequent calls at `limit` entries (< 0: no cap), so tests can force the exact all-pairs fallback
 * that runs when the list overflows (counts stay exact; items get CIL_ITEM_OVERFLOW). */
CIL_API void cil_diag_limit_recheck_list(int64_t limit);

/* cil_diag_recheck_sort_min — DIAGNOSTIC: on the calling host thread, re-check lists of at least `n`
 * entries take the row-bucketed pass (list counting-sorted by pattern row, each pair evaluated once;
 * recheck.cu), shorter ones the entry-by-entry pass.  Default 8192; n <= 0 restores it, n = 1 forces
 * the bucketed pass for every non-empty list (tests).  Results are identical either way. */
CIL_API void cil_diag_recheck_sort_min(int64_t n);

/* cil_diag_concurrent_engines — DIAGNOSTIC: on the calling host thread, when a call has both the
 * tensor-core family and the max family (AUTO / TC_I8 with Linf, W1inf or W1infsum), run the max
 * family's integer-pipe engine on a library-owned side stream concurrently with the tensor-core
 * engine (on = 1, default; the side stream is forked from and joined back into the caller's stream
 * with events, so the call stays asynchronous and graph-capturable) or serially on the caller's
 * stream (on = 0).  Results are identical either way. */
CIL_API void cil_diag_concurrent_engines(int32_t on);

/* ------------------------------------------------------------------------ */
/* Kernel timing (diagnostics, used by bench.py for the live roofline).  While enabled on
 * the calling host thread, every kernel the library launches is bracketed by CUDA events
 * recorded on its launching stream.  cil_prof_read waits for those events and returns, per
 * kernel class (0 prep, 1 pack, 2 tensor-core Gram, 3 CUDA-core tile engine, 4 L2 re-check,
 * 5 stats/loglik/SCIL tail, 6 bootstrap resampling), the summed milliseconds ms[7] and launch
 * counts launches[7], then clears the record.  Returns 7 (the number of classes) or -1 on a
 * CUDA error. */
CIL_API void cil_prof_enable(int32_t on);
CIL_API int32_t cil_prof_read(double* ms, int64_t* launches);

/* ------------------------------------------------------------------------ */
CIL_API const char* cil_status_string(cil_status s);
CIL_API int32_t cil_last_cuda_error(void);  /* cudaError_t of the last failed call on this thread */
CIL_API int32_t cil_version(void);          /* MAJOR*10000 + MINOR*100 + PATCH */
/* number of kernel launches the last successful call on this thread issued */
CIL_API int32_t cil_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CIL_H */
