/*
 * cil_oracle.c — plain, slow, obviously-correct FP64 CPU oracle for the CIL hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2203_14742_b200/, libcil.so) never links, imports or calls it, and this
 * file shares no code, header, table or constant with the CUDA path.
 *
 * Every function below is the plain definition written out, in the paper's order
 * and notation (arXiv 2203.14742 = /root/reference/PAPER.md):
 *   Eq. (1)  PAPER.md:96-100   C(R,s,s~,||.||) = 1/(N*N~) sum_i sum_j #(||s_i - s~_j|| < R)
 *   Eq. (2)  PAPER.md:102-107  y_m^{k,l} = C(R_m, s^k, s^l)
 *   Eq. (4)  PAPER.md:144-148  f = (y-mu)^T Sigma^{-1} (y-mu)
 *   Eqs. (5)-(10) PAPER.md:178-193  the six norms (discrete equivalents)
 *   Eq. (11)-(13) PAPER.md:236-258, Alg. 3 PAPER.md:260-297  SCIL
 *   Alg. A1 / A2 PAPER.md:648-723  bootstrap (resampled set pairs)
 *   mu/Sigma: PAPER.md:111, 131 (mean and covariance of the realisations)
 * Readings where the paper is silent are listed in DESIGN.md "Readings" (R1..R10)
 * and cited inline as [Rn].
 *
 * Precision: inputs are the FP32 patterns, up-cast exactly to FP64; every
 * arithmetic step is FP64.  No SIMD intrinsics, no fast-math (compiled -O2).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL 1
#define OR_NONFINITE 1
#define OR_NOTPD 2

/* Measure slots, in bit order (concatenation order, Eq. (5)..(10)) [R9]. */
enum { M_L2 = 0, M_LINF = 1, M_W12SUM = 2, M_W12 = 3, M_W1INF = 4, M_W1INFSUM = 5, N_MEAS_MAX = 6 };

typedef struct {
    int S, H, W;   /* species, rows, columns of one pattern; layout [S][H][W] row-major */
    double h;      /* grid spacing; <=0 -> 1/(W-1) [R2] */
    unsigned gs;   /* species with derivative terms (bit s); 0 = all [R18] */
} or_grid;

static double grid_h(const or_grid *g) {
    if (g->h > 0.0) return g->h;
    if (g->W >= 2) return 1.0 / (double)(g->W - 1); /* h = 1/(M_dim - 1) */
    return 1.0;
}

/*
 * Sub-norms of the difference u = a - b of two patterns (FP64).
 *   s0 = sum u^2,  sx = sum (D_x u)^2,  sy = sum (D_y u)^2
 *   m0 = max |u|,  mx = max |D_x u|,    my = max |D_y u|
 * D_h f(x_j) = (f(x_{j+1}) - f(x_j))/h, the forward difference of PAPER.md:823-826,
 * taken along each axis inside each species [R3]; the last node has the Neumann
 * ghost f_{M+1} = f_M, so its forward difference is 0 and it is
 * omitted from sums and maxima [R3].  Species are combined by summing inside L2-type
 * sub-norms and taking the max inside max-type sub-norms [R4].
 */
void oracle_subnorms(const float *a, const float *b, const or_grid *g, double out[6]) {
    const int S = g->S, H = g->H, W = g->W;
    const double h = grid_h(g);
    double s0 = 0, sx = 0, sy = 0, m0 = 0, mx = 0, my = 0;
    for (int s = 0; s < S; ++s) {
        const int grad = g->gs == 0 || ((g->gs >> s) & 1u);   /* derivative terms of species s [R18] */
        for (int r = 0; r < H; ++r) {
            for (int c = 0; c < W; ++c) {
                size_t e = ((size_t)s * H + r) * W + c;
                double u = (double)a[e] - (double)b[e];
                s0 += u * u;
                if (fabs(u) > m0) m0 = fabs(u);
                if (!grad) continue;
                if (c + 1 < W) {
                    double u1 = (double)a[e + 1] - (double)b[e + 1];
                    double dx = (u1 - u) / h;
                    sx += dx * dx;
                    if (fabs(dx) > mx) mx = fabs(dx);
                }
                if (r + 1 < H) {
                    double u1 = (double)a[e + W] - (double)b[e + W];
                    double dy = (u1 - u) / h;
                    sy += dy * dy;
                    if (fabs(dy) > my) my = fabs(dy);
                }
            }
        }
    }
    out[0] = s0; out[1] = sx; out[2] = sy; out[3] = m0; out[4] = mx; out[5] = my;
}

/*
 * The six distances (Eqs. (5)-(10)) from the sub-norms.
 * Quadrature weight w = h^dim on L2-type sub-norms, none on max-type [R1];
 * dim = 2 when H > 1, else 1 (1-D grids, Table 1).
 *   a_alpha = sqrt(w * s_alpha)
 *   (5)  L2      = a_0
 *   (6)  Linf    = m_0
 *   (7)  |||.|||_{W12}  = a_0 + a_x + a_y          (sum over |alpha| <= 1)
 *   (8)  ||.||_{W12}    = sqrt(a_0^2 + a_x^2 + a_y^2)
 *   (9)  ||.||_{W1inf}  = max(m_0, m_x, m_y)
 *   (10) |||.|||_{W1inf}= m_0 + m_x + m_y
 */
void oracle_measures(const double sub[6], const or_grid *g, double d[6]) {
    const double h = grid_h(g);
    const double w = (g->H > 1) ? h * h : h;
    double a0 = sqrt(w * sub[0]), ax = sqrt(w * sub[1]), ay = sqrt(w * sub[2]);
    double m0 = sub[3], mx = sub[4], my = sub[5];
    d[M_L2] = a0;
    d[M_LINF] = m0;
    d[M_W12SUM] = a0 + ax + ay;
    d[M_W12] = sqrt(a0 * a0 + ax * ax + ay * ay);
    double t = m0;
    if (mx > t) t = mx;
    if (my > t) t = my;
    d[M_W1INF] = t;
    d[M_W1INFSUM] = m0 + mx + my;
}

void oracle_pair_distances(const float *a, const float *b, const or_grid *g, double d[6]) {
    double sub[6];
    oracle_subnorms(a, b, g, sub);
    oracle_measures(sub, g, d);
}

static int popcount6(uint32_t mask) {
    int n = 0;
    for (int i = 0; i < N_MEAS_MAX; ++i) n += (mask >> i) & 1u;
    return n;
}

/* ---------------------------------------------------------------------------
 * Features (Eq. (1)/(2)): counts cnt[q][m] = #{(i,j): d_q(A_i, B_j) < R[q][m]}
 * (strict <), for every selected measure q (slots in bit order [R9]).
 * Band counts for parity: lo = #{d < R(1-band)}, hi = #{d < R(1+band)}; a GPU
 * count is correct iff lo <= gpu <= hi (pairs within band*R of a radius are the
 * ambiguous ones the north star excludes).
 * y[q][m] = cnt / (N * N~)  (the 1/(N x N~) normalisation of Eq. (1)).
 * ------------------------------------------------------------------------- */
typedef struct {
    const float *A; int64_t lda; int64_t N;
    const float *B; int64_t ldb; int64_t Nt;
    or_grid g; uint32_t mask; const double *radii; int M; double band;
    int64_t row0, row1;
    int64_t *cnt, *lo, *hi;   /* private per thread, [nq][M] */
    int64_t n_amb;
    int nonfinite;
} feat_job;

static void *feat_worker(void *arg) {
    feat_job *J = (feat_job *)arg;
    const int nq = popcount6(J->mask);
    int slot[N_MEAS_MAX], q = 0;
    for (int i = 0; i < N_MEAS_MAX; ++i)
        if ((J->mask >> i) & 1u) slot[q++] = i;
    const size_t K = (size_t)J->g.S * J->g.H * J->g.W;
    for (int64_t i = J->row0; i < J->row1; ++i) {
        const float *a = J->A + i * J->lda;
        for (size_t e = 0; e < K; ++e) if (!isfinite(a[e])) J->nonfinite = 1;
        for (int64_t j = 0; j < J->Nt; ++j) {
            const float *b = J->B + j * J->ldb;
            double d[6];
            oracle_pair_distances(a, b, &J->g, d);
            for (q = 0; q < nq; ++q) {
                double dq = d[slot[q]];
                for (int m = 0; m < J->M; ++m) {
                    double R = J->radii[q * J->M + m];
                    if (dq < R) J->cnt[q * J->M + m] += 1;
                    if (dq < R * (1.0 - J->band)) J->lo[q * J->M + m] += 1;
                    if (dq < R * (1.0 + J->band)) J->hi[q * J->M + m] += 1;
                    if (fabs(dq - R) <= J->band * R) J->n_amb += 1;
                }
            }
        }
    }
    return NULL;
}

/* returns 0 ok, 1 if any input is non-finite (counts still computed), -1 on bad args */
int oracle_features(const float *A, int64_t lda, int64_t N,
                    const float *B, int64_t ldb, int64_t Nt,
                    int S, int H, int W, double h, unsigned gs, uint32_t mask,
                    const double *radii, int M, double band,
                    int64_t *cnt, int64_t *lo, int64_t *hi, double *y,
                    int64_t *n_amb, int nthreads) {
    if (!A || !B || !radii || !cnt || N < 0 || Nt < 0 || M < 1 || mask == 0 || (mask >> 6)) return -1;
    or_grid g = {S, H, W, h, gs};
    const int nq = popcount6(mask);
    const size_t nc = (size_t)nq * M;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > N && N > 0) nthreads = (int)N;
    if (N == 0) nthreads = 1;
    feat_job *jobs = (feat_job *)calloc((size_t)nthreads, sizeof(feat_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    int64_t *buf = (int64_t *)calloc((size_t)nthreads * 3 * nc, sizeof(int64_t));
    for (int t = 0; t < nthreads; ++t) {
        feat_job *J = &jobs[t];
        J->A = A; J->lda = lda; J->N = N; J->B = B; J->ldb = ldb; J->Nt = Nt;
        J->g = g; J->mask = mask; J->radii = radii; J->M = M; J->band = band;
        J->row0 = N * t / nthreads; J->row1 = N * (t + 1) / nthreads;
        J->cnt = buf + (size_t)t * 3 * nc; J->lo = J->cnt + nc; J->hi = J->lo + nc;
        pthread_create(&th[t], NULL, feat_worker, J);
    }
    int nonfinite = 0;
    int64_t amb = 0;
    memset(cnt, 0, nc * sizeof(int64_t));
    if (lo) memset(lo, 0, nc * sizeof(int64_t));
    if (hi) memset(hi, 0, nc * sizeof(int64_t));
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        for (size_t c = 0; c < nc; ++c) {
            cnt[c] += jobs[t].cnt[c];
            if (lo) lo[c] += jobs[t].lo[c];
            if (hi) hi[c] += jobs[t].hi[c];
        }
        amb += jobs[t].n_amb;
        nonfinite |= jobs[t].nonfinite;
    }
    /* non-finite check of B as well */
    const size_t K = (size_t)S * H * W;
    for (int64_t j = 0; j < Nt; ++j)
        for (size_t e = 0; e < K; ++e) if (!isfinite(B[j * ldb + e])) nonfinite = 1;
    if (y) {
        const double NN = (double)N * (double)Nt;
        for (size_t c = 0; c < nc; ++c) y[c] = (NN > 0) ? (double)cnt[c] / NN : 0.0;
    }
    if (n_amb) *n_amb = amb;
    free(buf); free(th); free(jobs);
    return nonfinite ? OR_NONFINITE : OR_OK;
}

/* All pairwise distances for the selected measures, d[q][i][j] (tiny inputs only). */
int oracle_distance_matrix(const float *A, int64_t lda, int64_t N,
                           const float *B, int64_t ldb, int64_t Nt,
                           int S, int H, int W, double h, unsigned gs, uint32_t mask, double *D) {
    or_grid g = {S, H, W, h, gs};
    int slot[N_MEAS_MAX], nq = 0;
    for (int i = 0; i < N_MEAS_MAX; ++i)
        if ((mask >> i) & 1u) slot[nq++] = i;
    for (int64_t i = 0; i < N; ++i)
        for (int64_t j = 0; j < Nt; ++j) {
            double d[6];
            oracle_pair_distances(A + i * lda, B + j * ldb, &g, d);
            for (int q = 0; q < nq; ++q) D[((size_t)q * N + i) * Nt + j] = d[slot[q]];
        }
    return 0;
}

/* ---------------------------------------------------------------------------
 * mu, Sigma of n realisations y_p in R^D (Alg. 1 step 3 PAPER.md:131):
 * two-pass, mu = (1/n) sum_p y_p, Sigma = 1/(n-1) sum_p (y_p - mu)(y_p - mu)^T [R7].
 * ------------------------------------------------------------------------- */
int oracle_stats(const double *Y, int n, int D, double *mu, double *Sigma) {
    if (n < 2 || D < 1) return -1;
    for (int a = 0; a < D; ++a) {
        double s = 0;
        for (int p = 0; p < n; ++p) s += Y[(size_t)p * D + a];
        mu[a] = s / n;
    }
    for (int a = 0; a < D; ++a)
        for (int b = 0; b < D; ++b) {
            double s = 0;
            for (int p = 0; p < n; ++p)
                s += (Y[(size_t)p * D + a] - mu[a]) * (Y[(size_t)p * D + b] - mu[b]);
            Sigma[(size_t)a * D + b] = s / (n - 1);
        }
    return 0;
}

/* ---------------------------------------------------------------------------
 * Gaussian log-likelihood (Eq. (4), Eq. (12)) [R8]:
 *   Sigma + ridge*I = L L^T (Cholesky, no pivoting; a pivot <= 0 -> NOTPD)
 *   z = L^{-1}(y - mu);  quad = z^T z  (= the paper's f);
 *   logdet = 2 sum ln L_ii;  loglik = -quad/2 - logdet/2 - (D/2) ln(2 pi).
 * out = {quad, logdet, loglik}; returns 0 or OR_NOTPD (out = NaN).
 * ------------------------------------------------------------------------- */
int oracle_loglik(const double *mu, const double *Sigma, const double *y, int D,
                  double ridge, double out[3]) {
    double *L = (double *)calloc((size_t)D * D, sizeof(double));
    double *z = (double *)calloc((size_t)D, sizeof(double));
    int status = OR_OK;
    for (int j = 0; j < D && status == OR_OK; ++j) {
        double s = Sigma[(size_t)j * D + j] + ridge;
        for (int k = 0; k < j; ++k) s -= L[(size_t)j * D + k] * L[(size_t)j * D + k];
        if (!(s > 0.0)) { status = OR_NOTPD; break; }
        double Ljj = sqrt(s);
        L[(size_t)j * D + j] = Ljj;
        for (int i = j + 1; i < D; ++i) {
            double t = Sigma[(size_t)i * D + j];
            for (int k = 0; k < j; ++k) t -= L[(size_t)i * D + k] * L[(size_t)j * D + k];
            L[(size_t)i * D + j] = t / Ljj;
        }
    }
    if (status == OR_OK) {
        double quad = 0, logdet = 0;
        for (int i = 0; i < D; ++i) {
            double t = y[i] - mu[i];
            for (int k = 0; k < i; ++k) t -= L[(size_t)i * D + k] * z[k];
            z[i] = t / L[(size_t)i * D + i];
            quad += z[i] * z[i];
            logdet += 2.0 * log(L[(size_t)i * D + i]);
        }
        out[0] = quad;
        out[1] = logdet;
        out[2] = -0.5 * quad - 0.5 * logdet - 0.5 * D * log(2.0 * M_PI);
    } else {
        out[0] = out[1] = out[2] = NAN;
    }
    free(L); free(z);
    return status;
}

/* ---------------------------------------------------------------------------
 * SCIL at one theta, Alg. 3, Eqs. (11)-(13):
 *   subset k = pool rows [k*N, (k+1)*N), N = N_set + N~ (step 2) [R10];
 *   s^{k,1} = its first N_set rows, s^{k,2} = its last N~ rows;
 *   for k,l = 1..n_ens (all n_ens^2 combinations, k = l included):
 *       y^{k,l}_m = C(R_m, s^{k,1}, s^{l,2})  (Eq. (11)), vector index v = k*n_ens + l;
 *   mu_theta, Sigma_theta from the n_ens^2 vectors (step 4);
 *   y~_m = C(R_m, s_data, s^{k0,2})  (Eq. (13)), k0 given by the caller (step 5);
 *   f = (y~ - mu)^T Sigma^{-1} (y~ - mu) (Eq. (12)) -> out = {quad, logdet, loglik}.
 * Y (optional) receives the n_ens^2 + 1 vectors (the last one is y~), each D = nq*M.
 * ------------------------------------------------------------------------- */
int oracle_synth_loglik(const float *pool, int64_t ld, int n_ens, int N_set, int N_tilde,
                        const float *data, int64_t ld_data, int k0,
                        int S, int H, int W, double h, unsigned gs, uint32_t mask,
                        const double *radii, int M, double ridge, double out[3],
                        double *Y, int nthreads) {
    const int nq = popcount6(mask);
    const int D = nq * M;
    const int64_t N = (int64_t)N_set + N_tilde;
    const int nv = n_ens * n_ens;
    double *Yv = (double *)calloc((size_t)(nv + 1) * D, sizeof(double));
    int64_t *cnt = (int64_t *)calloc((size_t)D, sizeof(int64_t));
    int nonfinite = 0;
    for (int k = 0; k < n_ens; ++k)
        for (int l = 0; l < n_ens; ++l) {
            const float *s1 = pool + (int64_t)k * N * ld;
            const float *s2 = pool + ((int64_t)l * N + N_set) * ld;
            int st = oracle_features(s1, ld, N_set, s2, ld, N_tilde, S, H, W, h, gs, mask, radii, M,
                                     0.0, cnt, NULL, NULL, Yv + (size_t)(k * n_ens + l) * D,
                                     NULL, nthreads);
            if (st == OR_NONFINITE) nonfinite = 1;
        }
    {
        const float *s2 = pool + ((int64_t)k0 * N + N_set) * ld;
        int st = oracle_features(data, ld_data, N_set, s2, ld, N_tilde, S, H, W, h, gs, mask, radii, M,
                                 0.0, cnt, NULL, NULL, Yv + (size_t)nv * D, NULL, nthreads);
        if (st == OR_NONFINITE) nonfinite = 1;
    }
    double *mu = (double *)calloc((size_t)D, sizeof(double));
    double *Sig = (double *)calloc((size_t)D * D, sizeof(double));
    oracle_stats(Yv, nv, D, mu, Sig);
    int status = oracle_loglik(mu, Sig, Yv + (size_t)nv * D, D, ridge, out);
    if (Y) memcpy(Y, Yv, sizeof(double) * (size_t)(nv + 1) * D);
    free(mu); free(Sig); free(Yv); free(cnt);
    if (nonfinite) return OR_NONFINITE;
    return status;
}

/* ---------------------------------------------------------------------------
 * Bootstrap step 2 (Alg. A1 steps 2.1-2.3 PAPER.md:660-672, Alg. A2 steps 2.1-2.4
 * PAPER.md:698-712), written out literally: for replicate k the sets
 *   s^1 = { A[I1[k][i]] : i < n1 },  s^2 = { B[I2[k][j]] : j < n2 }
 * are CONSTRUCTED (copies of the drawn patterns, repetitions included; the draws are
 * the caller's [R14]) and the correlation-integral vector of (s^1, s^2) is computed
 * from their distances exactly as in Eq. (1) (oracle_features).  cnt / lo / hi receive
 * [n_rep][nq*M] (band counts as in oracle_features), y [n_rep][nq*M] (nullable).
 * Returns 0, OR_NONFINITE, or -1 (bad argument / index out of range).
 * ------------------------------------------------------------------------- */
int oracle_resample_features(const float *A, int64_t lda, int64_t N, const float *B, int64_t ldb, int64_t Nt,
                             int S, int H, int W, double h, unsigned gs, uint32_t mask, const double *radii, int M,
                             int n_rep, const int32_t *I1, int64_t n1, const int32_t *I2, int64_t n2,
                             double band, int64_t *cnt, int64_t *lo, int64_t *hi, double *y, int nthreads) {
    const int64_t K = (int64_t)S * H * W;
    const int nq = popcount6(mask);
    const size_t D = (size_t)nq * M;
    if (n_rep < 1 || n1 < 1 || n2 < 1) return -1;
    for (int64_t t = 0; t < (int64_t)n_rep * n1; ++t) if (I1[t] < 0 || I1[t] >= N) return -1;
    for (int64_t t = 0; t < (int64_t)n_rep * n2; ++t) if (I2[t] < 0 || I2[t] >= Nt) return -1;
    float *s1 = (float *)malloc(sizeof(float) * (size_t)(n1 * K));
    float *s2 = (float *)malloc(sizeof(float) * (size_t)(n2 * K));
    int nonfinite = 0;
    for (int k = 0; k < n_rep; ++k) {
        /* step 2.1 (and 2.2): construct the resampled sets */
        for (int64_t i = 0; i < n1; ++i)
            memcpy(s1 + i * K, A + (int64_t)I1[(int64_t)k * n1 + i] * lda, sizeof(float) * (size_t)K);
        for (int64_t j = 0; j < n2; ++j)
            memcpy(s2 + j * K, B + (int64_t)I2[(int64_t)k * n2 + j] * ldb, sizeof(float) * (size_t)K);
        /* distances between all patterns of s^1 and s^2 -> y^k via Eq. (1) */
        int st = oracle_features(s1, K, n1, s2, K, n2, S, H, W, h, gs, mask, radii, M, band,
                                 cnt + (size_t)k * D, lo ? lo + (size_t)k * D : NULL,
                                 hi ? hi + (size_t)k * D : NULL, y ? y + (size_t)k * D : NULL, NULL, nthreads);
        if (st == OR_NONFINITE) nonfinite = 1;
        if (st < 0) { free(s1); free(s2); return -1; }
    }
    free(s1); free(s2);
    return nonfinite ? OR_NONFINITE : OR_OK;
}

/* ---------------------------------------------------------------------------
 * SCIL with bootstrapping at one theta, Alg. A2:
 *   step 1: the pool s_syn (N_syn patterns) is given;
 *   step 2: for k < n_rep: s^1 = pool[I1[k]] (N_set draws), s^2 = pool[I2[k]] (N~ = N_syn - N_set
 *           draws), y^k = C(R, s^1, s^2)   (oracle_resample_features);
 *   step 3: mu_theta, Sigma_theta of the n_rep vectors (oracle_stats);
 *   step 4: s^2_theta = pool[J] (N~ patterns);
 *   step 5: y~ = C(R, s_data, s^2_theta) (Eq. (13) with s^2_theta), f from Eq. (12) ->
 *           out = {quad, logdet, loglik} (oracle_loglik).
 * Y (optional) receives the n_rep + 1 vectors (y~ last).
 * ------------------------------------------------------------------------- */
int oracle_synth_boot(const float *pool, int64_t ld, int N_syn, const float *data, int64_t ld_data, int N_set,
                      int n_rep, const int32_t *I1, const int32_t *I2, const int32_t *J,
                      int S, int H, int W, double h, unsigned gs, uint32_t mask, const double *radii, int M,
                      double ridge, double out[3], double *Y, int nthreads) {
    const int nq = popcount6(mask);
    const int D = nq * M;
    const int Nt = N_syn - N_set;
    double *Yv = (double *)calloc((size_t)(n_rep + 1) * D, sizeof(double));
    int64_t *cnt = (int64_t *)calloc((size_t)n_rep * D, sizeof(int64_t));
    int st = oracle_resample_features(pool, ld, N_syn, pool, ld, N_syn, S, H, W, h, gs, mask, radii, M, n_rep,
                                      I1, N_set, I2, Nt, 0.0, cnt, NULL, NULL, Yv, nthreads);
    if (st < 0) { free(Yv); free(cnt); return -1; }
    int nonfinite = st == OR_NONFINITE;
    /* steps 4-5: y~ from s_data and the subset pool[J] */
    int32_t *I0 = (int32_t *)malloc(sizeof(int32_t) * (size_t)N_set);
    for (int i = 0; i < N_set; ++i) I0[i] = i;                 /* s_data itself, no resampling */
    st = oracle_resample_features(data, ld_data, N_set, pool, ld, N_syn, S, H, W, h, gs, mask, radii, M, 1,
                                  I0, N_set, J, Nt, 0.0, cnt, NULL, NULL, Yv + (size_t)n_rep * D, nthreads);
    free(I0);
    if (st < 0) { free(Yv); free(cnt); return -1; }
    if (st == OR_NONFINITE) nonfinite = 1;
    double *mu = (double *)calloc((size_t)D, sizeof(double));
    double *Sig = (double *)calloc((size_t)D * D, sizeof(double));
    oracle_stats(Yv, n_rep, D, mu, Sig);
    int status = oracle_loglik(mu, Sig, Yv + (size_t)n_rep * D, D, ridge, out);
    if (Y) memcpy(Y, Yv, sizeof(double) * (size_t)(n_rep + 1) * D);
    free(mu); free(Sig); free(Yv); free(cnt);
    if (nonfinite) return OR_NONFINITE;
    return status;
}
