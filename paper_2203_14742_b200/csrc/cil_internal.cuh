// cil_internal.cuh — shared device/host definitions of libcil (CUDA path only).
// Nothing here is shared with oracle/: the oracle is an independent program.
#pragma once
#include <atomic>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/cil.h"

namespace cil {

// One-time, per-device setting of a kernel's maximum dynamic shared memory (thread-safe;
// a bit per device, so a process driving several GPUs sets it on each).
struct SmemAttrOnce {
    std::atomic<unsigned long long> mask{0ull};
    template <typename F>
    cudaError_t ensure(F* fn, int bytes) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        const unsigned long long bit = 1ull << (dev & 63);
        if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_release);
        return e;
    }
};


// Bounds-checked builds (-DCIL_BOUNDS_CHECK, tools/bounds_check.sh; compute-sanitizer is closed on
// this pool): CIL_CHECK counts index violations of the engines' computed global accesses in a
// per-translation-unit device counter (no trap, so a violation cannot take the GPU down);
// cil_diag_bounds_violations() sums the counters.  Compiled out otherwise.
#ifdef CIL_BOUNDS_CHECK
static __device__ unsigned int cil_oob_count;
#define CIL_CHECK(c)                                   \
    do {                                               \
        if (!(c)) atomicAdd(&cil_oob_count, 1u);       \
    } while (0)
#define CIL_OOB_READER(fn)                                                               \
    unsigned int fn() {                                                                  \
        unsigned int v = 0;                                                              \
        return cudaMemcpyFromSymbol(&v, cil_oob_count, sizeof(v)) == cudaSuccess ? v : ~0u; \
    }
#else
#define CIL_CHECK(c) \
    do {             \
    } while (0)
#define CIL_OOB_READER(fn) \
    unsigned int fn() { return 0u; }
#endif
unsigned int oob_gram3();
unsigned int oob_recheck();
unsigned int oob_simt();
unsigned int oob_max16();

constexpr int kMaxM = 64;        // radii per measure
constexpr int kMaxMeas = 6;
constexpr int kMaxD = 192;       // n_meas * M for loglik (packed Cholesky factor in smem)
constexpr int kSimtBK = 32;      // SIMT k-chunk (floats); region padding unit
constexpr int kMax16BK = 64;     // max16.cu k-chunk (int16 elements); its region padding unit
constexpr int kG3MaxSeg = 24;     // INT8 Gram: K segments (exact int32 chunks of <= 65536 per phase) per launch
constexpr int kTcBK = 128;       // K padding of the tensor-core operands (128 int8 = one 128-B row)

// Row sources: how panel row r of item p maps to a pattern in caller memory.
//  MODE_PLAIN : base + p*stride + r*ld
//  MODE_SYN_ROW: r <  n_ens*N_set : pool + p*stride + (k*N + i)*ld,  k = r / N_set, i = r % N_set
//                r >= n_ens*N_set : data + (r - n_ens*N_set)*ld_data   (s_data, Eq. (13))
//  MODE_SYN_COL: pool + p*stride + (l*N + N_set + j)*ld,  l = r / N_tilde, j = r % N_tilde
//  MODE_INDEXED: base + p*stride + idx[p*idx_stride + r]*ld  (an index outside [0, idx_range)
//                reads row 0; k_check_index flags the item CIL_ITEM_BADINDEX)
enum RowMode : int { MODE_PLAIN = 0, MODE_SYN_ROW = 1, MODE_SYN_COL = 2, MODE_INDEXED = 3 };

struct RowSrc {
    const float* base;
    int64_t stride;   // per item (floats)
    int64_t ld;       // per row (floats)
    int64_t rows;     // rows per item in the panel
    int mode;
    // synth parameters
    int n_ens, N_set, N_tilde;
    const float* data;
    int64_t ld_data;
    // indexed mode
    const int32_t* idx;
    int64_t idx_stride, idx_range;
};

__host__ __device__ inline const float* row_ptr(const RowSrc& s, int64_t p, int64_t r) {
    if (s.mode == MODE_PLAIN) return s.base + p * s.stride + r * s.ld;
    if (s.mode == MODE_INDEXED) {
        int64_t i = s.idx[p * s.idx_stride + r];
        if (i < 0 || i >= s.idx_range) i = 0;
        return s.base + p * s.stride + i * s.ld;
    }
    const int64_t N = (int64_t)s.N_set + s.N_tilde;
    if (s.mode == MODE_SYN_ROW) {
        const int64_t nr = (int64_t)s.n_ens * s.N_set;
        if (r >= nr) return s.data + (r - nr) * s.ld_data;
        const int64_t k = r / s.N_set, i = r % s.N_set;
        return s.base + p * s.stride + (k * N + i) * s.ld;
    }
    const int64_t l = r / s.N_tilde, j = r % s.N_tilde;
    return s.base + p * s.stride + (l * N + s.N_set + j) * s.ld;
}

// Geometry of the augmented SIMT operand: [value | D_x | D_y] regions, each
// zero-padded to a multiple of kSimtBK floats.
struct AugGeom {
    int S, H, W;
    int64_t K;          // S*H*W
    int64_t Kx, Ky;     // S*H*(W-1), S*(H-1)*W
    int64_t off[4];     // region starts (padded); off[3] = total row length
    int nreg;           // regions materialised (1 = value only, 2 = +D_x, 3 = +D_y)
    uint32_t gs;        // species with derivative terms (bit s; 0 = all): others get 0 derivatives
};

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// n / d (and n % d) for n < 2^31, d >= 1 by a multiply-high: m = floor((2^32 - 1) / d) leaves the
// quotient short by at most 1, fixed by one compare (checked on the host for d < 5000 and random n)
struct FastDiv {
    uint32_t d, m;
    __host__ __device__ explicit FastDiv(uint32_t d_) : d(d_), m(0xffffffffu / d_) {}
    __device__ __forceinline__ uint32_t div(uint32_t n, uint32_t& r) const {
        uint32_t q = __umulhi(n, m);
        r = n - q * d;
        if (r >= d) { ++q; r -= d; }
        return q;
    }
};

inline AugGeom make_aug_geom(int S, int H, int W, int nreg, uint32_t gs = 0, int64_t pad = kSimtBK) {
    AugGeom a{};
    a.S = S; a.H = H; a.W = W;
    a.gs = gs;
    a.K = (int64_t)S * H * W;
    a.Kx = (W > 1) ? (int64_t)S * H * (W - 1) : 0;
    a.Ky = (H > 1) ? (int64_t)S * (H - 1) * W : 0;
    if (nreg >= 3 && a.Ky == 0) nreg = 2;
    a.nreg = nreg;
    a.off[0] = 0;
    a.off[1] = round_up(a.K, pad);
    a.off[2] = a.off[1] + (nreg >= 2 ? round_up(a.Kx, pad) : 0);
    a.off[3] = a.off[2] + (nreg >= 3 ? round_up(a.Ky, pad) : 0);
    return a;
}

// Everything the engines need to bin one measure slot.
struct BinParams {
    int nq;                 // measures selected
    int M;
    int slot[kMaxMeas];     // measure id (0..5) of slot q
    double h;               // grid spacing
    double w;               // quadrature weight h^dim
};

// Segment layout of the count histogram hist[item][rs][cs][q][M+1] (uint64).
struct SegParams {
    int64_t row_seg, col_seg;   // rows (cols) per segment
    int n_rs, n_cs;             // segments per item
};

__host__ __device__ inline int64_t hist_index(const SegParams& sp, int nq, int M, int64_t p,
                                              int64_t rs, int64_t cs, int q, int b) {
    return ((((p * sp.n_rs + rs) * sp.n_cs + cs) * nq + q) * (M + 1)) + b;
}

// Launch bookkeeping (per host thread).
void note_launch(int n = 1);

// Kernel classes for the optional event timing (cil_prof_*).
enum KClass : int { K_PREP = 0, K_PACK = 1, K_GRAM_TC = 2, K_SIMT = 3, K_RECHECK = 4, K_TAIL = 5, K_RESAMPLE = 6,
                    K_NCLASS = 7 };
// RAII: when profiling is enabled on this thread, brackets the enclosed launch with
// CUDA events recorded on the launching stream.
struct ProfScope {
    int cls;
    cudaStream_t st;
    void* ev0;
    ProfScope(int c, cudaStream_t s);
    ~ProfScope();
};

}  // namespace cil

// ---- launchers implemented in the .cu files ----
namespace cil {

// pack.cu
cudaError_t launch_fill_f64(double* p, int n, double v, cudaStream_t st);
cudaError_t launch_prep(int P, int nq, int M, const double* radii, int64_t radii_stride,
                        const BinParams& bp, double* thr, float* thr2_l2, int32_t* status,
                        uint64_t* hist, int64_t hist_elems, uint32_t* recheck_ctr, cudaStream_t st,
                        bool keep_status = false);
cudaError_t launch_pack_aug(int P, const RowSrc& src, int64_t rows, const AugGeom& g,
                            float* out, float* rowstat, int32_t* status, cudaStream_t st);
cudaError_t launch_center(int P, const RowSrc& colsrc, int64_t nrows_center, int64_t K, int64_t Kp,
                          float* center, cudaStream_t st);
cudaError_t launch_pack_tc(int P, const RowSrc& src, int64_t rows, int64_t K, int64_t Kp,
                           const float* center, int split, void* hi, void* lo, float* nrm, float* q4,
                           int32_t* status, cudaStream_t st);


// simt_tile.cu
struct SimtArgs {
    const float* Aaug; const float* Baug;    // [P][rowsA][Kaug], [P][rowsB][Kaug]
    int64_t rowsA, rowsB, Kaug;
    AugGeom g;
    BinParams bp;
    SegParams sp;
    const double* thr;                        // [P or 1][nq][M]
    int64_t thr_stride;
    uint64_t* hist;
    const int32_t* status;                    // skip items flagged BADRADII
    int P;
    bool do_max, do_sum;
    uint32_t qmask;                           // slots binned by this engine
    uint8_t* binout;                          // non-null: bins[p][q][i][j] instead of counts
    unsigned long long* range;                // non-null: [P][nq][2] min (d > 0) / max of d as FP64 bits
    bool tri;                                 // skip tiles without a block k < l (Alg. 1 training)
    bool sym;                                 // bin matrix of a panel against itself: tiles with
                                              // i > j only are skipped, computed (i, j) also written at (j, i)
    int hist_cap;                             // shared histogram entries (set by the launcher)
    const float* statA; const float* statB;   // [P][rows][4] per-row derivative stats (k_pack_aug)
    uint4* list; uint32_t* ctr; uint32_t cap; // re-check list: (p, i, j, b_lo | measure id << 8)
};
cudaError_t launch_simt(const SimtArgs& a, cudaStream_t st);

// max16.cu — the max family on 15-bit fixed-point operands (integer pipes), rigorous interval + re-check
struct Max16Args {
    const int16_t* A; const int16_t* B;       // [P][rowsA][Kaug], [P][rowsB][Kaug] (B negated)
    int64_t rowsA, rowsB, Kaug;
    AugGeom g;                                // regions padded to kMax16BK elements
    const unsigned* maxbits;                  // [P][3][2] per-item range of each region (max16.cu)
    BinParams bp;
    SegParams sp;
    const double* thr;                        // [P][nq][M]
    int64_t thr_stride;
    uint64_t* hist;
    const int32_t* status;
    int P;
    uint32_t qmask;                           // slots binned by this engine (max family only)
    uint8_t* binout;
    bool tri, sym;
    int hist_cap;
    uint4* list; uint32_t* ctr; uint32_t cap;
    uint32_t one;                             // 1 (set by the launcher; keeps the adds on the FMA pipe)
    uint16_t* dmax;                           // [P][nreg][rowsA][rowsB] per-pair region maxima (workspace)
    int64_t dmax_elems;                       // its capacity (bounds-checked builds)
};
cudaError_t launch_pack16(int P, const RowSrc& asrc, int64_t rowsA, const RowSrc& bsrc, int64_t rowsB,
                          const AugGeom& g, unsigned* maxbits, int16_t* outA, int16_t* outB, int32_t* status,
                          cudaStream_t st);
cudaError_t launch_max16(const Max16Args& a, cudaStream_t st);

// gram_tc.cu
struct TcArgs {
    const void* hi; const void* lo;     // stacked [P*rowsA + P*rowsB][Kp] (A panels then B panels)
    const float* nrm; const float* q4;  // stacked like hi
    int64_t rowsA, rowsB, Kp, K;
    int P;
    int split;                          // 1 = 3xBF16, 2 = 3xTF32
    const float* thr2;                  // [P or 1][M] L2 thresholds R^2/w (FP32)
    int64_t thr_stride;
    int M;
    int q_l2;                           // slot of L2 in the hist
    int nq;
    SegParams sp;
    uint64_t* hist;
    uint4* recheck; uint32_t* recheck_ctr; uint32_t recheck_cap;
    const int32_t* status;
    float guard_k1, guard_rel;
    float* diag;                        // diagnostics only (see cil_diag_gram)
    int cta_group;                      // 2 (default): CTA-pair 256x256 tiles; 1: single-CTA 128x256
    int chunk_kb;                       // k-blocks per TMEM partial accumulation (precision control)
    int p0, np;                         // items covered by this launch (np = 0: all from p0)
    int sm_budget;                      // SMs the persistent grid may occupy (0 = all)
};
cudaError_t launch_gram_tc(const TcArgs& a, cudaStream_t st);

// rowdot.cu (bootstrap replicate counts as an integer GEMM, Alg. A1 / A2)
struct RowdotArgs {
    const int8_t* ops;                   // stacked operand rows: P*rowsA multiplicity rows M1, then P*rowsB rows E
    int64_t rowsA, rowsB, Kp;            // rowsB = rd_m * rd_nt (b-major E rows)
    int P;
    const uint16_t* m2;                  // [P][rowsA][rd_nt] column multiplicities
    int64_t rd_nt;
    int rd_m;
    unsigned long long* out;             // [P][rowsA][rd_m] counts (accumulated atomically)
};
cudaError_t launch_rowdot(const RowdotArgs& a, cudaStream_t st);

// gram3.cu (three-digit INT8 engine, the default L2 / L2-family engine; worst-case error bound)
struct G3Args {
    const int8_t* planes;                // [3][rows_tot][Kp] digits h, m, l (A panels then B panels)
    int64_t rows_tot, Kp;
    const float* meta;                   // [rows_tot][nph][8]: n, sigma, r, alpha, beta
    int64_t rowsA, rowsB, a_off, b_off;  // A rows at a_off + p rowsA, B rows at b_off + p rowsB
    int P, p0, np;
    int nph;                             // 1 (L2) or 3 (value, D_x, D_y blocks: L2, W12, W12SUM)
    int64_t ph_beg[3], ph_end[3];        // K byte ranges of the phases (multiples of 64, contiguous)
    const float* thr;                    // [P][8][M] (k_prep)
    int64_t thr_stride;
    int M, nq, q_l2;
    int q_k[3];                          // three-phase: slots of L2, W12, W12SUM (-1: absent)
    SegParams sp;
    uint64_t* hist;
    uint4* list; uint32_t* ctr; uint32_t cap;
    float ih_rd, ih_ru, ih2_rd, ih2_ru;  // 1/h and 1/h^2 rounded down / up
    float* part;                         // three-phase partials [2][P rowsA rowsB] float2
    uint8_t* binout;                     // non-null: bins [p][q][i][j] (or [p][q][j][i] with bin_t)
    bool bin_t;
    int skip;                            // 0 all tiles; 1 symmetric bin matrix; 2 Alg. 1 blocks k < l
    int tn_force;                        // 64: narrow B panel (<= 64 rows)
    float* diag;                         // diagnostics: (lo, hi) per pair of item 0, no binning
    int64_t hist_elems;                  // histogram size (bounds-checked builds)
};
cudaError_t launch_gram3(const G3Args& a, cudaStream_t st);
cudaError_t launch_pack3(int P, const RowSrc& src, int64_t rows, int64_t K, int64_t Kp, const float* center,
                         int8_t* planes, int64_t plane_stride, int64_t row0, float* meta, int32_t* status,
                         cudaStream_t st);
cudaError_t launch_pack3_aug(int P, const RowSrc& src, int64_t rows, const AugGeom& g, const int64_t* kp,
                             const float* center, int64_t Kc, int8_t* planes, int64_t plane_stride, int64_t row0,
                             float* meta, int32_t* status, cudaStream_t st);
bool gram_tc_supported();

// recheck.cu
struct RecheckArgs {
    RowSrc asrc, bsrc;
    int64_t K;
    const double* thr;   // FP64 radii: slot q of item p at thr[p*thr_stride + q*M + m]
    int64_t thr_stride;
    double w, h;         // quadrature weight h^dim, grid spacing
    int M, nq;
    int qslot[6];        // histogram / bin slot of measure id k (bit order), -1 if not requested
    uint32_t kinds;      // measure ids requested (bit k)
    SegParams sp;
    uint64_t* hist;
    const uint4* list; const uint32_t* ctr; uint32_t cap;   // entries (p, i, j, b_lo | kind << 8)
    int32_t* status;
    int P;
    uint8_t* binout;     // non-null: write the exact bin to bins[p][q][i][j] instead of moving counts
    bool mirror;         // symmetric bin matrix: also write [j][i]
    bool transpose;      // write bins[p][q][j][i] only (the INT8 engine's transposed narrow output)
    int64_t rowsA, rowsB;
    int S, H, W;
    uint32_t gs;
    int64_t hist_elems;  // bounds-checked builds
    uint32_t* rk;        // [P*rowsA + 1] per-A-row bucket counts -> offsets (row-bucketed pass)
    uint4* rk_list;      // [cap] the list sorted by (p, i)
    uint32_t sort_min;   // lists of >= sort_min entries take the row-bucketed pass
};
cudaError_t launch_recheck(const RecheckArgs& a, int64_t hist_elems, cudaStream_t st);

// stats.cu — chi^2 Gaussianity diagnostic (interior bin edges by value: no host-to-device copy)
constexpr int kMaxChi2Bins = 64;
struct Chi2Edges {
    int nb;                          // bins
    double e[kMaxChi2Bins - 1];      // interior edges, increasing
};
cudaError_t launch_chi2_pearson(int64_t n, const double* d2, const Chi2Edges& ed, double* out, cudaStream_t st);

// stats.cu
cudaError_t launch_finalize(int P, int nq, int M, const SegParams& sp, const uint64_t* hist,
                            uint64_t* counts, double* y, int64_t pairs_per_seg_rows,
                            int64_t pairs_per_seg_cols, const int32_t* status_in,
                            int32_t* status_out, cudaStream_t st);
cudaError_t launch_finalize_y(int P, int nq, int M, const SegParams& sp, const uint64_t* hist, double* y,
                              int64_t y_stride, double npairs, cudaStream_t st);
cudaError_t launch_stats(int P, const double* Y, int n, int D, double* mu, double* Sigma,
                         cudaStream_t st);
cudaError_t launch_normalize(int64_t n, const uint64_t* counts, double npairs, double* y, cudaStream_t st);

// resample.cu (bootstrap estimators, Alg. A1 / A2)
cudaError_t launch_check_index(int P, const int32_t* idx, int64_t per_item, int64_t range, int32_t* status,
                               cudaStream_t st);
cudaError_t launch_resample(int P, const uint8_t* bins, int64_t N, int64_t Nt, int nq, int M, int n_rep,
                            const int32_t* I1, int64_t n1, const int32_t* I2, int64_t n2, uint64_t* counts,
                            double* y, int64_t y_item_stride, int32_t* status, cudaStream_t st);
cudaError_t launch_minmax(int64_t n, const float* X, int64_t ldx, float* Y, int64_t ldy, int S, int64_t HW,
                          cudaStream_t st);
cudaError_t launch_range_init(int P, int nq, unsigned long long* range, cudaStream_t st);
cudaError_t launch_radii(int P, int nq, int M, const unsigned long long* range, int law, double margin, double* radii,
                         int32_t* status, cudaStream_t st);
cudaError_t launch_build_pairs(int P, int n_ens, int nq, int M, const SegParams& sp, const uint64_t* hist,
                               int64_t N, double* Y, cudaStream_t st);
cudaError_t launch_rd_mult(int P, int64_t N, int64_t Kp, int64_t Ntp, int n_rep, const int32_t* I1, int64_t n1,
                           const int32_t* I2, int64_t n2, int8_t* M1, uint16_t* M2, int32_t* status, cudaStream_t st);
cudaError_t launch_rd_build_E(int P, const uint8_t* bins, int64_t N, int nq, int q, int M, int64_t Kp, int64_t Ntp,
                              int8_t* E, cudaStream_t st);
cudaError_t launch_rd_final(const unsigned long long* cnt, int P, int n_rep, int M, int nq, int q, double npairs,
                            double* y, int64_t y_item_stride, cudaStream_t st);
cudaError_t launch_boot_tail(int P, int n_rep, int D, double ridge, double* out, int32_t* status, double* Y,
                             double* mu, double* Sigma, cudaStream_t st);
cudaError_t launch_loglik(int P, const double* mu, int64_t mu_stride, const double* Sigma,
                          int64_t Sigma_stride, const double* y, int D, double ridge, double* out,
                          int32_t* status, const int32_t* status_in, cudaStream_t st);
cudaError_t launch_synth_tail(int P, int n_ens, int nq, int M, const SegParams& sp, const uint64_t* hist,
                              int64_t N_set, int64_t N_tilde, const int32_t* k0, double ridge, double* out,
                              int32_t* status, double* Y, double* mu, double* Sigma, cudaStream_t st,
                              bool swapped = false);
}  // namespace cil
