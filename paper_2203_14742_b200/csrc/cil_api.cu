// cil_api.cu — the C ABI (include/cil.h): host validation, workspace layout,
// dispatch of the hot-path kernels on the caller's stream.  No device memory is
// allocated here and nothing synchronises the device.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "cil_internal.cuh"

#include <nvtx3/nvToolsExt.h>

#include <vector>

namespace cil {
static thread_local int32_t t_last_cuda = 0;
// diagnostics (cil_diag_limit_recheck_list): cap the re-check list below its allocated capacity on this
// thread so tests can exercise the exact all-pairs fallback; < 0 = no limit
static thread_local int64_t t_list_limit = -1;
// diagnostics (cil_diag_recheck_sort_min): list length from which the re-check is row-bucketed
static thread_local uint32_t t_sort_min = 8192;   // below: the sort costs more than it saves (C2: 3.3k cases)
static thread_local int32_t t_launches = 0;
// Items per call: grids put items on gridDim.y / .z (<= 65535), the max family's region kernel
// three per item.
constexpr int32_t kMaxItems = 21845;
// Rows per set (or panel): the CUDA-core engines put 32-row A tiles on gridDim.y (<= 65535).
constexpr int64_t kMaxRows = 65535ll * 32;
void note_launch(int n) { t_launches += n; }
// diagnostics (cil_diag_concurrent_engines): run the max family's engine on a side stream, concurrently
// with the tensor-core family (default on)
static thread_local bool t_concurrent = true;

// One library-owned side stream per host thread and device (non-blocking), with its two ordering
// events, for the concurrent engines: per thread, so one thread capturing a CUDA graph never shares a
// side stream with another thread's work (a captured stream must not receive uncaptured work).
// Created on a thread's first call that forks (which, like the kernel attribute setup, should be an
// eager call), destroyed at thread exit.
struct SideStreams {
    cudaStream_t s[64] = {};
    cudaEvent_t fork[64] = {}, join[64] = {};
    ~SideStreams() {
        for (int d = 0; d < 64; ++d) {
            if (s[d]) cudaStreamDestroy(s[d]);
            if (fork[d]) cudaEventDestroy(fork[d]);
            if (join[d]) cudaEventDestroy(join[d]);
        }
    }
};
static thread_local SideStreams t_side;
static int side_setup() {          // the device index with a ready side stream, or -1
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
    if (!t_side.s[dev]) {
        cudaStream_t st = nullptr;
        cudaEvent_t f = nullptr, j = nullptr;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return -1;
        if (cudaEventCreateWithFlags(&f, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&j, cudaEventDisableTiming) != cudaSuccess) {
            cudaStreamDestroy(st);
            if (f) cudaEventDestroy(f);
            return -1;
        }
        t_side.s[dev] = st; t_side.fork[dev] = f; t_side.join[dev] = j;
    }
    return dev;
}

// Fork / join of the side stream around the engines (event-ordered, so it is CUDA-graph capturable:
// the side stream joins the capture through the fork event and leaves it through the join).
struct Fork {
    cudaStream_t main, aux = nullptr;
    int dev = -1;
    bool joined = true;
    Fork(cudaStream_t m, bool on) : main(m) {
        if (!on || (dev = side_setup()) < 0) return;
        aux = t_side.s[dev];
        cudaEventRecord(t_side.fork[dev], main);
        cudaStreamWaitEvent(aux, t_side.fork[dev], 0);
        joined = false;
    }
    cudaStream_t side() const { return aux ? aux : main; }
    // work enqueued on the side stream from now on starts only after the main stream's work so far
    void side_after_main() {
        if (joined) return;
        cudaEventRecord(t_side.fork[dev], main);
        cudaStreamWaitEvent(aux, t_side.fork[dev], 0);
    }
    void join() {
        if (joined) return;
        joined = true;
        cudaEventRecord(t_side.join[dev], aux);
        cudaStreamWaitEvent(main, t_side.join[dev], 0);
    }
    ~Fork() { join(); }
};

// ---- optional per-kernel-class event timing (diagnostics for the roofline) ----
struct ProfRec {
    int cls;
    cudaEvent_t a, b;
};
static thread_local bool t_prof_on = false;
static thread_local std::vector<ProfRec>* t_prof = nullptr;
static thread_local std::vector<cudaEvent_t>* t_evpool = nullptr;

static cudaEvent_t ev_get() {
    if (!t_evpool) t_evpool = new std::vector<cudaEvent_t>();
    if (!t_evpool->empty()) {
        cudaEvent_t e = t_evpool->back();
        t_evpool->pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// NVTX ranges: one per public call (NvtxScope below) and one per kernel class launch (ProfScope),
// visible in Nsight timelines; no-ops when no tool is attached (NVTX v3, header-only)
static const char* const kClassName[K_NCLASS] = {"cil:prep",     "cil:pack", "cil:gram_tc", "cil:simt_tile",
                                                 "cil:recheck",  "cil:tail", "cil:resample"};
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
};

ProfScope::ProfScope(int c, cudaStream_t s) : cls(c), st(s), ev0(nullptr) {
    nvtxRangePushA(kClassName[c]);
    if (!t_prof_on) return;
    cudaEvent_t e = ev_get();
    cudaEventRecord(e, s);
    ev0 = e;
}
ProfScope::~ProfScope() {
    nvtxRangePop();
    if (!ev0) return;
    cudaEvent_t e = ev_get();
    cudaEventRecord(e, st);
    if (!t_prof) t_prof = new std::vector<ProfRec>();
    t_prof->push_back({cls, (cudaEvent_t)ev0, e});
}
}  // namespace cil

using namespace cil;

namespace {

struct Slots {
    int nq = 0;
    int slot[kMaxMeas] = {0};
    int q_l2 = -1;
};

Slots slots_of(uint32_t mask) {
    Slots s;
    for (int i = 0; i < kMaxMeas; ++i)
        if ((mask >> i) & 1u) {
            if (i == 0) s.q_l2 = s.nq;
            s.slot[s.nq++] = i;
        }
    return s;
}

double grid_h(const cil_grid& g) {
    if (g.h > 0) return g.h;
    return g.W >= 2 ? 1.0 / (double)(g.W - 1) : 1.0;
}

// Which engines a request uses.
struct Plan {
    bool tc = false;        // L2 on tensor cores
    int split = 1;          // 1 = 3xBF16, 2 = 3xTF32
    bool aug = false;       // three-phase INT8 engine: L2, W12, W12SUM on tensor cores
    uint32_t simt_mask = 0; // measures on the CUDA-core engine
    bool do_max = false, do_sum = false;
    int nreg = 1;
    bool max16 = false;     // max family alone on the 15-bit fixed-point integer engine (max16.cu)
    bool f32aug = false;    // FP32 augmented operands for k_simt (everything else on the CUDA cores)
};

// The max family goes to max16.cu when it runs without the sum family (the L2 type measures are on
// the tensor cores) and the engine is not the all-FP32 CUDA-core engine (SIMT, also the exact
// distance-range mode).
void plan_cuda_cores(Plan& pl, cil_engine engine) {
    pl.max16 = pl.do_max && !pl.do_sum && engine != CIL_ENGINE_SIMT;
    pl.f32aug = pl.simt_mask != 0 && !pl.max16;
}

// split: 1 = 3xBF16, 2 = 3xTF32, 3 = three-digit INT8 (gram3.cu).  The INT8 engine takes any K
// (exact int32 accumulation in chunks of 65536) and column segments of >= 21 columns (its
// per-thread byte histograms); otherwise AUTO / TC_I8 run L2 on the CUDA cores, whose bounds are
// rigorous too.  The float split engines are explicit options only.
constexpr int64_t kMinSegI8 = 21;
bool i8_ok(int64_t col_seg, int64_t rowsB) { return col_seg >= rowsB || col_seg >= kMinSegI8; }
// K segments of the INT8 Gram (launch_gram3: each phase in exact int32 chunks of <= 65536 bytes,
// an empty phase counts one): longer rows than kG3MaxSeg segments hold run on the CUDA cores
// (nph = 1: K <= 24 x 65536; three phases: about 8 x 65536 per block)
int i8_segments(const cil_grid& g, bool aug) {
    auto ch = [](int64_t n) { return n > 0 ? (int)((n + 65535) / 65536) : 1; };
    const int64_t K = (int64_t)g.S * g.H * g.W, Kp = round_up(K, kTcBK);
    if (!aug) return ch(Kp);
    const int64_t Ky = (int64_t)g.S * (g.H - 1) * g.W;
    return ch(Kp) + ch(Kp) + ch(round_up(Ky, kTcBK));
}
// The L2-type family (L2, W12, W12SUM) on the three-phase INT8 engine when the
// request has W12 or W12SUM, the engine is AUTO / TC_I8, and the per-thread histograms fit
// (column segments: >= 21 columns and M <= 16).
bool aug_ok(uint32_t mask, cil_engine engine, const cil_grid& g, int64_t col_seg, int64_t rowsB, int M) {
    if (!(mask & (CIL_W12 | CIL_W12SUM))) return false;
    if (engine != CIL_ENGINE_AUTO && engine != CIL_ENGINE_TC_I8) return false;
    if (g.W < 2) return false;
    if (i8_segments(g, true) > kG3MaxSeg) return false;
    const bool seg = col_seg < rowsB;
    if (seg && (col_seg < kMinSegI8 || M > 16)) return false;
    return M <= 64;
}
Plan make_plan(uint32_t mask, cil_engine engine, const cil_grid& g, int64_t col_seg = 1ll << 40,
               int64_t rowsB = 0, int M = 1, bool allow_aug = true) {
    Plan pl;
    if (allow_aug && aug_ok(mask, engine, g, col_seg, rowsB, M)) {
        pl.tc = true;
        pl.aug = true;
        pl.split = 3;
        pl.simt_mask = mask & ~(uint32_t)(CIL_L2 | CIL_W12 | CIL_W12SUM);
        pl.do_max = pl.simt_mask & (CIL_LINF | CIL_W1INF | CIL_W1INFSUM);
        pl.do_sum = false;
        pl.nreg = (pl.simt_mask & (CIL_W1INF | CIL_W1INFSUM)) ? (g.H > 1 ? 3 : 2) : 1;
        plan_cuda_cores(pl, engine);
        return pl;
    }
    pl.split = (engine == CIL_ENGINE_TC_3XTF32) ? 2 : (engine == CIL_ENGINE_TC_3XBF16) ? 1 : 3;
    pl.tc = (mask & CIL_L2) && engine != CIL_ENGINE_SIMT &&
            (pl.split != 3 || (i8_ok(col_seg, rowsB) && i8_segments(g, false) <= kG3MaxSeg));
    pl.simt_mask = pl.tc ? (mask & ~(uint32_t)CIL_L2) : mask;
    pl.do_max = pl.simt_mask & (CIL_LINF | CIL_W1INF | CIL_W1INFSUM);
    pl.do_sum = pl.simt_mask & (CIL_L2 | CIL_W12SUM | CIL_W12);
    const bool grad = pl.simt_mask & (CIL_W12SUM | CIL_W12 | CIL_W1INF | CIL_W1INFSUM);
    pl.nreg = grad ? (g.H > 1 ? 3 : 2) : 1;
    plan_cuda_cores(pl, engine);
    return pl;
}

// Bin-matrix mode (bootstrap): L2 (and W12 / W12SUM) on the INT8 engine, the rest on the CUDA cores;
// the float split engines have no bin-matrix epilogue.
bool plan_bins(uint32_t mask, cil_engine engine, const cil_grid& g, Plan* out) {
    if (engine == CIL_ENGINE_TC_3XBF16 || engine == CIL_ENGINE_TC_3XTF32) return false;
    const cil_engine e = engine == CIL_ENGINE_SIMT ? CIL_ENGINE_SIMT : CIL_ENGINE_TC_I8;
    *out = make_plan(mask, e, g, 1ll << 40, 0, 1, /*allow_aug=*/true);
    return true;
}

// Union of two plans (one workspace serving two engine runs in sequence).
Plan plan_union(const Plan& a, const Plan& b) {
    Plan u = a;
    u.tc = a.tc || b.tc;
    u.aug = a.aug || b.aug;
    // operand element size: split 2 (tf32) 4 B > split 1 (bf16) 2 B > split 3 (int8 digits)
    auto esz = [](const Plan& p) { return !p.tc ? 0 : p.split == 2 ? 4 : p.split == 3 ? 1 : 2; };
    u.split = esz(a) >= esz(b) ? a.split : b.split;
    u.simt_mask = a.simt_mask | b.simt_mask;
    u.do_max = a.do_max || b.do_max;
    u.do_sum = a.do_sum || b.do_sum;
    u.nreg = a.nreg > b.nreg ? a.nreg : b.nreg;
    u.max16 = a.max16 || b.max16;
    u.f32aug = a.f32aug || b.f32aug;
    return u;
}

// Workspace carve-up (identical in the size query and in the call).
struct Layout {
    size_t off_thr, off_thr2, off_hist, off_ctr, off_list, off_center, off_hi, off_lo, off_nrm, off_q4,
        off_aug, off_rowstat, off_aug16, off_max16, off_dmax16, off_rk, off_rk_list, off_Y, off_mu, off_sig, off_part, total;
    int64_t hist_elems = 0;
    uint32_t list_cap = 0;
    int64_t Kp = 0;
    int64_t kp[4] = {0, 0, 0, 0};   // three-phase engine: block starts of the augmented planes, kp[3] = row length
    int64_t rows_cap = 0;           // rows of the operand planes (A panels then B panels)
    int64_t Krow = 0;               // bytes per plane row (INT8 engine)
    int nph = 1;
    AugGeom geom{};
    AugGeom geom16{};               // max16.cu operands (regions padded to kMax16BK)
    int64_t dmax_rows_product = 0;  // P * rowsA * rowsB of the per-pair region maxima
};

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

Layout make_layout(int P, int64_t rowsA, int64_t rowsB, const cil_grid& g, int nq, int M, const Plan& pl,
                   const SegParams& sp, int64_t nY) {
    Layout L{};
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = al(o + bytes); return r; };
    const int64_t K = (int64_t)g.S * g.H * g.W;
    L.off_thr = take(sizeof(double) * (size_t)P * nq * M);
    L.off_thr2 = take(sizeof(float) * (size_t)P * 8 * M);      // [P][8][M] tensor-core thresholds (k_prep)
    L.hist_elems = (int64_t)P * sp.n_rs * sp.n_cs * nq * (M + 1);
    L.off_hist = take(sizeof(uint64_t) * (size_t)L.hist_elems);
    L.off_ctr = take(sizeof(uint32_t) * 2);
    const int64_t rows = (int64_t)P * (rowsA + rowsB);
    L.rows_cap = rows;
    if (pl.tc || pl.simt_mask) {
        // re-check list (16 B per entry): 1/128 of the (pair, measure) cases + 256 k; beyond that the
        // exact fallback of recheck.cu runs instead (counts stay exact)
        const double cases = (double)P * rowsA * rowsB * nq;
        L.list_cap = (uint32_t)fmin(fmin(cases, cases / 128.0 + 262144.0), 1.0e9);
        L.off_list = take(16 * (size_t)L.list_cap);
        L.off_rk = take(sizeof(uint32_t) * ((size_t)rows + 1));     // row buckets of the re-check
        L.off_rk_list = take(16 * (size_t)L.list_cap);
    }
    if (pl.tc) {
        L.Kp = round_up(K, kTcBK);
        L.off_center = take(sizeof(float) * (size_t)P * L.Kp);
        if (pl.split == 3) {
            L.Krow = L.Kp;
            if (pl.aug) {
                const AugGeom ag = make_aug_geom(g.S, g.H, g.W, 3);
                L.kp[0] = 0;
                L.kp[1] = L.Kp;
                L.kp[2] = L.kp[1] + round_up(ag.K, kTcBK);          // D_x rows padded to W (pack3_aug)
                L.kp[3] = L.kp[2] + round_up(ag.Ky, kTcBK);
                L.Krow = L.kp[3];
                L.nph = 3;
            }
            L.off_hi = take((size_t)3 * rows * L.Krow);                       // digit planes h, m, l
            L.off_nrm = take(sizeof(float) * 8 * (size_t)rows * L.nph);        // per-row metadata
            if (pl.aug) L.off_part = take(sizeof(float) * 4 * (size_t)P * rowsA * rowsB);
        } else {
            const size_t esz = pl.split == 2 ? 4 : 2;
            L.off_hi = take(esz * (size_t)rows * L.Kp);
            L.off_lo = take(esz * (size_t)rows * L.Kp);
            L.off_nrm = take(sizeof(float) * (size_t)rows);
            L.off_q4 = take(sizeof(float) * (size_t)rows);
        }
    }
    if (pl.f32aug) {
        L.geom = make_aug_geom(g.S, g.H, g.W, pl.nreg, g.gs);
        L.off_aug = take(sizeof(float) * (size_t)rows * L.geom.off[3]);
        L.off_rowstat = take(sizeof(float) * 4 * (size_t)rows);
    }
    if (pl.max16) {
        L.geom16 = make_aug_geom(g.S, g.H, g.W, pl.nreg, g.gs, kMax16BK);
        L.off_aug16 = take(sizeof(int16_t) * (size_t)rows * L.geom16.off[3]);
        L.off_max16 = take(sizeof(unsigned) * 8 * (size_t)P);
        L.off_dmax16 = take(sizeof(uint16_t) * 3 * (size_t)P * rowsA * rowsB);
        L.dmax_rows_product = (int64_t)P * rowsA * rowsB;
    }
    if (nY > 0) {
        L.off_Y = take(sizeof(double) * (size_t)nY);
        const int D = nq * M;
        L.off_mu = take(sizeof(double) * (size_t)P * D);
        L.off_sig = take(sizeof(double) * (size_t)P * D * D);
    }
    L.total = o + 256;   // slack for base alignment
    return L;
}

template <class T>
T* at(void* base, size_t off) { return reinterpret_cast<T*>(reinterpret_cast<char*>(base) + off); }

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// the two panels address the same pattern rows (plain mode, same base / strides)
bool same_rows(const RowSrc& a, const RowSrc& b) {
    return a.mode == MODE_PLAIN && b.mode == MODE_PLAIN && a.base == b.base && a.stride == b.stride &&
           a.ld == b.ld && a.rows == b.rows;
}

// shared-memory budget of k_resample: per-thread histograms + the two multiplicity tables
bool resample_fits(int64_t N, int64_t Nt, int M) {
    // histograms + m1 + m2 + the distinct-row list (<= N)
    return 4 * ((int64_t)(M + 1) * 256 + ((N + 3) & ~(int64_t)3) + ((Nt + 15) & ~(int64_t)15) + N) <= 200 * 1024;
}

cil_status fail_cuda(cudaError_t e) {
    t_last_cuda = (int32_t)e;
    return CIL_ECUDA;
}

#define CIL_CU(x)                                   \
    do {                                            \
        cudaError_t _e = (x);                       \
        if (_e != cudaSuccess) return fail_cuda(_e); \
    } while (0)

cil_status check_grid(const cil_grid& g, uint32_t mask) {
    if (g.S < 1 || g.H < 1 || g.W < 1) return CIL_EINVAL;
    if (mask == 0 || (mask & ~CIL_ALL_DISTS)) return CIL_EINVAL;
    if ((mask & (CIL_W12SUM | CIL_W12 | CIL_W1INF | CIL_W1INFSUM)) && g.W < 2) return CIL_EINVAL;
    if (!(g.h == g.h)) return CIL_EINVAL;
    return CIL_OK;
}

cil_status check_sets(int32_t P, const float* A, int64_t strideA, int64_t lda, int64_t N, const float* B,
                             int64_t strideB, int64_t ldb, int64_t Nt, const cil_grid& g) {
    if ((N > 0 && !A) || (Nt > 0 && !B)) return CIL_EINVAL;
    if (strideA < 0 || strideB < 0) return CIL_EINVAL;
    const int64_t K = (int64_t)g.S * g.H * g.W;
    if ((N > 0 && lda < K) || (Nt > 0 && ldb < K)) return CIL_EINVAL;
    if (N > 0 && P > 1 && strideA > 0 && strideA < (N - 1) * lda + K) return CIL_EINVAL;
    if (Nt > 0 && P > 1 && strideB > 0 && strideB < (Nt - 1) * ldb + K) return CIL_EINVAL;
    if (K % 4 || lda % 4 || ldb % 4 || strideA % 4 || strideB % 4) return CIL_EUNSUPPORTED;
    if ((A && !aligned16(A)) || (B && !aligned16(B))) return CIL_EUNSUPPORTED;
    return CIL_OK;
}

// 1/h (or 1/h^2) as the FP32 neighbours below and above the FP64 value
void f32_bracket(double v, float* rd, float* ru) {
    const float f = (float)v;
    *rd = (double)f <= v ? f : nextafterf(f, -INFINITY);
    *ru = (double)f >= v ? f : nextafterf(f, INFINITY);
    *rd = nextafterf(*rd, -INFINITY);       // one more ulp each way for the FP64 rounding of v itself
    *ru = nextafterf(*ru, INFINITY);
}

RecheckArgs recheck_args(const RowSrc& asrc, const RowSrc& bsrc, int64_t K, const cil_grid& g, const Slots& sl, int M,
                         const BinParams& bp, const SegParams& sp, const Layout& L, void* ws, int32_t* status, int P,
                         uint8_t* binout, int64_t rowsA, int64_t rowsB, uint32_t mask) {
    RecheckArgs r{};
    r.asrc = asrc; r.bsrc = bsrc; r.K = K;
    r.thr = at<double>(ws, L.off_thr); r.thr_stride = (int64_t)sl.nq * M;
    r.w = bp.w; r.h = bp.h;
    r.M = M; r.nq = sl.nq;
    for (int k = 0; k < 6; ++k) r.qslot[k] = -1;
    for (int q = 0; q < sl.nq; ++q) r.qslot[sl.slot[q]] = q;
    r.kinds = mask;
    r.sp = sp;
    r.hist = at<uint64_t>(ws, L.off_hist);
    r.list = at<uint4>(ws, L.off_list); r.ctr = at<uint32_t>(ws, L.off_ctr); r.cap = L.list_cap;
    r.status = status; r.P = P;
    r.binout = binout; r.rowsA = rowsA; r.rowsB = rowsB;
    r.mirror = binout != nullptr && same_rows(asrc, bsrc) && rowsA == rowsB;
    r.S = g.S; r.H = g.H; r.W = g.W; r.gs = g.gs;
    r.hist_elems = L.hist_elems;
    r.rk = at<uint32_t>(ws, L.off_rk);
    r.sort_min = t_sort_min;
    r.rk_list = at<uint4>(ws, L.off_rk_list);
    return r;
}

// Core: counts for P items of (row panel x col panel), into the workspace histogram.
cil_status run_engines(int P, const RowSrc& asrc, const RowSrc& bsrc, int64_t rowsA, int64_t rowsB,
                       const cil_grid& g, uint32_t mask, const Slots& sl, int M, const Plan& pl,
                       const SegParams& sp, const Layout& L, void* ws, const double* radii,
                       int64_t radii_stride, int32_t* status, cudaStream_t st, float* diag = nullptr,
                       uint8_t* binout = nullptr, bool keep_status = false,
                       unsigned long long* range = nullptr, int tile_skip = 0) {
    const int64_t K = (int64_t)g.S * g.H * g.W;
    // TMA row coordinates are int32: the tensor-core engines take < 2^31 packed rows per call
    if (pl.tc && (int64_t)P * (rowsA + rowsB) >= (1ll << 31)) return CIL_EUNSUPPORTED;
    BinParams bp{};
    bp.nq = sl.nq;
    bp.M = M;
    for (int q = 0; q < sl.nq; ++q) bp.slot[q] = sl.slot[q];
    bp.h = grid_h(g);
    bp.w = g.H > 1 ? bp.h * bp.h : bp.h;
    double* thr = at<double>(ws, L.off_thr);
    float* thr2 = pl.tc ? at<float>(ws, L.off_thr2) : nullptr;
    uint64_t* hist = at<uint64_t>(ws, L.off_hist);
    uint32_t* ctr = at<uint32_t>(ws, L.off_ctr);
    uint4* list = L.list_cap ? at<uint4>(ws, L.off_list) : nullptr;
    const uint32_t cap = (t_list_limit >= 0 && t_list_limit < (int64_t)L.list_cap) ? (uint32_t)t_list_limit : L.list_cap;
    CIL_CU(launch_prep(P, sl.nq, M, radii, radii_stride, bp, thr, thr2, status, hist, L.hist_elems, ctr, st,
                       keep_status));
    if (rowsA == 0 || rowsB == 0) return CIL_OK;
    const bool b_same = same_rows(asrc, bsrc) && rowsA == rowsB;

    // The max family's integer-pipe engine and the tensor-core family use different pipes and fit on
    // one SM together (one Gram CTA + one k_max16_reg CTA): with both, the former runs on a side stream.
    // the side stream exists after a thread's first call on a device (eager, like the kernel
    // attribute setup), so a later call with both families can be captured into a graph
    if (t_concurrent) side_setup();
    Fork fk(st, t_concurrent && pl.simt_mask && pl.max16 && pl.tc && range == nullptr && diag == nullptr);
    // With the concurrent engines the max family's tile kernels are enqueued after the INT8 Gram and
    // start only once the Gram's operands are packed: the Gram's CTAs (186 KB of shared memory each)
    // must be resident first — were the max family's CTAs there first, they would fill every SM and
    // keep the Gram out until the end (measured: C5 Gram overlapped by only ~10 %).
    Max16Args m16{};
    bool m16_pending = false;
    if (pl.simt_mask && pl.max16) {
        // max family alone: 15-bit fixed point on the integer pipes (never in distance-range mode,
        // whose plans use the SIMT engine)
        if (range != nullptr) return CIL_EUNSUPPORTED;
        const cudaStream_t sm = fk.side();
        int16_t* qa = at<int16_t>(ws, L.off_aug16);
        int16_t* qb = qa + (size_t)P * rowsA * L.geom16.off[3];
        unsigned* maxbits = at<unsigned>(ws, L.off_max16);
        const AugGeom& g16 = L.geom16;
        CIL_CU(launch_pack16(P, asrc, rowsA, bsrc, rowsB, g16, maxbits, qa, qb, status, sm));
        Max16Args a{};
        a.A = qa; a.B = qb;
        a.rowsA = rowsA; a.rowsB = rowsB; a.Kaug = L.geom16.off[3];
        a.g = g16;
        a.maxbits = maxbits;
        a.dmax = at<uint16_t>(ws, L.off_dmax16);
        a.dmax_elems = 3 * (int64_t)L.dmax_rows_product;
        a.bp = bp;
        a.sp = sp;
        a.thr = thr; a.thr_stride = (int64_t)sl.nq * M;
        a.hist = hist;
        a.status = status;
        a.P = P;
        a.qmask = 0;
        for (int q = 0; q < sl.nq; ++q)
            if ((pl.simt_mask >> sl.slot[q]) & 1u) a.qmask |= 1u << q;
        a.binout = binout;
        a.tri = tile_skip == 2;
        a.sym = binout != nullptr && b_same;
        a.list = list; a.ctr = ctr; a.cap = cap;
        if (!fk.joined && pl.tc && pl.split == 3) {
            m16 = a;
            m16_pending = true;
        } else {
            CIL_CU(launch_max16(a, sm));
        }
    } else if (pl.simt_mask) {
        float* aug = at<float>(ws, L.off_aug);
        float* augB = aug + (size_t)P * rowsA * L.geom.off[3];
        float* statA = at<float>(ws, L.off_rowstat);
        float* statB = statA + (size_t)P * rowsA * 4;
        CIL_CU(launch_pack_aug(P, asrc, rowsA, L.geom, aug, statA, status, st));
        CIL_CU(launch_pack_aug(P, bsrc, rowsB, L.geom, augB, statB, status, st));
        SimtArgs a{};
        a.Aaug = aug; a.Baug = augB;
        a.rowsA = rowsA; a.rowsB = rowsB; a.Kaug = L.geom.off[3];
        a.g = L.geom;
        a.bp = bp;
        a.sp = sp;
        a.thr = thr; a.thr_stride = (int64_t)sl.nq * M;
        a.hist = hist;
        a.status = status;
        a.P = P;
        a.do_max = pl.do_max; a.do_sum = pl.do_sum;
        // the SIMT engine bins only its own measures (L2 may be on the tensor cores)
        a.qmask = 0;
        for (int q = 0; q < sl.nq; ++q)
            if ((pl.simt_mask >> sl.slot[q]) & 1u) a.qmask |= 1u << q;
        a.binout = binout;
        a.range = range;
        a.tri = tile_skip == 2;
        a.sym = binout != nullptr && b_same;
        a.statA = statA; a.statB = statB;
        a.list = list; a.ctr = ctr; a.cap = cap;
        CIL_CU(launch_simt(a, st));
    }
    if (pl.tc) {
        if (!gram_tc_supported()) return CIL_EUNSUPPORTED;
        float* center = at<float>(ws, L.off_center);
        CIL_CU(launch_center(P, bsrc, rowsB < 16 ? rowsB : 16, K, L.Kp, center, st));
        if (pl.split == 3) {
            // ---- three-digit INT8 engine (default): L2, or with pl.aug L2, W12, W12SUM from the
            // Grams of [x~ | D_x x~ | D_y x~]; exact integer accumulation, worst-case bound
            int8_t* planes = at<int8_t>(ws, L.off_hi);
            float* meta = at<float>(ws, L.off_nrm);
            const int64_t pstride = L.rows_cap * L.Krow;
            const int64_t offB = b_same ? 0 : (int64_t)P * rowsA;
            if (pl.aug) {
                const AugGeom ag = make_aug_geom(g.S, g.H, g.W, 3, g.gs);
                CIL_CU(launch_pack3_aug(P, asrc, rowsA, ag, L.kp, center, L.Kp, planes, pstride, 0, meta, status, st));
                if (!b_same)
                    CIL_CU(launch_pack3_aug(P, bsrc, rowsB, ag, L.kp, center, L.Kp, planes, pstride, offB, meta, status,
                                            st));
            } else {
                CIL_CU(launch_pack3(P, asrc, rowsA, K, L.Kp, center, planes, pstride, 0, meta, status, st));
                if (!b_same)
                    CIL_CU(launch_pack3(P, bsrc, rowsB, K, L.Kp, center, planes, pstride, offB, meta, status, st));
            }
            G3Args t{};
            t.planes = planes; t.rows_tot = L.rows_cap; t.Kp = L.Krow; t.meta = meta;
            t.rowsA = rowsA; t.rowsB = rowsB; t.a_off = 0; t.b_off = offB;
            t.P = P; t.p0 = 0; t.np = P;
            t.nph = pl.aug ? 3 : 1;
            if (pl.aug) {
                for (int a = 0; a < 3; ++a) { t.ph_beg[a] = L.kp[a]; t.ph_end[a] = L.kp[a + 1]; }
            } else {
                t.ph_beg[0] = 0; t.ph_end[0] = L.Krow;
            }
            t.thr = thr2; t.thr_stride = 8 * M;
            t.M = M; t.nq = sl.nq; t.q_l2 = sl.q_l2;
            t.q_k[0] = t.q_k[1] = t.q_k[2] = -1;
            for (int q = 0; q < sl.nq; ++q) {
                if (sl.slot[q] == 0) t.q_k[0] = q;
                if (sl.slot[q] == 3) t.q_k[1] = q;
                if (sl.slot[q] == 2) t.q_k[2] = q;
            }
            t.sp = sp; t.hist = hist;
            t.list = list; t.ctr = ctr; t.cap = cap;
            f32_bracket(1.0 / bp.h, &t.ih_rd, &t.ih_ru);
            f32_bracket(1.0 / (bp.h * bp.h), &t.ih2_rd, &t.ih2_ru);
            t.part = pl.aug ? at<float>(ws, L.off_part) : nullptr;
            t.binout = binout;
            t.skip = (binout && b_same) ? 1 : (b_same ? tile_skip : 0);
            t.diag = diag;
            t.hist_elems = L.hist_elems;
            if (m16_pending) fk.side_after_main();          // the Gram's operands are packed
            CIL_CU(launch_gram3(t, st));
            if (m16_pending) {
                m16_pending = false;
                CIL_CU(launch_max16(m16, fk.side()));
            }
        } else {
            // ---- 3xBF16 / 3xTF32 split engine (histogram mode only)
            if (binout) return CIL_EUNSUPPORTED;
            const size_t esz = pl.split == 2 ? 4 : 2;
            char* hi = at<char>(ws, L.off_hi);
            char* lo = at<char>(ws, L.off_lo);
            float* nrm = at<float>(ws, L.off_nrm);
            float* q4 = at<float>(ws, L.off_q4);
            const size_t offB = (size_t)P * rowsA;
            CIL_CU(launch_pack_tc(P, asrc, rowsA, K, L.Kp, center, pl.split, hi, lo, nrm, q4, status, st));
            CIL_CU(launch_pack_tc(P, bsrc, rowsB, K, L.Kp, center, pl.split, hi + offB * L.Kp * esz,
                                  lo + offB * L.Kp * esz, nrm + offB, q4 + offB, status, st));
            TcArgs t{};
            t.hi = hi; t.lo = lo; t.nrm = nrm; t.q4 = q4;
            t.rowsA = rowsA; t.rowsB = rowsB; t.Kp = L.Kp; t.K = K;
            t.P = P; t.split = pl.split;
            t.thr2 = thr2 + 6 * M; t.thr_stride = 8 * M; t.M = M;
            t.q_l2 = sl.q_l2; t.nq = sl.nq;
            t.sp = sp; t.hist = hist;
            t.recheck = list; t.recheck_ctr = ctr; t.recheck_cap = cap;
            t.status = status;
            t.cta_group = 2;
            t.chunk_kb = 4;
            // E = k1 q_a q_b + rel (n_a + n_b): k1 = 8 sigma of the split residual (2^-16 per product
            // for 3xBF16, 2^-20 for 3xTF32, x2 for d^2); rel = truncation over the 12*chunk_kb MMA steps
            // of one chunk + RN adds of the chunk partials + FP32 evaluation / threshold rounding.
            const int64_t n_kb = (L.Kp * (int64_t)esz) / 128;
            const double nchunks = (double)((n_kb + t.chunk_kb - 1) / t.chunk_kb);
            t.guard_k1 = (float)(8.0 * (pl.split == 2 ? ldexp(1.0, -18) : ldexp(1.0, -15)));
            t.guard_rel = (float)(ldexp(1.0, -24) * (8.0 * t.chunk_kb + 3.0 * sqrt(nchunks) + 8.0));
            t.diag = diag;
            t.p0 = 0; t.np = P; t.sm_budget = 0;
            CIL_CU(launch_gram_tc(t, st));
        }
    }
    if (m16_pending) CIL_CU(launch_max16(m16, fk.side()));   // (not reached: the INT8 path launches it)
    fk.join();
    if (diag || range) return CIL_OK;
    if (L.list_cap) {
        RecheckArgs r = recheck_args(asrc, bsrc, K, g, sl, M, bp, sp, L, ws, status, P, binout, rowsA, rowsB, mask);
        r.cap = cap;
        CIL_CU(launch_recheck(r, L.hist_elems, st));
    }
    return CIL_OK;
}

}  // namespace

extern "C" {

size_t cil_features_workspace_size(int32_t P, int64_t N, int64_t Nt, cil_grid g, uint32_t dist_mask,
                                   int32_t M, cil_engine engine) {
    if (P < 1 || P > kMaxItems || N < 0 || Nt < 0 || N > kMaxRows || Nt > kMaxRows || M < 1 || check_grid(g, dist_mask) != CIL_OK) return 0;
    const Slots sl = slots_of(dist_mask);
    const Plan pl = make_plan(dist_mask, engine, g, Nt > 0 ? Nt : 1, Nt, M);
    SegParams sp{N > 0 ? N : 1, Nt > 0 ? Nt : 1, 1, 1};
    return make_layout(P, N, Nt, g, sl.nq, M, pl, sp, 0).total;
}

cil_status cil_features(int32_t P, const float* A, int64_t strideA, int64_t lda, int64_t N, const float* B,
                        int64_t strideB, int64_t ldb, int64_t Nt, cil_grid g, uint32_t dist_mask,
                        const double* radii, int64_t radii_stride, int32_t M, uint64_t* counts, double* y,
                        int32_t* item_status, cil_engine engine, void* ws, size_t ws_bytes, void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_features");
    if (P < 1 || P > kMaxItems || N < 0 || Nt < 0 || N > kMaxRows || Nt > kMaxRows || M < 1 || M > kMaxM) return CIL_EINVAL;
    if (check_grid(g, dist_mask) != CIL_OK) return CIL_EINVAL;
    if ((int)engine < 0 || (int)engine > 4) return CIL_EINVAL;
    if (!radii || !counts || !item_status || !ws) return CIL_EINVAL;
    if ((N > 0 && !A) || (Nt > 0 && !B)) return CIL_EINVAL;
    if (strideA < 0 || strideB < 0 || radii_stride < 0) return CIL_EINVAL;
    const int64_t K = (int64_t)g.S * g.H * g.W;
    if ((N > 0 && lda < K) || (Nt > 0 && ldb < K)) return CIL_EINVAL;
    if (N > 0 && P > 1 && strideA < (N - 1) * lda + K) return CIL_EINVAL;
    if (Nt > 0 && P > 1 && strideB < (Nt - 1) * ldb + K) return CIL_EINVAL;
    if (K % 4 || lda % 4 || ldb % 4 || strideA % 4 || strideB % 4) return CIL_EUNSUPPORTED;
    if ((A && !aligned16(A)) || (B && !aligned16(B))) return CIL_EUNSUPPORTED;
    const Slots sl = slots_of(dist_mask);
    const Plan pl = make_plan(dist_mask, engine, g, Nt > 0 ? Nt : 1, Nt, M);
    SegParams sp{N > 0 ? N : 1, Nt > 0 ? Nt : 1, 1, 1};
    const Layout L = make_layout(P, N, Nt, g, sl.nq, M, pl, sp, 0);
    if (ws_bytes < L.total) return CIL_ENOMEM;
    void* wsa = reinterpret_cast<void*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    RowSrc as{}, bs{};
    as.base = A; as.stride = strideA; as.ld = lda; as.rows = N; as.mode = MODE_PLAIN;
    bs.base = B; bs.stride = strideB; bs.ld = ldb; bs.rows = Nt; bs.mode = MODE_PLAIN;
    cil_status s = run_engines(P, as, bs, N, Nt, g, dist_mask, sl, M, pl, sp, L, wsa, radii, radii_stride,
                               item_status, st);
    if (s != CIL_OK) return s;
    CIL_CU(launch_finalize(P, sl.nq, M, sp, at<uint64_t>(wsa, L.off_hist), counts, y, N, Nt, nullptr,
                           nullptr, st));
    return CIL_OK;
}

cil_status cil_features_recheck_count(int32_t P, int64_t N, int64_t Nt, cil_grid g, uint32_t dist_mask, int32_t M,
                                      cil_engine engine, const void* ws, uint64_t* listed, uint64_t* capacity) {
    if (P < 1 || P > kMaxItems || N < 0 || Nt < 0 || N > kMaxRows || Nt > kMaxRows || M < 1 || !ws || !listed || !capacity || check_grid(g, dist_mask) != CIL_OK)
        return CIL_EINVAL;
    const Slots sl = slots_of(dist_mask);
    const Plan pl = make_plan(dist_mask, engine, g, Nt > 0 ? Nt : 1, Nt, M);
    SegParams sp{N > 0 ? N : 1, Nt > 0 ? Nt : 1, 1, 1};
    const Layout L = make_layout(P, N, Nt, g, sl.nq, M, pl, sp, 0);
    const void* wsa = reinterpret_cast<const void*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    uint32_t c = 0;
    CIL_CU(cudaMemcpy(&c, reinterpret_cast<const char*>(wsa) + L.off_ctr, sizeof(c), cudaMemcpyDeviceToHost));
    *listed = c;
    *capacity = L.list_cap;
    return CIL_OK;
}

cil_status cil_normalize(int64_t n, const uint64_t* counts, double npairs, double* y, void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_normalize");
    if (n < 0 || (n > 0 && (!counts || !y)) || !(npairs > 0.0)) return CIL_EINVAL;
    CIL_CU(launch_normalize(n, counts, npairs, y, reinterpret_cast<cudaStream_t>(stream)));
    return CIL_OK;
}

cil_status cil_stats(int32_t P, const double* Y, int32_t n, int32_t D, double* mu, double* Sigma,
                     void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_stats");
    if (P < 1 || n < 2 || D < 1 || !Y || !mu || !Sigma) return CIL_EINVAL;
    CIL_CU(launch_stats(P, Y, n, D, mu, Sigma, reinterpret_cast<cudaStream_t>(stream)));
    return CIL_OK;
}

namespace {
// Regularised lower incomplete gamma P(a, x) in FP64: the power series for x < a + 1, else
// 1 - Q(a, x) from the continued fraction (modified Lentz).
double gamma_p(double a, double x) {
    if (!(x > 0.0)) return 0.0;
    const double lpre = -x + a * log(x) - lgamma(a);
    if (x < a + 1.0) {
        double ap = a, del = 1.0 / a, sum = del;
        for (int it = 0; it < 10000; ++it) {
            ap += 1.0;
            del *= x / ap;
            sum += del;
            if (fabs(del) < fabs(sum) * 1e-17) break;
        }
        return fmin(1.0, sum * exp(lpre));
    }
    const double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i < 10000; ++i) {
        const double an = -i * (i - a);
        b += 2.0;
        d = an * d + b;
        if (fabs(d) < tiny) d = tiny;
        c = b + an / c;
        if (fabs(c) < tiny) c = tiny;
        d = 1.0 / d;
        const double del = d * c;
        h *= del;
        if (fabs(del - 1.0) < 1e-17) break;
    }
    return fmax(0.0, 1.0 - exp(lpre) * h);
}
}  // namespace

double cil_chi2_quantile(int32_t D, double prob) {
    if (D < 1 || !(prob > 0.0) || !(prob < 1.0)) return NAN;
    const double a = 0.5 * D;
    double lo = 0.0, hi = fmax(1.0, 2.0 * D);
    while (gamma_p(a, 0.5 * hi) < prob) hi *= 2.0;                // chi^2_D CDF(x) = P(D/2, x/2)
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (gamma_p(a, 0.5 * mid) < prob) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

cil_status cil_gaussianity_pearson(int64_t n, const double* d2, int32_t D, int32_t bins, double* out, void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_gaussianity_pearson");
    if (n < 1 || !d2 || !out || D < 1 || bins < 2 || bins > kMaxChi2Bins) return CIL_EINVAL;
    Chi2Edges ed{};
    ed.nb = bins;
    for (int b = 1; b < bins; ++b) ed.e[b - 1] = cil_chi2_quantile(D, (double)b / bins);
    CIL_CU(launch_chi2_pearson(n, d2, ed, out, reinterpret_cast<cudaStream_t>(stream)));
    return CIL_OK;
}

cil_status cil_loglik(int32_t P, const double* mu, int64_t mu_stride, const double* Sigma, int64_t Sigma_stride,
                      const double* y_obs, int32_t D, double ridge, double* out, int32_t* item_status,
                      void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_loglik");
    if (P < 1 || D < 1 || !mu || !Sigma || !y_obs || !out || !item_status) return CIL_EINVAL;
    if (D > kMaxD) return CIL_EUNSUPPORTED;
    if (mu_stride < 0 || Sigma_stride < 0 || !(ridge >= 0.0)) return CIL_EINVAL;
    CIL_CU(launch_loglik(P, mu, mu_stride, Sigma, Sigma_stride, y_obs, D, ridge, out, item_status, nullptr,
                         reinterpret_cast<cudaStream_t>(stream)));
    return CIL_OK;
}

namespace {
// SCIL panel geometry.  The INT8 Gram tiles 256 rows x 128 columns; when the row panel
// ((n_ens+1) N_set rows, e.g. 550) pads worse on the 256-row axis than the column panel
// (n_ens N~, e.g. 500), the panels are swapped (the column panel runs as the Gram's rows;
// segments become [l][k], k_build_Y reads them transposed).  Only for the INT8 engine.
struct SynthGeo {
    bool swap;
    int64_t rowsA, rowsB;     // Gram rows / columns
    SegParams sp;
    Plan pl;
};
int64_t pad_cols(int64_t n) { return (n + 127) / 128 * 128; }
SynthGeo synth_geo(int32_t n_ens, int32_t N_set, int32_t N_tilde, const cil_grid& g, uint32_t mask, int32_t M,
                   cil_engine engine) {
    SynthGeo s{};
    const int64_t R = (int64_t)(n_ens + 1) * N_set, C = (int64_t)n_ens * N_tilde;
    s.swap = false;
    s.rowsA = R; s.rowsB = C;
    s.sp = SegParams{N_set, N_tilde, n_ens + 1, n_ens};
    s.pl = make_plan(mask, engine, g, N_tilde, C, M);
    const int64_t cost = (R + 255) / 256 * 256 * pad_cols(C), cost_sw = (C + 255) / 256 * 256 * pad_cols(R);
    if (cost_sw < cost && s.pl.tc && s.pl.split == 3) {
        const Plan ps = make_plan(mask, engine, g, N_set, R, M);
        if (ps.tc && ps.split == 3 && ps.aug == s.pl.aug) {
            s.swap = true;
            s.rowsA = C; s.rowsB = R;
            s.sp = SegParams{N_tilde, N_set, n_ens, n_ens + 1};
            s.pl = ps;
        }
    }
    return s;
}
}  // namespace

size_t cil_synth_workspace_size(int32_t P, int32_t n_ens, int32_t N_set, int32_t N_tilde, cil_grid g,
                                uint32_t dist_mask, int32_t M, cil_engine engine) {
    if (P < 1 || P > kMaxItems || n_ens < 2 || N_set < 1 || N_tilde < 1 || (int64_t)(n_ens + 1) * N_set > kMaxRows || (int64_t)n_ens * N_tilde > kMaxRows || M < 1 || check_grid(g, dist_mask) != CIL_OK)
        return 0;
    const Slots sl = slots_of(dist_mask);
    const SynthGeo sg = synth_geo(n_ens, N_set, N_tilde, g, dist_mask, M, engine);
    const int64_t nY = (int64_t)P * (n_ens * n_ens + 1) * sl.nq * M;
    return make_layout(P, sg.rowsA, sg.rowsB, g, sl.nq, M, sg.pl, sg.sp, nY).total;
}

cil_status cil_synth_loglik(int32_t P, const float* pools, int64_t pool_stride, int64_t ld, int32_t n_ens,
                            int32_t N_set, int32_t N_tilde, const float* data, int64_t ld_data,
                            const int32_t* k0, cil_grid g, uint32_t dist_mask, const double* radii, int32_t M,
                            double ridge, double* out, int32_t* item_status, double* Y_out, cil_engine engine,
                            void* ws, size_t ws_bytes, void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_synth_loglik");
    if (P < 1 || P > kMaxItems || n_ens < 2 || N_set < 1 || N_tilde < 1 || M < 1 || M > kMaxM) return CIL_EINVAL;
    if ((int64_t)(n_ens + 1) * N_set > kMaxRows || (int64_t)n_ens * N_tilde > kMaxRows) return CIL_EINVAL;
    if (check_grid(g, dist_mask) != CIL_OK) return CIL_EINVAL;
    if ((int)engine < 0 || (int)engine > 4) return CIL_EINVAL;
    if (!pools || !data || !k0 || !radii || !out || !item_status || !ws) return CIL_EINVAL;
    if (!(ridge >= 0.0)) return CIL_EINVAL;
    const int64_t K = (int64_t)g.S * g.H * g.W;
    const int64_t Nsyn = (int64_t)n_ens * (N_set + N_tilde);
    if (ld < K || ld_data < K) return CIL_EINVAL;
    if (P > 1 && pool_stride < (Nsyn - 1) * ld + K) return CIL_EINVAL;
    if (K % 4 || ld % 4 || ld_data % 4 || pool_stride % 4) return CIL_EUNSUPPORTED;
    if (!aligned16(pools) || !aligned16(data)) return CIL_EUNSUPPORTED;
    const Slots sl = slots_of(dist_mask);
    if (sl.nq * M > kMaxD) return CIL_EUNSUPPORTED;
    const SynthGeo sg = synth_geo(n_ens, N_set, N_tilde, g, dist_mask, M, engine);
    const Plan& pl = sg.pl;
    const int64_t rowsA = (int64_t)(n_ens + 1) * N_set, rowsB = (int64_t)n_ens * N_tilde;
    const SegParams& sp = sg.sp;
    const int nv = n_ens * n_ens;
    const int64_t nY = (int64_t)P * (nv + 1) * sl.nq * M;
    const Layout L = make_layout(P, sg.rowsA, sg.rowsB, g, sl.nq, M, pl, sp, nY);
    if (ws_bytes < L.total) return CIL_ENOMEM;
    void* wsa = reinterpret_cast<void*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    RowSrc as{}, bs{};
    as.base = pools; as.stride = pool_stride; as.ld = ld; as.rows = rowsA; as.mode = MODE_SYN_ROW;
    as.n_ens = n_ens; as.N_set = N_set; as.N_tilde = N_tilde; as.data = data; as.ld_data = ld_data;
    bs = as;
    bs.rows = rowsB; bs.mode = MODE_SYN_COL;
    cil_status s = sg.swap ? run_engines(P, bs, as, rowsB, rowsA, g, dist_mask, sl, M, pl, sp, L, wsa, radii,
                                         (int64_t)sl.nq * M, item_status, st)
                           : run_engines(P, as, bs, rowsA, rowsB, g, dist_mask, sl, M, pl, sp, L, wsa, radii,
                                         (int64_t)sl.nq * M, item_status, st);
    if (s != CIL_OK) return s;
    double* Y = Y_out ? Y_out : at<double>(wsa, L.off_Y);
    CIL_CU(launch_synth_tail(P, n_ens, sl.nq, M, sp, at<uint64_t>(wsa, L.off_hist), N_set, N_tilde, k0, ridge,
                             out, item_status, Y, at<double>(wsa, L.off_mu), at<double>(wsa, L.off_sig), st,
                             sg.swap));
    return CIL_OK;
}

// ------------------------------------------------------------------ min-max scaled patterns
cil_status cil_minmax_scale(int64_t n, const float* X, int64_t ldx, float* Y, int64_t ldy, cil_grid g,
                            void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_minmax_scale");
    if (n < 0 || g.S < 1 || g.H < 1 || g.W < 1) return CIL_EINVAL;
    const int64_t K = (int64_t)g.S * g.H * g.W;
    if (n > 0 && (!X || !Y || ldx < K || ldy < K)) return CIL_EINVAL;
    CIL_CU(launch_minmax(n, X, ldx, Y, ldy, g.S, (int64_t)g.H * g.W, reinterpret_cast<cudaStream_t>(stream)));
    return CIL_OK;
}

// ------------------------------------------------------------------ adaptive radii
size_t cil_range_workspace_size(int32_t P, int64_t N, int64_t Nt, cil_grid g, uint32_t dist_mask) {
    if (P < 1 || P > kMaxItems || N < 0 || Nt < 0 || N > kMaxRows || Nt > kMaxRows || check_grid(g, dist_mask) != CIL_OK) return 0;
    const Slots sl = slots_of(dist_mask);
    const Plan pl = make_plan(dist_mask, CIL_ENGINE_SIMT, g);
    SegParams sp{N > 0 ? N : 1, Nt > 0 ? Nt : 1, 1, 1};
    return make_layout(P, N, Nt, g, sl.nq, 1, pl, sp, 0).total + 512;
}

cil_status cil_distance_range(int32_t P, const float* A, int64_t strideA, int64_t lda, int64_t N, const float* B,
                              int64_t strideB, int64_t ldb, int64_t Nt, cil_grid g, uint32_t dist_mask,
                              double* range, int32_t* item_status, void* ws, size_t ws_bytes, void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_distance_range");
    if (P < 1 || P > kMaxItems || N < 1 || Nt < 1 || N > kMaxRows || Nt > kMaxRows) return CIL_EINVAL;
    if (check_grid(g, dist_mask) != CIL_OK) return CIL_EINVAL;
    if (!range || !item_status || !ws) return CIL_EINVAL;
    cil_status s = check_sets(P, A, strideA, lda, N, B, strideB, ldb, Nt, g);
    if (s != CIL_OK) return s;
    const Slots sl = slots_of(dist_mask);
    const Plan pl = make_plan(dist_mask, CIL_ENGINE_SIMT, g);     // exact FP64 measures on CUDA cores
    SegParams sp{N, Nt, 1, 1};
    const Layout L = make_layout(P, N, Nt, g, sl.nq, 1, pl, sp, 0);
    if (ws_bytes < L.total + 512) return CIL_ENOMEM;
    void* wsa = reinterpret_cast<void*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    double* r = at<double>(wsa, L.total);                 // a dummy radius per measure (not binned)
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CIL_CU(launch_fill_f64(r, sl.nq, 1.0, st));          // device-side: stays asynchronous and capturable
    unsigned long long* rg = reinterpret_cast<unsigned long long*>(range);   // non-negative FP64 bits: ordered
    CIL_CU(launch_range_init(P, sl.nq, rg, st));
    RowSrc as{}, bs{};
    as.base = A; as.stride = strideA; as.ld = lda; as.rows = N; as.mode = MODE_PLAIN;
    bs.base = B; bs.stride = strideB; bs.ld = ldb; bs.rows = Nt; bs.mode = MODE_PLAIN;
    return run_engines(P, as, bs, N, Nt, g, dist_mask, sl, 1, pl, sp, L, wsa, r, 0, item_status, st, nullptr,
                       nullptr, false, rg);
}

cil_status cil_radii_from_range(int32_t P, int32_t n_meas, int32_t M, const double* range, int32_t law,
                                double margin, double* radii, int32_t* item_status, void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_radii_from_range");
    if (P < 1 || n_meas < 1 || n_meas > kMaxMeas || M < 1 || M > kMaxM || (law != 0 && law != 1)) return CIL_EINVAL;
    if (!range || !radii || !item_status || !(margin >= 0.0 && margin < 1.0)) return CIL_EINVAL;
    CIL_CU(launch_radii(P, n_meas, M, reinterpret_cast<const unsigned long long*>(range), law, margin, radii,
                        item_status, reinterpret_cast<cudaStream_t>(stream)));
    return CIL_OK;
}

// ------------------------------------------------------------------ Alg. 1 / Alg. 2 training vectors
size_t cil_train_workspace_size(int32_t P, int32_t n_ens, int32_t N, cil_grid g, uint32_t dist_mask, int32_t M,
                                cil_engine engine) {
    if (P < 1 || P > kMaxItems || n_ens < 2 || N < 1 || (int64_t)n_ens * N > kMaxRows || M < 1 || check_grid(g, dist_mask) != CIL_OK) return 0;
    const Slots sl = slots_of(dist_mask);
    const int64_t rows = (int64_t)n_ens * N;
    const Plan pl = make_plan(dist_mask, engine, g, N, rows, M);
    SegParams sp{N, N, n_ens, n_ens};
    return make_layout(P, rows, rows, g, sl.nq, M, pl, sp, 0).total;
}

cil_status cil_train_vectors(int32_t P, const float* X, int64_t stride, int64_t ld, int32_t n_ens, int32_t N,
                             cil_grid g, uint32_t dist_mask, const double* radii, int64_t radii_stride, int32_t M,
                             double* Y, int32_t* item_status, cil_engine engine, void* ws, size_t ws_bytes,
                             void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_train_vectors");
    if (P < 1 || P > kMaxItems || n_ens < 2 || N < 1 || (int64_t)n_ens * N > kMaxRows || M < 1 || M > kMaxM) return CIL_EINVAL;
    if (check_grid(g, dist_mask) != CIL_OK) return CIL_EINVAL;
    if ((int)engine < 0 || (int)engine > 4) return CIL_EINVAL;
    if (!X || !radii || !Y || !item_status || !ws || radii_stride < 0 || stride < 0) return CIL_EINVAL;
    const int64_t K = (int64_t)g.S * g.H * g.W;
    const int64_t rows = (int64_t)n_ens * N;
    if (ld < K || (P > 1 && stride < (rows - 1) * ld + K)) return CIL_EINVAL;
    if (K % 4 || ld % 4 || stride % 4 || !aligned16(X)) return CIL_EUNSUPPORTED;
    const Slots sl = slots_of(dist_mask);
    const Plan pl = make_plan(dist_mask, engine, g, N, rows, M);
    SegParams sp{N, N, n_ens, n_ens};
    const Layout L = make_layout(P, rows, rows, g, sl.nq, M, pl, sp, 0);
    if (ws_bytes < L.total) return CIL_ENOMEM;
    void* wsa = reinterpret_cast<void*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    RowSrc xs{};
    xs.base = X; xs.stride = stride; xs.ld = ld; xs.rows = rows; xs.mode = MODE_PLAIN;
    // one panel against itself, segmented by subset: block (k, l) = C(R, s^k, s^l)
    cil_status s = run_engines(P, xs, xs, rows, rows, g, dist_mask, sl, M, pl, sp, L, wsa, radii, radii_stride,
                               item_status, st, nullptr, nullptr, false, nullptr, /*tile_skip=*/2);
    if (s != CIL_OK) return s;
    CIL_CU(launch_build_pairs(P, n_ens, sl.nq, M, sp, at<uint64_t>(wsa, L.off_hist), N, Y, st));
    return CIL_OK;
}

// ------------------------------------------------------------------ bootstrap (Alg. A1 / A2)

size_t cil_bin_matrix_workspace_size(int32_t P, int64_t N, int64_t Nt, cil_grid g, uint32_t dist_mask, int32_t M,
                                     cil_engine engine) {
    if (P < 1 || P > kMaxItems || N < 0 || Nt < 0 || N > kMaxRows || Nt > kMaxRows || M < 1 || check_grid(g, dist_mask) != CIL_OK) return 0;
    Plan pl;
    if (!plan_bins(dist_mask, engine, g, &pl)) return 0;
    const Slots sl = slots_of(dist_mask);
    SegParams sp{N > 0 ? N : 1, Nt > 0 ? Nt : 1, 1, 1};
    return make_layout(P, N, Nt, g, sl.nq, M, pl, sp, 0).total;
}

cil_status cil_bin_matrix(int32_t P, const float* A, int64_t strideA, int64_t lda, int64_t N, const float* B,
                          int64_t strideB, int64_t ldb, int64_t Nt, cil_grid g, uint32_t dist_mask,
                          const double* radii, int64_t radii_stride, int32_t M, uint8_t* bins,
                          int32_t* item_status, cil_engine engine, void* ws, size_t ws_bytes, void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_bin_matrix");
    if (P < 1 || P > kMaxItems || N < 0 || Nt < 0 || N > kMaxRows || Nt > kMaxRows || M < 1 || M > kMaxM) return CIL_EINVAL;
    if (check_grid(g, dist_mask) != CIL_OK) return CIL_EINVAL;
    if ((int)engine < 0 || (int)engine > 4) return CIL_EINVAL;
    if (!radii || !item_status || !ws || (N > 0 && Nt > 0 && !bins) || radii_stride < 0) return CIL_EINVAL;
    cil_status s = check_sets(P, A, strideA, lda, N, B, strideB, ldb, Nt, g);
    if (s != CIL_OK) return s;
    Plan pl;
    if (!plan_bins(dist_mask, engine, g, &pl)) return CIL_EUNSUPPORTED;
    const Slots sl = slots_of(dist_mask);
    SegParams sp{N > 0 ? N : 1, Nt > 0 ? Nt : 1, 1, 1};
    const Layout L = make_layout(P, N, Nt, g, sl.nq, M, pl, sp, 0);
    if (ws_bytes < L.total) return CIL_ENOMEM;
    void* wsa = reinterpret_cast<void*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    RowSrc as{}, bs{};
    as.base = A; as.stride = strideA; as.ld = lda; as.rows = N; as.mode = MODE_PLAIN;
    bs.base = B; bs.stride = strideB; bs.ld = ldb; bs.rows = Nt; bs.mode = MODE_PLAIN;
    return run_engines(P, as, bs, N, Nt, g, dist_mask, sl, M, pl, sp, L, wsa, radii, radii_stride, item_status,
                       st, nullptr, bins);
}

cil_status cil_resample_counts(int32_t P, const uint8_t* bins, int64_t N, int64_t Nt, int32_t n_meas, int32_t M,
                               int32_t n_rep, const int32_t* I1, int64_t n1, const int32_t* I2, int64_t n2,
                               uint64_t* counts, double* y, int64_t y_item_stride, int32_t* item_status,
                               void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_resample_counts");
    if (P < 1 || P > kMaxItems || N < 1 || Nt < 1 || n_meas < 1 || n_meas > kMaxMeas || M < 1 || M > kMaxM) return CIL_EINVAL;
    if (n_rep < 1 || n1 < 1 || n2 < 1 || !bins || !I1 || !I2 || !item_status || (!counts && !y)) return CIL_EINVAL;
    if (y_item_stride < 0 || (y && y_item_stride > 0 && y_item_stride < (int64_t)n_rep * n_meas * M))
        return CIL_EINVAL;
    if (y_item_stride == 0) y_item_stride = (int64_t)n_rep * n_meas * M;
    if (!resample_fits(N, Nt, M)) return CIL_EUNSUPPORTED;
    CIL_CU(launch_resample(P, bins, N, Nt, n_meas, M, n_rep, I1, n1, I2, n2, counts, y, y_item_stride,
                           item_status, reinterpret_cast<cudaStream_t>(stream)));
    return CIL_OK;
}

namespace {
struct BootLayout {
    Layout L;
    size_t off_bins, total;
    Plan pb, ph;
    // tensor-core resample (steps 2.1-2.4 as one integer GEMM per measure, resample.cu)
    bool rd;
    int64_t kp_rd, ntp;
    size_t off_m1, off_m2, off_e, off_cnt;
};
// The GEMM form needs m1 <= 127 (int8 operand), m2 <= 65535 (u16) and n1 n2 < 2^32 (u32
// epilogue sums); the CUDA-core engine choice keeps the shared-atomic resample.
bool boot_rd(int32_t N_syn, int32_t N_set, int32_t n_rep, int32_t P, int nq, int32_t M, cil_engine engine) {
    if (engine == CIL_ENGINE_SIMT || N_set > 127) return false;
    const int64_t Nt = (int64_t)N_syn - N_set;
    if (Nt > 65535 || (int64_t)N_set * Nt >= (1ll << 32)) return false;
    const int64_t ntp = ((int64_t)N_syn + 255) / 256 * 256;   // rowdot.cu: b-blocks of 256
    if ((int64_t)P * (n_rep + (int64_t)M * ntp) >= (1ll << 31)) return false;
    const int64_t kp = ((int64_t)N_syn + kTcBK - 1) / kTcBK * kTcBK;
    return 2 * (kp + ntp) * 4 <= 200 * 1024 && nq >= 1;     // k_rd_mult: 4 warps x (kp + ntp) u16
}
bool boot_layout(int32_t P, int32_t N_syn, int32_t N_set, int32_t n_rep, const cil_grid& g, uint32_t mask,
                 int32_t M, cil_engine engine, BootLayout* B) {
    if (!plan_bins(mask, engine, g, &B->pb)) return false;
    const int32_t Nt = N_syn - N_set;
    B->ph = make_plan(mask, engine, g, Nt, Nt, M);
    const Plan u = plan_union(B->pb, B->ph);
    const Slots sl = slots_of(mask);
    SegParams sp{N_syn, N_syn, 1, 1};
    const int64_t nY = (int64_t)P * (n_rep + 1) * sl.nq * M;
    B->L = make_layout(P, N_syn, N_syn, g, sl.nq, M, u, sp, nY);
    B->off_bins = al(B->L.total);
    B->total = B->off_bins + al((size_t)P * sl.nq * N_syn * (size_t)N_syn);
    B->rd = boot_rd(N_syn, N_set, n_rep, P, sl.nq, M, engine);
    if (B->rd) {
        B->kp_rd = ((int64_t)N_syn + kTcBK - 1) / kTcBK * kTcBK;
        B->ntp = ((int64_t)N_syn + 255) / 256 * 256;
        B->off_m1 = B->total;                                        // M1 rows, then E rows (stacked planes)
        B->off_e = B->off_m1 + (size_t)P * n_rep * B->kp_rd;
        B->total = al(B->off_e + (size_t)P * M * B->ntp * B->kp_rd);
        B->off_m2 = B->total;
        B->total += al((size_t)P * n_rep * B->ntp * 2);
        B->off_cnt = B->total;
        B->total += al((size_t)P * n_rep * M * 8);
    }
    B->total += 256;
    return true;
}
}  // namespace

size_t cil_synth_boot_workspace_size(int32_t P, int32_t N_syn, int32_t N_set, int32_t n_rep, cil_grid g,
                                     uint32_t dist_mask, int32_t M, cil_engine engine) {
    if (P < 1 || P > kMaxItems || N_set < 1 || N_syn <= N_set || N_syn > kMaxRows || n_rep < 2 || M < 1 || check_grid(g, dist_mask) != CIL_OK) return 0;
    BootLayout B;
    if (!boot_layout(P, N_syn, N_set, n_rep, g, dist_mask, M, engine, &B)) return 0;
    return B.total;
}

cil_status cil_synth_loglik_boot(int32_t P, const float* pools, int64_t pool_stride, int64_t ld, int32_t N_syn,
                                 const float* data, int64_t ld_data, int32_t N_set, int32_t n_rep,
                                 const int32_t* I1, const int32_t* I2, const int32_t* J, cil_grid g,
                                 uint32_t dist_mask, const double* radii, int32_t M, double ridge, double* out,
                                 int32_t* item_status, double* Y_out, cil_engine engine, void* ws, size_t ws_bytes,
                                 void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_synth_loglik_boot");
    if (P < 1 || P > kMaxItems || N_set < 1 || N_syn <= N_set || N_syn > kMaxRows || n_rep < 2 || M < 1 || M > kMaxM) return CIL_EINVAL;
    if (check_grid(g, dist_mask) != CIL_OK) return CIL_EINVAL;
    if ((int)engine < 0 || (int)engine > 4) return CIL_EINVAL;
    if (!pools || !data || !I1 || !I2 || !J || !radii || !out || !item_status || !ws) return CIL_EINVAL;
    if (!(ridge >= 0.0)) return CIL_EINVAL;
    const int64_t K = (int64_t)g.S * g.H * g.W;
    if (ld < K || ld_data < K) return CIL_EINVAL;
    if (P > 1 && pool_stride < ((int64_t)N_syn - 1) * ld + K) return CIL_EINVAL;
    if (K % 4 || ld % 4 || ld_data % 4 || pool_stride % 4) return CIL_EUNSUPPORTED;
    if (!aligned16(pools) || !aligned16(data)) return CIL_EUNSUPPORTED;
    const Slots sl = slots_of(dist_mask);
    const int D = sl.nq * M;
    if (D > kMaxD) return CIL_EUNSUPPORTED;
    BootLayout B;
    if (!boot_layout(P, N_syn, N_set, n_rep, g, dist_mask, M, engine, &B)) return CIL_EUNSUPPORTED;
    if (!resample_fits(N_syn, N_syn, M)) return CIL_EUNSUPPORTED;
    if (ws_bytes < B.total) return CIL_ENOMEM;
    void* wsa = reinterpret_cast<void*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int32_t Nt = N_syn - N_set;
    uint8_t* bins = at<uint8_t>(wsa, B.off_bins);
    double* Y = Y_out ? Y_out : at<double>(wsa, B.L.off_Y);
    const int64_t Ystride = (int64_t)(n_rep + 1) * D;
    // step 2 (all pool pairs once): bin matrix of pool x pool
    RowSrc ps{};
    ps.base = pools; ps.stride = pool_stride; ps.ld = ld; ps.rows = N_syn; ps.mode = MODE_PLAIN;
    SegParams spb{N_syn, N_syn, 1, 1};
    cil_status s = run_engines(P, ps, ps, N_syn, N_syn, g, dist_mask, sl, M, B.pb, spb, B.L, wsa, radii, D,
                               item_status, st, nullptr, bins);
    if (s != CIL_OK) return s;
    // steps 2.1-2.4: the n_rep resampled vectors, straight into Y rows [0, n_rep)
    if (B.rd && gram_tc_supported()) {
        int8_t* M1 = at<int8_t>(wsa, B.off_m1);
        int8_t* E = at<int8_t>(wsa, B.off_e);
        uint16_t* M2 = at<uint16_t>(wsa, B.off_m2);
        unsigned long long* cnt = at<unsigned long long>(wsa, B.off_cnt);
        CIL_CU(launch_rd_mult(P, N_syn, B.kp_rd, B.ntp, n_rep, I1, N_set, I2, Nt, M1, M2, item_status, st));
        for (int q = 0; q < sl.nq; ++q) {
            CIL_CU(launch_rd_build_E(P, bins, N_syn, sl.nq, q, M, B.kp_rd, B.ntp, E, st));
            CIL_CU(cudaMemsetAsync(cnt, 0, (size_t)P * n_rep * M * 8, st));
            RowdotArgs t{};
            t.ops = M1;                                            // M1 rows, then the E rows (stacked)
            t.rowsA = n_rep; t.rowsB = (int64_t)M * B.ntp; t.Kp = B.kp_rd;
            t.P = P;
            t.m2 = M2; t.rd_nt = B.ntp; t.rd_m = M; t.out = cnt;
            CIL_CU(launch_rowdot(t, st));
            CIL_CU(launch_rd_final(cnt, P, n_rep, M, sl.nq, q, (double)N_set * (double)Nt, Y, Ystride, st));
        }
    } else {
        CIL_CU(launch_resample(P, bins, N_syn, N_syn, sl.nq, M, n_rep, I1, N_set, I2, Nt, nullptr, Y, Ystride,
                               item_status, st));
    }
    // steps 4-5: y~ = C(R, s_data, pool rows J[p]) into Y row n_rep
    CIL_CU(launch_check_index(P, J, Nt, N_syn, item_status, st));
    if (B.pb.tc && B.pb.split == 3 && !B.pb.aug && !B.pb.simt_mask && gram_tc_supported()) {
        // The pool rows are already packed (INT8 planes, centred on the item's pool): bin ALL
        // pool rows (A, 4 tiles of 256) against the s_data rows (B, one 64-wide tile) with
        // those planes (only s_data is packed), then count with the multiplicities of J:
        // C(R, s_data, pool[J]) = sum_b #{j : J_j = b} [...] (the resample kernel with one
        // replicate, identity rows, column draws J, on the transposed [s_data][pool] output).
        const int64_t K = (int64_t)g.S * g.H * g.W;
        const Layout& L = B.L;
        float* center = at<float>(wsa, L.off_center);
        int8_t* planes = at<int8_t>(wsa, L.off_hi);
        float* meta = at<float>(wsa, L.off_nrm);
        uint32_t* ctr = at<uint32_t>(wsa, L.off_ctr);
        const int64_t a_off = (int64_t)P * N_syn;                 // data rows after the pool rows
        RowSrc ds{};
        ds.base = data; ds.stride = 0; ds.ld = ld_data; ds.rows = N_set; ds.mode = MODE_PLAIN;
        CIL_CU(cudaMemsetAsync(ctr, 0, sizeof(uint32_t), st));
        CIL_CU(launch_pack3(P, ds, N_set, K, L.Kp, center, planes, L.rows_cap * L.Krow, a_off, meta, item_status, st));
        const bool narrow = N_set <= 64;                           // s_data as a 64-wide B tile
        SegParams sph = narrow ? SegParams{N_syn, N_set, 1, 1} : SegParams{N_set, N_syn, 1, 1};
        G3Args t{};
        t.planes = planes; t.rows_tot = L.rows_cap; t.Kp = L.Krow; t.meta = meta;
        t.rowsA = narrow ? N_syn : N_set; t.rowsB = narrow ? N_set : N_syn;
        t.a_off = narrow ? 0 : a_off; t.b_off = narrow ? a_off : 0;
        t.tn_force = narrow ? 64 : 0;
        t.P = P; t.p0 = 0; t.np = P;
        t.nph = 1; t.ph_beg[0] = 0; t.ph_end[0] = L.Krow;
        t.thr = at<float>(wsa, L.off_thr2); t.thr_stride = 8 * M; t.M = M; t.q_l2 = sl.q_l2; t.nq = sl.nq;
        t.q_k[0] = sl.q_l2; t.q_k[1] = t.q_k[2] = -1;
        t.sp = sph; t.hist = at<uint64_t>(wsa, L.off_hist);
        t.list = at<uint4>(wsa, L.off_list); t.ctr = ctr; t.cap = L.list_cap;
        t.binout = bins;                                          // [P][nq][N_set][N_syn] either way
        t.bin_t = narrow;                                         // (narrow: the transposed output)
        CIL_CU(launch_gram3(t, st));
        BinParams bp{};
        bp.h = grid_h(g);
        bp.w = g.H > 1 ? bp.h * bp.h : bp.h;
        RecheckArgs r = recheck_args(narrow ? ps : ds, narrow ? ds : ps, K, g, sl, M, bp, sph, L, wsa, item_status, P,
                                     bins, t.rowsA, t.rowsB, CIL_L2);
        r.mirror = false;
        r.transpose = narrow;
        CIL_CU(launch_recheck(r, 0, st));
        CIL_CU(launch_resample(P, bins, N_set, N_syn, sl.nq, M, 1, nullptr, N_set, J, Nt, nullptr,
                               Y + (int64_t)n_rep * D, Ystride, item_status, st));
        CIL_CU(launch_boot_tail(P, n_rep, D, ridge, out, item_status, Y, at<double>(wsa, B.L.off_mu),
                                at<double>(wsa, B.L.off_sig), st));
        return CIL_OK;
    }
    RowSrc ds{}, js{};
    ds.base = data; ds.stride = 0; ds.ld = ld_data; ds.rows = N_set; ds.mode = MODE_PLAIN;
    js.base = pools; js.stride = pool_stride; js.ld = ld; js.rows = Nt; js.mode = MODE_INDEXED;
    js.idx = J; js.idx_stride = Nt; js.idx_range = N_syn;
    SegParams sph{N_set, Nt, 1, 1};
    s = run_engines(P, ds, js, N_set, Nt, g, dist_mask, sl, M, B.ph, sph, B.L, wsa, radii, D, item_status, st,
                    nullptr, nullptr, /*keep_status=*/true);
    if (s != CIL_OK) return s;
    CIL_CU(launch_finalize_y(P, sl.nq, M, sph, at<uint64_t>(wsa, B.L.off_hist), Y + (int64_t)n_rep * D, Ystride,
                             (double)N_set * (double)Nt, st));
    // step 3 and 5: mu_theta, Sigma_theta over the n_rep vectors, loglik of y~
    CIL_CU(launch_boot_tail(P, n_rep, D, ridge, out, item_status, Y, at<double>(wsa, B.L.off_mu),
                            at<double>(wsa, B.L.off_sig), st));
    return CIL_OK;
}

cil_status cil_diag_gram(const float* A, int64_t lda, int64_t N, const float* B, int64_t ldb, int64_t Nt,
                         cil_grid g, cil_engine engine, float* d2E, void* ws, size_t ws_bytes, void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_diag_gram");
    if (N < 1 || Nt < 1 || !A || !B || !d2E || !ws) return CIL_EINVAL;
    if (engine != CIL_ENGINE_TC_3XBF16 && engine != CIL_ENGINE_TC_3XTF32 && engine != CIL_ENGINE_TC_I8)
        return CIL_EINVAL;
    if (check_grid(g, CIL_L2) != CIL_OK) return CIL_EINVAL;
    const int64_t K = (int64_t)g.S * g.H * g.W;
    if (lda < K || ldb < K) return CIL_EINVAL;
    if (K % 4 || lda % 4 || ldb % 4 || !aligned16(A) || !aligned16(B)) return CIL_EUNSUPPORTED;
    const Slots sl = slots_of(CIL_L2);
    const Plan pl = make_plan(CIL_L2, engine, g);
    if (!pl.tc) return CIL_EUNSUPPORTED;                  // rows beyond the engine's K segments
    SegParams sp{N, Nt, 1, 1};
    const Layout L = make_layout(1, N, Nt, g, sl.nq, 1, pl, sp, 0);
    if (ws_bytes < L.total + 512) return CIL_ENOMEM;
    void* wsa = reinterpret_cast<void*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    // a single dummy radius (the diagnostic path does not bin); it lives past the layout
    double* r = at<double>(wsa, L.total);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CIL_CU(launch_fill_f64(r, 1, 1.0, st));
    int32_t* status = reinterpret_cast<int32_t*>(r + 1);
    RowSrc as{}, bs{};
    as.base = A; as.ld = lda; as.rows = N; as.mode = MODE_PLAIN;
    bs.base = B; bs.ld = ldb; bs.rows = Nt; bs.mode = MODE_PLAIN;
    return run_engines(1, as, bs, N, Nt, g, CIL_L2, sl, 1, pl, sp, L, wsa, r, 0, status, st, d2E);
}

cil_status cil_diag_gram_family(const float* A, int64_t lda, int64_t N, const float* B, int64_t ldb, int64_t Nt,
                                cil_grid g, float* vE, void* ws, size_t ws_bytes, void* stream) {
    t_launches = 0;
    NvtxScope nv_("cil_diag_gram_family");
    if (N < 1 || Nt < 1 || !A || !B || !vE || !ws) return CIL_EINVAL;
    const uint32_t mask = CIL_L2 | CIL_W12SUM | CIL_W12;
    if (check_grid(g, mask) != CIL_OK) return CIL_EINVAL;
    const int64_t K = (int64_t)g.S * g.H * g.W;
    if (lda < K || ldb < K) return CIL_EINVAL;
    if (K % 4 || lda % 4 || ldb % 4 || !aligned16(A) || !aligned16(B)) return CIL_EUNSUPPORTED;
    const Slots sl = slots_of(mask);
    const int M = 1;
    const Plan pl = make_plan(mask, CIL_ENGINE_TC_I8, g, Nt, Nt, M);
    if (!pl.aug) return CIL_EUNSUPPORTED;
    SegParams sp{N, Nt, 1, 1};
    const Layout L = make_layout(1, N, Nt, g, sl.nq, M, pl, sp, 0);
    if (ws_bytes < L.total + 512) return CIL_ENOMEM;
    void* wsa = reinterpret_cast<void*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    double* r = at<double>(wsa, L.total);                 // one dummy radius per measure (not binned)
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CIL_CU(launch_fill_f64(r, 3, 1.0, st));
    int32_t* status = reinterpret_cast<int32_t*>(r + 3);
    RowSrc as{}, bs{};
    as.base = A; as.ld = lda; as.rows = N; as.mode = MODE_PLAIN;
    bs.base = B; bs.ld = ldb; bs.rows = Nt; bs.mode = MODE_PLAIN;
    return run_engines(1, as, bs, N, Nt, g, mask, sl, M, pl, sp, L, wsa, r, 0, status, st, vE);
}

const char* cil_status_string(cil_status s) {
    switch (s) {
        case CIL_OK: return "CIL_OK";
        case CIL_EINVAL: return "CIL_EINVAL: invalid argument";
        case CIL_EUNSUPPORTED: return "CIL_EUNSUPPORTED: valid request not supported by this build";
        case CIL_ENOMEM: return "CIL_ENOMEM: workspace too small";
        case CIL_ECUDA: return "CIL_ECUDA: CUDA launch failed (see cil_last_cuda_error)";
    }
    return "unknown cil_status";
}

void cil_prof_enable(int32_t on) { t_prof_on = on != 0; }

int32_t cil_prof_read(double* ms, int64_t* launches) {
    for (int c = 0; c < K_NCLASS; ++c) { ms[c] = 0.0; launches[c] = 0; }
    if (!t_prof) return 0;
    for (const ProfRec& r : *t_prof) {
        if (cudaEventSynchronize(r.b) != cudaSuccess) return -1;
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        ms[r.cls] += t;
        launches[r.cls] += 1;
        t_evpool->push_back(r.a);
        t_evpool->push_back(r.b);
    }
    t_prof->clear();
    return K_NCLASS;
}

void cil_diag_limit_recheck_list(int64_t limit) { t_list_limit = limit; }
void cil_diag_concurrent_engines(int32_t on) { t_concurrent = on != 0; }
void cil_diag_recheck_sort_min(int64_t n) { t_sort_min = n <= 0 ? 8192u : (uint32_t)(n > 0xffffffffll ? 0xffffffffll : n); }

int64_t cil_diag_bounds_violations(void) {
#ifdef CIL_BOUNDS_CHECK
    return (int64_t)oob_gram3() + oob_recheck() + oob_simt() + oob_max16();
#else
    return -1;
#endif
}

int32_t cil_last_cuda_error(void) { return t_last_cuda; }
int32_t cil_version(void) { return 100; }
int32_t cil_last_launch_count(void) { return t_launches; }

}  // extern "C"
