// gram3.cu — step a1 (pack) and a2 (L2 Gram + fused binning) of the hot path, default engine,
// and the L2-type family of SURVEY §8(f) 2, on tcgen05 kind::i8 with a WORST-CASE error bound.
//
// What it computes: for every pair (i, j) of an item, the L2 distance d = |a_i - b_j| of the caller's
// FP32 patterns (Eq. (5)) — or, in three-phase mode, the block distances of the
// augmented rows [x | D_x x | D_y x] that W12 (Eq. (8)) and W12SUM (Eq. (7)) are made of — and
// the count #{(i, j) : d < R_m} of Eq. (1) (strict <), without writing the N x Nt
// distance matrix anywhere.
//
// Representation (k_pack3_*): per row x~ = x - c (c = the item's centre, FP32), sigma = max|x~| / Q,
// q = rint(x~ / sigma) = 2^16 h + 2^8 m + l, int8 digits h in [-63, 63], m, l in [-128, 127]
// (22-bit fixed point, Q = 4 160 000).  Per-row metadata (8 floats):
//   n = sigma^2 sum q^2 (exact integer sum via dp4a of the digits), sigma,
//   r >= |x^ - (x - c)| with x^ = sigma q (quantisation AND FP32-centring residual, upper bound),
//   alpha >= sigma |l|, beta >= 2^8 sigma |m|.
// Gram (k_gram3): G' = 2^32 L32 + 2^24 L24 + 2^16 L16 with L32 = sum h_a h_b, L24 = sum (h_a m_b +
// m_a h_b), L16 = sum (h_a l_b + m_a m_b + l_a h_b) accumulated EXACTLY in three int32 TMEM
// accumulators, six MMAs per 32-byte K step (|L16| <= 32512 K < 2^31 for K <= 65536; longer K runs in
// chunks whose FP32 partials are summed in a fourth TMEM column block).  The dropped digit products
// obey |G - G'| <= 2^8 (|m_a||l_b| + |l_a||m_b|) + |l_a||l_b| (Cauchy-Schwarz), so with the FP32
// evaluation d~^2 = n_a + n_b - 2 sigma_a sigma_b G':
//   |d_q^2 - d~^2| <= Delta = 2 (alpha_a alpha_b + alpha_a beta_b + beta_a alpha_b) + rel (n_a + n_b)
// (d_q = |x^_a - x^_b|; rel >= the FP32 rounding of d~^2) and |d - d_q| <= rho = r_a + r_b (triangle
// inequality), hence for EVERY input
//   d in [ sqrt(max(d~^2 - Delta, 0)) - rho ,  sqrt(d~^2 + Delta) + rho ]
// evaluated with directed rounding (__f*_rd / __f*_ru).  A pair is binned in-kernel when no radius
// lies in its interval; otherwise it is listed for the exact FP64 re-check (recheck.cu).  Counts are
// therefore those of the plain definition (reading R13).
//
// Kernel anatomy (persistent CTA pairs, cta_group::2, tiles of 256 A rows x TN B columns, TN = 128
// (64 for a narrow B panel); TMEM columns [0,TN) L32, [TN,2TN) L24, [2TN,3TN) L16, [3TN,4TN) the
// chunk partial):
//   warp 0      TMA producer: one 3-D box (64 K-bytes x rows x 3 planes, SWIZZLE_64B) for A and one
//               for B per stage, 4-6 stages
//   warp 1      TMEM allocator + single-thread MMA issuer (leader CTA)
//   warps 2..   epilogue (12 warps; 8 in three-phase mode): tcgen05.ld of the accumulators ->
//               interval of d -> binary search over the radii -> per-thread shared histograms
//               (fire-and-forget ATOMS, flushed per tile as warp sums -> u64 atomics), or the bins as
//               bytes (bootstrap bin matrices); ambiguous pairs -> the re-check list.
#include <cuda.h>
#include <stdio.h>

#include <algorithm>

#include "cil_internal.cuh"
#include "tc_common.cuh"

namespace cil {
namespace g3 {
using tc::cluster_rank;
using tc::cluster_sync;
using tc::fence_after;
using tc::fence_before;
using tc::mbar_arrive_remote;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::mbar_wait;
using tc::mbar_wait_cluster;
using tc::named_bar;
using tc::smem_u32;
using tc::tmem_ld16;

// Build-time experiment switch (never set in the product build; tools/g3_exp.sh):
//   1 = the epilogue only hands the accumulators back (MMA + operand feed alone)
//   2 = no TMA loads (MMA + epilogue on whatever the stages hold)   3 = both (MMA alone)
#ifndef CIL_G3_EXP
#define CIL_G3_EXP 0
#endif
constexpr int KS = 128;         // K bytes per pipeline stage (one SWIZZLE_128B row)
constexpr int AR = 128;         // A rows per CTA (M = 256 per CTA pair)
constexpr int TILE_M = 256;
constexpr int MAXSEG = kG3MaxSeg;

struct Params {
    int64_t rowsA, rowsB, a_off, b_off;
    int P, p0, np;
    int tiles_m, tiles_n, tiles_act, tn, skip;
    int nseg;
    int seg_end[MAXSEG];               // K-block (64 B) end of each segment
    uint8_t seg_ph[MAXSEG], seg_first[MAXSEG], seg_last[MAXSEG], seg_empty[MAXSEG];
    int nph;
    const float* meta;                 // [rows_tot][nph][8]
    const float* thr;                  // [P][8][M]: kind k (L2 R/sqrt(w), W12 R^2/w, W12SUM R/sqrt(w)) at
                                       // rows 2k (rounded down) and 2k+1 (rounded up)
    int64_t thr_stride;
    int M, nq, q_l2;
    int q_k[3];                        // histogram slots of L2, W12, W12SUM (-1: not requested)
    SegParams sp;
    unsigned long long* hist;
    uint4* list; uint32_t* ctr; uint32_t cap;
    float rel;                         // FP32 evaluation bound of d~^2 relative to n_a + n_b
    float ih_rd, ih_ru, ih2_rd, ih2_ru;  // 1/h, 1/h^2 rounded down / up
    float2* part;                      // three-phase: [2][P rowsA rowsB] (lo, hi) of phases 0 and 1
    uint8_t* binout;
    int bin_t;
    float* diag;                       // diagnostics: per pair (lo, hi), item 0 only, no binning
    int64_t hist_elems;                // bounds-checked builds only
};

#ifndef CIL_PACK_WAVES
#define CIL_PACK_WAVES 16    // k_pack3 CTAs launched per resident CTA slot (rows per CTA follow)
#endif
#ifndef CIL_PACK_STRIDED
#define CIL_PACK_STRIDED 1   // k_pack3: rows j + k G per CTA (0: contiguous row blocks, experiment builds)
#endif
#ifndef CIL_G3_NARROW
#define CIL_G3_NARROW 1  // ragged last column tile at MMA N = round_up(columns, 16) (0: experiment builds)
#endif
#ifndef CIL_G3_WIDE
#define CIL_G3_WIDE 0   // 0: six N = TN MMAs per K step (product); 1: four wide MMAs (experiment builds)
#endif
template <int TN, int MAXM, bool SEG, bool AUG> struct Geo3 {
    static constexpr int BR = TN / 2;                           // B rows per CTA (N = TN MMA)
    static constexpr int A_PL = AR * KS;                        // 16 KB per plane
    static constexpr int B_PL = BR * KS;
    // wide layout: B per CTA = X (TN rows of one plane; rank 0: h, rank 1: m — the two halves of the
    // N = 2 TN operand [B_h | B_m]) + Y / Z (this CTA's half of B_l / B_h, the N = TN operands)
    static constexpr int B_X = TN * KS;
    static constexpr int B_Y = BR * KS;
    static constexpr int STAGE_W = 3 * A_PL + B_X + 2 * B_Y;    // 80 KB (TN 128)
    static constexpr int STAGE_N = 3 * (A_PL + B_PL);           // 72 KB (TN 128)
    static constexpr int NEPI = 8;
    static constexpr int NET = 32 * NEPI;
    static constexpr int NTHR = 64 + NET;
    // per-thread histograms of u32 cells [word][thread] (bank = thread), byte-packed (a thread bins
    // <= 64 pairs per tile and kind, flushed every tile):
    //   no segments: byte (b & 3) of word b >> 2 counts bin b (three-phase: one array per kind);
    //   column segments: word b, byte l counts local segment l (a thread's <= 64 columns of a tile
    //   meet <= 4 segments of >= 21 columns; three-phase: one array per kind)
    static constexpr int NLOC = SEG ? 4 : 1;
    static constexpr int NKA = AUG ? 3 : 1;
    static constexpr int HWORDS = SEG ? (MAXM + 1) : (MAXM + 4) / 4;
    static constexpr int HIST = NKA * HWORDS * NET * 4;
    static constexpr int NPHM = AUG ? 3 : 1;
    static constexpr int COLB = NPHM * TN * 20;                 // float4 (sigma, n, alpha, beta) + r
    static constexpr int THRB = 3 * 2 * 2 * MAXM * 4;           // [kind][rd/ru][2 MAXM]
    static constexpr int FIXED = 1024 + 1024 + COLB + THRB + HIST;
    // the wide layout needs two of its stages next to the fixed region (not: segmented MAXM = 64)
    static constexpr bool WIDE = CIL_G3_WIDE && (227 * 1024 - FIXED) / STAGE_W >= 2;
    static constexpr int STAGE = WIDE ? STAGE_W : STAGE_N;
    static constexpr int FIT = (227 * 1024 - FIXED) / STAGE;
#ifdef CIL_G3_MAXSTAGES
    static constexpr int STAGES = FIT > CIL_G3_MAXSTAGES ? CIL_G3_MAXSTAGES : FIT;   // experiment builds only
#else
    static constexpr int STAGES = FIT > 4 ? 4 : FIT;
#endif
    static constexpr int SMEM = STAGES * STAGE + FIXED;
    static constexpr int TCOLS = 4 * TN <= 256 ? 256 : 512;
    static_assert(FIT >= 2, "shared memory");
};

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
// one digit plane (box 128 K-bytes x rows x 1 plane, plane z); both CTAs of the pair signal the leader's barrier
__device__ __forceinline__ void tma1(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar) & 0xFEFFFFFFu)
        : "memory");
}
// 3-D TMA box (128 K-bytes x rows x 3 digit planes, SWIZZLE_128B); both CTAs of the pair signal the leader's barrier
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(0), "r"(smem_u32(bar) & 0xFEFFFFFFu)
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Tile enumeration.  With skipping, the active tiles of tile row mt are a suffix [start, tiles_n):
//   skip 1 (symmetric bin matrix, mirrored writes): the tiles holding a column >= the row tile's first row;
//   skip 2 (Alg. 1: blocks k < l only): the first tile whose last column lies in a later column
//          segment than the row tile's first row.
__host__ __device__ inline int row_start(int skip, int mt, int64_t row_seg, int64_t col_seg, int64_t rowsB, int tn) {
    if (skip == 1) return (int)((int64_t)mt * TILE_M / tn);
    const int64_t k0 = (int64_t)mt * TILE_M / row_seg;
    const int64_t need = (k0 + 1) * col_seg;
    if (need > rowsB - 1) return 1 << 30;
    return (int)(need / tn);
}
__host__ __device__ inline int tiles_active(int skip, int tiles_m, int tiles_n, int64_t row_seg, int64_t col_seg,
                                            int64_t rowsB, int tn) {
    if (skip == 0) return tiles_m * tiles_n;
    int n = 0;
    for (int mt = 0; mt < tiles_m; ++mt) {
        const int s = row_start(skip, mt, row_seg, col_seg, rowsB, tn);
        if (s < tiles_n) n += tiles_n - s;
    }
    return n;
}
// Without skipping the tiles of an item run in groups of up to 8 tile rows, column-major inside a group
// (row tile fastest): the clusters of one wave then share ~8 A tiles and ~9 B tiles, so both stay in
// L2 while the wave streams K — for long rows (C3, C5: one tile's planes exceed L2) this replaces a
// fresh B tile per cluster and wave.
constexpr int kGroupRows = 8;
__device__ __forceinline__ void tile_of(const Params& prm, int u, int& mt, int& nt) {
    if (prm.skip == 0) {
        const int per_group = kGroupRows * prm.tiles_n;
        const int g = u / per_group, r = u % per_group;
        const int rows_g = min(kGroupRows, prm.tiles_m - g * kGroupRows);
        mt = g * kGroupRows + r % rows_g;
        nt = r / rows_g;
        return;
    }
    for (mt = 0; mt < prm.tiles_m; ++mt) {
        const int s = row_start(prm.skip, mt, prm.sp.row_seg, prm.sp.col_seg, prm.rowsB, prm.tn);
        const int c = s < prm.tiles_n ? prm.tiles_n - s : 0;
        if (u < c) { nt = s + u; return; }
        u -= c;
    }
    mt = nt = 0;
}

// MMA N of column tile nt: the ragged last tile issues only round_up(its columns, 16) (M = 256 takes
// N % 16 == 0; each CTA of the pair then holds N / 2 B rows) — C4's swapped SCIL panel: 550 columns
// = 4 x 128 + 38 run the last tile at N = 48
template <int TN>
__device__ __forceinline__ int tile_n(const Params& prm, int nt) {
    if (!CIL_G3_NARROW) return TN;
    const int64_t left = prm.rowsB - (int64_t)nt * TN;
    return left >= TN ? TN : (int)((left + 15) / 16 * 16);
}

// b = #{m : v < T_m} over decreasing thresholds T[0..MAXM) padded with -inf to 2 MAXM
template <int MAXM>
__device__ __forceinline__ int bin_search(float v, const float* T) {
    int b = 0;
#pragma unroll
    for (int s = MAXM; s >= 1; s >>= 1)
        if (v < T[b + s - 1]) b += s;
    return b;
}

// Row metadata of one phase
struct RowV {
    float n, s, r, al, be;
};
__device__ __forceinline__ RowV row_meta(const float* meta, int64_t row, int nph, int ph) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(meta + (row * nph + ph) * 8));
    const float r = __ldg(meta + (row * nph + ph) * 8 + 4);
    RowV o;
    o.n = v.x; o.s = v.y; o.r = v.z; o.al = v.w; o.be = r;
    return o;
}

// sqrt with a rigorous one-sided bound: the hardware approximation (sqrt.approx.f32) inflated /
// deflated by 2^-21, directed rounding.  Its relative error is below 2^-22 for every normal input
// (checked exhaustively on the device: cil_diag_sqrt_approx_error, tests/test_gpu_parity.py);
// inputs below FLT_MIN are raised to it (upper) or give 0 (lower).
__device__ __forceinline__ float sqrt_up(float x) {
    float s;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(s) : "f"(fmaxf(x, 1.17549435e-38f)));
    return __fmul_ru(s, 1.000000476837158203125f);           // 1 + 2^-21
}
__device__ __forceinline__ float sqrt_dn(float x) {
    if (!(x >= 1.17549435e-38f)) return 0.f;
    float s;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(s) : "f"(x));
    return __fmul_rd(s, 0.999999523162841796875f);           // 1 - 2^-21
}

// Bounds of the squared distance of the quantised rows (see the header): lo2 <= d_q^2 <= hi2,
// and rho = r_a + r_b.  g = G' / 2^32 (FP32).  Every operation is symmetric in (a, b), so d(i, j)
// and d(j, i) give bit-identical results.
__device__ __forceinline__ void pair_interval(float g, const RowV& A, float sb, float nb, float alb, float beb,
                                              float rb, float rel, float& lo2, float& hi2, float& rho) {
    const float nn = A.n + nb;
    const float d2 = fmaf(A.s * sb * -8589934592.f, g, nn);           // -2^33 sigma_a sigma_b G'/2^32
    const float x = __fadd_ru(__fmul_ru(A.al, beb), __fmul_ru(A.be, alb));
    const float z = __fmaf_ru(A.al, alb, x);
    const float delta = __fmaf_ru(2.f, z, __fmul_ru(rel, nn));
    hi2 = __fadd_ru(d2, delta);
    lo2 = __fsub_rd(d2, delta);
    rho = __fadd_ru(A.r, rb);
}

// Epilogue (all modes).  Per tile: stage the column metadata and thresholds; per K segment, read
// the three accumulators, combine them (+ the running chunk partial) into one FP32 value per pair in
// TMEM columns [3TN, 4TN) and hand the accumulators back at once (the MMAs of the next segment or
// tile run while this one is binned); at a phase's last segment, bin from those columns, list
// ambiguous pairs, and finally flush the per-thread histograms.
template <int TN, int MAXM, bool SEG, bool AUG>
__device__ __forceinline__ void epilogue(const Params& prm, uint32_t tmem_base, uint64_t* tfull, uint64_t* tempty,
                                         float4* s_c4, float* s_cr, float* s_T, uint32_t* hist_s, int cluster_id,
                                         int n_clusters, int total_tiles, uint32_t rank, int warp, int lane) {
    using GG = Geo3<TN, MAXM, SEG, AUG>;
    constexpr int NET = GG::NET;
    const int quarter = warp & 3;
    const int ew = warp - 2;
    const int e0 = (quarter + 2) & 3;
    const int nwq = (GG::NEPI - e0 + 3) / 4;
    const int kq = ew >> 2;
    const int g0 = kq * (TN / 16) / nwq, g1 = (kq + 1) * (TN / 16) / nwq;
    const int ncol = (g1 - g0) * 16;
    const int et = threadIdx.x - 64;
    const int M = prm.M;
    const int nph = prm.nph;
    const int64_t npairs = (int64_t)prm.P * prm.rowsA * prm.rowsB;
    uint32_t* myh = hist_s + et;
    uint32_t tph = 0;
    for (int t = cluster_id; t < total_tiles; t += n_clusters) {
        const int p = prm.p0 + t / prm.tiles_act;
        int mt, nt;
        tile_of(prm, t % prm.tiles_act, mt, nt);
        const int64_t col0 = (int64_t)nt * TN;
        const int64_t browbase = prm.b_off + (int64_t)p * prm.rowsB;
        named_bar(1, NET);
        for (int i = et; i < nph * TN; i += NET) {
            const int ph = i / TN, c = i % TN;
            const int64_t j = col0 + c;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            float r = 0.f;
            if (j < prm.rowsB) {
                const RowV b = row_meta(prm.meta, browbase + j, nph, ph);
                v = make_float4(b.s, b.n, b.al, b.be);
                r = b.r;
            }
            s_c4[ph * TN + c] = v;
            s_cr[ph * TN + c] = r;
        }
        if (et < 2 * MAXM) {
            // kinds: 0 L2 (R/sqrt(w)), 1 W12 (R^2/w), 2 W12SUM (R/sqrt(w)); [kind][rd, ru][2 MAXM]
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const bool on = et < M && (AUG ? prm.q_k[k] >= 0 : k == 0);
                const float* T = prm.thr + (int64_t)p * prm.thr_stride;
                s_T[(k * 2 + 0) * 2 * MAXM + et] = on ? T[(2 * k) * M + et] : -INFINITY;
                s_T[(k * 2 + 1) * 2 * MAXM + et] = on ? T[(2 * k + 1) * M + et] : -INFINITY;
            }
        }
        named_bar(1, NET);
        const int64_t row = (int64_t)mt * TILE_M + rank * AR + quarter * 32 + lane;
        const bool row_ok = row < prm.rowsA;
        const int64_t arow = prm.a_off + (int64_t)p * prm.rowsA + (row_ok ? row : 0);
        const int hc0 = (int)(col0 + g0 * 16);
        const int nvalid = (int)min((int64_t)ncol, prm.rowsB - hc0);
        const uint32_t tl = tmem_base + ((uint32_t)(quarter * 32) << 16);
        const uint32_t tg = tl + 3 * TN;                         // combined FP32 values / chunk partials
        const int64_t cs_first = hc0 >= 0 ? (int64_t)hc0 / prm.sp.col_seg : 0;
        int bnd[GG::NLOC > 1 ? GG::NLOC - 1 : 1];
#pragma unroll
        for (int i = 0; i < GG::NLOC - 1; ++i) {
            const int64_t c = (cs_first + 1 + i) * prm.sp.col_seg - hc0;
            bnd[i] = SEG ? (int)(c < ncol ? c : (1 << 30)) : (1 << 30);
        }
        const bool diag_item = prm.diag != nullptr && p == 0;
        const bool no_bin = prm.diag != nullptr;
        // bin-matrix mode: symmetric layouts mirror tiles fully above the diagonal; in the diagonal
        // band both orders are computed here and the re-check list takes col >= row only
        const bool sym_up = prm.skip == 1 && (int64_t)(mt + 1) * TILE_M <= (int64_t)nt * TN;
        const bool sym_band = prm.skip == 1 && !sym_up;
        const int64_t pbase = (int64_t)p * prm.rowsA * prm.rowsB + (row_ok ? row : 0) * prm.rowsB;
        RowV A = row_meta(prm.meta, arow, nph, 0);

        for (int s = 0; s < prm.nseg; ++s) {
            const int ph = prm.seg_ph[s];
            const bool first = prm.seg_first[s], last = prm.seg_last[s], emp = prm.seg_empty[s];
            if (AUG && first && ph > 0) A = row_meta(prm.meta, arow, nph, ph);
            mbar_wait(&tfull[0], tph);
            fence_after();
            // ---- drain: g = 2^-32 G' (+ the running partial) into TMEM columns [3TN, 4TN)
#pragma unroll 1
            for (int gi = 0; gi < ((CIL_G3_EXP & 1) ? 0 : g1 - g0); ++gi) {
                if (gi * 16 >= nvalid) break;                       // warp-uniform
                const int tcol = (g0 + gi) * 16;
                uint32_t vr[16];
                if (emp) {
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) vr[jj] = 0u;
                } else {
                    uint32_t v32[16], v24[16], v16[16];
                    tmem_ld16(tl + tcol, v32);
                    tmem_ld16(tl + TN + tcol, v24);
                    tmem_ld16(tl + 2 * TN + tcol, v16);
                    if (!first) tmem_ld16(tg + tcol, vr);
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        float gv = fmaf((float)(int)v16[jj], 1.52587890625e-05f,
                                        fmaf((float)(int)v24[jj], 0.00390625f, (float)(int)v32[jj]));
                        if (!first) gv += __uint_as_float(vr[jj]);
                        vr[jj] = __float_as_uint(gv);
                    }
                }
                tmem_st16(tg + tcol, vr);
            }
            tmem_wait_st();
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(&tempty[0], 0);      // the accumulators are free again
            tph ^= 1;
            if (!last || (CIL_G3_EXP & 1)) continue;
            // ---- a phase's last segment: intervals and bins from the combined values
            const float4* c4 = s_c4 + ph * TN;
            const float* cr = s_cr + ph * TN;
#pragma unroll 1
            for (int gi = 0; gi < g1 - g0; ++gi) {
                if (gi * 16 >= nvalid) break;                       // warp-uniform
                const int tcol = (g0 + gi) * 16;
                uint32_t vr[16];
                tmem_ld16(tg + tcol, vr);
                if (!row_ok) continue;
                if (!AUG) {
                    // ---- one phase: the L2 distance; bin on the upper end, list if a radius is inside
                    const float* Tlo = s_T;                      // kind 0, rounded down
                    const float* Thi = s_T + 2 * MAXM;           // kind 0, rounded up
                    int bins[16];
                    uint32_t amb = 0;
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const int jc = tcol + jj;
                        const float4 cb = c4[jc];
                        float lo2, hi2, rho;
                        pair_interval(__uint_as_float(vr[jj]), A, cb.x, cb.y, cb.z, cb.w, cr[jc], prm.rel, lo2, hi2, rho);
                        const float up = __fadd_ru(sqrt_up(hi2), rho);
                        if (diag_item) {
                            if (gi * 16 + jj < nvalid) {
                                const float dn = fmaxf(__fsub_rd(sqrt_dn(lo2), rho), 0.f);
                                float* dg = prm.diag + ((int64_t)row * prm.rowsB + hc0 + gi * 16 + jj) * 2;
                                dg[0] = dn;
                                dg[1] = up;
                            }
                            continue;
                        }
                        const int b = bin_search<MAXM>(up, Tlo);
                        // a radius R_b possibly above d: d >= sqrt(lo2) - rho, so d < R_b is possible iff
                        // sqrt(lo2) < R_b + rho  <=>  lo2 < (R_b + rho)^2
                        const float u = __fadd_ru(Thi[b], rho);
                        const bool a = u > 0.f && lo2 < __fmul_ru(u, u);
                        int lcs = 0;
                        if (SEG) {
#pragma unroll
                            for (int i = 0; i < GG::NLOC - 1; ++i) lcs += (gi * 16 + jj >= bnd[i]) ? 1 : 0;
                        }
                        bins[jj] = b | (lcs << 8);
                        amb |= (a && gi * 16 + jj < nvalid) ? (1u << jj) : 0u;
                    }
                    if (no_bin) continue;
                    if (prm.binout != nullptr) {
                        const int64_t mb = ((int64_t)p * prm.nq + prm.q_l2) * prm.rowsA * prm.rowsB;
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            if (gi * 16 + jj >= nvalid) break;
                            const int64_t col = hc0 + gi * 16 + jj;
                            const uint8_t bv = (uint8_t)(bins[jj] & 255);
                            CIL_CHECK(row < prm.rowsA && col < prm.rowsB && mb + prm.rowsA * prm.rowsB <=
                                      (int64_t)prm.P * prm.nq * prm.rowsA * prm.rowsB);
                            if (prm.bin_t) prm.binout[mb + col * prm.rowsA + row] = bv;
                            else prm.binout[mb + row * prm.rowsB + col] = bv;
                            if (sym_up) prm.binout[mb + col * prm.rowsB + row] = bv;
                        }
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj)
                            if (gi * 16 + jj < nvalid)
                                atomicAdd(myh + (SEG ? (bins[jj] & 255) : ((bins[jj] & 255) >> 2)) * NET,
                                          SEG ? 1u << ((bins[jj] >> 5) & 24) : 1u << (8 * (bins[jj] & 3)));
                    }
                    if (amb) {
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            if (!((amb >> jj) & 1u)) continue;
                            const int64_t col = hc0 + gi * 16 + jj;
                            if (sym_band && col < row) continue;
                            const uint32_t idx = atomicAdd(prm.ctr, 1u);
                            if (idx < prm.cap)
                                prm.list[idx] = make_uint4((uint32_t)p, (uint32_t)row, (uint32_t)col,
                                                           (uint32_t)(bins[jj] & 255));   // kind 0 (L2)
                        }
                    }
                } else {
                    // ---- three phases: block intervals; phases 0, 1 parked, phase 2 forms the measures
#pragma unroll 4
                    for (int jj = 0; jj < 16; ++jj) {
                        if (gi * 16 + jj >= nvalid) break;
                        const int jc = tcol + jj;
                        const int64_t col = hc0 + gi * 16 + jj;
                        const float4 cb = c4[jc];
                        float lo2, hi2, rho;
                        pair_interval(__uint_as_float(vr[jj]), A, cb.x, cb.y, cb.z, cb.w, cr[jc], prm.rel, lo2, hi2, rho);
                        const float up = __fadd_ru(sqrt_up(hi2), rho);
                        const float dn = fmaxf(__fsub_rd(sqrt_dn(lo2), rho), 0.f);
                        const int64_t pi = pbase + col;
                        if (ph < 2) {
                            CIL_CHECK(pi >= 0 && pi < npairs && col < prm.rowsB);
                            prm.part[ph * npairs + pi] = make_float2(dn, up);
                            continue;
                        }
                        const float2 p0 = prm.part[pi], p1 = prm.part[npairs + pi];
                        int lcs = 0;
                        if (SEG) {
#pragma unroll
                            for (int i = 0; i < GG::NLOC - 1; ++i) lcs += (gi * 16 + jj >= bnd[i]) ? 1 : 0;
                        }
#pragma unroll
                        for (int k = 0; k < 3; ++k) {
                            if (prm.q_k[k] < 0) continue;
                            float vlo, vhi;
                            if (k == 0) {                        // L2 / sqrt(w) = d_0
                                vlo = p0.x; vhi = p0.y;
                            } else if (k == 1) {                 // W12^2 / w = d_0^2 + (d_x^2 + d_y^2) / h^2
                                vlo = __fmaf_rd(__fmaf_rd(p1.x, p1.x, __fmul_rd(dn, dn)), prm.ih2_rd, __fmul_rd(p0.x, p0.x));
                                vhi = __fmaf_ru(__fmaf_ru(p1.y, p1.y, __fmul_ru(up, up)), prm.ih2_ru, __fmul_ru(p0.y, p0.y));
                            } else {                             // W12SUM / sqrt(w) = d_0 + (d_x + d_y) / h
                                vlo = __fmaf_rd(__fadd_rd(p1.x, dn), prm.ih_rd, p0.x);
                                vhi = __fmaf_ru(__fadd_ru(p1.y, up), prm.ih_ru, p0.y);
                            }
                            if (diag_item) {
                                float* dg = prm.diag + (((int64_t)k * prm.rowsA + row) * prm.rowsB + col) * 2;
                                dg[0] = vlo;
                                dg[1] = vhi;
                                continue;
                            }
                            if (no_bin) continue;
                            const float* Tlo = s_T + (k * 2) * 2 * MAXM;
                            const float* Thi = s_T + (k * 2 + 1) * 2 * MAXM;
                            const int b = bin_search<MAXM>(vhi, Tlo);
                            if (prm.binout != nullptr) {
                                uint8_t* bm = prm.binout + ((int64_t)p * prm.nq + prm.q_k[k]) * prm.rowsA * prm.rowsB;
                                CIL_CHECK(row < prm.rowsA && col < prm.rowsB && prm.q_k[k] < prm.nq);
                                bm[row * prm.rowsB + col] = (uint8_t)b;
                                if (sym_up) bm[col * prm.rowsB + row] = (uint8_t)b;
                                if (sym_band && col < row) continue;
                            } else if (SEG) {
                                atomicAdd(myh + (k * GG::HWORDS + b) * NET, 1u << (8 * lcs));
                            } else {
                                atomicAdd(myh + (k * GG::HWORDS + (b >> 2)) * NET, 1u << (8 * (b & 3)));
                            }
                            if (vlo < Thi[b]) {
                                const uint32_t idx = atomicAdd(prm.ctr, 1u);
                                // measure ids (bit order): L2 0, W12SUM 2, W12 3
                                const uint32_t kind = k == 0 ? 0u : k == 1 ? 3u : 2u;
                                if (idx < prm.cap)
                                    prm.list[idx] = make_uint4((uint32_t)p, (uint32_t)row, (uint32_t)col,
                                                               (uint32_t)b | (kind << 8));
                            }
                        }
                    }
                }
            }
        }
        if (prm.binout != nullptr || no_bin) continue;
        // ---- flush the per-thread histograms (warp sums -> global u64 atomics) and reset them
        const int64_t rs = row_ok ? row / prm.sp.row_seg : 0;
        const int64_t rs0 = __shfl_sync(0xffffffffu, rs, 0);
        const bool uniform = __all_sync(0xffffffffu, rs == rs0 || !row_ok);
        for (int bb = 0; bb <= M; ++bb) {
#pragma unroll
            for (int k = 0; k < GG::NKA; ++k) {
                const int wd = SEG ? bb : (bb >> 2);
                uint32_t* cp = myh + (k * GG::HWORDS + wd) * NET;
                const uint32_t cell = *cp;
                if (SEG || (bb & 3) == 3 || bb == M) *cp = 0u;   // word done: reset
                const int q = AUG ? prm.q_k[k] : prm.q_l2;
                if (bb == 0 || q < 0) continue;                  // bin 0 (outside every radius) is not kept
#pragma unroll
                for (int l = 0; l < GG::NLOC; ++l) {
                    const int64_t cs = cs_first + l;
                    if (cs * prm.sp.col_seg >= prm.rowsB || cs * prm.sp.col_seg >= hc0 + ncol) break;
                    const uint32_t v = SEG ? ((cell >> (8 * l)) & 255u) : ((cell >> (8 * (bb & 3))) & 255u);
                    CIL_CHECK(hist_index(prm.sp, prm.nq, M, p, uniform ? rs0 : rs, cs, q, bb) < prm.hist_elems &&
                              cs < prm.sp.n_cs && (uniform ? rs0 : rs) < prm.sp.n_rs);
                    if (uniform) {
                        const uint32_t tot = __reduce_add_sync(0xffffffffu, v);
                        if (lane == 0 && tot)
                            atomicAdd(&prm.hist[hist_index(prm.sp, prm.nq, M, p, rs0, cs, q, bb)],
                                      (unsigned long long)tot);
                    } else if (v) {
                        atomicAdd(&prm.hist[hist_index(prm.sp, prm.nq, M, p, rs, cs, q, bb)], (unsigned long long)v);
                    }
                }
            }
        }
    }
}

template <int TN, int MAXM, bool SEG, bool AUG>
__global__ void __launch_bounds__(Geo3<TN, MAXM, SEG, AUG>::NTHR, 1)
k_gram3(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
        const __grid_constant__ CUtensorMap mB2, Params prm) {
    using GG = Geo3<TN, MAXM, SEG, AUG>;
    constexpr int STAGES = GG::STAGES;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* stages = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * GG::STAGE);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    float4* s_c4 = reinterpret_cast<float4*>(smem + STAGES * GG::STAGE + 1024);
    float* s_cr = reinterpret_cast<float*>(s_c4 + GG::NPHM * TN);
    float* s_T = s_cr + GG::NPHM * TN;
    uint32_t* hist_s = reinterpret_cast<uint32_t*>(s_T + 3 * 2 * 2 * MAXM);   // GG::HIST bytes

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int cluster_id = blockIdx.x / 2, n_clusters = gridDim.x / 2;
    const int total_tiles = prm.np * prm.tiles_act;
    const int n_kb = prm.seg_end[prm.nseg - 1];

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(&tfull[0], 1);
        mbar_init(&tempty[0], 2 * GG::NEPI);                 // epilogue warps x 2 CTAs
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mB) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mB2) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(GG::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (warp >= 2)
        for (int i = threadIdx.x - 64; i < GG::HIST / 4; i += GG::NET) hist_s[i] = 0u;
    fence_before();
    cluster_sync();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cluster_id; t < total_tiles; t += n_clusters) {
                const int p = prm.p0 + t / prm.tiles_act;
                int mt, nt;
                tile_of(prm, t % prm.tiles_act, mt, nt);
                const int ya = (int)(prm.a_off + p * prm.rowsA + (int64_t)mt * TILE_M + rank * AR);
                const int yb = (int)(prm.b_off + p * prm.rowsB + (int64_t)nt * TN +
                                     (GG::WIDE ? 0 : rank * (tile_n<TN>(prm, nt) / 2)));
                for (int kb = 0; kb < n_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char* st = stages + stage * GG::STAGE;
                    if (CIL_G3_EXP & 2) {
                        if (rank == 0) mbar_expect_tx(&full[stage], 0);
                    } else if (!GG::WIDE && (CIL_G3_EXP & 12)) {       // experiment: only B (4) / only A (8)
                        if (rank == 0) mbar_expect_tx(&full[stage], (CIL_G3_EXP & 4) ? 2 * 3 * GG::B_PL : 2 * 3 * GG::A_PL);
                        if (CIL_G3_EXP & 8) tma3(st, &mA, &full[stage], kb * KS, ya);
                        else tma3(st + 3 * GG::A_PL, &mB, &full[stage], kb * KS, yb);
                    } else {
                        if (rank == 0) mbar_expect_tx(&full[stage], 2 * GG::STAGE);
                        tma3(st, &mA, &full[stage], kb * KS, ya);
                        if constexpr (GG::WIDE) {
                            unsigned char* sbp = st + 3 * GG::A_PL;
                            tma1(sbp, &mB, &full[stage], kb * KS, yb, (int)rank);                            // X: h | m
                            tma1(sbp + GG::B_X, &mB2, &full[stage], kb * KS, yb + (int)rank * GG::BR, 2);       // Y: l
                            tma1(sbp + GG::B_X + GG::B_Y, &mB2, &full[stage], kb * KS, yb + (int)rank * GG::BR, 0);  // Z: h
                        } else {
                            tma3(st + 3 * GG::A_PL, &mB, &full[stage], kb * KS, yb);
                        }
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            const uint32_t id = idesc_i8(TILE_M, TN);
            const uint32_t id2 = idesc_i8(TILE_M, 2 * TN);
            (void)id2;
            const uint32_t d32 = tmem_base, d24 = tmem_base + TN, d16 = tmem_base + 2 * TN;
            int stage = 0;
            uint32_t phase = 0, tph = 0;
            for (int t = cluster_id; t < total_tiles; t += n_clusters) {
                uint32_t idt = id;
                if constexpr (!GG::WIDE) {
                    int mt_, nt_;
                    tile_of(prm, t % prm.tiles_act, mt_, nt_);
                    idt = idesc_i8(TILE_M, tile_n<TN>(prm, nt_));
                }
                for (int s = 0; s < prm.nseg; ++s) {
                    mbar_wait_cluster(&tempty[0], tph ^ 1);
                    fence_after();
                    const int kb0 = s ? prm.seg_end[s - 1] : 0, kb1 = prm.seg_end[s];
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        fence_after();
                        const uint32_t sa = smem_u32(stages + stage * GG::STAGE);
                        const uint32_t sb = sa + 3 * GG::A_PL;
                        const uint64_t ah = tc::sdesc(sa), am = tc::sdesc(sa + GG::A_PL), al = tc::sdesc(sa + 2 * GG::A_PL);
                        if constexpr (GG::WIDE) {
                            // [H | X] = A_h [B_h | B_m]; L = A_h B_l; [X | L] += A_m [B_h | B_m]; L += A_l B_h:
                            // the six digit products in four MMAs, A_h read twice instead of three times
                            const uint64_t bx = tc::sdesc(sb), by = tc::sdesc(sb + GG::B_X),
                                           bz = tc::sdesc(sb + GG::B_X + GG::B_Y);
#pragma unroll
                            for (int k = 0; k < KS / 32; ++k) {          // 32 int8 of K per MMA
                                const uint64_t adv = (uint64_t)(k * 2);  // +32 B in the start-address field
                                const uint32_t acc = (kb != kb0 || k != 0) ? 1u : 0u;
                                mma_i8(d32, ah + adv, bx + adv, id2, acc);
                                mma_i8(d16, ah + adv, by + adv, id, acc);
                                mma_i8(d24, am + adv, bx + adv, id2, 1u);
                                mma_i8(d16, al + adv, bz + adv, id, 1u);
                            }
                        } else {
                            const uint64_t bh = tc::sdesc(sb), bm = tc::sdesc(sb + GG::B_PL),
                                           bl = tc::sdesc(sb + 2 * GG::B_PL);
#pragma unroll
                            for (int k = 0; k < KS / 32; ++k) {          // 32 int8 of K per MMA
                                const uint64_t adv = (uint64_t)(k * 2);  // +32 B in the start-address field
                                const uint32_t acc = (kb != kb0 || k != 0) ? 1u : 0u;
                                mma_i8(d32, ah + adv, bh + adv, idt, acc);
                                mma_i8(d24, ah + adv, bm + adv, idt, acc);
                                mma_i8(d24, am + adv, bh + adv, idt, 1u);
                                mma_i8(d16, ah + adv, bl + adv, idt, acc);
                                mma_i8(d16, am + adv, bm + adv, idt, 1u);
                                mma_i8(d16, al + adv, bh + adv, idt, 1u);
                            }
                        }
                        tc::mma_commit<2>(&empty[stage]);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    tc::mma_commit<2>(&tfull[0]);
                    tph ^= 1;
                }
            }
        }
    } else {
        epilogue<TN, MAXM, SEG, AUG>(prm, tmem_base, tfull, tempty, s_c4, s_cr, s_T, hist_s, cluster_id, n_clusters,
                                     total_tiles, rank, warp, lane);
    }
    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(GG::TCOLS));
    }
}

// ------------------------------------------------------------------------------------ pack
#ifndef CIL_Q4_EXP
#define CIL_Q4_EXP 0     // 1: the earlier digit extraction (experiment builds)
#endif
// Quantisation constant: |q| <= Q (1 + 2^-22) < 2^22 (the magic-constant rint is exact) and
// (q + 128) >> 8 in [-16250, 16250], so h = (t1 + 128) >> 8 in [-63, 63].
constexpr float kQ = 4160000.f;
// Rows whose centred maximum lies outside [2^-38, 2^40] would under/overflow FP32 in the epilogue;
// they are packed as exact-only (r = +inf: every pair of theirs goes to the FP64 re-check).
constexpr float kMinMax = 3.637978807091713e-12f, kMaxMax = 1.099511627776e12f;

// Quantise 4 values: q = rint(t / sigma) by one FFMA with the 1.5 * 2^23 constant (exact rint of
// t * inv for |t * inv| < 2^22), raw = its bit pattern = q + 0x4B400000.  The balanced digits come
// straight from byte lanes: l = byte 0 of q = byte 0 of raw, m = byte 1 of (q + 128) = byte 1 of
// (raw + 128), h = byte 2 of (q + 32896) = byte 2 of (raw - 0x4B3F7F80) (q = 2^16 h + 2^8 m + l,
// h = (q + 32896) >> 16, m = ((q + 128) >> 8) - 2^8 h).  Digit words are gathered with byte
// permutes; S[0..5] += the exact digit dot products (hh, hm, hl, mm, ml, ll) by dp4a.
__device__ __forceinline__ void quant4(const float4 t, float inv, uint32_t& wh, uint32_t& wm, uint32_t& wl,
                                       int (&S)[6]) {
    const uint32_t r0 = __float_as_uint(fmaf(t.x, inv, 12582912.f));
    const uint32_t r1 = __float_as_uint(fmaf(t.y, inv, 12582912.f));
    const uint32_t r2 = __float_as_uint(fmaf(t.z, inv, 12582912.f));
    const uint32_t r3 = __float_as_uint(fmaf(t.w, inv, 12582912.f));
    const uint32_t c = 0x4B3F7F80u;
#if CIL_Q4_EXP == 1
    wl = __byte_perm(__byte_perm(r0, r1, 0x0040), __byte_perm(r2, r3, 0x0040), 0x5410);
    wm = __byte_perm(__byte_perm(r0 + 128u, r1 + 128u, 0x0051), __byte_perm(r2 + 128u, r3 + 128u, 0x0051), 0x5410);
    wh = __byte_perm(__byte_perm(r0 - c, r1 - c, 0x0062), __byte_perm(r2 - c, r3 - c, 0x0062), 0x5410);
#else
    // u = raw - c = q + 32896 = 2^16 h + 2^8 (m + 128) + (l + 128): bytes 0 / 1 are l / m biased by 128
    // (XOR 0x80 gives the two's-complement digit), byte 2 is h — one IADD per value for all three
    const uint32_t u0 = r0 - c, u1 = r1 - c, u2 = r2 - c, u3 = r3 - c;
    const uint32_t x = __byte_perm(u0, u1, 0x5140), y = __byte_perm(u2, u3, 0x5140);   // (l0 l1 m0 m1), (l2 l3 m2 m3)
    wl = __byte_perm(x, y, 0x5410) ^ 0x80808080u;
    wm = __byte_perm(x, y, 0x7632) ^ 0x80808080u;
    wh = __byte_perm(__byte_perm(u0, u1, 0x0062), __byte_perm(u2, u3, 0x0062), 0x5410);
#endif
    S[0] = __dp4a((int)wh, (int)wh, S[0]);
    S[1] = __dp4a((int)wh, (int)wm, S[1]);
    S[2] = __dp4a((int)wh, (int)wl, S[2]);
    S[3] = __dp4a((int)wm, (int)wm, S[3]);
    S[4] = __dp4a((int)wm, (int)wl, S[4]);
    S[5] = __dp4a((int)wl, (int)wl, S[5]);
}

// NaN-propagating 3-input |.|-max (FMNMX3 with |.| operands): a NaN input poisons the row maximum
__device__ __forceinline__ float absmax3_nan(float m, float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(m), "f"(fabsf(a)), "f"(fabsf(b)));
    return r;
}

// Row metadata from the block's digit sums (one thread).  cnt = elements of the block; tslack =
// extra FP32-rounding slack of the block values beyond the centring of the values themselves
// (derivative blocks: 2^-24 * 2 |x~|, see k_pack3_aug).  The quantisation residual is bounded
// analytically: q = rint(t inv) gives |t - sigma q| <= sigma/2 + delta |t| with delta = |1 - sigma inv|
// (exact in FP64), so |e| <= (sigma/2 sqrt(cnt) + delta sqrt(n)) / (1 - delta) (|t| <= sqrt(n) + |e|);
// the centring t = fl(x - c) adds <= 2^-24 |t| per element.
__device__ __forceinline__ void write_meta(float* out, float sg, float inv, const long long (&S)[6], double cnt,
                                           double tslack, bool exact_only, double tnorm_exact_only) {
    // sum q^2 = 2^32 hh + 2^25 hm + 2^17 hl + 2^16 mm + 2^9 ml + ll, exactly
    const long long Q = S[0] * (1ll << 32) + S[1] * (1ll << 25) + S[2] * (1ll << 17) + S[3] * (1ll << 16) +
                        S[4] * (1ll << 9) + S[5];
    const double s = (double)sg;
    const double n = (double)Q * s * s;
    const double delta = fabs(1.0 - (double)sg * (double)inv);
    const double e = (0.5 * s * sqrt(cnt) + delta * sqrt(n)) / (1.0 - delta);
    const double r = exact_only ? INFINITY
                                : (e + 5.9604644775390625e-08 * 1.001 * (sqrt(n) + e) + tslack) * (1.0 + 1e-9);
    (void)tnorm_exact_only;
    out[0] = (float)n;
    out[1] = sg;
    out[2] = __double2float_ru(r);
    out[3] = __double2float_ru(s * sqrt((double)S[5]) * (1.0 + 1e-12));
    out[4] = __double2float_ru(256.0 * s * sqrt((double)S[3]) * (1.0 + 1e-12));
    out[5] = 0.f; out[6] = 0.f; out[7] = 0.f;
}

// A CTA packs rpc consecutive rows of one item, each row whole in registers (NV float4 per thread,
// NT threads): x~ = x - c, max, quantise, store the three digit planes, exact digit sums.  The item's
// centre row is staged in shared memory once per CTA (re-reading it from L2 for every row cost ~16 %
// of the pack: an experiment build without centre loads took the C2 pack 1.02 -> 0.86 ms); thread 0
// prefetches the CTA's next row into L2 (cp.async.bulk.prefetch) while the current one is reduced /
// quantised / stored.
template <int NV, int NT>
__global__ void __launch_bounds__(NT) k_pack3(RowSrc src, int64_t rows, int64_t K, int64_t Kp, const float* __restrict__ center,
                                              int8_t* __restrict__ planes, int64_t plane_stride, int64_t row0,
                                              float* __restrict__ meta, int32_t* __restrict__ status, int rpc) {
    extern __shared__ float4 cs[];                        // the item's centre row, NV * NT float4 (0 past K)
    const int64_t p = blockIdx.y;
#if CIL_PACK_STRIDED
    // CTA j of the item packs rows j, j + G, j + 2G, ... (G = gridDim.x): the CTAs resident at any
    // moment work on neighbouring rows (a compact DRAM frontier), each still reusing its centre row
    const int64_t G = gridDim.x, rb = blockIdx.x, re = rows;
#else
    const int64_t G = 1, rb = (int64_t)blockIdx.x * rpc, re = min(rows, rb + rpc);
#endif
    const float* c = center + p * Kp;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int64_t k = ((int64_t)i * NT + threadIdx.x) * 4;
        cs[i * NT + threadIdx.x] = k < K ? __ldg(reinterpret_cast<const float4*>(c + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (threadIdx.x == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row_ptr(src, p, rb)), "r"((uint32_t)(K * 4)) : "memory");
    __syncthreads();
    __shared__ float red[NT / 32];
    __shared__ long long redl[NT / 32][6];
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    for (int64_t r = rb; r < re; r += G) {
        const float* x = row_ptr(src, p, r);
        const int64_t orow = row0 + p * rows + r;
        if (threadIdx.x == 0 && r + G < re)             // the CTA's next row streams into L2 meanwhile
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row_ptr(src, p, r + G)),
                         "r"((uint32_t)(K * 4)) : "memory");

        float4 v[NV];
        float mx = 0.f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int64_t k = ((int64_t)i * NT + threadIdx.x) * 4;
            if (k < K) {
                const float4 xv = __ldg(reinterpret_cast<const float4*>(x + k));
                const float4 cv = cs[i * NT + threadIdx.x];
                v[i] = make_float4(xv.x - cv.x, xv.y - cv.y, xv.z - cv.z, xv.w - cv.w);
            } else {
                v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            mx = absmax3_nan(absmax3_nan(mx, v[i].x, v[i].y), v[i].z, v[i].w);
        }
        for (int o = 16; o > 0; o >>= 1) {
            const float t = __shfl_xor_sync(0xffffffffu, mx, o);
            asm("max.NaN.f32 %0, %0, %1;" : "+f"(mx) : "f"(t));
        }
        if (ln == 0) red[w] = mx;
        __syncthreads();
        mx = 0.f;
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) asm("max.NaN.f32 %0, %0, %1;" : "+f"(mx) : "f"(red[i]));
        const bool nonfinite = !(mx <= 3.0e38f);                    // NaN or Inf somewhere in the row
        const bool ok = mx >= kMinMax && mx <= kMaxMax;
        const bool exact_only = mx > 0.f && !ok;
        const float sg = ok ? mx / kQ : 1.f;
        const float inv = 1.f / sg;
        int S[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int64_t k = ((int64_t)i * NT + threadIdx.x) * 4;
            if (k >= Kp) continue;
            uint32_t wh = 0, wm = 0, wl = 0;
            if (ok) quant4(v[i], inv, wh, wm, wl, S);
            int8_t* o = planes + orow * Kp + k;
            CIL_CHECK(orow * Kp + k + 4 <= plane_stride);
            *reinterpret_cast<uint32_t*>(o) = wh;
            *reinterpret_cast<uint32_t*>(o + plane_stride) = wm;
            *reinterpret_cast<uint32_t*>(o + 2 * plane_stride) = wl;
        }
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            long long a = S[i];
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (ln == 0) redl[w][i] = a;
        }
        __syncthreads();      // (red is re-written only after every thread has passed this barrier)
        if (threadIdx.x == 0) {
            long long Sl[6];
            for (int i = 0; i < 6; ++i) {
                long long a = 0;
                for (int j = 0; j < NT / 32; ++j) a += redl[j][i];
                Sl[i] = a;
            }
            write_meta(meta + orow * 8, sg, inv, Sl, (double)K, 0.0, exact_only, 0.0);
            if (nonfinite) atomicOr(&status[p], CIL_ITEM_NONFINITE);
        }
    }
}

// Rows too long for registers (K > 32768): pass 1 streams the row for max|x~|, pass 2 re-reads it
// (L2-resident: one row per CTA) to quantise.  Same arithmetic as k_pack3.
__global__ void __launch_bounds__(1024) k_pack3_2p(RowSrc src, int64_t rows, int64_t K, int64_t Kp,
                                                   const float* __restrict__ center, int8_t* __restrict__ planes,
                                                   int64_t plane_stride, int64_t row0, float* __restrict__ meta,
                                                   int32_t* __restrict__ status) {
    constexpr int NT = 1024;
    const int64_t p = blockIdx.y;
    const int64_t r = blockIdx.x;
    const float* x = row_ptr(src, p, r);
    const float* c = center + p * Kp;
    const int64_t orow = row0 + p * rows + r;
    __shared__ float red[NT / 32];
    __shared__ long long redl[NT / 32][6];
    float mx = 0.f;
    for (int64_t k = (int64_t)threadIdx.x * 4; k < K; k += NT * 4) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(x + k));
        const float4 cv = __ldg(reinterpret_cast<const float4*>(c + k));
        mx = absmax3_nan(absmax3_nan(mx, xv.x - cv.x, xv.y - cv.y), xv.z - cv.z, xv.w - cv.w);
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float t = __shfl_xor_sync(0xffffffffu, mx, o);
        asm("max.NaN.f32 %0, %0, %1;" : "+f"(mx) : "f"(t));
    }
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (ln == 0) red[w] = mx;
    __syncthreads();
    mx = 0.f;
    for (int i = 0; i < NT / 32; ++i) asm("max.NaN.f32 %0, %0, %1;" : "+f"(mx) : "f"(red[i]));
    const bool nonfinite = !(mx <= 3.0e38f);
    const bool ok = mx >= kMinMax && mx <= kMaxMax;
    const bool exact_only = mx > 0.f && !ok;
    const float sg = ok ? mx / kQ : 1.f;
    const float inv = 1.f / sg;
    int S[6] = {0, 0, 0, 0, 0, 0};
    long long SL[6] = {0, 0, 0, 0, 0, 0};
    int cnt = 0;
    for (int64_t k = (int64_t)threadIdx.x * 4; k < Kp; k += NT * 4) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < K) {
            const float4 xv = __ldg(reinterpret_cast<const float4*>(x + k));
            const float4 cv = __ldg(reinterpret_cast<const float4*>(c + k));
            v = make_float4(xv.x - cv.x, xv.y - cv.y, xv.z - cv.z, xv.w - cv.w);
        }
        uint32_t wh = 0, wm = 0, wl = 0;
        if (ok) quant4(v, inv, wh, wm, wl, S);
        int8_t* o = planes + orow * Kp + k;
        CIL_CHECK(orow * Kp + k + 4 <= plane_stride);
        *reinterpret_cast<uint32_t*>(o) = wh;
        *reinterpret_cast<uint32_t*>(o + plane_stride) = wm;
        *reinterpret_cast<uint32_t*>(o + 2 * plane_stride) = wl;
        if (++cnt == 64) {                                  // keep the int32 digit sums far from overflow
            for (int i = 0; i < 6; ++i) { SL[i] += S[i]; S[i] = 0; }
            cnt = 0;
        }
    }
    for (int i = 0; i < 6; ++i) {
        long long a = SL[i] + S[i];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (ln == 0) redl[w][i] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long Sl[6];
        for (int i = 0; i < 6; ++i) {
            long long a = 0;
            for (int j = 0; j < NT / 32; ++j) a += redl[j][i];
            Sl[i] = a;
        }
        write_meta(meta + orow * 8, sg, inv, Sl, (double)K, 0.0, exact_only, 0.0);
        if (nonfinite) atomicOr(&status[p], CIL_ITEM_NONFINITE);
    }
}

// Three-phase pack: row x~ = x - c expanded into the blocks value x~ (K), D_x x~ = x~[s][r][c+1] -
// x~[s][r][c] (S H (W-1)) and D_y x~ = x~[s][r+1][c] - x~[s][r][c] (S (H-1) W) (forward differences,
// last node omitted, reading R3; raw differences, 1/h applied to the distances; species masked by
// g.gs get 0 derivatives, reading R18), each quantised with its own scale into the three planes at
// columns kp[a] + idx.  Residual bound of a derivative block: the FP32 difference of FP32-centred
// values deviates from the exact (x - c) difference by <= 2^-24 (|D x~| + |x~_1| + |x~_0|) per
// element, hence the slack norm |D x~| + 2 |x~|.
__global__ void __launch_bounds__(256) k_pack3_aug(RowSrc src, int64_t rows, AugGeom g, int64_t kp0, int64_t kp1,
                                                   int64_t kp2, int64_t kp3, const float* __restrict__ center,
                                                   int64_t Kc, int8_t* __restrict__ planes, int64_t plane_stride,
                                                   int64_t Krow, int64_t row0, float* __restrict__ meta,
                                                   int32_t* __restrict__ status) {
    const int64_t p = blockIdx.y;
    const int64_t r = blockIdx.x;
    const float* x = row_ptr(src, p, r);
    const float* c = center + p * Kc;
    const int64_t orow = row0 + p * rows + r;
    const int W = g.W, H = g.H, SH = g.S * g.H;
    __shared__ float red[3][8];
    __shared__ long long redd[8][3][6];
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    auto xt = [&](int64_t e) -> float { return __ldg(x + e) - __ldg(c + e); };
    float m0 = 0.f, mx = 0.f, my = 0.f, nfa = 0.f;
    for (int sr = w; sr < SH; sr += 8) {
        const bool grad = g.gs == 0 || ((g.gs >> (sr / H)) & 1u);
        const bool has_dy = grad && (sr % H) + 1 < H;
        const int64_t base = (int64_t)sr * W;
        for (int c0 = 0; c0 < W; c0 += 32) {
            const int col = c0 + ln;
            const bool in = col < W;
            const float xv = in ? __ldg(x + base + col) : 0.f;
            nfa = fmaf(xv, 0.f, nfa);
            const float xe = in ? xv - __ldg(c + base + col) : 0.f;
            float xn = __shfl_down_sync(0xffffffffu, xe, 1);
            if (ln == 31 && col + 1 < W) xn = xt(base + col + 1);
            m0 = fmaxf(m0, fabsf(xe));
            if (grad && col + 1 < W) mx = fmaxf(mx, fabsf(xn - xe));
            if (has_dy && in) my = fmaxf(my, fabsf(xt(base + W + col) - xe));
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        my = fmaxf(my, __shfl_xor_sync(0xffffffffu, my, o));
    }
    const bool anynf = __syncthreads_or(nfa != nfa);
    if (ln == 0) { red[0][w] = m0; red[1][w] = mx; red[2][w] = my; }
    __syncthreads();
    float sg[3], inv[3];
    bool ex[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float m = 0.f;
        for (int i = 0; i < 8; ++i) m = fmaxf(m, red[a][i]);
        const bool ok = m >= kMinMax && m <= kMaxMax;
        ex[a] = m > 0.f && !ok;
        sg[a] = ok ? m / kQ : 1.f;
        inv[a] = 1.f / sg[a];
    }
    int8_t* ph = planes + orow * Krow;
    int S[3][6];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int i = 0; i < 6; ++i) S[a][i] = 0;
    // one value at a time (the block layouts are not 4-aligned); digits from the byte lanes of the
    // rint result (see quant4)
    auto put = [&](int a, int64_t col, float v) {
        int hh = 0, mm = 0, ll = 0;
        if (!ex[a]) {
            const uint32_t raw = __float_as_uint(fmaf(v, inv[a], 12582912.f));
            ll = (int)(signed char)(raw & 255u);
            mm = (int)(signed char)(((raw + 128u) >> 8) & 255u);
            hh = (int)(signed char)(((raw - 0x4B3F7F80u) >> 16) & 255u);
            S[a][0] += hh * hh; S[a][1] += hh * mm; S[a][2] += hh * ll;
            S[a][3] += mm * mm; S[a][4] += mm * ll; S[a][5] += ll * ll;
        }
        ph[col] = (int8_t)hh;
        ph[col + plane_stride] = (int8_t)mm;
        ph[col + 2 * plane_stride] = (int8_t)ll;
    };
    for (int sr = w; sr < SH; sr += 8) {
        const int s = sr / H;
        const bool grad = g.gs == 0 || ((g.gs >> s) & 1u);
        const bool has_dy = (sr % H) + 1 < H;
        const int64_t base = (int64_t)sr * W;
        for (int c0 = 0; c0 < W; c0 += 32) {
            const int col = c0 + ln;
            const bool in = col < W;
            const float xe = in ? xt(base + col) : 0.f;
            float xn = __shfl_down_sync(0xffffffffu, xe, 1);
            if (ln == 31 && col + 1 < W) xn = xt(base + col + 1);
            if (!in) continue;
            put(0, kp0 + base + col, xe);
            put(1, kp1 + base + col, grad && col + 1 < W ? xn - xe : 0.f);   // D_x rows padded to W
            if (has_dy) put(2, kp2 + base - (int64_t)s * W + col, grad ? xt(base + W + col) - xe : 0.f);
        }
    }
    const int64_t len[3] = {g.K, g.Kx, g.Ky}, beg[3] = {kp0, kp1, kp2}, end[3] = {kp1, kp2, kp3};
    const int64_t used[3] = {g.K, g.K, g.Ky};                   // D_x rows padded to W
#pragma unroll
    for (int a = 0; a < 3; ++a)
        for (int64_t col = beg[a] + used[a] + threadIdx.x; col < end[a]; col += 256) {
            ph[col] = 0; ph[col + plane_stride] = 0; ph[col + 2 * plane_stride] = 0;
        }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            long long v = S[a][i];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (ln == 0) redd[w][a][i] = v;
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        // value block first: its centred norm bounds the FP32 slack of the derivative blocks
        // (|fl(t1 - t0) - exact| <= 2^-24 (|D x~| + |t1| + |t0|) per element, |t| <= sqrt(n_0) + r_0)
        double tnorm = 0.0;
        for (int a = 0; a < 3; ++a) {
            long long Sl[6];
            for (int i = 0; i < 6; ++i) {
                long long v = 0;
                for (int j = 0; j < 8; ++j) v += redd[j][a][i];
                Sl[i] = v;
            }
            const double slack = a == 0 ? 0.0 : 2.0 * 5.9604644775390625e-08 * 1.001 * tnorm;
            float* out = meta + (orow * 3 + a) * 8;
            write_meta(out, sg[a], inv[a], Sl, (double)len[a], slack, ex[a], 0.0);
            if (a == 0) tnorm = sqrt((double)out[0]) * (1.0 + 1e-6) + (double)out[2];
        }
        if (anynf) atomicOr(&status[p], CIL_ITEM_NONFINITE);
    }
}

// k_pack3_aug for W % 4 == 0: a flat float4 sweep (4 elements of one grid row per thread, the
// x neighbour of the 4th from the next lane, the y neighbours one grid row on from L1 / L2), two
// passes (maxima, then quantise + store; the second reads the row from L2), one 32-bit store per
// plane and 4 values (the D_x rows are padded to W, so every block is 4-aligned).  Same values,
// digits, sums and metadata as k_pack3_aug.
__global__ void __launch_bounds__(512, 2) k_pack3_aug4(RowSrc src, int64_t rows, AugGeom g, int64_t kp0, int64_t kp1,
                                                    int64_t kp2, int64_t kp3, const float* __restrict__ center,
                                                    int64_t Kc, int8_t* __restrict__ planes, int64_t plane_stride,
                                                    int64_t Krow, int64_t row0, float* __restrict__ meta,
                                                    int32_t* __restrict__ status) {
    constexpr int NT = 512, NW = NT / 32;
    const int64_t p = blockIdx.y;
    const int64_t r = blockIdx.x;
    const float* x = row_ptr(src, p, r);
    const float* cc = center + p * Kc;
    const int64_t orow = row0 + p * rows + r;
    const uint32_t W = (uint32_t)g.W, H = (uint32_t)g.H, K = (uint32_t)g.K;
    const FastDiv fw(W), fh(H);
    __shared__ float red[3][NW];
    __shared__ long long redd[NW][3][6];
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    // one float4 of x~ = x - c and its derivative float4s (0 where there is no neighbour / masked)
    auto load = [&](uint32_t e, float4& t, float4& dx, float4& dy) {
        const bool ok = e < K;
        t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok) {
            const float4 xv = __ldg(reinterpret_cast<const float4*>(x + e));
            const float4 cv = __ldg(reinterpret_cast<const float4*>(cc + e));
            t = make_float4(xv.x - cv.x, xv.y - cv.y, xv.z - cv.z, xv.w - cv.w);
        }
        float nx = __shfl_down_sync(0xffffffffu, t.x, 1);
        dx = dy = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!ok) return;
        uint32_t c, hr;
        const uint32_t sr = fw.div(e, c), sp = fh.div(sr, hr);
        if (!(g.gs == 0 || ((g.gs >> sp) & 1u))) return;
        if (c + 4 < W && ln == 31) nx = (__ldg(x + e + 4) - __ldg(cc + e + 4));
        dx = make_float4(t.y - t.x, t.z - t.y, t.w - t.z, c + 4 < W ? nx - t.w : 0.f);
        if (hr + 1 < H) {
            const float4 xv = __ldg(reinterpret_cast<const float4*>(x + e + W));
            const float4 cv = __ldg(reinterpret_cast<const float4*>(cc + e + W));
            dy = make_float4((xv.x - cv.x) - t.x, (xv.y - cv.y) - t.y, (xv.z - cv.z) - t.z, (xv.w - cv.w) - t.w);
        }
    };
    float m0 = 0.f, mx = 0.f, my = 0.f;
    for (uint32_t base = 0; base < K; base += NT * 4) {
        float4 t, dx, dy;
        load(base + threadIdx.x * 4, t, dx, dy);
        m0 = absmax3_nan(absmax3_nan(m0, t.x, t.y), t.z, t.w);
        mx = fmaxf(fmaxf(mx, fmaxf(fabsf(dx.x), fabsf(dx.y))), fmaxf(fabsf(dx.z), fabsf(dx.w)));
        my = fmaxf(fmaxf(my, fmaxf(fabsf(dy.x), fabsf(dy.y))), fmaxf(fabsf(dy.z), fabsf(dy.w)));
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float t = __shfl_xor_sync(0xffffffffu, m0, o);
        asm("max.NaN.f32 %0, %0, %1;" : "+f"(m0) : "f"(t));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        my = fmaxf(my, __shfl_xor_sync(0xffffffffu, my, o));
    }
    if (ln == 0) { red[0][w] = m0; red[1][w] = mx; red[2][w] = my; }
    __syncthreads();
    float sg[3], inv[3];
    bool ex[3];
    bool anynf = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float m = 0.f;
        for (int i = 0; i < NW; ++i) {
            if (a == 0) asm("max.NaN.f32 %0, %0, %1;" : "+f"(m) : "f"(red[a][i]));
            else m = fmaxf(m, red[a][i]);
        }
        if (a == 0) anynf = !(m <= 3.0e38f);
        const bool ok = m >= kMinMax && m <= kMaxMax;
        ex[a] = m > 0.f && !ok;
        sg[a] = ok ? m / kQ : 1.f;
        inv[a] = 1.f / sg[a];
    }
    int8_t* ph = planes + orow * Krow;
    int S[3][6];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int i = 0; i < 6; ++i) S[a][i] = 0;
    auto put4 = [&](int a, int64_t col, const float4 v) {
        uint32_t wh = 0, wm = 0, wl = 0;
        if (!ex[a]) quant4(v, inv[a], wh, wm, wl, S[a]);
        CIL_CHECK(orow * Krow + col + 4 <= plane_stride);
        *reinterpret_cast<uint32_t*>(ph + col) = wh;
        *reinterpret_cast<uint32_t*>(ph + col + plane_stride) = wm;
        *reinterpret_cast<uint32_t*>(ph + col + 2 * plane_stride) = wl;
    };
    for (uint32_t base = 0; base < K; base += NT * 4) {
        const uint32_t e = base + threadIdx.x * 4;
        float4 t, dx, dy;
        load(e, t, dx, dy);
        if (e >= K) continue;
        uint32_t c, hr;
        const uint32_t sr = fw.div(e, c), sp = fh.div(sr, hr);
        (void)c;
        put4(0, kp0 + e, t);
        put4(1, kp1 + e, dx);
        if (hr + 1 < H) put4(2, kp2 + (int64_t)e - (int64_t)sp * W, dy);
    }
    const int64_t len[3] = {g.K, g.Kx, g.Ky}, beg[3] = {kp0, kp1, kp2}, end[3] = {kp1, kp2, kp3};
    const int64_t used[3] = {g.K, g.K, g.Ky};
#pragma unroll
    for (int a = 0; a < 3; ++a)
        for (int64_t col = beg[a] + used[a] + threadIdx.x; col < end[a]; col += NT) {
            ph[col] = 0; ph[col + plane_stride] = 0; ph[col + 2 * plane_stride] = 0;
        }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            long long v = S[a][i];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (ln == 0) redd[w][a][i] = v;
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tnorm = 0.0;
        for (int a = 0; a < 3; ++a) {
            long long Sl[6];
            for (int i = 0; i < 6; ++i) {
                long long v = 0;
                for (int j = 0; j < NW; ++j) v += redd[j][a][i];
                Sl[i] = v;
            }
            const double slack = a == 0 ? 0.0 : 2.0 * 5.9604644775390625e-08 * 1.001 * tnorm;
            float* out = meta + (orow * 3 + a) * 8;
            write_meta(out, sg[a], inv[a], Sl, (double)len[a], slack, ex[a], 0.0);
            if (a == 0) tnorm = sqrt((double)out[0]) * (1.0 + 1e-6) + (double)out[2];
        }
        if (anynf) atomicOr(&status[p], CIL_ITEM_NONFINITE);
    }
}

}  // namespace g3

// ------------------------------------------------------------------ host side
cudaError_t launch_pack3(int P, const RowSrc& src, int64_t rows, int64_t K, int64_t Kp, const float* center,
                         int8_t* planes, int64_t plane_stride, int64_t row0, float* meta, int32_t* status,
                         cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    dim3 grid((unsigned)rows, (unsigned)P);
    ProfScope ps_(K_PACK, st);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // rows per CTA: the centre row is read once per CTA; about 16 waves of resident CTAs remain (C2:
    // 6 rows per CTA; A/B: 4, 8, 32, 64 waves and a cap of 8 rows were slower or equal; without the
    // next-row prefetch the C2 pack takes 1.07 ms, with a second row prefetched 1.22 ms)
    auto rpc_for = [&](const void* fn, int nt, size_t smem) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, smem);
        const int64_t ctas = (int64_t)nsm * (per_sm > 0 ? per_sm : 1) * CIL_PACK_WAVES;
        const int64_t r = (rows * P + ctas - 1) / ctas;
        return (int)(r < 1 ? 1 : r > 16 ? 16 : r);
    };
#define PACK3(NV, NT)                                                                                              \
    do {                                                                                                           \
        static SmemAttrOnce attr_;                                                                                 \
        const size_t smem_ = sizeof(float4) * (NV) * (NT);                                                         \
        if (cudaError_t e_ = attr_.ensure(g3::k_pack3<NV, NT>, (int)smem_); e_ != cudaSuccess) return e_;          \
        const int rpc_ = rpc_for((const void*)g3::k_pack3<NV, NT>, NT, smem_);                                    \
        dim3 g_((unsigned)((rows + rpc_ - 1) / rpc_), (unsigned)P);                                                \
        g3::k_pack3<NV, NT><<<g_, NT, smem_, st>>>(src, rows, K, Kp, center, planes, plane_stride, row0, meta,     \
                                                   status, rpc_);                                                  \
    } while (0)
    if (Kp <= 1024)
        PACK3(1, 256);
    else if (Kp <= 4096)
        PACK3(4, 256);
    else if (Kp <= 8192)
        PACK3(16, 128);          // C2: 1.008-1.012 ms vs 1.045-1.057 for 8 x 256 (round 2, three planes)
    else if (Kp <= 16384)
        PACK3(16, 256);          // C4: 6.03-6.09 ms vs 6.40-6.42 for 8 x 512 (round 2, three planes)
    else if (Kp <= 32768)
        PACK3(8, 1024);
    else
        g3::k_pack3_2p<<<grid, 1024, 0, st>>>(src, rows, K, Kp, center, planes, plane_stride, row0, meta, status);
#undef PACK3
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_pack3_aug(int P, const RowSrc& src, int64_t rows, const AugGeom& g, const int64_t* kp,
                             const float* center, int64_t Kc, int8_t* planes, int64_t plane_stride, int64_t row0,
                             float* meta, int32_t* status, cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    dim3 grid((unsigned)rows, (unsigned)P);
    ProfScope ps_(K_PACK, st);
    if (g.W % 4 == 0 && g.K < (1ll << 31))
        g3::k_pack3_aug4<<<grid, 512, 0, st>>>(src, rows, g, kp[0], kp[1], kp[2], kp[3], center, Kc, planes,
                                               plane_stride, kp[3], row0, meta, status);
    else
        g3::k_pack3_aug<<<grid, 256, 0, st>>>(src, rows, g, kp[0], kp[1], kp[2], kp[3], center, Kc, planes,
                                              plane_stride, kp[3], row0, meta, status);
    note_launch();
    return cudaGetLastError();
}

typedef CUresult (*PFN_encodeTiled_g3)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 3-D map over the digit planes [3][rows_tot][Kp] (u8): box 128 x box_rows x 3, SWIZZLE_128B
static bool make_map3(CUtensorMap* m, const void* base, int64_t rows_tot, int64_t Kp, int box_rows, int box_planes = 3) {
    static PFN_encodeTiled_g3 enc = nullptr;
    if (!enc) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
        enc = reinterpret_cast<PFN_encodeTiled_g3>(p);
    }
    cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows_tot, 3};
    cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)(rows_tot * Kp)};
    cuuint32_t box[3] = {(cuuint32_t)g3::KS, (cuuint32_t)box_rows, (cuuint32_t)box_planes};
    cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int TN, int MAXM, bool SEG, bool AUG>
static cudaError_t launch_g3_t(const g3::Params& prm, const CUtensorMap* maps, int nsm, cudaStream_t st) {
    using GG = g3::Geo3<TN, MAXM, SEG, AUG>;
    static SmemAttrOnce attr;
    if (cudaError_t e = attr.ensure(g3::k_gram3<TN, MAXM, SEG, AUG>, GG::SMEM); e != cudaSuccess) return e;
    const int64_t tiles = (int64_t)prm.np * prm.tiles_act;
    const int clusters = (int)(tiles < nsm / 2 ? tiles : nsm / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(clusters * 2));
    cfg.blockDim = dim3(GG::NTHR);
    cfg.dynamicSmemBytes = GG::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope ps_(K_GRAM_TC, st);
    // maps: [0] A (3 planes), [1] B (3 planes x TN/2 rows), [2] B (1 plane x TN rows), [3] B (1 plane x TN/2)
    cudaError_t e = GG::WIDE ? cudaLaunchKernelEx(&cfg, g3::k_gram3<TN, MAXM, SEG, AUG>, maps[0], maps[2], maps[3], prm)
                             : cudaLaunchKernelEx(&cfg, g3::k_gram3<TN, MAXM, SEG, AUG>, maps[0], maps[1], maps[1], prm);
    note_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <int TN, bool AUG>
static cudaError_t dispatch_g3(const g3::Params& prm, const CUtensorMap* maps, int nsm, cudaStream_t st, bool seg,
                               int M) {
    if (M <= 16) return seg ? launch_g3_t<TN, 16, true, AUG>(prm, maps, nsm, st) : launch_g3_t<TN, 16, false, AUG>(prm, maps, nsm, st);
    if constexpr (AUG) {
        if (seg) return cudaErrorInvalidValue;              // the host routes these to the CUDA cores
        if (M <= 32) return launch_g3_t<TN, 32, false, AUG>(prm, maps, nsm, st);
        return launch_g3_t<TN, 64, false, AUG>(prm, maps, nsm, st);
    } else {
        if (M <= 32) return seg ? launch_g3_t<TN, 32, true, AUG>(prm, maps, nsm, st) : launch_g3_t<TN, 32, false, AUG>(prm, maps, nsm, st);
        return seg ? launch_g3_t<TN, 64, true, AUG>(prm, maps, nsm, st) : launch_g3_t<TN, 64, false, AUG>(prm, maps, nsm, st);
    }
}

cudaError_t launch_gram3(const G3Args& a, cudaStream_t st) {
    if (a.rowsA == 0 || a.rowsB == 0) return cudaSuccess;
    if (a.rows_tot >= (1ll << 31) || a.Kp % g3::KS) return cudaErrorInvalidValue;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int tn = a.tn_force == 64 ? 64 : 128;
    if (tn == 64 && (a.skip != 0 || a.nph != 1)) return cudaErrorInvalidValue;
    CUtensorMap maps[4];
    if (!make_map3(&maps[0], a.planes, a.rows_tot, a.Kp, g3::AR) || !make_map3(&maps[1], a.planes, a.rows_tot, a.Kp, tn / 2) ||
        !make_map3(&maps[2], a.planes, a.rows_tot, a.Kp, tn, 1) || !make_map3(&maps[3], a.planes, a.rows_tot, a.Kp, tn / 2, 1))
        return cudaErrorInvalidValue;
    g3::Params prm{};
    prm.rowsA = a.rowsA; prm.rowsB = a.rowsB; prm.a_off = a.a_off; prm.b_off = a.b_off;
    prm.P = a.P; prm.p0 = a.p0; prm.np = a.np > 0 ? a.np : a.P - a.p0;
    prm.tn = tn; prm.skip = a.skip;
    prm.tiles_m = (int)((a.rowsA + g3::TILE_M - 1) / g3::TILE_M);
    prm.tiles_n = (int)((a.rowsB + tn - 1) / tn);
    prm.tiles_act = g3::tiles_active(a.skip, prm.tiles_m, prm.tiles_n, a.sp.row_seg, a.sp.col_seg, a.rowsB, tn);
    if (prm.tiles_act == 0) return cudaSuccess;
    // K segments: each phase's k-blocks in chunks of <= 65536 bytes (exact int32 accumulation)
    prm.nph = a.nph == 3 ? 3 : 1;
    int ns = 0, max_chunks = 1;
    for (int ph = 0; ph < prm.nph; ++ph) {
        const int kb0 = (int)(a.ph_beg[ph] / g3::KS), kb1 = (int)(a.ph_end[ph] / g3::KS);
        const int per = 65536 / g3::KS;
        const int nch = kb1 > kb0 ? (kb1 - kb0 + per - 1) / per : 1;
        max_chunks = std::max(max_chunks, nch);
        for (int c = 0; c < nch; ++c) {
            if (ns >= g3::MAXSEG) return cudaErrorInvalidValue;
            prm.seg_end[ns] = std::min(kb1, kb0 + (c + 1) * per);
            prm.seg_ph[ns] = (uint8_t)ph;
            prm.seg_first[ns] = c == 0;
            prm.seg_last[ns] = c == nch - 1;
            prm.seg_empty[ns] = kb1 == kb0;
            ++ns;
        }
        if (a.ph_beg[ph] != (ph ? a.ph_end[ph - 1] : 0)) return cudaErrorInvalidValue;   // contiguous phases
    }
    prm.nseg = ns;
    prm.meta = a.meta;
    prm.thr = a.thr; prm.thr_stride = a.thr_stride;
    prm.M = a.M; prm.nq = a.nq; prm.q_l2 = a.q_l2;
    for (int k = 0; k < 3; ++k) prm.q_k[k] = a.q_k[k];
    prm.sp = a.sp;
    prm.hist = reinterpret_cast<unsigned long long*>(a.hist);
    prm.list = a.list; prm.ctr = a.ctr; prm.cap = a.cap;
    // FP32 evaluation of d~^2 = n_a + n_b - 2 s G': n (1 ulp each), their sum, the sigma product,
    // the digit combination (3 ulp) and one per chunk partial, the FMA; 16 + chunks ulps covers it
    prm.rel = (float)ldexp(16.0 + 2.0 * max_chunks, -24);
    prm.ih_rd = a.ih_rd; prm.ih_ru = a.ih_ru; prm.ih2_rd = a.ih2_rd; prm.ih2_ru = a.ih2_ru;
    prm.part = reinterpret_cast<float2*>(a.part);
    prm.binout = a.binout;
    prm.bin_t = a.bin_t ? 1 : 0;
    if (a.bin_t && (a.skip != 0 || !a.binout || prm.nph != 1)) return cudaErrorInvalidValue;
    prm.diag = a.diag;
    prm.hist_elems = a.hist_elems;
    const bool seg = a.sp.col_seg < a.rowsB;
    if (seg && a.sp.col_seg < 21) return cudaErrorInvalidValue;
    if (tn == 64) {
        if (seg) return cudaErrorInvalidValue;
        if (a.M <= 16) return launch_g3_t<64, 16, false, false>(prm, maps, nsm, st);
        if (a.M <= 32) return launch_g3_t<64, 32, false, false>(prm, maps, nsm, st);
        return launch_g3_t<64, 64, false, false>(prm, maps, nsm, st);
    }
    if (prm.nph == 3) return dispatch_g3<128, true>(prm, maps, nsm, st, seg, a.M);
    return dispatch_g3<128, false>(prm, maps, nsm, st, seg, a.M);
}

CIL_OOB_READER(oob_gram3)

}  // namespace cil
