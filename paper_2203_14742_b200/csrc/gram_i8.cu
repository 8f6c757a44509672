// gram_i8.cu — step a2 of the hot path, INT8 variant (default engine): L2 distances (Eq. (5),
// PAPER.md:181) of all pairs through d^2 = |a~|^2 + |b~|^2 - 2 a~.b~ on tcgen05 kind::i8,
// fused with the radius binning of Eq. (1).
//
// Operands (pack.cu k_pack_i8): per row a~ = sigma (256 h + l), h, l int8, sigma = max|a~|/32639.
//   a~.b~ = sigma_a sigma_b (65536 HH + 256 (HL + LH) + LL),   HH = sum h_a h_b, ...
// HH and X = HL + LH are accumulated EXACTLY in two int32 TMEM accumulators (3 MMAs per 32-byte
// k-step); LL (< 2^-16 of the total, noise-like) is dropped and covered by the error bound.
// Exact integer accumulation: no drift with K (|X| <= 32512 K < 2^31 for K <= 65536).
// The only approximation is the operand quantisation (|delta| <= sigma/2 per element), whose
// effect on d^2 is bounded per pair by
//   E = k_q d sqrt((sigma_a^2 + sigma_b^2)/3) + k_ll sigma_a sigma_b sqrt(K) + rel (n_a + n_b);
// pairs with a threshold T_m = R_m^2/w inside (d^2 - E, d^2 + E] go to the exact FP64 re-check.
//
// Kernel anatomy (persistent CTA pairs, cta_group::2, 256 x TN tiles, TN in {256, 192, 64}):
//   warp 0      TMA producer (h and l tiles of A and B, 128-byte SWIZZLE_128B rows, 2-3 stages)
//   warp 1      TMEM allocator + single-thread MMA issuer (leader CTA): HH -> cols [0,TN),
//               HL, LH -> cols [TN,2 TN)
//   warps 2..15 epilogue (14 warps; 8 for the three-phase AUG engine): tcgen05.ld of H and X ->
//               FP32 d^2 and its bound E per pair -> binary search over the thresholds ->
//               per-thread shared histograms [bin][thread] (fire-and-forget ATOMS), flushed per
//               tile as warp sums -> u64 atomics per (row segment, column segment); or, in
//               bin-matrix mode, the bins as bytes (row-major, mirrored for a symmetric matrix,
//               or transposed); ambiguous pairs -> the re-check list.
//   mode 1      (bootstrap resample, epilogue_rowdot): h planes only, one MMA per k-step, TMEM
//               double-buffered, A row block resident, weights applied in the epilogue.
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>


#include <algorithm>
#include "cil_internal.cuh"
#include "tc_common.cuh"

namespace cil {
namespace tc {

struct I8Params {
    int64_t rowsA, rowsB;
    int64_t b_off;             // first B row in the stacked planes: P*rowsA, or 0 when B = A (packed once)
    int64_t a_off;             // first A row in the stacked planes (0 unless the caller places A after B)
    int P, p0, np;
    int n_kb;
    int tiles_m, tiles_n;
    const float* nrm;          // stacked [P*rowsA + P*rowsB]: sigma^2 sum q^2
    const float* scl;          // stacked: sigma
    const float* thr2;         // [P][M] R^2/w
    int64_t thr_stride;
    int M, nq, q_l2;
    SegParams sp;
    unsigned long long* hist;
    uint4* list; uint32_t* ctr; uint32_t cap;
    float kq, kll, rel;
    float* diag;
    uint8_t* binout;           // non-null: bins[p][q_l2][i][j] (provisional; re-check fixes ambiguous ones)
    int pf;                    // L2 prefetch distance of the TMA producer in k-blocks (0 = off)
    // three-phase mode (AUG): blocks value / D_x / D_y, k-block ends per phase
    int nph;
    int kb_end[3];
    const float* nrm3; const float* scl3;   // [rows][4]
    float kll3[3];
    float2* part;              // [2][P*rowsA*rowsB] (d2, E) of phases 0 and 1
    int q_tc[3];               // histogram slots of L2, W12, W12SUM (-1: absent)
    float ih;                  // 1/h
    int mode;                  // 0 binning; 1 row-dot (bootstrap replicate counts, see epilogue_rowdot)
    int bin_t;                 // bin-matrix mode: write binout transposed ([p][q][col][row], stride rowsA)
    const uint16_t* m2;        // mode 1: [P][rowsA][rd_nt] column-draw multiplicities
    int64_t rd_nt;             // mode 1: columns per threshold block (B row = v * rd_nt + b)
    int rd_m;                  // mode 1: thresholds
    unsigned long long* rd_out;   // mode 1: [P][rowsA][rd_m] counts (atomic sums)
    int tn;                    // B columns per tile (the kernel's TN)
    int tiles_act;             // active tiles per item (tiles_m * tiles_n without skipping)
    int skip;                  // 0 all tiles; 1 symmetric bin matrix (tiles mt > nt skipped, mirrored
                               // by mt < nt); 2 only tiles meeting a block k < l (Alg. 1 triangle)
    int dbg;                   // diagnostic timing knob (CIL_DEBUG_I8): 1 skip binning, 2 skip the epilogue,
                               // 3 also skip the B loads, 4 all loads; mode 1: 1 hand-off only,
                               // 5 no weight loads, 6 streaming ring instead of the resident A
};

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
// Instruction descriptor for kind::i8: S32 accumulate (2), signed int8 A/B (1), K-major, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int MAXM, bool SEG, bool AUG = false, int TN = 256> struct I8Geo {
    // tile = 256 A rows (CTA pair) x TN B columns (TN = 256, or 192 to cut padding of ~550-row
    // panels, or 64 for a narrow B panel such as Alg. A2's 50 s_data rows); each CTA stages 128
    // A rows and TN/2 B rows per 128-byte K block
    static constexpr int B_ROWS = TN / 2;
    static constexpr int A_BYTES = A_ROWS * ROW_BYTES;
    static constexpr int B_BYTES = B_ROWS * ROW_BYTES;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // 64 KB (TN 256) / 56 KB (TN 192)
    static constexpr int HALF = TN / 2;                             // columns per epilogue warp
    static constexpr int NG = HALF / 16;                            // 16-column TMEM groups per warp
    // per-thread histograms [bin][thread] of u32 cells (bank = thread, conflict-free); with column
    // segments (SCIL blocks of >= 43 columns, so a 128-column half meets <= 4) byte l of a cell
    // counts local segment l (<= 128 pairs per tile, flushed every tile).  AUG (three measure
    // kinds): without segments byte k of a cell counts kind k; with segments one cell array
    // per kind.
    static constexpr int NLOC = SEG ? 4 : 1;
    static constexpr int NKIND = AUG ? 3 : 1;
    // epilogue warps: 14 (3-4 per SM sub-partition, more latency hiding while the MMA waits)
    // for the one-phase engine, 8 for the three-phase one (its register budget)
    static constexpr int NEPI = AUG ? 8 : 14;
    static constexpr int NET = 32 * NEPI;                           // epilogue threads
    static constexpr int NTHR = 64 + NET;
    static constexpr int HIST_BYTES = (AUG && SEG ? 3 : 1) * (MAXM + 1) * NET * 4;
    static constexpr int FIXED = 1024 /*align*/ + 1024 /*barriers*/ + 3 * TN * 4 /*norms, sigma, spare*/ +
                                 NKIND * 2 * MAXM * 4 + HIST_BYTES;
    static constexpr int STAGES = (3 * STAGE_BYTES + FIXED <= 227 * 1024) ? 3 : 2;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + FIXED;
};

// Which tiles a launch computes.  With tile skipping the active tiles of a tile row mt are a
// suffix [start(mt), tiles_n) of the row, so they are enumerated compactly (no idle clusters):
//   skip 1 (symmetric bin matrix, mirrored writes): start = mt (upper triangle incl. diagonal);
//   skip 2 (Alg. 1: blocks k < l only): start = first tile whose last column lies in a later
//          column segment than the tile's first row's segment.
__host__ __device__ inline int tile_row_start(int skip, int mt, int64_t row_seg, int64_t col_seg, int64_t rowsB,
                                              int tn) {
    if (skip == 1) return mt;
    const int64_t k0 = (int64_t)mt * Geo<2>::TILE_M / row_seg;      // segment of the tile's first row
    // smallest nt with min((nt+1)*tn, rowsB) - 1 >= (k0 + 1) * col_seg
    const int64_t need = (k0 + 1) * col_seg;                         // first column of segment k0 + 1
    if (need > rowsB - 1) return 1 << 30;
    return (int)(need / tn);
}
__host__ __device__ inline int tiles_active(int skip, int tiles_m, int tiles_n, int64_t row_seg, int64_t col_seg,
                                            int64_t rowsB, int tn) {
    if (skip == 0) return tiles_m * tiles_n;
    int n = 0;
    for (int mt = 0; mt < tiles_m; ++mt) {
        const int s = tile_row_start(skip, mt, row_seg, col_seg, rowsB, tn);
        if (s < tiles_n) n += tiles_n - s;
    }
    return n;
}
__device__ __forceinline__ void tile_of(const I8Params& prm, int u, int& mt, int& nt) {
    if (prm.skip == 0) { mt = u / prm.tiles_n; nt = u % prm.tiles_n; return; }
    for (mt = 0; mt < prm.tiles_m; ++mt) {
        const int s = tile_row_start(prm.skip, mt, prm.sp.row_seg, prm.sp.col_seg, prm.rowsB, prm.tn);
        const int cnt = s < prm.tiles_n ? prm.tiles_n - s : 0;
        if (u < cnt) { nt = s + u; return; }
        u -= cnt;
    }
    mt = nt = 0;                                                     // not reached
}

// sqrt for the error bound (one SFU op, relative error ~2^-22: immaterial for a bound with a
// >= 4x measured margin); d^2 >= 1e-30 > FLT_MIN so no denormal handling is needed
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// b = #{m : v < T_m} for decreasing thresholds T[0..MAXM) padded with -inf to 2*MAXM
template <int MAXM>
__device__ __forceinline__ int bin_search(float v, const float* T) {
    int b = 0;
#pragma unroll
    for (int s = MAXM; s >= 1; s >>= 1)
        if (v < T[b + s - 1]) b += s;
    return b;
}

// Three-phase epilogue (the L2-type family on tensor cores): phase a drains the Gram of block a
// (value, D_x, D_y) into (d2_a, E_a); phases 0 and 1 park theirs in global memory (L2-resident
// partials), phase 2 forms
//   L2^2/w = d2_0,   W12^2/w = d2_0 + (d2_x + d2_y)/h^2,   W12SUM/sqrt(w) = sqrt d2_0 + (sqrt d2_x + sqrt d2_y)/h
// (Eqs. (5), (8), (7) with readings R1, R3) with their bounds, bins the requested ones and
// sends pairs with a threshold inside the bound to the FP64 re-check (kind in bits 8-15).
template <int MAXM, bool SEG, int TN>
__device__ __forceinline__ void epilogue_aug(const I8Params& prm, uint32_t tmem_base, uint64_t* tfull,
                                             uint64_t* tempty, float* s_nb, float* s_sb, float* s_T,
                                             uint32_t* hist_s, int cluster_id, int n_clusters, int total_tiles,
                                             int tiles_per_item, uint32_t rank, int warp, int lane) {
    using G = Geo<2>;
    using IG = I8Geo<MAXM, SEG, true, TN>;
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;
    const int M = prm.M;
    const int64_t npairs = (int64_t)prm.P * prm.rowsA * prm.rowsB;
    uint32_t tph = 0;
    for (int t = cluster_id; t < total_tiles; t += n_clusters) {
        const int p = prm.p0 + t / tiles_per_item;
        int mt, nt;
        tile_of(prm, t % tiles_per_item, mt, nt);
        const int64_t col0 = (int64_t)nt * TN;
        const int64_t browbase = prm.b_off + (int64_t)p * prm.rowsB;
        const int64_t row = (int64_t)mt * G::TILE_M + rank * A_ROWS + quarter * 32 + lane;
        const bool row_ok = row < prm.rowsA;
        const int64_t arow = prm.a_off + (int64_t)p * prm.rowsA + (row_ok ? row : 0);
        const int hc0 = (int)(col0 + half * IG::HALF);
        const int nvalid = (int)min((int64_t)IG::HALF, prm.rowsB - hc0);
        const uint32_t tl = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(half * IG::HALF);
        const int64_t cs_first = (int64_t)hc0 / prm.sp.col_seg;
        int bnd[IG::NLOC > 1 ? IG::NLOC - 1 : 1];
#pragma unroll
        for (int i = 0; i < IG::NLOC - 1; ++i) {
            const int64_t c = (cs_first + 1 + i) * prm.sp.col_seg - hc0;
            bnd[i] = SEG ? (int)(c < IG::HALF ? c : (1 << 30)) : (1 << 30);
        }
        uint32_t* myh = hist_s + et;
        const int64_t pbase = (int64_t)p * prm.rowsA * prm.rowsB + (row_ok ? row : 0) * prm.rowsB;
        for (int ph = 0; ph < 3; ++ph) {
            named_bar(1, 256);
            {
                const int64_t c = col0 + et;
                const bool ok = c < prm.rowsB;
                if (et < TN) {                   // the tile's TN columns (s_nb / s_sb hold TN each)
                    s_nb[et] = ok ? prm.nrm3[(browbase + c) * 4 + ph] : 0.f;
                    s_sb[et] = ok ? prm.scl3[(browbase + c) * 4 + ph] : 0.f;
                }
                if (ph == 0 && et < 2 * MAXM)
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        s_T[k * 2 * MAXM + et] = (et < M && prm.q_tc[k] >= 0)
                                                     ? prm.thr2[(int64_t)p * prm.thr_stride + k * M + et]
                                                     : -INFINITY;
            }
            named_bar(1, 256);
            const float na = row_ok ? __ldg(&prm.nrm3[arow * 4 + ph]) : 0.f;
            const float sa = row_ok ? __ldg(&prm.scl3[arow * 4 + ph]) : 0.f;
            const float kq_sa = prm.kq * 0.81649658f;
            const float kll_sa = prm.kll3[ph] * sa;
            const float m2sa = -2.f * sa;
            const bool empty_ph = prm.kb_end[ph] == (ph ? prm.kb_end[ph - 1] : 0);
            mbar_wait(&tfull[0], tph);
            fence_after();
#pragma unroll 1
            for (int g = 0; g < IG::NG; ++g) {
                if (g * 16 >= nvalid) break;
                uint32_t hv[16], xv[16];
                tmem_ld16(tl + g * 16, hv);
                tmem_ld16(tl + TN + g * 16, xv);
                if (!row_ok) continue;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    const int j = g * 16 + jj;
                    if (j >= nvalid) break;
                    const int jc = half * IG::HALF + j;
                    const float sb = s_sb[jc], nb = s_nb[jc];
                    const float gi = empty_ph ? 0.f : fmaf((float)(int)hv[jj], 65536.f, (float)(int)xv[jj] * 256.f);
                    const float d2 = fmaxf(fmaf(m2sa * sb, gi, na + nb), 0.f);
                    const float dd = fmaxf(d2, 1e-30f);
                    const float E = fmaf(kq_sa * sqrt_approx(dd), fmaxf(sa, sb), fmaf(kll_sa, sb, prm.rel * (na + nb)));
                    const int64_t pi = pbase + hc0 + j;
                    if (ph < 2) {
                        prm.part[ph * npairs + pi] = make_float2(d2, E);
                        continue;
                    }
                    const float2 p0 = prm.part[pi], p1 = prm.part[npairs + pi];
                    const float ih = prm.ih, ih2 = ih * ih;
                    int lcs = 0;
                    if (SEG) {
#pragma unroll
                        for (int i = 0; i < IG::NLOC - 1; ++i) lcs += (j >= bnd[i]) ? 1 : 0;
                    }
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        if (prm.q_tc[k] < 0) continue;
                        float v, e;
                        if (k == 0) {
                            v = p0.x; e = p0.y;
                        } else if (k == 1) {
                            v = p0.x + (p1.x + d2) * ih2;
                            e = p0.y + (p1.y + E) * ih2 + v * 2.4e-7f;
                        } else {
                            // |u - d| <= E  =>  |sqrt u - sqrt d| = |u - d| / (sqrt u + sqrt d)
                            //   <= min(sqrt E, E / (sqrt u + sqrt max(u - E, 0)))   (d >= u - E)
                            const float r0 = sqrtf(p0.x), rx = sqrtf(p1.x), ry = sqrtf(d2);
                            auto eb = [](float u, float r, float Eu) {
                                return fminf(sqrtf(Eu), Eu / fmaxf(r + sqrtf(fmaxf(u - Eu, 0.f)), 1e-30f));
                            };
                            const float e0 = eb(p0.x, r0, p0.y), ex = eb(p1.x, rx, p1.y), ey = eb(d2, ry, E);
                            v = r0 + (rx + ry) * ih;
                            e = e0 + (ex + ey) * ih + v * 2.4e-7f;
                        }
                        if (prm.diag != nullptr) {        // diagnostics: (value, bound) per kind, item 0
                            if (p == 0) {
                                float* dg = prm.diag + (((int64_t)k * prm.rowsA + row) * prm.rowsB + hc0 + j) * 2;
                                dg[0] = v;
                                dg[1] = e;
                            }
                            continue;
                        }
                        const float* T = s_T + k * 2 * MAXM;
                        const int b = bin_search<MAXM>(v + e, T);
                        if (prm.binout != nullptr) {      // bin-matrix mode (bootstrap), measure q_tc[k]
                            uint8_t* bm = prm.binout + ((int64_t)p * prm.nq + prm.q_tc[k]) * prm.rowsA * prm.rowsB;
                            const int64_t col = hc0 + j;
                            bm[row * prm.rowsB + col] = (uint8_t)b;
                            if (prm.skip == 1 && mt < nt) bm[col * prm.rowsB + row] = (uint8_t)b;   // mirror
                            // a diagonal tile of a symmetric matrix lists each unordered pair once
                            if (prm.skip == 1 && mt == nt && col < row) continue;
                        } else if (SEG) {
                            atomicAdd(myh + ((k * (MAXM + 1) + b) << 8), 1u << (8 * lcs));
                        } else {
                            atomicAdd(myh + (b << 8), 1u << (8 * k));
                        }
                        if (v - e < T[b]) {
                            const uint32_t idx = atomicAdd(prm.ctr, 1u);
                            if (idx < prm.cap)
                                prm.list[idx] = make_uint4((uint32_t)p, (uint32_t)row, (uint32_t)(hc0 + j),
                                                           (uint32_t)(b | (k << 8)));
                        }
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(&tempty[0], 0);
            tph ^= 1;
        }
        if (prm.binout != nullptr) continue;           // bin-matrix mode: no histograms
        // ---- flush the per-thread histograms of the requested kinds
        const int64_t rs = row_ok ? row / prm.sp.row_seg : 0;
        const int64_t rs0 = __shfl_sync(0xffffffffu, rs, 0);
        const bool uniform = __all_sync(0xffffffffu, rs == rs0 || !row_ok);
        for (int bb = 0; bb <= M; ++bb) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                uint32_t* cp = SEG ? myh + ((k * (MAXM + 1) + bb) << 8) : myh + (bb << 8);
                const uint32_t cell = *cp;
                if (SEG || k == 2) *cp = 0u;
                if (bb == 0 || prm.q_tc[k] < 0) continue;          // bin 0 (outside every radius) is not kept
#pragma unroll
                for (int l = 0; l < IG::NLOC; ++l) {
                    const int64_t cs = cs_first + l;
                    if (cs * prm.sp.col_seg >= prm.rowsB || cs * prm.sp.col_seg >= hc0 + IG::HALF) break;
                    const uint32_t v = SEG ? ((cell >> (8 * l)) & 255u) : ((cell >> (8 * k)) & 255u);
                    if (uniform) {
                        const uint32_t tot = __reduce_add_sync(0xffffffffu, v);
                        if (lane == 0 && tot)
                            atomicAdd(&prm.hist[hist_index(prm.sp, prm.nq, M, p, rs0, cs, prm.q_tc[k], bb)],
                                      (unsigned long long)tot);
                    } else if (v) {
                        atomicAdd(&prm.hist[hist_index(prm.sp, prm.nq, M, p, rs, cs, prm.q_tc[k], bb)],
                                  (unsigned long long)v);
                    }
                }
            }
        }
    }
}

// mode 1 barriers after tfull[6]: the streaming ring (2 STAGES full + 2 STAGES empty) or, with
// the A panel resident, a_full, a_empty, then kRdSlots B full + kRdSlots B empty
constexpr int kRdSlots = 16;
constexpr int kRdBars = 2 + 2 * kRdSlots;
// Tile sequence of one cluster in mode 1 (the same for producer, MMA and epilogue).
// Resident A: clusters form groups of tiles_m; cluster (g, mt) keeps tile row mt and walks the
// group's contiguous range of (item, nt) columns, so the tiles_m clusters of a group read each
// B tile at about the same time (one HBM read of B, A loaded once per item).  Streaming: the
// persistent stride of the other modes.
struct RdSeq {
    bool resA;
    int n, mt, c0, tiles_n, stride, first;
    __device__ __forceinline__ void init(const I8Params& prm, bool resA_, int cluster_id, int n_clusters,
                                         int total_tiles) {
        resA = resA_;
        tiles_n = prm.tiles_n;
        if (resA) {
            const int G = n_clusters / prm.tiles_m;
            const int g = cluster_id / prm.tiles_m;
            mt = cluster_id % prm.tiles_m;
            const int C = prm.np * prm.tiles_n;
            c0 = g < G ? (int)((int64_t)g * C / G) : 0;
            n = g < G ? (int)((int64_t)(g + 1) * C / G) - c0 : 0;
        } else {
            first = cluster_id;
            stride = n_clusters;
            n = cluster_id < total_tiles ? (total_tiles - 1 - cluster_id) / n_clusters + 1 : 0;
        }
    }
    __device__ __forceinline__ void get(const I8Params& prm, int i, int tiles_per_item, int& p, int& mt_, int& nt) const {
        if (resA) {
            const int c = c0 + i;
            p = prm.p0 + c / tiles_n;
            nt = c % tiles_n;
            mt_ = mt;
        } else {
            const int t = first + i * stride;
            p = prm.p0 + t / tiles_per_item;
            tile_of(prm, t % tiles_per_item, mt_, nt);
        }
    }
};
template <typename IG, int STAGES>
__device__ __forceinline__ bool rd_resident_a(const I8Params& prm, int n_clusters) {
    return prm.skip == 0 && prm.tiles_m <= n_clusters && prm.dbg != 6 &&     // dbg 6: streaming ring
           prm.n_kb * IG::A_BYTES + 2 * IG::B_BYTES <= STAGES * IG::STAGE_BYTES;
}

// Row-dot epilogue (mode 1, bootstrap replicate counts on the tensor cores): the Gram of one-
// digit operands is C[k][c] = sum_a M1[k][a] E[c][a] (replicate k's row-draw multiplicities
// against the 0/1 threshold rows E[v*Nt + b][a] = [bins(a, b) > v]); the epilogue forms
//   counts[k][v] = sum_b C[k][v*Nt + b] * M2[k][b]   (M2 = column-draw multiplicities)
// = #{(i, j) : bins(I1[k][i], I2[k][j]) > v}, exactly (integers), and adds it atomically.
template <int MAXM, bool SEG, int TN>
__device__ __forceinline__ void epilogue_rowdot(const I8Params& prm, uint32_t tmem_base, uint64_t* tfull,
                                                uint64_t* tempty, int cluster_id, int n_clusters, int total_tiles,
                                                int tiles_per_item, uint32_t rank, int warp, int lane) {
    using G = Geo<2>;
    using IG = I8Geo<MAXM, SEG, false, TN>;
    const int quarter = warp & 3;
    const int ew = warp - 2;
    const int e0 = (quarter + 2) & 3;
    const int nwq = (IG::NEPI - e0 + 3) / 4;
    const int kq = ew >> 2;
    const int g0 = kq * (TN / 16) / nwq, g1 = (kq + 1) * (TN / 16) / nwq;
    const int ncol = (g1 - g0) * 16;
    // B rows are b-major: row (bt, v, i) = bt M TN + v TN + i holds column b = bt TN + i of
    // threshold v, so tile nt is (bt, v) = (nt / M, nt % M), all its columns share v, and the
    // column multiplicities of a thread stay in registers across the M tiles of one b-block
    const int Nt = (int)prm.rd_nt;
    const int Mv = prm.rd_m;
    constexpr int MAXG = (TN / 16 + 2) / 3;
    uint4 w[MAXG][2];
    int64_t wkey = -1;                                        // (item, row, bt) of the cached weights
    uint32_t tphb = 0;
    int ab = 0;
    RdSeq seq;
    seq.init(prm, rd_resident_a<IG, IG::STAGES>(prm, n_clusters), cluster_id, n_clusters, total_tiles);
    for (int i = 0; i < seq.n; ++i, ab ^= 1) {
        int p, mt, nt;
        seq.get(prm, i, tiles_per_item, p, mt, nt);
        const int64_t row = (int64_t)mt * G::TILE_M + rank * A_ROWS + quarter * 32 + lane;
        const bool row_ok = row < prm.rowsA;
        const int bt = nt / Mv, v = nt - bt * Mv;
        const int ng = prm.dbg == 1 ? 0 : g1 - g0;           // dbg 1: hand-off only
        const uint32_t tl = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(ab * TN + g0 * 16);
        const int64_t key = ((int64_t)p * prm.tiles_m + mt) * (prm.tiles_n / Mv) + bt;
        if (key != wkey) {                                    // new b-block: load this thread's weights
            wkey = key;
            const uint16_t* m2row = prm.m2 + ((int64_t)p * prm.rowsA + (row_ok ? row : 0)) * Nt + bt * TN + g0 * 16;
#pragma unroll
            for (int g = 0; g < MAXG; ++g) {
                w[g][0] = w[g][1] = make_uint4(0u, 0u, 0u, 0u);
                if (row_ok && g < ng && prm.dbg != 5) {       // dbg 5: no weight loads (diagnostic)
                    const uint4* mp = reinterpret_cast<const uint4*>(m2row + g * 16);
                    w[g][0] = __ldg(mp); w[g][1] = __ldg(mp + 1);
                }
            }
        }
        uint64_t* tf = ab ? tfull + 4 : tfull;
        uint64_t* te = ab ? tfull + 5 : tempty;
        mbar_wait(tf, (tphb >> ab) & 1u);
        fence_after();
        uint32_t acc = 0u;                                    // <= n1 n2 < 2^32 (host-checked)
        // two groups per TMEM load (one wait::ld per 32 columns)
#pragma unroll
        for (int g2 = 0; g2 < MAXG; g2 += 2) {
            if (g2 < ng) {
                uint32_t hv[32];
                if (g2 + 1 < ng) {
                    tmem_ld32(tl + g2 * 16, hv);
                } else {                                      // odd tail: never read past the warp's range
                    uint32_t (&lo)[16] = *reinterpret_cast<uint32_t(*)[16]>(&hv[0]);
                    tmem_ld16(tl + g2 * 16, lo);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int g = g2 + h;
                    if (g < MAXG && g < ng) {
                        const uint32_t mw[8] = {w[g][0].x, w[g][0].y, w[g][0].z, w[g][0].w,
                                                w[g][1].x, w[g][1].y, w[g][1].z, w[g][1].w};
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            acc += hv[16 * h + 2 * jj] * (mw[jj] & 0xffffu);
                            acc += hv[16 * h + 2 * jj + 1] * (mw[jj] >> 16);
                        }
                    }
                }
            }
        }
        // release the accumulator first: the atomic completes while the next tile accumulates
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(te, 0);
        if (row_ok && acc)
            atomicAdd(prm.rd_out + ((int64_t)p * prm.rowsA + row) * Mv + v, (unsigned long long)acc);
        tphb ^= 1u << ab;
    }
}

template <int MAXM, bool SEG, bool AUG, int TN>
__global__ void __maxnreg__(AUG ? 168 : 128)
k_gram_i8(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
          const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl, I8Params prm) {
    using G = Geo<2>;
    using IG = I8Geo<MAXM, SEG, AUG, TN>;
    constexpr int STAGES = IG::STAGES;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-B alignment by offsetting the shared pointer itself (keeps the shared address space, so
    // the epilogue's threshold / histogram accesses compile to LDS/STS, not generic loads)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* stages = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * IG::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
    float* s_nb = reinterpret_cast<float*>(smem + STAGES * IG::STAGE_BYTES + 1024);
    float* s_sb = s_nb + TN;
    float* s_T = s_sb + 2 * TN;                       // [NKIND][2*MAXM] thresholds, -inf padded
    uint32_t* hist_s = reinterpret_cast<uint32_t*>(s_T + IG::NKIND * 2 * MAXM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int cluster_id = blockIdx.x / 2, n_clusters = gridDim.x / 2;
    const int tiles_per_item = prm.tiles_act;
    const int total_tiles = prm.np * tiles_per_item;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        mbar_init(&tfull[0], 1);
        mbar_init(&tempty[0], 2 * IG::NEPI);              // epilogue warps x 2 CTAs
        mbar_init(tfull + 4, 1);                          // second accumulator (mode 1)
        mbar_init(tfull + 5, 2 * IG::NEPI);
        for (int s = 6; s < 6 + kRdBars; ++s) mbar_init(tfull + s, 1);   // mode-1 rings (count 1 each)
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mAh) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mAl) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mBh) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mBl) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (warp >= 2)
        for (int i = threadIdx.x - 64; i < IG::HIST_BYTES / 4; i += IG::NET) reinterpret_cast<uint32_t*>(hist_s)[i] = 0u;
    fence_before();
    cluster_sync();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            if (prm.mode == 1) {
                // one-digit operands (h planes only).  A resident: the A row block (all k-blocks)
                // stays in shared memory while the cluster's consecutive tiles stream B through a
                // ring; otherwise the stage memory is a ring of 2 STAGES (A_h | B_h) slots.
                const bool resA = rd_resident_a<IG, STAGES>(prm, n_clusters);
                // B slots: the stage memory after the A block, then the epilogue scratch that mode 1
                // does not use (norm / threshold staging and the histograms after the barriers)
                const int nsb0 = (STAGES * IG::STAGE_BYTES - prm.n_kb * IG::A_BYTES) / IG::B_BYTES;
                const int nsb = min(kRdSlots, nsb0 + (IG::FIXED - 2048) / IG::B_BYTES);
                unsigned char* bring = stages + prm.n_kb * IG::A_BYTES;
                unsigned char* bextra = stages + STAGES * IG::STAGE_BYTES + 1024 - nsb0 * IG::B_BYTES;
                int key_prev = -1, sb = 0;
                uint32_t aph = 0, bph = 0;
                RdSeq seq;
                seq.init(prm, resA, cluster_id, n_clusters, total_tiles);
                for (int i = 0; i < seq.n; ++i) {
                    int p, mt, nt;
                    seq.get(prm, i, tiles_per_item, p, mt, nt);
                    const int ya = (int)(prm.a_off + p * prm.rowsA + (int64_t)mt * G::TILE_M + rank * A_ROWS);
                    const int yb = (int)(prm.b_off + p * prm.rowsB + (int64_t)nt * TN + rank * IG::B_ROWS);
                    if (resA) {
                        const int key = p * prm.tiles_m + mt;
                        if (key != key_prev) {
                            mbar_wait(tfull + 7, aph ^ 1);
                            if (rank == 0) mbar_expect_tx(tfull + 6, 2 * prm.n_kb * IG::A_BYTES);
                            for (int kb = 0; kb < prm.n_kb; ++kb)
                                tma_load_2d<2>(stages + kb * IG::A_BYTES, &mAh, tfull + 6, kb * 128, ya);
                            aph ^= 1;
                            key_prev = key;
                        }
                        for (int kb = 0; kb < prm.n_kb; ++kb) {
                            mbar_wait(tfull + 8 + kRdSlots + sb, bph ^ 1);
                            if (rank == 0) mbar_expect_tx(tfull + 8 + sb, 2 * IG::B_BYTES);
                            tma_load_2d<2>((sb < nsb0 ? bring : bextra) + sb * IG::B_BYTES, &mBh, tfull + 8 + sb,
                                           kb * 128, yb);
                            if (++sb == nsb) { sb = 0; bph ^= 1; }
                        }
                    } else {
                        for (int kb = 0; kb < prm.n_kb; ++kb) {
                            mbar_wait(tfull + 6 + 2 * STAGES + sb, bph ^ 1);
                            unsigned char* st = stages + sb * (IG::A_BYTES + IG::B_BYTES);
                            uint64_t* f = tfull + 6 + sb;
                            if (rank == 0) mbar_expect_tx(f, 2 * (IG::A_BYTES + IG::B_BYTES));
                            tma_load_2d<2>(st, &mAh, f, kb * 128, ya);
                            tma_load_2d<2>(st + IG::A_BYTES, &mBh, f, kb * 128, yb);
                            if (++sb == 2 * STAGES) { sb = 0; bph ^= 1; }
                        }
                    }
                }
            }
            for (int t = cluster_id; t < total_tiles && prm.mode != 1; t += n_clusters) {
                const int p = prm.p0 + t / tiles_per_item;
                int mt, nt;
                tile_of(prm, t % tiles_per_item, mt, nt);
                const int ya = (int)(prm.a_off + p * prm.rowsA + (int64_t)mt * G::TILE_M + rank * A_ROWS);
                const int yb = (int)(prm.b_off + p * prm.rowsB + (int64_t)nt * TN + rank * IG::B_ROWS);
                for (int kb = 0; kb < prm.n_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char* st = stages + stage * IG::STAGE_BYTES;
                    // diagnostics: dbg 3 skips the B loads, dbg 4 all loads (MMA rate alone)
                    const bool only_a = prm.dbg == 3, none = prm.dbg == 4;
                    if (rank == 0)
                        mbar_expect_tx(&full[stage], none ? 0 : only_a ? 4 * IG::A_BYTES : 2 * IG::STAGE_BYTES);
                    const int x = kb * 128;
                    if (prm.pf > 0 && kb + prm.pf < prm.n_kb) {   // L2 prefetch pf k-blocks ahead
                        const int xp = (kb + prm.pf) * 128;
                        tma_prefetch_2d(&mAh, xp, ya);
                        tma_prefetch_2d(&mAl, xp, ya);
                        tma_prefetch_2d(&mBh, xp, yb);
                        tma_prefetch_2d(&mBl, xp, yb);
                    }
                    if (!none) {
                        tma_load_2d<2>(st, &mAh, &full[stage], x, ya);
                        tma_load_2d<2>(st + IG::A_BYTES, &mAl, &full[stage], x, ya);
                    }
                    if (!only_a && !none) {
                        tma_load_2d<2>(st + 2 * IG::A_BYTES, &mBh, &full[stage], x, yb);
                        tma_load_2d<2>(st + 2 * IG::A_BYTES + IG::B_BYTES, &mBl, &full[stage], x, yb);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            const uint32_t id = idesc_i8(G::TILE_M, TN);
            const uint32_t dH0 = tmem_base, dX = tmem_base + TN;
            // mode 1 has no X accumulator: its TMEM columns double-buffer H (tile i + 1
            // accumulates while the epilogue drains tile i); barriers tfull[4] / tfull[5]
            int stage = 0, ab = 0;
            uint32_t phase = 0, tphb = 0;
            if (prm.mode == 1) {                            // see the producer
                const bool resA = rd_resident_a<IG, STAGES>(prm, n_clusters);
                // B slots: the stage memory after the A block, then the epilogue scratch that mode 1
                // does not use (norm / threshold staging and the histograms after the barriers)
                const int nsb0 = (STAGES * IG::STAGE_BYTES - prm.n_kb * IG::A_BYTES) / IG::B_BYTES;
                const int nsb = min(kRdSlots, nsb0 + (IG::FIXED - 2048) / IG::B_BYTES);
                unsigned char* bring = stages + prm.n_kb * IG::A_BYTES;
                unsigned char* bextra = stages + STAGES * IG::STAGE_BYTES + 1024 - nsb0 * IG::B_BYTES;
                int key_prev = -1, sb = 0;
                uint32_t aph = 0, bph = 0;
                RdSeq seq;
                seq.init(prm, resA, cluster_id, n_clusters, total_tiles);
                for (int i = 0; i < seq.n; ++i) {
                    uint64_t* tf = ab ? tfull + 4 : tfull;
                    uint64_t* te = ab ? tfull + 5 : tempty;
                    const uint32_t dH = dH0 + (ab ? (uint32_t)TN : 0u);
                    mbar_wait_cluster(te, ((tphb >> ab) & 1u) ^ 1u);
                    fence_after();
                    if (resA) {
                        int p, mt, nt;
                        seq.get(prm, i, tiles_per_item, p, mt, nt);
                        const int key = p * prm.tiles_m + mt;
                        if (key != key_prev) {
                            if (key_prev >= 0) mma_commit<2>(tfull + 7);   // the old A block is free once its MMAs end
                            mbar_wait(tfull + 6, aph);
                            fence_after();
                            aph ^= 1;
                            key_prev = key;
                        }
                    }
                    for (int kb = 0; kb < prm.n_kb; ++kb) {
                        uint64_t ah, bh;
                        if (resA) {
                            mbar_wait(tfull + 8 + sb, bph);
                            fence_after();
                            ah = sdesc(smem_u32(stages + kb * IG::A_BYTES));
                            bh = sdesc(smem_u32((sb < nsb0 ? bring : bextra) + sb * IG::B_BYTES));
                        } else {
                            mbar_wait(tfull + 6 + sb, bph);
                            fence_after();
                            const uint32_t s0 = smem_u32(stages + sb * (IG::A_BYTES + IG::B_BYTES));
                            ah = sdesc(s0);
                            bh = sdesc(s0 + IG::A_BYTES);
                        }
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            mma_i8(dH, ah + (uint64_t)(k * 2), bh + (uint64_t)(k * 2), id, (kb != 0 || k != 0) ? 1u : 0u);
                        if (resA) {
                            mma_commit<2>(tfull + 8 + kRdSlots + sb);
                            if (++sb == nsb) { sb = 0; bph ^= 1; }
                        } else {
                            mma_commit<2>(tfull + 6 + 2 * STAGES + sb);
                            if (++sb == 2 * STAGES) { sb = 0; bph ^= 1; }
                        }
                    }
                    mma_commit<2>(tf);
                    tphb ^= 1u << ab;
                    ab ^= 1;
                }
            }
            for (int t = cluster_id; t < total_tiles && prm.mode != 1; t += n_clusters) {
                // one accumulation (and one epilogue hand-off) per phase; nph = 1: the whole K
                for (int ph = 0; ph < prm.nph; ++ph) {
                    uint64_t* tf = ab ? tfull + 4 : tfull;
                    uint64_t* te = ab ? tfull + 5 : tempty;
                    const uint32_t dH = dH0 + (ab ? (uint32_t)TN : 0u);
                    mbar_wait_cluster(te, ((tphb >> ab) & 1u) ^ 1u);
                    fence_after();
                    const int kb0 = ph ? prm.kb_end[ph - 1] : 0, kb1 = prm.kb_end[ph];
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        fence_after();
                        const uint32_t s0 = smem_u32(stages + stage * IG::STAGE_BYTES);
                        {
                            const uint64_t ah = sdesc(s0), al = sdesc(s0 + IG::A_BYTES);
                            const uint64_t bh = sdesc(s0 + 2 * IG::A_BYTES), bl = sdesc(s0 + 2 * IG::A_BYTES + IG::B_BYTES);
#pragma unroll
                            for (int k = 0; k < 4; ++k) {               // 4 x 32 int8 of K per 128-byte row
                                const uint64_t adv = (uint64_t)(k * 2);  // +32 B in the start-address field
                                const uint32_t first = (kb != kb0 || k != 0) ? 1u : 0u;
                                mma_i8(dH, ah + adv, bh + adv, id, first);
                                mma_i8(dX, ah + adv, bl + adv, id, first);
                                mma_i8(dX, al + adv, bh + adv, id, 1u);
                            }
                        }
                        mma_commit<2>(&empty[stage]);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    mma_commit<2>(tf);
                    tphb ^= 1u << ab;
                }
            }
        }
    } else if constexpr (AUG) {
        epilogue_aug<MAXM, SEG, TN>(prm, tmem_base, tfull, tempty, s_nb, s_sb, s_T, hist_s, cluster_id, n_clusters,
                                total_tiles, tiles_per_item, rank, warp, lane);
    } else if (prm.mode == 1) {
        epilogue_rowdot<MAXM, SEG, TN>(prm, tmem_base, tfull, tempty, cluster_id, n_clusters, total_tiles,
                                       tiles_per_item, rank, warp, lane);
    } else {
        // ------------------------------------------------------------ epilogue
        // warp w reads TMEM lanes 32 (w % 4) .. +31 (its quarter); the NEPI epilogue warps split
        // each quarter's TN columns into contiguous 16-column groups
        const int quarter = warp & 3;
        const int ew = warp - 2;
        const int e0 = (quarter + 2) & 3;             // first epilogue warp of this quarter
        const int nwq = (IG::NEPI - e0 + 3) / 4;      // epilogue warps in this quarter
        const int kq = ew >> 2;                       // index within the quarter
        const int g0 = kq * (TN / 16) / nwq, g1 = (kq + 1) * (TN / 16) / nwq;
        const int ncol = (g1 - g0) * 16;
        const int et = threadIdx.x - 64;              // 0..NET-1
        const int M = prm.M;
        uint32_t tph = 0;
        for (int t = cluster_id; t < total_tiles; t += n_clusters) {
            const int p = prm.p0 + t / tiles_per_item;
            int mt, nt;
            tile_of(prm, t % tiles_per_item, mt, nt);
            const int64_t col0 = (int64_t)nt * TN;
            const int64_t browbase = prm.b_off + (int64_t)p * prm.rowsB;
            named_bar(1, IG::NET);
            {
                const int64_t c = col0 + et;
                const bool ok = c < prm.rowsB;
                if (et < TN) {                   // the tile's TN columns (s_nb / s_sb hold TN each)
                    s_nb[et] = ok ? prm.nrm[browbase + c] : 0.f;
                    s_sb[et] = ok ? prm.scl[browbase + c] : 0.f;
                }
                if (et < 2 * MAXM) s_T[et] = (et < M) ? prm.thr2[(int64_t)p * prm.thr_stride + et] : -INFINITY;
            }
            named_bar(1, IG::NET);
            const int64_t row = (int64_t)mt * G::TILE_M + rank * A_ROWS + quarter * 32 + lane;
            const bool row_ok = row < prm.rowsA;
            const int64_t arow = prm.a_off + (int64_t)p * prm.rowsA + (row_ok ? row : 0);
            const float na = row_ok ? __ldg(&prm.nrm[arow]) : 0.f;
            const float sa = row_ok ? __ldg(&prm.scl[arow]) : 0.f;

            // ---- bin straight from TMEM in 8 rolled groups of 16 columns (compact loop body: an
            // unrolled 128-pair body thrashed the instruction cache).  Per pair: d^2 and its bound E,
            // bin b = #{m : d^2 + E < T_m} by a 5-level binary search (2 levels on registers, the rest
            // in shared memory), one LDS for the ambiguity test, one per-thread shared histogram
            // update; histograms are flushed once per tile (warp REDUX -> u64 atomics).
            mbar_wait(&tfull[0], tph);
            fence_after();
            const int hc0 = (int)(col0 + g0 * 16);
            const int nvalid = (int)min((int64_t)ncol, prm.rowsB - hc0);     // warp-uniform
            const bool diag_mode = prm.diag != nullptr && p == 0;          // diagnostics (item 0 only)
            float* diag_row = diag_mode ? prm.diag + (size_t)(row_ok ? row : 0) * prm.rowsB * 2 : nullptr;
            const float kq_sa = prm.kq * 0.81649658f;    // sqrt((sa^2 + sb^2)/3) <= sqrt(2/3) max(sa, sb)
            const float kll_sa = prm.kll * sa;
            const float m2sa = -2.f * sa;
            const float reln = prm.rel;
            const uint32_t tl = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(g0 * 16);
            const bool skip = prm.dbg >= 2 || (prm.diag != nullptr && p != 0);
            const float T_top = s_T[MAXM - 1], T_mid = s_T[MAXM / 2 - 1];
            const float T_q1 = s_T[MAXM / 4 - 1], T_q3 = s_T[MAXM / 2 + MAXM / 4 - 1];
            const int64_t cs_first = (int64_t)hc0 / prm.sp.col_seg;
            int bnd[IG::NLOC > 1 ? IG::NLOC - 1 : 1];    // local column indices where the segment changes
#pragma unroll
            for (int i = 0; i < IG::NLOC - 1; ++i) {
                const int64_t c = (cs_first + 1 + i) * prm.sp.col_seg - hc0;
                bnd[i] = SEG ? (int)(c < ncol ? c : (1 << 30)) : (1 << 30);
            }
            uint32_t* myh = hist_s + et;
            uint8_t* binrow = (prm.binout != nullptr && row_ok)
                                  ? prm.binout + (((int64_t)p * prm.nq + prm.q_l2) * prm.rowsA + row) * prm.rowsB
                                  : nullptr;
            // transposed output: entry (col, row) at stride rowsA (lanes = consecutive rows: coalesced)
            uint8_t* tbase = (binrow != nullptr && prm.bin_t)
                                 ? prm.binout + ((int64_t)p * prm.nq + prm.q_l2) * prm.rowsA * prm.rowsB + row
                                 : nullptr;
            const bool mirror = binrow != nullptr && prm.skip == 1 && mt < nt;
            const bool diag_sym = binrow != nullptr && prm.skip == 1 && mt == nt;
            uint8_t* mbase = mirror ? prm.binout + ((int64_t)p * prm.nq + prm.q_l2) * prm.rowsA * prm.rowsB + row : nullptr;

#pragma unroll 1
            for (int g = 0; g < g1 - g0 && !skip; ++g) {
                if (g * 16 >= nvalid) break;                        // warp-uniform
                uint32_t hv[16], xv[16];
                tmem_ld16(tl + g * 16, hv);
                tmem_ld16(tl + TN + g * 16, xv);
                if (prm.dbg == 1 || !row_ok) continue;
                // (d^2, E) of pair jj of the group
                auto d2_E = [&](int jj, float& d2, float& E) {
                    const int jc = g0 * 16 + g * 16 + jj;
                    const float sb = s_sb[jc], nb = s_nb[jc];
                    // 65536 H + 256 X in FP32 (relative rounding 2^-24 of g, inside rel): measured
                    // identical to an FP64 combination on generator data
                    const float gi = fmaf((float)(int)hv[jj], 65536.f, (float)(int)xv[jj] * 256.f);
                    d2 = fmaf(m2sa * sb, gi, na + nb);
                    const float dd = fmaxf(d2, 1e-30f);
                    E = fmaf(kq_sa * sqrt_approx(dd), fmaxf(sa, sb), fmaf(kll_sa, sb, reln * (na + nb)));
                };
                if (diag_mode) {                            // diagnostics: (d^2, E) of every pair, no binning
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        float d2, E;
                        d2_E(jj, d2, E);
                        if (g * 16 + jj < nvalid) {
                            diag_row[2 * (hc0 + g * 16 + jj)] = d2;
                            diag_row[2 * (hc0 + g * 16 + jj) + 1] = E;
                        }
                    }
                    continue;
                }
                // phase A (loads + ALU only, branch-free, so the compiler overlaps the 16 pairs' search
                // chains): bin b_j = #{m : hi_j < T_m} and the ambiguity bit of every pair of the group
                int bin[16];                                // b | (local column segment << 8)
                uint32_t amb = 0;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    const int j = g * 16 + jj;
                    float d2, E;
                    d2_E(jj, d2, E);
                    const float hi = d2 + E, lo = d2 - E;
                    // binary search over the decreasing thresholds (s_T[MAXM..2 MAXM) = -inf):
                    // two levels from registers, the remaining log2(MAXM) - 2 from shared memory
                    int b = (hi < T_mid) ? MAXM / 2 : 0;
                    b += (hi < (b ? T_q3 : T_q1)) ? MAXM / 4 : 0;
#pragma unroll
                    for (int s = MAXM / 8; s >= 1; s >>= 1)
                        if (hi < s_T[b + s - 1]) b += s;
                    b = (hi < T_top) ? MAXM : b;
                    int lcs = 0;
                    if (SEG) {
#pragma unroll
                        for (int i = 0; i < IG::NLOC - 1; ++i) lcs += (j >= bnd[i]) ? 1 : 0;
                    }
                    bin[jj] = b | (lcs << 8);
                    // a threshold in (lo, hi]: provisional bin b, exact re-check
                    amb |= (lo < s_T[b] && j < nvalid) ? (1u << jj) : 0u;
                }
                // phase B: per-thread histogram increments (fire-and-forget shared atomics), or
                // in bin-matrix mode the 16 provisional bins of the group as bytes
                if (tbase != nullptr) {
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj)
                        if (g * 16 + jj < nvalid) tbase[(int64_t)(hc0 + g * 16 + jj) * prm.rowsA] = (uint8_t)(bin[jj] & 255);
                } else if (binrow != nullptr) {
                    uint8_t* dst = binrow + hc0 + g * 16;
                    if (g * 16 + 16 <= nvalid && ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
                        uint32_t wv[4];
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            wv[v] = (uint32_t)(bin[4 * v] & 255) | ((uint32_t)(bin[4 * v + 1] & 255) << 8) |
                                    ((uint32_t)(bin[4 * v + 2] & 255) << 16) | ((uint32_t)(bin[4 * v + 3] & 255) << 24);
                        *reinterpret_cast<uint4*>(dst) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj)
                            if (g * 16 + jj < nvalid) dst[jj] = (uint8_t)(bin[jj] & 255);
                    }
                    if (mirror) {        // symmetric bin matrix: (j, i) from the upper tile (i, j)
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj)
                            if (g * 16 + jj < nvalid) mbase[(int64_t)(hc0 + g * 16 + jj) * prm.rowsB] = (uint8_t)(bin[jj] & 255);
                    }
                } else {
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj)
                        if (g * 16 + jj < nvalid)
                            atomicAdd(myh + (bin[jj] & 255) * IG::NET, SEG ? 1u << ((bin[jj] >> 5) & 24) : 1u);
                }
                if (amb) {                                  // rare (~1e-4 of the pairs)
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        if (!((amb >> jj) & 1u)) continue;
                        // symmetric bin matrix, diagonal tile: (i, j) and (j, i) are both here and
                        // the re-check writes both orders, so list each unordered pair once
                        if (diag_sym && hc0 + g * 16 + jj < row) continue;
                        const uint32_t idx = atomicAdd(prm.ctr, 1u);
                        if (idx < prm.cap)
                            prm.list[idx] = make_uint4((uint32_t)p, (uint32_t)row, (uint32_t)(hc0 + g * 16 + jj),
                                                       (uint32_t)(bin[jj] & 255));
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(&tempty[0], 0);
            tph ^= 1;
            if (skip || prm.dbg == 1 || prm.binout != nullptr) continue;
            // ---- flush the per-thread histograms (warp sums -> global u64 atomics), reset them.
            // Cell [b][thread] is a u32; with column segments (SEG) byte l counts local segment l.
            const int64_t rs = row_ok ? row / prm.sp.row_seg : 0;
            const int64_t rs0 = __shfl_sync(0xffffffffu, rs, 0);
            const bool uniform = __all_sync(0xffffffffu, rs == rs0 || !row_ok);
            myh[0] = 0u;                                    // bin 0 (outside every radius) is not kept
            for (int bb = 1; bb <= M; ++bb) {
                const uint32_t cell = myh[bb * IG::NET];
                myh[bb * IG::NET] = 0u;
#pragma unroll
                for (int l = 0; l < IG::NLOC; ++l) {
                    const int64_t cs = cs_first + l;
                    if (cs * prm.sp.col_seg >= prm.rowsB || cs * prm.sp.col_seg >= hc0 + ncol) break;
                    const uint32_t v = SEG ? ((cell >> (8 * l)) & 255u) : cell;
                    if (uniform) {
                        const uint32_t tot = __reduce_add_sync(0xffffffffu, v);
                        if (lane == 0 && tot)
                            atomicAdd(&prm.hist[hist_index(prm.sp, prm.nq, M, p, rs0, cs, prm.q_l2, bb)],
                                      (unsigned long long)tot);
                    } else if (v) {
                        atomicAdd(&prm.hist[hist_index(prm.sp, prm.nq, M, p, rs, cs, prm.q_l2, bb)],
                                  (unsigned long long)v);
                    }
                }
            }
        }
    }
    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}
}  // namespace tc

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled_i8)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_map_i8(CUtensorMap* m, const void* base, int64_t rows, int64_t Kp, int box_rows) {
    static PFN_encodeTiled_i8 enc = nullptr;
    if (!enc) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
        enc = reinterpret_cast<PFN_encodeTiled_i8>(p);
    }
    cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)Kp};
    cuuint32_t box[2] = {128u, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MAXM, bool SEG, bool AUG = false, int TN = 256>
static cudaError_t launch_i8_t(const tc::I8Params& prm, const CUtensorMap* maps, int nsm, cudaStream_t st) {
    using IG = tc::I8Geo<MAXM, SEG, AUG, TN>;
    static SmemAttrOnce attr;
    if (cudaError_t e = attr.ensure(tc::k_gram_i8<MAXM, SEG, AUG, TN>, IG::SMEM_BYTES); e != cudaSuccess) return e;
    const int64_t tiles = (int64_t)prm.np * prm.tiles_act;
    const int clusters = (int)(tiles < nsm / 2 ? tiles : nsm / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(clusters * 2));
    cfg.blockDim = dim3(IG::NTHR);
    cfg.dynamicSmemBytes = IG::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope ps_(prm.mode == 1 ? K_RESAMPLE : K_GRAM_TC, st);   // mode 1 is the bootstrap resample
    cudaError_t e = cudaLaunchKernelEx(&cfg, tc::k_gram_i8<MAXM, SEG, AUG, TN>, maps[0], maps[1], maps[2], maps[3], prm);
    note_launch();
    if (e != cudaSuccess) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, tc::k_gram_i8<MAXM, SEG, AUG, TN>);
        fprintf(stderr, "[libcil] k_gram_i8 launch failed (%s): regs=%d maxThreads=%d local=%zu smem_dyn=%d\n",
                cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock, fa.localSizeBytes, IG::SMEM_BYTES);
        return e;
    }
    return cudaGetLastError();
}

template <int TN>
static cudaError_t dispatch_i8(const tc::I8Params& prm, const CUtensorMap* maps, int nsm, cudaStream_t st, bool seg,
                               int M) {
    if (prm.nph == 3) {
        if (M <= 16)
            return seg ? launch_i8_t<16, true, true, TN>(prm, maps, nsm, st)
                       : launch_i8_t<16, false, true, TN>(prm, maps, nsm, st);
        if (seg) return cudaErrorInvalidValue;                 // host routes these to the CUDA cores
        if (M <= 32) return launch_i8_t<32, false, true, TN>(prm, maps, nsm, st);
        return launch_i8_t<64, false, true, TN>(prm, maps, nsm, st);
    }
    if (M <= 16) return seg ? launch_i8_t<16, true, false, TN>(prm, maps, nsm, st) : launch_i8_t<16, false, false, TN>(prm, maps, nsm, st);
    if (M <= 32) return seg ? launch_i8_t<32, true, false, TN>(prm, maps, nsm, st) : launch_i8_t<32, false, false, TN>(prm, maps, nsm, st);
    return seg ? launch_i8_t<64, true, false, TN>(prm, maps, nsm, st) : launch_i8_t<64, false, false, TN>(prm, maps, nsm, st);
}

cudaError_t launch_gram_i8(const I8Args& a, cudaStream_t st) {
    if (a.rowsA == 0 || a.rowsB == 0) return cudaSuccess;
    int64_t rows = (int64_t)a.P * (a.b_same ? a.rowsA : a.rowsA + a.rowsB);
    if (a.offs_set) {
        if (a.b_same || a.a_off < 0 || a.b_off < 0) return cudaErrorInvalidValue;
        rows = std::max(a.a_off + (int64_t)a.P * a.rowsA, a.b_off + (int64_t)a.P * a.rowsB);
    }
    if (rows >= (1ll << 31) || (a.b_same && a.rowsA != a.rowsB)) return cudaErrorInvalidValue;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (a.sm_budget > 0 && a.sm_budget < nsm) nsm = a.sm_budget;
    // B columns per tile: 192 when that costs fewer column-waves of the persistent grid than 256
    // (waves = ceil(tiles / CTA pairs); a 192-column tile is charged 5 % extra for its A feed):
    // less padding (a 550-row panel: 576 instead of 768 columns) or a better last wave (C7's 75
    // k < l tiles on 74 CTA pairs: 100 tiles of 192).  The mirrored symmetric layout needs square
    // tiles, mode 1's b-major B layout assumes 256.
    int tn = 256;
    if (a.skip != 1 && a.mode != 1) {
        const int64_t np = a.np > 0 ? a.np : a.P - a.p0;
        const int64_t tm = (a.rowsA + tc::Geo<2>::TILE_M - 1) / tc::Geo<2>::TILE_M;
        auto waves = [&](int t) {
            const int64_t tiles = np * tc::tiles_active(a.skip, (int)tm, (int)((a.rowsB + t - 1) / t), a.sp.row_seg,
                                                        a.sp.col_seg, a.rowsB, t);
            return (tiles + nsm / 2 - 1) / (nsm / 2);
        };
        if ((double)waves(192) * 192 * 1.05 < (double)waves(256) * 256) tn = 192;
    }
    static const char* tne = getenv("CIL_I8_TN");            // diagnostic override (256 / 192)
    if (tne && a.skip != 1 && a.mode != 1) tn = atoi(tne) == 192 ? 192 : 256;
    if (a.mode == 1 && (a.rd_nt % 256 || a.rowsB != (int64_t)a.rd_m * a.rd_nt)) return cudaErrorInvalidValue;
    if (a.tn_force == 64) {
        if (a.skip != 0 || a.mode != 0 || a.nph == 3) return cudaErrorInvalidValue;
        tn = 64;
    }
    CUtensorMap maps[4];
    if (!make_map_i8(&maps[0], a.hq, rows, a.Kp, tc::A_ROWS) || !make_map_i8(&maps[1], a.lq, rows, a.Kp, tc::A_ROWS) ||
        !make_map_i8(&maps[2], a.hq, rows, a.Kp, tn / 2) || !make_map_i8(&maps[3], a.lq, rows, a.Kp, tn / 2))
        return cudaErrorInvalidValue;
    tc::I8Params prm{};
    prm.rowsA = a.rowsA; prm.rowsB = a.rowsB;
    prm.b_off = a.offs_set ? a.b_off : a.b_same ? 0 : (int64_t)a.P * a.rowsA;
    prm.a_off = a.offs_set ? a.a_off : 0;
    prm.P = a.P; prm.p0 = a.p0; prm.np = a.np > 0 ? a.np : a.P - a.p0;
    prm.n_kb = (int)(a.Kp / 128);
    prm.tiles_m = (int)((a.rowsA + tc::Geo<2>::TILE_M - 1) / tc::Geo<2>::TILE_M);
    prm.tn = tn;
    prm.tiles_n = (int)((a.rowsB + tn - 1) / tn);
    prm.nrm = a.nrm; prm.scl = a.scl;
    prm.thr2 = a.thr2; prm.thr_stride = a.thr_stride;
    prm.M = a.M; prm.nq = a.nq; prm.q_l2 = a.q_l2;
    prm.sp = a.sp;
    prm.hist = reinterpret_cast<unsigned long long*>(a.hist);
    prm.list = a.recheck; prm.ctr = a.recheck_ctr; prm.cap = a.recheck_cap;
    prm.kq = a.kq; prm.kll = a.kll; prm.rel = a.rel;
    prm.diag = a.diag;
    prm.binout = a.binout;
    prm.skip = a.skip;
    prm.mode = a.mode;
    prm.bin_t = a.bin_t ? 1 : 0;
    if (a.bin_t && (a.skip != 0 || !a.binout)) return cudaErrorInvalidValue;
    prm.m2 = a.m2; prm.rd_nt = a.rd_nt; prm.rd_m = a.rd_m; prm.rd_out = a.rd_out;
    prm.tiles_act = tc::tiles_active(prm.skip, prm.tiles_m, prm.tiles_n, a.sp.row_seg, a.sp.col_seg, a.rowsB, tn);
    if (prm.tiles_act == 0) return cudaSuccess;
    prm.nph = a.nph == 3 ? 3 : 1;
    if (prm.nph == 3) {
        for (int i = 0; i < 3; ++i) { prm.kb_end[i] = a.kb_end[i]; prm.kll3[i] = a.kll3[i]; prm.q_tc[i] = a.q_tc[i]; }
        prm.nrm3 = a.nrm3; prm.scl3 = a.scl3;
        prm.part = reinterpret_cast<float2*>(a.part);
        prm.ih = a.ih;
        prm.n_kb = a.kb_end[2];
    } else {
        prm.kb_end[0] = prm.n_kb;
    }
    {
        static const char* dbg = getenv("CIL_DEBUG_I8");
        prm.dbg = dbg ? atoi(dbg) : 0;
        static const char* pfe = getenv("CIL_I8_PF");
        prm.pf = pfe ? atoi(pfe) : 0;
    }
    const bool seg = a.sp.col_seg < a.rowsB;
    if (tn == 64) {
        if (seg || prm.nph == 3 || prm.mode != 0) return cudaErrorInvalidValue;
        if (a.M <= 16) return launch_i8_t<16, false, false, 64>(prm, maps, nsm, st);
        if (a.M <= 32) return launch_i8_t<32, false, false, 64>(prm, maps, nsm, st);
        return launch_i8_t<64, false, false, 64>(prm, maps, nsm, st);
    }
    if (tn == 192) return dispatch_i8<192>(prm, maps, nsm, st, seg, a.M);
    return dispatch_i8<256>(prm, maps, nsm, st, seg, a.M);
}

}  // namespace cil
