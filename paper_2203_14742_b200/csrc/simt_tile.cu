// simt_tile.cu — step a3 of the hot path: the alternative distance measures
// (Eqs. (6)-(10)) — and L2 when the SIMT engine is chosen —
// on CUDA cores, fused with radius binning (Eq. (1)) so no N x Nt matrix is stored.
//
// Per pair (i,j) and region al in {value, D_x, D_y} of the augmented operands:
//   m_al = max_e |A_i[e] - B_j[e]|        (FADD2 + 3-input |.|-max)
//   s_al = sum_e (A_i[e] - B_j[e])^2      (FADD2 + FFMA2; FP32 chunks of 128 flushed to FP64)
// Epilogue (FP64): a_al = sqrt(w * s_al / h^2[al>0]), m_al /= h[al>0], then
//   L2 = a_0, Linf = m_0, W12sum = a_0+a_x+a_y, W12 = sqrt(a_0^2+a_x^2+a_y^2),
//   W1inf = max(m_0,m_x,m_y), W1infsum = m_0+m_x+m_y     (readings R1-R4)
// and bin b = #{m : d < R_m} (strict <) into a per-segment histogram.
//
// Tiling: CTA = 128 threads = 8 RI A-rows x 64 B-rows of pairs, RI x 4 pairs per (RI = 8 for the max family alone, else 4)
// thread; k-chunks of 32 floats double-buffered in smem with cp.async (rows
// padded to 36 floats -> conflict-free LDS.128).
#include "cil_internal.cuh"

namespace cil {

namespace {
constexpr int TB = 64, BK = kSimtBK, LDS = BK + 4;   // TA = 8 RI rows per CTA (template)
constexpr int NTHR = 128;
constexpr int FLUSH = 4;   // chunks between FP32 -> FP64 flushes (128 elements per pair)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float absmax3(float m, float x, float y) {
    return fmaxf(m, fmaxf(fabsf(x), fabsf(y)));
}
}  // namespace

// SYM (bin matrix of a panel against itself) is a template flag so that the counting kernels'
// code is not touched by the mirrored writes (as a runtime flag it cost the max family 16 %)
#ifndef CIL_SIMT_EXP
#define CIL_SIMT_EXP 0   // code-generation experiments (tools/simt_var.sh); 0 = product
#endif
template <bool DO_MAX, bool DO_SUM, int RI, bool SYM>
__global__ void __launch_bounds__(NTHR, (CIL_SIMT_EXP == 1 && !DO_SUM) ? 3 : (DO_SUM || RI == 8) ? 2 : 4)
    k_simt(SimtArgs a) {
    constexpr int TA = 8 * RI;     // A rows per CTA: RI x 4 pairs per thread
    constexpr int NP = RI * 4;     // pairs per thread
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* As = reinterpret_cast<float*>(smem_raw);                 // [2][TA][LDS]
    float* Bs = As + 2 * TA * LDS;                                   // [2][TB][LDS]
    double* thr_s = reinterpret_cast<double*>(Bs + 2 * TB * LDS);    // [nq*M]
    // per-thread region results for regions 0 and 1 (region 2 stays in registers)
    double* rs_sum = thr_s + kMaxMeas * kMaxM;                       // [2][NP][NTHR]
    float* rs_max = reinterpret_cast<float*>(rs_sum + (DO_SUM ? 2 * NP * NTHR : 0));  // [2][NP][NTHR]
    uint32_t* hist_s = reinterpret_cast<uint32_t*>(rs_max + (DO_MAX ? 2 * NP * NTHR : 0));

    const int p = blockIdx.z;
    if (a.status[p] & CIL_ITEM_BADRADII) return;
    const int64_t row0 = (int64_t)blockIdx.y * TA;
    const int64_t col0 = (int64_t)blockIdx.x * TB;
    // Alg. 1 triangle: a tile without any block k < l has nothing to count
    if (a.tri && row0 / a.sp.row_seg >= (min(col0 + TB, a.rowsB) - 1) / a.sp.col_seg) return;
    // symmetric bin matrix: the strictly lower tiles come from the mirrored writes
    if (SYM && row0 >= col0 + TB) return;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ty = (warp >> 1) * 4 + (lane >> 3);   // 0..7
    const int tx = (warp & 1) * 8 + (lane & 7);     // 0..15
    const int nq = a.bp.nq, M = a.bp.M;

    for (int t = tid; t < nq * M; t += NTHR) thr_s[t] = a.thr[(int64_t)p * a.thr_stride + t];

    // local segment window of this tile
    const int64_t rlast = min(row0 + TA, a.rowsA) - 1, clast = min(col0 + TB, a.rowsB) - 1;
    const int64_t rs0 = row0 / a.sp.row_seg, cs0 = col0 / a.sp.col_seg;
    const int nrs = (int)(rlast / a.sp.row_seg - rs0 + 1), ncs = (int)(clast / a.sp.col_seg - cs0 + 1);
    const int nloc = nrs * ncs;
    const int hist_len = nloc * nq * (M + 1);
    const bool use_sh = hist_len <= a.hist_cap;
    if (use_sh)
        for (int t = tid; t < hist_len; t += NTHR) hist_s[t] = 0u;

    const float* Ag = a.Aaug + ((int64_t)p * a.rowsA) * a.Kaug;
    const float* Bg = a.Baug + ((int64_t)p * a.rowsB) * a.Kaug;
    const int nchunks = (int)(a.g.off[a.g.nreg] / BK);
    const int c_end0 = (int)(a.g.off[1] / BK);
    const int c_end1 = (int)(a.g.off[2] / BK);

    auto load_chunk = [&](int c, int buf) {
        const int64_t k0 = (int64_t)c * BK;
        // A: TA rows x 8 x 16B, TA / 16 copies per thread
#pragma unroll
        for (int t = 0; t < (TA * BK / 4) / NTHR; ++t) {
            const int idx = tid + t * NTHR;
            const int r = idx >> 3, v = idx & 7;
            const int64_t gr = row0 + r;
            const bool ok = gr < a.rowsA;
            cp_async16(As + (buf * TA + r) * LDS + v * 4, Ag + (ok ? gr : 0) * a.Kaug + k0 + v * 4, ok);
        }
#pragma unroll
        for (int t = 0; t < (TB * BK / 4) / NTHR; ++t) {
            const int idx = tid + t * NTHR;
            const int r = idx >> 3, v = idx & 7;
            const int64_t gc = col0 + r;
            const bool ok = gc < a.rowsB;
            cp_async16(Bs + (buf * TB + r) * LDS + v * 4, Bg + (ok ? gc : 0) * a.Kaug + k0 + v * 4, ok);
        }
        cp_async_commit();
    };

    float2 acc[RI][4];     // FP32 chunk sums (even, odd elements)
    double tot[RI][4];     // FP64 region sums
    float mx[RI][4];       // region maxima
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            acc[i][j] = make_float2(0.f, 0.f);
            tot[i][j] = 0.0;
            mx[i][j] = 0.f;
        }

    load_chunk(0, 0);
    int region = 0, since_flush = 0;
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        if (c + 1 < nchunks) {
            load_chunk(c + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float* Ab = As + buf * TA * LDS;
        const float* Bb = Bs + buf * TB * LDS;
        // unroll 1 for the max family alone (28.8 vs 33.8 ms on C3, tools/simt_c3.py), 2 with sums
#if CIL_SIMT_EXP == 3
#pragma unroll
#else
#pragma unroll(DO_SUM ? 2 : 1)
#endif
        for (int kk = 0; kk < BK; kk += 4) {
            float4 av[RI], bv[4];
#pragma unroll
            for (int i = 0; i < RI; ++i) av[i] = *reinterpret_cast<const float4*>(Ab + (ty + 8 * i) * LDS + kk);
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = *reinterpret_cast<const float4*>(Bb + (tx + 16 * j) * LDS + kk);
#pragma unroll
            for (int i = 0; i < RI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 d0 = sub2(make_float2(av[i].x, av[i].y), make_float2(bv[j].x, bv[j].y));
                    const float2 d1 = sub2(make_float2(av[i].z, av[i].w), make_float2(bv[j].z, bv[j].w));
                    if (DO_MAX) {
#if CIL_SIMT_EXP == 4
                        const float t = fmaxf(fabsf(d0.x), fmaxf(fabsf(d0.y), fabsf(d1.x)));
                        mx[i][j] = fmaxf(mx[i][j], fmaxf(t, fabsf(d1.y)));
#else
                        mx[i][j] = absmax3(mx[i][j], d0.x, d0.y);
                        mx[i][j] = absmax3(mx[i][j], d1.x, d1.y);
#endif
                    }
                    if (DO_SUM) {
                        acc[i][j] = __ffma2_rn(d0, d0, acc[i][j]);
                        acc[i][j] = __ffma2_rn(d1, d1, acc[i][j]);
                    }
                }
        }
        __syncthreads();
        const bool region_end = (c + 1 == c_end0) || (c + 1 == c_end1) || (c + 1 == nchunks);
        if (DO_SUM && (++since_flush == FLUSH || region_end)) {
            since_flush = 0;
#pragma unroll
            for (int i = 0; i < RI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    tot[i][j] += (double)acc[i][j].x + (double)acc[i][j].y;
                    acc[i][j] = make_float2(0.f, 0.f);
                }
        }
        if (region_end && c + 1 < nchunks) {
#pragma unroll
            for (int i = 0; i < RI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int e = (region * NP + i * 4 + j) * NTHR + tid;
                    if (DO_SUM) { rs_sum[e] = tot[i][j]; tot[i][j] = 0.0; }
                    if (DO_MAX) { rs_max[e] = mx[i][j]; mx[i][j] = 0.f; }
                }
            ++region;
            since_flush = 0;
        }
    }

    // ------------------------------------------------------------- epilogue
    // Measures in FP64 from the region results, each with a rigorous bound E of its error against
    // the exact FP64 value of the plain definition (u = 2^-24):
    //  - value region: differences fl(a - b) carry relative error u; the max is then exact up to u
    //    (rounding is monotone), the FP32 sums of <= 64 squares carry relative error <= 67 u
    //    (FFMA chains of 64 terms, flushed to FP64), i.e. <= 34 u on a_0 = sqrt(w s_0);
    //  - derivative regions: the stored differences D a, D b are themselves rounded, so each element
    //    of D a - D b is within u (|D a| + |D b|) + u |result| of the exact D(a - b): the max moves by
    //    <= u (max|D a| + max|D b|) + u m, the root of the sum by <= u (|D a| + |D b|) + 35 u sqrt(s)
    //    (per-row max / norm of the stored differences: statA / statB);
    //  - the measures combine these monotonically (sums add bounds, max takes the max, the
    //    Euclidean combination of W12 is 1-Lipschitz in each part).
    // A pair is binned at the upper end d + E and listed for the FP64 re-check when a radius lies in
    // (d - E, d + E] (recheck.cu) — the counts are those of the plain definition.
    const double h = a.bp.h, w = a.bp.w, ih = 1.0 / h, ih2 = 1.0 / (h * h);
    const double U = 5.9604644775390625e-08;            // 2^-24
    const int nreg = a.g.nreg;
    // The last region's results leave the registers for the (free) operand buffers, so the epilogue
    // is a rolled loop over this thread's pairs: its code (FP64, per-measure) stays out of the main
    // loop's register allocation (the unrolled epilogue cost the max family ~20 % through a worse
    // allocation of the chunk loop, tools/simt_ab.sh) and the kernel stays small.
    double* last_sum = reinterpret_cast<double*>(As);                  // [NP][NTHR]
    float* last_max = reinterpret_cast<float*>(last_sum + (DO_SUM ? NP * NTHR : 0));   // [NP][NTHR]
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (DO_SUM) last_sum[(i * 4 + j) * NTHR + tid] = tot[i][j];
            if (DO_MAX) last_max[(i * 4 + j) * NTHR + tid] = mx[i][j];
        }
#pragma unroll 1
    for (int pi = 0; pi < NP; ++pi) {
        const int i = pi >> 2, j = pi & 3;
        const int64_t gi = row0 + ty + 8 * i;
        const int64_t gj = col0 + tx + 16 * j;
        if (gi >= a.rowsA || gj >= a.rowsB) continue;
        {
            float4 sa = make_float4(0.f, 0.f, 0.f, 0.f), sb = sa;
            if (nreg > 1) {
                sa = __ldg(reinterpret_cast<const float4*>(a.statA + ((int64_t)p * a.rowsA + gi) * 4));
                sb = __ldg(reinterpret_cast<const float4*>(a.statB + ((int64_t)p * a.rowsB + gj) * 4));
            }
            double s[3] = {0.0, 0.0, 0.0}, m[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                if (r >= nreg) break;
                const bool last = (r == nreg - 1);
                const int e = (r * NP + pi) * NTHR + tid;
                if (DO_SUM) s[r] = last ? last_sum[pi * NTHR + tid] : rs_sum[e];
                if (DO_MAX) m[r] = last ? (double)last_max[pi * NTHR + tid] : (double)rs_max[e];
            }
            const double sw = sqrt(w);
            const double a0 = sqrt(w * s[0]), ax = sqrt(w * s[1] * ih2), ay = sqrt(w * s[2] * ih2);
            const double m0 = m[0], mxx = m[1] * ih, myy = m[2] * ih;
            const double ea0 = 34.0 * U * a0;
            const double eax = sw * ih * (35.0 * U * sqrt(s[1]) + 1.0001 * U * ((double)sa.z + (double)sb.z));
            const double eay = sw * ih * (35.0 * U * sqrt(s[2]) + 1.0001 * U * ((double)sa.w + (double)sb.w));
            const double em0 = 1.0001 * U * m0;
            const double emx = ih * (1.0001 * U * ((double)sa.x + (double)sb.x) + 2.0 * U * m[1]);
            const double emy = ih * (1.0001 * U * ((double)sa.y + (double)sb.y) + 2.0 * U * m[2]);
            const int64_t rs = gi / a.sp.row_seg, cs = gj / a.sp.col_seg;
            for (int q = 0; q < nq; ++q) {
                if (!((a.qmask >> q) & 1u)) continue;
                const int kind = a.bp.slot[q];
                double d, E;
                switch (kind) {
                    case 0: d = a0; E = ea0; break;
                    case 1: d = m0; E = em0; break;
                    case 2: d = a0 + ax + ay; E = ea0 + eax + eay; break;
                    case 3: d = sqrt(a0 * a0 + ax * ax + ay * ay); E = ea0 + eax + eay; break;
                    case 4: d = fmax(m0, fmax(mxx, myy)); E = fmax(em0, fmax(emx, emy)); break;
                    default: d = m0 + mxx + myy; E = em0 + emx + emy; break;
                }
                E += 1e-14 * d;                  // FP64 evaluation of d and of the bound
                if (a.range) {               // distance-range mode (adaptive radii)
                    unsigned long long* rg = a.range + ((int64_t)p * nq + q) * 2;
                    if (d > 0.0) atomicMin(&rg[0], (unsigned long long)__double_as_longlong(d));
                    atomicMax(&rg[1], (unsigned long long)__double_as_longlong(d));
                    continue;
                }
                const double* T = thr_s + q * M;
                const double hi = d + E;
                int b = 0;
                while (b < M && hi < T[b]) ++b;
                if (b < M && d - E < T[b] && !(SYM && gi > gj)) {
                    const uint32_t idx = atomicAdd(a.ctr, 1u);
                    if (idx < a.cap)
                        a.list[idx] = make_uint4((uint32_t)p, (uint32_t)gi, (uint32_t)gj, (uint32_t)b | ((uint32_t)kind << 8));
                }
                if (a.binout) {              // bin-matrix mode (bootstrap, Alg. A1 / A2)
                    CIL_CHECK(gi < a.rowsA && gj < a.rowsB && q < nq);
                    a.binout[(((int64_t)p * nq + q) * a.rowsA + gi) * a.rowsB + gj] = (uint8_t)b;
                    // d(i, j) and d(j, i) are bit-identical here (exact negations, same order), so
                    // a straddling tile writing both orders writes equal bytes
                    if (SYM) a.binout[(((int64_t)p * nq + q) * a.rowsA + gj) * a.rowsB + gi] = (uint8_t)b;
                    continue;
                }
                if (b == 0) continue;
                if (use_sh) {
                    const int loc = (int)((rs - rs0) * ncs + (cs - cs0));
                    atomicAdd(&hist_s[(loc * nq + q) * (M + 1) + b], 1u);
                } else {
                    CIL_CHECK(rs < a.sp.n_rs && cs < a.sp.n_cs);
                    atomicAdd((unsigned long long*)&a.hist[hist_index(a.sp, nq, M, p, rs, cs, q, b)], 1ull);
                }
            }
        }
    }
    if (use_sh) {
        __syncthreads();
        for (int t = tid; t < hist_len; t += NTHR) {
            const uint32_t v = hist_s[t];
            if (v == 0u) continue;
            const int b = t % (M + 1);
            const int q = (t / (M + 1)) % nq;
            const int loc = t / ((M + 1) * nq);
            const int64_t rs = rs0 + loc / ncs, cs = cs0 + loc % ncs;
            atomicAdd((unsigned long long*)&a.hist[hist_index(a.sp, nq, M, p, rs, cs, q, b)],
                      (unsigned long long)v);
        }
    }
}

static size_t simt_smem(bool do_max, bool do_sum, int ri, int hist_cap) {
    size_t s = sizeof(float) * 2 * (8 * ri + TB) * LDS + sizeof(double) * kMaxMeas * kMaxM;
    if (do_sum) s += sizeof(double) * 2 * 4 * ri * NTHR;
    if (do_max) s += sizeof(float) * 2 * 4 * ri * NTHR;
    s += sizeof(uint32_t) * hist_cap;
    return s;
}

template <bool X, bool Y, int RI, bool SYM>
static cudaError_t launch_simt_t(const SimtArgs& a_in, cudaStream_t st) {
    // shared histogram sized for the segments one tile can touch (else global atomics)
    constexpr int TA = 8 * RI;
    SimtArgs a = a_in;
    const int64_t nrs = (TA + a.sp.row_seg - 1) / a.sp.row_seg + 1, ncs = (TB + a.sp.col_seg - 1) / a.sp.col_seg + 1;
    const int64_t need = nrs * ncs * a.bp.nq * (a.bp.M + 1);
    a.hist_cap = (int)(need < 4096 ? need : 4096);
    const size_t sm = simt_smem(X, Y, RI, a.hist_cap);
    static SmemAttrOnce attr;
    if (cudaError_t e = attr.ensure(k_simt<X, Y, RI, SYM>, (int)simt_smem(X, Y, RI, 4096)); e != cudaSuccess) return e;
    dim3 grid((unsigned)((a.rowsB + TB - 1) / TB), (unsigned)((a.rowsA + TA - 1) / TA), (unsigned)a.P);
    ProfScope ps_(K_SIMT, st);
    k_simt<X, Y, RI, SYM><<<grid, NTHR, sm, st>>>(a);
    note_launch();
    return cudaGetLastError();
}

template <bool SYM>
static cudaError_t launch_simt_s(const SimtArgs& a, cudaStream_t st) {
    if (a.do_max && a.do_sum) return launch_simt_t<true, true, 4, SYM>(a, st);
    if (a.do_max) {
        // max family alone: 8 x 4 pairs per thread (12 LDS.128 per 128 element-pairs instead of 8 per 64)
        return launch_simt_t<true, false, 8, SYM>(a, st);
    }
    return launch_simt_t<false, true, 4, SYM>(a, st);
}

cudaError_t launch_simt(const SimtArgs& a, cudaStream_t st) {
    if (a.rowsA == 0 || a.rowsB == 0) return cudaSuccess;
    return a.sym ? launch_simt_s<true>(a, st) : launch_simt_s<false>(a, st);
}

CIL_OOB_READER(oob_simt)

}  // namespace cil
