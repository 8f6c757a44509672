// max16.cu — step a3 for the max family (Linf, W1inf, W1infsum; Eqs. (6), (9), (10),
// PAPER.md:182-190) on the CUDA cores' integer pipes, fused with radius binning (Eq. (1)).
//
// The three max sub-norms m_al = max_e |D_al (a - b)_e| (al in {value, D_x, D_y}) are computed on
// 15-bit fixed-point copies of the operands: per item and region one scale over both panels (A and
// B must share it): centre c_al = (max v + min v) / 2, half range r_al, s_al = r_al / 16383,
// q = rint((v - c_al) / s_al) in [-16383, 16383] (a - b does not see c_al; the
// differences of the derivative regions are formed in FP64 first, so q is within 0.5 + 1e-11 of
// (v - c_al) / s_al of the EXACT v).  Then for one pair
//     |s_al * max_e |q_a - q_b| - m_al| <= (1 + 1e-9) s_al      (max is 1-Lipschitz in the sup norm)
// — a rigorous interval.  A pair is binned at the upper end d + E and listed for the exact FP64
// re-check (recheck.cu) when a radius lies in (d - E, d + E], so the counts are those of the plain
// definition.  For the paper's workloads the band is ~1e-4 d wide (re-check fraction in DESIGN.md).
//
// Why: FP32 |a - b| max costs FADD2 + FMNMX3 per two element-pairs and is bound by the FP32
// subtraction rate (57 element-pairs per SM-cycle measured, profiles/r02_maxmix.txt); this mix
// reaches 89-91 per SM-cycle register-only (tools/maxmix3_bench.cu, cil_diag_alu_ceiling(3)), and
// the operands are half the bytes.
//
// Kernels: k_max16_reg, CTA = 128 threads = 64 A rows x 64 B rows x one region, 8 x 4 pairs per
// thread; k_max16_bin, the binning epilogue over the per-pair region maxima.  Operands are stored
// biased, A as q + 16384 and B as -q + 16384 (both in [1, 32767]), so ONE 32-bit integer add of two
// packed words gives both 16-bit lanes t = q_a - q_b + 32768 in [2, 65534] with no carry between
// the lanes — issued as IMAD on the FMA pipe, which leaves the integer ALU pipe to the
// VIMNMX3.U16x2 running max / min of t (max |q_a - q_b| = max(max t - 32768, 32768 - min t)); an
// all-ALU VIADD.16x2 form ran at ~0.7 of this.  k-chunks of 64 elements (128 B per row) double-
// buffered in shared memory with cp.async (rows padded to 144 B -> conflict-free LDS.128).
#include "cil_internal.cuh"

namespace cil {

namespace {
constexpr int TB = 64;               // B rows per CTA
constexpr int RI = 8;                // A rows per thread (8 x 4 pairs)
constexpr int TA = 8 * RI;           // A rows per CTA
constexpr int NTHR = 128;
constexpr int BKW = kMax16BK / 2;    // 32-bit words per row per chunk
constexpr int LDW = BKW + 4;         // padded row stride (words)
constexpr double kQ = 16383.0;       // |q| <= 16383: q + 16384 in [1, 32767], t = q_a - q_b + 32768 in [2, 65534]

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Order-preserving map of FP32 onto uint32 (for atomicMax / atomicMin of signed values)
__device__ __forceinline__ unsigned ord_f(float f) {
    const unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f(unsigned u) {     // 0 (nothing merged) -> 0
    return u == 0u ? 0.f : __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
// centre and scale of region r of item p from the range pass: rng[p][r] = {ord(max), ord(-min)}
// (scale 0 for a constant region; both are exact FP64 functions of two floats, so the pack and the
// epilogue see the same values)
__device__ __forceinline__ double centre16(const unsigned* rng, int64_t p, int r) {
    return 0.5 * ((double)unord_f(rng[p * 8 + 2 * r]) - (double)unord_f(rng[p * 8 + 2 * r + 1]));
}
__device__ __forceinline__ double scale16(const unsigned* rng, int64_t p, int r) {
    const double hr = 0.5 * ((double)unord_f(rng[p * 8 + 2 * r]) + (double)unord_f(rng[p * 8 + 2 * r + 1]));
    return hr > 0.0 ? hr / kQ : 0.0;
}

constexpr int kBias = 16384;        // storage bias of both panels

// max |q_a - q_b| of one pair from its packed running max / min of t = q_a - q_b + 32768
__device__ __forceinline__ int absmax_pair(uint32_t mx, uint32_t mn) {
    const int hi = (int)max(mx & 0xffffu, mx >> 16) - 32768;
    const int lo = (int)min(mn & 0xffffu, mn >> 16) - 32768;
    return max(hi, -lo);
}
// a + b as IMAD a * one + b (one = 1 from the kernel arguments, so ptxas keeps the FMA-pipe form)
__device__ __forceinline__ uint32_t add_fma(uint32_t a, uint32_t one, uint32_t b) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(one), "r"(b));
    return d;
}
}  // namespace

// ----------------------------------------------------------------- pass 1: per-item range
// One CTA per panel row: max and min of x, D_x x, D_y x (differences in FP64, rounded outwards to
// FP32), atomically merged into rng[p][r] = {ord(max), ord(-min)} (both atomicMax; zero-initialised
// by launch_pack16, 0 = no value seen).
__global__ void __launch_bounds__(256) k_range16(RowSrc src, int64_t rows, AugGeom g, unsigned* rng,
                                                 int32_t* status) {
    const int64_t p = blockIdx.y, r = blockIdx.x;
    const float* x = row_ptr(src, p, r);
    float hi0 = -INFINITY, lo0 = INFINITY, nfa = 0.f;
    double hx = -INFINITY, lx = INFINITY, hy = -INFINITY, ly = INFINITY;
    const int W = g.W, H = g.H, SH = g.S * g.H;
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    const bool flat = g.nreg >= 2 && (W & 3) == 0 && g.K < (1ll << 31);
    if (!flat) {
        for (int64_t k = (int64_t)threadIdx.x * 4; k < g.K; k += 1024) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(x + k));
            nfa = fmaf(v.x, 0.f, fmaf(v.y, 0.f, fmaf(v.z, 0.f, fmaf(v.w, 0.f, nfa))));
            hi0 = fmaxf(fmaxf(hi0, v.x), fmaxf(fmaxf(v.y, v.z), v.w));
            lo0 = fminf(fminf(lo0, v.x), fminf(fminf(v.y, v.z), v.w));
        }
    }
    if (flat) {                       // one sweep: the value range rides along with the derivative ranges
        // flat float4 sweep: 4 elements of one grid row per thread, the x neighbour of the 4th from
        // the next lane (lane 31: a load), the y neighbours one grid row on (an L1 / L2 hit)
        const uint32_t K = (uint32_t)g.K, Wu = (uint32_t)W, Hu = (uint32_t)H;
        const FastDiv fw(Wu), fh(Hu);
        for (uint32_t base = 0; base < K; base += 1024) {
            const uint32_t e = base + threadIdx.x * 4;
            const bool ok = e < K;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ok) v = __ldg(reinterpret_cast<const float4*>(x + e));
            float nxv = __shfl_down_sync(0xffffffffu, v.x, 1);
            if (!ok) continue;
            nfa = fmaf(v.x, 0.f, fmaf(v.y, 0.f, fmaf(v.z, 0.f, fmaf(v.w, 0.f, nfa))));
            hi0 = fmaxf(fmaxf(hi0, v.x), fmaxf(fmaxf(v.y, v.z), v.w));
            lo0 = fminf(fminf(lo0, v.x), fminf(fminf(v.y, v.z), v.w));
            uint32_t c, hr;
            const uint32_t sr = fw.div(e, c), sp = fh.div(sr, hr);
            if (!(g.gs == 0 || ((g.gs >> sp) & 1u))) continue;     // species mask (R18): 0 derivatives
            const double x0 = v.x, x1 = v.y, x2 = v.z, x3 = v.w;
            hx = fmax(hx, fmax(fmax(x1 - x0, x2 - x1), x3 - x2));
            lx = fmin(lx, fmin(fmin(x1 - x0, x2 - x1), x3 - x2));
            if (c + 4 < Wu) {
                if (ln == 31) nxv = __ldg(x + e + 4);
                const double d = (double)nxv - x3;
                hx = fmax(hx, d); lx = fmin(lx, d);
            }
            if (g.nreg >= 3 && hr + 1 < Hu) {
                const float4 vd = __ldg(reinterpret_cast<const float4*>(x + e + Wu));
                const double d0 = (double)vd.x - x0, d1 = (double)vd.y - x1, d2 = (double)vd.z - x2,
                             d3 = (double)vd.w - x3;
                hy = fmax(hy, fmax(fmax(d0, d1), fmax(d2, d3)));
                ly = fmin(ly, fmin(fmin(d0, d1), fmin(d2, d3)));
            }
        }
    } else if (g.nreg >= 2) {
        for (int sr = w; sr < SH; sr += 8) {
            const int s = sr / H;
            if (!(g.gs == 0 || ((g.gs >> s) & 1u))) continue;     // species mask (R18): 0 derivatives
            const bool has_dy = g.nreg >= 3 && (sr % H) + 1 < H;
            const float* xr = x + (int64_t)sr * W;
            for (int c = ln; c < W; c += 32) {
                const double xe = __ldg(xr + c);
                if (c + 1 < W) {
                    const double d = (double)__ldg(xr + c + 1) - xe;
                    hx = fmax(hx, d); lx = fmin(lx, d);
                }
                if (has_dy) {
                    const double d = (double)__ldg(xr + W + c) - xe;
                    hy = fmax(hy, d); ly = fmin(ly, d);
                }
            }
        }
    }
    // masked species contribute zeros to the derivative regions
    if (g.gs != 0) { hx = fmax(hx, 0.0); lx = fmin(lx, 0.0); hy = fmax(hy, 0.0); ly = fmin(ly, 0.0); }
    float v[6] = {hi0, lo0, __double2float_ru(hx), __double2float_rd(lx), __double2float_ru(hy), __double2float_rd(ly)};
#pragma unroll
    for (int k = 0; k < 6; ++k)
        for (int o = 16; o > 0; o >>= 1) {
            const float t = __shfl_xor_sync(0xffffffffu, v[k], o);
            v[k] = (k & 1) ? fminf(v[k], t) : fmaxf(v[k], t);
        }
    if (ln == 0) {
        for (int rg = 0; rg < g.nreg; ++rg) {
            if (v[2 * rg] >= v[2 * rg + 1]) {           // the warp saw at least one value
                atomicMax(&rng[p * 8 + 2 * rg], ord_f(v[2 * rg]));
                atomicMax(&rng[p * 8 + 2 * rg + 1], ord_f(-v[2 * rg + 1]));
            }
        }
    }
    if (__syncthreads_or(nfa != nfa) && threadIdx.x == 0) atomicOr(&status[p], CIL_ITEM_NONFINITE);
}

// ----------------------------------------------------------------- pass 2: quantise
// One CTA per panel row: out = [q(x) | q(D_x x) | q(D_y x)], regions zero-padded to kMax16BK
// elements (in both panels, so padding adds |0 - 0| to the max), q = rint((v - c) / s) in FP64 (v of
// the derivative regions = the exact FP64 difference, 0 for masked species); negated for the B panel.
__global__ void __launch_bounds__(256) k_pack16(RowSrc src, int64_t rows, AugGeom g, const unsigned* rng,
                                                int16_t* __restrict__ out, int neg) {
    const int64_t p = blockIdx.y, r = blockIdx.x;
    const float* x = row_ptr(src, p, r);
    int16_t* o = out + (p * rows + r) * g.off[3];
    const double sgn = neg ? -1.0 : 1.0;
    double inv[3], cen[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double s = k < g.nreg ? scale16(rng, p, k) : 0.0;
        inv[k] = s > 0.0 ? sgn / s : 0.0;
        cen[k] = k < g.nreg ? centre16(rng, p, k) : 0.0;
    }
    for (int64_t k = (int64_t)threadIdx.x * 4; k < g.off[1]; k += 1024) {
        short4 q = make_short4(kBias, kBias, kBias, kBias);
        if (k < g.K) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(x + k));
            q = make_short4((short)(__double2int_rn((v.x - cen[0]) * inv[0]) + kBias),
                            (short)(__double2int_rn((v.y - cen[0]) * inv[0]) + kBias),
                            (short)(__double2int_rn((v.z - cen[0]) * inv[0]) + kBias),
                            (short)(__double2int_rn((v.w - cen[0]) * inv[0]) + kBias));
        }
        *reinterpret_cast<short4*>(o + k) = q;
    }
    if (g.nreg < 2) return;
    const int W = g.W, H = g.H, SH = g.S * g.H;
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if ((W & 3) == 0 && g.K < (1ll << 31)) {
        // flat float4 sweep (as in k_range16): D_x rows are W - 1 long (scalar 2-byte stores), D_y
        // rows W long (one 8-byte store per 4 values)
        const uint32_t K = (uint32_t)g.K, Wu = (uint32_t)W, Hu = (uint32_t)H;
        const FastDiv fw(Wu), fh(Hu);
        auto qz = [&](double d, int k) { return (int16_t)(__double2int_rn((d - cen[k]) * inv[k]) + kBias); };
        for (uint32_t base = 0; base < K; base += 1024) {
            const uint32_t e = base + threadIdx.x * 4;
            const bool ok = e < K;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ok) v = __ldg(reinterpret_cast<const float4*>(x + e));
            float nxv = __shfl_down_sync(0xffffffffu, v.x, 1);
            if (!ok) continue;
            uint32_t c, hr;
            const uint32_t sr = fw.div(e, c), sp = fh.div(sr, hr);
            const bool grad = g.gs == 0 || ((g.gs >> sp) & 1u);
            const double x0 = v.x, x1 = v.y, x2 = v.z, x3 = v.w;
            int16_t* ox = o + g.off[1] + (int64_t)sr * (W - 1) + c;
            ox[0] = qz(grad ? x1 - x0 : 0.0, 1);
            ox[1] = qz(grad ? x2 - x1 : 0.0, 1);
            ox[2] = qz(grad ? x3 - x2 : 0.0, 1);
            if (c + 4 < Wu) {
                if (ln == 31) nxv = __ldg(x + e + 4);
                ox[3] = qz(grad ? (double)nxv - x3 : 0.0, 1);
            }
            if (g.nreg >= 3 && hr + 1 < Hu) {
                double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
                if (grad) {
                    const float4 vd = __ldg(reinterpret_cast<const float4*>(x + e + Wu));
                    d0 = (double)vd.x - x0; d1 = (double)vd.y - x1; d2 = (double)vd.z - x2; d3 = (double)vd.w - x3;
                }
                *reinterpret_cast<short4*>(o + g.off[2] + (int64_t)(sr - sp) * W + c) =
                    make_short4(qz(d0, 2), qz(d1, 2), qz(d2, 2), qz(d3, 2));
            }
        }
    } else {
    for (int sr = w; sr < SH; sr += 8) {
        const int s = sr / H;
        const bool grad = g.gs == 0 || ((g.gs >> s) & 1u);
        const bool has_dy = g.nreg >= 3 && (sr % H) + 1 < H;
        const float* xr = x + (int64_t)sr * W;
        for (int c = ln; c < W; c += 32) {
            const double xe = __ldg(xr + c);
            const double dx = grad && c + 1 < W ? (double)__ldg(xr + c + 1) - xe : 0.0;
            const double dy = grad && has_dy ? (double)__ldg(xr + W + c) - xe : 0.0;
            if (c + 1 < W)
                o[g.off[1] + (int64_t)sr * (W - 1) + c] = (int16_t)(__double2int_rn((dx - cen[1]) * inv[1]) + kBias);
            if (has_dy)
                o[g.off[2] + (int64_t)sr * W - (int64_t)s * W + c] = (int16_t)(__double2int_rn((dy - cen[2]) * inv[2]) + kBias);
        }
    }
    }
    for (int64_t t = g.Kx + threadIdx.x; t < g.off[2] - g.off[1]; t += 256) o[g.off[1] + t] = kBias;
    if (g.nreg >= 3)
        for (int64_t t = g.Ky + threadIdx.x; t < g.off[3] - g.off[2]; t += 256) o[g.off[2] + t] = kBias;
}

// ----------------------------------------------------------------- the max-family tile kernels
// k_max16_reg: one CTA per (64 x 64 tile, region): the packed running max / min over the region's
// chunks, then the per-pair region maximum max |q_a - q_b| (u16) to dmax[p][r][i][j] (staged in
// shared memory, stored row-contiguous).  Splitting by region triples the work units (3072 for C3
// instead of 1024 tiles over 444 resident CTAs), so the last partial wave costs ~3 % instead of ~12 %.
// k_max16_bin: the epilogue over the same tile grid — interval, bin at the upper end, re-check list,
// histogram or bin matrix.
#ifndef CIL_M16_EXP
#define CIL_M16_EXP 0   // code-generation experiments (tools/simt_var_build.sh); 0 = product
#endif
template <bool SYM>
__global__ void __launch_bounds__(NTHR, CIL_M16_EXP == 1 ? 4 : 3) k_max16_reg(Max16Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* As = reinterpret_cast<uint32_t*>(smem_raw);           // [2][TA][LDW]
    uint32_t* Bs = As + 2 * TA * LDW;                                // [2][TB][LDW]

    const int nreg = a.g.nreg;
    const int p = blockIdx.z / nreg, region = blockIdx.z % nreg;
    if (a.status[p] & CIL_ITEM_BADRADII) return;
    const int64_t row0 = (int64_t)blockIdx.y * TA;
    const int64_t col0 = (int64_t)blockIdx.x * TB;
    if (a.tri && row0 / a.sp.row_seg >= (min(col0 + TB, a.rowsB) - 1) / a.sp.col_seg) return;
    if (SYM && row0 >= col0 + TB) return;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int ty = (warp >> 1) * 4 + (lane >> 3);   // 0..7
    const int tx = (warp & 1) * 8 + (lane & 7);     // 0..15

    const int16_t* Ag = a.A + ((int64_t)p * a.rowsA) * a.Kaug;
    const int16_t* Bg = a.B + ((int64_t)p * a.rowsB) * a.Kaug;
    const int cb = (int)(a.g.off[region] / kMax16BK), ce = (int)(a.g.off[region + 1] / kMax16BK);

    auto load_chunk = [&](int c, int buf) {
        const int64_t k0 = (int64_t)c * kMax16BK;
#pragma unroll
        for (int t = 0; t < (TA * 8) / NTHR; ++t) {      // 8 x 16 B per row
            const int idx = tid + t * NTHR;
            const int r = idx >> 3, v = idx & 7;
            const int64_t gr = row0 + r;
            const bool ok = gr < a.rowsA;
            cp_async16(As + (buf * TA + r) * LDW + v * 4, Ag + (ok ? gr : 0) * a.Kaug + k0 + v * 8, ok);
        }
#pragma unroll
        for (int t = 0; t < (TB * 8) / NTHR; ++t) {
            const int idx = tid + t * NTHR;
            const int r = idx >> 3, v = idx & 7;
            const int64_t gc = col0 + r;
            const bool ok = gc < a.rowsB;
            cp_async16(Bs + (buf * TB + r) * LDW + v * 4, Bg + (ok ? gc : 0) * a.Kaug + k0 + v * 8, ok);
        }
        cp_async_commit();
    };

    uint32_t mx[RI][4], mn[RI][4];   // packed (2 x u16) running max / min of t = q_a - q_b + 32768
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { mx[i][j] = 0u; mn[i][j] = 0xffffffffu; }

    const uint32_t one = a.one;
    if (cb < ce) load_chunk(cb, 0);
    for (int c = cb; c < ce; ++c) {
        const int buf = (c - cb) & 1;
        if (c + 1 < ce) {
            load_chunk(c + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const uint32_t* Ab = As + buf * TA * LDW;
        const uint32_t* Bb = Bs + buf * TB * LDW;
#if CIL_M16_EXP == 2
#pragma unroll 1
#elif CIL_M16_EXP == 3
#pragma unroll 2
#else
#pragma unroll 4
#endif
        for (int kk = 0; kk < BKW; kk += 4) {
            uint4 av[RI], bv[4];
#pragma unroll
            for (int i = 0; i < RI; ++i) av[i] = *reinterpret_cast<const uint4*>(Ab + (ty + 8 * i) * LDW + kk);
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = *reinterpret_cast<const uint4*>(Bb + (tx + 16 * j) * LDW + kk);
#pragma unroll
            for (int i = 0; i < RI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t d0 = add_fma(av[i].x, one, bv[j].x), d1 = add_fma(av[i].y, one, bv[j].y);
                    const uint32_t d2 = add_fma(av[i].z, one, bv[j].z), d3 = add_fma(av[i].w, one, bv[j].w);
                    mx[i][j] = __vimax3_u16x2(mx[i][j], d0, d1);
                    mn[i][j] = __vimin3_u16x2(mn[i][j], d0, d1);
                    mx[i][j] = __vimax3_u16x2(mx[i][j], d2, d3);
                    mn[i][j] = __vimin3_u16x2(mn[i][j], d2, d3);
                }
        }
        __syncthreads();
    }
    // stage the 64 x 64 region maxima (an empty region gives 0) and store them row-contiguous
    uint16_t* tile = reinterpret_cast<uint16_t*>(As);                // [TA][TB]
#pragma unroll
    for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
            tile[(ty + 8 * i) * TB + tx + 16 * j] = cb < ce ? (uint16_t)absmax_pair(mx[i][j], mn[i][j]) : (uint16_t)0;
    __syncthreads();
    uint16_t* out = a.dmax + ((int64_t)p * nreg + region) * a.rowsA * a.rowsB;
    for (int t = tid; t < TA * TB; t += NTHR) {
        const int r = t / TB, cc = t % TB;
        const int64_t gi = row0 + r, gj = col0 + cc;
        if (gi < a.rowsA && gj < a.rowsB) {
            CIL_CHECK(((int64_t)p * nreg + region + 1) * a.rowsA * a.rowsB <= a.dmax_elems);
            out[gi * a.rowsB + gj] = tile[t];
        }
    }
}

template <bool SYM>
__global__ void __launch_bounds__(256) k_max16_bin(Max16Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nq = a.bp.nq, M = a.bp.M;
    double* thr_s = reinterpret_cast<double*>(smem_raw);              // [nq*M]
    uint32_t* hist_s = reinterpret_cast<uint32_t*>(thr_s + ((nq * M + 1) & ~1));

    const int p = blockIdx.z;
    if (a.status[p] & CIL_ITEM_BADRADII) return;
    const int64_t row0 = (int64_t)blockIdx.y * TA;
    const int64_t col0 = (int64_t)blockIdx.x * TB;
    if (a.tri && row0 / a.sp.row_seg >= (min(col0 + TB, a.rowsB) - 1) / a.sp.col_seg) return;
    if (SYM && row0 >= col0 + TB) return;
    const int tid = threadIdx.x;
    for (int t = tid; t < nq * M; t += 256) thr_s[t] = a.thr[(int64_t)p * a.thr_stride + t];
    const int64_t rlast = min(row0 + TA, a.rowsA) - 1, clast = min(col0 + TB, a.rowsB) - 1;
    const int64_t rs0 = row0 / a.sp.row_seg, cs0 = col0 / a.sp.col_seg;
    const int nrs = (int)(rlast / a.sp.row_seg - rs0 + 1), ncs = (int)(clast / a.sp.col_seg - cs0 + 1);
    const int hist_len = nrs * ncs * nq * (M + 1);
    const bool use_sh = hist_len <= a.hist_cap;
    if (use_sh)
        for (int t = tid; t < hist_len; t += 256) hist_s[t] = 0u;
    __syncthreads();

    const double h = a.bp.h, ih = 1.0 / h;
    const int nreg = a.g.nreg;
    const double s0 = scale16(a.maxbits, p, 0);
    const double sx = nreg > 1 ? scale16(a.maxbits, p, 1) * ih : 0.0;
    const double sy = nreg > 2 ? scale16(a.maxbits, p, 2) * ih : 0.0;
    // per-region error: 2 (0.5 + 1e-11) s of the quantisation, FP64 products (1e-15 relative)
    const double E0 = (1.0 + 1e-9) * s0, Ex = (1.0 + 1e-9) * sx, Ey = (1.0 + 1e-9) * sy;
    const int64_t plane = a.rowsA * a.rowsB;
    const uint16_t* dm = a.dmax + (int64_t)p * nreg * plane;
    for (int t = tid; t < TA * TB; t += 256) {
        const int64_t gi = row0 + t / TB, gj = col0 + t % TB;
        if (gi >= a.rowsA || gj >= a.rowsB) continue;
        const int64_t o = gi * a.rowsB + gj;
        const double m0 = s0 * (double)dm[o];
        const double mxx = nreg > 1 ? sx * (double)dm[plane + o] : 0.0;
        const double myy = nreg > 2 ? sy * (double)dm[2 * plane + o] : 0.0;
        const int64_t rsg = gi / a.sp.row_seg, csg = gj / a.sp.col_seg;
        for (int q = 0; q < nq; ++q) {
            if (!((a.qmask >> q) & 1u)) continue;
            const int kind = a.bp.slot[q];
            double d, E;
            switch (kind) {
                case 1: d = m0; E = E0; break;                                                   // Eq. (6)
                case 4: d = fmax(m0, fmax(mxx, myy)); E = fmax(E0, fmax(Ex, Ey)); break;         // Eq. (9)
                default: d = m0 + mxx + myy; E = E0 + Ex + Ey; break;                            // Eq. (10)
            }
            E += 1e-14 * d;
            const double* T = thr_s + q * M;
            const double hi = d + E;
            int b = 0;
            while (b < M && hi < T[b]) ++b;
            if (b < M && d - E < T[b] && !(SYM && gi > gj)) {
                const uint32_t idx = atomicAdd(a.ctr, 1u);
                if (idx < a.cap)
                    a.list[idx] = make_uint4((uint32_t)p, (uint32_t)gi, (uint32_t)gj, (uint32_t)b | ((uint32_t)kind << 8));
            }
            if (a.binout) {
                CIL_CHECK(gi < a.rowsA && gj < a.rowsB && q < nq);
                a.binout[(((int64_t)p * nq + q) * a.rowsA + gi) * a.rowsB + gj] = (uint8_t)b;
                if (SYM) a.binout[(((int64_t)p * nq + q) * a.rowsA + gj) * a.rowsB + gi] = (uint8_t)b;
                continue;
            }
            if (b == 0) continue;
            if (use_sh) {
                const int loc = (int)((rsg - rs0) * ncs + (csg - cs0));
                atomicAdd(&hist_s[(loc * nq + q) * (M + 1) + b], 1u);
            } else {
                CIL_CHECK(rsg < a.sp.n_rs && csg < a.sp.n_cs);
                atomicAdd((unsigned long long*)&a.hist[hist_index(a.sp, nq, M, p, rsg, csg, q, b)], 1ull);
            }
        }
    }
    if (use_sh) {
        __syncthreads();
        for (int t = tid; t < hist_len; t += 256) {
            const uint32_t v = hist_s[t];
            if (v == 0u) continue;
            const int b = t % (M + 1);
            const int q = (t / (M + 1)) % nq;
            const int loc = t / ((M + 1) * nq);
            const int64_t rsg = rs0 + loc / ncs, csg = cs0 + loc % ncs;
            atomicAdd((unsigned long long*)&a.hist[hist_index(a.sp, nq, M, p, rsg, csg, q, b)], (unsigned long long)v);
        }
    }
}

static size_t max16_smem_reg() { return sizeof(uint32_t) * 2 * (TA + TB) * LDW; }
static size_t max16_smem_bin(int hist_cap, int nqM) {
    return sizeof(double) * ((nqM + 1) & ~1) + sizeof(uint32_t) * hist_cap;
}

cudaError_t launch_pack16(int P, const RowSrc& asrc, int64_t rowsA, const RowSrc& bsrc, int64_t rowsB,
                          const AugGeom& g, unsigned* maxbits, int16_t* outA, int16_t* outB, int32_t* status,
                          cudaStream_t st) {
    if (rowsA == 0 || rowsB == 0) return cudaSuccess;
    ProfScope ps_(K_PACK, st);
    if (cudaError_t e = cudaMemsetAsync(maxbits, 0, sizeof(unsigned) * 8 * (size_t)P, st); e != cudaSuccess) return e;
    k_range16<<<dim3((unsigned)rowsA, (unsigned)P), 256, 0, st>>>(asrc, rowsA, g, maxbits, status);
    k_range16<<<dim3((unsigned)rowsB, (unsigned)P), 256, 0, st>>>(bsrc, rowsB, g, maxbits, status);
    k_pack16<<<dim3((unsigned)rowsA, (unsigned)P), 256, 0, st>>>(asrc, rowsA, g, maxbits, outA, 0);
    k_pack16<<<dim3((unsigned)rowsB, (unsigned)P), 256, 0, st>>>(bsrc, rowsB, g, maxbits, outB, 1);
    note_launch(4);
    return cudaGetLastError();
}

template <bool SYM>
static cudaError_t launch_max16_t(const Max16Args& a_in, cudaStream_t st) {
    Max16Args a = a_in;
    a.one = 1u;
    const int64_t nrs = (TA + a.sp.row_seg - 1) / a.sp.row_seg + 1, ncs = (TB + a.sp.col_seg - 1) / a.sp.col_seg + 1;
    const int64_t need = nrs * ncs * a.bp.nq * (a.bp.M + 1);
    a.hist_cap = (int)(need < 4096 ? need : 4096);
    static SmemAttrOnce attr;
    if (cudaError_t e = attr.ensure(k_max16_reg<SYM>, (int)max16_smem_reg()); e != cudaSuccess) return e;
    const unsigned gx = (unsigned)((a.rowsB + TB - 1) / TB), gy = (unsigned)((a.rowsA + TA - 1) / TA);
    ProfScope ps_(K_SIMT, st);
    k_max16_reg<SYM><<<dim3(gx, gy, (unsigned)(a.P * a.g.nreg)), NTHR, max16_smem_reg(), st>>>(a);
    k_max16_bin<SYM><<<dim3(gx, gy, (unsigned)a.P), 256, max16_smem_bin(a.hist_cap, a.bp.nq * a.bp.M), st>>>(a);
    note_launch(2);
    return cudaGetLastError();
}

cudaError_t launch_max16(const Max16Args& a, cudaStream_t st) {
    if (a.rowsA == 0 || a.rowsB == 0) return cudaSuccess;
    return a.sym ? launch_max16_t<true>(a, st) : launch_max16_t<false>(a, st);
}

CIL_OOB_READER(oob_max16)

}  // namespace cil
