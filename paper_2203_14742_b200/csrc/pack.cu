// pack.cu — step a1 of the hot path: radii validation, centring,
// split-precision operands for the tensor-core Gram, augmented FP32 operands
// [value | D_x | D_y] for the CUDA-core engine.  HBM-bound, one pass per row.
//
// Definitions followed:
//  - distances of pattern differences u = a - b (Eq. (1));
//  - forward difference D_h f = f(x_{j+1}) - f(x_j), taken along
//    W (D_x) and H (D_y) inside each species; the last node is omitted (Neumann
//    ghost; reading R3).  The 1/h factor is applied in
//    the engines' epilogues in FP64, so the fields here are plain differences.
#include <stdlib.h>

#include "cil_internal.cuh"

namespace cil {

// -------------------------------------------------------------------------- prep
// Validates radii (> 0, strictly decreasing) and writes per-item thresholds:
//   thr[p][q][m]  = R (FP64, compared with the measure value)
//   thr2[p][m]    = R^2 / w (FP32), the L2 threshold on the unweighted sum of squares
__global__ void k_prep(int P, int nq, int M, const double* __restrict__ radii, int64_t radii_stride,
                       BinParams bp, double* __restrict__ thr, float* __restrict__ thr2_l2,
                       int32_t* __restrict__ status, int keep_status) {
    const int p = blockIdx.x;
    const double* R = radii + (int64_t)p * radii_stride;
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < nq * M; t += blockDim.x) {
        const int m = t % M;
        const double r = R[t];
        const bool ok = (r > 0.0) && isfinite(r) && (m == 0 || R[t - 1] > r);
        if (!ok) atomicOr(&bad, 1);
        thr[(int64_t)p * nq * M + t] = r;
    }
    if (thr2_l2 != nullptr) {
        // tensor-core thresholds [p][8][M] (FP32), rigorously bracketed for the INT8 engine's interval
        // tests: row 2k = rounded down, 2k + 1 = rounded up, for kind k = 0: L2 as R / sqrt(w) (the
        // engine bins the distance of the unweighted sums), 1: W12 as R^2 / w, 2: W12SUM as R / sqrt(w);
        // row 6: L2 as R^2 / w (nearest; the float split engines)
        const double sw = sqrt(bp.w);
        for (int q = 0; q < nq; ++q) {
            const int kind = bp.slot[q] == 0 ? 0 : bp.slot[q] == 3 ? 1 : bp.slot[q] == 2 ? 2 : -1;
            if (kind < 0) continue;
            for (int m = threadIdx.x; m < M; m += blockDim.x) {
                const double r = R[q * M + m];
                const double v = kind == 1 ? r * r / bp.w : r / sw;
                float* T = thr2_l2 + (int64_t)p * 8 * M;
                T[(2 * kind) * M + m] = __double2float_rd(v * (1.0 - 1e-15));
                T[(2 * kind + 1) * M + m] = __double2float_ru(v * (1.0 + 1e-15));
                if (kind == 0) T[6 * M + m] = (float)(r * r / bp.w);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) status[p] = (keep_status ? status[p] : 0) | (bad ? CIL_ITEM_BADRADII : 0);
}

cudaError_t launch_prep(int P, int nq, int M, const double* radii, int64_t radii_stride,
                        const BinParams& bp, double* thr, float* thr2_l2, int32_t* status,
                        uint64_t* hist, int64_t hist_elems, uint32_t* recheck_ctr, cudaStream_t st,
                        bool keep_status) {
    cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(uint64_t) * hist_elems, st);
    if (e != cudaSuccess) return e;
    if (recheck_ctr) {
        e = cudaMemsetAsync(recheck_ctr, 0, sizeof(uint32_t) * 2, st);
        if (e != cudaSuccess) return e;
    }
    ProfScope ps_(K_PREP, st);
    k_prep<<<P, 128, 0, st>>>(P, nq, M, radii, radii_stride, bp, thr, thr2_l2, status, keep_status ? 1 : 0);
    note_launch();
    return cudaGetLastError();
}

// Fill n doubles with v (device-side constants such as dummy radii: no pageable host copy, so the
// call stays asynchronous and capturable into a CUDA graph).
__global__ void k_fill_f64(double* p, int n, double v) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = v;
}
cudaError_t launch_fill_f64(double* p, int n, double v, cudaStream_t st) {
    k_fill_f64<<<1, 64, 0, st>>>(p, n, v);
    note_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------------------ centre
// c[p][k] = mean of the first nrc rows of the item's column panel, FP64
// accumulation, rounded to FP32.  A numerical device only (conditioning of the
// Gram, DESIGN.md §L2 engine): distances are translation invariant.
__global__ void __launch_bounds__(256) k_center(RowSrc src, int64_t nrc, int64_t K, int64_t Kp,
                                                float* __restrict__ center) {
    const int64_t p = blockIdx.y;
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;   // K % 4 == 0, Kp % 128 == 0
    if (k >= Kp) return;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (k < K) {
        float4 v[16];                                 // nrc <= 16: all loads in flight, then the sums
#pragma unroll
        for (int r = 0; r < 16; ++r)
            v[r] = r < nrc ? __ldg(reinterpret_cast<const float4*>(row_ptr(src, p, r) + k)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            s[0] += (double)v[r].x; s[1] += (double)v[r].y; s[2] += (double)v[r].z; s[3] += (double)v[r].w;
        }
    }
    float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < K && nrc > 0)
        c = make_float4((float)(s[0] / (double)nrc), (float)(s[1] / (double)nrc), (float)(s[2] / (double)nrc),
                        (float)(s[3] / (double)nrc));
    *reinterpret_cast<float4*>(center + p * Kp + k) = c;
}

cudaError_t launch_center(int P, const RowSrc& colsrc, int64_t nrc, int64_t K, int64_t Kp,
                          float* center, cudaStream_t st) {
    if (nrc > 16) return cudaErrorInvalidValue;
    dim3 grid((unsigned)((Kp / 4 + 255) / 256), (unsigned)P);
    ProfScope ps_(K_PACK, st);
    k_center<<<grid, 256, 0, st>>>(colsrc, nrc, K, Kp, center);
    note_launch();
    return cudaGetLastError();
}

// ----------------------------------------------------------------------- TC pack
// One CTA per panel row.  x~ = x - c (FP32), split:
//   split 1 (3xBF16): hi = bf16_rn(x~), lo = bf16_rn(x~ - hi)
//   split 2 (3xTF32): hi = x~ with the low 13 mantissa bits cleared, lo = x~ - hi (exact)
// nrm = sum x~^2 (FP64 accumulate -> FP32), q4 = (sum x~^4)^(1/4) (the error-bound scale
// of the split products, DESIGN.md §L2 engine).
template <int SPLIT>
__global__ void __launch_bounds__(256) k_pack_tc(RowSrc src, int64_t rows, int64_t K, int64_t Kp,
                                                 const float* __restrict__ center,
                                                 void* __restrict__ hi, void* __restrict__ lo,
                                                 float* __restrict__ nrm, float* __restrict__ q4,
                                                 int32_t* __restrict__ status) {
    const int64_t p = blockIdx.y;
    const int64_t r = blockIdx.x;
    const float* x = row_ptr(src, p, r);
    const float* c = center + p * Kp;
    const int64_t orow = p * rows + r;
    double s2 = 0.0, s4 = 0.0;
    bool nonfinite = false;
    for (int64_t k = (int64_t)threadIdx.x * 4; k < Kp; k += (int64_t)blockDim.x * 4) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < K) {
            float4 xv = __ldg(reinterpret_cast<const float4*>(x + k));
            float4 cv = *reinterpret_cast<const float4*>(c + k);
            nonfinite |= !(isfinite(xv.x) && isfinite(xv.y) && isfinite(xv.z) && isfinite(xv.w));
            v = make_float4(xv.x - cv.x, xv.y - cv.y, xv.z - cv.z, xv.w - cv.w);
        }
        const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const double d = (double)e[t];
            s2 += d * d;
            s4 += (d * d) * (d * d);
        }
        if (SPLIT == 1) {
            __nv_bfloat16 h[4], l[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                h[t] = __float2bfloat16_rn(e[t]);
                l[t] = __float2bfloat16_rn(e[t] - __bfloat162float(h[t]));
            }
            uint2 hv, lv;
            hv.x = (uint32_t)__bfloat16_as_ushort(h[0]) | ((uint32_t)__bfloat16_as_ushort(h[1]) << 16);
            hv.y = (uint32_t)__bfloat16_as_ushort(h[2]) | ((uint32_t)__bfloat16_as_ushort(h[3]) << 16);
            lv.x = (uint32_t)__bfloat16_as_ushort(l[0]) | ((uint32_t)__bfloat16_as_ushort(l[1]) << 16);
            lv.y = (uint32_t)__bfloat16_as_ushort(l[2]) | ((uint32_t)__bfloat16_as_ushort(l[3]) << 16);
            reinterpret_cast<uint2*>(hi)[(orow * Kp + k) / 4] = hv;
            reinterpret_cast<uint2*>(lo)[(orow * Kp + k) / 4] = lv;
        } else {
            float hh[4], ll[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                hh[t] = __uint_as_float(__float_as_uint(e[t]) & 0xFFFFE000u);
                ll[t] = e[t] - hh[t];
            }
            reinterpret_cast<float4*>(hi)[(orow * Kp + k) / 4] = make_float4(hh[0], hh[1], hh[2], hh[3]);
            reinterpret_cast<float4*>(lo)[(orow * Kp + k) / 4] = make_float4(ll[0], ll[1], ll[2], ll[3]);
        }
    }
    // block reduction of s2, s4
    __shared__ double red[2][32];
    __shared__ int nf;
    if (threadIdx.x == 0) nf = 0;
    for (int o = 16; o > 0; o >>= 1) {
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        s4 += __shfl_xor_sync(0xffffffffu, s4, o);
    }
    __syncthreads();
    if (nonfinite) atomicOr(&nf, 1);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { red[0][w] = s2; red[1][w] = s4; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a += red[0][i]; b += red[1][i]; }
        nrm[orow] = (float)a;
        q4[orow] = (float)sqrt(sqrt(b));
        if (nf) atomicOr(&status[p], CIL_ITEM_NONFINITE);
    }
}

cudaError_t launch_pack_tc(int P, const RowSrc& src, int64_t rows, int64_t K, int64_t Kp,
                           const float* center, int split, void* hi, void* lo, float* nrm, float* q4,
                           int32_t* status, cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    dim3 grid((unsigned)rows, (unsigned)P);
    ProfScope ps_(K_PACK, st);
    if (split == 2)
        k_pack_tc<2><<<grid, 256, 0, st>>>(src, rows, K, Kp, center, hi, lo, nrm, q4, status);
    else
        k_pack_tc<1><<<grid, 256, 0, st>>>(src, rows, K, Kp, center, hi, lo, nrm, q4, status);
    note_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------- min-max scaling
// Scaled-pattern mode: per pattern and species s,
//   y_s(x) = (s(x) - s_min) / (s_max - s_min)  over the species' H x W grid values,
// evaluated in FP64 and rounded to FP32; a constant species maps to 0 (reading R17).
// One CTA per pattern.
__global__ void __launch_bounds__(256) k_minmax(const float* __restrict__ X, int64_t ldx, float* __restrict__ Y,
                                                int64_t ldy, int S, int64_t HW) {
    const int64_t r = blockIdx.x;
    const float* x = X + r * ldx;
    float* y = Y + r * ldy;
    __shared__ float smin[8], smax[8];
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    for (int s = 0; s < S; ++s) {
        const float* xs = x + (int64_t)s * HW;
        float mn = INFINITY, mx = -INFINITY;
        for (int64_t e = threadIdx.x; e < HW; e += 256) {
            const float v = xs[e];
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
        for (int o = 16; o > 0; o >>= 1) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (ln == 0) { smin[w] = mn; smax[w] = mx; }
        __syncthreads();
        mn = smin[0];
        mx = smax[0];
        for (int i = 1; i < 8; ++i) { mn = fminf(mn, smin[i]); mx = fmaxf(mx, smax[i]); }
        __syncthreads();                                    // smin/smax reused by the next species
        const double lo = mn, span = (double)mx - (double)mn;
        float* ys = y + (int64_t)s * HW;
        for (int64_t e = threadIdx.x; e < HW; e += 256)
            ys[e] = span > 0.0 ? (float)(((double)xs[e] - lo) / span) : 0.f;
    }
}

cudaError_t launch_minmax(int64_t n, const float* X, int64_t ldx, float* Y, int64_t ldy, int S, int64_t HW,
                          cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    ProfScope ps_(K_PACK, st);
    k_minmax<<<(unsigned)n, 256, 0, st>>>(X, ldx, Y, ldy, S, HW);
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------------- aug pack
// One CTA per panel row: out = [x (K) | D_x x (S*H*(W-1)) | D_y x (S*(H-1)*W)], each
// region zero-padded to a multiple of kSimtBK, plain FP32 differences.  rowstat[row] = {max |D_x x|,
// max |D_y x|, |D_x x|, |D_y x|} of the stored FP32 differences (rounded up): the CUDA-core engine's
// error bound for the derivative terms needs them (the stored differences are rounded, so the
// engine's D(a) - D(b) is off the exact D(a - b) by <= 2^-24 (|D a| + |D b|) per element).
__global__ void __launch_bounds__(256) k_pack_aug(RowSrc src, int64_t rows, AugGeom g,
                                                  float* __restrict__ out, float* __restrict__ rowstat,
                                                  int32_t* __restrict__ status) {
    const int64_t p = blockIdx.y;
    const int64_t r = blockIdx.x;
    const float* x = row_ptr(src, p, r);
    float* o = out + (p * rows + r) * g.off[3];
    float nfa = 0.f;                               // NaN iff some value is not finite
    // value region: float4 copy (K % 4 == 0), zero padding
    for (int64_t k = (int64_t)threadIdx.x * 4; k < g.off[1]; k += 1024) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < g.K) v = __ldg(reinterpret_cast<const float4*>(x + k));
        nfa = fmaf(v.x, 0.f, fmaf(v.y, 0.f, fmaf(v.z, 0.f, fmaf(v.w, 0.f, nfa))));
        *reinterpret_cast<float4*>(o + k) = v;
    }
    // derivative regions: warp per grid row (s, r), lanes along the columns, no index division
    const int W = g.W, H = g.H, SH = g.S * g.H;
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
    float mxx = 0.f, myy = 0.f;
    double sxx = 0.0, syy = 0.0;
    if (g.nreg >= 2) {
        for (int sr = w; sr < SH; sr += 8) {
            const int64_t base = (int64_t)sr * W;
            const bool has_dy = g.nreg >= 3 && (sr % H) + 1 < H;
            const int s = sr / H;
            const bool grad = g.gs == 0 || ((g.gs >> s) & 1u);     // species mask (R18): else 0
            for (int c = ln; c < W; c += 32) {
                const float xe = __ldg(x + base + c);
                if (c + 1 < W) {
                    const float dx = grad ? __ldg(x + base + c + 1) - xe : 0.f;
                    o[g.off[1] + (int64_t)sr * (W - 1) + c] = dx;
                    mxx = fmaxf(mxx, fabsf(dx));
                    sxx += (double)dx * (double)dx;
                }
                if (has_dy) {
                    const float dy = grad ? __ldg(x + base + W + c) - xe : 0.f;
                    o[g.off[2] + base - (int64_t)s * W + c] = dy;
                    myy = fmaxf(myy, fabsf(dy));
                    syy += (double)dy * (double)dy;
                }
            }
        }
        for (int64_t t = g.Kx + threadIdx.x; t < g.off[2] - g.off[1]; t += 256) o[g.off[1] + t] = 0.f;
        if (g.nreg >= 3)
            for (int64_t t = g.Ky + threadIdx.x; t < g.off[3] - g.off[2]; t += 256) o[g.off[2] + t] = 0.f;
    }
    if (rowstat != nullptr) {
        __shared__ float smx[2][8];
        __shared__ double ssx[2][8];
        for (int off = 16; off > 0; off >>= 1) {
            mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, off));
            myy = fmaxf(myy, __shfl_xor_sync(0xffffffffu, myy, off));
            sxx += __shfl_xor_sync(0xffffffffu, sxx, off);
            syy += __shfl_xor_sync(0xffffffffu, syy, off);
        }
        if (ln == 0) { smx[0][w] = mxx; smx[1][w] = myy; ssx[0][w] = sxx; ssx[1][w] = syy; }
        __syncthreads();
        if (threadIdx.x == 0) {
            float a = 0.f, b = 0.f;
            double c = 0.0, d = 0.0;
            for (int i = 0; i < 8; ++i) { a = fmaxf(a, smx[0][i]); b = fmaxf(b, smx[1][i]); c += ssx[0][i]; d += ssx[1][i]; }
            float4 v = make_float4(a, b, __double2float_ru(sqrt(c) * (1.0 + 1e-12)), __double2float_ru(sqrt(d) * (1.0 + 1e-12)));
            *reinterpret_cast<float4*>(rowstat + (p * rows + r) * 4) = v;
        }
    }
    if (__syncthreads_or(nfa != nfa) && threadIdx.x == 0) atomicOr(&status[p], CIL_ITEM_NONFINITE);
}

cudaError_t launch_pack_aug(int P, const RowSrc& src, int64_t rows, const AugGeom& g, float* out, float* rowstat,
                            int32_t* status, cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    dim3 grid((unsigned)rows, (unsigned)P);
    ProfScope ps_(K_PACK, st);
    k_pack_aug<<<grid, 256, 0, st>>>(src, rows, g, out, rowstat, status);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cil
