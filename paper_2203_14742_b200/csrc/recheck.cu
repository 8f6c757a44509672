// recheck.cu — exact FP64 re-evaluation of the (pair, measure) cases an engine could not classify
// with certainty: the engine's rigorous interval of the distance contained a radius (gram3.cu,
// simt_tile.cu, gram_tc.cu).  Per listed pair, from the caller's original FP32 patterns:
//   s0 = sum u^2, s_x = sum (D_x u)^2, s_y = sum (D_y u)^2, m0 = max|u|, m_x = max|D_x u|, m_y = max|D_y u|
// with u = (double)a - (double)b and raw forward differences inside each species (last node
// omitted, reading R3; species mask gs, R18), then the measure of the entry's kind (Eqs. (5)-(10),
// PAPER.md:181-190; w = h^dim, R1) and its bin b = #{m : d < R_m} (Eq. (1), strict <).
// The pair is moved from the provisional bin the engine counted it in to b (hist[b_lo] -= 1,
// hist[b] += 1) or, in bin-matrix mode, b is written to the pair's entry (both orders when mirrored).
//
// List overflow: the engines stop appending at the list capacity and the counter keeps counting.
// Then k_fb_clear zeroes the histograms and k_recheck evaluates EVERY pair of every item exactly
// (the slow path; counts stay exact, CIL_ITEM_OVERFLOW records that it ran).
#include "cil_internal.cuh"

namespace cil {

namespace {
// The six FP64 sub-norms of u = x - y over one pattern, one CTA of 256 threads (warp per grid row).
// full = false: only s0 (a flat K-long loop with 4 float4 pairs in flight per thread).
__device__ void exact_subnorms(const float* x, const float* y, const RecheckArgs& a, bool full, double out[6],
                               double (*red)[8]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (!full) {
        int64_t k = (int64_t)threadIdx.x * 4;
        for (; k + 3 * 1024 < a.K; k += 4 * 1024) {
            float4 u[4], z[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                u[t] = __ldg(reinterpret_cast<const float4*>(x + k + t * 1024));
                z[t] = __ldg(reinterpret_cast<const float4*>(y + k + t * 1024));
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const double d0 = (double)u[t].x - (double)z[t].x, d1 = (double)u[t].y - (double)z[t].y;
                const double d2 = (double)u[t].z - (double)z[t].z, d3 = (double)u[t].w - (double)z[t].w;
                v[0] = fma(d0, d0, v[0]); v[0] = fma(d1, d1, v[0]); v[0] = fma(d2, d2, v[0]); v[0] = fma(d3, d3, v[0]);
            }
        }
        for (; k < a.K; k += 1024) {
            const float4 u = __ldg(reinterpret_cast<const float4*>(x + k));
            const float4 z = __ldg(reinterpret_cast<const float4*>(y + k));
            const double d0 = (double)u.x - (double)z.x, d1 = (double)u.y - (double)z.y;
            const double d2 = (double)u.z - (double)z.z, d3 = (double)u.w - (double)z.w;
            v[0] = fma(d0, d0, v[0]); v[0] = fma(d1, d1, v[0]); v[0] = fma(d2, d2, v[0]); v[0] = fma(d3, d3, v[0]);
        }
    } else {
        const int W = a.W, H = a.H, SH = a.S * a.H;
        for (int sr = w; sr < SH; sr += 8) {
            const bool grad = a.gs == 0 || ((a.gs >> (sr / H)) & 1u);
            const bool has_dy = grad && (sr % H) + 1 < H;
            const float* xr = x + (int64_t)sr * W;
            const float* yr = y + (int64_t)sr * W;
            for (int c = lane; c < W; c += 32) {
                const double u = (double)__ldg(xr + c) - (double)__ldg(yr + c);
                v[0] += u * u;
                v[3] = fmax(v[3], fabs(u));
                if (grad && c + 1 < W) {
                    const double dx = ((double)__ldg(xr + c + 1) - (double)__ldg(yr + c + 1)) - u;
                    v[1] += dx * dx;
                    v[4] = fmax(v[4], fabs(dx));
                }
                if (has_dy) {
                    const double dy = ((double)__ldg(xr + W + c) - (double)__ldg(yr + W + c)) - u;
                    v[2] += dy * dy;
                    v[5] = fmax(v[5], fabs(dy));
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        for (int o = 16; o > 0; o >>= 1) {
            const double t = __shfl_xor_sync(0xffffffffu, v[i], o);
            v[i] = i < 3 ? v[i] + t : fmax(v[i], t);
        }
        if (lane == 0) red[i][w] = v[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < 6; ++i) {
            double s = 0.0;
            for (int t = 0; t < 8; ++t) s = i < 3 ? s + red[i][t] : fmax(s, red[i][t]);
            out[i] = s;
        }
    }
    __syncthreads();
}

// The measure of kind k (measure id, bit order) from the sub-norms (raw differences: 1/h applied here)
__device__ double measure(int k, const double sub[6], double w, double h) {
    const double a0 = sqrt(w * sub[0]), ax = sqrt(w * sub[1] / (h * h)), ay = sqrt(w * sub[2] / (h * h));
    const double m0 = sub[3], mx = sub[4] / h, my = sub[5] / h;
    switch (k) {
        case 0: return a0;                                   // Eq. (5)
        case 1: return m0;                                   // Eq. (6)
        case 2: return a0 + ax + ay;                         // Eq. (7)
        case 3: return sqrt(a0 * a0 + ax * ax + ay * ay);    // Eq. (8)
        case 4: return fmax(m0, fmax(mx, my));               // Eq. (9)
        default: return m0 + mx + my;                        // Eq. (10)
    }
}

__device__ void settle(const RecheckArgs& a, int64_t p, int64_t i, int64_t j, int kind, int b_lo, double d,
                       bool add_only) {
    const int q = a.qslot[kind];
    CIL_CHECK(kind >= 0 && kind < 6 && q >= 0 && q < a.nq && p < a.P && i < a.rowsA && j < a.rowsB);
    const double* R = a.thr + p * a.thr_stride + (int64_t)q * a.M;
    int b = 0;
    while (b < a.M && d < R[b]) ++b;
    if (a.binout && a.transpose) {                       // [p][q][j][i] (the engine's transposed output)
        a.binout[(((int64_t)p * a.nq + q) * a.rowsB + j) * a.rowsA + i] = (uint8_t)b;
    } else if (a.binout) {
        a.binout[(((int64_t)p * a.nq + q) * a.rowsA + i) * a.rowsB + j] = (uint8_t)b;
        if (a.mirror) a.binout[(((int64_t)p * a.nq + q) * a.rowsA + j) * a.rowsB + i] = (uint8_t)b;
    } else {
        const int64_t rs = i / a.sp.row_seg, cs = j / a.sp.col_seg;
        unsigned long long* H = (unsigned long long*)a.hist;
        CIL_CHECK(hist_index(a.sp, a.nq, a.M, p, rs, cs, q, a.M) < a.hist_elems);
        if (add_only) {
            if (b > 0) atomicAdd(&H[hist_index(a.sp, a.nq, a.M, p, rs, cs, q, b)], 1ull);
        } else if (b != b_lo) {
            if (b_lo > 0) atomicAdd(&H[hist_index(a.sp, a.nq, a.M, p, rs, cs, q, b_lo)], ~0ull);
            if (b > 0) atomicAdd(&H[hist_index(a.sp, a.nq, a.M, p, rs, cs, q, b)], 1ull);
        }
    }
}
}  // namespace

// Overflow: zero the histograms (the exact pass below re-counts every pair).
__global__ void k_fb_clear(RecheckArgs a, int64_t hist_elems) {
    if (*a.ctr <= a.cap || a.binout) return;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < hist_elems; e += (int64_t)gridDim.x * blockDim.x)
        a.hist[e] = 0ull;
}

__global__ void __launch_bounds__(256) k_recheck(RecheckArgs a) {
    const uint32_t c = *a.ctr;
    const bool overflow = c > a.cap;
    __shared__ double red[6][8];
    __shared__ double sub[6];
    if (overflow) {
        if (blockIdx.x == 0 && threadIdx.x == 0)
            for (int p = 0; p < a.P; ++p) atomicOr(&a.status[p], CIL_ITEM_OVERFLOW);
        // exact pass over every pair (mirrored layouts: i <= j, written in both orders)
        const int64_t per = a.rowsA * a.rowsB;
        for (int64_t e = blockIdx.x; e < (int64_t)a.P * per; e += gridDim.x) {
            const int64_t p = e / per, i = (e % per) / a.rowsB, j = e % a.rowsB;
            if (a.mirror && j < i) continue;
            if (a.status[p] & CIL_ITEM_BADRADII) continue;
            exact_subnorms(row_ptr(a.asrc, p, i), row_ptr(a.bsrc, p, j), a, a.kinds & ~1u, sub, red);
            if (threadIdx.x == 0)
                for (int k = 0; k < 6; ++k)
                    if ((a.kinds >> k) & 1u) settle(a, p, i, j, k, 0, measure(k, sub, a.w, a.h), true);
            __syncthreads();
        }
        return;
    }
    for (uint32_t e = blockIdx.x; e < c; e += gridDim.x) {
        const uint4 ent = a.list[e];
        const int64_t p = ent.x, i = ent.y, j = ent.z;
        const int b_lo = (int)(ent.w & 255u);
        const int kind = (int)((ent.w >> 8) & 255u);
        exact_subnorms(row_ptr(a.asrc, p, i), row_ptr(a.bsrc, p, j), a, kind != 0, sub, red);
        if (threadIdx.x == 0) settle(a, p, i, j, kind, b_lo, measure(kind, sub, a.w, a.h), false);
        __syncthreads();
    }
}

cudaError_t launch_recheck(const RecheckArgs& a, int64_t hist_elems, cudaStream_t st) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    ProfScope ps_(K_RECHECK, st);
    if (!a.binout && hist_elems > 0) {
        k_fb_clear<<<nsm, 256, 0, st>>>(a, hist_elems);
        note_launch();
    }
    k_recheck<<<nsm * 8, 256, 0, st>>>(a);
    note_launch();
    return cudaGetLastError();
}

CIL_OOB_READER(oob_recheck)

}  // namespace cil
