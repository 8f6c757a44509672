// recheck.cu — exact re-evaluation of the L2 pairs the tensor-core epilogue could not
// classify with certainty (|d^2_approx - R_m^2/w| within the engine's error bound E).
// One CTA per listed pair (256 threads, grid-stride over the list): s0 = sum_e ((double)a_e -
// (double)b_e)^2 in FP64 from the caller's original FP32 patterns, bin b = #{m : s0 < R_m^2/w}
// (Eq. (1), strict <; L2 = sqrt(w s0), Eq. (5)); the pair is then moved from the
// provisional bin b_lo the epilogue gave it to b:  hist[b_lo] -= 1, hist[b] += 1 — or, in
// bin-matrix mode, b is written to the pair's entry.
#include "cil_internal.cuh"

namespace cil {

__global__ void __launch_bounds__(256) k_recheck(RecheckArgs a) {
    const uint32_t n = min(*a.ctr, a.cap);
    if (blockIdx.x == 0 && threadIdx.x == 0 && *a.ctr > a.cap) {
        // overflow: flag every item (we do not know which pairs were dropped)
        for (int p = 0; p < a.P; ++p) atomicOr(&a.status[p], CIL_ITEM_OVERFLOW);
    }
    __shared__ double red[8];
    __shared__ double red3[3][8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint32_t e = blockIdx.x; e < n; e += gridDim.x) {
        const uint4 ent = a.list[e];
        const int64_t p = ent.x, i = ent.y, j = ent.z;
        const int b_lo = (int)(ent.w & 255u);
        const int kind = (int)((ent.w >> 8) & 255u);
        const float* x = row_ptr(a.asrc, p, i);
        const float* y = row_ptr(a.bsrc, p, j);
        if (kind != 0) {
            // W12 (kind 1) / W12SUM (kind 2): the FP64 sub-norms of u = a - b exactly as the plain
            // definition (forward differences inside each species, last node omitted, R3)
            const int W = a.W, H = a.H, SH = a.S * a.H;
            const double h = a.h;
            double s0 = 0.0, sx = 0.0, sy = 0.0;
            // warp per grid row (s, r), lanes along the columns: coalesced, no index division
            for (int sr = w; sr < SH; sr += 8) {
                const bool grad = a.gs == 0 || ((a.gs >> (sr / H)) & 1u);   // species mask (R18)
                const bool has_dy = grad && (sr % H) + 1 < H;
                const float* xr = x + (int64_t)sr * W;
                const float* yr = y + (int64_t)sr * W;
                for (int c = lane; c < W; c += 32) {
                    const double u = (double)__ldg(xr + c) - (double)__ldg(yr + c);
                    s0 += u * u;
                    if (grad && c + 1 < W) {               // raw differences; the 1/h^2 is applied once
                        const double dx = ((double)__ldg(xr + c + 1) - (double)__ldg(yr + c + 1)) - u;
                        sx += dx * dx;
                    }
                    if (has_dy) {
                        const double dy = ((double)__ldg(xr + W + c) - (double)__ldg(yr + W + c)) - u;
                        sy += dy * dy;
                    }
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                s0 += __shfl_xor_sync(0xffffffffu, s0, o);
                sx += __shfl_xor_sync(0xffffffffu, sx, o);
                sy += __shfl_xor_sync(0xffffffffu, sy, o);
            }
            if (lane == 0) { red3[0][w] = s0; red3[1][w] = sx; red3[2][w] = sy; }
            __syncthreads();
            if (threadIdx.x == 0) {
                s0 = sx = sy = 0.0;
                for (int t = 0; t < 8; ++t) { s0 += red3[0][t]; sx += red3[1][t]; sy += red3[2][t]; }
                sx /= h * h;
                sy /= h * h;
                const double a0 = sqrt(a.w * s0), ax = sqrt(a.w * sx), ay = sqrt(a.w * sy);
                const double d = kind == 1 ? sqrt(a0 * a0 + ax * ax + ay * ay) : a0 + ax + ay;   // Eqs. (8), (7)
                const int q = a.q_tc[kind];
                const double* R = a.thr + p * a.thr_stride + (int64_t)q * a.M;
                int b = 0;
                while (b < a.M && d < R[b]) ++b;
                if (a.binout) {                          // bin-matrix mode: the exact bin, both orders
                    a.binout[(((int64_t)p * a.nq + q) * a.rowsA + i) * a.rowsB + j] = (uint8_t)b;
                    if (a.mirror) a.binout[(((int64_t)p * a.nq + q) * a.rowsA + j) * a.rowsB + i] = (uint8_t)b;
                } else if (b != b_lo) {
                    const int64_t rs = i / a.sp.row_seg, cs = j / a.sp.col_seg;
                    unsigned long long* Hh = (unsigned long long*)a.hist;
                    if (b_lo > 0) atomicAdd(&Hh[hist_index(a.sp, a.nq, a.M, p, rs, cs, q, b_lo)], ~0ull);
                    if (b > 0) atomicAdd(&Hh[hist_index(a.sp, a.nq, a.M, p, rs, cs, q, b)], 1ull);
                }
            }
            __syncthreads();
            continue;
        }
        double s = 0.0;
        // 4 independent float4 pairs in flight per thread (memory-level parallelism)
        int64_t k = (int64_t)threadIdx.x * 4;
        for (; k + 3 * 1024 < a.K; k += 4 * 1024) {
            float4 u[4], v[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                u[t] = __ldg(reinterpret_cast<const float4*>(x + k + t * 1024));
                v[t] = __ldg(reinterpret_cast<const float4*>(y + k + t * 1024));
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const double d0 = (double)u[t].x - (double)v[t].x, d1 = (double)u[t].y - (double)v[t].y;
                const double d2 = (double)u[t].z - (double)v[t].z, d3 = (double)u[t].w - (double)v[t].w;
                s = fma(d0, d0, s); s = fma(d1, d1, s); s = fma(d2, d2, s); s = fma(d3, d3, s);
            }
        }
        for (; k < a.K; k += 1024) {
            const float4 u = __ldg(reinterpret_cast<const float4*>(x + k));
            const float4 v = __ldg(reinterpret_cast<const float4*>(y + k));
            const double d0 = (double)u.x - (double)v.x, d1 = (double)u.y - (double)v.y;
            const double d2 = (double)u.z - (double)v.z, d3 = (double)u.w - (double)v.w;
            s = fma(d0, d0, s); s = fma(d1, d1, s); s = fma(d2, d2, s); s = fma(d3, d3, s);
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[w] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            s = 0.0;
            for (int t = 0; t < 8; ++t) s += red[t];
            const int ql = a.q_tc[0] >= 0 ? a.q_tc[0] : a.q_l2;
            const double* R = a.thr + p * a.thr_stride + (int64_t)ql * a.M;
            int b = 0;
            while (b < a.M && s < R[b] * R[b] / a.w) ++b;
            if (a.binout && a.transpose) {              // [p][q][j][i] (the engine's transposed output)
                a.binout[(((int64_t)p * a.nq + ql) * a.rowsB + j) * a.rowsA + i] = (uint8_t)b;
            } else if (a.binout) {
                a.binout[(((int64_t)p * a.nq + ql) * a.rowsA + i) * a.rowsB + j] = (uint8_t)b;
                if (a.mirror) a.binout[(((int64_t)p * a.nq + ql) * a.rowsA + j) * a.rowsB + i] = (uint8_t)b;
            } else if (b != b_lo) {
                const int64_t rs = i / a.sp.row_seg, cs = j / a.sp.col_seg;
                unsigned long long* H = (unsigned long long*)a.hist;
                if (b_lo > 0) atomicAdd(&H[hist_index(a.sp, a.nq, a.M, p, rs, cs, a.q_l2, b_lo)], ~0ull);
                if (b > 0) atomicAdd(&H[hist_index(a.sp, a.nq, a.M, p, rs, cs, a.q_l2, b)], 1ull);
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_recheck(const RecheckArgs& a, cudaStream_t st) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    ProfScope ps_(K_RECHECK, st);
    k_recheck<<<nsm * 8, 256, 0, st>>>(a);
    note_launch();
    return cudaGetLastError();
}

}  // namespace cil
