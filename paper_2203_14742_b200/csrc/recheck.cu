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
// Row-bucketed pass (lists of >= sort_min entries, 8192 unless a diagnostic changes it; VERDICT r1
// "restructure k_recheck around row reuse"): the list is counting-sorted by (p, i) (k_rk_count,
// k_rk_scan, k_rk_scatter) and walked entry-parallel, so the CTAs working at one time share a few A
// rows (one HBM read each, L2 hits for the rest) while the partners stream, and every pair is
// evaluated once for all its listed measures.  Pairs listed only for the max family (Eqs. (6),
// (9), (10)) are first evaluated in FP32 with a rigorous bound (fl is monotone: the FP32 max of
// |fl(a - b)| is within 2^-24 of the exact max, the differences of the derivative regions within
// 2^-24 (2 m_0 + |D|) + ...); only a pair whose FP32 interval still contains a radius goes on to the
// FP64 evaluation.
//
// List overflow: the engines stop appending at the list capacity and the counter keeps counting.
// Then k_fb_clear zeroes the histograms and k_recheck evaluates EVERY pair of every item exactly
// (the slow path; counts stay exact, CIL_ITEM_OVERFLOW records that it ran).
#include <cub/block/block_scan.cuh>

#include "cil_internal.cuh"
#include "tc_common.cuh"


namespace cil {

namespace {
// ---- the pair sweeps' operand ring: chunks of RCH elements of x and y streamed into shared memory
// by one thread with cp.async.bulk (TMA, 1-D) and an mbarrier per stage, RST stages in flight, so a
// CTA keeps 3 x 2 x 8 KB of its pair's rows in flight while it computes, 4 CTAs per SM (2 CTAs with
// 3 x 2 x 16 KB: slower; profiles/r02_recheck.txt)
#ifndef CIL_RK_EXP
#define CIL_RK_EXP 0     // experiment builds: 1 neighbour sweep for L-inf-only pairs too; 2 two stages;
#endif                   // 3 twice the CTAs; 4 chunks of 1024
constexpr uint32_t RCH = CIL_RK_EXP == 4 ? 1024 : 2048;
constexpr uint32_t RHALO = 256;      // each chunk also brings the next grid row (W <= RHALO): every x / y
                                     // neighbour of the chunk is in shared memory, the sweeps are branch-free
constexpr uint32_t RSTR = RCH + RHALO;
constexpr int RST = CIL_RK_EXP == 2 ? 2 : 3;
constexpr size_t kRingBytes = sizeof(float) * 2 * RSTR * RST;
struct Ring {
    float* buf;        // [RST][2][RSTR] (x chunk + halo, y chunk + halo)
    uint64_t* bar;     // [RST]
    uint32_t g;        // chunks streamed so far by this CTA (stage = g % RST, parity = (g / RST) & 1)
};
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     tc::smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
                 : "memory");
}
// chunk [e0, e0 + len) plus the halo [e0 + len, e0 + len + min(halo, K - e0 - len))
__device__ __forceinline__ void ring_issue(Ring& r, uint32_t gi, const float* x, const float* y, uint32_t e0,
                                           uint32_t len, uint32_t K, uint32_t halo) {
    const int st = (int)(gi % RST);
    float* dx = r.buf + (size_t)st * 2 * RSTR;
    const uint32_t n = len + min(halo, K - e0 - len);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the stage's generic reads are done
    tc::mbar_expect_tx(&r.bar[st], 8u * n);
    bulk_g2s(dx, x + e0, 4u * n, &r.bar[st]);
    bulk_g2s(dx + RSTR, y + e0, 4u * n, &r.bar[st]);
}
// Streams the K elements of x and y (16-B aligned, K % 4 == 0) through the ring, each chunk with a
// halo of `halo` (<= RHALO, % 4 == 0) further elements; all threads call f(base, sx, sy, len) once per
// chunk (elements [base, base + len), sx / sy valid up to base + len + halo where the pattern has them;
// reads up to RSTR stay inside the stage).
template <class F>
__device__ void ring_stream(Ring& r, const float* x, const float* y, uint32_t K, uint32_t halo, F f) {
    const uint32_t nch = (K + RCH - 1) / RCH, g0 = r.g;
    if (threadIdx.x == 0)
        for (uint32_t c = 0; c < nch && c < (uint32_t)RST; ++c)
            ring_issue(r, g0 + c, x, y, c * RCH, min(RCH, K - c * RCH), K, halo);
    for (uint32_t c = 0; c < nch; ++c) {
        const uint32_t gi = g0 + c, st = gi % RST;
        tc::mbar_wait(&r.bar[st], (gi / RST) & 1u);
        const float* sx = r.buf + (size_t)st * 2 * RSTR;
        f(c * RCH, sx, sx + RSTR, min(RCH, K - c * RCH));
        __syncthreads();                                   // every thread is done with the stage
        if (threadIdx.x == 0 && c + RST < nch)
            ring_issue(r, gi + RST, x, y, (c + RST) * RCH, min(RCH, K - (c + RST) * RCH), K, halo);
    }
    r.g = g0 + nch;
}

// The six FP64 sub-norms of u = x - y over one pattern, one CTA of 256 threads.
// full = false: only s0 (a flat K-long loop with 4 float4 pairs in flight per thread); full with
// W % 4 == 0 and the operand ring: a flat float4 sweep over the ring's chunks of x and y (the x / y
// neighbours from there); otherwise a warp per grid row.
__device__ void exact_subnorms(const float* x, const float* y, const RecheckArgs& a, bool full, double out[6],
                               double (*red)[8], Ring* ring = nullptr) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (full && ring != nullptr && (a.W & 3) == 0 && (uint32_t)a.W <= RHALO && a.K < (1ll << 31)) {
        const uint32_t W = (uint32_t)a.W, H = (uint32_t)a.H;
        const FastDiv fw(W), fh(H);
        ring_stream(*ring, x, y, (uint32_t)a.K, W, [&](uint32_t base, const float* sx, const float* sy, uint32_t len) {
#pragma unroll
            for (int t = 0; t < (int)(RCH / 1024); ++t) {
                const uint32_t l = t * 1024 + threadIdx.x * 4, e = base + l;
                if (l >= len) continue;
                const float4 xa = *reinterpret_cast<const float4*>(sx + l), yb = *reinterpret_cast<const float4*>(sy + l);
                const double u0 = (double)xa.x - (double)yb.x, u1 = (double)xa.y - (double)yb.y;
                const double u2 = (double)xa.z - (double)yb.z, u3 = (double)xa.w - (double)yb.w;
                v[0] += u0 * u0 + u1 * u1 + u2 * u2 + u3 * u3;
                v[3] = fmax(v[3], fmax(fmax(fabs(u0), fabs(u1)), fmax(fabs(u2), fabs(u3))));
                uint32_t c, hr;
                const uint32_t sr = fw.div(e, c), sp = fh.div(sr, hr);
                const bool g = a.gs == 0 || ((a.gs >> sp) & 1u);
                // neighbours from the stage (chunk + halo); masked where the pattern has none
                const double d0 = u1 - u0, d1 = u2 - u1, d2 = u3 - u2;
                const double d3 = c + 4 < W ? ((double)sx[l + 4] - (double)sy[l + 4]) - u3 : 0.0;
                const float4 xd = *reinterpret_cast<const float4*>(sx + l + W);
                const float4 yd = *reinterpret_cast<const float4*>(sy + l + W);
                const bool gy = g && hr + 1 < H;
                const double e0 = gy ? ((double)xd.x - (double)yd.x) - u0 : 0.0;
                const double e1 = gy ? ((double)xd.y - (double)yd.y) - u1 : 0.0;
                const double e2 = gy ? ((double)xd.z - (double)yd.z) - u2 : 0.0;
                const double e3 = gy ? ((double)xd.w - (double)yd.w) - u3 : 0.0;
                if (g) {
                    v[1] += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
                    v[4] = fmax(v[4], fmax(fmax(fabs(d0), fabs(d1)), fmax(fabs(d2), fabs(d3))));
                }
                v[2] += e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3;
                v[5] = fmax(v[5], fmax(fmax(fabs(e0), fabs(e1)), fmax(fabs(e2), fabs(e3))));
            }
        });
    } else if (!full) {
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

// The max sub-norms m0, m_x, m_y of u = x - y in FP32 (raw differences, no 1/h), one CTA of 256
// threads; |result - exact| <= 2^-24 m0, 3 2^-24 (m0 + m_x), 3 2^-24 (m0 + m_y).  W % 4 == 0 (and
// the operand ring): a flat float4 sweep over the ring's chunks; else a warp per grid row.
__device__ __forceinline__ float amax4(float m, float a, float b, float c, float d) {
    return fmaxf(fmaxf(m, fmaxf(fabsf(a), fabsf(b))), fmaxf(fabsf(c), fabsf(d)));
}
// GRAD = false (every listed measure of the pair is L-inf): the value block only, m_x = m_y = 0.
template <bool GRAD>
__device__ void max_subnorms32(const float* x, const float* y, const RecheckArgs& a, float out[3], float (*red)[8],
                               Ring* ring) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float v[3] = {0.f, 0.f, 0.f};
    const int W = a.W, H = a.H;
    if ((W & 3) == 0 && W <= (int)RHALO && ring != nullptr) {
        const uint32_t Wu = (uint32_t)W, Hu = (uint32_t)H;
        const FastDiv fw(Wu), fh(Hu);
        ring_stream(*ring, x, y, (uint32_t)a.K, Wu, [&](uint32_t base, const float* sx, const float* sy, uint32_t len) {
#pragma unroll
            for (int t = 0; t < (int)(RCH / 1024); ++t) {
                const uint32_t l = t * 1024 + threadIdx.x * 4, e = base + l;
                if (l >= len) continue;
                const float4 xa = *reinterpret_cast<const float4*>(sx + l), yb = *reinterpret_cast<const float4*>(sy + l);
                const float4 u = make_float4(xa.x - yb.x, xa.y - yb.y, xa.z - yb.z, xa.w - yb.w);
                v[0] = amax4(v[0], u.x, u.y, u.z, u.w);
                if (!GRAD) continue;
                uint32_t c, hr;
                const uint32_t sr = fw.div(e, c), sp = fh.div(sr, hr);
                const bool g = a.gs == 0 || ((a.gs >> sp) & 1u);
                // neighbours from the stage (chunk + halo); masked where the pattern has none
                const float nx = (sx[l + 4] - sy[l + 4]) - u.w;
                const float4 xd = *reinterpret_cast<const float4*>(sx + l + Wu);
                const float4 yd = *reinterpret_cast<const float4*>(sy + l + Wu);
                float dxm = fmaxf(fabsf(u.y - u.x), fmaxf(fabsf(u.z - u.y), fabsf(u.w - u.z)));
                dxm = c + 4 < Wu ? fmaxf(dxm, fabsf(nx)) : dxm;
                const float dym = amax4(0.f, (xd.x - yd.x) - u.x, (xd.y - yd.y) - u.y, (xd.z - yd.z) - u.z,
                                        (xd.w - yd.w) - u.w);
                v[1] = g ? fmaxf(v[1], dxm) : v[1];
                v[2] = (g && hr + 1 < Hu) ? fmaxf(v[2], dym) : v[2];
            }
        });
    } else {
        const int SH = a.S * a.H;
        for (int sr = w; sr < SH; sr += 8) {
            const bool grad = GRAD && (a.gs == 0 || ((a.gs >> (sr / H)) & 1u));
            const bool has_dy = grad && (sr % H) + 1 < H;
            const float* xr = x + (int64_t)sr * W;
            const float* yr = y + (int64_t)sr * W;
            for (int c = lane; c < W; c += 32) {
                const float u = __ldg(xr + c) - __ldg(yr + c);
                v[0] = fmaxf(v[0], fabsf(u));
                if (grad && c + 1 < W) v[1] = fmaxf(v[1], fabsf((__ldg(xr + c + 1) - __ldg(yr + c + 1)) - u));
                if (has_dy) v[2] = fmaxf(v[2], fabsf((__ldg(xr + W + c) - __ldg(yr + W + c)) - u));
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        for (int o = 16; o > 0; o >>= 1) v[i] = fmaxf(v[i], __shfl_xor_sync(0xffffffffu, v[i], o));
        if (lane == 0) red[i][w] = v[i];
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int i = 0; i < 3; ++i) {
            float m = 0.f;
            for (int t = 0; t < 8; ++t) m = fmaxf(m, red[i][t]);
            out[i] = m;
        }
    __syncthreads();
}

// FP32 interval of a max-family measure (kind 1, 4, 5) from max_subnorms32
__device__ void measure32(int k, const float m[3], double h, double* d, double* E) {
    const double U = 5.9604644775390625e-08;
    const double m0 = m[0], mx = (double)m[1] / h, my = (double)m[2] / h;
    const double e0 = 2.0 * U * m0, ex = 3.0 * U * ((double)m[0] + m[1]) / h, ey = 3.0 * U * ((double)m[0] + m[2]) / h;
    if (k == 1) { *d = m0; *E = e0; }
    else if (k == 4) { *d = fmax(m0, fmax(mx, my)); *E = fmax(e0, fmax(ex, ey)); }
    else { *d = m0 + mx + my; *E = e0 + ex + ey; }
    *E += 1e-14 * *d;
}

// Move pair (i, j) of measure `kind` from its provisional bin b_lo to its exact bin b (or write b).
__device__ void settle_bin(const RecheckArgs& a, int64_t p, int64_t i, int64_t j, int kind, int b_lo, int b,
                           bool add_only) {
    const int q = a.qslot[kind];
    CIL_CHECK(kind >= 0 && kind < 6 && q >= 0 && q < a.nq && p < a.P && i < a.rowsA && j < a.rowsB);
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

__device__ void settle(const RecheckArgs& a, int64_t p, int64_t i, int64_t j, int kind, int b_lo, double d,
                       bool add_only) {
    const double* R = a.thr + p * a.thr_stride + (int64_t)a.qslot[kind] * a.M;
    int b = 0;
    while (b < a.M && d < R[b]) ++b;
    settle_bin(a, p, i, j, kind, b_lo, b, add_only);
}

// #{m : v < R_m} of slot `kind` of item p, counted by the whole CTA (R is decreasing; M <= 64)
__device__ __forceinline__ int bin_of(const RecheckArgs& a, int64_t p, int kind, double v) {
    const double* R = a.thr + p * a.thr_stride + (int64_t)a.qslot[kind] * a.M;
    return __syncthreads_count((int)threadIdx.x < a.M && v < R[threadIdx.x]);
}
}  // namespace

// ---- counting sort of the list by (p, i): counts, exclusive scan (one CTA), scatter.  After the
// scatter rk[row] is the END of the row's range (= start of row + 1).
__global__ void k_rk_count(RecheckArgs a) {
    const uint32_t c = *a.ctr;
    if (c > a.cap || c < a.sort_min) return;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < c; e += gridDim.x * blockDim.x) {
        const uint4 ent = a.list[e];
        CIL_CHECK(ent.x < (uint32_t)a.P && ent.y < (uint64_t)a.rowsA);
        atomicAdd(&a.rk[(int64_t)ent.x * a.rowsA + ent.y], 1u);
    }
}

__global__ void __launch_bounds__(1024) k_rk_scan(RecheckArgs a, int64_t n) {
    const uint32_t c = *a.ctr;
    if (c > a.cap || c < a.sort_min) return;
    using BlockScan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename BlockScan::TempStorage tmp;
    uint32_t carry = 0;
    for (int64_t base = 0; base < n; base += 4096) {
        uint32_t v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int64_t idx = base + threadIdx.x * 4 + t;
            v[t] = idx < n ? a.rk[idx] : 0u;
        }
        uint32_t agg;
        BlockScan(tmp).ExclusiveSum(v, v, agg);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int64_t idx = base + threadIdx.x * 4 + t;
            if (idx < n) a.rk[idx] = v[t] + carry;
        }
        carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) a.rk[n] = carry;
}

__global__ void k_rk_scatter(RecheckArgs a) {
    const uint32_t c = *a.ctr;
    if (c > a.cap || c < a.sort_min) return;
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < c; e += gridDim.x * blockDim.x) {
        const uint4 ent = a.list[e];
        const uint32_t pos = atomicAdd(&a.rk[(int64_t)ent.x * a.rowsA + ent.y], 1u);
        CIL_CHECK(pos < c);
        a.rk_list[pos] = ent;
    }
}

// Overflow: zero the histograms (the exact pass below re-counts every pair).
__global__ void k_fb_clear(RecheckArgs a, int64_t hist_elems) {
    if (*a.ctr <= a.cap || a.binout) return;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < hist_elems; e += (int64_t)gridDim.x * blockDim.x)
        a.hist[e] = 0ull;
}

__global__ void __launch_bounds__(256, 4) k_recheck(RecheckArgs a) {
    const uint32_t c = *a.ctr;
    const bool overflow = c > a.cap;
    __shared__ double red[6][8];
    __shared__ double sub[6];
    extern __shared__ __align__(16) float ring_buf[];     // kRingBytes (the sweeps' operand ring)
    __shared__ __align__(8) uint64_t ring_bar[RST];
    if (threadIdx.x == 0) {
        for (int i = 0; i < RST; ++i) tc::mbar_init(&ring_bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    Ring ring{ring_buf, ring_bar, 0u};
    Ring* rp = a.K < (1ll << 31) ? &ring : nullptr;
    if (overflow) {
        if (blockIdx.x == 0 && threadIdx.x == 0)
            for (int p = 0; p < a.P; ++p) atomicOr(&a.status[p], CIL_ITEM_OVERFLOW);
        // exact pass over every pair (mirrored layouts: i <= j, written in both orders)
        const int64_t per = a.rowsA * a.rowsB;
        for (int64_t e = blockIdx.x; e < (int64_t)a.P * per; e += gridDim.x) {
            const int64_t p = e / per, i = (e % per) / a.rowsB, j = e % a.rowsB;
            if (a.mirror && j < i) continue;
            if (a.status[p] & CIL_ITEM_BADRADII) continue;
            exact_subnorms(row_ptr(a.asrc, p, i), row_ptr(a.bsrc, p, j), a, a.kinds & ~1u, sub, red, rp);
            if (threadIdx.x == 0)
                for (int k = 0; k < 6; ++k)
                    if ((a.kinds >> k) & 1u) settle(a, p, i, j, k, 0, measure(k, sub, a.w, a.h), true);
            __syncthreads();
        }
        return;
    }
    if (c < a.sort_min) {
        for (uint32_t e = blockIdx.x; e < c; e += gridDim.x) {
            const uint4 ent = a.list[e];
            const int64_t p = ent.x, i = ent.y, j = ent.z;
            const int b_lo = (int)(ent.w & 255u);
            const int kind = (int)((ent.w >> 8) & 255u);
            exact_subnorms(row_ptr(a.asrc, p, i), row_ptr(a.bsrc, p, j), a, kind != 0, sub, red, rp);
            if (threadIdx.x == 0) settle(a, p, i, j, kind, b_lo, measure(kind, sub, a.w, a.h), false);
            __syncthreads();
        }
        return;
    }
    // row-bucketed pass: the CTAs walk the SORTED list entry-parallel (consecutive entries share
    // their A row, so concurrent CTAs read it together: one HBM read, L2 hits for the rest); the
    // first entry of a pair (i, j) in its row bucket owns the pair and settles all its measures
    // (bins counted by the whole CTA over the radii, no serial loops over global memory)
    constexpr uint32_t kBucketScan = 1024;               // buckets up to this size pair their entries
    __shared__ uint32_t s_n, s_w[8];
    __shared__ double s_d[8], s_E[8];
    __shared__ float red32[3][8];
    __shared__ float m32[3];
    for (uint32_t e = blockIdx.x; e < c; e += gridDim.x) {
        const uint4 ent = a.rk_list[e];
        const int64_t p = ent.x, i = ent.y, j = ent.z;
        const int64_t row = p * a.rowsA + i;
        const uint32_t beg = row ? a.rk[row - 1] : 0u, end = a.rk[row];
        if (threadIdx.x == 0) s_n = 0u;
        __syncthreads();
        bool dup = false;
        if (end - beg <= kBucketScan) {
            for (uint32_t u = beg + threadIdx.x; u < end; u += blockDim.x) {
                const uint4 o = a.rk_list[u];
                if (o.z != ent.z) continue;
                if (u < e) dup = true;
                else {
                    const uint32_t k = atomicAdd(&s_n, 1u);
                    if (k < 8) s_w[k] = o.w;
                }
            }
        } else if (threadIdx.x == 0) {                       // a huge bucket: no pairing (each entry
            s_n = 1u;                                        // settles itself; bounded work, not
            s_w[0] = ent.w;                                  // quadratic in the bucket size)
        }
        if (__syncthreads_or(dup)) continue;
        const int n = (int)min(s_n, 8u);                  // a pair is listed at most once per measure
        uint32_t kmask = 0u;
        for (int k = 0; k < n; ++k) kmask |= 1u << ((s_w[k] >> 8) & 255u);
        const float* xa = row_ptr(a.asrc, p, i);
        const float* yb = row_ptr(a.bsrc, p, j);
        bool exact = true;
        if (!(kmask & 0x0Du)) {                              // max family only: FP32 interval first
            if ((kmask & ~0x2u) || CIL_RK_EXP == 1) max_subnorms32<true>(xa, yb, a, m32, red32, rp);
            else max_subnorms32<false>(xa, yb, a, m32, red32, rp);        // L-inf only: no neighbours
            if ((int)threadIdx.x < n) measure32((int)((s_w[threadIdx.x] >> 8) & 255u), m32, a.h, &s_d[threadIdx.x], &s_E[threadIdx.x]);
            __syncthreads();
            exact = false;
            for (int k = 0; k < n; ++k) {
                const int kind = (int)((s_w[k] >> 8) & 255u);
                const int bh = bin_of(a, p, kind, s_d[k] + s_E[k]), bl = bin_of(a, p, kind, s_d[k] - s_E[k]);
                if (bh == bl) {
                    if (threadIdx.x == 0) settle_bin(a, p, i, j, kind, (int)(s_w[k] & 255u), bh, false);
                    if (threadIdx.x == 0) s_w[k] |= 0x80000000u;      // settled
                } else {
                    exact = true;
                }
            }
            __syncthreads();
        }
        if (!exact) continue;
        exact_subnorms(xa, yb, a, (kmask & ~1u) != 0u, sub, red, rp);
        if ((int)threadIdx.x < n) s_d[threadIdx.x] = measure((int)((s_w[threadIdx.x] >> 8) & 255u), sub, a.w, a.h);
        __syncthreads();
        for (int k = 0; k < n; ++k) {
            if (s_w[k] & 0x80000000u) continue;
            const int kind = (int)((s_w[k] >> 8) & 255u);
            const int b = bin_of(a, p, kind, s_d[k]);
            if (threadIdx.x == 0) settle_bin(a, p, i, j, kind, (int)(s_w[k] & 255u), b, false);
        }
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
    const int64_t nrows = (int64_t)a.P * a.rowsA;
    if (cudaError_t e = cudaMemsetAsync(a.rk, 0, sizeof(uint32_t) * (size_t)(nrows + 1), st); e != cudaSuccess) return e;
    k_rk_count<<<nsm * 2, 256, 0, st>>>(a);
    k_rk_scan<<<1, 1024, 0, st>>>(a, nrows);
    k_rk_scatter<<<nsm * 2, 256, 0, st>>>(a);
    static SmemAttrOnce attr;
    if (cudaError_t e = attr.ensure(k_recheck, (int)kRingBytes); e != cudaSuccess) return e;
    k_recheck<<<nsm * (CIL_RK_EXP == 3 ? 16 : 8), 256, kRingBytes, st>>>(a);
    note_launch(4);
    return cudaGetLastError();
}

CIL_OOB_READER(oob_recheck)

}  // namespace cil
