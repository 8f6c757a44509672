// gram_tc.cu — step a2 of the hot path: L2 distances (Eq. (5)) of all
// pairs through the Gram identity d^2 = |a~|^2 + |b~|^2 - 2 a~.b~ on the 5th-generation
// tensor cores, fused with the radius binning of Eq. (1): the
// N x Nt distance matrix never leaves the SM.
//
// Split precision: a~ = hi + lo (3xBF16: bf16 pair; 3xTF32: tf32 pair) and
//   g = hi_a.hi_b + hi_a.lo_b + lo_a.hi_b        (3 tcgen05.mma per k-step, one FP32 TMEM accumulator)
// Error control: every pair with |d^2 - T_m| <= E(i,j) for some threshold T_m = R_m^2/w,
//   E = k1 * q_a * q_b + rel * (n_a + n_b),   q = (sum x~^4)^(1/4),
// is NOT binned here; it is appended to a re-check list and binned exactly (FP64) by
// recheck.cu.  All other pairs are classified correctly whenever the Gram error is
// below E (DESIGN.md §"L2 engine" derives k1, rel and tests their margin).
//
// Kernel anatomy (persistent, one CTA per SM, 192 threads):
//   warp 0      TMA producer: A_hi, A_lo (128 x 128 B) and B_hi, B_lo (BN x 128 B) per stage,
//               SWIZZLE_128B, mbarrier complete_tx
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, cta_group::1),
//               tcgen05.commit -> smem-slot release and accumulator-ready barriers
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> d^2 -> per-thread cumulative counters,
//               ambiguous pairs -> re-check list; double-buffered TMEM accumulator so the
//               epilogue of tile t overlaps the MMAs of tile t+1.
#include <cuda.h>
#include <stdio.h>

#include "cil_internal.cuh"
#include "tc_common.cuh"

namespace cil {

namespace tc {
// Tile geometry.  CG = CTAs per MMA (cta_group): the cluster tile is (128*CG) x 256;
// every CTA holds 128 A-rows and 256/CG B-rows of each operand stage, and its TMEM holds
// the FP32 accumulator of its own 128 rows x all 256 columns (double-buffered).

struct TcParams {
    int64_t rowsA, rowsB;     // rows per item of the A / B panel
    int P;                    // items in the stacked operand arrays
    int p0, np;               // this launch covers items [p0, p0 + np)
    int n_kb;                 // k-blocks of 128 bytes
    int tiles_m, tiles_n;     // per item (cluster tiles)
    int split;                // 1 = bf16, 2 = tf32
    const float* nrm;         // stacked [P*rowsA + P*rowsB]
    const float* q4;
    const float* thr2;        // [P][M]
    int64_t thr_stride;
    int M, nq, q_l2;
    SegParams sp;
    unsigned long long* hist;
    uint4* list; uint32_t* ctr; uint32_t cap;
    float k1, rel;
    float* diag;              // diagnostics: [rowsA][rowsB][2] = (d2, E) of item 0, no binning
    int chunk_kb;             // k-blocks accumulated per TMEM partial before the FP32 drain
};


template <int MAXM, int CG>
// 10 warps -> up to 3 per SM sub-partition (16K registers each): <= 168 registers/thread
__global__ void __maxnreg__(168)
k_gram_tc(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
          const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo, TcParams prm) {
    using G = Geo<CG>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    unsigned char* stages = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::STAGES * G::STAGE_BYTES);
    uint64_t* empty = full + G::STAGES;
    uint64_t* tfull = empty + G::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* s_nb = reinterpret_cast<float*>(smem + G::STAGES * G::STAGE_BYTES + 1024);
    float* s_qb = s_nb + TILE_N;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    const int cluster_id = blockIdx.x / CG, n_clusters = gridDim.x / CG;
    const int tiles_per_item = prm.tiles_m * prm.tiles_n;
    const int total_tiles = prm.np * tiles_per_item;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < G::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8 * CG); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mAhi) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mAlo) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mBhi) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mBlo) : "memory");
    }
    if (warp == 1) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    fence_before();
    if (CG == 2) cluster_sync(); else __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int kind_tf32 = prm.split == 2;
    const int bkE = kind_tf32 ? 32 : 64;    // elements per 128-byte row

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cluster_id; t < total_tiles; t += n_clusters) {
                const int p = prm.p0 + t / tiles_per_item, r = t % tiles_per_item;
                const int mt = r / prm.tiles_n, nt = r % prm.tiles_n;
                const int ya = (int)(p * prm.rowsA + (int64_t)mt * G::TILE_M + rank * A_ROWS);
                const int yb = (int)((int64_t)prm.P * prm.rowsA + p * prm.rowsB + (int64_t)nt * TILE_N + rank * G::B_ROWS);
                for (int kb = 0; kb < prm.n_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    unsigned char* st = stages + stage * G::STAGE_BYTES;
                    if (rank == 0) mbar_expect_tx(&full[stage], CG * G::STAGE_BYTES);
                    const int x = kb * bkE;
                    tma_load_2d<CG>(st, &mAhi, &full[stage], x, ya);
                    tma_load_2d<CG>(st + G::A_BYTES, &mAlo, &full[stage], x, ya);
                    tma_load_2d<CG>(st + 2 * G::A_BYTES, &mBhi, &full[stage], x, yb);
                    tma_load_2d<CG>(st + 2 * G::A_BYTES + G::B_BYTES, &mBlo, &full[stage], x, yb);
                    if (++stage == G::STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // K is accumulated in chunks of chunk_kb k-blocks into one of two TMEM partial
            // buffers (columns [0,256) and [256,512)); the epilogue drains each chunk into FP32
            // running sums in registers (round-to-nearest adds) while the tensor cores fill the
            // other buffer.  Long in-place tensor-core accumulation loses low bits
            // systematically (measured ~4e-5 relative d^2 at K = 8192); short
            // chunks bound that loss.
            const uint32_t id = idesc(kind_tf32 ? 2 : 1, G::TILE_M, TILE_N);
            int stage = 0;
            uint32_t phase = 0;
            int buf = 0;
            uint32_t bph = 0u;          // bit b = phase parity of partial buffer b
            for (int t = cluster_id; t < total_tiles; t += n_clusters) {
                for (int kb0 = 0; kb0 < prm.n_kb; kb0 += prm.chunk_kb) {
                    const int kb1 = min(kb0 + prm.chunk_kb, prm.n_kb);
                    if (CG == 2) mbar_wait_cluster(&tempty[buf], ((bph >> buf) & 1u) ^ 1u);
                    else mbar_wait(&tempty[buf], ((bph >> buf) & 1u) ^ 1u);
                    fence_after();
                    const uint32_t d = tmem_base + (uint32_t)(buf * TILE_N);
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        fence_after();
                        const uint32_t s0 = smem_u32(stages + stage * G::STAGE_BYTES);
                        const uint64_t ahi = sdesc(s0), alo = sdesc(s0 + G::A_BYTES);
                        const uint64_t bhi = sdesc(s0 + 2 * G::A_BYTES), blo = sdesc(s0 + 2 * G::A_BYTES + G::B_BYTES);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {           // 4 x 32 bytes of K per 128-byte row
                            const uint64_t adv = (uint64_t)(k * 2);  // +32 B in the start-address field (>>4)
                            mma<CG>(d, ahi + adv, bhi + adv, id, (kb != kb0 || k != 0) ? 1u : 0u, kind_tf32);
                            mma<CG>(d, ahi + adv, blo + adv, id, 1u, kind_tf32);
                            mma<CG>(d, alo + adv, bhi + adv, id, 1u, kind_tf32);
                        }
                        mma_commit<CG>(&empty[stage]);
                        if (++stage == G::STAGES) { stage = 0; phase ^= 1; }
                    }
                    mma_commit<CG>(&tfull[buf]);
                    bph ^= 1u << buf;
                    buf ^= 1;
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        // 8 warps: warp w owns TMEM lanes 32*(w&3).. (its 32 rows) and the column half
        // (w-2)>>2 of the 256-column tile; running sums of its 128 pairs live in registers.
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        const int et = threadIdx.x - 64;              // 0..255
        const int M = prm.M;
        int buf = 0;
        uint32_t bph = 0u;          // bit b = phase parity of partial buffer b
        for (int t = cluster_id; t < total_tiles; t += n_clusters) {
            const int p = prm.p0 + t / tiles_per_item, r = t % tiles_per_item;
            const int mt = r / prm.tiles_n, nt = r % prm.tiles_n;
            const int64_t col0 = (int64_t)nt * TILE_N;
            const int64_t browbase = (int64_t)prm.P * prm.rowsA + (int64_t)p * prm.rowsB;
            named_bar(1, 256);
            {
                const int64_t c = col0 + et;
                const bool ok = c < prm.rowsB;
                s_nb[et] = ok ? prm.nrm[browbase + c] : 0.f;
                s_qb[et] = ok ? prm.q4[browbase + c] : 0.f;
            }
            named_bar(1, 256);

            // ---- drain the K-chunks into registers
            float acc[128];
#pragma unroll
            for (int j = 0; j < 128; ++j) acc[j] = 0.f;
            const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
            for (int kb0 = 0; kb0 < prm.n_kb; kb0 += prm.chunk_kb) {
                mbar_wait(&tfull[buf], (bph >> buf) & 1u);
                fence_after();
                const uint32_t tp = tmem_base + lane_off + (uint32_t)(buf * TILE_N + half * 128);
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {
                    uint32_t v[16];
                    tmem_ld16(tp + ch * 16, v);
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) acc[ch * 16 + jj] += __uint_as_float(v[jj]);
                }
                if (kb0 + prm.chunk_kb < prm.n_kb) {      // release the buffer; keep the last one
                    fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (CG == 2) mbar_arrive_remote(&tempty[buf], 0);
                        else mbar_arrive(&tempty[buf]);
                    }
                    bph ^= 1u << buf;
                    buf ^= 1;
                }
            }
            // ---- park the final sums in the (still owned) last buffer, bin from there
            const uint32_t tp = tmem_base + lane_off + (uint32_t)(buf * TILE_N + half * 128);
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[32];
#pragma unroll
                for (int jj = 0; jj < 32; ++jj) v[jj] = __float_as_uint(acc[ch * 32 + jj]);
                tmem_st32(tp + ch * 32, v);
            }
            tmem_wait_st();

            float T[MAXM];
#pragma unroll
            for (int m = 0; m < MAXM; ++m) T[m] = (m < M) ? __ldg(&prm.thr2[(int64_t)p * prm.thr_stride + m]) : -INFINITY;
            const int64_t row = (int64_t)mt * G::TILE_M + rank * A_ROWS + quarter * 32 + lane;
            const bool row_ok = row < prm.rowsA;
            const int64_t arow = (int64_t)p * prm.rowsA + (row_ok ? row : 0);
            const float na = row_ok ? __ldg(&prm.nrm[arow]) : 0.f;
            const float k1qa = row_ok ? prm.k1 * __ldg(&prm.q4[arow]) : 0.f;
            const int64_t rs = row_ok ? row / prm.sp.row_seg : 0;
            uint32_t cnt[MAXM];
#pragma unroll
            for (int m = 0; m < MAXM; ++m) cnt[m] = 0;

            auto flush = [&](int64_t cs) {
                // all lanes share cs; rows of one warp may span two row segments
                const int64_t rs0 = __shfl_sync(0xffffffffu, rs, 0);
                const bool uniform = __all_sync(0xffffffffu, rs == rs0 || !row_ok);
                if (uniform) {
                    uint32_t prev = 0;
#pragma unroll
                    for (int m = MAXM - 1; m >= 0; --m) {
                        if (m >= M) continue;
                        const uint32_t tot = __reduce_add_sync(0xffffffffu, cnt[m]);
                        if (lane == 0 && tot != prev)
                            atomicAdd(&prm.hist[hist_index(prm.sp, prm.nq, M, p, rs0, cs, prm.q_l2, m + 1)],
                                      (unsigned long long)(tot - prev));
                        prev = tot;
                        cnt[m] = 0;
                    }
                } else {
                    uint32_t prev = 0;
#pragma unroll
                    for (int m = MAXM - 1; m >= 0; --m) {
                        if (m >= M) continue;
                        if (row_ok && cnt[m] != prev)
                            atomicAdd(&prm.hist[hist_index(prm.sp, prm.nq, M, p, rs, cs, prm.q_l2, m + 1)],
                                      (unsigned long long)(cnt[m] - prev));
                        prev = cnt[m];
                        cnt[m] = 0;
                    }
                }
            };

            const int64_t hcol0 = col0 + half * 128;
            int64_t cur_cs = hcol0 / prm.sp.col_seg;
#pragma unroll 1
            for (int ch = 0; ch < 4; ++ch) {
                uint32_t v[32];
                tmem_ld32(tp + ch * 32, v);
                if (hcol0 + ch * 32 >= prm.rowsB) break;   // warp-uniform
#pragma unroll 4
                for (int jj = 0; jj < 32; ++jj) {
                    const int j = half * 128 + ch * 32 + jj;
                    const int64_t c = col0 + j;
                    if (c >= prm.rowsB) break;             // warp-uniform
                    const int64_t cs = c / prm.sp.col_seg;
                    if (cs != cur_cs) { flush(cur_cs); cur_cs = cs; }
                    if (!row_ok) continue;
                    const float g = __uint_as_float(v[jj]);
                    const float nb = s_nb[j];
                    const float sab = na + nb;
                    const float d2 = fmaf(-2.f, g, sab);
                    const float E = fmaf(k1qa, s_qb[j], prm.rel * sab);
                    if (prm.diag) {
                        if (p == 0) {
                            prm.diag[(row * prm.rowsB + c) * 2] = d2;
                            prm.diag[(row * prm.rowsB + c) * 2 + 1] = E;
                        }
                        continue;
                    }
                    const float hi = d2 + E, lo = d2 - E;
                    uint32_t blo = 0;
#pragma unroll
                    for (int m = 0; m < MAXM; ++m) {
                        const uint32_t c1 = hi < T[m] ? 1u : 0u;
                        cnt[m] += c1;
                        blo += c1;
                    }
                    // ambiguous iff the next threshold below the certain prefix is within reach
                    float Tn = -INFINITY;
#pragma unroll
                    for (int m = 0; m < MAXM; ++m) Tn = (m == (int)blo) ? T[m] : Tn;
                    if (lo < Tn) {
                        const uint32_t idx = atomicAdd(prm.ctr, 1u);
                        if (idx < prm.cap) prm.list[idx] = make_uint4((uint32_t)p, (uint32_t)row, (uint32_t)c, blo);
                    }
                }
            }
            // release the last buffer of this tile
            fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CG == 2) mbar_arrive_remote(&tempty[buf], 0);
                else mbar_arrive(&tempty[buf]);
            }
            bph ^= 1u << buf;
            buf ^= 1;
            flush(cur_cs);
        }
    }
    __syncthreads();
    if (CG == 2) cluster_sync();
    if (warp == 1) {
        fence_after();
        if (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}
}  // namespace tc

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    }
    return fn;
}

bool gram_tc_supported() { return true; }

static bool make_map(CUtensorMap* m, const void* base, int split, int64_t rows, int64_t Kp, int box_rows) {
    PFN_encodeTiled enc = get_encode();
    if (!enc) return false;
    const size_t esz = split == 2 ? 4 : 2;
    cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(Kp * esz)};
    cuuint32_t box[2] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, split == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                     const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int MAXM, int CG>
static cudaError_t launch_t(const tc::TcParams& prm, const CUtensorMap* maps, int nsm, cudaStream_t st) {
    using G = tc::Geo<CG>;
    static SmemAttrOnce attr;
    if (cudaError_t e = attr.ensure(tc::k_gram_tc<MAXM, CG>, G::SMEM_BYTES); e != cudaSuccess) return e;
    const int64_t tiles = (int64_t)prm.np * prm.tiles_m * prm.tiles_n;
    const int clusters = (int)(tiles < nsm / CG ? tiles : nsm / CG);   // nsm = SM budget of this launch
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(clusters * CG));
    cfg.blockDim = dim3(tc::NTHREADS);
    cfg.dynamicSmemBytes = G::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope ps_(K_GRAM_TC, st);
    cudaError_t e = cudaLaunchKernelEx(&cfg, tc::k_gram_tc<MAXM, CG>, maps[0], maps[1], maps[2], maps[3], prm);
    note_launch();
    if (e != cudaSuccess) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, tc::k_gram_tc<MAXM, CG>);
        fprintf(stderr, "[libcil] k_gram_tc launch failed (%s): regs=%d maxThreads=%d local=%zu smem_dyn=%d\n",
                cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock, fa.localSizeBytes, G::SMEM_BYTES);
        return e;
    }
    return cudaGetLastError();
}

template <int CG>
static cudaError_t launch_cg(const TcArgs& a, cudaStream_t st) {
    using G = tc::Geo<CG>;
    const int64_t rows = (int64_t)a.P * (a.rowsA + a.rowsB);
    if (rows >= (1ll << 31)) return cudaErrorInvalidValue;
    const size_t esz = a.split == 2 ? 4 : 2;
    const char* hi = static_cast<const char*>(a.hi);
    const char* lo = static_cast<const char*>(a.lo);
    CUtensorMap maps[4];
    if (!make_map(&maps[0], hi, a.split, rows, a.Kp, tc::A_ROWS) ||
        !make_map(&maps[1], lo, a.split, rows, a.Kp, tc::A_ROWS) ||
        !make_map(&maps[2], hi, a.split, rows, a.Kp, G::B_ROWS) ||
        !make_map(&maps[3], lo, a.split, rows, a.Kp, G::B_ROWS))
        return cudaErrorInvalidValue;
    tc::TcParams prm{};
    prm.rowsA = a.rowsA; prm.rowsB = a.rowsB; prm.P = a.P;
    prm.n_kb = (int)((a.Kp * (int64_t)esz) / tc::ROW_BYTES);
    prm.tiles_m = (int)((a.rowsA + G::TILE_M - 1) / G::TILE_M);
    prm.tiles_n = (int)((a.rowsB + tc::TILE_N - 1) / tc::TILE_N);
    prm.split = a.split;
    prm.nrm = a.nrm; prm.q4 = a.q4;
    prm.thr2 = a.thr2; prm.thr_stride = a.thr_stride;
    prm.M = a.M; prm.nq = a.nq; prm.q_l2 = a.q_l2;
    prm.sp = a.sp;
    prm.hist = reinterpret_cast<unsigned long long*>(a.hist);
    prm.list = a.recheck; prm.ctr = a.recheck_ctr; prm.cap = a.recheck_cap;
    prm.k1 = a.guard_k1; prm.rel = a.guard_rel;
    prm.diag = a.diag;
    prm.chunk_kb = a.chunk_kb > 0 ? a.chunk_kb : 4;
    prm.p0 = a.p0;
    prm.np = a.np > 0 ? a.np : a.P - a.p0;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (a.sm_budget > 0 && a.sm_budget < nsm) nsm = a.sm_budget;
    if (a.M <= 16) return launch_t<16, CG>(prm, maps, nsm, st);
    if (a.M <= 32) return launch_t<32, CG>(prm, maps, nsm, st);
    return launch_t<64, CG>(prm, maps, nsm, st);
}

cudaError_t launch_gram_tc(const TcArgs& a, cudaStream_t st) {
    if (a.rowsA == 0 || a.rowsB == 0) return cudaSuccess;
    // CTA pairs (cta_group::2, 256 x 256 tiles) unless explicitly forced to single-CTA tiles
    if (a.cta_group == 1) return launch_cg<1>(a, st);
    return launch_cg<2>(a, st);
}

}  // namespace cil
