// rowdot.cu — the bootstrap's replicate counts (Alg. A1 step 2 / Alg. A2 steps 2.1-2.4,
// PAPER.md:648-723) as one integer GEMM per measure on tcgen05 kind::i8.
//
// A resampled set pair only contains patterns of the fixed sets, so (regrouping the (i, j) sum of
// Eq. (1); repeated draws count once per draw)
//   counts[k][v] = #{(i, j) : bins(I1[k][i], I2[k][j]) > v} = sum_b m2[k][b] sum_a m1[k][a] [bins(a, b) > v]
// with m1 / m2 the row / column draw multiplicities of replicate k.  The inner sum is the GEMM
//   C[k][(v, b)] = sum_a M1[k][a] E[(v, b)][a],   M1 int8 (multiplicities <= 127), E 0/1 bytes
// (resample.cu builds both), accumulated exactly in int32 TMEM; the epilogue forms
// sum_b C[k][(v, b)] m2[k][b] (u32, exact: <= n1 n2 < 2^32, host-checked) and adds it atomically.
//
// Kernel anatomy (persistent CTA pairs, cta_group::2, 256 x 256 tiles, one operand plane):
//   warp 0      TMA producer: with the A row block resident (all k-blocks of 256 replicates kept in
//               shared memory while B streams through a ring of up to 16 slots), else a streaming ring
//   warp 1      TMEM allocator + single-thread MMA issuer; the accumulator is double-buffered (tile
//               i + 1 accumulates while the epilogue drains tile i)
//   warps 2-15  epilogue: tcgen05.ld -> weighted sums with the m2 weights held in registers across the
//               M tiles of a b-block (E rows are b-major: row = (b / 256, v, b mod 256))
#include <cuda.h>
#include <stdio.h>

#include "cil_internal.cuh"
#include "tc_common.cuh"

namespace cil {
namespace rd {
using namespace tc;

constexpr int TN = 256;
constexpr int BROWS = TN / 2;                       // B rows per CTA
constexpr int A_BYTES = A_ROWS * ROW_BYTES;         // 16 KB (128 rows x 128 K-bytes)
constexpr int B_BYTES = BROWS * ROW_BYTES;          // 16 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int STAGES = 3;
constexpr int NEPI = 14;
constexpr int NET = 32 * NEPI;
constexpr int NTHR = 64 + NET;
constexpr int SCRATCH = 33600;                      // extra B ring slots after the barrier block
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 1024 /*barriers*/ + SCRATCH;
constexpr int kSlots = 16;                          // resident-A mode: B ring slots
constexpr int kBars = 2 + 2 * kSlots;

struct Params {
    int64_t rowsA, rowsB, b_off;
    int P, p0, np, n_kb, tiles_m, tiles_n;
    const uint16_t* m2;        // [P][rowsA][rd_nt] column-draw multiplicities
    int64_t rd_nt;             // columns per threshold block (B row = v * rd_nt + b)
    int rd_m;                  // thresholds
    unsigned long long* out;   // [P][rowsA][rd_m] counts (atomic sums)
};

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
                 "l"(a), "l"(b), "r"(id), "r"(acc));
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Tile sequence of one cluster (the same for producer, MMA and epilogue).  Resident A: clusters form
// groups of tiles_m; cluster (g, mt) keeps tile row mt and walks the group's contiguous range of
// (item, nt) columns, so the tiles_m clusters of a group read each B tile at about the same time (one
// HBM read of B, A loaded once per item).  Streaming: the plain persistent stride.
struct Seq {
    bool resA;
    int n, mt, c0, tiles_n, stride, first;
    __device__ __forceinline__ void init(const Params& prm, bool resA_, int cluster_id, int n_clusters, int total) {
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
            n = cluster_id < total ? (total - 1 - cluster_id) / n_clusters + 1 : 0;
        }
    }
    __device__ __forceinline__ void get(const Params& prm, int i, int& p, int& mt_, int& nt) const {
        if (resA) {
            const int c = c0 + i;
            p = prm.p0 + c / tiles_n;
            nt = c % tiles_n;
            mt_ = mt;
        } else {
            const int t = first + i * stride;
            const int per = prm.tiles_m * prm.tiles_n;
            p = prm.p0 + t / per;
            mt_ = (t % per) / prm.tiles_n;
            nt = (t % per) % prm.tiles_n;
        }
    }
};
__device__ __forceinline__ bool resident_a(const Params& prm, int n_clusters) {
    return prm.tiles_m <= n_clusters && prm.n_kb * A_BYTES + 2 * B_BYTES <= STAGES * STAGE_BYTES;
}

// Epilogue: counts[k][v] = sum_b C[k][(v, b)] m2[k][b] for the tile's 256 columns (one v, 256 b)
__device__ __forceinline__ void epilogue(const Params& prm, uint32_t tmem_base, uint64_t* tfull, uint64_t* tempty,
                                         int cluster_id, int n_clusters, int total, uint32_t rank, int warp,
                                         int lane) {
    const int quarter = warp & 3;
    const int ew = warp - 2;
    const int e0 = (quarter + 2) & 3;
    const int nwq = (NEPI - e0 + 3) / 4;
    const int kq = ew >> 2;
    const int g0 = kq * (TN / 16) / nwq, g1 = (kq + 1) * (TN / 16) / nwq;
    // B rows are b-major: row (bt, v, i) = bt M TN + v TN + i holds column b = bt TN + i of threshold
    // v, so tile nt is (bt, v) = (nt / M, nt % M), all its columns share v, and the multiplicities of a
    // thread stay in registers across the M tiles of one b-block
    const int Nt = (int)prm.rd_nt;
    const int Mv = prm.rd_m;
    constexpr int MAXG = (TN / 16 + 2) / 3;
    uint4 w[MAXG][2];
    int64_t wkey = -1;                                      // (item, row, bt) of the cached weights
    uint32_t tphb = 0;
    int ab = 0;
    Seq seq;
    seq.init(prm, resident_a(prm, n_clusters), cluster_id, n_clusters, total);
    for (int i = 0; i < seq.n; ++i, ab ^= 1) {
        int p, mt, nt;
        seq.get(prm, i, p, mt, nt);
        const int64_t row = (int64_t)mt * (2 * A_ROWS) + rank * A_ROWS + quarter * 32 + lane;
        const bool row_ok = row < prm.rowsA;
        const int bt = nt / Mv, v = nt - bt * Mv;
        const int ng = g1 - g0;
        const uint32_t tl = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(ab * TN + g0 * 16);
        const int64_t key = ((int64_t)p * prm.tiles_m + mt) * (prm.tiles_n / Mv) + bt;
        if (key != wkey) {                                  // new b-block: load this thread's weights
            wkey = key;
            const uint16_t* m2row = prm.m2 + ((int64_t)p * prm.rowsA + (row_ok ? row : 0)) * Nt + bt * TN + g0 * 16;
#pragma unroll
            for (int g = 0; g < MAXG; ++g) {
                w[g][0] = w[g][1] = make_uint4(0u, 0u, 0u, 0u);
                if (row_ok && g < ng) {
                    const uint4* mp = reinterpret_cast<const uint4*>(m2row + g * 16);
                    w[g][0] = __ldg(mp); w[g][1] = __ldg(mp + 1);
                }
            }
        }
        uint64_t* tf = ab ? tfull + 4 : tfull;
        uint64_t* te = ab ? tfull + 5 : tempty;
        mbar_wait(tf, (tphb >> ab) & 1u);
        fence_after();
        uint32_t acc = 0u;                                  // <= n1 n2 < 2^32 (host-checked)
        // two groups per TMEM load (one wait::ld per 32 columns)
#pragma unroll
        for (int g2 = 0; g2 < MAXG; g2 += 2) {
            if (g2 < ng) {
                uint32_t hv[32];
                if (g2 + 1 < ng) {
                    tmem_ld32(tl + g2 * 16, hv);
                } else {                                    // odd tail: never read past the warp's range
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
        if (row_ok && acc) atomicAdd(prm.out + ((int64_t)p * prm.rowsA + row) * Mv + v, (unsigned long long)acc);
        tphb ^= 1u << ab;
    }
}

__global__ void __launch_bounds__(NTHR, 1)
k_rowdot(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, Params prm) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* stages = smem;
    uint64_t* tfull = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 6 + kBars);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int cluster_id = blockIdx.x / 2, n_clusters = gridDim.x / 2;
    const int total = prm.np * prm.tiles_m * prm.tiles_n;

    if (warp == 0 && lane == 0) {
        mbar_init(&tfull[0], 1);
        mbar_init(&tempty[0], 2 * NEPI);                    // epilogue warps x 2 CTAs
        mbar_init(tfull + 4, 1);                            // second accumulator
        mbar_init(tfull + 5, 2 * NEPI);
        for (int s = 6; s < 6 + kBars; ++s) mbar_init(tfull + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mB) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const bool resA = resident_a(prm, n_clusters);
    // B slots (resident A): the stage memory after the A block, then the scratch after the barriers
    const int nsb0 = (STAGES * STAGE_BYTES - prm.n_kb * A_BYTES) / B_BYTES;
    const int nsb = min(kSlots, nsb0 + SCRATCH / B_BYTES);
    unsigned char* bring = stages + prm.n_kb * A_BYTES;
    unsigned char* bextra = stages + STAGES * STAGE_BYTES + 1024 - nsb0 * B_BYTES;

    if (warp == 0) {
        if (lane == 0) {
            int key_prev = -1, sb = 0;
            uint32_t aph = 0, bph = 0;
            Seq seq;
            seq.init(prm, resA, cluster_id, n_clusters, total);
            for (int i = 0; i < seq.n; ++i) {
                int p, mt, nt;
                seq.get(prm, i, p, mt, nt);
                const int ya = (int)(p * prm.rowsA + (int64_t)mt * (2 * A_ROWS) + rank * A_ROWS);
                const int yb = (int)(prm.b_off + p * prm.rowsB + (int64_t)nt * TN + rank * BROWS);
                if (resA) {
                    const int key = p * prm.tiles_m + mt;
                    if (key != key_prev) {
                        mbar_wait(tfull + 7, aph ^ 1);
                        if (rank == 0) mbar_expect_tx(tfull + 6, 2 * prm.n_kb * A_BYTES);
                        for (int kb = 0; kb < prm.n_kb; ++kb)
                            tma_load_2d<2>(stages + kb * A_BYTES, &mA, tfull + 6, kb * 128, ya);
                        aph ^= 1;
                        key_prev = key;
                    }
                    for (int kb = 0; kb < prm.n_kb; ++kb) {
                        mbar_wait(tfull + 8 + kSlots + sb, bph ^ 1);
                        if (rank == 0) mbar_expect_tx(tfull + 8 + sb, 2 * B_BYTES);
                        tma_load_2d<2>((sb < nsb0 ? bring : bextra) + sb * B_BYTES, &mB, tfull + 8 + sb, kb * 128, yb);
                        if (++sb == nsb) { sb = 0; bph ^= 1; }
                    }
                } else {
                    for (int kb = 0; kb < prm.n_kb; ++kb) {
                        mbar_wait(tfull + 6 + 2 * STAGES + sb, bph ^ 1);
                        unsigned char* st = stages + sb * (A_BYTES + B_BYTES);
                        uint64_t* f = tfull + 6 + sb;
                        if (rank == 0) mbar_expect_tx(f, 2 * (A_BYTES + B_BYTES));
                        tma_load_2d<2>(st, &mA, f, kb * 128, ya);
                        tma_load_2d<2>(st + A_BYTES, &mB, f, kb * 128, yb);
                        if (++sb == 2 * STAGES) { sb = 0; bph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            const uint32_t id = idesc_i8(2 * A_ROWS, TN);
            int key_prev = -1, sb = 0, ab = 0;
            uint32_t aph = 0, bph = 0, tphb = 0;
            Seq seq;
            seq.init(prm, resA, cluster_id, n_clusters, total);
            for (int i = 0; i < seq.n; ++i) {
                uint64_t* tf = ab ? tfull + 4 : tfull;
                uint64_t* te = ab ? tfull + 5 : tempty;
                const uint32_t dH = tmem_base + (ab ? (uint32_t)TN : 0u);
                mbar_wait_cluster(te, ((tphb >> ab) & 1u) ^ 1u);
                fence_after();
                if (resA) {
                    int p, mt, nt;
                    seq.get(prm, i, p, mt, nt);
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
                        ah = sdesc(smem_u32(stages + kb * A_BYTES));
                        bh = sdesc(smem_u32((sb < nsb0 ? bring : bextra) + sb * B_BYTES));
                    } else {
                        mbar_wait(tfull + 6 + sb, bph);
                        fence_after();
                        const uint32_t s0 = smem_u32(stages + sb * (A_BYTES + B_BYTES));
                        ah = sdesc(s0);
                        bh = sdesc(s0 + A_BYTES);
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mma_i8(dH, ah + (uint64_t)(k * 2), bh + (uint64_t)(k * 2), id, (kb != 0 || k != 0) ? 1u : 0u);
                    if (resA) {
                        mma_commit<2>(tfull + 8 + kSlots + sb);
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
    } else {
        epilogue(prm, tmem_base, tfull, tempty, cluster_id, n_clusters, total, rank, warp, lane);
    }
    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}
}  // namespace rd

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled_rd)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_map_rd(CUtensorMap* m, const void* base, int64_t rows, int64_t Kp, int box_rows) {
    static PFN_encodeTiled_rd enc = nullptr;
    if (!enc) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
        enc = reinterpret_cast<PFN_encodeTiled_rd>(p);
    }
    cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)Kp};
    cuuint32_t box[2] = {128u, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_rowdot(const RowdotArgs& a, cudaStream_t st) {
    if (a.rowsA == 0 || a.rowsB == 0) return cudaSuccess;
    const int64_t rows = (int64_t)a.P * (a.rowsA + a.rowsB);
    if (rows >= (1ll << 31) || a.Kp % 128 || a.rd_nt % rd::TN || a.rowsB != (int64_t)a.rd_m * a.rd_nt)
        return cudaErrorInvalidValue;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    CUtensorMap maps[2];
    if (!make_map_rd(&maps[0], a.ops, rows, a.Kp, tc::A_ROWS) || !make_map_rd(&maps[1], a.ops, rows, a.Kp, rd::BROWS))
        return cudaErrorInvalidValue;
    rd::Params prm{};
    prm.rowsA = a.rowsA; prm.rowsB = a.rowsB; prm.b_off = (int64_t)a.P * a.rowsA;
    prm.P = a.P; prm.p0 = 0; prm.np = a.P;
    prm.n_kb = (int)(a.Kp / 128);
    prm.tiles_m = (int)((a.rowsA + 2 * tc::A_ROWS - 1) / (2 * tc::A_ROWS));
    prm.tiles_n = (int)((a.rowsB + rd::TN - 1) / rd::TN);
    prm.m2 = a.m2; prm.rd_nt = a.rd_nt; prm.rd_m = a.rd_m; prm.out = a.out;
    static SmemAttrOnce attr;
    if (cudaError_t e = attr.ensure(rd::k_rowdot, rd::SMEM_BYTES); e != cudaSuccess) return e;
    const int64_t tiles = (int64_t)prm.np * prm.tiles_m * prm.tiles_n;
    const int clusters = (int)(tiles < nsm / 2 ? tiles : nsm / 2);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(clusters * 2));
    cfg.blockDim = dim3(rd::NTHR);
    cfg.dynamicSmemBytes = rd::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ProfScope ps_(K_RESAMPLE, st);
    cudaError_t e = cudaLaunchKernelEx(&cfg, rd::k_rowdot, maps[0], maps[1], prm);
    note_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace cil
