// Persistent warp-specialised bf16 GEMM on 5th-gen tensor cores (sm_100a).
//
//   C[M,N] (op)= A[M,K] * B[K,N]     fp32 accumulate in TMEM
//
// One CTA per SM, 192 threads:
//   warp 0      TMA producer: A/B tiles -> 128B-swizzled smem ring (mbarrier full/empty)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> fused op -> global
// Two TMEM accumulators (2 x BN fp32 columns) let the epilogue of tile i
// overlap the mainloop of tile i+1.
//
// Operand majors cover the three pass shapes of a pipeline stage without any
// transposes in HBM:
//   F  Y  = X  . W^T   A=[M][K] (K-major)   B=[N][K] (K-major)
//   B  dX = dY . W     A=[M][K] (K-major)   B=[K][N] (MN-major)
//   W  dW += dY^T . X  A=[K][M] (MN-major)  B=[K][N] (MN-major)
#include <cudaTypedefs.h>

#include <cstdlib>
#include <map>
#include <unordered_map>
#include <mutex>
#include <vector>
#include <stdexcept>
#include <string>

#include "gemm.hpp"
#include "sm100.cuh"

namespace pbk {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 192;
// EPI_F32 epilogue staging: 4 epilogue warps x 2 buffers x [32 rows][32 fp32] (128B-swizzled), drained
// by TMA bulk reduce-adds (accumulate) or stores
constexpr int kEpiStage = 4 * 2 * 4096;
#ifndef PB_GEMM_SMEM_KB
#define PB_GEMM_SMEM_KB 200  // operand ring budget (KB): 6 stages of 32 KB for the CTA-pair 256-wide tiles
#endif

// BM2 = 2: each CTA holds TWO 128-row A sub-tiles (a CTA pair covers 512 x BN) sharing one B
// stage, and the two accumulators fill all 512 TMEM columns (single-buffered): a quarter less
// operand traffic per FLOP than BM2 = 1 (48 KB per 2 x 4.2 MFLOP instead of 32 KB per 4.2).
template <int BN, int CG, int BM2 = 1>
struct Cfg {
    static constexpr int kBRows = BN / CG;  // B rows (N) held by each CTA of the pair
    static constexpr int kABytes = BM * BK * 2 * BM2;
    static constexpr int kBBytes = kBRows * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = (PB_GEMM_SMEM_KB * 1024) / kStageBytes > 8 ? 8 : (PB_GEMM_SMEM_KB * 1024) / kStageBytes;
    static constexpr int kAccStride = BN <= 128 ? 128 : 256;  // accumulator buffer pitch (TMEM columns)
    static constexpr int kAccBufs = BM2 == 2 ? 1 : 2;          // double-buffered unless BM2 fills TMEM
    static constexpr int kTmemCols = 2 * kAccStride;           // (power of 2)
    static_assert(BM2 == 1 || (BN == 256 && CG == 2), "BM2 = 2 is a CTA-pair 512 x 256 tile");
    static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
    // EPI_F32: the barriers take a 1 KB slot, then the epilogue warps' fp32 staging for TMA
    static constexpr int kSmemF32 = kStages * kStageBytes + 1024 /*align*/ + 1024 /*barriers*/ + kEpiStage;
    static_assert(kSmemF32 <= 232448, "gemm: EPI_F32 staging over the opt-in shared memory limit");
};

struct alignas(128) GroupProblem {
    CUtensorMap ta, tb, tc;  // tc: fp32 C, box 32 x 32 (EPI_F32 epilogue)
    void* C;
    int M, N, K, ldc, tile0, ntiles, num_m, pad;
};

struct KParams {
    int M, N, K;
    void* C;
    void* C2;
    const __nv_bfloat16* aux;
    int ldc, ldaux;
    int accumulate;
    const GroupProblem* group;  // grouped launch: tiles come from this table
    int ngroup, total_tiles;
    // row scale (RMSNorm folded into the consuming GEMM): acc(row, :) *= rsqrt(rs[row] * rs_inv_n + rs_eps),
    // rs = the row's sum of squares over the normalised width
    const float* rs;
    float rs_inv_n, rs_eps;
    // EPI_RESID: ss_out[row] = sum of bf16(out)^2 over the row (the next RMSNorm's statistic), from
    // per-128-column partials (ss_part, [M][N/128]) summed in column order by the row group's last tile
    float* ss_out;
    float* ss_part;
    int* ss_cnt;
};

// Resolves tile t of the launch: its problem's descriptors, origin, K blocks, output.
struct TileRef {
    const CUtensorMap* ta;
    const CUtensorMap* tb;
    const CUtensorMap* tc;
    void* C;
    int m_blk, n_blk, num_k, ldc;
};
template <int BN, int CG, int BM2 = 1>
__device__ __forceinline__ TileRef resolve_tile(const KParams& p, const CUtensorMap* ta, const CUtensorMap* tb,
                                                const CUtensorMap* tc, int t, int& cursor) {
    if (p.group == nullptr) {
        const int num_m = (p.M + BM * CG * BM2 - 1) / (BM * CG * BM2);  // the last M / N tile may be half empty
        return TileRef{ta, tb, tc, p.C, t % num_m, t / num_m, p.K / BK, p.ldc};
    }
    while (t >= p.group[cursor].tile0 + p.group[cursor].ntiles) ++cursor;  // tiles visited in increasing order
    const GroupProblem& g = p.group[cursor];
    const int lt = t - g.tile0;
    return TileRef{&g.ta, &g.tb, &g.tc, g.C, lt % g.num_m, lt / g.num_m, g.K / BK, g.ldc};
}

// Whole tiles round-robin over the persistent CTAs (pairs).
struct TileIter {
    int t, step, num_tiles;
    __device__ TileIter(int num_tiles_, int cid, int ncl) : t(cid), step(ncl), num_tiles(num_tiles_) {}
    __device__ bool next(int& tile) {
        if (t >= num_tiles) return false;
        tile = t;
        t += step;
        return true;
    }
};

// CG = 1: one CTA per 128 x BN tile.  CG = 2: a CTA pair (cluster of 2) per
// 256 x BN tile; each CTA stages its 128 rows of A and BN/2 rows of B, the
// leader issues tcgen05.mma.cta_group::2 (M=256) and commits to both CTAs.
template <int BN, bool A_MN, bool B_MN, int EPI, int CG, int BM2>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                const __grid_constant__ CUtensorMap tma_c, const __grid_constant__ CUtensorMap tma_c2, KParams p) {
    using C_ = Cfg<BN, CG, BM2>;
    constexpr int kPairRows = BM * CG;  // rows of one MMA (both CTAs of a pair)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C_::kStages * C_::kStageBytes);
    uint64_t* empty = full + C_::kStages;
    uint64_t* tfull = empty + C_::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    // EPI_F32 staging (1 KB-aligned, after the barriers' 1 KB slot): [epilogue warp][2][32 rows][128 B]
    uint8_t* epi_stage = smem + C_::kStages * C_::kStageBytes + 1024;

    const uint32_t warp = warp_id();
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;
    const bool leader = rank == 0;
    const int num_tiles =
        p.group ? p.total_tiles : ((p.M + kPairRows * BM2 - 1) / (kPairRows * BM2)) * ((p.N + BN - 1) / BN);
    const int cid = int(blockIdx.x) / CG, ncl = int(gridDim.x) / CG;

    if (warp == 0 && elect_one()) {
        if (!p.group) {
            tma_prefetch(&tma_a);
            tma_prefetch(&tma_b);
        }
        for (int s = 0; s < C_::kStages; ++s) {
            mbar_init(&full[s], 1);  // leader's expect_tx covers both CTAs' bytes
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4 * CG);  // one arrive per epilogue warp of each CTA
        }
        fence_barrier_init();
    }
    // TMEM is allocated after griddepcontrol.wait, and for a CTA pair only once both CTAs are
    // resident: a CTA launched early by PDL must not hold (or block in) tcgen05.alloc while its
    // peer or the previous kernel still owns the columns (observed: a pair hung in the prologue
    // with one CTA at the cluster barrier and the other never leaving the allocation).
    pdl_wait();
    pdl_launch();
    if constexpr (CG == 2) cluster_sync();
    if (warp == 1) tmem_alloc<C_::kTmemCols, CG>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            int cursor = 0;
            TileIter it(num_tiles, cid, ncl);
            int t;
            while (it.next(t)) {
                const TileRef tr = resolve_tile<BN, CG, BM2>(p, &tma_a, &tma_b, &tma_c, t, cursor);
                const CUtensorMap* pa = tr.ta;
                const CUtensorMap* pb = tr.tb;
                const int num_k = tr.num_k;
                const int m0 = tr.m_blk * kPairRows * BM2 + int(rank) * BM, n0 = tr.n_blk * BN + int(rank) * C_::kBRows;
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * C_::kStageBytes;
                    uint8_t* sb = sa + C_::kABytes;
                    const int k0 = kb * BK;
                    if constexpr (CG == 1) {
                        mbar_expect_tx(&full[stage], C_::kStageBytes);
#pragma unroll
                        for (int s2 = 0; s2 < BM2; ++s2) {
                            if constexpr (A_MN) {
                                tma_load_2d(sa + s2 * 16384, pa, &full[stage], m0 + s2 * kPairRows, k0);
                                tma_load_2d(sa + s2 * 16384 + 8192, pa, &full[stage], m0 + s2 * kPairRows + 64, k0);
                            } else {
                                tma_load_2d(sa + s2 * 16384, pa, &full[stage], k0, m0 + s2 * kPairRows);
                            }
                        }
                        if constexpr (B_MN) {
#pragma unroll
                            for (int j = 0; j < C_::kBRows / 64; ++j)
                                tma_load_2d(sb + j * 8192, pb, &full[stage], n0 + 64 * j, k0);
                        } else {
                            tma_load_2d(sb, pb, &full[stage], k0, n0);
                        }
                    } else {
                        // the peer's bytes may land before the leader arms this phase: the phase
                        // cannot complete before the leader's arrive, and the previous phase is
                        // complete (the peer waited on `empty`, released after it was consumed)
                        const uint32_t bar = map_peer(smem_u32(&full[stage]), 0);
                        if (leader) mbar_expect_tx(&full[stage], CG * C_::kStageBytes);
#pragma unroll
                        for (int s2 = 0; s2 < BM2; ++s2) {
                            if constexpr (A_MN) {
                                tma_load_2d_2sm(sa + s2 * 16384, pa, bar, m0 + s2 * kPairRows, k0);
                                tma_load_2d_2sm(sa + s2 * 16384 + 8192, pa, bar, m0 + s2 * kPairRows + 64, k0);
                            } else {
                                tma_load_2d_2sm(sa + s2 * 16384, pa, bar, k0, m0 + s2 * kPairRows);
                            }
                        }
                        if constexpr (B_MN) {
#pragma unroll
                            for (int j = 0; j < C_::kBRows / 64; ++j)
                                tma_load_2d_2sm(sb + j * 8192, pb, bar, n0 + 64 * j, k0);
                        } else {
                            tma_load_2d_2sm(sb, pb, bar, k0, n0);
                        }
                    }
                    if (++stage == C_::kStages) stage = 0, phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (leader CTA)
        if (leader) {
            constexpr uint32_t idesc = idesc_bf16(BM * CG, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            int cursor = 0;
            TileIter it(num_tiles, cid, ncl);
            int t;
            while (it.next(t)) {
                const int num_k = resolve_tile<BN, CG, BM2>(p, &tma_a, &tma_b, &tma_c, t, cursor).num_k;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * C_::kAccStride;  // (BM2 = 2: sub-tile s2 at + s2 * 256)
                for (int kb = 0; kb < num_k; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t sa = smem_u32(smem + stage * C_::kStageBytes);
                        const uint32_t sb = sa + C_::kABytes;
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            const uint64_t bd = B_MN ? sdesc(sb + k * 2048, 8192, 1024) : sdesc(sb + k * 32, 16, 1024);
                            const bool accum = kb != 0 || k != 0;
#pragma unroll
                            for (int s2 = 0; s2 < BM2; ++s2) {
                                const uint32_t sa2 = sa + s2 * 16384;
                                const uint64_t ad = A_MN ? sdesc(sa2 + k * 2048, 8192, 1024) : sdesc(sa2 + k * 32, 16, 1024);
                                if constexpr (CG == 1)
                                    tc_mma(d_tmem + s2 * 256, ad, bd, idesc, accum);
                                else
                                    tc_mma2(d_tmem + s2 * 256, ad, bd, idesc, accum);
                            }
                        }
                        if constexpr (CG == 1) {
                            tc_commit(&empty[stage]);  // smem slot free once these MMAs retire
                            if (kb == num_k - 1) tc_commit(&tfull[acc]);
                        } else {
                            tc_commit2(&empty[stage], 0x3);
                            if (kb == num_k - 1) tc_commit2(&tfull[acc], 0x3);
                        }
                    }
                    __syncwarp();
                    if (++stage == C_::kStages) stage = 0, phase ^= 1;
                }
                if (++acc == C_::kAccBufs) acc = 0, acc_phase ^= 1;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
        const int row_in_tile = int(q * 32 + lane_id());
        int epi_chunk = 0;  // EPI_F32: staged blocks issued by this warp (staging buffer parity)
        int acc = 0;
        uint32_t acc_phase = 0;
        int cursor = 0;
        TileIter it(num_tiles, cid, ncl);
        int t;
        while (it.next(t)) {
            const TileRef tr = resolve_tile<BN, CG, BM2>(p, &tma_a, &tma_b, &tma_c, t, cursor);
            const int m0 = tr.m_blk * kPairRows * BM2 + int(rank) * BM, n0 = tr.n_blk * BN;
            void* const Cout = tr.C;
            const int ldc = tr.ldc;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int row0 = m0 + row_in_tile;
            const uint32_t tbase0 = tmem_base + ((q * 32) << 16) + acc * C_::kAccStride;
            // residual / pre-activation operand of the next 32 columns is loaded one chunk ahead
            // (each element is read and written by the same thread, so C may alias aux)
            constexpr bool kAux = EPI == EPI_RESID || EPI == EPI_DGELU;
#pragma unroll 1
            for (int s2 = 0; s2 < BM2; ++s2) {  // BM2 = 2: the CTA's second 128-row sub-tile is 256 rows on
            const int row = row0 + s2 * kPairRows;
            const uint32_t tbase = tbase0 + s2 * 256;
            const float rsc = (p.rs && row < p.M) ? rsqrtf(p.rs[row] * p.rs_inv_n + p.rs_eps) : 1.f;
            float ssq = 0.f;  // EPI_RESID with ss_out: sum of squares of this row's stored outputs per 128 columns
            uint4 aux_next[4];
            // (aux epilogues run only on full tiles: layer GEMMs have M = tokens, N = h or 4h)
            if constexpr (kAux) {
                const uint4* s4 = reinterpret_cast<const uint4*>(p.aux + size_t(row) * p.ldaux + n0);
#pragma unroll
                for (int j = 0; j < 4; ++j) aux_next[j] = s4[j];
            }
            float vnext[32];  // the next 32 accumulator columns, loaded from TMEM while this chunk is processed
            tmem_ld32(tbase, vnext);
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint4 aux_cur[4];
                if constexpr (kAux) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) aux_cur[j] = aux_next[j];
                    if (c + 32 < BN && n0 + c + 32 < p.N) {  // (BN = 160 / 192: the last tile may be partial)
                        const uint4* s4 = reinterpret_cast<const uint4*>(p.aux + size_t(row) * p.ldaux + n0 + c + 32);
#pragma unroll
                        for (int j = 0; j < 4; ++j) aux_next[j] = s4[j];
                    }
                }
                float v[32];
                tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = vnext[e];
                if (c + 32 < BN) tmem_ld32(tbase + c + 32, vnext);
                if (p.rs) {  // warp-uniform: folded RMSNorm of this row
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] *= rsc;
                }
                const int col = n0 + c;
                // partial last tile (M or N = 128 mod 256): nothing to store outside the matrix
                if (!(p.group || (row < p.M && col < p.N))) continue;
                if constexpr (EPI == EPI_F32) {
                    // C (+)= acc through shared memory and the TMA: the warp's 32 rows x 32 columns go to a
                    // 128B-swizzled staging buffer (a thread writes its row: conflict-free), then one
                    // bulk tensor reduce-add (accumulate; one update per element per launch, so the result
                    // is deterministic) or store covers the whole 4 KB block in full 128 B lines
                    (void)Cout;
                    (void)ldc;
                    uint8_t* buf = epi_stage + (q * 2 + (epi_chunk & 1)) * 4096;
                    if (lane_id() == 0 && epi_chunk >= 2)  // this buffer's previous block has been read out
                        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        *reinterpret_cast<float4*>(buf + lane_id() * 128 + ((j ^ (lane_id() & 7)) << 4)) =
                            make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane_id() == 0) {
                        const int rowb = row - int(lane_id());  // the warp's first row
                        if (p.accumulate)
                            asm volatile(
                                "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                    reinterpret_cast<uint64_t>(tr.tc)),
                                "r"(smem_u32(buf)), "r"(col), "r"(rowb)
                                : "memory");
                        else
                            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                             reinterpret_cast<uint64_t>(tr.tc)),
                                         "r"(smem_u32(buf)), "r"(col), "r"(rowb)
                                         : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    ++epi_chunk;
                } else {
                    if constexpr (kAux) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint4 a = aux_cur[j];
                            uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                float lo = bf16_lo(w[e]), hi = bf16_hi(w[e]);
                                if constexpr (EPI == EPI_RESID) {
                                    v[8 * j + 2 * e] += lo;
                                    v[8 * j + 2 * e + 1] += hi;
                                } else {
                                    v[8 * j + 2 * e] *= gelu_grad(lo);
                                    v[8 * j + 2 * e + 1] *= gelu_grad(hi);
                                }
                            }
                        }
                    }
                    // single-output epilogues stage the bf16 block in shared memory ([32 rows][64 cols], 128B-
                    // swizzled: two 32-column chunks) and write it with one TMA tensor store per 64 columns
                    constexpr bool kStaged = EPI == EPI_STORE || EPI == EPI_RESID || EPI == EPI_DGELU;
                    uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.C) + size_t(row) * p.ldc + col);
                    const int half = (c >> 5) & 1;
                    // GELU (two outputs): u and gelu(u) blocks single-buffered in the warp's two slots
                    uint8_t* sbuf = epi_stage + (q * 2 + (EPI == EPI_GELU ? 0 : (epi_chunk & 1))) * 4096;
                    uint8_t* gbuf = epi_stage + (q * 2 + 1) * 4096;
                    if constexpr (kStaged || EPI == EPI_GELU) {
                        if (half == 0) {
                            if (lane_id() == 0 && epi_chunk >= (EPI == EPI_GELU ? 1 : 2)) {
                                if constexpr (EPI == EPI_GELU)  // both previous stores have read their blocks
                                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                                else  // this buffer's previous block has been read out
                                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                            }
                            __syncwarp();
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint4 o = make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                                   pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
                        if constexpr (kStaged || EPI == EPI_GELU)
                            *reinterpret_cast<uint4*>(sbuf + lane_id() * 128 + (((half * 4 + j) ^ (lane_id() & 7)) << 4)) = o;
                        else
                            d4[j] = o;
                        if constexpr (EPI == EPI_RESID) {
                            if (p.ss_out) {
                                const uint32_t w4[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const float lo = bf16_lo(w4[e]), hi = bf16_hi(w4[e]);
                                    ssq = fmaf(lo, lo, fmaf(hi, hi, ssq));
                                }
                            }
                        }
                    }
                    if constexpr (kStaged) {
                        if (half == 1) {  // the 64-column block is complete: one TMA store
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            __syncwarp();
                            if (lane_id() == 0) {
                                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                                 reinterpret_cast<uint64_t>(tr.tc)),
                                             "r"(smem_u32(sbuf)), "r"(col - 32), "r"(row - int(lane_id()))
                                             : "memory");
                                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                            }
                            ++epi_chunk;
                        }
                    }
                    if constexpr (EPI == EPI_RESID) {
                        if (p.ss_out && ((c + 32) & 127) == 0) {  // end of a 128-column chunk: its partial
                            p.ss_part[size_t(row) * (p.N >> 7) + (col >> 7)] = ssq;
                            ssq = 0.f;
                        }
                    }
                    if constexpr (EPI == EPI_GELU) {
                        // activation from the bf16-rounded pre-activation, as the backward sees it
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            float g[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e)
                                g[e] = gelu_f(__bfloat162float(__float2bfloat16_rn(v[8 * j + e])));
                            *reinterpret_cast<uint4*>(gbuf + lane_id() * 128 + (((half * 4 + j) ^ (lane_id() & 7)) << 4)) =
                                make_uint4(pack_bf16(g[0], g[1]), pack_bf16(g[2], g[3]), pack_bf16(g[4], g[5]),
                                           pack_bf16(g[6], g[7]));
                        }
                        if (half == 1) {  // both 64-column blocks complete: two TMA stores
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            __syncwarp();
                            if (lane_id() == 0) {
                                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                                 reinterpret_cast<uint64_t>(&tma_c)),
                                             "r"(smem_u32(sbuf)), "r"(col - 32), "r"(row - int(lane_id()))
                                             : "memory");
                                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                                 reinterpret_cast<uint64_t>(&tma_c2)),
                                             "r"(smem_u32(gbuf)), "r"(col - 32), "r"(row - int(lane_id()))
                                             : "memory");
                                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                            }
                            ++epi_chunk;
                        }
                    }
                }
            }
            if constexpr (EPI == EPI_RESID) {
                if (p.ss_out) {
                    // deterministic row reduction: the last of the row group's N tiles sums the
                    // partials in column order (threadfence reduction; the counter resets itself)
                    __threadfence();
                    __syncwarp();
                    int last = 0;
                    if (lane_id() == 0) last = atomicAdd(p.ss_cnt + (row >> 5), 1) == (p.N + BN - 1) / BN - 1;
                    if (__shfl_sync(0xffffffffu, last, 0)) {
                        __threadfence();
                        if (row < p.M) {
                            float sum = 0.f;
                            const int P = p.N >> 7;  // the row's partials are contiguous: vector loads, column order
                            const float* pr = p.ss_part + size_t(row) * P;
                            if ((P & 3) == 0) {
                                for (int q = 0; q < P; q += 4) {
                                    const float4 v4 = __ldcg(reinterpret_cast<const float4*>(pr + q));
                                    sum += v4.x;
                                    sum += v4.y;
                                    sum += v4.z;
                                    sum += v4.w;
                                }
                            } else {
                                for (int q = 0; q < P; ++q) sum += __ldcg(pr + q);
                            }
                            p.ss_out[row] = sum;
                        }
                        if (lane_id() == 0) p.ss_cnt[row >> 5] = 0;
                    }
                }
            }
            }  // s2
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) {
                if constexpr (CG == 1)
                    mbar_arrive(&tempty[acc]);
                else
                    mbar_arrive_cluster(map_peer(smem_u32(&tempty[acc]), 0));
            }
            if (++acc == C_::kAccBufs) acc = 0, acc_phase ^= 1;
        }
        if constexpr (EPI == EPI_F32 || EPI == EPI_STORE || EPI == EPI_RESID || EPI == EPI_DGELU || EPI == EPI_GELU) {
            if (lane_id() == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // staging stays valid
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_free<C_::kTmemCols, CG>(tmem_base);
    }
}

}  // namespace

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
            throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// 2-D tensor [outer][inner] with row stride `ld` elements; box = box_inner x box_outer; 128B swizzle.
// Descriptors are pure functions of these arguments, so they are cached per host thread (the
// executor re-issues the same few hundred GEMM / attention shapes on the same buffers every step:
// one hash lookup instead of a driver encode per operand per launch).
namespace {
struct MapKey {
    const void* base;
    uint64_t inner, outer, ld;
    uint32_t box_inner, box_outer, dt;
    bool operator==(const MapKey& o) const {
        return base == o.base && inner == o.inner && outer == o.outer && ld == o.ld && box_inner == o.box_inner &&
               box_outer == o.box_outer && dt == o.dt;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        uint64_t h = reinterpret_cast<uint64_t>(k.base) * 0x9E3779B97F4A7C15ull;
        for (uint64_t v : {k.inner, k.outer, k.ld, uint64_t(k.box_inner) << 32 | k.box_outer, uint64_t(k.dt)})
            h = (h ^ v) * 0x100000001B3ull;
        return size_t(h);
    }
};
}  // namespace

CUtensorMap make_map_t(const void* base, CUtensorMapDataType dt, uint32_t esize, uint64_t inner, uint64_t outer,
                       uint64_t ld, uint32_t box_inner, uint32_t box_outer) {
    thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
    const MapKey key{base, inner, outer, ld, box_inner, box_outer, uint32_t(dt) | (esize << 8)};
    if (auto it = cache.find(key); it != cache.end()) return it->second;
    if (cache.size() > 8192) cache.clear();
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld * esize};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    cache.emplace(key, m);
    return m;
}

CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                     uint32_t box_outer) {
    return make_map_t(base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, inner, outer, ld, box_inner, box_outer);
}

namespace {

int sm_count() {
    static int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

template <int BN, bool A_MN, bool B_MN, int EPI, int CG, int BM2 = 1>
void launch(const GemmArgs& g, cudaStream_t s) {
    using C_ = Cfg<BN, CG, BM2>;
    auto kern = gemm_kernel<BN, A_MN, B_MN, EPI, CG, BM2>;
    constexpr bool staged = EPI == EPI_F32 || EPI == EPI_STORE || EPI == EPI_RESID || EPI == EPI_DGELU || EPI == EPI_GELU;
    constexpr int smem = staged ? C_::kSmemF32 : C_::kSmem;
    static bool attr = [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (CG == 2) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
        return true;
    }();
    (void)attr;
    CUtensorMap ta = A_MN ? make_map(g.A, g.M, g.K, g.lda, 64, 64) : make_map(g.A, g.K, g.M, g.lda, 64, BM);
    CUtensorMap tb = B_MN ? make_map(g.B, g.N, g.K, g.ldb, 64, 64) : make_map(g.B, g.K, g.N, g.ldb, 64, C_::kBRows);
    CUtensorMap tc{};
    if constexpr (EPI == EPI_F32)
        tc = make_map_t(g.C, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, uint64_t(g.N), uint64_t(g.M), uint64_t(g.ldc), 32, 32);
    else if constexpr (staged)
        tc = make_map(g.C, uint64_t(g.N), uint64_t(g.M), uint64_t(g.ldc), 64, 32);
    CUtensorMap tc2{};
    if constexpr (EPI == EPI_GELU) tc2 = make_map(g.C2, uint64_t(g.N), uint64_t(g.M), uint64_t(g.ldc), 64, 32);
    KParams kp{g.M, g.N, g.K, g.C, g.C2, g.aux, g.ldc, g.ldaux, g.accumulate, nullptr, 0, 0,
               g.rs, g.rs_inv_n, g.rs_eps, g.ss_out, g.ss_part, g.ss_cnt};
    const int tiles = ((g.M + BM * CG * BM2 - 1) / (BM * CG * BM2)) * ((g.N + BN - 1) / BN);
    const int slots = sm_count() / CG;
    const int grid = (tiles < slots ? tiles : slots) * CG;
    launch_k(kern, dim3(grid), dim3(kThreads), smem, s, CG, ta, tb, tc, tc2, kp);
}

template <int BN, int CG, int BM2 = 1>
void dispatch(const GemmArgs& g, cudaStream_t s) {
    if (!g.a_mn && !g.b_mn) {
        switch (g.epi) {
            case EPI_STORE: return launch<BN, false, false, EPI_STORE, CG, BM2>(g, s);
            case EPI_GELU: return launch<BN, false, false, EPI_GELU, CG, BM2>(g, s);
            case EPI_RESID: return launch<BN, false, false, EPI_RESID, CG, BM2>(g, s);
            case EPI_F32: return launch<BN, false, false, EPI_F32, CG, BM2>(g, s);
            default: break;
        }
    } else if (!g.a_mn && g.b_mn) {
        switch (g.epi) {
            case EPI_STORE: return launch<BN, false, true, EPI_STORE, CG, BM2>(g, s);
            case EPI_DGELU: return launch<BN, false, true, EPI_DGELU, CG, BM2>(g, s);
            case EPI_RESID: return launch<BN, false, true, EPI_RESID, CG, BM2>(g, s);
            case EPI_F32: return launch<BN, false, true, EPI_F32, CG, BM2>(g, s);
            default: break;
        }
    } else if (g.a_mn && g.b_mn) {
        if (g.epi == EPI_F32) return launch<BN, true, true, EPI_F32, CG, BM2>(g, s);
        if (g.epi == EPI_STORE) return launch<BN, true, true, EPI_STORE, CG, BM2>(g, s);
    } else {
        if (g.epi == EPI_F32) return launch<BN, true, false, EPI_F32, CG, BM2>(g, s);
        if (g.epi == EPI_STORE) return launch<BN, true, false, EPI_STORE, CG, BM2>(g, s);
    }
    throw std::invalid_argument("gemm: unsupported operand-major / epilogue combination");
}

}  // namespace

int num_sms() { return sm_count(); }

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PB_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

int gemm_bn(const GemmArgs& g) {
    const int tiles256 = (g.N % 256 == 0) ? (g.M / BM) * (g.N / 256) : 0;
    return (tiles256 >= num_sms()) ? 256 : 128;
}

bool gemm_group_ok(const GemmArgs& g) {
    return g.a_mn && g.b_mn && g.epi == EPI_F32 && g.M % 256 == 0 && g.N % 256 == 0 && g.K % BK == 0;
}

GemmGroup gemm_group_create(const GemmArgs* probs, int n) {
    std::vector<GroupProblem> t(size_t(std::max(n, 1)));
    int tiles = 0;
    for (int i = 0; i < n; ++i) {
        const GemmArgs& g = probs[i];
        if (!gemm_group_ok(g) || g.accumulate != probs[0].accumulate)
            throw std::invalid_argument("gemm group: problems must be MN/MN fp32 with M, N % 256 == 0");
        GroupProblem& q = t[i];
        q.ta = make_map(g.A, g.M, g.K, g.lda, 64, 64);
        q.tb = make_map(g.B, g.N, g.K, g.ldb, 64, 64);
        q.tc = make_map_t(g.C, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, uint64_t(g.N), uint64_t(g.M), uint64_t(g.ldc), 32, 32);
        q.C = g.C;
        q.M = g.M, q.N = g.N, q.K = g.K, q.ldc = g.ldc;
        q.num_m = g.M / 256;
        q.tile0 = tiles;
        q.ntiles = (g.M / 256) * (g.N / 256);
        tiles += q.ntiles;
    }
    GemmGroup out;
    if (cudaMalloc(&out.table, sizeof(GroupProblem) * t.size()) != cudaSuccess)
        throw std::runtime_error("gemm group: table allocation failed");
    if (cudaMemcpy(out.table, t.data(), sizeof(GroupProblem) * t.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("gemm group: table upload failed");
    out.n = n;
    out.total_tiles = tiles;
    out.accumulate = probs[0].accumulate;
    return out;
}

void gemm_group_run(const GemmGroup& g, cudaStream_t s) {
    if (g.n == 0) return;
    using C_ = Cfg<256, 2, 1>;
    auto kern = gemm_kernel<256, true, true, EPI_F32, 2, 1>;
    static bool attr = [&] {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::kSmemF32);
        return true;
    }();
    (void)attr;
    KParams kp{0, 0, 0, nullptr, nullptr, nullptr, 0, 0, g.accumulate,
               static_cast<const GroupProblem*>(g.table), g.n, g.total_tiles, nullptr, 0.f, 0.f, nullptr, nullptr, nullptr};
    const int slots = sm_count() / 2;
    const int grid = (g.total_tiles < slots ? g.total_tiles : slots) * 2;
    CUtensorMap dummy{};
    launch_k(kern, dim3(grid), dim3(kThreads), C_::kSmemF32, s, 2, dummy, dummy, dummy, dummy, kp);
}

void gemm_group_destroy(GemmGroup& g) {
    if (g.table) cudaFree(g.table);
    g.table = nullptr;
    g.n = 0;
}

static int g_force_cg = -1;  // tests: -1 auto, 1 or 2 forced
void gemm_force_cta_group(int cg) { g_force_cg = cg; }

// 512 x 256 CTA-pair tiles (BM2 = 2) for full-tile launches (PB_GEMM_BM2=1 or the test hook);
// a pair's epilogue is then not overlapped with its next tile's main loop.  Default: K >= 8192 only:
// measured at T = 4096 it gains on long-K shapes (FC1 dX, K = 8192: 1399 -> 1454 TFLOP/s; FC2,
// K = 8192: 1355 -> 1375) but loses more on K = 2048 (FC1 + GELU 1317 -> 1016), where the exposed
// epilogue is a quarter of the tile; 82.5k vs 86.5k tokens/s in-step with it on everywhere.
static int g_force_bm2 = -1;  // tests: -1 environment, 0 off, 1 on
void gemm_force_bm2(int on) { g_force_bm2 = on; }
static bool use_bm2(const GemmArgs& g) {
    // PB_GEMM_BM2: 1 = every eligible launch, 0 = never, unset = long-K launches only (K >= 8192)
    static const int env = [] {
        const char* e = std::getenv("PB_GEMM_BM2");
        return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : -1;
    }();
    const int mode = g_force_bm2 >= 0 ? g_force_bm2 : env;
    const bool on = mode == 1 || (mode < 0 && g.K >= 8192);
    return on && g.M % 512 == 0 && g.N % 256 == 0;
}

void gemm(const GemmArgs& g, cudaStream_t s) {
    if (g.M % BM || g.N % 128 || g.K % BK || g.M <= 0 || g.N <= 0 || g.K <= 0)
        throw std::invalid_argument("gemm: M%128, N%128, K%64 must be 0 (M=" + std::to_string(g.M) +
                                    " N=" + std::to_string(g.N) + " K=" + std::to_string(g.K) + ")");
    // CTA pairs also take M or N = 128 (mod 256) (e.g. the LM head, V = 50304): TMA zero-fills
    // the empty half of the last tile and the epilogue skips its rows / columns
    const bool full = g.M % 256 == 0 && g.N % 256 == 0;
    const bool pair_ok = full || (g.M >= 256 && g.N >= 256 && g.epi != EPI_RESID && g.epi != EPI_DGELU);
    const int cg = g_force_cg > 0 ? (pair_ok ? g_force_cg : 1) : (pair_ok ? 2 : 1);
    if (g.rs && (g.epi == EPI_RESID || g.epi == EPI_F32))
        throw std::invalid_argument("gemm: a row scale applies to the store / GELU / dGELU epilogues");
    if (g.ss_out && g.epi != EPI_RESID) throw std::invalid_argument("gemm: ss_out needs the residual epilogue");
    if (g.ss_out && (!g.ss_part || !g.ss_cnt || g.N % 128))
        throw std::invalid_argument("gemm: ss_out needs the ss_part / ss_cnt workspace and N % 128 == 0");
    if (cg == 2 && use_bm2(g))
        dispatch<256, 2, 2>(g, s);
    else if (cg == 2)
        dispatch<256, 2>(g, s);
    else if (gemm_bn(g) == 256)
        dispatch<256, 1>(g, s);
    else
        dispatch<128, 1>(g, s);
}

}  // namespace pbk
