// Causal flash attention forward on 5th-gen tensor cores (sm_100a).
//
// One CTA per (128-query tile, head, sequence); 192 threads:
//   warp 0     TMA: Q tile once, then a 2-stage ring of K/V tiles (128 keys x 128 d)
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//                S_j  = Q K_j^T      (M=128 q, N=128 keys, K=128 d)  -> TMEM S[j%2]
//                O   += P_j V_j      (M=128 q, N=128 d,   K=128 keys) -> TMEM O
//   warps 2-5  softmax: thread = query row = TMEM lane; reads its S row with
//              tcgen05.ld, online softmax in registers (no shuffles), writes P
//              (bf16, 128B-swizzled K-major) to smem for the PV MMA.
// S_{j+1} is computed while the softmax of S_j runs (two S buffers).  P goes back to TMEM
// (bf16 pairs, two buffers) and feeds the PV MMA as its A operand, so the softmax of tile j
// overlaps PV_{j-1} and smem holds only Q and a 3-stage K/V ring.  The
// running max is rescaled lazily: O (in TMEM) is only rescaled when a row's
// max grows by more than 2^8, which keeps the result exact (O and the row sum
// share the same stale max) and avoids a TMEM round trip per tile.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "ops.hpp"
#include "sm100.cuh"

namespace pbk {

namespace {

constexpr int D = 128;
constexpr int BQ = 128;
constexpr int BK = 128;
constexpr int kTile = BQ * D * 2;  // 32 KB: two 128B-swizzled atoms of [128 rows][64]
constexpr float kLog2e = 1.4426950408889634f;

constexpr int kFwdStages = 3;  // K/V ring depth of the forward kernel
struct FwdSmem {
    static constexpr int q = 0;
    static constexpr int k0 = kTile;                       // [3]
    static constexpr int v0 = k0 + kFwdStages * kTile;     // [3]
    static constexpr int bars = v0 + kFwdStages * kTile;
    static constexpr int total = bars + 256 + 1024;
};
static_assert(FwdSmem::total <= 232448, "attn fwd: shared memory over the sm_100 opt-in limit");

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
// ------------------------------------------------------------------ backward helpers
// D[h][t] = sum_d dO * O (the softmax-backward row term) and zero the fp32 dQ accumulator.
__global__ void attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ dout, const __nv_bfloat16* __restrict__ out,
                                    float* __restrict__ dsum, float* __restrict__ dq_acc, int H, int T) {
    pdl_wait();
    pdl_launch();
    const int t = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 4
    for (int head = warp; head < H; head += blockDim.x >> 5) {
        const size_t off = size_t(t) * H * D + head * D + lane * 4;
        uint2 a = *reinterpret_cast<const uint2*>(dout + off);
        uint2 b = *reinterpret_cast<const uint2*>(out + off);
        float s = bf16_lo(a.x) * bf16_lo(b.x) + bf16_hi(a.x) * bf16_hi(b.x) + bf16_lo(a.y) * bf16_lo(b.y) +
                  bf16_hi(a.y) * bf16_hi(b.y);
#pragma unroll
        for (int k = 16; k; k >>= 1) s += __shfl_xor_sync(0xffffffff, s, k);
        if (lane == 0) dsum[size_t(head) * T + t] = s;
        *reinterpret_cast<float4*>(dq_acc + off) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (t == 0 && threadIdx.x == 0) reinterpret_cast<int*>(dsum + size_t(H) * T)[0] = 0;  // bwd work counter
}

// dQ (bf16, into the q columns of dqkv) = scale * dq_acc, times the row's folded-RMSNorm factor
// rsqrt(rs[t] * rs_inv_n + rs_eps) when rs is given (dqkv' = rstd1 * dqkv, see executor.cpp)
__global__ void attn_dq_store_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, int H,
                                     float scale, const float* __restrict__ rs, float rs_inv_n, float rs_eps) {
    pdl_wait();
    pdl_launch();
    const int t = blockIdx.x;
    const float f = rs ? scale * rsqrtf(rs[t] * rs_inv_n + rs_eps) : scale;
#pragma unroll 4  // the row's loads in flight together (one at a time: 4.8 TB/s under ncu)
    for (int c = threadIdx.x * 4; c < H * D; c += blockDim.x * 4) {
        float4 v = *reinterpret_cast<const float4*>(dq_acc + size_t(t) * H * D + c);
        uint2 o = make_uint2(pack_bf16(v.x * f, v.y * f), pack_bf16(v.z * f, v.w * f));
        *reinterpret_cast<uint2*>(dqkv + size_t(t) * 3 * H * D + c) = o;
    }
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// byte offset of (row, col) in a [128 rows][128 cols] bf16 tile stored as two
// 128B-swizzled K-major atoms (cols 0-63, 64-127)
__device__ __forceinline__ uint32_t sw128(int row, int col) {
    return uint32_t((col >> 6) * 16384 + row * 128 + ((((col & 63) >> 3) ^ (row & 7)) << 4) + (col & 7) * 2);
}

// Phase stamps (clock64) of block 0, compiled in only with -DPB_ATTN_TRACE_BUILD (build.py:
// PB_ATTN_TRACE_BUILD=1); read by PB_ATTN_TRACE / PB_ATTN_TRACE_FWD (tests/trace_attn_*.py)
__device__ unsigned long long* g_attn_trace = nullptr;
#ifdef PB_ATTN_TRACE_BUILD
#define ATRACE(i, ev)                                                                        \
    do {                                                                                     \
        if (g_attn_trace && blockIdx.x == 0 && (i) < 32) g_attn_trace[(i) * 16 + (ev)] = clock64(); \
    } while (0)
#else
#define ATRACE(i, ev) \
    do {              \
    } while (0)
#endif

__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}

__device__ __forceinline__ void tmem_st32u(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

__global__ void __launch_bounds__(192, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ lse2, int seq, int H, int T, float scale) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + FwdSmem::bars);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;   // [3]
    uint64_t* kv_empty = bars + 4;  // [3]
    uint64_t* s_full = bars + 7;    // [2]
    uint64_t* s_free = bars + 9;    // [2]
    uint64_t* p_full = bars + 11;   // [2]
    uint64_t* p_empty = bars + 13;  // [2]
    uint64_t* o_full = bars + 15;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

    const uint32_t warp = warp_id();
    const int nqb = seq / BQ;
    // 1-D grid ordered heaviest causal tile first across all (head, sequence): LPT dispatch
    const int hb = int(blockIdx.x) % (H * (T / seq));
    const int qb = nqb - 1 - int(blockIdx.x) / (H * (T / seq));
    const int head = hb % H, b = hb / H;
    const int row0 = b * seq + qb * BQ;        // first token row of this Q tile
    const int nkv = qb + 1;                    // causal: key tiles 0..qb

    if (warp == 0 && elect_one()) {
        tma_prefetch(&tm);
        mbar_init(q_full, 1);
        for (int i = 0; i < kFwdStages; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 4);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&p_full[i], 4);
            mbar_init(&p_empty[i], 1);
        }
        mbar_init(o_full, 1);
        fence_barrier_init();
    }
    // TMEM is allocated only once the previous kernel in the stream has finished: a CTA that
    // launched early (PDL) never holds TMEM while it waits (see gemm_tc.cu)
    pdl_wait();
    pdl_launch();
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;  // cols [0,128) S0, [128,256) S1, [256,384) O, [384,448) P0, [448,512) P1

    if (warp == 0) {
        if (elect_one()) {
            const int cq = head * D, ck = H * D + head * D, cv = 2 * H * D + head * D;
            mbar_expect_tx(q_full, kTile);
            tma_load_2d(sm + FwdSmem::q, &tm, q_full, cq, row0);
            tma_load_2d(sm + FwdSmem::q + 16384, &tm, q_full, cq + 64, row0);
            for (int j = 0; j < nkv; ++j) {
                const int st = j % kFwdStages;
                if (j >= kFwdStages) mbar_wait(&kv_empty[st], ((j - kFwdStages) / kFwdStages) & 1);
                mbar_expect_tx(&kv_full[st], 2 * kTile);
                const int kr = b * seq + j * BK;
                uint8_t* ks = sm + FwdSmem::k0 + st * kTile;
                uint8_t* vs = sm + FwdSmem::v0 + st * kTile;
                tma_load_2d(ks, &tm, &kv_full[st], ck, kr);
                tma_load_2d(ks + 16384, &tm, &kv_full[st], ck + 64, kr);
                tma_load_2d(vs, &tm, &kv_full[st], cv, kr);
                tma_load_2d(vs + 16384, &tm, &kv_full[st], cv + 64, kr);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc_s = idesc_bf16(128, 128, false, false);
        constexpr uint32_t idesc_o = idesc_bf16(128, 128, false, true);
        const uint32_t sq = smem_u32(sm + FwdSmem::q);
        mbar_wait(q_full, 0);
        auto issue_pv = [&](int j) {  // O += P_j V_j, P from TMEM
            const int pb = j & 1;
            const int kv = j % kFwdStages;
            if (lane_id() == 0) ATRACE(j, 11);
            mbar_wait(&p_full[pb], (j >> 1) & 1);
            tc_fence_after();
            if (lane_id() == 0) ATRACE(j, 12);
            if (elect_one()) {
                const uint32_t sv = smem_u32(sm + FwdSmem::v0 + kv * kTile);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    tc_mma_ts(tmem + 256, tmem + 384 + pb * 64 + kk * 8, sdesc(sv + kk * 2048, 16384, 1024), idesc_o,
                              (j | kk) != 0);
                tc_commit(&kv_empty[kv]);
                tc_commit(&p_empty[pb]);
            }
            __syncwarp();
        };
        for (int j = 0; j < nkv; ++j) {
            const int st = j & 1;
            const int kv = j % kFwdStages;
            if (lane_id() == 0) ATRACE(j, 8);
            mbar_wait(&kv_full[kv], (j / kFwdStages) & 1);
            if (lane_id() == 0) ATRACE(j, 9);
            if (j >= 2) mbar_wait(&s_free[st], ((j - 2) >> 1) & 1);
            tc_fence_after();
            if (lane_id() == 0) ATRACE(j, 10);
            if (elect_one()) {
                const uint32_t sk = smem_u32(sm + FwdSmem::k0 + kv * kTile);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t ad = sdesc(sq + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
                    const uint64_t bd = sdesc(sk + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
                    tc_mma(tmem + st * 128, ad, bd, idesc_s, kk != 0);
                }
                tc_commit(&s_full[st]);
            }
            __syncwarp();
            if (j >= 1) issue_pv(j - 1);
        }
        issue_pv(nkv - 1);
        if (elect_one()) tc_commit(o_full);
        __syncwarp();
    } else {
        // ------------------------------------------------------------ softmax
        const uint32_t q4 = warp & 3;
        const int r = int(q4 * 32 + lane_id());  // query row in tile == TMEM lane
        const uint32_t lane_base = (q4 * 32) << 16;
        const float sl2 = scale * kLog2e;
        float m_used = -INFINITY, l = 0.f;
        for (int j = 0; j < nkv; ++j) {
            const int st = j & 1;
            if (threadIdx.x == 64) ATRACE(j, 0);
            mbar_wait(&s_full[st], (j >> 1) & 1);
            tc_fence_after();
            if (threadIdx.x == 64) ATRACE(j, 1);
            float s[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tmem + lane_base + st * 128 + c * 32, *reinterpret_cast<float(*)[32]>(&s[c * 32]));
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&s_free[st]);
            if (threadIdx.x == 64) ATRACE(j, 2);
            // one warp per SM sub-partition runs this: keep the reductions as 8 independent
            // chains (a single 128-long chain would be latency-bound), scale folded into the exp
            float mx8[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
            // causal mask only on the diagonal tile: a separate (warp-uniform) branch, so the other
            // tiles do not pay a compare + select per element
            if (__builtin_expect(j == nkv - 1, 0)) {
#pragma unroll
                for (int c = 0; c < 128; ++c)
                    if (c > r) s[c] = -INFINITY;
            }
#pragma unroll
            for (int c = 0; c < 128; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
            const float m_new = fmaxf(m_used, mx);
            bool rescale = (j > 0) && (m_new > m_used + 8.f);
            const bool any_rescale = __any_sync(0xffffffff, rescale);
            if (any_rescale) {  // O must be stable: PV_{j-1} done
                mbar_wait(&p_empty[(j - 1) & 1], ((j - 1) >> 1) & 1);
                tc_fence_after();
            }
            if (j >= 2) {  // P buffer j&1 free: PV_{j-2} done
                mbar_wait(&p_empty[j & 1], ((j - 2) >> 1) & 1);
                tc_fence_after();
            }
            if (any_rescale) {
                const float f = rescale ? exp2f(m_used - m_new) : 1.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float o[32];
                    tmem_ld32(tmem + lane_base + 256 + c * 32, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] *= f;
                    tmem_st32(tmem + lane_base + 256 + c * 32, o);
                }
                tmem_st_wait();
                if (rescale) {
                    l *= f;
                    m_used = m_new;
                }
            }
            if (j == 0) m_used = m_new;
            if (threadIdx.x == 64) ATRACE(j, 4);
            float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t pk[32];
#pragma unroll
                for (int e2 = 0; e2 < 32; ++e2) {
                    const int c = h2 * 64 + 2 * e2;
                    const float2 x = __ffma2_rn(make_float2(s[c], s[c + 1]), make_float2(sl2, sl2),
                                                make_float2(-m_used, -m_used));
                    // every other pair on the FMA pipe (poly_exp2x2), see kFwdEmu
                    const float2 pv = (e2 & 1) ? poly_exp2x2(x) : make_float2(fast_exp2(x.x), fast_exp2(x.y));
                    rs8[(2 * e2) & 7] += pv.x;
                    rs8[(2 * e2 + 1) & 7] += pv.y;
                    pk[e2] = pack_bf16(pv.x, pv.y);
                }
                tmem_st32u(tmem + lane_base + 384 + (j & 1) * 64 + h2 * 32, pk);
            }
            l += ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (threadIdx.x == 64) ATRACE(j, 5);
            if (lane_id() == 0) mbar_arrive(&p_full[j & 1]);
        }
        // epilogue: O / l -> bf16
        mbar_wait(o_full, 0);
        tc_fence_after();
        const float inv = 1.f / l;
        __nv_bfloat16* orow = out + size_t(row0 + r) * (H * D) + head * D;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float o[32];
            tmem_ld32(tmem + lane_base + 256 + c * 32, o);
            tmem_ld_wait();
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                dst[e] = make_uint4(pack_bf16(o[8 * e] * inv, o[8 * e + 1] * inv), pack_bf16(o[8 * e + 2] * inv, o[8 * e + 3] * inv),
                                    pack_bf16(o[8 * e + 4] * inv, o[8 * e + 5] * inv), pack_bf16(o[8 * e + 6] * inv, o[8 * e + 7] * inv));
        }
        lse2[size_t(head) * T + row0 + r] = m_used + log2f(l);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_free<512>(tmem);
    }
}


// ------------------------------------------------------------------ backward
// (round 1's full-tile kernel v4 is superseded by v5 below: 6-9 % slower at every measured shape,
// profiles/r2_attn_vs_cudnn.json and DESIGN §4.)
constexpr int kBwdThreads = 384;

__device__ __forceinline__ void bar_sync_compute() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// ------------------------------------------------------------------ backward v5 (half-tile pipeline)
// One CTA per (128-key tile kb, head, sequence), looping over the query rows >= kb (as round 1's v4),
// but the query loop runs in 64-row HALF tiles j with two TMEM buffers, so the tensor pipe computes
// S^T / dP^T of half tile j+1 while the compute warps form P^T / dS^T of half tile j:
//   buffer b = j & 1:  [b*128, +64)  S^T_j  (128 keys x 64 queries); after the elementwise phase each
//                      32-query half h holds P^T bf16 pairs in [32h, 32h+16) and dS^T pairs in [32h+16, 32h+32)
//                      (the TMEM A operands of dV_j and dK_j)
//                      [b*128+64, +64) dP^T_j -> dQ^T_j (fp32, 128 d lanes x 64 queries)
//   [256,384) dV, [384,512) dK accumulators (as v4).
// dS^T_j also goes to shared memory ([key][q], one 128B-swizzled atom) as the B operand (MN-major)
// of dQ^T_j = K^T dS^T_j.  A operands come from TMEM wherever the layout allows: the kernel is bound
// by shared-memory bandwidth (128 B/clk/SM: SS MMAs with N = 64 read 6 KB per 32-cycle K step, plus
// the TMA fills, the dS^T tile and the fp32 dQ staging written and read back by the reduce).
// MMA issue order (one thread, in-order pipe):  S_0 dP_0 S_1 dP_1 | per j: [ds_full_j] dQ^T_j dK_j dV_j
// S_{j+2} [dq_free_j] dP_{j+2}: dQ^T_j first, over the consumed dP^T_j columns, so it can be drained
// while dK_j / dV_j run; S_{j+2} overwrites P^T_j after dV_j read it.
// Compute warps (thread = TMEM lane, column half hf of the 64 queries), per j: E_j (S, dP -> P, dS;
// lse2 / D as smem float4 broadcasts) -> ds_full_j -> read dQ^T_{j-1} (thread = d lane) ->
// dq_free_{j-1} -> stage it fp32 (128B-swizzled [64 q][32 d] chunks, a warp writes one 128 B row per
// store) -> dq_staged -> the reducer warp issues the TMA bulk reduce-add.  Per 64-row half tile the
// MMAs are 5 x 128x64x128-equivalent (~1.3k cycles at full rate); phase stamps
// (tests/trace_attn_bwd.py) put the period at ~2.9k cycles, bounded by the dP_{j+2} -> dQ^T_j drain
// dependency and the per-SM TMA reduce of 32 KB (~1.6k cycles to read out under full-chip load).
constexpr int BQH = 64;
constexpr int kHalf = BQH * D * 2;  // 16 KB: two 128B-swizzled atoms of [64 rows][64]
struct Bwd5Smem {
    static constexpr int k = 0;                 // [128 keys][128 d]: two atoms of 16 KB
    static constexpr int v = k + kTile;
    static constexpr int q = v + kTile;         // [3] half tiles
    static constexpr int dO = q + 3 * kHalf;    // [3]
    static constexpr int ds = dO + 3 * kHalf;   // [2] dS^T_j: [128 keys][64 q] bf16, one atom
    static constexpr int stg = ds + 2 * 16384;  // dQ staging: 4 chunks [64 q][32 d] fp32, 8 KB each
    static constexpr int lse = stg + 32768;     // [2][128] floats: lse2[64] | D[64]
    static constexpr int bars = lse + 1024;  // 36 barriers, the TMEM slot, a 4-entry item ring
    // 512 B of alignment slack: the 227 KB opt-in limit leaves no room for 1 KB; the dynamic window
    // starts 1 KB-aligned when the kernel has no static shared memory (checked at run time)
    static constexpr int total = bars + 384 + 512;
};
static_assert(Bwd5Smem::total <= 232448, "attn bwd v5: shared memory over the sm_100 opt-in limit");

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_tc5_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                        const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dq,
                        const float* __restrict__ lse2, const float* __restrict__ dsum,
                        __nv_bfloat16* __restrict__ dqkv, int seq, int H, int T, float scale,
                        const float* __restrict__ rs, float rs_inv_n, float rs_eps) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    if ((smem_u32(smem_raw) & 1023u) > 512u) __trap();  // alignment slack is 512 B
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Bwd5Smem::bars);
    uint64_t* kv_full = bars + 0;
    uint64_t* q_full = bars + 1;      // [3]
    uint64_t* q_empty = bars + 4;     // [3] MMA commit after dK_g
    uint64_t* do_full = bars + 7;     // [3]
    uint64_t* do_empty = bars + 10;   // [3] MMA commit after dV_g
    uint64_t* s_full = bars + 13;     // [2]
    uint64_t* dp_full = bars + 15;    // [2]
    uint64_t* ds_full = bars + 17;    // [2] 8 compute warps
    uint64_t* dq_full = bars + 19;    // [2]
    uint64_t* dq_free = bars + 21;    // [2] 8 compute warps
    uint64_t* stg_free = bars + 23;   // reducer: staging read out
    uint64_t* dq_staged = bars + 24;  // 8 compute warps
    uint64_t* dkv_full = bars + 25;   // MMA commit after an item's last dV
    uint64_t* kv_empty = bars + 26;   // (same commit) the item's K / V no longer read
    uint64_t* dkv_free = bars + 27;   // 8 compute warps: the item's dK / dV read out of TMEM
    uint64_t* item_full = bars + 28;  // [4] loader: the item index of ring slot k is published
    uint64_t* item_empty = bars + 32; // [4] the 11 consumer warps have read it
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 36);
    int* item_ring = reinterpret_cast<int*>(bars + 37);  // [4]
    float* sL = reinterpret_cast<float*>(sm + Bwd5Smem::lse);

    const uint32_t warp = warp_id();
    const int nqb = seq / BQ;
    const int HB = H * (T / seq);     // (head, sequence) pairs
    const int NI = nqb * HB;          // items: (128-key tile kb, head, sequence), heaviest kb first
    // Persistent CTAs with dynamic (greedy, heaviest-first) items: the loader warp takes the next item
    // index from a global counter (attn_bwd_pre zeroes it; the first item is blockIdx.x) and publishes it
    // in a 4-entry shared ring; every other warp reads the ring in the same order.  Half tiles are
    // numbered globally (g) across a CTA's items: ring slots, TMEM buffers and barrier phases follow g.
    int* work = reinterpret_cast<int*>(const_cast<float*>(dsum) + size_t(H) * T);
    auto next_item = [&](int k, bool whole_warp) {  // consumer warps: one arrival per warp
        mbar_wait(&item_full[k & 3], (k >> 2) & 1);
        const int idx = *reinterpret_cast<volatile int*>(&item_ring[k & 3]);
        if (whole_warp) __syncwarp();
        if (!whole_warp || lane_id() == 0) mbar_arrive(&item_empty[k & 3]);
        return idx;
    };

    if (warp == 0 && elect_one()) {
        tma_prefetch(&tm_kv);
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        tma_prefetch(&tm_dq);
        for (int i = 0; i < 36; ++i) {
            const bool eight = (i >= 17 && i < 19) || (i >= 21 && i < 23) || i == 24 || i == 27;
            mbar_init(&bars[i], i >= 32 ? 11 : (eight ? 8 : 1));
        }
        fence_barrier_init();
    }
    pdl_wait();
    pdl_launch();
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= 10) {
        if (warp == 10 && lane_id() == 0) {
            // dQ reducer: four 8 KB TMA bulk reduce-adds per half tile
            int u = 0;
            for (int r = 0;; ++r) {
                const int idx = next_item(r, false);
                if (idx >= NI) break;
                const int kb = idx / HB, hb = idx % HB, head = hb % H;
                const int qrow0 = (hb / H) * seq + kb * BQ, n = 2 * (nqb - kb);
                for (int j = 0; j < n; ++j, ++u) {
                    mbar_wait(dq_staged, u & 1);
                    ATRACE(u, 6);
                    const int row = qrow0 + j * BQH;
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc)
                        asm volatile(
                            "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                reinterpret_cast<uint64_t>(&tm_dq)),
                            "r"(smem_u32(sm + Bwd5Smem::stg + cc * 8192)), "r"(head * D + cc * 32), "r"(row)
                            : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    ATRACE(u, 7);
                    mbar_arrive(stg_free);
                }
            }
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
        if (warp == 11 && lane_id() == 0) {
            int g = 0;
            for (int r = 0;; ++r) {
                const int idx = next_item(r, false);
                if (idx >= NI) break;
                const int kb = idx / HB, hb = idx % HB, head = hb % H;
                const int qrow0 = (hb / H) * seq + kb * BQ, n = 2 * (nqb - kb);
                for (int j = 0; j < n; ++j, ++g) {
                    const int st = g % 3;
                    if (g >= 3) mbar_wait(&do_empty[st], ((g / 3) - 1) & 1);
                    uint8_t* dst = sm + Bwd5Smem::dO + st * kHalf;
                    mbar_expect_tx(&do_full[st], kHalf);
                    tma_load_2d(dst, &tm_do, &do_full[st], head * D, qrow0 + j * BQH);
                    tma_load_2d(dst + 8192, &tm_do, &do_full[st], head * D + 64, qrow0 + j * BQH);
                }
            }
        }
    } else if (warp == 0) {
        if (lane_id() == 0) {
            int g = 0;
            for (int r = 0;; ++r) {
                const int idx = r == 0 ? int(blockIdx.x) : int(gridDim.x) + atomicAdd(work, 1);
                if (r >= 4) mbar_wait(&item_empty[r & 3], ((r >> 2) - 1) & 1);
                item_ring[r & 3] = idx < NI ? idx : NI;  // NI: no more work
                mbar_arrive(&item_full[r & 3]);
                if (idx >= NI) break;
                const int kb = idx / HB, hb = idx % HB, head = hb % H;
                const int tok0 = (hb / H) * seq, qrow0 = tok0 + kb * BQ, n = 2 * (nqb - kb);
                const int ck = H * D + head * D, cv = 2 * H * D + head * D;
                const int kr = tok0 + kb * BK;
                if (r > 0) mbar_wait(kv_empty, (r - 1) & 1);  // the previous item's MMAs are done with K / V
                mbar_expect_tx(kv_full, 2 * kTile);
                tma_load_2d(sm + Bwd5Smem::k, &tm_kv, kv_full, ck, kr);
                tma_load_2d(sm + Bwd5Smem::k + 16384, &tm_kv, kv_full, ck + 64, kr);
                tma_load_2d(sm + Bwd5Smem::v, &tm_kv, kv_full, cv, kr);
                tma_load_2d(sm + Bwd5Smem::v + 16384, &tm_kv, kv_full, cv + 64, kr);
                for (int j = 0; j < n; ++j, ++g) {
                    const int st = g % 3;
                    if (g >= 3) mbar_wait(&q_empty[st], ((g / 3) - 1) & 1);
                    ATRACE(g, 11);
                    uint8_t* dst = sm + Bwd5Smem::q + st * kHalf;
                    mbar_expect_tx(&q_full[st], kHalf);
                    tma_load_2d(dst, &tm_q, &q_full[st], head * D, qrow0 + j * BQH);
                    tma_load_2d(dst + 8192, &tm_q, &q_full[st], head * D + 64, qrow0 + j * BQH);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t id_sd = idesc_bf16(128, 64, false, false);   // S^T, dP^T: K-major x K-major
        constexpr uint32_t id_kv = idesc_bf16(128, 128, false, true);   // dK, dV: A from TMEM, B MN-major
        constexpr uint32_t id_dq = idesc_bf16(128, 64, true, true);     // dQ^T = K^T dS^T: both MN-major
        const uint32_t sk = smem_u32(sm + Bwd5Smem::k), sv = smem_u32(sm + Bwd5Smem::v);
        auto issue_sd = [&](int g, bool dp) {  // S^T_g = K Q_g^T or dP^T_g = V dO_g^T
            const int st = g % 3;
            uint64_t* full = dp ? &do_full[st] : &q_full[st];
            const uint32_t sb = smem_u32(sm + (dp ? Bwd5Smem::dO : Bwd5Smem::q) + st * kHalf);
            const uint32_t sa = dp ? sv : sk;
            if (dp && g >= 2) {  // dP^T_g lands over dQ^T_{g-2}: wait until it is read out of TMEM
                mbar_wait(&dq_free[g & 1], ((g - 2) >> 1) & 1);
                if (lane_id() == 0) ATRACE(g - 2, 10);
            }
            mbar_wait(full, (g / 3) & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    tc_mma(tmem + (g & 1) * 128 + (dp ? 64 : 0), sdesc(sa + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                           sdesc(sb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), id_sd, kk != 0);
                tc_commit(dp ? &dp_full[g & 1] : &s_full[g & 1]);
            }
            __syncwarp();
        };
        int g = 0;
        for (int r = 0;; ++r) {
            const int idx = next_item(r, true);
            if (idx >= NI) break;
            const int kb = idx / HB, n = 2 * (nqb - kb);
            mbar_wait(kv_full, r & 1);
            tc_fence_after();
            issue_sd(g, false);
            issue_sd(g, true);
            issue_sd(g + 1, false);
            issue_sd(g + 1, true);
            for (int j = 0; j < n; ++j) {
                const int gg = g + j, bb = gg & 1, st = gg % 3;
                const uint32_t sq = smem_u32(sm + Bwd5Smem::q + st * kHalf);
                const uint32_t sdo = smem_u32(sm + Bwd5Smem::dO + st * kHalf);
                const uint32_t sds = smem_u32(sm + Bwd5Smem::ds + bb * 16384);
                mbar_wait(&ds_full[bb], (gg >> 1) & 1);
                if (j == 0 && r > 0) mbar_wait(dkv_free, (r - 1) & 1);  // previous item's dK / dV read out
                tc_fence_after();
                if (lane_id() == 0) ATRACE(gg, 8);
                if (elect_one()) {
                    // dQ^T_g = K^T dS^T_g over the consumed dP^T_g columns: first, so the compute warps can
                    // drain it while dK_g / dV_g run
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        tc_mma(tmem + bb * 128 + 64, sdesc(sk + kk * 2048, 16384, 1024),
                               sdesc(sds + kk * 2048, 8192, 1024), id_dq, kk != 0);
                    tc_commit(&dq_full[bb]);
                    // dK += dS^T_g Q_g (A = dS^T bf16 pairs in the S^T_g columns [16,32) / [48,64); K = 64)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        tc_mma_ts(tmem + 384, tmem + bb * 128 + (kk >> 1) * 32 + 16 + (kk & 1) * 8,
                                  sdesc(sq + kk * 2048, 8192, 1024), id_kv, (j | kk) != 0);
                    tc_commit(&q_empty[st]);
                    // dV += P^T_g dO_g (A = P^T bf16 pairs in TMEM)
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        tc_mma_ts(tmem + 256, tmem + bb * 128 + (kk >> 1) * 32 + (kk & 1) * 8,
                                  sdesc(sdo + kk * 2048, 8192, 1024), id_kv, (j | kk) != 0);
                    tc_commit(&do_empty[st]);
                    if (j == n - 1) {
                        tc_commit(dkv_full);
                        tc_commit(kv_empty);
                    }
                }
                __syncwarp();
                if (j + 2 < n) {
                    issue_sd(gg + 2, false);  // over P^T_g, after dV_g read it (in-order pipe)
                    issue_sd(gg + 2, true);
                }
            }
            g += n;
        }
    } else {
        const uint32_t q4 = warp & 3;
        const int hf = int(warp - 2) >> 2;  // query column half (32 of the 64) handled by this warp
        const int r = int(q4 * 32 + lane_id());
        const uint32_t lane_base = (q4 * 32) << 16;
        const float sl2 = scale * kLog2e;
        const int key = r;  // key row relative to the tile (queries relative to qrow0 below)
        auto drain_dq = [&](int u) {  // dQ^T_u: TMEM -> registers -> release -> fp32 staging
            const int pb = u & 1;
            mbar_wait(&dq_full[pb], (u >> 1) & 1);
            tc_fence_after();
            if (threadIdx.x == 64) ATRACE(u, 3);
            float v[32];
            tmem_ld32(tmem + lane_base + pb * 128 + 64 + hf * 32, v);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&dq_free[pb]);
            if (u >= 1) mbar_wait(stg_free, (u - 1) & 1);
            if (threadIdx.x == 64) ATRACE(u, 4);
            // thread = d row r (chunk q4 = r / 32, lane = r % 32), 32 query rows hf*32 + c
            uint8_t* chunk = sm + Bwd5Smem::stg + q4 * 8192;
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
                const int qq = hf * 32 + cc;
                *reinterpret_cast<float*>(chunk + qq * 128 + (((lane_id() >> 2) ^ (qq & 7)) << 4) + (lane_id() & 3) * 4) = v[cc];
            }
            fence_async_smem();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(dq_staged);
            if (threadIdx.x == 64) ATRACE(u, 5);
        };
        int g = 0;
        for (int ri = 0;; ++ri) {
            const int idx = next_item(ri, true);
            if (idx >= NI) break;
            const int kb = idx / HB, hb = idx % HB, head = hb % H;
            const int tok0 = (hb / H) * seq, qrow0 = tok0 + kb * BQ, n = 2 * (nqb - kb);
            auto lse_of = [&](int j) {  // staged value of this thread (r < 64): lse2 (hf 0) or D (hf 1)
                const size_t i2 = size_t(head) * T + qrow0 + j * BQH + (r & 63);
                return hf == 0 ? lse2[i2] : dsum[i2];
            };
            if (r < 64) sL[(g & 1) * 128 + hf * 64 + r] = lse_of(0);
            bar_sync_compute();
            for (int j = 0; j < n; ++j) {
                const int gg = g + j, bb = gg & 1;
                const float* Lb = sL + bb * 128;
                const float lnext = (j + 1 < n && r < 64) ? lse_of(j + 1) : 0.f;
                if (threadIdx.x == 64) ATRACE(gg, 0);
                mbar_wait(&s_full[bb], (gg >> 1) & 1);
                if (threadIdx.x == 64) ATRACE(gg, 12);
                mbar_wait(&dp_full[bb], (gg >> 1) & 1);
                tc_fence_after();
                if (threadIdx.x == 64) ATRACE(gg, 1);
                const int c0 = hf * 32;
                {
                    float sv[32], dp[32];
                    tmem_ld32(tmem + lane_base + bb * 128 + c0, sv);
                    tmem_ld32(tmem + lane_base + bb * 128 + 64 + c0, dp);
                    tmem_ld_wait();
                    if (threadIdx.x == 64) ATRACE(gg, 13);
                    if (__builtin_expect(j < 2, 0)) {  // causal mask: the two half tiles of the diagonal block
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (key > j * BQH + c0 + e) sv[e] = -INFINITY;
                    }
                    // lse2 / D of this half's 32 query columns: the same for every lane (smem broadcast),
                    // loaded as float4 so the 32 independent exp2 chains issue back to back
                    const float4* l4 = reinterpret_cast<const float4*>(Lb + c0);
                    const float4* d4 = reinterpret_cast<const float4*>(Lb + 64 + c0);
                    uint32_t pk[16], dk[16];
#pragma unroll
                    for (int e4 = 0; e4 < 8; ++e4) {
                        const float4 lq = l4[e4], dq = d4[e4];
                        const float lz[4] = {lq.x, lq.y, lq.z, lq.w}, dz[4] = {dq.x, dq.y, dq.z, dq.w};
                        // packed f32x2 FMA / ADD / MUL (FFMA2 & co. on sm_100): half the issue slots
#pragma unroll
                        for (int u = 0; u < 4; u += 2) {
                            const float2 x = __ffma2_rn(make_float2(sv[4 * e4 + u], sv[4 * e4 + u + 1]),
                                                        make_float2(sl2, sl2), make_float2(-lz[u], -lz[u + 1]));
                            const float2 pv = make_float2(fast_exp2(x.x), fast_exp2(x.y));
                            const float2 dd = __fadd2_rn(make_float2(dp[4 * e4 + u], dp[4 * e4 + u + 1]),
                                                         make_float2(-dz[u], -dz[u + 1]));
                            const float2 dsv = __fmul2_rn(pv, dd);
                            pk[2 * e4 + (u >> 1)] = pack_bf16(pv.x, pv.y);
                            dk[2 * e4 + (u >> 1)] = pack_bf16(dsv.x, dsv.y);
                        }
                    }
                    if (threadIdx.x == 64) ATRACE(gg, 14);
                    tmem_st16u(tmem + lane_base + bb * 128 + c0, pk);
                    tmem_st16u(tmem + lane_base + bb * 128 + c0 + 16, dk);
                    // dS^T_g to smem ([key][q], 128B-swizzled, one atom): B operand (MN-major) of dQ^T_g.
                    // Its last readers, dQ^T_{g-2} and dK_{g-2}, precede S_g in the MMA pipe, so s_full_g
                    // (waited above) covers them.
                    uint8_t* sds = sm + Bwd5Smem::ds + bb * 16384;
#pragma unroll
                    for (int e8 = 0; e8 < 4; ++e8)
                        *reinterpret_cast<uint4*>(sds + r * 128 + ((((c0 >> 3) + e8) ^ (r & 7)) << 4)) =
                            make_uint4(dk[4 * e8], dk[4 * e8 + 1], dk[4 * e8 + 2], dk[4 * e8 + 3]);
                }
                tmem_st_wait();
                if (threadIdx.x == 64) ATRACE(gg, 15);
                fence_async_smem();
                tc_fence_before();
                __syncwarp();
                if (lane_id() == 0) mbar_arrive(&ds_full[bb]);
                if (threadIdx.x == 64) ATRACE(gg, 2);
                if (j >= 1) drain_dq(gg - 1);
                if (j + 1 < n) {
                    if (r < 64) sL[((gg + 1) & 1) * 128 + hf * 64 + r] = lnext;  // buffer last read by E_{g-1}
                    bar_sync_compute();
                }
            }
            drain_dq(g + n - 1);
            // dV, dK rows (thread = key row, column half hf); then the columns go to the next item
            mbar_wait(dkv_full, ri & 1);
            tc_fence_after();
            const size_t rowoff = size_t(tok0 + kb * BK + r) * (3 * H * D);
            // folded RMSNorm of the QKV input: dqkv' = rstd1(row) * dqkv (executor.cpp, fold mode)
            const float fv = rs ? rsqrtf(rs[tok0 + kb * BK + r] * rs_inv_n + rs_eps) : 1.f;
            const float fk = fv * scale;
#pragma unroll 1
            for (int cc = 0; cc < 2; ++cc) {
                const int cq = hf * 2 + cc;
                float v[32], k[32];
                tmem_ld32(tmem + lane_base + 256 + cq * 32, v);
                tmem_ld32(tmem + lane_base + 384 + cq * 32, k);
                tmem_ld_wait();
                uint4* dv = reinterpret_cast<uint4*>(dqkv + rowoff + 2 * H * D + head * D + cq * 32);
                uint4* dkp = reinterpret_cast<uint4*>(dqkv + rowoff + H * D + head * D + cq * 32);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    dv[e] = make_uint4(pack_bf16(v[8 * e] * fv, v[8 * e + 1] * fv), pack_bf16(v[8 * e + 2] * fv, v[8 * e + 3] * fv),
                                       pack_bf16(v[8 * e + 4] * fv, v[8 * e + 5] * fv), pack_bf16(v[8 * e + 6] * fv, v[8 * e + 7] * fv));
                    dkp[e] = make_uint4(pack_bf16(k[8 * e] * fk, k[8 * e + 1] * fk),
                                        pack_bf16(k[8 * e + 2] * fk, k[8 * e + 3] * fk),
                                        pack_bf16(k[8 * e + 4] * fk, k[8 * e + 5] * fk),
                                        pack_bf16(k[8 * e + 6] * fk, k[8 * e + 7] * fk));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(dkv_free);
            g += n;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_free<512>(tmem);
    }
}

// ------------------------------------------------------------------ forward v3 (two CTAs per SM)
// Single-buffered per CTA so that TWO CTAs fit on an SM (96 KB smem: Q, K, V; 256 TMEM columns:
// S / P at [0,128), O at [128,256)): while one CTA runs its softmax the other CTA's S / PV MMAs
// keep the tensor pipe busy, and one CTA's prologue / epilogue hides under the other's main loop.
// Per CTA and key tile j:  S(j) = Q K(j)^T -> softmax (thread = query row; P written back over S as
// bf16 pairs) -> O += P(j) V(j) (A = P from TMEM).  The MMA pipe runs in issue order, so S(j+1)
// overwrites P(j) only after PV(j) has read it, and when s_full(j) completes PV(j-1) has too (the
// lazy O rescale needs no extra wait).  The softmax reads S from TMEM once (128 scores per thread in
// registers: 166 registers, under the 168 that two CTAs / SM allow) and applies the O rescale after
// P is written, when the scores' registers are free.
struct Fwd3Smem {
    static constexpr int q = 0;
    static constexpr int k = kTile;
    static constexpr int v = 2 * kTile;
    static constexpr int bars = 3 * kTile;
    static constexpr int total = bars + 128 + 1024;
};

// Exponentials: kFwdEmu of every 16 pairs go to the FMA pipe (poly_exp2x2), the rest to the SFU,
// whose 16 ex2 / clk / SM otherwise match the tensor pipe's S + PV time per tile exactly.
// Measured (tests/bench_attn.py), two-pass softmax: 0 / 4 / 6 / 8 of 16 -> 68.3 / 73.4 / 66.8 / 66.2 us at
// 2x2048x16, 160.5 / 163.7 / 153.8 / 154.1 us at 4096x32, 468 / 467 / 458 / 460 us at 6144x48; with the
// single-read softmax: 4 / 6 / 8 / 10 / 12 of 16 -> 62.7 / 62.4 / 62.5 / 66.8 / 68.9 us, 147.7 / 148.1 /
// 149.8 / 158.0 / 173.1 us, 449 / 451 / 460 / 474 / 515 us.
constexpr int kFwdEmu = 4;

__global__ void __launch_bounds__(192, 2)
    attn_fwd_tc3_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
                        float* __restrict__ lse2, int seq, int H, int T, float scale) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared-space pointer
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Fwd3Smem::bars);
    uint64_t* q_full = bars + 0;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = bars + 2;  // MMA commit after S(j)
    uint64_t* v_full = bars + 3;
    uint64_t* v_empty = bars + 4;  // MMA commit after PV(j)
    uint64_t* s_full = bars + 5;   // MMA commit after S(j)
    uint64_t* p_full = bars + 6;   // 4 softmax warps: P(j) in TMEM
    uint64_t* o_full = bars + 7;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

    const uint32_t warp = warp_id();
    const int nqb = seq / BQ;
    const int hb = int(blockIdx.x) % (H * (T / seq));
    const int qb = nqb - 1 - int(blockIdx.x) / (H * (T / seq));  // heaviest causal tile first (LPT)
    const int head = hb % H, b = hb / H;
    const int row0 = b * seq + qb * BQ;
    const int nkv = qb + 1;

    if (warp == 0 && elect_one()) {
        tma_prefetch(&tm);
        for (int i = 0; i < 8; ++i) mbar_init(&bars[i], i == 6 ? 4 : 1);
        fence_barrier_init();
    }
    // TMEM is allocated only once the previous kernel in the stream has finished: a CTA that
    // launched early (PDL) never holds TMEM while it waits (see gemm_tc.cu)
    pdl_wait();
    pdl_launch();
    if (warp == 1) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elect_one()) {
            const int cq = head * D, ck = H * D + head * D, cv = 2 * H * D + head * D;
            mbar_expect_tx(q_full, kTile);
            tma_load_2d(sm + Fwd3Smem::q, &tm, q_full, cq, row0);
            tma_load_2d(sm + Fwd3Smem::q + 16384, &tm, q_full, cq + 64, row0);
            for (int j = 0; j < nkv; ++j) {
                const int kr = b * seq + j * BK;
                if (j > 0) mbar_wait(k_empty, (j - 1) & 1);
                mbar_expect_tx(k_full, kTile);
                tma_load_2d(sm + Fwd3Smem::k, &tm, k_full, ck, kr);
                tma_load_2d(sm + Fwd3Smem::k + 16384, &tm, k_full, ck + 64, kr);
                if (j > 0) mbar_wait(v_empty, (j - 1) & 1);
                mbar_expect_tx(v_full, kTile);
                tma_load_2d(sm + Fwd3Smem::v, &tm, v_full, cv, kr);
                tma_load_2d(sm + Fwd3Smem::v + 16384, &tm, v_full, cv + 64, kr);
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc_s = idesc_bf16(128, 128, false, false);
        constexpr uint32_t idesc_o = idesc_bf16(128, 128, false, true);
        const uint32_t sq = smem_u32(sm + Fwd3Smem::q), sk = smem_u32(sm + Fwd3Smem::k);
        const uint32_t sv = smem_u32(sm + Fwd3Smem::v);
        mbar_wait(q_full, 0);
        for (int j = 0; j < nkv; ++j) {
            mbar_wait(k_full, j & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32;
                    tc_mma(tmem, sdesc(sq + o, 16, 1024), sdesc(sk + o, 16, 1024), idesc_s, kk != 0);
                }
                tc_commit(s_full);
                tc_commit(k_empty);
            }
            __syncwarp();
            mbar_wait(p_full, j & 1);
            mbar_wait(v_full, j & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    tc_mma_ts(tmem + 128, tmem + kk * 8, sdesc(sv + kk * 2048, 16384, 1024), idesc_o, (j | kk) != 0);
                tc_commit(v_empty);
            }
            __syncwarp();
        }
        if (elect_one()) tc_commit(o_full);
        __syncwarp();
    } else {
        const uint32_t q4 = warp & 3;
        const int r = int(q4 * 32 + lane_id());  // query row in tile == TMEM lane
        const uint32_t lane_base = (q4 * 32) << 16;
        const float sl2 = scale * kLog2e;
        float m_used = -INFINITY, l = 0.f;
        for (int j = 0; j < nkv; ++j) {
            mbar_wait(s_full, j & 1);
            tc_fence_after();
            const bool diag = j == nkv - 1;
            // S read from TMEM once (all 128 columns in flight, one wait); row max and P from registers
            float s[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tmem + lane_base + c * 32, s[c]);
            tmem_ld_wait();  // every S column is in registers before P overwrites [0,64)
            if (__builtin_expect(diag, 0)) {
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (c * 32 + e > r) s[c][e] = -INFINITY;
            }
            float mx8[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int e = 0; e < 32; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], s[c][e]);
            const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
            const float m_new = fmaxf(m_used, mx);
            const bool rescale = (j > 0) && (m_new > m_used + 8.f);
            // lazy O rescale: decided here, applied to O after P is written (O is stable until
            // p_full(j): s_full(j) implies PV(j-1) retired), so S's registers are dead by then
            const float f = rescale ? exp2f(m_used - m_new) : 1.f;
            if (rescale || j == 0) {
                l *= f;
                m_used = m_new;
            }
            // P = exp2(S*c - m) -> bf16 pairs over the consumed S columns [0,64)
            float2 rs4[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int e2 = 0; e2 < 16; ++e2) {  // packed f32x2 FMA / ADD (FFMA2, FADD2)
                    const float2 x = __ffma2_rn(make_float2(s[c][2 * e2], s[c][2 * e2 + 1]), make_float2(sl2, sl2),
                                                make_float2(-m_used, -m_used));
                    // Bresenham spread: kFwdEmu of the 16 pairs, evenly interleaved with the SFU pairs
                    const bool emu = (e2 * kFwdEmu) / 16 != ((e2 + 1) * kFwdEmu) / 16;
                    const float2 pv = emu ? poly_exp2x2(x) : make_float2(fast_exp2(x.x), fast_exp2(x.y));
                    rs4[e2 & 3] = __fadd2_rn(rs4[e2 & 3], pv);
                    pk[e2] = pack_bf16(pv.x, pv.y);
                }
                tmem_st16u(tmem + lane_base + c * 16, pk);
            }
            l += ((rs4[0].x + rs4[1].x) + (rs4[2].x + rs4[3].x)) + ((rs4[0].y + rs4[1].y) + (rs4[2].y + rs4[3].y));
            if (__any_sync(0xffffffff, rescale)) {
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    float o[32];
                    tmem_ld32(tmem + lane_base + 128 + c * 32, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e) o[e] *= f;
                    tmem_st32(tmem + lane_base + 128 + c * 32, o);
                }
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(p_full);
        }
        mbar_wait(o_full, 0);
        tc_fence_after();
        const float inv = 1.f / l;
        __nv_bfloat16* orow = out + size_t(row0 + r) * (H * D) + head * D;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float o[32];
            tmem_ld32(tmem + lane_base + 128 + c * 32, o);
            tmem_ld_wait();
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                dst[e] = make_uint4(pack_bf16(o[8 * e] * inv, o[8 * e + 1] * inv), pack_bf16(o[8 * e + 2] * inv, o[8 * e + 3] * inv),
                                    pack_bf16(o[8 * e + 4] * inv, o[8 * e + 5] * inv), pack_bf16(o[8 * e + 6] * inv, o[8 * e + 7] * inv));
        }
        lse2[size_t(head) * T + row0 + r] = m_used + log2f(l);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_free<256>(tmem);
    }
}


}  // namespace

// Phase-stamp buffer of block 0 (PB_ATTN_TRACE / PB_ATTN_TRACE_FWD with a -DPB_ATTN_TRACE_BUILD library)
static unsigned long long* trace_buffer(const char* env) {
    unsigned long long* t = nullptr;
    if (std::getenv(env)) {
        cudaMalloc(&t, 32 * 16 * 8);
        cudaMemset(t, 0, 32 * 16 * 8);
        cudaMemcpyToSymbol(g_attn_trace, &t, sizeof(t));
    }
    return t;
}
static void trace_dump(unsigned long long* t, const char* what, cudaStream_t s) {
    if (!t) return;
    unsigned long long h[32 * 16];
    cudaStreamSynchronize(s);
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 32 && h[i * 16 + 0]; ++i) {
        std::fprintf(stderr, "%s trace it %2d: t0=%lld", what, i, (long long)(h[i * 16] - h[0]));
        for (int e = 1; e < 16; ++e)
            if (h[i * 16 + e]) std::fprintf(stderr, " e%d=%lld", e, (long long)(h[i * 16 + e] - h[i * 16 + 0]));
        std::fprintf(stderr, "\n");
    }
}

void attn_bwd_pre(const __nv_bfloat16* dout, const __nv_bfloat16* out, float* dsum, float* dq_acc, int heads, int T,
                  cudaStream_t s) {
    launch_k(attn_bwd_pre_kernel, dim3(T), dim3(256), 0, s, 1, dout, out, dsum, dq_acc, heads, T);
}

void attn_dq_store(const float* dq_acc, __nv_bfloat16* dqkv, int heads, int T, cudaStream_t s, const float* rs,
                   float rs_inv_n, float rs_eps) {
    launch_k(attn_dq_store_kernel, dim3(T), dim3(256), 0, s, 1, dq_acc, dqkv, heads, 0.08838834764831845f, rs,
             rs_inv_n, rs_eps);
}

void attn_bwd_tc(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout, const float* lse2,
                 float* dsum, float* dq_acc, __nv_bfloat16* dqkv, int batch, int seq, int heads, cudaStream_t s,
                 const float* rs, float rs_inv_n, float rs_eps) {
    if (seq % 128) throw std::invalid_argument("attention: seq must be a multiple of 128");
    attn_bwd_pre(dout, out, dsum, dq_acc, heads, batch * seq, s);
    static bool once = [] {
        cudaFuncSetAttribute(attn_bwd_tc5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Bwd5Smem::total);
        return true;
    }();
    (void)once;
    const int T = batch * seq;
    const CUtensorMap tq = make_map(qkv, uint64_t(3) * heads * D, uint64_t(T), uint64_t(3) * heads * D, 64, 128);
    const CUtensorMap tq64 = make_map(qkv, uint64_t(3) * heads * D, uint64_t(T), uint64_t(3) * heads * D, 64, 64);
    const CUtensorMap td64 = make_map(dout, uint64_t(heads) * D, uint64_t(T), uint64_t(heads) * D, 64, 64);
    const CUtensorMap tdq = make_map_t(dq_acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, uint64_t(heads) * D, uint64_t(T),
                                       uint64_t(heads) * D, 32, 64);
    static unsigned long long* trace = trace_buffer("PB_ATTN_TRACE");
    const int items = seq / BK * heads * batch;  // persistent: one CTA per SM walks the items
    launch_k(attn_bwd_tc5_kernel, dim3(items < num_sms() ? items : num_sms()), dim3(kBwdThreads), Bwd5Smem::total, s, 1,
             tq, tq64,
             td64, tdq, lse2, static_cast<const float*>(dsum), dqkv, seq, heads, T, 0.08838834764831845f, rs, rs_inv_n,
             rs_eps);
    trace_dump(trace, "attn_bwd", s);
    attn_dq_store(dq_acc, dqkv, heads, T, s, rs, rs_inv_n, rs_eps);
}

// Two forward kernels, same contract: the single-CTA-per-SM kernel with double-buffered S / P
// (attn_fwd_tc_kernel, lowest per-tile latency: small grids) and the two-CTAs-per-SM kernel
// (attn_fwd_tc3_kernel: one CTA's MMAs run under the other's softmax) for grids of >= ~3 CTAs per
// SM.  PB_ATTN_FWD=1 / 3 forces one.
void attn_fwd_tc(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse2, int batch, int seq, int heads,
                 cudaStream_t s) {
    if (seq % 128) throw std::invalid_argument("attention: seq must be a multiple of 128");
    static bool once = [] {
        cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdSmem::total);
        cudaFuncSetAttribute(attn_fwd_tc3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd3Smem::total);
        return true;
    }();
    (void)once;
    const int T = batch * seq;
    const CUtensorMap tm = make_map(qkv, uint64_t(3) * heads * D, uint64_t(T), uint64_t(3) * heads * D, 64, 128);
    static const int fenv = [] {
        const char* e = std::getenv("PB_ATTN_FWD");
        return e && (e[0] == '1' || e[0] == '3') ? e[0] - '0' : 0;
    }();
    const int nblk = seq / BQ * heads * batch;
    const int fver = fenv ? fenv : (nblk >= 3 * num_sms() ? 3 : 1);
    if (fver == 3) {
        launch_k(attn_fwd_tc3_kernel, dim3(nblk), dim3(192), Fwd3Smem::total, s, 1, tm, out, lse2, seq, heads, T,
                 0.08838834764831845f);
    } else {
        static unsigned long long* trace = trace_buffer("PB_ATTN_TRACE_FWD");
        launch_k(attn_fwd_tc_kernel, dim3(nblk), dim3(192), FwdSmem::total, s, 1, tm, out, lse2, seq, heads, T,
                 0.08838834764831845f);
        trace_dump(trace, "attn_fwd", s);
    }
}

}  // namespace pbk
