// Causal multi-head attention, head_dim 128, fused forward (online softmax,
// log-sum-exp saved) and backward (dQ/dK/dV), flash-attention-2 dataflow.
//
// Layout: qkv [T, 3h] bf16 row-major (q | k | v, head j at columns j*128),
// T = micro_batch * seq tokens, sequences contiguous; o [T, h]; lse2 [H, T]
// fp32 (base-2 log-sum-exp of the scaled scores).
//
// Round-1 implementation on warp-level mma.sync (m16n8k16 bf16, fp32 acc)
// with ldmatrix from XOR-swizzled smem and cp.async double buffering.
#include <stdexcept>

#include "ops.hpp"
#include "sm100.cuh"

namespace pbk {
namespace {

constexpr int D = 128;   // head dim
constexpr int BQ = 64;   // query rows per tile
constexpr int BKV = 64;  // key rows per tile
constexpr float kLog2e = 1.4426950408889634f;

// byte offset of (row, col) in a [rows][128] bf16 tile, 16B chunks XOR-swizzled by row
__device__ __forceinline__ uint32_t swz(int row, int col) {
    return uint32_t(row * 256 + ((((col >> 3) ^ (row & 7))) << 4) + (col & 7) * 2);
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// load a [64][128] bf16 tile (row stride ld elements) into swizzled smem; 128 threads
__device__ __forceinline__ void load_tile(uint32_t sbase, const __nv_bfloat16* g, int ld, int tid) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        int idx = tid + i * 128;  // 1024 chunks of 16B
        int row = idx >> 4, ch = idx & 15;
        cp_async16(sbase + swz(row, ch * 8), g + size_t(row) * ld + ch * 8);
    }
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A fragment (16 rows x 16 k) from a row-major swizzled tile at (r0, k0)
__device__ __forceinline__ void frag_a(uint32_t base, int r0, int k0, int lane, uint32_t (&a)[4]) {
    int row = r0 + (lane & 7) + ((lane >> 3) & 1) * 8;
    int col = k0 + (lane >> 4) * 8;
    ldsm_x4(base + swz(row, col), a[0], a[1], a[2], a[3]);
}
// A fragment from a tile stored transposed ([k][m], m contiguous): rows of A = columns of the tile
__device__ __forceinline__ void frag_a_t(uint32_t base, int r0, int k0, int lane, uint32_t (&a)[4]) {
    // matrices: (m 0-7,k 0-7), (m 8-15,k 0-7), (m 0-7,k 8-15), (m 8-15,k 8-15); tile row = k
    int krow = k0 + (lane & 7) + (lane >> 4) * 8;
    int mcol = r0 + ((lane >> 3) & 1) * 8;
    ldsm_x4_t(base + swz(krow, mcol), a[0], a[1], a[2], a[3]);
}
// B fragments for two n-tiles (n0..n0+15) x k16, tile stored [n][k] (k contiguous)
__device__ __forceinline__ void frag_b_nk(uint32_t base, int n0, int k0, int lane, uint32_t (&b)[4]) {
    int row = n0 + (lane & 7) + (lane >> 4) * 8;
    int col = k0 + ((lane >> 3) & 1) * 8;
    ldsm_x4(base + swz(row, col), b[0], b[1], b[2], b[3]);  // b0,b1 -> ntile n0; b2,b3 -> n0+8
}
// B fragments for two n-tiles x k16, tile stored [k][n] (n contiguous)
__device__ __forceinline__ void frag_b_kn(uint32_t base, int n0, int k0, int lane, uint32_t (&b)[4]) {
    int row = k0 + (lane & 7) + ((lane >> 3) & 1) * 8;
    int col = n0 + (lane >> 4) * 8;
    ldsm_x4_t(base + swz(row, col), b[0], b[1], b[2], b[3]);
}

// ------------------------------------------------------------------ forward
__global__ void __launch_bounds__(128, 2)
    attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out, float* __restrict__ lse2,
                    int seq, int H, int T, float scale) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nqb = seq / BQ;
    const int qb = nqb - 1 - blockIdx.x;  // heaviest tiles first
    const int head = blockIdx.y, b = blockIdx.z;
    const int ld = 3 * H * D;
    const size_t tok0 = size_t(b) * seq;
    const __nv_bfloat16* Qg = qkv + (tok0 + size_t(qb) * BQ) * ld + head * D;
    const __nv_bfloat16* Kg = qkv + tok0 * ld + H * D + head * D;
    const __nv_bfloat16* Vg = qkv + tok0 * ld + 2 * H * D + head * D;

    const uint32_t sQ = smem_u32(sm);
    const uint32_t sK[2] = {sQ + 16384, sQ + 16384 * 2};
    const uint32_t sV[2] = {sQ + 16384 * 3, sQ + 16384 * 4};

    load_tile(sQ, Qg, ld, tid);
    load_tile(sK[0], Kg, ld, tid);
    load_tile(sV[0], Vg, ld, tid);
    cp_commit();

    float o[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    const float sl2 = scale * kLog2e;
    const int g = lane >> 2, t4 = lane & 3;
    const int qrow0 = qb * BQ + warp * 16 + g;  // rows g and g+8 of this warp, within the sequence

    uint32_t qf[8][4];
    for (int kb = 0; kb <= qb; ++kb) {
        const int buf = kb & 1;
        if (kb + 1 <= qb) {
            load_tile(sK[buf ^ 1], Kg + size_t(kb + 1) * BKV * ld, ld, tid);
            load_tile(sV[buf ^ 1], Vg + size_t(kb + 1) * BKV * ld, ld, tid);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (kb == 0) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) frag_a(sQ, warp * 16, kk * 16, lane, qf[kk]);
        }
        // S = Q K^T (16 x 64 per warp)
        float s[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                uint32_t bf[4];
                frag_b_nk(sK[buf], j * 8, kk * 16, lane, bf);
                mma16816(s[j], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], bf[0], bf[1]);
                mma16816(s[j + 1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], bf[2], bf[3]);
            }
        }
        // scale, causal mask on the diagonal tile, online softmax
        float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float v = s[j][e] * sl2;
                if (kb == qb) {
                    int key = kb * BKV + j * 8 + 2 * t4 + (e & 1);
                    int q = qrow0 + (e >> 1) * 8;
                    if (key > q) v = -INFINITY;
                }
                s[j][e] = v;
                mnew[e >> 1] = fmaxf(mnew[e >> 1], v);
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffff, mnew[r], 1));
            mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffff, mnew[r], 2));
        }
        float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
        for (int r = 0; r < 2; ++r) corr[r] = exp2f(mrow[r] - mnew[r]);
        uint32_t pf[4][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float p0 = exp2f(s[j][0] - mnew[0]), p1 = exp2f(s[j][1] - mnew[0]);
            float p2 = exp2f(s[j][2] - mnew[1]), p3 = exp2f(s[j][3] - mnew[1]);
            rs[0] += p0 + p1;
            rs[1] += p2 + p3;
            const int kk = j >> 1, hi = j & 1;
            pf[kk][hi * 2 + 0] = pack_bf16(p0, p1);
            pf[kk][hi * 2 + 1] = pack_bf16(p2, p3);
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            lrow[r] = lrow[r] * corr[r] + rs[r];
            mrow[r] = mnew[r];
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            o[i][0] *= corr[0];
            o[i][1] *= corr[0];
            o[i][2] *= corr[1];
            o[i][3] *= corr[1];
        }
        // O += P V   (P: 16 x 64 keys from registers; V: [key][d])
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                uint32_t bf[4];
                frag_b_kn(sV[buf], i * 8, kk * 16, lane, bf);
                mma16816(o[i], pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3], bf[0], bf[1]);
                mma16816(o[i + 1], pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3], bf[2], bf[3]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        lrow[r] += __shfl_xor_sync(0xffffffff, lrow[r], 1);
        lrow[r] += __shfl_xor_sync(0xffffffff, lrow[r], 2);
    }
    const float inv0 = 1.f / lrow[0], inv1 = 1.f / lrow[1];
    const size_t t0 = tok0 + qrow0, t1 = t0 + 8;
    __nv_bfloat16* O0 = out + t0 * (H * D) + head * D;
    __nv_bfloat16* O1 = out + t1 * (H * D) + head * D;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int c = i * 8 + 2 * t4;
        *reinterpret_cast<uint32_t*>(O0 + c) = pack_bf16(o[i][0] * inv0, o[i][1] * inv0);
        *reinterpret_cast<uint32_t*>(O1 + c) = pack_bf16(o[i][2] * inv1, o[i][3] * inv1);
    }
    if (t4 == 0) {
        lse2[size_t(head) * T + t0] = mrow[0] + log2f(lrow[0]);
        lse2[size_t(head) * T + t1] = mrow[1] + log2f(lrow[1]);
    }
}

// ------------------------------------------------------------------ backward
// Dsum[h][t] = sum_d dO * O ; also zero the fp32 dQ accumulator.
__global__ void attn_bwd_pre_kernel(const __nv_bfloat16* __restrict__ dout, const __nv_bfloat16* __restrict__ out,
                                    float* __restrict__ dsum, float* __restrict__ dq_acc, int H, int T) {
    pdl_wait();
    pdl_launch();
    const int t = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
}

// one CTA per (key tile, head, sequence); 4 warps x 16 keys
__global__ void __launch_bounds__(128, 1)
    attn_bwd_kernel(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
                    const float* __restrict__ lse2, const float* __restrict__ dsum, float* __restrict__ dq_acc,
                    __nv_bfloat16* __restrict__ dqkv, int seq, int H, int T, float scale) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nkb = seq / BKV;
    const int kb = blockIdx.x;
    const int head = blockIdx.y, b = blockIdx.z;
    const int ld = 3 * H * D, ldo = H * D;
    const size_t tok0 = size_t(b) * seq;
    const __nv_bfloat16* Qg = qkv + tok0 * ld + head * D;
    const __nv_bfloat16* Kg = qkv + (tok0 + size_t(kb) * BKV) * ld + H * D + head * D;
    const __nv_bfloat16* Vg = qkv + (tok0 + size_t(kb) * BKV) * ld + 2 * H * D + head * D;
    const __nv_bfloat16* dOg = dout + tok0 * ldo + head * D;

    const uint32_t sK = smem_u32(sm), sV = sK + 16384;
    const uint32_t sQ[2] = {sK + 16384 * 2, sK + 16384 * 3};
    const uint32_t sdO[2] = {sK + 16384 * 4, sK + 16384 * 5};
    const uint32_t sdS = sK + 16384 * 6;  // [64 keys][64 q] bf16, rows of 128B (swizzle on 8 chunks)
    float* sL = reinterpret_cast<float*>(sm + 16384 * 6 + 8192);  // lse2[64], dsum[64] x 2 buffers
    const float sl2 = scale * kLog2e;
    const int g = lane >> 2, t4 = lane & 3;

    load_tile(sK, Kg, ld, tid);
    load_tile(sV, Vg, ld, tid);
    const int qb0 = kb;
    load_tile(sQ[0], Qg + size_t(qb0) * BQ * ld, ld, tid);
    load_tile(sdO[0], dOg + size_t(qb0) * BQ * ldo, ldo, tid);
    cp_commit();

    float dk[16][4], dv[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;

    const int key_row0 = kb * BKV + warp * 16 + g;  // keys g, g+8 of this warp (within sequence)
    for (int qb = qb0; qb < nkb; ++qb) {
        const int buf = (qb - qb0) & 1;
        if (tid < 64) {
            sL[buf * 128 + tid] = lse2[size_t(head) * T + tok0 + size_t(qb) * BQ + tid];
            sL[buf * 128 + 64 + tid] = dsum[size_t(head) * T + tok0 + size_t(qb) * BQ + tid];
        }
        if (qb + 1 < nkb) {
            load_tile(sQ[buf ^ 1], Qg + size_t(qb + 1) * BQ * ld, ld, tid);
            load_tile(sdO[buf ^ 1], dOg + size_t(qb + 1) * BQ * ldo, ldo, tid);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const float* Ls = sL + buf * 128;
        // S^T = K Q^T (16 keys x 64 queries per warp); dP^T = V dO^T
        float st[8][4], dpt[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) st[j][e] = dpt[j][e] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t ka[4], va[4];
            frag_a(sK, warp * 16, kk * 16, lane, ka);
            frag_a(sV, warp * 16, kk * 16, lane, va);
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
                uint32_t qf[4], of[4];
                frag_b_nk(sQ[buf], j * 8, kk * 16, lane, qf);
                frag_b_nk(sdO[buf], j * 8, kk * 16, lane, of);
                mma16816(st[j], ka[0], ka[1], ka[2], ka[3], qf[0], qf[1]);
                mma16816(st[j + 1], ka[0], ka[1], ka[2], ka[3], qf[2], qf[3]);
                mma16816(dpt[j], va[0], va[1], va[2], va[3], of[0], of[1]);
                mma16816(dpt[j + 1], va[0], va[1], va[2], va[3], of[2], of[3]);
            }
        }
        // P^T, dS^T
        uint32_t pf[4][4], dsf[4][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float p[4], ds[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int ql = j * 8 + 2 * t4 + (e & 1);  // query within tile
                const int key = key_row0 + (e >> 1) * 8;
                float v = exp2f(st[j][e] * sl2 - Ls[ql]);
                if (qb == kb && key > qb * BQ + ql) v = 0.f;
                p[e] = v;
                ds[e] = v * (dpt[j][e] - Ls[64 + ql]);
            }
            const int kk = j >> 1, hi = j & 1;
            pf[kk][hi * 2 + 0] = pack_bf16(p[0], p[1]);
            pf[kk][hi * 2 + 1] = pack_bf16(p[2], p[3]);
            dsf[kk][hi * 2 + 0] = pack_bf16(ds[0], ds[1]);
            dsf[kk][hi * 2 + 1] = pack_bf16(ds[2], ds[3]);
            // stash dS^T (keys x queries) for the dQ product
            const int kr = warp * 16 + g;
            const int qc = j * 8 + 2 * t4;
            uint32_t a0 = uint32_t(kr * 128 + ((((qc >> 3) ^ (kr & 7))) << 4) + (qc & 7) * 2);
            uint32_t a1 = uint32_t((kr + 8) * 128 + ((((qc >> 3) ^ ((kr + 8) & 7))) << 4) + (qc & 7) * 2);
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(sdS + a0), "r"(dsf[kk][hi * 2 + 0]));
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(sdS + a1), "r"(dsf[kk][hi * 2 + 1]));
        }
        // dV += P^T dO ; dK += dS^T Q   (B operands stored [q][d])
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                uint32_t ob[4], qb4[4];
                frag_b_kn(sdO[buf], i * 8, kk * 16, lane, ob);
                frag_b_kn(sQ[buf], i * 8, kk * 16, lane, qb4);
                mma16816(dv[i], pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3], ob[0], ob[1]);
                mma16816(dv[i + 1], pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3], ob[2], ob[3]);
                mma16816(dk[i], dsf[kk][0], dsf[kk][1], dsf[kk][2], dsf[kk][3], qb4[0], qb4[1]);
                mma16816(dk[i + 1], dsf[kk][0], dsf[kk][1], dsf[kk][2], dsf[kk][3], qb4[2], qb4[3]);
            }
        }
        __syncthreads();
        // dQ (16 queries per warp x 128) += dS (q x 64 keys) K (64 keys x 128), atomically in fp32
        {
            float dq[16][4];
#pragma unroll
            for (int i = 0; i < 16; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                // A = dS[q][key] = transpose of sdS[key][q] tile (rows 128B)
                uint32_t a[4];
                {
                    int krow = kk * 16 + (lane & 7) + (lane >> 4) * 8;
                    int qcol = warp * 16 + ((lane >> 3) & 1) * 8;
                    uint32_t addr = sdS + uint32_t(krow * 128 + ((((qcol >> 3) ^ (krow & 7))) << 4));
                    ldsm_x4_t(addr, a[0], a[1], a[2], a[3]);
                }
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    uint32_t kbf[4];
                    frag_b_kn(sK, i * 8, kk * 16, lane, kbf);
                    mma16816(dq[i], a[0], a[1], a[2], a[3], kbf[0], kbf[1]);
                    mma16816(dq[i + 1], a[0], a[1], a[2], a[3], kbf[2], kbf[3]);
                }
            }
            const size_t q0 = tok0 + size_t(qb) * BQ + warp * 16 + g;
            float* r0 = dq_acc + q0 * (H * D) + head * D;
            float* r1 = r0 + 8 * size_t(H * D);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int c = i * 8 + 2 * t4;
                atomicAdd(r0 + c, dq[i][0]);
                atomicAdd(r0 + c + 1, dq[i][1]);
                atomicAdd(r1 + c, dq[i][2]);
                atomicAdd(r1 + c + 1, dq[i][3]);
            }
        }
        __syncthreads();
    }
    // write dK, dV (scale folds the softmax scale into dK)
    const size_t k0 = tok0 + key_row0, k1 = k0 + 8;
    __nv_bfloat16* dK0 = dqkv + k0 * ld + H * D + head * D;
    __nv_bfloat16* dK1 = dqkv + k1 * ld + H * D + head * D;
    __nv_bfloat16* dV0 = dqkv + k0 * ld + 2 * H * D + head * D;
    __nv_bfloat16* dV1 = dqkv + k1 * ld + 2 * H * D + head * D;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int c = i * 8 + 2 * t4;
        *reinterpret_cast<uint32_t*>(dK0 + c) = pack_bf16(dk[i][0] * scale, dk[i][1] * scale);
        *reinterpret_cast<uint32_t*>(dK1 + c) = pack_bf16(dk[i][2] * scale, dk[i][3] * scale);
        *reinterpret_cast<uint32_t*>(dV0 + c) = pack_bf16(dv[i][0], dv[i][1]);
        *reinterpret_cast<uint32_t*>(dV1 + c) = pack_bf16(dv[i][2], dv[i][3]);
    }
}

__global__ void attn_dq_store_kernel(const float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv, int H,
                                     float scale) {
    pdl_wait();
    pdl_launch();
    const int t = blockIdx.x;
    for (int c = threadIdx.x * 4; c < H * D; c += blockDim.x * 4) {
        float4 v = *reinterpret_cast<const float4*>(dq_acc + size_t(t) * H * D + c);
        uint2 o = make_uint2(pack_bf16(v.x * scale, v.y * scale), pack_bf16(v.z * scale, v.w * scale));
        *reinterpret_cast<uint2*>(dqkv + size_t(t) * 3 * H * D + c) = o;
    }
}

}  // namespace

void attn_fwd(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse2, int batch, int seq, int heads,
              cudaStream_t s) {
    if (seq % 64) throw std::invalid_argument("attention: seq must be a multiple of 64");
    static bool once = [] {
        cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 16384);
        return true;
    }();
    (void)once;
    dim3 grid(seq / BQ, heads, batch);
    attn_fwd_kernel<<<grid, 128, 5 * 16384, s>>>(qkv, out, lse2, seq, heads, batch * seq, 0.08838834764831845f);
}

void attn_bwd_pre(const __nv_bfloat16* dout, const __nv_bfloat16* out, float* dsum, float* dq_acc, int heads, int T,
                  cudaStream_t s) {
    launch_k(attn_bwd_pre_kernel, dim3(T), dim3(256), 0, s, 1, dout, out, dsum, dq_acc, heads, T);
}

void attn_dq_store(const float* dq_acc, __nv_bfloat16* dqkv, int heads, int T, cudaStream_t s) {
    launch_k(attn_dq_store_kernel, dim3(T), dim3(256), 0, s, 1, dq_acc, dqkv, heads, 0.08838834764831845f);
}

void attn_bwd(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout, const float* lse2,
              float* dsum, float* dq_acc, __nv_bfloat16* dqkv, int batch, int seq, int heads, cudaStream_t s) {
    constexpr int kSmem = 6 * 16384 + 8192 + 2 * 128 * 4;
    static bool once = [] {
        cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        return true;
    }();
    (void)once;
    const int T = batch * seq;
    attn_bwd_pre_kernel<<<T, 256, 0, s>>>(dout, out, dsum, dq_acc, heads, T);
    dim3 grid(seq / BKV, heads, batch);
    const float scale = 0.08838834764831845f;
    attn_bwd_kernel<<<grid, 128, kSmem, s>>>(qkv, dout, lse2, dsum, dq_acc, dqkv, seq, heads, T, scale);
    attn_dq_store_kernel<<<T, 256, 0, s>>>(dq_acc, dqkv, heads, scale);
}

}  // namespace pbk
