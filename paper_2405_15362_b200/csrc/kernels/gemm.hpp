// Host interface of the sm_100a kernels (kernels/*.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pbk {

enum Epi : int {
    EPI_STORE = 0,  // C(bf16) = acc
    EPI_GELU = 1,   // C(bf16) = acc (pre-activation u), C2(bf16) = gelu(u)
    EPI_RESID = 2,  // C(bf16) = acc + aux(bf16)      (residual add; C may alias aux)
    EPI_DGELU = 3,  // C(bf16) = acc * gelu'(aux)     (aux = pre-activation u)
    EPI_F32 = 4,    // C(f32) (+)= acc                (weight gradients, accumulate flag)
};

struct GemmArgs {
    int M = 0, N = 0, K = 0;
    const __nv_bfloat16* A = nullptr;
    int lda = 0;
    bool a_mn = false;  // A stored [K][M] (else [M][K])
    const __nv_bfloat16* B = nullptr;
    int ldb = 0;
    bool b_mn = false;  // B stored [K][N] (else [N][K])
    void* C = nullptr;
    int ldc = 0;
    void* C2 = nullptr;
    const __nv_bfloat16* aux = nullptr;
    int ldaux = 0;
    int epi = EPI_STORE;
    int accumulate = 0;
    // folded RMSNorm (STORE / GELU / DGELU): acc(row, :) *= rsqrt(rs[row] * rs_inv_n + rs_eps)
    const float* rs = nullptr;
    float rs_inv_n = 0.f, rs_eps = 0.f;
    // RESID: ss_out[row] = sum of squares of the row's stored (bf16) outputs, deterministic: every
    // tile writes one fp32 partial per 128 columns to ss_part ([M][N/128]); the last tile to finish a
    // 32-row group (ss_cnt[row / 32], zero before the launch and reset by that tile) sums the partials
    // in column order.  row_sumsq() (ops.hpp) computes the bit-identical value from a stored matrix.
    float* ss_out = nullptr;
    float* ss_part = nullptr;
    int* ss_cnt = nullptr;
};

void gemm(const GemmArgs& g, cudaStream_t s);

// Grouped weight-gradient GEMMs: independent dW (+)= dY^T X problems (A and B MN-major,
// fp32 epilogue) run as ONE persistent CTA-pair launch over their concatenated tiles,
// so the W pass of a whole stage pays one ramp and one tail.  Descriptor table lives
// in device memory; built once per (stage, activation slot).
struct GemmGroup {
    void* table = nullptr;  // device GroupProblem[n]
    int n = 0;
    int total_tiles = 0;
    int accumulate = 1;
};
GemmGroup gemm_group_create(const GemmArgs* problems, int n);
void gemm_group_run(const GemmGroup& g, cudaStream_t s);
void gemm_group_destroy(GemmGroup& g);
bool gemm_group_ok(const GemmArgs& g);  // eligible for a group
int gemm_bn(const GemmArgs& g);
int num_sms();
// tests: force the 1-CTA (1) or CTA-pair (2) variant where shapes allow; -1 = automatic
void gemm_force_cta_group(int cg);
void gemm_force_bm2(int on);  // tests: 512 x 256 CTA-pair tiles, -1 = PB_GEMM_BM2
// 2-D bf16 tensor map [outer][inner], row stride ld elements, box_inner x box_outer, 128B swizzle
CUtensorMap make_map_t(const void* base, CUtensorMapDataType dt, uint32_t esize, uint64_t inner, uint64_t outer,
                       uint64_t ld, uint32_t box_inner, uint32_t box_outer);
CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                     uint32_t box_outer);

}  // namespace pbk
