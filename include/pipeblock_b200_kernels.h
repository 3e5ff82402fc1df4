/*
 * pipeblock_b200_kernels.h — direct access to the individual sm_100a kernels
 * the executor chains into F/B/W passes.  For kernel parity tests and
 * micro-benchmarks only (device pointers in, device pointers out, optional
 * cudaStream_t); the executor does not go through these entry points.
 * bf16 tensors are passed as raw device pointers to 16-bit storage.
 */
#ifndef PIPEBLOCK_B200_KERNELS_H
#define PIPEBLOCK_B200_KERNELS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* C[M,N] (epi)= A . B ; a_mn: A stored [K][M], else [M][K]; b_mn: B stored [K][N], else [N][K].
 * epi: 0 store bf16, 1 gelu (C=u, C2=gelu(u)), 2 residual (C=acc+aux), 3 dgelu (C=acc*gelu'(aux)),
 *      4 fp32 (C f32, accumulate != 0 adds). */
int pbt_gemm(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, int32_t a_mn, const void* B, int32_t ldb,
             int32_t b_mn, void* C, int32_t ldc, void* C2, const void* aux, int32_t ldaux, int32_t epi,
             int32_t accumulate, void* stream);

/* Force the GEMM variant: 1 = one CTA per 128-row tile, 2 = CTA pair (cta_group::2) per 256-row tile
 * where M and N allow it, -1 = automatic (default). Process-wide; for tests and benchmarks. */
int pbt_gemm_set_cta_group(int32_t cg);
int pbt_gemm_set_pair_rows(int32_t rows); /* CTA-pair tile rows: 256, 512 (two A sub-tiles per CTA, M % 512 == 0), -1 = PB_GEMM_BM2 */
/* pbt_gemm plus the folded-RMSNorm hooks: rs (may be NULL) = per-row sum of squares, the accumulator row
 * is scaled by rsqrt(rs[row] * rs_inv_n + rs_eps) (epi 0 / 1 / 3); ss_out (may be NULL, epi 2) = the
 * row's sum of squares of the stored bf16 outputs (deterministic, bit-identical to pbt_row_sumsq). */
int pbt_gemm_rownorm(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, int32_t a_mn, const void* B,
                     int32_t ldb, int32_t b_mn, void* C, int32_t ldc, void* C2, const void* aux, int32_t ldaux,
                     int32_t epi, const float* rs, float rs_inv_n, float rs_eps, float* ss_out, void* stream);
/* ss[t] = sum of squares of row t of x [T,h] bf16 (h % 128 == 0), in the GEMM epilogue's order */
int pbt_row_sumsq(const void* x, float* ss, int32_t T, int32_t h, void* stream);
/* causal attention, head_dim 128, tcgen05/TMEM (the executor's forward attention): qkv [T,3h] -> out [T,h],
 * lse2 [heads,T] (base-2 LSE of scaled scores); seq % 128 == 0 */
int pbt_attn_fwd_tc(const void* qkv, void* out, float* lse2, int32_t batch, int32_t seq, int32_t heads, void* stream);
/* backward on tcgen05/TMEM (the executor's): dqkv [T,3h]; dsum [heads*T + 64] (the row terms, then the
 * persistent kernel's work counter), dq_acc [T,h] fp32 scratch */
int pbt_attn_bwd_tc(const void* qkv, const void* out, const void* dout, const float* lse2, float* dsum, float* dq_acc,
                    void* dqkv, int32_t batch, int32_t seq, int32_t heads, void* stream);
int pbt_rmsnorm_fwd(const void* x, const void* g, void* y, float* rstd, int32_t T, int32_t h, void* stream);
int pbt_rmsnorm_bwd(const void* dy, const void* x, const void* g, const float* rstd, const void* dres, void* dx,
                    float* dgamma, int32_t T, int32_t h, void* stream);
/* backward of y = rstd * x with gamma folded (the executor's norm backward): dyp = rstd * dy (the dX GEMM's
 * row-scaled output), ss = the forward row sums of squares; dx = dyp - x * mean(dyp * x) / (ss / h + eps)
 * (+ dres when not NULL); h % 256 == 0 */
int pbt_rmsnorm_bwd_x(const void* dyp, const void* x, const float* ss, const void* dres, void* dx, int32_t T,
                      int32_t h, float eps, void* stream);
int pbt_embed_fwd(const int32_t* tok, const void* emb, void* x, int32_t T, int32_t h, void* stream);
int pbt_embed_bwd(const int32_t* tok, const void* dx, float* demb, int32_t T, int32_t h, void* stream);
int pbt_cross_entropy(void* logits, const int32_t* labels, float* loss, int32_t T, int32_t V, float scale,
                      void* stream);
int pbt_adamw(float* w, void* wb, float* g, float* m, float* v, int64_t n, float lr, float b1, float b2, float eps,
              float wd, int32_t step, void* stream);

#ifdef __cplusplus
}
#endif
#endif
