// Host interface of the non-GEMM sm_100a kernels (attention.cu, ops.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "gemm.hpp"

namespace pbk {

// causal MHA, head_dim 128, tcgen05/TMEM (attention_tc.cu): qkv [T,3h] -> out [T,h], lse2 [heads,T]
// (base-2 LSE of the scaled scores); seq % 128 == 0
void attn_fwd_tc(const __nv_bfloat16* qkv, __nv_bfloat16* out, float* lse2, int batch, int seq, int heads,
                 cudaStream_t s);
// dqkv [T,3h] from dout [T,h]; dsum [heads,T] and dq_acc [T,h] fp32 are scratch.  rs (may be null):
// per-token sum of squares of the QKV GEMM's input; dqkv rows are then scaled by
// rsqrt(rs * rs_inv_n + rs_eps) (the folded RMSNorm's rstd, see executor.cpp)
void attn_bwd_tc(const __nv_bfloat16* qkv, const __nv_bfloat16* out, const __nv_bfloat16* dout, const float* lse2,
                 float* dsum, float* dq_acc, __nv_bfloat16* dqkv, int batch, int seq, int heads, cudaStream_t s,
                 const float* rs = nullptr, float rs_inv_n = 0.f, float rs_eps = 0.f);
void attn_bwd_pre(const __nv_bfloat16* dout, const __nv_bfloat16* out, float* dsum, float* dq_acc, int heads, int T,
                  cudaStream_t s);
void attn_dq_store(const float* dq_acc, __nv_bfloat16* dqkv, int heads, int T, cudaStream_t s,
                   const float* rs = nullptr, float rs_inv_n = 0.f, float rs_eps = 0.f);

// g may be null (unit gamma: the gamma is folded into the next projection)
void rmsnorm_fwd(const __nv_bfloat16* x, const __nv_bfloat16* g, __nv_bfloat16* y, float* rstd, int T, int h,
                 cudaStream_t s);
// dx = dres (may be null) + d/dx rmsnorm(x)*g applied to dy
void rmsnorm_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, const __nv_bfloat16* g, const float* rstd,
                 const __nv_bfloat16* dres, __nv_bfloat16* dx, int T, int h, cudaStream_t s);
// dgamma (fp32) += sum_t dy * x * rstd ; deterministic; scratch >= ceil(T/16) * h floats
void rmsnorm_dgamma(const __nv_bfloat16* dy, const __nv_bfloat16* x, const float* rstd, float* dgamma, float* scratch,
                    int T, int h, cudaStream_t s);
// ids outside [0, V) are never dereferenced: the row is zeroed / skipped and *err (may be null) |= 1
void embed_fwd(const int32_t* tok, const __nv_bfloat16* emb, __nv_bfloat16* x, int T, int h, int V, int* err,
               cudaStream_t s);
void embed_bwd(const int32_t* tok, const __nv_bfloat16* dx, float* demb, int T, int h, int V, int* err,
               cudaStream_t s);
// loss (fp32 scalar) += scale * sum_rows CE ; logits <- scale * (softmax - onehot), in place
// (a label outside [0, V) adds no loss and no one-hot, and sets *err); rs (may be null): the rows of
// dlogits are further scaled by rsqrt(rs * rs_inv_n + rs_eps) (folded final RMSNorm)
void cross_entropy(__nv_bfloat16* logits, const int32_t* labels, float* loss, int T, int V, float scale, int* err,
                   cudaStream_t s, const float* rs = nullptr, float rs_inv_n = 0.f, float rs_eps = 0.f);
// folded RMSNorm (executor fold mode): ss[row] = sum_c x^2 ; and the backward
// dx = dyp - x * rstd^2 * mean(dyp * x) + dres (dres may be null), rstd = rsqrt(ss / h + eps)
// dst[0, n) += src[0, n) (fp32; n % 4 == 0, 16-byte aligned)
void grad_add(float* dst, const float* src, size_t n, cudaStream_t s);
void row_sumsq(const __nv_bfloat16* x, float* ss, int T, int h, cudaStream_t s);
void rmsnorm_bwd_x(const __nv_bfloat16* dyp, const __nv_bfloat16* x, const float* ss, const __nv_bfloat16* dres,
                   __nv_bfloat16* dx, int T, int h, float eps, cudaStream_t s);
void adamw(float* w, __nv_bfloat16* wb, float* g, float* m, float* v, size_t n, float lr, float b1, float b2,
           float eps, float wd, int step, cudaStream_t s);
void f32_to_bf16(const float* src, __nv_bfloat16* dst, size_t n, cudaStream_t s);
// gamma folding (executor.cpp): wb = bf16(w * g[col]) ; and once per step
// dw += dwp * g[col], dg[col] += sum_rows dwp * w, dwp <- 0 (deterministic; scratch fp32)
void fold_weight(const float* w, const float* g, __nv_bfloat16* wb, int rows, int cols, cudaStream_t s);
void fold_grad(float* dwp, const float* w, const float* g, float* dw, float* dg, float* scratch, size_t scratch_floats,
               int rows, int cols, cudaStream_t s);
void init_normal(float* w, size_t n, uint64_t seed, float std, float constant, cudaStream_t s);

}  // namespace pbk
