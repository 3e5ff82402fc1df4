// Kernel-level test entry points (include/pipeblock_b200_kernels.h).
#include "../../include/pipeblock_b200_kernels.h"

#include <climits>
#include <cstdint>

#include "capi_common.hpp"
#include "kernels/gemm.hpp"
#include "kernels/ops.hpp"

namespace {
void cuda_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw pbx::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

extern "C" int pbt_gemm(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, int32_t a_mn, const void* B,
                        int32_t ldb, int32_t b_mn, void* C, int32_t ldc, void* C2, const void* aux, int32_t ldaux,
                        int32_t epi, int32_t accumulate, void* stream) {
    return pbx::guard([&] {
        pbk::GemmArgs g;
        g.M = M, g.N = N, g.K = K;
        g.A = static_cast<const __nv_bfloat16*>(A), g.lda = lda, g.a_mn = a_mn != 0;
        g.B = static_cast<const __nv_bfloat16*>(B), g.ldb = ldb, g.b_mn = b_mn != 0;
        g.C = C, g.ldc = ldc, g.C2 = C2;
        g.aux = static_cast<const __nv_bfloat16*>(aux), g.ldaux = ldaux;
        g.epi = epi, g.accumulate = accumulate;
        pbk::gemm(g, static_cast<cudaStream_t>(stream));
        cuda_check("pbt_gemm");
    });
}

extern "C" int pbt_gemm_rownorm(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, int32_t a_mn,
                                const void* B, int32_t ldb, int32_t b_mn, void* C, int32_t ldc, void* C2,
                                const void* aux, int32_t ldaux, int32_t epi, const float* rs, float rs_inv_n,
                                float rs_eps, float* ss_out, void* stream) {
    return pbx::guard([&] {
        pbk::GemmArgs g;
        g.M = M, g.N = N, g.K = K;
        g.A = static_cast<const __nv_bfloat16*>(A), g.lda = lda, g.a_mn = a_mn != 0;
        g.B = static_cast<const __nv_bfloat16*>(B), g.ldb = ldb, g.b_mn = b_mn != 0;
        g.C = C, g.ldc = ldc, g.C2 = C2;
        g.aux = static_cast<const __nv_bfloat16*>(aux), g.ldaux = ldaux;
        g.epi = epi;
        g.rs = rs, g.rs_inv_n = rs_inv_n, g.rs_eps = rs_eps, g.ss_out = ss_out;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (ss_out) {  // the row-statistic workspace (the executor keeps one per device)
            const size_t part = size_t(M) * (N / 128) * 4, cnt = size_t(M / 32 + 1) * 4;
            if (cudaMallocAsync(reinterpret_cast<void**>(&g.ss_part), part + cnt, st) != cudaSuccess)
                throw pbx::CudaError("ss workspace allocation failed");
            g.ss_cnt = reinterpret_cast<int*>(reinterpret_cast<char*>(g.ss_part) + part);
            cudaMemsetAsync(g.ss_cnt, 0, cnt, st);
        }
        pbk::gemm(g, st);
        if (ss_out) cudaFreeAsync(g.ss_part, st);
        cuda_check("pbt_gemm_rownorm");
    });
}

#define BF(p) static_cast<const __nv_bfloat16*>(p)
#define BFM(p) static_cast<__nv_bfloat16*>(p)
#define ST(s) static_cast<cudaStream_t>(s)

extern "C" int pbt_row_sumsq(const void* x, float* ss, int32_t T, int32_t h, void* stream) {
    return pbx::guard([&] {
        pbk::row_sumsq(BF(x), ss, T, h, ST(stream));
        cuda_check("pbt_row_sumsq");
    });
}

extern "C" int pbt_rmsnorm_fwd(const void* x, const void* g, void* y, float* rstd, int32_t T, int32_t h,
                               void* stream) {
    return pbx::guard([&] {
        pbk::rmsnorm_fwd(BF(x), BF(g), BFM(y), rstd, T, h, ST(stream));
        cuda_check("pbt_rmsnorm_fwd");
    });
}
extern "C" int pbt_rmsnorm_bwd_x(const void* dyp, const void* x, const float* ss, const void* dres, void* dx,
                                 int32_t T, int32_t h, float eps, void* stream) {
    return pbx::guard([&] {
        pbk::rmsnorm_bwd_x(BF(dyp), BF(x), ss, BF(dres), BFM(dx), T, h, eps, ST(stream));
        cuda_check("pbt_rmsnorm_bwd_x");
    });
}
extern "C" int pbt_rmsnorm_bwd(const void* dy, const void* x, const void* g, const float* rstd, const void* dres,
                               void* dx, float* dgamma, int32_t T, int32_t h, void* stream) {
    return pbx::guard([&] {
        pbk::rmsnorm_bwd(BF(dy), BF(x), BF(g), rstd, BF(dres), BFM(dx), T, h, ST(stream));
        if (dgamma) {
            float* scratch = nullptr;
            if (cudaMallocAsync(reinterpret_cast<void**>(&scratch), size_t((T + 15) / 16) * h * 4, ST(stream)) != cudaSuccess)
                throw pbx::CudaError("scratch allocation failed");
            pbk::rmsnorm_dgamma(BF(dy), BF(x), rstd, dgamma, scratch, T, h, ST(stream));
            cudaFreeAsync(scratch, ST(stream));
        }
        cuda_check("pbt_rmsnorm_bwd");
    });
}
extern "C" int pbt_embed_fwd(const int32_t* tok, const void* emb, void* x, int32_t T, int32_t h, void* stream) {
    return pbx::guard([&] {
        pbk::embed_fwd(tok, BF(emb), BFM(x), T, h, INT32_MAX, nullptr, ST(stream));
        cuda_check("pbt_embed_fwd");
    });
}
extern "C" int pbt_embed_bwd(const int32_t* tok, const void* dx, float* demb, int32_t T, int32_t h, void* stream) {
    return pbx::guard([&] {
        pbk::embed_bwd(tok, BF(dx), demb, T, h, INT32_MAX, nullptr, ST(stream));
        cuda_check("pbt_embed_bwd");
    });
}
extern "C" int pbt_cross_entropy(void* logits, const int32_t* labels, float* loss, int32_t T, int32_t V, float scale,
                                 void* stream) {
    return pbx::guard([&] {
        pbk::cross_entropy(BFM(logits), labels, loss, T, V, scale, nullptr, ST(stream));
        cuda_check("pbt_cross_entropy");
    });
}
extern "C" int pbt_adamw(float* w, void* wb, float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                         float eps, float wd, int32_t step, void* stream) {
    return pbx::guard([&] {
        pbk::adamw(w, BFM(wb), g, m, v, size_t(n), lr, b1, b2, eps, wd, step, ST(stream));
        cuda_check("pbt_adamw");
    });
}
extern "C" int pbt_attn_fwd_tc(const void* qkv, void* out, float* lse2, int32_t batch, int32_t seq, int32_t heads,
                               void* stream) {
    return pbx::guard([&] {
        pbk::attn_fwd_tc(BF(qkv), BFM(out), lse2, batch, seq, heads, ST(stream));
        cuda_check("pbt_attn_fwd_tc");
    });
}
extern "C" int pbt_attn_bwd_tc(const void* qkv, const void* out, const void* dout, const float* lse2, float* dsum,
                               float* dq_acc, void* dqkv, int32_t batch, int32_t seq, int32_t heads, void* stream) {
    return pbx::guard([&] {
        pbk::attn_bwd_tc(BF(qkv), BF(out), BF(dout), lse2, dsum, dq_acc, BFM(dqkv), batch, seq, heads, ST(stream));
        cuda_check("pbt_attn_bwd_tc");
    });
}
extern "C" int pbt_gemm_set_cta_group(int32_t cg) {
    return pbx::guard([&] { pbk::gemm_force_cta_group(cg); });
}

extern "C" int pbt_gemm_set_pair_rows(int32_t rows) {
    return pbx::guard([&] {
        if (rows != -1 && rows != 256 && rows != 512) throw std::invalid_argument("pair rows must be -1, 256 or 512");
        pbk::gemm_force_bm2(rows < 0 ? -1 : rows == 512 ? 1 : 0);
    });
}
