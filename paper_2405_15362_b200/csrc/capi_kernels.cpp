// Kernel-level test entry points (include/pipeblock_b200_kernels.h).
#include "../../include/pipeblock_b200_kernels.h"

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
