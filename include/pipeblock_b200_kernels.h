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

#ifdef __cplusplus
}
#endif
#endif
