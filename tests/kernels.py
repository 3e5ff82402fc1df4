"""ctypes access to the kernel test entry points (include/pipeblock_b200_kernels.h)."""
import ctypes as C

import torch

from paper_2405_15362_b200 import _lib


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def gemm(A, B, C_, *, a_mn=False, b_mn=False, epi=0, C2=None, aux=None, accumulate=0):
    """C (epi)= A . B with A [M,K] (or [K,M] if a_mn) and B [N,K] (or [K,N] if b_mn)."""
    if a_mn:
        K, M = A.shape
    else:
        M, K = A.shape
    N = B.shape[1] if b_mn else B.shape[0]
    L = _lib.lib()
    _lib.check(L.pbt_gemm(M, N, K, _p(A), A.stride(0), int(a_mn), _p(B), B.stride(0), int(b_mn), _p(C_),
                          C_.stride(0), _p(C2), _p(aux), aux.stride(0) if aux is not None else 0, epi, accumulate,
                          _s()))
