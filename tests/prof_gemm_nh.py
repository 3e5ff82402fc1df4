"""The N = h GEMMs of the bench shape (T=4096, h=2048) for ncu: F-pass O projection (+residual, row
sum of squares; K = h), FC2 (+residual, K = 4h, 512-row pair tiles), B-pass O dX (K = h) and FC1 dX
(K = 4h)."""
import torch

from tests import kernels as K

T, h = 4096, 2048
torch.manual_seed(0)
A = torch.randn(T, h, device="cuda").bfloat16()
Wo = torch.randn(h, h, device="cuda").bfloat16() * 0.02
R = torch.randn(T, h, device="cuda").bfloat16()
X = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
ss = torch.empty(T, device="cuda")
for _ in range(2):
    K.gemm_rownorm(A, Wo, X, epi=2, aux=R, ss_out=ss)          # F: O projection + residual + sum of squares
U = torch.randn(T, 4 * h, device="cuda").bfloat16()
W2 = torch.randn(h, 4 * h, device="cuda").bfloat16() * 0.02
K.gemm_rownorm(U, W2, X, epi=2, aux=R, ss_out=ss)               # F: FC2 + residual + sum of squares
K.gemm(A, Wo, X, b_mn=True)                                     # B: O dX
W1 = torch.randn(4 * h, h, device="cuda").bfloat16() * 0.02
K.gemm(U, W1, X, b_mn=True)                                     # B: FC1 dX
torch.cuda.synchronize()
print("ok")
