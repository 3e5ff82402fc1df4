"""One launch of each hot kernel at GPT-1.5B / seq 2048 / micro-batch 2 pass shapes (T=4096; for ncu captures)."""
import torch

from tests import kernels as K

B_, S_, h, H = 2, 2048, 2048, 16
T = B_ * S_
torch.manual_seed(0)
A = torch.randn(T, h, device="cuda").bfloat16()
W1 = torch.randn(4 * h, h, device="cuda").bfloat16()
U = torch.empty(T, 4 * h, device="cuda", dtype=torch.bfloat16)
G = torch.empty_like(U)
K.gemm(A, W1, U, epi=1, C2=G)                                   # F: fc1 + GELU
dY = torch.randn(T, h, device="cuda").bfloat16()
W2t = torch.randn(h, 4 * h, device="cuda").bfloat16()
K.gemm(dY, W2t, U, b_mn=True, epi=3, aux=U)                     # B: dgl * gelu'
dW = torch.zeros(h, 4 * h, device="cuda")
K.gemm(dY, G, dW, a_mn=True, b_mn=True, epi=4, accumulate=1)   # W: dW2 += dY^T gelu(u)
# folded RMSNorm (the executor's default F pass): FC1+GELU with the rstd row scale, FC2 + residual
# emitting the next norm's per-row sum of squares, and the stand-alone statistic of a stage input
ss = (torch.rand(T, device="cuda") + 0.5) * h
K.gemm_rownorm(A, W1, U, epi=1, C2=G, rs=ss, inv_n=1.0 / h)    # F: fc1 + GELU, rows scaled by rstd
W2 = torch.randn(h, 4 * h, device="cuda").bfloat16()
X1 = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
K.gemm_rownorm(G, W2, X1, epi=2, aux=A, ss_out=ss)              # F: fc2 + residual + sum of squares
K.row_sumsq(X1, ss)
qkv = torch.randn(T, 3 * h, device="cuda").bfloat16()
out, lse2 = K.attn_fwd_tc(qkv, B_, S_, H)
dout = torch.randn_like(out)
K.attn_bwd_tc(qkv, out, dout, lse2, B_, S_, H)
torch.cuda.synchronize()
print("ok")
