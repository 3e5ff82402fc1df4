"""Phase timestamps of block 0 of the tcgen05 attention backward (PB_ATTN_TRACE=1), at the bench shape.
    PB_ATTN_TRACE=1 python -m tests.trace_attn_bwd"""
import torch

from tests import kernels as K

qkv = torch.randn(4096, 3 * 2048, device="cuda").bfloat16()
out, lse2 = K.attn_fwd_tc(qkv, 2, 2048, 16)
dout = torch.randn_like(out)
for _ in range(3):
    K.attn_bwd_tc(qkv, out, dout, lse2, 2, 2048, 16)
torch.cuda.synchronize()
