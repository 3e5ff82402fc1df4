"""Phase timestamps of block 0 (the heaviest causal tile) of the tcgen05 attention forward.
    PB_ATTN_TRACE_FWD=1 python -m tests.trace_attn_fwd"""
import torch

from tests import kernels as K

qkv = torch.randn(4096, 3 * 2048, device="cuda").bfloat16()
for _ in range(2):
    K.attn_fwd_tc(qkv, 2, 2048, 16)
torch.cuda.synchronize()
