"""Three forward-attention launches at (batch, seq, heads) for an ncu capture:

    ncu --set full --import-source on -k regex:attn_fwd -s 2 -c 1 python tools/prof_attn_fwd.py 1 4096 32
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import kernels as K  # noqa: E402

b, s, h = (int(x) for x in sys.argv[1:4])
qkv = torch.randn(b * s, 3 * h * 128, device="cuda").bfloat16()
for _ in range(3):
    K.attn_fwd_tc(qkv, b, s, h)
torch.cuda.synchronize()
