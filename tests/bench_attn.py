"""Attention micro-benchmark (causal, head_dim 128): TFLOP/s of fwd kernels (causal FLOPs = 2*s^2*h per seq)."""
import json
import sys

import torch

from tests import kernels as K
from tests.bench_gemm import timeit


def main():
    for batch, seq, heads in [(1, 2048, 16), (2, 2048, 16), (1, 4096, 32), (1, 6144, 48)]:
        qkv = torch.randn(batch * seq, 3 * heads * 128, device="cuda").bfloat16()
        fl = 2.0 * seq * seq * heads * 128 * batch  # causal fwd: 4*s^2*d*H/2
        t_old = timeit(lambda: K.attn_fwd(qkv, batch, seq, heads))
        t_new = timeit(lambda: K.attn_fwd_tc(qkv, batch, seq, heads))
        out, lse2 = K.attn_fwd(qkv, batch, seq, heads)
        dout = torch.randn_like(out)
        t_bwd = timeit(lambda: K.attn_bwd(qkv, out, dout, lse2, batch, seq, heads))
        t_bwd_tc = timeit(lambda: K.attn_bwd_tc(qkv, out, dout, lse2, batch, seq, heads))
        # library reference point (cuDNN / flash SDPA through torch), fwd and fwd+bwd
        q = torch.randn(batch, heads, seq, 128, device="cuda", dtype=torch.bfloat16, requires_grad=True)
        k, v = torch.randn_like(q, requires_grad=True), torch.randn_like(q, requires_grad=True)
        sd = torch.nn.functional.scaled_dot_product_attention
        t_sdpa = timeit(lambda: sd(q, k, v, is_causal=True))
        o = sd(q, k, v, is_causal=True)
        go = torch.randn_like(o)
        t_sdpa_fb = timeit(lambda: torch.autograd.grad(sd(q, k, v, is_causal=True), (q, k, v), go))
        print(json.dumps({"sdpa_fwd_tflops": fl / t_sdpa / 1e9, "sdpa_bwd_tflops_est": 2.5 * fl / max(1e-9, t_sdpa_fb - t_sdpa) / 1e9}))
        print(json.dumps({"batch": batch, "seq": seq, "heads": heads, "fwd_mma_sync_us": t_old * 1e3,
                          "fwd_tcgen05_us": t_new * 1e3, "fwd_mma_sync_tflops": fl / t_old / 1e9,
                          "fwd_tcgen05_tflops": fl / t_new / 1e9, "bwd_mma_sync_us": t_bwd * 1e3,
                          "bwd_mma_sync_tflops": 2.5 * fl / t_bwd / 1e9,
                          "bwd_tcgen05_us": t_bwd_tc * 1e3, "bwd_tcgen05_tflops": 2.5 * fl / t_bwd_tc / 1e9}), flush=True)


if __name__ == "__main__":
    main()
