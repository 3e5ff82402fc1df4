"""Whole-tile vs stream-K GEMM on a ragged-wave pass shape (4096x2048x8192: 128 pair tiles on
74 CTA pairs), for ncu side by side:  ncu --set full -k regex:gemm_kernel -s 4 -c 2 python -m tests.prof_sk"""
import torch

from tests import kernels as K

M, N, Kd = 4096, 2048, 8192
torch.manual_seed(0)
A = torch.randn(M, Kd, device="cuda").bfloat16()
W = torch.randn(N, Kd, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for sk in (0, 1, 0, 1):  # two warm-up launches, then one of each
    K.set_stream_k(sk)
    K.gemm(A, W, C)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for sk in (0, 1):
    K.set_stream_k(sk)
    for _ in range(3):
        K.gemm(A, W, C)
    torch.cuda.synchronize()
    s.record()
    for _ in range(20):
        K.gemm(A, W, C)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"stream_k={sk}: {ms * 1e3:.1f} us  {2 * M * N * Kd / ms / 1e9:.0f} TFLOP/s")
