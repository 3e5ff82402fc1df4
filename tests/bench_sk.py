"""Whole tiles vs stream-K vs hybrid (full waves whole, ragged last wave split) on the bench's pass shapes."""
import json

import torch

from tests import kernels as K
from tests.bench_gemm import timeit

T, h = 4096, 2048
for name, (M, N, Kd, b_mn, epi) in {
    "F.o+res": (T, h, h, False, 2), "F.fc2+res": (T, h, 4 * h, False, 2), "F.qkv": (T, 3 * h, h, False, 0),
    "B.fc1": (T, h, 4 * h, True, 0), "B.qkv": (T, h, 3 * h, True, 0), "B.o": (T, h, h, True, 0),
}.items():
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    B = (torch.randn(Kd, N, device="cuda") if b_mn else torch.randn(N, Kd, device="cuda")).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    aux = torch.randn(M, N, device="cuda").bfloat16() if epi == 2 else None
    row = {"gemm": name, "M": M, "N": N, "K": Kd}
    for mode in (0, 1, 2):
        K.set_stream_k(mode)
        t = timeit(lambda: K.gemm(A, B, C, b_mn=b_mn, epi=epi, aux=aux))
        row[f"sk{mode}_tflops"] = 2.0 * M * N * Kd / t / 1e9
    K.set_stream_k(-1)
    print(json.dumps(row), flush=True)
