"""256- vs 512-row CTA-pair tiles on the bench's F / B pass shapes (T = 4096, h = 2048)."""
import json

import torch

from tests import kernels as K
from tests.bench_gemm import timeit

T, h = 4096, 2048
for name, (M, N, Kd, b_mn, epi) in {
    "F.qkv": (T, 3 * h, h, False, 0), "F.o+res": (T, h, h, False, 2), "F.fc1+gelu": (T, 4 * h, h, False, 1),
    "F.fc2+res": (T, h, 4 * h, False, 2), "B.fc2+dgelu": (T, 4 * h, h, True, 3), "B.fc1": (T, h, 4 * h, True, 0),
    "B.o": (T, h, h, True, 0), "B.qkv": (T, h, 3 * h, True, 0),
}.items():
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    B = (torch.randn(Kd, N, device="cuda") if b_mn else torch.randn(N, Kd, device="cuda")).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    C2 = torch.empty_like(C) if epi == 1 else None
    aux = torch.randn(M, N, device="cuda").bfloat16() if epi in (2, 3) else None
    row = {"gemm": name, "M": M, "N": N, "K": Kd}
    for rows in (256, 512):
        K.set_pair_rows(rows)
        t = timeit(lambda: K.gemm(A, B, C, b_mn=b_mn, epi=epi, C2=C2, aux=aux))
        row[f"r{rows}_tflops"] = round(2.0 * M * N * Kd / t / 1e9)
    K.set_pair_rows(-1)
    print(json.dumps(row), flush=True)
