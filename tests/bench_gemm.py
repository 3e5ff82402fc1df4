"""GEMM micro-benchmark: TFLOP/s of the tcgen05 kernel vs torch (cuBLAS) on pass shapes."""
import json
import sys

import torch

from tests import kernels as K


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    rows = []
    for h in (2048, 4096):
        for name, (M, N, Kd, mode) in {
            "F.qkv": (T, 3 * h, h, "F"), "F.fc1": (T, 4 * h, h, "F"), "F.fc2": (T, h, 4 * h, "F"),
            "B.fc1": (T, h, 4 * h, "B"), "B.qkv": (T, h, 3 * h, "B"),
            "W.fc1": (4 * h, h, T, "W"), "W.qkv": (3 * h, h, T, "W"), "W.o": (h, h, T, "W"),
        }.items():
            if mode == "F":
                A = torch.randn(M, Kd, device="cuda").bfloat16(); B = torch.randn(N, Kd, device="cuda").bfloat16()
                C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                f = lambda: K.gemm(A, B, C)
                ref = lambda: torch.matmul(A, B.t())
            elif mode == "B":
                A = torch.randn(M, Kd, device="cuda").bfloat16(); B = torch.randn(Kd, N, device="cuda").bfloat16()
                C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                f = lambda: K.gemm(A, B, C, b_mn=True)
                ref = lambda: torch.matmul(A, B)
            else:
                A = torch.randn(Kd, M, device="cuda").bfloat16(); B = torch.randn(Kd, N, device="cuda").bfloat16()
                C = torch.zeros(M, N, device="cuda")
                f = lambda: K.gemm(A, B, C, a_mn=True, b_mn=True, epi=4, accumulate=1)
                ref = lambda: torch.matmul(A.t(), B)
            fl = 2.0 * M * N * Kd
            K.set_cta_group(1)
            t_1 = timeit(f)
            K.set_cta_group(-1)
            t_ours, t_ref = timeit(f), timeit(ref)
            rows.append({"h": h, "gemm": name, "M": M, "N": N, "K": Kd, "ours_tflops": fl / t_ours / 1e9,
                         "ours_1cta_tflops": fl / t_1 / 1e9, "torch_tflops": fl / t_ref / 1e9})
            print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
