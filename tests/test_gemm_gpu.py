"""tcgen05 GEMM vs torch fp32 on the same bf16 inputs (all three pass shapes)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from tests import kernels as K  # noqa: E402


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


def gelu(x):
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


SHAPES = [(128, 128, 64), (256, 384, 128), (512, 1024, 512), (2048, 6144, 2048), (384, 2304, 768), (256, 256, 64),
          (1024, 768, 320)]


@pytest.fixture(params=[1, 2], ids=["cta1", "cta2"], autouse=True)
def cta_group(request):
    K.set_cta_group(request.param)
    yield request.param
    K.set_cta_group(-1)


@pytest.mark.parametrize("M,N,Kd", SHAPES)
def test_forward_shape(M, N, Kd):
    g = torch.Generator(device="cuda").manual_seed(M + N + Kd)
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    W = torch.randn(N, Kd, device="cuda", generator=g).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(A, W, C)
    torch.cuda.synchronize()
    ref = A.float() @ W.float().t()
    assert rel(C, ref) < 4e-3


@pytest.mark.parametrize("M,N,Kd", SHAPES)
def test_backward_shape(M, N, Kd):
    # dX[M,N] = dY[M,K] . W[K,N]  with W stored [K][N] (MN-major B)
    g = torch.Generator(device="cuda").manual_seed(7 + M)
    dY = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    W = torch.randn(Kd, N, device="cuda", generator=g).bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(dY, W, C, b_mn=True)
    torch.cuda.synchronize()
    assert rel(C, dY.float() @ W.float()) < 4e-3


@pytest.mark.parametrize("M,N,Kd", SHAPES)
def test_weight_shape_accumulate(M, N, Kd):
    # dW[M,N] += dY^T . X with dY stored [K][M], X stored [K][N]
    g = torch.Generator(device="cuda").manual_seed(11 + N)
    dY = torch.randn(Kd, M, device="cuda", generator=g).bfloat16()
    X = torch.randn(Kd, N, device="cuda", generator=g).bfloat16()
    C = torch.randn(M, N, device="cuda", generator=g)
    C0 = C.clone()
    K.gemm(dY, X, C, a_mn=True, b_mn=True, epi=4, accumulate=1)
    torch.cuda.synchronize()
    assert rel(C, C0 + dY.float().t() @ X.float()) < 1e-4 * max(1.0, Kd / 64)
    K.gemm(dY, X, C, a_mn=True, b_mn=True, epi=4, accumulate=0)
    torch.cuda.synchronize()
    assert rel(C, dY.float().t() @ X.float()) < 1e-5


def test_fused_epilogues():
    g = torch.Generator(device="cuda").manual_seed(3)
    M, N, Kd = 256, 512, 256
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    W = torch.randn(N, Kd, device="cuda", generator=g).bfloat16() * 0.1
    u = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    gg = torch.empty_like(u)
    K.gemm(A, W, u, epi=1, C2=gg)
    R = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    out = torch.empty_like(u)
    K.gemm(A, W, out, epi=2, aux=R)
    Wt = torch.randn(Kd, N, device="cuda", generator=g).bfloat16() * 0.1
    dg = torch.empty_like(u)
    K.gemm(A, Wt, dg, b_mn=True, epi=3, aux=u)
    torch.cuda.synchronize()
    ref_u = A.float() @ W.float().t()
    assert rel(u, ref_u) < 4e-3
    assert rel(gg, gelu(u.float())) < 4e-3
    assert rel(out, ref_u + R.float()) < 4e-3
    x = u.float().requires_grad_(True)
    (gl,) = torch.autograd.grad(gelu(x), x, torch.ones_like(x))
    assert rel(dg, (A.float() @ Wt.float()) * gl) < 5e-3


def test_rejects_bad_shapes():
    A = torch.zeros(100, 64, device="cuda", dtype=torch.bfloat16)
    W = torch.zeros(128, 64, device="cuda", dtype=torch.bfloat16)
    C = torch.zeros(100, 128, device="cuda", dtype=torch.bfloat16)
    from paper_2405_15362_b200._lib import ScheduleError
    with pytest.raises(ScheduleError):
        K.gemm(A, W, C)


@pytest.mark.parametrize("M,N,Kd", [(512, 2048, 256), (4096, 2048, 2048), (256, 768, 128)])
def test_folded_rmsnorm_epilogues(cta_group, M, N, Kd):
    """Folded RMSNorm hooks: the residual epilogue's per-row sum of squares of its bf16 outputs
    (atomic over the column tiles), and the row scale rsqrt(ss / n + eps) applied by the store /
    GELU / dGELU epilogues of the consuming GEMMs."""
    g = torch.Generator(device="cuda").manual_seed(M + N + Kd)
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    W = torch.randn(N, Kd, device="cuda", generator=g).bfloat16() * 0.05
    R = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ss = torch.full((M,), 0.5, device="cuda")  # overwritten
    K.gemm_rownorm(A, W, out, epi=2, aux=R, ss_out=ss)
    ss2 = torch.full((M,), -1.0, device="cuda")
    K.gemm_rownorm(A, W, out, epi=2, aux=R, ss_out=ss2)  # the row-group counters reset themselves
    ss_k = torch.empty(M, device="cuda")
    K.row_sumsq(out, ss_k)
    torch.cuda.synchronize()
    assert rel(out, A.float() @ W.float().t() + R.float()) < 4e-3
    assert rel(ss, out.float().pow(2).sum(1)) < 1e-5
    # deterministic, and bit-identical to the standalone statistic of a stage's input rows
    assert torch.equal(ss, ss2) and torch.equal(ss, ss_k)
    # consumer: rows of X scaled by rstd(ss) through the epilogue == GEMM of the normalised rows
    X = out
    W2 = torch.randn(Kd, N, device="cuda", generator=g).bfloat16() * 0.05
    rstd = torch.rsqrt(ss / N + 1e-5)
    xhat = X.float() * rstd[:, None]
    st = torch.empty(M, Kd, device="cuda", dtype=torch.bfloat16)
    K.gemm_rownorm(X, W2, st, rs=ss, inv_n=1.0 / N)
    u = torch.empty_like(st)
    gl = torch.empty_like(st)
    K.gemm_rownorm(X, W2, u, epi=1, C2=gl, rs=ss, inv_n=1.0 / N)
    Wt = W2.t().contiguous()  # [N][Kd]: B MN-major for the dGELU (B-pass) shape
    dg = torch.empty_like(st)
    K.gemm_rownorm(X, Wt, dg, b_mn=True, epi=3, aux=u, rs=ss, inv_n=1.0 / N)
    torch.cuda.synchronize()
    ref = xhat @ W2.float().t()
    assert rel(st, ref) < 5e-3
    assert rel(u, ref) < 5e-3 and rel(gl, gelu(u.float())) < 5e-3
    x = u.float().requires_grad_(True)
    (gp,) = torch.autograd.grad(gelu(x), x, torch.ones_like(x))
    assert rel(dg, ref * gp) < 6e-3


@pytest.mark.parametrize("M,N,Kd", [(4096, 50304, 256), (640, 896, 128)])
def test_half_empty_last_tile(M, N, Kd):
    """M or N = 128 (mod 256) on CTA pairs (the LM head: V = 50304): zero-filled loads, skipped stores."""
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    W = torch.randn(N, Kd, device="cuda", generator=g).bfloat16()
    guard = torch.full((M + 256, N + 256), 7.0, device="cuda", dtype=torch.bfloat16)
    C = guard[:M, :N]
    K.gemm(A, W, C)
    Wt = torch.randn(Kd, M, device="cuda", generator=g).bfloat16()
    X = torch.randn(Kd, N, device="cuda", generator=g).bfloat16()
    D = torch.zeros(M, N, device="cuda")
    K.gemm(Wt, X, D, a_mn=True, b_mn=True, epi=4, accumulate=1)
    torch.cuda.synchronize()
    assert rel(C, A.float() @ W.float().t()) < 4e-3
    assert (guard[M:, :] == 7.0).all() and (guard[:, N:] == 7.0).all()  # nothing written outside
    assert rel(D, Wt.float().t() @ X.float()) < 1e-4 * max(1.0, Kd / 64)


@pytest.mark.parametrize("M,N,Kd", [(512, 256, 128), (1024, 768, 384), (2048, 2048, 1024), (512, 6144, 512)])
def test_pair_512_row_tiles(cta_group, M, N, Kd):
    """512 x 256 CTA-pair tiles (two 128-row A sub-tiles per CTA, accumulators in all 512 TMEM
    columns): F (store / GELU / residual), B (store / dGELU) and W (fp32 accumulate) operand majors."""
    if cta_group != 2:
        pytest.skip("a CTA-pair variant")
    g = torch.Generator(device="cuda").manual_seed(M + 2 * N + Kd)
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    W = torch.randn(N, Kd, device="cuda", generator=g).bfloat16()
    Wt = W.t().contiguous()
    R = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    At = A.t().contiguous()
    X = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    K.set_pair_rows(512)
    try:
        u = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        gg = torch.empty_like(u)
        K.gemm(A, W, u, epi=1, C2=gg)
        res = torch.empty_like(u)
        K.gemm(A, W, res, epi=2, aux=R)
        st = torch.empty_like(u)
        K.gemm(A, Wt, st, b_mn=True)
        dg = torch.empty_like(u)
        K.gemm(A, Wt, dg, b_mn=True, epi=3, aux=u)
        C32 = torch.ones(Kd, N, device="cuda")
        K.gemm(A, X, C32, a_mn=True, b_mn=True, epi=4, accumulate=1)  # C += A^T X, A stored [M][Kd] = [K][M']
        torch.cuda.synchronize()
    finally:
        K.set_pair_rows(-1)
    ref = A.float() @ W.float().t()
    assert rel(u, ref) < 4e-3
    assert rel(gg, gelu(u.float())) < 4e-3
    assert rel(res, ref + R.float()) < 4e-3
    assert rel(st, ref) < 4e-3
    x = u.float().requires_grad_(True)
    (gl,) = torch.autograd.grad(gelu(x), x, torch.ones_like(x))
    assert rel(dg, ref * gl) < 5e-3
    assert rel(C32, 1 + At.float() @ X.float()) < 1e-4
