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


# pass shapes whose tile count leaves a ragged last wave on 74 CTA pairs -> stream-K split tiles
SK_SHAPES = [(2048, 2048, 8192), (2048, 2048, 2048), (2048, 6144, 2048), (2048, 8192, 2048), (4096, 2048, 512), (4096, 2048, 8192), (4096, 6144, 2048)]


@pytest.fixture(params=[0, 1, 2], ids=["tiles", "streamk", "hybrid"])
def stream_k(request):
    K.set_stream_k(request.param)
    yield request.param
    K.set_stream_k(-1)


@pytest.mark.parametrize("M,N,Kd", SK_SHAPES)
def test_stream_k_epilogues(M, N, Kd, stream_k):
    g = torch.Generator(device="cuda").manual_seed(M * 3 + N + Kd)
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    W = torch.randn(N, Kd, device="cuda", generator=g).bfloat16() * 0.05
    ref = A.float() @ W.float().t()
    u = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    gg = torch.empty_like(u)
    K.gemm(A, W, u, epi=1, C2=gg)
    R = torch.randn(M, N, device="cuda", generator=g).bfloat16()
    out = torch.empty_like(u)
    K.gemm(A, W, out, epi=2, aux=R)
    Wt = W.t().contiguous()
    dg = torch.empty_like(u)
    K.gemm(A, Wt, dg, b_mn=True, epi=3, aux=u)
    C32 = torch.zeros(M, N, device="cuda")
    K.gemm(A, W, C32, epi=4, accumulate=1)
    K.gemm(A, W, C32, epi=4, accumulate=1)
    torch.cuda.synchronize()
    assert rel(u, ref) < 4e-3
    assert rel(gg, gelu(u.float())) < 4e-3
    assert rel(out, ref + R.float()) < 4e-3
    x = u.float().requires_grad_(True)
    (gl,) = torch.autograd.grad(gelu(x), x, torch.ones_like(x))
    assert rel(dg, ref * gl) < 5e-3
    assert rel(C32, 2 * ref) < 1e-4
    # deterministic: same inputs, same bits
    u2 = torch.empty_like(u)
    K.gemm(A, W, u2, epi=1, C2=gg)
    torch.cuda.synchronize()
    assert torch.equal(u, u2)


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


@pytest.mark.parametrize("bn", [192, 160])
@pytest.mark.parametrize("M,N,Kd", [(512, 2048, 256), (256, 6144, 128), (768, 1024, 320), (256, 384, 64)])
@pytest.mark.parametrize("epi", ["store", "gelu", "resid"])
def test_forward_narrow_tiles(cta_group, bn, M, N, Kd, epi):
    """F-pass pair GEMMs on 256 x 192 / 256 x 160 tiles (gemm_f_bn): partial last column tile,
    GELU and residual epilogues."""
    if cta_group != 2:
        pytest.skip("narrow tiles are a CTA-pair variant")
    g = torch.Generator(device="cuda").manual_seed(3 * M + N + bn)
    A = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
    W = torch.randn(N, Kd, device="cuda", generator=g).bfloat16()
    C = torch.full((M, N + 64), 7.0, device="cuda", dtype=torch.bfloat16)  # padded: nothing past N is written
    C2 = torch.full((M, N + 64), 7.0, device="cuda", dtype=torch.bfloat16)
    aux = torch.randn(M, N + 64, device="cuda", generator=g).bfloat16()
    K.set_tile_n(bn)
    try:
        if epi == "store":
            K.gemm(A, W, C[:, :N])
        elif epi == "gelu":
            K.gemm(A, W, C[:, :N], epi=1, C2=C2[:, :N])
        else:
            K.gemm(A, W, C[:, :N], epi=2, aux=aux[:, :N])
        torch.cuda.synchronize()
    finally:
        K.set_tile_n(0)
    ref = A.float() @ W.float().t()
    if epi == "resid":
        ref = ref + aux[:, :N].float()
    assert rel(C[:, :N], ref) < 4e-3
    assert bool((C[:, N:] == 7.0).all())
    if epi == "gelu":
        assert rel(C2[:, :N], gelu(C[:, :N].float())) < 4e-3
        assert bool((C2[:, N:] == 7.0).all())


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
