"""ctypes access to the kernel test entry points (include/pipeblock_b200_kernels.h)."""
import ctypes as C

import torch

from paper_2405_15362_b200 import _lib


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def gemm(A, B, C_, *, a_mn=False, b_mn=False, epi=0, C2=None, aux=None, accumulate=0):
    """C (epi)= A . B with A [M,K] (or [K,M] if a_mn) and B [N,K] (or [K,N] if b_mn)."""
    if a_mn:
        K, M = A.shape
    else:
        M, K = A.shape
    N = B.shape[1] if b_mn else B.shape[0]
    L = _lib.lib()
    _lib.check(L.pbt_gemm(M, N, K, _p(A), A.stride(0), int(a_mn), _p(B), B.stride(0), int(b_mn), _p(C_),
                          C_.stride(0), _p(C2), _p(aux), aux.stride(0) if aux is not None else 0, epi, accumulate,
                          _s()))


def row_sumsq(x, ss):
    T, h = x.shape
    _lib.check(_lib.lib().pbt_row_sumsq(_p(x), _f(ss), T, h, _s()))


def gemm_rownorm(A, B, C_, *, b_mn=False, epi=0, C2=None, aux=None, rs=None, ss_out=None, inv_n=0.0, eps=1e-5):
    """gemm with the folded-RMSNorm hooks: row scale rsqrt(rs * inv_n + eps) / residual sum of squares."""
    M, K = A.shape
    N = B.shape[1] if b_mn else B.shape[0]
    _lib.check(_lib.lib().pbt_gemm_rownorm(M, N, K, _p(A), A.stride(0), 0, _p(B), B.stride(0), int(b_mn), _p(C_),
                                           C_.stride(0), _p(C2), _p(aux), aux.stride(0) if aux is not None else 0,
                                           epi, _f(rs), C.c_float(inv_n), C.c_float(eps), _f(ss_out), _s()))


def _f(t):
    return C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_float)) if t is not None else None


def _i(t):
    return C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_int32))


def rmsnorm_fwd(x, g):
    T, h = x.shape
    y = torch.empty_like(x)
    rstd = torch.empty(T, device="cuda", dtype=torch.float32)
    _lib.check(_lib.lib().pbt_rmsnorm_fwd(_p(x), _p(g), _p(y), _f(rstd), T, h, _s()))
    return y, rstd


def rmsnorm_bwd(dy, x, g, rstd, dres=None, dgamma=None):
    T, h = x.shape
    dx = torch.empty_like(x)
    _lib.check(_lib.lib().pbt_rmsnorm_bwd(_p(dy), _p(x), _p(g), _f(rstd), _p(dres), _p(dx), _f(dgamma), T, h, _s()))
    return dx


def rmsnorm_bwd_x(dyp, x, ss, dres=None, eps=1e-5):
    T, h = x.shape
    dx = torch.empty_like(x)
    _lib.check(_lib.lib().pbt_rmsnorm_bwd_x(_p(dyp), _p(x), _f(ss), _p(dres), _p(dx), T, h, C.c_float(eps), _s()))
    return dx


def embed_fwd(tok, emb):
    T, h = tok.numel(), emb.shape[1]
    x = torch.empty(T, h, device="cuda", dtype=torch.bfloat16)
    _lib.check(_lib.lib().pbt_embed_fwd(_i(tok), _p(emb), _p(x), T, h, _s()))
    return x


def embed_bwd(tok, dx, demb):
    _lib.check(_lib.lib().pbt_embed_bwd(_i(tok), _p(dx), _f(demb), tok.numel(), dx.shape[1], _s()))


def cross_entropy(logits, labels, loss, scale):
    T, V = logits.shape
    _lib.check(_lib.lib().pbt_cross_entropy(_p(logits), _i(labels), _f(loss), T, V, C.c_float(scale), _s()))


def adamw(w, wb, g, m, v, lr, b1, b2, eps, wd, step):
    _lib.check(_lib.lib().pbt_adamw(_f(w), _p(wb), _f(g), _f(m), _f(v), C.c_int64(w.numel()), C.c_float(lr),
                                    C.c_float(b1), C.c_float(b2), C.c_float(eps), C.c_float(wd), step, _s()))


def attn_fwd_tc(qkv, batch, seq, heads):
    T = batch * seq
    out = torch.empty(T, heads * 128, device="cuda", dtype=torch.bfloat16)
    lse2 = torch.empty(heads, T, device="cuda", dtype=torch.float32)
    _lib.check(_lib.lib().pbt_attn_fwd_tc(_p(qkv), _p(out), _f(lse2), batch, seq, heads, _s()))
    return out, lse2


def attn_bwd_tc(qkv, out, dout, lse2, batch, seq, heads):
    T = batch * seq
    dsum = torch.empty(heads * T + 64, device="cuda", dtype=torch.float32)  # + the work counter
    dq = torch.empty(T, heads * 128, device="cuda", dtype=torch.float32)
    dqkv = torch.empty_like(qkv)
    _lib.check(_lib.lib().pbt_attn_bwd_tc(_p(qkv), _p(out), _p(dout), _f(lse2), _f(dsum), _f(dq), _p(dqkv), batch,
                                          seq, heads, _s()))
    return dqkv


def set_pair_rows(rows: int) -> None:
    _lib.check(_lib.lib().pbt_gemm_set_pair_rows(rows))


def set_cta_group(cg: int) -> None:
    _lib.check(_lib.lib().pbt_gemm_set_cta_group(cg))
