"""TEST INFRASTRUCTURE ONLY — CPU fp32 numerics oracle for the executor.

The reference (pipeblock) has no F/B/W arithmetic, no model and no third-party
math dependency, so loss/gradient parity cannot be pinned on a
reference artefact.  This module is the builder-written restatement the
executor is checked against:

  * ``reference_step``  — plain non-pipelined fp32 autograd over the whole
    model and all microbatches (the ground truth);
  * ``schedule_step``   — the same model executed pass by pass in a
    GridSchedule's global start order with the F / B / W split of the
    reference's pass kinds (model.hpp:15; B = activation gradient,
    W = weight gradient, BW = both), stage inputs/outputs handed over exactly
    along the route dependencies (model.hpp:220-240).  Passes run before their
    prerequisites raise, so this also checks schedule semantics.

Model (matches csrc/exec/executor.cpp): token embedding; per layer pre-norm
RMSNorm (eps 1e-5) -> QKV -> causal MHA (head_dim 128) -> O + residual ->
RMSNorm -> FC1 -> GELU(tanh) -> FC2 + residual; final RMSNorm; untied LM head;
mean cross-entropy over all tokens of the step.  No biases.
"""
from __future__ import annotations

import math
from typing import Dict, Iterable, List, Tuple

import torch
import torch.nn.functional as F


def gelu(x):
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def rmsnorm(x, g, eps=1e-5):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def attention(qkv, mbs, seq, heads):
    T = mbs * seq
    q, k, v = qkv.view(mbs, seq, 3, heads, 128).unbind(2)
    q, k, v = (t.transpose(1, 2) for t in (q, k, v))
    s = q @ k.transpose(-1, -2) / math.sqrt(128)
    mask = torch.triu(torch.ones(seq, seq, dtype=torch.bool, device=qkv.device), 1)
    p = torch.softmax(s.masked_fill(mask, float("-inf")), -1)
    return (p @ v).transpose(1, 2).reshape(T, heads * 128)


def layer_forward(x, p: Dict[str, torch.Tensor], pre: str, cfg):
    a = rmsnorm(x, p[pre + "norm1"])
    qkv = a @ p[pre + "wqkv"].t()
    o = attention(qkv, cfg.micro_batch, cfg.seq, cfg.heads)
    x1 = x + o @ p[pre + "wo"].t()
    b = rmsnorm(x1, p[pre + "norm2"])
    return x1 + gelu(b @ p[pre + "w1"].t()) @ p[pre + "w2"].t()


def stage_layers(cfg, S: int) -> List[int]:
    """Layers per stage: cfg.stage_layers when given (uneven split), else layers // S each."""
    sl = getattr(cfg, "stage_layers", None)
    if sl is not None:
        assert len(sl) == S and sum(sl) == cfg.layers
        return list(sl)
    return [cfg.layers // S] * S


def stage_param_names(cfg, S: int, s: int) -> List[str]:
    Lc = stage_layers(cfg, S)[s - 1]
    names = ["s1.emb"] if s == 1 else []
    for l in range(Lc):
        names += [f"s{s}.l{l}.{w}" for w in ("norm1", "wqkv", "wo", "norm2", "w1", "w2")]
    if s == S:
        names += [f"s{S}.norm", f"s{S}.head"]
    return names


def shapes(cfg, S: int) -> Dict[str, Tuple[int, ...]]:
    h, V = cfg.hidden, cfg.vocab
    out = {}
    for s in range(1, S + 1):
        for n in stage_param_names(cfg, S, s):
            w = n.split(".")[-1]
            out[n] = {"emb": (V, h), "head": (V, h), "norm": (h,), "norm1": (h,), "norm2": (h,), "wqkv": (3 * h, h),
                      "wo": (h, h), "w1": (4 * h, h), "w2": (h, 4 * h)}[w]
    return out


def stage_forward(s: int, S: int, inp, p, cfg, tokens_mb=None, labels_mb=None, loss_scale=1.0):
    """Stage s on one microbatch: returns its output (s < S) or scaled CE sum (s == S)."""
    Lc = stage_layers(cfg, S)[s - 1]
    x = p["s1.emb"][tokens_mb] if s == 1 else inp
    for l in range(Lc):
        x = layer_forward(x, p, f"s{s}.l{l}.", cfg)
    if s < S:
        return x
    logits = rmsnorm(x, p[f"s{S}.norm"]) @ p[f"s{S}.head"].t()
    return F.cross_entropy(logits, labels_mb.long(), reduction="sum") * loss_scale


def rename_for(params: Dict[str, torch.Tensor], cfg, S_from: int, S_to: int, cfg_to=None) -> Dict[str, torch.Tensor]:
    """Map parameter names between stage partitions (global layer index is invariant).
    cfg gives the source split (its stage_layers, if any); cfg_to the target's (default: even)."""
    import types
    first_from = [0]
    for n in stage_layers(cfg, S_from):
        first_from.append(first_from[-1] + n)
    tgt = cfg_to if cfg_to is not None else types.SimpleNamespace(layers=cfg.layers, stage_layers=None)
    owner = []  # global layer -> (stage, local index) in the target split
    for s, n in enumerate(stage_layers(tgt, S_to), 1):
        owner += [(s, l) for l in range(n)]
    out = {}
    for n, t in params.items():
        parts = n.split(".")
        if parts[1] == "emb":
            out["s1.emb"] = t
        elif len(parts) == 2:
            out[f"s{S_to}.{parts[1]}"] = t
        else:
            gl = first_from[int(parts[0][1:]) - 1] + int(parts[1][1:])
            s2, l2 = owner[gl]
            out[f"s{s2}.l{l2}.{parts[2]}"] = t
    return out


def reference_step(params: Dict[str, torch.Tensor], tokens, labels, cfg, S: int, device: str = "cpu"):
    """Non-pipelined fp32 loss and gradients.  params named for an S-stage split.

    device="cuda" runs the same fp32 restatement on the GPU (full-fp32 matmuls, TF32 off) for the
    real-shape parity cases (h up to 6144, s up to 6144) that would take minutes on host cores;
    gradients are returned on the host either way."""
    prec = torch.get_float32_matmul_precision()
    torch.set_float32_matmul_precision("highest")
    try:
        p = {n: t.detach().to(device).float().clone().requires_grad_(True) for n, t in params.items()}
        m, T = tokens.shape
        scale = 1.0 / (m * T)
        total = 0.0
        for mb in range(m):
            x = None
            tok = torch.as_tensor(tokens[mb]).long().to(device)
            lab = torch.as_tensor(labels[mb]).to(device)
            for s in range(1, S + 1):
                x = stage_forward(s, S, x, p, cfg, tok, lab, scale)
            x.backward()
            total += x.item()
        return total, {n: t.grad.detach().cpu().clone() for n, t in p.items()}
    finally:
        torch.set_float32_matmul_precision(prec)


def schedule_step(params: Dict[str, torch.Tensor], tokens, labels, cfg, passes: Iterable, S: int):
    """Execute a GridSchedule's passes in global (start, device) order with split F/B/W."""
    p = {n: t.detach().float().clone() for n, t in params.items()}
    grads = {n: torch.zeros_like(t) for n, t in p.items()}
    m, T = tokens.shape
    scale = 1.0 / (m * T)
    store: Dict[Tuple[int, int], dict] = {}
    total = 0.0
    for op in sorted(passes, key=lambda q: (q.start, q.device, q.stage, q.microbatch)):
        s, mb, kind = op.stage, op.microbatch, op.kind
        if kind == "F":
            if s > 1 and (s - 1, mb) not in store:
                raise RuntimeError(f"F({s},{mb}) before F({s - 1},{mb})")
            leaf = {n: p[n].clone().requires_grad_(True) for n in stage_param_names(cfg, S, s)}
            inp = None if s == 1 else store[(s - 1, mb)]["out"].detach().requires_grad_(True)
            out = stage_forward(s, S, inp, leaf, cfg, torch.as_tensor(tokens[mb]).long(), torch.as_tensor(labels[mb]),
                                scale)
            if s == S:
                total += out.item()
            store[(s, mb)] = {"inp": inp, "out": out, "leaf": leaf}
        else:
            st = store.get((s, mb))
            if st is None:
                raise RuntimeError(f"{kind}({s},{mb}) before its F")
            if kind in ("B", "BW"):
                if s == S:
                    st["gout"] = torch.ones(())
                else:
                    nxt = store.get((s + 1, mb), {})
                    if "gin" not in nxt:
                        raise RuntimeError(f"B({s},{mb}) before B({s + 1},{mb})")
                    st["gout"] = nxt["gin"]
                if s > 1:
                    (st["gin"],) = torch.autograd.grad(st["out"], st["inp"], st["gout"], retain_graph=True)
                st["b_done"] = True
            if kind in ("W", "BW"):
                if not st.get("b_done"):
                    raise RuntimeError(f"W({s},{mb}) before its B")
                names = list(st["leaf"])
                gs = torch.autograd.grad(st["out"], [st["leaf"][n] for n in names], st["gout"], allow_unused=True)
                for n, g in zip(names, gs):
                    if g is not None:
                        grads[n] += g
                st["leaf"] = None
                st["out"] = st["out"].detach()
    return total, grads


def rel_l2(a, b) -> float:
    a, b = torch.as_tensor(a).float().ravel(), torch.as_tensor(b).float().ravel()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def cosine(a, b) -> float:
    a, b = torch.as_tensor(a).float().ravel(), torch.as_tensor(b).float().ravel()
    return float(a @ b / (a.norm() * b.norm()).clamp_min(1e-30))
