"""The CPU numerics oracle: schedule-driven F/B/W execution equals plain autograd,
and out-of-order passes are rejected.  (CPU only; small config.)"""
from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import numerics as N
from paper_2405_15362_b200 import pipeblock as pb

CFG = SimpleNamespace(layers=4, hidden=256, heads=2, seq=128, vocab=512, micro_batch=1)


def make_params(S, seed=0):
    g = torch.Generator().manual_seed(seed)
    out = {}
    for n, shp in N.shapes(CFG, S).items():
        if n.endswith(("norm", "norm1", "norm2")):
            out[n] = 1 + 0.1 * torch.randn(shp, generator=g)
        else:
            out[n] = 0.05 * torch.randn(shp, generator=g)
    return out


def batch(m, seed=1):
    rng = np.random.default_rng(seed)
    t = rng.integers(0, CFG.vocab, size=(m, CFG.seq + 1))
    return t[:, :-1].astype(np.int32), t[:, 1:].astype(np.int32)


@pytest.mark.parametrize("entry,p", [("zb-h1", 1), ("1f1b", 2), ("zb-h1", 4), ("v-min", 2), ("v-half", 2), ("v-zb", 2)])
def test_schedule_step_matches_autograd(entry, p):
    g = pb.assemble(pb.build_entry(entry, p), 4)
    S = g.topology.num_stages
    params = make_params(S)
    tok, lab = batch(4)
    l_ref, g_ref = N.reference_step(params, tok, lab, CFG, S)
    l_sch, g_sch = N.schedule_step(params, tok, lab, CFG, g.passes, S)
    assert abs(l_ref - l_sch) < 1e-5 * abs(l_ref)
    for n in g_ref:
        assert N.rel_l2(g_sch[n], g_ref[n]) < 1e-5, n


def test_partition_invariance():
    p2 = make_params(4)
    p1 = N.rename_for(p2, CFG, 4, 1)
    tok, lab = batch(2)
    l4, g4 = N.reference_step(p2, tok, lab, CFG, 4)
    l1, g1 = N.reference_step(p1, tok, lab, CFG, 1)
    assert abs(l4 - l1) < 1e-6 * abs(l1)
    g4r = N.rename_for(g4, CFG, 4, 1)
    for n in g1:
        assert N.rel_l2(g4r[n], g1[n]) < 1e-5


def test_out_of_order_passes_rejected():
    g = pb.assemble(pb.build_entry("v-half", 2), 2)
    bad = [q._replace(start=-1) if (q.kind == "W" and q.stage == 3 and q.microbatch == 0) else q for q in g.passes]
    tok, lab = batch(2)
    with pytest.raises(RuntimeError, match="before its"):
        N.schedule_step(make_params(4), tok, lab, CFG, bad, 4)


def test_uneven_stage_layers_partition_invariance():
    """Uneven split (fewer layers on the stages carrying embedding / head): same model, same numbers."""
    cfg_u = SimpleNamespace(**vars(CFG), stage_layers=(1, 2, 1))
    even = make_params(1)
    pu = N.rename_for(even, CFG, 1, 3, cfg_to=cfg_u)
    assert sorted(N.shapes(cfg_u, 3)) == sorted(pu)
    tok, lab = batch(2)
    l1, g1 = N.reference_step(even, tok, lab, CFG, 1)
    lu, gu = N.reference_step(pu, tok, lab, cfg_u, 3)
    assert abs(l1 - lu) < 1e-6 * abs(l1)
    back = N.rename_for(gu, cfg_u, 3, 1)
    for n in g1:
        assert N.rel_l2(back[n], g1[n]) < 1e-5, n
    g = pb.assemble(pb.build_entry("1f1b", 3), 3)
    ls, gs = N.schedule_step(pu, tok[:1].repeat(3, 0), lab[:1].repeat(3, 0), cfg_u, g.passes, 3)
    lr, gr = N.reference_step(pu, tok[:1].repeat(3, 0), lab[:1].repeat(3, 0), cfg_u, 3)
    assert abs(ls - lr) < 1e-5 * abs(lr)


def test_balanced_stage_layers():
    """The LM-head stage sheds layers until per-device work (layers + head ~ V/(12h+2s)) evens out."""
    from paper_2405_15362_b200.executor import ModelConfig, balanced_stage_layers
    cfg = ModelConfig(layers=32, hidden=2048, heads=16, seq=2048, vocab=50304)
    v8 = pb.assemble(pb.build_entry("v-half", 8), 16).topology
    L = balanced_stage_layers(cfg, v8)
    assert sum(L) == 32 and min(L) >= 1 and len(L) == 16
    head = cfg.vocab / (12 * cfg.hidden + 2 * cfg.seq)
    load = [0.0] * 8
    for s in range(1, 17):
        load[v8.device_of(s) - 1] += L[s - 1] + (head if s == 16 else 0)
    assert max(load) <= 5.0 + 1e-9            # even split: device 1 carries 4 + 1.75
    assert balanced_stage_layers(cfg, pb.assemble(pb.build_entry("1f1b", 8), 8).topology)[-1] < 4
    big = ModelConfig(layers=32, hidden=6144, heads=48, seq=6144, vocab=50304)  # head < 1 layer: unchanged
    assert balanced_stage_layers(big, v8) == (2,) * 16
