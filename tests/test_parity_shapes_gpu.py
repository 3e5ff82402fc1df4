"""Executor parity at the BASELINE model shapes: loss and every gradient of
one pipeline step on slices of the real configs, against the fp32 numerics oracle on the same
bf16-valued weights and tokens.

  * config 1 (SURVEY §8d "tiny"): L=8, h=512, 4 heads, s=256, V=1024, mbs=2, V-Half p=4, m=8
  * GPT-1.5B slice: h=2048, 16 heads, s=2048, V=50304, mbs=2, 4 layers, V-Half p=2
  * GPT-6B slice:   h=4096, 32 heads, s=4096, V=50304, mbs=1, 4 layers, V-ZB p=2 (and 1F1B p=2)
  * GPT-14B slice:  h=6144, 48 heads, s=6144, V=50304, mbs=1, 5 layers split (2,1,1,1), V-Min p=2
  * round 2: 14B V-Half p=2; 6B ZB-H1 p=2 with an uneven (3, 2) split; 1.5B interleaved-1F1B p=2 (looped)

The big slices run the oracle's fp32 restatement on the GPU (oracle.numerics.reference_step,
device="cuda", TF32 off): the same arithmetic, minutes faster than host cores.  Tolerances are
SURVEY §8c's (bf16 GPU vs fp32): loss rel <= 5e-3, gradient rel-L2 <= 3e-2, cosine >= 0.999.
"""
import gc

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import numerics as N  # noqa: E402
from paper_2405_15362_b200 import pipeblock as pb  # noqa: E402
from paper_2405_15362_b200.executor import ModelConfig, PipelineExecutor, synthetic_batch  # noqa: E402

LOSS_RTOL = 5e-3
GRAD_REL_L2 = 3e-2
GRAD_COS = 0.999

SLICES = {
    "config1": (ModelConfig(layers=8, hidden=512, heads=4, seq=256, vocab=1024, micro_batch=2, optimizer=False),
                "v-half", 4, 8, "cpu"),
    "1.5b": (ModelConfig(layers=4, hidden=2048, heads=16, seq=2048, vocab=50304, micro_batch=2, optimizer=False),
             "v-half", 2, 4, "cuda"),
    "6b": (ModelConfig(layers=4, hidden=4096, heads=32, seq=4096, vocab=50304, micro_batch=1, optimizer=False),
           "v-zb", 2, 4, "cuda"),
    "6b-1f1b": (ModelConfig(layers=4, hidden=4096, heads=32, seq=4096, vocab=50304, micro_batch=1,
                            optimizer=False), "1f1b", 2, 3, "cuda"),
    "14b": (ModelConfig(layers=5, hidden=6144, heads=48, seq=6144, vocab=50304, micro_batch=1, optimizer=False,
                        stage_layers=(2, 1, 1, 1)), "v-min", 2, 3, "cuda"),
    # round 2: the other schedule families at real layer shapes
    "14b-v-half": (ModelConfig(layers=4, hidden=6144, heads=48, seq=6144, vocab=50304, micro_batch=1,
                               optimizer=False), "v-half", 2, 4, "cuda"),
    "6b-zb-h1-uneven": (ModelConfig(layers=5, hidden=4096, heads=32, seq=4096, vocab=50304, micro_batch=1,
                                    optimizer=False, stage_layers=(3, 2)), "zb-h1", 2, 4, "cuda"),
    "1.5b-interleaved": (ModelConfig(layers=4, hidden=2048, heads=16, seq=2048, vocab=50304, micro_batch=2,
                                     optimizer=False), "interleaved-1f1b", 2, 4, "cuda"),
}


@pytest.mark.parametrize("name", list(SLICES))
def test_real_shape_step_matches_oracle(name):
    cfg, entry, p, m, oracle_dev = SLICES[name]
    sched = pb.assemble(pb.build_entry(entry, p), m)
    S = sched.topology.num_stages
    tokens, labels = synthetic_batch(cfg, m)
    ex = PipelineExecutor(cfg, sched)
    res = ex.step(tokens, labels)
    names = list(ex.params())
    shp = N.shapes(cfg, S)
    assert sorted(names) == sorted(shp)
    weights = {n: torch.from_numpy(ex.get(n, "weight").reshape(shp[n])) for n in names}
    grads = {n: ex.get(n, "grad") for n in names}
    peaks = pb.exact_peak(sched)
    for d, st in res.per_device.items():  # lifespan pool: slots == the reference's exact_peak
        assert st.pool_slots == int(peaks[d - 1])
    del ex
    gc.collect()
    torch.cuda.empty_cache()
    loss_ref, grads_ref = N.reference_step(weights, tokens, labels, cfg, S, device=oracle_dev)
    torch.cuda.empty_cache()
    assert np.isfinite(res.loss)
    assert abs(res.loss - loss_ref) <= LOSS_RTOL * abs(loss_ref), (res.loss, loss_ref)
    worst = []
    for n in names:
        g, r = grads[n], grads_ref[n].numpy().ravel()
        e, c = N.rel_l2(g, r), N.cosine(g, r)
        worst.append((e, n))
        assert e < GRAD_REL_L2, (n, e)
        assert c > GRAD_COS, (n, c)
    print(f"{name}: loss {res.loss:.6f} vs {loss_ref:.6f}; worst grad rel-L2 {max(worst)}")
