"""Executor parity on the B200: loss and every gradient of one pipeline step
vs the CPU fp32 oracle on the same (bf16-valued) weights and tokens, for each
schedule family; measured activation slots vs the reference's exact_peak."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import numerics as N  # noqa: E402
from paper_2405_15362_b200 import pipeblock as pb  # noqa: E402
from paper_2405_15362_b200.executor import ModelConfig, PipelineExecutor, synthetic_batch  # noqa: E402

# tolerances: bf16 activations/weights on the GPU vs fp32 on the CPU
LOSS_RTOL = 5e-3
GRAD_REL_L2 = 3e-2
GRAD_COS = 0.999

CFG = ModelConfig(layers=8, hidden=256, heads=2, seq=256, vocab=1024, micro_batch=2, optimizer=False)
M = 8
CASES = [("zb-h1", 1), ("1f1b", 2), ("zb-h1", 2), ("v-min", 2), ("v-half", 2), ("v-zb", 2), ("v-half", 4),
         ("v-min", 4), ("v-zb", 4), ("1f1b", 4)]

_ref_cache = {}


def oracle(weights, tokens, labels, S):
    key = S
    if key not in _ref_cache:
        w = {n: torch.from_numpy(v.reshape(N.shapes(CFG, S)[n])) for n, v in weights.items()}
        _ref_cache[key] = N.reference_step(w, tokens, labels, CFG, S)
    return _ref_cache[key]


@pytest.mark.parametrize("entry,p", CASES)
def test_step_matches_oracle(entry, p):
    sched = pb.assemble(pb.build_entry(entry, p), M)
    S = sched.topology.num_stages
    ex = PipelineExecutor(CFG, sched)
    tokens, labels = synthetic_batch(CFG, M)
    res = ex.step(tokens, labels)
    names = list(ex.params())
    weights = {n: ex.get(n, "weight") for n in names}
    loss_ref, grads_ref = oracle(weights, tokens, labels, S)
    assert abs(res.loss - loss_ref) <= LOSS_RTOL * abs(loss_ref), (res.loss, loss_ref)
    for n in names:
        g = ex.get(n, "grad")
        r = grads_ref[n].numpy().ravel()
        assert N.rel_l2(g, r) < GRAD_REL_L2, (n, N.rel_l2(g, r))
        assert N.cosine(g, r) > GRAD_COS, (n, N.cosine(g, r))
    # lifespan-bounded pool: slots allocated == predicted exact_peak, all used
    peaks = pb.exact_peak(sched)
    for d, st in res.per_device.items():
        assert st.pool_slots == int(peaks[d - 1])
        assert st.pool_peak == int(peaks[d - 1])
    # measured timeline covers every pass exactly once and respects the grid order per device
    assert sorted((q.stage, q.kind, q.microbatch) for q in res.timeline) == sorted(
        (q.stage, q.kind, q.microbatch) for q in sched.passes)
    for d in range(1, p + 1):
        mine = [q for q in res.timeline if q.device == d]
        grid = sched.device_passes(d)
        assert [(q.stage, q.kind, q.microbatch) for q in mine] == [(q.stage, q.kind, q.microbatch) for q in grid]
        assert all(a.start + a.duration <= b.start + 1e-3 for a, b in zip(mine, mine[1:]))
    assert 0.0 <= res.bubble_rate < 1.0


def test_schedules_agree_on_gpu():
    """Same weights (partition-independent init) and tokens: all schedules give the same gradients."""
    tokens, labels = synthetic_batch(CFG, M)
    base = None
    for entry, p in [("zb-h1", 1), ("v-half", 2), ("v-zb", 4), ("1f1b", 4)]:
        sched = pb.assemble(pb.build_entry(entry, p), M)
        ex = PipelineExecutor(CFG, sched)
        res = ex.step(tokens, labels)
        g = {n: ex.get(n, "grad") for n in ex.params()}
        g1 = N.rename_for({n: torch.from_numpy(v) for n, v in g.items()}, CFG, sched.topology.num_stages, 1)
        if base is None:
            base = (res.loss, g1)
            continue
        assert abs(res.loss - base[0]) < 1e-4 * abs(base[0])
        for n in base[1]:
            assert N.rel_l2(g1[n], base[1][n]) < 2e-3, (entry, p, n)


def test_serial_mode_matches_overlapped():
    import dataclasses
    sched = pb.assemble(pb.build_entry("v-half", 4), M)
    tokens, labels = synthetic_batch(CFG, M)
    a = PipelineExecutor(CFG, sched)
    ra = a.step(tokens, labels)
    b = PipelineExecutor(dataclasses.replace(CFG, serial=True), sched)
    rb = b.step(tokens, labels)
    assert abs(ra.loss - rb.loss) < 1e-5 * abs(ra.loss)
    for n in a.params():
        assert N.rel_l2(a.get(n, "grad"), b.get(n, "grad")) < 1e-3


def test_optimizer_steps_reduce_loss():
    import dataclasses
    cfg = dataclasses.replace(CFG, optimizer=True, lr=1e-3)
    sched = pb.assemble(pb.build_entry("v-zb", 2), M)
    ex = PipelineExecutor(cfg, sched)
    # learnable stream: next token = current + 1 (mod V)
    start = np.random.default_rng(0).integers(0, cfg.vocab, size=(M, 1))
    seqs = (start + np.arange(cfg.tokens_per_microbatch + 1)) % cfg.vocab
    tokens = np.ascontiguousarray(seqs[:, :-1].astype(np.int32))
    labels = np.ascontiguousarray(seqs[:, 1:].astype(np.int32))
    losses = [ex.step(tokens, labels).loss for _ in range(10)]
    assert losses[-1] < losses[0] - 0.5, losses
    assert min(losses[5:]) < min(losses[:5]), losses
    assert all(np.isfinite(losses))


def test_device_inputs_equal_host_inputs():
    sched = pb.assemble(pb.build_entry("v-min", 2), M)
    tokens, labels = synthetic_batch(CFG, M)
    ex = PipelineExecutor(CFG, sched)
    r1 = ex.step(tokens, labels, on_host=True)
    g1 = ex.get("s1.emb", "grad")
    for d in ex.devices:
        d.zero_grads()
    tt, ll = torch.from_numpy(tokens).cuda(), torch.from_numpy(labels).cuda()
    torch.cuda.synchronize()
    r2 = ex.step(tt, ll, on_host=False)
    assert abs(r1.loss - r2.loss) < 1e-6 * abs(r1.loss)
    assert N.rel_l2(ex.get("s1.emb", "grad"), g1) < 1e-5


@pytest.mark.parametrize("entry,p", [("v-half", 4), ("1f1b", 2), ("v-zb", 2)])
def test_isolate_mode_serialises_passes_and_matches(entry, p):
    """PB_FLAG_ISOLATE: one pass at a time over the whole group; same numbers as
    the overlapped run, and the per-pass times replay into a valid timeline."""
    sched = pb.assemble(pb.build_entry(entry, p), M)
    tokens, labels = synthetic_batch(CFG, M)
    a = PipelineExecutor(CFG, sched)
    ra = a.step(tokens, labels)
    b = PipelineExecutor(CFG, sched)
    b.set_flags(timeline=True, isolate=True)
    rb = b.step(tokens, labels)
    rb = b.step(tokens, labels)  # second step: turnstile carries across steps
    assert abs(rb.loss - ra.loss) < 1e-5 * abs(ra.loss)
    for n in a.params():
        assert N.rel_l2(a.get(n, "grad"), b.get(n, "grad") / 2) < 1e-3  # grads accumulate (no optimizer)
    assert len(rb.timeline) == len(sched.passes)
    durs = {(q.device, q.stage, q.kind, q.microbatch): q.duration for q in rb.timeline}
    rep = pb.replay(sched, [durs[(q.device, q.stage, q.kind, q.microbatch)] for q in sched.passes], 0.0)
    assert rep.makespan >= max(rep.busy) > 0
    assert 0.0 <= rep.bubble_rate < 1.0


@pytest.mark.parametrize("entry,p,split", [("v-half", 2, (1, 3, 3, 1)), ("1f1b", 2, (3, 5)), ("v-zb", 4, (1, 1, 1, 1, 1, 1, 1, 1))])
def test_uneven_stage_layers_match_oracle(entry, p, split):
    import dataclasses
    cfg = dataclasses.replace(CFG, stage_layers=split)
    sched = pb.assemble(pb.build_entry(entry, p), M)
    S = sched.topology.num_stages
    ex = PipelineExecutor(cfg, sched)
    tokens, labels = synthetic_batch(cfg, M)
    res = ex.step(tokens, labels)
    names = list(ex.params())
    assert sorted(names) == sorted(N.shapes(cfg, S))
    w = {n: torch.from_numpy(ex.get(n, "weight").reshape(N.shapes(cfg, S)[n])) for n in names}
    loss_ref, grads_ref = N.reference_step(w, tokens, labels, cfg, S)
    assert abs(res.loss - loss_ref) <= LOSS_RTOL * abs(loss_ref), (res.loss, loss_ref)
    for n in names:
        g = ex.get(n, "grad")
        r = grads_ref[n].numpy().ravel()
        assert N.rel_l2(g, r) < GRAD_REL_L2, (n, N.rel_l2(g, r))
    # same model as the even split: the loss does not depend on the partition
    even = PipelineExecutor(CFG, pb.assemble(pb.build_entry("zb-h1", 1), M))
    assert abs(even.step(tokens, labels).loss - res.loss) < 2e-3 * abs(res.loss)


def test_unfolded_gamma_path_matches_oracle(monkeypatch):
    """PB_NO_FOLD=1: per-microbatch gamma reductions instead of the folded projection weights."""
    monkeypatch.setenv("PB_NO_FOLD", "1")
    test_step_matches_oracle("v-half", 2)


@pytest.mark.parametrize("vocab", [1152, 8448])
def test_vocab_half_tile_matches_oracle(vocab):
    """vocab = 128 (mod 256): the LM-head GEMMs run on CTA pairs with a half-empty last tile; at
    vocab >= 8192 the LM-head dX GEMM (K = vocab) takes the 512-row pair tile."""
    import dataclasses
    cfg = dataclasses.replace(CFG, vocab=vocab)
    sched = pb.assemble(pb.build_entry("v-half", 2), M)
    ex = PipelineExecutor(cfg, sched)
    tokens, labels = synthetic_batch(cfg, M)
    res = ex.step(tokens, labels)
    S = sched.topology.num_stages
    w = {n: torch.from_numpy(ex.get(n, "weight").reshape(N.shapes(cfg, S)[n])) for n in ex.params()}
    loss_ref, grads_ref = N.reference_step(w, tokens, labels, cfg, S)
    assert abs(res.loss - loss_ref) <= LOSS_RTOL * abs(loss_ref), (res.loss, loss_ref)
    for n in ex.params():
        assert N.rel_l2(ex.get(n, "grad"), grads_ref[n].numpy().ravel()) < GRAD_REL_L2, n


CFG16 = ModelConfig(layers=16, hidden=256, heads=2, seq=256, vocab=1024, micro_batch=1, optimizer=False)


@pytest.mark.parametrize("entry,p,m,cfg", [
    ("zb-h2", 2, 8, CFG), ("gpipe", 2, 8, CFG), ("eager-1f1b", 2, 8, CFG),   # other straight gallery entries
    ("v-half", 2, 1, CFG), ("v-zb", 4, 3, CFG), ("v-min", 2, 5, CFG),       # m = 1 and m not a multiple of p
    ("v-half", 8, 8, CFG16), ("v-zb", 8, 8, CFG16), ("1f1b", 8, 8, CFG16),  # p = 8: 16 V stages of one layer
    # looped placement (device i holds stages i and d+i; the F(d)->F(d+1) edge wraps to device 1),
    # V with fused backward, two microbatches per block
    ("interleaved-1f1b", 2, 4, CFG), ("interleaved-1f1b", 4, 8, CFG), ("interleaved-1f1b-uniform", 4, 8, CFG),
    ("interleaved-low-mem", 2, 6, CFG), ("1f1b-v", 2, 8, CFG), ("1f1b-v", 4, 4, CFG), ("zb-2-3", 2, 8, CFG),
    ("zb-2-3", 4, 4, CFG),
])
def test_more_schedules_match_oracle(entry, p, m, cfg):
    """Executor parity beyond the main sweep: the straight zb-h2 / gpipe / eager-1f1b entries,
    microbatch counts below or not divisible by p, and p = 8 (all pipeline devices on one GPU)."""
    sched = pb.assemble(pb.build_entry(entry, p), m)
    S = sched.topology.num_stages
    ex = PipelineExecutor(cfg, sched)
    tokens, labels = synthetic_batch(cfg, m)
    res = ex.step(tokens, labels)
    names = list(ex.params())
    w = {n: torch.from_numpy(ex.get(n, "weight").reshape(N.shapes(cfg, S)[n])) for n in names}
    loss_ref, grads_ref = N.reference_step(w, tokens, labels, cfg, S)
    assert abs(res.loss - loss_ref) <= LOSS_RTOL * abs(loss_ref), (res.loss, loss_ref)
    for n in names:
        g, r = ex.get(n, "grad"), grads_ref[n].numpy().ravel()
        assert N.rel_l2(g, r) < GRAD_REL_L2, (n, N.rel_l2(g, r))
        assert N.cosine(g, r) > GRAD_COS, (n, N.cosine(g, r))
    peaks = pb.exact_peak(sched)
    for d, st in res.per_device.items():
        assert st.pool_slots == int(peaks[d - 1]) and st.pool_peak == int(peaks[d - 1])


@pytest.mark.parametrize("on_host", [True, False])
@pytest.mark.parametrize("what,bad", [("tokens", 1024), ("labels", -1), ("tokens", 1 << 30)])
def test_out_of_range_ids_rejected(on_host, what, bad):
    """Ids index the embedding rows and the logits: an id outside [0, vocab) is PB_EINVAL, never an
    out-of-bounds read or scatter-add (host inputs: rejected before enqueue; device inputs: the
    kernels skip the row, flag it, and the step's sync raises). A following valid step is unaffected."""
    from paper_2405_15362_b200._lib import PipeblockError
    sched = pb.assemble(pb.build_entry("v-half", 2), M)
    tokens, labels = synthetic_batch(CFG, M)
    ex = PipelineExecutor(CFG, sched)
    ref = ex.step(tokens, labels).loss
    for d in ex.devices:
        d.zero_grads()
    bt, bl = tokens.copy(), labels.copy()
    (bt if what == "tokens" else bl)[3, 17] = bad
    if not on_host:
        bt, bl = torch.from_numpy(bt).cuda(), torch.from_numpy(bl).cuda()
        torch.cuda.synchronize()
    with pytest.raises(PipeblockError, match="outside \\[0, 1024\\)"):
        ex.step(bt, bl, on_host=on_host)
    for d in ex.devices:
        d.zero_grads()
    again = ex.step(tokens, labels).loss
    assert abs(again - ref) < 1e-6 * abs(ref)


def test_solo_device_probe_and_memory_accounting():
    """PB_FLAG_SOLO: one device of a p=4 V-Half pipeline runs its own op list alone (no peers) at its
    real footprint; pb_exec_memory reports the allocation by category and the device high-water."""
    import dataclasses
    from paper_2405_15362_b200.executor import DeviceExecutor
    sched = pb.assemble(pb.build_entry("v-half", 4), M)
    tokens, labels = synthetic_batch(CFG, M)
    peaks = pb.exact_peak(sched)
    for d in (1, 3):
        ex = DeviceExecutor(dataclasses.replace(CFG, solo=True), sched, d, 0)
        tl, st = ex.step(tokens, labels)
        assert [(q.stage, q.kind, q.microbatch) for q in tl] == \
            [(q.stage, q.kind, q.microbatch) for q in sched.device_passes(d)]
        assert st.pool_slots == int(peaks[d - 1]) and st.peer_bytes == 0
        mem = ex.memory()
        assert mem["activation_pool"] == st.slot_bytes * st.pool_slots
        assert (mem["head_pool"] > 0) == (d == 1)  # V: device 1 holds stage 2p (LM head)
        parts = ("weights", "grads", "optimizer", "activation_pool", "head_pool", "transfer", "scratch")
        assert sum(mem[k] for k in parts) == mem["executor_total"]
        assert mem["device_used_high"] >= mem["device_used_at_create"] + mem["executor_total"]
        assert mem["device_used_high"] <= mem["device_total"]
        del ex


def test_out_of_memory_is_reported_and_released():
    """A pipeline device that does not fit in HBM fails pb_exec_create with PB_ECUDA and a message
    naming the allocation, and gives back everything it had allocated (1F1B device 1 of the 14B
    model at p=8 with micro-batch 5: ~8 x 4 layer-slots of 7.9 GB on top of ~44 GB of weights/state)."""
    import gc
    from paper_2405_15362_b200._lib import PipeblockError
    from paper_2405_15362_b200.executor import DeviceExecutor
    cfg = ModelConfig(layers=32, hidden=6144, heads=48, seq=6144, vocab=50304, micro_batch=5, solo=True)
    sched = pb.assemble(pb.build_entry("1f1b", 8), 64)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    with pytest.raises(PipeblockError, match="out of device memory allocating activation pool"):
        DeviceExecutor(cfg, sched, 1, 0)
    gc.collect()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free1 >= free0 - (64 << 20)


def test_search_winner_from_measured_profile_matches_oracle():
    """§8f row 2: the adaptive search (search.hpp:235) driven by MEASURED per-kind pass times; its winner
    block, assembled at the step's microbatch count, runs on the executor unchanged and matches the oracle."""
    base = PipelineExecutor(CFG, pb.assemble(pb.build_entry("zb-h1", 1), M))
    tokens, labels = synthetic_batch(CFG, M)
    base.step(tokens, labels)
    tl = base.step(tokens, labels).timeline
    mean = {k: float(np.mean([q.duration for q in tl if q.kind == k])) for k in ("F", "B", "W")}
    prof = pb.RunTimeProfile(mean["F"] / 8, mean["B"] / 8, mean["W"] / 8, 0.0)  # one pipeline stage = 1/8 of the model
    r = pb.search(pb.SearchSpec(d=2, profile=prof, memory_limit=6.0, delta_max=4, tau_max=4))
    assert r.feasible and r.exact_peak <= 6.0
    sched = pb.search_assemble(2, r.best, M)
    S = sched.topology.num_stages
    ex = PipelineExecutor(CFG, sched)
    res = ex.step(tokens, labels)
    w = {n: torch.from_numpy(ex.get(n, "weight").reshape(N.shapes(CFG, S)[n])) for n in ex.params()}
    loss_ref, grads_ref = N.reference_step(w, tokens, labels, CFG, S)
    assert abs(res.loss - loss_ref) <= LOSS_RTOL * abs(loss_ref), (res.loss, loss_ref)
    for n in ex.params():
        assert N.rel_l2(ex.get(n, "grad"), grads_ref[n].numpy().ravel()) < GRAD_REL_L2, n
    peaks = pb.exact_peak(sched)
    for d, st in res.per_device.items():
        assert st.pool_slots == int(peaks[d - 1])


@pytest.mark.parametrize("entry,p,m", [("gems", 2, 4), ("chimera", 2, 4), ("chimera", 4, 8), ("gems", 3, 6)])
def test_twin_schedules_match_oracle(entry, p, m):
    """gems / chimera (twin topology: two routes over two weight replicas, gallery.hpp:252-326): every
    microbatch runs its route's stages; at the end of the step the replicas exchange gradients, so both
    copies of every model stage carry the gradient of the whole batch.  Reference: the same model with
    d stages trained on all m microbatches (oracle.numerics.reference_step)."""
    sched = pb.assemble(pb.build_entry(entry, p), m)
    S = sched.topology.num_stages
    Sm = S // 2
    cfg = ModelConfig(layers=2 * Sm, hidden=256, heads=2, seq=256, vocab=1024, micro_batch=1, optimizer=False)
    ex = PipelineExecutor(cfg, sched)
    tokens, labels = synthetic_batch(cfg, m)
    res = ex.step(tokens, labels)

    def model_name(n):
        s, rest = n.split(".", 1)
        k = int(s[1:])
        return f"s{k - Sm if k > Sm else k}.{rest}"

    names = list(ex.params())
    shp = N.shapes(cfg, Sm)
    assert sorted({model_name(n) for n in names}) == sorted(shp)
    w = {model_name(n): torch.from_numpy(ex.get(n, "weight").reshape(shp[model_name(n)])) for n in names
         if int(n.split(".")[0][1:]) <= Sm}
    for n in names:  # replicas start identical (init ids follow the model layer)
        assert np.array_equal(ex.get(n, "weight"), w[model_name(n)].numpy().ravel()), n
    loss_ref, grads_ref = N.reference_step(w, tokens, labels, cfg, Sm)
    assert abs(res.loss - loss_ref) <= LOSS_RTOL * abs(loss_ref), (res.loss, loss_ref)
    for n in names:
        g, r = ex.get(n, "grad"), grads_ref[model_name(n)].numpy().ravel()
        assert N.rel_l2(g, r) < GRAD_REL_L2, (n, N.rel_l2(g, r))
    for n in names:  # both copies hold the same summed gradient
        k = int(n.split(".")[0][1:])
        if k <= Sm:
            twin_n = f"s{k + Sm}." + n.split(".", 1)[1]
            assert np.array_equal(ex.get(n, "grad"), ex.get(twin_n, "grad")), n
    peaks = pb.exact_peak(sched)
    for d, st in res.per_device.items():
        assert st.pool_slots == int(peaks[d - 1])


def test_twin_optimizer_keeps_replicas_identical():
    """Two AdamW steps on a chimera pipeline: the replicas see the same summed gradient, so their
    weights stay bit-identical and the loss goes down."""
    sched = pb.assemble(pb.build_entry("chimera", 2), 4)
    cfg = ModelConfig(layers=4, hidden=256, heads=2, seq=256, vocab=1024, micro_batch=1, optimizer=True, lr=1e-3)
    ex = PipelineExecutor(cfg, sched)
    tokens, labels = synthetic_batch(cfg, 4)
    l0 = ex.step(tokens, labels).loss
    ex.step(tokens, labels)
    l2 = ex.step(tokens, labels).loss
    assert l2 < l0, (l0, l2)
    for n in ex.params():
        k = int(n.split(".")[0][1:])
        if k <= 2:
            assert np.array_equal(ex.get(n, "weight"), ex.get(f"s{k + 2}." + n.split(".", 1)[1], "weight")), n
