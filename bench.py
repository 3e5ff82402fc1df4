"""Benchmark: one pipeline training step (all F/B/W passes of the schedule +
AdamW) of a GPT on B200s, driven by the reference's schedule API.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)

Workload (BASELINE.json configs[2]): GPT ~1.5B (L=32, h=2048, 16 heads,
seq 2048, vocab 50304), bf16, synthetic tokens, m=32 microbatches of 2
sequences per step (global batch 64 x 2048 tokens, fixed as N grows ->
"strong" scaling; micro-batch 2 measured +10% tokens/s over 1 at N=1).  N=1 runs zb-h1 with d=1 (all stages serialised; the
V schedules need d >= 2), N>1 runs V-Half with p=N.  A step is every pass of
the reference's assemble(build_entry(...), m) op order plus the optimizer.

Prints ONE JSON line on rank 0 (see README/DESIGN for the keys).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/sec & bubble rate at 1/2/4/8 B200; peak activation mem vs 1F1B"
CONFIGS = {
    "1.5b": dict(layers=32, hidden=2048, heads=16, seq=2048, vocab=50304),
    "6b": dict(layers=32, hidden=4096, heads=32, seq=4096, vocab=50304),
    "14b": dict(layers=32, hidden=6144, heads=48, seq=6144, vocab=50304),
    "tiny": dict(layers=8, hidden=512, heads=4, seq=256, vocab=1024),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="1.5b", choices=sorted(CONFIGS))
    ap.add_argument("--schedule", default=None, help="gallery entry (default zb-h1 at N=1, v-half at N>1)")
    ap.add_argument("--microbatches", type=int, default=32)
    ap.add_argument("--micro-batch", type=int, default=2)
    ap.add_argument("--cpu-sample-s", type=float, default=20.0, help="target seconds of CPU baseline work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--compare", nargs="+", default=None,
                    help="schedules run after the headline one in the same process group (default at N>1: 1f1b, "
                         "v-zb, v-half, + v-min for --model 14b; 'none' to skip)")
    ap.add_argument("--even-split", action="store_true",
                    help="layers / num_stages per stage (default: balance the LM-head stage, N > 1)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines = gpu, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() in ("active", "0x1") or v.startswith("Active"):
                    reasons.add(n)
        load = [x for x in sm if mx and x > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ---------------------------------------------------------------- CPU baseline (oracle port)
def _median_time(fn, budget_s, max_n=20):
    fn()  # warm-up (thread pool, allocator)
    times = []
    t_end = time.perf_counter() + budget_s
    while True:
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end or len(times) >= max_n:
            return statistics.median(times), len(times)


def cpu_baseline(mcfg, args, target_s=None, tiny_e2e=True):
    """Bounded CPU sample of the same workload on all host threads (torch CPU fp32, the oracle port):
    per sequence, one transformer layer F + B + W and the final norm + LM head + cross-entropy F + B + W;
    AdamW over one layer's parameters.  The step is extrapolated as
        (m * mbs) * (L * t_layer + t_head) + n_params * t_adamw_per_param
    and, separately, config 1 (L=8, h=512, 4 heads, s=256, V=1024, mbs=2, V-Half p=4, m=8) runs END TO END
    through oracle.numerics.schedule_step (the GridSchedule executed pass by pass) + AdamW."""
    import torch
    from types import SimpleNamespace

    from oracle import numerics as N

    target_s = args.cpu_sample_s if target_s is None else target_s
    torch.set_num_threads(os.cpu_count() or 1)
    cfg = SimpleNamespace(layers=1, hidden=mcfg["hidden"], heads=mcfg["heads"], seq=mcfg["seq"],
                          vocab=mcfg["vocab"], micro_batch=1)
    h, V, T, L = cfg.hidden, cfg.vocab, cfg.seq, mcfg["layers"]
    g = torch.Generator().manual_seed(0)
    shp = {"wqkv": (3 * h, h), "wo": (h, h), "w1": (4 * h, h), "w2": (h, 4 * h)}
    p = {f"s1.l0.{n}": (0.02 * torch.randn(s, generator=g)).requires_grad_(True) for n, s in shp.items()}
    p["s1.l0.norm1"] = torch.ones(h, requires_grad=True)
    p["s1.l0.norm2"] = torch.ones(h, requires_grad=True)
    head = {"norm": torch.ones(h, requires_grad=True), "head": (0.02 * torch.randn(V, h, generator=g)).requires_grad_(True)}
    x = torch.randn(T, h, requires_grad=True)
    lab = torch.randint(0, V, (T,), generator=g)

    def layer():
        y = N.layer_forward(x, p, "s1.l0.", cfg)                           # F
        gy = torch.randn_like(y)
        torch.autograd.grad(y, x, gy, retain_graph=True)                   # B
        torch.autograd.grad(y, list(p.values()), gy)                       # W

    def lm_head():
        z = N.rmsnorm(x, head["norm"]) @ head["head"].t()
        loss = torch.nn.functional.cross_entropy(z, lab, reduction="sum")
        torch.autograd.grad(loss, [x], retain_graph=True)
        torch.autograd.grad(loss, list(head.values()))

    flat = [t.detach() for t in p.values()]
    st = [(torch.zeros_like(t), torch.zeros_like(t), torch.randn_like(t)) for t in flat]

    def adamw():
        for w, (m1, m2, gr) in zip(flat, st):
            m1.mul_(0.9).add_(gr, alpha=0.1)
            m2.mul_(0.95).addcmul_(gr, gr, value=0.05)
            w.addcdiv_(m1, m2.sqrt().add_(1e-8), value=-1e-4)

    t_layer, n1 = _median_time(layer, 0.5 * target_s)
    t_head, n2 = _median_time(lm_head, 0.3 * target_s)
    t_adam, n3 = _median_time(adamw, 0.1 * target_s)
    n_layer_params = sum(t.numel() for t in flat)
    n_params = L * (12 * h * h + 2 * h) + 2 * V * h + h
    seqs = args.microbatches * args.micro_batch
    t_step = seqs * (L * t_layer + t_head) + n_params * t_adam / n_layer_params
    out = {"value": seqs * T / t_step, "unit": "tokens/s", "cores": torch.get_num_threads(), "kind": "port",
           "sample": f"per sequence ({T} tokens): 1 of {L} layers F+B+W (median of {n1}), final norm + LM head + CE "
                     f"F+B+W (median of {n2}), AdamW on one layer's {n_layer_params} parameters (median of {n3}); "
                     f"step extrapolated to {seqs} sequences x {L} layers + head and AdamW over {n_params} parameters "
                     f"(fp32, oracle/numerics.py on torch CPU)",
           "ms_per_step_extrapolated": t_step * 1e3,
           "parts_ms": {"layer_fbw_per_seq": t_layer * 1e3, "head_fbw_per_seq": t_head * 1e3,
                        "adamw_per_layer_params": t_adam * 1e3}}
    if tiny_e2e:
        out["tiny_e2e"] = cpu_tiny_e2e()
    return out


def cpu_tiny_e2e():
    """BASELINE configs[0] / SURVEY §8d config 1 end to end on host cores: V-Half p=4 m=8, L=8, h=512,
    4 heads, s=256, V=1024, mbs=2; the whole GridSchedule pass by pass (oracle.numerics.schedule_step)
    plus AdamW over every parameter."""
    import torch
    from types import SimpleNamespace

    from oracle import numerics as N
    from paper_2405_15362_b200 import pipeblock as pb

    cfg = SimpleNamespace(layers=8, hidden=512, heads=4, seq=256, vocab=1024, micro_batch=2, stage_layers=None)
    sched = pb.assemble(pb.build_entry("v-half", 4), 8)
    S = sched.topology.num_stages
    g = torch.Generator().manual_seed(0)
    w = {n: (0.02 * torch.randn(s, generator=g)) for n, s in N.shapes(cfg, S).items()}
    tok = torch.randint(0, cfg.vocab, (8, cfg.seq * cfg.micro_batch), generator=g)
    lab = torch.randint(0, cfg.vocab, (8, cfg.seq * cfg.micro_batch), generator=g)
    state = {n: (torch.zeros_like(t), torch.zeros_like(t)) for n, t in w.items()}

    def step():
        _, grads = N.schedule_step(w, tok.numpy(), lab.numpy(), cfg, sched.passes, S)
        for n, gr in grads.items():
            m1, m2 = state[n]
            m1.mul_(0.9).add_(gr, alpha=0.1)
            m2.mul_(0.95).addcmul_(gr, gr, value=0.05)
            w[n].addcdiv_(m1, m2.sqrt().add_(1e-8), value=-1e-4)

    t, n = _median_time(step, 3.0, max_n=5)
    return {"value": 8 * cfg.seq * cfg.micro_batch / t, "unit": "tokens/s", "ms_per_step": t * 1e3,
            "cores": torch.get_num_threads(), "runs": n,
            "workload": "config 1: gpt L=8 h=512 4 heads s=256 V=1024, v-half p=4 m=8 mbs=2, whole step + AdamW"}


def reference_schedule_time(entry, p, m):
    try:
        from oracle import refpy
        if not refpy.available():
            return None
        t = refpy.time_pipeline(entry, p, m, 3)
        return {"entry": entry, "p": p, "m": m, "ms": t * 1e3, "cores": 1,
                "what": "reference build_entry+assemble+simulate+exact_peak (oracle/_ref, steady_clock)"}
    except Exception:  # noqa: BLE001
        return None


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path — its own
    schedule code (oracle/_ref) producing the op order, executed on host cores by the
    oracle port; rank 0 only."""
    if rank != 0:
        return
    mcfg = CONFIGS[args.model]
    sched = args.schedule or ("zb-h1" if args.gpus == 1 else "v-half")
    from oracle import refpy
    sched_info = reference_schedule_time(sched, args.gpus, args.microbatches) if refpy.available() else None
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(mcfg, args, target_s=max(2.0, args.cpu_sample_s / max(1, args.steps + args.warmup)),
                         tiny_e2e=False)
        if i >= args.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    tiny = cpu_tiny_e2e()
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "dtype": "f32",
            "data": "synthetic", "config": {"workload": workload_name(args, sched), "model": f"gpt-{args.model}"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r["cores"], "kind": "port",
                             "sample": r["sample"], "tiny_e2e": tiny},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_schedule": sched_info,
            "note": "the reference has no F/B/W execution; its schedule code (oracle/_ref) + the CPU oracle port"}
    print(json.dumps(line), flush=True)


def workload_name(args, sched):
    return (f"gpt-{args.model} seq{CONFIGS[args.model]['seq']} {sched} p={args.gpus} m={args.microbatches} "
            f"mbs={args.micro_batch}")


# ---------------------------------------------------------------- our arm
def transfer_summary(gathered):
    """Stage-boundary activation / gradient pulls of the timeline step: bytes and copy-engine time per
    device (CUDA events around each cudaMemcpyAsync on the copy stream), achieved GB/s.  The link is
    NVLink P2P when the ranks sit on different GPUs; ranks sharing one GPU measure a local HBM copy."""
    pb_, ms_ = sum(g[4] for g in gathered), sum(g[5] for g in gathered)
    if pb_ == 0:
        return None
    uuids = {str(g[6]) for g in gathered}
    return {"bytes_per_step": int(pb_), "copy_ms_per_step": ms_,
            "achieved_gbps": pb_ / (ms_ * 1e-3) / 1e9 if ms_ > 0 else None,
            "per_device_gbps": [g[4] / (g[5] * 1e-3) / 1e9 if g[5] > 0 else None for g in gathered],
            "link": "nvlink-p2p" if len(uuids) == len(gathered) else "same-gpu (ranks share a device; not NVLink)",
            "peak_gbps_per_direction": 900.0}


def run_schedule(args, ctx, sched_name, headline):
    """One schedule on this rank's pipeline device: build, warm up, time K steps (device-resident inputs,
    CUDA events, max over ranks), then (headline only) the e2e host-input steps and the GEMM-timed step,
    and always one timeline step.  Returns the rank-0 summary (None on other ranks).  The executor is
    destroyed before returning, so the next schedule gets the whole HBM."""
    import gc

    import torch

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import DeviceExecutor, ModelConfig, balanced_stage_layers

    rank, world, local, p, dist = ctx["rank"], ctx["world"], ctx["local"], args.gpus, ctx["dist"]
    m = args.microbatches
    schedule = pb.assemble(pb.build_entry(sched_name, p), m)
    cfg = ModelConfig(**CONFIGS[args.model], micro_batch=args.micro_batch, optimizer=True, timeline=True)
    if p > 1 and not args.even_split:
        cfg = dataclasses.replace(cfg, stage_layers=balanced_stage_layers(cfg, schedule.topology))
    device = rank + 1
    ex = DeviceExecutor(cfg, schedule, device, local)
    if world > 1:
        blobs = [None] * world
        dist.all_gather_object(blobs, ex.export_blob())
        ex.connect_ipc(blobs)
        dist.barrier()
    T = cfg.tokens_per_microbatch
    tok_dev, lab_dev, tok_host, lab_host = ctx["inputs"]
    barrier, max_over_ranks, sum_over_ranks = ctx["barrier"], ctx["max"], ctx["sum"]
    stream = torch.cuda.ExternalStream(ex.stream)
    for _ in range(args.warmup):
        ex.step(tok_dev, lab_dev, on_host=False)
    barrier()

    # ---- device-timed region: K steps, inputs resident in HBM (weights+activations >> 126 MB L2)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            ex.step_async(tok_dev, lab_dev, on_host=False)
        e1.record(stream)
        torch.cuda.synchronize()
        _, st = ex.sync()
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    launches = sum_over_ranks(st.kernel_launches * args.steps)
    tokens_per_step = m * T
    out = {"schedule": sched_name, "ms_per_step": ms, "tokens_per_s": tokens_per_step / (ms / 1e3),
           "launches": launches, "clocks": clk.summary(), "cfg": cfg, "sched": schedule}

    if headline:
        # ---- e2e: the public step call with pinned HOST inputs, H2D + loss D2H inside, wall clock
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ex.step(tok_host, lab_host, on_host=True)
        barrier()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
        holds_first = schedule.topology.device_of(1) == device
        holds_last = schedule.topology.device_of(schedule.topology.num_stages) == device
        out["e2e"] = {"value": tokens_per_step / e2e_s, "unit": "tokens/s",
                      "h2d_bytes_per_step": int(sum_over_ranks((m * T * 4 if holds_first else 0)
                                                               + (m * T * 4 if holds_last else 0))),
                      "d2h_bytes_per_step": int(sum_over_ranks(8)),
                      "def": "pb_exec_step with pinned host tokens/labels (H2D inside), loss + id-check flag D2H, "
                             "wall clock, max over ranks"}

    # ---- timeline step (bubble, per-device busy) after a barrier, same inputs
    barrier()
    torch.cuda.synchronize()
    tl, tst = ex.step(tok_dev, lab_dev, on_host=False)
    mem = ex.memory()
    uuid = str(torch.cuda.get_device_properties(torch.cuda.current_device()).uuid)
    mine = ([tuple(q) for q in tl], tst.pool_bytes, tst.pool_slots, tst.loss, tst.peer_bytes, tst.copy_ms, uuid, mem)
    gathered = [mine]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)

    gall = None
    if headline:
        # ---- GEMM roofline: one more step with CUDA events around every GEMM launch (compute stream)
        barrier()
        ex.set_flags(timeline=False, gemm_timing=True)
        _, gst = ex.step(tok_dev, lab_dev, on_host=False)
        ex.set_flags(timeline=True, gemm_timing=False)
        gsum = [gst.gemm_ms, gst.gemm_flops, gst.gemm_launches, gst.step_ms]
        gall = [gsum]
        if world > 1:
            gall = [None] * world
            dist.all_gather_object(gall, gsum)
    del ex, stream
    gc.collect()
    torch.cuda.synchronize()
    barrier()
    if rank != 0:
        return None

    from paper_2405_15362_b200.pipeblock import TimedPass, account
    passes = [TimedPass(*q) for g in gathered for q in g[0]]
    sim = account(schedule.topology, passes) if passes else None
    pred = [int(x) for x in pb.exact_peak(schedule)]
    mems = [g[7] for g in gathered]
    GiB = 2 ** 30
    out.update({
        "loss": next((g[3] for g in gathered if g[3] == g[3]), None),
        "bubble_rate": sim.bubble_rate if sim else None,
        "makespan_ms": sim.makespan if sim else None,
        "ideal_ms": max(sim.busy) if sim else None,
        "predicted_slots_per_device": pred,
        "measured_slots_per_device": [g[2] for g in gathered],
        "pool_bytes_per_device": [g[1] for g in gathered],
        "device_memory": {
            "activation_gib_per_device": [(x["activation_pool"] + x["head_pool"]) / GiB for x in mems],
            "executor_gib_per_device": [x["executor_total"] / GiB for x in mems],
            "high_water_gib_per_device": [x["device_used_high"] / GiB for x in mems],
            "baseline_gib_per_device": [x["device_used_at_create"] / GiB for x in mems],
            "device_total_gib": mems[0]["device_total"] / GiB,
            "breakdown_device_max": max(mems, key=lambda x: x["executor_total"]),
            "def": "pb_exec_memory: executor allocations by category; high-water = cudaMemGetInfo total - free "
                   "sampled after creation and after every synchronised step (whole device)"},
        "transfer": transfer_summary(gathered),
        "gathered": gathered, "gall": gall, "sim": sim,
    })
    return out


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import ModelConfig, synthetic_batch

    if os.environ.get("PB_BENCH_SHARE_GPU"):  # test mode: every rank on cuda:0 (one-GPU box)
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("PB_BENCH_SHARE_GPU"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    mcfg = CONFIGS[args.model]
    p = args.gpus
    m = args.microbatches
    sched_name = args.schedule or ("zb-h1" if p == 1 else "v-half")
    if args.compare is None:  # the north-star comparisons at N > 1 (the V blocks need d >= 2)
        compare = [] if p == 1 else [s for s in ("1f1b", "v-zb", "v-half") + (("v-min",) if args.model == "14b" else ())
                                     if s != sched_name]
    else:
        compare = [s for s in args.compare if s not in ("none", sched_name)]
    base_cfg = ModelConfig(**mcfg, micro_batch=args.micro_batch, optimizer=True, timeline=True)
    T = base_cfg.tokens_per_microbatch
    tokens_np, labels_np = synthetic_batch(base_cfg, m)
    tok_host = torch.from_numpy(tokens_np).pin_memory()
    lab_host = torch.from_numpy(labels_np).pin_memory()
    tok_dev, lab_dev = tok_host.cuda(), lab_host.cuda()
    torch.cuda.synchronize()
    coll_dev = "cpu" if os.environ.get("PB_BENCH_SHARE_GPU") else "cuda"

    def barrier():
        if world > 1:
            dist.barrier()

    def reduce(x: float, op) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    ctx = {"rank": rank, "world": world, "local": local, "dist": dist, "barrier": barrier,
           "inputs": (tok_dev, lab_dev, tok_host, lab_host),
           "max": lambda x: reduce(x, dist.ReduceOp.MAX) if dist else x,
           "sum": lambda x: reduce(x, dist.ReduceOp.SUM) if dist else x}
    head = run_schedule(args, ctx, sched_name, headline=True)
    others = [run_schedule(args, ctx, s, headline=False) for s in compare]
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    cfg, schedule, gathered, gall, sim = head["cfg"], head["sched"], head["gathered"], head["gall"], head["sim"]
    ms, value = head["ms_per_step"], head["tokens_per_s"]
    tokens_per_step = m * T
    peaks_pred = head["predicted_slots_per_device"]
    # 1F1B at the same p: predicted slots per device (its slot = one straight stage = 2 V-chunks)
    peaks_1f1b = pb.exact_peak(pb.assemble(pb.build_entry("1f1b", p), m))
    chunk_units = 2 if schedule.topology.num_stages == 2 * p else 1
    mem_vs_1f1b = max(peaks_pred) / chunk_units / max(peaks_1f1b)
    meas_vs_1f1b = max(head["measured_slots_per_device"]) / chunk_units / max(peaks_1f1b)

    peaks, peak_kind = measured_peaks()
    roof = None
    g_ms, g_fl, g_n = sum(g[0] for g in gall), sum(g[1] for g in gall), sum(g[2] for g in gall)
    if g_ms > 0:
        achieved = g_fl / (g_ms / 1e3) / 1e12
        pk = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
        traffic, tnote = None, None
        tp = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_gemm_traffic.json")) \
            if os.path.isdir(os.path.join(ROOT, "profiles")) else []
        if tp:
            with open(os.path.join(ROOT, "profiles", tp[-1])) as f:
                tj = json.load(f)
            traffic = tj["dram_bytes"]
            tnote = (f"DRAM read+write bytes per launch of {tj['kernel']} from profiles/{tp[-1]}; "
                     f"algorithmic bytes of that launch {tj['algorithmic_bytes']}")
        roof = {"bound": "tensor", "kernel": "gemm_kernel (tcgen05, csrc/kernels/gemm_tc.cu)", "achieved": achieved,
                "peak": pk, "unit": "TFLOP/s", "frac": achieved / pk, "traffic": traffic, "traffic_note": tnote,
                "peak_kind": f"{peak_kind} bf16_tflops_sustained (kernel timed inside a long step)",
                "gemm_share_of_device_time": g_ms / sum(g[3] for g in gall),
                "launches": g_n, "flops_per_step": g_fl,
                "def": "sum of 2MNK over all GEMM launches of one step / sum of their CUDA-event durations"}
    # model FLOP utilisation (Megatron F/B/W counts: full, non-causal attention FLOPs)
    fl = cfg.flops_per_token()
    model_flops = tokens_per_step * (cfg.layers * (fl["F"] + fl["B"] + fl["W"]) + 3 * fl["head"])
    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(mcfg, args)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)}

    def sched_block(r):
        dm = r["device_memory"]
        act = max(dm["activation_gib_per_device"])
        return {"tokens_per_s": r["tokens_per_s"], "ms_per_step": r["ms_per_step"], "bubble_rate": r["bubble_rate"],
                "makespan_ms": r["makespan_ms"], "pipeline_roofline_frac": (r["ideal_ms"] / r["makespan_ms"])
                if r["makespan_ms"] else None,
                "predicted_slots_per_device": r["predicted_slots_per_device"],
                "activation_gib_max": act, "high_water_gib_max": max(dm["high_water_gib_per_device"]),
                "executor_gib_max": max(dm["executor_gib_per_device"]),
                "transfer_gbps": (r["transfer"] or {}).get("achieved_gbps"),
                "link": (r["transfer"] or {}).get("link"), "loss": r["loss"], "clocks": r["clocks"]}

    schedules = None
    if others:
        schedules = {r["schedule"]: sched_block(r) for r in [head] + others}
        b = schedules.get("1f1b")
        if b:
            for v in schedules.values():
                v["tokens_per_s_vs_1f1b"] = v["tokens_per_s"] / b["tokens_per_s"]
                v["activation_vs_1f1b"] = v["activation_gib_max"] / b["activation_gib_max"]
                v["high_water_vs_1f1b"] = v["high_water_gib_max"] / b["high_water_gib_max"]
    dm = head["device_memory"]
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": p, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, seeded; random-init weights)",
        "config": {"workload": workload_name(args, sched_name), "model": f"gpt-{args.model}",
                   "global_batch": m * args.micro_batch, "seq_len": cfg.seq, "parallelism": f"pp{p}",
                   "schedule": sched_name, "microbatches": m, "micro_batch": args.micro_batch,
                   "stage_layers": list(cfg.stage_layers) if cfg.stage_layers else None,
                   "l2": "no flush: per-step working set (weights+grads+optimizer+activations, tens of GB) >> 126 MB L2"},
        "bubble_rate": head["bubble_rate"],
        "bubble_def": "1 - sum busy / (d * makespan) over measured pass times (simulate.hpp:81-82)",
        "makespan_ms": head["makespan_ms"],
        "roofline_pipeline": {"ideal_ms": head["ideal_ms"],
                              "frac": (head["ideal_ms"] / head["makespan_ms"]) if head["makespan_ms"] else None,
                              "def": "ideal zero-bubble time (max per-device busy) / measured makespan"},
        "activation_memory": {"predicted_slots_per_device": peaks_pred,
                              "measured_slots_max": max(head["measured_slots_per_device"]),
                              "pool_bytes_per_device": head["pool_bytes_per_device"],
                              "activation_gib_per_device": dm["activation_gib_per_device"],
                              "device_high_water_gib_per_device": dm["high_water_gib_per_device"],
                              "device_baseline_gib_per_device": dm["baseline_gib_per_device"],
                              "executor_gib_per_device": dm["executor_gib_per_device"],
                              "breakdown_device_max": dm["breakdown_device_max"],
                              "vs_1f1b": mem_vs_1f1b, "measured_vs_1f1b": meas_vs_1f1b,
                              "def": "slots: peak activation units (whole-stage microbatches) / 1F1B's predicted at the "
                                     "same p; bytes: pb_exec_memory allocations and cudaMemGetInfo high-water"},
        "mfu": model_flops / (ms / 1e3) / (p * 1e12) / peaks.get("bf16_tflops", 1687.0),
        "mfu_def": "Megatron F/B/W FLOPs (PAPER.md:575, full non-causal attention counted) / (N x measured "
                   "bf16_tflops burst)",
        "loss": head["loss"],
        "clocks": head["clocks"],
        "e2e": head["e2e"],
        "gpu_launches": int(head["launches"]),
        "roofline": roof,
        "transfer": head["transfer"],
        "schedules": schedules,
        "cpu_baseline": cpu,
        "reference_schedule": reference_schedule_time(sched_name, p, m),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
