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
def cpu_layer_sample(mcfg, target_s: float):
    """Bounded CPU sample: one microbatch through one layer, F + B + W (fp32, torch CPU,
    all host threads), via the oracle's F/B/W split; extrapolated to the whole model."""
    import torch
    from types import SimpleNamespace

    from oracle import numerics as N

    torch.set_num_threads(os.cpu_count() or 1)
    cfg = SimpleNamespace(layers=1, hidden=mcfg["hidden"], heads=mcfg["heads"], seq=mcfg["seq"],
                          vocab=mcfg["vocab"], micro_batch=1)
    h = cfg.hidden
    g = torch.Generator().manual_seed(0)
    p = {f"s1.l0.{n}": (0.02 * torch.randn(shp, generator=g)).requires_grad_(True)
         for n, shp in {"wqkv": (3 * h, h), "wo": (h, h), "w1": (4 * h, h), "w2": (h, 4 * h)}.items()}
    p["s1.l0.norm1"] = torch.ones(h, requires_grad=True)
    p["s1.l0.norm2"] = torch.ones(h, requires_grad=True)
    T = cfg.seq
    times = []
    t_end = time.perf_counter() + target_s
    while True:
        x = torch.randn(T, h, requires_grad=True)
        t0 = time.perf_counter()
        y = N.layer_forward(x, p, "s1.l0.", cfg)                               # F
        gy = torch.randn_like(y)
        (gx,) = torch.autograd.grad(y, x, gy, retain_graph=True)              # B
        gw = torch.autograd.grad(y, list(p.values()), gy)                     # W
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end or len(times) >= 20:
            break
    per_layer = statistics.median(times)
    tokens_per_s = T / (per_layer * mcfg["layers"])
    return {"value": tokens_per_s, "unit": "tokens/s", "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"1 sequence ({T} tokens) through 1 of {mcfg['layers']} layers, F+B+W in fp32 "
                      f"(oracle/numerics.py, torch CPU), median of {len(times)} runs, x{mcfg['layers']} layers; "
                      f"LM head and optimizer excluded"}


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
        r = cpu_layer_sample(mcfg, target_s=max(2.0, args.cpu_sample_s / max(1, args.steps + args.warmup)))
        if i >= args.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "dtype": "f32",
            "data": "synthetic", "config": {"workload": workload_name(args, sched), "model": f"gpt-{args.model}"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r["cores"], "kind": "port",
                             "sample": r["sample"]},
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


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import DeviceExecutor, ModelConfig, synthetic_batch

    if os.environ.get("PB_BENCH_SHARE_GPU"):  # test mode: every rank on cuda:0 (one-GPU box)
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("PB_BENCH_SHARE_GPU"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    mcfg = CONFIGS[args.model]
    p = args.gpus
    sched_name = args.schedule or ("zb-h1" if p == 1 else "v-half")
    schedule = pb.assemble(pb.build_entry(sched_name, p), args.microbatches)
    cfg = ModelConfig(**mcfg, micro_batch=args.micro_batch, optimizer=True, timeline=True)
    if p > 1 and not args.even_split:
        from paper_2405_15362_b200.executor import balanced_stage_layers
        cfg = dataclasses.replace(cfg, stage_layers=balanced_stage_layers(cfg, schedule.topology))
    device = rank + 1
    ex = DeviceExecutor(cfg, schedule, device, local)
    if world > 1:
        blobs = [None] * world
        dist.all_gather_object(blobs, ex.export_blob())
        ex.connect_ipc(blobs)
        dist.barrier()

    T = cfg.tokens_per_microbatch
    m = args.microbatches
    tokens_np, labels_np = synthetic_batch(cfg, m)
    tok_host = torch.from_numpy(tokens_np).pin_memory()
    lab_host = torch.from_numpy(labels_np).pin_memory()
    tok_dev, lab_dev = tok_host.cuda(), lab_host.cuda()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    coll_dev = "cpu" if os.environ.get("PB_BENCH_SHARE_GPU") else "cuda"

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    stream = torch.cuda.ExternalStream(ex.stream)
    # warm-up (device-resident inputs)
    for _ in range(args.warmup):
        ex.step(tok_dev, lab_dev, on_host=False)
    barrier()

    # ---- device-timed region: K steps, inputs resident in HBM (weights+activations >> 126 MB L2)
    launches = 0
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
    ms = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms)
    launches = sum_over_ranks(st.kernel_launches * args.steps)
    tokens_per_step = m * T
    value = tokens_per_step / (ms / 1e3)

    # ---- e2e: the public step call with pinned HOST inputs, H2D + loss D2H inside, wall clock
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _, est = ex.step(tok_host, lab_host, on_host=True)
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.steps)
    holds_first = schedule.topology.device_of(1) == device
    holds_last = schedule.topology.device_of(schedule.topology.num_stages) == device
    h2d = sum_over_ranks((m * T * 4 if holds_first else 0) + (m * T * 4 if holds_last else 0))
    d2h = sum_over_ranks(4 if holds_last else 0)

    # ---- timeline step (bubble, per-device busy) after a barrier, same inputs
    barrier()
    torch.cuda.synchronize()
    tl, tst = ex.step(tok_dev, lab_dev, on_host=False)
    loss = tst.loss
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, ([tuple(q) for q in tl], tst.pool_bytes, tst.pool_slots, tst.loss,
                                          tst.peer_bytes, tst.copy_ms, str(torch.cuda.get_device_properties(torch.cuda.current_device()).uuid)))
    else:
        gathered = [([tuple(q) for q in tl], tst.pool_bytes, tst.pool_slots, tst.loss, tst.peer_bytes, tst.copy_ms,
                     None)]

    # ---- GEMM roofline: one more step with CUDA events around every GEMM launch (compute stream)
    barrier()
    ex.set_flags(timeline=False, gemm_timing=True)
    _, gst = ex.step(tok_dev, lab_dev, on_host=False)
    ex.set_flags(timeline=True, gemm_timing=False)
    gsum = [gst.gemm_ms, gst.gemm_flops, gst.gemm_launches, gst.step_ms]
    if world > 1:
        gall = [None] * world
        dist.all_gather_object(gall, gsum)
    else:
        gall = [gsum]

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    from paper_2405_15362_b200.pipeblock import TimedPass, account
    passes = [TimedPass(*q) for g in gathered for q in g[0]]
    sim = account(schedule.topology, passes) if passes else None
    peaks_pred = pb.exact_peak(schedule)
    pool_bytes = [g[1] for g in gathered]
    # 1F1B at the same p: predicted slots per device (its slot = one straight stage = 2 V-chunks)
    ref1 = pb.assemble(pb.build_entry("1f1b", p), m)
    peaks_1f1b = pb.exact_peak(ref1)
    chunk_units = 2 if schedule.topology.num_stages == 2 * p else 1
    ours_units = max(peaks_pred) / chunk_units
    peaks_meas_units = max(g[2] for g in gathered) / chunk_units
    mem_vs_1f1b = ours_units / max(peaks_1f1b)

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
    # model FLOP utilisation (Megatron F/B/W counts)
    fl = cfg.flops_per_token()
    model_flops = tokens_per_step * (cfg.layers * (fl["F"] + fl["B"] + fl["W"]) + 3 * fl["head"])
    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = cpu_layer_sample(mcfg, args.cpu_sample_s)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)}
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": p, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, seeded; random-init weights)",
        "config": {"workload": workload_name(args, sched_name), "model": f"gpt-{args.model}",
                   "global_batch": m * args.micro_batch, "seq_len": cfg.seq, "parallelism": f"pp{p}",
                   "schedule": sched_name, "microbatches": m, "micro_batch": args.micro_batch,
                   "stage_layers": list(cfg.stage_layers) if cfg.stage_layers else None,
                   "l2": "no flush: per-step working set (weights+grads+optimizer+activations, tens of GB) >> 126 MB L2"},
        "bubble_rate": sim.bubble_rate if sim else None,
        "bubble_def": "1 - sum busy / (d * makespan) over measured pass times (simulate.hpp:81-82)",
        "makespan_ms": sim.makespan if sim else None,
        "roofline_pipeline": {"ideal_ms": max(sim.busy) if sim else None,
                              "frac": (max(sim.busy) / sim.makespan) if sim else None,
                              "def": "ideal zero-bubble time (max per-device busy) / measured makespan"},
        "activation_memory": {"predicted_slots_per_device": peaks_pred, "measured_slots_max": max(g[2] for g in gathered),
                              "pool_bytes_per_device": pool_bytes,
                              "vs_1f1b": mem_vs_1f1b, "measured_vs_1f1b": peaks_meas_units / max(peaks_1f1b),
                              "def": "peak activation units (whole-stage microbatches) / 1F1B's at the same p"},
        "mfu": model_flops / (ms / 1e3) / (p * 1e12) / peaks.get("bf16_tflops", 1687.0),
        "loss": loss,
        "clocks": clocks,
        "e2e": {"value": tokens_per_step / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "def": "pb_exec_step with pinned host tokens/labels, wall clock"},
        "gpu_launches": int(launches),
        "roofline": roof,
        "transfer": transfer_summary(gathered),
        "cpu_baseline": cpu,
        "reference_schedule": reference_schedule_time(sched_name, p, m),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
