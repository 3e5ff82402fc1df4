"""Per-device probes of a p-device pipeline on ONE B200 (PB_FLAG_SOLO), and the projection built on them.

Each pipeline device d of the REAL schedule (assemble(build_entry(name, p), m)) is instantiated alone
on cuda:0 with PB_FLAG_SOLO: its own weights, gradients, AdamW state, lifespan activation pool
(exact_peak slots), LM-head pool and transfer buffers — its real memory footprint — and one step walks
its own op list in grid order with the real kernels (cross-device inputs are not pulled: the receive
slot keeps its contents; outputs are not signalled).  Per device this gives

  * memory: every allocation by category (pb_exec_memory) and the device high-water mark
    (cudaMemGetInfo, sampled after creation and after each synchronised step), or the out-of-memory
    error (PB_ECUDA) when the device does not fit in HBM;
  * per-pass CUDA-event durations of a continuous run of its op list (the same power-capped clock
    regime as a real step, unlike one-pass-at-a-time isolation).

When every device fits, the durations are replayed in each device's grid order with pb_replay
(simulate.hpp:44-56) plus an assumed per-crossing cost msg_bytes / NVLink GB/s + latency, giving the
projected p-GPU step time, tokens/s and bubble (simulate.hpp:81-82).

    python tools/device_probe.py --model 14b --p 8 --microbatches 64 --micro-batch 4 \\
        --schedules v-min v-half v-zb 1f1b --out profiles/r2_memory_regime_14b_mbs4.json
"""
from __future__ import annotations

import argparse
import dataclasses
import gc
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402

GiB = 2 ** 30


def probe_device(cfg, sched, d, tok, lab, steps):
    import torch

    from paper_2405_15362_b200._lib import PipeblockError
    from paper_2405_15362_b200.executor import DeviceExecutor

    torch.cuda.synchronize()
    free0, total = torch.cuda.mem_get_info()
    t0 = time.time()
    try:
        ex = DeviceExecutor(dataclasses.replace(cfg, solo=True), sched, d, 0)
    except PipeblockError as e:
        gc.collect()
        torch.cuda.synchronize()
        free1, _ = torch.cuda.mem_get_info()
        import re
        need = None
        mm = re.search(r"allocating .* \((\d+) B; executor holds (\d+) B", str(e))
        if mm:  # the allocation that failed + what was already held: a lower bound on the footprint
            need = (int(mm.group(1)) + int(mm.group(2))) / GiB
        return {"device": d, "fits": False, "error": str(e), "code": e.code, "needs_at_least_gib": need,
                "freed_after_error": free1 >= free0 - (64 << 20)}
    try:
        tl = st = None
        for i in range(steps + 1):  # first step: warm-up (lazy W-pass GEMM tables)
            tl, st = ex.step(tok, lab, on_host=False)
        mem = ex.memory()
        kinds = {}
        for q in tl:
            kinds.setdefault(q.kind, []).append(q.duration)
        return {"device": d, "fits": True, "memory": mem,
                "executor_gib": mem["executor_total"] / GiB,
                "high_water_gib": mem["device_used_high"] / GiB,
                "high_water_minus_baseline_gib": (mem["device_used_high"] - mem["device_used_at_create"]) / GiB,
                "activation_gib": (mem["activation_pool"] + mem["head_pool"]) / GiB,
                "pool_slots": st.pool_slots, "slot_bytes": st.slot_bytes, "step_ms": st.step_ms,
                "busy_ms": st.busy_ms, "mean_pass_ms": {k: sum(v) / len(v) for k, v in kinds.items()},
                "passes": [(q.stage, q.kind, q.microbatch, q.duration) for q in tl], "wall_s": time.time() - t0}
    finally:
        del ex
        gc.collect()
        torch.cuda.synchronize()


def probe_schedule(cfg, sched, name, devs, tok, lab, steps, comm_ms):
    """Probe the listed pipeline devices of `sched`; when all p devices fit, replay their measured
    per-pass durations (pb_replay, simulate.hpp:44-56) into the projected p-GPU step.  The returned
    run keeps "durations" ((device, stage, kind, mb) -> ms) and "replay" (the SimResult) for callers."""
    import sys as _sys

    from paper_2405_15362_b200 import pipeblock as pb

    T = cfg.tokens_per_microbatch
    m = sched.microbatches
    run = {"schedule": name, "stage_layers": list(cfg.stage_layers) if cfg.stage_layers else None,
           "predicted_peak_units": [int(x) for x in pb.exact_peak(sched)], "devices": []}
    for d in devs:
        r = probe_device(cfg, sched, d, tok, lab, steps)
        run["devices"].append(r)
        print(json.dumps({"schedule": name, "device": d, "fits": r["fits"],
                          "high_water_gib": r.get("high_water_gib"), "activation_gib": r.get("activation_gib"),
                          "step_ms": r.get("step_ms"), "error": r.get("error")}), file=_sys.stderr, flush=True)
    fits = [r for r in run["devices"] if r["fits"]]
    run["all_fit"] = len(fits) == len(run["devices"])
    if fits:
        run["max_high_water_gib"] = max(r["high_water_gib"] for r in fits)
        run["max_executor_gib"] = max(r["executor_gib"] for r in fits)
        run["max_activation_gib"] = max(r["activation_gib"] for r in fits)
    if run["all_fit"] and len(run["devices"]) == sched.topology.devices:
        dur = {}
        for r in run["devices"]:
            for (s, k, mb, t) in r["passes"]:
                dur[(r["device"], s, k, mb)] = t
        durations = [dur[(q.device, q.stage, q.kind, q.microbatch)] for q in sched.passes]
        rep = pb.replay(sched, durations, comm_ms)
        rep0 = pb.replay(sched, durations, 0.0)
        run.update({"projected_ms_per_step": rep.makespan,
                    "projected_tokens_per_s": m * T / (rep.makespan / 1e3),
                    "bubble_rate": rep.bubble_rate, "bubble_rate_zero_comm": rep0.bubble_rate,
                    "pipeline_roofline_frac": max(rep.busy) / rep.makespan, "ideal_ms": max(rep.busy),
                    "busy_ms_per_device": rep.busy, "durations": dur, "replay": rep})
    return run


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="1.5b", choices=sorted(CONFIGS))
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--microbatches", type=int, default=32)
    ap.add_argument("--micro-batch", type=int, default=2)
    ap.add_argument("--schedules", nargs="+", default=["1f1b", "zb-h1", "v-min", "v-half", "v-zb"])
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--balance", action="store_true", help="balanced_stage_layers (LM-head stage carries fewer layers)")
    ap.add_argument("--steps", type=int, default=1, help="timed solo steps per device (after one warm-up)")
    ap.add_argument("--devices", default="all", help="'all' or a comma list of 1-based pipeline devices")
    ap.add_argument("--nvlink-gbs", type=float, default=720.0, help="assumed achieved P2P GB/s per direction")
    ap.add_argument("--latency-us", type=float, default=8.0, help="assumed per-transfer latency")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import ModelConfig, balanced_stage_layers, synthetic_batch

    mcfg = dict(CONFIGS[args.model])
    if args.layers:
        mcfg["layers"] = args.layers
    base = ModelConfig(**mcfg, micro_batch=args.micro_batch, optimizer=True, timeline=True)
    T = base.tokens_per_microbatch
    m = args.microbatches
    tokens, labels = synthetic_batch(base, m)
    tok, lab = torch.from_numpy(tokens).cuda(), torch.from_numpy(labels).cuda()
    msg_bytes = T * base.hidden * 2
    comm_ms = (msg_bytes / (args.nvlink_gbs * 1e9) + args.latency_us * 1e-6) * 1e3
    free, total = torch.cuda.mem_get_info()
    out = {"model": f"gpt-{args.model}", "config": mcfg, "p": args.p, "microbatches": m,
           "micro_batch": args.micro_batch, "tokens_per_step": m * T, "gpu": torch.cuda.get_device_name(0),
           "device_total_gib": total / GiB,
           "method": "each pipeline device of the real schedule alone on one B200 (PB_FLAG_SOLO): real allocation "
                     "(weights, grads, AdamW, exact_peak activation slots, head pool, transfer buffers), one "
                     "continuous step of its own op list; per-pass CUDA-event durations replayed in grid order "
                     "(pb_replay) with comm = msg_bytes / nvlink_gbs + latency",
           "assumptions": {"nvlink_gbs": args.nvlink_gbs, "latency_us": args.latency_us, "msg_bytes": msg_bytes,
                           "comm_ms": comm_ms}, "runs": []}
    for name in args.schedules:
        sched = pb.assemble(pb.build_entry(name, args.p), m)
        cfg = base
        if args.balance:
            cfg = dataclasses.replace(base, stage_layers=balanced_stage_layers(base, sched.topology))
        devs = list(range(1, args.p + 1)) if args.devices == "all" else [int(x) for x in args.devices.split(",")]
        run = probe_schedule(cfg, sched, name, devs, tok, lab, args.steps, comm_ms)
        for r in run["devices"]:
            r.pop("passes", None)
        run.pop("durations", None)
        run.pop("replay", None)
        out["runs"].append(run)
    for r in out["runs"]:
        b = next((x for x in out["runs"] if x["schedule"] == "1f1b"), None)
        if b and r.get("max_activation_gib") and b.get("max_activation_gib"):
            r["activation_vs_1f1b"] = r["max_activation_gib"] / b["max_activation_gib"]
        if b and r.get("projected_tokens_per_s") and b.get("projected_tokens_per_s"):
            r["tokens_per_s_vs_1f1b"] = r["projected_tokens_per_s"] / b["projected_tokens_per_s"]
    text = json.dumps(out, indent=1)
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
