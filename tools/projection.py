"""Multi-GPU projection from ONE B200 (this round's GPU pool gives one GPU per call).

For each schedule, all p pipeline devices of the REAL schedule are instantiated in
one process on cuda:0 (PipelineExecutor, in-process transport) and one training
step runs with PB_FLAG_ISOLATE: passes execute one at a time over the whole group
(a GPU token taken after each pass's cross-device waits), each synchronised, so every pass's CUDA-event duration is
its stand-alone time on a B200 at the real chunk size (embedding / LM head / loss
on the right stages, real message copies, real activation pool).  The measured
per-pass durations are then replayed in each device's grid order with pb_replay
(simulate.hpp:44-56 with one duration per pass) plus a per-crossing latency of
msg_bytes / NVLink bandwidth (an assumption, stated in the output: no NVLink here).

--via-chunks (models too large to instantiate whole on one GPU: 6B, 14B): a probe
pipeline with the SAME chunk shapes runs instead — the same schedule family at p=2
(V: 4 stages = first / middle / middle / last chunk) or p=3 (straight: first /
middle / last stage), each chunk with the target's layers per chunk — and the
target schedule is replayed with the probe's mean isolated pass time per
(chunk class, kind).  Activation memory is then the plan's slot count times the
probe's measured slot bytes for that chunk class.

Output: one JSON object (stdout, and --out file) with, per schedule, the projected
p-GPU step time, tokens/s, bubble rate (simulate.hpp:81-82 on the replay), the
pipeline roofline fraction (max per-device busy / makespan), measured activation
pool bytes per device vs the exact_peak prediction and vs 1F1B.

    python tools/projection.py --model 1.5b --p 8 --microbatches 32 --out profiles/r1_projection_1p5b_p8.json
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="1.5b", choices=sorted(CONFIGS))
    ap.add_argument("--p", type=int, nargs="+", default=[8])
    ap.add_argument("--microbatches", type=int, default=32)
    ap.add_argument("--micro-batch", type=int, default=2)
    ap.add_argument("--schedules", nargs="+", default=["1f1b", "zb-h1", "v-min", "v-half", "v-zb"])
    ap.add_argument("--nvlink-gbs", type=float, default=720.0, help="assumed achieved P2P GB/s per direction")
    ap.add_argument("--latency-us", type=float, default=8.0, help="assumed per-transfer latency")
    ap.add_argument("--out", default=None)
    ap.add_argument("--via-chunks", action="store_true", help="probe-pipeline projection (see module doc)")
    ap.add_argument("--balance", action="store_true", help="balanced_stage_layers (LM-head stage carries fewer layers)")
    ap.add_argument("--layers", type=int, default=None,
                    help="override the model's layer count; with --via-chunks the last stage takes the remainder "
                         "(e.g. 31 layers on 16 V stages: 2 per stage, 1 on the LM-head stage)")
    args = ap.parse_args()

    import torch

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import ModelConfig, PipelineExecutor, synthetic_batch

    mcfg = dict(CONFIGS[args.model])
    if args.layers:
        mcfg["layers"] = args.layers
    cfg = ModelConfig(**mcfg, micro_batch=args.micro_batch, optimizer=True, timeline=True)
    T = cfg.tokens_per_microbatch
    m = args.microbatches
    tokens, labels = synthetic_batch(cfg, m)
    tok, lab = torch.from_numpy(tokens).cuda(), torch.from_numpy(labels).cuda()
    msg_bytes = T * cfg.hidden * 2
    comm_ms = (msg_bytes / (args.nvlink_gbs * 1e9) + args.latency_us * 1e-6) * 1e3
    out = {"model": f"gpt-{args.model}", "config": mcfg, "microbatches": m, "micro_batch": args.micro_batch,
           "tokens_per_step": m * T, "gpu": torch.cuda.get_device_name(0),
           "method": "all p pipeline devices on one B200, PB_FLAG_ISOLATE per-pass CUDA-event times, "
                     "replayed in grid order (pb_replay) with comm = msg_bytes/nvlink_gbs + latency",
           "assumptions": {"nvlink_gbs": args.nvlink_gbs, "latency_us": args.latency_us, "msg_bytes": msg_bytes,
                           "comm_ms": comm_ms}, "runs": []}
    out["power_cap"] = power_cap_factor(args, mcfg)
    for p in args.p:
        for name in args.schedules:
            t0 = time.time()
            if args.via_chunks:
                out["runs"].append(project_via_chunks(args, mcfg, name, p, m, comm_ms))
                print(json.dumps({k: out["runs"][-1][k] for k in ("schedule", "p", "projected_tokens_per_s",
                                                                  "bubble_rate", "max_pool_gib")}), file=sys.stderr)
                continue
            sched = pb.assemble(pb.build_entry(name, p), m)
            rcfg = cfg
            if args.balance:
                from paper_2405_15362_b200.executor import balanced_stage_layers
                rcfg = dataclasses.replace(cfg, stage_layers=balanced_stage_layers(cfg, sched.topology))
            ex = PipelineExecutor(rcfg, sched, [0] * p)
            ex.set_flags(timeline=True, isolate=True)
            ex.step(tok, lab, on_host=False)                  # warm-up
            res = ex.step(tok, lab, on_host=False)
            dur = {(q.device, q.stage, q.kind, q.microbatch): q.duration for q in res.timeline}
            durations = [dur[(q.device, q.stage, q.kind, q.microbatch)] for q in sched.passes]
            rep = pb.replay(sched, durations, comm_ms)
            rep0 = pb.replay(sched, durations, 0.0)
            per_kind = {}
            for q in sched.passes:
                per_kind.setdefault(q.kind, []).append(dur[(q.device, q.stage, q.kind, q.microbatch)])
            pred = pb.exact_peak(sched)
            pool = [res.per_device[d].pool_bytes for d in sorted(res.per_device)]
            slots = [res.per_device[d].pool_slots for d in sorted(res.per_device)]
            run = {"schedule": name, "p": p, "loss": res.loss,
                   "stage_layers": list(rcfg.stage_layers) if rcfg.stage_layers else None,
                   "projected_ms_per_step": rep.makespan, "projected_tokens_per_s": m * T / (rep.makespan / 1e3),
                   "bubble_rate": rep.bubble_rate, "bubble_rate_zero_comm": rep0.bubble_rate,
                   "pipeline_roofline_frac": max(rep.busy) / rep.makespan,
                   "ideal_ms": max(rep.busy), "busy_ms_per_device": rep.busy,
                   "mean_pass_ms": {k: sum(v) / len(v) for k, v in per_kind.items()},
                   "predicted_peak_units": pred, "measured_slots": slots, "pool_bytes_per_device": pool,
                   "max_pool_gib": max(pool) / 2**30, "wall_s": time.time() - t0}
            out["runs"].append(run)
            print(json.dumps({k: run[k] for k in ("schedule", "p", "projected_tokens_per_s", "bubble_rate",
                                                  "pipeline_roofline_frac", "max_pool_gib")}), file=sys.stderr)
            del ex, res
            import gc
            gc.collect()
            torch.cuda.synchronize()
    if args.via_chunks:
        out["method"] = ("probe pipeline with the target's chunk shapes on one B200 (PB_FLAG_ISOLATE pass times, "
                         "mean per chunk class and kind), target schedule replayed with pb_replay")
    # the same projection at the continuous (power-capped) pass speed
    f = out["power_cap"]["factor"]
    for r in out["runs"]:
        r["projected_tokens_per_s_at_cap"] = r["projected_tokens_per_s"] / f
    # activation memory vs 1F1B at the same p (measured pool bytes, max over devices)
    for r in out["runs"]:
        base = next((b for b in out["runs"] if b["schedule"] == "1f1b" and b["p"] == r["p"]), None)
        if base:
            r["pool_vs_1f1b"] = max(r["pool_bytes_per_device"]) / max(base["pool_bytes_per_device"])
            r["tokens_per_s_vs_1f1b"] = r["projected_tokens_per_s"] / base["projected_tokens_per_s"]
    text = json.dumps(out, indent=1)
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)


def power_cap_factor(args, mcfg):
    """Isolated passes run one at a time with a synchronise in between, so the GPU sits below its power
    cap and clocks higher than in a continuous step.  Calibrate: a zb-h1 p=1 pipeline of the same layer
    shapes (4 layers, real hidden / seq / vocab / micro-batch) runs once isolated and once continuously;
    factor = continuous makespan / sum of isolated pass times (>= 1 when power-capped)."""
    import torch

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import ModelConfig, PipelineExecutor, synthetic_batch

    cfg = ModelConfig(**dict(mcfg, layers=4), micro_batch=args.micro_batch, optimizer=True, timeline=True)
    m = 16
    sched = pb.assemble(pb.build_entry("zb-h1", 1), m)
    tokens, labels = synthetic_batch(cfg, m)
    tok, lab = torch.from_numpy(tokens).cuda(), torch.from_numpy(labels).cuda()
    ex = PipelineExecutor(cfg, sched, [0])
    ex.set_flags(timeline=True)
    for _ in range(3):
        ex.step(tok, lab, on_host=False)
    cont = [ex.step(tok, lab, on_host=False).per_device[1].step_ms for _ in range(3)]
    ex.set_flags(timeline=True, serial=True)  # one device: a synchronise after every pass = isolated passes
    ex.step(tok, lab, on_host=False)
    iso = [sum(q.duration for q in ex.step(tok, lab, on_host=False).timeline) for _ in range(3)]
    del ex
    torch.cuda.synchronize()
    c, i = sorted(cont)[1], sorted(iso)[1]
    return {"factor": c / i, "continuous_ms": c, "isolated_sum_ms": i,
            "what": "zb-h1 p=1, 4 layers of this model, m=16: continuous step / sum of isolated pass times "
                    "(median of 3); projected_tokens_per_s_at_cap = projected / factor"}


def chunk_class(stage: int, num_stages: int) -> str:
    return "first" if stage == 1 else ("last" if stage == num_stages else "middle")


def project_via_chunks(args, mcfg, name, p, m, comm_ms):
    import dataclasses

    import torch

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import ModelConfig, PipelineExecutor, synthetic_batch

    target = pb.assemble(pb.build_entry(name, p), m)
    S = target.topology.num_stages
    L = mcfg["layers"]
    per_chunk = -(-L // S)                 # ceil: every stage but the LM-head one carries this many
    last = L - per_chunk * (S - 1)         # the LM-head stage takes the remainder
    if last < 1:
        raise SystemExit(f"{L} layers do not split into {S} stages")
    v_shape = S == 2 * p
    probe_p = 2 if v_shape else 3
    probe_S = 2 * probe_p if v_shape else probe_p
    probe_m = min(m, 4 * probe_p)
    cfg = ModelConfig(**dict(mcfg, layers=per_chunk * (probe_S - 1) + last), micro_batch=args.micro_batch,
                      optimizer=True, timeline=True,
                      stage_layers=tuple([per_chunk] * (probe_S - 1) + [last]) if last != per_chunk else None)
    probe = pb.assemble(pb.build_entry(name, probe_p), probe_m)
    tokens, labels = synthetic_batch(cfg, probe_m)
    tok, lab = torch.from_numpy(tokens).cuda(), torch.from_numpy(labels).cuda()
    ex = PipelineExecutor(cfg, probe, [0] * probe_p)
    ex.set_flags(timeline=True, isolate=True)
    ex.step(tok, lab, on_host=False)
    res = ex.step(tok, lab, on_host=False)
    acc = {}
    for q in res.timeline:
        acc.setdefault((chunk_class(q.stage, probe_S), q.kind), []).append(q.duration)
    mean = {k: sum(v) / len(v) for k, v in acc.items()}
    # activation slot bytes per chunk class: the probe's slot size (largest chunk class on a device)
    slot_bytes = {d: res.per_device[d].slot_bytes for d in res.per_device}
    del ex
    torch.cuda.synchronize()
    durations = [mean[(chunk_class(q.stage, S), q.kind)] for q in target.passes]
    rep = pb.replay(target, durations, comm_ms)
    rep0 = pb.replay(target, durations, 0.0)
    pred = pb.exact_peak(target)
    # a device's activation slot is sized for its largest stage: take the slot bytes of the probe device
    # that holds the same chunk classes (V: {first, last} / {middle}; straight: {first} / {middle} / {last})
    def classes(topo, n_stages, d):
        return frozenset(chunk_class(st, n_stages) for st in range(1, n_stages + 1) if topo.device_of(st) == d)

    probe_bytes = {classes(probe.topology, probe_S, d): b for d, b in slot_bytes.items()}
    # the LM-head pool (logits + final hidden per live head microbatch) sits on the device holding stage
    # S, outside the activation slots: take the probe's (pool_bytes - slots * slot_bytes) on that device
    probe_last = probe.topology.device_of(probe_S)
    st_last = None
    for d, st in res.per_device.items():
        if d == probe_last:
            st_last = st
    head_bytes = int(st_last.pool_bytes - st_last.slot_bytes * st_last.pool_slots) if st_last else 0
    pool = []
    for d in range(1, p + 1):
        pool.append(int(pred[d - 1]) * probe_bytes[classes(target.topology, S, d)]
                    + (head_bytes if target.topology.device_of(S) == d else 0))
    T = cfg.tokens_per_microbatch
    return {"schedule": name, "p": p, "probe": f"{name} p={probe_p} m={probe_m}, {cfg.layers} layers "
                                                f"({per_chunk} per chunk, {last} on the LM-head chunk)",
            "target_stage_layers": [per_chunk] * (S - 1) + [last],
            "projected_ms_per_step": rep.makespan, "projected_tokens_per_s": m * T / (rep.makespan / 1e3),
            "bubble_rate": rep.bubble_rate, "bubble_rate_zero_comm": rep0.bubble_rate,
            "pipeline_roofline_frac": max(rep.busy) / rep.makespan, "ideal_ms": max(rep.busy),
            "busy_ms_per_device": rep.busy, "mean_pass_ms": {f"{c}.{k}": v for (c, k), v in sorted(mean.items())},
            "predicted_peak_units": pred, "pool_bytes_per_device": pool, "head_pool_bytes": head_bytes,
            "pool_def": "predicted peak slots x probe slot bytes (same chunk classes) + the probe's LM-head pool on "
                        "the device holding the last stage", "max_pool_gib": max(pool) / 2**30,
            "probe_slot_bytes": sorted(set(slot_bytes.values()))}


if __name__ == "__main__":
    main()
