"""Host enqueue cost vs device time per pass (no CUDA graphs; is the host fast
enough at p=8 pass sizes?).

One pipeline device of a p=8 schedule runs alone on cuda:0 (PB_FLAG_SOLO: its real op list, real
kernels, no cross-device pulls).  The host time of pb_exec_step_async (it only enqueues: every wait is
device-side in solo mode) is compared with the device time of the same step and of each pass
(CUDA events).  With the host far ahead of the device, launch overhead is hidden and CUDA graphs would
buy nothing.  The host figure is an upper bound (a full launch queue blocks the host); the device-side
idle time between passes is the direct measure of host-induced gaps.

    python tools/host_overhead.py --model 1.5b --p 8 --microbatches 32 --micro-batch 2 --out x.json
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="1.5b", choices=sorted(CONFIGS))
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--microbatches", type=int, default=32)
    ap.add_argument("--micro-batch", type=int, default=2)
    ap.add_argument("--schedules", nargs="+", default=["v-half", "1f1b"])
    ap.add_argument("--device", type=int, default=2, help="pipeline device (1-based) to run")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import DeviceExecutor, ModelConfig, synthetic_batch

    out = {"model": args.model, "p": args.p, "microbatches": args.microbatches, "micro_batch": args.micro_batch,
           "device": args.device, "runs": []}
    for name in args.schedules:
        sched = pb.assemble(pb.build_entry(name, args.p), args.microbatches)
        cfg = ModelConfig(**CONFIGS[args.model], micro_batch=args.micro_batch, optimizer=True, timeline=True,
                          solo=True)
        tok, lab = synthetic_batch(cfg, args.microbatches)
        tt, ll = torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda()
        ex = DeviceExecutor(cfg, sched, args.device, 0)
        for _ in range(2):
            ex.step(tt, ll, on_host=False)
        host, dev = [], []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ex.step_async(tt, ll, on_host=False)
            t1 = time.perf_counter()
            tl, st = ex.sync()
            host.append((t1 - t0) * 1e3)
            dev.append(st.step_ms)
        tl, st = ex.step(tt, ll, on_host=False)
        n = len(tl)
        durs = [q.duration for q in tl]
        busy = sum(durs)
        run = {"schedule": name, "passes": n, "kernel_launches_per_step": st.kernel_launches,
               "host_enqueue_ms_per_step": statistics.median(host), "device_ms_per_step": statistics.median(dev),
               "host_us_per_pass": 1e3 * statistics.median(host) / n,
               "host_us_per_launch": 1e3 * statistics.median(host) / max(st.kernel_launches, 1),
               "device_ms_per_pass_median": statistics.median(durs), "device_ms_per_pass_min": min(durs),
               "host_vs_device": statistics.median(host) / statistics.median(dev),
               "device_busy_ms": busy, "device_step_ms": st.step_ms,
               "idle_between_passes_ms": st.step_ms - busy,
               "note": "host time includes back-pressure once the launch queue is full; the device-side "
                       "idle time between passes (step - sum of pass durations, incl. the optimizer) is the "
                       "measure of host-induced gaps"}
        out["runs"].append(run)
        print(json.dumps(run), flush=True)
        del ex
        torch.cuda.synchronize()
    if args.out:
        json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
