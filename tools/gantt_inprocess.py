"""Gantt of a MEASURED pipeline step (not a replay): every pipeline device of the schedule runs as its
own executor on cuda:0 (in-process group, one host thread per device, device-side waits), one real
step, and the executor's CUDA-event timeline (pb_exec_step's TimedSchedule) is emitted as a "time"
ScheduleDocument (document.hpp:413) and rendered by the reference-identical renderer
(render.hpp:83-256).  The devices time-share one GPU here, so pass durations include contention;
the op order, dependencies and the measured bubble are those of the real run.

    python tools/gantt_inprocess.py --out-prefix profiles/r2_gantt_inprocess
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out-prefix", required=True)
    ap.add_argument("--cases", nargs="+", default=["v-half:2:8", "v-zb:4:8", "1f1b:4:8"])
    args = ap.parse_args()

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import ModelConfig, PipelineExecutor, synthetic_batch

    summary = []
    for case in args.cases:
        name, p, m = case.split(":")
        p, m = int(p), int(m)
        sched = pb.assemble(pb.build_entry(name, p), m)
        S = sched.topology.num_stages
        # 1.5B-shaped layers (h=2048, 16 heads, s=2048, V=50304), one layer per stage
        cfg = ModelConfig(layers=S, hidden=2048, heads=16, seq=2048, vocab=50304, micro_batch=1, optimizer=True)
        ex = PipelineExecutor(cfg, sched)
        tokens, labels = synthetic_batch(cfg, m)
        ex.step(tokens, labels)  # warm-up
        res = ex.step(tokens, labels)
        stem = f"{args.out_prefix}_{name}_p{p}_m{m}"
        title = f"{name} p={p} m={m}: measured step on one B200 (devices time-share the GPU)"
        open(stem + ".svg", "w").write(pb.render_timed(sched.topology, res.timeline, m, "svg", title))
        open(stem + ".txt", "w").write(pb.render_timed(sched.topology, res.timeline, m, "ascii", max_width=160))
        open(stem + ".time.json", "w").write(pb.emit_timed(sched.topology, res.timeline, m))
        row = {"schedule": name, "p": p, "m": m, "layers": S, "makespan_ms": res.makespan_ms,
               "bubble_rate": res.bubble_rate, "loss": res.loss,
               "slots": {d: st.pool_slots for d, st in res.per_device.items()},
               "predicted_peak": [int(x) for x in pb.exact_peak(sched)]}
        summary.append(row)
        print(json.dumps(row), flush=True)
        del ex
    json.dump(summary, open(args.out_prefix + "_summary.json", "w"), indent=1)


if __name__ == "__main__":
    main()
