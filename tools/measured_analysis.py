"""§8f rows 1-3 on MEASURED pass times (one B200, PB_FLAG_SOLO device probes, tools/device_probe.py).

For a model / p / m and each schedule, every pipeline device of the real schedule runs its own op list
alone on the GPU (real kernels, real footprint); the measured per-pass durations are replayed in each
device's grid order (pb_replay = simulate.hpp:44-56 with one duration per pass, comm per crossing
assumed: msg_bytes / NVLink GB/s + latency).  On that data:

  f3  the replayed measured timeline as a "time" ScheduleDocument (document.hpp:413) rendered to an SVG
      Gantt and an ASCII grid by the reference-identical renderer (render.hpp:83-256);
  f1  growth_rate (growth.hpp:141-187) under the measured per-kind profile (t_F, t_B, t_W means, comm)
      vs the measured-timeline per-microbatch makespan increment (replays of the same measured pass
      times over growing m: slope of makespan(m') for m' in [m/2, m]);
  f2  search / frontier (search.hpp:121-259) under the measured profile; each feasible winner is
      assembled at m (pb_search_assemble), probed on the GPU like the fixed blocks and replayed, so
      searched and gallery blocks are compared on measured pass times at equal memory.

    python tools/measured_analysis.py --model 1.5b --p 8 --microbatches 32 --micro-batch 2 \\
        --out profiles/r2_measured_analysis_1p5b_p8.json --svg-prefix profiles/r2_gantt_1p5b_p8
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from bench import CONFIGS  # noqa: E402
from device_probe import probe_schedule  # noqa: E402


def kind_profile(durations, comm_ms):
    """RunTimeProfile (model.hpp:189-206) of the measured means per kind; a fused BW pass counts as B + W
    in the same B:W proportion as the split passes (or 1:1 when the schedule has none)."""
    from paper_2405_15362_b200 import pipeblock as pb

    acc = {}
    for (_, _, k, _), t in durations.items():
        acc.setdefault(k, []).append(t)
    mean = {k: sum(v) / len(v) for k, v in acc.items()}
    f = mean.get("F", 0.0)
    if "B" in mean and "W" in mean:
        b, w = mean["B"], mean["W"]
    else:
        b = w = mean.get("BW", 0.0) / 2
    return pb.RunTimeProfile(f, b, w, comm_ms), mean


def growth_check(name, p, m, durations, prof, comm_ms):
    """growth_rate's predicted per-period time vs the slope of replayed measured makespans."""
    from paper_2405_15362_b200 import pipeblock as pb

    build = pb.build_entry(name, p)
    g = pb.growth_rate(build, prof)
    mpb = build.microbatches_per_block
    pts = []
    for m1 in range(max(mpb, (m // 2) // mpb * mpb), m + 1, mpb):
        s = pb.assemble(build, m1)
        rep = pb.replay(s, [durations[(q.device, q.stage, q.kind, q.microbatch)] for q in s.passes], comm_ms)
        sim = pb.simulate(s, prof)
        pts.append((m1, rep.makespan, sim.makespan))
    n = len(pts)
    xs = [x / mpb for x, _, _ in pts]
    def slope(ys):
        mx, my = sum(xs) / n, sum(ys) / n
        return sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    meas = slope([y for _, y, _ in pts])
    prof_slope = slope([y for _, _, y in pts])
    return {"schedule": name, "profile_ms": {"f": prof.f, "b": prof.b, "w": prof.w, "comm": prof.comm},
            "predicted_growth_ms_per_period": g.growth, "predicted_max_work_ms_per_period": g.max_work,
            "predicted_repeating_bubble": g.repeating_bubble, "linear_bubble": g.linear_bubble,
            "cycle_length": g.cycle_length, "witness_head": g.witness[:6],
            "measured_increment_ms_per_period": meas,
            "simulated_increment_ms_per_period_profile": prof_slope,
            "measured_vs_predicted": meas / g.growth if g.growth else None,
            "points": [{"m": a, "replayed_measured_ms": b, "simulated_profile_ms": c} for a, b, c in pts],
            "def": "period = one block repetition (microbatches_per_block microbatches); measured increment = "
                   "least-squares slope of the replayed measured makespan over m' in [m/2, m]"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="1.5b", choices=sorted(CONFIGS))
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--microbatches", type=int, default=32)
    ap.add_argument("--micro-batch", type=int, default=2)
    ap.add_argument("--schedules", nargs="+", default=["v-min", "v-half", "v-zb", "1f1b"])
    ap.add_argument("--limits", type=float, nargs="+", default=None,
                    help="search memory limits in units of m (default: the fixed V blocks' peaks)")
    ap.add_argument("--delta-max", type=int, default=3)
    ap.add_argument("--tau-max", type=int, default=3)
    ap.add_argument("--nvlink-gbs", type=float, default=720.0)
    ap.add_argument("--latency-us", type=float, default=8.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--svg-prefix", default=None)
    ap.add_argument("--layers", type=int, default=None,
                    help="override the layer count; the LM-head stage takes the remainder (ceil split), e.g. 31 = "
                         "2 per V stage + 1 on the LM-head stage at p=8")
    ap.add_argument("--balance", action="store_true", help="balanced_stage_layers: fewer layers on the LM-head stage")
    args = ap.parse_args()

    import torch

    from paper_2405_15362_b200 import pipeblock as pb
    from paper_2405_15362_b200.executor import ModelConfig, balanced_stage_layers, synthetic_batch

    mcfg = dict(CONFIGS[args.model])
    if args.layers:
        mcfg["layers"] = args.layers
    cfg0 = ModelConfig(**mcfg, micro_batch=args.micro_batch, optimizer=True, timeline=True)
    cfg = cfg0

    def split_for(topology):
        """Stage layers for this schedule's topology: balanced, the ceil split of --layers, or even."""
        S = topology.num_stages
        if args.balance:
            return tuple(balanced_stage_layers(cfg0, topology))
        if args.layers and args.layers % S:
            per = -(-args.layers // S)
            return tuple([per] * (S - 1) + [args.layers - per * (S - 1)])
        return None
    m, p, T = args.microbatches, args.p, cfg.tokens_per_microbatch
    tokens, labels = synthetic_batch(cfg, m)
    tok, lab = torch.from_numpy(tokens).cuda(), torch.from_numpy(labels).cuda()
    comm_ms = (T * cfg.hidden * 2 / (args.nvlink_gbs * 1e9) + args.latency_us * 1e-6) * 1e3
    out = {"model": f"gpt-{args.model}", "p": p, "microbatches": m, "micro_batch": args.micro_batch,
           "tokens_per_step": m * T, "comm_ms_assumed": comm_ms, "gpu": torch.cuda.get_device_name(0),
           "method": "PB_FLAG_SOLO device probes of every pipeline device (tools/device_probe.py), per-pass "
                     "CUDA-event durations replayed with pb_replay", "schedules": {}, "growth": [], "search": []}
    profiles = {}
    out["layers"] = cfg0.layers
    out["stage_layers"] = {}
    for name in args.schedules:
        sched = pb.assemble(pb.build_entry(name, p), m)
        cfg = dataclasses.replace(cfg0, stage_layers=split_for(sched.topology))
        out["stage_layers"][name] = list(cfg.stage_layers) if cfg.stage_layers else None
        run = probe_schedule(cfg, sched, name, list(range(1, p + 1)), tok, lab, 1, comm_ms)
        if "durations" not in run:
            out["schedules"][name] = {"all_fit": False, "devices": [{k: v for k, v in r.items() if k != "passes"}
                                                                   for r in run["devices"]]}
            continue
        dur, rep = run["durations"], run["replay"]
        prof, mean = kind_profile(dur, comm_ms)
        profiles[name] = prof
        out["schedules"][name] = {k: run[k] for k in ("projected_ms_per_step", "projected_tokens_per_s",
                                                      "bubble_rate", "bubble_rate_zero_comm",
                                                      "pipeline_roofline_frac", "max_activation_gib",
                                                      "max_high_water_gib", "predicted_peak_units")}
        out["schedules"][name]["mean_pass_ms"] = mean
        # f3: the replayed measured timeline through the reference-identical renderer
        if args.svg_prefix:
            title = f"{name} p={p} m={m} gpt-{args.model}: measured pass times (solo probes), replayed"
            svg = pb.render_timed(sched.topology, rep.schedule, m, "svg", title)
            with open(f"{args.svg_prefix}_{name}.svg", "w") as f:
                f.write(svg)
            with open(f"{args.svg_prefix}_{name}.txt", "w") as f:
                f.write(pb.render_timed(sched.topology, rep.schedule, m, "ascii", max_width=160))
            with open(f"{args.svg_prefix}_{name}.time.json", "w") as f:
                f.write(pb.emit_timed(sched.topology, rep.schedule, m))
        # f1: growth under the measured profile vs the measured-timeline increment
        if sched.topology.num_stages == 2 * p or name in ("1f1b", "zb-h1"):
            out["growth"].append(growth_check(name, p, m, dur, prof, comm_ms))
        print(json.dumps({"schedule": name, **{k: out["schedules"][name][k] for k in
                                               ("projected_tokens_per_s", "bubble_rate", "max_activation_gib")}}),
              file=sys.stderr, flush=True)
    # f2: search under the measured profile (the V-Half run's per-kind means), winners probed like the blocks
    src = profiles.get("v-half") or next(iter(profiles.values()), None)
    if src is not None:
        limits = args.limits or sorted({float(max(out["schedules"][s]["predicted_peak_units"]))
                                        for s in out["schedules"] if s.startswith("v-") and
                                        "predicted_peak_units" in out["schedules"][s]})
        spec = pb.SearchSpec(d=p, profile=src, delta_max=args.delta_max, tau_max=args.tau_max)
        for lim in limits:
            r = pb.search(dataclasses.replace(spec, memory_limit=lim))
            ent = {"memory_limit_m": lim, "feasible": r.feasible, "message": r.message,
                   "profile_ms": {"f": src.f, "b": src.b, "w": src.w, "comm": src.comm},
                   "enumerated": r.candidates_enumerated, "evaluated": r.candidates_evaluated}
            if r.feasible:
                ent.update({"best": r.best.str(), "predicted_bubble_eval_n": r.bubble_rate,
                            "exact_peak_m": r.exact_peak})
                sched = pb.search_assemble(p, r.best, m)
                cfg = dataclasses.replace(cfg0, stage_layers=split_for(sched.topology))
                run = probe_schedule(cfg, sched, "search", list(range(1, p + 1)), tok, lab, 1, comm_ms)
                if "durations" in run:
                    ent.update({k: run[k] for k in ("projected_tokens_per_s", "bubble_rate", "max_activation_gib",
                                                     "predicted_peak_units")})
            out["search"].append(ent)
            print(json.dumps({k: ent.get(k) for k in ("memory_limit_m", "best", "projected_tokens_per_s",
                                                      "bubble_rate")}), file=sys.stderr, flush=True)
    b = out["schedules"].get("1f1b")
    for v in list(out["schedules"].values()) + out["search"]:
        if b and b.get("projected_tokens_per_s") and v.get("projected_tokens_per_s"):
            v["tokens_per_s_vs_1f1b"] = v["projected_tokens_per_s"] / b["projected_tokens_per_s"]
            v["activation_vs_1f1b"] = v["max_activation_gib"] / b["max_activation_gib"]
    text = json.dumps(out, indent=1, default=str)
    print(text)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
