"""TEST INFRASTRUCTURE ONLY: regenerate tests/golden/analysis.json from the
reference's own growth / search / frontier / render code (oracle/_ref, built
in place from /root/reference by oracle/Makefile).

    python -m oracle.gen_golden_analysis

Pins vsched's §8f restatement (csrc/schedule/vanalysis.cpp) on the GPU box,
where /root/reference does not exist.
"""
from __future__ import annotations

import hashlib
import json
import os

from oracle import refpy

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "analysis.json")
ENTRIES = ["1f1b", "zb-h1", "v-min", "v-half", "v-zb", "zb-h2", "eager-1f1b", "gpipe", "gems", "chimera",
           "interleaved-1f1b", "interleaved-1f1b-uniform", "interleaved-low-mem", "1f1b-v", "zb-2-3"]
PROFILES = [[1, 1, 1, 0], [12.96, 13.22, 9.76, 0], [1, 2, 1, 0], [1, 1, 1, 0.5], [2.1, 2.6, 1.9, 0.05],
            [1, 3, 0.5, 0], [3, 1, 1, 0.25]]
SEARCHES = [dict(d=2, limit=4.0), dict(d=2, limit=3.0), dict(d=2, limit=2.0),
            dict(d=3, limit=4.0, delta_max=3, tau_max=3), dict(d=3, limit=6.0, delta_max=3, tau_max=3,
                                                             profile=[12.96, 13.22, 9.76, 0]),
            dict(d=4, limit=6.0, delta_max=3, tau_max=3, profile=[12.96, 13.22, 9.76, 0]),
            dict(d=4, limit=5.0, delta_max=2, tau_max=3, n=8, profile=[1, 2, 1, 0.1])]
FRONTIERS = [dict(d=2, limits=[1.0, 2.0, 3.0, 3.5, 4.0, 8.0]),
             dict(d=4, limits=[3.0, 4.0, 5.0, 6.0, 8.0], delta_max=2, tau_max=2, profile=[1, 2, 1, 0])]
RENDERS = [dict(entry=e, d=d, n=n) for e, d, n in [("v-half", 4, 8), ("v-min", 4, 16), ("1f1b", 4, 8),
                                                     ("zb-h1", 8, 32), ("v-zb", 8, 64), ("v-half", 2, 4)]]
RENDERS += [dict(entry=e, d=d, n=n) for e, d, n in [("interleaved-1f1b", 4, 8), ("interleaved-low-mem", 4, 8),
                                                      ("1f1b-v", 4, 8), ("zb-2-3", 4, 8), ("chimera", 4, 8),
                                                      ("gems", 2, 4)]]
RENDERS += [dict(entry="v-half", d=4, n=8, max_width=40), dict(entry="v-zb", d=2, n=4, color=True, title="a<b&c")]
RENDERS += [dict(entry=e, d=d, n=n, timed=True, profile=p) for e, d, n, p in
            [("v-half", 4, 8, [12.96, 13.22, 9.76, 0]), ("1f1b", 4, 8, [2.1, 2.6, 1.9, 0.05]),
             ("v-zb", 2, 6, [1, 1, 1, 0.5]), ("zb-h1", 8, 64, [0.37, 0.41, 0.29, 0.01])]]


def digest(text: str):
    """Long texts are pinned by SHA-256 (+ length) to keep the fixture small."""
    if len(text) <= 4000:
        return text
    return {"sha256": hashlib.sha256(text.encode()).hexdigest(), "len": len(text)}


def shrink(r: dict) -> dict:
    out = {k: digest(v) if isinstance(v, str) else v for k, v in r.items()}
    if "passes" in out:
        out["passes"] = digest("".join(",".join(map(str, q)) + "\n" for q in r["passes"]))
    return out


def main():
    assert refpy.build_if_possible(), "reference library unavailable"
    growth = []
    for e in ENTRIES:
        for d in (1, 2, 3, 4, 8):
            for p in PROFILES:
                r = refpy.analysis(op="growth", entry=e, d=d, profile=p)
                if "error" not in r:
                    growth.append({"entry": e, "d": d, "profile": p, **r})
    search = [{"spec": s, **shrink(refpy.analysis(op="search", **s))} for s in SEARCHES]
    front = [{"spec": s, "points": refpy.analysis(op="frontier", **s)} for s in FRONTIERS]
    render = [{"req": r, **shrink(refpy.analysis(op="render", **r))} for r in RENDERS]
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump({"source": "reference growth.hpp/search.hpp/render.hpp via oracle/_ref (oracle/gen_golden_analysis.py)",
                   "growth": growth, "search": search, "frontier": front, "render": render}, f, indent=0)
    print(f"wrote {OUT}: {len(growth)} growth, {len(search)} search, {len(front)} frontier, {len(render)} render")


if __name__ == "__main__":
    main()
