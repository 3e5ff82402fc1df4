"""TEST INFRASTRUCTURE ONLY: regenerate tests/golden/schedules.json from the
reference's own schedule code (oracle/_ref, built from /root/reference).

    python -m oracle.gen_golden

The fixture pins the product's schedule front end on the GPU box, where
/root/reference does not exist.  Hashes use SURVEY.md App. A's definition
(FNV-1a 64 over "device,stage,kind,mb,start,duration\\n" lines in canonical order).
"""
from __future__ import annotations

import json
import os

from oracle import refpy

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "schedules.json")
ENTRIES = ["1f1b", "zb-h1", "v-min", "v-half", "v-zb"]
PAPER = (12.96, 13.22, 9.76)  # PAPER.md:594-597 single-pass times (ms)


def fnv(lines) -> str:
    h = 0xCBF29CE484222325
    for b in "".join(f"{d},{s},{k},{m},{st},{du}\n" for d, s, k, m, st, du in lines).encode():
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def cell(entry, p, m):
    passes = refpy.assemble(entry, p, m)
    peaks, mk, ub = refpy.analyze(entry, p, m)
    _, _, pb = refpy.analyze(entry, p, m, *PAPER)
    _, mk_c, _ = refpy.analyze(entry, p, m, 1, 1, 1, 0.5)
    return {"entry": entry, "p": p, "m": m, "n_passes": len(passes), "makespan": mk, "unit_bubble": ub,
            "paper_bubble": pb, "comm_half_makespan": mk_c, "peaks": peaks, "fnv1a64": fnv(passes)}


def main():
    assert refpy.build_if_possible(), "reference library unavailable"
    sweep = [cell(e, p, m) for e in ENTRIES for p in (2, 4, 8) for m in (8, 16, 32, 64)]
    extra = [cell(e, p, 16) for e in ("v-min", "v-half", "v-zb") for p in (3, 5, 6, 7)]
    extra += [cell(e, 1, m) for e in ("1f1b", "zb-h1") for m in (1, 8, 32)]
    extra += [cell(e, p, m) for e in ENTRIES for p in (2, 4) for m in (1, 2, 3)]
    full = {}
    for e, p, m in [(e, 4, 8) for e in ENTRIES] + [("v-half", 8, 16), ("v-zb", 2, 4), ("zb-h1", 1, 4)]:
        full[f"{e}/{p}/{m}"] = refpy.assemble(e, p, m)
    # the other gallery entries (gallery.hpp:186-429): looped (interleaved-*), V with fused backward
    # (1f1b-v), two microbatches per block (zb-2-3) and the twin-route replicated-weight blocks
    more = ["interleaved-1f1b", "interleaved-1f1b-uniform", "interleaved-low-mem", "1f1b-v", "zb-2-3", "gems", "chimera"]
    gallery = [cell(e, p, m) for e in more for p in (2, 3, 4, 8) for m in (4, 8, 16)
               if not (e == "chimera" and p % 2)]
    gallery += [cell(e, 1, m) for e in ("zb-2-3", "gems") for m in (2, 8)]
    for e, p, m in [("interleaved-1f1b", 4, 8), ("interleaved-1f1b-uniform", 2, 4), ("interleaved-low-mem", 4, 8),
                    ("1f1b-v", 4, 8), ("zb-2-3", 4, 8), ("gems", 2, 4), ("chimera", 4, 4)]:
        full[f"{e}/{p}/{m}"] = refpy.assemble(e, p, m)
    squeeze_only = {f"{e}/4/16": max(st + du for _, _, _, _, st, du in refpy.assemble(e, 4, 16, True, False))
                    for e in ENTRIES}
    raw = {f"{e}/4/16": max(st + du for _, _, _, _, st, du in refpy.assemble(e, 4, 16, False, False))
           for e in ENTRIES}
    docs = {f"{e}/{p}/{m}": refpy.emit(e, p, m) for e, p, m in [("v-half", 4, 8), ("1f1b", 2, 2), ("v-zb", 2, 3),
                                                                 ("interleaved-1f1b", 2, 4), ("zb-2-3", 2, 4),
                                                                 ("chimera", 2, 2)]}
    errors = {}
    for e, p, m in [("v-min", 1, 4), ("v-half", 1, 4), ("nope", 4, 4), ("1f1b", 0, 4), ("1f1b", 4, 0),
                    ("chimera", 3, 4), ("interleaved-1f1b", 1, 4), ("interleaved-low-mem", 1, 4), ("1f1b-v", 1, 4),
                    ("zb-2-3", 4, 3), ("gems", 2, 5)]:
        try:
            refpy.assemble(e, p, m)
            errors[f"{e}/{p}/{m}"] = None
        except ValueError as ex:
            errors[f"{e}/{p}/{m}"] = str(ex)
    out = {"generator": "oracle/gen_golden.py over oracle/_ref/libpipeblock_ref.so (reference headers, unmodified)",
           "paper_profile": PAPER, "sweep": sweep, "extra": extra, "gallery": gallery, "passes": full, "squeeze_only_makespan": squeeze_only,
           "raw_makespan": raw, "documents": docs, "errors": errors}
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(f"wrote {OUT}: {len(sweep)} sweep cells, {len(extra)} extra, {len(gallery)} gallery, {len(full)} full lists")


if __name__ == "__main__":
    main()
