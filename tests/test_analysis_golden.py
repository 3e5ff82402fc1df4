"""§8f analysis rows — growth (growth.hpp), adaptive search / frontier (search.hpp),
SVG/ASCII rendering of grid and timed documents (render.hpp, document.hpp:413) —
bit-exact against the reference's own code (tests/golden/analysis.json, generated
by oracle/gen_golden_analysis.py from oracle/_ref)."""
import hashlib
import json
import os

import pytest

from paper_2405_15362_b200 import pipeblock as pb

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "analysis.json")))


def prof(p):
    return pb.RunTimeProfile(*p)


def same_text(ours: str, gold):
    if isinstance(gold, dict):
        assert len(ours) == gold["len"]
        assert hashlib.sha256(ours.encode()).hexdigest() == gold["sha256"]
    else:
        assert ours == gold


@pytest.mark.parametrize("g", GOLD["growth"], ids=lambda g: f"{g['entry']}-d{g['d']}-{g['profile']}")
def test_growth_matches_reference(g):
    blk = pb.build_entry(g["entry"], g["d"])
    r = pb.growth_rate(blk, prof(g["profile"]))
    assert r.cycle_length == g["cycle_length"]
    assert r.growth == g["growth"]
    assert r.work_per_period == g["work"]
    assert r.max_work == g["max_work"]
    assert r.repeating_bubble == g["repeating_bubble"]
    assert (r.linear_bubble, r.tie) == (g["linear_bubble"], g["tie"])
    assert r.witness == g["witness"]
    assert pb.growth_rate_unrolled(blk, prof(g["profile"]), 3) == g["unrolled3"]


def spec_of(s):
    return pb.SearchSpec(d=s["d"], n=s.get("n", 0), profile=prof(s.get("profile", [1, 1, 1, 0])),
                         memory_limit=s.get("limit", 0.0), delta_max=s.get("delta_max", 6),
                         tau_max=s.get("tau_max", 6))


@pytest.mark.parametrize("g", GOLD["search"], ids=lambda g: json.dumps(g["spec"]))
def test_search_matches_reference(g):
    r = pb.search(spec_of(g["spec"]))
    assert r.feasible == g["feasible"] and r.message == g["message"]
    assert list(r.best) == g["best"] and r.best.str() == g["best_str"]
    assert (r.bubble_rate, r.exact_peak) == (g["bubble_rate"], g["exact_peak"])
    assert (r.candidates_enumerated, r.candidates_evaluated) == (g["enumerated"], g["evaluated"])
    assert r.family_min_peak == g["family_min_peak"] and r.turn_devices_exercised == g["turn"]
    if r.feasible:
        kinds = {"F": 0, "B": 1, "W": 2, "BW": 3}
        text = "".join(f"{p.device},{p.stage},{kinds[p.kind]},{p.microbatch},{p.start},{p.duration}\n"
                       for p in r.schedule.passes)
        same_text(text, g["passes"])


def test_search_infeasible_message():
    r = pb.search(pb.SearchSpec(d=2, memory_limit=1.0, delta_max=2, tau_max=2))
    assert not r.feasible and r.schedule is None
    assert r.message == "infeasible: memory limit 1m is below the family minimum 4m"


@pytest.mark.parametrize("g", GOLD["frontier"], ids=lambda g: json.dumps(g["spec"]))
def test_frontier_matches_reference(g):
    pts = pb.frontier(spec_of(g["spec"]), g["spec"]["limits"])
    assert len(pts) == len(g["points"])
    for p, q in zip(pts, g["points"]):
        assert (p.limit, p.feasible, p.bubble_rate, p.exact_peak, list(p.best)) == \
            (q["limit"], q["feasible"], q["bubble_rate"], q["exact_peak"], q["best"])


@pytest.mark.parametrize("g", GOLD["render"], ids=lambda g: json.dumps(g["req"]))
def test_render_matches_reference(g):
    rq = g["req"]
    s = pb.assemble(pb.build_entry(rq["entry"], rq["d"]), rq["n"])
    if rq.get("timed"):
        sim = pb.simulate(s, prof(rq["profile"]))
        same_text(pb.emit_timed(s.topology, sim.schedule, s.microbatches), g["emit"])
        same_text(pb.render_timed(s.topology, sim.schedule, s.microbatches, "svg", rq.get("title", "")), g["svg"])
        same_text(pb.render_timed(s.topology, sim.schedule, s.microbatches, "ascii",
                                  max_width=rq.get("max_width", 200)), g["ascii"])
    else:
        same_text(pb.render_svg(s, rq.get("title", "")), g["svg"])
        same_text(pb.render_ascii(s, rq.get("max_width", 200), rq.get("color", False)), g["ascii"])


def test_growth_helpers():
    assert pb.vhalf_condition(pb.RunTimeProfile(1, 1, 1)) is True
    assert pb.vhalf_condition(pb.RunTimeProfile(3, 1, 0.5)) is False
    assert pb.lower_bound(16, 4, 8) == 96 and pb.lower_bound(4, 4, 1) == 44
    assert pb.min_memory_for_od_bubble(8) == 16.0
    with pytest.raises(pb.ScheduleError, match="k must be in"):
        pb.lower_bound(4, 4, 9)
    with pytest.raises(pb.ScheduleError, match="d must be positive"):
        pb.min_memory_for_od_bubble(0)


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference not mounted")
def test_live_random_growth_vs_reference():
    import random

    from oracle import refpy
    refpy.build_if_possible()
    rng = random.Random(11)
    for _ in range(40):
        e = rng.choice(["1f1b", "zb-h1", "v-min", "v-half", "v-zb"])
        d = rng.randint(2, 8)
        p = [round(rng.uniform(0.2, 3), 2) for _ in range(3)] + [round(rng.uniform(0, 0.5), 2)]
        g = refpy.analysis(op="growth", entry=e, d=d, profile=p)
        r = pb.growth_rate(pb.build_entry(e, d), prof(p))
        assert (r.growth, r.witness, r.cycle_length) == (g["growth"], g["witness"], g["cycle_length"])


def test_search_assemble_reproduces_the_winner():
    """pb_search_assemble(d, winner, eval_n) is the search's own winner schedule bit for bit; at another
    microbatch count it is the same block repeated (what the executor runs)."""
    r = pb.search(pb.SearchSpec(d=3, profile=pb.RunTimeProfile(1, 1.2, 0.8, 0), memory_limit=6.0, delta_max=3,
                                tau_max=3))
    assert r.feasible
    same = pb.search_assemble(3, r.best, r.schedule.microbatches)
    assert [tuple(x) for x in same.passes] == [tuple(x) for x in r.schedule.passes]
    big = pb.search_assemble(3, r.best, 24)
    assert big.microbatches == 24 and max(pb.exact_peak(big)) <= 6.0
    with pytest.raises(pb.ScheduleError if hasattr(pb, "ScheduleError") else Exception):
        pb.search_assemble(1, r.best, 8)
