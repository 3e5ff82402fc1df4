"""Schedule front end vs the reference, bit for bit.

Pinned by tests/golden/schedules.json, generated from the reference's own
headers (oracle/gen_golden.py over oracle/_ref).  When the reference library is
present (this container), the same checks also run live on extra cells.
"""
import pytest

from paper_2405_15362_b200 import pipeblock as pb

PAPER = pb.RunTimeProfile(12.96, 13.22, 9.76, 0.0)


def _check_cell(c):
    g = pb.assemble(pb.build_entry(c["entry"], c["p"]), c["m"])
    assert len(g.passes) == c["n_passes"]
    assert g.fnv1a64() == c["fnv1a64"], f"op order differs for {c['entry']} p={c['p']} m={c['m']}"
    assert pb.exact_peak(g) == c["peaks"]
    sim = pb.simulate(g, pb.RunTimeProfile.unit())
    assert sim.makespan == c["makespan"]
    assert sim.bubble_rate == pytest.approx(c["unit_bubble"], abs=1e-15)
    assert pb.simulate(g, PAPER).bubble_rate == pytest.approx(c["paper_bubble"], abs=1e-12)
    assert pb.simulate(g, pb.RunTimeProfile(1, 1, 1, 0.5)).makespan == pytest.approx(c["comm_half_makespan"])


def test_sweep_bit_exact(golden):
    # BASELINE configs[1]: p in {2,4,8} x m in {8,16,32,64} x five schedules
    assert len(golden["sweep"]) == 60
    for c in golden["sweep"]:
        _check_cell(c)


def test_extra_cells_bit_exact(golden):
    for c in golden["extra"]:
        _check_cell(c)


def test_gallery_entries_bit_exact(golden):
    # the other 10 gallery entries' newer half (gallery.hpp:186-429): interleaved-* (looped), 1f1b-v,
    # zb-2-3 and the replicated-weight twin blocks gems / chimera
    entries = {c["entry"] for c in golden["gallery"]}
    assert entries == {"interleaved-1f1b", "interleaved-1f1b-uniform", "interleaved-low-mem", "1f1b-v", "zb-2-3",
                       "gems", "chimera"}
    for c in golden["gallery"]:
        _check_cell(c)
    assert pb.gallery_names()[:5] == ["1f1b", "eager-1f1b", "gpipe", "gems", "chimera"]
    assert len(pb.gallery_names()) == 15
    for e in pb.gallery_names():
        b = pb.build_entry(e, 4)
        assert b.replicated_weights == (e in ("gems", "chimera"))
        assert b.microbatches_per_block == (2 if e in ("gems", "chimera", "zb-2-3") else 1)


def test_full_op_lists(golden):
    for key, passes in golden["passes"].items():
        e, p, m = key.split("/")
        g = pb.assemble(pb.build_entry(e, int(p)), int(m))
        assert [list(x) for x in g.passes] == [list(x) for x in passes], key


def test_appendix_a_values(golden):
    # SURVEY.md App. A (reference run during the survey): makespan and peaks
    want = {("v-half", 8, 64): (404, [10.0] * 8), ("v-min", 8, 8): (75, [6, 8, 8, 6, 8, 8, 6, 8]),
            ("v-zb", 8, 8): (55, [9, 10, 11, 12, 13, 14, 15, 16]), ("1f1b", 4, 8): (33, [4, 3, 2, 1]),
            ("zb-h1", 8, 64): (206, [8, 7, 6, 5, 4, 3, 2, 1])}
    for (e, p, m), (mk, peaks) in want.items():
        g = pb.assemble(pb.build_entry(e, p), m)
        assert g.makespan == mk
        assert pb.exact_peak(g) == [float(x) for x in peaks]


def test_squeeze_only_and_raw(golden):
    for key, mk in golden["squeeze_only_makespan"].items():
        e, p, m = key.split("/")
        assert pb.assemble(pb.build_entry(e, int(p)), int(m), True, False).makespan == mk
    for key, mk in golden["raw_makespan"].items():
        e, p, m = key.split("/")
        assert pb.assemble(pb.build_entry(e, int(p)), int(m), False, False).makespan == mk
    # test_assemble.cpp:334-345: V-Min d=4 n=16 squeezed span 107, full <= 107
    assert pb.assemble(pb.build_entry("v-min", 4), 16, True, False).makespan == 107


def test_documents_byte_identical(golden):
    for key, text in golden["documents"].items():
        e, p, m = key.split("/")
        g = pb.assemble(pb.build_entry(e, int(p)), int(m))
        assert pb.emit(g) == text, key
        back = pb.parse(text)
        assert pb.emit(back) == text
        assert back.passes == g.passes


def test_error_messages(golden):
    for key, msg in golden["errors"].items():
        e, p, m = key.split("/")
        if msg is None:
            continue
        with pytest.raises(pb.ScheduleError) as ei:
            pb.assemble(pb.BlockBuild(e, int(p)), int(m))
        assert str(ei.value) == msg


def test_vblock_cells_d4():
    # test_vblocks.cpp:52-71 frozen V-Half cells via the m=1 assembled block
    g = pb.assemble(pb.build_entry("v-half", 4), 1, False, False)
    cells = {(p.stage, p.kind): p.start for p in g.passes}
    assert [cells[(s, "F")] for s in range(1, 9)] == [0, 2, 4, 6, 8, 9, 10, 11]
    assert [cells[(s, "B")] for s in range(8, 0, -1)] == [15, 17, 19, 21, 22, 23, 24, 25]
    assert [cells[(s, "W")] for s in (8, 1, 7, 2, 6, 3, 5, 4)] == [16, 26, 19, 27, 20, 24, 23, 25]


def test_simulate_goldens():
    # test_simulate.cpp:12-58
    g = pb.assemble(pb.build_entry("1f1b", 4), 8)
    sim = pb.simulate(g)
    assert sim.makespan == 33 and sim.bubble_rate == pytest.approx(3 / 11)
    assert all(b == 24 for b in sim.busy) and all(v == 9 for v in sim.idle_total)
    assert sim.idle_span[3] == 0 and sim.idle_span[0] == 9
    assert pb.simulate(pb.assemble(pb.build_entry("1f1b", 2), 2), pb.RunTimeProfile(1, 1, 1, 1)).makespan == 11
    assert pb.simulate(pb.assemble(pb.build_entry("1f1b", 2), 3), pb.RunTimeProfile(1, 1, 1, 1)).makespan == 16
    for prof in [pb.RunTimeProfile(2, 2, 2, 0), pb.RunTimeProfile(1, 2, 1, 0), PAPER]:
        s = pb.simulate(g, prof)
        assert s.makespan == pytest.approx(11 * (prof.f + prof.b + prof.w))
        assert s.bubble_rate == pytest.approx(3 / 11)


def test_account_matches_simulate():
    g = pb.assemble(pb.build_entry("v-half", 4), 8)
    sim = pb.simulate(g, PAPER)
    acc = pb.account(g.topology, sim.schedule)
    assert acc.makespan == pytest.approx(sim.makespan)
    assert acc.bubble_rate == pytest.approx(sim.bubble_rate)
    assert acc.peak == sim.peak


def test_validation_messages():
    g = pb.assemble(pb.build_entry("1f1b", 2), 2)
    passes = [p for p in g.passes if not (p.stage == 1 and p.kind == "F" and p.microbatch == 0)]
    with pytest.raises(pb.ScheduleError, match="misses F of stage 1"):
        pb.schedule_from_passes(g.topology, passes, 2)
    moved = [p._replace(start=0) if (p.stage == 1 and p.kind == "F" and p.microbatch == 1) else p for p in g.passes]
    with pytest.raises(pb.ScheduleError, match="device 1 overlap"):
        pb.schedule_from_passes(g.topology, moved, 2)
    early = [p._replace(start=0) if (p.stage == 2 and p.kind == "F" and p.microbatch == 0) else p for p in g.passes]
    with pytest.raises(pb.ScheduleError, match="starts before its prerequisite ends"):
        pb.schedule_from_passes(g.topology, early, 2)
    ok = pb.schedule_from_passes(g.topology, g.passes, 2)
    assert ok.passes == g.passes


def test_document_errors():
    with pytest.raises(pb.DocumentError, match="malformed JSON"):
        pb.parse("{nope")
    doc = pb.emit(pb.assemble(pb.build_entry("1f1b", 2), 2))
    import json
    j = json.loads(doc)
    j["note"] = "hand edited"
    text = json.dumps(j, indent=2) + "\n"
    assert "hand edited" in pb.emit(pb.parse(text))
    with pytest.raises(pb.DocumentError, match="unknown field"):
        pb.parse(text, strict=True)
    j = json.loads(doc)
    j["passes"][1]["start"] = 0
    with pytest.raises(pb.DocumentError, match="collision on device 1 at cell"):
        pb.parse(json.dumps(j))
    j = json.loads(doc)
    j["format_version"] = 2
    with pytest.raises(pb.DocumentError, match="/format_version: unsupported format_version 2"):
        pb.parse(json.dumps(j))


def _ref():
    from oracle import refpy
    if not refpy.available():
        pytest.skip("reference library not built (no /root/reference here)")
    return refpy


def test_live_against_reference_random():
    refpy = _ref()
    import random
    rng = random.Random(7)
    for _ in range(60):
        e = rng.choice(["1f1b", "zb-h1", "v-min", "v-half", "v-zb"])
        p = rng.randint(1 if e in ("1f1b", "zb-h1") else 2, 9)
        m = rng.randint(1, 24)
        sq, re = rng.random() < 0.9, rng.random() < 0.8
        want = refpy.assemble(e, p, m, sq, re)
        got = pb.assemble(pb.build_entry(e, p), m, sq, re)
        assert [tuple(x) for x in got.passes] == want, (e, p, m, sq, re)
        peaks, mk, bub = refpy.analyze(e, p, m, 12.96, 13.22, 9.76, 0.3)
        assert pb.exact_peak(pb.assemble(pb.build_entry(e, p), m)) == peaks
        s = pb.simulate(pb.assemble(pb.build_entry(e, p), m), pb.RunTimeProfile(12.96, 13.22, 9.76, 0.3))
        assert s.makespan == mk and s.bubble_rate == bub


def test_live_document_roundtrip_reference():
    refpy = _ref()
    for e, p, m in [("v-min", 4, 4), ("zb-h1", 3, 5), ("v-zb", 8, 8)]:
        text = refpy.emit(e, p, m)
        assert pb.emit(pb.assemble(pb.build_entry(e, p), m)) == text
        rc, again = refpy.reemit(pb.emit(pb.parse(text)))
        assert rc == 0 and again == text
