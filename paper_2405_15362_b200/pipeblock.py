"""Python mirror of the reference's schedule API, backed by libpb200.so.

Names, argument meaning and error behaviour follow the reference headers:

    build_entry(name, d)               gallery.hpp:499-557
    assemble(build, n, opts)           assemble.hpp:405-419 (repeat -> squeeze -> reorder)
    exact_peak(schedule)               memory.hpp:63-91
    simulate(schedule, profile)        simulate.hpp:22-86
    validate_schedule(...)             assemble.hpp:138-183 (done on every construction)
    parse(text, strict) / emit(doc)    document.hpp:188-401
    growth_rate / vhalf_condition ...  growth.hpp:132-205
    search / frontier                  search.hpp:208-259
    render_svg / render_ascii          render.hpp:83-256
    emit_timed / render_timed          document_from_timed (document.hpp:413) + emit / render

Errors raise ScheduleError (the reference's std::invalid_argument) or
DocumentError (pipeblock::DocumentError) carrying the same messages.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, NamedTuple, Optional, Sequence

from ._lib import (KINDS, DocumentError, PipeblockError, ScheduleError, check, lib, pb_frontier_point,
                   pb_growth_report, pb_pass, pb_profile, pb_search_result, pb_search_spec, pb_sim_stats,
                   pb_timed_pass, pb_topology)

__all__ = ["GridPass", "TimedPass", "Topology", "RunTimeProfile", "BlockBuild", "GridSchedule", "SimResult",
           "build_entry", "assemble", "exact_peak", "simulate", "replay", "account", "parse", "emit", "schedule_from_passes",
           "fnv1a64", "ScheduleError", "DocumentError", "PipeblockError", "GrowthReport", "growth_rate",
           "growth_rate_unrolled", "vhalf_condition", "lower_bound", "min_memory_for_od_bubble", "SearchSpec",
           "SearchParams", "SearchResult", "FrontierPoint", "search", "frontier", "render_svg", "render_ascii",
           "emit_timed", "render_timed"]


class GridPass(NamedTuple):  # model.hpp:162-176 (ScheduledPassT<long long>)
    device: int
    stage: int
    kind: str
    microbatch: int
    start: int
    duration: int


class TimedPass(NamedTuple):  # model.hpp:176
    device: int
    stage: int
    kind: str
    microbatch: int
    start: float
    duration: float

    @property
    def end(self) -> float:
        return self.start + self.duration


@dataclass(frozen=True)
class Topology:  # model.hpp:50-125
    devices: int
    num_stages: int
    placement: tuple
    stage_mem: tuple

    def device_of(self, stage: int) -> int:
        return self.placement[stage - 1]

    @staticmethod
    def straight(d: int) -> "Topology":
        return Topology(d, d, tuple(range(1, d + 1)), (1.0,) * d)

    @staticmethod
    def v_shape(d: int) -> "Topology":
        return Topology(d, 2 * d, tuple(list(range(1, d + 1)) + list(range(d, 0, -1))), (1.0,) * (2 * d))

    def _c(self):
        pl = (C.c_int32 * self.num_stages)(*self.placement)
        mem = (C.c_double * self.num_stages)(*self.stage_mem)
        return pb_topology(self.devices, self.num_stages, pl, mem), (pl, mem)


@dataclass(frozen=True)
class RunTimeProfile:  # model.hpp:189-206
    f: float = 1.0
    b: float = 1.0
    w: float = 1.0
    comm: float = 0.0

    @staticmethod
    def unit() -> "RunTimeProfile":
        return RunTimeProfile()


@dataclass(frozen=True)
class BlockBuild:  # gallery.hpp:16-26 (the block itself lives in the library)
    entry: str
    devices: int
    microbatches_per_block: int = 1
    replicated_weights: bool = False


@dataclass
class SimResult:  # simulate.hpp:9-17
    schedule: List[TimedPass]
    makespan: float
    busy: List[float]
    idle_total: List[float]
    idle_span: List[float]
    bubble_rate: float
    peak: List[float]


class GridSchedule:
    """An immutable validated GridSchedule (model.hpp:185) held by the library."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        d, s, m, n = C.c_int32(), C.c_int32(), C.c_int32(), C.c_size_t()
        check(lib().pb_schedule_info(handle, C.byref(d), C.byref(s), C.byref(m), C.byref(n)))
        pl = (C.c_int32 * s.value)()
        mem = (C.c_double * s.value)()
        check(lib().pb_schedule_topology(handle, pl, mem))
        self.topology = Topology(d.value, s.value, tuple(pl), tuple(mem))
        self.microbatches = m.value
        buf = (pb_pass * n.value)()
        if n.value:
            check(lib().pb_schedule_passes(handle, buf, n.value))
        self.passes: List[GridPass] = [GridPass(p.device, p.stage, KINDS[p.kind], p.microbatch, p.start, p.duration)
                                       for p in buf]

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                lib().pb_schedule_destroy(h)
            except Exception:  # interpreter shutdown
                pass

    @property
    def handle(self):
        return self._h

    def device_passes(self, device: int) -> List[GridPass]:
        return [p for p in self.passes if p.device == device]

    @property
    def makespan(self) -> int:
        return max((p.start + p.duration for p in self.passes), default=0)

    def canonical_text(self) -> str:
        """The App. A line format: device,stage,kind,microbatch,start,duration per pass."""
        return "".join(f"{p.device},{p.stage},{p.kind},{p.microbatch},{p.start},{p.duration}\n" for p in self.passes)

    def fnv1a64(self) -> str:
        return fnv1a64(self.canonical_text().encode())


def fnv1a64(data: bytes) -> str:
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def build_entry(name: str, d: int) -> BlockBuild:
    """Checks the entry/device-count combination now (gallery.hpp:499-557)."""
    mpb, rep = C.c_int32(), C.c_int32()
    check(lib().pb_build_info(name.encode(), d, C.byref(mpb), C.byref(rep)))
    return BlockBuild(name, d, mpb.value, bool(rep.value))


def gallery_names() -> List[str]:
    """The reference gallery's 15 entries in listing order (gallery.hpp:474-497)."""
    return ["1f1b", "eager-1f1b", "gpipe", "gems", "chimera", "interleaved-1f1b", "interleaved-1f1b-uniform",
            "interleaved-low-mem", "zb-h1", "zb-h2", "1f1b-v", "zb-2-3", "v-min", "v-half", "v-zb"]


def assemble(build: BlockBuild, n: int, do_squeeze: bool = True, do_reorder: bool = True) -> GridSchedule:
    h = C.c_void_p()
    check(lib().pb_schedule_build(build.entry.encode(), build.devices, n, int(do_squeeze), int(do_reorder),
                                  C.byref(h)))
    return GridSchedule(h)


def schedule_from_passes(topology: Topology, passes: Sequence[GridPass], microbatches: int) -> GridSchedule:
    arr = (pb_pass * len(passes))()
    for i, p in enumerate(passes):
        arr[i] = pb_pass(p.device, p.stage, KINDS.index(p.kind), p.microbatch, p.start, p.duration)
    topo, keep = topology._c()
    h = C.c_void_p()
    check(lib().pb_schedule_create(C.byref(topo), arr, len(passes), microbatches, C.byref(h)))
    return GridSchedule(h)


def parse(text: str, strict: bool = False) -> GridSchedule:
    h = C.c_void_p()
    check(lib().pb_schedule_parse(text.encode(), int(strict), C.byref(h)))
    return GridSchedule(h)


def emit(schedule: GridSchedule) -> str:
    n = C.c_size_t()
    check(lib().pb_schedule_emit(schedule.handle, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().pb_schedule_emit(schedule.handle, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def exact_peak(schedule: GridSchedule) -> List[float]:
    out = (C.c_double * schedule.topology.devices)()
    check(lib().pb_schedule_exact_peak(schedule.handle, out))
    return list(out)


def simulate(schedule: GridSchedule, profile: RunTimeProfile = RunTimeProfile()) -> SimResult:
    d, n = schedule.topology.devices, len(schedule.passes)
    out = (pb_timed_pass * max(n, 1))()
    st = pb_sim_stats()
    arrs = [(C.c_double * d)() for _ in range(4)]
    prof = pb_profile(profile.f, profile.b, profile.w, profile.comm)
    check(lib().pb_simulate(schedule.handle, C.byref(prof), out, n, C.byref(st), *arrs))
    timed = [TimedPass(p.device, p.stage, KINDS[p.kind], p.microbatch, p.start, p.duration) for p in out[:n]]
    return SimResult(timed, st.makespan, list(arrs[0]), list(arrs[1]), list(arrs[2]), st.bubble_rate, list(arrs[3]))


def replay(schedule: GridSchedule, durations: Sequence[float], comm: float = 0.0) -> SimResult:
    """simulate() with one duration per pass (schedule.passes order): replays measured pass times."""
    d, n = schedule.topology.devices, len(schedule.passes)
    assert len(durations) == n
    dur = (C.c_double * max(n, 1))(*durations)
    out = (pb_timed_pass * max(n, 1))()
    st = pb_sim_stats()
    arrs = [(C.c_double * d)() for _ in range(4)]
    check(lib().pb_replay(schedule.handle, dur, C.c_size_t(n), C.c_double(comm), out, C.byref(st), *arrs))
    timed = [TimedPass(p.device, p.stage, KINDS[p.kind], p.microbatch, p.start, p.duration) for p in out[:n]]
    return SimResult(timed, st.makespan, list(arrs[0]), list(arrs[1]), list(arrs[2]), st.bubble_rate, list(arrs[3]))


def account(topology: Topology, passes: Sequence[TimedPass]) -> SimResult:
    """simulate()'s accounting over measured passes (bubble per simulate.hpp:81-82)."""
    arr = (pb_timed_pass * max(len(passes), 1))()
    for i, p in enumerate(passes):
        arr[i] = pb_timed_pass(p.device, p.stage, KINDS.index(p.kind), p.microbatch, p.start, p.duration)
    topo, keep = topology._c()
    st = pb_sim_stats()
    busy = (C.c_double * topology.devices)()
    peak = (C.c_double * topology.devices)()
    check(lib().pb_account(C.byref(topo), arr, len(passes), C.byref(st), busy, peak))
    return SimResult(sorted(passes, key=lambda p: (p.device, p.start, p.stage, p.microbatch)), st.makespan,
                     list(busy), [st.makespan - b for b in busy], [], st.bubble_rate, list(peak))


# ---------------------------------------------------------------- analysis
def _text(fn, *args) -> str:
    n = C.c_size_t()
    check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def _prof(p: RunTimeProfile) -> pb_profile:
    return pb_profile(p.f, p.b, p.w, p.comm)


@dataclass
class GrowthReport:  # growth.hpp:13-22
    cycle_length: int
    growth: float
    work_per_period: List[float]
    max_work: float
    repeating_bubble: float
    linear_bubble: bool
    tie: bool
    witness: List[str]


def _block_schedule(x) -> GridSchedule:
    # a BlockBuild names a gallery block; one instance carries it (growth needs the block only)
    return assemble(x, x.microbatches_per_block, False, False) if isinstance(x, BlockBuild) else x


def growth_rate(block, profile: RunTimeProfile = RunTimeProfile()) -> GrowthReport:
    """growth_rate(blk, profile) (growth.hpp:141-187); `block` is a BlockBuild or a GridSchedule carrying one."""
    s = _block_schedule(block)
    rep = pb_growth_report()
    work = (C.c_double * s.topology.devices)()
    prof = _prof(profile)
    wit = _text(lambda *a: lib().pb_growth_rate(s.handle, C.byref(prof), C.byref(rep), work, *a))
    return GrowthReport(rep.cycle_length, rep.growth, list(work), rep.max_work, rep.repeating_bubble,
                        bool(rep.linear_bubble), bool(rep.tie), wit.splitlines())


def growth_rate_unrolled(block, profile: RunTimeProfile, periods: int) -> float:
    s = _block_schedule(block)
    out = C.c_double()
    prof = _prof(profile)
    check(lib().pb_growth_rate_unrolled(s.handle, C.byref(prof), periods, C.byref(out)))
    return out.value


def vhalf_condition(profile: RunTimeProfile) -> bool:
    out = C.c_int32()
    prof = _prof(profile)
    check(lib().pb_vhalf_condition(C.byref(prof), C.byref(out)))
    return bool(out.value)


def lower_bound(n: int, d: int, k: int) -> int:
    out = C.c_int64()
    check(lib().pb_lower_bound(n, d, k, C.byref(out)))
    return out.value


def min_memory_for_od_bubble(d: int) -> float:
    out = C.c_double()
    check(lib().pb_min_memory_for_od_bubble(d, C.byref(out)))
    return out.value


@dataclass
class SearchSpec:  # search.hpp:15-25
    d: int
    n: int = 0
    profile: RunTimeProfile = RunTimeProfile()
    memory_limit: float = 0.0
    delta_max: int = 6
    tau_max: int = 6

    def _c(self):
        return pb_search_spec(self.d, self.n, _prof(self.profile), self.memory_limit, self.delta_max, self.tau_max)


class SearchParams(NamedTuple):  # search.hpp:27-42
    K: int
    d0_lo: int
    d1_lo: int
    d0_hi: int
    d1_hi: int
    tau1: int
    tau2: int
    tau3: int

    @staticmethod
    def _from(c) -> "SearchParams":
        return SearchParams(c.K, c.d0_lo, c.d1_lo, c.d0_hi, c.d1_hi, c.tau1, c.tau2, c.tau3)

    def str(self) -> str:
        return (f"K={self.K} d0=({self.d0_lo},{self.d0_hi}) d1=({self.d1_lo},{self.d1_hi}) "
                f"tau=({self.tau1},{self.tau2},{self.tau3})")


@dataclass
class SearchResult:  # search.hpp:44-56
    feasible: bool
    message: str
    best: SearchParams
    schedule: Optional[GridSchedule]
    bubble_rate: float
    exact_peak: float
    candidates_enumerated: int
    candidates_evaluated: int
    family_min_peak: float
    turn_devices_exercised: bool


def search(spec: SearchSpec) -> SearchResult:
    """search(spec) (search.hpp:235); the winner's schedule runs on the executor unchanged."""
    r = pb_search_result()
    h = C.c_void_p()
    c = spec._c()
    msg = _text(lambda *a: lib().pb_search(C.byref(c), C.byref(r), *a[:3], C.byref(h)) if a[0] is not None
                else lib().pb_search(C.byref(c), C.byref(r), *a, None))
    return SearchResult(bool(r.feasible), msg, SearchParams._from(r.best), GridSchedule(h) if h.value else None,
                        r.bubble_rate, r.exact_peak, r.enumerated, r.evaluated, r.family_min_peak,
                        bool(r.turn_devices_exercised))


def search_assemble(d: int, params: "SearchParams", n: int) -> GridSchedule:
    """The searched family block `params` at d devices assembled with n microbatches (run it on the executor)."""
    from ._lib import pb_search_params
    c = pb_search_params(*params)
    h = C.c_void_p()
    check(lib().pb_search_assemble(d, C.byref(c), n, C.byref(h)))
    return GridSchedule(h)


@dataclass
class FrontierPoint:  # search.hpp:58-64
    limit: float
    feasible: bool
    bubble_rate: float
    exact_peak: float
    best: SearchParams


def frontier(spec: SearchSpec, limits: Sequence[float]) -> List[FrontierPoint]:
    c = spec._c()
    arr = (C.c_double * max(1, len(limits)))(*limits)
    out = (pb_frontier_point * max(1, len(limits)))()
    check(lib().pb_frontier(C.byref(c), arr, len(limits), out))
    return [FrontierPoint(p.limit, bool(p.feasible), p.bubble_rate, p.exact_peak, SearchParams._from(p.best))
            for p in out[:len(limits)]]


PB_RENDER_SVG, PB_RENDER_ASCII = 0, 1


def render_svg(schedule: GridSchedule, title: str = "") -> str:
    """render_svg(document) (render.hpp:83-172) of the schedule's document."""
    return _text(lambda *a: lib().pb_render(schedule.handle, PB_RENDER_SVG, title.encode(), 0, 0, *a))


def render_ascii(schedule: GridSchedule, max_width: int = 200, color: bool = False) -> str:
    """render_ascii(document) (render.hpp:177-256)."""
    return _text(lambda *a: lib().pb_render(schedule.handle, PB_RENDER_ASCII, None, max_width, int(color), *a))


def _timed_c(passes: Sequence[TimedPass]):
    arr = (pb_timed_pass * max(len(passes), 1))()
    for i, p in enumerate(passes):
        arr[i] = pb_timed_pass(p.device, p.stage, KINDS.index(p.kind), p.microbatch, p.start, p.duration)
    return arr


def emit_timed(topology: Topology, passes: Sequence[TimedPass], microbatches: int) -> str:
    """emit(document_from_timed(...)) (document.hpp:188,413): a measured timeline as a 'time' document."""
    topo, keep = topology._c()
    arr = _timed_c(passes)
    return _text(lambda *a: lib().pb_timed_emit(C.byref(topo), arr, len(passes), microbatches, *a))


def render_timed(topology: Topology, passes: Sequence[TimedPass], microbatches: int, fmt: str = "svg",
                 title: str = "", max_width: int = 200) -> str:
    topo, keep = topology._c()
    arr = _timed_c(passes)
    f = PB_RENDER_ASCII if fmt == "ascii" else PB_RENDER_SVG
    return _text(lambda *a: lib().pb_timed_render(C.byref(topo), arr, len(passes), microbatches, f, title.encode(),
                                                  max_width, *a))
