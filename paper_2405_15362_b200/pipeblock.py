"""Python mirror of the reference's schedule API, backed by libpb200.so.

Names, argument meaning and error behaviour follow the reference headers:

    build_entry(name, d)               gallery.hpp:499-557
    assemble(build, n, opts)           assemble.hpp:405-419 (repeat -> squeeze -> reorder)
    exact_peak(schedule)               memory.hpp:63-91
    simulate(schedule, profile)        simulate.hpp:22-86
    validate_schedule(...)             assemble.hpp:138-183 (done on every construction)
    parse(text, strict) / emit(doc)    document.hpp:188-401

Errors raise ScheduleError (the reference's std::invalid_argument) or
DocumentError (pipeblock::DocumentError) carrying the same messages.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, NamedTuple, Optional, Sequence

from ._lib import (KINDS, DocumentError, PipeblockError, ScheduleError, check, lib, pb_pass, pb_profile,
                   pb_sim_stats, pb_timed_pass, pb_topology)

__all__ = ["GridPass", "TimedPass", "Topology", "RunTimeProfile", "BlockBuild", "GridSchedule", "SimResult",
           "build_entry", "assemble", "exact_peak", "simulate", "account", "parse", "emit", "schedule_from_passes",
           "fnv1a64", "ScheduleError", "DocumentError", "PipeblockError"]


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
    h = C.c_void_p()
    check(lib().pb_schedule_build(name.encode(), d, 1, 0, 0, C.byref(h)))
    lib().pb_schedule_destroy(h)
    return BlockBuild(name, d)


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
