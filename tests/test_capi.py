"""The C-ABI library loads on a CPU-only host and exports every symbol the
public headers declare (no compute calls here)."""
import ctypes
import pytest
import os
import re

from paper_2405_15362_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        if f.endswith(".h"):
            text = open(os.path.join(ROOT, "include", f)).read()
            names |= set(re.findall(r"\b(pb_[a-z_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    decl = declared_symbols()
    assert decl, "no declarations found"
    missing = [n for n in sorted(decl) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= decl


def test_abi_version_and_error_slot():
    lib = _lib.lib()
    assert lib.pb_abi_version() == 1
    h = ctypes.c_void_p()
    rc = lib.pb_schedule_build(b"v-half", 1, 4, 1, 1, ctypes.byref(h))
    assert rc == _lib.PB_EINVAL
    assert lib.pb_last_error() == b"v-half: needs d >= 2"


def test_no_gpu_executor_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    lib = _lib.lib()
    h = ctypes.c_void_p()
    assert lib.pb_schedule_build(b"zb-h1", 1, 2, 1, 1, ctypes.byref(h)) == 0
    cfg = _lib.pb_model_cfg(2, 256, 2, 128, 512, 1, 1, 1e-3, 0.9, 0.95, 1e-8, 0.0, 1, 0)
    e = ctypes.c_void_p()
    rc = lib.pb_exec_create(ctypes.byref(cfg), h, 1, 0, ctypes.byref(e))
    assert rc == _lib.PB_ECUDA
    assert lib.pb_last_error()
    lib.pb_schedule_destroy(h)


def test_twin_plans_follow_routes():
    """gems / chimera route microbatches over two weight replicas (twin topology, gallery.hpp:252-326,
    model.hpp:93-107): the execution plan sends F / B messages along each microbatch's route only —
    nothing crosses from the end of route 0 (stage d) into route 1 (stage d+1) or back."""
    from tests.test_multirank_cpu import device_plan
    from paper_2405_15362_b200 import pipeblock as pb
    for e, d in (("gems", 2), ("chimera", 2), ("chimera", 4)):
        sched = pb.assemble(pb.build_entry(e, d), 4)
        topo = sched.topology
        for dev in range(1, d + 1):
            ops, slots, _ = device_plan(sched, dev)
            for o in ops:
                route = list(range(1, d + 1)) if o["mb"] % 2 == 0 else list(range(d + 1, 2 * d + 1))
                assert o["stage"] in route, (e, o)
                pos = route.index(o["stage"])
                if o["kind"] == "F":  # to the next stage of the route, none from the route's last stage
                    nxt = route[pos + 1] if pos + 1 < d else None
                    assert o["send_to"] == (topo.device_of(nxt) if nxt else 0), (e, o)
                if o["kind"] in ("B", "BW"):  # back to the previous stage, none from the route's first
                    prv = route[pos - 1] if pos > 0 else None
                    assert o["send_to"] == (topo.device_of(prv) if prv else 0), (e, o)
