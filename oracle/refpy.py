"""TEST INFRASTRUCTURE ONLY: ctypes access to oracle/_ref/libpipeblock_ref.so,
the reference's unmodified schedule code (build recipe: oracle/Makefile)."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libpipeblock_ref.so")
KINDS = ("F", "B", "W", "BW")


class RefPass(C.Structure):
    _fields_ = [("device", C.c_int32), ("stage", C.c_int32), ("kind", C.c_int32), ("microbatch", C.c_int32),
                ("start", C.c_int64), ("duration", C.c_int64)]


_L = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def build_if_possible() -> bool:
    """Compile the shim when /root/reference is mounted (this container only)."""
    if os.path.isdir("/root/reference/proj/include"):
        import subprocess
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return available()


def lib():
    global _L
    if _L is None:
        L = C.CDLL(REF_LIB)
        L.ref_last_error.restype = C.c_char_p
        L.ref_time_pipeline.restype = C.c_double
        L.ref_time_pipeline.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
        L.ref_analyze.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _L = L
    return _L


def assemble(entry: str, d: int, n: int, squeeze: bool = True, reorder: bool = True):
    """Reference assemble(build_entry(entry, d), n): list of (device, stage, kind, mb, start, dur)."""
    cnt = C.c_size_t()
    rc = lib().ref_assemble(entry.encode(), d, n, int(squeeze), int(reorder), None, 0, C.byref(cnt))
    if rc:
        raise ValueError(lib().ref_last_error().decode())
    buf = (RefPass * cnt.value)()
    rc = lib().ref_assemble(entry.encode(), d, n, int(squeeze), int(reorder), buf, cnt.value, C.byref(cnt))
    if rc:
        raise ValueError(lib().ref_last_error().decode())
    return [(p.device, p.stage, KINDS[p.kind], p.microbatch, p.start, p.duration) for p in buf]


def analyze(entry: str, d: int, n: int, f=1.0, b=1.0, w=1.0, comm=0.0):
    peaks = (C.c_double * d)()
    mk, bub = C.c_double(), C.c_double()
    rc = lib().ref_analyze(entry.encode(), d, n, f, b, w, comm, peaks, C.byref(mk), C.byref(bub))
    if rc:
        raise ValueError(lib().ref_last_error().decode())
    return list(peaks), mk.value, bub.value


def emit(entry: str, d: int, n: int) -> str:
    ln = C.c_size_t()
    if lib().ref_emit(entry.encode(), d, n, None, 0, C.byref(ln)):
        raise ValueError(lib().ref_last_error().decode())
    buf = C.create_string_buffer(ln.value + 1)
    lib().ref_emit(entry.encode(), d, n, buf, ln.value + 1, C.byref(ln))
    return buf.value.decode()


def reemit(text: str, strict: bool = False):
    ln = C.c_size_t()
    lib().ref_reemit(text.encode(), int(strict), None, 0, C.byref(ln))
    buf = C.create_string_buffer(ln.value + 1)
    rc = lib().ref_reemit(text.encode(), int(strict), buf, ln.value + 1, C.byref(ln))
    return rc, buf.value.decode()


def time_pipeline(entry: str, d: int, n: int, iters: int = 3, prof=(1.0, 1.0, 1.0)) -> float:
    return lib().ref_time_pipeline(entry.encode(), d, n, iters, *prof)


def analysis(**request):
    """Reference growth / search / frontier / render through one JSON call (ref_shim.cpp ref_analysis)."""
    import json
    text = json.dumps(request).encode()
    ln = C.c_size_t()
    lib().ref_analysis(text, None, 0, C.byref(ln))
    buf = C.create_string_buffer(ln.value + 1)
    lib().ref_analysis(text, buf, ln.value + 1, C.byref(ln))
    return json.loads(buf.value.decode())
