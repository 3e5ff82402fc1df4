"""Host side of the executor: drive a GridSchedule on B200s through the C-ABI.

The executor is the real-hardware counterpart of the reference's simulate()
(simulate.hpp:22-86): it takes the same GridSchedule, runs every pass as
sm_100a kernels in each device's grid order, and returns a TimedSchedule with
measured times plus the same accounting (makespan, busy, bubble).

Two wirings, same device code:
  * ``PipelineExecutor`` — one process, one executor per pipeline device
    (several may share a GPU for tests), peers connected with plain pointers,
    one host thread per device.
  * ``DeviceExecutor`` + ``connect_ipc`` — one process per GPU (torchrun):
    each rank builds its own device, blobs with CUDA IPC handles are exchanged
    (e.g. ``torch.distributed.all_gather_object``), then each rank steps.
No CPU fallback: without an sm_100 GPU every call raises PipeblockError.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import pipeblock as pb
from ._lib import KINDS, check, lib, pb_exec_stats, pb_model_cfg, pb_timed_pass

PB_FLAG_SERIAL = 1
PB_FLAG_TIMELINE = 2
PB_FLAG_GEMM_TIMING = 4
PB_FLAG_KERNEL_TIMING = 8
PB_FLAG_ISOLATE = 16
PB_FLAG_SOLO = 32


@dataclass
class ModelConfig:
    layers: int
    hidden: int
    heads: int
    seq: int
    vocab: int
    micro_batch: int = 1
    seed: int = 1234
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.0
    optimizer: bool = True
    timeline: bool = True
    serial: bool = False
    gemm_timing: bool = False
    solo: bool = False  # PB_FLAG_SOLO: one device of a p-device pipeline run alone (memory / timing probe)
    stage_layers: Optional[tuple] = None  # layers per stage (None: layers / num_stages each)

    @property
    def tokens_per_microbatch(self) -> int:
        return self.seq * self.micro_batch

    def c(self) -> pb_model_cfg:
        flags = ((PB_FLAG_TIMELINE if self.timeline else 0) | (PB_FLAG_SERIAL if self.serial else 0)
                 | (PB_FLAG_GEMM_TIMING if self.gemm_timing else 0) | (PB_FLAG_SOLO if self.solo else 0))
        sl = None
        if self.stage_layers is not None:
            sl = (C.c_int32 * len(self.stage_layers))(*self.stage_layers)
        c = pb_model_cfg(self.layers, self.hidden, self.heads, self.seq, self.vocab, self.micro_batch, self.seed,
                         self.lr, self.beta1, self.beta2, self.eps, self.weight_decay, int(self.optimizer), flags, sl)
        c._keep = sl  # the array must outlive the call that reads it
        return c

    def params_per_layer(self) -> int:
        return 12 * self.hidden * self.hidden + 2 * self.hidden

    def flops_per_token(self) -> Dict[str, float]:
        """Megatron convention, per token per layer; LM head 2hV per pass."""
        h, s = self.hidden, self.seq
        return {"F": 24 * h * h + 4 * s * h, "B": 24 * h * h + 8 * s * h, "W": 24 * h * h, "head": 2 * h * self.vocab}


@dataclass
class StepStats:
    loss: float
    step_ms: float
    busy_ms: float
    pool_slots: int
    pool_peak: int
    slot_bytes: int
    pool_bytes: int
    peer_bytes: int
    kernel_launches: int
    gemm_ms: float = 0.0
    gemm_flops: float = 0.0
    gemm_launches: int = 0
    copy_ms: float = 0.0

    @staticmethod
    def of(s: pb_exec_stats) -> "StepStats":
        return StepStats(s.loss, s.step_ms, s.busy_ms, s.pool_slots, s.pool_peak, s.slot_bytes, s.pool_bytes,
                         s.peer_bytes, s.kernel_launches, s.gemm_ms, s.gemm_flops, s.gemm_launches, s.copy_ms)


def _i32(x) -> C.POINTER(C.c_int32):
    """numpy int32 array (host) or torch int32 tensor (host or device) -> pointer."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.dtype == np.int32 and x.flags["C_CONTIGUOUS"]
        return x.ctypes.data_as(C.POINTER(C.c_int32))
    assert str(x.dtype) == "torch.int32" and x.is_contiguous()
    return C.cast(C.c_void_p(x.data_ptr()), C.POINTER(C.c_int32))


class DeviceExecutor:
    """One pipeline device (1-based ``device`` of the schedule) on CUDA ordinal ``cuda_device``."""

    def __init__(self, cfg: ModelConfig, schedule: pb.GridSchedule, device: int, cuda_device: int = 0):
        self.cfg, self.schedule, self.device = cfg, schedule, device
        self._cfg_c = cfg.c()
        h = C.c_void_p()
        check(lib().pb_exec_create(C.byref(self._cfg_c), schedule.handle, device, cuda_device, C.byref(h)))
        self._h = h
        n = C.c_size_t()
        check(lib().pb_exec_num_passes(h, C.byref(n)))
        self.num_passes = n.value
        self._tl = (pb_timed_pass * max(self.num_passes, 1))()

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                lib().pb_exec_destroy(h)
            except Exception:  # interpreter shutdown
                pass

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return lib().pb_exec_stream(self._h)

    # ---- IPC wiring (one process per GPU)
    def export_blob(self) -> bytes:
        n = C.c_size_t()
        check(lib().pb_exec_export(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().pb_exec_export(self._h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def connect_ipc(self, blobs: Sequence[bytes]) -> None:
        arr = (C.c_void_p * len(blobs))()
        keep = [C.create_string_buffer(b, len(b)) for b in blobs]
        for i, k in enumerate(keep):
            arr[i] = C.cast(k, C.c_void_p)
        lens = (C.c_size_t * len(blobs))(*[len(b) for b in blobs])
        check(lib().pb_exec_connect_ipc(self._h, arr, lens, len(blobs)))

    # ---- stepping
    def step(self, tokens=None, labels=None, on_host: bool = True):
        st = pb_exec_stats()
        check(lib().pb_exec_step(self._h, _i32(tokens), _i32(labels), int(on_host), self._tl, self.num_passes,
                                 C.byref(st)))
        return self.timeline(), StepStats.of(st)

    def step_async(self, tokens=None, labels=None, on_host: bool = True) -> None:
        check(lib().pb_exec_step_async(self._h, _i32(tokens), _i32(labels), int(on_host)))

    def sync(self):
        st = pb_exec_stats()
        check(lib().pb_exec_sync(self._h, self._tl, self.num_passes, C.byref(st)))
        return self.timeline(), StepStats.of(st)

    def set_flags(self, timeline: bool = True, serial: bool = False, gemm_timing: bool = False,
                  kernel_timing: bool = False, isolate: bool = False, solo: Optional[bool] = None) -> None:
        solo = self.cfg.solo if solo is None else solo
        flags = ((PB_FLAG_TIMELINE if timeline else 0) | (PB_FLAG_SERIAL if serial else 0)
                 | (PB_FLAG_GEMM_TIMING if gemm_timing else 0) | (PB_FLAG_KERNEL_TIMING if kernel_timing else 0)
                 | (PB_FLAG_ISOLATE if isolate else 0) | (PB_FLAG_SOLO if solo else 0))
        check(lib().pb_exec_set_flags(self._h, flags))
        self.cfg = __import__("dataclasses").replace(self.cfg, timeline=timeline, serial=serial, gemm_timing=gemm_timing,
                                                     solo=solo)

    def memory(self) -> Dict[str, int]:
        """Device memory of this executor (pb_exec_memory): allocation per category, and the
        device's cudaMemGetInfo used bytes before creation and at the high-water mark."""
        from ._lib import pb_exec_memory_t
        m = pb_exec_memory_t()
        check(lib().pb_exec_memory(self._h, C.byref(m)))
        return {n: int(getattr(m, n)) for n, _ in m._fields_}

    def kernel_report(self) -> Dict[str, list]:
        import json
        n = C.c_size_t()
        check(lib().pb_exec_kernel_report(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib().pb_exec_kernel_report(self._h, buf, n.value + 1, C.byref(n)))
        return json.loads(buf.value.decode() or "{}")

    def timeline(self) -> List[pb.TimedPass]:
        if not self.cfg.timeline:
            return []
        return [pb.TimedPass(p.device, p.stage, KINDS[p.kind], p.microbatch, p.start, p.duration)
                for p in self._tl[: self.num_passes]]

    # ---- parameters (parity tests)
    def param_names(self) -> List[str]:
        n = C.c_int32()
        check(lib().pb_exec_param_count(self._h, C.byref(n)))
        out = []
        buf = C.create_string_buffer(256)
        for i in range(n.value):
            check(lib().pb_exec_param_info(self._h, i, buf, 256, None))
            out.append(buf.value.decode())
        return out

    def _index(self, name: str) -> int:
        return self.param_names().index(name)

    def get(self, name: str, which: str = "weight") -> np.ndarray:
        i = self._index(name)
        n = C.c_int64()
        check(lib().pb_exec_param_info(self._h, i, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype=np.float32)
        w = {"weight": 0, "grad": 1, "master": 2}[which]
        check(lib().pb_exec_param_get(self._h, i, w, out.ctypes.data_as(C.POINTER(C.c_float))))
        return out

    def set(self, name: str, value: np.ndarray) -> None:
        v = np.ascontiguousarray(value, dtype=np.float32).ravel()
        check(lib().pb_exec_param_set(self._h, self._index(name), v.ctypes.data_as(C.POINTER(C.c_float))))

    def zero_grads(self) -> None:
        check(lib().pb_exec_zero_grads(self._h))


@dataclass
class PipelineResult:
    loss: float
    timeline: List[pb.TimedPass]
    per_device: Dict[int, StepStats]
    sim: Optional[pb.SimResult] = None

    @property
    def bubble_rate(self) -> float:
        return self.sim.bubble_rate if self.sim else float("nan")

    @property
    def makespan_ms(self) -> float:
        return self.sim.makespan if self.sim else float("nan")


class PipelineExecutor:
    """All pipeline devices in this process (one host thread per device)."""

    def __init__(self, cfg: ModelConfig, schedule: pb.GridSchedule, cuda_devices: Optional[Sequence[int]] = None):
        d = schedule.topology.devices
        cuda_devices = list(cuda_devices) if cuda_devices is not None else [0] * d
        assert len(cuda_devices) == d
        self.cfg, self.schedule = cfg, schedule
        self.devices = [DeviceExecutor(cfg, schedule, i + 1, cuda_devices[i]) for i in range(d)]
        if d > 1:
            arr = (C.c_void_p * d)(*[x.handle.value for x in self.devices])
            check(lib().pb_exec_connect_local(arr, d))
        self.first = next(x for x in self.devices if x.device == schedule.topology.device_of(1))
        self.last = next(x for x in self.devices if x.device == schedule.topology.device_of(schedule.topology.num_stages))

    def step(self, tokens, labels, on_host: bool = True) -> PipelineResult:
        results, errors = {}, []

        def run(x: DeviceExecutor):
            try:
                results[x.device] = x.step(tokens, labels, on_host)
            except Exception as e:  # noqa: BLE001
                errors.append(e)

        threads = [threading.Thread(target=run, args=(x,)) for x in self.devices]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        tl = [p for dv in sorted(results) for p in results[dv][0]]
        stats = {dv: results[dv][1] for dv in results}
        sim = pb.account(self.schedule.topology, tl) if tl else None
        # every device holding a route's last stage reports its microbatches' share of the mean loss
        # (one device for single-route schedules, two for the gems / chimera twin)
        losses = [st.loss for st in stats.values() if st.loss == st.loss]
        return PipelineResult(float(sum(losses)) if losses else float("nan"), tl, stats, sim)

    def set_flags(self, **kw) -> None:
        for x in self.devices:
            x.set_flags(**kw)

    def params(self) -> Dict[str, DeviceExecutor]:
        return {n: x for x in self.devices for n in x.param_names()}

    def get(self, name: str, which: str = "weight") -> np.ndarray:
        return self.params()[name].get(name, which)

    def set(self, name: str, value) -> None:
        self.params()[name].set(name, value)


def balanced_stage_layers(cfg: ModelConfig, topology: pb.Topology) -> tuple:
    """Layers per stage that even out per-device work when the last stage also carries the
    LM head (+ loss): head ~ V / (12h + 2s) layer-equivalents of F+B+W FLOPs (Megatron
    counts).  The reference cannot express per-stage durations;
    the paper deducts layers at the ends — this does the same, greedily:
    move one layer from the most to the least loaded device while that lowers the
    sum of squared device loads.  Every stage keeps >= 1 layer."""
    S, d = topology.num_stages, topology.devices
    head = cfg.vocab / (12.0 * cfg.hidden + 2.0 * cfg.seq)
    L = [cfg.layers // S] * S
    for i in range(cfg.layers - sum(L)):
        L[i] += 1

    def loads(L):
        out = [0.0] * (d + 1)
        for s in range(1, S + 1):
            out[topology.device_of(s)] += L[s - 1] + (head if s == S else 0.0)
        return out[1:]

    def score(L):
        return sum(x * x for x in loads(L))

    for _ in range(4 * cfg.layers):
        ld = loads(L)
        hi, lo = ld.index(max(ld)) + 1, ld.index(min(ld)) + 1
        src = [s for s in range(1, S + 1) if topology.device_of(s) == hi and L[s - 1] > 1]
        dst = [s for s in range(1, S + 1) if topology.device_of(s) == lo]
        if not src or not dst:
            break
        a = max(src, key=lambda s: (L[s - 1], s))
        b = min(dst, key=lambda s: (L[s - 1], s))
        cand = list(L)
        cand[a - 1] -= 1
        cand[b - 1] += 1
        if score(cand) >= score(L) - 1e-9:
            break
        L = cand
    return tuple(L)


def synthetic_batch(cfg: ModelConfig, microbatches: int, seed: int = 1234):
    """Uniform tokens in [0, V) with labels = tokens shifted by one."""
    rng = np.random.default_rng(seed)
    T = cfg.tokens_per_microbatch
    stream = rng.integers(0, cfg.vocab, size=(microbatches, cfg.micro_batch, cfg.seq + 1), dtype=np.int64)
    tokens = np.ascontiguousarray(stream[..., :-1].reshape(microbatches, T).astype(np.int32))
    labels = np.ascontiguousarray(stream[..., 1:].reshape(microbatches, T).astype(np.int32))
    return tokens, labels


def param_name(stage: int, layer: Optional[int], what: str) -> str:
    return f"s{stage}.{what}" if layer is None else f"s{stage}.l{layer}.{what}"
