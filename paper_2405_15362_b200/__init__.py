"""B200-native executor for the V-shape building-block pipeline schedules of
arXiv 2405.15362 (V-Min, V-Half, V-ZB; 1F1B and ZB-H1 as baselines).

Layers:
  pipeblock  — the reference's schedule API (build_entry/assemble/simulate/parse/emit)
  executor   — runs a GridSchedule on B200s through the C-ABI (include/pipeblock_b200.h)
"""
import os as _os

# Cross-process pipeline transport uses stream memory operations; give every
# stream its own hardware queue so a device-side wait never blocks unrelated work
# (must be set before the CUDA context exists).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import pipeblock  # noqa: F401,E402

__all__ = ["pipeblock"]
