"""Per-kernel in-step time breakdown (CUDA events around every launch) for one bench-like step."""
import json
import sys

import torch

from paper_2405_15362_b200 import pipeblock as pb
from paper_2405_15362_b200.executor import DeviceExecutor, ModelConfig, synthetic_batch

mbs = int(sys.argv[1]) if len(sys.argv) > 1 else 1
m = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = ModelConfig(layers=32, hidden=2048, heads=16, seq=2048, vocab=50304, micro_batch=mbs)
sched = pb.assemble(pb.build_entry("zb-h1", 1), m)
ex = DeviceExecutor(cfg, sched, 1, 0)
tok, lab = synthetic_batch(cfg, m)
tt, ll = torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda()
for _ in range(2):
    ex.step(tt, ll, on_host=False)
_, st = ex.step(tt, ll, on_host=False)
ex.set_flags(timeline=False, kernel_timing=True)
_, st2 = ex.step(tt, ll, on_host=False)
rep = ex.kernel_report()
tot = sum(v[0] for v in rep.values())
print(json.dumps({"mbs": mbs, "m": m, "step_ms_plain": st.step_ms, "step_ms_timed": st2.step_ms,
                  "sum_kernel_event_ms": tot}))
for k, (ms, n) in sorted(rep.items(), key=lambda x: -x[1][0]):
    print(f"{k:16s} {ms:9.2f} ms {100 * ms / st.step_ms:5.1f}% of plain step  n={n:6d} avg={1e3 * ms / n:8.1f} us")
