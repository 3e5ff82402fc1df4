"""Helper for test_multiprocess_gpu: rank r runs pipeline device r+1 over CUDA IPC;
rank 0 compares loss/gradients with an in-process run of the same schedule."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2405_15362_b200 import pipeblock as pb  # noqa: E402
from paper_2405_15362_b200.executor import DeviceExecutor, ModelConfig, PipelineExecutor, synthetic_batch  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
torch.cuda.set_device(0)
cfg = ModelConfig(layers=8, hidden=256, heads=2, seq=256, vocab=1024, micro_batch=1, optimizer=False)
sched = pb.assemble(pb.build_entry("v-half", world), 8)
tok, lab = synthetic_batch(cfg, 8)
ex = DeviceExecutor(cfg, sched, rank + 1, 0)
blobs = [None] * world
dist.all_gather_object(blobs, ex.export_blob())
ex.connect_ipc(blobs)
dist.barrier()
losses = []
for _ in range(3):  # several steps: generations must carry over across steps
    ex.zero_grads()
    tl, st = ex.step(tok, lab)
    losses.append(st.loss)
grads = {n: ex.get(n, "grad") for n in ex.param_names()}
allg = [None] * world
dist.all_gather_object(allg, (grads, losses))
dist.barrier()
if rank == 0:
    merged = {k: v for g, _ in allg for k, v in g.items()}
    loss = [l for _, ls in allg for l in ls if np.isfinite(l)]
    ref = PipelineExecutor(cfg, sched)
    r = ref.step(tok, lab)
    assert all(abs(l - r.loss) < 1e-4 * abs(r.loss) for l in loss), (loss, r.loss)
    for n, g in merged.items():
        rg = ref.get(n, "grad")
        err = float(np.linalg.norm(g - rg) / max(np.linalg.norm(rg), 1e-30))
        assert err < 2e-3, (n, err)
    print("IPC_PARITY_OK", loss, r.loss, flush=True)
dist.barrier()
dist.destroy_process_group()
