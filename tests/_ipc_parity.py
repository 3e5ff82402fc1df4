"""Helper for test_multiprocess_gpu: rank r runs pipeline device r+1 over CUDA IPC;
rank 0 compares loss/gradients with an in-process run of the same schedule.

Options (argv):
  --distinct   rank r on cuda:r (distinct physical GPUs: NVLink P2P), else every rank on cuda:0
  --async-opt  optimizer on, 3 back-to-back pb_exec_step_async before one sync (pipelined steps,
               cross-step generations and the WAR guard); weights compared after the 3 steps
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2405_15362_b200 import pipeblock as pb  # noqa: E402
from paper_2405_15362_b200.executor import DeviceExecutor, ModelConfig, PipelineExecutor, synthetic_batch  # noqa: E402

distinct = "--distinct" in sys.argv
async_opt = "--async-opt" in sys.argv
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
gpu = rank if distinct else 0
torch.cuda.set_device(gpu)
cfg = ModelConfig(layers=8, hidden=256, heads=2, seq=256, vocab=1024, micro_batch=1, optimizer=async_opt, lr=1e-3)
sched = pb.assemble(pb.build_entry("v-half", world), 8)
tok, lab = synthetic_batch(cfg, 8)
ex = DeviceExecutor(cfg, sched, rank + 1, gpu)
blobs = [None] * world
dist.all_gather_object(blobs, ex.export_blob())
ex.connect_ipc(blobs)
dist.barrier()
losses = []
w0 = {n: ex.get(n, "weight") for n in ex.param_names()}
if async_opt:
    for _ in range(3):
        ex.step_async(tok, lab)
    tl, st = ex.sync()
    losses.append(st.loss)
    what = "weight"
else:
    for _ in range(3):  # several steps: generations must carry over across steps
        ex.zero_grads()
        tl, st = ex.step(tok, lab)
        losses.append(st.loss)
    what = "grad"
tensors = {n: ex.get(n, what) - (w0[n] if async_opt else 0) for n in ex.param_names()}  # grads / weight updates
peer = st.peer_bytes
allg = [None] * world
dist.all_gather_object(allg, (tensors, losses, peer, str(torch.cuda.get_device_properties(gpu).uuid)))
dist.barrier()
if rank == 0:
    merged = {k: v for g, *_ in allg for k, v in g.items()}
    loss = [l for _, ls, *_ in allg for l in ls if np.isfinite(l)]
    assert all(pb_ > 0 for _, _, pb_, _ in allg), "every device pulls stage-boundary tensors"
    if distinct:
        assert len({u for *_, u in allg}) == world, "ranks must sit on distinct GPUs"
    ref = PipelineExecutor(cfg, sched, [0] * world)
    r0 = {n: ref.get(n, "weight") for n in merged}
    for _ in range(3 if async_opt else 1):
        r = ref.step(tok, lab)
    assert all(abs(l - r.loss) < 1e-4 * abs(r.loss) for l in loss), (loss, r.loss)
    for n, g in merged.items():
        rg = ref.get(n, what) - (r0[n] if async_opt else 0)
        err = float(np.linalg.norm(g - rg) / max(np.linalg.norm(rg), 1e-30))
        assert err < (2e-2 if async_opt else 2e-3), (n, err)
    print("IPC_PARITY_OK", "distinct" if distinct else "shared", "async-opt" if async_opt else "sync", loss, r.loss,
          flush=True)
dist.barrier()
dist.destroy_process_group()
