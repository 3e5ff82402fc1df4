"""The one-process-per-GPU path (CUDA IPC outboxes + stream memory-op flags),
exercised with every rank on the single GPU of the test box: torchrun with 2 and
4 ranks running bench.py on the tiny model, and a direct parity check of the
multi-process step against the in-process executor."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def torchrun(n, *args, timeout=300):
    env = dict(os.environ, PB_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n), *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return r.stdout


@pytest.mark.parametrize("n,sched", [(2, "v-half"), (4, "v-zb"), (2, "1f1b")])
def test_bench_torchrun_shared_gpu(n, sched):
    out = torchrun(n, "bench.py", "--gpus", str(n), "--model", "tiny", "--steps", "2", "--warmup", "1",
                   "--microbatches", "8", "--schedule", sched, "--no-cpu-baseline")
    line = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == n and line["value"] > 0
    assert 0 <= line["bubble_rate"] < 1
    assert line["activation_memory"]["measured_slots_max"] == max(line["activation_memory"]["predicted_slots_per_device"])
    tr = line["transfer"]  # every stage crossing pulled once per step, timed on the copy stream
    assert tr["bytes_per_step"] > 0 and tr["copy_ms_per_step"] > 0 and tr["achieved_gbps"] > 0
    assert tr["link"].startswith("same-gpu")


def test_ipc_step_matches_in_process():
    out = torchrun(2, "tests/_ipc_parity.py", timeout=300)
    assert "IPC_PARITY_OK" in out, out
