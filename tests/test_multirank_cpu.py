"""N>1 host path on CPU: one process per pipeline device over torch.distributed
(gloo, 127.0.0.1), each rank driving ITS device's plan from the C-ABI
(pb_plan_device) in grid order with the executor's pull protocol — outbox
slot + generation per message, acknowledgement before an outbox slot is
reused, activation-pool slots from the plan.  The per-stage arithmetic is a
tiny float64 tanh layer so the gradients can be checked exactly against a
serial run; what is under test is the plan and the protocol (deadlock
freedom, message matching, WAR safety of outboxes and pool slots), i.e. the
same host logic the GPU ranks run over CUDA IPC."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_15362_b200 import _lib
from paper_2405_15362_b200 import pipeblock as pb

N = 8  # feature width of the toy stage


def device_plan(sched, device):
    n, slots, outboxes = C.c_size_t(), C.c_int32(), C.c_int32()
    L = _lib.lib()
    _lib.check(L.pb_plan_device(sched.handle, device, None, 0, C.byref(n), C.byref(slots), C.byref(outboxes)))
    buf = (_lib.pb_plan_op * max(1, n.value))()
    _lib.check(L.pb_plan_device(sched.handle, device, buf, n.value, C.byref(n), None, None))
    ops = [dict(stage=o.stage, kind=_lib.KINDS[o.kind],
                mb=o.microbatch, slot=o.slot, start=o.start, recv_from=o.recv_from, recv_outbox=o.recv_outbox,
                recv_gen=o.recv_gen, send_to=o.send_to, send_outbox=o.send_outbox, send_gen=o.send_gen)
           for o in buf[:n.value]]
    return ops, slots.value, outboxes.value


def weights(S):
    g = np.random.default_rng(5)
    return {s: g.standard_normal((N, N)) / np.sqrt(N) for s in range(1, S + 1)}


def inputs(m):
    return np.random.default_rng(9).standard_normal((m, N))


def serial_grads(S, m):
    W = weights(S)
    X = inputs(m)
    dW = {s: np.zeros((N, N)) for s in W}
    loss = 0.0
    for mb in range(m):
        xs, ys = [], []
        x = X[mb]
        for s in range(1, S + 1):
            y = np.tanh(W[s] @ x)
            xs.append(x)
            ys.append(y)
            x = y
        loss += 0.5 * float(x @ x)
        g = x
        for s in range(S, 0, -1):
            gz = g * (1 - ys[s - 1] ** 2)
            dW[s] += np.outer(gz, xs[s - 1])
            g = W[s].T @ gz
    return loss, dW


def tag(outbox, gen, ack):
    return ((outbox * 4096 + gen) << 1) | ack


def rank_main(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for entry, m in cases:
            sched = pb.assemble(pb.build_entry(entry, world), m)
            S = sched.topology.num_stages
            dev = rank + 1
            ops, nslots, noutbox = device_plan(sched, dev)
            # 1) every rank derives the same message layout: my sends == their receives
            allplans = [None] * world
            dist.all_gather_object(allplans, [(o["stage"], o["kind"], o["mb"], o["send_to"], o["send_outbox"],
                                               o["send_gen"], o["recv_from"], o["recv_outbox"], o["recv_gen"])
                                              for o in ops])
            sends = sorted((dev, t[3], t[4], t[5]) for d, pl in enumerate(allplans, 1) if d == dev for t in pl if t[3])
            recvs = sorted((t[6], d, t[7], t[8]) for d, pl in enumerate(allplans, 1) for t in pl if t[6] == dev)
            assert sends == recvs, (entry, sends, recvs)
            assert nslots == int(pb.exact_peak(sched)[rank]), (entry, nslots)
            # 2) run the step with the pull protocol
            W = weights(S)
            X = inputs(m)
            dW = {s: np.zeros((N, N)) for s in W if sched.topology.device_of(s) == dev}
            pool = [None] * nslots
            outbox = {}            # outbox slot -> (gen, payload) for local consumers
            last_use = {}          # outbox slot -> (gen, consumer device) of the current occupant
            pending = []
            loss = 0.0
            for o in ops:
                s, k, mb = o["stage"], o["kind"], o["mb"]
                inp = None
                if o["recv_from"]:
                    if o["recv_from"] == dev:
                        g_, inp = outbox[o["recv_outbox"]]
                        assert g_ == o["recv_gen"]
                    else:
                        t = torch.empty(N, dtype=torch.float64)
                        dist.recv(t, src=o["recv_from"] - 1, tag=tag(o["recv_outbox"], o["recv_gen"], 0))
                        inp = t.numpy()
                        ack = torch.zeros(1)
                        pending.append(dist.isend(ack, dst=o["recv_from"] - 1,
                                                  tag=tag(o["recv_outbox"], o["recv_gen"], 1)))
                out = None
                if k == "F":
                    assert pool[o["slot"]] is None, "activation slot still live (WAR)"
                    x = X[mb] if s == 1 else inp
                    y = np.tanh(W[s] @ x)
                    pool[o["slot"]] = {"x": x, "y": y}
                    out = y
                    if s == S:
                        loss += 0.5 * float(y @ y)
                else:
                    st = pool[o["slot"]]
                    if k in ("B", "BW"):
                        g = st["y"] if s == S else inp
                        st["gz"] = g * (1 - st["y"] ** 2)
                        out = W[s].T @ st["gz"]
                    if k in ("W", "BW"):
                        dW[s] += np.outer(st["gz"], st["x"])
                        pool[o["slot"]] = None
                if o["send_to"]:
                    kb, gen = o["send_outbox"], o["send_gen"]
                    prev = last_use.get(kb)
                    if prev is not None:
                        assert prev[0] == gen - 1
                        if prev[1] != dev:  # previous occupant pulled by a peer: wait for its ack
                            dist.recv(torch.zeros(1), src=prev[1] - 1, tag=tag(kb, prev[0], 1))
                    last_use[kb] = (gen, o["send_to"])
                    if o["send_to"] == dev:
                        outbox[kb] = (gen, out)
                    else:
                        t = torch.from_numpy(np.ascontiguousarray(out))
                        pending.append(dist.isend(t, dst=o["send_to"] - 1, tag=tag(kb, gen, 0)))
            for kb, (gen, cons) in last_use.items():  # drain the last acknowledgements of the step
                if cons != dev:
                    dist.recv(torch.zeros(1), src=cons - 1, tag=tag(kb, gen, 1))
            for p in pending:
                p.wait()
            assert all(x is None for x in pool), "activation slot leaked"
            res = [None] * world
            dist.all_gather_object(res, (loss, dW))
            if rank == 0:
                q.put((entry, m, sum(r[0] for r in res), {s: g for r in res for s, g in r[1].items()}))
            dist.barrier()
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,cases", [
    (2, [("v-half", 4), ("zb-h1", 4), ("v-zb", 6), ("1f1b", 3)]),
    (4, [("v-zb", 8), ("v-half", 8), ("v-min", 12), ("1f1b", 8), ("zb-h1", 5)]),
])
def test_pull_protocol_multirank(world, cases):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=rank_main, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in cases]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for entry, m, loss, dW in results:
        S = 2 * world if entry.startswith("v-") else world
        loss_ref, dW_ref = serial_grads(S, m)
        assert abs(loss - loss_ref) < 1e-9 * max(1, abs(loss_ref)), entry
        assert sorted(dW) == list(range(1, S + 1))
        for s in dW:
            np.testing.assert_allclose(dW[s], dW_ref[s], rtol=1e-10, atol=1e-12, err_msg=f"{entry} stage {s}")
