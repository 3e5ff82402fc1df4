"""compute-sanitizer evidence: one toy pipeline step (two pipeline devices sharing cuda:0,
V-Half p=2 m=4, every kernel the executor launches incl. folded-RMSNorm epilogues, attention fwd/bwd,
grouped dW, CE, AdamW), a chimera step (twin routes + replica-gradient exchange) and the stand-alone GEMM / attention entry points, run under
    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize.py
Small shapes: the sanitizer serialises and instruments every access."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import kernels as K  # noqa: E402
from paper_2405_15362_b200 import pipeblock as pb  # noqa: E402
from paper_2405_15362_b200.executor import ModelConfig, PipelineExecutor, synthetic_batch  # noqa: E402

cfg = ModelConfig(layers=4, hidden=256, heads=2, seq=256, vocab=1024, micro_batch=1, optimizer=True)
sched = pb.assemble(pb.build_entry("v-half", 2), 4)
ex = PipelineExecutor(cfg, sched, cuda_devices=[0, 0])
tokens, labels = synthetic_batch(cfg, 4)
res = ex.step(tokens, labels)
res = ex.step(tokens, labels)
print("step loss", res.loss)
# twin topology (chimera: two routes, replica-gradient exchange before AdamW)
sched2 = pb.assemble(pb.build_entry("chimera", 2), 4)
ex2 = PipelineExecutor(cfg, sched2, cuda_devices=[0, 0])
print("chimera loss", ex2.step(tokens, labels).loss)
# stand-alone GEMM (CTA pair, 512-row pair tiles) and attention at a multi-tile shape
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(512, 8192, device="cuda", generator=g).bfloat16()
W = torch.randn(256, 8192, device="cuda", generator=g).bfloat16()
C = torch.empty(512, 256, device="cuda", dtype=torch.bfloat16)
K.gemm(A, W, C)
qkv = torch.randn(512, 3 * 256, device="cuda", generator=g).bfloat16()
out, lse2 = K.attn_fwd_tc(qkv, 1, 512, 2)
dqkv = K.attn_bwd_tc(qkv, out, torch.randn_like(out), lse2, 1, 512, 2)
torch.cuda.synchronize()
print("sanitize workload done")
