"""In-tree build of libpb200.so (schedule front end + executor + sm_100a kernels).

Everything is compiled for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``)
with ``-lineinfo`` so ncu source pages map to the kernels.  cudart is linked
statically, so the library loads on a CPU-only host (schedule functions work;
executor calls report PB_ECUDA) and travels to the GPU box with the snapshot.
Incremental: an object is rebuilt when its source or any header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpb200.so")
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    out = []
    for d, _, files in os.walk(CSRC):
        for f in sorted(files):
            if f.endswith((".cpp", ".cu")):
                out.append(os.path.join(d, f))
    return sorted(out)


def _headers():
    hs = [os.path.join(ROOT, "include", "pipeblock_b200.h")]
    for d, _, files in os.walk(CSRC):
        hs += [os.path.join(d, f) for f in files if f.endswith((".hpp", ".cuh", ".h"))]
    return hs


def _flags(src):
    common = ["-O3", "-std=c++20", "-Xcompiler", "-fPIC", "-I" + CSRC, "-I" + os.path.join(ROOT, "include"),
              "-I" + JSON_DIR, "-DNDEBUG"] + ARCH
    if src.endswith(".cu"):
        extra = ["-DPB_ATTN_TRACE_BUILD"] if os.environ.get("PB_ATTN_TRACE_BUILD") else []
        extra += os.environ.get("PB_NVCC_EXTRA", "").split()  # experiments only (-D switches)
        return common + extra + ["-lineinfo", "--expt-relaxed-constexpr", "-Xptxas=-v" if os.environ.get("PB_PTXAS_V") else "-w"]
    return common


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr_mtime = max(os.path.getmtime(h) for h in _headers())
    todo, objs = [], []
    for src in _sources():
        rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
        obj = os.path.join(OBJ, rel + ".o")
        objs.append(obj)
        if not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hdr_mtime):
            todo.append((src, obj))

    def compile_one(item):
        src, obj = item
        cmd = [NVCC, "-c", src, "-o", obj] + _flags(src)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stdout + r.stderr, file=sys.stderr)
        return src

    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        for src in ex.map(compile_one, todo):
            if verbose:
                print("built", os.path.relpath(src, ROOT), file=sys.stderr)
    if todo or not os.path.exists(LIB):
        cmd = [NVCC, "-shared", "-o", LIB] + objs + ARCH + ["-cudart", "static", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
