"""Pipe utilisation and warp-stall summary of one kernel in an `ncu --set full --import-source on`
report (markdown on stdout).

    python tools/ncu_stalls.py report.ncu-rep [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys

PIPES = [
    ("tensor pipe active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
    ("XU (SFU) instructions", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    ("FMA pipe active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("shared memory (tensor wavefronts)", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("TMEM reads by MMA (C operand)", "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum.pct_of_peak_sustained_elapsed"),
    ("TMEM reads by tcgen05.ld", "smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed"),
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    kre = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
    raw = ncu_csv(rep, "raw")
    head = raw[0]
    rows = [r for r in raw[2:] if kre.search(r[head.index("Kernel Name")])]
    r = rows[0]
    print(f"kernel `{r[head.index('Kernel Name')][:90]}`, {r[head.index('gpu__time_duration.sum')]} us\n")
    print("| unit | % of peak |\n|---|---|")
    for name, key in PIPES:
        if key in head:
            print(f"| {name} | {float(r[head.index(key)]):.1f} |")
    src = ncu_csv(rep, "source", ["--print-source", "sass"])
    h = src[1]
    data = src[2:]
    i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    cols = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
    tot = sum(float(x[i_s] or 0) for x in data)
    agg = {}
    for x in data:
        for i in cols:
            agg[h[i]] = agg.get(h[i], 0.0) + float(x[i] or 0)
    print("\n| stall reason (all warps) | % of samples |\n|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]:
        print(f"| {k} | {100 * v / tot:.1f} |")
    print("\n| SASS (top sampled) | % of samples | main reason |\n|---|---|---|")
    for x in sorted(data, key=lambda x: -float(x[i_s] or 0))[:8]:
        top = max(cols, key=lambda i: float(x[i] or 0))
        print(f"| `{x[i_src].strip()[:70]}` | {100 * float(x[i_s]) / tot:.1f} | {h[top]} |")


if __name__ == "__main__":
    main()
