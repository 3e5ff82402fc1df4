"""Summarise `ncu --set full` captures (.ncu-rep) into a small JSON + markdown table.

    python tools/ncu_full_summary.py gpurun_out/gemm_full.ncu-rep gpurun_out/attn_full.ncu-rep > profiles/rN_ncu_full.md
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "tensor_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_throughput_pct": "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
    "sm_active_cycles": "sm__cycles_active.avg",
    "elapsed_cycles": "sm__cycles_elapsed.avg",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "regs": "launch__registers_per_thread",
}
SCALE = {"us": 1.0, "ms": 1e3, "ns": 1e-3, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        rec = {"kernel": row[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                v *= SCALE.get(units[i], 1.0) if k in ("duration_us", "dram_read_bytes", "dram_write_bytes", "sm_clock_ghz") else 1.0
                rec[k] = v
        yield rec


def main(paths):
    recs = [r for p in paths for r in rows(p)]
    print("| kernel | us | SM GHz | tensor active % | SM % | L2 % | DRAM % | DRAM read MB | DRAM write MB | SM active/elapsed |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in recs:
        act = r.get("sm_active_cycles", 0) / max(1.0, r.get("elapsed_cycles", 1))
        print(f"| `{r['kernel'][:60]}` | {r.get('duration_us', 0):.1f} | {r.get('sm_clock_ghz', 0):.2f} | "
              f"{r.get('tensor_active_pct', 0):.1f} | {r.get('sm_throughput_pct', 0):.1f} | {r.get('l2_throughput_pct', 0):.1f} | "
              f"{r.get('dram_throughput_pct', 0):.1f} | {r.get('dram_read_bytes', 0) / 1e6:.1f} | "
              f"{r.get('dram_write_bytes', 0) / 1e6:.1f} | {act:.2f} |")
    print()
    print("```json")
    print(json.dumps(recs, indent=1))
    print("```")


if __name__ == "__main__":
    main(sys.argv[1:])
