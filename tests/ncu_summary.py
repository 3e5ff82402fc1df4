"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import io
import re
import sys


def load(path):
    text = open(path).read()
    start = text.index('"ID"')
    return list(csv.DictReader(io.StringIO(text[start:])))


def key(name):
    m = re.search(r"(gemm_kernel<[^>]*>|\w+_kernel)", name)
    return m.group(1) if m else name[:60]


def main(path):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in load(path):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
        a = agg[key(r["Kernel Name"])]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>8s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:44s} {n:8d} {t / 1e3:9.2f} {t / tot * 100:5.1f}% {t / n:8.1f}")
    print(f"{'TOTAL':44s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:9.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
