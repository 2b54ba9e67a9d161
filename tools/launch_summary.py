"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch
list: launches, mean and total time, share of all kernel time.
usage: python tools/launch_summary.py launches.csv [--json out.json]"""
import collections
import csv
import json
import sys


def main():
    rows = []
    with open(sys.argv[1]) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(
            r["Metric Unit"], 1e-6)
        name = r["Kernel Name"].split("(")[0]
        tot[name][0] += 1
        tot[name][1] += v * scale
        rows.append(r)
    all_ms = sum(t for _, t in tot.values())
    out = {}
    for name, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        out[name] = {"launches": n, "total_ms": round(t, 4), "mean_ms": round(t / n, 4),
                     "share": round(t / all_ms, 4)}
        print(f"{100 * t / all_ms:5.1f}%  {n:5d} x {t / n:8.4f} ms  {name[:90]}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
