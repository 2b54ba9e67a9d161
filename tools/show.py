"""Summarise bench JSON lines: python tools/show.py file..."""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    p = d.get("passes") or {}
    out = {"cfg": d["config"]["workload"][:3], "prec": d["config"].get("precision"),
           "G/s": round(d["value"] / 1e9, 3), "ms": round(d["ms_per_step"], 3),
           "A": (round(p.get("pass_a_ms", 0), 3), round(p.get("frac_a", 0), 3)),
           "B": (round(p.get("pass_b_ms", 0), 3), round(p.get("frac_b", 0), 3)),
           "B/part": round(d["config"].get("device_bytes_per_particle") or 0)}
    if d.get("fp64"):
        out["fp64"] = round(d["fp64"]["value"] / 1e9, 3)
    if d.get("e2e"):
        out["e2e"] = round(d["e2e"]["value"] / 1e9, 3)
    if d.get("cpu_baseline") and d["cpu_baseline"].get("value"):
        out["cpu"] = round(d["cpu_baseline"]["value"] / 1e6, 3)
    out["clk"] = (d.get("clocks") or {}).get("sm_mhz")
    print(f, out)
