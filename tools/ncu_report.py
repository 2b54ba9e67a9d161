"""Key metrics + top stall reasons of every kernel in an .ncu-rep.
usage: python tools/ncu_report.py report.ncu-rep [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import ncu_io  # noqa: E402

KEYS = ['gpu__time_duration.sum', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.per_cycle_active', 'smsp__warps_eligible.avg.per_cycle_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'launch__shared_mem_per_block_dynamic', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active']


def main():
    out = ncu_io.raw(sys.argv[1])
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    summary = {}
    for r in rows[2:]:
        name = r[h.index('Kernel Name')]
        print(name[:70])
        d = {}
        for k in KEYS:
            if k in h:
                print(f"   {k:62s} {r[h.index(k)]} {rows[1][h.index(k)]}")
                d[k] = f"{r[h.index(k)]} {rows[1][h.index(k)]}".strip()
        st = [(k.replace('smsp__average_warps_issue_stalled_', '').replace(
            '_per_issue_active.ratio', ''), float(r[i])) for i, k in enumerate(h)
            if k.startswith('smsp__average_warps_issue_stalled') and
            k.endswith('per_issue_active.ratio') and r[i]]
        st.sort(key=lambda x: -x[1])
        print("   stalls", [(a, round(b, 2)) for a, b in st[:7]])
        d["top_stalls_per_issue"] = {a: round(b, 2) for a, b in st[:7]}
        summary[name] = d
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
