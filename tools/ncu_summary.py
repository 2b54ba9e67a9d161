"""Summarise an .ncu-rep: key throughput metrics, stall reasons, top SASS lines.
usage: python tools/ncu_summary.py report.ncu-rep [--sass N]"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'launch__shared_mem_per_block_dynamic', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed']


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (v, u) for h, v, u in zip(rows[0], rows[2], rows[1])}


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 0
    d = raw(rep)
    summary = {}
    for k in KEYS:
        if k in d:
            summary[k] = " ".join(d[k])
            print(f"{k:70s} {d[k][0]} {d[k][1]}")
    st = [(h, float(v)) for h, (v, u) in d.items()
          if 'smsp__average_warps_issue_stalled' in h and h.endswith('per_issue_active.ratio')]
    st.sort(key=lambda x: -x[1])
    for h, v in st[:8]:
        print("  stall", h.replace('smsp__average_warps_issue_stalled_', '')
              .replace('_per_issue_active.ratio', ''), round(v, 2))
    if nsass:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                              "sass"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr = rows[1]
        isrc, iss, iex = (hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"),
                          hdr.index("Instructions Executed"))
        data = [r for r in rows[2:] if len(r) > iex]
        tot = sum(float(r[iss] or 0) for r in data)
        for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:nsass]:
            print(f"  {100*float(r[iss] or 0)/tot:5.1f}%  {r[isrc][:60]:60s} exec={r[iex]}")
    return summary


if __name__ == "__main__":
    main()
