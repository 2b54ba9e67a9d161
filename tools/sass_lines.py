"""Join an ncu source page (SASS, per-instruction counts) with the cubin's
line table: instructions executed and stall samples per CUDA source line.

    python tools/sass_lines.py report.ncu-rep <kernel regex> <obj.o> <mangled substring> [top]

Needs the object compiled with -lineinfo (build.py does)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(obj, mangled):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True,
                         text=True).stdout
    table = {}
    cur_fn = None
    loc = None
    inner = "--inner" in sys.argv
    new_group = True
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            here = (os.path.basename(m.group(1)), int(m.group(2)))
            if inner:
                if new_group:
                    loc = here
            elif loc is None or "inlined at" not in ln:
                loc = here
            new_group = False
            continue
        new_group = True
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn is not None and mangled in cur_fn and "$" not in cur_fn:
            table[int(m.group(1), 16)] = loc
    return table


def main():
    rep, kre, obj, mangled_sub = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import ncu_io
    out = ncu_io.source(rep, kre)
    rows = list(csv.reader(io.StringIO(out)))
    name = mangled_sub
    hdr = rows[1]
    ia, iex, ist = hdr.index("Address"), hdr.index("Instructions Executed"), \
        hdr.index("Warp Stall Sampling (All Samples)")
    table = line_table(obj, name)
    if not table:
        print("no line table for", name)
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    tot_i = tot_s = 0.0
    base = None
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break                      # only the first kernel of the page
        if len(r) <= iex:
            continue
        try:
            a = int(r[ia], 16)
        except ValueError:
            continue
        base = a if base is None else base
        a -= base
        ex, st = float(r[iex] or 0), float(r[ist] or 0)
        loc = table.get(a, ("?", 0))
        agg[loc][0] += ex
        agg[loc][1] += st
        tot_i += ex
        tot_s += st
    print(f"{name}: {tot_i:.3e} warp instructions")
    for loc, (ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {loc[0]}:{loc[1]:<5d} inst {100 * ex / tot_i:5.1f}%  stall {100 * st / max(tot_s, 1):5.1f}%")


if __name__ == "__main__":
    main()
