"""Per-source-line stall breakdown of one kernel in an .ncu-rep.
usage: python tools/stall_lines.py rep kernel_regex obj mangled_substring [stall=long_sb] [top]"""
import collections
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
import ncu_io  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import sass_lines as S  # noqa: E402


def main():
    rep, kre, obj, mangled = sys.argv[1:5]
    which = sys.argv[5] if len(sys.argv) > 5 else "long_sb"
    top = int(sys.argv[6]) if len(sys.argv) > 6 else 15
    out = ncu_io.source(rep, kre)
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia = hdr.index("Address")
    cols = [c for c in hdr if c.startswith('stall_') and 'Not Issued' not in c]
    table = S.line_table(obj, mangled)
    agg = collections.defaultdict(collections.Counter)
    tot = collections.Counter()
    base = None
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break
        try:
            a = int(r[ia], 16)
        except (ValueError, IndexError):
            continue
        base = a if base is None else base
        loc = table.get(a - base, ('?', 0))
        for c in cols:
            v = float(r[hdr.index(c)] or 0)
            agg[loc][c] += v
            tot[c] += v
    T = sum(tot.values())
    print({c.replace('stall_', ''): round(100 * v / T, 1) for c, v in tot.most_common(8)})
    key = 'stall_' + which
    for loc, c in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        print(f"  {loc[0]}:{loc[1]:<5d} {which} {100 * c[key] / T:5.1f}%   all {100 * sum(c.values()) / T:5.1f}%")


if __name__ == "__main__":
    main()
