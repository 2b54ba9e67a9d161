"""Print registers / stack / spills per kernel from `nvcc -Xptxas -v` output (stdin)."""
import re
import sys

cur = None
info = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        info[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        info[cur]["stack"], info[cur]["spill_st"], info[cur]["spill_ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m:
        info[cur]["regs"] = int(m.group(1))
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for k, v in info.items():
    name = re.sub(r"_ZN\w*?(k_\w+?)I", r"\1<", k)
    if pat in name:
        print(f"{name[:60]:60s} regs={v.get('regs')} stack={v.get('stack')} spill={v.get('spill_st')}/{v.get('spill_ld')}")
