"""Registers / spills / stack of every kernel in a `-Xptxas -v` log
(default paper_2505_23254_b200/lib/obj/kernels.ptxas.txt), demangled names,
optionally filtered by a substring:  python tools/ptxas_regs.py [log] [filter]"""
import re
import subprocess
import sys

log = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else \
    "paper_2505_23254_b200/lib/obj/kernels.ptxas.txt"
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
rows = {}
for line in open(log):
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        rows.setdefault(cur, {})
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        rows.setdefault(cur, {})
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows[cur]["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for mangled, d in zip(names, dem):
    if flt in d and "regs" in rows[mangled]:
        r = rows[mangled]
        print(f"{r.get('regs', '?'):>4} regs  stack {r.get('stack', 0):>4}  spill {r.get('spill_st', 0)}/{r.get('spill_ld', 0)}  {d[:150]}")
