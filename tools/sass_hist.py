"""Opcode histogram of one kernel's SASS, optionally restricted to the
instructions between two address markers:  python tools/sass_hist.py <obj>
<mangled-substring> [lo_hex hi_hex]"""
import re
import subprocess
import sys
from collections import Counter

obj, name = sys.argv[1], sys.argv[2]
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 62
funcs = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
cur, body = None, {}
for line in funcs.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        body[cur] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and cur:
        body[cur].append((int(m.group(1), 16), m.group(2).strip()))
for fn, ins in body.items():
    if name not in fn:
        continue
    sel = [t for a, t in ins if lo <= a < hi]
    ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in sel)
    print(fn, len(ins), "instructions;", len(sel), "selected")
    print("  ", ", ".join(f"{k} {v}" for k, v in ops.most_common(40)))
