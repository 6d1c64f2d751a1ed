"""Registers / stack / spills per kernel from the build's ptxas logs (build/*.ptxas.txt)."""
import glob
import os
import re
import subprocess
import sys

root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2412_09734_b200", "build")
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for f in sorted(glob.glob(os.path.join(root, "*.ptxas.txt"))):
    cur = None
    rows = {}
    for ln in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", ln) or re.search(r"Function properties for (\S+)", ln)
        if m:
            cur = m.group(1)
            rows.setdefault(cur, {})
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
        if m and cur:
            rows[cur].update(stack=int(m.group(1)), st=int(m.group(2)), ld=int(m.group(3)))
        m = re.search(r"Used (\d+) registers", ln)
        if m and cur:
            rows[cur]["regs"] = int(m.group(1))
    names = list(rows)
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    for n, d in zip(names, dem):
        r = rows[n]
        if "regs" not in r or pat not in d:
            continue
        d = re.sub(r"mpax::\(anonymous namespace\)::", "", d)
        d = re.sub(r"\(.*\)$", "", d)
        print(f"{os.path.basename(f).split('.')[0]:16s} regs {r['regs']:3d} stack {r.get('stack', 0):5d} "
              f"spill st/ld {r.get('st', 0):5d}/{r.get('ld', 0):5d}  {d}")
