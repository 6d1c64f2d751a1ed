"""Per-instruction warp-stall samples of one ncu capture's source page (SASS), for the
instructions executed at least `min_exec` times: prints them in address order with their two top
stall reasons, so the attempt loop of a latency-bound kernel can be read off directly."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
min_exec = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[iS]) for r in rows[2:] if r[iS].isdigit())
loop = 0
for r in rows[2:]:
    e = int(r[iE]) if r[iE].isdigit() else 0
    if e < min_exec:
        continue
    s = int(r[iS])
    loop += s
    top = sorted(((int(r[i]) if r[i].isdigit() else 0, h[i][6:]) for i in sc), reverse=True)[:2]
    print(f"{r[0][-5:]} {e:8d} {s:5d} {r[1].strip()[:64]:64s} {top[0][1]}:{top[0][0]} {top[1][1]}:{top[1][0]}")
print(f"samples: loop {loop} of {tot} ({loop / max(tot, 1):.1%})")
