"""Hot SASS instructions of an ncu report (source page): samples, executed count, stall mix.
usage: python tools/ncu_sass_hot.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
si, ci, ei = h.index("# Samples"), h.index("Source"), h.index("Instructions Executed")
stalls = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
body = [r for r in rows[hi + 1:] if len(r) == len(h)]
tot = sum(int(r[si] or 0) for r in body)
texec = sum(int(r[ei] or 0) for r in body)
print(f"total samples {tot}, instructions executed {texec}")
agg = {}
for r in body:
    op = r[ci].split()[0] if r[ci] else "?"
    if op.startswith("@"):
        op = r[ci].split()[1]
    a = agg.setdefault(op, [0, 0])
    a[0] += int(r[si] or 0)
    a[1] += int(r[ei] or 0)
print("by opcode (samples, executed):")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:18]:
    print(f"  {k:28s} {v[0]:8d} {100 * v[0] / tot:5.1f}%  exec {v[1]:10d}")
print("hottest instructions:")
for idx, r in sorted(enumerate(body), key=lambda ir: -int(ir[1][si] or 0))[:top]:
    st = sorted(((int(r[i] or 0), h[i][6:]) for i in stalls), reverse=True)[:3]
    print(f"  #{idx:4d} {int(r[si] or 0):7d} {100 * int(r[si] or 0) / tot:5.1f}% exec {int(r[ei] or 0):9d}  {r[ci][:70]:70s} {st}")
