"""SASS opcode histogram (warp-level instructions executed) per kernel from an ncu report.
usage: python tools/ncu_ophist.py report.ncu-rep kernel_regex [topN]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name-base", "demangled", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
hist, tot, col, ci = {}, 0, None, None
for r in csv.reader(io.StringIO(out)):
    if len(r) < 2:
        continue
    if r[0] == "Address":
        col = r.index("Instructions Executed")
        ci = r.index("Source")
        continue
    if col is None or not r[0].startswith("0x"):
        continue
    try:
        v = int(float(r[col]))
    except ValueError:
        continue
    ins = r[ci].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1]
    op = ins.split()[0] if ins else "?"
    hist[op] = hist.get(op, 0) + v
    tot += v
print("total warp instructions", tot)
for op, v in sorted(hist.items(), key=lambda x: -x[1])[:top]:
    print(f"{op:24s} {v:12d} {100 * v / tot:5.1f}%")
