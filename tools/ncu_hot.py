"""Summarise an ncu report's source page: stall samples per CUDA source line (and top SASS).
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [topN]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
col_name = sys.argv[4] if len(sys.argv) > 4 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
agg, sass, fn_tot = {}, [], {}
cur_file, cur_fn, cur_line = "", "", ""
for r in csv.reader(io.StringIO(out)):
    if len(r) < 2:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if r[0] == "Line No":
        col = r.index(col_name, 3)
        continue
    if r[0]:
        cur_line = f"{cur_file}:{r[0]} {r[1].strip()[:80]}"
    try:
        v = int(float(r[col]))
    except (ValueError, IndexError):
        continue
    key = (cur_fn, cur_line)
    agg[key] = agg.get(key, 0) + v
    fn_tot[cur_fn] = fn_tot.get(cur_fn, 0) + v
    sass.append((v, cur_fn, r[3].strip()[:50], cur_line))
for fn, tot in fn_tot.items():
    print("=====", fn, "samples", tot)
    items = sorted(((v, l) for (f, l), v in agg.items() if f == fn), reverse=True)[:top]
    for v, l in items:
        print(f"{100 * v / max(tot, 1):5.1f}%  {l}")
    print("-- top SASS")
    for v, f, s, l in sorted([x for x in sass if x[1] == fn], reverse=True)[:12]:
        print(f"{100 * v / max(tot, 1):5.1f}%  {s:50s} {l[:60]}")
