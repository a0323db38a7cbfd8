"""Condense gpurun_out/ ncu artefacts into the tracked profiles/ summaries.

    python tools/make_profile_summary.py <round-tag> <config> <launches.csv | -> <full.ncu-rep>

Writes profiles/<tag>_launches.md (per-kernel launch counts and device-time shares of the
`ncu --metrics gpu__time_duration.sum` pass over bench.py), profiles/<tag>_ncu_full.md (key
`--set full` metrics of the sweep kernels) and updates profiles/ncu_summary.json: per config,
dram bytes per launch of the sweep's row kernel ("row") and column kernel ("col"), read by
bench.py for roofline.traffic."""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

tag, config, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)


def short(name):
    m = re.match(r"(?:void )?(?:<unnamed>::|bs::)?([\w]+)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


# ---- launch list
rows = [] if launches == "-" else [r for r in csv.reader(open(launches)) if len(r) > 14 and r[0].isdigit()]
agg = collections.OrderedDict()
for r in rows:
    k = short(r[4])
    t = float(r[14])
    c, s = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, s + t)
total = sum(s for _, s in agg.values())
for _ in [0] if rows else []:
  with open(os.path.join(out_dir, f"{tag}_launches.md"), "w") as fh:
    fh.write(f"# {tag} ({config}): kernel launch list of `python bench.py --no-cpu` under\n"
             f"`ncu --metrics gpu__time_duration.sum --clock-control none -c 3000`\n\n"
             f"Cold-cache, serialised per-launch times: compare SHARES, not absolutes.\n"
             f"{len(rows)} launches captured.\n\n| kernel | launches | total ms | mean us | share |\n|---|---|---|---|---|\n")
    for k, (c, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
        fh.write(f"| `{k}` | {c} | {s / 1e6:.3f} | {s / c / 1e3:.1f} | {100 * s / total:.1f}% |\n")

# ---- full set
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(out)))
hdr, units = raw[0], raw[1]
WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
        ("sm__warps_active.avg.per_cycle_active", "active warps / SM"),
        ("launch__registers_per_thread", "registers / thread"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
        ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard / issue"),
        ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue")]
summary = {}
with open(os.path.join(out_dir, f"{tag}_ncu_full.md"), "w") as fh:
    fh.write(f"# {tag}: `ncu --set full` of the {config} sweep kernels (tools/profile_sweep.py --config {config})\n\n")
    for r in raw[2:]:
        name = r[hdr.index("Kernel Name")]
        fh.write(f"## `{name}`\n\n| metric | value |\n|---|---|\n")
        vals = {}
        for m, label in WANT:
            if m in hdr:
                i = hdr.index(m)
                fh.write(f"| {label} (`{m}`) | {r[i]} {units[i]} |\n")
                vals[m] = (r[i], units[i])
        fh.write("\n")

        def to_bytes(v):
            x, u = float(v[0].replace(",", "")), v[1]
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        entry = {"kernel": name, "dram_bytes_per_launch":
                 to_bytes(vals["dram__bytes_read.sum"]) + to_bytes(vals["dram__bytes_write.sum"]),
                 "duration": " ".join(vals["gpu__time_duration.sum"])}
        # the sweep's row pass (R_SWEEP, or the c4 RC_A/RC_B pair) and its column pass
        if re.search(r"\brow_kernel<\d+, 3,|crow_kernel<\d+, 2,|prow_kernel", name):
            summary["row"] = entry
        if re.search(r"crow_kernel<\d+, 3,", name):
            summary["row_b"] = entry
        if re.search(r"tri_kernel|col_kernel<\d+, 1,|ccol_kernel<\d+, 1,", name):
            summary.setdefault("col", entry)
summary["source"] = f"profiles/{tag}_ncu_full.md (ncu --set full --clock-control none, tools/profile_sweep.py --config {config})"
path = os.path.join(out_dir, "ncu_summary.json")
try:
    doc = json.load(open(path))
    if "row_kernel" in doc:  # r01 layout (c1 only)
        doc = {}
except Exception:
    doc = {}
doc[config] = summary
json.dump(doc, open(path, "w"), indent=1)
print(json.dumps(summary, indent=1))
