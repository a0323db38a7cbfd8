"""Full-length solves of the BASELINE configs on the GPU, iteration counts pinned against the CPU
oracle where it finishes in minutes ("run the full-length oracle once to pin the
iteration counts").  Writes one JSON document (stdout, or --out).

    python tools/exp/full_length.py [--oracle-members 2] [--out profiles/r01c/full_length.json]

c1: all 64 members on the GPU to rtol 1e-6 (pointwise map), the oracle (plain C, OpenMP over the
transform rows) on the first --oracle-members members: iteration count and final-iterate rel-L2.
c0: GPU + oracle.  c2 / c3: GPU only (an oracle run would take hours), iteration counts recorded.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2603_18527_b200 as bs  # noqa: E402
from oracle import MAP_POINTWISE, MAP_SCALAR, Oracle, OracleProblem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--oracle-members", type=int, default=2)
ap.add_argument("--configs", default="c0,c1,c3,c2")
ap.add_argument("--out", default="")
args = ap.parse_args()
Oracle.set_threads(os.cpu_count() or 8)
MAX_ITERS = {"c0": 20000, "c1": 20000, "c2": 400000, "c3": 20000}
doc = {"host_threads": os.cpu_count()}
for name in args.configs.split(","):
    cfgd = bs.CONFIGS[name]
    dim = 3 if name == "c3" else 2
    k2, f, k0, eta = bs.config_instances(name)
    cmap = bs.PointwiseMap() if cfgd["map"] == "pointwise" else bs.ScalarMap(1.0)
    cfg = bs.IterationConfig(rtol=cfgd["rtol"], max_iters=MAX_ITERS[name])
    t0 = time.perf_counter()
    with bs.HelmholtzDirichlet(k2, k0, eta, dim=dim) as p:
        r = bs.run(p, cmap, f, cfg)
    gpu_s = time.perf_counter() - t0
    entry = {"gpu_seconds": round(gpu_s, 2), "rtol": cfgd["rtol"],
             "gpu_iters": [t.iters for t in r.traces],
             "gpu_terminated": [t.terminated for t in r.traces],
             "gpu_final_res_l2": [float(t.res_l2_rel[-1]) for t in r.traces][:4],
             "gpu_final_res_reta": [float(t.res_reta_rel[-1]) for t in r.traces][:4]}
    if name in ("c0", "c1"):
        checks = []
        for b in range(min(args.oracle_members, len(r.traces))):
            t1 = time.perf_counter()
            ref = OracleProblem(k2[b], k0[b], eta[b]).run(
                f[b], map_kind=MAP_POINTWISE if cfgd["map"] == "pointwise" else MAP_SCALAR,
                rtol=cfgd["rtol"], max_iters=MAX_ITERS[name])
            t = r.traces[b]
            k = min(t.iters, ref.iters) + 1
            checks.append({
                "member": b, "gpu_iters": t.iters, "oracle_iters": ref.iters,
                "gpu_terminated": t.terminated, "oracle_terminated": ref.terminated,
                "final_u_rel_l2": float(np.linalg.norm(r.u[b] - ref.u) / np.linalg.norm(ref.u)),
                "max_trace_rel_diff": float(np.max(np.abs(t.res_l2_rel[:k] - ref.res_l2[:k]) /
                                                   np.abs(ref.res_l2[:k]))),
                "oracle_seconds": round(time.perf_counter() - t1, 1)})
        entry["oracle_checks"] = checks
    doc[name] = entry
    print(name, json.dumps({k: v for k, v in entry.items() if k != "gpu_iters"})[:400], flush=True)
out = json.dumps(doc, indent=1)
if args.out:
    with open(args.out, "w") as fh:
        fh.write(out)
else:
    print(out)
