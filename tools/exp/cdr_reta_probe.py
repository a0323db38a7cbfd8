"""Probe: fnorm_reta of CDR runs on fresh vs set_medium handles, vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2603_18527_b200 as bs
from oracle import OracleProblem

bx, by, sg, s0, f = bs.make_cdr_instances(bs.CdrSpec(n=64, seed=5), 0, 2)
cfg = bs.IterationConfig("cbs", 1e-8, 200)
o = OracleProblem.cdr(bx[0], by[0], sg[0], float(s0[0])).run(f[0] + 0j, rtol=1e-8, max_iters=200)
print("oracle fnorm_reta", o.fnorm_reta)
with bs.CdrNeumann(bx, by, sg, s0) as p:
    r = bs.run(p, bs.ScalarMap(1.0), f, cfg); print("fresh run1", r.traces[0].fnorm_reta, r.traces[0].res_reta_rel[0])
    r = bs.run(p, bs.ScalarMap(1.0), f, cfg); print("fresh run2", r.traces[0].fnorm_reta, r.traces[0].res_reta_rel[0])
    p.set_medium(bx, by, sg, s0)
    r = bs.run(p, bs.ScalarMap(1.0), f, cfg); print("after set_medium", r.traces[0].fnorm_reta, r.traces[0].res_reta_rel[0])
with bs.CdrNeumann(bx, by, sg, s0) as p:
    p.set_medium(bx, by, sg, s0)
    r = bs.run(p, bs.ScalarMap(1.0), f, cfg); print("fresh+set_medium", r.traces[0].fnorm_reta, r.traces[0].res_reta_rel[0])
    p.set_kernel_timing(True)
    r = bs.run(p, bs.ScalarMap(1.0), f, cfg); print("timing", r.traces[0].fnorm_reta, r.traces[0].res_reta_rel[0])
