"""paper_2603_18527_b200 -- B200-native Born-series (CBS/NPBS) sweep.

The hot path of arxiv 2603.18527's solver (u <- u + M(G(Vu + f) - u) with the R_eta residual
metric), rebuilt as hand-written sm_100a CUDA behind a C ABI (include/bornsweep.h) and a
Python mirror of the reference's operator / map / driver API (api.py).
"""
from .api import (  # noqa: F401
    CdrNeumann,
    FourierDiagMap,
    HelmholtzDirichlet,
    HelmholtzPeriodic,
    IterationConfig,
    IterationTrace,
    OptimalScalarMap,
    Pipeline,
    PointwiseMap,
    RunResult,
    ScalarMap,
    run,
)
from .instances import (CONFIGS, CdrSpec, InstanceSpec, config_instances,  # noqa: F401
                        make_cdr_instances, make_instances)
from . import _native, bpfd, slab  # noqa: F401

__all__ = [
    "CdrNeumann", "FourierDiagMap", "HelmholtzDirichlet", "HelmholtzPeriodic", "IterationConfig", "IterationTrace", "OptimalScalarMap", "Pipeline", "PointwiseMap",
    "RunResult", "ScalarMap", "run", "CONFIGS", "InstanceSpec", "config_instances",
    "make_instances", "CdrSpec", "make_cdr_instances",
]
