"""The reference's file formats: BPFD field files, CSV exports, trace CSV and problem manifests.

Field files go through the native writer/reader (include/bornsweep_io.h, libbornsweep_host.so:
proj/src/field.cpp:37-133 layout); manifests are the reference's plain-text `key = value`
files (save_problem / load_problem, proj/src/problem_io.cpp:16-95, parsed with the rules of
Config::parse_string, proj/src/config.cpp:17-42).  Families:

  helmholtz            the reference's own periodic HelmholtzProblem (byte-compatible with the
                       reference's save_problem / load_problem) -> HelmholtzPeriodic
  helmholtz_dirichlet  the Dirichlet five-point family of configs c0-c2 (this project; same
                       keys, plus bc = dirichlet)                -> HelmholtzDirichlet
  cdr_neumann          config c4 (this project): bx / by / sigma real fields + sigma0 -> CdrNeumann
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as N

REAL64, COMPLEX128 = 0, 1


def _err(rc: int):
    msg = N.host_lib().bp_io_last_error().decode()
    raise (ValueError if rc == 1 else RuntimeError)(msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def save_field(path: str, field) -> None:
    """save_field (field.cpp:75-91): real -> real64, complex -> complex128."""
    a = np.asarray(field)
    if a.ndim != 2:
        raise ValueError("save_field: 2-D field expected")
    dtype = COMPLEX128 if np.iscomplexobj(a) else REAL64
    a = np.ascontiguousarray(a, np.complex128 if dtype else np.float64)
    rc = N.host_lib().bp_bpfd_save(os.fsencode(path), a.shape[0], a.shape[1], dtype, _dp(a))
    if rc:
        _err(rc)


def field_info(path: str):
    nx, ny, dt = C.c_int32(), C.c_int32(), C.c_int32()
    rc = N.host_lib().bp_bpfd_info(os.fsencode(path), C.byref(nx), C.byref(ny), C.byref(dt))
    if rc:
        _err(rc)
    return nx.value, ny.value, dt.value


def load_field(path: str, dtype: int | None = None) -> np.ndarray:
    """load_real_field / load_complex_field (field.cpp:93-113); dtype None = the file's."""
    nx, ny, dt = field_info(path)
    want = dt if dtype is None else dtype
    out = np.empty((nx, ny), np.complex128 if want == COMPLEX128 else np.float64)
    rc = N.host_lib().bp_bpfd_load(os.fsencode(path), nx, ny, want, _dp(out))
    if rc:
        _err(rc)
    return out


def export_csv(path: str, field) -> None:
    """export_csv (field.cpp:140-161)."""
    a = np.asarray(field)
    dtype = COMPLEX128 if np.iscomplexobj(a) else REAL64
    a = np.ascontiguousarray(a, np.complex128 if dtype else np.float64)
    rc = N.host_lib().bp_csv_export(os.fsencode(path), a.shape[0], a.shape[1], dtype, _dp(a))
    if rc:
        _err(rc)


def write_trace_csv(path: str, trace) -> None:
    """write_trace_csv (iterate.cpp:155-162) of an IterationTrace."""
    l2 = np.ascontiguousarray(trace.res_l2_rel, np.float64)
    rt = np.ascontiguousarray(trace.res_reta_rel, np.float64)
    rc = N.host_lib().bp_trace_csv_write(os.fsencode(path), len(l2), _dp(l2), _dp(rt))
    if rc:
        _err(rc)


# ---------------------------------------------------------------------------- manifests
def _g(v) -> str:
    """a double as the reference's manifest writer prints it (ostream precision 17)"""
    return "%.17g" % float(v)


def parse_manifest(text: str) -> dict:
    """Config::parse_string (config.cpp:17-42): '#' comments, [sections], key = value.
    Returns {section: {key: value}} with the unnamed section under ''."""
    out = {"": {}}
    section = ""
    for lineno, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("["):
            if not line.endswith("]"):
                raise RuntimeError(f"config line {lineno}: unterminated section header")
            section = line[1:-1].strip()
            out.setdefault(section, {})
            continue
        if "=" not in line:
            raise RuntimeError(f"config line {lineno}: expected key = value")
        k, v = line.split("=", 1)
        out.setdefault(section, {})[k.strip()] = v.strip()
    return out


def write_manifest(directory: str, stem: str, family: str, nx: int, ny: int, lx: float, ly: float,
                   scalars: list, fields: list) -> str:
    """The manifest + field files in save_problem's order (problem_io.cpp:16-60): family, nx,
    ny, lx, ly, then the family's scalars [(key, value)] and field files [(key, suffix, array)]."""
    os.makedirs(directory, exist_ok=True)
    path = os.path.join(directory, stem + ".problem")
    lines = [f"family = {family}", f"nx = {int(nx)}", f"ny = {int(ny)}", f"lx = {_g(lx)}", f"ly = {_g(ly)}"]
    lines += [f"{k} = {v if isinstance(v, str) else _g(v)}" for k, v in scalars]
    for key, suffix, arr in fields:
        fname = f"{stem}_{suffix}.bpfd"
        save_field(os.path.join(directory, fname), arr)
        lines.append(f"{key} = {fname}")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    return path


def save_problem(directory: str, stem: str, problem, member: int = 0) -> str:
    """save_problem (problem_io.cpp:16-60) for member `member` of a problem batch."""
    from .api import CdrNeumann, HelmholtzDirichlet, HelmholtzPeriodic
    if isinstance(problem, CdrNeumann):
        return write_manifest(directory, stem, "cdr_neumann", problem.nx, problem.ny, problem.lx,
                              problem.lx, [("sigma0", problem.sigma0[member])],
                              [("bx_file", "bx", problem.bx[member]), ("by_file", "by", problem.by[member]),
                               ("sigma_file", "sigma", problem.sigma[member])])
    if isinstance(problem, HelmholtzDirichlet):
        if problem.dim != 2:
            raise ValueError("save_problem: 2-D problems only (the BPFD format is 2-D)")
        periodic = isinstance(problem, HelmholtzPeriodic)
        scalars = ([] if periodic else [("bc", "dirichlet")]) + [("k0", problem.k0[member]),
                                                                  ("eta", problem.eta[member])]
        return write_manifest(directory, stem, "helmholtz" if periodic else "helmholtz_dirichlet",
                              problem.nx, problem.ny, problem.lx, problem.lx, scalars,
                              [("k2_file", "k2", problem.k2[member])])
    raise ValueError(f"save_problem: unknown problem family {type(problem).__name__}")


def read_problem(path: str) -> dict:
    """The manifest's family, grid and media as host arrays (no GPU needed)."""
    with open(path) as fh:
        cfg = parse_manifest(fh.read())[""]
    d = os.path.dirname(path)
    fam = cfg["family"]
    spec = {"family": fam, "nx": int(cfg.get("nx", 0)), "ny": int(cfg.get("ny", 0)),
            "lx": float(cfg.get("lx", 1.0)), "ly": float(cfg.get("ly", 1.0))}
    if fam in ("helmholtz", "helmholtz_dirichlet"):
        spec.update(k0=float(cfg["k0"]), eta=float(cfg["eta"]),
                    k2=load_field(os.path.join(d, cfg["k2_file"]), COMPLEX128))
    elif fam == "cdr_neumann":
        spec.update(sigma0=float(cfg["sigma0"]),
                    **{k: load_field(os.path.join(d, cfg[k + "_file"]), REAL64) for k in ("bx", "by", "sigma")})
    else:
        raise RuntimeError("load_problem: unknown family " + fam)
    return spec


def load_problem(path: str, device: int = 0):
    """load_problem (problem_io.cpp:62-93) -> a GPU problem handle of one member."""
    from .api import CdrNeumann, HelmholtzDirichlet, HelmholtzPeriodic
    s = read_problem(path)
    if s["lx"] != s["ly"]:
        raise NotImplementedError("GPU path needs lx == ly")
    if s["family"] == "helmholtz":
        return HelmholtzPeriodic(s["k2"], s["k0"], s["eta"], lx=s["lx"], device=device)
    if s["family"] == "helmholtz_dirichlet":
        return HelmholtzDirichlet(s["k2"], s["k0"], s["eta"], lx=s["lx"], device=device)
    return CdrNeumann(s["bx"], s["by"], s["sigma"], s["sigma0"], lx=s["lx"], device=device)
