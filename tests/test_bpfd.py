"""The reference's file formats through the native writer/reader (include/bornsweep_io.h):
byte-for-byte against files the reference's own field.cpp / problem_io.cpp wrote
(tests/golden/ref_io, make_golden.py io), cross-reads, the reference's error texts, and the
trace CSV format of write_trace_csv (iterate.cpp:155-162)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2603_18527_b200 import bpfd
from paper_2603_18527_b200.api import IterationTrace
from oracle import Reference

IO = os.path.join(GOLDEN, "ref_io")


@pytest.fixture(scope="module")
def inputs():
    return np.load(os.path.join(GOLDEN, "io_inputs.npz"))


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("name,key", [("field_c", "fc"), ("field_r", "fr")])
def test_field_files_byte_exact(tmp_path, inputs, name, key):
    ours = tmp_path / f"{name}.bpfd"
    bpfd.save_field(str(ours), inputs[key])
    assert _bytes(ours) == _bytes(os.path.join(IO, f"{name}.bpfd"))
    back = bpfd.load_field(os.path.join(IO, f"{name}.bpfd"))
    assert back.dtype == inputs[key].dtype and np.array_equal(back, inputs[key])


@pytest.mark.parametrize("name,key", [("field_c", "fc"), ("field_r", "fr")])
def test_csv_export_byte_exact(tmp_path, inputs, name, key):
    ours = tmp_path / f"{name}.csv"
    bpfd.export_csv(str(ours), inputs[key])
    assert _bytes(ours) == _bytes(os.path.join(IO, f"{name}.csv"))


def test_manifest_byte_exact_and_readable(tmp_path, inputs):
    path = bpfd.write_manifest(str(tmp_path), "helm", "helmholtz", 16, 16, 1.0, 1.0,
                               [("k0", float(inputs["k0"])), ("eta", float(inputs["eta"]))],
                               [("k2_file", "k2", inputs["k2"])])
    assert _bytes(path) == _bytes(os.path.join(IO, "helm.problem"))
    assert _bytes(tmp_path / "helm_k2.bpfd") == _bytes(os.path.join(IO, "helm_k2.bpfd"))
    spec = bpfd.read_problem(os.path.join(IO, "helm.problem"))
    assert spec["family"] == "helmholtz" and spec["nx"] == spec["ny"] == 16
    assert spec["k0"] == float(inputs["k0"]) and spec["eta"] == float(inputs["eta"])
    assert np.array_equal(spec["k2"], inputs["k2"])


def test_manifest_parser_rules():
    cfg = bpfd.parse_manifest("# c\nfamily = x  # tail\n\n[sec]\n a = 1 = 2 \n")
    assert cfg[""] == {"family": "x"} and cfg["sec"] == {"a": "1 = 2"}
    with pytest.raises(RuntimeError, match="unterminated section"):
        bpfd.parse_manifest("[sec\n")
    with pytest.raises(RuntimeError, match="expected key = value"):
        bpfd.parse_manifest("novalue\n")


def test_field_errors_follow_reference(tmp_path, inputs):
    good = os.path.join(IO, "field_c.bpfd")
    with pytest.raises(RuntimeError, match="cannot open for reading"):
        bpfd.load_field(str(tmp_path / "missing.bpfd"))
    bad = tmp_path / "bad.bpfd"
    bad.write_bytes(b"XXXX" + _bytes(good)[4:])
    with pytest.raises(RuntimeError, match="bad magic"):
        bpfd.load_field(str(bad))
    bad.write_bytes(_bytes(good)[:9])
    with pytest.raises(RuntimeError, match="truncated header"):
        bpfd.load_field(str(bad))
    bad.write_bytes(_bytes(good)[:-8])
    with pytest.raises(RuntimeError, match="truncated payload"):
        bpfd.load_field(str(bad))
    with pytest.raises(RuntimeError, match="expected real64"):
        bpfd.load_field(good, dtype=bpfd.REAL64)
    with pytest.raises(RuntimeError, match="expected complex128"):
        bpfd.load_field(os.path.join(IO, "field_r.bpfd"), dtype=bpfd.COMPLEX128)


@pytest.mark.skipif(not Reference.available(), reason="reference build absent")
def test_reference_reads_our_files(tmp_path, inputs):
    """the other direction, live: the reference's loaders read what the native writer wrote"""
    bpfd.save_field(str(tmp_path / "c.bpfd"), inputs["fc"])
    assert np.array_equal(Reference.load_field(str(tmp_path / "c.bpfd"), 5, 7, True), inputs["fc"])
    path = bpfd.write_manifest(str(tmp_path), "h", "helmholtz", 16, 16, 1.0, 1.0,
                               [("k0", float(inputs["k0"])), ("eta", float(inputs["eta"]))],
                               [("k2_file", "k2", inputs["k2"])])
    spec = Reference.load_problem_helmholtz(path)
    assert spec["k0"] == float(inputs["k0"]) and spec["eta"] == float(inputs["eta"])
    assert np.array_equal(spec["k2"], inputs["k2"])


def test_trace_csv_format(tmp_path):
    tr = IterationTrace(np.array([1.0, 0.5, 1e-10, 0.1]), np.array([1.0, 0.25, 3e-11, 1 / 3]), 3,
                        "converged", 2.0, 1.0)
    p = tmp_path / "t.csv"
    bpfd.write_trace_csv(str(p), tr)
    # ostream precision(17), default float field == printf %.17g (trailing zeros dropped; the
    # same engine export_csv's byte-exact pin above exercises against the reference's output)
    assert p.read_text() == ("step,res_l2_rel,res_Reta_rel\n0,1,1\n1,0.5,0.25\n"
                             "2,1e-10,3e-11\n"
                             "3,0.10000000000000001,0.33333333333333331\n")
