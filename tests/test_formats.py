"""TVQNVOL1 volumes and "tvqn-trace v1" CSVs (experiment_cli.py:35-137) are
byte-identical to files the reference harness wrote (tests/golden/ref_*)."""

from pathlib import Path

import numpy as np
import pytest

from paper_2307_02043_b200 import formats as F
from paper_2307_02043_b200.solvers import IterationTrace, TraceRow

GOLD = Path(__file__).parent / "golden"


def test_volume_bytes_match_reference(tmp_path):
    x = np.load(GOLD / "ref_formats.npz")["volume"]
    F.dump_volume(x, tmp_path / "v.tvqnvol")
    assert (tmp_path / "v.tvqnvol").read_bytes() == (GOLD / "ref_volume_5x4x3.tvqnvol").read_bytes()
    back = F.load_volume(GOLD / "ref_volume_5x4x3.tvqnvol")
    np.testing.assert_array_equal(back, x)
    # flat Fortran vector + dims (the device layout) gives the same bytes
    F.dump_volume(x.reshape(-1, order="F"), tmp_path / "w.tvqnvol", dims=(5, 4, 3))
    assert (tmp_path / "w.tvqnvol").read_bytes() == (GOLD / "ref_volume_5x4x3.tvqnvol").read_bytes()


def test_volume_errors(tmp_path):
    p = tmp_path / "bad"
    p.write_bytes(b"NOTAVOL!" + bytes(24))
    with pytest.raises(ValueError):
        F.load_volume(p)
    p.write_bytes((GOLD / "ref_volume_5x4x3.tvqnvol").read_bytes()[:-8])
    with pytest.raises(ValueError):
        F.load_volume(p)
    with pytest.raises(ValueError):
        F.dump_volume(np.zeros((2, 2, 2, 2)), tmp_path / "x")


def test_trace_bytes_match_reference(tmp_path):
    tr = IterationTrace(solver="bqnpm")
    for k in range(4):
        tr.rows.append(TraceRow(iteration=k, cost=float(1 / (k + 1) + 1e-13 * k), snr_db=float(3.25 * k + 1 / 3),
                                elapsed_s=0.125 * k, inner_iters=7 * k, grad_evals=k, full_grad_evals=0))
    F.write_trace(tr, tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_bytes() == (GOLD / "ref_trace_v1.csv").read_bytes()
    back = F.load_trace(GOLD / "ref_trace_v1.csv")
    assert back.solver == "bqnpm" and back.rows == tr.rows
    (tmp_path / "u.csv").write_text("# tvqn-trace v2\n")
    with pytest.raises(ValueError):
        F.load_trace(tmp_path / "u.csv")
