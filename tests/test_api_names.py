"""Every public name of the reference package (tvqn/__init__.py and each
module's __all__) exists in the device package, module for module (the
drop-in surface of SURVEY 8b).  Uses the unmodified reference installed under
baseline/_ref (skipped when it is not installed)."""

import importlib
import sys
from pathlib import Path

import pytest

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
MODULES = ["tv_ops", "wpm", "dual_tv_solver", "hessian_sr1", "forward_models", "solvers"]


@pytest.fixture(scope="module")
def tvqn():
    if not (REF / "tvqn" / "__init__.py").exists():
        pytest.skip("reference not installed under baseline/_ref")
    sys.path.insert(0, str(REF))
    try:
        return importlib.import_module("tvqn")
    finally:
        sys.path.remove(str(REF))


def test_top_level_names(tvqn):
    import paper_2307_02043_b200 as bq

    missing = [n for n in tvqn.__all__ if not hasattr(bq, n)]
    assert not missing, missing


@pytest.mark.parametrize("mod", MODULES)
def test_module_names(tvqn, mod):
    ref = importlib.import_module(f"tvqn.{mod}")
    ours = importlib.import_module(f"paper_2307_02043_b200.{mod}")
    missing = [n for n in ref.__all__ if not hasattr(ours, n)]
    assert not missing, missing
