import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs under `pytest -m gpu`)")


def _has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import restatement

    return restatement()


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    d = os.path.join(ROOT, "tests", "golden")
    return {n[:-4]: np.load(os.path.join(d, n)) for n in os.listdir(d) if n.endswith(".npz")}


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Print (and keep under gpurun_out/) the achieved max error of every tolerance check."""
    from tests._parity_log import ERRORS

    if not ERRORS:
        return
    import json

    worst = {}
    for e in ERRORS:
        key = (e["test"].split("[")[0], e["what"].split(" ")[0])
        if key not in worst or e["max_err"] / e["tol"] > worst[key]["max_err"] / worst[key]["tol"]:
            worst[key] = e
    terminalreporter.section("achieved parity errors (worst per test and quantity)")
    for (t, w), e in sorted(worst.items()):
        terminalreporter.write_line(f"{t:60s} {w:14s} max {e['max_err']:.3e}  (bar {e['tol']:.0e})")
    out = os.path.join(ROOT, "gpurun_out")
    try:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "parity_errors.json"), "w") as f:
            json.dump(ERRORS, f, indent=0)
    except OSError:
        pass
