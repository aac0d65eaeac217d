import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port

    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, ref_available

    if not ref_available():
        pytest.skip("oracle/_ref/libtaco_ref.so not built (reference sources absent)")
    return Ref()


def golden(name):
    import numpy as np

    return np.load(os.path.join(GOLDEN, name + ".npz"))


def golden_names(prefix=""):
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f.startswith(prefix))


def pytest_terminal_summary(terminalreporter):
    try:
        from parity import FLIP_RATE_MAX, FLIP_TALLY
    except Exception:
        return
    if FLIP_TALLY["codes"]:
        rate = FLIP_TALLY["flips"] / FLIP_TALLY["codes"]
        terminalreporter.write_line(
            f"TACO parity: {FLIP_TALLY['flips']} one-ulp code flips in {FLIP_TALLY['codes']} stage-isolated codes "
            f"(rate {rate:.3g}, gate {FLIP_RATE_MAX}), max distance {FLIP_TALLY['max_ulp']} ulp")
    if FLIP_TALLY["alphas"]:
        terminalreporter.write_line(
            f"TACO parity: alpha bit-exact in {FLIP_TALLY['alpha_exact']} of {FLIP_TALLY['alphas']} blocks, "
            f"max rel err {FLIP_TALLY['alpha_max_rel']:.3g} (gate 1e-6)")
