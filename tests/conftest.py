import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size cases (minutes of CPU oracle time)")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import PortOracle
    return PortOracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import RefOracle, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefOracle()


def load_cases(name="analyses.npz"):
    import numpy as np
    data = np.load(ROOT / "tests" / "golden" / name)
    cases = {}
    for key in data.files:
        case, field = key.split("__", 1)
        cases.setdefault(case, {})[field] = data[key]
    return cases


def case_kwargs(rec):
    kw = {k[2:]: rec[k].item() for k in rec if k.startswith("p_")}
    for k in ("n_steps", "minibatch_j", "seed", "cycle"):
        kw[k] = int(kw[k])
    return kw
