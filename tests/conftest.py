import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmdsx.so")
    config.addinivalue_line("markers", "slow: full-size BASELINE configurations")


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def sign_fixed_rel_err(got, ref) -> float:
    """Relative Frobenius error after per-column sign fixing (the north-star
    comparison); columns whose sign is ambiguous (zero dot) keep +."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    s = np.sign(np.sum(got * ref, axis=0))
    s[s == 0] = 1.0
    return float(np.linalg.norm(got * s - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2007_11919_b200  # noqa: F401
    from paper_2007_11919_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)
