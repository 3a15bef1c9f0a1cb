"""CPU-side checks: the C-ABI library loads and exports every symbol the
header declares (no device calls), the ctypes table covers them, and the
host-side parameter logic matches the reference (test_algorithms.py:38-62)."""

import re
from pathlib import Path

import pytest

from paper_2007_11919_b200 import AlgorithmParams, ParamError, run_algorithm
from paper_2007_11919_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "mdsx.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|int32_t|int64_t|const char\*)\s+(mdsx_\w+)\(", text, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "mdsx_divide_conquer" in syms and "mdsx_interpolation" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_ctypes_table_matches_header():
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_library_version_without_device():
    assert _lib.load().mdsx_version() == 1


class TestParamResolution:
    def test_defaults(self):
        d = AlgorithmParams(r=3).resolved("divide")
        assert d.l == 400 and d.c == 6
        f = AlgorithmParams(r=3).resolved("fast")
        assert f.l == 1000 and f.s == 6
        assert AlgorithmParams(r=3).resolved("interpolate").l == 1000

    @pytest.mark.parametrize("algorithm,params", [
        ("divide", AlgorithmParams(r=5, c=3)),
        ("divide", AlgorithmParams(r=2, l=4, c=4)),
        ("fast", AlgorithmParams(r=5, s=3)),
        ("fast", AlgorithmParams(r=2, l=6, s=4)),
        ("divide", AlgorithmParams(r=0)),
        ("interpolate", AlgorithmParams(r=2, l=1)),
        ("divide", AlgorithmParams(r=2, l=50_000)),
    ])
    def test_rejects_bad_params(self, algorithm, params):
        with pytest.raises(ParamError):
            params.resolved(algorithm)

    def test_unknown_algorithm(self):
        import numpy as np
        with pytest.raises(ParamError):
            run_algorithm("nope", np.zeros((10, 2)), AlgorithmParams(r=1))


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a device")
    import numpy as np
    from paper_2007_11919_b200 import divide_and_conquer_mds
    with pytest.raises(RuntimeError, match="CUDA device"):
        divide_and_conquer_mds(np.ones((10, 2)), AlgorithmParams(r=1))
