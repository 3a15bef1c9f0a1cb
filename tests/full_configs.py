"""BASELINE configurations 2-5 at their full sizes, shared by the full-size
golden generator (``tests/golden/make_full_golden.py``, which runs the
reference), the ``-m "gpu and slow"`` parity tests and bench.py's ``parity``
field.  Inputs are regenerated from seeds; see make_full_golden.py for what a
``full_<name>.npz`` fixture holds."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"

FULL = {
    # name: BASELINE config, algorithm and parameters (BASELINE.json configs[1..4])
    "dc2": dict(algo="divide", n=1_000_000, p=100, h=10, l=1000, c=20, r=10, data="gaussian",
                dtype="f64"),
    "fast3": dict(algo="fast", n=1_000_000, p=100, h=10, l=1000, s=20, r=10, data="gaussian",
                  dtype="f64"),
    "interp4": dict(algo="interpolate", n=10_000_000, p=100, h=10, l=2000, r=10, data="gaussian",
                    dtype="f32"),
    "img5interp": dict(algo="interpolate", n=814_255, p=784, l=1000, r=10, data="image",
                       dtype="f32"),
    "img5dc": dict(algo="divide", n=814_255, p=784, l=1000, c=20, r=10, data="image", dtype="f32"),
    "img5fast": dict(algo="fast", n=814_255, p=784, l=1000, s=20, r=10, data="image", dtype="f32"),
    # the two piece-pipeline routes once more on another draw: data seed 7, plan seed 7
    "dc2_s7": dict(algo="divide", n=1_000_000, p=100, h=10, l=1000, c=20, r=10, data="gaussian",
                   dtype="f64", seed=7),
    "fast3_s7": dict(algo="fast", n=1_000_000, p=100, h=10, l=1000, s=20, r=10, data="gaussian",
                     dtype="f64", seed=7),
}

N_SAMPLE = 4096
N_SKETCH = 4


def full_input(cfg: dict) -> np.ndarray:
    """The configuration's input from its seed (0 unless it names one): reference scenario stream
    (simulation.py:68-80; config 4 cast to float32 as BASELINE states) or the
    config-5 image-like stand-in."""
    from paper_2007_11919_b200.synthetic import image_like, scenario
    if cfg["data"] == "image":
        return image_like(cfg["n"], seed=cfg.get("seed", 0))
    x = scenario(cfg["n"], cfg["p"], cfg["h"], seed=cfg.get("seed", 0))
    return x.astype(np.float32) if cfg["dtype"] == "f32" else x


def sample_rows(n: int) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64(20071191))
    return np.sort(g.choice(n, size=min(N_SAMPLE, n), replace=False))


def full_sketch_weights(n: int) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64(11919))
    return g.random((n, N_SKETCH)) - 0.5


def load_golden(name: str) -> dict | None:
    path = GOLDEN / f"full_{name}.npz"
    if not path.exists():
        return None
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def compare(name: str, points: np.ndarray, estimates, g1: float, g2: float,
            gold: dict | None = None) -> dict:
    """Parity of a full-size result against the reference fixture:
    per-column sign from the sampled rows, then relative Frobenius errors of
    the sampled rows and of the all-row sketch, relative errors of the column
    sums of squares and of the eigenvalue estimates, absolute G1/G2 errors."""
    gold = gold if gold is not None else load_golden(name)
    if gold is None:
        return {"fixture": None}
    P = np.asarray(points, dtype=np.float64)
    rows = gold["sample_rows"]
    got_rows = P[rows]
    ref_rows = gold["sample_points"]
    s = np.sign(np.sum(got_rows * ref_rows, axis=0))
    s[s == 0] = 1.0
    rel = lambda a, b: float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))  # noqa: E731
    sketch = full_sketch_weights(P.shape[0]).T @ P
    est = np.asarray(estimates, dtype=np.float64)
    return {
        "fixture": f"tests/golden/full_{name}.npz",
        "points_rel_err": rel(got_rows * s, ref_rows),
        "sketch_rel_err": rel(sketch * s, gold["sketch"]),
        "col_sumsq_rel_err": rel(np.sum(P * P, axis=0), gold["col_sumsq"]),
        "estimates_rel_err": rel(est, gold["estimates"]),
        "g1_abs_err": abs(float(g1) - float(gold["g1"])),
        "g2_abs_err": abs(float(g2) - float(gold["g2"])),
        "signs_flipped": int(np.sum(s < 0)),
    }
