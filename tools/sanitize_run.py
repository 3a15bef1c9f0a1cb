"""Small invocations of every device route for compute-sanitizer
(memcheck / racecheck / synccheck on small configs):

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py

D&C (fused output route and the point-matrix route), fast MDS (one-call route
and the piece route), interpolation (bulk Gower kernel), classical MDS of a
distance matrix beyond the Jacobi size (block Krylov + device eigenvalues),
Procrustes, the staged H2D copy."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2007_11919_b200 as mds  # noqa: E402
from paper_2007_11919_b200.synthetic import image_like, scenario  # noqa: E402


def main():
    x = scenario(5000, 100, 10, seed=1)
    xs = scenario(3000, 20, 4, seed=2)
    runs = [
        ("divide", x, mds.AlgorithmParams(r=10, l=1000, c=20, seed=0)),
        ("fast", x, mds.AlgorithmParams(r=10, l=1000, s=20, seed=0)),
        ("interpolate", x.astype(np.float32), mds.AlgorithmParams(r=10, l=800, seed=0)),
        ("divide", xs, mds.AlgorithmParams(r=4, l=300, c=10, seed=0)),
        ("fast", xs, mds.AlgorithmParams(r=4, l=300, s=10, seed=0)),
        ("divide", image_like(2500, seed=0), mds.AlgorithmParams(r=10, l=1000, c=20, seed=0)),
    ]
    for name, data, prm in runs:
        cfg = mds.run_algorithm(name, data, prm)
        print(name, data.shape, data.dtype, "g1", round(cfg.gof_g1, 6), flush=True)
    os.environ["MDSX_DC_POINTS"] = "1"
    os.environ["MDSX_FAST_PIECES"] = "1"
    for name, data, prm in runs[:2]:
        cfg = mds.run_algorithm(name, data, prm)
        print(name, "(point-matrix route) g1", round(cfg.gof_g1, 6), flush=True)
    del os.environ["MDSX_DC_POINTS"], os.environ["MDSX_FAST_PIECES"]
    d = mds.euclidean_distance_matrix(scenario(300, 12, 4, seed=3))
    cfg = mds.classical_mds(d + 0.05 * (1 - np.eye(300)), 4)
    print("classical delta n=300 g1", round(cfg.gof_g1, 6), flush=True)
    tr = mds.fit_procrustes(xs[:50, :4], xs[50:100, :4])
    print("procrustes loss", round(tr.loss, 6), flush=True)


if __name__ == "__main__":
    main()
