"""Full-size (BASELINE n) golden fixtures, produced by running the REFERENCE.

Run in the build container only (imports ``scalemds`` from
/root/reference/pkg/src, absent on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_full_golden.py [cfg ...]

For each BASELINE configuration 2-5 the reference's own ``run_algorithm``
runs on the input regenerated from its seed (configs 2-4: the reference
scenario stream, config 4 cast to float32 exactly as BASELINE states;
config 5: ``synthetic.image_like``).  A full n x r result is too large to
commit, so each fixture keeps what a parity test needs to check every row:

* ``sample_rows`` / ``sample_points``: the configuration at 4096 seeded rows;
* ``sketch``: W^T P for a seeded n x 4 matrix W of uniforms in [-1/2, 1/2)
  (regenerated at test time by ``full_sketch_weights``) -- a checksum that
  touches every row; per-column signs flip it column-wise;
* ``col_sumsq``: sum_i P_ik^2 (sign invariant);
* ``g1``, ``g2``, ``estimates``;
* ``input_colsum``: column sums of the input (detects a generator mismatch);
* ``ref_seconds``, ``ref_threads``: wall time of the reference call here
  (8-core Xeon, pool of 8, OpenBLAS 1 thread).
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")
import scalemds as ref  # noqa: E402

sys.path.insert(0, str(HERE.parent))
from full_configs import FULL, full_input, full_sketch_weights, sample_rows  # noqa: E402


def main(names):
    threads = os.cpu_count() or 1
    for name in names:
        cfg = FULL[name]
        t0 = time.perf_counter()
        x = full_input(cfg)
        t_gen = time.perf_counter() - t0
        prm = ref.AlgorithmParams(r=cfg["r"], l=cfg["l"], c=cfg.get("c"), s=cfg.get("s"),
                                  seed=cfg.get("seed", 0))
        t0 = time.perf_counter()
        res = ref.run_algorithm(cfg["algo"], x, prm, threads=threads)
        dt = time.perf_counter() - t0
        P = np.asarray(res.points)
        n = P.shape[0]
        rows = sample_rows(n)
        W = full_sketch_weights(n)
        np.savez_compressed(
            HERE / f"full_{name}.npz",
            sample_rows=rows, sample_points=P[rows], sketch=W.T @ P,
            col_sumsq=np.sum(P * P, axis=0), g1=res.gof_g1, g2=res.gof_g2,
            estimates=np.asarray(res.eigenvalue_estimates),
            input_colsum=np.asarray(x, dtype=np.float64).sum(axis=0),
            ref_seconds=dt, ref_threads=threads)
        print(f"{name}: gen {t_gen:.1f}s reference {dt:.1f}s g1={res.gof_g1:.6f} "
              f"est={np.round(res.eigenvalue_estimates, 4)}", flush=True)
        del x, res, P, W


if __name__ == "__main__":
    main(sys.argv[1:] or list(FULL))
