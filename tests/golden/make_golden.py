"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (it imports ``scalemds`` from
/root/reference/pkg/src, which does not exist on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Inputs are regenerated at test time from seeds (configs 1-4: the reference
scenario generator; config 5: ``synthetic.image_like``), so only outputs,
plan digests and a few small inputs are stored.
"""

from __future__ import annotations

import hashlib
import importlib.util
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
import scalemds as ref  # noqa: E402

_spec = importlib.util.spec_from_file_location(
    "synthetic", REPO / "paper_2007_11919_b200" / "synthetic.py")
synthetic = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(synthetic)


def digest(arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
        h.update(np.int64(a.size).tobytes())
        h.update(a.tobytes())
    return h.hexdigest()


def fast_leaves_digest(plan) -> str:
    leaves = plan.leaves()
    return digest([leaf.indices for leaf in leaves])


def fast_positions_digest(plan) -> str:
    out = []
    stack = [plan.root]
    while stack:
        node = stack.pop()
        if node.sampling_positions is not None:
            out.append(node.sampling_positions)
        stack.extend(reversed(node.children))
    return digest(out)


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", **arrays)
    print("wrote", name, {k: np.asarray(v).shape for k, v in arrays.items()})


def cfg_arrays(cfg):
    return dict(points=cfg.points, estimates=cfg.eigenvalue_estimates,
                g1=np.float64(cfg.gof_g1), g2=np.float64(cfg.gof_g2))


def main():
    assert os.environ.get("OPENBLAS_NUM_THREADS") == "1", "pin OPENBLAS_NUM_THREADS=1"

    # ---- function-level seams (small, inputs stored) ----
    rng = np.random.default_rng(0)
    d40 = rng.standard_normal((40, 6))
    a43 = rng.standard_normal((4, 3))
    b63 = rng.standard_normal((6, 3))
    x60 = rng.standard_normal((60, 4)) * np.array([4.0, 2.0, 1.0, 0.5])
    c = ref.classical_mds_from_data(x60, 3)
    # non-Euclidean delta: perturbed symmetric with zero diagonal
    pert = ref.euclidean_distance_matrix(rng.standard_normal((30, 3)))
    noise = rng.uniform(0.0, 0.5, size=(30, 30))
    noise = noise + noise.T
    np.fill_diagonal(noise, 0.0)
    ne = pert + noise
    cne = ref.classical_mds(ne, 2)
    pt = rng.standard_normal((20, 10))
    ps = rng.standard_normal((20, 10))
    pf = ref.fit_procrustes(pt, ps)
    base = np.random.default_rng(21).standard_normal((200, 10)) * 2.0
    bcfg = ref.classical_mds_from_data(base, 5)
    ctx = ref.gower_context(base, bcfg.points)
    newrows = rng.standard_normal((50, 10)) * 2.0
    save("fn_small",
         d40=d40, dist_self=ref.euclidean_distance_matrix(d40),
         a43=a43, b63=b63, dist_cross=ref.cross_squared_distances(a43, b63),
         dcenter=ref.double_center(ref.euclidean_distance_matrix(d40)),
         x60=x60, c_points=c.points, c_est=c.eigenvalue_estimates,
         c_g=np.array([c.gof_g1, c.gof_g2]),
         ne=ne, ne_points=cne.points, ne_est=cne.eigenvalue_estimates,
         ne_g=np.array([cne.gof_g1, cne.gof_g2]),
         pt=pt, ps=ps, pf_rot=pf.rotation, pf_t=pf.translation, pf_loss=np.float64(pf.loss),
         base=base, base_points=bcfg.points, ctx_q=ctx.q_diag, ctx_cov=ctx.covariance,
         newrows=newrows, gower=ref.gower_interpolate(ctx, newrows))

    # ---- config 1 at full size ----
    x = ref.generate_scenario(ref.ScenarioSpec(n=10_000, k=10, h=2, seed=0), 0)
    plan = ref.plan_interpolation(10_000, 500, 0)
    cfg = ref.run_algorithm("interpolate", x, ref.AlgorithmParams(r=2, l=500, seed=0))
    save("cfg1_interp", sample=plan.subsets[0], plan_digest=np.array(digest(plan.subsets)),
         x_head=x[:5], **cfg_arrays(cfg))

    # ---- scaled-down configs 2 / 3 (same p, l, c, s, r) ----
    x = ref.generate_scenario(ref.ScenarioSpec(n=5000, k=100, h=10, seed=0), 0)
    cfg = ref.run_algorithm("divide", x, ref.AlgorithmParams(r=10, l=1000, c=20, seed=0))
    save("dc_n5000", **cfg_arrays(cfg))
    cfg = ref.run_algorithm("fast", x, ref.AlgorithmParams(r=10, l=1000, s=20, seed=0))
    save("fast_n5000", **cfg_arrays(cfg))
    # depth-2 recursion
    xd = ref.generate_scenario(ref.ScenarioSpec(n=3000, k=10, h=5, seed=4), 0)
    cfg = ref.run_algorithm("fast", xd, ref.AlgorithmParams(r=5, l=100, s=10, seed=4))
    save("fast_deep", **cfg_arrays(cfg))

    # ---- scaled-down config 4 (fp32 storage) ----
    x = ref.generate_scenario(ref.ScenarioSpec(n=8000, k=100, h=10, seed=0), 0).astype(np.float32)
    cfg = ref.run_algorithm("interpolate", x, ref.AlgorithmParams(r=10, l=2000, seed=0))
    save("interp_f32_n8000", **cfg_arrays(cfg))

    # ---- scaled-down config 5 (image-like stand-in) ----
    xi = synthetic.image_like(3000, seed=0)
    for name, prm in (("divide", ref.AlgorithmParams(r=10, l=1000, c=20, seed=0)),
                      ("fast", ref.AlgorithmParams(r=10, l=1000, s=20, seed=0)),
                      ("interpolate", ref.AlgorithmParams(r=10, l=1000, seed=0))):
        cfg = ref.run_algorithm(name, xi, prm)
        save(f"img_{name}_n3000", **cfg_arrays(cfg))

    # ---- full-size plan digests (bit-exact planner pin) ----
    dc = ref.plan_divide_conquer(1_000_000, 1000, 20, 0)
    fp = ref.plan_fast(1_000_000, 1000, 20, 0)
    ip = ref.plan_interpolation(10_000_000, 2000, 0)
    dc5 = ref.plan_divide_conquer(814_255, 1000, 20, 0)
    fp5 = ref.plan_fast(814_255, 1000, 20, 0)
    ip5 = ref.plan_interpolation(814_255, 1000, 0)
    save("plan_digests",
         dc_1e6=np.array(digest(dc.subsets)), dc_1e6_p=np.int64(dc.p),
         fast_1e6_leaves=np.array(fast_leaves_digest(fp)),
         fast_1e6_positions=np.array(fast_positions_digest(fp)),
         fast_1e6_root=np.array(digest([fp.root.indices])),
         interp_1e7=np.array(digest(ip.subsets)), interp_1e7_p=np.int64(ip.p),
         dc_cfg5=np.array(digest(dc5.subsets)),
         fast_cfg5_leaves=np.array(fast_leaves_digest(fp5)),
         fast_cfg5_positions=np.array(fast_positions_digest(fp5)),
         interp_cfg5=np.array(digest(ip5.subsets)))


if __name__ == "__main__":
    main()
