import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent)); sys.path.insert(0, "tests")
import numpy as np
import paper_2007_11919_b200 as mds
from oracle import mds_oracle as orc
from conftest import sign_fixed_rel_err
from paper_2007_11919_b200.synthetic import scenario
for (p, h, r) in [(150, 16, 13), (150, 16, 16), (150, 8, 14), (784, 0, 16)]:
    if h:
        x = scenario(2600, p, h, seed=3)
    else:
        from paper_2007_11919_b200.synthetic import image_like
        x = image_like(2600, seed=3)
    try:
        cfg = mds.divide_and_conquer_mds(x, mds.AlgorithmParams(r=r, l=1000, c=2 * r, seed=1))
        ref = orc.run("divide", x, r, l=1000, c=2 * r, seed=1, threads=1)
        print(p, h, r, "err", sign_fixed_rel_err(cfg.points, ref.points), np.max(np.abs(cfg.eigenvalue_estimates / ref.estimates - 1)))
    except Exception as e:
        print(p, h, r, "ERR", type(e).__name__, str(e)[:90])
