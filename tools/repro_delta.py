import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2007_11919_b200 as mds
from paper_2007_11919_b200 import _device as D
from oracle import mds_oracle as orc
from paper_2007_11919_b200.synthetic import scenario
x = scenario(300, 12, 4, seed=21)
for p_ in (12, 60, 150):
    x = scenario(300, p_, 4, seed=21)
    delta = orc.sqdist_self(x)
    dev = torch.device("cuda", 0)
    d = torch.from_numpy(delta).to(dev)
    n, r = 300, 4
    pts = D.empty((n, r), dev); est = D.empty((1, r), dev); gof = D.empty((1, 2), dev); st = D.status_tensor(1, dev)
    D.handle(dev).call("mdsx_classical_delta", d.data_ptr(), n, r, pts.data_ptr(), est.data_ptr(),
                       gof.data_ptr(), st.data_ptr(), D.stream_ptr(dev))
    print(p_, D.decode_status(st), est.cpu().numpy(), orc.mds_from_delta(delta, 4).estimates)
rng = np.random.default_rng(5)
for rank in (20, 60, 130):
    x = rng.standard_normal((3000, rank)) @ rng.standard_normal((rank, 150))
    try:
        cfg = mds.divide_and_conquer_mds(x, mds.AlgorithmParams(r=10, l=1000, c=20, seed=1))
        ref = orc.run("divide", x, 10, l=1000, c=20, seed=1, threads=1)
        sys.path.insert(0, "tests"); from conftest import sign_fixed_rel_err
        print("dc rank", rank, "ok err", sign_fixed_rel_err(cfg.points, ref.points))
    except Exception as e:
        print("dc rank", rank, "ERR", type(e).__name__, str(e)[:80])
