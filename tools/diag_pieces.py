"""Diagnostics: per-piece solver iterations and kernel times for a batch of
config-2-like pieces (run on a GPU box)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2007_11919_b200 as mds
from paper_2007_11919_b200 import _device as D
from paper_2007_11919_b200.primitives import classical_pieces
from paper_2007_11919_b200.synthetic import scenario

dev = torch.device("cuda", 0)
n, p, m = int(sys.argv[1]) if len(sys.argv) > 1 else 20000, 100, 1000
x = torch.from_numpy(scenario(n, p, 10, seed=0)).to(dev)
npc = n // m
idx = torch.arange(npc * m, dtype=torch.int64, device=dev)
off = np.arange(0, npc * m + 1, m, dtype=np.int64)
h = D.handle(dev)
for rep in range(3):
    h.timing(True)
    pts, est, gof, st = classical_pieces(x, idx, off, 10)
    torch.cuda.synchronize()
    h.timing(False)
    rep_t = h.timing_report()
stat = D.decode_status(st)
print("codes", np.unique(stat["code"], return_counts=True))
print("iterations (value)", np.unique(stat["value"], return_counts=True))
for k_, (ms, c) in sorted(rep_t.items()):
    print(f"{k_:28s} {ms:8.3f} ms  x{c}")

import ctypes
from paper_2007_11919_b200 import _lib
lib = _lib.load()




