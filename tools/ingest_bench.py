"""Ingestion throughput on the GPU box:
EMNIST-sized IDX file (814 255 x 28 x 28 u8) -> device matrix, native streamed
loader vs the reference-style host path (read + astype(float64) + H2D); and the
native CSV parser vs Python's csv module on a 200 000 x 20 matrix."""
import csv
import os
import struct
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2007_11919_b200 as m

tmp = Path(tempfile.mkdtemp(dir="/tmp"))
n, h, w = 814_255, 28, 28
pix = np.random.default_rng(0).integers(0, 256, (n, h * w), dtype=np.uint8)
p = tmp / "emnist-like-images-idx3-ubyte"
p.write_bytes(struct.pack(">IIII", 0x803, n, h, w) + pix.tobytes())
del pix
dev = torch.device("cuda", 0)
for dt in (torch.float64, torch.float32):
    m.load_idx_images(p, dtype=dt)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = m.load_idx_images(p, dtype=dt)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"native idx -> device {dt}: {t1 - t0:.3f} s ({x.numel() / (t1 - t0) / 1e9:.2f} Gelem/s)")
    del x
t0 = time.perf_counter()
host = np.fromfile(p, dtype=np.uint8, offset=16).reshape(n, h * w).astype(np.float64)
xd = torch.from_numpy(host).to(dev)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"reference-style read + astype(float64) + H2D: {t1 - t0:.3f} s")
del host, xd

rows, cols = 200_000, 20
mat = np.random.default_rng(1).standard_normal((rows, cols))
c = tmp / "m.csv"
m.write_csv_matrix(mat, c)
t0 = time.perf_counter()
got = m.read_csv_matrix(c)
t1 = time.perf_counter()
assert np.array_equal(got, mat)
print(f"native csv {rows}x{cols}: {t1 - t0:.3f} s ({os.cpu_count()} threads)")
t0 = time.perf_counter()
with open(c, newline="") as fh:
    ref = np.asarray([[float(v) for v in rec] for rec in csv.reader(fh)])
t1 = time.perf_counter()
assert np.array_equal(ref, mat)
print(f"python csv module (the reference's parser): {t1 - t0:.3f} s")
