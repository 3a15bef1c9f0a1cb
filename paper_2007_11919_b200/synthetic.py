"""Seeded synthetic inputs for the five BASELINE configurations.

Configs 1-4 use the reference scenario generator (``simulation.py:68-80``):
Box-Muller normals over ``PCG64(SeedSequence(seed, spawn_key=(rep,)))`` with
the first ``h`` columns scaled by sqrt(15).  ``scenario`` reproduces it bit
for bit (pinned in ``tests/test_oracle.py`` against the reference's own
output).

Config 5 has no generator in the reference (the EMNIST files are absent), so
``image_like`` is this build's own stand-in with the BASELINE description:
28x28 = 784 features in [0, 1] stored as float32, ~80% exact zeros per row;
row block k (65 536 rows) is drawn from PCG64 sub-stream (seed, 5, 1, k);
each row belongs to one of 47 seeded class prototypes, whose central blob
(an ellipse, jittered by up to one pixel per row) is the row's support; on
the support the value is 0.5*Beta(2,2) + 0.5*template_c(pixel) + N(0, 0.05),
clipped to [0, 1]; off the support it is exactly 0.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SIDE = 28
N_CLASSES = 47


def _gen(seed: int, *path: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence(entropy=seed, spawn_key=tuple(path))))


def normal_matrix(g: np.random.Generator, rows: int, cols: int, threads: int | None = None,
                  chunk: int = 1 << 22) -> np.ndarray:
    """Box-Muller normals from the generator's uniform doubles (rng.py:26-41):
    radius sqrt(-2 log1p(-u1)), angle 2 pi u2, cosines then sines.

    Bit-identical to the reference's serial draw, computed over `threads`
    host threads: the uniform stream u1 is the first `half` doubles of the
    PCG64 stream and u2 the next `half`, so a chunk [a, b) of both is drawn
    from copies of the bit generator advanced by a and half + a
    (``PCG64.advance``) and transformed independently (numpy ufuncs release
    the GIL).  Consumes the generator exactly like the serial version."""
    total = rows * cols
    half = (total + 1) // 2
    threads = threads or min(16, os.cpu_count() or 1)
    if half <= chunk or threads == 1:
        u = g.random(half)
        v = g.random(half)
        rad = np.sqrt(-2.0 * np.log1p(-u))
        ang = (2.0 * np.pi) * v
        return np.concatenate([rad * np.cos(ang), rad * np.sin(ang)])[:total].reshape(rows, cols)
    state = g.bit_generator.state
    out = np.empty(total)

    def work(a: int) -> None:
        b = min(half, a + chunk)
        streams = []
        for off in (a, half + a):
            bg = np.random.PCG64()
            bg.state = state
            bg.advance(off)
            streams.append(np.random.Generator(bg).random(b - a))
        u, v = streams
        rad = np.sqrt(-2.0 * np.log1p(-u))
        ang = (2.0 * np.pi) * v
        out[a:b] = rad * np.cos(ang)
        e = min(total, half + b)
        if e > half + a:
            out[half + a:e] = (rad * np.sin(ang))[:e - half - a]

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(0, half, chunk)))
    g.bit_generator.advance(2 * half)          # leave g where the serial draw would
    return out.reshape(rows, cols)


def scenario(n: int, p: int, h: int, seed: int = 0, rep: int = 0,
             threads: int | None = None) -> np.ndarray:
    """N(0, diag(15 x h, 1 x (p-h))) rows, float64, reference stream
    (simulation.py:68-80), bit-identical for any `threads`."""
    out = normal_matrix(_gen(seed, rep), n, p, threads)
    out[:, :h] *= np.sqrt(15.0)
    return out


def _prototypes(seed: int):
    g = _gen(seed, 5, 0)
    yy, xx = np.mgrid[0:SIDE, 0:SIDE].astype(np.float64)
    masks = np.zeros((N_CLASSES, SIDE, SIDE), dtype=bool)
    templates = np.zeros((N_CLASSES, SIDE, SIDE))
    for c in range(N_CLASSES):
        cy, cx = g.uniform(11.5, 16.5, size=2)
        ry, rx = g.uniform(6.0, 11.0), g.uniform(4.5, 7.0)
        th = g.uniform(0.0, np.pi)
        dy, dx = yy - cy, xx - cx
        u = (dy * np.cos(th) + dx * np.sin(th)) / ry
        w = (-dy * np.sin(th) + dx * np.cos(th)) / rx
        rr = u * u + w * w
        masks[c] = rr <= 1.0
        # smooth per-class intensity pattern inside the blob
        f1, f2 = g.uniform(0.15, 0.6, size=2)
        ph1, ph2 = g.uniform(0.0, 2 * np.pi, size=2)
        templates[c] = 0.5 + 0.5 * np.sin(f1 * yy + ph1) * np.cos(f2 * xx + ph2)
    return masks, templates


def _image_chunk(masks, templates, seed: int, k: int, m: int) -> np.ndarray:
    g = _gen(seed, 5, 1, k)
    cls = g.integers(0, N_CLASSES, size=m)
    sh = g.integers(-1, 2, size=(m, 2))
    # support = the class blob rolled by (dy, dx) per row (np.roll as a gather)
    yy = (np.arange(SIDE)[None, :, None] - sh[:, 0, None, None]) % SIDE
    xx = (np.arange(SIDE)[None, None, :] - sh[:, 1, None, None]) % SIDE
    sup = masks[cls][np.arange(m)[:, None, None], yy, xx]
    vals = 0.5 * g.beta(2.0, 2.0, size=(m, SIDE, SIDE)) + 0.5 * templates[cls] \
        + g.normal(0.0, 0.05, size=(m, SIDE, SIDE))
    vals = np.clip(vals, 0.0, 1.0) * sup
    return vals.reshape(m, -1).astype(np.float32)


def image_like(n: int, seed: int = 0, chunk: int = 65536, threads: int | None = None) -> np.ndarray:
    """Config-5 stand-in: n x 784 float32 in [0, 1], ~80% exact zeros.  Row
    block k (of `chunk` rows) is drawn from its own PCG64 sub-stream
    (seed, 5, 1, k), so blocks are generated in parallel and the result does
    not depend on `threads`."""
    masks, templates = _prototypes(seed)
    out = np.empty((n, SIDE * SIDE), dtype=np.float32)
    threads = threads or min(16, os.cpu_count() or 1)

    def work(k: int) -> None:
        a = k * chunk
        m = min(chunk, n - a)
        out[a:a + m] = _image_chunk(masks, templates, seed, k, m)

    nchunks = (n + chunk - 1) // chunk
    with ThreadPoolExecutor(max(1, min(threads, nchunks))) as ex:
        list(ex.map(work, range(nchunks)))
    return out
