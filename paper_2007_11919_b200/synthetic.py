"""Seeded synthetic inputs for the five BASELINE configurations.

Configs 1-4 use the reference scenario generator (``simulation.py:68-80``):
Box-Muller normals over ``PCG64(SeedSequence(seed, spawn_key=(rep,)))`` with
the first ``h`` columns scaled by sqrt(15).  ``scenario`` reproduces it bit
for bit (pinned in ``tests/test_oracle.py`` against the reference's own
output).

Config 5 has no generator in the reference (the EMNIST files are absent), so
``image_like`` is this build's own stand-in with the BASELINE description:
28x28 = 784 features in [0, 1] stored as float32, ~80% exact zeros per row;
each row belongs to one of 47 seeded class prototypes, whose central blob
(an ellipse, jittered by up to one pixel per row) is the row's support; on
the support the value is 0.5*Beta(2,2) + 0.5*template_c(pixel) + N(0, 0.05),
clipped to [0, 1]; off the support it is exactly 0.
"""

from __future__ import annotations

import numpy as np

SIDE = 28
N_CLASSES = 47


def _gen(seed: int, *path: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence(entropy=seed, spawn_key=tuple(path))))


def normal_matrix(g: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    """Box-Muller normals from the generator's uniform doubles (rng.py:26-41):
    radius sqrt(-2 log1p(-u1)), angle 2 pi u2, cosines then sines."""
    total = rows * cols
    half = (total + 1) // 2
    u = g.random(half)
    v = g.random(half)
    rad = np.sqrt(-2.0 * np.log1p(-u))
    ang = (2.0 * np.pi) * v
    return np.concatenate([rad * np.cos(ang), rad * np.sin(ang)])[:total].reshape(rows, cols)


def scenario(n: int, p: int, h: int, seed: int = 0, rep: int = 0) -> np.ndarray:
    """N(0, diag(15 x h, 1 x (p-h))) rows, float64, reference stream."""
    out = normal_matrix(_gen(seed, rep), n, p)
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


def image_like(n: int, seed: int = 0, chunk: int = 65536) -> np.ndarray:
    """Config-5 stand-in: n x 784 float32 in [0, 1], ~80% exact zeros."""
    masks, templates = _prototypes(seed)
    g = _gen(seed, 5, 1)
    out = np.zeros((n, SIDE * SIDE), dtype=np.float32)
    for start in range(0, n, chunk):
        m = min(chunk, n - start)
        cls = g.integers(0, N_CLASSES, size=m)
        sh = g.integers(-1, 2, size=(m, 2))
        sup = masks[cls]
        sup = np.stack([np.roll(sup[i], (sh[i, 0], sh[i, 1]), axis=(0, 1)) for i in range(m)])
        tpl = templates[cls]
        vals = 0.5 * g.beta(2.0, 2.0, size=(m, SIDE, SIDE)) + 0.5 * tpl \
            + g.normal(0.0, 0.05, size=(m, SIDE, SIDE))
        vals = np.clip(vals, 0.0, 1.0) * sup
        out[start:start + m] = vals.reshape(m, -1).astype(np.float32)
    return out


def image_like_device(n: int, seed: int = 0, device="cuda", chunk: int = 131072):
    """Same distribution as `image_like` (same 47 prototypes), drawn on the GPU
    with torch's generator — for benchmark-scale inputs only (parity tests use
    the numpy stream above)."""
    import torch

    masks_np, templates_np = _prototypes(seed)
    masks = torch.from_numpy(masks_np).to(device)
    templates = torch.from_numpy(templates_np).to(device=device, dtype=torch.float32)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    beta = torch.distributions.Beta(torch.tensor(2.0, device=device), torch.tensor(2.0, device=device))
    out = torch.empty((n, SIDE * SIDE), dtype=torch.float32, device=device)
    for start in range(0, n, chunk):
        m = min(chunk, n - start)
        cls = torch.randint(0, N_CLASSES, (m,), generator=g, device=device)
        sh = torch.randint(-1, 2, (m, 2), generator=g, device=device)
        sup = masks[cls]
        yy = (torch.arange(SIDE, device=device)[None, :, None] - sh[:, 0, None, None]) % SIDE
        xx = (torch.arange(SIDE, device=device)[None, None, :] - sh[:, 1, None, None]) % SIDE
        sup = sup[torch.arange(m, device=device)[:, None, None], yy, xx]
        torch.manual_seed(seed * 1000003 + start)      # Beta sampler uses the global stream
        vals = 0.5 * beta.sample((m, SIDE, SIDE)) + 0.5 * templates[cls] \
            + 0.05 * torch.randn((m, SIDE, SIDE), generator=g, device=device)
        out[start:start + m] = (vals.clamp_(0.0, 1.0) * sup).reshape(m, -1)
    return out
