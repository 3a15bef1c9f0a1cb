"""Host-side partition planner (drop-in for ``partition.py`` and ``rng.py``).

Plans are index arrays drawn from PCG64 streams keyed by
``SeedSequence(entropy=seed, spawn_key=path)`` (rng.py:14-17) with the same
Generator calls in the same order as the reference, so every plan is
bit-identical to the reference's (pinned against digests of the reference's
own plans in tests/test_plans.py).  The GPU path consumes plans in flattened
form (``flatten_*``): one int64 row-index array plus host offsets.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import weakref

import numpy as np

from .errors import ParamError


def spawned_generator(seed: int, *path: int) -> np.random.Generator:
    """rng.py:14-17."""
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence(entropy=seed, spawn_key=tuple(path))))


def sub_seed(seed: int, *path: int) -> int:
    """rng.py:20-23."""
    return int(np.random.SeedSequence(entropy=seed, spawn_key=tuple(path))
               .generate_state(1, np.uint64)[0])


_M64 = (1 << 64) - 1


def _permutation(g: np.random.Generator, arr: np.ndarray) -> np.ndarray:
    """== g.permutation(arr) for a 1-d int64 array, bit for bit, advancing g
    identically: the same PCG64 draws (numpy's masked-rejection interval on
    buffered 32-bit outputs), with the swaps done by libmdsx's native
    planner (mdsx_plan_permute: targets drawn first, swap targets
    prefetched).  numpy itself is used when the library is not built."""
    out = np.array(arr, dtype=np.int64, copy=True)
    bg = g.bit_generator
    if out.size < 4096 or type(bg) is not np.random.PCG64:
        return g.permutation(arr)
    try:
        from . import _lib
        lib = _lib.load()
    except (RuntimeError, OSError):
        return g.permutation(arr)
    import ctypes as C
    st = bg.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    state = np.array([s >> 64, s & _M64, inc >> 64, inc & _M64], dtype=np.uint64)
    has = C.c_int32(int(st["has_uint32"]))
    u32 = C.c_uint32(int(st["uinteger"]))
    rc = lib.mdsx_plan_permute(out.ctypes.data, out.size, state.ctypes.data, C.byref(has),
                               C.byref(u32))
    if rc != 0:
        return g.permutation(arr)
    st["state"]["state"] = (int(state[0]) << 64) | int(state[1])
    st["has_uint32"] = has.value
    st["uinteger"] = u32.value
    bg.state = st
    return out


def _choices_sorted(g: np.random.Generator, pops, s: int) -> list:
    """[np.sort(g.choice(pop, size=min(s, pop), replace=False)) for pop in pops],
    bit for bit and advancing g identically, in ONE native call
    (mdsx_plan_choices: numpy's Floyd / tail-shuffle methods on the same
    32-bit Lemire draws); numpy itself when the library is not built or a
    population needs another of numpy's paths."""
    pops = np.ascontiguousarray(pops, dtype=np.int64)
    bg = g.bit_generator
    lib = None
    if type(bg) is np.random.PCG64 and pops.size:
        try:
            from . import _lib
            lib = _lib.load()
        except (RuntimeError, OSError):
            lib = None
    if lib is not None:
        import ctypes as C
        st = bg.state
        st_s, inc = st["state"]["state"], st["state"]["inc"]
        state = np.array([st_s >> 64, st_s & _M64, inc >> 64, inc & _M64], dtype=np.uint64)
        has = C.c_int32(int(st["has_uint32"]))
        u32 = C.c_uint32(int(st["uinteger"]))
        out = np.empty(pops.size * s, dtype=np.int64)
        rc = lib.mdsx_plan_choices(pops.ctypes.data, pops.size, s, out.ctypes.data, state.ctypes.data,
                                   C.byref(has), C.byref(u32))
        if rc == 0:
            st["state"]["state"] = (int(state[0]) << 64) | int(state[1])
            st["has_uint32"] = has.value
            st["uinteger"] = u32.value
            bg.state = st
            return [np.sort(out[i * s:i * s + min(s, int(q))]) for i, q in enumerate(pops)]
    return [np.sort(g.choice(int(q), size=min(s, int(q)), replace=False)) for q in pops]


def _complement_sorted(n: int, taken: np.ndarray) -> np.ndarray:
    """== np.setdiff1d(np.arange(n), taken) for unique in-range ``taken``
    (a mask instead of a sort: O(n))."""
    keep = np.ones(n, dtype=bool)
    keep[taken] = False
    return np.flatnonzero(keep).astype(np.int64)


# ------------------------------------------------------------------ plan types
@dataclass(frozen=True)
class DcPlan:
    """partition.py:20-59 — every subset = connecting rows (ascending) then
    the subset's own rows (ascending); a single 0..n-1 subset when n <= l."""

    connecting_indices: np.ndarray
    subsets: list
    n: int
    l: int
    c: int
    seed: int

    @property
    def p(self) -> int:
        return len(self.subsets)

    def own_indices(self, j: int) -> np.ndarray:
        return self.subsets[0] if self.p == 1 else self.subsets[j][len(self.connecting_indices):]

    def to_dict(self) -> dict:
        return {"algorithm": "divide", "n": self.n, "l": self.l, "c": self.c, "seed": self.seed,
                "connecting_indices": self.connecting_indices.tolist(),
                "subsets": [q.tolist() for q in self.subsets]}

    def to_json(self) -> str:
        return json.dumps(self.to_dict())


@dataclass(frozen=True)
class InterpPlan:
    """partition.py:62-86 — sample subset first, then chunks of at most l."""

    subsets: list
    n: int
    l: int
    seed: int

    @property
    def p(self) -> int:
        return len(self.subsets)

    def to_dict(self) -> dict:
        return {"algorithm": "interpolate", "n": self.n, "l": self.l, "seed": self.seed,
                "subsets": [q.tolist() for q in self.subsets]}

    def to_json(self) -> str:
        return json.dumps(self.to_dict())


@dataclass
class FastNode:
    """partition.py:89-112 — ``indices`` in output-row order (leaves
    ascending, internal nodes = children concatenated); ``sampling_positions``
    index into ``indices`` and are assigned by the parent."""

    indices: np.ndarray
    children: list = field(default_factory=list)
    sampling_positions: np.ndarray | None = None

    @property
    def is_leaf(self) -> bool:
        return not self.children

    @property
    def size(self) -> int:
        return len(self.indices)

    def sampling_indices(self) -> np.ndarray:
        return self.indices[self.sampling_positions]


@dataclass(frozen=True)
class FastStats:
    """partition.py:115-121."""

    leaf_count: int
    mean_leaf_size: float
    depth: int


@dataclass(frozen=True)
class FastPlan:
    """partition.py:124-181."""

    root: FastNode
    n: int
    l: int
    s: int
    seed: int

    def leaves(self) -> list:
        found, todo = [], [self.root]
        while todo:
            node = todo.pop()
            if node.is_leaf:
                found.append(node)
            else:
                todo.extend(node.children[::-1])
        return found

    def stats(self) -> FastStats:
        sizes, depth, todo = [], 0, [(self.root, 0)]
        while todo:
            node, lvl = todo.pop()
            if node.is_leaf:
                sizes.append(node.size)
                depth = max(depth, lvl)
            else:
                todo.extend((ch, lvl + 1) for ch in node.children)
        return FastStats(leaf_count=len(sizes), mean_leaf_size=self.n / len(sizes), depth=depth)

    def _as_dict(self, node: FastNode) -> dict:
        d: dict = {"indices": node.indices.tolist()}
        if node.sampling_positions is not None:
            d["sampling_positions"] = node.sampling_positions.tolist()
        if node.children:
            d["children"] = [self._as_dict(ch) for ch in node.children]
        return d

    def to_dict(self) -> dict:
        return {"algorithm": "fast", "n": self.n, "l": self.l, "s": self.s, "seed": self.seed,
                "tree": self._as_dict(self.root)}

    def to_json(self) -> str:
        return json.dumps(self.to_dict())


# ------------------------------------------------------------------ planners
def plan_divide_conquer(n: int, l: int, c: int, seed: int) -> DcPlan:
    """partition.py:184-214."""
    if n < 1:
        raise ParamError(f"n must be >= 1, got {n}")
    if c < 1:
        raise ParamError(f"c must be >= 1, got {c}")
    if l <= c:
        raise ParamError(f"l must exceed c, got l={l}, c={c}")
    if n <= l:
        return DcPlan(np.empty(0, dtype=np.int64), [np.arange(n, dtype=np.int64)], n, l, c, seed)
    g = spawned_generator(seed)
    conn = np.sort(g.choice(n, size=c, replace=False)).astype(np.int64)
    dealt = _permutation(g, _complement_sorted(n, conn))
    step = l - c
    nb = (dealt.size + step - 1) // step          # chunks of `step` dealt rows, the last short
    if nb > 1 and dealt.size - (nb - 1) * step < c + 1:
        nb -= 1                                   # merge a short remainder into its predecessor
    full = nb - 1                                 # chunks of exactly `step` rows
    # [connecting | own sorted] for the full chunks in one 2-D block (row views)
    block = np.empty((full, l), dtype=np.int64)
    block[:, :c] = conn
    block[:, c:] = np.sort(dealt[:full * step].reshape(full, step), axis=1)
    last = np.concatenate([conn, np.sort(dealt[full * step:])])
    return DcPlan(conn, list(block) + [last], n, l, c, seed)


def interpolation_sample(n: int, l: int, seed: int) -> np.ndarray:
    """First draw of ``plan_interpolation``: the sorted landmark sample.  Every
    other row's Gower coordinates depend only on that row, so the GPU path
    needs nothing else from the plan."""
    if n <= l:
        return np.arange(n, dtype=np.int64)
    return np.sort(spawned_generator(seed).choice(n, size=l, replace=False)).astype(np.int64)


def plan_interpolation(n: int, l: int, seed: int) -> InterpPlan:
    """partition.py:217-232."""
    if n < 1:
        raise ParamError(f"n must be >= 1, got {n}")
    if l < 2:
        raise ParamError(f"l must be >= 2, got {l}")
    if n <= l:
        return InterpPlan([np.arange(n, dtype=np.int64)], n, l, seed)
    g = spawned_generator(seed)
    sample = np.sort(g.choice(n, size=l, replace=False)).astype(np.int64)
    dealt = _permutation(g, _complement_sorted(n, sample))
    return InterpPlan([sample] + [np.sort(dealt[a:a + l]) for a in range(0, dealt.size, l)],
                      n, l, seed)


def _check_fast(n: int, l: int, s: int) -> None:
    if n < 1:
        raise ParamError(f"n must be >= 1, got {n}")
    if s < 1:
        raise ParamError(f"s must be >= 1, got {s}")
    if l < 2 * s:
        raise ParamError(f"l must be >= 2*s so that at least two subsets form, got l={l}, s={s}")


def plan_fast(n: int, l: int, s: int, seed: int) -> FastPlan:
    """partition.py:244-274 — nodes above l rows are shuffled with the
    generator of their tree path and split into l//s near-equal parts, each
    sampled with min(s, size) positions by that same generator."""
    _check_fast(n, l, s)
    parts = l // s

    def grow(idx: np.ndarray, path: tuple) -> FastNode:
        if idx.size <= l:
            return FastNode(np.sort(idx))
        g = spawned_generator(seed, *path)
        pieces = np.array_split(_permutation(g, idx), parts)
        picks = _choices_sorted(g, [q.size for q in pieces], s)
        kids = []
        for i, (q, pos) in enumerate(zip(pieces, picks)):
            kid = grow(q, path + (i,))
            kid.sampling_positions = pos
            kids.append(kid)
        return FastNode(np.concatenate([k.indices for k in kids]), kids)

    return FastPlan(grow(np.arange(n, dtype=np.int64), ()), n, l, s, seed)


def fast_stats(n: int, l: int, s: int) -> FastStats:
    """partition.py:277-306 — leaf count / mean size / depth by arithmetic."""
    _check_fast(n, l, s)
    parts = l // s
    memo: dict = {}

    def count(size: int):
        if size <= l:
            return 1, 0
        if size not in memo:
            q, rem = divmod(size, parts)
            leaves, depth = 0, 0
            for sub, mult in ((q + 1, rem), (q, parts - rem)):
                if mult:
                    lv, dp = count(sub)
                    leaves += mult * lv
                    depth = max(depth, dp)
            memo[size] = (leaves, depth + 1)
        return memo[size]

    leaves, depth = count(n)
    return FastStats(leaf_count=leaves, mean_leaf_size=n / leaves, depth=depth)


# ------------------------------------------------------------------ flatteners
def flatten_subsets(subsets) -> tuple[np.ndarray, np.ndarray]:
    """(row_idx, piece_off) for mdsx_classical_pieces / mdsx_divide_conquer."""
    sizes = np.fromiter((len(q) for q in subsets), dtype=np.int64, count=len(subsets))
    off = np.zeros(len(subsets) + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    return np.concatenate(subsets).astype(np.int64, copy=False), off


_FLAT_CACHE: dict = {}


def flatten_subsets_cached(plan) -> tuple[np.ndarray, np.ndarray]:
    """flatten_subsets(plan.subsets), memoised per plan object (a plan passed
    explicitly to several calls is flattened once; plans are not mutated).
    Keyed by identity; the entry is dropped when the plan is collected."""
    key = id(plan)
    hit = _FLAT_CACHE.get(key)
    if hit is not None and hit[0]() is plan and hit[1] is plan.subsets:
        return hit[2]
    flat = flatten_subsets(plan.subsets)
    try:
        ref = weakref.ref(plan, lambda _r, k=key: _FLAT_CACHE.pop(k, None))
    except TypeError:
        return flat
    _FLAT_CACHE[key] = (ref, plan.subsets, flat, {})
    return flat


def plan_device_cache(plan) -> dict | None:
    """Per-plan dict for device copies of the plan's index arrays (keyed by
    the caller, e.g. (device, name)): a plan passed to several calls is
    uploaded once; dropped with the plan.  None when the plan cannot be
    weak-referenced (then nothing is cached)."""
    if isinstance(plan, FastPlan):
        flat = flatten_fast_cached(plan)
        cache = getattr(flat, "_dev_cache", None)
        if cache is None:
            cache = flat._dev_cache = {}
        return cache
    flatten_subsets_cached(plan)
    hit = _FLAT_CACHE.get(id(plan))
    return hit[3] if hit is not None and hit[0]() is plan else None


@dataclass
class FastLevel:
    """One bottom-up alignment wave of fast MDS (all nodes at one depth).

    For job t (a child of some node at this depth): Procrustes target rows
    ``tgt_rows[job_off[t]:job_off[t+1]]`` index the piece-points buffer
    (the parent's alignment-set configuration), source rows ``src_rows``
    index the working buffer (the child's sampled rows); the fitted
    transform is then applied in place to working rows
    [start[t], start[t] + length[t])."""

    tgt_rows: np.ndarray
    src_rows: np.ndarray
    job_off: np.ndarray
    start: np.ndarray
    length: np.ndarray


@dataclass
class FastFlat:
    """Flattened fast-MDS tree for the GPU.

    The working buffer holds one row per data row in ``order`` (=
    root.indices) order; leaf j occupies rows [leaf_off[j], leaf_off[j+1]).
    Piece list for classical MDS = leaves (rows ``order``) followed by the
    alignment sets of internal nodes (rows ``align_rows``)."""

    order: np.ndarray
    piece_rows: np.ndarray
    piece_off: np.ndarray
    n_leaves: int
    levels: list
    labels: list
    eval_order: list      # piece ids in the reference's evaluation (error) order


def flatten_fast(plan: FastPlan) -> FastFlat:
    """Walk the tree once: leaves in DFS order, alignment sets of every
    internal node, and per-depth Procrustes jobs (deepest first)."""
    return _flatten_fast(plan.root, None)


_FAST_CACHE: dict = {}


def flatten_fast_cached(plan: FastPlan) -> FastFlat:
    """flatten_fast(plan) memoised per plan object (plans are not mutated; the
    entry is dropped when the plan is collected), with the fast_route arrays
    attached on first use (``route_cached``)."""
    key = id(plan)
    hit = _FAST_CACHE.get(key)
    if hit is not None and hit[0]() is plan and hit[1] is plan.root:
        return hit[2]
    flat = flatten_fast(plan)
    try:
        ref = weakref.ref(plan, lambda _r, k=key: _FAST_CACHE.pop(k, None))
    except TypeError:
        return flat
    _FAST_CACHE[key] = (ref, plan.root, flat)
    return flat


def route_cached(flat: "FastFlat") -> "FastRoute":
    rt = getattr(flat, "_route", None)
    if rt is None:
        rt = fast_route(flat)
        flat._route = rt
    return rt


def flatten_fast_shard(plan: FastPlan, lo: int, hi: int) -> FastFlat:
    """The share of one rank in sharded fast MDS: the level-1 subtrees
    lo..hi-1 of the root (leaves, their alignment sets and internal jobs,
    labelled as in the full tree), then the root's alignment set over ALL
    children (computed redundantly by every rank) and the root-level jobs
    aligning children lo..hi-1 onto their slices of it.  ``order`` = the
    owned subtrees' rows; no other rank's rows appear."""
    if plan.root.is_leaf:
        raise ValueError("a single-leaf plan has no level-1 subtrees")
    return _flatten_fast(plan.root, (lo, hi))


def _flatten_fast(root: FastNode, span) -> FastFlat:
    leaves, aligns, labels_leaf, labels_align = [], [], [], []
    by_depth: dict = {}
    cursor = [0]
    post = []            # ("leaf"|"align", index) in algorithms.py:285-303 evaluation order

    def walk(node: FastNode, depth: int, label: str) -> int:
        start = cursor[0]
        if node.is_leaf:
            post.append(("leaf", len(leaves)))
            leaves.append(node.indices)
            labels_leaf.append(label or "leaf 1")
            cursor[0] += node.size
            return start
        kid_starts = [walk(ch, depth + 1, f"{label}.{i + 1}" if label else f"branch {i + 1}")
                      for i, ch in enumerate(node.children)]
        samp = np.concatenate([ch.indices[ch.sampling_positions] for ch in node.children])
        post.append(("align", len(aligns)))
        aligns.append(samp)
        labels_align.append(f"{label or 'root'} alignment set")
        by_depth.setdefault(depth, []).append((len(aligns) - 1, list(node.children), kid_starts, 0))
        return start

    if span is None:
        walk(root, 0, "")
        order = root.indices
    else:
        lo, hi = span
        kids = root.children[lo:hi]
        kid_starts = [walk(ch, 1, f"branch {lo + i + 1}") for i, ch in enumerate(kids)]
        samp = np.concatenate([ch.indices[ch.sampling_positions] for ch in root.children])
        post.append(("align", len(aligns)))
        aligns.append(samp)
        labels_align.append("root alignment set")
        off0 = int(sum(len(ch.sampling_positions) for ch in root.children[:lo]))
        by_depth.setdefault(0, []).append((len(aligns) - 1, list(kids), kid_starts, off0))
        order = (np.concatenate([ch.indices for ch in kids]) if kids
                 else np.empty(0, dtype=np.int64))
    n_leaves = len(leaves)
    pieces = leaves + aligns
    piece_rows, piece_off = flatten_subsets(pieces)
    levels = []
    for depth in sorted(by_depth, reverse=True):
        tg, sr, jo, st, ln = [], [], [0], [], []
        for a_idx, children, kid_starts, off0 in by_depth[depth]:
            a_base = piece_off[n_leaves + a_idx]
            off = off0
            for ch, ks in zip(children, kid_starts):
                cnt = len(ch.sampling_positions)
                tg.append(np.arange(a_base + off, a_base + off + cnt, dtype=np.int64))
                sr.append(ks + ch.sampling_positions.astype(np.int64))
                off += cnt
                jo.append(jo[-1] + cnt)
                st.append(ks)
                ln.append(ch.size)
        if len(st) == 0:
            continue
        levels.append(FastLevel(np.concatenate(tg), np.concatenate(sr), np.asarray(jo, np.int64),
                                np.asarray(st, np.int64), np.asarray(ln, np.int64)))
    eval_order = [i if kind == "leaf" else n_leaves + i for kind, i in post]
    return FastFlat(np.asarray(order).astype(np.int64, copy=False), piece_rows, piece_off,
                    n_leaves, levels, labels_leaf + labels_align, eval_order)


@dataclass
class FastRoute:
    """Host arrays of ``mdsx_fast_mds`` (include/mdsx.h) for a flattened plan:
    the TRACKED rows (working-buffer rows some alignment job samples) with
    their data rows and leaves, and per level (deepest first) the jobs'
    sources (tracked ids) and targets (rows of the alignment-set points, in
    piece order), the job owning each tracked row and each leaf at that
    level (-1: none)."""

    trk_pos: np.ndarray
    trk_row: np.ndarray
    trk_leaf: np.ndarray
    level_njobs: np.ndarray
    job_off: np.ndarray
    job_src: np.ndarray
    job_tgt: np.ndarray
    trk_job: np.ndarray
    leaf_job: np.ndarray


def fast_route(flat: FastFlat) -> FastRoute:
    nl = flat.n_leaves
    off = np.asarray(flat.piece_off, dtype=np.int64)
    leaf_total = int(off[nl])
    leaf_of = np.repeat(np.arange(nl, dtype=np.int32), np.diff(off[:nl + 1]))
    levels = flat.levels
    src_all = (np.concatenate([lv.src_rows for lv in levels]) if levels
               else np.empty(0, np.int64))
    trk_pos = np.unique(src_all).astype(np.int64)
    leaf_start = off[:nl]
    njobs, joffs, srcs, tgts, tj, lj = [], [], [], [], [], []
    for lv in levels:
        st = np.asarray(lv.start, np.int64)
        ln = np.asarray(lv.length, np.int64)
        njobs.append(len(st))
        joffs.append(np.asarray(lv.job_off, np.int64))
        srcs.append(np.searchsorted(trk_pos, lv.src_rows).astype(np.int64))
        tgts.append(np.asarray(lv.tgt_rows, np.int64) - leaf_total)

        def owner(pos):
            k = np.searchsorted(st, pos, side="right") - 1
            ok = (k >= 0) & (pos < st[np.maximum(k, 0)] + ln[np.maximum(k, 0)])
            return np.where(ok, k, -1).astype(np.int32)
        tj.append(owner(trk_pos))
        lj.append(owner(leaf_start))
    cat = (lambda parts, dt: np.concatenate(parts).astype(dt) if parts else np.empty(0, dt))  # noqa: E731
    return FastRoute(trk_pos, np.asarray(flat.piece_rows, np.int64)[trk_pos], leaf_of[trk_pos],
                     np.asarray(njobs, np.int32), cat(joffs, np.int64), cat(srcs, np.int64),
                     cat(tgts, np.int64), cat(tj, np.int32), cat(lj, np.int32))
