"""k-means and best-first multi-output CART behind the pruning strategies.

Restates reference pkg/src/kernelprune/clustering.py with identical
floating-point operation order, because the pruned config sets must be
bit-identical to the reference's given the same timing CSV:
  kmeans (k-means++ seeding, Lloyd, best-of-restarts)     (:60-120)
  fit_regression_tree / predict_tree / tree_leaves        (:336-476)
Tie conventions (reference module docstring :6-12): argmin ties -> lowest
index; split thresholds are midpoints of consecutive distinct sorted values;
equal splits prefer lower feature then lower threshold; x == threshold goes
right. HDBSCAN (reference :125-332) is outside the north_star path and is
provided by hdbscan.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DataError, DimensionMismatch
from .rng import KMEANS_STREAM, Xoshiro256StarStar, derive_seed


class KTooLarge(DataError):
    pass


class TooFewPoints(DataError):
    pass


@dataclass
class KMeansResult:
    centroids: np.ndarray     # (k, C)
    assignments: np.ndarray   # (P,)
    inertia: float
    iterations: int


# ------------------------------------------------------------------ k-means

def _sqnorm_rows(diff: np.ndarray) -> np.ndarray:
    return np.einsum("ij,ij->i", diff, diff)


def _distances(points: np.ndarray, centers: np.ndarray) -> np.ndarray:
    """Squared distance of every point to every center, one column per
    center (plain (x-c)^2 sums keep exact ties exact)."""
    out = np.empty((points.shape[0], centers.shape[0]))
    for j, c in enumerate(centers):
        out[:, j] = _sqnorm_rows(points - c)
    return out


def _seed_centers(points: np.ndarray, k: int, rng: Xoshiro256StarStar) -> np.ndarray:
    """k-means++: first center uniform, then D^2-weighted draws."""
    p = points.shape[0]
    picks = [rng.below(p)]
    nearest = _sqnorm_rows(points - points[picks[0]])
    for _ in range(1, k):
        mass = float(nearest.sum())
        if mass > 0.0:
            target = rng.random() * mass
            nxt = min(int(np.searchsorted(np.cumsum(nearest), target, side="right")), p - 1)
        else:
            nxt = rng.below(p)  # every point sits on a center already
        picks.append(nxt)
        nearest = np.minimum(nearest, _sqnorm_rows(points - points[nxt]))
    return points[picks].astype(np.float64, copy=True)


def _lloyd(points, centers, k, max_iter, trace):
    labels = _distances(points, centers).argmin(axis=1)
    steps = 0
    while steps < max_iter:
        for j in range(k):
            mine = points[labels == j]
            if len(mine):
                centers[j] = mine.mean(axis=0)
        d2 = _distances(points, centers)
        relabel = d2.argmin(axis=1)
        steps += 1
        if trace is not None:
            trace.append(float(d2[np.arange(len(points)), relabel].sum()))
        if np.array_equal(relabel, labels):
            break
        labels = relabel
    return labels, steps


def kmeans(points, k: int, seed: int, restarts: int = 10, max_iter: int = 300,
           _trace=None) -> KMeansResult:
    """Best-inertia Lloyd run over `restarts` k-means++ seedings.

    Restart r uses stream (seed, KMEANS_STREAM, r); empty clusters keep their
    previous center; a later restart replaces the best only if strictly
    better.
    """
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[0] == 0:
        raise DataError("points must be a non-empty 2-D array")
    if k < 1:
        raise ValueError("k must be >= 1")
    if k > pts.shape[0]:
        raise KTooLarge(f"k={k} exceeds point count {len(pts)}")
    if restarts < 1:
        raise ValueError("restarts must be >= 1")
    best: KMeansResult | None = None
    for r in range(restarts):
        centers = _seed_centers(pts, k, Xoshiro256StarStar(derive_seed(seed, KMEANS_STREAM, r)))
        labels, steps = _lloyd(pts, centers, k, max_iter, _trace)
        resid = pts - centers[labels]
        inertia = float(np.einsum("ij,ij->", resid, resid))
        if best is None or inertia < best.inertia:
            best = KMeansResult(centers.copy(), labels.copy(), inertia, steps)
    return best


# ------------------------------------------------------ multi-output CART

@dataclass
class TreeLeaf:
    value: np.ndarray  # mean target of member rows
    count: int


@dataclass
class TreeSplit:
    feature: int
    threshold: float
    left: "TreeSplit | TreeLeaf"
    right: "TreeSplit | TreeLeaf"


@dataclass
class RegressionTree:
    root: "TreeSplit | TreeLeaf"
    leaf_count: int
    n_features: int


def _sse(y: np.ndarray) -> float:
    return float(((y - y.mean(axis=0)) ** 2).sum())


def _scan_feature(sorted_vals, cum, cumsq, base_sse, tol, best, f):
    """Update `best` with the best midpoint split of one sorted feature."""
    n = len(sorted_vals)
    total, totalsq = cum[-1], cumsq[-1]
    for i in range(1, n):
        if sorted_vals[i] == sorted_vals[i - 1]:
            continue
        left = cum[i - 1]
        right = total - left
        sse_left = cumsq[i - 1] - float(left @ left) / i
        sse_right = (totalsq - cumsq[i - 1]) - float(right @ right) / (n - i)
        gain = base_sse - sse_left - sse_right
        if gain > tol and (best is None or gain > best[0]):
            best = (gain, f, (sorted_vals[i - 1] + sorted_vals[i]) / 2.0)
    return best


def _best_split(x: np.ndarray, y: np.ndarray, rows: np.ndarray, base_sse: float):
    """(SSE reduction, feature, threshold) of the best split, or None.

    Prefix sums give every candidate's SSE; the relative tolerance keeps
    cancellation noise from splitting constant targets.
    """
    if len(rows) < 2:
        return None
    tol = 1e-9 * (1.0 + base_sse)
    yr = y[rows]
    sq = np.einsum("ij,ij->i", yr, yr)
    best = None
    for f in range(x.shape[1]):
        vals = x[rows, f]
        order = np.argsort(vals, kind="stable")
        best = _scan_feature(vals[order], np.cumsum(yr[order], axis=0),
                             np.cumsum(sq[order]), base_sse, tol, best, f)
    return best


class _Grower:
    """Best-first growth bookkeeping: open leaves in creation order."""

    def __init__(self, x, y):
        self.x, self.y = x, y
        self.open: dict[int, tuple] = {}   # id -> (rows, best split or None)
        self.created: list[int] = []
        self.splits: dict[int, tuple] = {}  # id -> (feature, thr, left id, right id)

    def add(self, rows) -> int:
        nid = len(self.created)
        self.created.append(nid)
        self.open[nid] = (rows, _best_split(self.x, self.y, rows, _sse(self.y[rows])))
        return nid

    def pick(self):
        chosen, gain = None, None
        for nid in self.created:
            rec = self.open.get(nid)
            if rec is None or rec[1] is None:
                continue
            if chosen is None or rec[1][0] > gain:
                chosen, gain = nid, rec[1][0]
        return chosen

    def split(self, nid) -> None:
        rows, (_, f, thr) = self.open.pop(nid)
        goes_left = self.x[rows, f] < thr
        lid = self.add(rows[goes_left])
        rid = self.add(rows[~goes_left])
        self.splits[nid] = (f, thr, lid, rid)

    def node(self, nid):
        if nid in self.splits:
            f, thr, lid, rid = self.splits[nid]
            return TreeSplit(f, thr, self.node(lid), self.node(rid))
        rows = self.open[nid][0]
        return TreeLeaf(self.y[rows].mean(axis=0), len(rows))


def fit_regression_tree(features, targets, max_leaves: int) -> RegressionTree:
    """Best-first CART: repeatedly split the open leaf with the largest SSE
    reduction (earliest-created leaf on ties) until max_leaves or no gain."""
    x = np.atleast_2d(np.asarray(features, dtype=np.float64))
    y = np.atleast_2d(np.asarray(targets, dtype=np.float64))
    if len(x) == 0 or len(x) != len(y):
        raise DataError("features and targets must have the same non-zero length")
    if max_leaves < 1:
        raise ValueError("max_leaves must be >= 1")
    g = _Grower(x, y)
    root = g.add(np.arange(len(x)))
    while len(g.open) < max_leaves:
        nid = g.pick()
        if nid is None:
            break
        g.split(nid)
    return RegressionTree(g.node(root), len(g.open), x.shape[1])


def predict_tree(tree: RegressionTree, row) -> np.ndarray:
    """Leaf mean for one feature row (threshold ties go right)."""
    r = np.asarray(row, dtype=np.float64)
    if r.shape != (tree.n_features,):
        raise DimensionMismatch(f"expected {tree.n_features} features, got shape {r.shape}")
    node = tree.root
    while isinstance(node, TreeSplit):
        node = node.right if not r[node.feature] < node.threshold else node.left
    return node.value.copy()


def tree_leaves(tree: RegressionTree) -> list[TreeLeaf]:
    """Leaves left to right."""
    def walk(node):
        if isinstance(node, TreeLeaf):
            return [node]
        return walk(node.left) + walk(node.right)
    return walk(tree.root)


def __getattr__(name):
    # HDBSCAN lives in its own module; keep the reference's import path working
    if name in ("hdbscan", "HdbscanResult"):
        from . import hdbscan as _h
        return getattr(_h, name)
    raise AttributeError(name)
