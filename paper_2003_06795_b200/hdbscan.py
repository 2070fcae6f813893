"""HDBSCAN over performance rows (the reference's "hdbscan" pruning method).

Restates reference pkg/src/kernelprune/clustering.py:125-332. Outside the
north_star hot path (which names top-N / k-means / PCA / decision tree) but
kept so `prune(method="hdbscan")` and the report tables stay drop-in.

Pipeline: core distance = min_samples-th nearest other point; mutual
reachability max(core_a, core_b, d_ab); exact Prim MST from vertex 0 (ties to
the lowest vertex); single-linkage merge rows; condensation by
min_cluster_size with BFS cluster numbering; leaf-first excess-of-mass
selection with the root excluded unless nothing survives condensation;
medoid = member minimising summed mutual reachability (lowest index on ties).
"""

from __future__ import annotations

import math
from collections import deque
from dataclasses import dataclass

import numpy as np

from .clustering import TooFewPoints
from .errors import DataError


@dataclass
class HdbscanResult:
    labels: np.ndarray
    cluster_medoids: tuple[int, ...]
    stabilities: tuple[float, ...]


def _euclidean(points: np.ndarray) -> np.ndarray:
    p = len(points)
    d = np.empty((p, p))
    for i in range(p):
        diff = points - points[i]
        d[i] = np.sqrt(np.einsum("ij,ij->i", diff, diff))
    np.fill_diagonal(d, 0.0)
    return d


def _prim(weights: np.ndarray) -> list[tuple[int, int, float]]:
    p = len(weights)
    done = np.zeros(p, dtype=bool)
    done[0] = True
    key = weights[0].copy()
    via = np.zeros(p, dtype=np.int64)
    edges = []
    for _ in range(p - 1):
        v = int(np.where(done, np.inf, key).argmin())
        edges.append((int(via[v]), v, float(key[v])))
        done[v] = True
        improve = (weights[v] < key) & ~done
        key[improve] = weights[v][improve]
        via[improve] = v
    return edges


class _UnionFind:
    def __init__(self, n):
        self.parent = list(range(n))

    def find(self, x):
        root = x
        while self.parent[root] != root:
            root = self.parent[root]
        while self.parent[x] != root:
            self.parent[x], x = root, self.parent[x]
        return root


def _linkage(edges, p: int):
    ordered = sorted(((min(u, v), max(u, v), w) for u, v, w in edges),
                     key=lambda e: (e[2], e[0], e[1]))
    uf = _UnionFind(p)
    node_of = list(range(p))
    size_of = [1] * p
    merges = []
    for i, (a, b, w) in enumerate(ordered):
        ra, rb = uf.find(a), uf.find(b)
        na, nb = node_of[ra], node_of[rb]
        size = size_of[ra] + size_of[rb]
        merges.append((min(na, nb), max(na, nb), w, size))
        uf.parent[ra] = rb
        node_of[rb] = p + i
        size_of[rb] = size
    return merges


def _points_under(node: int, p: int, left, right) -> list[int]:
    out, todo = [], [node]
    while todo:
        cur = todo.pop()
        if cur < p:
            out.append(cur)
        else:
            todo.append(left[cur])
            todo.append(right[cur])
    return out


def _excess(lam: float, birth: float) -> float:
    if math.isinf(lam) and math.isinf(birth):
        return 0.0  # duplicate points: both infinite, no mass
    return lam - birth


def hdbscan(points, min_cluster_size: int = 3, min_samples: int = 2) -> HdbscanResult:
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or len(pts) == 0:
        raise DataError("points must be a non-empty 2-D array")
    p = len(pts)
    if min_cluster_size < 2:
        raise ValueError("min_cluster_size must be >= 2")
    if min_samples < 1:
        raise ValueError("min_samples must be >= 1")
    if p < min_cluster_size:
        raise TooFewPoints(f"need at least {min_cluster_size} points, got {p}")
    if min_samples > p - 1:
        raise TooFewPoints(f"min_samples={min_samples} needs at least {min_samples + 1} points")

    dist = _euclidean(pts)
    core = np.sort(dist, axis=1)[:, min_samples]
    mreach = np.maximum(np.maximum.outer(core, core), dist)
    np.fill_diagonal(mreach, 0.0)

    merges = _linkage(_prim(mreach), p)
    total_nodes = 2 * p - 1
    left = np.full(total_nodes, -1, dtype=np.int64)
    right = np.full(total_nodes, -1, dtype=np.int64)
    height = np.zeros(total_nodes)
    weight = np.ones(total_nodes, dtype=np.int64)
    for i, (a, b, w, s) in enumerate(merges):
        left[p + i], right[p + i], height[p + i], weight[p + i] = a, b, w, s

    # ---- condensation (clusters numbered in BFS creation order, root = 0)
    root = 2 * p - 2
    cluster_of = {root: 0}
    kids: dict[int, list[int]] = {0: []}
    birth = {0: 0.0}
    fallen: list[tuple[int, int, float]] = []          # (cluster, point, lambda)
    born: list[tuple[int, int, float, int]] = []       # (parent, child, lambda, size)
    next_id = 1
    queue = deque([root])
    while queue:
        node = queue.popleft()
        cid = cluster_of[node]
        a, b = int(left[node]), int(right[node])
        lam = math.inf if height[node] == 0.0 else 1.0 / height[node]
        sides = [(c, 1 if c < p else int(weight[c])) for c in (a, b)]
        large = [c for c, s in sides if s >= min_cluster_size]
        small = [c for c, s in sides if s < min_cluster_size]
        if len(large) == 2:
            for c in (a, b):
                cluster_of[c] = next_id
                kids[cid].append(next_id)
                kids[next_id] = []
                birth[next_id] = lam
                born.append((cid, next_id, lam, int(weight[c])))
                next_id += 1
                queue.append(c)
        else:
            for c in small:
                fallen.extend((cid, pt, lam) for pt in _points_under(c, p, left, right))
            if large:
                cluster_of[large[0]] = cid
                queue.append(large[0])

    stability = {c: 0.0 for c in kids}
    for cid, _, lam in fallen:
        stability[cid] += _excess(lam, birth[cid])
    for parent, _, lam, size in born:
        stability[parent] += _excess(lam, birth[parent]) * size

    # ---- leaf-first excess of mass (root never a candidate)
    keep: dict[int, bool] = {}
    best_below: dict[int, float] = {}
    for c in range(next_id - 1, 0, -1):
        below = sum(best_below[k] for k in kids[c])
        if kids[c] and below > stability[c]:
            keep[c], best_below[c] = False, below
        else:
            keep[c], best_below[c] = True, stability[c]
    chosen: list[int] = []
    stack = [(0, False)]
    while stack:
        c, covered = stack.pop()
        take = c != 0 and not covered and keep.get(c, False)
        if take:
            chosen.append(c)
        for k in kids[c]:
            stack.append((k, covered or take))
    chosen.sort()
    if not kids[0]:
        chosen = [0]

    rank = {c: i for i, c in enumerate(chosen)}
    parent_of: dict[int, int | None] = {0: None}
    for c, ks in kids.items():
        for k in ks:
            parent_of[k] = c
    labels = np.full(p, -1, dtype=np.int64)
    for cid, pt, _ in fallen:
        c = cid
        while c is not None:
            if c in rank:
                labels[pt] = rank[c]
                break
            c = parent_of[c]

    medoids, stabs = [], []
    for c in chosen:
        members = np.nonzero(labels == rank[c])[0]
        sub = mreach[np.ix_(members, members)]
        medoids.append(int(members[int(sub.sum(axis=1).argmin())]))
        stabs.append(float(stability[c]))
    return HdbscanResult(labels, tuple(medoids), tuple(stabs))
