"""TEST INFRASTRUCTURE ONLY — CPU oracle for the hash-octree voxel map.

Restates /root/reference/pkg/src/livsplat/voxmap.py: keys by floor(p / edge)
with true division (:41-65), grouping by leaf with a lexsort (:213-230),
leaf statistics [count, sum p, sum p p^T] (:204-211), capacity-1 insertion
(:171-182), the FoV leaf set under root voxels (:232-251) and the
iteration order (sorted root tuple, then octant DFS, :339-353).  The octree
is represented by its leaf set (an internal node exists iff a leaf below it
does).  Pinned by tests/test_oracle_golden.py against tests/golden/voxmap.npz.
"""

from __future__ import annotations

import numpy as np


def keys(points, edge):
    return np.floor(np.atleast_2d(np.asarray(points, dtype=float)) / edge).astype(np.int64)


class Map:
    def __init__(self, root_len, max_level):
        self.root_len = float(root_len)
        self.max_level = int(max_level)
        self.leaves = {}      # (ix, iy, iz) -> [count, sum(3), outer(3,3), has_gaussian]

    @property
    def leaf_len(self):
        return self.root_len / (1 << self.max_level)

    def _leaf(self, k):
        leaf = self.leaves.get(k)
        if leaf is None:
            leaf = [0, np.zeros(3), np.zeros((3, 3)), False]
            self.leaves[k] = leaf
        return leaf

    def accumulate_points(self, pts):
        pts = np.atleast_2d(np.asarray(pts, dtype=float))
        if pts.size == 0:
            return set()
        idx = keys(pts, self.leaf_len)
        order = np.lexsort((idx[:, 2], idx[:, 1], idx[:, 0]))
        idx, pts = idx[order], pts[order]
        cuts = np.nonzero(np.any(np.diff(idx, axis=0) != 0, axis=1))[0] + 1
        touched = set()
        for ki, kp in zip(np.split(idx, cuts), np.split(pts, cuts)):
            k = tuple(int(v) for v in ki[0])
            leaf = self._leaf(k)
            leaf[0] += len(kp)
            leaf[1] = leaf[1] + kp.sum(axis=0)
            leaf[2] = leaf[2] + kp.T @ kp
            touched.add(k)
        return touched

    def try_insert(self, mean):
        k = tuple(int(v) for v in keys(mean, self.leaf_len)[0])
        leaf = self._leaf(k)
        if leaf[3]:
            return False
        leaf[3] = True
        return True

    def leaf_keys_under_roots(self, roots):
        roots = {tuple(int(v) for v in r[:3]) for r in roots}
        L = self.max_level
        return {k for k, leaf in self.leaves.items() if leaf[3] and (k[0] >> L, k[1] >> L, k[2] >> L) in roots}

    def iter_keys(self):
        L = self.max_level

        def sort_key(k):
            digits = tuple((((k[0] >> b) & 1) | (((k[1] >> b) & 1) << 1) | (((k[2] >> b) & 1) << 2))
                           for b in range(L - 1, -1, -1))
            return (k[0] >> L, k[1] >> L, k[2] >> L) + digits

        return sorted(self.leaves, key=sort_key)
