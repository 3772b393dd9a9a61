"""Hash-indexed octree voxel map on the B200 — drop-in for livsplat.voxmap's
batch operations (voxmap.py:21-65, 99-251).

The device table (csrc/voxmap.cu) holds octree LEAVES keyed by their packed
integer key; internal nodes and roots are implied (a node exists iff a leaf
below it exists), so `_walk_create` becomes a single hash insert and
`leaf_keys_under_roots` a table scan against a root set.  Keys are computed
on the device as floor(p / edge) with f64 true division — bit-exact with the
reference.  Leaf statistics (count, sum p, sum p p^T) accumulate in f64.

Batch APIs take (n,3) point arrays and return device results; the
reference-shaped single-item calls (`locate_or_subdivide`, `try_insert`,
`get_leaf`, `leaf_keys_under_roots`, `iter_leaves`) wrap them.
"""

from __future__ import annotations

import ctypes
from typing import NamedTuple, Optional

import numpy as np
import torch

from . import _lib
from .errors import MissingVoxel

_P1, _P2, _P3 = 73856093, 19349669, 83492791


class VoxelKey(NamedTuple):
    """(ix, iy, iz, level) with the reference's prime-XOR hash (voxmap.py:21-38)."""

    ix: int
    iy: int
    iz: int
    level: int

    def __hash__(self):
        return (self.ix * _P1) ^ (self.iy * _P2) ^ (self.iz * _P3) ^ self.level

    def child(self, bx, by, bz):
        return VoxelKey(2 * self.ix + bx, 2 * self.iy + by, 2 * self.iz + bz, self.level + 1)

    def parent(self):
        return VoxelKey(self.ix // 2, self.iy // 2, self.iz // 2, self.level - 1)

    def root(self):
        s = 1 << self.level
        return VoxelKey(self.ix // s, self.iy // s, self.iz // s, 0)


def _iter_order(k: np.ndarray, L: int) -> np.ndarray:
    """Permutation of leaf keys (k,3) into iter_leaves order (voxmap.py:
    339-353): sorted root tuple, then octant DFS (x | y << 1 | z << 2 per level)."""
    roots = k >> L
    morton = np.zeros(len(k), dtype=np.int64)
    for d in range(L):             # level d+1 digit: bit (L-1-d) of each local coordinate
        b = L - 1 - d
        digit = ((k[:, 0] >> b) & 1) | (((k[:, 1] >> b) & 1) << 1) | (((k[:, 2] >> b) & 1) << 2)
        morton = morton * 8 + digit
    return np.lexsort((morton, roots[:, 2], roots[:, 1], roots[:, 0]))


def gaussian_row(g, width: Optional[int] = None) -> np.ndarray:
    """A Gaussian3D-like object as one f32 arena row (window.py:58-71):
    mean 3 | rot 9 | scale 3 | opacity 1 | sh 3K (K from `width` if given)."""
    sh = np.asarray(g.sh, dtype=np.float64).reshape(-1, 3)
    K = sh.shape[0] if width is None else (width - 16) // 3
    shk = np.zeros((K, 3))
    shk[: min(K, sh.shape[0])] = sh[:K]
    return np.concatenate([np.asarray(g.mean_w, float).ravel(), np.asarray(g.rot, float).ravel(),
                           np.asarray(g.scale, float).ravel(), [float(g.opacity)], shk.ravel()]).astype(np.float32)


def voxel_center(key, v_s: float) -> np.ndarray:
    """Centre of a voxel key at its level (voxmap.py:54-56)."""
    edge = v_s / (1 << key.level)
    return (np.array([key.ix, key.iy, key.iz], dtype=float) + 0.5) * edge


class LeafView:
    """A leaf of the device map seen through the reference's OctreeNode
    interface (voxmap.py:68-97): is_leaf, children (none), gaussians."""

    __slots__ = ("key", "gaussians", "count")
    is_leaf = True
    children = (None,) * 8

    def __init__(self, key, gaussians, count):
        self.key, self.gaussians, self.count = key, gaussians, count


class Inserted:
    pass


class Full:
    pass


def _dev_f64(points, device):
    t = torch.as_tensor(np.atleast_2d(np.asarray(points, dtype=np.float64))) if not torch.is_tensor(points) \
        else points
    return t.to(device=device, dtype=torch.float64).reshape(-1, 3).contiguous()


def keys_of_points_dev(points, edge: float, device=None) -> torch.Tensor:
    """Device (n,3) int64 floor(p / edge) (voxmap.py:59-65)."""
    _lib.require()
    device = device or torch.device("cuda")
    if edge <= 0:
        raise ValueError("root voxel length must be positive")
    pts = _dev_f64(points, device)
    out = torch.empty((pts.shape[0], 3), dtype=torch.int64, device=device)
    _lib.check(_lib.load().lsb_voxmap_keys(ctypes.c_void_p(pts.data_ptr()), pts.shape[0], float(edge),
                                           ctypes.c_void_p(out.data_ptr()), _lib.stream_ptr()), "voxmap_keys")
    return out


def keys_of_points(points, edge: float, level: int) -> list:
    """List of VoxelKey (voxmap.py:59-65)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    if pts.size == 0:
        return []
    k = keys_of_points_dev(pts, edge).cpu().numpy()
    return [VoxelKey(int(a), int(b), int(c), level) for a, b, c in k]


def hash_key(p, v_s: float) -> VoxelKey:
    if v_s <= 0:
        raise ValueError("root voxel length must be positive")
    return keys_of_points([p], v_s, 0)[0]


def leaf_key(p, v_s: float, max_level: int) -> VoxelKey:
    return keys_of_points([p], v_s / (1 << max_level), max_level)[0]


class HashOctree:
    """GPU voxel map: open-addressing table of octree leaves (voxmap.py:99-251)."""

    def __init__(self, root_len: float, max_level: int = 2, leaf_capacity: int = 1, capacity: int = 1 << 20,
                 device=None):
        if root_len <= 0:
            raise ValueError("root_len must be positive")
        if leaf_capacity != 1:
            raise ValueError("the device map stores one Gaussian per leaf (leaf_capacity == 1)")
        _lib.require()
        self.root_len = float(root_len)
        self.max_level = int(max_level)
        self.leaf_capacity = 1
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self._alloc(1 << max(10, int(np.ceil(np.log2(max(capacity, 2))))))
        self.gaussians: dict = {}        # gaussian id -> Gaussian3D-like payload (host, optional)
        self._next_gid = 0

    @property
    def leaf_len(self) -> float:
        return self.root_len / (1 << self.max_level)

    # ---- device storage -----------------------------------------------------
    def _alloc(self, cap: int):
        d = self.device
        self.cap = cap
        self.keys = torch.full((cap,), -1, dtype=torch.int64, device=d)       # 0xFF..FF = empty
        self.count = torch.zeros(cap, dtype=torch.int64, device=d)
        self.sum = torch.zeros((cap, 3), dtype=torch.float64, device=d)
        self.outer = torch.zeros((cap, 6), dtype=torch.float64, device=d)
        self.gslot = torch.full((cap,), -1, dtype=torch.int32, device=d)
        self.claim = torch.full((cap,), 0x7FFFFFFF, dtype=torch.int32, device=d)
        self.n_used = torch.zeros(1, dtype=torch.int64, device=d)
        self.flags = torch.zeros(1, dtype=torch.int64, device=d)
        # packed keys of the leaves that hold a Gaussian (append-only): the FoV
        # enumeration walks this list instead of the whole table
        self.gkeys = torch.empty(cap, dtype=torch.int64, device=d)
        self.n_gkeys = torch.zeros(1, dtype=torch.int64, device=d)

    def struct(self) -> _lib.VoxMap:
        return _lib.VoxMap(self.keys.data_ptr(), self.count.data_ptr(), self.sum.data_ptr(), self.outer.data_ptr(),
                           self.gslot.data_ptr(), self.claim.data_ptr(), self.n_used.data_ptr(),
                           self.flags.data_ptr(), self.cap, self.root_len, self.max_level, 0,
                           self.gkeys.data_ptr(), self.n_gkeys.data_ptr())

    def _reserve(self, extra: int):
        """Keep the load factor <= 1/2 (grow + rehash on the device; one sync)."""
        used = int(self.n_used.item())
        if used + extra <= self.cap // 2:
            return
        old = self.struct()
        keep = (self.keys, self.count, self.sum, self.outer, self.gslot, self.claim, self.n_used, self.flags,
                self.gkeys, self.n_gkeys)
        new_cap = self.cap
        while used + extra > new_cap // 2:
            new_cap *= 2
        self._alloc(new_cap)
        new = self.struct()
        _lib.check(_lib.load().lsb_voxmap_rehash(ctypes.byref(old), ctypes.byref(new), _lib.stream_ptr()), "rehash")
        self.gkeys[: keep[8].shape[0]].copy_(keep[8])         # packed keys do not move with the slots
        self.n_gkeys.copy_(keep[9])
        del keep

    def _check_flags(self):
        if int(self.flags.item()):
            raise RuntimeError("voxel map: table full or key outside the 21-bit range")

    # ---- batch operations (device) -------------------------------------------
    def accumulate_points_dev(self, points, accumulate: bool = True) -> torch.Tensor:
        """Add scan points to their leaves' statistics, creating leaves as
        needed (voxmap.py:184-190, 204-230); with accumulate=False only the
        leaves are created (ensure_leaf).  Returns per-point leaf slots."""
        pts = _dev_f64(points, self.device)
        n = pts.shape[0]
        self._reserve(n)
        slots = torch.empty(n, dtype=torch.int64, device=self.device)
        m = self.struct()
        lib = _lib.load()
        if accumulate:
            # deterministic: exact fixed-point group sums (integer atomics), one add per leaf
            nb = ctypes.c_size_t()
            _lib.check(lib.lsb_voxmap_accumulate_temp_bytes(n, ctypes.byref(nb)), "accumulate_temp")
            if getattr(self, "_acc_tmp", None) is None or self._acc_tmp.numel() < nb.value:
                self._acc_tmp = torch.empty(max(nb.value, 1), dtype=torch.uint8, device=self.device)
            _lib.check(lib.lsb_voxmap_accumulate(ctypes.byref(m), ctypes.c_void_p(pts.data_ptr()), n,
                                                 ctypes.c_void_p(slots.data_ptr()),
                                                 ctypes.c_void_p(self._acc_tmp.data_ptr()), self._acc_tmp.numel(),
                                                 _lib.stream_ptr()), "voxmap_accumulate")
            return slots
        _lib.check(lib.lsb_voxmap_insert_points(ctypes.byref(m), ctypes.c_void_p(pts.data_ptr()), n, 0,
                                                ctypes.c_void_p(slots.data_ptr()), _lib.stream_ptr()),
                   "voxmap_insert")
        return slots

    def accumulate_points(self, points_w) -> set:
        """Reference-shaped: returns the set of touched leaf keys."""
        slots = self.accumulate_points_dev(points_w)
        self._check_flags()
        from .sort import sort_pairs, unique_sorted
        u = unique_sorted(sort_pairs(slots)[0])
        return {self._key_of_slot(k) for k in self._keys_of_slots(u)}

    def try_insert_batch(self, means, first_gid: Optional[int] = None) -> torch.Tensor:
        """Batched try_insert (voxmap.py:171-182): status 1 Inserted / 0 Full.
        The lowest batch index wins an empty leaf (the reference's loop order)."""
        pts = _dev_f64(means, self.device)
        n = pts.shape[0]
        self._reserve(n)
        gid = self._next_gid if first_gid is None else int(first_gid)
        slots = torch.empty(n, dtype=torch.int64, device=self.device)
        status = torch.empty(n, dtype=torch.int32, device=self.device)
        m = self.struct()
        _lib.check(_lib.load().lsb_voxmap_try_insert(ctypes.byref(m), ctypes.c_void_p(pts.data_ptr()), n, gid,
                                                     ctypes.c_void_p(slots.data_ptr()),
                                                     ctypes.c_void_p(status.data_ptr()), _lib.stream_ptr()),
                   "voxmap_try_insert")
        self._next_gid = gid + n
        return status

    def lookup_dev(self, keys) -> torch.Tensor:
        k = torch.as_tensor(np.asarray(keys, dtype=np.int64)) if not torch.is_tensor(keys) else keys
        k = k.to(device=self.device, dtype=torch.int64).reshape(-1, 3).contiguous()
        out = torch.empty(k.shape[0], dtype=torch.int64, device=self.device)
        m = self.struct()
        _lib.check(_lib.load().lsb_voxmap_lookup(ctypes.byref(m), ctypes.c_void_p(k.data_ptr()), k.shape[0],
                                                 ctypes.c_void_p(out.data_ptr()), _lib.stream_ptr()), "lookup")
        return out

    def fov_leaf_keys_dev(self, points_w) -> torch.Tensor:
        """(k,3) int64 leaves holding a Gaussian under the root voxels the
        points touch (pipeline.py:190-191 -> voxmap.py:232-251)."""
        pts = _dev_f64(points_w, self.device)
        n = pts.shape[0]
        rcap = 1 << max(10, int(np.ceil(np.log2(max(2 * n, 2)))))
        rset = torch.empty(rcap, dtype=torch.int64, device=self.device)
        n_out = torch.zeros(1, dtype=torch.int64, device=self.device)
        out_cap = max(1024, int(self.n_used.item()))
        out = torch.empty((out_cap, 3), dtype=torch.int64, device=self.device)
        m = self.struct()
        _lib.check(_lib.load().lsb_voxmap_fov(ctypes.byref(m), ctypes.c_void_p(pts.data_ptr()), n,
                                              ctypes.c_void_p(rset.data_ptr()), rcap, ctypes.c_void_p(out.data_ptr()),
                                              ctypes.c_void_p(n_out.data_ptr()), out_cap, _lib.stream_ptr()), "fov")
        k = int(n_out.item())
        return out[:k]

    def dump_dev(self):
        """All occupied leaves: (keys (k,3) int64, slots (k,) int64)."""
        out_cap = max(1, int(self.n_used.item()))
        keys = torch.empty((out_cap, 3), dtype=torch.int64, device=self.device)
        slots = torch.empty(out_cap, dtype=torch.int64, device=self.device)
        n_out = torch.zeros(1, dtype=torch.int64, device=self.device)
        m = self.struct()
        _lib.check(_lib.load().lsb_voxmap_dump(ctypes.byref(m), ctypes.c_void_p(keys.data_ptr()),
                                               ctypes.c_void_p(slots.data_ptr()), ctypes.c_void_p(n_out.data_ptr()),
                                               out_cap, _lib.stream_ptr()), "dump")
        k = min(int(n_out.item()), out_cap)
        return keys[:k], slots[:k]

    # ---- plane fits (voxmap.py:255-335) ------------------------------------------
    def fit_planes_dev(self, keys, sensor_origin):
        """Batched plane fits of leaf keys (k,3): (normals (k,3), centroids
        (k,3), valid (k,) bool) on the device; NaN rows where no plane."""
        k = torch.as_tensor(np.asarray(keys, dtype=np.int64)) if not torch.is_tensor(keys) else keys
        k = k.to(device=self.device, dtype=torch.int64).reshape(-1, 3).contiguous()
        n = k.shape[0]
        normals = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        anchors = torch.empty((n, 3), dtype=torch.float64, device=self.device)
        valid = torch.empty(n, dtype=torch.uint8, device=self.device)
        o = (ctypes.c_double * 3)(*np.asarray(sensor_origin, dtype=np.float64).reshape(3).tolist())
        m = self.struct()
        _lib.check(_lib.load().lsb_voxmap_fit_planes(ctypes.byref(m), ctypes.c_void_p(k.data_ptr()), n, o,
                                                     ctypes.c_void_p(normals.data_ptr()),
                                                     ctypes.c_void_p(anchors.data_ptr()),
                                                     ctypes.c_void_p(valid.data_ptr()), _lib.stream_ptr()),
                   "fit_planes")
        return normals, anchors, valid.bool()

    def fit_planes(self, keys: list, sensor_origin) -> dict:
        """{key: (normal, centroid) or None}, like voxmap.py:297-335."""
        keys = list(keys)
        if not keys:
            return {}
        nrm, anc, ok = (t.cpu().numpy() for t in self.fit_planes_dev([[k[0], k[1], k[2]] for k in keys],
                                                                      sensor_origin))
        return {k: ((nrm[i], anc[i]) if ok[i] else None) for i, k in enumerate(keys)}

    def plane_at(self, key: VoxelKey, sensor_origin):
        """(normal, centroid) or None (voxmap.py:286-295)."""
        return self.fit_planes([key], sensor_origin)[key]

    def estimate_normal(self, key: VoxelKey, sensor_origin) -> np.ndarray:
        """Plane normal facing the sensor (voxmap.py:267-284); raises
        Degenerate when there is no plane.  (Evaluated like plane_at, so an
        empty leaf with populated neighbours is Degenerate here.)"""
        from .errors import Degenerate
        p = self.plane_at(key, sensor_origin)
        if p is None:
            raise Degenerate("no plane: fewer than 3 points, scatter rank < 2 or an empty leaf")
        return p[0]

    # ---- device Gaussian store (the map side of the sliding window) ------------
    def _store_reserve(self, rows: int, width: int) -> None:
        st = getattr(self, "store", None)
        if st is not None and st.shape[1] != width:
            raise ValueError(f"map rows have {st.shape[1]} floats, got {width}")
        if st is None or st.shape[0] < rows:
            cap = 1 << max(10, int(np.ceil(np.log2(max(rows, 2)))))
            new = torch.zeros((cap, width), dtype=torch.float32, device=self.device)
            if st is not None:
                new[: st.shape[0]] = st
            self.store = new

    def set_gaussians_dev(self, keys, rows) -> torch.Tensor:
        """Give each leaf key one Gaussian: rows (k, 16+3K) f32 in the
        reference's arena row layout (mean 3 | rot 9 | scale 3 | opacity 1 |
        sh 3K, window.py:58-60).  Leaves are created as needed (ensure_leaf);
        a leaf that already holds a Gaussian has it replaced (write_back,
        voxmap.py:190-194).  Returns the gids (k,) int32."""
        k = torch.as_tensor(np.asarray(keys, dtype=np.int64)) if not torch.is_tensor(keys) else keys
        k = k.to(device=self.device, dtype=torch.int64).reshape(-1, 3)
        rows = torch.as_tensor(rows, dtype=torch.float32).to(self.device).reshape(k.shape[0], -1)
        centers = (k.to(torch.float64) + 0.5) * self.leaf_len        # floor(centre / leaf_len) == key
        tslots = self.accumulate_points_dev(centers, accumulate=False)
        self._check_flags()
        g = self.gslot[tslots]
        new = g < 0
        n_new = int(new.sum().item())
        if n_new:
            g[new] = torch.arange(self._next_gid, self._next_gid + n_new, dtype=torch.int32, device=self.device)
            self._next_gid += n_new
            self.gslot[tslots] = g
            # new Gaussian leaves join the FoV list (tslots may repeat a key: once each)
            nk = torch.unique(self.keys[tslots[new]])
            pos = self.n_gkeys + torch.arange(nk.numel(), dtype=torch.int64, device=self.device)
            self.gkeys[pos] = nk
            self.n_gkeys += nk.numel()
        self._store_reserve(self._next_gid, rows.shape[1])
        self.store[g.long()] = rows
        return g

    def gaussian_rows_dev(self, keys) -> torch.Tensor:
        """Store rows of the leaves' Gaussians (NaN rows where none)."""
        t = self.lookup_dev(keys)
        g = torch.where(t >= 0, self.gslot[t.clamp(min=0)], torch.full_like(t, -1, dtype=torch.int32))
        out = torch.full((t.shape[0], self.store.shape[1]), float("nan"), dtype=torch.float32, device=self.device)
        ok = g >= 0
        out[ok] = self.store[g[ok].long()]
        return out

    # ---- persistence (voxmap.py:358-415) ---------------------------------------
    _MAGIC = b"LSMAP001"

    def _records(self):
        """(keys (r,3) int64, rows (r, 16+3K) f32) of the leaves holding a
        Gaussian, in the reference's iteration order (voxmap.py:339-353);
        one device gather, one copy to the host."""
        keys, slots = self.dump_dev()
        g = self.gslot[slots] if slots.numel() else torch.empty(0, dtype=torch.int32, device=self.device)
        has = g >= 0
        keys, g = keys[has], g[has]
        st = getattr(self, "store", None)
        if keys.shape[0] == 0 or st is None:
            return np.zeros((0, 3), np.int64), np.zeros((0, 19), np.float32)
        rows = st[g.long()].cpu().numpy()
        k = keys.cpu().numpy()
        order = _iter_order(k, self.max_level)
        return k[order], rows[order]

    def gaussian_count(self) -> int:
        return int(self._records()[0].shape[0])

    def save(self, path) -> None:
        """Binary snapshot, byte-identical to the reference's (voxmap.py:
        362-375): magic, <IdII Q header, per record <qqqI key + level and the
        f32 row (mean 3 | rot 9 | scale 3 | opacity 1 | sh 3K)."""
        import struct
        keys, rows = self._records()
        sh_k = (rows.shape[1] - 16) // 3 if len(keys) else 1
        rec = np.zeros(len(keys), dtype=np.dtype([("k", "<i8", (3,)), ("lv", "<u4"), ("f", "<f4", (16 + 3 * sh_k,))],
                                                  align=False))
        rec["k"] = keys
        rec["lv"] = self.max_level
        if len(keys):
            rec["f"] = rows
        with open(path, "wb") as f:
            f.write(self._MAGIC)
            f.write(struct.pack("<IdII Q", 1, self.root_len, self.max_level, sh_k, len(keys)))
            f.write(rec.tobytes())

    @classmethod
    def load(cls, path, device=None) -> "HashOctree":
        """Inverse of save (voxmap.py:377-399); the Gaussians go to the
        device store of a new map."""
        import struct
        with open(path, "rb") as f:
            if f.read(8) != cls._MAGIC:
                raise ValueError("not a map snapshot")
            hdr = struct.calcsize("<IdII Q")
            version, root_len, max_level, sh_k, n = struct.unpack("<IdII Q", f.read(hdr))
            if version != 1:
                raise ValueError(f"unsupported snapshot version {version}")
            rec = np.frombuffer(f.read(), dtype=np.dtype([("k", "<i8", (3,)), ("lv", "<u4"),
                                                          ("f", "<f4", (16 + 3 * sh_k,))]), count=n)
        m = cls(root_len, max_level, capacity=max(1 << 10, 2 * n), device=device)
        if n:
            if np.any(rec["lv"] != max_level):
                raise ValueError("the device map holds leaf-level Gaussians only")
            m.set_gaussians_dev(rec["k"].astype(np.int64), rec["f"].astype(np.float32))
        return m

    def export_ply(self, path) -> None:
        """ASCII PLY of the means and view-independent colours, text-identical
        to the reference's (voxmap.py:401-415)."""
        _, rows = self._records()
        c0 = 0.28209479177387814                      # sh.SH_C0
        rgb = np.clip(0.5 + c0 * rows[:, 16:19].astype(np.float64), 0.0, 1.0)
        q = np.round(rgb * 255).astype(int)
        mean = rows[:, 0:3].astype(np.float64)
        with open(path, "w") as f:
            f.write("ply\nformat ascii 1.0\n")
            f.write(f"element vertex {len(rows)}\n")
            f.write("property float x\nproperty float y\nproperty float z\n")
            f.write("property uchar red\nproperty uchar green\nproperty uchar blue\n")
            f.write("end_header\n")
            f.writelines(f"{a:.6f} {b:.6f} {c:.6f} {r} {g} {bl}\n"
                         for (a, b, c), (r, g, bl) in zip(mean.tolist(), q.tolist()))

    # ---- reference-shaped helpers ------------------------------------------------
    def _keys_of_slots(self, slots: torch.Tensor) -> np.ndarray:
        slots = slots[slots >= 0]
        packed = self.keys[slots].cpu().numpy().astype(np.uint64)
        mask = np.uint64((1 << 21) - 1)
        off = 1 << 20
        ix = (packed & mask).astype(np.int64) - off
        iy = ((packed >> np.uint64(21)) & mask).astype(np.int64) - off
        iz = ((packed >> np.uint64(42)) & mask).astype(np.int64) - off
        return np.stack([ix, iy, iz], axis=1)

    def _key_of_slot(self, k) -> VoxelKey:
        return VoxelKey(int(k[0]), int(k[1]), int(k[2]), self.max_level)

    def locate_or_subdivide(self, p) -> VoxelKey:
        """Leaf key containing p, creating it if needed (voxmap.py:156-160)."""
        self.accumulate_points_dev([p], accumulate=False)
        return leaf_key(p, self.root_len, self.max_level)

    def ensure_leaf(self, key: VoxelKey):
        center = (np.array([key.ix, key.iy, key.iz], dtype=float) + 0.5) * self.leaf_len
        self.accumulate_points_dev([center], accumulate=False)
        return self.get_leaf(key)

    def try_insert(self, g):
        status = self.try_insert_batch([np.asarray(g.mean_w, dtype=float)])
        ok = bool(int(status.item()))
        if ok:
            gid = self._next_gid - 1
            self.gaussians[gid] = g
            g.level = self.max_level
            if all(hasattr(g, a) for a in ("rot", "scale", "opacity", "sh")):    # full payload: device row
                row = gaussian_row(g, None if getattr(self, "store", None) is None else self.store.shape[1])
                self._store_reserve(gid + 1, row.shape[0])
                self.store[gid] = torch.as_tensor(row, device=self.device)
        return Inserted() if ok else Full()

    def get_leaf(self, key: VoxelKey):
        s = int(self.lookup_dev([[key.ix, key.iy, key.iz]]).item())
        if s < 0:
            return None
        return {"slot": s, "gid": int(self.gslot[s].item()), "count": int(self.count[s].item())}

    def write_back(self, key: VoxelKey, params) -> None:
        leaf = self.get_leaf(key)
        if leaf is None:
            raise MissingVoxel(key)
        if params and leaf["gid"] >= 0:
            self.gaussians[leaf["gid"]] = params[0]
        if params and getattr(self, "store", None) is not None:
            self.set_gaussians_dev([[key.ix, key.iy, key.iz]], gaussian_row(params[0], self.store.shape[1])[None])

    def leaf_stats(self, key: VoxelKey):
        leaf = self.get_leaf(key)
        if leaf is None or leaf["count"] == 0:
            return None
        s = leaf["slot"]
        o = self.outer[s].cpu().numpy()
        outer = np.array([[o[0], o[1], o[2]], [o[1], o[3], o[4]], [o[2], o[4], o[5]]])
        return [leaf["count"], self.sum[s].cpu().numpy(), outer]

    def leaf_stats_dev(self, keys):
        """Batched leaf_stats for (k,3) leaf keys: (count (k,) int64, sum
        (k,3) f64, outer (k,3,3) f64); zeros where the key has no leaf."""
        t = self.lookup_dev(keys)
        ok = t >= 0
        tc = t.clamp(min=0)
        cnt = torch.where(ok, self.count[tc], torch.zeros_like(self.count[tc]))
        sm = torch.where(ok[:, None], self.sum[tc], torch.zeros_like(self.sum[tc]))
        o = torch.where(ok[:, None], self.outer[tc], torch.zeros_like(self.outer[tc]))
        outer = torch.stack([o[:, 0], o[:, 1], o[:, 2], o[:, 1], o[:, 3], o[:, 4], o[:, 2], o[:, 4], o[:, 5]],
                            dim=1).reshape(-1, 3, 3)
        return cnt, sm, outer

    def fov_root_keys(self, points_w) -> set:
        return set(keys_of_points(points_w, self.root_len, 0))

    def leaf_keys_under_roots(self, root_keys) -> set:
        roots = np.array([[k[0], k[1], k[2]] for k in root_keys], dtype=np.float64).reshape(-1, 3)
        centers = (roots + 0.5) * self.root_len     # floor(center / root_len) == root key
        keys = self.fov_leaf_keys_dev(centers).cpu().numpy()
        return {VoxelKey(int(a), int(b), int(c), self.max_level) for a, b, c in keys}

    def fov_leaf_keys(self, points_w) -> set:
        """voxmap.py:187-188: the leaf keys of the points themselves."""
        return set(keys_of_points(points_w, self.leaf_len, self.max_level))

    def group_by_leaf(self, points_w) -> dict:
        """Leaf key -> stacked points (voxmap.py:213-230): keys ascend in
        (ix, iy, iz) order and each group keeps scan order.  The keys and
        the stable grouping sort run on the device; the groups are numpy
        arrays like the reference's."""
        pts = np.atleast_2d(np.asarray(points_w, dtype=float))
        if pts.size == 0:
            return {}
        keys = keys_of_points_dev(pts, self.leaf_len, self.device)
        from .window import order_keys
        from .sort import sort_pairs
        ok, order = sort_pairs(order_keys(keys))
        ok, order = ok.cpu().numpy(), order.cpu().numpy()
        idx = keys.cpu().numpy()[order]
        spts = pts[order]
        cuts = np.flatnonzero(ok[1:] != ok[:-1]) + 1
        groups = {}
        for ci, cp in zip(np.split(idx, cuts), np.split(spts, cuts)):
            groups[VoxelKey(int(ci[0, 0]), int(ci[0, 1]), int(ci[0, 2]), self.max_level)] = cp
        return groups

    def add_leaf_stats(self, key, pts) -> None:
        """voxmap.py:204-211: count += n; sum += pts.sum(axis=0); outer +=
        pts^T pts, the group's sums formed like the reference's and added to
        the leaf's device statistics (created if needed)."""
        pts = np.atleast_2d(np.asarray(pts, dtype=float))
        if pts.size == 0:
            return
        leaf = self.ensure_leaf(key)
        s = leaf["slot"]
        psum = pts.sum(axis=0)
        po = pts.T @ pts
        self.count[s] += len(pts)
        self.sum[s] += torch.as_tensor(psum, device=self.device)
        self.outer[s] += torch.as_tensor([po[0, 0], po[0, 1], po[0, 2], po[1, 1], po[1, 2], po[2, 2]],
                                         device=self.device)

    def iter_leaves(self):
        """(key, leaf) in the reference's order (voxmap.py:339-353): sorted
        root tuple, then octant DFS.  leaf.gaussians holds the leaf's
        Gaussian (the host payload given to try_insert, else one built from
        its device store row)."""
        from .geometry import Gaussian3D
        keys, slots = self.dump_dev()
        k = keys.cpu().numpy()
        if len(k) == 0:
            return
        order = _iter_order(k, self.max_level)
        sl = slots[torch.as_tensor(order, device=self.device)]
        gids = self.gslot[sl].cpu().numpy()
        counts = self.count[sl].cpu().numpy()
        rows = None
        if getattr(self, "store", None) is not None and (gids >= 0).any():
            g = torch.as_tensor(np.where(gids >= 0, gids, 0), device=self.device).long()
            rows = self.store[g].cpu().numpy()
        for i, (a, b, c) in enumerate(k[order]):
            key = VoxelKey(int(a), int(b), int(c), self.max_level)
            gs = []
            gid = int(gids[i])
            if gid >= 0:
                if gid in self.gaussians:
                    gs = [self.gaussians[gid]]
                elif rows is not None:
                    r = rows[i].astype(np.float64)
                    K = (r.shape[0] - 16) // 3
                    gs = [Gaussian3D(r[0:3], r[3:12].reshape(3, 3), r[12:15], float(r[15]), r[16:].reshape(K, 3),
                                     level=self.max_level)]
            yield key, LeafView(key, gs, int(counts[i]))

    def iter_leaf_keys(self) -> list:
        """Leaf keys in the reference's iteration order (voxmap.py:339-353):
        sorted root tuple, then octant DFS (x bit | y << 1 | z << 2 per level)."""
        keys, _ = self.dump_dev()
        k = keys.cpu().numpy()
        if len(k) == 0:
            return []
        L = self.max_level
        return [VoxelKey(int(a), int(b), int(c), L) for a, b, c in k[_iter_order(k, L)]]
