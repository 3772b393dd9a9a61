"""GPU-resident sliding window of Gaussians — drop-in for livsplat.window
(window.py:91-276), SURVEY.md §8(f) rank 1.

The reference keeps a host arena plus an emulated device mirror and moves
dirty rows between them every frame.  Here the window IS the device arena
the renderer reads (f32 SoA, `as_gaussian_arrays()` returns views of its
live prefix, no copies), the global map's Gaussians are rows of the voxel
map's device store (`HashOctree.store`, indexed by the leaf's gid), and
`maintain` runs the reference's protocol on the device (csrc/window.cu):

  diff        window hash (key -> slot) probed by the FoV keys          (window.py:136-143)
  write-back  deleted rows -> their leaves' store rows                   (window.py:145-150)
  compact     the i-th deleted slot below the new live count takes the
              i-th live slot at or above it, counted from the rear —
              the closed form of the reference's rear-pointer loop       (window.py:151-181)
  drop        over capacity: keep the adds nearest the sensor (f64
              distance as numpy computes it, ties by key)                (window.py:262-270)
  append      adds holding a Gaussian, in sorted key order, at the rear  (window.py:183-209)

Slot layout, rows and report counts are identical to the reference's
(tests/test_gpu_window.py against tests/golden/window_walk.npz, produced by
the reference itself).  There is no host mirror, so `sync_to_device` /
`sync_to_host` move nothing and the report's byte counters stay 0.  Key
sorting and de-duplication use the library's own stable radix sort
(csrc/sort.cu).  `init_fn` (Gaussian synthesis for FoV leaves without one) is a
host callback, as in the reference.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib
from .errors import WindowFull
from .raster import GaussianArrays
from .sort import sort_pairs, unique_sorted
from .voxmap import HashOctree, VoxelKey, gaussian_row

_KOFF = 1 << 20
_KMASK = (1 << 21) - 1


def order_keys(keys) -> torch.Tensor:
    """(k,3) int keys -> int64 order keys (integer order == sorted VoxelKey order)."""
    k = keys if torch.is_tensor(keys) else torch.as_tensor(np.asarray(keys, dtype=np.int64).reshape(-1, 3))
    k = k.to(torch.int64)
    return ((k[:, 0] + _KOFF) << 42) | ((k[:, 1] + _KOFF) << 21) | (k[:, 2] + _KOFF)


def _sorted(ok: torch.Tensor) -> torch.Tensor:
    """Order keys ascending (the library's radix sort; keys are < 2^63)."""
    return sort_pairs(ok, key_bits=63, signed=False)[0]


def _sorted_unique(ok: torch.Tensor) -> torch.Tensor:
    return unique_sorted(_sorted(ok))


def unpack_order_keys(ok: torch.Tensor) -> torch.Tensor:
    return torch.stack([((ok >> 42) & _KMASK) - _KOFF, ((ok >> 21) & _KMASK) - _KOFF, (ok & _KMASK) - _KOFF], dim=1)


@dataclass
class FrameDiff:
    overlap: list
    delete: list
    add: list


@dataclass
class MaintenanceReport:
    n_live: int = 0
    added: int = 0
    removed: int = 0
    moved: int = 0
    dropped: int = 0
    bytes_up: int = 0
    bytes_down: int = 0
    t_maintain_ms: float = 0.0


class GaussianWindow:
    """Device sliding window (window.py:91-276).  Leaf keys at the map's
    max_level; one Gaussian per slot."""

    def __init__(self, capacity: int = 100_000, sh_coeffs: int = 1, device=None):
        _lib.require()
        self.capacity = int(capacity)
        self.sh_coeffs = int(sh_coeffs)
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        d, C, K = self.device, self.capacity, self.sh_coeffs
        self.means = torch.zeros((C, 3), dtype=torch.float32, device=d)
        self.rots = torch.zeros((C, 3, 3), dtype=torch.float32, device=d)
        self.scales = torch.zeros((C, 3), dtype=torch.float32, device=d)
        self.opacities = torch.zeros(C, dtype=torch.float32, device=d)
        self.shs = torch.zeros((C, K, 3), dtype=torch.float32, device=d)
        self.wkeys = torch.full((C,), -1, dtype=torch.int64, device=d)      # order key per slot
        self.n = 0
        hcap = 1 << max(10, int(np.ceil(np.log2(2 * max(C, 1)))))
        self._hkeys = torch.empty(hcap, dtype=torch.int64, device=d)
        self._hslots = torch.empty(hcap, dtype=torch.int32, device=d)
        self._keep = torch.zeros(max(C, 1), dtype=torch.uint8, device=d)
        self._dels = torch.empty(max(C, 1), dtype=torch.int32, device=d)
        self._movers = torch.empty(max(C, 1), dtype=torch.int32, device=d)
        self._counts = torch.zeros(2, dtype=torch.int64, device=d)
        self._n_added = torch.zeros(1, dtype=torch.int64, device=d)
        self._pending: Optional[dict] = None

    def _tile_scratch(self, ints: int) -> torch.Tensor:
        """int32 scratch of the multi-CTA plan / append scans (kept, grown)."""
        t = getattr(self, "_tiles", None)
        if t is None or t.numel() < max(int(ints), 1):
            t = self._tiles = torch.empty(max(int(ints), 64), dtype=torch.int32, device=self.device)
        return t

    @property
    def row_floats(self) -> int:
        return 16 + 3 * self.sh_coeffs

    def _arena(self) -> _lib.Params:
        return _lib.Params(self.means.data_ptr(), self.rots.data_ptr(), self.scales.data_ptr(),
                           self.opacities.data_ptr(), self.shs.data_ptr(), self.capacity, self.sh_coeffs, 0)

    # ---- queries -------------------------------------------------------------
    def live_keys_dev(self) -> torch.Tensor:
        """(n,3) int64 live keys in slot order."""
        return unpack_order_keys(self.wkeys[: self.n])

    def live_keys(self, level: Optional[int] = None) -> set:
        lv = -1 if level is None else level
        return {VoxelKey(int(a), int(b), int(c), lv) for a, b, c in self.live_keys_dev().cpu().numpy()}

    def rows_dev(self) -> torch.Tensor:
        """(n, 16+3K) f32 live rows in slot order (the reference's row layout)."""
        n = self.n
        return torch.cat([self.means[:n], self.rots[:n].reshape(n, 9), self.scales[:n], self.opacities[:n, None],
                          self.shs[:n].reshape(n, -1)], dim=1)

    def gaussian_at(self, key, device: bool = False):
        """The live Gaussian of a leaf key (window.py:106-109; the window is
        the device arena, so `device` changes nothing).  KeyError if the key
        is not live."""
        from .geometry import Gaussian3D
        ok = order_keys(torch.as_tensor([[key[0], key[1], key[2]]], dtype=torch.int64, device=self.device))
        hit = (self.wkeys[: self.n] == ok[0]).nonzero().flatten()
        if hit.numel() == 0:
            raise KeyError(key)
        s = int(hit[0])
        r = self.rows_dev()[s].double().cpu().numpy()
        K = self.sh_coeffs
        return Gaussian3D(r[0:3], r[3:12].reshape(3, 3), r[12:15], float(r[15]), r[16:16 + 3 * K].reshape(K, 3),
                          level=int(key[3]) if len(key) > 3 else 0)

    def as_gaussian_arrays(self) -> GaussianArrays:
        """The live prefix as the renderer's arrays (views, no copy;
        window.py:109-120 upcasts a copy instead)."""
        n = self.n
        return GaussianArrays(self.means[:n], self.rots[:n], self.scales[:n], self.opacities[:n], self.shs[:n],
                              device=self.device)

    def audit(self) -> None:
        """Prefix liveness and key uniqueness (window.py:122-133)."""
        k = self.wkeys[: self.n]
        assert bool((k >= 0).all()), "free slot inside the live prefix"
        assert int(unique_sorted(sort_pairs(k, key_bits=63, signed=False)[0]).numel()) == self.n, \
            "key mapped twice"
        assert bool((self.wkeys[self.n:] < 0).all()), "live key outside the prefix"

    # ---- protocol --------------------------------------------------------------
    def _fov_order_keys(self, fov_keys) -> torch.Tensor:
        if torch.is_tensor(fov_keys):
            return order_keys(fov_keys.to(self.device).reshape(-1, 3))
        lst = [(k[0], k[1], k[2]) for k in fov_keys]
        return order_keys(torch.as_tensor(np.asarray(lst, dtype=np.int64).reshape(-1, 3), device=self.device))

    def _mark(self, fov_ok: torch.Tensor) -> torch.Tensor:
        m = int(fov_ok.numel())
        is_add = torch.empty(max(m, 1), dtype=torch.uint8, device=self.device)
        hcap = self._hkeys.numel()
        _lib.check(_lib.load().lsb_window_mark(
            ctypes.c_void_p(self.wkeys.data_ptr()), self.n, ctypes.c_void_p(self._hkeys.data_ptr()),
            ctypes.c_void_p(self._hslots.data_ptr()), hcap, ctypes.c_void_p(fov_ok.data_ptr()) if m else None, m,
            ctypes.c_void_p(self._keep.data_ptr()), ctypes.c_void_p(is_add.data_ptr()), _lib.stream_ptr()),
            "window_mark")
        return is_add[:m]

    def diff(self, fov_keys) -> FrameDiff:
        """Sorted overlap / delete / add key lists (window.py:136-143)."""
        fov_ok = _sorted_unique(self._fov_order_keys(fov_keys))
        is_add = self._mark(fov_ok).bool()
        live = self.wkeys[: self.n]
        keep = self._keep[: self.n].bool()
        lv = -1
        to_keys = lambda ok: [VoxelKey(int(a), int(b), int(c), lv)
                              for a, b, c in unpack_order_keys(_sorted(ok)).cpu().numpy()]
        return FrameDiff(overlap=to_keys(live[keep]), delete=to_keys(live[~keep]), add=to_keys(fov_ok[is_add]))

    def writeback_and_compact(self, vmap: HashOctree) -> tuple:
        """Write the deleted rows back to the map and compact (window.py:
        145-181).  Uses the keep marks of the last diff.  Returns (removed, moved)."""
        lib = _lib.load()
        n = self.n
        _lib.check(lib.lsb_window_plan(ctypes.c_void_p(self._keep.data_ptr()), n,
                                       ctypes.c_void_p(self._dels.data_ptr()),
                                       ctypes.c_void_p(self._movers.data_ptr()),
                                       ctypes.c_void_p(self._counts.data_ptr()),
                                       ctypes.c_void_p(self._tile_scratch(lib.lsb_window_plan_tiles(n)).data_ptr()),
                                       _lib.stream_ptr()), "window_plan")
        k, h = (int(v) for v in self._counts.cpu())
        if k:
            if getattr(vmap, "store", None) is None:
                raise ValueError("the map holds no Gaussian rows (HashOctree.set_gaussians_dev)")
            m = vmap.struct()
            a = self._arena()
            _lib.check(lib.lsb_window_compact(ctypes.byref(m), ctypes.byref(a), ctypes.c_void_p(self.wkeys.data_ptr()),
                                              ctypes.c_void_p(self._dels.data_ptr()), k,
                                              ctypes.c_void_p(self._movers.data_ptr()), h, n,
                                              ctypes.c_void_p(vmap.store.data_ptr()), _lib.stream_ptr()),
                       "window_compact")
            if int(vmap.flags.item()) & 2:
                from .errors import MissingVoxel
                vmap.flags.zero_()
                raise MissingVoxel("a window key has no leaf in the map")
        self.n = n - k
        return k, h

    def writeback_deleted(self, vmap: HashOctree, diff: FrameDiff) -> None:
        """Write the rows of diff.delete back to the map (window.py:145-150);
        compact() then closes the holes.  Marks the live keys of the diff's
        overlap as kept (the same marks diff() leaves)."""
        keep = list(diff.overlap)
        fov_ok = _sorted(self._fov_order_keys(keep)) if keep else torch.empty(0, dtype=torch.int64,
                                                                               device=self.device)
        self._mark(fov_ok)
        if diff.delete:
            rows = self.rows_dev()
            gone = ~self._keep[: self.n].bool()
            vmap.set_gaussians_dev(self.live_keys_dev()[gone], rows[gone])
        self._pending_vmap = vmap

    def compact(self) -> int:
        """Close the holes of the deleted slots (window.py:152-181: each
        deleted slot, ascending, takes the rearmost live slot).  Returns the
        number of moves."""
        vmap = getattr(self, "_pending_vmap", None)
        if vmap is None:
            return 0
        self._pending_vmap = None
        _, moved = self.writeback_and_compact(vmap)
        return moved

    def _leaf_gids(self, vmap: HashOctree, ok: torch.Tensor) -> torch.Tensor:
        gids = torch.empty(max(ok.numel(), 1), dtype=torch.int32, device=self.device)
        m = vmap.struct()
        _lib.check(_lib.load().lsb_window_leaf_gids(ctypes.byref(m), ctypes.c_void_p(ok.data_ptr()), ok.numel(),
                                                    ctypes.c_void_p(gids.data_ptr()), _lib.stream_ptr()),
                   "window_leaf_gids")
        return gids[: ok.numel()]

    def append_keys(self, vmap: HashOctree, add_ok: torch.Tensor, init_fn: Optional[Callable] = None) -> int:
        """Append the (sorted) add keys holding a Gaussian, synthesising
        missing ones with init_fn first (window.py:183-209).  Raises
        WindowFull before mutating the window if the rows cannot fit."""
        add_ok = add_ok.contiguous()
        gids = self._leaf_gids(vmap, add_ok) if add_ok.numel() else add_ok.to(torch.int32)
        if init_fn is not None and add_ok.numel():
            missing = (gids < 0).nonzero().flatten()
            if missing.numel():
                keys = unpack_order_keys(add_ok[missing]).cpu().numpy()
                new_keys, new_rows = [], []
                for a, b, c in keys:                      # sorted key order, like the reference
                    gs = init_fn(VoxelKey(int(a), int(b), int(c), vmap.max_level)) or []
                    if len(gs) > 1:
                        raise ValueError("window requires leaf_capacity == 1")
                    if gs:
                        new_keys.append((a, b, c))
                        new_rows.append(gaussian_row(gs[0], self.row_floats))
                if new_keys:
                    vmap.set_gaussians_dev(np.asarray(new_keys, dtype=np.int64), np.stack(new_rows))
                    gids = self._leaf_gids(vmap, add_ok)
        n_rows = int((gids >= 0).sum().item())
        if self.n + n_rows > self.capacity:
            raise WindowFull(f"{self.n} + {n_rows} > {self.capacity}")
        if n_rows == 0:
            return 0
        a = self._arena()
        _lib.check(_lib.load().lsb_window_append(ctypes.byref(a), ctypes.c_void_p(self.wkeys.data_ptr()),
                                                 ctypes.c_void_p(add_ok.data_ptr()), ctypes.c_void_p(gids.data_ptr()),
                                                 add_ok.numel(), ctypes.c_void_p(vmap.store.data_ptr()), self.n,
                                                 ctypes.c_void_p(self._n_added.data_ptr()),
                                                 ctypes.c_void_p(self._tile_scratch(
                                                     _lib.load().lsb_window_append_tiles(add_ok.numel())).data_ptr()),
                                                 _lib.stream_ptr()),
                   "window_append")
        self.n += n_rows
        return n_rows

    def append(self, vmap: HashOctree, add: list, init_fn: Optional[Callable] = None) -> int:
        """Reference-shaped append of a key list (window.py:183)."""
        ok = _sorted(self._fov_order_keys(add)) if len(add) else torch.empty(0, dtype=torch.int64,
                                                                            device=self.device)
        return self.append_keys(vmap, ok, init_fn)

    def sync_to_device(self) -> int:
        return 0            # the window is the device arena: nothing to mirror

    def sync_to_host(self) -> int:
        return 0

    def mark_device_dirty_live(self) -> None:
        pass

    def maintain(self, vmap: HashOctree, fov_keys, init_fn: Optional[Callable] = None,
                 sensor_pos: Optional[np.ndarray] = None) -> MaintenanceReport:
        """One frame of the incremental protocol (window.py:236-276).
        fov_keys: (k,3) int64 tensor (e.g. HashOctree.fov_leaf_keys_dev) or
        an iterable of VoxelKey."""
        t0 = time.perf_counter()
        rep = MaintenanceReport()
        # the FoV keys need no order: the hash marks give keep / add per key,
        # and only the adds (a few percent of the FoV) are sorted and
        # de-duplicated for the ordered append (window.py:254-276)
        fov_ok = self._fov_order_keys(fov_keys)
        is_add = self._mark(fov_ok).bool()
        rep.removed, rep.moved = self.writeback_and_compact(vmap)
        add_ok = _sorted_unique(fov_ok[is_add])                 # sorted, unique
        n_add = int(add_ok.numel())
        if self.n + n_add > self.capacity:
            if sensor_pos is None:
                raise WindowFull("capacity exceeded and no sensor position to rank drops")
            room = self.capacity - self.n
            origin = (ctypes.c_double * 3)(*np.asarray(sensor_pos, dtype=np.float64).reshape(3).tolist())
            dist = torch.empty(max(n_add, 1), dtype=torch.float64, device=self.device)
            _lib.check(_lib.load().lsb_window_dist(ctypes.c_void_p(add_ok.data_ptr()), n_add,
                                                   vmap.root_len / (1 << vmap.max_level), origin,
                                                   ctypes.c_void_p(dist.data_ptr()), _lib.stream_ptr()),
                       "window_dist")
            # stable ascending distance (non-negative f64: its bits order as int64); the
            # keys are already ascending, so ties keep key order
            order = sort_pairs(dist[:n_add].view(torch.int64), key_bits=63, signed=False)[1].long()
            rep.dropped = n_add - room
            add_ok = _sorted(add_ok[order[:room]])
        rep.added = self.append_keys(vmap, add_ok, init_fn)
        rep.n_live = self.n
        rep.t_maintain_ms = (time.perf_counter() - t0) * 1e3
        return rep
