"""TEST INFRASTRUCTURE ONLY — CPU oracle for the loss and the Adam step.

Restates /root/reference/pkg/src/livsplat/optimize.py: photometric_loss
(:48-74), AdamState.update (:103-119), the storage-coordinate parameter step
(:159-188), _batch_so3_exp (:77-88) and _orthonormalize (:91-100).  Pinned
by tests/test_oracle_golden.py against tests/golden/adam.npz and
optimize_plane.npz.
"""

from __future__ import annotations

import numpy as np

from . import raster as orc


def photometric_loss(rendered, observed, mask=None, kind="l1"):
    diff = np.asarray(rendered, float) - np.asarray(observed, float)
    if mask is None:
        mask = np.ones(diff.shape[:2], bool)
    npix = int(mask.sum())
    denom = 3.0 * npix
    m3 = mask[..., None]
    if kind == "l1":
        value = float(np.abs(diff[mask]).sum() / denom)
        grad = np.where(m3, np.sign(diff), 0.0) / denom
    else:
        value = float((diff[mask] ** 2).sum() / denom)
        grad = np.where(m3, 2.0 * diff, 0.0) / denom
    return value, float((diff[mask] ** 2).sum() / denom), grad


class Adam:
    def __init__(self, shapes, beta1=0.9, beta2=0.999, eps=1e-15):
        self.b1, self.b2, self.eps = beta1, beta2, eps
        self.step = 0
        self.m = {k: np.zeros(s) for k, s in shapes.items()}
        self.v = {k: np.zeros(s) for k, s in shapes.items()}

    def update(self, name, g, lr):
        m = self.m[name] = self.b1 * self.m[name] + (1 - self.b1) * g
        v = self.v[name] = self.b2 * self.v[name] + (1 - self.b2) * g ** 2
        return -lr * (m / (1 - self.b1 ** self.step)) / (np.sqrt(v / (1 - self.b2 ** self.step)) + self.eps)


def so3_exp_batch(phi):
    th = np.linalg.norm(phi, axis=1)
    S = np.zeros((len(phi), 3, 3))
    S[:, 0, 1], S[:, 0, 2] = -phi[:, 2], phi[:, 1]
    S[:, 1, 0], S[:, 1, 2] = phi[:, 2], -phi[:, 0]
    S[:, 2, 0], S[:, 2, 1] = -phi[:, 1], phi[:, 0]
    small = th < 1e-8
    with np.errstate(invalid="ignore", divide="ignore"):
        a = np.where(small, 1.0, np.sin(th) / np.where(small, 1.0, th))
        b = np.where(small, 0.5, (1.0 - np.cos(th)) / np.where(small, 1.0, th ** 2))
    return np.eye(3)[None] + a[:, None, None] * S + b[:, None, None] * (S @ S)


def orthonormalize(R):
    c0 = R[:, :, 0] / np.linalg.norm(R[:, :, 0], axis=1, keepdims=True)
    c1 = R[:, :, 1] - np.sum(R[:, :, 1] * c0, axis=1, keepdims=True) * c0
    c1 = c1 / np.linalg.norm(c1, axis=1, keepdims=True)
    return np.stack([c0, c1, np.cross(c0, c1)], axis=2)


def adam_param_step(P, grads, adam, cfg, touched):
    """One storage-coordinate step (optimize.py:169-188), in place on P (f64)."""
    adam.step += 1
    P["means"] = P["means"] + adam.update("mean", grads["mean"], cfg["lr_mean"] * cfg.get("scene_scale", 1.0))
    phi = adam.update("rot", grads["rot"], cfg["lr_rot"])
    rows = np.any(phi != 0.0, axis=1)
    if np.any(rows):
        P["rots"][rows] = P["rots"][rows] @ so3_exp_batch(phi[rows])
        touched |= rows
    s = P["scales"]
    st = adam.update("scale", grads["scale"] * s, cfg["lr_scale"])
    new = np.maximum(np.exp(np.log(np.maximum(s, 1e-6)) + st), 1e-6)
    P["scales"] = np.where(st == 0.0, s, new)
    op = P["opacities"]
    oc = np.clip(op, 1e-4, 1 - 1e-4)
    so = adam.update("opacity", grads["opacity"] * oc * (1.0 - oc), cfg["lr_opacity"])
    P["opacities"] = np.where(so == 0.0, op, 1.0 / (1.0 + np.exp(-(np.log(oc / (1.0 - oc)) + so))))
    P["shs"] = P["shs"] + adam.update("sh", grads["sh"], cfg["lr_sh"])


DEFAULT_CFG = dict(lr_mean=1.6e-4, lr_sh=2.5e-3, lr_opacity=5e-2, lr_scale=5e-3, lr_rot=1e-3, scene_scale=1.0)


def optimize_views(P, observed, poses_cw, cam, st, iters, cfg=DEFAULT_CFG):
    """Multi-view window optimisation: per iteration the gradient is the
    mean over views of the per-view reference gradients,
    then one Adam step; rotations re-orthonormalised at the end.  With one
    view this is optimize_window (optimize.py:122-202) in f64."""
    P = {k: np.array(v, dtype=np.float64, copy=True) for k, v in P.items()}
    n = len(P["means"])
    adam = Adam({"mean": (n, 3), "rot": (n, 3), "scale": (n, 3), "opacity": (n,), "sh": P["shs"].shape})
    touched = np.zeros(n, bool)
    history = []
    V = len(poses_cw)
    for _ in range(iters):
        acc = None
        losses = []
        for (R_cw, t_cw), obs in zip(poses_cw, observed):
            c = orc.render(P, R_cw, t_cw, cam, st)
            val, mse, g_img = photometric_loss(c["image"], obs)
            losses.append(val)
            g = orc.backward(c, g_img)["grads"]
            acc = g if acc is None else {k: acc[k] + g[k] for k in acc}
        grads = {k: v / V for k, v in acc.items()}
        adam_param_step(P, grads, adam, cfg, touched)
        history.append(losses)
    if np.any(touched):
        P["rots"][touched] = orthonormalize(P["rots"][touched])
    return P, history
