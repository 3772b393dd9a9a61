"""Host-side rigid-body math for the splat path (6-dof, numpy f64).

Pose conventions follow the reference (geometry.py:1-20): IMU poses are
perturbed on the right for rotation and additively for translation (boxplus);
camera poses T_CW on the left.  This is tiny per-call host math — the GPU
only ever sees the resulting T_cw — so it stays in numpy, evaluated with the
same expressions as the reference so the bits handed to the kernels match.
Reference objects (anything with .R/.t, or fx/fy/cx/cy/width/height) are
accepted wherever these types are.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def hat(v) -> np.ndarray:
    x, y, z = np.asarray(v, dtype=float).reshape(3)
    return np.array([[0.0, -z, y], [z, 0.0, -x], [-y, x, 0.0]])


def so3_exp(phi) -> np.ndarray:
    """Rodrigues with the second-order series below 1e-8 (geometry.py:43-53)."""
    phi = np.asarray(phi, dtype=float)
    theta = float(np.linalg.norm(phi))
    S = hat(phi)
    if theta < 1e-8:
        return np.eye(3) + S + 0.5 * (S @ S)
    return np.eye(3) + (np.sin(theta) / theta) * S + ((1.0 - np.cos(theta)) / theta**2) * (S @ S)


@dataclass
class SE3:
    """p_out = R p_in + t (geometry.py:125-171)."""

    R: np.ndarray = field(default_factory=lambda: np.eye(3))
    t: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        self.R = np.asarray(self.R, dtype=float).reshape(3, 3)
        self.t = np.asarray(self.t, dtype=float).reshape(3)

    @staticmethod
    def identity() -> "SE3":
        return SE3(np.eye(3), np.zeros(3))

    def inverse(self) -> "SE3":
        Rt = self.R.T
        return SE3(Rt, -Rt @ self.t)

    def __matmul__(self, other) -> "SE3":
        return SE3(self.R @ other.R, self.R @ other.t + self.t)

    def apply(self, p) -> np.ndarray:
        p = np.asarray(p, dtype=float)
        return self.R @ p + self.t if p.ndim == 1 else p @ self.R.T + self.t


@dataclass
class Twist:
    rho: np.ndarray
    tau: np.ndarray

    def __post_init__(self):
        self.rho = np.asarray(self.rho, dtype=float).reshape(3)
        self.tau = np.asarray(self.tau, dtype=float).reshape(3)


def boxplus(T, xi) -> SE3:
    """(R Exp(rho), t + tau) (geometry.py:186-188)."""
    return SE3(T.R @ so3_exp(xi.rho), T.t + xi.tau)


def as_se3(T) -> SE3:
    return T if isinstance(T, SE3) else SE3(np.asarray(T.R), np.asarray(T.t))


def imu_camera_adjoint(R_cw, T_ic) -> np.ndarray:
    """6x6 A with (rho_l, tau_l) = A (rho_r, tau_r) (geometry.py:202-228)."""
    R_ci = np.asarray(T_ic.R, dtype=float).T
    t_ci = -R_ci @ np.asarray(T_ic.t, dtype=float)
    A = np.zeros((6, 6))
    A[:3, :3] = -R_ci
    A[3:, :3] = -hat(t_ci) @ R_ci
    A[3:, 3:] = -np.asarray(R_cw, dtype=float)
    return A


@dataclass
class PinholeCamera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if not (0 <= self.cx < self.width and 0 <= self.cy < self.height):
            raise ValueError("principal point outside image")
