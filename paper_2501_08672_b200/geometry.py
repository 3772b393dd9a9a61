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


def so3_log(R) -> np.ndarray:
    """Inverse of so3_exp, theta in [0, pi] (geometry.py:56-79)."""
    R = np.asarray(R, dtype=float)
    cos_theta = np.clip(0.5 * (float(np.trace(R)) - 1.0), -1.0, 1.0)
    theta = float(np.arccos(cos_theta))
    w = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    if theta < 1e-8:
        return 0.5 * w
    if np.pi - theta > 1e-6:
        return (theta / (2.0 * np.sin(theta))) * w
    B = 0.5 * (R + np.eye(3))
    k = int(np.argmax(np.diag(B)))
    axis = B[:, k] / np.sqrt(max(B[k, k], 1e-12))
    axis = axis / np.linalg.norm(axis)
    if np.dot(w, axis) < 0.0:
        axis = -axis
    return theta * axis


def so3_left_jacobian(phi) -> np.ndarray:
    phi = np.asarray(phi, dtype=float)
    theta = float(np.linalg.norm(phi))
    S = hat(phi)
    if theta < 1e-6:
        return np.eye(3) + 0.5 * S + (S @ S) / 6.0
    return np.eye(3) + ((1.0 - np.cos(theta)) / theta**2) * S + ((theta - np.sin(theta)) / theta**3) * (S @ S)


def so3_right_jacobian_inv(phi) -> np.ndarray:
    """J_r^-1(phi) = J_l^-1(-phi) (geometry.py:96-107)."""
    phi = -np.asarray(phi, dtype=float)
    theta = float(np.linalg.norm(phi))
    S = hat(phi)
    if theta < 1e-6:
        return np.eye(3) - 0.5 * S + (S @ S) / 12.0
    b = (1.0 / theta**2) - 0.5 / (theta * np.tan(0.5 * theta))
    return np.eye(3) - 0.5 * S + b * (S @ S)


@dataclass
class Gaussian3D:
    """Planar-slice Gaussian primitive (geometry.py:271-309): the same fields
    and defaults as the reference's, so reference-built Gaussians and these
    are interchangeable at the boundary."""

    mean_w: np.ndarray
    rot: np.ndarray
    scale: np.ndarray
    opacity: float
    sh: np.ndarray
    level: int = 0

    def __post_init__(self):
        self.mean_w = np.asarray(self.mean_w, dtype=float).reshape(3)
        self.rot = np.asarray(self.rot, dtype=float).reshape(3, 3)
        self.scale = np.asarray(self.scale, dtype=float).reshape(3)
        self.sh = np.asarray(self.sh, dtype=float).reshape(-1, 3)

    def covariance(self) -> np.ndarray:
        B = self.rot * self.scale[None, :]
        return B @ B.T


@dataclass
class Gaussian2D:
    """Screen-space footprint of a splatted Gaussian (geometry.py:311-323)."""

    mean_i: np.ndarray
    cov_i: np.ndarray
    depth: float
    color: np.ndarray
    opacity: float

    def __post_init__(self):
        self.mean_i = np.asarray(self.mean_i, dtype=float).reshape(2)
        self.cov_i = np.asarray(self.cov_i, dtype=float).reshape(2, 2)
        self.color = np.asarray(self.color, dtype=float).reshape(3)
