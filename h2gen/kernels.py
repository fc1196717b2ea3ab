"""Kernel functions K(x, y) used to fill the H² data (generator side only).

exp:      K = exp(-r / ell)            2D set ell = 0.1a, 3D ell = 0.2a
gaussian: K = exp(-(r / ell)^2)        BASELINE config 3 wording ("3D Gaussian kernel"; reading R9)
poly:     K = (1 + x.y)^(p-1)          coordinate degree <= p-1: Chebyshev interpolation of order p is
                                       exact, so A~ = K to rounding (pin of SURVEY.md §8(c))
fd:       K = -2 sqrt(kappa_i kappa_j) / r^(2+2 beta), K_ii = 0   (reading R10)
"""
from dataclasses import dataclass, field
import numpy as np


@dataclass
class Kernel:
    name: str
    ell: float = 0.1
    p: int = 4                 # poly: order (degree p-1)
    beta: float = 0.75         # fd
    sign: float = -1.0         # fd: -1 for K, +1 for K^ (the D assembly)
    params: dict = field(default_factory=dict)

    def __call__(self, x, y):
        """x, y: broadcastable (..., dim) arrays -> (...) values."""
        if self.name == "exp":
            r = np.sqrt(_r2(x, y))
            r *= -1.0 / self.ell
            return np.exp(r, out=r)
        if self.name == "gaussian":
            r2 = _r2(x, y)
            r2 *= -1.0 / (self.ell * self.ell)
            return np.exp(r2, out=r2)
        if self.name == "poly":
            dot = x[..., 0] * y[..., 0]
            for d in range(1, x.shape[-1]):
                dot = dot + x[..., d] * y[..., d]
            return (1.0 + dot) ** (self.p - 1)
        if self.name == "fd":
            r2 = _r2(x, y)
            kx = fd_kappa(x)
            ky = fd_kappa(y)
            with np.errstate(divide="ignore", invalid="ignore"):
                v = 2.0 * self.sign * np.sqrt(kx * ky) / r2 ** (1.0 + self.beta)
            return np.where(r2 > 0, v, 0.0)
        if self.name == "zero":
            return np.zeros(np.broadcast_shapes(x.shape, y.shape)[:-1])
        raise ValueError(f"unknown kernel {self.name}")


def _r2(x, y):
    r2 = None
    for d in range(x.shape[-1]):
        t = x[..., d] - y[..., d]
        t *= t
        r2 = t if r2 is None else np.add(r2, t, out=r2)
    return r2


def fd_bump(x, c, ell):
    """f(x; c, l) = exp(-1 / (1 - r^2)) for |r| < 1, r = (x - c) / (l / 2); 0 otherwise."""
    r = (np.asarray(x, dtype=np.float64) - c) / (0.5 * ell)
    inside = np.abs(r) < 1.0
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        return np.where(inside, np.exp(-1.0 / np.maximum(1e-300, 1.0 - r * r)), 0.0)


def fd_kappa(x):
    """Diffusivity kappa(x) = 1 + f(x_1; 0, 1.5) f(x_2; 0, 2.0) (reading R10);
    kappa in [1, 1 + e^-2]."""
    return 1.0 + fd_bump(x[..., 0], 0.0, 1.5) * fd_bump(x[..., 1], 0.0, 2.0)
