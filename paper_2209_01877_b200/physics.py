"""Gas model, state containers and initial flows (host side).

Mirrors `hodg/physics.py:59-145` (AdmissibilityError, GasModel, Conserved,
Primitive) and `hodg/flows.py:23-74` with a third velocity component.  The
point physics itself (Roe / LLF flux, boundary states) lives in the CUDA
kernels (csrc/hodg_common.cuh).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "AdmissibilityError",
    "GasModel",
    "Conserved",
    "Primitive",
    "freestream_primitive",
    "freestream_conserved",
    "vortex_primitive",
    "vortex_density",
    "pulse_primitive",
]


class AdmissibilityError(Exception):
    """A state with non-positive density or pressure (hodg/physics.py:59-73)."""

    def __init__(self, message, cell=None, face=None, iteration=None):
        parts = [message]
        if cell is not None:
            parts.append(f"cell {cell}")
        if face is not None:
            parts.append(f"face {face}")
        if iteration is not None:
            parts.append(f"iteration {iteration}")
        super().__init__(", ".join(parts))
        self.cell = cell
        self.face = face
        self.iteration = iteration


@dataclass(frozen=True)
class GasModel:
    """Calorically perfect gas (hodg/physics.py:76-104).  The B200 path is
    the Euler residual: ivis must be 0 (the BR1 viscous terms are the next
    row of SURVEY.md §8(f))."""

    gamma: float = 1.4
    R: float = 1.0
    mu_dyn: float = 0.0
    Pr: float = 0.72
    ivis: int = 0

    def __post_init__(self):
        if not self.gamma > 1.0:
            raise ValueError("gamma must exceed 1")
        if self.R <= 0.0:
            raise ValueError("gas constant must be positive")
        if self.mu_dyn < 0.0:
            raise ValueError("viscosity must be non-negative")
        if self.Pr <= 0.0:
            raise ValueError("Prandtl number must be positive")
        if self.ivis not in (0, 1):
            raise ValueError("ivis must be 0 or 1")


@dataclass(frozen=True)
class Conserved:
    rho: float
    rho_u: float
    rho_v: float
    rho_w: float
    e: float

    def as_array(self) -> np.ndarray:
        return np.array([self.rho, self.rho_u, self.rho_v, self.rho_w, self.e])


@dataclass(frozen=True)
class Primitive:
    rho: object
    u: object
    v: object
    w: object
    p: object


def freestream_primitive(gas: GasModel, mach: float, angle_deg: float = 0.0) -> Primitive:
    """rho = T = 1, p = R, velocity Mach * a in the x-y plane (hodg/flows.py:23-29)."""
    a = np.sqrt(gas.gamma * gas.R)
    ang = np.deg2rad(angle_deg)
    return Primitive(1.0, mach * a * np.cos(ang), mach * a * np.sin(ang), 0.0, gas.R)


def freestream_conserved(gas: GasModel, mach: float, angle_deg: float = 0.0) -> Conserved:
    w = freestream_primitive(gas, mach, angle_deg)
    e = w.p / (gas.gamma - 1.0) + 0.5 * w.rho * (w.u * w.u + w.v * w.v + w.w * w.w)
    return Conserved(w.rho, w.rho * w.u, w.rho * w.v, w.rho * w.w, e)


def vortex_primitive(gas, mach, angle_deg, beta, x0, y0, t, x, y, z=None) -> Primitive:
    """Isentropic vortex (hodg/flows.py:38-53) extruded along z: an exact
    Euler solution advecting with the freestream (w = 0)."""
    fs = freestream_primitive(gas, mach, angle_deg)
    xr = np.asarray(x, dtype=np.float64) - x0 - fs.u * t
    yr = np.asarray(y, dtype=np.float64) - y0 - fs.v * t
    r2 = xr * xr + yr * yr
    g = gas.gamma
    env = np.exp(0.5 * (1.0 - r2))
    vs = np.sqrt(gas.R)
    u = fs.u - beta / (2.0 * np.pi) * yr * env * vs
    v = fs.v + beta / (2.0 * np.pi) * xr * env * vs
    T = 1.0 - (g - 1.0) * beta * beta / (8.0 * g * np.pi * np.pi) * np.exp(1.0 - r2)
    rho = T ** (1.0 / (g - 1.0))
    return Primitive(rho, u, v, np.zeros_like(u), rho * gas.R * T)


def vortex_density(gas, mach, angle_deg, beta, x0, y0, t, x, y, z=None):
    return np.asarray(vortex_primitive(gas, mach, angle_deg, beta, x0, y0, t, x, y).rho)


def pulse_primitive(gas, amplitude, sigma, x0, y0, z0, x, y, z, mach=0.0, angle_deg=0.0) -> Primitive:
    """Isentropic Gaussian pressure pulse on the freestream (hodg/flows.py:60-74)."""
    r2 = (np.asarray(x) - x0) ** 2 + (np.asarray(y) - y0) ** 2 + (np.asarray(z) - z0) ** 2
    p = gas.R * (1.0 + amplitude * np.exp(-0.5 * r2 / (sigma * sigma)))
    rho = (p / gas.R) ** (1.0 / gas.gamma)
    fs = freestream_primitive(gas, mach, angle_deg) if mach > 0.0 else Primitive(1.0, 0.0, 0.0, 0.0, gas.R)
    return Primitive(rho, np.full_like(p, fs.u), np.full_like(p, fs.v), np.zeros_like(p), p)
