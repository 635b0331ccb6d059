"""Synthetic phantom sinograms for tests and benchmarks.

Closed-form line integrals of constant ellipses (reference phantom.py:67-93),
extended with in-plane rotation for the Shepp-Logan composite (SURVEY.md
8d), on the reference grids (grids.py:61-62, 85-95).  Generated with torch
directly on the device in float64 and stored as float32 [S][A][n_t] -- input
synthesis only, not part of the reconstruction path.
"""

from __future__ import annotations

import math

import torch

__all__ = ["SHEPP_LOGAN", "ellipses_sinogram", "ellipsoid_volume"]

# modified Shepp-Logan (Toft): (rho, a, b, x0, y0, phi_deg)
SHEPP_LOGAN = (
    (1.0, 0.69, 0.92, 0.0, 0.0, 0.0),
    (-0.8, 0.6624, 0.8740, 0.0, -0.0184, 0.0),
    (-0.2, 0.1100, 0.3100, 0.22, 0.0, -18.0),
    (-0.2, 0.1600, 0.4100, -0.22, 0.0, 18.0),
    (0.1, 0.2100, 0.2500, 0.0, 0.35, 0.0),
    (0.1, 0.0460, 0.0460, 0.0, 0.1, 0.0),
    (0.1, 0.0460, 0.0460, 0.0, -0.1, 0.0),
    (0.1, 0.0460, 0.0230, -0.08, -0.605, 0.0),
    (0.1, 0.0230, 0.0230, 0.0, -0.606, 0.0),
    (0.1, 0.0230, 0.0460, 0.06, -0.605, 0.0),
)


def _grids(n_t, n_angles, full_turn, device):
    t = -1.0 + 2.0 * torch.arange(n_t, dtype=torch.float64, device=device) / (n_t - 1)
    span = 2.0 * math.pi if full_turn else math.pi
    th = torch.arange(n_angles, dtype=torch.float64, device=device) * (span / n_angles)
    return t, th


def ellipses_sinogram(ellipses, n_t: int, n_angles: int, full_turn: bool = False, device="cpu") -> torch.Tensor:
    """[A][n_t] float64 sinogram of a sum of rotated ellipses."""
    t, th = _grids(n_t, n_angles, full_turn, device)
    out = torch.zeros((n_angles, n_t), dtype=torch.float64, device=device)
    for rho, a, b, x0, y0, phi in ellipses:
        al = math.radians(phi)
        q2 = (a * torch.cos(th - al)) ** 2 + (b * torch.sin(th - al)) ** 2
        tp = t[None, :] - (x0 * torch.cos(th) + y0 * torch.sin(th))[:, None]
        under = torch.clamp(q2[:, None] - tp * tp, min=0.0)
        out += 2.0 * rho * a * b * torch.sqrt(under) / q2[:, None]
    return out


def ellipsoid_volume(n_slices: int, n_t: int, n_angles: int, a=0.5, b=0.4, c=0.5, center=(0.1, -0.05, 0.0),
                     rho=1.0, device="cpu", out: torch.Tensor | None = None, chunk: int = 64,
                     slices: tuple[int, int] | None = None) -> torch.Tensor:
    """float32 [S][A][n_t] sinogram volume of one off-centre ellipsoid sliced
    at s_k = -1 + 2(k + 1/2)/S (cli.py:156; phantom.py:44-50, 67-93).
    ``slices=(b, e)`` generates only the slab k in [b, e)."""
    first, last = slices if slices is not None else (0, n_slices)
    if out is None:
        out = torch.empty((last - first, n_angles, n_t), dtype=torch.float32, device=device)
    t, th = _grids(n_t, n_angles, False, out.device)
    cos_t, sin_t = torch.cos(th), torch.sin(th)
    shift = (center[0] * cos_t + center[1] * sin_t)[:, None]
    tp2 = (t[None, :] - shift) ** 2
    for k0 in range(first, last, chunk):
        k1 = min(last, k0 + chunk)
        s = -1.0 + 2.0 * (torch.arange(k0, k1, dtype=torch.float64, device=out.device) + 0.5) / n_slices
        srel = (s - center[2]) / c
        scale = torch.sqrt(torch.clamp(1.0 - srel * srel, min=0.0))
        as_, bs = a * scale, b * scale
        q2 = (as_[:, None] * cos_t[None, :]) ** 2 + (bs[:, None] * sin_t[None, :]) ** 2  # [k][A]
        under = torch.clamp(q2[:, :, None] - tp2[None], min=0.0)
        val = 2.0 * rho * (as_ * bs)[:, None, None] * torch.sqrt(under) / torch.clamp(q2, min=1e-300)[:, :, None]
        val = torch.where((srel.abs() <= 1.0)[:, None, None], val, torch.zeros_like(val))
        out[k0 - first:k1 - first].copy_(val.to(torch.float32))
    return out
