"""``tomoblocks.preprocess``-compatible normalisation on the B200 path.

``FlatDarkFrames`` and ``normalize`` keep the reference's names, validation
messages and float64 return type (preprocess.py:31-74); the arithmetic runs in
the sm_100a kernel ``tb_normalize`` (float32, fast natural log).  For
reconstruction, pass the frames to ``fourier_bp.fbp_volume(counts,
frames=...)``: the normalisation is then fused into the radial kernel's load
(tb_fbp_counts) instead of being a separate pass over the volume.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

__all__ = ["FlatDarkFrames", "normalize"]

_PLANS: dict = {}  # (n_angles, n_t) -> BstPlan carrying the device plan for tb_normalize


@dataclass(frozen=True)
class FlatDarkFrames:
    """Flat (no sample) and dark (no beam) detector frames."""

    flat: np.ndarray
    dark: np.ndarray

    def __post_init__(self):
        flat = np.asarray(self.flat, dtype=float)
        dark = np.asarray(self.dark, dtype=float)
        if flat.shape != dark.shape:
            raise ValueError(f"flat/dark shapes differ: {flat.shape} vs {dark.shape}")
        object.__setattr__(self, "flat", flat)
        object.__setattr__(self, "dark", dark)


def normalize(counts: np.ndarray, frames: FlatDarkFrames, eps: float = 1e-6, device=None) -> np.ndarray:
    """Transmission counts to line integrals: -log((I - D) / (I0 - D)), both
    differences clamped at ``eps`` (preprocess.py:59-74), on the GPU."""
    from . import fourier_bp as F
    if eps <= 0:
        raise ValueError("eps must be positive")
    counts = np.asarray(counts, dtype=float)
    if counts.shape != frames.flat.shape:
        raise ValueError(f"counts shape {counts.shape} does not match frames {frames.flat.shape}")
    if counts.ndim != 2:
        raise ValueError("counts must be a [n_angles][n_t] frame")
    a, n_t = counts.shape
    dev = F._device_index(device)
    plan = _PLANS.setdefault((a, n_t), F.BstPlan(n_t=max(n_t, 2), n_theta=max(a, 1)))
    nat = F.native_plan(plan, F.FilterPlan(), False, dev)
    c = torch.from_numpy(counts.astype(np.float32)).to(f"cuda:{dev}")
    flat, dark = F._frames_on(frames, dev, a, n_t)
    out = torch.empty_like(c)
    with torch.cuda.device(dev):
        nat.normalize(c, flat, dark, eps, out, 1)
    return out.cpu().numpy().astype(np.float64)
