"""``tomoblocks.preprocess``-compatible preprocessing on the B200 path.

``FlatDarkFrames`` / ``normalize`` (preprocess.py:31-74), ``CenteringResult``
/ ``CenteringError`` / ``estimate_center`` / ``apply_center``
(:27-28, :47-56, :88-138) and ``suppress_rings`` (:141-154) keep the
reference's names, validation messages and float64 containers; the
arithmetic runs in sm_100a kernels (tb_normalize, tb_center_estimate /
tb_center_apply and tb_rings; fp64 arithmetic for centering and rings like
the reference, fp32 fast log for normalisation).  ``preprocess_volume``
chains them over a device-resident volume (the pipeline's normalize ->
center -> rings stages, pipeline.py:447-484).  For reconstruction of raw
counts without centering / rings, ``fourier_bp.fbp_volume(counts,
frames=...)`` fuses the normalisation into the radial kernel's load
(tb_fbp_counts).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

__all__ = ["FlatDarkFrames", "normalize", "CenteringError", "CenteringResult", "estimate_center", "apply_center",
           "suppress_rings", "preprocess_volume"]

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
    nat = F.aux_plan(n_t, a, device=dev)
    c = torch.from_numpy(counts.astype(np.float32)).to(f"cuda:{dev}")
    flat, dark = F._frames_on(frames, dev, a, n_t)
    out = torch.empty_like(c)
    with torch.cuda.device(dev):
        nat.normalize(c, flat, dark, eps, out, 1)
    return out.cpu().numpy().astype(np.float64)


class CenteringError(ValueError):
    """Raised when the rotation center cannot be determined."""


@dataclass(frozen=True)
class CenteringResult:
    """Estimated detector-axis shift in bins, plus the match confidence."""

    beta: float
    confidence: float

    def __post_init__(self):
        if not np.isfinite(self.beta):
            raise ValueError("non-finite center estimate")


def _on_device(data, dev: int) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(data, dtype=np.float32)).to(f"cuda:{dev}")


def _raise_centering(status: int, beta: float) -> None:
    if status == 1:
        raise CenteringError("centering undetermined: constant sinogram")
    if status == 2:
        raise CenteringError(f"implausible center shift of {beta:.1f} bins")


def estimate_center(y, device=None) -> CenteringResult:
    """Rotation-centre shift from mirror consistency (preprocess.py:88-118),
    on the GPU (fp64 cross-correlation)."""
    from . import fourier_bp as F
    if y.n_angles < 2:
        raise CenteringError("need at least two projection angles")
    dev = F._device_index(device)
    nat = F.aux_plan(y.n_t, y.n_angles, device=dev)
    with torch.cuda.device(dev):
        bc, st = nat.center_estimate(_on_device(y.data, dev)[None], 1)
    beta, conf = (float(v) for v in bc[0].cpu())
    _raise_centering(int(st[0].item()), beta)
    return CenteringResult(beta=beta, confidence=conf)


def apply_center(y, beta: float, device=None):
    """Undo a detector shift of ``beta`` bins by linear interpolation
    (preprocess.py:121-138), on the GPU."""
    from . import fourier_bp as F
    from .slices import Sinogram
    if abs(beta) > y.n_t:
        raise ValueError(f"shift of {beta} bins exceeds the detector extent")
    dev = F._device_index(device)
    nat = F.aux_plan(y.n_t, y.n_angles, device=dev)
    x = _on_device(y.data, dev)[None]
    out = torch.empty_like(x)
    bc = torch.tensor([[float(beta), 0.0]], dtype=torch.float64, device=f"cuda:{dev}")
    with torch.cuda.device(dev):
        nat.center_apply(x, bc, out, 1)
    return Sinogram(y.detector, y.angles, out[0].cpu().numpy().astype(np.float64))


def suppress_rings(y, window: int = 9, device=None):
    """Remove angle-constant detector stripes (preprocess.py:141-154), on the GPU."""
    from . import fourier_bp as F
    from .slices import Sinogram
    if window < 3 or window % 2 == 0:
        raise ValueError(f"window must be an odd integer >= 3, got {window}")
    dev = F._device_index(device)
    nat = F.aux_plan(y.n_t, y.n_angles, device=dev)
    x = _on_device(y.data, dev)[None]
    out = torch.empty_like(x)
    with torch.cuda.device(dev):
        nat.rings(x, out, window, 1)
    return Sinogram(y.detector, y.angles, out[0].cpu().numpy().astype(np.float64))


def center_beta(sino: torch.Tensor, S: int, A: int, n_t: int, full_turn: bool, center) -> torch.Tensor:
    """Per-slice (beta, confidence) [S][2] float64 device tensor for the
    centre stage: "auto" estimates every slice (estimate_center,
    preprocess.py:88-116; CenteringError as the reference raises it), a
    number is that beta for every slice (apply_center's range check)."""
    from . import fourier_bp as F
    if isinstance(center, str):
        if center != "auto":
            raise ValueError(f"unknown center mode {center!r}")
        nat = F.aux_plan(n_t, A, full_turn, device=sino.device.index)
        bc, st = nat.center_estimate(sino, S)
        bad = torch.nonzero(st).flatten()
        if bad.numel():
            k = int(bad[0].item())
            _raise_centering(int(st[k].item()), float(bc[k, 0].item()))
        return bc
    if abs(float(center)) > n_t:
        raise ValueError(f"shift of {center} bins exceeds the detector extent")
    bc = torch.zeros((S, 2), dtype=torch.float64, device=sino.device)
    bc[:, 0] = float(center)
    return bc


def preprocess_volume(sino: torch.Tensor, plan, full_turn: bool = False, frames=None, eps: float = 1e-6,
                      center=None, rings: int | None = None) -> torch.Tensor:
    """normalize -> center -> rings over a device-resident volume [S][A][n_t]
    (pipeline.py:447-484), each a device pass; returns a new tensor.
    ``center``: None, "auto" (estimate per slice) or a fixed beta."""
    from . import fourier_bp as F
    S, A, n_t = sino.shape
    dev = sino.device.index
    nat = F.aux_plan(n_t, A, full_turn, device=dev)
    x = sino
    with torch.cuda.device(dev):
        if frames is not None:
            if not eps > 0:
                raise ValueError("eps must be positive")
            flat, dark = F._frames_on(frames, dev, A, n_t)
            y = torch.empty_like(x)
            nat.normalize(x, flat, dark, eps, y, S)
            x = y
        if center is not None:
            bc = center_beta(x, S, A, n_t, full_turn, center)
            y = torch.empty_like(x)
            nat.center_apply(x, bc, y, S)
            x = y
        if rings is not None:
            if rings < 3 or rings % 2 == 0:
                raise ValueError(f"window must be an odd integer >= 3, got {rings}")
            y = torch.empty_like(x)
            nat.rings(x, y, rings, S)
            x = y
    return x
