"""Forward projector and slant-stack (brute-force, O(V N^2) per slice)
backprojector on B200, mirroring reference projector.py.

``backproject_ss`` (projector.py:126-158): linear interpolation along t at
u . xi_j, zero contribution where the sample falls outside [-1, 1] (with the
reference's clip rule for the last bin), weight span / V.  It is the config-5
comparator of the BST kernel and the "ss" kernel of ``fbp``; kernel K5
(tb_ss).  ``forward_project`` (projector.py:94-123): midpoint-rule line
integrals of the image along each (theta, t) ray; kernel K6 (tb_forward).
The two are an adjoint pair under ``inner_product_image`` /
``inner_product_sino`` (projector.py:161-172).  No CPU path.
"""

from __future__ import annotations

import numpy as np
import torch

from .fourier_bp import FilterPlan, _device_index, aux_plan
from dataclasses import dataclass

from .slices import AngleAxis, DetectorAxis, ImageGrid, Sinogram

__all__ = ["RayTraceConfig", "forward_project", "backproject_ss", "inner_product_image", "inner_product_sino"]


@dataclass(frozen=True)
class RayTraceConfig:
    """Sampling step (as a fraction of pixel size) and interpolation mode
    (projector.py:36-47)."""

    step_length: float = 0.5
    interpolation: str = "bilinear"

    def __post_init__(self):
        if not 0.0 < self.step_length <= 1.0:
            raise ValueError(f"step_length must be in (0, 1], got {self.step_length}")
        if self.interpolation not in ("bilinear", "nearest"):
            raise ValueError(f"unknown interpolation {self.interpolation!r}")


def _ss_plan(y: Sinogram, n: int, device=None):
    """Table-free device plan carrying the slant-stack geometry: the
    detector axis, the angle span and count (any count, odd full turns
    included, like projector.py:126-158) and the n x n output grid."""
    return aux_plan(y.n_t, y.n_angles, y.angles.full_turn, n, FilterPlan(), device)


def backproject_ss(y: Sinogram, n: int, workers: int = 1, device=None) -> ImageGrid:
    """Slant-stack backprojection onto an n x n grid (projector.py:126-158)."""
    dev = _device_index(device)
    nat = _ss_plan(y, n, dev)
    rows = torch.from_numpy(np.ascontiguousarray(y.data, dtype=np.float32)).to(f"cuda:{dev}")
    img = torch.empty((n, n), dtype=torch.float32, device=f"cuda:{dev}")
    with torch.cuda.device(dev):
        nat.slant_stack(rows, img, 1, 1.0)
    out = img.cpu().numpy().astype(np.float64)
    if not np.isfinite(out).all():
        raise FloatingPointError("non-finite values in backprojection output")
    return ImageGrid(n, out)


def forward_project(image: ImageGrid, detector: DetectorAxis, angles: AngleAxis,
                    cfg: RayTraceConfig = RayTraceConfig(), workers: int = 1, device=None) -> Sinogram:
    """Line integrals of ``image`` on the (t, theta) grid (projector.py:94-123);
    ``workers`` is accepted and ignored."""
    y0 = Sinogram(detector, angles, np.zeros((angles.n_theta, detector.n_t)))
    dev = _device_index(device)
    nat = _ss_plan(y0, image.n, dev)
    img = torch.from_numpy(np.ascontiguousarray(image.data, dtype=np.float32)).to(f"cuda:{dev}")
    out = torch.empty((angles.n_theta, detector.n_t), dtype=torch.float32, device=f"cuda:{dev}")
    with torch.cuda.device(dev):
        nat.forward(img, out, 1, cfg.step_length, cfg.interpolation == "nearest")
    return Sinogram(detector, angles, out.cpu().numpy().astype(np.float64))


def inner_product_image(a: ImageGrid, b: ImageGrid) -> float:
    """Discrete L2 inner product weighted by pixel area (projector.py:161-165)."""
    if a.n != b.n:
        raise ValueError(f"image shapes differ: {a.n} vs {b.n}")
    return float(np.sum(a.data * b.data)) * a.pixel_size ** 2


def inner_product_sino(y: Sinogram, z: Sinogram) -> float:
    """Discrete L2 inner product weighted by the (t, theta) cell measure
    (projector.py:168-172)."""
    if y.data.shape != z.data.shape:
        raise ValueError(f"sinogram shapes differ: {y.data.shape} vs {z.data.shape}")
    return float(np.sum(y.data * z.data)) * y.detector.spacing * y.angles.spacing
