"""Slant-stack (brute-force, O(V N^2) per slice) backprojection on B200.

``backproject_ss`` mirrors reference projector.py:126-158: linear
interpolation along t at u . xi_j, zero contribution where the sample falls
outside [-1, 1] (with the reference's clip rule for the last bin), weight
span / V.  It is the config-5 comparator of the BST kernel and the "ss"
kernel of ``fbp``.  Runs kernel K5 (tb_ss); no CPU path.
"""

from __future__ import annotations

import numpy as np
import torch

from .fourier_bp import BstPlan, FilterPlan, _device_index, native_plan
from .slices import ImageGrid, Sinogram

__all__ = ["backproject_ss"]


def _next_pow2(n: int) -> int:
    m = 1
    while m < n:
        m <<= 1
    return m


def _ss_plan(y: Sinogram, n: int) -> BstPlan:
    """A device plan carrying the slant-stack geometry: the detector axis, the
    angle span (half or full turn) and the n x n output grid."""
    if y.angles.full_turn and y.n_angles % 2:
        raise NotImplementedError("full-turn input with an odd angle count is not supported on the GPU path")
    n_theta = y.n_angles // 2 if y.angles.full_turn else y.n_angles
    L = max(_next_pow2(2 * y.n_t), _next_pow2(n))
    return BstPlan(n_t=y.n_t, n_theta=n_theta, radial_samples=L, output_n=n)


def backproject_ss(y: Sinogram, n: int, workers: int = 1, device=None) -> ImageGrid:
    """Slant-stack backprojection onto an n x n grid (projector.py:126-158)."""
    plan = _ss_plan(y, n)
    dev = _device_index(device)
    nat = native_plan(plan, FilterPlan(), y.angles.full_turn, dev)
    rows = torch.from_numpy(np.ascontiguousarray(y.data, dtype=np.float32)).to(f"cuda:{dev}")
    img = torch.empty((n, n), dtype=torch.float32, device=f"cuda:{dev}")
    with torch.cuda.device(dev):
        nat.slant_stack(rows, img, 1, 1.0)
    out = img.cpu().numpy().astype(np.float64)
    if not np.isfinite(out).all():
        raise FloatingPointError("non-finite values in backprojection output")
    return ImageGrid(n, out)
