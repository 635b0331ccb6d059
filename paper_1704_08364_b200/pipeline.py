"""Pipeline stages for the reference's staged runtime (plugin contract).

The reference pipeline (pkg/src/tomoblocks/pipeline.py) calls
``spec.process(payload)`` (pipeline.py:275) on a ``VolumeBlock`` of Q
``Sinogram`` slices and expects a ``VolumeBlock`` back (pipeline.py:395-400).
The factories here build StageSpec-compatible stages whose ``process`` runs
a whole Q-block in one batched GPU call, with the ramp filter fused into the
backprojection (filter + backproject stages of pipeline.py:486-518 in one).
``StageSpec`` mirrors pipeline.py:48-67 so the stages plug into either
runtime; the generic thread/queue runtime itself is the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Callable

import numpy as np
import torch

from .fourier_bp import BstPlan, FilterPlan, FBP_SCALE, _device_index, aux_plan, fbp_volume
from .slices import ImageGrid, Sinogram, StageKind, VolumeBlock

__all__ = ["StageSpec", "block_descriptors", "make_fbp_stage", "make_backproject_stage", "make_filter_stage"]


@dataclass(frozen=True)
class StageSpec:
    """Stage descriptor with the reference's fields and checks (pipeline.py:48-67)."""

    name: str
    workers: int
    queue_capacity: int
    process: Callable[[Any], Any]
    workset_multiplier: float = 2.0

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError(f"stage {self.name!r}: workers must be >= 1")
        if self.queue_capacity < 1:
            raise ValueError(f"stage {self.name!r}: queue_capacity must be >= 1")


def block_descriptors(n_slices: int, q: int) -> list[tuple[int, int]]:
    """(first_slice, count) Q-blocks covering the volume (pipeline.py:552-554)."""
    return [(s, min(q, n_slices - s)) for s in range(0, n_slices, q)]


def _stack(block: VolumeBlock, dev: int) -> tuple[torch.Tensor, bool]:
    sl = block.slices
    full = sl[0].angles.full_turn
    arr = np.stack([np.asarray(s.data, dtype=np.float32) for s in sl])
    return torch.from_numpy(arr).to(f"cuda:{dev}"), full


def _images(vol: torch.Tensor, n: int) -> list[ImageGrid]:
    host = vol.cpu().numpy().astype(np.float64)
    return [ImageGrid(n, host[i]) for i in range(host.shape[0])]


def make_fbp_stage(plan: BstPlan, fplan: FilterPlan = FilterPlan(), kernel: str = "bst", workers: int = 1,
                   queue_capacity: int = 4, device=None, frames=None, eps: float = 1e-6, center=None,
                   rings: int | None = None) -> StageSpec:
    """Fused filter + backproject stage: Sinogram block -> ImageGrid block x 1/(2 pi)
    (pipeline.py:489-518 with cfg.kernel).  With ``frames`` (a
    preprocess.FlatDarkFrames) the blocks hold raw counts and the reference's
    normalize stage (pipeline.py:447-459) runs fused into the same launch.
    ``center`` ("auto": estimate_center per slice; a number: cfg.center_beta)
    and ``rings`` (cfg.ring_window) take over the center and rings stages
    (pipeline.py:461-484) as well: for kernel "bst" without frames they are
    applied on the radial kernel's row load."""
    if kernel not in ("ss", "bst"):
        raise ValueError(f"unknown kernel {kernel!r}")
    dev = _device_index(device)

    def process(block: VolumeBlock) -> VolumeBlock:
        vol, full = _stack(block, dev)
        out = fbp_volume(vol, plan, fplan, kernel=kernel, full_turn=full, frames=frames, eps=eps, center=center,
                         rings=rings)
        return VolumeBlock(block.first_slice, _images(out, plan.output_n), StageKind.BACKPROJECT)

    return StageSpec("backproject", workers, queue_capacity, process, 2.0)


def make_backproject_stage(plan: BstPlan, workers: int = 1, queue_capacity: int = 4, device=None,
                           scale: float = FBP_SCALE) -> StageSpec:
    """Backproject stage for already-filtered blocks (pipeline.py:511-518):
    bst_backproject x FBP_SCALE per slice."""
    dev = _device_index(device)

    def process(block: VolumeBlock) -> VolumeBlock:
        vol, full = _stack(block, dev)
        # the scale rides in K3's epilogue (tb_bst_scaled): no extra pass
        out = fbp_volume(vol, plan, FilterPlan(), kernel="none", full_turn=full, scale=scale)
        return VolumeBlock(block.first_slice, _images(out, plan.output_n), StageKind.BACKPROJECT)

    return StageSpec("backproject", workers, queue_capacity, process, 2.0)


def make_filter_stage(fplan: FilterPlan = FilterPlan(), workers: int = 1, queue_capacity: int = 4,
                      device=None) -> StageSpec:
    """Ramp-filter stage (pipeline.py:489-492) on the GPU."""
    dev = _device_index(device)

    def process(block: VolumeBlock) -> VolumeBlock:
        vol, full = _stack(block, dev)
        s0 = block.slices[0]
        nat = aux_plan(s0.n_t, s0.n_angles, fplan=fplan, device=dev)
        out = torch.empty_like(vol)
        with torch.cuda.device(dev):
            nat.ramp(vol, out, vol.shape[0])
        host = out.cpu().numpy().astype(np.float64)
        return VolumeBlock(block.first_slice,
                           [Sinogram(s.detector, s.angles, host[i]) for i, s in enumerate(block.slices)],
                           StageKind.FILTER)

    return StageSpec("filter", workers, queue_capacity, process, 2.0)
