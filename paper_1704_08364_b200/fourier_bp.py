"""BST filtered backprojection on B200 -- the reference's operator API.

Drop-in for ``tomoblocks.fourier_bp`` (reference pkg/src/tomoblocks/fourier_bp.py):

  ``BstPlan``, ``FilterPlan``   same fields, defaults and validation (:69-267)
  ``ramp_filter``               (:490-505)  -> tb_ramp
  ``bst_backproject``           (:435-461)  -> tb_bst  (K1 -> K1b -> K2 -> K3)
  ``fbp``                       (:508-530)  -> tb_fbp  / tb_fbp_ss
  ``FBP_SCALE``                 (:59)

plus the batched sinogram-volume call ``fbp_volume`` (device-resident or
host-pinned input, slab-sharded over devices).

Every call runs the hand-written sm_100a kernels of ``lib/libtb_bst.so``
through the C ABI in ``include/tb_bst.h``; there is no CPU path.  Inputs are
converted to float32 on the device; single-slice results come back as
float64 ``ImageGrid`` / ``Sinogram`` exactly like the reference's.
``workers`` is accepted for signature compatibility and ignored (the CUDA
grid replaces the thread pool, reference _parallel.py).
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .slices import AngleAxis, DetectorAxis, ImageGrid, Sinogram

__all__ = [
    "FBP_SCALE",
    "BstPlan",
    "FilterPlan",
    "ramp_filter",
    "bst_backproject",
    "fbp",
    "fbp_volume",
    "NativePlan",
]

FBP_SCALE = 1.0 / (2.0 * math.pi)


def _next_pow2(n: int) -> int:
    m = 1
    while m < n:
        m <<= 1
    return m


@dataclass(frozen=True)
class BstPlan:
    """Geometry, padding and window choices (fourier_bp.py:69-111)."""

    n_t: int
    n_theta: int
    pad_factor: int = 2
    radial_samples: int | None = None
    kb_beta: float = 10.0
    kb_support: float = 0.1
    sigma_min_bins: int = 1
    interp: str = "bilinear"
    output_n: int | None = None
    _cache: dict = field(default_factory=dict, repr=False, compare=False, init=False)

    def __post_init__(self):
        if self.n_t < 2 or self.n_theta < 1:
            raise ValueError("need n_t >= 2 and n_theta >= 1")
        if self.pad_factor < 2:
            raise ValueError(f"pad_factor must be >= 2, got {self.pad_factor}")
        if self.sigma_min_bins < 1:
            raise ValueError(f"sigma_min_bins must be >= 1, got {self.sigma_min_bins}")
        if self.interp not in ("bilinear", "nearest"):
            raise ValueError(f"unknown interp mode {self.interp!r}")
        L = self.radial_samples
        if L is None:
            L = _next_pow2(self.pad_factor * self.n_t)
            object.__setattr__(self, "radial_samples", L)
        if L & (L - 1) or L < self.pad_factor * self.n_t:
            raise ValueError(f"radial_samples must be a power of two >= pad_factor * n_t, got {L}")
        if self.output_n is None:
            object.__setattr__(self, "output_n", self.n_t)
        if not 1 <= self.output_n <= L:
            raise ValueError("output_n must be in [1, radial_samples]")
        object.__setattr__(self, "_lock", threading.RLock())

    @classmethod
    def for_sinogram(cls, y: Sinogram, **overrides) -> "BstPlan":
        # reference quirk kept: full-turn input is not halved (fourier_bp.py:113-115)
        return cls(n_t=y.n_t, n_theta=y.n_angles, **overrides)

    # derived geometry (fourier_bp.py:119-152)
    @property
    def delta_t(self) -> float:
        return 2.0 / (self.n_t - 1)

    @property
    def delta_f(self) -> float:
        return 1.0 / (self.radial_samples * self.delta_t)

    @property
    def sigma_min(self) -> float:
        return self.sigma_min_bins * self.delta_f

    @property
    def roll(self) -> int:
        return int(round((self.n_t - 1) / 2.0))

    @property
    def delta_u(self) -> float:
        return 2.0 / self.output_n

    @property
    def delta_nu(self) -> float:
        return 1.0 / (self.radial_samples * self.delta_u)

    @property
    def amplitude_scale(self) -> float:
        return (self.delta_nu * self.radial_samples) ** 2 * self.delta_t

    def _cached(self, key, builder):
        hit = self._cache.get(key)
        if hit is None:
            with self._lock:
                hit = self._cache.get(key)
                if hit is None:
                    hit = builder()
                    self._cache[key] = hit
        return hit


@dataclass(frozen=True)
class FilterPlan:
    """Ramp configuration; rolloff = 1 disables the taper (fourier_bp.py:252-267)."""

    kind: str = "ramp"
    rolloff: float = 1.0

    def __post_init__(self):
        if self.kind not in ("ramp", "ramp_apodized"):
            raise ValueError(f"unknown filter kind {self.kind!r}")
        if not 0.0 < self.rolloff <= 1.0:
            raise ValueError(f"rolloff must be in (0, 1], got {self.rolloff}")

    @property
    def effective_rolloff(self) -> float:
        return self.rolloff if self.kind == "ramp_apodized" else 1.0


# ---------------------------------------------------------------------------
# native plan handle
# ---------------------------------------------------------------------------


class NativePlan:
    """Owns one ``tb_plan`` (device constants for a BstPlan x FilterPlan x
    angle span on one device).  Immutable; safe to share across threads."""

    def __init__(self, plan: BstPlan, fplan: FilterPlan, full_turn: bool, device: int,
                 n_angles: int | None = None, grid: bool = True):
        lib = _native.lib()
        d = _native.tb_plan_desc()
        d.n_t = plan.n_t
        d.n_theta = plan.n_theta
        d.pad_factor = plan.pad_factor
        d.radial_samples = plan.radial_samples
        d.kb_beta = plan.kb_beta
        d.kb_support = plan.kb_support
        d.sigma_min_bins = plan.sigma_min_bins
        d.interp = 0 if plan.interp == "bilinear" else 1
        d.output_n = plan.output_n
        d.full_turn = 1 if full_turn else 0
        d.filter_kind = 1 if fplan.kind == "ramp_apodized" else 0
        d.rolloff = fplan.rolloff
        d.n_angles = 0 if n_angles is None else int(n_angles)
        d.flags = 0 if grid else _native.TB_PLAN_NO_GRID
        h = ctypes.c_void_p()
        _native.check(lib.tb_plan_create(ctypes.byref(d), int(device), ctypes.byref(h)), "tb_plan_create")
        self._h = h
        self._lib = lib
        self.device = int(device)
        info = _native.tb_plan_info()
        _native.check(lib.tb_plan_get_info(h, ctypes.byref(info)), "tb_plan_get_info")
        self.n_t = info.n_t
        self.n_theta = info.n_theta
        self.n_angles = info.n_angles
        self.L = info.radial_samples
        self.npad = info.ramp_samples
        self.n = info.output_n
        self.support = (info.support_lo, info.support_hi)
        self.full_turn = bool(full_turn)

    @property
    def handle(self):
        return self._h

    def workspace_bytes(self, batch: int) -> int:
        out = ctypes.c_size_t()
        _native.check(self._lib.tb_workspace_bytes(self._h, int(batch), ctypes.byref(out)), "tb_workspace_bytes")
        return int(out.value)

    def layout(self, batch: int) -> dict:
        lay = _native.tb_workspace_layout()
        _native.check(self._lib.tb_workspace_get_layout(self._h, int(batch), ctypes.byref(lay)), "layout")
        return {k: int(getattr(lay, k)) for k, _ in lay._fields_}

    def new_workspace(self, batch: int) -> torch.Tensor:
        return torch.empty(self.workspace_bytes(batch), dtype=torch.uint8, device=f"cuda:{self.device}")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.tb_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- execution (all asynchronous on `stream`) ---------------------------
    def _stream(self, stream):
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(stream.cuda_stream)

    def run(self, op: str, sino: torch.Tensor, image: torch.Tensor, n_slices: int, batch: int,
            workspace: torch.Tensor, stream=None, scale: float | None = None) -> None:
        """``scale`` (op "bst" only): multiply the backprojection in K3's
        epilogue (tb_bst_scaled) instead of a separate pass."""
        args = (self._h, ctypes.c_void_p(sino.data_ptr()), ctypes.c_void_p(image.data_ptr()), int(n_slices),
                int(batch), ctypes.c_void_p(workspace.data_ptr()), ctypes.c_size_t(workspace.numel()))
        if scale is not None and op == "bst":
            rc = self._lib.tb_bst_scaled(*args, ctypes.c_float(scale), self._stream(stream))
            _native.check(rc, "tb_bst_scaled")
            return
        if scale is not None:
            raise ValueError(f"scale applies to op 'bst' only, not {op!r}")
        fn = {"fbp": self._lib.tb_fbp, "bst": self._lib.tb_bst, "fbp_ss": self._lib.tb_fbp_ss,
              "fbp_frames": self._lib.tb_fbp_frames}[op]
        rc = fn(*args, self._stream(stream))
        _native.check(rc, f"tb_{op}")

    def run_counts(self, counts: torch.Tensor, flat: torch.Tensor, dark: torch.Tensor, eps: float,
                   image: torch.Tensor, n_slices: int, batch: int, workspace: torch.Tensor, stream=None) -> None:
        """fbp of transmission counts with the normalisation fused into K1
        (tb_fbp_counts); flat / dark are device frames [A][n_t] f32."""
        rc = self._lib.tb_fbp_counts(self._h, ctypes.c_void_p(counts.data_ptr()), ctypes.c_void_p(flat.data_ptr()),
                                     ctypes.c_void_p(dark.data_ptr()), ctypes.c_double(eps),
                                     ctypes.c_void_p(image.data_ptr()), int(n_slices), int(batch),
                                     ctypes.c_void_p(workspace.data_ptr()), ctypes.c_size_t(workspace.numel()),
                                     self._stream(stream))
        _native.check(rc, "tb_fbp_counts")

    def run_counts_const(self, counts: torch.Tensor, i0: float, dark: float, eps: float, image: torch.Tensor,
                         n_slices: int, batch: int, workspace: torch.Tensor, stream=None) -> None:
        """run_counts for constant frames (tb_fbp_counts_const: no frame loads)."""
        rc = self._lib.tb_fbp_counts_const(self._h, ctypes.c_void_p(counts.data_ptr()), ctypes.c_double(i0),
                                           ctypes.c_double(dark), ctypes.c_double(eps),
                                           ctypes.c_void_p(image.data_ptr()), int(n_slices), int(batch),
                                           ctypes.c_void_p(workspace.data_ptr()), ctypes.c_size_t(workspace.numel()),
                                           self._stream(stream))
        _native.check(rc, "tb_fbp_counts_const")

    def counts(self, counts: torch.Tensor, frames, eps: float, image: torch.Tensor, n_slices: int, batch: int,
               workspace: torch.Tensor, stream=None) -> None:
        """fbp of counts with `frames` = (flat, dark) device tensors or ("const", i0, dark)."""
        if frames[0] == "const":
            self.run_counts_const(counts, frames[1], frames[2], eps, image, n_slices, batch, workspace, stream)
        else:
            self.run_counts(counts, frames[0], frames[1], eps, image, n_slices, batch, workspace, stream)

    def normalize(self, counts: torch.Tensor, flat: torch.Tensor, dark: torch.Tensor, eps: float,
                  out: torch.Tensor, n_slices: int, stream=None) -> None:
        rc = self._lib.tb_normalize(self._h, ctypes.c_void_p(counts.data_ptr()), ctypes.c_void_p(flat.data_ptr()),
                                    ctypes.c_void_p(dark.data_ptr()), ctypes.c_double(eps),
                                    ctypes.c_void_p(out.data_ptr()), int(n_slices), self._stream(stream))
        _native.check(rc, "tb_normalize")

    def run_profiled(self, sino: torch.Tensor, image: torch.Tensor, n_slices: int, batch: int,
                     workspace: torch.Tensor, stream=None) -> dict:
        """tb_fbp with per-stage CUDA events; returns summed device ms per stage."""
        ms = (ctypes.c_double * 5)()
        rc = self._lib.tb_fbp_profiled(self._h, ctypes.c_void_p(sino.data_ptr()), ctypes.c_void_p(image.data_ptr()),
                                       int(n_slices), int(batch), ctypes.c_void_p(workspace.data_ptr()),
                                       ctypes.c_size_t(workspace.numel()), self._stream(stream), ms)
        _native.check(rc, "tb_fbp_profiled")
        return dict(zip(("ramp", "k1_radial", "k1b_common", "k2_columns", "k3_rows"), list(ms)))

    def ramp(self, sino: torch.Tensor, out: torch.Tensor, n_slices: int, stream=None) -> None:
        rc = self._lib.tb_ramp(self._h, ctypes.c_void_p(sino.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                               int(n_slices), self._stream(stream))
        _native.check(rc, "tb_ramp")

    def slant_stack(self, sino: torch.Tensor, image: torch.Tensor, n_slices: int, scale: float = 1.0,
                    stream=None) -> None:
        rc = self._lib.tb_ss(self._h, ctypes.c_void_p(sino.data_ptr()), ctypes.c_void_p(image.data_ptr()),
                             int(n_slices), ctypes.c_float(scale), self._stream(stream))
        _native.check(rc, "tb_ss")

    def forward(self, image: torch.Tensor, sino: torch.Tensor, n_slices: int, step_length: float = 0.5,
                nearest: bool = False, stream=None) -> None:
        """Forward projector (tb_forward): images [B][n][n] -> sinograms [B][A][n_t]."""
        rc = self._lib.tb_forward(self._h, ctypes.c_void_p(image.data_ptr()), ctypes.c_void_p(sino.data_ptr()),
                                  int(n_slices), ctypes.c_double(step_length), 1 if nearest else 0,
                                  self._stream(stream))
        _native.check(rc, "tb_forward")

    def center_estimate(self, sino: torch.Tensor, n_slices: int, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
        """(beta_conf [B][2] float64, status [B] int32) device tensors (tb_center_estimate)."""
        bc = torch.empty((n_slices, 2), dtype=torch.float64, device=f"cuda:{self.device}")
        st = torch.empty((n_slices,), dtype=torch.int32, device=f"cuda:{self.device}")
        rc = self._lib.tb_center_estimate(self._h, ctypes.c_void_p(sino.data_ptr()), int(n_slices),
                                          ctypes.c_void_p(bc.data_ptr()), ctypes.c_void_p(st.data_ptr()),
                                          self._stream(stream))
        _native.check(rc, "tb_center_estimate")
        return bc, st

    def center_apply(self, sino: torch.Tensor, beta_conf: torch.Tensor, out: torch.Tensor, n_slices: int,
                     stream=None) -> None:
        rc = self._lib.tb_center_apply(self._h, ctypes.c_void_p(sino.data_ptr()), ctypes.c_void_p(beta_conf.data_ptr()),
                                       ctypes.c_void_p(out.data_ptr()), int(n_slices), self._stream(stream))
        _native.check(rc, "tb_center_apply")

    def rings(self, sino: torch.Tensor, out: torch.Tensor, window: int, n_slices: int, stream=None) -> None:
        scratch = torch.empty((max(n_slices, 1), self.n_t), dtype=torch.float64, device=f"cuda:{self.device}")
        rc = self._lib.tb_rings(self._h, ctypes.c_void_p(sino.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                int(window), ctypes.c_void_p(scratch.data_ptr()), int(n_slices), self._stream(stream))
        _native.check(rc, "tb_rings")

    def pre_params(self, sino: torch.Tensor, n_slices: int, beta_conf: torch.Tensor | None, window: int,
                   stream=None) -> tuple[torch.Tensor, torch.Tensor | None]:
        """Fused centre / ring stage parameters (tb_pre_params): shift [S][2]
        f32 (floor(beta), frac(beta)) and, with window > 0, the stripe
        profile [S][n_t] f32 of the centred sinogram."""
        dev = f"cuda:{self.device}"
        shift = torch.empty((max(n_slices, 1), 2), dtype=torch.float32, device=dev)
        stripe = torch.empty((max(n_slices, 1), self.n_t), dtype=torch.float32, device=dev) if window else None
        scratch = torch.empty((max(n_slices, 1), self.n_t), dtype=torch.float64, device=dev) if window else None
        rc = self._lib.tb_pre_params(self._h, ctypes.c_void_p(sino.data_ptr()), int(n_slices),
                                     ctypes.c_void_p(beta_conf.data_ptr() if beta_conf is not None else None),
                                     int(window), ctypes.c_void_p(scratch.data_ptr() if window else None),
                                     ctypes.c_void_p(shift.data_ptr()),
                                     ctypes.c_void_p(stripe.data_ptr() if window else None), self._stream(stream))
        _native.check(rc, "tb_pre_params")
        return shift, stripe

    def run_pre(self, sino: torch.Tensor, image: torch.Tensor, n_slices: int, batch: int, workspace: torch.Tensor,
                shift: torch.Tensor, stripe: torch.Tensor | None, stream=None) -> None:
        """tb_fbp with the centre / ring stages applied on K1's load (tb_fbp_pre)."""
        rc = self._lib.tb_fbp_pre(self._h, ctypes.c_void_p(sino.data_ptr()), ctypes.c_void_p(image.data_ptr()),
                                  int(n_slices), int(batch), ctypes.c_void_p(workspace.data_ptr()),
                                  ctypes.c_size_t(workspace.numel()), ctypes.c_void_p(shift.data_ptr()),
                                  ctypes.c_void_p(stripe.data_ptr() if stripe is not None else None),
                                  self._stream(stream))
        _native.check(rc, "tb_fbp_pre")

    def polar(self, workspace: torch.Tensor, batch: int, stream=None) -> torch.Tensor:
        """K1 output of the last launch group (first lane) on this workspace:
        [batch][rows][L/2] complex64 (tb_copy_polar)."""
        rows = self.n_angles + 1  # + the angle-pi (half turn) / angle-2 pi (full turn) copy of row 0
        out = torch.empty((batch, rows, self.L // 2), dtype=torch.complex64, device=f"cuda:{self.device}")
        _native.check(self._lib.tb_copy_polar(self._h, ctypes.c_void_p(workspace.data_ptr()), int(batch),
                                              ctypes.c_void_p(out.data_ptr()), self._stream(stream)), "tb_copy_polar")
        return out

    def reset_status(self, workspace: torch.Tensor, stream=None) -> None:
        _native.check(self._lib.tb_reset_status(self._h, ctypes.c_void_p(workspace.data_ptr()),
                                                self._stream(stream)), "tb_reset_status")

    def read_status(self, workspace: torch.Tensor, stream=None) -> None:
        """Synchronise and raise ValueError (non-finite input) or
        FloatingPointError (non-finite output, fourier_bp.py:459-460)."""
        _native.check(self._lib.tb_read_status(self._h, ctypes.c_void_p(workspace.data_ptr()),
                                               self._stream(stream)), "tb_read_status")


def _device_index(device=None) -> int:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
        return torch.cuda.current_device()
    if isinstance(device, torch.device):
        return device.index if device.index is not None else torch.cuda.current_device()
    if isinstance(device, str):
        return _device_index(torch.device(device))
    return int(device)


def native_plan(plan: BstPlan, fplan: FilterPlan = FilterPlan(), full_turn: bool = False,
                device=None, n_angles: int | None = None, grid: bool = True) -> NativePlan:
    """Device plan for (plan, fplan, span) on `device`, cached on the BstPlan
    like the reference's lazily built tables (fourier_bp.py:154-162).
    ``grid=False`` skips the gridding tables (ramp / slant-stack / forward
    / preprocessing use); ``n_angles`` overrides the input row count (an odd
    full turn for the slant stack)."""
    dev = _device_index(device)
    key = ("native", fplan.kind, fplan.effective_rolloff, bool(full_turn), dev, n_angles, bool(grid))
    return plan._cached(key, lambda: NativePlan(plan, fplan, full_turn, dev, n_angles, grid))


_AUX_PLANS: dict = {}
_AUX_LOCK = threading.Lock()


def aux_plan(n_t: int, n_angles: int, full_turn: bool = False, output_n: int | None = None,
             fplan: FilterPlan = FilterPlan(), device=None) -> NativePlan:
    """Cached table-free device plan for the ramp, slant-stack, forward and
    preprocessing calls on a (n_t, n_angles) sinogram grid (and an output_n
    image grid): no gridding tables, built once per key and device."""
    dev = _device_index(device)
    n = n_t if output_n is None else int(output_n)
    n_theta = n_angles // 2 if full_turn else n_angles
    L = max(_next_pow2(2 * n_t), _next_pow2(n))
    key = (n_t, n_angles, bool(full_turn), n, fplan.kind, fplan.effective_rolloff, dev)
    hit = _AUX_PLANS.get(key)
    if hit is None:
        with _AUX_LOCK:
            hit = _AUX_PLANS.get(key)
            if hit is None:
                bp = BstPlan(n_t=max(n_t, 2), n_theta=max(n_theta, 1), radial_samples=L, output_n=n)
                hit = NativePlan(bp, fplan, full_turn, dev, n_angles=n_angles, grid=False)
                _AUX_PLANS[key] = hit
    return hit


def _to_device_rows(y: Sinogram, dev: int) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(y.data, dtype=np.float32)).to(f"cuda:{dev}")


def _check_plan(y: Sinogram, plan: BstPlan) -> None:
    half = y.n_angles // 2 if y.angles.full_turn else y.n_angles
    if y.n_t != plan.n_t or half != plan.n_theta:
        raise ValueError("sinogram dimensions do not match the plan")
    if y.angles.full_turn and y.n_angles != 2 * plan.n_theta:
        # the reference's resample_polar rejects it the same way (fourier_bp.py:331-332)
        raise ValueError("sinogram dimensions do not match the plan")


def _single_slice(op: str, y: Sinogram, plan: BstPlan, fplan: FilterPlan, device=None,
                  nat: NativePlan | None = None) -> ImageGrid:
    dev = _device_index(device)
    if nat is None:
        nat = native_plan(plan, fplan, y.angles.full_turn, dev)
    sino = _to_device_rows(y, dev)
    img = torch.empty((plan.output_n, plan.output_n), dtype=torch.float32, device=f"cuda:{dev}")
    ws = nat.new_workspace(1)
    with torch.cuda.device(dev):
        nat.reset_status(ws)
        nat.run(op, sino, img, 1, 1, ws)
        nat.read_status(ws)
    return ImageGrid(plan.output_n, img.cpu().numpy().astype(np.float64))


def ramp_filter(y: Sinogram, fplan: FilterPlan = FilterPlan(), workers: int = 1, device=None) -> Sinogram:
    """Ramp filtering along t on the GPU (fourier_bp.py:490-505)."""
    dev = _device_index(device)
    nat = aux_plan(y.n_t, y.n_angles, fplan=fplan, device=dev)
    sino = _to_device_rows(y, dev)
    out = torch.empty_like(sino)
    with torch.cuda.device(dev):
        nat.ramp(sino, out, 1)
    return Sinogram(y.detector, y.angles, out.cpu().numpy().astype(np.float64))


def bst_backproject(y: Sinogram, plan: BstPlan | None = None, workers: int = 1, device=None) -> ImageGrid:
    """Frequency-domain backprojection of a (filtered) sinogram (fourier_bp.py:435-461)."""
    if plan is None:
        plan = BstPlan.for_sinogram(y)
    _check_plan(y, plan)
    return _single_slice("bst", y, plan, FilterPlan(), device)


def fbp(y: Sinogram, plan: BstPlan | None = None, fplan: FilterPlan = FilterPlan(), kernel: str = "bst",
        workers: int = 1, device=None) -> ImageGrid:
    """Filtered backprojection with the selected kernel (fourier_bp.py:508-530)."""
    if kernel not in ("ss", "bst"):
        raise ValueError(f"unknown kernel {kernel!r}")
    if plan is None:
        plan = BstPlan.for_sinogram(y)
    if kernel == "ss":
        dev = _device_index(device)
        nat = aux_plan(y.n_t, y.n_angles, y.angles.full_turn, plan.output_n, fplan, dev)
        return _single_slice("fbp_ss", y, plan, fplan, dev, nat)
    _check_plan(y, plan)
    return _single_slice("fbp", y, plan, fplan, device)


# ---------------------------------------------------------------------------
# volume API
# ---------------------------------------------------------------------------


def default_batch(plan: BstPlan, full_turn: bool = False) -> int:
    """Slices per launch group (two groups in flight on two streams).  Larger
    groups fill the 148 SMs with fewer wave tails: at L = 4096 the measured
    step falls from 218 ms (4 slices) to 204 ms (24-31 slices,
    profiles/README.md).  Bounded by the polar texture's height,
    batch * polar rows <= 65000 (V + 1 rows per slice for half-turn input:
    31 slices at 2048 angles; 2V + 1 for full turn: 15), and at 64 slices."""
    L = plan.radial_samples
    rows = (2 * plan.n_theta if full_turn else plan.n_theta) + 1
    if L >= 1024:
        return max(1, min(64, 65000 // rows))
    return max(1, min(64, (4096 // L) ** 2, 65000 // rows))


def _split(n: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous [begin, end) slabs of n items over `parts` owners."""
    from .slabs import split
    return split(n, parts)


def _counts_frames(frames, dev: int, A: int, n_t: int):
    """Frames for NativePlan.counts: ("const", i0, dark) when both frames are
    constant (the reference pipeline's scalar i0 / dark, pipeline.py:447-451),
    else (flat, dark) device tensors."""
    f, d = frames.flat, frames.dark
    if (isinstance(f, np.ndarray) and isinstance(d, np.ndarray) and f.size and f.shape == (A, n_t)
            and d.shape == (A, n_t) and f.min() == f.max() and d.min() == d.max()):
        return ("const", float(f.flat[0]), float(d.flat[0]))
    return tuple(_frames_on(frames, dev, A, n_t))


def _frames_on(frames, dev: int, A: int, n_t: int):
    """(flat, dark) of a FlatDarkFrames as float32 [A][n_t] tensors on cuda:dev."""
    out = []
    for x in (frames.flat, frames.dark):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float32))
        t = t.to(device=f"cuda:{dev}", dtype=torch.float32).contiguous()
        if tuple(t.shape) != (A, n_t):
            raise ValueError(f"counts shape {(A, n_t)} does not match frames {tuple(t.shape)}")
        out.append(t)
    return out


def fbp_volume(sino, plan: BstPlan | None = None, fplan: FilterPlan = FilterPlan(), kernel: str = "bst",
               full_turn: bool = False, out: torch.Tensor | None = None, batch: int | None = None,
               devices=None, chunk: int | None = None, check: bool = True, frames=None,
               eps: float = 1e-6, center=None, rings: int | None = None,
               scale: float | None = None) -> torch.Tensor:
    """Reconstruct a sinogram volume [S][A][n_t] -> image volume [S][n][n].

    * CUDA tensor input: computed on that device, asynchronously on the
      current stream; returns a CUDA tensor (``out`` may be given).  With
      ``devices`` the volume is split into z-slabs over those GPUs: peer
      copies over NVLink to each GPU, reconstruction there, peer gather
      back into the output on the input's GPU.
    * CPU tensor / numpy input: streamed through ``devices`` (default: all
      visible GPUs) in contiguous z-slabs (pipeline.py:552-554 Q-blocks),
      with pinned async H2D / compute / D2H on three streams per device;
      returns a CPU tensor.  Pass pinned CPU tensors to avoid a staging copy.

    ``kernel`` is "bst" (fbp) or "ss" (ramp + slant stack); with
    ``kernel="none"`` the input is taken as already filtered
    (bst_backproject semantics, no 1/(2 pi)).

    With ``frames`` (a ``preprocess.FlatDarkFrames`` of [A][n_t] flat and
    dark fields) the input is raw transmission counts: the reference
    pipeline's normalize stage, -ln(max(I - D, eps) / max(I0 - D, eps))
    (preprocess.py:59-74, pipeline.py:447-459), runs fused into the radial
    kernel's load for kernel "bst" (device or host input), or as a separate
    pass before "ss" / "none" (device input).

    ``center`` ("auto": per-slice estimate_center; a float: that beta for
    every slice) and ``rings`` (odd window) run the reference pipeline's
    center and rings stages (pipeline.py:461-484) on the device (device
    input): for kernel "bst" without frames they are fused into the radial
    kernel's row load (tb_fbp_pre: per-slice shift and stripe profile, no
    extra sinogram passes), otherwise separate passes before the
    reconstruction; an implausible or undetermined centre raises
    CenteringError like the reference.

    ``scale`` (kernel "none" only) multiplies the backprojection inside the
    last kernel's epilogue (the pipeline's bst_backproject x FBP_SCALE).
    """
    if frames is not None and not eps > 0:
        raise ValueError("eps must be positive")
    if kernel not in ("bst", "ss", "none"):
        raise ValueError(f"unknown kernel {kernel!r}")
    if isinstance(sino, np.ndarray):
        sino = torch.from_numpy(np.ascontiguousarray(sino, dtype=np.float32))
    if sino.dtype != torch.float32 or sino.dim() != 3:
        raise ValueError("sinogram volume must be a float32 [S][A][n_t] tensor")
    sino = sino.contiguous()
    S, A, n_t = sino.shape
    if plan is None:
        plan = BstPlan(n_t=n_t, n_theta=A // 2 if full_turn else A)
    want_a = 2 * plan.n_theta if full_turn else plan.n_theta
    if n_t != plan.n_t or A != want_a:
        raise ValueError("sinogram dimensions do not match the plan")
    op = {"bst": "fbp", "ss": "fbp_ss", "none": "bst"}[kernel]
    if scale is not None and kernel != "none":
        raise ValueError("scale applies to kernel='none' (the fbp kernels carry 1/(2 pi))")
    n = plan.output_n
    if out is not None:
        _check_out(out, (S, n, n), sino)
    if batch is None:
        batch = default_batch(plan, full_turn)
    if (center is not None or rings is not None) and not sino.is_cuda:
        raise ValueError("center / rings stages run on device-resident volumes")
    pre = None
    if sino.is_cuda and S and (center is not None or rings is not None):
        from .preprocess import center_beta, preprocess_volume
        one_dev = devices is None or [_device_index(d) for d in devices] == [sino.device.index]
        if (frames is None and op == "fbp" and one_dev and plan.radial_samples == 2 * _next_pow2(n_t)):
            # centre and ring stages fused into K1's row load (tb_fbp_pre):
            # per-slice shift and stripe profile, no extra sinogram passes
            if rings is not None and (rings < 3 or rings % 2 == 0):
                raise ValueError(f"window must be an odd integer >= 3, got {rings}")
            dev = sino.device.index
            with torch.cuda.device(dev):
                bc = center_beta(sino, S, A, n_t, full_turn, center) if center is not None else None
                pre = native_plan(plan, fplan, full_turn, dev).pre_params(sino, S, bc, rings or 0)
        else:
            sino = preprocess_volume(sino, plan, full_turn, frames=frames, eps=eps, center=center, rings=rings)
            frames = None  # normalised by the preprocessing pass
    if sino.is_cuda and devices is not None and frames is None and S:
        devs = [_device_index(d) for d in devices]
        if devs != [sino.device.index]:
            return _device_volume_multi(sino, plan, fplan, op, full_turn, out, batch, devs, check, scale)
    if sino.is_cuda:
        dev = sino.device.index
        nat = native_plan(plan, fplan, full_turn, dev, grid=op != "fbp_ss")
        if out is None:
            out = torch.empty((S, n, n), dtype=torch.float32, device=sino.device)
        ws = nat.new_workspace(min(batch, max(S, 1)))
        with torch.cuda.device(dev):
            nat.reset_status(ws)
            if S and frames is not None:
                if op == "fbp":
                    nat.counts(sino, _counts_frames(frames, dev, A, n_t), eps, out, S, min(batch, S), ws)
                else:
                    flat, dark = _frames_on(frames, dev, A, n_t)
                    line = torch.empty_like(sino)
                    nat.normalize(sino, flat, dark, eps, line, S)
                    nat.run(op, line, out, S, min(batch, S), ws, scale=scale)
            elif S and pre is not None:
                nat.run_pre(sino, out, S, min(batch, S), ws, pre[0], pre[1])
            elif S:
                nat.run(op, sino, out, S, min(batch, S), ws, scale=scale)
            if check:
                nat.read_status(ws)
        return out
    if frames is not None and op != "fbp":
        raise ValueError("host-resident counts are supported for kernel 'bst' (fused normalisation)")
    return _host_volume(sino, plan, fplan, op, full_turn, out, batch, devices, chunk, check, frames, eps, scale)


def _device_volume_multi(sino, plan, fplan, op, full_turn, out, batch, devices, check, scale):
    """Device-resident input on one GPU, reconstructed as contiguous z-slabs
    on ``devices`` (pipeline.py:552-554 Q-blocks; no collective: slices are
    independent).  Each slab is copied peer-to-peer to its GPU
    (NVLink), reconstructed on its own stream and workspace, and gathered
    peer-to-peer into the output on the input's GPU; a slab on the input's
    GPU reads and writes in place.  The same device may appear more than once
    (independent streams / workspaces on one GPU).  Asynchronous on the
    input GPU's current stream, like the single-device call."""
    S = sino.shape[0]
    n = plan.output_n
    src = sino.device.index
    if out is None:
        out = torch.empty((S, n, n), dtype=torch.float32, device=sino.device)
    cur = torch.cuda.current_stream(src)
    ready = torch.cuda.Event()
    ready.record(cur)
    jobs = []
    for dev, (b, e) in zip(devices, _split(S, len(devices))):
        if e <= b:
            continue
        m = e - b
        nat = native_plan(plan, fplan, full_turn, dev, grid=op != "fbp_ss")
        with torch.cuda.device(dev):
            st = torch.cuda.Stream(dev)
            st.wait_event(ready)
            with torch.cuda.stream(st):
                x = sino[b:e] if dev == src else sino[b:e].to(f"cuda:{dev}", non_blocking=True)
                y = out[b:e] if dev == src else torch.empty((m, n, n), dtype=torch.float32, device=f"cuda:{dev}")
                ws = nat.new_workspace(min(batch, m))
                nat.reset_status(ws, st)
                nat.run(op, x, y, m, min(batch, m), ws, st, scale=scale)
                if dev != src:
                    out[b:e].copy_(y, non_blocking=True)  # peer copy back to the input's GPU
                done = torch.cuda.Event()
                done.record(st)
        jobs.append((nat, ws, st, done, x, y))
    for nat, ws, st, done, x, y in jobs:
        cur.wait_event(done)
        # keep the slab buffers alive until the input GPU's stream has
        # consumed them (the caching allocator reuses freed blocks per stream)
        for t in (x, y, ws):
            t.record_stream(st)
    if check:
        for nat, ws, st, *_ in jobs:
            nat.read_status(ws, st)
    return out


def _check_out(out, shape, sino) -> None:
    """A caller-supplied output must be exactly what the kernels write: the
    kernels take a raw pointer (no bounds, dtype or stride information)."""
    if not isinstance(out, torch.Tensor):
        raise ValueError("out must be a torch.Tensor")
    if tuple(out.shape) != tuple(shape):
        raise ValueError(f"out has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if out.dtype != torch.float32:
        raise ValueError(f"out must be float32, got {out.dtype}")
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")
    if sino.is_cuda and out.device != sino.device:
        raise ValueError(f"out is on {out.device}, the sinogram on {sino.device}")
    if not sino.is_cuda and out.is_cuda:
        raise ValueError("out must be a CPU tensor for host-resident input")


def _host_volume(sino, plan, fplan, op, full_turn, out, batch, devices, chunk, check, frames=None, eps=1e-6,
                 scale=None):
    S, A, n_t = sino.shape
    n = plan.output_n
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = [_device_index(d) for d in devices]
    if not devices:
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
    if out is None:
        out = torch.empty((S, n, n), dtype=torch.float32, pin_memory=True)
    if not sino.is_pinned():
        sino = sino.pin_memory()
    if chunk is None:
        # ~128 MiB of sinogram per copy: PCIe (not the kernels) bounds this
        # path, so small chunks shrink the un-overlapped first H2D / last D2H
        chunk = max(1, min(64, (128 << 20) // max(1, A * n_t * 4)))
    slabs = _split(S, len(devices))
    states = []
    for dev, (b, e) in zip(devices, slabs):
        if e <= b:
            continue
        nat = native_plan(plan, fplan, full_turn, dev, grid=op != "fbp_ss")
        m = min(chunk, e - b)
        with torch.cuda.device(dev):
            st = {
                "dev": dev, "nat": nat, "begin": b, "end": e, "next": b,
                "inb": [torch.empty((m, A, n_t), dtype=torch.float32, device=f"cuda:{dev}") for _ in range(2)],
                "outb": [torch.empty((m, n, n), dtype=torch.float32, device=f"cuda:{dev}") for _ in range(2)],
                "ws": nat.new_workspace(min(batch, m)),
                "s_in": torch.cuda.Stream(dev), "s_cmp": torch.cuda.Stream(dev), "s_out": torch.cuda.Stream(dev),
                "h2d": [torch.cuda.Event() for _ in range(2)],
                "cmp": [torch.cuda.Event() for _ in range(2)],
                "d2h": [torch.cuda.Event() for _ in range(2)],
                "k": 0, "chunk": m,
                "frames": _counts_frames(frames, dev, A, n_t) if frames is not None else None,
            }
            nat.reset_status(st["ws"], st["s_cmp"])
        states.append(st)
    active = list(states)
    while active:
        for st in list(active):
            b = st["next"]
            if b >= st["end"]:
                active.remove(st)
                continue
            e = min(st["end"], b + st["chunk"])
            m = e - b
            k = st["k"]
            dev = st["dev"]
            with torch.cuda.device(dev):
                with torch.cuda.stream(st["s_in"]):
                    st["s_in"].wait_event(st["cmp"][k])  # input buffer k free
                    st["inb"][k][:m].copy_(sino[b:e], non_blocking=True)
                    st["h2d"][k].record(st["s_in"])
                st["s_cmp"].wait_event(st["h2d"][k])
                st["s_cmp"].wait_event(st["d2h"][k])  # output buffer k free
                if st["frames"] is not None:
                    st["nat"].counts(st["inb"][k], st["frames"], eps, st["outb"][k], m, min(batch, st["chunk"]),
                                     st["ws"], st["s_cmp"])
                else:
                    st["nat"].run(op, st["inb"][k], st["outb"][k], m, min(batch, st["chunk"]), st["ws"], st["s_cmp"],
                                  scale=scale)
                st["cmp"][k].record(st["s_cmp"])
                with torch.cuda.stream(st["s_out"]):
                    st["s_out"].wait_event(st["cmp"][k])
                    out[b:e].copy_(st["outb"][k][:m], non_blocking=True)
                    st["d2h"][k].record(st["s_out"])
            st["next"] = e
            st["k"] = 1 - k
    for st in states:
        with torch.cuda.device(st["dev"]):
            st["s_out"].synchronize()
            if check:
                st["nat"].read_status(st["ws"], st["s_cmp"])
    return out
