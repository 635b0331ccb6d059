"""CPU oracle for the BST filtered-backprojection hot path.

TEST INFRASTRUCTURE ONLY.  This module is the checker, never the product:
only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it.  The product path
(``paper_1704_08364_b200``) runs hand-written sm_100a CUDA kernels and
fails loudly when the native library is missing.

What it restates (float64 numpy, independently written, same algebra):

* ``OraclePlan``       <- ``BstPlan`` / ``FilterPlan``
                          (reference ``pkg/src/tomoblocks/fourier_bp.py:69-267``)
* ``ramp_filter``      <- ``apply_ramp_rows`` + ``ramp_filter`` (``fourier_bp.py:469-505``)
* ``bst_backproject``  <- the P0..P8 chain of ``bst_backproject`` (``fourier_bp.py:302-461``)
* ``fbp``              <- ``fbp`` (``fourier_bp.py:508-530``)
* ``backproject_ss``   <- ``backproject_ss`` (``projector.py:126-158``)
* ``k1_polar`` / ``k1b_common`` / ``k2_columns`` / ``k3_image``
                       <- the same chain re-factored into the three GPU kernels
                          (SURVEY.md Appendix A); used to check each CUDA kernel
                          in isolation through the workspace.

Parity pinning: the reference ships no golden vectors, so
``tests/golden/make_golden.py`` runs the real reference package in the build
container and commits its outputs; ``tests/test_oracle_golden.py`` pins this
oracle against them to ~1e-12.

Third-party arithmetic used by the reference (not vendored there either):
numpy.fft (pocketfft, numpy 2.3.5 in the build image) and scipy.special.i0
(cephes, scipy 1.18.1).  The oracle calls the same two functions.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from concurrent.futures import ThreadPoolExecutor

import numpy as np

try:  # scipy is the reference's own dependency for the KB window (fourier_bp.py:37)
    from scipy.special import i0 as _i0
except Exception:  # pragma: no cover - scipy is present in the image
    _i0 = np.i0

FBP_SCALE = 1.0 / (2.0 * math.pi)  # fourier_bp.py:59


def next_pow2(n: int) -> int:
    """Smallest power of two >= n (fourier_bp.py:62-66)."""
    return 1 if n <= 1 else 1 << (int(n) - 1).bit_length()


# ---------------------------------------------------------------------------
# plan (fourier_bp.py:69-267)
# ---------------------------------------------------------------------------


@dataclass
class OraclePlan:
    n_t: int
    n_theta: int
    pad_factor: int = 2
    radial_samples: int | None = None
    kb_beta: float = 10.0
    kb_support: float = 0.1
    sigma_min_bins: int = 1
    interp: str = "bilinear"
    output_n: int | None = None
    rolloff: float = 1.0  # FilterPlan.effective_rolloff (fourier_bp.py:265-267)

    def _memo(self, key, build):
        cache = self.__dict__.setdefault("_tables", {})
        if key not in cache:
            cache[key] = build()
        return cache[key]

    def __post_init__(self):
        # validation mirrors fourier_bp.py:88-109
        if self.n_t < 2 or self.n_theta < 1:
            raise ValueError("need n_t >= 2 and n_theta >= 1")
        if self.pad_factor < 2:
            raise ValueError(f"pad_factor must be >= 2, got {self.pad_factor}")
        if self.sigma_min_bins < 1:
            raise ValueError(f"sigma_min_bins must be >= 1, got {self.sigma_min_bins}")
        if self.interp not in ("bilinear", "nearest"):
            raise ValueError(f"unknown interp mode {self.interp!r}")
        if self.radial_samples is None:
            self.radial_samples = next_pow2(self.pad_factor * self.n_t)
        L = self.radial_samples
        if L & (L - 1) or L < self.pad_factor * self.n_t:
            raise ValueError(
                f"radial_samples must be a power of two >= pad_factor * n_t, got {L}")
        if self.output_n is None:
            self.output_n = self.n_t
        if not 1 <= self.output_n <= L:
            raise ValueError("output_n must be in [1, radial_samples]")

    # scalar geometry (fourier_bp.py:119-152)
    @property
    def L(self) -> int:
        return int(self.radial_samples)

    @property
    def H(self) -> int:
        return self.L // 2

    @property
    def n(self) -> int:
        return int(self.output_n)

    @property
    def npad(self) -> int:
        return 2 * next_pow2(self.n_t)  # fourier_bp.py:494

    @property
    def dt(self) -> float:
        return 2.0 / (self.n_t - 1)

    @property
    def df(self) -> float:
        return 1.0 / (self.L * self.dt)

    @property
    def sigma_min(self) -> float:
        return self.sigma_min_bins * self.df

    @property
    def roll(self) -> int:
        return int(round((self.n_t - 1) / 2.0))  # Python half-to-even, fourier_bp.py:136

    @property
    def du(self) -> float:
        return 2.0 / self.n

    @property
    def dnu(self) -> float:
        return 1.0 / (self.L * self.du)

    @property
    def amp(self) -> float:
        return (self.dnu * self.L) ** 2 * self.dt

    # tables (fourier_bp.py:164-220), built once per plan like the reference's cache
    def t_samples(self) -> np.ndarray:
        return -1.0 + 2.0 * np.arange(self.n_t) / (self.n_t - 1)  # grids.py:61-62

    def _build_freqs(self) -> np.ndarray:
        return np.fft.fftfreq(self.L, d=self.dt)

    def _build_phase(self) -> np.ndarray:
        return np.exp(2j * np.pi * self.freqs() * (1.0 - self.roll * self.dt))

    def _build_bump(self) -> np.ndarray:
        t = self.t_samples()
        arg = np.sqrt(np.maximum(1.0 - (t / self.kb_support) ** 2, 0.0))
        val = _i0(self.kb_beta * arg) / _i0(self.kb_beta)
        return np.where(np.abs(t) <= self.kb_support, val, 0.0)

    def _build_ref_spectrum(self) -> np.ndarray:
        ones = np.zeros(self.L)
        ones[: self.n_t] = 1.0
        return np.fft.fft(np.roll(ones, -self.roll)) * self.phase()

    def _build_denom(self) -> np.ndarray:
        return np.maximum(np.abs(self.freqs()), self.sigma_min)

    def _build_coverage(self) -> np.ndarray:
        x = -1.0 + 2.0 * (np.arange(self.n) + 0.5) / self.n
        r = np.sqrt(x[None, :] ** 2 + x[:, None] ** 2)
        with np.errstate(divide="ignore", invalid="ignore"):
            far = 2.0 * np.arcsin(np.minimum(1.0, 1.0 / np.maximum(r, 1e-300)))
        return np.where(r > 1.0, far, np.pi)

    def _build_modulation(self) -> np.ndarray | None:
        """Half-node shift of inverse_dft2_and_shift (fourier_bp.py:424-430)."""
        L, n = self.L, self.n
        m0 = L // 2 - n // 2
        delta = (-1.0 + 1.0 / n) - (m0 - L // 2) * self.du
        if delta == 0.0:
            return None
        nu = np.fft.fftfreq(L) * L * self.dnu
        return np.exp(2j * np.pi * nu * delta)

    def _build_lattice_coords(self):
        """(ri, ti) of every Cartesian node, rows <-> nu2, cols <-> nu1
        (fourier_bp.py:226-232)."""
        L = self.L
        nu = np.fft.fftfreq(L) * L * self.dnu
        ri = np.hypot(nu[None, :], nu[:, None]) / self.df
        ang = np.mod(np.arctan2(nu[:, None], nu[None, :]), 2.0 * np.pi)
        ti = ang * (2 * self.n_theta / (2.0 * np.pi))
        return ri, ti

    def freqs(self):
        return self._memo('freqs', self._build_freqs)

    def phase(self):
        return self._memo('phase', self._build_phase)

    def bump(self):
        return self._memo('bump', self._build_bump)

    def ref_spectrum(self):
        return self._memo('ref_spectrum', self._build_ref_spectrum)

    def denom(self):
        return self._memo('denom', self._build_denom)

    def coverage(self):
        return self._memo('coverage', self._build_coverage)

    def modulation(self):
        return self._memo('modulation', self._build_modulation)

    def lattice_coords(self):
        return self._memo('lattice_coords', self._build_lattice_coords)


# ---------------------------------------------------------------------------
# direct restatement of the reference chain
# ---------------------------------------------------------------------------


def _sample_image(img: np.ndarray, u1, u2, nearest: bool) -> np.ndarray:
    """Image samples at points, pixel-centre convention, zero outside
    (projector.py:65-91)."""
    n = img.shape[0]
    du = 2.0 / n
    fx = (u1 + 1.0) / du - 0.5
    fy = (u2 + 1.0) / du - 0.5
    if nearest:
        ix, iy = np.rint(fx).astype(np.int64), np.rint(fy).astype(np.int64)
        ok = (ix >= 0) & (ix < n) & (iy >= 0) & (iy < n)
        return np.where(ok, img[np.clip(iy, 0, n - 1), np.clip(ix, 0, n - 1)], 0.0)
    x0, y0 = np.floor(fx).astype(np.int64), np.floor(fy).astype(np.int64)
    wx, wy = fx - x0, fy - y0
    out = np.zeros(np.broadcast(fx, fy).shape)
    for dy in (0, 1):
        for dx in (0, 1):
            ix, iy = x0 + dx, y0 + dy
            w = (wx if dx else 1.0 - wx) * (wy if dy else 1.0 - wy)
            ok = (ix >= 0) & (ix < n) & (iy >= 0) & (iy < n)
            out += np.where(ok, img[np.clip(iy, 0, n - 1), np.clip(ix, 0, n - 1)] * w, 0.0)
    return out


def forward_project(img: np.ndarray, n_t: int, n_angles: int, full_turn: bool = False,
                    step_length: float = 0.5, nearest: bool = False) -> np.ndarray:
    """Midpoint-rule line integrals along every (theta_j, t_i) ray over the
    circumscribed diameter (projector.py:94-123); [n_angles][n_t]."""
    n = img.shape[0]
    h = step_length * (2.0 / n)
    half = np.sqrt(2.0)
    m = int(np.ceil(2.0 * half / h))
    ell = -half + (np.arange(m) + 0.5) * h
    t = -1.0 + 2.0 * np.arange(n_t) / (n_t - 1)
    th = (2.0 * np.pi if full_turn else np.pi) / n_angles * np.arange(n_angles)
    out = np.empty((n_angles, n_t))
    for j in range(n_angles):
        c, s = np.cos(th[j]), np.sin(th[j])
        u1 = t[:, None] * c - ell[None, :] * s
        u2 = t[:, None] * s + ell[None, :] * c
        out[j] = _sample_image(img, u1, u2, nearest).sum(axis=1) * h
    return out


def _parabolic_peak(values: np.ndarray, k: int) -> float:
    """Sub-sample peak through k-1, k, k+1 (preprocess.py:77-85)."""
    if k <= 0 or k >= len(values) - 1:
        return float(k)
    y0, y1, y2 = values[k - 1], values[k], values[k + 1]
    denom = y0 - 2.0 * y1 + y2
    if denom == 0.0:
        return float(k)
    return k + 0.5 * (y0 - y2) / denom


def estimate_center(y: np.ndarray) -> tuple[float, float]:
    """(beta, confidence) from the mirror consistency of the first and the
    reversed last projection: full cross-correlation, first argmax,
    parabolic refinement, beta = lag / 2 (preprocess.py:88-118).  Raises
    ValueError where the reference raises CenteringError."""
    v, n_t = y.shape
    if v < 2:
        raise ValueError("need at least two projection angles")
    a = y[0].astype(float)
    b = y[-1][::-1].astype(float)
    a = a - a.mean()
    b = b - b.mean()
    norm = np.linalg.norm(a) * np.linalg.norm(b)
    if norm == 0.0:
        raise ValueError("centering undetermined: constant sinogram")
    corr = np.correlate(a, b, mode="full")
    k = int(np.argmax(corr))
    beta = (_parabolic_peak(corr, k) - (n_t - 1)) / 2.0
    if abs(beta) > n_t / 2:
        raise ValueError(f"implausible center shift of {beta:.1f} bins")
    return beta, float(np.clip(corr[k] / norm, 0.0, 1.0))


def apply_center(y: np.ndarray, beta: float) -> np.ndarray:
    """Undo a detector shift of beta bins by linear interpolation, zero out
    of range (preprocess.py:121-138)."""
    n_t = y.shape[1]
    idx = np.arange(n_t) + beta
    i0 = np.floor(idx).astype(np.int64)
    fr = idx - i0
    ok0 = (i0 >= 0) & (i0 <= n_t - 1)
    ok1 = (i0 + 1 >= 0) & (i0 + 1 <= n_t - 1)
    i0c, i1c = np.clip(i0, 0, n_t - 1), np.clip(i0 + 1, 0, n_t - 1)
    return y[:, i0c] * np.where(ok0, 1.0 - fr, 0.0) + y[:, i1c] * np.where(ok1, fr, 0.0)


def suppress_rings(y: np.ndarray, window: int = 9) -> np.ndarray:
    """Subtract the angle-constant stripe estimate: per-detector mean over
    angles minus its reflect-padded moving average (preprocess.py:141-154)."""
    m = y.mean(axis=0)
    padded = np.pad(m, window // 2, mode="reflect")
    smooth = np.convolve(padded, np.full(window, 1.0 / window), mode="valid")
    return y - (m - smooth)[None, :]


def normalize(counts: np.ndarray, flat: np.ndarray, dark: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    """Transmission counts to line integrals, -log(max(I - D, eps) / max(I0 - D, eps))
    (preprocess.py:59-74; np.maximum propagates NaN like the reference)."""
    if eps <= 0:
        raise ValueError("eps must be positive")
    counts = np.asarray(counts, dtype=np.float64)
    num = np.maximum(counts - np.asarray(dark, dtype=np.float64), eps)
    den = np.maximum(np.asarray(flat, dtype=np.float64) - np.asarray(dark, dtype=np.float64), eps)
    return -np.log(num / den)


def ramp_filter(y: np.ndarray, plan: OraclePlan) -> np.ndarray:
    """Rows of ``y`` through the padded 2*pi*|f| ramp (fourier_bp.py:469-505)."""
    y = np.asarray(y, dtype=np.float64)
    n_t = y.shape[-1]
    npad = 2 * next_pow2(n_t)
    f = np.fft.rfftfreq(npad, d=plan.dt)
    gain = 2.0 * np.pi * np.abs(f)
    if plan.rolloff < 1.0:
        fn = f[-1]
        f0 = plan.rolloff * fn
        zone = f > f0
        gain = gain.copy()
        gain[zone] *= 0.5 * (1.0 + np.cos(np.pi * (f[zone] - f0) / ((1.0 - plan.rolloff) * fn)))
    spec = np.fft.rfft(y, n=npad, axis=-1)
    return np.fft.irfft(spec * gain, n=npad, axis=-1)[..., :n_t]


def _polar_spectrum(h_full: np.ndarray, plan: OraclePlan) -> np.ndarray:
    """Window, pad, roll and radially transform the full-circle rows
    (fourier_bp.py:314-362), then split the rect component and apply the
    1/max(|f|, sigma_min) kernel (fourier_bp.py:452-455, 365-373)."""
    L = plan.L
    b = plan.bump()
    centre = h_full.mean(axis=0)
    win = h_full * (1.0 - b) + b * centre
    padded = np.zeros((h_full.shape[0], L))
    padded[:, : plan.n_t] = win
    padded = np.roll(padded, -plan.roll, axis=1)
    spec = np.fft.fft(padded, axis=1) * plan.phase()[None, :]
    ref = plan.ref_spectrum()
    coef = spec[:, 0].real / ref[0].real
    bal = (spec - coef[:, None] * ref[None, :]) / plan.denom()[None, :]
    return bal, coef


def _grid(bal: np.ndarray, plan: OraclePlan) -> np.ndarray:
    """Polar -> Cartesian interpolation on the L x L lattice (fourier_bp.py:376-410)."""
    ri, ti = plan.lattice_coords()
    rows = bal.shape[0]
    top = plan.L // 2 - 1
    if plan.interp == "nearest":
        ir = np.rint(ri).astype(np.int64)
        it = np.rint(ti).astype(np.int64) % rows
        keep = ir <= top
        return np.where(keep, bal[it, np.clip(ir, 0, top)], 0.0)
    r0 = np.floor(ri).astype(np.int64)
    fr = ri - r0
    tf = np.floor(ti)
    t0 = tf.astype(np.int64) % rows
    ft = ti - tf
    t1 = (t0 + 1) % rows
    ra = np.clip(r0, 0, top)
    rb = np.clip(r0 + 1, 0, top)
    val = ((1.0 - fr) * (1.0 - ft)) * bal[t0, ra]
    val = val + (fr * (1.0 - ft)) * bal[t0, rb]
    val = val + ((1.0 - fr) * ft) * bal[t1, ra]
    val = val + (fr * ft) * bal[t1, rb]
    return np.where(ri <= top, val, 0.0)


def _inverse(cart: np.ndarray, plan: OraclePlan) -> np.ndarray:
    """Half-node modulation, ifft2, fftshift, real part, crop (fourier_bp.py:413-432)."""
    L, n = plan.L, plan.n
    mod = plan.modulation()
    if mod is not None:
        cart = cart * mod[None, :] * mod[:, None]
    img = np.fft.fftshift(np.fft.ifft2(cart)).real * plan.amp
    m0 = L // 2 - n // 2
    return img[m0 : m0 + n, m0 : m0 + n]


def bst_backproject(y: np.ndarray, plan: OraclePlan, full_turn: bool = False) -> np.ndarray:
    """BST backprojection of one (already ramp-filtered) slice (fourier_bp.py:435-461)."""
    y = np.asarray(y, dtype=np.float64)
    full = y if full_turn else np.vstack([y, y[:, ::-1]])  # fourier_bp.py:302-311
    bal, coef = _polar_spectrum(full, plan)
    cart = _grid(bal, plan)
    out = _inverse(cart, plan) + coef.mean() * plan.coverage()
    if not np.all(np.isfinite(out)):
        raise FloatingPointError("non-finite values in backprojection output")
    return out


def backproject_ss(y: np.ndarray, n: int, full_turn: bool = False) -> np.ndarray:
    """Slant-stack Riemann sum with linear interpolation along t
    (projector.py:126-158): zero outside [-1, 1], weight span/V."""
    y = np.asarray(y, dtype=np.float64)
    n_ang, n_t = y.shape
    dt = 2.0 / (n_t - 1)
    span = 2.0 * np.pi if full_turn else np.pi
    th = np.arange(n_ang) * (span / n_ang)
    x = -1.0 + 2.0 * (np.arange(n) + 0.5) / n
    acc = np.zeros((n, n))
    for j in range(n_ang):
        pos = (x[None, :] * np.cos(th[j]) + x[:, None] * np.sin(th[j]) + 1.0) / dt
        base = np.floor(pos)
        frac = pos - base
        lo = np.clip(base.astype(np.int64), 0, n_t - 2)
        ok = (pos >= 0.0) & (pos <= n_t - 1)
        acc += np.where(ok, y[j, lo] * (1.0 - frac) + y[j, lo + 1] * frac, 0.0)
    return acc * (span / n_ang)


def fbp(y: np.ndarray, plan: OraclePlan, kernel: str = "bst", full_turn: bool = False) -> np.ndarray:
    """Ramp filter -> backprojection -> x 1/(2 pi) (fourier_bp.py:508-530)."""
    if kernel not in ("ss", "bst"):
        raise ValueError(f"unknown kernel {kernel!r}")
    h = ramp_filter(y, plan)
    if kernel == "ss":
        return backproject_ss(h, plan.n, full_turn) * FBP_SCALE
    return bst_backproject(h, plan, full_turn) * FBP_SCALE


def fbp_volume(vol: np.ndarray, plan: OraclePlan, kernel: str = "bst", workers: int = 1,
               full_turn: bool = False) -> np.ndarray:
    """Slice-parallel FBP over a [S][V][n_t] volume.  Slices are independent
    (pipeline.py:395-400, 552-554); a thread pool stands in for the reference
    pipeline's backproject-stage worker pool (numpy releases the GIL in FFTs)."""
    vol = np.asarray(vol)
    out = np.empty((vol.shape[0], plan.n, plan.n))

    def one(s):
        out[s] = fbp(vol[s], plan, kernel, full_turn)

    if workers <= 1:
        for s in range(vol.shape[0]):
            one(s)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(one, range(vol.shape[0])))
    return out


# ---------------------------------------------------------------------------
# three-kernel restatement: the per-kernel oracle
# ---------------------------------------------------------------------------


def _true_origin_dft(rows: np.ndarray, plan: OraclePlan) -> np.ndarray:
    """S_k = sum_i w_i exp(-2 pi i f_k t_i) for k < H; equal to the reference's
    roll + FFT + layout_phase (fourier_bp.py:345, 359) in exact arithmetic."""
    L, H = plan.L, plan.H
    padded = np.zeros(rows.shape[:-1] + (L,))
    padded[..., : plan.n_t] = rows
    f = np.arange(H) / (L * plan.dt)
    return np.fft.fft(padded, axis=-1)[..., :H] * np.exp(2j * np.pi * f)


def support_range(plan: OraclePlan) -> tuple[int, int]:
    """Index range [lo, hi] of the KB window, closed under i -> n_t-1-i."""
    nz = np.nonzero(np.abs(plan.t_samples()) <= plan.kb_support)[0]
    if nz.size == 0:
        return 0, -1
    lo = int(min(nz[0], plan.n_t - 1 - nz[-1]))
    hi = int(max(nz[-1], plan.n_t - 1 - nz[0]))
    return lo, hi


def _den_ref(plan: OraclePlan):
    H = plan.H
    f = np.arange(H) / (plan.L * plan.dt)
    den = np.maximum(np.abs(f), plan.sigma_min)
    ref = _true_origin_dft(np.ones(plan.n_t), plan)
    return den, ref


def k1_polar(h: np.ndarray, plan: OraclePlan):
    """K1: per processed row j, Ahat_j = (A_j - a_j ref)/den over k < H with
    A_j the true-origin spectrum of h_j (1 - bump); also a_j and the support
    column sums of h."""
    h = np.asarray(h, dtype=np.float64)
    b = plan.bump()
    den, ref = _den_ref(plan)
    A = _true_origin_dft(h * (1.0 - b), plan)
    a = A[:, 0].real / plan.n_t
    Ahat = (A - a[:, None] * ref[None, :]) / den[None, :]
    Ahat[:, 0] = 0.0
    lo, hi = support_range(plan)
    colsum = h[:, lo : hi + 1].sum(axis=0)
    return Ahat, a, colsum


def k1b_common(colsum: np.ndarray, a: np.ndarray, plan: OraclePlan, full_turn: bool = False):
    """K1b: the angle-independent row Chat (from the windowed angular mean row,
    fourier_bp.py:336-341) and coef.mean() (fourier_bp.py:458)."""
    lo, hi = support_range(plan)
    rows_total = 2 * plan.n_theta
    if full_turn:
        m = colsum / rows_total
    else:
        m = (colsum + colsum[::-1]) / rows_total
    b = plan.bump()
    bm = np.zeros(plan.n_t)
    bm[lo : hi + 1] = b[lo : hi + 1] * m
    den, ref = _den_ref(plan)
    Cm = _true_origin_dft(bm, plan)
    c = bm.sum() / plan.n_t
    Chat = (Cm - c * ref) / den
    Chat[0] = 0.0
    coef_mean = a.mean() + c
    return Chat, coef_mean


def _lattice_half(plan: OraclePlan):
    """Signed lattice indices of the half plane: columns a in [0, H] (a = H is
    the -L/2 node), all L rows."""
    L, H = plan.L, plan.H
    cols = np.arange(H + 1)
    acol = np.where(cols < H, cols, -H)
    rows = np.arange(L)
    brow = np.where(rows < H, rows, rows - L)
    return acol, brow


def _node_values(Ahat, Chat, plan, a_s, b_s, full_turn):
    """Interpolated C(a, b) for signed lattice indices (arrays)."""
    V = plan.n_theta
    rows = 2 * V
    top = plan.H - 1
    ratio = plan.dnu / plan.df
    ri = np.hypot(a_s * 1.0, b_s * 1.0) * ratio
    ti = np.mod(np.arctan2(b_s * 1.0, a_s * 1.0), 2 * np.pi) * (V / np.pi)

    def P(t, r):
        if full_turn:
            return Ahat[t, r] + Chat[r]
        tt = np.where(t < V, t, t - V)
        v = Ahat[tt, r]
        return np.where(t < V, v, np.conj(v)) + Chat[r]

    if plan.interp == "nearest":
        ir = np.rint(ri).astype(np.int64)
        it = np.rint(ti).astype(np.int64) % rows
        return np.where(ir <= top, P(it, np.clip(ir, 0, top)), 0.0)
    r0 = np.floor(ri).astype(np.int64)
    fr = ri - r0
    tfl = np.floor(ti)
    t0 = tfl.astype(np.int64) % rows
    ft = ti - tfl
    t1 = (t0 + 1) % rows
    ra, rb = np.clip(r0, 0, top), np.clip(r0 + 1, 0, top)
    val = ((1 - fr) * (1 - ft)) * P(t0, ra) + (fr * (1 - ft)) * P(t0, rb) \
        + ((1 - fr) * ft) * P(t1, ra) + (fr * ft) * P(t1, rb)
    return np.where(ri <= top, val, 0.0)


def k2_columns(Ahat: np.ndarray, Chat: np.ndarray, plan: OraclePlan, full_turn: bool = False):
    """K2: half-plane gather of the Hermitian part of the reference lattice,
    then the pruned inverse DFT along k2.  Returns G[a][m2], a in [0, H],
    m2 < n (unnormalised: no 1/L).

    ``.real`` of ``ifft2`` (fourier_bp.py:431) equals the ifft2 of the
    Hermitian part 0.5*(C[k] + conj(C[-k mod L])).  For half-turn input the
    point-reflected node is the conjugate mirror row, so only the Nyquist
    lines (index L/2 aliases to itself) need the explicit average; for
    full-turn input every node does."""
    L, H, n = plan.L, plan.H, plan.n
    acol, brow = _lattice_half(plan)
    A2, B2 = np.meshgrid(acol, brow, indexing="ij")  # [H+1][L] signed
    mod = plan.modulation()
    modm = np.ones(L, dtype=complex) if mod is None else mod

    def lattice_value(a_s, b_s):
        C = _node_values(Ahat, Chat, plan, a_s, b_s, full_turn)
        return C * modm[a_s % L] * modm[b_s % L]

    def partner(k):  # signed index of (-k mod L)
        return np.where(k == -H, -H, -k)

    C = 0.5 * (lattice_value(A2, B2) + np.conj(lattice_value(partner(A2), partner(B2))))
    g = np.fft.ifft(C, axis=1) * L  # unnormalised inverse along k2
    idx = (np.arange(n) - n // 2) % L
    return g[:, idx]


def k3_image(G: np.ndarray, coef_mean: float, plan: OraclePlan, scale: float = 1.0):
    """K3: C2R along k1 with crop, amplitude scale and coverage add-back."""
    L, H, n = plan.L, plan.H, plan.n
    half = G.copy()
    half[0] = half[0].real
    half[H] = half[H].real
    full = np.zeros((L, n), dtype=complex)
    full[: H + 1] = half
    full[H + 1 :] = np.conj(half[1:H][::-1])
    img = (np.fft.ifft(full, axis=0) * L).real  # [a -> m1][m2]
    idx = (np.arange(n) - n // 2) % L
    img = img[idx].T * (plan.amp / (L * L))  # [m2][m1]
    return (img + coef_mean * plan.coverage()) * scale


def bst_3k(h: np.ndarray, plan: OraclePlan, full_turn: bool = False, scale: float = 1.0):
    """Full BST through the three-kernel restatement."""
    Ahat, a, colsum = k1_polar(h, plan)
    Chat, coef_mean = k1b_common(colsum, a, plan, full_turn)
    G = k2_columns(Ahat, Chat, plan, full_turn)
    return k3_image(G, coef_mean, plan, scale)


# ---------------------------------------------------------------------------
# synthetic inputs (phantom.py:67-93 generalised with in-plane rotation)
# ---------------------------------------------------------------------------

# Modified Shepp-Logan (Toft) ellipses: (rho, a, b, x0, y0, phi_deg)
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


def ellipse_sinogram(ellipses, n_t: int, n_angles: int, full_turn: bool = False) -> np.ndarray:
    """Exact line integrals of a sum of rotated constant ellipses on the
    reference grids (detector grids.py:61-62, angles grids.py:85-95)."""
    t = -1.0 + 2.0 * np.arange(n_t) / (n_t - 1)
    span = 2.0 * np.pi if full_turn else np.pi
    th = np.arange(n_angles) * (span / n_angles)
    out = np.zeros((n_angles, n_t))
    for rho, a, b, x0, y0, phi in ellipses:
        al = np.deg2rad(phi)
        q2 = (a * np.cos(th - al)) ** 2 + (b * np.sin(th - al)) ** 2
        tp = t[None, :] - (x0 * np.cos(th) + y0 * np.sin(th))[:, None]
        under = np.clip(q2[:, None] - tp ** 2, 0.0, None)
        out += 2.0 * rho * a * b * np.sqrt(under) / q2[:, None]
    return out


def ellipsoid_volume_sinogram(n_slices: int, n_t: int, n_angles: int,
                              a=0.5, b=0.4, c=0.5, center=(0.1, -0.05, 0.0), rho=1.0,
                              slices: tuple[int, int] | None = None) -> np.ndarray:
    """Per-slice analytic sinogram of one off-centre ellipsoid at slice heights
    s_k = -1 + 2(k+1/2)/S (cli.py:156, phantom.py:44-50, 67-93); ``slices``
    restricts to the slab [b, e)."""
    first, last = slices if slices is not None else (0, n_slices)
    vol = np.zeros((last - first, n_angles, n_t))
    for k in range(first, last):
        s = -1.0 + 2.0 * (k + 0.5) / n_slices
        srel = (s - center[2]) / c
        if abs(srel) > 1.0:
            continue
        sc = math.sqrt(max(1.0 - srel * srel, 0.0))
        vol[k - first] = ellipse_sinogram([(rho, a * sc, b * sc, center[0], center[1], 0.0)], n_t, n_angles)
    return vol
