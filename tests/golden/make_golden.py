"""Generate the committed golden vectors by running the REAL reference package.

Run in the build container only (it imports ``/root/reference/pkg/src``, which
does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every case stores the float32 sinogram handed to both implementations, the
plan/filter parameters, and the reference's float64 outputs of
``tomoblocks.fourier_bp.fbp`` (``fourier_bp.py:508-530``; kernel "bst" and,
for some cases, "ss"), ``ramp_filter`` (``:490-505``) and ``bst_backproject``
(``:435-461``).  numpy / scipy versions are recorded in ``versions.json``.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

from oracle.bst_oracle import SHEPP_LOGAN, ellipse_sinogram  # noqa: E402  (input synthesis only)

from tomoblocks import fourier_bp as ref_fbp  # noqa: E402
from tomoblocks.grids import AngleAxis, DetectorAxis, Sinogram  # noqa: E402


def _case(name, sino, plan_kw, filt_kw=None, full_turn=False, ss=False):
    sino = np.asarray(sino, dtype=np.float32)
    n_ang, n_t = sino.shape
    filt_kw = filt_kw or {}
    n_theta = n_ang // 2 if full_turn else n_ang
    y = Sinogram(DetectorAxis(n_t), AngleAxis(n_ang, full_turn=full_turn), sino.astype(np.float64))
    plan = ref_fbp.BstPlan(n_t=n_t, n_theta=n_theta, **plan_kw)
    fplan = ref_fbp.FilterPlan(**filt_kw)
    out = {
        "sino": sino,
        "fbp_bst": ref_fbp.fbp(y, plan, fplan, kernel="bst").data,
        "ramp": ref_fbp.ramp_filter(y, fplan).data,
        "bst": ref_fbp.bst_backproject(y, plan).data,
        "params": np.array(json.dumps({"plan": plan_kw, "filter": filt_kw,
                                       "full_turn": full_turn, "n_theta": n_theta})),
    }
    if ss:
        out["fbp_ss"] = ref_fbp.fbp(y, plan, fplan, kernel="ss").data
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: sino {sino.shape} -> {out['fbp_bst'].shape}")


def _norm_case(name, y, i0, dark_level, rng, plan_kw=None):
    """Counts -> normalize -> fbp through the reference (preprocess.py:59-74,
    fourier_bp.py:508-530); frames vary per angle and detector, and a few
    samples fall below the dark level (the eps clamp)."""
    from tomoblocks import preprocess as ref_pre
    plan_kw = plan_kw or {}
    v, n_t = y.shape
    flat = (i0 * (1.0 + 0.02 * rng.standard_normal((v, n_t)))).astype(np.float32)
    dark = (dark_level * (1.0 + 0.1 * rng.random((v, n_t)))).astype(np.float32)
    counts = (flat - dark) * np.exp(-y) * (1.0 + 0.01 * rng.standard_normal((v, n_t))) + dark
    counts = counts.astype(np.float32)
    counts[3, 5] = dark[3, 5] - 1.0  # below dark: clamped at eps
    frames = ref_pre.FlatDarkFrames(flat=flat.astype(np.float64), dark=dark.astype(np.float64))
    line = ref_pre.normalize(counts.astype(np.float64), frames)
    ys = Sinogram(DetectorAxis(n_t), AngleAxis(v), line)
    plan = ref_fbp.BstPlan(n_t=n_t, n_theta=v, **plan_kw)
    out = {"counts": counts, "flat": flat, "dark": dark, "eps": np.float64(1e-6), "normalize": line,
           "fbp_bst": ref_fbp.fbp(ys, plan, ref_fbp.FilterPlan(), kernel="bst").data,
           "params": np.array(json.dumps({"plan": plan_kw}))}
    os.makedirs(os.path.join(HERE, "norm"), exist_ok=True)
    np.savez_compressed(os.path.join(HERE, "norm", f"{name}.npz"), **out)
    print(f"{name}: counts {counts.shape} -> {out['fbp_bst'].shape}")


def _proj_case(name, img, n_t, n_ang, full_turn=False, cfg_kw=None):
    """forward_project of an image through the reference (projector.py:94-123)."""
    from tomoblocks import projector as ref_proj
    from tomoblocks.grids import ImageGrid
    cfg_kw = cfg_kw or {}
    img = np.asarray(img, dtype=np.float32)
    y = ref_proj.forward_project(ImageGrid(img.shape[0], img.astype(np.float64)), DetectorAxis(n_t),
                                 AngleAxis(n_ang, full_turn=full_turn), ref_proj.RayTraceConfig(**cfg_kw))
    os.makedirs(os.path.join(HERE, "proj"), exist_ok=True)
    np.savez_compressed(os.path.join(HERE, "proj", f"{name}.npz"), image=img, sino=y.data,
                        params=np.array(json.dumps({"n_t": n_t, "n_angles": n_ang, "full_turn": full_turn,
                                                    "cfg": cfg_kw})))
    print(f"{name}: image {img.shape} -> sino {y.data.shape}")


def _phantom_image(n, rng):
    """Two ellipses plus noise on the n x n pixel-centre grid (input synthesis)."""
    x = -1.0 + (np.arange(n) + 0.5) * 2.0 / n
    u1, u2 = np.meshgrid(x, x)
    img = 1.0 * (((u1 - 0.1) / 0.6) ** 2 + ((u2 + 0.05) / 0.45) ** 2 <= 1.0)
    img += 0.5 * (((u1 + 0.3) / 0.2) ** 2 + ((u2 - 0.2) / 0.3) ** 2 <= 1.0)
    return img + 0.05 * rng.standard_normal((n, n))


def _pre_case(name, y, beta_true, window=9):
    """estimate_center / apply_center / suppress_rings through the reference
    (preprocess.py:88-154) on a sinogram shifted by beta_true bins with
    added detector stripes."""
    from tomoblocks import preprocess as ref_pre
    v, n_t = y.shape
    rng = np.random.default_rng(4)
    shifted = ref_pre.apply_center(Sinogram(DetectorAxis(n_t), AngleAxis(v), y.astype(np.float64)), -beta_true).data
    stripes = 0.05 * rng.standard_normal(n_t)
    sino = (shifted + stripes[None, :]).astype(np.float32)
    ys = Sinogram(DetectorAxis(n_t), AngleAxis(v), sino.astype(np.float64))
    cr = ref_pre.estimate_center(ys)
    centered = ref_pre.apply_center(ys, cr.beta)
    out = {"sino": sino, "beta": np.float64(cr.beta), "confidence": np.float64(cr.confidence),
           "centered": centered.data, "rings": ref_pre.suppress_rings(centered, window).data,
           "rings_raw": ref_pre.suppress_rings(ys, window).data,
           "params": np.array(json.dumps({"beta_true": beta_true, "window": window}))}
    os.makedirs(os.path.join(HERE, "pre"), exist_ok=True)
    np.savez_compressed(os.path.join(HERE, "pre", f"{name}.npz"), **out)
    print(f"{name}: beta {cr.beta:.4f} (true {beta_true}) conf {cr.confidence:.3f}")


def _vol_cases():
    """TOMOVOL1 bytes from the reference writer and blocks from its reader
    (volio.py:96-222) for the container round-trip tests."""
    from tomoblocks import volio as ref_vol
    from tomoblocks.grids import ImageGrid
    d = os.path.join(HERE, "vol")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(5)
    frames = rng.standard_normal((6, 5, 8)).astype(np.float32)  # [angle][slice][det]
    ref_vol.write_volume(os.path.join(d, "frames.tomovol"), ref_vol.VolumeHeader(0, frames.shape), frames)
    slices = np.ascontiguousarray(frames.transpose(1, 0, 2))
    ref_vol.write_volume(os.path.join(d, "slices.tomovol"), ref_vol.VolumeHeader(1, slices.shape), slices)
    with ref_vol.BlockReader(os.path.join(d, "frames.tomovol"), 2) as rd:
        blocks = [np.stack([s.data for s in b.slices]) for b in rd]
    imgs = rng.standard_normal((3, 4, 4))
    with ref_vol.VolumeWriter(os.path.join(d, "written.tomovol"), 3, 4) as wr:
        for k in (2, 0, 1):
            wr.write_slice(k, ImageGrid(4, imgs[k]))
    ref_vol.export_image(ImageGrid(4, imgs[0]), os.path.join(d, "img0.pgm"))
    np.savez_compressed(os.path.join(d, "expect.npz"), frames=frames, imgs=imgs,
                        block0=blocks[0], block1=blocks[1], block2=blocks[2])
    print("vol: frames/slices/written containers")


def main():
    rng0 = np.random.default_rng(0)
    rng1 = np.random.default_rng(1)
    # cfg1: Shepp-Logan 256^2, 256 angles (BASELINE.json configs[0])
    sl = ellipse_sinogram(SHEPP_LOGAN, 256, 256)
    _case("shepp256", sl, {}, ss=True)
    # off-centre ellipse + N(0, 0.05^2) noise (SURVEY.md 8d parity stress)
    el = ellipse_sinogram([(1.0, 0.5, 0.4, 0.1, -0.05, 0.0)], 256, 256)
    _case("ellipse_noise256", el + rng0.normal(0.0, 0.05, el.shape), {})
    # white noise, non power-of-two detector, V != n_t
    _case("white300x180", rng1.normal(0.0, 1.0, (180, 300)), {}, ss=True)
    # output_n != n_t puts the Nyquist lines inside the disc
    _case("outn128", sl, {"output_n": 128})
    # odd output grid (no half-node modulation when n is odd)
    sm = ellipse_sinogram(SHEPP_LOGAN, 65, 33)
    _case("odd65x33_n63", sm, {"output_n": 63}, ss=True)
    # nearest-neighbour gridding
    _case("nearest256", sl, {"interp": "nearest"})
    # apodized ramp, non-default KB window and sigma_min
    _case("apod128", ellipse_sinogram(SHEPP_LOGAN, 128, 96),
          {"kb_beta": 8.0, "kb_support": 0.15, "sigma_min_bins": 2},
          {"kind": "ramp_apodized", "rolloff": 0.7})
    # pad_factor 4: radial transform twice the ramp transform
    _case("pad4_128", ellipse_sinogram(SHEPP_LOGAN, 128, 128), {"pad_factor": 4})
    # full-turn input (2V angles on [0, 2pi)); plan must be explicit
    ft = ellipse_sinogram(SHEPP_LOGAN, 128, 256, full_turn=True)
    _case("fullturn128", ft + rng0.normal(0.0, 0.02, ft.shape), {}, full_turn=True, ss=True)
    # tiny detector
    _case("tiny16x12", rng1.normal(0.0, 1.0, (12, 16)), {}, ss=True)
    # transmission counts through the normalisation prologue
    rng2 = np.random.default_rng(2)
    _norm_case("norm_shepp128", ellipse_sinogram(SHEPP_LOGAN, 128, 128) * 0.5, 1.0e4, 100.0, rng2)
    _norm_case("norm_ellipse256x192", ellipse_sinogram([(1.0, 0.5, 0.4, 0.1, -0.05, 0.0)], 256, 192),
               4.0e3, 50.0, rng2, {"output_n": 200})
    # forward projector: bilinear / nearest / full turn / coarse step
    rng3 = np.random.default_rng(3)
    _proj_case("fp_bilinear64", _phantom_image(64, rng3), 80, 90)
    _proj_case("fp_nearest48", _phantom_image(48, rng3), 50, 36, cfg_kw={"interpolation": "nearest"})
    _proj_case("fp_fullturn40", _phantom_image(40, rng3), 41, 60, full_turn=True, cfg_kw={"step_length": 1.0})
    # centering + ring suppression
    _pre_case("pre_shepp128", ellipse_sinogram(SHEPP_LOGAN, 128, 128), 3.3)
    _pre_case("pre_ellipse200x90", ellipse_sinogram([(1.0, 0.5, 0.4, 0.1, -0.05, 0.0)], 200, 90), -5.75, 7)
    _vol_cases()
    import scipy
    with open(os.path.join(HERE, "versions.json"), "w") as f:
        json.dump({"numpy": np.__version__, "scipy": scipy.__version__,
                   "reference": "tomoblocks (/root/reference/pkg)"}, f, indent=1)


if __name__ == "__main__":
    main()
