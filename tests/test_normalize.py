"""Normalisation prologue: -ln(max(I - D, eps) /
max(I0 - D, eps)) (preprocess.py:59-74), alone and fused into the radial
kernel, against golden vectors produced by the real reference
(tests/golden/make_golden.py, tests/golden/norm/*.npz)."""
import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN_DIR, rel_l2, max_rel
from oracle import bst_oracle as O

NORM_DIR = os.path.join(GOLDEN_DIR, "norm")
NORM_CASES = sorted(f[:-4] for f in os.listdir(NORM_DIR) if f.endswith(".npz"))


def _load(name):
    z = np.load(os.path.join(NORM_DIR, name + ".npz"))
    d = {k: z[k] for k in z.files}
    d["params"] = json.loads(str(d["params"]))
    return d


@pytest.mark.parametrize("name", NORM_CASES)
def test_oracle_normalize_matches_reference(name):
    c = _load(name)
    got = O.normalize(c["counts"], c["flat"], c["dark"], float(c["eps"]))
    assert np.max(np.abs(got - c["normalize"])) <= 1e-12 * np.max(np.abs(c["normalize"]))


def test_frames_and_eps_validation_mirror_reference():
    from paper_1704_08364_b200.preprocess import FlatDarkFrames, normalize
    with pytest.raises(ValueError, match="flat/dark shapes differ"):
        FlatDarkFrames(flat=np.ones((2, 3)), dark=np.ones((3, 2)))
    fr = FlatDarkFrames(flat=np.ones((2, 3)), dark=np.zeros((2, 3)))
    with pytest.raises(ValueError, match="eps must be positive"):
        normalize(np.ones((2, 3)), fr, eps=0.0)
    with pytest.raises(ValueError, match="does not match frames"):
        normalize(np.ones((3, 3)), fr)


# --- GPU ------------------------------------------------------------------------

def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("name", NORM_CASES)
def test_gpu_normalize_matches_reference(name):
    _cuda()
    from paper_1704_08364_b200.preprocess import FlatDarkFrames, normalize
    c = _load(name)
    got = normalize(c["counts"], FlatDarkFrames(c["flat"], c["dark"]), float(c["eps"]))
    ref = c["normalize"]
    assert rel_l2(got, ref) <= 2e-6 and np.max(np.abs(got - ref)) <= 2e-5


@pytest.mark.gpu
@pytest.mark.parametrize("name", NORM_CASES)
def test_gpu_fused_counts_fbp_matches_reference(name):
    torch = _cuda()
    from paper_1704_08364_b200 import fourier_bp as F
    from paper_1704_08364_b200.preprocess import FlatDarkFrames
    c = _load(name)
    v, n_t = c["counts"].shape
    plan = F.BstPlan(n_t=n_t, n_theta=v, **c["params"]["plan"])
    frames = FlatDarkFrames(c["flat"], c["dark"])
    counts = torch.from_numpy(c["counts"])[None].repeat(3, 1, 1)
    dev = F.fbp_volume(counts.cuda(), plan, frames=frames, eps=float(c["eps"]))
    for k in range(3):
        got = dev[k].cpu().numpy()
        assert rel_l2(got, c["fbp_bst"]) <= 1e-4 and max_rel(got, c["fbp_bst"]) <= 1e-3
    # host-resident counts through the pinned pipeline: same kernels, bitwise
    host = F.fbp_volume(counts, plan, frames=frames, eps=float(c["eps"]), devices=[0])
    assert torch.equal(host, dev.cpu())
    # fused prologue == separate normalize pass + fbp (same fp32 line integrals)
    line = torch.empty_like(counts.cuda())
    nat = F.native_plan(plan, F.FilterPlan(), False, 0)
    fl, dk = F._frames_on(frames, 0, v, n_t)
    nat.normalize(counts.cuda(), fl, dk, float(c["eps"]), line, 3)
    two = F.fbp_volume(line, plan)
    assert (torch.linalg.norm(two - dev) / torch.linalg.norm(two)).item() <= 1e-6


@pytest.mark.gpu
def test_gpu_counts_nonfinite_raises():
    torch = _cuda()
    from paper_1704_08364_b200 import fourier_bp as F
    from paper_1704_08364_b200.preprocess import FlatDarkFrames
    c = _load(NORM_CASES[0])
    v, n_t = c["counts"].shape
    counts = torch.from_numpy(c["counts"].copy())[None].cuda()
    counts[0, 7, 9] = float("nan")
    with pytest.raises(ValueError):
        F.fbp_volume(counts, F.BstPlan(n_t, v), frames=FlatDarkFrames(c["flat"], c["dark"]))


@pytest.mark.gpu
def test_gpu_constant_frames_scalar_path_matches_table_path():
    """Constant frames (the reference pipeline's i0 / dark scalars) take the
    table-free kernel path; it equals the per-sample table path."""
    torch = _cuda()
    from paper_1704_08364_b200 import fourier_bp as F
    from paper_1704_08364_b200.preprocess import FlatDarkFrames
    rng = np.random.default_rng(9)
    v, n_t = 96, 128
    counts = torch.from_numpy((1e4 * np.exp(-rng.random((2, v, n_t))) + 100.0).astype(np.float32)).cuda()
    plan = F.BstPlan(n_t, v)
    const = FlatDarkFrames(np.full((v, n_t), 1e4 + 100.0), np.full((v, n_t), 100.0))
    a = F.fbp_volume(counts, plan, frames=const)
    nat = F.native_plan(plan, F.FilterPlan(), False, 0)
    fl, dk = F._frames_on(const, 0, v, n_t)
    b = torch.empty_like(a)
    ws = nat.new_workspace(2)
    nat.run_counts(counts, fl, dk, 1e-6, b, 2, 2, ws)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
