"""Centering and ring suppression (preprocess.py:88-154)
against golden vectors produced by the real reference
(tests/golden/make_golden.py -> tests/golden/pre/*.npz)."""
import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN_DIR, rel_l2, max_rel
from oracle import bst_oracle as O

PRE_DIR = os.path.join(GOLDEN_DIR, "pre")
PRE_CASES = sorted(f[:-4] for f in os.listdir(PRE_DIR) if f.endswith(".npz"))


def _load(name):
    z = np.load(os.path.join(PRE_DIR, name + ".npz"))
    d = {k: z[k] for k in z.files}
    d["params"] = json.loads(str(d["params"]))
    return d


@pytest.mark.parametrize("name", PRE_CASES)
def test_oracle_preprocessing_matches_reference(name):
    c = _load(name)
    y = c["sino"].astype(np.float64)
    beta, conf = O.estimate_center(y)
    assert abs(beta - c["beta"]) <= 1e-12 and abs(conf - c["confidence"]) <= 1e-12
    cen = O.apply_center(y, beta)
    assert np.max(np.abs(cen - c["centered"])) <= 1e-12
    w = c["params"]["window"]
    assert np.max(np.abs(O.suppress_rings(cen, w) - c["rings"])) <= 1e-12
    assert np.max(np.abs(O.suppress_rings(y, w) - c["rings_raw"])) <= 1e-12


def test_validation_mirrors_reference():
    from paper_1704_08364_b200.preprocess import CenteringError, apply_center, estimate_center, suppress_rings
    from paper_1704_08364_b200.slices import AngleAxis, DetectorAxis, Sinogram
    y = Sinogram(DetectorAxis(8), AngleAxis(1), np.zeros((1, 8)))
    with pytest.raises(CenteringError, match="need at least two projection angles"):
        estimate_center(y)
    with pytest.raises(ValueError, match="window must be an odd integer"):
        suppress_rings(y, 4)
    with pytest.raises(ValueError, match="exceeds the detector extent"):
        apply_center(y, 9.0)
    assert issubclass(CenteringError, ValueError)


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _sino(c):
    from paper_1704_08364_b200.slices import AngleAxis, DetectorAxis, Sinogram
    v, n_t = c["sino"].shape
    return Sinogram(DetectorAxis(n_t), AngleAxis(v), c["sino"].astype(np.float64))


@pytest.mark.gpu
@pytest.mark.parametrize("name", PRE_CASES)
def test_gpu_center_and_rings_match_reference(name):
    _cuda()
    from paper_1704_08364_b200.preprocess import apply_center, estimate_center, suppress_rings
    c = _load(name)
    y = _sino(c)
    cr = estimate_center(y)  # fp64 on fp32-exact data: same correlation peak
    assert abs(cr.beta - c["beta"]) <= 1e-9 and abs(cr.confidence - c["confidence"]) <= 1e-9
    cen = apply_center(y, cr.beta)
    assert max_rel(cen.data, c["centered"]) <= 1e-6
    w = c["params"]["window"]
    assert max_rel(suppress_rings(y, w).data, c["rings_raw"]) <= 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("name", PRE_CASES)
def test_gpu_volume_pipeline_center_rings_fbp(name):
    torch = _cuda()
    from paper_1704_08364_b200 import fourier_bp as F
    from paper_1704_08364_b200.preprocess import preprocess_volume
    c = _load(name)
    v, n_t = c["sino"].shape
    w = c["params"]["window"]
    plan = F.BstPlan(n_t=n_t, n_theta=v)
    vol = torch.from_numpy(c["sino"])[None].repeat(2, 1, 1).cuda()
    pre = preprocess_volume(vol, plan, center="auto", rings=w)
    for k in range(2):
        assert max_rel(pre[k].cpu().numpy(), c["rings"]) <= 1e-6
    img = F.fbp_volume(vol, plan, center="auto", rings=w)
    ref = O.fbp(c["rings"], O.OraclePlan(n_t, v))
    got = img[1].cpu().numpy()
    assert rel_l2(got, ref) <= 1e-4 and max_rel(got, ref) <= 1e-3


@pytest.mark.gpu
def test_gpu_constant_sinogram_raises_centering_error():
    torch = _cuda()
    from paper_1704_08364_b200 import fourier_bp as F
    from paper_1704_08364_b200.preprocess import CenteringError
    vol = torch.full((2, 16, 32), 3.0, device="cuda")
    with pytest.raises(CenteringError, match="constant sinogram"):
        F.fbp_volume(vol, F.BstPlan(32, 16), center="auto")


@pytest.mark.gpu
@pytest.mark.parametrize("center,rings", [("auto", 9), (3.25, None), (None, 5), (-7.5, 11)])
def test_gpu_fused_center_rings_equal_separate_passes(center, rings):
    """fbp_volume with the centre / ring stages fused into K1's row load
    (tb_fbp_pre) against the separate device passes (preprocess_volume, then
    fbp) on a 6-slice 512^2 volume over three launch groups."""
    torch = _cuda()
    from paper_1704_08364_b200 import fourier_bp as F
    from paper_1704_08364_b200 import phantom
    from paper_1704_08364_b200.preprocess import preprocess_volume
    N = 512
    plan = F.BstPlan(N, N)
    vol = phantom.ellipsoid_volume(6, N, N, device="cuda")
    g = torch.Generator("cuda").manual_seed(2)
    vol += 0.02 * torch.randn(vol.shape, device="cuda", generator=g)
    vol += 0.05 * torch.rand((1, 1, N), device="cuda", generator=g)  # detector stripes
    vol = torch.roll(vol, 3, dims=2)
    fused = F.fbp_volume(vol, plan, center=center, rings=rings, batch=2)
    sep = F.fbp_volume(preprocess_volume(vol, plan, center=center, rings=rings), plan, batch=2)
    for k in range(6):
        d = (torch.linalg.norm(fused[k] - sep[k]) / torch.linalg.norm(sep[k])).item()
        assert d < 1e-5, (k, d)


@pytest.mark.gpu
def test_gpu_fused_stages_fall_back_when_the_ramp_is_not_fused():
    """A plan whose ramp is a separate pass (pad_factor 4: npad != L) takes
    the separate preprocessing passes: same result as doing them by hand."""
    torch = _cuda()
    from paper_1704_08364_b200 import fourier_bp as F
    from paper_1704_08364_b200 import phantom
    from paper_1704_08364_b200.preprocess import preprocess_volume
    plan = F.BstPlan(128, 128, pad_factor=4)
    vol = phantom.ellipsoid_volume(2, 128, 128, device="cuda")
    g = torch.Generator("cuda").manual_seed(4)
    vol += 0.05 * torch.rand(vol.shape, device="cuda", generator=g)
    a = F.fbp_volume(vol, plan, center=2.5, rings=5)
    b = F.fbp_volume(preprocess_volume(vol, plan, center=2.5, rings=5), plan)
    assert torch.equal(a, b)
