"""Reentrancy and edge cases of the device path (SURVEY.md §8b "Threading":
one plan shared by concurrent callers on separate streams with separate
workspaces, like the reference's cfg.workers threads sharing one BstPlan,
pipeline.py:424-431, 511-518; empty volumes)."""
import threading

import pytest
import torch

pytestmark = pytest.mark.gpu


def _F():
    from paper_1704_08364_b200 import fourier_bp as F
    return F


def test_empty_volume_device_and_host():
    F = _F()
    plan = F.BstPlan(64, 48)
    dev = F.fbp_volume(torch.empty((0, 48, 64), device="cuda"), plan)
    assert dev.shape == (0, 64, 64) and dev.is_cuda
    host = F.fbp_volume(torch.empty((0, 48, 64)), plan, devices=[0])
    assert host.shape == (0, 64, 64) and not host.is_cuda


def test_concurrent_streams_share_one_plan():
    F = _F()
    from paper_1704_08364_b200 import phantom
    plan = F.BstPlan(256, 192)
    base = phantom.ellipsoid_volume(5, 256, 192, device="cuda")
    g = torch.Generator("cuda").manual_seed(11)
    vols = [base + 0.05 * k * torch.randn(base.shape, device="cuda", generator=g) for k in range(4)]
    torch.cuda.synchronize()
    serial = [F.fbp_volume(v, plan, batch=2) for v in vols]
    torch.cuda.synchronize()
    results, errors = [None] * len(vols), []

    def worker(k):
        try:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.default_stream())
            with torch.cuda.stream(s):
                for _ in range(3):
                    results[k] = F.fbp_volume(vols[k], plan, batch=2)
            s.synchronize()
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(vols))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for a, b in zip(serial, results):
        assert torch.equal(a, b)


def test_single_slice_api_equals_volume_slice():
    F = _F()
    import numpy as np
    from paper_1704_08364_b200 import phantom
    from paper_1704_08364_b200.slices import AngleAxis, DetectorAxis, Sinogram
    vol = phantom.ellipsoid_volume(3, 128, 128, device="cuda")
    plan = F.BstPlan(128, 128)
    v = F.fbp_volume(vol, plan)
    y = Sinogram(DetectorAxis(128), AngleAxis(128), vol[1].cpu().numpy().astype(np.float64))
    img = F.fbp(y, plan)
    assert np.array_equal(np.asarray(img.data, dtype=np.float32), v[1].cpu().numpy())


def test_plain_gather_path_matches_texture_path():
    """A launch group whose polar rows exceed the pitch-2D texture height
    (batch * (n_theta + 1) > 65000) gathers with plain loads instead of TLD4.
    Both read the same fp32 texels; the TLD4 path's weights come from the
    fp32 half-plane table, the plain path's from the unorm16 first-quadrant
    table (<= 2^-17 weight error), so they agree to ~1e-6, not bitwise."""
    F = _F()
    from paper_1704_08364_b200 import phantom
    plan = F.BstPlan(64, 2048)
    vol = phantom.ellipsoid_volume(40, 64, 2048, device="cuda")
    vol += 0.01 * torch.randn(vol.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    tex = F.fbp_volume(vol, plan, batch=1)     # 2049 rows: texture gathers
    plain = F.fbp_volume(vol, plan, batch=40)  # 81960 rows: plain loads
    rel = (torch.linalg.norm(tex - plain) / torch.linalg.norm(tex)).item()
    assert rel < 5e-6, rel


def test_odd_full_turn_bst_raises_value_error_and_ss_works():
    """Full-turn input with an odd angle count: the reference's BST path
    rejects it with ValueError (fourier_bp.py:331-332, 446-448); its slant
    stack handles any count (projector.py:126-158)."""
    import numpy as np
    from oracle import bst_oracle as O
    from paper_1704_08364_b200 import projector
    from paper_1704_08364_b200.slices import AngleAxis, DetectorAxis, Sinogram
    F = _F()
    rng = np.random.default_rng(3)
    n_t, A = 64, 63
    data = O.ellipse_sinogram(O.SHEPP_LOGAN, n_t, A, full_turn=True) + rng.normal(0, 0.01, (A, n_t))
    y = Sinogram(DetectorAxis(n_t), AngleAxis(A, full_turn=True), data)
    with pytest.raises(ValueError):
        F.fbp(y)
    with pytest.raises(ValueError):
        F.fbp(y, F.BstPlan(n_t, A // 2))
    with pytest.raises(ValueError):
        F.bst_backproject(y, F.BstPlan(n_t, A // 2))
    got = F.fbp(y, F.BstPlan(n_t, A // 2), kernel="ss").data
    ref = O.fbp(data, O.OraclePlan(n_t, A // 2), "ss", full_turn=True)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5
    bp = projector.backproject_ss(y, 48).data
    ref2 = O.backproject_ss(data, 48, full_turn=True)
    assert np.linalg.norm(bp - ref2) / np.linalg.norm(ref2) < 1e-5


def test_table_free_plan_rejects_bst_calls():
    F = _F()
    nat = F.aux_plan(64, 64)
    sino = torch.zeros((1, 64, 64), device="cuda")
    img = torch.empty((1, 64, 64), device="cuda")
    ws = nat.new_workspace(1)
    with pytest.raises(ValueError, match="gridding tables"):
        nat.run("fbp", sino, img, 1, 1, ws)


def test_plan_dropped_with_work_in_flight():
    """fbp_volume(check=False) returns with kernels queued; dropping the last
    reference to its plan destroys it, which must wait for those kernels
    (tb_plan_destroy drains the device) -- the result stays exact."""
    import gc
    F = _F()
    from paper_1704_08364_b200 import phantom
    vol = phantom.ellipsoid_volume(8, 256, 256, device="cuda")
    ref = F.fbp_volume(vol, F.BstPlan(256, 256))
    for _ in range(3):
        out = F.fbp_volume(vol, F.BstPlan(256, 256), check=False)  # plan=None path builds a fresh plan
        gc.collect()
        assert torch.equal(out, ref)


def test_backproject_stage_scale_rides_in_the_kernel():
    F = _F()
    from paper_1704_08364_b200 import phantom
    vol = phantom.ellipsoid_volume(2, 128, 128, device="cuda")
    plan = F.BstPlan(128, 128)
    raw = F.fbp_volume(vol, plan, kernel="none")
    scaled = F.fbp_volume(vol, plan, kernel="none", scale=F.FBP_SCALE)
    assert torch.allclose(scaled, raw * F.FBP_SCALE, rtol=2e-6, atol=1e-7)
