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
