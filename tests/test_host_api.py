"""Host-side API mirror (no GPU): plan/filter validation and defaults,
containers, Q-block descriptors, StageSpec checks, slab partitioning."""
import numpy as np
import pytest

from paper_1704_08364_b200 import grids
from paper_1704_08364_b200.fourier_bp import BstPlan, FilterPlan, FBP_SCALE, _split, default_batch
from paper_1704_08364_b200.pipeline import StageSpec, block_descriptors


def test_bstplan_defaults_and_geometry():
    p = BstPlan(256, 180)
    assert p.radial_samples == 512 and p.output_n == 256
    assert p.roll == 128 and p.delta_t == 2.0 / 255
    p2 = BstPlan(300, 10)
    assert p2.radial_samples == 1024 and p2.roll == int(round(299 / 2.0))
    assert p2.amplitude_scale == pytest.approx((p2.delta_nu * 1024) ** 2 * p2.delta_t)
    assert FBP_SCALE == pytest.approx(1 / (2 * np.pi))


@pytest.mark.parametrize("kw", [dict(n_t=1, n_theta=4), dict(n_t=8, n_theta=0), dict(n_t=8, n_theta=4, pad_factor=1),
                                dict(n_t=8, n_theta=4, sigma_min_bins=0), dict(n_t=8, n_theta=4, interp="cubic"),
                                dict(n_t=8, n_theta=4, radial_samples=24), dict(n_t=8, n_theta=4, output_n=99)])
def test_bstplan_validation(kw):
    with pytest.raises(ValueError):
        BstPlan(**kw)


def test_filterplan():
    assert FilterPlan().effective_rolloff == 1.0
    assert FilterPlan("ramp_apodized", 0.5).effective_rolloff == 0.5
    assert FilterPlan("ramp", 0.5).effective_rolloff == 1.0
    with pytest.raises(ValueError):
        FilterPlan("hann")
    with pytest.raises(ValueError):
        FilterPlan(rolloff=0.0)


def test_containers_match_reference_conventions():
    d = grids.DetectorAxis(5)
    assert d.coordinate(3) == 0.5 and d.samples[0] == -1.0 and d.samples[-1] == 1.0
    g = grids.ImageGrid(3, np.zeros((3, 3)))
    assert grids.pixel_center(g, 1, 1) == (0.0, 0.0)
    assert grids.pixel_center(grids.ImageGrid(2, np.zeros((2, 2))), 0, 0) == (-0.5, -0.5)
    a = grids.AngleAxis(4)
    assert np.allclose(a.angles, np.arange(4) * np.pi / 4)
    with pytest.raises(ValueError):
        grids.Sinogram(d, a, np.full((4, 5), np.nan))
    with pytest.raises(ValueError):
        grids.Sinogram(d, a, np.zeros((5, 4)))
    s = grids.Sinogram(d, a, np.ones((4, 5)))
    assert not s.data.flags.writeable
    with pytest.raises(ValueError):
        grids.VolumeBlock(0, [], grids.StageKind.READ)


def test_block_descriptors_and_stagespec():
    assert block_descriptors(10, 4) == [(0, 4), (4, 4), (8, 2)]
    with pytest.raises(ValueError):
        StageSpec("x", 0, 1, lambda b: b)
    with pytest.raises(ValueError):
        StageSpec("x", 1, 0, lambda b: b)


def test_slab_split_covers_volume():
    for n, parts in [(2048, 8), (7, 3), (2, 4)]:
        sl = _split(n, parts)
        assert sl[0][0] == 0 and sl[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
        sizes = [e - b for b, e in sl]
        assert max(sizes) - min(sizes) <= 1


def test_default_batch():
    assert default_batch(BstPlan(2048, 2048)) >= 1
    assert default_batch(BstPlan(256, 256)) > default_batch(BstPlan(1024, 1024))


@pytest.mark.parametrize("out,msg", [
    ("torch.empty((2, 8, 8))", "shape"),
    ("torch.empty((3, 8, 8), dtype=torch.float64)", "float32"),
    ("torch.empty((3, 8, 16))[:, :, ::2]", "contiguous"),
    ("[[0.0]]", "torch.Tensor"),
])
def test_fbp_volume_rejects_bad_out_before_any_device_work(out, msg):
    """The kernels write through a raw pointer: a wrong out must raise
    ValueError up front (no device needed to see it)."""
    import torch
    from paper_1704_08364_b200.fourier_bp import fbp_volume
    sino = torch.zeros((3, 8, 8))
    with pytest.raises(ValueError, match=msg):
        fbp_volume(sino, BstPlan(8, 8), out=eval(out))


def test_fbp_volume_scale_only_for_unfiltered_kernel():
    import torch
    from paper_1704_08364_b200.fourier_bp import fbp_volume
    with pytest.raises(ValueError, match="scale"):
        fbp_volume(torch.zeros((1, 8, 8)), BstPlan(8, 8), kernel="bst", scale=2.0)
