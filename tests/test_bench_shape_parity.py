"""Parity at the benchmark's real execution shape, the plugin-stage contract
and the multi-device orchestration (GPU).

* bench shape: ``fbp_volume`` on device-resident volumes with the DEFAULT
  launch-group size (31 slices at 2048, 63 at 1024, 64 at 512) on two
  lanes, i.e. the texture heights, lane-1 workspace regions and slice
  offsets inside the TLD4 row coordinate that ``bench.py`` exercises;
  slices at the group boundaries are compared with the CPU oracle
  (BASELINE north_star tolerance: rel-L2 <= 1e-4, max-abs <= 1e-3 max|ref|).
* plugin stages: ``make_fbp_stage(...).process(VolumeBlock)`` and friends,
  called exactly as the reference runtime calls ``spec.process(payload)``
  (pipeline.py:275) on Q-blocks (pipeline.py:395-400, 486-518).
* fake multi-GPU: the host slab pipeline with
  ``devices=[0, 0]`` (two slabs, two plan/stream sets on one GPU) is bitwise
  equal to ``devices=[0]``.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_util import rel_l2, max_rel  # noqa: E402
from oracle import bst_oracle as O  # noqa: E402

REL_L2_TOL = 1e-4
MAX_ABS_TOL = 1e-3


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _F():
    from paper_1704_08364_b200 import fourier_bp as F
    return F


def _assert_close(got, ref):
    r, m = rel_l2(got, ref), max_rel(got, ref)
    assert r <= REL_L2_TOL and m <= MAX_ABS_TOL, f"rel_l2={r:.3e} max_abs/max={m:.3e}"


def _noisy_volume(S, N, seed):
    from paper_1704_08364_b200 import phantom
    vol = phantom.ellipsoid_volume(S, N, N, device="cuda")
    g = torch.Generator("cuda").manual_seed(seed)
    vol += 0.05 * torch.randn(vol.shape, device="cuda", generator=g)
    return vol


@pytest.mark.parametrize("N,S,batch,check", [
    (2048, 64, 31, (0, 30, 31, 63)),     # groups 31 + 31 + 2 on 2 lanes; last group on lane 0
    (1024, 128, 63, (0, 62, 63, 127)),   # groups 63 + 63 + 2
    (512, 130, 64, (0, 63, 64, 129)),    # groups 64 + 64 + 2
])
def test_bench_shape_volume_against_oracle(N, S, batch, check):
    F = _F()
    plan = F.BstPlan(N, N)
    assert F.default_batch(plan) == batch  # the shape bench.py runs
    vol = _noisy_volume(S, N, seed=N)
    out = F.fbp_volume(vol, plan)  # default batch, two lanes
    op = O.OraclePlan(N, N)
    for k in check:
        ref = O.fbp(vol[k].cpu().numpy().astype(np.float64), op)
        _assert_close(out[k].cpu().numpy(), ref)
    # lanes and launch groups do not change any slice: bitwise equal to
    # single-slice groups on one lane
    one = F.fbp_volume(vol[:3].contiguous(), plan, batch=1)
    assert torch.equal(one, out[:3])


def test_devices_0_0_slabs_bitwise_equal_one_device():
    F = _F()
    vol = _noisy_volume(21, 256, seed=7).cpu()
    plan = F.BstPlan(256, 256)
    a = F.fbp_volume(vol, plan, devices=[0])
    b = F.fbp_volume(vol, plan, devices=[0, 0], chunk=4)
    assert not a.is_cuda and not b.is_cuda
    assert torch.equal(a, b)


def _block(vol, first, full_turn=False):
    from paper_1704_08364_b200.slices import AngleAxis, DetectorAxis, Sinogram, StageKind, VolumeBlock
    host = vol.cpu().numpy().astype(np.float64)
    S, A, n_t = host.shape
    sl = [Sinogram(DetectorAxis(n_t), AngleAxis(A, full_turn=full_turn), host[i]) for i in range(S)]
    return VolumeBlock(first, sl, StageKind.FILTER), host


def test_fbp_stage_process_volume_block_against_oracle():
    from paper_1704_08364_b200 import pipeline as P
    from paper_1704_08364_b200.slices import ImageGrid, StageKind
    F = _F()
    vol = _noisy_volume(5, 256, seed=11)
    blk, host = _block(vol, first=40)
    spec = P.make_fbp_stage(F.BstPlan(256, 256), workers=2, queue_capacity=3)
    assert spec.name == "backproject" and spec.workers == 2 and spec.queue_capacity == 3
    out = spec.process(blk)
    assert out.first_slice == 40 and out.stage_tag == StageKind.BACKPROJECT and len(out) == 5
    op = O.OraclePlan(256, 256)
    for i, img in enumerate(out.slices):
        assert isinstance(img, ImageGrid) and img.data.dtype == np.float64
        _assert_close(img.data, O.fbp(host[i], op))


def test_filter_then_backproject_stages_against_oracle():
    """The reference's two-stage form (pipeline.py:489-518): filter stage,
    then backproject stage x FBP_SCALE."""
    from paper_1704_08364_b200 import pipeline as P
    from paper_1704_08364_b200.slices import StageKind
    F = _F()
    vol = _noisy_volume(3, 128, seed=12)
    blk, host = _block(vol, first=0)
    plan = F.BstPlan(128, 128)
    op = O.OraclePlan(128, 128)
    filt = P.make_filter_stage().process(blk)
    assert filt.stage_tag == StageKind.FILTER
    for i, s in enumerate(filt.slices):
        _assert_close(s.data, O.ramp_filter(host[i], op))
    bp = P.make_backproject_stage(plan).process(filt)
    assert bp.stage_tag == StageKind.BACKPROJECT
    for i, img in enumerate(bp.slices):
        ref = O.bst_backproject(np.asarray(filt.slices[i].data), op) * O.FBP_SCALE
        _assert_close(img.data, ref)
    # unscaled backprojection (bst_backproject semantics)
    raw = P.make_backproject_stage(plan, scale=1.0).process(filt)
    _assert_close(raw.slices[1].data, O.bst_backproject(np.asarray(filt.slices[1].data), op))


def test_fbp_stage_ss_kernel_against_oracle():
    from paper_1704_08364_b200 import pipeline as P
    F = _F()
    vol = _noisy_volume(2, 96, seed=13)
    blk, host = _block(vol, first=2)
    out = P.make_fbp_stage(F.BstPlan(96, 96), kernel="ss").process(blk)
    for i, img in enumerate(out.slices):
        _assert_close(img.data, O.fbp(host[i], O.OraclePlan(96, 96), kernel="ss"))


def test_device_resident_slabs_over_devices_0_0_bitwise():
    """The device-resident multi-GPU path (slabs, per-slab stream and
    workspace, gather into the output on the input's GPU) on a fake
    two-device list: bitwise equal to the single-device call."""
    F = _F()
    vol = _noisy_volume(23, 256, seed=21)
    plan = F.BstPlan(256, 256)
    ref = F.fbp_volume(vol, plan, batch=4)
    out = F.fbp_volume(vol, plan, batch=4, devices=[0, 0])
    assert out.is_cuda and torch.equal(out, ref)
    three = F.fbp_volume(vol, plan, batch=5, devices=[0, 0, 0], kernel="none", scale=0.25)
    assert torch.equal(three, F.fbp_volume(vol, plan, batch=5, kernel="none", scale=0.25))


@pytest.mark.parametrize("N,S,batch", [(4096 // 2, 40, 12), (1024, 20, 6)])
def test_fused_schedule_bitwise_equals_per_group_launches(N, S, batch, monkeypatch):
    """TB_FUSE=2 (K2(g) + K1(g+1) + K3(g-1) in one grid, where it applies:
    L = 4096 / 8192), TB_FUSE=1 (K2 + K1) and TB_FUSE=0 (separate launches
    per group on two lanes, the default) run the same kernel bodies on the
    same data: bitwise equal outputs, including a short last group."""
    F = _F()
    plan = F.BstPlan(N, N)
    vol = _noisy_volume(S, N, seed=31)
    outs = {}
    for mode in ("0", "1", "2"):
        monkeypatch.setenv("TB_FUSE", mode)
        outs[mode] = F.fbp_volume(vol, plan, batch=batch)
    assert torch.equal(outs["0"], outs["1"]) and torch.equal(outs["0"], outs["2"])
    if N == 2048:
        ref = O.fbp(vol[S - 1].cpu().numpy().astype(np.float64), O.OraclePlan(N, N))
        _assert_close(outs["2"][S - 1].cpu().numpy(), ref)


def test_full_turn_texture_path_against_oracle_and_lattice_path(monkeypatch):
    """Full-turn input (2V rows over 2 pi) on the TLD4 path K2_TEXF: launch
    groups of 8 on two lanes (texture rows 8 (2V + 1) per lane), slices
    against the oracle, and the whole volume against the per-node
    lattice_value path (TB_NOTEX=1: no texture view -> K2_ANY), whose
    unorm16 table fractions carry up to 2^-17 weight error (measured
    difference 3.9e-6)."""
    F = _F()
    N, S = 512, 20
    plan = F.BstPlan(N, N)
    assert F.default_batch(plan, full_turn=True) == 65000 // (2 * N + 1)
    ell = O.ellipse_sinogram(O.SHEPP_LOGAN, N, 2 * N, full_turn=True)
    g = torch.Generator("cuda").manual_seed(5)
    vol = torch.from_numpy(ell.astype(np.float32)).cuda().expand(S, -1, -1).contiguous()
    vol += 0.05 * torch.randn(vol.shape, device="cuda", generator=g)
    out = F.fbp_volume(vol, plan, full_turn=True, batch=8)
    op = O.OraclePlan(N, N)
    for k in (0, 7, 8, 19):
        ref = O.fbp(vol[k].cpu().numpy().astype(np.float64), op, full_turn=True)
        _assert_close(out[k].cpu().numpy(), ref)
    monkeypatch.setenv("TB_NOTEX", "1")
    lat = F.fbp_volume(vol, plan, full_turn=True, batch=8)
    d = (torch.linalg.norm(lat - out) / torch.linalg.norm(lat)).item()
    assert d < 2e-5, d


def test_nearest_texture_path_against_oracle_and_lattice_path(monkeypatch):
    """interp="nearest" on the point-sampled texture path K2_TEXN (rounded
    indices decided in fp64 at plan time, the mirror node's own rounded row):
    three launch groups against the oracle, and against the lattice_value
    path (TB_NOTEX=1 -> K2_ANY)."""
    F = _F()
    N, S = 512, 20
    plan = F.BstPlan(N, N, interp="nearest")
    vol = _noisy_volume(S, N, seed=9)
    out = F.fbp_volume(vol, plan, batch=8)
    op = O.OraclePlan(N, N, interp="nearest")
    for k in (0, 7, 8, 19):
        ref = O.fbp(vol[k].cpu().numpy().astype(np.float64), op)
        _assert_close(out[k].cpu().numpy(), ref)
    monkeypatch.setenv("TB_NOTEX", "1")
    lat = F.fbp_volume(vol, plan, batch=8)
    d = (torch.linalg.norm(lat - out) / torch.linalg.norm(lat)).item()
    assert d < 2e-6, d


@pytest.mark.parametrize("n_t,V,full,interp,out_n,pad", [
    (128, 96, True, "bilinear", 100, 2),     # K2_TEXF without the half crop (per-node modulation)
    (65, 33, True, "bilinear", 63, 2),       # odd sizes, full turn
    (128, 96, False, "nearest", 100, 2),     # K2_TEXN without the half crop
    (65, 33, False, "nearest", 63, 2),       # odd sizes, nearest
    (64, 48, True, "bilinear", None, 4),     # full turn, separate ramp pass (npad != L)
    (64, 48, False, "nearest", None, 4),     # nearest, separate ramp pass
])
def test_texture_paths_edge_shapes_against_oracle(n_t, V, full, interp, out_n, pad):
    """The round-2 texture paths on shapes off the benchmark's: no n = L/2
    crop (modulation per node instead of fft_mod), odd sizes, pad_factor 4,
    three slices in launch groups of 2."""
    F = _F()
    plan = F.BstPlan(n_t, V, interp=interp, output_n=out_n, pad_factor=pad)
    A = 2 * V if full else V
    g = torch.Generator("cuda").manual_seed(n_t + V)
    ell = O.ellipse_sinogram(O.SHEPP_LOGAN, n_t, A, full_turn=full)
    vol = torch.from_numpy(ell.astype(np.float32)).cuda().expand(3, -1, -1).contiguous()
    vol += 0.05 * torch.randn(vol.shape, device="cuda", generator=g)
    out = F.fbp_volume(vol, plan, full_turn=full, batch=2)
    op = O.OraclePlan(n_t, V, interp=interp, output_n=out_n, pad_factor=pad)
    for k in range(3):
        ref = O.fbp(vol[k].cpu().numpy().astype(np.float64), op, full_turn=full)
        _assert_close(out[k].cpu().numpy(), ref)


@pytest.mark.parametrize("center", ["auto", 2.5])
def test_fbp_stage_with_center_and_rings_against_oracle(center):
    """make_fbp_stage taking over the reference pipeline's center and rings
    stages too (pipeline.py:461-518): the oracle runs estimate_center /
    apply_center, suppress_rings, then fbp per slice."""
    from paper_1704_08364_b200 import pipeline as P
    F = _F()
    vol = _noisy_volume(4, 128, seed=21)
    vol = torch.roll(vol, 2, dims=2).contiguous()
    blk, host = _block(vol, first=7)
    spec = P.make_fbp_stage(F.BstPlan(128, 128), center=center, rings=9)
    out = spec.process(blk)
    op = O.OraclePlan(128, 128)
    for i, img in enumerate(out.slices):
        beta = O.estimate_center(host[i])[0] if center == "auto" else center
        pre = O.suppress_rings(O.apply_center(host[i], beta), 9)
        _assert_close(img.data, O.fbp(pre, op))


@pytest.mark.parametrize("full,interp", [(True, "bilinear"), (False, "nearest")])
def test_texture_paths_at_2048_against_oracle(full, interp):
    """K2_TEXF / K2_TEXN at the headline size (L = 4096, the 5-CTA kernels,
    thread-0 mirror bookkeeping at 256 threads per column): the last slice
    of a 17-slice volume (two launch groups for full turn) vs the oracle."""
    F = _F()
    N, S = 2048, 17
    plan = F.BstPlan(N, N, interp=interp)
    A = 2 * N if full else N
    g = torch.Generator("cuda").manual_seed(17)
    vol = torch.randn((S, A, N), device="cuda", generator=g)
    out = F.fbp_volume(vol, plan, full_turn=full)
    ref = O.fbp(vol[S - 1].cpu().numpy().astype(np.float64), O.OraclePlan(N, N, interp=interp), full_turn=full)
    _assert_close(out[S - 1].cpu().numpy(), ref)
