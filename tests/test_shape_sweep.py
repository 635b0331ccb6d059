"""Shape sweep on the GPU against the oracle restatement (pinned to the
reference by tests/test_oracle_golden.py): small and odd detector counts,
odd angle counts, output_n above / below n_t, pad factors 2-4, half / full
turn, bilinear / nearest -- the small-L kernel shapes (sub-warp transforms,
RPT < 16) and the texture paths' slot / mirror bookkeeping."""
import numpy as np
import pytest

from golden_util import rel_l2, max_rel
from oracle import bst_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = [
    # n_t, V, full, interp, output_n, pad
    (2, 1, False, "bilinear", None, 2),
    (3, 2, False, "bilinear", None, 2),
    (5, 4, True, "bilinear", None, 2),
    (8, 3, False, "nearest", None, 2),
    (16, 9, True, "nearest", None, 2),
    (17, 11, False, "bilinear", 9, 3),
    (31, 7, True, "bilinear", 40, 2),
    (40, 25, False, "nearest", 64, 2),
    (64, 63, False, "bilinear", 33, 4),
    (100, 50, True, "bilinear", 100, 3),
    (129, 80, False, "bilinear", 129, 2),
    (200, 45, True, "nearest", 150, 2),
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("n_t,V,full,interp,out_n,pad", CASES)
def test_shape_sweep_against_oracle(n_t, V, full, interp, out_n, pad):
    from paper_1704_08364_b200 import fourier_bp as F
    rng = np.random.default_rng(n_t * 131 + V)
    A = 2 * V if full else V
    S = 3
    vol = rng.standard_normal((S, A, n_t)).astype(np.float32)
    plan = F.BstPlan(n_t, V, interp=interp, output_n=out_n, pad_factor=pad)
    got = F.fbp_volume(torch.from_numpy(vol).cuda(), plan, full_turn=full, batch=2).cpu().numpy()
    op = O.OraclePlan(n_t, V, interp=interp, output_n=out_n, pad_factor=pad)
    for k in range(S):
        ref = O.fbp(vol[k].astype(np.float64), op, full_turn=full)
        r, m = rel_l2(got[k], ref), max_rel(got[k], ref)
        assert r <= 1e-4 and m <= 1e-3, (k, r, m)


@pytest.mark.parametrize("n_t,V,full,kernel,rolloff,kb", [
    (33, 1, False, "bst", 1.0, (10.0, 0.1)),      # a single angle
    (48, 20, False, "ss", 1.0, (10.0, 0.1)),
    (48, 20, True, "ss", 0.5, (10.0, 0.1)),
    (64, 32, False, "bst", 0.3, (6.0, 0.2)),      # apodised ramp, other KB window
    (90, 61, True, "bst", 0.8, (14.0, 0.05)),
])
def test_kernels_filters_windows_against_oracle(n_t, V, full, kernel, rolloff, kb):
    from paper_1704_08364_b200 import fourier_bp as F
    rng = np.random.default_rng(n_t + 7 * V)
    A = 2 * V if full else V
    vol = rng.standard_normal((2, A, n_t)).astype(np.float32)
    plan = F.BstPlan(n_t, V, kb_beta=kb[0], kb_support=kb[1])
    fplan = F.FilterPlan(kind="ramp_apodized", rolloff=rolloff) if rolloff < 1.0 else F.FilterPlan()
    got = F.fbp_volume(torch.from_numpy(vol).cuda(), plan, fplan, kernel=kernel, full_turn=full).cpu().numpy()
    op = O.OraclePlan(n_t, V, kb_beta=kb[0], kb_support=kb[1], rolloff=rolloff)
    for k in range(2):
        ref = O.fbp(vol[k].astype(np.float64), op, kernel, full_turn=full)
        r, m = rel_l2(got[k], ref), max_rel(got[k], ref)
        assert r <= 1e-4 and m <= 1e-3, (k, r, m)
