"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, and validates plans like the reference (no GPU needed:
validation happens before any CUDA call)."""
import ctypes

import pytest

from paper_1704_08364_b200 import _native


def test_library_loads_and_exports_every_header_symbol():
    lib = _native.lib()
    names = _native.header_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    assert lib.tb_abi_version() == 3


def _desc(**kw):
    d = _native.tb_plan_desc()
    d.n_t, d.n_theta, d.pad_factor, d.radial_samples = 256, 256, 2, 0
    d.kb_beta, d.kb_support, d.sigma_min_bins = 10.0, 0.1, 1
    d.interp, d.output_n, d.full_turn, d.filter_kind, d.rolloff = 0, 0, 0, 0, 1.0
    for k, v in kw.items():
        setattr(d, k, v)
    return d


@pytest.mark.parametrize("kw,msg", [
    ({"n_t": 1}, "need n_t >= 2 and n_theta >= 1"),
    ({"n_theta": 0}, "need n_t >= 2 and n_theta >= 1"),
    ({"pad_factor": 1}, "pad_factor must be >= 2, got 1"),
    ({"sigma_min_bins": 0}, "sigma_min_bins must be >= 1, got 0"),
    ({"interp": 7}, "unknown interp mode"),
    ({"radial_samples": 500}, "radial_samples must be a power of two >= pad_factor * n_t, got 500"),
    ({"radial_samples": 256}, "radial_samples must be a power of two >= pad_factor * n_t, got 256"),
    ({"output_n": 1025}, "output_n must be in [1, radial_samples]"),
    ({"filter_kind": 5}, "unknown filter kind"),
    ({"rolloff": 0.0}, "rolloff must be in (0, 1]"),
    ({"n_angles": -1}, "n_angles must be >= 0"),
    ({"flags": 6}, "unknown plan flags"),
])
def test_plan_validation_mirrors_reference(kw, msg):
    lib = _native.lib()
    h = ctypes.c_void_p()
    rc = lib.tb_plan_create(ctypes.byref(_desc(**kw)), 0, ctypes.byref(h))
    assert rc == _native.TB_ERR_INVALID
    assert msg in _native.last_error()
    with pytest.raises(ValueError):
        _native.check(rc)


def test_unsupported_size_reports_unsupported():
    lib = _native.lib()
    h = ctypes.c_void_p()
    rc = lib.tb_plan_create(ctypes.byref(_desc(n_t=16384, n_theta=4)), 0, ctypes.byref(h))  # L = 32768
    assert rc == _native.TB_ERR_UNSUPPORTED


def test_null_arguments_do_not_crash():
    lib = _native.lib()
    assert lib.tb_plan_create(None, 0, None) == _native.TB_ERR_INVALID
    assert lib.tb_plan_destroy(None) == _native.TB_OK
    assert lib.tb_fbp(None, None, None, 1, 1, None, 0, None) == _native.TB_ERR_INVALID
    assert lib.tb_fbp_pre(None, None, None, 1, 1, None, 0, None, None, None) == _native.TB_ERR_INVALID
    assert lib.tb_pre_params(None, None, 1, None, 9, None, None, None, None) == _native.TB_ERR_INVALID


@pytest.mark.gpu
def test_fused_stage_entry_points_validate_like_the_reference():
    """tb_pre_params / tb_fbp_pre error paths on a real plan: ring window
    (suppress_rings' message), missing shift / stripe buffers, and a plan
    whose ramp is a separate pass (npad != L) -> TB_ERR_UNSUPPORTED."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = _native.lib()
    h = ctypes.c_void_p()
    assert lib.tb_plan_create(ctypes.byref(_desc(n_t=64, n_theta=32)), 0, ctypes.byref(h)) == _native.TB_OK
    h4 = ctypes.c_void_p()
    assert lib.tb_plan_create(ctypes.byref(_desc(n_t=64, n_theta=32, pad_factor=4)), 0,
                              ctypes.byref(h4)) == _native.TB_OK
    try:
        sino = torch.zeros((2, 32, 64), device="cuda")
        shift = torch.zeros((2, 2), device="cuda")
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        assert lib.tb_pre_params(h, p(sino), 2, None, 4, None, p(shift), None, None) == _native.TB_ERR_INVALID
        assert b"window must be an odd integer >= 3, got 4" in lib.tb_last_error()
        assert lib.tb_pre_params(h, p(sino), 2, None, 9, None, p(shift), None, None) == _native.TB_ERR_INVALID
        assert lib.tb_pre_params(h, p(sino), 2, None, 0, None, p(shift), None, None) == _native.TB_OK
        img = torch.empty((2, 64, 64), device="cuda")
        ws_bytes = ctypes.c_size_t()
        assert lib.tb_workspace_bytes(h4, 2, ctypes.byref(ws_bytes)) == _native.TB_OK
        ws = torch.empty(ws_bytes.value, dtype=torch.uint8, device="cuda")
        rc = lib.tb_fbp_pre(h4, p(sino), p(img), 2, 2, p(ws), ws_bytes, p(shift), None, None)
        assert rc == _native.TB_ERR_UNSUPPORTED
        rc = lib.tb_fbp_pre(h, p(sino), p(img), 2, 2, p(ws), ws_bytes, None, None, None)
        assert rc == _native.TB_ERR_INVALID
        torch.cuda.synchronize()
    finally:
        lib.tb_plan_destroy(h)
        lib.tb_plan_destroy(h4)
