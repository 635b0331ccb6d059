"""TOMOVOL1 container I/O (volio.py of the reference):
byte-exact against files written by the real reference
(tests/golden/make_golden.py -> tests/golden/vol/), and the GPU slab path
(frame-major slabs read in place by the radial kernel)."""
import os

import numpy as np
import pytest

from golden_util import GOLDEN_DIR

VOL = os.path.join(GOLDEN_DIR, "vol")


def _bytes(name):
    with open(os.path.join(VOL, name), "rb") as f:
        return f.read()


def test_header_and_writer_are_byte_exact(tmp_path):
    from paper_1704_08364_b200 import volio as V
    e = np.load(os.path.join(VOL, "expect.npz"))
    frames = e["frames"]
    V.write_volume(tmp_path / "f.tomovol", V.VolumeHeader(V.LAYOUT_FRAMES, frames.shape), frames)
    assert (tmp_path / "f.tomovol").read_bytes() == _bytes("frames.tomovol")
    sl = np.ascontiguousarray(frames.transpose(1, 0, 2))
    V.write_volume(tmp_path / "s.tomovol", V.VolumeHeader(V.LAYOUT_SLICES, sl.shape), sl)
    assert (tmp_path / "s.tomovol").read_bytes() == _bytes("slices.tomovol")
    from paper_1704_08364_b200.slices import ImageGrid
    with V.VolumeWriter(tmp_path / "w.tomovol", 3, 4) as wr:
        for k in (2, 0, 1):
            wr.write_slice(k, ImageGrid(4, e["imgs"][k]))
    assert (tmp_path / "w.tomovol").read_bytes() == _bytes("written.tomovol")
    V.export_image(ImageGrid(4, e["imgs"][0]), tmp_path / "i.pgm")
    assert (tmp_path / "i.pgm").read_bytes() == _bytes("img0.pgm")


@pytest.mark.parametrize("name", ["frames.tomovol", "slices.tomovol"])
def test_block_reader_matches_reference_blocks(name):
    from paper_1704_08364_b200 import volio as V
    e = np.load(os.path.join(VOL, "expect.npz"))
    with V.BlockReader(os.path.join(VOL, name), 2) as rd:
        assert rd.header.n_angles == 6 and rd.header.n_slices == 5 and rd.header.n_t == 8
        blocks = list(rd)
        assert V.read_block(rd) is None
    assert [b.first_slice for b in blocks] == [0, 2, 4]
    for k, b in enumerate(blocks):
        np.testing.assert_array_equal(np.stack([s.data for s in b.slices]), e[f"block{k}"])
    with V.BlockReader(os.path.join(VOL, name), 2) as rd:
        slab = rd.read_slab(1, 3).numpy()
        want = e["frames"][:, 1:4] if rd.header.layout == V.LAYOUT_FRAMES else e["frames"][:, 1:4].transpose(1, 0, 2)
        np.testing.assert_array_equal(slab, want)


def test_container_errors_mirror_reference(tmp_path):
    from paper_1704_08364_b200 import volio as V
    with pytest.raises(V.VolumeError, match="not a TOMOVOL1 file"):
        V.VolumeHeader.unpack(b"X" * 64)
    with pytest.raises(V.VolumeError, match="header truncated"):
        V.VolumeHeader.unpack(b"TOMOVOL1")
    raw = bytearray(_bytes("frames.tomovol")[:64])
    raw[21] = 3
    with pytest.raises(V.VolumeError, match="unsupported dtype"):
        V.VolumeHeader.unpack(bytes(raw))
    with pytest.raises(ValueError, match="unknown layout"):
        V.VolumeHeader(2, (1, 1, 1))
    (tmp_path / "t.tomovol").write_bytes(_bytes("frames.tomovol")[:-4])
    with pytest.raises(V.VolumeError, match="expected"):
        V.BlockReader(tmp_path / "t.tomovol", 1)
    with V.BlockReader(os.path.join(VOL, "frames.tomovol"), 2) as rd:
        with pytest.raises(ValueError, match="out of bounds"):
            rd.read_slices(4, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", [0, 1])
def test_gpu_reconstruct_file_equals_device_fbp(tmp_path, layout):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1704_08364_b200 import fourier_bp as F, phantom, volio as V
    S, n = 11, 128
    vol = phantom.ellipsoid_volume(S, n, n, device="cuda")
    vol += 0.02 * torch.randn(vol.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    host = vol.cpu().numpy()
    data = np.ascontiguousarray(host.transpose(1, 0, 2)) if layout == 0 else host
    V.write_volume(tmp_path / "in.tomovol", V.VolumeHeader(layout, data.shape), data)
    plan = F.BstPlan(n, n)
    V.reconstruct_file(tmp_path / "in.tomovol", tmp_path / "out.tomovol", plan, block=4, batch=2)
    ref = F.fbp_volume(vol, plan, batch=2).cpu()
    with V.BlockReader(tmp_path / "out.tomovol", S) as rd:
        assert rd.header.layout == V.LAYOUT_SLICES and rd.header.dims == (S, n, n)
        got = rd.read_slab(0, S)
    assert torch.equal(got, ref)  # same kernels; the frame-major slab is read in place
