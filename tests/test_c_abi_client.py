"""The C ABI from plain C99 (tests/c/abi_smoke.c): the header compiles as C,
the client links against libtb_bst.so, and on a GPU it reconstructs a
constant sinogram through tb_bst and checks the c * coverage identity."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "abi_smoke.c")
LIBDIR = os.path.join(ROOT, "paper_1704_08364_b200", "lib")
CUDA = "/usr/local/cuda"


def _gcc(args):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    return subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-D_DEFAULT_SOURCE",
                           "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CUDA, "include")] + args,
                          capture_output=True, text=True)


def _build(tmp_path):
    exe = str(tmp_path / "c_abi_smoke")
    r = _gcc([SRC, "-o", exe, "-L" + LIBDIR, "-ltb_bst", "-Wl,-rpath," + LIBDIR,
              "-L" + os.path.join(CUDA, "lib64"), "-lcudart", "-lm"])
    assert r.returncode == 0, r.stderr
    return exe


def test_header_is_c99_and_client_links(tmp_path):
    r = _gcc(["-c", SRC, "-o", str(tmp_path / "abi_smoke.o")])
    assert r.returncode == 0, r.stderr
    if os.path.exists(os.path.join(LIBDIR, "libtb_bst.so")):
        _build(tmp_path)


@pytest.mark.gpu
def test_c_client_reconstructs_constant_sinogram(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "c_abi_smoke ok" in r.stdout
