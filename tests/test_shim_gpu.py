"""GPU: the C++ shim (reference signatures) compiled against libtdg.so and run — the
reference's unit cases as a C++ caller would write them (tests/cpp/test_shim.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _build() -> str:
    from paper_1707_02000_b200._lib import LIB_DIR, ensure_built
    ensure_built()
    out_dir = os.path.join(ROOT, "tests", "cpp", "build")
    os.makedirs(out_dir, exist_ok=True)
    exe = os.path.join(out_dir, "test_shim")
    subprocess.run(["g++", "-O1", "-std=c++17", f"-I{ROOT}/include", f"-I{ROOT}/paper_1707_02000_b200/shim",
                    os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), f"-L{LIB_DIR}", "-ltrussdec_gpu", "-ltdg",
                    f"-Wl,-rpath,{LIB_DIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links():
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_shim_reference_cases_on_gpu():
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all shim checks passed" in r.stdout
