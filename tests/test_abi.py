"""CPU: the C-ABI library loads and exports every symbol include/*.h declares; the
product fails loudly (no CPU fallback) without a GPU; host-side plumbing."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared(header: str) -> list[str]:
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tdg_[a-z_0-9]+)\s*\(", txt)))


def test_tdg_exports_every_declared_symbol():
    from paper_1707_02000_b200 import _lib
    names = declared("tdg.h")
    assert "tdg_truss" in names and "tdg_support" in names and "tdg_process_sublevel" in names
    lib = C.CDLL(_lib.TDG_SO)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes signature table covers the header exactly
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == names


def test_gen_exports_every_declared_symbol():
    from paper_1707_02000_b200._lib import LIB_DIR
    names = declared("tdg_gen.h")
    lib = C.CDLL(os.path.join(LIB_DIR, "libtdg_gen.so"))
    assert [n for n in names if not hasattr(lib, n)] == []


def test_shim_library_exports_reference_names():
    import subprocess
    from paper_1707_02000_b200._lib import LIB_DIR
    out = subprocess.run(["nm", "-DC", os.path.join(LIB_DIR, "libtrussdec_gpu.so")], capture_output=True,
                         text=True, check=True).stdout
    for sym in ("trussdec_gpu::truss_parallel(", "trussdec_gpu::support_am4(", "trussdec_gpu::build_truss_graph(",
                "trussdec_gpu::scan(", "trussdec_gpu::process_sublevel(", "trussdec_gpu::stats("):
        assert sym in out, sym


def test_sm100a_cubin_present():
    import subprocess
    from paper_1707_02000_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.TDG_SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_without_gpu():
    import torch
    from paper_1707_02000_b200 import _lib, trussdec
    assert b"sm_100a" in _lib.tdg().tdg_version()
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        trussdec.Context(0)
    g = trussdec.CsrGraph.from_arrays(np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32))
    with pytest.raises(RuntimeError):
        trussdec.truss_parallel(g)


def test_counter_names_follow_the_header():
    """tdg_counters: the Python names list the header's TDG_CNT_* enum in order."""
    from paper_1707_02000_b200 import trussdec
    txt = open(os.path.join(ROOT, "include", "tdg.h")).read()
    i0 = txt.index("TDG_CNT_FILTER = 0")
    body = txt[i0: txt.index("TDG_NCOUNTERS", i0)]
    names = [n.lower() for n in re.findall(r"TDG_CNT_([A-Z_]+)", body)]
    assert names == list(trussdec.Context.COUNTER_NAMES)
