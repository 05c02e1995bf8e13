"""The C-ABI library loads on a CPU host and exports exactly what the header declares."""

import ctypes
import re

import numpy as np
import pytest

from paper_2211_15082_b200 import _lib


def header_functions():
    text = _lib.HEADER_PATH.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(glint_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/glint_b200.h but not exported"


def test_python_binding_covers_header_exactly():
    assert sorted(_lib.SIGNATURES) == header_functions()


def test_abi_version():
    assert _lib.query("glint_abi_version") == 1


def test_argument_errors_map_to_value_error_without_gpu():
    # validation happens on the host before any CUDA call
    with pytest.raises(ValueError, match="n_rows"):
        _lib.call("glint_spmm_mean_f32", -1, 4, None, None, None, 0, None, None, None, 4, None, 4,
                  None, 0, None, 0, None)
    with pytest.raises(ValueError, match="unknown kind"):
        _lib.call("glint_elementwise_f32", 99, 1, 1, 1, None, None, None, None, 1, None)
    with pytest.raises(ValueError, match="heads"):
        _lib.call("glint_gat_aggregate_f32", 1, 9, 4, 4, None, None, None, 0, None, None, None, 4,
                  None, None, 0.2, None, 4, None, 0, 0, None)
    assert "heads" in _lib.last_error()


def test_conv_mean_argument_errors_without_gpu():
    """K7's host-side validation (glint_conv_mean_f32) runs before any CUDA call."""
    args = dict(n_rows=10, dim_in=100, dim_out=256)

    def call(**kw):
        a = {**args, **kw}
        ws = 0 if kw.get("no_ws") else 4096
        _lib.call("glint_conv_mean_f32", a["n_rows"], a["dim_in"], a["dim_out"], 8, 16, None, 0,
                  None, None, 32, 100, 48, 100, None, kw.get("act", 0), 64, 256, None,
                  kw.get("max_ctas", 0), None if kw.get("no_ws") else 80, ws, None)

    with pytest.raises(ValueError, match="n_rows"):
        call(n_rows=-1)
    with pytest.raises(ValueError, match="act"):
        call(act=7)
    with pytest.raises(ValueError, match="max_ctas"):
        call(max_ctas=-2)
    with pytest.raises(ValueError, match="null"):
        call(no_ws=True)
    with pytest.raises(ValueError, match="workspace too small"):
        call()
    assert _lib.query("glint_conv_mean_supported", 100, 256) == 1
    assert _lib.query("glint_conv_mean_supported", 256, 256) == 0
    assert _lib.query("glint_conv_mean_supported", 100, 300) == 0
    assert _lib.query("glint_conv_mean_workspace_bytes", 100, 256) >= 256 + 13 * 2 * 256 * 8 * 4


def test_workspace_queries():
    assert _lib.query("glint_idset_workspace_bytes", 1000) >= 1000 // 8
    assert _lib.query("glint_scan_workspace_bytes", 10) >= 16
    assert _lib.query("glint_degree_schedule_workspace_bytes") == 1024


def test_native_rcmk_rejects_bad_ids():
    indptr = np.array([0, 1], dtype=np.int64)
    indices = np.array([5], dtype=np.int64)
    perm = np.zeros(1, dtype=np.int64)
    rc = _lib.load().glint_rcmk_host(1, indptr.ctypes.data_as(ctypes.c_void_p),
                                     indices.ctypes.data_as(ctypes.c_void_p),
                                     perm.ctypes.data_as(ctypes.c_void_p))
    assert rc == _lib.GLINT_EINVAL


def test_sm100a_code_in_library():
    """The .so carries sm_100a SASS (cross-compiled here, run on the B200 box)."""
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
