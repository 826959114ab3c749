"""The C-ABI library loads, exports every symbol include/tw/tw.h declares, and
its host-side validation follows the reference's error taxonomy.  CPU only:
no compute call needs a GPU here."""
import ctypes
import os
import re

import pytest

from tests.conftest import ROOT


def declared_symbols():
    with open(os.path.join(ROOT, "include", "tw", "tw.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^TW_API\s+[\w\s\*]+?\b(tw_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "tw_fused_allreduce_rmsnorm_group" in syms and "tw_rmsnorm_residual" in syms
    assert len(syms) >= 16


def test_library_exports_every_declared_symbol():
    import paper_2505_11329_b200._lib as L
    lib = ctypes.CDLL(L.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), f"libtw.so does not export {s}"
    assert sorted(L.exported_symbols()) == declared_symbols()


@pytest.mark.parametrize("header,lib", [("tw_split.h", "libweavesim_b200.so"),
                                        ("tw_workload.h", "libweavesim_b200.so"),
                                        ("tw_weave.h", "libtw_weave.so")])
def test_layer_libraries_export_their_headers(header, lib):
    with open(os.path.join(ROOT, "include", "tw", header)) as f:
        syms = set(re.findall(r"^TW_API\s+[\w\s\*]+?\b(tw_\w+)\s*\(", f.read(), flags=re.M))
    assert syms
    import paper_2505_11329_b200._lib  # noqa: F401  (libtw.so first, as a host would)
    so = ctypes.CDLL(os.path.join(ROOT, "paper_2505_11329_b200", "lib", lib))
    for s in sorted(syms):
        assert hasattr(so, s), f"{lib} does not export {s}"


def test_version_and_abi():
    import paper_2505_11329_b200 as tw
    from paper_2505_11329_b200 import _lib
    assert _lib.lib.tw_abi_version() == 1
    assert "sm_100a" in tw.version()


def test_shard_map_matches_reference_semantics():
    import paper_2505_11329_b200 as tw
    assert tw.token_shard_map(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert tw.token_shard_map(3, 8) == [(0, 1), (1, 2), (2, 3)] + [(3, 3)] * 5
    with pytest.raises(tw.ConfigError):
        tw.token_shard_map(16, 1)
    with pytest.raises(tw.DimensionError):
        tw.token_shard_map(-1, 4)
    tw.shard_map_validate([(0, 8), (8, 16)], 16)
    with pytest.raises(tw.ContractError):
        tw.shard_map_validate([(0, 8), (7, 16)], 16)
    with pytest.raises(tw.ContractError):
        tw.shard_map_validate([(0, 8), (8, 16)], 17)
    with pytest.raises(tw.ContractError):
        tw.shard_map_validate([], 0)


def test_shard_map_matches_oracle(orc):
    import paper_2505_11329_b200 as tw
    for T in (0, 1, 7, 8, 100, 1023, 8192):
        for W in (2, 3, 4, 8):
            assert tw.token_shard_map(T, W) == orc.token_shard_map(T, W)


def test_host_validation_before_any_device_work():
    from paper_2505_11329_b200 import _lib
    L = _lib.lib
    # negative epsilon -> NumericError (proj/src/numerics.cpp:43-45); bad dims -> DimensionError
    assert L.tw_rmsnorm_residual(None, None, None, None, None, 4, 8, -1.0, 0, 0, None) == _lib.TW_ERR_NUMERIC
    assert L.tw_rmsnorm_residual(None, None, None, None, None, 4, 0, 1e-5, 0, 0, None) == _lib.TW_ERR_DIMENSION
    assert L.tw_rmsnorm_residual(None, None, None, None, None, -1, 8, 1e-5, 0, 0, None) == _lib.TW_ERR_DIMENSION
    # T == 0 is a legal no-op
    assert L.tw_rmsnorm_residual(None, None, None, None, None, 0, 8, 1e-5, 0, 0, None) == _lib.TW_OK
    L.tw_rmsnorm_residual(None, None, None, None, None, 4, 8, -1.0, 0, 0, None)
    assert b"epsilon" in L.tw_last_error()


def test_c_abi_from_plain_c99(tmp_path):
    """The headers are C (not C++) and the libraries link from gcc -std=c99."""
    import subprocess
    exe = tmp_path / "test_capi"
    lib = os.path.join(ROOT, "paper_2505_11329_b200", "lib")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "test_capi.c"), "-o", str(exe), "-L", lib, "-ltw",
                    "-lweavesim_b200", "-ltw_weave", f"-Wl,-rpath,{lib}"], check=True)
    p = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "c-abi: ok" in p.stdout


def test_comm_requires_a_device_here():
    import paper_2505_11329_b200 as tw
    if tw.device_count() > 0:
        pytest.skip("GPU visible")
    with pytest.raises(tw.CudaError):
        tw.Communicator(2, [0, 0], 1 << 20)


def test_staged_copies_validate_on_the_host():
    """tw_memcpy_h2d_staged / tw_memcpy_d2h_staged reject bad arguments before
    any device work: null buffers and partial elements (DIMENSION), unknown
    dtypes and a destination / source that is not device memory (CONFIG; on
    a GPU-less host every pointer is host memory); zero bytes is a no-op."""
    import ctypes
    from paper_2505_11329_b200 import _lib
    L = _lib.lib
    buf = (ctypes.c_float * 16)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    nf = ctypes.c_int(7)
    assert L.tw_memcpy_h2d_staged(p, p, 0, _lib.TW_F32, 0, ctypes.byref(nf)) == _lib.TW_OK and nf.value == 0
    assert L.tw_memcpy_h2d_staged(None, p, 16, _lib.TW_F32, 0, None) == _lib.TW_ERR_DIMENSION
    assert L.tw_memcpy_h2d_staged(p, p, 6, _lib.TW_F32, 0, None) == _lib.TW_ERR_DIMENSION
    assert L.tw_memcpy_h2d_staged(p, p, 16, 7, 0, None) == _lib.TW_ERR_CONFIG
    assert L.tw_memcpy_h2d_staged(p, p, 16, _lib.TW_F32, 0, None) == _lib.TW_ERR_CONFIG
    assert b"not device memory" in L.tw_last_error()
    assert L.tw_memcpy_d2h_staged(p, None, 16) == _lib.TW_ERR_DIMENSION
    assert L.tw_memcpy_d2h_staged(p, p, 16) == _lib.TW_ERR_CONFIG
    assert L.tw_memcpy_d2h_staged(p, p, 0) == _lib.TW_OK


def test_gated_host_sync_validates_on_the_host():
    """tw_rmsnorm_residual_host_sync_gated (the drop-in's overlapped-fill
    path) rejects a malformed gate before anything else, then validates like
    tw_rmsnorm_residual_host_sync; T == 0 is a no-op."""
    import ctypes
    from paper_2505_11329_b200 import _lib
    L = _lib.lib
    ready = (ctypes.c_int64 * 2)(0, 0)
    assert L.tw_rmsnorm_residual_host_sync_gated(None, None, None, None, None, 4, 8, 1e-5, _lib.TW_F32, 0,
                                                  None, 2) == _lib.TW_ERR_DIMENSION
    assert b"gate" in L.tw_last_error()
    assert L.tw_rmsnorm_residual_host_sync_gated(None, None, None, None, None, 4, 8, 1e-5, _lib.TW_F32, 0,
                                                  ready, -1) == _lib.TW_ERR_DIMENSION
    assert L.tw_rmsnorm_residual_host_sync_gated(None, None, None, None, None, 4, 8, -1.0, _lib.TW_F32, 0,
                                                  ready, 2) == _lib.TW_ERR_NUMERIC
    assert L.tw_rmsnorm_residual_host_sync_gated(None, None, None, None, None, 4, 8, 1e-5, _lib.TW_F32, 0,
                                                  ready, 2) == _lib.TW_ERR_DIMENSION  # null buffers
    assert L.tw_rmsnorm_residual_host_sync_gated(None, None, None, None, None, 0, 8, 1e-5, _lib.TW_F32, 0,
                                                  ready, 2) == _lib.TW_OK
