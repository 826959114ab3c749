"""tw_memcpy_h2d_staged / tw_memcpy_d2h_staged (include/tw/tw.h): host <->
device copies staged through the pinned ring by the host thread pool -- the
drop-in's RankGroup path.  Byte-exact round trips over chunk boundaries from
pageable and pinned memory, the NaN/Inf scan flag (TokenMatrix::validate's
check, proj/src/numerics.cpp:25-27), and the error taxonomy."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CHUNK = 8 << 20


def _p(a):
    return ctypes.c_void_p(a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data)


@pytest.mark.parametrize("nbytes", [4, 4096, CHUNK - 4, CHUNK, CHUNK + 4, 3 * CHUNK + 1028, 5 * CHUNK + 8])
@pytest.mark.parametrize("pinned", [False, True])
def test_staged_round_trip(cuda, nbytes, pinned):
    import torch
    from paper_2505_11329_b200 import _lib
    n = nbytes // 4
    src = torch.from_numpy(np.random.default_rng(nbytes).standard_normal(n).astype(np.float32))
    if pinned:
        src = src.pin_memory()
    dev = torch.full((n + 16,), -7.0, device="cuda")  # guard words after the copy
    nf = ctypes.c_int(-1)
    _lib.check(_lib.lib.tw_memcpy_h2d_staged(_p(dev), _p(src), nbytes, _lib.TW_F32, _lib.TW_HOST_CHECK_FINITE,
                                             ctypes.byref(nf)))
    assert nf.value == 0
    assert torch.equal(dev[:n].cpu(), src) and bool((dev[n:] == -7.0).all())
    back = torch.full((n + 16,), 3.0)
    _lib.check(_lib.lib.tw_memcpy_d2h_staged(_p(back), _p(dev), nbytes))
    assert torch.equal(back[:n], src) and bool((back[n:] == 3.0).all())


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("where", [0, CHUNK - 2, 2 * CHUNK + 6, -1])
@pytest.mark.parametrize("bad", ["nan", "inf", "-inf"])
def test_staged_h2d_flags_nonfinite(cuda, dtype, where, bad):
    import torch
    from paper_2505_11329_b200 import _lib
    nbytes = 3 * CHUNK + 64
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    esz = 4 if dtype == "f32" else 2
    src = torch.ones(nbytes // esz, dtype=tdt)
    src[(where // esz) if where >= 0 else -1] = float(bad)
    dev = torch.empty_like(src, device="cuda")
    code = _lib.TW_F32 if dtype == "f32" else _lib.TW_BF16
    nf = ctypes.c_int(0)
    _lib.check(_lib.lib.tw_memcpy_h2d_staged(_p(dev), _p(src), nbytes, code, _lib.TW_HOST_CHECK_FINITE,
                                             ctypes.byref(nf)))
    assert nf.value == 1
    assert torch.equal(dev.cpu().float().nan_to_num(0.0, 9.0, -9.0), src.float().nan_to_num(0.0, 9.0, -9.0))
    # without the flag: no scan, the copy is the same
    nf = ctypes.c_int(5)
    _lib.check(_lib.lib.tw_memcpy_h2d_staged(_p(dev), _p(src), nbytes, code, 0, ctypes.byref(nf)))
    assert nf.value == 0


def test_staged_copy_errors(cuda):
    import torch
    from paper_2505_11329_b200 import _lib
    host = torch.zeros(1024)
    other = torch.zeros(1024)
    dev = torch.zeros(1024, device="cuda")
    st = _lib.lib.tw_memcpy_h2d_staged(_p(other), _p(host), 4096, _lib.TW_F32, 0, None)
    assert st == _lib.TW_ERR_CONFIG  # the destination is not device memory
    st = _lib.lib.tw_memcpy_d2h_staged(_p(other), _p(host), 4096)
    assert st == _lib.TW_ERR_CONFIG
    assert _lib.lib.tw_memcpy_h2d_staged(_p(dev), _p(host), 6, _lib.TW_F32, 0, None) == _lib.TW_ERR_DIMENSION
    assert _lib.lib.tw_memcpy_h2d_staged(None, _p(host), 16, _lib.TW_F32, 0, None) == _lib.TW_ERR_DIMENSION
    assert _lib.lib.tw_memcpy_h2d_staged(_p(dev), _p(host), 0, _lib.TW_F32, 0, None) == _lib.TW_OK
