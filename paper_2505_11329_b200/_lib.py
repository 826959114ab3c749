"""ctypes binding of libtw.so (include/tw/tw.h).

Python is plumbing here: tests and bench.py reach the product through the
same C-ABI a C++/cgo/JNI host would bind.  There is no Python or CPU compute
path -- if libtw.so is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_int64, c_size_t, c_uint, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libtw.so")

TW_OK, TW_ERR_DIMENSION, TW_ERR_NUMERIC, TW_ERR_CONFIG, TW_ERR_CONTRACT, TW_ERR_CUDA, TW_ERR_TIMEOUT, \
    TW_ERR_UNSUPPORTED, TW_ERR_PARSE = range(9)
TW_BF16, TW_F32 = 0, 1
TW_TRANSPORT_AUTO, TW_TRANSPORT_NVLS, TW_TRANSPORT_PEER, TW_TRANSPORT_NVLS_SIM = 0, 1, 2, 3
TW_BUF_INPUT, TW_BUF_OUTPUT, TW_BUF_RESIDUAL = 0, 1, 2
TW_HOST_CHECK_FINITE = 0x1
TW_GATHER_RESIDUAL = 0x1
TRANSPORT_NAMES = {TW_TRANSPORT_AUTO: "auto", TW_TRANSPORT_NVLS: "nvls", TW_TRANSPORT_PEER: "peer",
                   TW_TRANSPORT_NVLS_SIM: "nvls_sim"}


def TW_NVLS_DEPTH(d: int) -> int:
    """Flag bits of the NVLS kernel's pipeline depth (tw.h TW_NVLS_DEPTH)."""
    return (int(d) & 0x3) << 4


class TwError(RuntimeError):
    """Base of the error taxonomy (mirrors proj/include/weavesim/errors.hpp)."""


class DimensionError(TwError):
    pass


class NumericError(TwError):
    pass


class ConfigError(TwError):
    pass


class ContractError(TwError):
    pass


class CudaError(TwError):
    pass


class BarrierTimeout(TwError):
    pass


class Unsupported(TwError):
    pass


class ParseError(TwError):
    pass


_ERRORS = {
    TW_ERR_DIMENSION: DimensionError,
    TW_ERR_NUMERIC: NumericError,
    TW_ERR_CONFIG: ConfigError,
    TW_ERR_CONTRACT: ContractError,
    TW_ERR_CUDA: CudaError,
    TW_ERR_TIMEOUT: BarrierTimeout,
    TW_ERR_UNSUPPORTED: Unsupported,
    TW_ERR_PARSE: ParseError,
}

# (name, restype, argtypes) for every symbol tw.h declares.
_SIGNATURES = [
    ("tw_abi_version", c_int, []),
    ("tw_version", c_char_p, []),
    ("tw_last_error", c_char_p, []),
    ("tw_device_count", c_int, []),
    ("tw_rmsnorm_residual", c_int,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_float, c_int, c_int, c_void_p]),
    ("tw_rmsnorm_residual_host", c_int,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_float, c_int, c_int64, c_void_p]),
    ("tw_rmsnorm_residual_host_sync", c_int,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_float, c_int, c_uint]),
    ("tw_rmsnorm_residual_host_sync_gated", c_int,
     [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_float, c_int, c_uint,
      POINTER(c_int64), c_int]),
    ("tw_count_nonfinite", c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    ("tw_token_shard_map", c_int, [c_int64, c_int, POINTER(c_int64)]),
    ("tw_shard_map_validate", c_int, [POINTER(c_int64), c_int, c_int64]),
    ("tw_comm_create", c_int, [c_int, POINTER(c_int), c_size_t, c_int, POINTER(c_void_p)]),
    ("tw_comm_destroy", c_int, [c_void_p]),
    ("tw_comm_info", c_int, [c_void_p, POINTER(c_int), POINTER(c_int), POINTER(c_size_t)]),
    ("tw_comm_local_rank", c_int, [c_void_p, POINTER(c_int), POINTER(c_int)]),
    ("tw_comm_buffer", c_int, [c_void_p, c_int, c_int, POINTER(c_void_p)]),
    ("tw_comm_multicast_buffer", c_int, [c_void_p, c_int, c_int, POINTER(c_void_p)]),
    ("tw_fused_allreduce_rmsnorm_group", c_int,
     [c_void_p, c_int64, c_int64, c_int64, POINTER(c_int64), POINTER(c_void_p), POINTER(c_void_p), c_float, c_int, c_int,
      c_uint, POINTER(c_void_p)]),
    ("tw_allreduce_group", c_int, [c_void_p, c_int64, c_int64, c_int64, c_int, c_int, POINTER(c_void_p)]),
    ("tw_device_alloc", c_int, [c_int, c_size_t, POINTER(c_void_p)]),
    ("tw_device_free", c_int, [c_int, c_void_p]),
    ("tw_memcpy", c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    ("tw_memcpy_h2d_staged", c_int, [c_void_p, c_void_p, c_size_t, c_int, c_uint, POINTER(c_int)]),
    ("tw_memcpy_d2h_staged", c_int, [c_void_p, c_void_p, c_size_t]),
    ("tw_device_synchronize", c_int, [c_int]),
    ("tw_comm_check", c_int, [c_void_p]),
    ("tw_comm_create_mp", c_int, [c_int, c_int, c_int, c_size_t, c_char_p, c_int, POINTER(c_void_p)]),
    ("tw_fused_allreduce_rmsnorm", c_int,
     [c_void_p, c_int64, c_int64, c_int64, POINTER(c_int64), c_void_p, c_void_p, c_float, c_int, c_int, c_uint,
      c_void_p]),
    ("tw_allreduce", c_int, [c_void_p, c_int64, c_int64, c_int64, c_int, c_int, c_void_p]),
    ("tw_rendezvous_exchange_fd", c_int, [c_char_p, c_int, c_int, c_int, POINTER(c_int)]),
]


def _preload_cuda_cublas() -> None:
    """Bind the CUDA toolkit's cuBLAS (12.9, the one libtw_weave.so is built
    against) before anything else loads a libcublas.so.12: torch ships its own
    (12.8) and, loaded first, would serve the weave runner's GEMMs too -- with
    different kernel choices (the weave measured 1673 vs 1328 us per layer at
    Llama TP=8 shapes, T=8192).  A later `import torch` then
    reuses the already-loaded libraries (same SONAME).  No-op if torch's
    copy is already in the process or the toolkit is absent."""
    import sys
    if "torch" in sys.modules:
        return
    root = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    for name in ("libcublasLt.so.12", "libcublas.so.12"):
        path = os.path.join(root, "lib64", name)
        if os.path.exists(path):
            try:
                ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
            except OSError:
                return


def _load() -> ctypes.CDLL:
    _preload_cuda_cublas()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `make lib` (or __graft_entry__.build()); "
                          "there is no CPU fallback for the TokenWeave path")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in _SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int, message=None) -> None:
    """Raise the taxonomy's exception for a failing status; `message` is a
    callable returning the layer's last-error text (default: libtw's)."""
    if status != TW_OK:
        raw = message() if message is not None else lib.tw_last_error()
        msg = (raw or b"").decode()
        raise _ERRORS.get(status, TwError)(msg or f"tw status {status}")


def exported_symbols() -> list[str]:
    return [name for name, _, _ in _SIGNATURES]


def token_shard_map(num_tokens: int, world: int) -> list[tuple[int, int]]:
    buf = (c_int64 * (2 * max(world, 1)))()
    check(lib.tw_token_shard_map(num_tokens, world, buf))
    return [(buf[2 * r], buf[2 * r + 1]) for r in range(world)]


def shard_map_validate(ranges, total: int) -> None:
    flat = [v for rg in ranges for v in rg]
    buf = (c_int64 * max(len(flat), 1))(*flat)
    check(lib.tw_shard_map_validate(buf, len(ranges), total))
