"""B200-native TokenWeave hot path: fused AllReduce + residual-add + RMSNorm.

The product is libtw.so (hand-written sm_100a CUDA behind the C-ABI in
include/tw/tw.h) plus the drop-in C++ API libweavesim_b200.so
(include/weavesim/*.hpp).  This Python package is the plumbing tests and
bench.py use to reach that C-ABI with torch-allocated device memory; it has
no compute of its own and raises if the native library is missing.
"""
from __future__ import annotations

import ctypes
from ctypes import c_int, c_int64, c_size_t, c_void_p

from . import _lib
from ._lib import (TW_BF16, TW_F32, TW_BUF_INPUT, TW_BUF_OUTPUT, TW_BUF_RESIDUAL, TW_GATHER_RESIDUAL,
                   TW_TRANSPORT_AUTO, TW_TRANSPORT_NVLS, TW_TRANSPORT_NVLS_SIM, TW_TRANSPORT_PEER, TW_NVLS_DEPTH,
                   BarrierTimeout, ConfigError,
                   ContractError, CudaError, DimensionError, NumericError, TwError, Unsupported, check,
                   shard_map_validate, token_shard_map)

__all__ = [
    "rmsnorm_residual", "Communicator", "token_shard_map", "shard_map_validate", "TwError", "DimensionError",
    "NumericError", "ConfigError", "ContractError", "CudaError", "BarrierTimeout", "Unsupported", "TW_BF16",
    "TW_F32", "TW_GATHER_RESIDUAL", "TW_TRANSPORT_AUTO", "TW_TRANSPORT_NVLS", "TW_TRANSPORT_PEER",
    "TW_TRANSPORT_NVLS_SIM", "TW_NVLS_DEPTH",
    "device_count", "version",
]


def version() -> str:
    return _lib.lib.tw_version().decode()


def device_count() -> int:
    return _lib.lib.tw_device_count()


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.bfloat16:
        return TW_BF16
    if t.dtype == torch.float32:
        return TW_F32
    raise ConfigError(f"unsupported activation dtype {t.dtype} (bf16 or fp32)")


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _current_raw_stream(device=None) -> int:
    """The current CUDA stream handle of `device` (default: the current one);
    torch's raw accessor costs ~0.3 us where torch.cuda.current_stream() costs
    ~3 us per call, which is most of an op's host time at decode sizes
    (tools/host_overhead.py)."""
    import torch
    torch.cuda._lazy_init()  # a flag check once initialised
    if device is None:
        device = torch._C._cuda_getDevice()
    return torch._C._cuda_getCurrentRawStream(device)


def _stream_handle(stream) -> int | None:
    if stream is None:
        return _current_raw_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def rmsnorm_residual(inp, residual, weight, eps: float = 1e-5, *, residual_out=None, out=None, sm_budget: int = 0,
                     stream=None):
    """TP=1 fused residual-add + RMSNorm (kernel K2) on CUDA tensors.

    Mirrors weavesim::rmsnorm_residual (proj/src/numerics.cpp:30-64):
    returns (output, residual_out) with residual_out = inp + residual and
    output = residual_out * rsqrt(mean(residual_out^2) + eps) * weight.
    `residual_out` may be `residual` itself (in-place).  weight is fp32[H].
    """
    import torch
    if inp.dim() != 2 or residual.shape != inp.shape:
        raise DimensionError("rmsnorm_residual: input and residual shapes differ")
    T, H = inp.shape
    if weight.numel() != H:
        raise DimensionError("rmsnorm_residual: weight length must equal hidden size")
    if weight.dtype != torch.float32:
        raise ConfigError("rmsnorm_residual: weight must be fp32 (NormParams::weight)")
    if residual.dtype != inp.dtype:
        raise ConfigError("rmsnorm_residual: input and residual dtypes differ")
    if out is None:
        out = torch.empty_like(inp)
    if residual_out is None:
        residual_out = torch.empty_like(inp)
    for t in (inp, residual, residual_out, out, weight):
        if not t.is_cuda or not t.is_contiguous():
            raise ConfigError("rmsnorm_residual: tensors must be contiguous CUDA tensors")
    check(_lib.lib.tw_rmsnorm_residual(_ptr(inp), _ptr(residual), _ptr(residual_out), _ptr(out), _ptr(weight), T, H,
                                       float(eps), _dtype_code(inp), int(sm_budget), _stream_handle(stream)))
    return out, residual_out


def rmsnorm_residual_host(inp, residual, weight, eps: float = 1e-5, *, residual_out=None, out=None,
                          chunk_rows: int = 0, stream=None):
    """K2 over HOST (CPU) tensors -- pin them for full speed.  The C-ABI
    pipelines chunks (H2D | kernel | D2H overlapped); on return the work is
    enqueued on `stream` (synchronize before reading the outputs)."""
    import torch
    if inp.dim() != 2 or residual.shape != inp.shape:
        raise DimensionError("rmsnorm_residual_host: input and residual shapes differ")
    T, H = inp.shape
    if weight.numel() != H or weight.dtype != torch.float32 or weight.is_cuda:
        raise DimensionError("rmsnorm_residual_host: weight must be a host fp32 [H] tensor")
    if out is None:
        out = torch.empty_like(inp)
    if residual_out is None:
        residual_out = torch.empty_like(inp)
    for t in (inp, residual, residual_out, out):
        if t.is_cuda or not t.is_contiguous():
            raise ConfigError("rmsnorm_residual_host: tensors must be contiguous host tensors")
    check(_lib.lib.tw_rmsnorm_residual_host(_ptr(inp), _ptr(residual), _ptr(residual_out), _ptr(out), _ptr(weight),
                                            T, H, float(eps), _dtype_code(inp), int(chunk_rows),
                                            _stream_handle(stream)))
    return out, residual_out


class _DevBuf:
    """__cuda_array_interface__ view of communicator memory (no ownership)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class Communicator:
    """A tw_comm_t: `world` ranks on `devices` with symmetric INPUT/OUTPUT/RESIDUAL
    buffers (the B200 analogue of the reference's in-process RankGroup,
    proj/include/weavesim/collectives.hpp:36-46)."""

    def __init__(self, world: int, devices, buffer_bytes: int, transport: int = TW_TRANSPORT_AUTO):
        devs = (c_int * world)(*devices)
        h = c_void_p()
        check(_lib.lib.tw_comm_create(world, devs, buffer_bytes, transport, ctypes.byref(h)))
        self._h = h
        self.world = world
        self.devices = list(devices)
        w, tr, nb = c_int(), c_int(), c_size_t()
        check(_lib.lib.tw_comm_info(h, ctypes.byref(w), ctypes.byref(tr), ctypes.byref(nb)))
        self.transport = tr.value
        self.buffer_bytes = nb.value

    @property
    def transport_name(self) -> str:
        return _lib.TRANSPORT_NAMES[self.transport]

    def close(self) -> None:
        if self._h:
            check(_lib.lib.tw_comm_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def buffer_ptr(self, rank: int, which: int) -> int:
        p = c_void_p()
        check(_lib.lib.tw_comm_buffer(self._h, rank, which, ctypes.byref(p)))
        return p.value

    def buffer(self, rank: int, which: int, shape, dtype):
        """torch view of a symmetric buffer of `rank` (on its device)."""
        import torch
        typestr = {torch.bfloat16: "<V2", torch.float32: "<f4"}[dtype]
        n = 1
        for s in shape:
            n *= s
        if n * (2 if dtype == torch.bfloat16 else 4) > self.buffer_bytes:
            raise DimensionError("buffer view exceeds the communicator buffer size")
        with torch.cuda.device(self.devices[rank]):
            if dtype == torch.bfloat16:
                raw = torch.as_tensor(_DevBuf(self.buffer_ptr(rank, which), (n,), "<i2"), device="cuda")
                return raw.view(torch.bfloat16).view(*shape)
            return torch.as_tensor(_DevBuf(self.buffer_ptr(rank, which), tuple(shape), typestr), device="cuda")

    def fused_allreduce_rmsnorm(self, T: int, H: int, residual_shards, weights, eps: float = 1e-5, *, dtype=None,
                                shard_ranges=None, sm_budget: int = 8, gather_residual: bool = False, streams=None,
                                token_offset: int = 0, nvls_depth: int = 0):
        """Kernel K1 on every rank of this communicator (see tw.h).  nvls_depth:
        rows of ld_reduce in flight per row group on the NVLS kernel (1..3, 0 =
        the library default)."""
        import torch
        W = self.world
        if dtype is None:
            dtype = residual_shards[0].dtype
        code = TW_BF16 if dtype == torch.bfloat16 else TW_F32
        ranges = None
        if shard_ranges is not None:
            flat = [v for rg in shard_ranges for v in rg]
            ranges = (c_int64 * len(flat))(*flat)
        res = (c_void_p * W)(*[_ptr(t) if t is not None and t.numel() else None for t in residual_shards])
        wts = (c_void_p * W)(*[_ptr(t) for t in weights])
        strs = None
        if streams is not None:
            strs = (c_void_p * W)(*[_stream_handle(s) for s in streams])
        else:
            strs = (c_void_p * W)(*[_current_raw_stream(d) for d in self.devices])
        check(_lib.lib.tw_fused_allreduce_rmsnorm_group(self._h, T, H, token_offset, ranges, res, wts, float(eps), code,
                                                        int(sm_budget),
                                                        (TW_GATHER_RESIDUAL if gather_residual else 0)
                                                        | TW_NVLS_DEPTH(nvls_depth), strs))

    def allreduce(self, T: int, H: int, dtype, *, sm_budget: int = 8, streams=None, token_offset: int = 0):
        """Unfused AllReduce baseline (K3): OUTPUT = sum_r INPUT on every rank."""
        import torch
        W = self.world
        code = TW_BF16 if dtype == torch.bfloat16 else TW_F32
        if streams is not None:
            strs = (c_void_p * W)(*[_stream_handle(s) for s in streams])
        else:
            strs = (c_void_p * W)(*[_current_raw_stream(d) for d in self.devices])
        check(_lib.lib.tw_allreduce_group(self._h, T, H, token_offset, code, int(sm_budget), strs))

    def check(self) -> None:
        check(_lib.lib.tw_comm_check(self._h))
