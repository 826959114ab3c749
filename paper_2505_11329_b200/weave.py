"""ctypes plumbing for the weave: the token-split planner (tw_split.h, in
libweavesim_b200.so) and the two-stream layer runner (tw_weave.h, in
libtw_weave.so).  No compute here."""
from __future__ import annotations

import ctypes
import os
from ctypes import CFUNCTYPE, POINTER, Structure, c_double, c_float, c_int, c_int32, c_int64, c_void_p

from ._lib import check

_LIBDIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
MODES = {"fuseonly": 0, "tokenweave": 1, "nocomm": 2, "unfused": 3}
OPS = {0: "attention", 1: "ffn", 2: "fused_ar_norm"}
SPLITS = {0: "prefix", 1: "suffix", 2: "whole"}
SPLIT_MODES = {0: "NoSplit", 1: "FusedOnly", 2: "Overlap"}

# LayerSpec presets (proj/src/presets.cpp:72-97), per-GPU shapes at tp.
PRESETS = {
    "llama-70b": dict(hidden=8192, intermediate=28672, heads=64, kv_heads=8, head_dim=128, experts=1, top_k=1,
                      threshold=1024),
    "qwen-72b": dict(hidden=8192, intermediate=29568, heads=64, kv_heads=8, head_dim=128, experts=1, top_k=1,
                     threshold=1024),
    "mixtral-8x22b": dict(hidden=6144, intermediate=16384, heads=48, kv_heads=8, head_dim=128, experts=8, top_k=2,
                          threshold=4096),
}


def timeline_json(events, latency_us: float) -> dict:
    """Measured per-op timestamps of one layer in the reference's Timeline
    schema (proj/src/scheduler.cpp:301-317): seconds, ids, depends_on edges
    of build_layer_graph (:119-147 weave, :150-181 sequential chains)."""
    n = len(events)
    if n == 8:  # aa fa1 ab fb1 ffa fa2 ffb fb2
        deps = [[], [0], [0], [2, 1], [1], [4, 3], [3], [6, 5]]
    else:
        deps = [[]] + [[i - 1] for i in range(1, n)]
    t0 = min((e["start_us"] for e in events), default=0.0)
    return {"iteration_latency": latency_us * 1e-6,
            "events": [{"id": i, "op": e["op"], "split": e["split"], "stream": e["stream"],
                        "start": (e["start_us"] - t0) * 1e-6, "end": (e["end_us"] - t0) * 1e-6,
                        "depends_on": deps[i]} for i, e in enumerate(events)]}


class LayerSpec(Structure):
    _fields_ = [("hidden", c_int64), ("intermediate", c_int64), ("heads", c_int32), ("kv_heads", c_int32),
                ("head_dim", c_int32), ("experts", c_int32), ("top_k", c_int32), ("tp", c_int32)]


_FWD = CFUNCTYPE(c_double, c_int64, c_int64, c_void_p)


def _split_lib():
    lib = ctypes.CDLL(os.path.join(_LIBDIR, "libweavesim_b200.so"))
    lib.tw_make_split_plan.argtypes = [c_int64, c_int, c_int, c_int, c_int64, POINTER(c_int64), POINTER(c_int64),
                                       POINTER(c_int64), POINTER(c_int)]
    lib.tw_smart_offset_analytic.argtypes = [c_int64, c_int, c_int, c_int, POINTER(c_int64)]
    lib.tw_smart_offset_sweep.argtypes = [c_int64, POINTER(c_int64), c_int, _FWD, c_void_p, POINTER(c_int64)]
    lib.tw_place_sequence_boundaries.argtypes = [POINTER(c_int64), c_int, c_int64, c_int64, POINTER(c_int64)]
    for f in ("tw_make_split_plan", "tw_smart_offset_analytic", "tw_smart_offset_sweep",
              "tw_place_sequence_boundaries"):
        getattr(lib, f).restype = c_int
    return lib


_S = _split_lib()


def make_split_plan(T: int, num_sms: int = 148, tile_tokens: int = 128, cta_columns: int = 32,
                    threshold: int = 1024):
    """(prefix, suffix, offset, mode) -- weavesim::make_split_plan."""
    a, b, o, m = c_int64(), c_int64(), c_int64(), c_int()
    check(_S.tw_make_split_plan(T, num_sms, tile_tokens, cta_columns, threshold, ctypes.byref(a), ctypes.byref(b),
                                ctypes.byref(o), ctypes.byref(m)))
    return a.value, b.value, o.value, m.value


def smart_offset_analytic(T: int, num_sms: int = 148, tile_tokens: int = 128, cta_columns: int = 32) -> int:
    o = c_int64()
    check(_S.tw_smart_offset_analytic(T, num_sms, tile_tokens, cta_columns, ctypes.byref(o)))
    return o.value


def smart_offset_sweep(T: int, forward, grid=(0, 64, 128, 192, 256, 512)) -> int:
    """Algorithm 1: forward(prefix, suffix) -> time."""
    cb = _FWD(lambda a, b, _ctx: float(forward(a, b)))
    arr = (c_int64 * len(grid))(*grid)
    o = c_int64()
    check(_S.tw_smart_offset_sweep(T, arr, len(grid), cb, None, ctypes.byref(o)))
    return o.value


def place_sequence_boundaries(lengths, total: int, prefix: int):
    n = len(lengths)
    arr = (c_int64 * max(n, 1))(*lengths)
    out = (c_int64 * max(n, 1))()
    check(_S.tw_place_sequence_boundaries(arr, n, total, prefix, out))
    return list(out)[:n]


def _weave_lib():
    lib = ctypes.CDLL(os.path.join(_LIBDIR, "libtw_weave.so"))
    lib.tw_weave_create.argtypes = [POINTER(LayerSpec), c_int64, c_int, POINTER(c_void_p)]
    lib.tw_weave_create_tp.argtypes = [POINTER(LayerSpec), c_int64, c_void_p, POINTER(c_void_p)]
    lib.tw_weave_create_tp.restype = c_int
    lib.tw_weave_destroy.argtypes = [c_void_p]
    lib.tw_weave_run.argtypes = [c_void_p, c_int64, c_int64, c_int, c_int, c_int, c_int, POINTER(c_float)]
    lib.tw_weave_run_ex.argtypes = [c_void_p, c_int64, c_int64, c_int, c_int, c_int, c_int, ctypes.c_uint,
                                    POINTER(c_float)]
    lib.tw_weave_run_ex.restype = c_int
    lib.tw_weave_trace.argtypes = [c_void_p, c_int, POINTER(c_int), POINTER(c_int), POINTER(c_int), POINTER(c_int),
                                   POINTER(c_float), POINTER(c_float)]
    for f in ("tw_weave_create", "tw_weave_destroy", "tw_weave_run", "tw_weave_trace"):
        getattr(lib, f).restype = c_int
    return lib


class LayerRunner:
    """One GPU's layer DAG on real streams (include/tw/tw_weave.h)."""

    def __init__(self, model: str = "llama-70b", tp: int = 8, max_tokens: int = 8192, device: int = 0,
                 comm=None, **overrides):
        """comm: a multi-process tw_comm_t (c_void_p) -> TP mode, the boundary
        op is K1 over the communicator (tw_weave_create_tp)."""
        self._L = _weave_lib()
        cfg = dict(PRESETS[model])
        cfg.update(overrides)
        self.threshold = cfg.pop("threshold")
        self.spec = LayerSpec(tp=tp, **cfg)
        self.model = model
        h = c_void_p()
        if comm is not None:
            check(self._L.tw_weave_create_tp(ctypes.byref(self.spec), max_tokens, comm, ctypes.byref(h)))
        else:
            check(self._L.tw_weave_create(ctypes.byref(self.spec), max_tokens, device, ctypes.byref(h)))
        self._h = h

    def close(self):
        if self._h:
            self._L.tw_weave_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, T: int, mode: str, prefix: int = 0, boundary_sms: int = 16, gemm_sms: int = 0,
            layers: int = 4, graph: bool = False) -> float:
        """Device time per layer (us).  graph=True: the layers are captured in
        one CUDA graph and the replay is timed (no per-op trace)."""
        us = c_float()
        check(self._L.tw_weave_run_ex(self._h, T, prefix, MODES[mode], boundary_sms, gemm_sms, layers,
                                      1 if graph else 0, ctypes.byref(us)))
        return us.value

    def trace(self, max_events: int = 64):
        n = c_int()
        op, sp, st = (c_int * max_events)(), (c_int * max_events)(), (c_int * max_events)()
        a, b = (c_float * max_events)(), (c_float * max_events)()
        check(self._L.tw_weave_trace(self._h, max_events, ctypes.byref(n), op, sp, st, a, b))
        return [{"op": OPS[op[i]], "split": SPLITS[sp[i]], "stream": "comm" if st[i] else "compute",
                 "start_us": a[i], "end_us": b[i]} for i in range(n.value)]
