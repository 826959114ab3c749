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
    lib.tw_workload_last_error.restype = ctypes.c_char_p
    lib.tw_workload_last_error.argtypes = []
    lib.tw_synth_trace.argtypes = [c_int64, c_int64, c_int64, POINTER(Request)]
    lib.tw_load_trace.argtypes = [ctypes.c_char_p, POINTER(Request), c_int64, POINTER(c_int64)]
    lib.tw_save_trace.argtypes = [POINTER(Request), c_int64, ctypes.c_char_p]
    lib.tw_form_batches.argtypes = [POINTER(Request), c_int64, c_int64, POINTER(IterationBatch), c_int64,
                                    POINTER(PrefillSlice), c_int64, POINTER(c_int64), POINTER(c_int64)]
    for f in ("tw_make_split_plan", "tw_smart_offset_analytic", "tw_smart_offset_sweep",
              "tw_place_sequence_boundaries", "tw_synth_trace", "tw_load_trace", "tw_save_trace",
              "tw_form_batches"):
        getattr(lib, f).restype = c_int
    return lib


class Request(Structure):
    """tw_request = weavesim::Request (workloads.hpp:12-17)."""
    _fields_ = [("id", c_int64), ("prompt_tokens", c_int64), ("output_tokens", c_int64), ("arrival_s", c_double)]


class PrefillSlice(Structure):
    _fields_ = [("request_id", c_int64), ("start", c_int64), ("len", c_int64)]


class IterationBatch(Structure):
    _fields_ = [("total_tokens", c_int64), ("decode_token_count", c_int64), ("kv_context", c_int64),
                ("first_slice", c_int64), ("num_slices", c_int64)]


class ThroughputResult(Structure):
    _fields_ = [("tokens_per_sec", c_double), ("iterations", c_int64), ("total_tokens", c_int64),
                ("total_seconds", c_double), ("mean_iteration_latency", c_double)]


_S = _split_lib()


def _wcheck(status: int) -> None:
    check(status, _S.tw_workload_last_error)


def _requests(requests):
    """[(prompt, output[, arrival_s])] or Request structs -> a tw_request array."""
    arr = (Request * max(len(requests), 1))()
    for i, r in enumerate(requests):
        if isinstance(r, Request):
            arr[i] = r
        else:
            arr[i] = Request(i, r[0], r[1], float(r[2]) if len(r) > 2 else 0.0)
    return arr


def synth_trace(count: int, prompt_len: int, output_len: int):
    """weavesim::synth_trace -> [(prompt, output, arrival_s)]."""
    arr = (Request * max(count, 1))()
    _wcheck(_S.tw_synth_trace(count, prompt_len, output_len, arr))
    return [(arr[i].prompt_tokens, arr[i].output_tokens, arr[i].arrival_s) for i in range(count)]


def load_trace(path: str):
    """weavesim::load_trace (JSONL) -> [(prompt, output, arrival_s)]; ParseError like the reference."""
    n = c_int64()
    _wcheck(_S.tw_load_trace(path.encode(), None, 0, ctypes.byref(n)))
    arr = (Request * max(n.value, 1))()
    _wcheck(_S.tw_load_trace(path.encode(), arr, n.value, ctypes.byref(n)))
    return [(arr[i].prompt_tokens, arr[i].output_tokens, arr[i].arrival_s) for i in range(n.value)]


def save_trace(requests, path: str) -> None:
    _wcheck(_S.tw_save_trace(_requests(requests), len(requests), path.encode()))


def form_batches(requests, chunk_size: int):
    """weavesim::form_batches -> [(total_tokens, decode_token_count, kv_context, [(request_id, start, len)])]."""
    reqs = _requests(requests)
    nb, ns = c_int64(), c_int64()
    st = _S.tw_form_batches(reqs, len(requests), chunk_size, None, 0, None, 0, ctypes.byref(nb), ctypes.byref(ns))
    if st != 1:  # TW_ERR_DIMENSION = "arrays too small" (sizes reported)
        _wcheck(st)
    b = (IterationBatch * max(nb.value, 1))()
    sl = (PrefillSlice * max(ns.value, 1))()
    _wcheck(_S.tw_form_batches(reqs, len(requests), chunk_size, b, nb.value, sl, ns.value, ctypes.byref(nb),
                               ctypes.byref(ns)))
    out = []
    for k in range(nb.value):
        x = b[k]
        slices = [(sl[j].request_id, sl[j].start, sl[j].len) for j in range(x.first_slice, x.first_slice + x.num_slices)]
        out.append((x.total_tokens, x.decode_token_count, x.kv_context, slices))
    return out


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
    lib.tw_weave_run_batch.argtypes = [c_void_p, c_int64, c_int64, c_int64, c_int, c_int, c_int, c_int,
                                       ctypes.c_uint, POINTER(c_float)]
    lib.tw_weave_run_batch.restype = c_int
    lib.tw_weave_throughput.argtypes = [c_void_p, POINTER(Request), c_int64, c_int64, c_int, c_int64, c_int, c_int,
                                        c_int, c_int, ctypes.c_uint, POINTER(ThroughputResult), POINTER(c_double),
                                        c_int64]
    lib.tw_weave_throughput.restype = c_int
    lib.tw_weave_emulate_comm.argtypes = [c_void_p, POINTER(c_int64), POINTER(c_float), POINTER(c_float), c_int,
                                          c_int]
    lib.tw_weave_emulate_comm.restype = c_int
    lib.tw_weave_cublas_version.restype = c_int
    lib.tw_weave_cublas_version.argtypes = []
    lib.tw_weave_last_error.restype = ctypes.c_char_p
    lib.tw_weave_last_error.argtypes = []
    lib.tw_weave_trace.argtypes = [c_void_p, c_int, POINTER(c_int), POINTER(c_int), POINTER(c_int), POINTER(c_int),
                                   POINTER(c_float), POINTER(c_float)]
    lib.tw_weave_buffer.argtypes = [c_void_p, c_int, POINTER(c_void_p), POINTER(ctypes.c_size_t)]
    for f in ("tw_weave_create", "tw_weave_destroy", "tw_weave_run", "tw_weave_trace", "tw_weave_buffer"):
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
            self._check(self._L.tw_weave_create_tp(ctypes.byref(self.spec), max_tokens, comm, ctypes.byref(h)))
        else:
            self._check(self._L.tw_weave_create(ctypes.byref(self.spec), max_tokens, device, ctypes.byref(h)))
        self._h = h

    @property
    def cublas_version(self) -> int:
        """The cuBLAS version the runner's GEMMs bind (e.g. 120901)."""
        return int(self._L.tw_weave_cublas_version())

    def _check(self, status: int) -> None:
        check(status, self._L.tw_weave_last_error)

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
        self._check(self._L.tw_weave_run_ex(self._h, T, prefix, MODES[mode], boundary_sms, gemm_sms, layers,
                                      1 if graph else 0, ctypes.byref(us)))
        return us.value

    def run_batch(self, T: int, kv_context: int, mode: str, prefix: int = 0, boundary_sms: int = 16,
                  gemm_sms: int = 0, layers: int = 4, graph: bool = False) -> float:
        """run() for one serving batch with kv_context prior-context tokens attended."""
        us = c_float()
        self._check(self._L.tw_weave_run_batch(self._h, T, prefix, kv_context, MODES[mode], boundary_sms, gemm_sms, layers,
                                         1 if graph else 0, ctypes.byref(us)))
        return us.value

    def throughput(self, requests, chunk_size: int, mode: str, num_layers: int = 80, layers_measured: int = 2,
                   boundary_sms: int = -1, gemm_sms: int = 0, graph: bool = False, threshold: int | None = None):
        """Measured serving throughput over form_batches(requests, chunk_size)
        (tw_weave_throughput): a ThroughputResult dict with per-iteration latencies.
        boundary_sms = -1 (TW_WEAVE_AUTO_BUDGET): the weaved batches' fused-op SM
        budget is measured once per batch size over 16/32/64."""
        reqs = _requests(requests)
        n_iter = len(form_batches(requests, chunk_size))
        lat = (c_double * max(n_iter, 1))()
        res = ThroughputResult()
        self._check(self._L.tw_weave_throughput(self._h, reqs, len(requests), chunk_size, MODES[mode],
                                          self.threshold if threshold is None else threshold, num_layers,
                                          layers_measured, boundary_sms, gemm_sms, 1 if graph else 0,
                                          ctypes.byref(res), lat, n_iter))
        return {"tokens_per_sec": res.tokens_per_sec, "iterations": res.iterations,
                "total_tokens": res.total_tokens, "total_seconds": res.total_seconds,
                "mean_iteration_latency": res.mean_iteration_latency,
                "iteration_latencies": [lat[i] for i in range(min(n_iter, res.iterations))]}

    def emulate_comm(self, tokens=(), fused_us=(), allreduce_us=(), sms: int = 16):
        """What-if: the boundary op becomes an SM-holding emulation with the
        table's latency (tw_weave_emulate_comm); no arguments = the real op."""
        n = len(tokens)
        t = (c_int64 * max(n, 1))(*tokens)
        f = (c_float * max(n, 1))(*fused_us)
        a = (c_float * max(n, 1))(*allreduce_us)
        self._check(self._L.tw_weave_emulate_comm(self._h, t, f, a, n, sms))

    def trace(self, max_events: int = 64):
        n = c_int()
        op, sp, st = (c_int * max_events)(), (c_int * max_events)(), (c_int * max_events)()
        a, b = (c_float * max_events)(), (c_float * max_events)()
        self._check(self._L.tw_weave_trace(self._h, max_events, ctypes.byref(n), op, sp, st, a, b))
        return [{"op": OPS[op[i]], "split": SPLITS[sp[i]], "stream": "comm" if st[i] else "compute",
                 "start_us": a[i], "end_us": b[i]} for i in range(n.value)]

    BUFFERS = {"hidden": 0, "residual": 1, "partial": 2, "w_qkv": 3, "w_o": 4, "w_up": 5, "w_down": 6,
               "norm_weight": 7}

    def buffer(self, which: str):
        """torch view (no copy) of one of the runner's device buffers
        (tw_weave_buffer): bf16 1-D, or fp32 for "norm_weight"."""
        import torch
        from . import _DevBuf
        p, nb = c_void_p(), ctypes.c_size_t()
        self._check(self._L.tw_weave_buffer(self._h, self.BUFFERS[which], ctypes.byref(p), ctypes.byref(nb)))
        if which == "norm_weight":
            return torch.as_tensor(_DevBuf(p.value, (nb.value // 4,), "<f4"), device="cuda")
        raw = torch.as_tensor(_DevBuf(p.value, (nb.value // 2,), "<i2"), device="cuda")
        return raw.view(torch.bfloat16)
