"""Parity checkers for the TokenWeave hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker.  The product
(libtw.so, libweavesim_b200.so) never loads it.

  Oracle  : ctypes over liboracle.so, the C restatement (tw_oracle.c) of
            proj/src/{numerics,collectives,splitter,wavemodel}.cpp.
  RefLib  : ctypes over _ref/libweavesim_ref.so, the reference's own sources
            compiled unmodified (oracle/Makefile) + ref_capi.cpp adapter.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int64, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libweavesim_ref.so")

_F = POINTER(c_float)
_I64 = POINTER(c_int64)


def _fp(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_F)


def _ptr_array(arrs):
    return (c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


class StatusError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: status {code}")
        self.code = code


class Oracle:
    """The C restatement (parity pinned against RefLib and tests/golden)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make oracle)")
        L = ctypes.CDLL(path)
        L.orc_token_shard_map.argtypes = [c_int64, c_int, _I64]
        L.orc_shard_map_validate.argtypes = [_I64, c_int, c_int64]
        L.orc_rmsnorm_residual.argtypes = [_F, _F, _F, c_int64, c_int64, c_float, _F, _F]
        L.orc_all_reduce.argtypes = [c_int, c_void_p, c_int64, c_int64, _F]
        L.orc_fused_allreduce_rmsnorm.argtypes = [c_int, c_void_p, c_void_p, _I64, _F, c_int64, c_int64, c_float, _F]
        L.orc_cta_count.argtypes = [c_int64, c_int64, c_int64]
        L.orc_cta_count.restype = c_int64
        L.orc_wave_count.argtypes = [c_int64, c_int64]
        L.orc_wave_count.restype = c_int64
        L.orc_smart_offset_analytic.argtypes = [c_int64, c_int64, c_int64, c_int64]
        L.orc_smart_offset_analytic.restype = c_int64
        L.orc_make_split_plan.argtypes = [c_int64, c_int64, c_int64, c_int64, c_int64, _I64]
        L.orc_place_sequence_boundaries.argtypes = [_I64, c_int, c_int64, c_int64, _I64]
        L.orc_round_to_bf16.argtypes = [_F, _F, c_int64]
        _D = POINTER(c_double)
        L.orc_form_batches.argtypes = [_I64, _I64, _D, c_int64, c_int64, _I64, c_int64, _I64, c_int64, _I64]
        self.L = L

    def token_shard_map(self, T: int, world: int):
        buf = (c_int64 * (2 * max(world, 1)))()
        st = self.L.orc_token_shard_map(T, world, buf)
        if st:
            raise StatusError(st, "token_shard_map")
        return [(buf[2 * r], buf[2 * r + 1]) for r in range(world)]

    def shard_map_validate(self, ranges, total: int) -> int:
        flat = [v for rg in ranges for v in rg]
        buf = (c_int64 * max(len(flat), 1))(*flat)
        return self.L.orc_shard_map_validate(buf, len(ranges), total)

    def rmsnorm_residual(self, inp: np.ndarray, res: np.ndarray, weight: np.ndarray, eps: float = 1e-5):
        inp = np.ascontiguousarray(inp, np.float32)
        res = np.ascontiguousarray(res, np.float32)
        weight = np.ascontiguousarray(weight, np.float32)
        T, H = inp.shape
        out = np.empty_like(inp)
        rout = np.empty_like(inp)
        st = self.L.orc_rmsnorm_residual(_fp(inp), _fp(res), _fp(weight), T, H, eps, _fp(out), _fp(rout))
        if st:
            raise StatusError(st, "rmsnorm_residual")
        return out, rout

    def all_reduce(self, inputs):
        inputs = [np.ascontiguousarray(a, np.float32) for a in inputs]
        T, H = inputs[0].shape
        out = np.empty_like(inputs[0])
        st = self.L.orc_all_reduce(len(inputs), _ptr_array(inputs), T, H, _fp(out))
        if st:
            raise StatusError(st, "all_reduce")
        return out

    def fused_allreduce_rmsnorm(self, inputs, residual_shards, weight, ranges=None, eps: float = 1e-5):
        """Returns (output [T,H], updated residual shards); inputs untouched."""
        inputs = [np.ascontiguousarray(a, np.float32) for a in inputs]
        world = len(inputs)
        T, H = inputs[0].shape
        if ranges is None:
            ranges = self.token_shard_map(T, world)
        shards = [np.array(s, np.float32, copy=True).reshape(-1, H) for s in residual_shards]
        flat = (c_int64 * (2 * world))(*[v for rg in ranges for v in rg])
        out = np.empty((T, H), np.float32)
        w = np.ascontiguousarray(weight, np.float32)
        st = self.L.orc_fused_allreduce_rmsnorm(world, _ptr_array(inputs), _ptr_array(shards), flat, _fp(w), T, H,
                                                eps, _fp(out))
        if st:
            raise StatusError(st, "fused_allreduce_rmsnorm")
        return out, shards

    def smart_offset_analytic(self, T, num_sms, tile_tokens, cta_columns) -> int:
        return self.L.orc_smart_offset_analytic(T, num_sms, tile_tokens, cta_columns)

    def make_split_plan(self, T, threshold, num_sms, tile_tokens, cta_columns):
        out = (c_int64 * 4)()
        st = self.L.orc_make_split_plan(T, threshold, num_sms, tile_tokens, cta_columns, out)
        if st:
            raise StatusError(st, "make_split_plan")
        return tuple(out)

    def place_sequence_boundaries(self, lengths, total, prefix):
        n = len(lengths)
        arr = (c_int64 * max(n, 1))(*lengths)
        out = (c_int64 * max(n, 1))()
        st = self.L.orc_place_sequence_boundaries(arr, n, total, prefix, out)
        if st:
            raise StatusError(st, "place_sequence_boundaries")
        return list(out)[:n]

    def form_batches(self, requests, chunk_size):
        """requests: [(prompt, output, arrival_s)] -> [(total, decode, kv, [(id, start, len)])]."""
        n = len(requests)
        pr = (c_int64 * max(n, 1))(*[r[0] for r in requests])
        ou = (c_int64 * max(n, 1))(*[r[1] for r in requests])
        ar = (c_double * max(n, 1))(*[float(r[2]) if len(r) > 2 else 0.0 for r in requests])
        counts = (c_int64 * 2)()
        st = self.L.orc_form_batches(pr, ou, ar, n, chunk_size, None, 0, None, 0, counts)
        if st not in (0, 1):
            raise StatusError(st, "form_batches")
        nb, ns = counts[0], counts[1]
        out4 = (c_int64 * (4 * max(nb, 1)))()
        sl3 = (c_int64 * (3 * max(ns, 1)))()
        st = self.L.orc_form_batches(pr, ou, ar, n, chunk_size, out4, nb, sl3, ns, counts)
        if st:
            raise StatusError(st, "form_batches")
        return _unpack_batches(out4, sl3, nb)

    def round_bf16(self, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        out = np.empty_like(a)
        self.L.orc_round_to_bf16(_fp(a), _fp(out), a.size)
        return out


class RefLib:
    """The reference's own code (compiled unmodified), for pinning the oracle
    and as the reference CPU arm of bench.py."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make ref; needs /root/reference)")
        L = ctypes.CDLL(path)
        L.ref_rmsnorm_residual.argtypes = [_F, _F, _F, c_int64, c_int64, c_float, _F, _F]
        L.ref_token_shard_map.argtypes = [c_int64, c_int, _I64]
        L.ref_shard_map_validate.argtypes = [_I64, c_int, c_int64]
        L.ref_all_reduce.argtypes = [c_int, c_void_p, c_int64, c_int64, _F]
        L.ref_fused_allreduce_rmsnorm.argtypes = [c_int, c_void_p, c_void_p, _I64, _F, c_int64, c_int64, c_float,
                                                  c_int, _F]
        L.ref_fill_group.argtypes = [c_uint64, c_int, c_int64, c_int64, _F, _F, _F]
        L.ref_fill_group.restype = None
        L.ref_acceptance_seed.argtypes = [c_int, c_int64, c_int64, c_int]
        L.ref_acceptance_seed.restype = c_uint64
        L.ref_smart_offset_analytic.argtypes = [c_int64, c_int, c_int, c_int]
        L.ref_smart_offset_analytic.restype = c_int64
        L.ref_make_split_plan.argtypes = [c_char_p, c_char_p, c_int64, _I64, _I64]
        L.ref_layer_latency.argtypes = [c_char_p, c_char_p, c_int64, c_char_p, POINTER(c_double)]
        L.ref_time_fused.argtypes = [c_int, c_int64, c_int64, c_int, c_int, POINTER(c_double), POINTER(c_double)]
        L.ref_calibrate_file.argtypes = [c_char_p, POINTER(c_double)]
        L.ref_time_rmsnorm.argtypes = [c_int64, c_int64, c_int, c_int, POINTER(c_double), POINTER(c_double)]
        _D = POINTER(c_double)
        L.ref_form_batches.argtypes = [_I64, _D, c_int64, c_int64, _I64, c_int64, _I64, c_int64, _I64]
        L.ref_save_trace.argtypes = [_I64, _D, c_int64, c_char_p]
        L.ref_load_trace.argtypes = [c_char_p, _I64, _D, c_int64, _I64]
        L.ref_simulate_throughput.argtypes = [c_char_p, c_char_p, c_char_p, _I64, c_int64, c_int64, _D]
        L.ref_cmd_throughput_csv.argtypes = [c_char_p, c_char_p, c_int64, c_uint64, c_char_p, c_int64]
        L.ref_cmd_throughput_csv.restype = c_int64
        L.ref_chatlike_trace.argtypes = [c_int64, c_uint64, _I64]
        L.ref_timeline_json.argtypes = [c_char_p, c_char_p, c_int64, c_char_p, c_char_p, c_int64]
        L.ref_timeline_json.restype = c_int64
        self.L = L

    def rmsnorm_residual(self, inp, res, weight, eps=1e-5):
        inp = np.ascontiguousarray(inp, np.float32)
        res = np.ascontiguousarray(res, np.float32)
        weight = np.ascontiguousarray(weight, np.float32)
        T, H = inp.shape
        out = np.empty_like(inp)
        rout = np.empty_like(inp)
        st = self.L.ref_rmsnorm_residual(_fp(inp), _fp(res), _fp(weight), T, H, eps, _fp(out), _fp(rout))
        if st:
            raise StatusError(st, "ref_rmsnorm_residual")
        return out, rout

    def token_shard_map(self, T, world):
        buf = (c_int64 * (2 * max(world, 1)))()
        st = self.L.ref_token_shard_map(T, world, buf)
        if st:
            raise StatusError(st, "ref_token_shard_map")
        return [(buf[2 * r], buf[2 * r + 1]) for r in range(world)]

    def shard_map_validate(self, ranges, total) -> int:
        flat = [v for rg in ranges for v in rg]
        buf = (c_int64 * max(len(flat), 1))(*flat)
        return self.L.ref_shard_map_validate(buf, len(ranges), total)

    def all_reduce(self, inputs):
        inputs = [np.ascontiguousarray(a, np.float32) for a in inputs]
        T, H = inputs[0].shape
        out = np.empty_like(inputs[0])
        st = self.L.ref_all_reduce(len(inputs), _ptr_array(inputs), T, H, _fp(out))
        if st:
            raise StatusError(st, "ref_all_reduce")
        return out

    def fused_allreduce_rmsnorm(self, inputs, residual_shards, weight, ranges=None, eps=1e-5, parallel=False):
        inputs = [np.ascontiguousarray(a, np.float32) for a in inputs]
        world = len(inputs)
        T, H = inputs[0].shape
        shards = [np.array(s, np.float32, copy=True).reshape(-1, H) for s in residual_shards]
        flat = None
        if ranges is not None:
            flat = (c_int64 * (2 * world))(*[v for rg in ranges for v in rg])
        out = np.empty((T, H), np.float32)
        w = np.ascontiguousarray(weight, np.float32)
        st = self.L.ref_fused_allreduce_rmsnorm(world, _ptr_array(inputs), _ptr_array(shards), flat, _fp(w), T, H,
                                                eps, 1 if parallel else 0, _fp(out))
        if st:
            raise StatusError(st, "ref_fused_allreduce_rmsnorm")
        return out, shards

    def fill_group(self, seed: int, world: int, T: int, H: int):
        """Acceptance-test draw order (proj/tests/acceptance.cpp:45-66)."""
        inputs = np.empty((world, T, H), np.float32)
        residual = np.empty((T, H), np.float32)
        weight = np.empty((H,), np.float32)
        self.L.ref_fill_group(seed, world, T, H, _fp(inputs), _fp(residual), _fp(weight))
        return inputs, residual, weight

    def acceptance_seed(self, world, T, H, i) -> int:
        return self.L.ref_acceptance_seed(world, T, H, i)

    def smart_offset_analytic(self, T, num_sms, tile_tokens, cta_columns) -> int:
        return self.L.ref_smart_offset_analytic(T, num_sms, tile_tokens, cta_columns)

    def make_split_plan(self, profile: str, model: str, T: int):
        out = (c_int64 * 4)()
        geom = (c_int64 * 4)()
        st = self.L.ref_make_split_plan(profile.encode(), model.encode(), T, out, geom)
        if st:
            raise StatusError(st, "ref_make_split_plan")
        return tuple(out), tuple(geom)

    def layer_latency(self, profile, model, T, mode) -> float:
        s = c_double()
        st = self.L.ref_layer_latency(profile.encode(), model.encode(), T, mode.encode(), ctypes.byref(s))
        if st:
            raise StatusError(st, "ref_layer_latency")
        return s.value

    def calibrate_file(self, path: str) -> dict:
        """The reference calibrate() on a CalibrationTable JSON file."""
        out = (c_double * 6)()
        st = self.L.ref_calibrate_file(path.encode(), out)
        if st:
            raise StatusError(st, "ref_calibrate_file")
        keys = ("ar_intercept_us", "ar_slope_us_per_token", "rmsnorm_intercept_us", "rmsnorm_slope_us_per_token",
                "hbm_bandwidth_effective", "fused_extra_latency_s")
        return dict(zip(keys, list(out)))

    def time_fused(self, world, T, H, parallel, iters, each: bool = False):
        """weavesim::fused_allreduce_rmsnorm timed `iters` times on one set of
        inputs: the median (ms), or every iteration's time with each=True."""
        ms = c_double()
        per = (c_double * max(iters, 1))()
        st = self.L.ref_time_fused(world, T, H, 1 if parallel else 0, iters, ctypes.byref(ms), per)
        if st:
            raise StatusError(st, "ref_time_fused")
        return list(per)[:iters] if each else ms.value

    def time_rmsnorm(self, T, H, threads, iters, each: bool = False):
        """weavesim::rmsnorm_residual over T x H chunked across `threads` host
        threads: the median (ms), or every iteration's time with each=True."""
        ms = c_double()
        per = (c_double * max(iters, 1))()
        st = self.L.ref_time_rmsnorm(T, H, threads, iters, ctypes.byref(ms), per)
        if st:
            raise StatusError(st, "ref_time_rmsnorm")
        return list(per)[:iters] if each else ms.value

    @staticmethod
    def _req_arrays(requests):
        n = len(requests)
        r2 = (c_int64 * (2 * max(n, 1)))(*[v for r in requests for v in (r[0], r[1])])
        ar = (c_double * max(n, 1))(*[float(r[2]) if len(r) > 2 else 0.0 for r in requests])
        return n, r2, ar

    def form_batches(self, requests, chunk_size):
        """weavesim::form_batches itself; same return shape as Oracle.form_batches."""
        n, r2, ar = self._req_arrays(requests)
        counts = (c_int64 * 2)()
        st = self.L.ref_form_batches(r2, ar, n, chunk_size, (c_int64 * 4)(), 0, (c_int64 * 3)(), 0, counts)
        if st not in (0, 1):
            raise StatusError(st, "ref_form_batches")
        nb, ns = counts[0], counts[1]
        out4 = (c_int64 * (4 * max(nb, 1)))()
        sl3 = (c_int64 * (3 * max(ns, 1)))()
        st = self.L.ref_form_batches(r2, ar, n, chunk_size, out4, nb, sl3, ns, counts)
        if st:
            raise StatusError(st, "ref_form_batches")
        return _unpack_batches(out4, sl3, nb)

    def save_trace(self, requests, path: str) -> None:
        n, r2, ar = self._req_arrays(requests)
        st = self.L.ref_save_trace(r2, ar, n, path.encode())
        if st:
            raise StatusError(st, "ref_save_trace")

    def load_trace(self, path: str):
        """[(prompt, output, arrival_s)]; StatusError(5) is the reference ParseError."""
        cnt = c_int64()
        st = self.L.ref_load_trace(path.encode(), None, None, 0, ctypes.byref(cnt))
        if st:
            raise StatusError(st, "ref_load_trace")
        n = cnt.value
        r2 = (c_int64 * (2 * max(n, 1)))()
        ar = (c_double * max(n, 1))()
        self.L.ref_load_trace(path.encode(), r2, ar, n, ctypes.byref(cnt))
        return [(r2[2 * i], r2[2 * i + 1], ar[i]) for i in range(n)]

    def simulate_throughput(self, profile, model, mode, requests, chunk_size) -> dict:
        """The reference's MODELED throughput (scheduler + wave model)."""
        n, r2, _ = self._req_arrays(requests)
        out = (c_double * 4)()
        st = self.L.ref_simulate_throughput(profile.encode(), model.encode(), mode.encode(), r2, n, chunk_size, out)
        if st:
            raise StatusError(st, "ref_simulate_throughput")
        return {"tokens_per_sec": out[0], "iterations": int(out[1]), "total_tokens": int(out[2]),
                "total_seconds": out[3]}

    def cmd_throughput_csv(self, model="llama-70b", profile="b200", chunk=2048, seed=42) -> str:
        """The reference CLI `weavesim throughput` CSV, run as shipped."""
        n = self.L.ref_cmd_throughput_csv(model.encode(), profile.encode(), chunk, seed, None, 0)
        if n < 0:
            raise StatusError(9, "ref_cmd_throughput_csv")
        buf = ctypes.create_string_buffer(n + 1)
        self.L.ref_cmd_throughput_csv(model.encode(), profile.encode(), chunk, seed, buf, n + 1)
        return buf.value.decode()

    def timeline_json(self, profile, model, T, mode) -> str:
        """The reference's Timeline::to_json of iteration_timeline (modeled)."""
        n = self.L.ref_timeline_json(profile.encode(), model.encode(), T, mode.encode(), None, 0)
        if n < 0:
            raise StatusError(9, "ref_timeline_json")
        buf = ctypes.create_string_buffer(n + 1)
        self.L.ref_timeline_json(profile.encode(), model.encode(), T, mode.encode(), buf, n + 1)
        return buf.value.decode()

    def chatlike_trace(self, count=96, seed=42):
        out = (c_int64 * (2 * count))()
        st = self.L.ref_chatlike_trace(count, seed, out)
        if st:
            raise StatusError(st, "ref_chatlike_trace")
        return [(out[2 * i], out[2 * i + 1], 0.0) for i in range(count)]


def _unpack_batches(out4, sl3, nb):
    batches, s = [], 0
    for k in range(nb):
        ns = out4[4 * k + 3]
        slices = [(sl3[3 * j], sl3[3 * j + 1], sl3[3 * j + 2]) for j in range(s, s + ns)]
        s += ns
        batches.append((out4[4 * k], out4[4 * k + 1], out4[4 * k + 2], slices))
    return batches


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as fp32 (numpy; test helper)."""
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)
