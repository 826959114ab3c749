"""Shared input generators and tolerance rules for the parity tests."""
from __future__ import annotations

import numpy as np

from tests.golden.make_golden import group_inputs, norm_inputs  # noqa: F401  (re-export)


def bf16_round(a: np.ndarray) -> np.ndarray:
    """RNE to bf16, as fp32."""
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def assert_bf16_close(got: np.ndarray, want: np.ndarray, rel: float = 2e-2, what: str = "output") -> None:
    """north_star's bf16 bar, guarded for cancellation:
    |got - want| <= rel * max(|want|, rms_row(want)) elementwise."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    if want.size == 0:
        return
    rms = np.sqrt(np.mean(want * want, axis=-1, keepdims=True))
    bound = rel * np.maximum(np.abs(want), rms) + 1e-30
    err = np.abs(got - want)
    bad = err > bound
    assert not bad.any(), f"{what}: {bad.sum()} elements out of tolerance, max err/bound {np.max(err / bound):.3f}"


def assert_abs_close(got, want, atol: float = 1e-5, what: str = "output") -> None:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    if want.size:
        err = np.max(np.abs(got - want))
        assert err <= atol, f"{what}: max abs err {err:.3e} > {atol}"
