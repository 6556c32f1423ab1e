"""Host-side value containers and the counter-based RNG.

``Rng`` must reproduce the reference's draws exactly (``pkg/src/bnfuse/tensor.py:82-112``):
every call opens a fresh numpy Philox generator keyed by ``(seed, call index)``
and takes one bulk draw, so parameters and synthetic inputs generated here are
bit-identical to the reference's for the same seed and call order.  That is
what makes the GPU-vs-oracle parity tests compare like with like.
"""

from __future__ import annotations

import struct

import numpy as np

from .errors import InvalidRangeError, ShapeError

_U64 = (1 << 64) - 1


class Rng:
    """Deterministic stream keyed by (seed, call count) -- Philox under the hood."""

    def __init__(self, seed: int):
        self.seed = int(seed)
        self._calls = 0

    def _next(self) -> np.random.Generator:
        key = (self.seed & _U64, self._calls)
        self._calls += 1
        return np.random.Generator(np.random.Philox(key=key))

    def uniform(self, dims, lo: float, hi: float, dtype=np.float32) -> np.ndarray:
        if not lo < hi:
            raise InvalidRangeError(f"uniform needs lo < hi, got [{lo}, {hi})")
        u = self._next().random(tuple(int(d) for d in dims), dtype=np.float64)
        # same float64 expression order as the reference => bit-identical draws
        return ((hi - lo) * u + lo).astype(dtype)

    def normal(self, dims, dtype=np.float32) -> np.ndarray:
        z = self._next().standard_normal(tuple(int(d) for d in dims), dtype=np.float64)
        return z.astype(dtype)

    def integers(self, lo: int, hi: int) -> int:
        return int(self._next().integers(lo, hi))


def check_dims(dims) -> tuple:
    if len(dims) != 4:
        raise ShapeError(f"expected (n, c, h, w), got {dims!r}")
    dims = tuple(int(d) for d in dims)
    if min(dims) < 1:
        raise ShapeError(f"dims must be >= 1, got {dims}")
    if int(np.prod(dims, dtype=np.int64)) > 2**40:
        raise ShapeError(f"dims too large: {dims}")
    return dims


class Tensor4D:
    """NCHW host container with the reference's debug dump format
    (four little-endian u64 dims followed by f32 payload)."""

    __slots__ = ("data",)

    def __init__(self, data: np.ndarray):
        if data.ndim != 4:
            raise ShapeError(f"Tensor4D wants 4-D data, got ndim={data.ndim}")
        check_dims(data.shape)
        if data.dtype not in (np.float32, np.float64):
            data = data.astype(np.float32)
        self.data = np.ascontiguousarray(data)

    @property
    def dims(self):
        return self.data.shape

    @property
    def dtype(self):
        return self.data.dtype

    def dump_bytes(self) -> bytes:
        return struct.pack("<4Q", *self.dims) + self.data.astype("<f4").tobytes()

    @classmethod
    def load_bytes(cls, blob: bytes) -> "Tensor4D":
        dims = struct.unpack("<4Q", blob[:32])
        flat = np.frombuffer(blob[32:], dtype="<f4")
        if flat.size != int(np.prod(dims)):
            raise ShapeError(f"payload {flat.size} values, dims {dims}")
        return cls(flat.reshape(dims).astype(np.float32))


def tensor_approx_eq(a, b, rel_tol: float = 1e-5, abs_tol: float = 0.0):
    """|a-b| <= abs_tol + rel_tol*max(|a|,|b|) elementwise; returns (ok, worst_info)."""
    da = np.asarray(a.data if isinstance(a, Tensor4D) else a, dtype=np.float64)
    db = np.asarray(b.data if isinstance(b, Tensor4D) else b, dtype=np.float64)
    if da.shape != db.shape:
        raise ShapeError(f"shape mismatch {da.shape} vs {db.shape}")
    slack = abs_tol + rel_tol * np.maximum(np.abs(da), np.abs(db))
    excess = np.abs(da - db) - slack
    i = np.unravel_index(int(np.argmax(excess)), da.shape)
    return bool(np.all(excess <= 0)), (tuple(int(v) for v in i), float(abs(da[i] - db[i])), float(slack[i]))
