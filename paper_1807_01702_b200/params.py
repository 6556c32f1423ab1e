"""Layer parameter blocks and per-channel statistics (host side).

Mirrors the reference's ``ConvParams`` / ``BNParams`` / ``ChannelStats``
(``pkg/src/bnfuse/ops.py:37-143``): same field names, defaults, validation and
error types, so graphs built here carry parameters interchangeable with the
reference's.  Weights stay in the reference layout ``(out_c, in_c, kh, kw)``
on the host; the device engine re-lays them out once (see ``engine.py``).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ShapeError


@dataclass
class ConvParams:
    """2-D convolution; weights (out_c, in_c, kh, kw).  ops.py:37-69."""

    in_c: int
    out_c: int
    kh: int
    kw: int
    stride: int = 1
    pad: int = 0
    weights: np.ndarray = None
    bias: np.ndarray = None
    name: str = "conv"

    def __post_init__(self):
        if self.weights is None:
            self.weights = np.zeros((self.out_c, self.in_c, self.kh, self.kw), np.float32)
        if self.bias is None:
            self.bias = np.zeros(self.out_c, dtype=self.weights.dtype)
        want = (self.out_c, self.in_c, self.kh, self.kw)
        if tuple(self.weights.shape) != want:
            raise ShapeError(f"{self.name}: weights {tuple(self.weights.shape)} != {want}")
        if self.stride < 1 or self.pad < 0:
            raise ShapeError(f"{self.name}: need stride >= 1 and pad >= 0")

    def out_hw(self, h: int, w: int) -> tuple[int, int]:
        oh = (h + 2 * self.pad - self.kh) // self.stride + 1
        ow = (w + 2 * self.pad - self.kw) // self.stride + 1
        if oh < 1 or ow < 1:
            raise ShapeError(f"{self.name}: non-positive output for {h}x{w}")
        return oh, ow


@dataclass
class BNParams:
    """Per-channel gamma/beta with eps (default 1e-5).  ops.py:72-91."""

    gamma: np.ndarray
    beta: np.ndarray
    eps: float = 1e-5
    name: str = "bn"

    def __post_init__(self):
        self.gamma = np.asarray(self.gamma)
        self.beta = np.asarray(self.beta)
        if self.gamma.ndim != 1 or self.gamma.shape != self.beta.shape:
            raise ShapeError(f"{self.name}: gamma/beta must be equal-length vectors")
        if not self.eps > 0:
            raise ShapeError(f"{self.name}: eps must be positive")

    @property
    def channels(self) -> int:
        return int(self.gamma.shape[0])


@dataclass
class ChannelStats:
    """Population statistics from float64 running sums.  ops.py:94-125.

    ``count`` = n*h*w; ``var`` is clamped at 0 (E[x^2]-E[x]^2 can round
    negative).  On the device path the same record is produced by the
    ``bnff_stats_finalize`` kernel from per-tile partials.
    """

    sum_x: np.ndarray
    sum_x2: np.ndarray
    count: int
    mean: np.ndarray = field(default=None)
    var: np.ndarray = field(default=None)

    @classmethod
    def from_sums(cls, sum_x, sum_x2, count: int) -> "ChannelStats":
        mean = sum_x / count
        return cls(sum_x=sum_x, sum_x2=sum_x2, count=count, mean=mean,
                   var=np.maximum(sum_x2 / count - mean * mean, 0.0))

    def inv_std(self, eps: float) -> np.ndarray:
        return 1.0 / np.sqrt(np.maximum(self.var, 0.0) + eps)

    def slice(self, lo: int, hi: int) -> "ChannelStats":
        return ChannelStats(self.sum_x[lo:hi], self.sum_x2[lo:hi], self.count,
                            self.mean[lo:hi], self.var[lo:hi])


def concat_stats(parts: list[ChannelStats]) -> ChannelStats:
    """Stats of a channel concatenation = concatenated per-piece vectors (ops.py:128-143)."""
    count = parts[0].count
    if any(p.count != count for p in parts):
        raise ShapeError("concatenated pieces must share n*h*w")
    cat = np.concatenate
    return ChannelStats(cat([p.sum_x for p in parts]), cat([p.sum_x2 for p in parts]), count,
                        cat([p.mean for p in parts]), cat([p.var for p in parts]))
