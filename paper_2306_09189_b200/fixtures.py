"""Fixture I/O in the reference's text formats (reference io.cpp:31-103).

Host-side file handling for the network runner (net.py): the same headers,
value order and `%.17g` precision as the reference's load_* / save_*, so a
fixture written by either side loads bit-identically on the other.

  tensor  "c m\\n" + c*m*m values, one channel row per line        (io.cpp:31-46)
  filter  "c_in c_out kappa\\n" + weights ((f, g, r, s) order) + c_out biases (io.cpp:48-67)
  linear  "out in\\n" + out*in weights (row-major) + out biases      (io.cpp:69-86)
  poly    "degree bound\\n" + degree+1 Chebyshev coefficients        (io.cpp:88-103)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class ImageTensor:
    """tensor.hpp:18-37: data[(ch * m + i) * m + j]"""
    c: int
    m: int
    data: np.ndarray

    def __post_init__(self):
        self.data = np.ascontiguousarray(self.data, dtype=np.float64).reshape(-1)
        if self.data.size != self.c * self.m * self.m:
            raise ValueError("tensor size does not match its header")


@dataclass
class FilterTensor:
    """tensor.hpp:41-74: weights[((f * c_out + g) * kappa + r) * kappa + s]"""
    c_in: int
    c_out: int
    kappa: int
    weights: np.ndarray

    def __post_init__(self):
        self.weights = np.ascontiguousarray(self.weights, dtype=np.float64).reshape(-1)
        if self.weights.size != self.c_in * self.c_out * self.kappa * self.kappa:
            raise ValueError("filter size does not match its header")


@dataclass
class LinearWeights:
    """dense.hpp: w[o * in_features + i], b[o]"""
    out_features: int
    in_features: int
    w: np.ndarray
    b: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def __post_init__(self):
        self.w = np.ascontiguousarray(self.w, dtype=np.float64).reshape(-1)
        self.b = np.ascontiguousarray(self.b, dtype=np.float64).reshape(-1)
        if self.w.size != self.out_features * self.in_features or self.b.size != self.out_features:
            raise ValueError("linear weights do not match their header")


@dataclass
class ChebPoly:
    """act.hpp: sum_k coeffs[k] T_k(x / bound)"""
    coeffs: np.ndarray
    bound: float

    @property
    def degree(self) -> int:
        return len(self.coeffs) - 1


def _read(path: str) -> list[str]:
    try:
        with open(path) as f:
            return f.read().split()
    except OSError:
        raise RuntimeError("cannot open " + path) from None


def _values(tok: list[str], start: int, n: int, path: str) -> np.ndarray:
    if len(tok) < start + n:
        raise RuntimeError("truncated fixture: " + path)
    return np.array([float(x) for x in tok[start:start + n]], dtype=np.float64)


def _header(tok: list[str], n: int, what: str, path: str) -> list[str]:
    if len(tok) < n:
        raise RuntimeError(f"bad {what} header: " + path)
    return tok[:n]


def _fmt(v: float) -> str:
    return f"{v:.17g}"


def _open_out(path: str):
    try:
        return open(path, "w")
    except OSError:
        raise RuntimeError("cannot write " + path) from None


def load_tensor(path: str) -> ImageTensor:
    tok = _read(path)
    c, m = (int(x) for x in _header(tok, 2, "tensor", path))
    return ImageTensor(c, m, _values(tok, 2, c * m * m, path))


def save_tensor(path: str, t: ImageTensor) -> None:
    with _open_out(path) as f:
        f.write(f"{t.c} {t.m}\n")
        for i, v in enumerate(t.data):
            f.write(_fmt(v) + ("\n" if (i + 1) % t.m == 0 else " "))


def load_filter(path: str) -> tuple[FilterTensor, np.ndarray]:
    tok = _read(path)
    ci, co, k = (int(x) for x in _header(tok, 3, "filter", path))
    n = ci * co * k * k
    return FilterTensor(ci, co, k, _values(tok, 3, n, path)), _values(tok, 3 + n, co, path)


def save_filter(path: str, k: FilterTensor, bias=None) -> None:
    bias = np.zeros(0) if bias is None else np.asarray(bias, dtype=np.float64)
    if bias.size and bias.size != k.c_out:
        raise ValueError("bias size mismatch")
    with _open_out(path) as f:
        f.write(f"{k.c_in} {k.c_out} {k.kappa}\n")
        kk = k.kappa * k.kappa
        for i, v in enumerate(k.weights):
            f.write(_fmt(v) + ("\n" if (i + 1) % kk == 0 else " "))
        for g in range(k.c_out):
            f.write(_fmt(bias[g] if bias.size else 0.0) + ("\n" if g + 1 == k.c_out else " "))


def load_linear(path: str) -> LinearWeights:
    tok = _read(path)
    o, i = (int(x) for x in _header(tok, 2, "linear", path))
    return LinearWeights(o, i, _values(tok, 2, o * i, path), _values(tok, 2 + o * i, o, path))


def save_linear(path: str, w: LinearWeights) -> None:
    with _open_out(path) as f:
        f.write(f"{w.out_features} {w.in_features}\n")
        for i, v in enumerate(w.w):
            f.write(_fmt(v) + ("\n" if (i + 1) % w.in_features == 0 else " "))
        for o in range(w.out_features):
            f.write(_fmt(w.b[o]) + ("\n" if o + 1 == w.out_features else " "))


def load_poly(path: str) -> ChebPoly:
    tok = _read(path)
    d, bound = _header(tok, 2, "poly", path)
    d = int(d)
    return ChebPoly(_values(tok, 2, d + 1, path), float(bound))


def save_poly(path: str, p: ChebPoly) -> None:
    with _open_out(path) as f:
        f.write(f"{p.degree} {_fmt(p.bound)}\n")
        for i, v in enumerate(p.coeffs):
            f.write(_fmt(v) + ("\n" if i + 1 == len(p.coeffs) else " "))
