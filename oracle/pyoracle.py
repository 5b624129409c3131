"""TEST INFRASTRUCTURE ONLY — ctypes view of the parity checkers.

* ``Port``: the plain-C restatement (oracle/lmkan_oracle.c -> liblmkan_oracle.so).
* ``Ref``:  the unmodified reference headers behind oracle/ref_shim.cpp
            (oracle/_ref/liblmkan_ref.so, built here from /root/reference and
            shipped to the GPU box as a prebuilt .so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module. The product (paper_2509_07103_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liblmkan_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblmkan_ref.so")
_P = C.c_void_p


def _p(a):
    return C.c_void_p(a.ctypes.data)


def build(quiet: bool = True) -> None:
    """make -C oracle (C port always; _ref only where /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class Port:
    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.lmko_sigma.restype = C.c_double
        L.lmko_sigma.argtypes = [C.c_double]
        L.lmko_build_grid.argtypes = [C.c_int, _P, _P]
        L.lmko_interval_index.argtypes = [C.c_int, C.c_double]
        L.lmko_preamble.argtypes = [C.c_int, _P, _P, C.c_double, C.c_double, _P, _P, _P]
        L.lmko_locate.argtypes = [C.c_int, _P, _P, C.c_int, _P, C.c_int64, _P, _P, _P]
        L.lmko_forward.argtypes = [C.c_int, C.c_int, C.c_int, _P, _P, _P, C.c_double, _P, C.c_int64, _P, C.c_int]
        L.lmko_backward.argtypes = [C.c_int, C.c_int, C.c_int, _P, _P, _P, C.c_double, _P, _P, C.c_int64, _P, _P]
        L.lmko_thresholds_f64.argtypes = [C.c_int, _P]
        L.lmko_thresholds_f32.argtypes = [C.c_int, _P]
        L.lmko_verify_thresholds_f32.restype = C.c_int64
        L.lmko_verify_thresholds_f32.argtypes = [C.c_int, _P, C.c_uint32, C.c_uint32, C.c_int]
        self.L = L

    def sigma(self, x: float) -> float:
        return self.L.lmko_sigma(float(x))

    def build_grid(self, G: int):
        pts = np.zeros(G + 1)
        inv = np.zeros(G * G)
        if self.L.lmko_build_grid(G, _p(pts), _p(inv)) != 0:
            raise ValueError("build_grid: G must be >= 3")
        return pts, inv

    def interval_index(self, G: int, x: float) -> int:
        return self.L.lmko_interval_index(G, float(x))

    def locate(self, G: int, X: np.ndarray):
        X = np.ascontiguousarray(X, np.float64)
        rows, n_in = X.shape
        pts, inv = self.build_grid(G)
        i1 = np.zeros((rows, n_in // 2), np.int32)
        i2 = np.zeros_like(i1)
        w = np.zeros((rows, n_in // 2, 4))
        self.L.lmko_locate(G, _p(pts), _p(inv), n_in, _p(X), rows, _p(i1), _p(i2), _p(w))
        return i1, i2, w

    def forward(self, G: int, P: np.ndarray, X: np.ndarray, gamma: float = 1.0, threads: int = 1):
        X = np.ascontiguousarray(X, np.float64)
        P = np.ascontiguousarray(P, np.float64)
        rows, n_in = X.shape
        n_out = P.size // ((G + 1) ** 2 * (n_in // 2))
        pts, inv = self.build_grid(G)
        Y = np.zeros((rows, n_out))
        self.L.lmko_forward(n_in, n_out, G, _p(pts), _p(inv), _p(P), float(gamma), _p(X), rows, _p(Y), threads)
        return Y

    def backward(self, G: int, P: np.ndarray, X: np.ndarray, dY: np.ndarray, gamma: float = 1.0,
                 dP0: np.ndarray = None, workers: int = 1):
        """lmkan_backward (layer.hpp:141-202), one worker: (dP0 + dP, dX)."""
        X = np.ascontiguousarray(X, np.float64)
        dY = np.ascontiguousarray(dY, np.float64)
        P = np.ascontiguousarray(P, np.float64)
        rows, n_in = X.shape
        n_out = dY.shape[1]
        pts, inv = self.build_grid(G)
        dP = np.zeros(P.shape) if dP0 is None else np.array(dP0, np.float64, copy=True)
        dX = np.zeros((rows, n_in))
        self.L.lmko_backward(n_in, n_out, G, _p(pts), _p(inv), _p(P), float(gamma), _p(X), _p(dY), rows, _p(dP),
                             _p(dX))
        return dP, dX

    def thresholds_f64(self, G: int) -> np.ndarray:
        t = np.zeros(G - 1)
        self.L.lmko_thresholds_f64(G, _p(t))
        return t

    def thresholds_f32(self, G: int) -> np.ndarray:
        t = np.zeros(G - 1, np.float32)
        self.L.lmko_thresholds_f32(G, _p(t))
        return t

    def verify_thresholds_f32(self, G: int, t32: np.ndarray, lo: int, hi: int, threads: int = 8) -> int:
        t = np.ascontiguousarray(t32, np.float32)
        return int(self.L.lmko_verify_thresholds_f32(G, _p(t), lo, hi, threads))


class Ref:
    """The reference's own code (oracle/_ref). Raises if the .so is absent."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        L.lmkref_last_error.restype = C.c_char_p
        L.lmkref_sigma.restype = C.c_double
        L.lmkref_sigma.argtypes = [C.c_double]
        L.lmkref_build_grid.argtypes = [C.c_int, _P, _P]
        L.lmkref_interval_index.argtypes = [C.c_int, C.c_double]
        L.lmkref_interval_index_batch.argtypes = [C.c_int, _P, C.c_int64, _P]
        L.lmkref_locate.argtypes = [C.c_int, C.c_int, _P, C.c_int64, _P, _P, _P]
        L.lmkref_init_layer.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, _P]
        L.lmkref_layer_create.restype = _P
        L.lmkref_layer_create.argtypes = [C.c_int, C.c_int, C.c_int, _P, C.c_double]
        L.lmkref_layer_destroy.argtypes = [_P]
        L.lmkref_matrix_create.restype = _P
        L.lmkref_matrix_create.argtypes = [C.c_int64, C.c_int64, _P]
        L.lmkref_matrix_destroy.argtypes = [_P]
        L.lmkref_matrix_read.argtypes = [_P, _P]
        L.lmkref_forward.argtypes = [_P, _P, _P, C.c_uint64]
        L.lmkref_backward.argtypes = [_P, _P, _P, _P, _P, C.c_uint64]
        L.lmkref_worker_count.restype = C.c_uint64
        self.L = L

    def build_grid(self, G: int):
        pts = np.zeros(G + 1)
        inv = np.zeros(G * G)
        if self.L.lmkref_build_grid(G, _p(pts), _p(inv)) != 0:
            raise ValueError(self.L.lmkref_last_error().decode())
        return pts, inv

    def interval_index(self, G: int, x) -> np.ndarray:
        x = np.ascontiguousarray(np.atleast_1d(x), np.float64)
        out = np.zeros(x.size, np.int32)
        self.L.lmkref_interval_index_batch(G, _p(x), x.size, _p(out))
        return out

    def locate(self, G: int, X: np.ndarray):
        X = np.ascontiguousarray(X, np.float64)
        rows, n_in = X.shape
        i1 = np.zeros((rows, n_in // 2), np.int32)
        i2 = np.zeros_like(i1)
        w = np.zeros((rows, n_in // 2, 4))
        if self.L.lmkref_locate(n_in, G, _p(X), rows, _p(i1), _p(i2), _p(w)) != 0:
            raise ValueError(self.L.lmkref_last_error().decode())
        return i1, i2, w

    def init_table(self, n_in: int, n_out: int, G: int, seed: int, scale: float = -1.0) -> np.ndarray:
        P = np.zeros((G + 1, G + 1, n_in // 2, n_out))
        if self.L.lmkref_init_layer(n_in, n_out, G, seed, scale, _p(P)) != 0:
            raise ValueError(self.L.lmkref_last_error().decode())
        return P

    def forward(self, G: int, P: np.ndarray, X: np.ndarray, gamma: float = 1.0, workers: int = 0):
        X = np.ascontiguousarray(X, np.float64)
        P = np.ascontiguousarray(P, np.float64)
        rows, n_in = X.shape
        n_out = P.size // ((G + 1) ** 2 * (n_in // 2))
        lay = RefLayer(self, n_in, n_out, G, P, gamma)
        try:
            return lay.forward(X, workers)
        finally:
            lay.close()


def _ref_backward(self, G, P, X, dY, gamma=1.0, dP0=None, workers=1):
    """The reference's lmkan_backward (layer.hpp:141-202): (dP0 + dP, dX)."""
    X = np.ascontiguousarray(X, np.float64)
    dY = np.ascontiguousarray(dY, np.float64)
    P = np.ascontiguousarray(P, np.float64)
    rows, n_in = X.shape
    n_out = dY.shape[1]
    lay = RefLayer(self, n_in, n_out, G, P, gamma)
    dP = np.zeros(P.shape) if dP0 is None else np.array(dP0, np.float64, copy=True)
    xm = self.L.lmkref_matrix_create(rows, n_in, _p(X))
    gm = self.L.lmkref_matrix_create(rows, n_out, _p(dY))
    dxm = self.L.lmkref_matrix_create(rows, n_in, None)
    try:
        if self.L.lmkref_backward(lay.h, xm, gm, _p(dP), dxm, workers) != 0:
            raise ValueError(self.L.lmkref_last_error().decode())
        dX = np.zeros((rows, n_in))
        self.L.lmkref_matrix_read(dxm, _p(dX))
        return dP, dX
    finally:
        for m in (xm, gm, dxm):
            self.L.lmkref_matrix_destroy(m)
        lay.close()


Ref.backward = _ref_backward


class RefLayer:
    """Persistent reference LmKanLayer + Matrix handles (for timing lmkan_forward alone)."""

    def __init__(self, ref: Ref, n_in: int, n_out: int, G: int, P: np.ndarray, gamma: float):
        self.ref, self.n_in, self.n_out = ref, n_in, n_out
        P = np.ascontiguousarray(P, np.float64)
        self.h = ref.L.lmkref_layer_create(n_in, n_out, G, _p(P), float(gamma))
        if not self.h:
            raise ValueError(ref.L.lmkref_last_error().decode())

    def make_io(self, X: np.ndarray):
        X = np.ascontiguousarray(X, np.float64)
        xm = self.ref.L.lmkref_matrix_create(X.shape[0], X.shape[1], _p(X))
        ym = self.ref.L.lmkref_matrix_create(X.shape[0], self.n_out, None)
        return xm, ym

    def run(self, xm, ym, workers: int = 0) -> None:
        if self.ref.L.lmkref_forward(self.h, xm, ym, workers) != 0:
            raise ValueError(self.ref.L.lmkref_last_error().decode())

    def read(self, ym, rows: int) -> np.ndarray:
        Y = np.zeros((rows, self.n_out))
        self.ref.L.lmkref_matrix_read(ym, _p(Y))
        return Y

    def free_io(self, *ms) -> None:
        for m in ms:
            self.ref.L.lmkref_matrix_destroy(m)

    def forward(self, X: np.ndarray, workers: int = 0) -> np.ndarray:
        xm, ym = self.make_io(X)
        try:
            self.run(xm, ym, workers)
            return self.read(ym, X.shape[0])
        finally:
            self.free_io(xm, ym)

    def close(self) -> None:
        if self.h:
            self.ref.L.lmkref_layer_destroy(self.h)
            self.h = None


def ref_or_port():
    """The reference build when present, else the C restatement."""
    try:
        return Ref()
    except (FileNotFoundError, OSError):
        return Port()


def mixed_err(y, ref) -> np.ndarray:
    """|y - ref| / max(1, |ref|): the reference's own tolerance normalization
    (test_layer.cpp:96-97, test_func2d.cpp:25-27)."""
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    return np.abs(y - ref) / np.maximum(1.0, np.abs(ref))
