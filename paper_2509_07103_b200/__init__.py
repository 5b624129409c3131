"""B200-native (sm_100a) lmKAN layer forward — Python view of the C-ABI.

The product is the CUDA library ``lib/liblmkan_b200.so`` (sources in
``csrc/``) behind the C-ABI ``include/lmkan_b200.h`` and the C++ host API
``include/lmkan_b200/lmkan.hpp``. This module is the thin ctypes view used by
the tests and ``bench.py``; it mirrors the reference's C++ interface names
(paths relative to /root/reference/proj/include/lmkan/):

  build_grid(G)                       grid.hpp:44-68
  init_layer(n_in, n_out, G, seed)    layer.hpp:69-86   (bit-identical table)
  LmKanLayer                          layer.hpp:24-61
  lmkan_forward(layer, X, Y, workers) layer.hpp:108-134 (ValueError where the
                                       reference throws std::invalid_argument)

plus ``Layer``, the prepared device handle that the fast paths use. Device
tensors are torch CUDA tensors (torch is used for device memory and streams
only). Nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

from ._lib import LIB_PATH, FormatError, LmkanError, UnsupportedModelError, check, lib  # noqa: F401  (fails loudly if the .so is missing)

__all__ = ["SigmaGrid", "build_grid", "thresholds", "init_table", "Layer", "LmKanLayer", "init_layer",
           "Model", "load_model", "model_infer", "lmk1_inspect", "lmk1_block", "FormatError",
           "UnsupportedModelError",
           "lmkan_forward", "LmkanError", "LIB_PATH", "version"]


def _ptr(a) -> C.c_void_p:
    if a is None:
        return C.c_void_p(0)
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())  # torch tensor


def version() -> str:
    return lib.lmkan_b200_version().decode()


@dataclass
class SigmaGrid:
    """grid.hpp:33-39: G intervals, points[G+1] (ghost ends), inv_areas[G*G]."""
    G: int
    points: np.ndarray
    inv_areas: np.ndarray

    def inv_area(self, i1: int, i2: int) -> float:
        return float(self.inv_areas[i1 * self.G + i2])


def build_grid(G: int) -> SigmaGrid:
    pts = np.zeros(max(G, 0) + 1, np.float64)
    inv = np.zeros(max(G, 0) ** 2, np.float64)
    check(lib.lmkan_b200_build_grid(int(G), _ptr(pts), _ptr(inv)))
    return SigmaGrid(int(G), pts, inv)


def thresholds(G: int) -> Tuple[np.ndarray, np.ndarray]:
    """(t64, t32): interval_index(x) == #{k : x >= t[k]} (see include/lmkan_b200.h)."""
    t64 = np.zeros(max(G - 1, 0), np.float64)
    t32 = np.zeros(max(G - 1, 0), np.float32)
    check(lib.lmkan_b200_thresholds(int(G), _ptr(t64), _ptr(t32)))
    return t64, t32


def init_table(n_in: int, n_out: int, G: int, seed: int, init_scale: float = -1.0) -> np.ndarray:
    """init_layer's table (layer.hpp:69-86), reference layout [G+1][G+1][n_in/2][n_out]."""
    if n_in <= 0 or n_in % 2 or n_out <= 0 or G < 3:
        check(lib.lmkan_b200_init_table(int(n_in), int(n_out), int(G), int(seed), float(init_scale), None))
    P = np.empty((G + 1, G + 1, n_in // 2, n_out), np.float64)
    check(lib.lmkan_b200_init_table(int(n_in), int(n_out), int(G), int(seed) & (2**64 - 1), float(init_scale),
                                    _ptr(P)))
    return P


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class Layer:
    """Prepared device layer (opaque ``lmkan_b200_layer*``): fp32 table in the
    [out_tile][pair][node][OT] layout, grid constants and locate thresholds."""

    def __init__(self, handle: C.c_void_p, owned: bool = True):
        self._h = handle
        self._owned = owned  # False for layers borrowed from a Model
        n_in, n_out, G, dev, ot = (C.c_int() for _ in range(5))
        tb = C.c_size_t()
        check(lib.lmkan_b200_layer_info(self._h, C.byref(n_in), C.byref(n_out), C.byref(G), C.byref(dev),
                                        C.byref(tb), C.byref(ot)))
        self.n_in, self.n_out, self.G, self.device = n_in.value, n_out.value, G.value, dev.value
        self.table_bytes, self.out_tile = tb.value, ot.value
        self.pairs = self.n_in // 2

    # -- construction -------------------------------------------------------
    @classmethod
    def from_host(cls, n_in: int, n_out: int, G: int, P: np.ndarray, gamma: float = 1.0,
                  device: int = 0, precision: int = 32) -> "Layer":
        """precision 32: the fp32 gather (1e-5 contract); 64: the
        reference-precision kernel, bit-identical to the reference forward."""
        P = np.ascontiguousarray(P, dtype=np.float64)
        if P.size != (G + 1) ** 2 * (n_in // 2) * n_out:
            raise ValueError("layer_create: P has the wrong number of coefficients")
        if precision not in (32, 64):
            raise ValueError("layer_create: precision must be 32 or 64")
        h = C.c_void_p()
        fn = lib.lmkan_b200_layer_create_exact if precision == 64 else lib.lmkan_b200_layer_create
        check(fn(int(n_in), int(n_out), int(G), float(gamma), _ptr(P), int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, n_in: int, n_out: int, G: int, P_dev, gamma: float = 1.0, device: int = 0,
                    out_range: Optional[Tuple[int, int]] = None) -> "Layer":
        """P_dev: contiguous float32 CUDA tensor in reference layout."""
        import torch
        assert P_dev.dtype == torch.float32 and P_dev.is_cuda and P_dev.is_contiguous()
        ob, oe = out_range if out_range else (0, n_out)
        h = C.c_void_p()
        check(lib.lmkan_b200_layer_create_device_f32_slice(int(n_in), int(n_out), int(G), float(gamma),
                                                           _ptr(P_dev), int(ob), int(oe), int(device),
                                                           C.byref(h)))
        return cls(h)

    @classmethod
    def random(cls, n_in: int, n_out: int, G: int, seed: int = 1234, scale: float = -1.0,
               gamma: float = 1.0, device: int = 0, out_range: Optional[Tuple[int, int]] = None) -> "Layer":
        """Table generated on the device (counter-based RNG), N(0, scale^2);
        scale < 0 selects init_layer's (n_in/2)^-1/2 (layer.hpp:63-65)."""
        if scale < 0:
            scale = 1.0 / np.sqrt(max(n_in // 2, 1))
        ob, oe = out_range if out_range else (0, n_out)
        h = C.c_void_p()
        check(lib.lmkan_b200_layer_create_random(int(n_in), int(n_out), int(G), float(gamma), int(seed),
                                                 float(scale), int(ob), int(oe), int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def load_lmk1(cls, path: str, block: int = 0, out_range: Optional[Tuple[int, int]] = None,
                  device: int = 0) -> "Layer":
        """One lmkan block of an LMK1 file straight to the device (optionally an
        output slice [ob, oe)): the table is streamed from disk in chunks."""
        ob, oe = out_range if out_range else (0, -1)
        h = C.c_void_p()
        check(lib.lmkan_b200_layer_load_lmk1(str(path).encode(), int(block), int(ob), int(oe), int(device),
                                             C.byref(h)))
        return cls(h)

    # -- forward ------------------------------------------------------------
    def _check_x(self, X, dtypes=("float32", "float64")) -> None:
        """Shared checks of the device entry points: a 2-D contiguous CUDA tensor
        of the layer's width and an accepted dtype."""
        import torch
        if X.dim() != 2 or X.shape[1] != self.n_in:
            raise ValueError(f"lmkan_forward: expected width {self.n_in}, got {X.shape[-1]}")
        if not (X.is_cuda and X.is_contiguous()):
            raise ValueError("lmkan_forward: X must be a contiguous CUDA tensor")
        if X.dtype not in tuple(getattr(torch, d) for d in dtypes):
            raise ValueError(f"lmkan_forward: X dtype {X.dtype} not in {dtypes}")

    def forward_into(self, X, Y, stream=None) -> None:
        """Device path: X [rows, n_in], Y [rows, n_out] contiguous CUDA tensors
        (float32 or float64, same dtype); asynchronous on `stream`."""
        import torch
        self._check_x(X)
        if not (Y.is_cuda and Y.is_contiguous() and Y.shape == (X.shape[0], self.n_out) and Y.dtype == X.dtype):
            raise ValueError(f"lmkan_forward: Y must be a contiguous CUDA tensor [{X.shape[0]}, {self.n_out}] of X's dtype")
        fn = lib.lmkan_b200_forward_f32 if X.dtype == torch.float32 else lib.lmkan_b200_forward_f64
        check(fn(self._h, _ptr(X), _ptr(Y), int(X.shape[0]), _stream_ptr(stream)))

    def forward_dests(self, X, dest_ptrs, ld: int, col0: int, stream=None) -> None:
        """Forward (float32) storing this layer's output columns into every
        destination buffer: dest[r * ld + col0 + q] (device pointers, e.g. the
        full-width Y of every GPU of an output-sharded layer; this GPU's own
        buffer first: pair-block running sums live in dests[0])."""
        self._check_x(X, ("float32",))
        if col0 < 0 or ld < col0 + self.n_out:
            raise ValueError("forward_dests: ld must be >= col0 + n_out")
        arr = (C.c_void_p * len(dest_ptrs))(*[int(p) for p in dest_ptrs])
        check(lib.lmkan_b200_forward_f32_dests(self._h, _ptr(X), arr, len(dest_ptrs), int(ld), int(col0),
                                               int(X.shape[0]), _stream_ptr(stream)))

    def forward_into_timed(self, X, Y, ev_begin, ev_end, stream=None) -> None:
        """forward_into (float32) recording torch.cuda.Events around the gather kernel."""
        self._check_x(X, ("float32",))
        if not (Y.is_cuda and Y.is_contiguous() and Y.shape == (X.shape[0], self.n_out) and Y.dtype == X.dtype):
            raise ValueError(f"lmkan_forward: Y must be a contiguous CUDA tensor [{X.shape[0]}, {self.n_out}] of X's dtype")
        check(lib.lmkan_b200_forward_f32_timed(self._h, _ptr(X), _ptr(Y), int(X.shape[0]), _stream_ptr(stream),
                                               C.c_void_p(ev_begin.cuda_event), C.c_void_p(ev_end.cuda_event)))

    def conv_forward(self, img, k: int, s: int = 1, Y=None, stream=None):
        """Implicit-im2col conv: img [N, H, W, C] float32 CUDA tensor (NHWC) ->
        Y [N, out_h, out_w, n_out] (unfold_conv -> lmkan_forward -> fold_output,
        conv.hpp:39-71, without materializing the patch matrix)."""
        import torch
        assert img.dtype == torch.float32 and img.is_cuda and img.is_contiguous() and img.dim() == 4
        N, H, W, Cc = img.shape
        oh, ow = (H - k) // s + 1, (W - k) // s + 1
        if Y is None:
            Y = torch.empty((N, max(oh, 0), max(ow, 0), self.n_out), dtype=torch.float32, device=img.device)
        check(lib.lmkan_b200_conv_forward_f32(self._h, _ptr(img), int(N), int(H), int(W), int(Cc), int(k), int(s),
                                              _ptr(Y), _stream_ptr(stream)))
        return Y

    def conv_forward_host(self, img: np.ndarray, k: int, s: int = 1, Y: Optional[np.ndarray] = None) -> np.ndarray:
        """Host conv (synchronous, copies overlapped with the kernels): img
        [N, H, W, C] float32 -> Y [N, out_h, out_w, n_out] float32."""
        img = np.ascontiguousarray(img, np.float32)
        N, H, W, Cc = img.shape
        oh, ow = (H - k) // s + 1, (W - k) // s + 1
        if Y is None:
            Y = np.empty((N, max(oh, 0), max(ow, 0), self.n_out), np.float32)
        check(lib.lmkan_b200_conv_forward_host_f32(self._h, _ptr(img), int(N), int(H), int(W), int(Cc), int(k), int(s),
                                                   _ptr(Y), 0))
        return Y

    def conv_forward_host_ptr(self, img_ptr: int, N: int, H: int, W: int, Cc: int, k: int, s: int, Y_ptr: int) -> None:
        check(lib.lmkan_b200_conv_forward_host_f32(self._h, C.c_void_p(img_ptr), int(N), int(H), int(W), int(Cc),
                                                   int(k), int(s), C.c_void_p(Y_ptr), 0))

    def forward(self, X, stream=None):
        """torch CUDA tensor in -> CUDA tensor out; numpy in -> numpy out (host path)."""
        if isinstance(X, np.ndarray):
            return self.forward_host(X)
        import torch
        Y = torch.empty((X.shape[0], self.n_out), dtype=X.dtype, device=X.device)
        self.forward_into(X, Y, stream)
        return Y

    def forward_host(self, X: np.ndarray, Y: Optional[np.ndarray] = None) -> np.ndarray:
        """Synchronous host path (copies pipelined with the kernel by row chunk)."""
        if X.ndim != 2 or X.shape[1] != self.n_in:
            raise ValueError(f"lmkan_forward: expected width {self.n_in}, got {X.shape[-1]}")
        if X.dtype not in (np.float32, np.float64):
            X = X.astype(np.float64)
        X = np.ascontiguousarray(X)
        if Y is None or Y.shape != (X.shape[0], self.n_out) or Y.dtype != X.dtype:
            Y = np.empty((X.shape[0], self.n_out), X.dtype)
        fn = lib.lmkan_b200_forward_host_f32 if X.dtype == np.float32 else lib.lmkan_b200_forward_host_f64
        check(fn(self._h, _ptr(X), _ptr(Y), int(X.shape[0]), 0))
        return Y

    def forward_host_ptr(self, X_ptr: int, Y_ptr: int, rows: int, dtype=np.float32) -> None:
        fn = lib.lmkan_b200_forward_host_f32 if dtype == np.float32 else lib.lmkan_b200_forward_host_f64
        check(fn(self._h, C.c_void_p(X_ptr), C.c_void_p(Y_ptr), int(rows), 0))

    def locate(self, X, stream=None):
        """Stage 1 only: (i1, i2, w) CUDA tensors, w[..., :] = {w00, w10, w01, w11}."""
        import torch
        rows = X.shape[0]
        i1 = torch.empty((rows, self.pairs), dtype=torch.int32, device=X.device)
        i2 = torch.empty_like(i1)
        w = torch.empty((rows, self.pairs, 4), dtype=torch.float32, device=X.device)
        fn = lib.lmkan_b200_locate_f32 if X.dtype == torch.float32 else lib.lmkan_b200_locate_f64
        check(fn(self._h, _ptr(X), _ptr(i1), _ptr(i2), _ptr(w), int(rows), _stream_ptr(stream)))
        return i1, i2, w

    RECORD_VARIANTS = {"k1": 0, "k1_smem": 1, "in_kernel": 2}

    def records(self, X, variant: str = "k1", stream=None):
        """The PRODUCTION cell records (what the gather kernels consume), decoded:
        (i1, i2, ag) CUDA tensors [rows, pairs] / [rows, pairs, 2] with
        ag = {alpha, gamma}. variant: "k1" (records4_kernel of the staged plan),
        "k1_smem" (records_kernel), "in_kernel" (fused / global / narrow locate)."""
        import torch
        assert X.is_cuda and X.is_contiguous() and X.dim() == 2 and X.shape[1] == self.n_in
        assert X.dtype in (torch.float32, torch.float64)
        rows = X.shape[0]
        i1 = torch.empty((rows, self.pairs), dtype=torch.int32, device=X.device)
        i2 = torch.empty_like(i1)
        ag = torch.empty((rows, self.pairs, 2), dtype=torch.float32, device=X.device)
        fn = lib.lmkan_b200_records_f32 if X.dtype == torch.float32 else lib.lmkan_b200_records_f64
        check(fn(self._h, _ptr(X), _ptr(i1), _ptr(i2), _ptr(ag), int(rows), self.RECORD_VARIANTS[variant],
                 _stream_ptr(stream)))
        return i1, i2, ag

    # -- training path ------------------------------------------------------
    def backward(self, P, X, dY, dP=None, want_dx: bool = True, workers: int = 0, stream=None):
        """lmkan_backward (layer.hpp:141-202) in fp64. CUDA tensors: P (the fp64
        master table, reference layout), X [rows, n_in], dY [rows, n_out];
        dP is added into (zeros when None). Returns (dP, dX or None); bitwise
        equal to the reference run with the same `workers` (0 = GPU-filling
        count, see backward_workers). numpy in -> synchronous host path."""
        n_par = (self.G + 1) ** 2 * self.pairs * self.n_out

        def check_io(Xs, dYs, Ps):
            if len(Xs.shape) != 2 or Xs.shape[1] != self.n_in:
                raise ValueError(f"lmkan_backward: expected width {self.n_in}, got {Xs.shape[-1]}")
            if len(dYs.shape) != 2 or dYs.shape[1] != self.n_out:
                raise ValueError(f"lmkan_backward: expected width {self.n_out}, got {dYs.shape[-1]}")
            if dYs.shape[0] != Xs.shape[0]:
                raise ValueError("lmkan_backward: X and dY row counts differ")
            if int(np.prod(Ps.shape)) != n_par:
                raise ValueError(f"lmkan_backward: P has {int(np.prod(Ps.shape))} coefficients, the layer {n_par}")

        if isinstance(X, np.ndarray):
            P = np.ascontiguousarray(P, np.float64)
            X = np.ascontiguousarray(X, np.float64)
            dY = np.ascontiguousarray(dY, np.float64)
            check_io(X, dY, P)
            dP = np.zeros(P.shape) if dP is None else np.ascontiguousarray(dP, np.float64)
            if dP.size != n_par:
                raise ValueError("lmkan_backward: dP size mismatch")
            dX = np.zeros(X.shape) if want_dx else None
            check(lib.lmkan_b200_backward_host_f64(self._h, _ptr(P), _ptr(X), _ptr(dY), _ptr(dP), _ptr(dX),
                                                   int(X.shape[0]), int(workers)))
            return dP, dX
        import torch
        for name, t in (("P", P), ("X", X), ("dY", dY)):
            if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
                raise ValueError(f"lmkan_backward: {name} must be a contiguous float64 CUDA tensor")
        check_io(X, dY, P)
        if dP is None:
            dP = torch.zeros_like(P)
        elif not (dP.is_cuda and dP.dtype == torch.float64 and dP.is_contiguous() and dP.device == P.device):
            raise ValueError("lmkan_backward: dP must be a contiguous float64 tensor on P's device")
        elif dP.numel() != n_par:
            raise ValueError("lmkan_backward: dP size mismatch")
        if X.device != P.device or dY.device != P.device:
            raise ValueError("lmkan_backward: P, X and dY must be on the same device")
        dX = torch.empty_like(X) if want_dx else None
        check(lib.lmkan_b200_backward_f64(self._h, _ptr(P), _ptr(X), _ptr(dY), _ptr(dP), _ptr(dX), int(X.shape[0]),
                                          int(workers), _stream_ptr(stream)))
        return dP, dX

    def backward_workers(self, rows: int) -> int:
        """Worker count (row chunks) the backward uses for workers = 0."""
        return int(lib.lmkan_b200_backward_workers(self._h, int(rows)))

    # -- introspection ------------------------------------------------------
    def set_gamma(self, gamma: float) -> None:
        check(lib.lmkan_b200_layer_set_gamma(self._h, float(gamma)))

    def read_table(self, pair_begin: int = 0, pair_end: Optional[int] = None) -> np.ndarray:
        """Device table back in reference layout: [G+1, G+1, pairs, n_out] doubles."""
        pe = self.pairs if pair_end is None else pair_end
        out = np.empty((self.G + 1, self.G + 1, pe - pair_begin, self.n_out), np.float64)
        check(lib.lmkan_b200_layer_read_table(self._h, int(pair_begin), int(pe), _ptr(out)))
        return out

    def plan(self, rows: int) -> dict:
        v = [C.c_int() for _ in range(8)]
        check(lib.lmkan_b200_plan(self._h, int(rows), *[C.byref(x) for x in v]))
        d = dict(zip(["out_tile", "rows_per_thread", "nbuf", "rows_per_cta", "launches", "mode", "slabs",
                      "warps_per_cta"],
                     [x.value for x in v]))
        d["mode"] = {0: "fused", 1: "staged", 2: "global", 3: "narrow", 4: "exact"}[d["mode"]]
        if hasattr(lib, "lmkan_b200_layer_lane_vectors"):
            d["lane_vectors"] = int(lib.lmkan_b200_layer_lane_vectors(self._h))
        else:  # an older build under A/B (LMKAN_B200_LIB)
            d["lane_vectors"] = int(lib.lmkan_b200_lane_vectors(d["out_tile"]))
        if hasattr(lib, "lmkan_b200_plan_cta_group"):
            d["cta_group"] = int(lib.lmkan_b200_plan_cta_group(self._h, int(rows)))
        return d

    def conv_plan(self, N: int, H: int, W: int, Cc: int, k: int, s: int) -> dict:
        """Ring depth, rows per CTA and pixel-record use of a conv_forward call."""
        v = [C.c_int() for _ in range(3)]
        check(lib.lmkan_b200_conv_plan(self._h, int(N), int(H), int(W), int(Cc), int(k), int(s),
                                       *[C.byref(x) for x in v]))
        return {"nbuf": v[0].value, "rows_per_cta": v[1].value, "pixel_records": bool(v[2].value)}

    def close(self) -> None:
        if getattr(self, "_h", None):
            if getattr(self, "_owned", True):
                lib.lmkan_b200_layer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Peer memory for the fused output all-gather (sharding.PeerGather uses these).

def ipc_handle(t) -> Tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding CUDA tensor `t`,
    offset of t's data inside that allocation)."""
    buf = C.create_string_buffer(64)
    off = C.c_uint64()
    check(lib.lmkan_b200_ipc_get_handle(C.c_void_p(t.data_ptr()), buf, C.byref(off)))
    return buf.raw, off.value


def ipc_open(handle: bytes, offset: int, device: int) -> int:
    """Map a peer's allocation (from ipc_handle in another process); returns
    the device pointer of the peer tensor's data."""
    p = C.c_void_p()
    check(lib.lmkan_b200_ipc_open_handle(C.create_string_buffer(bytes(handle), 64), int(offset), int(device),
                                         C.byref(p)))
    return int(p.value)


def ipc_close(ptr: int) -> None:
    check(lib.lmkan_b200_ipc_close(C.c_void_p(ptr)))


def peer_barrier(flag_ptrs, rank: int, epoch: int, status, timeout_ms: int = 10000, stream=None) -> None:
    """Enqueue the device-side barrier (see include/lmkan_b200.h); `status` is
    an int32 tensor on the device or in pinned host memory."""
    arr = (C.c_void_p * len(flag_ptrs))(*[int(p) for p in flag_ptrs])
    check(lib.lmkan_b200_peer_barrier(arr, len(flag_ptrs), int(rank), int(epoch), int(timeout_ms),
                                      C.c_void_p(status.data_ptr()), _stream_ptr(stream)))


def device_pci_bus_id(device: int) -> str:
    buf = C.create_string_buffer(32)
    check(lib.lmkan_b200_device_pci_bus_id(int(device), buf, 32))
    return buf.value.decode()


def peer_access(device: int, peer_pci_bus_id: str) -> None:
    """Check and enable peer access from `device` to the GPU with that PCI bus
    id; RuntimeError naming both GPUs if the pair has no peer path."""
    rc = lib.lmkan_b200_peer_access(int(device), peer_pci_bus_id.encode())
    if rc != 0:
        raise RuntimeError((lib.lmkan_b200_last_error() or b"").decode())


# ---------------------------------------------------------------------------
# Models: the LMK1 container (serialize.hpp:185-301) and model_infer of a fused
# pure-lookup model (model.hpp:268-315, fuse.hpp:105-140) as one device chain.

_BLOCK_TYPES = {0: "lmkan", 1: "mlp", 2: "bn"}
_MODES = {0: "relu_first", 1: "relu_last", 2: "linear", 3: "none"}


def lmk1_inspect(path: str) -> dict:
    """load_model's validation only (host, no GPU); raises FormatError /
    ValueError exactly where load_model throws FormatError / invalid_argument."""
    nb, elem, pure = C.c_int(), C.c_int(), C.c_int()
    check(lib.lmkan_b200_lmk1_inspect(str(path).encode(), C.byref(nb), C.byref(elem), C.byref(pure)))
    return {"blocks": nb.value, "dtype": "f32" if elem.value == 4 else "f64", "pure_lookup": bool(pure.value)}


def lmk1_block(path: str, block: int) -> dict:
    t, n_in, n_out, G, mode, bn = (C.c_int() for _ in range(6))
    gamma, off = C.c_double(), C.c_uint64()
    check(lib.lmkan_b200_lmk1_block(str(path).encode(), int(block), C.byref(t), C.byref(n_in), C.byref(n_out),
                                    C.byref(G), C.byref(gamma), C.byref(mode), C.byref(bn), C.byref(off)))
    return {"type": _BLOCK_TYPES[t.value], "n_in": n_in.value, "n_out": n_out.value, "G": G.value,
            "gamma": gamma.value, "mode": _MODES[mode.value], "bn": bool(bn.value), "p_offset": off.value}


class Model:
    """Opaque ``lmkan_b200_model*``: a chain of device layers (a fused model)."""

    def __init__(self, handle: C.c_void_p, keep=None):
        self._h = handle
        self._keep = keep  # borrowed layers must outlive the model
        nb, di, do, dev = (C.c_int() for _ in range(4))
        check(lib.lmkan_b200_model_info(self._h, C.byref(nb), C.byref(di), C.byref(do), C.byref(dev)))
        self.n_blocks, self.in_dim, self.out_dim, self.device = nb.value, di.value, do.value, dev.value

    @classmethod
    def load(cls, path: str, device: int = 0) -> "Model":
        h = C.c_void_p()
        check(lib.lmkan_b200_model_load(str(path).encode(), int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def from_layers(cls, layers) -> "Model":
        arr = (C.c_void_p * len(layers))(*[lay._h for lay in layers])
        h = C.c_void_p()
        check(lib.lmkan_b200_model_create(arr, len(layers), C.byref(h)))
        return cls(h, keep=list(layers))

    def layer(self, block: int) -> Layer:
        h = C.c_void_p()
        check(lib.lmkan_b200_model_layer(self._h, int(block), C.byref(h)))
        lay = Layer(h, owned=False)
        lay._model = self  # keep the owner alive
        return lay

    def infer_into(self, X, Y, stream=None) -> None:
        """Device path (CUDA graph replay after the first call per shape/stream)."""
        import torch
        if X.dim() != 2 or X.shape[1] != self.in_dim:
            raise ValueError(f"precond_forward: expected width {self.in_dim}, got {X.shape[-1]}")
        assert X.is_cuda and Y.is_cuda and X.is_contiguous() and Y.is_contiguous() and X.dtype == Y.dtype
        assert Y.shape == (X.shape[0], self.out_dim)
        fn = lib.lmkan_b200_model_infer_f32 if X.dtype == torch.float32 else lib.lmkan_b200_model_infer_f64
        check(fn(self._h, _ptr(X), _ptr(Y), int(X.shape[0]), _stream_ptr(stream)))

    def infer(self, X, stream=None):
        if isinstance(X, np.ndarray):
            return self.infer_host(X)
        import torch
        Y = torch.empty((X.shape[0], self.out_dim), dtype=X.dtype, device=X.device)
        self.infer_into(X, Y, stream)
        return Y

    def infer_host(self, X: np.ndarray) -> np.ndarray:
        X = np.asarray(X)
        if X.ndim != 2 or X.shape[1] != self.in_dim:
            raise ValueError(f"precond_forward: expected width {self.in_dim}, got {X.shape[-1]}")
        if X.dtype not in (np.float32, np.float64):
            X = X.astype(np.float64)
        X = np.ascontiguousarray(X)
        Y = np.empty((X.shape[0], self.out_dim), X.dtype)
        fn = lib.lmkan_b200_model_infer_host_f32 if X.dtype == np.float32 else lib.lmkan_b200_model_infer_host_f64
        check(fn(self._h, _ptr(X), _ptr(Y), int(X.shape[0]), 0))
        return Y

    def infer_host_ptr(self, X_ptr: int, Y_ptr: int, rows: int, dtype=np.float32) -> None:
        fn = lib.lmkan_b200_model_infer_host_f32 if dtype == np.float32 else lib.lmkan_b200_model_infer_host_f64
        check(fn(self._h, C.c_void_p(X_ptr), C.c_void_p(Y_ptr), int(rows), 0))

    def conv_plan(self, N: int, H: int, W: int, Cc: int, k: int, s: int) -> dict:
        """Ring depth, rows per CTA and pixel-record use of a conv_forward call."""
        v = [C.c_int() for _ in range(3)]
        check(lib.lmkan_b200_conv_plan(self._h, int(N), int(H), int(W), int(Cc), int(k), int(s),
                                       *[C.byref(x) for x in v]))
        return {"nbuf": v[0].value, "rows_per_cta": v[1].value, "pixel_records": bool(v[2].value)}

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.lmkan_b200_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def load_model(path: str, device: int = 0) -> Model:
    """serialize.hpp:185-301 for fused pure-lookup models, onto `device`."""
    return Model.load(path, device)


def model_infer(model: Model, X: np.ndarray, workers: int = 0) -> np.ndarray:
    """model.hpp:313-316: host X [rows, in_dim] -> host Y; `workers` ignored."""
    return model.infer_host(np.ascontiguousarray(X, np.float64))


# ---------------------------------------------------------------------------
# Mirror of the reference host interface (layer.hpp:24-134) for Python callers.

@dataclass
class LmKanLayer:
    """layer.hpp:24-61. P is the reference table [G+1][G+1][n_in/2][n_out]."""
    n_in: int
    n_out: int
    grid: SigmaGrid
    P: np.ndarray
    gamma: float = 0.0
    device: int = 0
    _prepared: Optional[Layer] = field(default=None, repr=False, compare=False)
    _key: Optional[bytes] = field(default=None, repr=False, compare=False)

    def pairs(self) -> int:
        return self.n_in // 2

    def param_count(self) -> int:
        return int(self.P.size)

    def prepared(self) -> Layer:
        """Device handle, rebuilt when P changed since the last call (fingerprint
        of the full table, so in-place edits of P are never served stale)."""
        import hashlib
        P = np.ascontiguousarray(self.P, np.float64)
        key = hashlib.blake2b(P.view(np.uint8), digest_size=16).digest() + \
            np.array([self.n_in, self.n_out, self.grid.G], np.int64).tobytes()
        if self._prepared is None or key != self._key:
            if self._prepared is not None:
                self._prepared.close()
            self._prepared = Layer.from_host(self.n_in, self.n_out, self.grid.G, P, self.gamma, self.device)
            self._key = key
        self._prepared.set_gamma(self.gamma)
        return self._prepared


def init_layer(n_in: int, n_out: int, G: int, seed: int, init_scale: float = -1.0) -> LmKanLayer:
    """layer.hpp:69-86: same validation, same table, gamma = 0."""
    P = init_table(n_in, n_out, G, seed, init_scale)
    return LmKanLayer(n_in, n_out, build_grid(G), P, 0.0)


def lmkan_forward(layer: LmKanLayer, X: np.ndarray, Y: Optional[np.ndarray] = None,
                  workers: int = 0) -> np.ndarray:
    """layer.hpp:108-134 on the B200: X [rows, n_in] float64 host array; returns
    Y [rows, n_out] (reused when the shape matches, else reallocated, like
    layer.hpp:111-112). `workers` is accepted and ignored."""
    X = np.asarray(X)
    if X.ndim != 2 or X.shape[1] != layer.n_in:
        width = X.shape[1] if X.ndim == 2 else X.shape[-1]
        raise ValueError(f"lmkan_forward: expected width {layer.n_in}, got {width}")
    X = np.ascontiguousarray(X, np.float64)
    if Y is None or Y.shape != (X.shape[0], layer.n_out) or Y.dtype != np.float64 or not Y.flags.c_contiguous:
        Y = np.zeros((X.shape[0], layer.n_out), np.float64)
    if X.shape[0] == 0:
        return Y
    return layer.prepared().forward_host(X, Y)
