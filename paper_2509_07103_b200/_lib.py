"""ctypes binding of the C-ABI in include/lmkan_b200.h.

Loads the in-tree ``paper_2509_07103_b200/lib/liblmkan_b200.so`` (built by
``__graft_entry__.build()``). There is no fallback: if the library is missing
or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# LMKAN_B200_LIB points at another build of the same library (A/B experiments)
LIB_PATH = os.environ.get("LMKAN_B200_LIB") or os.path.join(_HERE, "lib", "liblmkan_b200.so")

OK, EINVAL, ECUDA, ENOMEM, ENOSYS, EFORMAT, EUNSUPPORTED = 0, 1, 2, 3, 4, 5, 6

# (name, restype, argtypes) — must match include/lmkan_b200.h exactly;
# tests/test_capi.py checks every declared symbol is exported.
_P = C.c_void_p
_SIGS = [
    ("lmkan_b200_last_error", C.c_char_p, []),
    ("lmkan_b200_version", C.c_char_p, []),
    ("lmkan_b200_build_grid", C.c_int, [C.c_int, _P, _P]),
    ("lmkan_b200_thresholds", C.c_int, [C.c_int, _P, _P]),
    ("lmkan_b200_init_table", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, _P]),
    ("lmkan_b200_layer_create", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, _P, C.c_int, C.POINTER(_P)]),
    ("lmkan_b200_layer_create_exact", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, _P, C.c_int, C.POINTER(_P)]),
    ("lmkan_b200_layer_create_device_f32", C.c_int,
     [C.c_int, C.c_int, C.c_int, C.c_double, _P, C.c_int, C.POINTER(_P)]),
    ("lmkan_b200_layer_create_device_f32_slice", C.c_int,
     [C.c_int, C.c_int, C.c_int, C.c_double, _P, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    ("lmkan_b200_layer_create_random", C.c_int,
     [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_double, C.c_int, C.c_int, C.c_int,
      C.POINTER(_P)]),
    ("lmkan_b200_layer_read_table", C.c_int, [_P, C.c_int, C.c_int, _P]),
    ("lmkan_b200_layer_set_gamma", C.c_int, [_P, C.c_double]),
    ("lmkan_b200_layer_info", C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    ("lmkan_b200_layer_destroy", C.c_int, [_P]),
    ("lmkan_b200_forward_f32", C.c_int, [_P, _P, _P, C.c_int64, _P]),
    ("lmkan_b200_forward_f32_timed", C.c_int, [_P, _P, _P, C.c_int64, _P, _P, _P]),
    ("lmkan_b200_forward_f64", C.c_int, [_P, _P, _P, C.c_int64, _P]),
    ("lmkan_b200_forward_f32_dests", C.c_int, [_P, _P, C.POINTER(_P), C.c_int, C.c_int64, C.c_int, C.c_int64, _P]),
    ("lmkan_b200_ipc_get_handle", C.c_int, [_P, _P, C.POINTER(C.c_uint64)]),
    ("lmkan_b200_ipc_open_handle", C.c_int, [_P, C.c_uint64, C.c_int, C.POINTER(_P)]),
    ("lmkan_b200_ipc_close", C.c_int, [_P]),
    ("lmkan_b200_peer_barrier", C.c_int, [C.POINTER(_P), C.c_int, C.c_int, C.c_int, C.c_int, _P, _P]),
    ("lmkan_b200_conv_forward_f32", C.c_int,
     [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P]),
    ("lmkan_b200_conv_forward_host_f32", C.c_int,
     [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, C.c_size_t]),
    ("lmkan_b200_device_pci_bus_id", C.c_int, [C.c_int, C.c_char_p, C.c_int]),
    ("lmkan_b200_peer_access", C.c_int, [C.c_int, C.c_char_p]),
    ("lmkan_b200_forward_host_f64", C.c_int, [_P, _P, _P, C.c_int64, C.c_size_t]),
    ("lmkan_b200_forward_host_f32", C.c_int, [_P, _P, _P, C.c_int64, C.c_size_t]),
    ("lmkan_b200_locate_f32", C.c_int, [_P, _P, _P, _P, _P, C.c_int64, _P]),
    ("lmkan_b200_locate_f64", C.c_int, [_P, _P, _P, _P, _P, C.c_int64, _P]),
    ("lmkan_b200_records_f32", C.c_int, [_P, _P, _P, _P, _P, C.c_int64, C.c_int, _P]),
    ("lmkan_b200_records_f64", C.c_int, [_P, _P, _P, _P, _P, C.c_int64, C.c_int, _P]),
    ("lmkan_b200_plan", C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("lmkan_b200_lane_vectors", C.c_int, [C.c_int]),
    ("lmkan_b200_layer_lane_vectors", C.c_int, [_P]),
    ("lmkan_b200_plan_cta_group", C.c_int, [_P, C.c_int64]),
    ("lmkan_b200_conv_plan", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P]),
    ("lmkan_b200_backward_f64", C.c_int, [_P, _P, _P, _P, _P, _P, C.c_int64, C.c_uint64, _P]),
    ("lmkan_b200_backward_workers", C.c_int64, [_P, C.c_int64]),
    ("lmkan_b200_backward_host_f64", C.c_int, [_P, _P, _P, _P, _P, _P, C.c_int64, C.c_size_t]),
    ("lmkan_b200_lmk1_inspect", C.c_int, [C.c_char_p, _P, _P, _P]),
    ("lmkan_b200_lmk1_block", C.c_int, [C.c_char_p, C.c_int, _P, _P, _P, _P, _P, _P, _P, _P]),
    ("lmkan_b200_layer_load_lmk1", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    ("lmkan_b200_model_load", C.c_int, [C.c_char_p, C.c_int, C.POINTER(_P)]),
    ("lmkan_b200_model_create", C.c_int, [C.POINTER(_P), C.c_int, C.POINTER(_P)]),
    ("lmkan_b200_model_info", C.c_int, [_P, _P, _P, _P, _P]),
    ("lmkan_b200_model_layer", C.c_int, [_P, C.c_int, C.POINTER(_P)]),
    ("lmkan_b200_model_infer_f32", C.c_int, [_P, _P, _P, C.c_int64, _P]),
    ("lmkan_b200_model_infer_f64", C.c_int, [_P, _P, _P, C.c_int64, _P]),
    ("lmkan_b200_model_infer_host_f64", C.c_int, [_P, _P, _P, C.c_int64, C.c_size_t]),
    ("lmkan_b200_model_infer_host_f32", C.c_int, [_P, _P, _P, C.c_int64, C.c_size_t]),
    ("lmkan_b200_model_destroy", C.c_int, [_P]),
]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in _SIGS:
        if os.environ.get("LMKAN_B200_LIB") and not hasattr(lib, name):
            continue  # an older build under test: bind what it has
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class LmkanError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class FormatError(LmkanError):
    """lmkan::FormatError (errors.hpp:23-26): malformed or truncated LMK1 file."""


class UnsupportedModelError(LmkanError):
    """A valid LMK1 model with blocks outside the B200 path (mlp / bn / preconditioned)."""


def check(rc: int) -> None:
    if rc != OK:
        msg = (lib.lmkan_b200_last_error() or b"").decode()
        if rc == EINVAL:
            # the reference raises std::invalid_argument for the same conditions
            raise ValueError(msg)
        if rc == EFORMAT:
            raise FormatError(rc, msg)
        if rc == EUNSUPPORTED:
            raise UnsupportedModelError(rc, msg)
        raise LmkanError(rc, msg)
