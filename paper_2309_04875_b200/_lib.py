"""ctypes binding of libhbrelu.so (the C ABI in include/hb_relu.h).

The library is built in-tree (``make -j8`` or ``__graft_entry__.build()``) and
loaded from ``paper_2309_04875_b200/lib``.  There is no fallback: if the
library or a CUDA device is missing, the first call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    ConfigError,
    DataFormatError,
    RingMpcError,
    TransportError,
    TripleExhaustedError,
)

LIB_PATH = os.environ.get("HB_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libhbrelu.so")

HB_OK, HB_ERR_CUDA, HB_ERR_CONFIG, HB_ERR_TRANSPORT, HB_ERR_DATA, HB_ERR_TRIPLES = range(6)
TAG_BY_CODE = {0: "Circuit", 1: "Mult", 2: "B2A", 3: "Other"}

EW = dict(SLICE=0, MSB=1, XOR=2, KS_RHS=3, KS_UPDATE=4, KS_FINISH=5, B2A_LIFT=6, DRELU_OUT=7, OWNER=8,
          STACK2=9, MASKW=10, DRELU_SHARES=11)

u64p = ctypes.c_void_p
i64 = ctypes.c_int64


class Triples(ctypes.Structure):
    """hb_triples_t: one party's (kind, width) stream with its cursor."""

    _fields_ = [
        ("a", ctypes.c_void_p),
        ("b", ctypes.c_void_p),
        ("c", ctypes.c_void_p),
        ("cursor", ctypes.c_int64),
        ("capacity", ctypes.c_int64),
        ("width", ctypes.c_int32),
    ]


EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_int64, ctypes.c_void_p)

_SIGS = {
    "hb_last_error": (ctypes.c_char_p, []),
    "hb_version": (ctypes.c_int, []),
    "hb_prefix_levels": (ctypes.c_int, [ctypes.c_int]),
    "hb_payload_bytes": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int]),
    "hb_relu_rounds": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "hb_relu_round_bytes": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int]),
    "hb_relu_round_tag": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "hb_relu_pair": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p, u64p, u64p, u64p,
                                    Triples, Triples, Triples, Triples, ctypes.c_int, ctypes.c_void_p]),
    "hb_relu_pair_range": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, u64p, u64p, u64p, u64p, Triples, Triples, Triples, Triples,
                                          ctypes.c_int, ctypes.c_void_p]),
    "hb_relu_pair_host": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p, u64p, u64p,
                                         u64p, Triples, Triples, Triples, Triples, ctypes.c_int, ctypes.c_int64, u64p,
                                         ctypes.c_void_p]),
    "hb_set_device": (ctypes.c_int, [ctypes.c_int]),
    "hb_relu_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int, ctypes.c_int64]),
    "hb_relu_p2p_bytes": (ctypes.c_uint64, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_int64)]),
    "hb_relu_p2p_wire_bytes": (ctypes.c_uint64, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int]),
    "hb_relu_p2p": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p, u64p,
                                   Triples, Triples, ctypes.c_void_p, u64p, ctypes.c_void_p, u64p, ctypes.c_uint64,
                                   ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_int, u64p,
                                   ctypes.c_void_p]),
    "hb_relu_p2p_pair": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p, u64p, u64p,
                                        u64p, Triples, Triples, Triples, Triples, ctypes.c_void_p, ctypes.c_void_p,
                                        u64p, u64p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_void_p, ctypes.c_int, u64p, ctypes.c_void_p]),
    "hb_relu_p2p_dev": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p,
                                       u64p, Triples, Triples, ctypes.c_void_p, u64p, ctypes.c_void_p, u64p, u64p,
                                       ctypes.c_uint64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_int,
                                       u64p, ctypes.c_void_p]),
    "hb_relu_p2p_pair_dev": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p, u64p,
                                            u64p, u64p, Triples, Triples, Triples, Triples, ctypes.c_void_p,
                                            ctypes.c_void_p, u64p, u64p, u64p, u64p, ctypes.c_uint64, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_int,
                                            u64p, ctypes.c_void_p]),
    "hb_dev_alloc": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    "hb_dev_free": (ctypes.c_int, [ctypes.c_void_p]),
    "hb_ipc_export": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p]),
    "hb_ipc_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "hb_ipc_close": (ctypes.c_int, [ctypes.c_void_p]),
    "hb_relu_round": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                     ctypes.c_int, u64p, u64p, Triples, Triples, ctypes.c_void_p, u64p, u64p,
                                     ctypes.c_int, ctypes.c_void_p]),
    "hb_relu_callback_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64]),
    "hb_relu": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p, u64p,
                               Triples, Triples, ctypes.c_void_p, ctypes.c_int, EXCHANGE_FN, ctypes.c_void_p,
                               ctypes.c_void_p]),
    "hb_pack": (ctypes.c_int, [u64p, ctypes.c_int64, ctypes.c_int, u64p, ctypes.c_void_p]),
    "hb_unpack": (ctypes.c_int, [u64p, ctypes.c_int64, ctypes.c_int, u64p, ctypes.c_void_p]),
    "hb_beaver_open": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p, u64p, Triples, u64p, u64p,
                                      ctypes.c_void_p]),
    "hb_beaver_close": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p, u64p, Triples,
                                       u64p, u64p, ctypes.c_void_p]),
    "hb_ewise": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int, u64p, u64p,
                                u64p, u64p, ctypes.c_void_p]),
    "hb_any_above_one": (ctypes.c_int, [u64p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int), ctypes.c_void_p]),
    "hb_im2col_limbs": (ctypes.c_int, [u64p] + [ctypes.c_int] * 8 + [ctypes.c_int64, u64p, ctypes.c_void_p]),
    "hb_limb_combine": (ctypes.c_int, [u64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, u64p,
                                       ctypes.c_int,
                                       ctypes.c_int, u64p, ctypes.c_int, ctypes.c_int64, u64p, ctypes.c_void_p]),
    "hb_avgpool": (ctypes.c_int, [u64p, ctypes.c_int64] + [ctypes.c_int] * 5 + [ctypes.c_uint64, ctypes.c_int,
                                                                                  ctypes.c_int, u64p, ctypes.c_void_p]),
    "hb_add_shares": (ctypes.c_int, [u64p, u64p, ctypes.c_int64, u64p, ctypes.c_void_p]),
    "hb_avgpool_nhwc": (ctypes.c_int, [u64p, ctypes.c_int64] + [ctypes.c_int] * 6 + [ctypes.c_uint64, ctypes.c_int,
                                                                                      ctypes.c_int, u64p,
                                                                                      ctypes.c_void_p]),
    "hb_deal_triples": (ctypes.c_int, [ctypes.c_uint64] * 4 + [ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                                                ctypes.c_int64, ctypes.c_int64] + [u64p] * 6
                        + [ctypes.c_void_p]),
    "hb_conv_limbs_tc": (ctypes.c_int, [u64p] + [ctypes.c_int] * 8 + [u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                                                        ctypes.c_int, ctypes.c_int, ctypes.c_int, u64p,
                                                                        u64p, ctypes.c_void_p]),
    "hb_sim_relu": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "hb_im2col_planes": (ctypes.c_int, [u64p] + [ctypes.c_int] * 8 + [u64p, ctypes.c_void_p]),
    "hb_limbs_nhwc": (ctypes.c_int, [u64p] + [ctypes.c_int] * 4 + [u64p, ctypes.c_void_p]),
    "hb_conv_limbs_tma": (ctypes.c_int, [u64p] + [ctypes.c_int] * 8 + [u64p] + [ctypes.c_int] * 5 + [u64p, u64p, u64p,
                                                                                                 ctypes.c_void_p]),
    "hb_conv_limbs_tma_pair": (ctypes.c_int, [u64p, u64p] + [ctypes.c_int] * 8 + [u64p] + [ctypes.c_int] * 4
                               + [u64p] * 5 + [ctypes.c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the library; raises RingMpcError if it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RingMpcError(f"CUDA library not built: {path} (run `make -j8` or __graft_entry__.build())")
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
            if hasattr(lib, "hb_debug_conv_stamps"):
                lib.hb_debug_conv_stamps.restype = ctypes.c_int
    return _lib


_ERRORS = {
    HB_ERR_CONFIG: ConfigError,
    HB_ERR_TRANSPORT: TransportError,
    HB_ERR_DATA: DataFormatError,
    HB_ERR_TRIPLES: TripleExhaustedError,
}


def check(rc: int) -> None:
    """Map a status code to the reference's exception classes (errors.py:8-47)."""
    if rc == HB_OK:
        return
    msg = load().hb_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, RingMpcError)(msg or f"libhbrelu status {rc}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
