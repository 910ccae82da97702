"""ctypes binding of libmergecomp.so (the C ABI in include/mergecomp.h).

There is no fallback: if the shared library is missing or cannot be loaded,
every compute entry point raises.  The library is built in-tree by
``python -m paper_2103_15195_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
from functools import lru_cache
from pathlib import Path

from .spec import McSpec

LIB_PATH = Path(__file__).resolve().parent / "libmergecomp.so"

MC_OK = 0
MC_EPEER = -4
MC_ERR_NONFINITE = 0x1
MC_ERR_INDEX_RANGE = 0x2
MC_ERR_INDEX_ORDER = 0x4
MC_ERR_HEADER = 0x8
MC_ERR_PEER_TIMEOUT = 0x10
MC_PIPE_NO_WAIT = ctypes.c_void_p(-1 & 0xFFFFFFFFFFFFFFFF)  # include/mergecomp.h: (void*)(intptr_t)-1


class McLayout(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("cap", ctypes.c_int64),
        ("n_val", ctypes.c_int64),
        ("n_bits", ctypes.c_int64),
        ("n_codes", ctypes.c_int64),
        ("off_idx", ctypes.c_int64),
        ("off_val", ctypes.c_int64),
        ("off_bits", ctypes.c_int64),
        ("off_codes", ctypes.c_int64),
        ("bytes", ctypes.c_int64),
    ]


class NativeError(RuntimeError):
    pass


_P = ctypes.c_void_p
_SPEC = ctypes.POINTER(McSpec)
_SIGS = {
    "mc_abi_version": (ctypes.c_int, []),
    "mc_last_error": (ctypes.c_char_p, []),
    "mc_kernel_launches": (ctypes.c_int64, []),
    "mc_set_sm_reserve": (ctypes.c_int, [ctypes.c_int32]),
    "mc_top_k_count": (ctypes.c_int64, [ctypes.c_double, ctypes.c_int64]),
    "mc_payload_bytes": (ctypes.c_int64, [_SPEC, ctypes.c_int64]),
    "mc_payload_layout": (ctypes.c_int, [_SPEC, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(McLayout)]),
    "mc_encode_workspace_bytes": (ctypes.c_int64, [_SPEC, ctypes.c_int64]),
    "mc_derive_seed": (ctypes.c_int, [ctypes.c_uint64] * 4 + [ctypes.POINTER(ctypes.c_uint64)] * 2),
    "mc_encode": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, _P, _P, ctypes.c_uint64, ctypes.c_uint64, _P, _P,
                                 ctypes.c_int64, _P, _P]),
    "mc_encode_decode": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, _P, _P, ctypes.c_uint64, ctypes.c_uint64, _P, _P,
                                        ctypes.c_int64, _P, _P, _P]),
    "mc_encode_range": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P, _P,
                                       ctypes.c_uint64, ctypes.c_uint64, _P, _P, ctypes.c_int64, _P, _P, _P]),
    "mc_decode_mean": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, _P, _P, _P]),
    "mc_decode_workspace_bytes": (ctypes.c_int64, [_SPEC, ctypes.c_int64, ctypes.c_int32]),
    "mc_decode_mean_ws": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, _P, _P,
                                         ctypes.c_int64, _P, _P]),
    "mc_pack": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_int64), ctypes.c_int32, _P, _P]),
    "mc_unpack": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_int64), ctypes.c_int32, _P]),
    "mc_serialize": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, _P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), _P]),
    "mc_deserialize": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, _P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                      _P]),
    "mc_encode_push": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, _P, _P, ctypes.c_uint64, ctypes.c_uint64, _P,
                                      ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.c_int32, ctypes.c_uint32, _P,
                                      ctypes.c_int64, _P, _P]),
    "mc_push_wait": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64, _P, _P]),
    "mc_encode_push_dev": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, _P, _P, _P, _P, ctypes.POINTER(_P),
                                          ctypes.POINTER(_P), ctypes.c_int32, _P, _P, ctypes.c_int64, _P, _P]),
    "mc_push_wait_dev": (ctypes.c_int, [_P, ctypes.c_int32, _P, ctypes.c_uint64, _P, _P]),
    "mc_mcast_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, ctypes.c_int64,
                                       ctypes.POINTER(_P)]),
    "mc_mcast_ptrs": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_int64)]),
    "mc_mcast_destroy": (None, [_P]),
    "mc_encode_push_mc": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, _P, _P, ctypes.c_uint64, ctypes.c_uint64, _P, _P,
                                         _P, ctypes.c_uint32, _P, ctypes.c_int64, _P, _P]),
    "mc_derive_keys": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, _P, ctypes.c_uint64, ctypes.c_int32, _P, _P]),
    "mc_encode_dk": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, _P, _P, _P, _P, _P, ctypes.c_int64, _P, _P]),
    "mc_encode_decode_dk": (ctypes.c_int, [_SPEC, _P, ctypes.c_int64, _P, _P, _P, _P, _P, ctypes.c_int64, _P, _P,
                                           _P]),
    "mc_peer_enable": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32]),
    "mc_peer_probe": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int32, ctypes.c_uint32, _P]),
    "mc_pipe_create": (ctypes.c_int, [ctypes.POINTER(_P)]),
    "mc_pipe_destroy": (None, [_P]),
    "mc_pipe_group": (ctypes.c_int, [_P, _SPEC, _P, _P, _P, ctypes.c_int64, ctypes.c_int64, _P, _P, ctypes.c_uint64,
                                     ctypes.c_uint64, _P, _P, ctypes.c_int64, _P, _P, _P, _P]),
    "mc_pipe_finish": (ctypes.c_int, [_P, _P, _P, _P]),
}
EXPORTED = tuple(_SIGS)


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    path = Path(os.environ.get("MERGECOMP_LIB", LIB_PATH))
    if not path.exists():
        raise NativeError(
            f"{path} is missing: build the CUDA library with `python -m paper_2103_15195_b200.build` "
            "(there is no CPU fallback)"
        )
    so = ctypes.CDLL(str(path))
    for name, (res, args) in _SIGS.items():
        fn = getattr(so, name)
        fn.restype = res
        fn.argtypes = args
    if so.mc_abi_version() != 1:
        raise NativeError("libmergecomp ABI version mismatch")
    return so


def check(status: int, what: str) -> None:
    if status != MC_OK:
        msg = lib().mc_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({status}): {msg}")


def layout(cspec: McSpec, n: int, cap: int = 0) -> McLayout:
    out = McLayout()
    check(lib().mc_payload_layout(ctypes.byref(cspec), n, cap, ctypes.byref(out)), "mc_payload_layout")
    return out


def workspace_bytes(cspec: McSpec, n: int) -> int:
    v = lib().mc_encode_workspace_bytes(ctypes.byref(cspec), n)
    if v < 0:
        check(int(v), "mc_encode_workspace_bytes")
    return int(v)


def derive_key(root: int, worker: int, iteration: int, group: int) -> tuple[int, int]:
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    check(lib().mc_derive_seed(root, worker, iteration, group, ctypes.byref(lo), ctypes.byref(hi)), "mc_derive_seed")
    return lo.value, hi.value
