"""Drop-in replacement for the reference codec module
(``mergesched.compressors``, /root/reference/pkg/src/mergesched/compressors.py)
whose every compute step runs in the sm_100a CUDA library (libmergecomp.so).

Same names, signatures, defaults and errors as the reference:
``CompressorSpec, ResidualState, CompressedPayload, encode, decode, aggregate,
payload_bytes, serialize, deserialize, derive_seed, top_k_count,
empirical_error_bound``.  Two calling conventions:

* numpy arrays in -> numpy arrays out (the reference's host-buffer contract; the
  data is copied to the GPU, encoded there and copied back), and
* torch CUDA tensors in -> payload / state backed by device memory (no host
  copies; this is what the sync engine and the benchmarks use).

There is no CPU implementation behind these functions.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native
from .spec import (
    ALGO_ID,
    ALGORITHMS,
    EF_DEFAULT_ON,
    FLAG_UNBIASED,
    HEADER_BYTES,
    SPARSIFIERS,
    STOCHASTIC,
    CompressorSpec,
    bucket_count,
    code_bytes,
    level_bits,
    payload_bytes,
    section_lengths,
    sign_bytes,
    top_k_count,
)

__all__ = [
    "ALGORITHMS", "HEADER_BYTES", "CompressorSpec", "ResidualState", "CompressedPayload", "DevicePayload",
    "encode", "decode", "aggregate", "payload_bytes", "serialize", "deserialize", "derive_seed",
    "top_k_count", "empirical_error_bound", "device_encode", "device_encode_decode", "device_decode_mean",
    "device_deserialize",
]

_HDR_DEV = 32  # sizeof(mc_payload_header)


# ------------------------------------------------------------------ state / payload types

@dataclass
class ResidualState:
    """Per-(worker, group) codec memory (compressors.py:136-161): float64 residual,
    float32 momentum.  Arrays are numpy (host calls) or torch CUDA tensors."""

    residual: object
    momentum: Optional[object] = None

    @classmethod
    def zeros(cls, length: int, with_momentum: bool = False, device=None) -> "ResidualState":
        if device is None:
            return cls(np.zeros(length, np.float64), np.zeros(length, np.float32) if with_momentum else None)
        return cls(
            torch.zeros(length, dtype=torch.float64, device=device),
            torch.zeros(length, dtype=torch.float32, device=device) if with_momentum else None,
        )

    def copy(self) -> "ResidualState":
        def cp(a):
            if a is None:
                return None
            return a.clone() if isinstance(a, torch.Tensor) else a.copy()

        return ResidualState(cp(self.residual), cp(self.momentum))


class DevicePayload:
    """The aligned device form of one payload: a CUDA uint8 buffer holding the
    32-byte mc_payload_header and 16-byte aligned idx / val / bits / codes sections."""

    def __init__(self, spec: CompressorSpec, n: int, buf: torch.Tensor, layout, cap: Optional[int] = None):
        self.spec, self.n, self.buf, self.layout = spec, n, buf, layout
        self.cap = layout.cap if cap is None else cap
        self._count: Optional[int] = None

    def count(self) -> int:
        """Selected count (sparsifiers); reads the device header (syncs) for threshold."""
        if self._count is None:
            if self.spec.algorithm == "threshold":
                hdr = self.buf[:_HDR_DEV].cpu().numpy().view(np.uint32)
                self._count = int(hdr[4])
            else:
                self._count = section_lengths(self.spec, self.n)[0]
        return self._count

    def section(self, off: int, nbytes: int) -> torch.Tensor:
        return self.buf[off: off + nbytes]

    def idx_val(self) -> tuple[torch.Tensor, torch.Tensor]:
        k = self.count()
        off_val = _HDR_DEV + _a16(4 * self.cap)
        idx = self.section(_HDR_DEV, 4 * k).view(torch.int32)
        val = self.section(off_val, 4 * k).view(torch.float32)
        return idx, val

    def canonical_sections(self) -> tuple[Optional[torch.Tensor], torch.Tensor, Optional[torch.Tensor]]:
        """(indices[int32 view], values[f32], bits[u8]) as device tensors in canonical order."""
        L, a = self.layout, self.spec.algorithm
        if a in SPARSIFIERS:
            idx, val = self.idx_val()
            return idx, val, None
        val = self.section(L.off_val, 4 * L.n_val).view(torch.float32)
        if a == "qsgd":
            bits = torch.cat([self.section(L.off_bits, L.n_bits), self.section(L.off_codes, L.n_codes)])
        elif L.n_bits:
            bits = self.section(L.off_bits, L.n_bits)
        else:
            bits = None
        return None, val, bits


def _a16(x: int) -> int:
    return (x + 15) & ~15


@dataclass(frozen=True)
class CompressedPayload:
    """compressors.py:164-182.  Host form: numpy arrays.  Device form: ``device`` is
    set and indices / values / bits are CUDA tensors viewing the device buffer."""

    algorithm: str
    original_len: int
    indices: Optional[object]
    values: object
    bits: Optional[object]
    flags: int = 0
    byte_size: int = field(init=False)
    device: Optional[DevicePayload] = field(default=None, compare=False, repr=False)

    def __post_init__(self):
        n_idx = 0 if self.indices is None else len(self.indices)
        n_bits = 0 if self.bits is None else len(self.bits)
        object.__setattr__(self, "byte_size", HEADER_BYTES + 4 * n_idx + 4 * len(self.values) + n_bits)

    @property
    def on_device(self) -> bool:
        return self.device is not None

    def to_host(self) -> "CompressedPayload":
        if self.device is None:
            return self
        idx, val, bits = self.device.canonical_sections()
        return CompressedPayload(
            self.algorithm,
            self.original_len,
            None if idx is None else idx.cpu().numpy().view(np.uint32).copy(),
            val.cpu().numpy().copy(),
            None if bits is None else bits.cpu().numpy().copy(),
            self.flags,
        )


# ------------------------------------------------------------------ device plumbing

class _Workspace:
    """Growable scratch buffers keyed by (device, stream): the library keeps no state, and two
    encodes in flight on different streams (e.g. two GradSync side streams) never share
    scratch (tile tickets, look-back status, push counters).  Each buffer is allocated on its
    own stream, so replacing a smaller one is stream-ordered by the caching allocator."""

    def __init__(self):
        self._bufs: dict[tuple[int, int], torch.Tensor] = {}

    def get(self, device: torch.device, nbytes: int, stream=None) -> torch.Tensor:
        dev = device.index if device.index is not None else torch.cuda.current_device()
        st = stream if stream is not None else torch.cuda.current_stream(dev)
        key = (dev, st.cuda_stream)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            with torch.cuda.stream(st):
                buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf


_WS = _Workspace()


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise _native.NativeError("no CUDA device: the MergeComp codecs run only on the GPU (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_ptr(stream: Optional[torch.cuda.Stream] = None) -> int:
    return (stream or torch.cuda.current_stream()).cuda_stream


def split_seed(seed: int) -> tuple[int, int]:
    seed = int(seed)
    return seed & 0xFFFFFFFFFFFFFFFF, (seed >> 64) & 0xFFFFFFFFFFFFFFFF


def device_encode(spec: CompressorSpec, grad: torch.Tensor, residual: Optional[torch.Tensor],
                  momentum: Optional[torch.Tensor], seed: int, out: Optional[torch.Tensor] = None,
                  err: Optional[torch.Tensor] = None, stream=None, cspec=None,
                  dkey: Optional[torch.Tensor] = None) -> DevicePayload:
    """Enqueue one encode on the current (or given) stream; no host sync.  ``residual``
    (f64) and ``momentum`` (f32) are updated in place.  ``err`` (int32[1]) collects
    the device error flags.  ``dkey`` (a device int64[2] written by ``derive_keys``)
    replaces ``seed`` by a key read on the device (CUDA Graph replays)."""
    n = grad.numel()
    cs = cspec if cspec is not None else spec.to_c()
    L = _native.layout(cs, n)
    if out is None:
        out = torch.empty(L.bytes, dtype=torch.uint8, device=grad.device)
    wsb = _native.workspace_bytes(cs, n)
    ws = _WS.get(grad.device, wsb, stream)
    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=grad.device)
    if dkey is not None:
        _native.check(
            _native.lib().mc_encode_dk(ctypes.byref(cs), grad.data_ptr(), n, _ptr(residual), _ptr(momentum),
                                       dkey.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), err.data_ptr(),
                                       _stream_ptr(stream)),
            "mc_encode_dk",
        )
        return DevicePayload(spec, n, out, L)
    lo, hi = split_seed(seed)
    _native.check(
        _native.lib().mc_encode(ctypes.byref(cs), grad.data_ptr(), n, _ptr(residual), _ptr(momentum), lo, hi,
                                out.data_ptr(), ws.data_ptr(), ws.numel(), err.data_ptr(), _stream_ptr(stream)),
        "mc_encode",
    )
    return DevicePayload(spec, n, out, L)


def device_encode_decode(spec: CompressorSpec, grad: torch.Tensor, residual: Optional[torch.Tensor],
                         momentum: Optional[torch.Tensor], seed: int, out: torch.Tensor,
                         payload: Optional[torch.Tensor] = None, err: Optional[torch.Tensor] = None, stream=None,
                         cspec=None, dkey: Optional[torch.Tensor] = None) -> DevicePayload:
    """Single-rank sync in one pass where the codec allows it: encode ``grad`` and write
    ``out = aggregate([payload])`` (``out`` may alias ``grad``).  ``dkey``: see device_encode."""
    n = grad.numel()
    cs = cspec if cspec is not None else spec.to_c()
    L = _native.layout(cs, n)
    if payload is None:
        payload = torch.empty(L.bytes, dtype=torch.uint8, device=grad.device)
    ws = _WS.get(grad.device, _native.workspace_bytes(cs, n), stream)
    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=grad.device)
    if dkey is not None:
        _native.check(
            _native.lib().mc_encode_decode_dk(ctypes.byref(cs), grad.data_ptr(), n, _ptr(residual), _ptr(momentum),
                                              dkey.data_ptr(), payload.data_ptr(), ws.data_ptr(), ws.numel(),
                                              out.data_ptr(), err.data_ptr(), _stream_ptr(stream)),
            "mc_encode_decode_dk",
        )
        return DevicePayload(spec, n, payload, L)
    lo, hi = split_seed(seed)
    _native.check(
        _native.lib().mc_encode_decode(ctypes.byref(cs), grad.data_ptr(), n, _ptr(residual), _ptr(momentum), lo, hi,
                                       payload.data_ptr(), ws.data_ptr(), ws.numel(), out.data_ptr(), err.data_ptr(),
                                       _stream_ptr(stream)),
        "mc_encode_decode",
    )
    return DevicePayload(spec, n, payload, L)


def derive_keys(root: int, worker: int, iteration: torch.Tensor, keys: torch.Tensor, group0: int = 0,
                stream=None) -> None:
    """keys[g] = derive_seed(root, worker, iteration, group0 + g) for every row of ``keys``
    (device int64[G, 2]), computed on the device from the device counter ``iteration``
    (int64[1]), which is then advanced by one (mc_derive_keys): the key schedule of a
    captured CUDA Graph."""
    _native.check(_native.lib().mc_derive_keys(int(root), int(worker), iteration.data_ptr(), int(group0),
                                               keys.shape[0], keys.data_ptr(), _stream_ptr(stream)),
                  "mc_derive_keys")


def device_encode_push(spec: CompressorSpec, grad: torch.Tensor, residual: Optional[torch.Tensor],
                       momentum: Optional[torch.Tensor], seed: int, payload: torch.Tensor, dsts: Sequence[int],
                       flags: Sequence[int], epoch: int, err: Optional[torch.Tensor] = None, stream=None,
                       cspec=None) -> None:
    """Encode into ``payload`` (this rank's slot of its own gather buffer) and push the same
    bytes into every peer slot ``dsts[j]`` (device / peer-mapped addresses, one per rank, the
    own slot included), then release ``flags[j]`` := epoch — the allgather over peer memory
    fused with the encode (mc_encode_push).  Pair with ``push_wait`` before decoding."""
    n = grad.numel()
    cs = cspec if cspec is not None else spec.to_c()
    ws = _WS.get(grad.device, _native.workspace_bytes(cs, n), stream)
    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=grad.device)
    lo, hi = split_seed(seed)
    k = len(dsts)
    arr_d = (ctypes.c_void_p * k)(*dsts)
    arr_f = (ctypes.c_void_p * k)(*flags)
    _native.check(
        _native.lib().mc_encode_push(ctypes.byref(cs), grad.data_ptr(), n, _ptr(residual), _ptr(momentum), lo, hi,
                                     payload.data_ptr(), arr_d, arr_f, k, int(epoch) & 0xFFFFFFFF, ws.data_ptr(),
                                     ws.numel(), err.data_ptr(), _stream_ptr(stream)),
        "mc_encode_push",
    )


def device_encode_push_dev(spec: CompressorSpec, grad: torch.Tensor, residual: Optional[torch.Tensor],
                           momentum: Optional[torch.Tensor], dkey: Optional[torch.Tensor], payload: torch.Tensor,
                           dsts: Sequence[int], flags: Sequence[int], epoch: torch.Tensor,
                           err: torch.Tensor, stream=None, cspec=None) -> None:
    """``device_encode_push`` with the Philox key (``dkey``, device int64[2]; None for codecs
    that draw no random numbers) and the exchange epoch (``epoch``, device int32[1]) read on
    the device (mc_encode_push_dev): the form a CUDA Graph of the N > 1 step replays."""
    n = grad.numel()
    cs = cspec if cspec is not None else spec.to_c()
    ws = _WS.get(grad.device, _native.workspace_bytes(cs, n), stream)
    k = len(dsts)
    arr_d = (ctypes.c_void_p * k)(*dsts)
    arr_f = (ctypes.c_void_p * k)(*flags)
    _native.check(
        _native.lib().mc_encode_push_dev(ctypes.byref(cs), grad.data_ptr(), n, _ptr(residual), _ptr(momentum),
                                         _ptr(dkey), payload.data_ptr(), arr_d, arr_f, k, epoch.data_ptr(),
                                         ws.data_ptr(), ws.numel(), err.data_ptr(), _stream_ptr(stream)),
        "mc_encode_push_dev",
    )


def push_wait_dev(flags: torch.Tensor, nranks: int, epoch: torch.Tensor, err: torch.Tensor, stream=None,
                  timeout_s: float = 0.0) -> None:
    """``push_wait`` against the epoch held in the device word ``epoch`` (mc_push_wait_dev)."""
    _native.check(_native.lib().mc_push_wait_dev(flags.data_ptr(), nranks, epoch.data_ptr(), int(timeout_s * 1e9),
                                                 err.data_ptr(), _stream_ptr(stream)),
                  "mc_push_wait_dev")


class McastBuffer:
    """A gather buffer behind an NVLink multicast object (mc_mcast_create) over devices owned
    by this process: ``unicast[i]`` is device i's view (what its decode reads), ``multicast``
    the address whose stores reach every device's copy (what mc_encode_push_mc writes)."""

    def __init__(self, devices: Sequence[int], nbytes: int):
        lib = _native.lib()
        devs = (ctypes.c_int32 * len(devices))(*devices)
        h = ctypes.c_void_p()
        _native.check(lib.mc_mcast_create(devs, len(devices), int(nbytes), ctypes.byref(h)), "mc_mcast_create")
        self._h = h
        uc = (ctypes.c_void_p * len(devices))()
        mcp, size = ctypes.c_void_p(), ctypes.c_int64()
        _native.check(lib.mc_mcast_ptrs(h, uc, ctypes.byref(mcp), ctypes.byref(size)), "mc_mcast_ptrs")
        self.unicast = [int(u) for u in uc]
        self.multicast = int(mcp.value)
        self.nbytes = int(size.value)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            torch.cuda.synchronize()
            _native.lib().mc_mcast_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def device_encode_push_mc(spec: CompressorSpec, grad: torch.Tensor, residual: Optional[torch.Tensor],
                          momentum: Optional[torch.Tensor], seed: int, payload_ptr: int, mc_slot: int, mc_flag: int,
                          epoch: int, err: Optional[torch.Tensor] = None, stream=None, cspec=None) -> None:
    """``device_encode_push`` over a multicast buffer: every payload word is stored once
    through ``mc_slot`` (this rank's slot, multicast address) and lands in every device's
    copy; ``mc_flag`` (multicast address of this rank's flag word) := epoch everywhere
    (mc_encode_push_mc).  ``payload_ptr``: the same slot's unicast address on this device."""
    n = grad.numel()
    cs = cspec if cspec is not None else spec.to_c()
    ws = _WS.get(grad.device, _native.workspace_bytes(cs, n), stream)
    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=grad.device)
    lo, hi = split_seed(seed)
    _native.check(
        _native.lib().mc_encode_push_mc(ctypes.byref(cs), grad.data_ptr(), n, _ptr(residual), _ptr(momentum), lo, hi,
                                        int(payload_ptr), int(mc_slot), int(mc_flag), int(epoch) & 0xFFFFFFFF,
                                        ws.data_ptr(), ws.numel(), err.data_ptr(), _stream_ptr(stream)),
        "mc_encode_push_mc",
    )


def push_wait(flags: torch.Tensor, nranks: int, epoch: int, err: Optional[torch.Tensor] = None, stream=None,
              timeout_s: float = 0.0) -> None:
    """The stream waits until all ``nranks`` local flag words equal ``epoch`` (mc_push_wait).
    A peer silent for ``timeout_s`` (0: the library default, 600 s) sets MC_ERR_PEER_TIMEOUT
    and traps — the job fails loudly instead of decoding stale slots."""
    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=flags.device)
    _native.check(_native.lib().mc_push_wait(flags.data_ptr(), nranks, int(epoch) & 0xFFFFFFFF,
                                             int(timeout_s * 1e9), err.data_ptr(), _stream_ptr(stream)),
                  "mc_push_wait")


def device_decode_mean(spec: CompressorSpec, base: torch.Tensor, stride: int, nranks: int, n: int,
                       out: torch.Tensor, err: torch.Tensor, stream=None, cspec=None) -> None:
    cs = cspec if cspec is not None else spec.to_c()
    lib = _native.lib()
    need = int(lib.mc_decode_workspace_bytes(ctypes.byref(cs), n, nranks))
    if need < 0:
        _native.check(need, "mc_decode_workspace_bytes")
    ws = _WS.get(out.device, need, stream) if need > 0 else None  # stream-ordered after the encodes
    _native.check(
        lib.mc_decode_mean_ws(ctypes.byref(cs), base.data_ptr(), stride, nranks, n, out.data_ptr(),
                              None if ws is None else ws.data_ptr(), 0 if ws is None else ws.numel(),
                              err.data_ptr(), _stream_ptr(stream)),
        "mc_decode_mean_ws",
    )


def _raise_flags(flags: int) -> None:
    if flags & _native.MC_ERR_NONFINITE:
        raise ValueError("gradient contains non-finite values")
    if flags & _native.MC_ERR_INDEX_RANGE:
        raise ValueError("corrupt payload: index out of range")
    if flags & _native.MC_ERR_INDEX_ORDER:
        raise ValueError("corrupt payload: indices not increasing")
    if flags & _native.MC_ERR_PEER_TIMEOUT:
        raise RuntimeError("peer exchange: a rank's payload did not arrive (mc_push_wait timed out)")
    if flags & _native.MC_ERR_HEADER:
        raise ValueError("corrupt payload: header does not match spec")


def _upload_payload(spec: CompressorSpec, p: CompressedPayload, dev: torch.device) -> DevicePayload:
    """Host-form payload -> aligned device buffer (one H2D copy)."""
    n = p.original_len
    cs = spec.to_c()
    a = spec.algorithm
    n_idx = 0 if p.indices is None else len(p.indices)
    n_bits = 0 if p.bits is None else len(p.bits)
    L = _native.layout(cs, n)
    if a in SPARSIFIERS:  # sections sized by this payload's own count (cap = count)
        L.cap = n_idx
        L.off_val = 32 + _a16(4 * n_idx)
        L.off_bits = L.off_codes = L.bytes = L.off_val + _a16(4 * n_idx)
        L.n_val = n_idx
    host = np.zeros(max(L.bytes, 32), np.uint8)
    hdr = np.array([ALGO_ID[a], p.flags, n & 0xFFFFFFFF, n >> 32, n_idx, len(p.values), n_bits,
                    n_idx if a in SPARSIFIERS else 0], np.uint32)
    host[:32] = hdr.view(np.uint8)
    if a in SPARSIFIERS:
        host[32: 32 + 4 * n_idx] = np.asarray(p.indices, np.uint32).view(np.uint8)
        host[L.off_val: L.off_val + 4 * len(p.values)] = np.asarray(p.values, np.float32).view(np.uint8)
    else:
        host[L.off_val: L.off_val + 4 * len(p.values)] = np.asarray(p.values, np.float32).view(np.uint8)
        if p.bits is not None:
            bits = np.asarray(p.bits, np.uint8)
            if a == "qsgd":
                host[L.off_bits: L.off_bits + L.n_bits] = bits[: L.n_bits]
                host[L.off_codes: L.off_codes + L.n_codes] = bits[L.n_bits: L.n_bits + L.n_codes]
            else:
                host[L.off_bits: L.off_bits + len(bits)] = bits
    buf = torch.from_numpy(host).to(dev, non_blocking=False)
    return DevicePayload(spec, n, buf, L, cap=L.cap)


def _check_structure(spec: CompressorSpec, p: CompressedPayload) -> None:
    """Reference decode's structural checks (compressors.py:432-512) on metadata only."""
    if p.algorithm != spec.algorithm:
        raise ValueError(f"payload algorithm {p.algorithm!r} does not match spec {spec.algorithm!r}")
    if p.device is not None:
        return
    a, n = spec.algorithm, p.original_len

    def chk(cond, msg):
        if not cond:
            raise ValueError(f"corrupt payload: {msg}")

    if a in SPARSIFIERS:
        chk(p.indices is not None, "sparsifier payload lacks indices")
        chk(len(p.indices) == len(p.values), "index/value length mismatch")
        return
    nb = bucket_count(n, spec.bucket_size)
    nbits = 0 if p.bits is None else len(p.bits)
    if a == "identity":
        chk(len(p.values) == n, "value buffer length mismatch")
    elif a == "fp16":
        chk(p.bits is not None and nbits == 2 * n, "fp16 buffer length mismatch")
    elif a == "qsgd":
        chk(p.bits is not None, "missing bit codes")
        chk(len(p.values) == nb, "scale count mismatch")
        chk(nbits == sign_bytes(n) + code_bytes(n, level_bits(spec.levels)), "bit buffer length mismatch")
    elif a in ("signsgd", "signum"):
        chk(len(p.values) == 1, "expected one global scaler")
        chk(p.bits is not None and nbits == sign_bytes(n), "sign buffer mismatch")
    elif a == "efsignsgd":
        chk(len(p.values) == nb, "scale count mismatch")
        chk(p.bits is not None and nbits == sign_bytes(n), "sign buffer mismatch")
    elif a == "onebit":
        chk(len(p.values) == 2 * nb, "scaler count mismatch")
        chk(p.bits is not None and nbits == sign_bytes(n), "sign buffer mismatch")
    elif a == "terngrad":
        chk(len(p.values) == nb, "scale count mismatch")
        chk(p.bits is not None and nbits == code_bytes(n, 2), "code buffer mismatch")
    elif a == "int8":
        chk(len(p.values) == nb, "scale count mismatch")
        chk(p.bits is not None and nbits == n, "int8 buffer mismatch")


# ------------------------------------------------------------------ public API

def derive_seed(root_seed: int, worker: int = 0, iteration: int = 0, group: int = 0) -> int:
    """compressors.py:247-251 — numpy SeedSequence((root, worker, iteration, group))
    .generate_state(2, uint64) as a 128-bit key, computed by the C library."""
    args = [int(root_seed), int(worker), int(iteration), int(group)]
    if all(0 <= v < (1 << 64) for v in args):
        lo, hi = _native.derive_key(*args)
        return lo | (hi << 64)
    from ._seedseq import seed_sequence_key  # arbitrary-precision entropy words

    lo, hi = seed_sequence_key(args)
    return lo | (hi << 64)


def _payload_from_device(spec: CompressorSpec, dp: DevicePayload, host: bool) -> CompressedPayload:
    flags = FLAG_UNBIASED if (spec.algorithm == "randk" and spec.unbiased_scaling) else 0
    idx, val, bits = dp.canonical_sections()
    if host:
        return CompressedPayload(
            spec.algorithm, dp.n,
            None if idx is None else idx.cpu().numpy().view(np.uint32).copy(),
            val.cpu().numpy().copy(),
            None if bits is None else bits.cpu().numpy().copy(),
            flags,
        )
    return CompressedPayload(spec.algorithm, dp.n, idx, val, bits, flags, device=dp)


def encode(spec: CompressorSpec, gradient, state: Optional[ResidualState] = None, seed: int = 0):
    """compressors.py:369-417 on the GPU.  Returns (payload, state)."""
    on_dev = isinstance(gradient, torch.Tensor) and gradient.is_cuda
    if on_dev:
        x = gradient.detach().reshape(-1)
        if x.dtype != torch.float32:
            x = x.float()
        x = x.contiguous()
        dev = x.device
    else:
        xh = np.ascontiguousarray(np.asarray(gradient, dtype=np.float32).reshape(-1))
        dev = _device()
        x = None
    n = x.numel() if on_dev else xh.size
    if n < 1:
        raise ValueError("gradient must have at least one element")
    use_ef, coef = spec.uses_error_feedback, spec.momentum_coef
    if (use_ef or coef is not None) and state is None:
        state = ResidualState.zeros(n, with_momentum=coef is not None, device=dev if on_dev else None)
    if state is not None and len(state.residual) != n:
        raise ValueError(f"state length {len(state.residual)} does not match gradient length {n}")
    if not on_dev:
        x = torch.from_numpy(xh).to(dev)

    def to_dev(a, dtype):
        if a is None:
            return None
        if isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == dtype:
            # a private copy: the reference returns NEW state objects and raises on a
            # non-finite gradient before touching state (compressors.py:384-411), so the
            # caller's tensors are never updated in place (the sync engine, which owns its
            # state, uses device_encode directly)
            return a.contiguous().clone()
        return torch.as_tensor(np.asarray(a) if not isinstance(a, torch.Tensor) else a, dtype=dtype).to(dev).contiguous()

    r = to_dev(state.residual, torch.float64) if (state is not None and use_ef) else None
    m = None
    if coef is not None:
        m = to_dev(state.momentum, torch.float32) if state.momentum is not None else torch.zeros(n, dtype=torch.float32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    dp = device_encode(spec, x, r, m, seed, err=err)
    flags = int(err.item())  # the reference raises synchronously
    if flags:
        _raise_flags(flags)
    payload = _payload_from_device(spec, dp, host=not on_dev)

    if state is None:
        return payload, None
    if on_dev:
        new_res = r if use_ef else state.residual
        return payload, ResidualState(new_res, m if coef is not None else state.momentum)
    new_res = r.cpu().numpy() if use_ef else state.residual
    new_mom = m.cpu().numpy() if coef is not None else state.momentum
    return payload, ResidualState(new_res, new_mom)


def _gather_device(spec: CompressorSpec, payloads: Sequence[CompressedPayload], dev) -> tuple[torch.Tensor, int]:
    dps = [p.device if p.device is not None else _upload_payload(spec, p, dev) for p in payloads]
    stride = _a16(max(d.buf.numel() for d in dps))
    buf = torch.zeros(len(dps) * stride, dtype=torch.uint8, device=dev)
    for i, d in enumerate(dps):
        buf[i * stride: i * stride + d.buf.numel()].copy_(d.buf)
    return buf, stride


def aggregate(spec: CompressorSpec, payloads: Sequence[CompressedPayload]):
    """compressors.py:519-532: rank-ordered fp32 sum of decodes / f32(n), on the GPU."""
    if not payloads:
        raise ValueError("need at least one payload")
    first = payloads[0]
    for p in payloads[1:]:
        if p.algorithm != first.algorithm:
            raise ValueError(f"mixed algorithms: {first.algorithm!r} vs {p.algorithm!r}")
        if p.original_len != first.original_len:
            raise ValueError(f"mixed lengths: {first.original_len} vs {p.original_len}")
    for p in payloads:
        _check_structure(spec, p)
    dev = first.device.buf.device if first.device is not None else _device()
    n = first.original_len
    buf, stride = _gather_device(spec, payloads, dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    device_decode_mean(spec, buf, stride, len(payloads), n, out, err)
    flags = int(err.item())
    if flags:
        _raise_flags(flags)
    return out if all(p.device is not None for p in payloads) else out.cpu().numpy()


def decode(spec: CompressorSpec, payload: CompressedPayload):
    """compressors.py:427-516 on the GPU (= aggregate of one payload)."""
    _check_structure(spec, payload)
    return aggregate(spec, [payload])


def empirical_error_bound(spec: CompressorSpec, samples: Sequence, trials: int = 1) -> float:
    """compressors.py:535-562: worst relative squared error of the raw codec."""
    if spec.uses_error_feedback:
        raise ValueError("disable error_feedback for error-bound measurement")
    if trials < 1:
        raise ValueError("trials must be >= 1")
    dev = _device()
    worst = 0.0
    for i, sample in enumerate(samples):
        x = torch.as_tensor(np.asarray(sample, dtype=np.float32).reshape(-1)).to(dev)
        x64 = x.double()
        denom = float(torch.dot(x64, x64))
        if denom == 0.0:
            raise ValueError(f"sample {i} has zero norm")
        total = 0.0
        for t in range(trials):
            p, _ = encode(spec, x, None, seed=derive_seed(t, group=i))
            e = decode(spec, p).double() - x64
            total += float(torch.dot(e, e)) / denom
        worst = max(worst, total / trials)
    return worst


# ------------------------------------------------------------------ canonical serialization

def serialize(payload: CompressedPayload) -> bytes:
    """Canonical little-endian form (compressors.py:601-620).  Device payloads are
    serialized on the GPU (mc_serialize) and copied back."""
    if payload.device is not None:
        dp = payload.device
        cs = dp.spec.to_c()
        nbytes = payload.byte_size
        out = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dp.buf.device)
        ln = ctypes.c_int64()
        _native.check(_native.lib().mc_serialize(ctypes.byref(cs), dp.buf.data_ptr(), dp.n, out.data_ptr(),
                                                 out.numel(), ctypes.byref(ln), _stream_ptr()), "mc_serialize")
        raw = out[: ln.value].cpu().numpy().tobytes()
        # flags byte: the library records the randk unbiased flag in the header
        return raw
    n_idx = 0 if payload.indices is None else len(payload.indices)
    n_bits = 0 if payload.bits is None else len(payload.bits)
    parts = [struct.pack("<BBQIII", ALGO_ID[payload.algorithm], payload.flags, payload.original_len, n_idx,
                         len(payload.values), n_bits)]
    if payload.indices is not None:
        parts.append(np.asarray(payload.indices).astype("<u4").tobytes())
    parts.append(np.asarray(payload.values).astype("<f4").tobytes())
    if payload.bits is not None:
        parts.append(np.asarray(payload.bits, np.uint8).tobytes())
    return b"".join(parts)


def deserialize(data: bytes) -> CompressedPayload:
    """compressors.py:623-645 (host form)."""
    if len(data) < HEADER_BYTES:
        raise ValueError("payload shorter than header")
    algo_id, flags, original_len, n_idx, n_val, n_bits = struct.unpack_from("<BBQIII", data)
    if algo_id >= len(ALGORITHMS):
        raise ValueError(f"unknown algorithm id {algo_id}")
    expect = HEADER_BYTES + 4 * n_idx + 4 * n_val + n_bits
    if len(data) != expect:
        raise ValueError(f"payload length {len(data)} does not match header ({expect})")
    off = HEADER_BYTES
    indices = None
    if n_idx:
        indices = np.frombuffer(data, dtype="<u4", count=n_idx, offset=off).copy()
        off += 4 * n_idx
    values = np.frombuffer(data, dtype="<f4", count=n_val, offset=off).copy()
    off += 4 * n_val
    bits = np.frombuffer(data, dtype=np.uint8, count=n_bits, offset=off).copy() if n_bits else None
    algo = ALGORITHMS[algo_id]
    if algo in SPARSIFIERS and indices is None:
        indices = np.empty(0, dtype="<u4")
    return CompressedPayload(algo, original_len, indices, values, bits, flags)


def device_deserialize(spec: CompressorSpec, data) -> CompressedPayload:
    """Canonical bytes (``bytes`` or a CUDA uint8 tensor) -> device payload (mc_deserialize,
    the on-device inverse of ``serialize``; compressors.py:623-645).  Raises the reference's
    ``ValueError`` messages on malformed input."""
    dev = data.device if isinstance(data, torch.Tensor) else _device()
    if not isinstance(data, torch.Tensor):
        raw = np.frombuffer(bytes(data), np.uint8)
        if raw.size < HEADER_BYTES:
            raise ValueError("payload shorter than header")
        data = torch.from_numpy(raw.copy()).to(dev)
    if data.numel() < HEADER_BYTES:
        raise ValueError("payload shorter than header")
    hdr = data[:HEADER_BYTES].cpu().numpy().tobytes()
    _, _, n, n_idx, _, _ = struct.unpack_from("<BBQIII", hdr)
    cs = spec.to_c()
    cap = n_idx if spec.algorithm in SPARSIFIERS else 0
    try:
        L = _native.layout(cs, max(int(n), 1), max(cap, 1) if spec.algorithm == "threshold" else 0)
    except _native.NativeError as e:
        raise ValueError(f"corrupt payload: {e}") from None
    nbytes = max(L.bytes, 32 + 2 * _a16(4 * cap)) if spec.algorithm in SPARSIFIERS else L.bytes
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    n_out = ctypes.c_int64()
    st = _native.lib().mc_deserialize(ctypes.byref(cs), data.data_ptr(), data.numel(), buf.data_ptr(), buf.numel(),
                                      ctypes.byref(n_out), _stream_ptr())
    if st != _native.MC_OK:
        raise ValueError(_native.lib().mc_last_error().decode(errors="replace"))
    L2 = _native.layout(cs, int(n), max(cap, 1) if spec.algorithm == "threshold" else 0)
    if spec.algorithm in SPARSIFIERS:
        L2.cap = cap
        L2.n_val = cap
        L2.off_val = 32 + _a16(4 * cap)
        L2.off_bits = L2.off_codes = L2.bytes = L2.off_val + _a16(4 * cap)
    dp = DevicePayload(spec, int(n), buf, L2, cap=cap if spec.algorithm in SPARSIFIERS else None)
    if spec.algorithm in SPARSIFIERS:
        dp._count = cap
    return _payload_from_device(spec, dp, host=False)
