"""CPU oracle for the MergeComp compressed-gradient-sync path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The shipped package never imports it and has no
CPU fallback.

It restates, in numpy, the reference codec semantics of
``/root/reference/pkg/src/mergesched/compressors.py`` (cited per function as
``compressors.py:LINE``).  The arithmetic is chosen op-for-op so numpy rounds
exactly as the reference does (float32 pairwise means, float64 residuals,
float32 RNE casts, Philox streams).

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
package (``mergesched``) in the build container and records its outputs on
seeded inputs into ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks this oracle against every one of them bit for bit.

Documented deviation (the top-k tie contract): the reference
uses ``np.argpartition`` whose choice among equal magnitudes at the k-th
boundary is implementation defined (it even changes with numpy's SIMD
dispatch).  This oracle — like the GPU kernels — takes the LOWEST indices among
ties.  On tie-free inputs the two are identical; golden vectors are tie-free.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

ALGORITHMS = (
    "identity", "fp16", "topk", "randk", "dgc_lite", "threshold", "qsgd",
    "signsgd", "efsignsgd", "onebit", "signum", "terngrad", "int8",
)  # compressors.py:29-43 (order = wire algorithm id)
ALGO_ID = {a: i for i, a in enumerate(ALGORITHMS)}
SPARSE = frozenset({"topk", "randk", "dgc_lite", "threshold"})  # compressors.py:50
HEADER = 22  # struct "<BBQIII", compressors.py:53


@dataclass(frozen=True)
class Payload:
    """Host form of one encoded group (compressors.py:164-182)."""

    algorithm: str
    original_len: int
    indices: Optional[np.ndarray]
    values: np.ndarray
    bits: Optional[np.ndarray]
    flags: int = 0

    @property
    def byte_size(self) -> int:
        ni = 0 if self.indices is None else len(self.indices)
        nb = 0 if self.bits is None else len(self.bits)
        return HEADER + 4 * ni + 4 * len(self.values) + nb


@dataclass
class State:
    residual: np.ndarray  # float64 (compressors.py:141-145)
    momentum: Optional[np.ndarray] = None  # float32


# ---------------------------------------------------------------- spec helpers

def ef_on(spec) -> bool:
    """compressors.py:94-98"""
    if spec.error_feedback is not None:
        return bool(spec.error_feedback)
    return spec.algorithm in ("topk", "dgc_lite", "efsignsgd", "onebit")


def momentum_of(spec) -> Optional[float]:
    """compressors.py:100-107"""
    if spec.algorithm == "signum":
        return 0.9 if spec.momentum is None else spec.momentum
    if spec.algorithm == "dgc_lite":
        return spec.momentum
    return None


def keep_count(sparsity: float, n: int) -> int:
    """k = max(1, ceil(round((1-s)*n, 9)))  — compressors.py:185-194"""
    if n < 1:
        raise ValueError("length must be >= 1")
    return max(1, math.ceil(round((1.0 - sparsity) * n, 9)))


def n_buckets(n: int, b: int) -> int:
    return -(-n // b)


def code_width(levels: int) -> int:
    """compressors.py:241-242"""
    return max(1, (levels - 1).bit_length())


# ---------------------------------------------------------------- bit packing

def pack_msb(codes: np.ndarray, width: int) -> np.ndarray:
    """MSB-first concatenation of ``width``-bit codes (compressors.py:199-205)."""
    if width == 8:
        return codes.astype(np.uint8)
    bitplanes = (codes.astype(np.uint32)[:, None] >> np.arange(width - 1, -1, -1, dtype=np.uint32)) & 1
    return np.packbits(bitplanes.astype(np.uint8).ravel())


def unpack_msb(packed: np.ndarray, count: int, width: int) -> np.ndarray:
    """compressors.py:208-213"""
    if width == 8:
        return packed[:count].astype(np.uint32)
    planes = np.unpackbits(packed)[: count * width].reshape(count, width).astype(np.uint32)
    return (planes << np.arange(width - 1, -1, -1, dtype=np.uint32)).sum(axis=1, dtype=np.uint32)


def sign_bits(x: np.ndarray) -> np.ndarray:
    """bit = (x >= 0), -0.0 counts as non-negative (compressors.py:216-217)."""
    return np.packbits((x >= 0).astype(np.uint8))


def signs_pm1(packed: np.ndarray, count: int) -> np.ndarray:
    """compressors.py:220-222"""
    return np.where(np.unpackbits(packed)[:count] == 1, np.float32(1.0), np.float32(-1.0))


# ---------------------------------------------------------------- numpy semantics restated

def pairwise_f32(a: np.ndarray) -> np.float32:
    """numpy's float32 pairwise summation tree (umath loops_utils pairwise_sum),
    as the ufunc reduce applies it: 0 + P(a).  Used to *document and test* the
    order the GPU reproduces; the codecs below call ``.mean()`` directly."""
    def rec(lo: int, n: int) -> np.float32:
        if n < 8:
            acc = np.float32(-0.0)
            for i in range(lo, lo + n):
                acc = np.float32(acc + a[i])
            return acc
        if n <= 128:
            r = [np.float32(a[lo + j]) for j in range(8)]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] = np.float32(r[j] + a[lo + i + j])
                i += 8
            s = np.float32(np.float32(np.float32(r[0] + r[1]) + np.float32(r[2] + r[3]))
                           + np.float32(np.float32(r[4] + r[5]) + np.float32(r[6] + r[7])))
            while i < n:
                s = np.float32(s + a[lo + i])
                i += 1
            return s
        half = n // 2
        half -= half % 8
        return np.float32(rec(lo, half) + rec(lo + half, n - half))

    return np.float32(np.float32(0.0) + rec(0, len(a)))


def mean_f32(a: np.ndarray) -> np.float32:
    """np.mean of a float32 array: f32(f64(0 + P(a)) / len)."""
    return np.float32(np.float64(pairwise_f32(a)) / len(a))


def stream_key(seed: int) -> tuple[int, int]:
    """Philox 128-bit key words used by ``_rng(seed)`` (compressors.py:254-256)."""
    return seed & ((1 << 64) - 1), seed >> 64


def derive_seed(root: int, worker: int = 0, iteration: int = 0, group: int = 0) -> int:
    """compressors.py:247-251 (numpy SeedSequence → two u64 words)."""
    w = np.random.SeedSequence(entropy=(int(root), int(worker), int(iteration), int(group))).generate_state(2, np.uint64)
    return int(w[0]) | (int(w[1]) << 64)


def generator(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=seed))


def philox_uniforms(seed: int, count: int) -> np.ndarray:
    """Uniform #i of the stream = (word_i >> 11) * 2^-53; word_i is 64-bit word
    i%4 of Philox4x64-10(counter = 1 + i//4, key)."""
    return generator(seed).random(count)


# Philox4x64-10 restated — used to pin the GPU stream bit-exactly.
_M0, _M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_W0, _W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_MASK = (1 << 64) - 1


def philox4x64_block(counter: int, key: tuple[int, int]) -> tuple[int, int, int, int]:
    c = [counter & _MASK, (counter >> 64) & _MASK, 0, 0]
    k0, k1 = key
    for rnd in range(10):
        if rnd:
            k0, k1 = (k0 + _W0) & _MASK, (k1 + _W1) & _MASK
        p0, p1 = _M0 * c[0], _M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & _MASK, (p0 >> 64) ^ c[3] ^ k1, p0 & _MASK]
    return tuple(c)


def floyd_choice(seed: int, n: int, k: int) -> np.ndarray:
    """numpy Generator.choice(n, k, replace=False) restated for the Floyd branch
    (k <= n//50 or n <= 10000): bounded draws are 32-bit Lemire with rejection
    over the Philox stream consumed 32 bits at a time (low half first)."""
    key = stream_key(seed)
    words: list[int] = []

    def next32() -> int:
        if not words:
            blk_idx = next32.block
            next32.block += 1
            for w in philox4x64_block(blk_idx, key):
                words.append(w & 0xFFFFFFFF)
                words.append(w >> 32)
        return words.pop(0)

    next32.block = 1

    def bounded(rng: int) -> int:
        if rng == 0:
            return 0
        excl = rng + 1
        m = next32() * excl
        if (m & 0xFFFFFFFF) < excl:
            thr = ((1 << 32) - excl) % excl
            while (m & 0xFFFFFFFF) < thr:
                m = next32() * excl
        return m >> 32

    chosen: set[int] = set()
    for j in range(n - k, n):
        t = bounded(j)
        chosen.add(j if t in chosen else t)
    return np.array(sorted(chosen), dtype=np.uint32)


# ---------------------------------------------------------------- codecs (encode side)

def _bucket_bounds(n: int, b: int):
    return [(lo, min(lo + b, n)) for lo in range(0, n, b)]


def _enc_identity(spec, x, seed):
    return None, x.copy(), None  # compressors.py:265-266


def _enc_fp16(spec, x, seed):
    return None, np.empty(0, np.float32), x.astype(np.float16).view(np.uint8).copy()  # :268-270


def _topk_indices(mag: np.ndarray, k: int) -> np.ndarray:
    # lowest-index tie rule: stable descending order of |x|
    order = np.argsort(-mag.astype(np.float64), kind="stable")[:k]
    return np.sort(order).astype(np.uint32)


def _enc_topk(spec, x, seed):
    k = keep_count(spec.sparsity, len(x))  # :272-276
    idx = _topk_indices(np.abs(x), k)
    return idx, x[idx].copy(), None


def _enc_randk(spec, x, seed):
    n = len(x)  # :278-285
    k = keep_count(spec.sparsity, n)
    idx = np.sort(generator(seed).choice(n, size=k, replace=False)).astype(np.uint32)
    vals = x[idx].copy()
    if spec.unbiased_scaling:
        vals = (vals * np.float32(n / k)).astype(np.float32)
    return idx, vals, None


def _enc_threshold(spec, x, seed):
    idx = np.flatnonzero(np.abs(x) >= spec.threshold).astype(np.uint32)  # :287-289
    return idx, x[idx].copy(), None


def _enc_qsgd(spec, x, seed):
    n = len(x)  # :291-310
    top = spec.levels - 1
    scales = np.empty(n_buckets(n, spec.bucket_size), np.float32)
    codes = np.zeros(n, np.uint32)
    rng = generator(seed)
    for b, (lo, hi) in enumerate(_bucket_bounds(n, spec.bucket_size)):
        seg = x[lo:hi]
        s = np.float32(np.linalg.norm(seg.astype(np.float64)))
        scales[b] = s
        if s == 0:
            continue  # zero bucket: codes 0, no draws
        t = np.minimum(np.abs(seg) / s, 1.0) * top
        fl = np.floor(t)
        up = rng.random(hi - lo) < (t - fl)
        codes[lo:hi] = np.minimum(fl + up, top).astype(np.uint32)
    return None, scales, np.concatenate([sign_bits(x), pack_msb(codes, code_width(spec.levels))])


def _enc_sign_global(spec, x, seed):
    s = np.float32(np.abs(x).mean())  # :312-314
    return None, np.array([s], np.float32), sign_bits(x)


def _enc_efsign(spec, x, seed):
    bounds = _bucket_bounds(len(x), spec.bucket_size)  # :316-321
    scales = np.array([np.abs(x[lo:hi]).mean() for lo, hi in bounds], np.float32)
    return None, scales, sign_bits(x)


def _enc_onebit(spec, x, seed):
    bounds = _bucket_bounds(len(x), spec.bucket_size)  # :323-336
    scales = np.zeros(2 * len(bounds), np.float32)
    for b, (lo, hi) in enumerate(bounds):
        seg = x[lo:hi]
        neg, pos = seg[seg < 0], seg[seg >= 0]
        if neg.size:
            scales[2 * b] = neg.mean()
        if pos.size:
            scales[2 * b + 1] = pos.mean()
    return None, scales, sign_bits(x)


def _enc_terngrad(spec, x, seed):
    n = len(x)  # :338-351
    scales = np.empty(n_buckets(n, spec.bucket_size), np.float32)
    codes = np.ones(n, np.uint32)
    rng = generator(seed)
    for b, (lo, hi) in enumerate(_bucket_bounds(n, spec.bucket_size)):
        seg = x[lo:hi]
        s = np.float32(np.abs(seg).max())
        scales[b] = s
        if s == 0:
            continue  # zero bucket: code 1 (= 0), no draws
        keep = rng.random(hi - lo) < (np.abs(seg) / s)
        codes[lo:hi] = (np.sign(seg) * keep + 1).astype(np.uint32)
    return None, scales, pack_msb(codes, 2)


def _enc_int8(spec, x, seed):
    n = len(x)  # :353-364
    scales = np.empty(n_buckets(n, spec.bucket_size), np.float32)
    q = np.zeros(n, np.int8)
    for b, (lo, hi) in enumerate(_bucket_bounds(n, spec.bucket_size)):
        seg = x[lo:hi]
        s = np.float32(np.abs(seg).max())
        scales[b] = s
        if s != 0:
            q[lo:hi] = np.clip(np.rint(seg / s * 127.0), -127, 127).astype(np.int8)
    return None, scales, q.view(np.uint8).copy()


_ENCODERS = {
    "identity": _enc_identity, "fp16": _enc_fp16, "topk": _enc_topk, "dgc_lite": _enc_topk,
    "randk": _enc_randk, "threshold": _enc_threshold, "qsgd": _enc_qsgd,
    "signsgd": _enc_sign_global, "signum": _enc_sign_global, "efsignsgd": _enc_efsign,
    "onebit": _enc_onebit, "terngrad": _enc_terngrad, "int8": _enc_int8,
}


def compress(spec, x: np.ndarray, seed: int) -> Payload:
    """compressors.py:259-366 (corrected float32 buffer -> payload sections)."""
    flags = 1 if (spec.algorithm == "randk" and spec.unbiased_scaling) else 0
    idx, vals, bits = _ENCODERS[spec.algorithm](spec, x, seed)
    return Payload(spec.algorithm, len(x), idx, vals, bits, flags)


def encode(spec, gradient, state: Optional[State] = None, seed: int = 0):
    """compressors.py:369-417: momentum, error feedback (float64), compress."""
    x = np.asarray(gradient, dtype=np.float32).reshape(-1)
    if x.size < 1:
        raise ValueError("gradient must have at least one element")
    if not np.isfinite(x).all():
        raise ValueError("gradient contains non-finite values")
    ef, beta = ef_on(spec), momentum_of(spec)
    if state is None and (ef or beta is not None):
        state = State(np.zeros(x.size, np.float64), np.zeros(x.size, np.float32) if beta is not None else None)
    if state is not None and len(state.residual) != x.size:
        raise ValueError(f"state length {len(state.residual)} does not match gradient length {x.size}")
    work, mom = x, (None if state is None else state.momentum)
    if beta is not None:
        m_old = state.momentum if state.momentum is not None else np.zeros(x.size, np.float32)
        b32 = np.float32(beta)
        if spec.algorithm == "signum":
            mom = b32 * m_old + (np.float32(1.0) - b32) * x
        else:
            mom = b32 * m_old + x
        work = mom
    if ef:
        corrected = work + state.residual  # float64
        payload = compress(spec, corrected.astype(np.float32), seed)
        return payload, State(corrected - decode(spec, payload), mom)
    payload = compress(spec, work, seed)
    return payload, (None if state is None else State(state.residual, mom))


# ---------------------------------------------------------------- decode / aggregate

def _corrupt(msg: str):
    raise ValueError(f"corrupt payload: {msg}")


def decode(spec, p: Payload) -> np.ndarray:
    """compressors.py:427-516"""
    if p.algorithm != spec.algorithm:
        raise ValueError(f"payload algorithm {p.algorithm!r} does not match spec {spec.algorithm!r}")
    a, n, B = spec.algorithm, p.original_len, spec.bucket_size
    if a in SPARSE:
        if p.indices is None:
            _corrupt("sparsifier payload lacks indices")
        if len(p.indices) != len(p.values):
            _corrupt("index/value length mismatch")
        if len(p.indices):
            if int(p.indices[-1]) >= n:
                _corrupt("index out of range")
            if not np.all(np.diff(p.indices.astype(np.int64)) > 0):
                _corrupt("indices not increasing")
        out = np.zeros(n, np.float32)
        out[p.indices] = p.values
        return out
    if a == "identity":
        if len(p.values) != n:
            _corrupt("value buffer length mismatch")
        return p.values.copy()
    if a == "fp16":
        if p.bits is None or len(p.bits) != 2 * n:
            _corrupt("fp16 buffer length mismatch")
        return p.bits.view(np.float16).astype(np.float32)
    nb = n_buckets(n, B)
    bounds = _bucket_bounds(n, B)
    sb = (n + 7) // 8
    if a == "qsgd":
        w = code_width(spec.levels)
        if p.bits is None:
            _corrupt("missing bit codes")
        if len(p.values) != nb:
            _corrupt("scale count mismatch")
        if len(p.bits) != sb + (n * w + 7) // 8:
            _corrupt("bit buffer length mismatch")
        sg = signs_pm1(p.bits[:sb], n)
        cf = unpack_msb(p.bits[sb:], n, w).astype(np.float32)
        out = np.empty(n, np.float32)
        for b, (lo, hi) in enumerate(bounds):
            out[lo:hi] = sg[lo:hi] * p.values[b] * (cf[lo:hi] / np.float32(spec.levels - 1))
        return out
    if a in ("signsgd", "signum"):
        if len(p.values) != 1:
            _corrupt("expected one global scaler")
        if p.bits is None or len(p.bits) != sb:
            _corrupt("sign buffer mismatch")
        return signs_pm1(p.bits, n) * p.values[0]
    if a == "efsignsgd":
        if len(p.values) != nb:
            _corrupt("scale count mismatch")
        if p.bits is None or len(p.bits) != sb:
            _corrupt("sign buffer mismatch")
        sg = signs_pm1(p.bits, n)
        out = np.empty(n, np.float32)
        for b, (lo, hi) in enumerate(bounds):
            out[lo:hi] = sg[lo:hi] * p.values[b]
        return out
    if a == "onebit":
        if len(p.values) != 2 * nb:
            _corrupt("scaler count mismatch")
        if p.bits is None or len(p.bits) != sb:
            _corrupt("sign buffer mismatch")
        positive = np.unpackbits(p.bits)[:n] == 1
        out = np.empty(n, np.float32)
        for b, (lo, hi) in enumerate(bounds):
            out[lo:hi] = np.where(positive[lo:hi], p.values[2 * b + 1], p.values[2 * b])
        return out
    if a == "terngrad":
        if len(p.values) != nb:
            _corrupt("scale count mismatch")
        if p.bits is None or len(p.bits) != (2 * n + 7) // 8:
            _corrupt("code buffer mismatch")
        t = unpack_msb(p.bits, n, 2).astype(np.float32) - np.float32(1.0)
        out = np.empty(n, np.float32)
        for b, (lo, hi) in enumerate(bounds):
            out[lo:hi] = t[lo:hi] * p.values[b]
        return out
    if a == "int8":
        if len(p.values) != nb:
            _corrupt("scale count mismatch")
        if p.bits is None or len(p.bits) != n:
            _corrupt("int8 buffer mismatch")
        q = p.bits.view(np.int8).astype(np.float32)
        out = np.empty(n, np.float32)
        for b, (lo, hi) in enumerate(bounds):
            out[lo:hi] = q[lo:hi] * (p.values[b] / np.float32(127.0))
        return out
    raise AssertionError(a)


def aggregate(spec, payloads: Sequence[Payload]) -> np.ndarray:
    """Rank-ordered float32 sum of decodes, then / f32(n) — compressors.py:519-532."""
    if not payloads:
        raise ValueError("need at least one payload")
    first = payloads[0]
    for p in payloads[1:]:
        if p.algorithm != first.algorithm:
            raise ValueError(f"mixed algorithms: {first.algorithm!r} vs {p.algorithm!r}")
        if p.original_len != first.original_len:
            raise ValueError(f"mixed lengths: {first.original_len} vs {p.original_len}")
    acc = np.zeros(first.original_len, np.float32)
    for p in payloads:
        acc += decode(spec, p)
    return acc / np.float32(len(payloads))


def payload_bytes(spec, n: int) -> int:
    """Canonical serialized size incl. the 22-byte header — compressors.py:565-596."""
    if n < 1:
        raise ValueError("group_size must be >= 1")
    a = spec.algorithm
    nb, sb = n_buckets(n, spec.bucket_size), (n + 7) // 8
    body = {
        "identity": lambda: 4 * n,
        "fp16": lambda: 2 * n,
        "qsgd": lambda: 4 * nb + sb + (n * code_width(spec.levels) + 7) // 8,
        "signsgd": lambda: 4 + sb,
        "signum": lambda: 4 + sb,
        "efsignsgd": lambda: 4 * nb + sb,
        "onebit": lambda: 8 * nb + sb,
        "terngrad": lambda: 4 * nb + (2 * n + 7) // 8,
        "int8": lambda: 4 * nb + n,
    }
    if a in SPARSE:
        return HEADER + 8 * keep_count(spec.sparsity, n)
    return HEADER + body[a]()


def serialize(p: Payload) -> bytes:
    """Canonical little-endian form (compressors.py:601-620)."""
    ni = 0 if p.indices is None else len(p.indices)
    nb = 0 if p.bits is None else len(p.bits)
    out = [struct.pack("<BBQIII", ALGO_ID[p.algorithm], p.flags, p.original_len, ni, len(p.values), nb)]
    if p.indices is not None:
        out.append(p.indices.astype("<u4").tobytes())
    out.append(p.values.astype("<f4").tobytes())
    if p.bits is not None:
        out.append(p.bits.tobytes())
    return b"".join(out)


# ---------------------------------------------------------------- sync loop (one group, n workers)

def sync_group(spec, grads: Sequence[np.ndarray], states: list, seeds: Sequence[int]):
    """Trainer.step's per-group body (trainer.py:377-389): encode per worker in
    order, then aggregate.  Returns (mean, payloads, new_states)."""
    payloads, new_states = [], []
    for w, g in enumerate(grads):
        p, s = encode(spec, g, states[w], seed=seeds[w])
        payloads.append(p)
        new_states.append(s)
    return aggregate(spec, payloads), payloads, new_states
