"""numpy SeedSequence key derivation for entropy words wider than 64 bits
(host arithmetic only; the common case goes through mc_derive_seed in C)."""

from __future__ import annotations

M32 = 0xFFFFFFFF


def _words(v: int) -> list[int]:
    if v < 0:
        raise ValueError("expected non-negative integer entropy")
    if v == 0:
        return [0]
    out = []
    while v:
        out.append(v & M32)
        v >>= 32
    return out


def seed_sequence_key(entropy: list[int]) -> tuple[int, int]:
    ent = [w for v in entropy for w in _words(int(v))]
    hc = 0x43B0D7E5

    def hashmix(v):
        nonlocal hc
        v ^= hc
        hc = (hc * 0x931E8875) & M32
        v = (v * hc) & M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (0xCA01F9DD * x - 0x4973F715 * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    hb = 0x8B51F9DD
    st = []
    for i in range(4):
        v = pool[i % 4] ^ hb
        hb = (hb * 0x58F38DED) & M32
        v = (v * hb) & M32
        st.append(v ^ (v >> 16))
    return st[0] | (st[1] << 32), st[2] | (st[3] << 32)
