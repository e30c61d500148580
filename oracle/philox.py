"""Pure-Python restatement of numpy's SeedSequence + Philox4x64-10 streams
as the reference's tuple-keyed RNG uses them (envs/rng.py:26-29,
render/augment.py:51-52) -- TEST INFRASTRUCTURE ONLY.

numpy (>= 1.17, pinned here at 2.3) is the third-party dependency whose
published algorithm the device implementation in csrc/augment.cu restates:
SeedSequence entropy mixing (pool of 4 uint32, hashmix / mix constants),
generate_state(2, uint64) as the Philox key, counter pre-incremented before
each 4-word block, next_double = (u64 >> 11) * 2^-53, uniform = low + range *
next_double, and Generator.permutation via Fisher-Yates with masked
rejection sampling on buffered 32-bit draws.  tests/test_augment.py pins
this restatement against numpy itself.
"""
from __future__ import annotations

M32 = 0xFFFFFFFF
M64 = 0xFFFFFFFFFFFFFFFF
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715


def entropy_words(key):
    """Each int -> little-endian 32-bit words (at least one), concatenated."""
    out = []
    for k in key:
        k = int(k)
        if k < 0:
            raise ValueError("negative seed")
        if k == 0:
            out.append(0)
        while k > 0:
            out.append(k & M32)
            k >>= 32
    return out


def seed_pool(key, pool_size=4):
    h = INIT_A

    def hashmix(v):
        nonlocal h
        v ^= h
        h = (h * MULT_A) & M32
        v = (v * h) & M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (MIX_L * x - MIX_R * y) & M32
        return r ^ (r >> 16)

    ent = entropy_words(key)
    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(pool_size)]
    for s in range(pool_size):
        for d in range(pool_size):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(pool_size, len(ent)):
        for d in range(pool_size):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    return pool


def philox_key(key):
    pool = seed_pool(key)
    h = INIT_B
    words = []
    for i in range(4):
        v = pool[i % 4] ^ h
        h = (h * MULT_B) & M32
        v = (v * h) & M32
        words.append(v ^ (v >> 16))
    return (words[0] | (words[1] << 32), words[2] | (words[3] << 32))


def _mulhilo(a, b):
    p = a * b
    return (p >> 64) & M64, p & M64


def philox4x64_10(ctr, key):
    c = list(ctr)
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B97F4A7C15) & M64
            k1 = (k1 + 0xBB67AE8584CAA73B) & M64
        hi0, lo0 = _mulhilo(0xD2E7470EE14C6C93, c[0])
        hi1, lo1 = _mulhilo(0xCA5A826395121157, c[2])
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return c


class Stream:
    """np.random.Generator(np.random.Philox(np.random.SeedSequence(key)))."""

    def __init__(self, key):
        self.key = philox_key(key)
        self.ctr = [0, 0, 0, 0]
        self.buf, self.pos = [0, 0, 0, 0], 4
        self.has32, self.u32 = False, 0

    def next64(self):
        if self.pos < 4:
            v = self.buf[self.pos]
            self.pos += 1
            return v
        for i in range(4):
            self.ctr[i] = (self.ctr[i] + 1) & M64
            if self.ctr[i]:
                break
        self.buf = philox4x64_10(self.ctr, self.key)
        self.pos = 1
        return self.buf[0]

    def next32(self):
        if self.has32:
            self.has32 = False
            return self.u32
        v = self.next64()
        self.has32, self.u32 = True, v >> 32
        return v & M32

    def uniform(self, low, high):
        return low + (high - low) * ((self.next64() >> 11) * (1.0 / 9007199254740992.0))

    def interval(self, mx):
        if mx == 0:
            return 0
        mask = mx
        for s in (1, 2, 4, 8, 16, 32):
            mask |= mask >> s
        while True:
            v = (self.next32() if mx <= M32 else self.next64()) & mask
            if v <= mx:
                return v

    def permutation(self, n):
        a = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.interval(i)
            a[i], a[j] = a[j], a[i]
        return a
