"""Structural hash, hash buckets, hierarchical-sampling representatives and
the beam cut (restates reference `loopnest.py:87-165`, `sampling.py:45-59`,
`search.py:63-201`), plus a from-scratch NumPy SeedSequence / PCG64 /
`permutation` / `gumbel` replica that pins the CUDA RNG (search.py:154,
189-190 call `np.random.default_rng((phase_seed, h))`)."""

from __future__ import annotations

import hashlib
import math

import numpy as np


def kernel_of(dmap, func):
    """loopnest.py:87-94."""
    d = dmap.get(func)
    while d is not None and d.kind in ("fuse_at_block", "fuse_at_thread"):
        func = d.consumer
        d = dmap.get(func)
    return None if d is None or d.kind == "inline" else func


def canonical_bytes(decisions, depth: int) -> bytes:
    """Bytes fed to blake2b (loopnest.py:131-165): repr of the canonical tuple."""
    if depth < 0:
        raise ValueError("depth must be >= 0")
    depth = min(depth, 3)
    dmap = dict(decisions)
    if depth == 0:
        canon = ("kernels", tuple(sorted(f for f, d in decisions if d.kind == "compute_root")))
    else:
        ents = []
        for f in sorted(dmap):
            d = dmap[f]
            e = (f, d.kind, kernel_of(dmap, f))
            if depth >= 2:
                e += (d.consumer,)
            if depth >= 3:
                e += (d.serial is not None, d.thread is not None)
            ents.append(e)
        canon = (depth, tuple(ents))
    return repr(canon).encode()


def structural_hash(decisions, depth: int) -> int:
    return int.from_bytes(hashlib.blake2b(canonical_bytes(decisions, depth),
                                          digest_size=8).digest(), "little")


def quota(b: int) -> int:
    """sampling.py:45-48."""
    if b < 1:
        raise ValueError("empty bucket")
    return max(1, int(math.floor(math.log2(b))))


def buckets(hashes):
    """hash -> member indices in insertion order (sampling.py:51-59)."""
    out = {}
    for i, h in enumerate(hashes):
        out.setdefault(int(h), []).append(i)
    return out


def select_reps(hashes, valid, phase_seed):
    """Indices of representatives in (hash asc, permutation position) order
    and indices of drawn rejects (search.py:127-165)."""
    reps, rejects = [], []
    bs = buckets(hashes)
    for h in sorted(bs):
        members = bs[h]
        q = quota(len(members))
        taken = 0
        for i in np.random.default_rng((phase_seed, h)).permutation(len(members)):
            m = members[int(i)]
            if valid[m]:
                reps.append(m)
                taken += 1
                if taken == q:
                    break
            else:
                rejects.append(m)
    return reps, rejects


def cut(reps, costs, pass_hashes, flagged, penalty, beam_size,
        temperature=0.0, phase_seed=0):
    """Beam cut over costed representatives (search.py:168-201, 76-87).

    reps        — candidate indices in representative order
    costs       — unpenalized totals per rep
    pass_hashes — hash at depth pass_index per rep
    flagged     — set of flagged hashes at depth pass_index
    Returns (kept rep positions, bottom-half rep positions for memo update).
    """
    keys = [c * penalty if h in flagged else c for c, h in zip(costs, pass_hashes)]
    if temperature > 0:
        noise = np.random.default_rng((phase_seed, 0x657870)).gumbel(size=len(keys)) * temperature
        keys = [math.log(max(k, 1e-300)) + n for k, n in zip(keys, noise)]
    order = sorted(range(len(keys)), key=lambda i: keys[i])
    bottom = []
    if len(costs) > 1:
        by_cost = sorted(range(len(costs)), key=lambda i: costs[i])
        bottom = by_cost[len(by_cost) // 2:]
    return order[:beam_size], bottom


# ---------------------------------------------------------------------------
# From-scratch replica of NumPy's SeedSequence -> PCG64 -> permutation/gumbel
# ---------------------------------------------------------------------------

_M32 = 0xFFFFFFFF
_INIT_A, _MULT_A = 0x43B0D7E5, 0x931E8875
_INIT_B, _MULT_B = 0x8B51F9DD, 0x58F38DED
_MIX_L, _MIX_R = 0xCA01F9DD, 0x4973F715
_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
_M128 = (1 << 128) - 1


def _words(x: int):
    if x == 0:
        return [0]
    out = []
    while x:
        out.append(x & _M32)
        x >>= 32
    return out


def seed_state(entropy, n_words64=4):
    """SeedSequence(entropy).generate_state(n, uint64)."""
    ent = []
    for e in entropy:
        ent += _words(int(e))
    pool = [0] * 4
    hc = _INIT_A

    def hashmix(v):
        nonlocal hc
        v = (v ^ hc) & _M32
        hc = (hc * _MULT_A) & _M32
        v = (v * hc) & _M32
        return (v ^ (v >> 16)) & _M32

    def mix(x, y):
        r = ((_MIX_L * x) & _M32) - ((_MIX_R * y) & _M32)
        r &= _M32
        return (r ^ (r >> 16)) & _M32

    for i in range(4):
        pool[i] = hashmix(ent[i] if i < len(ent) else 0)
    for src in range(4):
        for dst in range(4):
            if src != dst:
                pool[dst] = mix(pool[dst], hashmix(pool[src]))
    for src in range(4, len(ent)):
        for dst in range(4):
            pool[dst] = mix(pool[dst], hashmix(ent[src]))
    out32 = []
    hc = _INIT_B
    for i in range(2 * n_words64):
        v = pool[i % 4]
        v = (v ^ hc) & _M32
        hc = (hc * _MULT_B) & _M32
        v = (v * hc) & _M32
        out32.append((v ^ (v >> 16)) & _M32)
    return [out32[2 * i] | (out32[2 * i + 1] << 32) for i in range(n_words64)]


class PCG64:
    def __init__(self, entropy):
        s = seed_state(entropy)
        seed = (s[0] << 64) | s[1]
        inc = (s[2] << 64) | s[3]
        self.inc = ((inc << 1) | 1) & _M128
        self.state = 0
        self._step()
        self.state = (self.state + seed) & _M128
        self._step()
        self.buf = None

    def _step(self):
        self.state = (self.state * _PCG_MULT + self.inc) & _M128

    def next64(self) -> int:
        self._step()
        s = self.state
        x = ((s >> 64) ^ s) & 0xFFFFFFFFFFFFFFFF
        rot = s >> 122
        return ((x >> rot) | (x << ((64 - rot) & 63))) & 0xFFFFFFFFFFFFFFFF

    def next32(self) -> int:
        if self.buf is not None:
            v, self.buf = self.buf, None
            return v
        v = self.next64()
        self.buf = v >> 32
        return v & _M32

    def interval(self, mx: int) -> int:
        if mx == 0:
            return 0
        mask = mx
        for sh in (1, 2, 4, 8, 16, 32):
            mask |= mask >> sh
        if mx <= _M32:
            while True:
                v = self.next32() & mask
                if v <= mx:
                    return v
        while True:
            v = self.next64() & mask
            if v <= mx:
                return v

    def permutation(self, n: int):
        a = list(range(n))
        for i in range(n - 1, 0, -1):
            j = self.interval(i)
            a[i], a[j] = a[j], a[i]
        return a

    def integers(self, n: int) -> int:
        """Generator.integers(n) for 1 <= n < 2**32: Lemire's bounded
        rejection on next_uint32 (numpy distributions.c
        buffered_bounded_lemire_uint32); no draw when n == 1."""
        rng = n - 1
        if rng == 0:
            return 0
        m = self.next32() * n
        lo = m & 0xFFFFFFFF
        if lo < n:
            th = (0xFFFFFFFF - rng) % n
            while lo < th:
                m = self.next32() * n
                lo = m & 0xFFFFFFFF
        return m >> 32

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def gumbel(self) -> float:
        while True:
            u = 1.0 - self.next_double()
            if u < 1.0:
                return -math.log(-math.log(u))
