"""Bit generators and the bridge between numpy Generators and the device stream.

Mirrors ``sampler.py:131-133 make_rng`` of the reference (numpy
``Generator(Philox(seed))``) and adds the minstd / pcg32 / sfc64 kinds the
north star names.  The device draws the momenta from a stream described by
an ``rsv_prng_state`` (kind, seed words, position); this module converts a
numpy Generator's state into that description and writes the advanced
position back, so ``hmc_update_volatility(h, ..., rng)`` consumes exactly
the raw words numpy's own ``rng.standard_normal(T)`` + ``rng.random()``
would have consumed.

Conventions (also in include/rsvhmc_b200.h):
  * philox: numpy Philox4x64-10, key = SeedSequence(seed).generate_state(2)
  * sfc64 : numpy SFC64, (a, b, c) = SeedSequence(seed).generate_state(3)
  * pcg32 : pcg_basic, (initstate, initseq) = SeedSequence(seed).generate_state(2);
            64-bit word = out0 << 32 | out1
  * minstd: std::minstd_rand, x0 = SeedSequence(seed).generate_state(1) mod (2^31-1);
            64-bit word = x1 << 33 | x2 << 2 | x3 >> 29
  * next_double = (word >> 11) * 2**-53 for all kinds.
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as N

KINDS = tuple(N.KINDS)


def seed_material(kind: str, seed) -> np.ndarray:
    if kind not in N.KINDS:
        raise ValueError(f"unknown bit generator kind {kind!r}; expected one of {KINDS}")
    ss = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
    n = {"philox": 2, "minstd": 1, "pcg32": 2, "sfc64": 3}[kind]
    out = np.zeros(4, dtype=np.uint64)
    out[:n] = ss.generate_state(n, np.uint64)
    return out


class RsvBitGenerator:
    """A numpy-compatible bit generator (duck-typed: ``capsule`` + ``lock``)
    backed by the library's host stream code, so ``numpy.random.Generator``
    can draw from it and the device can continue it."""

    def __init__(self, kind: str = "pcg32", seed=None, state: N.PrngState | None = None):
        self._st = N.PrngState()
        if state is not None:
            ctypes.memmove(ctypes.byref(self._st), ctypes.byref(state), ctypes.sizeof(N.PrngState))
        else:
            mat = np.ascontiguousarray(seed_material(kind, seed))
            N.check(N.lib().rsv_stream_seed(ctypes.byref(self._st), N.KINDS[kind],
                                            mat.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
        self._bg = N.Bitgen()
        N.check(N.lib().rsv_stream_bitgen(ctypes.byref(self._st), ctypes.byref(self._bg)))
        new = ctypes.pythonapi.PyCapsule_New
        new.restype = ctypes.py_object
        new.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
        self.capsule = new(ctypes.addressof(self._bg), b"BitGenerator", None)
        self.lock = threading.Lock()

    @property
    def kind(self) -> str:
        return N.KIND_NAMES[self._st.kind]

    @property
    def prng_state(self) -> N.PrngState:
        st = N.PrngState()
        ctypes.memmove(ctypes.byref(st), ctypes.byref(self._st), ctypes.sizeof(N.PrngState))
        return st

    @prng_state.setter
    def prng_state(self, st: N.PrngState) -> None:
        ctypes.memmove(ctypes.byref(self._st), ctypes.byref(st), ctypes.sizeof(N.PrngState))

    @property
    def state(self) -> dict:
        return {"bit_generator": "Rsv" + self.kind, "s": [int(x) for x in self._st.s], "pos": int(self._st.pos)}

    def random_raw(self, size=None):
        n = 1 if size is None else int(size)
        out = np.fromiter((N.lib().rsv_stream_next_u64(ctypes.byref(self._st)) for _ in range(n)),
                          dtype=np.uint64, count=n)
        return int(out[0]) if size is None else out


def make_rng(seed: int = 0, kind: str = "philox") -> np.random.Generator:
    """sampler.py:131-133 make_rng.  kind='philox' returns exactly the
    reference's ``Generator(Philox(seed))``; 'sfc64' numpy's SFC64; 'minstd'
    and 'pcg32' a Generator over :class:`RsvBitGenerator`."""
    if kind == "philox":
        return np.random.Generator(np.random.Philox(seed))
    if kind == "sfc64":
        return np.random.Generator(np.random.SFC64(seed))
    return np.random.Generator(RsvBitGenerator(kind, seed))


def _bitgen(rng):
    return rng.bit_generator if isinstance(rng, np.random.Generator) else rng


def stream_state(rng) -> N.PrngState:
    """Device stream description of a Generator's (or bit generator's) position."""
    bg = _bitgen(rng)
    st = N.PrngState()
    if isinstance(bg, RsvBitGenerator):
        return bg.prng_state
    if isinstance(bg, np.random.Philox):
        s = bg.state
        ctr = s["state"]["counter"]
        if int(ctr[1]) or int(ctr[2]) or int(ctr[3]):
            raise ValueError("Philox counter beyond 2^64 blocks is not supported")
        c0 = int(ctr[0])
        pos = 0 if c0 == 0 else 4 * (c0 - 1) + int(s["buffer_pos"])
        st.kind = N.KINDS["philox"]
        st.s[0], st.s[1] = int(s["state"]["key"][0]), int(s["state"]["key"][1])
        st.pos = pos
        return st
    if isinstance(bg, np.random.SFC64):
        s = bg.state["state"]["state"]
        st.kind = N.KINDS["sfc64"]
        for i in range(4):
            st.s[i] = int(s[i])
        st.pos = 0
        return st
    raise TypeError(f"unsupported bit generator {type(bg).__name__}: use Philox, SFC64 or make_rng(kind=...)")


def store_stream_state(rng, st: N.PrngState) -> None:
    """Write an advanced device stream position back into the Generator."""
    bg = _bitgen(rng)
    if isinstance(bg, RsvBitGenerator):
        bg.prng_state = st
        return
    if isinstance(bg, np.random.Philox):
        s = bg.state
        pos = int(st.pos)
        k0, k1 = int(st.s[0]), int(st.s[1])
        if pos % 4 == 0:
            c0, bpos, buf = pos // 4, 4, s["buffer"]
        else:
            c0, bpos = pos // 4 + 1, pos % 4
            out = (ctypes.c_uint64 * 4)()
            N.lib().rsv_philox_block(c0 - 1, k0, k1, out)
            buf = np.array(list(out), dtype=np.uint64)
        s["state"]["counter"] = np.array([c0, 0, 0, 0], dtype=np.uint64)
        s["buffer"] = np.asarray(buf, dtype=np.uint64)
        s["buffer_pos"] = bpos
        bg.state = s
        return
    if isinstance(bg, np.random.SFC64):
        s = bg.state
        s["state"]["state"] = np.array([int(st.s[i]) for i in range(4)], dtype=np.uint64)
        bg.state = s
        return
    raise TypeError(f"unsupported bit generator {type(bg).__name__}")
