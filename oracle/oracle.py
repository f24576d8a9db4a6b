"""ctypes wrapper of the CPU oracle (``oracle/liboracle.so``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline leg and ``--impl reference``).  The product
package ``paper_1603_08114_b200`` never imports this module.

Each wrapper names the reference function it restates (paths relative to
/root/reference).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

KINDS = {"philox": 0, "minstd": 1, "pcg32": 2, "sfc64": 3}


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "rsv_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class _Stream(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("s", ctypes.c_uint64 * 4), ("pos", ctypes.c_uint64),
                ("cache_pos", ctypes.c_uint64), ("cache_state", ctypes.c_uint64),
                ("cache_ok", ctypes.c_int32), ("pad2", ctypes.c_int32)]


class _Bitgen(ctypes.Structure):
    _fields_ = [("state", ctypes.c_void_p), ("next_uint64", ctypes.c_void_p),
                ("next_uint32", ctypes.c_void_p), ("next_double", ctypes.c_void_p),
                ("next_raw", ctypes.c_void_p)]


class _Params(ctypes.Structure):
    _fields_ = [("phi", ctypes.c_double), ("mu", ctypes.c_double), ("xi", ctypes.c_double),
                ("sigma_eta_sq", ctypes.c_double), ("sigma_u_sq", ctypes.c_double)]


_lib = None
_D = ctypes.POINTER(ctypes.c_double)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        S = ctypes.POINTER(_Stream)
        P = ctypes.POINTER(_Params)
        i64 = ctypes.c_int64
        L.orc_stream_init.argtypes = [S, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
        L.orc_next_u64.argtypes = [S]; L.orc_next_u64.restype = ctypes.c_uint64
        L.orc_next_double.argtypes = [S]; L.orc_next_double.restype = ctypes.c_double
        L.orc_fill_u64.argtypes = [S, ctypes.POINTER(ctypes.c_uint64), i64]
        L.orc_fill_normal.argtypes = [S, _D, i64]
        L.orc_standard_normal.argtypes = [S]; L.orc_standard_normal.restype = ctypes.c_double
        L.orc_bitgen_bind.argtypes = [ctypes.POINTER(_Bitgen), S]
        L.orc_log1p.argtypes = [ctypes.c_double]; L.orc_log1p.restype = ctypes.c_double
        L.orc_log_posterior.argtypes = [_D, P, _D, _D, i64]; L.orc_log_posterior.restype = ctypes.c_double
        L.orc_hamiltonian.argtypes = [_D, _D, P, _D, _D, i64]; L.orc_hamiltonian.restype = ctypes.c_double
        L.orc_gradient.argtypes = [_D, P, _D, _D, _D, i64]; L.orc_gradient.restype = ctypes.c_int
        L.orc_elementary_step.argtypes = [_D, _D, P, _D, _D, i64, ctypes.c_double, ctypes.c_int]
        L.orc_elementary_step.restype = ctypes.c_int
        L.orc_integrate.argtypes = [_D, _D, P, _D, _D, i64, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_integrate.restype = ctypes.c_int
        L.orc_hmc_update.argtypes = [_D, P, _D, _D, i64, ctypes.c_double, ctypes.c_int, S, _D, _D, ctypes.c_int,
                                     ctypes.c_int]
        L.orc_hmc_update.restype = ctypes.c_int
        L.orc_suff_stats.argtypes = [_D, _D, i64, ctypes.c_double, ctypes.c_double, _D]
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_pool_shutdown.argtypes = []
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def seed_material(kind: str, seed) -> np.ndarray:
    """Raw seed words from numpy.SeedSequence (numpy's own convention for
    Philox/SFC64; the same convention is adopted for minstd and pcg32)."""
    ss = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
    n = {"philox": 2, "minstd": 1, "pcg32": 2, "sfc64": 3}[kind]
    out = np.zeros(4, dtype=np.uint64)
    out[:n] = ss.generate_state(n, np.uint64)
    return out


class Stream:
    """A positioned raw-word stream (see orc_stream in rsv_oracle.c)."""

    def __init__(self, kind: str = "philox", seed=0, material=None):
        self.kind = kind
        self._st = _Stream()
        mat = seed_material(kind, seed) if material is None else np.asarray(material, dtype=np.uint64)
        mat = np.ascontiguousarray(mat)
        lib().orc_stream_init(ctypes.byref(self._st), KINDS[kind],
                              mat.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        self._bg = None

    @property
    def pos(self) -> int:
        return int(self._st.pos)

    def state_words(self):
        return [int(x) for x in self._st.s], int(self._st.pos)

    def raw(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        lib().orc_fill_u64(ctypes.byref(self._st), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), n)
        return out

    def normals(self, n: int) -> np.ndarray:
        """numpy Generator.standard_normal(n) restated (sampler.py:141)."""
        out = np.empty(n, dtype=np.float64)
        lib().orc_fill_normal(ctypes.byref(self._st), _dp(out), n)
        return out

    def next_double(self) -> float:
        return float(lib().orc_next_double(ctypes.byref(self._st)))

    # duck-typed numpy BitGenerator: numpy.random.Generator(stream) works
    @property
    def capsule(self):
        if self._bg is None:
            self._bg = _Bitgen()
            lib().orc_bitgen_bind(ctypes.byref(self._bg), ctypes.byref(self._st))
            new = ctypes.pythonapi.PyCapsule_New
            new.restype = ctypes.py_object
            new.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
            self._capsule = new(ctypes.addressof(self._bg), b"BitGenerator", None)
            self.lock = threading.Lock()
        return self._capsule

    def generator(self) -> np.random.Generator:
        _ = self.capsule
        return np.random.Generator(self)


def _params(p):
    return _Params(float(p.phi), float(p.mu), float(p.xi), float(p.sigma_eta_sq), float(p.sigma_u_sq))


def log1p(x: float) -> float:
    return float(lib().orc_log1p(float(x)))


def log_posterior(h, params, y, lrv) -> float:
    """model.py:134-163."""
    h = np.ascontiguousarray(h, dtype=np.float64)
    return float(lib().orc_log_posterior(_dp(h), ctypes.byref(_params(params)), _dp(y), _dp(lrv), h.size))


def hamiltonian(h, p, params, y, lrv) -> float:
    """model.py:178-182."""
    h = np.ascontiguousarray(h, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    return float(lib().orc_hamiltonian(_dp(h), _dp(p), ctypes.byref(_params(params)), _dp(y), _dp(lrv), h.size))


def gradient(h, params, y, lrv):
    """_kernels.py:57-67 gradient_fill.  Returns (g, diverged)."""
    h = np.ascontiguousarray(h, dtype=np.float64)
    out = np.empty_like(h)
    f = lib().orc_gradient(_dp(h), ctypes.byref(_params(params)), _dp(y), _dp(lrv), _dp(out), h.size)
    return out, bool(f)


def elementary_step(h, p, params, y, lrv, dt, nthreads=1):
    """integrator.py:139-146, in place on copies; returns (h, p, diverged)."""
    h = np.array(h, dtype=np.float64)
    p = np.array(p, dtype=np.float64)
    f = lib().orc_elementary_step(_dp(h), _dp(p), ctypes.byref(_params(params)), _dp(y), _dp(lrv),
                                  h.size, float(dt), int(nthreads))
    return h, p, bool(f)


def integrate(h, p, params, y, lrv, dt, n_steps, fuse=False, nthreads=1):
    """integrator.py:149-179 on copies; returns (h, p, diverged)."""
    h = np.array(h, dtype=np.float64)
    p = np.array(p, dtype=np.float64)
    f = lib().orc_integrate(_dp(h), _dp(p), ctypes.byref(_params(params)), _dp(y), _dp(lrv), h.size,
                            float(dt), int(n_steps), int(bool(fuse)), int(nthreads))
    return h, p, bool(f)


def hmc_update(h, params, y, lrv, dt, n_steps, stream: Stream, nthreads=1, fuse=False):
    """sampler.py:144-167 (fuse: integrate_trajectory(fuse_half_steps=True),
    integrator.py:149).  Returns (h_new, accept, delta_h); advances stream."""
    h = np.array(h, dtype=np.float64)
    work = np.empty(2 * h.size, dtype=np.float64)
    dh = ctypes.c_double(0.0)
    acc = lib().orc_hmc_update(_dp(h), ctypes.byref(_params(params)), _dp(y), _dp(lrv), h.size, float(dt),
                               int(n_steps), ctypes.byref(stream._st), ctypes.byref(dh), _dp(work), int(nthreads),
                               int(bool(fuse)))
    return h, bool(acc), float(dh.value)


def suff_stats(h, lrv, c_mu, c_xi) -> np.ndarray:
    h = np.ascontiguousarray(h, dtype=np.float64)
    out = np.empty(7, dtype=np.float64)
    lib().orc_suff_stats(_dp(h), _dp(lrv), h.size, float(c_mu), float(c_xi), _dp(out))
    return out


def max_threads() -> int:
    return int(lib().orc_max_threads())
