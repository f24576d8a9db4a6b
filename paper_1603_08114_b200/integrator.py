"""Leapfrog integrator on the B200 (mirror of the reference's ``integrator.py``).

The reference advances the phase state with three barrier-separated range
kernels per step (``integrator.py:111-146``) run by a pluggable backend
(``integrator.py:50-105``).  Here:

* :class:`CudaBackend` is a drop-in ``backend=`` object.  Its ``run(kernel,
  n, args)`` implements the reference's backend protocol for the
  reference's own kernels (``_kernels.position_update`` /
  ``momentum_update`` / ``gradient_fill``) on the GPU, so the unmodified
  reference can run on it; the package's functions below use its fused
  paths instead.
* :func:`elementary_step` runs K1->K2->K3 as one streamed kernel.
* :func:`integrate_trajectory` runs the whole trajectory as one launch of the
  tiled, register-resident trajectory kernel (csrc/leapfrog.cu).
"""
from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .model import Dataset, Params, PhaseState, _f64, is_frozen, scalar_pack

DEFAULT_CHUNK = 512
DH_DIVERGENCE_THRESHOLD = 1000.0  # integrator.py:29; applied on device


@dataclass(frozen=True)
class MDConfig:
    """Step size and step count of one trajectory (integrator.py:32-47)."""

    step_size: float
    n_steps: int

    def __post_init__(self):
        if not self.step_size > 0.0:
            raise ValueError(f"step_size must be positive, got {self.step_size}")
        if self.n_steps < 1:
            raise ValueError(f"n_steps must be >= 1, got {self.n_steps}")

    @property
    def trajectory_length(self) -> float:
        return self.n_steps * self.step_size


class _Lease:
    """Owner object of one hand-out of a pooled page-locked buffer.  A
    read-only lease exposes no writable buffer, so neither the array over it
    nor any view of it can be made writable again."""

    __slots__ = ("__array_interface__", "buf", "__weakref__")

    def __init__(self, buf: np.ndarray, readonly: bool = False):
        self.buf = buf
        ai = dict(buf.__array_interface__)
        ai["data"] = (ai["data"][0], bool(readonly))
        self.__array_interface__ = ai


class DeviceChain:
    """One ``rsv_ctx``: a length-T chain resident on one GPU."""

    def __init__(self, T: int, device: int = 0):
        self.T = int(T)
        self.device = device
        self._lib = N.lib()
        h = ctypes.c_void_p()
        N.check(self._lib.rsv_create(ctypes.byref(h), int(device), self.T))
        self.ctx = h.value
        self._data_key = None
        self._params_key = None
        self._resident = None  # weakref to the lease of the returned path the device holds

    # -- lifecycle --
    def close(self):
        if self.ctx:
            self._lib.rsv_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, code, keeps_path: bool = False):
        """Check a C-ABI return code.  Every call that may move the device's
        path (or its cur index) drops the resident-path link of
        hmc_update_host; calls that leave it alone say keeps_path."""
        if not keeps_path:
            self._resident = None
        N.check(code, self.ctx)

    # -- state --
    def set_data(self, data: Dataset, force: bool = False):
        """Upload y and ln RV.  The upload is reused only while both arrays
        are read-only (``Dataset`` freezes its arrays), so no in-place edit
        can leave the device on stale data; writable arrays are uploaded on
        every call."""
        key = (id(data), id(data.returns), id(data.log_rv), data.returns.ctypes.data, data.log_rv.ctypes.data)
        if not (is_frozen(data.returns) and is_frozen(data.log_rv)):
            key = None
        if force or key is None or key != self._data_key:
            if data.length != self.T:
                raise ValueError(f"dataset length {data.length} does not match chain length {self.T}")
            y = np.ascontiguousarray(data.returns, dtype=np.float64)
            lrv = np.ascontiguousarray(data.log_rv, dtype=np.float64)
            self._ck(self._lib.rsv_set_data(self.ctx, y.ctypes.data, lrv.ctypes.data, 0), keeps_path=True)
            self._data_key = key
            self._data_ref = data  # keep ids alive

    def set_params(self, params: Params):
        key = (params.phi, params.mu, params.xi, params.sigma_eta_sq, params.sigma_u_sq)
        if key != self._params_key:
            self._ck(self._lib.rsv_set_params(self.ctx, ctypes.byref(N.to_params(params))), keeps_path=True)
            self._params_key = key

    def set_latent(self, h: np.ndarray):
        h = _f64(h)
        if h.shape != (self.T,):
            raise ValueError(f"latent path length {h.shape[0]} does not match chain length {self.T}")
        self._ck(self._lib.rsv_set_latent(self.ctx, h.ctypes.data, 0))

    def _pinned_out(self, readonly: bool = False) -> np.ndarray:
        """A page-locked host array for a returned path.  Each hand-out is an
        array over a fresh ``_Lease`` of a pool buffer, tracked by a weak
        reference: the lease is the memory owner numpy records for the
        returned array and for every view derived from it, so a buffer is
        reused only once all of them are gone -- a returned path is never
        overwritten."""
        pool = self.__dict__.setdefault("_pool", [])  # [buffer, weakref to the view handed out]
        if not pool:  # allocate the pool at once (page-locking is slow)
            try:
                import torch
                ts = [torch.empty(self.T, dtype=torch.float64, pin_memory=True) for _ in range(3)]
                self.__dict__["_pool_t"] = ts
                pool.extend([t.numpy(), None] for t in ts)
            except Exception:
                pass
        for ent in pool:
            if ent[1] is None or ent[1]() is None:
                lease = _Lease(ent[0], readonly)
                ent[1] = weakref.ref(lease)
                return np.asarray(lease)
        out = np.empty(self.T)
        if readonly:
            out.flags.writeable = False
        return out

    def get_latent(self, out: np.ndarray | None = None) -> np.ndarray:
        out = self._pinned_out() if out is None else out
        self._ck(self._lib.rsv_get_latent(self.ctx, N.ptr(out), 0), keeps_path=True)
        return out

    def set_stream(self, st: N.PrngState):
        self._ck(self._lib.rsv_set_prng_state(self.ctx, ctypes.byref(st)), keeps_path=True)

    def get_stream(self) -> N.PrngState:
        st = N.PrngState()
        self._ck(self._lib.rsv_get_prng_state(self.ctx, ctypes.byref(st)), keeps_path=True)
        return st

    # -- hot path --
    def hmc_update(self, step_size: float, n_steps: int, fuse: bool = False, stats: bool = True) -> N.Result:
        """One proposal; with stats=False the theta statistics of the kept
        path are not evaluated (the reference's hmc_update_volatility)."""
        if not stats:
            return self.hmc_update_many(step_size, n_steps, 1, fuse)[0]
        r = N.Result()
        self._ck(self._lib.rsv_hmc_update(self.ctx, float(step_size), int(n_steps), int(bool(fuse)),
                                          ctypes.byref(r)))
        return r

    def run_chain_device(self, step_size: float, n_steps: int, fuse: bool, prior, n_burnin: int, n_samples: int,
                         thin: int):
        """rsv_run_chain: every sweep on the device.  Returns (iters, params
        [n x 5], accept, delta_h); raises NativeError subclass StormError on
        a divergence storm (with .sweep)."""
        pr = N.Prior(*(float(getattr(prior, f)) for f, _ in N.Prior._fields_))
        iters = np.empty(n_samples, dtype=np.int64)
        par = np.empty((n_samples, 5))
        acc = np.empty(n_samples, dtype=np.int32)
        dh = np.empty(n_samples)
        storm = ctypes.c_int64(-1)
        code = self._lib.rsv_run_chain(self.ctx, float(step_size), int(n_steps), int(bool(fuse)), ctypes.byref(pr),
                                       int(n_burnin), int(n_samples), int(thin), iters.ctypes.data, par.ctypes.data,
                                       acc.ctypes.data, dh.ctypes.data, ctypes.byref(storm))
        self._params_key = None  # the device holds the final parameters now
        try:
            self._ck(code)
        except N.StormError as e:
            e.sweep = int(storm.value)
            raise
        return iters, par, acc.astype(bool), dh

    def set_blocked_streams(self, seed: int | None, block_len: int = 4096):
        """Config-5 momenta layout: sites [j*B, (j+1)*B) draw from
        SFC64(SeedSequence([seed, j])); seed=None restores one stream."""
        if seed is None:
            self._ck(self._lib.rsv_set_blocked_streams(self.ctx, 0, 0, None))
            return
        if self.T % block_len:
            raise ValueError(f"block length {block_len} does not divide T={self.T}")
        from .ensemble import sfc64_states
        st = sfc64_states(seed, self.T // block_len)
        self._ck(self._lib.rsv_set_blocked_streams(self.ctx, int(block_len), self.T // block_len, st.ctypes.data))
        self._block_len = block_len

    def blocked_streams(self) -> np.ndarray:
        n = self.T // max(1, getattr(self, "_block_len", 1))
        out = np.empty((n, 4), dtype=np.uint64)
        self._ck(self._lib.rsv_get_blocked_streams(self.ctx, out.ctypes.data))
        return out

    def get_params(self) -> Params:
        p = N.Params()
        self._ck(self._lib.rsv_get_params(self.ctx, ctypes.byref(p)), keeps_path=True)
        return N.to_params(p)

    def _holds(self, h) -> bool:
        """h is the read-only path this chain returned last and the device
        still holds it (no call since has moved the device's path)."""
        lease = self._resident() if self._resident is not None else None
        return (lease is not None and isinstance(h, np.ndarray) and h.base is lease and not h.flags.writeable
                and h.dtype == np.float64 and h.shape == (self.T,) and h.strides == (8,)
                and h.ctypes.data == lease.__array_interface__["data"][0])

    def hmc_update_host(self, h: np.ndarray, st: N.PrngState, step_size: float, n_steps: int,
                        fuse: bool = False):
        """One proposal from a host path (rsv_hmc_update_host): returns
        (result, path_out) where path_out is a read-only page-locked array
        holding the proposal when accepted (None otherwise); st is advanced in
        place.  A path this chain returned (read-only, so unchanged since) and
        still holds on the device is not sent again: the proposal runs from
        the device's copy and only the stream state crosses the link."""
        resident = self._holds(h)
        if not resident:
            h = _f64(h)
            if h.shape != (self.T,):
                raise ValueError(f"latent path length {h.shape[0]} does not match chain length {self.T}")
        out = self._pinned_out(readonly=True)
        r = N.Result()
        code = self._lib.rsv_hmc_update_host(self.ctx, None if resident else h.ctypes.data, out.ctypes.data,
                                             ctypes.byref(st), float(step_size), int(n_steps), int(bool(fuse)),
                                             ctypes.byref(r))
        self._ck(code, keeps_path=resident and code == 0)
        self._last_resident = resident
        if r.accept and isinstance(out.base, _Lease):
            self._resident = weakref.ref(out.base)  # the device's path is now the returned one
        return r, (out if r.accept else None)

    @property
    def last_update_resident(self) -> bool:
        """The last hmc_update_host proposed from the device's resident path."""
        return bool(getattr(self, "_last_resident", False))

    @property
    def last_update_zero_copy(self) -> bool:
        """The last hmc_update_host read the (page-locked) path in place."""
        return bool(self._lib.rsv_last_update_zero_copy(self.ctx))

    def hmc_update_many(self, step_size: float, n_steps: int, n: int, fuse: bool = False,
                        results: bool = True):
        out = (N.Result * n)() if results else None
        self._ck(self._lib.rsv_hmc_update_many(self.ctx, float(step_size), int(n_steps), int(bool(fuse)), int(n),
                                               out))
        return out

    def integrate(self, h, p, step_size, n_steps, fuse=False):
        h = _f64(h)
        p = _f64(p, "p")
        ho, po = np.empty_like(h), np.empty_like(p)
        div = ctypes.c_int32(0)
        self._ck(self._lib.rsv_integrate(self.ctx, h.ctypes.data, p.ctypes.data, float(step_size), int(n_steps),
                                         int(bool(fuse)), ho.ctypes.data, po.ctypes.data, ctypes.byref(div), 0))
        return ho, po, bool(div.value)

    def elementary_step_inplace(self, h: np.ndarray, p: np.ndarray, step_size: float) -> bool:
        div = ctypes.c_int32(0)
        self._ck(self._lib.rsv_elementary_step(self.ctx, N.ptr(h), N.ptr(p), float(step_size),
                                               ctypes.byref(div), 0))
        return bool(div.value)

    def refresh_momenta(self) -> np.ndarray:
        out = np.empty(self.T)
        self._ck(self._lib.rsv_refresh_momenta(self.ctx, out.ctypes.data, 0))
        return out

    def hamiltonian(self, h, p) -> float:
        v = ctypes.c_double()
        self._ck(self._lib.rsv_hamiltonian(self.ctx, N.ptr(h), N.ptr(p), ctypes.byref(v), 0))
        return float(v.value)

    def log_posterior(self, h) -> float:
        v = ctypes.c_double()
        self._ck(self._lib.rsv_log_posterior(self.ctx, N.ptr(h), ctypes.byref(v), 0))
        return float(v.value)

    def suff_stats(self, c_mu: float, c_xi: float) -> np.ndarray:
        out = np.empty(7)
        self._ck(self._lib.rsv_suff_stats(self.ctx, float(c_mu), float(c_xi),
                                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def last_stats(self) -> np.ndarray:
        out = np.empty(7)
        self._ck(self._lib.rsv_last_stats(self.ctx, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out

    def set_timing(self, level):
        """0/False off, 1/True per-proposal total, 2 with the momenta /
        trajectory breakdown (graph event nodes, slightly slower)."""
        self._ck(self._lib.rsv_set_timing(self.ctx, int(level)))

    def kernel_stamps(self) -> dict:
        """In-kernel %globaltimer split of the last proposal (microseconds):
        momenta kernel, gap, trajectory kernel, and the gap since the
        previous proposal's trajectory ended."""
        st = (ctypes.c_uint64 * 5)()
        self._ck(self._lib.rsv_kernel_stamps(self.ctx, st))
        t = [int(x) for x in st]
        return {"momenta_us": (t[1] - t[0]) / 1e3, "gap_us": (t[2] - t[1]) / 1e3,
                "trajectory_us": (t[3] - t[2]) / 1e3, "since_prev_us": (t[0] - t[4]) / 1e3 if t[4] else None}

    def timing(self):
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        self._ck(self._lib.rsv_get_timing(self.ctx, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return a.value, b.value, c.value

    def set_l2_flush(self, nbytes: int):
        self._ck(self._lib.rsv_set_l2_flush(self.ctx, int(nbytes)))

    def fp64_peak_tflops(self) -> float:
        v = ctypes.c_double()
        self._ck(self._lib.rsv_measure_fp64_peak(self.ctx, ctypes.byref(v)))
        return float(v.value)

    def launch_count(self) -> int:
        return int(self._lib.rsv_launch_count(self.ctx))

    def bench_trajectory(self, step_size: float, n_steps: int, n: int = 20) -> float:
        """Per-launch ms of the trajectory kernel alone (rsv_bench_trajectory)."""
        ms = ctypes.c_float()
        self._ck(self._lib.rsv_bench_trajectory(self.ctx, float(step_size), int(n_steps), int(n), ctypes.byref(ms)))
        return float(ms.value)


class CudaBackend:
    """Drop-in ``backend=`` for the reference API (integrator.py:50-105).

    Holds one :class:`DeviceChain` per series length.  ``run`` speaks the
    reference's kernel-level protocol; ``workers`` is 1 because a single GPU
    executes every kernel (results never depend on it)."""

    workers = 1

    def __init__(self, device: int = 0):
        self.device = device
        self._chains: dict[int, DeviceChain] = {}
        self._aux: DeviceChain | None = None

    def chain(self, data: Dataset | None = None, params: Params | None = None, T: int | None = None) -> DeviceChain:
        T = data.length if data is not None else int(T)
        ch = self._chains.get(T)
        if ch is None:
            ch = self._chains[T] = DeviceChain(T, self.device)
        if data is not None:
            ch.set_data(data)
        if params is not None:
            ch.set_params(params)
        return ch

    def _any_chain(self) -> DeviceChain:
        if self._chains:
            return next(iter(self._chains.values()))
        if self._aux is None:
            self._aux = DeviceChain(2, self.device)
        return self._aux

    # -- the reference's backend protocol: run(kernel, n, args) -> int --
    def run(self, kernel, n: int, args: tuple) -> int:
        name = getattr(kernel, "__name__", getattr(getattr(kernel, "py_func", None), "__name__", ""))
        ch = self._any_chain()
        lib = ch._lib
        if name == "position_update":
            h, p, c = args
            self._f64_arrays(h, p)
            ch._ck(lib.rsv_position_update(ch.ctx, h.ctypes.data, p.ctypes.data, float(c), int(n), 0, int(n), 0))
            return 0
        if name == "momentum_update":
            h, p, y, lrv, dt = args[:5]
            self._f64_arrays(h, p, y, lrv)
            scal = np.array([float(v) for v in args[5:12]], dtype=np.float64)
            flag = ctypes.c_int32(0)
            ch._ck(lib.rsv_momentum_update(ch.ctx, h.ctypes.data, p.ctypes.data, y.ctypes.data, lrv.ctypes.data,
                                           float(dt), scal.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                           int(n), 0, int(n), ctypes.byref(flag), 0))
            return int(flag.value)
        if name == "gradient_fill":
            h, y, lrv, out = args[:4]
            self._f64_arrays(h, y, lrv, out)
            scal = np.array([float(v) for v in args[4:11]], dtype=np.float64)
            flag = ctypes.c_int32(0)
            ch._ck(lib.rsv_gradient(ch.ctx, h.ctypes.data, y.ctypes.data, lrv.ctypes.data,
                                    scal.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.ctypes.data,
                                    int(n), 0, int(n), ctypes.byref(flag), 0))
            return int(flag.value)
        raise NotImplementedError(f"CudaBackend cannot run kernel {name!r}")

    # -- the proposal-level hook of INTEGRATION.md (level 2): a reference
    # function that finds these methods on its backend forwards to them --
    def hmc_update_volatility(self, h, params, data, md, rng):
        """sampler.py:144-167 for the reference's own objects (duck-typed
        Dataset / Params / MDConfig, a numpy Generator): one fused proposal."""
        from .sampler import hmc_update_volatility
        return hmc_update_volatility(h, params, data, md, rng, backend=self)

    def integrate_trajectory(self, state, config, params, data, fuse_half_steps: bool = False):
        """integrator.py:149-179 for the reference's objects; returns the
        caller's PhaseState type."""
        ps, diverged = integrate_trajectory(state, config, params, data, backend=self,
                                            fuse_half_steps=fuse_half_steps)
        return type(state)(ps.h, ps.p), diverged

    @staticmethod
    def _f64_arrays(*arrs):
        for a in arrs:
            if a.dtype == np.float32:
                raise NotImplementedError("the B200 path computes in float64 only")
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError("CudaBackend.run needs C-contiguous float64 arrays")

    def gradient(self, h: np.ndarray, params: Params, data: Dataset) -> np.ndarray:
        out = np.empty_like(h)
        scal = np.array(scalar_pack(params, np.float64), dtype=np.float64)
        y = np.ascontiguousarray(data.returns, dtype=np.float64)
        lrv = np.ascontiguousarray(data.log_rv, dtype=np.float64)
        ch = self._any_chain()
        flag = ctypes.c_int32(0)
        ch._ck(ch._lib.rsv_gradient(ch.ctx, h.ctypes.data, y.ctypes.data, lrv.ctypes.data,
                                    scal.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.ctypes.data,
                                    h.size, 0, h.size, ctypes.byref(flag), 0))
        return out

    def close(self):
        for ch in self._chains.values():
            ch.close()
        self._chains.clear()
        if self._aux is not None:
            self._aux.close()
            self._aux = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


_DEFAULT: CudaBackend | None = None


def default_backend() -> CudaBackend:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = CudaBackend(0)
    return _DEFAULT


def _resolve(backend) -> CudaBackend:
    if backend is None:
        return default_backend()
    if not isinstance(backend, CudaBackend):
        raise TypeError("this package runs on the GPU: pass a CudaBackend (or None for the default)")
    return backend


def kernel1_half_position(state: PhaseState, dt: float, backend=None) -> PhaseState:
    """integrator.py:111-116: h += (dt/2) p in place (exact reference arithmetic)."""
    b = _resolve(backend)
    t = state.h.dtype.type
    b.run(_named("position_update"), state.size, (state.h, state.p, t(0.5) * t(dt)))
    return state


def kernel2_momentum(state: PhaseState, dt: float, params: Params, data: Dataset,
                     backend=None) -> tuple[PhaseState, bool]:
    """integrator.py:119-131: p -= dt * grad, divergence flag."""
    b = _resolve(backend)
    dtype = state.h.dtype
    args = (state.h, state.p, np.ascontiguousarray(data.returns, dtype=dtype),
            np.ascontiguousarray(data.log_rv, dtype=dtype), dtype.type(dt)) + scalar_pack(params, dtype)
    flag = b.run(_named("momentum_update"), state.size, args)
    return state, bool(flag)


def kernel3_half_position(state: PhaseState, dt: float, backend=None) -> PhaseState:
    """integrator.py:134-136."""
    return kernel1_half_position(state, dt, backend)


def elementary_step(state: PhaseState, config: MDConfig, params: Params, data: Dataset,
                    backend=None) -> tuple[PhaseState, bool]:
    """integrator.py:139-146: K1 -> K2 -> K3 in place, one streamed kernel."""
    b = _resolve(backend)
    if state.h.dtype != np.float64:
        raise NotImplementedError("the B200 path computes in float64 only")
    ch = b.chain(data, params)
    diverged = ch.elementary_step_inplace(state.h, state.p, config.step_size)
    return state, diverged


def integrate_trajectory(state: PhaseState, config: MDConfig, params: Params, data: Dataset, backend=None,
                         fuse_half_steps: bool = False) -> tuple[PhaseState, bool]:
    """integrator.py:149-179: n_steps leapfrog steps on a copy of ``state``,
    as one launch of the fused trajectory kernel."""
    b = _resolve(backend)
    if state.h.dtype != np.float64:
        raise NotImplementedError("the B200 path computes in float64 only")
    ch = b.chain(data, params)
    h, p, diverged = ch.integrate(state.h, state.p, config.step_size, config.n_steps, fuse_half_steps)
    return PhaseState(h, p), diverged


class _named:
    """Stand-in carrying a reference kernel name for CudaBackend.run."""

    def __init__(self, name):
        self.__name__ = name
