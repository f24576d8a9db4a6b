"""ctypes binding of ``librsvhmc_b200.so`` (the C ABI in include/rsvhmc_b200.h).

There is no fallback: if the library is missing or no B200 is visible, the
calls raise.  Build it with ``python -c "import __graft_entry__ as g; g.build()"``
(or ``make -C paper_1603_08114_b200/csrc``).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RSV_LIB=checked selects the build with device-side invariant checks
# (make -C paper_1603_08114_b200/csrc checked; tools/checked_run.sh)
LIB_PATH = os.path.join(_HERE, "librsvhmc_b200_checked.so" if os.environ.get("RSV_LIB") == "checked"
                        else "librsvhmc_b200.so")

RSV_E_INVALID = -1
RSV_E_CUDA = -2
RSV_E_STATE = -3
RSV_E_STORM = -4

KINDS = {"philox": 0, "minstd": 1, "pcg32": 2, "sfc64": 3}
KIND_NAMES = {v: k for k, v in KINDS.items()}


class PrngState(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("s", ctypes.c_uint64 * 4), ("pos", ctypes.c_uint64)]


class Prior(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("mu_mean", "mu_var", "xi_mean", "xi_var", "var_shape", "var_scale",
                                               "phi_a", "phi_b")]


class Params(ctypes.Structure):
    _fields_ = [("phi", ctypes.c_double), ("mu", ctypes.c_double), ("xi", ctypes.c_double),
                ("sigma_eta_sq", ctypes.c_double), ("sigma_u_sq", ctypes.c_double)]


class Result(ctypes.Structure):
    _fields_ = [("accept", ctypes.c_int32), ("diverged", ctypes.c_int32), ("delta_h", ctypes.c_double),
                ("h_old", ctypes.c_double), ("h_new", ctypes.c_double), ("words_used", ctypes.c_uint64),
                ("u", ctypes.c_double)]


class ShardTotals(ctypes.Structure):  # rsv_shard_totals: 23 8-byte words
    _fields_ = [("dh", ctypes.c_int64 * 2), ("h_old", ctypes.c_int64 * 2), ("h_new", ctypes.c_int64 * 2),
                ("stats_old", ctypes.c_double * 5), ("stats_new", ctypes.c_double * 5), ("flag", ctypes.c_double),
                ("ends", ctypes.c_double * 4), ("u_word", ctypes.c_uint64), ("words_used", ctypes.c_uint64)]


class Bitgen(ctypes.Structure):  # numpy/random/bitgen.h
    _fields_ = [("state", ctypes.c_void_p), ("next_uint64", ctypes.c_void_p),
                ("next_uint32", ctypes.c_void_p), ("next_double", ctypes.c_void_p),
                ("next_raw", ctypes.c_void_p)]


_lib = None
_D = ctypes.POINTER(ctypes.c_double)
_I32P = ctypes.POINTER(ctypes.c_int32)
_CTX = ctypes.c_void_p

# name: (restype, argtypes)
_SIGS = {
    "rsv_last_error": (ctypes.c_char_p, [_CTX]),
    "rsv_version": (ctypes.c_char_p, []),
    "rsv_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int64]),
    "rsv_destroy": (ctypes.c_int, [_CTX]),
    "rsv_set_data": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "rsv_set_params": (ctypes.c_int, [_CTX, ctypes.POINTER(Params)]),
    "rsv_set_latent": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_int]),
    "rsv_get_latent": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_int]),
    "rsv_set_prng_state": (ctypes.c_int, [_CTX, ctypes.POINTER(PrngState)]),
    "rsv_get_prng_state": (ctypes.c_int, [_CTX, ctypes.POINTER(PrngState)]),
    "rsv_refresh_momenta": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_int]),
    "rsv_hmc_update": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.POINTER(Result)]),
    "rsv_hmc_update_many": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(Result)]),
    "rsv_integrate": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, _I32P, ctypes.c_int]),
    "rsv_elementary_step": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, _I32P,
                                           ctypes.c_int]),
    "rsv_bench_elementary": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                                            ctypes.c_void_p]),
    "rsv_bench_fused": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                                       ctypes.c_void_p]),
    "rsv_bench_state": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p]),
    "rsv_bench_trajectory": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_float)]),
    "rsv_position_update": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int]),
    "rsv_momentum_update": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_double, _D, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, _I32P, ctypes.c_int]),
    "rsv_gradient": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _D,
                                    ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _I32P,
                                    ctypes.c_int]),
    "rsv_hamiltonian": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p, _D, ctypes.c_int]),
    "rsv_log_posterior": (ctypes.c_int, [_CTX, ctypes.c_void_p, _D, ctypes.c_int]),
    "rsv_suff_stats": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_double, _D]),
    "rsv_last_stats": (ctypes.c_int, [_CTX, _D]),
    "rsv_set_timing": (ctypes.c_int, [_CTX, ctypes.c_int]),
    "rsv_get_timing": (ctypes.c_int, [_CTX, _D, _D, _D]),
    "rsv_launch_count": (ctypes.c_int64, [_CTX]),
    "rsv_kernel_stamps": (ctypes.c_int, [_CTX, ctypes.c_void_p]),
    "rsv_last_update_zero_copy": (ctypes.c_int, [_CTX]),
    "rsv_hmc_update_host": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
    "rsv_run_chain": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "rsv_get_params": (ctypes.c_int, [_CTX, ctypes.c_void_p]),
    "rsv_set_blocked_streams": (ctypes.c_int, [_CTX, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]),
    "rsv_set_stream": (ctypes.c_int, [_CTX, ctypes.c_void_p]),
    "rsv_simulate": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]),
    "rsv_shard_propose_async": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_void_p]),
    "rsv_shard_decide_async": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_int]),
    "rsv_shard_set_momenta": (ctypes.c_int, [_CTX, ctypes.c_int]),
    "rsv_shard_prepare": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "rsv_shard_momenta_async": (ctypes.c_int, [_CTX, ctypes.c_void_p]),
    "rsv_shard_place_async": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]),
    "rsv_shard_p2p_init": (ctypes.c_int, [_CTX, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.POINTER(ctypes.c_uint64)]),
    "rsv_shard_p2p_connect": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p]),
    "rsv_shard_p2p_push_async": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_int]),
    "rsv_shard_p2p_collect_async": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_int]),
    "rsv_shard_set_blocked_streams": (ctypes.c_int, [_CTX, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                                     ctypes.c_void_p]),
    "rsv_shard_run_begin": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64]),
    "rsv_shard_theta_async": (ctypes.c_int, [_CTX]),
    "rsv_shard_run_end": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "rsv_shard_halo_async": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                            ctypes.c_int]),
    "rsv_shard_results": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    "rsv_get_blocked_streams": (ctypes.c_int, [_CTX, ctypes.c_void_p]),
    "rsv_ens_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int, ctypes.c_int64]),
    "rsv_ens_set_streams": (ctypes.c_int, [_CTX, ctypes.c_void_p]),
    "rsv_ens_get_streams": (ctypes.c_int, [_CTX, ctypes.c_void_p]),
    "rsv_ens_refresh_momenta": (ctypes.c_int, [_CTX, ctypes.c_void_p]),
    "rsv_ens_hmc_update": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p]),
    "rsv_ens_counts": (ctypes.c_int, [_CTX, ctypes.c_void_p, ctypes.c_void_p]),
    "rsv_set_l2_flush": (ctypes.c_int, [_CTX, ctypes.c_int64]),
    "rsv_measure_fp64_peak": (ctypes.c_int, [_CTX, _D]),
    "rsv_create_shard": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                        ctypes.POINTER(ctypes.c_int64)]),
    "rsv_shard_propose": (ctypes.c_int, [_CTX, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ShardTotals)]),
    "rsv_shard_apply": (ctypes.c_int, [_CTX, ctypes.c_int, ctypes.c_int]),
    "rsv_latent_slice": (ctypes.c_int, [_CTX, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                        ctypes.c_int]),
    "rsv_stream_seed": (ctypes.c_int, [ctypes.POINTER(PrngState), ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]),
    "rsv_stream_next_u64": (ctypes.c_uint64, [ctypes.POINTER(PrngState)]),
    "rsv_stream_next_double": (ctypes.c_double, [ctypes.POINTER(PrngState)]),
    "rsv_stream_bitgen": (ctypes.c_int, [ctypes.POINTER(PrngState), ctypes.POINTER(Bitgen)]),
    "rsv_philox_block": (None, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]),
}

EXPORTED = tuple(_SIGS)


def lib() -> ctypes.CDLL:
    """Load the CUDA library; raises if it was not built (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a library first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class NativeError(RuntimeError):
    pass


class StormError(NativeError):
    """RSV_E_STORM from rsv_run_chain (re-raised as DivergenceStormError)."""


def check(code: int, ctx=None) -> None:
    if code == 0:
        return
    msg = lib().rsv_last_error(ctx)
    msg = msg.decode() if msg else "unknown error"
    if code == RSV_E_INVALID:
        raise ValueError(msg)
    if code == RSV_E_STORM:
        raise StormError(msg)
    raise NativeError(msg)


def ptr(a: np.ndarray) -> int:
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise ValueError("expected a C-contiguous float64 array")
    return a.ctypes.data


def to_params(p) -> Params:
    return Params(float(p.phi), float(p.mu), float(p.xi), float(p.sigma_eta_sq), float(p.sigma_u_sq))
