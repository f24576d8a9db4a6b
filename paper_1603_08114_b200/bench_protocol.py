"""The paper's scaling protocol for the elementary leapfrog step, on the GPU.

Mirrors the reference's `bench.py` (its module docstring and
`time_elementary_step` `bench.py:121-190`, `fit_linear` :193-210,
`compute_gain` / `asymptotic_gain` :213-230, `run_scaling_study` :240-267,
`emit_report` :274-309): for each B, T = 512*B sites; warm-up, then `reps`
consecutive elementary steps (K1 -> K2 -> K3, `integrator.py:139-146`) timed
in segments of 100 with untimed momentum refreshes in between, `repeats`
times for a standard error; divergence retries with half the step size; the
mean step times are fit to f(B) = A + C*B.

Differences, by design: the state stays resident on the device and each
step is one streamed kernel (`estep_kernel`), so the time is the device time
of the step launches (CUDA events), not a Python wall clock; the backend is
the GPU ("cuda").  The CSV report has the reference's layout.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from datetime import datetime, timezone
from pathlib import Path

import numpy as np

from . import _native as N
from .data import simulate_rsv
from .integrator import DeviceChain
from .model import Dataset, Params
from .rng import make_rng

SITES_PER_UNIT = 512
BENCH_PARAMS = Params(phi=0.97, mu=-1.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)  # bench.py:41-42
_REFRESH_EVERY = 100
_MAX_RETRIES = 3


class NumericError(RuntimeError):
    """A numeric procedure failed (degenerate fit, diverging timing run)."""


@dataclass(frozen=True)
class TimingFit:
    intercept_a: float
    slope_c: float
    r_squared: float

    def predict(self, b: float) -> float:
        return self.intercept_a + self.slope_c * b


@dataclass(frozen=True)
class TimingPoint:
    b: int
    mean_seconds: float
    se_seconds: float
    step_size: float


@dataclass(frozen=True)
class BenchConfig:
    b_values: tuple[int, ...] = (2, 4, 8, 16, 32, 64, 128, 256, 512)
    reps: int = 10000
    repeats: int = 5
    step_size: float = 0.01
    seed: int = 0
    device: int = 0

    def __post_init__(self):
        if not self.b_values or any(b < 1 for b in self.b_values):
            raise ValueError(f"b_values must be positive integers, got {self.b_values}")
        if self.reps < 1:
            raise ValueError(f"reps must be >= 1, got {self.reps}")
        if self.repeats < 1:
            raise ValueError(f"repeats must be >= 1, got {self.repeats}")


@dataclass
class ScalingStudy:
    config: BenchConfig
    timings: dict[str, list[TimingPoint]] = field(default_factory=dict)
    fits: dict[str, TimingFit] = field(default_factory=dict)


def _steps(ch: DeviceChain, dt: float, n: int, fused: bool = False) -> tuple[float, bool]:
    ms = ctypes.c_float()
    div = ctypes.c_int32(0)
    fn = ch._lib.rsv_bench_fused if fused else ch._lib.rsv_bench_elementary
    ch._ck(fn(ch.ctx, float(dt), int(n), ctypes.byref(ms), ctypes.byref(div)))
    return ms.value * 1e-3, bool(div.value)


def _set_state(ch: DeviceChain, h: np.ndarray | None, p: np.ndarray | None):
    h = None if h is None else np.ascontiguousarray(h, dtype=np.float64)
    p = None if p is None else np.ascontiguousarray(p, dtype=np.float64)
    ch._ck(ch._lib.rsv_bench_state(ch.ctx, None if h is None else h.ctypes.data,
                                   None if p is None else p.ctypes.data))


def time_elementary_step(b: int, backend, reps: int, params: Params, data: Dataset, *, step_size: float = 0.01,
                         repeats: int = 5, n_warmup: int = 10, precision: str = "double", seed: int = 0,
                         device: int | None = None, fused: bool = False) -> TimingPoint:
    """Mean device seconds of one elementary step at T = 512*b (bench.py:121-190,
    same signature; `backend` is a CudaBackend or None, only its device is used).
    fused=True (this package's addition): each 100-step segment is one launch
    of the persistent trajectory kernel instead of 100 streamed step kernels."""
    if precision != "double":
        raise NotImplementedError("the B200 path computes in float64 only (FP32 bench mode is out of scope)")
    if device is None:
        device = getattr(backend, "device", 0) if backend is not None else 0
    t_len = SITES_PER_UNIT * b
    if data.length != t_len:
        raise ValueError(f"dataset length {data.length} does not match 512*B = {t_len}")
    h_start = data.log_rv - params.xi
    ch = DeviceChain(t_len, device)
    try:
        ch.set_data(data)
        ch.set_params(params)
        dt = step_size
        for _ in range(_MAX_RETRIES + 1):
            rng = make_rng(seed)
            per_rep: list[float] = []
            diverged = False
            for _ in range(repeats):
                _set_state(ch, h_start, rng.standard_normal(t_len))
                _, diverged = _steps(ch, dt, n_warmup, fused)
                if diverged:
                    break
                total, done = 0.0, 0
                while done < reps:
                    seg = min(_REFRESH_EVERY, reps - done)
                    t, diverged = _steps(ch, dt, seg, fused)
                    total += t
                    if diverged:
                        break
                    done += seg
                    _set_state(ch, None, rng.standard_normal(t_len))
                if diverged:
                    break
                per_rep.append(total / reps)
            if not diverged:
                mean = float(np.mean(per_rep))
                se = float(np.std(per_rep, ddof=1) / math.sqrt(len(per_rep))) if len(per_rep) > 1 else 0.0
                return TimingPoint(b=b, mean_seconds=mean, se_seconds=se, step_size=dt)
            dt /= 2
        raise NumericError(f"timing at B={b} kept diverging after {_MAX_RETRIES} retries")
    finally:
        ch.close()


def fit_linear(points) -> TimingFit:
    """OLS fit of (B, seconds) to f(B) = A + C*B with R^2 (bench.py:193-210)."""
    pts = [(float(b), float(y)) for b, y in points]
    if len(pts) < 2:
        raise NumericError(f"need >= 2 points for a line, got {len(pts)}")
    b = np.array([p[0] for p in pts])
    y = np.array([p[1] for p in pts])
    if np.all(b == b[0]):
        raise NumericError("degenerate fit: all B values identical")
    slope, intercept = np.polyfit(b, y, 1)
    resid = y - (intercept + slope * b)
    ss_res = float(resid @ resid)
    ss_tot = float(((y - y.mean()) ** 2).sum())
    r2 = (1.0 if ss_res <= 1e-30 else 0.0) if ss_tot == 0.0 else 1.0 - ss_res / ss_tot
    return TimingFit(float(intercept), float(slope), r2)


def compute_gain(fit_slow: TimingFit, fit_fast: TimingFit, b: float) -> float:
    fast = fit_fast.predict(b)
    if fast <= 0.0:
        raise NumericError(f"fast backend has non-positive predicted time {fast} at B={b}")
    return fit_slow.predict(b) / fast


def asymptotic_gain(fit_slow: TimingFit, fit_fast: TimingFit) -> float:
    if fit_fast.slope_c <= 0.0:
        raise NumericError(f"fast backend has non-positive slope {fit_fast.slope_c}")
    return fit_slow.slope_c / fit_fast.slope_c


def run_scaling_study(config: BenchConfig = BenchConfig(), params: Params = BENCH_PARAMS,
                      fused: bool = False) -> ScalingStudy:
    """The reference's study on the GPU ("cuda": one streamed kernel per
    step); with fused=True also "cuda_fused" (100-step segments in one
    launch of the persistent trajectory kernel)."""
    study = ScalingStudy(config=config)
    for name, fz in (("cuda", False), ("cuda_fused", True)) if fused else (("cuda", False),):
        pts = []
        for b in config.b_values:
            data = simulate_rsv(params, SITES_PER_UNIT * b, seed=config.seed + b).dataset
            pts.append(time_elementary_step(b, None, config.reps, params, data, step_size=config.step_size,
                                            repeats=config.repeats, seed=config.seed, device=config.device,
                                            fused=fz))
        study.timings[name] = pts
        if len(set(config.b_values)) >= 2:
            study.fits[name] = fit_linear([(p.b, p.mean_seconds) for p in pts])
    return study


def emit_report(study: ScalingStudy, out_dir) -> dict[str, Path]:
    """timings_<backend>.csv and fits.csv in the reference's layout (bench.py:274-309)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    stamp = f"# generated={datetime.now(timezone.utc).isoformat()}\n"
    paths = {}
    for name, points in study.timings.items():
        path = out / f"timings_{name}.csv"
        with open(path, "w", newline="\n", encoding="utf-8") as fh:
            fh.write(stamp)
            fh.write("B,T,mean_seconds,se_seconds\n")
            for p in points:
                fh.write(f"{p.b},{SITES_PER_UNIT * p.b},{p.mean_seconds!r},{p.se_seconds!r}\n")
        paths[f"timings_{name}"] = path
    path = out / "fits.csv"
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        fh.write(stamp)
        fh.write("backend,intercept_a,slope_c,r_squared\n")
        for name, f in study.fits.items():
            fh.write(f"{name},{f.intercept_a!r},{f.slope_c!r},{f.r_squared!r}\n")
    paths["fits"] = path
    return paths
