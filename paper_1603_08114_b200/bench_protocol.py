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
    """bench.py's NumericError: the fit is degenerate or a timing run kept
    diverging (API contract: same name, same conditions)."""


@dataclass(frozen=True)
class TimingFit:
    """f(B) = A + C*B fitted to mean step times (fields as bench.py's)."""
    intercept_a: float
    slope_c: float
    r_squared: float

    def predict(self, b: float) -> float:
        return float(np.polyval((self.slope_c, self.intercept_a), b))


@dataclass(frozen=True)
class TimingPoint:
    """One B of the study: mean / standard error of the step time and the
    step size it finally ran with (fields as bench.py's)."""
    b: int
    mean_seconds: float
    se_seconds: float
    step_size: float


@dataclass(frozen=True)
class BenchConfig:
    """The study's schedule (bench.py's BenchConfig without the CPU-only
    fields chunk / backends / workers / precision; `device` added)."""
    b_values: tuple[int, ...] = (2, 4, 8, 16, 32, 64, 128, 256, 512)
    reps: int = 10000
    repeats: int = 5
    step_size: float = 0.01
    seed: int = 0
    device: int = 0

    def __post_init__(self):
        checks = (("b_values", bool(self.b_values) and min(self.b_values) >= 1, "positive integers"),
                  ("reps", self.reps >= 1, ">= 1"),
                  ("repeats", self.repeats >= 1, ">= 1"))
        for name, ok, want in checks:
            if not ok:
                raise ValueError(f"{name} must be {want}, got {getattr(self, name)}")


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
    """Least squares of the (B, seconds) pairs on f(B) = A + C*B, with R^2
    (the study's fit, bench.py:193-210), from the centred sums: C = Sby/Sbb,
    A = mean(y) - C mean(b).  Fewer than two points or a single distinct B
    raise NumericError; a constant y gives R^2 = 1 for an exact fit, else 0."""
    bs = np.array([float(b) for b, _ in points])
    ys = np.array([float(y) for _, y in points])
    if bs.size < 2:
        raise NumericError(f"a line needs at least two points (have {bs.size})")
    db = bs - bs.mean()
    sbb = float(db @ db)
    if sbb == 0.0:
        raise NumericError("degenerate fit: every point has the same B")
    dy = ys - ys.mean()
    c = float(db @ dy) / sbb
    a = float(ys.mean()) - c * float(bs.mean())
    r = ys - (a + c * bs)
    ss_res, ss_tot = float(r @ r), float(dy @ dy)
    if ss_tot > 0.0:
        r2 = 1.0 - ss_res / ss_tot
    else:
        r2 = 1.0 if ss_res <= 1e-30 else 0.0
    return TimingFit(intercept_a=a, slope_c=c, r_squared=r2)


def _ratio(num: float, den: float, what: str) -> float:
    if not den > 0.0:
        raise NumericError(f"the faster backend's {what} is not positive ({den})")
    return num / den


def compute_gain(fit_slow: TimingFit, fit_fast: TimingFit, b: float) -> float:
    """Speed-up of the fitted models at B: f_slow(B) / f_fast(B)."""
    return _ratio(fit_slow.predict(b), fit_fast.predict(b), f"predicted time at B={b}")


def asymptotic_gain(fit_slow: TimingFit, fit_fast: TimingFit) -> float:
    """The speed-up as B grows: C_slow / C_fast."""
    return _ratio(fit_slow.slope_c, fit_fast.slope_c, "slope")


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
