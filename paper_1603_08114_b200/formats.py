"""File formats on either side of the sampler.

The reference keeps its data and results in plain CSV (`data.py:98-327`):
datasets `date,return,rv`, intraday panels `date,time,return`, chains
`iter,phi,mu,xi,sigma_eta_sq,sigma_u_sq,accept,delta_h` with the latent
snapshots in a companion `<stem>.latent<suffix>` file `iter,h1..hT`, and the
ground truth of a simulation as `# name=value` comment lines over `date,h`.
Floats are written with 17 significant digits (a loss-free round trip),
UTF-8, LF line endings; blank lines are skipped and `#` lines are comments;
errors name the offending file and line.  This module reads and writes those
files byte-compatibly (tests/test_formats.py checks against files written by
the reference itself) and adds one thing the reference lacks: a binary
sidecar for multi-GB latent snapshots (T = 2^26 x n samples would be tens of
GB of decimal text) -- `<stem>.latent.npy`, used when `latent="npy"` and
picked up by `load_chain` in preference to the CSV companion.
"""
from __future__ import annotations

import csv
import io
import logging
import math
from dataclasses import dataclass
from datetime import date, timedelta
from pathlib import Path

import numpy as np

from .model import PARAM_NAMES, Dataset, Params

logger = logging.getLogger(__name__)

RV_FLOOR = 1e-12                 # data.py: days with zero realized variance are floored here
_FIRST_DAY = date(2000, 1, 3)    # synthesized dates start here (data.py: _DATE_BASE)
CHAIN_COLUMNS = ("iter", *PARAM_NAMES, "accept", "delta_h")


class DataFormatError(ValueError):
    """A file could not be parsed into the expected shape."""


def fmt_float(v) -> str:
    """17 significant digits: parses back to the same double."""
    return format(float(v), ".17g")


def synth_dates(n: int) -> list[str]:
    return [(_FIRST_DAY + timedelta(days=k)).isoformat() for k in range(n)]


class _Table:
    """A parsed CSV file: comment lines, the header, numbered data rows."""

    def __init__(self, path):
        self.path = Path(path)
        if not self.path.exists():
            raise DataFormatError(f"no such file: {self.path}")
        self.comments: list[str] = []
        self.header: list[str] | None = None
        self.rows: list[tuple[int, list[str]]] = []
        with open(self.path, newline="", encoding="utf-8") as fh:
            for lineno, line in enumerate(fh, start=1):
                text = line.strip()
                if not text:
                    continue
                if text.startswith("#"):
                    self.comments.append(text)
                    continue
                cells = next(csv.reader([line]))
                if self.header is None:
                    self.header = [c.strip() for c in cells]
                else:
                    self.rows.append((lineno, cells))
        if self.header is None:
            raise DataFormatError(f"{self.path}: file has no header row")

    def expect_header(self, cols, what=None):
        if self.header != list(cols):
            want = ",".join(cols)
            raise DataFormatError(what or f"{self.path}: expected header '{want}', got {','.join(self.header)!r}")

    def number(self, raw: str, lineno: int, column: str) -> float:
        try:
            return float(raw)
        except ValueError:
            raise DataFormatError(f"{self.path}, line {lineno}: cannot parse {column}={raw!r} as a number") from None

    def width(self, lineno: int, cells, n: int):
        if len(cells) != n:
            raise DataFormatError(f"{self.path}, line {lineno}: expected {n} columns, got {len(cells)}")


def _write_text(path, text: str):
    with open(path, "w", newline="\n", encoding="utf-8") as fh:
        fh.write(text)


# ---------------------------------------------------------------- datasets
def save_dataset(dataset: Dataset, path) -> None:
    """`date,return,rv` (dates synthesized when the dataset has none)."""
    dates = dataset.dates or synth_dates(dataset.length)
    buf = io.StringIO()
    buf.write("date,return,rv\n")
    for d, r, v in zip(dates, dataset.returns, dataset.rv):
        buf.write(f"{d},{fmt_float(r)},{fmt_float(v)}\n")
    _write_text(path, buf.getvalue())


def load_dataset(path) -> Dataset:
    t = _Table(path)
    t.expect_header(("date", "return", "rv"))
    if not t.rows:
        raise DataFormatError(f"{path}: empty dataset")
    dates, ret, rv = [], [], []
    for lineno, cells in t.rows:
        t.width(lineno, cells, 3)
        r = t.number(cells[1], lineno, "return")
        v = t.number(cells[2], lineno, "rv")
        if not math.isfinite(r):
            raise DataFormatError(f"{path}, line {lineno}: non-finite return")
        if not math.isfinite(v):
            raise DataFormatError(f"{path}, line {lineno}: non-finite rv")
        if v <= 0.0:
            raise DataFormatError(f"{path}, line {lineno}: rv={cells[2]} is not positive (its log is undefined)")
        dates.append(cells[0])
        ret.append(r)
        rv.append(v)
    if len(ret) < 2:
        raise DataFormatError(f"{path}: dataset needs at least 2 rows")
    return Dataset(returns=np.array(ret), rv=np.array(rv), dates=dates)


# ---------------------------------------------------------------- intraday panels
@dataclass
class IntradayPanel:
    """Per-day sequences of intraday log-returns (data.py)."""

    returns_per_day: list
    dates: list | None = None

    def __post_init__(self):
        self.returns_per_day = [np.asarray(r, dtype=np.float64) for r in self.returns_per_day]
        if not self.returns_per_day:
            raise ValueError("panel has no days")
        for k, r in enumerate(self.returns_per_day):
            if r.ndim != 1 or r.size < 1:
                raise ValueError(f"day {k} must hold at least one return")
            if not np.all(np.isfinite(r)):
                raise ValueError(f"day {k} contains non-finite returns")
        if self.dates is not None and len(self.dates) != len(self.returns_per_day):
            raise ValueError("dates length does not match number of days")

    @property
    def n_days(self) -> int:
        return len(self.returns_per_day)


def compute_rv(panel: IntradayPanel) -> np.ndarray:
    """Daily realized variance = sum of squared intraday returns, floored at
    RV_FLOOR for all-zero days (with a warning)."""
    rv = np.array([float(np.sum(r * r)) for r in panel.returns_per_day])
    low = rv < RV_FLOOR
    if low.any():
        logger.warning("%d day(s) with zero realized variance floored at %g", int(low.sum()), RV_FLOOR)
        rv[low] = RV_FLOOR
    return rv


def load_intraday(path) -> IntradayPanel:
    t = _Table(path)
    t.expect_header(("date", "time", "return"))
    if not t.rows:
        raise DataFormatError(f"{path}: empty intraday file")
    days: dict[str, list[float]] = {}
    for lineno, cells in t.rows:
        t.width(lineno, cells, 3)
        r = t.number(cells[2], lineno, "return")
        if not math.isfinite(r):
            raise DataFormatError(f"{path}, line {lineno}: non-finite return")
        days.setdefault(cells[0], []).append(r)
    names = list(days)
    return IntradayPanel(returns_per_day=[np.array(days[d]) for d in names], dates=names)


# ---------------------------------------------------------------- chains
def latent_companion(path) -> Path:
    p = Path(path)
    return p.with_name(p.stem + ".latent" + (p.suffix or ".csv"))


def latent_sidecar(path) -> Path:
    """Binary latent snapshots (this package's addition): <stem>.latent.npy."""
    p = Path(path)
    return p.with_name(p.stem + ".latent.npy")


def save_chain(chain, path, latent: str = "csv") -> None:
    """The chain table; latent snapshots (if stored) to the CSV companion
    (latent="csv", the reference's format) or to the .npy sidecar
    (latent="npy", with the iteration indices in the first column)."""
    if latent not in ("csv", "npy"):
        raise ValueError(f"latent must be 'csv' or 'npy', got {latent!r}")
    buf = io.StringIO()
    buf.write(",".join(CHAIN_COLUMNS) + "\n")
    series = [chain.param_series(n) for n in PARAM_NAMES]
    for k in range(len(chain)):
        cells = [str(int(chain.iters[k]))] + [fmt_float(s[k]) for s in series]
        cells += ["1" if chain.accept[k] else "0", fmt_float(chain.delta_h[k])]
        buf.write(",".join(cells) + "\n")
    _write_text(path, buf.getvalue())
    if chain.latent is None:
        return
    if latent == "npy":
        np.save(latent_sidecar(path), np.column_stack([np.asarray(chain.iters, dtype=np.float64), chain.latent]))
        return
    T = chain.latent.shape[1]
    lines = ["iter," + ",".join(f"h{t + 1}" for t in range(T))]
    for k in range(len(chain)):
        lines.append(str(int(chain.iters[k])) + "," + ",".join(fmt_float(v) for v in chain.latent[k]))
    _write_text(latent_companion(path), "\n".join(lines) + "\n")


def load_chain(path):
    from .sampler import Chain
    t = _Table(path)
    t.expect_header(CHAIN_COLUMNS, f"{path}: expected header {','.join(CHAIN_COLUMNS)!r}, "
                                   f"got {','.join(t.header)!r}")
    n = len(t.rows)
    iters = np.empty(n, dtype=np.int64)
    cols = {name: np.empty(n) for name in PARAM_NAMES}
    accept = np.empty(n, dtype=bool)
    delta_h = np.empty(n)
    for k, (lineno, cells) in enumerate(t.rows):
        t.width(lineno, cells, len(CHAIN_COLUMNS))
        try:
            iters[k] = int(cells[0])
        except ValueError:
            raise DataFormatError(f"{path}, line {lineno}: bad iteration index {cells[0]!r}") from None
        for j, name in enumerate(PARAM_NAMES, start=1):
            cols[name][k] = t.number(cells[j], lineno, name)
        accept[k] = cells[6].strip() == "1"
        delta_h[k] = t.number(cells[7], lineno, "delta_h")
    latent = None
    side = latent_sidecar(path)
    comp = latent_companion(path)
    if side.exists():
        arr = np.load(side)
        if arr.ndim != 2 or arr.shape[0] != n:
            raise DataFormatError(f"{side}: {arr.shape[0] if arr.ndim == 2 else '?'} latent rows for {n} chain rows")
        latent = np.ascontiguousarray(arr[:, 1:])
    elif comp.exists():
        lt = _Table(comp)
        if len(lt.rows) != n:
            raise DataFormatError(f"{comp}: {len(lt.rows)} latent rows for {n} chain rows")
        T = len(lt.header) - 1
        latent = np.empty((n, T))
        for k, (lineno, cells) in enumerate(lt.rows):
            lt.width(lineno, cells, T + 1)
            latent[k] = [lt.number(c, lineno, "h") for c in cells[1:]]
    return Chain(iters=iters, accept=accept, delta_h=delta_h, latent=latent, **cols)


# ---------------------------------------------------------------- simulation truth
def save_truth(truth, path) -> None:
    """`# name=value` lines for the generating parameters over `date,h`."""
    dates = truth.dataset.dates or synth_dates(truth.dataset.length)
    buf = io.StringIO()
    for name in PARAM_NAMES:
        buf.write(f"# {name}={fmt_float(getattr(truth.params, name))}\n")
    buf.write("date,h\n")
    for d, v in zip(dates, truth.latent):
        buf.write(f"{d},{fmt_float(v)}\n")
    _write_text(path, buf.getvalue())


def load_truth(path) -> tuple[Params, np.ndarray]:
    t = _Table(path)
    t.expect_header(("date", "h"), f"{path}: expected header 'date,h'")
    found = {}
    for c in t.comments:
        body = c.lstrip("#").strip()
        if "=" in body:
            key, _, raw = body.partition("=")
            found[key.strip()] = float(raw)
    missing = [n for n in PARAM_NAMES if n not in found]
    if missing:
        raise DataFormatError(f"{path}: missing parameter lines for {missing}")
    h = np.array([t.number(cells[1], lineno, "h") for lineno, cells in t.rows])
    return Params(**{n: found[n] for n in PARAM_NAMES}), h
