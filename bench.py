#!/usr/bin/env python
"""bench.py -- HMC site-updates/s of the RSV volatility update on B200.

Metric (BASELINE.json): HMC site-updates/sec (T x leapfrog steps / s) and
trajectories/s.  One "step" is one full HMC proposal of the reference's
hmc_update_volatility (sampler.py:144-167): numpy-exact momenta, H_old, an
L-step leapfrog trajectory, H_new, dH and the Metropolis test -- on one
synthetic series of T sites (config 3 of BASELINE.json at N=1: a single long
chain, T=2^20, L=20, dt=0.02, pcg32).  With N>1 (torchrun) the SAME chain is
time-sharded over the N GPUs (strong scaling): per proposal one
margin-halo exchange after an accepted move (NCCL send/recv), local momenta +
trajectory per GPU, an all_gather of the shards' energy totals and the same
Metropolis decision on every rank (sharded.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HMC site-updates/sec (T x leapfrog steps/s)"
UNIT = "site-updates/s"
THETA = dict(phi=0.97, mu=-9.0, xi=-0.3, sigma_eta_sq=0.05, sigma_u_sq=0.1)
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
# algorithmic FP64 work of one site-update of the leapfrog (DESIGN.md 4.2,
# SURVEY 8d): 2 half drifts (2 FMA), the kick (3 FMA + 2 ADD) and e^{-d}
# (a degree-3 polynomial after range reduction: 4 FMA-class + 3 ADD +
# rounding) -- counted as 26 flops.  The kernel issues 13 FP64 instructions
# per site-update for them (one full drift between kicks, the kick, and the
# scaled-state exp: 3 DADD + 3 DFMA/DMUL + 1 DFMA).
FLOPS_PER_SITE_UPDATE = 26
FP64_INSTR_PER_SITE_UPDATE = 13  # DFMA-pipe instructions (FMA, ADD, MUL each one issue slot)
HBM_BYTES_PER_SITE = 48  # streamed elementary step: r h,p,(y/2)y,lnRV; w h,p
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--T", type=int, default=1 << 20)
    ap.add_argument("--L", type=int, default=20)
    ap.add_argument("--dt", type=float, default=0.02)
    ap.add_argument("--prng", default="pcg32")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-ensemble", action="store_true")
    ap.add_argument("--no-protocol", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    ap.add_argument("--no-chain", action="store_true")
    ap.add_argument("--c5-T", type=int, default=1 << 26)
    ap.add_argument("--ens-chains", type=int, default=4096)
    ap.add_argument("--ens-T", type=int, default=4096)
    ap.add_argument("--sharded", action="store_true",
                    help="use the time-sharded path even at N=1 (exercises the N>1 code on one GPU)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.1)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(s[0]) for s in self.samples if len(s) >= 6 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 6 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples if len(s) >= 6 for i in range(4)
                          if s[2 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def config5_run(P, theta, T, block=4096, sweeps=60, dt=0.005):
    """Config 5 on one GPU: T = 2^26 sites, full theta update every sweep
    (run_chain with the theta draws on the device), sfc64 in the blocked
    layout (sites [j*4096, (j+1)*4096) from SFC64(SeedSequence([1, j])),
    the chain's own SFC64 stream for the uniforms and theta draws).  dt is
    0.005 here: at T = 2^26 the reference default 0.02 accepts nothing (the
    energy error grows with T).  The timed region is rsv_run_chain on the
    device-resident chain (the path was uploaded by the warm-up run);
    HBM-resident (T >> L2)."""
    be = P.CudaBackend(0)
    tr = P.simulate_rsv(theta, T, seed=11, backend=be)  # data generation on the device
    ch = be.chain(tr.dataset, theta)
    ch.set_blocked_streams(1, block)
    cfg = P.SamplerConfig(seed=1, md=P.MDConfig(dt, 20), n_burnin=0, n_samples=3, prng="sfc64")
    P.run_chain(tr.dataset, cfg, backend=be, init_params=theta, init_h=tr.latent)
    t0 = time.perf_counter()
    it, par, acc, dh = ch.run_chain_device(dt, 20, False, P.PriorSpec(), 0, sweeps, 1)
    el = time.perf_counter() - t0
    be.close()
    return {"workload": f"config 5 on 1 GPU: T={T}, L=20, dt={dt}, full theta update per sweep (device), sfc64 "
                        f"blocked momenta ({block}-site blocks, SeedSequence([1, j])), sfc64 main stream",
            "sweeps": sweeps, "sweeps_per_s": sweeps / el, "ms_per_sweep": el / sweeps * 1e3,
            "site_updates_per_s": T * 20 * sweeps / el, "accept_rate": float(acc.mean()),
            "timing": "wall clock around rsv_run_chain (device-resident chain; includes the samples' D2H)"}


def formats_run(P, theta, T=1 << 18, n_lat=8):
    """The data formats on either side of the sampler (host):
    dataset CSV save/load at T=2^18 and n_lat latent snapshots in the CSV
    companion vs the binary .npy sidecar."""
    import tempfile
    tr = P.simulate_rsv(theta, T, seed=7)
    out = {"T": T, "latent_snapshots": n_lat}
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "data.csv")
        t0 = time.perf_counter(); P.save_dataset(tr.dataset, f); out["dataset_save_s"] = time.perf_counter() - t0
        t0 = time.perf_counter(); back = P.load_dataset(f); out["dataset_load_s"] = time.perf_counter() - t0
        out["dataset_round_trip_exact"] = bool(np.array_equal(back.returns, tr.dataset.returns)
                                               and np.array_equal(back.rv, tr.dataset.rv))
        lat = tr.latent[None, :] + np.zeros((n_lat, 1))
        ch = P.Chain(iters=np.arange(n_lat), phi=np.full(n_lat, 0.97), mu=np.full(n_lat, -9.0),
                     xi=np.full(n_lat, -0.3), sigma_eta_sq=np.full(n_lat, 0.05), sigma_u_sq=np.full(n_lat, 0.1),
                     accept=np.ones(n_lat, bool), delta_h=np.zeros(n_lat), latent=lat)
        for kind in ("csv", "npy"):
            f = os.path.join(d, f"chain_{kind}.csv")
            t0 = time.perf_counter(); P.save_chain(ch, f, latent=kind); ts = time.perf_counter() - t0
            t0 = time.perf_counter(); b2 = P.load_chain(f); tl = time.perf_counter() - t0
            out[f"chain_latent_{kind}"] = {"save_s": ts, "load_s": tl, "exact": bool(np.array_equal(b2.latent, lat))}
    return out


def chain_run(P, be, theta):
    """Config 1 as a full sampler: run_chain (sampler.py:291-358) on T=2000,
    L=20, dt=0.02, minstd, every sweep (proposal + the five theta draws) on
    the device; sweeps/s by wall clock around run_chain (host arrays in and
    out, samples copied back at the end)."""
    tr = P.simulate_rsv(theta, 2000, seed=0)
    out = {}
    for T, tr_ in ((2000, tr), (1 << 20, P.simulate_rsv(theta, 1 << 20, seed=0))):
        cfg = P.SamplerConfig(seed=1, md=P.MDConfig(0.02, 20), n_burnin=0, n_samples=50, prng="minstd")
        P.run_chain(tr_.dataset, cfg, backend=be, init_params=theta, init_h=tr_.latent)
        n = 2000 if T == 2000 else 300
        cfg = P.SamplerConfig(seed=1, md=P.MDConfig(0.02, 20), n_burnin=0, n_samples=n, prng="minstd")
        t0 = time.perf_counter()
        ch = P.run_chain(tr_.dataset, cfg, backend=be, init_params=theta, init_h=tr_.latent)
        el = time.perf_counter() - t0
        out[f"T={T}"] = {"sweeps_per_s": n / el, "us_per_sweep": el / n * 1e6, "sweeps": n,
                         "accept_rate": float(ch.accept.mean()), "theta_on": "device"}
        be._chains.pop(T, None)
    out["workload"] = "run_chain, L=20, dt=0.02, minstd, theta draws on the device, init at the true path/params"
    return out


def paper_protocol(no_cpu):
    """Config 2 as the paper measures it (reference bench.py:121-267): the
    elementary step at T = 512*B, B = 2..512, 10^4 reps in segments of 100,
    5 repeats, fit A + C*B; beside it the CPU port with one thread (the
    reference's SerialBackend role) on fewer reps, and the gain curve."""
    from paper_1603_08114_b200 import bench_protocol as BP
    cfg = BP.BenchConfig()
    study = BP.run_scaling_study(cfg, fused=True)
    pts = study.timings["cuda"]
    fit = study.fits["cuda"]
    fpts = study.timings["cuda_fused"]
    ffit = study.fits["cuda_fused"]
    out = {"protocol": "reference bench.py:121-267 (device time of the step launches; state device-resident)",
           "params": "BENCH_PARAMS (phi .97, mu -1, xi -.3, se2 .05, su2 .1), dt 0.01, seed 0",
           "points": [{"B": p.b, "T": 512 * p.b, "mean_s": p.mean_seconds, "se_s": p.se_seconds,
                       "site_updates_per_s": 512 * p.b / p.mean_seconds} for p in pts],
           "fit_cuda": {"A_s": fit.intercept_a, "C_s_per_B": fit.slope_c, "r2": fit.r_squared},
           "fused": {"what": "the same protocol with each 100-step segment one launch of the persistent "
                             "trajectory kernel (halo tiles, no per-step synchronisation)",
                     "points": [{"B": p.b, "mean_s": p.mean_seconds, "se_s": p.se_seconds,
                                 "site_updates_per_s": 512 * p.b / p.mean_seconds} for p in fpts],
                     "fit": {"A_s": ffit.intercept_a, "C_s_per_B": ffit.slope_c, "r2": ffit.r_squared}}}
    if not no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        import paper_1603_08114_b200 as P
        cpu = []
        for b in cfg.b_values:
            data = P.simulate_rsv(BP.BENCH_PARAMS, 512 * b, seed=b).dataset
            h = data.log_rv - BP.BENCH_PARAMS.xi
            pm = np.random.default_rng(0).standard_normal(h.size)
            reps = max(20, int(2e6 // (512 * b)))
            O.integrate(h, pm, BP.BENCH_PARAMS, data.returns, data.log_rv, 0.01, 5, nthreads=1)
            t0 = time.perf_counter()
            O.integrate(h, pm, BP.BENCH_PARAMS, data.returns, data.log_rv, 0.01, reps, nthreads=1)
            cpu.append((b, (time.perf_counter() - t0) / reps))
        cfit = BP.fit_linear(cpu)
        out["cpu_port_serial"] = {"points": [{"B": b, "mean_s": t} for b, t in cpu],
                                  "fit": {"A_s": cfit.intercept_a, "C_s_per_B": cfit.slope_c, "r2": cfit.r_squared},
                                  "cores": 1}
        cpu_t = dict(cpu)
        out["gain_measured"] = [{"B": p.b, "gain": cpu_t[p.b] / p.mean_seconds} for p in pts]
        out["asymptotic_gain_fit"] = BP.asymptotic_gain(cfit, fit)
        out["fused"]["gain_measured"] = [{"B": p.b, "gain": cpu_t[p.b] / p.mean_seconds} for p in fpts]
        out["fused"]["asymptotic_gain_fit"] = BP.asymptotic_gain(cfit, ffit)
    return out


def ensemble_run(P, theta, dt, L, C, Tc, steps):
    """Config 4: C independent chains x Tc sites, one numpy SFC64 stream per
    chain (SeedSequence([seed, c])); one round = one HMC proposal of every
    chain.  Device-timed per round (event pair); the working set (>= 6 x 8 B
    x C x Tc = 768 MiB at 4096 x 4096) exceeds L2, so no flush is needed."""
    tr = P.simulate_rsv(theta, Tc, seed=5)
    ens = P.Ensemble(C, Tc)
    ens.set_data(tr.dataset.returns, tr.dataset.log_rv)
    ens.set_params(theta)
    ens.set_latent(tr.latent)
    ens.seed(1)
    ens.hmc_update(dt, L, rounds=3)
    ens.set_timing(1)
    n0 = ens.launch_count()
    ens.hmc_update(dt, L, rounds=steps)
    launches = ens.launch_count() - n0
    ms = ens.timing_ms()
    ens.set_timing(0)
    acc, _ = ens.counts()
    out = {"workload": f"config 4: {C} chains x T={Tc}, L={L}, dt={dt}, sfc64 per chain (SeedSequence([1, c]))",
           "metric": METRIC, "value": C * Tc * L / (ms * 1e-3), "unit": UNIT, "ms_per_round": ms,
           "chain_trajectories_per_s": C / (ms * 1e-3), "accept_rate": float(acc.sum()) / ((steps + 3) * C),
           "rounds": steps, "gpu_launches": int(launches),
           "data": "one simulate_rsv series (seed 5) shared by every chain; latent starts at the true path",
           "l2": "working set > L2 (768 MiB): not flushed"}
    ens.close()
    return out


def cpu_model() -> str:
    """The host CPU's model name (the baseline's hardware)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def config_dict(T, L, dt, prng):
    """The workload description shared verbatim by both arms (the driver
    compares the two lines' `config`)."""
    return {"workload": f"config 3: single chain T={T}, L={L}, dt={dt}, {prng}; one step = one full "
                        "HMC proposal of hmc_update_volatility (momenta + H_old + trajectory + H_new + Metropolis)",
            "T": T, "L": L, "dt": dt, "prng": prng}


def import_reference():
    """The unmodified reference package (`rsvhmc`, installed into
    baseline/_ref by pip --target) -- None when absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "rsvhmc")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "rsvhmc_numba_cache"))
    try:
        import rsvhmc
    except Exception:  # numba or numpy missing on the host
        return None
    if not os.path.abspath(rsvhmc.__file__).startswith(REF_DIR):
        return None
    return rsvhmc


def time_reference(T, L, dt, prng, steps, warmup, seconds=None, parallel_steps=2):
    """The reference's own CPU path on this host: rsvhmc.hmc_update_volatility
    (sampler.py:144-167) with its numba kernels, once with SerialBackend (one
    core; integrator.py:50-65) and once with ParallelBackend(nproc)
    (integrator.py:68-105, default 512-site chunks) -- the stock code path,
    nothing of this repository on it except the bit generator object feeding
    numpy's Generator (oracle Stream: the pcg32 / minstd words of DESIGN 6;
    the reference itself only ships Philox).  Data: the reference's own
    simulate_rsv(theta, T, seed=0); the chain starts at the true path.
    Returns None when the reference cannot be imported here."""
    ref = import_reference()
    if ref is None:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from rsvhmc import integrator as RI
    from rsvhmc import sampler as RS
    theta = ref.Params(**THETA)
    truth = ref.simulate_rsv(theta, T, seed=0)
    md = RI.MDConfig(dt, L)
    out = {}
    for name, mk, n_steps in (("serial", lambda: RI.SerialBackend(), steps),
                              ("parallel", lambda: RI.ParallelBackend(os.cpu_count()), parallel_steps)):
        if n_steps <= 0:
            continue
        gen = O.Stream(prng, 1).generator()
        h = truth.latent.copy()
        with mk() as be:
            for _ in range(max(1, warmup if name == "serial" else 1)):  # numba JIT + caches
                h, _, _ = RS.hmc_update_volatility(h, theta, truth.dataset, md, gen, backend=be)
            times = []
            while len(times) < n_steps:
                t0 = time.perf_counter()
                h, _, _ = RS.hmc_update_volatility(h, theta, truth.dataset, md, gen, backend=be)
                times.append(time.perf_counter() - t0)
                if seconds is not None and sum(times) >= seconds:
                    break
        tot = sum(times)
        out[name] = {"value": T * L * len(times) / tot, "unit": UNIT, "proposals": len(times),
                     "seconds": tot, "s_per_proposal": tot / len(times),
                     "cores": 1 if name == "serial" else os.cpu_count()}
    best = max(out.values(), key=lambda r: r["value"])
    out["best"] = "serial" if best is out.get("serial") else "parallel"
    return out


def cpu_port(T, L, dt, kind, seconds, data, h0):
    """The reference algorithm restated in C (oracle/, kind 'port'), all host
    threads for the leapfrog kernels, on a bounded sample of proposals."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    import paper_1603_08114_b200 as P
    nth = O.max_threads()
    theta = P.Params(**THETA)
    st = O.Stream(kind, 1)
    h = h0.copy()
    O.hmc_update(h, theta, data.returns, data.log_rv, dt, L, st, nthreads=nth)  # warm the pool
    n, t0 = 0, time.perf_counter()
    while True:
        h, _, _ = O.hmc_update(h, theta, data.returns, data.log_rv, dt, L, st, nthreads=nth)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 200:
            break
    O.lib().orc_pool_shutdown()
    return {"value": T * L * n / el, "unit": UNIT, "cores": nth, "kind": "port",
            "sample": f"{n} HMC proposals (momenta+2H+{L}-step trajectory+Metropolis) at T={T}, {el:.1f} s",
            "trajectories_per_s": n / el}


def cpu_baseline(T, L, dt, kind, seconds, data, h0):
    """cpu_baseline of the b200 line: the reference itself (rsvhmc + numba,
    SerialBackend -- the faster of its two backends at this size) on a
    bounded sample, the C port beside it; the port alone when the reference
    cannot be imported on this host."""
    port = cpu_port(T, L, dt, kind, seconds, data, h0)
    ref = time_reference(T, L, dt, kind, steps=10 ** 6, warmup=1, seconds=seconds, parallel_steps=0)
    host = {"cpu_model": cpu_model(), "nproc": os.cpu_count()}
    if ref is None:
        return dict(port, **host, note="reference (baseline/_ref) not importable on this host: the C port")
    r = ref["serial"]
    return {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"{r['proposals']} proposals of rsvhmc.hmc_update_volatility (SerialBackend, numba) at T={T}, "
                      f"{r['seconds']:.1f} s",
            "trajectories_per_s": 1.0 / r["s_per_proposal"], **host, "port": port}


def run_reference(args, ws, rank):
    """--impl reference: the unmodified reference (baseline/_ref) on this
    host's cores, same metric / config as the b200 arm; rank 0 only."""
    if rank != 0:
        return
    ref = time_reference(args.T, args.L, args.dt, args.prng, args.steps, args.warmup)
    host = {"cpu_model": cpu_model(), "nproc": os.cpu_count()}
    if ref is None:  # fall back to the C restatement, and say so
        import paper_1603_08114_b200 as P
        truth = P.simulate_rsv(P.Params(**THETA), args.T, seed=0)
        port = cpu_port(args.T, args.L, args.dt, args.prng, 1e9, truth.dataset, truth.latent)
        value, cores, kind = port["value"], port["cores"], "port"
        sample, extra = port["sample"], {"note": "rsvhmc not importable from baseline/_ref: oracle port timed"}
    else:
        best = ref[ref["best"]]
        value, cores, kind = best["value"], best["cores"], "reference"
        sample = (f"{best['proposals']} proposals of rsvhmc.hmc_update_volatility at T={args.T} "
                  f"({ref['best']} backend, numba)")
        extra = {"backends": {k: ref[k] for k in ("serial", "parallel") if k in ref}}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * args.T * args.L / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (simulate_rsv, theta of SURVEY \u00a78d, seed 0)", "impl": "reference",
            "config": config_dict(args.T, args.L, args.dt, args.prng),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample, **host},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "trajectories_per_s": value / (args.T * args.L), **extra}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import torch
    dist = None
    if ws > 1 or args.sharded:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            dist.init_process_group("nccl", rank=0, world_size=1)
        else:
            dist.init_process_group("nccl")
    import paper_1603_08114_b200 as P

    theta = P.Params(**THETA)
    T, L, dt = args.T, args.L, args.dt
    truth = P.simulate_rsv(theta, T, seed=0)
    data = truth.dataset
    be = P.CudaBackend(local)
    if dist is not None:
        sharded_run(args, P, theta, truth, rank, ws, local, dist, torch)
        be.close()
        dist.destroy_process_group()
        return
    ch = be.chain(data, theta)
    ch.set_latent(truth.latent)
    ch.set_stream(P.stream_state(P.make_rng(1 + rank, args.prng)))
    # warm-up (graph capture + clocks)
    ch.hmc_update_many(dt, L, max(3, args.warmup), results=False)

    # ---------------- timed region: K proposals, device-timed per step
    ch.set_l2_flush(L2_FLUSH_BYTES)
    clocks = ClockSampler(local)
    clocks.start()
    # keep the GPU under the same load for ~0.4 s so nvidia-smi samples the
    # clocks of this workload (the timed region itself is milliseconds long)
    t_load = time.perf_counter()
    while time.perf_counter() - t_load < 0.4:
        ch.hmc_update_many(dt, L, 20, results=False)
    ch.set_timing(1)  # one event pair per proposal around the proposal graph
    torch.cuda.synchronize(local)
    n0 = ch.launch_count()
    t_wall = time.perf_counter()
    res = ch.hmc_update_many(dt, L, args.steps, results=True)
    bracket_s = time.perf_counter() - t_wall
    torch.cuda.synchronize(local)
    launches = ch.launch_count() - n0
    clk = clocks.stop()
    clk["window"] = "0.4 s of the same proposals immediately before + the timed region"
    _, _, step_ms = ch.timing()
    # breakdown pass (not the headline): event nodes inside the graph around
    # the momenta and trajectory kernels (their own latency inflates both a bit)
    ch.set_timing(2)
    ch.hmc_update_many(dt, L, args.steps, results=False)
    traj_ms, mom_ms, bd_total_ms = ch.timing()
    ch.set_timing(0)
    ch.set_l2_flush(0)
    ch.hmc_update_many(dt, L, 4, results=False)
    stamps = ch.kernel_stamps()  # in-kernel %globaltimer split (no events, no flush)
    accept_rate = float(np.mean([r.accept for r in res]))
    step_s = step_ms * 1e-3
    value = T * L / step_s

    # ---------------- roofline of the dominant kernel (trajectory, FP64-bound):
    # its launch duration = CUDA events around 20 back-to-back launches of the
    # proposal's trajectory kernel on the context's stream (bench_trajectory)
    fp64_peak = ch.fp64_peak_tflops()
    traj_launch_ms = ch.bench_trajectory(dt, L, 20)
    achieved = FLOPS_PER_SITE_UPDATE * T * L / (traj_launch_ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traj_dram_bytes.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(str(T))
        except Exception:
            traffic = None

    # ---------------- e2e through the public API (host buffers, copies timed)
    rng = P.make_rng(7 + rank, args.prng)
    md = P.MDConfig(dt, L)
    h_host = torch.empty(T, dtype=torch.float64, pin_memory=True).numpy()
    h_host[:] = truth.latent
    h = h_host
    for _ in range(max(3, args.warmup)):  # warm: graph, pinned result buffers
        h, _, _ = P.hmc_update_volatility(h.view(), theta, data, md, rng, backend=be)
    e2e_steps = max(3, min(args.steps, 20))
    n_acc = 0
    # the path crosses the link every step: a view of the returned array is
    # not the chain's own returned path, so it is read from host memory again
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        h, acc, _ = P.hmc_update_volatility(h.view(), theta, data, md, rng, backend=be)
        n_acc += int(acc)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    ch_e2e = be.chain(data, theta)
    zero_copy = ch_e2e.last_update_zero_copy  # h read in place by the trajectory kernel
    assert not ch_e2e.last_update_resident
    # a chain loop passing the returned path straight back (the reference's
    # run_chain does): the device keeps the path, only the stream state goes
    # in and an accepted proposal comes out
    hr = h
    for _ in range(400):  # until a returned path is in hand (an accepted proposal)
        if not hr.flags.writeable:
            break
        hr, _, _ = P.hmc_update_volatility(hr, theta, data, md, rng, backend=be)
    for _ in range(3):
        hr, _, _ = P.hmc_update_volatility(hr, theta, data, md, rng, backend=be)
    n_acc_r = 0
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        hr, acc, _ = P.hmc_update_volatility(hr, theta, data, md, rng, backend=be)
        n_acc_r += int(acc)
    e2e_res_s = (time.perf_counter() - t0) / e2e_steps
    resident = ch_e2e.last_update_resident
    # the same call with a plain (pageable) numpy path, the reference user's usual case
    # (every step proposes from the same pageable path, so each call copies it in)
    hp = np.array(h)
    for _ in range(2):
        P.hmc_update_volatility(hp, theta, data, md, rng, backend=be)
    n_acc_p = 0
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        _, acc, _ = P.hmc_update_volatility(hp, theta, data, md, rng, backend=be)
        n_acc_p += int(acc)
    e2e_pg_s = (time.perf_counter() - t0) / e2e_steps
    state_bytes = 48 + 40  # stream state + params structs
    e2e = {"value": T * L / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * T + state_bytes,
           "d2h_bytes_per_step": int(8 * T * n_acc / e2e_steps) + 48 + 56,
           "h_in": "read in place over PCIe by the trajectory kernel (zero copy)" if zero_copy else "copied in",
           "path": "paper_1603_08114_b200.hmc_update_volatility(h numpy[pinned], params, data, md, rng) -> C ABI",
           "resident_chain": {"value": T * L / e2e_res_s, "unit": UNIT, "h2d_bytes_per_step": state_bytes,
                              "d2h_bytes_per_step": int(8 * T * n_acc_r / e2e_steps) + 48 + 56,
                              "resident": resident,
                              "h_in": "the returned (read-only) path passed back: proposed from the device's "
                                      "copy, only the stream state crosses the link"},
           "pageable": {"value": T * L / e2e_pg_s, "unit": UNIT, "h2d_bytes_per_step": 8 * T + state_bytes,
                        "d2h_bytes_per_step": int(8 * T * n_acc_p / e2e_steps) + 48 + 56,
                        "h_in": "pageable numpy array: copied in (cudaMemcpy from pageable memory); every "
                                "step proposes from the same path"}}

    extra = {}
    if rank == 0:
        # ---------------- HBM roofline of the streamed one-step kernel (T >> L2)
        Ts = 1 << 24
        tr2 = P.simulate_rsv(theta, Ts, seed=3)
        ch2 = be.chain(tr2.dataset, theta)
        hh = tr2.latent.copy()
        pp = np.random.default_rng(0).standard_normal(Ts)
        ch2.elementary_step_inplace(hh, pp, dt)
        import ctypes
        ms = ctypes.c_float()
        ch2._ck(ch2._lib.rsv_bench_elementary(ch2.ctx, dt, 50, ctypes.byref(ms), None))
        per = ms.value / 50 * 1e-3
        peaks = json.load(open(PEAKS)) if os.path.exists(PEAKS) else {}
        hbm_peak = peaks.get("hbm_gbs", 6650.0)
        gbs = HBM_BYTES_PER_SITE * Ts / per / 1e9
        extra["roofline_hbm"] = {"kernel": "estep_kernel (one streamed leapfrog step, integrator.py:139-146)",
                                 "bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                                 "frac": gbs / hbm_peak, "traffic": HBM_BYTES_PER_SITE * Ts,
                                 "site_updates_per_s": Ts / per, "T": Ts,
                                 "peak_source": "MEASURED_PEAKS.json" if peaks else "fallback 6.65 TB/s"}
        be._chains.pop(Ts, None)
        ch2.close()
        # ---------------- paper-style sweep (config 2): trajectories/s vs T
        if not args.no_sweep:
            sweep = []
            for Tq in (1 << 10, 1 << 14, 1 << 18):
                trq = P.simulate_rsv(theta, Tq, seed=4)
                cq = be.chain(trq.dataset, theta)
                cq.set_latent(trq.latent)
                cq.set_stream(P.stream_state(P.make_rng(2, args.prng)))
                cq.hmc_update_many(dt, L, 5, results=False)
                cq.set_timing(1)
                cq.hmc_update_many(dt, L, 50, results=False)
                _, _, sq = cq.timing()
                cq.set_timing(2)
                cq.hmc_update_many(dt, L, 50, results=False)
                tq, mq, _ = cq.timing()
                cq.set_timing(0)
                # throughput of back-to-back proposals: hmc_update_many without
                # per-proposal events runs them in graphs of 8 with programmatic
                # dependent launches (the per-graph gap dominates at small T)
                nb_ = 400
                cq.hmc_update_many(dt, L, 16)
                t0 = time.perf_counter()
                cq.hmc_update_many(dt, L, nb_)
                bq = (time.perf_counter() - t0) / nb_ * 1e3
                sweep.append({"T": Tq, "ms_per_proposal": sq, "traj_kernel_ms": tq, "momenta_ms": mq,
                              "trajectories_per_s": 1e3 / sq, "site_updates_per_s": Tq * L / (sq * 1e-3),
                              "batched": {"ms_per_proposal": bq, "trajectories_per_s": 1e3 / bq,
                                          "how": f"one hmc_update_many({nb_}) call, wall clock incl. the result "
                                                 "copy; proposals in graphs of 8, L2 not flushed"}})
                be._chains.pop(Tq, None)
                cq.close()
            extra["sweep"] = sweep
        if not args.no_ensemble:
            extra["ensemble"] = ensemble_run(P, theta, dt, L, args.ens_chains, args.ens_T, args.steps)
        if not args.no_protocol:
            extra["paper_protocol"] = paper_protocol(args.no_cpu)
        if not args.no_chain:
            extra["chain_config1"] = chain_run(P, be, theta)
        if not args.no_config5:
            extra["config5"] = config5_run(P, theta, args.c5_T)
        extra["formats"] = formats_run(P, theta)
        if not args.no_cpu:
            extra["cpu_baseline"] = cpu_baseline(T, L, dt, args.prng, args.cpu_seconds, data, truth.latent)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (simulate_rsv, theta of SURVEY §8d, seed 0)",
            "config": config_dict(T, L, dt, args.prng),
            "parallelism": "single chain, 1 GPU; device-resident, one CUDA graph per proposal",
            "l2": f"flushed between steps ({L2_FLUSH_BYTES >> 20} MiB memset, not timed)",
            "trajectories_per_s": 1.0 / step_s, "accept_rate": accept_rate,
            "breakdown_ms": {"momenta": mom_ms, "trajectory": traj_ms, "proposal_with_event_nodes": bd_total_ms},
            "in_kernel_us": stamps,
            "bracket_ms_per_step_incl_flush": bracket_s * 1e3 / args.steps,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "roofline": {"kernel": "traj_persistent_kernel (fused L-step trajectory)", "bound": "fp64",
                         "achieved": achieved, "launch_ms": traj_launch_ms,
                         "launch_timing": "CUDA events around 20 back-to-back launches on the context's stream "
                                          "(integrate-only, the proposal's geometry; L2 warm as inside a proposal)",
                         "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak, "traffic": traffic,
                         "flops_per_site_update": FLOPS_PER_SITE_UPDATE,
                         "peak_source": "measured live: DFMA microbenchmark (rsv_measure_fp64_peak)",
                         "fp64_pipe": {"instr_per_site_update": FP64_INSTR_PER_SITE_UPDATE,
                                       "frac": FP64_INSTR_PER_SITE_UPDATE * 2 / FLOPS_PER_SITE_UPDATE * achieved / fp64_peak,
                                       "note": "issue-slot view: every FP64 instruction occupies the pipe like an FMA"},
                         "in_kernel": {"trajectory_us": stamps["trajectory_us"],
                                       "achieved_tflops": FLOPS_PER_SITE_UPDATE * T * L / (stamps["trajectory_us"] * 1e-6) / 1e12}},
            "clocks": clk,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    be.close()


def sharded_run(args, P, theta, truth, rank, ws, local, dist, torch):
    """N > 1 (config 3): ONE chain of T sites time-sharded over the N GPUs
    (strong scaling), orchestrated on the device: per proposal each GPU
    parses only its window of the momenta stream (window records
    all-gathered, normals placed bit for bit as the whole-series draw), runs
    the trajectory on its sites plus an 8(L+1)-site margin, writes its
    23-word record (fixed-point dH / H parts: the same dH bits as one GPU);
    NCCL all-gathers the records and every GPU takes the same Metropolis
    decision on the device; the margins are exchanged (NCCL send/recv) every
    7 proposals, which keeps the owned sites exact whatever was accepted in
    between.  The host only enqueues; timed with CUDA events per proposal
    (max over ranks).  Beside it: e2e with host buffers, and config 5
    (T=2^26, run_chain) sharded the same way."""
    T, L, dt = args.T, args.L, args.dt
    dev = f"cuda:{local}"
    margin = 8 * (L + 1)
    windowed = args.prng != "sfc64"

    def make_chain():
        ch = P.ShardedChain(truth.dataset, theta, rank, ws, margin=margin, device=local)
        ch.set_latent_global(truth.latent)
        ch.set_stream(P.stream_state(P.make_rng(1, args.prng)))
        if windowed:
            ch.set_windowed_momenta(True)
        return ch

    # the per-proposal records go through the peer-memory boxes (NVLink
    # stores) unless RSV_P2P=0 or any rank cannot map its peers' boxes; a run
    # in which some rank's records never arrive (the collect kernel's 5 s
    # timeout) falls back to the NCCL exchange on every rank
    p2p = P.sharded._p2p_default(ws)
    chain = make_chain()
    ok = True
    try:
        P.sharded.hmc_update_distributed_device(chain, dt, L, max(3, args.warmup), p2p=p2p)
    except P._native.NativeError:
        ok = False
    agreed = torch.tensor([1 if ok else 0], dtype=torch.int32, device=f"cuda:{local}")
    dist.all_reduce(agreed, op=dist.ReduceOp.MIN)
    if not int(agreed.item()):
        chain.shard.close()
        p2p = False
        chain = make_chain()
        P.sharded.hmc_update_distributed_device(chain, dt, L, max(3, args.warmup), p2p=False)
    exchange = P.sharded.exchange_kind(chain)
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    t_load = time.perf_counter()
    while time.perf_counter() - t_load < 0.4:
        P.sharded.hmc_update_distributed_device(chain, dt, L, 21, graph=True, p2p=p2p)
    # L2 flushed before every proposal (a 256 MiB write, not timed), one event
    # pair per proposal around it on the proposal stream (as at N=1)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    dist.barrier()
    torch.cuda.synchronize(local)
    n0 = chain.shard.launch_count()
    times = []
    res = P.sharded.hmc_update_distributed_device(chain, dt, L, args.steps, l2_flush=flush, times=times, graph=True,
                                                  p2p=p2p)
    torch.cuda.synchronize(local)
    launches = chain.shard.launch_count() - n0
    dist.barrier()
    ms = sum(times) / len(times)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    clk = clocks.stop() if clocks else None

    # ---- e2e with host buffers: each step the rank's local slice of the path
    # goes in from page-locked host memory, one proposal runs, the decision
    # and the owned slice come back (wall clock, max over ranks)
    ls, le, lo, hi = chain.ls, chain.le, chain.lo, chain.hi
    h_host = torch.empty(T, dtype=torch.float64, pin_memory=True).numpy()
    h_host[:] = truth.latent
    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(2):
        chain.shard.set_latent(h_host[ls:le])
        chain.halo_valid = True
        P.sharded.hmc_update_distributed_device(chain, dt, L, 1, p2p=p2p)
    dist.barrier()
    n_acc = 0
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        chain.shard.set_latent(h_host[ls:le])
        chain.halo_valid = True
        r = P.sharded.hmc_update_distributed_device(chain, dt, L, 1, p2p=p2p)
        if r[0].accept:
            h_host[lo:hi] = chain.owned_latent()
            n_acc += 1
    dist.barrier()
    e2e_s = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_s[0])

    # ---- config 5 sharded: T = 2^26, full theta update per sweep, blocked sfc64
    c5 = None
    if not args.no_config5:
        c5 = config5_sharded(args, P, theta, rank, ws, local, dist, torch, p2p=p2p)

    if rank == 0:
        v = T * L / (ms * 1e-3)
        acc = sum(bool(x.accept) for x in res) / max(1, len(res))
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (simulate_rsv, theta of SURVEY \u00a78d, seed 0)",
                "config": config_dict(T, L, dt, args.prng),
                "parallelism": f"time-sharded x{ws} (margin {margin} sites, halo every "
                               f"{P.sharded.halo_period(margin, L)} proposals, "
                               + ("windowed momenta (each GPU parses its window of the stream), " if windowed else
                                  "replicated momenta (sfc64: no jump-ahead), ")
                               + ("shard records exchanged by NVLink stores into every GPU's box (peer memory), "
                                  if exchange == "p2p" else "NCCL all_gather of the shard records, ")
                               + "decision on the device)",
                "exchange": exchange,
                "l2": "flushed before every proposal (256 MiB write per GPU, outside the event pairs)",
                "trajectories_per_s": 1e3 / ms, "accept_rate": acc, "clocks": clk,
                "e2e": {"value": T * L / e2e_s, "unit": UNIT,
                        "h2d_bytes_per_step": 8 * (le - ls),
                        "d2h_bytes_per_step": int(8 * (hi - lo) * n_acc / e2e_steps) + 48,
                        "path": "per rank: local path slice from pinned host memory -> ShardedChain -> "
                                "sharded.hmc_update_distributed_device (one proposal) -> decision + owned slice "
                                "back to host; wall clock, max over ranks; bytes are rank 0's"},
                "gpu_launches": int(launches)}
        if c5 is not None:
            line["config5"] = c5
        print(json.dumps(line), flush=True)


def config5_sharded(args, P, theta, rank, ws, local, dist, torch, block=4096, sweeps=30, dt=0.005, p2p=None):
    """Config 5 across the N GPUs: T = 2^26, run_chain with the theta draws
    on every GPU from the all-gathered statistics, sfc64 blocked momenta
    (each GPU draws the blocks its sites touch).  Wall clock around the
    sweeps (device-orchestrated; includes the samples' D2H), max over ranks."""
    T = args.c5_T
    truth = P.simulate_rsv(theta, T, seed=11, backend=P.CudaBackend(local))
    margin = 8 * 21
    ch = P.ShardedChain(truth.dataset, theta, rank, ws, margin=margin, device=local)
    ch.set_latent_global(truth.latent)
    ch.set_stream(P.stream_state(P.make_rng(1, "sfc64")))
    ch.set_blocked_streams(1, block)
    prior = P.PriorSpec()
    P.sharded.run_chain_sharded([ch], dt, 20, prior, 0, 2, 1, p2p=p2p)
    ch.set_params(theta)
    dist.barrier()
    torch.cuda.synchronize(local)
    t0 = time.perf_counter()
    it, par, acc, dh = P.sharded.run_chain_sharded([ch], dt, 20, prior, 0, sweeps, 1, p2p=p2p)
    torch.cuda.synchronize(local)
    el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(el, op=dist.ReduceOp.MAX)
    el = float(el[0])
    ch.shard.close()
    return {"workload": f"config 5 on {ws} GPUs: T={T}, L=20, dt={dt}, full theta update per sweep (on every GPU "
                        f"from all-gathered statistics), sfc64 blocked momenta ({block}-site blocks), time-sharded",
            "sweeps": sweeps, "sweeps_per_s": sweeps / el, "ms_per_sweep": el / sweeps * 1e3,
            "site_updates_per_s": T * 20 * sweeps / el, "accept_rate": float(np.mean(acc)),
            "timing": "wall clock around run_chain_sharded (device-orchestrated; samples' D2H), max over ranks"}


if __name__ == "__main__":
    main()
