"""B200-native HMC volatility update of the realized stochastic volatility
model (arXiv 1603.08114).

A drop-in for the hot path of the reference package ``rsvhmc``
(pkg/src/rsvhmc/__init__.py:34-50): the same names and signatures for the
model types, the integrator, the HMC proposal and the Gibbs driver, with the
leapfrog trajectory, the numpy-exact momenta, dH, the Metropolis test and the
theta sufficient statistics running as sm_100a CUDA kernels behind the C ABI
in include/rsvhmc_b200.h.  There is no CPU fallback.
"""
from .data import SyntheticTruth, ar1_path, simulate_rsv
from .integrator import (DH_DIVERGENCE_THRESHOLD, CudaBackend, DeviceChain, MDConfig, default_backend,
                         elementary_step, integrate_trajectory, kernel1_half_position, kernel2_momentum,
                         kernel3_half_position)
from .model import (PARAM_NAMES, Dataset, Params, PhaseState, grad_neg_log_posterior, hamiltonian,
                    log_posterior, scalar_pack)
from .bench_protocol import (BenchConfig, NumericError, ScalingStudy, TimingFit, TimingPoint, asymptotic_gain,
                             compute_gain, emit_report, fit_linear, run_scaling_study, time_elementary_step)
from .ensemble import Ensemble, sfc64_states
from .formats import (DataFormatError, IntradayPanel, compute_rv, load_chain, load_dataset, load_intraday,
                      load_truth, save_chain, save_dataset, save_truth)
from .sharded import ShardedChain, hmc_update_distributed, hmc_update_local, shard_bounds
from .rng import RsvBitGenerator, make_rng, seed_material, store_stream_state, stream_state
from .sampler import (Chain, ChainSample, DivergenceStormError, PriorSpec, SamplerConfig, default_init,
                      hmc_update_volatility, phi_log_accept_ratio, refresh_momenta, run_chain, update_mu,
                      update_phi, update_sigma_eta_sq, update_sigma_u_sq, update_xi)

__version__ = "0.1.0"

__all__ = [
    "BenchConfig", "DataFormatError", "IntradayPanel", "NumericError", "ScalingStudy", "TimingFit", "TimingPoint",
    "asymptotic_gain", "compute_gain", "compute_rv", "emit_report", "fit_linear", "load_chain", "load_dataset",
    "load_intraday", "load_truth", "run_scaling_study", "save_chain", "save_dataset", "save_truth",
    "time_elementary_step",
    "Chain", "ChainSample", "CudaBackend", "Ensemble", "sfc64_states", "DH_DIVERGENCE_THRESHOLD", "Dataset", "DeviceChain",
    "DivergenceStormError", "MDConfig", "PARAM_NAMES", "Params", "PhaseState", "PriorSpec", "RsvBitGenerator",
    "SamplerConfig", "ShardedChain", "SyntheticTruth", "hmc_update_distributed", "hmc_update_local", "shard_bounds", "ar1_path", "default_backend", "default_init", "elementary_step",
    "grad_neg_log_posterior", "hamiltonian", "hmc_update_volatility", "integrate_trajectory",
    "kernel1_half_position", "kernel2_momentum", "kernel3_half_position", "log_posterior", "make_rng",
    "phi_log_accept_ratio", "refresh_momenta", "run_chain", "scalar_pack", "seed_material", "simulate_rsv",
    "store_stream_state", "stream_state", "update_mu", "update_phi", "update_sigma_eta_sq", "update_sigma_u_sq",
    "update_xi",
]
