"""B200-native ISRS-GN NLI engine (arXiv 2401.18022 hot path).

The compute path is libuwbnli.so (hand-written sm_100a CUDA behind the C-ABI
in include/uwb_nli.h); this package is its Python mirror of the reference's
uwblink API.  See DESIGN.md.
"""
from .gn_integral import (  # noqa: F401
    BetaCoefficients, ChannelGrid, ConfigError, CudaError, DistanceGrid, Engine, FibreSpec,
    GnSolverConfig, LinkConfig, LinkReport, NliResult, PowerEvolution, RamanSolveOptions,
    ResidentLink, SolverError, U1Sampling, all_channels_nli, beta_from_dispersion,
    cfm_all_channels_nli,
    build_distance_grid, channel_nli, default_fibre, evaluate_link, flat_fibre, gamma_at,
    get_engine, make_default_uwb_grid, make_uniform_grid, nli_psd_at, set_launch,
    set_uniform_launch, solve_power_evolution,
)

__all__ = [n for n in dir() if not n.startswith("_")]
