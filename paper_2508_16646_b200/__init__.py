"""B200-native Equinox per-step scheduling path (arXiv 2508.16646).

The package is a drop-in for the reference's scheduling hot path only: host mirror of the
reference types (scheduler.py) over the C ABI in include/eqx.h, implemented by sm_100a
kernels in csrc/ (libeqx_b200.so).  See DESIGN.md and INTEGRATION.md.
"""
from .scheduler import (  # noqa: F401
    ClientState,
    ConfigError,
    EngineError,
    EquinoxParams,
    GpuProfile,
    GpuScheduler,
    MopeModel,
    ParseError,
    PerfParams,
    PolicySpec,
    ProfileEntry,
    StepResult,
    TrainingError,
    default_bucket_bounds,
    rfc_increment,
    ufc_increment,
)

__version__ = "0.1.0"
