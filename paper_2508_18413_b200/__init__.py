"""chainscan-b200: B200-native parallel-in-time MCMC (arXiv 2508.18413 hot path).

Drop-in mirror of the reference ``chainscan`` solver/sampler API
(/root/reference/pkg/src/chainscan): the same names, argument meanings and
exceptions, backed by hand-written sm_100a CUDA kernels in
``_build/libchainscan_b200.so`` (C-ABI: include/chainscan_b200.h).  There is
no CPU fallback; every compute call needs a CUDA device.
"""

from . import core, deer, noise, pscan, samplers, targets  # noqa: F401
from .core import (  # noqa: F401
    ChainDivergedError,
    ConfigurationError,
    StructuralError,
    TargetModel,
    TransitionSystem,
    sequential_evaluate,
)
from .deer import DeerConfig, DeerResult, converged, deer_iterate, default_max_iters, hutchinson_diag, run_deer  # noqa: F401
from .noise import NoiseTable, SlotSpec, rademacher_probe  # noqa: F401
from .pscan import (  # noqa: F401
    Block2x2Elements,
    DenseElements,
    DiagElements,
    apply_element,
    compose,
    default_chunk,
    identity_element,
    parallel_affine_solve,
    sequential_affine_solve,
)
from .samplers import (  # noqa: F401
    EightSchoolsData,
    EightSchoolsHyper,
    GibbsKernel,
    HmcKernel,
    LeapfrogSystem,
    MalaKernel,
    generate_eight_schools,
)
from .targets import blr, gaussian, model_logp_grad_hvp, mog, rosenbrock, std_normal, synthetic_credit_like  # noqa: F401

from .basis import OrthogonalBasis, orthogonal_basis, transform_system  # noqa: F401
from .tracefile import TraceFormatError, export_csv, read_trace, write_trace  # noqa: F401

__version__ = "0.1.0"
