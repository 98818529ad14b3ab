"""gaplra-b200: the shift-and-invert hot path of arXiv 1607.02925 on B200 (sm_100a).

The product is libgaplra_cuda.so (C ABI: include/gaplra_cuda.h); this package
is its Python mirror of the reference `gaplra` interface.
"""
from .gaplra import (  # noqa: F401
    Context, ContractViolation, DeviceError, DeviceMatrix, Error, GramOperator, IndefiniteShift,
    NoPreconditioningNeeded, OutOfMemory, RankDeficient, ShiftInvertResult, ShiftOutOfRange, ShiftState,
    ShiftTuningStalled, SIConfig, SolverReport, SolverStalled, SymmetricEigen, default_context, estimate_top,
    gaussian_init, gram_apply, gram_block, index_stream, jacobi_eigh, orthonormality_defect, qr_orthonormalize,
    restricted_projection, shift_invert, solve_svrg, svrg_epoch, tune_shift, solve_cg, error_report,
    principal_angles, detect_multiplicative_gap, detect_additive_gap, estimate_eigenvalues, approximate,
    RankKProjection, find_gap_budget, NoUsableGap, DegenerateProgress, solve_accelerated_svrg,
)

__version__ = "0.1.0"
