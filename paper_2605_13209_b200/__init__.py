"""B200-native (sm_100a) SPD-solve path of arXiv 2605.13209: GP
squared-exponential assembly, blocked CG and tiled Cholesky, behind the
reference ``hsolve`` API (see ``hsolve.py`` and include/hs_cuda.h)."""
from .hsolve import (  # noqa: F401
    BlockedSPDMatrix, BlockVector, CgIteration, CgResult, ConfigError, DeviceError,
    DeviceMatrix, FactorizeStats, HsolveError, KernelParams, NotSpdError, NumericalError,
    Partition, Runtime, SingularBlockError, SolverConfig, SpdSolveResult, back_substitute,
    block_index, cholesky_border, factorize, forward_substitute, generate_inputs,
    generate_rhs, generate_spd, generate_spd_device, median_pairwise_distance,
    partition_for_fraction, partition_rows, potrf_device, solve_cg, solve_cg_device,
    solve_spd, solve_spd_device, symv_device, trsv_device, true_residual_device,
    FormatError, IoError, ResidencyError, TransferEntry, TruncatedFileError,
    VersionMismatchError, load_matrix, load_vector, save_matrix, save_vector,
)
