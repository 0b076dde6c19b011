"""B200-native alpha-complex construction (arXiv 1908.05944) -- a drop-in for
the hot path of the reference package ``alphax``:

    from paper_1908_05944_b200 import Ball, PipelineConfig, compute_alpha_complex

Python/PyTorch host code over hand-written sm_100a CUDA kernels behind a thin
C-ABI (``include/alphax_b200.h``).  No CPU fallback: computing without the
built library or without a GPU raises ``NativeLibraryMissing``.
"""

__version__ = "0.1.0"

from .errors import (
    AlphaxError,
    DegenerateSimplex,
    DuplicateCenter,
    EmptyInput,
    MalformedLine,
    MalformedRecord,
    NativeLibraryMissing,
    NoAtoms,
    NonFiniteCoordinate,
    NonFiniteValue,
    NonPositiveRadius,
    UnsupportedMode,
)
from .types import DEFAULT_TOLERANCE, Ball, OrthoResult, SimplexKey, TolerancePolicy, simplex_compare
from .pipeline import (
    STAGE_NAMES,
    AlphaComplex,
    ComplexStats,
    Engine,
    PipelineConfig,
    as_ball_arrays,
    closure_ok,
    complex_stats,
    compute_alpha_complex,
    compute_alpha_complex_arrays,
    compute_alpha_sweep,
    default_engine,
)
from .io import (format_xyzr, format_xyzr_arrays, parse_xyzr, parse_xyzr_arrays, read_complex, stats_csv,
                 write_complex)
from .stages import (CellKey, Grid, PotentialLevel, PotentialSets, ac2_mask, build_grid, cell_of, neighborhood,
                     potential_edges, potential_tets, potential_triangles, prune)
from .validate import ValidationReport, validate_complex
from . import synth

__all__ = [
    "AlphaComplex", "AlphaxError", "Ball", "ComplexStats", "DEFAULT_TOLERANCE", "DegenerateSimplex",
    "DuplicateCenter", "EmptyInput", "Engine", "MalformedLine", "MalformedRecord", "NativeLibraryMissing",
    "NoAtoms", "NonFiniteCoordinate", "NonFiniteValue", "NonPositiveRadius", "OrthoResult", "PipelineConfig",
    "STAGE_NAMES", "SimplexKey", "TolerancePolicy", "as_ball_arrays", "closure_ok", "complex_stats",
    "compute_alpha_complex", "compute_alpha_complex_arrays", "default_engine", "simplex_compare", "synth",
    "CellKey", "Grid", "PotentialLevel", "PotentialSets", "build_grid", "potential_edges", "potential_triangles",
    "potential_tets", "prune", "read_complex", "stats_csv", "write_complex", "parse_xyzr", "parse_xyzr_arrays",
    "format_xyzr", "format_xyzr_arrays", "UnsupportedMode", "ac2_mask", "cell_of", "neighborhood", "compute_alpha_sweep", "validate_complex", "ValidationReport",
]
