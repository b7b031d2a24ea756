"""B200-native batched DC loadflow engine (arXiv 2501.17529 hot path).

Drop-in for the reference's session binding (`batchdc_session.session_open`,
`solve_batch`) and library entry point (`batchdc.solve_batch`), with the
numerical work on hand-written sm_100a CUDA kernels behind the C ABI in
``include/bdc.h`` (``libbdc.so``, built in-tree by ``build.py``).
"""

from .errors import (
    BatchDcError,
    DegenerateSplit,
    DisconnectedTopology,
    EngineUnavailable,
    InvalidReduction,
    IslandingError,
    ParseError,
    SingularSplit,
    SingularSystem,
    UnsupportedFeature,
    ValidationError,
)
from .grid import (
    Branch,
    ContingencyCase,
    Grid,
    Injection,
    SplittableSubstation,
    branch_bridges,
    build_grid,
    replace_stub_branches,
    static_injection_fold,
)
from .io import grid_from_dict, grid_to_dict, load_grid, result_to_dict
from .ptdf import PtdfMatrix, compute_ptdf, prepare_base_ptdf, reduce_static
from .solver import (
    CaseFlows,
    Instrumentation,
    SolveConfig,
    SolveResult,
    SparseReport,
    SplitAction,
    TaskDiagnostics,
    TopologyTask,
    candidate_case_flows,
    canonicalize_task,
    solve_batch,
)

__version__ = "0.1.0"
