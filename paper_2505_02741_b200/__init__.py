"""B200-native dyGRASS batched incremental / decremental sparsifier update.

The device path (libdyg.so: hand-written sm_100a CUDA behind the C-ABI in
include/dyg.h) is the product; this package is the host-side mirror of the
reference's interface (see api.py). There is no CPU fallback.
"""
from .api import (  # noqa: F401
    BatchReport,
    DeletionOutcome,
    DynamicGraph,
    Error,
    ErrorKind,
    Decision,
    InsertionDecision,
    SparsifierOptions,
    SparsifierState,
    StreamGenOptions,
    UpdateReport,
    UpdateStream,
    WalkConfig,
    build_initial_sparsifier,
    build_initial_sparsifier_gpu,
    device_count,
    generate_update_stream,
    generate_update_stream_gpu,
    load_matrix_market,
    load_update_stream,
    make_grid4,
    make_mesh,
    make_random_connected,
    run_batch,
    save_matrix_market,
    save_update_stream,
)
from .spectral import (  # noqa: F401,E402
    ConditionEstimate,
    ConditionMethod,
    ConditionOptions,
    PcgResult,
    calibrate_budget,
    condition_number,
    pcg_solve,
    random_rhs,
)
