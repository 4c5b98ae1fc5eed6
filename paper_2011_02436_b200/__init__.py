"""B200-native (sm_100a) RBP-ELM training hot path (arXiv 2011.02436).

The reference's train/predict API (proj/include/rbpelm) re-exposed over a C ABI
to hand-written FP64 tensor-core (DMMA) kernels.  See DESIGN.md.
"""
from .api import (  # noqa: F401
    ColumnPermutation,
    Context,
    DeviceError,
    ElmModel,
    ElmParams,
    HiddenLayer,
    NotSupportedError,
    RankRevealingFactor,
    ShapeError,
    SingularMatrix,
    SingularSplit,
    SolveDiagnostics,
    SolverStrategy,
    accuracy,
    accuracy_stage_device,
    apply_permutation,
    context,
    duplicate_nodes,
    gram,
    gram_device,
    gram_stage_device,
    hidden_matrix,
    init_hidden,
    invert_permutation_rows,
    pinv_svd,
    predict,
    pseudo_inverse,
    pseudo_inverse_stage_device,
    rank_revealing_factor,
    rank_revealing_permutation,
    solve_beta,
    solve_direct,
    solve_factored_gram,
    solve_spd,
    solve_stage_device,
    synth_classification,
    synth_rank_deficient,
    train,
    train_device,
)

__all__ = [n for n in dir() if not n.startswith("_")]
