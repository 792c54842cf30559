"""tensortrack_b200 — B200-native online tensor-subspace tracking for
dynamic MRI (arXiv 1609.04104), a drop-in for the hot path of the reference
package ``tensortrack`` (`pkg/src/tensortrack/__init__.py:3-62`).

The public names mirror the reference modules; the arithmetic runs in the
sm_100a CUDA library ``libtensortrack_b200.so`` (C ABI in
``include/tensortrack_b200.h``). There is no CPU fallback: importing works
anywhere, but every compute call needs a CUDA device and the built library.
"""

from . import checkpoint
from .core import (TensorSubspace, outer_rank_one, rank_surrogate, rebalance, refold, singular_values,
                   synthesize_slice, unfold)
from .engine import (AdaptiveSchedule, BatchResult, EntryEngine, Informative, InformativeEntries, LocalShardedEngine, OnlineEngine,
                     OnlineResult, RowShardedEngine, StaticEntries, StaticRows, run_batch, run_online, warm_up)
from .mri import FrameEstimate, PatchGrid, interp_track_step, patch_assemble, patch_partition, reconstruct_frame
from .observation import (
    EntryMask,
    FourierMask,
    MeasurementBatch,
    build_phi,
    row_distances,
    rows_to_entries,
    unitary_dft2,
    unitary_dft_matrix,
    variable_density_rows,
    weighted_draw_without_replacement,
)
from .sampler import (
    SamplePlan,
    SamplingDistribution,
    adaptive_step,
    draw_samples,
    entry_scores,
    expected_count_trace,
    expected_sample_count,
    row_scores,
)
from .tracker import (
    Fixed,
    HessianBound,
    StepConfig,
    StepReport,
    TrackerState,
    empirical_cost,
    empirical_cost_gradient,
    factor_gradient,
    hessian_bound,
    init_state,
    instantaneous_cost,
    random_subspace,
    run,
    solve_gamma,
    track_step,
)
from ._lib import NumericalError
from .config import ConfigError
from .metrics import nmse, nmse_frames
from .acquisition import StreamingProvider, measure, project
from .patches import PatchedResult, draw_frame_entries, full_entries, init_patch_factors, run_tracking_patched
from .cten import CtenFormatError, read_cten, read_cten_tensor, write_cten
from .reports import (MetricRow, online_budget_rows, online_mask_rows, write_budget_csv, write_mask_csv,
                      write_manifest, write_metrics_csv, write_trace_csv)

__all__ = [
    "TensorSubspace", "rebalance", "synthesize_slice", "outer_rank_one", "singular_values", "rank_surrogate",
    "unfold", "refold",
    "EntryMask", "FourierMask", "MeasurementBatch", "build_phi", "row_distances", "rows_to_entries",
    "unitary_dft2", "unitary_dft_matrix", "variable_density_rows", "weighted_draw_without_replacement",
    "Fixed", "HessianBound", "StepConfig", "StepReport", "TrackerState", "init_state", "random_subspace",
    "run", "solve_gamma", "track_step", "factor_gradient", "hessian_bound", "instantaneous_cost",
    "empirical_cost", "empirical_cost_gradient",
    "SamplePlan", "SamplingDistribution", "adaptive_step", "draw_samples", "entry_scores",
    "expected_count_trace", "expected_sample_count", "row_scores",
    "FrameEstimate", "interp_track_step", "reconstruct_frame", "PatchGrid", "patch_partition", "patch_assemble",
    "PatchedResult", "run_tracking_patched", "init_patch_factors", "draw_frame_entries", "full_entries",
    "OnlineEngine", "OnlineResult", "StaticRows", "Informative", "AdaptiveSchedule", "run_online", "warm_up", "RowShardedEngine",
    "EntryEngine", "InformativeEntries", "StaticEntries", "run_batch", "BatchResult", "LocalShardedEngine",
    "NumericalError", "ConfigError", "nmse", "nmse_frames", "StreamingProvider", "measure", "project",
    "CtenFormatError", "read_cten", "read_cten_tensor", "write_cten",
    "MetricRow", "write_metrics_csv", "write_mask_csv", "write_trace_csv", "write_budget_csv",
    "online_mask_rows", "online_budget_rows", "write_manifest", "checkpoint",
]
