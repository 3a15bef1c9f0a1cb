"""B200-native big-data MDS (interpolation, divide-and-conquer, fast MDS).

Drop-in for the hot path of the reference ``scalemds`` package: same public
names, arguments and exceptions; all arithmetic runs in libmdsx.so
(hand-written sm_100a CUDA behind the C-ABI in include/mdsx.h).
"""

from .algorithms import (DivideRun, FastRun, InterpolationRun, divide_and_conquer_mds,
                         fast_mds, interpolation_mds, run_algorithm)
from .dataio import (IdxImageSet, load_idx_images, read_csv_matrix, read_idx_images,
                     read_idx_labels)
from .errors import (DegenerateRankError, FormatError, InvalidInputError, JoinError, MdsError,
                     MetricError, NumericalError, ParamError, ShapeError, UsageError)
from .params import (ALGORITHM_NAMES, EXACT_SIZE_GUARD, AlgorithmParams)
from .plans import (DcPlan, FastNode, FastPlan, FastStats, InterpPlan, fast_stats,
                    plan_divide_conquer, plan_fast, plan_interpolation, spawned_generator,
                    sub_seed)
from .primitives import (apply_procrustes, classical_mds, classical_mds_from_data,
                         cross_squared_distances, double_center, euclidean_distance_matrix,
                         fit_procrustes, gof_breakdown, goodness_of_fit, gower_context,
                         gower_interpolate)
from .simulation import aligned_correlations, g1_curve, gof_sweep
from .results import (EigenSystem, GofBreakdown, GowerContext, MdsConfiguration,
                      ProcrustesTransform)

__version__ = "0.1.0"

__all__ = [
    "ALGORITHM_NAMES", "AlgorithmParams", "DcPlan", "DegenerateRankError", "DivideRun",
    "EXACT_SIZE_GUARD", "EigenSystem", "FastNode", "FastPlan", "FastRun", "FastStats",
    "FormatError", "GofBreakdown", "GowerContext", "InterpPlan", "InterpolationRun",
    "InvalidInputError", "JoinError", "MdsConfiguration", "MdsError", "MetricError",
    "NumericalError", "ParamError", "ProcrustesTransform", "ShapeError", "UsageError",
    "apply_procrustes", "classical_mds", "classical_mds_from_data", "cross_squared_distances",
    "divide_and_conquer_mds", "double_center", "euclidean_distance_matrix", "fast_mds",
    "fast_stats", "fit_procrustes", "gof_breakdown", "goodness_of_fit", "gower_context",
    "gower_interpolate", "interpolation_mds", "plan_divide_conquer", "plan_fast",
    "plan_interpolation", "run_algorithm", "spawned_generator", "sub_seed",
    "IdxImageSet", "load_idx_images", "read_csv_matrix", "read_idx_images", "read_idx_labels",
    "aligned_correlations", "g1_curve", "gof_sweep",
]
