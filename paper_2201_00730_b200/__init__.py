"""B200-native (sm_100a) implementation of the hot paths of arXiv 2201.00730.

Mirrors the reference package's public solver API (uotkit, src/__init__.py:10-70)
for the paths in SURVEY.md §8: TI/F-Sinkhorn, the 1-D OT oracle, batched 1-D
Frank-Wolfe, and the multimarginal barycenter.  All arithmetic runs in the
CUDA kernels of ``csrc/`` through the C-ABI declared in ``include/uot_b200.h``;
there is no CPU fallback.
"""

from .duality import (
    DualPair,
    UotProblem,
    dual_feasibility_violation,
    eval_F,
    eval_primal,
    updated_marginals,
    eval_G,
    eval_H,
    kl_scalars,
    lambda_star,
    translate,
)
from .entropies import (KL, Balanced, Berg, aprox, conj, conj_grad, conj_hess, divergence,
                        logdotexp, softmin)
from .exceptions import (
    InfeasibleDualError,
    MassBalanceError,
    NewtonError,
    SubmodularityError,
    UnsupportedEntropyError,
    UotError,
)
from .measures import (
    DiscreteMeasure,
    ExplicitMatrix,
    PowerDistance,
    SqEuclideanPoints,
    build_cost_matrix,
    cost_quadruple_diameter,
)
from .barycenter import (
    BarycenterProblem,
    MultiDual,
    MultiPlan,
    barycentric_cost_fn,
    dual_feasibility_exhaustive,
    extract_barycenter,
    fw_barycenter,
    fw_barycenter_batched,
    mot_certificate,
    mot_certify_batched,
    multimarginal_cost,
    multimarginal_lambda,
    plan_cost,
    solve_mot_1d,
    solve_mot_1d_batched,
)
from .certify import Certificate, assemble_certificate
from .fw import (AtomStore, FwConfig, feasibility_violation, fw_solve, fw_solve_batched,
                 line_search_h0, pfw_step, ternary_max)
from .ot1d import SparsePlan, check_complementary_slackness, solve_ot_1d, solve_ot_1d_batched
from .sinkhorn import (
    AndersonConfig,
    AndersonWindow,
    SinkhornConfig,
    SolverReport,
    anderson_weights,
    birkhoff_rate_bound,
    estimate_rate,
    f_sinkhorn_step,
    g_sinkhorn_step,
    h_optimality_residual,
    h_sinkhorn_step,
    run,
    sinkhorn_batched,
    verify_batched,
    write_trace_csv,
)
from .formats import (
    read_measure_csv,
    read_measure_json,
    read_multiplan_csv,
    read_plan_csv,
    write_gap_csv,
    write_measure_csv,
    write_measure_json,
    write_multiplan_csv,
    write_plan_csv,
)
from .synthetic import mixture_measure, uniform_measure

__version__ = "0.1.0"
