"""B200-native reconstruction hot path of arXiv 2102.08514 (splineplan drop-in).

Public API mirrors the reference package (/root/reference/pkg/src/splineplan):
lattice and coset construction, spline/plan selection, and the reconstruct call
`PlanInterpreter(plan).eval_batch(grid, pts)`, executed by hand-written sm_100a CUDA
kernels in libsplinerecon.so.
"""

from .lattice import (  # noqa: F401
    CoefficientIndex,
    CosetDecomposition,
    IntegerLattice,
    LatticeError,
    decompose_cartesian,
    format_lattice_file,
    named_lattice,
    parse_lattice_file,
    rho,
)
from .plan import (  # noqa: F401
    ClassTransform,
    EvaluationPlan,
    FetchGroup,
    PlanError,
    PlanKernel,
    PlanOptions,
    deserialize_plan,
    plan_from_dict,
    plan_to_dict,
    serialize_plan,
)
from .corpus import build_plan, load_plan, DIRECTION_SETS, CORPUS, REFERENCE_LOOKUPS  # noqa: F401
from .minilang import KernelProgram, build_program, emit_kernel, execute, parse_kernel  # noqa: F401
from .boxplan import box_spline_plan, compile_pp_plan, extract_pp_form  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # runtime pulls in torch; import lazily so plan/lattice tooling stays light
    if name in ("CoefficientGrid", "PlanInterpreter", "RuntimeError_", "eval_plan", "morton_order", "grid_extents"):
        from . import runtime

        return getattr(runtime, name)
    raise AttributeError(name)
