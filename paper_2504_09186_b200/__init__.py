"""B200-native tensor-network-contraction engine (hot path of arXiv 2504.09186).

Drop-in for the reference package ``tncsim``'s public API
(``pkg/src/tncsim/__init__.py:17-60``): the same names and semantics, with the
numeric hot path -- permutation, pairwise contraction, split-K, step fusion,
slice accumulation -- running in hand-written sm_100a CUDA kernels behind the
C-ABI of ``include/tnc_b200.h`` (``libtnc_b200.so``).  Host planning (paths,
slicing, reuse programs) is integer logic in Python that reproduces the
reference's choices exactly.
"""

from .errors import (
    CircuitParseError,
    ContractionError,
    DeviceError,
    InvalidPermutationError,
    MemoryBudgetError,
    NetworkError,
    PlanningError,
    SlicingError,
    TensorError,
    TncError,
)
from .labels import Index, PermutationPlan, classify_permutation
from .tensor import DenseTensor, permute, project
from .contract import (
    ContractionShape,
    contract_pair,
    contraction_permutations,
    contraction_shape,
    multiply_cost,
    split_common_contract,
    ttgt_plan,
)
from .network import TensorNetwork
from .circuit import Circuit, Gate, circuit_to_network, gate_matrix, open_output_order, parse_circuit
from .tree import ContractionTree, LinearSchedule, TreeMetrics, greedy_path, linearize, tree_metrics
from .slicing import (
    Lifetime,
    SliceEntry,
    SliceSpec,
    branch_exchange_nest,
    compute_lifetimes,
    index_overhead,
    select_slices,
    slicing_overhead,
)
from .reuse import (
    ReuseAction,
    ReusePlanReport,
    ReuseSchedule,
    choose_reuse_subset,
    interpret,
    plan_spindle,
    plan_tree_reuse,
    tune_memory,
)

__version__ = "0.1.0"


def __getattr__(name):
    # the executor imports torch.distributed lazily; keep `import` cheap
    if name in {"ReductionTopology", "RunResult", "RunStats", "hierarchical_reduce", "run_direct",
                "run_reuse", "run_reuse_open", "run_sliced", "run_open", "SliceExecutor", "read_partials",
                "write_partials"}:
        from . import execute

        return getattr(execute, name)
    raise AttributeError(name)
