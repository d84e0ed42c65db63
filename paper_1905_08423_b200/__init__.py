"""B200-native Galerkin triple product C = P^T A P (arXiv 1905.08423).

Drop-in for the reference ``ptap`` package's triple-product path: the same
entry points and data model (int64/float64 CSR, 1D block-row DistMatrix),
with every symbolic and numeric phase executed by hand-written sm_100a CUDA
kernels behind a C ABI (include/ptap_b200.h).  PyTorch supplies device
buffers, streams and torch.distributed (NCCL over NVLink) only.
"""

from .comm import RankContext, RemoteRows, init_from_env, single_rank_context, spawn_ranks
from .device import DeviceCsr, DeviceLocalMatrix, DeviceOperands
from .errors import (AssemblyError, DeadlockError, DeviceError, MatrixMarketError, OwnershipError,
                     PartitionMismatchError, SizeCapError, StructuralDriftError)
from .ledger import MemoryLedger, PhaseTimer, PlanCounters
from .partition import (DistMatrix, LocalMatrix, NeighborList, RowPartition, assemble_global,
                        build_neighbor_list, dist_from_global, make_partition, owner, split_local)
from .hierarchy import GalerkinHierarchy, HierarchyLevel
from .matio import load_npz, read_matrix_market, save_npz, write_matrix_market
from .problems import model_problem_global, random_instance
from .sparse import CsrMatrix, RowAccumulator, RowSet, Triplet, csr_from_triplets, relative_difference, transpose
from .tripleproduct import (ALGORITHMS, ALL_AT_ONCE, CACHE_FREE, CACHE_KEEP, MERGED, TWO_STEP,
                            TripleProductPlan, aao_numeric, aao_symbolic, merged_numeric, merged_symbolic, ptap,
                            run_numeric, run_numeric_device, run_symbolic, two_step_numeric, two_step_symbolic)


def distribute(a: CsrMatrix, p: CsrMatrix, nranks: int, rank: int):
    """Split global (A, P) into one rank's operands (src/problems.py:147-154)."""
    row_part = make_partition(a.nrows, nranks)
    col_part = make_partition(p.ncols, nranks)
    return (dist_from_global(a, row_part, row_part, rank), dist_from_global(p, row_part, col_part, rank))


__version__ = "0.1.0"
