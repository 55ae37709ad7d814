"""B200-native D3M factorisation hot path (arXiv 2002.05018).

Drop-in for the hot-path API of the reference package ``ddsolve``
(pkg/src/ddsolve/__init__.py:10-39): Schur reduction of the subdomains,
assembly of the block-sparse interface matrix, restricted-Bunch-Kaufman
block LDL^T, block substitution and primal recovery, computed by
hand-written sm_100a kernels in libd3m.so (no CPU fallback).
"""

from ._lib import D3MError, D3MUnavailable
from .blockmat import BlockMatrixError, BlockSparseSym, CliqueGraph, clique_graph, from_blocks, load_blk, \
    save_blk
from .device import DeviceArray
from .factor import DEFAULT_PIVOT_TOL, BlockFactor, DenseFactor, FactorConsistencyError, FactorStats, \
    SingularBlockError, block_ldlt, block_solve, dense_ldlt_bk, scatter_factor
from .ordering import Ordering, OrderingError, identity_ordering, load_ordering_file, reorder
from .subdomain import Coupling, ReducedSystem, SingularDomainError, SolverStateError, SubdomainSystem, \
    assemble_reduced, interface_lambda_nodes, recover_primal, reduce_domain, reduce_domains
from .symbolic import EliminationPlan, fill_blocks, format_plan, symbolic_factor

__version__ = "0.1.0"

BK_ALPHA = (1.0 + 17.0 ** 0.5) / 8.0      # kernels.py:33

__all__ = [
    "BK_ALPHA", "BlockFactor", "BlockMatrixError", "BlockSparseSym", "CliqueGraph", "Coupling",
    "D3MError", "D3MUnavailable", "DEFAULT_PIVOT_TOL", "DenseFactor", "DeviceArray", "EliminationPlan",
    "FactorConsistencyError", "FactorStats", "Ordering", "OrderingError", "ReducedSystem",
    "SingularBlockError", "SingularDomainError", "SolverStateError", "SubdomainSystem",
    "assemble_reduced", "block_ldlt", "block_solve", "clique_graph", "dense_ldlt_bk", "fill_blocks",
    "format_plan", "from_blocks", "identity_ordering", "interface_lambda_nodes", "load_blk",
    "load_ordering_file", "recover_primal", "reduce_domain", "reduce_domains", "reorder", "save_blk",
    "scatter_factor", "symbolic_factor",
]
