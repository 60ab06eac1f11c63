"""B200-native TOCAB (GraphCage, arXiv 1904.02241) graph engine.

Drop-in for the reference package ``gcb``'s hot path: same module layout
(graph, blocking, kernels, traversal, util) and call signatures, with every
compute step running as hand-written sm_100a CUDA in libgcb_b200.so.
"""

from . import _lib
from .blocking import (
    DEFAULT_BLOCK_WIDTH,
    BlockedGraph,
    BlockStats,
    SubgraphBlock,
    block_stats,
    num_blocks_for,
    partition_cb,
    partition_tocab,
    read_gcb,
    width_for_l2,
    write_gcb,
)
from .components import CcResult, cc
from .graph import (
    CsrGraph,
    GraphCapacityError,
    GraphFormatError,
    GraphGenSpec,
    from_edges,
    generate,
    generate_rmat,
    load_edge_list,
    load_graph,
    load_matrix_market,
    symmetrize,
    transpose,
    write_edge_list,
)
from .kernels import (
    PrParams,
    PrResult,
    ScheduleStrategy,
    VertexValueSet,
    accumulate_ranges,
    compute_contributions,
    pr_baseline,
    pr_blocked,
    process_block_pull,
    process_block_push,
    segment_row_sums,
    spmv,
    spmv_blocked,
)
from .traversal import (
    INF_DEPTH,
    INF_DIST,
    BcResult,
    BfsResult,
    DirectionPolicy,
    SsspResult,
    TraversalState,
    bc,
    bc_backward,
    bc_single_source,
    bfs,
    choose_direction,
    forward_pull_step,
    forward_push_step,
    sample_sources,
    sssp,
)
from .util import parse_size, result_checksum

__version__ = "0.1.0"
