"""B200-native compress-and-eliminate (CE) factorization hot path.

Python mirror of the reference's public interface for this path
(``proj/include/ce/``): ``ce_factorize`` -> ``CEFactorization.solve`` used as
the preconditioner of a Krylov solve (``pcg`` here, with the ``minres``
contract of ``proj/include/ce/minres.hpp:46-47``).  Every call goes through
the C-ABI library ``libce_gpu.so`` (``include/ce_gpu.h``), which runs
hand-written sm_100a CUDA; there is no CPU fallback.
"""

from ._lib import lib, LibraryMissing  # noqa: F401
from .ce import (  # noqa: F401
    BlockSparseMatrix,
    BreakdownError,
    CoarseningPlan,
    CEFactorization,
    CompressionStrategy,
    Context,
    CsvTable,
    DeviceMatrix,
    FactorOptions,
    LocalShardComm,
    MinresOptions,
    PcgOptions,
    Problem,
    ShardComm,
    SolveReport,
    ce_factorize,
    ce_factorize_sharded,
    device_count,
    factor_stats_table,
    factor_summary_table,
    fmt_double,
    fmt_index,
    minres,
    pattern_coarsen,
    pattern_square,
    pcg,
    shard_plan_summary,
    solve_report_table,
    trace_table,
)

__all__ = [
    "BlockSparseMatrix",
    "BreakdownError",
    "CoarseningPlan",
    "CEFactorization",
    "CompressionStrategy",
    "Context",
    "CsvTable",
    "DeviceMatrix",
    "FactorOptions",
    "LocalShardComm",
    "MinresOptions",
    "PcgOptions",
    "Problem",
    "ShardComm",
    "SolveReport",
    "ce_factorize",
    "ce_factorize_sharded",
    "device_count",
    "factor_stats_table",
    "factor_summary_table",
    "fmt_double",
    "fmt_index",
    "minres",
    "pattern_coarsen",
    "pattern_square",
    "pcg",
    "shard_plan_summary",
    "solve_report_table",
    "trace_table",
]
