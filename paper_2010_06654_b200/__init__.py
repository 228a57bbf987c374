"""B200-native exact Lloyd k-means (the hot path of arXiv 2010.06654's UniK /
the reference package lloydkit), behind the reference's own entry points.

    from paper_2010_06654_b200 import run_lloyd, run_pruner, run_engine, KnobConfig

The compute runs in liblloydkit_b200.so (hand-written sm_100a CUDA behind the
C ABI in include/lloydkit_b200.h); there is no CPU fallback.
"""

from .core import ContractError, Counters, RunContext, make_init, sse
from .engine import BOUND_STRATEGIES, INDEX_MODES, KnobConfig, run_engine
from .lloyd import IterationStats, RunResult, run_lloyd
from .pruners import STRATEGIES, run_pruner
from .runlog import RunLog, read_runlogs, runlog_from_result, write_runlogs
from .harness import load_dataset, make_report, run_benchmark, summarize

__version__ = "0.1.0"

__all__ = [
    "BOUND_STRATEGIES",
    "ContractError",
    "Counters",
    "INDEX_MODES",
    "IterationStats",
    "KnobConfig",
    "RunContext",
    "RunLog",
    "RunResult",
    "STRATEGIES",
    "load_dataset",
    "make_init",
    "make_report",
    "read_runlogs",
    "run_engine",
    "run_lloyd",
    "run_benchmark",
    "run_pruner",
    "runlog_from_result",
    "sse",
    "summarize",
    "write_runlogs",
    "__version__",
]
