"""Generate tests/golden/runlog_ref.jsonl with the REFERENCE harness
(run in the build container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_runlog_golden.py

Two run-log lines (Lloyd and Hamerly) for a small gen_gaussian dataset, written
by lloydkit's own runlog_from_result / write_runlogs (bench.py:181-209)."""
import os

from lloydkit import KnobConfig, RunContext, make_init, run_engine
from lloydkit.bench import gen_gaussian, runlog_from_result, write_runlogs

HERE = os.path.dirname(os.path.abspath(__file__))
data, _ = gen_gaussian(300, 4, 6, 0.05, seed=3)
k = 6
init = make_init(RunContext(seed=1), data, k)
logs = []
for strat in ("none", "hamerly"):
    cfg = KnobConfig(bound_strategy=strat, t_max=6)
    res = run_engine(data, k, cfg, init=init, ctx=RunContext(seed=1))
    logs.append(runlog_from_result(res, dataset_id="gauss300", n=300, d=4, k=k, config=cfg,
                                   init_seed=1))
write_runlogs(os.path.join(HERE, "runlog_ref.jsonl"), logs)
print("wrote", len(logs))
