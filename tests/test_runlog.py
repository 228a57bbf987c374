"""Run logs in the reference's JSONL schema (bench.py:129-209): the drop-in
reads the reference's own lines (tests/golden/runlog_ref.jsonl, written by
lloydkit) and writes lines with the same keys and value types."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

REF = os.path.join(GOLDEN, "runlog_ref.jsonl")


def test_reads_reference_runlogs():
    from paper_2010_06654_b200.runlog import read_runlogs
    logs = read_runlogs(REF)
    assert [lg.label for lg in logs] == ["lloyd", "hamerly"]
    assert all(lg.schema_version == 1 for lg in logs)


def test_totals_check_rejects_tampering(tmp_path):
    from paper_2010_06654_b200.core import ContractError
    from paper_2010_06654_b200.runlog import read_runlogs
    obj = json.loads(open(REF).readline())
    obj["totals"]["dist_comps"] += 1
    p = tmp_path / "bad.jsonl"
    p.write_text(json.dumps(obj) + "\n")
    with pytest.raises(ContractError):
        read_runlogs(str(p))


def _schema(obj):
    """Key structure and value types of a run-log line."""
    if isinstance(obj, dict):
        return {k: _schema(v) for k, v in obj.items()}
    if isinstance(obj, list):
        return [_schema(obj[0])] if obj else []
    return type(obj).__name__


@pytest.mark.gpu
def test_gpu_runlog_has_reference_schema(tmp_path):
    import paper_2010_06654_b200 as lk
    from paper_2010_06654_b200.runlog import read_runlogs, runlog_from_result, write_runlogs
    ref = json.loads(open(REF).readlines()[1])
    rng = np.random.default_rng(3)
    data = (rng.normal(size=(300, 4)) + rng.integers(0, 6, size=(300, 1))).astype(np.float64)
    cfg = lk.KnobConfig(bound_strategy="hamerly", t_max=6)
    init = lk.make_init(lk.RunContext(seed=1), data, 6, "random")
    res = lk.run_engine(data, 6, cfg, init=init)
    log = runlog_from_result(res, dataset_id="gauss300", n=300, d=4, k=6, config=cfg, init_seed=1)
    path = tmp_path / "gpu.jsonl"
    write_runlogs(str(path), [log])
    got = json.loads(path.read_text())
    for key in ("run_id", "footprint_bytes_estimate", "error"):
        got.pop(key)
        ref.pop(key)
    assert _schema(got) == _schema(ref)
    assert read_runlogs(str(path))[0].label == "hamerly"
