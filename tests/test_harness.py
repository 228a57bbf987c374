"""Harness integration (harness.py; reference bench.py:30-58, :249-349): the
.npy loader beside the text loader, the sweep driver's aggregation and report
on CPU; GPU cells of the sweep in test_gpu_harness below."""

import numpy as np
import pytest

from paper_2010_06654_b200 import ContractError, KnobConfig
from paper_2010_06654_b200.harness import load_dataset, make_report, save_dataset, summarize
from paper_2010_06654_b200.runlog import RunLog


def test_npy_round_trip(tmp_path):
    x = np.random.default_rng(0).normal(size=(50, 3)).astype(np.float32)
    p = str(tmp_path / "x.npy")
    save_dataset(p, x.astype(np.float64))
    assert np.load(p).dtype == np.float32          # exact float32 data stays float32 on disk
    y = load_dataset(p)
    assert y.dtype == np.float64 and np.array_equal(y, x.astype(np.float64))


def test_npy_rejects_bad_arrays(tmp_path):
    p = str(tmp_path / "bad.npy")
    a = np.ones((4, 2))
    a[2, 1] = np.nan
    np.save(p, a)
    with pytest.raises(ContractError, match="row 3"):
        load_dataset(p)
    np.save(p, np.ones(5))
    with pytest.raises(ContractError):
        load_dataset(p)


def test_text_loader_matches_reference_errors(tmp_path):
    p = tmp_path / "x.csv"
    p.write_text("1,2\n3,4\n\n5,6\n")
    assert load_dataset(str(p)).tolist() == [[1, 2], [3, 4], [5, 6]]
    p.write_text("1 2\n3 4 5\n")
    with pytest.raises(ContractError, match="row 2: expected 2 columns"):
        load_dataset(str(p))
    p.write_text("1,x\n")
    with pytest.raises(ContractError, match="row 1"):
        load_dataset(str(p))


def _log(label, cell, wall, power):
    it = {"iter": 1, "wall_nanos": wall, "dist_comps": 10, "data_accesses": 11,
          "bound_accesses": 0, "bound_updates": 0, "pruning_power": power, "sse": 1.0}
    return RunLog(run_id=f"{label}-{cell}", dataset_id=cell[0], n=10, d=2, k=cell[1],
                  config=KnobConfig(bound_strategy=label if label != "lloyd" else "none").__dict__,
                  init_seed=cell[2], iterations=[it],
                  totals={"wall_nanos": wall, "dist_comps": 10, "data_accesses": 11,
                          "bound_accesses": 0, "bound_updates": 0})


def test_report_speedups_against_lloyd_in_the_same_cell():
    logs = [_log("lloyd", ("a", 4, 0), 1000, 0.0), _log("hamerly", ("a", 4, 0), 250, 0.5),
            _log("lloyd", ("b", 4, 0), 2000, 0.0), _log("hamerly", ("b", 4, 0), 1000, 0.3)]
    s = summarize(logs)
    assert s["hamerly"]["mean_speedup"] == pytest.approx(3.0)
    assert s["hamerly"]["median_speedup"] == pytest.approx(3.0)
    rows = make_report(logs)
    assert [r["label"] for r in rows] == ["hamerly", "lloyd"]
    with pytest.raises(ContractError):
        make_report([])


@pytest.mark.gpu
def test_gpu_sweep_cells(tmp_path):
    """run_benchmark on the GPU: Lloyd anchors every cell, bounded strategies
    report speedups and pruning power, tree index modes are failed cells, and
    the logs round-trip through the schema-v1 JSONL."""
    from paper_2010_06654_b200 import read_runlogs, write_runlogs
    from paper_2010_06654_b200 import datasets
    from paper_2010_06654_b200.harness import run_benchmark
    x = datasets.generate("cfg1", 30000)
    p = str(tmp_path / "cfg1.npy")
    save_dataset(p, x)
    data = load_dataset(p)
    cfgs = [KnobConfig(bound_strategy=s, t_max=15) for s in ("hamerly", "yinyang", "elkan")]
    cfgs.append(KnobConfig(index_mode="pure", t_max=15))
    logs, summary = run_benchmark([("cfg1", data)], [50, 100], cfgs, seeds=(0, 1),
                                  init_method="random", validate=True)
    assert summary["lloyd"]["runs"] == 4 and summary["lloyd"]["failed"] == 0
    for s in ("hamerly", "yinyang", "elkan"):
        assert summary[s]["failed"] == 0
        assert summary[s]["mean_speedup"] == summary[s]["mean_speedup"]  # (not NaN)
        assert summary[s]["mean_pruning_power"] > 0.0
    assert summary["ball-pure"]["failed"] == 4
    out = str(tmp_path / "logs.jsonl")
    write_runlogs(out, [g for g in logs if g.error is None])
    back = read_runlogs(out)
    assert len(back) == 16
    rows = make_report(back)
    assert {r["label"] for r in rows} == {"lloyd", "hamerly", "yinyang", "elkan"}
