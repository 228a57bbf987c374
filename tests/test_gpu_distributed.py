"""The sharded protocol on the real CUDA engine: two ranks on the one GPU of
the box, exchanging the int64 delta buffer through gloo (host-staged; no
kernel of one rank ever waits on the other).  Centroids must be bit-identical
to the single-process run and the trajectory must be the oracle's."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_2010_06654_b200 import datasets
    from paper_2010_06654_b200.core import RunContext, init_random
    x = datasets.generate("cfg1", 20000)
    init = init_random(RunContext(seed=7), x, 64)
    return x, init


def _rank(rank, world, port, strategy, out, backend="gloo"):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    # gloo: every rank on the box's one GPU (host-staged exchange); nccl: one
    # GPU per rank
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2010_06654_b200.device import DeviceLloyd
    from paper_2010_06654_b200.distributed import (DeviceEngine, ShardedLloyd, gather_labels,
                                                   shard_rows)
    x, init = _case()
    r0, r1 = shard_rows(len(x), world, rank)
    eng = DeviceLloyd(x[r0:r1], 64, strategy, 40, n_total=len(x), record_history=False,
                      groups=7 if strategy == "yinyang" else 0, comm=dist.group.WORLD)
    drv = ShardedLloyd(DeviceEngine(eng), group=dist.group.WORLD)
    drv.bind()
    res = drv.run(init, 40)
    labels = gather_labels(res.local_labels)
    np.savez(out + f".r{rank}.npz", centroids=res.centroids, labels=labels,
             iters=res.iterations, changed=np.array(res.changed),
             graphed=bool(getattr(eng, "graph_ready", False)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("strategy", ["lloyd", "hamerly", "yinyang"])
def test_two_ranks_on_device_match_one_rank(tmp_path, oracle, strategy):
    out2, out1 = str(tmp_path / "w2"), str(tmp_path / "w1")
    mp.spawn(_rank, args=(2, _free_port(), strategy, out2), nprocs=2, join=True)
    mp.spawn(_rank, args=(1, _free_port(), strategy, out1), nprocs=1, join=True)
    a0, a1, b = (np.load(out2 + ".r0.npz"), np.load(out2 + ".r1.npz"), np.load(out1 + ".r0.npz"))
    assert np.array_equal(a0["centroids"], a1["centroids"])
    assert np.array_equal(a0["centroids"], b["centroids"])
    assert np.array_equal(a0["labels"], b["labels"])
    assert int(a0["iters"]) == int(b["iters"])
    x, init = _case()
    ref = oracle.run_lloyd(x, 64, init, 40)
    assert int(a0["iters"]) == ref["iterations"]
    assert a0["changed"].tolist() == ref["changed"].tolist()
    assert np.all(np.abs(a0["centroids"] - ref["centroids"])
                  <= 1e-5 * np.abs(ref["centroids"]) + 1e-9 * np.abs(x).max())


def _check_against(out, ref_out, oracle, world):
    parts = [np.load(out + f".r{r}.npz") for r in range(world)]
    b = np.load(ref_out + ".r0.npz")
    for p in parts:
        assert np.array_equal(p["centroids"], b["centroids"])
    assert np.array_equal(parts[0]["labels"], b["labels"])
    assert int(parts[0]["iters"]) == int(b["iters"])
    x, init = _case()
    ref = oracle.run_lloyd(x, 64, init, 40)
    assert int(parts[0]["iters"]) == ref["iterations"]
    assert parts[0]["changed"].tolist() == ref["changed"].tolist()
    return parts


@pytest.mark.parametrize("strategy", ["lloyd", "yinyang"])
def test_nccl_graph_captured_protocol_single_gpu(tmp_path, oracle, strategy):
    """One rank over NCCL on the box's GPU: the iteration (assign, NCCL
    all-reduce of the delta payload, update) is captured as one CUDA graph and
    replayed without a host sync per iteration; the result equals the gloo
    (eager) protocol bit for bit and the oracle's trajectory."""
    out_n, out_g = str(tmp_path / "nccl"), str(tmp_path / "gloo")
    mp.spawn(_rank, args=(1, _free_port(), strategy, out_n, "nccl"), nprocs=1, join=True)
    mp.spawn(_rank, args=(1, _free_port(), strategy, out_g, "gloo"), nprocs=1, join=True)
    parts = _check_against(out_n, out_g, oracle, 1)
    assert bool(parts[0]["graphed"]), "the NCCL iteration was not graph-captured"


@pytest.mark.skipif(not __import__("torch").cuda.is_available()
                    or __import__("torch").cuda.device_count() < 2,
                    reason="needs >= 2 GPUs (one NCCL rank per GPU)")
@pytest.mark.parametrize("strategy", ["lloyd", "hamerly", "yinyang"])
def test_two_nccl_ranks_match_one_rank(tmp_path, oracle, strategy):
    out2, out1 = str(tmp_path / "n2"), str(tmp_path / "n1")
    mp.spawn(_rank, args=(2, _free_port(), strategy, out2, "nccl"), nprocs=2, join=True)
    mp.spawn(_rank, args=(1, _free_port(), strategy, out1, "gloo"), nprocs=1, join=True)
    _check_against(out2, out1, oracle, 2)
