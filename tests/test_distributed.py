"""Multi-rank protocol (paper_2010_06654_b200.distributed) on CPU: world_size 2
over gloo, each rank holding a contiguous row shard.

The compute engine here is a CPU stand-in with the device's exact semantics
(per-dimension fixed-point scales from an all-reduced MAX exponent, int64
member-sum deltas of moved rows only, empty clusters keep their centroid);
assignments come from the oracle.  What is under test is the product's
sharding, bind-time MAX reduction, per-iteration SUM reduction, stop rule and
label gathering: the 2-rank run must equal the 1-rank run bit for bit and
follow the oracle's Lloyd trajectory.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_06654_b200.distributed import ShardedLloyd, gather_labels, shard_rows


class CpuFixedPointEngine:
    def __init__(self, x, k, n_total):
        self.x = np.ascontiguousarray(x, dtype=np.float64)
        self.n, self.d = self.x.shape
        self.k = k
        self.n_total = n_total

    def qexp(self):
        e = np.full(self.d + 1, -1100, dtype=np.int32)
        for z in range(self.d):
            m = np.max(np.abs(self.x[:, z])) if self.n else 0.0
            if m > 0:
                e[z] = math.frexp(m)[1]
        s = np.max(np.sum(self.x * self.x, axis=1)) if self.n else 0.0
        if s > 0:
            e[self.d] = math.frexp(s * (1 + 1e-9))[1]
        self._q = torch.from_numpy(e)
        return self._q

    def set_quant(self):
        lg = 0
        while (1 << lg) <= self.n_total:
            lg += 1
        B = 62 - lg
        e = np.where(self._q.numpy() < -1000, 0, self._q.numpy()).astype(np.int64)
        self.scale = np.ldexp(1.0, B - e)
        self.inv = np.ldexp(1.0, e - B)

    def set_centroids(self, init):
        self._done = False
        self._chg, self._sses = [], []
        self.c = np.array(init, dtype=np.float64, copy=True)
        self.labels_ = np.full(self.n, -1, dtype=np.int64)
        self.sums = np.zeros((self.k, self.d), dtype=np.int64)
        self.cnt = np.zeros(self.k, dtype=np.int64)
        self.qs = np.zeros(self.k, dtype=np.int64)

    def assign(self, t):
        from oracle import oracle as O
        if self._done:  # (the device's no-op iterations after convergence)
            self._delta = torch.zeros(self.k * self.d + 2 * self.k + 8, dtype=torch.int64)
            return self._delta
        new = O.assign_full(self.x, self.c, nthreads=1)[0] if self.n else np.empty(0, np.int64)
        moved = np.nonzero(new != self.labels_)[0]
        q = np.rint(self.x[moved] * self.scale[None, : self.d]).astype(np.int64)
        qq = np.rint(np.sum(self.x[moved] ** 2, axis=1) * self.scale[self.d]).astype(np.int64)
        ds = np.zeros((self.k, self.d), dtype=np.int64)
        dn = np.zeros(self.k, dtype=np.int64)
        dq = np.zeros(self.k, dtype=np.int64)
        for r, i in enumerate(moved):
            a, b = self.labels_[i], new[i]
            ds[b] += q[r]; dn[b] += 1; dq[b] += qq[r]
            if a >= 0:
                ds[a] -= q[r]; dn[a] -= 1; dq[a] -= qq[r]
        self.labels_ = new
        delta = np.concatenate([ds.ravel(), dn, dq, [len(moved)], np.zeros(7, np.int64)])
        self._delta = torch.from_numpy(delta)
        return self._delta

    def update(self, t):
        if self._done:
            self._chg.append(0)
            self._sses.append(self._sse)
            return
        kd, k = self.k * self.d, self.k
        dl = self._delta.numpy()
        self.sums += dl[:kd].reshape(self.k, self.d)
        self.cnt += dl[kd: kd + k]
        self.qs += dl[kd + k: kd + 2 * k]
        self._changed = int(dl[kd + 2 * k])
        nz = self.cnt > 0
        self.c[nz] = (self.sums[nz] * self.inv[None, : self.d]) / self.cnt[nz, None]
        sr = self.sums * self.inv[None, : self.d]
        self._sse = float(np.sum(np.where(nz, self.qs * self.inv[self.d]
                                          - np.sum(sr * sr, axis=1) / np.maximum(self.cnt, 1), 0)))
        self._chg.append(self._changed)
        self._sses.append(self._sse)
        self._done = self._changed == 0

    def changed_range(self, t0, t1):
        return list(self._chg[t0:t1])

    def sse_range(self, t0, t1):
        return list(self._sses[t0:t1])

    def centroids(self):
        return self.c.copy()

    def labels(self):
        return self.labels_.copy()


def _data():
    rng = np.random.default_rng(11)
    centres = rng.uniform(-5, 5, size=(6, 3))
    lab = rng.integers(0, 6, size=301)
    x = (centres[lab] + rng.normal(0, 0.7, size=(301, 3))).astype(np.float32).astype(np.float64)
    init = x[rng.choice(301, size=6, replace=False)].copy()
    return x, init


def _run(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, init = _data()
    r0, r1 = shard_rows(len(x), world, rank)
    eng = CpuFixedPointEngine(x[r0:r1], 6, len(x))
    drv = ShardedLloyd(eng)
    drv.bind()
    res = drv.run(init, 30)
    labels = gather_labels(res.local_labels)
    if rank == 0:
        np.savez(out_path, centroids=res.centroids, labels=labels, iters=res.iterations,
                 changed=np.array(res.changed), sse=np.array(res.sse))
    else:
        np.savez(out_path + f".r{rank}", centroids=res.centroids)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_rows_cover_and_balance():
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_rows(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


def test_two_ranks_equal_one_rank_and_follow_the_oracle(tmp_path, oracle):
    out2 = str(tmp_path / "w2.npz")
    mp.spawn(_run, args=(2, _free_port(), out2), nprocs=2, join=True)
    out1 = str(tmp_path / "w1.npz")
    mp.spawn(_run, args=(1, _free_port(), out1), nprocs=1, join=True)
    a, b = np.load(out2), np.load(out1)
    b_r1 = np.load(out2 + ".r1.npz")
    # exact integer reduction: identical centroids on every rank and at every world size
    assert np.array_equal(a["centroids"], b_r1["centroids"])
    assert np.array_equal(a["centroids"], b["centroids"])
    assert np.array_equal(a["labels"], b["labels"])
    assert int(a["iters"]) == int(b["iters"])
    assert np.array_equal(a["changed"], b["changed"])
    # and the trajectory is Lloyd's
    x, init = _data()
    ref = oracle.run_lloyd(x, 6, init, 30)
    assert int(a["iters"]) == ref["iterations"]
    assert np.array_equal(a["labels"], ref["labels"])
    assert np.allclose(a["centroids"], ref["centroids"], rtol=1e-9, atol=1e-12)
    assert a["changed"].tolist() == ref["changed"].tolist()
    assert np.allclose(a["sse"], ref["sse"], rtol=1e-9)
