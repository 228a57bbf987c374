#!/usr/bin/env python
"""Group-tile worklist statistics of one cfg5-like trajectory: how many
(row tile, group tile) products the pass evaluates with the current order
(rows sorted by label) against orders that also sort by the rows' group masks
inside a label.  Debug tool (reads the internal worklist records).

    python tools/tile_stats.py cfg5 12 0
"""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def tiles(mask, torch):
    """sum over 128-row tiles of popcount(OR of the tile's masks)"""
    m = mask.numel()
    pad = (-m) % 128
    if pad:
        mask = torch.cat([mask, torch.zeros(pad, dtype=mask.dtype, device=mask.device)])
    mt = mask.view(-1, 128)
    tot = 0
    for b in range(32):
        tot += int(((mt >> b) & 1).amax(dim=1).sum())
    return tot


def main():
    import torch

    from paper_2010_06654_b200 import _native as nat
    from paper_2010_06654_b200 import datasets
    from paper_2010_06654_b200.core import RunContext, init_random
    from paper_2010_06654_b200.device import DeviceLloyd
    from paper_2010_06654_b200.pruners import gpu_groups

    wl, T, n_rows = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) or None
    cfg = datasets.CONFIGS[wl]
    x = datasets.generate(wl, n_rows)
    init = init_random(RunContext(seed=cfg.seed_init), x, cfg.k)
    n, k = x.shape[0], cfg.k
    g = gpu_groups("yinyang", n, k, cfg.d)
    eng = DeviceLloyd(x, k, "yinyang", T, kernel="auto", groups=g, group_seed=cfg.seed_init,
                      record_history=False)
    eng.set_centroids(init)
    off, size = ctypes.c_uint64(), ctypes.c_uint64()
    nat.check(eng.lib.lk_buffer(eng.ctx, 1000, ctypes.byref(off), ctypes.byref(size)), "lk_buffer")
    meta = eng.ws[off.value: off.value + size.value].view(torch.int32).view(-1, 8)
    for t in range(1, T + 1):
        lab0 = eng.labels.clone()
        eng.step(t)
        torch.cuda.synchronize()
        s = eng.stats[t - 1].to("cpu").numpy()
        m = int(s[3])
        if t < 7 or m == 0:
            continue
        row = meta[:m, 6].long()
        mask = meta[:m, 7].long() & 0xFFFFFFFF
        lab = lab0[row].long()
        own = 0
        for b in range(32):
            own += int(((mask >> b) & 1).sum())
        out = {"t": t, "listed": m, "dist_tiles": int(s[4]) // (128 * 128), "row_groups": own,
               "rows_x_tiles_now": tiles(mask, torch)}
        pc = torch.zeros_like(mask)
        for b in range(32):
            pc += (mask >> b) & 1
        for name, key in (("label_mask", lab * (1 << 32) + mask),
                          ("label_popc_mask", (lab * 64 + pc) * (1 << 32) + mask)):
            order = torch.argsort(key)
            out["rows_x_tiles_" + name] = tiles(mask[order], torch)
        # coarse second keys a counting sort could take
        gof = eng._view("group_of", torch.int32, (k,)).long()
        cnt = torch.bincount(lab, minlength=k).double()
        F = torch.stack([torch.bincount(lab, weights=((mask >> b) & 1).double(), minlength=k)
                         for b in range(32)], dim=1)          # [k, 32]
        F[torch.arange(k, device=F.device), gof] = 0.0        # own group: always set
        pfr = F / cnt.clamp(min=1).unsqueeze(1)
        score = 1.0 - (1.0 - pfr) ** 128 - pfr
        for nb in (2, 3, 4, 5):
            bits = torch.topk(score, nb, dim=1).indices      # [k, nb]
            kb = torch.zeros_like(mask)
            for j in range(nb):
                kb |= ((mask >> bits[lab, j]) & 1) << j
            order = torch.argsort(lab * 64 + kb, stable=True)
            out[f"score_top{nb}"] = tiles(mask[order], torch)
        for B in (8, 16):
            hb = ((mask * 2654435761) >> 13) % B
            order = torch.argsort(lab * 64 + hb, stable=True)
            out[f"hash{B}"] = tiles(mask[order], torch)
        # popcount buckets (1, 2, 3, 4, 5-6, 7+ groups)
        pb = torch.clamp(pc, max=8)
        order = torch.argsort(lab * 64 + pb, stable=True)
        out["popc_bucket"] = tiles(mask[order], torch)
        # histogram of popcounts
        out["popc_hist"] = torch.bincount(pc, minlength=33)[:12].tolist()
        print(json.dumps(out), flush=True)
        del row, mask, lab, pc
    eng.close()


if __name__ == "__main__":
    main()
