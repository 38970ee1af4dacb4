"""CPU, world size 2 (gloo): the period-shard host logic.

Each rank owns a contiguous period range, builds its local view of the
global problem through the shard index maps, and exchanges exactly the halo
the device path needs (boundary set-points both ways, boundary-row sigma_s
backward) with torch.distributed send/recv.  Checked against the bit-exact
oracle's global problem: the received halo equals the global values and every
owned ramp row (including the boundary row of step t0) evaluates to the global
constraint value from local data alone."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_14032_b200.shard import ShardMap, partition


def test_partition():
    assert partition(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert partition(96 * 8, 8)[-1] == (672, 96)
    assert sum(T for _, T in partition(97, 8)) == 97
    with pytest.raises(ValueError):
        partition(2, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, T_total, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    from helpers import golden_network, interior_point, sigmas
    from oracle import bindings as B
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        net = golden_network("synth")
        scale = np.ones((T_total, net.n_load))
        orc = B.OracleModel(net, T_total, scale)
        xl, xu, xs, _, _ = orc.bounds()
        x = interior_point(xl, xu, xs, 7)
        ok, g, _ = orc.eval_g(x)
        assert ok
        _, ss = sigmas(1, orc.sizes[1], 8)
        ramp_gens = np.nonzero(np.isfinite(net.gen_ramp))[0]
        t0, T = partition(T_total, world)[rank]
        mp_ = ShardMap(net.n_bus, net.n_line, net.n_gen, int(np.isfinite(net.line_smax).sum()),
                       ramp_gens, T_total, t0, T)
        vg, rg = mp_.var_global(), mp_.row_global()
        xl_ = x[vg].copy()
        sl_ = ss[rg].copy()
        xl_[mp_.ghost_prev()] = np.nan
        xl_[mp_.ghost_next()] = np.nan
        sl_[mp_.ghost_rows()] = np.nan
        # ---- halo exchange: the function bench.py runs over NCCL, here over gloo
        from paper_2405_14032_b200.shard import exchange_halo
        xt, st = torch.from_numpy(xl_), torch.from_numpy(sl_)
        exchange_halo(mp_.halo_plan(), xt, st, rank)
        xl_, sl_ = xt.numpy(), st.numpy()
        assert np.array_equal(xl_, x[vg]), "halo set-points"
        assert np.array_equal(sl_, ss[rg]), "halo sigma_s"
        # ---- owned ramp rows from local data (pg(s) - pg(s-1), opf.hpp:343-351)
        own = mp_.row_owned()
        k = np.repeat(np.arange(mp_.GR), mp_.loc.R)
        s = np.tile(mp_.ramp_steps(), mp_.GR)
        g_idx = ramp_gens[k]

        def var(sv):
            v = g_idx * T + sv
            v = np.where(sv < 0, mp_.loc.n_base + k, v)
            return np.where(sv >= T, mp_.loc.n_base + (mp_.GR if mp_.prev else 0) + k, v)
        ramp_local = xl_[var(s)] - xl_[var(s - 1)]
        rows = mp_.loc.ramp0 + np.arange(mp_.GR * mp_.loc.R)
        owned = own[rows]
        assert np.array_equal(ramp_local[owned], g[rg[rows]][owned])
        # ---- global objective: rank-order sum of the shard partials, equal on every rank
        from paper_2405_14032_b200.shard import global_objective
        ok, f_all, _ = orc.eval_f(x)
        assert ok
        orc_loc = B.OracleModel(net, T, scale[t0:t0 + T])
        xo = np.ascontiguousarray(x[vg][:orc_loc.sizes[0]])  # owned block precedes the ghosts
        ok, f_loc, _ = orc_loc.eval_f(xo)
        assert ok
        ft = global_objective(torch.tensor([f_loc], dtype=torch.float64), world)
        f_ranks = [torch.empty(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(f_ranks, ft)
        assert all(float(v) == float(ft) for v in f_ranks)
        assert abs(float(ft) - f_all) <= 1e-12 * abs(f_all)
        # every global row is owned by exactly one rank
        owned_global = torch.zeros(orc.sizes[1], dtype=torch.int32)
        owned_global[torch.from_numpy(rg[own])] = 1
        dist.all_reduce(owned_global)
        out[rank] = int(owned_global.min()), int(owned_global.max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T_total", [3, 8])
def test_period_shards_gloo(T_total):
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), T_total, out), nprocs=world, join=True)
    assert dict(out) == {0: (1, 1), 1: (1, 1)}
