"""GPU: the period-shard halo over peer memory (gn_halo, csrc/gn_halo.cu).

Ranks must live on different GPUs for the fused exchange (its kernel waits for the
neighbours' step flags).  On one GPU the same device code is exercised without any
kernel waiting on another launch:

* SEND for every rank, then RECV for every rank (the flags are already released when a
  RECV kernel runs): ghosts and the rank-order objective equal the global problem's;
* every rank's exchange in ONE cooperative launch (gn_halo_exchange_emulated, CTA r =
  rank r): the release / acquire flag protocol itself, both directions, two steps;
* two processes on cuda:0, each holding a device shard context: the halo over gloo with
  CPU staging and over CUDA IPC (each process maps the other's region; SEND, host
  barrier, RECV), and then every owned row of g, row of A and column of M of each
  process's shard equals the global problem's bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch

from helpers import DELTAS, interior_point, row_weights, sigmas
from paper_2405_14032_b200.opf import CondensedKkt, OpfNlp, load_profile
from paper_2405_14032_b200.shard import DeviceHalo, ShardMap, partition

pytestmark = pytest.mark.gpu


def _setup(net, T_total, world, seed):
    scale = load_profile(net.n_load, T_total)
    glob = OpfNlp(net, T_total, scale)
    xl, xu, xs, _, _ = glob.bounds()
    x = interior_point(xl, xu, xs, seed)
    _, ss = sigmas(1, glob.n_cons(), seed + 1)
    ok, f_glob = glob.eval_f(x)
    assert ok
    ramp = glob.shard_info()["ramp_gens"]
    LT = int(np.isfinite(net.line_smax).sum())
    shards = []
    for r, (t0, T) in enumerate(partition(T_total, world)):
        nlp = OpfNlp(net, T, scale[t0:t0 + T], shard=(T_total, t0))
        mp = ShardMap(net.n_bus, net.n_line, net.n_gen, LT, ramp, T_total, t0, T)
        shards.append((nlp, mp))
    return glob, x, ss, f_glob, shards


def _local(mp, x, ss, dev):
    xl_ = x[mp.var_global()].copy()
    sl_ = ss[mp.row_global()].copy()
    xl_[mp.ghost_prev()] = np.nan
    xl_[mp.ghost_next()] = np.nan
    sl_[mp.ghost_rows()] = np.nan
    return torch.from_numpy(xl_).to(dev), torch.from_numpy(sl_).to(dev)


def _check_filled(mp, xt, st, x, ss):
    assert np.array_equal(xt.cpu().numpy(), x[mp.var_global()]), "ghost set-points"
    assert np.array_equal(st.cpu().numpy(), ss[mp.row_global()]), "ghost sigma_s"


@pytest.mark.parametrize("world,T_total", [(2, 6), (3, 7), (4, 9)])
@pytest.mark.parametrize("mode", ["phases", "emulated"])
def test_device_halo_one_gpu(gpu, world, T_total, mode):
    from test_gpu_parity import _edge_network
    net = _edge_network(seed=60 + world)
    dev = torch.device("cuda", 0)
    glob, x, ss, f_glob, shards = _setup(net, T_total, world, 11)
    halos = [DeviceHalo(nlp, r, world) for r, (nlp, _) in enumerate(shards)]
    DeviceHalo.link(halos)
    for step in range(3):  # successive steps alternate the region buffers
        if step:
            x = interior_point(*glob.bounds()[:3], 100 + step)
            _, ss = sigmas(1, glob.n_cons(), 200 + step)
            ok, f_glob = glob.eval_f(x)
            assert ok
        loc = [_local(mp, x, ss, dev) for _, mp in shards]
        torch.cuda.synchronize()
        if mode == "emulated":
            DeviceHalo.exchange_emulated(halos, [a for a, _ in loc], [b for _, b in loc])
        else:
            for h, (xt, st) in zip(halos, loc):
                h.exchange(xt, st, DeviceHalo.SEND)
            for h, (xt, st) in zip(halos, loc):
                h.exchange(xt, st, DeviceHalo.RECV)
        torch.cuda.synchronize()
        for (_, mp), (xt, st) in zip(shards, loc):
            _check_filled(mp, xt, st, x, ss)
        # objective partials -> the rank-order sum on every rank
        fl = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in shards]
        fg = [torch.full((1,), np.nan, dtype=torch.float64, device=dev) for _ in shards]
        for (nlp, _), (xt, _), f in zip(shards, loc, fl):
            assert nlp.eval_device("f", xt, f)
        for h, a, b in zip(halos, fl, fg):
            h.objective(a, b, DeviceHalo.SEND)
        for h, a, b in zip(halos, fl, fg):
            h.objective(a, b, DeviceHalo.RECV)
        torch.cuda.synchronize()
        parts = [float(f) for f in fl]
        expect = parts[0]
        for p in parts[1:]:
            expect += p
        assert all(float(b) == expect for b in fg)
        assert abs(expect - f_glob) <= 1e-12 * abs(f_glob)
    for h in halos:
        h.close()


# ------------------------------------------------------------------- two processes
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _columns(colptr, rowidx, vals, cols):
    return {int(c): dict(zip(rowidx[colptr[c]:colptr[c + 1]].tolist(),
                             vals[colptr[c]:colptr[c + 1]].tolist())) for c in cols}


def _worker(rank, world, port, T_total, out):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    import torch.distributed as dist
    from paper_2405_14032_b200.shard import exchange_halo
    from test_gpu_parity import _edge_network
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        net = _edge_network(seed=77)
        glob, x, ss, f_glob, shards = _setup(net, T_total, world, 5)
        nlp, mp = shards[rank]
        # the global problem's KKT at the same point (each process builds it: small)
        glob.lift(1e-4)
        GK = CondensedKkt(nlp=glob)
        w = row_weights(glob.n_cons(), 4, zero_every=7)
        sx_g, _ = sigmas(glob.sizes.n_free, glob.n_cons(), 6)
        dw, dc = DELTAS[1]
        GK.update_x(x, w, 1.0, sx_g, ss, dw, dc)
        ga, gm = GK.values()
        g_rowptr, g_colidx, g_colptr, g_rowidx = GK.structure()
        ok, g_glob = glob.eval_g(x)
        assert ok
        gfree = glob.lifted_structure()["free_to_full"]
        g_lift = np.full(glob.n_vars(), -1, np.int64)
        g_lift[gfree] = np.arange(len(gfree))
        # (1) halo over gloo with CPU staging (the NCCL path of bench.py, on the CPU)
        xt, st = _local(mp, x, ss, dev)
        xc, sc = xt.cpu(), st.cpu()
        exchange_halo(mp.halo_plan(), xc, sc, rank)
        xt.copy_(xc)
        st.copy_(sc)
        _check_filled(mp, xt, st, x, ss)
        # (2) halo over CUDA IPC: map the other process's region, SEND, barrier, RECV
        halo = DeviceHalo(nlp, rank, world)
        halo.connect()
        xt2, st2 = _local(mp, x, ss, dev)
        torch.cuda.synchronize()
        halo.exchange(xt2, st2, DeviceHalo.SEND)
        torch.cuda.synchronize()
        dist.barrier()
        halo.exchange(xt2, st2, DeviceHalo.RECV)
        torch.cuda.synchronize()
        _check_filled(mp, xt2, st2, x, ss)
        fl = torch.zeros(1, dtype=torch.float64, device=dev)
        fg = torch.zeros(1, dtype=torch.float64, device=dev)
        assert nlp.eval_device("f", xt2, fl)
        halo.objective(fl, fg, DeviceHalo.SEND)
        torch.cuda.synchronize()
        dist.barrier()
        halo.objective(fl, fg, DeviceHalo.RECV)
        torch.cuda.synchronize()
        assert abs(float(fg) - f_glob) <= 1e-12 * abs(f_glob)
        allf = [None] * world
        dist.all_gather_object(allf, float(fg))
        assert len(set(allf)) == 1
        dist.barrier()  # every process done with the others' regions before closing
        halo.close()
        # (3) the device shard on the halo-filled x: owned g / A / M = global, bit for bit
        xx = xt2.cpu().numpy()
        rg, own = mp.row_global(), mp.row_owned()
        ok, g = nlp.eval_g(xx)
        assert ok and np.array_equal(g[own], g_glob[rg[own]]), "owned g"
        nlp.lift(1e-4)
        K = CondensedKkt(nlp=nlp)
        free = nlp.lifted_structure()["free_to_full"]
        loc2glob = g_lift[mp.var_global()[free]]
        K.update_x(xx, w[rg], 1.0, sx_g[loc2glob], st2.cpu().numpy(), dw, dc)
        a, m = K.values()
        rowptr, colidx, colptr, rowidx = K.structure()
        owned = nlp.shard_info()["owned_lifted"]
        bad = 0
        for c_l, col in _columns(colptr, rowidx, m, range(owned)).items():
            c_g = int(loc2glob[c_l])
            gcol = _columns(g_colptr, g_rowidx, gm, [c_g])[c_g]
            mapped = {int(loc2glob[rw]): v for rw, v in col.items()}
            bad += mapped != gcol
        gset = set(loc2glob.tolist())
        for rl in np.nonzero(own)[0]:
            loc = {int(loc2glob[colidx[k]]): a[k] for k in range(rowptr[rl], rowptr[rl + 1])}
            rgl = rg[rl]
            glo = {int(g_colidx[k]): ga[k] for k in range(g_rowptr[rgl], g_rowptr[rgl + 1])
                   if g_colidx[k] in gset}
            bad += loc != glo
        out[rank] = bad
        K.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T_total", [5, 8])
def test_two_processes_device_shards(gpu, T_total):
    import torch.multiprocessing as mp
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), T_total, out), nprocs=world, join=True)
    assert dict(out) == {0: 0, 1: 0}
