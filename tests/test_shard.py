"""GPU: period sharding is exact.

The global T_total-period problem and its period shards run on the same GPU
(sequentially — no rank waits on another).  After the halo fill, every owned
constraint value and every owned lifted column of M / row of A equals the
global problem's bit for bit: the ghost set-points and ghost ramp rows
reproduce the boundary contributions in the reference's summation order."""
import numpy as np
import pytest

from helpers import interior_point, row_weights, sigmas, DELTAS, assert_bitexact
from paper_2405_14032_b200.opf import CondensedKkt, OpfNlp, load_profile
from paper_2405_14032_b200.shard import ShardMap, halo_exchange, partition
from test_gpu_parity import _edge_network

pytestmark = pytest.mark.gpu


def _columns(colptr, rowidx, vals, cols):
    """{col: {row: value}} for the given columns."""
    return {int(c): dict(zip(rowidx[colptr[c]:colptr[c + 1]].tolist(),
                             vals[colptr[c]:colptr[c + 1]].tolist())) for c in cols}


@pytest.mark.parametrize("T_total,world", [(7, 2), (10, 3), (5, 5)])
def test_shards_reproduce_global_problem(gpu, T_total, world):
    net = _edge_network(seed=50 + world)
    scale = load_profile(net.n_load, T_total)
    glob = OpfNlp(net, T_total, scale)
    glob.lift(1e-4)
    GK = CondensedKkt(nlp=glob)
    xl, xu, xs, _, _ = glob.bounds()
    x = interior_point(xl, xu, xs, 3)
    w = row_weights(glob.n_cons(), 4, zero_every=7)
    sx_g, ss_g = sigmas(glob.sizes.n_free, glob.n_cons(), 5)
    ok, g_glob = glob.eval_g(x)
    assert ok
    GL = glob.lifted_structure()
    g_free = GL["free_to_full"]
    g_lifted_of_full = np.full(glob.n_vars(), -1, np.int64)
    g_lifted_of_full[g_free] = np.arange(len(g_free))
    dw, dc = DELTAS[1]
    GK.set_jacobian_x(x)
    GK.assemble_x(x, w, 1.0, sx_g, ss_g, dw, dc)
    ga, gm = GK.values()
    g_rowptr, g_colidx, g_colptr, g_rowidx = GK.structure()

    parts = partition(T_total, world)
    info0 = glob.shard_info()
    maps, nlps, xs_, ss_ = [], [], [], []
    for t0, T in parts:
        nlp = OpfNlp(net, T, scale[t0:t0 + T], shard=(T_total, t0))
        mp = ShardMap(net.n_bus, net.n_line, net.n_gen, int(np.isfinite(net.line_smax).sum()),
                      info0["ramp_gens"], T_total, t0, T)
        assert nlp.n_vars() == mp.n_local and nlp.n_cons() == mp.m_local
        vg, rg = mp.var_global(), mp.row_global()
        xl_loc = x[vg].copy()
        xs_.append(xl_loc)
        ss_.append(ss_g[rg].copy())
        maps.append(mp)
        nlps.append(nlp)
    # zero the ghosts, then fill them through the exchange protocol
    for mp, xx in zip(maps, xs_):
        xx[mp.ghost_prev()] = np.nan
        xx[mp.ghost_next()] = np.nan
    halo_exchange(maps, xs_, ss_)
    for mp, xx in zip(maps, xs_):
        assert_bitexact(xx, x[mp.var_global()], "halo-filled x")

    for r, (mp, nlp, xx, ss) in enumerate(zip(maps, nlps, xs_, ss_)):
        rg, own = mp.row_global(), mp.row_owned()
        ok, g = nlp.eval_g(xx)
        assert ok
        assert_bitexact(g[own], g_glob[rg[own]], f"rank {r} owned g")
        wl = w[rg]
        nlp.lift(1e-4)
        K = CondensedKkt(nlp=nlp)
        assert K.fused_ready == 1
        L = nlp.lifted_structure()
        free = L["free_to_full"]
        vg = mp.var_global()
        loc2glob = g_lifted_of_full[vg[free]]  # local lifted -> global lifted
        sx = sx_g[loc2glob]
        K.set_jacobian_x(xx)
        K.assemble_x(xx, wl, 1.0, sx, ss, dw, dc)
        a, m = K.values()
        rowptr, colidx, colptr, rowidx = K.structure()
        owned = nlp.shard_info()["owned_lifted"]
        # owned M columns: same rows (mapped) and bit-identical values
        loc_cols = _columns(colptr, rowidx, m, range(owned))
        for c_l, col in loc_cols.items():
            c_g = int(loc2glob[c_l])
            gcol = _columns(g_colptr, g_rowidx, gm, [c_g])[c_g]
            mapped = {int(loc2glob[rw]): v for rw, v in col.items()}
            assert mapped.keys() == gcol.keys(), (r, c_l)
            for rw, v in mapped.items():
                assert v == gcol[rw], (r, c_l, rw, v, gcol[rw])
        # owned A rows: same values at mapped (row, col)
        for rl in np.nonzero(own)[0][:: max(1, len(own) // 400)]:
            rgl = rg[rl]
            loc = {int(loc2glob[colidx[k]]): a[k] for k in range(rowptr[rl], rowptr[rl + 1])}
            glo = {int(g_colidx[k]): ga[k] for k in range(g_rowptr[rgl], g_rowptr[rgl + 1])
                   if g_colidx[k] in set(loc2glob.tolist())}
            assert loc == glo, (r, rl)

