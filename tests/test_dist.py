"""Host logic of the partitioned solve on CPU: the Morton-range partition and
the halo plans of octmg_partition_plan_host, checked with the fp64 oracle's operators.

A rank holds only its owned tiles plus what the halo plan sends it; with everything else
NaN, the composite operator (PCG apply) and the level operator (RBGS / residual) evaluated
on its owned rows must equal the global evaluation.  The world-size-2 test performs the
exchange for real over torch.distributed (gloo)."""
import os

import numpy as np
import pytest

from octgen import make_config
from oracle.oracle import Oracle

B3 = 512


def _plan(o, nranks, gather=0):
    import paper_2604_18886_b200 as om
    tb = o.tables()
    counts = np.zeros(4 * (o.L + 1), dtype=np.int32)
    for l in range(o.L + 1):
        counts[4 * l:4 * l + 4] = [o.leaf_begin[l], o.leaf_count[l], o.inner_begin[l], o.inner_count[l]]
    return om.partition_plan_host(tb, o.L, o.NL, o.NI, counts, nranks, gather)


def _cells(kind):
    if kind == 6:
        return np.arange(B3)
    ax, layer = kind >> 1, (7 if kind & 1 else 0)
    o1, o2 = (1, 2) if ax == 0 else ((0, 2) if ax == 1 else (0, 1))
    c = np.arange(64)
    xyz = [None, None, None]
    xyz[ax] = np.full(64, layer)
    xyz[o1] = c & 7
    xyz[o2] = c >> 3
    return xyz[0] + 8 * xyz[1] + 64 * xyz[2]


def _owned_mask(o, owner, rank, lg, leaf_only):
    tiles = o.tables()["tiles"]
    T = o.NL if leaf_only else o.T
    own = np.array([(owner[t] == rank) or (tiles[t, 0] < lg) for t in range(T)])
    return np.repeat(own, B3)


def _fill(local, ref, items, leaf_only, NL):
    for t, kind in items:
        if leaf_only and t >= NL:
            continue
        idx = t * B3 + _cells(int(kind))
        local[idx] = ref[idx]


CASES = ["sphere_small", "tank_small", "uniform32"]


@pytest.mark.parametrize("gather", [0, 1])
@pytest.mark.parametrize("name", CASES + ["sphere_35"])
@pytest.mark.parametrize("nranks", [2, 3])
def test_partition_ownership(name, nranks, gather):
    cfg = make_config(name, with_fields=False)
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    lg, owner, items = _plan(o, nranks, gather)
    tb = o.tables()
    lev = tb["tiles"][:, 0]
    assert np.all(owner[lev < lg] == -1) and np.all((owner[lev >= lg] >= 0) & (owner[lev >= lg] < nranks))
    assert lg <= min(lev[:o.NL])  # every leaf is owned
    for t in range(o.T):  # a tile at level > lg is owned by its parent's owner
        if lev[t] > lg:
            assert owner[t] == owner[tb["parent"][t]]
    # an item is a tile of the sender's level, owned by the sender
    for (l, a, b), it in items.items():
        for t, kind in it:
            assert owner[t] == a and lev[t] == l and a != b and 0 <= kind <= 6
    # the partition is a set of contiguous Morton ranges at level lg
    at = np.where(lev == lg)[0]
    from octgen.trees import morton3
    m = morton3(tb["tiles"][at, 1], tb["tiles"][at, 2], tb["tiles"][at, 3])
    seq = owner[at[np.argsort(m)]]
    assert np.all(np.diff(seq) >= 0)
    # whole parents: the children of a level-(lg-1) tile belong to one rank
    if lg >= 1:
        for pt in np.unique(tb["parent"][at]):
            assert len(np.unique(owner[at[tb["parent"][at] == pt]])) == 1


def test_gather_threshold_chooses_partition_level():
    """gather_below_cells (north_star: coarse levels below a size threshold are gathered): lg
    is the coarsest level <= the coarsest leaf level with >= 8 tiles per rank and >= the
    threshold in cells.  sphere_35: levels 0..3 have 1, 8, 64, 512 tiles, leaves from 3."""
    cfg = make_config("sphere_35", with_fields=False)
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    assert [int(c) for c in (np.asarray(o.leaf_count) + np.asarray(o.inner_count))[:4]] == [1, 8, 64, 512]
    assert _plan(o, 2, 1)[0] == 2            # as deep as 8 tiles per rank allow (64 >= 16)
    assert _plan(o, 8, 1)[0] == 2            # 64 >= 64
    assert _plan(o, 9, 1)[0] == 3            # 64 < 72
    assert _plan(o, 2, 64 * 512)[0] == 2     # level 2 holds exactly the threshold
    assert _plan(o, 2, 64 * 512 + 1)[0] == 3
    assert _plan(o, 2, 0)[0] == 3            # default 2^21 cells: nothing reaches it, lg = leaf level
    assert _plan(o, 2, 1 << 40)[0] == 3      # never above the coarsest leaf level


def _check_rank(o, owner, items, lg, rank, nranks, x, u_all, Ax, Au):
    # composite operator on the leaf vector (PCG direction): exchange every level's leaves
    loc = np.where(_owned_mask(o, owner, rank, lg, True), x, np.nan)
    for l in range(lg, o.L + 1):
        for a in range(nranks):
            if a != rank:
                _fill(loc, x, items[(l, a, rank)], True, o.NL)
    y = o.apply(loc)
    mine = _owned_mask(o, owner, rank, -1, True) & _owned_mask(o, owner, rank, lg, True)
    assert np.all(np.isfinite(y[mine])) and np.array_equal(y[mine], Ax[mine])
    # level operator at every partitioned level: exchange levels l and l-1
    tiles = o.tables()["tiles"]
    for l in range(max(lg, 1), o.L + 1):
        locu = np.where(_owned_mask(o, owner, rank, lg, False), u_all, np.nan)
        for ll in (l, l - 1):
            if ll < lg:
                continue
            for a in range(nranks):
                if a != rank:
                    _fill(locu, u_all, items[(ll, a, rank)], False, o.NL)
        yl = o.apply_level(l, locu)
        rows = np.repeat((tiles[:, 0] == l) & (owner == rank), B3)
        assert np.all(np.isfinite(yl[rows])) and np.array_equal(yl[rows], Au[l][rows])


@pytest.mark.parametrize("name", CASES)
def test_halo_plan_covers_every_read(name):
    cfg = make_config(name)
    o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
    o.setup(cfg["kind"], cfg["w"])
    rng = np.random.default_rng(3)
    act = o.coefs()[:, 0] != 0
    x = rng.standard_normal(o.N) * act[:o.N]
    u_all = rng.standard_normal(o.T * B3) * act
    Ax = o.apply(x)
    Au = {l: o.apply_level(l, u_all) for l in range(o.L + 1)}
    for nranks in (2, 3):
        for gather in (0, 1):
            lg, owner, items = _plan(o, nranks, gather)
            for rank in range(nranks):
                _check_rank(o, owner, items, lg, rank, nranks, x, u_all, Ax, Au)
    # negative control: the check notices one missing item of each kind class
    lg, owner, items = _plan(o, 2)
    for kinds in ((0, 1, 2, 3, 4, 5), (6,)):
        for key, it in items.items():
            sel = np.where(np.isin(it[:, 1], kinds) & (it[:, 0] < o.NL))[0]
            if key[2] == 0 and len(sel):
                bad = dict(items)
                bad[key] = np.delete(it, sel[0], axis=0)
                with pytest.raises(AssertionError):
                    _check_rank(o, owner, bad, lg, 0, 2, x, u_all, Ax, Au)
                break


def _worker(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = make_config(name)
        o = Oracle(cfg["tiles"], cfg["ext"], cfg["wall_bc"])
        o.setup(cfg["kind"], cfg["w"])
        act = o.coefs()[:o.N, 0] != 0
        x = np.random.default_rng(11).standard_normal(o.N) * act  # same on every rank
        lg, owner, items = _plan(o, world)
        loc = np.where(_owned_mask(o, owner, rank, lg, True), x, np.nan)
        # real exchange: each rank packs its items for every peer and sends them
        reqs, bufs = [], {}
        for l in range(lg, o.L + 1):
            for peer in range(world):
                if peer == rank:
                    continue
                send = items[(l, rank, peer)]
                send = [(t, k) for t, k in send if t < o.NL]
                if send:
                    pk = np.concatenate([loc[t * B3 + _cells(int(k))] for t, k in send])
                    reqs.append(dist.isend(torch.from_numpy(pk.astype(np.float64)), dst=peer, tag=l))
                recv = [(t, k) for t, k in items[(l, peer, rank)] if t < o.NL]
                if recv:
                    n = sum(len(_cells(int(k))) for _, k in recv)
                    buf = torch.empty(n, dtype=torch.float64)
                    reqs.append(dist.irecv(buf, src=peer, tag=l))
                    bufs[(l, peer)] = (recv, buf)
        for r in reqs:
            r.wait()
        for (l, peer), (recv, buf) in bufs.items():
            v, k0 = buf.numpy(), 0
            for t, k in recv:
                c = _cells(int(k))
                loc[t * B3 + c] = v[k0:k0 + len(c)]
                k0 += len(c)
        y = o.apply(loc)
        mine = _owned_mask(o, owner, rank, -1, True)
        ok = bool(np.all(np.isfinite(y[mine])) and np.array_equal(y[mine], o.apply(x)[mine]))
        # the fp64 dot over owned cells, summed by allreduce, equals the global dot
        part = torch.tensor([float((x[mine] * y[mine]).sum())], dtype=torch.float64)
        dist.all_reduce(part)
        tot = float((x * o.apply(x)).sum())
        ok = ok and abs(part.item() - tot) <= 1e-12 * abs(tot)
        # gather below the partition level: each rank restricts the residual of its level-lg
        # tiles into their (whole, rank-owned) parents, R r = sum of the 8 children / alpha,
        # and the all-gather leaves every rank with the full replicated level lg - 1
        if lg >= 1:
            tb = o.tables()
            lev, par = tb["tiles"][:, 0], tb["parent"]
            u_all = np.random.default_rng(5).standard_normal(o.T * B3) * (o.coefs()[:, 0] != 0)
            r_all = -o.apply_level(lg, u_all)
            def restrict(tiles_):
                out = np.zeros(o.T * B3)
                for t in tiles_:
                    p, (i, j, k) = par[t], tb["tiles"][t, 1:4]
                    for c in range(B3):
                        x_, y_, z_ = c & 7, (c >> 3) & 7, c >> 6
                        pc = ((i & 1) * 4 + (x_ >> 1)) + 8 * ((j & 1) * 4 + (y_ >> 1)) + 64 * ((k & 1) * 4 + (z_ >> 1))
                        out[p * B3 + pc] += r_all[t * B3 + c] / 2.0
                return out
            at = np.where(lev == lg)[0]
            full = restrict(at)
            mine_p = restrict(at[owner[at] == rank])
            parents = np.unique(par[at[owner[at] == rank]])
            got = [None] * world
            dist.all_gather_object(got, {int(p_): mine_p[p_ * B3:(p_ + 1) * B3] for p_ in parents})
            gathered = np.zeros(o.T * B3)
            for d in got:
                for p_, v in d.items():
                    assert not gathered[p_ * B3:(p_ + 1) * B3].any()  # each parent from one rank
                    gathered[p_ * B3:(p_ + 1) * B3] = v
            pall = np.unique(par[at])
            idx = np.concatenate([np.arange(p_ * B3, (p_ + 1) * B3) for p_ in pall])
            ok = ok and np.array_equal(gathered[idx], full[idx])
        q.put((rank, ok))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put((rank, repr(e)))


def test_gloo_world2_halo_exchange():
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, "sphere_small", q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(60)
    assert sorted(res) == [(0, True), (1, True)], res
