"""Multi-rank plumbing: world_size-2 process groups.

CPU (gloo): the Sharding partition/collectives, and the solver's block loop
driven by a test-only oracle-backed problem -> bitwise identical to one rank.
GPU (gloo, 2 processes on one GPU): the real device sweeps sharded over two
ranks, bitwise identical to the single-process result.  (NCCL is the
production backend; its collectives are the same two calls.)
"""
import ctypes
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _spawn(fn, world, *args):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=fn, args=(r, world, port, q, *args)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return {r: v for r, v in out}


# ------------------------------------------------------------- primitives
def _prim_worker(rank, world, port, q):
    _init(rank, world, port)
    from paper_1908_04489_b200.distributed import Sharding, from_process_group

    sh = from_process_group()
    res = {}
    for d in (1, 2, 3, 7, 201, 1000):
        b, e = sh.bounds(d)
        buf = sh.out_buffer(d, "cpu")
        buf.fill_(-1.0)
        buf[b:e] = torch.arange(b, e, dtype=torch.float64)
        sh.allgather_(buf)
        res[d] = (b, e, buf[:d].numpy().copy())
    # work-balanced, uneven shards: padded slots + compaction
    d = 1000
    w = torch.ones(d, dtype=torch.int64)
    w[:100] = 50  # heavy head
    bounds = sh.plan(d, w)
    b, e = sh.shard(bounds)
    buf = sh.padded_buffer(bounds, "cpu")
    base = sh.rank_ptr(buf, bounds)
    view = torch.from_numpy(np.ctypeslib.as_array((ctypes.c_double * (e - b)).from_address(base + 8 * b)))
    view[:] = torch.arange(b, e, dtype=torch.float64)
    res["balanced"] = (bounds, sh.gather(buf, bounds, d).numpy().copy())
    t = torch.tensor([10 + rank, 5 - rank, (1 << 63) - 1], dtype=torch.int64)
    sh.allreduce_min_(t)
    res["min"] = t.numpy().copy()
    dist.destroy_process_group()
    q.put((rank, res))


def test_sharding_primitives_world2():
    out = _spawn(_prim_worker, 2)
    for d in (1, 2, 3, 7, 201, 1000):
        (b0, e0, g0), (b1, e1, g1) = out[0][d], out[1][d]
        assert b0 == 0 and e0 == b1 and e1 == d  # contiguous cover, no overlap
        np.testing.assert_array_equal(g0, np.arange(d, dtype=np.float64))
        np.testing.assert_array_equal(g1, g0)
    np.testing.assert_array_equal(out[0]["min"], [10, 4, (1 << 63) - 1])
    for r in (0, 1):
        bounds, full = out[r]["balanced"]
        assert bounds[0] == 0 and bounds[-1] == 1000 and 0 < bounds[1] < 500  # the heavy head shrinks shard 0
        np.testing.assert_array_equal(full, np.arange(1000, dtype=np.float64))


# ------------------------------------- solver block loop over an oracle fake
def _make_fake(orc, P, d):
    p = orc.OracleWitsenhausen(grid0=(-25.0, 25.0, d), grid1=(-25.0, 25.0, d))
    ocfg = orc.OracleConfig()

    class OracleSharded(P.Problem):
        """Test-only stand-in for the device sweeps: each rank computes its
        shard with the oracle, then the shared Sharding all-gather."""

        name = "witsenhausen"

        def default_grid_specs(self):
            return [(-25.0, 25.0, d)] * 2

        def marginal_cost_segmented(self, *a):
            raise NotImplementedError

        def objective(self, U):
            return orc.objective(p, U.values(0), U.values(1))

        def _sweep(self, fn, m, U, sharding):
            b, e = sharding.bounds(d)
            buf = sharding.out_buffer(d, "cpu")
            buf[b:e] = torch.from_numpy(fn(p, m, np.array(U.values(0)), np.array(U.values(1)), ocfg,
                                           points=np.arange(b, e)))
            sharding.allgather_(buf)
            return buf[:d].numpy().copy()

        def device_local_update(self, m, U, cfg, sharding):
            return self._sweep(orc.local_update_phase, m, U, sharding)

        def device_exhaustion(self, m, U, cfg, sharding):
            return self._sweep(orc.partial_exhaustion_phase, m, U, sharding)

    return OracleSharded(), p


def _block_worker(rank, world, port, q, d):
    _init(rank, world, port)
    import paper_1908_04489_b200 as P
    from oracle import oracle as orc

    prob, p = _make_fake(orc, P, d)
    sh = P.from_process_group()
    rng = np.random.default_rng(3)
    U = P.ControllerSet(tuple(P.SampledController(g, g.points + rng.uniform(-1, 1, d)) for g in prob.grids))
    V = P.run_block(prob, U, P.SolverConfig(), 2, "local", sh)
    V = P.run_block(prob, V, P.SolverConfig(), 1, "exhaustion", sh)
    dist.destroy_process_group()
    q.put((rank, (np.array(V.values(0)), np.array(V.values(1)))))


@pytest.mark.parametrize("d", [201, 64])
def test_block_loop_shard_invariant(oracle_mod, d):
    import paper_1908_04489_b200 as P

    out = _spawn(_block_worker, 2, d)
    prob, p = _make_fake(oracle_mod, P, d)
    rng = np.random.default_rng(3)
    U = P.ControllerSet(tuple(P.SampledController(g, g.points + rng.uniform(-1, 1, d)) for g in prob.grids))
    V = P.run_block(prob, U, P.SolverConfig(), 2, "local")
    V = P.run_block(prob, V, P.SolverConfig(), 1, "exhaustion")
    for r in (0, 1):
        for m in (0, 1):
            np.testing.assert_array_equal(out[r][m].view(np.uint64), np.asarray(V.values(m)).view(np.uint64))


# ------------------------------------------------ real device sweeps, 2 ranks
def _gpu_solve_worker(rank, world, port, q, d):
    _init(rank, world, port)
    import paper_1908_04489_b200 as P

    torch.cuda.set_device(0)
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)
    res = P.solve(prob, P.SolverConfig(max_rounds=3), sharding=P.from_process_group())
    out = (np.array(res.controllers.values(0)), np.array(res.controllers.values(1)), res.final_objective,
           [r.objective for r in res.rounds])
    dist.destroy_process_group()
    q.put((rank, out))


@pytest.mark.gpu
@pytest.mark.parametrize("balanced", [False, True])
def test_sharded_device_solve_bitwise_world2(balanced, monkeypatch):
    import paper_1908_04489_b200 as P

    d = 301
    # work-balanced (uneven) shards are used above UCP_BALANCE_MIN_POINTS points
    monkeypatch.setenv("UCP_BALANCE_MIN_POINTS", "16" if balanced else str(1 << 20))
    out = _spawn(_gpu_solve_worker, 2, d)
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)
    ref = P.solve(prob, P.SolverConfig(max_rounds=3))
    for r in (0, 1):
        u0, u1, J, Js = out[r]
        np.testing.assert_array_equal(u0.view(np.uint64), np.asarray(ref.controllers.values(0)).view(np.uint64))
        np.testing.assert_array_equal(u1.view(np.uint64), np.asarray(ref.controllers.values(1)).view(np.uint64))
        assert np.float64(J).view(np.uint64) == np.float64(ref.final_objective).view(np.uint64)
        assert Js == [rr.objective for rr in ref.rounds]


# ------------------------------------ device Monte-Carlo estimate, 2/3 ranks
def _gpu_mc_worker(rank, world, port, q, n):
    _init(rank, world, port)
    import paper_1908_04489_b200 as P

    torch.cuda.set_device(0)
    prob = P.Inventory(stages=3, grids=[(-3.0, 3.0, 121)] * 3)
    U = prob.identity_controllers()
    out = P.device_monte_carlo_objective(prob, U, n, seed=11, sharding=P.from_process_group())
    dist.destroy_process_group()
    q.put((rank, out))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_device_monte_carlo_rank_invariant(world):
    """Chunks split over ranks, partials all-gathered: every rank gets the
    single-process bits."""
    import paper_1908_04489_b200 as P

    n = 5 * 4096 + 123
    out = _spawn(_gpu_mc_worker, world, n)
    prob = P.Inventory(stages=3, grids=[(-3.0, 3.0, 121)] * 3)
    ref = P.device_monte_carlo_objective(prob, prob.identity_controllers(), n, seed=11)
    for r in range(world):
        assert np.array(out[r]).view(np.uint64).tolist() == np.array(ref).view(np.uint64).tolist()


# ------------------------- config 4 across ranks: instances k % world, batched
def _gpu_many_worker(rank, world, port, q):
    _init(rank, world, port)
    import paper_1908_04489_b200 as P

    torch.cuda.set_device(0)
    probs = [P.Witsenhausen(k=0.1 + 0.2 * i, sigma=(3.0, 5.0)[i % 2], grids=[(-25.0, 25.0, 201)] * 2)
             for i in range(6)]
    res = P.solve_many(probs, P.SolverConfig(max_rounds=3), sharding=P.from_process_group())
    out = {k: (r.final_objective, np.asarray(r.controllers.values(0))) for k, r in enumerate(res) if r is not None}
    dist.destroy_process_group()
    q.put((rank, out))


@pytest.mark.gpu
def test_solve_many_replicas_world2():
    """Each rank solves its instances (k % world) with the batched engine;
    every instance is bitwise its single-process solve."""
    import paper_1908_04489_b200 as P

    out = _spawn(_gpu_many_worker, 2)
    assert sorted(out[0]) == [0, 2, 4] and sorted(out[1]) == [1, 3, 5]
    for r in (0, 1):
        for k, (J, u0) in out[r].items():
            p = P.Witsenhausen(k=0.1 + 0.2 * k, sigma=(3.0, 5.0)[k % 2], grids=[(-25.0, 25.0, 201)] * 2)
            ref = P.solve(p, P.SolverConfig(max_rounds=3))
            assert J == ref.final_objective
            assert np.array_equal(u0.view(np.uint64), np.asarray(ref.controllers.values(0)).view(np.uint64))


# ---------------------------- config 5 sharded over two ranks (grid points)
def _gpu_c5_worker(rank, world, port, q):
    _init(rank, world, port)
    import paper_1908_04489_b200 as P

    torch.cuda.set_device(0)
    out = {}
    for name, prob in (("inv3", P.Inventory(stages=3, grids=[(-3.0, 3.0, 121)] * 3)),
                       ("zd", P.ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)]))):
        res = P.solve(prob, P.SolverConfig(max_rounds=3), sharding=P.from_process_group())
        out[name] = (res.final_objective, [np.asarray(res.controllers.values(m)) for m in range(prob.M)])
    dist.destroy_process_group()
    q.put((rank, out))


@pytest.mark.gpu
def test_config5_sharded_solve_bitwise_world2():
    import paper_1908_04489_b200 as P

    out = _spawn(_gpu_c5_worker, 2)
    refs = {"inv3": P.solve(P.Inventory(stages=3, grids=[(-3.0, 3.0, 121)] * 3), P.SolverConfig(max_rounds=3)),
            "zd": P.solve(P.ZeroDelay(grids=[(-5.0, 5.0, 201), (-6.0, 6.0, 241)]), P.SolverConfig(max_rounds=3))}
    for r in (0, 1):
        for name, (J, us) in out[r].items():
            ref = refs[name]
            assert J == ref.final_objective, (name, r)
            for m, u in enumerate(us):
                assert np.array_equal(u.view(np.uint64), np.asarray(ref.controllers.values(m)).view(np.uint64))


# --------------------- no host synchronisation inside a multi-rank phase
@pytest.mark.gpu
def test_sharded_phases_do_not_synchronise(monkeypatch):
    """Rank 0 of a 2-rank work-balanced plan (collectives stubbed: this is about
    the host side): once a solve has cached the plans, every phase -- plan,
    sweep, gather -- queues its work without one host<->device synchronisation
    (torch sync debug mode "error" raises on any).  The plans are refreshed
    from the objective's own read-back (Witsenhausen.device_objective)."""
    import paper_1908_04489_b200 as P
    from paper_1908_04489_b200 import witsenhausen

    class Stub(P.Sharding):
        def allgather_(self, buf):
            pass

        def allgather_uneven_(self, buf, bounds):
            pass

        def allreduce_min_(self, t):
            pass

    monkeypatch.setattr(witsenhausen, "BALANCE_MIN_POINTS", 1024)
    sh = Stub(rank=0, world=2)
    d = 4096
    prob = P.Witsenhausen(grids=[(-25.0, 25.0, d)] * 2)
    cfg = P.SolverConfig(max_rounds=1)
    res = P.solve(prob, cfg, sharding=sh)  # fills and refreshes the plan cache
    plans = prob.device_context().plans
    assert {k[0] for k in plans} == {(0, None), (0, cfg.radius_for(prob.grids[0])), (1, None)}
    assert all(b != sh.equal_plan(d) for b in plans.values())  # uneven: the balanced path
    U = res.controllers
    torch.cuda.synchronize()
    torch.cuda.set_sync_debug_mode("error")
    try:
        for m in (0, 1):
            prob.device_local_update(m, U, cfg, sh)
            prob.device_exhaustion(m, U, cfg, sh)
    finally:
        torch.cuda.set_sync_debug_mode("default")
    prob.flush_errors(sh)


# ------------- the library-communicator backend routes every exchange to it
def test_comm_sharding_routes_collectives():
    """CommSharding (paper_1908_04489_b200.comm) sends the phase all-gathers --
    equal plans in place, work-balanced plans as the uneven all-gather with the
    plan's bounds -- and the error-slot MIN all-reduce to its communicator
    (host logic; the NCCL calls themselves run in tests/test_gpu_parity.py)."""
    from paper_1908_04489_b200.comm import CommSharding

    class FakeComm:
        def __init__(self):
            self.calls = []

        def allgather_(self, buf):
            self.calls.append(("allgather", buf.numel()))

        def allgatherv_(self, buf, bounds):
            self.calls.append(("allgatherv", tuple(bounds)))

        def allreduce_min_(self, t):
            self.calls.append(("min", t.numel()))

    comm = FakeComm()
    sh = CommSharding(rank=1, world=2, comm=comm)
    d = 1000
    eq = sh.equal_plan(d)
    buf = sh.padded_buffer(eq, "cpu")
    assert sh.gather(buf, eq, d).numel() == d
    w = torch.ones(d, dtype=torch.int64)
    w[:100] = 50
    bal = sh.plan_from_cuts(d, sh.plan_cuts(w).tolist())
    assert bal != eq and bal[0] == 0 and bal[-1] == d
    out = sh.gather(sh.padded_buffer(bal, "cpu"), bal, d)
    assert out.numel() == d
    sh.allreduce_min_(torch.zeros(6, dtype=torch.int64))
    assert comm.calls == [("allgather", 1000), ("allgatherv", bal), ("min", 6)]
    one = CommSharding(rank=0, world=1, comm=comm)
    one.allreduce_min_(torch.zeros(3, dtype=torch.int64))
    assert len(comm.calls) == 3  # a single rank exchanges nothing


def test_moments_weights_model_matches_tile_rule():
    """The stage-1 shard weights (Witsenhausen._moments_weights: live-tile
    pairs per query from two sorted counts) equal a direct application of the
    moments kernel's tile-skipping rule per 128-query block, NaN tiles live."""
    from paper_1908_04489_b200.witsenhausen import Witsenhausen

    rng = np.random.default_rng(5)
    d = 5000
    y = torch.from_numpy(np.linspace(-25.0, 25.0, d))
    x1 = y + torch.from_numpy(np.where(rng.random(d) < 0.5, 6.0, -6.0) - 0.9 * y.numpy())
    x1[1234] = float("nan")
    w = Witsenhausen._moments_weights(x1, y)
    xs, ys = x1.numpy(), y.numpy()
    for b in range(0, -(-d // 128)):
        q = ys[b * 128:(b + 1) * 128]
        live = 0
        for t in range(-(-d // 256)):
            xt = xs[t * 256:(t + 1) * 256]
            if np.isnan(xt).any() or not (q.min() - np.nanmax(xt) > 12 or q.max() - np.nanmin(xt) < -12):
                live += 1
        assert int(w[b * 128]) == max(live, 1) * 256, b
