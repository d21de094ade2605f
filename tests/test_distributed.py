"""CPU, world_size 2 over gloo: the N>1 path of solve_batch_sharded. Each
rank solves its column slice (here with the C restatement standing in for
the GPU solver, so the test runs without a GPU) and the final all_gather
must reassemble exactly the per-slice results, in original column order."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _port_solver(shard, cfg):
    from oracle import port
    from paper_2601_21990_b200.solver import (BatchSolveSummary, Residuals, SolveResult,
                                              SolveStatus)
    pre = [(q.column, int(q.result.status), q.result.objective) for q in shard.presets]
    s, res, *_ = port.solve_batch(shard.batch.base(), shard.batch.batch_width(),
                                  int(shard.batch.objective_mode()), shard.batch.overrides(),
                                  cfg, pre)
    out = BatchSolveSummary(iterations=int(s.iterations), restarts=int(s.restarts),
                            sparse_products=int(s.sparse_products))
    for r in res:
        out.per_problem.append(SolveResult(
            status=SolveStatus(r.status), objective=r.objective, iterations=int(r.iterations),
            restarts=int(r.restarts), residuals=Residuals(r.gap, r.primal, r.dual, r.fixed_point),
            bound_support=r.bound_support, row_support=r.row_support,
            base_bound_support=r.base_bound_support, vectors_exist=bool(r.vectors_exist)))
    return out


def _worker(rank, world, port, kind, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2601_21990_b200 as bl
        from paper_2601_21990_b200 import distributed as D
        from paper_2601_21990_b200 import instances as I
        if kind == "fsb":
            p = I.set_cover(50, 80, 0.08, 1)
            x, frac = I.synthetic_branch_point(p, 6)
            fb = bl.build_fsb_batch(bl.FsbRequest(p, x, frac))
            batch, presets = fb.batch, fb.presets
        else:
            p = I.boxed_feasible(30, 25, 4, 3)
            ob = bl.build_obbt_batch(p, bl.ObbtConfig())
            batch, presets = ob.batch, ob.presets
        cfg = bl.SolverConfig()
        got = D.solve_batch_sharded(batch, cfg, presets, rank=rank, world=world,
                                    solver=_port_solver)
        if rank == 0:
            # reference: every slice solved on its own
            want = []
            for r in range(world):
                sh = D.shard_batch(batch, presets, r, world)
                want.extend(_port_solver(sh, cfg).per_problem)
            ok = len(got.per_problem) == batch.batch_width() == len(want)
            for a, b in zip(got.per_problem, want):
                ok = ok and int(a.status) == int(b.status) and a.iterations == b.iterations
                ok = ok and (a.objective == b.objective or
                             (np.isnan(a.objective) and np.isnan(b.objective)))
            q.put(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["fsb", "obbt"])
def test_sharded_solve_gathers_per_slice_results(kind):
    from oracle import port
    if not port.available():
        pytest.fail("oracle port not built")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    p = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, p, kind, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    assert q.get(timeout=10) is True


def test_signed_unit_shard_is_the_same_lps():
    """A slice of an OBBT batch is rewritten as a shared-objective batch with
    +-1 objective entries; every column's effective cost and bounds match."""
    import paper_2601_21990_b200 as bl
    from paper_2601_21990_b200 import distributed as D
    from paper_2601_21990_b200 import instances as I
    p = I.boxed_feasible(12, 9, 3, 2)
    ob = bl.build_obbt_batch(p, bl.ObbtConfig())
    for r in range(3):
        sh = D.shard_batch(ob.batch, ob.presets, r, 3)
        for j in range(sh.batch.batch_width()):
            a = bl.resolve_column(sh.batch, j)
            b = bl.resolve_column(ob.batch, sh.start + j)
            for i in range(p.num_cols()):
                assert (a.cost(i), a.lower(i), a.upper(i)) == (b.cost(i), b.lower(i), b.upper(i))
