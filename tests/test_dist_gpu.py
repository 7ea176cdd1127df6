"""GPU: the library's distributed CG loop (owned-DOF dots, halo pack/unpack,
rank-local folds + allreduce).

* 1 rank over the library's own NCCL communicator (tfem_nccl_create,
  tfem_operator_set_nccl; ncclAllReduce inside the captured CG graphs):
  bit-identical iterates to the single-device solver.
* 2 ranks sharing the one GPU over gloo (host-staged hooks; no kernel waits
  on another process): same iteration count as the single-device solve of
  the global problem, same solution on owned DOFs.
* the halo / direction overlap of the NCCL path (side stream, fork / join,
  graph-captured) against the synchronous hook path on a self-exchange plan:
  bit-identical iterates.
"""
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def single_device_solution(dev, n_global, p, tol, its, seed):
    import paper_1911_09220_b200 as tf
    from paper_1911_09220_b200.dist import lattice
    sp = tf.FeSpace.cartesian(dev, n_global, p)
    a = tf.BilinearForm(sp)
    a.add_diffusion(1.0)
    a.assemble()
    ess = sp.essential_true_dofs()
    op = tf.ConstrainedOperator(a, ess)
    L = lattice(sp.element_dofs(), n_global, p, sp.n_dofs)
    return sp, op, ess, L


def test_one_rank_nccl_matches_single_device(dev):
    import torch
    import torch.distributed as tdist
    import paper_1911_09220_b200 as tf
    from paper_1911_09220_b200.dist import DistOperator, partition
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0,
                             world_size=1)
    try:
        n, p = (40, 30), 3
        d = DistOperator(dev, partition(2, n, p, 0, 1))
        assert d.transport == "nccl" and d.nccl  # the library's own communicator
        sp, op, ess, _ = single_device_solution(dev, n, p, 1e-10, 2000, 0)
        assert (d.plan.ess == ess).all() and len(d.plan.not_owned) == 0
        b = np.random.default_rng(4).uniform(-1, 1, sp.n_dofs)
        b[ess] = 0.0
        r1 = tf.cg_solve(d.op, b, 1e-10, 2000, d.diag)
        r2 = tf.cg_solve(op, b, 1e-10, 2000, op.diagonal())
        assert r1.iterations == r2.iterations and r1.converged and r2.converged
        assert (r1.x.numpy() == r2.x.numpy()).all()
        r3 = tf.cg_solve(d.op, b, 0.0, 37, d.diag)       # exhaustion path
        r4 = tf.cg_solve(op, b, 0.0, 37, op.diagonal())
        assert r3.iterations == r4.iterations == 37
        assert (r3.x.numpy() == r4.x.numpy()).all()
        d.close()
    finally:
        tdist.destroy_process_group()


def _rank(rank, world, port, n, p, q):
    sys.path.insert(0, str(ROOT))
    try:
        import torch
        import torch.distributed as tdist
        import paper_1911_09220_b200 as tf
        from paper_1911_09220_b200.dist import DistOperator, lattice, partition
        torch.cuda.set_device(0)
        tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                 world_size=world)
        dev = tf.Device(0)
        d = DistOperator(dev, partition(len(n), n, p, rank, world))
        sp, op, ess, Lg = single_device_solution(dev, n, p, 1e-10, 3000, 0)
        dims = tuple(k * p + 1 for k in n)
        table = np.full(int(np.prod(dims)), -1, dtype=np.int64)
        table[np.ravel_multi_index(tuple(Lg.T), dims, order="F")] = np.arange(len(Lg))
        L = d.lattice.copy()
        L[:, -1] += d.slab.lo * p
        l2g = table[np.ravel_multi_index(tuple(L.T), dims, order="F")]
        # smooth right-hand side: random ones amplify round-off over hundreds
        # of iterations (the reference's CG fixtures are smooth, too)
        bg = np.prod([np.sin(np.pi * Lg[:, k] / (n[k] * p)) for k in range(len(n))], axis=0)
        bg[ess] = 0.0
        # operator on owned DOFs: bit-identical to the global device operator
        xg = np.random.default_rng(9).uniform(-1, 1, sp.n_dofs)
        y = tf.Vector(dev, d.space.n_dofs)
        plain = tf.BilinearForm(d.space)
        plain.add_diffusion(1.0)
        plain.assemble()
        plain.mult_true(xg[l2g], y)
        yg = tf.Vector(dev, sp.n_dofs)
        a = tf.BilinearForm(sp)
        a.add_diffusion(1.0)
        a.assemble()
        a.mult_true(xg, yg)
        own = d.plan.owned
        assert (y.numpy()[own] == yg.numpy()[l2g[own]]).all()
        rd = tf.cg_solve(d.op, bg[l2g], 1e-9, 3000, d.diag)
        rg = tf.cg_solve(op, bg, 1e-9, 3000, op.diagonal())
        assert rd.converged and rg.converged and rd.iterations == rg.iterations, \
            (rd.iterations, rg.iterations)
        err = np.abs(rd.x.numpy()[own] - rg.x.numpy()[l2g[own]]).max()
        assert err <= 1e-9 * np.abs(rg.x.numpy()).max(), err
        q.put((rank, "ok", rd.iterations))
    except Exception:
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        try:
            import torch.distributed as tdist
            if tdist.is_initialized():
                tdist.destroy_process_group()
        except Exception:
            pass


@pytest.mark.parametrize("n,p", [((24, 18), 3), ((24, 18), 4), ((6, 5, 8), 2), ((5, 4, 6), 3)])
def test_two_ranks_share_one_gpu_gloo(dev, n, p):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, n, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    # a rank that fails leaves its peer blocked in a collective: report the
    # first failure (or a dead rank) instead of waiting for both results
    import queue
    import time
    res, deadline = [], time.monotonic() + 240
    while len(res) < 2 and time.monotonic() < deadline:
        try:
            res.append(q.get(timeout=2))
        except queue.Empty:
            dead = [(i, pr.exitcode) for i, pr in enumerate(procs)
                    if pr.exitcode not in (None, 0)]
            if dead:
                break
        if res and res[-1][1] != "ok":
            break
    for pr in procs:
        pr.join(timeout=5 if len(res) < 2 else 60)
        if pr.is_alive():
            pr.kill()
    bad = [r for r in res if r[1] != "ok"]
    assert not bad, bad[0][2]
    assert len(res) == 2, ("rank(s) died or hung", res, [pr.exitcode for pr in procs])


def test_overlapped_nccl_halo_matches_the_synchronous_path(dev):
    """The NCCL halo overlap (pack of the new direction's send planes, the
    exchange on a side stream while the direction kernel runs, unpack after
    the join; graph-captured) against the same plan through synchronous
    host hooks: one rank exchanging with itself, receiving into DOFs other
    than the ones it sends, so a missing join or a wrong pack shows up as
    different iterates.  Bitwise equal over 30 iterations."""
    import ctypes as C
    import torch
    import paper_1911_09220_b200 as tf
    from paper_1911_09220_b200 import abi
    n, p = (40, 30), 3
    sp = tf.FeSpace.cartesian(dev, n, p)
    ess = sp.essential_true_dofs()
    free = np.setdiff1d(np.arange(sp.n_dofs), ess)
    rng = np.random.default_rng(5)
    pick = rng.choice(free, 400, replace=False)
    A = np.ascontiguousarray(np.sort(pick[:200]), dtype=np.int32)   # sent
    B = np.ascontiguousarray(np.sort(pick[200:]), dtype=np.int32)   # received into

    def operator():
        a = tf.BilinearForm(sp)
        a.add_diffusion(1.0)
        a.assemble()
        return a, tf.ConstrainedOperator(a, ess)

    b = rng.uniform(-1, 1, sp.n_dofs)
    b[ess] = 0.0
    # overlapped: the library's NCCL communicator (1 rank, peer = itself)
    fa, op_a = operator()
    idbuf = C.create_string_buffer(abi.NCCL_ID_BYTES)
    abi.check(tf.lib().tfem_nccl_unique_id(idbuf))
    h = abi.vp()
    abi.check(tf.lib().tfem_nccl_create(dev.h, 1, 0, idbuf, C.byref(h)))
    one = lambda t, v: (t * 1)(v)
    abi.check(tf.lib().tfem_operator_set_nccl(
        op_a.h, h, 1, one(C.c_int, 0), one(C.c_int64, len(A)), one(abi.i32p, A.ctypes.data_as(abi.i32p)),
        one(C.c_int64, len(B)), one(abi.i32p, B.ctypes.data_as(abi.i32p)), 0, None))
    tf.lib().tfem_nccl_destroy(h)  # the operator keeps it alive
    # synchronous: host hooks copying the send buffer into the receive buffer
    fb, op_b = operator()
    gpu = torch.device("cuda", 0)
    stream = torch.cuda.ExternalStream(dev.stream)
    sb = torch.empty(len(A), dtype=torch.float64, device=gpu)
    rb = torch.empty(len(B), dtype=torch.float64, device=gpu)
    red = torch.zeros(4, dtype=torch.float64, device=gpu)

    def exchange(_u):
        with torch.cuda.stream(stream):
            rb.copy_(sb)

    hooks = (abi.EXCHANGE_HOOK(exchange), abi.ALLREDUCE_HOOK(lambda k, u: None))
    comm = abi.Comm(hooks[0], hooks[1], None)
    halo = abi.Halo()
    halo.n_peers = 1
    halo.n_send[0], halo.n_recv[0] = len(A), len(B)
    halo.send_idx[0], halo.recv_idx[0] = A.ctypes.data_as(abi.i32p), B.ctypes.data_as(abi.i32p)
    halo.send_buf[0], halo.recv_buf[0] = sb.data_ptr(), rb.data_ptr()
    halo.red = red.data_ptr()
    abi.check(tf.lib().tfem_operator_set_comm(op_b.h, C.byref(comm), C.byref(halo), 0, None))
    diag = op_b.diagonal()
    ra = tf.cg_solve(op_a, b, 0.0, 30, diag)
    rb_ = tf.cg_solve(op_b, b, 0.0, 30, diag)
    assert ra.iterations == rb_.iterations == 30
    xa, xb = ra.x.numpy(), rb_.x.numpy()
    assert np.isfinite(xa).all() and (xa == xb).all()
    # and the exchange mattered: the plain operator gives other iterates
    rc = tf.cg_solve(tf.ConstrainedOperator(fa, ess), b, 0.0, 30, diag)
    assert not (rc.x.numpy() == xa).all()
    del op_a, op_b
