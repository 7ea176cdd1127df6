"""Multi-rank path on CPU (torch.distributed gloo, world sizes 2 and 3).

The partition / lattice / halo / ownership / essential-DOF plan of
paper_1911_09220_b200/dist.py drives a numpy mirror of the library's
distributed CG loop with the oracle as the element kernel.  Checks:
  * every rank's operator on its owned DOFs is bit-identical to the global
    operator (ghost-layer design keeps the global element order);
  * the halo update makes every ghost copy equal to its owner's value;
  * distributed Jacobi-CG takes the same number of iterations as the global
    CG and lands on the same solution (owned DOFs, 1e-10).
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def global_index(Lg, dims_lat):
    """lattice -> global DOF lookup table."""
    table = np.full(int(np.prod(dims_lat)), -1, dtype=np.int64)
    lin = np.ravel_multi_index(tuple(Lg.T), dims_lat, order="F")
    table[lin] = np.arange(len(Lg))
    return table


def worker(rank, world, port, dim, n_global, p, out_q):
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as dist
    from oracle.pyoracle import OrcCartesian
    from paper_1911_09220_b200.dist import box_ctrl, halo_plan, lattice, partition

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        s = partition(dim, n_global, p, rank, world)
        oc = OrcCartesian(dim, s.n_local, p)
        qd = oc.setup("diffusion", ctrl=box_ctrl(s, [1.0] * dim))
        L = lattice(oc.elem_dofs, s.n_local, p, oc.ndofs)
        plan = halo_plan(s, L)

        og = OrcCartesian(dim, n_global, p)
        qg = og.setup("diffusion")
        Lg = lattice(og.elem_dofs, n_global, p, og.ndofs)
        dims_lat = tuple(k * p + 1 for k in n_global)
        table = global_index(Lg, dims_lat)
        Lglob = L.copy()
        Lglob[:, -1] += s.lo * p
        l2g = table[np.ravel_multi_index(tuple(Lglob.T), dims_lat, order="F")]
        assert (l2g >= 0).all()

        # 1) operator on owned DOFs == global operator, bit for bit
        xg = np.random.default_rng(0).uniform(-1, 1, og.ndofs)
        y_loc = oc.apply("diffusion", qd, xg[l2g])
        y_g = og.apply("diffusion", qg, xg)
        assert (y_loc[plan.owned] == y_g[l2g[plan.owned]]).all()
        # ownership partitions the global DOFs
        owned_g = torch.zeros(og.ndofs, dtype=torch.int64)
        owned_g[torch.from_numpy(l2g[plan.owned])] = 1
        dist.all_reduce(owned_g)
        assert (owned_g == 1).all()
        # essential DOFs are exactly the global boundary
        ess_g = set(og.boundary_dofs().tolist())
        assert set(l2g[plan.ess].tolist()) == ess_g & set(l2g.tolist())

        def exchange(v):
            reqs, recv = [], []
            for peer, s_idx, r_idx in plan.peers:
                sb = torch.from_numpy(np.ascontiguousarray(v[s_idx]))
                rb = torch.empty(len(r_idx), dtype=torch.float64)
                reqs.append(dist.isend(sb, peer))
                reqs.append(dist.irecv(rb, peer))
                recv.append((r_idx, rb))
            for r in reqs:
                r.wait()
            for r_idx, rb in recv:
                v[r_idx] = rb.numpy()

        # 2) halo update: start with garbage on not-owned DOFs
        v = xg[l2g].copy()
        v[plan.not_owned] = np.nan
        exchange(v)
        assert (v == xg[l2g]).all()

        # 3) distributed Jacobi-CG (mirror of cg.cu's dist loop)
        def gsum(vals):
            t = torch.tensor(vals, dtype=torch.float64)
            dist.all_reduce(t)
            return t.numpy()

        own = plan.owned
        op = oc.operator(["diffusion"], [qd], plan.ess)
        d = oc.diagonal("diffusion", qd)
        d[plan.ess] = 1.0
        bg = np.random.default_rng(1).uniform(-1, 1, og.ndofs)
        bg[og.boundary_dofs()] = 0.0
        b = bg[l2g].copy()
        tol, max_it = 1e-10, 3000
        bnorm = np.sqrt(gsum([b[own] @ b[own]])[0])
        x = np.zeros_like(b)
        r = b.copy()
        z = r / d
        pv = z.copy()
        rr, rz = gsum([r[own] @ r[own], r[own] @ z[own]])
        rnorm = np.sqrt(rr)
        it_done = None
        for it in range(1, max_it + 1):
            if rnorm <= tol * bnorm:
                it_done = it - 1
                break
            exchange(pv)
            q = oc.op_mult(op, pv)
            pq = gsum([pv[own] @ q[own]])[0]
            alpha = rz / pq
            x = x + alpha * pv
            r = r + (-alpha) * q
            z = r / d
            rr, rz_next = gsum([r[own] @ r[own], r[own] @ z[own]])
            rnorm = np.sqrt(rr)
            beta = rz_next / rz
            rz = rz_next
            pv = z + beta * pv
        assert it_done is not None

        dg = og.diagonal("diffusion", qg)
        ess = og.boundary_dofs()
        dg[ess] = 1.0
        xg_sol, it_g, conv = og.cg(og.operator(["diffusion"], [qg], ess), bg, tol, max_it, dg)
        assert conv and it_g == it_done, (it_g, it_done)
        err = np.abs(x[own] - xg_sol[l2g[own]]).max() / np.abs(xg_sol).max()
        assert err <= 1e-10, err
        out_q.put((rank, "ok", it_done))
    except Exception as e:  # report, don't hang the parent
        import traceback
        out_q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("dim,n_global,p,world", [
    (2, (6, 8), 3, 2),
    (2, (5, 7), 2, 3),
    (3, (3, 3, 4), 2, 2),
])
def test_distributed_cpu(oracle_built, dim, n_global, p, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, dim, n_global, p, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    bad = [r for r in results if r[1] != "ok"]
    assert not bad, bad[0][2]
    iters = {r[2] for r in results}
    assert len(iters) == 1


def test_partition_covers_all_layers():
    from paper_1911_09220_b200.dist import partition
    for N in (7, 8, 13):
        for world in (1, 2, 3, 4):
            if world > N:
                continue
            slabs = [partition(2, (5, N), 3, r, world) for r in range(world)]
            assert slabs[0].lo == 0 and slabs[-1].hi == N
            for a, b in zip(slabs, slabs[1:]):
                assert a.hi == b.lo
            assert max(s.hi - s.lo for s in slabs) - min(s.hi - s.lo for s in slabs) <= 1
