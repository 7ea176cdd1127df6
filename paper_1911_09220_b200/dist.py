"""Element-partitioned multi-GPU PA-CG.

Partition: the Cartesian mesh is cut along its last axis into contiguous
cell slabs, one per rank (one process per GPU).  Each rank also holds ONE
ghost cell layer above its slab, so every DOF it owns receives all element
contributions locally and in ascending global element order (own rows, then
the ghost row = the next rank's first row): the distributed operator is
bit-identical to the single-device / reference operator on owned DOFs.

Ownership: rank r owns the DOF lattice planes J in [1 if r > 0 else 0, top]
of its slab (top = its upper interface plane); the bottom interface plane
belongs to rank r-1, the planes above `top` to rank r+1.

Per CG iteration (inside the library's loop):
  halo update of p      owner -> ghost copies: send my planes J in [1, p] down,
                        my plane J = top up; receive J = 0 from below and
                        J in (top, top+p] from above
  allreduce(p.q), allreduce(r.r, r.z)   dots over owned DOFs only
Transport: "nccl" (default) -- the library's own NCCL communicator
(tfem_nccl_create / tfem_operator_set_nccl): ncclSend/ncclRecv and
ncclAllReduce on the library stream, captured into the CG's CUDA graphs, no
Python per iteration; torch.distributed only ships the NCCL id and times the
run.  "hooks" -- host callbacks through torch.distributed (gloo test path:
several ranks sharing one GPU, which NCCL refuses).

The plan (partition, lattice coordinates, halo lists, ownership, essential
DOFs) is plain numpy shared by the GPU driver and the CPU test backend
(tests/test_dist.py, gloo, world sizes 2-3).
"""
from __future__ import annotations

import ctypes as C
import json
import time
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np


# ------------------------------------------------------------------- plan
@dataclass
class Slab:
    dim: int
    n_global: Tuple[int, ...]
    p: int
    rank: int
    world: int
    lo: int  # own cell layers [lo, hi) along the last axis
    hi: int

    @property
    def ghost(self) -> bool:
        return self.rank < self.world - 1

    @property
    def n_local(self) -> Tuple[int, ...]:
        return tuple(self.n_global[:-1]) + (self.hi - self.lo + (1 if self.ghost else 0),)

    @property
    def origin(self) -> Tuple[int, ...]:
        return (0,) * (self.dim - 1) + (self.lo,)

    @property
    def top(self) -> int:
        """Local lattice index of the upper interface plane."""
        return (self.hi - self.lo) * self.p


def partition(dim: int, n_global: Sequence[int], p: int, rank: int, world: int) -> Slab:
    N = n_global[-1]
    if world > N:
        raise ValueError("partition: more ranks than cell layers")
    base, extra = divmod(N, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return Slab(dim, tuple(n_global), p, rank, world, lo, hi)


def lattice(elem_dofs: np.ndarray, n_cells: Sequence[int], p: int, ndofs: int) -> np.ndarray:
    """Lattice coordinates (I, J[, K]) of every local DOF from the element
    map: element (i, j, k), local slot (a, b, c) x fastest -> (i p + a, ...)."""
    dim = len(n_cells)
    ne = int(np.prod(n_cells))
    D1 = p + 1
    e = np.arange(ne, dtype=np.int64)
    l = np.arange(D1 ** dim, dtype=np.int64)
    cell = [e % n_cells[0], (e // n_cells[0]) % n_cells[1]]
    loc = [l % D1, (l // D1) % D1]
    if dim == 3:
        cell.append(e // (n_cells[0] * n_cells[1]))
        loc.append(l // (D1 * D1))
    L = np.empty((ndofs, dim), dtype=np.int64)
    flat = elem_dofs.reshape(-1)
    for d in range(dim):
        L[flat, d] = (cell[d][:, None] * p + loc[d][None, :]).reshape(-1)
    return L


@dataclass
class Plan:
    not_owned: np.ndarray           # local DOFs owned by another rank
    ess: np.ndarray                 # local DOFs on the global boundary (sorted)
    peers: List[Tuple[int, np.ndarray, np.ndarray]]  # (rank, send_idx, recv_idx)
    owned: np.ndarray               # local DOFs this rank owns (sorted)


def halo_plan(s: Slab, L: np.ndarray) -> Plan:
    p, top = s.p, s.top
    J = L[:, -1]
    # transverse key: first axis fastest (same order on both sides of a cut)
    key = L[:, 0].copy()
    if s.dim == 3:
        key = key + (s.n_global[0] * p + 1) * L[:, 1]
    idx = np.arange(len(J), dtype=np.int64)

    def sel(mask):
        i = idx[mask]
        return i[np.lexsort((key[i], J[i]))].astype(np.int32)

    not_owned = (J > top) | ((J == 0) & (s.rank > 0))
    peers = []
    if s.rank > 0:
        peers.append((s.rank - 1, sel((J >= 1) & (J <= p)), sel(J == 0)))
    if s.rank < s.world - 1:
        peers.append((s.rank + 1, sel(J == top), sel((J > top) & (J <= top + p))))
    Jg = s.lo * p + J
    bnd = (Jg == 0) | (Jg == s.n_global[-1] * p)
    for d in range(s.dim - 1):
        bnd |= (L[:, d] == 0) | (L[:, d] == s.n_global[d] * p)
    return Plan(idx[not_owned].astype(np.int32), idx[bnd].astype(np.int32), peers,
                idx[~not_owned].astype(np.int32))


def box_ctrl(s: Slab, ext: Sequence[float]) -> np.ndarray:
    """Straight-element control points of the local block with the global
    make_cartesian vertex coordinates ext * i_global / n_global."""
    n = s.n_local
    dim = s.dim
    ne = int(np.prod(n))
    e = np.arange(ne)
    cell = [e % n[0], (e // n[0]) % n[1]] + ([e // (n[0] * n[1])] if dim == 3 else [])
    out = np.empty((ne, 2 ** dim, dim))
    for l in range(2 ** dim):
        for d in range(dim):
            i = cell[d] + ((l >> d) & 1) + s.origin[d]
            out[:, l, d] = ext[d] * i.astype(np.float64) / s.n_global[d]
    return out


# ------------------------------------------------------- GPU (one rank)
class DistOperator:
    """One rank's constrained PA diffusion operator with the halo / allreduce
    hooks wired to torch.distributed on the library stream."""

    def __init__(self, dev, slab: Slab, ext=None, kind="diffusion", transport=None):
        import torch
        import torch.distributed as tdist
        from . import abi
        from .tensorfem import BilinearForm, ConstrainedOperator, FeSpace
        self.slab = slab
        self.dev = dev
        ext = list(ext or [1.0] * slab.dim)
        self.space = FeSpace.cartesian_box(dev, slab.n_local, slab.origin, slab.n_global,
                                           slab.p, ext)
        L = lattice(self.space.element_dofs(), slab.n_local, slab.p, self.space.n_dofs)
        self.lattice = L
        self.plan = halo_plan(slab, L)
        self.form = BilinearForm(self.space)
        (self.form.add_diffusion if kind == "diffusion" else self.form.add_mass)(1.0)
        self.form.assemble()
        self.op = ConstrainedOperator(self.form, self.plan.ess)
        gpu = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.ExternalStream(dev.stream)
        if transport is None:
            transport = "nccl" if tdist.get_backend() == "nccl" else "hooks"
        self.transport = transport
        self.nccl = None
        if transport == "nccl":
            self._init_nccl(abi, tdist)
            self.diag = self.op.diagonal()
            return
        self.red = torch.zeros(4, dtype=torch.float64, device=gpu)
        self.bufs = []
        halo = abi.Halo()
        halo.n_peers = len(self.plan.peers)
        self._keep = []
        for k, (peer, s_idx, r_idx) in enumerate(self.plan.peers):
            sb = torch.empty(len(s_idx), dtype=torch.float64, device=gpu)
            rb = torch.empty(len(r_idx), dtype=torch.float64, device=gpu)
            self.bufs.append((peer, sb, rb))
            halo.n_send[k], halo.n_recv[k] = len(s_idx), len(r_idx)
            halo.send_idx[k] = s_idx.ctypes.data_as(abi.i32p)
            halo.recv_idx[k] = r_idx.ctypes.data_as(abi.i32p)
            halo.send_buf[k], halo.recv_buf[k] = sb.data_ptr(), rb.data_ptr()
            self._keep += [s_idx, r_idx]
        halo.red = self.red.data_ptr()

        nccl = tdist.get_backend() == "nccl"

        def exchange(_user):
            with torch.cuda.stream(self.stream):
                if nccl:
                    ops = []
                    for peer, sb, rb in self.bufs:
                        ops.append(tdist.P2POp(tdist.isend, sb, peer))
                        ops.append(tdist.P2POp(tdist.irecv, rb, peer))
                    if ops:
                        for w in tdist.batch_isend_irecv(ops):
                            w.wait()
                    return
                # host-staged fallback (gloo): correctness path for tests
                reqs, back = [], []
                for peer, sb, rb in self.bufs:
                    sc, rc = sb.cpu(), torch.empty(rb.shape, dtype=rb.dtype)
                    reqs += [tdist.isend(sc, peer), tdist.irecv(rc, peer)]
                    back.append((rb, rc, sc))
                for w in reqs:
                    w.wait()
                for rb, rc, _ in back:
                    rb.copy_(rc)

        def allreduce(k, _user):
            with torch.cuda.stream(self.stream):
                if nccl:
                    tdist.all_reduce(self.red[:k])
                else:
                    t = self.red[:k].cpu()
                    tdist.all_reduce(t)
                    self.red[:k].copy_(t)

        self._hooks = (abi.EXCHANGE_HOOK(exchange), abi.ALLREDUCE_HOOK(allreduce))
        self.comm = abi.Comm(self._hooks[0], self._hooks[1], None)
        no = self.plan.not_owned
        abi.check(abi.lib().tfem_operator_set_comm(self.op.h, C.byref(self.comm), C.byref(halo),
                                                   len(no),
                                                   no.ctypes.data_as(abi.i32p) if len(no) else None))
        self._halo = halo
        self.diag = self.op.diagonal()

    def _init_nccl(self, abi, tdist):
        """The library's own communicator: rank 0's NCCL id over
        torch.distributed, then the halo plan with library-owned buffers."""
        rank, world = self.slab.rank, self.slab.world
        idbuf = C.create_string_buffer(abi.NCCL_ID_BYTES)
        if rank == 0:
            abi.check(abi.lib().tfem_nccl_unique_id(idbuf))
        obj = [idbuf.raw if rank == 0 else None]
        tdist.broadcast_object_list(obj, src=0)
        idbuf = C.create_string_buffer(obj[0], abi.NCCL_ID_BYTES)
        h = abi.vp()
        abi.check(abi.lib().tfem_nccl_create(self.dev.h, world, rank, idbuf, C.byref(h)))
        self.nccl = h
        peers = self.plan.peers
        k = len(peers)
        peer = (C.c_int * max(k, 1))(*[pr for pr, _, _ in peers])
        n_send = (C.c_int64 * max(k, 1))(*[len(s) for _, s, _ in peers])
        n_recv = (C.c_int64 * max(k, 1))(*[len(r) for _, _, r in peers])
        self._keep = [x for _, s, r in peers for x in (s, r)]
        s_idx = (abi.i32p * max(k, 1))(*[s.ctypes.data_as(abi.i32p) for _, s, _ in peers])
        r_idx = (abi.i32p * max(k, 1))(*[r.ctypes.data_as(abi.i32p) for _, _, r in peers])
        no = self.plan.not_owned
        abi.check(abi.lib().tfem_operator_set_nccl(
            self.op.h, h, k, peer, n_send, s_idx, n_recv, r_idx, len(no),
            no.ctypes.data_as(abi.i32p) if len(no) else None))

    def close(self):
        from . import abi
        if getattr(self, "op", None) is not None:
            self.op = None  # the operator references the communicator
        if getattr(self, "nccl", None):
            abi.lib().tfem_nccl_destroy(self.nccl)
            self.nccl = None

    @property
    def n_owned(self) -> int:
        return len(self.plan.owned)


def bench_distributed(args, rank: int, world: int, local: int):
    """Weak-scaling BP3: ~10M DOFs per rank, global mesh n x (world n)."""
    import torch
    import torch.distributed as tdist
    import paper_1911_09220_b200 as tf

    if getattr(args, "bp", 3) != 3:
        raise SystemExit("bench: the distributed run is BP3 (diffusion, Jacobi) only")
    # one GPU per rank; the CG's halo / dots go through the library's own
    # NCCL communicator (DistOperator, transport "nccl"); the process group
    # ships its id, and times the run (barrier, max over ranks)
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl", rank=rank, world_size=world,
                             device_id=torch.device("cuda", local))
    dev = tf.Device(local, numerics=args.numerics)
    n = args.cells or {2: round((10.0e6 ** 0.5 - 1) / args.order),
                   3: round((10.0e6 ** (1 / 3) - 1) / args.order)}[args.dim]
    # weak (default): ~10M DOFs per rank, the last axis grows with the ranks;
    # strong (--strong): one fixed global mesh n^dim cut into `world` slabs
    # (C2 at 10M, or C5's 333^3 ~ 1B DOFs in 3D)
    strong = getattr(args, "strong", False)
    n_global = (n,) * args.dim if strong else (n,) * (args.dim - 1) + (n * world,)
    slab = partition(args.dim, n_global, args.order, rank, world)
    t0 = time.perf_counter()
    d = DistOperator(dev, slab)
    setup_s = time.perf_counter() - t0
    N_local = d.space.n_dofs
    b_host = np.random.default_rng(2020 + rank).uniform(-1.0, 1.0, N_local)
    b_host[d.plan.ess] = 0.0
    b = tf.Vector.from_numpy(dev, b_host)
    x = tf.Vector(dev, N_local)
    n_owned = torch.tensor([d.n_owned], dtype=torch.float64, device="cuda")
    tdist.all_reduce(n_owned)
    N_global = int(n_owned.item())

    def step():
        return tf.cg_solve(d.op, b, 0.0, args.iters, d.diag, x=x)

    for _ in range(args.warmup):
        res = step()
    assert res.iterations == args.iters
    stream = d.stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = dev.launch_count()
    torch.cuda.synchronize()
    tdist.barrier()
    dev.sync()
    from bench import Clocks  # noqa: E402  (repo root on sys.path)
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    tdist.barrier()
    t = torch.tensor([ev0.elapsed_time(ev1) / 1e3], dtype=torch.float64, device="cuda")
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    t_max = float(t.item())
    launches = dev.launch_count() - launches0
    value = N_global * args.iters * args.steps / t_max / 1e9

    # e2e: host buffers through the C ABI on every rank
    e2e = None
    if not args.no_e2e:
        bp = torch.from_numpy(b_host).pin_memory()
        dp = torch.from_numpy(d.diag.numpy()).pin_memory()
        xp = torch.empty(N_local, dtype=torch.float64).pin_memory()
        tf.cg_solve_host(d.op, bp.numpy(), 0.0, args.iters, dp.numpy(), out=xp.numpy())
        tdist.barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            tf.cg_solve_host(d.op, bp.numpy(), 0.0, args.iters, dp.numpy(), out=xp.numpy())
        dev.sync()
        te = torch.tensor([time.perf_counter() - w0], dtype=torch.float64, device="cuda")
        tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
        e2e = {"value": N_global * args.iters * args.steps / float(te.item()) / 1e9,
               "unit": "GDOF/s", "h2d_bytes_per_step": 16 * N_local * world,
               "d2h_bytes_per_step": 8 * N_local * world,
               "api": "tfem_cg_solve_host on every rank"}
    if rank == 0:
        from bench import METRIC, config_of, peaks
        peak, _ = peaks()
        # algorithmic bytes per DOF-iteration of BP3, this rank's slab
        nc, nq = (3 if args.dim == 2 else 6), args.order + 2
        E = d.space.n_elements
        b_op = E * (nc * nq ** args.dim * 8 + (args.order + 1) ** args.dim * 4) + 16 * N_local
        b_it = (b_op + 96 * N_local) / N_local
        line = {
            "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": config_of(args, n, args.order, N_global // world, world=world),
            # the distributed run times the whole CG iteration (no per-kernel
            # split): algorithmic bytes of an iteration per GPU / its time
            "roofline": {"bound": "hbm", "achieved": b_it * value / world, "peak": peak,
                         "unit": "GB/s", "frac": b_it * value / world / peak, "traffic": None,
                         "kernel": "whole CG iteration per GPU (operator + vector kernels "
                                   "+ halo / allreduce)",
                         "bytes_per_dof_iteration": b_it},
            "cg_roofline": {"achieved_per_gpu": b_it * value / world, "unit": "GB/s",
                            "frac": b_it * value / world / peak},
            "e2e": e2e, "cpu_baseline": None, "clocks": clk.summary(),
            "gpu_launches": launches, "setup_s": setup_s,
            "partition": f"{world} slabs of {slab.hi - slab.lo} cell layers + 1 ghost layer",
            "transport": "library NCCL (ncclSend/ncclRecv halo + ncclAllReduce dots, "
                         "captured in the CG graphs)",
        }
        print(json.dumps(line))
    tdist.barrier()
    d.close()
    tdist.destroy_process_group()
