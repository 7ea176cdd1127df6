"""Debug helper: 2 gloo ranks on one GPU vs the single-device solve, step by step."""
import socket, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def rank_main(rank, world, port, n, p):
    import torch, torch.distributed as tdist
    import paper_1911_09220_b200 as tf
    from paper_1911_09220_b200 import abi
    from paper_1911_09220_b200.dist import DistOperator, lattice, partition
    import ctypes as C
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    dev = tf.Device(0)
    d = DistOperator(dev, partition(len(n), n, p, rank, world))
    sp = tf.FeSpace.cartesian(dev, n, p)
    a = tf.BilinearForm(sp); a.add_diffusion(1.0); a.assemble()
    ess = sp.essential_true_dofs()
    op = tf.ConstrainedOperator(a, ess)
    Lg = lattice(sp.element_dofs(), n, p, sp.n_dofs)
    dims = tuple(k * p + 1 for k in n)
    table = np.full(int(np.prod(dims)), -1, dtype=np.int64)
    table[np.ravel_multi_index(tuple(Lg.T), dims, order="F")] = np.arange(len(Lg))
    L = d.lattice.copy(); L[:, -1] += d.slab.lo * p
    l2g = table[np.ravel_multi_index(tuple(L.T), dims, order="F")]
    own = d.plan.owned
    bg = np.random.default_rng(8).uniform(-1, 1, sp.n_dofs); bg[ess] = 0.0
    dg = op.diagonal().numpy()
    print(rank, "diag owned equal:", (d.diag.numpy()[own] == dg[l2g[own]]).all(), flush=True)
    print(rank, "ess local", len(d.plan.ess), "notown", len(d.plan.not_owned), "peers",
          [(pp, len(s), len(r)) for pp, s, r in d.plan.peers], flush=True)
    for its in (0, 1, 2, 3, 5, 10):
        rd = abi.CgResult(); rg = abi.CgResult()
        xd = tf.Vector(dev, d.space.n_dofs); xg = tf.Vector(dev, sp.n_dofs)
        bd = tf.Vector.from_numpy(dev, bg[l2g]); bgv = tf.Vector.from_numpy(dev, bg)
        abi.check(abi.lib().tfem_cg_solve(dev.h, d.op.h, bd.h, 0.0, its, d.diag.h, xd.h, C.byref(rd), abi.CG_CALLBACK(0), None))
        dgv = tf.Vector.from_numpy(dev, dg)
        abi.check(abi.lib().tfem_cg_solve(dev.h, op.h, bgv.h, 0.0, its, dgv.h, xg.h, C.byref(rg), abi.CG_CALLBACK(0), None))
        xdn, xgn = xd.numpy(), xg.numpy()
        err = np.abs(xdn[own] - xgn[l2g[own]]).max() if its else 0
        print(rank, its, "bnorm", rd.initial_norm, rg.initial_norm, "rnorm", rd.final_norm, rg.final_norm, "xerr", err, flush=True)
    tdist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    n = (24, 18); p = 3
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=rank_main, args=(r, 2, port, n, p)) for r in range(2)]
    [x.start() for x in ps]; [x.join(timeout=200) for x in ps]
