# Debug aid: device CG residual / threshold around the reference stop on NC forests
# (PYTHONPATH=. python tools/nc_cg_probe.py on a GPU box).
import numpy as np
from oracle.pyoracle import RefSpace, RefForm, RefSystem
import paper_1911_09220_b200 as tf
import sys
sys.path.insert(0, "tests")
from test_gpu_nc import nc_space
dev = tf.Device(0, numerics="reference")
for p in (1, 2, 3):
    rs, sp = nc_space(dev, 4, p, 10, 21 + p)
    f = RefForm(rs, [("diffusion", "const", 1.0)])
    rsys = RefSystem(f, "front")
    a = tf.BilinearForm(sp); a.add_diffusion(1.0); a.assemble()
    op = tf.ConstrainedOperator(a, rsys.ess); d = op.diagonal()
    xr, itr, cr, _ = rsys.cg(1e-12, 3000, True)
    thr = 1e-12 * np.linalg.norm(rsys.rhs)
    for k in (itr - 1, itr, itr + 1):
        r = tf.cg_solve(op, rsys.rhs, 0.0, k, d)
        print(p, itr, k, r.final_norm / thr)
