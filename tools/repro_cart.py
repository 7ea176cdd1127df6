# tools/repro_cart.py P KIND -- one small Cartesian apply + diagonal (debug aid)
import sys
import numpy as np
import paper_1911_09220_b200 as tf
p, kind = int(sys.argv[1]), sys.argv[2]
numerics = sys.argv[3] if len(sys.argv) > 3 else "reference"
dev = tf.Device(0, numerics=numerics)
sp = tf.FeSpace.cartesian(dev, (5, 4), p, extents=(2.0, 1.0))
pa = tf.pa_setup(sp, kind, lambda q: 1.0 + q[..., 0] + 2.0 * q[..., 1])
print("qdata", pa.qdata().shape, flush=True)
y = tf.Vector(dev, sp.n_dofs)
tf.pa_apply_local(pa, sp, tf.Vector.from_numpy(dev, np.ones(sp.n_dofs)), y)
print("apply ok", y.numpy().sum(), flush=True)
print("diag", tf.pa_diagonal(pa, sp).numpy().sum(), flush=True)
