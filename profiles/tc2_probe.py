"""Layout probe of the CTA-pair tensor-core MMA (tcgen05.mma.cta_group::2,
M = 256): which CTA's shared memory must hold which half of B, and where the
results land (hivf_debug_tc2_dot).  Prints, per configuration, the columns of
each CTA's rows that equal the exact A.B^T."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2507_09138_b200 import Context, lib
Context(0)
rng = np.random.default_rng(3)
D = 64
tf = lambda x: (x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
A = tf(rng.standard_normal((256, D)))
for n in (16, 32):
    B = tf(rng.standard_normal((n, D)))
    ex = A.astype(np.float64) @ B.astype(np.float64).T
    for bsplit in (1, 0):
        out = np.zeros((256, n), np.float32)
        rc = lib().hivf_debug_tc2_dot(A.ctypes.data, B.ctypes.data, D, n, bsplit, out.ctypes.data)
        ok = np.abs(out - ex) <= 1e-3 * (1 + np.abs(ex))
        print(f"n={n} bsplit={bsplit} rc={rc}: CTA0 rows ok cols {np.where(ok[:128].all(0))[0].tolist()}; "
              f"CTA1 rows ok cols {np.where(ok[128:].all(0))[0].tolist()}; all_ok={bool(ok.all())}")
        if not ok.all():
            # which B row does each output column of CTA0 / CTA1 correspond to?
            for c0, c1 in ((0, 128), (128, 256)):
                m = []
                for j in range(n):
                    errs = [np.abs(out[c0:c1, j] - ex[c0:c1, jj]).max() for jj in range(n)]
                    m.append(int(np.argmin(errs)) if min(errs) < 1e-2 else -1)
                print(f"   rows {c0}-{c1}: out col -> B row {m}")
