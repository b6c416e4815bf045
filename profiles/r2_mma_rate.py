"""Issue rate of tcgen05.mma step shapes in isolation (hivf_debug_mma_rate):
SS f16 / SS tf32 / f16 with A in TMEM / tcgen05.cp + TS f16, M=128, N = 8..256.
Also checks that modes 0, 2, 3 produce identical accumulators.
    python profiles/r2_mma_rate.py > gpurun_out/mma_rate.txt"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2507_09138_b200 import Context, lib  # noqa: E402

Context(0)
L = lib()
rng = np.random.default_rng(1)
A = rng.standard_normal((128, 32)).astype(np.float32)
B = rng.standard_normal((256, 32)).astype(np.float32)
names = {0: "f16 SS", 1: "tf32 SS", 2: "f16 TS (A in TMEM)", 3: "cp + f16 TS"}
for n in (8, 16, 32, 64, 128, 256):
    row = []
    outs = {}
    for mode in range(4):
        cyc = C.c_double()
        d = np.zeros((128, 32), np.float32)
        rc = L.hivf_debug_mma_rate(mode, n, 4096, A.ctypes.data, B.ctypes.data, C.byref(cyc), d.ctypes.data)
        assert rc == 0, rc
        outs[mode] = d
        row.append("%s %.1f" % (names[mode], cyc.value))
    same = all(np.array_equal(outs[0], outs[m]) for m in (2, 3))
    print("N=%3d  " % n + " | ".join(row) + "  | f16 modes identical: %s" % same)
print("stage blocks (8 MMAs per warp-collective asm, mma_stage8_f16): cycles per MMA")
for n in (8, 16, 32, 64, 128, 256):
    cyc = C.c_double()
    d = np.zeros((128, 32), np.float32)
    assert L.hivf_debug_mma_rate(12, n, 4096, A.ctypes.data, B.ctypes.data, C.byref(cyc), d.ctypes.data) == 0
    print("N=%3d  stage8 %.1f" % (n, cyc.value))
print("independent accumulators (f16 SS, round robin): cycles per MMA")
for n in (16, 32):
    row = []
    for nd in (1, 2, 4, 8):
        cyc = C.c_double()
        d = np.zeros((128, 32), np.float32)
        assert L.hivf_debug_mma_rate(3 + nd, n, 4096, A.ctypes.data, B.ctypes.data, C.byref(cyc), d.ctypes.data) == 0
        row.append("%d acc: %.1f" % (nd, cyc.value))
    print("N=%3d  " % n + " | ".join(row))
