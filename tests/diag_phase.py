"""Diagnostic (not collected): phase breakdown of k_assemble_direct (GRIP_PHASE_TIMING build)."""
import ctypes, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench
sys.argv = ["bench.py", "--no-cpu", "--steps", "100", "--warmup", "200"]
bench.main()
from paper_2503_05020_b200 import _native as nv
out = (ctypes.c_ulonglong * 16)()
assert nv._lib.grip_debug_phase(out) == 0
v = np.array(list(out), float)
names = ["prologue", "dense_assemble", "cholesky", "solve", "refine", "converge"]
tot = v[:6].sum()
for k, nm in enumerate(names):
    print(f"{nm:16s} {100 * v[k] / tot:5.1f}%  {v[k] / v[8]:10.0f} cyc/CTA")
print("CTAs", v[8], "mean n", v[9] / v[8], "mean contact elems", v[10] / v[8], "regularized", v[11])
