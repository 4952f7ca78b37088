"""Diagnostic (not collected): phase breakdown of k_assemble_direct (GRIP_PHASE_TIMING build)."""
import ctypes, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench
sys.argv = ["bench.py", "--no-cpu", "--steps", "100", "--warmup", "200"] + sys.argv[1:]
bench.main()
from paper_2503_05020_b200 import _native as nv
out = (ctypes.c_ulonglong * 64)()
assert nv._lib.grip_debug_phase(out) == 0
v = np.array(list(out), float)
names = ["prologue", "static", "scatter", "cholesky", "solve", "refine", "converge"]
print(f"CTAs {v[8]:.0f} mean nce {v[9] / v[8]:.1f}  heavy(>128) CTAs {v[24]:.0f} mean nce {v[25] / max(v[24], 1):.1f}  max nce {v[41]:.0f}  max CTA cyc {v[40]:.0f}  smem {v[42]:.0f}")
for k, nm in enumerate(names):
    print(f"{nm:10s} all {v[k] / v[8]:10.0f}   heavy {v[16 + k] / max(v[24], 1):10.0f}")
print("nseg>=2", v[43], "shifted", v[44], "chol cyc when nseg<2", v[45] / max(v[46], 1), v[46])
pn = ["incidence", "energy", "grad_sv", "grad_nodes+abd", "nonfinite", "static_blocks"]
for k, nm in enumerate(pn):
    print(f"  prologue.{nm:15s} {v[48 + k] / v[8]:10.0f}")
print(f"cholesky: segment panels {v[56] / v[8]:.0f}  tail x tail {v[57] / v[8]:.0f}  hub panels {v[58] / v[8]:.0f}"
      f"  mean segments {v[59] / v[8]:.2f}  mean n {v[60] / v[8]:.1f}  mean tail {v[61] / v[8]:.1f}")
