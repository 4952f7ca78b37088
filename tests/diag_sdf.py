"""Diagnostic (not collected): phase timing of sdf.build_sdf at the metrics' resolutions."""
import json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2503_05020_b200 import sdf as sdfm
from test_metrics import _golden_env  # noqa: E402
env, _ = _golden_env()
g = json.loads((ROOT / "tests" / "golden" / "metrics.json").read_text())
r = env.records[g["object_body"]]
v, t = np.asarray(r["xi"]), np.asarray(r["body"].surface.triangles)
for res in (32, 128):
    T = {}
    t0 = time.perf_counter()
    s = sdfm.build_sdf(v, t, resolution=res, timings=T)
    print(res, s.values.shape, f"total {time.perf_counter() - t0:.2f} s", {k: round(x, 3) for k, x in T.items()})
