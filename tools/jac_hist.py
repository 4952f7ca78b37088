"""Jacobi sweep histogram of the eigen-clamp in the bench's steady state (diagnostic).

Loads the GRIP_JAC_HIST build (build/libgripipc_jachist.so, __graft_entry__.build_variant) through
GRIP_LIB, runs the config-2 bench workload (400 envs, 3 lanes, device protocol) until every slot
finished a trial, resets the counters, runs `--rounds` more rounds of the main lane and prints how
many sweeps each deferred matrix took: tets (warm-started from the previous Newton iteration's
eigenbasis) and contact / friction elements (cold).

  GRIP_LIB=build/libgripipc_jachist.so python tools/jac_hist.py [--rounds 64] [--out gpurun_out/jac_hist.json]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=64)
    ap.add_argument("--maxsweep", type=int, default=30)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "jac_hist.json"))
    args = ap.parse_args()
    os.environ.setdefault("GRIP_LIB", str(ROOT / "build" / "libgripipc_jachist.so"))
    import bench
    from paper_2503_05020_b200 import _native

    class A:
        global_envs = 0
        protocol = "auto"
        record = None
        lanes_per_kind = 3
        rounds_per_call = 1
        lane_priority = True

    runner, _, _, _ = bench.build_runner(A, 2, 400, 0, 1)
    runner.run(main_calls=8, min_trials=runner.n_slots)
    lib = _native.load()
    h = np.zeros((2, args.maxsweep + 1), np.uint64)
    fn = lib.grip_jac_hist
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    fn(h.ctypes.data, 1)
    runner.run(main_calls=max(1, args.rounds // A.rounds_per_call))
    fn(h.ctypes.data, 1)
    out = {}
    for k, name in enumerate(("tets", "contacts")):
        c = h[k].astype(np.int64)
        n = int(c.sum())
        mean = float((np.arange(len(c)) * c).sum() / max(n, 1))
        out[name] = {"matrices": n, "mean_sweeps": mean, "hist": c.tolist(),
                     "at_cap": int(c[-1])}
        print(name, json.dumps(out[name]))
    Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
