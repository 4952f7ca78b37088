"""Per-CTA wall-time histogram of the CTA-per-env kernels in the bench's steady state.

Loads the GRIP_CTA_TIMING diagnostic build (build/libgripipc_ctatime.so, __graft_entry__.build_ctatime)
through GRIP_LIB, runs the config-2 bench workload (400 envs, 3 lanes, device protocol) to a steady
phase mix, then records every CTA of k_begin / k_candidates / k_assemble_direct / k_linesearch /
k_finalize for `--rounds` rounds.  Per kernel: launch span (first CTA start to last CTA end), mean /
p50 / p90 / max duration of the CTAs that did work, span / mean-CTA ratio (the "heavy-env tail"),
and a log2 histogram of CTA durations.

  GRIP_LIB=build/libgripipc_ctatime.so python tools/cta_hist.py [--rounds 64] [--out profiles/r2_cta_hist.json]
"""

from __future__ import annotations

import argparse
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
    ap.add_argument("--envs", type=int, default=400)
    ap.add_argument("--min-ns", type=int, default=3000, help="CTAs shorter than this did no work (skipped env)")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r2_cta_hist.json"))
    args = ap.parse_args()
    if "GRIP_LIB" not in os.environ:
        os.environ["GRIP_LIB"] = str(ROOT / "build" / "libgripipc_ctatime.so")
    import bench
    from paper_2503_05020_b200._native import DeviceBatch

    class A:
        global_envs = 0
        protocol = "auto"
        record = None
        lanes_per_kind = 3
        rounds_per_call = 1
        lane_priority = True

    runner, jobs, _, _ = bench.build_runner(A, 2, args.envs, 0, 1)
    runner.run(main_calls=8, min_trials=runner.n_slots)
    for ln in runner.lanes:
        ln.dev.cta_records(reset=True)
    runner.run(main_calls=max(1, args.rounds // A.rounds_per_call))
    out = {"workload": "bench config 2 (400 envs, 3 lanes by object kind, device protocol), steady state",
           "lib": os.environ["GRIP_LIB"], "rounds_main_lane": args.rounds, "min_ns": args.min_ns, "kernels": {}}
    recs = []
    for li, ln in enumerate(runner.lanes):
        r = ln.dev.cta_records(reset=True)
        recs.append((li, int(ln.key), r))
    for k, name in enumerate(DeviceBatch.CTA_KERNELS):
        spans, ratios, durs, per_lane = [], [], [], {}
        infos, longest_info = [], []
        for li, key, r in recs:
            rk = r[r["kernel"] == k]
            for seq in np.unique(rk["seq"]):
                c = rk[rk["seq"] == seq]
                t0 = c["t0"].astype(np.int64)
                t0 = (t0 - t0.min()) % (1 << 32)            # low 32 bits of the ns timer
                end = t0 + c["dur"].astype(np.int64)
                work = c["dur"] >= args.min_ns
                if not work.any():
                    continue
                span = float(end[work].max() - t0[work].min())
                m = float(c["dur"][work].mean())
                spans.append(span)
                ratios.append(span / m)
                durs.extend(c["dur"][work].tolist())
                infos.extend(c["info"][work].tolist())
                longest_info.append(int(c["info"][work][np.argmax(c["dur"][work])]))
                per_lane.setdefault(key, []).append(span)
        if not durs:
            continue
        d = np.array(durs, float)
        bins = [int(2 ** b) for b in range(10, 24)]
        hist, _ = np.histogram(d, bins=bins)
        out["kernels"][name] = {
            "launches": len(spans), "ctas_with_work": int(len(d)),
            "launch_span_us": {"mean": float(np.mean(spans)) / 1e3, "p90": float(np.percentile(spans, 90)) / 1e3},
            "cta_us": {"mean": float(d.mean()) / 1e3, "p50": float(np.median(d)) / 1e3,
                       "p90": float(np.percentile(d, 90)) / 1e3, "max": float(d.max()) / 1e3},
            "span_over_mean_cta": {"mean": float(np.mean(ratios)), "p90": float(np.percentile(ratios, 90))},
            "span_us_by_lane_key": {str(kk): float(np.mean(v)) / 1e3 for kk, v in per_lane.items()},
            "hist_ns_log2_edges": bins, "hist_counts": hist.tolist(),
        }
        # kernel-specific CTA detail (CTA_INFO): line search bit 0 = fresh broad phase, bit 1 =
        # tet filter halvings, bits 8.. = extra energy passes; candidates bit 0 = superset rebuild
        iv = np.array(infos)
        by = {}
        for v in np.unique(iv):
            sel = iv == v
            by[str(int(v))] = {"ctas": int(sel.sum()), "mean_us": float(d[sel].mean()) / 1e3,
                               "max_us": float(d[sel].max()) / 1e3,
                               "launches_where_longest": int(sum(1 for x in longest_info if x == v))}
        out["kernels"][name]["by_info"] = by
        print(name, json.dumps({kk: out["kernels"][name][kk] for kk in ("launch_span_us", "cta_us", "span_over_mean_cta")}))
    Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
