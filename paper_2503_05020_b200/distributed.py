"""Environment sharding across GPUs and the one collective of the path.

Envs are independent (multienv.py:1-12), so a run over G GPUs is G
independent batches: rank r owns its own candidates (a contiguous shard of the job list)
and steps them with no per-step communication.  The only exchange is at the end: every
rank's finished-trial outcome records (fixed size, 13 doubles per trial) are gathered to
all ranks with one ``all_gather`` -- NCCL over NVLink 5 / NVSwitch on the GPU box, gloo in
the CPU tests.  Trajectories and stress stay rank-local: each rank writes its own dataset
shard and rank 0 merges the shard manifests (dataset.py:150-171 ``emit_dataset``'s manifest).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

VERDICTS = ("stable", "unstable", "sim-failed")

# fixed-size outcome record per finished trial (float64 fields)
OUTCOME_FIELDS = ("job", "verdict", "n_steps", "final_com_disp", "halt_step0", "halt_step1", "halt_force0",
                  "halt_force1", "final_contact", "fail_reason", "min_distance", "min_J", "rank")


def shard(n_envs, world, rank):
    """Contiguous env range [lo, hi) of `rank` (ceil split, last ranks may get fewer)."""
    per = -(-n_envs // world)
    lo = min(rank * per, n_envs)
    return lo, min(lo + per, n_envs)


def pack_outcomes(records, job_ids, finger_names=("finger0", "finger1"), rank=0, reasons=None):
    """Finished TrialRecords -> (n, len(OUTCOME_FIELDS)) float64 array."""
    inv = {v: k for k, v in (reasons or {}).items()}
    out = np.full((len(records), len(OUTCOME_FIELDS)), np.nan)
    for k, (r, j) in enumerate(zip(records, job_ids)):
        out[k, 0] = j
        out[k, 1] = VERDICTS.index(r.verdict) if r.verdict in VERDICTS else -1   # -1: trial still running
        out[k, 2] = r.n_steps
        out[k, 3] = r.metrics.get("final_phase_com_disp", np.nan)
        for i, f in enumerate(finger_names[:2]):
            h = r.halt_forces.get(f)
            if h:
                out[k, 4 + i] = h["step"]
                out[k, 6 + i] = h["force"]
        out[k, 8] = float(r.metrics.get("final_contact", False))
        out[k, 9] = inv.get(r.failure.get("reason"), -1) if r.failure else 0
        out[k, 10] = getattr(r, "min_distance", np.inf)
        out[k, 11] = getattr(r, "min_J", np.inf)
        out[k, 12] = rank
    return out


def gather_outcomes(local, device=None):
    """All-gather every rank's outcome rows (any count per rank) and return them sorted by job
    (then rank).  One all_gather of the counts, one of the rows padded to the largest count."""
    import torch
    import torch.distributed as dist

    def order(a):
        return a[np.lexsort((a[:, 12], a[:, 0]))] if len(a) else a

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return order(local)
    world = dist.get_world_size()
    n = torch.tensor([len(local)], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    per = max(int(c.item()) for c in counts)
    pad = np.full((max(per, 1), len(OUTCOME_FIELDS)), np.nan)
    pad[:len(local)] = local
    t = torch.as_tensor(pad, dtype=torch.float64, device=device)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t)
    allr = torch.cat(bufs).cpu().numpy()
    allr = allr[~np.isnan(allr[:, 0])]
    return order(allr)


def rank_dir(out_dir, rank):
    """Rank-local dataset shard directory (trajectories and stress never leave their rank)."""
    return Path(out_dir) / f"rank{rank:02d}"


def merge_manifests(out_dir, world, fmt):
    """Rank 0, after a barrier: one top-level manifest over every rank's shard manifest, trial
    dirs relative to out_dir (dataset.py:150-171)."""
    out = Path(out_dir)
    trials = []
    for r in range(world):
        d = rank_dir(out, r)
        m = json.loads((d / "manifest.json").read_text())
        for t in m["trials"]:
            t = dict(t)
            t["dir"] = f"{d.name}/{t['dir']}"
            t["rank"] = r
            trials.append(t)
    trials.sort(key=lambda t: (t["id"], t["rank"]))
    manifest = {"format": fmt, "n_trials": len(trials), "trials": trials}
    (out / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True))
    return manifest
