"""Environment sharding across GPUs and the one collective of the path.

Envs are independent (multienv.py:1-12), so a run over G GPUs is G
independent batches: rank r owns a contiguous env range and steps it with no
per-step communication.  The only exchange is at the end: every rank's
per-env outcome records (fixed size, ~100 B per env) are gathered to all
ranks with one ``all_gather`` -- NCCL over NVLink 5 / NVSwitch on the GPU box,
gloo in the CPU tests.
"""

from __future__ import annotations

import numpy as np

VERDICTS = ("stable", "unstable", "sim-failed")

# fixed-size outcome record per env (float64 fields)
OUTCOME_FIELDS = ("env", "verdict", "n_steps", "final_com_disp", "halt_step0", "halt_step1", "halt_force0",
                  "halt_force1", "final_contact")


def shard(n_envs, world, rank):
    """Contiguous env range [lo, hi) of `rank` (ceil split, last ranks may get fewer)."""
    per = -(-n_envs // world)
    lo = min(rank * per, n_envs)
    return lo, min(lo + per, n_envs)


def pack_outcomes(records, env_ids, finger_names=("finger0", "finger1")):
    """TrialRecords -> (n, len(OUTCOME_FIELDS)) float64 array."""
    out = np.full((len(records), len(OUTCOME_FIELDS)), np.nan)
    for k, (r, e) in enumerate(zip(records, env_ids)):
        out[k, 0] = e
        out[k, 1] = VERDICTS.index(r.verdict) if r.verdict in VERDICTS else -1   # -1: trial still running
        out[k, 2] = r.n_steps
        out[k, 3] = r.metrics.get("final_phase_com_disp", np.nan)
        for j, f in enumerate(finger_names[:2]):
            h = r.halt_forces.get(f)
            if h:
                out[k, 4 + j] = h["step"]
                out[k, 6 + j] = h["force"]
        out[k, 8] = float(r.metrics.get("final_contact", False))
    return out


def gather_outcomes(local, n_envs, device=None):
    """All-gather every rank's outcome rows (padded to the shard size) and return them sorted by env."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return local[np.argsort(local[:, 0])] if len(local) else local
    world = dist.get_world_size()
    per = -(-n_envs // world)
    pad = np.full((per, local.shape[1]), np.nan)
    pad[:len(local)] = local
    t = torch.as_tensor(pad, dtype=torch.float64, device=device)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t)
    allr = torch.cat(bufs).cpu().numpy()
    allr = allr[~np.isnan(allr[:, 0])]
    return allr[np.argsort(allr[:, 0])]
