"""Diagnostic (not collected): snapshots of every env's surface positions during the bench's
steady state, for offline broad-phase cost analysis (gpurun_out/bp_snap.npz)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2503_05020_b200 import scene as sc
from paper_2503_05020_b200.multienv import DeviceEnvGroup
from paper_2503_05020_b200.protocol import BatchedGraspTrials
from paper_2503_05020_b200.solver import Environment

cands = sc.load_cfg2_candidates()
scenes = [sc.cfg2_scene(i, cands) for i in range(400)]
envs = [Environment(s.bodies, collide_pairs_off=s.collide_pairs_off) for s in scenes]
group = DeviceEnvGroup(envs, device=0)
trials = BatchedGraspTrials(group, scenes)
snaps, phases = [], []
for r in range(400):
    trials.advance_round()
    if r % 20 == 19:
        snaps.append(group.dev.surface())
        phases.append(trials.phase.copy())
np.savez_compressed(ROOT / "gpurun_out" / "bp_snap.npz", sv=np.array(snaps), phase=np.array(phases),
                    sv_off=group.packed.sv_off)
print("saved", len(snaps))
