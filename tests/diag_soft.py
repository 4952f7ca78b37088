"""Diagnostic (not collected by pytest): per-step Newton path of the soft-object scene,
GPU vs oracle, both restarted from the reference's recorded state every step."""

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import solver as osv  # noqa: E402
from paper_2503_05020_b200 import scene as sc  # noqa: E402
from paper_2503_05020_b200.solver import Environment  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "soft"
rtol = float(sys.argv[2]) if len(sys.argv) > 2 else None
d = np.load(ROOT / "tests" / "golden" / f"traj_{name}.npz")
golden = json.loads(str(d["reports_json"]))


def scene():
    return sc.build_trial_scene(sc.ObjectSpec(kind=str(d["kind"]), soft=bool(d["soft_object"])),
                                sc.GripperSpec(soft_fingers=bool(d["soft_fingers"])),
                                d["cand_R"], d["cand_T"], float(d["cand_opening"]))


s1, s2 = scene(), scene()
sp = sc.SolverParams()
if rtol:
    sp.pcg_rtol = rtol
env = Environment(s1.bodies, collide_pairs_off=s1.collide_pairs_off, solver_params=sp)
ref = osv.OracleEnv(s2.bodies, collide_pairs_off=s2.collide_pairs_off)
for f, ids in s1.finger_links.items():
    for b in ids:
        env.bodies[b].velocity = s1.closing_dirs[f] * 0.05
        ref.bodies[b].velocity = s1.closing_dirs[f] * 0.05
halted = {f: False for f in s1.finger_links}
ell = 0.1
for k in range(min(len(golden), 25)):
    if k == 18:
        env.gravity = np.array([0, 0, -9.8])
        ref.gravity = np.array([0, 0, -9.8])
    r = env.step()
    rr = ref.step()
    ev = ref.events_now()
    forces = {f: osv.finger_force(ev, ids) for f, ids in s1.finger_links.items()}
    err = np.abs(env.x - ref.x).max() / ell
    ga = np.array(r.alpha_history)
    oa = np.array(rr["alphas"])
    first = next((i for i in range(min(len(ga), len(oa))) if ga[i] != oa[i]), None)
    m = min(len(ga), len(oa))
    first = (first, float(np.abs(ga[:m] - oa[:m]).max() / max(oa[:m].max(), 1e-300)) if m else 0.0)
    print(f"step {k:2d} it gpu {r.iterations:3d} ora {rr['iterations']:3d} gold {golden[k]['iterations']:3d} "
          f"res {r.residual:.6e} {rr['residual']:.6e} |dx|/l {err:.2e} pcg {r.pcg_iterations} "
          f"first-alpha-diff {first}", flush=True)
    # resync the GPU env to the oracle state so each step starts identical
    grp = env._owner()
    kin = np.zeros((env.n_sv, 3))
    svr = ref.surface_positions()
    for rec in env.layout.records:
        if rec.kind == "kinematic":
            kin[rec.surf0:rec.surf0 + rec.n_sv] = svr[rec.surf0:rec.surf0 + rec.n_sv]
    grp.dev.set_state(ref.x.reshape(-1, 3), ref.v.reshape(-1, 3), kin)
    grp.invalidate()
    for f in s1.finger_links:
        if not halted[f] and forces[f] > 50:
            halted[f] = True
            for b in s1.finger_links[f]:
                env.bodies[b].velocity = np.zeros(3)
                ref.bodies[b].velocity = np.zeros(3)
