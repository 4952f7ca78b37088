"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
fixtures and the CPU oracle on the same seeded scenes.

Bars (BASELINE.json north star): candidate sets bit-exact; per-step vertex
positions within 1e-6 * ell (ell = max(bbox diagonal, 0.05), solver.py:644);
identical step status / failure reason and Newton iteration counts.
"""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TRAJ_TOL = 1e-6   # x error / ell


def _scene(d):
    from paper_2503_05020_b200 import scene as sc
    if str(d["kind"]) == "bimanual":
        return sc.bimanual_scene()
    return sc.build_trial_scene(sc.ObjectSpec(kind=str(d["kind"]), soft=bool(d["soft_object"])),
                                sc.GripperSpec(soft_fingers=bool(d["soft_fingers"])),
                                d["cand_R"], d["cand_T"], float(d["cand_opening"]))


def _rollout(env, scene, n_steps, gravity_after=None, halt=50.0):
    """Closing rollout with per-finger force halt, on the device."""
    halted = {f: False for f in scene.finger_links}
    for f, ids in scene.finger_links.items():
        for b in ids:
            env.bodies[b].velocity = scene.closing_dirs[f] * 0.05
    xs, reps, forces = [], [], []
    for k in range(n_steps):
        if gravity_after is not None and k == gravity_after:
            env.gravity = np.array([0.0, 0.0, -9.8])
        rep = env.step()
        fb, _, _ = env.contact_forces()
        fr = {f: float(sum(fb[b] for b in ids)) for f, ids in scene.finger_links.items()}
        xs.append(env.x.copy())
        reps.append(rep)
        forces.append(fr)
        for f in scene.finger_links:
            if not halted[f] and fr[f] > halt:
                halted[f] = True
                for b in scene.finger_links[f]:
                    env.bodies[b].velocity = np.zeros(3)
        if rep.status == "failed":
            break
    return xs, reps, forces


@pytest.mark.parametrize("name,grav,solver", [("cfg1", None, None), ("cylfail", None, None), ("cyl", None, None),
                                               ("sphere", None, None), ("soft", 18, None), ("softsphere", 18, None),
                                               ("bimanual", None, None),
                                               ("cfg1", None, "pcg"), ("soft", 18, "pcg")])
def test_trajectory_matches_reference(golden, name, grav, solver, monkeypatch):
    """Every recorded step of the reference's trajectory (full fixture length: cfg1 50, cylinder /
    sphere 20, soft box / soft sphere object 25, bimanual 12).  solver="pcg": the block-Jacobi PCG alternative
    (GRIP_SOLVER=pcg, the north star's solver) instead of the default skyline Cholesky."""
    from paper_2503_05020_b200.solver import Environment
    if solver:
        monkeypatch.setenv("GRIP_SOLVER", solver)
    d = np.load(golden / f"traj_{name}.npz")
    scene = _scene(d)
    env = Environment(scene.bodies, collide_pairs_off=scene.collide_pairs_off)
    golden_reps = json.loads(str(d["reports_json"]))
    golden_forces = json.loads(str(d["forces_json"]))
    n = len(golden_reps)
    stress = []
    if "stress" in d.files:   # the recorder's stress field, every step (materials.py:191-205)
        orig_step = env.step

        def step_and_stress():
            rep = orig_step()
            stress.append(env.stress_rows().copy())
            return rep
        env.step = step_and_stress
    xs, reps, forces = _rollout(env, scene, n, gravity_after=grav)
    ell = max(float(np.linalg.norm(d["sv"][0].max(0) - d["sv"][0].min(0))), 0.05)
    worst = 0.0
    for k in range(n):
        g = golden_reps[k]
        r = reps[k]
        assert (r.status, r.reason) == (g["status"], g["reason"]), (k, r.status, r.reason, g["status"], g["reason"])
        assert r.iterations == g["iterations"], (k, r.iterations, g["iterations"])
        err = float(np.abs(xs[k] - d["x"][k]).max()) / ell
        worst = max(worst, err)
        assert err <= TRAJ_TOL, (k, err)
        if stress:
            # stress is a derived field: positions within 1e-6 ell allow strain errors ~1e-5 on the
            # pads' ~1 cm tets, i.e. stress errors ~1e-5 of the field's scale (1e-4 bound here)
            ref = d["stress"][k]
            np.testing.assert_allclose(stress[k], ref, rtol=0, atol=1e-4 * np.abs(ref).max())
        for f, v in golden_forces[k].items():
            assert abs(forces[k][f] - v) <= 1e-6 * max(1.0, abs(v)), (k, f, forces[k][f], v)
        if r.status == "failed":
            break
    assert len(reps) == n or reps[-1].status == "failed"
    print(f"{name}: {n} steps, worst |dx|/ell = {worst:.3e}")


@pytest.mark.parametrize("name,bp", [("cfg1", None), ("sphere", None), ("soft", None), ("softsphere", None),
                                     ("bimanual", None), ("cyl", None),
                                     ("cfg1", "grid"), ("sphere", "grid"), ("soft", "grid"), ("bimanual", "grid"),
                                     ("cyl", "grid")])
def test_candidate_sets_bit_exact(golden, name, bp, monkeypatch):
    """Broad phase on the reference's own recorded states equals its candidate sets: the default
    direct broad phase and the grid broad phase (GRIP_BP=grid, the automatic fallback for large
    culled sets)."""
    from paper_2503_05020_b200.solver import Environment
    if bp:
        monkeypatch.setenv("GRIP_BP", bp)
    d = np.load(golden / f"traj_{name}.npz")
    scene = _scene(d)
    env = Environment(scene.bodies, collide_pairs_off=scene.collide_pairs_off)
    off_pt = np.concatenate([[0], np.cumsum(d["pt_counts"])])
    off_ee = np.concatenate([[0], np.cumsum(d["ee_counts"])])
    grp = env._owner()
    for k in range(len(d["pt_counts"])):
        # set nodes and the kinematic surfaces of that step
        sv = d["sv"][k]
        kin = np.zeros_like(sv)
        for r in env.layout.records:
            if r.kind == "kinematic":
                kin[r.surf0:r.surf0 + r.n_sv] = sv[r.surf0:r.surf0 + r.n_sv]
        grp.dev.set_state(d["x"][k].reshape(-1, 3), None, kin)
        grp.invalidate()
        pt, ee = env.candidates(1.05e-3)
        assert np.array_equal(pt, d["pt_rows"][off_pt[k]:off_pt[k + 1]]), (k, len(pt), d["pt_counts"][k])
        assert np.array_equal(ee, d["ee_rows"][off_ee[k]:off_ee[k + 1]]), (k, len(ee), d["ee_counts"][k])


def test_batch_bitwise_equals_single(golden):
    """SPEC invariant: batch-of-N bitwise equals batch-of-1 (multienv isolation)."""
    from paper_2503_05020_b200 import scene as sc
    from paper_2503_05020_b200.multienv import Batch
    from paper_2503_05020_b200.solver import Environment
    c = sc.load_cfg2_candidates()
    scenes = [sc.cfg2_scene(i, c) for i in range(6)]
    envs = [Environment(s.bodies, collide_pairs_off=s.collide_pairs_off) for s in scenes]
    solo_scene = sc.cfg2_scene(4, c)
    solo = Environment(solo_scene.bodies, collide_pairs_off=solo_scene.collide_pairs_off)
    for s, e in list(zip(scenes, envs)) + [(solo_scene, solo)]:
        for f, ids in s.finger_links.items():
            for b in ids:
                e.bodies[b].velocity = s.closing_dirs[f] * 0.05
    batch = Batch(envs)
    for _ in range(6):
        batch.step()
        solo.step()
        assert np.array_equal(envs[4].x, solo.x)


def test_stress_matches_oracle(golden):
    from oracle import energies as oen
    from paper_2503_05020_b200.solver import Environment
    d = np.load(golden / "traj_bimanual.npz")
    scene = _scene(d)
    env = Environment(scene.bodies, collide_pairs_off=scene.collide_pairs_off)
    grp = env._owner()
    grp.dev.set_state(d["x"][5].reshape(-1, 3), None, None)
    grp.invalidate()
    rows = env.stress_rows()
    np.testing.assert_allclose(rows, d["stress"][5], rtol=1e-9, atol=1e-6 * np.abs(d["stress"][5]).max())
    assert oen is not None


@pytest.mark.parametrize("lockstep,small_caps", [(True, False), (False, False), (False, True), ("device", False),
                                                  ("device", True)])
def test_protocol_labels_match_reference(golden, lockstep, small_caps, monkeypatch):
    """Grasp labels (stable / unstable / sim-failed), step counts, halts and phase markers of the
    full protocol (protocol.py:152-277) on the reference's own seeds, all envs batched, in
    lockstep (Batch.step semantics) and with continuous batching (grip_round).  small_caps starts
    every candidate / contact / anchor / grid buffer tiny, so the rounds overflow and the
    per-stage growth-and-redo path runs many times; the labels must not change."""
    if small_caps:
        monkeypatch.setenv("GRIP_SMALL_CAPS", "1")
    from paper_2503_05020_b200 import scene as sc
    from paper_2503_05020_b200.multienv import DeviceEnvGroup
    from paper_2503_05020_b200.protocol import BatchedGraspTrials
    from paper_2503_05020_b200.solver import Environment
    ref = json.loads((golden / "verdicts.json").read_text())
    scenes = [sc.build_trial_scene(sc.ObjectSpec(kind=r["kind"], soft=r["soft_object"]), sc.GripperSpec(soft_fingers=True),
                                   np.array(r["R"]), np.array(r["T"]), r["opening"]) for r in ref]
    envs = [Environment(s.bodies, collide_pairs_off=s.collide_pairs_off) for s in scenes]
    grp = DeviceEnvGroup(envs)
    if lockstep == "device":   # the state machine as a kernel, 8 rounds per host call
        from paper_2503_05020_b200.protocol import DeviceProtocolTrials
        recs = DeviceProtocolTrials(grp, scenes).run(rounds_per_call=8)
    else:
        recs = BatchedGraspTrials(grp, scenes).run(lockstep=lockstep)
    for r, g in zip(recs, ref):
        assert r.verdict == g["verdict"], (g["seed"], r.verdict, g["verdict"])
        assert r.n_steps == g["n_steps"], (g["seed"], r.n_steps, g["n_steps"])
        assert r.phase_markers == g["phase_markers"], (g["seed"], r.phase_markers, g["phase_markers"])
        if g["failure"]:
            assert r.failure["reason"] == g["failure"]["reason"] and r.failure["phase"] == g["failure"]["phase"]
        for f, h in g["halt_forces"].items():
            assert r.halt_forces[f]["step"] == h["step"]
            # small_caps: a sweep redone after buffer growth restarts the eigensolves from warm
            # starts one Newton iteration newer (rounding-level H), which the barrier amplifies
            # near the 50 N halt (force ~ 1/d); labels, steps and markers stay exact
            assert abs(r.halt_forces[f]["force"] - h["force"]) <= (1e-3 if small_caps else 1e-5) * h["force"]
        for k, v in g["com_displacement"].items():
            assert abs(r.com_displacement[k] - v) <= 1e-6 * 0.1 + 1e-9, (g["seed"], k, r.com_displacement[k], v)


def test_device_element_kernels_vs_reference(golden):
    """The warp-per-element kernels against the reference's per-stencil / per-tet outputs."""
    from oracle import energies as oen
    from paper_2503_05020_b200._native import debug_elements
    K = dict(np.load(golden / "kernels.npz"))
    X, pt, ee, epsx = K["pot_x"], K["pot_pt"], K["pot_ee"], K["pot_epsx"]
    rows = {tuple(r): k for k, r in enumerate(K["pot_idx"])}
    inp = np.array([np.concatenate([X[r].ravel(), [3e6, 1e-3]]) for r in pt])
    E, g, H, fl = debug_elements(0, inp)
    inp = np.array([np.concatenate([X[r].ravel(), [epsx[n], 3e6, 1e-3]]) for n, r in enumerate(ee)])
    E2, g2, H2, fl2 = debug_elements(1, inp)
    Es, gs, n_act = 0.0, np.zeros_like(X), 0
    for rr, EE, gg, HH, ff in ((pt, E, g, H, fl), (ee, E2, g2, H2, fl2)):
        for n, r in enumerate(rr):
            if ff[n] & 1:
                n_act += 1
                Es += EE[n]
                np.add.at(gs, r, gg[n].reshape(4, 3))
                Hr = K["pot_H"][rows[tuple(r)]]
                assert np.abs(HH[n] - Hr).max() <= 1e-9 * np.abs(Hr).max(), n
    assert n_act == len(K["pot_idx"])
    np.testing.assert_allclose(Es, K["pot_E"], rtol=1e-12)
    np.testing.assert_allclose(gs, K["pot_g"], rtol=1e-9, atol=1e-11 * np.abs(K["pot_g"]).max())
    # Neo-Hookean
    rest, cur = K["nh_rest"], K["nh_cur"]
    Dmi, V0, _ = oen.tet_rest(rest.reshape(-1, 3), np.arange(4 * len(rest)).reshape(-1, 4))
    inp = np.array([np.concatenate([cur[n].ravel(), Dmi[n].ravel(), [V0[n], K["nh_mu"], K["nh_lam"]]])
                    for n in range(len(rest))])
    E, g, H, fl = debug_elements(2, inp)
    assert not np.any(fl & 4)
    np.testing.assert_allclose(E, K["nh_Ee"], rtol=1e-11, atol=1e-18)
    for n in range(len(rest)):
        assert np.abs(H[n] - K["nh_H"][n]).max() <= 1e-9 * np.abs(K["nh_H"][n]).max(), n
    np.testing.assert_allclose(g.reshape(-1, 3), K["nh_g"], rtol=1e-9, atol=1e-10 * np.abs(K["nh_g"]).max())
    # ABD
    inp = np.array([np.concatenate([A.ravel(), [1e8 * 1.25e-4]]) for A in K["abd_A"]])
    E, g, H, _ = debug_elements(3, inp)
    np.testing.assert_allclose(E, K["abd_E"], rtol=1e-12)
    for n in range(len(inp)):
        assert np.abs(H[n] - K["abd_H"][n]).max() <= 1e-9 * np.abs(K["abd_H"][n]).max()


@pytest.mark.parametrize("mode", ["device", "host"])
def test_protocol_labels_match_reference_cfg2(golden, mode):
    """Full-protocol labels of bench (config 2) envs with cylinder and sphere objects, the
    reference's own trials on the bench's candidates (verdicts_cfg2.json), batched together,
    with the device-resident protocol (the bench default) and the host state machine."""
    from paper_2503_05020_b200 import scene as sc
    from paper_2503_05020_b200.multienv import DeviceEnvGroup
    from paper_2503_05020_b200.protocol import BatchedGraspTrials, DeviceProtocolTrials
    from paper_2503_05020_b200.solver import Environment
    path = golden / "verdicts_cfg2.json"
    if not path.exists():
        pytest.skip("verdicts_cfg2.json not generated")
    ref = json.loads(path.read_text())
    cands = sc.load_cfg2_candidates()
    scenes = [sc.cfg2_scene(r["seed"], cands) for r in ref]
    for s, r in zip(scenes, ref):
        np.testing.assert_allclose(cands["R"][r["seed"]], r["R"])
    envs = [Environment(s.bodies, collide_pairs_off=s.collide_pairs_off) for s in scenes]
    grp = DeviceEnvGroup(envs)
    recs = DeviceProtocolTrials(grp, scenes).run(rounds_per_call=4) if mode == "device" else \
        BatchedGraspTrials(grp, scenes).run()
    for r, g in zip(recs, ref):
        key = (g["kind"], g["seed"])
        assert r.verdict == g["verdict"], (key, r.verdict, g["verdict"])
        assert r.n_steps == g["n_steps"], (key, r.n_steps, g["n_steps"])
        assert r.phase_markers == g["phase_markers"], (key, r.phase_markers, g["phase_markers"])
        if g["failure"]:
            assert r.failure["reason"] == g["failure"]["reason"] and r.failure["phase"] == g["failure"]["phase"]
        for f, h in g["halt_forces"].items():
            assert r.halt_forces[f]["step"] == h["step"], key
            assert abs(r.halt_forces[f]["force"] - h["force"]) <= 1e-5 * h["force"], key
        for k, v in g["com_displacement"].items():
            assert abs(r.com_displacement[k] - v) <= 1e-6 * 0.1 + 1e-9, (key, k, r.com_displacement[k], v)


def test_device_friction_vs_reference(golden):
    """The production friction element (w_friction, the code k_elements_w runs) against the
    reference's friction_potential (contact.py:475-524) on tests/golden/friction.npz."""
    from paper_2503_05020_b200._native import debug_elements
    F = np.load(golden / "friction.npz")
    n = len(F["fr_E"])
    inp = np.array([np.concatenate([F["fr_x"][k].ravel(), F["fr_xp"][k].ravel(), F["fr_gamma"][k], F["fr_T"][k].ravel(),
                                    [F["fr_lam"][k], F["fr_mu"][k], float(F["eps_v"]), float(F["dt"])]])
                    for k in range(n)])
    E, g, H, _ = debug_elements(4, inp)
    np.testing.assert_allclose(E, F["fr_E"], rtol=1e-11, atol=1e-20)
    for k in range(n):
        gr, Hr = F["fr_g"][k].ravel(), F["fr_H"][k]
        np.testing.assert_allclose(g[k], gr, rtol=1e-9, atol=1e-11 * max(np.abs(gr).max(), 1e-300))
        np.testing.assert_allclose(H[k], Hr, rtol=1e-9, atol=1e-11 * max(np.abs(Hr).max(), 1e-300))


def test_production_element_chain_vs_reference(golden):
    """The element chain a Newton sweep actually runs (grip_debug_chain): PT / EE stencils through
    the k_elements_w code with deferred clamps -> k_tet_jacobi2 -> k_tet_finish; NH tets through
    k_tet_front (Gershgorin pass-through or deferral) -> k_tet_jacobi2 -> k_tet_back, cold (identity
    warm starts) and warm (the bases the cold pass left, as in the next Newton iteration) -- all
    against the reference's SPD-projected blocks (materials.py:101-113, contact.py:271-344)."""
    from oracle import energies as oen
    from paper_2503_05020_b200._native import debug_chain
    K = dict(np.load(golden / "kernels.npz"))
    X, pt, ee, epsx = K["pot_x"], K["pot_pt"], K["pot_ee"], K["pot_epsx"]
    rows = {tuple(r): k for k, r in enumerate(K["pot_idx"])}
    n_act = 0
    for etype, rr, inp in ((0, pt, np.array([np.concatenate([X[r].ravel(), [3e6, 1e-3]]) for r in pt])),
                           (1, ee, np.array([np.concatenate([X[r].ravel(), [epsx[n], 3e6, 1e-3]])
                                             for n, r in enumerate(ee)]))):
        E, g, H, fl = debug_chain(etype, inp)
        for n, r in enumerate(rr):
            if fl[n] & 1:
                n_act += 1
                Hr = K["pot_H"][rows[tuple(r)]]
                assert np.abs(H[n] - Hr).max() <= 1e-9 * np.abs(Hr).max(), (etype, n)
    assert n_act == len(K["pot_idx"])
    rest, cur = K["nh_rest"], K["nh_cur"]
    Dmi, V0, _ = oen.tet_rest(rest.reshape(-1, 3), np.arange(4 * len(rest)).reshape(-1, 4))
    inp = np.array([np.concatenate([cur[n].ravel(), Dmi[n].ravel(), [V0[n], K["nh_mu"], K["nh_lam"]]])
                    for n in range(len(rest))])
    eig = np.zeros((len(rest), 9, 9))
    eig[:] = np.eye(9)
    for rnd in ("cold", "warm"):
        E, g, H, fl = debug_chain(2, inp, eig)
        assert not np.any(fl & 4), rnd
        np.testing.assert_allclose(E, K["nh_Ee"], rtol=1e-11, atol=1e-18)
        np.testing.assert_allclose(g.reshape(-1, 3), K["nh_g"], rtol=1e-9, atol=1e-10 * np.abs(K["nh_g"]).max())
        for n in range(len(rest)):
            assert np.abs(H[n] - K["nh_H"][n]).max() <= 1e-9 * np.abs(K["nh_H"][n]).max(), (rnd, n)
        # the warm starts are orthonormal eigenbases
        np.testing.assert_allclose(np.einsum("nij,nkj->nik", eig, eig), np.broadcast_to(np.eye(9), eig.shape),
                                   atol=1e-12)
