"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Run here (the build container), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 OMP_NUM_THREADS=1 \
        python tests/golden/make_golden.py [--only NAME ...]

Everything below calls the reference's own public functions (gripsim 0.1.0,
/root/reference/pkg/src/gripsim) on seeded synthetic inputs and records what
they return.  The fixtures pin two things:

* the oracle restatement in ``oracle/`` (CPU tests compare it with these), and
* the CUDA path (GPU tests compare it with the oracle and with these).

Outputs are small ``.npz`` / ``.json`` files; the 400 bench grasp candidates go
to ``paper_2503_05020_b200/data/cfg2_candidates.npz`` because bench.py needs
them on the GPU box.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent

from gripsim import contact as ct  # noqa: E402  (reference, read-only)
from gripsim import materials as mat  # noqa: E402
from gripsim import solver as sv  # noqa: E402
from gripsim import synth as sy  # noqa: E402
from gripsim.geometry import broadphase as bp  # noqa: E402
from gripsim.geometry import ccd  # noqa: E402
from gripsim.geometry import distances as dist  # noqa: E402
from gripsim.geometry import mesh as gm  # noqa: E402
from gripsim.geometry.sdf import build_sdf  # noqa: E402
from gripsim.pipeline import config as cfg  # noqa: E402
from gripsim.pipeline import protocol as proto  # noqa: E402

KINDS = ("box", "cylinder", "sphere")
CYL_RADIUS = 0.02
CYL_HEIGHT = 0.05
CYL_SEGMENTS = 20


# ---------------------------------------------------------------------------
# scenes
# ---------------------------------------------------------------------------


def cylinder_surface():
    prof = [(0.0, 0.0), (CYL_RADIUS, 0.0), (CYL_RADIUS, CYL_HEIGHT), (0.0, CYL_HEIGHT)]
    return gm.revolved_surface(prof, segments=CYL_SEGMENTS, center=(0.0, 0.0, -0.5 * CYL_HEIGHT))


_OBJ_DIR = Path(tempfile.gettempdir()) / "grip_golden_obj"


def scene_for(kind, soft_object=False, soft_fingers=True):
    sc = cfg.SceneConfig()
    sc.object.soft = soft_object
    sc.gripper.soft_fingers = soft_fingers
    if kind == "cylinder":
        _OBJ_DIR.mkdir(exist_ok=True)
        path = _OBJ_DIR / "cylinder.obj"
        if not path.exists():
            tmp = _OBJ_DIR / f"cylinder.{os.getpid()}.obj"
            gm.save_obj(cylinder_surface(), tmp)
            os.replace(tmp, path)
        sc.object.kind = "mesh"
        sc.object.mesh_path = str(path)
    else:
        sc.object.kind = kind
    return sc


_SDF_CACHE = {}


def candidate(kind, seed, soft_object=False):
    sc = scene_for(kind, soft_object=soft_object)
    surf = sc.object.surface()
    key = (kind, soft_object)
    if key not in _SDF_CACHE:
        _SDF_CACHE[key] = build_sdf(surf, resolution=sc.synth.sdf_resolution)
    cands = sy.sample_antipodal(
        surf, sc.gripper.gripper, 1, seed=seed, sdf=_SDF_CACHE[key], mu=sc.synth.mu,
        dhat=sc.contact.dhat, n_surface_points=sc.synth.surface_points,
        approach_attempts=sc.synth.approach_attempts,
    )
    return cands[0] if cands else None


def cand_arrays(c):
    return {"R": np.asarray(c.rotation), "T": np.asarray(c.translation), "opening": float(c.joints[0])}


# ---------------------------------------------------------------------------
# kernel-level vectors
# ---------------------------------------------------------------------------


def gen_kernels(out):
    rng = np.random.default_rng(20250305)
    res = {}

    # point-triangle closest: random + structured (vertex / edge / face regions)
    n = 3000
    tri = rng.normal(size=(n, 3, 3))
    p = rng.normal(size=(n, 3)) * 1.5
    # structured: points exactly at vertices, on edges, in the plane
    k = 300
    p[:k] = tri[:k, rng.integers(0, 3)]
    w = rng.random((k, 1))
    p[k:2 * k] = (1 - w) * tri[k:2 * k, 0] + w * tri[k:2 * k, 1]
    bw = rng.dirichlet(np.ones(3), size=k)
    p[2 * k:3 * k] = np.einsum("nk,nkj->nj", bw, tri[2 * k:3 * k])
    D, bary, region = dist.point_triangle_closest(p, tri[:, 0], tri[:, 1], tri[:, 2])
    res.update(ptc_p=p, ptc_tri=tri, ptc_D=D, ptc_bary=bary, ptc_region=region)

    # edge-edge closest: random + parallel + shared-plane cases
    a0, a1, b0, b1 = (rng.normal(size=(n, 3)) for _ in range(4))
    d = a1[:k] - a0[:k]
    b0[:k] = a0[:k] + rng.normal(size=(k, 3)) * 0.3
    b1[:k] = b0[:k] + d * rng.uniform(-2, 2, size=(k, 1))
    D, s, t = dist.edge_edge_closest(a0, a1, b0, b1)
    res.update(eec_x=np.stack([a0, a1, b0, b1], axis=1), eec_D=D, eec_s=s, eec_t=t)

    # barrier / mollifier scalars
    dh = 1e-3
    Dq = np.concatenate([np.linspace(1e-10, 1.2e-6, 500), rng.uniform(1e-9, 1e-6, 500)])
    b, f1, f2 = ct.barrier_sq(Dq, dh)
    y = np.linspace(0, 3e-5, 400)
    f0m, f1m = ct.friction_mollifier(y, 1e-3, 0.01)
    res.update(bar_D=Dq, bar_b=b, bar_f1=f1, bar_f2=f2, fm_y=y, fm_f0=f0m, fm_f1=f1m)

    # contact potential on near-contact stencils (all regions), project=True
    m = 300
    base = rng.normal(size=(m, 4, 3)) * 2e-3
    # PT: point hovering slightly above triangle plane
    pt_x = base.copy()
    nrm = np.cross(pt_x[:, 2] - pt_x[:, 1], pt_x[:, 3] - pt_x[:, 1])
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    bw = rng.dirichlet(np.ones(3), size=m) * 1.6 - 0.2
    foot = np.einsum("nk,nkj->nj", bw, pt_x[:, 1:])
    pt_x[:, 0] = foot + nrm * rng.uniform(1e-5, 9e-4, size=(m, 1))
    # EE: crossing edges separated slightly, some near-parallel
    ee_x = base.copy()
    mid = 0.5 * (ee_x[:, 0] + ee_x[:, 1])
    off = rng.normal(size=(m, 3))
    off /= np.linalg.norm(off, axis=1, keepdims=True)
    dirb = rng.normal(size=(m, 3))
    dirb[: m // 5] = (ee_x[: m // 5, 1] - ee_x[: m // 5, 0]) + rng.normal(size=(m // 5, 3)) * 1e-5
    dirb /= np.linalg.norm(dirb, axis=1, keepdims=True)
    shift = rng.uniform(-0.6, 0.6, size=(m, 1)) * 3e-3
    cen = mid + off * rng.uniform(1e-5, 9e-4, size=(m, 1))
    ee_x[:, 2] = cen - dirb * 2e-3 + shift * dirb
    ee_x[:, 3] = cen + dirb * 2e-3 + shift * dirb
    X = np.concatenate([pt_x.reshape(-1, 3), ee_x.reshape(-1, 3)])
    pt = np.arange(4 * m).reshape(m, 4)
    ee = 4 * m + np.arange(4 * m).reshape(m, 4)
    eps_x = rng.uniform(0.5, 2.0, size=m) * 1.6e-11
    cs = ct.ContactSet(pt, ee, eps_x)
    E, g, idx, H = cs.potential(X, ct.ContactParams(), order=2, project=True)
    E0, _, _, _ = cs.potential(X, ct.ContactParams(), order=0)
    # raw (unprojected) blocks too, to pin region dispatch separately from projection
    _, _, idx_r, H_r = cs.potential(X, ct.ContactParams(), order=2, project=False)
    res.update(pot_x=X, pot_pt=pt, pot_ee=ee, pot_epsx=eps_x, pot_E=E, pot_E0=E0, pot_g=g,
               pot_idx=idx, pot_H=H, pot_Hraw=H_r)

    # spd_project on random symmetric matrices (+ rank-deficient ones)
    A = rng.normal(size=(200, 12, 12))
    A = A + A.transpose(0, 2, 1)
    v = rng.normal(size=(100, 12, 1))
    A[:100] = v @ v.transpose(0, 2, 1) * rng.uniform(0.1, 10, size=(100, 1, 1))
    res.update(spd_in=A, spd_out=mat.spd_project(A))

    # Neo-Hookean on random tets (some compressed / sheared)
    nt = 300
    rest = rng.normal(size=(nt, 4, 3)) * 5e-3
    vol = gm.tet_volumes(rest.reshape(-1, 3), np.arange(4 * nt).reshape(nt, 4))
    bad = vol < 0
    rest[bad] = rest[bad][:, [0, 2, 1, 3]]
    Fd = np.eye(3) + rng.normal(size=(nt, 3, 3)) * 0.15
    Fd[: nt // 4] *= 0.6  # strong compression
    cur = np.einsum("nij,nkj->nki", Fd, rest) + rng.normal(size=(nt, 1, 3)) * 1e-2
    tets = np.arange(4 * nt).reshape(nt, 4)
    el = mat.TetElements(rest.reshape(-1, 3), tets)
    mu_l, lam_l = mat.lame_from_young_poisson(9.4e6, 0.3)
    vols_cur = gm.tet_volumes(cur.reshape(-1, 3), tets)
    keep = vols_cur > 0
    tets_k = np.arange(4 * int(keep.sum())).reshape(-1, 4)
    el = mat.TetElements(rest[keep].reshape(-1, 3), tets_k)
    e, g, H = mat.neo_hookean_energy(el, cur[keep].reshape(-1, 3), mu_l, lam_l, with_hessian=True, project=True)
    e_np, g_np, H_np = mat.neo_hookean_energy(el, cur[keep].reshape(-1, 3), mu_l, lam_l, with_hessian=True, project=False)
    # per-element energies/hessians: evaluate element by element for per-tet pins
    per_e = np.array([
        mat.neo_hookean_energy(mat.TetElements(rest[keep][i], np.arange(4)[None]),
                               cur[keep][i], mu_l, lam_l, with_hessian=False)[0]
        for i in range(int(keep.sum()))
    ])
    res.update(nh_rest=rest[keep], nh_cur=cur[keep], nh_mu=mu_l, nh_lam=lam_l, nh_E=e, nh_Ee=per_e,
               nh_g=g, nh_H=H, nh_Hraw=H_np)
    st = mat.compute_stress(el, cur[keep].reshape(-1, 3), mat.MaterialParams(9.4e6, 0.3, 1000.0, 3.5))
    res.update(stress_cauchy=st.cauchy, stress_vm=st.von_mises)

    # ABD orthogonality (+ projection as the solver does it)
    na = 50
    As = np.eye(3)[None] + rng.normal(size=(na, 3, 3)) * 0.05
    ab_E, ab_g, ab_H = [], [], []
    for Ai in As:
        st_ = mat.AffineBodyState(np.zeros(3), Ai, kappa=1e8)
        e_, g_, H_ = mat.abd_orthogonality_energy(st_, 1.25e-4, with_hessian=True)
        ab_E.append(e_); ab_g.append(g_); ab_H.append(mat.spd_project(H_[None])[0])
    res.update(abd_A=As, abd_E=np.array(ab_E), abd_g=np.array(ab_g), abd_H=np.array(ab_H))

    # CCD: random PT/EE stencils with displacements, incl. min_separation 0.1
    nc = 300
    cx = rng.normal(size=(nc, 4, 3)) * 1e-2
    cp = rng.normal(size=(nc, 4, 3)) * 1e-2
    Xc = cx.reshape(-1, 3)
    Pc = cp.reshape(-1, 3)
    ccd_out = []
    for i in range(nc):
        rows = np.arange(4 * i, 4 * i + 4)[None]
        a_pt = ccd.ccd_max_step(Xc, Pc, rows, np.zeros((0, 4), np.int64))
        a_ee = ccd.ccd_max_step(Xc, Pc, np.zeros((0, 4), np.int64), rows)
        a_pt2 = ccd.ccd_max_step(Xc, Pc, rows, np.zeros((0, 4), np.int64), min_separation=0.1)
        ccd_out.append((a_pt, a_ee, a_pt2))
    res.update(ccd_x=cx, ccd_p=cp, ccd_alpha=np.array(ccd_out))
    # SPEC example: point at height 1 above large triangle, displacement (0,0,-2)
    xs = np.array([[0.2, 0.2, 1.0], [-5, -5, 0], [5, -5, 0], [0, 5, 0]], float)
    ps = np.array([[0, 0, -2.0], [0, 0, 0], [0, 0, 0], [0, 0, 0]])
    res["ccd_spec"] = ccd.ccd_max_step(xs, ps, np.array([[0, 1, 2, 3]]), np.zeros((0, 4), np.int64))

    # tet inversion filter / pencil
    nf = 300
    M0 = np.eye(3)[None] * 1e-2 + rng.normal(size=(nf, 3, 3)) * 2e-3
    det0 = np.linalg.det(M0)
    M0[det0 < 0] = M0[det0 < 0][:, :, [1, 0, 2]]
    dM = rng.normal(size=(nf, 3, 3)) * 1e-2
    pen = np.array([ccd.pencil_det_positive_step(M0[i:i + 1], dM[i:i + 1]) for i in range(nf)])
    c0, c1, c2, c3 = rng.normal(size=(4, 400))
    roots = ccd.smallest_positive_cubic_root(c0, c1, c2, c3)
    res.update(pen_M0=M0, pen_dM=dM, pen_alpha=pen, cub_c=np.stack([c0, c1, c2, c3], 1), cub_root=roots)
    np.savez_compressed(out / "kernels.npz", **res)


# ---------------------------------------------------------------------------
# meshes
# ---------------------------------------------------------------------------


def gen_friction(out):
    """Lagged-friction golden vectors (contact.py:475-524 friction_potential, 403-410 tangent basis):
    single anchors with random stencils, weights and normals, slips below, at and above the
    mollifier width h = eps_v dt (the three branches of f0 / f1 / f1')."""
    rng = np.random.default_rng(7)
    eps_v, dt = 1e-3, 0.01
    h = eps_v * dt
    params = ct.ContactParams()
    n = 64
    rows = {k: [] for k in ("x", "xp", "gamma", "T", "lam", "mu", "E", "g", "H")}
    for k in range(n):
        x = rng.normal(scale=0.01, size=(4, 3))
        slip_scale = h * (0.0 if k % 8 == 0 else 10.0 ** rng.uniform(-3, 1.5))
        xp = x - rng.normal(size=(4, 3)) * slip_scale
        a = rng.uniform()
        gam = np.array([1.0, -a, -(1 - a) * 0.5, -(1 - a) * 0.5]) if k % 2 else \
            np.array([1 - a, a, -(1 - rng.uniform()), 0.0])
        if k % 2 == 0:
            gam[3] = -1.0 - gam[2]
        nrm = rng.normal(size=(1, 3))
        nrm /= np.linalg.norm(nrm)
        T = ct._tangent_basis(nrm)[0]
        lam, mu = float(10.0 ** rng.uniform(-2, 2)), float(rng.uniform(0.1, 2.0))
        anc = ct.FrictionAnchors(verts=np.arange(4)[None], gamma=gam[None], tangent=T[None], lam=np.array([lam]),
                                 mu=np.array([mu]), bodies=np.zeros((1, 2), np.int64))
        params.eps_v = eps_v
        E, g, _, H = ct.friction_potential(anc, x, xp, params, dt)
        for key, v in (("x", x), ("xp", xp), ("gamma", gam), ("T", T), ("lam", lam), ("mu", mu), ("E", E),
                       ("g", g), ("H", H[0])):
            rows[key].append(v)
    np.savez_compressed(out / "friction.npz", eps_v=eps_v, dt=dt, **{f"fr_{k}": np.array(v) for k, v in rows.items()})
    print("friction", n)


def gen_meshes(out):
    res = {}
    b = gm.box_surface(0.05, subdivisions=3)
    res.update(box_v=b.vertices, box_t=b.triangles, box_e=b.edges())
    s = gm.icosphere(0.025, level=3)
    res.update(sph_v=s.vertices, sph_t=s.triangles)
    c = cylinder_surface()
    res.update(cyl_v=c.vertices, cyl_t=c.triangles)
    L = gm.box_tet_lattice((0.01, 0.02, 0.05), (2, 2, 4), center=(0.03, 0.0, 0.025))
    surf, vmap = L.boundary_surface()
    res.update(lat_v=L.vertices, lat_T=L.tets, lat_sv=vmap, lat_st=surf.triangles, lat_se=surf.edges())
    L3 = gm.box_tet_lattice(0.05, 3)
    s3, m3 = L3.boundary_surface()
    res.update(cube3_v=L3.vertices, cube3_T=L3.tets, cube3_sv=m3, cube3_st=s3.triangles)
    SL = gm.sphere_tet_lattice(0.025, 6)
    ss, sm = SL.boundary_surface()
    res.update(sphl_v=SL.vertices, sphl_T=SL.tets, sphl_sv=sm, sphl_st=ss.triangles)
    mass, com, sec = gm.surface_mass_properties(b, 500.0)
    res.update(box_mass=mass, box_com=com, box_second=sec, box_vol=b.enclosed_volume())
    for name, srf in (("sph", s), ("cyl", c)):
        mass, com, sec = gm.surface_mass_properties(srf, 500.0)
        res.update(**{f"{name}_mass": mass, f"{name}_com": com, f"{name}_second": sec,
                      f"{name}_vol": srf.enclosed_volume()})
    res["lat_mass"] = mat.lumped_vertex_masses(L, 1000.0)
    np.savez_compressed(out / "meshes.npz", **res)


# ---------------------------------------------------------------------------
# trajectories
# ---------------------------------------------------------------------------


def _cands_now(env):
    cs = env.contact_set_now()
    return cs.pt.copy(), cs.ee.copy()


def rollout(env, finger_links, n_steps, close_speed=0.05, halt=50.0, gravity_after=None,
            gravity=(0.0, 0.0, -9.8), record_stress=False, record_bp=False):
    """Closing rollout: fingers close, each halts once its force > halt."""
    halted = {f: False for f in finger_links}
    for f, ids in finger_links.items():
        d = env.records[ids[0]].get("closing_dir")
        for bid in ids:
            env.records[bid]["body"].velocity = d * close_speed
    rec = {"x": [], "v": [], "kin": [], "sv": [], "reports": [], "forces": [], "stress": [],
           "pt": [], "ee": [], "events": []}
    soft_recs = [r for r in env.records if r["kind"] == "soft"]
    for step in range(n_steps):
        if gravity_after is not None and step == gravity_after:
            env.gravity = np.asarray(gravity, float)
        rep = env.step()
        events = proto.contact_events_now(env)
        forces = {f: proto.finger_contact_force(env, ids, events) for f, ids in finger_links.items()}
        rec["x"].append(env.x.copy())
        rec["v"].append(env.v.copy())
        rec["sv"].append(env.surface_positions().copy())
        rec["reports"].append(rep.to_dict())
        rec["forces"].append(forces)
        rec["events"].append(len(events))
        if record_bp:
            pt, ee = _cands_now(env)
            rec["pt"].append(pt)
            rec["ee"].append(ee)
        if record_stress:
            rows = []
            for r in soft_recs:
                xs = env.x[r["dof0"]: r["dof0"] + r["ndof"]].reshape(-1, 3)
                sf = mat.compute_stress(r["elements"], xs, r["body"].material)
                c = sf.cauchy
                rows.append(np.stack([c[:, 0, 0], c[:, 1, 1], c[:, 2, 2], c[:, 0, 1], c[:, 1, 2],
                                      c[:, 0, 2], sf.von_mises], 1))
            rec["stress"].append(np.concatenate(rows))
        for f in finger_links:
            if not halted[f] and forces[f] > halt:
                halted[f] = True
                for bid in finger_links[f]:
                    env.records[bid]["body"].velocity = np.zeros(3)
        if rep.status == "failed":
            break
    return rec


def pack_rollout(rec, extra):
    out = dict(extra)
    out["x"] = np.array(rec["x"])
    out["v"] = np.array(rec["v"])
    out["sv"] = np.array(rec["sv"])
    if rec["stress"]:
        out["stress"] = np.array(rec["stress"])
    if rec["pt"]:
        out["pt_counts"] = np.array([len(a) for a in rec["pt"]])
        out["ee_counts"] = np.array([len(a) for a in rec["ee"]])
        out["pt_rows"] = np.concatenate(rec["pt"]) if rec["pt"] else np.zeros((0, 4), np.int64)
        out["ee_rows"] = np.concatenate(rec["ee"]) if rec["ee"] else np.zeros((0, 4), np.int64)
    out["reports_json"] = np.array(json.dumps(rec["reports"]))
    out["forces_json"] = np.array(json.dumps(rec["forces"]))
    return out


def traj_cfg(kind, seed, n_steps, soft_object=False, soft_fingers=True, gravity_after=None):
    sc = scene_for(kind, soft_object=soft_object, soft_fingers=soft_fingers)
    c = candidate(kind, seed, soft_object=soft_object)
    env, ob, fl = cfg.build_trial_env(sc, c)
    rec = rollout(env, fl, n_steps, gravity_after=gravity_after, record_bp=True,
                  record_stress=soft_object)
    ca = cand_arrays(c)
    return pack_rollout(rec, {"cand_R": ca["R"], "cand_T": ca["T"], "cand_opening": ca["opening"],
                              "kind": kind, "seed": seed, "soft_object": soft_object,
                              "soft_fingers": soft_fingers})


# config-3 object: the soft sphere lattice (sphere_tet_lattice, mesh.py:400) under kinematic fingers
SOFT_SPHERE_JOBS = [("softsphere", dict(kind="sphere", seed=1, n_steps=25, soft_object=True, soft_fingers=False,
                                        gravity_after=18))]


def _traj_job(args):
    name, kw = args
    t0 = time.time()
    res = traj_cfg(**kw)
    np.savez_compressed(HERE / f"traj_{name}.npz", **res)
    return name, time.time() - t0


def bimanual_env():
    """Config 4: two top-down soft-pad parallel grippers on one soft cube."""
    sc = cfg.SceneConfig()
    sc.object.kind = "box"
    sc.object.soft = True
    obj = sc.object.build_body()
    g = sc.gripper.gripper
    opening = 0.05 + 2 * 2e-3
    bodies = [obj]
    fingers = {}
    pairs_off = []
    for gi, yoff in enumerate((-0.0125, 0.0125)):
        T = np.array([0.0, yoff, -0.01])
        pad_ids = []
        for side in (0, 1):
            body = cfg._soft_finger_body(sc.gripper, side, opening)
            body.mesh.vertices[:] = body.mesh.vertices + T
            body.mesh.rest_vertices[:] = body.mesh.vertices
            body.mesh.__post_init__()
            body.name = f"g{gi}finger{side}"
            bodies.append(body)
            pad_ids.append(len(bodies) - 1)
            fingers[f"g{gi}finger{side}"] = (len(bodies) - 1,)
        _, _, palm_surf = g.body_meshes(opening)
        palm_surf = gm.TriSurface(palm_surf.vertices + np.array([0.0, 0.0, sc.gripper.palm_gap]) + T,
                                  palm_surf.triangles)
        palm = sv.KinematicBody(palm_surf, mat.MaterialParams(1e9, 0.3, 2000.0, 0.3), name=f"g{gi}palm")
        bodies.append(palm)
        for pid in pad_ids:
            pairs_off.append((pid, len(bodies) - 1))
    env = sv.Environment(bodies, gravity=(0, 0, 0), contact_params=sc.contact, solver_params=sc.solver,
                         name="bimanual", collide_pairs_off=pairs_off)
    for name, (bid,) in fingers.items():
        side = int(name[-1])
        env.records[bid]["closing_dir"] = np.array([1.0, 0, 0]) if side == 0 else np.array([-1.0, 0, 0])
    return env, fingers


def gen_bimanual(out):
    env, fingers = bimanual_env()
    rec = rollout(env, fingers, 12, record_stress=True, record_bp=True)
    np.savez_compressed(out / "traj_bimanual.npz", **pack_rollout(rec, {"kind": "bimanual"}))


def _verdict_job(args):
    kind, seed, soft_object = args
    sc = scene_for(kind, soft_object=soft_object)
    c = candidate(kind, seed, soft_object=soft_object)
    if c is None:
        return None
    env, ob, fl = cfg.build_trial_env(sc, c)
    t0 = time.time()
    r = proto.run_grasp_trial(env, sc.protocol, ob, fl)
    iters = [rep["iterations"] for rep in r.step_reports]
    return {"kind": kind, "seed": seed, "soft_object": soft_object, "verdict": r.verdict,
            "failure": r.failure, "n_steps": r.n_steps, "phase_markers": r.phase_markers,
            "com_displacement": r.com_displacement,
            "halt_forces": {k: {"force": float(v["force"]), "step": int(v["step"])} for k, v in r.halt_forces.items()},
            "metrics": {k: (float(v) if not isinstance(v, bool) else v) for k, v in r.metrics.items()},
            "iterations": iters, "wall_s": time.time() - t0,
            "R": np.asarray(c.rotation).tolist(), "T": np.asarray(c.translation).tolist(),
            "opening": float(c.joints[0]),
            "positions": r.positions.tolist() if (seed == 0 and kind == "box" and not soft_object) else None}


def gen_dataset(out):
    """One config-1 trial (box, seed 0) under a shortened protocol, emitted by the reference's own
    dataset writer (pipeline/dataset.py:121-167): the byte-level and value-level fixture of §8f-3."""
    import shutil
    from gripsim.pipeline import dataset as ds
    sc = scene_for("box")
    c = candidate("box", 0)
    env, ob, fl = cfg.build_trial_env(sc, c)
    prot = proto.TrialProtocol(settle_duration=0.02, steady_max_duration=0.05, gravity_phase_duration=0.02)
    rec = proto.run_grasp_trial(env, prot, ob, fl)
    rec.candidate = {"R": np.asarray(c.rotation).tolist(), "T": np.asarray(c.translation).tolist(),
                     "opening": float(c.joints[0])}
    dest = out / "dataset_cfg1"
    if dest.exists():
        shutil.rmtree(dest)
    manifest = ds.emit_dataset([rec], dest, params={"protocol": "short", "seed": 0})
    (out / "dataset_cfg1_protocol.json").write_text(json.dumps(
        {"settle_duration": 0.02, "steady_max_duration": 0.05, "gravity_phase_duration": 0.02,
         "R": rec.candidate["R"], "T": rec.candidate["T"], "opening": rec.candidate["opening"]}))
    print("dataset", rec.verdict, rec.n_steps, manifest["trials"][0]["files"])
    gen_metrics(out, env, ob, rec)


def gen_metrics(out, env, ob, rec):
    """D1/D2 grasp-quality metrics (pipeline/metrics.py:99-164) of the dataset trial's final state,
    plus the SDF build (geometry/sdf.py:117-178) and the surface sampler they rest on."""
    from gripsim.geometry.mesh import TriSurface
    from gripsim.pipeline import metrics as qm
    res = {"x": env.x.tolist(), "object_body": ob, "gripper_bodies": list(rec.gripper_bodies)}
    for resolution in (32, 128):
        t0 = time.time()
        d1, d2, h = qm.trial_quality_metrics(env, ob, rec.gripper_bodies, resolution=resolution)
        res[f"res{resolution}"] = {"D1": d1, "D2": d2, "spacing": h, "wall_s": time.time() - t0}
    grips = qm.gripper_surfaces_from_env(env, rec.gripper_bodies)
    pts = qm._sample_surfaces(grips, 50_000, 0)
    # per-sample d_o (positive inside) at resolution 32: the interior (trilinear) and far-field
    # branches value by value -- D1 / D2 alone are 0.0 here (samples inside the posed grid's
    # world AABB but outside the rotated grid get -|0| = -0.0, metrics.py:58-75)
    sdf32 = qm.object_sdf_from_env(env, ob, resolution=32)
    res["d_o_res32"] = qm._object_signed_inside(sdf32, pts).tolist()
    res["samples_head"] = pts[:32].tolist()
    res["samples_sum"] = pts.sum(axis=0).tolist()
    r = env.records[ob]
    rest = TriSurface(r["xi"], r["body"].surface.triangles)
    sdf = build_sdf(rest, resolution=32)
    q = env.x[r["dof0"]:r["dof0"] + 12]
    res["polar_R"] = qm._polar_rotation(q[3:].reshape(3, 3)).tolist()
    np.savez_compressed(out / "sdf_box32.npz", values=sdf.values, origin=sdf.origin, spacing=sdf.spacing)
    soft = {}
    for name, mesh in (("cube", gm.box_tet_lattice((0.04, 0.04, 0.04), resolution=3)),):
        surf, _ = mesh.boundary_surface()
        s2 = build_sdf(surf, resolution=24)
        np.savez_compressed(out / f"sdf_soft_{name}24.npz", values=s2.values, origin=s2.origin, spacing=s2.spacing,
                            vertices=surf.vertices, triangles=surf.triangles)
    (out / "metrics.json").write_text(json.dumps(res))
    print("metrics", {k: v for k, v in res.items() if k.startswith("res")})


def _verdict_compact(r, wall):
    return {"verdict": r.verdict, "failure": r.failure, "n_steps": r.n_steps,
            "phase_markers": r.phase_markers, "com_displacement": r.com_displacement,
            "halt_forces": {k: {"force": float(v["force"]), "step": int(v["step"])} for k, v in r.halt_forces.items()},
            "iterations": [rep["iterations"] for rep in r.step_reports], "wall_s": wall}


def _verdict_job_cfg2(i):
    """Full-protocol reference trial of bench env i (config 2: kind i % 3, candidate seed i)."""
    kind = KINDS[i % 3]
    sc = scene_for(kind)
    c = candidate(kind, i)
    if c is None:
        return None
    env, ob, fl = cfg.build_trial_env(sc, c)
    t0 = time.time()
    r = proto.run_grasp_trial(env, sc.protocol, ob, fl)
    return {"i": i, "kind": kind, **_verdict_compact(r, time.time() - t0)}


CFG3_KINDS = ("box", "sphere")
CFG3_SEED = 0   # validate_candidates seed: material rng = default_rng(seed + 7919 * i)


def cfg3_material(i):
    """Config 3's domain-randomized object material of trial i, by the reference's own
    randomized_material (config.py:311-318) with the pipeline's seeding (pipeline/__init__.py:29)."""
    sc = cfg.SceneConfig()
    sc.randomization.enabled = True
    rng = np.random.default_rng(CFG3_SEED + 7919 * i)
    return cfg.randomized_material(sc.object.material, sc.randomization, rng)


def _cfg3_cand_job(i):
    kind = CFG3_KINDS[i % 2]
    c = candidate(kind, i, soft_object=True)
    return i, kind, None if c is None else cand_arrays(c)


def gen_candidates_cfg3(pool, n=400):
    """Config 3: soft NH box / sphere (kind i % 2), kinematic fingers, antipodal
    candidate seed i on the soft object's surface, randomized material per trial."""
    rows = pool.map(_cfg3_cand_job, range(n), chunksize=4)
    R = np.zeros((n, 3, 3)); T = np.zeros((n, 3)); op = np.zeros(n); kind = np.zeros(n, np.int64)
    ok = np.zeros(n, bool); E = np.zeros(n); mu = np.zeros(n); nu = np.zeros(n); rho = np.zeros(n)
    for i, k, ca in rows:
        kind[i] = CFG3_KINDS.index(k)
        m = cfg3_material(i)
        E[i], mu[i], nu[i], rho[i] = m.young_modulus, m.friction_coefficient, m.poisson_ratio, m.density
        if ca is not None:
            R[i], T[i], op[i], ok[i] = ca["R"], ca["T"], ca["opening"], True
    dest = REPO / "paper_2503_05020_b200" / "data"
    np.savez_compressed(dest / "cfg3_candidates.npz", R=R, T=T, opening=op, kind=kind, ok=ok,
                        kinds=np.array(CFG3_KINDS), E=E, mu=mu, nu=nu, rho=rho)
    print("cfg3 candidates ok:", int(ok.sum()), "of", n)


def _verdict_job_cfg3(i):
    kind = CFG3_KINDS[i % 2]
    sc = scene_for(kind, soft_object=True, soft_fingers=False)
    c = candidate(kind, i, soft_object=True)
    if c is None:
        return None
    env, ob, fl = cfg.build_trial_env(sc, c, env_id=i, material_override=cfg3_material(i))
    t0 = time.time()
    r = proto.run_grasp_trial(env, sc.protocol, ob, fl)
    return {"i": i, "kind": kind, **_verdict_compact(r, time.time() - t0)}


def _cand_job(i):
    kind = KINDS[i % 3]
    c = candidate(kind, i)
    if c is None:
        return i, kind, None
    return i, kind, cand_arrays(c)


def gen_candidates(pool, n=400):
    """Bench candidates i = 0..n-1 (kind i % 3, antipodal sample of seed i).  400 for one GPU;
    GRIP_CFG2_CANDIDATES=3200 gives every rank of an 8-GPU run (and the config-5 sweep up to
    3200 envs) its own candidates -- the first 400 are the same either way (same seeds)."""
    rows = pool.map(_cand_job, range(n), chunksize=4)
    R = np.zeros((n, 3, 3)); T = np.zeros((n, 3)); op = np.zeros(n); kind = np.zeros(n, np.int64)
    ok = np.zeros(n, bool)
    for i, k, ca in rows:
        kind[i] = KINDS.index(k)
        if ca is not None:
            R[i], T[i], op[i], ok[i] = ca["R"], ca["T"], ca["opening"], True
    dest = REPO / "paper_2503_05020_b200" / "data"
    dest.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(dest / "cfg2_candidates.npz", R=R, T=T, opening=op, kind=kind, ok=ok,
                        kinds=np.array(KINDS), cyl=np.array([CYL_RADIUS, CYL_HEIGHT, CYL_SEGMENTS]))
    print("candidates ok:", int(ok.sum()), "of", n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    args = ap.parse_args()
    want = set(args.only or ["kernels", "friction", "meshes", "traj", "bimanual", "verdicts", "candidates", "dataset"])
    out = HERE
    ctx = mp.get_context("fork")
    scene_for("cylinder")  # write the cylinder OBJ once, before forking
    t0 = time.time()
    if "kernels" in want:
        gen_kernels(out); print("kernels", time.time() - t0)
    if "friction" in want:
        gen_friction(out)
    if "meshes" in want:
        gen_meshes(out); print("meshes", time.time() - t0)
    if "dataset" in want:
        gen_dataset(out); print("dataset", time.time() - t0)
    with ctx.Pool(os.cpu_count()) as pool:
        if "traj" in want:
            jobs = [
                ("cfg1", dict(kind="box", seed=0, n_steps=50)),
                ("cyl", dict(kind="cylinder", seed=3, n_steps=20)),
                ("cylfail", dict(kind="cylinder", seed=1, n_steps=3)),
                ("sphere", dict(kind="sphere", seed=2, n_steps=20)),
                ("soft", dict(kind="box", seed=0, n_steps=25, soft_object=True, soft_fingers=False,
                              gravity_after=18)),
            ]
            if os.environ.get("GRIP_TRAJ_ONLY"):
                jobs = [j for j in jobs + SOFT_SPHERE_JOBS if j[0] in os.environ["GRIP_TRAJ_ONLY"].split(",")]
            else:
                jobs += SOFT_SPHERE_JOBS
            for name, dt_ in pool.map(_traj_job, jobs):
                print("traj", name, round(dt_, 1))
        if "bimanual" in want:
            gen_bimanual(out); print("bimanual", time.time() - t0)
        if "verdicts" in want:
            jobs = [("box", s, False) for s in range(8)] + [("box", 0, True)]
            res = [r for r in pool.map(_verdict_job, jobs) if r is not None]
            (out / "verdicts.json").write_text(json.dumps(res))
            print("verdicts", [(r["seed"], r["verdict"], r["n_steps"]) for r in res], time.time() - t0)
        if "verdicts_cfg2" in want:
            # full-protocol labels of bench (config 2) envs: cylinder / sphere candidates i % 3 = 1, 2
            jobs = [(("box", "cylinder", "sphere")[i % 3], i, False) for i in (1, 2, 4, 5, 7, 8, 10, 11)]
            res = [r for r in pool.map(_verdict_job, jobs) if r is not None]
            (out / "verdicts_cfg2.json").write_text(json.dumps(res))
            print("verdicts_cfg2", [(r["kind"], r["seed"], r["verdict"], r["n_steps"]) for r in res], time.time() - t0)
        if "verdicts_cfg2_all" in want:
            # every one of the 400 bench envs (config 2), full protocol, unmodified reference
            res = [r for r in pool.imap(_verdict_job_cfg2, range(400), chunksize=1) if r is not None]
            (out / "verdicts_cfg2_all.json").write_text(json.dumps(res))
            print("verdicts_cfg2_all", len(res), {v: sum(r["verdict"] == v for r in res)
                                                  for v in ("stable", "unstable", "sim-failed")}, time.time() - t0)
        if "candidates_cfg3" in want:
            gen_candidates_cfg3(pool); print("candidates_cfg3", time.time() - t0)
        if "verdicts_cfg3" in want:
            n3 = int(os.environ.get("GRIP_CFG3_VERDICTS", "32"))
            res = [r for r in pool.imap(_verdict_job_cfg3, range(n3), chunksize=1) if r is not None]
            (out / "verdicts_cfg3.json").write_text(json.dumps(res))
            print("verdicts_cfg3", len(res), [(r["kind"], r["verdict"], r["n_steps"]) for r in res], time.time() - t0)
        if "candidates" in want:
            gen_candidates(pool, int(os.environ.get("GRIP_CFG2_CANDIDATES", "400"))); print("candidates", time.time() - t0)


if __name__ == "__main__":
    main()
