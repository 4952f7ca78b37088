"""Pin the CPU oracle (oracle/) against golden vectors from the unmodified reference.

The fixtures come from tests/golden/make_golden.py (reference run in the build
container).  These tests run on CPU (-m "not gpu").
"""

import json

import numpy as np
import pytest

from oracle import energies as en
from oracle import geometry as geo
from oracle import solver as osv
from paper_2503_05020_b200 import geometry as gm
from paper_2503_05020_b200 import scene as sc


@pytest.fixture(scope="module")
def K(golden):
    return dict(np.load(golden / "kernels.npz"))


def test_pt_closest(K):
    tri = K["ptc_tri"]
    D, bary, reg = geo.pt_closest(K["ptc_p"], tri[:, 0], tri[:, 1], tri[:, 2])
    assert np.array_equal(reg, K["ptc_region"])
    np.testing.assert_allclose(D, K["ptc_D"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(bary, K["ptc_bary"], rtol=1e-12, atol=1e-14)


def test_ee_closest(K):
    x = K["eec_x"]
    D, s, t = geo.ee_closest(x[:, 0], x[:, 1], x[:, 2], x[:, 3])
    np.testing.assert_allclose(D, K["eec_D"], rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(s, K["eec_s"])
    np.testing.assert_array_equal(t, K["eec_t"])


def test_barrier_and_mollifier(K):
    b, f1, f2 = en.barrier_D(K["bar_D"], 1e-3)
    for a, r in ((b, "bar_b"), (f1, "bar_f1"), (f2, "bar_f2")):
        np.testing.assert_allclose(a, K[r], rtol=1e-13, atol=0)
    f0, f1m = en.friction_f0_f1(K["fm_y"], 1e-3, 0.01)
    np.testing.assert_allclose(f0, K["fm_f0"], rtol=1e-13)
    np.testing.assert_allclose(f1m, K["fm_f1"], rtol=1e-13)
    # SPEC known answers
    assert abs(en.barrier_d(np.array([5e-4]), 1e-3)[0][0] - 1.7329e-7) < 1e-10
    f0, f1v = en.friction_f0_f1(np.array([0.0, 5e-6, 1e-5]), 1e-3, 0.01)
    np.testing.assert_allclose(f1v, [0.0, 0.75, 1.0])


def test_spd_clamp(K):
    np.testing.assert_allclose(en.spd_clamp(K["spd_in"]), K["spd_out"], rtol=1e-10, atol=1e-10)


def test_contact_potential(K):
    x, pt, ee, epsx = K["pot_x"], K["pot_pt"], K["pot_ee"], K["pot_epsx"]
    E, g, idx, H = en.contact_potential(x, pt, ee, epsx, 3e6, 1e-3, order=2, project=False)
    assert np.array_equal(idx, K["pot_idx"])
    np.testing.assert_allclose(E, K["pot_E"], rtol=1e-12)
    scale = np.abs(K["pot_g"]).max()
    np.testing.assert_allclose(g, K["pot_g"], rtol=1e-9, atol=1e-12 * scale)
    hs = np.abs(K["pot_Hraw"]).max(axis=(1, 2), keepdims=True)
    assert np.all(np.abs(H - K["pot_Hraw"]) <= 1e-9 * hs)
    _, _, _, Hp = en.contact_potential(x, pt, ee, epsx, 3e6, 1e-3, order=2, project=True)
    hs = np.abs(K["pot_H"]).max(axis=(1, 2), keepdims=True)
    assert np.all(np.abs(Hp - K["pot_H"]) <= 1e-9 * hs)
    E0 = en.contact_potential(x, pt, ee, epsx, 3e6, 1e-3, order=0)[0]
    np.testing.assert_allclose(E0, K["pot_E0"], rtol=1e-12)


def test_neo_hookean(K):
    rest, cur = K["nh_rest"], K["nh_cur"]
    n = len(rest)
    tets = np.arange(4 * n).reshape(n, 4)
    Dmi, V0, w = en.tet_rest(rest.reshape(-1, 3), tets)
    E, g, H, _ = en.neo_hookean(cur.reshape(-1, 3), tets, Dmi, V0, w, K["nh_mu"], K["nh_lam"], 2, project=False)
    np.testing.assert_allclose(E, K["nh_E"], rtol=1e-12)
    np.testing.assert_allclose(g, K["nh_g"], rtol=1e-9, atol=1e-9 * np.abs(K["nh_g"]).max())
    hs = np.abs(K["nh_Hraw"]).max(axis=(1, 2), keepdims=True)
    assert np.all(np.abs(H - K["nh_Hraw"]) <= 1e-10 * hs)
    _, _, Hp, _ = en.neo_hookean(cur.reshape(-1, 3), tets, Dmi, V0, w, K["nh_mu"], K["nh_lam"], 2, project=True)
    assert np.all(np.abs(Hp - K["nh_H"]) <= 1e-9 * hs)
    st = en.cauchy_stress(cur.reshape(-1, 3), tets, Dmi, *en.lame(9.4e6, 0.3))
    c = K["stress_cauchy"]
    ref = np.stack([c[:, 0, 0], c[:, 1, 1], c[:, 2, 2], c[:, 0, 1], c[:, 1, 2], c[:, 0, 2], K["stress_vm"]], 1)
    np.testing.assert_allclose(st, ref, rtol=1e-9, atol=1e-6)


def test_abd(K):
    for A, E, g, H in zip(K["abd_A"], K["abd_E"], K["abd_g"], K["abd_H"]):
        e, gg, HH = en.abd_ortho(A, 1e8 * 1.25e-4)
        np.testing.assert_allclose(e, E, rtol=1e-12)
        np.testing.assert_allclose(gg, g, rtol=1e-10, atol=1e-6)
        assert np.abs(HH - H).max() <= 1e-9 * np.abs(H).max()


def test_ccd_and_filters(K):
    cx, cp = K["ccd_x"], K["ccd_p"]
    X, P = cx.reshape(-1, 3), cp.reshape(-1, 3)
    out = []
    for i in range(len(cx)):
        rows = np.arange(4 * i, 4 * i + 4)[None]
        none = np.zeros((0, 4), np.int64)
        out.append((geo.ccd_max_step(X, P, rows, none), geo.ccd_max_step(X, P, none, rows),
                    geo.ccd_max_step(X, P, rows, none, min_separation=0.1)))
    np.testing.assert_allclose(np.array(out), K["ccd_alpha"], rtol=1e-12, atol=1e-15)
    xs = np.array([[0.2, 0.2, 1.0], [-5, -5, 0], [5, -5, 0], [0, 5, 0]], float)
    ps = np.array([[0, 0, -2.0], [0, 0, 0], [0, 0, 0], [0, 0, 0]])
    a = geo.ccd_max_step(xs, ps, np.array([[0, 1, 2, 3]]), np.zeros((0, 4), np.int64))
    assert a == K["ccd_spec"] and 0.45 < a <= 0.5
    pen = np.array([geo.pencil_step(K["pen_M0"][i:i + 1], K["pen_dM"][i:i + 1]) for i in range(len(K["pen_M0"]))])
    np.testing.assert_allclose(pen, K["pen_alpha"], rtol=1e-12)
    c = K["cub_c"]
    np.testing.assert_allclose(geo.cubic_smallest_root(c[:, 0], c[:, 1], c[:, 2], c[:, 3]), K["cub_root"], rtol=1e-12)


def test_meshes(golden):
    M = np.load(golden / "meshes.npz")
    b = gm.box_surface(0.05, subdivisions=3)
    assert np.array_equal(b.vertices, M["box_v"]) and np.array_equal(b.triangles, M["box_t"])
    assert np.array_equal(b.edges(), M["box_e"])
    s = gm.icosphere(0.025, level=3)
    assert np.array_equal(s.vertices, M["sph_v"]) and np.array_equal(s.triangles, M["sph_t"])
    c = gm.cylinder_surface()
    assert np.array_equal(c.vertices, M["cyl_v"]) and np.array_equal(c.triangles, M["cyl_t"])
    L = gm.box_tet_lattice((0.01, 0.02, 0.05), (2, 2, 4), center=(0.03, 0.0, 0.025))
    surf, vmap = L.boundary_surface()
    assert np.array_equal(L.vertices, M["lat_v"]) and np.array_equal(L.tets, M["lat_T"])
    assert np.array_equal(vmap, M["lat_sv"]) and np.array_equal(surf.triangles, M["lat_st"])
    assert np.array_equal(surf.edges(), M["lat_se"])
    SL = gm.sphere_tet_lattice(0.025, 6)
    ss, sm = SL.boundary_surface()
    assert np.array_equal(SL.vertices, M["sphl_v"]) and np.array_equal(SL.tets, M["sphl_T"])
    assert np.array_equal(ss.triangles, M["sphl_st"])
    mass, com, sec = gm.surface_mass_properties(b, 500.0)
    assert mass == M["box_mass"] and np.array_equal(com, M["box_com"]) and np.array_equal(sec, M["box_second"])
    np.testing.assert_array_equal(gm.lumped_vertex_masses(L, 1000.0), M["lat_mass"])


def _scene_from_traj(d):
    kind = str(d["kind"])
    obj = sc.ObjectSpec(kind=kind, soft=bool(d["soft_object"]))
    gs = sc.GripperSpec(soft_fingers=bool(d["soft_fingers"]))
    return sc.build_trial_scene(obj, gs, d["cand_R"], d["cand_T"], float(d["cand_opening"]))


def _oracle_env(scene):
    return osv.OracleEnv(scene.bodies, collide_pairs_off=scene.collide_pairs_off)


@pytest.mark.parametrize("name,steps", [("cfg1", 8), ("cylfail", 1), ("sphere", 4)])
def test_oracle_trajectory(golden, name, steps):
    d = np.load(golden / f"traj_{name}.npz")
    scene = _scene_from_traj(d)
    env = _oracle_env(scene)
    reps = json.loads(str(d["reports_json"]))
    out = osv.closing_rollout(env, scene.finger_links, scene.closing_dirs, min(steps, len(reps)))
    ell = max(float(np.linalg.norm(d["sv"][0].max(0) - d["sv"][0].min(0))), 0.05)
    for k, (x, rep) in enumerate(zip(out["x"], out["reports"])):
        ref = reps[k]
        assert rep["status"] == ref["status"] and rep["reason"] == ref["reason"], (k, rep, ref)
        assert rep["iterations"] == ref["iterations"], (k, rep["iterations"], ref["iterations"])
        assert np.abs(x - d["x"][k]).max() <= 1e-9 * ell, (k, np.abs(x - d["x"][k]).max() / ell)
    # broad phase: candidate sets at the recorded state are bit-exact
    off_pt = np.concatenate([[0], np.cumsum(d["pt_counts"])])
    off_ee = np.concatenate([[0], np.cumsum(d["ee_counts"])])
    for k in range(min(steps, len(reps))):
        env.x = d["x"][k].copy()
        s = d["sv"][k]
        c = env.candidates(s, 1.05e-3)
        assert np.array_equal(c["pt"], d["pt_rows"][off_pt[k]:off_pt[k + 1]])
        assert np.array_equal(c["ee"], d["ee_rows"][off_ee[k]:off_ee[k + 1]])
