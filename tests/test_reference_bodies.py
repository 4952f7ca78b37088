"""The drop-in claim at the body level: gripsim's OWN body objects -- the
SoftBody / AffineBody / KinematicBody list that its pipeline.config.build_trial_env(...) builds
(config.py:241-308) -- go through this package's layout (packing.layout_env, the host half of
grip_create) unchanged, and the layout equals the reference Environment's own arrays
(solver.py:214-363): DOFs, free mask, lumped / ABD mass blocks, surface map G, collision soup
(edges, triangles, vertex bodies, rest lengths) and the body pair mask.

CPU only; needs the reference importable (/root/reference in the build container), skipped
elsewhere.  Nothing here runs the reference's step."""

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference sources not present")


@pytest.fixture(scope="module")
def gs():
    sys.path.insert(0, str(REF))
    try:
        from gripsim.pipeline import config as cfg
        from gripsim.synth import GraspCandidate
        yield cfg, GraspCandidate
    finally:
        sys.path.remove(str(REF))


def _ref_env(cfg, GraspCandidate, kind, soft_object, soft_fingers, c, i):
    sc = cfg.SceneConfig()
    sc.object.soft = soft_object
    sc.gripper.soft_fingers = soft_fingers
    if kind == "cylinder":
        pytest.skip("cylinder needs a mesh file; covered by the box / sphere cases")
    sc.object.kind = kind
    cand = GraspCandidate("parallel", c["R"][i], c["T"][i], [c["opening"][i]], [])
    return cfg.build_trial_env(sc, cand)


@pytest.mark.parametrize("kind,soft_object,soft_fingers,which", [("box", False, True, 0), ("sphere", False, True, 2),
                                                                ("box", True, False, 0), ("sphere", True, False, 1)])
def test_reference_bodies_layout(gs, kind, soft_object, soft_fingers, which):
    cfg, GraspCandidate = gs
    from paper_2503_05020_b200 import packing
    from paper_2503_05020_b200 import scene as sc
    c = sc.load_cfg3_candidates() if soft_object else sc.load_cfg2_candidates()
    env, ob, fl = _ref_env(cfg, GraspCandidate, kind, soft_object, soft_fingers, c, which)
    pairs_off = [tuple(int(v) for v in np.nonzero(~env.soup.collide[a])[0]) for a in range(len(env.records))]
    off = [(a, b) for a, bs in enumerate(pairs_off) for b in bs if a < b
           and not (env.soup.body_kinematic[a] and env.soup.body_kinematic[b])]
    lay = packing.layout_env([r["body"] for r in env.records], off)   # gripsim's own body objects
    # DOFs and state
    assert lay.n_node * 3 == env.n_dofs and lay.n_sv == env.n_sv
    np.testing.assert_array_equal(lay.x0.reshape(-1), env.x)
    np.testing.assert_array_equal(np.repeat(lay.free, 3), env.free)
    # mass blocks (materials.py:208-213, solver.py:261-271)
    M = env.M.toarray()
    Mb = lay._arrays["Mb"]
    for n in range(lay.n_node):
        np.testing.assert_array_equal(Mb[n], M[3 * n:3 * n + 3, 3 * n:3 * n + 3])
    # collision soup (solver.py:320-335) and the rest lengths of the EE mollifier
    np.testing.assert_array_equal(lay.tris, env.soup.triangles)
    np.testing.assert_array_equal(lay.edges, env.soup.edges)
    np.testing.assert_array_equal(lay.vbody, env.soup.vertex_body)
    pk = packing.Packed([lay], [np.zeros(14)], [np.zeros(3)], packing.body_velocities(lay_bodies(env)))
    np.testing.assert_array_equal(pk.edge_rest_sq, env.soup.edge_rest_len_sq)
    # pair mask: collide and not both kinematic (CollisionSoup.pair_ok, broadphase.py:50-51)
    kin = env.soup.body_kinematic
    want = env.soup.collide & ~(kin[:, None] & kin[None, :])
    np.testing.assert_array_equal(lay.pair_ok, want)
    # surface map: G x == surface_positions (solver.py:277-286, 367-372)
    sv = env.surface_positions()
    for r in lay.records:
        sl = slice(r.surf0, r.surf0 + r.n_sv)
        if r.kind == "soft":
            np.testing.assert_array_equal(lay.x0[r.node0 + r.vmap], sv[sl])
        elif r.kind == "affine":
            np.testing.assert_allclose(lay.x0[r.node0][None] + r.xi @ lay.x0[r.node0 + 1:r.node0 + 4].T, sv[sl],
                                       rtol=0, atol=1e-15)
        else:
            np.testing.assert_array_equal(lay.kin0[sl], sv[sl])


def lay_bodies(env):
    return [r["body"] for r in env.records]
