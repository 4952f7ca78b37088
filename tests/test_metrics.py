"""D1/D2 grasp-quality metrics and the SDF build against the reference
(tests/golden/metrics.json, sdf_*.npz from gripsim's own trial_quality_metrics / build_sdf,
tests/golden/make_golden.py gen_metrics)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2503_05020_b200 import metrics as qm
from paper_2503_05020_b200 import scene as sc
from paper_2503_05020_b200 import sdf as sdfm

GOLD = Path(__file__).resolve().parent / "golden"


def _golden_env():
    from paper_2503_05020_b200.solver import Environment
    pj = json.loads((GOLD / "dataset_cfg1_protocol.json").read_text())
    s = sc.build_trial_scene(sc.ObjectSpec(kind="box"), sc.GripperSpec(soft_fingers=True), np.array(pj["R"]),
                             np.array(pj["T"]), float(pj["opening"]))
    return Environment(s.bodies, collide_pairs_off=s.collide_pairs_off), s


def test_gripper_samples_match_reference_generator():
    g = json.loads((GOLD / "metrics.json").read_text())
    env, _ = _golden_env()
    surfs = qm.gripper_surfaces_from_env(env, g["gripper_bodies"], x=np.array(g["x"]))
    pts = qm.sample_surfaces(surfs, 50_000, 0)
    assert np.array_equal(pts[:32], np.array(g["samples_head"]))
    np.testing.assert_allclose(pts.sum(axis=0), g["samples_sum"], rtol=1e-13)


def test_polar_rotation_and_watertight():
    g = json.loads((GOLD / "metrics.json").read_text())
    env, _ = _golden_env()
    r = env.records[g["object_body"]]
    q = np.array(g["x"])[r["dof0"]:r["dof0"] + 12]
    np.testing.assert_allclose(qm.polar_rotation(q[3:].reshape(3, 3)), g["polar_R"], atol=1e-14)
    tris = np.asarray(r["body"].surface.triangles)
    assert sdfm.is_watertight(tris)
    assert not sdfm.is_watertight(tris[:-1])


@pytest.mark.gpu
def test_build_sdf_matches_reference():
    """Rest-shape box SDF at resolution 32 and a soft cube's boundary SDF at 24: grid, far field
    and the GPU narrow band against the reference's build_sdf values."""
    env, _ = _golden_env()
    g = json.loads((GOLD / "metrics.json").read_text())
    r = env.records[g["object_body"]]
    ref = np.load(GOLD / "sdf_box32.npz")
    ours = sdfm.build_sdf(np.asarray(r["xi"]), np.asarray(r["body"].surface.triangles), resolution=32)
    assert ours.values.shape == ref["values"].shape
    np.testing.assert_array_equal(ours.origin, ref["origin"])
    np.testing.assert_array_equal(ours.spacing, ref["spacing"])
    np.testing.assert_allclose(ours.values, ref["values"], rtol=0, atol=1e-12)
    soft = np.load(GOLD / "sdf_soft_cube24.npz")
    o2 = sdfm.build_sdf(soft["vertices"], soft["triangles"], resolution=24)
    np.testing.assert_allclose(o2.values, soft["values"], rtol=0, atol=1e-12)
    off = np.abs(soft["values"]) > 1e-12   # grid points on the surface carry either sign of ~0
    assert np.array_equal(np.sign(o2.values[off]), np.sign(soft["values"][off]))


@pytest.mark.gpu
def test_trial_metrics_match_reference():
    """D1, D2, spacing and every sample's d_o (resolution 32) of the golden trial's final state;
    D1 / D2 at the default resolution 128 too."""
    env, s = _golden_env()
    g = json.loads((GOLD / "metrics.json").read_text())
    env.x = np.array(g["x"])
    gb = g["gripper_bodies"]
    for res in (32, 128):
        d1, d2, h = qm.trial_quality_metrics(env, g["object_body"], gb, resolution=res)
        assert (d1, d2, h) == (g[f"res{res}"]["D1"], g[f"res{res}"]["D2"], g[f"res{res}"]["spacing"]), res
    sdf = qm.object_sdf_from_env(env, g["object_body"], resolution=32)
    pts = qm.sample_surfaces(qm.gripper_surfaces_from_env(env, gb), 50_000, 0)
    dmax, d_o = qm.signed_inside_max(sdf, pts, want_values=True)
    ref = np.array(g["d_o_res32"])
    np.testing.assert_allclose(d_o, ref, rtol=0, atol=1e-12)
    assert dmax == ref.max()
