"""Dataset emission: byte compatibility with the reference's writer and, on the
GPU, a recorded trial against the trial the reference recorded (tests/golden/dataset_cfg1,
written by gripsim.pipeline.dataset.emit_dataset in tests/golden/make_golden.py)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2503_05020_b200 import dataset as ds
from paper_2503_05020_b200.protocol import TrialRecord

GOLD = Path(__file__).resolve().parent / "golden" / "dataset_cfg1"


def _sha(p):
    return hashlib.sha256(Path(p).read_bytes()).hexdigest()


def _record_from_golden(tr):
    meta = tr["meta"]
    steps = [json.loads(line) for line in (GOLD / "trial_0000" / "steps.jsonl").read_text().splitlines()]
    rec = TrialRecord(candidate=meta["candidate"], verdict=meta["verdict"], failure=meta["failure"],
                      phase_markers=meta["phase_markers"], positions=tr["positions"], velocities=tr["velocities"],
                      times=tr["times"], stress=tr["stress"], step_reports=steps,
                      com_displacement=meta["com_displacement"], halt_forces=meta["halt_forces"],
                      finger_forces=meta["finger_forces"], metrics=meta["metrics"], object_body=meta["object_body"],
                      gripper_bodies=tuple(meta["gripper_bodies"]), n_steps=meta["n_steps"])
    rec.contacts = [c["events"] for c in tr["contacts"]]
    return rec, meta["params"]


def test_loaders_read_reference_files():
    man = ds.load_manifest(GOLD)
    assert man["format"] == "gripsim-dataset-v1" and man["n_trials"] == 1
    tr = ds.load_trial(GOLD / "trial_0000")
    n = tr["meta"]["n_steps"]
    assert tr["positions"].shape == (n, tr["positions"].shape[1], 3) and tr["velocities"].shape == tr["positions"].shape
    assert tr["stress"].shape[0] == n and tr["stress"].shape[2] == 7
    assert len(tr["contacts"]) == n and [c["step"] for c in tr["contacts"]] == list(range(n))
    for f, h in man["trials"][0]["files"].items():
        assert _sha(GOLD / "trial_0000" / f) == h


def test_writer_reproduces_reference_bytes(tmp_path):
    tr = ds.load_trial(GOLD / "trial_0000")
    rec, params = _record_from_golden(tr)
    man = ds.emit_dataset([rec], tmp_path, params=params)
    gold = ds.load_manifest(GOLD)
    assert man == gold
    assert (tmp_path / "manifest.json").read_bytes() == (GOLD / "manifest.json").read_bytes()


def test_traj_loader_rejects_bad_files(tmp_path):
    p = tmp_path / "t.bin"
    ds.write_traj(p, np.arange(3) * 0.01, np.zeros((3, 2, 3)), np.zeros((3, 2, 3)))
    raw = bytearray(p.read_bytes())
    raw[24] = 7  # frame 0 index
    p.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="index"):
        ds.load_traj(p)
    p.write_bytes(b"NOTATRAJ" + bytes(16))
    with pytest.raises(ValueError, match="magic"):
        ds.load_traj(p)
    q = tmp_path / "s.bin"
    ds.write_stress(q, np.zeros((0, 0, 7)))
    assert ds.load_stress(q).shape == (0, 0, 7)


@pytest.mark.gpu
def test_recorded_trial_matches_reference(tmp_path):
    """Our run_grasp_trial (device step, device contact events, device stress) under the same
    shortened protocol as the golden trial, emitted by our writer: same verdict, markers, step
    count, Newton iterations and contact stencils; positions within 1e-6 ell."""
    from paper_2503_05020_b200 import scene as sc
    from paper_2503_05020_b200.protocol import TrialProtocol, run_grasp_trial
    from paper_2503_05020_b200.solver import Environment

    pj = json.loads((GOLD.parent / "dataset_cfg1_protocol.json").read_text())
    s = sc.build_trial_scene(sc.ObjectSpec(kind="box"), sc.GripperSpec(soft_fingers=True), np.array(pj["R"]),
                             np.array(pj["T"]), float(pj["opening"]))
    env = Environment(s.bodies, collide_pairs_off=s.collide_pairs_off)
    prot = TrialProtocol(settle_duration=pj["settle_duration"], steady_max_duration=pj["steady_max_duration"],
                         gravity_phase_duration=pj["gravity_phase_duration"])
    ell = max(env.bbox_diagonal(), 0.05)
    rec = run_grasp_trial(env, prot, s.object_body, s.finger_links, record=True, closing_dirs=s.closing_dirs)
    rec.candidate = {"R": pj["R"], "T": pj["T"], "opening": pj["opening"]}
    ds.emit_dataset([rec], tmp_path, params={"protocol": "short", "seed": 0})
    ours = ds.load_trial(tmp_path / "trial_0000")
    ref = ds.load_trial(GOLD / "trial_0000")
    mo, mr = ours["meta"], ref["meta"]
    for k in ("verdict", "failure", "phase_markers", "n_steps", "object_body", "gripper_bodies"):
        assert mo[k] == mr[k], k
    assert set(mo["halt_forces"]) == set(mr["halt_forces"])
    for f in mr["halt_forces"]:
        assert mo["halt_forces"][f]["step"] == mr["halt_forces"][f]["step"]
        assert np.isclose(mo["halt_forces"][f]["force"], mr["halt_forces"][f]["force"], rtol=1e-6)
    assert ours["positions"].shape == ref["positions"].shape
    assert np.abs(ours["positions"] - ref["positions"]).max() <= 1e-6 * ell
    assert np.abs(ours["velocities"] - ref["velocities"]).max() <= 1e-6 * ell / 0.01
    np.testing.assert_allclose(ours["times"], ref["times"], rtol=0, atol=1e-12)
    sr = np.abs(ref["stress"]).max()
    assert np.abs(ours["stress"] - ref["stress"]).max() <= 1e-6 * sr
    for co, cr in zip(ours["contacts"], ref["contacts"]):
        assert [(e["kind"], e["bodies"], e["verts"]) for e in co["events"]] == \
               [(e["kind"], e["bodies"], e["verts"]) for e in cr["events"]]
        for eo, er in zip(co["events"], cr["events"]):
            assert abs(eo["d"] - er["d"]) <= 1e-6 * ell
            assert np.isclose(eo["lambda"], er["lambda"], rtol=1e-5, atol=1e-9)
    so = [json.loads(x) for x in (tmp_path / "trial_0000" / "steps.jsonl").read_text().splitlines()]
    sref = [json.loads(x) for x in (GOLD / "trial_0000" / "steps.jsonl").read_text().splitlines()]
    assert [(r["step"], r["status"], r["iterations"], r["reason"]) for r in so] == \
           [(r["step"], r["status"], r["iterations"], r["reason"]) for r in sref]


@pytest.mark.gpu
def test_batched_recording_matches_single_env(tmp_path):
    """BatchedGraspTrials(record=True): the golden trial recorded inside a batch of 3 (continuous
    batching) gives the same emitted trial as the single-env recorder, byte for byte."""
    from paper_2503_05020_b200 import scene as sc
    from paper_2503_05020_b200.multienv import DeviceEnvGroup
    from paper_2503_05020_b200.protocol import BatchedGraspTrials, TrialProtocol, run_grasp_trial
    from paper_2503_05020_b200.solver import Environment

    pj = json.loads((GOLD.parent / "dataset_cfg1_protocol.json").read_text())
    prot = TrialProtocol(settle_duration=pj["settle_duration"], steady_max_duration=pj["steady_max_duration"],
                         gravity_phase_duration=pj["gravity_phase_duration"])
    cands = sc.load_cfg2_candidates()
    scenes = [sc.build_trial_scene(sc.ObjectSpec(kind="box"), sc.GripperSpec(soft_fingers=True), np.array(pj["R"]),
                                   np.array(pj["T"]), float(pj["opening"]))] + [sc.cfg2_scene(i, cands) for i in (3, 6)]
    envs = [Environment(s.bodies, collide_pairs_off=s.collide_pairs_off) for s in scenes]
    trials = BatchedGraspTrials(DeviceEnvGroup(envs), scenes, prot, record=True)
    recs = trials.run()
    one = sc.build_trial_scene(sc.ObjectSpec(kind="box"), sc.GripperSpec(soft_fingers=True), np.array(pj["R"]),
                               np.array(pj["T"]), float(pj["opening"]))
    env1 = Environment(one.bodies, collide_pairs_off=one.collide_pairs_off)
    r1 = run_grasp_trial(env1, prot, one.object_body, one.finger_links, record=True, closing_dirs=one.closing_dirs)
    for r in (recs[0], r1):
        r.candidate = {"R": pj["R"], "T": pj["T"], "opening": pj["opening"]}
    ma = ds.emit_dataset([recs[0]], tmp_path / "batched")
    mb = ds.emit_dataset([r1], tmp_path / "single")
    a = json.loads((tmp_path / "batched" / "trial_0000" / "meta.json").read_text())
    b = json.loads((tmp_path / "single" / "trial_0000" / "meta.json").read_text())
    assert [k for k in a if a[k] != b[k]] == []
    assert ma["trials"][0]["files"] == mb["trials"][0]["files"]
    assert recs[1].positions is not None and len(recs[1].contacts) == recs[1].n_steps


def test_event_block_lines_match_reference_json():
    """The array fast path of contacts.jsonl writes exactly the reference's json.dumps text."""
    from paper_2503_05020_b200._native import EventBlock
    for line in (GOLD / "trial_0000" / "contacts.jsonl").read_text().splitlines():
        o = json.loads(line)
        ev = o["events"]
        i = np.array([[0 if e["kind"] == "point-triangle" else 1, *e["bodies"], *e["verts"]] for e in ev],
                     np.int32).reshape(-1, 7)
        d = np.array([[e["d"], e["lambda"]] for e in ev]).reshape(-1, 2)
        blk = EventBlock(i, d)
        assert ds._events_line(o["step"], blk) == line + "\n"
        assert blk.as_dicts() == [dict(e, bodies=tuple(e["bodies"])) for e in ev]
