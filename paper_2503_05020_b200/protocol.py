"""Grasp validation protocol (gripsim/pipeline/protocol.py:1-277) on the device step.

``run_grasp_trial`` keeps the reference's per-env semantics for a single
Environment.  ``run_grasp_trials`` is the batched driver: one
host-side phase state machine per env, all envs advanced by one lockstep
device step per iteration, finger forces and contact flags read back as one
small array per step.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

GRAVITY_DIRECTIONS = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], np.float64)
PHASES = ["gravity+x", "gravity-x", "gravity+y", "gravity-y", "gravity+z", "gravity-z"]


@dataclass
class TrialProtocol:
    """protocol.py:25-46."""

    settle_duration: float = 0.05
    closing_speed: float = 0.05
    force_halt: float = 50.0
    gravity_magnitude: float = 9.8
    gravity_phase_duration: float = 0.1
    steady_speed_steps: int = 5
    steady_max_duration: float = 1.0
    stability_constant: float = 1.0

    def __post_init__(self):
        if min(self.settle_duration, self.gravity_phase_duration, self.steady_max_duration) <= 0:
            raise ValueError("durations must be positive")
        if self.force_halt <= 0 or self.closing_speed <= 0:
            raise ValueError("closing speed and halt threshold must be positive")


@dataclass
class TrialRecord:
    """protocol.py:49-69 (positions/stress recorded on request)."""

    candidate: dict = field(default_factory=dict)
    verdict: str = "unstable"
    failure: dict = field(default_factory=dict)
    phase_markers: dict = field(default_factory=dict)
    positions: np.ndarray = None
    velocities: np.ndarray = None
    times: np.ndarray = None
    stress: np.ndarray = None
    step_reports: list = field(default_factory=list)
    contacts: list = field(default_factory=list)      # per step: list of contact events
    com_displacement: dict = field(default_factory=dict)
    halt_forces: dict = field(default_factory=dict)
    finger_forces: list = field(default_factory=list)
    metrics: dict = field(default_factory=dict)
    object_body: int = 0
    gripper_bodies: tuple = ()
    n_steps: int = 0
    # safety report over the completed steps (not part of the reference record or the dataset
    # files): min stencil distance (> 0: no intersection) and min J = det F / det A (> 0: no
    # inverted element); filled by the device protocol
    min_distance: float = float("inf")
    min_J: float = float("inf")


# ---------------------------------------------------------------------------
# contact readout (protocol.py:72-98, contact.py:348-372)
# ---------------------------------------------------------------------------


def contact_events_now(env):
    """protocol.py:72-75: the active stencils of the fresh 1.05 dhat candidate set at the current
    state as {kind, bodies, verts, d, lambda} dicts, computed on the device (grip_contacts_now)."""
    return env._owner()._events_now(env._slot)[0]


def finger_contact_force(env, finger_bodies, events=None):
    """Sum of barrier forces over stencils touching the finger (protocol.py:78-86)."""
    ids = {finger_bodies} if np.isscalar(finger_bodies) else set(finger_bodies)
    bad = [b for b in ids if b < 0 or b >= len(env.records)]
    if bad:
        raise KeyError(f"unknown finger link id(s): {bad}")
    if events is None:
        events = contact_events_now(env)
    return sum(ev["lambda"] for ev in events if ids.intersection(ev["bodies"]))


def object_gripper_contact(env, object_body, gripper_bodies, events=None):
    """protocol.py:89-98."""
    if events is None:
        events = contact_events_now(env)
    g = set(gripper_bodies)
    return any(object_body in ev["bodies"] and set(ev["bodies"]) & g for ev in events)


# ---------------------------------------------------------------------------
# single-env trial (protocol.py:152-277)
# ---------------------------------------------------------------------------


def run_grasp_trial(env, protocol, object_body, finger_links, record=True, closing_dirs=None):
    """Full validation protocol on one Environment, reference semantics."""
    dt = env.solver_params.dt
    rec = TrialRecord(object_body=object_body,
                      gripper_bodies=tuple(sorted({b for ids in finger_links.values() for b in ids})))
    markers, halt_forces, positions, reps, times, forces_log, stress = {}, {}, [], [], [], [], []
    velocities, contacts_log = [], []
    n_done = [0]
    group = env._owner()
    group.set_recording(True)   # the step's contact events straight from the device finalize
    kin_recs = [r for r in env.records if r["kind"] == "kinematic"]

    def snapshot(events, report, forces):
        """protocol.py:113-146 (_Recorder.snapshot)."""
        kp = [r["positions"] for r in kin_recs]
        kv = [np.tile(np.asarray(r["body"].velocity, np.float64), (r["n_sv"], 1)) for r in kin_recs]
        positions.append(np.concatenate([env.node_positions()] + kp) if kp else env.node_positions().copy())
        velocities.append(np.concatenate([env.v.reshape(-1, 3)] + kv) if kv else env.v.reshape(-1, 3).copy())
        stress.append(env.stress_rows())
        contacts_log.append(events)
        reps.append(report.to_dict())
        forces_log.append(forces)

    def fail(phase, report):
        rec.verdict = "sim-failed"
        rec.failure = {"phase": phase, "reason": report.reason if report else env.fail_reason, "step": env.step_index}

    last_events = [None]

    def run_phase(name, n_steps, per_step=None, early_stop=None):
        start = n_done[0]
        for _ in range(n_steps):
            report = env.step()
            events = group._events(env._slot)
            last_events[0] = events
            forces = {f: finger_contact_force(env, ids, events) for f, ids in finger_links.items()}
            n_done[0] += 1
            times.append(env.time)
            if record:
                snapshot(events, report, forces)
            if per_step is not None:
                per_step(forces)
            if report.status == "failed":
                fail(name, report)
                return False
            if early_stop is not None and early_stop():
                break
        markers[name] = [start, n_done[0]]
        return True

    env.gravity = np.zeros(3)
    for ids in finger_links.values():
        for b in ids:
            env.records[b]["body"].velocity = np.zeros(3)
    ok = run_phase("settle", int(np.ceil(protocol.settle_duration / dt)))
    if ok:
        halted = {f: False for f in finger_links}
        for f, ids in finger_links.items():
            d = (closing_dirs or {}).get(f, env.records[ids[0]].get("closing_dir"))
            d = np.zeros(3) if d is None else np.asarray(d)
            for b in ids:
                env.records[b]["body"].velocity = d * protocol.closing_speed
        opening = float(np.asarray(env.records[finger_links[list(finger_links)[0]][0]].get("opening", 0.08)))
        max_close = int(np.ceil((opening / 2.0) / (protocol.closing_speed * dt))) + 5

        def per_step(forces):
            for f in finger_links:
                if not halted[f] and forces[f] > protocol.force_halt:
                    halted[f] = True
                    halt_forces[f] = {"force": forces[f], "step": n_done[0] - 1}
                    for b in finger_links[f]:
                        env.records[b]["body"].velocity = np.zeros(3)

        ok = run_phase("close", max_close, per_step=per_step, early_stop=lambda: all(halted.values()))
        for ids in finger_links.values():
            for b in ids:
                env.records[b]["body"].velocity = np.zeros(3)
    if ok:
        quiet = [0]

        def steady():
            quiet[0] = quiet[0] + 1 if env.max_point_speed() < env.contact_params.eps_v else 0
            return quiet[0] >= protocol.steady_speed_steps

        ok = run_phase("hold", int(np.ceil(protocol.steady_max_duration / dt)), early_stop=steady)
    com_disp = {}
    n_grav = int(np.ceil(protocol.gravity_phase_duration / dt))
    if ok:
        for name, direction in zip(PHASES, GRAVITY_DIRECTIONS):
            env.gravity = protocol.gravity_magnitude * direction
            com0 = env.body_com(object_body).copy()
            ok = run_phase(name, n_grav)
            com_disp[name] = float(np.linalg.norm(env.body_com(object_body) - com0))
            if not ok:
                break
    if rec.verdict != "sim-failed":
        thr = protocol.stability_constant * n_grav * env.contact_params.eps_v * dt
        events = last_events[0] if last_events[0] is not None else contact_events_now(env)
        in_contact = object_gripper_contact(env, object_body, rec.gripper_bodies, events)
        final = com_disp.get(PHASES[-1], np.inf)
        rec.verdict = "stable" if (in_contact and final < thr) else "unstable"
        rec.metrics.update(final_phase_com_disp=final, stability_threshold=thr, final_contact=bool(in_contact))
    rec.phase_markers = markers
    rec.com_displacement = com_disp
    rec.halt_forces = halt_forces
    rec.n_steps = n_done[0]
    if record:
        rec.positions = np.array(positions)
        rec.velocities = np.array(velocities)
        rec.times = np.array(times)
        n_tets = env.layout.n_tet
        rec.stress = np.array(stress) if n_tets else np.zeros((len(times), 0, 7))
        rec.contacts = contacts_log
        rec.step_reports = reps
        rec.finger_forces = forces_log
    return rec


# ---------------------------------------------------------------------------
# batched trials: one state machine per env, lockstep device steps
# ---------------------------------------------------------------------------

_SETTLE, _CLOSE, _HOLD, _GRAV, _DONE = range(5)
_PHASE_NAMES = {_SETTLE: "settle", _CLOSE: "close", _HOLD: "hold"}


class BatchedGraspTrials:
    """The grasp protocol (protocol.py:152-277) for every env of a device group at once.

    Per-env phase state lives in numpy arrays; controls (finger velocities,
    gravity) go to the device as two arrays per step and the protocol's
    per-step observables (finger forces, contact flags, object COM, max
    point speed) come back from the device's finalize as small arrays, so no
    full state is read back.  Each env follows exactly the reference's
    sequence of controls and decisions; envs are only batched, never coupled.
    """

    def __init__(self, group, scenes, protocol=None, record=False):
        self.group = group
        self.dev = group.dev
        self.record = record
        if record:   # per-step frames for dataset emission (protocol.py:113-146, dataset.py)
            group.set_recording(True)
            p0 = group.packed
            self._kin_sl = []
            for i, env in enumerate(group.envs):
                sl = [(int(p0.sv_off[i]) + r.surf0, int(p0.sv_off[i]) + r.surf0 + r.n_sv, r.id)
                      for r in env.layout.records if r.kind == "kinematic"]
                self._kin_sl.append(sl)
            self._frames = [self._empty_frames() for _ in group.envs]
        self.protocol = pr = protocol or TrialProtocol()
        p = group.packed
        E = p.n_env
        self.E = E
        env0 = group.envs[0]
        self.dt = dt = env0.solver_params.dt
        self.eps_v = np.array([e.contact_params.eps_v for e in group.envs])
        self.n_settle = int(np.ceil(pr.settle_duration / dt))
        self.n_hold = int(np.ceil(pr.steady_max_duration / dt))
        self.n_grav = int(np.ceil(pr.gravity_phase_duration / dt))
        boff = p.body_off[:-1].astype(np.int64)
        self.fnames = [list(s.finger_links) for s in scenes]
        nf = len(self.fnames[0])
        self.fb = np.zeros((E, nf), np.int64)
        self.cd = np.zeros((E, nf, 3))
        for i, s in enumerate(scenes):
            for j, f in enumerate(self.fnames[i]):
                ids = s.finger_links[f]
                if len(ids) != 1:
                    raise ValueError("batched trials expect one body per finger link")
                self.fb[i, j] = boff[i] + ids[0]
                self.cd[i, j] = np.asarray(s.closing_dirs[f], np.float64)
        self.obj = boff + np.array([s.object_body for s in scenes], np.int64)
        self.gbits = np.array([sum(1 << b for ids in s.finger_links.values() for b in ids) for s in scenes], np.int64)
        self.max_close = np.array([int(np.ceil((s.opening / 2.0) / (pr.closing_speed * dt))) + 5 for s in scenes])
        self.vel = np.zeros((p.n_body_total, 3))
        self.grav = np.zeros((E, 3))
        self.phase = np.full(E, _SETTLE)
        self.pstep = np.zeros(E, np.int64)
        self.gphase = np.zeros(E, np.int64)
        self.quiet = np.zeros(E, np.int64)
        self.halted = np.zeros((E, nf), bool)
        self.nsteps = np.zeros(E, np.int64)
        self.phase_start = np.zeros(E, np.int64)
        self.com0 = np.zeros((E, 3))
        self.com_disp = np.full((E, 6), np.nan)
        self.records = [TrialRecord(object_body=s.object_body,
                                    gripper_bodies=tuple(sorted({b for ids in s.finger_links.values() for b in ids})))
                        for s in scenes]
        self.env_steps = 0
        self.reports = []

    @staticmethod
    def _empty_frames():
        return {"x": [], "v": [], "t": [], "stress": [], "events": [], "reports": [], "forces": []}

    def _snapshot(self, ids, rep, alphas, events, ff):
        """Record one frame for every env in ids (the reference's _Recorder.snapshot)."""
        from paper_2503_05020_b200.solver import report_from_row
        p = self.group.packed
        m = np.zeros(self.E, np.uint8)
        m[ids] = 1
        x, v, kin, st = self.dev.frames(m)   # the finalized envs only, packed in env order
        boff = p.body_off
        on = os_ = ot = 0
        assert np.all(np.diff(ids) > 0)   # frames come packed in env order
        for k, e in enumerate(ids):
            nn, ns, nt = p.node_off[e + 1] - p.node_off[e], p.sv_off[e + 1] - p.sv_off[e], p.tet_off[e + 1] - p.tet_off[e]
            s0 = p.sv_off[e]
            kp = [kin[os_ + a - s0:os_ + b - s0] for a, b, _ in self._kin_sl[e]]
            kv = [np.tile(self.vel[boff[e] + bid], (b - a, 1)) for a, b, bid in self._kin_sl[e]]
            fr = self._frames[e]
            fr["x"].append(np.concatenate([x[on:on + nn]] + kp))
            fr["v"].append(np.concatenate([v[on:on + nn]] + kv))
            env = self.group.envs[e]
            fr["t"].append(env._time + env.solver_params.dt)   # env.time after the step, accumulated
            fr["stress"].append(st[ot:ot + nt])
            on, os_, ot = on + nn, os_ + ns, ot + nt
            fr["events"].append(events[e])
            r = report_from_row(rep[e], alphas[e], self.group.envs[e].env_id)
            r.time = env._time
            r.step_index = env._step
            fr["reports"].append(r.to_dict())
            fr["forces"].append({self.fnames[e][j]: ff[k][j] for j in range(len(ff[k]))})

    def _close_record(self, e):
        """Move env e's frames into its TrialRecord (trial finished)."""
        fr = self._frames[e]
        r = self.records[e]
        r.positions = np.array(fr["x"])
        r.velocities = np.array(fr["v"])
        r.times = np.array(fr["t"])
        nt = self.group.packed.tet_off[e + 1] - self.group.packed.tet_off[e]
        r.stress = np.array(fr["stress"]) if nt else np.zeros((len(fr["t"]), 0, 7))
        r.contacts = fr["events"]
        r.step_reports = fr["reports"]
        r.finger_forces = fr["forces"]
        self._frames[e] = self._empty_frames()

    @property
    def done(self):
        return bool(np.all(self.phase == _DONE))

    # -- continuous refill (dataset-generation mode) ------------------------------------------
    @staticmethod
    def scene_payload(scene):
        """Device reset payload of a grasp scene: its one-env Packed arrays (a new candidate for the
        same meshes changes only the pose- / material-dependent ones, grip_reset_envs)."""
        from paper_2503_05020_b200 import packing
        lay = packing.layout_env(scene.bodies, scene.collide_pairs_off)
        pk = packing.Packed([lay], [np.zeros(14)], [np.zeros(3)], packing.body_velocities(scene.bodies))
        return {"packed": pk, "scene": scene}

    def refill(self, slots, payloads):
        """Start a fresh trial in each finished slot with a new candidate of the same topology."""
        mask = _reset_slots(self, slots, payloads)
        pr = self.protocol
        for e, pl in zip(slots, payloads):
            sc = pl["scene"]
            for j, f in enumerate(self.fnames[e]):
                self.cd[e, j] = np.asarray(sc.closing_dirs[f], np.float64)
            self.max_close[e] = int(np.ceil((sc.opening / 2.0) / (pr.closing_speed * self.dt))) + 5
            self.vel[self.fb[e]] = 0.0
            self.grav[e] = 0.0
            self.phase[e] = _SETTLE
            self.pstep[e] = self.gphase[e] = self.quiet[e] = self.nsteps[e] = self.phase_start[e] = 0
            self.halted[e] = False
            self.com_disp[e] = np.nan
            self.records[e] = TrialRecord(object_body=sc.object_body, gripper_bodies=self.records[e].gripper_bodies)
            if self.record:
                self._frames[e] = self._empty_frames()
        del mask
        if hasattr(self, "_iter"):
            self._iter[list(slots)] = False
            self._need[list(slots)] = True

    def advance(self, keep_reports=False):
        """One lockstep protocol step over every unfinished env; returns env-steps executed."""
        ids = np.nonzero(self.phase != _DONE)[0]
        if len(ids) == 0:
            return 0
        mask = np.zeros(self.E, np.uint8)
        mask[ids] = 1
        self.dev.set_controls(self.grav, self.vel)
        rep, alphas = self.dev.step(mask)
        self._after_step(ids, rep, keep_reports, alphas)
        return len(ids)

    def advance_round(self, keep_reports=False):
        """One continuous-batching round (grip_round): envs that finished their previous
        protocol step begin the next one, every unfinished env gets one Newton sweep, envs
        whose step converged are finalized and advance their protocol.  Returns the number
        of env-steps completed in this round."""
        if not hasattr(self, "_iter"):
            self._iter = np.zeros(self.E, bool)
            self._need = self.phase != _DONE
        begin = self._need & (self.phase != _DONE)
        if not begin.any() and not self._iter.any():
            return 0
        if begin.any():
            self.dev.set_controls(self.grav, self.vel)
        fin, rep, alphas = self.dev.round(begin, self._iter)
        self._iter = (self._iter | begin) & ~fin
        self._need = np.zeros(self.E, bool)
        ids = np.nonzero(fin)[0]
        if len(ids):
            self._after_step(ids, rep, keep_reports, alphas)
            self._need[ids] = self.phase[ids] != _DONE
        return len(ids)

    def _after_step(self, ids, rep, keep_reports=False, alphas=None):
        """Protocol bookkeeping after envs `ids` completed a time step (protocol.py:176-188)."""
        pr = self.protocol
        force, cmask, _ = self.dev.contacts()
        com, speed = self.dev.body_state()
        self.group.invalidate()
        if self.record:
            m = np.zeros(self.E, np.uint8)
            m[ids] = 1
            events = self.dev.event_blocks(m)
            # finger forces from the recorded events, as the reference sums them (protocol.py:78-86)
            boff = self.group.packed.body_off
            fsum = [[events[e].force_on(self.fb[e, j] - boff[e]) for j in range(self.fb.shape[1])] for e in ids]
            ffr = np.array(fsum, np.float64).reshape(len(ids), self.fb.shape[1])
            self._snapshot(ids, rep, alphas, events, fsum)
        for e in ids:
            env = self.group.envs[e]
            env._time += env.solver_params.dt
            env._step += 1
        if keep_reports:
            self.reports.append((ids.copy(), rep[ids].copy()))
        self.env_steps += len(ids)
        self.nsteps[ids] += 1
        self.pstep[ids] += 1
        ph = self.phase[ids]
        ff = force[self.fb[ids]]                       # (n, fingers)
        if self.record:
            ff = ffr   # the recorded events' sums, exactly as the single-env recorder halts on
        # close-phase halting happens before the failure check (protocol.py:181-186)
        closing = ph == _CLOSE
        newly = closing[:, None] & ~self.halted[ids] & (ff > pr.force_halt)
        if newly.any():
            for k, j in zip(*np.nonzero(newly)):
                e = ids[k]
                self.halted[e, j] = True
                self.records[e].halt_forces[self.fnames[e][j]] = {"force": float(ff[k, j]), "step": int(self.nsteps[e] - 1)}
                self.vel[self.fb[e, j]] = 0.0
        failed = rep["status"][ids] == 2
        for k in np.nonzero(failed)[0]:
            e = ids[k]
            name = _PHASE_NAMES.get(int(ph[k]), PHASES[int(self.gphase[e])] if ph[k] == _GRAV else "")
            r = self.records[e]
            r.verdict = "sim-failed"
            from paper_2503_05020_b200._native import REASONS
            r.failure = {"phase": name, "reason": REASONS.get(int(rep["reason"][e]), "unknown"),
                         "step": int(self.nsteps[e])}
            if ph[k] == _GRAV:
                r.com_displacement[name] = float(np.linalg.norm(com[self.obj[e]] - self.com0[e]))
            self.phase[e] = _DONE
        ok = ~failed
        ended = np.zeros(len(ids), bool)
        ended |= (ph == _SETTLE) & (self.pstep[ids] >= self.n_settle)
        ended |= closing & (self.halted[ids].all(axis=1) | (self.pstep[ids] >= self.max_close[ids]))
        hold = ph == _HOLD
        if hold.any():
            q = np.where(speed[ids] < self.eps_v[ids], self.quiet[ids] + 1, 0)
            self.quiet[ids] = np.where(hold, q, self.quiet[ids])
            ended |= hold & ((self.quiet[ids] >= pr.steady_speed_steps) | (self.pstep[ids] >= self.n_hold))
        ended |= (ph == _GRAV) & (self.pstep[ids] >= self.n_grav)
        ended &= ok
        for k in np.nonzero(ended)[0]:
            e = ids[k]
            r = self.records[e]
            name = _PHASE_NAMES.get(int(ph[k]), PHASES[int(self.gphase[e])] if ph[k] == _GRAV else "")
            r.phase_markers[name] = [int(self.phase_start[e]), int(self.nsteps[e])]
            self.phase_start[e] = self.nsteps[e]
            self.pstep[e] = 0
            fbe = self.fb[e]
            if ph[k] == _SETTLE:
                self.phase[e] = _CLOSE
                self.vel[fbe] = self.cd[e] * pr.closing_speed
            elif ph[k] == _CLOSE:
                self.vel[fbe] = 0.0
                self.phase[e] = _HOLD
            elif ph[k] == _HOLD:
                self.phase[e] = _GRAV
                self.gphase[e] = 0
                self.grav[e] = pr.gravity_magnitude * GRAVITY_DIRECTIONS[0]
                self.com0[e] = com[self.obj[e]]
            else:
                g = int(self.gphase[e])
                d = float(np.linalg.norm(com[self.obj[e]] - self.com0[e]))
                r.com_displacement[PHASES[g]] = d
                self.gphase[e] = g + 1
                if g + 1 >= 6:
                    self.phase[e] = _DONE
                    thr = pr.stability_constant * self.n_grav * self.eps_v[e] * self.dt
                    in_contact = bool(int(cmask[self.obj[e]]) & int(self.gbits[e]))
                    r.verdict = "stable" if (in_contact and d < thr) else "unstable"
                    r.metrics.update(final_phase_com_disp=d, stability_threshold=thr, final_contact=in_contact)
                else:
                    self.grav[e] = pr.gravity_magnitude * GRAVITY_DIRECTIONS[g + 1]
                    self.com0[e] = com[self.obj[e]]
        for e in ids:
            self.records[e].n_steps = int(self.nsteps[e])
            if self.record and self.phase[e] == _DONE:
                self._close_record(e)

    def run(self, max_steps=None, lockstep=False):
        n = 0
        while not self.done and (max_steps is None or n < max_steps):
            self.advance() if lockstep else self.advance_round()
            n += 1
        return self.records


def run_grasp_trials(group, scenes, protocol=None, max_steps=None, lockstep=False, record=False):
    """Protocol for all envs of a group; returns TrialRecords (labels, markers, COM, halts; with
    record=True also the per-step frames the reference's recorder keeps, for dataset emission)."""
    return BatchedGraspTrials(group, scenes, protocol, record=record).run(max_steps, lockstep=lockstep)


# ---------------------------------------------------------------------------
# device-resident protocol: the state machine above as a kernel (grip_run_rounds)
# ---------------------------------------------------------------------------
_MARK_NAMES = ["settle", "close", "hold"] + PHASES
_VERDICTS = {1: "stable", 2: "unstable", 3: "sim-failed"}


def _reset_slots(trials, slots, payloads):
    """Write the payloads (BatchedGraspTrials.scene_payload: a one-env Packed) of the refilled slots
    into a full-size host copy of the batch's scene arrays and reset those envs on the device
    (grip_reset_envs: pose, rest shape, masses, rest lengths, materials; every other per-env state
    as in a fresh batch)."""
    import copy

    from paper_2503_05020_b200._native import DeviceBatch
    p = trials.group.packed
    if not hasattr(trials, "_host"):
        trials._host = copy.copy(p)
        for name, _, _ in DeviceBatch.RESET_FIELDS:
            setattr(trials._host, name, np.array(getattr(p, name), copy=True))
        trials._host.env_cell_hint = np.array(p.env_cell_hint, copy=True)
    h = trials._host
    mask = np.zeros(trials.E, np.uint8)
    for e, pl in zip(slots, payloads):
        q = pl["packed"]
        for off in ("node_off", "sv_off", "tri_off", "edge_off", "tet_off", "abd_off", "body_off"):
            if getattr(p, off)[e + 1] - getattr(p, off)[e] != getattr(q, off)[1]:
                raise ValueError("refill needs the same topology as the slot's current scene")
        for name, k, off in DeviceBatch.RESET_FIELDS:
            lo, hi = getattr(p, off)[e], getattr(p, off)[e + 1]
            getattr(h, name)[k * lo:k * hi] = np.asarray(getattr(q, name)).reshape(-1)
        h.env_cell_hint[e] = q.env_cell_hint[0]
        env = trials.group.envs[e]
        env._time, env._step, env.status = 0.0, 0, "active"
        mask[e] = 1
    trials.dev.reset_envs(mask, h)
    return mask


class DeviceProtocolTrials:
    """The grasp protocol (protocol.py:152-277) run on the device (k_protocol): after every
    finalize the kernel makes BatchedGraspTrials' decisions itself -- finger halts, phase ends,
    controls of the next step, the verdict -- so ``advance(R)`` runs R continuous-batching
    rounds with one synchronisation.  Records are read back when trials end."""

    def __init__(self, group, scenes, protocol=None):
        from paper_2503_05020_b200._native import REASONS
        self._reasons = REASONS
        self.group = group
        self.dev = group.dev
        self.protocol = pr = protocol or TrialProtocol()
        E = group.packed.n_env
        self.E = E
        env0 = group.envs[0]
        self.dt = dt = env0.solver_params.dt
        self.fnames = [list(s.finger_links) for s in scenes]
        fb = np.zeros((E, 2), np.int32)
        cd = np.zeros((E, 2, 3))
        for i, s in enumerate(scenes):
            if len(self.fnames[i]) != 2:
                raise ValueError("device protocol expects two finger links")
            for j, f in enumerate(self.fnames[i]):
                ids = s.finger_links[f]
                if len(ids) != 1:
                    raise ValueError("device protocol expects one body per finger link")
                fb[i, j] = ids[0]
                cd[i, j] = np.asarray(s.closing_dirs[f], np.float64)
        obj = np.array([s.object_body for s in scenes], np.int32)
        gbits = np.array([sum(1 << b for ids in s.finger_links.values() for b in ids) for s in scenes], np.int32)
        self.max_close = np.array([int(np.ceil((s.opening / 2.0) / (pr.closing_speed * dt))) + 5 for s in scenes],
                                  np.int32)
        self.cd = cd
        cfg = [int(np.ceil(pr.settle_duration / dt)), int(np.ceil(pr.steady_max_duration / dt)),
               int(np.ceil(pr.gravity_phase_duration / dt)), pr.closing_speed, pr.force_halt, pr.gravity_magnitude,
               pr.steady_speed_steps, pr.stability_constant]
        self.gripper_bodies = [tuple(sorted({b for ids in s.finger_links.values() for b in ids})) for s in scenes]
        self.object_body = [s.object_body for s in scenes]
        self.dev.protocol_setup(fb, cd, obj, gbits, self.max_close, cfg)
        self.finished = np.zeros(E, bool)
        self.env_steps = 0

    def advance(self, rounds=1):
        """R device rounds; returns the env-steps completed."""
        n = self.dev.run_rounds(rounds)
        self.group.invalidate()
        self.env_steps += n
        return n

    def advance_async(self, rounds=1):
        """Enqueue R device rounds and their readout; returns a ticket for wait()."""
        return self.dev.run_rounds_async(rounds)

    def wait(self, ticket):
        """(env-steps, protocol records) of an advance_async call, once it finished."""
        n, out = self.dev.rounds_wait(ticket)
        self.group.invalidate()
        self.env_steps += n
        return n, out

    def record(self, e, out=None):
        """TrialRecord of env e from the device protocol state."""
        o = (out if out is not None else self.dev.protocol_read())[e]
        r = TrialRecord(object_body=self.object_body[e], gripper_bodies=self.gripper_bodies[e])
        r.n_steps = int(o.n_steps)
        r.verdict = _VERDICTS.get(int(o.verdict), "running")
        r.min_distance, r.min_J = float(o.min_distance), float(o.min_J)
        r.phase_markers = {_MARK_NAMES[k]: [int(o.markers[2 * k]), int(o.markers[2 * k + 1])]
                           for k in range(9) if o.markers[2 * k] >= 0}
        for j, f in enumerate(self.fnames[e]):
            if (o.halted >> j) & 1:
                r.halt_forces[f] = {"force": float(o.halt_force[j]), "step": int(o.halt_step[j])}
        ng = min(6, len([k for k in range(3, 9) if o.markers[2 * k] >= 0]) + (1 if o.verdict == 3 and o.fail_phase >= 3 else 0))
        for g in range(ng):
            r.com_displacement[PHASES[g]] = float(o.com_disp[g])
        if o.verdict == 3:
            r.failure = {"phase": _MARK_NAMES[int(o.fail_phase)], "reason": self._reasons.get(int(o.fail_reason), "unknown"),
                         "step": int(o.fail_step)}
        elif o.verdict in (1, 2):
            r.metrics.update(final_phase_com_disp=float(o.final_disp), stability_threshold=float(o.threshold),
                             final_contact=bool(o.final_contact))
        return r

    def done_envs(self, out=None):
        o = out if out is not None else self.dev.protocol_read()
        return np.array([o[e].phase == 4 for e in range(self.E)])

    def refill(self, slots, payloads):
        """New trials in `slots` with new candidates of the same topology (BatchedGraspTrials.refill)."""
        _reset_slots(self, slots, payloads)
        pr = self.protocol
        cds, mcs = [], []
        for e, pl in zip(slots, payloads):
            sc = pl["scene"]
            cds.append(np.array([np.asarray(sc.closing_dirs[f], np.float64) for f in self.fnames[e]]))
            mcs.append(int(np.ceil((sc.opening / 2.0) / (pr.closing_speed * self.dt))) + 5)
        self.restart(slots, cds, mcs)

    def restart(self, slots, closing_dirs, max_close):
        """New trials in `slots` (after grip_reset_envs gave them new candidates)."""
        m = np.zeros(self.E, np.uint8)
        m[list(slots)] = 1
        for e, c, mc in zip(slots, closing_dirs, max_close):
            self.cd[e] = c
            self.max_close[e] = mc
        self.dev.protocol_reset(m, self.cd, self.max_close)

    def run(self, rounds_per_call=8, max_rounds=100000):
        n = 0
        while n < max_rounds:
            self.advance(rounds_per_call)
            n += rounds_per_call
            out = self.dev.protocol_read()
            if self.done_envs(out).all():
                break
        out = self.dev.protocol_read()
        return [self.record(e, out) for e in range(self.E)]
