"""Batched execution of independent environments on one GPU.

``Batch`` mirrors gripsim.multienv.Batch (multienv.py:73-178): lockstep time
steps, per-env freezing, quarantine of failures with tombstones, per-env
step reports.  The difference is where the sweeps run: the reference loops
``newton_iteration`` over pending envs in Python (or forks a process pool);
here one device launch sequence advances every pending env per sweep, and an
env that converged simply drops out of the pending list (frozen) until the
step ends.
"""

from __future__ import annotations

import hashlib
import os
import time
from dataclasses import dataclass, field

import numpy as np

from paper_2503_05020_b200 import _native as nv
from paper_2503_05020_b200 import packing
from paper_2503_05020_b200.solver import StepReport, report_from_row


@dataclass
class SchedulerConfig:
    """multienv.py:25-29 (max_workers is accepted; the device path needs no process pool)."""

    max_workers: int = 0
    deterministic: bool = True
    seed: int = 0


@dataclass
class BatchReport:
    step_reports: list = field(default_factory=list)
    wall_clock: dict = field(default_factory=dict)
    counts: dict = field(default_factory=dict)

    def update_counts(self, batch):
        c = {"active": 0, "frozen": 0, "failed": 0, "done": 0}
        for s in batch.statuses:
            c[s] = c.get(s, 0) + 1
        self.counts = c
        return c


class AssetCache:
    """Content-hash keyed read-only assets (multienv.py:48-70)."""

    def __init__(self):
        self._store = {}

    @staticmethod
    def key_of(*arrays):
        h = hashlib.sha256()
        for a in arrays:
            a = np.ascontiguousarray(a)
            h.update(str(a.dtype).encode())
            h.update(str(a.shape).encode())
            h.update(a.tobytes())
        return h.hexdigest()

    def get_or_build(self, key, builder):
        if key not in self._store:
            self._store[key] = builder()
        return self._store[key]

    def __len__(self):
        return len(self._store)


class DeviceEnvGroup:
    """Envs sharing one DeviceBatch; every Environment facade reads/writes through it."""

    def __init__(self, envs, device=None):
        self.envs = list(envs)
        lays = [e.layout for e in self.envs]
        params = [e.params_row() for e in self.envs]
        grav = [e.gravity for e in self.envs]
        vel = np.concatenate([packing.body_velocities(e.bodies) for e in self.envs]) if self.envs else np.zeros((0, 3))
        self.packed = packing.Packed(lays, params, grav, vel)
        # carry over state of envs that were stepped elsewhere before joining
        self.dev = nv.DeviceBatch(self.packed, device=device)
        x0 = []
        v0 = []
        kin0 = []
        moved = False
        for e in self.envs:
            if e._batch is not None:
                moved = True
            x0.append(e.x.reshape(-1, 3))
            v0.append(e.v.reshape(-1, 3))
            kin0.append(np.concatenate([e._kin_positions(r) if r.kind == "kinematic" else np.zeros((r.n_sv, 3))
                                        for r in e.layout.records]) if e.layout.n_sv else np.zeros((0, 3)))
        if moved:
            self.dev.set_state(np.concatenate(x0), np.concatenate(v0), np.concatenate(kin0))
        for i, e in enumerate(self.envs):
            e._batch = self
            e._slot = i
        self._cache = None
        self._sv_cache = None

    # -- controls ---------------------------------------------------------------------
    def push_controls(self):
        g = np.stack([e.gravity for e in self.envs])
        v = np.concatenate([packing.body_velocities(e.bodies) for e in self.envs])
        self.dev.set_controls(g, v)

    # -- cached state --------------------------------------------------------------------
    def invalidate(self):
        self._cache = None
        self._sv_cache = None

    def _state(self):
        if self._cache is None:
            self._cache = self.dev.get_state(True)
        return self._cache

    def _node_slice(self, slot, which):
        x, v, _ = self._state()
        a, b = self.packed.node_off[slot], self.packed.node_off[slot + 1]
        return (x if which == "x" else v)[a:b]

    def _set_node_slice(self, slot, which, val):
        x, v, kin = (a.copy() for a in self._state())
        a, b = self.packed.node_off[slot], self.packed.node_off[slot + 1]
        (x if which == "x" else v)[a:b] = val
        self.dev.set_state(x, v, kin)
        self.invalidate()

    def _sv_slice(self, slot, which):
        _, _, kin = self._state()
        a, b = self.packed.sv_off[slot], self.packed.sv_off[slot + 1]
        return kin[a:b]

    def _surface(self, slot):
        if self._sv_cache is None:
            self._sv_cache = self.dev.surface()
        a, b = self.packed.sv_off[slot], self.packed.sv_off[slot + 1]
        return self._sv_cache[a:b].copy()

    def _candidates(self, slot, radius):
        return self.dev.candidates(slot, radius)

    def _contacts(self, slot):
        f, m, md = self.dev.contacts()
        a, b = self.packed.body_off[slot], self.packed.body_off[slot + 1]
        return f[a:b], m[a:b], float(md[slot])

    def _events(self, slot):
        """Device contact events of the slot's last finalize (recording switched on here)."""
        if not getattr(self, "_recording", False):
            raise RuntimeError("contact-event recording is off for this device group")
        return self.dev.events(self._mask([slot]))[slot]

    def _events_now(self, slot, radius_factor=1.05):
        """Contact events at the slot's current state, computed on the device (grip_contacts_now)."""
        m = self._mask([slot])
        md = self.dev.contacts_now(m, radius_factor)
        return self.dev.events(m)[slot], float(md[slot])

    def set_recording(self, on=True):
        self.dev.set_recording(on)
        self._recording = bool(on)

    def _stress(self, slot):
        s = self.dev.stress()
        a, b = self.packed.tet_off[slot], self.packed.tet_off[slot + 1]
        return s[a:b]

    # -- stepping ----------------------------------------------------------------------------
    def _mask(self, slots):
        m = np.zeros(len(self.envs), np.uint8)
        m[list(slots)] = 1
        return m

    def _reports(self, rep, alphas, slots):
        out = {}
        for s in slots:
            e = self.envs[s]
            r = report_from_row(rep[s], alphas[s], e.env_id)
            r.time = e._time
            r.step_index = e._step
            e._time += e.solver_params.dt
            e._step += 1
            if r.status == "failed":
                e.status = "failed"
                e.fail_reason = r.reason
            out[s] = r
        return out

    def _begin(self, slots):
        self.push_controls()
        self.dev.begin_step(self._mask(slots))
        self.invalidate()

    def _iterate(self, slots):
        pend = self.dev.newton_iteration(self._mask(slots))
        self.invalidate()
        return ~pend

    def _finalize(self, slots):
        rep, alphas = self.dev.finalize_step(self._mask(slots))
        self.invalidate()
        return self._reports(rep, alphas, slots)

    def _step(self, slots):
        self.push_controls()
        rep, alphas = self.dev.step(self._mask(slots))
        self.invalidate()
        return self._reports(rep, alphas, slots)


class Batch:
    """A set of isolated environments stepped together (multienv.py:73-178)."""

    def __init__(self, envs, scheduler=None, device=None):
        self.envs = list(envs)
        self.scheduler = scheduler or SchedulerConfig()
        self.statuses = ["active"] * len(self.envs)
        self.report = BatchReport(step_reports=[[] for _ in self.envs])
        for i, env in enumerate(self.envs):
            env.env_id = i
            if env.status == "failed":
                self.statuses[i] = "failed"
        self.group = DeviceEnvGroup(self.envs, device=device)

    def active_ids(self):
        return [i for i, s in enumerate(self.statuses) if s == "active"]

    def quarantine_failures(self):
        """Fail envs with non-finite state or a failed solve; keep a tombstone (multienv.py:98-123).
        The non-finite test runs on the device (grip_check_finite: one flag per env comes back)."""
        nonfinite = self.group.dev.check_finite()
        for i, env in enumerate(self.envs):
            if self.statuses[i] in ("failed", "done"):
                continue
            bad = env.status == "failed"
            reason = env.fail_reason
            if not bad and env.n_dofs and nonfinite[i]:
                bad, reason = True, "non-finite state"
                env.status, env.fail_reason = "failed", reason
            if bad:
                self.statuses[i] = "failed"
                self.report.step_reports[i].append({"env": i, "status": "failed", "reason": reason,
                                                    "step": env.step_index})
                self.envs[i] = _FailedEnvTombstone(i, env.name, reason, env.step_index)
        return list(self.statuses)

    def mark_done(self, i):
        self.statuses[i] = "done"

    def step(self):
        """One lockstep time step over all active envs with per-env freezing (multienv.py:130-156)."""
        self.quarantine_failures()
        ids = self.active_ids()
        t0 = time.perf_counter()
        reports = []
        if ids:
            out = self.group._step(ids)
            reports = [out[i] for i in ids]
        self.report.wall_clock["step"] = self.report.wall_clock.get("step", 0.0) + (time.perf_counter() - t0)
        for i, rep in zip(ids, reports):
            self.report.step_reports[i].append(rep.to_dict())
        self.quarantine_failures()
        self.report.update_counts(self)
        return reports


class _FailedEnvTombstone:
    """multienv.py:181-191."""

    def __init__(self, env_id, name, reason, step_index):
        self.env_id = env_id
        self.name = name
        self.status = "failed"
        self.fail_reason = reason
        self.step_index = step_index
        self.n_dofs = 0
        self.x = np.zeros(0)


def _run_trial_worker(args):
    fn, env, payload = args
    return fn(env, payload)


def run_batch_trials(trial_fn, envs_payloads, max_workers=0, chunksize=1):
    """One trial per (env, payload), results in input order (multienv.py:204-216).

    The reference forks a process pool (max_workers) around an arbitrary Python trial function.
    A CUDA context does not survive fork, so this generic form runs the trials in-process, one
    after another, and ignores max_workers / chunksize.  The batched device path for grasp
    trials is ``runner.TrialRunner`` (many trials per device batch, continuous refill) or
    ``protocol.run_grasp_trials`` / ``protocol.DeviceProtocolTrials`` on a fixed set of envs.
    """
    return [_run_trial_worker((trial_fn, env, payload)) for env, payload in envs_payloads]
