"""Drop-in ``Environment`` with the reference's constructor and stepping API.

Mirrors gripsim.solver (solver.py:37-773): ``Environment(bodies, gravity,
contact_params, solver_params, name, env_id, collide_pairs_off)`` with
``begin_step`` / ``newton_iteration`` / ``finalize_step`` / ``step`` and the
state queries the protocol and metrics use.  State lives on the GPU in a
``DeviceBatch`` (the C ABI of include/grip_ipc.h); an Environment is either
standalone (its own one-env batch, created on first use) or a slot of a
``multienv.Batch``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2503_05020_b200 import _native as nv
from paper_2503_05020_b200 import packing
from paper_2503_05020_b200.scene import (  # noqa: F401  (re-exported like the reference)
    AffineBody,
    ContactParams,
    KinematicBody,
    MaterialParams,
    SoftBody,
    SolverParams,
)


@dataclass
class StepReport:
    """Outcome of one implicit time step of one environment (solver.py:59-84)."""

    status: str
    iterations: int
    residual: float
    alpha_history: list
    min_distance: float
    energy: float
    kinematic_blocked: bool = False
    regularized: bool = False
    reason: str = ""
    env_id: int = 0
    step_index: int = 0
    time: float = 0.0
    newton_calls: int = 0
    pcg_iterations: int = 0

    def to_dict(self):
        return {
            "env": self.env_id, "step": self.step_index, "t": self.time,
            "status": self.status, "iterations": self.iterations,
            "residual": self.residual, "alphas": list(self.alpha_history),
            "min_distance": self.min_distance, "energy": self.energy,
            "kinematic_blocked": self.kinematic_blocked,
            "regularized": self.regularized, "reason": self.reason,
        }


class NewtonState:
    """Host view of one env's device Newton state (solver.py:180-192)."""

    def __init__(self):
        self.done = False
        self.status = "running"
        self.iterations = 0
        self.reason = ""


def report_from_row(row, alphas, env_id):
    st = int(row["status"])
    status = {nv.NS_CONVERGED: "converged", nv.NS_FAILED: "failed"}.get(st, "running")
    n = int(row["n_alphas"])
    en = float(row["energy"])
    return StepReport(status=status, iterations=int(row["iterations"]), residual=float(row["residual"]),
                      alpha_history=[float(a) for a in alphas[:n]], min_distance=float(row["min_distance"]),
                      energy=en if np.isfinite(en) else float("inf"), kinematic_blocked=bool(row["kinematic_blocked"]),
                      regularized=bool(row["regularized"]), reason=nv.REASONS.get(int(row["reason"]), "unknown"),
                      env_id=env_id, step_index=int(row["step_index"]), time=float(row["time"]) - 0.0,
                      newton_calls=int(row["newton_calls"]), pcg_iterations=int(row["pcg_iters"]))


class _Record(dict):
    """env.records[b] entry; "positions" of kinematic bodies is read from the device."""

    def __init__(self, env, rec):
        super().__init__()
        self._env = env
        self._rec = rec
        self.update({"body": rec.body, "id": rec.id, "kind": rec.kind, "dof0": rec.dof0, "surf0": rec.surf0,
                     "name": rec.name, "ndof": 12 if rec.kind == "affine" else rec.ndof, "n_sv": rec.n_sv})
        if rec.kind == "soft":
            self["masses"] = rec.masses
            self["surf_map"] = rec.vmap
        if rec.kind == "affine":
            self["xi"] = rec.xi
            self["mass"] = rec.mass
            self["volume"] = rec.volume

    def __getitem__(self, k):
        if k == "positions" and self._rec.kind == "kinematic":
            return self._env._kin_positions(self._rec)
        return super().__getitem__(k)

    def get(self, k, default=None):
        if k == "positions" and self._rec.kind == "kinematic":
            return self._env._kin_positions(self._rec)
        return super().get(k, default)


class Environment:
    """One independent scene (solver.py:195-773), stepped on the GPU."""

    def __init__(self, bodies, gravity=(0.0, 0.0, 0.0), contact_params=None, solver_params=None, name="env",
                 env_id=0, collide_pairs_off=()):
        self.bodies = list(bodies)
        self._gravity = np.asarray(gravity, np.float64).reshape(3)
        self.contact_params = contact_params or ContactParams()
        self.solver_params = solver_params or SolverParams()
        self.name = name
        self.env_id = env_id
        self.status = "active"
        self.fail_reason = ""
        self.collide_pairs_off = list(collide_pairs_off)
        self.layout = packing.layout_env(self.bodies, self.collide_pairs_off)
        self.records = [_Record(self, r) for r in self.layout.records]
        self.n_dofs = 3 * self.layout.n_node
        self.n_sv = self.layout.n_sv
        self._batch = None      # multienv.Batch or _Solo
        self._slot = 0
        self._time = 0.0
        self._step = 0

    # -- device attachment ------------------------------------------------------
    def _owner(self):
        if self._batch is None:
            self._batch = _Solo(self)
        return self._batch

    @property
    def time(self):
        return self._time

    @property
    def step_index(self):
        return self._step

    @property
    def gravity(self):
        return self._gravity

    @gravity.setter
    def gravity(self, g):
        self._gravity = np.asarray(g, np.float64).reshape(3)

    def params_row(self):
        return packing.env_params(self.contact_params, self.solver_params)

    # -- state access (solver.py:367-481) -----------------------------------------
    @property
    def x(self):
        if self._batch is None:
            return self.layout.x0.reshape(-1).copy()
        return self._batch._node_slice(self._slot, "x").reshape(-1).copy()

    @x.setter
    def x(self, val):
        self._owner()._set_node_slice(self._slot, "x", np.asarray(val, np.float64).reshape(-1, 3))

    @property
    def v(self):
        if self._batch is None:
            return np.zeros(self.n_dofs)
        return self._batch._node_slice(self._slot, "v").reshape(-1).copy()

    @v.setter
    def v(self, val):
        self._owner()._set_node_slice(self._slot, "v", np.asarray(val, np.float64).reshape(-1, 3))

    def _kin_positions(self, rec):
        if self._batch is None:
            return self.layout.kin0[rec.surf0:rec.surf0 + rec.n_sv].copy()
        return self._batch._sv_slice(self._slot, "kin")[rec.surf0:rec.surf0 + rec.n_sv].copy()

    def node_positions(self, x=None):
        return (self.x if x is None else np.asarray(x)).reshape(-1, 3)

    def surface_positions(self, x=None):
        if x is not None:
            return self._surface_host(np.asarray(x, np.float64).reshape(-1, 3))
        return self._owner()._surface(self._slot)

    def _surface_host(self, nodes):
        lay = self.layout
        out = np.zeros((lay.n_sv, 3))
        kin = None
        for r in lay.records:
            sl = slice(r.surf0, r.surf0 + r.n_sv)
            if r.kind == "soft":
                out[sl] = nodes[r.node0 + r.vmap]
            elif r.kind == "affine":
                q = nodes[r.node0:r.node0 + 4]
                out[sl] = q[0][None] + r.xi @ q[1:4].T
            else:
                kin = self._kin_positions(r) if kin is None else kin
                out[sl] = self._kin_positions(r)
        return out

    def bbox_diagonal(self):
        sv = self.surface_positions()
        return float(np.linalg.norm(sv.max(axis=0) - sv.min(axis=0))) if len(sv) else 0.0

    def body_com(self, bid):
        r = self.layout.records[bid]
        nodes = self.node_positions()
        if r.kind == "soft":
            xs = nodes[r.node0:r.node0 + r.n_node]
            return (r.masses[:, None] * xs).sum(axis=0) / r.masses.sum()
        if r.kind == "affine":
            return nodes[r.node0].copy()
        return self._kin_positions(r).mean(axis=0)

    def body_velocity_com(self, bid):
        r = self.layout.records[bid]
        vs = self.v.reshape(-1, 3)
        if r.kind == "soft":
            xs = vs[r.node0:r.node0 + r.n_node]
            return (r.masses[:, None] * xs).sum(axis=0) / r.masses.sum()
        if r.kind == "affine":
            return vs[r.node0].copy()
        return np.asarray(r.body.velocity, np.float64).copy()

    def total_linear_momentum(self):
        vs = self.v.reshape(-1, 3)
        mom = np.zeros(3)
        for r in self.layout.records:
            if r.kind == "soft":
                mom += (r.masses[:, None] * vs[r.node0:r.node0 + r.n_node]).sum(axis=0)
            elif r.kind == "affine":
                mom += r.mass * vs[r.node0]
        return mom

    def max_point_speed(self):
        """Max surface-vertex speed, prescribed bodies included (solver.py:414-428)."""
        vs = self.v.reshape(-1, 3)
        sp = [0.0]
        for r in self.layout.records:
            if r.kind == "soft":
                sp.append(float(np.linalg.norm(vs[r.node0:r.node0 + r.n_node], axis=1).max()))
            elif r.kind == "affine":
                q = vs[r.node0:r.node0 + 4]
                sp.append(float(np.linalg.norm(q[0][None] + r.xi @ q[1:4].T, axis=1).max()))
            else:
                sp.append(float(np.linalg.norm(r.body.velocity)))
        return max(sp)

    def min_tet_volume(self):
        nodes = self.node_positions()
        vols = [np.inf]
        T = self.layout.tets
        if len(T):
            d1, d2, d3 = (nodes[T[:, k]] - nodes[T[:, 0]] for k in (1, 2, 3))
            vols.append(float((np.einsum("ij,ij->i", np.cross(d1, d2), d3) / 6.0).min()))
        for r in self.layout.records:
            if r.kind == "affine":
                vols.append(float(np.linalg.det(nodes[r.node0 + 1:r.node0 + 4])))
        return min(vols)

    def candidates(self, radius):
        """Canonical candidate stencils at `radius` (broadphase.py:101-214), env-local sv ids."""
        return self._owner()._candidates(self._slot, radius)

    def contact_forces(self):
        """Per-body summed barrier force of the active stencils at the current state."""
        return self._owner()._contacts(self._slot)

    def min_contact_distance(self, radius_factor=2.0):
        """solver.py:449-453: min stencil distance of the candidate set at radius_factor * dhat
        (computed on the device, grip_contacts_now)."""
        return self._owner()._events_now(self._slot, radius_factor)[1]

    def stress_rows(self):
        return self._owner()._stress(self._slot)

    # -- stepping (solver.py:590-773) ---------------------------------------------------
    def begin_step(self):
        self._owner()._begin([self._slot])
        return NewtonState()

    def newton_iteration(self, ns):
        done = self._owner()._iterate([self._slot])
        ns.done = bool(done[self._slot])
        return ns

    def finalize_step(self, ns):
        rep = self._owner()._finalize([self._slot])[self._slot]
        ns.status = rep.status
        return rep

    def newton_step(self):
        if self.status != "active":
            raise RuntimeError(f"stepping a {self.status} environment")
        return self._owner()._step([self._slot])[self._slot]

    step = newton_step


class _Solo:
    """A one-env device batch owned by a standalone Environment."""

    def __new__(cls, env):
        from paper_2503_05020_b200.multienv import DeviceEnvGroup
        return DeviceEnvGroup([env])
