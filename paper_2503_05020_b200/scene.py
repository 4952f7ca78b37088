"""Scene description: materials, bodies, parameters and grasp-trial construction.

Mirrors the reference's constructor surface so a reference user can switch
(gripsim/solver.py:37-177, contact.py:34-46, materials.py:20-49,
pipeline/config.py:56-110,230-308, synth.py:143-207).  Objects from the
reference (its TetMesh / TriSurface / bodies) are accepted as-is by
``Environment`` because everything here is duck-typed on the same attributes.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from paper_2503_05020_b200 import geometry as gm


@dataclass
class MaterialParams:
    """E (Pa), nu, rho (kg/m^3), friction coefficient (materials.py:20-40)."""

    young_modulus: float = 1e5
    poisson_ratio: float = 0.3
    density: float = 1000.0
    friction_coefficient: float = 0.5

    def __post_init__(self):
        if self.young_modulus <= 0.0:
            raise ValueError("young_modulus must be > 0")
        if not (0.0 <= self.poisson_ratio < 0.5):
            raise ValueError("poisson_ratio must be in [0, 0.5)")
        if self.density <= 0.0:
            raise ValueError("density must be > 0")
        if self.friction_coefficient < 0.0:
            raise ValueError("friction_coefficient must be >= 0")

    def lame(self):
        return lame_from_young_poisson(self.young_modulus, self.poisson_ratio)


def lame_from_young_poisson(E, nu):
    """(mu, lambda); materials.py:43-49."""
    if nu >= 0.5:
        raise ValueError("poisson_ratio must be < 0.5")
    return E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))


@dataclass
class ContactParams:
    """kappa, dhat (m), eps_v (m/s), friction rule (contact.py:34-46)."""

    kappa: float = 3e6
    dhat: float = 1e-3
    eps_v: float = 1e-3
    friction_combination: str = "geometric"
    friction_iterations: int = 1

    def __post_init__(self):
        if self.kappa <= 0.0 or self.dhat <= 0.0 or self.eps_v <= 0.0:
            raise ValueError("kappa, dhat, eps_v must all be positive")
        if self.friction_combination not in ("geometric", "min"):
            raise ValueError(f"unknown friction combination rule: {self.friction_combination}")


@dataclass
class SolverParams:
    """Time step, Newton tolerances, line-search/CCD knobs (solver.py:37-56).

    ``linear_solver`` is accepted for API compatibility; the device path
    always uses block-Jacobi PCG at ``pcg_rtol`` on the relative residual: 1e-13
    keeps long soft-body Newton solves on the reference's direct-solve path
    (measured: 1e-9 flips line-search halvings within 10 steps, 1e-11 drifts to
    2e-7 ell per step, 1e-13 stays below 2e-9 ell; SURVEY §7 hard part 1).
    """

    dt: float = 0.01
    rel_tol: float = 1e-3
    max_iters: int = 100
    fp_precision: str = "fp64"
    linear_solver: str = "direct"
    length_scale_floor: float = 0.05
    max_line_search: int = 50
    ccd_scaling: float = 0.9
    ccd_max_iters: int = 32
    kinematic_ccd_guard: float = 0.1
    pcg_rtol: float = 1e-13

    def __post_init__(self):
        if self.dt <= 0.0 or self.rel_tol <= 0.0 or self.max_iters < 1:
            raise ValueError("invalid solver parameters")
        if self.fp_precision != "fp64":
            raise ValueError("only fp64 is supported")


def _vec3(v):
    return np.asarray(v, np.float64).reshape(3)


@dataclass
class SoftBody:
    """FEM body; kinematic_mask marks prescribed vertices driven at velocity (solver.py:139-154)."""

    mesh: object
    material: MaterialParams
    name: str = "soft"
    kinematic_mask: np.ndarray = None
    velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    collide_self: bool = False
    kind = "soft"

    def __post_init__(self):
        if self.kinematic_mask is None:
            self.kinematic_mask = np.zeros(self.mesh.n_vertices, bool)
        self.kinematic_mask = np.asarray(self.kinematic_mask, bool)
        self.velocity = _vec3(self.velocity)


@dataclass
class AffineBody:
    """Rigid body as a 12-DOF affine map of its surface (solver.py:157-164)."""

    surface: object
    material: MaterialParams
    name: str = "rigid"
    kappa: float = 1e8
    kind = "affine"


@dataclass
class KinematicBody:
    """Scripted collider without DOFs (solver.py:167-177)."""

    surface: object
    material: MaterialParams
    name: str = "kinematic"
    velocity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    kind = "kinematic"

    def __post_init__(self):
        self.velocity = _vec3(self.velocity)


def body_kind(body):
    k = getattr(body, "kind", None)
    if isinstance(k, str):
        return k
    return {"SoftBody": "soft", "AffineBody": "affine", "KinematicBody": "kinematic"}[type(body).__name__]


# ---------------------------------------------------------------------------
# parallel gripper and grasp-trial scenes (synth.py:143-207, config.py:56-110,230-308)
# ---------------------------------------------------------------------------


@dataclass
class ParallelGripper:
    max_opening: float = 0.08
    finger_length: float = 0.05
    finger_width: float = 0.02
    finger_thickness: float = 0.01
    palm_thickness: float = 0.015
    finger_subdiv: int = 2

    def finger_center(self, side, opening):
        s = -1.0 if side == 0 else 1.0
        return np.array([s * (opening / 2.0 + self.finger_thickness / 2.0), 0.0, self.finger_length / 2.0])

    def body_meshes(self, opening):
        dims = (self.finger_thickness, self.finger_width, self.finger_length)
        f0 = gm.box_surface(dims, center=self.finger_center(0, opening), subdivisions=self.finger_subdiv)
        f1 = gm.box_surface(dims, center=self.finger_center(1, opening), subdivisions=self.finger_subdiv)
        palm = gm.box_surface((opening + 2.0 * self.finger_thickness, self.finger_width, self.palm_thickness),
                              center=(0.0, 0.0, self.finger_length + self.palm_thickness / 2.0),
                              subdivisions=self.finger_subdiv)
        return f0, f1, palm


OBJECT_MATERIAL = dict(young_modulus=1e5, poisson_ratio=0.4, density=500.0, friction_coefficient=0.5)
PAD_MATERIAL = dict(young_modulus=9.4e6, poisson_ratio=0.3, density=1000.0, friction_coefficient=3.5)


@dataclass
class ObjectSpec:
    """box | sphere | cylinder, rigid (ABD) or soft (config.py:56-100; cylinder per SURVEY §8d-2)."""

    kind: str = "box"
    soft: bool = False
    size: float = 0.05
    resolution: int = 3
    material: MaterialParams = field(default_factory=lambda: MaterialParams(**OBJECT_MATERIAL))
    cylinder: tuple = (0.02, 0.05, 20)

    def surface(self):
        s = self.size
        if self.kind == "box":
            return gm.box_surface(s, subdivisions=max(2, self.resolution))
        if self.kind == "sphere":
            return gm.icosphere(s / 2.0, level=3)
        if self.kind == "cylinder":
            r, h, seg = self.cylinder
            return gm.cylinder_surface(r, h, int(seg))
        raise ValueError(f"unknown object kind {self.kind!r}")

    def build_body(self):
        s = self.size
        if self.soft:
            if self.kind == "box":
                mesh = gm.box_tet_lattice(s, self.resolution)
            elif self.kind == "sphere":
                mesh = gm.sphere_tet_lattice(s / 2.0, max(4, 2 * self.resolution))
            else:
                raise ValueError(f"soft {self.kind} is not supported")
            return SoftBody(mesh, self.material, name="object")
        return AffineBody(self.surface(), self.material, name="object")


@dataclass
class GripperSpec:
    soft_fingers: bool = True
    gripper: ParallelGripper = field(default_factory=ParallelGripper)
    pad_material: MaterialParams = field(default_factory=lambda: MaterialParams(**PAD_MATERIAL))
    pad_resolution: int = 2
    palm_gap: float = 2e-3


def soft_finger_body(gspec, side, opening):
    """Soft pad glued to the jaw by its outer face (config.py:230-238)."""
    g = gspec.gripper
    res = (gspec.pad_resolution, gspec.pad_resolution, 2 * gspec.pad_resolution)
    c = g.finger_center(side, opening)
    mesh = gm.box_tet_lattice((g.finger_thickness, g.finger_width, g.finger_length), res, center=c)
    outer_x = c[0] + (0.5 if side == 1 else -0.5) * g.finger_thickness
    mask = np.isclose(mesh.rest_vertices[:, 0], outer_x, atol=1e-9)
    return SoftBody(mesh, gspec.pad_material, name=f"finger{side}", kinematic_mask=mask)


@dataclass
class GraspScene:
    """Bodies plus the wiring a grasp trial needs (what config.build_trial_env returns)."""

    bodies: list
    collide_pairs_off: list
    object_body: int
    finger_links: dict
    closing_dirs: dict
    opening: float


def build_trial_scene(obj: ObjectSpec, gspec: GripperSpec, R, T, opening):
    """Object + posed gripper for one candidate (config.py:241-308)."""
    R = np.asarray(R, np.float64).reshape(3, 3)
    T = np.asarray(T, np.float64).reshape(3)
    g = gspec.gripper
    bodies = [obj.build_body()]
    links = {}
    f0s, f1s, palm_s = g.body_meshes(opening)
    palm_s = gm.TriSurface(palm_s.vertices + np.array([0.0, 0.0, gspec.palm_gap]), palm_s.triangles)
    if gspec.soft_fingers:
        for side in (0, 1):
            b = soft_finger_body(gspec, side, opening)
            b.mesh.vertices[:] = b.mesh.vertices @ R.T + T
            b.mesh.rest_vertices[:] = b.mesh.vertices
            bodies.append(b)
            links[f"finger{side}"] = (len(bodies) - 1,)
        for side in (0, 1):
            bodies[1 + side].mesh.refresh()
    else:
        for side, s in ((0, f0s), (1, f1s)):
            bodies.append(KinematicBody(s.transformed(rotation=R, translation=T),
                                        MaterialParams(1e9, 0.3, 2000.0, gspec.pad_material.friction_coefficient),
                                        name=f"finger{side}"))
            links[f"finger{side}"] = (len(bodies) - 1,)
    bodies.append(KinematicBody(palm_s.transformed(rotation=R, translation=T),
                                MaterialParams(1e9, 0.3, 2000.0, 0.3), name="palm"))
    palm = len(bodies) - 1
    off = [(links[f"finger{s}"][0], palm) for s in (0, 1)]
    axis = R @ np.array([1.0, 0.0, 0.0])
    dirs = {"finger0": axis, "finger1": -axis}
    return GraspScene(bodies, off, 0, links, dirs, float(opening))


# ---------------------------------------------------------------------------
# config-2 bench scenes: 400 envs, soft pads on rigid box/cylinder/sphere
# ---------------------------------------------------------------------------

DATA = Path(__file__).resolve().parent / "data"


def load_cfg2_candidates():
    """Antipodal candidates (seed i, kind [box, cylinder, sphere][i % 3]) precomputed by the
    reference's sampler (synth.py:227) in tests/golden/make_golden.py."""
    d = np.load(DATA / "cfg2_candidates.npz")
    return {k: d[k] for k in d.files}


def cfg2_scene(i, cands=None):
    """Environment i of BASELINE config 2."""
    c = cands if cands is not None else load_cfg2_candidates()
    kinds = [str(k) for k in c["kinds"]]
    kind = kinds[int(c["kind"][i])]
    r, h, seg = c["cyl"]
    obj = ObjectSpec(kind=kind, cylinder=(float(r), float(h), int(seg)))
    return build_trial_scene(obj, GripperSpec(soft_fingers=True), c["R"][i], c["T"][i], float(c["opening"][i]))


def load_cfg3_candidates():
    """Config 3: antipodal candidates on the soft box / sphere (kind i % 2, seed i)
    and each trial's randomized object material (E, mu; config.py:311-318 with the pipeline's
    seeding seed + 7919 i, pipeline/__init__.py:29), precomputed by the reference in
    tests/golden/make_golden.py."""
    d = np.load(DATA / "cfg3_candidates.npz")
    return {k: d[k] for k in d.files}


def cfg3_scene(i, cands=None):
    """Environment i of BASELINE config 3: soft Neo-Hookean object, kinematic ("rigid") fingers."""
    c = cands if cands is not None else load_cfg3_candidates()
    kind = [str(k) for k in c["kinds"]][int(c["kind"][i])]
    mat = MaterialParams(young_modulus=float(c["E"][i]), poisson_ratio=float(c["nu"][i]), density=float(c["rho"][i]),
                         friction_coefficient=float(c["mu"][i]))
    return build_trial_scene(ObjectSpec(kind=kind, soft=True, material=mat), GripperSpec(soft_fingers=False),
                             c["R"][i], c["T"][i], float(c["opening"][i]))


def soft_object_scene(R, T, opening, kind="box"):
    """Config 3 in the form the reference can express: soft NH object, kinematic fingers."""
    return build_trial_scene(ObjectSpec(kind=kind, soft=True), GripperSpec(soft_fingers=False), R, T, opening)


def bimanual_scene(yaw=0.0):
    """Config 4: two top-down soft-pad grippers (offset +-12.5 mm in y) on one soft cube.  yaw
    rotates the grippers about the vertical axis through the cube (bench envs get distinct poses;
    yaw=0 is the reference scene of tests/golden/traj_bimanual.npz)."""
    obj = ObjectSpec(kind="box", soft=True)
    gs = GripperSpec(soft_fingers=True)
    g = gs.gripper
    opening = 0.05 + 2 * 2e-3
    c, s_ = np.cos(yaw), np.sin(yaw)
    Rz = np.array([[c, -s_, 0.0], [s_, c, 0.0], [0.0, 0.0, 1.0]])
    bodies = [obj.build_body()]
    links, dirs, off = {}, {}, []
    for gi, yoff in enumerate((-0.0125, 0.0125)):
        T = np.array([0.0, yoff, -0.01])
        pads = []
        for side in (0, 1):
            b = soft_finger_body(gs, side, opening)
            b.mesh.vertices[:] = b.mesh.vertices + T
            if yaw:
                b.mesh.vertices[:] = b.mesh.vertices @ Rz.T
            b.mesh.rest_vertices[:] = b.mesh.vertices
            b.mesh.refresh()
            b.name = f"g{gi}finger{side}"
            bodies.append(b)
            pads.append(len(bodies) - 1)
            links[b.name] = (len(bodies) - 1,)
            dirs[b.name] = Rz @ (np.array([1.0, 0.0, 0.0]) if side == 0 else np.array([-1.0, 0.0, 0.0]))
        _, _, palm_s = g.body_meshes(opening)
        pv = palm_s.vertices + np.array([0.0, 0.0, gs.palm_gap]) + T
        palm_s = gm.TriSurface(pv @ Rz.T if yaw else pv, palm_s.triangles)
        bodies.append(KinematicBody(palm_s, MaterialParams(1e9, 0.3, 2000.0, 0.3), name=f"g{gi}palm"))
        off += [(p, len(bodies) - 1) for p in pads]
    return GraspScene(bodies, off, 0, links, dirs, opening)
