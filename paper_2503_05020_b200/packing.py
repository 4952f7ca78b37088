"""Flatten N environments into the SoA arrays of GripSceneDesc (include/grip_ipc.h).

Per env this restates the reference's DOF/surface layout (solver.py:214-363):
nodes are soft vertices (3 DOFs) and 4 pseudo-nodes (p, A rows) per affine
body, in body order, so ``x.reshape(-1, 3)`` of the reference equals the
node array here; surface vertices are stacked per body (soft: boundary
vertices in boundary order; affine / kinematic: all surface vertices).
All index arrays are env-local; *_off arrays give each env's slice.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2503_05020_b200 import _native as nv
from paper_2503_05020_b200 import geometry as gm
from paper_2503_05020_b200.scene import ContactParams, SolverParams, body_kind


@dataclass
class BodyRecord:
    """Per-body layout, shaped like the reference's env.records entries."""

    body: object
    id: int
    kind: str
    node0: int
    n_node: int
    surf0: int
    n_sv: int
    name: str = ""
    vmap: np.ndarray = None      # soft: tet vertex of each surface vertex
    masses: np.ndarray = None    # soft lumped masses
    xi: np.ndarray = None        # affine: surface vertex offsets from the COM
    mass: float = 0.0
    volume: float = 0.0
    tet0: int = 0
    n_tet: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def dof0(self):
        return 3 * self.node0

    @property
    def ndof(self):
        return 3 * self.n_node


@dataclass
class EnvLayout:
    records: list
    n_node: int
    n_sv: int
    n_tet: int
    n_abd: int
    n_body: int
    free: np.ndarray             # per node
    tets: np.ndarray             # (n_tet, 4) local nodes
    tris: np.ndarray
    edges: np.ndarray
    surf_rest: np.ndarray
    vbody: np.ndarray
    pair_ok: np.ndarray
    x0: np.ndarray               # (n_node, 3)
    kin0: np.ndarray             # (n_sv, 3)


def layout_env(bodies, collide_pairs_off=()):
    """DOF, surface and collision layout of one env (solver.py:214-363)."""
    recs = []
    node0 = surf0 = tet0 = 0
    x0, Mb, free, nbody, nkind, nsv = [], [], [], [], [], []
    svk, svn, svxi, svb, kin0 = [], [], [], [], []
    rest_chunks, tri_chunks, edge_chunks, tets, tet_par = [], [], [], [], []
    abd = []
    nb = len(bodies)
    kin = np.zeros(nb, bool)
    for bid, body in enumerate(bodies):
        kind = body_kind(body)
        if kind == "soft":
            mesh = body.mesh
            rest = np.asarray(mesh.rest_vertices, np.float64)
            T = np.asarray(mesh.tets, np.int64)
            nv_ = len(rest)
            if hasattr(mesh, "boundary_surface"):
                surf, vmap = mesh.boundary_surface()
                stris = np.asarray(surf.triangles, np.int64)
                sedges = np.asarray(surf.edges(), np.int64)
            else:  # pragma: no cover - duck-typed meshes always provide it
                raise TypeError("soft body mesh must provide boundary_surface()")
            masses = np.zeros(nv_)
            np.add.at(masses, T.reshape(-1), np.repeat(body.material.density * gm.tet_volumes(rest, T) / 4.0, 4))
            rec = BodyRecord(body, bid, kind, node0, nv_, surf0, len(vmap), getattr(body, "name", ""), vmap=vmap,
                             masses=masses, tet0=tet0, n_tet=len(T))
            x0.append(np.asarray(mesh.vertices, np.float64).reshape(-1, 3))
            Mb.append(masses[:, None, None] * np.eye(3)[None])
            kmask = np.asarray(getattr(body, "kinematic_mask", np.zeros(nv_, bool)), bool)
            free.append(~kmask)
            nbody += [bid] * nv_
            nkind += [0] * nv_
            node_sv = np.full(nv_, -1, np.int64)
            node_sv[vmap] = surf0 + np.arange(len(vmap))
            nsv.append(node_sv)
            svk += [0] * len(vmap)
            svn.append(node0 + vmap)
            svxi.append(np.zeros((len(vmap), 3)))
            svb += [bid] * len(vmap)
            kin0.append(np.zeros((len(vmap), 3)))
            rest_chunks.append(rest[vmap])
            tri_chunks.append(stris + surf0)
            edge_chunks.append(sedges + surf0)
            tets.append(T + node0)
            mu, lam = body.material.lame()
            tet_par.append((T, rest, mu, lam))
            node0 += nv_
            surf0 += len(vmap)
            tet0 += len(T)
        elif kind == "affine":
            v = np.asarray(body.surface.vertices, np.float64)
            tr = np.asarray(body.surface.triangles, np.int64)
            mass, com, second = gm.surface_mass_properties(body.surface, body.material.density)
            xi = v - com
            vol = body.surface.enclosed_volume()
            rec = BodyRecord(body, bid, kind, node0, 4, surf0, len(xi), getattr(body, "name", ""), xi=xi, mass=mass,
                             volume=vol)
            rec.extra["second"] = second
            x0.append(np.concatenate([com[None], np.eye(3)]))
            Mb.append(np.stack([mass * np.eye(3), second, second, second]))
            free.append(np.ones(4, bool))
            nbody += [bid] * 4
            nkind += [1, 2, 2, 2]
            nsv.append(np.full(4, -1, np.int64))
            svk += [1] * len(xi)
            svn.append(np.full(len(xi), node0, np.int64))
            svxi.append(xi)
            svb += [bid] * len(xi)
            kin0.append(np.zeros((len(xi), 3)))
            rest_chunks.append(xi)
            tri_chunks.append(tr + surf0)
            edge_chunks.append(np.asarray(body.surface.edges(), np.int64) + surf0)
            abd.append((node0, float(getattr(body, "kappa", 1e8)) * vol, bid))
            node0 += 4
            surf0 += len(xi)
        elif kind == "kinematic":
            v = np.asarray(body.surface.vertices, np.float64)
            tr = np.asarray(body.surface.triangles, np.int64)
            rest = np.asarray(getattr(body.surface, "rest_vertices", v), np.float64)
            rec = BodyRecord(body, bid, kind, node0, 0, surf0, len(v), getattr(body, "name", ""))
            kin[bid] = True
            svk += [2] * len(v)
            svn.append(np.full(len(v), -1, np.int64))
            svxi.append(np.zeros((len(v), 3)))
            svb += [bid] * len(v)
            kin0.append(v.copy())
            rest_chunks.append(rest)
            tri_chunks.append(tr + surf0)
            edge_chunks.append(np.asarray(body.surface.edges(), np.int64) + surf0)
            surf0 += len(v)
        else:
            raise TypeError(f"unknown body kind {kind}")
        recs.append(rec)
    collide = np.ones((nb, nb), bool)
    for bid, body in enumerate(bodies):
        collide[bid, bid] = bool(getattr(body, "collide_self", False))
    for a, b in collide_pairs_off:
        collide[a, b] = collide[b, a] = False
    pair_ok = collide & ~(kin[:, None] & kin[None, :])
    rest = np.concatenate(rest_chunks)
    edges = np.concatenate(edge_chunks)
    lay = EnvLayout(recs, node0, surf0, tet0, len(abd), nb,
                    np.concatenate(free) if free else np.zeros(0, bool),
                    np.concatenate(tets) if tets else np.zeros((0, 4), np.int64),
                    np.concatenate(tri_chunks), edges, rest, np.asarray(svb, np.int64), pair_ok,
                    np.concatenate(x0) if x0 else np.zeros((0, 3)), np.concatenate(kin0))
    tri_n = [len(t) for t in tri_chunks]
    edge_n = [len(e) for e in edge_chunks]
    lay.body_tri = np.stack([np.cumsum([0] + tri_n)[:-1], np.cumsum(tri_n)], 1)
    lay.body_edge = np.stack([np.cumsum([0] + edge_n)[:-1], np.cumsum(edge_n)], 1)
    lay._arrays = dict(Mb=np.concatenate(Mb) if Mb else np.zeros((0, 3, 3)), nbody=np.asarray(nbody, np.int64),
                       nkind=np.asarray(nkind, np.int64), nsv=np.concatenate(nsv) if nsv else np.zeros(0, np.int64),
                       svk=np.asarray(svk, np.int64), svn=np.concatenate(svn), svxi=np.concatenate(svxi),
                       tet_par=tet_par, abd=abd)
    return lay


def env_params(contact: ContactParams, solver: SolverParams):
    p = np.zeros(nv.NPARAM)
    p[nv.P_DT] = solver.dt
    p[nv.P_KAPPA] = contact.kappa
    p[nv.P_DHAT] = contact.dhat
    p[nv.P_EPSV] = contact.eps_v
    p[nv.P_RELTOL] = solver.rel_tol
    p[nv.P_MAXIT] = solver.max_iters
    p[nv.P_ELLFLOOR] = solver.length_scale_floor
    p[nv.P_MAXLS] = solver.max_line_search
    p[nv.P_CCDSCALE] = solver.ccd_scaling
    p[nv.P_CCDIT] = solver.ccd_max_iters
    p[nv.P_KINGUARD] = solver.kinematic_ccd_guard
    p[nv.P_MURULE] = 0.0 if contact.friction_combination == "geometric" else 1.0
    p[nv.P_PCGRTOL] = getattr(solver, "pcg_rtol", 1e-13)
    return p


class Packed:
    """All envs flattened; attribute names match GripSceneDesc fields."""

    def __init__(self, layouts, params, gravity, body_vel):
        E = len(layouts)
        self.n_env = E
        self.layouts = layouts
        off = lambda k: np.concatenate([[0], np.cumsum([k(l) for l in layouts])]).astype(np.int32)  # noqa: E731
        self.node_off = off(lambda l: l.n_node)
        self.sv_off = off(lambda l: l.n_sv)
        self.tri_off = off(lambda l: len(l.tris))
        self.edge_off = off(lambda l: len(l.edges))
        self.tet_off = off(lambda l: l.n_tet)
        self.abd_off = off(lambda l: l.n_abd)
        self.body_off = off(lambda l: l.n_body)
        self.n_node_total = int(self.node_off[-1])
        self.n_sv_total = int(self.sv_off[-1])
        self.n_tet_total = int(self.tet_off[-1])
        self.n_body_total = int(self.body_off[-1])
        cat = lambda f, dt: (np.concatenate([f(l) for l in layouts]).astype(dt) if E else np.zeros(0, dt))  # noqa: E731
        self.node_x0 = cat(lambda l: l.x0, np.float64).reshape(-1)
        self.node_M = cat(lambda l: l._arrays["Mb"].reshape(-1, 9), np.float64).reshape(-1)
        self.node_free = cat(lambda l: l.free, np.uint8)
        self.node_body = cat(lambda l: l._arrays["nbody"], np.int32)
        self.node_kind = cat(lambda l: l._arrays["nkind"], np.uint8)
        self.node_sv = cat(lambda l: l._arrays["nsv"], np.int32)
        self.sv_kind = cat(lambda l: l._arrays["svk"], np.uint8)
        self.sv_node = cat(lambda l: l._arrays["svn"], np.int32)
        self.sv_xi = cat(lambda l: l._arrays["svxi"], np.float64).reshape(-1)
        self.sv_body = cat(lambda l: l.vbody, np.int32)
        self.sv_kin0 = cat(lambda l: l.kin0, np.float64).reshape(-1)
        self.tris = cat(lambda l: l.tris, np.int32).reshape(-1)
        self.edges = cat(lambda l: l.edges, np.int32).reshape(-1)
        self.edge_rest_sq = cat(lambda l: np.einsum("ij,ij->i", l.surf_rest[l.edges[:, 1]] - l.surf_rest[l.edges[:, 0]],
                                                    l.surf_rest[l.edges[:, 1]] - l.surf_rest[l.edges[:, 0]]), np.float64)
        tn, dmi, v0, tmu, tlam = [], [], [], [], []
        for l in layouts:
            for (T, rest, mu, lam) in l._arrays["tet_par"]:
                Dm = np.stack([rest[T[:, k + 1]] - rest[T[:, 0]] for k in range(3)], axis=-1)
                V0 = np.linalg.det(Dm) / 6.0
                if np.any(V0 <= 0.0):
                    raise ValueError("non-positive rest volume")
                dmi.append(np.linalg.inv(Dm).reshape(-1, 9))
                v0.append(V0)
                tmu.append(np.full(len(T), mu))
                tlam.append(np.full(len(T), lam))
            tn.append(l.tets)
        self.tet_nodes = (np.concatenate(tn) if tn else np.zeros((0, 4))).astype(np.int32).reshape(-1)
        self.tet_Dmi = (np.concatenate(dmi) if dmi else np.zeros((0, 9))).reshape(-1)
        self.tet_V0 = np.concatenate(v0) if v0 else np.zeros(0)
        self.tet_mu = np.concatenate(tmu) if tmu else np.zeros(0)
        self.tet_lam = np.concatenate(tlam) if tlam else np.zeros(0)
        self.abd_node = cat(lambda l: np.array([a[0] for a in l._arrays["abd"]], np.int64), np.int32)
        self.abd_kV = cat(lambda l: np.array([a[1] for a in l._arrays["abd"]], np.float64), np.float64)
        self.abd_body = cat(lambda l: np.array([a[2] for a in l._arrays["abd"]], np.int64), np.int32)
        self.body_kind = cat(lambda l: np.array([{"soft": 0, "affine": 1, "kinematic": 2}[r.kind] for r in l.records]),
                             np.uint8)
        self.body_mu = cat(lambda l: np.array([r.body.material.friction_coefficient for r in l.records]), np.float64)
        self.body_pairmask = cat(lambda l: np.array([sum(1 << j for j in range(l.n_body) if l.pair_ok[i, j])
                                                     for i in range(l.n_body)], np.int64), np.uint32)
        if np.any(self.body_off[1:] - self.body_off[:-1] > 32):
            raise ValueError("at most 32 bodies per environment")
        self.body_vel0 = np.asarray(body_vel, np.float64).reshape(-1)
        self.body_tri_lo = cat(lambda l: l.body_tri[:, 0], np.int32)
        self.body_tri_hi = cat(lambda l: l.body_tri[:, 1], np.int32)
        self.body_edge_lo = cat(lambda l: l.body_edge[:, 0], np.int32)
        self.body_edge_hi = cat(lambda l: l.body_edge[:, 1], np.int32)
        self.env_params = np.asarray(params, np.float64).reshape(E, nv.NPARAM)
        self.env_gravity = np.asarray(gravity, np.float64).reshape(-1)
        hint = []
        for l in layouts:
            tv = l.surf_rest[l.tris] if len(l.tris) else np.zeros((1, 3, 3))
            hint.append(float(np.median((tv.max(axis=1) - tv.min(axis=1)).max(axis=1))))
        self.env_cell_hint = np.asarray(hint, np.float64)


def body_velocities(bodies):
    out = np.zeros((len(bodies), 3))
    for i, b in enumerate(bodies):
        v = getattr(b, "velocity", None)
        if v is not None:
            out[i] = np.asarray(v, np.float64).reshape(3)
    return out
