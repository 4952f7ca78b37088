"""Oracle per-environment solver and lockstep batch — TEST INFRASTRUCTURE ONLY.

Restates /root/reference/pkg/src/gripsim/solver.py (Environment build, begin /
newton_iteration / finalize, direct linear solve), multienv.py (Batch
lockstep sweeps with freeze / quarantine) and the per-step parts of
pipeline/protocol.py (contact events, finger force, grasp trial).

Bodies are duck-typed like the reference's: ``SoftBody``-likes expose
``mesh`` (vertices, rest_vertices, tets), ``material``, ``kinematic_mask``,
``velocity``, ``collide_self``; ``AffineBody``-likes expose ``surface``
(vertices, triangles), ``material``, ``kappa``; ``KinematicBody``-likes expose
``surface`` (vertices, rest_vertices, triangles), ``material``, ``velocity``.
The kind is read from ``body.kind`` when present, else from the class name.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import energies as en
from oracle import geometry as geo

_TET_FACES = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]], np.int64)   # mesh.py:19


class SolveBreakdown(RuntimeError):
    """solver.py:87."""


# ---------------------------------------------------------------------------
# mesh-derived data (restating the pieces of geometry/mesh.py the build uses)
# ---------------------------------------------------------------------------


def boundary(tets, n_vertices):
    """(triangles in compact ids, vertex map); mesh.py:185-209."""
    faces = tets[:, _TET_FACES].reshape(-1, 3)
    _, inv, cnt = np.unique(np.sort(faces, axis=1), axis=0, return_inverse=True, return_counts=True)
    faces = faces[cnt[inv.reshape(-1)] == 1]
    used = np.unique(faces)
    remap = np.full(n_vertices, -1, np.int64)
    remap[used] = np.arange(len(used))
    return remap[faces], used


def unique_edges(tris):
    """Lexicographically sorted undirected edges; mesh.py:72-79."""
    e = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]])
    return np.unique(np.sort(e, axis=1), axis=0)


def tet_volumes(v, tets):
    """mesh.py:143-148."""
    d1, d2, d3 = (v[tets[:, k]] - v[tets[:, 0]] for k in (1, 2, 3))
    return np.einsum("ij,ij->i", np.cross(d1, d2), d3) / 6.0


def enclosed_volume(v, t):
    """mesh.py:99-102."""
    return float(np.einsum("ij,ij->i", v[t[:, 0]], np.cross(v[t[:, 1]], v[t[:, 2]])).sum() / 6.0)


def mass_properties(v, t, rho):
    """(mass, com, second moment at com); mesh.py:544-571."""
    a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    vols = np.einsum("ij,ij->i", a, np.cross(b, c)) / 6.0
    V = vols.sum()
    if V <= 0.0:
        raise ValueError("surface encloses non-positive volume")
    com = (vols[:, None] * ((a + b + c) / 4.0)).sum(axis=0) / V
    s = a + b + c
    o = lambda q: q[:, :, None] * q[:, None, :]  # noqa: E731
    second = (vols[:, None, None] / 20.0 * (o(a) + o(b) + o(c) + o(s))).sum(axis=0)
    mass = rho * V
    return mass, com, rho * second - mass * np.outer(com, com)


def body_kind(body):
    k = getattr(body, "kind", None)
    if isinstance(k, str):
        return k
    name = type(body).__name__
    return {"SoftBody": "soft", "AffineBody": "affine", "KinematicBody": "kinematic"}[name]


# ---------------------------------------------------------------------------
# environment
# ---------------------------------------------------------------------------


class NewtonState:
    """solver.py:180-192."""

    def __init__(self):
        self.energy = np.inf
        self.iterations = 0
        self.alphas = []
        self.done = False
        self.status = "running"
        self.residual = np.inf
        self.reason = ""
        self.regularized = False
        self.kinematic_blocked = False


def linear_solve(H, g):
    """Direct solve with one refinement and a regularized retry; solver.py:91-131."""
    if g.size == 0:
        return np.zeros(0), False
    ng = np.linalg.norm(g)
    if ng == 0.0:
        return np.zeros_like(g), False
    H = H.tocsc()
    reg = False
    for attempt in range(2):
        try:
            lu = spla.splu(H)
            p = lu.solve(-g)
            if not np.all(np.isfinite(p)):
                raise RuntimeError("non-finite solution")
            r = H @ p + g
            if np.linalg.norm(r) > 1e-10 * ng:
                p -= lu.solve(r)
                r = H @ p + g
            if np.linalg.norm(r) <= 1e-8 * ng:
                return p, reg
            raise RuntimeError("residual too large")
        except RuntimeError:
            if attempt == 1:
                raise SolveBreakdown("linear solve failed after regularization")
            H = (H + 1e-8 * max(float(H.diagonal().max()), 1.0) * sp.identity(H.shape[0], format="csc")).tocsc()
            reg = True
    raise SolveBreakdown("unreachable")


class OracleEnv:
    """One environment; restates solver.Environment (solver.py:195-773)."""

    def __init__(self, bodies, gravity=(0.0, 0.0, 0.0), contact=None, solver=None, collide_pairs_off=(),
                 env_id=0):
        c = contact or {}
        s = solver or {}
        self.kappa = float(c.get("kappa", 3e6))
        self.dhat = float(c.get("dhat", 1e-3))
        self.eps_v = float(c.get("eps_v", 1e-3))
        self.mu_rule = c.get("friction_combination", "geometric")
        self.dt = float(s.get("dt", 0.01))
        self.rel_tol = float(s.get("rel_tol", 1e-3))
        self.max_iters = int(s.get("max_iters", 100))
        self.ell_floor = float(s.get("length_scale_floor", 0.05))
        self.max_ls = int(s.get("max_line_search", 50))
        self.ccd_scaling = float(s.get("ccd_scaling", 0.9))
        self.ccd_iters = int(s.get("ccd_max_iters", 32))
        self.kin_guard = float(s.get("kinematic_ccd_guard", 0.1))
        self.bodies = list(bodies)
        self.gravity = np.asarray(gravity, np.float64).reshape(3)
        self.status = "active"
        self.fail_reason = ""
        self.time = 0.0
        self.step_index = 0
        self.env_id = env_id
        self._build(collide_pairs_off)

    # -- construction (solver.py:214-363) ------------------------------------
    def _build(self, pairs_off):
        nb = len(self.bodies)
        self.recs = []
        dof0 = surf0 = 0
        rest_chunks, e_chunks, t_chunks, vbody = [], [], [], []
        Gr, Gc, Gv, Mr, Mc, Mv, tets_node = [], [], [], [], [], [], []
        self.mu_body = np.zeros(nb)
        kin = np.zeros(nb, bool)
        x0 = []
        for bid, body in enumerate(self.bodies):
            kind = body_kind(body)
            rec = {"body": body, "kind": kind, "dof0": dof0, "surf0": surf0}
            self.mu_body[bid] = body.material.friction_coefficient
            if kind == "soft":
                mesh = body.mesh
                tets = np.asarray(mesh.tets, np.int64)
                rest = np.asarray(mesh.rest_vertices, np.float64)
                nv = len(rest)
                tris, vmap = boundary(tets, nv)
                Dmi, V0, w = en.tet_rest(rest, tets)
                rec.update(ndof=3 * nv, n_sv=len(vmap), tets=tets, Dmi=Dmi, V0=V0, w=w,
                           lame=en.lame(body.material.young_modulus, body.material.poisson_ratio))
                masses = np.zeros(nv)
                np.add.at(masses, tets.reshape(-1), np.repeat(body.material.density * tet_volumes(rest, tets) / 4.0, 4))
                rec["masses"] = masses
                rest_chunks.append(rest[vmap])
                t_chunks.append(tris + surf0)
                e_chunks.append(unique_edges(tris) + surf0)
                vbody += [bid] * len(vmap)
                Gr.append((3 * (surf0 + np.arange(len(vmap)))[:, None] + np.arange(3)).ravel())
                Gc.append((dof0 + 3 * vmap[:, None] + np.arange(3)).ravel())
                Gv.append(np.ones(3 * len(vmap)))
                Mr.append(dof0 + np.arange(3 * nv)); Mc.append(dof0 + np.arange(3 * nv))
                Mv.append(np.repeat(masses, 3))
                tets_node.append(tets + dof0 // 3)
                x0.append(np.asarray(mesh.vertices, np.float64).reshape(-1))
                mask = getattr(body, "kinematic_mask", None)
                rec["kmask"] = np.zeros(nv, bool) if mask is None else np.asarray(mask, bool)
                surf0 += len(vmap); dof0 += 3 * nv
            elif kind == "affine":
                v = np.asarray(body.surface.vertices, np.float64)
                tr = np.asarray(body.surface.triangles, np.int64)
                mass, com, second = mass_properties(v, tr, body.material.density)
                xi = v - com
                rec.update(ndof=12, n_sv=len(xi), xi=xi, mass=mass, volume=enclosed_volume(v, tr),
                           kappa=float(getattr(body, "kappa", 1e8)))
                M12 = np.zeros((12, 12))
                M12[:3, :3] = mass * np.eye(3)
                for a in range(3):
                    M12[3 + 3 * a:6 + 3 * a, 3 + 3 * a:6 + 3 * a] = second
                rest_chunks.append(xi)
                t_chunks.append(tr + surf0)
                e_chunks.append(unique_edges(tr) + surf0)
                vbody += [bid] * len(xi)
                for loc, xv in enumerate(xi):
                    base = 3 * (surf0 + loc)
                    for a in range(3):
                        Gr.append(np.array([base + a])); Gc.append(np.array([dof0 + a])); Gv.append(np.array([1.0]))
                        Gr.append(np.full(3, base + a)); Gc.append(dof0 + 3 + 3 * a + np.arange(3)); Gv.append(xv)
                ii, jj = np.nonzero(M12)
                Mr.append(dof0 + ii); Mc.append(dof0 + jj); Mv.append(M12[ii, jj])
                q0 = np.zeros(12); q0[:3] = com; q0[3:] = np.eye(3).reshape(-1)
                x0.append(q0)
                surf0 += len(xi); dof0 += 12
            elif kind == "kinematic":
                v = np.asarray(body.surface.vertices, np.float64)
                tr = np.asarray(body.surface.triangles, np.int64)
                restv = np.asarray(getattr(body.surface, "rest_vertices", v), np.float64)
                rec.update(ndof=0, n_sv=len(v), positions=v.copy())
                kin[bid] = True
                rest_chunks.append(restv)
                t_chunks.append(tr + surf0)
                e_chunks.append(unique_edges(tr) + surf0)
                vbody += [bid] * len(v)
                surf0 += len(v)
            else:
                raise TypeError(f"unknown body kind {kind}")
            self.recs.append(rec)
        self.n_dofs, self.n_sv = dof0, surf0
        self.x = np.concatenate(x0) if x0 else np.zeros(0)
        self.v = np.zeros(self.n_dofs)
        rest = np.concatenate(rest_chunks)
        self.edges = np.concatenate(e_chunks)
        self.tris = np.concatenate(t_chunks)
        self.vbody = np.asarray(vbody, np.int64)
        collide = np.ones((nb, nb), bool)
        for bid, body in enumerate(self.bodies):
            collide[bid, bid] = bool(getattr(body, "collide_self", False))
        for a, b in pairs_off:
            collide[a, b] = collide[b, a] = False
        self.pair_ok = collide & ~(kin[:, None] & kin[None, :])
        de = rest[self.edges[:, 1]] - rest[self.edges[:, 0]]
        self.edge_rest_sq = np.einsum("ij,ij->i", de, de)
        self.G = sp.coo_matrix((np.concatenate(Gv), (np.concatenate(Gr), np.concatenate(Gc))),
                               shape=(3 * self.n_sv, self.n_dofs)).tocsr()
        self.M = sp.coo_matrix((np.concatenate(Mv), (np.concatenate(Mr), np.concatenate(Mc))),
                               shape=(self.n_dofs, self.n_dofs)).tocsr()
        free = np.ones(self.n_dofs, bool)
        for rec in self.recs:
            if rec["kind"] == "soft":
                free[rec["dof0"]:rec["dof0"] + rec["ndof"]] = ~np.repeat(rec["kmask"], 3)
        self.free = free
        self.free_idx = np.nonzero(free)[0]
        self.tets_node = np.concatenate(tets_node) if tets_node else np.zeros((0, 4), np.int64)
        self.anchors = en.empty_anchors()

    # -- state access (solver.py:367-481) -------------------------------------
    def surface_positions(self, x=None):
        x = self.x if x is None else x
        sv_ = (self.G @ x).reshape(-1, 3)
        for rec in self.recs:
            if rec["kind"] == "kinematic":
                sv_[rec["surf0"]:rec["surf0"] + rec["n_sv"]] = rec["positions"]
        return sv_

    def node_positions(self):
        return self.x.reshape(-1, 3)

    def bbox_diagonal(self):
        s = self.surface_positions()
        return float(np.linalg.norm(s.max(axis=0) - s.min(axis=0))) if len(s) else 0.0

    def body_com(self, bid):
        rec = self.recs[bid]
        if rec["kind"] == "soft":
            xs = self.x[rec["dof0"]:rec["dof0"] + rec["ndof"]].reshape(-1, 3)
            return (rec["masses"][:, None] * xs).sum(axis=0) / rec["masses"].sum()
        if rec["kind"] == "affine":
            return self.x[rec["dof0"]:rec["dof0"] + 3].copy()
        return rec["positions"].mean(axis=0)

    def max_point_speed(self):
        sp_ = [0.0]
        for rec in self.recs:
            if rec["kind"] == "soft":
                vs = self.v[rec["dof0"]:rec["dof0"] + rec["ndof"]].reshape(-1, 3)
                sp_.append(float(np.linalg.norm(vs, axis=1).max()))
            elif rec["kind"] == "affine":
                vq = self.v[rec["dof0"]:rec["dof0"] + 12]
                vs = vq[None, :3] + rec["xi"] @ vq[3:].reshape(3, 3).T
                sp_.append(float(np.linalg.norm(vs, axis=1).max()))
            else:
                sp_.append(float(np.linalg.norm(rec["body"].velocity)))
        return max(sp_)

    # -- contact plumbing (solver.py:432-467) ----------------------------------
    def candidates(self, sv_, r):
        return geo.broad_phase(sv_, self.tris, self.edges, self.vbody, self.pair_ok, r)

    def contact_set(self, c):
        pt, ee = c["pt"], c["ee"]
        cs = {"pt": pt, "ee": ee,
              "pt_bodies": np.stack([self.vbody[pt[:, 0]], self.vbody[pt[:, 1]]], 1) if len(pt) else np.zeros((0, 2), np.int64),
              "ee_bodies": np.stack([self.vbody[ee[:, 0]], self.vbody[ee[:, 2]]], 1) if len(ee) else np.zeros((0, 2), np.int64),
              "eps_x": (self.edge_rest_sq[c["ee_edges"][:, 0]] * self.edge_rest_sq[c["ee_edges"][:, 1]]) if len(ee) else np.zeros(0)}
        cs["pt_mu"] = en.combine_mu(self.mu_body[cs["pt_bodies"][:, 0]], self.mu_body[cs["pt_bodies"][:, 1]], self.mu_rule) if len(pt) else np.zeros(0)
        cs["ee_mu"] = en.combine_mu(self.mu_body[cs["ee_bodies"][:, 0]], self.mu_body[cs["ee_bodies"][:, 1]], self.mu_rule) if len(ee) else np.zeros(0)
        return cs

    def contact_set_now(self, factor=1.05):
        return self.contact_set(self.candidates(self.surface_positions(), self.dhat * factor))

    @staticmethod
    def min_distance(cs, sv_):
        best = np.inf
        if len(cs["pt"]):
            p = cs["pt"]
            best = min(best, float(geo.pt_closest(sv_[p[:, 0]], sv_[p[:, 1]], sv_[p[:, 2]], sv_[p[:, 3]])[0].min()))
        if len(cs["ee"]):
            e = cs["ee"]
            best = min(best, float(geo.ee_closest(sv_[e[:, 0]], sv_[e[:, 1]], sv_[e[:, 2]], sv_[e[:, 3]])[0].min()))
        return float(np.sqrt(best))

    def events_now(self):
        """protocol.py:72-75."""
        cs = self.contact_set_now()
        return en.stencil_forces(self.surface_positions(), cs["pt"], cs["ee"], cs["eps_x"],
                                 cs["pt_bodies"], cs["ee_bodies"], self.kappa, self.dhat)

    # -- energy and assembly (solver.py:485-586) ------------------------------
    def _elastic(self, x, order):
        E = 0.0
        g = np.zeros(self.n_dofs) if order >= 1 else None
        blocks = []
        for rec in self.recs:
            sl = slice(rec["dof0"], rec["dof0"] + rec["ndof"])
            if rec["kind"] == "soft":
                mu, lam = rec["lame"]
                e, gg, H, _ = en.neo_hookean(x[sl].reshape(-1, 3), rec["tets"], rec["Dmi"], rec["V0"], rec["w"],
                                             mu, lam, order=max(order, 1), project=True)
                E += e
                if order >= 1:
                    g[sl] += gg.reshape(-1)
                if order >= 2:
                    blocks.append((rec["dof0"] + (3 * rec["tets"][:, :, None] + np.arange(3)).reshape(-1, 12), H))
            elif rec["kind"] == "affine":
                q = x[sl]
                e, gg, H = en.abd_ortho(q[3:].reshape(3, 3), rec["kappa"] * rec["volume"], order=order)
                E += e
                if order >= 1:
                    g[sl] += gg
                if order >= 2:
                    blocks.append(((rec["dof0"] + np.arange(12))[None], H[None]))
        return E, g, blocks

    def energy(self, x, cs, xhat, surf_prev):
        """Incremental potential, +inf when invalid; solver.py:518-533."""
        dx = x - xhat
        E = 0.5 * float(dx @ (self.M @ dx))
        try:
            e_el, _, _ = self._elastic(x, 0)
            s = self.surface_positions(x)
            e_c = en.contact_potential(s, cs["pt"], cs["ee"], cs["eps_x"], self.kappa, self.dhat, order=0)[0]
            e_f = en.friction_potential(self.anchors, s, surf_prev, self.eps_v, self.dt, order=0)[0]
        except ValueError:
            return np.inf
        tot = E + self.dt * self.dt * (e_el + e_c + e_f)
        return tot if np.isfinite(tot) else np.inf

    @staticmethod
    def _coo(idx, blocks):
        n, w = idx.shape
        return (np.repeat(idx, w, axis=1).reshape(-1), np.tile(idx[:, None, :], (1, w, 1)).reshape(-1),
                blocks.reshape(-1))

    def assemble(self, x, cs, xhat, surf_prev):
        dt2 = self.dt * self.dt
        dx = x - xhat
        Mdx = self.M @ dx
        E = 0.5 * float(dx @ Mdx)
        g = Mdx.copy()
        rows, cols, vals = [], [], []
        e_el, g_el, blk = self._elastic(x, 2)
        E += dt2 * e_el
        g += dt2 * g_el
        for idx, H in blk:
            r, c, v = self._coo(idx, dt2 * H)
            rows.append(r); cols.append(c); vals.append(v)
        s = self.surface_positions(x)
        e_c, g_c, idx_c, H_c = en.contact_potential(s, cs["pt"], cs["ee"], cs["eps_x"], self.kappa, self.dhat, 2)
        e_f, g_f, idx_f, H_f = en.friction_potential(self.anchors, s, surf_prev, self.eps_v, self.dt, 2)
        E += dt2 * (e_c + e_f)
        g += self.G.T @ (dt2 * (g_c + g_f)).reshape(-1)
        sr, sc_, sv_ = [], [], []
        for idx, H in ((idx_c, H_c), (idx_f, H_f)):
            if len(idx):
                r, c, v = self._coo((3 * idx[:, :, None] + np.arange(3)).reshape(len(idx), 12), dt2 * H)
                sr.append(r); sc_.append(c); sv_.append(v)
        if sr:
            Hsv = sp.coo_matrix((np.concatenate(sv_), (np.concatenate(sr), np.concatenate(sc_))),
                                shape=(3 * self.n_sv, 3 * self.n_sv)).tocsr()
            Hcf = (self.G.T @ Hsv @ self.G).tocoo()
            rows.append(Hcf.row); cols.append(Hcf.col); vals.append(Hcf.data)
        Mc = self.M.tocoo()
        rows.append(Mc.row); cols.append(Mc.col); vals.append(Mc.data)
        H = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.n_dofs, self.n_dofs)).tocsr()
        return E, g, H

    # -- stepping (solver.py:590-773) --------------------------------------------
    def begin_step(self):
        dt = self.dt
        self._x_t = self.x.copy()
        self._surf_prev = self.surface_positions()
        ns = NewtonState()
        dx = np.zeros(self.n_dofs)
        kd = np.zeros((self.n_sv, 3))
        moving = False
        for rec in self.recs:
            vel = getattr(rec["body"], "velocity", None)
            if rec["kind"] == "kinematic" and np.any(vel):
                kd[rec["surf0"]:rec["surf0"] + rec["n_sv"]] = vel * dt
                moving = True
            elif rec["kind"] == "soft" and np.any(rec["kmask"]) and np.any(vel):
                loc = np.zeros(rec["ndof"])
                loc[np.repeat(rec["kmask"], 3)] = np.tile(vel * dt, int(rec["kmask"].sum()))
                dx[rec["dof0"]:rec["dof0"] + rec["ndof"]] = loc
                moving = True
        ak = 1.0
        if moving:
            s = self.surface_positions()
            disp = (self.G @ dx).reshape(-1, 3) + kd
            md = float(np.linalg.norm(disp, axis=1).max())
            c = self.candidates(s, self.dhat + 2.0 * md)
            if len(c["pt"]) or len(c["ee"]):
                ak = geo.ccd_max_step(s, disp, c["pt"], c["ee"], self.ccd_scaling, self.ccd_iters, self.kin_guard)
            self.x += ak * dx
            for rec in self.recs:
                if rec["kind"] == "kinematic":
                    rec["positions"] = rec["positions"] + ak * rec["body"].velocity * dt
            ns.kinematic_blocked = ak < 1.0 - 1e-12
        a = np.zeros(self.n_dofs)
        for rec in self.recs:
            if rec["kind"] == "soft":
                a[rec["dof0"]:rec["dof0"] + rec["ndof"]] = np.tile(self.gravity, rec["ndof"] // 3)
            elif rec["kind"] == "affine":
                a[rec["dof0"]:rec["dof0"] + 3] = self.gravity
        xh = self.x + dt * self.v + dt * dt * a
        xh[~self.free] = self.x[~self.free]
        self._xhat = xh
        self._ell = max(self.bbox_diagonal(), self.ell_floor)
        return ns

    def newton_iteration(self, ns):
        try:
            cs = self.contact_set(self.candidates(self.surface_positions(), self.dhat * 1.05))
            E, g, H = self.assemble(self.x, cs, self._xhat, self._surf_prev)
            if not (np.isfinite(E) and np.all(np.isfinite(g))):
                raise FloatingPointError("non-finite assembly")
            gf = g[self.free_idx]
            Hff = H[self.free_idx][:, self.free_idx]
            pf, reg = linear_solve(Hff, gf)
            ns.regularized |= reg
            tol = self.rel_tol * self.dt * self._ell
            res = float(np.abs(pf).max()) if len(pf) else 0.0
            ns.residual = res
            if res < tol:
                ns.done, ns.status, ns.energy = True, "converged", E
                return ns
            if ns.iterations >= self.max_iters:
                ns.done, ns.status, ns.reason = True, "failed", "non-convergence"
                return ns
            p = np.zeros(self.n_dofs)
            p[self.free_idx] = pf
            disp = (self.G @ p).reshape(-1, 3)
            md = float(np.linalg.norm(disp, axis=1).max()) if len(disp) else 0.0
            s = self.surface_positions()
            cs2 = self.contact_set(self.candidates(s, self.dhat + 2.0 * md))
            a0 = 1.0
            if len(cs2["pt"]) + len(cs2["ee"]):
                a0 = min(a0, geo.ccd_max_step(s, disp, cs2["pt"], cs2["ee"], self.ccd_scaling, self.ccd_iters))
            if len(self.tets_node):
                a0 = min(a0, geo.tet_filter(self.node_positions(), p.reshape(-1, 3), self.tets_node, self.ccd_scaling))
            for rec in self.recs:
                if rec["kind"] == "affine":
                    A = self.x[rec["dof0"] + 3:rec["dof0"] + 12].reshape(1, 3, 3)
                    dA = p[rec["dof0"] + 3:rec["dof0"] + 12].reshape(1, 3, 3)
                    if np.any(dA):
                        a0 = min(a0, geo.pencil_step(A, dA, self.ccd_scaling))
            E0 = self.energy(self.x, cs2, self._xhat, self._surf_prev)
            alpha = a0
            for _ in range(self.max_ls):
                Et = self.energy(self.x + alpha * p, cs2, self._xhat, self._surf_prev)
                if Et < E0:
                    break
                alpha *= 0.5
            else:
                if res < 10.0 * tol:
                    ns.done, ns.status, ns.energy = True, "converged", E0
                    return ns
                ns.done, ns.status, ns.reason = True, "failed", "line-search-failure"
                return ns
            self.x = self.x + alpha * p
            ns.iterations += 1
            ns.alphas.append(float(alpha))
            ns.energy = Et
            return ns
        except (np.linalg.LinAlgError, FloatingPointError, SolveBreakdown, ValueError, geo.IntersectionError) as exc:
            ns.done, ns.status = True, "failed"
            ns.reason = type(exc).__name__ + ": " + str(exc)
            return ns

    def finalize_step(self, ns):
        md = np.inf
        if ns.status == "failed":
            self.status = "failed"
            self.fail_reason = ns.reason
        else:
            self.v = (self.x - self._x_t) / self.dt
            cs = self.contact_set_now()
            s = self.surface_positions()
            self.anchors = en.friction_anchors(s, cs["pt"], cs["ee"], cs["eps_x"], cs["pt_mu"], cs["ee_mu"],
                                               cs["pt_bodies"], cs["ee_bodies"], self.kappa, self.dhat)
            if len(cs["pt"]) + len(cs["ee"]):
                md = self.min_distance(cs, s)
        rep = {"env": self.env_id, "step": self.step_index, "t": self.time, "status": ns.status,
               "iterations": ns.iterations, "residual": ns.residual, "alphas": list(ns.alphas),
               "min_distance": float(md), "energy": float(ns.energy) if np.isfinite(ns.energy) else float("inf"),
               "kinematic_blocked": ns.kinematic_blocked, "regularized": ns.regularized, "reason": ns.reason}
        self.time += self.dt
        self.step_index += 1
        return rep

    def step(self):
        if self.status != "active":
            raise RuntimeError(f"stepping a {self.status} environment")
        ns = self.begin_step()
        self.n_calls = getattr(self, "n_calls", 0)
        while not ns.done:
            self.newton_iteration(ns)
            self.n_calls += 1
        return self.finalize_step(ns)

    # -- per-step outputs used by the protocol ----------------------------------
    def stress_rows(self):
        rows = []
        for rec in self.recs:
            if rec["kind"] == "soft":
                mu, lam = rec["lame"]
                xs = self.x[rec["dof0"]:rec["dof0"] + rec["ndof"]].reshape(-1, 3)
                rows.append(en.cauchy_stress(xs, rec["tets"], rec["Dmi"], mu, lam))
        return np.concatenate(rows) if rows else np.zeros((0, 7))


# ---------------------------------------------------------------------------
# batch (multienv.py:73-178) and closing rollout
# ---------------------------------------------------------------------------


class OracleBatch:
    """Lockstep stepping with per-env freezing and quarantine; multienv.py:73-178."""

    def __init__(self, envs):
        self.envs = list(envs)
        self.statuses = ["failed" if e.status == "failed" else "active" for e in self.envs]
        for i, e in enumerate(self.envs):
            e.env_id = i

    def quarantine(self):
        for i, e in enumerate(self.envs):
            if self.statuses[i] in ("failed", "done"):
                continue
            if e.status == "failed" or (e.n_dofs and not np.all(np.isfinite(e.x))):
                if e.status != "failed":
                    e.status, e.fail_reason = "failed", "non-finite state"
                self.statuses[i] = "failed"

    def step(self):
        self.quarantine()
        ids = [i for i, s in enumerate(self.statuses) if s == "active"]
        states = {i: self.envs[i].begin_step() for i in ids}
        pending = [i for i in ids if not states[i].done]
        while pending:
            for i in pending:
                self.envs[i].newton_iteration(states[i])
            pending = [i for i in pending if not states[i].done]
        reps = [self.envs[i].finalize_step(states[i]) for i in ids]
        self.quarantine()
        return dict(zip(ids, reps))


def finger_force(events, ids):
    """protocol.py:78-86."""
    ids = set(ids)
    return sum(ev["lambda"] for ev in events if ids.intersection(ev["bodies"]))


def closing_rollout(env, fingers, closing_dirs, n_steps, speed=0.05, halt=50.0, gravity_after=None,
                    gravity=(0.0, 0.0, -9.8)):
    """Fingers close at `speed`, each halting once its force exceeds `halt`."""
    halted = {f: False for f in fingers}
    for f, ids in fingers.items():
        for b in ids:
            env.bodies[b].velocity = np.asarray(closing_dirs[f], np.float64) * speed
    out = {"x": [], "reports": [], "forces": []}
    for k in range(n_steps):
        if gravity_after is not None and k == gravity_after:
            env.gravity = np.asarray(gravity, np.float64)
        rep = env.step()
        ev = env.events_now()
        forces = {f: finger_force(ev, ids) for f, ids in fingers.items()}
        out["x"].append(env.x.copy()); out["reports"].append(rep); out["forces"].append(forces)
        for f in fingers:
            if not halted[f] and forces[f] > halt:
                halted[f] = True
                for b in fingers[f]:
                    env.bodies[b].velocity = np.zeros(3)
        if rep["status"] == "failed":
            break
    return out
