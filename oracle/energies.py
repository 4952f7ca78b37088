"""Oracle energies: barrier contact, lagged friction, Neo-Hookean, ABD, stress.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
/root/reference/pkg/src/gripsim/{contact,materials}.py.
"""

from __future__ import annotations

import numpy as np

from oracle.geometry import (
    cross_norm_sq,
    ee_closest,
    ee_plane,
    pe_derivs,
    pp_derivs,
    pt_closest,
    pt_plane,
)

_I3 = np.eye(3)


# ---------------------------------------------------------------------------
# scalar profiles (contact.py:49-98)
# ---------------------------------------------------------------------------


def barrier_d(d, dhat):
    """b, b', b'' in d for 0<d<dhat else 0; contact.py:49-64."""
    d = np.asarray(d, np.float64)
    if np.any(d <= 0.0):
        raise ValueError("barrier evaluated at non-positive distance")
    inside = d < dhat
    dd = d - dhat
    with np.errstate(divide="ignore", invalid="ignore"):
        ln = np.where(inside, np.log(d / dhat), 0.0)
    b = np.where(inside, -dd * dd * ln, 0.0)
    b1 = np.where(inside, -2.0 * dd * ln - dd * dd / d, 0.0)
    b2 = np.where(inside, -2.0 * ln - 4.0 * dd / d + (dd / d) ** 2, 0.0)
    return b, b1, b2


def barrier_D(D, dhat):
    """Barrier through D=d^2: (b, f1=db/dD, f2=d2b/dD2); contact.py:67-76."""
    D = np.asarray(D, np.float64)
    if np.any(D <= 0.0):
        raise ValueError("barrier evaluated at non-positive squared distance")
    d = np.sqrt(D)
    b, b1, b2 = barrier_d(d, dhat)
    return b, b1 / (2.0 * d), (b2 * d - b1) / (4.0 * d * D)


def friction_f0_f1(y, eps_v, dt):
    """C1 static/dynamic transition; contact.py:79-90."""
    y = np.asarray(y, np.float64)
    h = eps_v * dt
    inside = y < h
    f1 = np.where(inside, 2.0 * y / h - (y / h) ** 2, 1.0)
    f0 = np.where(inside, y * y / h - y ** 3 / (3.0 * h * h), y - h / 3.0)
    return f0, f1


def combine_mu(mu_a, mu_b, rule="geometric"):
    """contact.py:93-98."""
    if rule == "geometric":
        return np.sqrt(np.asarray(mu_a) * np.asarray(mu_b))
    if rule == "min":
        return np.minimum(mu_a, mu_b)
    raise ValueError(f"unknown friction combination rule: {rule}")


def spd_clamp(H, rel_floor=1e-12):
    """Eigen-clamp to max(lambda, rel_floor*max|lambda|); materials.py:101-113."""
    H = 0.5 * (H + H.transpose(0, 2, 1))
    lam, V = np.linalg.eigh(H)
    lam = np.maximum(lam, rel_floor * np.abs(lam).max(axis=1, keepdims=True))
    out = np.einsum("nik,nk,njk->nij", V, lam, V)
    return 0.5 * (out + out.transpose(0, 2, 1))


# ---------------------------------------------------------------------------
# contact (contact.py:178-344)
# ---------------------------------------------------------------------------

_PT_EDGE = {3: (1, 2), 4: (2, 3), 5: (3, 1)}   # contact.py:102


def _embed_grad(g_small, slots):
    """Place k-point gradients into the 12-slot layout (the grad half of contact.py:105-114)."""
    out = np.zeros((len(g_small), 12))
    rows = np.arange(len(g_small))
    for a in range(slots.shape[1]):
        for c in range(3):
            out[rows, 3 * slots[:, a] + c] = g_small[:, 3 * a + c]
    return out


def pt_terms(x4, order):
    """D, grad, hess of PT stencils with region dispatch; contact.py:178-211.

    Non-face regions contribute their gradient only: the reference's
    ``_expand_rows`` writes their Hessian through an advanced-index copy
    (contact.py:116-125), so it stays zero.  Reproduced on purpose.
    """
    D, _, region = pt_closest(x4[:, 0], x4[:, 1], x4[:, 2], x4[:, 3])
    if order == 0:
        return D, None, None, region
    n = len(x4)
    g = np.zeros((n, 12))
    H = np.zeros((n, 12, 12)) if order >= 2 else None
    face = region == 6
    if face.any():
        gf, Hf = pt_plane(x4[face])
        g[face] = gf
        if order >= 2:
            H[face] = Hf
    for code, (sa, sb) in _PT_EDGE.items():
        m = region == code
        if m.any():
            gs = pe_derivs(x4[m, 0], x4[m, sa], x4[m, sb])
            g[m] = _embed_grad(gs, np.tile([0, sa, sb], (int(m.sum()), 1)))
    for code in range(3):
        m = region == code
        if m.any():
            gs = pp_derivs(x4[m, 0], x4[m, 1 + code])
            g[m] = _embed_grad(gs, np.tile([0, 1 + code], (int(m.sum()), 1)))
    return D, g, H, region


def ee_terms(x4, order):
    """EE stencils, pre-mollifier; contact.py:213-256 (same Hessian quirk as pt_terms)."""
    D, s, t = ee_closest(x4[:, 0], x4[:, 1], x4[:, 2], x4[:, 3])
    if order == 0:
        return D, None, None, (s, t)
    n = len(x4)
    g = np.zeros((n, 12))
    H = np.zeros((n, 12, 12)) if order >= 2 else None
    s_in = (s > 0.0) & (s < 1.0)
    t_in = (t > 0.0) & (t < 1.0)
    both = s_in & t_in
    if both.any():
        gb, Hb = ee_plane(x4[both])
        g[both] = gb
        if order >= 2:
            H[both] = Hb
    rows = np.arange(n)
    # point of edge b against edge a
    m = s_in & ~t_in
    if m.any():
        ps = np.where(t[m] < 0.5, 2, 3)
        gs = pe_derivs(x4[rows[m], ps], x4[m, 0], x4[m, 1])
        g[m] = _embed_grad(gs, np.stack([ps, np.zeros_like(ps), np.ones_like(ps)], 1))
    m = ~s_in & t_in
    if m.any():
        ps = np.where(s[m] < 0.5, 0, 1)
        gs = pe_derivs(x4[rows[m], ps], x4[m, 2], x4[m, 3])
        g[m] = _embed_grad(gs, np.stack([ps, np.full_like(ps, 2), np.full_like(ps, 3)], 1))
    m = ~s_in & ~t_in
    if m.any():
        sa = np.where(s[m] < 0.5, 0, 1)
        sb = np.where(t[m] < 0.5, 2, 3)
        gs = pp_derivs(x4[rows[m], sa], x4[rows[m], sb])
        g[m] = _embed_grad(gs, np.stack([sa, sb], 1))
    return D, g, H, (s, t)


def mollifier(x4, eps_x, order):
    """EE parallel mollifier m(c), c=|u x v|^2, eps=1e-3*eps_x; contact.py:258-269."""
    c, gc, Hc = cross_norm_sq(x4)
    eps = 1e-3 * eps_x
    xr = c / eps
    inside = xr < 1.0
    m = np.where(inside, xr * (2.0 - xr), 1.0)
    if order == 0:
        return m, None, None, None, None
    dm = np.where(inside, (2.0 - 2.0 * xr) / eps, 0.0)
    d2m = np.where(inside, -2.0 / (eps * eps), 0.0)
    return m, dm, d2m, gc, Hc


def contact_potential(x, pt, ee, eps_x, kappa, dhat, order=2, project=True):
    """kappa*sum m*b(d) over active stencils; contact.py:271-344.

    Returns (E, grad (n_sv,3), idx (G,4), blocks (G,12,12)); raises
    ValueError on a non-positive candidate distance, like the reference.
    """
    E = 0.0
    grad = np.zeros((len(x), 3))
    idx_out, blk_out = [], []
    if len(pt):
        D, gD, HD, _ = pt_terms(x[pt], order)
        if np.any(D <= 0.0):
            raise ValueError("contact stencil at non-positive distance")
        act = D < dhat * dhat
        if act.any():
            b, f1, f2 = barrier_D(D[act], dhat)
            E += kappa * float(b.sum())
            if order >= 1:
                np.add.at(grad, pt[act].reshape(-1), (kappa * f1[:, None] * gD[act]).reshape(-1, 3))
            if order >= 2:
                g = gD[act]
                H = kappa * (f2[:, None, None] * g[:, :, None] * g[:, None, :] + f1[:, None, None] * HD[act])
                blk_out.append(spd_clamp(H) if project else H)
                idx_out.append(pt[act])
    if len(ee):
        D, gD, HD, _ = ee_terms(x[ee], order)
        if np.any(D <= 0.0):
            raise ValueError("contact stencil at non-positive distance")
        act = D < dhat * dhat
        if act.any():
            m, dm, d2m, gc, Hc = mollifier(x[ee[act]], eps_x[act], order)
            b, f1, f2 = barrier_D(D[act], dhat)
            E += kappa * float((m * b).sum())
            if order >= 1:
                gb = f1[:, None] * gD[act]
                gm = dm[:, None] * gc
                np.add.at(grad, ee[act].reshape(-1), (kappa * (m[:, None] * gb + b[:, None] * gm)).reshape(-1, 3))
            if order >= 2:
                g = gD[act]
                Hb = f2[:, None, None] * g[:, :, None] * g[:, None, :] + f1[:, None, None] * HD[act]
                Hm = d2m[:, None, None] * gc[:, :, None] * gc[:, None, :] + dm[:, None, None] * Hc
                cr = gm[:, :, None] * gb[:, None, :]
                H = kappa * (m[:, None, None] * Hb + b[:, None, None] * Hm + cr + cr.transpose(0, 2, 1))
                blk_out.append(spd_clamp(H) if project else H)
                idx_out.append(ee[act])
    idx = np.concatenate(idx_out) if idx_out else np.zeros((0, 4), np.int64)
    blocks = np.concatenate(blk_out) if blk_out else np.zeros((0, 12, 12))
    return E, grad, idx, blocks


def stencil_forces(x, pt, ee, eps_x, pt_bodies, ee_bodies, kappa, dhat):
    """Per active stencil (kind, bodies, verts, d, lambda); contact.py:348-372."""
    out = []
    if len(pt):
        D, _, _ = pt_closest(x[pt[:, 0]], x[pt[:, 1]], x[pt[:, 2]], x[pt[:, 3]])
        act = D < dhat * dhat
        if act.any():
            d = np.sqrt(D[act])
            lam = kappa * np.abs(barrier_d(d, dhat)[1])
            for row, bb, dd, ll in zip(pt[act], pt_bodies[act], d, lam):
                out.append({"kind": "point-triangle", "bodies": tuple(int(v) for v in bb),
                            "verts": [int(v) for v in row], "d": float(dd), "lambda": float(ll)})
    if len(ee):
        D, _, _ = ee_closest(x[ee[:, 0]], x[ee[:, 1]], x[ee[:, 2]], x[ee[:, 3]])
        act = D < dhat * dhat
        if act.any():
            d = np.sqrt(D[act])
            m = mollifier(x[ee[act]], eps_x[act], 0)[0]
            lam = kappa * m * np.abs(barrier_d(d, dhat)[1])
            for row, bb, dd, ll in zip(ee[act], ee_bodies[act], d, lam):
                out.append({"kind": "edge-edge", "bodies": tuple(int(v) for v in bb),
                            "verts": [int(v) for v in row], "d": float(dd), "lambda": float(ll)})
    return out


# ---------------------------------------------------------------------------
# lagged friction (contact.py:380-524)
# ---------------------------------------------------------------------------


def empty_anchors():
    return {"verts": np.zeros((0, 4), np.int64), "gamma": np.zeros((0, 4)), "tangent": np.zeros((0, 3, 2)),
            "lam": np.zeros(0), "mu": np.zeros(0), "bodies": np.zeros((0, 2), np.int64)}


def tangent_basis(n):
    """contact.py:403-410 (argmin picks the first smallest |n_i|)."""
    ref = np.zeros_like(n)
    ref[np.arange(len(n)), np.argmin(np.abs(n), axis=1)] = 1.0
    t1 = np.cross(ref, n)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(n, t1)
    return np.stack([t1, t2], axis=2)


def friction_anchors(x, pt, ee, eps_x, pt_mu, ee_mu, pt_bodies, ee_bodies, kappa, dhat):
    """Anchors from the converged state; contact.py:413-472."""
    vs, gs, ns, ls, ms, bs = [], [], [], [], [], []
    if len(pt):
        D, bary, _ = pt_closest(x[pt[:, 0]], x[pt[:, 1]], x[pt[:, 2]], x[pt[:, 3]])
        act = D < dhat * dhat
        if act.any():
            d = np.sqrt(D[act])
            lam = kappa * np.abs(barrier_d(d, dhat)[1])
            pa = x[pt[act, 0]]
            pb = np.einsum("nk,nkj->nj", bary[act], x[pt[act, 1:]])
            ns.append((pa - pb) / d[:, None])
            vs.append(pt[act]); gs.append(np.concatenate([np.ones((int(act.sum()), 1)), -bary[act]], 1))
            ls.append(lam); ms.append(pt_mu[act]); bs.append(pt_bodies[act])
    if len(ee):
        D, s, t = ee_closest(x[ee[:, 0]], x[ee[:, 1]], x[ee[:, 2]], x[ee[:, 3]])
        act = D < dhat * dhat
        if act.any():
            d = np.sqrt(D[act])
            m = mollifier(x[ee], eps_x, 0)[0][act]
            lam = kappa * m * np.abs(barrier_d(d, dhat)[1])
            sa, ta = s[act], t[act]
            pa = (1.0 - sa)[:, None] * x[ee[act, 0]] + sa[:, None] * x[ee[act, 1]]
            pb = (1.0 - ta)[:, None] * x[ee[act, 2]] + ta[:, None] * x[ee[act, 3]]
            ns.append((pa - pb) / d[:, None])
            vs.append(ee[act]); gs.append(np.stack([1.0 - sa, sa, -(1.0 - ta), -ta], 1))
            ls.append(lam); ms.append(ee_mu[act]); bs.append(ee_bodies[act])
    if not vs:
        return empty_anchors()
    return {"verts": np.concatenate(vs), "gamma": np.concatenate(gs), "tangent": tangent_basis(np.concatenate(ns)),
            "lam": np.concatenate(ls), "mu": np.concatenate(ms), "bodies": np.concatenate(bs)}


def friction_potential(anc, x, x_prev, eps_v, dt, order=2):
    """sum mu*lam*f0(|slip|); contact.py:475-524 (blocks are PSD, not projected)."""
    nv = len(x)
    if len(anc["lam"]) == 0:
        return 0.0, np.zeros((nv, 3)), np.zeros((0, 4), np.int64), np.zeros((0, 12, 12))
    h = eps_v * dt
    V, gam, T = anc["verts"], anc["gamma"], anc["tangent"]
    u = np.einsum("nk,nkj->nj", gam, x[V] - x_prev[V])
    slip = np.einsum("nji,nj->ni", T, u)
    y = np.linalg.norm(slip, axis=1)
    f0, f1 = friction_f0_f1(y, eps_v, dt)
    sc = anc["mu"] * anc["lam"]
    E = float((sc * f0).sum())
    if order == 0:
        return E, None, None, None
    ratio = np.where(y > 1e-14, f1 / np.maximum(y, 1e-300), 2.0 / h)
    g3 = np.einsum("nij,nj->ni", T, ratio[:, None] * slip)
    grad = np.zeros((nv, 3))
    np.add.at(grad, V.reshape(-1), (sc[:, None, None] * gam[:, :, None] * g3[:, None, :]).reshape(-1, 3))
    if order < 2:
        return E, grad, V, None
    df1 = np.where(y < h, 2.0 / h - 2.0 * y / (h * h), 0.0)
    uh = np.where(y[:, None] > 1e-14, slip / np.maximum(y, 1e-300)[:, None], 0.0)
    uu = uh[:, :, None] * uh[:, None, :]
    M2 = df1[:, None, None] * uu + ratio[:, None, None] * (np.eye(2)[None] - uu)
    M3 = np.einsum("nik,nkl,njl->nij", T, M2, T)
    blk = (sc[:, None, None, None, None] * gam[:, :, None, None, None] * gam[:, None, :, None, None]
           * M3[:, None, None, :, :])
    return E, grad, V, blk.transpose(0, 1, 3, 2, 4).reshape(-1, 12, 12)


# ---------------------------------------------------------------------------
# elasticity (materials.py:43-213)
# ---------------------------------------------------------------------------


def lame(E, nu):
    """materials.py:43-49."""
    return E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))


def tet_rest(rest, tets):
    """(Dm_inv, V0, w) per tet; materials.py:73-98."""
    Dm = np.stack([rest[tets[:, k + 1]] - rest[tets[:, 0]] for k in range(3)], axis=-1)
    V0 = np.linalg.det(Dm) / 6.0
    if np.any(V0 <= 0.0):
        raise ValueError("non-positive rest volume")
    Dmi = np.linalg.inv(Dm)
    w = np.concatenate([-Dmi.sum(axis=1)[:, None, :], Dmi], axis=1)
    return Dmi, V0, w


def neo_hookean(nodes, tets, Dmi, V0, w, mu, lam, order=2, project=True):
    """Classic compressible NH energy/grad/per-tet Hessians; materials.py:116-158.

    mu/lam may be scalars or per-tet arrays.  Raises on J<=0.
    """
    Ds = np.stack([nodes[tets[:, k + 1]] - nodes[tets[:, 0]] for k in range(3)], axis=-1)
    F = Ds @ Dmi
    J = np.linalg.det(F)
    if np.any(J <= 0.0):
        raise ValueError("inverted element passed to elastic energy")
    mu = np.broadcast_to(np.asarray(mu, np.float64), J.shape)
    lam = np.broadcast_to(np.asarray(lam, np.float64), J.shape)
    A = np.linalg.inv(F).transpose(0, 2, 1)
    Ic = np.einsum("nab,nab->n", F, F)
    psi = 0.5 * mu * (Ic - 3.0) - mu * np.log(J) + 0.5 * lam * (J - 1.0) ** 2
    E = float(np.sum(V0 * psi))
    if order == 0:
        return E, None, None, V0 * psi
    P = mu[:, None, None] * F + (lam * (J - 1.0) * J - mu)[:, None, None] * A
    gt = np.einsum("nmb,ncb->nmc", w, P) * V0[:, None, None]
    grad = np.zeros((len(nodes), 3))
    np.add.at(grad, tets.reshape(-1), gt.reshape(-1, 3))
    if order < 2:
        return E, grad, None, gt
    c2 = mu - lam * (J - 1.0) * J
    c3 = lam * (2.0 * J - 1.0) * J
    dP = (mu[:, None, None, None, None] * np.einsum("ac,bd->abcd", _I3, _I3)[None]
          + c2[:, None, None, None, None] * np.einsum("nad,ncb->nabcd", A, A)
          + c3[:, None, None, None, None] * np.einsum("nab,ncd->nabcd", A, A))
    H = np.einsum("ncbCB,nmb,nMB->nmcMC", dP, w, w).reshape(-1, 12, 12) * V0[:, None, None]
    if project:
        H = spd_clamp(H)
    return E, grad, H, gt


def abd_ortho(A, kV, order=2):
    """kappa*V*||A^T A - I||_F^2 over q=(p, A rows); materials.py:161-188 (+ solver.py:509-515 projection)."""
    S = A.T @ A - _I3
    E = kV * float(np.sum(S * S))
    g = np.zeros(12)
    g[3:] = (4.0 * kV * (A @ S)).reshape(-1)
    if order < 2:
        return E, g, None
    H9 = 4.0 * kV * (np.einsum("ac,db->abcd", _I3, S) + np.einsum("ad,cb->abcd", A, A)
                     + np.einsum("ac,bd->abcd", A @ A.T, _I3)).reshape(9, 9)
    H = np.zeros((12, 12))
    H[3:, 3:] = H9
    return E, g, spd_clamp(H[None])[0]


def cauchy_stress(nodes, tets, Dmi, mu, lam):
    """Per-tet [sxx, syy, szz, sxy, syz, sxz, von Mises]; materials.py:191-205 + protocol.py:131-146."""
    Ds = np.stack([nodes[tets[:, k + 1]] - nodes[tets[:, 0]] for k in range(3)], axis=-1)
    F = Ds @ Dmi
    J = np.linalg.det(F)
    if np.any(J <= 0.0):
        raise ValueError("inverted element passed to stress computation")
    mu = np.broadcast_to(np.asarray(mu, np.float64), J.shape)
    lam = np.broadcast_to(np.asarray(lam, np.float64), J.shape)
    A = np.linalg.inv(F).transpose(0, 2, 1)
    P = mu[:, None, None] * F + (lam * (J - 1.0) * J - mu)[:, None, None] * A
    s = np.einsum("n,nab,ncb->nac", 1.0 / J, P, F)
    s = 0.5 * (s + s.transpose(0, 2, 1))
    dev = s - (np.trace(s, axis1=1, axis2=2) / 3.0)[:, None, None] * _I3
    vm = np.sqrt(1.5 * np.einsum("nab,nab->n", dev, dev))
    return np.stack([s[:, 0, 0], s[:, 1, 1], s[:, 2, 2], s[:, 0, 1], s[:, 1, 2], s[:, 0, 2], vm], 1)
