"""Oracle geometry: closest points, squared-distance derivatives, broad phase, CCD.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
/root/reference/pkg/src/gripsim/geometry/{distances,broadphase,ccd}.py.
All arrays are float64; stencil arrays are (n, 3) per vertex slot.
"""

from __future__ import annotations

import numpy as np

EPS_DIST = 1e-14  # ccd.py:16


def _dot(a, b):
    return np.einsum("...i,...i->...", a, b)


# ---------------------------------------------------------------------------
# closest points (distances.py:61-152)
# ---------------------------------------------------------------------------


def pt_closest(p, t0, t1, t2):
    """Ericson point-triangle closest point; distances.py:61-121.

    Region codes: 0..2 vertex t0/t1/t2, 3 edge t0t1, 4 edge t1t2, 5 edge t2t0,
    6 face.  Tests are applied in the reference's priority order
    (vertex t0, t1, t2, edge 3, edge 5, edge 4, face) so ties resolve the same.
    """
    p, t0, t1, t2 = (np.atleast_2d(np.asarray(a, np.float64)) for a in (p, t0, t1, t2))
    ab, ac = t1 - t0, t2 - t0
    ap, bp, cp = p - t0, p - t1, p - t2
    d1, d2 = _dot(ab, ap), _dot(ac, ap)
    d3, d4 = _dot(ab, bp), _dot(ac, bp)
    d5, d6 = _dot(ab, cp), _dot(ac, cp)
    va = d3 * d6 - d5 * d4
    vb = d5 * d2 - d1 * d6
    vc = d1 * d4 - d3 * d2
    with np.errstate(divide="ignore", invalid="ignore"):
        s_ab = np.where(d1 != d3, d1 / (d1 - d3), 0.0)
        s_ac = np.where(d2 != d6, d2 / (d2 - d6), 0.0)
        den_bc = (d4 - d3) + (d5 - d6)
        s_bc = np.where(den_bc != 0.0, (d4 - d3) / den_bc, 0.0)
        den = va + vb + vc
        fv = np.where(den != 0.0, vb / den, 0.0)
        fw = np.where(den != 0.0, vc / den, 0.0)
    conds = [
        (d1 <= 0.0) & (d2 <= 0.0),
        (d3 >= 0.0) & (d4 <= d3),
        (d6 >= 0.0) & (d5 <= d6),
        (vc <= 0.0) & (d1 >= 0.0) & (d3 <= 0.0),
        (vb <= 0.0) & (d2 >= 0.0) & (d6 <= 0.0),
        (va <= 0.0) & (d4 - d3 >= 0.0) & (d5 - d6 >= 0.0),
    ]
    codes = [0, 1, 2, 3, 5, 4]
    region = np.select(conds, codes, default=6).astype(np.int64)
    zero = np.zeros_like(d1)
    one = np.ones_like(d1)
    b0 = np.select(conds, [one, zero, zero, 1.0 - s_ab, 1.0 - s_ac, zero], default=1.0 - fv - fw)
    b1 = np.select(conds, [zero, one, zero, s_ab, zero, 1.0 - s_bc], default=fv)
    b2 = np.select(conds, [zero, zero, one, zero, s_ac, s_bc], default=fw)
    bary = np.stack([b0, b1, b2], axis=1)
    closest = b0[:, None] * t0 + b1[:, None] * t1 + b2[:, None] * t2
    diff = p - closest
    return _dot(diff, diff), bary, region


def ee_closest(a0, a1, b0, b1):
    """Clamped segment-segment closest parameters; distances.py:124-152."""
    a0, a1, b0, b1 = (np.atleast_2d(np.asarray(a, np.float64)) for a in (a0, a1, b0, b1))
    d1, d2, r = a1 - a0, b1 - b0, a0 - b0
    a, e = _dot(d1, d1), _dot(d2, d2)
    f, c, b = _dot(d2, r), _dot(d1, r), _dot(d1, d2)
    den = a * e - b * b
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(den > 0.0, np.clip((b * f - c * e) / den, 0.0, 1.0), 0.0)
        t = (b * s + f) / e
        s = np.where(t < 0.0, np.clip(-c / a, 0.0, 1.0),
                     np.where(t > 1.0, np.clip((b - c) / a, 0.0, 1.0), s))
    t = np.clip(t, 0.0, 1.0)
    diff = (a0 + s[:, None] * d1) - (b0 + t[:, None] * d2)
    return _dot(diff, diff), s, t


# ---------------------------------------------------------------------------
# squared-distance derivatives (distances.py:160-382), in reduced variables
# ---------------------------------------------------------------------------

_I3 = np.eye(3)


def _outer(a, b):
    return a[:, :, None] * b[:, None, :]


def pp_derivs(a, b):
    """D=|a-b|^2 over (a, b); distances.py:160-174.  Returns grad (n,6)."""
    d = a - b
    return np.concatenate([2.0 * d, -2.0 * d], axis=1)


def pe_derivs(p, e0, e1):
    """Interior point-edge squared distance gradient over (p, e0, e1); distances.py:177-227.

    Only the gradient is returned: the reference never lands this Hessian in
    the stencil layout (contact.py:116-125, see contact_terms).
    """
    w, u = p - e0, e1 - e0
    q = _dot(u, u)
    sq = _dot(w, u) / q
    gw = 2.0 * w - 2.0 * sq[:, None] * u
    gu = -2.0 * sq[:, None] * w + 2.0 * (sq * sq)[:, None] * u
    return np.concatenate([gw, -gw - gu, gu], axis=1)


def _skew(c):
    z = np.zeros(len(c))
    return np.stack([
        np.stack([z, -c[:, 2], c[:, 1]], 1),
        np.stack([c[:, 2], z, -c[:, 0]], 1),
        np.stack([-c[:, 1], c[:, 0], z], 1),
    ], 1)


def plane_derivs(w, u, v):
    """D=(w.n)^2/|n|^2, n=u x v: grad (n,9) and Hessian (n,9,9) over (w,u,v); distances.py:230-277."""
    n = np.cross(u, v)
    iq = 1.0 / _dot(n, n)
    sq = _dot(w, n) * iq
    gw = 2.0 * sq[:, None] * n
    gn = 2.0 * sq[:, None] * w - 2.0 * (sq * sq)[:, None] * n
    nn, nw, ww = _outer(n, n), _outer(n, w), _outer(w, w)
    Hww = 2.0 * iq[:, None, None] * nn
    Hwn = (2.0 * iq[:, None, None] * nw + 2.0 * sq[:, None, None] * _I3
           - 4.0 * (sq * iq)[:, None, None] * nn)
    Hnn = (2.0 * iq[:, None, None] * ww - 4.0 * (sq * iq)[:, None, None] * (nw + nw.transpose(0, 2, 1))
           - 2.0 * (sq * sq)[:, None, None] * _I3 + 8.0 * (sq * sq * iq)[:, None, None] * nn)
    Ju, Jv = -_skew(v), _skew(u)          # dn/du, dn/dv
    gu = np.einsum("nki,nk->ni", Ju, gn)
    gv = np.einsum("nki,nk->ni", Jv, gn)
    g = np.concatenate([gw, gu, gv], axis=1)
    H = np.empty((len(w), 9, 9))
    H[:, 0:3, 0:3] = Hww
    H[:, 0:3, 3:6] = Hwn @ Ju
    H[:, 0:3, 6:9] = Hwn @ Jv
    H[:, 3:6, 3:6] = Ju.transpose(0, 2, 1) @ Hnn @ Ju
    H[:, 6:9, 6:9] = Jv.transpose(0, 2, 1) @ Hnn @ Jv
    H[:, 3:6, 6:9] = Ju.transpose(0, 2, 1) @ Hnn @ Jv - _skew(gn)
    H[:, 3:6, 0:3] = H[:, 0:3, 3:6].transpose(0, 2, 1)
    H[:, 6:9, 0:3] = H[:, 0:3, 6:9].transpose(0, 2, 1)
    H[:, 6:9, 3:6] = H[:, 3:6, 6:9].transpose(0, 2, 1)
    return g, H


# incidence of (w, u, v) on the 4 stencil points, as 3x12 signed selector rows
_PT_CHAIN = np.array([[1, -1, 0, 0], [0, -1, 1, 0], [0, -1, 0, 1]], np.float64)   # w=p-t0, u=t1-t0, v=t2-t0
_EE_CHAIN = np.array([[-1, 0, 1, 0], [-1, 1, 0, 0], [0, 0, -1, 1]], np.float64)   # w=b0-a0, u=a1-a0, v=b1-b0
_PT_C = np.kron(_PT_CHAIN, _I3)   # (9, 12)
_EE_C = np.kron(_EE_CHAIN, _I3)


def pt_plane(x4):
    """Interior point-triangle over the 4-point layout; distances.py:310-325."""
    g9, H9 = plane_derivs(x4[:, 0] - x4[:, 1], x4[:, 2] - x4[:, 1], x4[:, 3] - x4[:, 1])
    return g9 @ _PT_C, np.einsum("ia,nij,jb->nab", _PT_C, H9, _PT_C)


def ee_plane(x4):
    """Interior edge-edge over the 4-point layout; distances.py:328-343."""
    g9, H9 = plane_derivs(x4[:, 2] - x4[:, 0], x4[:, 1] - x4[:, 0], x4[:, 3] - x4[:, 2])
    return g9 @ _EE_C, np.einsum("ia,nij,jb->nab", _EE_C, H9, _EE_C)


def cross_norm_sq(x4):
    """c=|u x v|^2 by the Lagrange identity with grad/Hessian; distances.py:346-382."""
    u, v = x4[:, 1] - x4[:, 0], x4[:, 3] - x4[:, 2]
    qu, qv, s = _dot(u, u), _dot(v, v), _dot(u, v)
    c = qu * qv - s * s
    gu = 2.0 * qv[:, None] * u - 2.0 * s[:, None] * v
    gv = 2.0 * qu[:, None] * v - 2.0 * s[:, None] * u
    Huu = 2.0 * qv[:, None, None] * _I3 - 2.0 * _outer(v, v)
    Hvv = 2.0 * qu[:, None, None] * _I3 - 2.0 * _outer(u, u)
    Huv = 4.0 * _outer(u, v) - 2.0 * _outer(v, u) - 2.0 * s[:, None, None] * _I3
    g = np.concatenate([-gu, gu, -gv, gv], axis=1)
    sgn = np.array([-1.0, 1.0, -1.0, 1.0])
    H = np.empty((len(u), 12, 12))
    blk = {(0, 0): Huu, (0, 1): Huv, (1, 0): Huv.transpose(0, 2, 1), (1, 1): Hvv}
    for k in range(4):
        for m in range(4):
            H[:, 3 * k:3 * k + 3, 3 * m:3 * m + 3] = sgn[k] * sgn[m] * blk[(k // 2, m // 2)]
    return c, g, H


# ---------------------------------------------------------------------------
# broad phase (broadphase.py:101-214): exact predicate set, brute force
# ---------------------------------------------------------------------------


_HB = 20
_HOFF = 1 << (_HB - 1)


def _cell_keys(cells):
    """Pack integer cells into one int64 key per row (broadphase.py:57-67, single env)."""
    c = cells + _HOFF
    if np.any((c < 0) | (c >= (1 << _HB))):
        raise ValueError("scene exceeds spatial hash coordinate range")
    return (c[:, 0] << (2 * _HB)) | (c[:, 1] << _HB) | c[:, 2]


def _boxes_to_cells(lo, hi):
    """(row id, cell) for every integer cell of every box [lo, hi] (broadphase.py:70-85)."""
    span = hi - lo + 1
    cnt = span.prod(axis=1)
    rows = np.repeat(np.arange(len(lo)), cnt)
    local = np.arange(int(cnt.sum())) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    sy, sz = np.repeat(span[:, 1], cnt), np.repeat(span[:, 2], cnt)
    off = np.stack([local // (sz * sy), (local // sz) % sy, local % sz], axis=1)
    return rows, np.repeat(lo, cnt, axis=0) + off


def _hash_pairs(tab_lo, tab_hi, q_lo, q_hi, inv):
    """All (query row, table row) pairs sharing a cell; broadphase.py:88-98."""
    t_rows, t_cells = _boxes_to_cells(np.floor(tab_lo * inv).astype(np.int64), np.floor(tab_hi * inv).astype(np.int64))
    tk = _cell_keys(t_cells)
    order = np.argsort(tk, kind="stable")
    tk, t_rows = tk[order], t_rows[order]
    q_rows, q_cells = _boxes_to_cells(np.floor(q_lo * inv).astype(np.int64), np.floor(q_hi * inv).astype(np.int64))
    qk = _cell_keys(q_cells)
    left = np.searchsorted(tk, qk, "left")
    cnt = np.searchsorted(tk, qk, "right") - left
    tot = int(cnt.sum())
    if tot == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    flat = np.arange(tot) - np.repeat(np.cumsum(cnt) - cnt, cnt) + np.repeat(left, cnt)
    return np.repeat(q_rows, cnt), t_rows[flat]


def broad_phase(x, tris, edges, vbody, pair_ok, r):
    """Candidate stencils of ONE environment at search radius r; broadphase.py:101-214.

    Pairs are generated by the reference's spatial hash (cell = max(r, median
    triangle extent), tight insertion, r-inflated queries) and membership is
    decided by its exact predicates (:177-183 PT, :202-209 EE).  Output order
    is canonical: sorted by (v, tri) and (edge i, edge j).
    Returns dict(pt (n,4), ee (m,4), ee_edges (m,2), pt_tri (n,)).
    """
    if r <= 0.0:
        raise ValueError("search_radius must be positive")
    out = {"pt": np.zeros((0, 4), np.int64), "pt_tri": np.zeros(0, np.int64),
           "ee": np.zeros((0, 4), np.int64), "ee_edges": np.zeros((0, 2), np.int64)}
    ext = [r]
    if len(tris):
        tv = x[tris]
        ext.append(float(np.median((tv.max(axis=1) - tv.min(axis=1)).max(axis=1))))
    inv = 1.0 / max(max(ext), 1e-9)
    if len(tris) and len(x):
        tlo, thi = tv.min(axis=1), tv.max(axis=1)
        vi, ti = _hash_pairs(tlo, thi, x - r, x + r, inv)
        if len(vi):
            nt = np.int64(len(tris))
            u = np.unique(vi * nt + ti)
            vi, ti = u // nt, u % nt
            tr = tris[ti]
            keep = (tr[:, 0] != vi) & (tr[:, 1] != vi) & (tr[:, 2] != vi)
            keep &= pair_ok[vbody[vi], vbody[tr[:, 0]]]
            keep &= np.all(x[vi] >= tlo[ti] - r, axis=1) & np.all(x[vi] <= thi[ti] + r, axis=1)
            vi, ti = vi[keep], ti[keep]
            out["pt"] = np.concatenate([vi[:, None], tris[ti]], axis=1)
            out["pt_tri"] = ti
    if len(edges):
        ev = x[edges]
        lo, hi = ev.min(axis=1), ev.max(axis=1)
        ei, ej = _hash_pairs(lo, hi, lo - r, hi + r, inv)
        m = ej > ei
        ei, ej = ei[m], ej[m]
        if len(ei):
            ne = np.int64(len(edges))
            u = np.unique(ei * ne + ej)
            ei, ej = u // ne, u % ne
            ea, eb = edges[ei], edges[ej]
            keep = ((ea[:, 0] != eb[:, 0]) & (ea[:, 0] != eb[:, 1]) & (ea[:, 1] != eb[:, 0]) & (ea[:, 1] != eb[:, 1]))
            keep &= pair_ok[vbody[ea[:, 0]], vbody[eb[:, 0]]]
            keep &= np.all(hi[ej] >= lo[ei] - r, axis=1) & np.all(lo[ej] <= hi[ei] + r, axis=1)
            ei, ej = ei[keep], ej[keep]
            out["ee_edges"] = np.stack([ei, ej], axis=1)
            out["ee"] = np.concatenate([edges[ei], edges[ej]], axis=1)
    return out


def broad_phase_brute(x, tris, edges, vbody, pair_ok, r):
    """Same predicate set by exhaustive pair testing (test helper, small scenes only)."""
    out = {"pt": np.zeros((0, 4), np.int64), "ee": np.zeros((0, 4), np.int64)}
    if len(tris):
        tv = x[tris]
        lo, hi = tv.min(axis=1) - r, tv.max(axis=1) + r
        ins = np.all((x[:, None] >= lo[None]) & (x[:, None] <= hi[None]), axis=2)
        vi = np.arange(len(x))[:, None]
        ins &= (tris[None, :, 0] != vi) & (tris[None, :, 1] != vi) & (tris[None, :, 2] != vi)
        ins &= pair_ok[vbody[:, None], vbody[tris[:, 0]][None, :]]
        v, t = np.nonzero(ins)
        out["pt"] = np.concatenate([v[:, None], tris[t]], axis=1)
    if len(edges):
        ev = x[edges]
        lo, hi = ev.min(axis=1), ev.max(axis=1)
        ii, jj = np.triu_indices(len(edges), k=1)
        ok = np.all((hi[jj] >= lo[ii] - r) & (lo[jj] <= hi[ii] + r), axis=1)
        ii, jj = ii[ok], jj[ok]
        ea, eb = edges[ii], edges[jj]
        ok = ((ea[:, 0] != eb[:, 0]) & (ea[:, 0] != eb[:, 1]) & (ea[:, 1] != eb[:, 0]) & (ea[:, 1] != eb[:, 1]))
        ok &= pair_ok[vbody[ea[:, 0]], vbody[eb[:, 0]]]
        out["ee"] = np.concatenate([edges[ii[ok]], edges[jj[ok]]], axis=1)
    return out


# ---------------------------------------------------------------------------
# CCD and inversion filters (ccd.py:34-204)
# ---------------------------------------------------------------------------


class IntersectionError(RuntimeError):
    """ccd.py:19."""


def _stencil_dist(q, split):
    if split == 1:
        D, _, _ = pt_closest(q[:, 0], q[:, 1], q[:, 2], q[:, 3])
    else:
        D, _, _ = ee_closest(q[:, 0], q[:, 1], q[:, 2], q[:, 3])
    return np.sqrt(D)


def ccd_max_step(x, p, pt, ee, scaling=0.9, max_iters=32, min_separation=0.0):
    """Additive conservative advancement, per stencil, min over the env; ccd.py:34-95."""
    pt = np.asarray(pt, np.int64).reshape(-1, 4)
    ee = np.asarray(ee, np.int64).reshape(-1, 4)
    if len(pt) == 0 and len(ee) == 0:
        return 1.0
    alpha = 1.0
    for idx, split in ((pt, 1), (ee, 2)):
        if not len(idx):
            continue
        xs, ps = x[idx], p[idx]
        rel = ps - ps.mean(axis=1, keepdims=True)
        nrm = np.linalg.norm(rel, axis=2)
        lp = nrm[:, :split].max(axis=1) + nrm[:, split:].max(axis=1)
        t = np.zeros(len(idx))
        d = _stencil_dist(xs, split)
        if np.any(d <= EPS_DIST):
            raise IntersectionError("CCD called from an intersecting or touching state")
        gap = min_separation * d
        active = lp > 0.0
        t[~active] = 1.0
        for _ in range(max_iters):
            if not active.any():
                break
            a = np.nonzero(active)[0]
            t_new = t[a] + scaling * np.maximum(d[a] - gap[a], 0.0) / lp[a]
            fin = t_new >= 1.0
            t[a[fin]] = 1.0
            a = a[~fin]
            active[:] = False
            active[a] = True
            if not len(a):
                break
            t[a] = t_new[~fin]
            d[a] = _stencil_dist(xs[a] + t[a][:, None, None] * ps[a], split)
            stalled = d[a] <= gap[a] + EPS_DIST
            active[a[stalled]] = False
        alpha = min(alpha, float(t.min()))
    return max(alpha, 0.0)


def _det3(M):
    return np.linalg.det(M)


def _cof(M):
    """Cofactor matrix (columns = cross products of column pairs); ccd.py:98-103."""
    c0 = np.cross(M[..., :, 1], M[..., :, 2], axis=-1)
    c1 = np.cross(M[..., :, 2], M[..., :, 0], axis=-1)
    c2 = np.cross(M[..., :, 0], M[..., :, 1], axis=-1)
    return np.stack([c0, c1, c2], axis=-1)


def cubic_smallest_root(c0, c1, c2, c3, t_max=1.0):
    """Smallest real root in (1e-12, t_max] of c0+c1 t+c2 t^2+c3 t^3 else t_max+1; ccd.py:106-163."""
    c0, c1, c2, c3 = np.broadcast_arrays(*(np.atleast_1d(np.asarray(c, np.float64)) for c in (c0, c1, c2, c3)))
    n = len(c0)
    roots = np.full((n, 3), np.inf)
    scale = np.maximum.reduce([np.abs(c0), np.abs(c1), np.abs(c2), np.abs(c3), np.full(n, 1e-30)])
    cub = np.abs(c3) > 1e-14 * scale
    quad = ~cub & (np.abs(c2) > 1e-14 * scale)
    lin = ~cub & ~quad & (np.abs(c1) > 1e-14 * scale)
    roots[lin, 0] = -c0[lin] / c1[lin]
    if quad.any():
        a, b, c = c2[quad], c1[quad], c0[quad]
        disc = b * b - 4.0 * a * c
        sq = np.sqrt(np.maximum(disc, 0.0))
        roots[quad, 0] = np.where(disc >= 0.0, (-b - sq) / (2.0 * a), np.inf)
        roots[quad, 1] = np.where(disc >= 0.0, (-b + sq) / (2.0 * a), np.inf)
    if cub.any():
        a = c2[cub] / c3[cub]
        b = c1[cub] / c3[cub]
        c = c0[cub] / c3[cub]
        p = b - a * a / 3.0
        q = 2.0 * a ** 3 / 27.0 - a * b / 3.0 + c
        disc = (q / 2.0) ** 2 + (p / 3.0) ** 3
        blk = np.full((len(a), 3), np.inf)
        one = disc > 0.0
        if one.any():
            sq = np.sqrt(disc[one])
            blk[one, 0] = np.cbrt(-q[one] / 2.0 + sq) + np.cbrt(-q[one] / 2.0 - sq) - a[one] / 3.0
        thr = ~one
        if thr.any():
            pm = np.minimum(p[thr], -1e-300)
            rr = np.sqrt(-pm / 3.0)
            phi = np.arccos(np.clip(3.0 * q[thr] / (2.0 * pm * rr), -1.0, 1.0))
            for k in range(3):
                blk[thr, k] = 2.0 * rr * np.cos((phi - 2.0 * np.pi * k) / 3.0) - a[thr] / 3.0
        roots[cub] = blk
    roots = np.where((roots > 1e-12) & (roots <= t_max), roots, np.inf)
    best = roots.min(axis=1)
    return np.where(np.isfinite(best), best, t_max + 1.0)


def pencil_step(M0, dM, scaling=0.9):
    """Step keeping det(M0 + t dM) > 0 for every pencil; ccd.py:166-188."""
    M0 = np.asarray(M0, np.float64).reshape(-1, 3, 3)
    dM = np.asarray(dM, np.float64).reshape(-1, 3, 3)
    det0 = _det3(M0)
    if np.any(det0 <= 0.0):
        raise IntersectionError("step filter called with non-positive determinant state")
    c1 = np.einsum("nij,nij->n", _cof(M0), dM)
    c2 = np.einsum("nij,nij->n", _cof(dM), M0)
    t = cubic_smallest_root(det0, c1, c2, _det3(dM), 1.0)
    t_min = float(t.min())
    if t_min > 1.0:
        return 1.0
    alpha = scaling * t_min
    for _ in range(60):
        if np.all(_det3(M0 + alpha * dM) > 0.0):
            return alpha
        alpha *= 0.5
    return 0.0


def tet_filter(nodes, p, tets, scaling=0.9):
    """Inversion step bound over all tets; ccd.py:191-204."""
    if len(tets) == 0 or not np.any(p[tets]):
        return 1.0
    M0 = np.stack([nodes[tets[:, k]] - nodes[tets[:, 0]] for k in (1, 2, 3)], axis=-1)
    dM = np.stack([p[tets[:, k]] - p[tets[:, 0]] for k in (1, 2, 3)], axis=-1)
    return pencil_step(M0, dM, scaling)
