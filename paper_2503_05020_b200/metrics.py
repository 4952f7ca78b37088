"""Grasp-quality metrics D1 / D2 over the object's SDF (gripsim/pipeline/metrics.py), B200 path.

    D1 = max(0, max_p d_o(p))    penetration depth          (metrics.py:87-91)
    D2 = |max_p d_o(p)|          unsigned gripper-object gap (metrics.py:94-98)

d_o is positive inside (the geometry SDF negated once).  The gripper surface is sampled
with the reference's seeded area-weighted sampler (metrics.py:78-84); the samples are
evaluated on the GPU (grip_sdf_query: posed trilinear inside the grid, far field outside,
max-reduction).  Rigid (affine) objects reuse one rest-shape SDF per mesh, posed through the
polar rotation of the body's linear map; soft objects rebuild the SDF from the deformed
surface (sdf.build_sdf, narrow band on the GPU).  Reference quirk kept: a sample inside the
posed grid's world AABB but outside the rotated grid box gets d_o = -|0| (metrics.py:58-75).
"""

from __future__ import annotations

import hashlib

import numpy as np

from paper_2503_05020_b200 import _native as nv
from paper_2503_05020_b200 import sdf as sdfm


class PosedSdf:
    """Rest-shape SDF queried through a rigid pose (metrics.py:21-45)."""

    def __init__(self, base, rotation, translation):
        self.base = base
        self.rotation = np.asarray(rotation, np.float64)
        self.translation = np.asarray(translation, np.float64)
        self.spacing = base.spacing

    def bounds(self):
        lo, hi = self.base.bounds()
        corners = np.array([[a, b, c] for a in (lo[0], hi[0]) for b in (lo[1], hi[1]) for c in (lo[2], hi[2])])
        world = corners @ self.rotation.T + self.translation
        return world.min(axis=0), world.max(axis=0)


def polar_rotation(A):
    """metrics.py:48-54."""
    U, _, Vt = np.linalg.svd(A)
    R = U @ Vt
    if np.linalg.det(R) < 0:
        U[:, -1] *= -1
        R = U @ Vt
    return R


def sample_surfaces(surfaces, n_samples, seed):
    """metrics.py:78-84; surfaces = [(vertices, triangles), ...]."""
    rng = np.random.default_rng(seed)
    areas = np.array([sdfm.triangle_areas(v, t).sum() for v, t in surfaces])
    counts = np.maximum(1, np.floor(n_samples * areas / areas.sum()).astype(int))
    counts[0] += n_samples - counts.sum()
    return np.concatenate([sdfm.sample_surface(v, t, int(c), rng) for (v, t), c in zip(surfaces, counts)])


def signed_inside_max(sdf, points, want_values=False):
    """max over points of d_o (metrics.py:58-75), on the GPU; also every d_o if asked."""
    pts = np.atleast_2d(np.asarray(points, np.float64))
    if isinstance(sdf, PosedSdf):
        base = sdf.base
        wlo, whi = sdf.bounds()
        return nv.sdf_query(base.values, base.origin, base.spacing, pts, rot=sdf.rotation, trans=sdf.translation,
                            world_lo=wlo, world_hi=whi, want_values=want_values)
    return nv.sdf_query(sdf.values, sdf.origin, sdf.spacing, pts, want_values=want_values)


def _surface_tris(rec):
    body = rec["body"]
    if rec["kind"] == "soft":
        surf, _ = body.mesh.boundary_surface()
        return np.asarray(surf.triangles, np.int64)
    return np.asarray(body.surface.triangles, np.int64)


def gripper_surfaces_from_env(env, gripper_bodies, x=None):
    """metrics.py:101-115: (vertices, triangles) of each gripper body at the current state
    (or at node positions x)."""
    sv = env.surface_positions(x)
    out = []
    for bid in gripper_bodies:
        rec = env.records[bid]
        a = rec["surf0"]
        out.append((sv[a:a + rec["n_sv"]], _surface_tris(rec)))
    return out


class SdfCache:
    """Rest-shape SDFs keyed by mesh content (multienv.AssetCache semantics)."""

    def __init__(self):
        self._d = {}

    @staticmethod
    def key_of(*arrays):
        h = hashlib.sha256()
        for a in arrays:
            a = np.ascontiguousarray(a)
            h.update(str(a.dtype).encode() + str(a.shape).encode() + a.tobytes())
        return h.hexdigest()

    def get_or_build(self, key, builder):
        if key not in self._d:
            self._d[key] = builder()
        return self._d[key]


def object_sdf_from_env(env, object_body, resolution=128, cache=None):
    """metrics.py:130-160."""
    rec = env.records[object_body]
    tris = _surface_tris(rec)
    if rec["kind"] == "affine":
        xi = np.asarray(rec["xi"], np.float64)
        build = lambda: sdfm.build_sdf(xi, tris, resolution=resolution)  # noqa: E731
        base = cache.get_or_build(SdfCache.key_of(xi, tris, np.array([resolution])), build) if cache else build()
        q = env.x[rec["dof0"]:rec["dof0"] + 12]
        return PosedSdf(base, polar_rotation(q[3:].reshape(3, 3)), q[:3])
    sv = env.surface_positions()
    verts = sv[rec["surf0"]:rec["surf0"] + rec["n_sv"]]
    build = lambda: sdfm.build_sdf(verts, tris, resolution=resolution)  # noqa: E731
    return cache.get_or_build(SdfCache.key_of(verts, tris, np.array([resolution])), build) if cache else build()


def trial_quality_metrics(env, object_body, gripper_bodies, resolution=128, n_samples=50_000, seed=0, cache=None):
    """(D1, D2, grid spacing) of the env's current state (metrics.py:163-171)."""
    sdf = object_sdf_from_env(env, object_body, resolution=resolution, cache=cache)
    pts = sample_surfaces(gripper_surfaces_from_env(env, gripper_bodies), n_samples, seed)
    dmax, _ = signed_inside_max(sdf, pts)
    return float(max(0.0, dmax)), float(abs(dmax)), float(sdf.spacing.max())
