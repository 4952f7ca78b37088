"""Grid signed distance fields for the D1/D2 metrics (gripsim/geometry/sdf.py), B200 path.

Same grid, same far field, same sign labelling as the reference's ``build_sdf``
(sdf.py:117-178): negative inside; the far field is the distance to a dense seeded surface
point cloud signed by a leak-free flood fill of the cells no triangle cuts; the narrow
band (cloud distance <= band_cells * h, or a cut cell) is the exact point-triangle distance
signed by the angle-weighted pseudonormal of the closest feature.

What runs where: the grid, the seeded cloud (numpy's generator, the reference's call
sequence) and the flood fill (scipy.ndimage.label) are host preprocessing.  On the GPU:
the far field -- the exact nearest cloud point of every grid node (the reference's cKDTree;
here a Morton-ordered box tree walked per node, grip_sdf_nn) -- and the narrow band -- the
reference's costly part, a Python loop over kd-tree candidates with certificates
(sdf.py:181-241), here one kernel over all band points against all triangles
(grip_sdf_exact).  Queries (trilinear, posed) run on the GPU too (metrics.py, grip_sdf_query).
"""

from __future__ import annotations

import numpy as np

from paper_2503_05020_b200 import _native as nv

SDF_MAGIC = b"GRIPSDF1"


def triangle_areas(v, t):
    """mesh.py:61-65."""
    n = np.cross(v[t[:, 1]] - v[t[:, 0]], v[t[:, 2]] - v[t[:, 0]])
    return 0.5 * np.linalg.norm(n, axis=1)


def triangle_normals(v, t):
    """mesh.py:67-70."""
    n = np.cross(v[t[:, 1]] - v[t[:, 0]], v[t[:, 2]] - v[t[:, 0]])
    return n / np.linalg.norm(n, axis=1, keepdims=True)


def vertex_normals(v, t):
    """Angle-weighted vertex pseudonormals (mesh.py:104-115)."""
    fn = triangle_normals(v, t)
    out = np.zeros_like(v)
    for k in range(3):
        a = v[t[:, (k + 1) % 3]] - v[t[:, k]]
        b = v[t[:, (k + 2) % 3]] - v[t[:, k]]
        cosang = np.einsum("ij,ij->i", a, b) / (np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1))
        np.add.at(out, t[:, k], np.arccos(np.clip(cosang, -1.0, 1.0))[:, None] * fn)
    return out / np.maximum(np.linalg.norm(out, axis=1, keepdims=True), 1e-300)


def sample_surface(v, t, n, rng):
    """Area-weighted uniform samples (mesh.py:117-130), the reference's generator calls."""
    areas = triangle_areas(v, t)
    tri = rng.choice(len(t), size=n, p=areas / areas.sum())
    r1 = np.sqrt(rng.random(n))
    r2 = rng.random(n)
    w0, w1, w2 = 1.0 - r1, r1 * (1.0 - r2), r1 * r2
    tt = t[tri]
    return w0[:, None] * v[tt[:, 0]] + w1[:, None] * v[tt[:, 1]] + w2[:, None] * v[tt[:, 2]]


def is_watertight(t):
    """mesh.py:81-94: every edge shared by exactly two consistently oriented triangles."""
    directed = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    _, counts = np.unique(np.sort(directed, axis=1), axis=0, return_counts=True)
    if np.any(counts != 2):
        return False
    _, dcounts = np.unique(directed, axis=0, return_counts=True)
    return bool(np.all(dcounts == 1))


def feature_pseudonormals(v, t):
    """Face normals, per-(triangle, edge) edge pseudonormals, vertex pseudonormals (sdf.py:98-114).
    Edge k of a triangle is (k, k+1 mod 3), the reference's region order 3, 4, 5."""
    fn = triangle_normals(v, t)
    vn = vertex_normals(v, t)
    keys = np.sort(np.stack([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]], axis=1), axis=2).reshape(-1, 2)
    uniq, inv = np.unique(keys, axis=0, return_inverse=True)
    acc = np.zeros((len(uniq), 3))
    # the reference accumulates each edge's face normals in triangle order
    for j, f in zip(inv.reshape(-1), np.repeat(fn, 3, axis=0)):
        acc[j] += f
    en = acc / np.maximum(np.linalg.norm(acc, axis=1, keepdims=True), 1e-300)
    return fn, en[inv.reshape(-1)].reshape(len(t), 3, 3), vn


class Sdf:
    """Sampled signed distance grid (sdf.py:24-60)."""

    def __init__(self, origin, spacing, values, source=""):
        self.origin = np.asarray(origin, np.float64).reshape(3)
        self.spacing = np.asarray(spacing, np.float64).reshape(3)
        self.values = np.ascontiguousarray(values, np.float64)
        self.source = source

    @property
    def resolution(self):
        return self.values.shape

    def bounds(self):
        return self.origin.copy(), self.origin + self.spacing * (np.array(self.values.shape) - 1)

    def query(self, points):
        """Trilinear signed distance at points inside the grid (sdf.py:62-87), on the GPU."""
        pts = np.atleast_2d(np.asarray(points, np.float64))
        lo, hi = self.bounds()
        if np.any(pts < lo - 1e-9 * self.spacing) or np.any(pts > hi + 1e-9 * self.spacing):
            raise ValueError("query point outside SDF grid bounds")
        _, d_o = nv.sdf_query(self.values, self.origin, self.spacing, pts, want_values=True)
        return -d_o


def build_sdf(vertices, triangles, resolution=128, padding_cells=4, band_cells=4.0, seed=0, timings=None):
    """The reference's build_sdf (sdf.py:117-178) with the narrow band on the GPU.
    timings: optional dict that receives the wall time of each phase (s)."""
    import time

    from scipy import ndimage

    clock = [time.perf_counter()]

    def lap(name):
        if timings is not None:
            now = time.perf_counter()
            timings[name] = timings.get(name, 0.0) + now - clock[0]
            clock[0] = now

    v = np.asarray(vertices, np.float64).reshape(-1, 3)
    t = np.asarray(triangles, np.int64).reshape(-1, 3)
    if not is_watertight(t):
        raise ValueError("SDF requires a watertight surface")
    lo, hi = v.min(axis=0), v.max(axis=0)
    extent = hi - lo
    h = float(extent.max()) / float(resolution)
    dims = np.ceil(extent / h).astype(np.int64) + 1 + 2 * padding_cells
    origin = lo - padding_cells * h
    X, Y, Z = np.meshgrid(*(origin[a] + h * np.arange(dims[a]) for a in range(3)), indexing="ij")
    pts = np.stack([X, Y, Z], axis=-1).reshape(-1, 3)
    lap("grid")

    rng = np.random.default_rng(seed)
    n_cloud = int(min(400_000, max(20_000, 4.0 * triangle_areas(v, t).sum() / (h * h))))
    cloud = np.concatenate([sample_surface(v, t, n_cloud, rng), v])
    lap("cloud")
    d_cloud = nv.sdf_nn(pts, cloud)   # exact nearest cloud point on the GPU (the reference: cKDTree)
    lap("cloud_nn")

    occupied = np.zeros(tuple(dims), dtype=bool)
    tv = v[t]
    tlo = np.clip(((tv.min(axis=1) - origin) / h).astype(np.int64), 0, dims - 1)
    thi = np.clip(np.ceil((tv.max(axis=1) - origin) / h).astype(np.int64), 0, dims - 1)
    for a, b in zip(tlo, thi):
        occupied[a[0]:b[0] + 1, a[1]:b[1] + 1, a[2]:b[2] + 1] = True
    labels, _ = ndimage.label(~occupied)
    faces = np.concatenate([labels[0].ravel(), labels[-1].ravel(), labels[:, 0].ravel(), labels[:, -1].ravel(),
                            labels[:, :, 0].ravel(), labels[:, :, -1].ravel()])
    boundary = np.unique(faces)
    outside = np.isin(labels, boundary[boundary != 0])
    lap("flood_fill")
    values = np.where(outside.reshape(-1), 1.0, -1.0) * d_cloud
    band = (d_cloud <= band_cells * h) | occupied.reshape(-1)
    if band.any():
        fn, en, vn = feature_pseudonormals(v, t)
        lap("pseudonormals")
        values[band] = nv.sdf_exact(pts[band], v, t, fn, en, vn)
        lap("band_gpu")
        if timings is not None:
            timings["band_points"] = int(band.sum())
    return Sdf(origin, np.full(3, h), values.reshape(tuple(dims)), source=f"grid{resolution}")


def save_sdf(sdf, path):
    """sdf.py:244-252."""
    with open(path, "wb") as f:
        f.write(SDF_MAGIC)
        f.write(np.array([*[float(r) for r in sdf.values.shape], *sdf.origin, *sdf.spacing], "<f8").tobytes())
        f.write(np.ascontiguousarray(sdf.values, "<f8").tobytes())


def load_sdf(path):
    """sdf.py:255-265."""
    raw = open(path, "rb").read()
    if raw[:8] != SDF_MAGIC:
        raise ValueError(f"bad SDF magic: {raw[:8]!r}")
    hdr = np.frombuffer(raw, "<f8", 9, 8)
    dims = tuple(int(x) for x in hdr[:3])
    vals = np.frombuffer(raw, "<f8", dims[0] * dims[1] * dims[2], 80).reshape(dims)
    return Sdf(hdr[3:6].copy(), hdr[6:9].copy(), vals.copy())
