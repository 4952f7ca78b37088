"""Surfaces, tet meshes and the primitive generators used to build scenes.

Scene construction is outside the accelerated step: it runs
once per environment on the host.  These generators reproduce the reference's
vertex and triangle ORDER exactly (gripsim/geometry/mesh.py:224-409), because
candidate stencils are compared index-for-index with the reference; the
golden mesh fixtures (tests/golden/meshes.npz) pin that.
"""

from __future__ import annotations

import numpy as np

_TET_FACES = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]], np.int64)  # mesh.py:19
_MIN_TRI_AREA = 1e-12


class TriSurface:
    """Triangle surface with current and rest vertex positions (mesh.py:30-140)."""

    def __init__(self, vertices, triangles, rest_vertices=None):
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        self.triangles = np.ascontiguousarray(triangles, dtype=np.int64).reshape(-1, 3)
        self.rest_vertices = (self.vertices.copy() if rest_vertices is None
                              else np.ascontiguousarray(rest_vertices, dtype=np.float64).reshape(-1, 3))
        t = self.triangles
        if t.size and (t.min() < 0 or t.max() >= len(self.vertices)):
            raise ValueError("triangle index out of range")
        if np.any(self.triangle_areas() <= _MIN_TRI_AREA):
            raise ValueError("degenerate triangle (area <= 1e-12 m^2)")
        self._edges = None

    @property
    def n_vertices(self):
        return len(self.vertices)

    @property
    def n_triangles(self):
        return len(self.triangles)

    def triangle_areas(self):
        v, t = self.vertices, self.triangles
        return 0.5 * np.linalg.norm(np.cross(v[t[:, 1]] - v[t[:, 0]], v[t[:, 2]] - v[t[:, 0]]), axis=1)

    def edges(self):
        """Unique undirected edges in lexicographic order (mesh.py:72-79)."""
        if self._edges is None:
            t = self.triangles
            e = np.sort(np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]]), axis=1)
            self._edges = np.unique(e, axis=0)
        return self._edges

    def enclosed_volume(self):
        v, t = self.vertices, self.triangles
        return float(np.einsum("ij,ij->i", v[t[:, 0]], np.cross(v[t[:, 1]], v[t[:, 2]])).sum() / 6.0)

    def transformed(self, rotation=None, translation=None, scale=None):
        v = self.vertices
        if scale is not None:
            v = v * float(scale)
        if rotation is not None:
            v = v @ np.asarray(rotation, np.float64).T
        if translation is not None:
            v = v + np.asarray(translation, np.float64)
        return TriSurface(v, self.triangles.copy())


def tet_volumes(v, tets):
    d1, d2, d3 = (v[tets[:, k]] - v[tets[:, 0]] for k in (1, 2, 3))
    return np.einsum("ij,ij->i", np.cross(d1, d2), d3) / 6.0


class TetMesh:
    """Tetrahedral mesh with rest state and boundary extraction (mesh.py:151-209)."""

    def __init__(self, vertices, tets, rest_vertices=None):
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        self.tets = np.ascontiguousarray(tets, dtype=np.int64).reshape(-1, 4)
        self.rest_vertices = (self.vertices.copy() if rest_vertices is None
                              else np.ascontiguousarray(rest_vertices, dtype=np.float64).reshape(-1, 3))
        self.refresh()

    def refresh(self):
        """Re-derive rest volumes after the rest state was edited in place (config.py:274-277)."""
        if self.tets.size and (self.tets.min() < 0 or self.tets.max() >= len(self.vertices)):
            raise ValueError("tet index out of range")
        self.rest_volumes = tet_volumes(self.rest_vertices, self.tets)
        if np.any(self.rest_volumes <= 0.0):
            raise ValueError("tet with non-positive rest volume")
        self._boundary = None

    __post_init__ = refresh   # name the reference's scene code calls

    @property
    def n_vertices(self):
        return len(self.vertices)

    @property
    def n_tets(self):
        return len(self.tets)

    def boundary_surface(self):
        """(TriSurface over boundary vertices, vertex map); faces seen once, in tet order."""
        if self._boundary is None:
            faces = self.tets[:, _TET_FACES].reshape(-1, 3)
            _, inv, cnt = np.unique(np.sort(faces, axis=1), axis=0, return_inverse=True, return_counts=True)
            faces = faces[cnt[inv.reshape(-1)] == 1]
            used = np.unique(faces)
            remap = np.full(self.n_vertices, -1, np.int64)
            remap[used] = np.arange(len(used))
            surf = TriSurface(self.vertices[used], remap[faces], rest_vertices=self.rest_vertices[used])
            self._boundary = (surf, used)
        return self._boundary


def _outward(v, t):
    s = TriSurface(v, t)
    return s if s.enclosed_volume() >= 0.0 else TriSurface(v, t[:, [0, 2, 1]])


def box_surface(size, center=(0.0, 0.0, 0.0), subdivisions=1):
    """Box surface, each face a subdivisions^2 grid of quad pairs (mesh.py:224-256).

    Vertex ids are assigned on first sight of the 12-decimal-rounded unit
    coordinate, which is also the coordinate used (the reference keys by it).
    """
    size = np.broadcast_to(np.asarray(size, np.float64), (3,))
    n = int(subdivisions)
    ids: dict = {}
    tris = []
    for axis in range(3):
        ua, va = (axis + 1) % 3, (axis + 2) % 3
        for sign in (-1.0, 1.0):
            for i in range(n):
                for j in range(n):
                    q = []
                    for di, dj in ((0, 0), (1, 0), (1, 1), (0, 1)):
                        c = [0.0, 0.0, 0.0]
                        c[axis] = sign * 0.5
                        c[ua] = -0.5 + (i + di) / n
                        c[va] = -0.5 + (j + dj) / n
                        key = tuple(round(float(x), 12) for x in c)
                        q.append(ids.setdefault(key, len(ids)))
                    a, b, c_, d = q
                    tris += [[a, b, c_], [a, c_, d]] if sign > 0 else [[a, c_, b], [a, d, c_]]
    v = np.array(list(ids), np.float64) * size + np.asarray(center, np.float64)
    return _outward(v, np.array(tris, np.int64))


_ICO_FACES = np.array([
    [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4], [11, 10, 2],
    [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5],
    [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], np.int64)


def icosphere(radius=0.5, level=2, center=(0.0, 0.0, 0.0)):
    """Midpoint-subdivided icosahedron (mesh.py:259-299)."""
    g = (1.0 + np.sqrt(5.0)) / 2.0
    base = np.array([[-1, g, 0], [1, g, 0], [-1, -g, 0], [1, -g, 0], [0, -1, g], [0, 1, g], [0, -1, -g],
                     [0, 1, -g], [g, 0, -1], [g, 0, 1], [-g, 0, -1], [-g, 0, 1]], np.float64)
    base /= np.linalg.norm(base, axis=1, keepdims=True)
    verts = list(base)
    faces = _ICO_FACES
    for _ in range(level):
        cache: dict = {}

        def mid(a, b):
            k = (min(a, b), max(a, b))
            if k not in cache:
                m = verts[a] + verts[b]
                m /= np.linalg.norm(m)
                cache[k] = len(verts)
                verts.append(m)
            return cache[k]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        faces = np.array(nf, np.int64)
    v = np.array(verts) * radius + np.asarray(center, np.float64)
    return _outward(v, faces)


def revolved_surface(profile, segments=24, center=(0.0, 0.0, 0.0)):
    """Revolve a closed (r, z) polygon about z (mesh.py:316-359); r=0 points become apexes."""
    prof = [(float(r), float(z)) for r, z in profile]
    theta = np.linspace(0.0, 2.0 * np.pi, segments, endpoint=False)
    ids: dict = {}
    verts = []

    def vid(i, k):
        r, z = prof[i]
        key = (i, -1) if r == 0.0 else (i, k % segments)
        if key not in ids:
            th = theta[k % segments]
            verts.append([0.0, 0.0, z] if r == 0.0 else [r * np.cos(th), r * np.sin(th), z])
            ids[key] = len(verts) - 1
        return ids[key]

    tris = []
    for i in range(len(prof)):
        j = (i + 1) % len(prof)
        r1, r2 = prof[i][0], prof[j][0]
        if r1 == 0.0 and r2 == 0.0:
            continue
        for k in range(segments):
            if r1 > 0.0 and r2 > 0.0:
                a, b, c, d = vid(i, k), vid(j, k), vid(j, k + 1), vid(i, k + 1)
                tris += [[a, b, c], [a, c, d]]
            elif r1 == 0.0:
                tris.append([vid(i, 0), vid(j, k), vid(j, k + 1)])
            else:
                tris.append([vid(i, k), vid(j, 0), vid(i, k + 1)])
    v = np.array(verts, np.float64) + np.asarray(center, np.float64)
    return _outward(v, np.array(tris, np.int64))


def cylinder_surface(radius=0.02, height=0.05, segments=20):
    """Closed cylinder centred at the origin (config 2's third primitive)."""
    return revolved_surface([(0.0, 0.0), (radius, 0.0), (radius, height), (0.0, height)],
                            segments=segments, center=(0.0, 0.0, -0.5 * height))


# Freudenthal 6-tet split of a cube; corner bits are (x<<2 | y<<1 | z)  (mesh.py:363-373)
_CUBE_TETS = np.array([[0, 4, 6, 7], [0, 6, 2, 7], [0, 2, 3, 7], [0, 3, 1, 7], [0, 1, 5, 7], [0, 5, 4, 7]],
                      np.int64)


def box_tet_lattice(size, resolution=3, center=(0.0, 0.0, 0.0)):
    """Lattice tetrahedralisation of a box, 6 tets per cell (mesh.py:376-397)."""
    size = np.broadcast_to(np.asarray(size, np.float64), (3,))
    res = [int(r) for r in np.broadcast_to(np.asarray(resolution, np.int64), (3,))]
    axes = [np.linspace(-0.5 * size[i], 0.5 * size[i], res[i] + 1) for i in range(3)]
    grid = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3) + np.asarray(center, np.float64)
    nx, ny, nz = res
    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    cells = np.stack([ci.ravel(), cj.ravel(), ck.ravel()], 1)               # (i, j, k) row-major
    bits = np.arange(8)
    off = np.stack([(bits >> 2) & 1, (bits >> 1) & 1, bits & 1], 1)           # corner offsets
    c = cells[:, None, :] + off[None]
    corner = (c[..., 0] * (ny + 1) + c[..., 1]) * (nz + 1) + c[..., 2]       # (n_cells, 8)
    tets = corner[:, _CUBE_TETS].reshape(-1, 4)
    return TetMesh(grid, tets)


def sphere_tet_lattice(radius=0.05, resolution=6, center=(0.0, 0.0, 0.0)):
    """Lattice tets whose centroid lies inside the ball (mesh.py:400-409)."""
    full = box_tet_lattice(2.0 * radius, resolution, center=center)
    cen = full.vertices[full.tets].mean(axis=1)
    tets = full.tets[np.linalg.norm(cen - np.asarray(center), axis=1) <= radius]
    used = np.unique(tets)
    remap = np.full(full.n_vertices, -1, np.int64)
    remap[used] = np.arange(len(used))
    return TetMesh(full.vertices[used], remap[tets])


def surface_mass_properties(surface, density):
    """(mass, com, second moment about com) of the enclosed solid (mesh.py:544-571)."""
    v, t = surface.vertices, surface.triangles
    a, b, c = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
    vols = np.einsum("ij,ij->i", a, np.cross(b, c)) / 6.0
    V = vols.sum()
    if V <= 0.0:
        raise ValueError("surface encloses non-positive volume")
    com = (vols[:, None] * ((a + b + c) / 4.0)).sum(axis=0) / V
    s = a + b + c
    sec = (vols[:, None, None] / 20.0 * (np.einsum("ni,nj->nij", a, a) + np.einsum("ni,nj->nij", b, b)
                                         + np.einsum("ni,nj->nij", c, c) + np.einsum("ni,nj->nij", s, s))).sum(axis=0)
    mass = density * V
    return mass, com, density * sec - mass * np.outer(com, com)


def lumped_vertex_masses(mesh, density):
    """rho*V0/4 to each tet corner (materials.py:208-213)."""
    m = np.zeros(mesh.n_vertices)
    np.add.at(m, mesh.tets.reshape(-1), np.repeat(density * mesh.rest_volumes / 4.0, 4))
    return m
