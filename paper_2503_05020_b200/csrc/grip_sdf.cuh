// Signed distance fields for the D1/D2 grasp-quality metrics (
// gripsim/geometry/sdf.py, gripsim/pipeline/metrics.py).
//
// k_sdf_exact : the narrow band of build_sdf (sdf.py:168-241): thread per grid point, the
//               exact closest point over ALL triangles of the surface (brute force: the
//               surfaces here have <= a few thousand triangles, so every band point is one
//               warp-coherent sweep), signed by the angle-weighted pseudonormal of the
//               closest feature (face / edge / vertex, the reference's region codes).
// k_sdf_query : metrics.py:58-75 with sdf.py:62-87: per sample, d_o = -trilinear(SDF) inside
//               the grid box of the (posed) SDF, else -|gap to the world AABB|; a max-reduction
//               of d_o gives D1 = max(0, max d_o) and D2 = |max d_o|.
#pragma once
#include "grip_device.cuh"

namespace grip {

__global__ void k_sdf_exact(const double* pts, long long n, const double* V, const int* T, int nt, const double* fn,
                            const double* en, const double* vn, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const V3 p = ld3(pts + 3 * i);
    double best = INFINITY, bb[3] = {0, 0, 0};
    int bt = 0, br = 6;
    for (int t = 0; t < nt; ++t) {
      const int a = T[3 * t], b = T[3 * t + 1], c = T[3 * t + 2];
      double bary[3];
      int reg;
      const double D = pt_closest(p, ld3(V + 3 * a), ld3(V + 3 * b), ld3(V + 3 * c), bary, &reg);
      if (D < best) {   // first minimum in triangle order
        best = D;
        bt = t;
        br = reg;
        bb[0] = bary[0]; bb[1] = bary[1]; bb[2] = bary[2];
      }
    }
    const int a = T[3 * bt], b = T[3 * bt + 1], c = T[3 * bt + 2];
    const V3 cl = bb[0] * ld3(V + 3 * a) + bb[1] * ld3(V + 3 * b) + bb[2] * ld3(V + 3 * c);
    V3 nrm;
    if (br == 6) nrm = ld3(fn + 3 * bt);
    else if (br >= 3) nrm = ld3(en + 9 * bt + 3 * (br - 3));   // edges (0,1), (1,2), (2,0)
    else nrm = ld3(vn + 3 * T[3 * bt + br]);
    const V3 dp = p - cl;
    const double s = dot(dp, nrm) >= 0.0 ? 1.0 : -1.0;
    out[i] = s * sqrt(best);
  }
}

struct SdfGridDev {
  const double* values;
  int nx, ny, nz;
  double ox, oy, oz, hx, hy, hz;
};

__device__ __forceinline__ double sdf_trilinear(const SdfGridDev& G, V3 q) {
  const double gx = fmin(fmax((q.x - G.ox) / G.hx, 0.0), (G.nx - 1) - 1e-12);
  const double gy = fmin(fmax((q.y - G.oy) / G.hy, 0.0), (G.ny - 1) - 1e-12);
  const double gz = fmin(fmax((q.z - G.oz) / G.hz, 0.0), (G.nz - 1) - 1e-12);
  const int ix = min((int)gx, G.nx - 2), iy = min((int)gy, G.ny - 2), iz = min((int)gz, G.nz - 2);
  const double fx = gx - ix, fy = gy - iy, fz = gz - iz;
  const double wx[2] = {1.0 - fx, fx}, wy[2] = {1.0 - fy, fy}, wz[2] = {1.0 - fz, fz};
  double s = 0.0;
  for (int dx = 0; dx < 2; ++dx)
    for (int dy = 0; dy < 2; ++dy)
      for (int dz = 0; dz < 2; ++dz)
        s += G.values[((size_t)(ix + dx) * G.ny + (iy + dy)) * G.nz + (iz + dz)] * wx[dx] * wy[dy] * wz[dz];
  return s;
}

// R (row-major) / T: the SDF's pose (body = (p - T) R); lo/hi: its grid box in the body
// frame; wlo/whi: the world AABB of that box (PosedSdf.bounds, metrics.py:33-37)
__global__ void k_sdf_query(SdfGridDev G, const double* R, V3 Tr, V3 lo, V3 hi, V3 wlo, V3 whi, const double* pts,
                            long long n, double* d_o, unsigned long long* dmax_bits) {
  double m = -INFINITY;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const V3 p = ld3(pts + 3 * i);
    V3 q = p;
    if (R) {
      const V3 d = p - Tr;   // (p - T) @ R
      q = V3{d.x * R[0] + d.y * R[3] + d.z * R[6], d.x * R[1] + d.y * R[4] + d.z * R[7],
             d.x * R[2] + d.y * R[5] + d.z * R[8]};
    }
    double v;
    if (q.x >= lo.x && q.y >= lo.y && q.z >= lo.z && q.x <= hi.x && q.y <= hi.y && q.z <= hi.z) {
      v = -sdf_trilinear(G, q);
    } else {
      const double gx = fmax(wlo.x - p.x, 0.0) + fmax(p.x - whi.x, 0.0);
      const double gy = fmax(wlo.y - p.y, 0.0) + fmax(p.y - whi.y, 0.0);
      const double gz = fmax(wlo.z - p.z, 0.0) + fmax(p.z - whi.z, 0.0);
      v = -sqrt(gx * gx + gy * gy + gz * gz);
    }
    if (d_o) d_o[i] = v;
    m = fmax(m, v);
  }
  m = wmax(m);
  // order-preserving map of doubles to unsigned keys: the max is exact and schedule-independent
  if ((threadIdx.x & 31) == 0) {
    unsigned long long u = __double_as_longlong(m);
    u = (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
    atomicMax(dmax_bits, u);
  }
}

}  // namespace grip

namespace grip {

// Exact nearest-neighbour distance from every query to a point cloud (the far field of
// build_sdf, sdf.py:150-151, there a scipy cKDTree).  The cloud is sorted by Morton code on
// the host and grouped into leaves of SDF_LEAF points under an implicit complete binary tree
// of boxes (heap order, node k -> children 2k+1, 2k+2); one thread per query walks it depth
// first, nearer child first, pruning boxes farther than the best distance so far.  Squared
// distances are summed without FMA contraction, in x, y, z order, as cKDTree does, so the
// minimum is the same double.
constexpr int SDF_LEAF = 8;

__device__ __forceinline__ double d2_rn(V3 a, V3 b) {
  const double dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y), dz = __dsub_rn(a.z, b.z);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

__device__ __forceinline__ double box_d2(V3 q, const double* lo, const double* hi) {
  const double gx = fmax(fmax(lo[0] - q.x, q.x - hi[0]), 0.0);
  const double gy = fmax(fmax(lo[1] - q.y, q.y - hi[1]), 0.0);
  const double gz = fmax(fmax(lo[2] - q.z, q.z - hi[2]), 0.0);
  return gx * gx + gy * gy + gz * gz;
}

__global__ void k_sdf_nn(const double* pts, long long n, const double* cloud, long long m, const double* blo,
                         const double* bhi, int levels, double* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const V3 q = ld3(pts + 3 * i);
    double best = INFINITY;
    int stack[64];
    int sp = 0;
    stack[sp++] = 0;
    const int first_leaf = (1 << levels) - 1;
    while (sp) {
      const int k = stack[--sp];
      // the box test is a strict prune with a small relative margin: it only skips work,
      // the exact distances below decide
      if (box_d2(q, blo + 3 * (size_t)k, bhi + 3 * (size_t)k) * (1.0 - 1e-12) > best) continue;
      if (k >= first_leaf) {
        const long long p0 = (long long)(k - first_leaf) * SDF_LEAF;
        const long long p1 = p0 + SDF_LEAF < m ? p0 + SDF_LEAF : m;
        for (long long p = p0; p < p1; ++p) best = fmin(best, d2_rn(q, ld3(cloud + 3 * p)));
        continue;
      }
      const int c0 = 2 * k + 1, c1 = 2 * k + 2;
      const double d0 = box_d2(q, blo + 3 * (size_t)c0, bhi + 3 * (size_t)c0);
      const double d1 = box_d2(q, blo + 3 * (size_t)c1, bhi + 3 * (size_t)c1);
      // push the farther child first so the nearer one is visited next
      const double m0 = d0 * (1.0 - 1e-12), m1 = d1 * (1.0 - 1e-12);
      if (d0 <= d1) {
        if (m1 <= best) stack[sp++] = c1;
        if (m0 <= best) stack[sp++] = c0;
      } else {
        if (m0 <= best) stack[sp++] = c0;
        if (m1 <= best) stack[sp++] = c1;
      }
    }
    out[i] = sqrt(best);
  }
}

}  // namespace grip
