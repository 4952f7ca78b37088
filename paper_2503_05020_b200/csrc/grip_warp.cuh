// Warp-per-element element kernel math: one warp evaluates one element (tet, affine body,
// contact stencil or friction anchor), its 12x12 Hessian and the reference's eigen-clamp,
// with the element's matrices staged in a per-warp shared-memory workspace.  Lanes own
// matrix entries; the 9x9 symmetric eigenproblem uses parallel-ordered Jacobi (4 disjoint
// rotations per round).  Nothing is kept in per-thread arrays, so there is no local-memory
// traffic (the per-thread versions in grip_elements.cuh remain the host-checked spec).
#pragma once
#include "grip_elements.cuh"

namespace grip {

struct WarpWS {
  double H[144];
  double S[81];
  double V[81];
  double T[108];
  double sc[48];      // broadcast scalars / small vectors
  double g[12];       // element gradient
  double al[10], be[10];
  int pi[10];
  int flag;
};

__device__ __forceinline__ double wred_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// S = Q^T H Q (9x9), Q = Helmert (x) I3 ; symmetric result
__device__ void w_S_from_H(WarpWS& w, int lane) {
  for (int e = lane; e < 108; e += 32) {          // T = H Q : T[r][(j,b)]
    const int r = e / 9, jb = e % 9, j = jb / 3, b = jb % 3;
    double s = 0.0;
    for (int l = 0; l < 4; ++l) s += w.H[r * 12 + 3 * l + b] * helmert(j, l);
    w.T[e] = s;
  }
  __syncwarp();
  for (int e = lane; e < 81; e += 32) {           // S = Q^T T
    const int ia = e / 9, c = e % 9, i = ia / 3, a = ia % 3;
    double s = 0.0;
    for (int k = 0; k < 4; ++k) s += helmert(i, k) * w.T[(3 * k + a) * 9 + c];
    w.S[e] = s;
  }
  __syncwarp();
  for (int e = lane; e < 81; e += 32) {
    const int i = e / 9, j = e % 9;
    if (i < j) {
      const double v = 0.5 * (w.S[e] + w.S[j * 9 + i]);
      w.S[e] = v;
      w.S[j * 9 + i] = v;
    }
  }
  __syncwarp();
}

// true iff S - shift I is positive definite (parallel right-looking Cholesky in w.V)
__device__ bool w_chol_pd9(WarpWS& w, double shift, int lane) {
  for (int e = lane; e < 81; e += 32) w.V[e] = w.S[e] - ((e / 9 == e % 9) ? shift : 0.0);
  if (lane == 0) w.flag = 1;
  __syncwarp();
  for (int k = 0; k < 9; ++k) {
    if (lane == 0) {
      const double d = w.V[k * 10];
      if (!(d > 0.0)) w.flag = 0;
      else w.V[k * 10] = sqrt(d);
    }
    __syncwarp();
    if (!w.flag) return false;
    const double lkk = w.V[k * 10];
    if (lane > k && lane < 9) w.V[lane * 9 + k] /= lkk;
    __syncwarp();
    for (int e = lane; e < 81; e += 32) {
      const int i = e / 9, j = e % 9;
      if (j > k && i >= j) w.V[e] -= w.V[i * 9 + k] * w.V[j * 9 + k];
    }
    __syncwarp();
  }
  return true;
}

// largest eigenvalue estimate of SPD S by power iteration (only scales the 1e-12 floor)
__device__ double w_power9(WarpWS& w, int lane) {
  double* v = w.sc;
  if (lane < 9) v[lane] = 1.0 + 0.1 * lane;
  __syncwarp();
  double lam = 0.0;
  for (int it = 0; it < 12; ++it) {
    double wi = 0.0;
    if (lane < 9)
      for (int j = 0; j < 9; ++j) wi += w.S[lane * 9 + j] * v[j];
    const double vi = lane < 9 ? v[lane] : 0.0;
    const double nn = sqrt(wred_sum(wi * wi));
    const double vw = wred_sum(vi * wi), vv = wred_sum(vi * vi);
    if (nn == 0.0) break;
    lam = vw / vv;
    __syncwarp();
    if (lane < 9) v[lane] = wi / nn;
    __syncwarp();
  }
  return lam;
}

// Jacobi eigendecomposition of the symmetric 9x9 w.S (-> diagonal), eigenvectors in w.V.
// Round-robin ordering over 10 players (index 9 is a bye): every pair once per sweep.
// Lane l owns entries l, l+32, l+64 of S and V (row/column indices precomputed).
__device__ __constant__ signed char kRR[9][5][2] = {
    {{0, 1}, {2, 9}, {3, 8}, {4, 7}, {5, 6}}, {{0, 2}, {3, 1}, {4, 9}, {5, 8}, {6, 7}},
    {{0, 3}, {4, 2}, {5, 1}, {6, 9}, {7, 8}}, {{0, 4}, {5, 3}, {6, 2}, {7, 1}, {8, 9}},
    {{0, 5}, {6, 4}, {7, 3}, {8, 2}, {9, 1}}, {{0, 6}, {7, 5}, {8, 4}, {9, 3}, {1, 2}},
    {{0, 7}, {8, 6}, {9, 5}, {1, 4}, {2, 3}}, {{0, 8}, {9, 7}, {1, 6}, {2, 5}, {3, 4}},
    {{0, 9}, {1, 8}, {2, 7}, {3, 6}, {4, 5}}};

__device__ void w_jacobi9(WarpWS& w, int lane, bool init_identity = true) {
  if (init_identity) {
    for (int e = lane; e < 81; e += 32) w.V[e] = (e / 9 == e % 9) ? 1.0 : 0.0;
    __syncwarp();
  }
  int ei[3], ej[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int e = lane + 32 * c;
    ei[c] = e < 81 ? e / 9 : 0;
    ej[c] = e < 81 ? e % 9 : 0;
  }
  const int nown = lane < 17 ? 3 : 2;   // 81 = 2*32 + 17
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (c < nown) {
        const double v = w.S[lane + 32 * c];
        tot += v * v;
        if (ei[c] != ej[c]) off += v * v;
      }
    }
    off = wred_sum(off);
    tot = wred_sum(tot);
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int r = 0; r < 9; ++r) {
      if (lane < 5) {
        const int a = kRR[r][lane][0], b = kRR[r][lane][1];
        const int p = min(a, b), q = max(a, b);
        if (q == 9) {
          w.al[p] = 1.0; w.be[p] = 0.0; w.pi[p] = p;
        } else {
          const double apq = w.S[p * 9 + q];
          double c = 1.0, sn = 0.0;
          if (apq != 0.0) {
            // t = sgn(theta) / (|theta| + sqrt(theta^2 + 1)), theta = (aqq - app) / (2 apq)
            const double d = w.S[q * 9 + q] - w.S[p * 9 + p];
            const double sg = ((d >= 0.0) == (apq > 0.0)) ? 1.0 : -1.0;
            const double t = sg * 2.0 * fabs(apq) / (fabs(d) + sqrt(d * d + 4.0 * apq * apq));
            c = rsqrt(t * t + 1.0);
            sn = t * c;
          }
          w.al[p] = c; w.be[p] = -sn; w.pi[p] = q;
          w.al[q] = c; w.be[q] = sn; w.pi[q] = p;
        }
      }
      __syncwarp();
      double ns[3], nv[3];
      bool z[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (c < nown) {
          const int i = ei[c], j = ej[c];
          const double ai = w.al[i], bi = w.be[i], aj = w.al[j], bj = w.be[j];
          const int pi_ = w.pi[i], pj = w.pi[j];
          ns[c] = ai * aj * w.S[i * 9 + j] + ai * bj * w.S[i * 9 + pj] + bi * aj * w.S[pi_ * 9 + j] +
                  bi * bj * w.S[pi_ * 9 + pj];
          nv[c] = aj * w.V[i * 9 + j] + bj * w.V[i * 9 + pj];
          // the rotated pair's off-diagonal is exactly zero after its rotation
          z[c] = i != j && pi_ == j && bi != 0.0;
        }
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (c < nown) {
          const int e = lane + 32 * c;
          w.S[e] = z[c] ? 0.0 : ns[c];
          w.V[e] = nv[c];
        }
      }
      __syncwarp();
    }
  }
}

// Warm start: S <- V0^T S V0 with the element's eigenvectors from its previous Newton iteration
// (V0 orthogonal), so Jacobi starts near diagonal; the accumulated V is then the eigenbasis of
// the ORIGINAL S.  Same converged spectral decomposition, typically 1-2 sweeps instead of ~7.
__device__ void w_rotate_into(WarpWS& w, const double* V0, int lane) {
  for (int e = lane; e < 81; e += 32) w.V[e] = V0[e];
  __syncwarp();
  for (int e = lane; e < 81; e += 32) {   // T = S V0
    const int i = e / 9, j = e % 9;
    double acc = 0.0;
    for (int k = 0; k < 9; ++k) acc += w.S[i * 9 + k] * w.V[k * 9 + j];
    w.T[e] = acc;
  }
  __syncwarp();
  for (int e = lane; e < 81; e += 32) {   // S = V0^T T
    const int i = e / 9, j = e % 9;
    double acc = 0.0;
    for (int k = 0; k < 9; ++k) acc += w.V[k * 9 + i] * w.T[k * 9 + j];
    w.S[e] = acc;
  }
  __syncwarp();
  for (int e = lane; e < 81; e += 32) {
    const int i = e / 9, j = e % 9;
    if (i < j) {
      const double v = 0.5 * (w.S[e] + w.S[j * 9 + i]);
      w.S[e] = v;
      w.S[j * 9 + i] = v;
    }
  }
  __syncwarp();
}

// reference clamp (materials.py:101-113) of a translation-invariant 4-point stencil Hessian in w.H
// (Vwarm: previous eigenvectors of this element or null; Vout: where to keep the new ones)
// defer_S: when the eigensolve is needed, write S (warm-rotated S~ for tets; upper triangle, 45)
// there and return true without clamping; k_tet_jacobi2 / k_tet_finish complete the clamp
__device__ bool w_clamp_stencil(WarpWS& w, int lane, const double* Vwarm = nullptr, double* Vout = nullptr,
                                double* defer_S = nullptr) {
  for (int e = lane; e < 144; e += 32) {
    const int i = e / 12, j = e % 12;
    if (i < j) {
      const double v = 0.5 * (w.H[e] + w.H[j * 12 + i]);
      w.H[e] = v;
      w.H[j * 12 + i] = v;
    }
  }
  __syncwarp();
  w_S_from_H(w, lane);
  double fro = 0.0;
  for (int e = lane; e < 81; e += 32) fro += w.S[e] * w.S[e];
  fro = sqrt(wred_sum(fro));
  double f;
  bool pd = false;
  if (!Vwarm && w_chol_pd9(w, 1e-12 * fro, lane)) {
    f = 1e-12 * w_power9(w, lane);
    pd = true;
  } else if (Vwarm) {
    // S~ = V0^T S V0 is near diagonal; when every Gershgorin disc of S~ lies above the clamp
    // floor 1e-12 max|lambda|, no eigenvalue is clamped and H passes through unchanged
    w_rotate_into(w, Vwarm, lane);
    if (lane < 9) {
      double rad = 0.0;
      for (int j = 0; j < 9; ++j)
        if (j != lane) rad += fabs(w.S[lane * 9 + j]);
      const double dg = w.S[lane * 10];
      w.sc[lane] = dg - rad;
      w.sc[9 + lane] = dg + rad;
      w.sc[18 + lane] = fabs(dg);
    }
    __syncwarp();
    double lo = w.sc[0], hi = w.sc[9], dm = w.sc[18];
    for (int k = 1; k < 9; ++k) {
      lo = fmin(lo, w.sc[k]);
      hi = fmax(hi, w.sc[9 + k]);
      dm = fmax(dm, w.sc[18 + k]);
    }
    __syncwarp();
    if (lo > 1e-12 * hi) {
      f = 1e-12 * dm;
      pd = true;
    }
  }
  if (!pd && defer_S) {
    for (int q = lane; q < 45; q += 32) {
      int i = 0, rem = q;
      while (rem >= 9 - i) { rem -= 9 - i; ++i; }
      defer_S[q] = w.S[i * 9 + i + rem];
    }
    __syncwarp();
    return true;
  }
  if (!pd) {
    w_jacobi9(w, lane, Vwarm == nullptr);
    if (Vout)
      for (int e = lane; e < 81; e += 32) Vout[e] = w.V[e];
    double amax = 0.0;
    for (int k = 0; k < 9; ++k) amax = fmax(amax, fabs(w.S[k * 10]));
    f = 1e-12 * amax;
    // eigenvalue shifts d_k = max(lam_k, f) - lam_k, staged before S is reused
    if (lane < 9) {
      const double lk = w.S[lane * 10];
      w.sc[lane] = fmax(lk, f) - lk;
    }
    __syncwarp();
    // H += U diag(d) U^T with U = Q V (12x9): only the clamped eigenpairs (d_k != 0) contribute
    for (int e = lane; e < 108; e += 32) {
      const int r = e / 9, k = e - 9 * r, n = r / 3, a = r - 3 * n;
      double u = 0.0;
      if (w.sc[k] != 0.0)
        for (int i = 0; i < 3; ++i) u += helmert(i, n) * w.V[(3 * i + a) * 9 + k];
      w.T[e] = u;
    }
    __syncwarp();
  }
  // plus the reference's lifted translation modes (f/4 on equal components); both terms are
  // symmetric and added to the mirrored entries identically, so H stays exactly symmetric
  for (int t = lane; t < 78; t += 32) {
    int i = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    while (i * (i + 1) / 2 > t) --i;
    const int j = t - i * (i + 1) / 2;
    double s = (i % 3 == j % 3) ? 0.25 * f : 0.0;
    if (!pd)
      for (int k = 0; k < 9; ++k) {
        const double d = w.sc[k];
        if (d != 0.0) s += d * (w.T[i * 9 + k] * w.T[j * 9 + k]);
      }
    w.H[i * 12 + j] += s;
    if (i != j) w.H[j * 12 + i] += s;
  }
  __syncwarp();
  return false;
}

// rank-one clamp: H = c g g^T + f (I - g g^T/|g|^2), f = 1e-12 c |g|^2 ; g in w.sc[0..11]
__device__ void w_rank1(WarpWS& w, double c, int lane) {
  double gg = 0.0;
  for (int i = 0; i < 12; ++i) gg += w.sc[i] * w.sc[i];
  const double f = 1e-12 * fabs(c * gg);
  const double ig = gg > 0.0 ? 1.0 / gg : 0.0;
  for (int e = lane; e < 144; e += 32) {
    const int i = e / 12, j = e % 12;
    const double gi = w.sc[i], gj = w.sc[j];
    w.H[e] = c * gi * gj + f * ((i == j ? 1.0 : 0.0) - gi * gj * ig);
  }
  __syncwarp();
}

// plane-distance Hessian over 4 points (distances.py:230-343) into w.H; chain C[r][k]
__device__ void w_plane12(WarpWS& w, V3 wv, V3 u, V3 v, const double C[3][4], int lane) {
  // small 3x3 blocks redundantly per lane (cheap), H9 entries parallel over lanes
  V3 n = cross(u, v);
  const double iq = 1.0 / dot(n, n);
  const double sq = dot(wv, n) * iq;
  const double nvv[3] = {n.x, n.y, n.z}, wvv[3] = {wv.x, wv.y, wv.z};
  double gn[3];
  for (int i = 0; i < 3; ++i) gn[i] = 2.0 * sq * wvv[i] - 2.0 * sq * sq * nvv[i];
  double Ju[9], Jv[9], cu[9];
  skew(v, Ju);
  for (int i = 0; i < 9; ++i) Ju[i] = -Ju[i];
  skew(u, Jv);
  skew(V3{gn[0], gn[1], gn[2]}, cu);
  auto Hww = [&](int i, int j) { return 2.0 * iq * nvv[i] * nvv[j]; };
  auto Hwn = [&](int i, int j) {
    return 2.0 * iq * nvv[i] * wvv[j] + (i == j ? 2.0 * sq : 0.0) - 4.0 * sq * iq * nvv[i] * nvv[j];
  };
  auto Hnn = [&](int i, int j) {
    return 2.0 * iq * wvv[i] * wvv[j] - 4.0 * sq * iq * (nvv[i] * wvv[j] + wvv[i] * nvv[j]) - (i == j ? 2.0 * sq * sq : 0.0) +
           8.0 * sq * sq * iq * nvv[i] * nvv[j];
  };
  // H9 blocks (r, s) with r,s in {w,u,v} -> w.T[0..80]
  for (int e = lane; e < 81; e += 32) {
    const int ra = e / 9, sb = e % 9, r = ra / 3, a = ra % 3, s = sb / 3, b = sb % 3;
    double val = 0.0;
    if (r == 0 && s == 0) {
      val = Hww(a, b);
    } else if (r == 0 || s == 0) {  // Hw? = Hwn J?
      const int ii = r == 0 ? a : b, jj = r == 0 ? b : a, o = r == 0 ? s : r;
      const double* J = o == 1 ? Ju : Jv;
      for (int k = 0; k < 3; ++k) val += Hwn(ii, k) * J[3 * k + jj];
    } else {                        // J_r^T Hnn J_s (+ curvature on u-v)
      const double* Jr = r == 1 ? Ju : Jv;
      const double* Js = s == 1 ? Ju : Jv;
      for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) val += Jr[3 * k + a] * Hnn(k, l) * Js[3 * l + b];
      if (r == 1 && s == 2) val -= cu[3 * a + b];
      if (r == 2 && s == 1) val -= cu[3 * b + a];
    }
    w.T[e] = val;
  }
  __syncwarp();
  for (int e = lane; e < 144; e += 32) {
    const int ka = e / 12, lb = e % 12, k = ka / 3, a = ka % 3, l = lb / 3, b = lb % 3;
    double s = 0.0;
    for (int r = 0; r < 3; ++r) {
      if (C[r][k] == 0.0) continue;
      for (int q = 0; q < 3; ++q) {
        if (C[q][l] == 0.0) continue;
        s += C[r][k] * C[q][l] * w.T[(3 * r + a) * 9 + 3 * q + b];
      }
    }
    w.H[e] = s;
  }
  __syncwarp();
}

}  // namespace grip
