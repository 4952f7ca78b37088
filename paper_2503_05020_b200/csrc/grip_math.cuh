// Small fp64 linear algebra shared by the device kernels and the host check library.
//
// Everything here is __host__ __device__ so tests/ can pin the element math on
// the CPU (libgrip_hostcheck.so) before it ever runs on a B200.
#pragma once
#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define GHD __host__ __device__ __forceinline__
#else
#define GHD inline
#endif

namespace grip {

struct V3 {
  double x, y, z;
};

GHD V3 v3(double a, double b, double c) { return V3{a, b, c}; }
GHD V3 ld3(const double* p) { return V3{p[0], p[1], p[2]}; }
GHD void st3(double* p, V3 a) { p[0] = a.x; p[1] = a.y; p[2] = a.z; }
GHD V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
GHD V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
GHD V3 operator*(double s, V3 a) { return V3{s * a.x, s * a.y, s * a.z}; }
GHD double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
GHD V3 cross(V3 a, V3 b) { return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
GHD double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
GHD double norm(V3 a) { return sqrt(dot(a, a)); }
GHD V3 vmin(V3 a, V3 b) { return V3{fmin(a.x, b.x), fmin(a.y, b.y), fmin(a.z, b.z)}; }
GHD V3 vmax(V3 a, V3 b) { return V3{fmax(a.x, b.x), fmax(a.y, b.y), fmax(a.z, b.z)}; }

// 3x3 row-major
GHD double det3(const double* m) {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) + m[2] * (m[3] * m[7] - m[4] * m[6]);
}
GHD void inv3(const double* m, double* o) {
  double d = det3(m);
  double id = 1.0 / d;
  o[0] = (m[4] * m[8] - m[5] * m[7]) * id;
  o[1] = (m[2] * m[7] - m[1] * m[8]) * id;
  o[2] = (m[1] * m[5] - m[2] * m[4]) * id;
  o[3] = (m[5] * m[6] - m[3] * m[8]) * id;
  o[4] = (m[0] * m[8] - m[2] * m[6]) * id;
  o[5] = (m[2] * m[3] - m[0] * m[5]) * id;
  o[6] = (m[3] * m[7] - m[4] * m[6]) * id;
  o[7] = (m[1] * m[6] - m[0] * m[7]) * id;
  o[8] = (m[0] * m[4] - m[1] * m[3]) * id;
}
GHD void mul33(const double* a, const double* b, double* o) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}

// ---------------------------------------------------------------------------
// Symmetric eigen-clamp (materials.py:101-113 semantics): sym -> eig ->
// lambda <- max(lambda, 1e-12 * max|lambda|) -> V diag V^T -> sym.
// Cyclic Jacobi with eigenvector accumulation on an n x n (n <= 12) matrix
// held in caller storage (row-major, leading dimension n).
// ---------------------------------------------------------------------------
template <int N>
GHD void jacobi_eig(double* A, double* V) {
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) V[i * N + j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        double a2 = A[i * N + j] * A[i * N + j];
        tot += a2;
        if (i != j) off += a2;
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < N - 1; ++p) {
      for (int q = p + 1; q < N; ++q) {
        double apq = A[p * N + q];
        if (apq == 0.0) continue;
        double app = A[p * N + p], aqq = A[q * N + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        // A <- J^T A J  with J = rotation in (p, q)
        for (int k = 0; k < N; ++k) {
          double akp = A[k * N + p], akq = A[k * N + q];
          A[k * N + p] = c * akp - s * akq;
          A[k * N + q] = s * akp + c * akq;
        }
        for (int k = 0; k < N; ++k) {
          double apk = A[p * N + k], aqk = A[q * N + k];
          A[p * N + k] = c * apk - s * aqk;
          A[q * N + k] = s * apk + c * aqk;
        }
        A[p * N + q] = 0.0;
        A[q * N + p] = 0.0;
        for (int k = 0; k < N; ++k) {
          double vkp = V[k * N + p], vkq = V[k * N + q];
          V[k * N + p] = c * vkp - s * vkq;
          V[k * N + q] = s * vkp + c * vkq;
        }
      }
    }
  }
}

// Cholesky test: true iff (S - shift I) is positive definite.  S is n x n, row-major.
template <int N>
GHD bool chol_pd(const double* S, double shift) {
  double L[N * (N + 1) / 2];
#define LI(i, j) L[(i) * ((i) + 1) / 2 + (j)]
  for (int i = 0; i < N; ++i) {
    for (int j = 0; j <= i; ++j) {
      double s = S[i * N + j] - (i == j ? shift : 0.0);
      for (int k = 0; k < j; ++k) s -= LI(i, k) * LI(j, k);
      if (i == j) {
        if (!(s > 0.0)) return false;
        LI(i, i) = sqrt(s);
      } else {
        LI(i, j) = s / LI(j, j);
      }
    }
  }
#undef LI
  return true;
}

// Generic clamp of an n x n symmetric matrix in place (full eigen path).
// Returns the clamp floor used.
template <int N>
GHD double spd_clamp_full(double* A) {
  double V[N * N];
  for (int i = 0; i < N; ++i)
    for (int j = i + 1; j < N; ++j) {
      double s = 0.5 * (A[i * N + j] + A[j * N + i]);
      A[i * N + j] = s;
      A[j * N + i] = s;
    }
  jacobi_eig<N>(A, V);
  double lam[N];
  double amax = 0.0;
  for (int i = 0; i < N; ++i) {
    lam[i] = A[i * N + i];
    amax = fmax(amax, fabs(lam[i]));
  }
  double fl = 1e-12 * amax;
  for (int i = 0; i < N; ++i) lam[i] = fmax(lam[i], fl);
  for (int i = 0; i < N; ++i)
    for (int j = i; j < N; ++j) {
      double s = 0.0;
      for (int k = 0; k < N; ++k) s += V[i * N + k] * lam[k] * V[j * N + k];
      A[i * N + j] = s;
      A[j * N + i] = s;
    }
  return fl;
}

// Helmert basis of the 4-point translation complement: Q = H4 (x) I3, 12 x 9.
// q1=(1,-1,0,0)/sqrt2, q2=(1,1,-2,0)/sqrt6, q3=(1,1,1,-3)/sqrt12.
GHD double helmert(int i, int k) {
  const double r2 = 0.70710678118654752440, r6 = 0.40824829046386301637, r12 = 0.28867513459481288225;
  if (i == 0) return k == 0 ? r2 : (k == 1 ? -r2 : 0.0);
  if (i == 1) return k < 2 ? r6 : (k == 2 ? -2.0 * r6 : 0.0);
  return k < 3 ? r12 : -3.0 * r12;
}

// Eigen-clamp of a translation-invariant 4-point stencil Hessian (12x12, in place).
//
// Such an H has the 3 rigid translations T in its null space, so
// eig(H) = eig(S) (+) {0,0,0} with S = Q^T H Q (9x9).  The reference's
// full 12x12 clamp therefore equals  Q clamp(S) Q^T + f T T^T  with
// f = 1e-12 max|lambda(S)|.  If S - f I is positive definite no eigenvalue
// of S is clamped and the result is H + f T T^T (the Cholesky fast path).
GHD void spd_clamp_stencil(double* H) {
  for (int i = 0; i < 12; ++i)
    for (int j = i + 1; j < 12; ++j) {
      double s = 0.5 * (H[i * 12 + j] + H[j * 12 + i]);
      H[i * 12 + j] = s;
      H[j * 12 + i] = s;
    }
  // S = Q^T H Q, indices (i,a) -> 3*i+a
  double S[81];
  double HQ[12 * 9];
  for (int r = 0; r < 12; ++r)
    for (int j = 0; j < 3; ++j)
      for (int b = 0; b < 3; ++b) {
        double s = 0.0;
        for (int l = 0; l < 4; ++l) s += H[r * 12 + 3 * l + b] * helmert(j, l);
        HQ[r * 9 + 3 * j + b] = s;
      }
  for (int i = 0; i < 3; ++i)
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 9; ++c) {
        double s = 0.0;
        for (int k = 0; k < 4; ++k) s += helmert(i, k) * HQ[(3 * k + a) * 9 + c];
        S[(3 * i + a) * 9 + c] = s;
      }
  for (int i = 0; i < 9; ++i)
    for (int j = i + 1; j < 9; ++j) {
      double s = 0.5 * (S[i * 9 + j] + S[j * 9 + i]);
      S[i * 9 + j] = s;
      S[j * 9 + i] = s;
    }
  double fro = 0.0;
  for (int i = 0; i < 81; ++i) fro += S[i] * S[i];
  fro = sqrt(fro);
  double f;
  bool fast = chol_pd<9>(S, 1e-12 * fro);
  if (fast) {
    // spectral radius by power iteration (only scales the 1e-12 floor)
    double v[9], w[9];
    for (int i = 0; i < 9; ++i) v[i] = 1.0 + 0.1 * i;
    double lam = 0.0;
    for (int it = 0; it < 12; ++it) {
      double nn = 0.0;
      for (int i = 0; i < 9; ++i) {
        double s = 0.0;
        for (int j = 0; j < 9; ++j) s += S[i * 9 + j] * v[j];
        w[i] = s;
        nn += s * s;
      }
      nn = sqrt(nn);
      if (nn == 0.0) break;
      double vv = 0.0, vw = 0.0;
      for (int i = 0; i < 9; ++i) {
        vv += v[i] * v[i];
        vw += v[i] * w[i];
      }
      lam = vw / vv;
      for (int i = 0; i < 9; ++i) v[i] = w[i] / nn;
    }
    f = 1e-12 * lam;
  } else {
    double V[81];
    jacobi_eig<9>(S, V);
    double lam[9], amax = 0.0;
    for (int i = 0; i < 9; ++i) {
      lam[i] = S[i * 9 + i];
      amax = fmax(amax, fabs(lam[i]));
    }
    f = 1e-12 * amax;
    // correction C = V diag(max(lam,f) - lam) V^T  (only clamped modes contribute)
    double C[81];
    for (int i = 0; i < 81; ++i) C[i] = 0.0;
    for (int k = 0; k < 9; ++k) {
      double d = fmax(lam[k], f) - lam[k];
      if (d == 0.0) continue;
      for (int i = 0; i < 9; ++i)
        for (int j = 0; j < 9; ++j) C[i * 9 + j] += d * V[i * 9 + k] * V[j * 9 + k];
    }
    // H += Q C Q^T
    double QC[12 * 9];
    for (int k = 0; k < 4; ++k)
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 9; ++c) {
          double s = 0.0;
          for (int i = 0; i < 3; ++i) s += helmert(i, k) * C[(3 * i + a) * 9 + c];
          QC[(3 * k + a) * 9 + c] = s;
        }
    for (int r = 0; r < 12; ++r)
      for (int l = 0; l < 4; ++l)
        for (int b = 0; b < 3; ++b) {
          double s = 0.0;
          for (int j = 0; j < 3; ++j) s += QC[r * 9 + 3 * j + b] * helmert(j, l);
          H[r * 12 + 3 * l + b] += s;
        }
  }
  // + f T T^T, T T^T[(k,a),(l,b)] = delta_ab / 4
  for (int k = 0; k < 4; ++k)
    for (int l = 0; l < 4; ++l)
      for (int a = 0; a < 3; ++a) H[(3 * k + a) * 12 + 3 * l + a] += 0.25 * f;
  for (int i = 0; i < 12; ++i)
    for (int j = i + 1; j < 12; ++j) {
      double s = 0.5 * (H[i * 12 + j] + H[j * 12 + i]);
      H[i * 12 + j] = s;
      H[j * 12 + i] = s;
    }
}

// Rank-one stencil Hessian H = c g g^T (c >= 0): eigenvalues c|g|^2 and eleven 0s,
// so the clamp is H + f (I - g g^T/|g|^2) with f = 1e-12 c |g|^2.
GHD void rank1_clamped(const double* g, double c, double* H) {
  double gg = 0.0;
  for (int i = 0; i < 12; ++i) gg += g[i] * g[i];
  double lam = c * gg;
  double f = 1e-12 * fabs(lam);
  double ig = gg > 0.0 ? 1.0 / gg : 0.0;
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j) H[i * 12 + j] = c * g[i] * g[j] + f * ((i == j ? 1.0 : 0.0) - g[i] * g[j] * ig);
}

}  // namespace grip
