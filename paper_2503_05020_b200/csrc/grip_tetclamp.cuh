// Batched completion of the eigen-clamp (materials.py:101-113) of the matrices the element
// kernels deferred (tets: k_tet_front stores the warm-rotated S~ = Y^T S Y; contacts:
// k_elements_w stores S and the unclamped H).
//   k_tet_jacobi2 : two threads per matrix, cyclic Jacobi on S~ entirely in registers (45 upper
//                   entries duplicated, rows of the rotation R split, the round-robin schedule
//                   unrolled so every index is static) -> eigenvalues + R.
//   k_tet_back    : (grip_tet.cuh) tets: V = Y R, H = Q V max(L, f) V^T Q^T + f/4.
//   k_tet_finish  : contacts: H += Q R diag(max(l, f) - l) R^T Q^T + f/4 (translations),
//                   f = 1e-12 max|l|.
#pragma once
#include "grip_warp_elements.cuh"

namespace grip {

constexpr int TJ = 128;   // threads per k_tet_jacobi2 block (64 matrices)
#ifndef GRIP_JAC_TOL
#define GRIP_JAC_TOL 1e-32   // stop when the squared off-diagonal Frobenius norm is below this fraction
#endif
#ifndef GRIP_JAC_MAXSWEEP
#define GRIP_JAC_MAXSWEEP 30
#endif
#ifdef GRIP_JAC_HIST   // diagnostic build: histogram of Jacobi sweeps, [0] tets (warm) / [1] contacts (cold)
__device__ unsigned long long g_jac_hist[2][GRIP_JAC_MAXSWEEP + 1];
#endif

__host__ __device__ constexpr int up9(int i, int j) { return i * 9 - i * (i - 1) / 2 + (j - i); }   // i <= j

// Cyclic Jacobi, two threads per matrix (Numerical Recipes rotation; same t, c, s as w_jacobi9).
// Both threads of a pair hold the whole S (identical instruction streams, the rotation
// parameters computed redundantly, no communication) and half of the rotation R: thread h
// owns rows 5h .. 5h+4 (thread 1's fifth row is padding).  No shared memory, so the kernel
// co-resides with the CTA-per-env kernels of other lanes.
template <int P, int Q>
__device__ __forceinline__ void jrot2(double* s, double (&Rr)[5][9]) {
  const double apq = s[up9(P, Q)];
  const double d = s[up9(Q, Q)] - s[up9(P, P)];
  const double sg = ((d >= 0.0) == (apq > 0.0)) ? 1.0 : -1.0;
  const double den = fabs(d) + sqrt(d * d + 4.0 * apq * apq);
  const double t = apq != 0.0 ? sg * 2.0 * fabs(apq) / den : 0.0;
  const double c = rsqrt(t * t + 1.0), sn = t * c;
  s[up9(P, P)] -= t * apq;
  s[up9(Q, Q)] += t * apq;
  s[up9(P, Q)] = 0.0;
#pragma unroll
  for (int r = 0; r < 9; ++r) {
    if (r == P || r == Q) continue;
    const int rp = r < P ? up9(r, P) : up9(P, r);
    const int rq = r < Q ? up9(r, Q) : up9(Q, r);
    const double a = s[rp], b = s[rq];
    s[rp] = c * a - sn * b;
    s[rq] = sn * a + c * b;
  }
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const double a = Rr[r][P], b = Rr[r][Q];
    Rr[r][P] = c * a - sn * b;
    Rr[r][Q] = sn * a + c * b;
  }
}

template <int RND>
__device__ __forceinline__ void jround2(double* s, double (&Rr)[5][9]) {
  constexpr int A1 = 1 + (RND + 1) % 9, B1 = 1 + (RND + 8) % 9;
  constexpr int A2 = 1 + (RND + 2) % 9, B2 = 1 + (RND + 7) % 9;
  constexpr int A3 = 1 + (RND + 3) % 9, B3 = 1 + (RND + 6) % 9;
  constexpr int A4 = 1 + (RND + 4) % 9, B4 = 1 + (RND + 5) % 9;
  constexpr int A0 = 0, B0 = 1 + RND % 9;
  if constexpr (B0 != 9) jrot2<(A0 < B0 ? A0 : B0), (A0 < B0 ? B0 : A0)>(s, Rr);
  if constexpr (A1 != 9 && B1 != 9) jrot2<(A1 < B1 ? A1 : B1), (A1 < B1 ? B1 : A1)>(s, Rr);
  if constexpr (A2 != 9 && B2 != 9) jrot2<(A2 < B2 ? A2 : B2), (A2 < B2 ? B2 : A2)>(s, Rr);
  if constexpr (A3 != 9 && B3 != 9) jrot2<(A3 < B3 ? A3 : B3), (A3 < B3 ? B3 : A3)>(s, Rr);
  if constexpr (A4 != 9 && B4 != 9) jrot2<(A4 < B4 ? A4 : B4), (A4 < B4 ? B4 : A4)>(s, Rr);
}

__global__ void __launch_bounds__(TJ) k_tet_jacobi2(const int2* list, const int* n_ptr, const double* Sbuf, double* Wbuf) {
  const int n = *n_ptr;
  const int h = threadIdx.x & 1;
  for (int idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 1; idx < n; idx += (gridDim.x * blockDim.x) >> 1) {
    const int t = list[idx].x;
    const double* Sg = Sbuf + 45 * (size_t)t;
    double s[45];
#pragma unroll
    for (int q = 0; q < 45; ++q) s[q] = Sg[q];
    double Rr[5][9];
#pragma unroll
    for (int r = 0; r < 5; ++r)
#pragma unroll
      for (int c = 0; c < 9; ++c) Rr[r][c] = (5 * h + r == c) ? 1.0 : 0.0;
    int sweep = 0;
    for (; sweep < GRIP_JAC_MAXSWEEP; ++sweep) {
      double off = 0.0, dg = 0.0;
#pragma unroll
      for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int j = i; j < 9; ++j) {
          const double v = s[up9(i, j)];
          if (i == j) dg += v * v;
          else off += v * v;
        }
      off *= 2.0;
      if (off <= GRIP_JAC_TOL * (dg + off) || off == 0.0) break;
      jround2<0>(s, Rr); jround2<1>(s, Rr); jround2<2>(s, Rr);
      jround2<3>(s, Rr); jround2<4>(s, Rr); jround2<5>(s, Rr);
      jround2<6>(s, Rr); jround2<7>(s, Rr); jround2<8>(s, Rr);
    }
#ifdef GRIP_JAC_HIST
    if (h == 0) atomicAdd(&g_jac_hist[gridDim.x == 148 ? 1 : 0][sweep], 1ull);   // contacts: the 148-block launch
#else
    (void)sweep;
#endif
    double* W = Wbuf + 90 * (size_t)t;
    if (h == 0) {
#pragma unroll
      for (int k = 0; k < 9; ++k) W[k] = s[up9(k, k)];
    }
#pragma unroll
    for (int r = 0; r < 5; ++r)
      if (5 * h + r < 9)
#pragma unroll
        for (int c = 0; c < 9; ++c) W[9 + (5 * h + r) * 9 + c] = Rr[r][c];
  }
}

// eig: the tets' warm-start eigenbases (V = V0 R is stored back), or null for cold matrices (V = R)
__global__ void __launch_bounds__(EW * 32) k_tet_finish(Dev D, const int2* list, const int* n_ptr, const double* Wbuf,
                                                        double* eig) {
  __shared__ WarpWS ws[EW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpWS& w = ws[warp];
  const int n = *n_ptr;
  for (int idx = blockIdx.x * EW + warp; idx < n; idx += gridDim.x * EW) {
    const int2 it = list[idx];
    const size_t t = it.x, slot = it.y;
    double* Hg = D.el_H + slot * 144;
    const double* W = Wbuf + 90 * t;
    double* V0 = eig ? eig + 81 * t : nullptr;
    for (int e = lane; e < 144; e += 32) w.H[e] = Hg[e];
    for (int e = lane; e < 81; e += 32) {
      w.S[e] = V0 ? V0[e] : ((e / 9 == e % 9) ? 1.0 : 0.0);   // V0
      w.T[e] = W[9 + e];                                     // R
    }
    double amax = 0.0;
    for (int k = 0; k < 9; ++k) amax = fmax(amax, fabs(W[k]));
    const double f = 1e-12 * amax;
    if (lane < 9) {
      const double lk = W[lane];
      w.sc[lane] = fmax(lk, f) - lk;
    }
    __syncwarp();
    for (int e = lane; e < 81; e += 32) {   // V = V0 R
      const int i = e / 9, j = e - 9 * i;
      double a = 0.0;
      for (int k = 0; k < 9; ++k) a += w.S[i * 9 + k] * w.T[k * 9 + j];
      w.V[e] = a;
    }
    __syncwarp();
    if (V0)
      for (int e = lane; e < 81; e += 32) V0[e] = w.V[e];
    for (int e = lane; e < 108; e += 32) {  // U = Q V, clamped columns only
      const int r = e / 9, k = e - 9 * r, nd = r / 3, a = r - 3 * nd;
      double u = 0.0;
      if (w.sc[k] != 0.0)
        for (int i = 0; i < 3; ++i) u += helmert(i, nd) * w.V[(3 * i + a) * 9 + k];
      w.T[e] = u;
    }
    __syncwarp();
    for (int q = lane; q < 78; q += 32) {
      int i = (int)((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
      while ((i + 1) * (i + 2) / 2 <= q) ++i;
      while (i * (i + 1) / 2 > q) --i;
      const int j = q - i * (i + 1) / 2;
      double s = (i % 3 == j % 3) ? 0.25 * f : 0.0;
      for (int k = 0; k < 9; ++k) {
        const double d = w.sc[k];
        if (d != 0.0) s += d * (w.T[i * 9 + k] * w.T[j * 9 + k]);
      }
      const double v = w.H[i * 12 + j] + s;
      Hg[i * 12 + j] = v;
      if (i != j) Hg[j * 12 + i] = v;
    }
    __syncwarp();
  }
}

}  // namespace grip
