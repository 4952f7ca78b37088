// Batched completion of the tets' eigen-clamp (materials.py:101-113) that k_elements_w deferred.
//
// k_elements_w evaluates every tet warp-per-element and rotates its 9x9 translation-deflated
// S = Q^T H Q into the tet's eigenbasis of the previous Newton iteration (S~ = V0^T S V0).  When
// the Gershgorin discs of S~ do not already prove that nothing is clamped, it stores S~ and the
// unclamped H and appends the tet to jac_list.  Then
//   k_tet_jacobi  : one THREAD per tet, cyclic Jacobi on S~ with the 45 upper entries in
//                   registers (the round-robin schedule is unrolled, every index static) and the
//                   rotation R in shared memory -> eigenvalues + R.  A warp thus works on 32
//                   matrices at once instead of one.
//   k_tet_finish  : one warp per tet, V = V0 R (kept for the next warm start), the reference's
//                   clamp H += Q V diag(max(l, f) - l) V^T Q^T + f/4 (translations), f = 1e-12 max|l|.
#pragma once
#include "grip_warp_elements.cuh"

namespace grip {

constexpr int TJ = 128;   // threads per k_tet_jacobi block (R in shared memory: 81 x TJ doubles)

__host__ __device__ constexpr int up9(int i, int j) { return i * 9 - i * (i - 1) / 2 + (j - i); }   // i <= j

// one Jacobi rotation zeroing s[p][q] (Numerical Recipes form; same t, c, s as w_jacobi9)
template <int P, int Q>
__device__ __forceinline__ void jrot(double* s, double* R, int tid) {
  // branch-free: apq == 0 gives t = 0, c = 1, s = 0 (an exact no-op)
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
  for (int r = 0; r < 9; ++r) {
    double* vp = R + (r * 9 + P) * TJ + tid;
    double* vq = R + (r * 9 + Q) * TJ + tid;
    const double a = *vp, b = *vq;
    *vp = c * a - sn * b;
    *vq = sn * a + c * b;
  }
  asm volatile("" ::: "memory");   // keep each rotation's R traffic local (register pressure)
}

// one round-robin round: the 4 disjoint pairs of round RND (kRR, player 9 = bye)
template <int RND>
__device__ __forceinline__ void jround(double* s, double* R, int tid) {
  constexpr int A1 = 1 + (RND + 1) % 9, B1 = 1 + (RND + 8) % 9;
  constexpr int A2 = 1 + (RND + 2) % 9, B2 = 1 + (RND + 7) % 9;
  constexpr int A3 = 1 + (RND + 3) % 9, B3 = 1 + (RND + 6) % 9;
  constexpr int A4 = 1 + (RND + 4) % 9, B4 = 1 + (RND + 5) % 9;
  constexpr int A0 = 0, B0 = 1 + RND % 9;
  // each pair (min, max); the one touching player 9 is the bye
  if constexpr (B0 != 9) jrot<(A0 < B0 ? A0 : B0), (A0 < B0 ? B0 : A0)>(s, R, tid);
  if constexpr (A1 != 9 && B1 != 9) jrot<(A1 < B1 ? A1 : B1), (A1 < B1 ? B1 : A1)>(s, R, tid);
  if constexpr (A2 != 9 && B2 != 9) jrot<(A2 < B2 ? A2 : B2), (A2 < B2 ? B2 : A2)>(s, R, tid);
  if constexpr (A3 != 9 && B3 != 9) jrot<(A3 < B3 ? A3 : B3), (A3 < B3 ? B3 : A3)>(s, R, tid);
  if constexpr (A4 != 9 && B4 != 9) jrot<(A4 < B4 ? A4 : B4), (A4 < B4 ? B4 : A4)>(s, R, tid);
}

// list[i].x indexes the S (45) / W (90) scratch of the matrix
__global__ void __launch_bounds__(TJ) k_tet_jacobi(const int2* list, const int* n_ptr, const double* Sbuf, double* Wbuf) {
  extern __shared__ double rsm[];   // R: [81][TJ]
  const int n = *n_ptr;
  const int tid = threadIdx.x;
  for (int idx = blockIdx.x * TJ + tid; idx < n; idx += gridDim.x * TJ) {
    const int t = list[idx].x;
    const double* Sg = Sbuf + 45 * (size_t)t;
    double s[45];
#pragma unroll
    for (int q = 0; q < 45; ++q) s[q] = Sg[q];
#pragma unroll
    for (int e = 0; e < 81; ++e) rsm[e * TJ + tid] = (e / 9 == e % 9) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 30; ++sweep) {
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
      if (off <= 1e-32 * (dg + off) || off == 0.0) break;
      jround<0>(s, rsm, tid); jround<1>(s, rsm, tid); jround<2>(s, rsm, tid);
      jround<3>(s, rsm, tid); jround<4>(s, rsm, tid); jround<5>(s, rsm, tid);
      jround<6>(s, rsm, tid); jround<7>(s, rsm, tid); jround<8>(s, rsm, tid);
    }
    double* W = Wbuf + 90 * (size_t)t;
#pragma unroll
    for (int k = 0; k < 9; ++k) W[k] = s[up9(k, k)];
#pragma unroll
    for (int e = 0; e < 81; ++e) W[9 + e] = rsm[e * TJ + tid];
  }
}

// ---- register-only variant: two threads per matrix ----
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
  for (int idx = (blockIdx.x * TJ + threadIdx.x) >> 1; idx < n; idx += (gridDim.x * TJ) >> 1) {
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
    for (int sweep = 0; sweep < 30; ++sweep) {
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
      if (off <= 1e-32 * (dg + off) || off == 0.0) break;
      jround2<0>(s, Rr); jround2<1>(s, Rr); jround2<2>(s, Rr);
      jround2<3>(s, Rr); jround2<4>(s, Rr); jround2<5>(s, Rr);
      jround2<6>(s, Rr); jround2<7>(s, Rr); jround2<8>(s, Rr);
    }
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
