// Neo-Hookean tets (materials.py:116-158) with the reference's eigen-clamp (materials.py:101-113),
// thread-per-tet in registers.
//
// The tet Hessian is H[(m,c),(M,C)] = V0 [mu d_cC WW_mM + c2 WA_Mc WA_mC + c3 WA_mc WA_MC]
// (WA = w A, WW = w w^T, w the 4x3 incidence of Dm^-1, A = F^-T).  Its translation-deflated
// 9x9 block S = Q^T H Q (Q = Helmert (x) I3) has the SAME form with the 4 points contracted
// onto the 3 Helmert rows (wh = h w):
//     S[(i,a),(j,b)] = V0 [mu d_ab WWh_ij + c2 WAh_ja WAh_ib + c3 WAh_ia WAh_jb],
// so S is built from two 3x3 matrices without forming H (no 144-entry matrix, no Q^T H Q).
//
// k_tet_front (one thread per tet): energy, gradient, S in registers, S~ = Y^T S Y with the
//   tet's eigenbasis Y of its previous Newton iteration, Gershgorin test of S~.  When every
//   disc lies above the clamp floor nothing is clamped: H (direct formula) + the lifted
//   translations is written.  Otherwise S~ goes to tet_S and the tet to jac_list.
// k_tet_jacobi2 (grip_tetclamp.cuh): eigenvalues + rotation R of S~, two threads per tet.
// k_tet_back (one warp per deferred tet): V = Y R (the next warm start), S_proj =
//   V diag(max(l, f)) V^T, H = Q S_proj Q^T + f/4 on equal components (translations lifted to
//   f = 1e-12 max|l|, exactly the reference's clamp of the 12x12 matrix).
// Both write H packed (tri12): 624 B per tet instead of the 1152 B of the full matrix.
#pragma once
#include "grip_tetclamp.cuh"

namespace grip {

constexpr int TF = 128;   // threads per k_tet_front block

// Helmert basis (q1 = (1,-1,0,0)/sqrt2, q2 = (1,1,-2,0)/sqrt6, q3 = (1,1,1,-3)/sqrt12) and the
// lower-triangle (row << 4 | column) list of a 12x12 matrix, for k_tet_back
__constant__ double kHelm[3][4] = {{0.70710678118654752440, -0.70710678118654752440, 0.0, 0.0},
                                   {0.40824829046386301637, 0.40824829046386301637, -2.0 * 0.40824829046386301637, 0.0},
                                   {0.28867513459481288225, 0.28867513459481288225, 0.28867513459481288225,
                                    -3.0 * 0.28867513459481288225}};   // the same doubles as helmert()
__constant__ unsigned char kTri78[78] = {
    0x00, 0x10, 0x11, 0x20, 0x21, 0x22, 0x30, 0x31, 0x32, 0x33, 0x40, 0x41, 0x42, 0x43, 0x44, 0x50, 0x51, 0x52, 0x53, 0x54,
    0x55, 0x60, 0x61, 0x62, 0x63, 0x64, 0x65, 0x66, 0x70, 0x71, 0x72, 0x73, 0x74, 0x75, 0x76, 0x77, 0x80, 0x81, 0x82, 0x83,
    0x84, 0x85, 0x86, 0x87, 0x88, 0x90, 0x91, 0x92, 0x93, 0x94, 0x95, 0x96, 0x97, 0x98, 0x99, 0xa0, 0xa1, 0xa2, 0xa3, 0xa4,
    0xa5, 0xa6, 0xa7, 0xa8, 0xa9, 0xaa, 0xb0, 0xb1, 0xb2, 0xb3, 0xb4, 0xb5, 0xb6, 0xb7, 0xb8, 0xb9, 0xba, 0xbb};


__device__ __forceinline__ double helm_c(int i, int k) {   // compile-time foldable Helmert entry
  const double r2 = 0.70710678118654752440, r6 = 0.40824829046386301637, r12 = 0.28867513459481288225;
  return i == 0 ? (k == 0 ? r2 : (k == 1 ? -r2 : 0.0))
                : (i == 1 ? (k < 2 ? r6 : (k == 2 ? -2.0 * r6 : 0.0)) : (k < 3 ? r12 : -3.0 * r12));
}

__global__ void __launch_bounds__(TF) k_tet_front(Dev D, const int* list, int n) {
  const int total = D.twork_off[n];
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int item = blockIdx.x * TF + threadIdx.x; item - lane < total; item += gridDim.x * TF) {
    const bool live = item < total;
    bool defer = false;
    int t = 0;
    size_t slot = 0;
    if (live) {
      int lo = 0, hi = n;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (D.twork_off[mid] <= item) lo = mid;
        else hi = mid;
      }
      const int e = list[lo];
      const int k = item - D.twork_off[lo];
      t = D.tet_off[e] + k;
      slot = (size_t)e * D.cap_el + k;
      const int n0 = D.node_off[e];
      int idx[4];
      V3 x[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        idx[j] = D.tet_nodes[4 * (size_t)t + j];
        x[j] = ld3(D.x + 3 * (size_t)(n0 + idx[j]));
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) D.el_idx[slot * 4 + j] = idx[j];
      double Dmi[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) Dmi[j] = D.tet_Dmi[9 * (size_t)t + j];
      const double V0 = D.tet_V0[t], mu = D.tet_mu[t], lam = D.tet_lam[t];
      double F[9];
      tet_F(x, Dmi, F);
      const double J = det3(F);
      double* Hg = D.el_H + slot * 144;
      if (!(J > 0.0)) {
        atomicOr(&D.tflag[e], ERR_INVERTED);
        D.el_E[slot] = 0.0;
#pragma unroll
        for (int j = 0; j < 12; ++j) D.el_g[slot * 12 + j] = 0.0;
        for (int j = 0; j < 78; ++j) Hg[j] = 0.0;
      } else {
        double A[9];
        {
          double Fi[9];
          inv3(F, Fi);
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) A[3 * i + j] = Fi[3 * j + i];
        }
        double Ic = 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) Ic += F[i] * F[i];
        D.el_E[slot] = V0 * (0.5 * mu * (Ic - 3.0) - mu * log(J) + 0.5 * lam * (J - 1.0) * (J - 1.0));
        const double c1 = lam * (J - 1.0) * J - mu;
        const double c2 = mu - lam * (J - 1.0) * J;
        const double c3 = lam * (2.0 * J - 1.0) * J;
        double w[12];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          w[b] = -(Dmi[b] + Dmi[3 + b] + Dmi[6 + b]);
#pragma unroll
          for (int m = 1; m < 4; ++m) w[3 * m + b] = Dmi[3 * (m - 1) + b];
        }
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < 3; ++b) s += w[3 * m + b] * (mu * F[3 * c + b] + c1 * A[3 * c + b]);
            D.el_g[slot * 12 + 3 * m + c] = s * V0;
          }
        // Helmert-contracted incidence and the two 3x3 factors of S
        double WAh[9], WWh[9];
        {
          double wh[9];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              double s = 0.0;
#pragma unroll
              for (int k = 0; k < 4; ++k) s += helm_c(i, k) * w[3 * k + b];
              wh[3 * i + b] = s;
            }
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              WAh[3 * i + a] = wh[3 * i] * A[3 * a] + wh[3 * i + 1] * A[3 * a + 1] + wh[3 * i + 2] * A[3 * a + 2];
              WWh[3 * i + a] = wh[3 * i] * wh[3 * a] + wh[3 * i + 1] * wh[3 * a + 1] + wh[3 * i + 2] * wh[3 * a + 2];
            }
        }
        double S[45];
#pragma unroll
        for (int p = 0; p < 9; ++p)
#pragma unroll
          for (int q = p; q < 9; ++q) {
            const int i = p / 3, a = p % 3, j = q / 3, b = q % 3;
            S[up9(p, q)] = V0 * ((a == b ? mu * WWh[3 * i + j] : 0.0) + c2 * WAh[3 * j + a] * WAh[3 * i + b] +
                                 c3 * WAh[3 * i + a] * WAh[3 * j + b]);
          }
        // S~ = Y^T S Y (Y = previous eigenbasis, row-major), streamed column by column of Y;
        // upper entries to tet_S, Gershgorin bounds on the fly
        const double* Y = tet_eig_cur(D, e, t);
        double* St = D.tet_S + 45 * (size_t)t;
        double rad[9], dg[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) rad[i] = 0.0;
#pragma unroll
        for (int j = 0; j < 9; ++j) {
          double tj[9];
          {
            double y[9];
#pragma unroll
            for (int r = 0; r < 9; ++r) y[r] = Y[r * 9 + j];
#pragma unroll
            for (int r = 0; r < 9; ++r) {
              double s = 0.0;
#pragma unroll
              for (int c = 0; c < 9; ++c) s += S[r <= c ? up9(r, c) : up9(c, r)] * y[c];
              tj[r] = s;
            }
          }
#pragma unroll
          for (int i = 0; i <= j; ++i) {
            double s = 0.0;
#pragma unroll
            for (int r = 0; r < 9; ++r) s += Y[r * 9 + i] * tj[r];
            St[up9(i, j)] = s;
            if (i == j) {
              dg[i] = s;
            } else {
              rad[i] += fabs(s);
              rad[j] += fabs(s);
            }
          }
        }
        double glo = dg[0] - rad[0], ghi = dg[0] + rad[0], dm = fabs(dg[0]);
#pragma unroll
        for (int i = 1; i < 9; ++i) {
          glo = fmin(glo, dg[i] - rad[i]);
          ghi = fmax(ghi, dg[i] + rad[i]);
          dm = fmax(dm, fabs(dg[i]));
        }
        if (glo > 1e-12 * ghi) {
          // nothing clamped: the warm start carries over to the next half; H itself plus the
          // reference's lifted translation modes
          {
            double* Yn = tet_eig_next(D, e, t);
            for (int q = 0; q < 81; ++q) Yn[q] = Y[q];
          }
          const double f4 = 0.25 * (1e-12 * dm);
          double WA[12], WW[16];
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int c = 0; c < 3; ++c) WA[3 * m + c] = w[3 * m] * A[3 * c] + w[3 * m + 1] * A[3 * c + 1] + w[3 * m + 2] * A[3 * c + 2];
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int M = 0; M < 4; ++M) WW[4 * m + M] = w[3 * m] * w[3 * M] + w[3 * m + 1] * w[3 * M + 1] + w[3 * m + 2] * w[3 * M + 2];
#pragma unroll
          for (int q = 0; q < 12; ++q)
#pragma unroll
            for (int r = 0; r <= q; ++r) {
              const int m = r / 3, c = r % 3, M = q / 3, C = q % 3;
              const double v = V0 * ((c == C ? mu * WW[4 * m + M] : 0.0) + c2 * WA[3 * M + c] * WA[3 * m + C] +
                                     c3 * WA[3 * m + c] * WA[3 * M + C]) + (c == C ? f4 : 0.0);
              Hg[tri12(q, r)] = v;
            }
        } else {
          defer = true;
        }
      }
    }
    // warp-aggregated append of the deferred tets
    const unsigned m = __ballot_sync(0xffffffffu, defer);   // the loop is warp-uniform
    if (m) {
      int base = 0;
      if (lane == 0) base = atomicAdd(D.jac_n, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (defer) D.jac_list[base + __popc(m & lt)] = make_int2(t, (int)slot);
    }
  }
}

// deferred tets: finish the clamp from (eigenvalues, R) -- see the file header
// The next warm start V = Y R goes to the env's other warm-start half (tet_eig_next); the line
// search makes it current unless the env's sweep is redone after a buffer growth (a redone sweep
// must start from the same warm starts, so results do not depend on when buffers grew).
__global__ void __launch_bounds__(EW * 32) k_tet_back(Dev D, const int2* list, const int* n_ptr, const double* Wbuf) {
  __shared__ WarpWS ws[EW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpWS& w = ws[warp];
  const int n = *n_ptr;
  for (int idx = blockIdx.x * EW + warp; idx < n; idx += gridDim.x * EW) {
    const int2 it = list[idx];
    const size_t t = it.x, slot = it.y;
    const int env = (int)(slot / D.cap_el);
    const double* W = Wbuf + 90 * t;
    const double* Y = tet_eig_cur(D, env, t);
    for (int e = lane; e < 81; e += 32) {
      w.S[e] = Y[e];       // Y
      w.T[e] = W[9 + e];   // R
    }
    double amax = 0.0;
    for (int k = 0; k < 9; ++k) amax = fmax(amax, fabs(W[k]));
    const double f = 1e-12 * amax;
    if (lane < 9) w.sc[lane] = fmax(W[lane], f);
    __syncwarp();
    for (int e = lane; e < 81; e += 32) {   // V = Y R
      const int i = e / 9, j = e - 9 * i;
      double a = 0.0;
      for (int k = 0; k < 9; ++k) a += w.S[i * 9 + k] * w.T[k * 9 + j];
      w.V[e] = a;
    }
    __syncwarp();
    {
      double* Yn = tet_eig_next(D, env, t);
      for (int q = lane; q < 81; q += 32) Yn[q] = w.V[q];   // next warm start
    }
    for (int e = lane; e < 81; e += 32) {   // S_proj = V diag(max(l, f)) V^T
      const int i = e / 9, j = e - 9 * i;
      double a = 0.0;
      if (i <= j)
        for (int k = 0; k < 9; ++k) a += w.V[i * 9 + k] * w.sc[k] * w.V[j * 9 + k];
      w.S[e] = a;
    }
    __syncwarp();
    // H = Q S_proj Q^T + f/4 on equal components, as two 3-term contractions:
    // T[(i,c)][(M,C)] = sum_j S[(i,c),(j,C)] h(j,M), then H[(m,c),(M,C)] = sum_i h(i,m) T[(i,c)][(M,C)]
    for (int e = lane; e < 108; e += 32) {
      const int pr = e / 12, q = e - 12 * pr, M = q / 3, C = q - 3 * M;
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int pc = 3 * j + C;
        a += (pr <= pc ? w.S[pr * 9 + pc] : w.S[pc * 9 + pr]) * kHelm[j][M];
      }
      w.T[e] = a;
    }
    __syncwarp();
    double* Hg = D.el_H + slot * 144;
    for (int q = lane; q < 78; q += 32) {   // kTri78 is the packed lower-triangle order: q = tri12(r, c12)
      const int rc = kTri78[q], r = rc >> 4, c12 = rc & 15;   // column <= row
      const int m = r / 3, c = r - 3 * m;
      double s = (c == c12 % 3) ? 0.25 * f : 0.0;
#pragma unroll
      for (int i = 0; i < 3; ++i) s += kHelm[i][m] * w.T[(3 * i + c) * 12 + c12];
      Hg[q] = s;
    }
    __syncwarp();
  }
}

}  // namespace grip
