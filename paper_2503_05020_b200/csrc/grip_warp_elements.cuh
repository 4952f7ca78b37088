// Warp-cooperative element evaluators (one warp per element) and the flat element kernel.
// Same math as grip_elements.cuh (the host-checked spec), re-laid out so lanes own matrix
// entries and every 12x12 / 9x9 matrix lives in the warp's shared-memory workspace.
#pragma once
#include "grip_device.cuh"
#include "grip_warp.cuh"

namespace grip {

using WarpEl = WarpWS;
__device__ __forceinline__ WarpWS& ws_of(WarpWS& e) { return e; }

// lane-select store of a register vector into shared memory (static indices only)
template <int N>
__device__ __forceinline__ void put_vec(double* dst, const double* v, int lane) {
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (lane == i) dst[i] = v[i];
}

__device__ void plane_grad12(V3 wv, V3 u, V3 v, const double C[3][4], double* g12) {
  V3 n = cross(u, v);
  const double iq = 1.0 / dot(n, n);
  const double sq = dot(wv, n) * iq;
  const double nvv[3] = {n.x, n.y, n.z}, wvv[3] = {wv.x, wv.y, wv.z};
  double gn[3], g9[9];
  for (int i = 0; i < 3; ++i) {
    g9[i] = 2.0 * sq * nvv[i];
    gn[i] = 2.0 * sq * wvv[i] - 2.0 * sq * sq * nvv[i];
  }
  double Ju[9], Jv[9];
  skew(v, Ju);
  for (int i = 0; i < 9; ++i) Ju[i] = -Ju[i];
  skew(u, Jv);
  for (int i = 0; i < 3; ++i) {
    double su = 0.0, sv = 0.0;
    for (int k = 0; k < 3; ++k) {
      su += Ju[3 * k + i] * gn[k];
      sv += Jv[3 * k + i] * gn[k];
    }
    g9[3 + i] = su;
    g9[6 + i] = sv;
  }
  for (int k = 0; k < 4; ++k)
    for (int a = 0; a < 3; ++a) {
      double s = 0.0;
      for (int r = 0; r < 3; ++r) s += C[r][k] * g9[3 * r + a];
      g12[3 * k + a] = s;
    }
}

__device__ __constant__ double kPT_C[3][4] = {{1, -1, 0, 0}, {0, -1, 1, 0}, {0, -1, 0, 1}};
__device__ __constant__ double kEE_C[3][4] = {{-1, 0, 1, 0}, {-1, 1, 0, 0}, {0, 0, -1, 1}};

// ---- Neo-Hookean tet (materials.py:116-158); H[(m,c),(M,C)] = V0 [mu d_cC WW_mM + c2 WA_Mc WA_mC + c3 WA_mc WA_MC]
__device__ int w_nh(WarpEl& W, const V3* x, const double* Dmi, double V0, double mu, double lam, double* E, int lane,
                    double* Vtet = nullptr, double* defer_S = nullptr) {
  double F[9];
  tet_F(x, Dmi, F);
  const double J = det3(F);
  if (!(J > 0.0)) return EL_INVERTED;
  double Fi[9], A[9];
  inv3(F, Fi);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) A[3 * i + j] = Fi[3 * j + i];
  double Ic = 0.0;
  for (int i = 0; i < 9; ++i) Ic += F[i] * F[i];
  *E = V0 * (0.5 * mu * (Ic - 3.0) - mu * log(J) + 0.5 * lam * (J - 1.0) * (J - 1.0));
  const double c1 = lam * (J - 1.0) * J - mu;
  const double c2 = mu - lam * (J - 1.0) * J;
  const double c3 = lam * (2.0 * J - 1.0) * J;
  double w[12];
  for (int b = 0; b < 3; ++b) {
    w[b] = -(Dmi[b] + Dmi[3 + b] + Dmi[6 + b]);
    for (int m = 1; m < 4; ++m) w[3 * m + b] = Dmi[3 * (m - 1) + b];
  }
  double g[12], WA[12], WW[16];
  for (int m = 0; m < 4; ++m)
    for (int c = 0; c < 3; ++c) {
      double s = 0.0, t = 0.0;
      for (int b = 0; b < 3; ++b) {
        s += w[3 * m + b] * (mu * F[3 * c + b] + c1 * A[3 * c + b]);
        t += w[3 * m + b] * A[3 * c + b];
      }
      g[3 * m + c] = s * V0;
      WA[3 * m + c] = t;
    }
  for (int m = 0; m < 4; ++m)
    for (int M = 0; M < 4; ++M) WW[4 * m + M] = w[3 * m] * w[3 * M] + w[3 * m + 1] * w[3 * M + 1] + w[3 * m + 2] * w[3 * M + 2];
  put_vec<12>(W.g, g, lane);
  put_vec<12>(W.sc, WA, lane);
  put_vec<16>(W.sc + 12, WW, lane);
  __syncwarp();
  for (int e = lane; e < 144; e += 32) {
    const int mc = e / 12, MC = e % 12, m = mc / 3, c = mc % 3, M = MC / 3, C = MC % 3;
    const double* wa = W.sc;
    W.H[e] = V0 * ((c == C ? mu * W.sc[12 + 4 * m + M] : 0.0) + c2 * wa[3 * M + c] * wa[3 * m + C] +
                   c3 * wa[3 * m + c] * wa[3 * M + C]);
  }
  __syncwarp();
  return w_clamp_stencil(ws_of(W), lane, Vtet, Vtet, defer_S) ? EL_DEFERRED : 0;
}

// ---- point-triangle stencil (contact.py:178-211, 283-303)
__device__ int w_pt(WarpEl& W, const V3* x, double kappa, double dhat, double* E, int lane, double* defer_S = nullptr) {
  double bary[3];
  int reg;
  const double D = pt_closest(x[0], x[1], x[2], x[3], bary, &reg);
  if (!(D > 0.0)) return EL_BAD_D;
  if (!(D < dhat * dhat)) return 0;
  double b, f1, f2;
  barrier_D(D, dhat, &b, &f1, &f2);
  *E = kappa * b;
  double gD[12];
  if (reg == 6) {
    plane_grad12(x[0] - x[1], x[2] - x[1], x[3] - x[1], kPT_C, gD);
  } else if (reg >= 3) {
    const int sa = reg == 3 ? 1 : (reg == 4 ? 2 : 3);
    const int sb = reg == 3 ? 2 : (reg == 4 ? 3 : 1);
    pe_grad12(x[0], x[sa], x[sb], 0, sa, sb, gD);
  } else {
    pp_grad12(x[0], x[1 + reg], 0, 1 + reg, gD);
  }
  double g[12];
  for (int i = 0; i < 12; ++i) g[i] = kappa * f1 * gD[i];
  put_vec<12>(W.g, g, lane);
  put_vec<12>(W.sc, gD, lane);
  __syncwarp();
  if (reg == 6) {
    w_plane12(ws_of(W), x[0] - x[1], x[2] - x[1], x[3] - x[1], kPT_C, lane);
    for (int e = lane; e < 144; e += 32) {
      const int i = e / 12, j = e % 12;
      W.H[e] = kappa * (f2 * W.sc[i] * W.sc[j] + f1 * W.H[e]);
    }
    __syncwarp();
    if (w_clamp_stencil(ws_of(W), lane, nullptr, nullptr, defer_S)) return EL_ACTIVE | EL_DEFERRED;
  } else {
    w_rank1(ws_of(W), kappa * f2, lane);
  }
  return EL_ACTIVE;
}

// ---- edge-edge stencil with the parallel mollifier (contact.py:213-269, 305-340)
__device__ int w_ee(WarpEl& W, const V3* x, double eps_x, double kappa, double dhat, double* E, int lane,
                    double* defer_S = nullptr) {
  double s, t;
  const double D = ee_closest(x[0], x[1], x[2], x[3], &s, &t);
  if (!(D > 0.0)) return EL_BAD_D;
  if (!(D < dhat * dhat)) return 0;
  const double c = cross_norm_sq(x, nullptr, nullptr);
  double m, dm, d2m;
  edge_mollifier(c, eps_x, &m, &dm, &d2m);
  double b, f1, f2;
  barrier_D(D, dhat, &b, &f1, &f2);
  *E = kappa * m * b;
  const bool s_in = s > 0.0 && s < 1.0, t_in = t > 0.0 && t < 1.0;
  const bool plane = s_in && t_in;
  const bool moll = dm != 0.0 || d2m != 0.0;
  double gD[12], gc[12];
  if (plane) {
    plane_grad12(x[2] - x[0], x[1] - x[0], x[3] - x[2], kEE_C, gD);
  } else if (s_in) {
    const int ps = t < 0.5 ? 2 : 3;
    pe_grad12(x[ps], x[0], x[1], ps, 0, 1, gD);
  } else if (t_in) {
    const int ps = s < 0.5 ? 0 : 1;
    pe_grad12(x[ps], x[2], x[3], ps, 2, 3, gD);
  } else {
    const int sa = s < 0.5 ? 0 : 1, sb = t < 0.5 ? 2 : 3;
    pp_grad12(x[sa], x[sb], sa, sb, gD);
  }
  for (int i = 0; i < 12; ++i) gc[i] = 0.0;
  if (moll) cross_norm_sq(x, gc, nullptr);
  double g[12];
  for (int i = 0; i < 12; ++i) g[i] = kappa * (m * f1 * gD[i] + b * dm * gc[i]);
  put_vec<12>(W.g, g, lane);
  put_vec<12>(W.sc, gD, lane);
  put_vec<12>(W.sc + 12, gc, lane);
  __syncwarp();
  if (!plane && !moll) {
    w_rank1(ws_of(W), kappa * m * f2, lane);
    return EL_ACTIVE;
  }
  if (plane) w_plane12(ws_of(W), x[2] - x[0], x[1] - x[0], x[3] - x[2], kEE_C, lane);
  // mollifier curvature d2c (cross_norm_sq Hessian) per entry
  const V3 u = x[1] - x[0], v = x[3] - x[2];
  const double qu = dot(u, u), qv = dot(v, v), suv = dot(u, v);
  const double uv[3] = {u.x, u.y, u.z}, vv[3] = {v.x, v.y, v.z};
  for (int e = lane; e < 144; e += 32) {
    const int i = e / 12, j = e % 12;
    const double gi = W.sc[i], gj = W.sc[j], ci = W.sc[12 + i], cj = W.sc[12 + j];
    const double hb = f2 * gi * gj + (plane ? f1 * W.H[e] : 0.0);
    double hm = 0.0;
    if (moll) {
      const int k = i / 3, l = j / 3, a = i % 3, bb = j % 3;
      const double sg = ((k & 1) ? 1.0 : -1.0) * ((l & 1) ? 1.0 : -1.0);
      double blk;
      const double dab = a == bb ? 1.0 : 0.0;
      if (k < 2 && l < 2) blk = 2.0 * qv * dab - 2.0 * vv[a] * vv[bb];
      else if (k >= 2 && l >= 2) blk = 2.0 * qu * dab - 2.0 * uv[a] * uv[bb];
      else if (k < 2) blk = 4.0 * uv[a] * vv[bb] - 2.0 * vv[a] * uv[bb] - 2.0 * suv * dab;
      else blk = 4.0 * uv[bb] * vv[a] - 2.0 * vv[bb] * uv[a] - 2.0 * suv * dab;
      hm = d2m * ci * cj + dm * sg * blk;
    }
    W.H[e] = kappa * (m * hb + b * hm + dm * ci * f1 * gj + f1 * gi * dm * cj);
  }
  __syncwarp();
  if (w_clamp_stencil(ws_of(W), lane, nullptr, nullptr, defer_S)) return EL_ACTIVE | EL_DEFERRED;
  return EL_ACTIVE;
}

// ---- lagged friction anchor (contact.py:475-524), PSD by construction
__device__ double w_friction(WarpEl& W, const V3* x, const V3* xp, const double* gamma, const double* T, double lam,
                             double mu, double eps_v, double dt, int lane) {
  double g[12];
  const double h = eps_v * dt;
  V3 u = V3{0.0, 0.0, 0.0};
  for (int k = 0; k < 4; ++k) u = u + gamma[k] * (x[k] - xp[k]);
  const double s0 = T[0] * u.x + T[2] * u.y + T[4] * u.z;
  const double s1 = T[1] * u.x + T[3] * u.y + T[5] * u.z;
  const double y = sqrt(s0 * s0 + s1 * s1);
  double f0, f1;
  if (y < h) {
    f1 = 2.0 * y / h - (y / h) * (y / h);
    f0 = y * y / h - y * y * y / (3.0 * h * h);
  } else {
    f1 = 1.0;
    f0 = y - h / 3.0;
  }
  const double sc = mu * lam;
  const double ratio = y > 1e-14 ? f1 / fmax(y, 1e-300) : 2.0 / h;
  const double q0 = ratio * s0, q1 = ratio * s1;
  const double g3[3] = {T[0] * q0 + T[1] * q1, T[2] * q0 + T[3] * q1, T[4] * q0 + T[5] * q1};
  for (int k = 0; k < 4; ++k)
    for (int a = 0; a < 3; ++a) g[3 * k + a] = sc * gamma[k] * g3[a];
  const double df1 = y < h ? 2.0 / h - 2.0 * y / (h * h) : 0.0;
  double u0 = 0.0, u1 = 0.0;
  if (y > 1e-14) {
    const double iy = 1.0 / fmax(y, 1e-300);
    u0 = s0 * iy;
    u1 = s1 * iy;
  }
  const double M2[4] = {df1 * u0 * u0 + ratio * (1.0 - u0 * u0), df1 * u0 * u1 - ratio * u0 * u1,
                        df1 * u1 * u0 - ratio * u1 * u0, df1 * u1 * u1 + ratio * (1.0 - u1 * u1)};
  double M3[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l) s += T[2 * i + k] * M2[2 * k + l] * T[2 * j + l];
      M3[3 * i + j] = s;
    }
  put_vec<12>(W.g, g, lane);
  put_vec<9>(W.sc, M3, lane);
  double gm[4] = {gamma[0], gamma[1], gamma[2], gamma[3]};
  put_vec<4>(W.sc + 9, gm, lane);
  __syncwarp();
  for (int e = lane; e < 144; e += 32) {
    const int ka = e / 12, lb = e % 12;
    W.H[e] = sc * W.sc[9 + ka / 3] * W.sc[9 + lb / 3] * W.sc[3 * (ka % 3) + lb % 3];
  }
  __syncwarp();
  return sc * f0;
}

// ---- ABD orthogonality (materials.py:161-188) + clamp (solver.py:509-515)
__device__ double w_abd(WarpEl& W, const double* A, double kV, int lane) {
  double S[9], AAt[9], g[12];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0, t = 0.0;
      for (int k = 0; k < 3; ++k) {
        s += A[3 * k + i] * A[3 * k + j];
        t += A[3 * i + k] * A[3 * j + k];
      }
      S[3 * i + j] = s - (i == j ? 1.0 : 0.0);
      AAt[3 * i + j] = t;
    }
  double E = 0.0;
  for (int i = 0; i < 9; ++i) E += S[i] * S[i];
  E *= kV;
  for (int i = 0; i < 3; ++i) g[i] = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += A[3 * a + k] * S[3 * k + b];
      g[3 + 3 * a + b] = 4.0 * kV * s;
    }
  put_vec<12>(W.g, g, lane);
  WarpWS& w = ws_of(W);
  for (int e = lane; e < 81; e += 32) {
    const int ab = e / 9, cd = e % 9, a = ab / 3, b = ab % 3, c = cd / 3, d = cd % 3;
    w.S[e] = 4.0 * kV * ((a == c ? S[3 * d + b] : 0.0) + A[3 * a + d] * A[3 * c + b] + (b == d ? AAt[3 * a + c] : 0.0));
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
  w_jacobi9(w, lane);
  double amax = 0.0;
  for (int k = 0; k < 9; ++k) amax = fmax(amax, fabs(w.S[k * 10]));
  const double f = 1e-12 * amax;
  for (int e = lane; e < 81; e += 32) {
    const int i = e / 9, j = e % 9;
    double s = 0.0;
    for (int k = 0; k < 9; ++k) s += w.V[i * 9 + k] * fmax(w.S[k * 10], f) * w.V[j * 9 + k];
    w.T[e] = s;
  }
  __syncwarp();
  for (int e = lane; e < 144; e += 32) {
    const int i = e / 12, j = e % 12;
    double v;
    if (i < 3 || j < 3) v = (i == j) ? f : 0.0;
    else v = 0.5 * (w.T[(i - 3) * 9 + (j - 3)] + w.T[(j - 3) * 9 + (i - 3)]);
    w.H[e] = v;
  }
  __syncwarp();
  return E;
}

// write one element's outputs (coalesced 144-entry Hessian store)
__device__ __forceinline__ void w_store(const Dev& D, size_t slot, WarpEl& W, double E, const int* idx, int lane) {
  double* H = D.el_H + slot * 144;
  for (int e = lane; e < 144; e += 32) H[e] = W.H[e];
  if (lane < 12) D.el_g[slot * 12 + lane] = W.g[lane];
  if (lane == 0) D.el_E[slot] = E;
  if (lane < 4) D.el_idx[slot * 4 + lane] = idx[lane];
}

constexpr int EW = 8;  // warps per block of k_elements_w

// Newton sweep 2/4 (warp per element): element slots per env [tets | abd | contacts | anchors]
#ifndef GRIP_EW_MINB
#define GRIP_EW_MINB 2   // blocks per SM k_elements_w is compiled for (register cap 128)
#endif
__global__ void __launch_bounds__(EW * 32, GRIP_EW_MINB) k_elements_w(Dev D, const int* list, int n) {
  __shared__ WarpEl ws[EW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpEl& W = ws[warp];
  const int total = D.cwork_off[n];   // contacts + anchors (tets and ABD bodies: second stream)
  for (int item = blockIdx.x * EW + warp; item < total; item += gridDim.x * EW) {
    int lo = 0, hi = n;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (D.cwork_off[mid] <= item) lo = mid;
      else hi = mid;
    }
    const int e = list[lo];
    const EnvIx E = env_ix(D, e);
    const double* P = P_(D, e);
    int k = item - D.cwork_off[lo];
    const size_t elbase = (size_t)e * D.cap_el;
    double Eel = 0.0;
    int idx[4];
    size_t slot;
    if (k < D.n_act[e]) {
      slot = elbase + D.max_tet + D.max_abd + k;
      const int code = D.act[(size_t)e * D.cap_act + k];
      const bool is_ee = code >= D.cap_pt;
      const int* row = is_ee ? D.c1_ee + ((size_t)e * D.cap_ee + (code - D.cap_pt)) * 4
                             : D.c1_pt + ((size_t)e * D.cap_pt + code) * 4;
      V3 x[4];
      for (int j = 0; j < 4; ++j) {
        idx[j] = row[j];
        x[j] = ld3(D.sv_pos + 3 * (size_t)(E.s0 + idx[j]));
      }
      const size_t cs = (size_t)e * D.cap_act + k;
      double* dS = D.cjac_S + 45 * cs;
      int fl;
      if (is_ee) {
        const int* eid = D.c1_eid + ((size_t)e * D.cap_ee + (code - D.cap_pt)) * 2;
        const double epsx = D.edge_rest_sq[E.ed0 + eid[0]] * D.edge_rest_sq[E.ed0 + eid[1]];
        fl = w_ee(W, x, epsx, P[GRIP_P_KAPPA], P[GRIP_P_DHAT], &Eel, lane, dS);
      } else {
        fl = w_pt(W, x, P[GRIP_P_KAPPA], P[GRIP_P_DHAT], &Eel, lane, dS);
      }
      if ((fl & EL_DEFERRED) && lane == 0) D.cjac_list[atomicAdd(D.cjac_n, 1)] = make_int2((int)cs, (int)slot);
    } else {
      k -= D.n_act[e];
      slot = elbase + D.max_tet + D.max_abd + D.cap_act + k;
      const size_t ai = (size_t)e * D.cap_anc + k;
      V3 x[4], xp[4];
      for (int j = 0; j < 4; ++j) {
        idx[j] = D.anc_v[4 * ai + j];
        x[j] = ld3(D.sv_pos + 3 * (size_t)(E.s0 + idx[j]));
        xp[j] = ld3(D.surf_prev + 3 * (size_t)(E.s0 + idx[j]));
      }
      Eel = w_friction(W, x, xp, D.anc_gamma + 4 * ai, D.anc_T + 6 * ai, D.anc_lam[ai], D.anc_mu[ai], P[GRIP_P_EPSV],
                       P[GRIP_P_DT], lane);
    }
    w_store(D, slot, W, Eel, idx, lane);
    __syncwarp();
  }
}

// ABD orthogonality elements (materials.py:161-188) of the listed envs, warp per env: they depend on
// x only, so they run on the second stream with the tets, ahead of the static blocks
__global__ void __launch_bounds__(EW * 32) k_abd_w(Dev D, const int* list, int n) {
  __shared__ WarpEl ws[EW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpEl& W = ws[warp];
  for (int pos = blockIdx.x * EW + warp; pos < n; pos += gridDim.x * EW) {
    const int e = list[pos];
    if (D.ns_done[e]) continue;
    const EnvIx E = env_ix(D, e);
    const size_t elbase = (size_t)e * D.cap_el;
    for (int k = 0; k < E.na; ++k) {
      const int a = E.a0 + k;
      const size_t slot = elbase + D.max_tet + k;
      const int pn = D.abd_node[a];
      int idx[4];
      for (int j = 0; j < 4; ++j) idx[j] = pn + j;
      const double Eel = w_abd(W, D.x + 3 * (size_t)(E.n0 + pn) + 3, D.abd_kV[a], lane);
      w_store(D, slot, W, Eel, idx, lane);
      __syncwarp();
    }
  }
}

// standalone element evaluation for GPU unit tests (type: 0 PT, 1 EE, 2 NH, 3 ABD, 4 friction)
__global__ void k_debug_elements(int type, int n, const double* in, int stride, double* E, double* g, double* H,
                                 int* flags) {
  __shared__ WarpEl ws[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpEl& W = ws[warp];
  for (int item = blockIdx.x * 4 + warp; item < n; item += gridDim.x * 4) {
    const double* p = in + (size_t)item * stride;
    V3 x[4];
    for (int j = 0; j < 4; ++j) x[j] = ld3(p + 3 * j);
    double e = 0.0;
    int fl = 0;
    for (int i = lane; i < 144; i += 32) W.H[i] = 0.0;
    if (lane < 12) W.g[lane] = 0.0;
    __syncwarp();
    if (type == 0) fl = w_pt(W, x, p[12], p[13], &e, lane);
    else if (type == 1) fl = w_ee(W, x, p[12], p[13], p[14], &e, lane);
    else if (type == 2) fl = w_nh(W, x, p + 12, p[21], p[22], p[23], &e, lane);
    else if (type == 3) e = w_abd(W, p, p[9], lane);
    else {
      V3 xp[4];
      for (int j = 0; j < 4; ++j) xp[j] = ld3(p + 12 + 3 * j);
      e = w_friction(W, x, xp, p + 24, p + 28, p[34], p[35], p[36], p[37], lane);
    }
    for (int i = lane; i < 144; i += 32) H[(size_t)item * 144 + i] = W.H[i];
    if (lane < 12) g[(size_t)item * 12 + lane] = W.g[lane];
    if (lane == 0) {
      E[item] = e;
      flags[item] = fl;
    }
    __syncwarp();
  }
}

// grip_debug_chain, contacts: the production path of k_elements_w for standalone PT / EE stencils
// (in: x(12), kappa, dhat / x(12), eps_x, kappa, dhat): clamps that fail the cold Cholesky test are
// deferred to the batched eigensolve (D.cjac_*: k_tet_jacobi2 + k_tet_finish), exactly as in a sweep
__global__ void k_debug_contacts(Dev D, int type, int n, const double* in, int stride, int* flags) {
  __shared__ WarpEl ws[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpEl& W = ws[warp];
  for (int item = blockIdx.x * 4 + warp; item < n; item += gridDim.x * 4) {
    const double* p = in + (size_t)item * stride;
    V3 x[4];
    for (int j = 0; j < 4; ++j) x[j] = ld3(p + 3 * j);
    double e = 0.0;
    int fl = 0;
    for (int i = lane; i < 144; i += 32) W.H[i] = 0.0;
    if (lane < 12) W.g[lane] = 0.0;
    __syncwarp();
    double* dS = D.cjac_S + 45 * (size_t)item;
    if (type == 0) fl = w_pt(W, x, p[12], p[13], &e, lane, dS);
    else fl = w_ee(W, x, p[12], p[13], p[14], &e, lane, dS);
    if ((fl & EL_DEFERRED) && lane == 0) D.cjac_list[atomicAdd(D.cjac_n, 1)] = make_int2(item, item);
    int idx[4] = {0, 1, 2, 3};
    w_store(D, (size_t)item, W, e, idx, lane);
    if (lane == 0) flags[item] = fl;
    __syncwarp();
  }
}

}  // namespace grip
