// Per-element physics of the IPC step: closest points, squared-distance
// derivatives, barrier / mollifier / friction / Neo-Hookean / ABD element
// energies with projected Hessians, CCD per stencil, cubic pencils, stress.
//
// One function per reference routine, each citing the gripsim file:line it
// follows (reference: /root/reference/pkg/src/gripsim).  All fp64.
#pragma once
#include "grip_math.cuh"

namespace grip {

// ---------------------------------------------------------------------------
// closest points (geometry/distances.py:61-152)
// ---------------------------------------------------------------------------

// region: 0..2 vertex t0/t1/t2, 3 edge t0t1, 4 edge t1t2, 5 edge t2t0, 6 face.
// Priority order vertex0, vertex1, vertex2, edge3, edge5, edge4, face (distances.py:97-117).
GHD double pt_closest(V3 p, V3 t0, V3 t1, V3 t2, double* bary, int* region) {
  V3 ab = t1 - t0, ac = t2 - t0;
  V3 ap = p - t0, bp = p - t1, cp = p - t2;
  double d1 = dot(ab, ap), d2 = dot(ac, ap);
  double d3 = dot(ab, bp), d4 = dot(ac, bp);
  double d5 = dot(ab, cp), d6 = dot(ac, cp);
  double va = d3 * d6 - d5 * d4;
  double vb = d5 * d2 - d1 * d6;
  double vc = d1 * d4 - d3 * d2;
  double b0, b1, b2;
  int r;
  if (d1 <= 0.0 && d2 <= 0.0) {
    b0 = 1.0; b1 = 0.0; b2 = 0.0; r = 0;
  } else if (d3 >= 0.0 && d4 <= d3) {
    b0 = 0.0; b1 = 1.0; b2 = 0.0; r = 1;
  } else if (d6 >= 0.0 && d5 <= d6) {
    b0 = 0.0; b1 = 0.0; b2 = 1.0; r = 2;
  } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double v = (d1 != d3) ? d1 / (d1 - d3) : 0.0;
    b0 = 1.0 - v; b1 = v; b2 = 0.0; r = 3;
  } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double w = (d2 != d6) ? d2 / (d2 - d6) : 0.0;
    b0 = 1.0 - w; b1 = 0.0; b2 = w; r = 5;
  } else if (va <= 0.0 && d4 - d3 >= 0.0 && d5 - d6 >= 0.0) {
    double den = (d4 - d3) + (d5 - d6);
    double w = (den != 0.0) ? (d4 - d3) / den : 0.0;
    b0 = 0.0; b1 = 1.0 - w; b2 = w; r = 4;
  } else {
    double den = va + vb + vc;
    double v = (den != 0.0) ? vb / den : 0.0;
    double w = (den != 0.0) ? vc / den : 0.0;
    b0 = 1.0 - v - w; b1 = v; b2 = w; r = 6;
  }
  if (bary) { bary[0] = b0; bary[1] = b1; bary[2] = b2; }
  if (region) *region = r;
  V3 c = b0 * t0 + b1 * t1 + b2 * t2;
  V3 d = p - c;
  return dot(d, d);
}

GHD double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

GHD double ee_closest(V3 a0, V3 a1, V3 b0, V3 b1, double* s_out, double* t_out) {
  V3 d1 = a1 - a0, d2 = b1 - b0, r = a0 - b0;
  double a = dot(d1, d1), e = dot(d2, d2), f = dot(d2, r), c = dot(d1, r), b = dot(d1, d2);
  double den = a * e - b * b;
  double s = den > 0.0 ? clip01((b * f - c * e) / den) : 0.0;
  double t = (b * s + f) / e;
  if (t < 0.0) s = clip01(-c / a);
  else if (t > 1.0) s = clip01((b - c) / a);
  t = clip01(t);
  V3 d = (a0 + s * d1) - (b0 + t * d2);
  if (s_out) *s_out = s;
  if (t_out) *t_out = t;
  return dot(d, d);
}

// ---------------------------------------------------------------------------
// squared-distance derivatives (distances.py:160-382)
// ---------------------------------------------------------------------------

// gradient of |a-b|^2 placed at stencil slots (sa, sb) of a 12-vector
GHD void pp_grad12(V3 a, V3 b, int sa, int sb, double* g) {
  for (int i = 0; i < 12; ++i) g[i] = 0.0;
  V3 d = a - b;
  g[3 * sa + 0] = 2.0 * d.x; g[3 * sa + 1] = 2.0 * d.y; g[3 * sa + 2] = 2.0 * d.z;
  g[3 * sb + 0] = -2.0 * d.x; g[3 * sb + 1] = -2.0 * d.y; g[3 * sb + 2] = -2.0 * d.z;
}

// gradient of the interior point-edge squared distance, slots (sp, s0, s1); distances.py:177-227
GHD void pe_grad12(V3 p, V3 e0, V3 e1, int sp, int s0, int s1, double* g) {
  for (int i = 0; i < 12; ++i) g[i] = 0.0;
  V3 w = p - e0, u = e1 - e0;
  double sq = dot(w, u) / dot(u, u);
  V3 gw = 2.0 * w - (2.0 * sq) * u;
  V3 gu = (-2.0 * sq) * w + (2.0 * sq * sq) * u;
  V3 g0 = V3{-gw.x - gu.x, -gw.y - gu.y, -gw.z - gu.z};
  st3(g + 3 * sp, gw);
  st3(g + 3 * s0, g0);
  st3(g + 3 * s1, gu);
}

GHD void skew(V3 c, double* M) {
  M[0] = 0.0;  M[1] = -c.z; M[2] = c.y;
  M[3] = c.z;  M[4] = 0.0;  M[5] = -c.x;
  M[6] = -c.y; M[7] = c.x;  M[8] = 0.0;
}

// D = (w.n)^2/|n|^2, n = u x v: grad g9 and Hessian H9 over (w,u,v); distances.py:230-277
GHD void plane_derivs(V3 w, V3 u, V3 v, double* g9, double* H9) {
  V3 n = cross(u, v);
  double iq = 1.0 / dot(n, n);
  double sq = dot(w, n) * iq;
  double nv[3] = {n.x, n.y, n.z}, wv[3] = {w.x, w.y, w.z};
  double gn[3];
  for (int i = 0; i < 3; ++i) {
    g9[i] = 2.0 * sq * nv[i];
    gn[i] = 2.0 * sq * wv[i] - 2.0 * sq * sq * nv[i];
  }
  double Hww[9], Hwn[9], Hnn[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double dij = (i == j) ? 1.0 : 0.0;
      Hww[3 * i + j] = 2.0 * iq * nv[i] * nv[j];
      Hwn[3 * i + j] = 2.0 * iq * nv[i] * wv[j] + 2.0 * sq * dij - 4.0 * sq * iq * nv[i] * nv[j];
      Hnn[3 * i + j] = 2.0 * iq * wv[i] * wv[j] - 4.0 * sq * iq * (nv[i] * wv[j] + wv[i] * nv[j]) - 2.0 * sq * sq * dij
                       + 8.0 * sq * sq * iq * nv[i] * nv[j];
    }
  double Ju[9], Jv[9], cu[9];
  skew(v, Ju);
  for (int i = 0; i < 9; ++i) Ju[i] = -Ju[i];
  skew(u, Jv);
  skew(V3{gn[0], gn[1], gn[2]}, cu);
  for (int i = 0; i < 3; ++i) {
    double su = 0.0, sv = 0.0;
    for (int k = 0; k < 3; ++k) {
      su += Ju[3 * k + i] * gn[k];
      sv += Jv[3 * k + i] * gn[k];
    }
    g9[3 + i] = su;
    g9[6 + i] = sv;
  }
  // blocks: Hwu = Hwn Ju, Hwv = Hwn Jv, Huu = Ju^T Hnn Ju, Hvv = Jv^T Hnn Jv, Huv = Ju^T Hnn Jv - [gn]x
  double HnJu[9], HnJv[9];
  mul33(Hnn, Ju, HnJu);
  mul33(Hnn, Jv, HnJv);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double wu = 0.0, wv2 = 0.0, uu = 0.0, vv = 0.0, uv = 0.0;
      for (int k = 0; k < 3; ++k) {
        wu += Hwn[3 * i + k] * Ju[3 * k + j];
        wv2 += Hwn[3 * i + k] * Jv[3 * k + j];
        uu += Ju[3 * k + i] * HnJu[3 * k + j];
        vv += Jv[3 * k + i] * HnJv[3 * k + j];
        uv += Ju[3 * k + i] * HnJv[3 * k + j];
      }
      uv -= cu[3 * i + j];
      H9[(0 + i) * 9 + 0 + j] = Hww[3 * i + j];
      H9[(0 + i) * 9 + 3 + j] = wu;
      H9[(3 + j) * 9 + 0 + i] = wu;
      H9[(0 + i) * 9 + 6 + j] = wv2;
      H9[(6 + j) * 9 + 0 + i] = wv2;
      H9[(3 + i) * 9 + 3 + j] = uu;
      H9[(6 + i) * 9 + 6 + j] = vv;
      H9[(3 + i) * 9 + 6 + j] = uv;
      H9[(6 + j) * 9 + 3 + i] = uv;
    }
}

// chain (w,u,v) derivatives onto 4 stencil points: coefficient of reduced
// variable r on point k is C[r][k] (PT: w=p-t0,u=t1-t0,v=t2-t0; EE: w=b0-a0,u=a1-a0,v=b1-b0)
GHD void chain4(const double C[3][4], const double* g9, const double* H9, double* g12, double* H12) {
  for (int k = 0; k < 4; ++k)
    for (int a = 0; a < 3; ++a) {
      double s = 0.0;
      for (int r = 0; r < 3; ++r) s += C[r][k] * g9[3 * r + a];
      g12[3 * k + a] = s;
    }
  for (int k = 0; k < 4; ++k)
    for (int l = 0; l < 4; ++l)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          double s = 0.0;
          for (int r = 0; r < 3; ++r) {
            if (C[r][k] == 0.0) continue;
            for (int q = 0; q < 3; ++q) {
              if (C[q][l] == 0.0) continue;
              s += C[r][k] * C[q][l] * H9[(3 * r + a) * 9 + 3 * q + b];
            }
          }
          H12[(3 * k + a) * 12 + 3 * l + b] = s;
        }
}

GHD void pt_plane12(const V3* x, double* g12, double* H12) {
  const double C[3][4] = {{1, -1, 0, 0}, {0, -1, 1, 0}, {0, -1, 0, 1}};
  double g9[9], H9[81];
  plane_derivs(x[0] - x[1], x[2] - x[1], x[3] - x[1], g9, H9);
  chain4(C, g9, H9, g12, H12);
}

GHD void ee_plane12(const V3* x, double* g12, double* H12) {
  const double C[3][4] = {{-1, 0, 1, 0}, {-1, 1, 0, 0}, {0, 0, -1, 1}};
  double g9[9], H9[81];
  plane_derivs(x[2] - x[0], x[1] - x[0], x[3] - x[2], g9, H9);
  chain4(C, g9, H9, g12, H12);
}

// c = |u x v|^2 (Lagrange identity), grad/Hessian over 4 points; distances.py:346-382
GHD double cross_norm_sq(const V3* x, double* g, double* H) {
  V3 u = x[1] - x[0], v = x[3] - x[2];
  double qu = dot(u, u), qv = dot(v, v), s = dot(u, v);
  double c = qu * qv - s * s;
  if (g) {
    V3 gu = (2.0 * qv) * u - (2.0 * s) * v;
    V3 gv = (2.0 * qu) * v - (2.0 * s) * u;
    st3(g + 0, (-1.0) * gu);
    st3(g + 3, gu);
    st3(g + 6, (-1.0) * gv);
    st3(g + 9, gv);
  }
  if (H) {
    double uv[3] = {u.x, u.y, u.z}, vv[3] = {v.x, v.y, v.z};
    double Huu[9], Hvv[9], Huv[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double dij = i == j ? 1.0 : 0.0;
        Huu[3 * i + j] = 2.0 * qv * dij - 2.0 * vv[i] * vv[j];
        Hvv[3 * i + j] = 2.0 * qu * dij - 2.0 * uv[i] * uv[j];
        Huv[3 * i + j] = 4.0 * uv[i] * vv[j] - 2.0 * vv[i] * uv[j] - 2.0 * s * dij;
      }
    const double sg[4] = {-1.0, 1.0, -1.0, 1.0};
    for (int k = 0; k < 4; ++k)
      for (int l = 0; l < 4; ++l)
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            double b;
            if (k < 2 && l < 2) b = Huu[3 * i + j];
            else if (k >= 2 && l >= 2) b = Hvv[3 * i + j];
            else if (k < 2) b = Huv[3 * i + j];
            else b = Huv[3 * j + i];
            H[(3 * k + i) * 12 + 3 * l + j] = sg[k] * sg[l] * b;
          }
  }
  return c;
}

// ---------------------------------------------------------------------------
// barrier, mollifiers (contact.py:49-90, 258-269)
// ---------------------------------------------------------------------------

GHD void barrier_d(double d, double dhat, double* b, double* b1, double* b2) {
  if (d < dhat) {
    double dd = d - dhat;
    double ln = log(d / dhat);
    *b = -dd * dd * ln;
    *b1 = -2.0 * dd * ln - dd * dd / d;
    double r = dd / d;
    *b2 = -2.0 * ln - 4.0 * dd / d + r * r;
  } else {
    *b = 0.0; *b1 = 0.0; *b2 = 0.0;
  }
}

// b and derivatives with respect to D = d^2 (contact.py:67-76)
GHD void barrier_D(double D, double dhat, double* b, double* f1, double* f2) {
  double d = sqrt(D), b1, b2;
  barrier_d(d, dhat, b, &b1, &b2);
  *f1 = b1 / (2.0 * d);
  *f2 = (b2 * d - b1) / (4.0 * d * D);
}

GHD void edge_mollifier(double c, double eps_x, double* m, double* dm, double* d2m) {
  double eps = 1e-3 * eps_x;
  double xr = c / eps;
  if (xr < 1.0) {
    *m = xr * (2.0 - xr);
    *dm = (2.0 - 2.0 * xr) / eps;
    *d2m = -2.0 / (eps * eps);
  } else {
    *m = 1.0; *dm = 0.0; *d2m = 0.0;
  }
}

// ---------------------------------------------------------------------------
// contact elements (contact.py:178-344) -- energy, grad, SPD-projected Hessian
// ---------------------------------------------------------------------------

enum { EL_ACTIVE = 1, EL_BAD_D = 2, EL_INVERTED = 4, EL_DEFERRED = 8 };

// Point-triangle stencil x[0]=point, x[1..3]=triangle.  Returns EL_* flags.
// Non-face regions keep only their gradient: the reference's _expand_rows writes
// their Hessian into an advanced-index copy (contact.py:116-125), so d2D == 0 there.
GHD int pt_element(const V3* x, double kappa, double dhat, double* E, double* g, double* H, int want_hess) {
  double bary[3];
  int reg;
  double D = pt_closest(x[0], x[1], x[2], x[3], bary, &reg);
  if (!(D > 0.0)) return EL_BAD_D;
  if (!(D < dhat * dhat)) return 0;
  double b, f1, f2;
  barrier_D(D, dhat, &b, &f1, &f2);
  *E = kappa * b;
  if (!g) return EL_ACTIVE;
  double gD[12];
  double* HD = want_hess ? H : nullptr;  // reuse H storage for d2D
  if (reg == 6) {
    double tmp[144];
    pt_plane12(x, gD, want_hess ? H : tmp);
  } else if (reg >= 3) {
    const int sa = reg == 3 ? 1 : (reg == 4 ? 2 : 3);
    const int sb = reg == 3 ? 2 : (reg == 4 ? 3 : 1);
    pe_grad12(x[0], x[sa], x[sb], 0, sa, sb, gD);
  } else {
    pp_grad12(x[0], x[1 + reg], 0, 1 + reg, gD);
  }
  for (int i = 0; i < 12; ++i) g[i] = kappa * f1 * gD[i];
  if (!want_hess) return EL_ACTIVE;
  if (reg == 6) {
    for (int i = 0; i < 12; ++i)
      for (int j = 0; j < 12; ++j) HD[i * 12 + j] = kappa * (f2 * gD[i] * gD[j] + f1 * HD[i * 12 + j]);
    spd_clamp_stencil(H);
  } else {
    rank1_clamped(gD, kappa * f2, H);
  }
  return EL_ACTIVE;
}

// Edge-edge stencil x = (a0, a1, b0, b1) with mollifier scale eps_x (contact.py:213-256, 305-340).
GHD int ee_element(const V3* x, double eps_x, double kappa, double dhat, double* E, double* g, double* H,
                   int want_hess) {
  double s, t;
  double D = ee_closest(x[0], x[1], x[2], x[3], &s, &t);
  if (!(D > 0.0)) return EL_BAD_D;
  if (!(D < dhat * dhat)) return 0;
  double c = cross_norm_sq(x, nullptr, nullptr);
  double m, dm, d2m;
  edge_mollifier(c, eps_x, &m, &dm, &d2m);
  double b, f1, f2;
  barrier_D(D, dhat, &b, &f1, &f2);
  *E = kappa * m * b;
  if (!g) return EL_ACTIVE;
  bool s_in = s > 0.0 && s < 1.0, t_in = t > 0.0 && t < 1.0;
  double gD[12];
  bool plane = s_in && t_in;
  if (plane) {
    ee_plane12(x, gD, H);  // H holds d2D
  } else if (s_in) {
    int ps = t < 0.5 ? 2 : 3;
    pe_grad12(x[ps], x[0], x[1], ps, 0, 1, gD);
  } else if (t_in) {
    int ps = s < 0.5 ? 0 : 1;
    pe_grad12(x[ps], x[2], x[3], ps, 2, 3, gD);
  } else {
    int sa = s < 0.5 ? 0 : 1, sb = t < 0.5 ? 2 : 3;
    pp_grad12(x[sa], x[sb], sa, sb, gD);
  }
  double gc[12];
  bool moll = dm != 0.0 || d2m != 0.0;
  for (int i = 0; i < 12; ++i) gc[i] = 0.0;
  double Hc[144];
  if (moll) cross_norm_sq(x, gc, want_hess ? Hc : nullptr);
  for (int i = 0; i < 12; ++i) g[i] = kappa * (m * f1 * gD[i] + b * dm * gc[i]);
  if (!want_hess) return EL_ACTIVE;
  if (!plane && !moll) {
    rank1_clamped(gD, kappa * m * f2, H);
    return EL_ACTIVE;
  }
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j) {
      double hb = f2 * gD[i] * gD[j] + (plane ? f1 * H[i * 12 + j] : 0.0);
      double hm = moll ? (d2m * gc[i] * gc[j] + dm * Hc[i * 12 + j]) : 0.0;
      double gmi = dm * gc[i], gmj = dm * gc[j], gbi = f1 * gD[i], gbj = f1 * gD[j];
      H[i * 12 + j] = kappa * (m * hb + b * hm + gmi * gbj + gbi * gmj);
    }
  spd_clamp_stencil(H);
  return EL_ACTIVE;
}

// ---------------------------------------------------------------------------
// lagged friction (contact.py:79-90, 475-524); per-anchor blocks are PSD, not projected
// ---------------------------------------------------------------------------
GHD double friction_element(const V3* x, const V3* xp, const double* gamma, const double* T /*3x2 row-major*/,
                            double lam, double mu, double eps_v, double dt, double* g, double* H) {
  double h = eps_v * dt;
  V3 u = V3{0.0, 0.0, 0.0};
  for (int k = 0; k < 4; ++k) u = u + gamma[k] * (x[k] - xp[k]);
  double s0 = T[0] * u.x + T[2] * u.y + T[4] * u.z;
  double s1 = T[1] * u.x + T[3] * u.y + T[5] * u.z;
  double y = sqrt(s0 * s0 + s1 * s1);
  double f0, f1;
  if (y < h) {
    f1 = 2.0 * y / h - (y / h) * (y / h);
    f0 = y * y / h - y * y * y / (3.0 * h * h);
  } else {
    f1 = 1.0;
    f0 = y - h / 3.0;
  }
  double sc = mu * lam;
  double E = sc * f0;
  if (!g) return E;
  double ratio = y > 1e-14 ? f1 / fmax(y, 1e-300) : 2.0 / h;
  double q0 = ratio * s0, q1 = ratio * s1;
  double g3[3] = {T[0] * q0 + T[1] * q1, T[2] * q0 + T[3] * q1, T[4] * q0 + T[5] * q1};
  for (int k = 0; k < 4; ++k)
    for (int a = 0; a < 3; ++a) g[3 * k + a] = sc * gamma[k] * g3[a];
  if (!H) return E;
  double df1 = y < h ? 2.0 / h - 2.0 * y / (h * h) : 0.0;
  double u0 = 0.0, u1 = 0.0;
  if (y > 1e-14) {
    double iy = 1.0 / fmax(y, 1e-300);
    u0 = s0 * iy;
    u1 = s1 * iy;
  }
  double M2[4] = {df1 * u0 * u0 + ratio * (1.0 - u0 * u0), df1 * u0 * u1 + ratio * (-u0 * u1),
                  df1 * u1 * u0 + ratio * (-u1 * u0), df1 * u1 * u1 + ratio * (1.0 - u1 * u1)};
  double M3[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 2; ++k)
        for (int l = 0; l < 2; ++l) s += T[2 * i + k] * M2[2 * k + l] * T[2 * j + l];
      M3[3 * i + j] = s;
    }
  for (int k = 0; k < 4; ++k)
    for (int l = 0; l < 4; ++l)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) H[(3 * k + a) * 12 + 3 * l + b] = sc * gamma[k] * gamma[l] * M3[3 * a + b];
  return E;
}

// ---------------------------------------------------------------------------
// Neo-Hookean tet (materials.py:116-158) and stress (materials.py:191-205)
// ---------------------------------------------------------------------------

GHD bool tet_F(const V3* x, const double* Dmi, double* F) {
  double Ds[9];
  for (int k = 0; k < 3; ++k) {
    V3 d = x[k + 1] - x[0];
    Ds[0 * 3 + k] = d.x;
    Ds[1 * 3 + k] = d.y;
    Ds[2 * 3 + k] = d.z;
  }
  mul33(Ds, Dmi, F);
  return true;
}

// Returns EL_INVERTED if J <= 0; else energy (and grad/H if asked, H projected).
GHD int nh_element(const V3* x, const double* Dmi, double V0, double mu, double lam, double* E, double* g, double* H) {
  double F[9];
  tet_F(x, Dmi, F);
  double J = det3(F);
  if (!(J > 0.0)) return EL_INVERTED;
  double Fi[9];
  inv3(F, Fi);
  double A[9];  // F^{-T}
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) A[3 * i + j] = Fi[3 * j + i];
  double Ic = 0.0;
  for (int i = 0; i < 9; ++i) Ic += F[i] * F[i];
  double lnJ = log(J);
  *E = V0 * (0.5 * mu * (Ic - 3.0) - mu * lnJ + 0.5 * lam * (J - 1.0) * (J - 1.0));
  if (!g) return 0;
  double c1 = lam * (J - 1.0) * J - mu;
  double P[9];
  for (int i = 0; i < 9; ++i) P[i] = mu * F[i] + c1 * A[i];
  double w[12];  // w[m][b]
  for (int b = 0; b < 3; ++b) {
    w[0 * 3 + b] = -(Dmi[0 * 3 + b] + Dmi[1 * 3 + b] + Dmi[2 * 3 + b]);
    for (int m = 1; m < 4; ++m) w[m * 3 + b] = Dmi[(m - 1) * 3 + b];
  }
  for (int m = 0; m < 4; ++m)
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int b = 0; b < 3; ++b) s += w[m * 3 + b] * P[c * 3 + b];
      g[3 * m + c] = s * V0;
    }
  if (!H) return 0;
  double c2 = mu - lam * (J - 1.0) * J;
  double c3 = lam * (2.0 * J - 1.0) * J;
  // T[c][b][M][C] = sum_B dP[c][b][C][B] w[M][B]
  double Tt[3 * 3 * 4 * 3];
  for (int c = 0; c < 3; ++c)
    for (int b = 0; b < 3; ++b)
      for (int M = 0; M < 4; ++M)
        for (int C = 0; C < 3; ++C) {
          double s = 0.0;
          for (int B = 0; B < 3; ++B) {
            double dp = (c == C && b == B ? mu : 0.0) + c2 * A[3 * c + B] * A[3 * C + b] + c3 * A[3 * c + b] * A[3 * C + B];
            s += dp * w[M * 3 + B];
          }
          Tt[((c * 3 + b) * 4 + M) * 3 + C] = s;
        }
  for (int m = 0; m < 4; ++m)
    for (int c = 0; c < 3; ++c)
      for (int M = 0; M < 4; ++M)
        for (int C = 0; C < 3; ++C) {
          double s = 0.0;
          for (int b = 0; b < 3; ++b) s += w[m * 3 + b] * Tt[((c * 3 + b) * 4 + M) * 3 + C];
          H[(3 * m + c) * 12 + 3 * M + C] = s * V0;
        }
  spd_clamp_stencil(H);
  return 0;
}

// Cauchy stress row [sxx, syy, szz, sxy, syz, sxz, von Mises]; returns false if J <= 0
GHD bool nh_stress(const V3* x, const double* Dmi, double mu, double lam, double* row) {
  double F[9];
  tet_F(x, Dmi, F);
  double J = det3(F);
  if (!(J > 0.0)) return false;
  double Fi[9], A[9], P[9];
  inv3(F, Fi);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) A[3 * i + j] = Fi[3 * j + i];
  double c1 = lam * (J - 1.0) * J - mu;
  for (int i = 0; i < 9; ++i) P[i] = mu * F[i] + c1 * A[i];
  double s[9];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) {
      double v = 0.0;
      for (int b = 0; b < 3; ++b) v += P[3 * a + b] * F[3 * c + b];
      s[3 * a + c] = v / J;
    }
  double sym[9];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) sym[3 * a + c] = 0.5 * (s[3 * a + c] + s[3 * c + a]);
  double tr = (sym[0] + sym[4] + sym[8]) / 3.0;
  double dd = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) {
      double v = sym[3 * a + c] - (a == c ? tr : 0.0);
      dd += v * v;
    }
  row[0] = sym[0]; row[1] = sym[4]; row[2] = sym[8];
  row[3] = sym[1]; row[4] = sym[5]; row[5] = sym[2];
  row[6] = sqrt(1.5 * dd);
  return true;
}

// ---------------------------------------------------------------------------
// ABD orthogonality (materials.py:161-188 + projection at solver.py:509-515)
// q = (p, A rows); grad/H over the 4 pseudo-nodes (p, A0, A1, A2)
// ---------------------------------------------------------------------------
GHD double abd_element(const double* A, double kV, double* g, double* H) {
  double S[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += A[3 * k + i] * A[3 * k + j];
      S[3 * i + j] = s - (i == j ? 1.0 : 0.0);
    }
  double E = 0.0;
  for (int i = 0; i < 9; ++i) E += S[i] * S[i];
  E *= kV;
  if (!g) return E;
  for (int i = 0; i < 3; ++i) g[i] = 0.0;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += A[3 * a + k] * S[3 * k + b];
      g[3 + 3 * a + b] = 4.0 * kV * s;
    }
  if (!H) return E;
  double AAt[9];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += A[3 * a + k] * A[3 * c + k];
      AAt[3 * a + c] = s;
    }
  double H9[81];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d)
          H9[(3 * a + b) * 9 + 3 * c + d] =
              4.0 * kV * ((a == c ? S[3 * d + b] : 0.0) + A[3 * a + d] * A[3 * c + b] + (b == d ? AAt[3 * a + c] : 0.0));
  double f = spd_clamp_full<9>(H9);
  for (int i = 0; i < 144; ++i) H[i] = 0.0;
  for (int i = 0; i < 3; ++i) H[i * 12 + i] = f;
  for (int i = 0; i < 9; ++i)
    for (int j = 0; j < 9; ++j) H[(3 + i) * 12 + 3 + j] = H9[i * 9 + j];
  return E;
}

// ---------------------------------------------------------------------------
// CCD (geometry/ccd.py:34-95) for one stencil: returns the advanced time t in [0,1];
// *bad = 1 if the stencil starts at distance <= 1e-14.
// ---------------------------------------------------------------------------
GHD double stencil_dist(const V3* q, int is_ee) {
  double D = is_ee ? ee_closest(q[0], q[1], q[2], q[3], nullptr, nullptr)
                   : pt_closest(q[0], q[1], q[2], q[3], nullptr, nullptr);
  return sqrt(D);
}

GHD double ccd_stencil(const V3* x, const V3* p, int is_ee, double scaling, int max_iters, double min_sep, int* bad) {
  const int split = is_ee ? 2 : 1;
  V3 mean = 0.25 * (((p[0] + p[1]) + p[2]) + p[3]);
  double la = 0.0, lb = 0.0;
  for (int k = 0; k < 4; ++k) {
    double l = norm(p[k] - mean);
    if (k < split) la = fmax(la, l);
    else lb = fmax(lb, l);
  }
  double lp = la + lb;
  double d = stencil_dist(x, is_ee);
  *bad = !(d > 1e-14);
  if (*bad) return 0.0;
  if (!(lp > 0.0)) return 1.0;
  double gap = min_sep * d;
  double t = 0.0;
  for (int it = 0; it < max_iters; ++it) {
    double tn = t + scaling * fmax(d - gap, 0.0) / lp;
    if (tn >= 1.0) return 1.0;
    t = tn;
    V3 q[4];
    for (int k = 0; k < 4; ++k) q[k] = x[k] + t * p[k];
    d = stencil_dist(q, is_ee);
    if (d <= gap + 1e-14) return t;
  }
  return t;
}

// ---------------------------------------------------------------------------
// cubic pencils (ccd.py:98-188)
// ---------------------------------------------------------------------------
GHD double cubic_smallest_root(double c0, double c1, double c2, double c3, double t_max) {
  double sc = fmax(fmax(fmax(fabs(c0), fabs(c1)), fmax(fabs(c2), fabs(c3))), 1e-30);
  double r[3] = {INFINITY, INFINITY, INFINITY};
  if (fabs(c3) > 1e-14 * sc) {
    double a = c2 / c3, b = c1 / c3, c = c0 / c3;
    double p = b - a * a / 3.0;
    double q = 2.0 * a * a * a / 27.0 - a * b / 3.0 + c;
    double disc = (q / 2.0) * (q / 2.0) + (p / 3.0) * (p / 3.0) * (p / 3.0);
    if (disc > 0.0) {
      double sq = sqrt(disc);
      r[0] = cbrt(-q / 2.0 + sq) + cbrt(-q / 2.0 - sq) - a / 3.0;
    } else {
      double pm = fmin(p, -1e-300);
      double rr = sqrt(-pm / 3.0);
      double arg = 3.0 * q / (2.0 * pm * rr);
      arg = arg < -1.0 ? -1.0 : (arg > 1.0 ? 1.0 : arg);
      double phi = acos(arg);
      const double pi = 3.14159265358979323846;
      for (int k = 0; k < 3; ++k) r[k] = 2.0 * rr * cos((phi - 2.0 * pi * k) / 3.0) - a / 3.0;
    }
  } else if (fabs(c2) > 1e-14 * sc) {
    double a = c2, b = c1, c = c0;
    double disc = b * b - 4.0 * a * c;
    if (disc >= 0.0) {
      double sq = sqrt(fmax(disc, 0.0));
      r[0] = (-b - sq) / (2.0 * a);
      r[1] = (-b + sq) / (2.0 * a);
    }
  } else if (fabs(c1) > 1e-14 * sc) {
    r[0] = -c0 / c1;
  }
  double best = INFINITY;
  for (int k = 0; k < 3; ++k)
    if (r[k] > 1e-12 && r[k] <= t_max) best = fmin(best, r[k]);
  return isfinite(best) ? best : t_max + 1.0;
}

// cofactor-based pencil coefficients of det(M0 + t dM) (ccd.py:98-103,173-176)
GHD void cofactor(const double* M, double* C) {
  // columns of C are cross products of column pairs of M
  V3 m0 = V3{M[0], M[3], M[6]}, m1 = V3{M[1], M[4], M[7]}, m2 = V3{M[2], M[5], M[8]};
  V3 c0 = cross(m1, m2), c1 = cross(m2, m0), c2 = cross(m0, m1);
  C[0] = c0.x; C[3] = c0.y; C[6] = c0.z;
  C[1] = c1.x; C[4] = c1.y; C[7] = c1.z;
  C[2] = c2.x; C[5] = c2.y; C[8] = c2.z;
}

GHD double pencil_root(const double* M0, const double* dM, double det0) {
  double C0[9], C1[9];
  cofactor(M0, C0);
  cofactor(dM, C1);
  double c1 = 0.0, c2 = 0.0;
  for (int i = 0; i < 9; ++i) {
    c1 += C0[i] * dM[i];
    c2 += C1[i] * M0[i];
  }
  return cubic_smallest_root(det0, c1, c2, det3(dM), 1.0);
}

// tet edge matrix M = [x1-x0, x2-x0, x3-x0] as columns (ccd.py:198-203)
GHD void tet_edge_matrix(const V3* x, double* M) {
  for (int k = 0; k < 3; ++k) {
    V3 d = x[k + 1] - x[0];
    M[0 * 3 + k] = d.x;
    M[1 * 3 + k] = d.y;
    M[2 * 3 + k] = d.z;
  }
}

}  // namespace grip
