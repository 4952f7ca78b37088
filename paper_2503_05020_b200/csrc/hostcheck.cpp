// Host build of the device element math (grip_elements.cuh) for CPU unit tests.
// Test infrastructure: lets tests/ pin every per-element routine against the
// oracle without a GPU.  Not used by the product path.
#include <cmath>
#include <cstdint>

#include "grip_elements.cuh"

using namespace grip;

static void ld4(const double* x, V3* o) {
  for (int k = 0; k < 4; ++k) o[k] = ld3(x + 3 * k);
}

extern "C" {
double hc_pt_closest(const double* x, double* bary, int* region) {
  V3 v[4];
  ld4(x, v);
  return pt_closest(v[0], v[1], v[2], v[3], bary, region);
}
double hc_ee_closest(const double* x, double* s, double* t) {
  V3 v[4];
  ld4(x, v);
  return ee_closest(v[0], v[1], v[2], v[3], s, t);
}
int hc_pt_element(const double* x, double kappa, double dhat, double* E, double* g, double* H, int want) {
  V3 v[4];
  ld4(x, v);
  return pt_element(v, kappa, dhat, E, g, H, want);
}
int hc_ee_element(const double* x, double epsx, double kappa, double dhat, double* E, double* g, double* H, int want) {
  V3 v[4];
  ld4(x, v);
  return ee_element(v, epsx, kappa, dhat, E, g, H, want);
}
int hc_nh_element(const double* x, const double* Dmi, double V0, double mu, double lam, double* E, double* g, double* H) {
  V3 v[4];
  ld4(x, v);
  return nh_element(v, Dmi, V0, mu, lam, E, g, H);
}
double hc_abd_element(const double* A, double kV, double* g, double* H) { return abd_element(A, kV, g, H); }
double hc_friction(const double* x, const double* xp, const double* gamma, const double* T, double lam, double mu,
                   double eps_v, double dt, double* g, double* H) {
  V3 v[4], vp[4];
  ld4(x, v);
  ld4(xp, vp);
  return friction_element(v, vp, gamma, T, lam, mu, eps_v, dt, g, H);
}
double hc_ccd(const double* x, const double* p, int is_ee, double scaling, int iters, double min_sep, int* bad) {
  V3 v[4], q[4];
  ld4(x, v);
  ld4(p, q);
  return ccd_stencil(v, q, is_ee, scaling, iters, min_sep, bad);
}
double hc_cubic(double c0, double c1, double c2, double c3) { return cubic_smallest_root(c0, c1, c2, c3, 1.0); }
double hc_pencil(const double* M0, const double* dM) { return pencil_root(M0, dM, det3(M0)); }
void hc_clamp_stencil(double* H) { spd_clamp_stencil(H); }
void hc_clamp12(double* H) { spd_clamp_full<12>(H); }
int hc_stress(const double* x, const double* Dmi, double mu, double lam, double* row) {
  V3 v[4];
  ld4(x, v);
  return nh_stress(v, Dmi, mu, lam, row) ? 1 : 0;
}
}
