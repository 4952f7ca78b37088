// Kernels of the batched IPC step.  Two shapes:
//   *_env kernels: one CTA (NT threads) per environment, blockIdx.x indexes a
//     device list of env ids; everything an env needs between two global
//     decisions (broad phase, assembly + PCG, CCD + line search) runs inside it.
//   k_elements: flat grid-stride kernel over the element work of all pending
//     envs (Neo-Hookean tets, ABD, contact stencils, friction anchors) -- the
//     fp64-heavy part with the 12x12 eigen-clamps, load-balanced chip-wide.
#pragma once
#include "grip_device.cuh"

namespace grip {

// ---------------------------------------------------------------------------
// shared per-env helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ void fail_env(const Dev& D, int e, int reason) {
  if (threadIdx.x == 0) {
    D.ns_status[e] = GRIP_NS_FAILED;
    D.reason[e] = reason;
    D.ns_done[e] = 1;
    D.needs_ls[e] = 0;
  }
}

// radius of the candidate superset: covers 1.05 dhat, optionally the next line search's
// dhat + 2 max_disp predicted from the last step (ss_k * md_prev, GRIP_SS_K; default 0: measured,
// the grid cost grows faster with R than the line search saves) and the kinematic CCD radius;
// capped so a huge Newton step does not blow the set up (that line search runs its own)
__device__ __forceinline__ double superset_radius(const Dev& D, int e, double dhat) {
  double R = fmax(1.05 * dhat, dhat + D.ss_k * D.md_prev[e]);
  R = fmax(R, dhat + 2.0 * D.md_kin[e]);
  return fmin(R, 12.0 * dhat);
}

// Verlet skin: a superset built at radius R from positions X0 is still a superset at radius
// R - 2 drift for positions X, if no surface vertex moved more than drift (any norm >= the max
// norm) between X0 and X: both reference predicates are per-axis box tests (broadphase.py:
// 177-183, 195-210), and a vertex coordinate and an AABB face each move by at most drift.  The
// relative / absolute margins cover the rounding of the drift sums and of the predicates.
// With drift == 0 (positions unchanged since the build) the superset covers exactly R.
__device__ __forceinline__ bool cs_covers(const Dev& D, int e, double need) {
  if (!D.cs_valid[e]) return false;
  const double dr = D.cs_drift[e];
  return dr == 0.0 ? D.cs_R[e] >= need : D.cs_R[e] - 2.0 * dr * (1.0 + 1e-9) - 1e-12 >= need;
}

// surfaces of env e moved by at most dmax since the last call (thread 0)
__device__ __forceinline__ void cs_moved(const Dev& D, int e, double dmax) {
  if (threadIdx.x == 0) {
    if (D.ss_skin > 0.0) D.cs_drift[e] += dmax;
    else D.cs_valid[e] = 0;
  }
}

// make D.cs_* a superset at radius >= need for the current positions (D.sv_pos); built with
// the skin GRIP_SKIN * dhat on top, so that it survives the next small moves
__device__ bool ensure_superset(const Dev& D, const EnvIx& E, double need, double dhat, BPShared& S, Red& sm,
                                const BPCl& cl = BPCl{0, 1}) {
  const int e = E.e;
  const bool valid = cs_covers(D, e, need);
  __syncthreads();
  if (valid) return true;
  const double R = fmax(need, superset_radius(D, e, dhat)) + D.ss_skin * dhat;
  const bool ok = broad_phase_env(D, E, R, D.cs_pt + (size_t)e * 4 * D.cap_pt, D.cs_ee + (size_t)e * 4 * D.cap_ee,
                                  D.cs_eid + (size_t)e * 2 * D.cap_ee, D.cs_n + 2 * e, S, sm, cl);
  if (cl.rank == 0 && threadIdx.x == 0) {
    D.cs_R[e] = R;
    D.cs_drift[e] = 0.0;
    D.cs_valid[e] = ok ? 1 : 0;
  }
  __syncthreads();
  return ok;
}

__device__ __forceinline__ void filter_from_superset(const Dev& D, const EnvIx& E, double r, int* pt, int* ee, int* eid,
                                                     int* n, Red& sm) {
  const int e = E.e;
  filter_set(D, E, r, D.cs_pt + (size_t)e * 4 * D.cap_pt, D.cs_ee + (size_t)e * 4 * D.cap_ee,
             D.cs_eid + (size_t)e * 2 * D.cap_ee, D.cs_n + 2 * e, pt, ee, eid, n, sm);
}

// write sv positions of node array xs into D.sv_pos (env slice)
__device__ void env_sv_positions(const Dev& D, const EnvIx& E, const double* xs) {
  for (int i = threadIdx.x; i < E.ns; i += NT) st3(D.sv_pos + 3 * (size_t)(E.s0 + i), sv_at(D, E, i, xs));
  __syncthreads();
}

// additive CCD over a candidate set, min over stencils (ccd.py:34-95).  disp: per-sv D.sv_disp.
// returns alpha; *bad set if any stencil starts at d <= 1e-14
__device__ double env_ccd(const Dev& D, const EnvIx& E, const int* pt, int npt, const int* ee, int nee, double scaling,
                          int iters, double min_sep, int* bad, Red& sm) {
  const double* X = D.sv_pos + 3 * (size_t)E.s0;
  const double* U = D.sv_disp + 3 * (size_t)E.s0;
  double amin = 1.0;
  int b = 0;
  for (int k = threadIdx.x; k < npt + nee; k += NT) {
    const int is_ee = k >= npt;
    const int* row = is_ee ? ee + 4 * (k - npt) : pt + 4 * k;
    V3 x[4], p[4];
    for (int j = 0; j < 4; ++j) {
      x[j] = ld3(X + 3 * row[j]);
      p[j] = ld3(U + 3 * row[j]);
    }
    int bk = 0;
    double t = ccd_stencil(x, p, is_ee, scaling, iters, min_sep, &bk);
    b |= bk;
    amin = fmin(amin, t);
  }
  *bad = block_or(b, sm);
  return fmax(block_min(amin, sm), 0.0);
}

// ---------------------------------------------------------------------------
// begin_step (solver.py:590-645)
// ---------------------------------------------------------------------------
__device__ void begin_env(const Dev& D, int e, Red& sm, BPShared& S, const BPCl& cl);

// A cluster of BP_CL CTAs per env, for the kinematic CCD's broad phase (see k_linesearch); rank 0
// does everything else.
__global__ void __cluster_dims__(BP_CL, 1, 1) __launch_bounds__(NT) k_begin(Dev D, const int* list) {
  __shared__ Red sm;
  __shared__ BPShared S;
  const BPCl cl{(int)cooperative_groups::this_cluster().block_rank(), BP_CL};
  const int e = list[blockIdx.x / BP_CL];
  CTA_TIMER_IF(cl.rank == 0, 0, e);
  // device protocol: only envs whose protocol asked for a new step
  if (D.round_mode && !D.pr_i[(size_t)e * PI_N + PI_NEEDBEGIN]) return;
  begin_env(D, e, sm, S, cl);
  if (cl.rank != 0) return;
  if (D.round_mode) {
    __syncthreads();
    if (threadIdx.x == 0 && !(D.flags[e] & FLAG_OVERFLOW)) {   // an overflowed begin is redone later
      D.pr_i[(size_t)e * PI_N + PI_NEEDBEGIN] = 0;
      D.pr_i[(size_t)e * PI_N + PI_INSTEP] = 1;
    }
  }
}

__device__ void begin_env(const Dev& D, int e, Red& sm, BPShared& S, const BPCl& cl) {
  const EnvIx E = env_ix(D, e);
  const double* P = P_(D, e);
  const double dt = P[GRIP_P_DT], dhat = P[GRIP_P_DHAT];
  const bool r0 = cl.rank == 0;
  if (r0 && threadIdx.x == 0) D.fin_done[e] = 0;
  if (r0) {
    for (int i = threadIdx.x; i < 3 * E.nn; i += NT) D.x_t[3 * (size_t)E.n0 + i] = D.x[3 * (size_t)E.n0 + i];
    env_sv_positions(D, E, D.x);
    for (int i = threadIdx.x; i < 3 * E.ns; i += NT) D.surf_prev[3 * (size_t)E.s0 + i] = D.sv_pos[3 * (size_t)E.s0 + i];
  }
  // which bodies move: kinematic with v != 0, soft with a prescribed mask and v != 0
  int moving = 0;
  for (int b = threadIdx.x; b < E.nb; b += NT) {
    const double* vb = D.body_vel + 3 * (size_t)(E.b0 + b);
    const bool nz = vb[0] != 0.0 || vb[1] != 0.0 || vb[2] != 0.0;
    const int kind = D.body_kind[E.b0 + b];
    if (nz && kind == 2) moving = 1;
    if (nz && kind == 0) {
      for (int n = 0; n < E.nn; ++n)
        if (D.node_body[E.n0 + n] == b && !D.node_free[E.n0 + n]) { moving = 1; break; }
    }
  }
  moving = block_or(moving, sm);
  if (!moving && !r0) return;   // no broad phase: nothing for the other ranks (inputs are static)
  double alpha = 1.0;
  if (moving) {
    double md = 0.0;
    for (int i = threadIdx.x; i < E.ns; i += NT) {
      const int g = E.s0 + i;
      V3 d = V3{0.0, 0.0, 0.0};
      const int kind = D.sv_kind[g];
      const double* vb = D.body_vel + 3 * (size_t)(E.b0 + D.sv_body[g]);
      if (kind == 2) d = V3{vb[0] * dt, vb[1] * dt, vb[2] * dt};
      if (kind == 0 && !D.node_free[E.n0 + D.sv_node[g]]) d = V3{vb[0] * dt, vb[1] * dt, vb[2] * dt};
      if (r0) st3(D.sv_disp + 3 * (size_t)g, d);
      md = fmax(md, norm(d));
    }
    md = block_max(md, sm);
    int* cn = D.c2_n + 2 * e;
    const double rk = dhat + 2.0 * md;
    const bool reuse = cs_covers(D, e, rk);
    cl_sync(cl);   // every rank has its decision before rank 0 changes its inputs
    if (!r0 && reuse) return;
    if (r0 && threadIdx.x == 0) D.md_kin[e] = md;
    if (reuse) {
      filter_from_superset(D, E, rk, D.c2_pt + (size_t)e * 4 * D.cap_pt, D.c2_ee + (size_t)e * 4 * D.cap_ee,
                           D.c2_eid + (size_t)e * 2 * D.cap_ee, cn, sm);
    } else if (!broad_phase_env(D, E, rk, D.c2_pt + (size_t)e * 4 * D.cap_pt, D.c2_ee + (size_t)e * 4 * D.cap_ee,
                                D.c2_eid + (size_t)e * 2 * D.cap_ee, cn, S, sm, cl)) {
      if (r0 && threadIdx.x == 0) D.flags[e] |= FLAG_OVERFLOW | FLAG_OVF_BEGIN;
      return;
    }
    if (!r0) return;
    if (cn[0] + cn[1] > 0) {
      int bad = 0;
      alpha = env_ccd(D, E, D.c2_pt + (size_t)e * 4 * D.cap_pt, cn[0], D.c2_ee + (size_t)e * 4 * D.cap_ee, cn[1],
                      P[GRIP_P_CCDSCALE], (int)P[GRIP_P_CCDIT], P[GRIP_P_KINGUARD], &bad, sm);
      if (bad) {
        // the reference raises out of begin_step here; the env is quarantined instead
        fail_env(D, e, GRIP_R_CCD);
        return;
      }
    }
    // pre-move: masked soft nodes by alpha*(v dt); kinematic surfaces by (alpha v) dt
    for (int n = threadIdx.x; n < E.nn; n += NT) {
      const int g = E.n0 + n;
      if (D.node_kind[g] == 0 && !D.node_free[g]) {
        const double* vb = D.body_vel + 3 * (size_t)(E.b0 + D.node_body[g]);
        for (int c = 0; c < 3; ++c) D.x[3 * (size_t)g + c] += alpha * (vb[c] * dt);
      }
    }
    for (int i = threadIdx.x; i < E.ns; i += NT) {
      const int g = E.s0 + i;
      if (D.sv_kind[g] == 2) {
        const double* vb = D.body_vel + 3 * (size_t)(E.b0 + D.sv_body[g]);
        for (int c = 0; c < 3; ++c) D.kin_pos[3 * (size_t)g + c] += alpha * vb[c] * dt;
      }
    }
    cs_moved(D, e, alpha * md);  // surfaces moved
    __syncthreads();
  } else {
    if (threadIdx.x == 0) D.md_kin[e] = 0.0;
  }
  // implicit-Euler target: gravity on soft nodes and affine translations only
  const double* gr = D.gravity + 3 * e;
  for (int n = threadIdx.x; n < E.nn; n += NT) {
    const int g = E.n0 + n;
    const int kind = D.node_kind[g];
    for (int c = 0; c < 3; ++c) {
      const double a = kind == 2 ? 0.0 : gr[c];
      const double xv = D.x[3 * (size_t)g + c];
      D.xhat[3 * (size_t)g + c] = D.node_free[g] ? xv + dt * D.v[3 * (size_t)g + c] + dt * dt * a : xv;
    }
  }
  __syncthreads();
  env_sv_positions(D, E, D.x);
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = threadIdx.x; i < E.ns; i += NT)
    for (int c = 0; c < 3; ++c) {
      const double v = D.sv_pos[3 * (size_t)(E.s0 + i) + c];
      lo[c] = fmin(lo[c], v);
      hi[c] = fmax(hi[c], v);
    }
  for (int c = 0; c < 3; ++c) {
    lo[c] = block_min(lo[c], sm);
    hi[c] = block_max(hi[c], sm);
  }
  if (threadIdx.x == 0) {
    const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
    const double diag = E.ns ? sqrt(dx * dx + dy * dy + dz * dz) : 0.0;
    const double ell = fmax(diag, P[GRIP_P_ELLFLOOR]);
    D.ell[e] = ell;
    D.tol[e] = P[GRIP_P_RELTOL] * dt * ell;
    D.kin_blocked[e] = moving && alpha < 1.0 - 1e-12;
    D.iters[e] = 0;
    D.ns_status[e] = GRIP_NS_RUNNING;
    D.reason[e] = GRIP_R_NONE;
    D.ns_done[e] = 0;
    D.needs_ls[e] = 0;
    D.residual[e] = INFINITY;
    D.energy[e] = INFINITY;
    D.regularized[e] = 0;
    D.newton_calls[e] = 0;
    D.pcg_iters[e] = 0;
    D.flags[e] = 0;
    D.fin_done[e] = 0;
  }
}

// ---------------------------------------------------------------------------
// Newton sweep 1/4: surface positions, candidate set at 1.05 dhat, active stencils
// (solver.py:652-653, contact.py:283-309)
// ---------------------------------------------------------------------------
// A cluster of BP_CL CTAs per env: a superset rebuild is split over the cluster (BPCl), the rest
// runs on rank 0; the other ranks of an env whose superset still covers exit at once.
__device__ void work_scan_body(const Dev& D, const int* list, int n, Red& sm);

__device__ __forceinline__ void cand_env(const Dev& D, int e, const BPCl& cl, BPShared& S, Red& sm) {
  const EnvIx E = env_ix(D, e);
  const double* P = P_(D, e);
  const double dhat = P[GRIP_P_DHAT];
  // finished (or failed in begin_step) envs of a round list; an env whose begin_step overflowed
  // this round keeps its flag and is re-run by the host after growth (rank 0 clears the flags
  // of a live env only: every rank reads the same skip decision)
  const bool skip = D.ns_done[e] || (D.flags[e] & FLAG_OVERFLOW);
  const bool covered = cs_covers(D, e, 1.05 * dhat);
  __syncthreads();
  if (skip || (cl.rank != 0 && covered)) return;
  if (cl.rank == 0 && threadIdx.x == 0) {
    D.flags[e] = 0;
    D.newton_calls[e] += 1;
  }
  if (cl.rank == 0) env_sv_positions(D, E, D.x);
  if (!covered) cl_sync(cl);   // the positions rank 0 wrote, before the cluster's broad phase
  int* cn = D.c1_n + 2 * e;
  int* cpt = D.c1_pt + (size_t)e * 4 * D.cap_pt;
  int* cee = D.c1_ee + (size_t)e * 4 * D.cap_ee;
  if (!ensure_superset(D, E, 1.05 * dhat, dhat, S, sm, covered ? BPCl{0, 1} : cl)) {
    if (cl.rank == 0 && threadIdx.x == 0) D.flags[e] |= FLAG_OVERFLOW;
    return;
  }
  if (cl.rank != 0) return;
  filter_from_superset(D, E, dhat * 1.05, cpt, cee, D.c1_eid + (size_t)e * 2 * D.cap_ee, cn, sm);
  const int npt = cn[0], nee = cn[1];
  const double* X = D.sv_pos + 3 * (size_t)E.s0;
  // active stencils in candidate order (PT first, then EE), non-positive distance check
  int* act = D.act + (size_t)e * D.cap_act;
  int base = 0, bad = 0;
  for (int s = 0; s < npt + nee; s += NT) {
    const int k = s + threadIdx.x;
    int a = 0;
    if (k < npt + nee) {
      const bool is_ee = k >= npt;
      const int* row = is_ee ? cee + 4 * (k - npt) : cpt + 4 * k;
      V3 x0 = ld3(X + 3 * row[0]), x1 = ld3(X + 3 * row[1]), x2 = ld3(X + 3 * row[2]), x3 = ld3(X + 3 * row[3]);
      const double Dq = is_ee ? ee_closest(x0, x1, x2, x3, nullptr, nullptr) : pt_closest(x0, x1, x2, x3, nullptr, nullptr);
      if (!(Dq > 0.0)) bad = 1;
      a = Dq < dhat * dhat;
    }
    int tot;
    const int pre = block_scan(a, sm, &tot);
    if (a && base + pre < D.cap_act) act[base + pre] = k >= npt ? D.cap_pt + (k - npt) : k;
    base += tot;
  }
  bad = block_or(bad, sm);
  if (threadIdx.x == 0) {
    D.n_act[e] = base;
    if (bad) D.flags[e] |= ERR_CONTACT_D;
    if (base > D.cap_act) {
      D.flags[e] |= FLAG_OVERFLOW;
      atomicMax(&D.need[2], (unsigned)base);
    }
  }
}

// Newton sweep 1/4 (see cand_env).  The last env CTA to finish also scans the per-env contact
// work for the element kernels (the scan used to be its own single-CTA launch on the critical
// path): every rank-0 CTA publishes its env's results, fences and counts itself in.
__global__ void __cluster_dims__(BP_CL, 1, 1) __launch_bounds__(NT, NT_MINB3) k_candidates(Dev D, const int* list) {
  __shared__ Red sm;
  __shared__ BPShared S;
  __shared__ int last;
  const BPCl cl{(int)cooperative_groups::this_cluster().block_rank(), BP_CL};
  const int e = list[blockIdx.x / BP_CL];
  CTA_TIMER_IF(cl.rank == 0, 1, e);
  cand_env(D, e, cl, S, sm);
  if (cl.rank != 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const int n = gridDim.x / BP_CL;
    last = atomicAdd(D.cand_done, 1u) == (unsigned)(n - 1);
    if (last) {
      __threadfence();
      *D.cand_done = 0u;
    }
  }
  __syncthreads();
  if (last) work_scan_body(D, list, gridDim.x / BP_CL, sm);
}

// exclusive scan of per-env contact / friction element work over the pending list (one CTA)
__device__ void work_scan_body(const Dev& D, const int* list, int n, Red& sm) {
  int base = 0;
  double cc = 0.0, cf = 0.0, cn = 0.0;   // cn: envs iterating (newton_iteration calls)
  int cbase = 0;
  for (int s = 0; s < n; s += NT) {
    const int i = s + threadIdx.x;
    int w = 0, wc = 0;
    if (i < n) {
      const int e = list[i];
      if (!(D.flags[e] & FLAG_OVERFLOW) && !D.ns_done[e]) {
        const int nt = D.tet_off[e + 1] - D.tet_off[e], na = D.abd_off[e + 1] - D.abd_off[e];
        wc = D.n_act[e] + D.n_anc[e];
        w = nt + na + wc;
        cc += D.n_act[e]; cf += D.n_anc[e]; cn += 1.0;
      }
    }
    if (i < n) D.asm_key[i] = wc;
    int tot;
    const int pre = block_scan(w, sm, &tot);
    if (i < n) D.work_off[i] = base + pre;
    base += tot;
    const int cpre = block_scan(wc, sm, &tot);
    if (i < n) D.cwork_off[i] = cbase + cpre;
    cbase += tot;
  }
  __syncthreads();
  // heavy envs first: rank by (contact work descending, list position ascending)
  for (int i = threadIdx.x; i < n; i += NT) {
    const int ki = D.asm_key[i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const int kj = D.asm_key[j];
      r += (kj > ki) || (kj == ki && j < i);
    }
    D.asm_order[r] = list[i];
  }
  cc = block_sum(cc, sm); cf = block_sum(cf, sm);
  cn = block_sum(cn, sm);
  if (threadIdx.x == 0) {
    D.work_off[n] = base;
    D.cwork_off[n] = cbase;
    *D.cjac_n = 0;   // k_elements_w appends deferred contact clamps
    D.stats[2] += cc; D.stats[3] += cf;
    D.stats[7] += cn;
  }
}

// The tet chain's scan (second stream): tets of every pending env that is not done.  It cannot
// read the overflow flags k_candidates is writing concurrently; an env whose candidates
// overflow computes its tets anyway (its assembly is skipped, its warm starts not committed).
__global__ void __launch_bounds__(NT) k_tet_scan(Dev D, const int* list, int n) {
  __shared__ Red sm;
  double ct = 0.0, ca = 0.0;
  int tbase = 0, sbase = 0;
  for (int s = 0; s < n; s += NT) {
    const int i = s + threadIdx.x;
    int wt = 0, ws = 0;
    if (i < n) {
      const int e = list[i];
      D.tflag[e] = 0;
      D.eig_swept[e] = !D.ns_done[e];
      if (!D.ns_done[e]) {
        wt = D.tet_off[e + 1] - D.tet_off[e];
        const int f0 = D.free_off[e], f1 = D.free_off[e + 1];
        ws = D.sb_rowptr[f1] - D.sb_rowptr[f0];
        ct += wt;
        ca += D.abd_off[e + 1] - D.abd_off[e];
      }
    }
    int tot;
    const int tpre = block_scan(wt, sm, &tot);
    if (i < n) D.twork_off[i] = tbase + tpre;
    tbase += tot;
    const int spre = block_scan(ws, sm, &tot);
    if (i < n) D.swork_off[i] = sbase + spre;
    sbase += tot;
  }
  ct = block_sum(ct, sm);
  ca = block_sum(ca, sm);
  if (threadIdx.x == 0) {
    D.twork_off[n] = tbase;
    D.swork_off[n] = sbase;
    *D.jac_n = 0;   // k_tet_front appends deferred tet clamps
    D.stats[0] += ct;
    D.stats[1] += ca;
  }
}

// Static block values of H_ff (mass + dt^2 x tet / ABD element blocks, solver.py:542-586's
// M + dt^2 H_el part) for every listed env, thread per 3x3 block, chip-wide on the second stream
// after the tet back-end (each block's contributions in their stored order: the same sums the
// assembly kernel formed itself before)
__global__ void __launch_bounds__(NT) k_static(Dev D, const int* list, int n) {
  const int total = D.swork_off[n];
  for (int item = blockIdx.x * blockDim.x + threadIdx.x; item < total; item += gridDim.x * blockDim.x) {
    int lo = 0, hi = n;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (D.swork_off[mid] <= item) lo = mid;
      else hi = mid;
    }
    const int e = list[lo];
    const int f0 = D.free_off[e];
    const int b = D.sb_rowptr[f0] + item - D.swork_off[lo];
    const int f = D.sb_row[b] - f0;
    const size_t elbase = (size_t)e * D.cap_el;
    const double dt = D.params[(size_t)e * GRIP_NPARAM + GRIP_P_DT], dt2 = dt * dt;
    double v[9];
    for (int i = 0; i < 9; ++i) v[i] = 0.0;
    for (int q = D.sbc_ptr[b]; q < D.sbc_ptr[b + 1]; ++q) {
      const int code = D.sbc[q];
      const int sl = code >> 4, sa = (code >> 2) & 3, sbb = code & 3;
      const double* H = D.el_H + (elbase + sl) * 144;
      if (sl < D.max_tet) {   // tets: packed lower triangle (grip_tet.cuh)
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) {
            const int r = 3 * sa + i, c = 3 * sbb + j;
            v[3 * i + j] += H[r >= c ? tri12(r, c) : tri12(c, r)];
          }
      } else {
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) v[3 * i + j] += H[(3 * sa + i) * 12 + 3 * sbb + j];
      }
    }
    const bool diag = D.sb_col[b] == f;
    const double* M = D.node_M + 9 * (size_t)(D.node_off[e] + D.free_node[f0 + f]);
    for (int i = 0; i < 9; ++i) D.sb_val[9 * (size_t)b + i] = (diag ? M[i] : 0.0) + dt2 * v[i];
  }
}

// Newton sweep 2/4 (element energies, gradients, SPD-projected Hessians): grip_tet.cuh
// (k_tet_front / k_tet_back), grip_warp_elements.cuh (k_elements_w), grip_tetclamp.cuh.

// ---------------------------------------------------------------------------
// Newton sweep 3/4: assembly + block-Jacobi PCG (solver.py:542-586, 654-676, 91-131)
// ---------------------------------------------------------------------------

// contact/friction element slots of env e: k in [0, n_ce) -> slot
__device__ __forceinline__ int ce_slot(const Dev& D, int e, int k) {
  const int na = D.n_act[e];
  return k < na ? D.max_tet + D.max_abd + k : D.max_tet + D.max_abd + D.cap_act + (k - na);
}

struct AsmShared {
  Red sm;
  double abd_red[NWARP][12];
  double chol[144];
};

// y = H_ff p over free nodes (static blocks + G^T H_sv G for contacts/friction)
__device__ void spmv(const Dev& D, const EnvIx& E, double dt2, const double* p, double* y, AsmShared& A) {
  const int e = E.e;
  const size_t vb = (size_t)e * 3 * D.max_free;
  // static blocks
  for (int f = threadIdx.x; f < E.nf; f += NT) {
    const int fg = E.f0 + f;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int b = D.sb_rowptr[fg]; b < D.sb_rowptr[fg + 1]; ++b) {
      const double* B = D.sb_val + 9 * (size_t)b;
      const double* q = p + vb + 3 * D.sb_col[b];
      s0 += B[0] * q[0] + B[1] * q[1] + B[2] * q[2];
      s1 += B[3] * q[0] + B[4] * q[1] + B[5] * q[2];
      s2 += B[6] * q[0] + B[7] * q[1] + B[8] * q[2];
    }
    y[vb + 3 * f] = s0; y[vb + 3 * f + 1] = s1; y[vb + 3 * f + 2] = s2;
  }
  const int nce = D.n_act[e] + D.n_anc[e];
  if (nce == 0) { __syncthreads(); return; }
  // u = G p (sv space)
  double* U = D.c_u + (size_t)e * 3 * D.max_sv;
  for (int i = threadIdx.x; i < E.ns; i += NT) {
    const int g = E.s0 + i;
    const int kind = D.sv_kind[g];
    V3 u = V3{0.0, 0.0, 0.0};
    if (kind == 0) {
      const int f = D.node_fidx[E.n0 + D.sv_node[g]];
      if (f >= 0) u = ld3(p + vb + 3 * f);
    } else if (kind == 1) {
      const int f = D.node_fidx[E.n0 + D.sv_node[g]];
      const double* q = p + vb + 3 * f;
      V3 xi = ld3(D.sv_xi + 3 * g);
      u = V3{q[0] + xi.x * q[3] + xi.y * q[4] + xi.z * q[5], q[1] + xi.x * q[6] + xi.y * q[7] + xi.z * q[8],
             q[2] + xi.x * q[9] + xi.y * q[10] + xi.z * q[11]};
    }
    st3(U + 3 * i, u);
  }
  __syncthreads();
  // r_e = dt^2 H_e u_e, one thread per element row
  double* R = D.c_r + (size_t)e * 12 * (D.cap_act + D.cap_anc);
  const size_t elbase = (size_t)e * D.cap_el;
  for (int t = threadIdx.x; t < 12 * nce; t += NT) {
    const int k = t / 12, row = t - 12 * k;
    const size_t sl = elbase + ce_slot(D, e, k);
    const double* H = D.el_H + sl * 144 + row * 12;
    const int* ix = D.el_idx + sl * 4;
    double s = 0.0;
    for (int j = 0; j < 4; ++j) {
      const double* u = U + 3 * ix[j];
      s += H[3 * j] * u[0] + H[3 * j + 1] * u[1] + H[3 * j + 2] * u[2];
    }
    R[t] = dt2 * s;
  }
  __syncthreads();
  // w_sv = sum over incident (element, slot), fixed order
  double* W = D.c_w + (size_t)e * 3 * D.max_sv;
  const int* ip = D.inc_ptr + (size_t)e * (D.max_sv + 1);
  const int* inc = D.inc + (size_t)e * 4 * (D.cap_act + D.cap_anc);
  for (int i = threadIdx.x; i < E.ns; i += NT) {
    double w0 = 0.0, w1 = 0.0, w2 = 0.0;
    for (int q = ip[i]; q < ip[i + 1]; ++q) {
      const int code = inc[q];
      const double* r = R + 12 * (code >> 2) + 3 * (code & 3);
      w0 += r[0]; w1 += r[1]; w2 += r[2];
    }
    W[3 * i] = w0; W[3 * i + 1] = w1; W[3 * i + 2] = w2;
  }
  __syncthreads();
  // y += G^T w : soft free nodes directly, affine bodies by block reduction
  for (int i = threadIdx.x; i < E.ns; i += NT) {
    const int g = E.s0 + i;
    if (D.sv_kind[g] == 0) {
      const int f = D.node_fidx[E.n0 + D.sv_node[g]];
      if (f >= 0)
        for (int c = 0; c < 3; ++c) y[vb + 3 * f + c] += W[3 * i + c];
    }
  }
  for (int a = 0; a < E.na; ++a) {
    const int pn = D.abd_node[E.a0 + a];
    double acc[12];
    for (int c = 0; c < 12; ++c) acc[c] = 0.0;
    for (int i = threadIdx.x; i < E.ns; i += NT) {
      const int g = E.s0 + i;
      if (D.sv_kind[g] != 1 || D.sv_node[g] != pn) continue;
      V3 xi = ld3(D.sv_xi + 3 * g);
      const double* w = W + 3 * i;
      for (int c = 0; c < 3; ++c) {
        acc[c] += w[c];
        acc[3 + 3 * c] += w[c] * xi.x;
        acc[4 + 3 * c] += w[c] * xi.y;
        acc[5 + 3 * c] += w[c] * xi.z;
      }
    }
    for (int c = 0; c < 12; ++c) {
      double v = wsum(acc[c]);
      if ((threadIdx.x & 31) == 0) A.abd_red[threadIdx.x >> 5][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < 12) {
      double s = 0.0;
      for (int w = 0; w < NWARP; ++w) s += A.abd_red[w][threadIdx.x];
      const int f = D.node_fidx[E.n0 + pn];
      y[vb + 3 * f + threadIdx.x] += s;
    }
    __syncthreads();
  }
  __syncthreads();
}

__device__ void precond(const Dev& D, const EnvIx& E, const double* r, double* z) {
  const size_t vb = (size_t)E.e * 3 * D.max_free;
  for (int f = threadIdx.x; f < E.nf; f += NT) {
    const int n = D.free_node[E.f0 + f];
    if (D.node_kind[E.n0 + n] != 0) continue;
    const double* M = D.pcg_pinv + 9 * (size_t)(E.f0 + f);
    const double* q = r + vb + 3 * f;
    for (int c = 0; c < 3; ++c) z[vb + 3 * f + c] = M[3 * c] * q[0] + M[3 * c + 1] * q[1] + M[3 * c + 2] * q[2];
  }
  for (int t = threadIdx.x; t < 12 * E.na; t += NT) {
    const int a = t / 12, i = t - 12 * a;
    const int f = D.node_fidx[E.n0 + D.abd_node[E.a0 + a]];
    const double* M = D.abd_pinv + 144 * (size_t)(E.a0 + a) + 12 * i;
    const double* q = r + vb + 3 * f;
    double s = 0.0;
    for (int j = 0; j < 12; ++j) s += M[j] * q[j];
    z[vb + 3 * f + i] = s;
  }
  __syncthreads();
}

__device__ double vdot(const Dev& D, const EnvIx& E, const double* a, const double* b, Red& sm) {
  const size_t vb = (size_t)E.e * 3 * D.max_free;
  double s = 0.0;
  for (int i = threadIdx.x; i < 3 * E.nf; i += NT) s += a[vb + i] * b[vb + i];
  return block_sum(s, sm);
}

// 12x12 SPD inverse by Cholesky (single thread; tiny)
__device__ bool chol_inv12(double* A) {
  double L[144];
  for (int i = 0; i < 144; ++i) L[i] = 0.0;
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = A[i * 12 + j];
      for (int k = 0; k < j; ++k) s -= L[i * 12 + k] * L[j * 12 + k];
      if (i == j) {
        if (!(s > 0.0)) return false;
        L[i * 12 + i] = sqrt(s);
      } else {
        L[i * 12 + j] = s / L[j * 12 + j];
      }
    }
  // inverse = L^-T L^-1 : solve column by column
  for (int c = 0; c < 12; ++c) {
    double y[12];
    for (int i = 0; i < 12; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[i * 12 + k] * y[k];
      y[i] = s / L[i * 12 + i];
    }
    for (int i = 11; i >= 0; --i) {
      double s = y[i];
      for (int k = i + 1; k < 12; ++k) s -= L[k * 12 + i] * A[k * 12 + c];
      A[i * 12 + c] = s / L[i * 12 + i];
    }
  }
  return true;
}

// solution x (free dofs, pcg layout) -> pdir, residual, convergence / iteration cap (solver.py:663-676)
__device__ void asm_converge(const Dev& D, const EnvIx& E, const double* X, double Etot, Red& sm) {
  const int e = E.e;
  const double* P = P_(D, e);
  const size_t vb = (size_t)e * 3 * D.max_free;
  const int nf3 = 3 * E.nf;
  double res = 0.0;
  for (int i = threadIdx.x; i < nf3; i += NT) res = fmax(res, fabs(X[vb + i]));
  res = block_max(res, sm);
  for (int n = threadIdx.x; n < E.nn; n += NT) {
    const int f = D.node_fidx[E.n0 + n];
    for (int c = 0; c < 3; ++c) D.pdir[3 * (size_t)(E.n0 + n) + c] = f >= 0 ? X[vb + 3 * f + c] : 0.0;
  }
  if (threadIdx.x == 0) {
    D.residual[e] = res;
    const double tol = D.tol[e];
    if (res < tol) {
      D.ns_done[e] = 1;
      D.ns_status[e] = GRIP_NS_CONVERGED;
      D.energy[e] = Etot;
      D.needs_ls[e] = 0;
    } else if (D.iters[e] >= (int)P[GRIP_P_MAXIT]) {
      D.ns_done[e] = 1;
      D.ns_status[e] = GRIP_NS_FAILED;
      D.reason[e] = GRIP_R_NONCONV;
      D.needs_ls[e] = 0;
    } else {
      D.needs_ls[e] = 1;
    }
  }
}

// Assembly shared by both solvers (solver.py:542-586): contact incidence, energy, gradient
// (-g over free dofs in pcg_b) and the static block values (mass + dt^2 element blocks).
// Returns false if the env failed (element error or non-finite assembly).
__device__ bool asm_prologue(const Dev& D, const EnvIx& E, AsmShared& A, double dt2, double* Etot_out) {
#ifdef GRIP_PHASE_TIMING   // sub-phases of the prologue (tests/diag_phase.py)
  long long tl = clock64();
#define PPH(k)                                 \
  do {                                         \
    __syncthreads();                           \
    if (threadIdx.x == 0) {                    \
      const long long t = clock64();           \
      GSTAT(48 + (k), t - tl);                 \
      tl = t;                                  \
    }                                          \
  } while (0)
#else
#define PPH(k) do {} while (0)
#endif
  Red& sm = A.sm;
  const int e = E.e;
  // element-level failures, in the reference's raise order (_elastic before contact)
  if (D.tflag[e] & ERR_INVERTED) { fail_env(D, e, GRIP_R_INVERTED); return false; }
  if (D.flags[e] & ERR_CONTACT_D) { fail_env(D, e, GRIP_R_CONTACT_D); return false; }
  const size_t elbase = (size_t)e * D.cap_el;
  const int nce = D.n_act[e] + D.n_anc[e];
  // ---- contact incidence per sv (element order), used by gradient and SpMV ----
  // counting sort over the 4 nce (element, vertex) items: counts, scan, scatter, then each
  // sv's short list sorted by code = (k << 2) | j, i.e. element order
  int* ip = D.inc_ptr + (size_t)e * (D.max_sv + 1);
  int* inc = D.inc + (size_t)e * 4 * (D.cap_act + D.cap_anc);
  int* cur = D.bp_cnt + (size_t)e * (max(D.max_sv, D.max_edge) + 1);   // broad-phase scratch, free here
  for (int i = threadIdx.x; i < E.ns; i += NT) ip[i] = 0;
  __syncthreads();
  for (int it = threadIdx.x; it < 4 * nce; it += NT)
    atomicAdd(&ip[D.el_idx[(elbase + ce_slot(D, e, it >> 2)) * 4 + (it & 3)]], 1);
  __syncthreads();
  const int tot_inc = block_scan_array(ip, E.ns, sm);
  if (threadIdx.x == 0) ip[E.ns] = tot_inc;
  for (int i = threadIdx.x; i < E.ns; i += NT) cur[i] = ip[i];
  __syncthreads();
  for (int it = threadIdx.x; it < 4 * nce; it += NT) {
    const int v = D.el_idx[(elbase + ce_slot(D, e, it >> 2)) * 4 + (it & 3)];
    inc[atomicAdd(&cur[v], 1)] = it;   // it == (k << 2) | j
  }
  __syncthreads();
  // short lists: insertion sort by one thread; long ones (vertices of the grasped body that
  // many contacts share): rank sort by a warp, every lane ranks its items against the list
  constexpr int INC_SHORT = 12, INC_RANK = 4;   // warp rank sort up to 32 * INC_RANK items
  for (int i = threadIdx.x; i < E.ns; i += NT) {
    const int lo = ip[i], hi = ip[i + 1];
    if (hi - lo > INC_SHORT && hi - lo <= 32 * INC_RANK) continue;
    for (int a = lo + 1; a < hi; ++a) {
      const int t = inc[a];
      int b = a - 1;
      while (b >= lo && inc[b] > t) {
        inc[b + 1] = inc[b];
        --b;
      }
      inc[b + 1] = t;
    }
  }
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int seen = 0;   // long lists are dealt out to warps in sv order (ballot over 32 svs)
    for (int c0 = 0; c0 < E.ns; c0 += 32) {
      const int len = c0 + lane < E.ns ? ip[c0 + lane + 1] - ip[c0 + lane] : 0;
      unsigned m = __ballot_sync(0xffffffffu, len > INC_SHORT && len <= 32 * INC_RANK);
      while (m) {
        const int i = c0 + __ffs(m) - 1;
        m &= m - 1;
        if (seen++ % NWARP != warp) continue;
        const int lo = ip[i], hi = ip[i + 1];
        int t[INC_RANK], r[INC_RANK];
#pragma unroll
        for (int u = 0; u < INC_RANK; ++u) {
          const int a = lo + lane + 32 * u;
          t[u] = a < hi ? inc[a] : 0;
          r[u] = 0;
        }
        for (int b = lo; b < hi; ++b) {   // codes (k << 2) | j are distinct
          const int v = inc[b];
#pragma unroll
          for (int u = 0; u < INC_RANK; ++u) r[u] += v < t[u];
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < INC_RANK; ++u)
          if (lo + lane + 32 * u < hi) inc[lo + r[u]] = t[u];
        __syncwarp();
      }
    }
  }
  __syncthreads();
  PPH(0);
  // ---- energy (solver.py:543-562) ----
  double ein = 0.0;
  for (int n = threadIdx.x; n < E.nn; n += NT) {
    const size_t g = E.n0 + n;
    const double* M = D.node_M + 9 * g;
    double d[3];
    for (int c = 0; c < 3; ++c) d[c] = D.x[3 * g + c] - D.xhat[3 * g + c];
    for (int r = 0; r < 3; ++r) ein += d[r] * (M[3 * r] * d[0] + M[3 * r + 1] * d[1] + M[3 * r + 2] * d[2]);
  }
  ein = 0.5 * block_sum(ein, sm);
  double eel = 0.0;
  for (int k = threadIdx.x; k < E.ntet + E.na; k += NT)
    eel += D.el_E[elbase + (k < E.ntet ? k : D.max_tet + (k - E.ntet))];
  eel = block_sum(eel, sm);
  double ecf = 0.0;
  for (int k = threadIdx.x; k < nce; k += NT) ecf += D.el_E[elbase + ce_slot(D, e, k)];
  ecf = block_sum(ecf, sm);
  const double Etot = ein + dt2 * eel + dt2 * ecf;
  PPH(1);
  // ---- gradient: g = M dx + dt^2 (g_el + G^T g_sv) ----
  double* SG = D.sv_g + (size_t)e * 3 * D.max_sv;
  for (int i = threadIdx.x; i < E.ns; i += NT) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int q = ip[i]; q < ip[i + 1]; ++q) {
      const int code = inc[q];
      const double* gg = D.el_g + (elbase + ce_slot(D, e, code >> 2)) * 12 + 3 * (code & 3);
      s0 += gg[0]; s1 += gg[1]; s2 += gg[2];
    }
    SG[3 * i] = s0; SG[3 * i + 1] = s1; SG[3 * i + 2] = s2;
  }
  __syncthreads();
  PPH(2);
  const size_t vb = (size_t)e * 3 * D.max_free;
  double* RHS = D.pcg_b;  // -g over free dofs
  int nonfinite = !isfinite(Etot);
  for (int n = threadIdx.x; n < E.nn; n += NT) {
    const size_t g = E.n0 + n;
    const double* M = D.node_M + 9 * g;
    double d[3], gr[3];
    for (int c = 0; c < 3; ++c) d[c] = D.x[3 * g + c] - D.xhat[3 * g + c];
    for (int r = 0; r < 3; ++r) gr[r] = M[3 * r] * d[0] + M[3 * r + 1] * d[1] + M[3 * r + 2] * d[2];
    double ge[3] = {0.0, 0.0, 0.0};
    for (int q = D.tinc_ptr[g]; q < D.tinc_ptr[g + 1]; ++q) {
      const int code = D.tinc[q];
      const double* gg = D.el_g + (elbase + (code >> 2)) * 12 + 3 * (code & 3);
      for (int c = 0; c < 3; ++c) ge[c] += gg[c];
    }
    const int kind = D.node_kind[g];
    if (kind == 0) {
      const int s = D.node_sv[g];
      if (s >= 0)
        for (int c = 0; c < 3; ++c) ge[c] += SG[3 * s + c];
    }
    for (int c = 0; c < 3; ++c) {
      gr[c] += dt2 * ge[c];
      if (!isfinite(gr[c])) nonfinite = 1;
    }
    const int f = D.node_fidx[g];
    if (f >= 0 && kind == 0)
      for (int c = 0; c < 3; ++c) RHS[vb + 3 * f + c] = -gr[c];
    if (kind != 0) {  // affine: contact part added below
      if (f >= 0)
        for (int c = 0; c < 3; ++c) RHS[vb + 3 * f + c] = -gr[c];
    }
  }
  __syncthreads();
  for (int a = 0; a < E.na; ++a) {
    const int pn = D.abd_node[E.a0 + a];
    double acc[12];
    for (int c = 0; c < 12; ++c) acc[c] = 0.0;
    for (int i = threadIdx.x; i < E.ns; i += NT) {
      const int g = E.s0 + i;
      if (D.sv_kind[g] != 1 || D.sv_node[g] != pn) continue;
      V3 xi = ld3(D.sv_xi + 3 * g);
      const double* w = SG + 3 * i;
      for (int c = 0; c < 3; ++c) {
        acc[c] += w[c];
        acc[3 + 3 * c] += w[c] * xi.x;
        acc[4 + 3 * c] += w[c] * xi.y;
        acc[5 + 3 * c] += w[c] * xi.z;
      }
    }
    for (int c = 0; c < 12; ++c) {
      double v = wsum(acc[c]);
      if ((threadIdx.x & 31) == 0) A.abd_red[threadIdx.x >> 5][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < 12) {
      double s = 0.0;
      for (int w = 0; w < NWARP; ++w) s += A.abd_red[w][threadIdx.x];
      const int f = D.node_fidx[E.n0 + pn];
      RHS[vb + 3 * f + threadIdx.x] -= dt2 * s;
    }
    __syncthreads();
  }
  PPH(3);
  for (int i = threadIdx.x; i < 3 * E.nf; i += NT) nonfinite |= !isfinite(RHS[vb + i]);
  nonfinite = block_or(nonfinite, sm);
  if (nonfinite) { fail_env(D, e, GRIP_R_NONFINITE); return false; }
  PPH(4);
  // static block values (mass + dt^2 * element blocks): k_static, on the second stream
  PPH(5);
#undef PPH
  *Etot_out = Etot;
  return true;
}

__global__ void __launch_bounds__(NT) k_assemble_solve(Dev D, const int* list) {
  __shared__ AsmShared A;
  Red& sm = A.sm;
  const int e = list[blockIdx.x];
  if (D.ns_done[e] || (D.flags[e] & FLAG_OVERFLOW)) return;
  const EnvIx E = env_ix(D, e);
  const double* P = P_(D, e);
  const double dt = P[GRIP_P_DT], dt2 = dt * dt;
  const size_t elbase = (size_t)e * D.cap_el;
  const int nce = D.n_act[e] + D.n_anc[e];
  int* ip = D.inc_ptr + (size_t)e * (D.max_sv + 1);
  int* inc = D.inc + (size_t)e * 4 * (D.cap_act + D.cap_anc);
  const size_t vb = (size_t)e * 3 * D.max_free;
  double* RHS = D.pcg_b;
  double Etot = 0.0;
  if (!asm_prologue(D, E, A, dt2, &Etot)) return;
  // ---- preconditioner: soft 3x3 diagonal blocks, affine 12x12 body blocks ----
  for (int f = threadIdx.x; f < E.nf; f += NT) {
    const int fg = E.f0 + f;
    const int n = D.free_node[fg];
    if (D.node_kind[E.n0 + n] != 0) continue;
    double Bd[9];
    for (int i = 0; i < 9; ++i) Bd[i] = D.sb_val[9 * (size_t)D.sb_diag[fg] + i];
    const int s = D.node_sv[E.n0 + n];
    if (s >= 0)
      for (int q = ip[s]; q < ip[s + 1]; ++q) {
        const int code = inc[q];
        const int sl = code & 3;
        const double* H = D.el_H + (elbase + ce_slot(D, e, code >> 2)) * 144;
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) Bd[3 * i + j] += dt2 * H[(3 * sl + i) * 12 + 3 * sl + j];
      }
    inv3(Bd, D.pcg_pinv + 9 * (size_t)fg);
  }
  for (int a = 0; a < E.na; ++a) {
    const int pn = D.abd_node[E.a0 + a];
    const int fp = D.node_fidx[E.n0 + pn];
    // static part: blocks among the 4 pseudo-nodes
    for (int t = threadIdx.x; t < 144; t += NT) {
      const int i = t / 12, j = t % 12;
      const int fg = E.f0 + fp + i / 3;
      double s = 0.0;
      for (int b = D.sb_rowptr[fg]; b < D.sb_rowptr[fg + 1]; ++b)
        if (D.sb_col[b] == fp + j / 3) s = D.sb_val[9 * (size_t)b + 3 * (i % 3) + (j % 3)];
      // contacts: sum_e sum_{k,l on body} J_k^T H_kl J_l
      double c = 0.0;
      const int ni = i / 3, ci = i % 3, nj = j / 3, cj = j % 3;
      for (int k = 0; k < nce; ++k) {
        const size_t sl = elbase + ce_slot(D, e, k);
        const int* ix = D.el_idx + sl * 4;
        const double* H = D.el_H + sl * 144;
        for (int u = 0; u < 4; ++u) {
          const int gu = E.s0 + ix[u];
          if (D.sv_kind[gu] != 1 || D.sv_node[gu] != pn) continue;
          const double au = ni == 0 ? 1.0 : D.sv_xi[3 * (size_t)gu + ci];
          const int ra = ni == 0 ? ci : ni - 1;
          for (int w2 = 0; w2 < 4; ++w2) {
            const int gw = E.s0 + ix[w2];
            if (D.sv_kind[gw] != 1 || D.sv_node[gw] != pn) continue;
            const double aw = nj == 0 ? 1.0 : D.sv_xi[3 * (size_t)gw + cj];
            const int cb = nj == 0 ? cj : nj - 1;
            c += au * aw * H[(3 * u + ra) * 12 + 3 * w2 + cb];
          }
        }
      }
      A.chol[t] = s + dt2 * c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (!chol_inv12(A.chol)) {
        // fall back to the diagonal (still SPD direction) if the block is not PD
        for (int i = 0; i < 144; ++i) A.chol[i] = (i % 13 == 0 && A.chol[i] != 0.0) ? 1.0 / A.chol[i] : 0.0;
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 144; t += NT) D.abd_pinv[144 * (size_t)(E.a0 + a) + t] = A.chol[t];
    __syncthreads();
  }
  // ---- PCG on H_ff p = -g_f (rtol P[PCGRTOL]); regularized retry (solver.py:111-131) ----
  double* X = D.pcg_x;
  double* R = D.pcg_r;
  double* Z = D.pcg_z;
  double* Pp = D.pcg_p;
  double* Q = D.pcg_q;
  const int nf3 = 3 * E.nf;
  double bnorm2 = 0.0;
  for (int i = threadIdx.x; i < nf3; i += NT) bnorm2 += RHS[vb + i] * RHS[vb + i];
  bnorm2 = block_sum(bnorm2, sm);
  const double rtol = P[GRIP_P_PCGRTOL];
  int pcg_total = 0;
  bool solved = false;
  double shift = 0.0;
  if (bnorm2 == 0.0) {
    for (int i = threadIdx.x; i < nf3; i += NT) X[vb + i] = 0.0;
    solved = true;
  }
  const int maxit = max(200, 4 * nf3);
  for (int attempt = 0; attempt < 2 && !solved; ++attempt) {
    if (attempt == 1) {
      // shift = 1e-8 * max(max diag, 1) on every diagonal entry
      double md = -INFINITY;
      for (int f = threadIdx.x; f < E.nf; f += NT) {
        const double* Bd = D.sb_val + 9 * (size_t)D.sb_diag[E.f0 + f];
        md = fmax(md, fmax(Bd[0], fmax(Bd[4], Bd[8])));
      }
      md = block_max(md, sm);
      shift = 1e-8 * fmax(md, 1.0);
      for (int f = threadIdx.x; f < E.nf; f += NT) {
        double* Bd = D.sb_val + 9 * (size_t)D.sb_diag[E.f0 + f];
        Bd[0] += shift; Bd[4] += shift; Bd[8] += shift;
      }
      if (threadIdx.x == 0) D.regularized[e] = 1;
      __syncthreads();
    }
    // r = b (stored in R), x = 0
    for (int i = threadIdx.x; i < nf3; i += NT) {
      X[vb + i] = 0.0;
      R[vb + i] = RHS[vb + i];
    }
    __syncthreads();
    precond(D, E, R, Z);
    for (int i = threadIdx.x; i < nf3; i += NT) Pp[vb + i] = Z[vb + i];
    __syncthreads();
    double rz = vdot(D, E, R, Z, sm);
    const double stop2 = rtol * rtol * bnorm2;
    int it = 0;
    bool conv = false, broke = false;
    for (; it < maxit; ++it) {
      spmv(D, E, dt2, Pp, Q, A);
      const double pq = vdot(D, E, Pp, Q, sm);
      if (!(pq > 0.0) || !isfinite(pq)) { broke = true; break; }
      const double alpha = rz / pq;
      double rr = 0.0;
      for (int i = threadIdx.x; i < nf3; i += NT) {
        X[vb + i] += alpha * Pp[vb + i];
        const double rv = R[vb + i] - alpha * Q[vb + i];
        R[vb + i] = rv;
        rr += rv * rv;
      }
      rr = block_sum(rr, sm);
      if (!isfinite(rr)) { broke = true; break; }
      if (rr <= stop2) { conv = true; ++it; break; }
      precond(D, E, R, Z);
      const double rz2 = vdot(D, E, R, Z, sm);
      const double beta = rz2 / rz;
      rz = rz2;
      for (int i = threadIdx.x; i < nf3; i += NT) Pp[vb + i] = Z[vb + i] + beta * Pp[vb + i];
      __syncthreads();
    }
    pcg_total += it;
    // accept on the TRUE residual |b - H x| <= 1e-8 |b| (the reference's acceptance bound,
    // solver.py:121) when the recursive residual stalled short of rtol
    if (!conv) {
      spmv(D, E, dt2, X, Q, A);
      double tr = 0.0;
      for (int i = threadIdx.x; i < nf3; i += NT) {
        const double rv = RHS[vb + i] - Q[vb + i];
        tr += rv * rv;
      }
      tr = block_sum(tr, sm);
      conv = isfinite(tr) && tr <= 1e-16 * bnorm2;
    }
    (void)broke;
    solved = conv;
  }
  if (threadIdx.x == 0) {
    D.pcg_iters[e] += pcg_total;
    atomicAdd(&D.stats[4], (double)pcg_total);   // PCG iterations (bench statistics)
    atomicAdd(&D.stats[5], 1.0);                 // linear solves
    atomicAdd(&D.stats[6], (double)(3 * E.nf));  // unknowns (sum)
  }
  if (!solved) { fail_env(D, e, GRIP_R_SOLVE); return; }
  asm_converge(D, E, X, Etot, sm);

}

// ---------------------------------------------------------------------------
// Newton sweep 4/4: CCD + inversion filters + backtracking line search
// (solver.py:678-726, _energy_only :518-533)
// ---------------------------------------------------------------------------

// incremental potential at x + a p with candidate set c2; +inf if invalid
// Total incremental potential at the NA trial points x + a[k] p (solver.py:518-533 _energy_only):
// inertia + dt^2 (elastic + orthogonality + barrier over the frozen candidate set + friction),
// +inf on an inverted element, a non-positive distance or a non-finite total.  One pass over the
// elements serves all NA points (their loads shared); every value goes through the same per-thread
// order and reduction tree as a single evaluation, so each out[k] is bitwise the 1-point result.
constexpr int LS_NA = 4;
template <int NA>
__device__ void env_energy_n(const Dev& D, const EnvIx& E, const double* a, const int* cpt, int npt, const int* cee,
                             const int* ceid, int nee, double* out, Red& sm) {
  const int e = E.e;
  const double* P = P_(D, e);
  const double dt = P[GRIP_P_DT], kappa = P[GRIP_P_KAPPA], dhat = P[GRIP_P_DHAT];
  const size_t ys = 3 * (size_t)D.max_sv;
  double* Y = D.ls_y + (size_t)e * LS_NA * ys;   // trial sv positions (scratch), NA slices
  // trial surface positions: surface_positions(x + a p) (solver.py:525)
  for (int i = threadIdx.x; i < E.ns; i += NT) {
    const int g = E.s0 + i;
    const int kind = D.sv_kind[g];
    if (kind == 2) {
      const V3 y = ld3(D.kin_pos + 3 * (size_t)g);
#pragma unroll
      for (int k = 0; k < NA; ++k) st3(Y + k * ys + 3 * i, y);
      continue;
    }
    const size_t nb = E.n0 + D.sv_node[g];
    if (kind == 0) {
      const V3 xv = ld3(D.x + 3 * nb), pv = ld3(D.pdir + 3 * nb);
#pragma unroll
      for (int k = 0; k < NA; ++k) st3(Y + k * ys + 3 * i, xv + a[k] * pv);
    } else {
      double xq[12], pq[12];
      for (int c = 0; c < 12; ++c) {
        xq[c] = D.x[3 * nb + c];
        pq[c] = D.pdir[3 * nb + c];
      }
      const V3 xi = ld3(D.sv_xi + 3 * g);
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        double q[12];
        for (int c = 0; c < 12; ++c) q[c] = xq[c] + a[k] * pq[c];
        st3(Y + k * ys + 3 * i, V3{q[0] + xi.x * q[3] + xi.y * q[4] + xi.z * q[5],
                                   q[1] + xi.x * q[6] + xi.y * q[7] + xi.z * q[8],
                                   q[2] + xi.x * q[9] + xi.y * q[10] + xi.z * q[11]});
      }
    }
  }
  __syncthreads();
  int bad = 0;   // bit k: trial point k is invalid
  double ein[NA], eel[NA], ec[NA], ef[NA];
#pragma unroll
  for (int k = 0; k < NA; ++k) ein[k] = eel[k] = ec[k] = ef[k] = 0.0;
  for (int n = threadIdx.x; n < E.nn; n += NT) {
    const size_t g = E.n0 + n;
    const double* M = D.node_M + 9 * g;
    double xg[3], pg[3], xh[3];
    for (int c = 0; c < 3; ++c) {
      xg[c] = D.x[3 * g + c];
      pg[c] = D.pdir[3 * g + c];
      xh[c] = D.xhat[3 * g + c];
    }
#pragma unroll
    for (int k = 0; k < NA; ++k) {
      double d[3];
      for (int c = 0; c < 3; ++c) d[c] = (xg[c] + a[k] * pg[c]) - xh[c];
      for (int r = 0; r < 3; ++r) ein[k] += d[r] * (M[3 * r] * d[0] + M[3 * r + 1] * d[1] + M[3 * r + 2] * d[2]);
    }
  }
  for (int t = threadIdx.x; t < E.ntet; t += NT) {
    const int tg = E.te0 + t;
    V3 xv[4], pv[4];
    for (int j = 0; j < 4; ++j) {
      const size_t g = E.n0 + D.tet_nodes[4 * (size_t)tg + j];
      xv[j] = ld3(D.x + 3 * g);
      pv[j] = ld3(D.pdir + 3 * g);
    }
    const double* Dmi = D.tet_Dmi + 9 * (size_t)tg;
    const double V0 = D.tet_V0[tg], mu = D.tet_mu[tg], lam = D.tet_lam[tg];
#pragma unroll
    for (int k = 0; k < NA; ++k) {
      V3 x[4];
      for (int j = 0; j < 4; ++j) x[j] = xv[j] + a[k] * pv[j];
      double el = 0.0;
      if (nh_element(x, Dmi, V0, mu, lam, &el, nullptr, nullptr) & EL_INVERTED) bad |= 1 << k;
      else eel[k] += el;
    }
  }
  for (int m = threadIdx.x; m < E.na; m += NT) {
    const size_t g = E.n0 + D.abd_node[E.a0 + m];
#pragma unroll
    for (int k = 0; k < NA; ++k) {
      double Am[9];
      for (int c = 0; c < 9; ++c) Am[c] = D.x[3 * g + 3 + c] + a[k] * D.pdir[3 * g + 3 + c];
      eel[k] += abd_element(Am, D.abd_kV[E.a0 + m], nullptr, nullptr);
    }
  }
  for (int m = threadIdx.x; m < npt + nee; m += NT) {
    const bool is_ee = m >= npt;
    const int* row = is_ee ? cee + 4 * (m - npt) : cpt + 4 * m;
    int rv[4];
    for (int j = 0; j < 4; ++j) rv[j] = row[j];
    const double epsx = is_ee ? D.edge_rest_sq[E.ed0 + ceid[2 * (m - npt)]] * D.edge_rest_sq[E.ed0 + ceid[2 * (m - npt) + 1]]
                              : 0.0;
#pragma unroll
    for (int k = 0; k < NA; ++k) {
      V3 x[4];
      for (int j = 0; j < 4; ++j) x[j] = ld3(Y + k * ys + 3 * rv[j]);
      double el = 0.0;
      const int fl = is_ee ? ee_element(x, epsx, kappa, dhat, &el, nullptr, nullptr, 0)
                           : pt_element(x, kappa, dhat, &el, nullptr, nullptr, 0);
      if (fl & EL_BAD_D) bad |= 1 << k;
      else if (fl & EL_ACTIVE) ec[k] += el;
    }
  }
  const int nanc = D.n_anc[e];
  for (int m = threadIdx.x; m < nanc; m += NT) {
    const size_t ai = (size_t)e * D.cap_anc + m;
    int sv[4];
    V3 xp[4];
    for (int j = 0; j < 4; ++j) {
      sv[j] = D.anc_v[4 * ai + j];
      xp[j] = ld3(D.surf_prev + 3 * (size_t)(E.s0 + sv[j]));
    }
#pragma unroll
    for (int k = 0; k < NA; ++k) {
      V3 x[4];
      for (int j = 0; j < 4; ++j) x[j] = ld3(Y + k * ys + 3 * sv[j]);
      ef[k] += friction_element(x, xp, D.anc_gamma + 4 * ai, D.anc_T + 6 * ai, D.anc_lam[ai], D.anc_mu[ai],
                                P[GRIP_P_EPSV], dt, nullptr, nullptr);
    }
  }
  bad = block_or(bad, sm);
  double v[4];
#pragma unroll
  for (int k = 0; k < NA; ++k) v[k] = ein[k];
  block_sum_n<NA>(v, sm);
#pragma unroll
  for (int k = 0; k < NA; ++k) ein[k] = 0.5 * v[k], v[k] = eel[k];
  block_sum_n<NA>(v, sm);
#pragma unroll
  for (int k = 0; k < NA; ++k) eel[k] = v[k], v[k] = ec[k];
  block_sum_n<NA>(v, sm);
#pragma unroll
  for (int k = 0; k < NA; ++k) ec[k] = v[k], v[k] = ef[k];
  block_sum_n<NA>(v, sm);
#pragma unroll
  for (int k = 0; k < NA; ++k) {
    const double tot = ein[k] + dt * dt * (eel[k] + ec[k] + v[k]);
    out[k] = ((bad >> k) & 1) || !isfinite(tot) ? INFINITY : tot;
  }
}

// A cluster of BP_CL CTAs per env: every rank computes the step's max surface displacement and
// whether the candidate superset covers dhat + 2 md; after one cluster barrier (the decision's
// inputs are only written by rank 0 after it) the other ranks exit, or join a fresh broad phase
// (BPCl) and then exit; rank 0 runs the line search.
__global__ void __cluster_dims__(BP_CL, 1, 1) __launch_bounds__(NT) k_linesearch(Dev D, const int* list) {
  __shared__ Red sm;
  __shared__ BPShared S;
  const BPCl cl{(int)cooperative_groups::this_cluster().block_rank(), BP_CL};
  const int e = list[blockIdx.x / BP_CL];
  CTA_TIMER_IF(cl.rank == 0, 3, e);
  EigCommit commit_(D, e, cl.rank == 0);   // on every return path of rank 0
  if (D.ns_done[e] || !D.needs_ls[e] || (D.flags[e] & FLAG_OVERFLOW)) return;
  const EnvIx E = env_ix(D, e);
  const double* P = P_(D, e);
  const double dhat = P[GRIP_P_DHAT], scaling = P[GRIP_P_CCDSCALE];
  // disp = G p and its max norm
  if (cl.rank == 0) env_sv_positions(D, E, D.x);
  double md = 0.0;
  for (int i = threadIdx.x; i < E.ns; i += NT) {
    V3 d = sv_dir(D, E, i, D.pdir);
    if (cl.rank == 0) st3(D.sv_disp + 3 * (size_t)(E.s0 + i), d);
    md = fmax(md, norm(d));
  }
  md = block_max(md, sm);
  int* cn = D.c2_n + 2 * e;
  int* cpt = D.c2_pt + (size_t)e * 4 * D.cap_pt;
  int* cee = D.c2_ee + (size_t)e * 4 * D.cap_ee;
  int* ceid = D.c2_eid + (size_t)e * 2 * D.cap_ee;
  const double r2 = dhat + 2.0 * md;
  const bool reuse = cs_covers(D, e, r2);
  cl_sync(cl);
  if (cl.rank != 0 && reuse) return;
  if (cl.rank == 0 && threadIdx.x == 0) D.md_prev[e] = md;
  if (reuse) {
    filter_from_superset(D, E, r2, cpt, cee, ceid, cn, sm);
  } else if (!broad_phase_env(D, E, r2, cpt, cee, ceid, cn, S, sm, cl)) {
    if (cl.rank == 0 && threadIdx.x == 0) D.flags[e] |= FLAG_OVERFLOW;
    return;
  }
  if (cl.rank != 0) return;
  if (!reuse) CTA_INFO(1u);
  const int npt = cn[0], nee = cn[1];
  double alpha0 = 1.0;
  if (npt + nee > 0) {
    int bad = 0;
    const double a = env_ccd(D, E, cpt, npt, cee, nee, scaling, (int)P[GRIP_P_CCDIT], 0.0, &bad, sm);
    if (bad) { fail_env(D, e, GRIP_R_CCD); return; }
    alpha0 = fmin(alpha0, a);
  }
  // tet inversion filter (ccd.py:191-204)
  if (E.ntet > 0) {
    int anyp = 0, bad = 0;
    double tmin = INFINITY;
    for (int t = threadIdx.x; t < E.ntet; t += NT) {
      const int tg = E.te0 + t;
      V3 x[4], p[4];
      for (int j = 0; j < 4; ++j) {
        const size_t g = E.n0 + D.tet_nodes[4 * (size_t)tg + j];
        x[j] = ld3(D.x + 3 * g);
        p[j] = ld3(D.pdir + 3 * g);
        if (p[j].x != 0.0 || p[j].y != 0.0 || p[j].z != 0.0) anyp = 1;
      }
      double M0[9], dM[9];
      tet_edge_matrix(x, M0);
      tet_edge_matrix(p, dM);
      const double d0 = det3(M0);
      if (!(d0 > 0.0)) bad = 1;
      else tmin = fmin(tmin, pencil_root(M0, dM, d0));
    }
    anyp = block_or(anyp, sm);
    if (anyp) {
      bad = block_or(bad, sm);
      if (bad) { fail_env(D, e, GRIP_R_DET); return; }
      tmin = block_min(tmin, sm);
      if (tmin <= 1.0) {
        double a = scaling * tmin;
        bool okall = false;
        CTA_INFO(2u);
        for (int it = 0; it < 60; ++it) {
          int neg = 0;
          for (int t = threadIdx.x; t < E.ntet; t += NT) {
            const int tg = E.te0 + t;
            V3 x[4], p[4];
            for (int j = 0; j < 4; ++j) {
              const size_t g = E.n0 + D.tet_nodes[4 * (size_t)tg + j];
              x[j] = ld3(D.x + 3 * g);
              p[j] = ld3(D.pdir + 3 * g);
            }
            double M0[9], dM[9], Mt[9];
            tet_edge_matrix(x, M0);
            tet_edge_matrix(p, dM);
            for (int c = 0; c < 9; ++c) Mt[c] = M0[c] + a * dM[c];
            if (!(det3(Mt) > 0.0)) neg = 1;
          }
          neg = block_or(neg, sm);
          if (!neg) { okall = true; break; }
          a *= 0.5;
        }
        alpha0 = fmin(alpha0, okall ? a : 0.0);
      }
    }
  }
  // affine bodies: det(A + t dA) > 0 (solver.py:695-700)
  for (int k = 0; k < E.na; ++k) {
    const size_t g = E.n0 + D.abd_node[E.a0 + k];
    double A0[9], dA[9];
    bool any = false;
    for (int c = 0; c < 9; ++c) {
      A0[c] = D.x[3 * g + 3 + c];
      dA[c] = D.pdir[3 * g + 3 + c];
      any |= dA[c] != 0.0;
    }
    if (!any) continue;
    const double d0 = det3(A0);
    if (!(d0 > 0.0)) { fail_env(D, e, GRIP_R_DET); return; }
    const double t = pencil_root(A0, dA, d0);
    if (t > 1.0) continue;
    double a = scaling * t;
    bool okv = false;
    for (int it = 0; it < 60; ++it) {
      double Mt[9];
      for (int c = 0; c < 9; ++c) Mt[c] = A0[c] + a * dA[c];
      if (det3(Mt) > 0.0) { okv = true; break; }
      a *= 0.5;
    }
    alpha0 = fmin(alpha0, okv ? a : 0.0);
  }
  // backtracking on strict decrease (solver.py:702-720): E0 and the first trial share one energy
  // pass; after a rejection the next LS_NA halvings are evaluated together (the first that
  // decreases is taken, exactly the sequential loop's choice: alpha halves exactly)
  const int maxls = (int)P[GRIP_P_MAXLS];
  double alpha = alpha0, Et = INFINITY, E0;
  bool accepted = false;
  {
    const double a2[2] = {0.0, alpha};
    double e2[2];
    env_energy_n<2>(D, E, a2, cpt, npt, cee, ceid, nee, e2, sm);
    E0 = e2[0];
    if (maxls > 0) {
      Et = e2[1];
      if (Et < E0) accepted = true;
      else alpha *= 0.5;
    }
  }
  for (int it = 1; it < maxls && !accepted; it += LS_NA) {
    double av[LS_NA], ev[LS_NA];
    for (int k = 0; k < LS_NA; ++k) av[k] = k == 0 ? alpha : av[k - 1] * 0.5;
    env_energy_n<LS_NA>(D, E, av, cpt, npt, cee, ceid, nee, ev, sm);
    CTA_INFO_ADD(1u << 8);
    for (int k = 0; k < LS_NA && it + k < maxls; ++k) {
      Et = ev[k];
      alpha = av[k];
      if (Et < E0) { accepted = true; break; }
    }
    if (!accepted) alpha *= 0.5;
  }
  if (!accepted) {
    if (threadIdx.x == 0) {
      D.ns_done[e] = 1;
      D.needs_ls[e] = 0;
      if (D.residual[e] < 10.0 * D.tol[e]) {
        D.ns_status[e] = GRIP_NS_CONVERGED;
        D.energy[e] = E0;
      } else {
        D.ns_status[e] = GRIP_NS_FAILED;
        D.reason[e] = GRIP_R_LINESEARCH;
      }
    }
    return;
  }
  for (int i = threadIdx.x; i < 3 * E.nn; i += NT) {
    const size_t g = 3 * (size_t)E.n0 + i;
    D.x[g] = D.x[g] + alpha * D.pdir[g];
  }
  cs_moved(D, e, alpha * md);  // x moved
  if (threadIdx.x == 0) {
    const int it = D.iters[e];
    if (it < D.max_alpha) D.alphas[(size_t)e * D.max_alpha + it] = alpha;
    D.iters[e] = it + 1;
    D.energy[e] = Et;
    D.needs_ls[e] = 0;
  }
}

// pending list compaction: keep envs still iterating (including overflowed ones)
__global__ void __launch_bounds__(NT) k_compact(Dev D, const int* list, int n, int* out, int* out_n, int* any_overflow) {
  __shared__ Red sm;
  int base = 0, ov = 0;
  for (int s = 0; s < n; s += NT) {
    const int i = s + threadIdx.x;
    int keep = 0, e = -1;
    if (i < n) {
      e = list[i];
      keep = !D.ns_done[e];
      ov |= (D.flags[e] & FLAG_OVERFLOW) ? 1 : 0;
    }
    int tot;
    const int pre = block_scan(keep, sm, &tot);
    if (keep) out[base + pre] = e;
    base += tot;
  }
  ov = block_or(ov, sm);
  if (threadIdx.x == 0) {
    *out_n = base;
    *any_overflow = ov;
  }
}

// ---------------------------------------------------------------------------
// finalize_step (solver.py:733-762) + contact readout (protocol.py:72-98)
// ---------------------------------------------------------------------------
__device__ void finalize_env(const Dev& D, int e, int only_done, Red& sm, BPShared& S, unsigned int* cmask);

__global__ void __launch_bounds__(NT) k_finalize(Dev D, const int* list, int only_done = 0) {
  __shared__ Red sm;
  __shared__ BPShared S;
  __shared__ unsigned int cmask[32];
  const int e = list[blockIdx.x];
  CTA_TIMER(4, e);
  finalize_env(D, e, only_done, sm, S, cmask);
}

__device__ void finalize_env(const Dev& D, int e, int only_done, Red& sm, BPShared& S, unsigned int* cmask) {
  if (only_done && (!D.ns_done[e] || D.fin_done[e] || (D.flags[e] & FLAG_OVERFLOW))) return;
  const EnvIx E = env_ix(D, e);
  const double* P = P_(D, e);
  const double dt = P[GRIP_P_DT], kappa = P[GRIP_P_KAPPA], dhat = P[GRIP_P_DHAT];
  __syncthreads();
  if (threadIdx.x == 0) D.flags[e] = 0;
  // a failed step keeps x, v and the anchors (solver.py:736-738); the contact readout the
  // protocol does after every step (protocol.py:179-180) is still produced
  const bool failed = D.ns_status[e] == GRIP_NS_FAILED;
  if (!failed)
    for (int i = threadIdx.x; i < 3 * E.nn; i += NT) {
      const size_t g = 3 * (size_t)E.n0 + i;
      D.v[g] = (D.x[g] - D.x_t[g]) / dt;
    }
  env_sv_positions(D, E, D.x);
  int* cn = D.c1_n + 2 * e;
  int* cpt = D.c1_pt + (size_t)e * 4 * D.cap_pt;
  int* cee = D.c1_ee + (size_t)e * 4 * D.cap_ee;
  int* ceid = D.c1_eid + (size_t)e * 2 * D.cap_ee;
  if (!ensure_superset(D, E, 1.05 * dhat, dhat, S, sm)) {
    if (threadIdx.x == 0) D.flags[e] |= FLAG_OVERFLOW | FLAG_OVF_FIN;
    return;
  }
  filter_from_superset(D, E, dhat * 1.05, cpt, cee, ceid, cn, sm);
  const int npt = cn[0], nee = cn[1];
  const double* X = D.sv_pos + 3 * (size_t)E.s0;
  if (threadIdx.x < 32) cmask[threadIdx.x] = 0u;
  __syncthreads();
  // anchors from active stencils, PT then EE in candidate order (contact.py:413-472)
  double dmin = INFINITY;
  int base = 0;
  double fsum[32];
  const int nbl = min(E.nb, 32);
  for (int b = 0; b < nbl; ++b) fsum[b] = 0.0;
  for (int s = 0; s < npt + nee; s += NT) {
    const int k = s + threadIdx.x;
    int act = 0;
    double lam = 0.0, gam[4], Tm[6], mu = 0.0, dmin_k = 0.0;
    int rowv[4], bb[2];
    if (k < npt + nee) {
      const bool is_ee = k >= npt;
      const int* row = is_ee ? cee + 4 * (k - npt) : cpt + 4 * k;
      V3 x[4];
      for (int j = 0; j < 4; ++j) {
        rowv[j] = row[j];
        x[j] = ld3(X + 3 * row[j]);
      }
      double Dq, bary[3], sp = 0.0, tp = 0.0;
      Dq = is_ee ? ee_closest(x[0], x[1], x[2], x[3], &sp, &tp) : pt_closest(x[0], x[1], x[2], x[3], bary, nullptr);
      dmin = fmin(dmin, Dq);
      dmin_k = Dq;
      if (Dq < dhat * dhat) {
        act = 1;
        const double d = sqrt(Dq);
        double b0, b1, b2;
        barrier_d(d, dhat, &b0, &b1, &b2);
        V3 pa, pb;
        if (is_ee) {
          double c = cross_norm_sq(x, nullptr, nullptr);
          const int* eid = ceid + 2 * (k - npt);
          double m, dm, d2m;
          edge_mollifier(c, D.edge_rest_sq[E.ed0 + eid[0]] * D.edge_rest_sq[E.ed0 + eid[1]], &m, &dm, &d2m);
          lam = kappa * m * fabs(b1);
          pa = (1.0 - sp) * x[0] + sp * x[1];
          pb = (1.0 - tp) * x[2] + tp * x[3];
          gam[0] = 1.0 - sp; gam[1] = sp; gam[2] = -(1.0 - tp); gam[3] = -tp;
          bb[0] = D.sv_body[E.s0 + row[0]];
          bb[1] = D.sv_body[E.s0 + row[2]];
        } else {
          lam = kappa * fabs(b1);
          pa = x[0];
          pb = bary[0] * x[1] + bary[1] * x[2] + bary[2] * x[3];
          gam[0] = 1.0; gam[1] = -bary[0]; gam[2] = -bary[1]; gam[3] = -bary[2];
          bb[0] = D.sv_body[E.s0 + row[0]];
          bb[1] = D.sv_body[E.s0 + row[1]];
        }
        const double ma = D.body_mu[E.b0 + bb[0]], mb = D.body_mu[E.b0 + bb[1]];
        mu = P[GRIP_P_MURULE] == 0.0 ? sqrt(ma * mb) : fmin(ma, mb);
        const double id = 1.0 / d;
        V3 n = V3{(pa.x - pb.x) / d, (pa.y - pb.y) / d, (pa.z - pb.z) / d};
        (void)id;
        // tangent basis (contact.py:403-410): ref = e_argmin|n|
        const double ax = fabs(n.x), ay = fabs(n.y), az = fabs(n.z);
        V3 ref = (ax <= ay && ax <= az) ? V3{1, 0, 0} : ((ay <= az) ? V3{0, 1, 0} : V3{0, 0, 1});
        V3 t1 = cross(ref, n);
        const double l1 = norm(t1);
        t1 = V3{t1.x / l1, t1.y / l1, t1.z / l1};
        V3 t2 = cross(n, t1);
        Tm[0] = t1.x; Tm[1] = t2.x; Tm[2] = t1.y; Tm[3] = t2.y; Tm[4] = t1.z; Tm[5] = t2.z;
        for (int b = 0; b < nbl; ++b)
          if (bb[0] == b || bb[1] == b) fsum[b] += lam;
        if (bb[0] < 32 && bb[1] < 32) {
          atomicOr(&cmask[bb[0]], 1u << bb[1]);
          atomicOr(&cmask[bb[1]], 1u << bb[0]);
        }
      }
    }
    int tot;
    const int pre = block_scan(act, sm, &tot);
    if (act && D.ev_on && base + pre < D.cap_anc) {
      const size_t vi = (size_t)e * D.cap_anc + base + pre;
      int* ei = D.ev_i + 7 * vi;
      ei[0] = k >= npt;
      ei[1] = bb[0];
      ei[2] = bb[1];
      for (int j = 0; j < 4; ++j) ei[3 + j] = rowv[j];
      D.ev_d[2 * vi] = sqrt(dmin_k);
      D.ev_d[2 * vi + 1] = lam;
    }
    if (act && !failed && base + pre < D.cap_anc) {
      const size_t ai = (size_t)e * D.cap_anc + base + pre;
      for (int j = 0; j < 4; ++j) {
        D.anc_v[4 * ai + j] = rowv[j];
        D.anc_gamma[4 * ai + j] = gam[j];
      }
      for (int j = 0; j < 6; ++j) D.anc_T[6 * ai + j] = Tm[j];
      D.anc_lam[ai] = lam;
      D.anc_mu[ai] = mu;
      D.anc_b[2 * ai] = bb[0];
      D.anc_b[2 * ai + 1] = bb[1];
    }
    base += tot;
  }
  if (base > D.cap_anc && !failed) {
    if (threadIdx.x == 0) {
      D.flags[e] |= FLAG_OVERFLOW | FLAG_OVF_FIN;
      atomicMax(&D.need[3], (unsigned)base);
    }
    return;
  }
  dmin = block_min(dmin, sm);
  for (int b = 0; b < nbl; ++b) {
    const double f = block_sum(fsum[b], sm);
    if (threadIdx.x == 0) D.body_force[E.b0 + b] = f;
  }
  // per-body centre of mass and the env's max point speed (solver.py:384-428), for the protocol
  for (int b = 0; b < E.nb; ++b) {
    const int kind = D.body_kind[E.b0 + b];
    double m = 0.0, cx = 0.0, cy = 0.0, cz = 0.0;
    if (kind == 0) {
      for (int n = threadIdx.x; n < E.nn; n += NT) {
        const size_t g = E.n0 + n;
        if (D.node_body[g] != b) continue;
        const double mn = D.node_M[9 * g];
        m += mn; cx += mn * D.x[3 * g]; cy += mn * D.x[3 * g + 1]; cz += mn * D.x[3 * g + 2];
      }
    } else if (kind == 2) {
      for (int i = threadIdx.x; i < E.ns; i += NT) {
        const size_t g = E.s0 + i;
        if (D.sv_body[g] != b) continue;
        m += 1.0; cx += D.kin_pos[3 * g]; cy += D.kin_pos[3 * g + 1]; cz += D.kin_pos[3 * g + 2];
      }
    }
    m = block_sum(m, sm); cx = block_sum(cx, sm); cy = block_sum(cy, sm); cz = block_sum(cz, sm);
    if (threadIdx.x == 0) {
      double* o = D.body_com + 3 * (size_t)(E.b0 + b);
      if (kind == 1) {
        for (int a = 0; a < E.na; ++a) {
          const int pn = D.abd_node[E.a0 + a];
          if (D.node_body[E.n0 + pn] == b)
            for (int c = 0; c < 3; ++c) o[c] = D.x[3 * (size_t)(E.n0 + pn) + c];
        }
      } else {
        o[0] = cx / m; o[1] = cy / m; o[2] = cz / m;
      }
    }
  }
  {
    double sp = 0.0;
    for (int n = threadIdx.x; n < E.nn; n += NT) {
      const size_t g = E.n0 + n;
      if (D.node_kind[g] == 0) sp = fmax(sp, norm(ld3(D.v + 3 * g)));
    }
    for (int i = threadIdx.x; i < E.ns; i += NT)
      if (D.sv_kind[E.s0 + i] == 1) sp = fmax(sp, norm(sv_dir(D, E, i, D.v)));
    for (int b = threadIdx.x; b < E.nb; b += NT)
      if (D.body_kind[E.b0 + b] == 2) sp = fmax(sp, norm(ld3(D.body_vel + 3 * (size_t)(E.b0 + b))));
    sp = block_max(sp, sm);
    if (threadIdx.x == 0) D.max_speed[e] = sp;
  }
  {   // inversion report: min J = det F = det(Ds) det(Dm^-1) over tets (materials.py:116-131), det A
      // over affine bodies (ccd.py:191-204's determinant)
    double mj = INFINITY;
    for (int k = threadIdx.x; k < E.ntet; k += NT) {
      const int t = E.te0 + k;
      const int* tn = D.tet_nodes + 4 * (size_t)t;
      const V3 x0 = ld3(D.x + 3 * (size_t)(E.n0 + tn[0]));
      const V3 a = ld3(D.x + 3 * (size_t)(E.n0 + tn[1])) - x0, b = ld3(D.x + 3 * (size_t)(E.n0 + tn[2])) - x0,
               c = ld3(D.x + 3 * (size_t)(E.n0 + tn[3])) - x0;
      const double* M = D.tet_Dmi + 9 * (size_t)t;
      const double dM = M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
                        M[2] * (M[3] * M[7] - M[4] * M[6]);
      mj = fmin(mj, dot(cross(a, b), c) * dM);
    }
    for (int k = threadIdx.x; k < E.na; k += NT) {
      const size_t pn = E.n0 + D.abd_node[E.a0 + k];
      const V3 r0 = ld3(D.x + 3 * (pn + 1)), r1 = ld3(D.x + 3 * (pn + 2)), r2 = ld3(D.x + 3 * (pn + 3));
      mj = fmin(mj, dot(cross(r0, r1), r2));
    }
    mj = block_min(mj, sm);
    if (threadIdx.x == 0) D.min_J[e] = mj;
  }
  // quarantine check (multienv.py:105-108)
  int nonfin = 0;
  for (int i = threadIdx.x; i < 3 * E.nn; i += NT) nonfin |= !isfinite(D.x[3 * (size_t)E.n0 + i]);
  nonfin = block_or(nonfin, sm);
  if (threadIdx.x < nbl) D.contact_mask[E.b0 + threadIdx.x] = cmask[threadIdx.x];
  if (threadIdx.x == 0) {
    D.fin_done[e] = 1;
    if (D.ev_on) D.ev_n[e] = base;
    if (!failed) D.n_anc[e] = base;
    D.min_dist[e] = (!failed && (npt + nee) > 0) ? sqrt(dmin) : INFINITY;
    D.time[e] += dt;
    D.step_index[e] += 1;
    if (nonfin && !failed) {
      D.ns_status[e] = GRIP_NS_FAILED;
      D.reason[e] = GRIP_R_NONFINITE_STATE;
    }
  }
}

// ---------------------------------------------------------------------------
// Device-resident grasp protocol (protocol.py:152-277), one thread per env, after k_finalize:
// the same decisions as BatchedGraspTrials._after_step, in the same order (close-phase halting
// before the failure check, phase ends, the verdict of the last gravity phase).
// ---------------------------------------------------------------------------
__constant__ double kGravDir[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};

__device__ void protocol_env(const Dev& D, int e);

__global__ void k_protocol(Dev D) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= D.n_env) return;
  protocol_env(D, e);
}

// One round boundary of the device protocol in one launch: finalize_step of the envs that finished
// the previous round's sweep, their protocol decision (thread 0), then begin_step of the envs the
// protocol asks to step (a cluster per env, as k_begin).  The decision inputs of begin (the
// protocol state, body velocities, supersets) are written by rank 0 before one cluster barrier.
__global__ void __cluster_dims__(BP_CL, 1, 1) __launch_bounds__(NT) k_bound(Dev D, const int* list) {
  __shared__ Red sm;
  __shared__ BPShared S;
  __shared__ unsigned int cmask[32];
  const BPCl cl{(int)cooperative_groups::this_cluster().block_rank(), BP_CL};
  const int e = list[blockIdx.x / BP_CL];
  CTA_TIMER_IF(cl.rank == 0, 5, e);
  if (cl.rank == 0) {
    finalize_env(D, e, 1, sm, S, cmask);
    __syncthreads();
    if (threadIdx.x == 0) protocol_env(D, e);
  }
  cl_sync(cl);
  if (!D.pr_i[(size_t)e * PI_N + PI_NEEDBEGIN]) return;
  begin_env(D, e, sm, S, cl);
  if (cl.rank != 0) return;
  __syncthreads();
  if (threadIdx.x == 0 && !(D.flags[e] & FLAG_OVERFLOW)) {   // an overflowed begin is redone later
    D.pr_i[(size_t)e * PI_N + PI_NEEDBEGIN] = 0;
    D.pr_i[(size_t)e * PI_N + PI_INSTEP] = 1;
  }
}

// finalize_step + the protocol decision of the envs that finished the round's sweep, one CTA per env
// (the device protocol's round end; the next round's begin_step is a cluster launch of its own)
__global__ void __launch_bounds__(NT) k_finalize_protocol(Dev D, const int* list) {
  __shared__ Red sm;
  __shared__ BPShared S;
  __shared__ unsigned int cmask[32];
  const int e = list[blockIdx.x];
  CTA_TIMER(4, e);
  finalize_env(D, e, 1, sm, S, cmask);
  __syncthreads();
  if (threadIdx.x == 0) protocol_env(D, e);
}

__device__ void protocol_env(const Dev& D, int e) {
  int* I = D.pr_i + (size_t)e * PI_N;
  double* R = D.pr_d + (size_t)e * PD_N;
  if (!I[PI_INSTEP] || !D.fin_done[e] || (D.flags[e] & FLAG_OVERFLOW)) return;
  I[PI_INSTEP] = 0;
  atomicAdd(D.pr_steps, 1ull);
  const double* C = D.pr_cfg;   // settle, hold, grav steps, speed, halt, g, steady, stability
  const int b0 = D.body_off[e];
  const double dt = D.params[(size_t)e * GRIP_NPARAM + GRIP_P_DT];
  const double eps_v = D.params[(size_t)e * GRIP_NPARAM + GRIP_P_EPSV];
  const int fb[2] = {I[PI_FB0], I[PI_FB1]};
  const int obj = I[PI_OBJ];
  I[PI_NSTEPS] += 1;
  I[PI_PSTEP] += 1;
  const int ph = I[PI_PHASE];
  if (ph == 1)
    for (int j = 0; j < 2; ++j) {
      const double f = D.body_force[b0 + fb[j]];
      if (!((I[PI_HALTED] >> j) & 1) && f > C[4]) {
        I[PI_HALTED] |= 1 << j;
        R[PD_HF + j] = f;
        I[PI_HSTEP0 + j] = I[PI_NSTEPS] - 1;
        for (int c = 0; c < 3; ++c) D.body_vel[3 * (size_t)(b0 + fb[j]) + c] = 0.0;
      }
    }
  const double* com = D.body_com + 3 * (size_t)(b0 + obj);
  auto disp = [&]() {
    const double dx = com[0] - R[PD_COM0], dy = com[1] - R[PD_COM0 + 1], dz = com[2] - R[PD_COM0 + 2];
    return sqrt(dx * dx + dy * dy + dz * dz);
  };
  if (D.ns_status[e] != GRIP_NS_FAILED) {   // a failed step keeps its pre-step state
    R[PD_MIND] = fmin(R[PD_MIND], D.min_dist[e]);
    R[PD_MINJ] = fmin(R[PD_MINJ], D.min_J[e]);
  }
  if (D.ns_status[e] == GRIP_NS_FAILED) {
    I[PI_VERDICT] = 3;
    I[PI_FPHASE] = ph == 3 ? 3 + I[PI_GPHASE] : ph;
    I[PI_FREASON] = D.reason[e];
    I[PI_FSTEP] = I[PI_NSTEPS];
    if (ph == 3) R[PD_CDISP + I[PI_GPHASE]] = disp();
    I[PI_PHASE] = 4;
    return;
  }
  bool ended = false;
  if (ph == 0) ended = I[PI_PSTEP] >= (int)C[0];
  else if (ph == 1) ended = I[PI_HALTED] == 3 || I[PI_PSTEP] >= I[PI_MAXCLOSE];
  else if (ph == 2) {
    I[PI_QUIET] = D.max_speed[e] < eps_v ? I[PI_QUIET] + 1 : 0;
    ended = I[PI_QUIET] >= (int)C[6] || I[PI_PSTEP] >= (int)C[1];
  } else if (ph == 3) ended = I[PI_PSTEP] >= (int)C[2];
  if (ended) {
    const int mk = ph == 3 ? 3 + I[PI_GPHASE] : ph;
    I[PI_MARK + 2 * mk] = I[PI_PSTART];
    I[PI_MARK + 2 * mk + 1] = I[PI_NSTEPS];
    I[PI_PSTART] = I[PI_NSTEPS];
    I[PI_PSTEP] = 0;
    double* gr = D.gravity + 3 * (size_t)e;
    if (ph == 0) {
      I[PI_PHASE] = 1;
      for (int j = 0; j < 2; ++j)
        for (int c = 0; c < 3; ++c) D.body_vel[3 * (size_t)(b0 + fb[j]) + c] = R[PD_CD + 3 * j + c] * C[3];
    } else if (ph == 1) {
      for (int j = 0; j < 2; ++j)
        for (int c = 0; c < 3; ++c) D.body_vel[3 * (size_t)(b0 + fb[j]) + c] = 0.0;
      I[PI_PHASE] = 2;
    } else if (ph == 2) {
      I[PI_PHASE] = 3;
      I[PI_GPHASE] = 0;
      for (int c = 0; c < 3; ++c) gr[c] = C[5] * kGravDir[0][c];
      for (int c = 0; c < 3; ++c) R[PD_COM0 + c] = com[c];
    } else {
      const int g = I[PI_GPHASE];
      const double d = disp();
      R[PD_CDISP + g] = d;
      I[PI_GPHASE] = g + 1;
      if (g + 1 >= 6) {
        I[PI_PHASE] = 4;
        const double thr = C[7] * (int)C[2] * eps_v * dt;
        const bool in_contact = (D.contact_mask[b0 + obj] & (unsigned)I[PI_GBITS]) != 0u;
        I[PI_VERDICT] = (in_contact && d < thr) ? 1 : 2;
        R[PD_FDISP] = d;
        R[PD_THR] = thr;
        I[PI_FCONTACT] = in_contact;
      } else {
        for (int c = 0; c < 3; ++c) gr[c] = C[5] * kGravDir[g + 1][c];
        for (int c = 0; c < 3; ++c) R[PD_COM0 + c] = com[c];
      }
    }
  }
  if (I[PI_PHASE] != 4) I[PI_NEEDBEGIN] = 1;
}

// protocol (re)start of n envs (grip_protocol_setup / grip_protocol_reset), thread per env:
// hd = closing dirs (PINIT_D per env), hi = {env, max_close, finger 0, finger 1, object, gripper
// bits} (-1: keep the current wiring).  Settle starts with the fingers still and gravity off
// (protocol.py:193-198).
__global__ void k_protocol_init(Dev D, int n, const double* hd, const int* hi) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int* q = hi + PINIT_I * k;
  const int e = q[0];
  int* I = D.pr_i + (size_t)e * PI_N;
  double* R = D.pr_d + (size_t)e * PD_N;
  const int fb0 = q[2] >= 0 ? q[2] : I[PI_FB0], fb1 = q[3] >= 0 ? q[3] : I[PI_FB1];
  const int obj = q[4] >= 0 ? q[4] : I[PI_OBJ], gb = q[5] >= 0 ? q[5] : I[PI_GBITS];
  for (int j = 0; j < PI_N; ++j) I[j] = 0;
  for (int j = 0; j < PD_N; ++j) R[j] = 0.0;
  I[PI_FB0] = fb0; I[PI_FB1] = fb1; I[PI_OBJ] = obj; I[PI_GBITS] = gb;
  I[PI_MAXCLOSE] = q[1];
  I[PI_NEEDBEGIN] = 1;
  for (int j = 0; j < 18; ++j) I[PI_MARK + j] = -1;
  I[PI_HSTEP0] = I[PI_HSTEP1] = -1;
  for (int j = 0; j < 6; ++j) R[PD_CD + j] = hd[PINIT_D * k + j];
  R[PD_MIND] = R[PD_MINJ] = INFINITY;
  const int b0 = D.body_off[e];
  for (int c = 0; c < 3; ++c) {
    D.body_vel[3 * (size_t)(b0 + fb0) + c] = 0.0;
    D.body_vel[3 * (size_t)(b0 + fb1) + c] = 0.0;
    D.gravity[3 * (size_t)e + c] = 0.0;
  }
}

// packed recorder frame of the envs with m[4e] >= 0 (grip_get_frames): CTA per env
__global__ void k_frames(Dev D, const int* m, double* fx, double* fv, double* fk, double* fs) {
  const int e = blockIdx.x;
  const int on = m[4 * e], os = m[4 * e + 1], ot = m[4 * e + 2];
  if (on < 0) return;
  const int n0 = D.node_off[e], nn = D.node_off[e + 1] - n0;
  const int s0 = D.sv_off[e], ns = D.sv_off[e + 1] - s0;
  const int t0 = D.tet_off[e], nt = D.tet_off[e + 1] - t0;
  for (int i = threadIdx.x; i < 3 * nn; i += blockDim.x) {
    fx[3 * (size_t)on + i] = D.x[3 * (size_t)n0 + i];
    fv[3 * (size_t)on + i] = D.v[3 * (size_t)n0 + i];
  }
  for (int i = threadIdx.x; i < 3 * ns; i += blockDim.x) fk[3 * (size_t)os + i] = D.kin_pos[3 * (size_t)s0 + i];
  for (int k = threadIdx.x; k < nt; k += blockDim.x) {
    const int t = t0 + k;
    V3 x[4];
    for (int j = 0; j < 4; ++j) x[j] = ld3(D.x + 3 * (size_t)(n0 + D.tet_nodes[4 * (size_t)t + j]));
    double row[7];
    if (!nh_stress(x, D.tet_Dmi + 9 * (size_t)t, D.tet_mu[t], D.tet_lam[t], row))
      for (int c = 0; c < 7; ++c) row[c] = NAN;
    for (int c = 0; c < 7; ++c) fs[7 * ((size_t)ot + k) + c] = row[c];
  }
}

// Slot refill (grip_reset_envs): CTA per refilled env.  The env gets the new candidate's pose,
// rest shape and materials from the staged slice and EVERY piece of per-env state a fresh
// grip_create starts from (zeros, identity Jacobi warm starts), so a refilled trial is bitwise a
// fresh trial.  Staged slice per env (doubles): x0 (3 nn) | M (9 nn) | kin0 (3 ns) | xi (3 ns) |
// Dmi (9 nt) | V0 | mu | lam (nt each) | body mu (nb) | edge rest len^2 (ne) | kappa V (na) | cell hint
// (pose-dependent rounding: lumped masses and rest lengths of posed pads differ in the last bits)
__global__ void k_reset_envs(Dev D, const int* lst, const long long* off, const double* stage) {
  const int e = lst[blockIdx.x];
  const double* s = stage + off[blockIdx.x];
  const int n0 = D.node_off[e], nn = D.node_off[e + 1] - n0;
  const int s0 = D.sv_off[e], ns = D.sv_off[e + 1] - s0;
  const int t0 = D.tet_off[e], nt = D.tet_off[e + 1] - t0;
  const int b0 = D.body_off[e], nb = D.body_off[e + 1] - b0;
  const int e0 = D.edge_off[e], ne = D.edge_off[e + 1] - e0;
  const int a0 = D.abd_off[e], na = D.abd_off[e + 1] - a0;
  auto put = [&](const double* dst_c, size_t first, int cnt) {
    double* dst = const_cast<double*>(dst_c) + first;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) dst[i] = s[i];
    s += cnt;
  };
  put(D.x, 3 * (size_t)n0, 3 * nn);
  put(D.node_M, 9 * (size_t)n0, 9 * nn);
  put(D.kin_pos, 3 * (size_t)s0, 3 * ns);
  put(D.sv_xi, 3 * (size_t)s0, 3 * ns);
  put(D.tet_Dmi, 9 * (size_t)t0, 9 * nt);
  put(D.tet_V0, t0, nt);
  put(D.tet_mu, t0, nt);
  put(D.tet_lam, t0, nt);
  put(D.body_mu, b0, nb);
  put(D.edge_rest_sq, e0, ne);
  put(D.abd_kV, a0, na);
  put(D.cell_hint, e, 1);
  for (int i = threadIdx.x; i < 3 * nn; i += blockDim.x) {
    const size_t g = 3 * (size_t)n0 + i;
    D.v[g] = D.x_t[g] = D.xhat[g] = D.pdir[g] = 0.0;
  }
  for (int i = threadIdx.x; i < 3 * ns; i += blockDim.x) {
    const size_t g = 3 * (size_t)s0 + i;
    D.sv_pos[g] = D.surf_prev[g] = D.sv_disp[g] = 0.0;
  }
  for (int i = threadIdx.x; i < 81 * nt; i += blockDim.x)   // Jacobi warm start: identity, in half 0
    D.tet_eig[81 * (size_t)t0 + i] = (i % 81) % 10 == 0 ? 1.0 : 0.0;
  if (threadIdx.x == 0) {
    D.eig_par[e] = 0;
    D.eig_swept[e] = 0;
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    D.body_force[b0 + i] = 0.0;
    D.contact_mask[b0 + i] = 0u;
    for (int c = 0; c < 3; ++c) D.body_com[3 * (size_t)(b0 + i) + c] = 0.0;
  }
  for (int i = threadIdx.x; i < D.max_alpha; i += blockDim.x) D.alphas[(size_t)e * D.max_alpha + i] = 0.0;
  if (threadIdx.x == 0) {
    D.ell[e] = D.tol[e] = D.residual[e] = D.energy[e] = D.min_dist[e] = D.time[e] = 0.0;
    D.max_speed[e] = D.cs_R[e] = D.cs_drift[e] = D.md_prev[e] = D.md_kin[e] = 0.0;
    D.iters[e] = D.ns_status[e] = D.reason[e] = D.regularized[e] = D.kin_blocked[e] = D.needs_ls[e] = 0;
    D.ns_done[e] = D.flags[e] = D.step_index[e] = D.newton_calls[e] = D.pcg_iters[e] = D.fin_done[e] = 0;
    D.cs_valid[e] = D.n_act[e] = D.n_anc[e] = D.ev_n[e] = 0;
    for (int c = 0; c < 2; ++c) D.cs_n[2 * e + c] = D.c1_n[2 * e + c] = D.c2_n[2 * e + c] = 0;
  }
}

// per-tet stress rows (materials.py:191-205), flat over all tets
__global__ void k_stress(Dev D, int n_tet_total, const int* tet_env, double* out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tet_total; t += gridDim.x * blockDim.x) {
    const int e = tet_env[t];
    const int n0 = D.node_off[e];
    V3 x[4];
    for (int j = 0; j < 4; ++j) x[j] = ld3(D.x + 3 * (size_t)(n0 + D.tet_nodes[4 * (size_t)t + j]));
    double row[7];
    if (!nh_stress(x, D.tet_Dmi + 9 * (size_t)t, D.tet_mu[t], D.tet_lam[t], row))
      for (int c = 0; c < 7; ++c) row[c] = NAN;
    for (int c = 0; c < 7; ++c) out[7 * (size_t)t + c] = row[c];
  }
}

// surface positions of every env (state readout)
__global__ void k_surface_all(Dev D, const int* list) {
  const int e = list[blockIdx.x];
  const EnvIx E = env_ix(D, e);
  for (int i = threadIdx.x; i < E.ns; i += blockDim.x) st3(D.sv_pos + 3 * (size_t)(E.s0 + i), sv_at(D, E, i, D.x));
}

// candidate query on current positions
__global__ void __launch_bounds__(NT) k_query(Dev D, const int* list, double r) {
  __shared__ Red sm;
  __shared__ BPShared S;
  const int e = list[blockIdx.x];
  const EnvIx E = env_ix(D, e);
  env_sv_positions(D, E, D.x);
  if (!broad_phase_env(D, E, r, D.c2_pt + (size_t)e * 4 * D.cap_pt, D.c2_ee + (size_t)e * 4 * D.cap_ee,
                       D.c2_eid + (size_t)e * 2 * D.cap_ee, D.c2_n + 2 * e, S, sm)) {
    if (threadIdx.x == 0) D.flags[e] |= FLAG_OVERFLOW;
  }
}

// Contact readout at the CURRENT state, no step taken (protocol.py:72-75 contact_events_now,
// solver.py:449-453 min_contact_distance, contact.py:348-372 stencil_forces): the canonical
// candidate set at radius r (the c2 buffers, as k_query), the min distance over all of its
// stencils, and every active stencil (d < dhat) as an event row in the ev_* buffers with
// lambda = kappa m |b'(d)|; per-body force sums and the body contact bits as k_finalize makes
// them.  v, anchors, time and the step's min_dist are untouched.
__global__ void __launch_bounds__(NT) k_contacts_now(Dev D, const int* list, double radius_factor, double* md_out) {
  __shared__ Red sm;
  __shared__ BPShared S;
  __shared__ unsigned int cmask[32];
  const int e = list[blockIdx.x];
  const EnvIx E = env_ix(D, e);
  const double* P = P_(D, e);
  const double kappa = P[GRIP_P_KAPPA], dhat = P[GRIP_P_DHAT];
  env_sv_positions(D, E, D.x);
  int* cn = D.c2_n + 2 * e;
  int* cpt = D.c2_pt + (size_t)e * 4 * D.cap_pt;
  int* cee = D.c2_ee + (size_t)e * 4 * D.cap_ee;
  int* ceid = D.c2_eid + (size_t)e * 2 * D.cap_ee;
  if (!broad_phase_env(D, E, radius_factor * dhat, cpt, cee, ceid, cn, S, sm)) {
    if (threadIdx.x == 0) D.flags[e] |= FLAG_OVERFLOW;
    return;
  }
  const int npt = cn[0], nee = cn[1];
  const double* X = D.sv_pos + 3 * (size_t)E.s0;
  if (threadIdx.x < 32) cmask[threadIdx.x] = 0u;
  __syncthreads();
  double dmin = INFINITY;
  int base = 0;
  double fsum[32];
  const int nbl = min(E.nb, 32);
  for (int b = 0; b < nbl; ++b) fsum[b] = 0.0;
  for (int s = 0; s < npt + nee; s += NT) {
    const int k = s + threadIdx.x;
    int act = 0, rowv[4], bb[2];
    double lam = 0.0, Dq = 0.0;
    if (k < npt + nee) {
      const bool is_ee = k >= npt;
      const int* row = is_ee ? cee + 4 * (k - npt) : cpt + 4 * k;
      V3 x[4];
      for (int j = 0; j < 4; ++j) {
        rowv[j] = row[j];
        x[j] = ld3(X + 3 * row[j]);
      }
      double bary[3], sp = 0.0, tp = 0.0;
      Dq = is_ee ? ee_closest(x[0], x[1], x[2], x[3], &sp, &tp) : pt_closest(x[0], x[1], x[2], x[3], bary, nullptr);
      dmin = fmin(dmin, Dq);
      if (Dq < dhat * dhat) {
        act = 1;
        double b0, b1, b2;
        barrier_d(sqrt(Dq), dhat, &b0, &b1, &b2);
        double m = 1.0;
        if (is_ee) {
          double dm, d2m;
          const int* eid = ceid + 2 * (k - npt);
          edge_mollifier(cross_norm_sq(x, nullptr, nullptr), D.edge_rest_sq[E.ed0 + eid[0]] * D.edge_rest_sq[E.ed0 + eid[1]],
                         &m, &dm, &d2m);
        }
        lam = kappa * m * fabs(b1);
        bb[0] = D.sv_body[E.s0 + row[0]];
        bb[1] = D.sv_body[E.s0 + row[is_ee ? 2 : 1]];
        for (int b = 0; b < nbl; ++b)
          if (bb[0] == b || bb[1] == b) fsum[b] += lam;
        if (bb[0] < 32 && bb[1] < 32) {
          atomicOr(&cmask[bb[0]], 1u << bb[1]);
          atomicOr(&cmask[bb[1]], 1u << bb[0]);
        }
      }
    }
    int tot;
    const int pre = block_scan(act, sm, &tot);
    if (act && base + pre < D.cap_anc) {
      const size_t vi = (size_t)e * D.cap_anc + base + pre;
      int* ei = D.ev_i + 7 * vi;
      ei[0] = k >= npt;
      ei[1] = bb[0];
      ei[2] = bb[1];
      for (int j = 0; j < 4; ++j) ei[3 + j] = rowv[j];
      D.ev_d[2 * vi] = sqrt(Dq);
      D.ev_d[2 * vi + 1] = lam;
    }
    base += tot;
  }
  if (base > D.cap_anc) {   // more active stencils than event rows: grow and redo
    if (threadIdx.x == 0) {
      D.flags[e] |= FLAG_OVERFLOW;
      atomicMax(&D.need[3], (unsigned)base);
    }
    return;
  }
  dmin = block_min(dmin, sm);
  for (int b = 0; b < nbl; ++b) {
    const double f = block_sum(fsum[b], sm);
    if (threadIdx.x == 0) D.body_force[E.b0 + b] = f;
  }
  if (threadIdx.x < nbl) D.contact_mask[E.b0 + threadIdx.x] = cmask[threadIdx.x];
  if (threadIdx.x == 0) {
    D.ev_n[e] = base;
    md_out[e] = (npt + nee) > 0 ? sqrt(dmin) : INFINITY;
  }
}

// quarantine test of Batch.quarantine_failures (multienv.py:98-123): 1 per env whose x holds a
// non-finite value, CTA per env (no state copy to the host)
__global__ void __launch_bounds__(NT) k_check_finite(Dev D, int* out) {
  __shared__ Red sm;
  const int e = blockIdx.x;
  const size_t a = 3 * (size_t)D.node_off[e], b = 3 * (size_t)D.node_off[e + 1];
  int bad = 0;
  for (size_t i = a + threadIdx.x; i < b; i += NT) bad |= !isfinite(D.x[i]);
  bad = block_or(bad, sm);
  if (threadIdx.x == 0) out[e] = bad;
}

}  // namespace grip
