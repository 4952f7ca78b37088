// Device-side context, CTA-wide reductions/scans and the per-environment
// broad phase.  One CTA owns one environment in every *_env kernel, so all
// per-env reductions are block reductions with a fixed tree: results are
// bitwise reproducible and independent of how many envs share the launch
// (SPEC "batch-of-N bitwise equals batch-of-1").
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/grip_ipc.h"
#include "grip_elements.cuh"

namespace grip {

// Tet Hessians are stored as their packed lower triangle (78 of the slot's 144 doubles): the
// symmetric 12x12 written and read once instead of twice (k_static is the only reader).
__host__ __device__ constexpr int tri12(int r, int c) { return r * (r + 1) / 2 + c; }   // c <= r

#ifdef GRIP_PHASE_TIMING
__device__ unsigned long long g_phase[64];   // diagnostic counters (grip_debug_phase)
#define GSTAT(k, v) atomicAdd(&g_phase[k], (unsigned long long)(v))
#else
#define GSTAT(k, v) do {} while (0)
#endif


#ifndef GRIP_NT
#define GRIP_NT 256
#endif
constexpr int NT = GRIP_NT;       // threads per env CTA (256; GRIP_NT=512 builds are an A/B experiment)
constexpr int NWARP = NT / 32;
#ifndef GRIP_MINB
#define GRIP_MINB 3
#endif
constexpr int NT_MINB3 = NT == 256 ? GRIP_MINB : 1;   // CTAs per SM the heavy CTA-per-env kernels are built for
constexpr int MAXC = 4096;        // broad-phase grid cells per env

// error / flag bits per env and Newton sweep
enum { ERR_INVERTED = 1, ERR_CONTACT_D = 2, FLAG_OVERFLOW = 4, FLAG_OVF_BEGIN = 8, FLAG_OVF_FIN = 16 };  // OVF_*: stage

// device protocol state layout (per env)
enum {
  PI_PHASE = 0, PI_PSTEP, PI_GPHASE, PI_QUIET, PI_NSTEPS, PI_PSTART, PI_HALTED, PI_MAXCLOSE, PI_INSTEP,
  PI_NEEDBEGIN, PI_VERDICT, PI_FPHASE, PI_FREASON, PI_FSTEP, PI_FCONTACT, PI_FB0, PI_FB1, PI_OBJ, PI_GBITS,
  PI_HSTEP0, PI_HSTEP1, PI_MARK, PI_N = PI_MARK + 18
};
// PD_MIND / PD_MINJ: min stencil distance / min element J = det F (tets) or det A (affine bodies)
// over the trial's completed steps (the north star's intersection / inversion report)
enum { PINIT_D = 6, PINIT_I = 6 };   // k_protocol_init staging per env: closing dirs | ints
// k_reset_envs staged doubles per node (x0, M), surface vertex (kin0, xi), tet (Dmi, V0, mu, lam)
enum { RESET_PER_NODE = 12, RESET_PER_SV = 6, RESET_PER_TET = 12 };   // k_protocol_init staging per env: closing dirs | ints
enum { PD_CD = 0, PD_COM0 = 6, PD_HF = 9, PD_CDISP = 11, PD_FDISP = 17, PD_THR = 18, PD_MIND = 19, PD_MINJ = 20, PD_N = 21 };

struct Dev {
  int n_env;
  // env slices
  const int *node_off, *sv_off, *tri_off, *edge_off, *tet_off, *abd_off, *body_off, *free_off;
  // scene
  const double* node_M;
  const uint8_t* node_free;
  const int* node_body;
  const uint8_t* node_kind;
  const int* node_sv;
  const int* node_fidx;      // local free index or -1
  const int* free_node;      // per global free idx: local node
  const int* dense_perm;     // per global free idx: position in the env's dense system (hub bodies last)
  const int* dense_fc;       // per env-dense position (global free offset): lowest statically coupled position
  const int* dense_tail;     // per env: first dense position of the hub (last) body
  const int* sb_row;         // per block: global free row
  const int* sb_dst;         // per block: dense (row, col) node positions << 16 | ..., -1 above the diagonal
  double* tet_S;             // per tet 45: warm-rotated S~ (upper) awaiting the batched eigensolve
  double* tet_W;             // per tet 90: its eigenvalues (9) and rotation R (81, row-major)
  int2* jac_list;            // (tet, element slot) of the tets whose clamp was deferred this sweep
  int* jac_n;
  double* cjac_S;            // contacts (cold clamps), per active slot env*cap_act + k: S (45)
  double* cjac_W;            // ... eigenvalues + eigenvectors (90)
  int2* cjac_list;           // (active slot, element slot)
  int* cjac_n;
  const int* sv_code;        // per surface vertex: dense node position << 2 | kind (0 soft, 1 affine), -1 none
  const uint8_t* sv_kind;
  const int* sv_node;
  const double* sv_xi;
  const int* sv_body;
  const int* tris;
  const int* edges;
  const double* edge_rest_sq;
  const int* tet_nodes;
  const double* tet_Dmi;
  const double* tet_V0;
  const double* tet_mu;
  const double* tet_lam;
  double* tet_eig;           // per tet 9x9: eigenvectors of its deflated Hessian (Jacobi warm start),
                             // two halves of eig_half doubles: env e reads half eig_par[e], its
                             // deferred tets' next bases go to the other half (tet_eig_cur / _next)
  size_t eig_half;
  int* eig_par;              // per env: the half holding its current warm starts
  int* eig_swept;            // per env: its tets went through this sweep (k_tet_scan; k_linesearch commits)
  const int* abd_node;
  const double* abd_kV;
  const uint8_t* body_kind;
  const double* body_mu;
  const uint32_t* body_pairmask;
  const int *body_tri_lo, *body_tri_hi, *body_edge_lo, *body_edge_hi;
  double* body_vel;
  double* gravity;
  const double* params;
  const double* cell_hint;
  // static block structure over free nodes (global free index rows)
  const int* sb_rowptr;      // [n_free_total + 1] global block ids
  const int* sb_col;         // local free col
  const int* sb_diag;        // per global free idx
  const int* sbc_ptr;        // [n_blocks + 1]
  const int* sbc;            // contribution code: (elem_slot << 4) | (sa << 2) | sb ; elem_slot local el index
  const int* tinc_ptr;       // per global node: tet/abd gradient incidence
  const int* tinc;           // (elem_slot << 2) | slot
  // state
  double *x, *v, *x_t, *xhat, *pdir;
  double *sv_pos, *surf_prev, *kin_pos, *sv_disp;
  double *ell, *tol, *residual, *energy, *alphas, *min_dist, *time;
  int *iters, *ns_status, *reason, *regularized, *kin_blocked, *needs_ls, *ns_done, *flags, *step_index;
  int *newton_calls, *pcg_iters;
  int* fin_done;       // finalize ran for the current step (round API)
  double* body_force;
  unsigned int* contact_mask;
  double* body_com;    // 3 per body, after finalize
  double* max_speed;   // per env, after finalize (solver.py:414-428)
  double* min_J;       // per env, after finalize: min det F over its tets and det A over its affine bodies
  double* stats;       // [0..3] element counts of the last sweep (tets, abd, contacts, anchors)
  int max_alpha;
  // candidates (uniform capacity per env)
  int cap_pt, cap_ee;
  unsigned* cand_done;   // k_candidates: env CTAs finished (the last one scans the contact work)
  unsigned* need;    // 4: the largest pt / ee / active / anchor count that overflowed its capacity (growth sizes)
  int *c1_pt, *c1_ee, *c1_eid, *c1_n;   // c1_n[2e]=n_pt, [2e+1]=n_ee
  int *c2_pt, *c2_ee, *c2_eid, *c2_n;
  // candidate superset at radius cs_R >= every radius needed before x changes; exact sets are
  // order-preserving filters of it with the reference predicate (identical membership)
  int *cs_pt, *cs_ee, *cs_eid, *cs_n;
  double* cs_R;
  int* cs_valid;
  double* cs_drift;  // summed max surface displacement since the superset was built (Verlet skin)
  double ss_skin;    // extra radius (units of dhat) a superset is built with, GRIP_SKIN
  double ss_k;        // superset covers dhat + ss_k * (last Newton step's max displacement)
  double* md_prev;   // last Newton step's max surface displacement
  double* md_kin;    // this step's prescribed (kinematic) displacement bound
  // elements (uniform capacity per env): [tets | abd | contacts | anchors]
  int max_tet, max_abd, cap_act, cap_anc, cap_el;
  int* act;          // per env cap_act: candidate code (ee ? cap_pt + k : k)
  int* n_act;
  int* n_anc;
  double *el_E, *el_g, *el_H;
  int* el_idx;
  int* tflag;        // per env: ERR_INVERTED from k_tet_front this sweep (its own word: the tet chain runs
                     // on the second stream, concurrently with k_candidates writing flags)
  int* work_off;     // per list position (n+1)
  int* cwork_off;    // per list position (n+1): contact / friction elements only
  int* asm_key;      // per list position: contact / friction elements (the work scan)
  int* asm_order;    // the list's envs by descending contact work: the assembly and line search
                     // launch their heavy envs first (a launch lasts as long as its heaviest CTA)
  int* twork_off;    // per list position (n+1): tets only (k_tet_front)
  int* swork_off;    // per list position (n+1): static 3x3 blocks of H_ff (k_static)
  // anchors (persist across steps)
  int* anc_v;        // 4
  double *anc_gamma, *anc_T, *anc_lam, *anc_mu;   // 4, 6, 1, 1
  int* anc_b;        // 2
  // contact events of the last finalize (protocol.py:72-75 contact_events_now; recorded when ev_on):
  // per env cap_anc slots, active stencils in candidate order (PT then EE)
  // device-resident protocol (k_protocol, grip_run_rounds): per env PI_N ints, PD_N doubles
  int round_mode;
  int* pr_i;
  double* pr_d;
  double* pr_cfg;          // 8 (grip_protocol_setup)
  unsigned long long* pr_steps;  // env-steps completed (counter)
  int ev_on;
  int* ev_i;         // 7 per event: kind (0 PT, 1 EE), body a, body b, 4 vertices
  double* ev_d;      // 2 per event: d, lambda
  int* ev_n;         // per env: event count (may exceed cap_anc: truncated)
  // scratch
  int max_sv, max_tri, max_edge, max_free, max_node;
  int cap_cells;
  int bp_qm_min;     // direct broad phase: groups with > bp_qm_min lane-mode iterations use query mode
  float bp_qm_fac;   //   when that costs <= bp_qm_fac x the lane-mode iterations (GRIP_BP_QM=min,fac)
  int bp_mode;       // broad phase: 0 direct over culled primitives with grid fallback, 1 grid only (GRIP_BP)
  int* bp_cells;     // per env cap_cells (grid path)
  int* bp_scr;       // per env 4 max(max_tri, max_edge) + max_sv (direct path: compacted ids, vertices, queries)
  double* bp_aabb;   // per env 6*max(max_tri, max_edge)
  int* bp_cnt;       // per env max(max_sv, max_edge) + 1
  int* bp_tmp;       // per env max(cap_pt, cap_ee)
  int* bp_lc;        // per env 3*max(max_tri, max_edge): lowest grid cell of each primitive
  double *pcg_x, *pcg_r, *pcg_z, *pcg_p, *pcg_q, *pcg_b;  // per env 3*max_free
  double* pcg_pinv;  // per global free node 9
  double* abd_pinv;  // per abd 144
  double* sb_val;    // per block 9
  double* dense_L;   // per env dense_stride doubles (direct solve when the matrix exceeds shared memory)
  size_t dense_stride;
  double *c_u, *c_w; // per env 3*max_sv
  double* ls_y;       // per env LS_NA*3*max_sv: trial surface positions of the line search's energy passes
  double* c_r;       // per env 12*(cap_act+cap_anc)
  int *inc_ptr, *inc; // per env max_sv+1 ; 4*(cap_act+cap_anc)
  double* el_K;       // direct solve, per contact slot (env (cap_act+cap_anc)): dt^2 J^T H J, lower triangle over
                      // the element's DOFs in dense order (<= 24 DOFs -> 300 entries)
  int* el_kn;         // per contact slot 9: node count, then the element's dense node positions (ascending)
  int* sc_lst;        // direct solve scratch, per env 8*(cap_act+cap_anc): contact (element, node slot) items by node
  int* sc_off;        // ... per env 2*(max_free+1): per dense node item offsets, fill cursors
  int dense_k;        // 1: the element kernel writes el_K / el_kn (direct solver)
  double* sv_g;      // per env 3*max_sv
  unsigned long long launch_seq;   // host launch counter, captured by value at every launch
  unsigned long long* cta_rec;     // GRIP_CTA_TIMING builds: 4 per CTA (seq, kernel << 32 | env, smid, t0 << 32 | t1)
  unsigned int* cta_n;
  unsigned int cta_cap;
};

// per-CTA wall time (GRIP_CTA_TIMING builds only; the per-env CTA histograms of profiles/):
// thread 0 stamps %globaltimer at entry and, through the destructor, at every exit
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct CtaTimer {
  const Dev& D;
  int kid, env;
  bool on;
  unsigned info = 0;   // kernel-specific detail bits (CTA_INFO), stored above the SM id
  unsigned long long t0;
  __device__ CtaTimer(const Dev& d, int k, int e, bool o = true)
      : D(d), kid(k), env(e), on(o), t0(threadIdx.x == 0 ? gtimer() : 0ull) {}
  __device__ ~CtaTimer() {
    if (!on || threadIdx.x != 0 || !D.cta_rec) return;
    const unsigned long long t1 = gtimer();
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    const unsigned i = atomicAdd(D.cta_n, 1u);
    if (i >= D.cta_cap) return;
    unsigned long long* r = D.cta_rec + 4 * (size_t)i;
    r[0] = D.launch_seq;
    r[1] = ((unsigned long long)kid << 32) | (unsigned)env;
    r[2] = sm | ((unsigned long long)info << 16);
    r[3] = ((t0 & 0xffffffffull) << 32) | (t1 - t0 > 0xffffffffull ? 0xffffffffull : t1 - t0);
  }
};
#ifdef GRIP_CTA_TIMING
#define CTA_TIMER(kid, e) CtaTimer cta_timer_(D, kid, e)
#define CTA_TIMER_IF(on, kid, e) CtaTimer cta_timer_(D, kid, e, on)
#define CTA_INFO(v) (cta_timer_.info |= (v))
#define CTA_INFO_ADD(v) (cta_timer_.info += (v))
#else
#define CTA_INFO(v) do {} while (0)
#define CTA_INFO_ADD(v) do {} while (0)
#define CTA_TIMER(kid, e) do {} while (0)
#define CTA_TIMER_IF(on, kid, e) do {} while (0)
#endif

__device__ __forceinline__ const double* P_(const Dev& D, int e) { return D.params + (size_t)e * GRIP_NPARAM; }

// the warm-start halves of env e (see Dev::tet_eig)
__device__ __forceinline__ double* tet_eig_cur(const Dev& D, int e, size_t t) {
  return D.tet_eig + (D.eig_par[e] ? D.eig_half : 0) + 81 * t;
}
__device__ __forceinline__ double* tet_eig_next(const Dev& D, int e, size_t t) {
  return D.tet_eig + (D.eig_par[e] ? 0 : D.eig_half) + 81 * t;
}

// At the end of an env's line search (the sweep's last kernel that can flag an overflow): a swept
// env without overflow makes its new warm starts current; an overflowed env's sweep is redone from
// the same bases (results independent of when buffers grew).
struct EigCommit {
  const Dev& D;
  int e;
  bool on;
  __device__ EigCommit(const Dev& d, int env, bool o) : D(d), e(env), on(o) {}
  __device__ ~EigCommit() {
    if (!on || threadIdx.x != 0 || !D.eig_swept[e]) return;
    if (!(D.flags[e] & FLAG_OVERFLOW)) D.eig_par[e] ^= 1;
    D.eig_swept[e] = 0;
  }
};

// ---------------------------------------------------------------------------
// block reductions (fixed shuffle tree -> deterministic)
// ---------------------------------------------------------------------------
struct Red {
  double d[4 * NWARP + 8];   // block_sum_n: 4 values per warp, then its results; block_red: [0, NWARP), [32]
  int i[40];
};

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double wmax(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double wmin(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int OP>  // 0 sum 1 max 2 min
__device__ double block_red(double v, Red& sm) {
  v = OP == 0 ? wsum(v) : (OP == 1 ? wmax(v) : wmin(v));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm.d[w] = v;
  __syncthreads();
  if (w == 0) {
    double r = l < NWARP ? sm.d[l] : (OP == 0 ? 0.0 : (OP == 1 ? -INFINITY : INFINITY));
    r = OP == 0 ? wsum(r) : (OP == 1 ? wmax(r) : wmin(r));
    if (l == 0) sm.d[32] = r;
  }
  __syncthreads();
  return sm.d[32];
}
// N <= 4 block sums at once, each through exactly block_red<0>'s tree (bitwise the same values)
template <int N>
__device__ void block_sum_n(double* v, Red& sm) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = wsum(v[k]);
  __syncthreads();
  if (l == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) sm.d[4 * w + k] = v[k];
  __syncthreads();
  if (w == 0)
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double r = l < NWARP ? sm.d[4 * l + k] : 0.0;
      r = wsum(r);
      if (l == 0) sm.d[4 * NWARP + k] = r;
    }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) v[k] = sm.d[4 * NWARP + k];
  __syncthreads();
}
__device__ __forceinline__ double block_sum(double v, Red& sm) { return block_red<0>(v, sm); }
__device__ __forceinline__ double block_max(double v, Red& sm) { return block_red<1>(v, sm); }
__device__ __forceinline__ double block_min(double v, Red& sm) { return block_red<2>(v, sm); }

__device__ int block_or(int v, Red& sm) {
  v = __reduce_or_sync(0xffffffffu, (unsigned)v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm.i[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int r = 0;
    for (int k = 0; k < NWARP; ++k) r |= sm.i[k];
    sm.i[32] = r;
  }
  __syncthreads();
  return sm.i[32];
}

// exclusive scan of one int per thread; returns prefix, writes block total to *total
__device__ int block_scan(int v, Red& sm, int* total) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  int inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (l >= o) inc += t;
  }
  __syncthreads();
  if (l == 31) sm.i[w] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int k = 0; k < NWARP; ++k) {
      int t = sm.i[k];
      sm.i[k] = run;
      run += t;
    }
    sm.i[32] = run;
  }
  __syncthreads();
  *total = sm.i[32];
  return sm.i[w] + inc - v;
}

// in-place exclusive scan of cnt[0..n) (global or shared), returns total
__device__ int block_scan_array(int* cnt, int n, Red& sm) {
  int base = 0;
  for (int s = 0; s < n; s += NT) {
    int i = s + threadIdx.x;
    int v = i < n ? cnt[i] : 0;
    int tot;
    int pre = block_scan(v, sm, &tot);
    if (i < n) cnt[i] = base + pre;
    base += tot;
  }
  __syncthreads();
  return base;
}

// ---------------------------------------------------------------------------
// state access
// ---------------------------------------------------------------------------
struct EnvIx {
  int e, n0, nn, s0, ns, t0, nt, ed0, ne, te0, ntet, a0, na, b0, nb, f0, nf;
};
__device__ __forceinline__ EnvIx env_ix(const Dev& D, int e) {
  EnvIx r;
  r.e = e;
  r.n0 = D.node_off[e]; r.nn = D.node_off[e + 1] - r.n0;
  r.s0 = D.sv_off[e]; r.ns = D.sv_off[e + 1] - r.s0;
  r.t0 = D.tri_off[e]; r.nt = D.tri_off[e + 1] - r.t0;
  r.ed0 = D.edge_off[e]; r.ne = D.edge_off[e + 1] - r.ed0;
  r.te0 = D.tet_off[e]; r.ntet = D.tet_off[e + 1] - r.te0;
  r.a0 = D.abd_off[e]; r.na = D.abd_off[e + 1] - r.a0;
  r.b0 = D.body_off[e]; r.nb = D.body_off[e + 1] - r.b0;
  r.f0 = D.free_off[e]; r.nf = D.free_off[e + 1] - r.f0;
  return r;
}

// surface position of env-local sv i from node array xs (global base), G x (solver.py:367-372)
__device__ __forceinline__ V3 sv_at(const Dev& D, const EnvIx& E, int i, const double* xs) {
  const int g = E.s0 + i;
  const int k = D.sv_kind[g];
  if (k == 0) return ld3(xs + 3 * (E.n0 + D.sv_node[g]));
  if (k == 1) {
    const double* q = xs + 3 * (E.n0 + D.sv_node[g]);
    V3 xi = ld3(D.sv_xi + 3 * g);
    return V3{q[0] + xi.x * q[3] + xi.y * q[4] + xi.z * q[5], q[1] + xi.x * q[6] + xi.y * q[7] + xi.z * q[8],
              q[2] + xi.x * q[9] + xi.y * q[10] + xi.z * q[11]};
  }
  return ld3(D.kin_pos + 3 * g);
}
// G applied to a node-space direction (kinematic rows are zero)
__device__ __forceinline__ V3 sv_dir(const Dev& D, const EnvIx& E, int i, const double* ps) {
  const int g = E.s0 + i;
  const int k = D.sv_kind[g];
  if (k == 0) return ld3(ps + 3 * (E.n0 + D.sv_node[g]));
  if (k == 1) {
    const double* q = ps + 3 * (E.n0 + D.sv_node[g]);
    V3 xi = ld3(D.sv_xi + 3 * g);
    return V3{q[0] + xi.x * q[3] + xi.y * q[4] + xi.z * q[5], q[1] + xi.x * q[6] + xi.y * q[7] + xi.z * q[8],
              q[2] + xi.x * q[9] + xi.y * q[10] + xi.z * q[11]};
  }
  return V3{0.0, 0.0, 0.0};
}

// ---------------------------------------------------------------------------
// Per-environment broad phase (geometry/broadphase.py:101-214 semantics).
//
// Candidate MEMBERSHIP is the reference's exact predicate set
//   PT: v not in t, pair_ok(body v, body t), x_v in [tri_lo - r, tri_hi + r]   (:177-183)
//   EE: i < j, no shared vertex, pair_ok, hi_j >= lo_i - r and lo_j <= hi_i + r (:195-210)
// and the output is in the reference's canonical order ((v, t) / (i, j)).
// Pairs are generated by an env-local uniform grid held in shared memory
// (cell >= r, triangles / edges inserted over their tight AABB cells, queries
// over the r-inflated box, each pair visited in exactly one cell: the lowest
// cell common to both boxes).  The grid only prunes; the predicate decides,
// so the cell size cannot change the result.
// ---------------------------------------------------------------------------
constexpr int BP_TILE = 512;      // direct broad phase: partner primitives staged per tile
constexpr int BP_MAXG = 512;      // direct broad phase: query groups with a recorded traversal mode
struct BPShared {
  union {
    struct {
      int head[MAXC + 1];
      int cur[MAXC];
    };
    struct {                        // direct path: one tile of compacted partners
      double pb[6][BP_TILE];        // tight AABB (lo, hi), SoA: conflict-free across lanes
      int pv[3][BP_TILE];           // vertices (edges: 2)
      int pid[BP_TILE];             // primitive id
    };
  };
  double bb[32][6];   // per-body surface AABB (culling: primitives far from every partner body)
  int rs[32], re[32]; // per-body range of the compacted primitive list (direct path)
  unsigned char gmode[BP_MAXG];   // direct path: per 32-query group, 1 = queries one by one
  int cl_val[4];                  // cluster broad phase: rank 0's counts, read by the other ranks (DSMEM)
};

// A thread-block cluster working on ONE env's broad phase (the rebuild of a candidate superset
// is the heavy-env tail of its kernel: an O(queries x partners) pass that would otherwise run on
// one SM while the launch waits for it).  Rank 0 compacts the culled primitives / queries; the
// 32-query groups are dealt out round-robin over the ranks for both passes; rank 0 turns the
// per-query counts into write offsets between the passes; counts travel through distributed
// shared memory.  n == 1 is the plain CTA-per-env path.
struct BPCl {
  int rank, n;
};
#ifndef GRIP_BP_CL
#define GRIP_BP_CL 4
#endif
constexpr int BP_CL = GRIP_BP_CL;   // CTAs per env cluster of k_begin / k_candidates / k_linesearch
__device__ __forceinline__ BPCl bp_solo() { return BPCl{0, 1}; }
__device__ __forceinline__ void cl_sync(const BPCl& c) {
  if (c.n > 1) {
    __threadfence();   // rank 0's global writes (compacted lists, offsets) before the other ranks read them
    cooperative_groups::this_cluster().sync();
  } else {
    __syncthreads();
  }
}
// value rank 0 left in its shared slot before a cl_sync; ends with a cl_sync so rank 0's shared
// memory outlives every remote read
__device__ __forceinline__ int cl_from0(const BPCl& c, int* slot) {
  if (c.n == 1) return *slot;
  const int v = *cooperative_groups::this_cluster().map_shared_rank(slot, 0);
  cl_sync(c);
  return v;
}

struct Grid {
  double lox, loy, loz, ih;
  int nx, ny, nz;
  __device__ __forceinline__ int cx(double v) const {
    double f = floor((v - lox) * ih);
    return f < 0.0 ? 0 : (f >= nx ? nx - 1 : (int)f);
  }
  __device__ __forceinline__ int cy(double v) const {
    double f = floor((v - loy) * ih);
    return f < 0.0 ? 0 : (f >= ny ? ny - 1 : (int)f);
  }
  __device__ __forceinline__ int cz(double v) const {
    double f = floor((v - loz) * ih);
    return f < 0.0 ? 0 : (f >= nz ? nz - 1 : (int)f);
  }
};

// shell sort of a small int segment (per-thread; segments are the candidates of one query)
__device__ void sort_ints(int* a, int n) {
  const int gaps[8] = {701, 301, 132, 57, 23, 10, 4, 1};
  for (int gi = 0; gi < 8; ++gi) {
    const int g = gaps[gi];
    for (int i = g; i < n; ++i) {
      int t = a[i];
      int j = i;
      while (j >= g && a[j - g] > t) {
        a[j] = a[j - g];
        j -= g;
      }
      a[j] = t;
    }
  }
}

// Builds the grid over `n` primitive AABBs (aabb[6*i]: lo, hi), each inserted into its
// tight cell range.  Returns false on scratch overflow.
__device__ bool grid_build(const Grid& G, const double* aabb, int n, int* cells, int* lc, int cap, BPShared& S, Red& sm) {
  const int ncell = G.nx * G.ny * G.nz;
  for (int c = threadIdx.x; c <= ncell; c += NT) S.head[c] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += NT) {
    const double* b = aabb + 6 * i;
    if (!(b[0] <= b[3])) continue;   // culled primitive
    int x0 = G.cx(b[0]), y0 = G.cy(b[1]), z0 = G.cz(b[2]);
    int x1 = G.cx(b[3]), y1 = G.cy(b[4]), z1 = G.cz(b[5]);
    for (int a = x0; a <= x1; ++a)
      for (int bb = y0; bb <= y1; ++bb)
        for (int c = z0; c <= z1; ++c) atomicAdd(&S.head[(a * G.ny + bb) * G.nz + c], 1);
  }
  __syncthreads();
  int total = block_scan_array(S.head, ncell, sm);
  if (total > cap) return false;
  for (int c = threadIdx.x; c < ncell; c += NT) S.cur[c] = S.head[c];
  if (threadIdx.x == 0) S.head[ncell] = total;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += NT) {
    const double* b = aabb + 6 * i;
    if (!(b[0] <= b[3])) continue;
    int x0 = G.cx(b[0]), y0 = G.cy(b[1]), z0 = G.cz(b[2]);
    int x1 = G.cx(b[3]), y1 = G.cy(b[4]), z1 = G.cz(b[5]);
    lc[3 * i] = x0; lc[3 * i + 1] = y0; lc[3 * i + 2] = z0;
    for (int a = x0; a <= x1; ++a)
      for (int bb = y0; bb <= y1; ++bb)
        for (int c = z0; c <= z1; ++c) cells[atomicAdd(&S.cur[(a * G.ny + bb) * G.nz + c], 1)] = i;
  }
  __syncthreads();
  // each cell's list ascending by primitive id (atomic fill order is arbitrary)
  for (int c = threadIdx.x; c < ncell; c += NT) {
    const int lo = S.head[c], hi = S.head[c + 1];
    for (int k = lo + 1; k < hi; ++k) {
      const int t = cells[k];
      int j = k - 1;
      while (j >= lo && cells[j] > t) {
        cells[j + 1] = cells[j];
        --j;
      }
      cells[j + 1] = t;
    }
  }
  __syncthreads();
  return true;
}

// Candidate stencils of one env at radius r from the sv positions in D.sv_pos.
// out_n[0] = n_pt, out_n[1] = n_ee (true counts, even past capacity).
// Returns false if an output or scratch capacity was exceeded; the host then
// grows the buffers and re-runs the whole sweep for that env.
__device__ bool broad_phase_grid(const Dev& D, const EnvIx& E, double r, int* out_pt, int* out_ee, int* out_eid,
                                 int* out_n, BPShared& S, Red& sm) {
  const double* X = D.sv_pos + 3 * (size_t)E.s0;
  const int* tris = D.tris + 3 * (size_t)E.t0;
  const int* edges = D.edges + 2 * (size_t)E.ed0;
  double* aabb = D.bp_aabb + (size_t)E.e * 6 * max(D.max_tri, D.max_edge);
  int* cells = D.bp_cells + (size_t)E.e * D.cap_cells;
  int* cnt = D.bp_cnt + (size_t)E.e * (max(D.max_sv, D.max_edge) + 1);
  int* tmp = D.bp_tmp + (size_t)E.e * max(D.cap_pt, D.cap_ee);
  int* lc = D.bp_lc + (size_t)E.e * 3 * max(D.max_tri, D.max_edge);
  if (E.ns == 0) {
    if (threadIdx.x == 0) { out_n[0] = 0; out_n[1] = 0; }
    __syncthreads();
    return true;
  }
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = threadIdx.x; i < E.ns; i += NT)
    for (int c = 0; c < 3; ++c) {
      lo[c] = fmin(lo[c], X[3 * i + c]);
      hi[c] = fmax(hi[c], X[3 * i + c]);
    }
  for (int c = 0; c < 3; ++c) {
    lo[c] = block_min(lo[c], sm);
    hi[c] = block_max(hi[c], sm);
  }
  const uint32_t* pm = D.body_pairmask + E.b0;
  const int* vb = D.sv_body + E.s0;
  // per-body AABBs: a primitive can only pair with bodies its pair mask allows, and every such
  // pair needs the primitive's r-box to reach that body's AABB -> primitives (and query
  // vertices) that reach no partner body are culled before the grid (membership unchanged)
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = warp; b < E.nb; b += NWARP) {
      double l[3] = {INFINITY, INFINITY, INFINITY}, u[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int i = lane; i < E.ns; i += 32)
        if (vb[i] == b)
          for (int c = 0; c < 3; ++c) {
            l[c] = fmin(l[c], X[3 * i + c]);
            u[c] = fmax(u[c], X[3 * i + c]);
          }
      for (int c = 0; c < 3; ++c) {
        l[c] = wmin(l[c]);
        u[c] = wmax(u[c]);
      }
      if (lane == 0)
        for (int c = 0; c < 3; ++c) { S.bb[b][c] = l[c]; S.bb[b][3 + c] = u[c]; }
    }
    __syncthreads();
  }
  // does box [l, u] inflated by rc reach a partner body of body bo (mask m)?
  auto reaches = [&](const double* l, const double* u, uint32_t m, int bo, double rc) {
    for (int b = 0; b < E.nb; ++b) {
      if (!((m >> b) & 1u)) continue;
      const double* q = S.bb[b];
      if (l[0] - rc <= q[3] && l[1] - rc <= q[4] && l[2] - rc <= q[5] && u[0] + rc >= q[0] && u[1] + rc >= q[1] &&
          u[2] + rc >= q[2])
        return true;
    }
    return false;
  };
  double h = fmax(r, D.cell_hint[E.e]);
  int npt = 0, nee = 0;
  bool ok = true;
  for (int attempt = 0; attempt < 12; ++attempt) {
    Grid G;
    G.lox = lo[0] - r; G.loy = lo[1] - r; G.loz = lo[2] - r;
    for (;;) {
      G.ih = 1.0 / h;
      G.nx = (int)fmin(floor((hi[0] + r - G.lox) * G.ih) + 1.0, 1e6);
      G.ny = (int)fmin(floor((hi[1] + r - G.loy) * G.ih) + 1.0, 1e6);
      G.nz = (int)fmin(floor((hi[2] + r - G.loz) * G.ih) + 1.0, 1e6);
      if ((long long)G.nx * G.ny * G.nz <= MAXC) break;
      h *= 1.3;
    }
    const double eps = 1e-9 * h;
    npt = nee = 0;
    ok = true;
    bool regrid = false;
    // ---------------- point-triangle ----------------
    if (E.nt && E.ns) {
      for (int t = threadIdx.x; t < E.nt; t += NT) {
        V3 a = ld3(X + 3 * tris[3 * t]), b = ld3(X + 3 * tris[3 * t + 1]), c = ld3(X + 3 * tris[3 * t + 2]);
        V3 l = vmin(vmin(a, b), c), u = vmax(vmax(a, b), c);
        double* o = aabb + 6 * t;
        o[0] = l.x; o[1] = l.y; o[2] = l.z; o[3] = u.x; o[4] = u.y; o[5] = u.z;
        const int bt = vb[tris[3 * t]];
        const uint32_t m = pm[bt] & (((pm[bt] >> bt) & 1u) ? ~0u : ~(1u << bt));
        if (!reaches(o, o + 3, m, bt, r + eps)) o[0] = INFINITY;   // culled
      }
      __syncthreads();
      if (!grid_build(G, aabb, E.nt, cells, lc, D.cap_cells, S, sm)) {
        regrid = true;
      } else {
        for (int pass = 0; pass < 2; ++pass) {
          for (int v = threadIdx.x; v < E.ns; v += NT) {
            V3 p = ld3(X + 3 * v);
            const int qx0 = G.cx(p.x - r - eps), qy0 = G.cy(p.y - r - eps), qz0 = G.cz(p.z - r - eps);
            const int qx1 = G.cx(p.x + r + eps), qy1 = G.cy(p.y + r + eps), qz1 = G.cz(p.z + r + eps);
            const uint32_t okmask = pm[vb[v]];
            const int base = pass ? cnt[v] : 0;
            const int lim = pass ? cnt[v + 1] - base : 0;
            // bodies without self-collision never pair with their own triangles
            const int bv = vb[v];
            const bool selfc = (okmask >> bv) & 1u;
            const int own_lo = selfc ? 0 : D.body_tri_lo[E.b0 + bv];
            const int own_hi = selfc ? 0 : D.body_tri_hi[E.b0 + bv];
            int count = 0;
            const double pv[3] = {p.x, p.y, p.z};
            const bool live = reaches(pv, pv, okmask & (selfc ? ~0u : ~(1u << bv)), bv, r + eps);
            for (int a = qx0; a <= (live ? qx1 : qx0 - 1); ++a)
              for (int bb = qy0; bb <= qy1; ++bb)
                for (int c = qz0; c <= qz1; ++c) {
                  const int cell = (a * G.ny + bb) * G.nz + c;
                  const int kend = S.head[cell + 1];
                  for (int k = S.head[cell]; k < kend; ++k) {
                    int t = cells[k];
                    if (t >= own_lo && t < own_hi) {   // own body's run (lists ascending): jump over it
                      int lo2 = k, hi2 = kend;
                      while (lo2 < hi2) {
                        const int mid = (lo2 + hi2) >> 1;
                        if (cells[mid] < own_hi) lo2 = mid + 1;
                        else hi2 = mid;
                      }
                      k = lo2;
                      if (k >= kend) break;
                      t = cells[k];
                    }
                    if (max(qx0, lc[3 * t]) != a || max(qy0, lc[3 * t + 1]) != bb || max(qz0, lc[3 * t + 2]) != c)
                      continue;
                    const double* bx = aabb + 6 * t;
                    const int t0 = tris[3 * t], t1 = tris[3 * t + 1], t2 = tris[3 * t + 2];
                    if (t0 == v || t1 == v || t2 == v) continue;
                    if (!((okmask >> vb[t0]) & 1u)) continue;
                    if (!(p.x >= bx[0] - r && p.y >= bx[1] - r && p.z >= bx[2] - r)) continue;
                    if (!(p.x <= bx[3] + r && p.y <= bx[4] + r && p.z <= bx[5] + r)) continue;
                    if (pass && count < lim) tmp[base + count] = t;
                    ++count;
                  }
                }
            if (!pass) {
              cnt[v] = count;
            } else {
              sort_ints(tmp + base, lim);
              for (int k = 0; k < lim; ++k) {
                const int t = tmp[base + k];
                int* row = out_pt + 4 * (base + k);
                row[0] = v; row[1] = tris[3 * t]; row[2] = tris[3 * t + 1]; row[3] = tris[3 * t + 2];
              }
            }
          }
          __syncthreads();
          if (!pass) {
            npt = block_scan_array(cnt, E.ns, sm);
            if (threadIdx.x == 0) cnt[E.ns] = npt;
            __syncthreads();
            if (npt > D.cap_pt) {
            if (threadIdx.x == 0) atomicMax(&D.need[0], (unsigned)npt);
            ok = false;
            break;
          }
          }
        }
      }
    }
    if (regrid) { h *= 2.0; continue; }
    // ---------------- edge-edge ----------------
    if (E.ne && ok) {
      for (int i = threadIdx.x; i < E.ne; i += NT) {
        V3 a = ld3(X + 3 * edges[2 * i]), b = ld3(X + 3 * edges[2 * i + 1]);
        V3 l = vmin(a, b), u = vmax(a, b);
        double* o = aabb + 6 * i;
        o[0] = l.x; o[1] = l.y; o[2] = l.z; o[3] = u.x; o[4] = u.y; o[5] = u.z;
        const int be = vb[edges[2 * i]];
        const uint32_t m = pm[be] & (((pm[be] >> be) & 1u) ? ~0u : ~(1u << be));
        if (!reaches(o, o + 3, m, be, r + eps)) o[0] = INFINITY;   // culled
      }
      __syncthreads();
      if (!grid_build(G, aabb, E.ne, cells, lc, D.cap_cells, S, sm)) { h *= 2.0; continue; }
      for (int pass = 0; pass < 2; ++pass) {
        for (int i = threadIdx.x; i < E.ne; i += NT) {
          const double* bi = aabb + 6 * i;
          if (!(bi[0] <= bi[3])) {   // culled: no partner body within reach
            if (!pass) cnt[i] = 0;
            continue;
          }
          const double lx = bi[0] - r, ly = bi[1] - r, lz = bi[2] - r;
          const double ux = bi[3] + r, uy = bi[4] + r, uz = bi[5] + r;
          const int qx0 = G.cx(lx - eps), qy0 = G.cy(ly - eps), qz0 = G.cz(lz - eps);
          const int qx1 = G.cx(ux + eps), qy1 = G.cy(uy + eps), qz1 = G.cz(uz + eps);
          const int a0 = edges[2 * i], a1 = edges[2 * i + 1];
          const uint32_t okmask = pm[vb[a0]];
          const int base = pass ? cnt[i] : 0;
          const int lim = pass ? cnt[i + 1] - base : 0;
          // pairs are (i < j); without self-collision the first candidate j is the next body's
          const int ebody = vb[a0];
          const int jmin = ((okmask >> ebody) & 1u) ? i + 1 : max(i + 1, D.body_edge_hi[E.b0 + ebody]);
          int count = 0;
          for (int a = qx0; a <= qx1; ++a)
            for (int bb = qy0; bb <= qy1; ++bb)
              for (int c = qz0; c <= qz1; ++c) {
                const int cell = (a * G.ny + bb) * G.nz + c;
                const int kbeg = S.head[cell];
                for (int k = S.head[cell + 1] - 1; k >= kbeg; --k) {
                  const int j = cells[k];
                  if (j < jmin) break;  // list ascending: nothing at or above jmin remains
                  if (max(qx0, lc[3 * j]) != a || max(qy0, lc[3 * j + 1]) != bb || max(qz0, lc[3 * j + 2]) != c)
                    continue;
                  const double* bj = aabb + 6 * j;
                  const int b0 = edges[2 * j], b1 = edges[2 * j + 1];
                  if (a0 == b0 || a0 == b1 || a1 == b0 || a1 == b1) continue;
                  if (!((okmask >> vb[b0]) & 1u)) continue;
                  if (!(bj[3] >= lx && bj[4] >= ly && bj[5] >= lz)) continue;
                  if (!(bj[0] <= ux && bj[1] <= uy && bj[2] <= uz)) continue;
                  if (pass && count < lim) tmp[base + count] = j;
                  ++count;
                }
              }
          if (!pass) {
            cnt[i] = count;
          } else {
            sort_ints(tmp + base, lim);
            for (int k = 0; k < lim; ++k) {
              const int j = tmp[base + k];
              int* row = out_ee + 4 * (base + k);
              row[0] = a0; row[1] = a1; row[2] = edges[2 * j]; row[3] = edges[2 * j + 1];
              out_eid[2 * (base + k)] = i;
              out_eid[2 * (base + k) + 1] = j;
            }
          }
        }
        __syncthreads();
        if (!pass) {
          nee = block_scan_array(cnt, E.ne, sm);
          if (threadIdx.x == 0) cnt[E.ne] = nee;
          __syncthreads();
          if (nee > D.cap_ee) {
            if (threadIdx.x == 0) atomicMax(&D.need[1], (unsigned)nee);
            ok = false;
            break;
          }
        }
      }
    }
    break;
  }
  if (threadIdx.x == 0) {
    out_n[0] = npt;
    out_n[1] = nee;
  }
  __syncthreads();
  return ok;
}

// ---------------------------------------------------------------------------
// Direct broad phase over the culled primitives (the default; the grid above is the fallback
// for envs whose culled sets are large).  Same membership predicates and canonical order:
//   1. per-body AABBs; a primitive (query vertex) survives iff its (r+eps)-box reaches the
//      AABB of a body its pair mask allows -- every predicate-true pair survives (see above);
//   2. survivors are compacted in ascending id order (ids ascend body by body, so each body
//      is one contiguous range of the compacted list);
//   3. one warp per query walks the allowed bodies' ranges 32 primitives at a time; the
//      ballot of the exact predicate gives each hit its rank, so a query's candidates come
//      out in ascending primitive id with no sort: (v, t) and (i, j) canonical order.
// Two passes (count, block scan, fill).  Work is balanced across the warps of the CTA and
// every load of a 32-chunk is contiguous.
// ---------------------------------------------------------------------------
constexpr long long BP_DIRECT_MAX = 1ll << 21;   // estimated pair tests above which the grid is used

__device__ __forceinline__ bool reaches_body(const BPShared& S, int nb, V3 l, V3 u, uint32_t m, double rc) {
  for (int b = 0; b < nb; ++b) {
    if (!((m >> b) & 1u)) continue;
    const double* q = S.bb[b];
    if (l.x - rc <= q[3] && l.y - rc <= q[4] && l.z - rc <= q[5] && u.x + rc >= q[0] && u.y + rc >= q[1] &&
        u.z + rc >= q[2])
      return true;
  }
  return false;
}

__device__ __forceinline__ int lower_bound_int(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// compacts the K-vertex primitives (K = 3 triangles, 2 edges) that survive the body cull:
// ids -> cid[c], vertices -> cv[K c + k], tight AABBs -> cb[6 c]; per-body compact ranges
// -> S.rs / S.re.  Returns the survivor count.
template <int K>
__device__ int bp_compact(const Dev& D, const EnvIx& E, const double* X, const int* prim, int n, const int* blo,
                          const int* bhi, double rc, int* cid, int* cv, double* cb, BPShared& S, Red& sm,
                          const BPCl& cl) {
  const uint32_t* pm = D.body_pairmask + E.b0;
  const int* vb = D.sv_body + E.s0;
  int ns = 0;
  if (cl.rank == 0)
  for (int s0 = 0; s0 < n; s0 += NT) {
    const int i = s0 + threadIdx.x;
    int keep = 0;
    int w[K];
    V3 l = V3{0, 0, 0}, u = V3{0, 0, 0};
    if (i < n) {
      for (int k = 0; k < K; ++k) w[k] = prim[K * i + k];
      const V3 a = ld3(X + 3 * w[0]), b = ld3(X + 3 * w[1]);
      l = vmin(a, b);
      u = vmax(a, b);
      if (K == 3) {
        const V3 c = ld3(X + 3 * w[K - 1]);
        l = vmin(l, c);
        u = vmax(u, c);
      }
      const int bt = vb[w[0]];
      keep = reaches_body(S, E.nb, l, u, pm[bt], rc);
    }
    int tot;
    const int pre = block_scan(keep, sm, &tot);
    if (keep) {
      const int c = ns + pre;
      cid[c] = i;
      for (int k = 0; k < K; ++k) cv[K * c + k] = w[k];
      double* o = cb + 6 * c;
      o[0] = l.x; o[1] = l.y; o[2] = l.z; o[3] = u.x; o[4] = u.y; o[5] = u.z;
    }
    ns += tot;
  }
  if (cl.n > 1) {
    if (cl.rank == 0 && threadIdx.x == 0) S.cl_val[0] = ns;
    cl_sync(cl);
    ns = cl_from0(cl, &S.cl_val[0]);
  }
  __syncthreads();
  if (threadIdx.x < E.nb) {
    S.rs[threadIdx.x] = lower_bound_int(cid, ns, blo[E.b0 + threadIdx.x]);
    S.re[threadIdx.x] = lower_bound_int(cid, ns, bhi[E.b0 + threadIdx.x]);
  }
  __syncthreads();
  return ns;
}

// One query against staged partner k (tile-local kt) -- the reference's exact predicates.
//   PT (broadphase.py:177-183): v not in t, x_v in [tri_lo - r, tri_hi + r]
//   EE (:195-210): no shared vertex, hi_j >= lo_i - r and lo_j <= hi_i + r
template <int K>
__device__ __forceinline__ bool bp_hit(const BPShared& S, int kt, const double* q, int q0, int q1, double r) {
  const double b0x = S.pb[0][kt], b0y = S.pb[1][kt], b0z = S.pb[2][kt];
  const double b1x = S.pb[3][kt], b1y = S.pb[4][kt], b1z = S.pb[5][kt];
  if (K == 3) {
    const int t0 = S.pv[0][kt], t1 = S.pv[1][kt], t2 = S.pv[2][kt];
    return t0 != q0 && t1 != q0 && t2 != q0 && (q[0] >= b0x - r && q[1] >= b0y - r && q[2] >= b0z - r) &&
           (q[0] <= b1x + r && q[1] <= b1y + r && q[2] <= b1z + r);
  } else {
    const int b0 = S.pv[0][kt], b1 = S.pv[1][kt];
    return !(q0 == b0 || q0 == b1 || q1 == b0 || q1 == b1) &&
           (b1x >= q[0] - r && b1y >= q[1] - r && b1z >= q[2] - r) &&
           (b0x <= q[3] + r && b0y <= q[4] + r && b0z <= q[5] + r);
  }
}

// Pairs of the nq queries with the np compacted partners (tiles of BP_TILE in shared memory).
// K = 3: PT, queries are sv ids qid[q]; K = 2: EE, queries are the compacted edges themselves
// (partner index > query index, i.e. i < j).  Per 32-query group and tile the cheaper of two
// traversals is used:
//   lane mode : lane per query, a uniform loop over the group's partner ranges (broadcast
//               shared reads);
//   query mode: one query at a time, lanes over 32 partners (ballot ranks).  These queries
//               are dealt out to the warps one by one, so a few heavy groups (e.g. the pad
//               vertices against a sphere's triangles) are spread over the whole CTA.
// Both emit each query's hits in ascending partner order; cnt[q] carries the count (pass 0)
// or the write cursor (pass 1) across tiles.  Returns the total (pass 0).
template <int K>
struct BPQuery {
  double qd[6];
  int q0, q1, qi;
  uint32_t allow;
};

template <int K>
__device__ __forceinline__ BPQuery<K> bp_load_query(const Dev& D, const EnvIx& E, const double* X, int q,
                                                    const int* qid, const int* cv, const double* cb) {
  BPQuery<K> Q;
  const uint32_t* pm = D.body_pairmask + E.b0;
  const int* vb = D.sv_body + E.s0;
  if (K == 3) {
    Q.q0 = qid[q];
    Q.q1 = -1;
    Q.qi = 0;
    const V3 pq = ld3(X + 3 * Q.q0);
    Q.qd[0] = pq.x; Q.qd[1] = pq.y; Q.qd[2] = pq.z;
    Q.qd[3] = Q.qd[4] = Q.qd[5] = 0.0;
  } else {
    for (int c = 0; c < 6; ++c) Q.qd[c] = cb[6 * q + c];
    Q.q0 = cv[2 * q];
    Q.q1 = cv[2 * q + 1];
    Q.qi = q;
  }
  Q.allow = pm[vb[Q.q0]];
  return Q;
}

template <int K>
__device__ __forceinline__ void bp_emit(const BPShared& S, int kt, int q0, int q1, int qid_global, int pos, int* out,
                                        int* out_eid) {
  int* row = out + 4 * pos;
  row[0] = q0;
  if (K == 3) {
    row[1] = S.pv[0][kt]; row[2] = S.pv[1][kt]; row[3] = S.pv[2][kt];
  } else {
    row[1] = q1; row[2] = S.pv[0][kt]; row[3] = S.pv[1][kt];
    out_eid[2 * pos] = qid_global;
    out_eid[2 * pos + 1] = S.pid[kt];
  }
}

template <int K>
__device__ int bp_pairs(const Dev& D, const EnvIx& E, const double* X, int nq, const int* qid, int np, const int* cid,
                        const int* cv, const double* cb, double r, int* cnt, int* out, int* out_eid, int cap,
                        BPShared& S, Red& sm, const BPCl& cl) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int ngroups = (nq + 31) >> 5;
  const bool modes = ngroups <= BP_MAXG;   // else every group runs in lane mode
  int total = 0;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 0)
      for (int q = threadIdx.x; q < nq; q += NT)
        if ((q >> 5) % cl.n == cl.rank) cnt[q] = 0;
    for (int p0 = 0; p0 < np; p0 += BP_TILE) {
      const int p1 = min(np, p0 + BP_TILE);
      __syncthreads();
      if (pass == 0 || np > BP_TILE) {   // a single tile stays staged for the second pass
        for (int k = p0 + threadIdx.x; k < p1; k += NT) {
          const int kt = k - p0;
          for (int c = 0; c < 6; ++c) S.pb[c][kt] = cb[6 * k + c];
          for (int c = 0; c < K; ++c) S.pv[c][kt] = cv[K * k + c];
          S.pid[kt] = cid[k];
        }
        __syncthreads();
      }
      // phase 1: each warp takes whole groups, decides their mode, runs the lane-mode ones
      for (int g = cl.rank + cl.n * warp; g < ngroups; g += cl.n * NWARP) {   // this rank's groups
        const int q = 32 * g + lane;
        const bool valid = q < nq;
        BPQuery<K> Q;
        if (valid) Q = bp_load_query<K>(D, E, X, q, qid, cv, cb);
        else { Q.allow = 0; Q.q0 = Q.q1 = -1; Q.qi = 0; for (int c = 0; c < 6; ++c) Q.qd[c] = 0.0; }
        const uint32_t uni = __reduce_or_sync(0xffffffffu, Q.allow);
        const int kmin = K == 2 ? __reduce_min_sync(0xffffffffu, valid ? Q.qi + 1 : 0x7fffffff) : 0;
        int wl = 0, ww = 0;
        for (int b = 0; b < E.nb; ++b) {
          const int hi = min(S.re[b], p1);
          const int lo = max(max(S.rs[b], p0), kmin);
          if (((uni >> b) & 1u) && hi > lo) wl += hi - lo;
          if (valid && ((Q.allow >> b) & 1u)) {
            const int lq = max(max(S.rs[b], p0), K == 2 ? Q.qi + 1 : 0);
            if (hi > lq) ww += (hi - lq + 31) >> 5;
          }
        }
        ww = __reduce_add_sync(0xffffffffu, ww);
        const bool qmode = modes && (ww <= wl || (wl > D.bp_qm_min && ww <= D.bp_qm_fac * wl));
        if (modes && lane == 0) S.gmode[g] = qmode;
        if (qmode) continue;
        int run = valid ? cnt[q] : 0;
        for (int b = 0; b < E.nb; ++b) {
          if (!((uni >> b) & 1u)) continue;
          const int lo = max(max(S.rs[b], p0), kmin), hi = min(S.re[b], p1);
          const bool mine = valid && ((Q.allow >> b) & 1u);
          for (int k = lo; k < hi; ++k) {
            const int kt = k - p0;
            if (mine && (K == 3 || k > Q.qi) && bp_hit<K>(S, kt, Q.qd, Q.q0, Q.q1, r)) {
              if (pass) bp_emit<K>(S, kt, Q.q0, Q.q1, K == 2 ? cid[Q.qi] : 0, run, out, out_eid);
              ++run;
            }
          }
        }
        if (valid) cnt[q] = run;
      }
      __syncthreads();
      // phase 2: query-mode queries, dealt out one by one: warp w takes queries base + w + 8 l
      // (l = lane), loads their data in one go and walks them with broadcasts
      if (modes)
        for (int base = 0; base < nq; base += 32 * NWARP) {
          const int q = base + warp + NWARP * lane;
          const bool mine = q < nq && (q >> 5) % cl.n == cl.rank && S.gmode[q >> 5];
          const unsigned todo = __ballot_sync(0xffffffffu, mine);
          if (!todo) continue;
          BPQuery<K> Q;
          int run = 0;
          if (mine) {
            Q = bp_load_query<K>(D, E, X, q, qid, cv, cb);
            run = cnt[q];
          } else {
            Q.allow = 0; Q.q0 = Q.q1 = -1; Q.qi = 0;
            for (int c = 0; c < 6; ++c) Q.qd[c] = 0.0;
          }
          for (unsigned left = todo; left; left &= left - 1) {
            const int j = __ffs(left) - 1;
            double qj[6];
            for (int c = 0; c < 6; ++c) qj[c] = __shfl_sync(0xffffffffu, Q.qd[c], j);
            const int j0 = __shfl_sync(0xffffffffu, Q.q0, j), j1 = __shfl_sync(0xffffffffu, Q.q1, j);
            const int ji = __shfl_sync(0xffffffffu, Q.qi, j);
            const uint32_t aj = __shfl_sync(0xffffffffu, Q.allow, j);
            int rj = __shfl_sync(0xffffffffu, run, j);
            const int gid = K == 2 ? cid[ji] : 0;
            for (int b = 0; b < E.nb; ++b) {
              if (!((aj >> b) & 1u)) continue;
              const int lo = max(max(S.rs[b], p0), K == 2 ? ji + 1 : 0), hi = min(S.re[b], p1);
              for (int s0 = lo; s0 < hi; s0 += 32) {
                const int k = s0 + lane;
                const bool hit = k < hi && bp_hit<K>(S, k - p0, qj, j0, j1, r);
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                if (pass && hit) bp_emit<K>(S, k - p0, j0, j1, gid, rj + __popc(m & lt), out, out_eid);
                rj += __popc(m);
              }
            }
            if (lane == j) run = rj;
          }
          if (mine) cnt[q] = run;
        }
    }
    __syncthreads();
    if (pass == 0) {
      if (cl.n == 1) {
        total = block_scan_array(cnt, nq, sm);
      } else {   // every rank's counts -> rank 0 turns them into write offsets -> every rank
        cl_sync(cl);
        if (cl.rank == 0) {
          total = block_scan_array(cnt, nq, sm);
          if (threadIdx.x == 0) S.cl_val[2] = total;
        }
        cl_sync(cl);
        total = cl_from0(cl, &S.cl_val[2]);
      }
      if (total > cap) return total;
    }
  }
  if (cl.n > 1) cl_sync(cl);   // every rank done with the compacted lists before they are reused
  return total;
}

// returns false on output overflow (*too_big: the culled sets are too large for the direct
// path; nothing was written and the caller runs the grid)
__device__ bool broad_phase_direct(const Dev& D, const EnvIx& E, double r, int* out_pt, int* out_ee, int* out_eid,
                                   int* out_n, BPShared& S, Red& sm, bool* too_big, const BPCl& cl) {
  const double* X = D.sv_pos + 3 * (size_t)E.s0;
  const int* tris = D.tris + 3 * (size_t)E.t0;
  const int* edges = D.edges + 2 * (size_t)E.ed0;
  const int Mx = max(D.max_tri, D.max_edge);
  double* cb = D.bp_aabb + (size_t)E.e * 6 * Mx;
  int* cid = D.bp_scr + (size_t)E.e * (4 * Mx + D.max_sv);   // [0, Mx) ids, [Mx, 4 Mx) vertices, [4 Mx, ..) queries
  int* cv = cid + Mx;
  int* qid = cid + 4 * Mx;
  int* cnt = D.bp_cnt + (size_t)E.e * (max(D.max_sv, D.max_edge) + 1);
  const uint32_t* pm = D.body_pairmask + E.b0;
  const int* vb = D.sv_body + E.s0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  *too_big = false;
  // per-body AABBs
  for (int b = warp; b < E.nb; b += NWARP) {
    double l[3] = {INFINITY, INFINITY, INFINITY}, u[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = lane; i < E.ns; i += 32)
      if (vb[i] == b)
        for (int c = 0; c < 3; ++c) {
          l[c] = fmin(l[c], X[3 * i + c]);
          u[c] = fmax(u[c], X[3 * i + c]);
        }
    for (int c = 0; c < 3; ++c) {
      l[c] = wmin(l[c]);
      u[c] = wmax(u[c]);
    }
    if (lane == 0)
      for (int c = 0; c < 3; ++c) { S.bb[b][c] = l[c]; S.bb[b][3 + c] = u[c]; }
  }
  __syncthreads();
  const double rc = r + 1e-9 * fmax(r, D.cell_hint[E.e]);
  // ---------------- point-triangle ----------------
  const int nts = bp_compact<3>(D, E, X, tris, E.nt, D.body_tri_lo, D.body_tri_hi, rc, cid, cv, cb, S, sm, cl);
  int nq = 0;
  if (cl.rank == 0)
  for (int s0 = 0; s0 < E.ns; s0 += NT) {
    const int v = s0 + threadIdx.x;
    int keep = 0;
    if (v < E.ns && nts) {
      const V3 p = ld3(X + 3 * v);
      keep = reaches_body(S, E.nb, p, p, pm[vb[v]], rc);
    }
    int tot;
    const int pre = block_scan(keep, sm, &tot);
    if (keep) qid[nq + pre] = v;
    nq += tot;
  }
  if (cl.n > 1) {
    if (cl.rank == 0 && threadIdx.x == 0) S.cl_val[1] = nq;
    cl_sync(cl);
    nq = cl_from0(cl, &S.cl_val[1]);
  }
  __syncthreads();
  if ((double)nq * nts + 0.5 * (1.5 * nts) * (1.5 * nts) > (double)BP_DIRECT_MAX) {
    *too_big = true;
    return false;
  }
  const int npt = bp_pairs<3>(D, E, X, nq, qid, nts, cid, cv, cb, r, cnt, out_pt, nullptr, D.cap_pt, S, sm, cl);
  int nee = 0;
  bool ok = npt <= D.cap_pt;
  if (!ok && cl.rank == 0 && threadIdx.x == 0) atomicMax(&D.need[0], (unsigned)npt);
  // ---------------- edge-edge ----------------
  if (ok) {
    const int nes = bp_compact<2>(D, E, X, edges, E.ne, D.body_edge_lo, D.body_edge_hi, rc, cid, cv, cb, S, sm, cl);
    nee = bp_pairs<2>(D, E, X, nes, nullptr, nes, cid, cv, cb, r, cnt, out_ee, out_eid, D.cap_ee, S, sm, cl);
    ok = nee <= D.cap_ee;
    if (!ok && cl.rank == 0 && threadIdx.x == 0) atomicMax(&D.need[1], (unsigned)nee);
  }
  if (cl.rank == 0 && threadIdx.x == 0) {
    out_n[0] = npt;
    out_n[1] = nee;
  }
  __syncthreads();
  return ok;
}

// Candidate stencils of one env at radius r (see broad_phase_grid for the contract).
__device__ bool broad_phase_env(const Dev& D, const EnvIx& E, double r, int* out_pt, int* out_ee, int* out_eid,
                                int* out_n, BPShared& S, Red& sm, const BPCl& cl = BPCl{0, 1}) {
  if (D.bp_mode == 0 && E.ns > 0) {
    bool too_big = false;
    const bool ok = broad_phase_direct(D, E, r, out_pt, out_ee, out_eid, out_n, S, sm, &too_big, cl);
    if (!too_big) return ok;
  }
  if (cl.n == 1) return broad_phase_grid(D, E, r, out_pt, out_ee, out_eid, out_n, S, sm);
  // the grid fallback (rare: very large culled sets) runs on rank 0, the others wait for its verdict
  if (cl.rank == 0) {
    const bool ok = broad_phase_grid(D, E, r, out_pt, out_ee, out_eid, out_n, S, sm);
    if (threadIdx.x == 0) S.cl_val[3] = ok ? 1 : 0;
  }
  cl_sync(cl);
  return cl_from0(cl, &S.cl_val[3]) != 0;
}

// Exact candidate set at radius r as an order-preserving filter of a superset computed at
// R >= r from the same positions: identical predicates (broadphase.py:177-183, :202-209),
// so identical membership and canonical order.
__device__ void filter_set(const Dev& D, const EnvIx& E, double r, const int* spt, const int* see, const int* seid,
                           const int* sn, int* dpt, int* dee, int* deid, int* dn, Red& sm) {
  const double* X = D.sv_pos + 3 * (size_t)E.s0;
  const int npt = sn[0], nee = sn[1];
  int base = 0;
  for (int s = 0; s < npt; s += NT) {
    const int k = s + threadIdx.x;
    int keep = 0;
    int row[4];
    if (k < npt) {
      for (int j = 0; j < 4; ++j) row[j] = spt[4 * k + j];
      V3 p = ld3(X + 3 * row[0]), a = ld3(X + 3 * row[1]), b = ld3(X + 3 * row[2]), c = ld3(X + 3 * row[3]);
      V3 l = vmin(vmin(a, b), c), u = vmax(vmax(a, b), c);
      keep = (p.x >= l.x - r && p.y >= l.y - r && p.z >= l.z - r) && (p.x <= u.x + r && p.y <= u.y + r && p.z <= u.z + r);
    }
    int tot;
    const int pre = block_scan(keep, sm, &tot);
    if (keep)
      for (int j = 0; j < 4; ++j) dpt[4 * (base + pre) + j] = row[j];
    base += tot;
  }
  const int mpt = base;
  base = 0;
  for (int s = 0; s < nee; s += NT) {
    const int k = s + threadIdx.x;
    int keep = 0;
    int row[4];
    if (k < nee) {
      for (int j = 0; j < 4; ++j) row[j] = see[4 * k + j];
      V3 a0 = ld3(X + 3 * row[0]), a1 = ld3(X + 3 * row[1]), b0 = ld3(X + 3 * row[2]), b1 = ld3(X + 3 * row[3]);
      V3 li = vmin(a0, a1), ui = vmax(a0, a1), lj = vmin(b0, b1), uj = vmax(b0, b1);
      keep = (uj.x >= li.x - r && uj.y >= li.y - r && uj.z >= li.z - r) &&
             (lj.x <= ui.x + r && lj.y <= ui.y + r && lj.z <= ui.z + r);
    }
    int tot;
    const int pre = block_scan(keep, sm, &tot);
    if (keep) {
      for (int j = 0; j < 4; ++j) dee[4 * (base + pre) + j] = row[j];
      deid[2 * (base + pre)] = seid[2 * k];
      deid[2 * (base + pre) + 1] = seid[2 * k + 1];
    }
    base += tot;
  }
  if (threadIdx.x == 0) {
    dn[0] = mpt;
    dn[1] = base;
  }
  __syncthreads();
}

}  // namespace grip
