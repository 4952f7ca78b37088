/*
 * grip_ipc.h -- C ABI of the B200-native multi-environment IPC step.
 *
 * The reference (gripsim 0.1.0, /root/reference/pkg/src/gripsim) has no FFI:
 * its boundary is the Python object API.  Each entry point below replaces one
 * reference call site; the Python host side (paper_2503_05020_b200) binds them
 * with ctypes exactly where the reference calls its own methods:
 *
 *   grip_create / grip_destroy     <- Environment.__init__ / _build (solver.py:198-363),
 *                                     Batch.__init__ (multienv.py:76-84)
 *   grip_set_controls              <- writes of env.gravity and body.velocity
 *                                     (protocol.py:193-225, solver.py:599-613)
 *   grip_begin_step                <- Environment.begin_step (solver.py:590-645)
 *   grip_newton_iteration          <- Environment.newton_iteration (solver.py:647-731), one
 *                                     sweep over the pending envs (multienv.py:163-167)
 *   grip_finalize_step             <- Environment.finalize_step (solver.py:733-762)
 *   grip_step                      <- Batch.step / _step_serial_sweeps (multienv.py:130-168)
 *   grip_get_state / grip_set_state<- env.x / env.v reads and writes (solver.py:314-315)
 *   grip_get_surface               <- Environment.surface_positions (solver.py:367-372)
 *   grip_get_contacts              <- protocol.contact_events_now + finger_contact_force
 *                                     (protocol.py:72-98, contact.py:348-372)
 *   grip_query_candidates          <- broad_phase (geometry/broadphase.py:101-155)
 *   grip_stress                    <- materials.compute_stress (materials.py:191-205)
 *
 * Pointers are HOST pointers except in the *_device entry points (device pointers, e.g. torch
 * tensors' data_ptr()); the library owns its device memory and by default its CUDA stream
 * (grip_set_stream hands it a caller's stream).  Per-environment failures are data (GripStepReport.status),
 * never return codes.  Return codes: 0 ok, <0 error (see grip_last_error()).
 */
#ifndef GRIP_IPC_H
#define GRIP_IPC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GRIP_ABI_VERSION 4

/* Flattened description of N environments (all arrays host, row-major).
 * Index spaces are ENV-LOCAL (node / surface-vertex / body ids restart at 0 in
 * every env); *_off arrays (length n_env+1) give each env's slice. */
typedef struct GripSceneDesc {
  int32_t abi_version;
  int32_t n_env;
  const int32_t* node_off; /* nodes: soft vertices, then 4 pseudo-nodes (p, A rows) per affine body */
  const int32_t* sv_off;   /* surface vertices (collision vertices) */
  const int32_t* tri_off;
  const int32_t* edge_off;
  const int32_t* tet_off;
  const int32_t* abd_off;
  const int32_t* body_off;
  /* nodes */
  const double* node_x0;   /* 3 per node: initial positions / q */
  const double* node_M;    /* 9 per node: 3x3 mass block */
  const uint8_t* node_free;
  const int32_t* node_body;
  const uint8_t* node_kind; /* 0 soft, 1 affine p, 2 affine A-row */
  const int32_t* node_sv;   /* soft node -> its surface vertex, or -1 */
  /* surface vertices */
  const uint8_t* sv_kind;   /* 0 soft, 1 affine, 2 kinematic */
  const int32_t* sv_node;   /* soft: node; affine: p-node; kinematic: -1 */
  const double* sv_xi;      /* 3 per sv (affine body frame offset) */
  const int32_t* sv_body;
  const double* sv_kin0;    /* 3 per sv: initial kinematic positions */
  /* topology */
  const int32_t* tris;      /* 3 per tri (sv ids) */
  const int32_t* edges;     /* 2 per edge (sv ids) */
  const double* edge_rest_sq;
  const int32_t* tet_nodes; /* 4 per tet (node ids) */
  const double* tet_Dmi;    /* 9 per tet */
  const double* tet_V0;
  const double* tet_mu;
  const double* tet_lam;
  const int32_t* abd_node;  /* p-node of each affine body */
  const double* abd_kV;     /* kappa * enclosed volume */
  const int32_t* abd_body;
  /* bodies */
  const uint8_t* body_kind;
  const double* body_mu;
  const uint32_t* body_pairmask; /* bit j: may collide with env-local body j */
  const double* body_vel0;  /* 3 per body */
  const int32_t* body_tri_lo;  /* env-local triangle range [lo, hi) of each body */
  const int32_t* body_tri_hi;
  const int32_t* body_edge_lo; /* env-local edge range [lo, hi) of each body */
  const int32_t* body_edge_hi;
  /* per-env parameters (14 doubles each, see GRIP_P_* ) and gravity (3 each) */
  const double* env_params;
  const double* env_gravity;
  const double* env_cell_hint; /* broad-phase cell size hint (m) */
} GripSceneDesc;

enum {
  GRIP_P_DT = 0, GRIP_P_KAPPA, GRIP_P_DHAT, GRIP_P_EPSV, GRIP_P_RELTOL, GRIP_P_MAXIT, GRIP_P_ELLFLOOR,
  GRIP_P_MAXLS, GRIP_P_CCDSCALE, GRIP_P_CCDIT, GRIP_P_KINGUARD, GRIP_P_MURULE, GRIP_P_PCGRTOL, GRIP_P_SPARE,
  GRIP_NPARAM
};

/* status codes */
enum { GRIP_NS_RUNNING = 0, GRIP_NS_CONVERGED = 1, GRIP_NS_FAILED = 2 };
enum {
  GRIP_R_NONE = 0,
  GRIP_R_NONCONV = 1,            /* "non-convergence" */
  GRIP_R_LINESEARCH = 2,         /* "line-search-failure" */
  GRIP_R_INVERTED = 3,           /* "ValueError: inverted element passed to elastic energy" */
  GRIP_R_CONTACT_D = 4,          /* "ValueError: contact stencil at non-positive distance" */
  GRIP_R_NONFINITE = 5,          /* "FloatingPointError: non-finite assembly" */
  GRIP_R_SOLVE = 6,              /* "SolveBreakdown: linear solve failed after regularization" */
  GRIP_R_CCD = 7,                /* "IntersectionError: CCD called from an intersecting or touching state" */
  GRIP_R_DET = 8,                /* "IntersectionError: step filter called with non-positive determinant state" */
  GRIP_R_NONFINITE_STATE = 9,    /* "non-finite state" (quarantine) */
  GRIP_R_CAPACITY = 10           /* device buffer capacity exceeded (never silent) */
};

typedef struct GripStepReport {
  int32_t status;      /* GRIP_NS_* */
  int32_t reason;      /* GRIP_R_* */
  int32_t iterations;
  int32_t n_alphas;
  double residual;
  double min_distance;
  double energy;
  double time;
  int32_t step_index;
  int32_t kinematic_blocked;
  int32_t regularized;
  int32_t newton_calls; /* newton_iteration calls this step (incl. the final check) */
  int32_t pcg_iters;    /* total PCG iterations this step */
  int32_t pad;
} GripStepReport;

typedef struct GripBatch GripBatch;

int grip_abi_version(void);
const char* grip_last_error(void);
int grip_create(const GripSceneDesc* desc, int device, GripBatch** out);
int grip_destroy(GripBatch* b);
int grip_set_controls(GripBatch* b, const double* gravity /* n_env*3 or NULL */,
                      const double* body_vel /* n_body*3 or NULL */);
int grip_begin_step(GripBatch* b, const uint8_t* active /* n_env */);
/* one Newton sweep over envs with pending[e]=1; clears pending for envs that finished */
int grip_newton_iteration(GripBatch* b, uint8_t* pending /* n_env, in/out */);
int grip_finalize_step(GripBatch* b, const uint8_t* active, GripStepReport* reports /* n_env */,
                       double* alphas /* n_env * max_iters, or NULL */);
int grip_step(GripBatch* b, const uint8_t* active, GripStepReport* reports, double* alphas);
/* Continuous batching (no lockstep): begin_step for envs with begin[e]=1, one Newton sweep
 * over every unfinished env in begin|iter, finalize_step for the envs that finished this round
 * (finalized[e]=1, reports[e] filled).  Each env still follows solver.py:590-773 exactly;
 * envs simply no longer wait for the slowest env of the batch between time steps. */
int grip_round(GripBatch* b, const uint8_t* begin, const uint8_t* iter, uint8_t* finalized,
               GripStepReport* reports, double* alphas);
int grip_get_state(GripBatch* b, double* x, double* v, double* kin /* n_sv*3, or NULL */);
/* Run the batch on a caller's cudaStream_t (NULL: the library's own stream again); queued work on
 * the previous stream is finished first; the caller keeps ownership of its stream. */
int grip_set_stream(GripBatch* b, void* stream);
/* Device-pointer forms (torch tensors): stream-ordered copies on the batch's stream, no sync.
 * x, v: n_node*3, kin: n_sv*3; gravity: n_env*3, body_vel: n_body*3 (any may be NULL). */
int grip_get_state_device(GripBatch* b, double* x, double* v, double* kin);
int grip_set_controls_device(GripBatch* b, const double* gravity, const double* body_vel);
int grip_set_state(GripBatch* b, const double* x, const double* v, const double* kin);
int grip_get_surface(GripBatch* b, double* sv /* n_sv*3 */);
/* per env-local body pair: summed barrier force (lambda) of active stencils at the
 * current state (1.05*dhat candidate set) and a contact bit matrix */
int grip_get_contacts(GripBatch* b, double* body_force /* n_body */, uint32_t* contact_mask /* n_body */,
                      double* min_distance /* n_env */);
/* canonical candidate stencils of env `env` at radius r, env-local sv ids */
int grip_query_candidates(GripBatch* b, int env, double radius, int32_t* pt, int32_t cap_pt, int32_t* n_pt,
                          int32_t* ee, int32_t cap_ee, int32_t* n_ee);
int grip_stress(GripBatch* b, double* out /* n_tet*7 */);
/* Contact-event recording (protocol.py:72-75 contact_events_now, contact.py:348-372
 * ContactSet.stencil_forces): while on, every finalize_step also stores the env's active
 * stencils of the fresh 1.05*dhat candidate set, PT then EE in canonical order.
 * grip_get_events copies them for the envs with mask[e]=1, packed in env order:
 * counts[e] (n_env) = events of env e copied (bounded by the anchor capacity),
 * ev_i (7 per event: kind 0 PT / 1 EE, body a, body b, 4 env-local sv ids), ev_d (2 per event:
 * d, lambda = kappa m |b'(d)|).  cap = rows available in ev_i / ev_d. */
int grip_set_recording(GripBatch* b, int on);
/* stream priority of the batch (0 default, larger = scheduled first among concurrent batches) */
int grip_set_priority(GripBatch* b, int priority);
/* Device-resident grasp protocol (protocol.py:152-277): the phase state machine
 * runs on the device after every finalize (k_protocol), sets the fingers' velocities and the
 * gravity of the next step itself, and keeps the trial record, so many rounds run back to back
 * with no host decision.  Setup (per env, n_env entries each): finger_body[2] (env-local body
 * ids of finger 0 / 1), closing_dir[2*3], object_body, gripper_bits (bit b = body b is a finger
 * link), max_close (close-phase step cap); cfg[8] = {settle steps, hold steps, gravity-phase
 * steps, closing speed, force halt, gravity magnitude, steady speed steps, stability constant}.
 * Every env starts a trial (settle, fingers still, gravity off). */
typedef struct GripTrialOut {
  double halt_force[2];
  double com_disp[6];     /* gravity+x, -x, +y, -y, +z, -z */
  double final_disp, threshold;
  int32_t phase;          /* 0 settle 1 close 2 hold 3 gravity 4 done */
  int32_t verdict;        /* 0 running 1 stable 2 unstable 3 sim-failed */
  int32_t n_steps;
  int32_t fail_phase;     /* 0 settle 1 close 2 hold 3+g gravity phase g */
  int32_t fail_reason;    /* GRIP_R_* */
  int32_t fail_step;
  int32_t halted;         /* bit j: finger j halted */
  int32_t final_contact;
  int32_t halt_step[2];
  int32_t markers[18];    /* [start, end) per phase 0..8, -1 = phase not completed */
  /* safety report over the trial's completed steps (the north star's "zero intersections and
   * zero inverted elements"): min stencil distance of the finalize contact set (> 0: no
   * intersection; inf: no stencil ever within 1.05 dhat) and min J = det F over every tet,
   * det A over every affine body (> 0: nothing inverted) */
  double min_distance;
  double min_J;
} GripTrialOut;
int grip_protocol_setup(GripBatch* b, const int32_t* finger_body, const double* closing_dir, const int32_t* object_body,
                        const int32_t* gripper_bits, const int32_t* max_close, const double* cfg);
/* restart the protocol of the masked envs (after grip_reset_envs gave them a new candidate) */
int grip_protocol_reset(GripBatch* b, const uint8_t* mask, const double* closing_dir, const int32_t* max_close);
/* run `rounds` continuous-batching rounds on the device (begin / sweep / finalize / protocol)
 * with one synchronisation at the end; capacity overflows are grown there and the affected
 * envs simply resume.  *env_steps = time steps completed. */
int grip_run_rounds(GripBatch* b, int rounds, int64_t* env_steps);
int grip_protocol_read(GripBatch* b, GripTrialOut* out /* n_env */);
/* Pipelined form of grip_run_rounds + grip_protocol_read (replaces the same reference loop,
 * pipeline/__init__.py:51-70 around protocol.py:152-277): enqueue the rounds and an async
 * readout of the env-step counter and every env's GripTrialOut, return at once with a ticket;
 * at most two calls in flight.  grip_rounds_wait blocks until that call's readout landed and
 * returns it (out may be NULL); a capacity overflow seen there drains the stream and grows.
 * Refills (grip_reset_envs / grip_protocol_reset) issued between the two queue behind the
 * call in flight, so the host's collect-and-refill overlaps the device's next call. */
int grip_run_rounds_async(GripBatch* b, int rounds, int32_t* ticket);
int grip_rounds_wait(GripBatch* b, int32_t ticket, int64_t* env_steps, GripTrialOut* out /* n_env or NULL */);
/* One recorder frame (protocol.py:113-146) of the envs with mask[e]=1, packed in env order:
 * x, v (their nodes * 3), kin (their surface vertices * 3: kinematic positions, zeros for
 * the others) and stress (their tets * 7, materials.py:191-205).  Any output may be NULL. */
int grip_get_frames(GripBatch* b, const uint8_t* mask, double* x, double* v, double* kin, double* stress);
/* SDFs for the D1/D2 grasp-quality metrics (gripsim/geometry/sdf.py, pipeline/metrics.py).
 * grip_sdf_exact replaces the narrow-band loop of build_sdf (sdf.py:168-241): for every point
 * the exact distance to the closest of the n_tris triangles, signed by the angle-weighted
 * pseudonormal of the closest feature (face_n: n_tris*3; edge_n: n_tris*9, edges (0,1),
 * (1,2), (2,0); vert_n: n_verts*3).  grip_sdf_query evaluates metrics.py:58-75 on n samples:
 * d_o = -(trilinear SDF) inside the grid box (in the frame body = (p - trans) rot, rot
 * row-major 3x3 or NULL for identity) and -|gap to [world_lo, world_hi]| outside; it returns
 * max d_o in *d_max and, if d_o is not NULL, every value. */
int grip_sdf_exact(const double* pts, int64_t n, const double* verts, int32_t n_verts, const int32_t* tris,
                   int32_t n_tris, const double* face_n, const double* edge_n, const double* vert_n, double* out);
/* Exact nearest-neighbour distance of n points to a cloud of m points (the SDF far field,
 * sdf.py:150-151): cloud sorted by the caller into leaves of 8 under an implicit complete
 * binary tree of `levels` levels of boxes (heap order, 2^(levels+1)-1 nodes, box_lo / box_hi
 * 3 per node, empty leaves as inverted boxes). */
int grip_sdf_nn(const double* pts, int64_t n, const double* cloud, int64_t m, const double* box_lo, const double* box_hi,
                int32_t levels, double* out);
int grip_sdf_query(const double* values, const int32_t* dims, const double* origin, const double* spacing,
                   const double* rot, const double* trans, const double* world_lo, const double* world_hi,
                   const double* pts, int64_t n, double* d_o, double* d_max);
/* Contact readout at the CURRENT state without stepping (protocol.py:72-75 contact_events_now,
 * solver.py:449-453 min_contact_distance, contact.py:348-372 stencil_forces), for the envs with
 * mask[e]=1: the canonical candidate set at radius_factor * dhat, min_distance[e] (n_env, may be
 * NULL) = min stencil distance over it (inf when empty), its active stencils (d < dhat) as event
 * rows for grip_get_events, per-body force sums and contact bits for grip_get_contacts. */
/* nonfinite[e] (n_env) = 1 when env e's state x holds a NaN / inf: the quarantine test of
 * Batch.quarantine_failures (multienv.py:98-123), evaluated on the device. */
int grip_check_finite(GripBatch* b, uint8_t* nonfinite);
int grip_contacts_now(GripBatch* b, const uint8_t* mask, double radius_factor, double* min_distance);
int grip_get_events(GripBatch* b, const uint8_t* mask, int32_t* counts, int32_t* ev_i, double* ev_d, int64_t cap);
/* per-body centre of mass (n_body*3) and per-env max point speed after the last finalize
 * (solver.py:384-428; read by the protocol's steady / COM tests, protocol.py:231-249) */
int grip_get_body_state(GripBatch* b, double* body_com, double* max_speed);
/* per-kernel CUDA-event timing on the library stream (0 begin, 1 candidates, 2 work-scan,
 * 3 elements, 4 assemble+PCG, 5 line search, 6 finalize); units (8 doubles) = element counts
 * (tets, affine, contacts, anchors) of kernel 3, then PCG iterations, linear solves and
 * summed unknowns of kernel 4, since profiling was enabled */
int grip_set_profiling(GripBatch* b, int on);
int grip_kernel_stats(GripBatch* b, int kernel, double* ms, int64_t* launches, double* units);
/* CUDA events on the library stream: start=1 marks, start=0 returns ms since the mark */
int grip_stream_timer(GripBatch* b, int start, double* ms);
/* Re-initialise the envs with mask[e]=1 to a new scene of the SAME topology (a new grasp
 * candidate for the same object / gripper meshes, possibly a new material: the slot refill of
 * run_batch_trials, multienv.py:204-216, done in place).  desc describes a full batch of the same
 * n_env and offsets; the masked envs' slices of every pose- or material-dependent array are read
 * from it (node_x0, node_M, sv_kin0, sv_xi, tet_Dmi, tet_V0, tet_mu, tet_lam, body_mu,
 * edge_rest_sq, abd_kV, env_cell_hint -- posed rest shapes differ from the previous candidate's in
 * the last bits), staged through one pinned buffer and scattered by one kernel.  Every other piece
 * of per-env state returns to what grip_create starts from (v, anchors, time, step index, Jacobi
 * warm starts, candidate superset, ...), so a refilled env is bitwise a fresh one.  An env whose
 * offsets differ is an error (nothing is reset). */
int grip_reset_envs(GripBatch* b, const uint8_t* mask, const GripSceneDesc* desc);
/* Evaluate n standalone elements with the device element kernels (test / parity hook).
 * type 0 PT  in[x(12), kappa, dhat]; 1 EE in[x(12), eps_x, kappa, dhat];
 * 2 NH in[x(12), Dm^-1(9), V0, mu, lambda]; 3 ABD in[A(9), kappa*V];
 * 4 friction in[x(12), x_prev(12), gamma(4), T(6), lambda, mu, eps_v, dt]
 * outputs per element: energy, grad (12), SPD-projected 12x12 Hessian, flags (1 active, 2 bad d, 4 inverted) */
int grip_debug_elements(int type, int n, const double* in, int stride, double* E, double* g, double* H, int* flags);
/* The same element evaluations through the PRODUCTION element chain of a Newton sweep (test /
 * parity hook): types 0 / 1 (PT / EE stencils) via the k_elements_w element code with its clamp
 * deferral -> k_tet_jacobi2 -> k_tet_finish; type 2 (NH tets) via k_tet_front (Gershgorin
 * pass-through or deferral) -> k_tet_jacobi2 -> k_tet_back, warm-started from eig (n*81
 * row-major 9x9 eigenbases, updated in place; NULL = identity). */
int grip_debug_chain(int type, int n, const double* in, int stride, double* E, double* g, double* H, double* eig,
                     int* flags);
/* Per-CTA wall-time records of the CTA-per-env kernels (builds with -DGRIP_CTA_TIMING only; 0
 * records otherwise): 4 uint64 per CTA = launch sequence number, kernel << 32 | env (kernel 0 begin,
 * 1 candidates, 2 assemble_direct, 3 line search, 4 finalize), SM id, start (low 32 bits of the ns
 * globaltimer) << 32 | duration (ns); kernel 5 = k_bound (finalize + protocol + begin).  reset=1 clears the buffer after the copy. */
int grip_cta_records(GripBatch* b, uint64_t* out, int64_t cap, int64_t* n, int reset);
/* timing of the last grip_step: device ms (CUDA events) and kernel launches */
int grip_last_step_stats(GripBatch* b, double* device_ms, int64_t* launches, int64_t* newton_sweeps);

#ifdef __cplusplus
}
#endif
#endif /* GRIP_IPC_H */
