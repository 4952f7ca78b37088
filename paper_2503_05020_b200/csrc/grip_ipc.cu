// C ABI of the batched IPC step (include/grip_ipc.h): device memory, the
// static block structure of every env's Hessian, and the host loop that
// drives begin / Newton sweeps / finalize over the pending-env lists.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "grip_kernels.cuh"
#include "grip_warp_elements.cuh"
#include "grip_tet.cuh"
#include "grip_direct.cuh"
#include "grip_tetclamp.cuh"
#include "grip_sdf.cuh"

using namespace grip;

namespace {

thread_local std::string g_err;

#define CK(call)                                                                            \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess) {                                                                \
      g_err = std::string(#call) + ": " + cudaGetErrorString(_e);                           \
      return -1;                                                                            \
    }                                                                                       \
  } while (0)

// in void launch helpers: remember the first error; the caller's next CK'd call reports it
#define CK_VOID(call)                                                                       \
  do {                                                                                      \
    cudaError_t _e = (call);                                                                \
    if (_e != cudaSuccess && g_err.empty()) g_err = std::string(#call) + ": " + cudaGetErrorString(_e); \
  } while (0)

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
};

}  // namespace

struct GripBatch {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;   // the library's stream (stream may be a caller's, grip_set_stream)
  cudaStream_t aux = nullptr;          // second stream: the tet chain of a sweep, forked / joined by events
  cudaStream_t aux2 = nullptr;         // third stream: the ABD elements (one warp-level element per env)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_abd = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  Dev D{};
  int n_env = 0, n_node = 0, n_sv = 0, n_tet = 0, n_abd = 0, n_body = 0, n_free = 0, n_blk = 0;
  std::vector<void*> owned;     // device allocations released at destroy
  // host copies of the env slices
  std::vector<int> node_off, sv_off, tri_off, edge_off, tet_off, abd_off, body_off;
  std::vector<int> tet_env;
  int* d_list = nullptr;        // active / pending lists
  int* d_list2 = nullptr;
  int* d_tet_env = nullptr;
  int* d_ident = nullptr;       // 0..n_env-1 (device protocol rounds run over every env)
  double* d_stress = nullptr;   // persistent: stress rows (n_tet * 7)
  double* d_frame = nullptr;    // persistent: packed frame of the masked envs (grip_get_frames)
  double* h_frame = nullptr;    // pinned staging of the same
  double* d_md_now = nullptr;   // grip_contacts_now: per env min distance at the queried radius
  int* d_nonfin = nullptr;      // grip_check_finite: per env flag
  bool ev_now = false;          // the ev_* buffers hold a grip_contacts_now readout
  char* h_pinit = nullptr;      // pinned staging of the protocol (re)starts
  char* d_pinit = nullptr;
  size_t pinit_cap = 0;
  char* h_reset = nullptr;      // pinned staging of grip_reset_envs (env list, offsets, slices)
  char* d_reset = nullptr;
  size_t reset_cap = 0;
  int* d_fmask = nullptr;       // per env: packed offsets (node, sv, tet) or -1
  int* h_fmask = nullptr;
  int* h_pin = nullptr;         // pinned small readbacks
  int* h_lists = nullptr;       // pinned: round lists (begin | iterating), 2 n_env
  // pinned per-round snapshot: everything the host reads after a round, one D2H batch
  char* h_snap = nullptr;
  int *s_flags = nullptr, *s_done = nullptr, *s_st = nullptr, *s_rs = nullptr, *s_it = nullptr, *s_kb = nullptr,
      *s_rg = nullptr, *s_si = nullptr, *s_nc = nullptr, *s_pi = nullptr;
  double *s_res = nullptr, *s_md = nullptr, *s_en = nullptr, *s_tm = nullptr, *s_alpha = nullptr, *s_force = nullptr,
         *s_com = nullptr, *s_speed = nullptr;
  uint32_t* s_cmask = nullptr;
  bool snap_valid = false;      // snapshot equals device state (no state change since the round)
  int max_it = 100;
  double last_ms = 0.0;
  long long launches = 0, sweeps = 0;
  unsigned long long seq_ctr = 0;   // D.launch_seq source (per-CTA timing records)
  // optional per-kernel timing on the library stream (grip_set_profiling)
  bool prof = false;
  // grids of the flat element kernels (k_tet_front, k_elements_w, k_tet_jacobi2, k_tet_back), in
  // blocks; GRIP_EGRID="f,w,j,b" (blocks per SM) overrides
  int eg[4] = {148 * 2, 148 * 2, 148 * 2, 148 * 4};
  bool direct = getenv("GRIP_SOLVER") == nullptr || std::string(getenv("GRIP_SOLVER")) != "pcg";
  int env_cap = 0;        // direct solve: skyline capacity (doubles) in shared memory
  size_t dyn_smem = 0;
  static constexpr int NK = 8;
  std::vector<cudaEvent_t> kev;   // pairs
  std::vector<int> kev_free;      // event pairs whose times were collected
  std::vector<std::pair<int, int>> pending_k;  // (kernel id, event pair index), in launch order
  // pipelined device-protocol calls (grip_run_rounds_async / grip_rounds_wait): up to two calls
  // in flight, each with a pinned readout (env-step counter, flags, protocol records) and an event
  struct RoundSlot {
    char* h = nullptr;
    cudaEvent_t ev = nullptr;
    bool busy = false;
    size_t kt_mark = 0;   // pending_k entries of this call (and of calls before it)
  };
  RoundSlot rslot[2];
  int rslot_next = 0;
  // the pipelined call's launch sequence as a CUDA graph, one per readout slot (a graph's timing
  // events are not re-recorded before that slot's readout was waited for); re-captured whenever
  // the kernels' arguments (the Dev struct: buffers grow), the stream, the round count or the
  // profiling switch change
  struct RoundGraph {
    cudaGraphExec_t exec = nullptr;
    Dev D{};
    cudaStream_t stream = nullptr;
    int rounds = 0, env_cap = 0;
    size_t dyn_smem = 0;
    bool prof = false;
    std::vector<std::pair<int, int>> kt;   // the captured timing event pairs
    long long launches = 0;
  };
  RoundGraph rgraph[2];
  std::vector<char> kev_owned;   // event pair owned by a captured graph (never freed by kt_collect)
  cudaEvent_t ev_reset_st = nullptr, ev_pinit_st = nullptr;   // staging consumed (copy + kernel done)
  double k_ms[NK] = {0};
  long long k_n[NK] = {0};
  cudaEvent_t r0 = nullptr, r1 = nullptr;

  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    if (n == 0) n = 1;
    if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) return nullptr;
    cudaMemsetAsync(p, 0, n * sizeof(T), stream);
    owned.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const T* h, size_t n) {
    T* d = alloc<T>(n);
    if (d && h && n) cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, stream);
    return d;
  }
  void release(void* p) {
    auto it = std::find(owned.begin(), owned.end(), p);
    if (it != owned.end()) {
      cudaFree(p);
      owned.erase(it);
    }
  }
};

namespace {

// (re)allocate every buffer whose size depends on the candidate / element capacities
int alloc_dynamic(GripBatch* b, bool keep_anchors, int old_cap_anc) {
  Dev& D = b->D;
  const size_t E = b->n_env;
  auto swap_alloc = [&](auto*& ptr, size_t n) {
    using T = std::remove_reference_t<decltype(*ptr)>;
    if (ptr) b->release((void*)ptr);
    ptr = b->alloc<std::remove_const_t<T>>(n);
    return ptr != nullptr;
  };
  bool ok = true;
  ok &= swap_alloc(D.c1_pt, E * 4 * D.cap_pt);
  ok &= swap_alloc(D.c1_ee, E * 4 * D.cap_ee);
  ok &= swap_alloc(D.c1_eid, E * 2 * D.cap_ee);
  ok &= swap_alloc(D.c2_pt, E * 4 * D.cap_pt);
  ok &= swap_alloc(D.c2_ee, E * 4 * D.cap_ee);
  ok &= swap_alloc(D.c2_eid, E * 2 * D.cap_ee);
  ok &= swap_alloc(D.act, E * D.cap_act);
  D.cap_el = D.max_tet + D.max_abd + D.cap_act + D.cap_anc;
  ok &= swap_alloc(D.el_E, E * D.cap_el);
  ok &= swap_alloc(D.el_g, E * D.cap_el * 12);
  ok &= swap_alloc(D.el_H, E * D.cap_el * 144);
  ok &= swap_alloc(D.el_idx, E * D.cap_el * 4);
  ok &= swap_alloc(D.c_r, E * 12 * (D.cap_act + D.cap_anc));
  ok &= swap_alloc(D.inc, E * 4 * (D.cap_act + D.cap_anc));
  ok &= swap_alloc(D.cjac_S, E * 45 * D.cap_act);
  ok &= swap_alloc(D.cjac_W, E * 90 * D.cap_act);
  ok &= swap_alloc(D.cjac_list, E * D.cap_act);
  if (!D.cjac_n) ok &= swap_alloc(D.cjac_n, 1);
  if (b->direct) {
    ok &= swap_alloc(D.el_K, E * 300 * (D.cap_act + D.cap_anc));
    ok &= swap_alloc(D.el_kn, E * 9 * (D.cap_act + D.cap_anc));
    ok &= swap_alloc(D.sc_lst, E * 8 * (D.cap_act + D.cap_anc));
    ok &= swap_alloc(D.sc_off, E * 2 * ((size_t)D.max_free + 1));
  } else if (!D.el_K) {
    ok &= swap_alloc(D.el_K, 1);
    ok &= swap_alloc(D.el_kn, 1);
    ok &= swap_alloc(D.sc_lst, 1);
    ok &= swap_alloc(D.sc_off, 1);
  }
  ok &= swap_alloc(D.bp_tmp, E * std::max(D.cap_pt, D.cap_ee));
  ok &= swap_alloc(D.cs_pt, E * 4 * D.cap_pt);
  ok &= swap_alloc(D.cs_ee, E * 4 * D.cap_ee);
  ok &= swap_alloc(D.cs_eid, E * 2 * D.cap_ee);
  if (D.cs_valid) cudaMemsetAsync(D.cs_valid, 0, sizeof(int) * E, b->stream);  // supersets were dropped
  ok &= swap_alloc(D.bp_cells, E * D.cap_cells);
  // anchors persist: copy with the new pitch
  auto grow_anc = [&](auto*& ptr, int width) {
    using T = std::remove_reference_t<decltype(*ptr)>;
    T* np = b->alloc<T>(E * D.cap_anc * width);
    if (!np) return false;
    if (ptr && keep_anchors)
      cudaMemcpy2DAsync(np, sizeof(T) * width * D.cap_anc, ptr, sizeof(T) * width * old_cap_anc,
                        sizeof(T) * width * old_cap_anc, E, cudaMemcpyDeviceToDevice, b->stream);
    if (ptr) b->release((void*)ptr);
    ptr = np;
    return true;
  };
  ok &= grow_anc(D.anc_v, 4);
  ok &= grow_anc(D.anc_gamma, 4);
  ok &= grow_anc(D.anc_T, 6);
  ok &= grow_anc(D.anc_lam, 1);
  ok &= grow_anc(D.anc_mu, 1);
  ok &= grow_anc(D.anc_b, 2);
  ok &= swap_alloc(D.ev_i, E * 7 * D.cap_anc);   // events: per step, not preserved across growth
  ok &= swap_alloc(D.ev_d, E * 2 * D.cap_anc);
  if (!ok) {
    g_err = "out of device memory growing candidate/element buffers";
    return -1;
  }
  return 0;
}

// Grow only the capacities that overflowed, to 1.25x the largest count the kernels reported
// (D.need); buffers are per-env uniform, so one heavy env must not double every array of a
// 3200-env batch.  A flagged overflow with no recorded need (should not happen) doubles all.
int grow(GripBatch* b) {
  Dev& D = b->D;
  const int old_anc = D.cap_anc;
  unsigned need[4] = {0, 0, 0, 0};
  CK(cudaMemcpyAsync(need, D.need, sizeof(need), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  int* caps[4] = {&D.cap_pt, &D.cap_ee, &D.cap_act, &D.cap_anc};
  bool any = false;
  for (int k = 0; k < 4; ++k)
    if ((long long)need[k] > *caps[k]) {
      *caps[k] = std::max(*caps[k] + 1, (int)std::min<long long>((long long)need[k] * 5 / 4 + 8, 1ll << 30));
      any = true;
    }
  if (!any)
    for (int k = 0; k < 4; ++k) *caps[k] *= 2;
  CK(cudaMemsetAsync(D.need, 0, sizeof(need), b->stream));
  return alloc_dynamic(b, true, old_anc);
}

int upload_list(GripBatch* b, const std::vector<int>& L, int* dst) {
  if (!L.empty()) CK(cudaMemcpyAsync(dst, L.data(), L.size() * sizeof(int), cudaMemcpyHostToDevice, b->stream));
  return 0;
}

// run an env kernel over a list until no env overflows its buffers
template <class Launch>
int run_with_growth(GripBatch* b, int n, Launch launch) {
  for (int attempt = 0; attempt < 8; ++attempt) {
    launch();
    b->launches++;
    int* ov = b->D.flags;  // scan flags of listed envs on the host
    (void)ov;
    std::vector<int> fl(b->n_env);
    CK(cudaMemcpyAsync(fl.data(), b->D.flags, sizeof(int) * b->n_env, cudaMemcpyDeviceToHost, b->stream));
    CK(cudaStreamSynchronize(b->stream));
    bool any = false;
    for (int e = 0; e < b->n_env; ++e) any |= (fl[e] & FLAG_OVERFLOW) != 0;
    if (!any) return 0;
    if (grow(b)) return -1;
    CK(cudaMemsetAsync(b->D.flags, 0, sizeof(int) * b->n_env, b->stream));
  }
  g_err = "buffer growth did not converge";
  return -1;
}

}  // namespace

extern "C" {

int grip_abi_version(void) { return GRIP_ABI_VERSION; }
const char* grip_last_error(void) { return g_err.c_str(); }

int grip_create(const GripSceneDesc* d, int device, GripBatch** out) {
  if (!d || !out) {
    g_err = "null argument";
    return -1;
  }
  if (d->abi_version != GRIP_ABI_VERSION) {
    g_err = "ABI version mismatch";
    return -1;
  }
  CK(cudaSetDevice(device));
  GripBatch* b = new GripBatch();
  b->device = device;
  CK(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
  b->own_stream = b->stream;
  CK(cudaStreamCreateWithFlags(&b->aux, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&b->aux2, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&b->ev_abd, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&b->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&b->ev_join, cudaEventDisableTiming));
  CK(cudaEventCreate(&b->ev0));
  CK(cudaEventCreate(&b->ev1));
  const int E = d->n_env;
  b->n_env = E;
  auto vec = [&](const int32_t* p) { return std::vector<int>(p, p + E + 1); };
  b->node_off = vec(d->node_off);
  b->sv_off = vec(d->sv_off);
  b->tri_off = vec(d->tri_off);
  b->edge_off = vec(d->edge_off);
  b->tet_off = vec(d->tet_off);
  b->abd_off = vec(d->abd_off);
  b->body_off = vec(d->body_off);
  const int NN = b->node_off[E], NS = b->sv_off[E], NTR = b->tri_off[E], NE = b->edge_off[E], NTET = b->tet_off[E],
            NA = b->abd_off[E], NB = b->body_off[E];
  b->n_node = NN; b->n_sv = NS; b->n_tet = NTET; b->n_abd = NA; b->n_body = NB;
  Dev& D = b->D;
  D.n_env = E;
  int max_sv = 1, max_tri = 1, max_edge = 1, max_tet = 1, max_abd = 1, max_node = 1;
  for (int e = 0; e < E; ++e) {
    max_sv = std::max(max_sv, b->sv_off[e + 1] - b->sv_off[e]);
    max_tri = std::max(max_tri, b->tri_off[e + 1] - b->tri_off[e]);
    max_edge = std::max(max_edge, b->edge_off[e + 1] - b->edge_off[e]);
    max_tet = std::max(max_tet, b->tet_off[e + 1] - b->tet_off[e]);
    max_abd = std::max(max_abd, b->abd_off[e + 1] - b->abd_off[e]);
    max_node = std::max(max_node, b->node_off[e + 1] - b->node_off[e]);
  }
  // ---- free nodes, static block structure, gradient incidence (host) ----
  std::vector<int> node_fidx(NN, -1), free_off(E + 1, 0), free_node;
  int max_free = 1;
  for (int e = 0; e < E; ++e) {
    int f = 0;
    for (int n = b->node_off[e]; n < b->node_off[e + 1]; ++n)
      if (d->node_free[n]) {
        node_fidx[n] = f++;
        free_node.push_back(n - b->node_off[e]);
      }
    free_off[e + 1] = free_off[e] + f;
    max_free = std::max(max_free, f);
  }
  const int NF = free_off[E];
  b->n_free = NF;
  // dense-solve ordering: free nodes grouped by body, bodies with the fewest DOF-carrying collision
  // partners first and the hub (e.g. the grasped object every pad touches) last, so pad-pad blocks
  // stay structurally zero in the Cholesky factor
  std::vector<int> dense_perm(std::max(NF, 1), 0);
  for (int e = 0; e < E; ++e) {
    const int b0 = b->body_off[e], nb = b->body_off[e + 1] - b0;
    std::vector<int> partners(nb, 0);
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < nb; ++j)
        if (i != j && ((d->body_pairmask[b0 + i] >> j) & 1u) && d->body_kind[b0 + j] != 2) partners[i]++;
    std::vector<int> order(nb);
    for (int i = 0; i < nb; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
      if (partners[x] != partners[y]) return partners[x] < partners[y];
      return x > y;
    });
    // within a soft body: reverse Cuthill-McKee on the tet graph of its free nodes (small
    // envelope for the skyline Cholesky); affine bodies keep their [t, A rows] node order
    const int n0 = b->node_off[e], nn = b->node_off[e + 1] - n0;
    std::vector<std::vector<int>> nbr(nn);
    for (int t = b->tet_off[e]; t < b->tet_off[e + 1]; ++t) {
      const int* tn = d->tet_nodes + 4 * (size_t)t;
      for (int a = 0; a < 4; ++a)
        for (int c = 0; c < 4; ++c)
          if (a != c && node_fidx[n0 + tn[a]] >= 0 && node_fidx[n0 + tn[c]] >= 0) nbr[tn[a]].push_back(tn[c]);
    }
    for (auto& v : nbr) {
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
    }
    int pos = 0;
    for (int bi : order) {
      std::vector<int> nodes;
      for (int n = 0; n < nn; ++n)
        if (node_fidx[n0 + n] >= 0 && d->node_body[n0 + n] == bi) nodes.push_back(n);
      if (d->body_kind[b0 + bi] == 0) {
        std::vector<int> cm, mark(nn, 0);
        auto deg = [&](int n) { return (int)nbr[n].size(); };
        for (;;) {
          int start = -1;
          for (int n : nodes)
            if (!mark[n] && (start < 0 || deg(n) < deg(start))) start = n;
          if (start < 0) break;
          size_t head = cm.size();
          cm.push_back(start);
          mark[start] = 1;
          while (head < cm.size()) {
            const int u = cm[head++];
            std::vector<int> nx;
            for (int w : nbr[u])
              if (!mark[w] && d->node_body[n0 + w] == bi) { mark[w] = 1; nx.push_back(w); }
            std::stable_sort(nx.begin(), nx.end(), [&](int x, int y) { return deg(x) < deg(y); });
            cm.insert(cm.end(), nx.begin(), nx.end());
          }
        }
        nodes.assign(cm.rbegin(), cm.rend());
      }
      for (int n : nodes) dense_perm[free_off[e] + node_fidx[n0 + n]] = pos++;
    }
  }
  std::vector<int> sb_rowptr(NF + 1, 0), sb_col, sb_diag(NF, -1), sbc_ptr(1, 0), sbc;
  std::vector<int> tinc_ptr(NN + 1, 0), tinc;
  {
    std::vector<std::vector<std::pair<int, int>>> tin(NN);  // per global node: (slot, k)
    for (int e = 0; e < E; ++e) {
      const int n0 = b->node_off[e];
      const int nf = free_off[e + 1] - free_off[e];
      // per free row: map col -> list of contribution codes
      std::vector<std::vector<std::pair<int, std::vector<int>>>> rows(nf);
      auto add = [&](int rn, int cn, int code) {
        const int fr = node_fidx[n0 + rn], fc = node_fidx[n0 + cn];
        if (fr < 0 || fc < 0) return;
        auto& R = rows[fr];
        for (auto& pr : R)
          if (pr.first == fc) {
            pr.second.push_back(code);
            return;
          }
        R.push_back({fc, {code}});
      };
      for (int t = 0; t < b->tet_off[e + 1] - b->tet_off[e]; ++t) {
        const int* tn = d->tet_nodes + 4 * (size_t)(b->tet_off[e] + t);
        for (int a = 0; a < 4; ++a) {
          tin[n0 + tn[a]].push_back({t, a});
          for (int c = 0; c < 4; ++c) add(tn[a], tn[c], (t << 4) | (a << 2) | c);
        }
      }
      for (int j = 0; j < b->abd_off[e + 1] - b->abd_off[e]; ++j) {
        const int pn = d->abd_node[b->abd_off[e] + j];
        const int slot = max_tet + j;
        for (int a = 0; a < 4; ++a) {
          tin[n0 + pn + a].push_back({slot, a});
          for (int c = 0; c < 4; ++c) add(pn + a, pn + c, (slot << 4) | (a << 2) | c);
        }
      }
      for (int f = 0; f < nf; ++f) {  // every free row has its diagonal (mass)
        const int n = free_node[free_off[e] + f];
        add(n, n, -1);
      }
      for (int f = 0; f < nf; ++f) {
        auto& R = rows[f];
        std::sort(R.begin(), R.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        const int fg = free_off[e] + f;
        for (auto& pr : R) {
          if (pr.first == f) sb_diag[fg] = (int)sb_col.size();
          sb_col.push_back(pr.first);
          for (int code : pr.second)
            if (code >= 0) sbc.push_back(code);
          sbc_ptr.push_back((int)sbc.size());
        }
        sb_rowptr[fg + 1] = (int)sb_col.size();
      }
    }
    for (int n = 0; n < NN; ++n) {
      for (auto& pr : tin[n]) tinc.push_back((pr.first << 2) | pr.second);
      tinc_ptr[n + 1] = (int)tinc.size();
    }
  }
  b->n_blk = (int)sb_col.size();
  // skyline (envelope) data for the direct solve: block -> row, per dense position the lowest
  // dense position it couples to statically; the shared-memory envelope capacity assumes the
  // hub rows (last body) fill up through contact
  std::vector<int> sb_row(std::max((int)sb_col.size(), 1), 0), dense_fc(std::max(NF, 1), 0), dense_tail(E, 0);
  size_t env_need = 0;
  for (int e = 0; e < E; ++e) {
    const int f0 = free_off[e], nf = free_off[e + 1] - f0;
    if (nf == 0) continue;
    const int* pm = dense_perm.data() + f0;
    int hub_pos = nf;   // first dense position of the last body
    {
      const int n0 = b->node_off[e];
      int last = -1;
      for (int f = 0; f < nf; ++f)
        if (pm[f] == nf - 1) last = d->node_body[n0 + free_node[f0 + f]];
      for (int f = 0; f < nf; ++f)
        if (d->node_body[n0 + free_node[f0 + f]] == last) hub_pos = std::min(hub_pos, pm[f]);
    }
    std::vector<int> fcn(nf);
    for (int f = 0; f < nf; ++f) {
      int m = pm[f];
      for (int q = sb_rowptr[f0 + f]; q < sb_rowptr[f0 + f + 1]; ++q) {
        sb_row[q] = f0 + f;
        m = std::min(m, pm[sb_col[q]]);
      }
      dense_fc[f0 + pm[f]] = m;
    }
    dense_tail[e] = hub_pos;
    for (int p = 0; p < nf; ++p) fcn[p] = p >= hub_pos ? 0 : dense_fc[f0 + p];
    size_t tot = 0;
    for (int i = 0; i < 3 * nf; ++i) tot += i - ((3 * fcn[i / 3]) & ~7) + 1;
    env_need = std::max(env_need, tot);
  }
  // ---- uploads ----
  D.node_off = b->upload(b->node_off.data(), E + 1);
  D.sv_off = b->upload(b->sv_off.data(), E + 1);
  D.tri_off = b->upload(b->tri_off.data(), E + 1);
  D.edge_off = b->upload(b->edge_off.data(), E + 1);
  D.tet_off = b->upload(b->tet_off.data(), E + 1);
  D.abd_off = b->upload(b->abd_off.data(), E + 1);
  D.body_off = b->upload(b->body_off.data(), E + 1);
  D.free_off = b->upload(free_off.data(), E + 1);
  D.node_M = b->upload(d->node_M, 9 * (size_t)NN);
  D.node_free = b->upload(d->node_free, NN);
  D.node_body = b->upload(d->node_body, NN);
  D.node_kind = b->upload(d->node_kind, NN);
  D.node_sv = b->upload(d->node_sv, NN);
  D.node_fidx = b->upload(node_fidx.data(), NN);
  D.free_node = b->upload(free_node.data(), std::max(NF, 1));
  D.dense_perm = b->upload(dense_perm.data(), std::max(NF, 1));
  D.dense_fc = b->upload(dense_fc.data(), std::max(NF, 1));
  {   // per surface vertex: (dense node position << 2 | kind), -1 when it carries no free DOF
    std::vector<int> sv_code(std::max(NS, 1), -1);
    for (int e = 0; e < E; ++e)
      for (int g = b->sv_off[e]; g < b->sv_off[e + 1]; ++g) {
        const int kind = d->sv_kind[g];
        if (kind == 2) continue;
        const int f = node_fidx[b->node_off[e] + d->sv_node[g]];
        if (f >= 0) sv_code[g] = (dense_perm[free_off[e] + f] << 2) | kind;
      }
    D.sv_code = b->upload(sv_code.data(), sv_code.size());
  }
  D.dense_tail = b->upload(dense_tail.data(), E);
  D.sb_row = b->upload(sb_row.data(), sb_row.size());
  {   // per static block: its dense (row node, column node) positions packed, -1 for upper-triangle
      // blocks (their mirror carries the values): one load per block in the skyline fill
    std::vector<int> sb_dst(sb_row.size(), -1);
    for (int e = 0; e < E; ++e) {
      const int f0 = free_off[e];
      for (int q = sb_rowptr[f0]; q < sb_rowptr[free_off[e + 1]]; ++q) {
        const int pf = dense_perm[sb_row[q]], pf2 = dense_perm[f0 + sb_col[q]];
        if (pf2 <= pf) sb_dst[q] = (pf << 16) | pf2;
      }
    }
    D.sb_dst = b->upload(sb_dst.data(), sb_dst.size());
  }
  D.sv_kind = b->upload(d->sv_kind, NS);
  D.sv_node = b->upload(d->sv_node, NS);
  D.sv_xi = b->upload(d->sv_xi, 3 * (size_t)NS);
  D.sv_body = b->upload(d->sv_body, NS);
  D.tris = b->upload(d->tris, 3 * (size_t)NTR);
  D.edges = b->upload(d->edges, 2 * (size_t)NE);
  D.edge_rest_sq = b->upload(d->edge_rest_sq, NE);
  D.tet_nodes = b->upload(d->tet_nodes, 4 * (size_t)NTET);
  D.tet_Dmi = b->upload(d->tet_Dmi, 9 * (size_t)NTET);
  D.tet_V0 = b->upload(d->tet_V0, NTET);
  D.tet_mu = b->upload(d->tet_mu, NTET);
  D.tet_lam = b->upload(d->tet_lam, NTET);
  {
    std::vector<double> eye(81 * (size_t)std::max(NTET, 1), 0.0);
    for (int t = 0; t < std::max(NTET, 1); ++t)
      for (int k = 0; k < 9; ++k) eye[81 * (size_t)t + 10 * k] = 1.0;
    eye.resize(2 * eye.size(), 0.0);   // both warm-start halves (Dev::tet_eig)
    for (size_t q = eye.size() / 2; q < eye.size(); ++q) eye[q] = eye[q - eye.size() / 2];
    D.tet_eig = b->upload(eye.data(), eye.size());
    D.eig_half = eye.size() / 2;
  D.tet_S = b->alloc<double>(45 * (size_t)std::max(NTET, 1));
  D.tet_W = b->alloc<double>(90 * (size_t)std::max(NTET, 1));
  {
    std::vector<int> z(std::max(E, 1), 0);
    D.eig_par = b->upload(z.data(), z.size());
    D.eig_swept = b->upload(z.data(), z.size());
  }
  D.jac_list = b->alloc<int2>((size_t)std::max(NTET, 1));
  D.jac_n = b->alloc<int>(1);
  }
  D.abd_node = b->upload(d->abd_node, NA);
  D.abd_kV = b->upload(d->abd_kV, NA);
  D.body_kind = b->upload(d->body_kind, NB);
  D.body_mu = b->upload(d->body_mu, NB);
  D.body_pairmask = b->upload(d->body_pairmask, NB);
  D.body_vel = b->upload(d->body_vel0, 3 * (size_t)NB);
  D.body_tri_lo = b->upload(d->body_tri_lo, NB);
  D.body_tri_hi = b->upload(d->body_tri_hi, NB);
  D.body_edge_lo = b->upload(d->body_edge_lo, NB);
  D.body_edge_hi = b->upload(d->body_edge_hi, NB);
  D.gravity = b->upload(d->env_gravity, 3 * (size_t)E);
  D.params = b->upload(d->env_params, (size_t)GRIP_NPARAM * E);
  D.cell_hint = b->upload(d->env_cell_hint, E);
  D.sb_rowptr = b->upload(sb_rowptr.data(), NF + 1);
  D.sb_col = b->upload(sb_col.data(), sb_col.size());
  D.sb_diag = b->upload(sb_diag.data(), std::max(NF, 1));
  D.sbc_ptr = b->upload(sbc_ptr.data(), sbc_ptr.size());
  D.sbc = b->upload(sbc.data(), sbc.size());
  D.tinc_ptr = b->upload(tinc_ptr.data(), NN + 1);
  D.tinc = b->upload(tinc.data(), tinc.size());
  // state
  D.x = b->upload(d->node_x0, 3 * (size_t)NN);
  D.v = b->alloc<double>(3 * (size_t)NN);
  D.x_t = b->alloc<double>(3 * (size_t)NN);
  D.xhat = b->alloc<double>(3 * (size_t)NN);
  D.pdir = b->alloc<double>(3 * (size_t)NN);
  D.sv_pos = b->alloc<double>(3 * (size_t)NS);
  D.surf_prev = b->alloc<double>(3 * (size_t)NS);
  D.kin_pos = b->upload(d->sv_kin0, 3 * (size_t)NS);
  D.sv_disp = b->alloc<double>(3 * (size_t)NS);
  D.ell = b->alloc<double>(E);
  D.tol = b->alloc<double>(E);
  D.residual = b->alloc<double>(E);
  D.energy = b->alloc<double>(E);
  D.min_dist = b->alloc<double>(E);
  D.time = b->alloc<double>(E);
  int maxit = 1;
  for (int e = 0; e < E; ++e) maxit = std::max(maxit, (int)d->env_params[(size_t)e * GRIP_NPARAM + GRIP_P_MAXIT]);
  b->max_it = maxit;
  D.max_alpha = maxit + 1;
  D.alphas = b->alloc<double>((size_t)E * D.max_alpha);
  D.iters = b->alloc<int>(E);
  D.ns_status = b->alloc<int>(E);
  D.reason = b->alloc<int>(E);
  D.regularized = b->alloc<int>(E);
  D.kin_blocked = b->alloc<int>(E);
  D.needs_ls = b->alloc<int>(E);
  D.ns_done = b->alloc<int>(E);
  D.flags = b->alloc<int>(E);
  D.step_index = b->alloc<int>(E);
  D.newton_calls = b->alloc<int>(E);
  D.pcg_iters = b->alloc<int>(E);
  D.fin_done = b->alloc<int>(E);
  D.body_force = b->alloc<double>(NB);
  D.contact_mask = b->alloc<unsigned int>(NB);
  D.body_com = b->alloc<double>(3 * (size_t)NB);
  D.max_speed = b->alloc<double>(E);
  D.min_J = b->alloc<double>(E);
  D.stats = b->alloc<double>(8);
  D.cs_n = b->alloc<int>(2 * (size_t)E);
  D.cs_R = b->alloc<double>(E);
  D.ss_k = getenv("GRIP_SS_K") ? atof(getenv("GRIP_SS_K")) : 0.0;
  if (getenv("GRIP_EGRID")) {
    float m[4] = {2, 2, 2, 4};
    sscanf(getenv("GRIP_EGRID"), "%f,%f,%f,%f", &m[0], &m[1], &m[2], &m[3]);
    for (int k = 0; k < 4; ++k) b->eg[k] = std::max(1, (int)(148 * m[k] + 0.5f));
  }
  D.bp_mode = (getenv("GRIP_BP") && std::string(getenv("GRIP_BP")) == "grid") ? 1 : 0;
  D.bp_qm_min = 1 << 30;   // measured: plain cost comparison is best (GRIP_BP_QM to experiment)
  D.bp_qm_fac = 1.0f;
  if (getenv("GRIP_BP_QM")) sscanf(getenv("GRIP_BP_QM"), "%d,%f", &D.bp_qm_min, &D.bp_qm_fac);
  D.cs_valid = b->alloc<int>(E);
  D.cs_drift = b->alloc<double>(E);
  D.ss_skin = getenv("GRIP_SKIN") ? atof(getenv("GRIP_SKIN")) : 2.0;   // measured: 0 -> 61.1k, 2 -> 63.5k
  D.md_prev = b->alloc<double>(E);
  D.md_kin = b->alloc<double>(E);
  D.bp_lc = b->alloc<int>((size_t)E * 3 * std::max(max_tri, max_edge));
  D.need = b->alloc<unsigned>(4);
  D.cand_done = b->alloc<unsigned>(1);
  D.c1_n = b->alloc<int>(2 * (size_t)E);
  D.c2_n = b->alloc<int>(2 * (size_t)E);
  D.n_act = b->alloc<int>(E);
  D.n_anc = b->alloc<int>(E);
  D.tflag = b->alloc<int>(E);
  D.work_off = b->alloc<int>(E + 1);
  D.cwork_off = b->alloc<int>(E + 1);
  D.asm_key = b->alloc<int>(E + 1);
  D.asm_order = b->alloc<int>(E + 1);
  D.twork_off = b->alloc<int>(E + 1);
  D.ev_n = b->alloc<int>(E);
  D.ev_on = 0;
  D.swork_off = b->alloc<int>(E + 1);
  D.max_sv = max_sv; D.max_tri = max_tri; D.max_edge = max_edge; D.max_free = max_free;
  D.max_node = max_node; D.max_tet = max_tet; D.max_abd = max_abd;
  D.cap_pt = std::max(2048, 16 * max_sv);
  D.cap_ee = std::max(4096, 16 * max_edge);
  D.cap_act = 512;
  D.cap_anc = 512;
  D.cap_cells = 32 * std::max(max_tri, max_edge) + 4096;
  if (getenv("GRIP_SMALL_CAPS")) {   // test hook: start tiny so every growth / redo path runs
    D.cap_pt = D.cap_ee = 8;
    D.cap_act = D.cap_anc = 4;
    D.cap_cells = 64;
  }
  D.bp_aabb = b->alloc<double>((size_t)E * 6 * std::max(max_tri, max_edge));
  D.bp_scr = b->alloc<int>((size_t)E * (4 * std::max(max_tri, max_edge) + max_sv));
  D.bp_cnt = b->alloc<int>((size_t)E * (std::max(max_sv, max_edge) + 1));
  D.pcg_x = b->alloc<double>((size_t)E * 3 * max_free);
  D.pcg_r = b->alloc<double>((size_t)E * 3 * max_free);
  D.pcg_z = b->alloc<double>((size_t)E * 3 * max_free);
  D.pcg_p = b->alloc<double>((size_t)E * 3 * max_free);
  D.pcg_q = b->alloc<double>((size_t)E * 3 * max_free);
  D.pcg_b = b->alloc<double>((size_t)E * 3 * max_free);
  D.pcg_pinv = b->alloc<double>(9 * (size_t)std::max(NF, 1));
  D.abd_pinv = b->alloc<double>(144 * (size_t)std::max(NA, 1));
  D.sb_val = b->alloc<double>(9 * (size_t)std::max(b->n_blk, 1));
  {
    // direct solve storage: the skyline of H_ff in shared memory (capacity env_cap doubles, sized
    // from the static envelope + 15%); an env whose envelope outgrows it this iteration uses its
    // global slot (full packed triangle, so any envelope fits)
    const int nd = 3 * max_free;
    const size_t packed = (size_t)nd * (nd + 1) / 2;
    int dev_smem = 0;
    cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    const size_t aux = dir_aux_bytes(nd, max_free);
    const size_t avail = (size_t)dev_smem - sizeof(DirShared) - 1024 - aux;
    size_t cap = std::min(packed, (env_need * 115 / 100 + 63) / 64 * 64);
    if (getenv("GRIP_DENSE_GLOBAL")) cap = 0;
    cap = std::min(cap, avail / sizeof(double));
    b->env_cap = (int)cap;
    b->dyn_smem = aux + cap * sizeof(double);
    D.dense_stride = packed;
    D.dense_L = b->alloc<double>(packed * (size_t)E);
    CK(cudaFuncSetAttribute(k_assemble_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b->dyn_smem));
  }
  D.c_u = b->alloc<double>((size_t)E * 3 * max_sv);
  D.c_w = b->alloc<double>((size_t)E * 3 * max_sv);
  D.ls_y = b->alloc<double>((size_t)E * LS_NA * 3 * max_sv);
  D.sv_g = b->alloc<double>((size_t)E * 3 * max_sv);
  D.inc_ptr = b->alloc<int>((size_t)E * (max_sv + 1));
  D.dense_k = b->direct ? 1 : 0;
  if (alloc_dynamic(b, false, 0)) return -1;
  b->tet_env.resize(NTET);
  for (int e = 0; e < E; ++e)
    for (int t = b->tet_off[e]; t < b->tet_off[e + 1]; ++t) b->tet_env[t] = e;
  b->d_tet_env = b->upload(b->tet_env.data(), std::max(NTET, 1));
  b->d_list = b->alloc<int>(E + 1);
  b->d_list2 = b->alloc<int>(E + 1);
  CK(cudaMallocHost(&b->h_pin, 64 * sizeof(int)));
  CK(cudaMallocHost(&b->h_lists, 2 * sizeof(int) * std::max(b->n_env, 1)));
  {
    const size_t E = std::max(b->n_env, 1), NBd = std::max(b->n_body, 1), A = std::max(b->D.max_alpha, 1);
    const size_t bytes = 10 * 4 * E + (8 * E + A * E + NBd + 3 * NBd) * 8 + 4 * NBd + 64;
    CK(cudaMallocHost(&b->h_snap, bytes));
    char* q = b->h_snap;
    auto take = [&](auto*& ptr, size_t n) {
      using T = std::remove_reference_t<decltype(*ptr)>;
      q = (char*)(((uintptr_t)q + 7) & ~(uintptr_t)7);
      ptr = reinterpret_cast<T*>(q);
      q += n * sizeof(T);
    };
    take(b->s_res, E); take(b->s_md, E); take(b->s_en, E); take(b->s_tm, E); take(b->s_alpha, A * E);
    take(b->s_force, NBd); take(b->s_com, 3 * NBd); take(b->s_speed, E);
    take(b->s_flags, E); take(b->s_done, E); take(b->s_st, E); take(b->s_rs, E); take(b->s_it, E); take(b->s_kb, E);
    take(b->s_rg, E); take(b->s_si, E); take(b->s_nc, E); take(b->s_pi, E); take(b->s_cmask, NBd);
  }
#ifdef GRIP_CTA_TIMING
  D.cta_cap = 1u << 21;
  D.cta_rec = b->alloc<unsigned long long>(4 * (size_t)D.cta_cap);
  D.cta_n = b->alloc<unsigned int>(1);
#endif
  for (void* p : b->owned)
    if (!p) {
      g_err = "out of device memory";
      return -1;
    }
  {
    // every pointer member of Dev must be set (catches a forgotten allocation at create time)
    const void* ptrs[] = {
        D.node_off, D.sv_off, D.tri_off, D.edge_off, D.tet_off, D.abd_off, D.body_off, D.free_off, D.node_M,
        D.node_free, D.node_body, D.node_kind, D.node_sv, D.node_fidx, D.free_node, D.sv_kind, D.sv_node, D.sv_xi,
        D.sv_body, D.tris, D.edges, D.edge_rest_sq, D.tet_nodes, D.tet_Dmi, D.tet_V0, D.tet_mu, D.tet_lam, D.abd_node,
        D.abd_kV, D.body_kind, D.body_mu, D.body_pairmask, D.body_vel, D.gravity, D.params, D.cell_hint, D.sb_rowptr,
        D.sb_col, D.sb_diag, D.sbc_ptr, D.sbc, D.tinc_ptr, D.tinc, D.x, D.v, D.x_t, D.xhat, D.pdir, D.sv_pos,
        D.surf_prev, D.kin_pos, D.sv_disp, D.ell, D.tol, D.residual, D.energy, D.alphas, D.min_dist, D.time, D.iters,
        D.ns_status, D.reason, D.regularized, D.kin_blocked, D.needs_ls, D.ns_done, D.flags, D.step_index,
        D.newton_calls, D.pcg_iters, D.body_force, D.contact_mask, D.c1_pt, D.c1_ee, D.c1_eid, D.c1_n, D.c2_pt,
        D.c2_ee, D.c2_eid, D.c2_n, D.act, D.n_act, D.n_anc, D.el_E, D.el_g, D.el_H, D.el_idx, D.tflag, D.work_off, D.cwork_off, D.twork_off, D.swork_off, D.anc_v,
        D.anc_gamma, D.anc_T, D.anc_lam, D.anc_mu, D.anc_b, D.ev_i, D.ev_d, D.ev_n, D.bp_cells, D.bp_scr, D.need, D.cand_done, D.bp_aabb, D.bp_cnt, D.bp_tmp, D.pcg_x,
        D.pcg_r, D.pcg_z, D.pcg_p, D.pcg_q, D.pcg_b, D.pcg_pinv, D.abd_pinv, D.sb_val, D.c_u, D.c_w, D.ls_y, D.c_r,
        D.inc_ptr, D.inc, D.sv_g, D.body_com, D.max_speed, D.min_J, D.stats, D.fin_done, D.cs_pt, D.cs_ee, D.cs_eid,
        D.cs_n, D.cs_R, D.cs_valid, D.cs_drift, D.md_prev, D.md_kin, D.bp_lc, D.dense_L, D.tet_eig, D.body_tri_lo,
        D.body_tri_hi, D.body_edge_lo, D.body_edge_hi, D.dense_perm, D.dense_fc, D.dense_tail, D.sb_row, D.sb_dst, D.el_K, D.el_kn, D.sc_lst, D.sc_off, D.sv_code, D.tet_S, D.tet_W, D.jac_list, D.jac_n, D.cjac_S, D.cjac_W, D.cjac_list, D.cjac_n, D.eig_par, D.eig_swept, D.asm_key, D.asm_order};
    for (size_t i = 0; i < sizeof(ptrs) / sizeof(ptrs[0]); ++i)
      if (!ptrs[i]) {
        g_err = "internal: device buffer " + std::to_string(i) + " not allocated";
        return -1;
      }
  }
  CK(cudaStreamSynchronize(b->stream));
  CK(cudaGetLastError());
  *out = b;
  return 0;
}

// host-side time split of grip_round (GRIP_TRACE_HOST=1 prints it at grip_destroy)
static double g_host_enq = 0.0, g_host_wait = 0.0, g_host_post = 0.0;
static long long g_host_rounds = 0;
static double host_now() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int grip_destroy(GripBatch* b) {
  if (!b) return 0;
  if (getenv("GRIP_TRACE_HOST") && g_host_rounds)
    fprintf(stderr, "GRIP_TRACE_HOST rounds %lld enqueue %.3f ms wait %.3f ms post %.3f ms (per round)\n", g_host_rounds,
            g_host_enq / g_host_rounds, g_host_wait / g_host_rounds, g_host_post / g_host_rounds);
  cudaStreamSynchronize(b->stream);
  for (void* p : b->owned) cudaFree(p);
  for (auto ev : b->kev) cudaEventDestroy(ev);
  if (b->r0) cudaEventDestroy(b->r0);
  if (b->r1) cudaEventDestroy(b->r1);
  if (b->h_pin) cudaFreeHost(b->h_pin);
  if (b->h_lists) cudaFreeHost(b->h_lists);
  if (b->h_snap) cudaFreeHost(b->h_snap);
  if (b->h_frame) cudaFreeHost(b->h_frame);
  if (b->h_fmask) cudaFreeHost(b->h_fmask);
  for (auto& rs : b->rslot) {
    if (rs.h) cudaFreeHost(rs.h);
    if (rs.ev) cudaEventDestroy(rs.ev);
  }
  for (auto& g : b->rgraph)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (b->ev_reset_st) cudaEventDestroy(b->ev_reset_st);
  if (b->ev_pinit_st) cudaEventDestroy(b->ev_pinit_st);
  if (b->h_reset) cudaFreeHost(b->h_reset);
  if (b->h_pinit) cudaFreeHost(b->h_pinit);
  if (b->d_pinit) cudaFree(b->d_pinit);
  if (b->d_reset) cudaFree(b->d_reset);
  cudaEventDestroy(b->ev0);
  cudaEventDestroy(b->ev1);
  cudaStreamDestroy(b->own_stream);   // a caller's stream (grip_set_stream) is the caller's
  cudaStreamDestroy(b->aux);
  cudaStreamDestroy(b->aux2);
  cudaEventDestroy(b->ev_abd);
  cudaEventDestroy(b->ev_fork);
  cudaEventDestroy(b->ev_join);
  delete b;
  return 0;
}

int grip_set_controls(GripBatch* b, const double* gravity, const double* body_vel) {
  if (gravity) CK(cudaMemcpyAsync(b->D.gravity, gravity, 3 * sizeof(double) * b->n_env, cudaMemcpyHostToDevice, b->stream));
  if (body_vel)
    CK(cudaMemcpyAsync(b->D.body_vel, body_vel, 3 * sizeof(double) * b->n_body, cudaMemcpyHostToDevice, b->stream));
  return 0;
}

static std::vector<int> mask_to_list(const GripBatch* b, const uint8_t* m) {
  std::vector<int> L;
  for (int e = 0; e < b->n_env; ++e)
    if (!m || m[e]) L.push_back(e);
  return L;
}

int grip_begin_step(GripBatch* b, const uint8_t* active) {
  b->snap_valid = false;
  std::vector<int> L = mask_to_list(b, active);
  if (L.empty()) return 0;
  if (upload_list(b, L, b->d_list)) return -1;
  const int n = (int)L.size();
  return run_with_growth(b, n, [&] { k_begin<<<n * BP_CL, NT, 0, b->stream>>>(b->D, b->d_list); });
}

// kernel ids for grip_kernel_stats
enum { K_BEGIN = 0, K_CAND, K_SCAN, K_ELEM, K_ASM, K_LS, K_FIN, K_TET };

// a timing event: inside a captured round graph it must be an external record (a real event
// node, not only a dependency); outside a capture that flag is illegal
static void kt_record(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  else cudaEventRecord(ev, st);
}
static int kt_begin(GripBatch* b, int kid, cudaStream_t st = nullptr) {
  if (!b->prof) return -1;
  int pair;
  if (!b->kev_free.empty()) {
    pair = b->kev_free.back();
    b->kev_free.pop_back();
  } else {
    pair = (int)b->kev.size() / 2;
    for (int k = 0; k < 2; ++k) {
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      b->kev.push_back(ev);
    }
  }
  kt_record(b->kev[2 * pair], st ? st : b->stream);
  b->pending_k.push_back({kid, pair});
  return pair;
}
static void kt_end(GripBatch* b, int pair, cudaStream_t st = nullptr) {
  if (pair >= 0) kt_record(b->kev[2 * pair + 1], st ? st : b->stream);
}
// fold the recorded launch times into the per-kernel totals: the first `upto` pending launches
// (all when negative), which must have completed
static void kt_collect(GripBatch* b, int n_listed = -1, long long upto = -1) {
  static const bool trace = getenv("GRIP_TRACE") != nullptr;
  double per[GripBatch::NK] = {0};
  const size_t m = upto < 0 ? b->pending_k.size() : std::min((size_t)upto, b->pending_k.size());
  for (size_t i = 0; i < m; ++i) {
    const auto& pk = b->pending_k[i];
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, b->kev[2 * pk.second], b->kev[2 * pk.second + 1]) != cudaSuccess) {
      (void)cudaGetLastError();   // a timing gap, never an error of the product path
      ms = 0.0f;
    }
    b->k_ms[pk.first] += ms;
    b->k_n[pk.first] += 1;
    per[pk.first] += ms;
    if ((size_t)pk.second >= b->kev_owned.size() || !b->kev_owned[pk.second]) b->kev_free.push_back(pk.second);
  }
  if (trace && n_listed >= 0 && m)
    fprintf(stderr, "GRIP_TRACE n=%d cand=%.3f elem=%.3f asm=%.3f ls=%.3f\n", n_listed, per[1], per[3], per[4], per[5]);
  b->pending_k.erase(b->pending_k.begin(), b->pending_k.begin() + m);
  for (auto& rs : b->rslot)
    if (rs.busy) rs.kt_mark = rs.kt_mark > m ? rs.kt_mark - m : 0;
}

// one Newton sweep over the pending envs (list in b->d_list, n entries); returns new pending count
static void sweep_launch(GripBatch* b, int n, const int* list);

static int newton_sweep(GripBatch* b, int n, int* n_out) {
  Dev& D = b->D;
  for (int attempt = 0; attempt < 8; ++attempt) {
    sweep_launch(b, n, b->d_list);
    CK(cudaGetLastError());
    std::vector<int> fl(b->n_env);
    CK(cudaMemcpyAsync(fl.data(), D.flags, sizeof(int) * b->n_env, cudaMemcpyDeviceToHost, b->stream));
    std::vector<int> done(b->n_env);
    CK(cudaMemcpyAsync(done.data(), D.ns_done, sizeof(int) * b->n_env, cudaMemcpyDeviceToHost, b->stream));
    std::vector<int> L(n);
    CK(cudaMemcpyAsync(L.data(), b->d_list, sizeof(int) * n, cudaMemcpyDeviceToHost, b->stream));
    CK(cudaStreamSynchronize(b->stream));
    kt_collect(b, n);
    bool ov = false;
    for (int i = 0; i < n; ++i) ov |= (fl[L[i]] & FLAG_OVERFLOW) != 0;
    if (ov) {
      if (grow(b)) return -1;
      CK(cudaMemsetAsync(D.flags, 0, sizeof(int) * b->n_env, b->stream));
      // the overflowed envs did not move; sweep again with the same pending list
      std::vector<int> keep;
      for (int i = 0; i < n; ++i)
        if (!done[L[i]]) keep.push_back(L[i]);
      if (upload_list(b, keep, b->d_list)) return -1;
      n = (int)keep.size();
      if (n == 0) { *n_out = 0; return 0; }
      continue;
    }
    std::vector<int> keep;
    for (int i = 0; i < n; ++i)
      if (!done[L[i]]) keep.push_back(L[i]);
    if (upload_list(b, keep, b->d_list)) return -1;
    *n_out = (int)keep.size();
    return 0;
  }
  g_err = "buffer growth did not converge";
  return -1;
}

int grip_newton_iteration(GripBatch* b, uint8_t* pending) {
  b->snap_valid = false;
  std::vector<int> L = mask_to_list(b, pending);
  if (L.empty()) return 0;
  if (upload_list(b, L, b->d_list)) return -1;
  int n2 = 0;
  if (newton_sweep(b, (int)L.size(), &n2)) return -1;
  std::vector<int> done(b->n_env);
  CK(cudaMemcpy(done.data(), b->D.ns_done, sizeof(int) * b->n_env, cudaMemcpyDeviceToHost));
  for (int e = 0; e < b->n_env; ++e)
    if (pending[e] && done[e]) pending[e] = 0;
  return 0;
}

static int read_reports(GripBatch* b, const std::vector<int>& L, GripStepReport* reports, double* alphas) {
  const int E = b->n_env;
  Dev& D = b->D;
  std::vector<int> st(E), rs(E), it(E), kb(E), rg(E), si(E), nc(E), pi(E);
  std::vector<double> res(E), md(E), en(E), tm(E);
  CK(cudaMemcpyAsync(st.data(), D.ns_status, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(rs.data(), D.reason, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(it.data(), D.iters, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(kb.data(), D.kin_blocked, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(rg.data(), D.regularized, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(si.data(), D.step_index, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(nc.data(), D.newton_calls, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(pi.data(), D.pcg_iters, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(res.data(), D.residual, sizeof(double) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(md.data(), D.min_dist, sizeof(double) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(en.data(), D.energy, sizeof(double) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(tm.data(), D.time, sizeof(double) * E, cudaMemcpyDeviceToHost, b->stream));
  if (alphas)
    CK(cudaMemcpyAsync(alphas, D.alphas, sizeof(double) * (size_t)E * D.max_alpha, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  const double* P = nullptr;
  (void)P;
  for (int e : L) {
    GripStepReport& r = reports[e];
    r.status = st[e];
    r.reason = rs[e];
    r.iterations = it[e];
    r.n_alphas = std::min(it[e], D.max_alpha);
    r.residual = res[e];
    r.min_distance = md[e];
    r.energy = en[e];
    r.step_index = si[e] - 1;
    r.time = tm[e];
    r.kinematic_blocked = kb[e];
    r.regularized = rg[e];
    r.newton_calls = nc[e];
    r.pcg_iters = pi[e];
  }
  return 0;
}

int grip_finalize_step(GripBatch* b, const uint8_t* active, GripStepReport* reports, double* alphas) {
  b->ev_now = false;   // a finalize rewrites (or, recording off, invalidates) the event rows
  b->snap_valid = false;
  std::vector<int> L = mask_to_list(b, active);
  if (L.empty()) return 0;
  if (upload_list(b, L, b->d_list)) return -1;
  const int n = (int)L.size();
  if (run_with_growth(b, n, [&] { k_finalize<<<n, NT, 0, b->stream>>>(b->D, b->d_list); })) return -1;
  if (reports) return read_reports(b, L, reports, alphas);
  return 0;
}

int grip_step(GripBatch* b, const uint8_t* active, GripStepReport* reports, double* alphas) {
  b->ev_now = false;   // a finalize rewrites (or, recording off, invalidates) the event rows
  b->snap_valid = false;
  std::vector<int> L = mask_to_list(b, active);
  if (L.empty()) return 0;
  const long long l0 = b->launches;
  CK(cudaEventRecord(b->ev0, b->stream));
  if (upload_list(b, L, b->d_list)) return -1;
  int n = (int)L.size();
  if (run_with_growth(b, n, [&] {
        int t = kt_begin(b, K_BEGIN);
        k_begin<<<n * BP_CL, NT, 0, b->stream>>>(b->D, b->d_list);
        kt_end(b, t);
      }))
    return -1;
  kt_collect(b);
  // envs that failed in begin_step are done
  std::vector<int> done(b->n_env);
  CK(cudaMemcpy(done.data(), b->D.ns_done, sizeof(int) * b->n_env, cudaMemcpyDeviceToHost));
  std::vector<int> P;
  for (int e : L)
    if (!done[e]) P.push_back(e);
  if (upload_list(b, P, b->d_list)) return -1;
  n = (int)P.size();
  while (n > 0) {
    int n2 = 0;
    if (newton_sweep(b, n, &n2)) return -1;
    n = n2;
  }
  if (upload_list(b, L, b->d_list)) return -1;
  n = (int)L.size();
  if (run_with_growth(b, n, [&] {
        int t = kt_begin(b, K_FIN);
        k_finalize<<<n, NT, 0, b->stream>>>(b->D, b->d_list);
        kt_end(b, t);
      }))
    return -1;
  kt_collect(b);
  CK(cudaEventRecord(b->ev1, b->stream));
  CK(cudaEventSynchronize(b->ev1));
  float ms = 0.0f;
  CK(cudaEventElapsedTime(&ms, b->ev0, b->ev1));
  b->last_ms = ms;
  (void)l0;
  if (reports) return read_reports(b, L, reports, alphas);
  return 0;
}

// the sweep kernels over a device list of n envs, no host synchronisation
static void sweep_launch(GripBatch* b, int n, const int* list) {
  Dev& D = b->D;
  // fork: the tet chain (energy, gradient, deflated Hessian, batched eigen-clamp) depends on x
  // only, so it runs on the second stream while the candidates and the contact / ABD / friction
  // elements run on the main one; they join before the assembly
  CK_VOID(cudaEventRecord(b->ev_fork, b->stream));
  CK_VOID(cudaStreamWaitEvent(b->aux, b->ev_fork, 0));
  CK_VOID(cudaStreamWaitEvent(b->aux2, b->ev_fork, 0));
  k_abd_w<<<(n + EW - 1) / EW, EW * 32, 0, b->aux2>>>(D, list, n);   // third stream: x only
  CK_VOID(cudaEventRecord(b->ev_abd, b->aux2));
  int t = kt_begin(b, K_TET, b->aux);
  k_tet_scan<<<1, NT, 0, b->aux>>>(D, list, n);
  k_tet_front<<<b->eg[0], TF, 0, b->aux>>>(D, list, n);
  k_tet_jacobi2<<<b->eg[2], TJ, 0, b->aux>>>(D.jac_list, D.jac_n, D.tet_S, D.tet_W);
  k_tet_back<<<b->eg[3], EW * 32, 0, b->aux>>>(D, D.jac_list, D.jac_n, D.tet_W);
  CK_VOID(cudaStreamWaitEvent(b->aux, b->ev_abd, 0));   // the ABD blocks, before the static sums
  k_static<<<148 * 4, NT, 0, b->aux>>>(D, list, n);
  kt_end(b, t, b->aux);
  CK_VOID(cudaEventRecord(b->ev_join, b->aux));
  t = kt_begin(b, K_CAND);
  D.launch_seq = ++b->seq_ctr;
  k_candidates<<<n * BP_CL, NT, 0, b->stream>>>(D, list);
  kt_end(b, t);
  t = kt_begin(b, K_ELEM);
  k_elements_w<<<b->eg[1], EW * 32, 0, b->stream>>>(D, list, n);
  k_tet_jacobi2<<<148, TJ, 0, b->stream>>>(D.cjac_list, D.cjac_n, D.cjac_S, D.cjac_W);
  k_tet_finish<<<148 * 2, EW * 32, 0, b->stream>>>(D, D.cjac_list, D.cjac_n, D.cjac_W, nullptr);
  kt_end(b, t);
  CK_VOID(cudaStreamWaitEvent(b->stream, b->ev_join, 0));   // join
  t = kt_begin(b, K_ASM);
  if (b->direct) {
    k_contact_K<<<148 * 2, KT, 0, b->stream>>>(D, list, n);
    D.launch_seq = ++b->seq_ctr;
    k_assemble_direct<<<n, NT, b->dyn_smem, b->stream>>>(D, D.asm_order, b->env_cap);   // heavy envs first
  } else {
    k_assemble_solve<<<n, NT, 0, b->stream>>>(D, list);
  }
  kt_end(b, t);
  t = kt_begin(b, K_LS);
  D.launch_seq = ++b->seq_ctr;
  k_linesearch<<<n * BP_CL, NT, 0, b->stream>>>(D, D.asm_order);   // heavy envs first
  kt_end(b, t);
  b->launches += 6 + 2 + 3 + (b->direct ? 2 : 1) + 1;
  b->sweeps += 1;
}

// queue the D2H copies of everything the host reads after a round into the pinned snapshot
static int snapshot_async(GripBatch* b) {
  Dev& D = b->D;
  const size_t E = b->n_env, NBd = b->n_body;
  auto cp = [&](void* dst, const void* src, size_t bytes) {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, b->stream);
  };
  CK(cp(b->s_flags, D.flags, 4 * E));
  CK(cp(b->s_done, D.ns_done, 4 * E));
  CK(cp(b->s_st, D.ns_status, 4 * E));
  CK(cp(b->s_rs, D.reason, 4 * E));
  CK(cp(b->s_it, D.iters, 4 * E));
  CK(cp(b->s_kb, D.kin_blocked, 4 * E));
  CK(cp(b->s_rg, D.regularized, 4 * E));
  CK(cp(b->s_si, D.step_index, 4 * E));
  CK(cp(b->s_nc, D.newton_calls, 4 * E));
  CK(cp(b->s_pi, D.pcg_iters, 4 * E));
  CK(cp(b->s_res, D.residual, 8 * E));
  CK(cp(b->s_md, D.min_dist, 8 * E));
  CK(cp(b->s_en, D.energy, 8 * E));
  CK(cp(b->s_tm, D.time, 8 * E));
  CK(cp(b->s_alpha, D.alphas, 8 * E * D.max_alpha));
  CK(cp(b->s_force, D.body_force, 8 * NBd));
  CK(cp(b->s_cmask, D.contact_mask, 4 * NBd));
  CK(cp(b->s_com, D.body_com, 24 * NBd));
  CK(cp(b->s_speed, D.max_speed, 8 * E));
  return 0;
}

// One continuous-batching round: begin_step for envs in `begin` (their controls must be set),
// one Newton sweep over every unfinished env in begin|iter, finalize for every env that finished
// in this round.  finalized[e] is set for those envs and reports[e] filled.
//
// The round is one queue of launches over device lists and one synchronisation: the envs
// that overflowed a buffer (flagged, state untouched) are redone after growth on the
// synchronous per-stage path (rare: capacities only grow early in a run).
int grip_round(GripBatch* b, const uint8_t* begin, const uint8_t* iter, uint8_t* finalized, GripStepReport* reports,
               double* alphas) {
  b->ev_now = false;   // a finalize rewrites (or, recording off, invalidates) the event rows
  Dev& D = b->D;
  b->snap_valid = false;
  const double h0 = host_now();
  const int E = b->n_env;
  int nb = 0, n = 0;
  for (int e = 0; e < E; ++e) {
    if (begin && begin[e]) b->h_lists[nb++] = e;
    if ((begin && begin[e]) || (iter && iter[e])) b->h_lists[E + n++] = e;
  }
  if (finalized) memset(finalized, 0, (size_t)(E > 0 ? E : 0));
  if (n == 0) return 0;
  if (nb) CK(cudaMemcpyAsync(b->d_list, b->h_lists, sizeof(int) * nb, cudaMemcpyHostToDevice, b->stream));
  CK(cudaMemcpyAsync(b->d_list2, b->h_lists + E, sizeof(int) * n, cudaMemcpyHostToDevice, b->stream));
  if (nb) {
    const int t = kt_begin(b, K_BEGIN);
    k_begin<<<nb * BP_CL, NT, 0, b->stream>>>(D, b->d_list);
    kt_end(b, t);
    b->launches++;
  }
  sweep_launch(b, n, b->d_list2);
  {
    const int t = kt_begin(b, K_FIN);
    k_finalize<<<n, NT, 0, b->stream>>>(D, b->d_list2, 1);
    kt_end(b, t);
    b->launches++;
  }
  CK(cudaGetLastError());
  if (snapshot_async(b)) return -1;
  const double h1 = host_now();
  CK(cudaStreamSynchronize(b->stream));
  const double h2 = host_now();
  g_host_enq += h1 - h0;
  g_host_wait += h2 - h1;
  g_host_rounds += 1;
  kt_collect(b, n);
  const std::vector<int> L(b->h_lists + E, b->h_lists + E + n);
  std::vector<int> ovB, ovS, ovF;
  for (int e : L) {
    const int fl = b->s_flags[e];
    if (!(fl & FLAG_OVERFLOW)) continue;
    if (fl & FLAG_OVF_BEGIN) ovB.push_back(e);
    else if (fl & FLAG_OVF_FIN) ovF.push_back(e);
    else ovS.push_back(e);
  }
  if (!ovB.empty() || !ovS.empty() || !ovF.empty()) {
    if (grow(b)) return -1;
    CK(cudaMemsetAsync(D.flags, 0, sizeof(int) * E, b->stream));
    if (!ovB.empty()) {
      if (upload_list(b, ovB, b->d_list)) return -1;
      const int m = (int)ovB.size();
      if (run_with_growth(b, m, [&] { k_begin<<<m * BP_CL, NT, 0, b->stream>>>(D, b->d_list); })) return -1;
    }
    std::vector<int> S2 = ovB;
    S2.insert(S2.end(), ovS.begin(), ovS.end());
    std::sort(S2.begin(), S2.end());
    if (!S2.empty()) {
      if (upload_list(b, S2, b->d_list)) return -1;
      int n2 = 0;
      if (newton_sweep(b, (int)S2.size(), &n2)) return -1;
    }
    std::vector<int> F2 = S2;
    F2.insert(F2.end(), ovF.begin(), ovF.end());
    std::sort(F2.begin(), F2.end());
    if (upload_list(b, F2, b->d_list)) return -1;
    const int m = (int)F2.size();
    if (run_with_growth(b, m, [&] { k_finalize<<<m, NT, 0, b->stream>>>(D, b->d_list, 1); })) return -1;
    kt_collect(b);
    if (snapshot_async(b)) return -1;
    CK(cudaStreamSynchronize(b->stream));
  }
  b->snap_valid = true;
  for (int e : L) {
    if (!b->s_done[e]) continue;
    if (finalized) finalized[e] = 1;
    if (!reports) continue;
    GripStepReport& r = reports[e];
    r.status = b->s_st[e];
    r.reason = b->s_rs[e];
    r.iterations = b->s_it[e];
    r.n_alphas = std::min(b->s_it[e], D.max_alpha);
    r.residual = b->s_res[e];
    r.min_distance = b->s_md[e];
    r.energy = b->s_en[e];
    r.step_index = b->s_si[e] - 1;
    r.time = b->s_tm[e];
    r.kinematic_blocked = b->s_kb[e];
    r.regularized = b->s_rg[e];
    r.newton_calls = b->s_nc[e];
    r.pcg_iters = b->s_pi[e];
  }
  if (alphas) memcpy(alphas, b->s_alpha, sizeof(double) * (size_t)E * D.max_alpha);
  g_host_post += host_now() - h0;
  return 0;
}

// ---------------------------------------------------------------------------
// Device-resident protocol (k_protocol): setup, restart, rounds, readout
// ---------------------------------------------------------------------------
// (Re)start the protocol of the masked envs (all when mask is NULL) on the device: one pinned
// staging buffer of the per-env inputs, one H2D copy, k_protocol_init (no state round trip).
static int protocol_init_envs(GripBatch* b, const uint8_t* mask, const double* closing_dir, const int32_t* max_close,
                              const int32_t* finger_body, const int32_t* object_body, const int32_t* gripper_bits) {
  const int E = b->n_env;
  std::vector<int> L;
  for (int e = 0; e < E; ++e)
    if (!mask || mask[e]) L.push_back(e);
  if (L.empty()) return 0;
  const size_t n = L.size();
  const size_t bytes = n * (sizeof(double) * PINIT_D + sizeof(int) * PINIT_I);
  if (b->ev_pinit_st) CK(cudaEventSynchronize(b->ev_pinit_st));   // the staging may still feed a previous restart
  if (bytes > b->pinit_cap) {
    if (b->h_pinit) cudaFreeHost(b->h_pinit);
    if (b->d_pinit) cudaFree(b->d_pinit);
    b->h_pinit = b->d_pinit = nullptr;
    b->pinit_cap = std::max(bytes, 2 * b->pinit_cap);
    CK(cudaMallocHost(&b->h_pinit, b->pinit_cap));
    CK(cudaMalloc(&b->d_pinit, b->pinit_cap));
  }
  double* hd = reinterpret_cast<double*>(b->h_pinit);
  int* hi = reinterpret_cast<int*>(b->h_pinit + n * sizeof(double) * PINIT_D);
  for (size_t k = 0; k < n; ++k) {
    const int e = L[k];
    for (int c = 0; c < 6; ++c) hd[PINIT_D * k + c] = closing_dir[6 * (size_t)e + c];
    int* q = hi + PINIT_I * k;
    q[0] = e;
    q[1] = max_close[e];
    q[2] = finger_body ? finger_body[2 * e] : -1;   // -1: keep the env's current wiring
    q[3] = finger_body ? finger_body[2 * e + 1] : -1;
    q[4] = object_body ? object_body[e] : -1;
    q[5] = gripper_bits ? gripper_bits[e] : -1;
  }
  CK(cudaMemcpyAsync(b->d_pinit, b->h_pinit, bytes, cudaMemcpyHostToDevice, b->stream));
  k_protocol_init<<<(int)((n + 127) / 128), 128, 0, b->stream>>>(
      b->D, (int)n, reinterpret_cast<const double*>(b->d_pinit),
      reinterpret_cast<const int*>(b->d_pinit + n * sizeof(double) * PINIT_D));
  b->launches++;
  CK(cudaGetLastError());
  if (!b->ev_pinit_st) CK(cudaEventCreateWithFlags(&b->ev_pinit_st, cudaEventDisableTiming));
  CK(cudaEventRecord(b->ev_pinit_st, b->stream));
  b->snap_valid = false;
  return 0;
}

int grip_protocol_setup(GripBatch* b, const int32_t* finger_body, const double* closing_dir, const int32_t* object_body,
                        const int32_t* gripper_bits, const int32_t* max_close, const double* cfg) {
  Dev& D = b->D;
  const int E = b->n_env;
  if (!D.pr_i) {
    D.pr_i = b->alloc<int>((size_t)E * PI_N);
    D.pr_d = b->alloc<double>((size_t)E * PD_N);
    D.pr_cfg = b->alloc<double>(8);
    D.pr_steps = b->alloc<unsigned long long>(1);
    b->d_ident = b->alloc<int>(E);
    if (!D.pr_i || !D.pr_d || !D.pr_cfg || !D.pr_steps || !b->d_ident) {
      g_err = "out of device memory (protocol state)";
      return -1;
    }
    std::vector<int> id(E);
    for (int e = 0; e < E; ++e) id[e] = e;
    CK(cudaMemcpyAsync(b->d_ident, id.data(), sizeof(int) * E, cudaMemcpyHostToDevice, b->stream));
  }
  CK(cudaMemcpyAsync(D.pr_cfg, cfg, sizeof(double) * 8, cudaMemcpyHostToDevice, b->stream));
  return protocol_init_envs(b, nullptr, closing_dir, max_close, finger_body, object_body, gripper_bits);
}

int grip_protocol_reset(GripBatch* b, const uint8_t* mask, const double* closing_dir, const int32_t* max_close) {
  if (!b->D.pr_i) {
    g_err = "grip_protocol_reset before grip_protocol_setup";
    return -1;
  }
  return protocol_init_envs(b, mask, closing_dir, max_close, nullptr, nullptr, nullptr);
}

// enqueue `rounds` device-protocol rounds over every env and the closing finalize + protocol
static int enqueue_rounds(GripBatch* b, int rounds) {
  b->ev_now = false;   // a finalize rewrites (or, recording off, invalidates) the event rows
  Dev& D = b->D;
  if (!D.pr_i) {
    g_err = "grip_run_rounds before grip_protocol_setup";
    return -1;
  }
  const int E = b->n_env;
  b->snap_valid = false;
  D.round_mode = 1;
  CK(cudaMemsetAsync(D.pr_steps, 0, sizeof(unsigned long long), b->stream));
  // round r: [begin] sweep [finalize + protocol]; the finalize / protocol of round r and the begin
  // of round r + 1 are one 4-CTA cluster launch (k_bound). GRIP_SPLIT_BOUND=1 splits it into
  // finalize + protocol (CTA per env) then begin (cluster), so no cluster rank idles through the
  // finalize: measured 1-2 % slower on the bench (one more launch on the lane's critical path).
  static const bool fuse = getenv("GRIP_SPLIT_BOUND") == nullptr;
  for (int r = 0; r < rounds; ++r) {
    int t = kt_begin(b, K_BEGIN);
    D.launch_seq = ++b->seq_ctr;
    if (r > 0 && fuse) {
      k_bound<<<E * BP_CL, NT, 0, b->stream>>>(D, b->d_ident);
    } else {
      if (r > 0) {
        k_finalize_protocol<<<E, NT, 0, b->stream>>>(D, b->d_ident);
        b->launches += 1;
      }
      k_begin<<<E * BP_CL, NT, 0, b->stream>>>(D, b->d_ident);
    }
    kt_end(b, t);
    sweep_launch(b, E, b->d_ident);
    b->launches += 1;
  }
  int t = kt_begin(b, K_FIN);
  D.launch_seq = ++b->seq_ctr;
  k_finalize_protocol<<<E, NT, 0, b->stream>>>(D, b->d_ident);
  kt_end(b, t);
  b->launches += 1;
  D.round_mode = 0;
  CK(cudaGetLastError());
  return 0;
}

// after a call whose flags showed an overflow: drain the stream, grow, clear the flags; the
// overflowed envs' state is untouched and they resume in the next call
static int grow_after_overflow(GripBatch* b) {
  CK(cudaStreamSynchronize(b->stream));
  if (grow(b)) return -1;
  CK(cudaMemsetAsync(b->D.flags, 0, sizeof(int) * b->n_env, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

int grip_run_rounds(GripBatch* b, int rounds, int64_t* env_steps) {
  for (auto& rs : b->rslot)
    if (rs.busy) {
      g_err = "grip_run_rounds: a pipelined call is in flight (grip_rounds_wait first)";
      return -1;
    }
  if (enqueue_rounds(b, rounds)) return -1;
  Dev& D = b->D;
  const int E = b->n_env;
  unsigned long long steps = 0;
  std::vector<int> fl(E);
  CK(cudaMemcpyAsync(&steps, D.pr_steps, sizeof(steps), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(fl.data(), D.flags, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  kt_collect(b);
  bool ovf = false;
  for (int e = 0; e < E; ++e) ovf |= (fl[e] & FLAG_OVERFLOW) != 0;
  if (ovf && grow_after_overflow(b)) return -1;
  if (env_steps) *env_steps = (int64_t)steps;
  return 0;
}

static size_t rslot_bytes(int E) {
  return 8 + ((4 * (size_t)E * (1 + PI_N) + 7) & ~(size_t)7) + 8 * (size_t)E * PD_N;
}

static void decode_trial_out(const int* hi, const double* hd, int E, GripTrialOut* out) {
  for (int e = 0; e < E; ++e) {
    const int* I = hi + (size_t)e * PI_N;
    const double* R = hd + (size_t)e * PD_N;
    GripTrialOut& o = out[e];
    o.halt_force[0] = R[PD_HF]; o.halt_force[1] = R[PD_HF + 1];
    for (int k = 0; k < 6; ++k) o.com_disp[k] = R[PD_CDISP + k];
    o.final_disp = R[PD_FDISP];
    o.threshold = R[PD_THR];
    o.phase = I[PI_PHASE];
    o.verdict = I[PI_VERDICT];
    o.n_steps = I[PI_NSTEPS];
    o.fail_phase = I[PI_FPHASE];
    o.fail_reason = I[PI_FREASON];
    o.fail_step = I[PI_FSTEP];
    o.halted = I[PI_HALTED];
    o.final_contact = I[PI_FCONTACT];
    o.halt_step[0] = I[PI_HSTEP0]; o.halt_step[1] = I[PI_HSTEP1];
    for (int k = 0; k < 18; ++k) o.markers[k] = I[PI_MARK + k];
    o.min_distance = R[PD_MIND];
    o.min_J = R[PD_MINJ];
  }
}

int grip_run_rounds_async(GripBatch* b, int rounds, int32_t* ticket) {
  GripBatch::RoundSlot& rs = b->rslot[b->rslot_next];
  if (rs.busy) {
    g_err = "grip_run_rounds_async: two calls already in flight (grip_rounds_wait first)";
    return -1;
  }
  const int E = b->n_env;
  if (!rs.h) {
    CK(cudaMallocHost(&rs.h, rslot_bytes(E)));
    // GRIP_BLOCKING_SYNC=1: the waiting host thread sleeps instead of spinning (bench.py sets it
    // when its ranks' lane threads would outnumber the host cores); spinning is ~0.5 % faster
    const unsigned fl = cudaEventDisableTiming | (getenv("GRIP_BLOCKING_SYNC") ? cudaEventBlockingSync : 0u);
    CK(cudaEventCreateWithFlags(&rs.ev, fl));
  }
  const bool graphs = getenv("GRIP_GRAPH") != nullptr && !b->D.cta_rec;   // opt-in: see DESIGN §6
  if (graphs && !b->D.cta_rec) {
    GripBatch::RoundGraph& g = b->rgraph[b->rslot_next];
    Dev cur = b->D;
    cur.launch_seq = 0;   // diagnostic only (per-CTA timing builds, which do not use graphs)
    const bool valid = g.exec && g.rounds == rounds && g.prof == b->prof && g.stream == b->stream &&
                       g.env_cap == b->env_cap && g.dyn_smem == b->dyn_smem && memcmp(&g.D, &cur, sizeof(Dev)) == 0;
    if (!valid) {
      if (g.exec) {
        cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
        for (auto& pk : g.kt) {
          b->kev_owned[pk.second] = 0;
          b->kev_free.push_back(pk.second);
        }
        g.kt.clear();
      }
      const size_t k0 = b->pending_k.size();
      const long long l0 = b->launches;
      CK(cudaStreamBeginCapture(b->stream, cudaStreamCaptureModeThreadLocal));
      const int rc = enqueue_rounds(b, rounds);
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(b->stream, &graph);
      if (rc) return -1;
      CK(ce);
      CK(cudaGraphInstantiate(&g.exec, graph, 0));
      cudaGraphDestroy(graph);
      g.kt.assign(b->pending_k.begin() + k0, b->pending_k.end());
      b->pending_k.resize(k0);
      for (auto& pk : g.kt) {
        if ((size_t)pk.second >= b->kev_owned.size()) b->kev_owned.resize(pk.second + 1, 0);
        b->kev_owned[pk.second] = 1;
      }
      g.launches = b->launches - l0;
      b->launches = l0;
      g.D = cur;
      g.stream = b->stream;
      g.rounds = rounds;
      g.prof = b->prof;
      g.env_cap = b->env_cap;
      g.dyn_smem = b->dyn_smem;
    }
    b->ev_now = false;
    b->snap_valid = false;
    CK(cudaGraphLaunch(g.exec, b->stream));
    b->pending_k.insert(b->pending_k.end(), g.kt.begin(), g.kt.end());
    b->launches += g.launches;
  } else if (enqueue_rounds(b, rounds)) {
    return -1;
  }
  Dev& D = b->D;
  char* h = rs.h;
  int* hf = reinterpret_cast<int*>(h + 8);
  int* hi = hf + E;
  double* hd = reinterpret_cast<double*>(h + 8 + ((4 * (size_t)E * (1 + PI_N) + 7) & ~(size_t)7));
  CK(cudaMemcpyAsync(h, D.pr_steps, 8, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(hf, D.flags, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(hi, D.pr_i, sizeof(int) * (size_t)E * PI_N, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(hd, D.pr_d, sizeof(double) * (size_t)E * PD_N, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaEventRecord(rs.ev, b->stream));
  rs.busy = true;
  rs.kt_mark = b->pending_k.size();
  *ticket = b->rslot_next;
  b->rslot_next ^= 1;
  return 0;
}

int grip_rounds_wait(GripBatch* b, int32_t ticket, int64_t* env_steps, GripTrialOut* out) {
  if (ticket < 0 || ticket > 1 || !b->rslot[ticket].busy) {
    g_err = "grip_rounds_wait: no such call in flight";
    return -1;
  }
  GripBatch::RoundSlot& rs = b->rslot[ticket];
  CK(cudaEventSynchronize(rs.ev));
  kt_collect(b, -1, (long long)rs.kt_mark);
  rs.busy = false;
  const int E = b->n_env;
  const char* h = rs.h;
  unsigned long long steps = 0;
  memcpy(&steps, h, 8);
  const int* hf = reinterpret_cast<const int*>(h + 8);
  const int* hi = hf + E;
  const double* hd = reinterpret_cast<const double*>(h + 8 + ((4 * (size_t)E * (1 + PI_N) + 7) & ~(size_t)7));
  if (out) decode_trial_out(hi, hd, E, out);
  bool ovf = false;
  for (int e = 0; e < E; ++e) ovf |= (hf[e] & FLAG_OVERFLOW) != 0;
  if (ovf && grow_after_overflow(b)) return -1;
  if (env_steps) *env_steps = (int64_t)steps;
  return 0;
}

int grip_protocol_read(GripBatch* b, GripTrialOut* out) {
  Dev& D = b->D;
  if (!D.pr_i) {
    g_err = "grip_protocol_read before grip_protocol_setup";
    return -1;
  }
  const int E = b->n_env;
  std::vector<int> hi((size_t)E * PI_N);
  std::vector<double> hd((size_t)E * PD_N);
  CK(cudaMemcpyAsync(hi.data(), D.pr_i, sizeof(int) * hi.size(), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(hd.data(), D.pr_d, sizeof(double) * hd.size(), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  decode_trial_out(hi.data(), hd.data(), E, out);
  return 0;
}

// Scheduling priority of the batch's stream (0 = default, larger = more urgent, clamped to the
// device's range): lanes sharing a GPU can favour the batch with the longest per-env chains.
int grip_set_priority(GripBatch* b, int priority) {
  int lo = 0, hi = 0;   // CUDA: numerically lower = higher priority (hi <= lo)
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  const int p = std::max(hi, std::min(lo, lo - priority));
  const bool using_own = b->stream == b->own_stream;
  CK(cudaStreamSynchronize(b->stream));
  cudaStream_t s = nullptr;
  CK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, p));
  CK(cudaStreamDestroy(b->own_stream));
  b->own_stream = s;
  if (using_own) b->stream = s;
  CK(cudaStreamSynchronize(b->aux));
  cudaStream_t a = nullptr;
  CK(cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, p));
  CK(cudaStreamDestroy(b->aux));
  b->aux = a;
  CK(cudaStreamSynchronize(b->aux2));
  CK(cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, p));
  CK(cudaStreamDestroy(b->aux2));
  b->aux2 = a;
  return 0;
}

// Run the batch on a caller's CUDA stream (e.g. a torch.cuda.Stream's handle) from now on, or on
// the library's own stream again with stream == NULL.  Work already queued on the previous stream
// is finished first; the caller keeps ownership of its stream.
int grip_set_stream(GripBatch* b, void* stream) {
  CK(cudaStreamSynchronize(b->stream));
  b->stream = stream ? static_cast<cudaStream_t>(stream) : b->own_stream;
  return 0;
}

// Device-pointer forms of the state / control transfers (torch tensors' data pointers): copies
// queued on the batch's stream, no synchronisation (stream order is the caller's contract).
int grip_get_state_device(GripBatch* b, double* x, double* v, double* kin) {
  if (x) CK(cudaMemcpyAsync(x, b->D.x, 3 * sizeof(double) * b->n_node, cudaMemcpyDeviceToDevice, b->stream));
  if (v) CK(cudaMemcpyAsync(v, b->D.v, 3 * sizeof(double) * b->n_node, cudaMemcpyDeviceToDevice, b->stream));
  if (kin) CK(cudaMemcpyAsync(kin, b->D.kin_pos, 3 * sizeof(double) * b->n_sv, cudaMemcpyDeviceToDevice, b->stream));
  return 0;
}

int grip_set_controls_device(GripBatch* b, const double* gravity, const double* body_vel) {
  if (gravity)
    CK(cudaMemcpyAsync(b->D.gravity, gravity, 3 * sizeof(double) * b->n_env, cudaMemcpyDeviceToDevice, b->stream));
  if (body_vel)
    CK(cudaMemcpyAsync(b->D.body_vel, body_vel, 3 * sizeof(double) * b->n_body, cudaMemcpyDeviceToDevice, b->stream));
  b->snap_valid = false;
  return 0;
}

int grip_set_recording(GripBatch* b, int on) {
  b->D.ev_on = on ? 1 : 0;
  return 0;
}

int grip_check_finite(GripBatch* b, uint8_t* nonfinite) {
  if (b->n_env == 0) return 0;
  if (!b->d_nonfin) {
    b->d_nonfin = b->alloc<int>(b->n_env);
    if (!b->d_nonfin) {
      g_err = "out of device memory";
      return -1;
    }
  }
  k_check_finite<<<b->n_env, NT, 0, b->stream>>>(b->D, b->d_nonfin);
  b->launches++;
  CK(cudaGetLastError());
  std::vector<int> h(b->n_env);
  CK(cudaMemcpyAsync(h.data(), b->d_nonfin, sizeof(int) * b->n_env, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  for (int e = 0; e < b->n_env; ++e) nonfinite[e] = (uint8_t)(h[e] != 0);
  return 0;
}

int grip_contacts_now(GripBatch* b, const uint8_t* mask, double radius_factor, double* min_distance) {
  std::vector<int> L = mask_to_list(b, mask);
  if (L.empty()) return 0;
  if (upload_list(b, L, b->d_list)) return -1;
  const int n = (int)L.size();
  if (!b->d_md_now) {
    b->d_md_now = b->alloc<double>(std::max(b->n_env, 1));
    if (!b->d_md_now) {
      g_err = "out of device memory";
      return -1;
    }
  }
  if (run_with_growth(b, n, [&] {
        k_contacts_now<<<n, NT, 0, b->stream>>>(b->D, b->d_list, radius_factor, b->d_md_now);
      }))
    return -1;
  b->snap_valid = false;   // body forces / contact bits now describe this state
  b->ev_now = true;
  if (min_distance) {
    CK(cudaMemcpyAsync(min_distance, b->d_md_now, sizeof(double) * b->n_env, cudaMemcpyDeviceToHost, b->stream));
    CK(cudaStreamSynchronize(b->stream));
  }
  return 0;
}

int grip_get_events(GripBatch* b, const uint8_t* mask, int32_t* counts, int32_t* ev_i, double* ev_d, int64_t cap) {
  Dev& D = b->D;
  if (!D.ev_on && !b->ev_now) {
    g_err = "grip_get_events: no events (grip_set_recording off and no grip_contacts_now)";
    return -1;
  }
  const int E = b->n_env;
  CK(cudaMemcpyAsync(counts, D.ev_n, sizeof(int) * E, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  int64_t off = 0;
  for (int e = 0; e < E; ++e) {
    if (!mask[e]) continue;
    const int n = std::min(counts[e], D.cap_anc);
    counts[e] = n;   // rows copied (a step with more active stencils than cap_anc is truncated)
    if (off + n > cap) {
      g_err = "grip_get_events: output capacity too small";
      return -1;
    }
    if (n) {
      const size_t s = (size_t)e * D.cap_anc;
      CK(cudaMemcpyAsync(ev_i + 7 * off, D.ev_i + 7 * s, sizeof(int) * 7 * n, cudaMemcpyDeviceToHost, b->stream));
      CK(cudaMemcpyAsync(ev_d + 2 * off, D.ev_d + 2 * s, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, b->stream));
    }
    off += n;
  }
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

int grip_reset_envs(GripBatch* b, const uint8_t* mask, const GripSceneDesc* d) {
  b->snap_valid = false;
  if (!d || d->abi_version != GRIP_ABI_VERSION || d->n_env != b->n_env) {
    g_err = "grip_reset_envs: scene description missing or of another batch size / ABI";
    return -1;
  }
  // stage the masked envs' slices in one pinned buffer -> one H2D copy -> k_reset_envs scatters them
  std::vector<int> L;
  std::vector<long long> off;
  long long n = 0;
  for (int e = 0; e < b->n_env; ++e) {
    if (!mask[e]) continue;
    auto same = [&](const int32_t* o, const std::vector<int>& mine) {
      return o[e] == mine[e] && o[e + 1] == mine[e + 1];
    };
    if (!same(d->node_off, b->node_off) || !same(d->sv_off, b->sv_off) || !same(d->tri_off, b->tri_off) ||
        !same(d->edge_off, b->edge_off) || !same(d->tet_off, b->tet_off) || !same(d->abd_off, b->abd_off) ||
        !same(d->body_off, b->body_off)) {
      g_err = "grip_reset_envs: env " + std::to_string(e) + " changes topology (a refill keeps the slot's meshes)";
      return -1;
    }
    const long long nn = b->node_off[e + 1] - b->node_off[e], ns = b->sv_off[e + 1] - b->sv_off[e];
    const long long nt = b->tet_off[e + 1] - b->tet_off[e], nb = b->body_off[e + 1] - b->body_off[e];
    const long long ne = b->edge_off[e + 1] - b->edge_off[e], na = b->abd_off[e + 1] - b->abd_off[e];
    L.push_back(e);
    off.push_back(n);
    n += RESET_PER_NODE * nn + RESET_PER_SV * ns + RESET_PER_TET * nt + nb + ne + na + 1;
  }
  if (L.empty()) return 0;
  const size_t head = L.size() * (sizeof(int) + sizeof(long long));
  const size_t bytes = ((head + 15) & ~(size_t)15) + n * sizeof(double);
  if (b->ev_reset_st) CK(cudaEventSynchronize(b->ev_reset_st));   // the staging may still feed a previous refill
  if (bytes > b->reset_cap) {
    if (b->h_reset) cudaFreeHost(b->h_reset);
    if (b->d_reset) cudaFree(b->d_reset);
    b->h_reset = nullptr;
    b->d_reset = nullptr;
    b->reset_cap = std::max(bytes, 2 * b->reset_cap);
    CK(cudaMallocHost(&b->h_reset, b->reset_cap));
    CK(cudaMalloc(&b->d_reset, b->reset_cap));
  }
  char* h = b->h_reset;
  long long* h_off = reinterpret_cast<long long*>(h);
  int* h_lst = reinterpret_cast<int*>(h + L.size() * sizeof(long long));
  double* h_st = reinterpret_cast<double*>(h + ((head + 15) & ~(size_t)15));
  for (size_t k = 0; k < L.size(); ++k) {
    const int e = L[k];
    h_off[k] = off[k];
    h_lst[k] = e;
    double* q = h_st + off[k];
    auto put = [&](const double* src, size_t o, size_t cnt) {
      memcpy(q, src + o, cnt * sizeof(double));
      q += cnt;
    };
    const size_t n0 = b->node_off[e], nn = b->node_off[e + 1] - n0;
    const size_t s0 = b->sv_off[e], ns = b->sv_off[e + 1] - s0;
    const size_t t0 = b->tet_off[e], nt = b->tet_off[e + 1] - t0;
    const size_t b0 = b->body_off[e], nb = b->body_off[e + 1] - b0;
    const size_t e0 = b->edge_off[e], ne = b->edge_off[e + 1] - e0;
    const size_t a0 = b->abd_off[e], na = b->abd_off[e + 1] - a0;
    put(d->node_x0, 3 * n0, 3 * nn);
    put(d->node_M, 9 * n0, 9 * nn);
    put(d->sv_kin0, 3 * s0, 3 * ns);
    put(d->sv_xi, 3 * s0, 3 * ns);
    put(d->tet_Dmi, 9 * t0, 9 * nt);
    put(d->tet_V0, t0, nt);
    put(d->tet_mu, t0, nt);
    put(d->tet_lam, t0, nt);
    put(d->body_mu, b0, nb);
    put(d->edge_rest_sq, e0, ne);
    put(d->abd_kV, a0, na);
    put(d->env_cell_hint, e, 1);
  }
  CK(cudaMemcpyAsync(b->d_reset, b->h_reset, bytes, cudaMemcpyHostToDevice, b->stream));
  const char* dd = b->d_reset;
  k_reset_envs<<<(int)L.size(), NT, 0, b->stream>>>(
      b->D, reinterpret_cast<const int*>(dd + L.size() * sizeof(long long)), reinterpret_cast<const long long*>(dd),
      reinterpret_cast<const double*>(dd + ((head + 15) & ~(size_t)15)));
  b->launches++;
  CK(cudaGetLastError());
  if (!b->ev_reset_st) CK(cudaEventCreateWithFlags(&b->ev_reset_st, cudaEventDisableTiming));
  CK(cudaEventRecord(b->ev_reset_st, b->stream));
  return 0;
}

int grip_debug_elements(int type, int n, const double* in, int stride, double* E, double* g, double* H, int* flags) {
  if (n <= 0) return 0;
  double *d_in, *d_E, *d_g, *d_H;
  int* d_f;
  CK(cudaMalloc(&d_in, sizeof(double) * (size_t)n * stride));
  CK(cudaMalloc(&d_E, sizeof(double) * n));
  CK(cudaMalloc(&d_g, sizeof(double) * 12 * (size_t)n));
  CK(cudaMalloc(&d_H, sizeof(double) * 144 * (size_t)n));
  CK(cudaMalloc(&d_f, sizeof(int) * n));
  CK(cudaMemcpy(d_in, in, sizeof(double) * (size_t)n * stride, cudaMemcpyHostToDevice));
  k_debug_elements<<<std::min(1024, (n + 3) / 4), 128>>>(type, n, d_in, stride, d_E, d_g, d_H, d_f);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(E, d_E, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(g, d_g, sizeof(double) * 12 * (size_t)n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(H, d_H, sizeof(double) * 144 * (size_t)n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(flags, d_f, sizeof(int) * n, cudaMemcpyDeviceToHost));
  cudaFree(d_in); cudaFree(d_E); cudaFree(d_g); cudaFree(d_H); cudaFree(d_f);
  return 0;
}

// Element-level test hook of the PRODUCTION element chain (the launches of sweep_launch on a
// scratch device context): type 2 NH tets through k_tet_front (Gershgorin pass-through or
// deferral) -> k_tet_jacobi2 -> k_tet_back with the warm-start eigenbases eig (n*81, in/out;
// NULL = identity, the first Newton iteration); types 0 / 1 PT / EE stencils through the
// k_elements_w element code with clamp deferral -> k_tet_jacobi2 -> k_tet_finish.  Same input
// rows and outputs as grip_debug_elements.
int grip_debug_chain(int type, int n, const double* in, int stride, double* E, double* g, double* H, double* eig,
                     int* flags) {
  if (n <= 0) return 0;
  if (type < 0 || type > 2) {
    g_err = "grip_debug_chain: type must be 0 (PT), 1 (EE) or 2 (NH)";
    return -1;
  }
  std::vector<void*> mem;
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 8)) != cudaSuccess) return (void*)nullptr;
    cudaMemset(p, 0, std::max<size_t>(bytes, 8));
    mem.push_back(p);
    return p;
  };
  auto up = [&](const void* h, size_t bytes) {
    void* p = dalloc(bytes);
    if (p && bytes) cudaMemcpy(p, h, bytes, cudaMemcpyHostToDevice);
    return p;
  };
  int rc = 0;
  Dev D{};
  D.n_env = 1;
  D.cap_el = n;
  D.el_E = (double*)dalloc(sizeof(double) * n);
  D.el_g = (double*)dalloc(sizeof(double) * 12 * (size_t)n);
  D.el_H = (double*)dalloc(sizeof(double) * 144 * (size_t)n);
  D.el_idx = (int*)dalloc(sizeof(int) * 4 * (size_t)n);
  D.flags = (int*)dalloc(sizeof(int));
  D.tflag = (int*)dalloc(sizeof(int));
  int* d_flags = (int*)dalloc(sizeof(int) * n);
  double* d_in = (double*)up(in, sizeof(double) * (size_t)n * stride);
  if (type == 2) {
    std::vector<double> x(12 * (size_t)n), Dmi(9 * (size_t)n), V0(n), mu(n), lam(n), Y(81 * (size_t)n, 0.0);
    std::vector<int> tn(4 * (size_t)n), off_n{0, 4 * n}, off_t{0, n}, zero{0};
    for (int k = 0; k < n; ++k) {
      const double* r = in + (size_t)k * stride;
      for (int j = 0; j < 12; ++j) x[12 * (size_t)k + j] = r[j];
      for (int j = 0; j < 9; ++j) Dmi[9 * (size_t)k + j] = r[12 + j];
      V0[k] = r[21]; mu[k] = r[22]; lam[k] = r[23];
      for (int j = 0; j < 4; ++j) tn[4 * (size_t)k + j] = 4 * k + j;
      for (int j = 0; j < 81; ++j) Y[81 * (size_t)k + j] = eig ? eig[81 * (size_t)k + j] : (j % 10 == 0 ? 1.0 : 0.0);
    }
    D.x = (double*)up(x.data(), sizeof(double) * x.size());
    D.tet_nodes = (const int*)up(tn.data(), sizeof(int) * tn.size());
    D.tet_Dmi = (const double*)up(Dmi.data(), sizeof(double) * Dmi.size());
    D.tet_V0 = (const double*)up(V0.data(), sizeof(double) * n);
    D.tet_mu = (const double*)up(mu.data(), sizeof(double) * n);
    D.tet_lam = (const double*)up(lam.data(), sizeof(double) * n);
    Y.resize(2 * Y.size(), 0.0);   // warm-start halves: the bases in half 0, the new ones land in half 1
    D.tet_eig = (double*)up(Y.data(), sizeof(double) * Y.size());
    D.eig_half = 81 * (size_t)n;
    D.eig_par = (int*)up(zero.data(), sizeof(int));
    D.eig_swept = (int*)up(zero.data(), sizeof(int));
    D.tet_S = (double*)dalloc(sizeof(double) * 45 * (size_t)n);
    D.tet_W = (double*)dalloc(sizeof(double) * 90 * (size_t)n);
    D.jac_list = (int2*)dalloc(sizeof(int2) * n);
    D.jac_n = (int*)dalloc(sizeof(int));
    D.node_off = (const int*)up(off_n.data(), sizeof(int) * 2);
    D.tet_off = (const int*)up(off_t.data(), sizeof(int) * 2);
    D.twork_off = (int*)up(off_t.data(), sizeof(int) * 2);
    int* d_list = (int*)up(zero.data(), sizeof(int));
    k_tet_front<<<std::max(1, std::min(1024, (n + TF - 1) / TF)), TF>>>(D, d_list, 1);
    k_tet_jacobi2<<<148, TJ>>>(D.jac_list, D.jac_n, D.tet_S, D.tet_W);
    k_tet_back<<<148, EW * 32>>>(D, D.jac_list, D.jac_n, D.tet_W);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) rc = -1;
    if (!rc && eig) cudaMemcpy(eig, D.tet_eig + D.eig_half, sizeof(double) * 81 * (size_t)n, cudaMemcpyDeviceToHost);
    int ff = 0;
    cudaMemcpy(&ff, D.tflag, sizeof(int), cudaMemcpyDeviceToHost);
    for (int k = 0; k < n; ++k) flags[k] = ff;
  } else {
    D.cjac_S = (double*)dalloc(sizeof(double) * 45 * (size_t)n);
    D.cjac_W = (double*)dalloc(sizeof(double) * 90 * (size_t)n);
    D.cjac_list = (int2*)dalloc(sizeof(int2) * n);
    D.cjac_n = (int*)dalloc(sizeof(int));
    k_debug_contacts<<<std::max(1, std::min(1024, (n + 3) / 4)), 128>>>(D, type, n, d_in, stride, d_flags);
    k_tet_jacobi2<<<148, TJ>>>(D.cjac_list, D.cjac_n, D.cjac_S, D.cjac_W);
    k_tet_finish<<<148, EW * 32>>>(D, D.cjac_list, D.cjac_n, D.cjac_W, nullptr);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) rc = -1;
    if (!rc) cudaMemcpy(flags, d_flags, sizeof(int) * n, cudaMemcpyDeviceToHost);
  }
  for (void* p : mem)
    if (!p) rc = -1;
  if (!rc) {
    cudaMemcpy(E, D.el_E, sizeof(double) * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(g, D.el_g, sizeof(double) * 12 * (size_t)n, cudaMemcpyDeviceToHost);
    cudaMemcpy(H, D.el_H, sizeof(double) * 144 * (size_t)n, cudaMemcpyDeviceToHost);
    if (type == 2)   // tets: unpack the stored lower triangle (tri12) in place, last slot entry first
      for (int k = 0; k < n; ++k) {
        double* h = H + 144 * (size_t)k;
        double lo[78];
        memcpy(lo, h, sizeof lo);
        for (int r = 0; r < 12; ++r)
          for (int c = 0; c <= r; ++c) h[r * 12 + c] = h[c * 12 + r] = lo[tri12(r, c)];
      }
  }
  for (void* p : mem)
    if (p) cudaFree(p);
  if (rc) g_err = "grip_debug_chain: device error";
  return rc;
}

#ifdef GRIP_JAC_HIST
// diagnostic build only (tools/jac_hist.py): the Jacobi sweep histogram, [2][GRIP_JAC_MAXSWEEP + 1]
int grip_jac_hist(unsigned long long* out, int reset) {
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyFromSymbol(out, g_jac_hist, sizeof(g_jac_hist)));
  if (reset) {
    static unsigned long long z[2][GRIP_JAC_MAXSWEEP + 1] = {};
    CK(cudaMemcpyToSymbol(g_jac_hist, z, sizeof(z)));
  }
  return 0;
}
#endif

int grip_cta_records(GripBatch* b, uint64_t* out, int64_t cap, int64_t* n, int reset) {
  *n = 0;
  if (!b->D.cta_rec) return 0;   // not a GRIP_CTA_TIMING build
  unsigned cnt = 0;
  CK(cudaMemcpyAsync(&cnt, b->D.cta_n, sizeof(unsigned), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  const int64_t m = std::min<int64_t>({(int64_t)cnt, (int64_t)b->D.cta_cap, cap});
  if (out && m > 0) CK(cudaMemcpy(out, b->D.cta_rec, sizeof(uint64_t) * 4 * (size_t)m, cudaMemcpyDeviceToHost));
  *n = m;
  if (reset) CK(cudaMemsetAsync(b->D.cta_n, 0, sizeof(unsigned), b->stream));
  return 0;
}

int grip_get_state(GripBatch* b, double* x, double* v, double* kin) {
  if (x) CK(cudaMemcpyAsync(x, b->D.x, 3 * sizeof(double) * b->n_node, cudaMemcpyDeviceToHost, b->stream));
  if (v) CK(cudaMemcpyAsync(v, b->D.v, 3 * sizeof(double) * b->n_node, cudaMemcpyDeviceToHost, b->stream));
  if (kin) CK(cudaMemcpyAsync(kin, b->D.kin_pos, 3 * sizeof(double) * b->n_sv, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

int grip_set_state(GripBatch* b, const double* x, const double* v, const double* kin) {
  b->snap_valid = false;
  CK(cudaMemsetAsync(b->D.cs_valid, 0, sizeof(int) * b->n_env, b->stream));
  if (x) CK(cudaMemcpyAsync(b->D.x, x, 3 * sizeof(double) * b->n_node, cudaMemcpyHostToDevice, b->stream));
  if (v) CK(cudaMemcpyAsync(b->D.v, v, 3 * sizeof(double) * b->n_node, cudaMemcpyHostToDevice, b->stream));
  if (kin) CK(cudaMemcpyAsync(b->D.kin_pos, kin, 3 * sizeof(double) * b->n_sv, cudaMemcpyHostToDevice, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

int grip_get_surface(GripBatch* b, double* sv) {
  std::vector<int> L = mask_to_list(b, nullptr);
  if (upload_list(b, L, b->d_list)) return -1;
  k_surface_all<<<b->n_env, 128, 0, b->stream>>>(b->D, b->d_list);
  b->launches++;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(sv, b->D.sv_pos, 3 * sizeof(double) * b->n_sv, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

int grip_get_contacts(GripBatch* b, double* body_force, uint32_t* contact_mask, double* min_distance) {
  if (b->snap_valid) {   // unchanged since the round's snapshot
    if (body_force) memcpy(body_force, b->s_force, sizeof(double) * b->n_body);
    if (contact_mask) memcpy(contact_mask, b->s_cmask, sizeof(uint32_t) * b->n_body);
    if (min_distance) memcpy(min_distance, b->s_md, sizeof(double) * b->n_env);
    return 0;
  }
  if (body_force) CK(cudaMemcpyAsync(body_force, b->D.body_force, sizeof(double) * b->n_body, cudaMemcpyDeviceToHost, b->stream));
  if (contact_mask)
    CK(cudaMemcpyAsync(contact_mask, b->D.contact_mask, sizeof(uint32_t) * b->n_body, cudaMemcpyDeviceToHost, b->stream));
  if (min_distance) CK(cudaMemcpyAsync(min_distance, b->D.min_dist, sizeof(double) * b->n_env, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

int grip_query_candidates(GripBatch* b, int env, double radius, int32_t* pt, int32_t cap_pt, int32_t* n_pt, int32_t* ee,
                          int32_t cap_ee, int32_t* n_ee) {
  if (env < 0 || env >= b->n_env) {
    g_err = "env out of range";
    return -1;
  }
  std::vector<int> L{env};
  if (upload_list(b, L, b->d_list)) return -1;
  if (run_with_growth(b, 1, [&] { k_query<<<1, NT, 0, b->stream>>>(b->D, b->d_list, radius); })) return -1;
  int cn[2];
  CK(cudaMemcpy(cn, b->D.c2_n + 2 * env, 2 * sizeof(int), cudaMemcpyDeviceToHost));
  *n_pt = cn[0];
  *n_ee = cn[1];
  if (pt) CK(cudaMemcpy(pt, b->D.c2_pt + (size_t)env * 4 * b->D.cap_pt, 4 * sizeof(int) * std::min(cn[0], cap_pt),
                        cudaMemcpyDeviceToHost));
  if (ee) CK(cudaMemcpy(ee, b->D.c2_ee + (size_t)env * 4 * b->D.cap_ee, 4 * sizeof(int) * std::min(cn[1], cap_ee),
                        cudaMemcpyDeviceToHost));
  return 0;
}

int grip_stress(GripBatch* b, double* out) {
  if (b->n_tet == 0) return 0;
  if (!b->d_stress && !(b->d_stress = b->alloc<double>(7 * (size_t)b->n_tet))) {
    g_err = "out of device memory";
    return -1;
  }
  k_stress<<<std::min(148 * 8, (b->n_tet + 127) / 128), 128, 0, b->stream>>>(b->D, b->n_tet, b->d_tet_env, b->d_stress);
  b->launches++;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, b->d_stress, 7 * sizeof(double) * b->n_tet, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

// One recorded frame of every masked env (protocol.py:113-146 _Recorder.snapshot), packed in
// env order: node positions and velocities (nn*3 each), surface-vertex kinematic positions
// (ns*3) and stress rows (n_tet*7).  One kernel gathers them on the device, one D2H moves
// them through a pinned buffer.
int grip_get_frames(GripBatch* b, const uint8_t* mask, double* x, double* v, double* kin, double* stress) {
  const int E = b->n_env;
  const size_t cap = 6 * (size_t)b->n_node + 3 * (size_t)b->n_sv + 7 * (size_t)b->n_tet;
  if (!b->d_frame) {
    b->d_frame = b->alloc<double>(cap);
    b->d_fmask = b->alloc<int>(4 * (size_t)E);
    if (!b->d_stress) b->d_stress = b->alloc<double>(7 * (size_t)std::max(b->n_tet, 1));
    if (cudaMallocHost(&b->h_frame, sizeof(double) * std::max<size_t>(cap, 1)) != cudaSuccess ||
        cudaMallocHost(&b->h_fmask, sizeof(int) * 4 * E) != cudaSuccess || !b->d_frame || !b->d_fmask) {
      g_err = "out of memory (frame buffers)";
      return -1;
    }
  }
  size_t on = 0, os = 0, ot = 0;
  for (int e = 0; e < E; ++e) {
    int* m = b->h_fmask + 4 * e;
    m[0] = mask[e] ? (int)on : -1;
    m[1] = (int)os;
    m[2] = (int)ot;
    m[3] = 0;
    if (mask[e]) {
      on += b->node_off[e + 1] - b->node_off[e];
      os += b->sv_off[e + 1] - b->sv_off[e];
      ot += b->tet_off[e + 1] - b->tet_off[e];
    }
  }
  if (on + os + ot == 0) return 0;
  CK(cudaMemcpyAsync(b->d_fmask, b->h_fmask, sizeof(int) * 4 * E, cudaMemcpyHostToDevice, b->stream));
  double* fx = b->d_frame;
  double* fv = fx + 3 * on;
  double* fk = fv + 3 * on;
  double* fs = fk + 3 * os;
  k_frames<<<E, 128, 0, b->stream>>>(b->D, b->d_fmask, fx, fv, fk, fs);
  b->launches++;
  CK(cudaGetLastError());
  const size_t tot = 6 * on + 3 * os + 7 * ot;
  CK(cudaMemcpyAsync(b->h_frame, b->d_frame, sizeof(double) * tot, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  const double* h = b->h_frame;
  if (x) memcpy(x, h, sizeof(double) * 3 * on);
  if (v) memcpy(v, h + 3 * on, sizeof(double) * 3 * on);
  if (kin) memcpy(kin, h + 6 * on, sizeof(double) * 3 * os);
  if (stress) memcpy(stress, h + 6 * on + 3 * os, sizeof(double) * 7 * ot);
  return 0;
}

int grip_get_body_state(GripBatch* b, double* body_com, double* max_speed) {
  if (b->snap_valid) {
    if (body_com) memcpy(body_com, b->s_com, 3 * sizeof(double) * b->n_body);
    if (max_speed) memcpy(max_speed, b->s_speed, sizeof(double) * b->n_env);
    return 0;
  }
  if (body_com) CK(cudaMemcpyAsync(body_com, b->D.body_com, 3 * sizeof(double) * b->n_body, cudaMemcpyDeviceToHost, b->stream));
  if (max_speed) CK(cudaMemcpyAsync(max_speed, b->D.max_speed, sizeof(double) * b->n_env, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

int grip_set_profiling(GripBatch* b, int on) {
  b->prof = on != 0;
  for (int k = 0; k < GripBatch::NK; ++k) {
    b->k_ms[k] = 0.0;
    b->k_n[k] = 0;
  }
  CK(cudaMemsetAsync(b->D.stats, 0, 8 * sizeof(double), b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return 0;
}

int grip_kernel_stats(GripBatch* b, int kernel, double* ms, int64_t* launches, double* units /* 4 or NULL */) {
  if (kernel < 0 || kernel >= GripBatch::NK) {
    g_err = "kernel id out of range";
    return -1;
  }
  if (ms) *ms = b->k_ms[kernel];
  if (launches) *launches = b->k_n[kernel];
  if (units) CK(cudaMemcpy(units, b->D.stats, 8 * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

int grip_stream_timer(GripBatch* b, int start, double* ms) {
  if (!b->r0) {
    CK(cudaEventCreate(&b->r0));
    CK(cudaEventCreate(&b->r1));
  }
  if (start) {
    CK(cudaEventRecord(b->r0, b->stream));
    return 0;
  }
  CK(cudaEventRecord(b->r1, b->stream));
  CK(cudaEventSynchronize(b->r1));
  float f = 0.0f;
  CK(cudaEventElapsedTime(&f, b->r0, b->r1));
  if (ms) *ms = f;
  return 0;
}

#ifdef GRIP_PHASE_TIMING
int grip_debug_phase(unsigned long long* out) {
  CK(cudaMemcpyFromSymbol(out, g_phase, sizeof(unsigned long long) * 64));
  return 0;
}
#endif

int grip_last_step_stats(GripBatch* b, double* device_ms, int64_t* launches, int64_t* newton_sweeps) {
  if (device_ms) *device_ms = b->last_ms;
  if (launches) *launches = b->launches;
  if (newton_sweeps) *newton_sweeps = b->sweeps;
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// SDF kernels for the D1/D2 metrics; stateless, default stream, device 0
// of the calling thread's current device
// ---------------------------------------------------------------------------
namespace {
template <class T>
struct DevBuf {
  T* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  bool put(const T* h, size_t n) {
    if (cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)) != cudaSuccess) return false;
    return !n || cudaMemcpy(p, h, sizeof(T) * n, cudaMemcpyHostToDevice) == cudaSuccess;
  }
  bool alloc(size_t n) { return cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)) == cudaSuccess; }
};
}  // namespace

int grip_sdf_exact(const double* pts, int64_t n, const double* verts, int32_t n_verts, const int32_t* tris,
                   int32_t n_tris, const double* face_n, const double* edge_n, const double* vert_n, double* out) {
  if (n <= 0) return 0;
  DevBuf<double> dp, dv, dfn, den, dvn, dout;
  DevBuf<int> dt;
  if (!dp.put(pts, 3 * (size_t)n) || !dv.put(verts, 3 * (size_t)n_verts) || !dt.put(tris, 3 * (size_t)n_tris) ||
      !dfn.put(face_n, 3 * (size_t)n_tris) || !den.put(edge_n, 9 * (size_t)n_tris) ||
      !dvn.put(vert_n, 3 * (size_t)n_verts) || !dout.alloc(n)) {
    g_err = "grip_sdf_exact: device allocation / copy failed";
    return -1;
  }
  const int blocks = (int)std::min<int64_t>((n + 127) / 128, 148 * 16);
  k_sdf_exact<<<blocks, 128>>>(dp.p, n, dv.p, dt.p, n_tris, dfn.p, den.p, dvn.p, dout.p);
  CK(cudaGetLastError());
  CK(cudaMemcpy(out, dout.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return 0;
}

int grip_sdf_query(const double* values, const int32_t* dims, const double* origin, const double* spacing,
                   const double* rot, const double* trans, const double* world_lo, const double* world_hi,
                   const double* pts, int64_t n, double* d_o, double* d_max) {
  const size_t nv = (size_t)dims[0] * dims[1] * dims[2];
  DevBuf<double> dvals, dp, dR, dout;
  DevBuf<unsigned long long> dm;
  if (!dvals.put(values, nv) || !dp.put(pts, 3 * (size_t)std::max<int64_t>(n, 0)) || !dm.alloc(1) ||
      (rot && !dR.put(rot, 9)) || (d_o && !dout.alloc(std::max<int64_t>(n, 1)))) {
    g_err = "grip_sdf_query: device allocation / copy failed";
    return -1;
  }
  CK(cudaMemset(dm.p, 0, sizeof(unsigned long long)));
  SdfGridDev G{dvals.p, dims[0], dims[1], dims[2], origin[0], origin[1], origin[2], spacing[0], spacing[1], spacing[2]};
  const V3 lo{origin[0], origin[1], origin[2]};
  const V3 hi{origin[0] + spacing[0] * (dims[0] - 1), origin[1] + spacing[1] * (dims[1] - 1),
              origin[2] + spacing[2] * (dims[2] - 1)};
  const V3 T = trans ? V3{trans[0], trans[1], trans[2]} : V3{0, 0, 0};
  const V3 wlo = world_lo ? V3{world_lo[0], world_lo[1], world_lo[2]} : lo;
  const V3 whi = world_hi ? V3{world_hi[0], world_hi[1], world_hi[2]} : hi;
  if (n > 0) {
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_sdf_query<<<blocks, 256>>>(G, rot ? dR.p : nullptr, T, lo, hi, wlo, whi, dp.p, n, d_o ? dout.p : nullptr, dm.p);
    CK(cudaGetLastError());
  }
  unsigned long long u = 0;
  CK(cudaMemcpy(&u, dm.p, sizeof(u), cudaMemcpyDeviceToHost));
  if (d_o && n > 0) CK(cudaMemcpy(d_o, dout.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  if (n <= 0) {
    *d_max = -INFINITY;
  } else {
    u = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
    memcpy(d_max, &u, sizeof(double));
  }
  return 0;
}

int grip_sdf_nn(const double* pts, int64_t n, const double* cloud, int64_t m, const double* box_lo, const double* box_hi,
                int32_t levels, double* out) {
  if (n <= 0) return 0;
  const size_t nodes = ((size_t)2 << levels) - 1;
  DevBuf<double> dp, dc, dl, dh, dout;
  if (!dp.put(pts, 3 * (size_t)n) || !dc.put(cloud, 3 * (size_t)m) || !dl.put(box_lo, 3 * nodes) ||
      !dh.put(box_hi, 3 * nodes) || !dout.alloc(n)) {
    g_err = "grip_sdf_nn: device allocation / copy failed";
    return -1;
  }
  const int blocks = (int)std::min<int64_t>((n + 127) / 128, 148 * 32);
  k_sdf_nn<<<blocks, 128>>>(dp.p, n, dc.p, m, dl.p, dh.p, levels, dout.p);
  CK(cudaGetLastError());
  CK(cudaMemcpy(out, dout.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return 0;
}
