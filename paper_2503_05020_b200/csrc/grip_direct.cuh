// Direct linear solve of the Newton system (solver.py:91-131) for one env in one CTA:
// dense H_ff assembled in packed lower-triangular form (shared memory when it fits, else a
// per-env global scratch), right-looking Cholesky, forward/back substitution by one warp,
// then the reference's recipe: one refinement if |H p + g| > 1e-10 |g|, accept if
// <= 1e-8 |g|, else add 1e-8 max(diag, 1) to the diagonal and retry once, else
// SolveBreakdown.  H_ff is SPD (every element block is clamped PSD and M > 0), so
// Cholesky replaces SuperLU's LU with the same solution up to rounding.
#pragma once
#include "grip_kernels.cuh"

namespace grip {

__device__ __forceinline__ int pidx(int i, int j) { return i * (i + 1) / 2 + j; }  // i >= j

struct ElemMap {     // one contact element's slot -> free node map (per warp)
  int nn;            // distinct free nodes of the element
  int fnode[8];      // their free indices
  int skind[4];      // per slot: 0 soft free, 1 affine, 2 none
  int sf[4];         // per slot: free index (soft node or affine p-node)
  double sxi[4][3];
};

struct DirShared {
  AsmShared A;
  ElemMap em[NWARP];
  int ok;
};

// dense H_ff (+ shift on the diagonal) into packed L
__device__ void dense_assemble(const Dev& D, const EnvIx& E, double dt2, double shift, double* L, int n,
                               DirShared& S, double* kbuf) {
  const int e = E.e;
  const int* perm = D.dense_perm + E.f0;   // free node -> dense position (hub bodies last)
  const size_t elbase = (size_t)e * D.cap_el;
  const int tot = n * (n + 1) / 2;
  for (int i = threadIdx.x; i < tot; i += NT) L[i] = 0.0;
  __syncthreads();
  for (int f = threadIdx.x; f < E.nf; f += NT) {
    const int fg = E.f0 + f;
    for (int b = D.sb_rowptr[fg]; b < D.sb_rowptr[fg + 1]; ++b) {
      const int f2 = D.sb_col[b];
      const int pf = perm[f], pf2 = perm[f2];
      if (pf2 > pf) continue;   // keep the block that lands in the lower triangle
      const double* B = D.sb_val + 9 * (size_t)b;
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) {
          const int i = 3 * pf + c, j = 3 * pf2 + d;
          if (i >= j) L[pidx(i, j)] = B[3 * c + d] + (i == j ? shift : 0.0);
        }
    }
  }
  __syncthreads();
  // contact / friction elements, NWARP at a time: warp w computes K = J^T (dt^2 H) J of element
  // chunk+w into shared memory; then every warp adds, for the free nodes it owns
  // (f % NWARP == w), the chunk's K rows in element order -> deterministic, no write conflicts.
  const int nce = D.n_act[e] + D.n_anc[e];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < nce; c0 += NWARP) {
    const int k = c0 + warp;
    ElemMap& M = S.em[warp];
    double* K = kbuf + (size_t)warp * 576;
    if (k < nce) {
      const size_t sl = elbase + ce_slot(D, e, k);
      const int* ix = D.el_idx + sl * 4;
      const double* H = D.el_H + sl * 144;
      if (lane == 0) {
        int nn = 0;
        for (int u = 0; u < 4; ++u) {
          const int g = E.s0 + ix[u];
          const int kind = D.sv_kind[g];
          M.skind[u] = 2;
          if (kind == 2) continue;
          const int f = D.node_fidx[E.n0 + D.sv_node[g]];
          if (f < 0) continue;
          M.sf[u] = f;
          M.skind[u] = kind;  // 0 soft, 1 affine
          const int cnt = kind == 0 ? 1 : 4;
          for (int q = 0; q < cnt; ++q) {
            bool have = false;
            for (int r = 0; r < nn; ++r) have |= M.fnode[r] == f + q;
            if (!have) M.fnode[nn++] = f + q;
          }
          if (kind == 1)
            for (int c = 0; c < 3; ++c) M.sxi[u][c] = D.sv_xi[3 * (size_t)g + c];
        }
        M.nn = nn;
      }
      __syncwarp();
      const int nd = 3 * M.nn;
      for (int t = lane; t < nd * nd; t += 32) {
        const int r = t / nd, q = t % nd;
        const int Nr = M.fnode[r / 3], cr = r % 3, Nq = M.fnode[q / 3], cq = q % 3;
        double v = 0.0;
        for (int u = 0; u < 4; ++u) {
          int au = -1;
          double cu = 1.0;
          if (M.skind[u] == 0) {
            if (M.sf[u] == Nr) au = cr;
          } else if (M.skind[u] == 1) {
            const int o = Nr - M.sf[u];
            if (o == 0) au = cr;
            else if (o >= 1 && o <= 3) { au = o - 1; cu = M.sxi[u][cr]; }
          }
          if (au < 0) continue;
          for (int w = 0; w < 4; ++w) {
            int aw = -1;
            double cw = 1.0;
            if (M.skind[w] == 0) {
              if (M.sf[w] == Nq) aw = cq;
            } else if (M.skind[w] == 1) {
              const int o = Nq - M.sf[w];
              if (o == 0) aw = cq;
              else if (o >= 1 && o <= 3) { aw = o - 1; cw = M.sxi[w][cq]; }
            }
            if (aw < 0) continue;
            v += cu * cw * H[(3 * u + au) * 12 + 3 * w + aw];
          }
        }
        K[t] = dt2 * v;
      }
    }
    __syncthreads();
    const int kmax = min(NWARP, nce - c0);
    for (int w2 = 0; w2 < kmax; ++w2) {   // element order within the chunk
      const ElemMap& Mw = S.em[w2];
      const double* Kw = kbuf + (size_t)w2 * 576;
      const int nd = 3 * Mw.nn;
      for (int a = 0; a < Mw.nn; ++a) {
        const int Nr = Mw.fnode[a];
        if (Nr % NWARP != warp) continue;
        const int pr = perm[Nr];
        for (int t = lane; t < 3 * nd; t += 32) {
          const int cr = t / nd, q = t % nd;
          const int i = 3 * pr + cr, j = 3 * perm[Mw.fnode[q / 3]] + q % 3;
          if (i >= j) L[pidx(i, j)] += Kw[(3 * a + cr) * nd + q];
        }
      }
    }
    __syncthreads();
  }
}

// Blocked right-looking Cholesky of packed L in place (panel width 8); false on a
// non-positive pivot.  One warp factors each 8-column panel (warp barriers only), then all
// warps apply the rank-8 trailing update (8 FMAs per read-modify-write): 2 block barriers
// per panel instead of 3 per column.
constexpr int PW = 8;

__device__ bool dense_cholesky(double* L, int n, DirShared& S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int kb = 0; kb < n; kb += PW) {
    const int wb = min(PW, n - kb);
    if (warp == 0) {  // diagonal wb x wb block
      int ok = 1;
      for (int c = 0; c < wb; ++c) {
        const int k = kb + c;
        const double d = L[pidx(k, k)];
        ok = d > 0.0;
        if (!ok) break;
        const double lkk = sqrt(d);
        __syncwarp();
        if (lane == 0) L[pidx(k, k)] = lkk;
        const int i = k + 1 + lane;
        if (i < kb + wb) L[pidx(i, k)] /= lkk;
        __syncwarp();
        // remaining diagonal-block entries (i, j), k < j <= i < kb+wb: at most 28, one per lane
        int t = lane, ii = k + 1, jj = k + 1;
        for (;;) {   // lane -> (ii, jj) in the trailing diagonal triangle
          if (ii >= kb + wb) { ii = -1; break; }
          const int len = ii - (k + 1) + 1;
          if (t < len) { jj = k + 1 + t; break; }
          t -= len;
          ++ii;
        }
        if (ii >= 0) L[pidx(ii, jj)] -= L[pidx(ii, k)] * L[pidx(jj, k)];
        __syncwarp();
      }
      if (lane == 0) S.ok = ok;
    }
    __syncthreads();
    if (!S.ok) return false;
    const int j0 = kb + wb;
    // panel rows below the diagonal block: solve row * L_kk^T = row (one thread per row)
    for (int i = j0 + threadIdx.x; i < n; i += NT) {
      double* pi = L + pidx(i, kb);
      double r[PW];
      bool nz = false;
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        r[c] = c < wb ? pi[c] : 0.0;
        nz |= r[c] != 0.0;
      }
      if (!nz) continue;   // structurally decoupled row (e.g. the other pad): stays zero
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        if (c >= wb) break;
        const double* dc = L + pidx(kb + c, kb);
        double v = r[c];
#pragma unroll
        for (int q = 0; q < PW; ++q)
          if (q < c) v -= r[q] * dc[q];
        r[c] = v / dc[c];
      }
#pragma unroll
      for (int c = 0; c < PW; ++c)
        if (c < wb) pi[c] = r[c];
    }
    __syncthreads();
    // trailing: L[i][j] -= sum_{k in panel} L[i][k] L[j][k], j0 <= j <= i
    for (int i = j0 + warp; i < n; i += NWARP) {
      double li[PW];
      const double* pi = L + pidx(i, kb);
      bool nz = false;
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        li[c] = c < wb ? pi[c] : 0.0;
        nz |= li[c] != 0.0;
      }
      if (!nz) continue;   // L[i][panel] == 0 -> no update of row i
      double* row = L + pidx(i, 0);
      for (int j = j0 + lane; j <= i; j += 32) {
        const double* pj = L + pidx(j, kb);
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < PW; ++c)
          if (c < wb) acc += li[c] * pj[c];
        row[j] -= acc;
      }
    }
    __syncthreads();
  }
  return true;
}

// Solve L L^T x = b with all warps (blocked by 32: warp 0 solves each diagonal block, all
// warps update the rest).  x may alias b.  Call with the whole CTA.
__device__ void dense_solve(const double* L, int n, const double* b, double* x) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < n; i += NT) x[i] = b[i];
  __syncthreads();
  for (int kb = 0; kb < n; kb += 32) {            // forward: L y = b
    const int kend = min(kb + 32, n);
    if (warp == 0) {
      for (int k = kb; k < kend; ++k) {
        const double yk = x[k] / L[pidx(k, k)];
        __syncwarp();
        if (lane == 0) x[k] = yk;
        const int i = kb + lane;
        if (i > k && i < kend) x[i] -= L[pidx(i, k)] * yk;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = kend + threadIdx.x; i < n; i += NT) {
      const double* row = L + pidx(i, 0);
      double acc = 0.0;
      for (int k = kb; k < kend; ++k) acc += row[k] * x[k];
      x[i] -= acc;
    }
    __syncthreads();
  }
  for (int kb = ((n - 1) / 32) * 32; kb >= 0; kb -= 32) {  // backward: L^T x = y
    const int kend = min(kb + 32, n);
    if (warp == 0) {
      for (int k = kend - 1; k >= kb; --k) {
        const double xk = x[k] / L[pidx(k, k)];
        __syncwarp();
        if (lane == 0) x[k] = xk;
        const int i = kb + lane;
        if (i < k) x[i] -= L[pidx(k, i)] * xk;
        __syncwarp();
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kb; i += NT) {
      double acc = 0.0;
      for (int k = kb; k < kend; ++k) acc += L[pidx(k, i)] * x[k];
      x[i] -= acc;
    }
    __syncthreads();
  }
}

extern __shared__ double dyn_smem[];

#ifdef GRIP_PHASE_TIMING
__device__ unsigned long long g_phase[16];
#define PHASE(k)                                                   \
  do {                                                             \
    __syncthreads();                                               \
    if (threadIdx.x == 0) {                                        \
      const long long t = clock64();                               \
      atomicAdd(&g_phase[k], (unsigned long long)(t - t_last));    \
      t_last = t;                                                  \
    }                                                              \
  } while (0)
#else
#define PHASE(k) do {} while (0)
#endif

// Newton sweep 3/4 (direct): assembly + dense Cholesky solve of H_ff p = -g_f
__global__ void __launch_bounds__(NT) k_assemble_direct(Dev D, const int* list, int smem_dofs) {
  __shared__ DirShared S;
  AsmShared& A = S.A;
  Red& sm = A.sm;
  const int e = list[blockIdx.x];
  if (D.ns_done[e] || (D.flags[e] & FLAG_OVERFLOW)) return;
  const EnvIx E = env_ix(D, e);
  const double* P = P_(D, e);
  const double dt = P[GRIP_P_DT], dt2 = dt * dt;
  double Etot = 0.0;
#ifdef GRIP_PHASE_TIMING
  long long t_last = clock64();
#endif
  if (!asm_prologue(D, E, A, dt2, &Etot)) return;
  PHASE(0);
  const int n = 3 * E.nf;
  const size_t vb = (size_t)e * 3 * D.max_free;
  double* L = (n <= smem_dofs) ? dyn_smem : D.dense_L + (size_t)e * D.dense_stride;
  double* kbuf = dyn_smem + (size_t)smem_dofs * (smem_dofs + 1) / 2;   // NWARP x 576 element blocks
  double* X = D.pcg_x;
  double* Q = D.pcg_q;
  double* RHS = D.pcg_b;
  double bn2 = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) bn2 += RHS[vb + i] * RHS[vb + i];
  bn2 = block_sum(bn2, sm);
  bool solved = false;
  double shift = 0.0;
  if (bn2 == 0.0) {
    for (int i = threadIdx.x; i < n; i += NT) X[vb + i] = 0.0;
    __syncthreads();
    solved = true;
  }
  for (int attempt = 0; attempt < 2 && !solved; ++attempt) {
    if (attempt == 1) {
      double md = -INFINITY;
      for (int f = threadIdx.x; f < E.nf; f += NT) {
        const double* Bd = D.sb_val + 9 * (size_t)D.sb_diag[E.f0 + f];
        md = fmax(md, fmax(Bd[0], fmax(Bd[4], Bd[8])));
      }
      md = block_max(md, sm);
      shift = 1e-8 * fmax(md, 1.0);
      for (int f = threadIdx.x; f < E.nf; f += NT) {   // the refinement SpMV must see the shift too
        double* Bd = D.sb_val + 9 * (size_t)D.sb_diag[E.f0 + f];
        Bd[0] += shift; Bd[4] += shift; Bd[8] += shift;
      }
      if (threadIdx.x == 0) D.regularized[e] = 1;
      __syncthreads();
    }
    dense_assemble(D, E, dt2, 0.0, L, n, S, kbuf);   // sb_val already carries the shift
    PHASE(1);
    if (!dense_cholesky(L, n, S)) continue;
    PHASE(2);
    {
      const int* perm = D.dense_perm + E.f0;
      for (int f = threadIdx.x; f < E.nf; f += NT)
        for (int c = 0; c < 3; ++c) D.pcg_p[vb + 3 * perm[f] + c] = RHS[vb + 3 * f + c];
      __syncthreads();
      dense_solve(L, n, D.pcg_p + vb, D.pcg_z + vb);
      for (int f = threadIdx.x; f < E.nf; f += NT)
        for (int c = 0; c < 3; ++c) X[vb + 3 * f + c] = D.pcg_z[vb + 3 * perm[f] + c];
      __syncthreads();
    }
    PHASE(3);
    // refinement on the true residual (solver.py:117-122)
    int fin = 1;
    for (int i = threadIdx.x; i < n; i += NT) fin &= isfinite(X[vb + i]);
    fin = !block_or(!fin, sm);
    if (!fin) continue;
    spmv(D, E, dt2, X, Q, A);
    double r2 = 0.0;
    for (int i = threadIdx.x; i < n; i += NT) {
      const double r = RHS[vb + i] - Q[vb + i];
      D.pcg_r[vb + i] = r;
      r2 += r * r;
    }
    r2 = block_sum(r2, sm);
    if (r2 > 1e-20 * bn2) {
      const int* perm = D.dense_perm + E.f0;
      for (int f = threadIdx.x; f < E.nf; f += NT)
        for (int c = 0; c < 3; ++c) D.pcg_p[vb + 3 * perm[f] + c] = D.pcg_r[vb + 3 * f + c];
      __syncthreads();
      dense_solve(L, n, D.pcg_p + vb, D.pcg_z + vb);
      for (int f = threadIdx.x; f < E.nf; f += NT)
        for (int c = 0; c < 3; ++c) X[vb + 3 * f + c] += D.pcg_z[vb + 3 * perm[f] + c];
      __syncthreads();
      spmv(D, E, dt2, X, Q, A);
      r2 = 0.0;
      for (int i = threadIdx.x; i < n; i += NT) {
        const double r = RHS[vb + i] - Q[vb + i];
        r2 += r * r;
      }
      r2 = block_sum(r2, sm);
    }
    solved = isfinite(r2) && r2 <= 1e-16 * bn2;
  }
  PHASE(4);
  if (!solved) { fail_env(D, e, GRIP_R_SOLVE); return; }
  asm_converge(D, E, X, Etot, sm);
  PHASE(5);
}

}  // namespace grip
