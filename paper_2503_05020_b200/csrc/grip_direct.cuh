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

struct DirShared {
  AsmShared A;
  int nn;            // distinct free nodes of the current element
  int fnode[8];      // their free indices
  int skind[4];      // per slot: 0 soft free, 1 affine, 2 none
  int sf[4];         // per slot: free index (soft node or affine p-node)
  double sxi[4][3];
  int ok;
};

// dense H_ff (+ shift on the diagonal) into packed L
__device__ void dense_assemble(const Dev& D, const EnvIx& E, double dt2, double shift, double* L, int n,
                               DirShared& S) {
  const int e = E.e;
  const size_t elbase = (size_t)e * D.cap_el;
  const int tot = n * (n + 1) / 2;
  for (int i = threadIdx.x; i < tot; i += NT) L[i] = 0.0;
  __syncthreads();
  for (int f = threadIdx.x; f < E.nf; f += NT) {
    const int fg = E.f0 + f;
    for (int b = D.sb_rowptr[fg]; b < D.sb_rowptr[fg + 1]; ++b) {
      const int f2 = D.sb_col[b];
      if (f2 > f) continue;
      const double* B = D.sb_val + 9 * (size_t)b;
      for (int c = 0; c < 3; ++c)
        for (int d = 0; d < 3; ++d) {
          const int i = 3 * f + c, j = 3 * f2 + d;
          if (i >= j) L[pidx(i, j)] = B[3 * c + d] + (i == j ? shift : 0.0);
        }
    }
  }
  __syncthreads();
  // contact / friction elements: J^T (dt^2 H) J, element by element (fixed order -> deterministic)
  const int nce = D.n_act[e] + D.n_anc[e];
  for (int k = 0; k < nce; ++k) {
    const size_t sl = elbase + ce_slot(D, e, k);
    const int* ix = D.el_idx + sl * 4;
    const double* H = D.el_H + sl * 144;
    if (threadIdx.x == 0) {
      int nn = 0;
      for (int u = 0; u < 4; ++u) {
        const int g = E.s0 + ix[u];
        const int kind = D.sv_kind[g];
        S.skind[u] = 2;
        if (kind == 2) continue;
        const int f = D.node_fidx[E.n0 + D.sv_node[g]];
        if (f < 0) continue;
        S.sf[u] = f;
        S.skind[u] = kind;  // 0 soft, 1 affine
        const int cnt = kind == 0 ? 1 : 4;
        for (int q = 0; q < cnt; ++q) {
          bool have = false;
          for (int r = 0; r < nn; ++r) have |= S.fnode[r] == f + q;
          if (!have) S.fnode[nn++] = f + q;
        }
        if (kind == 1)
          for (int c = 0; c < 3; ++c) S.sxi[u][c] = D.sv_xi[3 * (size_t)g + c];
      }
      S.nn = nn;
    }
    __syncthreads();
    const int nd = 3 * S.nn;
    for (int t = threadIdx.x; t < nd * nd; t += NT) {
      const int r = t / nd, q = t % nd;
      const int Nr = S.fnode[r / 3], cr = r % 3, Nq = S.fnode[q / 3], cq = q % 3;
      const int i = 3 * Nr + cr, j = 3 * Nq + cq;
      if (i < j) continue;
      double v = 0.0;
      for (int u = 0; u < 4; ++u) {
        int au = -1;
        double cu = 1.0;
        if (S.skind[u] == 0) {
          if (S.sf[u] == Nr) au = cr;
        } else if (S.skind[u] == 1) {
          const int o = Nr - S.sf[u];
          if (o == 0) au = cr;
          else if (o >= 1 && o <= 3) { au = o - 1; cu = S.sxi[u][cr]; }
        }
        if (au < 0) continue;
        for (int w = 0; w < 4; ++w) {
          int aw = -1;
          double cw = 1.0;
          if (S.skind[w] == 0) {
            if (S.sf[w] == Nq) aw = cq;
          } else if (S.skind[w] == 1) {
            const int o = Nq - S.sf[w];
            if (o == 0) aw = cq;
            else if (o >= 1 && o <= 3) { aw = o - 1; cw = S.sxi[w][cq]; }
          }
          if (aw < 0) continue;
          v += cu * cw * H[(3 * u + au) * 12 + 3 * w + aw];
        }
      }
      L[pidx(i, j)] += dt2 * v;
    }
    __syncthreads();
  }
}

// right-looking Cholesky of packed L in place; false if a pivot is not positive
__device__ bool dense_cholesky(double* L, int n, DirShared& S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = 0; k < n; ++k) {
    if (threadIdx.x == 0) {
      const double d = L[pidx(k, k)];
      S.ok = d > 0.0;
      if (d > 0.0) L[pidx(k, k)] = sqrt(d);
    }
    __syncthreads();
    if (!S.ok) return false;
    const double lkk = L[pidx(k, k)];
    for (int i = k + 1 + threadIdx.x; i < n; i += NT) L[pidx(i, k)] /= lkk;
    __syncthreads();
    for (int i = k + 1 + warp; i < n; i += NWARP) {
      const double lik = L[pidx(i, k)];
      double* row = L + pidx(i, 0);
      for (int j = k + 1 + lane; j <= i; j += 32) row[j] -= lik * L[pidx(j, k)];
    }
    __syncthreads();
  }
  return true;
}

// solve L L^T x = b (warp 0), x and b may alias
__device__ void dense_solve(const double* L, int n, const double* b, double* x) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32) x[i] = b[i];
  __syncwarp();
  for (int k = 0; k < n; ++k) {
    const double yk = x[k] / L[pidx(k, k)];
    __syncwarp();
    if (lane == 0) x[k] = yk;
    for (int i = k + 1 + lane; i < n; i += 32) x[i] -= L[pidx(i, k)] * yk;
    __syncwarp();
  }
  for (int k = n - 1; k >= 0; --k) {
    const double xk = x[k] / L[pidx(k, k)];
    __syncwarp();
    if (lane == 0) x[k] = xk;
    const double* row = L + pidx(k, 0);
    for (int i = lane; i < k; i += 32) x[i] -= row[i] * xk;
    __syncwarp();
  }
}

extern __shared__ double dyn_smem[];

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
  if (!asm_prologue(D, E, A, dt2, &Etot)) return;
  const int n = 3 * E.nf;
  const size_t vb = (size_t)e * 3 * D.max_free;
  double* L = (n <= smem_dofs) ? dyn_smem : D.dense_L + (size_t)e * D.dense_stride;
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
    dense_assemble(D, E, dt2, 0.0, L, n, S);   // sb_val already carries the shift
    if (!dense_cholesky(L, n, S)) continue;
    dense_solve(L, n, RHS + vb, X + vb);
    __syncthreads();
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
      dense_solve(L, n, D.pcg_r + vb, D.pcg_z + vb);
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += NT) X[vb + i] += D.pcg_z[vb + i];
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
  if (!solved) { fail_env(D, e, GRIP_R_SOLVE); return; }
  asm_converge(D, E, X, Etot, sm);
}

}  // namespace grip
