// Direct linear solve of the Newton system (solver.py:91-131) for one env in one CTA: H_ff in
// skyline (envelope) storage, right-looking blocked Cholesky restricted to the envelope,
// forward/back substitution, then the reference's recipe: one refinement if |H p + g| >
// 1e-10 |g|, accept if <= 1e-8 |g|, else add 1e-8 max(diag, 1) to the diagonal and retry
// once, else SolveBreakdown.  H_ff is SPD (every element block is clamped PSD and M > 0),
// so Cholesky replaces SuperLU's LU with the same solution up to rounding.
//
// Dense ordering (host, grip_create): bodies grouped, hub bodies (the grasped object) last,
// reverse Cuthill-McKee inside every soft body.  Row i of the factor is stored from its first
// coupled column fc[i] (rounded down to the panel width) to the diagonal; fill-in of a
// Cholesky factor never leaves the envelope, so the pad blocks never couple and a pad's band
// stays narrow (config 1: 5.9k stored entries instead of 18.5k).
#pragma once
#include "grip_kernels.cuh"

namespace grip {

constexpr int PW = 8;       // panel width = envelope alignment
constexpr int RE_MAXP = 128;  // panels per segment with a row bound (longer segments: no pruning)
constexpr int MAXSEG = 8;   // independent segments factored concurrently (2 warp groups)

struct DirShared {
  AsmShared A;
  int ok[2];
  int nseg;                // independent row segments ahead of the tail (hub) rows
  int sc_next;             // sky_scatter_rows: next node (dynamic schedule)
  int seg[MAXSEG + 1];     // segment starts, seg[nseg] = tail start (DOFs)
  int rend[2][RE_MAXP];    // sky_panels: per panel, end of the rows whose envelope reaches it (per group)
};

// dynamic shared memory in front of the skyline: rdiag[nd] | xv[nd] | fcd[nd] | ro[nd+1] | fcn[max_free]
__host__ __device__ inline size_t dir_aux_bytes(int nd, int max_free) {
  const size_t b = (size_t)nd * 16 + ((size_t)2 * nd + 1 + max_free) * 4;
  return (b + 15) / 16 * 16;
}

struct Sky {
  double* L;
  const int* ro;   // row start offsets (ro[n] = stored entries)
  const int* fc;   // first stored column per row (multiple of PW)
  __device__ __forceinline__ double& at(int i, int j) const { return L[ro[i] + j - fc[i]]; }
};

// Per-iteration envelope: static first columns lowered by every contact element's node set
// (min is order independent, so the shared-memory atomics are deterministic).  Returns the
// stored entry count.
__device__ int sky_build(const Dev& D, const EnvIx& E, int* fcn, int* fcd, int* ro, DirShared& sh) {
  Red& sm = sh.A.sm;
  const int e = E.e, nf = E.nf, n = 3 * nf;
  for (int p = threadIdx.x; p < nf; p += NT) fcn[p] = D.dense_fc[E.f0 + p];
  __syncthreads();
  const int na = D.n_act[e], nce = na + D.n_anc[e];
  const size_t cs0 = (size_t)e * (D.cap_act + D.cap_anc);
  for (int t = threadIdx.x; t < 8 * nce; t += NT) {   // (element, node) pairs
    const int k = t >> 3, q = t & 7;
    const int* kn = D.el_kn + (cs0 + (k < na ? k : D.cap_act + (k - na))) * 9;
    if (q < kn[0]) atomicMin(&fcn[kn[1 + q]], kn[1]);   // nodes ascending: kn[1] is the lowest
  }
  __syncthreads();
  // independent segments of the rows ahead of the tail: a boundary at node p when no row
  // at or after p (before the tail) reaches a column before p
  if (threadIdx.x == 0) {
    const int hn = min(D.dense_tail[e], nf);
    int b[MAXSEG], nb = 0, m = 1 << 29;
    for (int p = hn - 1; p >= 1 && nb < MAXSEG - 1; --p) {
      m = min(m, fcn[p]);
      if (m >= p) b[nb++] = p;
    }
    int ns = 0;
    if (hn > 0) {
      sh.seg[ns++] = 0;
      for (int q = nb - 1; q >= 0; --q) sh.seg[ns++] = 3 * b[q];
    }
    sh.seg[ns] = 3 * hn;
    sh.nseg = ns;
  }
  __syncthreads();
  const int ns = sh.nseg;
  for (int i = threadIdx.x; i < n; i += NT) {
    const int f = 3 * fcn[i / 3];
    int ss = sh.seg[ns];   // alignment origin: the segment (or the tail) holding column f
    if (f < ss)
      for (int q = ns - 1; q >= 0; --q)
        if (sh.seg[q] <= f) { ss = sh.seg[q]; break; }
    const int fa = ss + ((f - ss) & ~(PW - 1));
    fcd[i] = fa;
    ro[i] = i - fa + 1;
  }
  __syncthreads();
  const int tot = block_scan_array(ro, n, sm);
  if (threadIdx.x == 0) ro[n] = tot;
  __syncthreads();
  return tot;
}

// H_ff into the skyline: the static blocks from sb_val (mass, dt^2 element blocks and any
// shift), then dt^2 J^T H J of the contact / friction elements (sky_scatter_contacts)
__device__ void sky_static(const Dev& D, const EnvIx& E, const Sky& S, int n) {
  const int tot = S.ro[n];
  for (int i = threadIdx.x; i < tot; i += NT) S.L[i] = 0.0;
  __syncthreads();
  const int b0 = D.sb_rowptr[E.f0], nb = D.sb_rowptr[E.f0 + E.nf] - b0;
  for (int t = threadIdx.x; t < nb; t += NT) {   // a block per thread, its 9 values loaded at once
    const int b = b0 + t;
    const int dst = D.sb_dst[b];
    if (dst < 0) continue;   // the mirrored block lands in the lower triangle
    const int pf = dst >> 16, pf2 = dst & 0xffff;
    double v[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) v[q] = D.sb_val[9 * (size_t)b + q];
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const int i = 3 * pf + q / 3, j = 3 * pf2 + q % 3;
      if (i >= j) S.at(i, j) = v[q];
    }
  }
  __syncthreads();
}

// The contact / friction elements' K into the skyline, row node by row node: every entry of
// the lower triangle belongs to the rows of exactly one dense node I, so the warp that owns I
// adds, for each element containing I in ascending element order, that element's entries of
// I's rows (columns of its nodes at or before I).  Rows of different nodes never share an
// entry, so the warps run without synchronisation, and each entry still accumulates its
// elements in element order (bitwise the same sums as the former turn-ordered scatter).
// Node lists: counting sort of the (element, node slot) items by node; short lists are then
// sorted by element, long ones (the hub nodes every object contact touches) are walked by
// scanning all elements in order instead.
constexpr int SC_LONG = 48;
__device__ void sky_scatter_rows(const Dev& D, const EnvIx& E, const Sky& S, DirShared& sh) {
  Red& sm = sh.A.sm;
  const int e = E.e, nf = E.nf;
  const int na = D.n_act[e];
  const int nce = na + D.n_anc[e];
  const size_t cs0 = (size_t)e * (D.cap_act + D.cap_anc);
  int* off = D.sc_off + (size_t)e * 2 * (D.max_free + 1);
  int* cur = off + (D.max_free + 1);
  int* lst = D.sc_lst + (size_t)e * 8 * (D.cap_act + D.cap_anc);
  const int lane = threadIdx.x & 31;
  auto slot_of = [&](int k) { return cs0 + (k < na ? k : D.cap_act + (k - na)); };
  for (int p = threadIdx.x; p < nf; p += NT) off[p] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < 8 * nce; t += NT) {
    const int* kn = D.el_kn + slot_of(t >> 3) * 9;
    if ((t & 7) < kn[0]) atomicAdd(&off[kn[1 + (t & 7)]], 1);
  }
  __syncthreads();
  const int tot = block_scan_array(off, nf, sm);
  if (threadIdx.x == 0) off[nf] = tot;
  for (int p = threadIdx.x; p < nf; p += NT) cur[p] = off[p];
  __syncthreads();
  for (int t = threadIdx.x; t < 8 * nce; t += NT) {
    const int* kn = D.el_kn + slot_of(t >> 3) * 9;
    if ((t & 7) < kn[0]) lst[atomicAdd(&cur[kn[1 + (t & 7)]], 1)] = t;   // t == (k << 3) | slot
  }
  __syncthreads();
  for (int p = threadIdx.x; p < nf; p += NT) {
    const int lo = off[p], hi = off[p + 1];
    if (hi - lo > SC_LONG) continue;
    for (int a = lo + 1; a < hi; ++a) {
      const int t = lst[a];
      int b = a - 1;
      while (b >= lo && lst[b] > t) {
        lst[b + 1] = lst[b];
        --b;
      }
      lst[b + 1] = t;
    }
  }
  if (threadIdx.x == 0) sh.sc_next = 0;
  __syncthreads();
  // nodes are dealt out to the warps one at a time, last node first: the hub nodes (last in
  // the dense order, with the long element walks) start at once and the other warps share the
  // short lists, instead of a hub walk queued behind a warp's share of short ones
  for (;;) {
    int R = 0;
    if (lane == 0) R = atomicAdd(&sh.sc_next, 1);
    R = __shfl_sync(0xffffffffu, R, 0);
    if (R >= nf) break;
    const int I = nf - 1 - R;
    const int lo = off[I], hi = off[I + 1];
    if (hi == lo) continue;
    const bool scan_all = hi - lo > SC_LONG;
    const int cnt = scan_all ? nce : hi - lo;
    // chunks of SCH elements: every lane gathers its (address, value) pairs of all of them
    // first (the loads overlap), then they are added element by element, in order
    constexpr int SCH = 4;
    for (int u0 = 0; u0 < cnt; u0 += SCH) {
      int addr[SCH][3];
      double val[SCH][3];
#pragma unroll
      for (int c = 0; c < SCH; ++c) {
        const int u = u0 + c;
        int k = -1, a = -1;
        if (u < cnt) {
          if (scan_all) {
            const int* kn = D.el_kn + slot_of(u) * 9;
            const int nn = kn[0];
#pragma unroll
            for (int q = 0; q < 8; ++q) {   // all nine loads issued at once (no nn-dependent loop)
              const int v = kn[1 + q];
              if (q < nn && v == I) a = q;
            }
            k = a >= 0 ? u : -1;
          } else {
            const int t = lst[lo + u];
            k = t >> 3;
            a = t & 7;
          }
        }
        const int* kn = k >= 0 ? D.el_kn + slot_of(k) * 9 : nullptr;
        const double* K = k >= 0 ? D.el_K + slot_of(k) * 300 : nullptr;
        const int nent = k >= 0 ? 9 * a + 6 : 0;   // rows 3a..3a+2, columns 0..row
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          const int t = lane + 32 * m;
          addr[c][m] = -1;
          val[c][m] = 0.0;
          if (t < nent) {
            const int ri = t < 3 * a + 1 ? 0 : (t < 6 * a + 3 ? 1 : 2);
            const int q = t - (ri == 0 ? 0 : (ri == 1 ? 3 * a + 1 : 6 * a + 3));
            const int r = 3 * a + ri;
            const int i = 3 * I + ri, j = 3 * kn[1 + q / 3] + q % 3;
            addr[c][m] = S.ro[i] + j - S.fc[i];
            val[c][m] = K[r * (r + 1) / 2 + q];
          }
        }
      }
#pragma unroll
      for (int c = 0; c < SCH; ++c) {   // one element at a time: an address shared by two
#pragma unroll                          // elements may sit in different lanes
        for (int m = 0; m < 3; ++m)
          if (addr[c][m] >= 0) S.L[addr[c][m]] += val[c][m];
        __syncwarp();
      }
    }
  }
  __syncthreads();
}

// A warp group: the whole CTA (barrier 0) or half of it (named barriers 1, 2)
struct Grp {
  int t, nt, w, nw, id;
  __device__ __forceinline__ void sync() const {
    if (id == 0) __syncthreads();
    else if (id == 1) asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory");
    else asm volatile("bar.sync 2, %0;" ::"r"(nt) : "memory");
  }
};

// Factor the wb x wb diagonal block at kb in registers (lane j holds column j); false on a
// non-positive pivot.  Call with one full warp.
__device__ __forceinline__ bool diag_factor(const Sky& S, double* rdiag, int kb, int wb, int lane) {
  double a[PW];
#pragma unroll
  for (int i = 0; i < PW; ++i)
    a[i] = (lane < wb && i < wb && i >= lane) ? S.at(kb + i, kb + lane) : (i == lane ? 1.0 : 0.0);
  bool ok = true;
#pragma unroll
  for (int c = 0; c < PW; ++c) {
    if (c < wb) {
      const double d = __shfl_sync(0xffffffffu, a[c], c);
      if (!(d > 0.0)) { ok = false; break; }
      const double rk = rsqrt(d);
      double lc[PW];
#pragma unroll
      for (int i = 0; i < PW; ++i) lc[i] = i > c ? __shfl_sync(0xffffffffu, a[i], c) * rk : 0.0;
      double lj = 0.0;
#pragma unroll
      for (int i = 0; i < PW; ++i)
        if (i == lane) lj = lc[i];
      if (lane == c) {
        a[c] = d * rk;
#pragma unroll
        for (int i = 0; i < PW; ++i)
          if (i > c) a[i] = lc[i];
        rdiag[kb + c] = rk;
      } else if (lane > c) {
#pragma unroll
        for (int i = 0; i < PW; ++i)
          if (i >= lane) a[i] -= lc[i] * lj;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < PW; ++i)
    if (ok && lane < wb && i < wb && i >= lane) S.at(kb + i, kb + lane) = a[i];
  return ok;
}

// Right-looking panels over columns [c0, c1): the diagonal blocks, the panel solve and the
// rank-PW update of rows [j0, c1) and of the extra rows [x0, n) (the tail, whose updates are
// limited to columns < c1).  Rows / columns whose envelope starts after a panel are
// structurally zero in it and skipped.  Look-ahead: the group's first warp updates the next
// panel's diagonal block (rows [j0, j0 + PW) of the trailing update) and factors it while the
// other warps update the remaining rows, so a panel costs two barriers and the serial diagonal
// factorisation overlaps the trailing update.  Returns false on a non-positive pivot.
__device__ __forceinline__ void trail_row(const Sky& S, int i, int kb, int wb, int j0, int c1, int lane) {
  if (S.fc[i] > kb) return;   // L[i][j] -= L[i][panel] . L[j][panel]
  const double* pi = &S.at(i, kb);
  double li[PW];
  bool nz = false;
#pragma unroll
  for (int c = 0; c < PW; ++c) {
    li[c] = c < wb ? pi[c] : 0.0;
    nz |= li[c] != 0.0;
  }
  if (!nz) return;
  double* row = S.L + S.ro[i] - S.fc[i];
  const int jend = min(i, c1 - 1);
  for (int j = j0 + lane; j <= jend; j += 32) {
    const int fj = S.fc[j];
    if (fj > kb) continue;
    const double* pj = S.L + S.ro[j] + kb - fj;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < PW; ++c)
      if (c < wb) acc += li[c] * pj[c];
    row[j] -= acc;
  }
}

// L[i][j] -= L[i][panel] . L[j][panel] for one entry (the same c order as a row-wise update, so
// the same doubles); rows whose envelope starts after the panel are structurally zero in it
__device__ __forceinline__ void trail_pair(const Sky& S, int i, int j, int kb, int wb) {
  if (S.fc[i] > kb || S.fc[j] > kb) return;
  const double* pi = &S.at(i, kb);
  const double* pj = &S.at(j, kb);
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < PW; ++c)
    if (c < wb) acc += pi[c] * pj[c];
  S.at(i, j) -= acc;
}

// Trailing update of a panel as a flat list of (row, column) entries (not a warp per row: a
// banded row has only ~ the bandwidth of columns, so most lanes of a row-wise warp idled).
// Rows [j0, re) (re: the last row whose envelope reaches the panel, from the group's rend
// table) x columns [j0, row], then the extra rows [x0, n) x columns [j0, c1).  The group's first
// warp takes the next diagonal block's rows [j0, j0 + nb) (look-ahead), the other warps the rest.
__device__ bool sky_panels(const Sky& S, double* rdiag, int c0, int c1, int x0, int n, const Grp& G, int* okf,
                           int* rend) {
  static_assert(NT / 64 >= 2, "look-ahead needs two warps per group");
  const int lane = G.t & 31;
  if (c0 >= c1) return true;
  const int np = (c1 - c0 + PW - 1) / PW;
  const bool pruned = np <= RE_MAXP;
  if (pruned) {   // rend[p] = 1 + last row whose envelope starts in panel p (prefix max below)
    for (int p = G.t; p < np; p += G.nt) rend[p] = 0;
    G.sync();
    for (int i = c0 + G.t; i < c1; i += G.nt)   // (tail rows' envelopes start before the tail)
      atomicMax(&rend[S.fc[i] <= c0 ? 0 : (S.fc[i] - c0) / PW], i + 1);
  }
  if (G.w == 0) {
    const bool ok = diag_factor(S, rdiag, c0, min(PW, c1 - c0), lane);
    if (lane == 0) *okf = ok;
  }
  G.sync();
  int reach = c0;   // running prefix max of rend
  for (int kb = c0; kb < c1; kb += PW) {
    if (!*okf) return false;
    const int wb = min(PW, c1 - kb);
    const int j0 = kb + wb;
    if (pruned) reach = max(reach, rend[(kb - c0) / PW]);
    const int re = pruned ? min(max(reach, j0), c1) : c1;
    const int nband = re - j0, ntail = n - x0;
    const int nrow = nband + ntail;
    for (int t = G.t; t < nrow; t += G.nt) {   // panel rows: r * L_kk^T = row
      const int i = t < nband ? j0 + t : x0 + t - nband;
      if (S.fc[i] > kb) continue;
      double* pi = &S.at(i, kb);
      double r[PW];
      bool nz = false;
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        r[c] = c < wb ? pi[c] : 0.0;
        nz |= r[c] != 0.0;
      }
      if (!nz) continue;
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        if (c >= wb) break;
        const double* dc = &S.at(kb + c, kb);
        double v = r[c];
#pragma unroll
        for (int q = 0; q < PW; ++q)
          if (q < c) v -= r[q] * dc[q];
        r[c] = v * rdiag[kb + c];
      }
#pragma unroll
      for (int c = 0; c < PW; ++c)
        if (c < wb) pi[c] = r[c];
    }
    G.sync();
    const int nb = min(PW, c1 - j0);   // rows of the next diagonal block
    if (G.w == 0) {
      for (int u = lane; u < nb * (nb + 1) / 2; u += 32) {
        int ii = 0;
        while ((ii + 1) * (ii + 2) / 2 <= u) ++ii;
        trail_pair(S, j0 + ii, j0 + u - ii * (ii + 1) / 2, kb, wb);
      }
      if (nb > 0) {
        __syncwarp();
        const bool ok = diag_factor(S, rdiag, j0, nb, lane);
        if (lane == 0) *okf = ok;
      }
    } else {
      const int m = nband, t0 = nb * (nb + 1) / 2;
      const int nbandp = m > nb ? m * (m + 1) / 2 - t0 : 0;
      const int ntot = nbandp + ntail * (c1 - j0);
      for (int u = G.t - 32; u < ntot; u += G.nt - 32) {
        if (u < nbandp) {
          const int t = u + t0;
          int ii = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
          while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
          while (ii * (ii + 1) / 2 > t) --ii;
          trail_pair(S, j0 + ii, j0 + t - ii * (ii + 1) / 2, kb, wb);
        } else {
          const int v = u - nbandp, w = c1 - j0;
          trail_pair(S, x0 + v / w, j0 + v % w, kb, wb);
        }
      }
    }
    G.sync();
  }
  return true;   // the last panel has no next block: *okf was checked at its top (and is not
}                // re-read here, the caller's next segment may already be writing it)

__device__ __forceinline__ Grp seg_group(int nseg) {
  const int G2 = nseg >= 2;
  Grp g;
  if (G2) {
    const int half = NT / 2;
    g.id = 1 + (threadIdx.x >= half);
    g.t = threadIdx.x - (g.id - 1) * half;
    g.nt = half;
  } else {
    g.id = 0;
    g.t = threadIdx.x;
    g.nt = NT;
  }
  g.w = g.t >> 5;
  g.nw = g.nt >> 5;
  return g;
}

// Skyline Cholesky in place: the independent segments concurrently (two warp groups), the
// segment x segment products into the tail x tail block, then the tail.  False on a
// non-positive pivot (all threads agree).
__device__ bool sky_cholesky(const Sky& S, double* rdiag, int n, DirShared& sh) {
  const int ns = sh.nseg, h = sh.seg[ns];
  const Grp G = seg_group(ns);
  const int gi = G.id == 0 ? 0 : G.id - 1, ng = G.id == 0 ? 1 : 2;
  if (threadIdx.x == 0) { sh.ok[0] = 1; sh.ok[1] = 1; }
  __syncthreads();
#ifdef GRIP_PHASE_TIMING
  long long c_t0 = clock64();
#endif
  for (int q = gi; q < ns; q += ng)
    if (!sky_panels(S, rdiag, sh.seg[q], sh.seg[q + 1], h, n, G, &sh.ok[gi], sh.rend[gi])) break;
  __syncthreads();
#ifdef GRIP_PHASE_TIMING
  long long c_t1 = clock64();
  if (threadIdx.x == 0) {
    GSTAT(56, c_t1 - c_t0);
    GSTAT(59, ns);
    GSTAT(60, n);
    GSTAT(61, n - h);
  }
#endif
  if (!sh.ok[0] || !sh.ok[1]) return false;
  if (h > 0) {   // tail x tail -= sum over segment columns (fixed-order warp reduction)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = n - h, ne = m * (m + 1) / 2;
    for (int t = warp; t < ne; t += NWARP) {
      int ii = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
      while ((ii + 1) * (ii + 2) / 2 <= t) ++ii;
      while (ii * (ii + 1) / 2 > t) --ii;
      const int jj = t - ii * (ii + 1) / 2;
      const int i = h + ii, j = h + jj;
      const int lo = max(S.fc[i], S.fc[j]);
      const double* ri = S.L + S.ro[i] - S.fc[i];
      const double* rj = S.L + S.ro[j] - S.fc[j];
      double acc = 0.0;
      for (int k = lo + lane; k < h; k += 32) acc += ri[k] * rj[k];
      acc = wsum(acc);
      if (lane == 0) S.at(i, j) -= acc;
    }
    __syncthreads();
  }
  const Grp A{(int)threadIdx.x, NT, (int)threadIdx.x >> 5, NWARP, 0};
#ifdef GRIP_PHASE_TIMING
  long long c_t2 = clock64();
  if (threadIdx.x == 0) GSTAT(57, c_t2 - c_t1);
#endif
  const bool ok = sky_panels(S, rdiag, h, n, n, n, A, &sh.ok[0], sh.rend[0]);
#ifdef GRIP_PHASE_TIMING
  if (threadIdx.x == 0) GSTAT(58, clock64() - c_t2);
#endif
  return ok;
}

// Forward / backward substitution over columns [c0, c1) by one group, blocks of 32 (the
// group's first warp solves each diagonal block, the group updates rows [c0, c1)).
__device__ void seg_forward(const Sky& S, const double* rdiag, int c0, int c1, double* x, const Grp& G) {
  const int lane = G.t & 31;
  for (int kb = c0; kb < c1; kb += 32) {
    const int kend = min(kb + 32, c1);
    if (G.w == 0) {   // diagonal block in registers: lane i holds x[i], y_k by shuffle
      const int i = kb + lane;
      const bool in = i < kend;
      const int fi = in ? S.fc[i] : c1;
      const double* row = S.L + (in ? S.ro[i] - fi : 0);
      double xi = in ? x[i] : 0.0;
      const double rd = in ? rdiag[i] : 0.0;
      for (int k = kb; k < kend; ++k) {
        const double yk = __shfl_sync(0xffffffffu, xi * rd, k - kb);
        if (i == k) xi = yk;
        if (i > k && in && fi <= k) xi -= row[k] * yk;
      }
      if (in) x[i] = xi;
    }
    G.sync();
    for (int i = kend + G.t; i < c1; i += G.nt) {
      const int fi = S.fc[i], lo = max(kb, fi);
      if (lo >= kend) continue;
      const double* row = S.L + S.ro[i] - fi;
      double acc = 0.0;
      for (int k = lo; k < kend; ++k) acc += row[k] * x[k];
      x[i] -= acc;
    }
    G.sync();
  }
}

__device__ void seg_backward(const Sky& S, const double* rdiag, int c0, int c1, double* x, const Grp& G) {
  const int lane = G.t & 31;
  for (int kb = c0 + ((c1 - 1 - c0) / 32) * 32; kb >= c0; kb -= 32) {
    const int kend = min(kb + 32, c1);
    if (G.w == 0) {   // diagonal block in registers: lane i holds x[i], x_k by shuffle
      const int i = kb + lane;
      const bool in = i < kend;
      double xi = in ? x[i] : 0.0;
      const double rd = in ? rdiag[i] : 0.0;
      for (int k = kend - 1; k >= kb; --k) {
        const double xk = __shfl_sync(0xffffffffu, xi * rd, k - kb);
        if (i == k) xi = xk;
        const int fk = S.fc[k];
        if (i < k && i >= fk) xi -= S.L[S.ro[k] + i - fk] * xk;
      }
      if (in) x[i] = xi;
    }
    G.sync();
    for (int i = c0 + G.t; i < kb; i += G.nt) {
      double acc = 0.0;
      for (int k = kb; k < kend; ++k) {
        const int fk = S.fc[k];
        if (fk <= i) acc += S.L[S.ro[k] + i - fk] * x[k];
      }
      x[i] -= acc;
    }
    G.sync();
  }
}

// Solve L L^T x = b in place (x in shared memory).  Call with the whole CTA.
__device__ void sky_solve(const Sky& S, const double* rdiag, int n, double* x, const DirShared& sh) {
  const int ns = sh.nseg, h = sh.seg[ns];
  const Grp G = seg_group(ns);
  const int gi = G.id == 0 ? 0 : G.id - 1, ng = G.id == 0 ? 1 : 2;
  const Grp A{(int)threadIdx.x, NT, (int)threadIdx.x >> 5, NWARP, 0};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = gi; q < ns; q += ng) seg_forward(S, rdiag, sh.seg[q], sh.seg[q + 1], x, G);
  __syncthreads();
  if (h > 0) {
    for (int i = h + warp; i < n; i += NWARP) {   // tail rows -= L[i][segments] . y
      const double* ri = S.L + S.ro[i] - S.fc[i];
      double acc = 0.0;
      for (int k = S.fc[i] + lane; k < h; k += 32) acc += ri[k] * x[k];
      acc = wsum(acc);
      if (lane == 0) x[i] -= acc;
    }
    __syncthreads();
  }
  seg_forward(S, rdiag, h, n, x, A);
  seg_backward(S, rdiag, h, n, x, A);
  if (h > 0) {
    for (int i = threadIdx.x; i < h; i += NT) {   // segment rows -= L[tail][i]^T . x_tail
      double acc = 0.0;
      for (int k = h; k < n; ++k) {
        const int fk = S.fc[k];
        if (fk <= i) acc += S.L[S.ro[k] + i - fk] * x[k];
      }
      x[i] -= acc;
    }
    __syncthreads();
  }
  for (int q = gi; q < ns; q += ng) seg_backward(S, rdiag, sh.seg[q], sh.seg[q + 1], x, G);
  __syncthreads();
}

// Per contact / friction element: K = dt^2 J^T H J over its free DOFs, J the surface-vertex ->
// DOF map (soft vertex: identity on its node; ABD vertex: [I, xi0 I, xi1 I, xi2 I] on the
// body's translation and A-row nodes), stored as the lower triangle in dense order with the
// element's node list (el_K / el_kn), so the assembly only adds entries (solver.py:542-586).
// CTA per env, warp per element: T = H J then K = J^T T from per-DOF slot tables.
struct KWS {
  double H[144];
  double kx[12];   // affine-slot material coordinates
  double kj[96];   // per DOF: the 4 slot coefficients of its J column
  double kt[288];  // H J (12 x nd)
  int kr[96];      // ... and the H rows they pick
  int kc[4];       // slot codes (sv_code)
  int kn[8];       // node list (dense positions, ascending)
  int knn;
};

constexpr int KT = 256;   // k_contact_K: flat kernel, warp per element
__global__ void __launch_bounds__(KT) k_contact_K(Dev D, const int* list, int n) {
  constexpr int NWARP = KT / 32;
  __shared__ KWS ws[NWARP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  KWS& w = ws[warp];
  const int total = D.cwork_off[n];
  // flat over the contact elements of all listed envs (cwork_off from k_candidates' last CTA), warp each
  for (int item = blockIdx.x * NWARP + warp; item < total; item += gridDim.x * NWARP) {
    int lo = 0, hi = n;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (D.cwork_off[mid] <= item) lo = mid;
      else hi = mid;
    }
    const int e = list[lo], k = item - D.cwork_off[lo];
    const int s0 = D.sv_off[e];
    const size_t elbase = (size_t)e * D.cap_el;
    const int na = D.n_act[e];
    const double dt = P_(D, e)[GRIP_P_DT], dt2 = dt * dt;
    const int kk = k < na ? k : D.cap_act + (k - na);
    const size_t slot = elbase + D.max_tet + D.max_abd + kk;
    const size_t cs = (size_t)e * (D.cap_act + D.cap_anc) + kk;
    for (int t = lane; t < 144; t += 32) w.H[t] = D.el_H[slot * 144 + t];
    const int src = lane < 12 ? lane / 3 : 0;
    const int g = s0 + D.el_idx[slot * 4 + src];
    const int cd = D.sv_code[g];   // affine: translation node, A rows follow
    const double xv = lane < 12 ? D.sv_xi[3 * (size_t)g + lane % 3] : 0.0;
    const int kcv = __shfl_sync(0xffffffffu, cd, lane < 4 ? 3 * lane : 0);
    if (lane < 4) w.kc[lane] = kcv;
    if (lane < 12) w.kx[lane] = (cd >= 0 && (cd & 3)) ? xv : 0.0;
    __syncwarp();
    if (lane == 0) {
      int m = 0;
      for (int u = 0; u < 4; ++u) {
        const int c = w.kc[u];
        if (c < 0) continue;
        const int P = c >> 2, cnt = (c & 3) ? 4 : 1;
        bool have = false;
        for (int r = 0; r < m; ++r) have |= w.kn[r] == P;
        if (have) continue;   // second slot on the same affine body (or the same node)
        for (int q = 0; q < cnt; ++q) w.kn[m++] = P + q;
      }
      w.knn = m;
    }
    __syncwarp();
    const int nn = w.knn;
    {
      const int my = lane < nn ? w.kn[lane] : 0;
      int rank = 0;
      for (int q = 0; q < nn; ++q) rank += w.kn[q] < my;
      __syncwarp();
      if (lane < nn) w.kn[rank] = my;
      __syncwarp();
    }
    const int nd = 3 * nn, ne = nd * (nd + 1) / 2;
    if (lane < nd) {   // J column of DOF lane: per slot the H row it picks and its coefficient
      const int Nr = w.kn[lane / 3], cr = lane % 3;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = w.kc[u];
        int row = 0;
        double cf = 0.0;
        if (c >= 0) {
          const int o = Nr - (c >> 2);
          if ((c & 3) == 0) {
            if (o == 0) { row = 3 * u + cr; cf = 1.0; }
          } else if (o == 0) {
            row = 3 * u + cr; cf = 1.0;
          } else if (o >= 1 && o <= 3) {
            row = 3 * u + o - 1; cf = w.kx[3 * u + cr];
          }
        }
        w.kj[4 * lane + u] = cf;
        w.kr[4 * lane + u] = row;
      }
    }
    __syncwarp();
    double* kt = w.kt;
    for (int t = lane; t < 12 * nd; t += 32) {   // T = H J
      const int a = t / nd, d = t - a * nd;
      double v = 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) v += w.kj[4 * d + u] * w.H[12 * a + w.kr[4 * d + u]];
      kt[t] = v;
    }
    __syncwarp();
    double* Ko = D.el_K + cs * 300;
    for (int t = lane; t < ne; t += 32) {        // K = J^T T, lower triangle
      int r = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
      while ((r + 1) * (r + 2) / 2 <= t) ++r;
      while (r * (r + 1) / 2 > t) --r;
      const int q = t - r * (r + 1) / 2;
      double v = 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) v += w.kj[4 * r + u] * kt[w.kr[4 * r + u] * nd + q];
      Ko[t] = dt2 * v;
    }
    if (lane < 9) D.el_kn[cs * 9 + lane] = lane == 0 ? nn : (lane - 1 < nn ? w.kn[lane - 1] : -1);
    __syncwarp();
  }
}

extern __shared__ double dyn_smem[];

#ifdef GRIP_PHASE_TIMING
#define PHASE(k)                                  \
  do {                                            \
    __syncthreads();                              \
    if (threadIdx.x == 0) {                       \
      const long long t = clock64();              \
      ph[k] += t - t_last;                        \
      t_last = t;                                 \
    }                                             \
  } while (0)
#else
#define PHASE(k) do {} while (0)
#endif

// Newton sweep 3/4 (direct): assembly + skyline Cholesky solve of H_ff p = -g_f
__global__ void __launch_bounds__(NT, NT_MINB3) k_assemble_direct(Dev D, const int* list, int env_cap) {
  __shared__ DirShared S;
  AsmShared& A = S.A;
  Red& sm = A.sm;
  const int e = list[blockIdx.x];
  CTA_TIMER(2, e);
  if (D.ns_done[e] || (D.flags[e] & FLAG_OVERFLOW)) return;
  const EnvIx E = env_ix(D, e);
  const double* P = P_(D, e);
  const double dt = P[GRIP_P_DT], dt2 = dt * dt;
  double Etot = 0.0;
#ifdef GRIP_PHASE_TIMING
  long long t_last = clock64(), ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  if (!asm_prologue(D, E, A, dt2, &Etot)) return;
  PHASE(0);
  const int n = 3 * E.nf;
  const int nd = 3 * D.max_free;
  double* rdiag = dyn_smem;
  double* xv = rdiag + nd;
  int* fcd = reinterpret_cast<int*>(xv + nd);
  int* ro = fcd + nd;
  int* fcn = ro + nd + 1;
  double* Lsm = dyn_smem + dir_aux_bytes(nd, D.max_free) / sizeof(double);
  const size_t vb = (size_t)e * 3 * D.max_free;
  const int* perm = D.dense_perm + E.f0;
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
  Sky L{nullptr, ro, fcd};
  if (!solved) {
    const int tot = sky_build(D, E, fcn, fcd, ro, S);
    L.L = tot <= env_cap ? Lsm : D.dense_L + (size_t)e * D.dense_stride;
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
    sky_static(D, E, L, n);
    PHASE(1);
    sky_scatter_rows(D, E, L, S);
    PHASE(2);
    const bool chol_ok = sky_cholesky(L, rdiag, n, S);
    PHASE(3);
    if (!chol_ok) continue;
    for (int f = threadIdx.x; f < E.nf; f += NT)
      for (int c = 0; c < 3; ++c) xv[3 * perm[f] + c] = RHS[vb + 3 * f + c];
    __syncthreads();
    sky_solve(L, rdiag, n, xv, S);
    for (int f = threadIdx.x; f < E.nf; f += NT)
      for (int c = 0; c < 3; ++c) X[vb + 3 * f + c] = xv[3 * perm[f] + c];
    __syncthreads();
    PHASE(4);
    // refinement on the true residual (solver.py:117-122)
    int fin = 1;
    for (int i = threadIdx.x; i < n; i += NT) fin &= isfinite(X[vb + i]);
    fin = !block_or(!fin, sm);
    if (!fin) continue;
    spmv(D, E, dt2, X, Q, A);
    double r2 = 0.0;
    for (int f = threadIdx.x; f < E.nf; f += NT)
      for (int c = 0; c < 3; ++c) {
        const double r = RHS[vb + 3 * f + c] - Q[vb + 3 * f + c];
        xv[3 * perm[f] + c] = r;
        r2 += r * r;
      }
    r2 = block_sum(r2, sm);
    if (r2 > 1e-20 * bn2) {
      sky_solve(L, rdiag, n, xv, S);
      for (int f = threadIdx.x; f < E.nf; f += NT)
        for (int c = 0; c < 3; ++c) X[vb + 3 * f + c] += xv[3 * perm[f] + c];
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
  PHASE(5);
  if (!solved) { fail_env(D, e, GRIP_R_SOLVE); return; }
  asm_converge(D, E, X, Etot, sm);
  PHASE(6);
#ifdef GRIP_PHASE_TIMING
  if (threadIdx.x == 0) {
    const int nce = D.n_act[e] + D.n_anc[e];
    const bool heavy = nce > 128;
    long long tot = 0;
    for (int k = 0; k < 7; ++k) {
      GSTAT(k, ph[k]);
      if (heavy) GSTAT(16 + k, ph[k]);
      tot += ph[k];
    }
    GSTAT(8, 1);
    GSTAT(9, nce);
    if (heavy) { GSTAT(24, 1); GSTAT(25, nce); }
    atomicMax(&g_phase[40], (unsigned long long)tot);
    atomicMax(&g_phase[41], (unsigned long long)nce);
    GSTAT(42, L.L == Lsm);
    GSTAT(43, S.nseg >= 2);
    GSTAT(44, shift != 0.0);
    if (S.nseg < 2) { GSTAT(45, ph[3]); GSTAT(46, 1); }
  }
#endif
}

}  // namespace grip
