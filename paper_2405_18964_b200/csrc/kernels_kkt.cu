// Time-marching all-at-once KKT matvec y = A x (eq. (FinalA)), 2-D.
//
// Block rows of A (A2), for every time block s = 0..n_b-1 with v_{-1} := 0 and
// lam_{n_b} := 0 (backward Euler, E (x) M):
//   y1v_s = tau M v_s + M lam_s - M lam_{s+1} + tau L^T lam_s + tau B^T mu_s      (row half 0)
//   y2v_s = M v_s - M v_{s-1} - (tau/beta) M lam_s + tau L v_s + tau B^T p_s      (row half 1)
//   y1p_s = tau B lam_s,   y2p_s = tau B v_s
// with L = nu K (+ N for Oseen).  The operator applications M u, K u, B u, B^T q are computed ONCE per
// input slice and time step; the time coupling is a register carry (M v_{s-1}) and a deferred output
// (y1v_{s-1} = A_{s-1} - M lam_s).  A CTA owns a 64 x 32 tile of Q2 nodes (all components, both
// halves, and the Q1 pressure nodes under it) for a chunk of time blocks, and marches through time:
// every input slice is read from HBM once (plus a 2-node halo that neighbouring tiles fetch through L2
// at about the same time), every output is written once.  Slices are staged in shared memory with
// cp.async (zero-fill for masked / outside nodes = the elimination of S:85-86), double-buffered so the
// next time step streams in while the current one is computed.
//
// On a uniform mesh every interior 1-D row of the Q2 mass / stiffness / mixed matrices is one of two
// generic rows (vertex: even index, 5 taps; midpoint: odd index, 3 taps).  Rows next to the boundary
// differ only in the couplings to eliminated (boundary) columns, whose staged values are exact zeros,
// so the generic rows give the eliminated operator exactly; they are kernel parameters (constant bank).
// The x-direction 1-D products are formed per staged row and scattered into the y-direction sums
// (sum factorisation of the Kronecker forms).
#include <algorithm>
#include <cstdlib>

#include "aao_internal.h"

namespace aao {
namespace {

constexpr int KM_TX = 64, KM_TY = 32;          // owned Q2 tile
constexpr int KM_SX = KM_TX + 6, KM_SY = KM_TY + 5;   // staged Q2 tile: cols x0-2..x0+67, rows y0-2..y0+34
constexpr int KM_PX = 36, KM_PY = 20;          // staged Q1 tile: cols x0/2-1.., rows y0/2-1..
constexpr int KM_THREADS = 256;                // 32 column pairs x 8 row groups of 4 rows
constexpr int KM_Q2 = KM_SX * KM_SY, KM_Q1 = KM_PX * KM_PY;
constexpr int KM_STAGE = 4 * KM_Q2 + 2 * KM_Q1;  // doubles: v0, v1, lam0, lam1, p, mu

// generic 1-D rows (uniform mesh).  Q2-Q2: vertex taps -2..2, midpoint taps -1..1 (in [1..3]).
// B^T (Q2 node -> Q1 cols): vertex 2e -> e-1..e+1, midpoint 2e+1 -> e..e+2.  B (Q1 node I -> Q2 cols
// 2I-2..2I+2).  P = int psi phi, G = int psi phi' (B_c = -(G on axis c) (x) (P on the other axes)).
struct KMRows {
  double mv[5], kv[5], mm[5], km[5];
  double tpv[3], tgv[3], tpm[3], tgm[3];
  double bp[5], bg[5];
};

struct KMArgs {
  const double* x;
  double* y;
  const double* conv;    // Oseen: N  [n_s][25] (node-major, taps (ob, oa)); nullptr for Stokes
  const double* convT;   // Oseen: N^T
  int n1, m1, n_b, ntx, tiles;
  long nblk, n_s, n_v;
  double tau, tnu, tob;  // tau, tau nu, tau / beta
};

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// stage time block s: fields bit 0 = v (both comps) and p, bit 1 = lam and mu
__device__ __forceinline__ void km_stage(const KMArgs& a, double* st, int s, int fields, int x0, int y0, int tid) {
  const int n1 = a.n1, m1 = a.m1;
  for (int f = 0; f < 2; ++f) {
    if (!((fields >> f) & 1)) continue;
    const double* row = a.x + ((long)f * a.n_b + s) * a.nblk;   // half f: (v, p) or (lam, mu)
    for (int c = 0; c < 2; ++c) {
      const double* src = row + c * a.n_s;
      double* dst = st + (2 * f + c) * KM_Q2;
      for (int e = tid; e < KM_Q2; e += KM_THREADS) {
        const int lj = e / KM_SX, li = e - lj * KM_SX;
        const int gi = x0 - 2 + li, gj = y0 - 2 + lj;
        const bool ok = gi >= 1 && gi <= n1 - 2 && gj >= 1 && gj <= n1 - 2;
        cp_async8(dst + e, ok ? src + (long)gj * n1 + gi : a.x, ok);
      }
    }
    const double* q = row + a.n_v;
    double* dq = st + 4 * KM_Q2 + f * KM_Q1;
    for (int e = tid; e < KM_Q1; e += KM_THREADS) {
      const int lj = e / KM_PX, li = e - lj * KM_PX;
      const int I = x0 / 2 - 1 + li, J = y0 / 2 - 1 + lj;
      const bool ok = I >= 0 && I < m1 && J >= 0 && J < m1 && (I | J) != 0;   // node 0 pinned
      cp_async8(dq + e, ok ? q + (long)J * m1 + I : a.x, ok);
    }
  }
}

// y-direction scatter table: input row q (0..6, rows j0-2..j0+4) -> output row jj (j0+jj), tap index
// into the generic row (vertex rows: o = q - jj in 0..4; midpoint rows: o = q - jj in 1..3)
__device__ __forceinline__ constexpr bool ytap(int q, int jj) {
  return (jj & 1) ? (q - jj >= 1 && q - jj <= 3) : (q - jj >= 0 && q - jj <= 4);
}

// one segment: tile `tile`, output time blocks [t0, t1)
template <bool CONV>
__device__ __forceinline__ void km_segment(const KMArgs& a, const KMRows& R, double* kms, int tile, int t0, int t1) {
  const int tx = tile % a.ntx, ty = tile / a.ntx;
  const int x0 = tx * KM_TX, y0 = ty * KM_TY;
  const int n1 = a.n1, m1 = a.m1, n_b = a.n_b;
  const int tid = threadIdx.x, lane = tid & 31, g = tid >> 5;
  const int i0 = x0 + 2 * lane, j0 = y0 + 4 * g;      // velocity: cols i0, i0+1, rows j0..j0+3
  const int Ip = x0 / 2 + lane, Jp = y0 / 2 + 2 * g;  // pressure: col Ip, rows Jp, Jp+1
  const bool xlast = x0 + KM_TX == n1 - 1, ylast = y0 + KM_TY == n1 - 1;
  const double tau = a.tau, tnu = a.tnu, tob = a.tob;
  const long nblk = a.nblk;

  // carries: M v_{s-1} and A_{s-1} = tau M v + M lam + tau L^T lam + tau B^T mu, per [comp][row][col]
  double cMv[2][4][2], cA[2][4][2];
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < 2; ++k) cMv[c][r][k] = cA[c][r][k] = 0.0;

  const int s_begin = t0 > 0 ? t0 - 1 : 0;
  const int s_end = t1 < n_b ? t1 : n_b - 1;     // inclusive
  const int nsteps = s_end - s_begin + 1;
  auto fields_of = [&](int s) { return s < t0 ? 1 : (s >= t1 ? 2 : 3); };

  km_stage(a, kms, s_begin, fields_of(s_begin), x0, y0, tid);
  cp_commit();
  for (int k = 0; k < nsteps; ++k) {
    const int s = s_begin + k;
    if (k + 1 < nsteps) {
      km_stage(a, kms + ((k + 1) & 1) * KM_STAGE, s + 1, fields_of(s + 1), x0, y0, tid);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const double* st = kms + (k & 1) * KM_STAGE;
    const bool main = s >= t0 && s < t1;
    const bool pro = s < t0, epi = s >= t1;
    const double* sq = st + 4 * KM_Q2;   // p
    const double* smu = sq + KM_Q1;      // mu
    double Bv[2] = {0.0, 0.0}, Bl[2] = {0.0, 0.0};   // pressure rows: (B v)(Ip, Jp+jj), (B lam)(..)

#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double* sv = st + c * KM_Q2;
      const double* sl = st + (2 + c) * KM_Q2;
      double Mv[4][2], Kv[4][2], Ml[4][2], Kl[4][2];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) Mv[r][kk] = Kv[r][kk] = Ml[r][kk] = Kl[r][kk] = 0.0;
#pragma unroll
      for (int q = 0; q < 7; ++q) {
        const int off = (4 * g + q) * KM_SX + 2 * lane;
        const double2 va = *reinterpret_cast<const double2*>(sv + off);
        const double2 vb = *reinterpret_cast<const double2*>(sv + off + 2);
        const double vc = sv[off + 4];
        const double2 la = *reinterpret_cast<const double2*>(sl + off);
        const double2 lb = *reinterpret_cast<const double2*>(sl + off + 2);
        const double lc = sl[off + 4];
        const double V[5] = {va.x, va.y, vb.x, vb.y, vc};
        const double L[5] = {la.x, la.y, lb.x, lb.y, lc};
        // x-direction products: column i0 (vertex, taps 0..4), column i0+1 (midpoint, taps 1..3 -> V[1+o])
        double mxv[2] = {0, 0}, kxv[2] = {0, 0}, mxl[2] = {0, 0}, kxl[2] = {0, 0};
#pragma unroll
        for (int o = 0; o < 5; ++o) {
          mxv[0] = fma(R.mv[o], V[o], mxv[0]);
          kxv[0] = fma(R.kv[o], V[o], kxv[0]);
          if (o < 3) {
            mxv[1] = fma(R.mm[o + 1], V[o + 2], mxv[1]);
            kxv[1] = fma(R.km[o + 1], V[o + 2], kxv[1]);
          }
        }
        if (!pro) {
#pragma unroll
          for (int o = 0; o < 5; ++o) {
            mxl[0] = fma(R.mv[o], L[o], mxl[0]);
            kxl[0] = fma(R.kv[o], L[o], kxl[0]);
            if (o < 3) {
              mxl[1] = fma(R.mm[o + 1], L[o + 2], mxl[1]);
              kxl[1] = fma(R.km[o + 1], L[o + 2], kxl[1]);
            }
          }
        }
        // y-direction scatter into the 4 owned rows
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          if (!ytap(q, jj)) continue;
          const int o = q - jj;
          const double my = (jj & 1) ? R.mm[o] : R.mv[o];
          const double ky = (jj & 1) ? R.km[o] : R.kv[o];
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            Mv[jj][kk] = fma(my, mxv[kk], Mv[jj][kk]);
            Kv[jj][kk] = fma(ky, mxv[kk], fma(my, kxv[kk], Kv[jj][kk]));
            Ml[jj][kk] = fma(my, mxl[kk], Ml[jj][kk]);
            Kl[jj][kk] = fma(ky, mxl[kk], fma(my, kxl[kk], Kl[jj][kk]));
          }
        }
        // pressure rows: x-direction B_c products on the same staged values (cols 2Ip-2..2Ip+2)
        if (main) {
          const double* bx = c == 0 ? R.bg : R.bp;
          const double* by = c == 0 ? R.bp : R.bg;
          double bxv = 0.0, bxl = 0.0;
#pragma unroll
          for (int o = 0; o < 5; ++o) {
            bxv = fma(bx[o], V[o], bxv);
            bxl = fma(bx[o], L[o], bxl);
          }
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int o = q - 2 * jj;
            if (o < 0 || o > 4) continue;
            Bv[jj] = fma(by[o], bxv, Bv[jj]);
            Bl[jj] = fma(by[o], bxl, Bl[jj]);
          }
        }
      }
      if (pro) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) cMv[c][r][kk] = Mv[r][kk];
        continue;
      }
      // deferred output y1v_{s-1} = A_{s-1} - M lam_s (s > t0), or the epilogue
      if (s > t0) {
        double* yo = a.y + (long)(s - 1) * nblk + c * a.n_s;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int j = j0 + r;
          if (j >= n1) continue;
          const bool rin = j >= 1 && j <= n1 - 2;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int i = i0 + kk;
            if (i >= n1) continue;
            const bool in = rin && i >= 1 && i <= n1 - 2;
            yo[(long)j * n1 + i] = in ? cA[c][r][kk] - Ml[r][kk] : 0.0;
          }
        }
      }
      if (epi) continue;
      // B^T p and B^T mu for component c (Q1 tile, sum factorised): x then y
      double Tp[4][2], Tm[4][2];
#pragma unroll
      for (int r = 0; r < 4; ++r) Tp[r][0] = Tp[r][1] = Tm[r][0] = Tm[r][1] = 0.0;
      {
        const double* fxv = c == 0 ? R.tgv : R.tpv;   // axis x: G for comp 0, P otherwise
        const double* fxm = c == 0 ? R.tgm : R.tpm;
        const double* fyv = c == 1 ? R.tgv : R.tpv;   // axis y: G for comp 1
        const double* fym = c == 1 ? R.tgm : R.tpm;
#pragma unroll
        for (int qr = 0; qr < 5; ++qr) {   // Q1 rows (local 2g + qr)
          const int off = (2 * g + qr) * KM_PX + lane;   // Q1 cols lane..lane+3 (local)
          double P4[4], U4[4];
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            P4[o] = sq[off + o];
            U4[o] = smu[off + o];
          }
          double xp[2], xm[2];
          xp[0] = fma(fxv[0], P4[0], fma(fxv[1], P4[1], fxv[2] * P4[2]));
          xp[1] = fma(fxm[0], P4[1], fma(fxm[1], P4[2], fxm[2] * P4[3]));
          xm[0] = fma(fxv[0], U4[0], fma(fxv[1], U4[1], fxv[2] * U4[2]));
          xm[1] = fma(fxm[0], U4[1], fma(fxm[1], U4[2], fxm[2] * U4[3]));
          // output row j0+jj uses Q1 local rows base(jj) + o, base = 2g + {0,1,1,2}
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int base = jj == 0 ? 0 : (jj == 3 ? 2 : 1);
            const int o = qr - base;
            if (o < 0 || o > 2) continue;
            const double fy = (jj & 1) ? fym[o] : fyv[o];
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              Tp[jj][kk] = fma(fy, xp[kk], Tp[jj][kk]);
              Tm[jj][kk] = fma(fy, xm[kk], Tm[jj][kk]);
            }
          }
        }
      }
      double Nv[4][2], Nl[4][2];
#pragma unroll
      for (int r = 0; r < 4; ++r) Nv[r][0] = Nv[r][1] = Nl[r][0] = Nl[r][1] = 0.0;
      if constexpr (CONV) {
#pragma unroll 1
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int i = i0 + kk, j = j0 + r;
            if (i < 1 || i > n1 - 2 || j < 1 || j > n1 - 2) continue;
            const double* cn = a.conv + ((long)j * n1 + i) * 25;
            const double* ct = a.convT + ((long)j * n1 + i) * 25;
            double nv = 0.0, nl = 0.0;
#pragma unroll
            for (int ob = 0; ob < 5; ++ob)
#pragma unroll
              for (int oa = 0; oa < 5; ++oa) {
                const int so = (4 * g + r + ob) * KM_SX + 2 * lane + kk + oa;
                nv = fma(__ldg(cn + ob * 5 + oa), sv[so], nv);
                nl = fma(__ldg(ct + ob * 5 + oa), sl[so], nl);
              }
            Nv[r][kk] = nv;
            Nl[r][kk] = nl;
          }
      }
      // y2v_s = M v_s - M v_{s-1} - tau/beta M lam_s + tau (nu K + N) v_s + tau B^T p_s;  new carries
      double* y2 = a.y + ((long)n_b + s) * nblk + c * a.n_s;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int j = j0 + r;
        const bool rin = j >= 1 && j <= n1 - 2;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int i = i0 + kk;
          const bool in = rin && i >= 1 && i <= n1 - 2;
          const double val = Mv[r][kk] - cMv[c][r][kk] - tob * Ml[r][kk] + tnu * Kv[r][kk] + tau * Nv[r][kk] -
                             tau * Tp[r][kk];
          if (j < n1 && i < n1) y2[(long)j * n1 + i] = in ? val : 0.0;
          cMv[c][r][kk] = Mv[r][kk];
          cA[c][r][kk] = tau * Mv[r][kk] + Ml[r][kk] + tnu * Kl[r][kk] + tau * Nl[r][kk] - tau * Tm[r][kk];
        }
      }
    }
    if (main) {
      // pressure rows y1p_s = tau B lam_s, y2p_s = tau B v_s  (B = -(G (x) P) per component)
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const int J = Jp + jj;
        if (Ip < m1 && J < m1) {
          const long pn = (long)J * m1 + Ip;
          const bool pin = pn == 0;
          a.y[(long)s * nblk + a.n_v + pn] = pin ? 0.0 : -tau * Bl[jj];
          a.y[((long)n_b + s) * nblk + a.n_v + pn] = pin ? 0.0 : -tau * Bv[jj];
        }
      }
      // the last Q2 line / Q1 line of the grid when it lies just past the owned tile
      if (xlast || ylast) {
        // Q2 boundary line: zero outputs (both halves, both components)
        const int cnt = (xlast ? KM_TY : 0) + (ylast ? KM_TX : 0) + (xlast && ylast ? 1 : 0);
        for (int e = tid; e < 2 * cnt; e += KM_THREADS) {
          const int c = e / cnt, m = e % cnt;
          int i, j;
          if (xlast && m < KM_TY) {
            i = n1 - 1;
            j = y0 + m;
          } else {
            const int mm = m - (xlast ? KM_TY : 0);
            i = mm < KM_TX ? x0 + mm : n1 - 1;
            j = n1 - 1;
          }
          if (i >= n1 || j >= n1) continue;
          a.y[(long)s * nblk + c * a.n_s + (long)j * n1 + i] = 0.0;
          a.y[((long)n_b + s) * nblk + c * a.n_s + (long)j * n1 + i] = 0.0;
        }
        // Q1 line: full 5 x 5 products from the staged tile
        const int pc = (xlast ? KM_TY / 2 : 0) + (ylast ? KM_TX / 2 : 0) + (xlast && ylast ? 1 : 0);
        for (int e = tid; e < pc; e += KM_THREADS) {
          int I, J;
          if (xlast && e < KM_TY / 2) {
            I = m1 - 1;
            J = y0 / 2 + e;
          } else {
            const int mm = e - (xlast ? KM_TY / 2 : 0);
            I = mm < KM_TX / 2 ? x0 / 2 + mm : m1 - 1;
            J = m1 - 1;
          }
          if (I >= m1 || J >= m1) continue;
          double bv = 0.0, bl = 0.0;
          for (int c = 0; c < 2; ++c) {
            const double* sv = st + c * KM_Q2;
            const double* sl = st + (2 + c) * KM_Q2;
            const double* bx = c == 0 ? R.bg : R.bp;
            const double* by = c == 0 ? R.bp : R.bg;
            for (int ob = 0; ob < 5; ++ob)
              for (int oa = 0; oa < 5; ++oa) {
                const int so = (2 * J - y0 + ob) * KM_SX + (2 * I - x0 + oa);
                const double w = by[ob] * bx[oa];
                bv = fma(w, sv[so], bv);
                bl = fma(w, sl[so], bl);
              }
          }
          const long pn = (long)J * m1 + I;
          a.y[(long)s * nblk + a.n_v + pn] = -tau * bl;
          a.y[((long)n_b + s) * nblk + a.n_v + pn] = -tau * bv;
        }
      }
    }
    __syncthreads();
  }
  // last time block: y1v_{n_b-1} = A_{n_b-1} (lam_{n_b} = 0)
  if (t1 == n_b) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      double* yo = a.y + (long)(n_b - 1) * nblk + c * a.n_s;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int j = j0 + r;
        if (j >= n1) continue;
        const bool rin = j >= 1 && j <= n1 - 2;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int i = i0 + kk;
          if (i >= n1) continue;
          const bool in = rin && i >= 1 && i <= n1 - 2;
          yo[(long)j * n1 + i] = in ? cA[c][r][kk] : 0.0;
        }
      }
    }
  }
}

// Work is the linearised (tile, time block) space, split evenly over the grid (one CTA per SM slot):
// a CTA marches through at most a few contiguous segments, so there is no partial last wave.
template <bool CONV>
__global__ void __launch_bounds__(KM_THREADS, 1) k_kkt_march(KMArgs a, KMRows R) {
  extern __shared__ double kms[];
  const long total = (long)a.tiles * a.n_b;
  const long per = (total + gridDim.x - 1) / gridDim.x;
  long gbeg = (long)blockIdx.x * per;
  const long gend = min(total, gbeg + per);
  while (gbeg < gend) {
    const int tile = (int)(gbeg / a.n_b), t0 = (int)(gbeg % a.n_b);
    const int t1 = (int)min((long)a.n_b, t0 + (gend - gbeg));
    km_segment<CONV>(a, R, kms, tile, t0, t1);
    gbeg += t1 - t0;
    __syncthreads();
  }
}

}  // namespace

// true if the time-marching kernel handles this context (2-D); launched on stream s
bool launch_kkt_march(const Ctx& c, const double* x, double* y, cudaStream_t s) {
  if (c.dim != 2) return false;
  static const bool off = std::getenv("AAO_KKT_TILED") != nullptr;
  if (off) return false;
  if (c.n1q2 < 9) return false;   // generic rows need an interior vertex and midpoint (N_c >= 4)
  // Oseen: the per-node convection stencils (25 coefficients per node and time block, read through L2)
  // make the marching kernel slower than the tiled one (c3: 2.92 vs 2.07 ms) -- opt-in until restructured
  static const bool march_oseen = std::getenv("AAO_KKT_MARCH_OSEEN") != nullptr;
  if (c.oseen && !march_oseen) return false;
  // generic rows from the assembled 1-D tables at an interior vertex (even) and midpoint (odd) index
  KMRows R;
  const int iv = 2 * ((c.n1q2 - 1) / 4), im = iv + 1;
  for (int o = 0; o < 5; ++o) {
    R.mv[o] = c.h_M2[iv * 5 + o];
    R.kv[o] = c.h_K2[iv * 5 + o];
    R.mm[o] = c.h_M2[im * 5 + o];
    R.km[o] = c.h_K2[im * 5 + o];
  }
  for (int o = 0; o < 3; ++o) {
    R.tpv[o] = c.h_PmT[iv * 3 + o];
    R.tgv[o] = c.h_GmT[iv * 3 + o];
    R.tpm[o] = c.h_PmT[im * 3 + o];
    R.tgm[o] = c.h_GmT[im * 3 + o];
  }
  const int I = (c.n1q1 - 1) / 2;   // interior Q1 node
  for (int o = 0; o < 5; ++o) {
    R.bp[o] = c.h_Pm[I * 5 + o];
    R.bg[o] = c.h_Gm[I * 5 + o];
  }
  KMArgs a;
  a.x = x;
  a.y = y;
  a.conv = c.oseen ? c.vel.grids[0].conv : nullptr;
  a.convT = c.oseen ? c.vel.grids[0].convT : nullptr;
  a.n1 = c.n1q2;
  a.m1 = c.n1q1;
  a.n_b = c.n_b;
  a.nblk = c.nblk;
  a.n_s = c.n_s;
  a.n_v = c.n_v;
  a.tau = c.tau;
  a.tnu = c.tau * c.nu;
  a.tob = c.tau / c.beta;
  a.ntx = (c.n1q2 - 1 + KM_TX - 1) / KM_TX;
  const int nty = (c.n1q2 - 1 + KM_TY - 1) / KM_TY;
  const int tiles = a.ntx * nty;
  a.tiles = tiles;
  // one CTA per SM (shared memory bound); at least 4 time blocks per CTA
  const long total = (long)tiles * c.n_b;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = (int)std::max(1L, std::min((long)sms, (total + 3) / 4));
  const size_t smem = 2 * KM_STAGE * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_kkt_march<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_kkt_march<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (c.oseen)
    k_kkt_march<true><<<grid, KM_THREADS, smem, s>>>(a, R);
  else
    k_kkt_march<false><<<grid, KM_THREADS, smem, s>>>(a, R);
  return true;
}

}  // namespace aao
