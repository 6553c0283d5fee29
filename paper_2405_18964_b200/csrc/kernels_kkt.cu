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


// ------------------------------------------------------------------------------------------ 3-D
// Same time march in 3-D (Stokes).  A CTA owns a 16 x 8 x 8 box of Q2 nodes (+ the boundary layer past
// the last box in each direction, whose velocity outputs are zeros and whose Q1 nodes are unknowns).
// The pipeline unit is one (time block, component) sub-step: the component's v and lam boxes (+2 halo)
// are staged with cp.async while the previous sub-step is computed.  A thread owns one (x, y) column
// and 4 consecutive z outputs: per staged z-plane it forms the x-direction products on the 3 or 5 rows
// of its y (y parity is warp-uniform), the y-direction combinations, and scatters them into its 4 z
// outputs (sum factorisation of M = Mz (x) My (x) Mx, K = Kz My Mx + Mz Ky Mx + Mz My Kx).
// B^T p, B^T mu (all components) are formed at the component-0 sub-step from the staged Q1 boxes;
// B v, B lam accumulate over the three component sub-steps (one (Q1 node, field) item per thread).
constexpr int K3_TX = 16, K3_TY = 8, K3_TZ = 8;
constexpr int K3_SX = 22, K3_SY = 13, K3_SZ = 13;   // staged: x0-2..x0+19, y0-2..y0+10, z0-2..z0+10
constexpr int K3_PX = 12, K3_PY = 8, K3_PZ = 8;     // staged Q1: from (x0/2-1, y0/2-1, z0/2-1)
constexpr int K3_Q2 = K3_SX * K3_SY * K3_SZ, K3_Q1 = K3_PX * K3_PY * K3_PZ;
constexpr int K3_STAGE = 2 * K3_Q2 + 2 * K3_Q1;     // v_c, lam_c, p, mu

struct K3Args {
  const double* x;
  double* y;
  int n1, m1, n_b, ntx, nty, tiles;
  long nblk, n_s, n_v;
  double tau, tnu, tob;
};

__device__ __forceinline__ void k3_stage(const K3Args& a, double* st, int s, int c, bool wv, bool wl, bool wp,
                                         int x0, int y0, int z0, int tid) {
  const int n1 = a.n1, m1 = a.m1;
  for (int f = 0; f < 2; ++f) {
    if (!(f == 0 ? wv : wl)) continue;
    const double* src = a.x + ((long)f * a.n_b + s) * a.nblk + c * a.n_s;
    double* dst = st + f * K3_Q2;
    for (int e = tid; e < K3_Q2; e += 256) {
      const int li = e % K3_SX, r = e / K3_SX, lj = r % K3_SY, lk = r / K3_SY;
      const int gi = x0 - 2 + li, gj = y0 - 2 + lj, gk = z0 - 2 + lk;
      const bool ok = gi >= 1 && gi <= n1 - 2 && gj >= 1 && gj <= n1 - 2 && gk >= 1 && gk <= n1 - 2;
      cp_async8(dst + e, ok ? src + ((long)gk * n1 + gj) * n1 + gi : a.x, ok);
    }
  }
  if (!wp) return;
  for (int f = 0; f < 2; ++f) {
    const double* q = a.x + ((long)f * a.n_b + s) * a.nblk + a.n_v;
    double* dq = st + 2 * K3_Q2 + f * K3_Q1;
    for (int e = tid; e < K3_Q1; e += 256) {
      const int li = e % K3_PX, r = e / K3_PX, lj = r % K3_PY, lk = r / K3_PY;
      const int I = x0 / 2 - 1 + li, J = y0 / 2 - 1 + lj, K = z0 / 2 - 1 + lk;
      const bool ok = I >= 0 && I < m1 && J >= 0 && J < m1 && K >= 0 && K < m1 && (I | J | K) != 0;
      cp_async8(dq + e, ok ? q + ((long)K * m1 + J) * m1 + I : a.x, ok);
    }
  }
}

// M and K products of one staged field at the thread's 4 z outputs (PY: y parity of the thread's row)
template <int PY>
__device__ __forceinline__ void k3_mk(const KMRows& R, const double* U, int xl, int yl, int zq0, bool xodd,
                                      double* Mo, double* Ko) {
  constexpr int B0 = PY ? 1 : 0, B1 = PY ? 4 : 5;
  double mx[5], kx[5];
#pragma unroll
  for (int o = 0; o < 5; ++o) {
    mx[o] = xodd ? R.mm[o] : R.mv[o];
    kx[o] = xodd ? R.km[o] : R.kv[o];
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) Mo[r] = Ko[r] = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {   // planes z_out0 - 2 + q
    const double* P = U + (zq0 + q) * (K3_SX * K3_SY) + yl * K3_SX + xl;
    double pmm = 0.0, pkm = 0.0, pmk = 0.0;
#pragma unroll
    for (int ob = B0; ob < B1; ++ob) {
      const double* row = P + ob * K3_SX;
      double rm = 0.0, rk = 0.0;
#pragma unroll
      for (int oa = 0; oa < 5; ++oa) {
        const double u = row[oa];
        rm = fma(mx[oa], u, rm);
        rk = fma(kx[oa], u, rk);
      }
      const double my = PY ? R.mm[ob] : R.mv[ob], ky = PY ? R.km[ob] : R.kv[ob];
      pmm = fma(my, rm, pmm);
      pkm = fma(ky, rm, pkm);
      pmk = fma(my, rk, pmk);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {   // output z parity = parity of r (z0 and 4 zh even)
      const int o = q - r;
      const bool ok = (r & 1) ? (o >= 1 && o <= 3) : (o >= 0 && o <= 4);
      if (!ok) continue;
      const double mz = (r & 1) ? R.mm[o] : R.mv[o], kz = (r & 1) ? R.km[o] : R.kv[o];
      Mo[r] = fma(mz, pmm, Mo[r]);
      Ko[r] = fma(kz, pmm, fma(mz, pkm + pmk, Ko[r]));
    }
  }
}

// B^T q (all 3 components) at the thread's 4 z outputs from the staged Q1 box
template <int PY>
__device__ __forceinline__ void k3_bt(const KMRows& R, const double* Q, int x, int yq0, int zq0, bool xodd,
                                      double T[3][4]) {
  // Q1 cols for the thread's x: vertex x = 2e -> e-1..e+1, midpoint 2e+1 -> e..e+2; local = e - 1 - (x0/2 - 1)
  const int xq0 = (x >> 1) + (xodd ? 1 : 0);   // local Q1 col of tap 0 (x local, x0 even)
  double fpx[3], fgx[3];
#pragma unroll
  for (int o = 0; o < 3; ++o) {
    fpx[o] = xodd ? R.tpm[o] : R.tpv[o];
    fgx[o] = xodd ? R.tgm[o] : R.tgv[o];
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 4; ++r) T[c][r] = 0.0;
#pragma unroll
  for (int kq = 0; kq < 5; ++kq) {   // Q1 planes zq0 + kq
    double xy[3] = {0.0, 0.0, 0.0};  // comp 0: Gx Py, comp 1: Px Gy, comp 2: Px Py
#pragma unroll
    for (int jq = 0; jq < 3; ++jq) {
      const double* row = Q + (zq0 + kq) * (K3_PX * K3_PY) + (yq0 + jq) * K3_PX + xq0;
      double sp = 0.0, sg = 0.0;
#pragma unroll
      for (int o = 0; o < 3; ++o) {
        const double v = row[o];
        sp = fma(fpx[o], v, sp);
        sg = fma(fgx[o], v, sg);
      }
      const double py = PY ? R.tpm[jq] : R.tpv[jq], gy = PY ? R.tgm[jq] : R.tgv[jq];
      xy[0] = fma(py, sg, xy[0]);
      xy[1] = fma(gy, sp, xy[1]);
      xy[2] = fma(py, sp, xy[2]);
    }
    // z: output r uses Q1 planes base(r) + o, base = {0, 1, 1, 2}[r] relative to zq0 (as in 2-D)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int base = r == 0 ? 0 : (r == 3 ? 2 : 1);
      const int o = kq - base;
      if (o < 0 || o > 2) continue;
      const double pz = (r & 1) ? R.tpm[o] : R.tpv[o], gz = (r & 1) ? R.tgm[o] : R.tgv[o];
      T[0][r] = fma(pz, xy[0], T[0][r]);
      T[1][r] = fma(pz, xy[1], T[1][r]);
      T[2][r] = fma(gz, xy[2], T[2][r]);
    }
  }
}

__device__ __forceinline__ void k3_segment(const K3Args& a, const KMRows& R, double* sm, int tile, int t0, int t1) {
  const int tx = tile % a.ntx, ty = (tile / a.ntx) % a.nty, tz = tile / (a.ntx * a.nty);
  const int x0 = tx * K3_TX, y0 = ty * K3_TY, z0 = tz * K3_TZ;
  const int n1 = a.n1, m1 = a.m1, n_b = a.n_b;
  const bool xlast = x0 + K3_TX == n1 - 1, ylast = y0 + K3_TY == n1 - 1, zlast = z0 + K3_TZ == n1 - 1;
  const int tid = threadIdx.x, xl = tid & 15, zh = (tid >> 4) & 1, yl = tid >> 5;
  const int xg = x0 + xl, yg = y0 + yl, zg0 = z0 + 4 * zh;
  const bool xodd = xg & 1, yodd = yg & 1;
  const double tau = a.tau, tnu = a.tnu, tob = a.tob;
  const long nblk = a.nblk, ns = a.n_s;
  // owned Q1 box (+1 layer past the last tile) and this thread's (node, field) items
  const int nIx = K3_TX / 2 + (xlast ? 1 : 0), nIy = K3_TY / 2 + (ylast ? 1 : 0), nIz = K3_TZ / 2 + (zlast ? 1 : 0);
  const int nitems = 2 * nIx * nIy * nIz;
  double cMv[3][4], cA[3][4], Tp[3][4], Tm[3][4], Bacc[2];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 4; ++r) cMv[c][r] = cA[c][r] = Tp[c][r] = Tm[c][r] = 0.0;
  const int s_begin = t0 > 0 ? t0 - 1 : 0;
  const int s_end = t1 < n_b ? t1 : n_b - 1;
  const int nsub = 3 * (s_end - s_begin + 1);
  auto stage = [&](int k, double* buf) {
    const int s = s_begin + k / 3, c = k % 3;
    const bool pro = s < t0, epi = s >= t1;
    k3_stage(a, buf, s, c, !epi, !pro, !pro && !epi && c == 0, x0, y0, z0, tid);
  };
  stage(0, sm);
  cp_commit();
  for (int k = 0; k < nsub; ++k) {
    if (k + 1 < nsub) {
      stage(k + 1, sm + ((k + 1) & 1) * K3_STAGE);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const double* st = sm + (k & 1) * K3_STAGE;
    const int s = s_begin + k / 3, c = k % 3;
    const bool pro = s < t0, epi = s >= t1, main = !pro && !epi;
    double Mv[4], Kv[4], Ml[4], Kl[4];
    if (!epi) {
      if (yodd) k3_mk<1>(R, st, xl, yl, 4 * zh, xodd, Mv, Kv);
      else k3_mk<0>(R, st, xl, yl, 4 * zh, xodd, Mv, Kv);
    }
    if (!pro) {
      if (yodd) k3_mk<1>(R, st + K3_Q2, xl, yl, 4 * zh, xodd, Ml, Kl);
      else k3_mk<0>(R, st + K3_Q2, xl, yl, 4 * zh, xodd, Ml, Kl);
    }
    if (main && c == 0) {
      // Q1 rows/planes of the thread's y and z outputs: local base (y0 even) = yl/2 (+ parity shift)
      const double* sp = st + 2 * K3_Q2;
      const int yq0 = (yl >> 1) + (yodd ? 1 : 0), zq0 = 2 * zh;
      if (yodd) {
        k3_bt<1>(R, sp, xl, yq0, zq0, xodd, Tp);
        k3_bt<1>(R, sp + K3_Q1, xl, yq0, zq0, xodd, Tm);
      } else {
        k3_bt<0>(R, sp, xl, yq0, zq0, xodd, Tp);
        k3_bt<0>(R, sp + K3_Q1, xl, yq0, zq0, xodd, Tm);
      }
      Bacc[0] = Bacc[1] = 0.0;
    }
    const bool rin = xg >= 1 && xg <= n1 - 2 && yg >= 1 && yg <= n1 - 2;
    if (pro) {
#pragma unroll
      for (int r = 0; r < 4; ++r) cMv[0][r] = Mv[r];
    } else {
      // deferred y1v_{s-1} = A_{s-1} - M lam_s
      if (s > t0) {
        double* yo = a.y + (long)(s - 1) * nblk + c * ns;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int zg = zg0 + r;
          if (xg < n1 && yg < n1 && zg < n1) {
            const bool in = rin && zg >= 1 && zg <= n1 - 2;
            yo[((long)zg * n1 + yg) * n1 + xg] = in ? cA[0][r] - Ml[r] : 0.0;
          }
        }
      }
      if (main) {
        double* y2 = a.y + ((long)n_b + s) * nblk + c * ns;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int zg = zg0 + r;
          const double val = Mv[r] - cMv[0][r] - tob * Ml[r] + tnu * Kv[r] - tau * Tp[0][r];
          if (xg < n1 && yg < n1 && zg < n1) {
            const bool in = rin && zg >= 1 && zg <= n1 - 2;
            y2[((long)zg * n1 + yg) * n1 + xg] = in ? val : 0.0;
          }
          cMv[0][r] = Mv[r];
          cA[0][r] = tau * Mv[r] + Ml[r] + tnu * Kl[r] - tau * Tm[0][r];
        }
        // pressure rows: B_c v_c and B_c lam_c of the owned Q1 nodes (item = (node, field))
        const double* bx = c == 0 ? R.bg : R.bp;
        const double* by = c == 1 ? R.bg : R.bp;
        const double* bz = c == 2 ? R.bg : R.bp;
#pragma unroll
        for (int it = 0; it < 2; ++it) {
          const int item = tid + 256 * it;
          if (item >= nitems) continue;
          const int f = item & 1, nd = item >> 1;
          const int Il = nd % nIx, Jl = (nd / nIx) % nIy, Kl2 = nd / (nIx * nIy);
          const double* U = st + f * K3_Q2;
          // Q2 cols 2I-2..2I+2 -> local 2 Il (x0 even): box origin x0 - 2
          double acc = 0.0;
          for (int oc = 0; oc < 5; ++oc) {
            double pl = 0.0;
#pragma unroll
            for (int ob = 0; ob < 5; ++ob) {
              const double* row = U + (2 * Kl2 + oc) * (K3_SX * K3_SY) + (2 * Jl + ob) * K3_SX + 2 * Il;
              double rs = 0.0;
#pragma unroll
              for (int oa = 0; oa < 5; ++oa) rs = fma(bx[oa], row[oa], rs);
              pl = fma(by[ob], rs, pl);
            }
            acc = fma(bz[oc], pl, acc);
          }
          Bacc[it] += acc;
        }
        if (c == 2) {
#pragma unroll
          for (int it = 0; it < 2; ++it) {
            const int item = tid + 256 * it;
            if (item >= nitems) continue;
            const int f = item & 1, nd = item >> 1;
            const int I = x0 / 2 + nd % nIx, J = y0 / 2 + (nd / nIx) % nIy, K = z0 / 2 + nd / (nIx * nIy);
            if (I >= m1 || J >= m1 || K >= m1) continue;
            const long pn = ((long)K * m1 + J) * m1 + I;
            // field 1 (lam) -> y1p (half 0), field 0 (v) -> y2p (half 1)
            a.y[((long)(f == 1 ? 0 : n_b) + s) * nblk + a.n_v + pn] = pn == 0 ? 0.0 : -tau * Bacc[it];
          }
        }
        // zero velocity outputs on the boundary layer past the last box (all comps at c == 0)
        if (c == 0 && (xlast || ylast || zlast)) {
          const int ex = K3_TX + (xlast ? 1 : 0), ey = K3_TY + (ylast ? 1 : 0), ez = K3_TZ + (zlast ? 1 : 0);
          const int tot = ex * ey * ez;
          for (int e = tid; e < tot; e += 256) {
            const int li = e % ex, lj = (e / ex) % ey, lk = e / (ex * ey);
            if (li < K3_TX && lj < K3_TY && lk < K3_TZ) continue;
            const int gi = x0 + li, gj = y0 + lj, gk = z0 + lk;
            if (gi >= n1 || gj >= n1 || gk >= n1) continue;
            const long nd = ((long)gk * n1 + gj) * n1 + gi;
            for (int cc = 0; cc < 3; ++cc) {
              a.y[(long)s * nblk + cc * ns + nd] = 0.0;
              a.y[((long)n_b + s) * nblk + cc * ns + nd] = 0.0;
            }
          }
        }
      }
    }
    // the current component's carries live in slot 0: rotate so the next component's move there
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      double t;
      t = cMv[0][r]; cMv[0][r] = cMv[1][r]; cMv[1][r] = cMv[2][r]; cMv[2][r] = t;
      t = cA[0][r]; cA[0][r] = cA[1][r]; cA[1][r] = cA[2][r]; cA[2][r] = t;
      t = Tp[0][r]; Tp[0][r] = Tp[1][r]; Tp[1][r] = Tp[2][r]; Tp[2][r] = t;
      t = Tm[0][r]; Tm[0][r] = Tm[1][r]; Tm[1][r] = Tm[2][r]; Tm[2][r] = t;
    }
    __syncthreads();
  }
  if (t1 == n_b) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double* yo = a.y + (long)(n_b - 1) * nblk + c * ns;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int zg = zg0 + r;
        if (xg < n1 && yg < n1 && zg < n1) {
          const bool in = xg >= 1 && xg <= n1 - 2 && yg >= 1 && yg <= n1 - 2 && zg >= 1 && zg <= n1 - 2;
          yo[((long)zg * n1 + yg) * n1 + xg] = in ? cA[c][r] : 0.0;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(256, 1) k_kkt_march3(K3Args a, KMRows R) {
  extern __shared__ double k3s[];
  const long total = (long)a.tiles * a.n_b;
  const long per = (total + gridDim.x - 1) / gridDim.x;
  long gbeg = (long)blockIdx.x * per;
  const long gend = min(total, gbeg + per);
  while (gbeg < gend) {
    const int tile = (int)(gbeg / a.n_b), t0 = (int)(gbeg % a.n_b);
    const int t1 = (int)min((long)a.n_b, t0 + (gend - gbeg));
    k3_segment(a, R, k3s, tile, t0, t1);
    gbeg += t1 - t0;
    __syncthreads();
  }
}

}  // namespace

// true if the time-marching kernel handles this context (2-D); launched on stream s
bool launch_kkt_march(const Ctx& c, const double* x, double* y, cudaStream_t s) {
  if (c.n1q2 < 9) return false;   // generic rows need an interior vertex and midpoint (N_c >= 4)
  if (c.dim == 3 && c.oseen) return false;
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
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (c.dim == 3) {
    K3Args a;
    a.x = x;
    a.y = y;
    a.n1 = c.n1q2;
    a.m1 = c.n1q1;
    a.n_b = c.n_b;
    a.nblk = c.nblk;
    a.n_s = c.n_s;
    a.n_v = c.n_v;
    a.tau = c.tau;
    a.tnu = c.tau * c.nu;
    a.tob = c.tau / c.beta;
    a.ntx = (c.n1q2 - 1 + K3_TX - 1) / K3_TX;
    a.nty = (c.n1q2 - 1 + K3_TY - 1) / K3_TY;
    const int ntz = (c.n1q2 - 1 + K3_TZ - 1) / K3_TZ;
    a.tiles = a.ntx * a.nty * ntz;
    const long total = (long)a.tiles * c.n_b;
    const int grid = (int)std::max(1L, std::min((long)sms, (total + 3) / 4));
    const size_t smem = 2 * K3_STAGE * sizeof(double);
    static bool attr3 = false;
    if (!attr3) {
      cudaFuncSetAttribute(k_kkt_march3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr3 = true;
    }
    k_kkt_march3<<<grid, 256, smem, s>>>(a, R);
    return true;
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
