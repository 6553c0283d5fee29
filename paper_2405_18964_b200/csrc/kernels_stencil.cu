// Batched-over-frequency stencil kernels for the per-frequency block solves
// (SURVEY 8(a) A4-A7): operator application, multicolour SOR, residual,
// restriction / prolongation, coarsest-level dense solve, Chebyshev steps,
// fused linear combinations.  sm_100a, fp64 / complex128.
//
// Every constant-coefficient operator is evaluated from 1-D assembled rows
// (Kronecker structure of Q2/Q1 on a uniform box mesh), so no matrix is
// stored except the convection N of the Oseen problem (per-node stencil).
// All problems of a batch share the real stencil; per-frequency complex scalars
// (alpha M + beta K + gamma N) come from a small coefficient table.
#include "aao_internal.h"

namespace aao {

#ifndef MG_THREADS
#define MG_THREADS 512
#endif
#ifndef MG_THREADS_TAB
#define MG_THREADS_TAB 512
#endif
// 2-D Q1 (pressure) solves: threads per CTA and CTAs per SM of the CTA-resident MG and Chebyshev kernels
#ifndef MG_THREADS_Q1
#define MG_THREADS_Q1 512
#endif
#ifndef MG_MINB_Q1
#define MG_MINB_Q1 1
#endif
// M_p Chebyshev of the 2-D Q1 space: pure streaming (five vectors per step), so several smaller CTAs per SM
#ifndef CHEB_THREADS_Q1
#define CHEB_THREADS_Q1 512
#endif
#ifndef CHEB_MINB_Q1
#define CHEB_MINB_Q1 2   // measured c4_512: pressure solves 27.1 (512 x 1) / 24.35 (512 x 2) / 25.8 ms (256 x 3, 256 x 4)
#endif
template <int DIM, int ORD>
constexpr int cheb_threads() {
  return DIM == 2 && ORD == 1 ? CHEB_THREADS_Q1 : MG_THREADS;
}
template <int DIM, int ORD>
constexpr int cheb_minb() {
  return DIM == 2 && ORD == 1 ? CHEB_MINB_Q1 : 1;
}

// ---------------------------------------------------------------- complex helpers
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cfma(double s, double2 a, double2 acc) {
  return make_double2(fma(s, a.x, acc.x), fma(s, a.y, acc.y));
}
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  double den = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / den, (a.y * b.x - a.x * b.y) / den);
}

__device__ __forceinline__ long voff(const View& v, int p, long n) {
  return (long)(p / v.per_group) * v.gstride + (long)(p % v.per_group) * n;
}

template <int DIM>
__device__ __forceinline__ void coords(long idx, int n1, int* c) {
  // per-problem node indices fit in 32 bits (n1^3 < 2^31 for every supported grid)
  const unsigned u = (unsigned)idx, un = (unsigned)n1;
  const unsigned q = u / un;
  c[0] = (int)(u - q * un);
  if (DIM == 2) {
    c[1] = (int)q;
  } else {
    const unsigned q2 = q / un;
    c[1] = (int)(q - q2 * un);
    c[2] = (int)q2;
  }
}

template <int DIM, int ORD>
__device__ __forceinline__ bool masked(const int* c, long idx, int n1) {
  if (ORD == 1) return idx == 0;  // pinned pressure node
  bool m = false;
#pragma unroll
  for (int a = 0; a < DIM; ++a) m |= (c[a] == 0) | (c[a] == n1 - 1);  // Dirichlet velocity
  return m;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Mx = (M x)_i, Kx = (K x)_i, Cx = (C x)_i at one node; dM, dK, dC = diagonal entries.
// Generic version (clamped taps): used for the Q1 pressure space.
template <int DIM, int ORD, bool CONV>
__device__ __forceinline__ void apply_MKC_generic(const Grid& g, const double* __restrict__ cv,
                                          const double2* x, const int* c, long idx,
                                          double2& Mx, double2& Kx, double2& Cx, double& dM, double& dK,
                                          double& dC) {
  constexpr int W = 2 * ORD + 1;
  double mx[W], kx[W];
#pragma unroll
  for (int o = 0; o < W; ++o) {
    mx[o] = __ldg(g.tM + c[0] * W + o);
    kx[o] = __ldg(g.tK + c[0] * W + o);
  }
  const int n1 = g.n1;
  Mx = Kx = Cx = make_double2(0.0, 0.0);
  const double* cvr = CONV ? cv + idx * (DIM == 2 ? W * W : W * W * W) : nullptr;
  const int nz = DIM == 3 ? W : 1;
  double mzc = 1.0, kzc = 0.0;  // z-row diagonal (3-D)
  double myc = 0.0, kyc = 0.0;  // y-row diagonal
#pragma unroll 1
  for (int oc = 0; oc < nz; ++oc) {
    double mz = 1.0, kz = 0.0;
    int zoff = 0;
    if (DIM == 3) {
      mz = __ldg(g.tM + c[2] * W + oc);
      kz = __ldg(g.tK + c[2] * W + oc);
      if (oc == ORD) {
        mzc = mz;
        kzc = kz;
      }
      zoff = clampi(c[2] + oc - ORD, 0, n1 - 1) * n1 * n1;
    }
#pragma unroll
    for (int ob = 0; ob < W; ++ob) {
      const double my = __ldg(g.tM + c[1] * W + ob);
      const double ky = __ldg(g.tK + c[1] * W + ob);
      if (ob == ORD) {
        myc = my;
        kyc = ky;
      }
      const double mzy = mz * my;
      const double kzy = kz * my + mz * ky;
      const int row = zoff + clampi(c[1] + ob - ORD, 0, n1 - 1) * n1;
#pragma unroll
      for (int oa = 0; oa < W; ++oa) {
        const double2 v = x[row + clampi(c[0] + oa - ORD, 0, n1 - 1)];
        Mx = cfma(mzy * mx[oa], v, Mx);
        Kx = cfma(kzy * mx[oa] + mzy * kx[oa], v, Kx);
        if (CONV) Cx = cfma(__ldg(cvr + (oc * W + ob) * W + oa), v, Cx);
      }
    }
  }
  dM = mzc * myc * mx[ORD];
  dK = kzc * myc * mx[ORD] + mzc * kyc * mx[ORD] + mzc * myc * kx[ORD];
  dC = CONV ? __ldg(cvr + (DIM == 3 ? (ORD * W + ORD) * W + ORD : ORD * W + ORD)) : 0.0;
}

// Q2 specialisation.  A Q2 node with an odd index along an axis is an element midpoint and
// couples only to offsets -1..1 along that axis; even (vertex) nodes couple to -2..2.  Taking the
// parity as a template argument gives 16 taps on average in 2-D (64 in 3-D) instead of 25 (125),
// and no tap of an interior node ever leaves the grid, so no clamping is needed.  The Kronecker
// coefficients are applied row by row (sum factorisation): per row rm = sum mx v, rk = sum kx v.
template <int DIM, bool CONV, int PY, int PZ>
__device__ __forceinline__ void q2_MKC(const Grid& g, const double* __restrict__ cv, const double2* x, const int* c,
                                       int idx, double2& Mx, double2& Kx, double2& Cx, double& dM, double& dK,
                                       double& dC) {
  constexpr int AY0 = PY ? 1 : 0, AY1 = PY ? 4 : 5;
  constexpr int AZ0 = DIM == 3 ? (PZ ? 1 : 0) : 2, AZ1 = DIM == 3 ? (PZ ? 4 : 5) : 3;
  const int n1 = g.n1;
  double mx[5], kx[5];
#pragma unroll
  for (int oa = 0; oa < 5; ++oa) {
    mx[oa] = __ldg(g.tM + c[0] * 5 + oa);   // zero outside the element support (odd nodes: oa = 0, 4)
    kx[oa] = __ldg(g.tK + c[0] * 5 + oa);
  }
  // the two outer x-taps may leave the grid next to the boundary (with zero coefficient): clamp them
  const int xl = c[0] >= 2 ? c[0] - 2 : c[0], xr = c[0] + 2 <= n1 - 1 ? c[0] + 2 : c[0];
  Mx = Kx = Cx = make_double2(0.0, 0.0);
  const double* cvr = CONV ? cv + (long)idx * (DIM == 2 ? 25 : 125) : nullptr;
  double mzc = 1.0, kzc = 0.0, myc = 0.0, kyc = 0.0;
#pragma unroll
  for (int oc = AZ0; oc < AZ1; ++oc) {
    double mz = 1.0, kz = 0.0;
    int zrow = 0;
    if (DIM == 3) {
      mz = __ldg(g.tM + c[2] * 5 + oc);
      kz = __ldg(g.tK + c[2] * 5 + oc);
      zrow = (c[2] + oc - 2) * n1;
      if (oc == 2) {
        mzc = mz;
        kzc = kz;
      }
    }
#pragma unroll
    for (int ob = AY0; ob < AY1; ++ob) {
      const double my = __ldg(g.tM + c[1] * 5 + ob);
      const double ky = __ldg(g.tK + c[1] * 5 + ob);
      if (ob == 2) {
        myc = my;
        kyc = ky;
      }
      const double2* row = x + (zrow + c[1] + ob - 2) * n1;
      double2 rm = make_double2(0.0, 0.0), rk = rm;
#pragma unroll
      for (int oa = 0; oa < 5; ++oa) {
        const int col = oa == 0 ? xl : (oa == 4 ? xr : c[0] + oa - 2);
        const double2 v = row[col];
        rm = cfma(mx[oa], v, rm);
        rk = cfma(kx[oa], v, rk);
        if (CONV) Cx = cfma(__ldg(cvr + ((DIM == 3 ? oc * 5 : 0) + ob) * 5 + oa), v, Cx);
      }
      const double mzy = mz * my, kzy = kz * my + mz * ky;
      Mx = cfma(mzy, rm, Mx);
      Kx = cfma(kzy, rm, cfma(mzy, rk, Kx));
    }
  }
  dM = mzc * myc * mx[2];
  dK = kzc * myc * mx[2] + mzc * kyc * mx[2] + mzc * myc * kx[2];
  dC = CONV ? __ldg(cvr + (DIM == 3 ? 62 : 12)) : 0.0;
}

template <int DIM, bool CONV>
__device__ __forceinline__ void q2_dispatch(const Grid& g, const double* __restrict__ cv, const double2* x,
                                            const int* c, int idx, double2& Mx, double2& Kx, double2& Cx, double& dM,
                                            double& dK, double& dC) {
  const int cls = (c[1] & 1) | (DIM == 3 ? ((c[2] & 1) << 1) : 0);
#define Q2C(b, cc) q2_MKC<DIM, CONV, b, cc>(g, cv, x, c, idx, Mx, Kx, Cx, dM, dK, dC)
  switch (cls) {
    case 0: Q2C(0, 0); break;
    case 1: Q2C(1, 0); break;
    case 2: if (DIM == 3) Q2C(0, 1); break;
    default: if (DIM == 3) Q2C(1, 1); break;
  }
#undef Q2C
}

template <int DIM, int ORD, bool CONV>
__device__ __forceinline__ void apply_MKC(const Grid& g, const double* __restrict__ cv, const double2* x,
                                          const int* c, long idx, double2& Mx, double2& Kx, double2& Cx, double& dM,
                                          double& dK, double& dC) {
  if constexpr (ORD == 2) {
    q2_dispatch<DIM, CONV>(g, cv, x, c, (int)idx, Mx, Kx, Cx, dM, dK, dC);
  } else {
    apply_MKC_generic<DIM, ORD, CONV>(g, cv, x, c, idx, Mx, Kx, Cx, dM, dK, dC);
  }
}

// (A x)_i and A_ii for A = a M + b K + c C
template <int DIM, int ORD>
__device__ __forceinline__ void apply_op(const Grid& g, const OpSel& op, int p, const double2* x,
                                         const int* c, long idx, double2& Ax, double2& D) {
  const Coef cf = op.coef[p / op.per_group];
  double2 Mx, Kx, Cx;
  double dM, dK, dC;
  if (op.conv_sel == 0) {
    apply_MKC<DIM, ORD, false>(g, nullptr, x, c, idx, Mx, Kx, Cx, dM, dK, dC);
  } else {
    apply_MKC<DIM, ORD, true>(g, op.conv_sel == 1 ? g.conv : g.convT, x, c, idx, Mx, Kx, Cx, dM, dK, dC);
  }
  Ax = cadd(cadd(cmul(cf.a, Mx), cmul(cf.b, Kx)), cmul(cf.c, Cx));
  D = cadd(cadd(cscale(dM, cf.a), cscale(dK, cf.b)), cscale(dC, cf.c));
}

// real-coefficient operator without convection (Stokes W_k, K_p): A = a M + b K, a, b real
template <int DIM, int ORD>
__device__ __forceinline__ void apply_op_real(const Grid& g, double ca, double cb, const double2* x, const int* c,
                                              long idx, double2& Ax, double& D) {
  double2 Mx, Kx, Cx;
  double dM, dK, dC;
  apply_MKC<DIM, ORD, false>(g, nullptr, x, c, idx, Mx, Kx, Cx, dM, dK, dC);
  Ax = make_double2(ca * Mx.x + cb * Kx.x, ca * Mx.y + cb * Kx.y);
  D = ca * dM + cb * dK;
}

// complex coefficients with convection (Oseen Q_k, Q_k^H): A = a M + b K + c C
template <int DIM, int ORD>
__device__ __forceinline__ void apply_op_conv(const Grid& g, const Coef& cf, const double* cv, const double2* x,
                                              const int* c, long idx, double2& Ax, double2& D) {
  double2 Mx, Kx, Cx;
  double dM, dK, dC;
  apply_MKC<DIM, ORD, true>(g, cv, x, c, idx, Mx, Kx, Cx, dM, dK, dC);
  Ax = cadd(cadd(cmul(cf.a, Mx), cmul(cf.b, Kx)), cmul(cf.c, Cx));
  D = cadd(cadd(cscale(dM, cf.a), cscale(dK, cf.b)), cscale(dC, cf.c));
}

// ---------------------------------------------------------------- multicolour SOR
// x_i <- x_i + omega (b_i - (A x)_i) / A_ii for the nodes of one colour (DESIGN.md reading:
// colour = sum_a (c_a mod C1) C1^a, C1 = 3 for Q2, 2 for Q1; no same-colour couplings).
template <int DIM, int ORD>
__global__ void k_gs(Grid g, OpSel op, View xv, View bv, int colour, double omega) {
  constexpr int C1 = ORD == 2 ? 3 : 2;
  const int p = blockIdx.y;
  int res[DIM], cnt[DIM];
  int cc = colour;
  long total = 1;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    res[a] = cc % C1;
    cc /= C1;
    cnt[a] = (g.n1 - res[a] + C1 - 1) / C1;
    total *= cnt[a];
  }
  long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total) return;
  int c[DIM];
  long idx = 0, stride = 1;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    c[a] = res[a] + C1 * (int)(t % cnt[a]);
    t /= cnt[a];
    idx += c[a] * stride;
    stride *= g.n1;
  }
  if (masked<DIM, ORD>(c, idx, g.n1)) return;
  double2* x = xv.p + voff(xv, p, g.n);
  const double2* b = bv.p + voff(bv, p, g.n);
  double2 Ax, D;
  apply_op<DIM, ORD>(g, op, p, x, c, idx, Ax, D);
  const double2 upd = cdiv(csub(b[idx], Ax), D);
  x[idx] = cadd(x[idx], cscale(omega, upd));
}

// r = b - A x  (masked entries -> 0)
template <int DIM, int ORD>
__global__ void k_residual(Grid g, OpSel op, View xv, View bv, View rv) {
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.n) return;
  int c[DIM];
  coords<DIM>(idx, g.n1, c);
  double2* r = rv.p + voff(rv, p, g.n);
  if (masked<DIM, ORD>(c, idx, g.n1)) {
    r[idx] = make_double2(0.0, 0.0);
    return;
  }
  const double2* x = xv.p + voff(xv, p, g.n);
  const double2* b = bv.p + voff(bv, p, g.n);
  double2 Ax, D;
  apply_op<DIM, ORD>(g, op, p, x, c, idx, Ax, D);
  r[idx] = csub(b[idx], Ax);
}

// ---------------------------------------------------------------- transfers
// restriction b_c = P^T r_f: coarse node I gathers fine nodes 2I-R..2I+R per axis (R = 3 Q2, 1 Q1)
template <int DIM, int ORD>
__global__ void k_restrict(Grid gf, Grid gc, Transfer t, View rv, View bv) {
  constexpr int R = ORD == 2 ? 3 : 1;
  constexpr int WR = 2 * R + 1;
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= gc.n) return;
  int c[DIM];
  coords<DIM>(idx, gc.n1, c);
  double2* b = bv.p + voff(bv, p, gc.n);
  if (masked<DIM, ORD>(c, idx, gc.n1)) {
    b[idx] = make_double2(0.0, 0.0);
    return;
  }
  const double2* r = rv.p + voff(rv, p, gf.n);
  const int o7 = ORD == 2 ? 0 : 2;  // Q1 rows use entries [2..4] of the 7-wide table
  double w[DIM][WR];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int o = 0; o < WR; ++o) w[a][o] = __ldg(t.tR + c[a] * 7 + o7 + o);
  double2 acc = make_double2(0.0, 0.0);
  const int n1 = gf.n1;
  if constexpr (DIM == 2) {
#pragma unroll
    for (int ob = 0; ob < WR; ++ob) {
      if (w[1][ob] == 0.0) continue;
      const int jj = 2 * c[1] + ob - R;
#pragma unroll
      for (int oa = 0; oa < WR; ++oa) {
        if (w[0][oa] == 0.0) continue;
        const int ii = 2 * c[0] + oa - R;
        acc = cfma(w[1][ob] * w[0][oa], r[(long)jj * n1 + ii], acc);
      }
    }
  } else {
    for (int oc = 0; oc < WR; ++oc) {
      if (w[2][oc] == 0.0) continue;
      const int kk = 2 * c[2] + oc - R;
      for (int ob = 0; ob < WR; ++ob) {
        if (w[1][ob] == 0.0) continue;
        const int jj = 2 * c[1] + ob - R;
#pragma unroll
        for (int oa = 0; oa < WR; ++oa) {
          if (w[0][oa] == 0.0) continue;
          const int ii = 2 * c[0] + oa - R;
          acc = cfma(w[2][oc] * w[1][ob] * w[0][oa], r[((long)kk * n1 + jj) * n1 + ii], acc);
        }
      }
    }
  }
  b[idx] = acc;
}

// prolongation + correction x_f += P x_c (nodal interpolation; masked fine nodes untouched)
template <int DIM, int ORD>
__global__ void k_prolong(Grid gf, Grid gc, Transfer t, View xcv, View xfv) {
  constexpr int NW = ORD == 2 ? 3 : 2;
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= gf.n) return;
  int c[DIM];
  coords<DIM>(idx, gf.n1, c);
  if (masked<DIM, ORD>(c, idx, gf.n1)) return;
  const double2* xc = xcv.p + voff(xcv, p, gc.n);
  double2* xf = xfv.p + voff(xfv, p, gf.n);
  int base[DIM];
  double w[DIM][NW];
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    base[a] = (int)__ldg(t.tP + c[a] * 4);
#pragma unroll
    for (int o = 0; o < NW; ++o) w[a][o] = __ldg(t.tP + c[a] * 4 + 1 + o);
  }
  const int n1 = gc.n1;
  double2 acc = make_double2(0.0, 0.0);
  if constexpr (DIM == 2) {
#pragma unroll
    for (int ob = 0; ob < NW; ++ob) {
      if (w[1][ob] == 0.0) continue;
#pragma unroll
      for (int oa = 0; oa < NW; ++oa) {
        if (w[0][oa] == 0.0) continue;
        acc = cfma(w[1][ob] * w[0][oa], xc[(long)(base[1] + ob) * n1 + base[0] + oa], acc);
      }
    }
  } else {
#pragma unroll
    for (int oc = 0; oc < NW; ++oc) {
      if (w[2][oc] == 0.0) continue;
#pragma unroll
      for (int ob = 0; ob < NW; ++ob) {
        if (w[1][ob] == 0.0) continue;
#pragma unroll
        for (int oa = 0; oa < NW; ++oa) {
          if (w[0][oa] == 0.0) continue;
          acc = cfma(w[2][oc] * w[1][ob] * w[0][oa],
                     xc[((long)(base[2] + oc) * n1 + base[1] + ob) * n1 + base[0] + oa], acc);
        }
      }
    }
  }
  xf[idx] = cadd(xf[idx], acc);
}

// coarsest level: x[unk] = inv_g * b[unk] (dense inverse per coefficient group)
__global__ void k_coarse(long nc, const double2* __restrict__ inv, int inv_per_group, const int* __restrict__ unk,
                         int nu, View bv, View xv) {
  const int p = blockIdx.x;
  const double2* b = bv.p + voff(bv, p, nc);
  double2* x = xv.p + voff(xv, p, nc);
  const double2* A = inv + (long)(p / inv_per_group) * nu * nu;
  extern __shared__ double2 sb[];
  for (int i = threadIdx.x; i < nu; i += blockDim.x) sb[i] = b[unk[i]];
  __syncthreads();
  for (int i = threadIdx.x; i < nu; i += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < nu; ++j) acc = cadd(acc, cmul(A[(long)i * nu + j], sb[j]));
    x[unk[i]] = acc;
  }
}

__global__ void k_zero(View xv, long n) {
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  xv.p[voff(xv, p, n) + idx] = make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------- Chebyshev on a mass matrix
// x0 = 0, r0 = f, d0 = D^-1 r0 / theta; per step x += d; r -= M d; d' = c1 d + c2 D^-1 r.
template <int DIM, int ORD>
__device__ __forceinline__ double mass_diag(const Grid& g, const int* c) {
  constexpr int W = 2 * ORD + 1;
  double d = 1.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) d *= __ldg(g.tM + c[a] * W + ORD);
  return d;
}

template <int DIM, int ORD>
__global__ void k_cheb_init(Grid g, View bv, View xv, View rv, View dv, double inv_theta) {
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.n) return;
  int c[DIM];
  coords<DIM>(idx, g.n1, c);
  const long o = voff(bv, p, g.n) + idx;
  double2 bb = bv.p[o];
  double2 z = make_double2(0.0, 0.0);
  double2 dd = z;
  if (masked<DIM, ORD>(c, idx, g.n1)) {
    bb = z;
  } else {
    dd = cscale(1.0 / mass_diag<DIM, ORD>(g, c), bb);
    dd = cscale(inv_theta, dd);
  }
  xv.p[voff(xv, p, g.n) + idx] = z;
  rv.p[voff(rv, p, g.n) + idx] = bb;
  dv.p[voff(dv, p, g.n) + idx] = dd;
}

template <int DIM, int ORD>
__global__ void k_cheb_step(Grid g, View xv, View rv, View dov, View dnv, double c1, double c2) {
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.n) return;
  int c[DIM];
  coords<DIM>(idx, g.n1, c);
  const long oo = voff(dnv, p, g.n) + idx;
  if (masked<DIM, ORD>(c, idx, g.n1)) {
    dnv.p[oo] = make_double2(0.0, 0.0);
    return;
  }
  const double2* dold = dov.p + voff(dov, p, g.n);
  double2 Mx, Kx, Cx;
  double dM, dK, dC;
  apply_MKC<DIM, ORD, false>(g, nullptr, dold, c, idx, Mx, Kx, Cx, dM, dK, dC);
  const long ox = voff(xv, p, g.n) + idx, orr = voff(rv, p, g.n) + idx;
  const double2 d = dold[idx];
  xv.p[ox] = cadd(xv.p[ox], d);
  const double2 r = csub(rv.p[orr], Mx);
  rv.p[orr] = r;
  dnv.p[oo] = cadd(cscale(c1, d), cscale(c2, cscale(1.0 / dM, r)));
}

template <int DIM, int ORD>
__global__ void k_cheb_final(Grid g, View xv, View dv, double scale) {
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.n) return;
  const long ox = voff(xv, p, g.n) + idx;
  xv.p[ox] = cscale(scale, cadd(xv.p[ox], dv.p[voff(dv, p, g.n) + idx]));
}

// ---------------------------------------------------------------- fused linear combinations
template <int DIM, int ORD>
__global__ void k_lincomb(Grid g, View ov, double cb, View bv, OpSel A1, View x1, OpSel A2, View x2, int two) {
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.n) return;
  int c[DIM];
  coords<DIM>(idx, g.n1, c);
  double2* out = ov.p + voff(ov, p, g.n);
  if (masked<DIM, ORD>(c, idx, g.n1)) {
    out[idx] = make_double2(0.0, 0.0);
    return;
  }
  double2 acc = make_double2(0.0, 0.0);
  if (cb != 0.0) acc = cscale(cb, bv.p[voff(bv, p, g.n) + idx]);
  double2 Ax, D;
  apply_op<DIM, ORD>(g, A1, p, x1.p + voff(x1, p, g.n), c, idx, Ax, D);
  acc = cadd(acc, Ax);
  if (two) {
    apply_op<DIM, ORD>(g, A2, p, x2.p + voff(x2, p, g.n), c, idx, Ax, D);
    acc = cadd(acc, Ax);
  }
  out[idx] = acc;
}

template <int DIM, int ORD>
__global__ void k_axpby(Grid g, View yv, double2 a, View xv, double2 bc) {
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.n) return;
  const long oy = voff(yv, p, g.n) + idx;
  yv.p[oy] = cadd(cmul(a, yv.p[oy]), cmul(bc, xv.p[voff(xv, p, g.n) + idx]));
}

// pressure out_q = sb * bp_q + sB * sum_c (B_c v_c)_q, B = -[int psi d_c phi]
// tPm/tGm: [n1q1][5] 1-D rows int psi_I phi_j, int psi_I phi_j' for j = 2I-2..2I+2 (Dirichlet cols 0)
// v view: problem p (pressure problem) -> velocity components at p*DIMgroups (see launcher)
template <int DIM>
__global__ void k_Bv(Grid g2, Grid g1, const double* __restrict__ tPm, const double* __restrict__ tGm, View vv,
                     View bpv, View ov, double sb, double sB) {
  const int p = blockIdx.y;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g1.n) return;
  int c[DIM];
  coords<DIM>(idx, g1.n1, c);
  double2* out = ov.p + voff(ov, p, g1.n);
  if (idx == 0) {
    out[0] = make_double2(0.0, 0.0);
    return;
  }
  double Pm[DIM][5], Gm[DIM][5];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int o = 0; o < 5; ++o) {
      Pm[a][o] = __ldg(tPm + c[a] * 5 + o);
      Gm[a][o] = __ldg(tGm + c[a] * 5 + o);
    }
  double2 acc = make_double2(0.0, 0.0);
  const int n1 = g2.n1;
  for (int comp = 0; comp < DIM; ++comp) {
    const double2* v = vv.p + voff(vv, p * DIM + comp, g2.n);
    if constexpr (DIM == 2) {
#pragma unroll
      for (int ob = 0; ob < 5; ++ob) {
        const int jj = clampi(2 * c[1] + ob - 2, 0, n1 - 1);
        const double fy = comp == 1 ? Gm[1][ob] : Pm[1][ob];
#pragma unroll
        for (int oa = 0; oa < 5; ++oa) {
          const int ii = clampi(2 * c[0] + oa - 2, 0, n1 - 1);
          const double fx = comp == 0 ? Gm[0][oa] : Pm[0][oa];
          acc = cfma(-fy * fx, v[(long)jj * n1 + ii], acc);
        }
      }
    } else {
      for (int oc = 0; oc < 5; ++oc) {
        const int kk = clampi(2 * c[2] + oc - 2, 0, n1 - 1);
        const double fz = comp == 2 ? Gm[2][oc] : Pm[2][oc];
#pragma unroll
        for (int ob = 0; ob < 5; ++ob) {
          const int jj = clampi(2 * c[1] + ob - 2, 0, n1 - 1);
          const double fy = comp == 1 ? Gm[1][ob] : Pm[1][ob];
#pragma unroll
          for (int oa = 0; oa < 5; ++oa) {
            const int ii = clampi(2 * c[0] + oa - 2, 0, n1 - 1);
            const double fx = comp == 0 ? Gm[0][oa] : Pm[0][oa];
            acc = cfma(-fz * fy * fx, v[((long)kk * n1 + jj) * n1 + ii], acc);
          }
        }
      }
    }
  }
  double2 res = cscale(sB, acc);
  if (sb != 0.0) res = cadd(res, cscale(sb, bpv.p[voff(bpv, p, g1.n) + idx]));
  out[idx] = res;
}

// ---------------------------------------------------------------- class stencils (Q2, real operators)
// Masked nodes of an iterate are exact zeros, so every interior Q2 node can use the UN-eliminated
// interior 1-D rows: a vertex row (even index) or a midpoint row (odd index) per axis.  A level of
// a real operator A = a M + b K therefore has only 2^d distinct stencils, precomputed per CTA (per
// frequency) in shared memory together with 1/A_ii: one coefficient lookup and two FMAs per tap.
template <int DIM>
struct ClassTab {
  static constexpr int NT = DIM == 2 ? 25 : 125;   // taps
  static constexpr int NCL = 1 << DIM;             // classes (parity per axis, x fastest)
  static constexpr int PER_LEVEL = NCL * (NT + 1); // + 1/diag per class
};

// build the class stencils of level g for A = ca M + cb K into tab (ClassTab::PER_LEVEL doubles)
template <int DIM>
__device__ void build_class_tab(const Grid& g, double ca, double cb, double* tab, int tid, int nth) {
  using CT = ClassTab<DIM>;
  // un-eliminated interior rows: index 4 (vertex) and 3 (midpoint); needs n1 >= 9
  for (int e = tid; e < CT::NCL * CT::NT; e += nth) {
    const int cls = e / CT::NT, tap = e % CT::NT;
    const int oa = tap % 5, ob = (tap / 5) % 5, oc = tap / 25;
    const int rx = (cls & 1) ? 3 : 4, ry = ((cls >> 1) & 1) ? 3 : 4, rz = ((cls >> 2) & 1) ? 3 : 4;
    const double mx = g.tM[rx * 5 + oa], kx = g.tK[rx * 5 + oa];
    const double my = g.tM[ry * 5 + ob], ky = g.tK[ry * 5 + ob];
    double mz = 1.0, kz = 0.0;
    if (DIM == 3) {
      mz = g.tM[rz * 5 + oc];
      kz = g.tK[rz * 5 + oc];
    }
    const double m = mz * my * mx;
    const double k = kz * my * mx + mz * ky * mx + mz * my * kx;
    tab[cls * (CT::NT + 1) + tap] = ca * m + cb * k;
  }
  __syncthreads();
  for (int cls = tid; cls < CT::NCL; cls += nth) {
    const int centre = DIM == 2 ? 12 : 62;
    tab[cls * (CT::NT + 1) + CT::NT] = 1.0 / tab[cls * (CT::NT + 1) + centre];
  }
}

// complex coefficients (Oseen Q_k = a M + b K + c N): class table of a M + b K (double2 per tap);
// the convection part is per node (stored stencil), accumulated separately and scaled by c.
template <int DIM>
__device__ void build_class_tab_c(const Grid& g, double2 ca, double2 cb, double2* tab, int tid, int nth) {
  using CT = ClassTab<DIM>;
  for (int e = tid; e < CT::NCL * CT::NT; e += nth) {
    const int cls = e / CT::NT, tap = e % CT::NT;
    const int oa = tap % 5, ob = (tap / 5) % 5, oc = tap / 25;
    const int rx = (cls & 1) ? 3 : 4, ry = ((cls >> 1) & 1) ? 3 : 4, rz = ((cls >> 2) & 1) ? 3 : 4;
    const double mx = g.tM[rx * 5 + oa], kx = g.tK[rx * 5 + oa];
    const double my = g.tM[ry * 5 + ob], ky = g.tK[ry * 5 + ob];
    double mz = 1.0, kz = 0.0;
    if (DIM == 3) {
      mz = g.tM[rz * 5 + oc];
      kz = g.tK[rz * 5 + oc];
    }
    const double m = mz * my * mx;
    const double k = kz * my * mx + mz * ky * mx + mz * my * kx;
    tab[cls * CT::NT + tap] = cadd(cscale(m, ca), cscale(k, cb));
  }
}

template <int DIM, int PY, int PZ>
__device__ __forceinline__ void class_eval_conv_rows(const double2* T, const double* cvr, const double2* x,
                                                     const int* c, int n1, double2& acc, double2& nacc) {
  constexpr int AY0 = PY ? 1 : 0, AY1 = PY ? 4 : 5;
  constexpr int AZ0 = DIM == 3 ? (PZ ? 1 : 0) : 2, AZ1 = DIM == 3 ? (PZ ? 4 : 5) : 3;
  const int xl = c[0] >= 2 ? c[0] - 2 : c[0], xr = c[0] + 2 <= n1 - 1 ? c[0] + 2 : c[0];
#pragma unroll
  for (int oc = AZ0; oc < AZ1; ++oc) {
    const int zrow = DIM == 3 ? (c[2] + oc - 2) * n1 : 0;
#pragma unroll
    for (int ob = AY0; ob < AY1; ++ob) {
      const double2* row = x + (zrow + c[1] + ob - 2) * n1;
      const int t0 = ((DIM == 3 ? oc * 5 : 0) + ob) * 5;
#pragma unroll
      for (int oa = 0; oa < 5; ++oa) {
        const double2 v = row[oa == 0 ? xl : (oa == 4 ? xr : c[0] + oa - 2)];
        acc = cadd(acc, cmul(T[t0 + oa], v));
        nacc = cfma(__ldg(cvr + t0 + oa), v, nacc);
      }
    }
  }
}

template <int DIM>
__device__ __forceinline__ double2 class_eval_conv(const double2* tabl, const double* cv, double2 cc,
                                                   const double2* x, const int* c, int idx, int n1, double2& D) {
  using CT = ClassTab<DIM>;
  const int cls = (c[0] & 1) | ((c[1] & 1) << 1) | (DIM == 3 ? ((c[2] & 1) << 2) : 0);
  const double2* T = tabl + cls * CT::NT;
  const double* cvr = cv + (long)idx * CT::NT;
  double2 acc = make_double2(0.0, 0.0), nacc = acc;
  const int ycls = (c[1] & 1) | (DIM == 3 ? ((c[2] & 1) << 1) : 0);
  switch (ycls) {
    case 0: class_eval_conv_rows<DIM, 0, 0>(T, cvr, x, c, n1, acc, nacc); break;
    case 1: class_eval_conv_rows<DIM, 1, 0>(T, cvr, x, c, n1, acc, nacc); break;
    case 2: class_eval_conv_rows<DIM, 0, 1>(T, cvr, x, c, n1, acc, nacc); break;
    default: class_eval_conv_rows<DIM, 1, 1>(T, cvr, x, c, n1, acc, nacc); break;
  }
  const int centre = DIM == 2 ? 12 : 62;
  D = cadd(T[centre], cscale(__ldg(cvr + centre), cc));
  return cadd(acc, cmul(cc, nacc));
}

// (A x)_i with the class stencil; returns 1/A_ii in invD.  Rows with zero taps for odd y/z are skipped.
template <int DIM, int PY, int PZ>
__device__ __forceinline__ double2 class_eval_rows(const double* T, const double2* x, const int* c, int n1) {
  constexpr int AY0 = PY ? 1 : 0, AY1 = PY ? 4 : 5;
  constexpr int AZ0 = DIM == 3 ? (PZ ? 1 : 0) : 2, AZ1 = DIM == 3 ? (PZ ? 4 : 5) : 3;
  const int xl = c[0] >= 2 ? c[0] - 2 : c[0], xr = c[0] + 2 <= n1 - 1 ? c[0] + 2 : c[0];
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int oc = AZ0; oc < AZ1; ++oc) {
    const int zrow = DIM == 3 ? (c[2] + oc - 2) * n1 : 0;
#pragma unroll
    for (int ob = AY0; ob < AY1; ++ob) {
      const double2* row = x + (zrow + c[1] + ob - 2) * n1;
      const double* t = T + ((DIM == 3 ? oc * 5 : 0) + ob) * 5;
      acc = cfma(t[0], row[xl], acc);
      acc = cfma(t[1], row[c[0] - 1], acc);
      acc = cfma(t[2], row[c[0]], acc);
      acc = cfma(t[3], row[c[0] + 1], acc);
      acc = cfma(t[4], row[xr], acc);
    }
  }
  return acc;
}

template <int DIM>
__device__ __forceinline__ double2 class_eval(const double* tabl, const double2* x, const int* c, int n1,
                                              double& invD) {
  using CT = ClassTab<DIM>;
  const int cls = (c[0] & 1) | ((c[1] & 1) << 1) | (DIM == 3 ? ((c[2] & 1) << 2) : 0);
  const double* T = tabl + cls * (CT::NT + 1);
  invD = T[CT::NT];
  const int ycls = (c[1] & 1) | (DIM == 3 ? ((c[2] & 1) << 1) : 0);
  switch (ycls) {
    case 0: return class_eval_rows<DIM, 0, 0>(T, x, c, n1);
    case 1: return class_eval_rows<DIM, 1, 0>(T, x, c, n1);
    case 2: return class_eval_rows<DIM, 0, 1>(T, x, c, n1);
    default: return class_eval_rows<DIM, 1, 1>(T, x, c, n1);
  }
}

// Branch-free 2-D class-stencil evaluation (all 25 taps; rows and columns clamped into the grid where the
// class coefficient is zero) with one accumulator per stencil row: for the small, latency-bound levels,
// where one node per thread and one colour per barrier phase leave nothing to overlap, a single
// warp-convergent pass with short dependency chains beats the parity-split visits.
__device__ __forceinline__ double2 class_eval_flat2(const double* tabl, const double2* x, int i, int j, int n1,
                                                    double& invD) {
  const int cls = (i & 1) | ((j & 1) << 1);
  const double* T = tabl + cls * (ClassTab<2>::NT + 1);
  invD = T[ClassTab<2>::NT];
  const int xl = i >= 2 ? i - 2 : i, xr = i + 2 <= n1 - 1 ? i + 2 : i;
  double2 acc[5];
#pragma unroll
  for (int ob = 0; ob < 5; ++ob) {
    int r = j + ob - 2;
    r = r < 0 ? 0 : (r > n1 - 1 ? n1 - 1 : r);
    const double2* row = x + r * n1;
    const double* t = T + ob * 5;
    double2 a = make_double2(t[0] * row[xl].x, t[0] * row[xl].y);
    a = cfma(t[1], row[i - 1], a);
    a = cfma(t[2], row[i], a);
    a = cfma(t[3], row[i + 1], a);
    acc[ob] = cfma(t[4], row[xr], a);
  }
  return cadd(cadd(cadd(acc[0], acc[1]), cadd(acc[2], acc[3])), acc[4]);
}

// Branch-free 2-D evaluation with complex class coefficients and the per-node convection stencil
// (Oseen Q_k, Q_k^H: A = a M + b K + c N), for the small levels (as class_eval_flat2).
__device__ __forceinline__ double2 class_eval_conv_flat2(const double2* tabl, const double* cv, double2 cc,
                                                         const double2* x, int i, int j, int idx, int n1,
                                                         double2& D) {
  const int cls = (i & 1) | ((j & 1) << 1);
  const double2* T = tabl + cls * ClassTab<2>::NT;
  const double* cvr = cv + (long)idx * ClassTab<2>::NT;
  const int xl = i >= 2 ? i - 2 : i, xr = i + 2 <= n1 - 1 ? i + 2 : i;
  double2 acc[5], nac[5];
#pragma unroll
  for (int ob = 0; ob < 5; ++ob) {
    int r = j + ob - 2;
    r = r < 0 ? 0 : (r > n1 - 1 ? n1 - 1 : r);
    const double2* row = x + r * n1;
    const double2 v[5] = {row[xl], row[i - 1], row[i], row[i + 1], row[xr]};
    double2 a = cmul(T[ob * 5], v[0]);
    double2 nn = cscale(__ldg(cvr + ob * 5), v[0]);
#pragma unroll
    for (int oa = 1; oa < 5; ++oa) {
      a = cadd(a, cmul(T[ob * 5 + oa], v[oa]));
      nn = cfma(__ldg(cvr + ob * 5 + oa), v[oa], nn);
    }
    acc[ob] = a;
    nac[ob] = nn;
  }
  D = cadd(T[12], cscale(__ldg(cvr + 12), cc));
  const double2 A = cadd(cadd(cadd(acc[0], acc[1]), cadd(acc[2], acc[3])), acc[4]);
  const double2 N = cadd(cadd(cadd(nac[0], nac[1]), cadd(nac[2], nac[3])), nac[4]);
  return cadd(A, cmul(cc, N));
}

// ---------------------------------------------------------------- class stencils (2-D Q1, real operators)
// The Q1 pressure operators (Neumann K_p, M_p; every node an unknown except the pinned corner, whose iterate is an
// exact zero) have one stencil per position class: first / interior / last node along each axis, 3 x 3 classes of
// 9 taps + 1 / A_ii.  Taps that would leave the grid have zero coefficients and are read at a clamped index.  One
// table per level in shared memory replaces the per-node 1-D row loads and the separate M and K sums of
// apply_MKC_generic (the pressure MG was bound by the L1 data path: 12 table loads per node, lanes diverging).
constexpr int Q1TAB = 90;   // doubles per level: 9 classes x (9 taps + 1 / diagonal)

__device__ void build_class_tab_q1(const Grid& g, double ca, double cb, double* tab, int tid, int nth) {
  const int n1 = g.n1;
  for (int e = tid; e < 81; e += nth) {
    const int cls = e / 9, tap = e % 9;
    const int oa = tap % 3, ob = tap / 3;
    const int cx = cls % 3, cy = cls / 3;
    const int ix = cx == 0 ? 0 : (cx == 2 ? n1 - 1 : 1), iy = cy == 0 ? 0 : (cy == 2 ? n1 - 1 : 1);
    const double mx = g.tM[ix * 3 + oa], kx = g.tK[ix * 3 + oa];
    const double my = g.tM[iy * 3 + ob], ky = g.tK[iy * 3 + ob];
    tab[cls * 10 + tap] = ca * (my * mx) + cb * (ky * mx + my * kx);
  }
  __syncthreads();
  for (int cls = tid; cls < 9; cls += nth) tab[cls * 10 + 9] = 1.0 / tab[cls * 10 + 4];
}

// (A x)_i at node (i, j) of a 2-D Q1 level from its class stencil; 1 / A_ii in invD
__device__ __forceinline__ double2 class_eval_q1(const double* tabl, const double2* x, int i, int j, int n1,
                                                 double& invD) {
  const int cx = i == 0 ? 0 : (i == n1 - 1 ? 2 : 1), cy = j == 0 ? 0 : (j == n1 - 1 ? 2 : 1);
  const double* T = tabl + (cy * 3 + cx) * 10;
  invD = T[9];
  const int xl = i > 0 ? i - 1 : i, xr = i < n1 - 1 ? i + 1 : i;
  const int yl = j > 0 ? j - 1 : j, yr = j < n1 - 1 ? j + 1 : j;
  const double2* r0 = x + yl * n1;
  const double2* r1 = x + j * n1;
  const double2* r2 = x + yr * n1;
  double2 a0 = cscale(T[0], r0[xl]);
  a0 = cfma(T[1], r0[i], a0);
  a0 = cfma(T[2], r0[xr], a0);
  double2 a1 = cscale(T[3], r1[xl]);
  a1 = cfma(T[4], r1[i], a1);
  a1 = cfma(T[5], r1[xr], a1);
  double2 a2 = cscale(T[6], r2[xl]);
  a2 = cfma(T[7], r2[i], a2);
  a2 = cfma(T[8], r2[xr], a2);
  return cadd(cadd(a0, a1), a2);
}

// ---------------------------------------------------------------- CTA-resident solvers
// One CTA owns one problem (one frequency / slot / component) and runs the WHOLE fixed-count
// solve -- every level, colour, transfer and V-cycle -- with block barriers only.  The problems
// of a batch are independent, so the batch supplies the parallelism and no grid-wide
// synchronisation is ever needed; the iterate stays L1/L2-resident between colour steps.
template <int DIM, int ORD>
__device__ __forceinline__ long colour_count(int n1, int colour, int* res, int* cnt) {
  constexpr int C1 = ORD == 2 ? 3 : 2;
  long total = 1;
  int cc = colour;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    res[a] = cc % C1;
    cc /= C1;
    cnt[a] = (n1 - res[a] + C1 - 1) / C1;
    total *= cnt[a];
  }
  return total;
}

// node update of one multicolour SOR step: x_i += omega (b_i - (A x)_i) / A_ii
template <int DIM, int ORD, bool CONV>
__device__ __forceinline__ void sor_node(const Grid& g, const Coef& cf, const double* cv, double2* x, const double2* b,
                                         const int* c, int idx, double omega) {
  if (CONV) {
    double2 Ax, D;
    apply_op_conv<DIM, ORD>(g, cf, cv, x, c, idx, Ax, D);
    x[idx] = cadd(x[idx], cscale(omega, cdiv(csub(b[idx], Ax), D)));
  } else {
    double2 Ax;
    double D;
    apply_op_real<DIM, ORD>(g, cf.a.x, cf.b.x, x, c, idx, Ax, D);
    x[idx] = cadd(x[idx], cscale(omega / D, csub(b[idx], Ax)));
  }
}

// Thread groups for the CTA-resident solves: the whole block (big levels, __syncthreads) or one
// warp (the tiny bottom levels of each V-cycle, __syncwarp -- their phases are pure latency).
template <bool W>
__device__ __forceinline__ void gsync() {
  if (W)
    __syncwarp();
  else
    __syncthreads();
}

// Visit the unknown nodes with per-axis start s[a] and stride st[a] (interior range [lo, hi]),
// distributing them over the group's threads (tid, nth).
template <int DIM, class F>
__device__ __forceinline__ void cta_visit(int n1, const int* s0, const int* sta, int lo, int hi, int tid, int nth,
                                          F&& f) {
  int cnt[DIM], start[DIM], stv[DIM];
  int total = 1;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    int s = s0[a];
    while (s < lo) s += sta[a];
    start[a] = s;
    stv[a] = sta[a];
    cnt[a] = s > hi ? 0 : (hi - s) / sta[a] + 1;
    total *= cnt[a];
  }
  if (total == 0) return;
  for (int t = tid; t < total; t += nth) {
    int c[DIM];
    const unsigned q = (unsigned)t / (unsigned)cnt[0];
    c[0] = start[0] + stv[0] * (int)((unsigned)t - q * (unsigned)cnt[0]);
    if (DIM == 2) {
      c[1] = start[1] + stv[1] * (int)q;
    } else {
      const unsigned q2 = q / (unsigned)cnt[1];
      c[1] = start[1] + stv[1] * (int)(q - q2 * (unsigned)cnt[1]);
      c[2] = start[2] + stv[2] * (int)q2;
    }
    const int idx = DIM == 2 ? c[1] * n1 + c[0] : (c[2] * n1 + c[1]) * n1 + c[0];
    f(c, idx);
  }
}

// all unknowns of a level: Q2 in y/z parity classes (uniform taps per warp), Q1 in one pass
template <int DIM, int ORD, class F>
__device__ __forceinline__ void cta_all_unknowns(int n1, int tid, int nth, F&& f) {
  if (ORD == 2) {
    for (int cls = 0; cls < (1 << (DIM - 1)); ++cls) {
      int s0[DIM], st[DIM];
      s0[0] = 1;
      st[0] = 1;
#pragma unroll
      for (int a = 1; a < DIM; ++a) {
        s0[a] = ((cls >> (a - 1)) & 1) ? 1 : 2;
        st[a] = 2;
      }
      cta_visit<DIM>(n1, s0, st, 1, n1 - 2, tid, nth, f);
    }
  } else {
    int s0[DIM], st[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      s0[a] = 0;
      st[a] = 1;
    }
    cta_visit<DIM>(n1, s0, st, 0, n1 - 1, tid, nth, [&](const int* c, int idx) {
      if (idx != 0) f(c, idx);  // pinned node
    });
  }
}

// ---- band-wavefront multicolour SOR (2-D Q2, real class stencils) --------------------------------
// The 9 colour steps of one sweep are fused into ONE pass over the grid.  Rows are grouped in bands of
// H rows; a row j of class c = (j mod 3) (c' = 2 - c for the reversed colour order) is updated at step
// tau(j) = floor(j / H) + 2 c'.  For rows at distance <= 2 (the stencil reach) this orders every
// earlier colour before and every later colour after, exactly as the 9 separate colour steps do
// (|floor(j/H) - floor(j'/H)| <= 1 < 2 |c - c'|), and rows active in one step are >= H + 1 apart.
// Each step runs the three x-colours (i mod 3) of its three active bands in order.  The rows the
// active bands can touch (bands T-5 .. T+1) live in a shared-memory ring of 8 bands: a band is
// streamed in (cp.async) two steps ahead and written back when no later step can read it, so every
// value of the iterate crosses L2/HBM once per sweep instead of once per colour, and every stencil tap
// is a shared-memory load.  Same updates, same values as cta_sweep (only the summation schedule of
// independent nodes differs: none, each node's stencil sum is evaluated in the same order).
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_commit_all() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// TMA bulk copies (cp.async.bulk) and mbarriers for the band ring of q2_wave_pass
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* mb) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(mb)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(mb)), "r"(parity) : "memory");
}

// Q2 transfer weights in closed form (nodal interpolation between N_c and 2 N_c cells, reading 12): the
// same values as the host tables tP / tR (every product of them is exact in binary), without their loads.
// Restriction row of coarse node I (fine offsets -3..3 around 2 I): vertex (even I) {-1/8, 0, 3/8, 1, 3/8, 0, -1/8},
// midpoint (odd I) {0, 0, 3/4, 1, 3/4, 0, 0}.
__device__ __forceinline__ void q2_rrow(int I, double* w) {
  const bool mid = I & 1;
  w[0] = w[6] = mid ? 0.0 : -0.125;
  w[1] = w[5] = 0.0;
  w[2] = w[4] = mid ? 0.75 : 0.375;
  w[3] = 1.0;
}
// Prolongation of fine node f (interior): coarse nodes 2 (f >> 2) + {0, 1, 2}; f mod 4 = 0: {1, 0, 0}, 1: {3/8, 3/4,
// -1/8}, 2: {0, 1, 0}, 3: {-1/8, 3/4, 3/8}
__device__ __forceinline__ int q2_prow(int f, double* w) {
  const int r = f & 3;
  w[0] = r == 0 ? 1.0 : (r == 1 ? 0.375 : (r == 3 ? -0.125 : 0.0));
  w[1] = (r & 1) ? 0.75 : (r == 2 ? 1.0 : 0.0);
  w[2] = r == 1 ? -0.125 : (r == 3 ? 0.375 : 0.0);
  return 2 * (f >> 2);
}

template <int RR, int PY>
__device__ __forceinline__ double2 ring_eval_conv(const double2* T, const double* cvr, double2 cc, const double2* ring,
                                                  int r0, int i, int n1) {
  constexpr int AY0 = PY ? 1 : 0, AY1 = PY ? 4 : 5;
  const int xl = i >= 2 ? i - 2 : i, xr = i + 2 <= n1 - 1 ? i + 2 : i;
  double2 acc = make_double2(0.0, 0.0), nacc = acc;
#pragma unroll
  for (int ob = AY0; ob < AY1; ++ob) {
    int r = r0 + ob - 2;
    r += r < 0 ? RR : 0;
    r -= r >= RR ? RR : 0;
    const double2* row = ring + r * n1;
    const double2 v[5] = {row[xl], row[i - 1], row[i], row[i + 1], row[xr]};
#pragma unroll
    for (int oa = 0; oa < 5; ++oa) {
      acc = cadd(acc, cmul(T[ob * 5 + oa], v[oa]));
      nacc = cfma(__ldg(cvr + ob * 5 + oa), v[oa], nacc);
    }
  }
  return cadd(acc, cmul(cc, nacc));
}

template <int H>
__device__ void q2_wave_pass(const double* tabl, double2* x, const double2* __restrict__ b, double2* ring, int n1,
                             bool reverse, double omega, int tid, int nth, const double* cv = nullptr,
                             double2 cc = make_double2(0.0, 0.0), double2* rout = nullptr,
                             const double2* xcoarse = nullptr, int n1c = 0, unsigned long long* mbar = nullptr) {
  static_assert(H % 3 == 0, "band height must be a multiple of the 3 row classes");
  constexpr int RR = 8 * H;   // ring rows: 8 bands
  const int nb = (n1 + H - 1) / H;
  auto band_rows = [&](int band, int& j0, int& cnt) {
    j0 = band * H;
    cnt = (min(n1, j0 + H) - j0) * n1;
  };
  // Band copies.  Plain sweeps stream a band of the iterate into the ring with one TMA bulk copy (cp.async.bulk,
  // 3 H n1 complex values, contiguous in both places) completing on the slot's mbarrier, and write a final band back
  // with one bulk store; the CTA's threads only wait on the mbarrier.  With xcoarse (first post-smoothing sweep) the
  // coarse-grid correction x += P x_c (nodal interpolation, mg_up's arithmetic) is applied on the way in by the
  // threads instead of in a separate pass over the level.
  // mbarriers (8 slots) and their phase bits: after the finest level's ring (initialised at kernel start)
  unsigned* phase_word = reinterpret_cast<unsigned*>(mbar + MG_TRI_SLOTS);
  unsigned phase = *phase_word;          // bit s: parity of the next completion of slot s
  const bool tma = xcoarse == nullptr;
  auto load_band = [&](int band) {
    int j0, cnt;
    band_rows(band, j0, cnt);
    double2* dst = ring + (j0 % RR) * n1;
    const double2* src = x + (long)j0 * n1;
    if (tma) {
      if (tid == 0) bulk_load(dst, src, (unsigned)cnt * sizeof(double2), mbar + band % 8);
      return;
    }
    for (int e = tid; e < cnt; e += nth) {
      const int jj = e / n1, j = j0 + jj, i = e - jj * n1;
      double2 v = src[e];
      if (j >= 1 && j <= n1 - 2 && i >= 1 && i <= n1 - 2) {
        double wy[3], wx[3];
        const int by = q2_prow(j, wy), bx = q2_prow(i, wx);
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int ob = 0; ob < 3; ++ob)
#pragma unroll
          for (int oa = 0; oa < 3; ++oa) {
            const double ww = wy[ob] * wx[oa];
            if (ww != 0.0) acc = cfma(ww, xcoarse[(by + ob) * n1c + bx + oa], acc);
          }
        v = cadd(v, acc);
      }
      dst[e] = v;
    }
  };
  auto wait_band = [&](int band) {      // TMA loads: wait for the slot's completion (all threads)
    if (!tma) return;
    const int sl = band % 8;
    mbar_wait(mbar + sl, (phase >> sl) & 1u);
    phase ^= 1u << sl;
  };
  auto store_band = [&](int band) {     // by thread 0, after a fence + barrier of all writers
    int j0, cnt;
    band_rows(band, j0, cnt);
    bulk_store(x + (long)j0 * n1, ring + (j0 % RR) * n1, (unsigned)cnt * sizeof(double2));
  };
  auto copy_back = [&](int band) {      // write a band back by the threads (prolongation sweep)
    int j0, cnt;
    band_rows(band, j0, cnt);
    const double2* src = ring + (j0 % RR) * n1;
    double2* dst = x + (long)j0 * n1;
    for (int e = tid; e < cnt; e += nth) dst[e] = src[e];
  };
  // generic writes of the iterate (previous passes, zeroing) before the async-proxy reads
  fence_async_global();
  __syncthreads();
  load_band(0);
  if (nb > 1) load_band(1);
  // Work items of x-colour step q (x residue i0 = i0s[rx]): t = p per + kk cx + m covers the three active bands
  // T - 2p (p = 0, 1, 2; row class cls = p, reversed 2 - p), rows band H + cls + 3 kk (kk < H / 3), columns
  // i0 + 3 m.  H is a multiple of 3, so a work item keeps its (p, row offset, column) from one band step to the next
  // and only its band advances: the mapping is decoded once per thread (at most 2 items per thread and step:
  // 3 H cx <= 2 nth for every level that uses the wavefront) and packed as i | off << 11 | p << 20.
  const int i0s[3] = {3, 1, 2};
  int item[3][2];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int i0 = i0s[reverse ? 2 - q : q];
    const int cx = i0 > n1 - 2 ? 0 : (n1 - 2 - i0) / 3 + 1;
    const int per = (H / 3) * cx;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int t = tid + u * nth;
      item[q][u] = -1;
      if (t < 3 * per) {
        const int p = t / per, rem = t - p * per;
        const int kk = rem / cx, m = rem - kk * cx;
        const int cls = reverse ? 2 - p : p;
        item[q][u] = (i0 + 3 * m) | ((cls + 3 * kk) << 11) | (p << 20);
      }
    }
  }
  for (int T = 0; T <= nb + 3; ++T) {
    // bands T - 5 .. T + 1 are touched in this step; band T + 1 (issued in step T - 1) must have landed
    if (T == 0) wait_band(0);
    if (T + 1 < nb) wait_band(T + 1);
    if (tma) fence_async_smem();       // this thread's ring writes (step T - 1) -> visible to the bulk store
    __syncthreads();
    if (tma) {
      if (tid == 0) {
        bulk_wait_read();               // the store of band T - 6 (issued in step T - 1) has read its slot
        if (T + 2 < nb) load_band(T + 2);
        if (T - 5 >= 0 && T - 5 < nb) store_band(T - 5);   // final since step T - 1; only read from now on
      }
    } else {
      if (T >= 6) {
        copy_back(T - 6);
        __syncthreads();
      }
      if (T + 2 < nb) load_band(T + 2);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int it = item[q][u];
        if (it < 0) continue;
        const int band = T - 2 * (it >> 20);
        const int j = band * H + ((it >> 11) & 511);
        if (band < 0 || band >= nb || j < 1 || j > n1 - 2) continue;
        const int i = it & 2047;
        const double2 bb = b[(long)j * n1 + i];
        const int r0 = j % RR;
        const int ccls = (i & 1) | ((j & 1) << 1);
        double2* xp = ring + r0 * n1 + i;
        const double2* Tc = reinterpret_cast<const double2*>(tabl) + ccls * ClassTab<2>::NT;
        const double* cvr = cv + ((long)j * n1 + i) * ClassTab<2>::NT;
        const double2 Ax = (j & 1) ? ring_eval_conv<RR, 1>(Tc, cvr, cc, ring, r0, i, n1)
                                   : ring_eval_conv<RR, 0>(Tc, cvr, cc, ring, r0, i, n1);
        const double2 D = cadd(Tc[12], cscale(__ldg(cvr + 12), cc));
        const double2 xo = *xp;
        *xp = cadd(xo, cscale(omega, cdiv(csub(bb, Ax), D)));
      }
      __syncthreads();
    }
    // fused residual (last pre-smoothing sweep, forward colour order): band T - 4 has had its last row class
    // updated in this step, and every row its stencils reach is final (band T - 5 and the first two row classes of
    // band T - 3); r = b - A x on its interior nodes, from the ring (same taps, same order as the separate pass)
    if (rout != nullptr) {
      const int F = T - 4;
      if (F >= 0 && F < nb) {
        const int j0 = max(1, F * H), j1 = min(n1 - 2, F * H + H - 1);
        const int w = n1 - 2, cnt = (j1 - j0 + 1) * w;
        for (int e = tid; e < cnt; e += nth) {
          const int jj = e / w, j = j0 + jj, i = 1 + (e - jj * w);
          const int r0 = j % RR;
          const double2 bb = b[(long)j * n1 + i];
          const int ccls = (i & 1) | ((j & 1) << 1);
          const double2* Tc = reinterpret_cast<const double2*>(tabl) + ccls * ClassTab<2>::NT;
          const double* cvr = cv + ((long)j * n1 + i) * ClassTab<2>::NT;
          const double2 Ax = (j & 1) ? ring_eval_conv<RR, 1>(Tc, cvr, cc, ring, r0, i, n1)
                                     : ring_eval_conv<RR, 0>(Tc, cvr, cc, ring, r0, i, n1);
          rout[(long)j * n1 + i] = csub(bb, Ax);
        }
      }
    }
  }
  if (tma) {
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      if (nb - 1 > nb + 3 - 5) store_band(nb - 1);   // the last band (final after step nb + 3)
      bulk_wait_all();
      fence_async_global();
      *phase_word = phase;
    }
  } else {
    for (int band = max(0, nb - 2); band < nb; ++band)
      if (band + 6 > nb + 3) copy_back(band);
  }
  __syncthreads();
}

// ---- band-wavefront sweeps in triple form (2-D Q2, real class stencils) ------------------------------------------
// The same schedule of updates as q2_wave_pass (bands of H rows; a row of class c' in band B is updated at step
// B + 2 c'; the three x-colours of a step run in order), reorganised so that the barrier-separated x-colour phases
// carry almost no work.  A thread owns the three consecutive nodes (3m, 3m+1, 3m+2) of one active row: one node of
// each x-colour.  Rows j +- 1, j +- 2 belong to other row classes and are not written during the step, and within
// row j only the triple itself and the colour-0 / colour-1 nodes of the neighbouring triple (m + 1; m - 1 for the
// reversed colour order) change before the triple's last update.  So every tap that cannot change is accumulated up
// front in one phase with all loads independent -- 7 columns x 5 rows serve the three nodes, 35 shared-memory loads
// instead of 3 x 25 -- and each x-colour phase only adds its one or two fresh values and updates its node.  The
// reversed order is the mirror image: local column c stands for i0 + 4 - c, local tap oa for 4 - oa.
// Columns -2, -1 (m = 0) and n1 .. n1 + 2 (last triple) fall into the neighbouring ring rows or the zeroed guard
// around the ring; they only meet zero coefficients (midpoint rows have three taps) or inactive boundary nodes.
// lanes a row of ntr triples takes in the thread mapping of q2_tri_pass
__host__ __device__ __forceinline__ int tri_lanes_per_row(int ntr) {
  if (ntr >= 32) return (ntr + 31) / 32 * 32;
  int l = 1;
  while (l < ntr) l *= 2;
  return l;
}

template <bool REV, int PY, bool FULL>
__device__ __forceinline__ void tri_accumulate(const double* __restrict__ Ta, const double* __restrict__ Tb,
                                               const double2* ring, int r0, int RR, int n1, int cb, double2* acc,
                                               double2* xo) {
  constexpr int AY0 = PY ? 1 : 0, AY1 = PY ? 4 : 5;
#pragma unroll
  for (int ob = AY0; ob < AY1; ++ob) {
    int r = r0 + ob - 2;
    r += r < 0 ? RR : 0;
    r -= r >= RR ? RR : 0;
    const double2* row = ring + r * n1 + cb;
    double ta[5], tb[5];
#pragma unroll
    for (int oa = 0; oa < 5; ++oa) {
      ta[oa] = Ta[ob * 5 + (REV ? 4 - oa : oa)];
      tb[oa] = Tb[ob * 5 + (REV ? 4 - oa : oa)];
    }
    if (FULL || ob != 2) {
      double2 v[7];
#pragma unroll
      for (int c = 0; c < 7; ++c) v[c] = row[REV ? -c : c];
#pragma unroll
      for (int oa = 0; oa < 5; ++oa) {
        acc[0] = cfma(ta[oa], v[oa], acc[0]);
        acc[1] = cfma(tb[oa], v[1 + oa], acc[1]);
        acc[2] = cfma(ta[oa], v[2 + oa], acc[2]);
      }
    } else {
      // row j: node 0 (first colour) sees only old values; nodes 1 and 2 take their fresh taps in their own phase
      double2 v[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) v[c] = row[REV ? -c : c];
      xo[0] = v[2];
      xo[1] = v[3];
      xo[2] = v[4];
#pragma unroll
      for (int oa = 0; oa < 5; ++oa) acc[0] = cfma(ta[oa], v[oa], acc[0]);
      acc[1] = cfma(tb[0], v[1], acc[1]);
      acc[1] = cfma(tb[2], v[3], acc[1]);
      acc[1] = cfma(tb[3], v[4], acc[1]);
      acc[2] = cfma(ta[2], v[4], acc[2]);
    }
  }
}

// one band step of the triple-form sweep for this thread's item (see q2_tri_pass)
// x-colour phases synchronise only the threads of one row class (named barrier 1 + p, a whole number of warps):
// updates of different row classes touch rows at least four apart and never exchange values within a step.
__device__ __forceinline__ void class_sync(int bar_id, int bar_threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_threads) : "memory");
}

template <bool REV>
__device__ __forceinline__ void tri_step(const double* tabl, double2* ring, int n1, int RR, int j, int r0, int i0,
                                         int px, bool on, const bool* act, double omega, double2* acc, int bar_id,
                                         int bar_threads) {
  const int cb = REV ? i0 + 4 : i0 - 2;
  const int py = j & 1;
  // class stencils of the x-parity of nodes 0 and 2 (Ta) and of node 1 (Tb); lanes alternate in parity, the two
  // addresses of a warp fall into different banks (a select from two broadcast loads was measured no faster)
  const double* Ta = tabl + (px | (py << 1)) * (ClassTab<2>::NT + 1);
  const double* Tb = tabl + ((px ^ 1) | (py << 1)) * (ClassTab<2>::NT + 1);
  double2 xo[3] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  double2* rowj = ring + r0 * n1 + cb;
  double wa = 0.0, wb = 0.0, tb1 = 0.0, tb4 = 0.0, ta0 = 0.0, ta1 = 0.0, ta3 = 0.0, ta4 = 0.0;
  if (on) {
    if (py) tri_accumulate<REV, 1, false>(Ta, Tb, ring, r0, RR, n1, cb, acc, xo);
    else tri_accumulate<REV, 0, false>(Ta, Tb, ring, r0, RR, n1, cb, acc, xo);
    wa = omega * Ta[ClassTab<2>::NT];
    wb = omega * Tb[ClassTab<2>::NT];
    tb1 = Tb[10 + (REV ? 3 : 1)];
    tb4 = Tb[10 + (REV ? 0 : 4)];
    ta0 = Ta[10 + (REV ? 4 : 0)];
    ta1 = Ta[10 + (REV ? 3 : 1)];
    ta3 = Ta[10 + (REV ? 1 : 3)];
    ta4 = Ta[10 + (REV ? 0 : 4)];
  }
  // first x-colour
  double2 x0n = xo[0];
  if (on && act[0]) {
    x0n = make_double2(xo[0].x - wa * acc[0].x, xo[0].y - wa * acc[0].y);
    rowj[REV ? -2 : 2] = x0n;
  }
  class_sync(bar_id, bar_threads);
  // second x-colour: fresh taps = own first node and the first node of the next triple
  double2 x1n = xo[1];
  double2 v5 = make_double2(0.0, 0.0);
  if (on) {
    v5 = rowj[REV ? -5 : 5];
    if (act[1]) {
      double2 a1 = cfma(tb1, x0n, acc[1]);
      a1 = cfma(tb4, v5, a1);
      x1n = make_double2(xo[1].x - wb * a1.x, xo[1].y - wb * a1.y);
      rowj[REV ? -3 : 3] = x1n;
    }
  }
  class_sync(bar_id, bar_threads);
  // third x-colour
  if (on && act[2]) {
    const double2 v6 = rowj[REV ? -6 : 6];
    double2 a2 = cfma(ta0, x0n, acc[2]);
    a2 = cfma(ta1, x1n, a2);
    a2 = cfma(ta3, v5, a2);
    a2 = cfma(ta4, v6, a2);
    rowj[REV ? -4 : 4] = make_double2(xo[2].x - wa * a2.x, xo[2].y - wa * a2.y);
  }
}

// Ring of MG_TRI_SLOTS = 9 band slots.  At step T the bands T - 4 .. T are updated (rows up to band T + 1 and down to
// band T - 5 are read), band T + 1 has landed, band T + 2 is being loaded, band T - 5 (final since step T - 1) is
// stored and, in the sweep that also produces the residual, r = b - A x of band T - 5 is formed from final values
// (its stencils reach the last rows of band T - 6 and the first two rows -- row classes 0 and 1, final -- of band
// T - 4): nothing this step writes is read by it, so it needs no barrier of its own.  The slot loaded at step T held
// band T - 7, whose store was issued two steps earlier, so the copy thread never waits for the latest store to drain.
// N1C / HC: the level size and band height as compile-time constants for the two big levels of the BASELINE
// meshes (513 / 3 and 257 / 6), 0 = the run-time values (every other level; same code).
template <int N1C, int HC>
__device__ __forceinline__ void q2_tri_pass(const double* tabl, double2* x, const double2* __restrict__ b, double2* ring,
                                            int n1r, int Hr, bool reverse, double omega, int tid, int nth, double2* rout,
                                            const double2* xcoarse, int n1c, unsigned long long* mbar,
                                            unsigned long long* clk = nullptr) {
  const int n1 = N1C ? N1C : n1r, H = HC ? HC : Hr;
  constexpr int NS = MG_TRI_SLOTS;
  const int RR = NS * H;
  const int nb = (n1 + H - 1) / H;
  auto band_rows = [&](int band, int& j0, int& cnt) {
    j0 = band * H;
    cnt = (min(n1, j0 + H) - j0) * n1;
  };
  // band copies: TMA bulk copies on the slot mbarriers, issued by the copy thread.  With xcoarse (first
  // post-smoothing sweep) the coarse-grid correction x += P x_c (nodal interpolation, mg_up's arithmetic) is added
  // to a band in the ring once it has landed -- at the end of the step that issued its load, one step before it is
  // first read -- instead of in a separate pass over the level.
  unsigned* phase_word = reinterpret_cast<unsigned*>(mbar + NS);
  unsigned phase = *phase_word;
  const bool corr = xcoarse != nullptr;
  auto load_band = [&](int band) {
    int j0, cnt;
    band_rows(band, j0, cnt);
    bulk_load(ring + (band % NS) * H * n1, x + (long)j0 * n1, (unsigned)cnt * sizeof(double2), mbar + band % NS);
  };
  auto wait_band = [&](int band) {
    const int sl = band % NS;
    mbar_wait(mbar + sl, (phase >> sl) & 1u);
    phase ^= 1u << sl;
  };
  auto correct_band = [&](int band) {   // ring band += P x_c (all threads; the band has landed)
    int j0, cnt;
    band_rows(band, j0, cnt);
    double2* dst = ring + (band % NS) * H * n1;
    for (int e = tid; e < cnt; e += nth) {
      const int jj = e / n1, j = j0 + jj, i = e - jj * n1;
      if (j >= 1 && j <= n1 - 2 && i >= 1 && i <= n1 - 2) {
        double wy[3], wx[3];
        const int by = q2_prow(j, wy), bx = q2_prow(i, wx);
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int ob = 0; ob < 3; ++ob)
#pragma unroll
          for (int oa = 0; oa < 3; ++oa) {
            const double ww = wy[ob] * wx[oa];
            if (ww != 0.0) acc = cfma(ww, xcoarse[(by + ob) * n1c + bx + oa], acc);
          }
        dst[e] = cadd(dst[e], acc);
      }
    }
  };
  auto store_band = [&](int band) {
    int j0, cnt;
    band_rows(band, j0, cnt);
    bulk_store(x + (long)j0 * n1, ring + (band % NS) * H * n1, (unsigned)cnt * sizeof(double2));
  };
  // this thread's item: row class slot p (band lag 2 p), row kk of that class within the band, triple m.  A row
  // takes lpr lanes (tri_lanes_per_row: whole warps, or a power-of-two fraction of a warp on small levels), so the
  // threads of a row class are whole warps: they synchronise among themselves, and on the big levels a warp works
  // on one row (one row parity: no divergence between the 5-row and 3-row stencils).
  const int ntr = (n1 - 2) / 3 + 1;
  const int lpr = tri_lanes_per_row(ntr);
  const int per = (H / 3) * lpr;            // threads of one row class
  // the copy thread: the block's last thread (a spare lane: ntr < lpr on every level with n1 = 2^k + 1)
  const bool copier = tid == nth - 1;
  fence_async_global();   // generic writes of the iterate (previous passes, zeroing) before the async-proxy reads
  __syncthreads();
  if (copier) {
    load_band(0);
    if (nb > 1) load_band(1);
  }
  if (corr) {   // the first two bands are corrected before step 0 reads them
    wait_band(0);
    correct_band(0);
    if (nb > 1) {
      wait_band(1);
      correct_band(1);
    }
  }
  int p = 0, kk = 0, m = 0;
  bool has = tid < 3 * per;
  if (has) {
    p = tid / per;
    const int rem = tid - p * per;
    kk = rem / lpr;
    m = rem - kk * lpr;
    has = m < ntr;
  }
  // barrier group of the x-colour phases: the row class (whole warps), or the whole block where a class is a
  // fraction of a warp (small levels with forced 3- or 6-row bands)
  const bool grouped = (per & 31) == 0;
  const bool in_class = !grouped || tid < 3 * per;
  const int bar_id = grouped ? 1 + p : 0, bar_threads = grouped ? per : nth;
  const int rowoff = (reverse ? 2 - p : p) + 3 * kk;
  const int i0 = 3 * m, px = m & 1;
  int gc[3];     // global columns of the local nodes (update order)
  bool act[3];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    gc[n] = reverse ? i0 + 2 - n : i0 + n;
    act[n] = gc[n] >= 1 && gc[n] <= n1 - 2;
  }
  const int rrow = p * (H / 3) + kk;   // residual item: row rrow of band T - 5, the same triple
  const double2 zero = make_double2(0.0, 0.0);
  double2 bn[3] = {zero, zero, zero};
  if (has && p == 0 && rowoff >= 1 && rowoff <= n1 - 2) {   // step 0: band 0 for p = 0
#pragma unroll
    for (int n = 0; n < 3; ++n)
      if (act[n]) bn[n] = b[rowoff * n1 + gc[n]];
  }
  int slot = (NS - 2 * p) % NS;   // ring slot of this item's band T - 2 p at T = 0 (p <= 2)
#ifdef AAO_TRI_CLOCK   // per-phase cycle accounting of the steps (build with -DAAO_TRI_CLOCK, run with AAO_MG_CLOCK)
  unsigned long long pt = clk ? clock64() : 0ull;
  auto pmark = [&](int sl) {
    if (clk) {
      const unsigned long long t1 = clock64();
      clk[sl] += t1 - pt;
      pt = t1;
    }
  };
#else
  auto pmark = [](int) {};
#endif
  for (int T = 0; T <= nb + 4; ++T) {
    if (!corr) {   // (with the correction, a band was waited for when it was corrected)
      if (T == 0) wait_band(0);
      if (T + 1 < nb) wait_band(T + 1);
    }
    pmark(16);
    fence_async_smem();   // this thread's ring writes (step T - 1) -> visible to the bulk store
    __syncthreads();
    pmark(17);
    if (copier) {
      bulk_wait_read1();          // all but the latest store have read their slot: band T - 7's slot is free
      if (T + 2 < nb) load_band(T + 2);
      if (T - 5 >= 0 && T - 5 < nb) store_band(T - 5);
    }
    pmark(18);
    const int band = T - 2 * p;
    const int j = band * H + rowoff;
    const bool on = has && band >= 0 && band < nb && j >= 1 && j <= n1 - 2;
    const int r0 = slot * H + rowoff;
    slot = slot == NS - 1 ? 0 : slot + 1;
    double2 acc[3] = {make_double2(-bn[0].x, -bn[0].y), make_double2(-bn[1].x, -bn[1].y),
                      make_double2(-bn[2].x, -bn[2].y)};
    {   // right-hand side of the next step's row
      const int j1 = j + H;
      const bool on1 = has && band + 1 >= 0 && band + 1 < nb && j1 >= 1 && j1 <= n1 - 2;
#pragma unroll
      for (int n = 0; n < 3; ++n) bn[n] = (on1 && act[n]) ? b[j1 * n1 + gc[n]] : zero;
    }
    if (in_class) {
      if (reverse) tri_step<true>(tabl, ring, n1, RR, j, r0, i0, px, on, act, omega, acc, bar_id, bar_threads);
      else tri_step<false>(tabl, ring, n1, RR, j, r0, i0, px, on, act, omega, acc, bar_id, bar_threads);
    }
    pmark(19);
    // fused residual (last pre-smoothing sweep, forward order) of band T - 5
    if (rout != nullptr) {
      const int F = T - 5;
      const int jr = F * H + rrow;
      if (has && F >= 0 && F < nb && jr >= 1 && jr <= n1 - 2) {
        double2 bb[3];
#pragma unroll
        for (int n = 0; n < 3; ++n) bb[n] = act[n] ? b[jr * n1 + i0 + n] : zero;
        double2 ra[3] = {zero, zero, zero};
        const int rr0 = (F % NS) * H + rrow;
        const int pyr = jr & 1;
        const double* Ta = tabl + (px | (pyr << 1)) * (ClassTab<2>::NT + 1);
        const double* Tb = tabl + ((px ^ 1) | (pyr << 1)) * (ClassTab<2>::NT + 1);
        if (pyr) tri_accumulate<false, 1, true>(Ta, Tb, ring, rr0, RR, n1, i0 - 2, ra, nullptr);
        else tri_accumulate<false, 0, true>(Ta, Tb, ring, rr0, RR, n1, i0 - 2, ra, nullptr);
#pragma unroll
        for (int n = 0; n < 3; ++n)
          if (act[n]) rout[jr * n1 + i0 + n] = csub(bb[n], ra[n]);
      }
      pmark(14);
    }
    if (corr && T + 2 < nb) {   // band T + 2 (issued at the top of this step): correct it once it has landed
      wait_band(T + 2);
      correct_band(T + 2);
    }
  }
  __syncthreads();
  if (copier) {
    bulk_wait_all();
    fence_async_global();
  }
  if (tid == 0) *phase_word = phase;
  __syncthreads();
}

// ---- band-wavefront sweeps in pair form (2-D Q1, real position-class stencils: the pressure MG) --------------------
// The Q1 analogue of q2_tri_pass.  Colours (i mod 2) + 2 (j mod 2); bands of H rows (H even); the rows of class c'
// (j mod 2, mirrored for the reversed order) of band B are updated at step B + 2 c' (a row's neighbours j +- 1 of the
// other class may sit in the next or previous band: the lag of two steps orders them as the colour steps do).  A
// thread owns the pair (2m, 2m + 1) of one active row: its first node sees only old values (rows j +- 1 are not
// written during the step), its second needs the fresh first node and the fresh first node of the next pair.
// Ring of MG_TRI_SLOTS band slots filled and drained by TMA bulk copies as in q2_tri_pass: at step T band T + 1 has
// landed, band T + 2 is loading, band T - 3 (final since step T - 1) is stored.  Taps that leave the grid have zero
// coefficients in the position classes and read finite ring or guard entries.
__device__ __forceinline__ void q1_pair_pass(const double* tabl, double2* x, const double2* __restrict__ b, double2* ring,
                                             int n1, int H, bool reverse, double omega, int tid, int nth,
                                             unsigned long long* mbar) {
  constexpr int NS = MG_TRI_SLOTS;
  const int RR = NS * H;
  const int nb = (n1 + H - 1) / H;
  auto band_rows = [&](int band, int& j0, int& cnt) {
    j0 = band * H;
    cnt = (min(n1, j0 + H) - j0) * n1;
  };
  unsigned* phase_word = reinterpret_cast<unsigned*>(mbar + NS);
  unsigned phase = *phase_word;
  auto load_band = [&](int band) {
    int j0, cnt;
    band_rows(band, j0, cnt);
    bulk_load(ring + (band % NS) * H * n1, x + (long)j0 * n1, (unsigned)cnt * sizeof(double2), mbar + band % NS);
  };
  auto wait_band = [&](int band) {
    const int sl = band % NS;
    mbar_wait(mbar + sl, (phase >> sl) & 1u);
    phase ^= 1u << sl;
  };
  auto store_band = [&](int band) {
    int j0, cnt;
    band_rows(band, j0, cnt);
    bulk_store(x + (long)j0 * n1, ring + (band % NS) * H * n1, (unsigned)cnt * sizeof(double2));
  };
  const int np = (n1 + 1) / 2;                 // pairs per row
  const int lpr = tri_lanes_per_row(np);
  // a thread owns its pair in U rows of its class (U = 2 when H is a multiple of 4: half the band steps for the
  // same per-step overhead -- wait, fence, barriers -- which dominates a step of so little arithmetic)
  constexpr int UMAX = 2;
  const int U = (H & 3) == 0 ? 2 : 1;
  const int per = (H / 2 / U) * lpr;           // threads of one row class
  const bool copier = tid == nth - 1;
  fence_async_global();
  __syncthreads();
  if (copier) {
    load_band(0);
    if (nb > 1) load_band(1);
  }
  int p = 0, kk = 0, m = 0;
  bool has = tid < 2 * per;
  if (has) {
    p = tid / per;
    const int rem = tid - p * per;
    kk = rem / lpr;
    m = rem - kk * lpr;
    has = m < np;
  }
  const bool grouped = (per & 31) == 0;
  const bool in_class = !grouped || tid < 2 * per;
  const int bar_id = grouped ? 1 + p : 0, bar_threads = grouped ? per : nth;
  const int rowoff0 = (reverse ? 1 - p : p) + 2 * kk * U;   // row u of this thread: rowoff0 + 2 u
  // local frame: column c = 0..3 stands for 2m - 1 + c (2m + 2 - c for the reversed order); nodes at c = 1, 2
  const int cb = reverse ? 2 * m + 2 : 2 * m - 1;
  const int sgn = reverse ? -1 : 1;
  const int g0 = reverse ? 2 * m + 1 : 2 * m, g1 = reverse ? 2 * m : 2 * m + 1;
  const int cx0 = g0 == 0 ? 0 : (g0 == n1 - 1 ? 2 : 1), cx1 = g1 == 0 ? 0 : (g1 == n1 - 1 ? 2 : 1);
  const bool in0 = has && g0 <= n1 - 1, in1 = has && g1 <= n1 - 1;
  const double2 zero = make_double2(0.0, 0.0);
  double2 bn0[UMAX] = {zero, zero}, bn1[UMAX] = {zero, zero};
#pragma unroll
  for (int u = 0; u < UMAX; ++u) {   // step 0: band 0 for p = 0
    const int jr = rowoff0 + 2 * u;
    if (u < U && p == 0 && jr <= n1 - 1) {
      if (in0) bn0[u] = b[jr * n1 + g0];
      if (in1) bn1[u] = b[jr * n1 + g1];
    }
  }
  int slot = (NS - 2 * p) % NS;
  for (int T = 0; T <= nb + 2; ++T) {
    if (T == 0) wait_band(0);
    if (T + 1 < nb) wait_band(T + 1);
    fence_async_smem();
    __syncthreads();
    if (copier) {
      bulk_wait_read1();
      if (T + 2 < nb) load_band(T + 2);
      if (T - 3 >= 0 && T - 3 < nb) store_band(T - 3);
    }
    const int band = T - 2 * p;
    const bool bandon = has && band >= 0 && band < nb;
    const bool band1on = band + 1 >= 0 && band + 1 < nb;
    const int rs = slot * H;
    slot = slot == NS - 1 ? 0 : slot + 1;
    double2 acc0[UMAX], acc1[UMAX], xo0[UMAX], xo1[UMAX], x0n[UMAX];
    double t10[UMAX], t12[UMAX], w0[UMAX], w1[UMAX];
    bool act0[UMAX], act1[UMAX];
#pragma unroll
    for (int u = 0; u < UMAX; ++u) {
      acc0[u] = make_double2(-bn0[u].x, -bn0[u].y);
      acc1[u] = make_double2(-bn1[u].x, -bn1[u].y);
      const int j1 = (band + 1) * H + rowoff0 + 2 * u;
      const bool on1 = u < U && band1on && j1 >= 0 && j1 <= n1 - 1;
      bn0[u] = (on1 && in0) ? b[j1 * n1 + g0] : zero;
      bn1[u] = (on1 && in1) ? b[j1 * n1 + g1] : zero;
    }
    if (!in_class) continue;
#pragma unroll
    for (int u = 0; u < UMAX; ++u) {
      const int ro = rowoff0 + 2 * u;
      const int j = band * H + ro;
      const bool on = u < U && bandon && j >= 0 && j <= n1 - 1;
      const int r0 = rs + ro;
      const int cy = j == 0 ? 0 : (j == n1 - 1 ? 2 : 1);
      const double* T0 = tabl + (cy * 3 + cx0) * 10;
      const double* T1 = tabl + (cy * 3 + cx1) * 10;
      act0[u] = on && in0 && !(j == 0 && g0 == 0);   // (pinned corner)
      act1[u] = on && in1 && !(j == 0 && g1 == 0);
      xo0[u] = xo1[u] = zero;
      t10[u] = t12[u] = w0[u] = w1[u] = 0.0;
      if (on) {
#pragma unroll
        for (int ob = 0; ob < 3; ++ob) {
          int r = r0 + ob - 1;
          r += r < 0 ? RR : 0;
          r -= r >= RR ? RR : 0;
          const double2* row = ring + r * n1 + cb;
          const double2 v0 = row[0], v1 = row[sgn], v2 = row[2 * sgn], v3 = row[3 * sgn];
          const double a0 = T0[ob * 3 + (reverse ? 2 : 0)], a1 = T0[ob * 3 + 1], a2 = T0[ob * 3 + (reverse ? 0 : 2)];
          const double c0 = T1[ob * 3 + (reverse ? 2 : 0)], c1 = T1[ob * 3 + 1], c2 = T1[ob * 3 + (reverse ? 0 : 2)];
          acc0[u] = cfma(a0, v0, acc0[u]);
          acc0[u] = cfma(a1, v1, acc0[u]);
          acc0[u] = cfma(a2, v2, acc0[u]);
          if (ob != 1) {
            acc1[u] = cfma(c0, v1, acc1[u]);
            acc1[u] = cfma(c1, v2, acc1[u]);
            acc1[u] = cfma(c2, v3, acc1[u]);
          } else {   // row j: the second node takes its two fresh taps after the first colour
            xo0[u] = v1;
            xo1[u] = v2;
            acc1[u] = cfma(c1, v2, acc1[u]);
            t10[u] = c0;
            t12[u] = c2;
          }
        }
        w0[u] = omega * T0[9];
        w1[u] = omega * T1[9];
      }
      x0n[u] = xo0[u];
      if (act0[u]) {
        x0n[u] = make_double2(xo0[u].x - w0[u] * acc0[u].x, xo0[u].y - w0[u] * acc0[u].y);
        ring[r0 * n1 + cb + sgn] = x0n[u];
      }
    }
    class_sync(bar_id, bar_threads);
#pragma unroll
    for (int u = 0; u < UMAX; ++u) {
      if (act1[u]) {
        double2* rowj = ring + (rs + rowoff0 + 2 * u) * n1 + cb;
        const double2 v3 = rowj[3 * sgn];
        double2 a = cfma(t10[u], x0n[u], acc1[u]);
        a = cfma(t12[u], v3, a);
        rowj[2 * sgn] = make_double2(xo1[u].x - w1[u] * a.x, xo1[u].y - w1[u] * a.y);
      }
    }
  }
  __syncthreads();
  if (copier) {
    bulk_wait_all();
    fence_async_global();
  }
  if (tid == 0) *phase_word = phase;
  __syncthreads();
}

// ---- z-band wavefront sweeps in line form (3-D Q2, real class stencils) -------------------------------------------
// The schedule of the 3-D z-band wavefront (planes in bands of 3, band B updates its plane of z-class c' at step
// B + 2 c', the 9 xy-colours of a step in order), with the work of a step given to warps line by line: a warp owns
// one x-line (y = j, z = k) of the current y-class and each lane the triple (3m, 3m+1, 3m+2) of it, as in the 2-D
// triple form.  The up to 25 neighbouring lines (j + dy, k + dz) are not written while the line is updated; the
// warp copies each of them once, coalesced, into a small shared-memory stage and every lane takes its 7 columns
// from there (the per-node form re-read them from L1 with stride-3 lane addresses: 3 x 125 taps per triple, twelve
// cache lines per warp load).  The x-colours of a line are ordered inside the warp -- the two fresh neighbour
// values come by shuffle -- so a step needs one block barrier per y-class instead of one per xy-colour.
// Lines of one y-class are three apart and the three active planes five apart: no line read here is being written.
constexpr int ZL_PAD = 4;   // zeroed entries before and after a staged line
#ifndef ZL_STAGES
#define ZL_STAGES MG_ZL_STAGES   // staged lines per warp (ring of cp.async copies)
#endif

template <bool REV, int PY, int PZ>
__device__ __forceinline__ void zline_accumulate(const double* __restrict__ Ta, const double* __restrict__ Tb,
                                                 const double2* x, int n1, int j, int k, int cb, bool has, int lane,
                                                 double2* stage, int& buf, double2* acc, double2* xo,
                                                 double2& v5old, double2& v6old) {
  constexpr int AY0 = PY ? 1 : 0, NY = PY ? 3 : 5;
  constexpr int AZ0 = PZ ? 1 : 0, NZ = PZ ? 3 : 5;
  constexpr int NL = NY * NZ;
  constexpr int D = ZL_STAGES;
  const int SL = n1 + 2 * ZL_PAD;
  // the neighbouring lines stream through a ring of D stages per warp: line t + D - 1 is issued (cp.async, 16 bytes
  // per lane and copy) while line t is processed, so D - 1 lines are in flight per warp
  auto issue = [&](int t, int slot) {
    const int oc = AZ0 + t / NY, ob = AY0 + t % NY;
    const double2* L = x + ((long)(k + oc - 2) * n1 + (j + ob - 2)) * n1;
    double2* st = stage + slot * SL + ZL_PAD;
    for (int e = lane; e < n1; e += 32) cp_async16(st + e, L + e);
  };
#pragma unroll
  for (int t = 0; t < D - 1; ++t) {
    if (t < NL) issue(t, (buf + t) % D);
    cp_commit_all();
  }
#pragma unroll 1
  for (int t = 0; t < NL; ++t) {
    const int oc = AZ0 + t / NY, ob = AY0 + t % NY;
    if (t + D - 1 < NL) issue(t + D - 1, (buf + t + D - 1) % D);
    cp_commit_all();
    asm volatile("cp.async.wait_group %0;\n" ::"n"(D - 1));
    __syncwarp();
    const double2* st = stage + ((buf + t) % D) * SL + ZL_PAD;
    if (has) {
    const double2* row = st + cb;
    const double* pa = Ta + (oc * 5 + ob) * 5;
    const double* pb = Tb + (oc * 5 + ob) * 5;
    double ta[5], tb[5];
#pragma unroll
    for (int oa = 0; oa < 5; ++oa) {
      ta[oa] = pa[REV ? 4 - oa : oa];
      tb[oa] = pb[REV ? 4 - oa : oa];
    }
    double2 v[7];
#pragma unroll
    for (int c = 0; c < 7; ++c) v[c] = row[REV ? -c : c];
    if (oc != 2 || ob != 2) {
#pragma unroll
      for (int oa = 0; oa < 5; ++oa) {
        acc[0] = cfma(ta[oa], v[oa], acc[0]);
        acc[1] = cfma(tb[oa], v[1 + oa], acc[1]);
        acc[2] = cfma(ta[oa], v[2 + oa], acc[2]);
      }
    } else {   // the line itself: node 0 (first colour) sees only old values; nodes 1, 2 take their fresh taps later
      xo[0] = v[2];
      xo[1] = v[3];
      xo[2] = v[4];
      v5old = v[5];
      v6old = v[6];
#pragma unroll
      for (int oa = 0; oa < 5; ++oa) acc[0] = cfma(ta[oa], v[oa], acc[0]);
      acc[1] = cfma(tb[0], v[1], acc[1]);
      acc[1] = cfma(tb[2], v[3], acc[1]);
      acc[1] = cfma(tb[3], v[4], acc[1]);
      acc[2] = cfma(ta[2], v[4], acc[2]);
    }
    }
    __syncwarp();   // every lane is done with this stage before a later issue reuses it
  }
  buf = (buf + NL) % D;
}

template <bool REV>
__device__ __forceinline__ void zline_update(const double* tabl, double2* x, const double2* __restrict__ b, int n1,
                                             int j, int k, int m, int ntr, int lane, double omega, double2* stage,
                                             int& buf) {
  const bool has = m < ntr;
  const int i0 = 3 * m, px = m & 1, py = j & 1, pz = k & 1;
  const int cb = REV ? i0 + 4 : i0 - 2;
  int gc[3];
  bool act[3];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    gc[n] = REV ? i0 + 2 - n : i0 + n;
    act[n] = has && gc[n] >= 1 && gc[n] <= n1 - 2;
  }
  const long line = ((long)k * n1 + j) * n1;
  const double* Ta = tabl + (px | (py << 1) | (pz << 2)) * (ClassTab<3>::NT + 1);
  const double* Tb = tabl + ((px ^ 1) | (py << 1) | (pz << 2)) * (ClassTab<3>::NT + 1);
  const double2 zero = make_double2(0.0, 0.0);
  double2 acc[3], xo[3] = {zero, zero, zero}, v5old = zero, v6old = zero;
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    const double2 bb = act[n] ? b[line + gc[n]] : zero;
    acc[n] = make_double2(-bb.x, -bb.y);
  }
  switch (py | (pz << 1)) {
    case 0: zline_accumulate<REV, 0, 0>(Ta, Tb, x, n1, j, k, cb, has, lane, stage, buf, acc, xo, v5old, v6old); break;
    case 1: zline_accumulate<REV, 1, 0>(Ta, Tb, x, n1, j, k, cb, has, lane, stage, buf, acc, xo, v5old, v6old); break;
    case 2: zline_accumulate<REV, 0, 1>(Ta, Tb, x, n1, j, k, cb, has, lane, stage, buf, acc, xo, v5old, v6old); break;
    default: zline_accumulate<REV, 1, 1>(Ta, Tb, x, n1, j, k, cb, has, lane, stage, buf, acc, xo, v5old, v6old); break;
  }
  const double wa = omega * Ta[ClassTab<3>::NT], wb = omega * Tb[ClassTab<3>::NT];
  const double* ra = Ta + 62 - 2;   // the centre row (oc = ob = 2) of the two stencils
  const double* rb = Tb + 62 - 2;
  const double tb1 = rb[REV ? 3 : 1], tb4 = rb[REV ? 0 : 4];
  const double ta0 = ra[REV ? 4 : 0], ta1 = ra[REV ? 3 : 1], ta3 = ra[REV ? 1 : 3], ta4 = ra[REV ? 0 : 4];
  // the triple that holds local columns 5 and 6: m + 1 (m - 1 in the mirrored frame of the reversed order)
  const int nbr = REV ? lane - 1 : lane + 1;
  const bool nbr_ok = has && nbr >= 0 && nbr < ntr;
  const int src = nbr_ok ? nbr : lane;
  // first x-colour
  double2 x0n = xo[0];
  if (act[0]) x0n = make_double2(xo[0].x - wa * acc[0].x, xo[0].y - wa * acc[0].y);
  // second x-colour: fresh taps = own first node and the first node of the neighbouring triple
  double2 v5 = make_double2(__shfl_sync(0xffffffffu, x0n.x, src), __shfl_sync(0xffffffffu, x0n.y, src));
  if (!nbr_ok) v5 = v5old;
  double2 x1n = xo[1];
  if (act[1]) {
    double2 a1 = cfma(tb1, x0n, acc[1]);
    a1 = cfma(tb4, v5, a1);
    x1n = make_double2(xo[1].x - wb * a1.x, xo[1].y - wb * a1.y);
  }
  // third x-colour
  double2 v6 = make_double2(__shfl_sync(0xffffffffu, x1n.x, src), __shfl_sync(0xffffffffu, x1n.y, src));
  if (!nbr_ok) v6 = v6old;
  if (act[0]) x[line + gc[0]] = x0n;
  if (act[1]) x[line + gc[1]] = x1n;
  if (act[2]) {
    double2 a2 = cfma(ta0, x0n, acc[2]);
    a2 = cfma(ta1, x1n, a2);
    a2 = cfma(ta3, v5, a2);
    a2 = cfma(ta4, v6, a2);
    x[line + gc[2]] = make_double2(xo[2].x - wa * a2.x, xo[2].y - wa * a2.y);
  }
}

// one sweep (all 27 colours in order, reversed if `reverse`) of a 3-D level with (n1 - 2) / 3 + 1 <= 32 triples per line
__device__ __noinline__ void q2_zline_sweep(const double* tabl, double2* x, const double2* __restrict__ b, int n1,
                                            bool reverse, double omega, int tid, int nth, double2* stage_all) {
  const int lane = tid & 31, warp = tid >> 5, nwarp = nth >> 5;
  const int ntr = (n1 - 2) / 3 + 1;
  const int SL = n1 + 2 * ZL_PAD;
  double2* stage = stage_all + warp * ZL_STAGES * SL;
  for (int e = lane; e < ZL_STAGES * SL; e += 32) stage[e] = make_double2(0.0, 0.0);   // pads stay zero
  __syncwarp();
  int buf = 0;
  const int nbz = (n1 + 2) / 3;
  for (int T = 0; T <= nbz + 3; ++T)
    for (int q = 0; q < 3; ++q) {
      const int cy = reverse ? 2 - q : q;
      const int j0 = cy ? cy : 3;
      const int nj = j0 > n1 - 2 ? 0 : (n1 - 2 - j0) / 3 + 1;
      for (int ln = warp; ln < 3 * nj; ln += nwarp) {
        const int pp = ln / nj, mj = ln - pp * nj;
        const int band = T - 2 * pp;
        if (band < 0 || band >= nbz) continue;
        const int k = 3 * band + (reverse ? 2 - pp : pp);
        if (k < 1 || k > n1 - 2) continue;
        const int j = j0 + 3 * mj;
        if (reverse) zline_update<true>(tabl, x, b, n1, j, k, lane, ntr, lane, omega, stage, buf);
        else zline_update<false>(tabl, x, b, n1, j, k, lane, ntr, lane, omega, stage, buf);
      }
      __syncthreads();
    }
}

// Returns true if the band-wavefront path also wrote the residual b - A x of the final iterate to rout.
template <int DIM, int ORD, bool CONV, bool W, bool TAB>
__device__ __forceinline__ bool cta_sweep(const Grid& g, const Coef& cf, const double* cv, double2* x,
                                          const double2* b, int sweeps, bool reverse, double omega, int tid, int nth,
                                          const double* tabl, double2* ring = nullptr,
                                          int waveH = 0, int flat_max = 0, double2* rout = nullptr,
                                          const double2* xcoarse = nullptr, int n1c = 0, bool zwave = false,
                                          unsigned long long* mbar = nullptr, unsigned long long* clk = nullptr,
                                          double2* zstage = nullptr) {
  constexpr int C1 = ORD == 2 ? 3 : 2;
  constexpr int NC = DIM == 2 ? C1 * C1 : C1 * C1 * C1;
  if constexpr (TAB && ORD == 2 && DIM == 2 && !W) {
    if (ring && waveH) {
      for (int sw = 0; sw < sweeps; ++sw) {
        double2* rr = (sw == sweeps - 1 && !reverse) ? rout : nullptr;
        const double2* xcs = sw == 0 ? xcoarse : nullptr;
        if constexpr (CONV) {
          if (waveH == 6)
            q2_wave_pass<6>(tabl, x, b, ring, g.n1, reverse, omega, tid, nth, cv, cf.c, rr, xcs, n1c, mbar);
          else
            q2_wave_pass<3>(tabl, x, b, ring, g.n1, reverse, omega, tid, nth, cv, cf.c, rr, xcs, n1c, mbar);
        } else {
          if (g.n1 == 513 && waveH == 3)
            q2_tri_pass<513, 3>(tabl, x, b, ring, 513, 3, reverse, omega, tid, nth, rr, xcs, n1c, mbar, clk);
          else if (g.n1 == 257 && waveH == 6)
            q2_tri_pass<257, 6>(tabl, x, b, ring, 257, 6, reverse, omega, tid, nth, rr, xcs, n1c, mbar, clk);
          else
            q2_tri_pass<0, 0>(tabl, x, b, ring, g.n1, waveH, reverse, omega, tid, nth, rr, xcs, n1c, mbar, clk);
        }
      }
      return rout != nullptr && sweeps > 0 && !reverse;
    }
  }
  if constexpr (DIM == 2 && ORD == 1 && !CONV && !W) {
    if (ring && waveH && tabl) {
      for (int sw = 0; sw < sweeps; ++sw) q1_pair_pass(tabl, x, b, ring, g.n1, waveH, reverse, omega, tid, nth, mbar);
      return false;
    }
  }
  if constexpr (DIM == 3 && ORD == 2 && TAB && !W && !CONV) {
    if (zwave && zstage != nullptr && (g.n1 - 2) / 3 + 1 <= 32) {
      for (int sw = 0; sw < sweeps; ++sw) q2_zline_sweep(tabl, x, b, g.n1, reverse, omega, tid, nth, zstage);
      return false;
    }
  }
  if constexpr (DIM == 3 && ORD == 2 && TAB && !W) {
    if (zwave) {
      // z-band wavefront (3-D Q2): planes are grouped in bands of 3 (one plane per z-colour class); at band step T
      // the bands T, T - 2, T - 4 update their plane of z-class 0, 1, 2 (colour order), and within a step the 9
      // xy-colours run in order.  Planes within the stencil reach (2) of each other are updated in exactly the
      // order of the 27 colour steps (as q2_wave_pass for rows), so the sweep is the same map -- but it moves
      // through the volume once, touching a window of ~21 planes, instead of streaming the whole level once per
      // colour (27 times per sweep).
      const int n1 = g.n1;
      const int nbz = (n1 + 2) / 3;
      for (int sw = 0; sw < sweeps; ++sw)
        for (int T = 0; T <= nbz + 3; ++T)
          for (int q = 0; q < 9; ++q) {
            const int xy = reverse ? 8 - q : q;
            const int cx = xy % 3, cy = xy / 3;
            const int ni = cx > n1 - 2 ? 0 : (n1 - 2 - (cx ? cx : 3)) / 3 + 1;   // i = cx + 3m in [1, n1 - 2]
            const int i0 = cx ? cx : 3;
            const int j0 = cy ? cy : 3;
            const int nj = j0 > n1 - 2 ? 0 : (n1 - 2 - j0) / 3 + 1;
            // rows of one plane ordered by parity (uniform taps per warp): even-m rows first, then odd-m rows
            const int per_plane = ni * nj;
            const int total = 3 * per_plane;
            const int nje = (nj + 1) / 2;
            for (int t = tid; t < total; t += nth) {
              const int pp = t / per_plane, rem = t - pp * per_plane;
              const int band = T - 2 * pp;
              if (band < 0 || band >= nbz) continue;
              const int cz = reverse ? 2 - pp : pp;
              const int k = 3 * band + cz;
              if (k < 1 || k > n1 - 2) continue;
              const int rr = rem / ni, mi = rem - rr * ni;
              const int mj = rr < nje ? 2 * rr : 2 * (rr - nje) + 1;
              int c[DIM] = {i0 + 3 * mi, j0 + 3 * mj, k};
              const int idx = (k * n1 + c[1]) * n1 + c[0];
              if constexpr (CONV) {
                double2 D;
                const double2 Ax = class_eval_conv<DIM>(reinterpret_cast<const double2*>(tabl), cv, cf.c, x, c, idx,
                                                        n1, D);
                x[idx] = cadd(x[idx], cscale(omega, cdiv(csub(b[idx], Ax), D)));
              } else {
                double invD;
                const double2 Ax = class_eval<DIM>(tabl, x, c, n1, invD);
                x[idx] = cadd(x[idx], cscale(omega * invD, csub(b[idx], Ax)));
              }
            }
            __syncthreads();
          }
      return false;
    }
  }
  for (int sw = 0; sw < sweeps; ++sw)
    for (int cc = 0; cc < NC; ++cc) {
      const int colour = reverse ? NC - 1 - cc : cc;
      int res[DIM];
      int col = colour;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        res[a] = col % C1;
        col /= C1;
      }
      auto upd = [&](const int* c, int idx) {
        if constexpr (TAB && CONV) {
          double2 D;
          const double2 Ax = class_eval_conv<DIM>(reinterpret_cast<const double2*>(tabl), cv, cf.c, x, c, idx, g.n1, D);
          x[idx] = cadd(x[idx], cscale(omega, cdiv(csub(b[idx], Ax), D)));
        } else if constexpr (TAB) {
          double invD;
          const double2 Ax = class_eval<DIM>(tabl, x, c, g.n1, invD);
          x[idx] = cadd(x[idx], cscale(omega * invD, csub(b[idx], Ax)));
        } else {
          if constexpr (ORD == 1 && DIM == 2 && !CONV) {
            if (tabl) {
              double invD;
              const double2 Ax = class_eval_q1(tabl, x, c[0], c[1], g.n1, invD);
              x[idx] = cadd(x[idx], cscale(omega * invD, csub(b[idx], Ax)));
              return;
            }
          }
          sor_node<DIM, ORD, CONV>(g, cf, cv, x, b, c, idx, omega);
        }
      };
      if (ORD == 2 && TAB && CONV && DIM == 2 && g.n1 <= flat_max) {
        int st[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) st[a] = 3;
        cta_visit<DIM>(g.n1, res, st, 1, g.n1 - 2, tid, nth, [&](const int* c, int idx) {
          double2 D;
          const double2 Ax = class_eval_conv_flat2(reinterpret_cast<const double2*>(tabl), cv, cf.c, x, c[0], c[1],
                                                   idx, g.n1, D);
          const double2 xo = x[idx], bb = b[idx];
          x[idx] = cadd(xo, cscale(omega, cdiv(csub(bb, Ax), D)));
        });
      } else if (ORD == 2 && TAB && !CONV && DIM == 2 && g.n1 <= flat_max) {
        // small level: one visit of the whole colour (stride 3 in x and y), branch-free evaluation
        int st[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) st[a] = 3;
        cta_visit<DIM>(g.n1, res, st, 1, g.n1 - 2, tid, nth, [&](const int* c, int idx) {
          double invD;
          const double2 Ax = class_eval_flat2(tabl, x, c[0], c[1], g.n1, invD);
          const double2 xo = x[idx], bb = b[idx];
          x[idx] = cadd(xo, cscale(omega * invD, csub(bb, Ax)));
        });
      } else if (ORD == 2) {
        // colour residue r: x nodes r + 3m (coalesced); y/z in parity classes r + 3p + 6m so that
        // the row taps are warp-uniform
        for (int cls = 0; cls < (1 << (DIM - 1)); ++cls) {
          int s0[DIM], st[DIM];
          s0[0] = res[0];
          st[0] = 3;
#pragma unroll
          for (int a = 1; a < DIM; ++a) {
            s0[a] = res[a] + 3 * ((cls >> (a - 1)) & 1);
            st[a] = 6;
          }
          cta_visit<DIM>(g.n1, s0, st, 1, g.n1 - 2, tid, nth, upd);
        }
      } else {
        int st[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) st[a] = 2;
        cta_visit<DIM>(g.n1, res, st, 0, g.n1 - 1, tid, nth, [&](const int* c, int idx) {
          if (idx != 0) upd(c, idx);
        });
      }
      gsync<W>();
    }
  return false;
}

// level storage of one problem inside the CTA-resident MG
struct MGLevels {
  const MGArgs& a;
  double2* smem;
  int p;
  double* ctab;   // class stencils per smoothing level (ORD 2, real operators) or nullptr
  __device__ double2* X(int l) const {
    if (l == 0) return a.x0.p + voff(a.x0, p, a.g[0].n);
    return l >= a.lsm ? smem + a.sm_x[l] : a.xw[l] + (long)p * a.g[l].n;
  }
  __device__ double2* B(int l) const {
    if (l == 0) return a.b0.p + voff(a.b0, p, a.g[0].n);
    return l >= a.lsm ? smem + a.sm_b[l] : a.bw[l] + (long)p * a.g[l].n;
  }
  __device__ double2* R(int l) const { return a.rw[l] + (long)p * a.g[l].n; }
  __device__ const double* CV(int l) const { return a.op.conv_sel == 1 ? a.g[l].conv : a.g[l].convT; }
  __device__ double2* ZSTAGE() const { return a.zstage_off >= 0 ? smem + a.zstage_off : nullptr; }
  __device__ unsigned long long* MBAR() const {
    return a.wave_h ? reinterpret_cast<unsigned long long*>(smem + a.mbar_off) : nullptr;
  }
};

// down-leg of level l: (x_l = 0 for l > 0), pre-smoothing, residual, restriction to b_{l+1}
template <int DIM, int ORD, bool CONV, bool W, bool TAB>
__device__ void mg_down(const MGLevels& S, const Coef& cf, int l, int tid, int nth) {
  constexpr int R = ORD == 2 ? 3 : 1;
  constexpr int WR = 2 * R + 1;
  const MGArgs& a = S.a;
  const Grid g = a.g[l];
  double2* xl = S.X(l);
  const double2* bl = S.B(l);
  if (l > 0) {
    for (int i = tid; i < (int)g.n; i += nth) xl[i] = make_double2(0.0, 0.0);
    gsync<W>();
  }
  const double* tabl = S.ctab ? S.ctab + l * (ORD == 1 ? Q1TAB
                                                       : (CONV ? 2 * ClassTab<DIM>::NCL * ClassTab<DIM>::NT
                                                               : ClassTab<DIM>::PER_LEVEL)) : nullptr;
  // profiling (AAO_MG_CLOCK): split of the level-0 down-leg into sweeps / residual / restriction
  const bool pclk = DIM == 2 && a.clk != nullptr && blockIdx.x == a.clk_block && tid == 0 && l == 0;
  unsigned long long pt = pclk ? clock64() : 0ull;
  auto pmark = [&](int slot) {
    if (pclk) {
      const unsigned long long t1 = clock64();
      a.clk[slot] += t1 - pt;
      pt = t1;
    }
  };
  const bool wv = a.wave_hl[l] > 0;
  double2* rl = S.R(l);
  const bool fused = cta_sweep<DIM, ORD, CONV, W, TAB>(g, cf, S.CV(l), xl, bl, a.pre, false, a.omega, tid, nth, tabl,
                                                       wv ? S.smem + a.ring_off : nullptr, a.wave_hl[l],
                                                       a.flat_max, wv ? rl : nullptr, nullptr, 0,
                                                       DIM == 3 && l < a.lsm && g.n1 >= a.zwave_min, S.MBAR(),
                                                       pclk ? a.clk : nullptr, S.ZSTAGE());
  pmark(2 * MG_MAXL - 2);
  const double* cvl = S.CV(l);
  if (fused) {
    // residual written by the last wavefront sweep
  } else if (TAB && CONV && ORD == 2 && DIM == 2 && g.n1 <= a.flat_max) {
    int s1[DIM], st1[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      s1[d] = 1;
      st1[d] = 1;
    }
    cta_visit<DIM>(g.n1, s1, st1, 1, g.n1 - 2, tid, nth, [&](const int* c, int i) {
      double2 D;
      const double2 Ax = class_eval_conv_flat2(reinterpret_cast<const double2*>(tabl), cvl, cf.c, xl, c[0], c[1], i,
                                               g.n1, D);
      rl[i] = csub(bl[i], Ax);
    });
  } else if (TAB && !CONV && ORD == 2 && DIM == 2 && g.n1 <= a.flat_max) {
    int s1[DIM], st1[DIM];
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      s1[d] = 1;
      st1[d] = 1;
    }
    cta_visit<DIM>(g.n1, s1, st1, 1, g.n1 - 2, tid, nth, [&](const int* c, int i) {
      double invD;
      const double2 Ax = class_eval_flat2(tabl, xl, c[0], c[1], g.n1, invD);
      rl[i] = csub(bl[i], Ax);
    });
  } else
  cta_all_unknowns<DIM, ORD>(g.n1, tid, nth, [&](const int* c, int i) {
    double2 Ax;
    if constexpr (TAB && CONV) {
      double2 D;
      Ax = class_eval_conv<DIM>(reinterpret_cast<const double2*>(tabl), cvl, cf.c, xl, c, i, g.n1, D);
    } else if constexpr (TAB) {
      double invD;
      Ax = class_eval<DIM>(tabl, xl, c, g.n1, invD);
    } else if (CONV) {
      double2 D;
      apply_op_conv<DIM, ORD>(g, cf, cvl, xl, c, i, Ax, D);
    } else if (ORD == 1 && DIM == 2 && tabl != nullptr) {
      double invD;
      Ax = class_eval_q1(tabl, xl, c[0], c[1], g.n1, invD);
    } else {
      double D;
      apply_op_real<DIM, ORD>(g, cf.a.x, cf.b.x, xl, c, i, Ax, D);
    }
    rl[i] = csub(bl[i], Ax);
  });
  gsync<W>();
  pmark(2 * MG_MAXL - 3);
  const Grid gc = a.g[l + 1];
  const Transfer t = a.t[l];
  const int o7 = ORD == 2 ? 0 : 2;
  double2* bn = S.B(l + 1);
  const int n1 = g.n1;
  // b_{l+1}[I] = (P^T r_l)[I]; two coarse nodes per thread and round so that their gathers overlap
  auto restrict_node = [&](int I) -> double2 {
    int c[DIM];
    coords<DIM>(I, gc.n1, c);
    if (masked<DIM, ORD>(c, I, gc.n1)) return make_double2(0.0, 0.0);
    double w[DIM][WR];
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      if constexpr (ORD == 2) {
        q2_rrow(c[d], w[d]);
      } else {
#pragma unroll
        for (int o = 0; o < WR; ++o) w[d][o] = __ldg(t.tR + c[d] * 7 + o7 + o);
      }
    }
    double2 acc = make_double2(0.0, 0.0);
    if constexpr (DIM == 2) {
#pragma unroll
      for (int ob = 0; ob < WR; ++ob) {
        if (w[1][ob] == 0.0) continue;
        const double2* rrow = rl + (2 * c[1] + ob - R) * n1 + 2 * c[0] - R;
#pragma unroll
        for (int oa = 0; oa < WR; ++oa)
          if (w[0][oa] != 0.0) acc = cfma(w[1][ob] * w[0][oa], rrow[oa], acc);
      }
    } else {
      for (int oc = 0; oc < WR; ++oc) {
        if (w[2][oc] == 0.0) continue;
#pragma unroll
        for (int ob = 0; ob < WR; ++ob) {
          if (w[1][ob] == 0.0) continue;
          const double2* rrow = rl + ((2 * c[2] + oc - R) * n1 + 2 * c[1] + ob - R) * n1 + 2 * c[0] - R;
#pragma unroll
          for (int oa = 0; oa < WR; ++oa)
            if (w[0][oa] != 0.0) acc = cfma(w[2][oc] * w[1][ob] * w[0][oa], rrow[oa], acc);
        }
      }
    }
    return acc;
  };
  const int ncn = (int)gc.n;
  for (int I = tid; I < ncn; I += 2 * nth) {
    const int I2 = I + nth;
    const double2 v1 = restrict_node(I);
    const double2 v2 = I2 < ncn ? restrict_node(I2) : make_double2(0.0, 0.0);
    bn[I] = v1;
    if (I2 < ncn) bn[I2] = v2;
  }
  gsync<W>();
  pmark(2 * MG_MAXL - 4);
}

// coarsest level: dense inverse (masked entries of the coarsest iterate read as 0 in the prolongation)
template <int DIM, int ORD, bool W>
__device__ void mg_coarse(const MGLevels& S, int tid, int nth) {
  const MGArgs& a = S.a;
  const int L = a.nlev;
  double2* xL = S.X(L - 1);
  const double2* bL = S.B(L - 1);
  for (int i = tid; i < (int)a.g[L - 1].n; i += nth) xL[i] = make_double2(0.0, 0.0);
  gsync<W>();
  const double2* A = a.inv + (long)(S.p / a.inv_pg) * a.nu * a.nu;
  for (int i = tid; i < a.nu; i += nth) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < a.nu; ++j) acc = cadd(acc, cmul(A[(long)i * a.nu + j], bL[a.unk[j]]));
    xL[a.unk[i]] = acc;
  }
  gsync<W>();
}

// up-leg of level l: prolongate x_{l+1} and correct, post-smoothing
template <int DIM, int ORD, bool CONV, bool W, bool TAB>
__device__ void mg_up(const MGLevels& S, const Coef& cf, int l, int tid, int nth) {
  constexpr int NW = ORD == 2 ? 3 : 2;
  const MGArgs& a = S.a;
  const Grid g = a.g[l];
  const Grid gc = a.g[l + 1];
  const Transfer t = a.t[l];
  double2* xl = S.X(l);
  const double2* xc = S.X(l + 1);
  const bool wv = a.wave_hl[l] > 0;
  const bool fuse_prolong = TAB && ORD == 2 && DIM == 2 && !W && wv && a.post > 0 && a.fuse_prolong;
  if (!fuse_prolong) {
  cta_all_unknowns<DIM, ORD>(g.n1, tid, nth, [&](const int* c, int i) {
    int base[DIM];
    double w[DIM][NW];
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      if constexpr (ORD == 2) {
        base[d] = q2_prow(c[d], w[d]);
      } else {
        base[d] = (int)__ldg(t.tP + c[d] * 4);
#pragma unroll
        for (int o = 0; o < NW; ++o) w[d][o] = __ldg(t.tP + c[d] * 4 + 1 + o);
      }
    }
    const int n1 = gc.n1;
    double2 acc = make_double2(0.0, 0.0);
    if constexpr (DIM == 2) {
#pragma unroll
      for (int ob = 0; ob < NW; ++ob)
#pragma unroll
        for (int oa = 0; oa < NW; ++oa) {
          const double ww = w[1][ob] * w[0][oa];
          if (ww != 0.0) acc = cfma(ww, xc[(base[1] + ob) * n1 + base[0] + oa], acc);
        }
    } else {
#pragma unroll
      for (int oc = 0; oc < NW; ++oc)
#pragma unroll
        for (int ob = 0; ob < NW; ++ob)
#pragma unroll
          for (int oa = 0; oa < NW; ++oa) {
            const double ww = w[2][oc] * w[1][ob] * w[0][oa];
            if (ww != 0.0) acc = cfma(ww, xc[((base[2] + oc) * n1 + base[1] + ob) * n1 + base[0] + oa], acc);
          }
    }
    xl[i] = cadd(xl[i], acc);
  });
  gsync<W>();
  }
  const double* tabl = S.ctab ? S.ctab + l * (ORD == 1 ? Q1TAB
                                                   : (CONV ? 2 * ClassTab<DIM>::NCL * ClassTab<DIM>::NT
                                                           : ClassTab<DIM>::PER_LEVEL)) : nullptr;
  cta_sweep<DIM, ORD, CONV, W, TAB>(g, cf, S.CV(l), xl, S.B(l), a.post, true, a.omega, tid, nth, tabl,
                                    wv ? S.smem + a.ring_off : nullptr, a.wave_hl[l], a.flat_max, nullptr,
                                    fuse_prolong ? xc : nullptr, gc.n1, DIM == 3 && l < a.lsm && g.n1 >= a.zwave_min,
                                    S.MBAR(), nullptr, S.ZSTAGE());
}

// threads per CTA of the CTA-resident MG; 3-D measured: 512 (spills at 128 registers) 205 ms vs 256 (no
// spills, half the warps) 224 ms on c5
#ifndef MG_THREADS_3D
#define MG_THREADS_3D 512
#endif
template <int DIM, bool TAB, bool CONV, int ORD = 2>
constexpr int mg_threads() {
  // 2-D real class stencils: one thread per triple of the band-wavefront sweeps (3 x 171 triples on a 513^2 level)
  return DIM == 3 ? MG_THREADS_3D
                  : (TAB ? (CONV ? MG_THREADS_TAB : MG_TRI_THREADS) : (ORD == 1 ? MG_THREADS_Q1 : MG_THREADS));
}
template <int DIM, int ORD>
constexpr int mg_minb() {
  return DIM == 2 && ORD == 1 ? MG_MINB_Q1 : 1;
}

template <int DIM, int ORD, bool CONV, bool TAB>
__global__ void __launch_bounds__(mg_threads<DIM, TAB, CONV, ORD>(), mg_minb<DIM, ORD>()) k_mg_cta(MGArgs a) {
  extern __shared__ double2 smem[];
  const int p = blockIdx.x;
  const int L = a.nlev;
  const Coef cf = a.op.coef[p / a.op.per_group];
  const int tid = threadIdx.x, nth = blockDim.x;
  // class stencils of every smoothing level (real Q2 operators) at the start of dynamic smem
  double* ctab = nullptr;
  if constexpr (ORD == 1 && DIM == 2 && !CONV) {
    if (a.use_ctab == 2) {   // Q1 position-class stencils of every smoothing level
      ctab = reinterpret_cast<double*>(smem);
      for (int l = 0; l < L - 1; ++l) {
        build_class_tab_q1(a.g[l], cf.a.x, cf.b.x, ctab + l * Q1TAB, tid, nth);
        __syncthreads();
      }
    }
  }
  if constexpr (ORD == 1 && DIM == 2 && !CONV) {
    if (a.wave_h) {   // pair-form wavefront sweeps: zeroed ring with guards, band-slot mbarriers
      for (long e = a.ring_off - MG_RING_GUARD + tid; e < a.mbar_off; e += nth) smem[e] = make_double2(0.0, 0.0);
      if (tid == 0) {
        unsigned long long* mb = reinterpret_cast<unsigned long long*>(smem + a.mbar_off);
        for (int sl = 0; sl < MG_TRI_SLOTS; ++sl) mbar_init(mb + sl, 1);
        *reinterpret_cast<unsigned*>(mb + MG_TRI_SLOTS) = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();
    }
  }
  if (TAB) {
    ctab = reinterpret_cast<double*>(smem);
    for (int l = 0; l < L - 1; ++l) {
      if (CONV)
        build_class_tab_c<DIM>(a.g[l], cf.a, cf.b,
                               reinterpret_cast<double2*>(ctab) + l * ClassTab<DIM>::NCL * ClassTab<DIM>::NT, tid, nth);
      else
        build_class_tab<DIM>(a.g[l], cf.a.x, cf.b.x, ctab + l * ClassTab<DIM>::PER_LEVEL, tid, nth);
    }
    __syncthreads();
  }
  if constexpr (TAB && ORD == 2 && DIM == 2) {
    if (a.wave_h) {
      // the ring and its guard columns start as zeros: the triple-form sweeps read up to three entries beyond a row
      // (they only meet zero coefficients or inactive nodes, but must be finite)
      for (long e = a.ring_off - MG_RING_GUARD + tid; e < a.mbar_off; e += nth) smem[e] = make_double2(0.0, 0.0);
      if (tid == 0) {   // band-ring mbarriers (8 slots) and their phase word, after the ring
        unsigned long long* mb = reinterpret_cast<unsigned long long*>(smem + a.mbar_off);
        for (int sl = 0; sl < MG_TRI_SLOTS; ++sl) mbar_init(mb + sl, 1);
        *reinterpret_cast<unsigned*>(mb + MG_TRI_SLOTS) = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
    }
    __syncthreads();
  }
  const MGLevels S{a, smem, p, ctab};
  const int lw = a.lwarp;   // levels >= lw run inside warp 0
  double2* x0 = S.X(0);
  for (int i = tid; i < (int)a.g[0].n; i += nth) x0[i] = make_double2(0.0, 0.0);
  __syncthreads();
  const bool clk = a.clk != nullptr && blockIdx.x == a.clk_block && tid == 0;
  unsigned long long t0 = clk ? clock64() : 0ull;
  auto mark = [&](int slot) {
    if (clk) {
      const unsigned long long t1 = clock64();
      a.clk[slot] += t1 - t0;
      t0 = t1;
    }
  };
  for (int cyc = 0; cyc < a.cycles; ++cyc) {
    for (int l = 0; l < lw && l < L - 1; ++l) {
      mg_down<DIM, ORD, CONV, false, TAB>(S, cf, l, tid, nth);
      mark(2 * l);
    }
    if (lw < L) {
      if (tid < 32) {
        for (int l = lw; l < L - 1; ++l) mg_down<DIM, ORD, CONV, true, TAB>(S, cf, l, tid, 32);
        mg_coarse<DIM, ORD, true>(S, tid, 32);
        for (int l = L - 2; l >= lw; --l) mg_up<DIM, ORD, CONV, true, TAB>(S, cf, l, tid, 32);
      }
      __syncthreads();
      mark(2 * MG_MAXL - 1);
    } else {
      mg_coarse<DIM, ORD, false>(S, tid, nth);
      mark(2 * MG_MAXL - 1);
    }
    for (int l = (lw < L ? lw : L - 1) - 1; l >= 0; --l) {
      mg_up<DIM, ORD, CONV, false, TAB>(S, cf, l, tid, nth);
      mark(2 * l + 1);
    }
  }
}

// Chebyshev semi-iteration on a mass matrix, one CTA per problem
template <int DIM, int ORD>
__global__ void __launch_bounds__(cheb_threads<DIM, ORD>(), cheb_minb<DIM, ORD>()) k_cheb_cta(Grid g, View bv, View xv, double2* rw, double2* d0w, double2* d1w,
                                                   double theta, double sigma, double delta, int iters, double scale) {
  const int p = blockIdx.x;
  const double2* b = bv.p + voff(bv, p, g.n);
  double2* x = xv.p + voff(xv, p, g.n);
  double2* r = rw + (long)p * g.n;
  double2* d0 = d0w + (long)p * g.n;
  double2* d1 = d1w + (long)p * g.n;
  const double2 z = make_double2(0.0, 0.0);
  // Q2 mass: class stencils (a = 1, b = 0) when the level has an interior vertex row (n1 >= 9)
  __shared__ double mtab[ClassTab<DIM>::PER_LEVEL];
  static_assert(ClassTab<DIM>::PER_LEVEL >= Q1TAB, "the Q1 mass table shares mtab");
  const bool tab = ORD == 2 && g.n1 >= 9;
  const bool tabq1 = ORD == 1 && DIM == 2 && g.n1 >= 3;
  if (tab) {
    build_class_tab<DIM>(g, 1.0, 0.0, mtab, threadIdx.x, blockDim.x);
    __syncthreads();
  } else if (tabq1) {
    build_class_tab_q1(g, 1.0, 0.0, mtab, threadIdx.x, blockDim.x);
    __syncthreads();
  }
  for (int i = threadIdx.x; i < (int)g.n; i += blockDim.x) {
    int c[DIM];
    coords<DIM>(i, g.n1, c);
    x[i] = z;
    d1[i] = z;
    if (masked<DIM, ORD>(c, i, g.n1)) {
      r[i] = z;
      d0[i] = z;
    } else {
      const double2 bb = b[i];
      r[i] = bb;
      d0[i] = cscale(1.0 / theta, cscale(1.0 / mass_diag<DIM, ORD>(g, c), bb));
    }
  }
  __syncthreads();
  double rho = 1.0 / sigma;
  for (int k = 0; k < iters - 1; ++k) {
    const double rho1 = 1.0 / (2.0 * sigma - rho);
    const double c1 = rho1 * rho, c2 = 2.0 * rho1 / delta;
    const double2* dold = d0;
    double2* dnew = d1;
    cta_all_unknowns<DIM, ORD>(g.n1, threadIdx.x, blockDim.x, [&](const int* c, int i) {
      double2 Mx;
      double invM;
      if (ORD == 2 && tab) {
        Mx = class_eval<DIM>(mtab, dold, c, g.n1, invM);
      } else if (DIM == 2 && tabq1) {
        Mx = class_eval_q1(mtab, dold, c[0], c[1], g.n1, invM);
      } else {
        double2 Kx, Cx;
        double dM, dK, dC;
        apply_MKC<DIM, ORD, false>(g, nullptr, dold, c, i, Mx, Kx, Cx, dM, dK, dC);
        invM = 1.0 / dM;
      }
      const double2 d = dold[i];
      x[i] = cadd(x[i], d);
      const double2 rr = csub(r[i], Mx);
      r[i] = rr;
      dnew[i] = cadd(cscale(c1, d), cscale(c2, cscale(invM, rr)));
    });
    __syncthreads();
    double2* tmp = d0;
    d0 = d1;
    d1 = tmp;
    rho = rho1;
  }
  for (int i = threadIdx.x; i < (int)g.n; i += blockDim.x) x[i] = cscale(scale, cadd(x[i], d0[i]));
}

// ---------------------------------------------------------------- launchers
static inline dim3 grid1(long n, int nprob, int bs) { return dim3((unsigned)((n + bs - 1) / bs), nprob); }
constexpr int BS = 128;

template <int DIM, int ORD>
static void gs_t(const Grid& g, const OpSel& op, View x, View b, int nprob, int colour, double omega,
                 cudaStream_t s) {
  constexpr int C1 = ORD == 2 ? 3 : 2;
  long total = 1;
  int cc = colour;
  for (int a = 0; a < DIM; ++a) {
    int r = cc % C1;
    cc /= C1;
    total *= (g.n1 - r + C1 - 1) / C1;
  }
  k_gs<DIM, ORD><<<grid1(total, nprob, BS), BS, 0, s>>>(g, op, x, b, colour, omega);
}

#define SWITCH_DO(g, FN, ...)                         \
  switch ((g).dim * 10 + (g).order) {                 \
    case 22: FN<2, 2>(__VA_ARGS__); break;            \
    case 21: FN<2, 1>(__VA_ARGS__); break;            \
    case 32: FN<3, 2>(__VA_ARGS__); break;            \
    case 31: FN<3, 1>(__VA_ARGS__); break;            \
  }

void launch_gs(const Grid& g, const OpSel& op, View x, View b, int nprob, int colour, double omega,
               cudaStream_t s) {
  SWITCH_DO(g, gs_t, g, op, x, b, nprob, colour, omega, s);
}

template <int DIM, int ORD>
static void res_t(const Grid& g, const OpSel& op, View x, View b, View r, int nprob, cudaStream_t s) {
  k_residual<DIM, ORD><<<grid1(g.n, nprob, BS), BS, 0, s>>>(g, op, x, b, r);
}
void launch_residual(const Grid& g, const OpSel& op, View x, View b, View r, int nprob, cudaStream_t s) {
  SWITCH_DO(g, res_t, g, op, x, b, r, nprob, s);
}

template <int DIM, int ORD>
static void restr_t(const Grid& gf, const Grid& gc, const Transfer& t, View rf, View bc, int nprob,
                    cudaStream_t s) {
  k_restrict<DIM, ORD><<<grid1(gc.n, nprob, BS), BS, 0, s>>>(gf, gc, t, rf, bc);
}
void launch_restrict(const Grid& gf, const Grid& gc, const Transfer& t, View rf, View bc, int nprob,
                     cudaStream_t s) {
  SWITCH_DO(gf, restr_t, gf, gc, t, rf, bc, nprob, s);
}

template <int DIM, int ORD>
static void prol_t(const Grid& gf, const Grid& gc, const Transfer& t, View xc, View xf, int nprob,
                   cudaStream_t s) {
  k_prolong<DIM, ORD><<<grid1(gf.n, nprob, BS), BS, 0, s>>>(gf, gc, t, xc, xf);
}
void launch_prolong(const Grid& gf, const Grid& gc, const Transfer& t, View xc, View xf, int nprob,
                    cudaStream_t s) {
  SWITCH_DO(gf, prol_t, gf, gc, t, xc, xf, nprob, s);
}

void launch_coarse(const Grid& gc, const double2* inv, int inv_per_group, const int* unk, int nu, View b,
                   View x, int nprob, cudaStream_t s) {
  k_coarse<<<nprob, 32, nu * sizeof(double2), s>>>(gc.n, inv, inv_per_group, unk, nu, b, x);
}

void launch_zero(View x, long n, int nprob, cudaStream_t s) {
  k_zero<<<grid1(n, nprob, 256), 256, 0, s>>>(x, n);
}

template <int DIM, int ORD>
static void chi_t(const Grid& g, View b, View x, View r, View d, double it, int nprob, cudaStream_t s) {
  k_cheb_init<DIM, ORD><<<grid1(g.n, nprob, BS), BS, 0, s>>>(g, b, x, r, d, it);
}
void launch_cheb_init(const Grid& g, View b, View x, View r, View d, double inv_theta, int nprob,
                      cudaStream_t s) {
  SWITCH_DO(g, chi_t, g, b, x, r, d, inv_theta, nprob, s);
}
template <int DIM, int ORD>
static void chs_t(const Grid& g, View x, View r, View dold, View dnew, double c1, double c2, int nprob,
                  cudaStream_t s) {
  k_cheb_step<DIM, ORD><<<grid1(g.n, nprob, BS), BS, 0, s>>>(g, x, r, dold, dnew, c1, c2);
}
void launch_cheb_step(const Grid& g, View x, View r, View dold, View dnew, double c1, double c2, int nprob,
                      cudaStream_t s) {
  SWITCH_DO(g, chs_t, g, x, r, dold, dnew, c1, c2, nprob, s);
}
template <int DIM, int ORD>
static void chf_t(const Grid& g, View x, View d, double scale, int nprob, cudaStream_t s) {
  k_cheb_final<DIM, ORD><<<grid1(g.n, nprob, 256), 256, 0, s>>>(g, x, d, scale);
}
void launch_cheb_final(const Grid& g, View x, View d, double scale, int nprob, cudaStream_t s) {
  SWITCH_DO(g, chf_t, g, x, d, scale, nprob, s);
}

template <int DIM, int ORD>
static void lc_t(const Grid& g, View out, double cb, View b, const OpSel& A1, View x1, const OpSel& A2, View x2,
                 int nprob, cudaStream_t s) {
  k_lincomb<DIM, ORD><<<grid1(g.n, nprob, BS), BS, 0, s>>>(g, out, cb, b, A1, x1, A2, x2, x2.p != nullptr);
}
void launch_lincomb(const Grid& g, View out, double cb, View b, const OpSel& A1, View x1, const OpSel& A2,
                    View x2, int nprob, cudaStream_t s) {
  SWITCH_DO(g, lc_t, g, out, cb, b, A1, x1, A2, x2, nprob, s);
}

template <int DIM, int ORD>
static void ax_t(const Grid& g, View y, double2 a, View x, double2 bc, int nprob, cudaStream_t s) {
  k_axpby<DIM, ORD><<<grid1(g.n, nprob, 256), 256, 0, s>>>(g, y, a, x, bc);
}
void launch_axpby(const Grid& g, View y, double2 a, View x, double2 bcoef, int nprob, cudaStream_t s) {
  SWITCH_DO(g, ax_t, g, y, a, x, bcoef, nprob, s);
}

template <int DIM, int ORD>
static void mgcta_t(const MGArgs& a, int nprob, size_t smem, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_mg_cta<DIM, ORD, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, MG_SMEM_MAX);
    cudaFuncSetAttribute(k_mg_cta<DIM, ORD, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, MG_SMEM_MAX);
    if (ORD == 2) {
      cudaFuncSetAttribute(k_mg_cta<DIM, ORD, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, MG_SMEM_MAX);
      cudaFuncSetAttribute(k_mg_cta<DIM, ORD, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, MG_SMEM_MAX);
    }
    attr = true;
  }
  if (a.op.conv_sel != 0 && ORD == 2 && a.use_ctab)
    k_mg_cta<DIM, ORD, true, (ORD == 2)><<<nprob, mg_threads<DIM, true, true>(), smem, s>>>(a);
  else if (a.op.conv_sel != 0)
    k_mg_cta<DIM, ORD, true, false><<<nprob, mg_threads<DIM, false, true, ORD>(), smem, s>>>(a);
  else if (ORD == 2 && a.use_ctab)
    k_mg_cta<DIM, ORD, false, (ORD == 2)><<<nprob, mg_threads<DIM, true, false>(), smem, s>>>(a);
  else
    k_mg_cta<DIM, ORD, false, false><<<nprob, mg_threads<DIM, false, false, ORD>(), smem, s>>>(a);
}
void launch_mg_cta(const MGArgs& a, int nprob, size_t smem, cudaStream_t s) {
  SWITCH_DO(a.g[0], mgcta_t, a, nprob, smem, s);
}

template <int DIM, int ORD>
static void chcta_t(const Grid& g, View b, View x, double2* r, double2* d0, double2* d1, double theta, double sigma,
                    double delta, int iters, double scale, int nprob, cudaStream_t s) {
  k_cheb_cta<DIM, ORD><<<nprob, cheb_threads<DIM, ORD>(), 0, s>>>(g, b, x, r, d0, d1, theta, sigma, delta, iters,
                                                                  scale);
}
void launch_cheb_cta(const Grid& g, View b, View x, double2* r, double2* d0, double2* d1, double theta, double sigma,
                     double delta, int iters, double scale, int nprob, cudaStream_t s) {
  SWITCH_DO(g, chcta_t, g, b, x, r, d0, d1, theta, sigma, delta, iters, scale, nprob, s);
}

void launch_Bv(const Grid& g2, const Grid& g1, const double* tPm, const double* tGm, View v, View bp, View out,
               double sb, double sB, int nprob, cudaStream_t s) {
  if (g1.dim == 2)
    k_Bv<2><<<grid1(g1.n, nprob, BS), BS, 0, s>>>(g2, g1, tPm, tGm, v, bp, out, sb, sB);
  else
    k_Bv<3><<<grid1(g1.n, nprob, BS), BS, 0, s>>>(g2, g1, tPm, tGm, v, bp, out, sb, sB);
}

}  // namespace aao
