// Time-axis transforms fused with the T-transforms, and the all-at-once KKT matvec.
//
//  k_fft_fwd : r (paper order, real) -> T_l^{-1} F r  in the frequency layout
//              (steps A3; Oseen: no T transform)
//  k_fft_inv : T_r^{-1} x  -> F^{-1} (...) (paper order, real)  (step A8)
//  k_kkt_*   : y = A x of eq. (FinalA) (step A2)
//
// Layout choice: the Krylov vectors keep the paper's
// order [half][t][field][node] -- SPACE is contiguous.  A CTA owns a tile of TD
// consecutive spatial columns for all n_b time rows of both halves: every global
// load/store is a coalesced row segment, the time DFT runs along the tile in
// shared memory, and the frequency layout [k][half][field][node] (space
// contiguous again) falls out of the same tile.  No separate transpose pass.
#include <cmath>
#include <cstdlib>

#include "aao_internal.h"

namespace aao {

namespace {

struct InvSrc {
  const double2* v1;   // slot 1 (x1) velocity, element (k, comp, node) at k*vstride + comp*n_s + node
  const double2* v2;   // slot 2 (x2)
  long vstride;
  const double2* pA;   // pressure, (k, h, node) at k*pstride + h*phoff + node
  const double2* pB;   // Stokes only: Chebyshev(M_p) part
  long pstride, phoff;
  int stokes;
  double pscale;       // Oseen: slots 3/4 = pscale * pA
};

__device__ __forceinline__ bool q2_interior(long node, int n1, int dim) {
  int i = (int)(node % n1), j = (int)((node / n1) % n1);
  bool in = i > 0 && i < n1 - 1 && j > 0 && j < n1 - 1;
  if (dim == 3) {
    int k = (int)(node / ((long)n1 * n1));
    in = in && k > 0 && k < n1 - 1;
  }
  return in;
}

struct Geo {
  int dim, n1q2, n1q1, n_b, n_f;
  long n_s, n_v, n_p, nblk;
  double tau, nu, beta;
  double rst;          // 1 / sqrt(tau)
};

// slot values y_h0, y_h1 of column `col` at frequency k (after T_r^{-1} for Stokes)
__device__ __forceinline__ void slot_values(const Geo& G, const InvSrc& S, const FreqConst& f, int k, long col,
                                            double2& y0, double2& y1) {
  const double rs = G.rst;   // 1 / sqrt(tau)
  if (col < G.n_v) {
    const long comp = col / G.n_s, node = col % G.n_s;
    const double2 x1 = S.v1[k * S.vstride + comp * G.n_s + node];
    const double2 x2 = S.v2[k * S.vstride + comp * G.n_s + node];
    if (S.stokes) {
      // T_r^{-1}: y2 = x2 c2 / sqrt(tau); y1 = (x1 + i (dc/sqrt(tau)) y2) / sqrt(tau)
      const double g = f.c2 * rs;
      const double2 yy2 = make_double2(x2.x * g, x2.y * g);
      const double a = f.dc * rs;
      y0 = make_double2((x1.x - a * yy2.y) * rs, (x1.y + a * yy2.x) * rs);
      y1 = yy2;
    } else {
      y0 = x1;
      y1 = x2;
    }
  } else {
    const long node = col - G.n_v;
    const double2 a0 = S.pA[k * S.pstride + node];
    const double2 a1 = S.pA[k * S.pstride + S.phoff + node];
    if (S.stokes) {
      // x3 = (1+c1) K_p^{-1} s3 + nu c2 M_p^{-1} s3, same for x4 (pB == nullptr: already combined)
      double2 x3 = a0, x4 = a1;
      if (S.pB) {
        const double2 b0 = S.pB[k * S.pstride + node];
        const double2 b1 = S.pB[k * S.pstride + S.phoff + node];
        const double ca = 1.0 + f.c1, cb = G.nu * f.c2;
        x3 = make_double2(ca * a0.x + cb * b0.x, ca * a0.y + cb * b0.y);
        x4 = make_double2(ca * a1.x + cb * b1.x, ca * a1.y + cb * b1.y);
      }
      // T_r^{-1}: y4 = x4 / sqrt(tau); y3 = (x3 + i (dc c2 / sqrt(tau)) y4) / (sqrt(tau) c2)
      const double2 yy4 = make_double2(x4.x * rs, x4.y * rs);
      const double a = f.dc * f.c2 * rs, rden = rs * f.rc2;
      y0 = make_double2((x3.x - a * yy4.y) * rden, (x3.y + a * yy4.x) * rden);
      y1 = yy4;
    } else {
      y0 = make_double2(S.pscale * a0.x, S.pscale * a0.y);
      y1 = make_double2(S.pscale * a1.x, S.pscale * a1.y);
    }
  }
}

__device__ __forceinline__ bool col_masked(const Geo& G, long col) {
  if (col < G.n_v) return !q2_interior(col % G.n_s, G.n1q2, G.dim);
  return (col - G.n_v) == 0;
}

// ------------------------------------------------------------------ forward transform
// store T_l^{-1} r_hat_k of one column (Stokes; Oseen: no T transform) in the frequency layout
__device__ __forceinline__ void fwd_store(const Geo& G, double2* __restrict__ Fv, double2* __restrict__ Fp,
                                          const FreqConst& f, int k, long col, double2 s0, double2 s1, int stokes) {
  const double rs = G.rst;
  if (col < G.n_v) {
    if (stokes) {
      // T_l^{-1}: s1 = r1/sqrt(tau); s2 = (r2 - i (dc/sqrt(tau)) s1) c2 / sqrt(tau)
      const double2 q1 = make_double2(s0.x * rs, s0.y * rs);
      const double a = f.dc * rs, g = f.c2 * rs;
      s1 = make_double2((s1.x + a * q1.y) * g, (s1.y - a * q1.x) * g);
      s0 = q1;
    }
    const long comp = col / G.n_s, node = col % G.n_s;
    Fv[(((long)k * 2 + 0) * G.dim + comp) * G.n_s + node] = s0;
    Fv[(((long)k * 2 + 1) * G.dim + comp) * G.n_s + node] = s1;
  } else {
    if (stokes) {
      // s3 = r3 / (sqrt(tau) c2); s4 = (r4 - i (dc c2 / sqrt(tau)) s3) / sqrt(tau)
      const double rden = rs * f.rc2;
      const double2 q3 = make_double2(s0.x * rden, s0.y * rden);
      const double a = f.dc * f.c2 * rs;
      s1 = make_double2((s1.x + a * q3.y) * rs, (s1.y - a * q3.x) * rs);
      s0 = q3;
    }
    const long node = col - G.n_v;
    Fp[((long)k * 2 + 0) * G.n_p + node] = s0;
    Fp[((long)k * 2 + 1) * G.n_p + node] = s1;
  }
}

__global__ void k_fft_fwd(Geo G, const double* __restrict__ r, double2* __restrict__ Fv, double2* __restrict__ Fp,
                          const FreqConst* __restrict__ fc, const double2* __restrict__ tw, int TD, int stokes) {
  extern __shared__ double sm[];
  const int n_b = G.n_b;
  double2* stw = reinterpret_cast<double2*>(sm);
  double* xs = sm + 2 * n_b;  // [2 n_b][TD]
  const int tx = threadIdx.x, ty = threadIdx.y, KY = blockDim.y;
  const int tid = ty * blockDim.x + tx;
  for (int m = tid; m < n_b; m += blockDim.x * KY) stw[m] = tw[m];
  const long col = (long)blockIdx.x * TD + tx;
  const bool valid = col < G.nblk;
  const bool msk = !valid || col_masked(G, col);
  for (int row = ty; row < 2 * n_b; row += KY)
    xs[row * TD + tx] = msk ? 0.0 : __ldg(r + (long)row * G.nblk + col);
  __syncthreads();
  if (!valid) return;
  const double st = sqrt(G.tau);
  for (int k = ty; k < G.n_f; k += KY) {
    // r_hat_k = sum_t r_{t} omega^{k t}, omega = exp(-2 pi i / n_b)   (reading C.2 #2)
    double a0r = 0, a0i = 0, a1r = 0, a1i = 0;
    int m = 0;
    for (int t = 0; t < n_b; ++t) {
      const double2 w = stw[m];
      const double x0 = xs[t * TD + tx], x1 = xs[(n_b + t) * TD + tx];
      a0r = fma(x0, w.x, a0r);
      a0i = fma(-x0, w.y, a0i);
      a1r = fma(x1, w.x, a1r);
      a1i = fma(-x1, w.y, a1i);
      m += k;
      if (m >= n_b) m -= n_b;
    }
    fwd_store(G, Fv, Fp, fc[k], k, col, make_double2(a0r, a0i), make_double2(a1r, a1i), stokes);
  }
}

// Forward transform with the real-input symmetry (the time series are real):
//   r_hat_k = r_0 + sum_{t=1}^{(n-1)/2} [(r_t + r_{n-t}) cos(2 pi k t / n) - i (r_t - r_{n-t}) sin(2 pi k t / n)]
//             (+ r_{n/2} (-1)^k for even n)
// -- half the multiply-adds of the plain sum.  The pair sums/differences are formed in place in shared
// memory; every thread keeps KB frequencies of one column in registers, so each staged value is read
// once per KB outputs and each twiddle load is a warp broadcast.
template <int KB>
__global__ void __launch_bounds__(256) k_fft_fwd_sym(Geo G, const double* __restrict__ r, double2* __restrict__ Fv,
                                                     double2* __restrict__ Fp, const FreqConst* __restrict__ fc,
                                                     const double2* __restrict__ tw, int TD, int stokes) {
  extern __shared__ double sm[];
  const int n = G.n_b;
  double2* stw = reinterpret_cast<double2*>(sm);
  double* xs = sm + 2 * n;  // [2 n][TD]
  const int tx = threadIdx.x, ty = threadIdx.y, KY = blockDim.y;
  const int tid = ty * blockDim.x + tx;
  for (int m = tid; m < n; m += blockDim.x * KY) stw[m] = tw[m];
  const long col = (long)blockIdx.x * TD + tx;
  const bool valid = col < G.nblk;
  const bool msk = !valid || col_masked(G, col);
  for (int row = ty; row < 2 * n; row += KY)
    xs[row * TD + tx] = msk ? 0.0 : __ldg(r + (long)row * G.nblk + col);
  __syncthreads();
  const int hh = (n - 1) / 2;   // pairs t, n - t (t = 1..hh); even n: t = n/2 unpaired
  for (int t = 1 + ty; t <= hh; t += KY)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double a = xs[(h * n + t) * TD + tx], b = xs[(h * n + n - t) * TD + tx];
      xs[(h * n + t) * TD + tx] = a + b;
      xs[(h * n + n - t) * TD + tx] = a - b;
    }
  __syncthreads();
  if (!valid) return;
  const bool even = (n & 1) == 0;
  int kk[KB], m[KB];
  double re[KB][2], im[KB][2];
  const double x00 = xs[tx], x10 = xs[n * TD + tx];
  const double xn0 = even ? xs[(n / 2) * TD + tx] : 0.0, xn1 = even ? xs[(n + n / 2) * TD + tx] : 0.0;
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    kk[j] = ty + KY * j;
    m[j] = 0;
    const double sg = (kk[j] & 1) ? -1.0 : 1.0;
    re[j][0] = x00 + sg * xn0;
    re[j][1] = x10 + sg * xn1;
    im[j][0] = im[j][1] = 0.0;
  }
  for (int t = 1; t <= hh; ++t) {
    const double p0 = xs[t * TD + tx], q0 = xs[(n - t) * TD + tx];
    const double p1 = xs[(n + t) * TD + tx], q1 = xs[(2 * n - t) * TD + tx];
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      m[j] += kk[j];
      if (m[j] >= n) m[j] -= n;
      const double2 w = stw[m[j]];
      re[j][0] = fma(p0, w.x, re[j][0]);
      im[j][0] = fma(-q0, w.y, im[j][0]);
      re[j][1] = fma(p1, w.x, re[j][1]);
      im[j][1] = fma(-q1, w.y, im[j][1]);
    }
  }
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    const int k = kk[j];
    if (k >= G.n_f) continue;
    fwd_store(G, Fv, Fp, fc[k], k, col, make_double2(re[j][0], im[j][0]), make_double2(re[j][1], im[j][1]), stokes);
  }
}

// Inverse transform with the same symmetry: for t and n - t
//   y_t, y_{n-t} = (1/n) [y_hat_0 + 2 (C_t -+ S_t) (+ Nyquist)],  C_t = sum_k Re y_hat_k cos(2 pi k t / n),
//   S_t = sum_k Im y_hat_k sin(2 pi k t / n),  k = 1..n_f-1 (even n: y_hat_{n/2} (-1)^t once).
template <int TB>
__global__ void __launch_bounds__(256) k_fft_inv_sym(Geo G, InvSrc S, double* __restrict__ z,
                                                     const FreqConst* __restrict__ fc, const double2* __restrict__ tw,
                                                     int TD) {
  extern __shared__ double sm[];
  const int n = G.n_b, n_f = G.n_f;
  double2* stw = reinterpret_cast<double2*>(sm);
  double2* ys = stw + n;  // [2][n_f][TD]
  const int tx = threadIdx.x, ty = threadIdx.y, KY = blockDim.y;
  const int tid = ty * blockDim.x + tx;
  for (int m = tid; m < n; m += blockDim.x * KY) stw[m] = tw[m];
  const long col = (long)blockIdx.x * TD + tx;
  const bool valid = col < G.nblk;
  const bool msk = !valid || col_masked(G, col);
  for (int k = ty; k < n_f; k += KY) {
    double2 y0 = make_double2(0, 0), y1 = y0;
    if (!msk) slot_values(G, S, fc[k], k, col, y0, y1);
    ys[(0 * n_f + k) * TD + tx] = y0;
    ys[(1 * n_f + k) * TD + tx] = y1;
  }
  __syncthreads();
  if (!valid) return;
  const bool even = (n & 1) == 0;
  const int kend = even ? n_f - 1 : n_f;   // k = 1..kend-1 with weight 2; even n: Nyquist k = n/2 once
  const int thalf = n / 2;                 // t = 0..thalf (mirror n - t)
  int tt[TB], m[TB];
  double C[TB][2], Sn[TB][2];
#pragma unroll
  for (int j = 0; j < TB; ++j) {
    tt[j] = ty + KY * j;
    m[j] = 0;
    C[j][0] = C[j][1] = Sn[j][0] = Sn[j][1] = 0.0;
  }
  for (int k = 1; k < kend; ++k) {
    const double2 a = ys[(0 * n_f + k) * TD + tx], b = ys[(1 * n_f + k) * TD + tx];
#pragma unroll
    for (int j = 0; j < TB; ++j) {
      m[j] += tt[j];
      while (m[j] >= n) m[j] -= n;
      const double2 w = stw[m[j]];
      C[j][0] = fma(a.x, w.x, C[j][0]);
      Sn[j][0] = fma(a.y, w.y, Sn[j][0]);
      C[j][1] = fma(b.x, w.x, C[j][1]);
      Sn[j][1] = fma(b.y, w.y, Sn[j][1]);
    }
  }
  const double inv_n = 1.0 / n;
  const double2 a0 = ys[tx], b0 = ys[n_f * TD + tx];
  const double2 an = even ? ys[(n_f - 1) * TD + tx] : make_double2(0, 0);
  const double2 bn = even ? ys[(2 * n_f - 1) * TD + tx] : make_double2(0, 0);
#pragma unroll
  for (int j = 0; j < TB; ++j) {
    const int t = tt[j];
    if (t > thalf) continue;
    const double sg = (t & 1) ? -1.0 : 1.0;
    const double base0 = a0.x + sg * an.x, base1 = b0.x + sg * bn.x;
    z[(long)t * G.nblk + col] = msk ? 0.0 : (base0 + 2.0 * (C[j][0] - Sn[j][0])) * inv_n;
    z[(long)(n + t) * G.nblk + col] = msk ? 0.0 : (base1 + 2.0 * (C[j][1] - Sn[j][1])) * inv_n;
    if (t > 0 && 2 * t != n) {
      z[(long)(n - t) * G.nblk + col] = msk ? 0.0 : (base0 + 2.0 * (C[j][0] + Sn[j][0])) * inv_n;
      z[(long)(2 * n - t) * G.nblk + col] = msk ? 0.0 : (base1 + 2.0 * (C[j][1] + Sn[j][1])) * inv_n;
    }
  }
}

// ------------------------------------------------------------------ prime-factor (Good-Thomas) transforms
// n_b = P Q with gcd(P, Q) = 1 (511 = 7 x 73, 255 = 15 x 17, 63 = 7 x 9, 15 = 3 x 5): the DFT of P:332-344,
//   r_hat_k = sum_t r_t omega^{k t},  omega = exp(-2 pi i / n_b),
// is evaluated exactly (up to rounding order) as a 2-D DFT through the index maps
//   t = (Q t1 + P t2) mod n_b,   k = (k1 Q (Q^-1 mod P) + k2 P (P^-1 mod Q)) mod n_b,
// for which omega^{k t} = omega_P^{k1 t1} omega_Q^{k2 t2} (no twiddle factors):
//   stage A: Y[t1][k2] = sum_t2 r[t(t1, t2)] omega_Q^{k2 t2}   (real input: k2 <= (Q-1)/2, pair sums/differences)
//   stage B: X[k1][k2] = sum_t1 Y[t1][k2] omega_P^{k1 t1}
// and the Hermitian half X[n_b - k] = conj(X[k]) covers every k < n_f.  Work per series ~ n_b (Q/2 + P) multiply-
// adds instead of the dense sum's ~n_b^2/2 (c4 at n_t = 512: 43 n_b vs 255 n_b).
// Thread layout: a CTA owns 16 spatial columns x 2 halves = 32 series (lane = column + 16 half, warp w = t1 for
// stage A); every thread loads its Q inputs straight from global memory (rows t(t1, .) of its column: 2 x 128-byte
// segments per warp load), keeps the pair sums in registers, and exchanges Y through shared memory in blocks of P
// values of k2.  T_l^{-1} (Stokes) is applied at the store; the halves meet by a lane shuffle.
template <int P, int Q>
struct Pfa {
  static constexpr int HQ = (Q - 1) / 2;           // pairs t2, Q - t2
  static constexpr int NK2 = HQ + 1;               // k2 = 0..HQ
  // k2 per block: stage A computes 4 k2 at a time (4 independent accumulator pairs per pass over the pairs); up to 4
  // per warp in stage B
  static constexpr int KB = (NK2 + 3) / 4 * 4 <= 4 * P ? (NK2 + 3) / 4 * 4 : 4 * P;
  static constexpr int NBLK = (NK2 + KB - 1) / KB;
  static constexpr int THREADS = 32 * P;
  // dynamic shared memory (double2 units): twiddles omega_Q^{k2 (j + 1)} [NK2][HQ], omega_P [P], frequency
  // constants [n_f] (FreqConst = 5 doubles, rounded to 3 double2), then the exchange buffers
  static constexpr int TW2 = NK2 * HQ;
  static size_t smem(int n_f, int nbuf) {
    return (size_t)(TW2 + P + 3 * n_f + nbuf * KB * P * 32) * sizeof(double2);
  }
};

struct PfaMap {
  int QA, PB;   // Q (Q^-1 mod P), P (P^-1 mod Q)
};

__device__ __forceinline__ double2 cj(double2 a) { return make_double2(a.x, -a.y); }

// T_l^{-1} of one column at frequency k with the two halves (s0: half 0, s1: half 1); returns half h
__device__ __forceinline__ double2 tl_inv_half(const Geo& G, const FreqConst& f, long col, double2 s0, double2 s1,
                                               int stokes, int h) {
  if (!stokes) return h ? s1 : s0;
  const double rs = G.rst;
  if (col < G.n_v) {
    const double2 q1 = make_double2(s0.x * rs, s0.y * rs);
    if (h == 0) return q1;
    const double a = f.dc * rs, g = f.c2 * rs;
    return make_double2((s1.x + a * q1.y) * g, (s1.y - a * q1.x) * g);
  }
  const double rden = rs * f.rc2;
  const double2 q3 = make_double2(s0.x * rden, s0.y * rden);
  if (h == 0) return q3;
  const double a = f.dc * f.c2 * rs;
  return make_double2((s1.x + a * q3.y) * rs, (s1.y - a * q3.x) * rs);
}

// shared tables of the prime-factor kernels: tw2[k2][j] = (cos, sin)(2 pi k2 (j + 1) / Q), twP[m] = (cos, sin)(2 pi m / P),
// fcs[k] = the frequency constants (k < n_f)
template <int P, int Q>
__device__ __forceinline__ void pfa_tables(const Geo& G, const double2* __restrict__ tw, const FreqConst* __restrict__ fc,
                                           double2* tw2, double2* twP, FreqConst* fcs) {
  using PF = Pfa<P, Q>;
  for (int e = threadIdx.x; e < PF::TW2; e += PF::THREADS) {
    const int k2 = e / PF::HQ, j = e - k2 * PF::HQ;
    tw2[e] = tw[((k2 * (j + 1)) % Q) * P];          // exp(2 pi i m / Q) = tw[m P] (tw: n_b-th roots)
  }
  for (int m = threadIdx.x; m < P; m += PF::THREADS) twP[m] = tw[m * Q];
  for (int k = threadIdx.x; k < G.n_f; k += PF::THREADS) fcs[k] = fc[k];
}

template <int P, int Q>
__global__ void __launch_bounds__(Pfa<P, Q>::THREADS) k_fft_fwd_pfa(Geo G, const double* __restrict__ r,
                                                                    double2* __restrict__ Fv, double2* __restrict__ Fp,
                                                                    const FreqConst* __restrict__ fc,
                                                                    const double2* __restrict__ tw, PfaMap mp,
                                                                    int stokes) {
  using PF = Pfa<P, Q>;
  constexpr int n = P * Q;
  extern __shared__ double2 pfa_sm[];
  double2* tw2 = pfa_sm;
  double2* twP = tw2 + PF::TW2;
  FreqConst* fcs = reinterpret_cast<FreqConst*>(twP + P);
  double2 (*Ys)[P][32] = reinterpret_cast<double2 (*)[P][32]>(twP + P + 3 * G.n_f);   // [k2 - block start][t1][series]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int h = lane >> 4;
  const long col = (long)blockIdx.x * 16 + (lane & 15);
  pfa_tables<P, Q>(G, tw, fc, tw2, twP, fcs);
  const bool valid = col < G.nblk;
  const bool msk = !valid || col_masked(G, col);
  // destination of this series: Fv[k][h][comp][node] (velocity) or Fp[k][h][node]; element k at dst + k * dstride
  double2* dst;
  long dstride;
  if (col < G.n_v) {
    const long comp = col / G.n_s, node = col - comp * G.n_s;
    dst = Fv + ((long)h * G.dim + comp) * G.n_s + node;
    dstride = 2L * G.dim * G.n_s;
  } else {
    dst = Fp + (long)h * G.n_p + (col - G.n_v);
    dstride = 2L * G.n_p;
  }
  // stage A inputs of series (col, h), t1 = w: y[t2] = r[h][t(w, t2)][col]; pair sums / differences in registers
  const double* rc = r + (long)h * n * G.nblk + col;
  double ps[PF::HQ], pd[PF::HQ];
  auto ld = [&](int t2) { return msk ? 0.0 : __ldg(rc + (long)((Q * w + P * t2) % n) * G.nblk); };
  const double y0 = ld(0);
#pragma unroll
  for (int j = 0; j < PF::HQ; ++j) {
    const double a = ld(1 + j), b = ld(Q - 1 - j);
    ps[j] = a + b;
    pd[j] = a - b;
  }
  __syncthreads();
  for (int blk = 0; blk < PF::NBLK; ++blk) {
    // stage A: Y[w][k2] for k2 = blk KB + i, four at a time:  Re = y0 + sum_j ps_j cos, Im = -sum_j pd_j sin
#pragma unroll 1
    for (int i0 = 0; i0 < PF::KB; i0 += 4) {
      const int kb = blk * PF::KB + i0;
      double re[4], im[4];
      const double2* tr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        re[u] = y0;
        im[u] = 0.0;
        tr[u] = tw2 + min(kb + u, PF::HQ) * PF::HQ;   // rows past HQ are computed but never stored
      }
#pragma unroll
      for (int j = 0; j < PF::HQ; ++j) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 wq = tr[u][j];                  // warp-uniform broadcast
          re[u] = fma(ps[j], wq.x, re[u]);
          im[u] = fma(-pd[j], wq.y, im[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (kb + u <= PF::HQ) Ys[i0 + u][w][lane] = make_double2(re[u], im[u]);
    }
    __syncthreads();
    // stage B: X[k1][k2] = sum_t1 Y[t1][k2] omega_P^{k1 t1}, k1 = 0..P-1; then T_l^{-1} and the store
    for (int i = w; i < PF::KB; i += P) {
      const int k2 = blk * PF::KB + i;
      if (k2 > PF::HQ) break;
      double2 yv[P];
#pragma unroll
      for (int t1 = 0; t1 < P; ++t1) yv[t1] = Ys[i][t1][lane];
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) {
        double2 x = yv[0];
#pragma unroll
        for (int t1 = 1; t1 < P; ++t1) {
          const double2 wp = twP[(k1 * t1) % P];   // exp(-2 pi i k1 t1 / P) = (cos, -sin)
          x.x += yv[t1].x * wp.x + yv[t1].y * wp.y;
          x.y += yv[t1].y * wp.x - yv[t1].x * wp.y;
        }
        int k = (k1 * mp.QA + k2 * mp.PB) % n;
        if (k >= G.n_f) {               // X[n - k] = conj(X[k]); k2 = 0 entries above n_f are their own mirror
          if (k2 == 0) continue;
          k = n - k;
          x = cj(x);
        }
        double2 other;
        other.x = __shfl_xor_sync(0xffffffffu, x.x, 16);
        other.y = __shfl_xor_sync(0xffffffffu, x.y, 16);
        if (!valid) continue;
        const double2 s0 = h ? other : x, s1 = h ? x : other;
        dst[k * dstride] = tl_inv_half(G, fcs[k], col, s0, s1, stokes, h);
      }
    }
    __syncthreads();
  }
}

// Inverse (step A8): y_t = (1/n_b) sum_k y_hat_k omega^{-k t} with y_hat_{n_b - k} = conj(y_hat_k), through the same
// maps:  Z[t1][k2] = sum_k1 Yh[k1][k2] omega_P^{-k1 t1}  (k2 <= HQ; Yh gathered from the half spectrum after
// T_r^{-1}),  y[t1][t2] = (1/n_b) [Z[t1][0] + 2 sum_{k2 >= 1} Re(Z[t1][k2] omega_Q^{-k2 t2})]  (pairs t2, Q - t2).
template <int P, int Q>
__global__ void __launch_bounds__(Pfa<P, Q>::THREADS) k_fft_inv_pfa(Geo G, InvSrc S, double* __restrict__ z,
                                                                    const FreqConst* __restrict__ fc,
                                                                    const double2* __restrict__ tw, PfaMap mp) {
  using PF = Pfa<P, Q>;
  constexpr int n = P * Q;
  extern __shared__ double2 pfa_sm[];
  double2* tw2 = pfa_sm;
  double2* twP = tw2 + PF::TW2;
  FreqConst* fcs = reinterpret_cast<FreqConst*>(twP + P);
  double2 (*Hs)[P][32] = reinterpret_cast<double2 (*)[P][32]>(twP + P + 3 * G.n_f);   // gathered spectrum [k2][k1][s],
                                                                                       // then Z [k2][t1][s] in place
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int h = lane >> 4;
  const long col = (long)blockIdx.x * 16 + (lane & 15);
  pfa_tables<P, Q>(G, tw, fc, tw2, twP, fcs);
  const bool valid = col < G.nblk;
  const bool msk = !valid || col_masked(G, col);
  double a0 = 0.0, s0 = 0.0;            // Z[w][0].re and sum_{k2>=1} Re Z[w][k2] (t2 = 0)
  double C[PF::HQ], Sn[PF::HQ];
#pragma unroll
  for (int j = 0; j < PF::HQ; ++j) C[j] = Sn[j] = 0.0;
  __syncthreads();
  for (int blk = 0; blk < PF::NBLK; ++blk) {
    // gather: Yh[k1][k2] for the block's k2 (T_r^{-1} applied, both halves read, own half kept); the P entries of
    // an item are independent, so their loads are all in flight together
    for (int i = w; i < PF::KB; i += P) {
      const int k2g = blk * PF::KB + i;
      if (k2g > PF::HQ) break;
      double2 v[P];
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) {
        int k = (k1 * mp.QA + k2g * mp.PB) % n;
        const bool cjg = k >= G.n_f;
        if (cjg) k = n - k;
        double2 v0 = make_double2(0.0, 0.0), v1 = v0;
        if (!msk) slot_values(G, S, fcs[k], k, col, v0, v1);
        v[k1] = h ? v1 : v0;
        if (cjg) v[k1] = cj(v[k1]);
      }
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) Hs[i][k1][lane] = v[k1];
    }
    __syncthreads();
    // stage B^-1: Z[t1] = sum_k1 Yh[k1] omega_P^{-k1 t1}, written over Yh (each lane owns its entries)
    for (int i = w; i < PF::KB; i += P) {
      const int k2g = blk * PF::KB + i;
      if (k2g > PF::HQ) break;
      double2 hv[P];
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) hv[k1] = Hs[i][k1][lane];
#pragma unroll
      for (int t1 = 0; t1 < P; ++t1) {
        double2 x = hv[0];
#pragma unroll
        for (int k1 = 1; k1 < P; ++k1) {
          const double2 wp = twP[(k1 * t1) % P];   // omega_P^{-k1 t1} = (cos, +sin)
          x.x += hv[k1].x * wp.x - hv[k1].y * wp.y;
          x.y += hv[k1].y * wp.x + hv[k1].x * wp.y;
        }
        Hs[i][t1][lane] = x;
      }
    }
    __syncthreads();
    // stage A^-1 partial sums for t1 = w over this block's k2
    for (int i = 0; i < PF::KB; ++i) {
      const int k2 = blk * PF::KB + i;
      if (k2 > PF::HQ) break;
      const double2 zz = Hs[i][w][lane];
      if (k2 == 0) {
        a0 = zz.x;
        continue;
      }
      s0 += zz.x;
      const double2* tr = tw2 + k2 * PF::HQ;
#pragma unroll
      for (int j = 0; j < PF::HQ; ++j) {
        const double2 wq = tr[j];        // cos, sin of 2 pi k2 (j + 1) / Q
        C[j] = fma(zz.x, wq.x, C[j]);
        Sn[j] = fma(zz.y, wq.y, Sn[j]);
      }
    }
    __syncthreads();
  }
  if (!valid) return;
  const double inv_n = 1.0 / n;
  double* zc = z + (long)h * n * G.nblk + col;
  zc[(long)((Q * w) % n) * G.nblk] = msk ? 0.0 : (a0 + 2.0 * s0) * inv_n;
#pragma unroll
  for (int j = 0; j < PF::HQ; ++j) {
    const int t2 = j + 1;
    const int ta = (Q * w + P * t2) % n, tb = (Q * w + P * (Q - t2)) % n;
    zc[(long)ta * G.nblk] = msk ? 0.0 : (a0 + 2.0 * (C[j] - Sn[j])) * inv_n;
    zc[(long)tb * G.nblk] = msk ? 0.0 : (a0 + 2.0 * (C[j] + Sn[j])) * inv_n;
  }
}

// ------------------------------------------------------------------ inverse transform
__global__ void k_fft_inv(Geo G, InvSrc S, double* __restrict__ z, const FreqConst* __restrict__ fc,
                          const double2* __restrict__ tw, int TD) {
  extern __shared__ double sm[];
  const int n_b = G.n_b, n_f = G.n_f;
  double2* stw = reinterpret_cast<double2*>(sm);
  double2* ys = stw + n_b;  // [2][n_f][TD]
  const int tx = threadIdx.x, ty = threadIdx.y, KY = blockDim.y;
  const int tid = ty * blockDim.x + tx;
  for (int m = tid; m < n_b; m += blockDim.x * KY) stw[m] = tw[m];
  const long col = (long)blockIdx.x * TD + tx;
  const bool valid = col < G.nblk;
  const bool msk = !valid || col_masked(G, col);
  for (int k = ty; k < n_f; k += KY) {
    double2 y0 = make_double2(0, 0), y1 = y0;
    if (!msk) slot_values(G, S, fc[k], k, col, y0, y1);
    ys[(0 * n_f + k) * TD + tx] = y0;
    ys[(1 * n_f + k) * TD + tx] = y1;
  }
  __syncthreads();
  if (!valid) return;
  const bool even = (n_b % 2) == 0;
  const double inv_n = 1.0 / n_b;
  for (int t = ty; t < n_b; t += KY) {
    // y_t = (1/n_b) sum_k y_hat_k omega^{-k t}, using y_hat_{n_b-k} = conj(y_hat_k)
    double acc0 = ys[(0 * n_f) * TD + tx].x, acc1 = ys[(1 * n_f) * TD + tx].x;
    int m = 0;
    for (int k = 1; k < n_f; ++k) {
      m += t;
      if (m >= n_b) m -= n_b;
      const double2 w = stw[m];
      const double wk = (even && 2 * k == n_b) ? 1.0 : 2.0;
      const double2 a = ys[(0 * n_f + k) * TD + tx], b = ys[(1 * n_f + k) * TD + tx];
      acc0 = fma(wk, a.x * w.x - a.y * w.y, acc0);
      acc1 = fma(wk, b.x * w.x - b.y * w.y, acc1);
    }
    z[(long)t * G.nblk + col] = msk ? 0.0 : acc0 * inv_n;
    z[(long)(n_b + t) * G.nblk + col] = msk ? 0.0 : acc1 * inv_n;
  }
}

__global__ void k_debug_block(Geo G, InvSrc S, const FreqConst* __restrict__ fc, int k, double2* out) {
  const long col = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= G.nblk) return;
  double2 y0 = make_double2(0, 0), y1 = y0;
  if (!col_masked(G, col)) slot_values(G, S, fc[k], k, col, y0, y1);
  out[col] = y0;
  out[G.nblk + col] = y1;
}

// ------------------------------------------------------------------ KKT matvec (real)
struct KKTTab {
  const double *tM, *tK, *conv, *convT;   // fine Q2 (eliminated columns zero)
  const double *tPmT, *tGmT;              // B^T rows [n1q2][3]
  const double *tPm, *tGm;                // B rows [n1q1][5]
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Velocity rows of eq. (FinalA) expanded block-row by block-row (E (x) M = backward-Euler difference):
//   half 0  y1v_t = M(tau v_t + lam_t - lam_{t+1}) + tau L^T lam_t + tau B^T mu_t
//   half 1  y2v_t = M(v_t - v_{t-1} - tau/beta lam_t) + tau L v_t + tau B^T p_t
// (used for Oseen and as the fallback of the time-marching kernels).  A CTA owns a TX x TY (x TZ) tile of one
// (half, t, component) slice; it forms the mass operand w = cA v_t + cB lam_t + cO other and the
// L-operand u once per node of the tile + 2-halo in shared memory (masked / outside nodes = 0,
// which is exactly the elimination), plus the pressure tile for B^T.
template <int DIM>
struct KT {
  static constexpr int TX = 32, TY = DIM == 2 ? 8 : 4, TZ = DIM == 2 ? 1 : 2;
  static constexpr int SX = TX + 4, SY = TY + 4, SZ = DIM == 2 ? 1 : TZ + 4;
  static constexpr int PX = TX / 2 + 4, PY = TY / 2 + 4, PZ = DIM == 2 ? 1 : TZ / 2 + 4;
};

template <int DIM>
__global__ void __launch_bounds__(256) k_kkt_vel_tiled(Geo G, KKTTab T, const double* __restrict__ x,
                                                       double* __restrict__ y, int oseen, int tiles_x, int tiles_y) {
  using K = KT<DIM>;
  __shared__ double sw[K::SZ][K::SY][K::SX];
  __shared__ double su[K::SZ][K::SY][K::SX];
  __shared__ double sq[K::PZ][K::PY][K::PX];
  const int row = blockIdx.y;  // h * n_b + t
  const int h = row / G.n_b, t = row % G.n_b;
  const int comp = blockIdx.z;
  const int tile = blockIdx.x;
  const int txi = tile % tiles_x, tyi = (tile / tiles_x) % tiles_y, tzi = tile / (tiles_x * tiles_y);
  const int x0 = txi * K::TX, y0 = tyi * K::TY, z0 = DIM == 3 ? tzi * K::TZ : 0;
  const int n1 = G.n1q2, m1 = G.n1q1;
  const long nblk = G.nblk, n_b = G.n_b, ns = G.n_s;
  const double tau = G.tau;
  const double* xv = x + (long)t * nblk + comp * ns;
  const double* xl = x + (long)(n_b + t) * nblk + comp * ns;
  const double* xo = nullptr;
  double cA, cB, cO;
  if (h == 0) {
    cA = tau; cB = 1.0; cO = -1.0;
    if (t + 1 < n_b) xo = x + (long)(n_b + t + 1) * nblk + comp * ns;
  } else {
    cA = 1.0; cB = -tau / G.beta; cO = -1.0;
    if (t >= 1) xo = x + (long)(t - 1) * nblk + comp * ns;
  }
  const int tid = threadIdx.x;
  const int NS = K::SX * K::SY * K::SZ;
  for (int e = tid; e < NS; e += blockDim.x) {
    const int li = e % K::SX, lj = (e / K::SX) % K::SY, lk = e / (K::SX * K::SY);
    const int gi = x0 - 2 + li, gj = y0 - 2 + lj, gk = DIM == 3 ? z0 - 2 + lk : 0;
    double wv = 0.0, uv = 0.0;
    bool in = gi > 0 && gi < n1 - 1 && gj > 0 && gj < n1 - 1;
    if (DIM == 3) in = in && gk > 0 && gk < n1 - 1;
    if (in) {
      const long nd = ((long)gk * n1 + gj) * n1 + gi;
      const double a = xv[nd], l = xl[nd];
      wv = cA * a + cB * l;
      if (xo) wv += cO * xo[nd];
      uv = h == 0 ? l : a;
    }
    sw[lk][lj][li] = wv;
    su[lk][lj][li] = uv;
  }
  // pressure tile: Q1 nodes from floor((x0-1)/2)
  const int P0x = (x0 >= 1) ? (x0 - 1) / 2 : -1, P0y = (y0 >= 1) ? (y0 - 1) / 2 : -1;
  const int P0z = DIM == 3 ? ((z0 >= 1) ? (z0 - 1) / 2 : -1) : 0;
  const double* q = x + (long)(h == 0 ? (n_b + t) : t) * nblk + G.n_v;
  const int NP = K::PX * K::PY * K::PZ;
  for (int e = tid; e < NP; e += blockDim.x) {
    const int li = e % K::PX, lj = (e / K::PX) % K::PY, lk = e / (K::PX * K::PY);
    const int I = P0x + li, J = P0y + lj, Kk = DIM == 3 ? P0z + lk : 0;
    double v = 0.0;
    if (I >= 0 && I < m1 && J >= 0 && J < m1 && Kk >= 0 && Kk < m1) {
      const long pn = ((long)Kk * m1 + J) * m1 + I;
      if (pn != 0) v = q[pn];  // pinned pressure node: eliminated column
    }
    sq[lk][lj][li] = v;
  }
  __syncthreads();
  const int lx = tid % K::TX, ly = (tid / K::TX) % K::TY, lz = DIM == 3 ? tid / (K::TX * K::TY) : 0;
  const int i = x0 + lx, j = y0 + ly, k = z0 + lz;
  if (i >= n1 || j >= n1 || (DIM == 3 && k >= n1)) return;
  const long node = ((long)k * n1 + j) * n1 + i;
  double* yo = y + (long)row * nblk + comp * ns + node;
  bool interior = i > 0 && i < n1 - 1 && j > 0 && j < n1 - 1;
  if (DIM == 3) interior = interior && k > 0 && k < n1 - 1;
  if (!interior) {
    *yo = 0.0;
    return;
  }
  double mx[5], kx[5];
#pragma unroll
  for (int o = 0; o < 5; ++o) {
    mx[o] = __ldg(T.tM + i * 5 + o);
    kx[o] = __ldg(T.tK + i * 5 + o);
  }
  const double* cv = oseen ? ((h == 0 ? T.convT : T.conv) + node * (DIM == 2 ? 25 : 125)) : nullptr;
  double Mw = 0, KL = 0, CL = 0;
  const int zb = DIM == 3 ? 0 : 2, ze = DIM == 3 ? 5 : 3;
  for (int oc = zb; oc < ze; ++oc) {
    const double mz = DIM == 3 ? __ldg(T.tM + k * 5 + oc) : 1.0;
    const double kz = DIM == 3 ? __ldg(T.tK + k * 5 + oc) : 0.0;
    if (DIM == 3 && mz == 0.0 && kz == 0.0) continue;
    const int sz = DIM == 3 ? lz + oc : 0;
#pragma unroll
    for (int ob = 0; ob < 5; ++ob) {
      const double my = __ldg(T.tM + j * 5 + ob), ky = __ldg(T.tK + j * 5 + ob);
      if (my == 0.0 && ky == 0.0) continue;
      const double* wr = &sw[sz][ly + ob][lx];
      const double* ur = &su[sz][ly + ob][lx];
      double rmw = 0, rmu = 0, rku = 0;
#pragma unroll
      for (int oa = 0; oa < 5; ++oa) {
        rmw = fma(mx[oa], wr[oa], rmw);
        rmu = fma(mx[oa], ur[oa], rmu);
        rku = fma(kx[oa], ur[oa], rku);
        if (oseen) CL = fma(__ldg(cv + ((DIM == 3 ? oc * 5 : 0) + ob) * 5 + oa), ur[oa], CL);
      }
      const double mzy = mz * my, kzy = kz * my + mz * ky;
      Mw = fma(mzy, rmw, Mw);
      KL = fma(kzy, rmu, fma(mzy, rku, KL));
    }
  }
  // B^T q from the pressure tile
  double P[DIM][3], Gd[DIM][3];
  int I0[DIM];
  const int cc[3] = {i, j, k};
  const int P0[3] = {P0x, P0y, P0z};
  for (int a = 0; a < DIM; ++a) {
    I0[a] = ((cc[a] - 1 >= 0) ? (cc[a] - 1) / 2 : -1) - P0[a];
    for (int o = 0; o < 3; ++o) {
      P[a][o] = __ldg(T.tPmT + cc[a] * 3 + o);
      Gd[a][o] = __ldg(T.tGmT + cc[a] * 3 + o);
    }
  }
  double BTq = 0;
  for (int oc = 0; oc < (DIM == 3 ? 3 : 1); ++oc) {
    const double fz = DIM == 3 ? (comp == 2 ? Gd[2][oc] : P[2][oc]) : 1.0;
    const int lzq = DIM == 3 ? I0[2] + oc : 0;
#pragma unroll
    for (int ob = 0; ob < 3; ++ob) {
      const double fy = comp == 1 ? Gd[1][ob] : P[1][ob];
#pragma unroll
      for (int oa = 0; oa < 3; ++oa) {
        const double fx = comp == 0 ? Gd[0][oa] : P[0][oa];
        BTq = fma(-fz * fy * fx, sq[lzq][I0[1] + ob][I0[0] + oa], BTq);
      }
    }
  }
  *yo = Mw + tau * (G.nu * KL + CL) + tau * BTq;
}

// pressure rows: half 0 y1p_t = tau B lam_t ; half 1 y2p_t = tau B v_t
template <int DIM>
__global__ void k_kkt_pres(Geo G, KKTTab T, const double* __restrict__ x, double* __restrict__ y) {
  const long node = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= G.n_p) return;
  const int row = blockIdx.y;
  const int h = row / G.n_b, t = row % G.n_b;
  double* yo = y + (long)row * G.nblk + G.n_v + node;
  if (node == 0) {
    *yo = 0.0;
    return;
  }
  const int m1 = G.n1q1, n1 = G.n1q2;
  int c[3];
  c[0] = (int)(node % m1);
  c[1] = (int)((node / m1) % m1);
  c[2] = DIM == 3 ? (int)(node / ((long)m1 * m1)) : 0;
  const double* u = x + (long)(h == 0 ? (G.n_b + t) : t) * G.nblk;
  double Pm[DIM][5], Gm[DIM][5];
  for (int a = 0; a < DIM; ++a)
    for (int o = 0; o < 5; ++o) {
      Pm[a][o] = __ldg(T.tPm + c[a] * 5 + o);
      Gm[a][o] = __ldg(T.tGm + c[a] * 5 + o);
    }
  double acc = 0;
  for (int comp = 0; comp < DIM; ++comp) {
    const double* uc = u + comp * G.n_s;
    for (int oc = 0; oc < (DIM == 3 ? 5 : 1); ++oc) {
      double fz = 1.0;
      int kk = 0;
      if (DIM == 3) {
        fz = comp == 2 ? Gm[2][oc] : Pm[2][oc];
        kk = clampi(2 * c[2] + oc - 2, 0, n1 - 1);
      }
      for (int ob = 0; ob < 5; ++ob) {
        const double fy = comp == 1 ? Gm[1][ob] : Pm[1][ob];
        const int jj = clampi(2 * c[1] + ob - 2, 0, n1 - 1);
#pragma unroll
        for (int oa = 0; oa < 5; ++oa) {
          const double fx = comp == 0 ? Gm[0][oa] : Pm[0][oa];
          const int ii = clampi(2 * c[0] + oa - 2, 0, n1 - 1);
          acc = fma(-fz * fy * fx, __ldg(uc + ((long)kk * n1 + jj) * n1 + ii), acc);
        }
      }
    }
  }
  *yo = G.tau * acc;
}

__global__ void k_mask_copy(Geo G, const double* __restrict__ in, double* __restrict__ out, long N) {
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const long col = i % G.nblk;
  out[i] = col_masked(G, col) ? 0.0 : in[i];
}

// b = tau (M_full v_d)|_interior in the adjoint-velocity rows (half 0), 0 elsewhere
template <int DIM>
__global__ void k_rhs(Geo G, const double* __restrict__ tMf, const double* __restrict__ vd, double* __restrict__ b) {
  const long col = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= G.nblk) return;
  const int row = blockIdx.y;
  double* bo = b + (long)row * G.nblk + col;
  if (row >= G.n_b || col >= G.n_v || col_masked(G, col)) {
    *bo = 0.0;
    return;
  }
  const long comp = col / G.n_s, node = col % G.n_s;
  const int n1 = G.n1q2;
  int c[3];
  c[0] = (int)(node % n1);
  c[1] = (int)((node / n1) % n1);
  c[2] = DIM == 3 ? (int)(node / ((long)n1 * n1)) : 0;
  const double* v = vd + comp * G.n_s;
  double acc = 0;
  for (int oc = 0; oc < (DIM == 3 ? 5 : 1); ++oc) {
    const double fz = DIM == 3 ? tMf[c[2] * 5 + oc] : 1.0;
    const int kk = DIM == 3 ? clampi(c[2] + oc - 2, 0, n1 - 1) : 0;
    for (int ob = 0; ob < 5; ++ob) {
      const double fy = tMf[c[1] * 5 + ob];
      const int jj = clampi(c[1] + ob - 2, 0, n1 - 1);
      for (int oa = 0; oa < 5; ++oa) {
        const double fx = tMf[c[0] * 5 + oa];
        const int ii = clampi(c[0] + oa - 2, 0, n1 - 1);
        acc = fma(fz * fy * fx, v[((long)kk * n1 + jj) * n1 + ii], acc);
      }
    }
  }
  *bo = G.tau * acc;
}

// Right-hand side with time-dependent data and lifting of inhomogeneous Dirichlet data (
// NEXT-2: the paper's manufactured problem).  Row block m = j + 1 (t_m = m tau), component c:
//   adjoint rows (half 0):   tau [M (v_d^m - G^m)]_i
//   state rows   (half 1):   [M (tau f^m - G^m + H^{m-1}) - tau (nu K + N) G^m]_i,  H^0 = v0, H^{m-1} = G^{m-1}
//   divergence rows (half 1): -tau [B G^m]_I  (B = -(int psi d_c phi))
// with G^m = g^m on boundary nodes and 0 inside, all operators un-eliminated (boundary columns kept).
// vd, f: [n_b][d][n_s]; g: [n_b + 1][d][n_s]; v0: [d][n_s]; any may be null (= 0; v0 null -> g^0).
struct RhsData {
  const double *vd, *f, *g, *v0;
  const double *tM, *tK, *tPm, *tGm;   // full 1-D rows
  const double* conv;                  // Oseen: un-eliminated convection stencil per node, or null
};

__device__ __forceinline__ bool q2_boundary(int i, int j, int k, int n1, int dim) {
  bool b = i == 0 || i == n1 - 1 || j == 0 || j == n1 - 1;
  if (dim == 3) b = b || k == 0 || k == n1 - 1;
  return b;
}

template <int DIM>
__global__ void k_rhs_gen(Geo G, RhsData D, double* __restrict__ b) {
  const long col = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= G.nblk) return;
  const int row = blockIdx.y, h = row / G.n_b, j = row % G.n_b, m = j + 1;
  double* bo = b + (long)row * G.nblk + col;
  const int n1 = G.n1q2;
  const long ns = G.n_s;
  auto gb = [&](int mm, int comp, long nd, int ii, int jj, int kk) -> double {   // G^mm (boundary data only)
    return (D.g && q2_boundary(ii, jj, kk, n1, DIM)) ? D.g[((long)mm * G.dim + comp) * ns + nd] : 0.0;
  };
  if (col < G.n_v) {
    const int comp = (int)(col / ns);
    const long node = col % ns;
    int c[3];
    c[0] = (int)(node % n1);
    c[1] = (int)((node / n1) % n1);
    c[2] = DIM == 3 ? (int)(node / ((long)n1 * n1)) : 0;
    if (q2_boundary(c[0], c[1], c[2], n1, DIM)) {
      *bo = 0.0;
      return;
    }
    double accM = 0.0, accK = 0.0;
    for (int oc = 0; oc < (DIM == 3 ? 5 : 1); ++oc) {
      const int kk = DIM == 3 ? c[2] + oc - 2 : 0;
      if (DIM == 3 && (kk < 0 || kk >= n1)) continue;
      const double mz = DIM == 3 ? D.tM[c[2] * 5 + oc] : 1.0, kz = DIM == 3 ? D.tK[c[2] * 5 + oc] : 0.0;
      for (int ob = 0; ob < 5; ++ob) {
        const int jj = c[1] + ob - 2;
        if (jj < 0 || jj >= n1) continue;
        const double my = D.tM[c[1] * 5 + ob], ky = D.tK[c[1] * 5 + ob];
        for (int oa = 0; oa < 5; ++oa) {
          const int ii = c[0] + oa - 2;
          if (ii < 0 || ii >= n1) continue;
          const double mx = D.tM[c[0] * 5 + oa], kx = D.tK[c[0] * 5 + oa];
          const double wm = mz * my * mx;
          const double wk = kz * my * mx + mz * ky * mx + mz * my * kx;
          const long nd = ((long)kk * n1 + jj) * n1 + ii;
          const double Gm = gb(m, comp, nd, ii, jj, kk);
          double w;
          if (h == 0) {
            w = (D.vd ? D.vd[((long)j * G.dim + comp) * ns + nd] : 0.0) - Gm;
          } else {
            const double fm = D.f ? D.f[((long)j * G.dim + comp) * ns + nd] : 0.0;
            const double H = m == 1 ? (D.v0 ? D.v0[(long)comp * ns + nd] : gb(0, comp, nd, ii, jj, kk))
                                    : gb(m - 1, comp, nd, ii, jj, kk);
            w = G.tau * fm - Gm + H;
            accK = fma(wk, Gm, accK);
          }
          accM = fma(wm, w, accM);
        }
      }
    }
    double accN = 0.0;   // Oseen: (N G^m)_i with the un-eliminated stencil (taps (oc, ob, oa), x fastest)
    if (h == 1 && D.conv && D.g) {
      constexpr int NT = DIM == 2 ? 25 : 125;
      const double* cv = D.conv + node * NT;
      for (int t = 0; t < NT; ++t) {
        const int oa = t % 5, ob = (t / 5) % 5, oc = t / 25;
        const int ii = c[0] + oa - 2, jj = c[1] + ob - 2, kk = DIM == 3 ? c[2] + oc - 2 : 0;
        if (ii < 0 || ii >= n1 || jj < 0 || jj >= n1 || kk < 0 || kk >= n1) continue;
        accN = fma(cv[t], gb(m, comp, ((long)kk * n1 + jj) * n1 + ii, ii, jj, kk), accN);
      }
    }
    *bo = h == 0 ? G.tau * accM : accM - G.tau * (G.nu * accK + accN);
    return;
  }
  // pressure rows
  const long pn = col - G.n_v;
  if (h == 0 || pn == 0 || !D.g) {
    *bo = 0.0;
    return;
  }
  const int m1 = G.n1q1;
  int c[3];
  c[0] = (int)(pn % m1);
  c[1] = (int)((pn / m1) % m1);
  c[2] = DIM == 3 ? (int)(pn / ((long)m1 * m1)) : 0;
  double acc = 0.0;   // (B G^m)_I = -sum_c sum (G_c on axis c)(P elsewhere) G^m_c
  for (int comp = 0; comp < DIM; ++comp)
    for (int oc = 0; oc < (DIM == 3 ? 5 : 1); ++oc) {
      const int kk = DIM == 3 ? 2 * c[2] + oc - 2 : 0;
      if (DIM == 3 && (kk < 0 || kk >= n1)) continue;
      const double fz = DIM == 3 ? (comp == 2 ? D.tGm : D.tPm)[c[2] * 5 + oc] : 1.0;
      for (int ob = 0; ob < 5; ++ob) {
        const int jj = 2 * c[1] + ob - 2;
        if (jj < 0 || jj >= n1) continue;
        const double fy = (comp == 1 ? D.tGm : D.tPm)[c[1] * 5 + ob];
        for (int oa = 0; oa < 5; ++oa) {
          const int ii = 2 * c[0] + oa - 2;
          if (ii < 0 || ii >= n1) continue;
          const double fx = (comp == 0 ? D.tGm : D.tPm)[c[0] * 5 + oa];
          const long nd = ((long)kk * n1 + jj) * n1 + ii;
          acc = fma(-fz * fy * fx, gb(m, comp, nd, ii, jj, kk), acc);
        }
      }
    }
  *bo = -G.tau * acc;
}

Geo geo_of(const Ctx& c) {
  Geo g;
  g.dim = c.dim;
  g.n1q2 = c.n1q2;
  g.n1q1 = c.n1q1;
  g.n_b = c.n_b;
  g.n_f = c.n_f;
  g.n_s = c.n_s;
  g.n_v = c.n_v;
  g.n_p = c.n_p;
  g.nblk = c.nblk;
  g.tau = c.tau;
  g.nu = c.nu;
  g.beta = c.beta;
  g.rst = 1.0 / std::sqrt(c.tau);
  return g;
}

InvSrc src_of(const Ctx& c) {
  InvSrc S;
  if (!c.oseen) {
    S.v1 = c.Xv;
    S.v2 = c.Xv + (long)c.dim * c.n_s;
    S.vstride = 2L * c.dim * c.n_s;
    S.pA = c.XpA;
    S.pB = c.XpB;
    S.stokes = 1;
    S.pscale = 0.0;
  } else {
    S.v1 = c.X1;
    S.v2 = c.X2;
    S.vstride = (long)c.dim * c.n_s;
    S.pA = c.XpA;
    S.pB = nullptr;
    S.stokes = 0;
    S.pscale = -1.0 / c.tau;   // (y3, y4) = -S_hat^{-1}(...), with the 1/tau of [[0,tau K_p],[tau K_p,0]]^{-1}
  }
  S.pstride = 2L * c.n_p;
  S.phoff = c.n_p;
  return S;
}

int tile_width(int n_b, int n_f, size_t* smem_fwd, size_t* smem_inv) {
  int TD = 32;
  for (;;) {
    size_t f = (size_t)n_b * 16 + 2ull * n_b * TD * 8;
    size_t i = (size_t)n_b * 16 + 2ull * n_f * TD * 16;
    if ((f <= 160 * 1024 && i <= 160 * 1024) || TD == 8) {
      *smem_fwd = f;
      *smem_inv = i;
      return TD;
    }
    TD /= 2;
  }
}

}  // namespace

namespace {
bool dense_fft_env() {
  static const bool d = std::getenv("AAO_FFT_DENSE") != nullptr;
  return d;
}
// frequencies (forward) / time pairs (inverse) per thread: 1, 2, 4 or 8
int per_thread(int count, int ky) {
  const int need = (count + ky - 1) / ky;
  return need <= 1 ? 1 : (need <= 2 ? 2 : (need <= 4 ? 4 : 8));
}
// tile width for the symmetric kernels: fits shared memory and needs at most 8 outputs per thread
int sym_tile(const Ctx& c, int count, size_t* sf, size_t* si) {
  int TD = tile_width(c.n_b, c.n_f, sf, si);
  // at most 4 outputs per thread on tiles wider than 16 columns (c4_128: TD 32 -> 16, 8 -> 4 outputs per thread,
  // DFT pair 4.53 -> 3.89 ms; profiles/r01_fft_td.log), else at most 8
  while (TD > 8 && (count + 256 / TD - 1) / (256 / TD) > (TD > 16 ? 4 : 8)) TD /= 2;
  *sf = (size_t)c.n_b * 16 + 2ull * c.n_b * TD * 8;
  *si = (size_t)c.n_b * 16 + 2ull * c.n_f * TD * 16;
  return TD;
}
// dense (plain-sum) kernels: on request, or when a 256-thread tile cannot cover the outputs in 8 per thread
bool dense_fft(const Ctx& c) {
  return dense_fft_env() || (c.n_b / 2 + 1 > 8 * 32) || (c.n_f > 8 * 32);
}
void launch_inv_sym(const Ctx& c, const InvSrc& S, double* z, cudaStream_t s) {
  size_t sf, si;
  const int TD = sym_tile(c, c.n_b / 2 + 1, &sf, &si);
  const int KY = 256 / TD;
  const int TB = per_thread(c.n_b / 2 + 1, KY);
  dim3 blk(TD, KY), grd((unsigned)((c.nblk + TD - 1) / TD));
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)si);
    kern<<<grd, blk, si, s>>>(geo_of(c), S, z, c.fc, c.tw, TD);
  };
  if (TB == 1) go(k_fft_inv_sym<1>);
  else if (TB == 2) go(k_fft_inv_sym<2>);
  else if (TB == 4) go(k_fft_inv_sym<4>);
  else go(k_fft_inv_sym<8>);
}
}  // namespace

// prime-factor plan n_b = P Q (gcd 1) for the instantiated pairs; false: the dense symmetric kernels
static bool pfa_plan(int n_b, int* P, int* Q, PfaMap* mp) {
  static const int pairs[][2] = {{7, 73}, {15, 17}, {7, 9}, {3, 5}};
  for (auto& pq : pairs) {
    if (pq[0] * pq[1] != n_b) continue;
    *P = pq[0];
    *Q = pq[1];
    int a = 1, b = 1;
    while ((pq[1] * a) % pq[0] != 1) ++a;   // Q^-1 mod P
    while ((pq[0] * b) % pq[1] != 1) ++b;   // P^-1 mod Q
    mp->QA = pq[1] * a;
    mp->PB = pq[0] * b;
    return true;
  }
  return false;
}
static bool pfa_off() {
  static const bool off = std::getenv("AAO_FFT_DENSE") != nullptr;
  return off;
}
template <int P, int Q>
static void fwd_pfa_t(const Ctx& c, const double* r, PfaMap mp, cudaStream_t s) {
  const size_t sm = Pfa<P, Q>::smem(c.n_f, 1);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_fwd_pfa<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  k_fft_fwd_pfa<P, Q><<<(unsigned)((c.nblk + 15) / 16), Pfa<P, Q>::THREADS, sm, s>>>(geo_of(c), r, c.Fv, c.Fp, c.fc,
                                                                                      c.tw, mp, c.oseen ? 0 : 1);
}
template <int P, int Q>
static void inv_pfa_t(const Ctx& c, const InvSrc& S, double* z, PfaMap mp, cudaStream_t s) {
  const size_t sm = Pfa<P, Q>::smem(c.n_f, 1);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_inv_pfa<P, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  k_fft_inv_pfa<P, Q><<<(unsigned)((c.nblk + 15) / 16), Pfa<P, Q>::THREADS, sm, s>>>(geo_of(c), S, z, c.fc, c.tw, mp);
}
static bool launch_pfa_fwd(const Ctx& c, const double* r, cudaStream_t s) {
  int P, Q;
  PfaMap mp;
  if (pfa_off() || !pfa_plan(c.n_b, &P, &Q, &mp)) return false;
  switch (P * 1000 + Q) {
    case 7073: fwd_pfa_t<7, 73>(c, r, mp, s); break;
    case 15017: fwd_pfa_t<15, 17>(c, r, mp, s); break;
    case 7009: fwd_pfa_t<7, 9>(c, r, mp, s); break;
    default: fwd_pfa_t<3, 5>(c, r, mp, s); break;
  }
  return true;
}
static bool launch_pfa_inv(const Ctx& c, const InvSrc& S, double* z, cudaStream_t s) {
  int P, Q;
  PfaMap mp;
  if (pfa_off() || !pfa_plan(c.n_b, &P, &Q, &mp)) return false;
  switch (P * 1000 + Q) {
    case 7073: inv_pfa_t<7, 73>(c, S, z, mp, s); break;
    case 15017: inv_pfa_t<15, 17>(c, S, z, mp, s); break;
    case 7009: inv_pfa_t<7, 9>(c, S, z, mp, s); break;
    default: inv_pfa_t<3, 5>(c, S, z, mp, s); break;
  }
  return true;
}

void launch_fft_fwd(const Ctx& c, const double* r, cudaStream_t s) {
  if (launch_pfa_fwd(c, r, s)) return;
  size_t sf, si;
  const int TD = tile_width(c.n_b, c.n_f, &sf, &si);
  dim3 blk(TD, 256 / TD);
  dim3 grd((unsigned)((c.nblk + TD - 1) / TD));
  if (dense_fft(c)) {
    cudaFuncSetAttribute(k_fft_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
    k_fft_fwd<<<grd, blk, sf, s>>>(geo_of(c), r, c.Fv, c.Fp, c.fc, c.tw, TD, c.oseen ? 0 : 1);
    return;
  }
  const int TDs = sym_tile(c, c.n_f, &sf, &si);
  const int KB = per_thread(c.n_f, 256 / TDs);
  blk = dim3(TDs, 256 / TDs);
  grd = dim3((unsigned)((c.nblk + TDs - 1) / TDs));
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
    kern<<<grd, blk, sf, s>>>(geo_of(c), r, c.Fv, c.Fp, c.fc, c.tw, TDs, c.oseen ? 0 : 1);
  };
  if (KB == 1) go(k_fft_fwd_sym<1>);
  else if (KB == 2) go(k_fft_fwd_sym<2>);
  else if (KB == 4) go(k_fft_fwd_sym<4>);
  else go(k_fft_fwd_sym<8>);
}

void launch_fft_inv(const Ctx& c, double* z, cudaStream_t s) {
  if (launch_pfa_inv(c, src_of(c), z, s)) return;
  if (!dense_fft(c)) {
    launch_inv_sym(c, src_of(c), z, s);
    return;
  }
  size_t sf, si;
  const int TD = tile_width(c.n_b, c.n_f, &sf, &si);
  cudaFuncSetAttribute(k_fft_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)si);
  dim3 blk(TD, 256 / TD);
  dim3 grd((unsigned)((c.nblk + TD - 1) / TD));
  k_fft_inv<<<grd, blk, si, s>>>(geo_of(c), src_of(c), z, c.fc, c.tw, TD);
}

InvSrc src_of_fvec(const Ctx& c, FVec x) {
  InvSrc S;
  S.v1 = x.v;
  S.v2 = x.v + (long)c.dim * c.n_s;
  S.vstride = 2L * c.dim * c.n_s;
  S.pA = x.p;
  S.pB = nullptr;
  S.pstride = 2L * c.n_p;
  S.phoff = c.n_p;
  S.stokes = c.oseen ? 0 : 1;
  S.pscale = 1.0;
  return S;
}

void launch_debug_block(const Ctx& c, int k, double2* out, cudaStream_t s) {
  const InvSrc S = c.debug_block_src_v ? src_of_fvec(c, FVec{c.debug_block_src_v, c.debug_block_src_p}) : src_of(c);
  k_debug_block<<<(unsigned)((c.nblk + 255) / 256), 256, 0, s>>>(geo_of(c), S, c.fc, k, out);
}

void launch_fft_inv_from(const Ctx& c, FVec x, double* z, cudaStream_t s) {
  if (launch_pfa_inv(c, src_of_fvec(c, x), z, s)) return;
  if (!dense_fft(c)) {
    launch_inv_sym(c, src_of_fvec(c, x), z, s);
    return;
  }
  size_t sf, si;
  const int TD = tile_width(c.n_b, c.n_f, &sf, &si);
  cudaFuncSetAttribute(k_fft_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)si);
  dim3 blk(TD, 256 / TD);
  dim3 grd((unsigned)((c.nblk + TD - 1) / TD));
  k_fft_inv<<<grd, blk, si, s>>>(geo_of(c), src_of_fvec(c, x), z, c.fc, c.tw, TD);
}

void launch_kkt(const Ctx& c, const double* x, double* y, cudaStream_t s) {
  if (launch_kkt_march(c, x, y, s)) return;   // 2-D: time-marching kernel (kernels_kkt.cu)
  KKTTab T;
  T.tM = c.vel.grids[0].tM;
  T.tK = c.vel.grids[0].tK;
  T.conv = c.vel.grids[0].conv;
  T.convT = c.vel.grids[0].convT;
  T.tPmT = c.tPmT;
  T.tGmT = c.tGmT;
  T.tPm = c.tPm;
  T.tGm = c.tGm;
  const Geo G = geo_of(c);
  dim3 gp((unsigned)((c.n_p + 127) / 128), 2 * c.n_b);
  if (c.dim == 2) {
    const int tx = (c.n1q2 + KT<2>::TX - 1) / KT<2>::TX, ty = (c.n1q2 + KT<2>::TY - 1) / KT<2>::TY;
    k_kkt_vel_tiled<2><<<dim3(tx * ty, 2 * c.n_b, 2), 256, 0, s>>>(G, T, x, y, c.oseen ? 1 : 0, tx, ty);
    k_kkt_pres<2><<<gp, 128, 0, s>>>(G, T, x, y);
  } else {
    const int tx = (c.n1q2 + KT<3>::TX - 1) / KT<3>::TX, ty = (c.n1q2 + KT<3>::TY - 1) / KT<3>::TY;
    const int tz = (c.n1q2 + KT<3>::TZ - 1) / KT<3>::TZ;
    k_kkt_vel_tiled<3><<<dim3(tx * ty * tz, 2 * c.n_b, 3), 256, 0, s>>>(G, T, x, y, c.oseen ? 1 : 0, tx, ty);
    k_kkt_pres<3><<<gp, 128, 0, s>>>(G, T, x, y);
  }
}

void launch_mask_copy(const Ctx& c, const double* in, double* out, cudaStream_t s) {
  k_mask_copy<<<(unsigned)((c.N + 255) / 256), 256, 0, s>>>(geo_of(c), in, out, c.N);
}

void launch_rhs_general(const Ctx& c, const double* vd, const double* f, const double* g, const double* v0, double* b,
                        cudaStream_t s) {
  RhsData D{vd, f, g, v0, c.tMfull, c.tKfull, c.tPmfull, c.tGmfull, c.oseen ? c.convFull : nullptr};
  dim3 grd((unsigned)((c.nblk + 127) / 128), 2 * c.n_b);
  if (c.dim == 2)
    k_rhs_gen<2><<<grd, 128, 0, s>>>(geo_of(c), D, b);
  else
    k_rhs_gen<3><<<grd, 128, 0, s>>>(geo_of(c), D, b);
}

void launch_rhs(const Ctx& c, const double* vd, double* b, cudaStream_t s) {
  dim3 g((unsigned)((c.nblk + 127) / 128), 2 * c.n_b);
  if (c.dim == 2)
    k_rhs<2><<<g, 128, 0, s>>>(geo_of(c), c.tMfull, vd, b);
  else
    k_rhs<3><<<g, 128, 0, s>>>(geo_of(c), c.tMfull, vd, b);
}

}  // namespace aao
