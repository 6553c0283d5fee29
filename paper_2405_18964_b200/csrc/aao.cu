// C-ABI library: setup (step A9), KKT apply (A2), Algorithm-1 preconditioner (A3-A8)
// and GMRES (A1) for the all-at-once Stokes/Oseen control system of arXiv 2405.18964.
// See include/aao.h for the contract and DESIGN.md for the design.
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <stdexcept>

#include "aao_internal.h"

using cplx = std::complex<double>;

namespace aao {

long& launch_counter() {
  static long c = 0;
  return c;
}

namespace {

struct CudaError : std::runtime_error {
  aao_status st;
  CudaError(aao_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw CudaError(e_ == cudaErrorMemoryAllocation ? AAO_ERR_OOM : AAO_ERR_CUDA,           \
                      std::string(#call) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

template <class T>
T* dalloc(Ctx& c, size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(&p, count * sizeof(T));
  if (e != cudaSuccess) throw CudaError(AAO_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  c.allocs.push_back(p);
  c.bytes += count * sizeof(T);
  return static_cast<T*>(p);
}

template <class T>
T* upload(Ctx& c, const std::vector<T>& h) {
  T* d = dalloc<T>(c, h.size());
  CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

// ------------------------------------------------------------------ 1-D finite elements
// 3-point Gauss-Legendre on [0,1]; quadratic (nodes 0, 1/2, 1) and linear Lagrange bases.
struct Ref1D {
  double gp[3], gw[3];
  double phi[3][3], dphi[3][3];  // [basis][point]
  double psi[2][3], dpsi[2][3];
  double m2[3][3], k2[3][3], m1[2][2], k1[2][2], pm[2][3], gm[2][3];
  Ref1D() {
    const double s = std::sqrt(3.0 / 5.0);
    const double xi[3] = {-s, 0.0, s}, w[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
    for (int q = 0; q < 3; ++q) {
      gp[q] = 0.5 * (xi[q] + 1.0);
      gw[q] = 0.5 * w[q];
      const double x = gp[q];
      phi[0][q] = 2 * (x - 0.5) * (x - 1);
      phi[1][q] = 4 * x * (1 - x);
      phi[2][q] = 2 * x * (x - 0.5);
      dphi[0][q] = 4 * x - 3;
      dphi[1][q] = 4 - 8 * x;
      dphi[2][q] = 4 * x - 1;
      psi[0][q] = 1 - x;
      psi[1][q] = x;
      dpsi[0][q] = -1;
      dpsi[1][q] = 1;
    }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        m2[i][j] = k2[i][j] = 0;
        for (int q = 0; q < 3; ++q) {
          m2[i][j] += gw[q] * phi[i][q] * phi[j][q];
          k2[i][j] += gw[q] * dphi[i][q] * dphi[j][q];
        }
      }
    for (int i = 0; i < 2; ++i) {
      for (int j = 0; j < 2; ++j) {
        m1[i][j] = k1[i][j] = 0;
        for (int q = 0; q < 3; ++q) {
          m1[i][j] += gw[q] * psi[i][q] * psi[j][q];
          k1[i][j] += gw[q] * dpsi[i][q] * dpsi[j][q];
        }
      }
      for (int j = 0; j < 3; ++j) {
        pm[i][j] = gm[i][j] = 0;
        for (int q = 0; q < 3; ++q) {
          pm[i][j] += gw[q] * psi[i][q] * phi[j][q];
          gm[i][j] += gw[q] * psi[i][q] * dphi[j][q];
        }
      }
    }
  }
};

// assembled 1-D rows on N cells of width h
struct Tables1D {
  std::vector<double> M2, K2, M2full, K2full, M1, K1, Pm, Gm, Pmfull, Gmfull, PmT, GmT;
};

Tables1D tables_1d(const Ref1D& R, int N, double h) {
  Tables1D T;
  const int n1 = 2 * N + 1, m1 = N + 1;
  T.M2.assign(n1 * 5, 0.0);
  T.K2.assign(n1 * 5, 0.0);
  for (int e = 0; e < N; ++e)
    for (int li = 0; li < 3; ++li)
      for (int lj = 0; lj < 3; ++lj) {
        const int i = 2 * e + li, j = 2 * e + lj;
        T.M2[i * 5 + (j - i + 2)] += h * R.m2[li][lj];
        T.K2[i * 5 + (j - i + 2)] += R.k2[li][lj] / h;
      }
  T.M2full = T.M2;
  T.K2full = T.K2;
  for (int i = 0; i < n1; ++i)
    for (int o = 0; o < 5; ++o) {
      const int j = i + o - 2;
      if (j <= 0 || j >= n1 - 1) {  // Dirichlet columns eliminated (and out of range)
        T.M2[i * 5 + o] = 0.0;
        T.K2[i * 5 + o] = 0.0;
      }
      if (j < 0 || j > n1 - 1) T.M2full[i * 5 + o] = T.K2full[i * 5 + o] = 0.0;
    }
  T.M1.assign(m1 * 3, 0.0);
  T.K1.assign(m1 * 3, 0.0);
  for (int e = 0; e < N; ++e)
    for (int li = 0; li < 2; ++li)
      for (int lj = 0; lj < 2; ++lj) {
        const int i = e + li, j = e + lj;
        T.M1[i * 3 + (j - i + 1)] += h * R.m1[li][lj];
        T.K1[i * 3 + (j - i + 1)] += R.k1[li][lj] / h;
      }
  // B rows: Q1 node I, Q2 columns 2I-2..2I+2
  T.Pm.assign(m1 * 5, 0.0);
  T.Gm.assign(m1 * 5, 0.0);
  for (int e = 0; e < N; ++e)
    for (int li = 0; li < 2; ++li)
      for (int lj = 0; lj < 3; ++lj) {
        const int I = e + li, j = 2 * e + lj;
        T.Pm[I * 5 + (j - 2 * I + 2)] += h * R.pm[li][lj];
        T.Gm[I * 5 + (j - 2 * I + 2)] += R.gm[li][lj];
      }
  T.Pmfull = T.Pm;   // boundary (Dirichlet) Q2 columns kept: lifting of boundary data (aao_build_rhs_general)
  T.Gmfull = T.Gm;
  for (int I = 0; I < m1; ++I)
    for (int o = 0; o < 5; ++o) {
      const int j = 2 * I + o - 2;
      if (j <= 0 || j >= n1 - 1) T.Pm[I * 5 + o] = T.Gm[I * 5 + o] = 0.0;
      if (j < 0 || j > n1 - 1) T.Pmfull[I * 5 + o] = T.Gmfull[I * 5 + o] = 0.0;
    }
  T.PmT.assign(n1 * 3, 0.0);
  T.GmT.assign(n1 * 3, 0.0);
  for (int i = 0; i < n1; ++i) {
    const int I0 = i >= 1 ? (i - 1) / 2 : -1;
    for (int o = 0; o < 3; ++o) {
      const int I = I0 + o;
      if (I < 0 || I >= m1) continue;
      const int off = i - 2 * I + 2;
      if (off < 0 || off > 4) continue;
      T.PmT[i * 3 + o] = T.Pm[I * 5 + off];
      T.GmT[i * 3 + o] = T.Gm[I * 5 + off];
    }
  }
  return T;
}

// prolongation tables, coarse N cells -> fine 2N cells (nodal interpolation; DESIGN.md reading)
void transfer_1d(const Ref1D&, int Nc, int order, std::vector<double>& tP, std::vector<double>& tR) {
  const int nf = order * 2 * Nc + 1, nc = order * Nc + 1;
  std::vector<double> P((size_t)nf * nc, 0.0);
  tP.assign((size_t)nf * 4, 0.0);
  for (int f = 0; f < nf; ++f) {
    const double x = f / (2.0 * order);
    int e = (int)std::floor(x);
    if (e > Nc - 1) e = Nc - 1;
    const double xi = x - e;
    double w[3];
    if (order == 2) {
      w[0] = 2 * (xi - 0.5) * (xi - 1);
      w[1] = 4 * xi * (1 - xi);
      w[2] = 2 * xi * (xi - 0.5);
    } else {
      w[0] = 1 - xi;
      w[1] = xi;
      w[2] = 0;
    }
    for (int a = 0; a < 3; ++a)
      if (std::fabs(w[a]) < 1e-15) w[a] = 0.0;
    tP[f * 4 + 0] = order * e;
    for (int a = 0; a <= order; ++a) {
      tP[f * 4 + 1 + a] = w[a];
      P[(size_t)f * nc + order * e + a] += w[a];
    }
  }
  tR.assign((size_t)nc * 7, 0.0);
  for (int I = 0; I < nc; ++I)
    for (int o = 0; o < 7; ++o) {
      const int f = 2 * I + o - 3;
      if (f < 0 || f >= nf) continue;
      tR[I * 7 + o] = P[(size_t)f * nc + I];
    }
}

// convection stencils N_ij = int phi_i (w_h . grad phi_j) by an element loop (3^d Gauss points)
// on the Q2 space (order 2) or Q1 space (order 1) with the Q2 nodal wind of the level.
void convection(const Ref1D& R, int dim, int N, double h, int order, const std::vector<double>& wind,
                std::vector<double>& conv, std::vector<double>& convT, std::vector<double>* conv_full = nullptr) {
  const int n1q2 = 2 * N + 1;
  const long ns = (long)std::pow(n1q2, dim);
  const int n1 = order * N + 1, W = 2 * order + 1, nl1 = order + 1;
  const long n = (long)std::pow(n1, dim);
  const int NS = (int)std::pow(W, dim);
  const int nloc = (int)std::pow(nl1, dim), nq = (int)std::pow(3, dim), nw = (int)std::pow(3, dim);
  // reference basis at tensor Gauss points
  std::vector<double> bv(nloc * nq), bg(nloc * nq * dim), wv(nw * nq), wq(nq);
  for (int q = 0; q < nq; ++q) {
    int qa[3] = {q % 3, (q / 3) % 3, q / 9};
    wq[q] = 1.0;
    for (int a = 0; a < dim; ++a) wq[q] *= R.gw[qa[a]];
    for (int l = 0; l < nloc; ++l) {
      int la[3] = {l % nl1, (l / nl1) % nl1, l / (nl1 * nl1)};
      double v = 1.0;
      for (int a = 0; a < dim; ++a) v *= order == 2 ? R.phi[la[a]][qa[a]] : R.psi[la[a]][qa[a]];
      bv[l * nq + q] = v;
      for (int c = 0; c < dim; ++c) {
        double g = 1.0;
        for (int a = 0; a < dim; ++a) {
          const double val = order == 2 ? (a == c ? R.dphi[la[a]][qa[a]] : R.phi[la[a]][qa[a]])
                                        : (a == c ? R.dpsi[la[a]][qa[a]] : R.psi[la[a]][qa[a]]);
          g *= val;
        }
        bg[(l * nq + q) * dim + c] = g;
      }
    }
    for (int l = 0; l < nw; ++l) {
      int la[3] = {l % 3, (l / 3) % 3, l / 9};
      double v = 1.0;
      for (int a = 0; a < dim; ++a) v *= R.phi[la[a]][qa[a]];
      wv[l * nq + q] = v;
    }
  }
  conv.assign((size_t)n * NS, 0.0);
  const long E = (long)std::pow(N, dim);
  const double scale = std::pow(h, dim - 1);
  std::vector<double> wc(nq * dim);
  for (long e = 0; e < E; ++e) {
    int ec[3] = {(int)(e % N), (int)((e / N) % N), (int)(e / ((long)N * N))};
    for (int q = 0; q < nq; ++q)
      for (int c = 0; c < dim; ++c) {
        double s = 0;
        for (int l = 0; l < nw; ++l) {
          int la[3] = {l % 3, (l / 3) % 3, l / 9};
          long g = 0, st = 1;
          for (int a = 0; a < dim; ++a) {
            g += (2 * ec[a] + la[a]) * st;
            st *= n1q2;
          }
          s += wind[(size_t)c * ns + g] * wv[l * nq + q];
        }
        wc[q * dim + c] = s;
      }
    for (int i = 0; i < nloc; ++i) {
      int ia[3] = {i % nl1, (i / nl1) % nl1, i / (nl1 * nl1)};
      long gi = 0, st = 1;
      for (int a = 0; a < dim; ++a) {
        gi += (order * ec[a] + ia[a]) * st;
        st *= n1;
      }
      for (int j = 0; j < nloc; ++j) {
        int ja[3] = {j % nl1, (j / nl1) % nl1, j / (nl1 * nl1)};
        double val = 0;
        for (int q = 0; q < nq; ++q) {
          double adv = 0;
          for (int c = 0; c < dim; ++c) adv += wc[q * dim + c] * bg[(j * nq + q) * dim + c];
          val += wq[q] * bv[i * nq + q] * adv;
        }
        int off = 0, sw = 1;
        for (int a = 0; a < dim; ++a) {
          off += (ja[a] - ia[a] + order) * sw;
          sw *= W;
        }
        conv[(size_t)gi * NS + off] += scale * val;
      }
    }
  }
  if (conv_full) *conv_full = conv;   // un-eliminated (boundary columns kept): lifting of Dirichlet data
  // eliminate: rows/columns of masked nodes (Dirichlet boundary for Q2, pinned node 0 for Q1)
  auto is_masked = [&](long node) {
    if (order == 1) return node == 0;
    long t = node;
    for (int a = 0; a < dim; ++a) {
      const int ca = (int)(t % n1);
      t /= n1;
      if (ca == 0 || ca == n1 - 1) return true;
    }
    return false;
  };
  for (long i = 0; i < n; ++i) {
    int ia[3] = {(int)(i % n1), (int)((i / n1) % n1), (int)(i / ((long)n1 * n1))};
    const bool mi = is_masked(i);
    for (int o = 0; o < NS; ++o) {
      int oa[3] = {o % W, (o / W) % W, o / (W * W)};
      long j = 0, st = 1;
      bool inr = true;
      for (int a = 0; a < dim; ++a) {
        const int ja = ia[a] + oa[a] - order;
        if (ja < 0 || ja >= n1) inr = false;
        j += ja * st;
        st *= n1;
      }
      if (mi || !inr || is_masked(j)) conv[(size_t)i * NS + o] = 0.0;
    }
  }
  convT.assign((size_t)n * NS, 0.0);
  for (long i = 0; i < n; ++i) {
    int ia[3] = {(int)(i % n1), (int)((i / n1) % n1), (int)(i / ((long)n1 * n1))};
    for (int o = 0; o < NS; ++o) {
      int oa[3] = {o % W, (o / W) % W, o / (W * W)};
      long j = 0, st = 1;
      bool inr = true;
      int oT = 0, sw = 1;
      for (int a = 0; a < dim; ++a) {
        const int ja = ia[a] + oa[a] - order;
        if (ja < 0 || ja >= n1) inr = false;
        j += ja * st;
        st *= n1;
        oT += (2 * order - oa[a]) * sw;
        sw *= W;
      }
      if (inr) convT[(size_t)i * NS + o] = conv[(size_t)j * NS + oT];
    }
  }
}

// dense operator a M + b K + c C on the unknowns of a (small) grid, host evaluation of the stencil
std::vector<cplx> dense_coarse(int dim, int order, int n1, const std::vector<double>& tM, const std::vector<double>& tK,
                               const std::vector<double>* conv, cplx a, cplx b, cplx c, const std::vector<int>& unk) {
  const int W = 2 * order + 1, NS = (int)std::pow(W, dim);
  const int nu = (int)unk.size();
  std::vector<cplx> A((size_t)nu * nu, 0.0);
  for (int r = 0; r < nu; ++r) {
    const int gi = unk[r];
    int ia[3] = {gi % n1, (gi / n1) % n1, gi / (n1 * n1)};
    for (int s = 0; s < nu; ++s) {
      const int gj = unk[s];
      int ja[3] = {gj % n1, (gj / n1) % n1, gj / (n1 * n1)};
      bool ok = true;
      int oa[3];
      for (int x = 0; x < dim; ++x) {
        oa[x] = ja[x] - ia[x] + order;
        if (oa[x] < 0 || oa[x] >= W) ok = false;
      }
      if (!ok) continue;
      double m = 1.0, k = 0.0;
      for (int x = 0; x < dim; ++x) m *= tM[ia[x] * W + oa[x]];
      for (int x = 0; x < dim; ++x) {
        double t = tK[ia[x] * W + oa[x]];
        for (int y = 0; y < dim; ++y)
          if (y != x) t *= tM[ia[y] * W + oa[y]];
        k += t;
      }
      cplx v = a * m + b * k;
      if (conv) {
        int off = 0, sw = 1;
        for (int x = 0; x < dim; ++x) {
          off += oa[x] * sw;
          sw *= W;
        }
        v += c * (*conv)[(size_t)gi * NS + off];
      }
      A[(size_t)r * nu + s] = v;
    }
  }
  return A;
}

// Gauss-Jordan inverse with partial pivoting
bool invert(std::vector<cplx>& A, int n) {
  std::vector<cplx> I((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) I[(size_t)i * n + i] = 1.0;
  double amax = 0;
  for (auto& v : A) amax = std::max(amax, std::abs(v));
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::abs(A[(size_t)r * n + col]) > std::abs(A[(size_t)piv * n + col])) piv = r;
    if (std::abs(A[(size_t)piv * n + col]) <= 1e-14 * amax) return false;
    if (piv != col)
      for (int j = 0; j < n; ++j) {
        std::swap(A[(size_t)piv * n + j], A[(size_t)col * n + j]);
        std::swap(I[(size_t)piv * n + j], I[(size_t)col * n + j]);
      }
    const cplx p = A[(size_t)col * n + col];
    for (int j = 0; j < n; ++j) {
      A[(size_t)col * n + j] /= p;
      I[(size_t)col * n + j] /= p;
    }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const cplx f = A[(size_t)r * n + col];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        A[(size_t)r * n + j] -= f * A[(size_t)col * n + j];
        I[(size_t)r * n + j] -= f * I[(size_t)col * n + j];
      }
    }
  }
  A = I;
  return true;
}

inline double2 d2(cplx z) { return make_double2(z.real(), z.imag()); }
inline Coef coef(cplx a, cplx b, cplx c) { return Coef{d2(a), d2(b), d2(c)}; }

struct HostLevel {
  int N;
  double h;
  Tables1D t;
  std::vector<double> wind, conv, convT;    // Q2 (Oseen)
};

// ------------------------------------------------------------------ setup
void setup(Ctx& c, const aao_config& cfg) {
  c.cfg = cfg;
  c.dim = cfg.dim;
  c.Nc = cfg.n_cells;
  c.n_t = cfg.n_t;
  c.n_b = cfg.n_t - 1;
  c.n_f = c.n_b / 2 + 1;
  c.tau = cfg.T / cfg.n_t;
  c.beta = cfg.beta;
  c.nu = cfg.nu;
  c.oseen = cfg.problem == AAO_OSEEN;
  c.n1q2 = 2 * c.Nc + 1;
  c.n1q1 = c.Nc + 1;
  c.n_s = (long)std::pow(c.n1q2, c.dim);
  c.n_p = (long)std::pow(c.n1q1, c.dim);
  c.n_v = c.dim * c.n_s;
  c.nblk = c.n_v + c.n_p;
  c.N = 2L * c.n_b * c.nblk;
  const int dim = c.dim;
  const Ref1D R;

  // levels N_c, N_c/2, ..., 2 (reading C.2 #12)
  std::vector<HostLevel> L;
  for (int N = c.Nc; N >= 2; N /= 2) {
    HostLevel hl;
    hl.N = N;
    hl.h = (cfg.x_hi - cfg.x_lo) / N;
    hl.t = tables_1d(R, N, hl.h);
    L.push_back(std::move(hl));
  }
  const int nlev = (int)L.size();
  if (c.oseen) {
    L[0].wind.assign(cfg.wind_q2, cfg.wind_q2 + (size_t)dim * c.n_s);
    for (int l = 1; l < nlev; ++l) {  // injection: coarse node I <-> fine node 2I
      const int nf1 = 2 * L[l - 1].N + 1, nc1 = 2 * L[l].N + 1;
      const long ncn = (long)std::pow(nc1, dim), nfn = (long)std::pow(nf1, dim);
      L[l].wind.assign((size_t)dim * ncn, 0.0);
      for (long I = 0; I < ncn; ++I) {
        long f = 0, st = 1, t = I;
        for (int a = 0; a < dim; ++a) {
          f += 2 * (t % nc1) * st;
          t /= nc1;
          st *= nf1;
        }
        for (int comp = 0; comp < dim; ++comp) L[l].wind[(size_t)comp * ncn + I] = L[l - 1].wind[(size_t)comp * nfn + f];
      }
    }
    std::vector<double> conv_full;
    for (int l = 0; l < nlev; ++l)
      convection(R, dim, L[l].N, L[l].h, 2, L[l].wind, L[l].conv, L[l].convT, l == 0 ? &conv_full : nullptr);
    c.convFull = upload(c, conv_full);
  }

  // MG spaces
  for (int sp = 0; sp < 2; ++sp) {
    MGSpace& S = sp == 0 ? c.vel : c.pres;
    const int order = sp == 0 ? 2 : 1;
    S.order = order;
    S.nlev = nlev;
    S.grids.resize(nlev);
    S.transfers.resize(nlev);
    for (int l = 0; l < nlev; ++l) {
      Grid& g = S.grids[l];
      g.dim = dim;
      g.order = order;
      g.n1 = order * L[l].N + 1;
      g.n = (long)std::pow(g.n1, dim);
      g.tM = upload(c, order == 2 ? L[l].t.M2 : L[l].t.M1);
      g.tK = upload(c, order == 2 ? L[l].t.K2 : L[l].t.K1);
      g.conv = g.convT = nullptr;
      if (order == 2 && c.oseen) {
        g.conv = upload(c, L[l].conv);
        g.convT = upload(c, L[l].convT);
      }
      if (l + 1 < nlev) {
        std::vector<double> tP, tR;
        transfer_1d(R, L[l + 1].N, order, tP, tR);
        S.transfers[l].tP = upload(c, tP);
        S.transfers[l].tR = upload(c, tR);
      }
    }
    // coarsest-level unknowns
    const Grid& gc = S.grids[nlev - 1];
    std::vector<int> unk;
    for (long i = 0; i < gc.n; ++i) {
      bool m;
      if (order == 1) {
        m = i == 0;
      } else {
        m = false;
        long t = i;
        for (int a = 0; a < dim; ++a) {
          const int ca = (int)(t % gc.n1);
          t /= gc.n1;
          m = m || ca == 0 || ca == gc.n1 - 1;
        }
      }
      if (!m) unk.push_back((int)i);
    }
    S.ncoarse_unk = (int)unk.size();
    S.coarse_unk = upload(c, unk);
  }
  // fine pressure convection (Oseen Schur complement)
  if (c.oseen) {
    std::vector<double> cp, cpT;
    convection(R, dim, c.Nc, L[0].h, 1, L[0].wind, cp, cpT);
    c.pres.grids[0].conv = upload(c, cp);
    c.pres.grids[0].convT = upload(c, cpT);
  }
  c.tPm = upload(c, L[0].t.Pm);
  c.tGm = upload(c, L[0].t.Gm);
  c.tPmT = upload(c, L[0].t.PmT);
  c.tGmT = upload(c, L[0].t.GmT);
  c.tMfull = upload(c, L[0].t.M2full);
  c.tKfull = upload(c, L[0].t.K2full);
  c.tPmfull = upload(c, L[0].t.Pmfull);
  c.tGmfull = upload(c, L[0].t.Gmfull);
  c.h_M2 = L[0].t.M2;
  c.h_K2 = L[0].t.K2;
  c.h_Pm = L[0].t.Pm;
  c.h_Gm = L[0].t.Gm;
  c.h_PmT = L[0].t.PmT;
  c.h_GmT = L[0].t.GmT;

  // frequency constants: d_k = 1 - exp(-2 pi i k / n_b) (reading C.2 #2)
  const int n_f = c.n_f, n_b = c.n_b;
  const double tau = c.tau, beta = c.beta, nu = c.nu;
  std::vector<cplx> d(n_f);
  c.fch.resize(n_f);
  for (int k = 0; k < n_f; ++k) {
    const double th = 2.0 * M_PI * (double)k / n_b;
    d[k] = cplx(1.0 - std::cos(th), std::sin(th));
    FreqConst& f = c.fch[k];
    f.dr = d[k].real();
    f.dc = d[k].imag();
    f.c1 = f.dr / std::sqrt(tau * tau / beta + f.dc * f.dc);       // squared reading (C.2 #1)
    f.c2 = 1.0 / std::sqrt(1.0 / beta + f.dc * f.dc / (tau * tau));
    f.rc2 = 1.0 / f.c2;
  }
  c.fc = upload(c, c.fch);
  std::vector<double2> tw(n_b);
  for (int m = 0; m < n_b; ++m) {
    const double th = 2.0 * M_PI * (double)m / n_b;
    tw[m] = make_double2(std::cos(th), std::sin(th));
  }
  c.tw = upload(c, tw);

  // coefficient tables and coarse inverses
  const Grid& gv = c.vel.grids[nlev - 1];
  const Grid& gp = c.pres.grids[nlev - 1];
  std::vector<int> unk_v(c.vel.ncoarse_unk), unk_p(c.pres.ncoarse_unk);
  CK(cudaMemcpy(unk_v.data(), c.vel.coarse_unk, unk_v.size() * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(unk_p.data(), c.pres.coarse_unk, unk_p.size() * sizeof(int), cudaMemcpyDeviceToHost));
  const HostLevel& LC = L[nlev - 1];
  auto inv_of = [&](int order, cplx a, cplx b, cplx cc, const std::vector<double>* conv, const std::vector<int>& unk) {
    const Tables1D& t = LC.t;
    std::vector<cplx> A = dense_coarse(dim, order, order == 2 ? gv.n1 : gp.n1, order == 2 ? t.M2 : t.M1,
                                       order == 2 ? t.K2 : t.K1, conv, a, b, cc, unk);
    if (!invert(A, (int)unk.size())) throw CudaError(AAO_ERR_NUMERIC, "singular coarse-grid matrix");
    std::vector<double2> out(A.size());
    for (size_t i = 0; i < A.size(); ++i) out[i] = d2(A[i]);
    return out;
  };
  auto append = [](std::vector<double2>& dst, const std::vector<double2>& src) {
    dst.insert(dst.end(), src.begin(), src.end());
  };
  c.coefKp = upload(c, std::vector<Coef>{coef(0.0, 1.0, 0.0)});
  c.coefMass = upload(c, std::vector<Coef>{coef(1.0, 0.0, 0.0)});
  c.coefNegMass = upload(c, std::vector<Coef>{coef(-1.0, 0.0, 0.0)});
  c.invKp = upload(c, inv_of(1, 0.0, 1.0, 0.0, nullptr, unk_p));
  if (!c.oseen) {
    std::vector<Coef> cw(n_f);
    std::vector<double2> iw;
    for (int k = 0; k < n_f; ++k) {
      // W_k = (1 + c_{k,1}) M + c_{k,2} L, L = nu K
      const cplx a = 1.0 + c.fch[k].c1, b = c.fch[k].c2 * nu;
      cw[k] = coef(a, b, 0.0);
      append(iw, inv_of(2, a, b, 0.0, nullptr, unk_v));
    }
    c.coefW = upload(c, cw);
    c.invW = upload(c, iw);
    std::vector<Coef> zx(n_f);
    for (int k = 0; k < n_f; ++k) zx[k] = coef(c.fch[k].c1, c.fch[k].c2 * nu, 0.0);   // X = c1 M + c2 L
    c.coefZX = upload(c, zx);
  } else {
    // Q_k = d_k M + tau L + (tau/sqrt(beta)) M, L = nu K + N; Q_k^H uses N^T
    std::vector<Coef> cq(n_f), cqh(n_f), u2(n_f), u3(n_f), s2(n_f), s3(n_f);
    std::vector<double2> iq, iqh;
    const double sb = tau / std::sqrt(beta);
    for (int k = 0; k < n_f; ++k) {
      const cplx sh = d[k] + sb;
      cq[k] = coef(sh, tau * nu, tau);
      cqh[k] = coef(std::conj(sh), tau * nu, tau);
      append(iq, inv_of(2, sh, tau * nu, tau, &LC.conv, unk_v));
      append(iqh, inv_of(2, std::conj(sh), tau * nu, tau, &LC.convT, unk_v));
      u2[k] = coef(-std::conj(d[k]), -tau * nu, -tau);   // -(d^* M + tau L^T)       (Uzawa x1 update)
      u3[k] = coef(-d[k], -tau * nu, -tau);              // -(d M + tau L)           (Uzawa x2 update)
      s2[k] = coef(std::conj(d[k]), tau * nu, tau);      // d^* M_p + tau L_p^T      (Schur middle block)
      s3[k] = coef(d[k], tau * nu, tau);                 // d M_p + tau L_p
    }
    c.coefQ = upload(c, cq);
    c.coefQH = upload(c, cqh);
    c.invQ = upload(c, iq);
    c.invQH = upload(c, iqh);
    c.coefU1 = upload(c, std::vector<Coef>{coef(-tau, 0.0, 0.0)});
    c.coefU2 = upload(c, u2);
    c.coefU3 = upload(c, u3);
    c.coefU4 = upload(c, std::vector<Coef>{coef(tau / beta, 0.0, 0.0)});
    c.coefS1 = upload(c, std::vector<Coef>{coef(tau, 0.0, 0.0)});
    c.coefS2 = upload(c, s2);
    c.coefS3 = upload(c, s3);
    c.coefS4 = upload(c, std::vector<Coef>{coef(-tau / beta, 0.0, 0.0)});
  }

  // frequency-domain arrays and workspaces
  const long fv = (long)n_f * 2 * dim * c.n_s, fp = (long)n_f * 2 * c.n_p;
  c.Fv = dalloc<double2>(c, fv);
  c.Fp = dalloc<double2>(c, fp);
  c.XpA = dalloc<double2>(c, fp);
  const int nprob_v = c.oseen ? n_f * dim : n_f * 2 * dim;
  const int nprob_p = 2 * n_f;
  long cheb_len = (long)nprob_p * c.n_p;
  if (c.oseen) {
    const long vv = (long)n_f * dim * c.n_s;
    c.X1 = dalloc<double2>(c, vv);
    c.X2 = dalloc<double2>(c, vv);
    c.T1 = dalloc<double2>(c, vv);
    c.T2 = dalloc<double2>(c, vv);
    c.T3 = dalloc<double2>(c, vv);
    c.Qp = dalloc<double2>(c, fp);
    c.Sp = dalloc<double2>(c, fp);
    c.Tp = dalloc<double2>(c, fp);
    cheb_len = std::max(cheb_len, vv);
  } else {
    c.Xv = dalloc<double2>(c, fv);
    c.XpB = dalloc<double2>(c, fp);
  }
  c.Cr = dalloc<double2>(c, cheb_len);
  c.Cd0 = dalloc<double2>(c, cheb_len);
  c.Cd1 = dalloc<double2>(c, cheb_len);
  // MG level workspaces.  The velocity solves run in chunks of c.freq_chunk frequencies (aao_config.freq_chunk;
  // 0 = auto: all frequencies when the workspace fits in 2 GiB, else the largest multiple of a full wave of
  // 148 problems that does), so the per-level workspace is bounded independently of n_t.
  {
    const int ppf = nprob_v / n_f;   // velocity problems per frequency
    double per_prob = 0;
    for (int l = 0; l < nlev; ++l) per_prob += (l == 0 ? 1.0 : 3.0) * c.vel.grids[l].n * sizeof(double2);
    const double per_freq = per_prob * ppf;
    int F = cfg.freq_chunk > 0 ? std::min(cfg.freq_chunk, n_f) : n_f;
    if (cfg.freq_chunk <= 0 && per_freq * n_f > 2.0 * (1 << 30)) {
      F = std::max(1, (int)(2.0 * (1 << 30) / per_freq));
      int q = 1;                       // frequencies per full wave of 148 problems (when it divides)
      while ((q * ppf) % 148 != 0 && q < 148) ++q;
      if (F >= q) F = F / q * q;
    }
    c.freq_chunk = F;
  }
  for (int sp = 0; sp < 2; ++sp) {
    MGSpace& S = sp == 0 ? c.vel : c.pres;
    const int np = sp == 0 ? c.freq_chunk * (nprob_v / n_f) : nprob_p;
    S.nprob_max = np;
    S.x.assign(nlev, nullptr);
    S.b.assign(nlev, nullptr);
    S.r.assign(nlev, nullptr);
    for (int l = 0; l < nlev; ++l) {
      const long n = S.grids[l].n * (long)np;
      S.r[l] = dalloc<double2>(c, n);
      CK(cudaMemset(S.r[l], 0, n * sizeof(double2)));
      if (l > 0) {
        S.x[l] = dalloc<double2>(c, n);
        S.b[l] = dalloc<double2>(c, n);
        CK(cudaMemset(S.x[l], 0, n * sizeof(double2)));
        CK(cudaMemset(S.b[l], 0, n * sizeof(double2)));
      }
    }
  }
  // Algorithm 2 workspace: inner Krylov basis V_0..V_m plus Zt, U (frequency vectors)
  if (cfg.pmode == AAO_PRECOND_NONLINEAR) {
    c.nonlinear = true;
    c.inner_eps = cfg.inner_eps;
    const size_t fvec = (size_t)(fv + fp) * sizeof(double2);
    size_t freeb = 0, totb = 0;
    CK(cudaMemGetInfo(&freeb, &totb));
    const long fit = (long)((freeb * 0.6) / fvec) - 3;
    int m = std::min<long>(cfg.inner_maxit, std::max<long>(fit, 1));
    c.inner_maxit = m;
    c.nlV.resize(m + 3);
    for (int j = 0; j < m + 3; ++j) {
      c.nlV[j].v = dalloc<double2>(c, fv);
      c.nlV[j].p = dalloc<double2>(c, fp);
      CK(cudaMemset(c.nlV[j].v, 0, fv * sizeof(double2)));
      CK(cudaMemset(c.nlV[j].p, 0, fp * sizeof(double2)));
    }
    c.nlVdev = upload(c, std::vector<FVec>(c.nlV.begin(), c.nlV.begin() + m + 1));
    c.nlH = dalloc<double2>(c, (size_t)(m + 2) * n_f);
    c.nlPart = dalloc<double2>(c, fdot_partial_len(n_f));
    c.nlY = dalloc<double2>(c, (size_t)n_f * (m + 1));
    c.nlFrozen = dalloc<int>(c, n_f);
    if (!c.oseen && !c.Xv) c.Xv = dalloc<double2>(c, fv);
  }
  CK(cudaMemset(c.Fv, 0, fv * sizeof(double2)));
  CK(cudaMemset(c.Fp, 0, fp * sizeof(double2)));
  CK(cudaMemset(c.XpA, 0, fp * sizeof(double2)));
  if (c.Xv) CK(cudaMemset(c.Xv, 0, fv * sizeof(double2)));
  if (c.XpB) CK(cudaMemset(c.XpB, 0, fp * sizeof(double2)));
  if (c.X1) {
    CK(cudaMemset(c.X1, 0, (size_t)n_f * dim * c.n_s * sizeof(double2)));
    CK(cudaMemset(c.X2, 0, (size_t)n_f * dim * c.n_s * sizeof(double2)));
  }
  CK(cudaDeviceSynchronize());
}

// ------------------------------------------------------------------ block solvers
inline View contig(double2* p, long n) { return View{p, 1, n}; }

// brackets a run of launches of the dominant kernel class with events when profiling is on
struct SweepTimer {
  Ctx& c;
  bool on;
  cudaStream_t s;
  SweepTimer(Ctx& c_, bool active, cudaStream_t s_, double bytes, long launches)
      : c(c_), on(c_.prof && active), s(s_) {
    if (!on) return;
    if (c.prof_used + 2 > c.prof_ev.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c.prof_ev.push_back(e);
      }
    }
    cudaEventRecord(c.prof_ev[c.prof_used], s);
    c.prof_bytes += bytes;
    c.prof_launches += launches;
  }
  ~SweepTimer() {
    if (!on) return;
    cudaEventRecord(c.prof_ev[c.prof_used + 1], s);
    c.prof_used += 2;
  }
};

long unknowns(const Grid& g) {
  long u = 1;
  for (int a = 0; a < g.dim; ++a) u *= (g.order == 2 ? g.n1 - 2 : g.n1);
  return g.order == 1 ? u - 1 : u;
}

// algorithmic bytes of one MG solve (all cycles): per level and V-cycle, sweeps 48 B/unknown each,
// residual 48, restriction 16 (+16 per coarse unknown), prolongation + correction 32 (+16 per coarse
// unknown), coarsest solve 32 (~1579 B per fine unknown in 2-D)
double mg_bytes(const Ctx& c, const MGSpace& S, int nprob) {
  double b = 0;
  for (int l = 0; l + 1 < S.nlev; ++l) {
    const double u = unknowns(S.grids[l]), uc = unknowns(S.grids[l + 1]);
    b += u * (48.0 * (c.cfg.pre_sweeps + c.cfg.post_sweeps) + 48 + 16 + 32) + uc * 32.0;
  }
  b += 32.0 * unknowns(S.grids[S.nlev - 1]);
  return b * c.cfg.mg_cycles * nprob;
}

// one V-cycle on levels >= l, one launch per level / colour (AAO_MG_MODE=1; the parity-tested reference
// schedule of the CTA-resident solve)
void mg_vcycle(Ctx& c, MGSpace& S, int l, const OpSel& op, const double2* inv, int inv_pg, View x, View b, int nprob,
               cudaStream_t s) {
  const Grid& g = S.grids[l];
  auto& cnt = launch_counter();
  if (l == S.nlev - 1) {
    launch_coarse(g, inv, inv_pg, S.coarse_unk, S.ncoarse_unk, b, x, nprob, s);
    ++cnt;
    return;
  }
  const int C = S.order == 2 ? (c.dim == 2 ? 9 : 27) : (c.dim == 2 ? 4 : 8);
  for (int sw = 0; sw < c.cfg.pre_sweeps; ++sw)
    for (int col = 0; col < C; ++col) {
      launch_gs(g, op, x, b, nprob, col, c.cfg.omega, s);
      ++cnt;
    }
  View r = contig(S.r[l], g.n);
  launch_residual(g, op, x, b, r, nprob, s);
  const Grid& gc = S.grids[l + 1];
  View bc = contig(S.b[l + 1], gc.n), xc = contig(S.x[l + 1], gc.n);
  launch_restrict(g, gc, S.transfers[l], r, bc, nprob, s);
  launch_zero(xc, gc.n, nprob, s);
  cnt += 3;
  mg_vcycle(c, S, l + 1, op, inv, inv_pg, xc, bc, nprob, s);
  launch_prolong(g, gc, S.transfers[l], xc, x, nprob, s);
  ++cnt;
  for (int sw = 0; sw < c.cfg.post_sweeps; ++sw)
    for (int col = C - 1; col >= 0; --col) {
      launch_gs(g, op, x, b, nprob, col, c.cfg.omega, s);
      ++cnt;
    }
}

// CTA-resident solve: `cycles` V-cycles from x = 0, one CTA per problem, all levels in one launch.
void launch_cta_levels(Ctx& c, MGSpace& S, const OpSel& op, const double2* inv, int inv_pg, View x, View b, int nprob,
                       int cycles, cudaStream_t s) {
  MGArgs a;
  std::memset(&a, 0, sizeof(a));
  a.nlev = S.nlev;
  a.cycles = cycles;
  a.pre = c.cfg.pre_sweeps;
  a.post = c.cfg.post_sweeps;
  a.omega = c.cfg.omega;
  for (int i = 0; i < a.nlev; ++i) {
    a.g[i] = S.grids[i];
    a.t[i] = S.transfers[i];
    a.xw[i] = S.x[i];
    a.bw[i] = S.b[i];
    a.rw[i] = S.r[i];
  }
  a.x0 = x;
  a.b0 = b;
  a.op = op;
  a.inv = inv;
  a.inv_pg = inv_pg;
  a.unk = S.coarse_unk;
  a.nu = S.ncoarse_unk;
  // class stencil tables (Q2, smoothing levels need n1 >= 9): first in dynamic smem.  AAO_NO_CTAB=1 evaluates
  // every stencil from the 1-D rows instead (same map, parity-tested; used to measure summation-order drift)
  static const bool no_ctab = std::getenv("AAO_NO_CTAB") != nullptr;
  size_t tab_bytes = 0;
  a.use_ctab = 0;
  if (!no_ctab && S.order == 2 && a.nlev >= 2 && a.g[a.nlev - 2].n1 >= 9) {
    a.use_ctab = 1;
    const size_t nt = c.dim == 2 ? 25 : 125;
    const size_t per = (size_t)(1 << c.dim) * (op.conv_sel == 0 ? (nt + 1) : 2 * nt);
    tab_bytes = (a.nlev - 1) * per * sizeof(double);
    tab_bytes = (tab_bytes + 15) / 16 * 16;
  } else if (!no_ctab && S.order == 1 && c.dim == 2 && op.conv_sel == 0 && a.nlev >= 2) {
    a.use_ctab = 2;   // 2-D Q1 real operators: position-class stencils (90 doubles per smoothing level)
    tab_bytes = ((size_t)(a.nlev - 1) * 90 * sizeof(double) + 15) / 16 * 16;
  }
  // shared-memory residency of the coarse levels (coarsest first while x and b fit).  Measured: 2-D Q2 with the
  // merged small-level visits keeps no level in shared memory (the L1 cache serves every level better than a
  // split: c2 2.216 -> 2.175 ms); elsewhere the smallest levels within 20 KB (c2 3.02 vs 3.17 ms, c3 277 vs 437 ms)
  const bool flat2d = c.dim == 2 && S.order == 2 && a.use_ctab;
  const size_t budget = flat2d ? 0 : 20 * 1024;
  size_t used = tab_bytes;
  a.lsm = a.nlev;
  for (int l = a.nlev - 1; l >= 1; --l) {
    const size_t need = 2 * a.g[l].n * sizeof(double2);
    if (used + need > budget + tab_bytes) break;
    a.sm_x[l] = (long)(used / sizeof(double2));
    a.sm_b[l] = (long)(used / sizeof(double2)) + a.g[l].n;
    used += need;
    a.lsm = l;
  }
  // the bottom levels (<= 256 unknowns) run warp-synchronously -- their phases are pure latency -- except for
  // the 2-D Q2 merged branch-free visits, which run faster block-wide (c2 precond 2.25 -> 2.22 ms)
  const long wmax = flat2d ? 0 : 256;
  a.lwarp = a.nlev;
  for (int l = 1; l < a.nlev; ++l)
    if (unknowns(a.g[l]) <= wmax) {
      a.lwarp = l;
      break;
    }
  // band-wavefront sweeps (2-D Q2) on the levels with n1 >= wave_min (default 65): the iterate crosses HBM once
  // per sweep instead of once per colour, every tap is a shared-memory load (measured with the first, node-per-thread
  // form: c4_64 precond 43.6 -> 35.2 ms, c4_128 87.8 -> 73.5 ms; slower with the stored per-node convection stencils,
  // c3 255 -> 330 ms, so Oseen operators use it only when forced).  AAO_WAVE=0/1 forces it off/on for every eligible
  // level >= AAO_WAVE_MIN (parity-tested).  Real operators sweep in triple form, one thread per node triple: the band
  // height of a level is the largest H in {24, 12, 6, 3} whose H rows of triples fit the CTA's threads and whose
  // 9-slot ring fits the shared memory left (513^2: 3, 257^2: 6, 129^2: 6, 65^2: 12, 33^2: 24); a row takes whole warps.
  a.wave_h = 0;
  for (int l = 0; l < MG_MAXL; ++l) a.wave_hl[l] = 0;
  const bool wave_on = c.wave_force >= 0 ? c.wave_force != 0 : (op.conv_sel == 0 && a.g[0].n1 >= c.wave_min);
  const bool wave_conv = c.wave_force == 1;
  if (wave_on && c.dim == 2 && S.order == 2 && a.use_ctab && (op.conv_sel == 0 || wave_conv)) {
    const size_t mbars = 5 * sizeof(double2);   // 9 mbarriers (72 B) + phase word
    const size_t guard = 2 * MG_RING_GUARD * sizeof(double2);
    used = (used + 15) / 16 * 16;
    const size_t cap = (size_t)MG_SMEM_MAX > used + mbars + guard ? (size_t)MG_SMEM_MAX - used - mbars - guard : 0;
    size_t ring = 0;
    for (int l = 0; l < a.nlev - 1 && l < a.lsm; ++l) {
      const int n1 = a.g[l].n1;
      if (n1 < c.wave_min || n1 < 9) break;
      int h = 0;
      if (op.conv_sel != 0) {
        h = n1 <= 129 ? 6 : 3;                       // node-per-thread form (q2_wave_pass)
        if ((size_t)8 * h * n1 * sizeof(double2) > cap) h = 0;
      } else {
        const int ntr = (n1 - 2) / 3 + 1;
        for (int cand = c.wave_hmax; cand >= 3 && !h; cand /= 2)
          if (cand * mg_tri_lanes_per_row(ntr) <= MG_TRI_THREADS &&
              (size_t)MG_TRI_SLOTS * cand * n1 * sizeof(double2) <= cap)
            h = cand;
      }
      a.wave_hl[l] = h;
      if (h) ring = std::max(ring, (size_t)(op.conv_sel != 0 ? 8 : MG_TRI_SLOTS) * h * n1 * sizeof(double2));
    }
    if (ring) {
      a.wave_h = 1;
      a.ring_off = (long)(used / sizeof(double2)) + MG_RING_GUARD;
      used += ring + guard;
      a.mbar_off = (long)(used / sizeof(double2));
      used += mbars;
    }
  }
  // 2-D Q1 real operators (pressure MG): pair-form wavefront sweeps on the levels with n1 >= wave_min_q1; band
  // height = the largest even H <= 8 whose rows of pairs (padded to whole warps; two rows per thread when 4 | H) fit
  // the CTA's 512 threads
  static const int wave_q1 = std::getenv("AAO_WAVE_Q1") ? std::atoi(std::getenv("AAO_WAVE_Q1")) : 1;
  if (wave_q1 && c.wave_force != 0 && c.dim == 2 && S.order == 1 && a.use_ctab == 2 && op.conv_sel == 0) {
    const int wmin = c.wave_force == 1 ? std::max(c.wave_min, 5) : 129;
    const size_t mbars = 5 * sizeof(double2), guard = 2 * MG_RING_GUARD * sizeof(double2);
    used = (used + 15) / 16 * 16;
    const size_t cap = (size_t)MG_SMEM_MAX > used + mbars + guard ? (size_t)MG_SMEM_MAX - used - mbars - guard : 0;
    size_t ring = 0;
    for (int l = 0; l < a.nlev - 1 && l < a.lsm && l < a.lwarp; ++l) {
      const int n1 = a.g[l].n1;
      if (n1 < wmin) break;
      const int lpr = mg_tri_lanes_per_row((n1 + 1) / 2);
      int h = 0;
      // (a thread takes two rows of its class when H is a multiple of 4: H / U rows of lanes)
      for (int cand = std::min(8, c.wave_hmax >= 6 ? 8 : 2); cand >= 2 && !h; cand -= 2)
        if ((cand % 4 == 0 ? cand / 2 : cand) * lpr <= 512 &&
            (size_t)MG_TRI_SLOTS * cand * n1 * sizeof(double2) <= cap)
          h = cand;
      a.wave_hl[l] = h;
      if (h) ring = std::max(ring, (size_t)MG_TRI_SLOTS * h * n1 * sizeof(double2));
    }
    if (ring) {
      a.wave_h = 1;
      a.ring_off = (long)(used / sizeof(double2)) + MG_RING_GUARD;
      used += ring + guard;
      a.mbar_off = (long)(used / sizeof(double2));
      used += mbars;
    }
  }
  a.flat_max = 33;   // measured: 33 best (c2 precond 2.371 -> 2.249 ms)
  // x += P x_c fused into the first post-smoothing wavefront sweep (AAO_FUSE_PROLONG=0: a separate pass; measured
  // c4_512 precond 184 vs 175 ms with the fusion)
  static const bool no_fuse_pro = std::getenv("AAO_FUSE_PROLONG") != nullptr && std::atoi(std::getenv("AAO_FUSE_PROLONG")) == 0;
  a.fuse_prolong = no_fuse_pro ? 0 : 1;
  // 3-D: z-band wavefront sweeps on the levels whose iterate does not stay in L2 across the 27 colour steps
  // (n1 >= 65 by default; AAO_WAVE=1 forces every level >= AAO_WAVE_MIN, AAO_WAVE=0 none)
  a.zwave_min = c.wave_force == 0 ? (1 << 30) : (c.wave_force == 1 ? c.wave_min : 65);
  // line form of the z-band wavefront (real operators): a ring of staged lines of n1 + 8 entries per warp of the CTA
  a.zstage_off = -1;
  static const bool no_zline = std::getenv("AAO_NO_ZLINE") != nullptr;
  if (c.dim == 3 && S.order == 2 && a.use_ctab == 1 && op.conv_sel == 0 && !no_zline) {
    used = (used + 15) / 16 * 16;
    const size_t st = (size_t)16 * MG_ZL_STAGES * (a.g[0].n1 + 8) * sizeof(double2);   // 512 threads = 16 warps
    if (used + st <= (size_t)MG_SMEM_MAX) {
      a.zstage_off = (long)(used / sizeof(double2));
      used += st;
    }
  }
  // profiling only: per-level SM-cycle accounting of CTA 0, printed per launch (AAO_MG_CLOCK=1)
  static const bool mg_clock = std::getenv("AAO_MG_CLOCK") != nullptr;
  static unsigned long long* clk_dev = nullptr;
  if (mg_clock) {
    if (!clk_dev) cudaMalloc(&clk_dev, 2 * MG_MAXL * sizeof(unsigned long long));
    cudaMemsetAsync(clk_dev, 0, 2 * MG_MAXL * sizeof(unsigned long long), s);
    a.clk = clk_dev;
    a.clk_block = std::min(std::atoi(std::getenv("AAO_MG_CLOCK")), nprob - 1);
  }
  launch_mg_cta(a, nprob, used, s);
  ++launch_counter();
  if (mg_clock) {
    unsigned long long h[2 * MG_MAXL];
    cudaMemcpyAsync(h, clk_dev, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "mg_clock order %d nprob %d lwarp %d:", S.order, nprob, a.lwarp);
    for (int l = 0; l < a.nlev - 1; ++l) std::fprintf(stderr, " L%d(n1=%d) %llu/%llu", l, a.g[l].n1, h[2 * l], h[2 * l + 1]);
    std::fprintf(stderr, " bottom %llu | L0 down: sweeps %llu residual %llu restrict %llu | tri steps: band wait %llu "
                 "barrier %llu tma issue %llu update %llu residual %llu\n", h[2 * MG_MAXL - 1], h[2 * MG_MAXL - 2],
                 h[2 * MG_MAXL - 3], h[2 * MG_MAXL - 4], h[16], h[17], h[18], h[19], h[14]);
  }
}

// problems [p0, p0 + ...) of a batch view (p0 a multiple of the view's group size)
inline View sub_view(View v, long n, int p0) {
  return View{v.p + (long)(p0 / v.per_group) * v.gstride + (long)(p0 % v.per_group) * n, v.per_group, v.gstride};
}

// x = MG(A; b): mg_cycles V-cycles from x = 0, in chunks of at most S.nprob_max problems
// (the workspace size; frequency-aligned chunks, so coefficient groups and coarse inverses shift with them)
void mg_solve(Ctx& c, MGSpace& S, const OpSel& op, const double2* inv, int inv_pg, View x, View b, int nprob,
              cudaStream_t s) {
  const long n = S.grids[0].n;
  for (int p0 = 0; p0 < nprob; p0 += S.nprob_max) {
    const int np = std::min(S.nprob_max, nprob - p0);
    OpSel opc = op;
    if (op.per_group < (1 << 30)) opc.coef = op.coef + p0 / op.per_group;
    const double2* invc = inv_pg < (1 << 30) ? inv + (long)(p0 / inv_pg) * S.ncoarse_unk * S.ncoarse_unk : inv;
    const View xc = sub_view(x, n, p0), bc = sub_view(b, n, p0);
    if (c.mg_mode == 0) {
      SweepTimer tm(c, S.order == 2, s, mg_bytes(c, S, np), 1);
      launch_cta_levels(c, S, opc, invc, inv_pg, xc, bc, np, c.cfg.mg_cycles, s);
    } else {
      SweepTimer tm(c, S.order == 2, s, mg_bytes(c, S, np), 0);
      launch_zero(xc, n, np, s);
      ++launch_counter();
      for (int cyc = 0; cyc < c.cfg.mg_cycles; ++cyc) mg_vcycle(c, S, 0, opc, invc, inv_pg, xc, bc, np, s);
    }
  }
}

// x = scale * Chebyshev(M; b), Jacobi-preconditioned, Wathen bounds
void cheb_solve(Ctx& c, const Grid& g, View b, View x, int nprob, double scale, cudaStream_t s) {
  const double lo1 = 0.5, hi1 = g.order == 2 ? 1.25 : 1.5;
  const double lo = std::pow(lo1, c.dim), hi = std::pow(hi1, c.dim);
  const double theta = 0.5 * (hi + lo), delta = 0.5 * (hi - lo), sigma = theta / delta;
  if (c.mg_mode != 1) {
    launch_cheb_cta(g, b, x, c.Cr, c.Cd0, c.Cd1, theta, sigma, delta, c.cfg.cheb_iters, scale, nprob, s);
    ++launch_counter();
    return;
  }
  View r = contig(c.Cr, g.n), d0 = contig(c.Cd0, g.n), d1 = contig(c.Cd1, g.n);
  launch_cheb_init(g, b, x, r, d0, 1.0 / theta, nprob, s);
  double rho = 1.0 / sigma;
  for (int k = 0; k < c.cfg.cheb_iters - 1; ++k) {
    const double rho1 = 1.0 / (2.0 * sigma - rho);
    launch_cheb_step(g, x, r, d0, d1, rho1 * rho, 2.0 * rho1 / delta, nprob, s);
    std::swap(d0, d1);
    rho = rho1;
  }
  launch_cheb_final(g, x, d0, scale, nprob, s);
  launch_counter() += c.cfg.cheb_iters + 1;
}

// Stokes block solves P~_k^{-1} without the T transforms, on the frequency vector `in`
// (velocity slots -> outV; pressure slots: K_p-MG -> outPA, M_p-Chebyshev -> outPB)
void stokes_blocks(Ctx& c, FVec in, double2* outV, double2* outPA, double2* outPB, cudaStream_t s) {
  const int dim = c.dim, n_f = c.n_f;
  const Grid& gv = c.vel.grids[0];
  const Grid& gp = c.pres.grids[0];
  // x1 = MG(W; s1), x2 = MG(W; s2) per velocity component
  OpSel opW{c.coefW, 2 * dim, 0};
  // The pressure slots (independent of the velocity slots) -- K_p^{-1} by MG and M_p^{-1} by Chebyshev, combined
  // later -- run on two side streams, concurrently with each other (each fills the partial last wave of
  // the other: 512 problems on 148 SMs at c4_512).  When the velocity solve is chunked into several full-width
  // launches they start after it: interleaved with it, their short CTAs take the SMs that free up at every
  // launch boundary and every velocity launch then waits for them (measured c4_512: 20.8 ms per launch with the
  // same total as 15.9 ms per launch alone + the pressure solves at full width).  A single velocity launch that
  // leaves SMs idle (small configs) still overlaps with them.
  cudaStream_t sp = c.s2, sq = c.s3;
  OpSel opKp{c.coefKp, 1 << 30, 0};
  const int nprob_v = n_f * 2 * dim;
  static const int after_env = std::getenv("AAO_PRESSURE_AFTER") ? std::atoi(std::getenv("AAO_PRESSURE_AFTER")) : -1;
  const bool after = after_env >= 0 ? after_env != 0 : nprob_v > c.vel.nprob_max;
  auto pressure = [&]() {
    cudaEventRecord(c.ev_fork, s);
    cudaStreamWaitEvent(sp, c.ev_fork, 0);
    cudaStreamWaitEvent(sq, c.ev_fork, 0);
    mg_solve(c, c.pres, opKp, c.invKp, 1 << 30, contig(outPA, gp.n), contig(in.p, gp.n), 2 * n_f, sp);
    cheb_solve(c, gp, contig(in.p, gp.n), contig(outPB, gp.n), 2 * n_f, 1.0, sq);
    cudaEventRecord(c.ev_join, sp);
    cudaEventRecord(c.ev_join2, sq);
  };
  if (!after) pressure();
  mg_solve(c, c.vel, opW, c.invW, 2 * dim, contig(outV, gv.n), contig(in.v, gv.n), nprob_v, s);
  if (c.timing) cudaEventRecord(c.ev[2], s);
  if (after) pressure();
  cudaStreamWaitEvent(s, c.ev_join, 0);
  cudaStreamWaitEvent(s, c.ev_join2, 0);
}

void precond_stokes(Ctx& c, cudaStream_t s) { stokes_blocks(c, FVec{c.Fv, c.Fp}, c.Xv, c.XpA, c.XpB, s); }

// Oseen block solves (P~_k^(UZ))^{-1} (Algorithm 3) on the frequency vector `in`: outputs X1, X2
// (velocity slots, [k][comp][node]) and XpA (pressure slots, to be scaled by -1/tau)
void oseen_blocks(Ctx& c, FVec in, cudaStream_t s) {
  const int dim = c.dim, n_f = c.n_f;
  const Grid& gv = c.vel.grids[0];
  const Grid& gp = c.pres.grids[0];
  const long nv = gv.n, np = gp.n;
  const int nprob = n_f * dim;
  const double tau = c.tau, mu = c.cfg.uzawa_mu;
  View B1{in.v, dim, 2L * dim * nv}, B2{in.v + (long)dim * nv, dim, 2L * dim * nv};
  View X1 = contig(c.X1, nv), X2 = contig(c.X2, nv), T1 = contig(c.T1, nv), T2 = contig(c.T2, nv),
       T3 = contig(c.T3, nv);
  OpSel U1{c.coefU1, 1 << 30, 0}, U2{c.coefU2, dim, 2}, U3{c.coefU3, dim, 1}, U4{c.coefU4, 1 << 30, 0};
  OpSel Mass{c.coefMass, 1 << 30, 0};
  OpSel opQ{c.coefQ, dim, 1}, opQH{c.coefQH, dim, 2};
  auto& cnt = launch_counter();
  launch_zero(X1, nv, nprob, s);
  launch_zero(X2, nv, nprob, s);
  cnt += 2;
  for (int it = 0; it < c.cfg.uzawa_iters; ++it) {
    // x1 <- x1 + (1/tau) Mhat^{-1}(b1 - tau M x1 - (d M + tau L)^H x2)     (eq. Uzawa11)
    launch_lincomb(gv, T1, 1.0, B1, U1, X1, U2, X2, nprob, s);
    cheb_solve(c, gv, T1, T2, nprob, 1.0, s);
    launch_axpby(gv, X1, make_double2(1, 0), T2, make_double2(1.0 / tau, 0), nprob, s);
    // x2 <- x2 - (1/mu) S^{-1}(b2 - (d M + tau L) x1 + (tau/beta) M x2),  S^{-1} = tau Q^{-H} M Q^{-1}
    launch_lincomb(gv, T1, 1.0, B2, U3, X1, U4, X2, nprob, s);
    cnt += 3;
    mg_solve(c, c.vel, opQ, c.invQ, dim, T2, T1, nprob, s);
    launch_lincomb(gv, T3, 0.0, T1, Mass, T2, Mass, View{nullptr, 1, 0}, nprob, s);
    ++cnt;
    mg_solve(c, c.vel, opQH, c.invQH, dim, T2, T3, nprob, s);
    launch_axpby(gv, X2, make_double2(1, 0), T2, make_double2(-tau / mu, 0), nprob, s);
    ++cnt;
  }
  if (c.timing) cudaEventRecord(c.ev[2], s);
  // (y3, y4) = -S_hat^{-1}((r3, r4) - tau (B y2, B y1))   (Algorithm 3)
  View Xv2{c.X2, dim, (long)dim * nv}, Xv1{c.X1, dim, (long)dim * nv};
  View P3{in.p, 1, 2 * np}, P4{in.p + np, 1, 2 * np};
  View Q3{c.Qp, 1, 2 * np}, Q4{c.Qp + np, 1, 2 * np};
  launch_Bv(gv, gp, c.tPm, c.tGm, Xv2, P3, Q3, 1.0, -tau, n_f, s);
  launch_Bv(gv, gp, c.tPm, c.tGm, Xv1, P4, Q4, 1.0, -tau, n_f, s);
  // S_hat^{-1}: [[0,tau M_p],[tau M_p,0]]^{-1} -> Sp[k][0] = s2 = M_p^{-1} q3 / tau, Sp[k][1] = s1 = M_p^{-1} q4 / tau
  cheb_solve(c, gp, contig(c.Qp, np), contig(c.Sp, np), 2 * n_f, 1.0 / tau, s);
  View s2v{c.Sp, 1, 2 * np}, s1v{c.Sp + np, 1, 2 * np};
  View t2v{c.Tp, 1, 2 * np}, t1v{c.Tp + np, 1, 2 * np};
  OpSel S1{c.coefS1, 1 << 30, 0}, S2{c.coefS2, 1, 2}, S3{c.coefS3, 1, 1}, S4{c.coefS4, 1 << 30, 0};
  // t1 = tau M_p s1 + (d^* M_p + tau L_p^T) s2 ;  t2 = (d M_p + tau L_p) s1 - (tau/beta) M_p s2
  launch_lincomb(gp, t1v, 0.0, t1v, S1, s1v, S2, s2v, n_f, s);
  launch_lincomb(gp, t2v, 0.0, t2v, S3, s1v, S4, s2v, n_f, s);
  cnt += 4;
  // [[0,tau K_p],[tau K_p,0]]^{-1}: XpA[k][0] = K_p^{-1} t2, XpA[k][1] = K_p^{-1} t1 (scaled by -1/tau on output)
  OpSel opKp{c.coefKp, 1 << 30, 0};
  mg_solve(c, c.pres, opKp, c.invKp, 1 << 30, contig(c.XpA, np), contig(c.Tp, np), 2 * n_f, s);
}

void precond_oseen(Ctx& c, cudaStream_t s) { oseen_blocks(c, FVec{c.Fv, c.Fp}, s); }

// ------------------------------------------------------------------ Algorithm 2 (nonlinear)
// P~ applied to a frequency vector: out = blkdiag-preconditioner(in)   (Stokes: P~_k^{-1} of P:416-426
// without T transforms; Oseen: (P~_k^(UZ))^{-1}, Algorithm 3)
void pt_apply(Ctx& c, FVec in, FVec out, cudaStream_t s) {
  const long LP = 2L * c.n_p;
  if (!c.oseen) {
    stokes_blocks(c, in, out.v, c.XpA, c.XpB, s);
    launch_combine_p(out.p, c.XpA, c.XpB, c.fc, c.nu, LP, c.n_f, s);
  } else {
    oseen_blocks(c, in, s);
    launch_oseen_scatter(out, c.X1, c.X2, c.XpA, -1.0 / c.tau, (long)c.dim * c.n_s, LP, c.n_f, s);
  }
  ++launch_counter();
}

// y = A_k x per frequency: Z_k of P:392-397 (Stokes) or G_k of eq. (SubBlockG) (Oseen)
void op_apply(Ctx& c, FVec x, FVec y, cudaStream_t s) {
  const int dim = c.dim, n_f = c.n_f;
  const Grid& gv = c.vel.grids[0];
  const Grid& gp = c.pres.grids[0];
  const long nv = gv.n, np = gp.n;
  auto vh = [&](double2* base, int h) { return View{base + (long)h * dim * nv, dim, 2L * dim * nv}; };
  auto ph = [&](double2* base, int h) { return View{base + (long)h * np, 1, 2 * np}; };
  const int nprob = n_f * dim;
  const View none{nullptr, 1, 0};
  if (!c.oseen) {
    // r1 = M x1 + X x2 + B^T x4 ; r2 = X x1 - M x2 + B^T x3 ; r3 = B x2 ; r4 = B x1,  X = c1 M + c2 nu K
    OpSel Mass{c.coefMass, 1 << 30, 0}, NegMass{c.coefNegMass, 1 << 30, 0}, X{c.coefZX, dim, 0};
    launch_lincomb(gv, vh(y.v, 0), 0.0, none, Mass, vh(x.v, 0), X, vh(x.v, 1), nprob, s);
    launch_lincomb(gv, vh(y.v, 1), 0.0, none, X, vh(x.v, 0), NegMass, vh(x.v, 1), nprob, s);
    launch_fBT(c, y, 0, x, 1, 1.0, s);
    launch_fBT(c, y, 1, x, 0, 1.0, s);
    launch_Bv(gv, gp, c.tPm, c.tGm, vh(x.v, 1), none, ph(y.p, 0), 0.0, 1.0, n_f, s);
    launch_Bv(gv, gp, c.tPm, c.tGm, vh(x.v, 0), none, ph(y.p, 1), 0.0, 1.0, n_f, s);
  } else {
    // r1 = tau M x1 + (d^* M + tau L^T) x2 + tau B^T x4 ; r2 = (d M + tau L) x1 - tau/beta M x2 + tau B^T x3
    // r3 = tau B x2 ; r4 = tau B x1
    const double tau = c.tau;
    OpSel G11{c.coefS1, 1 << 30, 0}, G12{c.coefS2, dim, 2}, G21{c.coefS3, dim, 1}, G22{c.coefS4, 1 << 30, 0};
    launch_lincomb(gv, vh(y.v, 0), 0.0, none, G11, vh(x.v, 0), G12, vh(x.v, 1), nprob, s);
    launch_lincomb(gv, vh(y.v, 1), 0.0, none, G21, vh(x.v, 0), G22, vh(x.v, 1), nprob, s);
    launch_fBT(c, y, 0, x, 1, tau, s);
    launch_fBT(c, y, 1, x, 0, tau, s);
    launch_Bv(gv, gp, c.tPm, c.tGm, vh(x.v, 1), none, ph(y.p, 0), 0.0, tau, n_f, s);
    launch_Bv(gv, gp, c.tPm, c.tGm, vh(x.v, 0), none, ph(y.p, 1), 0.0, tau, n_f, s);
  }
  launch_counter() += 6;
}

// Algorithm 2: z = F^{-1} T_r^{-1} GMRES_k(A_k, P~_k, T_l^{-1} (F r)_k, eps)  per frequency,
// inner GMRES right-preconditioned, x0 = 0, MGS, no restart, |g_{j+1}| <= eps ||s_k|| (C.2 #20)
void nl_precond_apply(Ctx& c, const double* r, double* z, cudaStream_t s) {
  const int nf = c.n_f, m = c.inner_maxit;
  const long LV = 2L * c.dim * c.n_s, LP = 2L * c.n_p;
  launch_fft_fwd(c, r, s);
  ++launch_counter();
  FVec S0{c.Fv, c.Fp};
  FVec* V = c.nlV.data();
  FVec Zt = c.nlV[m + 1], U = c.nlV[m + 2];
  std::vector<double2> hh((size_t)(m + 2) * nf);
  std::vector<std::complex<double>> H((size_t)nf * (m + 1) * m), cs((size_t)nf * m), sn((size_t)nf * m),
      g((size_t)nf * (m + 1));
  std::vector<double> beta(nf);
  std::vector<int> its(nf, 0), done(nf, 0);
  // beta_k = ||s_k||, V_0 = s / beta_k
  launch_fdot(S0, S0, LV, LP, nf, c.nlPart, c.nlH, 1, s);
  CK(cudaMemcpyAsync(hh.data(), c.nlH, nf * sizeof(double2), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int k = 0; k < nf; ++k) {
    beta[k] = hh[k].x;
    done[k] = beta[k] == 0.0;
    g[(size_t)k * (m + 1)] = beta[k];
  }
  CK(cudaMemcpyAsync(c.nlFrozen, done.data(), nf * sizeof(int), cudaMemcpyHostToDevice, s));
  launch_fscale(V[0], S0, c.nlH, c.nlFrozen, LV, LP, nf, s);
  launch_counter() += 3;
  int jmax = 0;
  for (int j = 0; j < m; ++j) {
    bool all = true;
    for (int k = 0; k < nf; ++k) all = all && done[k];
    if (all) break;
    pt_apply(c, V[j], Zt, s);
    op_apply(c, Zt, V[j + 1], s);
    for (int i = 0; i <= j; ++i) {                       // modified Gram-Schmidt, per frequency
      launch_fdot(V[i], V[j + 1], LV, LP, nf, c.nlPart, c.nlH + (size_t)i * nf, 0, s);
      launch_faxpy(V[j + 1], V[i], c.nlH + (size_t)i * nf, -1.0, LV, LP, nf, s);
      launch_counter() += 3;
    }
    launch_fdot(V[j + 1], V[j + 1], LV, LP, nf, c.nlPart, c.nlH + (size_t)(j + 1) * nf, 1, s);
    launch_counter() += 2;
    CK(cudaMemcpyAsync(hh.data(), c.nlH, (size_t)(j + 2) * nf * sizeof(double2), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    jmax = j + 1;
    for (int k = 0; k < nf; ++k) {
      if (done[k]) continue;
      std::complex<double>* Hk = &H[(size_t)k * (m + 1) * m];
      for (int i = 0; i <= j + 1; ++i) Hk[(size_t)i * m + j] = std::complex<double>(hh[(size_t)i * nf + k].x, hh[(size_t)i * nf + k].y);
      std::complex<double>* csk = &cs[(size_t)k * m];
      std::complex<double>* snk = &sn[(size_t)k * m];
      std::complex<double>* gk = &g[(size_t)k * (m + 1)];
      for (int i = 0; i < j; ++i) {                      // previous complex Givens rotations
        const std::complex<double> t = std::conj(csk[i]) * Hk[(size_t)i * m + j] + std::conj(snk[i]) * Hk[(size_t)(i + 1) * m + j];
        Hk[(size_t)(i + 1) * m + j] = -snk[i] * Hk[(size_t)i * m + j] + csk[i] * Hk[(size_t)(i + 1) * m + j];
        Hk[(size_t)i * m + j] = t;
      }
      const std::complex<double> a = Hk[(size_t)j * m + j], b = Hk[(size_t)(j + 1) * m + j];
      const double den = std::sqrt(std::norm(a) + std::norm(b));
      csk[j] = a / den;
      snk[j] = b / den;
      Hk[(size_t)j * m + j] = den;
      Hk[(size_t)(j + 1) * m + j] = 0.0;
      gk[j + 1] = -snk[j] * gk[j];
      gk[j] = std::conj(csk[j]) * gk[j];
      its[k] = j + 1;
      if (std::abs(gk[j + 1]) <= c.inner_eps * beta[k] || std::abs(b) < 1e-14 * beta[k]) done[k] = 1;
    }
    CK(cudaMemcpyAsync(c.nlFrozen, done.data(), nf * sizeof(int), cudaMemcpyHostToDevice, s));
    launch_fscale(V[j + 1], V[j + 1], c.nlH + (size_t)(j + 1) * nf, c.nlFrozen, LV, LP, nf, s);
    ++launch_counter();
  }
  // y_k = H_k^{-1} g_k (its_k columns), u_k = sum_i y_k[i] V_i,k, x = P~(u)
  std::vector<double2> Y((size_t)nf * std::max(jmax, 1), make_double2(0.0, 0.0));
  c.inner_its = its;
  for (int k = 0; k < nf; ++k) {
    const int n = its[k];
    const std::complex<double>* Hk = &H[(size_t)k * (m + 1) * m];
    const std::complex<double>* gk = &g[(size_t)k * (m + 1)];
    std::vector<std::complex<double>> y(n);
    for (int i = n - 1; i >= 0; --i) {
      std::complex<double> acc = gk[i];
      for (int l = i + 1; l < n; ++l) acc -= Hk[(size_t)i * m + l] * y[l];
      y[i] = acc / Hk[(size_t)i * m + i];
    }
    for (int i = 0; i < n; ++i) Y[(size_t)k * std::max(jmax, 1) + i] = make_double2(y[i].real(), y[i].imag());
    c.inner_total += n;
    c.inner_max = std::max(c.inner_max, n);
  }
  CK(cudaMemcpyAsync(c.nlY, Y.data(), Y.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
  launch_fmulti(U, c.nlVdev, c.nlY, std::max(jmax, 1), LV, LP, nf, s);
  pt_apply(c, U, Zt, s);
  c.debug_block_src_v = Zt.v;
  c.debug_block_src_p = Zt.p;
  launch_fft_inv_from(c, Zt, z, s);
  launch_counter() += 2;
  CK(cudaStreamSynchronize(s));   // host vectors H, g, Y go out of scope
}

// r == z is allowed internally: r is read only by the forward transform, z written only by the inverse
void precond_apply(Ctx& c, const double* r, double* z, cudaStream_t s) {
  c.phase_valid = false;
  if (c.nonlinear) {
    nl_precond_apply(c, r, z, s);
    return;
  }
  c.debug_block_src_v = c.debug_block_src_p = nullptr;
  if (c.timing) cudaEventRecord(c.ev[0], s);
  launch_fft_fwd(c, r, s);
  ++launch_counter();
  if (c.timing) cudaEventRecord(c.ev[1], s);
  if (c.oseen)
    precond_oseen(c, s);
  else
    precond_stokes(c, s);
  if (c.timing) cudaEventRecord(c.ev[3], s);
  launch_fft_inv(c, z, s);
  ++launch_counter();
  if (c.timing) {
    cudaEventRecord(c.ev[4], s);
    c.phase_valid = true;
  }
}

void kkt_apply(Ctx& c, const double* x, double* y, cudaStream_t s) {
  launch_kkt(c, x, y, s);
  launch_counter() += 2;
}

// ------------------------------------------------------------------ GMRES
// Workspace: the basis V_0..V_m and ONE work vector z (the Arnoldi z_k = P^{-1} v_k, and at a restart the update
// u = V y and P^{-1} u in place); the residual b - A x is formed directly in V_0.  With the caller's b and x that is
// m + 4 vectors of N doubles (c4 at n_t = 512: 34 x 4.84 GB), plus m more when the preconditioned vectors are kept.
void gmres_alloc(Ctx& c, int m) {
  if (c.gm_m >= m) return;
  if (c.gm_m > 0) throw CudaError(AAO_ERR_CONFIG, "GMRES restart larger than the first solve's is not supported");
  const long N = c.N;
  c.gV = dalloc<double>(c, (size_t)(m + 1) * N);
  c.gz = dalloc<double>(c, N);
  c.gH = dalloc<double>(c, (size_t)(m + 2) * (m + 1));
  c.gpart = dalloc<double>(c, std::max((long)dot_blocks(), (long)(2 * m + 4) * 4 * mgs_blocks()));
  c.gG = dalloc<double>(c, (size_t)(m + 2) * (m + 2));
  c.gscal = dalloc<double>(c, 4 * (m + 2));
  std::vector<double*> ptr(m + 1);
  for (int i = 0; i <= m; ++i) ptr[i] = c.gV + (size_t)i * N;
  c.gVptr = upload(c, ptr);
  CK(cudaMallocHost(&c.hostH, sizeof(double) * (m + 2) * 2));
  for (int i = 0; i < 2; ++i) CK(cudaEventCreateWithFlags(&c.gm_ev[i], cudaEventDisableTiming));
  for (int i = 0; i < 4; ++i) CK(cudaEventCreate(&c.gt_ev[i]));
  c.gm_m = m;
}

// The m preconditioned vectors Z_k = P^{-1} v_k: always for FGMRES; for the linear mode only when the
// caller asks (aao_krylov.store_z): the restart update x += Z y then needs no extra preconditioner application
// (Algorithm 1 is a fixed linear map, so Z y = P^{-1}(V y) up to rounding).  A deterministic choice: an
// allocation failure is AAO_ERR_OOM, never a silent switch to the other update.
void gmres_alloc_z(Ctx& c, int m) {
  if (c.gZ_m >= m) return;
  if (c.gZ_m > 0) throw CudaError(AAO_ERR_CONFIG, "stored-Z restart larger than the first solve's is not supported");
  c.gZ = dalloc<double>(c, (size_t)m * c.N);
  std::vector<double*> zp(m);
  for (int i = 0; i < m; ++i) zp[i] = c.gZ + (size_t)i * c.N;
  c.gZptr = upload(c, zp);
  c.gZ_m = m;
}

double dot_host(Ctx& c, const double* x, const double* y, int mode, cudaStream_t s) {
  launch_dot(x, y, c.N, c.gpart, dot_blocks(), c.gscal, mode, s);
  launch_counter() += 2;
  CK(cudaMemcpyAsync(c.hostH, c.gscal, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return c.hostH[0];
}

aao_status gmres(Ctx& c, const double* b, double* x, const aao_krylov& kry, aao_info* info, double* hist, int hist_cap,
                 cudaStream_t s) {
  const int m = kry.restart;
  gmres_alloc(c, m);
  c.store_z = c.nonlinear || kry.store_z != 0;
  if (c.store_z) gmres_alloc_z(c, m);
  const long N = c.N;
  auto t0 = std::chrono::steady_clock::now();
  aao_info inf;
  std::memset(&inf, 0, sizeof(inf));
  inf.store_z = c.store_z ? 1 : 0;
  const long inner0 = c.inner_total;
  c.inner_max = 0;
  const double bnorm = dot_host(c, b, b, 1, s);
  int nh = 0;
  if (bnorm == 0.0) {
    CK(cudaMemsetAsync(x, 0, N * sizeof(double), s));
    CK(cudaStreamSynchronize(s));
    inf.converged = 1;
    if (info) *info = inf;
    return AAO_OK;
  }
  double* V0 = c.gV;
  // r = b - A x0, formed in V_0
  kkt_apply(c, x, V0, s);
  launch_copy_sub(V0, b, V0, N, s);
  ++launch_counter();
  int it = 0;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
  bool stop = false;
  for (;;) {
    const double beta0 = dot_host(c, V0, V0, 1, s);
    launch_scale_dev(V0, V0, c.gscal, N, s);
    ++launch_counter();
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta0;
    int kdone = 0;
    // Iteration k on the device: z_k = P^{-1} v_k, w = A z_k, MGS against v_0..v_k with w normalised on
    // the device (v_{k+1}), and the Hessenberg column copied to host buffer k & 1.  The linear path
    // enqueues iteration k+1 before the host has read column k (the host's Givens update and
    // convergence test overlap the next iteration); a solve that stops at k leaves one speculative
    // iteration in the stream whose results are never used.  Same arithmetic, same history.
    auto enqueue = [&](int k) {
      double* Vk = c.gV + (size_t)k * N;
      double* w = c.gV + (size_t)(k + 1) * N;
      double* zk = c.store_z ? c.gZ + (size_t)k * N : c.gz;
      if (c.timing) CK(cudaEventRecord(c.gt_ev[0], s));
      precond_apply(c, Vk, zk, s);
      if (c.timing) CK(cudaEventRecord(c.gt_ev[1], s));
      kkt_apply(c, zk, w, s);
      if (c.timing) CK(cudaEventRecord(c.gt_ev[2], s));
      double* hcol = c.gH + (size_t)k * (m + 1);
      int w_scaled = 0;
      CK(launch_mgs(w, (const double* const*)c.gVptr, k, N, hcol, c.gpart, c.gG, m + 2, s, &w_scaled));
      ++launch_counter();
      if (!w_scaled) {
        launch_scale_dev(w, w, hcol + k + 1, N, s);
        ++launch_counter();
      }
      if (c.timing) CK(cudaEventRecord(c.gt_ev[3], s));
      CK(cudaMemcpyAsync(c.hostH + (k & 1) * (m + 2), hcol, sizeof(double) * (k + 2), cudaMemcpyDeviceToHost, s));
      CK(cudaEventRecord(c.gm_ev[k & 1], s));
    };
    // Algorithm 2 synchronises inside precond_apply; phase timing reuses one event set per iteration
    const bool speculate = !c.nonlinear && !c.timing;
    enqueue(0);
    for (int k = 0; k < m; ++k) {
      if (speculate && k + 1 < m && it + 1 < kry.max_iters) enqueue(k + 1);
      CK(cudaEventSynchronize(c.gm_ev[k & 1]));
      inf.precond_applies++;
      if (c.timing) {
        float t01 = 0.f, t12 = 0.f, t23 = 0.f;
        CK(cudaEventElapsedTime(&t01, c.gt_ev[0], c.gt_ev[1]));
        CK(cudaEventElapsedTime(&t12, c.gt_ev[1], c.gt_ev[2]));
        CK(cudaEventElapsedTime(&t23, c.gt_ev[2], c.gt_ev[3]));
        inf.ms_precond += t01;
        inf.ms_kkt += t12;
        inf.ms_orth += t23;
      }
      const double* hh = c.hostH + (k & 1) * (m + 2);
      for (int i = 0; i <= k + 1; ++i) H[(size_t)i * m + k] = hh[i];
      // Givens rotations (same arithmetic as oracle/gmres.py)
      for (int i = 0; i < k; ++i) {
        const double t = cs[i] * H[(size_t)i * m + k] + sn[i] * H[(size_t)(i + 1) * m + k];
        H[(size_t)(i + 1) * m + k] = -sn[i] * H[(size_t)i * m + k] + cs[i] * H[(size_t)(i + 1) * m + k];
        H[(size_t)i * m + k] = t;
      }
      const double hkk = H[(size_t)k * m + k], hk1 = H[(size_t)(k + 1) * m + k];
      const double den = std::hypot(hkk, hk1);
      cs[k] = hkk / den;
      sn[k] = hk1 / den;
      H[(size_t)k * m + k] = den;
      H[(size_t)(k + 1) * m + k] = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      ++it;
      kdone = k + 1;
      const double rel = std::fabs(g[k + 1]) / bnorm;
      if (hist && nh < hist_cap) hist[nh++] = rel;
      inf.final_relres = rel;
      if (!std::isfinite(rel)) throw CudaError(AAO_ERR_NUMERIC, "NaN/Inf in GMRES");
      if (std::fabs(g[k + 1]) <= kry.tol * bnorm) {
        inf.converged = 1;
        stop = true;
        break;
      }
      if (hk1 < 1e-14 * bnorm) {
        inf.breakdown = 1;
        stop = true;
        break;
      }
      if (it >= kry.max_iters) {
        stop = true;
        break;
      }
      if (!speculate && k + 1 < m) enqueue(k + 1);
    }
    // x += P^{-1}(V_k y), H_k y = g_k
    for (int i = kdone - 1; i >= 0; --i) {
      double acc = g[i];
      for (int j = i + 1; j < kdone; ++j) acc -= H[(size_t)i * m + j] * y[j];
      y[i] = acc / H[(size_t)i * m + i];
    }
    CK(cudaMemcpyAsync(c.gscal + 8, y.data(), sizeof(double) * kdone, cudaMemcpyHostToDevice, s));
    if (c.store_z) {     // FGMRES, or linear with stored Z: x += Z_k y
      launch_multi_axpy(c.gz, (const double* const*)c.gZptr, c.gscal + 8, kdone, N, s);
      ++launch_counter();
    } else {             // GMRES: x += P^{-1}(V_k y)  (u = V y and P^{-1} u in place, in z)
      launch_multi_axpy(c.gz, (const double* const*)c.gVptr, c.gscal + 8, kdone, N, s);
      ++launch_counter();
      precond_apply(c, c.gz, c.gz, s);
      inf.precond_applies++;
    }
    launch_axpy(x, c.gz, 1.0, N, s);
    kkt_apply(c, x, V0, s);
    launch_copy_sub(V0, b, V0, N, s);
    launch_counter() += 2;
    inf.true_relres = dot_host(c, V0, V0, 1, s) / bnorm;
    if (stop) break;
    inf.restarts++;
  }
  inf.iterations = it;
  inf.inner_its_total = c.inner_total - inner0;
  inf.inner_its_max = c.inner_max;
  inf.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (info) *info = inf;
  return inf.converged ? AAO_OK : AAO_NOT_CONVERGED;
}

// m steps of Arnoldi on A P^{-1}, the GMRES iteration without the Givens update:
// v_0 = v0 / ||v0||, w = A P^{-1} v_k, MGS against v_0..v_k, h_{k+1,k} = ||w||.  H (host, row-major
// (m+1) x m, unrotated) receives the columns done; returns the number of steps (stops at breakdown).
int arnoldi(Ctx& c, const double* v0, int m, double* H, cudaStream_t s) {
  gmres_alloc(c, m);
  const long N = c.N;
  const double nrm = dot_host(c, v0, v0, 1, s);
  std::memset(H, 0, sizeof(double) * (size_t)(m + 1) * m);
  if (nrm == 0.0) return 0;
  launch_scale_dev(c.gV, v0, c.gscal, N, s);
  ++launch_counter();
  for (int k = 0; k < m; ++k) {
    double* Vk = c.gV + (size_t)k * N;
    double* w = c.gV + (size_t)(k + 1) * N;
    precond_apply(c, Vk, c.gz, s);
    kkt_apply(c, c.gz, w, s);
    double* hcol = c.gH + (size_t)k * (m + 1);
    int w_scaled = 0;
    CK(launch_mgs(w, (const double* const*)c.gVptr, k, N, hcol, c.gpart, c.gG, m + 2, s, &w_scaled));
    ++launch_counter();
    if (!w_scaled) {
      launch_scale_dev(w, w, hcol + k + 1, N, s);
      ++launch_counter();
    }
    CK(cudaMemcpyAsync(c.hostH, hcol, sizeof(double) * (k + 2), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int i = 0; i <= k + 1; ++i) H[(size_t)i * m + k] = c.hostH[i];
    if (!std::isfinite(c.hostH[k + 1])) throw CudaError(AAO_ERR_NUMERIC, "NaN/Inf in Arnoldi");
    if (c.hostH[k + 1] < 1e-14 * nrm) return k + 1;
  }
  return m;
}

}  // namespace
}  // namespace aao

// ====================================================================== C ABI
struct aao_ctx {
  aao::Ctx c;
  long launches_last = 0;
};

using aao::CudaError;

static aao_status fail(aao_ctx* ctx, aao_status st, const std::string& msg) {
  if (ctx) ctx->c.err = msg;
  return st;
}

#define ABI_GUARD(ctx, body)                                         \
  try {                                                              \
    ctx->c.err.clear();                                              \
    const long l0_ = aao::launch_counter();                          \
    body;                                                            \
    ctx->launches_last = aao::launch_counter() - l0_;                \
    cudaError_t e_ = cudaGetLastError();                             \
    if (e_ != cudaSuccess) return fail(ctx, AAO_ERR_CUDA, cudaGetErrorString(e_)); \
  } catch (const CudaError& e) {                                     \
    return fail(ctx, e.st, e.what());                                \
  } catch (const std::exception& e) {                                \
    return fail(ctx, AAO_ERR_CUDA, e.what());                        \
  }

extern "C" {

void aao_config_defaults(aao_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->dim = 2;
  cfg->n_cells = 8;
  cfg->x_lo = 0.0;
  cfg->x_hi = 1.0;
  cfg->n_t = 16;
  cfg->T = 1.0;
  cfg->beta = 1e-2;
  cfg->nu = 1e-2;
  cfg->problem = AAO_STOKES;
  cfg->wind_q2 = nullptr;
  cfg->mg_cycles = 4;
  cfg->pre_sweeps = 2;
  cfg->post_sweeps = 2;
  cfg->omega = 1.0;
  cfg->cheb_iters = 10;
  cfg->uzawa_iters = 6;
  cfg->uzawa_mu = 0.75;
  cfg->pmode = AAO_PRECOND_LINEAR;
  cfg->inner_eps = 1e-2;
  cfg->inner_maxit = 60;
  cfg->freq_chunk = 0;
}

aao_status aao_create(const aao_config* cfg, aao_ctx** out) {
  if (!cfg || !out) return AAO_ERR_SHAPE;
  *out = nullptr;
  const int N = cfg->n_cells;
  const bool pow2 = N >= 4 && (N & (N - 1)) == 0;
  if ((cfg->dim != 2 && cfg->dim != 3) || !pow2 || cfg->n_t < 3 || !(cfg->T > 0) || !(cfg->beta > 0) ||
      !(cfg->nu > 0) || !(cfg->x_hi > cfg->x_lo) || (cfg->problem != AAO_STOKES && cfg->problem != AAO_OSEEN) ||
      (cfg->problem == AAO_OSEEN && cfg->wind_q2 == nullptr) || cfg->mg_cycles < 1 || cfg->cheb_iters < 1 ||
      cfg->uzawa_iters < 1 || !(cfg->uzawa_mu > 0) || cfg->pre_sweeps < 0 || cfg->post_sweeps < 0 ||
      (cfg->pmode != AAO_PRECOND_LINEAR && cfg->pmode != AAO_PRECOND_NONLINEAR) ||
      (cfg->pmode == AAO_PRECOND_NONLINEAR && (!(cfg->inner_eps > 0) || !(cfg->inner_eps < 1) || cfg->inner_maxit < 1)) ||
      cfg->freq_chunk < 0)
    return AAO_ERR_CONFIG;
  aao_ctx* ctx = new aao_ctx();
  try {
    const char* mm = std::getenv("AAO_MG_MODE");
    ctx->c.mg_mode = (mm && std::atoi(mm) == 1) ? 1 : 0;
    const char* we = std::getenv("AAO_WAVE");
    ctx->c.wave_force = we ? std::atoi(we) : -1;
    const char* wm = std::getenv("AAO_WAVE_MIN");
    ctx->c.wave_min = wm ? std::atoi(wm) : 65;   // measured (triple form): c4_512 precond 175.9 (257) / 170.1 (129) /
                                                 // 169.3 ms (65); c2 2.07 / 1.92 / 1.84 ms
    const char* wh = std::getenv("AAO_WAVE_H");      // largest band height tried (24, 12, 6 or 3): tests force 3
    const int whv = wh ? std::atoi(wh) : 24;
    ctx->c.wave_hmax = (whv == 3 || whv == 6 || whv == 12) ? whv : 24;
    aao::setup(ctx->c, *cfg);
    for (auto& e : ctx->c.ev) cudaEventCreate(&e);
    cudaStreamCreateWithFlags(&ctx->c.s2, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&ctx->c.s3, cudaStreamNonBlocking);

    cudaEventCreateWithFlags(&ctx->c.ev_join2, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->c.ev_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->c.ev_join, cudaEventDisableTiming);
  } catch (const CudaError& e) {
    std::fprintf(stderr, "aao_create: %s\n", e.what());
    aao_status st = e.st;
    aao_destroy(ctx);
    return st;
  }
  *out = ctx;
  return AAO_OK;
}

void aao_destroy(aao_ctx* ctx) {
  if (!ctx) return;
  for (void* p : ctx->c.allocs) cudaFree(p);
  if (ctx->c.hostH) cudaFreeHost(ctx->c.hostH);
  for (auto e : ctx->c.gm_ev)
    if (e) cudaEventDestroy(e);
  for (auto e : ctx->c.gt_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->c.ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->c.prof_ev) cudaEventDestroy(e);
  if (ctx->c.s2) cudaStreamDestroy(ctx->c.s2);
  if (ctx->c.s3) cudaStreamDestroy(ctx->c.s3);
  if (ctx->c.ev_join2) cudaEventDestroy(ctx->c.ev_join2);
  if (ctx->c.ev_fork) cudaEventDestroy(ctx->c.ev_fork);
  if (ctx->c.ev_join) cudaEventDestroy(ctx->c.ev_join);
  delete ctx;
}

const char* aao_last_error(const aao_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }
size_t aao_vector_len(const aao_ctx* ctx) { return ctx ? (size_t)ctx->c.N : 0; }
size_t aao_device_bytes(const aao_ctx* ctx) { return ctx ? ctx->c.bytes : 0; }
long aao_last_launch_count(const aao_ctx* ctx) { return ctx ? ctx->launches_last : 0; }

aao_status aao_pack(aao_ctx* ctx, const double* in, double* out, void* stream) {
  if (!ctx || !in || !out) return AAO_ERR_SHAPE;
  ABI_GUARD(ctx, { aao::launch_mask_copy(ctx->c, in, out, (cudaStream_t)stream); ++aao::launch_counter(); });
  return AAO_OK;
}

aao_status aao_unpack(aao_ctx* ctx, const double* in, double* out, void* stream) {
  return aao_pack(ctx, in, out, stream);
}

aao_status aao_build_rhs(aao_ctx* ctx, const double* vd, double* b, void* stream) {
  if (!ctx || !vd || !b) return AAO_ERR_SHAPE;
  ABI_GUARD(ctx, { aao::launch_rhs(ctx->c, vd, b, (cudaStream_t)stream); ++aao::launch_counter(); });
  return AAO_OK;
}

aao_status aao_build_rhs_general(aao_ctx* ctx, const double* vd, const double* f, const double* g, const double* v0,
                                 double* b, void* stream) {
  if (!ctx || !b) return AAO_ERR_SHAPE;
  ABI_GUARD(ctx, { aao::launch_rhs_general(ctx->c, vd, f, g, v0, b, (cudaStream_t)stream); ++aao::launch_counter(); });
  return AAO_OK;
}

aao_status aao_arnoldi(aao_ctx* ctx, const double* v0, int m, double* H, int* m_done, void* stream) {
  if (!ctx || !v0 || !H || m < 1) return AAO_ERR_SHAPE;
  int k = 0;
  ABI_GUARD(ctx, { k = aao::arnoldi(ctx->c, v0, m, H, (cudaStream_t)stream); });
  if (m_done) *m_done = k;
  return AAO_OK;
}

aao_status aao_kkt_apply(aao_ctx* ctx, const double* x, double* y, void* stream) {
  if (!ctx || !x || !y || x == y) return AAO_ERR_SHAPE;
  ABI_GUARD(ctx, { aao::kkt_apply(ctx->c, x, y, (cudaStream_t)stream); });
  return AAO_OK;
}

aao_status aao_precond_apply(aao_ctx* ctx, const double* r, double* z, void* stream) {
  if (!ctx || !r || !z || r == z) return AAO_ERR_SHAPE;
  ABI_GUARD(ctx, { aao::precond_apply(ctx->c, r, z, (cudaStream_t)stream); });
  return AAO_OK;
}

static bool krylov_ok(const aao_krylov* kry) {
  return kry && kry->restart >= 1 && kry->restart <= 64 && kry->tol > 0 && kry->max_iters >= 1 &&
         (kry->store_z == 0 || kry->store_z == 1);
}

aao_status aao_gmres_solve(aao_ctx* ctx, const double* b, double* x, const aao_krylov* kry, aao_info* info,
                           double* hist, int hist_cap, void* stream) {
  if (!ctx || !b || !x || !krylov_ok(kry) || b == x) return AAO_ERR_SHAPE;
  aao_status st = AAO_OK;
  ABI_GUARD(ctx, { st = aao::gmres(ctx->c, b, x, *kry, info, hist, hist_cap, (cudaStream_t)stream); });
  return st;
}

aao_status aao_gmres_solve_host(aao_ctx* ctx, const double* b_host, double* x_host, const aao_krylov* kry,
                                aao_info* info, double* hist, int hist_cap, void* stream) {
  if (!ctx || !b_host || !x_host || b_host == x_host || !krylov_ok(kry)) return AAO_ERR_SHAPE;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = ctx->c.N * sizeof(double);
  try {
    ctx->c.err.clear();
    aao::gmres_alloc(ctx->c, kry->restart);
    // device staging for b and x, allocated once per context (owned, freed by aao_destroy)
    if (!ctx->c.stage_b) {
      ctx->c.stage_b = aao::dalloc<double>(ctx->c, ctx->c.N);
      ctx->c.stage_x = aao::dalloc<double>(ctx->c, ctx->c.N);
    }
  } catch (const CudaError& e) {
    return fail(ctx, e.st, e.what());
  }
  double *db = ctx->c.stage_b, *dx = ctx->c.stage_x;
  cudaError_t e1 = cudaMemcpyAsync(db, b_host, bytes, cudaMemcpyHostToDevice, s);
  cudaError_t e2 = e1 == cudaSuccess ? cudaMemcpyAsync(dx, x_host, bytes, cudaMemcpyHostToDevice, s) : e1;
  if (e2 != cudaSuccess) return fail(ctx, AAO_ERR_CUDA, std::string("host -> device copy: ") + cudaGetErrorString(e2));
  const aao_status st = aao_gmres_solve(ctx, db, dx, kry, info, hist, hist_cap, stream);
  if (st < 0) return st;   // x_host untouched on error
  cudaError_t e3 = cudaMemcpyAsync(x_host, dx, bytes, cudaMemcpyDeviceToHost, s);
  if (e3 == cudaSuccess) e3 = cudaStreamSynchronize(s);
  if (e3 != cudaSuccess) return fail(ctx, AAO_ERR_CUDA, std::string("device -> host copy: ") + cudaGetErrorString(e3));
  return st;
}

aao_status aao_debug_freq_block(aao_ctx* ctx, int k, double* out, void* stream) {
  if (!ctx || !out || k < 0 || k >= ctx->c.n_f) return AAO_ERR_SHAPE;
  ABI_GUARD(ctx, {
    cudaStream_t s = (cudaStream_t)stream;
    double2* tmp = nullptr;
    if (cudaMalloc(&tmp, 2 * ctx->c.nblk * sizeof(double2)) != cudaSuccess)
      throw CudaError(AAO_ERR_OOM, "debug block alloc");
    aao::launch_debug_block(ctx->c, k, tmp, s);
    cudaMemcpyAsync(out, tmp, 2 * ctx->c.nblk * sizeof(double2), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(tmp);
  });
  return AAO_OK;
}

int aao_last_inner_iterations(const aao_ctx* ctx, int* out, int cap) {
  if (!ctx || !out || cap < 0) return AAO_ERR_SHAPE;
  const int n = std::min<int>(cap, (int)ctx->c.inner_its.size());
  for (int i = 0; i < n; ++i) out[i] = ctx->c.inner_its[i];
  return n;
}

aao_status aao_set_timing(aao_ctx* ctx, int on) {
  if (!ctx) return AAO_ERR_SHAPE;
  ctx->c.timing = on != 0;
  return AAO_OK;
}

aao_status aao_profile_smoother(aao_ctx* ctx, int on) {
  if (!ctx || on < 0) return AAO_ERR_SHAPE;
  auto& c = ctx->c;
  c.prof = on != 0;
  c.prof_used = 0;
  c.prof_bytes = 0;
  c.prof_launches = 0;
  // on > 1: create the events for `on` launches now, so that none is created inside a timed region
  while (on > 1 && c.prof_ev.size() < 2 * (size_t)on) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return fail(ctx, AAO_ERR_CUDA, "cudaEventCreate");
    c.prof_ev.push_back(e);
  }
  return AAO_OK;
}

aao_status aao_profile_read(aao_ctx* ctx, double* out3) {
  if (!ctx || !out3) return AAO_ERR_SHAPE;
  auto& c = ctx->c;
  double ms = 0;
  if (c.prof_used) cudaEventSynchronize(c.prof_ev[c.prof_used - 1]);
  for (size_t i = 0; i + 1 < c.prof_used; i += 2) {
    float t = 0;
    cudaEventElapsedTime(&t, c.prof_ev[i], c.prof_ev[i + 1]);
    ms += t;
  }
  out3[0] = ms;
  out3[1] = c.prof_bytes;
  out3[2] = (double)c.prof_launches;
  c.prof_used = 0;
  c.prof_bytes = 0;
  c.prof_launches = 0;
  return AAO_OK;
}

aao_status aao_last_phase_ms(aao_ctx* ctx, double* ms4) {
  if (!ctx || !ms4) return AAO_ERR_SHAPE;
  for (int i = 0; i < 4; ++i) ms4[i] = 0.0;
  if (!ctx->c.timing) return fail(ctx, AAO_ERR_CONFIG, "timing not enabled (aao_set_timing)");
  if (!ctx->c.phase_valid)
    return fail(ctx, AAO_ERR_CONFIG, "no linear precond_apply recorded with timing on since the last apply");
  if (cudaEventSynchronize(ctx->c.ev[4]) != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(ctx, AAO_ERR_CUDA, "phase event synchronisation failed");
  }
  for (int i = 0; i < 4; ++i) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, ctx->c.ev[i], ctx->c.ev[i + 1]) != cudaSuccess) {
      (void)cudaGetLastError();   // leave no pending error for the next ABI call
      return fail(ctx, AAO_ERR_CUDA, "phase event elapsed time failed");
    }
    ms4[i] = t;
  }
  return AAO_OK;
}

}  // extern "C"
