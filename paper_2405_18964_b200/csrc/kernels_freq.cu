// Batched frequency-vector kernels for the nonlinear preconditioner (Algorithm 2):
// one inner GMRES per frequency, all frequencies in lockstep.  A "frequency vector" is the pair
// (velocity part [k][half][comp][node], pressure part [k][half][node]) in the layout of Fv / Fp;
// every kernel works per frequency k with deterministic fixed-order reductions.
#include "aao_internal.h"

namespace aao {

namespace {

__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;
}

__device__ __forceinline__ double2 block_sum2(double2 v) {
  __shared__ double2 ws[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum2(v);
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  v = threadIdx.x < nw ? ws[threadIdx.x] : make_double2(0.0, 0.0);
  if (wid == 0) v = warp_sum2(v);
  return v;
}

constexpr int FD_BLOCKS = 16;   // blocks per frequency for the dot partials
constexpr int FD_THREADS = 256;

// partial[k][blk] = sum over this block's share of  conj(a_k) . b_k  (velocity then pressure part)
__global__ void k_fdot_partial(FVec a, FVec b, long LV, long LP, double2* partial) {
  const int k = blockIdx.y;
  const double2* av = a.v + (long)k * LV;
  const double2* bv = b.v + (long)k * LV;
  const double2* ap = a.p + (long)k * LP;
  const double2* bp = b.p + (long)k * LP;
  double2 acc = make_double2(0.0, 0.0);
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < LV; i += stride) {
    const double2 t = cmulc(av[i], bv[i]);
    acc.x += t.x;
    acc.y += t.y;
  }
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < LP; i += stride) {
    const double2 t = cmulc(ap[i], bp[i]);
    acc.x += t.x;
    acc.y += t.y;
  }
  acc = block_sum2(acc);
  if (threadIdx.x == 0) partial[(long)k * gridDim.x + blockIdx.x] = acc;
}

// out[k] = sum of the partials (mode 1: sqrt of the real part, imaginary 0)
__global__ void k_fdot_final(const double2* partial, int nb, int nf, double2* out, int mode) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nf) return;
  double2 s = make_double2(0.0, 0.0);
  for (int b = 0; b < nb; ++b) {
    s.x += partial[(long)k * nb + b].x;
    s.y += partial[(long)k * nb + b].y;
  }
  out[k] = mode == 1 ? make_double2(sqrt(s.x), 0.0) : s;
}

// y_k += sign * coef[k] * x_k
__global__ void k_faxpy(FVec y, FVec x, const double2* coef, double sign, long LV, long LP) {
  const int k = blockIdx.y;
  const double2 c = make_double2(sign * coef[k].x, sign * coef[k].y);
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < LV + LP; i += stride) {
    double2* yy = i < LV ? y.v + (long)k * LV + i : y.p + (long)k * LP + (i - LV);
    const double2 xx = i < LV ? x.v[(long)k * LV + i] : x.p[(long)k * LP + (i - LV)];
    *yy = make_double2(yy->x + c.x * xx.x - c.y * xx.y, yy->y + c.x * xx.y + c.y * xx.x);
  }
}

// y_k = x_k / den[k].x (0 where den is 0 or the frequency is frozen)
__global__ void k_fscale(FVec y, FVec x, const double2* den, const int* frozen, long LV, long LP) {
  const int k = blockIdx.y;
  const double d = den[k].x;
  const double s = (frozen[k] || d == 0.0) ? 0.0 : 1.0 / d;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < LV + LP; i += stride) {
    if (i < LV) {
      const double2 xx = x.v[(long)k * LV + i];
      y.v[(long)k * LV + i] = make_double2(s * xx.x, s * xx.y);
    } else {
      const double2 xx = x.p[(long)k * LP + (i - LV)];
      y.p[(long)k * LP + (i - LV)] = make_double2(s * xx.x, s * xx.y);
    }
  }
}

// u_k = sum_j Y[k][j] V_j,k  (V_j = basis vector j; Y row-major [nf][m])
__global__ void k_fmulti(FVec u, const FVec* V, const double2* Y, int m, long LV, long LP) {
  const int k = blockIdx.y;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < LV + LP; i += stride) {
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < m; ++j) {
      const double2 c = Y[(long)k * m + j];
      const double2 xx = i < LV ? V[j].v[(long)k * LV + i] : V[j].p[(long)k * LP + (i - LV)];
      acc.x += c.x * xx.x - c.y * xx.y;
      acc.y += c.x * xx.y + c.y * xx.x;
    }
    if (i < LV)
      u.v[(long)k * LV + i] = acc;
    else
      u.p[(long)k * LP + (i - LV)] = acc;
  }
}

// Stokes pressure slots of P~_k^{-1}: out = (1 + c_{k,1}) K_p^{-1} s + nu c_{k,2} M_p^{-1} s
__global__ void k_combine_p(double2* out, const double2* A, const double2* Bc, const FreqConst* fc, double nu, long LP) {
  const int k = blockIdx.y;
  const double ca = 1.0 + fc[k].c1, cb = nu * fc[k].c2;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < LP; i += stride) {
    const long o = (long)k * LP + i;
    out[o] = make_double2(ca * A[o].x + cb * Bc[o].x, ca * A[o].y + cb * Bc[o].y);
  }
}

// Oseen P~^(UZ) outputs (X1, X2 as [k][comp][node]; XpA as [k][half][node]) into a frequency vector
__global__ void k_oseen_scatter(FVec out, const double2* X1, const double2* X2, const double2* XpA, double pscale,
                                long ncomp_nodes, long LP) {
  const int k = blockIdx.y;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * ncomp_nodes + LP; i += stride) {
    if (i < ncomp_nodes)
      out.v[(long)k * 2 * ncomp_nodes + i] = X1[(long)k * ncomp_nodes + i];
    else if (i < 2 * ncomp_nodes)
      out.v[(long)k * 2 * ncomp_nodes + i] = X2[(long)k * ncomp_nodes + (i - ncomp_nodes)];
    else {
      const double2 a = XpA[(long)k * LP + (i - 2 * ncomp_nodes)];
      out.p[(long)k * LP + (i - 2 * ncomp_nodes)] = make_double2(pscale * a.x, pscale * a.y);
    }
  }
}

// out velocity (half h, comp c) += s * (B^T q)_c, q = pressure half qh of the same frequency
// B_c = -(prod of Pm, Gm on axis c); pinned pressure node contributes nothing (q_0 = 0)
template <int DIM>
__global__ void k_fBT(FVec out, int h, FVec q, int qh, double s, int n1, int m1, long ns, long np,
                      const double* __restrict__ tPmT, const double* __restrict__ tGmT) {
  const long node = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= ns) return;
  const int k = blockIdx.y / DIM, comp = blockIdx.y % DIM;
  int c[3];
  c[0] = (int)(node % n1);
  c[1] = (int)((node / n1) % n1);
  c[2] = DIM == 3 ? (int)(node / ((long)n1 * n1)) : 0;
  for (int a = 0; a < DIM; ++a)
    if (c[a] == 0 || c[a] == n1 - 1) return;
  const double2* qq = q.p + ((long)k * 2 + qh) * np;
  double2 acc = make_double2(0.0, 0.0);
  int I0[3];
  for (int a = 0; a < DIM; ++a) I0[a] = (c[a] - 1) / 2;
  for (int oc = 0; oc < (DIM == 3 ? 3 : 1); ++oc) {
    const int Kz = DIM == 3 ? I0[2] + oc : 0;
    const double fz = DIM == 3 ? (comp == 2 ? tGmT[c[2] * 3 + oc] : tPmT[c[2] * 3 + oc]) : 1.0;
    if (fz == 0.0 || Kz >= m1) continue;
    for (int ob = 0; ob < 3; ++ob) {
      const int J = I0[1] + ob;
      const double fy = comp == 1 ? tGmT[c[1] * 3 + ob] : tPmT[c[1] * 3 + ob];
      if (fy == 0.0 || J >= m1) continue;
      for (int oa = 0; oa < 3; ++oa) {
        const int I = I0[0] + oa;
        const double fx = comp == 0 ? tGmT[c[0] * 3 + oa] : tPmT[c[0] * 3 + oa];
        if (fx == 0.0 || I >= m1) continue;
        const long pn = ((long)Kz * m1 + J) * m1 + I;
        const double2 v = qq[pn];
        const double w = -fz * fy * fx;
        acc.x += w * v.x;
        acc.y += w * v.y;
      }
    }
  }
  double2* o = out.v + (((long)k * 2 + h) * DIM + comp) * ns + node;
  *o = make_double2(o->x + s * acc.x, o->y + s * acc.y);
}

dim3 fgrid(long len, int nf) {
  long b = (len + 255) / 256;
  if (b > 256) b = 256;
  return dim3((unsigned)b, nf);
}

}  // namespace

void launch_fdot(FVec a, FVec b, long LV, long LP, int nf, double2* partial, double2* out, int mode, cudaStream_t s) {
  k_fdot_partial<<<dim3(FD_BLOCKS, nf), FD_THREADS, 0, s>>>(a, b, LV, LP, partial);
  k_fdot_final<<<(nf + 127) / 128, 128, 0, s>>>(partial, FD_BLOCKS, nf, out, mode);
}
size_t fdot_partial_len(int nf) { return (size_t)FD_BLOCKS * nf; }

void launch_faxpy(FVec y, FVec x, const double2* coef, double sign, long LV, long LP, int nf, cudaStream_t s) {
  k_faxpy<<<fgrid(LV + LP, nf), 256, 0, s>>>(y, x, coef, sign, LV, LP);
}
void launch_fscale(FVec y, FVec x, const double2* den, const int* frozen, long LV, long LP, int nf, cudaStream_t s) {
  k_fscale<<<fgrid(LV + LP, nf), 256, 0, s>>>(y, x, den, frozen, LV, LP);
}
void launch_fmulti(FVec u, const FVec* V, const double2* Y, int m, long LV, long LP, int nf, cudaStream_t s) {
  k_fmulti<<<fgrid(LV + LP, nf), 256, 0, s>>>(u, V, Y, m, LV, LP);
}
void launch_combine_p(double2* out, const double2* A, const double2* B, const FreqConst* fc, double nu, long LP, int nf,
                      cudaStream_t s) {
  k_combine_p<<<fgrid(LP, nf), 256, 0, s>>>(out, A, B, fc, nu, LP);
}
void launch_oseen_scatter(FVec out, const double2* X1, const double2* X2, const double2* XpA, double pscale,
                          long ncomp_nodes, long LP, int nf, cudaStream_t s) {
  k_oseen_scatter<<<fgrid(2 * ncomp_nodes + LP, nf), 256, 0, s>>>(out, X1, X2, XpA, pscale, ncomp_nodes, LP);
}
void launch_fBT(const Ctx& c, FVec out, int h, FVec q, int qh, double sc, cudaStream_t s) {
  dim3 g((unsigned)((c.n_s + 127) / 128), c.n_f * c.dim);
  if (c.dim == 2)
    k_fBT<2><<<g, 128, 0, s>>>(out, h, q, qh, sc, c.n1q2, c.n1q1, c.n_s, c.n_p, c.tPmT, c.tGmT);
  else
    k_fBT<3><<<g, 128, 0, s>>>(out, h, q, qh, sc, c.n1q2, c.n1q1, c.n_s, c.n_p, c.tPmT, c.tGmT);
}

}  // namespace aao
