// GMRES vector kernels (step A1): deterministic two-stage reductions with warp
// shuffles (fixed grid, fixed order -> bitwise reproducible), device-scalar axpys
// so Gram-Schmidt coefficients never round-trip through the host.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "aao_internal.h"

namespace cg = cooperative_groups;

namespace aao {

constexpr int DOT_BLOCKS = 4 * 148;
constexpr int DOT_THREADS = 256;
int dot_blocks() { return DOT_BLOCKS; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  v = threadIdx.x < nw ? ws[threadIdx.x] : 0.0;
  if (wid == 0) v = warp_sum(v);
  return v;  // valid in thread 0
}

__global__ void k_dot_partial(const double* __restrict__ x, const double* __restrict__ y, long n,
                              double* __restrict__ partial) {
  double acc = 0.0;
  const long stride = (long)gridDim.x * blockDim.x;
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  // 2-way unrolled grid-stride loop with vectorised loads when aligned
  for (; i < n; i += stride) acc = fma(__ldg(x + i), __ldg(y + i), acc);
  acc = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void k_dot_final(const double* __restrict__ partial, int nb, double* out, int mode) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += partial[i];
  acc = block_sum(acc);
  if (threadIdx.x == 0) *out = mode == 1 ? sqrt(acc) : acc;
}

void launch_dot(const double* x, const double* y, long n, double* partial, int nblk, double* out, int mode,
                cudaStream_t s) {
  k_dot_partial<<<nblk, DOT_THREADS, 0, s>>>(x, y, n, partial);
  k_dot_final<<<1, 1024, 0, s>>>(partial, nblk, out, mode);
}

__global__ void k_axpy_dev(double* __restrict__ y, const double* __restrict__ x, const double* __restrict__ alpha,
                           double sign, long n) {
  const double a = sign * *alpha;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = fma(a, x[i], y[i]);
}
void launch_axpy_dev(double* y, const double* x, const double* alpha, double sign, long n, cudaStream_t s) {
  k_axpy_dev<<<DOT_BLOCKS, 256, 0, s>>>(y, x, alpha, sign, n);
}

// y and x may alias (in-place scaling)
__global__ void k_scale_dev(double* y, const double* x, const double* __restrict__ den,
                            long n) {
  const double a = 1.0 / *den;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = x[i] * a;
}
void launch_scale_dev(double* y, const double* x, const double* denom, long n, cudaStream_t s) {
  k_scale_dev<<<DOT_BLOCKS, 256, 0, s>>>(y, x, denom, n);
}

__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ x, double a, long n) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = fma(a, x[i], y[i]);
}
void launch_axpy(double* y, const double* x, double alpha, long n, cudaStream_t s) {
  k_axpy<<<DOT_BLOCKS, 256, 0, s>>>(y, x, alpha, n);
}

// y and ax may alias (r = b - A x formed in place)
__global__ void k_copy_sub(double* y, const double* __restrict__ b, const double* ax,
                           long n) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) y[i] = b[i] - ax[i];
}
void launch_copy_sub(double* y, const double* b, const double* ax, long n, cudaStream_t s) {
  k_copy_sub<<<DOT_BLOCKS, 256, 0, s>>>(y, b, ax, n);
}

// u = sum_{i<k} coef[i] * V_i, V_i = V[i]
__global__ void k_multi_axpy(double* __restrict__ u, const double* const* __restrict__ V,
                             const double* __restrict__ coef, int k, long n) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long j = (long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    double acc = 0.0;
    for (int i = 0; i < k; ++i) acc = fma(coef[i], V[i][j], acc);
    u[j] = acc;
  }
}
void launch_multi_axpy(double* u, const double* const* V, const double* coef, int k, long n, cudaStream_t s) {
  k_multi_axpy<<<DOT_BLOCKS, 256, 0, s>>>(u, V, coef, k, n);
}

// Modified Gram-Schmidt of w against V_0..V_k in ONE cooperative launch (step A1):
//   h_i = <w, V_i>; w -= h_i V_i  (i = 0..k, sequentially, as MGS requires);  h_{k+1} = ||w||.
// Each block owns a fixed contiguous chunk; the dot for step i+1 is fused into the update pass of
// step i, so every step costs one pass over the chunk and one grid barrier.  Block partials are
// reduced in a fixed order by every block (deterministic, bitwise reproducible).
#ifndef MGS_THREADS
#define MGS_THREADS 512
#endif
#ifndef MGS_PER_SM
#define MGS_PER_SM 1
#endif

// Streaming version for vectors too large for the on-chip variant below: the update/dot pass works on double2
// (n even: N = 2 n_b (n_v + n_p)) with four elements per thread in flight per round (12 independent 16-byte loads),
// enough memory-level parallelism for one 1024-thread CTA per SM to stream at HBM rate.
constexpr int MGS_U = 4;

__global__ void __launch_bounds__(MGS_THREADS) k_mgs(double* __restrict__ w, const double* const* __restrict__ V,
                                                     int k, long n, double* __restrict__ H,
                                                     double* __restrict__ partial) {
  cg::grid_group grid = cg::this_grid();
  const int nb = gridDim.x;
  const long chunk = ((n + nb - 1) / nb + 1) / 2 * 2;   // even: double2 aligned
  const long lo = min(n, blockIdx.x * chunk), hi = min(n, lo + chunk);
  __shared__ double hs;
  // dot for step 0
  double acc = 0.0;
  {
    const double2* v0 = reinterpret_cast<const double2*>(V[0] + lo);
    const double2* w2 = reinterpret_cast<const double2*>(w + lo);
    const long m = (hi - lo) / 2;
    for (long e = threadIdx.x; e < m; e += blockDim.x) {
      const double2 a = w2[e], b = __ldcg(v0 + e);
      acc = fma(a.x, b.x, acc);
      acc = fma(a.y, b.y, acc);
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
  grid.sync();
  for (int i = 0; i <= k; ++i) {
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int b = threadIdx.x; b < nb; b += 32) s += partial[(long)i * nb + b];
      s = warp_sum(s);
      if (threadIdx.x == 0) {
        hs = s;
        if (blockIdx.x == 0) H[i] = s;
      }
    }
    __syncthreads();
    const double h = hs;
    const double2* vi = reinterpret_cast<const double2*>(V[i] + lo);
    const double2* vn = reinterpret_cast<const double2*>((i < k ? V[i + 1] : w) + lo);
    double2* w2 = reinterpret_cast<double2*>(w + lo);
    const long m = (hi - lo) / 2;                 // double2 elements of this chunk
    const long step = (long)blockDim.x * MGS_U;
    double a2 = 0.0;
    for (long base = threadIdx.x; base < m; base += step) {
      double2 ww[MGS_U], vv[MGS_U], nn[MGS_U];
#pragma unroll
      for (int u = 0; u < MGS_U; ++u) {
        const long e = base + (long)u * blockDim.x;
        if (e < m) {
          ww[u] = w2[e];
          vv[u] = __ldcs(vi + e);
          if (i < k) nn[u] = __ldcg(vn + e);
        }
      }
#pragma unroll
      for (int u = 0; u < MGS_U; ++u) {
        const long e = base + (long)u * blockDim.x;
        if (e < m) {
          double2 x;
          x.x = fma(-h, vv[u].x, ww[u].x);
          x.y = fma(-h, vv[u].y, ww[u].y);
          w2[e] = x;
          const double2 y = i < k ? nn[u] : x;
          a2 = fma(x.x, y.x, a2);
          a2 = fma(x.y, y.y, a2);
        }
      }
    }
    a2 = block_sum(a2);
    if (threadIdx.x == 0) partial[(long)(i + 1) * nb + blockIdx.x] = a2;
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nb; b += 32) s += partial[(long)(k + 1) * nb + b];
    s = warp_sum(s);
    if (threadIdx.x == 0) H[k + 1] = sqrt(s);
  }
}

// ---- MGS in its inverse-compact-WY form for vectors too large for the on-chip variant (c4 at n_t >= 32).
// MGS computes h_i = <v_i, w^(i)>, w^(i+1) = w^(i) - h_i v_i (i = 0..k).  Since w^(i) = w - sum_{j<i} h_j v_j,
//   h_i = s_i - sum_{j<i} <v_i, v_j> h_j,   s_i = <v_i, w>,
// a forward substitution with the strictly lower Gram matrix of the basis (Swirydowicz et al., "Low
// synchronization Gram-Schmidt and GMRES algorithms", 2020: the same loss of orthogonality as MGS).  The
// Gram row of v_{k+1} is formed in the update pass that creates it, so one step is two passes over the
// basis instead of k+1: pass 1 reads w and v_0..v_k once (all k+1 dots); pass 2 reads them again and
// writes w_new = w - h_0 v_0 - ... - h_k v_k (the same per-element FMA order as MGS), accumulating
// <w_new, v_j> (-> Gram row k+1) and ||w_new||^2.  HBM traffic per step (2k+5) vectors instead of
// 4(k+1)+2.  Gram rows live in G (ld = ldg), row i valid for the current restart cycle once v_i exists.
constexpr int MGSW_THREADS = 256;

__device__ __forceinline__ double dot2(double2 a, double2 b) { return fma(a.x, b.x, a.y * b.y); }

// Block sums of acc[i] for i < cnt and of acc[NA - 1] (when last), written to out[i] / out[NA - 1].
template <int NA>
__device__ __forceinline__ void block_sum_many(const double* acc, int cnt, bool last, double* red /* [nw][NA] */,
                                               double* out /* [NA] */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NA; ++i) {
    if (i < cnt || (last && i == NA - 1)) {
      const double v = warp_sum(acc[i]);
      if (lane == 0) red[wid * NA + i] = v;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NA; i += blockDim.x) {
    if (i < cnt || (last && i == NA - 1)) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += red[w * NA + i];
      out[i] = s;
    }
  }
  __syncthreads();
}

// KMAX = 32 runs one CTA per SM so that a thread can hold the 32 basis values of its element in registers between
// the update and the Gram dots of pass 2 (with two CTAs per SM and 128 registers the second use re-read them through
// L2: measured 2.9-3.4 TB/s against 5.8 TB/s for KMAX = 16 on c4 at n_t = 512).
template <int KMAX>
__global__ void __launch_bounds__(MGSW_THREADS, KMAX > 16 ? 1 : 2)
    k_mgs_icwy(double* __restrict__ w, const double* const* __restrict__ V, int k, long n2,
               double* __restrict__ H, double* __restrict__ partial, double* __restrict__ G, int ldg) {
  constexpr int NA = KMAX + 1;
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[(MGSW_THREADS / 32) * NA];
  __shared__ double bs[NA], hs[KMAX];
  __shared__ const double2* vp[KMAX];
  const int nb = gridDim.x, T = blockDim.x, tid = threadIdx.x;
  const long chunk = (n2 + nb - 1) / nb;
  const long lo = min(n2, (long)blockIdx.x * chunk), cnt = min(n2, lo + chunk) - lo;
  const int K1 = k + 1;
  if (tid < K1) vp[tid] = reinterpret_cast<const double2*>(V[tid]) + lo;
  double2* w2 = reinterpret_cast<double2*>(w) + lo;
  __syncthreads();
  // pass 1: s_i = <v_i, w>, i = 0..k
  double acc[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) acc[i] = 0.0;
  for (long e = tid; e < cnt; e += T) {
    const double2 x = w2[e];
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < K1) acc[i] += dot2(x, __ldcs(vp[i] + e));
  }
  block_sum_many<NA>(acc, K1, false, red, bs);
  for (int i = tid; i < K1; i += T) partial[(long)i * nb + blockIdx.x] = bs[i];
  grid.sync();
  // every block: s_i summed in a fixed order, then h_i = s_i - sum_{j<i} G_ij h_j
  for (int i = tid; i < K1; i += T) {
    double sm = 0.0;
    for (int b = 0; b < nb; ++b) sm += partial[(long)i * nb + b];
    bs[i] = sm;
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 0; i < K1; ++i) {
      double h = bs[i];
      for (int j = 0; j < i; ++j) h -= G[(long)i * ldg + j] * hs[j];
      hs[i] = h;
      if (blockIdx.x == 0) H[i] = h;
    }
  }
  __syncthreads();
  // pass 2: w_new = w - h_0 v_0 - ... - h_k v_k (MGS order), q_j = <w_new, v_j>, ||w_new||^2 (acc[KMAX])
#pragma unroll
  for (int i = 0; i < NA; ++i) acc[i] = 0.0;
  for (long e = tid; e < cnt; e += T) {
    double2 x = w2[e];
    double2 v[KMAX];
#pragma unroll
    for (int i = 0; i < KMAX; ++i) v[i] = i < K1 ? __ldcs(vp[i] + e) : make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
      if (i < K1) {
        x.x = fma(-hs[i], v[i].x, x.x);
        x.y = fma(-hs[i], v[i].y, x.y);
      }
    }
    w2[e] = x;
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i < K1) acc[i] += dot2(x, v[i]);
    acc[KMAX] += dot2(x, x);
  }
  block_sum_many<NA>(acc, K1, true, red, bs);
  for (int i = tid; i < K1; i += T) partial[(long)(K1 + i) * nb + blockIdx.x] = bs[i];
  if (tid == 0) partial[(long)(2 * K1) * nb + blockIdx.x] = bs[KMAX];
  grid.sync();
  if (blockIdx.x == 0) {
    for (int i = tid; i <= K1; i += T) {
      double sm = 0.0;
      for (int b = 0; b < nb; ++b) sm += partial[(long)(K1 + i) * nb + b];
      bs[i] = sm;
    }
    __syncthreads();
    const double hn = sqrt(bs[K1]);
    if (tid == 0) H[K1] = hn;
    for (int j = tid; j < K1; j += T) G[(long)K1 * ldg + j] = hn > 0.0 ? bs[j] / hn : 0.0;
  }
}

// ---- MGS with the new vector w held on chip (registers + shared memory) for all k+1 passes.
// One 1024-thread CTA per SM owns a contiguous chunk of w (in double2 units): the first R2*1024
// double2 in registers (slot r of thread t holds element r*1024+t, coalesced), the rest in
// dynamic shared memory.  Pass i reads only v_i (just streamed by the previous pass as v_{i+1},
// so it is served by L2) and v_{i+1} from HBM: one vector of HBM traffic per pass instead of the
// streaming kernel's four.  The last pass also forms ||w|| and writes w back scaled by
// 1/h_{k+1,k} (the next basis vector), removing the separate scale pass.  Same arithmetic per
// element as k_mgs (h_i = <w, v_i>, w -= h_i v_i), different (fixed) reduction partition.
constexpr int MGS_OC_THREADS = 1024;
constexpr int MGS_OC_R2 = 4;

template <int R2>
__global__ void __launch_bounds__(MGS_OC_THREADS, 1)
    k_mgs_oc(double* __restrict__ w, const double* const* __restrict__ V, int k, long n2, long C2,
             double* __restrict__ H, double* __restrict__ partial, int scale) {
  extern __shared__ double2 wsm[];
  cg::grid_group grid = cg::this_grid();
  const int nb = gridDim.x, T = MGS_OC_THREADS, tid = threadIdx.x;
  const long lo = (long)blockIdx.x * C2;
  const int cnt = (int)max(0L, min(n2, lo + C2) - lo);
  const int nsm = max(0, cnt - R2 * T);
  double2* w2 = reinterpret_cast<double2*>(w) + lo;
  __shared__ double hs;
  double2 wr[R2];
  {
    const double2* v0 = reinterpret_cast<const double2*>(V[0]) + lo;
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < R2; ++r) {
      const int e = r * T + tid;
      wr[r] = e < cnt ? w2[e] : make_double2(0.0, 0.0);
      if (e < cnt) acc += dot2(wr[r], __ldcg(v0 + e));
    }
#pragma unroll 4
    for (int e = tid; e < nsm; e += T) {
      const double2 x = w2[R2 * T + e];
      wsm[e] = x;
      acc += dot2(x, __ldcg(v0 + R2 * T + e));
    }
    acc = block_sum(acc);
    if (tid == 0) partial[blockIdx.x] = acc;
  }
  grid.sync();
  for (int i = 0; i <= k; ++i) {
    if (tid < 32) {
      double sm = 0.0;
      for (int b = tid; b < nb; b += 32) sm += partial[(long)i * nb + b];
      sm = warp_sum(sm);
      if (tid == 0) {
        hs = sm;
        if (blockIdx.x == 0) H[i] = sm;
      }
    }
    __syncthreads();
    const double h = hs;
    const double2* vi = reinterpret_cast<const double2*>(V[i]) + lo;
    const double2* vn = reinterpret_cast<const double2*>(i < k ? V[i + 1] : w) + lo;
    const bool last = i == k;
    double a2 = 0.0;
#pragma unroll
    for (int r = 0; r < R2; ++r) {
      const int e = r * T + tid;
      if (e < cnt) {
        const double2 a = __ldcg(vi + e);
        double2 x = wr[r];
        x.x = fma(-h, a.x, x.x);
        x.y = fma(-h, a.y, x.y);
        wr[r] = x;
        a2 += dot2(x, last ? x : __ldcg(vn + e));
      }
    }
#pragma unroll 4
    for (int e = tid; e < nsm; e += T) {
      const double2 a = __ldcg(vi + R2 * T + e);
      double2 x = wsm[e];
      x.x = fma(-h, a.x, x.x);
      x.y = fma(-h, a.y, x.y);
      wsm[e] = x;
      a2 += dot2(x, last ? x : __ldcg(vn + R2 * T + e));
    }
    a2 = block_sum(a2);
    if (tid == 0) partial[(long)(i + 1) * nb + blockIdx.x] = a2;
    grid.sync();
  }
  // ||w|| (every CTA forms the same fixed-order sum), then write w back (scaled: next basis vector)
  if (tid < 32) {
    double sm = 0.0;
    for (int b = tid; b < nb; b += 32) sm += partial[(long)(k + 1) * nb + b];
    sm = warp_sum(sm);
    if (tid == 0) {
      hs = sqrt(sm);
      if (blockIdx.x == 0) H[k + 1] = hs;
    }
  }
  __syncthreads();
  const double f = (scale && hs > 0.0) ? 1.0 / hs : 1.0;
#pragma unroll
  for (int r = 0; r < R2; ++r) {
    const int e = r * T + tid;
    if (e < cnt) w2[e] = make_double2(wr[r].x * f, wr[r].y * f);
  }
  for (int e = tid; e < nsm; e += T) w2[R2 * T + e] = make_double2(wsm[e].x * f, wsm[e].y * f);
}

int mgs_blocks() {
  static int nb = 0;
  if (nb == 0) {
    int dev, sms;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    nb = sms;
  }
  return nb;
}

// Returns the on-chip plan for vectors of n doubles: dynamic smem bytes, or -1 if w does not fit.
static long mgs_oc_smem(long n, long* C2out) {
  static int max_smem = -1;
  if (max_smem < 0) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    max_smem -= 8 * 1024;   // static smem of block_sum / hs and headroom
  }
  if (n % 2 != 0) return -1;
  const long C2 = (n / 2 + mgs_blocks() - 1) / mgs_blocks();
  const long bytes = std::max(0L, C2 - (long)MGS_OC_R2 * MGS_OC_THREADS) * (long)sizeof(double2);
  if (bytes > max_smem) return -1;
  *C2out = C2;
  return bytes;
}

cudaError_t launch_mgs(double* w, const double* const* V, int k, long n, double* H, double* partial, double* G,
                       int ldg, cudaStream_t s, int* scaled) {
  long C2 = 0;
  const long smem = mgs_oc_smem(n, &C2);
  if (smem >= 0) {
    static long attr_set = -1;
    if (attr_set < smem) {
      cudaFuncSetAttribute(k_mgs_oc<MGS_OC_R2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_set = smem;
    }
    long n2 = n / 2;
    int scale = 1;
    int nb = mgs_blocks();
    void* args[] = {&w, (void*)&V, &k, &n2, &C2, &H, &partial, &scale};
    *scaled = 1;
    return cudaLaunchCooperativeKernel((void*)k_mgs_oc<MGS_OC_R2>, dim3(nb), dim3(MGS_OC_THREADS), args,
                                       (size_t)smem, s);
  }
  if (n % 2 != 0) return cudaErrorInvalidValue;   // N = 2 n_b (n_v + n_p) is even (double2 passes)
  *scaled = 0;
  if (k < 32 && G) {   // inverse-compact-WY form: two passes over the basis per step
    long n2 = n / 2;
    void* args[] = {&w, (void*)&V, &k, &n2, &H, &partial, &G, &ldg};
    void* fn = k < 8 ? (void*)k_mgs_icwy<8> : k < 16 ? (void*)k_mgs_icwy<16> : (void*)k_mgs_icwy<32>;
    static int bpsm16 = 0, bpsm32 = 0;
    if (bpsm16 == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm16, k_mgs_icwy<16>, MGSW_THREADS, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm32, k_mgs_icwy<32>, MGSW_THREADS, 0);
      bpsm16 = std::max(1, std::min(bpsm16, 2));
      bpsm32 = std::max(1, std::min(bpsm32, 1));
    }
    const int bpsm = k < 16 ? bpsm16 : bpsm32;
    return cudaLaunchCooperativeKernel(fn, dim3(bpsm * mgs_blocks()), dim3(MGSW_THREADS), args, 0, s);
  }
  int nb = mgs_blocks();
  void* args[] = {&w, (void*)&V, &k, &n, &H, &partial};
  return cudaLaunchCooperativeKernel((void*)k_mgs, dim3(nb), dim3(MGS_THREADS), args, 0, s);
}

}  // namespace aao
