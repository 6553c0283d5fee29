// Micro-benchmark of one 2-D Q2 multicolour-SOR sweep set on c2-sized problems (one CTA per problem),
// isolating the finest level of the CTA-resident multigrid: which layout / mapping is fastest?
//   V0  natural layout, lanes over x with stride 3 (current k_mg_cta), per-node class lookup
//   V1  x-residue-blocked rows (x = r mod 3 contiguous), lanes consecutive -> coalesced taps
//   V2  natural layout, 2 nodes per thread with all loads issued before any store
// Timing: clock64 per CTA (max over CTAs) and cudaEvent over the launch.  Synthetic data; the class
// table is 4 x 25 arbitrary diagonally dominant coefficients (values do not affect timing).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__constant__ double ctab[4 * 26];

template <int PY>
__device__ __forceinline__ double2 eval_nat(const double2* x, int i, int j, int n1, int cls) {
  const double* T = ctab + cls * 26;
  double ax = 0, ay = 0;
  const int xl = i >= 2 ? i - 2 : i, xr = i + 2 <= n1 - 1 ? i + 2 : i;
#pragma unroll
  for (int ob = PY ? 1 : 0; ob < (PY ? 4 : 5); ++ob) {
    const double2* row = x + (j + ob - 2) * n1;
    const double2 v0 = row[xl], v1 = row[i - 1], v2 = row[i], v3 = row[i + 1], v4 = row[xr];
    ax = fma(T[ob * 5 + 0], v0.x, ax); ay = fma(T[ob * 5 + 0], v0.y, ay);
    ax = fma(T[ob * 5 + 1], v1.x, ax); ay = fma(T[ob * 5 + 1], v1.y, ay);
    ax = fma(T[ob * 5 + 2], v2.x, ax); ay = fma(T[ob * 5 + 2], v2.y, ay);
    ax = fma(T[ob * 5 + 3], v3.x, ax); ay = fma(T[ob * 5 + 3], v3.y, ay);
    ax = fma(T[ob * 5 + 4], v4.x, ax); ay = fma(T[ob * 5 + 4], v4.y, ay);
  }
  return make_double2(ax, ay);
}

// V0 / V2: natural layout
template <int NB, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_v0(double2* X, const double2* B, int n1, int sweeps, long long* cyc) {
  double2* x = X + (long)blockIdx.x * n1 * n1;
  const double2* b = B + (long)blockIdx.x * n1 * n1;
  const long long t0 = clock64();
  for (int sw = 0; sw < sweeps; ++sw)
    for (int colour = 0; colour < 9; ++colour) {
      const int rx = colour % 3, ry = colour / 3;
      for (int py = 0; py < 2; ++py) {
        int sy = ry + 3 * py; if (sy < 1) sy += 6;
        const int sx = rx < 1 ? rx + 3 : rx;
        const int cx = (n1 - 2 - sx) / 3 + 1, cy = sy > n1 - 2 ? 0 : (n1 - 2 - sy) / 6 + 1;
        const int total = cx * cy;
        for (int t = threadIdx.x; t < total; t += NB * blockDim.x) {
          int idx[NB];
          double2 ax[NB], bb[NB], xc[NB];
          bool ok[NB];
#pragma unroll
          for (int k = 0; k < NB; ++k) {
            const int tt = t + k * blockDim.x;
            ok[k] = tt < total;
            const int q = (ok[k] ? tt : t) / cx;
            const int i = sx + 3 * ((ok[k] ? tt : t) - q * cx), j = sy + 6 * q;
            idx[k] = j * n1 + i;
            const int cls = (i & 1) | ((j & 1) << 1);
            bb[k] = b[idx[k]];
            xc[k] = x[idx[k]];
            ax[k] = (sy & 1) ? eval_nat<1>(x, i, j, n1, cls) : eval_nat<0>(x, i, j, n1, cls);
          }
#pragma unroll
          for (int k = 0; k < NB; ++k)
            if (ok[k]) {
              const int cls = (idx[k] % n1 & 1) | (((idx[k] / n1) & 1) << 1);
              const double oi = ctab[cls * 26 + 25];
              x[idx[k]] = make_double2(xc[k].x + oi * (bb[k].x - ax[k].x), xc[k].y + oi * (bb[k].y - ax[k].y));
            }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

// V1: x-residue-blocked rows: row j stores [i = 0 mod 3 | 1 mod 3 | 2 mod 3]
__device__ __forceinline__ int rcol(int i, int c0, int c01) {
  const int q = i / 3, r = i - 3 * q;
  return (r == 0 ? 0 : (r == 1 ? c0 : c01)) + q;
}
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_v1(double2* X, const double2* B, int n1, int sweeps, long long* cyc) {
  double2* x = X + (long)blockIdx.x * n1 * n1;
  const double2* b = B + (long)blockIdx.x * n1 * n1;
  const int c0 = (n1 + 2) / 3, c01 = c0 + (n1 + 1) / 3;
  const long long t0 = clock64();
  for (int sw = 0; sw < sweeps; ++sw)
    for (int colour = 0; colour < 9; ++colour) {
      const int rx = colour % 3, ry = colour / 3;
      int K[5];
#pragma unroll
      for (int o = 0; o < 5; ++o) {
        const int tt = rx + o - 2;
        const int q = tt >= 0 ? tt / 3 : -1;
        const int r = tt - 3 * q;
        K[o] = (r == 0 ? 0 : (r == 1 ? c0 : c01)) + q;
      }
      const int own = (rx == 0 ? 0 : (rx == 1 ? c0 : c01));
      for (int py = 0; py < 2; ++py) {
        int sy = ry + 3 * py; if (sy < 1) sy += 6;
        const int sx = rx < 1 ? rx + 3 : rx;
        const int m0 = (sx - rx) / 3;
        const int cx = (n1 - 2 - sx) / 3 + 1, cy = sy > n1 - 2 ? 0 : (n1 - 2 - sy) / 6 + 1;
        const int total = cx * cy;
        for (int t = threadIdx.x; t < total; t += blockDim.x) {
          const int q = t / cx;
          const int m = m0 + (t - q * cx);
          const int i = rx + 3 * m, j = sy + 6 * q;
          const int cls = (i & 1) | ((j & 1) << 1);
          const double* T = ctab + cls * 26;
          double ax = 0, ay = 0;
#pragma unroll
          for (int ob = 0; ob < 5; ++ob) {
            if ((sy & 1) && (ob == 0 || ob == 4)) continue;
            const double2* row = x + (j + ob - 2) * n1 + m;
#pragma unroll
            for (int oa = 0; oa < 5; ++oa) {
              const double2 v = row[K[oa]];
              ax = fma(T[ob * 5 + oa], v.x, ax);
              ay = fma(T[ob * 5 + oa], v.y, ay);
            }
          }
          const int id = j * n1 + own + m;
          const double2 bb = b[id], xc = x[id];
          const double oi = T[25];
          x[id] = make_double2(xc.x + oi * (bb.x - ax), xc.y + oi * (bb.y - ay));
        }
      }
      __syncthreads();
    }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}


// V3: rows stored 6-residue-blocked: [i = 0 mod 6 | 1 mod 6 | ... | 5 mod 6]; a colour (rx, ry) splits
// into sub-lattices s = rx or rx + 3 (mod 6) with fixed x parity; lanes take consecutive m (contiguous),
// taps are compile-time by parity; per tap one pointer add.
struct R6 { int off[7]; };
__device__ __forceinline__ int r6col(const R6& R, int i) { const int q = i / 6; return R.off[i - 6 * q] + q; }
template <int PX, int PY>
__device__ __forceinline__ void v3_sub(double2* x, const double2* b, int n1, const R6& R, int sx, int sy, int tid, int nth) {
  constexpr int OA0 = PX ? 1 : 0, OA1 = PX ? 4 : 5, OB0 = PY ? 1 : 0, OB1 = PY ? 4 : 5;
  const int hi = n1 - 2;
  const int cx = sx > hi ? 0 : (hi - sx) / 6 + 1, cy = sy > hi ? 0 : (hi - sy) / 6 + 1;
  const int total = cx * cy;
  if (!total) return;
  // column offset of tap oa for node i = sx + 6m: block of residue (sx+oa-2) mod 6, index m + floor((sx+oa-2)/6)
  int K[5];
#pragma unroll
  for (int oa = 0; oa < 5; ++oa) {
    const int t = sx + oa - 2;
    const int q = t >= 0 ? t / 6 : -1;
    K[oa] = R.off[t - 6 * q] + q;
  }
  const int m0 = (sx - (sx % 6)) / 6;   // 0
  const int own = K[2];
  const double* T = ctab + (PX | (PY << 1)) * 26;
  const float rc = 1.0f / cx;
  for (int t = tid; t < total; t += nth) {
    int n = __float2int_rz((t + 0.5f) * rc);
    int m = t - n * cx;
    if (m >= cx) { m -= cx; ++n; } else if (m < 0) { m += cx; --n; }
    m += m0;
    const int j = sy + 6 * n;
    const double2* base = x + (j - 2) * n1 + m;
    double a0 = 0, a1 = 0, c0 = 0, c1 = 0;
#pragma unroll
    for (int ob = OB0; ob < OB1; ++ob) {
      const double2* row = base + ob * n1;
#pragma unroll
      for (int oa = OA0; oa < OA1; ++oa) {
        const double2 v = row[K[oa]];
        const double w = T[ob * 5 + oa];
        if ((oa + ob) & 1) { a1 = fma(w, v.x, a1); c1 = fma(w, v.y, c1); }
        else { a0 = fma(w, v.x, a0); c0 = fma(w, v.y, c0); }
      }
    }
    const int id = j * n1 + own + m;
    const double2 bb = b[id], xc = x[id];
    const double oi = T[25];
    x[id] = make_double2(xc.x + oi * (bb.x - a0 - a1), xc.y + oi * (bb.y - c0 - c1));
  }
}
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_v3(double2* X, const double2* B, int n1, int sweeps, long long* cyc) {
  double2* x = X + (long)blockIdx.x * n1 * n1;
  const double2* b = B + (long)blockIdx.x * n1 * n1;
  R6 R;
  R.off[0] = 0;
  for (int r = 0; r < 6; ++r) R.off[r + 1] = R.off[r] + (n1 - r + 5) / 6;
  const long long t0 = clock64();
  for (int sw = 0; sw < sweeps; ++sw)
    for (int colour = 0; colour < 9; ++colour) {
      const int rx = colour % 3, ry = colour / 3;
      for (int qy = 0; qy < 2; ++qy)
        for (int qx = 0; qx < 2; ++qx) {
          int sx = rx + 3 * qx, sy = ry + 3 * qy;
          if (sx == 0) sx = 6;
          if (sy == 0) sy = 6;
          // sx in 1..6: residue sx % 6, first node sx
          switch ((sx & 1) | ((sy & 1) << 1)) {
            case 0: v3_sub<0, 0>(x, b, n1, R, sx, sy, threadIdx.x, blockDim.x); break;
            case 1: v3_sub<1, 0>(x, b, n1, R, sx, sy, threadIdx.x, blockDim.x); break;
            case 2: v3_sub<0, 1>(x, b, n1, R, sx, sy, threadIdx.x, blockDim.x); break;
            default: v3_sub<1, 1>(x, b, n1, R, sx, sy, threadIdx.x, blockDim.x); break;
          }
        }
      __syncthreads();
    }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

// V5: V0 with the iterate resident in shared memory (copied in once; n1^2 * 16 B must fit)
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_v5(double2* X, const double2* B, int n1, int sweeps, long long* cyc) {
  extern __shared__ double2 xs[];
  double2* xg = X + (long)blockIdx.x * n1 * n1;
  const double2* b = B + (long)blockIdx.x * n1 * n1;
  for (int i = threadIdx.x; i < n1 * n1; i += blockDim.x) xs[i] = xg[i];
  __syncthreads();
  double2* x = xs;
  const long long t0 = clock64();
  for (int sw = 0; sw < sweeps; ++sw)
    for (int colour = 0; colour < 9; ++colour) {
      const int rx = colour % 3, ry = colour / 3;
      for (int py = 0; py < 2; ++py) {
        int sy = ry + 3 * py; if (sy < 1) sy += 6;
        const int sx = rx < 1 ? rx + 3 : rx;
        const int cx = (n1 - 2 - sx) / 3 + 1, cy = sy > n1 - 2 ? 0 : (n1 - 2 - sy) / 6 + 1;
        const int total = cx * cy;
        for (int t = threadIdx.x; t < total; t += blockDim.x) {
          const int q = t / cx;
          const int i = sx + 3 * (t - q * cx), j = sy + 6 * q;
          const int idx = j * n1 + i;
          const int cls = (i & 1) | ((j & 1) << 1);
          const double2 bb = b[idx];
          const double2 ax = (sy & 1) ? eval_nat<1>(x, i, j, n1, cls) : eval_nat<0>(x, i, j, n1, cls);
          const double2 xc = x[idx];
          const double oi = ctab[cls * 26 + 25];
          x[idx] = make_double2(xc.x + oi * (bb.x - ax.x), xc.y + oi * (bb.y - ax.y));
        }
      }
      __syncthreads();
    }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  for (int i = threadIdx.x; i < n1 * n1; i += blockDim.x) xg[i] = xs[i];
}

int main(int argc, char** argv) {
  const int n1 = argc > 1 ? atoi(argv[1]) : 129;
  const int P = argc > 2 ? atoi(argv[2]) : 128;
  const int sweeps = 4;
  const long n = (long)n1 * n1;
  std::vector<double2> h(n * P);
  srand(1);
  for (long p = 0; p < P; ++p)
    for (long k = 0; k < n; ++k) {
      const int i = k % n1, j = k / n1;
      const bool in = i > 0 && j > 0 && i < n1 - 1 && j < n1 - 1;
      h[p * n + k] = in ? make_double2(rand() / (double)RAND_MAX, rand() / (double)RAND_MAX) : make_double2(0, 0);
    }
  double ht[104];
  for (int c = 0; c < 4; ++c) {
    for (int t = 0; t < 25; ++t) ht[c * 26 + t] = (t == 12) ? 4.0 : -0.1;
    ht[c * 26 + 25] = 0.25;
  }
  CK(cudaMemcpyToSymbol(ctab, ht, sizeof(ht)));
  double2 *X, *B;
  long long* cyc;
  CK(cudaMalloc(&X, n * P * 16));
  CK(cudaMalloc(&B, n * P * 16));
  CK(cudaMalloc(&cyc, P * 8));
  CK(cudaMemcpy(B, h.data(), n * P * 16, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemcpy(X, h.data(), n * P * 16, cudaMemcpyHostToDevice));
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(P);
    cudaMemcpy(c.data(), cyc, P * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (auto v : c) mx = v > mx ? v : mx;
    printf("%-28s n1=%d P=%d: %.3f ms, max CTA cycles %lld, per phase %lld cycles\n", name, n1, P, ms, mx,
           mx / (9 * sweeps));
  };
  run("V0 natural t512", [&] { k_v0<1, 512><<<P, 512>>>(X, B, n1, sweeps, cyc); });
  run("V0 natural t1024", [&] { k_v0<1, 1024><<<P, 1024>>>(X, B, n1, sweeps, cyc); });
  run("V0 natural t256", [&] { k_v0<1, 256><<<P, 256>>>(X, B, n1, sweeps, cyc); });
  run("V2 natural 2/thr t512", [&] { k_v0<2, 512><<<P, 512>>>(X, B, n1, sweeps, cyc); });
  run("V2 natural 2/thr t1024", [&] { k_v0<2, 1024><<<P, 1024>>>(X, B, n1, sweeps, cyc); });
  run("V1 residue t512", [&] { k_v1<512><<<P, 512>>>(X, B, n1, sweeps, cyc); });
  run("V1 residue t1024", [&] { k_v1<1024><<<P, 1024>>>(X, B, n1, sweeps, cyc); });
  run("V3 residue6 t512", [&] { k_v3<512><<<P, 512>>>(X, B, n1, sweeps, cyc); });
  if (n * 16 <= 220 * 1024) {
    cudaFuncSetAttribute(k_v5<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_v5<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    run("V5 smem-resident t512", [&] { k_v5<512><<<P, 512, n * 16>>>(X, B, n1, sweeps, cyc); });
    run("V5 smem-resident t1024", [&] { k_v5<1024><<<P, 1024, n * 16>>>(X, B, n1, sweeps, cyc); });
  }
  run("V3 residue6 t1024", [&] { k_v3<1024><<<P, 1024>>>(X, B, n1, sweeps, cyc); });
  return 0;
}
