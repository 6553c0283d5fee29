// Internal declarations of the B200 all-at-once library (not part of the C ABI).
// Device descriptors are passed to kernels by value.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/aao.h"

namespace aao {

// One multigrid level of one scalar finite-element space on the full node grid.
//   order 2: Q2 velocity component, 5-point 1-D rows, Dirichlet boundary nodes masked;
//   order 1: Q1 pressure, 3-point 1-D rows, corner node 0 pinned.
// Constant-coefficient operators are Kronecker sums of 1-D assembled rows:
//   M = M_z (x) M_y (x) M_x,  K = sum_a (K_a (x) prod_{b!=a} M_b)     (x fastest)
// tM/tK rows are indexed by the 1-D node index i, entry o is the coupling to
// node i + o - order; entries to eliminated (boundary) columns are 0.
struct Grid {
  int dim;
  int order;
  int n1;
  long n;
  const double* tM;     // [n1][2*order+1]
  const double* tK;     // [n1][2*order+1]
  const double* conv;   // [n][(2*order+1)^dim] convection N (Oseen) or nullptr
  const double* convT;  // its transpose N^T, same layout, or nullptr
};

// A = a*M + b*K + c*C, C = conv (sel 1) or convT (sel 2); coefficients per group.
struct Coef { double2 a, b, c; };
struct OpSel {
  const Coef* coef;    // device, [n_groups]
  int per_group;       // problems per coefficient group
  int conv_sel;        // 0: none, 1: N, 2: N^T
};

// A batch of complex vectors of length n: problem p lives at
//   p + (p / per_group) * gstride + (p % per_group) * n   (in double2 units)
struct View {
  double2* p;
  int per_group;
  long gstride;
};

// MG transfer tables between a fine level f and the coarse level c = f+1 (1-D).
struct Transfer {
  const double* tP;    // [n1_fine][4]: base coarse index, 3 weights (Q1: 2 used)
  const double* tR;    // [n1_coarse][7]: weights on fine nodes 2I-3..2I+3 (Q1: 2I-1..2I+1 in [2..4])
};

// per-frequency constants for the time kernels (k < n_f)
struct FreqConst {
  double c1, c2;       // c_{k,1}, c_{k,2} (squared reading)
  double dr, dc;       // Re d_k, Im d_k
  double rc2;          // 1 / c_{k,2} (the T transforms multiply instead of dividing)
};

// Arguments of the CTA-resident multigrid solve (one CTA per problem, all levels and cycles).
constexpr int MG_MAXL = 12;
constexpr int MG_TRI_THREADS = 576;    // threads per CTA of the 2-D Q2 real class-stencil MG: one per triple of a
                                       // band-wavefront step, rows padded to whole warps (3 rows x 192 lanes for the
                                       // 171 triples of a 513^2 level); 96 registers (as for any count in 513..640)
// lanes a row of ntr triples takes in that mapping
inline int mg_tri_lanes_per_row(int ntr) {
  if (ntr >= 32) return (ntr + 31) / 32 * 32;
  int l = 1;
  while (l < ntr) l *= 2;
  return l;
}
constexpr int MG_RING_GUARD = 4;       // zeroed double2 entries before and after the band ring
constexpr int MG_ZL_STAGES = 6;        // 3-D line-form sweeps: staged lines per warp (= ZL_STAGES of kernels_stencil.cu)
constexpr int MG_TRI_SLOTS = 9;        // band slots of the triple-form ring (8 for the node-per-thread Oseen form)
constexpr int MG_SMEM_MAX = 232448;    // dynamic shared memory per CTA (227 KB opt-in on sm_100)
struct MGArgs {
  int nlev, cycles, pre, post;
  double omega;
  Grid g[MG_MAXL];
  Transfer t[MG_MAXL];
  double2* xw[MG_MAXL];   // levels >= 1: [nprob][n_l]
  double2* bw[MG_MAXL];
  double2* rw[MG_MAXL];   // all levels: [nprob][n_l]
  View x0, b0;            // finest level solution / right-hand side
  OpSel op;
  const double2* inv;     // coarsest-level dense inverses [groups][nu][nu]
  int inv_pg;
  const int* unk;
  int nu;
  int lsm;                // levels >= lsm keep x and b in shared memory (offsets below, in double2)
  int lwarp;              // levels >= lwarp run inside one warp (tiny bottom of the V-cycle)
  int use_ctab;           // Q2 operators: per-level class stencils at the start of dynamic smem
  long sm_x[MG_MAXL], sm_b[MG_MAXL];
  int wave_h;               // band-wavefront sweeps (2-D Q2) on some level: the ring and its mbarriers exist
  int wave_hl[MG_MAXL];     // per level: band height H (rows per band, a multiple of 3), 0 = colour-by-colour sweeps
  int zwave_min;            // 3-D Q2: levels with n1 >= zwave_min sweep as a z-band wavefront (global memory)
  long zstage_off;          // 3-D Q2 real: per-warp line stages of the line-form wavefront (double2 units), -1 = none
  long ring_off;            // ring buffer offset in dynamic smem (double2 units)
  long mbar_off;            // 9 band-slot mbarriers + their phase word after the ring (double2 units)
  int flat_max;             // 2-D Q2 real: levels with n1 <= flat_max use merged branch-free colour visits
  int fuse_prolong;         // wavefront levels: x += P x_c applied while the first post-smoothing sweep loads its bands
  unsigned long long* clk;  // profiling (AAO_MG_CLOCK=<block>): that CTA accumulates SM cycles per [level][down, up]
  int clk_block;
};

// a frequency vector: velocity part [k][half][comp][node] and pressure part [k][half][node] (complex)
struct FVec {
  double2* v;
  double2* p;
};

struct MGSpace {       // an MG hierarchy for one space, with batch workspace
  int order;
  int nlev;
  std::vector<Grid> grids;
  std::vector<Transfer> transfers;
  std::vector<double2*> x, b, r;     // per level (level 0 x/b external), nprob_max problems each
  int ncoarse_unk;                   // unknowns on the coarsest grid
  int* coarse_unk;                   // device, node indices
  int nprob_max;
};

// The context: configuration, device operators, per-frequency data, workspace.
struct Ctx {
  aao_config cfg;
  int dim = 2, Nc = 0, n_t = 0, n_b = 0, n_f = 0;
  double tau = 0, beta = 0, nu = 0;
  bool oseen = false;
  int n1q2 = 0, n1q1 = 0;
  long n_s = 0, n_p = 0, n_v = 0, nblk = 0, N = 0;
  MGSpace vel, pres;             // MG hierarchies (Q2 velocity component, Q1 pressure)
  double *tPm = nullptr, *tGm = nullptr;    // [n1q1][5] B rows: int psi_I phi_j, int psi_I phi_j'
  double *tPmT = nullptr, *tGmT = nullptr;  // [n1q2][3] B^T rows, Q1 cols floor((i-1)/2)+o
  double* tMfull = nullptr;                 // [n1q2][5] un-eliminated Q2 mass rows (RHS)
  double *tKfull = nullptr, *tPmfull = nullptr, *tGmfull = nullptr;  // un-eliminated K rows, B rows (lifting)
  double* convFull = nullptr;   // Oseen: un-eliminated fine convection stencil [n_s][5^d] (lifting)
  std::vector<double> h_M2, h_K2, h_Pm, h_Gm, h_PmT, h_GmT;  // host copies of the fine 1-D rows
  FreqConst* fc = nullptr;                  // device [n_f]
  std::vector<FreqConst> fch;
  double2* tw = nullptr;                    // [n_b] (cos, sin)(2 pi m / n_b)
  // frequency-domain arrays: Fv [n_f][2][d][n_s], Fp [n_f][2][n_p]
  double2 *Fv = nullptr, *Fp = nullptr, *Xv = nullptr, *XpA = nullptr, *XpB = nullptr;
  // Oseen work arrays (velocity [n_f][d][n_s], pressure [n_f][2][n_p])
  double2 *X1 = nullptr, *X2 = nullptr, *T1 = nullptr, *T2 = nullptr, *T3 = nullptr;
  double2 *Qp = nullptr, *Sp = nullptr, *Tp = nullptr;
  // Chebyshev work (r, d_old, d_new) sized for the largest batch
  double2 *Cr = nullptr, *Cd0 = nullptr, *Cd1 = nullptr;
  // operator coefficient tables (device)
  Coef *coefW = nullptr, *coefKp = nullptr, *coefMass = nullptr;
  Coef *coefZX = nullptr, *coefNegMass = nullptr;  // Z_k apply (Algorithm 2, Stokes)
  Coef *coefQ = nullptr, *coefQH = nullptr;        // MG operators Q_k, Q_k^H (per k)
  Coef *coefU1 = nullptr, *coefU2 = nullptr, *coefU3 = nullptr, *coefU4 = nullptr;  // Uzawa combos
  Coef *coefS1 = nullptr, *coefS2 = nullptr, *coefS3 = nullptr, *coefS4 = nullptr;  // Schur combos
  // coarse-grid inverses
  double2 *invW = nullptr, *invKp = nullptr, *invQ = nullptr, *invQH = nullptr;
  // nonlinear preconditioner (Algorithm 2): batched inner GMRES per frequency
  bool nonlinear = false;
  double inner_eps = 1e-2;
  int inner_maxit = 0;                   // basis size actually allocated
  std::vector<FVec> nlV;                 // basis V_0..V_m (device), then Zt, U
  FVec* nlVdev = nullptr;                // device copy of the basis descriptors
  double2 *nlH = nullptr, *nlPart = nullptr, *nlY = nullptr;
  int* nlFrozen = nullptr;
  std::vector<int> inner_its;            // per frequency, last application
  long inner_total = 0;
  int inner_max = 0;
  double2* debug_block_src_v = nullptr;  // frequency vector of the last NL solution (debug block)
  double2* debug_block_src_p = nullptr;
  bool store_z = false;                  // this solve keeps Z_k = P^{-1} v_k (FGMRES always; linear on request)
  int gZ_m = 0;                          // stored-Z vectors allocated
  double* gZ = nullptr;                  // preconditioned basis (FGMRES, or aao_krylov.store_z)
  double** gZptr = nullptr;
  // GMRES workspace (allocated on first solve): basis V_0..V_m and one work vector (z / update)
  int gm_m = 0;
  double *gV = nullptr, *gz = nullptr;
  double *gH = nullptr, *gpart = nullptr, *gscal = nullptr, *gG = nullptr;
  double **gVptr = nullptr;
  double *stage_b = nullptr, *stage_x = nullptr;   // device staging of aao_gmres_solve_host
  double* hostH = nullptr;   // pinned, 2 x (m + 2): Hessenberg columns of iterations k, k+1
  cudaEvent_t gm_ev[2] = {nullptr, nullptr};
  cudaEvent_t gt_ev[4] = {nullptr, nullptr, nullptr, nullptr};   // GMRES phase timing (aao_set_timing)
  // bookkeeping
  std::vector<void*> allocs;
  size_t bytes = 0;
  std::string err;
  long launches = 0;
  bool timing = false;
  cudaEvent_t ev[5] = {};
  double phase_ms[4] = {0, 0, 0, 0};
  // live timing of the dominant kernel class (finest-level multicolour SOR sweeps)
  cudaStream_t s2 = nullptr, s3 = nullptr; // side streams: the two pressure solves overlap the velocity MG
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr;
  int wave_force = -1, wave_min = 65;   // band-wavefront sweeps: AAO_WAVE (-1 auto), AAO_WAVE_MIN
  int wave_hmax = 24;                    // largest band height tried per level (AAO_WAVE_H)
  int mg_mode = 0;       // MG schedule: 0 CTA-resident (default), 1 per level / colour launches (AAO_MG_MODE=1)
  int freq_chunk = 0;    // frequencies per velocity-MG launch (aao_config.freq_chunk; workspace sized for it)
  bool phase_valid = false;   // ev[0..4] recorded by the last linear precond_apply (aao_last_phase_ms)
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;   // pairs (start, end)
  size_t prof_used = 0;
  double prof_bytes = 0;
  long prof_launches = 0;
};

// ---- kernel launchers (kernels_*.cu) --------------------------------------
void launch_gs(const Grid& g, const OpSel& op, View x, View b, int nprob, int colour, double omega,
               cudaStream_t s);
void launch_residual(const Grid& g, const OpSel& op, View x, View b, View r, int nprob, cudaStream_t s);
void launch_restrict(const Grid& gf, const Grid& gc, const Transfer& t, View rf, View bc, int nprob,
                     cudaStream_t s);
void launch_prolong(const Grid& gf, const Grid& gc, const Transfer& t, View xc, View xf, int nprob,
                    cudaStream_t s);
void launch_coarse(const Grid& gc, const double2* inv, int inv_per_group, const int* unk, int nu,
                   View b, View x, int nprob, cudaStream_t s);
void launch_zero(View x, long n, int nprob, cudaStream_t s);
void launch_cheb_init(const Grid& g, View b, View x, View r, View d, double inv_theta, int nprob,
                      cudaStream_t s);
void launch_cheb_step(const Grid& g, View x, View r, View dold, View dnew, double c1, double c2,
                      int nprob, cudaStream_t s);
void launch_cheb_final(const Grid& g, View x, View d, double scale, int nprob, cudaStream_t s);
// out = cb*b + A1 x1 + A2 x2  (A2 optional: x2.p == nullptr)
void launch_lincomb(const Grid& g, View out, double cb, View b, const OpSel& A1, View x1,
                    const OpSel& A2, View x2, int nprob, cudaStream_t s);
// y = a*y + bcoef*x  (pointwise, masked entries stay 0)
void launch_axpby(const Grid& g, View y, double2 a, View x, double2 bcoef, int nprob, cudaStream_t s);
void launch_mg_cta(const MGArgs& a, int nprob, size_t smem, cudaStream_t s);

void launch_cheb_cta(const Grid& g, View b, View x, double2* r, double2* d0, double2* d1, double theta, double sigma,
                     double delta, int iters, double scale, int nprob, cudaStream_t s);
// pressure: out = sb*bp + sB * sum_c B_c v_c (v: d components per problem group)
void launch_Bv(const Grid& g2, const Grid& g1, const double* tPm, const double* tGm, View v, View bp,
               View out, double sb, double sB, int nprob, cudaStream_t s);

// time transforms and KKT (kernels_time.cu)
void launch_fft_fwd(const Ctx& c, const double* r, cudaStream_t s);
void launch_fft_inv(const Ctx& c, double* z, cudaStream_t s);
void launch_kkt(const Ctx& c, const double* x, double* y, cudaStream_t s);
bool launch_kkt_march(const Ctx& c, const double* x, double* y, cudaStream_t s);
void launch_mask_copy(const Ctx& c, const double* in, double* out, cudaStream_t s);
void launch_rhs(const Ctx& c, const double* vd, double* b, cudaStream_t s);
void launch_rhs_general(const Ctx& c, const double* vd, const double* f, const double* g, const double* v0, double* b,
                        cudaStream_t s);
void launch_debug_block(const Ctx& c, int k, double2* out, cudaStream_t s);

// frequency-vector kernels (kernels_freq.cu)
void launch_fdot(FVec a, FVec b, long LV, long LP, int nf, double2* partial, double2* out, int mode, cudaStream_t s);
size_t fdot_partial_len(int nf);
void launch_faxpy(FVec y, FVec x, const double2* coef, double sign, long LV, long LP, int nf, cudaStream_t s);
void launch_fscale(FVec y, FVec x, const double2* den, const int* frozen, long LV, long LP, int nf, cudaStream_t s);
void launch_fmulti(FVec u, const FVec* V, const double2* Y, int m, long LV, long LP, int nf, cudaStream_t s);
void launch_combine_p(double2* out, const double2* A, const double2* B, const FreqConst* fc, double nu, long LP, int nf,
                      cudaStream_t s);
void launch_oseen_scatter(FVec out, const double2* X1, const double2* X2, const double2* XpA, double pscale,
                          long ncomp_nodes, long LP, int nf, cudaStream_t s);
void launch_fBT(const Ctx& c, FVec out, int h, FVec q, int qh, double sc, cudaStream_t s);
void launch_fft_inv_from(const Ctx& c, FVec x, double* z, cudaStream_t s);   // T_r^{-1} (Stokes) + inverse DFT of x

// blas (kernels_blas.cu): deterministic two-stage reductions
void launch_dot(const double* x, const double* y, long n, double* partial, int nblk, double* out,
                int mode, cudaStream_t s);   // mode 0: out = dot; 1: out = sqrt(dot)
void launch_axpy_dev(double* y, const double* x, const double* alpha, double sign, long n, cudaStream_t s);
void launch_scale_dev(double* y, const double* x, const double* denom, long n, cudaStream_t s);
void launch_axpy(double* y, const double* x, double alpha, long n, cudaStream_t s);
void launch_copy_sub(double* y, const double* b, const double* ax, long n, cudaStream_t s);  // y = b - ax
void launch_multi_axpy(double* u, const double* const* V, const double* coef, int k, long n, cudaStream_t s);
int dot_blocks();
int mgs_blocks();
// whole MGS sweep (dots, updates, norm) in one cooperative launch; partial: [(2k+3) * 4 * mgs_blocks()]
// MGS of w against V[0..k] -> H[0..k+1]; sets *scaled = 1 if w was also overwritten by w / H[k+1].
// G (ld ldg, rows 0..k+1): Gram rows <v_i, v_j> (j < i) of the current cycle, written and read by the
// inverse-compact-WY form used for vectors that do not fit on chip (row k+1 is written by step k).
cudaError_t launch_mgs(double* w, const double* const* V, int k, long n, double* H, double* partial, double* G,
                       int ldg, cudaStream_t s, int* scaled);

}  // namespace aao
