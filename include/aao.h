/*
 * aao.h -- all-at-once Stokes/Oseen optimal control on one B200:
 *          KKT matvec, block-circulant preconditioner, outer GMRES.
 *
 * Implements the hot path of arXiv 2405.18964 (PAPER.md = P:n line refs):
 *   - the permuted all-at-once KKT matrix A of eq. (FinalA), P:120-149;
 *   - the block-circulant preconditioner of Algorithm 1: time DFT
 *     of every v, p, lambda, mu series, one complex-shifted
 *     saddle-point solve per frequency, inverse DFT.  Stokes blocks use
 *     T_l^{-1}, P~_j^{-1}, T_r^{-1}; Oseen blocks use
 *     (P~_j^(UZ))^{-1} of Algorithm 3;
 *   - restarted right-preconditioned GMRES(m).
 * Readings of points the paper leaves open: DESIGN.md "Readings" (= SURVEY 8(c) C.2).
 *
 * Conventions (all entry points):
 *   - Vectors are fp64, length aao_vector_len() = N = 2 (n_t - 1)(n_v + n_p),
 *     in "paper order" (P:96-100 permuted as in eq. FinalA):
 *        index = ((half * n_b + t) * (n_v + n_p)) + field
 *     half 0 = (v, p), half 1 = (lambda, mu); t = 0..n_b-1 is time block j = t+1
 *     (n_b = n_t - 1); field = [velocity component c: Q2 node] (c*n_s + node)
 *     then [Q1 pressure node] (n_v + node); nodes on the full grid, lexicographic,
 *     x fastest.  n_s = (2 N_c + 1)^d, n_v = d n_s, n_p = (N_c + 1)^d.
 *   - Masked entries -- Dirichlet velocity nodes (boundary), the pinned pressure
 *     node 0 -- are IGNORED on input (must be finite) and WRITTEN AS 0 on output.
 *   - Vector pointers passed to *_apply / gmres are DEVICE memory owned by the
 *     caller.  The context owns all workspace (allocated in aao_create).
 *   - *_apply calls allocate nothing, do not synchronise, and are ordered on
 *     `stream` (a cudaStream_t passed as void*; NULL = legacy default stream).
 *   - One context must not be used from two threads at once.
 *   - Errors: a negative aao_status; aao_last_error() returns a message.
 */
#ifndef AAO_H
#define AAO_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  AAO_OK = 0,
  AAO_NOT_CONVERGED = 1,   /* status, not error: x holds the last iterate       */
  AAO_ERR_CONFIG = -1,     /* invalid configuration (see aao_create)            */
  AAO_ERR_SHAPE = -2,      /* bad argument (NULL pointer, index out of range)   */
  AAO_ERR_CUDA = -3,       /* a CUDA runtime error                              */
  AAO_ERR_OOM = -4,        /* device allocation failed                          */
  AAO_ERR_NUMERIC = -5     /* NaN/Inf, singular coarse-grid matrix              */
} aao_status;

typedef enum { AAO_STOKES = 0, AAO_OSEEN = 1 } aao_problem;

typedef struct aao_ctx aao_ctx;

typedef struct {
  int dim;               /* space dimension d, 2 or 3                          */
  int n_cells;           /* N_c cells per direction, power of 2, >= 4                  */
  double x_lo, x_hi;     /* Omega = [x_lo, x_hi]^d, uniform Q2-Q1 mesh          */
  int n_t;               /* time steps; n_b = n_t - 1 unknown blocks; >= 3 */
  double T;              /* final time; tau = T / n_t                           */
  double beta;           /* regularisation beta > 0                             */
  double nu;             /* viscosity nu > 0                                    */
  int problem;           /* aao_problem; Oseen (w != 0) or Stokes (w = 0)       */
  const double* wind_q2; /* HOST, [d][n_s] Q2 nodal wind (Oseen only, else NULL);
                            copied during aao_create (caller keeps ownership)          */
  int mg_cycles;         /* V-cycles per MG application (4)                      */
  int pre_sweeps;        /* multicolour SOR sweeps before / after the coarse           */
  int post_sweeps;       /*   correction (paper silent; DESIGN.md reading: 2 / 2)       */
  double omega;          /* SOR relaxation (reading: 1.0)                              */
  int cheb_iters;        /* Chebyshev semi-iterations (10)                      */
  int uzawa_iters;       /* Uzawa iterations, Oseen (6)                         */
  double uzawa_mu;       /* Uzawa parameter mu (3/4)                            */
  int pmode;             /* aao_pmode: AAO_PRECOND_LINEAR (Algorithm 1, default) or
                            AAO_PRECOND_NONLINEAR (Algorithm 2: per-frequency inner
                            GMRES to inner_eps; aao_gmres_solve then runs FGMRES)  */
  double inner_eps;      /* inner relative tolerance (1e-2)                      */
  int inner_maxit;       /* inner iteration cap = inner Krylov basis size (reading: 60;
                            reduced at create if the basis does not fit in memory)     */
  int freq_chunk;        /* frequencies per velocity-MG launch; the MG level workspace is sized for
                            freq_chunk frequencies instead of all n_f.  0 = auto: all
                            when the workspace fits in 2 GiB, else the largest multiple of a full
                            148-problem wave that does.  Changes no arithmetic (independent
                            per-frequency solves).  < 0: AAO_ERR_CONFIG                  */
} aao_config;

typedef enum { AAO_PRECOND_LINEAR = 0, AAO_PRECOND_NONLINEAR = 1 } aao_pmode;

/* Fill *cfg with the paper's defaults (4 V-cycles, 2/2 sweeps, omega 1, 10 Chebyshev,
   6 Uzawa, mu 3/4); geometry / time / beta / nu must still be set by the caller. */
void aao_config_defaults(aao_config* cfg);

typedef struct {
  double tol;            /* relative residual target on ||b|| (reading: 1e-6)            */
  int restart;           /* GMRES restart m (30), 1 <= m <= 64                     */
  int max_iters;         /* iteration cap                                                 */
  int store_z;           /* linear mode: 0 = restart update x += P^{-1}(V y) (the oracle's form, one
                            extra preconditioner application per cycle); 1 = keep the m vectors
                            Z_k = P^{-1} v_k and update x += Z y (m more vectors of device memory,
                            AAO_ERR_OOM if they do not fit -- never a silent switch).  FGMRES
                            (nonlinear mode) always stores Z.  Other values: AAO_ERR_SHAPE      */
} aao_krylov;

typedef struct {
  int iterations;        /* GMRES iterations (= preconditioned matvecs of the Arnoldi loop) */
  int restarts;
  int converged;         /* 1 if |g_{k+1}| <= tol ||b||                                     */
  int breakdown;         /* 1 if h_{k+1,k} < 1e-14 ||b||                                    */
  double final_relres;   /* last recurrence residual / ||b||                                */
  double true_relres;    /* ||b - A x|| / ||b|| recomputed at exit                           */
  int precond_applies;   /* Arnoldi applications, plus one per cycle when the preconditioned vectors
                            are not stored (x += P^{-1}(V y))                                  */
  double ms_total;       /* wall time of the solve (host clock around device work)           */
  long inner_its_total;  /* nonlinear mode: inner GMRES iterations summed over frequencies and
                            preconditioner applications of this solve                        */
  int inner_its_max;     /* nonlinear mode: largest inner iteration count of one frequency    */
  double ms_precond;     /* device time summed over the Arnoldi iterations: preconditioner,   */
  double ms_kkt;         /*   KKT matvec and Gram-Schmidt (+ normalisation); filled only after */
  double ms_orth;        /*   aao_set_timing(ctx, 1) (events; the speculative enqueue is off)  */
  int store_z;           /* 1 if the restart update used the stored Z (x += Z y)               */
} aao_info;

/* Assemble operators and per-frequency data, allocate all device workspace (step A9).
   Rejects with AAO_ERR_CONFIG: dim not in {2,3}; n_cells not a power of 2 or < 4;
   n_t < 3; T, beta, nu <= 0; Oseen without wind_q2; mg_cycles < 1; cheb_iters < 1;
   uzawa_iters < 1; uzawa_mu <= 0; pmode not in {0,1}; nonlinear with inner_eps not in (0,1)
   or inner_maxit < 1.  Ownership of *out passes to the caller
   (release with aao_destroy).  Runs on the current CUDA device. */
aao_status aao_create(const aao_config* cfg, aao_ctx** out);
void aao_destroy(aao_ctx* ctx);
const char* aao_last_error(const aao_ctx* ctx);   /* never NULL; "" when no error */

size_t aao_vector_len(const aao_ctx* ctx);         /* N = 2 n_b (n_v + n_p) */
/* Workspace owned by the context, bytes.  aao_gmres_solve adds (m + 1) + 1 vectors of N doubles at the first
   solve (+ m with stored Z or in nonlinear mode); aao_gmres_solve_host 2 more (device staging of b, x). */
size_t aao_device_bytes(const aao_ctx* ctx);       /* workspace owned by the context */

/* Paper order -> internal layout.  The internal (layout-T) vector IS the paper's ordering
   [half][time block][field][full-grid node] (P:118-149 block structure), so packing
   is a masked copy: out = in with masked entries (Dirichlet nodes, pinned pressure node) set to 0.
   Device pointers; in == out allowed. */
aao_status aao_pack(aao_ctx* ctx, const double* in, double* out, void* stream);

/* Internal layout -> paper order: the same masked copy (the layouts coincide).  Device pointers. */
aao_status aao_unpack(aao_ctx* ctx, const double* in, double* out, void* stream);

/* Right-hand side for v_0 = 0, f = 0, h = 0:
   b = tau * (M_full v_d)|_interior in every adjoint-velocity block (half 0), 0 elsewhere.
   vd_q2: DEVICE, [d][n_s] Q2 nodal desired state (time-constant). */
aao_status aao_build_rhs(aao_ctx* ctx, const double* vd_q2, double* b, void* stream);

/* Right-hand side with time-dependent data and inhomogeneous Dirichlet data moved to the right-hand
   side by lifting (the paper's manufactured problem P:812-824).
   For time block m = 1..n_b (t_m = m tau), component c, with G^m = g^m on boundary nodes and 0 inside:
     adjoint rows (half 0):    tau [M (v_d^m - G^m)] on interior velocity nodes
     state rows (half 1):      [M (tau f^m - G^m + H^{m-1}) - tau L G^m],  H^0 = v0, H^{m-1} = G^{m-1},
                               L = nu K (Stokes) or nu K + N (Oseen, the context's wind)
     divergence rows (half 1): -tau [B G^m] on unknown pressure nodes;  all other rows 0,
   M, K, B un-eliminated (boundary columns kept).  All pointers DEVICE, full Q2 grids, x fastest:
     vd, f: [n_b][d][n_s] at t_1..t_{n_b};  g: [n_b + 1][d][n_s] at t_0..t_{n_b} (only boundary entries
     are read);  v0: [d][n_s] on every node.  Any of vd, f, g, v0 may be NULL (= 0; v0 NULL -> g^0).
   b: DEVICE, length aao_vector_len (paper order).  Errors: AAO_ERR_SHAPE (null ctx/b). */
aao_status aao_build_rhs_general(aao_ctx* ctx, const double* vd, const double* f, const double* g, const double* v0,
                                 double* b, void* stream);

/* Arnoldi process on A P^{-1} (right preconditioning, the GMRES iteration of aao_gmres_solve without the
   Givens update, the spectra of P:359-367 and P:607-632): v_0 = v0 / ||v0||, then for
   k = 0..m-1  w = A P^{-1} v_k, modified Gram-Schmidt against v_0..v_k, h_{k+1,k} = ||w||.
   v0: DEVICE, length aao_vector_len (masked entries ignored).  H: HOST, row-major (m + 1) x m, receives
   the unrotated Hessenberg matrix (zeros beyond the steps done); *m_done (may be NULL) = steps done
   (< m at breakdown, h_{k+1,k} < 1e-14 ||v0||).  Eigenvalues of H[:k, :k] (Ritz values) estimate those
   of P^{-1} A.  Uses the GMRES workspace: m must not exceed the restart of the first solve on ctx.
   Synchronises the stream once per step.  Errors: AAO_ERR_SHAPE, AAO_ERR_CONFIG, AAO_ERR_NUMERIC. */
aao_status aao_arnoldi(aao_ctx* ctx, const double* v0, int m, double* H, int* m_done, void* stream);

/* y = A x, eq. (FinalA) (step A2).  Device pointers, x != y (else AAO_ERR_SHAPE). */
aao_status aao_kkt_apply(aao_ctx* ctx, const double* x, double* y, void* stream);

/* z = Pbar_C^{-1} r, Algorithm 1 (steps A3-A8).  Device pointers, r != z.
   A fixed linear map (fixed-count inner solvers).  With pmode = AAO_PRECOND_NONLINEAR:
   Algorithm 2 (a nonlinear map; synchronises the stream once per inner iteration). */
aao_status aao_precond_apply(aao_ctx* ctx, const double* r, double* z, void* stream);

/* Restarted right-preconditioned GMRES(m), MGS + Givens (step A1); flexible GMRES (FGMRES,
   storing the preconditioned basis) when pmode = AAO_PRECOND_NONLINEAR.
   b, x: DEVICE; x is the initial guess on input (pass zeros for x0 = 0) and the
   solution on output.  hist: HOST, may be NULL; receives |g_{k+1}|/||b|| per
   iteration (up to hist_cap entries).  Synchronises `stream` before returning;
   info (HOST, may be NULL) is filled.  Returns AAO_OK, AAO_NOT_CONVERGED or an error. */
aao_status aao_gmres_solve(aao_ctx* ctx, const double* b, double* x, const aao_krylov* kry,
                           aao_info* info, double* hist, int hist_cap, void* stream);

/* Same solve with HOST b and x (pinned or pageable; each N doubles, caller-owned, b != x): copies b and x0
   in and x out inside the call -- the end-to-end entry point.  On an error (negative status) x_host is not
   written.  The binding checks the host buffers' dtype / length / contiguity before the call. */
aao_status aao_gmres_solve_host(aao_ctx* ctx, const double* b_host, double* x_host,
                                const aao_krylov* kry, aao_info* info, double* hist,
                                int hist_cap, void* stream);

/* Debug / sampled parity: copy frequency block k (0 <= k < n_f,
   n_f = n_b/2 + 1) of the LAST aao_precond_apply, i.e. y_hat_k after T_r^{-1}
   (Stokes) or after Algorithm 3 (Oseen), to HOST memory `out` as complex128
   pairs (re, im): [half 0..1][n_v + n_p] in the field order above.  Synchronises. */
aao_status aao_debug_freq_block(aao_ctx* ctx, int k, double* out, void* stream);

/* Nonlinear mode: inner GMRES iteration counts of the last aao_precond_apply, one per stored
   frequency k < n_f (HOST out, up to cap entries); returns the number written (>= 0) or an error. */
int aao_last_inner_iterations(const aao_ctx* ctx, int* out, int cap);

/* Per-phase device timings of the last aao_precond_apply, milliseconds
   (fft_fwd, velocity block solves, pressure block solves, fft_inv); requires
   aao_set_timing(ctx, 1) beforehand (adds events; off by default) and a LINEAR-mode apply since;
   otherwise AAO_ERR_CONFIG with ms4 zeroed. */
aao_status aao_set_timing(aao_ctx* ctx, int on);
aao_status aao_last_phase_ms(aao_ctx* ctx, double* ms4);

/* Live timing of the dominant kernel class -- the velocity multigrid: in the default CTA-resident
   mode the k_mg_cta solve launches, in the per-level mode (env AAO_MG_MODE=1) the finest-level
   multicolour SOR sweeps -- with CUDA events on the launching stream around each launch (run).
   aao_profile_smoother(ctx, on) resets and enables (on = 1), disables (on = 0), or enables and pre-creates the
   events for `on` > 1 launches (so that no event is created inside a timed region); aao_profile_read
   synchronises and returns
   out3 = {milliseconds, algorithmic bytes, number of kernel launches} accumulated since, then
   resets.  Algorithmic bytes: a sweep reads x, b and writes x once per unknown (48 B, complex128);
   a whole MG solve adds residual (48), restriction (16 + 16/coarse unknown), prolongation (32 +
   16/coarse unknown) per level and V-cycle and the coarsest solve (32) -- DESIGN.md "Roofline". */
aao_status aao_profile_smoother(aao_ctx* ctx, int on);
aao_status aao_profile_read(aao_ctx* ctx, double* out3);

/* Number of kernel launches issued by the last aao_precond_apply / aao_kkt_apply /
   aao_gmres_solve (counted on the host as they are enqueued). */
long aao_last_launch_count(const aao_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* AAO_H */
