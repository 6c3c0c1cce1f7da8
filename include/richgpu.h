/*
 * richgpu.h — C-ABI of the B200 (sm_100a) Richardson(m) solve-loop library.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `richlab` (arXiv 2412.08076).  The reference is pure Python; its hot path
 * calls SciPy's CSR matvec, NumPy ufuncs, BLAS ddot and pocketfft.  Each
 * entry point below replaces one of those reference call sites (cited as
 * file:line into /root/reference/pkg/src/richlab/).  The Python shim in
 * paper_2412_08076_b200/ binds these with ctypes.
 *
 * Conventions
 *  - Plain C types only.  Every array pointer is CALLER-OWNED DEVICE memory
 *    unless the comment says "host".  `stream` is a cudaStream_t passed as
 *    void* (NULL = legacy default stream).
 *  - Grids: one "system" is the (side x side) interior of an (side+1)-cell
 *    Dirichlet grid, flattened row-major with x the slow axis:
 *    index = (ix-1)*side + (iy-1)   (problems.py:131-133).  A batch of B
 *    systems is B such vectors back to back.
 *  - Scalar type of vectors follows the operator dtype: RG_F32 -> float,
 *    RG_F64 -> double, RG_C128 -> interleaved (re, im) doubles.
 *  - Return value: RG_OK (0) or a negative rg_err; rg_last_error() gives the
 *    text (thread-local).  Numerical divergence is NOT a call failure: it is
 *    reported per system through rg_report.status (reference
 *    DivergenceError, richardson.py:20-23,126-129).
 *  - Handles are immutable after creation except rg_solver (one solve in
 *    flight per solver).  Operators may be shared by concurrent solvers
 *    (mirrors "multiple solves over shared immutable A may run concurrently").
 */
#ifndef RICHGPU_H
#define RICHGPU_H

#ifdef __cplusplus
extern "C" {
#endif

#define RG_ABI_VERSION 1

enum rg_dtype   { RG_F32 = 1, RG_F64 = 2, RG_C128 = 3 };
/* Operator kinds.  CONST9: one 9-point stencil per system (bilinear-FEM
 * anisotropic operator, problems.py:121-154).  DIAG5: 5-point stencil with
 * constant off-diagonals and a per-node diagonal (damped Helmholtz,
 * problems.py:174-200).  VAR9: 9 per-node coefficient planes (Galerkin
 * coarse operators, multigrid.py:62-68). */
enum rg_kind    { RG_CONST9 = 1, RG_DIAG5 = 2, RG_VAR9 = 3 };
/* schedules.py:8 VARIANTS */
enum rg_variant { RG_PLAIN = 0, RG_MOM = 1, RG_NAG = 2, RG_NAGEX = 3 };
/* precond.py:71-77 weighted Jacobi (scale = relax/diag).  SCALAR: one scale
 * per system (constant diagonal); FIELD: one scale per node. */
enum rg_precond { RG_PRECOND_NONE = 0, RG_PRECOND_JACOBI_SCALAR = 1,
                  RG_PRECOND_JACOBI_FIELD = 2 };
/* richardson.py:77-90 `check` */
enum rg_check   { RG_CHECK_OUTER = 0, RG_CHECK_INNER = 1 };
enum rg_status  { RG_ACTIVE = 0, RG_CONVERGED = 1, RG_DIVERGED = 2,
                  RG_MAXED = 3 };
enum rg_err     { RG_OK = 0, RG_EINVAL = -1, RG_ESIZE = -2, RG_ENULL = -3,
                  RG_EUNSUPPORTED = -4, RG_ECUDA = -5, RG_ESTATE = -6 };

typedef struct rg_op rg_op;
typedef struct rg_solver rg_solver;

/* Operator description.  Coefficient arrays are device pointers that must
 * outlive the handle (no copy is taken).
 *   CONST9 : stencil = [batch][9] in CSR column order (di,dj) =
 *            (-1,-1),(-1,0),(-1,1),(0,-1),(0,0),(0,1),(1,-1),(1,0),(1,1)
 *   DIAG5  : stencil = [batch][4] off-diagonals in CSR order
 *            (-1,0),(0,-1),(0,1),(1,0);  diag = [batch][side*side]
 *   VAR9   : stencil = [batch][9][side*side] planes, same offset order,
 *            absent CSR entries stored as 0.                               */
typedef struct rg_op_desc {
    int dtype;
    int kind;
    int batch;         /* systems (vectors) the operator is applied to */
    int side;
    const void* stencil;
    const void* diag;
    int shared;        /* 1: the arrays hold ONE system's coefficients, applied
                          to all `batch` systems (e.g. 4 right-hand sides of
                          one Helmholtz problem); 0: one set per system */
} rg_op_desc;

/* Weight schedule for all systems of a batch (schedules.py:11-54).
 * omega/alpha/alpha_tilde are device double arrays [batch][m]; alpha and
 * alpha_tilde may be NULL for RG_PLAIN.  scale: device array of the op's
 * scalar type, [batch] (SCALAR) or [batch][side*side] (FIELD).            */
typedef struct rg_sched {
    int variant;
    int m;
    const double* omega;
    const double* alpha;
    const double* alpha_tilde;
    int precond;
    const void* scale;
} rg_sched;

/* Per-system outcome of a solve (richardson.py:38-46 SolveReport plus the
 * DivergenceError payload).  Filled on the host by rg_solver_report. */
typedef struct rg_report {
    int status;            /* rg_status */
    int iterations;        /* outer sweeps, a trailing partial sweep counts */
    int inner_iterations;  /* also the DivergenceError.inner_iteration */
    int ans_buf;           /* which of the two u buffers holds the answer */
    double final_relative_residual;
    double trace0;
    double fnorm;
    double bad_rel;        /* relative residual that triggered divergence */
} rg_report;

int         rg_version(void);
const char* rg_last_error(void);

/* ---- operator (sparse.py:13-133 SparseMatrix, duck-typed by the solvers) */
int rg_op_create(rg_op** out, const rg_op_desc* desc);
int rg_op_destroy(rg_op* op);

/* y = A x for every system (sparse.py:101-106 -> scipy csr_matvec).  Summed
 * in CSR column order without FMA contraction: bitwise equal to SciPy. */
int rg_matvec(const rg_op* A, const void* x, void* y, void* stream);

/* r = f - A u (r may be NULL) and norm2[b] = ||r_b||^2 (device, may be NULL)
 * (richardson.py:105-106,124-125; np.linalg.norm -> deterministic
 * fixed-order reduction, not bitwise BLAS). */
int rg_residual(const rg_op* A, const void* u, const void* f, void* r,
                double* norm2, void* stream);

/* n_steps power-iteration steps (spectral.py:31-57, the loop body of
 * _power_iteration) for every system of a float64 operator, one fused launch
 * per step:  x = y_prev / ny_prev ;  y = A x  (shifted: y = sigma x - A x,
 * spectral.py:75-76) ;  lam[k][b] = <x, y> ;  ny[k][b] = ||y||.
 * Step 0 reads (y_prev, ny_prev) -- ny_prev NULL means y_prev already is the
 * normalised start vector; step k > 0 reads the previous step's y and ny.
 * y of step k goes to (k even ? y0 : y1); y_prev must not alias y0.
 * x_last (may be NULL) receives x of the last step.  lam and ny are device
 * arrays [n_steps][batch]. */
int rg_power_steps(const rg_op* A, int n_steps, const double* y_prev, const double* ny_prev,
                   double* y0, double* y1, double sigma, int shifted, double* lam,
                   double* ny, double* x_last, void* stream);

/* One inner update of _inner_update (richardson.py:49-59) for every system:
 *   plain/mom: r = f - A u ;  nag/nagex: r = f - A (u + at_i v)
 *   v_out = a_i v + w_i B^{-1} r ;  u_out = u + v_out
 * u_in/u_out and v_in/v_out must not alias (neighbour reads).  v_in may be
 * NULL (treated as 0) for plain.  If nonfinite_at (device int[batch]) is
 * given, the first `tag` at which u_out or v_out held a non-finite entry is
 * recorded with atomicMin (outer_sweep's check, richardson.py:67-70). */
int rg_inner_update(const rg_op* A, const rg_sched* s, int i,
                    const void* u_in, const void* v_in,
                    void* u_out, void* v_out, const void* f,
                    int* nonfinite_at, int tag, void* stream);

/* n_steps free-running inner updates (schedule index (i0 + t) mod m), with
 * no residual norms and no status: the smoothing loops of fns_lite_step
 * (fns.py:78-79, plain, weights cycled) and multigrid._smooth
 * (multigrid.py:126-138, fresh v, no preconditioner).  u0 holds the input
 * (and v0 the input velocity); u0/u1, v0/v1 are ping-pong buffers and
 * *out_buf (host int) says which one holds the result.  block_T as for the
 * solver (CONST9 real operators run temporally blocked). */
int rg_sweep(const rg_op* A, const rg_sched* s, int i0, int n_steps, int block_T,
             void* u0, void* u1, void* v0, void* v1, const void* f, int* out_buf,
             void* stream);
/* rg_sweep whose input v (zero_mask bit 0) and / or u (bit 1) are all zero,
 * as at the start of every smoothing call (multigrid.py:128 fresh v; :154
 * zero coarse guess): the caller need not clear u0 / v0, and the blocked
 * complex sweeps do not read them in their first launch.  zero_mask 0 is
 * rg_sweep. */
int rg_sweep_from_zero(const rg_op* A, const rg_sched* s, int i0, int n_steps, int block_T,
                       void* u0, void* u1, void* v0, void* v1, const void* f, int zero_mask,
                       int* out_buf, void* stream);
/* rg_sweep that also returns norm2_first[b] = ||f - A u0_b||^2, the residual
 * norm of the INPUT iterate (device [batch]): the first step computes that
 * residual anyway, so on the wavefront path the norm rides on the sweep's
 * fused reduction (fns.py:99 -- the relative residual after a correction is
 * the first residual of the next alternation's smoothing); other paths take
 * one rg_residual pass first. */
int rg_sweep_norm(const rg_op* A, const rg_sched* s, int i0, int n_steps, int block_T,
                  void* u0, void* u1, void* v0, void* v1, const void* f,
                  double* norm2_first, int* out_buf, void* stream);

/* ---- DST-I / FNS correction (transforms.py:24-35, fns.py:30-84) ----------
 * A plan holds the twiddle table and one [batch][side][side] workspace; one
 * call in flight per plan.  side+1 a power of two (4 .. 8192): FFT path;
 * any other side <= 4096: dense orthonormal sine-matrix products. */
typedef struct rg_dst rg_dst;
int rg_dst_create(rg_dst** out, int batch, int side);
int rg_dst_destroy(rg_dst* plan);
/* out = dst2(in) for every system (orthonormal 2D DST-I, involutory);
 * in and out may alias.  float64. */
int rg_dst2(const rg_dst* plan, const double* in, double* out, void* stream);
/* u += dst2(lam * dst2(f - A u)) for every system (SpectralCorrection.apply,
 * fns.py:43-44,80); lam is [batch][side*side] float64. */
int rg_fns_correct(const rg_op* A, const rg_dst* plan, const double* lam, double* u,
                   const double* f, void* stream);

/* ---- V-cycle pieces (multigrid.py:24-59,151-163) ---------------------------
 * n = cells per side of the FINE grid (even); fine vectors have (n-1)^2
 * entries, coarse ones (n/2-1)^2.  Bitwise equal to the reference's CSR
 * R.matvec / P.matvec (power-of-two weights, CSR summation order). */
int rg_restrict(int dtype, int batch, int n, const void* fine, void* coarse,
                void* stream);
/* fine += P coarse  (u = u + P.matvec(ec), multigrid.py:162) */
int rg_prolong_add(int dtype, int batch, int n, const void* coarse, void* fine,
                   void* stream);
/* y[b] = M x[b] with M dense [n][n] row-major (one per system, or one shared
 * when shared != 0): the coarsest-level solve with a precomputed inverse
 * (replaces scipy.linalg.lu_solve, multigrid.py:155; ~1e-15 relative). */
int rg_dense_apply(int dtype, int batch, int n, const void* M, int shared,
                   const void* x, void* y, void* stream);

/* ---- FGMRES building block (fgmres.py:76-78) -------------------------------
 * One fused modified Gram-Schmidt index for `batch` systems (vectors of n
 * float64 / complex128, system b at w + b*ldw etc.):
 *     w -= h[b] * v          (skipped when v is NULL)
 *     hn[b] = vdot(vn, w)    (skipped when vn is NULL; conj(vn) . w)
 *     wnorm2[b] = ||w||^2    (when wnorm2 is not NULL)
 * h, hn, wnorm2 are device arrays [batch]. */
int rg_mgs_step(int dtype, int batch, int n, void* w, long long ldw, const void* v,
                long long ldv, const void* h, const void* vn, long long ldvn, void* hn,
                double* wnorm2, void* stream);
/* One whole modified Gram-Schmidt orthogonalisation of w against
 * v_0 .. v_k (fgmres.py:76-78), k + 2 rg_mgs_step launches from one call:
 * v_i = V + i * n elements (system stride ldv), H is [k + 1][batch]
 * (H[i][b] = h_{i,k} of system b), wnorm2[b] = ||w||^2 afterwards. */
int rg_mgs_arnoldi(int dtype, int batch, int n, void* w, long long ldw, const void* V,
                   long long ldv, int k, void* H, double* wnorm2, void* stream);

/* Tail of an Arnoldi step (fgmres.py:79-80,106-107) for `batch` systems at
 * index k: hk1 = sqrt(wnorm2[b]); vnext_b = w_b / hk1; hcol[b][0..k+1] =
 * (H[0..k][b], hk1) packed for one device->host copy.  vnext is computed
 * unconditionally (the host ignores it after a stop). */
int rg_arnoldi_tail(int dtype, int batch, int n, const void* w, long long ldw, void* vnext,
                    long long ldv, const void* H, int k, const double* wnorm2, void* hcol,
                    void* stream);
/* u += Z[:, :k] y for one system (fgmres.py:119); Z column j at Z + j*ldz
 * elements, y device [k]. */
int rg_krylov_update(int dtype, int n, void* u, const void* Z, long long ldz, const void* y, int k,
                     void* stream);

/* ---- Gauss-Seidel / SOR / SSOR preconditioners (precond.py:79-118) --------
 * z = B^{-1} r for every system of any operator (CONST9 / DIAG5 / VAR9,
 * real or complex128; constant real stencils take a thread-block-cluster
 * wavefront, the rest a general one-CTA-per-system wavefront):
 *   RG_TRI_SOR  : z = relax (D + relax L)^{-1} r          (gauss_seidel: relax 1)
 *   RG_TRI_SSOR : z = c (D + relax U)^{-1} D (D + relax L)^{-1} r,
 *                 c = relax (2 - relax)
 * L, U: strict lower / upper parts of A in lexicographic order.  Replaces the
 * SuperLU triangular solves of precond.py:36-45 (agreement to rounding,
 * ~1e-15; the reference's own bar is 1e-13).  relax in (0, 2); a zero
 * diagonal is RG_EINVAL (ZeroDiagonalError) for CONST9 real operators and
 * the caller's check otherwise (the coefficients live on the device).  work: [batch][side*side]
 * scratch for SSOR (may be NULL for SOR).  r and z must not alias. */
enum rg_tri { RG_TRI_SOR = 1, RG_TRI_SSOR = 2,
              /* the transposed maps B^{-T} (Preconditioner.apply_transpose,
               * precond.py:94,112-113), used by the training adjoint */
              RG_TRI_SOR_T = 3, RG_TRI_SSOR_T = 4 };
int rg_tri_apply(const rg_op* A, int kind, double relax, const void* r, void* z,
                 void* work, void* stream);
/* The Richardson update from an externally preconditioned residual z
 * (richardson.py:120-121): v = a_i v + w_i z; u = u + v (in place), and when
 * y != NULL the next look-ahead y = u + at_{(i+1) mod m} v (nag/nagex).
 * z == NULL: only y = u + at_i v.  v may be NULL for plain. */
int rg_precond_update(const rg_op* A, const rg_sched* s, int i, const void* z,
                      void* u, void* v, void* y, void* stream);

/* ---- training unroll adjoint (training.py:84-104, tape.py:191-199) --------
 * Reverse pass of the K-step unroll from u_0 = v_0 = 0 whose loss is
 * L = ||f - A u_K|| / ||f|| (float64, CONST9 or VAR9; At = the operator
 * holding A^T, equal to A for the symmetric anisotropic stencils).  The
 * forward histories u_k, v_k come from rg_inner_update.
 * init: loss[b] = L_b, ubar = dL/du_K, vbar = 0 (rwork: [batch][P] scratch).
 * step (k = K-1 .. 0, i = k mod m): ubar/vbar go from the adjoints of
 * u_{k+1}, v_{k+1} to those of u_k, v_k in place, and dots[3][batch] gets
 * the contributions of step k to dL/dalpha_i, dL/domega_i and
 * dL/dalpha_tilde_i (the last zero for plain/mom).  Jacobi (scalar/field)
 * or no preconditioner.  Deterministic fixed-order reductions. */
int rg_unroll_adjoint_init(const rg_op* A, const rg_op* At, const void* uK,
                           const void* f, void* rwork, void* ubar, void* vbar,
                           double* loss, void* stream);
int rg_unroll_adjoint_step(const rg_op* A, const rg_op* At, const rg_sched* s,
                           int i, const void* f, const void* u_k, const void* v_k,
                           void* ubar, void* vbar, void* rbar, double* dots,
                           void* stream);

/* The same reverse step with a GS / SOR / SSOR preconditioner, in two
 * phases around the host's rg_tri_apply(RG_TRI_*_T, rbar_pre -> rbar):
 * phase 1 reads p_k (the forward's B^{-1} r_k history) and writes
 * rbar_pre = w_i vbar_total and dots[0..1][batch]; phase 2 reads rbar
 * (= B^{-T} rbar_pre), updates ubar / vbar and writes dots[2][batch]. */
int rg_unroll_adjoint_step_ext(const rg_op* A, const rg_op* At, const rg_sched* s,
                               int i, const void* v_k, const void* p_k, void* ubar,
                               void* vbar, void* rbar_pre, void* rbar, double* dots,
                               int phase, void* stream);

/* ---- solve_stationary engine (richardson.py:77-141) ----------------------
 * A solver owns device workspace (per-system status, trace, reduction
 * partials) and runs the whole loop on the device: convergence, divergence
 * and max_outer decisions are taken by the last CTA of each launch, and
 * finished systems are skipped by later launches, so the host only polls.
 * Iterates live in two caller-owned ping-pong buffers u0/u1 (and v0/v1 for
 * mom/nag/nagex); rg_report.ans_buf says which one holds the answer.
 * block_T: temporal-blocking depth (inner steps fused per HBM pass) for the
 * CONST9 real path; 0 = automatic, 1 = off.                              */
int rg_solver_create(rg_solver** out, const rg_op* A, const rg_sched* s,
                     double tol, int max_outer, int check, int block_T);
int rg_solver_destroy(rg_solver* S);
/* u0 holds the initial guess on entry; u1, v0, v1 are scratch. v0/v1 may be
 * NULL for plain. Computes ||f||, the initial residual and trace[0]. */
int rg_solver_begin(rg_solver* S, void* u0, void* u1, void* v0, void* v1,
                    const void* f, void* stream);
/* Enqueue exactly one kernel launch of the sweep schedule (no host sync).
 * *steps_out = inner steps it covers (0 once max_outer sweeps are queued). */
int rg_solver_step(rg_solver* S, void* stream, int* steps_out);
/* Enqueue n_sweeps outer sweeps (or up to max_outer) plus the trailing
 * residual check; no host sync. */
int rg_solver_run(rg_solver* S, int n_sweeps, void* stream);
/* Enqueue the residual check of the current iterate (resolves the lagged
 * convergence test of the last queued sweep). */
int rg_solver_flush(rg_solver* S, void* stream);
/* Synchronise `stream`, copy the per-system state to the host.
 * *n_active = systems still iterating; *done = 1 when nothing is left to do
 * (all systems finished or max_outer sweeps queued and flushed). */
int rg_solver_poll(rg_solver* S, void* stream, int* n_active, int* done);
int rg_solver_report(const rg_solver* S, int b, rg_report* out);
/* Copy trace[0..iterations] of system b into host buffer out (cap entries). */
int rg_solver_trace(const rg_solver* S, int b, double* out, int cap,
                    int* n_out);
/* The sweep kernel a solver uses (for measurement and reporting):
 * kernel = RG_KERNEL_STEP (one inner step per launch), RG_KERNEL_TILE
 * (overlapped-tile temporal blocking), RG_KERNEL_WAVE (wavefront strips,
 * seg_rows rows per segment) or RG_KERNEL_CLUSTER (the whole solve in one
 * launch); block_T = inner steps fused per launch. */
enum { RG_KERNEL_STEP = 0, RG_KERNEL_TILE = 1, RG_KERNEL_WAVE = 2, RG_KERNEL_CLUSTER = 3 };
int rg_solver_plan(const rg_solver* S, int* kernel, int* block_T, int* seg_rows);
/* Inner steps queued so far and the temporal-blocking depth in use. */
int rg_solver_info(const rg_solver* S, long long* steps_queued,
                   int* block_T, int* launches);

#ifdef __cplusplus
}
#endif
#endif /* RICHGPU_H */
