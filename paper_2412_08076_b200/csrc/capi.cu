// capi.cu — extern "C" boundary of librichgpu (declared in include/richgpu.h).
//
// Host-side dispatch, argument validation and the solve_stationary launch
// planner.  No torch types cross this boundary: plain pointers, ints and a
// cudaStream_t passed as void*.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <string>
#include <vector>

#include "../../include/richgpu.h"
#include "block.cuh"
#include "dst.cuh"
#include "dstw.cuh"
#include "mg.cuh"
#include "cluster.cuh"
#include "krylov.cuh"
#include <type_traits>
#include "cblock.cuh"
#include "tri.cuh"
#include "trigen.cuh"
#include "resid.cuh"
#include "adjoint.cuh"
#include "psweep.cuh"
#include "power.cuh"
#include "wave.cuh"

using namespace rg;

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
    char b[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(b, sizeof b, fmt, ap);
    va_end(ap);
    g_err = b;
    return code;
}

#define CUDA_TRY(expr)                                                              \
    do {                                                                            \
        cudaError_t e_ = (expr);                                                    \
        if (e_ != cudaSuccess)                                                      \
            return fail(RG_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),  \
                        __FILE__, __LINE__);                                        \
    } while (0)

#define LAUNCH_CHECK()                                                              \
    do {                                                                            \
        cudaError_t e_ = cudaGetLastError();                                        \
        if (e_ != cudaSuccess)                                                      \
            return fail(RG_ECUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                        \
    } while (0)

struct rg_op {
    rg_op_desc d;
    int P;
    std::vector<double> hcoef;   // CONST9 real: host copy of [batch][9] (kernel params)
    bool cblock_ok = false;      // DIAG5 c128 with one set of off-diagonals: blocked sweep
    double2 hoff[4];
    // VAR9 c128 whose rows mostly repeat one stencil (Galerkin levels of the
    // sponge Helmholtz operator: ~96% of rows bit-identical to the centre
    // row): that stencil as kernel parameters + a per-node "row == stencil"
    // flag, so the blocked sweep reads coefficient planes only in the band
    // where they vary.
    bool var9h = false;
    double2 hc9[9];
    unsigned char* mask = nullptr;  // device [P] (owned)
    ~rg_op() {
        if (mask) cudaFree(mask);
    }
};

struct rg_solver {
    const rg_op* A;
    rg_sched s;
    SolveCfg cfg;
    int check;
    int block_T;
    bool use_block;
    bool use_wave;    // plain sweeps take the wavefront kernel (wave.cuh)
    int wave_L;       // its segment rows
    bool use_small;   // whole solve in one launch (grid fits in shared memory)
    bool small_done;  // that launch has been queued
    int cl_nc, cl_rows, cl_ppt;   // cluster shape of the resident solver
    SysState* d_st;
    double* d_trace;
    double* d_part;
    int ncta_cap;
    int trace_stride;
    SysState* h_st;
    void* u[2];
    void* v[2];
    const void* f;
    std::vector<double> hscale;   // Jacobi scale per system (blocked path)
    long long k;
    long long kmax;
    long long flushed_k;
    int cur;
    int launches;
    bool need_flush;
    bool begun;
};

// ---------------------------------------------------------------- helpers
static size_t scalar_bytes(int dtype) {
    return dtype == RG_F32 ? 4 : dtype == RG_F64 ? 8 : 16;
}

static dim3 step_grid(const rg_op* A) {
    const int side = A->d.side;
    return dim3((side + STEP_BX - 1) / STEP_BX, (side + STEP_BY * STEP_RPT - 1) / (STEP_BY * STEP_RPT),
                A->d.batch);
}

template <typename S>
static OpView<S> view(const rg_op* A) {
    OpView<S> v;
    v.stencil = (const CT<S>*)A->d.stencil;
    v.diag = (const CT<S>*)A->d.diag;
    v.side = A->d.side;
    v.P = A->P;
    v.shared = A->d.shared;
    return v;
}

// ------------------------------------------------------- step1 dispatch
template <typename S, int KIND>
static int launch_step1_k(const rg_op* A, StepArgs<S>& a, cudaStream_t st) {
    step1_kernel<S, KIND><<<step_grid(A), dim3(STEP_BX, STEP_BY), 0, st>>>(a);
    LAUNCH_CHECK();
    return RG_OK;
}

template <typename S>
static int launch_step1(const rg_op* A, StepArgs<S>& a, cudaStream_t st) {
    switch (A->d.kind) {
        case RG_CONST9: return launch_step1_k<S, K_CONST9>(A, a, st);
        case RG_DIAG5: return launch_step1_k<S, K_DIAG5>(A, a, st);
        case RG_VAR9: return launch_step1_k<S, K_VAR9>(A, a, st);
    }
    return fail(RG_EINVAL, "bad operator kind %d", A->d.kind);
}

// Generic "one step" request independent of the scalar type.
struct StepReq {
    const void *u_in, *v_in, *f, *scale;
    void *u_out, *v_out, *r_out;
    const double *omega, *alpha, *atil;
    int m, i, variant, precond, update, norm_u, use_status;
    int* nonfinite_at;
    int tag;
    double* partials;
    EpiArgs epi;
};

template <typename S>
static int do_step1(const rg_op* A, const StepReq& q, cudaStream_t st) {
    StepArgs<S> a;
    a.A = view<S>(A);
    a.u_in = (const S*)q.u_in;
    a.v_in = (const S*)q.v_in;
    a.u_out = (S*)q.u_out;
    a.v_out = (S*)q.v_out;
    a.f = (const S*)q.f;
    a.r_out = (S*)q.r_out;
    a.omega = q.omega;
    a.alpha = q.alpha;
    a.atil = q.atil;
    a.scale = (const CT<S>*)q.scale;
    a.m = q.m;
    a.i = q.i;
    a.variant = q.variant;
    a.precond = q.precond;
    a.update = q.update;
    a.norm_u = q.norm_u;
    a.use_status = q.use_status;
    a.nonfinite_at = q.nonfinite_at;
    a.tag = q.tag;
    a.partials = q.partials;
    a.epi = q.epi;
    return launch_step1<S>(A, a, st);
}

static int step1(const rg_op* A, const StepReq& q, cudaStream_t st) {
    switch (A->d.dtype) {
        case RG_F32: return do_step1<float>(A, q, st);
        case RG_F64: return do_step1<double>(A, q, st);
        case RG_C128: return do_step1<double2>(A, q, st);
    }
    return fail(RG_EINVAL, "bad dtype %d", A->d.dtype);
}

// wavefront sweep tuning (env overrides for measurement: RG_WAVE=0 disables,
// RG_WAVE_T sets the default depth, RG_WAVE_L the segment rows)
static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}
// Segment rows of the wavefront sweep for a batch, or 0 when the grid gives
// too few strips x segments to fill the GPU (one-warp CTAs, 8 resident per
// SM at ~206 registers): then the overlapped-tile kernel, which cuts a system
// into ~4x more CTAs, is faster.  Measured on cfg3's 1023^2 systems
// (profiles/wave_batch_r02.json): 8 systems L = 64 352 vs tile 279 G upd/s;
// 4 systems L = 32 279 vs 250; 1-2 systems the tile kernel wins.
// RG_WAVE_L overrides (read per solver, so measurement scripts vary it).
static int wave_seg_rows(int side, int batch) {
    const int forced = env_int("RG_WAVE_L", 0);
    if (forced > 0) return forced < 8 ? 8 : forced;
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long slots = 8ll * nsm;
    for (int L = RG_WV_L; L >= 32; L /= 2) {
        int nstrip = 0;
        const long long n = (long long)batch * wave_ntiles(side, 4, L, &nstrip);
        if (n * 100 >= slots * 85) return L;
    }
    return 0;
}
static bool wave_enabled() { return env_int("RG_WAVE", 1) != 0; }
constexpr int WV_MIN_SIDE = 128;

// ------------------------------------------------------- block dispatch
template <typename S>
static int do_wave(rg_solver* S_, int T, cudaStream_t st) {
    const rg_op* A = S_->A;
    static thread_local WaveArgs<S> a;   // ~5 KB of kernel parameters
    a.side = A->d.side;
    a.P = A->P;
    a.u_in = (const S*)S_->u[S_->cur];
    a.u_out = (S*)S_->u[S_->cur ^ 1];
    a.f = (const S*)S_->f;
    a.omega = S_->s.omega;
    a.m = S_->s.m;
    a.k0 = (int)S_->k;
    a.seg_rows = S_->wave_L;
    wave_ntiles(A->d.side, T, a.seg_rows, &a.nstrip);
    const bool jac = S_->s.precond == RG_PRECOND_JACOBI_SCALAR;
    EpiArgs& e = a.epi;
    e.st = S_->d_st;
    e.trace = S_->d_trace;
    e.trace_stride = S_->trace_stride;
    e.partials = S_->d_part;
    e.ncta_cap = S_->ncta_cap;
    e.cfg = S_->cfg;
    e.j0 = (int)S_->k;
    e.nslots = T;
    e.with_f = 0;
    e.buf = S_->cur;
    const int B = A->d.batch;
    for (int b0 = 0; b0 < B; b0 += BLK_MAXB) {
        const int nsys = B - b0 < BLK_MAXB ? B - b0 : BLK_MAXB;
        a.b0 = b0;
        for (int j = 0; j < nsys; ++j) {
            for (int d = 0; d < 9; ++d) a.coef[j][d] = A->hcoef[(size_t)(b0 + j) * 9 + d];
            a.scale[j] = jac ? S_->hscale[b0 + j] : 0.0;
        }
        cudaError_t err = launch_wave<S>(a, T, jac, nsys, st);
        if (err != cudaSuccess) return fail(RG_ECUDA, "wave sweep launch: %s", cudaGetErrorString(err));
    }
    return RG_OK;
}

template <typename S>
static int do_block(rg_solver* S_, int T, int norm_first_u, cudaStream_t st) {
    const rg_op* A = S_->A;
    if (S_->use_wave && T <= WV_TMAX) return do_wave<S>(S_, T, st);
    static thread_local BlockArgs<S> a;   // ~5 KB of kernel parameters
    a.side = A->d.side;
    a.P = A->P;
    a.u_in = (const S*)S_->u[S_->cur];
    a.u_out = (S*)S_->u[S_->cur ^ 1];
    a.v_in = (const S*)S_->v[S_->cur];
    a.v_out = (S*)S_->v[S_->cur ^ 1];
    a.r_out = nullptr;
    a.f = (const S*)S_->f;
    a.omega = S_->s.omega;
    a.alpha = S_->s.alpha;
    a.atil = S_->s.alpha_tilde;
    a.m = S_->s.m;
    a.k0 = (int)S_->k;
    const bool nag = S_->s.variant >= RG_NAG;
    const bool jac = S_->s.precond == RG_PRECOND_JACOBI_SCALAR;
    a.norm_first_u = norm_first_u;
    a.norm_every = nag ? 0 : 1;
    block_ntiles(A->d.side, T, &a.nty);
    EpiArgs& e = a.epi;
    e.st = S_->d_st;
    e.trace = S_->d_trace;
    e.trace_stride = S_->trace_stride;
    e.partials = S_->d_part;
    e.ncta_cap = S_->ncta_cap;
    e.cfg = S_->cfg;
    e.j0 = (int)S_->k;
    e.nslots = nag ? (norm_first_u ? 1 : 0) : T;
    e.with_f = 0;
    e.buf = S_->cur;
    const int B = A->d.batch;
    for (int b0 = 0; b0 < B; b0 += BLK_MAXB) {
        const int nsys = B - b0 < BLK_MAXB ? B - b0 : BLK_MAXB;
        a.b0 = b0;
        for (int j = 0; j < nsys; ++j) {
            for (int d = 0; d < 9; ++d) a.coef[j][d] = A->hcoef[(size_t)(b0 + j) * 9 + d];
            a.scale[j] = jac ? S_->hscale[b0 + j] : 0.0;
        }
        cudaError_t err;
        switch (S_->s.variant) {
            case RG_PLAIN: err = launch_block<S, V_PLAIN>(a, T, jac, nsys, st); break;
            case RG_MOM: err = launch_block<S, V_MOM>(a, T, jac, nsys, st); break;
            default: err = launch_block<S, V_NAG>(a, T, jac, nsys, st); break;
        }
        if (err != cudaSuccess) return fail(RG_ECUDA, "block sweep launch: %s", cudaGetErrorString(err));
    }
    return RG_OK;
}

// ------------------------------------------------------------- validation
static int check_op(const rg_op* A) {
    if (!A) return fail(RG_ENULL, "null operator");
    return RG_OK;
}

static int check_sched(const rg_op* A, const rg_sched* s) {
    if (!s) return fail(RG_ENULL, "null schedule");
    if (s->m < 1) return fail(RG_EINVAL, "schedule needs at least one weight (m=%d)", s->m);
    if (s->variant < RG_PLAIN || s->variant > RG_NAGEX)
        return fail(RG_EINVAL, "unknown variant %d", s->variant);
    if (!s->omega) return fail(RG_ENULL, "null omega");
    if (s->variant != RG_PLAIN && !s->alpha) return fail(RG_ENULL, "variant needs alpha");
    if (s->variant >= RG_NAG && !s->alpha_tilde) return fail(RG_ENULL, "variant needs alpha_tilde");
    if (s->precond < RG_PRECOND_NONE || s->precond > RG_PRECOND_JACOBI_FIELD)
        return fail(RG_EINVAL, "unknown preconditioner %d", s->precond);
    if (s->precond != RG_PRECOND_NONE && !s->scale) return fail(RG_ENULL, "Jacobi needs scale");
    (void)A;
    return RG_OK;
}

struct rg_dst {
    int batch, side, M, logM, lpc;
    double2* tw;     // [M]
    double* work;    // [batch][side][side] residual / intermediate
    // lean kernels (dstw.cu, M = 512 / 1024 / 2048): the intermediate lives in
    // a padded [batch][M][M] array (entry (i, k) at i * M + k, row / column 0
    // unused), so rows start 16-byte aligned and 4 adjacent columns of a row
    // are one 32-byte sector
    bool lean = false;
    double* wpad = nullptr;
    int num_sms = 148;
    // dense path (side + 1 not a power of two): the orthonormal DST-I matrix
    bool dense = false;
    double* S = nullptr;      // [side][side]
    double* work2 = nullptr;  // [batch][side][side]
};

// C = P Q for every system (dense DST path); P or Q may be the shared S.
static int dst_gemm(const rg_dst* D, const double* P, bool p_batched, const double* Q,
                    bool q_batched, double* C, int mode, const double* lam, cudaStream_t st) {
    GemmArgs g;
    const size_t NN = (size_t)D->side * D->side;
    g.P = P; g.sP = p_batched ? NN : 0;
    g.Q = Q; g.sQ = q_batched ? NN : 0;
    g.C = C; g.sC = NN;
    g.lam = lam;
    g.N = D->side;
    g.mode = mode;
    const int nb = (D->side + GM_T - 1) / GM_T;
    dst_gemm_kernel<<<dim3(nb, nb, D->batch), GM_NT, 0, st>>>(g);
    LAUNCH_CHECK();
    return RG_OK;
}

// Lines per CTA of the compile-time M = 1024 kernels (cfg4's size), per axis;
// RG_DST_LPC_ROW / RG_DST_LPC_COL (2 or 4) override for tuning.
static int dst_lpc_1024(int axis) {
    static int v[2] = {-1, -1};
    if (v[axis] < 0) {
        const char* ev = getenv(axis == 0 ? "RG_DST_LPC_ROW" : "RG_DST_LPC_COL");
        v[axis] = ev ? atoi(ev) : 4;   // measured: 4 / 4 best (0.380 ms per FNS alternation)
        if (v[axis] != 2) v[axis] = 4;
    }
    return v[axis];
}

static int dst_pass(const rg_dst* D, int axis, int mode, const double* in, double* out,
                    const double* lam, cudaStream_t st) {
    const bool cm = D->M == 1024;   // compile-time indexing
    const int lpc = cm ? dst_lpc_1024(axis) : D->lpc;
    DstArgs a;
    a.in = in;
    a.out = out;
    a.tw = D->tw;
    a.lam = lam;
    a.N = D->side;
    a.M = D->M;
    a.logM = D->logM;
    a.lpc = lpc;
    a.mode = mode;
    a.scale = sqrt(2.0 / D->M);
    // in-place FFT: lpc lines + the twiddle table (M <= DST_SMEM_TW_MAX) + lam staging
    const size_t smem = ((size_t)lpc * dst_ls(D->M) + (D->M <= DST_SMEM_TW_MAX ? D->M : 0)) * sizeof(double2) +
                        (mode == DST_TWICE_LAM ? (size_t)lpc * (D->M + 8) * sizeof(double) : 0);
    const int nt = lpc * (D->M / dst_vpt(D->M));
    const dim3 grid((D->side + lpc - 1) / lpc, D->batch);
    auto go = [&](auto kern) -> int {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<grid, nt, smem, st>>>(a);
        return RG_OK;
    };
    int rc;
    if (cm && lpc == 2) rc = axis == 0 ? go(dst_lines_kernel<0, 256, 10, 2>) : go(dst_lines_kernel<1, 256, 10, 2>);
    else if (cm) rc = axis == 0 ? go(dst_lines_kernel<0, 256, 10, 4>) : go(dst_lines_kernel<1, 256, 10, 4>);
    else if (nt <= 256) rc = axis == 0 ? go(dst_lines_kernel<0, 256, 0, 0>) : go(dst_lines_kernel<1, 256, 0, 0>);
    else rc = axis == 0 ? go(dst_lines_kernel<0, 512, 0, 0>) : go(dst_lines_kernel<1, 512, 0, 0>);
    if (rc) return rc;
    LAUNCH_CHECK();
    return RG_OK;
}

// Views of the lean kernels (dstw.cuh): unpadded [side][side] arrays and the
// padded intermediate, walked by rows or by columns.
static DstwView dstw_view(const double* p, int side, bool padded, bool by_cols) {
    DstwView v;
    const long long M = side + 1;
    v.base = const_cast<double*>(p);
    const long long rs = padded ? M : side;          // row stride
    v.bs = rs * rs;
    v.off = padded ? 0 : -(long long)(side + 1);     // (1, 1) is entry 0 of an unpadded array
    v.ls = by_cols ? 1 : rs;
    v.es = by_cols ? rs : 1;
    return v;
}

static int dstw_pass(const rg_dst* D, bool col, int mode, const double* in, bool in_padded, double* out,
                     bool out_padded, const double* lam, cudaStream_t st) {
    DstwArgs a;
    a.in = dstw_view(in, D->side, in_padded, col);
    a.out = dstw_view(out, D->side, out_padded, col);
    a.lam = dstw_view(lam, D->side, false, col);
    a.tw = D->tw;
    a.B = D->batch;
    a.N = D->side;
    a.s4 = -0.25 * sqrt(2.0 / D->M);
    const cudaError_t e = launch_dstw(a, D->logM, col, mode, D->num_sms, st);
    if (e != cudaSuccess) return fail(RG_ECUDA, "dst launch: %s", cudaGetErrorString(e));
    return RG_OK;
}

// Free-running inner steps (no norms, no status): see rg_sweep in the header.
template <typename S>
static int sweep_block(const rg_op* A, const rg_sched* s, int k0, int T, bool jac_scalar,
                       const std::vector<double>& hscale, void* uin, void* uout, void* vin,
                       void* vout, const void* f, cudaStream_t st) {
    static thread_local BlockArgs<S> a;
    memset(&a.epi, 0, sizeof a.epi);
    a.side = A->d.side;
    a.P = A->P;
    a.u_in = (const S*)uin;
    a.u_out = (S*)uout;
    a.v_in = (const S*)vin;
    a.v_out = (S*)vout;
    a.r_out = nullptr;
    a.f = (const S*)f;
    a.omega = s->omega;
    a.alpha = s->alpha;
    a.atil = s->alpha_tilde;
    a.m = s->m;
    a.k0 = k0;
    a.norm_first_u = 0;
    a.norm_every = 0;
    block_ntiles(A->d.side, T, &a.nty);
    const int B = A->d.batch;
    for (int b0 = 0; b0 < B; b0 += BLK_MAXB) {
        const int nsys = B - b0 < BLK_MAXB ? B - b0 : BLK_MAXB;
        a.b0 = b0;
        for (int j = 0; j < nsys; ++j) {
            for (int d = 0; d < 9; ++d) a.coef[j][d] = A->hcoef[(size_t)(b0 + j) * 9 + d];
            a.scale[j] = jac_scalar ? hscale[b0 + j] : 0.0;
        }
        cudaError_t err;
        switch (s->variant) {
            case RG_PLAIN: err = launch_block<S, V_PLAIN>(a, T, jac_scalar, nsys, st); break;
            case RG_MOM: err = launch_block<S, V_MOM>(a, T, jac_scalar, nsys, st); break;
            default: err = launch_block<S, V_NAG>(a, T, jac_scalar, nsys, st); break;
        }
        if (err != cudaSuccess) return fail(RG_ECUDA, "sweep launch: %s", cudaGetErrorString(err));
    }
    return RG_OK;
}

// The same T plain steps through the wavefront-strip kernel (wave.cuh), no
// norm epilogue: rg_sweep's smoothing calls (FNS alternations, real V-cycles).
template <typename S>
static int sweep_wave(const rg_op* A, const rg_sched* s, int k0, int T, int seg_rows, bool jac_scalar,
                      const std::vector<double>& hscale, void* uin, void* uout, const void* f,
                      cudaStream_t st, const EpiArgs* epi = nullptr) {
    static thread_local WaveArgs<S> a;
    if (epi) a.epi = *epi;
    else a.epi = EpiArgs{};
    a.side = A->d.side;
    a.P = A->P;
    a.u_in = (const S*)uin;
    a.u_out = (S*)uout;
    a.f = (const S*)f;
    a.omega = s->omega;
    a.m = s->m;
    a.k0 = k0;
    a.seg_rows = seg_rows;
    wave_ntiles(A->d.side, T, seg_rows, &a.nstrip);
    const int B = A->d.batch;
    for (int b0 = 0; b0 < B; b0 += BLK_MAXB) {
        const int nsys = B - b0 < BLK_MAXB ? B - b0 : BLK_MAXB;
        a.b0 = b0;
        for (int j = 0; j < nsys; ++j) {
            for (int d = 0; d < 9; ++d) a.coef[j][d] = A->hcoef[(size_t)(b0 + j) * 9 + d];
            a.scale[j] = jac_scalar ? hscale[b0 + j] : 0.0;
        }
        cudaError_t err = launch_wave<S>(a, T, jac_scalar, nsys, st);
        if (err != cudaSuccess) return fail(RG_ECUDA, "wave sweep launch: %s", cudaGetErrorString(err));
    }
    return RG_OK;
}

// Length of the blocked chunk that starts at step i of an n-step run: n is
// split into round(n / T) nearly equal chunks (at most 8 steps each), so a
// 32-step sweep at T=5 runs as 6,6,5,5,5,5 instead of 5,5,5,5,5,5,2.
static int chunk_len(int n, int T, int i) {
    int nc = (n + T / 2) / T;
    if (nc < 1) nc = 1;
    if (nc < (n + 7) / 8) nc = (n + 7) / 8;
    const int base = n / nc, rem = n % nc;
    int start = 0;
    for (int c = 0; c < nc; ++c) {
        const int len = base + (c < rem ? 1 : 0);
        if (i < start + len) return start + len - i;   // steps left in this chunk
        start += len;
    }
    return 1;
}

// smallest side that takes the blocked 9-point complex sweep automatically
static int cb9_min_side() {
    static int v = -1;
    if (v < 0) {
        const char* ev = getenv("RG_CB9_MINSIDE");   // tuning override
        v = ev ? atoi(ev) : 200;
    }
    return v;
}

// balanced chunks of at most T steps (the complex blocked sweeps instantiate T <= 4)
static int chunk_cap(int n, int T, int i) {
    const int nc = (n + T - 1) / T;
    const int base = n / nc, rem = n % nc;
    int start = 0;
    for (int c = 0; c < nc; ++c) {
        const int len = base + (c < rem ? 1 : 0);
        if (i < start + len) return start + len - i;
        start += len;
    }
    return 1;
}

// ==================================================================== C ABI
// CONST9 / VAR9 dispatch for the adjoint kernels
template <typename K>
static cudaError_t by_kind(int kind, K k) {
    if (kind == RG_CONST9) k(std::integral_constant<int, K_CONST9>());
    else k(std::integral_constant<int, K_VAR9>());
    return cudaGetLastError();
}

// Stream-ordered scratch (reduction partials) comes from the device's
// default memory pool.  Its default release threshold (0) hands memory back
// to the driver at every synchronisation, which made the first allocation
// after each host sync cost ~0.9 ms (measured in the FGMRES loop); keep it.
static void ensure_pool() {
    static bool done[64] = {false};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

extern "C" {

int rg_version(void) { return RG_ABI_VERSION; }

const char* rg_last_error(void) { return g_err.c_str(); }

int rg_op_create(rg_op** out, const rg_op_desc* d) {
    if (!out || !d) return fail(RG_ENULL, "null argument");
    if (d->dtype != RG_F32 && d->dtype != RG_F64 && d->dtype != RG_C128)
        return fail(RG_EINVAL, "bad dtype %d", d->dtype);
    if (d->kind != RG_CONST9 && d->kind != RG_DIAG5 && d->kind != RG_VAR9)
        return fail(RG_EINVAL, "bad operator kind %d", d->kind);
    if (d->batch < 1 || d->side < 1) return fail(RG_ESIZE, "batch=%d side=%d", d->batch, d->side);
    if ((long long)d->side * d->side > (1ll << 30)) return fail(RG_ESIZE, "grid too large");
    if (!d->stencil) return fail(RG_ENULL, "null stencil");
    if (d->kind == RG_DIAG5 && !d->diag) return fail(RG_ENULL, "DIAG5 needs a diagonal");
    rg_op* A = new rg_op;
    A->d = *d;
    A->P = d->side * d->side;
    if (d->kind == RG_CONST9 && (d->dtype == RG_F64 || d->dtype == RG_F32)) {
        // the blocked sweep takes the 9 coefficients as kernel parameters
        const size_t n = (size_t)(d->shared ? 1 : d->batch) * 9;
        A->hcoef.resize(n);
        cudaError_t e;
        // coefficients are float64 for both F64 and F32 operators
        e = cudaMemcpy(A->hcoef.data(), d->stencil, n * sizeof(double), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            delete A;
            return fail(RG_ECUDA, "reading CONST9 coefficients: %s", cudaGetErrorString(e));
        }
        if (d->shared) {   // replicate for the per-system parameter table
            A->hcoef.resize((size_t)d->batch * 9);
            for (int b = 1; b < d->batch; ++b)
                for (int q = 0; q < 9; ++q) A->hcoef[(size_t)b * 9 + q] = A->hcoef[q];
        }
    }
    if (d->kind == RG_DIAG5 && d->dtype == RG_C128) {
        const int nsets = d->shared ? 1 : d->batch;
        std::vector<double2> off((size_t)nsets * 4);
        if (cudaMemcpy(off.data(), d->stencil, off.size() * sizeof(double2), cudaMemcpyDeviceToHost) ==
            cudaSuccess) {
            bool same = true;
            for (int b = 1; b < nsets && same; ++b)
                for (int q = 0; q < 4; ++q)
                    same = same && off[b * 4 + q].x == off[q].x && off[b * 4 + q].y == off[q].y;
            A->cblock_ok = same;
            for (int q = 0; q < 4; ++q) A->hoff[q] = off[q];
        }
    }
    if (d->kind == RG_VAR9 && d->dtype == RG_C128 && (d->shared || d->batch == 1)) {
        // one coefficient set: find the rows equal (on their in-grid entries)
        // to the centre row; worth it when they are the large majority
        const int side = d->side;
        const size_t P = A->P;
        std::vector<double2> pl(9 * P);
        if (cudaMemcpy(pl.data(), d->stencil, pl.size() * sizeof(double2), cudaMemcpyDeviceToHost) ==
                cudaSuccess && side >= 3) {
            const size_t ic = (size_t)(side / 2) * side + side / 2;
            double2 c[9];
            for (int q = 0; q < 9; ++q) c[q] = pl[q * P + ic];
            std::vector<unsigned char> m(P);
            size_t same = 0;
            for (int i = 0; i < side; ++i)
                for (int j = 0; j < side; ++j) {
                    const size_t idx = (size_t)i * side + j;
                    bool eq = true;
                    for (int q = 0; q < 9 && eq; ++q) {
                        const int ii = i + q / 3 - 1, jj = j + q % 3 - 1;
                        if (ii < 0 || ii >= side || jj < 0 || jj >= side) continue;   // zero-padded
                        const double2 v = pl[q * P + idx];
                        // bitwise equality (distinguishes +0 / -0)
                        eq = memcmp(&v, &c[q], sizeof(double2)) == 0;
                    }
                    m[idx] = eq ? 1 : 0;
                    same += eq;
                }
            if (same * 4 >= P * 3 && cudaMalloc((void**)&A->mask, P) == cudaSuccess) {
                if (cudaMemcpy(A->mask, m.data(), P, cudaMemcpyHostToDevice) == cudaSuccess) {
                    A->var9h = true;
                    for (int q = 0; q < 9; ++q) A->hc9[q] = c[q];
                } else {
                    cudaFree(A->mask);
                    A->mask = nullptr;
                }
            }
        }
    }
    *out = A;
    return RG_OK;
}

int rg_op_destroy(rg_op* A) {
    delete A;
    return RG_OK;
}

int rg_matvec(const rg_op* A, const void* x, void* y, void* stream) {
    int rc = check_op(A);
    if (rc) return rc;
    if (!x || !y) return fail(RG_ENULL, "null vector");
    cudaStream_t st = (cudaStream_t)stream;
    const dim3 g((A->d.side + STEP_BX - 1) / STEP_BX, (A->d.side + STEP_BY - 1) / STEP_BY, A->d.batch);
    const dim3 blk(STEP_BX, STEP_BY);
#define MV(S, K) matvec_kernel<S, K><<<g, blk, 0, st>>>(view<S>(A), (const S*)x, (S*)y)
    switch (A->d.dtype * 10 + A->d.kind) {
        case RG_F32 * 10 + RG_CONST9: MV(float, K_CONST9); break;
        case RG_F32 * 10 + RG_DIAG5: MV(float, K_DIAG5); break;
        case RG_F32 * 10 + RG_VAR9: MV(float, K_VAR9); break;
        case RG_F64 * 10 + RG_CONST9: MV(double, K_CONST9); break;
        case RG_F64 * 10 + RG_DIAG5: MV(double, K_DIAG5); break;
        case RG_F64 * 10 + RG_VAR9: MV(double, K_VAR9); break;
        case RG_C128 * 10 + RG_CONST9: MV(double2, K_CONST9); break;
        case RG_C128 * 10 + RG_DIAG5: MV(double2, K_DIAG5); break;
        case RG_C128 * 10 + RG_VAR9: MV(double2, K_VAR9); break;
        default: return fail(RG_EINVAL, "bad dtype/kind");
    }
#undef MV
    LAUNCH_CHECK();
    return RG_OK;
}

// r = f - A u (+ per-CTA partials of ||r||^2) for constant real stencils (resid.cuh)
static int resid9_ncta(const rg_op* A) {
    return ((A->d.side + RS_TC - 1) / RS_TC) * ((A->d.side + RS_TR - 1) / RS_TR);
}
static int launch_resid9(const rg_op* A, const void* u, const void* f, void* r, double* part,
                         cudaStream_t st) {
    const dim3 g((A->d.side + RS_TC - 1) / RS_TC, (A->d.side + RS_TR - 1) / RS_TR, A->d.batch);
    if (A->d.dtype == RG_F64) {
        ResidArgs<double> a{(const double*)A->d.stencil, A->d.shared, A->d.side, A->P,
                            (const double*)u, (const double*)f, (double*)r, part};
        resid9_kernel<double><<<g, RS_NT, 0, st>>>(a);
    } else {
        ResidArgs<float> a{(const double*)A->d.stencil, A->d.shared, A->d.side, A->P,
                           (const float*)u, (const float*)f, (float*)r, part};
        resid9_kernel<float><<<g, RS_NT, 0, st>>>(a);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RG_OK : fail(RG_ECUDA, "residual launch: %s", cudaGetErrorString(e));
}

int rg_residual(const rg_op* A, const void* u, const void* f, void* r, double* norm2,
                void* stream) {
    int rc = check_op(A);
    if (rc) return rc;
    if (!u || !f) return fail(RG_ENULL, "null vector");
    cudaStream_t st = (cudaStream_t)stream;
    if (A->d.kind == RG_CONST9 && A->d.dtype != RG_C128 && env_int("RG_RESID_TILED", 1)) {
        // constant real stencils: the shared-memory tiled pass (resid.cuh)
        const int ncta = resid9_ncta(A);
        double* part = nullptr;
        if (norm2) {
            ensure_pool();
            CUDA_TRY(cudaMallocAsync((void**)&part, sizeof(double) * ncta * A->d.batch, st));
        }
        if ((rc = launch_resid9(A, u, f, r, part, st))) return rc;
        if (norm2) {
            sum_partials_kernel<256><<<A->d.batch, 256, 0, st>>>(part, ncta, norm2);
            const cudaError_t e = cudaGetLastError();
            CUDA_TRY(cudaFreeAsync(part, st));
            if (e != cudaSuccess) return fail(RG_ECUDA, "reduce launch: %s", cudaGetErrorString(e));
        }
        return RG_OK;
    }
    StepReq q;
    memset(&q, 0, sizeof q);
    q.u_in = u;
    q.f = f;
    q.r_out = r;
    q.m = 1;
    q.norm_u = norm2 ? 1 : 0;
    const dim3 g = step_grid(A);
    const int ncta = g.x * g.y;
    if (norm2) {
        ensure_pool();
        CUDA_TRY(cudaMallocAsync((void**)&q.partials, sizeof(double) * ncta * A->d.batch, st));
    }
    rc = step1(A, q, st);
    if (rc == RG_OK && norm2) {
        sum_partials_kernel<256><<<A->d.batch, 256, 0, st>>>(q.partials, ncta, norm2);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(RG_ECUDA, "reduce launch: %s", cudaGetErrorString(e));
    }
    if (norm2) CUDA_TRY(cudaFreeAsync(q.partials, st));
    return rc;
}

int rg_power_steps(const rg_op* A, int n_steps, const double* y_prev, const double* ny_prev,
                   double* y0, double* y1, double sigma, int shifted, double* lam, double* ny,
                   double* x_last, void* stream) {
    int rc = check_op(A);
    if (rc) return rc;
    if (A->d.dtype != RG_F64) return fail(RG_EUNSUPPORTED, "power steps run on float64 operators");
    if (!y_prev || !y0 || !y1 || !lam || !ny) return fail(RG_ENULL, "null argument");
    if (n_steps < 0) return fail(RG_EINVAL, "n_steps=%d", n_steps);
    if ((const double*)y_prev == y0 || y0 == y1) return fail(RG_EINVAL, "y_prev / y0 / y1 alias");
    if (n_steps == 0) return RG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const dim3 g((A->d.side + STEP_BX - 1) / STEP_BX, (A->d.side + STEP_BY - 1) / STEP_BY, A->d.batch);
    const int ncta = g.x * g.y;
    const int B = A->d.batch;
    ensure_pool();
    char* ws = nullptr;
    const size_t part_bytes = sizeof(double) * 2 * (size_t)ncta * B;
    CUDA_TRY(cudaMallocAsync((void**)&ws, part_bytes + sizeof(int) * B, st));
    int* counter = (int*)(ws + part_bytes);
    CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int) * B, st));
    PowerArgs a;
    a.A = view<double>(A);
    a.sigma = sigma;
    a.shifted = shifted ? 1 : 0;
    a.part = (double*)ws;
    a.ncta_cap = ncta;
    a.counter = counter;
    for (int k = 0; k < n_steps && rc == RG_OK; ++k) {
        a.y_prev = k == 0 ? y_prev : ((k - 1) & 1 ? y1 : y0);
        a.ny_prev = k == 0 ? ny_prev : ny + (size_t)(k - 1) * B;
        a.y_out = (k & 1) ? y1 : y0;
        a.x_out = k == n_steps - 1 ? x_last : nullptr;
        a.lam_out = lam + (size_t)k * B;
        a.ny_out = ny + (size_t)k * B;
        switch (A->d.kind) {
            case RG_CONST9: power_step_kernel<K_CONST9><<<g, dim3(STEP_BX, STEP_BY), 0, st>>>(a); break;
            case RG_DIAG5: power_step_kernel<K_DIAG5><<<g, dim3(STEP_BX, STEP_BY), 0, st>>>(a); break;
            default: power_step_kernel<K_VAR9><<<g, dim3(STEP_BX, STEP_BY), 0, st>>>(a); break;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(RG_ECUDA, "power step launch: %s", cudaGetErrorString(e));
    }
    CUDA_TRY(cudaFreeAsync(ws, st));
    return rc;
}

int rg_inner_update(const rg_op* A, const rg_sched* s, int i, const void* u_in, const void* v_in,
                    void* u_out, void* v_out, const void* f, int* nonfinite_at, int tag,
                    void* stream) {
    int rc = check_op(A);
    if (rc) return rc;
    if ((rc = check_sched(A, s))) return rc;
    if (i < 0 || i >= s->m) return fail(RG_EINVAL, "inner index %d outside [0, %d)", i, s->m);
    if (!u_in || !u_out || !f) return fail(RG_ENULL, "null vector");
    if (u_in == u_out) return fail(RG_EINVAL, "u_in and u_out must not alias");
    if (s->variant >= RG_NAG && v_in && v_in == v_out)
        return fail(RG_EINVAL, "v_in and v_out must not alias for nag/nagex");
    StepReq q;
    memset(&q, 0, sizeof q);
    q.u_in = u_in;
    q.v_in = v_in;
    q.u_out = u_out;
    q.v_out = v_out;
    q.f = f;
    q.omega = s->omega;
    q.alpha = s->alpha;
    q.atil = s->alpha_tilde;
    q.scale = s->scale;
    q.m = s->m;
    q.i = i;
    q.variant = s->variant;
    q.precond = s->precond;
    q.update = 1;
    q.nonfinite_at = nonfinite_at;
    q.tag = tag;
    return step1(A, q, (cudaStream_t)stream);
}

int rg_tri_apply(const rg_op* A, int kind, double relax, const void* r, void* z, void* work,
                 void* stream) {
    int rc = check_op(A);
    if (rc) return rc;
    if (kind < RG_TRI_SOR || kind > RG_TRI_SSOR_T) return fail(RG_EINVAL, "bad triangular kind %d", kind);
    const bool needs_work = kind == RG_TRI_SSOR || kind == RG_TRI_SSOR_T;
    if (!(relax > 0.0 && relax < 2.0)) return fail(RG_EINVAL, "relaxation must be in (0, 2), got %g", relax);
    if (!r || !z || (needs_work && !work)) return fail(RG_ENULL, "null vector");
    if (r == z || work == r || work == z) return fail(RG_EINVAL, "r, z and work must not alias");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if (A->d.kind == RG_CONST9 && A->d.dtype != RG_C128) {
        // constant real stencils: the cluster wavefront (tri.cuh)
        for (int b = 0; b < (A->d.shared ? 1 : A->d.batch); ++b)
            if (A->hcoef[(size_t)b * 9 + 4] == 0.0) return fail(RG_EINVAL, "zero diagonal entry in system %d", b);
        if (A->d.dtype == RG_F64) {
            TriArgs<double> a{(const double*)A->d.stencil, A->d.shared, A->d.side, A->P, relax,
                              (const double*)r, (double*)z, (double*)work};
            e = launch_tri(a, kind, A->d.batch, st);
        } else {
            TriArgs<float> a{(const double*)A->d.stencil, A->d.shared, A->d.side, A->P, relax,
                             (const float*)r, (float*)z, (float*)work};
            e = launch_tri(a, kind, A->d.batch, st);
        }
    } else {
        // per-node coefficients and complex scalars (trigen.cuh); the caller
        // has checked the diagonal (it lives on the device)
#define RG_TG(S, C)                                                                               \
    {                                                                                             \
        TriGenArgs<S> a{(const C*)A->d.stencil, (const C*)A->d.diag, A->d.shared, A->d.side, A->P, \
                        relax, (const S*)r, (S*)z, (S*)work};                                     \
        e = A->d.kind == RG_CONST9 ? launch_trigen<S, K_CONST9>(a, kind, A->d.batch, st)          \
            : A->d.kind == RG_DIAG5 ? launch_trigen<S, K_DIAG5>(a, kind, A->d.batch, st)          \
                                    : launch_trigen<S, K_VAR9>(a, kind, A->d.batch, st);          \
    }
        if (A->d.dtype == RG_C128) RG_TG(double2, double2)
        else if (A->d.dtype == RG_F64) RG_TG(double, double)
        else RG_TG(float, double)
#undef RG_TG
    }
    return e == cudaSuccess ? RG_OK : fail(RG_ECUDA, "triangular solve launch: %s", cudaGetErrorString(e));
}

int rg_precond_update(const rg_op* A, const rg_sched* s, int i, const void* z, void* u, void* v,
                      void* y, void* stream) {
    int rc = check_op(A);
    if (rc) return rc;
    if ((rc = check_sched(A, s))) return rc;
    if (i < 0 || i >= s->m) return fail(RG_EINVAL, "inner index %d outside [0, %d)", i, s->m);
    if (!u) return fail(RG_ENULL, "null u");
    if (s->variant != RG_PLAIN && !v) return fail(RG_ENULL, "variant needs v");
    if (!z && !y) return fail(RG_ENULL, "nothing to compute");
    if ((y || !z) && !s->alpha_tilde) return fail(RG_ENULL, "look-ahead needs alpha_tilde");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = (size_t)A->d.batch * A->P;
    const int nb = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
    const int var = s->variant;
    switch (A->d.dtype) {
        case RG_F64:
            pupdate_kernel<double><<<nb, 256, 0, st>>>(A->d.batch, A->P, (const double*)z, (double*)u,
                                                      (double*)v, (double*)y, s->omega, s->alpha,
                                                      s->alpha_tilde, s->m, i, var);
            break;
        case RG_F32:
            pupdate_kernel<float><<<nb, 256, 0, st>>>(A->d.batch, A->P, (const float*)z, (float*)u,
                                                     (float*)v, (float*)y, s->omega, s->alpha,
                                                     s->alpha_tilde, s->m, i, var);
            break;
        default:
            return fail(RG_EUNSUPPORTED, "external-preconditioner update needs a real operator");
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RG_OK : fail(RG_ECUDA, "update launch: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------- adjoint
static int check_adj_ops(const rg_op* A, const rg_op* At) {
    int rc = check_op(A);
    if (rc) return rc;
    if ((rc = check_op(At))) return rc;
    if (A->d.dtype != RG_F64 || At->d.dtype != RG_F64)
        return fail(RG_EUNSUPPORTED, "the unroll adjoint runs on float64 operators");
    if (A->d.kind != At->d.kind || (A->d.kind != RG_CONST9 && A->d.kind != RG_VAR9))
        return fail(RG_EUNSUPPORTED, "the unroll adjoint needs CONST9 or VAR9 operators A, A^T");
    if (A->d.side != At->d.side || A->d.batch != At->d.batch)
        return fail(RG_ESIZE, "A and A^T disagree in side or batch");
    return RG_OK;
}

int rg_unroll_adjoint_init(const rg_op* A, const rg_op* At, const void* uK, const void* f,
                           void* rwork, void* ubar, void* vbar, double* loss, void* stream) {
    int rc = check_adj_ops(A, At);
    if (rc) return rc;
    if (!uK || !f || !rwork || !ubar || !vbar || !loss) return fail(RG_ENULL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const dim3 g = step_grid(A), blk(STEP_BX, STEP_BY);
    const int ncta = g.x * g.y, B = A->d.batch;
    double *part = nullptr, *sums = nullptr;
    ensure_pool();
    CUDA_TRY(cudaMallocAsync((void**)&part, sizeof(double) * 2 * B * ncta, st));
    ensure_pool();
    CUDA_TRY(cudaMallocAsync((void**)&sums, sizeof(double) * 2 * B, st));
    const OpView<double> av = view<double>(A), tv = view<double>(At);
    cudaError_t e = by_kind(A->d.kind, [&](auto kk) {
        constexpr int KIND = decltype(kk)::value;
        adj_seed_a_kernel<KIND><<<g, blk, 0, st>>>(av, (const double*)uK, (const double*)f,
                                                   (double*)rwork, part);
        sum_partials_kernel<256><<<2 * B, 256, 0, st>>>(part, ncta, sums);
        adj_seed_scale_kernel<<<dim3(64, B), 256, 0, st>>>(B, A->P, sums, (double*)rwork, loss);
        adj_seed_b_kernel<KIND><<<g, blk, 0, st>>>(tv, (const double*)rwork, (double*)ubar,
                                                   (double*)vbar);
    });
    if (e != cudaSuccess) rc = fail(RG_ECUDA, "adjoint seed launch: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaFreeAsync(part, st));
    CUDA_TRY(cudaFreeAsync(sums, st));
    return rc;
}

int rg_unroll_adjoint_step(const rg_op* A, const rg_op* At, const rg_sched* s, int i,
                           const void* f, const void* u_k, const void* v_k, void* ubar,
                           void* vbar, void* rbar, double* dots, void* stream) {
    int rc = check_adj_ops(A, At);
    if (rc) return rc;
    if ((rc = check_sched(A, s))) return rc;
    if (i < 0 || i >= s->m) return fail(RG_EINVAL, "inner index %d outside [0, %d)", i, s->m);
    if (!f || !u_k || !v_k || !ubar || !vbar || !rbar || !dots) return fail(RG_ENULL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const dim3 g = step_grid(A), blk(STEP_BX, STEP_BY);
    const int ncta = g.x * g.y, B = A->d.batch;
    AdjArgs a;
    a.A = view<double>(A);
    a.At = view<double>(At);
    a.f = (const double*)f;
    a.u = (const double*)u_k;
    a.v = (const double*)v_k;
    a.ubar = (double*)ubar;
    a.vbar = (double*)vbar;
    a.rbar = (double*)rbar;
    a.omega = s->omega;
    a.alpha = s->variant == RG_PLAIN ? nullptr : s->alpha;
    a.atil = s->alpha_tilde;
    a.scale = (const double*)s->scale;
    a.precond = s->precond;
    a.m = s->m;
    a.i = i;
    a.nag = s->variant >= RG_NAG;
    ensure_pool();
    CUDA_TRY(cudaMallocAsync((void**)&a.part, sizeof(double) * 3 * B * ncta, st));
    cudaError_t e = by_kind(A->d.kind, [&](auto kk) {
        constexpr int KIND = decltype(kk)::value;
        adj_a_kernel<KIND><<<g, blk, 0, st>>>(a);
        adj_b_kernel<KIND><<<g, blk, 0, st>>>(a);
        sum_partials_kernel<256><<<3 * B, 256, 0, st>>>(a.part, ncta, dots);
    });
    if (e != cudaSuccess) rc = fail(RG_ECUDA, "adjoint step launch: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaFreeAsync(a.part, st));
    return rc;
}

int rg_unroll_adjoint_step_ext(const rg_op* A, const rg_op* At, const rg_sched* s, int i,
                               const void* v_k, const void* p_k, void* ubar, void* vbar,
                               void* rbar_pre, void* rbar, double* dots, int phase, void* stream) {
    int rc = check_adj_ops(A, At);
    if (rc) return rc;
    if ((rc = check_sched(A, s))) return rc;
    if (i < 0 || i >= s->m) return fail(RG_EINVAL, "inner index %d outside [0, %d)", i, s->m);
    if (phase != 1 && phase != 2) return fail(RG_EINVAL, "phase must be 1 or 2");
    if (!v_k || !ubar || !vbar || !dots || (phase == 1 && (!p_k || !rbar_pre)) || (phase == 2 && !rbar))
        return fail(RG_ENULL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const dim3 g = step_grid(A), blk(STEP_BX, STEP_BY);
    const int ncta = g.x * g.y, B = A->d.batch;
    AdjArgs a;
    memset(&a, 0, sizeof a);
    a.A = view<double>(A);
    a.At = view<double>(At);
    a.v = (const double*)v_k;
    a.pk = (const double*)p_k;
    a.ubar = (double*)ubar;
    a.vbar = (double*)vbar;
    a.rbar = (double*)rbar;
    a.rbar_pre = (double*)rbar_pre;
    a.omega = s->omega;
    a.alpha = s->variant == RG_PLAIN ? nullptr : s->alpha;
    a.atil = s->alpha_tilde;
    a.m = s->m;
    a.i = i;
    a.nag = s->variant >= RG_NAG;
    ensure_pool();
    CUDA_TRY(cudaMallocAsync((void**)&a.part, sizeof(double) * 3 * B * ncta, st));
    cudaError_t e;
    if (phase == 1) {
        adj_a_ext_kernel<<<g, blk, 0, st>>>(a);
        sum_partials_kernel<256><<<2 * B, 256, 0, st>>>(a.part, ncta, dots);
        e = cudaGetLastError();
    } else {
        e = by_kind(A->d.kind, [&](auto kk) {
            constexpr int KIND = decltype(kk)::value;
            adj_b_kernel<KIND><<<g, blk, 0, st>>>(a);
            sum_partials_kernel<256><<<B, 256, 0, st>>>(a.part + (size_t)2 * B * ncta, ncta, dots + 2 * B);
        });
    }
    if (e != cudaSuccess) rc = fail(RG_ECUDA, "adjoint step launch: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaFreeAsync(a.part, st));
    return rc;
}

int rg_sweep(const rg_op* A, const rg_sched* s, int i0, int n_steps, int block_T, void* u0,
             void* u1, void* v0, void* v1, const void* f, int* out_buf, void* stream) {
    return rg_sweep_from_zero(A, s, i0, n_steps, block_T, u0, u1, v0, v1, f, 0, out_buf, stream);
}

static int sweep_impl(const rg_op* A, const rg_sched* s, int i0, int n_steps, int block_T, void* u0,
                      void* u1, void* v0, void* v1, const void* f, int zero_mask, double* norm2_first,
                      int* out_buf, void* stream);

int rg_sweep_from_zero(const rg_op* A, const rg_sched* s, int i0, int n_steps, int block_T, void* u0,
                       void* u1, void* v0, void* v1, const void* f, int zero_mask, int* out_buf,
                       void* stream) {
    return sweep_impl(A, s, i0, n_steps, block_T, u0, u1, v0, v1, f, zero_mask, nullptr, out_buf, stream);
}

int rg_sweep_norm(const rg_op* A, const rg_sched* s, int i0, int n_steps, int block_T, void* u0,
                  void* u1, void* v0, void* v1, const void* f, double* norm2_first, int* out_buf,
                  void* stream) {
    if (!norm2_first) return fail(RG_ENULL, "null norm output");
    return sweep_impl(A, s, i0, n_steps, block_T, u0, u1, v0, v1, f, 0, norm2_first, out_buf, stream);
}

static int sweep_impl(const rg_op* A, const rg_sched* s, int i0, int n_steps, int block_T, void* u0,
                      void* u1, void* v0, void* v1, const void* f, int zero_mask, double* norm2_first,
                      int* out_buf, void* stream) {
    int rc = check_op(A);
    if (rc) return rc;
    if ((rc = check_sched(A, s))) return rc;
    if (!u0 || !u1 || !f || !out_buf) return fail(RG_ENULL, "null argument");
    if (s->variant != RG_PLAIN && (!v0 || !v1)) return fail(RG_ENULL, "variant needs v0/v1");
    if (n_steps < 0 || i0 < 0) return fail(RG_EINVAL, "negative step count or index");
    if (block_T < 0 || block_T > 8) return fail(RG_EINVAL, "block_T must be in [0, 8]");
    cudaStream_t st = (cudaStream_t)stream;
    void* u[2] = {u0, u1};
    void* v[2] = {v0, v1};
    int cur = 0;
    const bool real = A->d.dtype == RG_F32 || A->d.dtype == RG_F64;
    const bool blocked = real && A->d.kind == RG_CONST9 &&
                         s->precond != RG_PRECOND_JACOBI_FIELD && block_T != 1;
    // complex 5-point Helmholtz smoother (V-cycle fine level): blocked sweep
    const bool cblocked = !blocked && A->cblock_ok && s->precond == RG_PRECOND_NONE && block_T != 1;
    // (side >= 200: with 16 x 64 windows, 16 steps at 255^2 take 129 us
    // against 203 us with one-step launches; at 127^2 the resident cluster
    // sweep is faster, 46 against 71 us)
    const bool cblocked9 = !blocked && A->var9h && s->precond == RG_PRECOND_NONE &&
                           block_T != 1 && (block_T > 1 || A->d.side >= cb9_min_side());
    // zero_mask: the blocked complex sweeps skip reading an all-zero u / v in
    // their first launch; every other path gets the zeros written
    if (zero_mask & ~3) return fail(RG_EINVAL, "bad zero mask %d", zero_mask);
    int zero_in = zero_mask;
    if (zero_mask && !((cblocked || cblocked9) && n_steps > 0)) {
        const size_t bytes = (size_t)A->d.batch * A->P *
                             (A->d.dtype == RG_C128 ? 16 : (A->d.dtype == RG_F64 ? 8 : 4));
        if ((zero_mask & 1) && v0) CUDA_TRY(cudaMemsetAsync(v0, 0, bytes, st));
        if (zero_mask & 2) CUDA_TRY(cudaMemsetAsync(u0, 0, bytes, st));
        zero_in = 0;
    }
    std::vector<double> hscale;
    const bool jac = s->precond == RG_PRECOND_JACOBI_SCALAR;
    if (blocked && jac) {
        const int B = A->d.batch;
        hscale.resize(B);
        CUDA_TRY(cudaMemcpyAsync(hscale.data(), s->scale, B * sizeof(double), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    // plain sweeps of enough systems: wavefront strips at depth 4 (as the
    // solver engine chooses them, rg_solver_create)
    const int wave_L = (blocked && s->variant == RG_PLAIN && A->d.side >= WV_MIN_SIDE && wave_enabled() &&
                        block_T == 0)
                           ? wave_seg_rows(A->d.side, A->d.batch)
                           : 0;
    const int T = block_T == 0 ? (wave_L > 0 ? env_int("RG_WAVE_T", 4) : 5) : block_T;
    // ||f - A u0||^2 per system: the first wavefront launch computes that
    // residual anyway and reduces its norm in the fused epilogue (stateless
    // mode); every other path takes a residual pass first
    const bool norm_fused = norm2_first && wave_L > 0 && n_steps > 0 && A->d.dtype == RG_F64 &&
                            chunk_len(n_steps, T, 0) <= WV_TMAX;
    if (norm2_first && !norm_fused) {
        if ((rc = rg_residual(A, u0, f, nullptr, norm2_first, stream))) return rc;
    }
    int k = i0;
    int left = n_steps;
    // automatic depth of the complex blocked sweeps: 4 for the 32-row 5-point
    // windows, 3 for the 16-row Galerkin windows (511^2: 305 us per 16-step
    // call at T=3 against 373 at T=4, 304 at T=2); RG_CB_T / RG_CB9_T override
    int TC = block_T == 0 ? (cblocked9 ? 3 : 4) : (block_T < 4 ? block_T : 4);
    if (block_T == 0) {
        if (const char* ev = getenv(cblocked9 ? "RG_CB9_T" : "RG_CB_T"))
            TC = atoi(ev) < 1 ? 1 : (atoi(ev) > 4 ? 4 : atoi(ev));
    }
    // small grids (coarse V-cycle levels): every step in one cluster launch
    // with the stencil input resident in distributed shared memory
    // (psweep.cuh; up to 16 x 1024 unknowns per system)
    int cs_nc = 0;
    csweep_shape(A->d.side, CS_NT_BIG, &cs_nc);
    const bool small = !blocked && !cblocked && !cblocked9 && block_T == 0 && n_steps >= 2 &&
                       (A->d.dtype == RG_F64 || A->d.dtype == RG_C128) && cs_nc > 0;
    if (small) {
        cudaError_t err;
        if (A->d.dtype == RG_F64) {
            PsArgs<double> pa;
            pa.A = view<double>(A);
            pa.u = (double*)u[0];
            pa.v = (double*)v[0];
            pa.f = (const double*)f;
            pa.omega = s->omega;
            pa.alpha = s->alpha;
            pa.atil = s->alpha_tilde;
            pa.scale = (const double*)s->scale;
            pa.precond = s->precond;
            pa.m = s->m;
            pa.k0 = i0;
            pa.n_steps = n_steps;
            pa.B = A->d.batch;
            err = launch_psweep(pa, A->d.kind, s->variant, st);
        } else {
            PsArgs<double2> pa;
            pa.A = view<double2>(A);
            pa.u = (double2*)u[0];
            pa.v = (double2*)v[0];
            pa.f = (const double2*)f;
            pa.omega = s->omega;
            pa.alpha = s->alpha;
            pa.atil = s->alpha_tilde;
            pa.scale = (const double2*)s->scale;
            pa.precond = s->precond;
            pa.m = s->m;
            pa.k0 = i0;
            pa.n_steps = n_steps;
            pa.B = A->d.batch;
            err = launch_psweep(pa, A->d.kind, s->variant, st);
        }
        if (err != cudaSuccess) return fail(RG_ECUDA, "small-grid sweep launch: %s", cudaGetErrorString(err));
        *out_buf = 0;
        return RG_OK;
    }
    while (left > 0) {
        const int t = blocked ? chunk_len(n_steps, T, n_steps - left)
                              : ((cblocked || cblocked9) ? chunk_cap(n_steps, TC, n_steps - left) : 1);
        if (cblocked9) {
            CBlock9Args ca;
            for (int q = 0; q < 9; ++q) ca.c9[q] = A->hc9[q];
            ca.planes = (const double2*)A->d.stencil;
            ca.mask = A->mask;
            ca.side = A->d.side;
            ca.P = A->P;
            ca.u_in = (const double2*)u[cur];
            ca.u_out = (double2*)u[cur ^ 1];
            ca.v_in = (const double2*)v[cur];
            ca.v_out = (double2*)v[cur ^ 1];
            ca.f = (const double2*)f;
            ca.omega = s->omega;
            ca.alpha = s->alpha;
            ca.atil = s->alpha_tilde;
            ca.m = s->m;
            ca.k0 = k;
            ca.zero_in = left == n_steps ? zero_in : 0;
            cudaError_t err;
            switch (s->variant) {
                case RG_PLAIN: err = launch_cblock9<V_PLAIN>(ca, t, A->d.batch, st); break;
                case RG_MOM: err = launch_cblock9<V_MOM>(ca, t, A->d.batch, st); break;
                default: err = launch_cblock9<V_NAG>(ca, t, A->d.batch, st); break;
            }
            rc = err == cudaSuccess ? RG_OK : fail(RG_ECUDA, "complex 9-point sweep launch: %s", cudaGetErrorString(err));
        } else if (cblocked) {
            CBlockArgs ca;
            for (int q = 0; q < 4; ++q) ca.off[q] = A->hoff[q];
            ca.diag = (const double2*)A->d.diag;
            ca.diag_shared = A->d.shared;
            ca.side = A->d.side;
            ca.P = A->P;
            ca.u_in = (const double2*)u[cur];
            ca.u_out = (double2*)u[cur ^ 1];
            ca.v_in = (const double2*)v[cur];
            ca.v_out = (double2*)v[cur ^ 1];
            ca.f = (const double2*)f;
            ca.omega = s->omega;
            ca.alpha = s->alpha;
            ca.atil = s->alpha_tilde;
            ca.m = s->m;
            ca.k0 = k;
            ca.zero_in = left == n_steps ? zero_in : 0;
            cudaError_t err;
            switch (s->variant) {
                case RG_PLAIN: err = launch_cblock<V_PLAIN>(ca, t, A->d.batch, st); break;
                case RG_MOM: err = launch_cblock<V_MOM>(ca, t, A->d.batch, st); break;
                default: err = launch_cblock<V_NAG>(ca, t, A->d.batch, st); break;
            }
            rc = err == cudaSuccess ? RG_OK : fail(RG_ECUDA, "complex sweep launch: %s", cudaGetErrorString(err));
        } else if (blocked && wave_L > 0 && t <= WV_TMAX) {
            if (norm_fused && left == n_steps) {
                const int ncta = wave_ntiles(A->d.side, t, wave_L, nullptr);
                const int B = A->d.batch;
                char* ws = nullptr;
                const size_t pbytes = sizeof(double) * (size_t)B * NSLOT * ncta;
                ensure_pool();
                CUDA_TRY(cudaMallocAsync((void**)&ws, pbytes + sizeof(int) * B, st));
                CUDA_TRY(cudaMemsetAsync(ws + pbytes, 0, sizeof(int) * B, st));
                EpiArgs e = {};
                e.partials = (double*)ws;
                e.ncta_cap = ncta;
                e.nslots = 1;
                e.counters = (int*)(ws + pbytes);
                e.norm_out = norm2_first;
                rc = sweep_wave<double>(A, s, k, t, wave_L, jac, hscale, u[cur], u[cur ^ 1], f, st, &e);
                CUDA_TRY(cudaFreeAsync(ws, st));
            } else {
                rc = A->d.dtype == RG_F64
                         ? sweep_wave<double>(A, s, k, t, wave_L, jac, hscale, u[cur], u[cur ^ 1], f, st)
                         : sweep_wave<float>(A, s, k, t, wave_L, jac, hscale, u[cur], u[cur ^ 1], f, st);
            }
        } else if (blocked) {
            rc = A->d.dtype == RG_F64
                     ? sweep_block<double>(A, s, k, t, jac, hscale, u[cur], u[cur ^ 1], v[cur], v[cur ^ 1], f, st)
                     : sweep_block<float>(A, s, k, t, jac, hscale, u[cur], u[cur ^ 1], v[cur], v[cur ^ 1], f, st);
        } else {
            StepReq q;
            memset(&q, 0, sizeof q);
            q.u_in = u[cur];
            q.u_out = u[cur ^ 1];
            q.v_in = v[cur];
            q.v_out = v[cur ^ 1];
            q.f = f;
            q.omega = s->omega;
            q.alpha = s->alpha;
            q.atil = s->alpha_tilde;
            q.scale = s->scale;
            q.m = s->m;
            q.i = k % s->m;
            q.variant = s->variant;
            q.precond = s->precond;
            q.update = 1;
            rc = step1(A, q, st);
        }
        if (rc) return rc;
        cur ^= 1;
        k += t;
        left -= t;
    }
    *out_buf = cur;
    return RG_OK;
}

int rg_dst_create(rg_dst** out, int batch, int side) {
    if (!out) return fail(RG_ENULL, "null out");
    const int M = side + 1;
    if (batch < 1 || side < 1) return fail(RG_EINVAL, "DST needs batch >= 1 and side >= 1");
    if ((M & (M - 1)) != 0 || M < 4 || M > 8192) {
        // any other size: dense sine-matrix products (S X S)
        if (side > 4096) return fail(RG_EUNSUPPORTED, "DST side %d: not a power of two minus one, "
                                     "and above the dense path's 4096", side);
        rg_dst* D = new rg_dst();
        D->batch = batch;
        D->side = side;
        D->M = M;
        D->dense = true;
        const size_t NN = (size_t)side * side;
        std::vector<double> S(NN);
        const double sc = sqrt(2.0 / M);
        for (int j = 0; j < side; ++j)
            for (int k = 0; k < side; ++k) {
                const long long a = ((long long)(j + 1) * (k + 1)) % (2LL * M);   // sin is 2M-periodic in a
                S[(size_t)j * side + k] = sc * sin(M_PI * (double)a / (double)M);
            }
        cudaError_t e;
        if ((e = cudaMalloc((void**)&D->S, sizeof(double) * NN)) != cudaSuccess ||
            (e = cudaMalloc((void**)&D->work, sizeof(double) * batch * NN)) != cudaSuccess ||
            (e = cudaMalloc((void**)&D->work2, sizeof(double) * batch * NN)) != cudaSuccess ||
            (e = cudaMemcpy(D->S, S.data(), sizeof(double) * NN, cudaMemcpyHostToDevice)) != cudaSuccess) {
            cudaFree(D->S);
            cudaFree(D->work);
            cudaFree(D->work2);
            delete D;
            return fail(RG_ECUDA, "dst plan: %s", cudaGetErrorString(e));
        }
        *out = D;
        return RG_OK;
    }
    rg_dst* D = new rg_dst();
    D->batch = batch;
    D->side = side;
    D->M = M;
    D->logM = 0;
    while ((1 << D->logM) < M) ++D->logM;
    // lines per CTA: <= 256 threads (M / dst_vpt(M) per line; 512 for M = 8192)
    const int tpl = M / dst_vpt(M);
    int lpc = 256 / tpl;
    if (const char* ev = getenv("RG_DST_LPC")) lpc = atoi(ev);   // tuning override
    if (lpc * tpl > 256) lpc = 256 / tpl;
    if (lpc < 1) lpc = 1;
    while (lpc & (lpc - 1)) lpc &= lpc - 1;   // a power of two (index shifts in the kernel)
    D->lpc = lpc;
    std::vector<double2> tw(M);
    for (int k = 0; k < M; ++k) {
        // (cos, sin)(pi k / M), symmetric evaluation for accuracy
        const double ang = M_PI * (double)k / (double)M;
        tw[k] = make_double2(cos(ang), sin(ang));
    }
    D->lean = dstw_supported(M) && env_int("RG_DSTW", 1) != 0;
    cudaError_t e;
    if ((e = cudaMalloc((void**)&D->tw, sizeof(double2) * M)) != cudaSuccess ||
        (e = cudaMalloc((void**)&D->work, sizeof(double) * (size_t)batch * side * side)) != cudaSuccess ||
        (D->lean && ((e = cudaMalloc((void**)&D->wpad, sizeof(double) * (size_t)batch * M * M)) != cudaSuccess ||
                     (e = cudaMemset(D->wpad, 0, sizeof(double) * (size_t)batch * M * M)) != cudaSuccess)) ||
        (e = cudaMemcpy(D->tw, tw.data(), sizeof(double2) * M, cudaMemcpyHostToDevice)) != cudaSuccess) {
        cudaFree(D->tw);
        cudaFree(D->work);
        cudaFree(D->work2);
        cudaFree(D->wpad);
        delete D;
        return fail(RG_ECUDA, "dst plan: %s", cudaGetErrorString(e));
    }
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&D->num_sms, cudaDevAttrMultiProcessorCount, dev);
    *out = D;
    return RG_OK;
}

int rg_dst_destroy(rg_dst* D) {
    if (!D) return RG_OK;
    cudaFree(D->tw);
    cudaFree(D->work);
    cudaFree(D->S);
    cudaFree(D->work2);
    cudaFree(D->wpad);
    delete D;
    return RG_OK;
}

int rg_dst2(const rg_dst* D, const double* in, double* out, void* stream) {
    if (!D || !in || !out) return fail(RG_ENULL, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    if (D->dense) {   // out = S (in S)
        int rc = dst_gemm(D, in, true, D->S, false, D->work2, GEMM_STORE, nullptr, st);
        if (rc) return rc;
        return dst_gemm(D, D->S, false, D->work2, true, out, GEMM_STORE, nullptr, st);
    }
    if (D->lean) {   // rows into the padded intermediate, columns out of it
        int rc = dstw_pass(D, false, DSTW_PLAIN, in, false, D->wpad, true, nullptr, st);
        if (rc) return rc;
        return dstw_pass(D, true, DSTW_PLAIN, D->wpad, true, out, false, nullptr, st);
    }
    int rc = dst_pass(D, 0, DST_PLAIN, in, out, nullptr, st);
    if (rc) return rc;
    return dst_pass(D, 1, DST_PLAIN, out, out, nullptr, st);
}

// r = f - A u for a CONST9 float64 operator through the blocked kernel's
// residual-only T = 1 launch (64 x 64 windows staged in shared memory, the
// stencil as kernel parameters): ~2x the one-point-per-thread step1 kernel.
static int resid_const9(const rg_op* A, const double* u, const double* f, double* r, cudaStream_t st) {
    static thread_local BlockArgs<double> a;
    memset(&a.epi, 0, sizeof a.epi);
    a.side = A->d.side;
    a.P = A->P;
    a.u_in = u;
    a.v_in = nullptr;
    a.u_out = nullptr;
    a.v_out = nullptr;
    a.r_out = r;
    a.f = f;
    a.omega = a.alpha = a.atil = nullptr;
    a.m = 1;
    a.k0 = 0;
    a.norm_first_u = 0;
    a.norm_every = 0;
    block_ntiles(A->d.side, 1, &a.nty);
    const int B = A->d.batch;
    for (int b0 = 0; b0 < B; b0 += BLK_MAXB) {
        const int nsys = B - b0 < BLK_MAXB ? B - b0 : BLK_MAXB;
        a.b0 = b0;
        for (int j = 0; j < nsys; ++j) {
            for (int d = 0; d < 9; ++d) a.coef[j][d] = A->hcoef[(size_t)(b0 + j) * 9 + d];
            a.scale[j] = 0.0;
        }
        const cudaError_t err = launch_block<double, V_PLAIN>(a, 1, false, nsys, st);
        if (err != cudaSuccess) return fail(RG_ECUDA, "residual launch: %s", cudaGetErrorString(err));
    }
    return RG_OK;
}

int rg_fns_correct(const rg_op* A, const rg_dst* D, const double* lam, double* u, const double* f,
                   void* stream) {
    int rc = check_op(A);
    if (rc) return rc;
    if (!D || !lam || !u || !f) return fail(RG_ENULL, "null argument");
    if (A->d.dtype != RG_F64) return fail(RG_EUNSUPPORTED, "FNS correction is float64 (fns.py:36)");
    if (A->d.side != D->side || A->d.batch != D->batch) return fail(RG_ESIZE, "plan/operator shape mismatch");
    cudaStream_t st = (cudaStream_t)stream;
    // r = f - A u (a separate pass: measured faster than recomputing the
    // stencil inside the row transform's load)
    if (A->d.kind == RG_CONST9 && env_int("RG_RESID_TILED", 1)) {
        if ((rc = launch_resid9(A, u, f, D->work, nullptr, st))) return rc;
    } else if (A->d.kind == RG_CONST9 && !A->hcoef.empty()) {
        if ((rc = resid_const9(A, u, f, D->work, st))) return rc;
    } else {
        StepReq q;
        memset(&q, 0, sizeof q);
        q.u_in = u;
        q.f = f;
        q.r_out = D->work;
        q.m = 1;
        if ((rc = step1(A, q, st))) return rc;
    }
    if (D->dense) {   // u += S ((S (r S)) * lam) S
        if ((rc = dst_gemm(D, D->work, true, D->S, false, D->work2, GEMM_STORE, nullptr, st))) return rc;
        if ((rc = dst_gemm(D, D->S, false, D->work2, true, D->work, GEMM_LAM, lam, st))) return rc;
        if ((rc = dst_gemm(D, D->work, true, D->S, false, D->work2, GEMM_STORE, nullptr, st))) return rc;
        return dst_gemm(D, D->S, false, D->work2, true, u, GEMM_ADD, nullptr, st);
    }
    if (D->lean) {
        if ((rc = dstw_pass(D, false, DSTW_PLAIN, D->work, false, D->wpad, true, nullptr, st))) return rc;
        if ((rc = dstw_pass(D, true, DSTW_TWICE_LAM, D->wpad, true, D->wpad, true, lam, st))) return rc;
        return dstw_pass(D, false, DSTW_ADD, D->wpad, true, u, false, nullptr, st);
    }
    if ((rc = dst_pass(D, 0, DST_PLAIN, D->work, D->work, nullptr, st))) return rc;
    if ((rc = dst_pass(D, 1, DST_TWICE_LAM, D->work, D->work, lam, st))) return rc;
    return dst_pass(D, 0, DST_ADD, D->work, u, nullptr, st);
}

static int mg_dtype_ok(int dtype) { return dtype == RG_F64 || dtype == RG_C128 || dtype == RG_F32; }

int rg_restrict(int dtype, int batch, int n, const void* fine, void* coarse, void* stream) {
    if (!fine || !coarse) return fail(RG_ENULL, "null vector");
    if (!mg_dtype_ok(dtype)) return fail(RG_EINVAL, "bad dtype %d", dtype);
    if (n < 4 || (n & 1) || batch < 1) return fail(RG_ESIZE, "grid side %d must be even and >= 4", n);
    const int nf = n - 1, nc = n / 2 - 1;
    const dim3 g((nc + MG_BX - 1) / MG_BX, (nc + MG_BY - 1) / MG_BY, batch), blk(MG_BX, MG_BY);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == RG_F64) restrict_kernel<double><<<g, blk, 0, st>>>((const double*)fine, (double*)coarse, nf, nc);
    else if (dtype == RG_F32) restrict_kernel<float><<<g, blk, 0, st>>>((const float*)fine, (float*)coarse, nf, nc);
    else restrict_kernel<double2><<<g, blk, 0, st>>>((const double2*)fine, (double2*)coarse, nf, nc);
    LAUNCH_CHECK();
    return RG_OK;
}

int rg_prolong_add(int dtype, int batch, int n, const void* coarse, void* fine, void* stream) {
    if (!fine || !coarse) return fail(RG_ENULL, "null vector");
    if (!mg_dtype_ok(dtype)) return fail(RG_EINVAL, "bad dtype %d", dtype);
    if (n < 4 || (n & 1) || batch < 1) return fail(RG_ESIZE, "grid side %d must be even and >= 4", n);
    const int nf = n - 1, nc = n / 2 - 1;
    const dim3 g((nf + MG_BX - 1) / MG_BX, (nf + MG_BY - 1) / MG_BY, batch), blk(MG_BX, MG_BY);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == RG_F64) prolong_add_kernel<double><<<g, blk, 0, st>>>((const double*)coarse, (double*)fine, nf, nc);
    else if (dtype == RG_F32) prolong_add_kernel<float><<<g, blk, 0, st>>>((const float*)coarse, (float*)fine, nf, nc);
    else prolong_add_kernel<double2><<<g, blk, 0, st>>>((const double2*)coarse, (double2*)fine, nf, nc);
    LAUNCH_CHECK();
    return RG_OK;
}

int rg_dense_apply(int dtype, int batch, int n, const void* M, int shared, const void* x, void* y,
                   void* stream) {
    if (!M || !x || !y) return fail(RG_ENULL, "null argument");
    if (!mg_dtype_ok(dtype)) return fail(RG_EINVAL, "bad dtype %d", dtype);
    if (n < 1 || batch < 1) return fail(RG_ESIZE, "bad size");
    const dim3 g((n + 7) / 8, batch);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == RG_F64) dense_apply_kernel<double><<<g, 256, 0, st>>>((const double*)M, shared, (const double*)x, (double*)y, n);
    else if (dtype == RG_F32) dense_apply_kernel<float><<<g, 256, 0, st>>>((const float*)M, shared, (const float*)x, (float*)y, n);
    else dense_apply_kernel<double2><<<g, 256, 0, st>>>((const double2*)M, shared, (const double2*)x, (double2*)y, n);
    LAUNCH_CHECK();
    return RG_OK;
}

int rg_mgs_step(int dtype, int batch, int n, void* w, long long ldw, const void* v, long long ldv,
                const void* h, const void* vn, long long ldvn, void* hn, double* wnorm2,
                void* stream) {
    if (!w) return fail(RG_ENULL, "null w");
    if (dtype != RG_F64 && dtype != RG_C128) return fail(RG_EINVAL, "mgs: float64 or complex128");
    if (batch < 1 || n < 1) return fail(RG_ESIZE, "bad size");
    if (v && !h) return fail(RG_ENULL, "projection needs h");
    if (vn && !hn) return fail(RG_ENULL, "dot needs hn");
    cudaStream_t st = (cudaStream_t)stream;
    int ncta = (n + MGS_NT * 4 - 1) / (MGS_NT * 4);
    if (ncta > 512) ncta = 512;
    double* part = nullptr;
    ensure_pool();
    CUDA_TRY(cudaMallocAsync((void**)&part, sizeof(double) * 3 * ncta * batch, st));
    const dim3 g(ncta, batch);
    if (dtype == RG_F64) {
        MgsArgs<double> a{(double*)w, ldw, (const double*)v, ldv, (const double*)h,
                          (const double*)vn, ldvn, part, n, wnorm2 != nullptr,
                          nullptr, nullptr, nullptr};
        mgs_kernel<double><<<g, MGS_NT, 0, st>>>(a);
        mgs_finish_kernel<double><<<batch, MGS_NT, 0, st>>>(part, ncta, (double*)hn, wnorm2);
    } else {
        MgsArgs<double2> a{(double2*)w, ldw, (const double2*)v, ldv, (const double2*)h,
                           (const double2*)vn, ldvn, part, n, wnorm2 != nullptr,
                           nullptr, nullptr, nullptr};
        mgs_kernel<double2><<<g, MGS_NT, 0, st>>>(a);
        mgs_finish_kernel<double2><<<batch, MGS_NT, 0, st>>>(part, ncta, (double2*)hn, wnorm2);
    }
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(part, st);
    if (e != cudaSuccess) return fail(RG_ECUDA, "mgs launch: %s", cudaGetErrorString(e));
    return RG_OK;
}

}  // extern "C"

// Whole MGS orthogonalisation (fgmres.py:76-78): k + 2 fused passes per
// system.  Systems are processed in chunks small enough that a chunk's w
// plus the two basis vectors a pass touches stay resident in L2 (126 MB),
// so a pass streams only the next basis vector from HBM; each pass is ONE
// launch (the partial sums are finished by the last CTA of each system).
// Persistent single-launch MGS when a CTA per SM can hold its slices of w
// and of the basis vector in shared memory (cooperative launch for
// guaranteed co-residency); returns -1 when it does not apply.
template <typename S>
static int mgs_persist(int batch, int n, S* w, long long ldw, const S* V, long long ldv, int k,
                       S* H, double* wnorm2, cudaStream_t st) {
    if (env_int("RG_MGS_PERSIST", 1) == 0) return -1;
    int dev = 0, nsm = 0, coop = 0, smem_optin = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (!coop || nsm < 1) return -1;
    const int slice = (n + nsm - 1) / nsm;
    const size_t smem = 2 * (size_t)slice * sizeof(S);
    if (smem + 2048 > (size_t)smem_optin || slice > MGSP_NT * MGSP_R) return -1;   // 1.6 KB static
    // fewest slice elements per thread that cover the slice (registers)
    const void* kern = slice <= MGSP_NT * 12 ? (const void*)mgs_persist_kernel<S, 12>
                       : slice <= MGSP_NT * 14 ? (const void*)mgs_persist_kernel<S, 14>
                                               : (const void*)mgs_persist_kernel<S, 16>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem_optin - 2048)) !=
        cudaSuccess)
        return -1;
    char* ws = nullptr;
    const size_t part_bytes = sizeof(double) * MGSP_NV * 2 * (size_t)nsm;   // two parities
    ensure_pool();
    if (cudaMallocAsync((void**)&ws, part_bytes + 2 * sizeof(unsigned int), st) != cudaSuccess) return -1;
    unsigned int* cnt = (unsigned int*)(ws + part_bytes);
    if (cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned int), st) != cudaSuccess) return -1;
    MgsPArgs<S> a;
    a.w = w; a.ldw = ldw; a.V = V; a.ldv = ldv; a.H = H; a.wnorm2 = wnorm2;
    a.part = (double*)ws; a.bar.count = cnt; a.bar.gen = cnt + 1;
    a.n = n; a.k = k; a.B = batch; a.slice = slice;
    void* args[] = {&a};
    cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(nsm),
                                                dim3(MGSP_NT), args, smem, st);
    cudaFreeAsync(ws, st);
    if (e != cudaSuccess) {        // e.g. co-residency refused: take the multi-launch path
        cudaGetLastError();
        return -1;
    }
    return RG_OK;
}

template <typename S>
static int mgs_arnoldi_t(int batch, int n, S* w, long long ldw, const S* V, long long ldv, int k,
                         S* H, double* wnorm2, cudaStream_t st) {
    {
        const int rc = mgs_persist<S>(batch, n, w, ldw, V, ldv, k, H, wnorm2, st);
        if (rc != -1) return rc;
    }
    int ncta = (n + MGS_NT * 4 - 1) / (MGS_NT * 4);
    if (ncta > 1024) ncta = 1024;
    const double L2_BUDGET = (double)env_int("RG_MGS_L2MB", 96) * 1024 * 1024;
    int chunk = (int)(L2_BUDGET / (3.0 * (double)n * sizeof(S)));
    if (chunk < 1) chunk = 1;
    if (chunk > batch) chunk = batch;
    char* ws = nullptr;
    const size_t part_bytes = sizeof(double) * 3 * (size_t)ncta * batch;
    ensure_pool();
    CUDA_TRY(cudaMallocAsync((void**)&ws, part_bytes + sizeof(int) * batch, st));
    int* counter = (int*)(ws + part_bytes);
    CUDA_TRY(cudaMemsetAsync(counter, 0, sizeof(int) * batch, st));
    auto vi = [&](int i) { return V + (size_t)i * n; };
    auto hi = [&](int i) { return H + (size_t)i * batch; };
    for (int b0 = 0; b0 < batch; b0 += chunk) {
        const int nb = batch - b0 < chunk ? batch - b0 : chunk;
        const dim3 g(ncta, nb);
        for (int i = 0; i <= k + 1; ++i) {
            // pass i: w -= h_{i-1} v_{i-1} ; h_i = <v_i, w>  (last pass: ||w||^2)
            const bool last = i == k + 1;
            MgsArgs<S> a{w + b0 * ldw, ldw,
                         i ? vi(i - 1) + b0 * ldv : nullptr, ldv,
                         i ? hi(i - 1) + b0 : nullptr,
                         last ? nullptr : vi(i) + b0 * ldv, ldv,
                         (double*)ws + (size_t)3 * ncta * b0, n, last ? 1 : 0,
                         counter + b0, last ? nullptr : hi(i) + b0, last ? wnorm2 + b0 : nullptr};
            mgs_kernel<S><<<g, MGS_NT, 0, st>>>(a);
        }
    }
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(ws, st);
    if (e != cudaSuccess) return fail(RG_ECUDA, "mgs launch: %s", cudaGetErrorString(e));
    return RG_OK;
}

extern "C" {

int rg_mgs_arnoldi(int dtype, int batch, int n, void* w, long long ldw, const void* V, long long ldv,
                   int k, void* H, double* wnorm2, void* stream) {
    if (!w || !V || !H || !wnorm2) return fail(RG_ENULL, "null argument");
    if (k < 0) return fail(RG_EINVAL, "k must be >= 0");
    if (dtype != RG_F64 && dtype != RG_C128) return fail(RG_EINVAL, "mgs: float64 or complex128");
    if (batch < 1 || n < 1) return fail(RG_ESIZE, "bad size");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == RG_F64)
        return mgs_arnoldi_t<double>(batch, n, (double*)w, ldw, (const double*)V, ldv, k, (double*)H,
                                     wnorm2, st);
    return mgs_arnoldi_t<double2>(batch, n, (double2*)w, ldw, (const double2*)V, ldv, k, (double2*)H,
                                  wnorm2, st);
}

int rg_arnoldi_tail(int dtype, int batch, int n, const void* w, long long ldw, void* vnext,
                    long long ldv, const void* H, int k, const double* wnorm2, void* hcol,
                    void* stream) {
    if (!w || !vnext || !H || !wnorm2 || !hcol) return fail(RG_ENULL, "null argument");
    if (dtype != RG_F64 && dtype != RG_C128) return fail(RG_EINVAL, "arnoldi: float64 or complex128");
    if (batch < 1 || n < 1 || k < 0) return fail(RG_ESIZE, "bad size");
    cudaStream_t st = (cudaStream_t)stream;
    int nx = (n + MGS_NT * 4 - 1) / (MGS_NT * 4);
    if (nx > 256) nx = 256;
    const dim3 g(nx, batch);
    if (dtype == RG_F64)
        arnoldi_tail_kernel<double><<<g, MGS_NT, 0, st>>>((const double*)w, ldw, (double*)vnext,
                                                          ldv, (const double*)H, k, wnorm2,
                                                          (double*)hcol, n);
    else
        arnoldi_tail_kernel<double2><<<g, MGS_NT, 0, st>>>((const double2*)w, ldw, (double2*)vnext,
                                                           ldv, (const double2*)H, k, wnorm2,
                                                           (double2*)hcol, n);
    LAUNCH_CHECK();
    return RG_OK;
}

int rg_krylov_update(int dtype, int n, void* u, const void* Z, long long ldz, const void* y, int k,
                     void* stream) {
    if (!u || (k > 0 && (!Z || !y))) return fail(RG_ENULL, "null argument");
    if (dtype != RG_F64 && dtype != RG_C128) return fail(RG_EINVAL, "update: float64 or complex128");
    if (k <= 0) return RG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int nx = (n + MGS_NT * 2 - 1) / (MGS_NT * 2);
    if (nx > 1184) nx = 1184;
    if (dtype == RG_F64)
        krylov_update_kernel<double><<<nx, MGS_NT, 0, st>>>((double*)u, (const double*)Z, ldz,
                                                            (const double*)y, k, n);
    else
        krylov_update_kernel<double2><<<nx, MGS_NT, 0, st>>>((double2*)u, (const double2*)Z, ldz,
                                                             (const double2*)y, k, n);
    LAUNCH_CHECK();
    return RG_OK;
}

int rg_solver_create(rg_solver** out, const rg_op* A, const rg_sched* s, double tol,
                     int max_outer, int check, int block_T) {
    if (!out) return fail(RG_ENULL, "null out");
    int rc = check_op(A);
    if (rc) return rc;
    if ((rc = check_sched(A, s))) return rc;
    if (!(tol > 0)) return fail(RG_EINVAL, "tol must be positive");
    if (check != RG_CHECK_OUTER && check != RG_CHECK_INNER)
        return fail(RG_EINVAL, "check must be 'outer' or 'inner'");
    if (max_outer < 0) return fail(RG_EINVAL, "max_outer must be >= 0");
    if ((long long)max_outer * s->m > 2000000000ll) return fail(RG_ESIZE, "max_outer*m too large");
    if (block_T < 0 || block_T > 8) return fail(RG_EINVAL, "block_T must be in [0, 8]");
    rg_solver* S = new rg_solver();
    S->A = A;
    S->s = *s;
    S->cfg.tol = tol;
    S->cfg.div_factor = 1e12;
    S->cfg.m = s->m;
    S->cfg.max_outer = max_outer;
    S->cfg.check_inner = check == RG_CHECK_INNER;
    S->check = check;
    const bool real = A->d.dtype == RG_F32 || A->d.dtype == RG_F64;
    S->use_block = real && A->d.kind == RG_CONST9 && check == RG_CHECK_OUTER &&
                   s->precond != RG_PRECOND_JACOBI_FIELD && block_T != 1;
    S->wave_L = wave_seg_rows(A->d.side, A->d.batch);
    S->use_wave = S->use_block && s->variant == RG_PLAIN && A->d.side >= WV_MIN_SIDE &&
                  wave_enabled() && S->wave_L > 0;
    // automatic depth: measured optima on B200 (profiles/): 5 for the 64x64
    // overlapped tile, 4 for the wavefront strip
    S->block_T = block_T != 0 ? block_T : (S->use_wave ? env_int("RG_WAVE_T", 4) : 5);
    if (S->block_T > 8) S->block_T = 8;
    if (!S->use_block) S->block_T = 1;
    {
        // resident cluster solver: the whole solve in one launch when the grid
        // fits in the distributed shared memory of <= 16 CTAs
        int nc = 0, rows = 0, ppt = 0;
        cluster_shape(A->d.side, &nc, &rows, &ppt);
        const int v = s->variant >= RG_NAG ? V_NAG : s->variant;
        const size_t smem = nc == 0 ? 0 : (A->d.dtype == RG_F32 ? cluster_smem_bytes<float>(A->d.side, rows, v)
                                                                : cluster_smem_bytes<double>(A->d.side, rows, v));
        S->use_small = real && A->d.kind == RG_CONST9 && block_T == 0 && nc > 0 &&
                       s->precond != RG_PRECOND_JACOBI_FIELD && smem <= 200 * 1024;
        S->cl_nc = nc;
        S->cl_rows = rows;
        S->cl_ppt = ppt;
    }
    S->kmax = (long long)max_outer * s->m;
    const dim3 g = step_grid(A);
    int cap = g.x * g.y;
    for (int T = 1; T <= 8; ++T) {
        const int nt = block_ntiles(A->d.side, T, nullptr);
        if (nt > cap) cap = nt;
        if (S->use_wave && T <= WV_TMAX) {
            const int nw = wave_ntiles(A->d.side, T, S->wave_L, nullptr);
            if (nw > cap) cap = nw;
        }
    }
    S->ncta_cap = cap;
    S->trace_stride = max_outer + 1;
    const int B = A->d.batch;
    cudaError_t e;
    if ((e = cudaMalloc((void**)&S->d_st, sizeof(SysState) * B)) != cudaSuccess ||
        (e = cudaMalloc((void**)&S->d_trace, sizeof(double) * B * (size_t)S->trace_stride)) !=
            cudaSuccess ||
        (e = cudaMalloc((void**)&S->d_part, sizeof(double) * B * (size_t)NSLOT * cap)) !=
            cudaSuccess ||
        !(S->h_st = (SysState*)calloc(B, sizeof(SysState)))) {
        if (e == cudaSuccess) e = cudaErrorMemoryAllocation;
        cudaFree(S->d_st);
        cudaFree(S->d_trace);
        cudaFree(S->d_part);
        delete S;
        return fail(RG_ECUDA, "solver workspace: %s", cudaGetErrorString(e));
    }
    *out = S;
    return RG_OK;
}

int rg_solver_destroy(rg_solver* S) {
    if (!S) return RG_OK;
    cudaFree(S->d_st);
    cudaFree(S->d_trace);
    cudaFree(S->d_part);
    free(S->h_st);
    delete S;
    return RG_OK;
}

static EpiArgs solver_epi(rg_solver* S, int j0, int nslots, int with_f) {
    EpiArgs e = {};
    e.st = S->d_st;
    e.trace = S->d_trace;
    e.trace_stride = S->trace_stride;
    e.partials = S->d_part;
    e.ncta_cap = S->ncta_cap;
    e.cfg = S->cfg;
    e.j0 = j0;
    e.nslots = nslots;
    e.with_f = with_f;
    e.buf = S->cur;
    return e;
}

int rg_solver_begin(rg_solver* S, void* u0, void* u1, void* v0, void* v1, const void* f,
                    void* stream) {
    if (!S) return fail(RG_ENULL, "null solver");
    if (!u0 || !u1 || !f) return fail(RG_ENULL, "null vector");
    if (S->s.variant != RG_PLAIN && (!v0 || !v1)) return fail(RG_ENULL, "variant needs v0/v1");
    cudaStream_t st = (cudaStream_t)stream;
    const rg_op* A = S->A;
    const size_t vbytes = scalar_bytes(A->d.dtype) * (size_t)A->P * A->d.batch;
    S->u[0] = u0;
    S->u[1] = u1;
    S->v[0] = v0;
    S->v[1] = v1;
    S->f = f;
    S->k = 0;
    S->cur = 0;
    S->launches = 0;
    S->flushed_k = 0;
    S->need_flush = false;
    if (S->use_block && S->s.precond == RG_PRECOND_JACOBI_SCALAR) {
        // the blocked sweep takes the per-system Jacobi scale as a kernel parameter
        const int B = A->d.batch;
        S->hscale.resize(B);   // Jacobi scales are float64 for F64 and F32 operators
        CUDA_TRY(cudaMemcpyAsync(S->hscale.data(), S->s.scale, B * sizeof(double),
                                 cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    CUDA_TRY(cudaMemsetAsync(S->d_st, 0, sizeof(SysState) * A->d.batch, st));
    CUDA_TRY(cudaMemsetAsync(S->d_trace, 0, sizeof(double) * A->d.batch * (size_t)S->trace_stride, st));
    if (v0) CUDA_TRY(cudaMemsetAsync(v0, 0, vbytes, st));  // v = 0 at entry (:95)
    if (S->use_small) {   // the single-launch solver computes ||f|| and trace[0] itself
        S->small_done = false;
        S->begun = true;
        return RG_OK;
    }
    StepReq q;
    memset(&q, 0, sizeof q);
    q.u_in = u0;
    q.f = f;
    q.m = S->s.m;
    q.norm_u = 1;
    q.use_status = 0;
    q.epi = solver_epi(S, 0, 1, 1);
    int rc = step1(A, q, st);
    if (rc) return rc;
    S->begun = true;
    return RG_OK;
}

int rg_solver_step(rg_solver* S, void* stream, int* steps_out) {
    if (!S) return fail(RG_ENULL, "null solver");
    if (!S->begun) return fail(RG_ESTATE, "rg_solver_begin not called");
    if (steps_out) *steps_out = 0;
    if (S->use_small ? S->small_done : S->k >= S->kmax) return RG_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int m = S->s.m;
    if (S->use_small) {   // the whole solve (even max_outer = 0) in one launch
        const rg_op* A = S->A;
        cudaError_t err;
        auto fill = [&](auto& a) {
            a.coef = (const double*)A->d.stencil;
            a.scale = S->s.precond == RG_PRECOND_JACOBI_SCALAR ? (const double*)S->s.scale : nullptr;
            a.omega = S->s.omega; a.alpha = S->s.alpha; a.atil = S->s.alpha_tilde;
            a.side = A->d.side; a.P = A->P; a.m = m; a.shared = A->d.shared; a.cfg = S->cfg;
            a.nc = S->cl_nc; a.rows = S->cl_rows;
            a.st = S->d_st; a.trace = S->d_trace; a.trace_stride = S->trace_stride;
        };
        const int var = S->s.variant >= RG_NAG ? V_NAG : S->s.variant;
        const bool jac = S->s.precond == RG_PRECOND_JACOBI_SCALAR;
        if (A->d.dtype == RG_F64) {
            ClusterArgs<double> a;
            fill(a);
            a.u = (double*)S->u[0];
            a.f = (const double*)S->f;
            err = launch_cluster<double>(a, var, jac, S->cl_ppt, A->d.batch, st);
        } else {
            ClusterArgs<float> a;
            fill(a);
            a.u = (float*)S->u[0];
            a.f = (const float*)S->f;
            err = launch_cluster<float>(a, var, jac, S->cl_ppt, A->d.batch, st);
        }
        if (err != cudaSuccess) return fail(RG_ECUDA, "cluster solve launch: %s", cudaGetErrorString(err));
        if (steps_out) *steps_out = (int)(S->kmax - S->k);
        S->k = S->kmax;
        S->small_done = true;
        S->launches += 1;
        S->need_flush = false;
        return RG_OK;
    }
    const int i = (int)(S->k % m);
    const bool nag = S->s.variant >= RG_NAG;
    const bool boundary_norm = nag && i == 0 && S->k > 0 && S->flushed_k != S->k;
    int T = 1;
    int rc;
    if (S->use_block) {
        T = chunk_len(m, S->block_T, i);
        if (S->A->d.dtype == RG_F64) rc = do_block<double>(S, T, boundary_norm ? 1 : 0, st);
        else rc = do_block<float>(S, T, boundary_norm ? 1 : 0, st);
    } else {
        StepReq q;
        memset(&q, 0, sizeof q);
        q.u_in = S->u[S->cur];
        q.u_out = S->u[S->cur ^ 1];
        q.v_in = S->v[S->cur];
        q.v_out = S->v[S->cur ^ 1];
        q.f = S->f;
        q.omega = S->s.omega;
        q.alpha = S->s.alpha;
        q.atil = S->s.alpha_tilde;
        q.scale = S->s.scale;
        q.m = m;
        q.i = i;
        q.variant = S->s.variant;
        q.precond = S->s.precond;
        q.update = 1;
        q.norm_u = (!nag || S->cfg.check_inner || boundary_norm) ? 1 : 0;
        q.use_status = 1;
        q.epi = solver_epi(S, (int)S->k, q.norm_u, 0);
        rc = step1(S->A, q, st);
    }
    if (rc) return rc;
    S->cur ^= 1;
    S->k += T;
    S->launches += 1;
    S->need_flush = true;
    if (steps_out) *steps_out = T;
    return RG_OK;
}

int rg_solver_flush(rg_solver* S, void* stream) {
    if (!S) return fail(RG_ENULL, "null solver");
    if (!S->begun) return fail(RG_ESTATE, "rg_solver_begin not called");
    if (!S->need_flush) return RG_OK;
    S->need_flush = false;
    const int m = S->s.m;
    const bool nag = S->s.variant >= RG_NAG;
    if (nag && !S->cfg.check_inner && (S->k % m) != 0) return RG_OK;  // no test mid-sweep
    StepReq q;
    memset(&q, 0, sizeof q);
    q.u_in = S->u[S->cur];
    q.f = S->f;
    q.m = m;
    q.norm_u = 1;
    q.use_status = 1;
    q.epi = solver_epi(S, (int)S->k, 1, 0);
    int rc = step1(S->A, q, (cudaStream_t)stream);
    if (rc) return rc;
    S->flushed_k = S->k;
    return RG_OK;
}

int rg_solver_run(rg_solver* S, int n_sweeps, void* stream) {
    if (!S) return fail(RG_ENULL, "null solver");
    if (!S->begun) return fail(RG_ESTATE, "rg_solver_begin not called");
    if (n_sweeps < 1) return fail(RG_EINVAL, "n_sweeps must be >= 1");
    const long long m = S->s.m;
    long long target = (S->k / m + n_sweeps) * m;
    if (target > S->kmax) target = S->kmax;
    if (S->use_small) {
        int steps = 0;
        int rc = rg_solver_step(S, stream, &steps);
        if (rc) return rc;
        return RG_OK;
    }
    while (S->k < target) {
        int steps = 0;
        int rc = rg_solver_step(S, stream, &steps);
        if (rc) return rc;
        if (steps == 0) break;
    }
    return rg_solver_flush(S, stream);
}

int rg_solver_poll(rg_solver* S, void* stream, int* n_active, int* done) {
    if (!S) return fail(RG_ENULL, "null solver");
    cudaStream_t st = (cudaStream_t)stream;
    const int B = S->A->d.batch;
    CUDA_TRY(cudaMemcpyAsync(S->h_st, S->d_st, sizeof(SysState) * B, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    int act = 0;
    for (int b = 0; b < B; ++b) act += S->h_st[b].status == ST_ACTIVE;
    if (n_active) *n_active = act;
    if (done) *done = (act == 0) || (S->use_small ? S->small_done : (S->k >= S->kmax && !S->need_flush));
    return RG_OK;
}

int rg_solver_report(const rg_solver* S, int b, rg_report* out) {
    if (!S || !out) return fail(RG_ENULL, "null argument");
    if (b < 0 || b >= S->A->d.batch) return fail(RG_ESIZE, "system %d out of range", b);
    const SysState& s = S->h_st[b];
    out->status = s.status;
    out->iterations = s.outer;
    out->inner_iterations = s.inner;
    out->ans_buf = s.ans_buf;
    out->final_relative_residual = s.rel;
    out->trace0 = s.trace0;
    out->fnorm = s.fnorm;
    out->bad_rel = s.bad_rel;
    return RG_OK;
}

int rg_solver_trace(const rg_solver* S, int b, double* out, int cap, int* n_out) {
    if (!S || !out) return fail(RG_ENULL, "null argument");
    if (b < 0 || b >= S->A->d.batch) return fail(RG_ESIZE, "system %d out of range", b);
    int n = S->h_st[b].outer + 1;
    if (n > S->trace_stride) n = S->trace_stride;
    if (n > cap) n = cap;
    CUDA_TRY(cudaMemcpy(out, S->d_trace + (size_t)b * S->trace_stride, sizeof(double) * n,
                        cudaMemcpyDeviceToHost));
    if (n_out) *n_out = n;
    return RG_OK;
}

int rg_solver_plan(const rg_solver* S, int* kernel, int* block_T, int* seg_rows) {
    if (!S) return fail(RG_ENULL, "null solver");
    if (kernel)
        *kernel = S->use_small ? RG_KERNEL_CLUSTER
                  : !S->use_block ? RG_KERNEL_STEP
                  : (S->use_wave && S->block_T <= WV_TMAX) ? RG_KERNEL_WAVE : RG_KERNEL_TILE;
    if (block_T) *block_T = S->block_T;
    if (seg_rows) *seg_rows = S->use_wave ? S->wave_L : 0;
    return RG_OK;
}

int rg_solver_info(const rg_solver* S, long long* steps_queued, int* block_T, int* launches) {
    if (!S) return fail(RG_ENULL, "null solver");
    if (steps_queued) *steps_queued = S->k;
    if (block_T) *block_T = S->block_T;
    if (launches) *launches = S->launches;
    return RG_OK;
}

}  // extern "C"
