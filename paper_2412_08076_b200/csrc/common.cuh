// common.cuh — scalar arithmetic with the reference's exact rounding.
//
// The library is compiled with --fmad=false: every a*b+c below is a
// separate multiply and add, which is what SciPy's csr_matvec
// (sparsetools, compiled without FMA) and NumPy's elementwise ufuncs do
// (SURVEY.md Appendix A).  Only the norm accumulation, which the reference
// does in BLAS ddot and therefore cannot be matched bitwise anyway, uses an
// explicit fma().
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

namespace rg {

enum { DT_F32 = 1, DT_F64 = 2, DT_C128 = 3 };
enum { K_CONST9 = 1, K_DIAG5 = 2, K_VAR9 = 3 };
enum { V_PLAIN = 0, V_MOM = 1, V_NAG = 2, V_NAGEX = 3 };
enum { P_NONE = 0, P_JSCALAR = 1, P_JFIELD = 2 };
enum { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_DIVERGED = 2, ST_MAXED = 3 };

// ---- scalar ops: float, double, double2 (= complex128, (re, im)) ----------
template <typename S> struct Real { typedef S type; };
template <> struct Real<double2> { typedef double type; };

// Arithmetic type for a storage type: float32 vectors are computed in
// float64 (loaded -> widened, rounded once on store), so the f32 mode keeps
// f32 HBM traffic but the reference's float64 arithmetic; coefficients and
// Jacobi scales of an f32 operator are float64.
template <typename S> struct Compute { typedef S type; };
template <> struct Compute<float> { typedef double type; };
template <typename S> using CT = typename Compute<S>::type;

__device__ __forceinline__ double  to_c(float x)   { return (double)x; }
__device__ __forceinline__ double  to_c(double x)  { return x; }
__device__ __forceinline__ double2 to_c(double2 x) { return x; }
template <typename S> __device__ __forceinline__ S to_s(CT<S> x);
template <> __device__ __forceinline__ float   to_s<float>(double x)    { return (float)x; }
template <> __device__ __forceinline__ double  to_s<double>(double x)   { return x; }
template <> __device__ __forceinline__ double2 to_s<double2>(double2 x) { return x; }
// value as stored and reloaded: the rounding a state vector sees per step
template <typename S> __device__ __forceinline__ CT<S> stored(CT<S> x) { return to_c(to_s<S>(x)); }

__device__ __forceinline__ float   zero(float*)   { return 0.f; }
__device__ __forceinline__ double  zero(double*)  { return 0.0; }
__device__ __forceinline__ double2 zero(double2*) { return make_double2(0.0, 0.0); }
template <typename S> __device__ __forceinline__ S szero() { return zero((S*)nullptr); }

__device__ __forceinline__ float  add(float a, float b)   { return a + b; }
__device__ __forceinline__ double add(double a, double b) { return a + b; }
__device__ __forceinline__ double2 add(double2 a, double2 b) {
    return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ float  sub(float a, float b)   { return a - b; }
__device__ __forceinline__ double sub(double a, double b) { return a - b; }
__device__ __forceinline__ double2 sub(double2 a, double2 b) {
    return make_double2(a.x - b.x, a.y - b.y);
}
// scalar * scalar; complex product is the unfused textbook formula that
// SciPy's std::complex CSR kernel evaluates.
__device__ __forceinline__ float  mul(float a, float b)   { return a * b; }
__device__ __forceinline__ double mul(double a, double b) { return a * b; }
__device__ __forceinline__ double2 mul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// real scalar (float64 weight) * vector entry.  NumPy promotes the scalar
// to the array dtype first: float32 arrays see a float32 weight, complex
// arrays see (w + 0j) whose product is FMA-invariant and equals (w*re, w*im)
// for finite entries.
__device__ __forceinline__ float  rmul(double w, float x)  { return (float)w * x; }
__device__ __forceinline__ double rmul(double w, double x) { return w * x; }
__device__ __forceinline__ double2 rmul(double w, double2 x) {
    return make_double2(w * x.x, w * x.y);
}
__device__ __forceinline__ double sq(float x)   { return (double)x * (double)x; }
__device__ __forceinline__ double sq(double x)  { return x * x; }
__device__ __forceinline__ double sq(double2 x) { return fma(x.y, x.y, x.x * x.x); }
__device__ __forceinline__ double sqacc(double acc, float x)  { return fma((double)x, (double)x, acc); }
__device__ __forceinline__ double sqacc(double acc, double x) { return fma(x, x, acc); }
__device__ __forceinline__ double sqacc(double acc, double2 x) {
    return fma(x.y, x.y, fma(x.x, x.x, acc));
}
__device__ __forceinline__ float shfl_down(float v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ double shfl_down(double v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ double2 shfl_down(double2 v, int o) {
    return make_double2(__shfl_down_sync(0xffffffffu, v.x, o), __shfl_down_sync(0xffffffffu, v.y, o));
}
__device__ __forceinline__ bool finite(float x)   { return isfinite(x); }
__device__ __forceinline__ bool finite(double x)  { return isfinite(x); }
__device__ __forceinline__ bool finite(double2 x) { return isfinite(x.x) && isfinite(x.y); }

// ---- asynchronous global -> shared element copies (zero-filled when !valid)
template <int BYTES>
__device__ __forceinline__ void cp_async_el(void* sdst, const void* gsrc, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(sa), "l"(gsrc), "n"(BYTES),
                 "r"(valid ? BYTES : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- per-system solver state (device) ------------------------------------
// Mirrors the local variables of solve_stationary (richardson.py:92-136).
struct SysState {
    double fnorm;    // ||f||                       (:96)
    double trace0;   // trace[0]                    (:106-107)
    double rel;      // last relative residual      (:106,125)
    double bad_rel;  // rel that raised DivergenceError (:126-129)
    int status;      // ST_*
    int outer;       // outer sweeps completed      (:133)
    int inner;       // inner iterations            (:122)
    int ans_buf;     // ping-pong buffer holding the returned u
    int counter;     // last-CTA ticket for the fused reduction
    int last_j;      // last inner index whose residual was decided
    int pad[2];
};

struct SolveCfg {
    double tol;
    double div_factor;   // DIVERGENCE_FACTOR = 1e12 (richardson.py:17)
    int m;
    int max_outer;
    int check_inner;
};

}  // namespace rg
