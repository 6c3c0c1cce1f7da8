// Explicit instantiation of the general triangular wavefront (parallel build); see trigen.cuh.
#include "trigen.cuh"
namespace rg {
#define RG_TRIGEN_INST(S)                                                                         \
    template cudaError_t launch_trigen<S, K_CONST9>(const TriGenArgs<S>&, int, int, cudaStream_t); \
    template cudaError_t launch_trigen<S, K_DIAG5>(const TriGenArgs<S>&, int, int, cudaStream_t);  \
    template cudaError_t launch_trigen<S, K_VAR9>(const TriGenArgs<S>&, int, int, cudaStream_t);
RG_TRIGEN_INST(float)
RG_TRIGEN_INST(double)
RG_TRIGEN_INST(double2)
#undef RG_TRIGEN_INST
}
