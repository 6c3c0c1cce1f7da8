// Explicit instantiation of the cluster SOR/SSOR wavefront (parallel build); see tri.cuh.
#include "tri.cuh"
namespace rg {
template cudaError_t launch_tri<double>(const TriArgs<double>&, int, int, cudaStream_t);
template cudaError_t launch_tri<float>(const TriArgs<float>&, int, int, cudaStream_t);
}
