// Explicit instantiation of the wavefront sweep for double storage (parallel build).
#include "wave.cuh"
namespace rg {
template cudaError_t launch_wave<double>(const WaveArgs<double>&, int, bool, int, cudaStream_t);
}
