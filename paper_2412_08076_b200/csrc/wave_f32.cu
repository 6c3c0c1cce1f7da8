// Explicit instantiation of the wavefront sweep for float storage (parallel build).
#include "wave.cuh"
namespace rg {
template cudaError_t launch_wave<float>(const WaveArgs<float>&, int, bool, int, cudaStream_t);
}
