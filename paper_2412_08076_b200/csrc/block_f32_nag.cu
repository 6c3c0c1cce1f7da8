// Instantiates the temporally blocked sweep for (float, nag); see block.cuh.
#include "block.cuh"
namespace rg {
template cudaError_t launch_block<float, V_NAG>(const BlockArgs<float>&, int, bool, int, cudaStream_t);
}
