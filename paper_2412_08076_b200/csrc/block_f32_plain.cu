// Instantiates the temporally blocked sweep for (float, plain); see block.cuh.
#include "block.cuh"
namespace rg {
template cudaError_t launch_block<float, V_PLAIN>(const BlockArgs<float>&, int, bool, int, cudaStream_t);
}
