// Instantiates the temporally blocked sweep for (double, plain); see block.cuh.
#include "block.cuh"
namespace rg {
template cudaError_t launch_block<double, V_PLAIN>(const BlockArgs<double>&, int, bool, int, cudaStream_t);
}
