// Instantiates the temporally blocked sweep for (double, nag); see block.cuh.
#include "block.cuh"
namespace rg {
template cudaError_t launch_block<double, V_NAG>(const BlockArgs<double>&, int, bool, int, cudaStream_t);
}
