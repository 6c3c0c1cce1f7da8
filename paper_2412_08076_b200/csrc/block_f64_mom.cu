// Instantiates the temporally blocked sweep for (double, mom); see block.cuh.
#include "block.cuh"
namespace rg {
template cudaError_t launch_block<double, V_MOM>(const BlockArgs<double>&, int, bool, int, cudaStream_t);
}
