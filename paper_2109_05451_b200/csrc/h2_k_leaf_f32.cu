// h2_k_leaf_f32.cu -- explicit instantiations (leaf, float) of the launchers in h2_kernels.cuh
#include "h2_kernels.cuh"

namespace h2 {
#define T float
    template cudaError_t launch_leaf_dense<T>(const Task *, const Task *, int, const Blk *, const T *, int64_t, const CallArgs<T> *, const T *, int, int, int, int, cudaStream_t);
#undef T
}  // namespace h2
