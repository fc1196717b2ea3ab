// h2_k_rows_f32.cu -- explicit instantiations (rows, float) of the launchers in h2_kernels.cuh
#include "h2_kernels.cuh"

namespace h2 {
#define T float
    template cudaError_t launch_rows<T>(int, const Task *, int, const Blk *, const T *, int64_t, T *, int64_t, int, int, cudaStream_t);
#undef T
}  // namespace h2
