// h2_k_rows_f64.cu -- explicit instantiations (rows, double) of the launchers in h2_kernels.cuh
#include "h2_kernels.cuh"

namespace h2 {
#define T double
    template cudaError_t launch_rows<T>(int, const Task *, int, const Blk *, const T *, int64_t, T *, int64_t, int, int, cudaStream_t);
#undef T
}  // namespace h2
