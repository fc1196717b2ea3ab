// h2_k_a_f32.cu -- explicit instantiations (a, float) of the launchers in h2_kernels.cuh
#include "h2_kernels.cuh"

namespace h2 {
#define T float
    template cudaError_t launch_set_args<T>(CallArgs<T> *, const T *, int64_t, T *, int64_t, T, T, cudaStream_t);
    template cudaError_t launch_up_leaf<T>(const Task *, int, const Blk *, const CallArgs<T> *, T *, int64_t, int, int, cudaStream_t);
    template cudaError_t launch_scale<T>(T *, int64_t, int64_t, int, T, cudaStream_t);
    template cudaError_t launch_transpose<T>(const T *, T *, int64_t, int, int, cudaStream_t);
    template cudaError_t launch_pack<T>(const PackSeg *, int64_t, const T *, int64_t, const CallArgs<T> *, T *, int, cudaStream_t);
    template cudaError_t launch_sweep<T>(int, const SweepParams &, int, int, T *, int64_t, int, int, cudaStream_t);
    template cudaError_t launch_tree<T>(int, const TreeStage &, int, const Task *, const Blk *, T *, int64_t, int, int, cudaStream_t);
#undef T
}  // namespace h2
