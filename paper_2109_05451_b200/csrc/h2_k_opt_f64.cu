// h2_k_opt_f64.cu -- explicit instantiations (opt, double) of the launchers in h2_kernels.cuh
#include "h2_kernels.cuh"

namespace h2 {
#define T double
    template cudaError_t launch_mega_up<T>(const SchedEntry *, int, const MegaParams &, const Task *, const Blk *, const Task *, T *, int64_t, T *, int64_t, int32_t *, int32_t *, CallArgs<T> *, int, int, int, cudaStream_t);
    template cudaError_t launch_mega_down<T>(const SchedEntry *, int, const MegaParams &, const Task *, const Task *, const Blk *, T *, int64_t, const T *, int32_t *, CallArgs<T> *, int, int, int, cudaStream_t);
    template cudaError_t launch_chain<T>(int, const Task *, const ChainDep *, int, const Blk *, T *, int64_t, int, int, int32_t *, CallArgs<T> *, int, int, cudaStream_t);
    template cudaError_t launch_tree<T>(int, const TreeStage &, int, const Task *, const Blk *, T *, int64_t, int, int, cudaStream_t);
#undef T
}  // namespace h2
