// h2_k_sym.cu -- explicit instantiations of the symmetric-storage launchers (h2_sym.cuh)
#include "h2_sym.cuh"

namespace h2 {
#define INST(T)                                                                                                    \
    template cudaError_t launch_sym_rows<T>(const Task *, int, const Blk *, const T *, T *, int, cudaStream_t);    \
    template cudaError_t launch_sym_leaf<T>(const Task *, const Task *, int, const Blk *, const T *,               \
                                            const CallArgs<T> *, int, cudaStream_t);                               \
    template cudaError_t launch_beta<T>(const CallArgs<T> *, int64_t, int, cudaStream_t);
INST(double)
INST(float)
#undef INST
}  // namespace h2
