// h2_k_mono.cu -- explicit instantiations of the single-launch latency path (h2_mono.cuh)
#include "h2_mono.cuh"

namespace h2 {
template cudaError_t launch_mono<double>(const MonoPlan &, const Task *, const Blk *, double *, double *, int64_t,
                                         const CallArgs<double> *, int, int, int, cudaStream_t);
template cudaError_t launch_mono<float>(const MonoPlan &, const Task *, const Blk *, float *, float *, int64_t,
                                        const CallArgs<float> *, int, int, int, cudaStream_t);
}  // namespace h2
