// h2_k_umma_f32.cu -- the tcgen05 FP32 row engine (h2_umma.cuh) and its launcher
#include <cstring>
#include <type_traits>
#include "h2_kernels.cuh"
#include "h2_umma.cuh"
