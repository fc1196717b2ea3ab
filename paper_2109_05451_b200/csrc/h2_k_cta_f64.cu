// h2_k_cta_f64.cu -- the CTA-tile FP64 engine (h2_cta.cuh) and its launcher
#include "h2_kernels.cuh"
#include "h2_cta.cuh"
