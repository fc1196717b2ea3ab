// h2_k_p2p.cu -- the signal kernels of the device-initiated peer exchange (h2_internal.h,
// SURVEY.md §8(f) NEXT-1; PAPER.md:477-480, 505-509 for the exchange they replace).  One thread
// each: flags are int32 epochs in the handles' signal blocks, written across GPUs through CUDA-IPC
// mappings (st.release.sys) and polled with ld.acquire.sys.
#include "h2_internal.h"

#include <cstdio>

namespace h2 {
namespace {

__device__ __forceinline__ int ld_acq(const int32_t *p)
{
    int v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(int32_t *p, int v)
{
    asm volatile("st.release.sys.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until(const int32_t *p, int target, int slot)
{
    unsigned long long n = 0;
    while (ld_acq(p) < target) {
        __nanosleep(128);
        if (++n > 150000000ull) {             // ~20 s: a peer is gone; fail loudly instead of hanging
            printf("h2 p2p: signal slot %d stuck at %d (waiting for %d)\n", slot, ld_acq(p), target);
            __trap();
        }
    }
}

__global__ void k_p2p_begin(int32_t *sig, const int32_t *waits, int nwait)
{
    const int e = sig[SIG_EPOCH] + 1;
    sig[SIG_EPOCH] = e;
    for (int i = 0; i < nwait; ++i) spin_until(sig + waits[i], e - 1, waits[i]);
    __threadfence_system();
}

__global__ void k_p2p_signal(const int32_t *sig, int32_t *const *targets, int n)
{
    const int e = sig[SIG_EPOCH];
    __threadfence_system();
    for (int i = 0; i < n; ++i) st_rel(targets[i], e);
}

__global__ void k_p2p_wait(const int32_t *sig, const int32_t *offs, int n)
{
    const int e = sig[SIG_EPOCH];
    for (int i = 0; i < n; ++i) spin_until(sig + offs[i], e, offs[i]);
    __threadfence_system();
}

}  // namespace

cudaError_t launch_p2p_begin(int32_t *sig, const int32_t *waits, int nwait, cudaStream_t s)
{
    k_p2p_begin<<<1, 1, 0, s>>>(sig, waits, nwait);
    return cudaGetLastError();
}
cudaError_t launch_p2p_signal(const int32_t *sig, int32_t *const *targets, int n, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    k_p2p_signal<<<1, 1, 0, s>>>(sig, targets, n);
    return cudaGetLastError();
}
cudaError_t launch_p2p_wait(const int32_t *sig, const int32_t *offs, int n, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    k_p2p_wait<<<1, 1, 0, s>>>(sig, offs, n);
    return cudaGetLastError();
}

}  // namespace h2
