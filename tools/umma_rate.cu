// Microbenchmark (dev tool): cycles per tcgen05.mma.kind::tf32 for small shapes, SS operands,
// nmma back-to-back MMAs issued by one thread into NCH independent accumulators, then one commit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o umma_rate tools/umma_rate.cu && ./umma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);
}
__global__ void rate(int M, int N, int nmma, int nch, long long *out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint32_t tb;
    __shared__ __align__(8) uint64_t bar;
    float *f = reinterpret_cast<float *>(sm);
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) f[i] = 0.001f * (i % 13);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&tb)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tm = tb;
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x < 32) {          // whole warp, converged; one elected lane issues
        const uint32_t a = su32(sm), b = su32(sm + 32768);
        __syncwarp();
        t0 = clock64();
        const uint64_t da0 = sdesc(a, 128, 2048), db0 = sdesc(b, 128, 2048);
        for (int i0 = 0; i0 < nmma; i0 += 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (i0 + i >= nmma) break;
                // descriptor start address advances 256 B per k-step: +16 in the (addr >> 4) field
                const uint64_t da = da0 + (uint64_t)(i * 16), db = db0 + (uint64_t)(i * 16);
                const uint32_t d = tm + (uint32_t)((nch == 1 ? 0 : i) * N);
                asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(d), "l"(da), "l"(db), "r"(id), "r"(i0 + i >= nch ? 1 : 0));
            }
        }
        long long ti = clock64();
        asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(&bar)));
        asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(su32(&bar)));
        t1 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = ti - t0; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tm));
}

int main()
{
    long long *d, h[2];
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    struct S { int M, N; } shapes[] = {{64, 16}, {128, 16}, {128, 32}, {128, 64}, {128, 128}};
    for (auto sh : shapes)
        for (int nch : {1, 8})
            for (int nmma : {1, 8, 64, 256}) {
                if (sh.N * nch > 512) continue;
                rate<<<1, 128, 64 * 1024>>>(sh.M, sh.N, nmma, nch, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                rate<<<1, 128, 64 * 1024>>>(sh.M, sh.N, nmma, nch, d);
                cudaDeviceSynchronize();
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                printf("M=%3d N=%3d chains=%d nmma=%2d: %6lld cycles (%.1f per MMA), issue %lld\n", sh.M, sh.N, nch, nmma,
                       h[0], (double)h[0] / nmma, h[1]);
            }
    return 0;
}
