// Probe of tcgen05.mma kind::tf32 on sm_100a (dev tool, not part of the library):
//  (1) where the rows of an M=64 accumulator land in TMEM (lanes), (2) K-major and MN-major
//  no-swizzle shared-memory descriptors, (3) whether TF32 operands are truncated or rounded.
//  nvcc -gencode arch=compute_100a,code=sm_100a -o umma_probe tools/umma_probe.cu && ./umma_probe
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;   // version (sm_100)
    return d;                 // layout type 0 = SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int amaj, int bmaj)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// mode 0: A K-major, mode 1: A MN-major.  B always K-major (N x K).
__global__ void probe(const float *A, const float *B, float *out, int mode, int M, int swap)
{
    __shared__ __align__(1024) float As[128 * 8];
    __shared__ __align__(1024) float Bs[16 * 8];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < M * 8; i += blockDim.x) {
        const int m = i / 8, k = i % 8;
        int off;
        if (mode == 0) off = (m / 8) * 64 + (k / 4) * 32 + (m % 8) * 4 + (k % 4);        // SBO 256 B, LBO 128 B
        else off = (m / 4) * 32 + (k % 8) * 4 + (m % 4);                                   // SBO 128 B (M groups of 4)
        As[off] = A[m * 8 + k];
    }
    for (int i = tid; i < 16 * 8; i += blockDim.x) {
        const int n = i / 8, k = i % 8;
        Bs[(n / 8) * 64 + (k / 4) * 32 + (n % 8) * 4 + (k % 4)] = B[n * 8 + k];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tm = tbase;
    if (tid == 0) {
        const uint64_t da = mode == 0 ? sdesc(su32(As), 128, 256) : (swap ? sdesc(su32(As), 128, 128 * 16) : sdesc(su32(As), 128 * 16, 128));
        const uint64_t db = sdesc(su32(Bs), 128, 256);
        const uint32_t id = idesc_tf32(M, 16, mode, 0);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(id), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
    }
    // wait phase 0
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    uint32_t v[16];
    const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int c = 0; c < 16; ++c) out[tid * 16 + c] = __uint_as_float(v[c]);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tm));
}

__global__ void probe_sw128(const float *A, const float *B, float *out, int M, int variant)
{
    __shared__ __align__(1024) float As[128 * 8];
    __shared__ __align__(1024) float Bs[16 * 8];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < M * 8; i += blockDim.x) {
        const int m = i / 8, k = i % 8;
        const int g = m / 32, mm = m % 32;                      // MN group, element within the 128 B row
        const int chunk = mm / 4, w = mm % 4;
        const int byte = g * 1024 + k * 128 + (((chunk ^ (k & 7)) * 16)) + w * 4;
        As[byte / 4] = A[m * 8 + k];
    }
    for (int i = tid; i < 16 * 8; i += blockDim.x) {
        const int n = i / 8, k = i % 8;
        Bs[(n / 8) * 64 + (k / 4) * 32 + (n % 8) * 4 + (k % 4)] = B[n * 8 + k];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tm = tbase;
    if (tid == 0) {
        uint64_t da = variant == 0 ? sdesc(su32(As), 1024, 8192) : sdesc(su32(As), 8192, 1024);
        da |= (uint64_t)2 << 61;                                  // SWIZZLE_128B
        const uint64_t db = sdesc(su32(Bs), 128, 256);
        const uint32_t id = idesc_tf32(M, 16, 1, 0);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(id), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
    }
    asm volatile("{\n.reg .pred P;\nW2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W2;\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    uint32_t v[16];
    const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int c = 0; c < 16; ++c) out[tid * 16 + c] = __uint_as_float(v[c]);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tm));
}

__global__ void probe_ksw128(const float *A, const float *B, float *out, int M, int ks)
{
    __shared__ __align__(1024) float As[128 * 32];
    __shared__ __align__(1024) float Bs[16 * 8];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    // rows of 128 B (32 K values); 16-byte chunk c of row r stored at chunk c ^ (r & 7)
    for (int i = tid; i < M * 32; i += blockDim.x) {
        const int m = i / 32, k = i % 32;
        const int chunk = k / 4, w = k % 4;
        As[m * 32 + ((chunk ^ (m & 7)) * 4) + w] = A[m * 32 + k];
    }
    for (int i = tid; i < 16 * 8; i += blockDim.x) {
        const int n = i / 8, k = i % 8;
        Bs[(n / 8) * 64 + (k / 4) * 32 + (n % 8) * 4 + (k % 4)] = B[n * 8 + k];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tm = tbase;
    if (tid == 0) {
        uint64_t da = sdesc(su32(As) + ks * 32, 16, 1024);       // SBO = 8 rows x 128 B
        da |= (uint64_t)2 << 61;                                  // SWIZZLE_128B
        const uint64_t db = sdesc(su32(Bs), 128, 256);
        const uint32_t id = idesc_tf32(M, 16, 0, 0);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(tm), "l"(da), "l"(db), "r"(id), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)));
    }
    asm volatile("{\n.reg .pred P;\nW3: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W3;\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    uint32_t v[16];
    const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int c = 0; c < 16; ++c) out[tid * 16 + c] = __uint_as_float(v[c]);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tm));
}

int main()
{
    float hA[128 * 8], hB[16 * 8], hO[128 * 16];
    float *dA, *dB, *dO;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dO, sizeof hO);
    int fails = 0;
    for (int M : {64, 128})
    for (int mode = 0; mode < 3; ++mode) {
        const int swap = mode == 2;
        for (int m = 0; m < M; ++m) for (int k = 0; k < 8; ++k) hA[m * 8 + k] = k == 0 ? (float)(m + 1) : (float)((m * 3 + k * 7) % 11 - 5);
        for (int n = 0; n < 16; ++n) for (int k = 0; k < 8; ++k) hB[n * 8 + k] = (float)((n * 5 + k * 3) % 7 - 3);
        cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
        cudaMemset(dO, 0xff, sizeof hO);
        probe<<<1, 128>>>(dA, dB, dO, mode ? 1 : 0, M, swap);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("M=%d mode %d: %s\n", M, mode, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
        // map each expected row to the TMEM lane holding it
        printf("M=%d A-%s: row->lane:", M, mode == 0 ? "K" : (swap ? "MN(lbo/sbo swapped)" : "MN"));
        int bad = 0;
        for (int m = 0; m < M; ++m) {
            int lane = -1;
            for (int l = 0; l < 128 && lane < 0; ++l) {
                bool ok = true;
                for (int n = 0; n < 16 && ok; ++n) {
                    float s = 0;
                    for (int k = 0; k < 8; ++k) s += hA[m * 8 + k] * hB[n * 8 + k];
                    ok = hO[l * 16 + n] == s;
                }
                if (ok) lane = l;
            }
            if (lane < 0) ++bad;
            if (m < 20 || m % 8 == 0 || m == M - 1) printf(" %d:%d", m, lane);
        }
        printf("  (%d rows not found)\n", bad);
        fails += bad;
    }
    // MN-major decode: A[m][k] = m + 128 k, B = identity (n = k < 8) -> D[m][n] = the A element the
    // tensor core read for (m, n); print it as (row, col)
    for (int swap = 0; swap < 2; ++swap) {
        const int M = 64;
        for (int m = 0; m < 128; ++m) for (int k = 0; k < 8; ++k) hA[m * 8 + k] = (float)(m + 128 * k);
        for (int n = 0; n < 16; ++n) for (int k = 0; k < 8; ++k) hB[n * 8 + k] = (n == k) ? 1.f : 0.f;
        cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
        probe<<<1, 128>>>(dA, dB, dO, 1, M, swap);
        cudaDeviceSynchronize();
        cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
        printf("MN decode swap=%d (lane: read (row,col) for col 0..7):\n", swap);
        for (int l : {0, 1, 2, 3, 4, 5, 8, 15, 32, 33}) {
            printf("  lane %3d:", l);
            for (int n = 0; n < 8; ++n) {
                const int v = (int)hO[l * 16 + n];
                printf(" (%d,%d)", v % 128, v / 128);
            }
            printf("\n");
        }
    }
    // MN-major A with 128-byte swizzle: M = 128 (4 groups of 32), K = 8: atom (mgroup) = 8 K rows x
    // 128 B, 16-byte chunk c of row r stored at chunk c ^ (r & 7); LBO = MN-group stride (1 KB),
    // SBO = K-group stride (unused for K = 8)
    {
        const int M = 128;
        for (int m = 0; m < 128; ++m) for (int k = 0; k < 8; ++k) hA[m * 8 + k] = (float)(m + 128 * k);
        for (int n = 0; n < 16; ++n) for (int k = 0; k < 8; ++k) hB[n * 8 + k] = (n == k) ? 1.f : 0.f;
        cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
        for (int variant = 0; variant < 2; ++variant) {
            probe_sw128<<<1, 128>>>(dA, dB, dO, M, variant);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("sw128 variant %d: %s\n", variant, cudaGetErrorString(e)); return 1; }
            cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
            int good = 0;
            for (int l = 0; l < 128; ++l) {
                bool ok = true;
                for (int n = 0; n < 8 && ok; ++n) ok = hO[l * 16 + n] == hA[l * 8 + n];
                good += ok;
            }
            printf("MN-major SW128 variant %d (lbo/sbo %s): %d of 128 rows correct; lane 0: (%g %g %g) lane 33: (%g %g)\n",
                   variant, variant ? "swapped" : "LBO=MN", good, hO[0], hO[1], hO[2], hO[33 * 16], hO[33 * 16 + 1]);
        }
    }
    // K-major A with 128-byte swizzle (the GEMM layout): A = 128 (M) x 32 (K) per atom row; one MMA
    // with K = 8 at K offset koff (start address + 32 B per 8-column step inside the 128 B row)
    {
        const int M = 128;
        static float hA2[128 * 32];
        for (int m = 0; m < 128; ++m) for (int k = 0; k < 32; ++k) hA2[m * 32 + k] = (float)(m + 128 * k);
        float *dA2;
        cudaMalloc(&dA2, sizeof hA2);
        cudaMemcpy(dA2, hA2, sizeof hA2, cudaMemcpyHostToDevice);
        for (int n = 0; n < 16; ++n) for (int k = 0; k < 8; ++k) hB[n * 8 + k] = (n == k) ? 1.f : 0.f;
        cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
        for (int ks = 0; ks < 4; ++ks) {
            probe_ksw128<<<1, 128>>>(dA2, dB, dO, M, ks);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("ksw128: %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
            int good = 0;
            for (int l = 0; l < 128; ++l) {
                bool ok = true;
                for (int n = 0; n < 8 && ok; ++n) ok = hO[l * 16 + n] == hA2[l * 32 + ks * 8 + n];
                good += ok;
            }
            printf("K-major SW128 k-step %d: %d of 128 rows correct (lane 1 col 0: %g want %g)\n", ks, good, hO[16],
                   hA2[32 + ks * 8]);
        }
    }
    // rounding probe: A = 1 + 3*2^-12 (between two TF32 values, nearer the upper), B = 1
    {
        const int M = 128;
        for (int i = 0; i < 128 * 8; ++i) hA[i] = 0.f;
        for (int i = 0; i < 16 * 8; ++i) hB[i] = 0.f;
        hA[0] = 1.0f + 3.0f * ldexpf(1.f, -12);
        hA[8] = 1.0f + 1.0f * ldexpf(1.f, -12);
        hA[16] = -(1.0f + 3.0f * ldexpf(1.f, -12));
        hB[0] = 1.f;
        cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
        probe<<<1, 128>>>(dA, dB, dO, 0, M, 0);
        cudaDeviceSynchronize();
        cudaMemcpy(hO, dO, sizeof hO, cudaMemcpyDeviceToHost);
        printf("rounding: 1+3*2^-12 -> 1 + %g ulp(2^-10); 1+2^-12 -> 1 + %g; -(1+3*2^-12) -> -(1 + %g)\n",
               (hO[0] - 1.f) / ldexpf(1.f, -10), (hO[16] - 1.f) / ldexpf(1.f, -10), (-hO[32] - 1.f) / ldexpf(1.f, -10));
        printf("  (truncation gives 0 0 0; round-to-nearest gives 1 0 1)\n");
    }
    printf(fails ? "FAIL\n" : "OK\n");
    return 0;
}
