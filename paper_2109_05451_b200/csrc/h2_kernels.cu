// h2_kernels.cu -- sm_100a kernels of the H^2 matvec hot path.
//
// Every phase is a set of warp tasks over a static plan built once by h2_create (the paper's
// per-level marshaling, done at setup instead of per call).  A task owns one
// output node (row-owner computes: no atomics, no conflict batches) and
// accumulates   y_rows (r x nv) += sum_b A_b (r x c) x_b (c x nv)   with lanes <-> output rows
// (RPL rows per lane), A streamed once from HBM with coalesced column loads (evict-first),
// and the x operand staged per block in warp-private shared memory (broadcast reads).
//
//   up_leaf   x^_s = V_s^T x_s                         PAPER.md:239, 262 (alg:upsweep2 line 3)
//   rows/W    x^_p = F_{c1}^T x^_{c1} + F_{c2}^T x^_{c2} PAPER.md:241-253, 267-268
//   rows/W    y^_t = sum_s S_ts x^_s  (all levels)      PAPER.md:328-331, 344-356 (alg:mult)
//   rows/A    y^_c += E_c y^_parent                     PAPER.md:389-399, 408-412 (alg:downsweep)
//   leaf      z_t = y^_t + E_t y^_parent ; y_t = U_t z_t + sum_s D_ts x_s ;
//             Y = alpha y + beta Y                      PAPER.md:399, 414, 225; reading R11/R12
#include "h2_internal.h"

namespace h2 {

template <typename T>
__device__ __forceinline__ T ld_stream(const T *p) { return __ldcs(p); }

// x operand (c x NVB) of one block into warp smem xs[n * XLD + j]; rows >= xrows and vectors
// >= nvc are zero (ragged leaves / partial vector chunk).
template <typename T, int NVB>
__device__ __forceinline__ void stage_x(T *xs, const T *__restrict__ src, int64_t ld, int xrows,
                                        int c, int nvc, int lane)
{
#pragma unroll
    for (int n = 0; n < NVB; ++n) {
        for (int j = lane; j < c; j += 32)
            xs[n * XLD + j] = (n < nvc && j < xrows) ? src[j + n * ld] : T(0);
    }
}

// acc[ri][n] += sum_j A[(j) * r + lane + 32 ri] * xs[n * XLD + j]
template <typename T, int RPL, int NVB>
__device__ __forceinline__ void acc_block(T (&acc)[RPL][NVB], const T *__restrict__ A, int r,
                                          int c, const T *xs, int lane)
{
    int j = 0;
    for (; j + 8 <= c; j += 8) {
        T a[8][RPL];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int ri = 0; ri < RPL; ++ri) {
                int i = lane + 32 * ri;
                a[u][ri] = (i < r) ? ld_stream(A + (int64_t)(j + u) * r + i) : T(0);
            }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int n = 0; n < NVB; ++n) {
                T xv = xs[n * XLD + j + u];
#pragma unroll
                for (int ri = 0; ri < RPL; ++ri) acc[ri][n] = fma(a[u][ri], xv, acc[ri][n]);
            }
    }
    for (; j < c; ++j) {
        T a[RPL];
#pragma unroll
        for (int ri = 0; ri < RPL; ++ri) {
            int i = lane + 32 * ri;
            a[ri] = (i < r) ? ld_stream(A + (int64_t)j * r + i) : T(0);
        }
#pragma unroll
        for (int n = 0; n < NVB; ++n) {
            T xv = xs[n * XLD + j];
#pragma unroll
            for (int ri = 0; ri < RPL; ++ri) acc[ri][n] = fma(a[ri], xv, acc[ri][n]);
        }
    }
}

template <typename T, int RPL, int NVB>
__device__ __forceinline__ void zero_acc(T (&acc)[RPL][NVB])
{
#pragma unroll
    for (int ri = 0; ri < RPL; ++ri)
#pragma unroll
        for (int n = 0; n < NVB; ++n) acc[ri][n] = T(0);
}

// ---------------------------------------------------------------------------------------
// Upsweep leaves: x^_s (k x nv) = Vt_s (k x m) x_s (m x nv), Vt = V^T re-laid out at create.
template <typename T, int RPL, int NVB>
__global__ void __launch_bounds__(WPB * 32)
k_up_leaf(const Task *__restrict__ tasks, int ntask, const Blk *__restrict__ blks,
          const T *__restrict__ X, int64_t ldx, T *__restrict__ xh, int64_t xh_ld, int nv)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int task = blockIdx.x * WPB + wid;
    if (task >= ntask) return;
    T *xs = reinterpret_cast<T *>(smem_raw) + wid * NVB * XLD;
    const Task tk = tasks[task];
    const Blk b = blks[tk.blk0];
    const T *A = static_cast<const T *>(b.A);
    for (int n0 = 0; n0 < nv; n0 += NVB) {
        const int nvc = min(NVB, nv - n0);
        T acc[RPL][NVB];
        zero_acc(acc);
        __syncwarp();
        stage_x<T, NVB>(xs, X + b.x + n0 * ldx, ldx, b.xrows, tk.c, nvc, lane);
        __syncwarp();
        acc_block<T, RPL, NVB>(acc, A, tk.r, tk.c, xs, lane);
#pragma unroll
        for (int ri = 0; ri < RPL; ++ri) {
            int i = lane + 32 * ri;
            if (i < tk.r)
#pragma unroll
                for (int n = 0; n < NVB; ++n)
                    if (n < nvc) xh[tk.out + i + (int64_t)(n0 + n) * xh_ld] = acc[ri][n];
        }
    }
}

// ---------------------------------------------------------------------------------------
// Generic row tasks whose x operands and output live in the x^/y^ workspaces:
//   MODE_WRITE  out  = sum_b A_b x_b    (upsweep transfers, coupling multiply)
//   MODE_ACCUM  out += sum_b A_b x_b    (downsweep transfers, off-diagonal coupling pass)
template <typename T, int RPL, int NVB, int MODE>
__global__ void __launch_bounds__(WPB * 32)
k_rows(const Task *__restrict__ tasks, int ntask, const Blk *__restrict__ blks,
       const T *__restrict__ src, int64_t src_ld, T *__restrict__ dst, int64_t dst_ld, int nv)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int task = blockIdx.x * WPB + wid;
    if (task >= ntask) return;
    T *xs = reinterpret_cast<T *>(smem_raw) + wid * NVB * XLD;
    const Task tk = tasks[task];
    for (int n0 = 0; n0 < nv; n0 += NVB) {
        const int nvc = min(NVB, nv - n0);
        T acc[RPL][NVB];
        if (MODE == MODE_ACCUM) {
#pragma unroll
            for (int ri = 0; ri < RPL; ++ri) {
                int i = lane + 32 * ri;
#pragma unroll
                for (int n = 0; n < NVB; ++n)
                    acc[ri][n] = (i < tk.r && n < nvc)
                                     ? dst[tk.out + i + (int64_t)(n0 + n) * dst_ld] : T(0);
            }
        } else {
            zero_acc(acc);
        }
        for (int bi = 0; bi < tk.nblk; ++bi) {
            const Blk b = blks[tk.blk0 + bi];
            const int64_t ld = b.xld ? (int64_t)b.xld : src_ld;
            __syncwarp();
            stage_x<T, NVB>(xs, src + b.x + (int64_t)n0 * ld, ld, b.xrows, tk.c, nvc, lane);
            __syncwarp();
            acc_block<T, RPL, NVB>(acc, static_cast<const T *>(b.A), tk.r, tk.c, xs, lane);
        }
#pragma unroll
        for (int ri = 0; ri < RPL; ++ri) {
            int i = lane + 32 * ri;
            if (i < tk.r)
#pragma unroll
                for (int n = 0; n < NVB; ++n)
                    if (n < nvc) dst[tk.out + i + (int64_t)(n0 + n) * dst_ld] = acc[ri][n];
        }
    }
}

// ---------------------------------------------------------------------------------------
// Leaf kernel: last downsweep transfer + leaf expansion + dense near field + epilogue.
// blocks: [E_t (if flags&1), x = parent y^ offset] [U_t, x = own y^ offset] [D_ts ...]
template <typename T, int RPLK, int RPLM, int NVB>
__global__ void __launch_bounds__(WPB * 32)
k_leaf(const Task *__restrict__ tasks, int ntask, const Blk *__restrict__ blks,
       const T *__restrict__ yh, int64_t yh_ld, const T *__restrict__ X, int64_t ldx,
       const T *__restrict__ halo, int64_t halo_ld, T *__restrict__ Y, int64_t ldy, T alpha,
       T beta, int nv, int k, int kp)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int task = blockIdx.x * WPB + wid;
    if (task >= ntask) return;
    T *xs = reinterpret_cast<T *>(smem_raw) + wid * NVB * XLD;
    const Task tk = tasks[task];
    const bool hasE = tk.flags & 1;
    const Blk bU = blks[tk.blk0 + (hasE ? 1 : 0)];
    for (int n0 = 0; n0 < nv; n0 += NVB) {
        const int nvc = min(NVB, nv - n0);
        // z_t = y^_t + E_t y^_parent   (lanes <-> rank rows)
        T z[RPLK][NVB];
#pragma unroll
        for (int ri = 0; ri < RPLK; ++ri) {
            int i = lane + 32 * ri;
#pragma unroll
            for (int n = 0; n < NVB; ++n)
                z[ri][n] = (i < k && n < nvc) ? yh[bU.x + i + (int64_t)(n0 + n) * yh_ld] : T(0);
        }
        if (hasE) {
            const Blk bE = blks[tk.blk0];
            __syncwarp();
            stage_x<T, NVB>(xs, yh + bE.x + (int64_t)n0 * yh_ld, yh_ld, bE.xrows, kp, nvc, lane);
            __syncwarp();
            acc_block<T, RPLK, NVB>(z, static_cast<const T *>(bE.A), k, kp, xs, lane);
        }
        __syncwarp();
#pragma unroll
        for (int ri = 0; ri < RPLK; ++ri) {
            int i = lane + 32 * ri;
            if (i < k)
#pragma unroll
                for (int n = 0; n < NVB; ++n) xs[n * XLD + i] = z[ri][n];
        }
        __syncwarp();
        // y_t = U_t z_t  (lanes <-> leaf rows)
        T acc[RPLM][NVB];
        zero_acc(acc);
        acc_block<T, RPLM, NVB>(acc, static_cast<const T *>(bU.A), tk.r, k, xs, lane);
        // dense near field y_t += sum_s D_ts x_s
        const int64_t d0 = tk.blk0 + (hasE ? 2 : 1), d1 = tk.blk0 + tk.nblk;
        for (int64_t bi = d0; bi < d1; ++bi) {
            const Blk b = blks[bi];
            const T *src;
            int64_t ld;
            if (b.x >= 0) { src = X + b.x; ld = ldx; }
            else          { src = halo + (-b.x - 1); ld = b.xld ? (int64_t)b.xld : halo_ld; }
            __syncwarp();
            stage_x<T, NVB>(xs, src + (int64_t)n0 * ld, ld, b.xrows, tk.r, nvc, lane);
            __syncwarp();
            acc_block<T, RPLM, NVB>(acc, static_cast<const T *>(b.A), tk.r, tk.r, xs, lane);
        }
        // epilogue Y = alpha y + beta Y (beta == 0: Y not read)
#pragma unroll
        for (int ri = 0; ri < RPLM; ++ri) {
            int i = lane + 32 * ri;
            if (i < tk.rows)
#pragma unroll
                for (int n = 0; n < NVB; ++n)
                    if (n < nvc) {
                        T *p = Y + tk.out + i + (int64_t)(n0 + n) * ldy;
                        *p = (beta == T(0)) ? alpha * acc[ri][n] : fma(alpha, acc[ri][n], beta * *p);
                    }
        }
    }
}

template <typename T>
__global__ void k_scale(T *Y, int64_t ldy, int64_t n, int nv, T beta)
{
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * nv;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = e / n, r = e - c * n;
        T *p = Y + r + c * ldy;
        *p = (beta == T(0)) ? T(0) : beta * *p;
    }
}

// batched transpose of column-major r x c matrices into column-major c x r
template <typename T>
__global__ void k_transpose(const T *__restrict__ src, T *__restrict__ dst, int64_t batch, int r,
                            int c)
{
    const int64_t per = (int64_t)r * c;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < batch * per;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t bidx = e / per, w = e - bidx * per;
        int j = (int)(w / r), i = (int)(w - (int64_t)j * r);   // src (i, j)
        dst[bidx * per + i * (int64_t)c + j] = src[e];
    }
}

// gather segments (pack for the halo exchange): one warp per segment,
// dst[seg.dst + j + n * seg.dst_ld] = src[seg.src + j + n * src_ld], j < seg.len, n < nv
template <typename T>
__global__ void k_pack(const PackSeg *__restrict__ segs, int64_t nseg, const T *__restrict__ src,
                       int64_t src_ld, T *__restrict__ dst, int nv)
{
    const int lane = threadIdx.x & 31;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nseg;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const PackSeg sg = segs[w];
        for (int n = 0; n < nv; ++n)
            for (int j = lane; j < sg.len; j += 32)
                dst[sg.dst + j + (int64_t)n * sg.dst_ld] = src[sg.src + j + (int64_t)n * src_ld];
    }
}

// ---------------------------------------------------------------------------------------
// launchers
static inline int grid_for(int ntask) { return (ntask + WPB - 1) / WPB; }

template <typename K>
static cudaError_t set_smem(K kernel, size_t bytes)
{
    if (bytes > 48 * 1024)
        return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return cudaSuccess;
}

static inline int nvb_for(int nv) { return nv <= 1 ? 1 : nv <= 2 ? 2 : nv <= 4 ? 4 : nv <= 8 ? 8 : 16; }

#define H2_NVB_SWITCH(nvb, ...)                                  \
    switch (nvb) {                                               \
    case 1: { constexpr int NVB = 1; __VA_ARGS__; } break;       \
    case 2: { constexpr int NVB = 2; __VA_ARGS__; } break;       \
    case 4: { constexpr int NVB = 4; __VA_ARGS__; } break;       \
    case 8: { constexpr int NVB = 8; __VA_ARGS__; } break;       \
    default: { constexpr int NVB = 16; __VA_ARGS__; } break;     \
    }
#define H2_RPL_SWITCH(rpl, NAME, ...)                                  \
    if ((rpl) <= 1) { constexpr int NAME = 1; __VA_ARGS__; }           \
    else            { constexpr int NAME = 2; __VA_ARGS__; }

template <typename T>
cudaError_t launch_up_leaf(const Task *t, int ntask, const Blk *b, const T *X, int64_t ldx,
                           T *xh, int64_t xh_ld, int nv, int rpl, cudaStream_t s)
{
    if (ntask == 0) return cudaSuccess;
    cudaError_t err = cudaSuccess;
    H2_NVB_SWITCH(nvb_for(nv), H2_RPL_SWITCH(rpl, RPL, {
        size_t sm = (size_t)WPB * NVB * XLD * sizeof(T);
        err = set_smem(k_up_leaf<T, RPL, NVB>, sm);
        if (err == cudaSuccess)
            k_up_leaf<T, RPL, NVB><<<grid_for(ntask), WPB * 32, sm, s>>>(t, ntask, b, X, ldx, xh, xh_ld, nv);
    }))
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_rows(int mode, const Task *t, int ntask, const Blk *b, const T *src,
                        int64_t src_ld, T *dst, int64_t dst_ld, int nv, int rpl, cudaStream_t s)
{
    if (ntask == 0) return cudaSuccess;
    cudaError_t err = cudaSuccess;
    H2_NVB_SWITCH(nvb_for(nv), H2_RPL_SWITCH(rpl, RPL, {
        size_t sm = (size_t)WPB * NVB * XLD * sizeof(T);
        if (mode == MODE_WRITE) {
            err = set_smem(k_rows<T, RPL, NVB, MODE_WRITE>, sm);
            if (err == cudaSuccess)
                k_rows<T, RPL, NVB, MODE_WRITE><<<grid_for(ntask), WPB * 32, sm, s>>>(
                    t, ntask, b, src, src_ld, dst, dst_ld, nv);
        } else {
            err = set_smem(k_rows<T, RPL, NVB, MODE_ACCUM>, sm);
            if (err == cudaSuccess)
                k_rows<T, RPL, NVB, MODE_ACCUM><<<grid_for(ntask), WPB * 32, sm, s>>>(
                    t, ntask, b, src, src_ld, dst, dst_ld, nv);
        }
    }))
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_leaf(const Task *t, int ntask, const Blk *b, const T *yh, int64_t yh_ld,
                             const T *X, int64_t ldx, const T *halo, int64_t halo_ld, T *Y,
                             int64_t ldy, T alpha, T beta, int nv, int k, int kp, int rplk,
                             int rplm, cudaStream_t s)
{
    if (ntask == 0) return cudaSuccess;
    cudaError_t err = cudaSuccess;
    H2_NVB_SWITCH(nvb_for(nv), H2_RPL_SWITCH(rplk, RK, H2_RPL_SWITCH(rplm, RM, {
        size_t sm = (size_t)WPB * NVB * XLD * sizeof(T);
        err = set_smem(k_leaf<T, RK, RM, NVB>, sm);
        if (err == cudaSuccess)
            k_leaf<T, RK, RM, NVB><<<grid_for(ntask), WPB * 32, sm, s>>>(
                t, ntask, b, yh, yh_ld, X, ldx, halo, halo_ld, Y, ldy, alpha, beta, nv, k, kp);
    })))
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_scale(T *Y, int64_t ldy, int64_t n, int nv, T beta, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    k_scale<T><<<1184, 256, 0, s>>>(Y, ldy, n, nv, beta);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_transpose(const T *src, T *dst, int64_t batch, int r, int c, cudaStream_t s)
{
    if (batch == 0) return cudaSuccess;
    k_transpose<T><<<1184, 256, 0, s>>>(src, dst, batch, r, c);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pack(const PackSeg *segs, int64_t nseg, const T *src, int64_t src_ld, T *dst,
                        int nv, cudaStream_t s)
{
    if (nseg == 0) return cudaSuccess;
    int64_t blocks = (nseg + 7) / 8;
    k_pack<T><<<(int)(blocks < 1184 ? blocks : 1184), 256, 0, s>>>(segs, nseg, src, src_ld, dst, nv);
    return cudaGetLastError();
}

#define H2_INSTANTIATE(T)                                                                     \
    template cudaError_t launch_up_leaf<T>(const Task *, int, const Blk *, const T *, int64_t, \
                                           T *, int64_t, int, int, cudaStream_t);             \
    template cudaError_t launch_rows<T>(int, const Task *, int, const Blk *, const T *,       \
                                        int64_t, T *, int64_t, int, int, cudaStream_t);       \
    template cudaError_t launch_leaf<T>(    const Task *, int, const Blk *, const T *,       \
                                             int64_t, const T *, int64_t, const T *, int64_t, \
                                             T *, int64_t, T, T, int, int, int, int, int,     \
                                             cudaStream_t);                                   \
    template cudaError_t launch_scale<T>(T *, int64_t, int64_t, int, T, cudaStream_t);         \
    template cudaError_t launch_transpose<T>(const T *, T *, int64_t, int, int, cudaStream_t); \
    template cudaError_t launch_pack<T>(const PackSeg *, int64_t, const T *, int64_t, T *, int, \
                                        cudaStream_t);

H2_INSTANTIATE(double)
H2_INSTANTIATE(float)

}  // namespace h2
