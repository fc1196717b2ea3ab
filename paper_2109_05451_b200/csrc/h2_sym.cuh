// h2_sym.cuh -- symmetric-storage kernels (DESIGN.md §7 "Symmetric storage"; SURVEY.md §8(f)
// NEXT-2; PAPER.md:145-150 for the blocks A_ts = U_t S_ts V_s^T of a symmetric H² matrix).
//
// With U = V, E = F, S^l_st = (S^l_ts)^T and D_st = D_ts^T only the blocks with t <= s are stored
// (h2_desc.flags & H2_SYMMETRIC).  A warp owns block row t and applies every stored block (t, s)
// of it twice from ONE read of the block: directly, y_t += A x_s (registers), and -- for s > t,
// the "mirrored" blocks -- transposed, y_s += A^T x_t, by a 32-column reduce-scatter across the
// lanes (16 shuffles per 16 columns) and one red.global.add per column.  Outputs therefore
// accumulate with atomics: the coupling rows into a zeroed y^, the leaves into Y after a beta pass.
// nv = 1 (the HBM-bound case the halved bytes pay for).
#pragma once
#include "h2_internal.h"

namespace h2 {
// CTAs per SM the sym kernels' registers are sized for (memory-latency-bound: more warps in flight)
#ifndef SYM_MINB
#define SYM_MINB 4
#endif
namespace sym {

constexpr unsigned FULL = 0xffffffffu;

// lanes c and c + 16 end with the sum over all lanes of v[c] (in v[0]): a 16-value reduce-scatter
// over the lane bits 0..3 (15 shuffles), then one exchange across bit 4
template <typename T>
__device__ __forceinline__ void reduce_scatter16(T (&v)[16], int lane)
{
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
        const bool hi = lane & o;
#pragma unroll
        for (int i = 0; i < o; ++i) {
            const T send = hi ? v[i] : v[i + o];
            const T keep = hi ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(FULL, send, o);
        }
    }
    v[0] += __shfl_xor_sync(FULL, v[0], 16);
}

// acc (r rows: lane, lane + 32) += A (r x c, column-major) x_s, x_s held as xs0 / xs1 (rows lane,
// lane + 32); if MIRROR: ymir[j] += alpha * (A^T x_t)[j], x_t held as xt0 / xt1.
template <typename T, int RPL, bool MIRROR>
__device__ __forceinline__ void block(T (&acc)[RPL], const T *__restrict__ A, int r, int c, T xs0, T xs1, T xt0,
                                      T xt1, T *ymir, T alpha, int lane)
{
    for (int j0 = 0; j0 < c; j0 += 16) {
        T v[16];
        const T xsrc = j0 < 32 ? xs0 : xs1;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int j = j0 + u;
            const T a0 = (j < c && lane < r) ? __ldcs(A + (int64_t)j * r + lane) : T(0);
            const T a1 = (RPL == 2 && j < c && lane + 32 < r) ? __ldcs(A + (int64_t)j * r + lane + 32) : T(0);
            const T xj = __shfl_sync(FULL, xsrc, (j0 & 31) + u);
            acc[0] = fma(a0, xj, acc[0]);
            if (RPL == 2) acc[RPL - 1] = fma(a1, xj, acc[RPL - 1]);
            if (MIRROR) v[u] = RPL == 2 ? fma(a1, xt1, a0 * xt0) : a0 * xt0;
        }
        if (MIRROR) {
            reduce_scatter16(v, lane);
            if (lane < 16 && j0 + lane < c) atomicAdd(ymir + j0 + lane, alpha * v[0]);
        }
    }
}

template <typename T, int RPL>
__device__ __forceinline__ void apply(T (&acc)[RPL], const Blk &b, int r, int c, const T *xs_base, const T *xt,
                                      int xt_rows, T *ymir_base, T alpha, int lane)
{
    const T *xs = xs_base + b.x;
    const T xs0 = lane < b.xrows ? xs[lane] : T(0);
    const T xs1 = lane + 32 < b.xrows ? xs[lane + 32] : T(0);
    const T *A = static_cast<const T *>(b.A);
    if (b.xld == -1) {
        const T xt0 = lane < xt_rows ? xt[lane] : T(0);
        const T xt1 = lane + 32 < xt_rows ? xt[lane + 32] : T(0);
        block<T, RPL, true>(acc, A, r, c, xs0, xs1, xt0, xt1, ymir_base + b.x, alpha, lane);
    } else {
        block<T, RPL, false>(acc, A, r, c, xs0, xs1, T(0), T(0), nullptr, alpha, lane);
    }
}

}  // namespace sym

// Coupling rows (all levels of one class): y^_t += sum_{s >= t} S_ts x^_s ; y^_s += S_ts^T x^_t.
// x^ and y^ share the plane layout, so Blk::x addresses both x^_s and y^_s and Task::out both y^_t
// and x^_t.  y^ was zeroed before the launch.
template <typename T, int RPL>
__global__ void __launch_bounds__(256, SYM_MINB) k_sym_rows(const Task *__restrict__ tasks, int ntask, const Blk *__restrict__ blks,
                                                  const T *__restrict__ xh, T *yh)
{
    const int lane = threadIdx.x & 31;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ntask; w += (gridDim.x * blockDim.x) >> 5) {
        const Task tk = tasks[w];
        T acc[RPL] = {};
        const T *xt = xh + tk.out;
        // the next block's descriptor is loaded while this block streams (latency-bound kernel)
        Blk nb = tk.nblk > 0 ? blks[tk.blk0] : Blk{};
        for (int bi = 0; bi < tk.nblk; ++bi) {
            const Blk b = nb;
            if (bi + 1 < tk.nblk) nb = blks[tk.blk0 + bi + 1];
            sym::apply<T, RPL>(acc, b, tk.r, tk.c, xh, xt, tk.r, yh, T(1), lane);
        }
#pragma unroll
        for (int ri = 0; ri < RPL; ++ri)
            if (lane + 32 * ri < tk.r) atomicAdd(yh + tk.out + lane + 32 * ri, acc[ri]);
    }
}

// Leaves: z = y^_t + E_t y^_parent ; Y_t += alpha (U_t z + sum_{s >= t} D_ts x_s) ;
// Y_s += alpha D_ts^T x_t (s > t).  Y was scaled by beta before the launch.
template <typename T, int RPL>
__global__ void __launch_bounds__(256, SYM_MINB) k_sym_leaf(const Task *__restrict__ ltasks, const Task *__restrict__ dtasks,
                                                  int ntask, const Blk *__restrict__ blks, const T *__restrict__ yh,
                                                  const CallArgs<T> *__restrict__ args)
{
    const int lane = threadIdx.x & 31;
    const T *__restrict__ X = args->X;
    T *Y = args->Y;
    const T alpha = args->alpha;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < ntask; w += (gridDim.x * blockDim.x) >> 5) {
        const Task tk = ltasks[w];
        const Task dk = dtasks[w];
        const bool hasE = tk.flags & TF_HAS_E;
        const Blk bU = blks[tk.blk0 + (hasE ? 1 : 0)];
        const int k = bU.xrows;
        // z (k rows) = y^_t + E_t y^_parent
        T z[2];
        z[0] = lane < k ? yh[bU.x + lane] : T(0);
        z[1] = lane + 32 < k ? yh[bU.x + lane + 32] : T(0);
        if (hasE) {
            const Blk bE = blks[tk.blk0];
            if (k > 32) {
                T zz[2] = {z[0], z[1]};
                sym::apply<T, 2>(zz, bE, k, bE.xrows, yh, nullptr, 0, nullptr, T(1), lane);
                z[0] = zz[0];
                z[1] = zz[1];
            } else {
                T zz[1] = {z[0]};
                sym::apply<T, 1>(zz, bE, k, bE.xrows, yh, nullptr, 0, nullptr, T(1), lane);
                z[0] = zz[0];
            }
        }
        // y (m rows) = U_t z + dense row
        T acc[RPL] = {};
        sym::block<T, RPL, false>(acc, static_cast<const T *>(bU.A), tk.r, k, z[0], z[1], T(0), T(0), nullptr,
                                  alpha, lane);
        const T *xt = X + tk.out;
        Blk nb = dk.nblk > 0 ? blks[dk.blk0] : Blk{};
        for (int bi = 0; bi < dk.nblk; ++bi) {
            const Blk b = nb;
            if (bi + 1 < dk.nblk) nb = blks[dk.blk0 + bi + 1];
            sym::apply<T, RPL>(acc, b, dk.r, dk.c, X, xt, tk.rows, Y, alpha, lane);
        }
#pragma unroll
        for (int ri = 0; ri < RPL; ++ri)
            if (lane + 32 * ri < tk.rows) atomicAdd(Y + tk.out + lane + 32 * ri, alpha * acc[ri]);
    }
}

// Y := beta Y on the call's Y (read from the device CallArgs: graph-capturable)
template <typename T>
__global__ void k_beta(const CallArgs<T> *__restrict__ args, int64_t n, int nv)
{
    T *Y = args->Y;
    const int64_t ldy = args->ldy;
    const T beta = args->beta;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * nv; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / n, r = e - c * n;
        T *p = Y + r + c * ldy;
        *p = (beta == T(0)) ? T(0) : beta * *p;
    }
}

template <typename T>
cudaError_t launch_beta(const CallArgs<T> *args, int64_t n, int nv, cudaStream_t s)
{
    if (n == 0) return cudaSuccess;
    k_beta<T><<<592, 256, 0, s>>>(args, n, nv);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_sym_rows(const Task *t, int ntask, const Blk *b, const T *xh, T *yh, int r, cudaStream_t s)
{
    if (ntask == 0) return cudaSuccess;
    const int grid = (ntask + 7) / 8;
    if (r > 32) k_sym_rows<T, 2><<<grid, 256, 0, s>>>(t, ntask, b, xh, yh);
    else        k_sym_rows<T, 1><<<grid, 256, 0, s>>>(t, ntask, b, xh, yh);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_sym_leaf(const Task *lt, const Task *dt, int ntask, const Blk *b, const T *yh,
                            const CallArgs<T> *args, int m, cudaStream_t s)
{
    if (ntask == 0) return cudaSuccess;
    const int grid = (ntask + 7) / 8;
    if (m > 32) k_sym_leaf<T, 2><<<grid, 256, 0, s>>>(lt, dt, ntask, b, yh, args);
    else        k_sym_leaf<T, 1><<<grid, 256, 0, s>>>(lt, dt, ntask, b, yh, args);
    return cudaGetLastError();
}

}  // namespace h2
