// h2_mono.cuh -- the whole matvec in ONE cooperative launch for L2-resident problems (DESIGN.md §7
// "Latency path"; "latency ... report µs and launches").
//
// For an operator that fits in L2 the matvec is bound by launch and dependency latency, not by
// bytes: round 1's 13 launches (plus a side-stream fork / join) cost ~70 µs for 13 MB of data.
// Here one persistent grid runs every phase of the plan in order -- leaf projection, the upsweep
// levels, all coupling rows, the downsweep levels, the leaves (expansion + dense + epilogue) --
// with a grid-wide barrier between dependent phases.
// One warp per task, the SIMT engine at nv = 1; FP64 / FP32; one rank.
#pragma once
#include "h2_kernels.cuh"

#include <cooperative_groups.h>

namespace h2 {

template <typename T, int RPLK, int RPLM>
__global__ void __launch_bounds__(256) k_mono(const __grid_constant__ MonoPlan mp, const Task *__restrict__ tasks,
                                              const Blk *__restrict__ blks, T *xh, T *yh, int64_t plane,
                                              const CallArgs<T> *__restrict__ args)
{
    namespace cg = cooperative_groups;
    using EK = Simt<T, RPLK, 1>;
    using EM = Simt<T, RPLM, 1>;
    __shared__ __align__(16) T zsh[8][KMAX];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const T *__restrict__ X = args->X;
    T *__restrict__ Y = args->Y;
    const int64_t ldx = args->ldx;
    const T alpha = args->alpha, beta = args->beta;
    for (int p = 0; p < mp.nph; ++p) {
        const MonoPhase ph = mp.ph[p];
        for (int w = gw; w < ph.n; w += nw) {
            const Task tk = tasks[ph.t0 + w];
            if (ph.kind == MONO_UPLEAF) {
                typename EK::Acc acc;
                acc_zero(acc, lane);
                const Blk b = blks[tk.blk0];
                EK::block(acc, static_cast<const T *>(b.A), tk.r, tk.c, X + b.x, ldx, b.xrows, 1, lane);
                acc_store(acc, xh + tk.out, plane, tk.r, 1, lane);
            } else if (ph.kind == MONO_LEAF) {
                const Task dk = tasks[mp.dense_t0 + w];
                const bool hasE = tk.flags & TF_HAS_E;
                const Blk bU = blks[tk.blk0 + (hasE ? 1 : 0)];
                typename EK::Acc z;
                acc_load(z, yh + bU.x, plane, mp.k, 1, lane);
                if (hasE) {
                    const Blk bE = blks[tk.blk0];
                    EK::block(z, static_cast<const T *>(bE.A), mp.k, mp.kp, yh + bE.x, plane, bE.xrows, 1, lane);
                }
                __syncwarp();
                acc_store(z, &zsh[wid][0], (int64_t)KMAX, mp.k, 1, lane);
                __syncwarp();
                typename EM::Acc acc;
                acc_zero(acc, lane);
                EM::block(acc, static_cast<const T *>(bU.A), tk.r, mp.k, &zsh[wid][0], (int64_t)KMAX, mp.k, 1, lane);
                for (int bi = 0; bi < dk.nblk; ++bi) {
                    const Blk b = blks[dk.blk0 + bi];
                    EM::block(acc, static_cast<const T *>(b.A), dk.r, dk.c, X + b.x, ldx, b.xrows, 1, lane);
                }
                T *Yb = Y + tk.out;
                const int rows = tk.rows;
                acc.each(lane, [&](int row, int n, auto &v) {
                    if (row < rows && n < 1) Yb[row] = (beta == T(0)) ? alpha * v : fma(alpha, (T)v, beta * Yb[row]);
                });
                __syncwarp();
            } else {
                // transfer or coupling row: out (+)= sum_b A_b x_b, x^ -> x^ (up), x^ -> y^ (coupling),
                // y^ -> y^ (down, accumulating)
                const T *src = (ph.kind == MONO_DOWN) ? yh : xh;
                T *dst = (ph.kind == MONO_UP) ? xh : yh;
                typename EK::Acc acc;
                if (ph.kind == MONO_DOWN) acc_load(acc, dst + tk.out, plane, tk.r, 1, lane);
                else acc_zero(acc, lane);
                for (int bi = 0; bi < tk.nblk; ++bi) {
                    const Blk b = blks[tk.blk0 + bi];
                    EK::block(acc, static_cast<const T *>(b.A), tk.r, tk.c, src + b.x, plane, b.xrows, 1, lane);
                }
                acc_store(acc, dst + tk.out, plane, tk.r, 1, lane);
            }
        }
        if (ph.sync) cg::this_grid().sync();
    }
}

// Cooperative launch of k_mono: every CTA resident at once (the grid barrier needs it).
template <typename T>
cudaError_t launch_mono(const MonoPlan &mp, const Task *tasks, const Blk *blks, T *xh, T *yh, int64_t plane,
                        const CallArgs<T> *args, int kmax, int m, int nsm, cudaStream_t s)
{
    auto go = [&](auto kern) -> cudaError_t {
        int per = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0);
        if (e != cudaSuccess) return e;
        const int grid = (per < 2 ? per : 2) * nsm;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, mp, tasks, blks, xh, yh, plane, args);
    };
    cudaError_t e;
    if (kmax <= 32) e = m <= 32 ? go(k_mono<T, 1, 1>) : go(k_mono<T, 1, 2>);
    else            e = m <= 32 ? go(k_mono<T, 2, 1>) : go(k_mono<T, 2, 2>);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace h2
