// h2_kernels.cuh -- sm_100a kernels of the H^2 matvec hot path.
// Included by the h2_k_*.cu translation units, each instantiating a subset of the launchers
// for one element type (parallel compilation).
//
// Every phase is a set of warp tasks over a static plan built once by h2_create (the paper's
// per-level marshaling, done at setup instead of per call).  A task owns one
// output node (row-owner computes: no atomics, no conflict batches) and
// accumulates   y (r x nv) += sum_b A_b (r x c) x_b (c x nv),   A_b streamed once from HBM.
//
// Two warp engines compute the block products:
//   Simt  (any T, nv chunks of 1..16): lanes <-> output rows (RPL rows per lane); each A column
//         is one coalesced warp load (evict-first); the x operand is held distributed in
//         registers (lane j holds rows j, j+32) and broadcast with shuffles.
//   Mma   (double, nv chunks of 8 / 16): FP64 tensor-core tiles mma.sync.m8n8k4.f64 (SASS DMMA);
//         A fragments straight from global memory (each element loaded once), B fragments from
//         the x^ / X source (L2) or from shared memory, accumulators in registers across all
//         blocks of the task.
//
//   up_leaf   x^_s = V_s^T x_s                         PAPER.md:239, 262 (alg:upsweep2 line 3)
//   rows/W    x^_p = F_{c1}^T x^_{c1} + F_{c2}^T x^_{c2} PAPER.md:241-253, 267-268
//   rows/W    y^_t = sum_s S_ts x^_s  (all levels)      PAPER.md:328-331, 344-356 (alg:mult)
//   rows/A    y^_c += E_c y^_parent                     PAPER.md:389-399, 408-412 (alg:downsweep)
//   leaf      z_t = y^_t + E_t y^_parent ; y_t = U_t z_t + sum_s D_ts x_s ;
//             Y = alpha y + beta Y                      PAPER.md:399, 414, 225; reading R11/R12
#include "h2_internal.h"

#include <algorithm>
#include <utility>
#include <cstdlib>
#include <type_traits>

namespace h2 {

constexpr unsigned FULL = 0xffffffffu;
constexpr size_t SWEEP_STAGE_SMEM = 200 * 1024;   // dynamic smem cap of a staged k_sweep CTA
#ifndef H2_APF
#define H2_APF 4          // k-steps of L2 prefetch ahead of the DMMA A-fragment loads (0 = off;
                          // the same prefetch in the SIMT streams measured slower)
#endif
constexpr int XCAP_BYTES = 4096;   // per-warp staging of the stacked x in the Simt stream
constexpr int ZLD = KMAX + 4;   // smem leading dimension of the z hand-over (2 wavefronts per
                                // DMMA B-fragment load: no extra bank conflicts)

template <typename T>
__device__ __forceinline__ T ld_stream(const T *p) { return __ldcs(p); }

// =========================================================================== Simt engine
template <typename T, int RPL, int NVB>
struct SimtAcc {
    T v[RPL][NVB];
    template <typename F>
    __device__ __forceinline__ void each(int lane, F f) {
#pragma unroll
        for (int ri = 0; ri < RPL; ++ri)
#pragma unroll
            for (int n = 0; n < NVB; ++n) f(lane + 32 * ri, n, v[ri][n]);
    }
};

// x operand rows lane / lane+32 of vectors [0, nvc); rows >= xrows -> 0
template <typename T, int NVB>
__device__ __forceinline__ void simt_load_x(T (&x0)[NVB], T (&x1)[NVB], const T *__restrict__ src,
                                            int64_t ld, int xrows, int nvc, int lane)
{
#pragma unroll
    for (int n = 0; n < NVB; ++n) {
        x0[n] = (n < nvc && lane < xrows) ? src[lane + n * ld] : T(0);
        x1[n] = (n < nvc && lane + 32 < xrows) ? src[lane + 32 + n * ld] : T(0);
    }
}

template <typename T, int RPL, int NVB, int U>
__device__ __forceinline__ void simt_cols(SimtAcc<T, RPL, NVB> &acc, const T *__restrict__ A, int r,
                                          int j, const T (&x0)[NVB], const T (&x1)[NVB], int lane)
{
    T a[U][RPL];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int ri = 0; ri < RPL; ++ri) {
            int i = lane + 32 * ri;
            a[u][ri] = (i < r) ? ld_stream(A + (int64_t)(j + u) * r + i) : T(0);
        }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int jj = j + u;                       // warp-uniform
#pragma unroll
        for (int n = 0; n < NVB; ++n) {
            T xv = __shfl_sync(FULL, jj < 32 ? x0[n] : x1[n], jj & 31);
#pragma unroll
            for (int ri = 0; ri < RPL; ++ri) acc.v[ri][n] = fma(a[u][ri], xv, acc.v[ri][n]);
        }
    }
}

// acc += A (r x c, col-major) * x (c x nvc) with x in registers (x0/x1)
// column unroll of the Simt engines: 16 (2 CTAs/SM budget) or 8 (3-4 CTAs/SM budget)
template <int RPL, int NVB>
__host__ __device__ constexpr int simt_unroll() { return NVB <= 2 ? 8 : 16; }

template <typename T, int RPL, int U>
__device__ __forceinline__ void simt_load_cols(T (&a)[U][RPL], const T *__restrict__ A, int r, int j, int K,
                                               int lane)
{
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int ri = 0; ri < RPL; ++ri) {
            const int i = lane + 32 * ri;
            a[u][ri] = (i < r && j + u < K) ? ld_stream(A + (int64_t)(j + u) * r + i) : T(0);
        }
}

template <typename T, int RPL, int NVB, int U>
__device__ __forceinline__ void simt_fma_cols_regs(SimtAcc<T, RPL, NVB> &acc, const T (&a)[U][RPL], int j,
                                                   const T (&x0)[NVB], const T (&x1)[NVB])
{
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int jj = j + u;                       // warp-uniform; columns >= c have a == 0
#pragma unroll
        for (int n = 0; n < NVB; ++n) {
            T xv = __shfl_sync(FULL, jj < 32 ? x0[n] : x1[n], jj & 31);
#pragma unroll
            for (int ri = 0; ri < RPL; ++ri) acc.v[ri][n] = fma(a[u][ri], xv, acc.v[ri][n]);
        }
    }
}

// acc += A (r x c, col-major) * x (c x nvc) with x in registers (x0/x1), columns in batches
// (a two-group register pipeline here measured slower at nv = 1: the single-block tasks are
// short and the deeper pipeline spilled at the 3-4 CTA/SM register budget)
template <typename T, int RPL, int NVB, bool WIDE = false>
__device__ __forceinline__ void simt_block_regs(SimtAcc<T, RPL, NVB> &acc, const T *__restrict__ A,
                                                int r, int c, const T (&x0)[NVB], const T (&x1)[NVB],
                                                int lane)
{
    if (WIDE && RPL == 1 && NVB == 1 && c <= 32) {
        // small block (a transfer or coupling block, k <= 32): every column load in flight at
        // once -- one HBM round trip per block instead of one per batch of 8 columns
        T a[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) a[u] = (lane < r && u < c) ? ld_stream(A + (int64_t)u * r + lane) : T(0);
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const T xv = __shfl_sync(FULL, x0[0], u);
            acc.v[0][0] = fma(a[u], xv, acc.v[0][0]);
        }
        return;
    }
    int j = 0;
    if (simt_unroll<RPL, NVB>() >= 16)
        for (; j + 16 <= c; j += 16) simt_cols<T, RPL, NVB, 16>(acc, A, r, j, x0, x1, lane);
    for (; j + 8 <= c; j += 8) simt_cols<T, RPL, NVB, 8>(acc, A, r, j, x0, x1, lane);
    if (j + 4 <= c) { simt_cols<T, RPL, NVB, 4>(acc, A, r, j, x0, x1, lane); j += 4; }
    for (; j < c; ++j) simt_cols<T, RPL, NVB, 1>(acc, A, r, j, x0, x1, lane);
}

template <typename T, int RPL, int NVB, bool WIDE = false>
__device__ __forceinline__ void simt_block(SimtAcc<T, RPL, NVB> &acc, const T *__restrict__ A, int r,
                                           int c, const T *__restrict__ src, int64_t ld, int xrows,
                                           int nvc, int lane)
{
    T x0[NVB], x1[NVB];
    simt_load_x<T, NVB>(x0, x1, src, ld, xrows, nvc, lane);
    simt_block_regs<T, RPL, NVB, WIDE>(acc, A, r, c, x0, x1, lane);
}

// =========================================================================== Mma engine
template <int MT, int NT>
struct MmaAcc {
    double v[MT][NT][2];
    template <typename F>
    __device__ __forceinline__ void each(int lane, F f) {
        const int g = lane >> 2, t = lane & 3;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < 2; ++i) f(mt * 8 + g, nt * 8 + 2 * t + i, v[mt][nt][i]);
    }
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// acc += A (r x c, col-major, global) * B (c x nvc; element (j, n) at src[j + n*ld], global or
// shared).  Fragments (PTX m8n8k4 .f64): A row = 8mt + lane/4, col = 4ks + lane%4;
// B row = 4ks + lane%4, col = 8nt + lane/4; rows >= xrows / cols >= nvc read as 0.
template <int MT, int NT, bool A_STREAM>
__device__ __forceinline__ void mma_block_step(double (&a)[MT], double (&b)[NT], const double *__restrict__ A,
                                               int r, int c, const double *src, int64_t ld, int xrows,
                                               int nvc, int ks, int g, int t, int lda)
{
    const int col = ks * 4 + t;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        const int row = mt * 8 + g;
        const double *p = A + (int64_t)col * lda + row;
        a[mt] = (row < r && col < c) ? (A_STREAM ? ld_stream(p) : *p) : 0.0;
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        const int n = nt * 8 + g;
        b[nt] = (col < xrows && n < nvc) ? src[col + n * ld] : 0.0;
    }
}

// acc += A (r x c, col-major, global) * B (c x nvc; element (j, n) at src[j + n*ld], global or
// shared).  Fragments (PTX m8n8k4 .f64): A row = 8mt + lane/4, col = 4ks + lane%4;
// B row = 4ks + lane%4, col = 8nt + lane/4; rows >= xrows / cols >= nvc read as 0.
// Two fragment sets in flight (loads of k-step ks+2 issued behind the DMMAs of k-step ks).
template <int MT, int NT, bool A_STREAM>
__device__ __forceinline__ void mma_block(MmaAcc<MT, NT> &acc, const double *__restrict__ A, int r,
                                          int c, const double *src, int64_t ld, int xrows, int nvc,
                                          int lane, int lda = -1)
{
    const int g = lane >> 2, t = lane & 3;
    if (lda < 0) lda = r;
    const int ksn = (c + 3) >> 2;
    constexpr int PD = MT <= 4 ? 3 : 2;      // fragment sets in flight (see mma_stream)
    double a[PD][MT], b[PD][NT];
#pragma unroll
    for (int p = 0; p < PD; ++p)
        mma_block_step<MT, NT, A_STREAM>(a[p], b[p], A, r, c, src, ld, xrows, nvc, p, g, t, lda);
    int ks = 0;
    for (; ks + PD <= ksn; ks += PD) {
#pragma unroll
        for (int p = 0; p < PD; ++p) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma(acc.v[mt][nt], a[p][mt], b[p][nt]);
            mma_block_step<MT, NT, A_STREAM>(a[p], b[p], A, r, c, src, ld, xrows, nvc, ks + PD + p, g, t, lda);
        }
    }
#pragma unroll
    for (int p = 0; p < PD; ++p)
        if (ks + p < ksn) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma(acc.v[mt][nt], a[p][mt], b[p][nt]);
        }
}

// =========================================================================== streaming rows
// A task whose blocks A_b are CONTIGUOUS (flag TF_ACONTIG: A_b = A_0 + b r c, e.g. the CSR run
// of a coupling row, the dense row of a leaf, the two child transfers of a parent) is one
// GEMM  y (r x nv) += [A_1 .. A_n] (r x n c) [x_1; ..; x_n] (n c x nv):  its A columns are
// streamed back to back with no per-block dependent descriptor loads, and the stacked x is
// gathered per block from its own source (x^ slots, X leaf rows or the halo buffer).
template <typename T>
struct Src {
    const T *pos;     // x >= 0: pos + x, leading dimension pos_ld (or the block's xld)
    int64_t pos_ld;
    const T *neg;     // x < 0: neg + (-x - 1), leading dimension xld (halo buffer)
    int n0;           // first vector of the current chunk
};

template <typename T>
__device__ __forceinline__ const T *resolve(const Src<T> &s, int64_t x, int32_t xld, int64_t &ld)
{
    if (x >= 0) { ld = xld ? (int64_t)xld : s.pos_ld; return s.pos + x + s.n0 * ld; }
    ld = xld;
    return s.neg + (-x - 1) + s.n0 * ld;
}

// acc += A (r x K, col-major, contiguous) * xs (K x nvc in shared memory, ld xld): columns in
// groups of U with two groups in flight (the loads of group g+2 are issued behind the FMAs of
// group g), so each warp keeps 2U column loads outstanding without exposing HBM latency.
// x row j (NVB vectors, contiguous: the stream stages x vector-fastest) into registers with 16-byte
// shared loads (broadcast: every lane reads the same row) -- NVB / (16 / sizeof(T)) loads per column
// instead of NVB scalar loads
template <typename T, int NVB>
__device__ __forceinline__ void smem_row(T (&xv)[NVB], const T *p)
{
    if constexpr ((NVB * sizeof(T)) % 16 == 0) {
#pragma unroll
        for (int n = 0; n < NVB; n += 16 / (int)sizeof(T)) {
            const float4 q = *reinterpret_cast<const float4 *>(p + n);
            const T *qt = reinterpret_cast<const T *>(&q);
#pragma unroll
            for (int i = 0; i < 16 / (int)sizeof(T); ++i) xv[n + i] = qt[i];
        }
    } else {
#pragma unroll
        for (int n = 0; n < NVB; ++n) xv[n] = p[n];
    }
}

// acc += a (U columns in registers) * xs rows j .. j+U-1 (row e at xs + e * NVB; rows >= K are zero)
template <typename T, int RPL, int NVB, int U>
__device__ __forceinline__ void simt_fma_cols(SimtAcc<T, RPL, NVB> &acc, const T (&a)[U][RPL], int j, int K,
                                              const T *xs, int xld)
{
#pragma unroll
    for (int u = 0; u < U; ++u) {
        T xv[NVB];
        smem_row<T, NVB>(xv, xs + (int64_t)(j + u) * NVB);
#pragma unroll
        for (int n = 0; n < NVB; ++n)
#pragma unroll
            for (int ri = 0; ri < RPL; ++ri) acc.v[ri][n] = fma(a[u][ri], xv[n], acc.v[ri][n]);
    }
}

template <typename T, int RPL, int NVB>
__device__ __forceinline__ void simt_cols_pipelined(SimtAcc<T, RPL, NVB> &acc, const T *__restrict__ A, int r,
                                                    int K, const T *xs, int xld, int lane)
{
    constexpr int U = RPL == 1 ? 8 : 4;
    T a0[U][RPL], a1[U][RPL];
    simt_load_cols<T, RPL, U>(a0, A, r, 0, K, lane);
    simt_load_cols<T, RPL, U>(a1, A, r, U, K, lane);
    for (int j = 0; j < K; j += 2 * U) {
        simt_fma_cols<T, RPL, NVB, U>(acc, a0, j, K, xs, xld);
        simt_load_cols<T, RPL, U>(a0, A, r, j + 2 * U, K, lane);
        simt_fma_cols<T, RPL, NVB, U>(acc, a1, j + U, K, xs, xld);
        simt_load_cols<T, RPL, U>(a1, A, r, j + 3 * U, K, lane);
    }
}

template <typename T, int RPL, int NVB>
__device__ __forceinline__ void simt_stream(SimtAcc<T, RPL, NVB> &acc, const T *__restrict__ A0, int r,
                                            int c, int nblk, const Blk *__restrict__ blks,
                                            const Src<T> &src, int nvc, int lane, T *xs, int xcap)
{
    int per = (xcap - 16 * NVB) / (c * NVB);          // room for the 2U zero rows of the tail
    per = per < 1 ? 1 : (per > 32 ? 32 : per);
    for (int b0 = 0; b0 < nblk; b0 += per) {
        const int nb = min(per, nblk - b0);
        const int K = nb * c;
        int64_t xo = 0;
        int xr = 0, xl = 0;
        if (lane < nb) {
            const Blk b = blks[b0 + lane];
            xo = b.x; xr = b.xrows; xl = b.xld;
        }
        __syncwarp();
        for (int e0 = 0; e0 < K; e0 += 32) {           // gather the stacked x of the chunk
            const int e = e0 + lane;
            const int bb = min(e / c, nb - 1), j = e - bb * c;
            const int64_t bxo = __shfl_sync(FULL, xo, bb);
            const int bxr = __shfl_sync(FULL, xr, bb), bxl = __shfl_sync(FULL, xl, bb);
            if (e < K) {
                int64_t ld;
                const T *p = resolve(src, bxo, bxl, ld);
#pragma unroll
                for (int n = 0; n < NVB; ++n) xs[e * NVB + n] = (j < bxr && n < nvc) ? p[j + n * ld] : T(0);
            }
        }
        // rows K .. K + 2U - 1 are read by the pipelined tail (their A columns are zero): keep them 0
        constexpr int UP = RPL == 1 ? 8 : 4;
        for (int e = K * NVB + lane; e < (K + 2 * UP) * NVB; e += 32) xs[e] = T(0);
        __syncwarp();
        simt_cols_pipelined<T, RPL, NVB>(acc, A0 + (int64_t)b0 * r * c, r, K, xs, K, lane);
        __syncwarp();
    }
}

struct MmaDesc {
    const double *p;
    int64_t ld;
    int32_t xrows;
    int32_t pad;
};

template <int MT, int NT>
struct MmaFrag {
    double a[MT], b[NT];
};

// Load cursor of the stacked-B operand: lane's row j of block bb (descriptor d)
struct BCursor {
    int j, bb;
    MmaDesc d;
};

template <int MT, int NT>
__device__ __forceinline__ void mma_load_step(MmaFrag<MT, NT> &f, const double *__restrict__ A, int r, int K,
                                              int ks, int g, int t, const BCursor &cur, int nvc, int lda)
{
    const int col = ks * 4 + t;
    if (H2_APF > 0) {
        // L2 prefetch of the A columns H2_APF k-steps ahead: lanes g < ceil(8 MT / 16) each
        // touch one 128-byte line of their column (no registers, no wait)
        const int pcol = (ks + H2_APF) * 4 + t;
        const int prow = g * 16;
        if (pcol < K && prow < r && g < (MT * 8 + 15) / 16)
            asm volatile("prefetch.global.L2 [%0];\n" ::"l"(A + (int64_t)pcol * lda + prow));
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
        const int row = mt * 8 + g;
        f.a[mt] = (row < r && col < K) ? ld_stream(A + (int64_t)col * lda + row) : 0.0;
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        const int n = nt * 8 + g;
        f.b[nt] = (col < K && cur.j < cur.d.xrows && n < nvc) ? cur.d.p[cur.j + n * cur.d.ld] : 0.0;
    }
}

__device__ __forceinline__ void bcursor_advance(BCursor &cur, int c, int nb, const MmaDesc *ds)
{
    cur.j += 4;
    if (cur.j >= c) {
        do { cur.j -= c; ++cur.bb; } while (cur.j >= c);
        cur.d = ds[min(cur.bb, nb - 1)];
    }
}

template <int MT, int NT>
__device__ __forceinline__ void mma_frag_mma(MmaAcc<MT, NT> &acc, const MmaFrag<MT, NT> &f)
{
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma(acc.v[mt][nt], f.a[mt], f.b[nt]);
}

// DMMA over a contiguous run with an explicit two-stage register pipeline: the fragments of
// k-step ks+2 are loaded before the tensor-core work of k-step ks is issued, so HBM latency is
// covered by two k-steps of DMMA instead of being exposed every k-step (ncu round 1: the
// unpipelined loop kept the FP64 tensor pipe 45 % busy at 54 % DRAM).
template <int MT, int NT>
__device__ __forceinline__ void mma_stream(MmaAcc<MT, NT> &acc, const double *__restrict__ A0, int r,
                                           int c, int nblk, const Blk *__restrict__ blks,
                                           const Src<double> &src, int nvc, int lane, MmaDesc *ds, int lda = -1)
{
    const int g = lane >> 2, t = lane & 3;
    if (lda < 0) lda = r;
    for (int b0 = 0; b0 < nblk; b0 += 32) {
        const int nb = min(32, nblk - b0);
        const int K = nb * c;
        __syncwarp();
        if (lane < nb) {
            const Blk b = blks[b0 + lane];
            int64_t ld;
            const double *p = resolve(src, b.x, b.xld, ld);
            ds[lane] = MmaDesc{p, ld, b.xrows, 0};
        }
        __syncwarp();
        const double *A = A0 + (int64_t)b0 * lda * c;
        BCursor cur;
        cur.j = t;
        cur.bb = 0;
        while (cur.j >= c) { cur.j -= c; ++cur.bb; }
        cur.d = ds[min(cur.bb, nb - 1)];
        const int ksn = (K + 3) >> 2;
        // PD fragment sets in flight (k-steps ks .. ks+PD-1); after the DMMAs of a set are issued,
        // the set is refilled with the k-step PD ahead
        constexpr int PD = MT <= 4 ? 3 : 2;
        MmaFrag<MT, NT> f[PD];
#pragma unroll
        for (int p = 0; p < PD; ++p) {
            mma_load_step(f[p], A, r, K, p, g, t, cur, nvc, lda);
            bcursor_advance(cur, c, nb, ds);
        }
        int ks = 0;
        for (; ks + PD <= ksn; ks += PD) {
#pragma unroll
            for (int p = 0; p < PD; ++p) {
                mma_frag_mma(acc, f[p]);
                mma_load_step(f[p], A, r, K, ks + PD + p, g, t, cur, nvc, lda);
                bcursor_advance(cur, c, nb, ds);
            }
        }
#pragma unroll
        for (int p = 0; p < PD; ++p)
            if (ks + p < ksn) mma_frag_mma(acc, f[p]);
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

// =========================================================================== common helpers
template <typename Acc>
__device__ __forceinline__ void acc_zero(Acc &acc, int lane)
{
    acc.each(lane, [](int, int, auto &v) { v = 0; });
}

template <typename Acc, typename T>
__device__ __forceinline__ void acc_load(Acc &acc, const T *base, int64_t ld, int r, int nvc, int lane)
{
    acc.each(lane, [&](int row, int n, auto &v) { v = (row < r && n < nvc) ? base[row + n * ld] : T(0); });
}

template <typename Acc, typename T>
__device__ __forceinline__ void acc_store(Acc &acc, T *base, int64_t ld, int r, int nvc, int lane)
{
    acc.each(lane, [&](int row, int n, auto &v) {
        if (row < r && n < nvc) base[row + n * ld] = v;
    });
}

// Engine selector: Simt<T, RPL, NVB> or Mma<MT, NT> behind one interface
template <typename T, int RPL, int NVB>
struct Simt {
    using Acc = SimtAcc<T, RPL, NVB>;
    static constexpr int NV = NVB;
    // CTAs per SM the register budget is sized for (__launch_bounds__ min blocks): the nv <= 2
    // streaming engines are latency-bound at 2 CTAs (16 warps, 25 % occupancy; ncu round 1)
    static constexpr int MINB = NVB <= 2 ? (RPL == 1 ? 4 : 3) : 2;
    static constexpr bool SIMT1 = (RPL == 1 && NVB == 1);
    static constexpr bool MMA = false;
    // per-warp smem for the stream staging: >= one 64-column block of x plus the 16 zero tail rows
    static constexpr int SCRATCH = (int)(80 * NVB * sizeof(T)) > XCAP_BYTES ? (int)(80 * NVB * sizeof(T)) : XCAP_BYTES;
    __device__ static void block(Acc &acc, const T *A, int r, int c, const T *src, int64_t ld, int xrows,
                                 int nvc, int lane, int lda = -1)
    { simt_block<T, RPL, NVB>(acc, A, r, c, src, ld, xrows, nvc, lane); }
    // all columns of a small block in flight at once (needs ~2x the registers: k_sweep only)
    __device__ static void block_wide(Acc &acc, const T *A, int r, int c, const T *src, int64_t ld, int xrows,
                                      int nvc, int lane)
    { simt_block<T, RPL, NVB, true>(acc, A, r, c, src, ld, xrows, nvc, lane); }
    __device__ static void stream(Acc &acc, const T *A0, int r, int c, int nblk, const Blk *blks,
                                  const Src<T> &src, int nvc, int lane, void *scratch)
    { simt_stream<T, RPL, NVB>(acc, A0, r, c, nblk, blks, src, nvc, lane, (T *)scratch, SCRATCH / (int)sizeof(T)); }
    // acc += As (r x c, col-major ld r, shared) * xs (c x nvc, ld xld, shared): outer products,
    // column j of As and row j of xs per step (RPL + NVB shared loads for RPL x NVB FMAs)
    __device__ static void smem_block(Acc &acc, const T *As, int r, int c, const T *xs, int xld, int nvc, int lane)
    {
#pragma unroll 4
        for (int j = 0; j < c; ++j) {
            T a[RPL];
#pragma unroll
            for (int ri = 0; ri < RPL; ++ri) a[ri] = (lane + 32 * ri < r) ? As[j * r + lane + 32 * ri] : T(0);
#pragma unroll
            for (int n = 0; n < NVB; ++n) {
                const T xv = n < nvc ? xs[j + n * xld] : T(0);
#pragma unroll
                for (int ri = 0; ri < RPL; ++ri) acc.v[ri][n] = fma(a[ri], xv, acc.v[ri][n]);
            }
        }
    }
};

template <int MT, int NT>
struct Mma {
    using Acc = MmaAcc<MT, NT>;
    static constexpr int NV = 8 * NT;
    static constexpr int MINB = 2;
    static constexpr bool SIMT1 = false;
    static constexpr bool MMA = true;
    static constexpr int SCRATCH = 32 * sizeof(MmaDesc);
    __device__ static void block(Acc &acc, const double *A, int r, int c, const double *src, int64_t ld,
                                 int xrows, int nvc, int lane, int lda = -1)
    { mma_block<MT, NT, true>(acc, A, r, c, src, ld, xrows, nvc, lane, lda); }
    __device__ static void block_wide(Acc &acc, const double *A, int r, int c, const double *src, int64_t ld,
                                      int xrows, int nvc, int lane)
    { mma_block<MT, NT, true>(acc, A, r, c, src, ld, xrows, nvc, lane); }
    __device__ static void stream(Acc &acc, const double *A0, int r, int c, int nblk, const Blk *blks,
                                  const Src<double> &src, int nvc, int lane, void *scratch, int lda = -1)
    { mma_stream<MT, NT>(acc, A0, r, c, nblk, blks, src, nvc, lane, (MmaDesc *)scratch, lda); }
    __device__ static void smem_block(Acc &acc, const double *As, int r, int c, const double *xs, int xld, int nvc,
                                      int lane)
    { mma_block<MT, NT, false>(acc, As, r, c, xs, xld, c, nvc, lane, r); }
};

// =========================================================================== FP32 tensor engine
// FP32 on the tensor cores by the 3xTF32 split: a = a_hi + a_lo with a_hi =
// tf32(a), a_lo = tf32(a - a_hi); a b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi (the dropped a_lo b_lo is
// ~2^-22 relative), accumulated in FP32 by mma.sync.m16n8k8.tf32 -- FP32-level accuracy (parity
// <= 1e-5 against the FP64 oracle) at tensor-core throughput, so FP32 at nv >= 5 is bound by HBM
// instead of by FFMA issue (the SIMT stream reached 0.32-0.37 of HBM on cfg5).
// Fragments (PTX m16n8k8 .tf32, g = lane / 4, t = lane % 4):
//   A 16x8: a0 (g, t), a1 (g+8, t), a2 (g, t+4), a3 (g+8, t+4);  B 8x8: b0 (t, g), b1 (t+4, g);
//   C 16x8: c0 (g, 2t), c1 (g, 2t+1), c2 (g+8, 2t), c3 (g+8, 2t+1).
template <int MT, int NT>
struct TfAcc {
    float v[MT][NT][4];
    template <typename F>
    __device__ __forceinline__ void each(int lane, F f) {
        const int g = lane >> 2, t = lane & 3;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < 4; ++i) f(mt * 16 + g + (i >> 1) * 8, nt * 8 + 2 * t + (i & 1), v[mt][nt][i]);
    }
};

__device__ __forceinline__ void tf32_split(float x, uint32_t &hi, uint32_t &lo)
{
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(hi) : "f"(x));
    const float r = x - __uint_as_float(hi);
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(lo) : "f"(r));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};\n"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int MT, int NT>
struct TfFrag {
    float a[MT][4], b[NT][2];
};

// fragments of k-step ks (columns 8ks .. 8ks+7) of A (r x c, col-major, lda) and B (c x nvc at
// src[j + n ld]; rows >= xrows and vectors >= nvc are zero)
template <int MT, int NT, bool A_STREAM>
__device__ __forceinline__ void tf_load(TfFrag<MT, NT> &f, const float *__restrict__ A, int r, int c, int lda,
                                        const float *src, int64_t ld, int xrows, int nvc, int ks, int g, int t)
{
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int row = mt * 16 + g + (i & 1) * 8, col = ks * 8 + t + (i >> 1) * 4;
            const float *p = A + (int64_t)col * lda + row;
            f.a[mt][i] = (row < r && col < c) ? (A_STREAM ? __ldcs(p) : *p) : 0.f;
        }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int row = ks * 8 + t + i * 4, n = nt * 8 + g;
            f.b[nt][i] = (row < xrows && row < c && n < nvc) ? src[row + n * ld] : 0.f;
        }
}

template <int MT, int NT>
__device__ __forceinline__ void tf_mma(TfAcc<MT, NT> &acc, const TfFrag<MT, NT> &f)
{
    uint32_t ah[MT][4], al[MT][4], bh[NT][2], bl[NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) tf32_split(f.a[mt][i], ah[mt][i], al[mt][i]);
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) tf32_split(f.b[nt][i], bh[nt][i], bl[nt][i]);
    // the three products of this k-step go into a zeroed tile and are added to the accumulator with
    // IEEE FP32 adds: the tensor cores' own accumulation is not round-to-nearest, and its bias over
    // hundreds of k-steps of a coupling row measured 1.6e-5 (cfg5) against the 1e-5 bar
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            float d[4] = {0.f, 0.f, 0.f, 0.f};
            mma_tf32(d, al[mt], bh[nt][0], bh[nt][1]);     // small terms first
            mma_tf32(d, ah[mt], bl[nt][0], bl[nt][1]);
            mma_tf32(d, ah[mt], bh[nt][0], bh[nt][1]);
#pragma unroll
            for (int i = 0; i < 4; ++i) acc.v[mt][nt][i] += d[i];
        }
}

// acc += A (r x c) B (c x nvc), fragments of k-step ks+1 loaded behind the MMAs of k-step ks
template <int MT, int NT, bool A_STREAM>
__device__ __forceinline__ void tf_block(TfAcc<MT, NT> &acc, const float *__restrict__ A, int r, int c, int lda,
                                         const float *src, int64_t ld, int xrows, int nvc, int lane)
{
    const int g = lane >> 2, t = lane & 3;
    const int ksn = (c + 7) >> 3;
    TfFrag<MT, NT> f[2];
    tf_load<MT, NT, A_STREAM>(f[0], A, r, c, lda, src, ld, xrows, nvc, 0, g, t);
    for (int ks = 0; ks < ksn; ++ks) {
        if (ks + 1 < ksn) tf_load<MT, NT, A_STREAM>(f[(ks + 1) & 1], A, r, c, lda, src, ld, xrows, nvc, ks + 1, g, t);
        tf_mma(acc, f[ks & 1]);
    }
}

template <int MT, int NT>
struct Tf3 {
    using Acc = TfAcc<MT, NT>;
    static constexpr int NV = 8 * NT;
    static constexpr int MINB = 2;
    static constexpr bool SIMT1 = false;
    static constexpr bool MMA = true;
    static constexpr int SCRATCH = 32;
    __device__ static void block(Acc &acc, const float *A, int r, int c, const float *src, int64_t ld, int xrows,
                                 int nvc, int lane, int lda = -1)
    { tf_block<MT, NT, true>(acc, A, r, c, lda < 0 ? r : lda, src, ld, xrows, nvc, lane); }
    __device__ static void block_wide(Acc &acc, const float *A, int r, int c, const float *src, int64_t ld, int xrows,
                                      int nvc, int lane)
    { tf_block<MT, NT, true>(acc, A, r, c, r, src, ld, xrows, nvc, lane); }
    // a contiguous run of blocks: one block at a time, each with its own x source
    __device__ static void stream(Acc &acc, const float *A0, int r, int c, int nblk, const Blk *blks,
                                  const Src<float> &src, int nvc, int lane, void *, int lda = -1)
    {
        const int la = lda < 0 ? r : lda;
        for (int b = 0; b < nblk; ++b) {
            const Blk bk = blks[b];
            int64_t ld;
            const float *x = resolve(src, bk.x, bk.xld, ld);
            tf_block<MT, NT, true>(acc, A0 + (int64_t)b * la * c, r, c, la, x, ld, bk.xrows, nvc, lane);
        }
    }
    __device__ static void smem_block(Acc &acc, const float *As, int r, int c, const float *xs, int xld, int nvc,
                                      int lane)
    { tf_block<MT, NT, false>(acc, As, r, c, r, xs, xld, c, nvc, lane); }
};

// ---------------------------------------------------------------------------------------
// Upsweep leaves: x^_s (k x nv) = Vt_s (k x m) x_s (m x nv), Vt = V^T re-laid out at create.
template <typename T, typename Eng>
__global__ void __launch_bounds__(WPB * 32, Eng::MINB < 3 ? Eng::MINB : 3)
k_up_leaf(const Task *__restrict__ tasks, int ntask, const Blk *__restrict__ blks,
          const CallArgs<T> *__restrict__ args, T *__restrict__ xh, int64_t xh_ld, int nv)
{
    const int lane = threadIdx.x & 31;
    // one warp per (leaf, vector chunk) when the launcher sized the grid for it (see k_rows)
    const int nch = (nv + Eng::NV - 1) / Eng::NV;
    const int S = (int64_t)ntask * nch <= (int64_t)gridDim.x * WPB ? nch : 1;
    const int vt = blockIdx.x * WPB + (threadIdx.x >> 5);
    if (vt >= ntask * S) return;
    const int task = vt / S;
    const int ch0 = S == 1 ? 0 : vt - task * S, ch1 = S == 1 ? nch : ch0 + 1;
    const T *__restrict__ X = args->X;
    const int64_t ldx = args->ldx;
    const Task tk = tasks[task];
    const Blk b = blks[tk.blk0];
    for (int n0 = ch0 * Eng::NV; n0 < ch1 * Eng::NV && n0 < nv; n0 += Eng::NV) {
        const int nvc = min(Eng::NV, nv - n0);
        typename Eng::Acc acc;
        acc_zero(acc, lane);
        Eng::block(acc, static_cast<const T *>(b.A), tk.r, tk.c, X + b.x + (int64_t)n0 * ldx, ldx,
                   b.xrows, nvc, lane);
        acc_store(acc, xh + tk.out + (int64_t)n0 * xh_ld, xh_ld, tk.r, nvc, lane);
    }
}

// ---------------------------------------------------------------------------------------
// Generic row tasks whose x operands and output live in the x^/y^ workspaces:
//   MODE_WRITE  out  = sum_b A_b x_b    (upsweep transfers, coupling multiply)
//   MODE_ACCUM  out += sum_b A_b x_b    (downsweep transfers, off-diagonal coupling pass)
template <typename T, typename Eng, int MODE>
__global__ void __launch_bounds__(WPB * 32, Eng::MINB)
k_rows(const Task *__restrict__ tasks, int ntask, const Blk *__restrict__ blks,
       const T *__restrict__ src, int64_t src_ld, T *__restrict__ dst, int64_t dst_ld, int nv)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // (row, vector chunk) tasks when the launcher sized the grid for them:
    // the chunks of one row run on adjacent warps instead of in series on one warp
    const int nch = (nv + Eng::NV - 1) / Eng::NV;
    const int S = (int64_t)ntask * nch <= (int64_t)gridDim.x * WPB ? nch : 1;
    if (blockIdx.x * WPB + wid >= ntask * S) return;
    void *scratch = smem_raw + (size_t)wid * Eng::SCRATCH;
    for (int vt = blockIdx.x * WPB + wid; vt < ntask * S; vt += gridDim.x * WPB) {
    const int task = vt / S;
    const int ch0 = S == 1 ? 0 : vt - task * S, ch1 = S == 1 ? nch : ch0 + 1;
    const Task tk = tasks[task];
    for (int n0 = ch0 * Eng::NV; n0 < ch1 * Eng::NV && n0 < nv; n0 += Eng::NV) {
        const int nvc = min(Eng::NV, nv - n0);
        typename Eng::Acc acc;
        if (MODE == MODE_ACCUM) acc_load(acc, dst + tk.out + (int64_t)n0 * dst_ld, dst_ld, tk.r, nvc, lane);
        else acc_zero(acc, lane);
        if ((tk.flags & TF_ACONTIG) && tk.nblk > 0) {
            const Blk b0 = blks[tk.blk0];
            const Src<T> sr{src, src_ld, nullptr, n0};
            Eng::stream(acc, static_cast<const T *>(b0.A), tk.r, tk.c, tk.nblk, blks + tk.blk0, sr, nvc, lane,
                        scratch);
            acc_store(acc, dst + tk.out + (int64_t)n0 * dst_ld, dst_ld, tk.r, nvc, lane);
            continue;
        }
        for (int bi = 0; bi < tk.nblk; ++bi) {
            const Blk b = blks[tk.blk0 + bi];
            const int64_t ld = b.xld ? (int64_t)b.xld : src_ld;
            Eng::block(acc, static_cast<const T *>(b.A), tk.r, tk.c, src + b.x + (int64_t)n0 * ld, ld,
                       b.xrows, nvc, lane);
        }
        acc_store(acc, dst + tk.out + (int64_t)n0 * dst_ld, dst_ld, tk.r, nvc, lane);
    }
    }
}

// ---------------------------------------------------------------------------------------
// Heap-addressed transfer sweep (see SweepParams): one warp per output node, no descriptor
// loads -- the A blocks and x operands are computed from the slot index, so a task is a single
// round of independent loads.  nlev > 1 only with one CTA (barrier between levels).
template <typename T>
__device__ __forceinline__ void cp_async_elem(T *dst, const T *src)
{
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <typename T, typename Eng, int MODE, bool STAGE>
__global__ void __launch_bounds__(512, 1)
k_sweep(const __grid_constant__ SweepParams p, T *__restrict__ buf, int64_t ld, int nv, int wstride)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // programmatic dependent launch: the next level's grid may be scheduled now (its CTAs wait
    // below for this grid's completion and memory flush), hiding the per-level launch latency;
    // a no-op when launched without the attribute
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    for (int lv = 0; lv < p.nlev; ++lv) {
        const SweepLevel L = p.lv[lv];
        const int64_t blk = (int64_t)L.r * L.c;
        // a multi-level launch gives every CTA a contiguous node range per level -- a subtree: the
        // parents (upsweep) / children (downsweep) of its nodes are its own, so a CTA barrier
        // between levels suffices; single-level launches stride over the whole level
        const bool multi = p.nlev > 1;
        const int64_t per = multi ? (L.n + gridDim.x - 1) / gridDim.x : L.n;
        const int64_t lo = multi ? (int64_t)blockIdx.x * per : 0;
        const int64_t hi = multi ? min((int64_t)L.n, lo + per) : L.n;
        const int64_t i0 = multi ? lo + wid : (int64_t)blockIdx.x * nw + wid;
        const int64_t istep = multi ? nw : (int64_t)gridDim.x * nw;
        if constexpr (STAGE) {
            // latency-bound levels: the node's whole operand set (its transfer block(s) and source
            // x^ slots, r x cc and cc x nvc) is pulled into the warp's shared memory by cp.async
            // in ONE round of independent copies, then multiplied from shared memory -- one HBM
            // round trip per node instead of one per pipelined k-step group
            extern __shared__ __align__(128) unsigned char smem_raw[];
            T *As = reinterpret_cast<T *>(smem_raw) + (int64_t)wid * wstride;
            const int cc = MODE == MODE_ACCUM ? L.c : 2 * L.c;
            T *xs = As + L.r * cc;
            for (int64_t i = i0; i < hi; i += istep) {
                const T *Ag = static_cast<const T *>(L.A) + (MODE == MODE_ACCUM ? (int64_t)i : 2 * (int64_t)i) * blk;
                const T *xg = buf + L.xbase + (MODE == MODE_ACCUM ? (int64_t)(i >> 1) : 2 * (int64_t)i) * L.c;
                for (int n0 = 0; n0 < nv; n0 += Eng::NV) {
                    const int nvc = min(Eng::NV, nv - n0);
                    T *out = buf + L.obase + (int64_t)i * L.r + (int64_t)n0 * ld;
                    __syncwarp();
                    if (n0 == 0)
                        for (int e = lane; e < L.r * cc; e += 32) cp_async_elem(As + e, Ag + e);
                    for (int e = lane; e < cc * nvc; e += 32) {
                        const int n = e / cc, j = e - n * cc;
                        cp_async_elem(xs + e, xg + j + (int64_t)(n0 + n) * ld);
                    }
                    typename Eng::Acc acc;
                    if (MODE == MODE_ACCUM) acc_load(acc, out, ld, L.r, nvc, lane);
                    else                    acc_zero(acc, lane);
                    cp_async_wait_all();
                    __syncwarp();
                    Eng::smem_block(acc, As, L.r, cc, xs, cc, nvc, lane);
                    acc_store(acc, out, ld, L.r, nvc, lane);
                }
            }
            if (p.nlev > 1) __syncthreads();
            continue;
        }
        // task = (node, vector chunk) when the grid has a warp for each (nv > Eng::NV): the
        // chunks of one node run on adjacent warps instead of in series on one warp, which is
        // what bounds the small levels at large k and nv (cfg3s: ~80 us per level otherwise);
        // the launch sizes the single-level grid by the chunk count (launch_sweep)
        const int nch = (nv + Eng::NV - 1) / Eng::NV;
        const int S = (multi || (int64_t)L.n * nch <= (int64_t)gridDim.x * nw) ? nch : 1;
        for (int64_t t = (multi ? lo * S : 0) + (i0 - (multi ? lo : 0)); t < hi * S; t += istep) {
            const int64_t i = t / S;
            const int ch0 = S == 1 ? 0 : (int)(t - i * S);
            const int ch1 = S == 1 ? nch : ch0 + 1;
            for (int n0 = ch0 * Eng::NV; n0 < ch1 * Eng::NV && n0 < nv; n0 += Eng::NV) {
                const int nvc = min(Eng::NV, nv - n0);
                typename Eng::Acc acc;
                T *out = buf + L.obase + i * L.r + (int64_t)n0 * ld;
                if (MODE == MODE_ACCUM) {
                    acc_load(acc, out, ld, L.r, nvc, lane);
                    Eng::block_wide(acc, static_cast<const T *>(L.A) + i * blk, L.r, L.c,
                               buf + L.xbase + (int64_t)(i >> 1) * L.c + (int64_t)n0 * ld, ld, L.c, nvc, lane);
                } else {
                    acc_zero(acc, lane);
                    const T *A2 = static_cast<const T *>(L.A) + 2 * (int64_t)i * blk;
                    const T *x2 = buf + L.xbase + 2 * (int64_t)i * L.c + (int64_t)n0 * ld;
                    if constexpr (!Eng::MMA) {
#pragma unroll
                        for (int ch = 0; ch < 2; ++ch)
                            Eng::block_wide(acc, A2 + ch * blk, L.r, L.c, x2 + ch * L.c, ld, L.c, nvc, lane);
                    } else {
                        // the two children's Ft blocks (r x c each, column-major, adjacent) form
                        // one r x 2c block over the two adjacent child x^ slots
                        Eng::block_wide(acc, A2, L.r, 2 * L.c, x2, ld, 2 * L.c, nvc, lane);
                    }
                }
                acc_store(acc, out, ld, L.r, nvc, lane);
            }
        }
        if (p.nlev > 1) __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// Fused tree stage: one CTA owns a subtree and runs `nlev` consecutive transfer levels of it,
// level by level, with a CTA barrier between levels (the upsweep levels q-1 .. 0 or the
// downsweep levels 1 .. q-1 in a few launches instead of one launch per level, PAPER.md:263,
// 408).  Level i's tasks of CTA c are [t0[i] + c * per[i], t0[i] + (c + 1) * per[i]).
template <typename T, typename Eng, int MODE>
__global__ void __launch_bounds__(WPB * 32, Eng::MINB)
k_tree(TreeStage st, const Task *__restrict__ tasks, const Blk *__restrict__ blks, T *__restrict__ buf,
       int64_t ld, int nv)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    void *scratch = smem_raw + wid * Eng::SCRATCH;
    for (int lv = 0; lv < st.nlev; ++lv) {
        const int per = st.per[lv];
        const int64_t first = (int64_t)blockIdx.x * per;
        const int64_t base = st.t0[lv] + first;
        const int my = (int)min((int64_t)per, (int64_t)st.cnt[lv] - first);
        for (int ti = wid; ti < my; ti += WPB) {
            const Task tk = tasks[base + ti];
            for (int n0 = 0; n0 < nv; n0 += Eng::NV) {
                const int nvc = min(Eng::NV, nv - n0);
                typename Eng::Acc acc;
                if (MODE == MODE_ACCUM) acc_load(acc, buf + tk.out + (int64_t)n0 * ld, ld, tk.r, nvc, lane);
                else acc_zero(acc, lane);
                if (tk.flags & TF_ACONTIG) {
                    const Src<T> sr{buf, ld, nullptr, n0};
                    Eng::stream(acc, static_cast<const T *>(blks[tk.blk0].A), tk.r, tk.c, tk.nblk,
                                blks + tk.blk0, sr, nvc, lane, scratch);
                } else {
                    for (int bi = 0; bi < tk.nblk; ++bi) {
                        const Blk b = blks[tk.blk0 + bi];
                        Eng::block(acc, static_cast<const T *>(b.A), tk.r, tk.c, buf + b.x + (int64_t)n0 * ld,
                                   ld, b.xrows, nvc, lane);
                    }
                }
                acc_store(acc, buf + tk.out + (int64_t)n0 * ld, ld, tk.r, nvc, lane);
            }
        }
        __syncthreads();   // level lv complete (global writes visible to the CTA) before lv + 1
    }
}

// Fused leaf kernel (default schedule): last transfer + leaf expansion + dense near field +
// epilogue, Y written once:  z_t = y^_t + E_t y^_p ;  Y_t = alpha (U_t z_t + sum_s D_ts x_s) + beta Y_t
// (reading R11).  Leaf task t = ltasks[t] ([E][U]) and dtasks[t] (dense row).
template <typename T, typename EngK, typename EngM>
__global__ void __launch_bounds__(WPB * 32, (EngM::MINB < EngK::MINB ? EngM::MINB : EngK::MINB))
k_leaf_dense(const Task *__restrict__ ltasks, const Task *__restrict__ dtasks, int ntask,
             const Blk *__restrict__ blks, const T *__restrict__ yh, int64_t yh_ld,
             const CallArgs<T> *__restrict__ args, const T *__restrict__ halo, int nv, int k, int kp)
{
    const T *__restrict__ X = args->X;
    T *__restrict__ Y = args->Y;
    const int64_t ldx = args->ldx, ldy = args->ldy;
    const T alpha = args->alpha, beta = args->beta;
    static_assert(EngK::NV == EngM::NV, "engines must agree on the vector chunk");
    constexpr int NV = EngM::NV;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T *zs = reinterpret_cast<T *>(smem_raw) + wid * NV * ZLD;
    void *scratch = smem_raw + (size_t)WPB * NV * ZLD * sizeof(T) + wid * EngM::SCRATCH;
    for (int task = blockIdx.x * WPB + wid; task < ntask; task += gridDim.x * WPB) {
        const Task tk = ltasks[task];
        const Task dk = dtasks[task];
        const bool hasE = tk.flags & TF_HAS_E;
        const Blk bU = blks[tk.blk0 + (hasE ? 1 : 0)];
        for (int n0 = 0; n0 < nv; n0 += NV) {
            const int nvc = min(NV, nv - n0);
            typename EngK::Acc z;
            acc_load(z, yh + bU.x + (int64_t)n0 * yh_ld, yh_ld, k, nvc, lane);
            if (hasE) {
                const Blk bE = blks[tk.blk0];
                EngK::block(z, static_cast<const T *>(bE.A), k, kp, yh + bE.x + (int64_t)n0 * yh_ld, yh_ld,
                            bE.xrows, nvc, lane);
            }
            __syncwarp();
            acc_store(z, zs, (int64_t)ZLD, k, nvc, lane);
            __syncwarp();
            typename EngM::Acc acc;
            acc_zero(acc, lane);
            EngM::block(acc, static_cast<const T *>(bU.A), tk.r, k, zs, (int64_t)ZLD, k, nvc, lane);
            if ((dk.flags & TF_ACONTIG) && dk.nblk > 0) {
                const Src<T> sr{X, ldx, halo, n0};
                EngM::stream(acc, static_cast<const T *>(blks[dk.blk0].A), dk.r, dk.c, dk.nblk, blks + dk.blk0, sr,
                             nvc, lane, scratch);
            } else {
                for (int bi = 0; bi < dk.nblk; ++bi) {
                    const Blk b = blks[dk.blk0 + bi];
                    const T *src;
                    int64_t ld;
                    if (b.x >= 0) { src = X + b.x; ld = ldx; }
                    else          { src = halo + (-b.x - 1); ld = b.xld; }
                    EngM::block(acc, static_cast<const T *>(b.A), dk.r, dk.c, src + (int64_t)n0 * ld, ld,
                                b.xrows, nvc, lane);
                }
            }
            T *Yb = Y + tk.out + (int64_t)n0 * ldy;
            const int rows = tk.rows;
            acc.each(lane, [&](int row, int n, auto &v) {
                if (row < rows && n < nvc) {
                    T *p = Yb + row + n * ldy;
                    *p = (beta == T(0)) ? alpha * v : fma(alpha, (T)v, beta * *p);
                }
            });
            __syncwarp();
        }
    }
}

// Row-split fused leaf kernel for the DMMA path with m > 32 (nv >= 5): two warps per leaf, each
// owning 32 rows of U_t and of the dense row (lda = m), so the accumulator is Mma<4,NT> instead
// of Mma<8,NT> (no register spills, twice the warps in flight).  z_t is computed by both.
template <typename T, typename EngK, typename EngH>
__global__ void __launch_bounds__(WPB * 32, 2)
k_leaf_dense_split(const Task *__restrict__ ltasks, const Task *__restrict__ dtasks, int ntask2,
                   const Blk *__restrict__ blks, const T *__restrict__ yh, int64_t yh_ld,
                   const CallArgs<T> *__restrict__ args, const T *__restrict__ halo, int nv, int k, int kp, int m)
{
    const T *__restrict__ X = args->X;
    T *__restrict__ Y = args->Y;
    const int64_t ldx = args->ldx, ldy = args->ldy;
    const T alpha = args->alpha, beta = args->beta;
    static_assert(EngK::NV == EngH::NV, "engines must agree on the vector chunk");
    constexpr int NV = EngH::NV;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T *zs = reinterpret_cast<T *>(smem_raw) + wid * NV * ZLD;
    void *scratch = smem_raw + (size_t)WPB * NV * ZLD * sizeof(T) + wid * EngH::SCRATCH;
    // (leaf half, vector chunk) tasks when the launcher sized the grid for them (see k_rows)
    const int nch = (nv + NV - 1) / NV;
    const int S = (int64_t)ntask2 * nch <= (int64_t)gridDim.x * WPB ? nch : 1;
    for (int vt = blockIdx.x * WPB + wid; vt < ntask2 * S; vt += gridDim.x * WPB) {
        const int task2 = vt / S;
        const int ch0 = S == 1 ? 0 : vt - task2 * S, ch1 = S == 1 ? nch : ch0 + 1;
        const int task = task2 >> 1, half = task2 & 1;
        const Task tk = ltasks[task];
        const Task dk = dtasks[task];
        const bool hasE = tk.flags & TF_HAS_E;
        const Blk bU = blks[tk.blk0 + (hasE ? 1 : 0)];
        const int r0 = 32 * half;
        const int rh = min(32, m - r0);
        for (int n0 = ch0 * NV; n0 < ch1 * NV && n0 < nv; n0 += NV) {
            const int nvc = min(NV, nv - n0);
            typename EngK::Acc z;
            acc_load(z, yh + bU.x + (int64_t)n0 * yh_ld, yh_ld, k, nvc, lane);
            if (hasE) {
                const Blk bE = blks[tk.blk0];
                EngK::block(z, static_cast<const T *>(bE.A), k, kp, yh + bE.x + (int64_t)n0 * yh_ld, yh_ld,
                            bE.xrows, nvc, lane);
            }
            __syncwarp();
            acc_store(z, zs, (int64_t)ZLD, k, nvc, lane);
            __syncwarp();
            typename EngH::Acc acc;
            acc_zero(acc, lane);
            EngH::block(acc, static_cast<const T *>(bU.A) + r0, rh, k, zs, (int64_t)ZLD, k, nvc, lane, m);
            if ((dk.flags & TF_ACONTIG) && dk.nblk > 0) {
                const Src<T> sr{X, ldx, halo, n0};
                EngH::stream(acc, static_cast<const T *>(blks[dk.blk0].A) + r0, rh, dk.c, dk.nblk, blks + dk.blk0,
                             sr, nvc, lane, scratch, m);
            } else {
                for (int bi = 0; bi < dk.nblk; ++bi) {
                    const Blk b = blks[dk.blk0 + bi];
                    const T *src;
                    int64_t ld;
                    if (b.x >= 0) { src = X + b.x; ld = ldx; }
                    else          { src = halo + (-b.x - 1); ld = b.xld; }
                    EngH::block(acc, static_cast<const T *>(b.A) + r0, rh, dk.c, src + (int64_t)n0 * ld, ld,
                                b.xrows, nvc, lane, m);
                }
            }
            T *Yb = Y + tk.out + r0 + (int64_t)n0 * ldy;
            const int rows = tk.rows - r0;
            acc.each(lane, [&](int row, int n, auto &v) {
                if (row < rows && n < nvc) {
                    T *p = Yb + row + n * ldy;
                    *p = (beta == T(0)) ? alpha * v : fma(alpha, (T)v, beta * *p);
                }
            });
            __syncwarp();
        }
    }
}

template <typename T>
__global__ void k_set_args(CallArgs<T> *a, const T *X, int64_t ldx, T *Y, int64_t ldy, T alpha, T beta)
{
    a->X = X; a->ldx = ldx; a->Y = Y; a->ldy = ldy; a->alpha = alpha; a->beta = beta;
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
                       int64_t src_ld, const CallArgs<T> *__restrict__ args, T *__restrict__ dst, int nv)
{
    const int lane = threadIdx.x & 31;
    if (!src) { src = args->X; src_ld = args->ldx; }   // halo pack reads the caller's X
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nseg;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const PackSeg sg = segs[w];
        for (int n = 0; n < nv; ++n)
            for (int j = lane; j < sg.len; j += 32)
                dst[sg.dst + j + (int64_t)n * sg.dst_ld] = src[sg.src + j + (int64_t)n * src_ld];
    }
}

// ---------------------------------------------------------------------------------------
// dispatch: Simt for float or nv <= 4; Mma (DMMA) for double with nv >= 5
static inline int grid_for(int ntask) { return (ntask + WPB - 1) / WPB; }

// kernel launch with programmatic stream serialization (PDL): the kernel may start before its
// in-stream predecessor completes and must execute griddepcontrol.wait before reading its output
template <typename... KArgs, typename... Args>
static inline void launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t s,
                              Args &&...args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    // H2_PDL=0: plain stream order (A/B switch)
    static const bool pdl = [] { const char *e = getenv("H2_PDL"); return !(e && e[0] == '0'); }();
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// dynamic shared memory opt-in, once per kernel instantiation
template <typename K>
static inline cudaError_t smem_opt_in(K kern, size_t bytes)
{
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <typename T>
struct Dispatch {
    // f(Eng) with Eng chosen from (rows r -> RPL / MT, nv -> NVB / NT): FP32 runs SIMT up to nv = 4
    // and the 3xTF32 tensor engine above
    template <typename F>
    static void run(int r, int nv, F f)
    {
        const int rpl = r > 32 ? 2 : 1;
        if (nv <= 1) { if (rpl == 1) f(Simt<T, 1, 1>{}); else f(Simt<T, 2, 1>{}); }
        else if (nv <= 2) { if (rpl == 1) f(Simt<T, 1, 2>{}); else f(Simt<T, 2, 2>{}); }
        else if (nv <= 4) { if (rpl == 1) f(Simt<T, 1, 4>{}); else f(Simt<T, 2, 4>{}); }
        else if (nv <= 8) {
            if (r <= 16) f(Tf3<1, 1>{}); else if (r <= 32) f(Tf3<2, 1>{}); else f(Tf3<4, 1>{});
        } else {
            if (r <= 16) f(Tf3<1, 2>{}); else if (r <= 32) f(Tf3<2, 2>{}); else f(Tf3<4, 2>{});
        }
    }
    template <typename F>
    static void run2(int rk, int rm, int nv, F f)
    {
        run(rk, nv, [&](auto ek) {
            using EK = decltype(ek);
            run(rm, nv, [&](auto em) {
                using EM = decltype(em);
                if constexpr (EK::NV == EM::NV) f(ek, em);
            });
        });
    }
};

template <>
struct Dispatch<double> {
    template <typename F>
    static void run(int r, int nv, F f)
    {
        using T = double;
        const int rpl = r > 32 ? 2 : 1;
        if (nv <= 1) { if (rpl == 1) f(Simt<T, 1, 1>{}); else f(Simt<T, 2, 1>{}); }
        else if (nv <= 2) { if (rpl == 1) f(Simt<T, 1, 2>{}); else f(Simt<T, 2, 2>{}); }
        else if (nv <= 4) { if (rpl == 1) f(Simt<T, 1, 4>{}); else f(Simt<T, 2, 4>{}); }
        else if (nv <= 8) {
            if (r <= 16) f(Mma<2, 1>{}); else if (r <= 32) f(Mma<4, 1>{}); else f(Mma<8, 1>{});
        } else {
            if (r <= 16) f(Mma<2, 2>{}); else if (r <= 32) f(Mma<4, 2>{}); else f(Mma<8, 2>{});
        }
    }
    template <typename F>
    static void run2(int rk, int rm, int nv, F f)
    {
        run(rk, nv, [&](auto ek) {
            using EK = decltype(ek);
            run(rm, nv, [&](auto em) {
                using EM = decltype(em);
                if constexpr (EK::NV == EM::NV) f(ek, em);
            });
        });
    }
};

template <typename T>
cudaError_t launch_set_args(CallArgs<T> *a, const T *X, int64_t ldx, T *Y, int64_t ldy, T alpha, T beta,
                            cudaStream_t s)
{
    k_set_args<T><<<1, 1, 0, s>>>(a, X, ldx, Y, ldy, alpha, beta);
    return cudaGetLastError();
}

// Grids of the warp-task kernels carry one warp per (task, vector chunk): when nv exceeds the
// engine's chunk, the chunks of one task run on adjacent warps instead of in series on one warp
// (the repeated block reads then hit L2).
template <typename T>
cudaError_t launch_up_leaf(const Task *t, int ntask, const Blk *b, const CallArgs<T> *args,
                           T *xh, int64_t xh_ld, int nv, int r, cudaStream_t s)
{
    if (ntask == 0) return cudaSuccess;
    Dispatch<T>::run(r, nv, [&](auto e) {
        const int nch = (nv + decltype(e)::NV - 1) / decltype(e)::NV;
        k_up_leaf<T, decltype(e)><<<grid_for(ntask * nch), WPB * 32, 0, s>>>(t, ntask, b, args, xh, xh_ld, nv);
    });
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_rows(int mode, const Task *t, int ntask, const Blk *b, const T *src, int64_t src_ld, T *dst,
                        int64_t dst_ld, int nv, int r, cudaStream_t s)
{
    if (ntask == 0) return cudaSuccess;
    cudaError_t err = cudaSuccess;
    Dispatch<T>::run(r, nv, [&](auto e) {
        using E = decltype(e);
        const size_t sm = (size_t)WPB * E::SCRATCH;
        auto kw = k_rows<T, E, MODE_WRITE>;
        auto ka = k_rows<T, E, MODE_ACCUM>;
        static cudaError_t attr = [&] {
            cudaError_t e1 = smem_opt_in(kw, sm);
            return e1 == cudaSuccess ? smem_opt_in(ka, sm) : e1;
        }();
        if ((err = attr) != cudaSuccess) return;
        const int nch = (nv + E::NV - 1) / E::NV;
        if (mode == MODE_WRITE) kw<<<grid_for(ntask * nch), WPB * 32, sm, s>>>(t, ntask, b, src, src_ld, dst, dst_ld, nv);
        else                    ka<<<grid_for(ntask * nch), WPB * 32, sm, s>>>(t, ntask, b, src, src_ld, dst, dst_ld, nv);
    });
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_tree(int mode, const TreeStage &st, int nctas, const Task *t, const Blk *b, T *buf,
                        int64_t ld, int nv, int r, cudaStream_t s)
{
    if (nctas == 0 || st.nlev == 0) return cudaSuccess;
    Dispatch<T>::run(r, nv, [&](auto e) {
        using E = decltype(e);
        const size_t sm = (size_t)WPB * E::SCRATCH;
        if (mode == MODE_WRITE)
            k_tree<T, E, MODE_WRITE><<<nctas, WPB * 32, sm, s>>>(st, t, b, buf, ld, nv);
        else
            k_tree<T, E, MODE_ACCUM><<<nctas, WPB * 32, sm, s>>>(st, t, b, buf, ld, nv);
    });
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_leaf_dense(const Task *lt, const Task *dt, int ntask, const Blk *b, const T *yh, int64_t yh_ld,
                              const CallArgs<T> *args, const T *halo, int nv, int k, int kp, int m, cudaStream_t s)
{
    if (ntask == 0) return cudaSuccess;
    cudaError_t err = cudaSuccess;
    if constexpr (std::is_same<T, double>::value) {
        if (nv >= 5 && m > 32) {
            // DMMA path with 64-row leaves: two warps per leaf (k_leaf_dense_split)
            auto go = [&](auto ek, auto eh) {
                using EK = decltype(ek);
                using EH = decltype(eh);
                auto kern = k_leaf_dense_split<double, EK, EH>;
                const size_t sm = (size_t)WPB * (EH::NV * ZLD * sizeof(double) + EH::SCRATCH);
                static cudaError_t attr = smem_opt_in(kern, sm);
                if ((err = attr) != cudaSuccess) return;
                const int nch = (nv + EH::NV - 1) / EH::NV;
                kern<<<grid_for(2 * ntask * nch), WPB * 32, sm, s>>>(lt, dt, 2 * ntask, b, yh, yh_ld, args, halo,
                                                                     nv, k, kp, m);
            };
            Dispatch<double>::run(k, nv, [&](auto ek) {
                using EK = decltype(ek);
                if constexpr (EK::NV == 8) go(ek, Mma<4, 1>{});
                else if constexpr (EK::NV == 16) go(ek, Mma<4, 2>{});
            });
            if (err != cudaSuccess) return err;
            return cudaGetLastError();
        }
    }
    Dispatch<T>::run2(k, m, nv, [&](auto ek, auto em) {
        using EK = decltype(ek);
        using EM = decltype(em);
        auto kern = k_leaf_dense<T, EK, EM>;
        const size_t sm = (size_t)WPB * (EM::NV * ZLD * sizeof(T) + EM::SCRATCH);
        static cudaError_t attr = smem_opt_in(kern, sm);
        if ((err = attr) != cudaSuccess) return;
        kern<<<grid_for(ntask), WPB * 32, sm, s>>>(lt, dt, ntask, b, yh, yh_ld, args, halo, nv, k, kp);
    });
    if (err != cudaSuccess) return err;
    return cudaGetLastError();
}

// Heap-addressed transfer sweep launch (k_sweep).  SIMT engines stage every node's operands
// with cp.async (one round of copies per node); DMMA engines read them straight from L2.
// Consecutive sweep launches overlap through programmatic dependent launch.
template <typename T>
cudaError_t launch_sweep(int mode, const SweepParams &p, int nctas, int threads, T *buf, int64_t ld, int nv,
                         int r, cudaStream_t s)
{
    if (p.nlev == 0 || nctas == 0) return cudaSuccess;
    int maxn = 0, rmax = 0, cmax = 0;
    for (int l = 0; l < p.nlev; ++l) {
        maxn = std::max(maxn, (int)p.lv[l].n);
        rmax = std::max(rmax, (int)p.lv[l].r);
        cmax = std::max(cmax, (int)p.lv[l].c);
    }
    const int cc = mode == MODE_ACCUM ? cmax : 2 * cmax;
    cudaError_t err = cudaSuccess;
    Dispatch<T>::run(r, nv, [&](auto e) {
        using E = decltype(e);
        const int wstride = ((rmax * cc + cc * E::NV) + 1) & ~1;          // elements, 16-byte multiple
        const size_t wbytes = (size_t)wstride * sizeof(T);
        int warps = threads / 32;
        while (warps > 1 && warps * wbytes > SWEEP_STAGE_SMEM) warps >>= 1;
        const bool stage = !E::MMA && warps * wbytes <= SWEEP_STAGE_SMEM;
        if (stage) {
            const int ctas = p.nlev > 1 ? nctas : (int)((maxn + warps - 1) / warps);
            const size_t sm = warps * wbytes;
            auto kw = k_sweep<T, E, MODE_WRITE, true>;
            auto ka = k_sweep<T, E, MODE_ACCUM, true>;
            static cudaError_t attr = [&] {
                cudaError_t e1 = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SWEEP_STAGE_SMEM);
                return e1 == cudaSuccess
                           ? cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SWEEP_STAGE_SMEM)
                           : e1;
            }();
            if ((err = attr) != cudaSuccess) return;
            launch_pdl(mode == MODE_WRITE ? kw : ka, ctas, warps * 32, sm, s, p, buf, ld, nv, wstride);
        } else {
            // single-level launches get a warp per (node, vector chunk); see k_sweep
            const int nch = (nv + E::NV - 1) / E::NV;
            const int grid = p.nlev > 1 ? nctas : nctas * nch;
            launch_pdl(mode == MODE_WRITE ? k_sweep<T, E, MODE_WRITE, false> : k_sweep<T, E, MODE_ACCUM, false>, grid,
                       threads, 0, s, p, buf, ld, nv, 0);
        }
    });
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
cudaError_t launch_pack(const PackSeg *segs, int64_t nseg, const T *src, int64_t src_ld,
                        const CallArgs<T> *args, T *dst, int nv, cudaStream_t s)
{
    if (nseg == 0) return cudaSuccess;
    int64_t blocks = (nseg + 7) / 8;
    k_pack<T><<<(int)(blocks < 1184 ? blocks : 1184), 256, 0, s>>>(segs, nseg, src, src_ld, args, dst, nv);
    return cudaGetLastError();
}

}  // namespace h2
