// h2_cta.cuh -- the CTA-tile FP64 engine (DESIGN.md §7 "CTA-tile engine").
//
// One CTA computes one output node at a time,  y (r x nv) (+)= sum_b A_b (r x c) x_b (c x nv),
// for the transfer, coupling, leaf-projection and leaf (expansion + dense + epilogue) tasks of the
// plan (PAPER.md:239-254 upsweep, 328-331 coupling, 389-414 downsweep and leaves, 225 dense).
// Every block A_b and its operand x_b pass through a multi-stage shared-memory ring filled by
// cp.async (LDGSTS, 16-byte chunks where aligned): A_b is read from HBM exactly once per task
// whatever nv is, and ALL warps of the CTA consume it -- warp (wr, wc) owns rows
// [8 MT wr, 8 MT (wr+1)) and vectors [16 wc, 16 wc + 16) of the output tile and multiplies with
// mma.sync.m8n8k4.f64 (SASS DMMA) from shared memory.  The ring's leading dimensions
// (lda, ldx = 4 mod 8 doubles) make the fragment loads conflict-free (two wavefronts per 256 B).
// Tasks are distributed statically over persistent CTAs (longest rows first from the plan), and
// the copies of the next NS-1 blocks -- across task boundaries -- run behind the DMMAs of the
// current one.
#pragma once
#include "h2_internal.h"

namespace h2 {

namespace cta {

constexpr int CMAX = 64;       // max block columns
constexpr int LDM = 68;        // max leading dimension of a staged operand (doubles)
__host__ __device__ constexpr int ld_for(int rows) { return ((rows + 3) / 8) * 8 + 4; }   // 4 mod 8, >= rows

struct Step {
    const double *A;
    const double *x;           // nullptr: the operand is the z tile the consumer writes (leaf U step)
    int64_t xld;
    int r, c, xrows;
};

__device__ __forceinline__ void cp8(double *dst, const double *src, bool valid)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp16(double *dst, const double *src, int bytes)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ const double *resolve_x(const CtaJob &j, const double *pos, int64_t pos_ld, int64_t x,
                                                   int32_t xld, int64_t &ld)
{
    if (x >= 0) { ld = xld ? (int64_t)xld : pos_ld; return pos + x; }
    ld = xld;
    return j.halo + (-x - 1);
}

// Number of steps of task t and the descriptor of step s.
__device__ __forceinline__ int task_steps(const CtaJob &j, int t)
{
    const Task tk = j.tasks[t];
    if (j.kind == CK_LEAF) return tk.nblk + j.dtasks[t].nblk;    // [E] U D...
    return tk.nblk;
}

__device__ __forceinline__ Step task_step(const CtaJob &j, int t, int s)
{
    const Task tk = j.tasks[t];
    Step st;
    if (j.kind == CK_LEAF) {
        const bool hasE = tk.flags & TF_HAS_E;
        if (s < tk.nblk) {
            const Blk b = j.blks[tk.blk0 + s];
            if (hasE && s == 0) {       // E_t (k x kp) times the parent's y^
                st.A = static_cast<const double *>(b.A);
                st.x = j.yh + b.x;
                st.xld = j.yh_ld;
                st.r = j.blks[tk.blk0 + 1].xrows;   // k: the U block's column count
                st.c = b.xrows;                     // kp
                st.xrows = b.xrows;
                return st;
            }
            st.A = static_cast<const double *>(b.A);   // U_t (m x k) times z
            st.x = nullptr;
            st.xld = 0;
            st.r = tk.r;
            st.c = b.xrows;
            st.xrows = b.xrows;
            return st;
        }
        const Task dk = j.dtasks[t];
        const Blk b = j.blks[dk.blk0 + (s - tk.nblk)];
        int64_t ld;
        st.A = static_cast<const double *>(b.A);
        st.x = resolve_x(j, j.args->X, j.args->ldx, b.x, b.xld, ld);
        st.xld = ld;
        st.r = dk.r;
        st.c = dk.c;
        st.xrows = b.xrows;
        return st;
    }
    const Blk b = j.blks[tk.blk0 + s];
    int64_t ld;
    if (j.kind == CK_UPLEAF) st.x = resolve_x(j, j.args->X, j.args->ldx, b.x, b.xld, ld);
    else                     st.x = resolve_x(j, j.src, j.src_ld, b.x, b.xld, ld);
    st.A = static_cast<const double *>(b.A);
    st.xld = ld;
    st.r = tk.r;
    st.c = tk.c;
    st.xrows = b.xrows;
    return st;
}

// Issue the copies of one step into stage buffers As (CMAX x LDM) and Xs (NVT x LDM).
template <int NW>
__device__ __forceinline__ void issue(const Step &st, double *As, double *Xs, int nv, int wid, int lane)
{
    const int lda = ld_for(st.r), c4 = (st.c + 3) & ~3;
    const bool a16 = ((reinterpret_cast<uintptr_t>(st.A) & 15) == 0) && !(st.r & 1);
    for (int col = wid; col < st.c; col += NW) {
        const double *src = st.A + (int64_t)col * st.r;
        double *dst = As + col * lda;
        if (a16) {
            if (2 * lane < st.r) cp16(dst + 2 * lane, src + 2 * lane, 16);
        } else {
            for (int i = lane; i < st.r; i += 32) cp8(dst + i, src + i, true);
        }
    }
    for (int e = threadIdx.x; e < (c4 - st.c) * lda; e += NW * 32) As[st.c * lda + e] = 0.0;   // k-step padding
    if (!st.x) return;
    const int ldx = ld_for(st.c);
    const bool x16 = ((reinterpret_cast<uintptr_t>(st.x) & 15) == 0) && !(st.xld & 1);
    for (int n = wid; n < nv; n += NW) {
        const double *src = st.x + (int64_t)n * st.xld;
        double *dst = Xs + n * ldx;
        if (x16) {
            if (2 * lane < c4) {
                const int left = st.xrows - 2 * lane;
                cp16(dst + 2 * lane, src + (left > 0 ? 2 * lane : 0), left >= 2 ? 16 : (left == 1 ? 8 : 0));
            }
        } else {
            for (int i = lane; i < c4; i += 32) cp8(dst + i, src + (i < st.xrows ? i : 0), i < st.xrows);
        }
    }
}

}  // namespace cta

// NS-stage ring, WR x WC warps, MT m-tiles x 2 n-tiles per warp.
template <int MT, int WR, int WC, int NS>
__global__ void __launch_bounds__(WR *WC * 32, 1) k_cta(const __grid_constant__ CtaJob j)
{
    using namespace cta;
    constexpr int NW = WR * WC, NVT = 16 * WC, NT = 2;
    constexpr int AEL = CMAX * LDM, XEL = NVT * LDM, STAGE = AEL + XEL;
    extern __shared__ __align__(128) double sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int wr = wid % WR, wc = wid / WR;
    const int g = lane >> 2, t4 = lane & 3;
    const int row0 = wr * 8 * MT, col0 = wc * 16;
    const int nv = j.nv;
    const int G = gridDim.x;

    // producer cursor: my task (blockIdx.x + pt * G) and its step ps
    int pt = 0, ps = 0, pn = 0;
    auto ptask = [&](int i) { return (int)blockIdx.x + i * G; };
    auto padvance = [&]() {       // move to the next step that exists
        ++ps;
        while (ptask(pt) < j.ntask && ps >= pn) {
            ++pt;
            ps = 0;
            pn = ptask(pt) < j.ntask ? task_steps(j, ptask(pt)) : 0;
        }
    };
    if (ptask(0) < j.ntask) {
        pn = task_steps(j, ptask(0));
        ps = -1;
        padvance();
    }
    int issued = 0;
    auto produce = [&]() {
        if (ptask(pt) < j.ntask) {
            const Step st = task_step(j, ptask(pt), ps);
            double *base = sm + (issued % NS) * STAGE;
            issue<NW>(st, base, base + AEL, nv, wid, lane);
            padvance();
        }
        cp_commit();
        ++issued;
    };
#pragma unroll 1
    for (int i = 0; i < NS - 1; ++i) produce();

    int consumed = 0;
    for (int ti = 0; ptask(ti) < j.ntask; ++ti) {
        const int t = ptask(ti);
        const Task tk = j.tasks[t];
        const int nsteps = task_steps(j, t);
        double acc[MT][NT][2];
        // ---- accumulator init
        auto acc_fill = [&](const double *base, int64_t ld, int rows) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int row = row0 + 8 * mt + g, n = col0 + 8 * nt + 2 * t4 + i;
                        acc[mt][nt][i] = (base && row < rows && n < nv) ? base[row + n * ld] : 0.0;
                    }
        };
        const bool leaf = j.kind == CK_LEAF;
        const bool hasE = leaf && (tk.flags & TF_HAS_E);
        int kz = 0;                                   // leaf: rows of z (= k)
        if (leaf) {
            const Blk bU = j.blks[tk.blk0 + (hasE ? 1 : 0)];
            kz = bU.xrows;
            acc_fill(j.yh + bU.x, j.yh_ld, kz);       // z starts at the leaf's own y^
        } else if (j.kind == CK_ROWS && j.mode == MODE_ACCUM) {
            acc_fill(j.dst + tk.out, j.dst_ld, tk.r);
        } else {
            acc_fill(nullptr, 0, 0);
        }
        if (nsteps == 0) {                            // empty coupling row (WRITE): y^ = 0
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int row = row0 + 8 * mt + g, n = col0 + 8 * nt + 2 * t4 + i;
                        if (row < tk.r && n < nv) j.dst[tk.out + row + n * j.dst_ld] = acc[mt][nt][i];
                    }
            continue;
        }
        for (int s = 0; s < nsteps; ++s, ++consumed) {
            cp_wait<NS - 2>();
            __syncthreads();
            produce();
            double *As = sm + (consumed % NS) * STAGE;
            double *Xs = As + AEL;
            const Step st = task_step(j, t, s);
            if (!st.x) {
                // leaf U step: hand z (k x nv, in the accumulator) over through this stage's x area
                const int ldz = ld_for(st.c), c4 = (st.c + 3) & ~3;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            const int row = row0 + 8 * mt + g, n = col0 + 8 * nt + 2 * t4 + i;
                            if (row < c4 && n < NVT) Xs[row + n * ldz] = row < kz ? acc[mt][nt][i] : 0.0;
                            acc[mt][nt][i] = 0.0;
                        }
                __syncthreads();
            }
            const int lda = ld_for(st.r), ldx = ld_for(st.c), ksn = (st.c + 3) >> 2;
            const double *Ap = As + t4 * lda + row0 + g;
            const double *Bp = Xs + t4 + (col0 + g) * ldx;
            double a[2][MT], b[2][NT];
            auto ldfr = [&](int p, int ks) {
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) a[p][mt] = Ap[4 * ks * lda + 8 * mt];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) b[p][nt] = Bp[4 * ks + 8 * nt * ldx];
            };
            auto mma = [&](int p) {
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) h2::dmma(acc[mt][nt], a[p][mt], b[p][nt]);
            };
            if (col0 < nv) {
                ldfr(0, 0);
                int ks = 0;
                for (; ks + 2 <= ksn; ks += 2) {
                    ldfr(1, ks + 1);
                    mma(0);
                    if (ks + 2 < ksn) ldfr(0, ks + 2);
                    mma(1);
                }
                if (ks < ksn) mma(0);
            }
        }
        // ---- store
        if (leaf) {
            double *Y = j.args->Y;
            const int64_t ldy = j.args->ldy;
            const double alpha = j.args->alpha, beta = j.args->beta;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int row = row0 + 8 * mt + g, n = col0 + 8 * nt + 2 * t4 + i;
                        if (row < tk.rows && n < nv) {
                            double *p = Y + tk.out + row + n * ldy;
                            *p = (beta == 0.0) ? alpha * acc[mt][nt][i] : fma(alpha, acc[mt][nt][i], beta * *p);
                        }
                    }
        } else {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int row = row0 + 8 * mt + g, n = col0 + 8 * nt + 2 * t4 + i;
                        if (row < tk.r && n < nv) j.dst[tk.out + row + n * j.dst_ld] = acc[mt][nt][i];
                    }
        }
    }
    cp_wait<0>();
}

}  // namespace h2

namespace h2 {
// Engine shape from the widest output tile (rmax rows) and nv: WC vector chunks of 16, WR warp
// rows of 8 MT rows each; NS ring stages (the largest that fits 227 KB of shared memory).
cudaError_t launch_cta(const CtaJob &j, int rmax, int nsm, cudaStream_t s)
{
    if (j.ntask == 0) return cudaSuccess;
    const int grid = j.ntask < nsm ? j.ntask : nsm;
    cudaError_t err = cudaSuccess;
    auto go = [&](void (*kern)(CtaJob), int warps, int nvt, int ns) {
        const size_t smem = (size_t)ns * (cta::CMAX * cta::LDM + nvt * cta::LDM) * sizeof(double);
        static void *done[16] = {};
        bool set = false;
        for (void *d : done) set = set || d == (void *)kern;
        if (!set) {
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (err != cudaSuccess) return;
            for (void *&d : done)
                if (!d) { d = (void *)kern; break; }
        }
        kern<<<grid, warps * 32, smem, s>>>(j);
        err = cudaGetLastError();
    };
    const bool big = rmax > 32;
    if (j.nv <= 16) {
        if (big) go(k_cta<2, 4, 1, 4>, 4, 16, 4); else go(k_cta<1, 4, 1, 4>, 4, 16, 4);
    } else if (j.nv <= 32) {
        if (big) go(k_cta<2, 4, 2, 3>, 8, 32, 3); else go(k_cta<1, 4, 2, 3>, 8, 32, 3);
    } else {
        if (big) go(k_cta<4, 2, 4, 3>, 8, 64, 3); else go(k_cta<2, 2, 4, 3>, 8, 64, 3);
    }
    return err;
}
}  // namespace h2
