// h2_cta.cuh -- the CTA-tile FP64 engine (DESIGN.md §7 "CTA-tile engine").
//
// One CTA computes one output node at a time,  y (r x nv) (+)= sum_b A_b (r x c) x_b (c x nv),
// for the transfer, coupling, leaf-projection and leaf (expansion + dense + epilogue) tasks of the
// plan (PAPER.md:239-254 upsweep, 328-331 coupling, 389-414 downsweep and leaves, 225 dense).
// Warp-specialised: one PRODUCER warp walks this CTA's task list and streams every block A_b and
// its operand x_b into an NS-stage shared-memory ring with cp.async (16-byte chunks where
// aligned), completing on per-stage mbarriers; the CONSUMER warps multiply from shared memory with
// mma.sync.m8n8k4.f64 (SASS DMMA) -- warp (wr, wc) owns rows [8 MT wr, 8 MT (wr+1)) and vectors
// [16 wc, 16 wc + 16) of the output tile -- and release the stage.  A_b is read from HBM once per
// task whatever nv is; the producer runs up to NS blocks ahead across task boundaries, so
// descriptor and HBM latency stay off the DMMA path.  The ring's leading dimensions
// (lda, ldx = 4 mod 8 doubles) make the fragment loads conflict-free (two wavefronts per 256 B).
// Tasks are distributed statically over persistent CTAs (longest rows first from the plan).
#pragma once
#include "h2_internal.h"

namespace h2 {
namespace cta {

constexpr int CMAX = 64;       // max block columns
constexpr int LDM = 68;        // max leading dimension of a staged operand (doubles)
__host__ __device__ constexpr int ld_for(int rows) { return ((rows + 3) / 8) * 8 + 4; }   // 4 mod 8, >= rows

enum { MF_Z = 1, MF_EMPTY = 2, MF_END = 4 };

// Per-stage descriptor written by the producer for the consumers.
struct Meta {
    int64_t out;      // output offset of the task (plane element / Y row)
    int64_t zsrc;     // leaf: y^ offset of the leaf's own y^ (z starts there)
    int32_t s, nst;   // step within the task, steps of the task
    int32_t r, c;     // block shape of this step
    int32_t tr;       // output rows of the task (r of its steps; leaf: m)
    int32_t rows;     // leaf: real rows of the leaf
    int32_t kz;       // leaf: rows of z (= k)
    int32_t flags;
};

struct Step {
    const double *A;
    const double *x;           // nullptr: the operand is the z tile the consumers write (leaf U step)
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
__device__ __forceinline__ void mb_init(uint64_t *b, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mb_arrive_cp(uint64_t *b)     // when this thread's cp.asyncs land
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads)
{
    asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ const double *resolve_x(const CtaJob &j, const double *pos, int64_t pos_ld, int64_t x,
                                                   int32_t xld, int64_t &ld)
{
    if (x >= 0) { ld = xld ? (int64_t)xld : pos_ld; return pos + x; }
    ld = xld;
    return j.halo + (-x - 1);
}

// Index of the block descriptor of step s of task tk (leaf tasks: [E] U, then the dense row dk).
__device__ __forceinline__ int64_t step_blk(const CtaJob &j, const Task &tk, const Task &dk, int s)
{
    return (j.kind == CK_LEAF && s >= tk.nblk) ? dk.blk0 + (s - tk.nblk) : tk.blk0 + s;
}

// Step s of task tk from its block descriptor b (kz: the leaf's k, the U block's column count).
__device__ __forceinline__ Step make_step(const CtaJob &j, const Task &tk, const Task &dk, int s, const Blk &b,
                                          int kz)
{
    Step st;
    int64_t ld;
    st.A = static_cast<const double *>(b.A);
    st.xrows = b.xrows;
    if (j.kind == CK_LEAF) {
        if (s < tk.nblk) {
            if ((tk.flags & TF_HAS_E) && s == 0) {      // E_t (k x kp) times the parent's y^
                st.x = j.yh + b.x;
                st.xld = j.yh_ld;
                st.r = kz;
                st.c = b.xrows;
            } else {                                    // U_t (m x k) times z
                st.x = nullptr;
                st.xld = 0;
                st.r = tk.r;
                st.c = b.xrows;
            }
            return st;
        }
        st.x = resolve_x(j, j.args->X, j.args->ldx, b.x, b.xld, ld);
        st.xld = ld;
        st.r = dk.r;
        st.c = dk.c;
        return st;
    }
    if (j.kind == CK_UPLEAF) st.x = resolve_x(j, j.args->X, j.args->ldx, b.x, b.xld, ld);
    else                     st.x = resolve_x(j, j.src, j.src_ld, b.x, b.xld, ld);
    st.xld = ld;
    st.r = tk.r;
    st.c = tk.c;
    return st;
}

__device__ __forceinline__ Blk shfl_blk(const Blk &b, int src)
{
    Blk o;
    o.A = reinterpret_cast<const void *>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(b.A), src));
    o.x = __shfl_sync(0xffffffffu, b.x, src);
    o.xrows = __shfl_sync(0xffffffffu, b.xrows, src);
    o.xld = __shfl_sync(0xffffffffu, b.xld, src);
    return o;
}

// The producer warp's copies of one step into stage buffers As (CMAX x LDM) and Xs (NVT x LDM);
// padding (A columns c..c4-1, x rows xrows..c4-1) is zero-filled by the copies themselves.
__device__ __forceinline__ void issue(const Step &st, double *As, double *Xs, int nv, int lane)
{
    const int lda = ld_for(st.r), c4 = (st.c + 3) & ~3;
    const bool a16 = ((reinterpret_cast<uintptr_t>(st.A) & 15) == 0) && !(st.r & 1);
    if (a16) {
        const int half = st.r >> 1;                       // 16-byte chunks per column (<= 32)
        if (lane < half)
            for (int col = 0; col < c4; ++col) {
                const bool v = col < st.c;
                cp16(As + col * lda + 2 * lane, st.A + (v ? (int64_t)col * st.r + 2 * lane : 0), v ? 16 : 0);
            }
    } else {
        for (int col = 0; col < c4; ++col) {
            const bool v = col < st.c;
            for (int i = lane; i < st.r; i += 32) cp8(As + col * lda + i, st.A + (v ? (int64_t)col * st.r + i : 0), v);
        }
    }
    if (!st.x) return;
    const int ldx = ld_for(st.c);
    const bool x16 = ((reinterpret_cast<uintptr_t>(st.x) & 15) == 0) && !(st.xld & 1);
    if (x16) {
        const int half = c4 >> 1;
        const int left = st.xrows - 2 * lane;
        if (lane < half)
            for (int n = 0; n < nv; ++n)
                cp16(Xs + n * ldx + 2 * lane, st.x + (int64_t)n * st.xld + (left > 0 ? 2 * lane : 0),
                     left >= 2 ? 16 : (left == 1 ? 8 : 0));
    } else {
        for (int n = 0; n < nv; ++n)
            for (int i = lane; i < c4; i += 32) {
                const bool v = i < st.xrows;
                cp8(Xs + n * ldx + i, st.x + (int64_t)n * st.xld + (v ? i : 0), v);
            }
    }
}

}  // namespace cta

// NS-stage ring, WR x WC consumer warps (MT m-tiles x NT n-tiles each) + 1 producer warp.
template <int MT, int NT, int WR, int WC, int NS>
__global__ void __launch_bounds__((WR * WC + 1) * 32, 1) k_cta(const __grid_constant__ CtaJob j)
{
    using namespace cta;
    constexpr int NW = WR * WC, NVT = 8 * NT * WC;
    constexpr int AEL = CMAX * LDM, XEL = NVT * LDM, STAGE = AEL + XEL;
    extern __shared__ __align__(128) double sm[];
    Meta *meta = reinterpret_cast<Meta *>(sm + NS * STAGE);
    uint64_t *full = reinterpret_cast<uint64_t *>(meta + NS);
    uint64_t *empty = full + NS;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nv = j.nv;
    const int G = gridDim.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mb_init(full + i, 64);     // 32 producer lanes x (cp.async completion + release of generic stores)
            mb_init(empty + i, NW);    // one arrive per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (wid == NW) {
        // ================================================================ producer warp
        int it = 0;
        auto next_stage = [&]() {
            const int stg = it % NS;
            if (it >= NS) mb_wait(empty + stg, ((it / NS) - 1) & 1);
            return stg;
        };
        // descriptors are fetched ahead: the next task's Task / dense Task while this task streams,
        // and the Blk of 32 steps at a time (one per lane, broadcast by shuffles)
        const Task none{};
        auto load_task = [&](int t, Task &tk, Task &dk) {
            tk = t < j.ntask ? j.tasks[t] : none;
            dk = (t < j.ntask && j.kind == CK_LEAF) ? j.dtasks[t] : none;
        };
        Task ntk, ndk;
        load_task(blockIdx.x, ntk, ndk);
        for (int t = blockIdx.x; t < j.ntask; t += G) {
            const Task tk = ntk, dk = ndk;
            load_task(t + G, ntk, ndk);
            const int nst = j.kind == CK_LEAF ? tk.nblk + dk.nblk : tk.nblk;
            Meta m{};
            m.out = tk.out;
            m.nst = nst;
            m.tr = tk.r;
            m.rows = tk.rows;
            if (j.kind == CK_LEAF) {
                const Blk bU = j.blks[tk.blk0 + ((tk.flags & TF_HAS_E) ? 1 : 0)];
                m.zsrc = bU.x;
                m.kz = bU.xrows;
            }
            if (nst == 0) {
                const int stg = next_stage();
                m.flags = MF_EMPTY;
                if (lane == 0) meta[stg] = m;
                mb_arrive_cp(full + stg);
                mb_arrive(full + stg);
                ++it;
                continue;
            }
            for (int s0 = 0; s0 < nst; s0 += 32) {
                Blk mine{};
                if (s0 + lane < nst) mine = j.blks[step_blk(j, tk, dk, s0 + lane)];
                const int s1 = min(nst, s0 + 32);
                for (int s = s0; s < s1; ++s) {
                    const Step st = make_step(j, tk, dk, s, shfl_blk(mine, s - s0), m.kz);
                    const int stg = next_stage();
                    double *As = sm + stg * STAGE;
                    issue(st, As, As + AEL, nv, lane);
                    m.s = s;
                    m.r = st.r;
                    m.c = st.c;
                    m.flags = st.x ? 0 : MF_Z;
                    if (lane == 0) meta[stg] = m;
                    mb_arrive_cp(full + stg);
                    mb_arrive(full + stg);
                    ++it;
                }
            }
        }
        const int stg = next_stage();
        if (lane == 0) meta[stg].flags = MF_END;
        mb_arrive_cp(full + stg);
        mb_arrive(full + stg);
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        return;
    }

    // ==================================================================== consumer warps
    const int wr = wid % WR, wc = wid / WR;
    const int g = lane >> 2, t4 = lane & 3;
    const int row0 = wr * 8 * MT, col0 = wc * 8 * NT;
    const bool active = col0 < nv;
    double acc[MT][NT][2];
    auto each = [&](auto f) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int i = 0; i < 2; ++i) f(row0 + 8 * mt + g, col0 + 8 * nt + 2 * t4 + i, acc[mt][nt][i]);
    };
    for (int it = 0;; ++it) {
        const int stg = it % NS;
        mb_wait(full + stg, (it / NS) & 1);
        const Meta m = meta[stg];
        if (m.flags & MF_END) break;
        double *As = sm + stg * STAGE;
        double *Xs = As + AEL;
        if (m.flags & MF_EMPTY) {                      // empty coupling row (WRITE): y^ = 0
            each([&](int row, int n, double &) {
                if (row < m.tr && n < nv) j.dst[m.out + row + n * j.dst_ld] = 0.0;
            });
            __syncwarp();
            if (lane == 0) mb_arrive(empty + stg);
            continue;
        }
        if (m.s == 0) {                                // accumulator init
            const double *base = nullptr;
            int64_t ld = 0;
            int rows = 0;
            if (j.kind == CK_LEAF) { base = j.yh + m.zsrc; ld = j.yh_ld; rows = m.kz; }
            else if (j.kind == CK_ROWS && j.mode == MODE_ACCUM) { base = j.dst + m.out; ld = j.dst_ld; rows = m.tr; }
            each([&](int row, int n, double &v) { v = (base && row < rows && n < nv) ? base[row + n * ld] : 0.0; });
        }
        if (m.flags & MF_Z) {
            // leaf U step: hand z (k x nv, in the accumulators) over through this stage's x area
            const int ldz = ld_for(m.c), c4 = (m.c + 3) & ~3;
            each([&](int row, int n, double &v) {
                if (row < c4 && n < NVT) Xs[row + n * ldz] = row < m.kz ? v : 0.0;
                v = 0.0;
            });
            consumer_sync(NW * 32);
        }
        if (active) {
            const int lda = ld_for(m.r), ldx = ld_for(m.c), ksn = (m.c + 3) >> 2;
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
        __syncwarp();
        if (lane == 0) mb_arrive(empty + stg);
        if (m.s == m.nst - 1) {                        // store
            if (j.kind == CK_LEAF) {
                double *Y = j.args->Y;
                const int64_t ldy = j.args->ldy;
                const double alpha = j.args->alpha, beta = j.args->beta;
                each([&](int row, int n, double &v) {
                    if (row < m.rows && n < nv) {
                        double *p = Y + m.out + row + n * ldy;
                        *p = (beta == 0.0) ? alpha * v : fma(alpha, v, beta * *p);
                    }
                });
            } else {
                each([&](int row, int n, double &v) {
                    if (row < m.tr && n < nv) j.dst[m.out + row + n * j.dst_ld] = v;
                });
            }
        }
    }
}

// Engine shape from the widest output tile (rmax rows) and nv: WC vector chunks of 16, WR warp
// rows of 8 MT rows each; NS ring stages (the largest that fits 227 KB of shared memory).
cudaError_t launch_cta(const CtaJob &j, int rmax, int nsm, cudaStream_t s)
{
    if (j.ntask == 0) return cudaSuccess;
    const int grid = j.ntask < nsm ? j.ntask : nsm;
    cudaError_t err = cudaSuccess;
    auto go = [&](void (*kern)(CtaJob), int warps, int nvt, int ns) {
        const size_t smem = (size_t)ns * (cta::CMAX * cta::LDM + nvt * cta::LDM) * sizeof(double) +
                            ns * (sizeof(cta::Meta) + 2 * sizeof(uint64_t));
        static void *done[16] = {};
        bool set = false;
        for (void *d : done) set = set || d == (void *)kern;
        if (!set) {
            err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (err != cudaSuccess) return;
            for (void *&d : done)
                if (!d) { d = (void *)kern; break; }
        }
        kern<<<grid, (warps + 1) * 32, smem, s>>>(j);
        err = cudaGetLastError();
    };
    const bool big = rmax > 32;
    if (j.nv <= 16) {
        if (big) go(k_cta<2, 2, 4, 1, 4>, 4, 16, 4); else go(k_cta<1, 2, 4, 1, 4>, 4, 16, 4);
    } else if (j.nv <= 32) {
        if (big) go(k_cta<2, 2, 4, 2, 3>, 8, 32, 3); else go(k_cta<1, 2, 4, 2, 3>, 8, 32, 3);
    } else {
        // (MT, NT) = (4, 4) on 2 x 2 warps and (2, 4) on 4 x 2 warps measured 12 % / 0 % slower on cfg3
        if (big) go(k_cta<4, 2, 2, 4, 3>, 8, 64, 3); else go(k_cta<2, 2, 2, 4, 3>, 8, 64, 3);
    }
    return err;
}

}  // namespace h2
