// h2_umma.cuh -- FP32 row tasks on the 5th-generation tensor cores (DESIGN.md §7 "tcgen05 engine").
//
//   y (r x nv) (+)= sum_b A_b (r x c) x_b (c x nv)      (coupling PAPER.md:328-331, transfers 263-270)
//
// in split TF32: every operand v is split v = hi + lo with hi = v truncated to TF32 and
// lo = rn_tf32(v - hi) (hi + lo reproduces v to < 2^-21), and ONE tcgen05.mma.kind::tf32 per 8 columns computes all four
// products: the operand tiles are stacked, A' = [A_hi; A_lo] (M = 128) and x' = [x_hi, x_lo]
// (N = 2 nv), so D' = A' x' holds A_hi x_hi, A_hi x_lo, A_lo x_hi, A_lo x_lo in its four quadrants and
// y = their sum carries FP32 accuracy (north_star: FP32 runs <= 1e-5 against the FP64 oracle).
// (Three separate M = 64 MMAs per 8 columns -- 3xTF32 -- were issue-bound: ~94 cycles per MMA.)
//
// One CTA per SM, warp-specialised, one output node (x one chunk of N <= 64 vectors) at a time:
//   warp 4      PRODUCER   per block ONE bulk copy (cp.async.bulk, the TMA engine) of A_b -- r x c
//                          contiguous, column-major -- and ONE 4-D tensor copy of x_b (all N vectors,
//                          landing in the K-major layout; per-vector bulk copies for received rows)
//                          into an NR-stage raw ring, completing on raw_full[s] by transaction count;
//                          task / block descriptors fetched ahead (32 per warp load)
//   warps 6-13  CONVERTERS split every element into hi / lo and write both into an NC-stage
//                          operand ring in the K-major canonical no-swizzle layout (A transposed:
//                          each thread gathers 4 columns of one row), then fence.proxy.async so the
//                          tensor cores see the generic-proxy stores, and free the raw stage;
//   warp 5      MMA        the whole warp, one elected lane issuing all 8 tcgen05.mma (M=128,
//                          N=2 nv, K=8, both operands from shared memory) of a block in one asm
//                          statement, k-step k into partial accumulator k % NACC of one of NB TMEM
//                          buffers, fresh per block; commits to op_empty[s] and acc_full[b];
//   warps 0-3   EPILOGUE   tcgen05.ld the block's partial products (warp w reads TMEM lanes
//                          32w..32w+31: warps 0-1 hold the A_hi rows, 2-3 the A_lo rows) and add
//                          both column halves to a running sum in registers with IEEE FP32 adds --
//                          the tensor cores' own accumulation is not round-to-nearest and its bias
//                          over a whole coupling row measured 1.6e-5 on cfg5 (3xTF32 warp engine);
//                          per block it stays ~1e-6 -- then, per task, the A_lo half hands its sums
//                          to the A_hi half through shared memory, which stores / accumulates y.
// (MN-major A straight from the column-major copy would skip the transpose, but kind::tf32 with
// an MN-major descriptor -- no swizzle or 128-byte swizzle -- returned zeros on this B200
// (tools/umma_probe.cu).)
// A_b is read from HBM once per (task, vector chunk).  The converters and the MMA warp consume a
// descriptor-free block stream (an end marker closes it); the producer and the epilogue walk the
// task list in the same order (static round robin over persistent CTAs).
#pragma once
#include <cuda.h>
#include "h2_internal.h"

namespace h2 {
namespace umma {

constexpr int MM = 64;                 // UMMA M: output rows per tile (tasks with r <= 64)
constexpr int KC = 64;                 // max block columns
constexpr int W_PROD = 4, W_MMA = 5, W_CONV0 = 6, NCONV = 8, NEPI = 4, NWARPS = 14;

template <int N>
struct Cfg {
    static constexpr int AEL = MM * KC;             // floats of an A tile
    static constexpr int XEL = N * KC;              // floats of an x tile
    static constexpr int XLDR = KC + 4;             // raw x row pitch (272 B: conflict-free 16 B reads)
    static constexpr int RAW = AEL + N * XLDR;      // raw stage: A as in HBM (ld r), x vectors (ld XLDR)
    static constexpr int OPS = 2 * (AEL + XEL);     // operand stage: A hi, A lo, x hi, x lo
    static constexpr int NR = N <= 32 ? 4 : 2;
    static constexpr int NC = N <= 16 ? 3 : 2;
    // accumulators per block: k-step k accumulates into partial k % NACC, so the MMAs of a block
    // form NACC independent chains -- dependent MMAs on one accumulator serialise on the MMA
    // latency (measured: a 2-chain block of 8 M=128 x N=32 MMAs took ~1 us)
    static constexpr int NACC = 2;
    // accumulator buffers in flight (MMA of block b waits for the epilogue to drain block b - NB)
    static constexpr int NB = 512 / (NACC * 2 * N) < 4 ? 512 / (NACC * 2 * N) : 4;   // >= 2
    static constexpr int TCOLS = NB * NACC * 2 * N; // buffers x NACC partials x 2N columns (128..512)
    static constexpr int CMB = 64 * N;              // floats: the A_lo half's sums handed to the A_hi half
    static constexpr size_t SMEM = (size_t)(NR * RAW + NC * OPS + CMB) * sizeof(float) + 512;
};

// K-major canonical no-swizzle layout (core matrix = 8 rows x 16 bytes): element (row, j) of an
// operand with KC columns; 4-column chunks at 128 B (LBO), 8-row groups at KC * 32 B (SBO); the MMA
// of columns [8 ks, 8 ks + 8) starts at ks * 256 B.  Rows are output rows (A) or vectors (x).
__device__ __forceinline__ int k_off(int row, int j) { return (row >> 3) * (KC * 8) + (j >> 2) * 32 + (row & 7) * 4 + (j & 3); }
constexpr uint32_t KSTEP_BYTES = 256, LBO = 128, SBO = KC * 32;

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46);     // version 1, SWIZZLE_NONE
}
// kind::tf32 instruction descriptor: D F32, A/B TF32, both K-major, N, M
template <int M, int N>
__host__ __device__ constexpr uint32_t idesc()
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp4(float *dst, const float *src, bool valid)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(su32(dst)), "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(float *dst, const float *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
// 4-D tiled tensor copy (the x^ operand: see make_xmap) completing on an mbarrier
__device__ __forceinline__ void tensor4_g2s(float *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar)
{
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
                 ::"r"(su32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
                   "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_init(uint64_t *b, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_arrive_cp(uint64_t *b)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
// issued by the whole (converged) warp: one elected lane executes the MMA / commit
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc)
{
    asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
// The 8 MMAs of a full 64-column block in one asm statement: one elect, descriptors advanced by
// 256 B (+16 in the address field) per k-step, k-step k into partial k % NACC (fresh for k < NACC),
// partials PCOLS TMEM columns apart.  One statement per MMA cost ~48 cycles of issue each (elect +
// vote + moves on the uniform datapath, tools/umma_rate.cu) against a 16-cycle execution floor.
template <int NACC, int PCOLS>
__device__ __forceinline__ void mma8_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id)
{
    asm volatile(
        "{\n.reg .pred e, f, p<8>;\n.reg .b32 d<8>;\n.reg .b64 a<8>, b<8>;\n"
        "setp.ne.b32 f, 0, 0;\nelect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p1, %11, 0;\nsetp.ne.b32 p2, %12, 0;\nsetp.ne.b32 p3, %13, 0;\nsetp.ne.b32 p4, %14, 0;\n"
        "setp.ne.b32 p5, %15, 0;\nsetp.ne.b32 p6, %16, 0;\nsetp.ne.b32 p7, %17, 0;\n"
        "add.u32 d0, %0, 0;\nadd.u32 d1, %0, %4;\nadd.u32 d2, %0, %5;\nadd.u32 d3, %0, %6;\n"
        "add.u32 d4, %0, %7;\nadd.u32 d5, %0, %8;\nadd.u32 d6, %0, %9;\nadd.u32 d7, %0, %10;\n"
        "add.s64 a0, %1, 0;\nadd.s64 a1, %1, 16;\nadd.s64 a2, %1, 32;\nadd.s64 a3, %1, 48;\n"
        "add.s64 a4, %1, 64;\nadd.s64 a5, %1, 80;\nadd.s64 a6, %1, 96;\nadd.s64 a7, %1, 112;\n"
        "add.s64 b0, %2, 0;\nadd.s64 b1, %2, 16;\nadd.s64 b2, %2, 32;\nadd.s64 b3, %2, 48;\n"
        "add.s64 b4, %2, 64;\nadd.s64 b5, %2, 80;\nadd.s64 b6, %2, 96;\nadd.s64 b7, %2, 112;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d0], a0, b0, %3, f;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d1], a1, b1, %3, p1;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d2], a2, b2, %3, p2;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d3], a3, b3, %3, p3;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d4], a4, b4, %3, p4;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d5], a5, b5, %3, p5;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d6], a6, b6, %3, p6;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d7], a7, b7, %3, p7;\n}\n"
        ::"r"(d), "l"(a), "l"(b), "r"(id),
          "n"((1 % NACC) * PCOLS), "n"((2 % NACC) * PCOLS), "n"((3 % NACC) * PCOLS), "n"((4 % NACC) * PCOLS),
          "n"((5 % NACC) * PCOLS), "n"((6 % NACC) * PCOLS), "n"((7 % NACC) * PCOLS),
          "n"(1 >= NACC), "n"(2 >= NACC), "n"(3 >= NACC), "n"(4 >= NACC), "n"(5 >= NACC), "n"(6 >= NACC),
          "n"(7 >= NACC)
        : "memory");
}

__device__ __forceinline__ void commit(uint64_t *b)
{
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                 ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t ta, float *v)
{
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld8(uint32_t ta, float *v)
{
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// Round to the nearest TF32 value (ties away from zero) on the bit pattern: add half a TF32 ulp to
// the magnitude, clear the 13 dropped mantissa bits (2 integer ops; cvt.rna.tf32.f32 lowers to a
// branchy NaN-aware sequence).  Finite inputs only -- the operands of a matvec.
__device__ __forceinline__ float tf32_rn(float v) { return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xffffe000u); }
// hi = v truncated to TF32 (what the tensor core reads from v itself: measured truncation), lo =
// the exact remainder rounded to TF32: |v - hi - lo| <= 2^-11 |lo| < 2^-21 |v| (one integer op
// less per element than a round-to-nearest hi)
__device__ __forceinline__ float tf32_tr(float v) { return __uint_as_float(__float_as_uint(v) & 0xffffe000u); }
__device__ __forceinline__ void split4(const float4 &v, float4 &h, float4 &l)
{
    h.x = tf32_tr(v.x); l.x = tf32_rn(v.x - h.x);
    h.y = tf32_tr(v.y); l.y = tf32_rn(v.y - h.y);
    h.z = tf32_tr(v.z); l.z = tf32_rn(v.z - h.z);
    h.w = tf32_tr(v.w); l.w = tf32_rn(v.w - h.w);
}


}  // namespace umma

// One launch's work description (kernel parameter).  Rows (LEAF = false): task t = output node
// tasks[t], blocks blks[blk0 .. blk0 + nblk), x from src (plane ld src_ld, or per-block xld), output
// dst (+)= .  Leaf (LEAF = true): task t = leaf tasks[t] ([E][U]; E already applied to y^ by a
// rows launch) and dense row dtasks[t]; block 0 is U_t (x = y^_t from src), blocks 1.. the dense
// row (x = rows of the caller's X, or of the halo); output Y = alpha (U y^_t + sum D x) + beta Y.
struct UJob {
    const Task *tasks;
    const Task *dtasks;
    const Blk *blks;
    int ntask;
    int nv;
    const float *src;          // rows: x^ plane; leaf: y^ plane
    int64_t src_ld;
    float *dst;                // rows
    int64_t dst_ld;
    const CallArgs<float> *args;   // leaf: X, Y, ldx, ldy, alpha, beta
    const float *halo;             // leaf: x rows received from peers (Blk::x < 0)
    const CUtensorMap *xmap;       // leaf: tensor map of X in global memory (written per call, followed by
                                   // an int: valid for this call), or null
    int use_tm;                    // the kernel-parameter map (of src) is valid
};

namespace umma {
struct BInfo {
    const float *A;
    const float *x;
    int64_t ld;
    int r, c, xr;
    int tm;        // 0: no tensor copy, 1: the src map (kernel parameter), 2: the X map (global)
    int tc2;       // tensor coordinate of the block's first x row (row / 4)
};

__device__ __forceinline__ Blk shfl_blk(const Blk &b, int src)
{
    Blk o;
    o.A = reinterpret_cast<const void *>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(b.A), src));
    o.x = __shfl_sync(0xffffffffu, b.x, src);
    o.xrows = __shfl_sync(0xffffffffu, b.xrows, src);
    o.xld = __shfl_sync(0xffffffffu, b.xld, src);
    return o;
}

template <bool LEAF>
__device__ __forceinline__ int nblocks(const UJob &j, const Task &tk, int t)
{
    return LEAF ? 1 + j.dtasks[t].nblk : tk.nblk;
}

}  // namespace umma

template <int N, int MODE, bool LEAF>
__global__ void __launch_bounds__(umma::NWARPS * 32, 1)
k_umma(const __grid_constant__ UJob j, const __grid_constant__ CUtensorMap tmx)
{
    using namespace umma;
    using C = Cfg<N>;
    constexpr int NR = C::NR, NC = C::NC;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *ops = reinterpret_cast<float *>(smem_raw);                  // NC operand stages (MMA reads)
    float *raw = ops + NC * C::OPS;                                    // NR raw stages (copies land)
    uint64_t *bars = reinterpret_cast<uint64_t *>(raw + NR * C::RAW);
    uint64_t *raw_full = bars, *raw_empty = bars + NR, *op_full = bars + 2 * NR, *op_empty = op_full + NC;
    uint64_t *acc_full = op_empty + NC, *acc_empty = acc_full + C::NB;
    int4 *meta = reinterpret_cast<int4 *>(acc_empty + C::NB);          // per raw stage: c, A ld, x rows, c8
    int *opmeta = reinterpret_cast<int *>(meta + NR);                  // per operand stage: k-steps (0: end)
    uint32_t *tbase_p = reinterpret_cast<uint32_t *>(opmeta + NC);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int G = gridDim.x;
    const int nv = j.nv;
    const int nch = (nv + N - 1) / N;
    const int nwork = j.ntask * nch;

    if (threadIdx.x == 0) {
        for (int i = 0; i < NR; ++i) {
            mb_init(raw_full + i, 1);        // producer lane 0 (expect_tx, or after its 4-byte copies)
            mb_init(raw_empty + i, NCONV);
        }
        for (int i = 0; i < NC; ++i) {
            mb_init(op_full + i, NCONV);
            mb_init(op_empty + i, 1);        // tcgen05.commit
        }
        for (int i = 0; i < C::NB; ++i) {
            mb_init(acc_full + i, 1);
            mb_init(acc_empty + i, NEPI);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (wid == W_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tbase_p)),
                     "n"(C::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tbase_p;

    if (wid == W_PROD) {
        // ===================================================================== producer
        // A_b (r x c, contiguous) as one bulk copy; x either as ONE tensor copy of all N vectors
        // straight into the K-major layout (plane sources, the caller's X through the per-call
        // map), or one bulk copy per vector into [n][XLDR] (received rows), or 4-byte cp.async
        // (odd shapes), then a plain arrive once those landed.  (The TMA engine serialises
        // requests at ~125 cycles each: 17 requests per block -- A plus 16 vectors -- paced the
        // kernel at ~2 us per block.)
        bool xmap_ok = false;
        if (LEAF && j.xmap) {
            xmap_ok = *reinterpret_cast<const volatile int *>(reinterpret_cast<const char *>(j.xmap) + 128) != 0;
            if (xmap_ok && lane == 0)
                asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(j.xmap) : "memory");
        }
        __syncwarp();
        // descriptors are fetched ahead -- the next work item's task (and dense row) while this one
        // streams, and the Blk of 32 blocks at a time (one per lane, broadcast by shuffles) -- so
        // the producer's per-block work is a few register operations and the copies (dependent
        // descriptor loads from L2 per block measured ~1 us per block on the single producer warp)
        const float *X = nullptr;
        int64_t ldx = 0;
        if (LEAF) { X = j.args->X; ldx = j.args->ldx; }
        const Task none{};
        Task tn = blockIdx.x < nwork ? j.tasks[blockIdx.x / nch] : none;
        Task dn = (LEAF && blockIdx.x < nwork) ? j.dtasks[blockIdx.x / nch] : none;
        int it = 0;
        for (int w = blockIdx.x; w < nwork; w += G) {
            const int t = w / nch, n0 = (w - t * nch) * N;
            const int nvc = min(N, nv - n0);
            const Task tk = tn, dk = dn;
            if (w + G < nwork) {
                tn = j.tasks[(w + G) / nch];
                if (LEAF) dn = j.dtasks[(w + G) / nch];
            }
            const int nb = LEAF ? 1 + dk.nblk : tk.nblk;
            const int64_t ublk = tk.blk0 + ((LEAF && (tk.flags & TF_HAS_E)) ? 1 : 0);
            for (int s0 = 0; s0 < nb; s0 += 32) {
                Blk mine{};
                {
                    const int q = s0 + lane;
                    if (q < nb) mine = j.blks[LEAF ? (q == 0 ? ublk : dk.blk0 + q - 1) : tk.blk0 + q];
                }
                const int s1 = min(nb, s0 + 32);
                for (int bi = s0; bi < s1; ++bi, ++it) {
                const Blk b = shfl_blk(mine, bi - s0);
                const int s = it % NR;
                if (it >= NR) mb_wait(raw_empty + s, ((it / NR) - 1) & 1);
                BInfo bk;
                bk.A = static_cast<const float *>(b.A);
                bk.xr = b.xrows;
                bk.tc2 = (int)(b.x >> 2);
                if (!LEAF) {
                    bk.r = tk.r;
                    bk.c = tk.c;
                    bk.ld = b.xld ? (int64_t)b.xld : j.src_ld;
                    bk.x = j.src + b.x + (int64_t)n0 * bk.ld;
                    bk.tm = (j.use_tm && !b.xld && !(b.x & 3) && b.xrows == bk.c) ? 1 : 0;
                } else if (bi == 0) {
                    bk.r = tk.r;
                    bk.c = b.xrows;
                    bk.ld = j.src_ld;
                    bk.x = j.src + b.x + (int64_t)n0 * bk.ld;
                    bk.tm = (j.use_tm && !(b.x & 3)) ? 1 : 0;
                } else {
                    bk.r = dk.r;
                    bk.c = dk.c;
                    if (b.x >= 0) {
                        bk.ld = ldx;
                        bk.x = X + b.x + (int64_t)n0 * ldx;
                        bk.tm = (xmap_ok && !(b.x & 3) && b.xrows == bk.c) ? 2 : 0;
                    } else {
                        bk.ld = b.xld;
                        bk.x = j.halo + (-b.x - 1) + (int64_t)n0 * bk.ld;
                        bk.tm = 0;
                    }
                }
                const int r = bk.r, c = bk.c, c8 = max(16, (c + 7) & ~7), xr = bk.xr;   // >= 2 k-steps
                const float *A = bk.A, *x = bk.x;
                const int64_t ld = bk.ld;
                float *As = raw + s * C::RAW, *Xs = As + C::AEL;
                const bool abulk = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && !((r * c) & 3) && !(r & 3);
                const bool xbulk = ((reinterpret_cast<uintptr_t>(x) & 15) == 0) && !(ld & 3) && !(xr & 3) && xr > 0;
                const int xtm = (n0 & 7) ? 0 : bk.tm;
                if (lane == 0) meta[s] = make_int4(c, abulk ? r : MM, xr, c8 | (xtm ? 0x10000 : 0));
                if (abulk && (xtm || xbulk)) {
                    if (lane == 0) {
                        mb_expect_tx(raw_full + s, (uint32_t)(r * c) * 4u +
                                                       (xtm ? (uint32_t)C::XEL * 4u : (uint32_t)(nvc * xr) * 4u));
                        bulk_g2s(As, A, (uint32_t)(r * c) * 4u, raw_full + s);
                        if (xtm == 1) tensor4_g2s(Xs, &tmx, 0, 0, bk.tc2, n0 >> 3, raw_full + s);
                        else if (xtm == 2) tensor4_g2s(Xs, j.xmap, 0, 0, bk.tc2, n0 >> 3, raw_full + s);
                    }
                    __syncwarp();
                    if (!xtm)
                        for (int n = lane; n < nvc; n += 32)
                            bulk_g2s(Xs + n * C::XLDR, x + (int64_t)n * ld, (uint32_t)xr * 4u, raw_full + s);
                } else {
                    const int la = abulk ? r : MM;
                    for (int q = lane; q < c * r; q += 32) {
                        const int m = q % r, jj = q / r;
                        cp4(As + jj * la + m, A + (int64_t)jj * r + m, true);
                    }
                    for (int q = lane; q < nvc * xr; q += 32) {
                        const int jj = q % xr, n = q / xr;
                        cp4(Xs + n * C::XLDR + jj, x + (int64_t)n * ld + jj, true);
                    }
                    asm volatile("cp.async.wait_all;\n" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mb_arrive(raw_full + s);
                }
                }
            }
        }
        // end of this CTA's block stream: converters and the MMA warp need no task descriptors
        const int s = it % NR;
        if (it >= NR) mb_wait(raw_empty + s, ((it / NR) - 1) & 1);
        if (lane == 0) {
            meta[s] = make_int4(-1, 0, 0, 0);
            mb_arrive(raw_full + s);
        }
    } else if (wid >= W_CONV0) {
        // ===================================================================== converters
        const int ct = threadIdx.x - W_CONV0 * 32;              // 0 .. NCONV * 32 - 1
        constexpr int CJ = NCONV * 32 / MM;                     // 4-column chunk groups (4)
        const int cm = ct & (MM - 1), cjh = ct / MM;            // A: row, first 4-column chunk
        for (int it = 0;; ++it) {
            {
                const int rs = it % NR, cs = it % NC;
                mb_wait(raw_full + rs, (it / NR) & 1);
                if (it >= NC) mb_wait(op_empty + cs, ((it / NC) - 1) & 1);
                const int4 mt = meta[rs];
                if (mt.x < 0) {                                  // end marker: pass it on
                    __syncwarp();
                    if (lane == 0) {
                        if (ct == 0) opmeta[cs] = 0;
                        mb_arrive(op_full + cs);
                    }
                    break;
                }
                const int c = mt.x, la = mt.y, xr = mt.z, c8 = mt.w & 0xffff;
                const bool xk = mt.w >> 16;
                const float *Ar = raw + rs * C::RAW, *Xr = Ar + C::AEL;
                float *Ah = ops + cs * C::OPS, *Al = Ah + C::AEL, *Xh = Al + C::AEL, *Xl = Xh + C::XEL;
                // A: thread = (row m, every CJ-th 4-column chunk); a warp reads 32 consecutive rows of
                // one column per LDS (conflict-free) and writes 32 rows' 16-byte chunks (8 distinct
                // banks per phase).  Columns >= c are zero (x rows there are zero too, but 0 x stale
                // could be NaN); rows >= r are zero.
                if (la == MM && c == KC) {
                    // full 64 x 64 block (every coupling block of a rank-64 level): constant offsets,
                    // all loads of the thread's 16 columns in flight at once
                    const float *ap = Ar + cm;
#pragma unroll
                    for (int i = 0; i < KC / (4 * CJ); ++i) {
                        const int jj = 4 * (cjh + CJ * i);
                        float4 v = make_float4(ap[(jj + 0) * MM], ap[(jj + 1) * MM], ap[(jj + 2) * MM], ap[(jj + 3) * MM]);
                        float4 h, l;
                        split4(v, h, l);
                        const int o = k_off(cm, jj);
                        *reinterpret_cast<float4 *>(Ah + o) = h;
                        *reinterpret_cast<float4 *>(Al + o) = l;
                    }
                } else {
                    const bool mrow = cm < la;
                    for (int jj = 4 * cjh; jj < c8; jj += 4 * CJ) {
                        float4 v;
                        v.x = (mrow && jj + 0 < c) ? Ar[(jj + 0) * la + cm] : 0.f;
                        v.y = (mrow && jj + 1 < c) ? Ar[(jj + 1) * la + cm] : 0.f;
                        v.z = (mrow && jj + 2 < c) ? Ar[(jj + 2) * la + cm] : 0.f;
                        v.w = (mrow && jj + 3 < c) ? Ar[(jj + 3) * la + cm] : 0.f;
                        float4 h, l;
                        split4(v, h, l);
                        const int o = k_off(cm, jj);
                        *reinterpret_cast<float4 *>(Ah + o) = h;
                        *reinterpret_cast<float4 *>(Al + o) = l;
                    }
                }
                if (xk) {
                    // x already in the K-major layout (tensor copy): split in place, rows >= xr zero
                    for (int q = ct; q < C::XEL / 4; q += NCONV * 32) {
                        const int jj = 4 * ((q & 127) >> 3);
                        if (jj >= c8) continue;
                        float4 v = *reinterpret_cast<const float4 *>(Xr + 4 * q);
                        if (jj + 4 > xr) {
                            if (jj + 0 >= xr) v.x = 0.f;
                            if (jj + 1 >= xr) v.y = 0.f;
                            if (jj + 2 >= xr) v.z = 0.f;
                            if (jj + 3 >= xr) v.w = 0.f;
                        }
                        float4 h, l;
                        split4(v, h, l);
                        *reinterpret_cast<float4 *>(Xh + 4 * q) = h;
                        *reinterpret_cast<float4 *>(Xl + 4 * q) = l;
                    }
                } else {
                    // x: vector-fastest over (vector, 4-row chunk); rows >= xr are zero (vectors >= nvc
                    // are stale: their output columns are never stored)
                    const int nq = c8 >> 2;
                    for (int q = ct; q < N * nq; q += NCONV * 32) {
                        const int n = q % N, jj = 4 * (q / N);
                        float4 v = *reinterpret_cast<const float4 *>(Xr + n * C::XLDR + jj);
                        if (jj + 4 > xr) {
                            if (jj + 0 >= xr) v.x = 0.f;
                            if (jj + 1 >= xr) v.y = 0.f;
                            if (jj + 2 >= xr) v.z = 0.f;
                            if (jj + 3 >= xr) v.w = 0.f;
                        }
                        float4 h, l;
                        split4(v, h, l);
                        const int o = k_off(n, jj);
                        *reinterpret_cast<float4 *>(Xh + o) = h;
                        *reinterpret_cast<float4 *>(Xl + o) = l;
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    if (ct == 0) opmeta[cs] = c8 >> 3;
                    mb_arrive(raw_empty + rs);
                    mb_arrive(op_full + cs);
                }
            }
        }
    } else if (wid == W_MMA) {
        // ===================================================================== MMA issuer (whole warp)
        constexpr uint32_t ID = idesc<128, 2 * N>();
        const uint32_t ops_a = su32(ops);
        for (int it = 0;; ++it) {
            {
                const int cs = it % NC, ab = it % C::NB;
                mb_wait(op_full + cs, (it / NC) & 1);
                const int ksn = opmeta[cs];
                if (ksn == 0) break;                              // end marker
                if (it >= C::NB) mb_wait(acc_empty + ab, ((it / C::NB) - 1) & 1);
                tc_fence_after();
                const uint32_t hA = ops_a + (uint32_t)(cs * C::OPS) * 4u;     // [A_hi; A_lo], 128 rows
                const uint32_t hX = hA + 2 * C::AEL * 4u;                     // [x_hi, x_lo], 2N rows
                const uint32_t d0 = tmem + (uint32_t)(ab * C::NACC * 2 * N);
                if (ksn == 8) {
                    mma8_tf32<C::NACC, 2 * N>(d0, sdesc(hA, LBO, SBO), sdesc(hX, LBO, SBO), ID);
                } else {
                    for (int k = 0; k < ksn; ++k)
                        mma_tf32(d0 + (uint32_t)((k % C::NACC) * 2 * N), sdesc(hA + k * KSTEP_BYTES, LBO, SBO),
                                 sdesc(hX + k * KSTEP_BYTES, LBO, SBO), ID, k >= C::NACC);
                }
                commit(op_empty + cs);
                commit(acc_full + ab);
            }
        }
    } else {
        // ===================================================================== epilogue (warps 0-3)
        const int row = threadIdx.x & 63, half = threadIdx.x >> 6;   // TMEM lane = M row: A_hi / A_lo half
        const uint32_t tl = tmem + ((uint32_t)(wid * 32) << 16);
        float *cmb = reinterpret_cast<float *>(smem_raw + (size_t)(NC * C::OPS + NR * C::RAW) * 4 + 512);
        int it = 0;
        for (int w = blockIdx.x; w < nwork; w += G) {
            const int t = w / nch, n0 = (w - t * nch) * N;
            const int nvc = min(N, nv - n0);
            const Task tk = j.tasks[t];
            const int nb = nblocks<LEAF>(j, tk, t);
            const bool live = row < (LEAF ? (int)tk.rows : (int)tk.r);
            float *out;
            int64_t old;
            if (LEAF) { old = j.args->ldy; out = j.args->Y + tk.out + row + (int64_t)n0 * old; }
            else      { old = j.dst_ld; out = j.dst + tk.out + row + (int64_t)n0 * old; }
            float acc[N];
#pragma unroll
            for (int n = 0; n < N; ++n)
                acc[n] = (!LEAF && MODE == MODE_ACCUM && half == 0 && live && n < nvc) ? out[(int64_t)n * old] : 0.f;
            for (int bi = 0; bi < nb; ++bi, ++it) {
                constexpr int npart = C::NACC;                  // every block has >= NACC k-steps
                const int ab = it % C::NB;
                mb_wait(acc_full + ab, (it / C::NB) & 1);
                tc_fence_after();
#pragma unroll
                for (int a = 0; a < npart; ++a) {
                    const uint32_t ta = tl + (uint32_t)((ab * C::NACC + a) * 2 * N);
#pragma unroll
                    for (int q = 0; q < N; q += 16) {
                        float v[16], u[16];
                        if constexpr (N >= 16) { tmem_ld16(ta + (uint32_t)q, v); tmem_ld16(ta + (uint32_t)(N + q), u); }
                        else { tmem_ld8(ta + (uint32_t)q, v); tmem_ld8(ta + (uint32_t)(N + q), u); }
#pragma unroll
                        for (int i = 0; i < (N >= 16 ? 16 : N); ++i) acc[q + i] += v[i] + u[i];
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mb_arrive(acc_empty + ab);
            }
            // the A_lo half hands its sums to the A_hi half (conflict-free: row fastest)
            if (half == 1) {
#pragma unroll
                for (int n = 0; n < N; ++n) cmb[n * 64 + row] = acc[n];
            }
            asm volatile("bar.sync 1, 128;\n" ::: "memory");
            if (half == 0 && live) {
                if (LEAF) {
                    const float alpha = j.args->alpha, beta = j.args->beta;
#pragma unroll
                    for (int n = 0; n < N; ++n)
                        if (n < nvc) {
                            float *p = out + (int64_t)n * old;
                            const float v = acc[n] + cmb[n * 64 + row];
                            *p = (beta == 0.f) ? alpha * v : fmaf(alpha, v, beta * *p);
                        }
                } else {
#pragma unroll
                    for (int n = 0; n < N; ++n)
                        if (n < nvc) out[(int64_t)n * old] = acc[n] + cmb[n * 64 + row];
                }
            }
            asm volatile("bar.sync 1, 128;\n" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (wid == W_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(C::TCOLS));
    }
}

// Tensor map of an x^ plane workspace (or of the caller's X: the same column-major form) for one
// N-vector chunk: 4-D view (j % 4, n % 8, j / 4, n / 8) with strides (4 B, ld, 16 B, 8 ld) so a
// {4, 8, 16, N / 8} box lands in shared memory in exactly the K-major canonical layout of k_off
// (row = vector).  Needs nv % 8 == 0 (no plane past the last one is addressed) and 16-byte
// aligned planes.
static bool make_xmap(CUtensorMap *m, const float *src, int64_t ld, int nv, int N)
{
    using Encode = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode encode = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<Encode>(fn);
    }();
    if (!encode || !src || (nv & 7) || (ld & 3) || ld <= 0 || (reinterpret_cast<uintptr_t>(src) & 15)) return false;
    const cuuint64_t dims[4] = {4, 8, (cuuint64_t)(ld / 4), (cuuint64_t)(nv / 8)};
    const cuuint64_t strides[3] = {(cuuint64_t)ld * 4, 16, (cuuint64_t)ld * 32};
    const cuuint32_t box[4] = {4, 8, (cuuint32_t)(umma::KC / 4), (cuuint32_t)(N / 8)};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(src), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static inline int umma_chunk(int nv) { return nv <= 8 ? 8 : (nv <= 16 ? 16 : (nv <= 32 ? 32 : 64)); }

template <bool LEAF>
static cudaError_t launch_umma(int mode, UJob j, int nsm, cudaStream_t s)
{
    if (j.ntask == 0) return cudaSuccess;
    cudaError_t err = cudaSuccess;
    auto go = [&](auto nt) {
        constexpr int N = decltype(nt)::value;
        using C = umma::Cfg<N>;
        auto kw = k_umma<N, MODE_WRITE, LEAF>;
        auto ka = k_umma<N, MODE_ACCUM, LEAF>;
        static cudaError_t attr = [&] {
            cudaError_t e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
            return e == cudaSuccess ? cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) : e;
        }();
        if ((err = attr) != cudaSuccess) return;
        const int nwork = j.ntask * ((j.nv + N - 1) / N);
        const int grid = nwork < nsm ? nwork : nsm;
        alignas(64) CUtensorMap tm;
        memset(&tm, 0, sizeof tm);
        j.use_tm = make_xmap(&tm, j.src, j.src_ld, j.nv, N) ? 1 : 0;
        if (mode == MODE_WRITE || LEAF) kw<<<grid, umma::NWARPS * 32, C::SMEM, s>>>(j, tm);
        else                            ka<<<grid, umma::NWARPS * 32, C::SMEM, s>>>(j, tm);
        err = cudaGetLastError();
    };
    switch (umma_chunk(j.nv)) {
    case 8: go(std::integral_constant<int, 8>{}); break;
    case 16: go(std::integral_constant<int, 16>{}); break;
    case 32: go(std::integral_constant<int, 32>{}); break;
    default: go(std::integral_constant<int, 64>{}); break;
    }
    return err;
}

cudaError_t launch_umma_rows(int mode, const Task *t, int ntask, const Blk *b, const float *src, int64_t src_ld,
                             float *dst, int64_t dst_ld, int nv, int nsm, cudaStream_t s)
{
    UJob j{};
    j.tasks = t;
    j.blks = b;
    j.ntask = ntask;
    j.nv = nv;
    j.src = src;
    j.src_ld = src_ld;
    j.dst = dst;
    j.dst_ld = dst_ld;
    return launch_umma<false>(mode, j, nsm, s);
}

cudaError_t launch_umma_leaf(const Task *lt, const Task *dt, int ntask, const Blk *b, const float *yh, int64_t yh_ld,
                             const CallArgs<float> *args, const float *halo, const void *xmap, int nv, int nsm,
                             cudaStream_t s)
{
    UJob j{};
    j.tasks = lt;
    j.dtasks = dt;
    j.blks = b;
    j.ntask = ntask;
    j.nv = nv;
    j.src = yh;
    j.src_ld = yh_ld;
    j.args = args;
    j.halo = halo;
    j.xmap = static_cast<const CUtensorMap *>(xmap);
    return launch_umma<true>(MODE_WRITE, j, nsm, s);
}

// Per call, before the (captured) matvec: the X tensor map written into device memory by a
// one-thread kernel (stream-ordered: no host buffer reuse race), released to the tensormap proxy.
__global__ void k_set_xmap(CUtensorMap *dst, const __grid_constant__ CUtensorMap m, int valid)
{
    const uint4 *s4 = reinterpret_cast<const uint4 *>(&m);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    for (int i = threadIdx.x; i < (int)(sizeof(CUtensorMap) / 16); i += blockDim.x) d4[i] = s4[i];
    if (threadIdx.x == 0) reinterpret_cast<int *>(dst)[32] = valid;
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("fence.proxy.tensormap::generic.release.gpu;\n" ::: "memory");
}

cudaError_t launch_set_xmap(void *dmap, const float *X, int64_t ldx, int nv, cudaStream_t s)
{
    alignas(64) CUtensorMap m;
    memset(&m, 0, sizeof m);
    const int valid = make_xmap(&m, X, ldx, nv, umma_chunk(nv)) ? 1 : 0;
    k_set_xmap<<<1, 8, 0, s>>>(static_cast<CUtensorMap *>(dmap), m, valid);
    return cudaGetLastError();
}

}  // namespace h2
