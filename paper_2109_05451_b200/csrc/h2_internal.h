// h2_internal.h -- shared between the host plan (h2_api.cpp) and the kernels (h2_kernels.cu).
// Not part of the public ABI (include/h2.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace h2 {

constexpr int KMAX = 64;   // max rank k^l and leaf size m supported by the kernels
constexpr int XLD = 64;    // leading dimension of a staged x operand in shared memory
constexpr int WPB = 8;     // warps per CTA of the row kernels

// One block of a row task: y_rows += A (r x c, column-major) * x (c x nv)
//   A     : device pointer to the block (already in the operand order the kernel wants)
//   x     : element offset of the x operand's first row in its source (plane layout:
//           element (j, n) at x + j + n * ld); for dense blocks x < 0 encodes a halo row
//           offset (-x - 1) into the received-leaf buffer
//   xrows : rows of x that are real (rows >= xrows are treated as 0: ragged leaves)
//   xld   : leading dimension (between vectors) of this block's x source; 0 = the launch's
//           default (per-peer receive chunks carry their own)
struct Blk {
    const void *A;
    int64_t x;
    int32_t xrows;
    int32_t xld;
};

// Task flags
constexpr uint8_t TF_HAS_E = 1;     // leaf kernel: first block is the parent transfer E_t
constexpr uint8_t TF_ACONTIG = 2;   // the task's (dense, for leaves) blocks are contiguous in
                                    // memory: A_b = A_0 + b * r * c  (streamed as one GEMM)

// One warp task: an output node / leaf and its list of blocks [blk0, blk0 + nblk).
struct Task {
    int64_t out;     // element offset of the output's first row (plane layout)
    int64_t blk0;
    int32_t nblk;
    uint8_t r;       // output rows (rank k, or leaf size m for the leaf kernel)
    uint8_t c;       // columns of every block in this task (k of the source level, or m)
    uint8_t rows;    // leaf kernel: real rows of this leaf (<= m)
    uint8_t flags;   // leaf kernel: bit0 = first block is the parent transfer E_t
};

// One contiguous run copied by the pack kernel: len rows of every vector.
struct PackSeg {
    int64_t src;     // element offset in the source (x^ workspace or X)
    int64_t dst;     // element offset in the send buffer
    int32_t len;
    int32_t dst_ld;  // distance between vectors in the destination (per-peer chunk)
};

// Kernel launchers (h2_kernels.cu).  T = double or float.  Each returns cudaGetLastError().
// Per-call arguments read by the kernels from device memory, so one captured CUDA graph per nv
// serves every call (k_set_args writes them, stream-ordered, before each graph launch).
template <typename T>
struct CallArgs {
    const T *X;
    T *Y;
    int64_t ldx, ldy;
    T alpha, beta;
    int32_t epoch;           // call counter: completion flags of the chain kernels hold it
    uint32_t ticket[4];      // work tickets of the chain kernels (reset every call)
    int32_t *counters;       // level-complete counters of the scheduled upsweep (reset per call)
    int32_t ncounters;
};

// Dependencies of one chain task (k_chain): it may start once flags[dep0] and flags[dep1]
// (-1 = none) equal the call's epoch; on completion it sets flags[self].
struct ChainDep {
    int32_t self, dep0, dep1, pad;
};
template <typename T>
cudaError_t launch_chain(int mode, const Task *t, const ChainDep *deps, int ntask, const Blk *b, T *buf,
                         int64_t ld, int nv, int r, int32_t *flags, CallArgs<T> *args, int which,
                         int max_ctas, cudaStream_t s);

template <typename T>
cudaError_t launch_set_args(CallArgs<T> *a, const T *X, int64_t ldx, T *Y, int64_t ldy, T alpha, T beta,
                            cudaStream_t s);
// r = output rows of the phase's tasks (selects lanes-per-row / DMMA m-tiles)
template <typename T>
cudaError_t launch_up_leaf(const Task *t, int ntask, const Blk *b, const CallArgs<T> *args,
                           T *xh, int64_t xh_ld, int nv, int r, cudaStream_t s);
// tma: stream contiguous block runs through the cp.async.bulk ring (else register loads)
// max_ctas > 0: cap the grid (tasks are grid-strided): persistent bandwidth kernels that leave
// SM room for the latency-bound tree chain running concurrently
template <typename T>
cudaError_t launch_rows(int mode, const Task *t, int ntask, const Blk *b, const T *src,
                        int64_t src_ld, T *dst, int64_t dst_ld, int nv, int r, bool tma, int max_ctas,
                        cudaStream_t s);
template <typename T>
cudaError_t launch_leaf_dense(const Task *lt, const Task *dt, int ntask, const Blk *b, const T *yh, int64_t yh_ld,
                              const CallArgs<T> *args, const T *halo, int nv, int k, int kp, int m, cudaStream_t s);
template <typename T>
cudaError_t launch_leaf_u(const Task *t, int ntask, const Blk *b, const T *yh, int64_t yh_ld,
                          const CallArgs<T> *args, int nv, int k, int kp, int m, cudaStream_t s);
template <typename T>
cudaError_t launch_dense(const Task *t, int ntask, const Blk *b, const CallArgs<T> *args, const T *halo,
                         int nv, int m, bool tma, int max_ctas, cudaStream_t s);
template <typename T>
cudaError_t launch_scale(T *Y, int64_t ldy, int64_t n, int nv, T beta, cudaStream_t s);
template <typename T>
cudaError_t launch_transpose(const T *src, T *dst, int64_t batch, int r, int c, cudaStream_t s);
// src == nullptr: read the caller's X from args (halo pack)
template <typename T>
cudaError_t launch_pack(const PackSeg *segs, int64_t nseg, const T *src, int64_t src_ld,
                        const CallArgs<T> *args, T *dst, int nv, cudaStream_t s);

enum { MODE_WRITE = 0, MODE_ACCUM = 1 };

// Launch priority for the next launches (0 = the stream's own).  Set by the host plan around the
// side-stream bandwidth kernels (low) and the sweep chain (high); applied with
// cudaLaunchKernelEx + cudaLaunchAttributePriority so it is also recorded in captured graphs.
inline int g_launch_priority = 0;

// A fused run of consecutive tree levels (see k_tree): per level, the first task of the phase
// and the number of tasks each CTA owns.
constexpr int TREE_MAXLEV = 8;
struct TreeStage {
    int64_t t0[TREE_MAXLEV];
    int32_t per[TREE_MAXLEV];   // tasks per CTA
    int32_t cnt[TREE_MAXLEV];   // tasks of the level
    int32_t nlev;
};
template <typename T>
cudaError_t launch_tree(int mode, const TreeStage &st, int nctas, const Task *t, const Blk *b, T *buf,
                        int64_t ld, int nv, int r, cudaStream_t s);

// Heap-addressed transfer levels (no task / block descriptors: every address follows from the
// node index, PAPER.md:135-142 nested bases; children of slot i are slots 2i, 2i+1):
//   up   (MODE_WRITE): out slot i of level l-1 = Ft_l[2i] x_l[2i] + Ft_l[2i+1] x_l[2i+1]
//   down (MODE_ACCUM): out slot c of level l  += E_l[c] y_{l-1}[c >> 1]
// Levels are processed in the order given; with one CTA the whole list runs in one launch with
// a CTA barrier between levels (the small top levels), with more CTAs exactly one level.
constexpr int SWEEP_MAXLEV = 32;
struct SweepLevel {
    const void *A;      // Ft_l (up) or E_l (down), first held node
    int64_t xbase;      // element offset of the source level's slot 0
    int64_t obase;      // element offset of the output level's slot 0
    int32_t n;          // output nodes of the level
    int16_t r, c;       // block rows (output rank) / columns (source rank)
};
struct SweepParams {
    SweepLevel lv[SWEEP_MAXLEV];
    int32_t nlev;
};
template <typename T>
cudaError_t launch_sweep(int mode, const SweepParams &p, int nctas, int threads, T *buf, int64_t ld, int nv,
                         int r, cudaStream_t s);
// Persistent scheduled kernels ("megakernels"): every warp takes the next entry of a
// topologically ordered schedule from an atomic ticket and waits on completion flags / level
// counters for its dependencies, so the latency-bound tree sweeps overlap with the bandwidth-
// bound coupling and dense work in ONE launch per sweep direction.
enum { ST_UPLEAF = 0, ST_UP = 1, ST_COUP = 2, ST_DOWN = 3, ST_LEAF = 4 };
struct SchedEntry {
    int16_t type, level;   // level: child level (ST_UP), row level (ST_COUP / ST_DOWN)
    int32_t idx;           // leaf / node slot, or task index (ST_COUP)
};
struct MegaParams {
    SweepLevel up[SWEEP_MAXLEV];     // by child level lc (parents at lc - 1), like the sweeps
    SweepLevel dn[SWEEP_MAXLEV];     // by level l
    int64_t fbase[SWEEP_MAXLEV + 1]; // flat node index of slot 0 of each level
    int32_t nodes[SWEEP_MAXLEV];     // held nodes per level (level-complete counter target)
    int32_t q;
    int32_t dn_first;                // first level computed by the downsweep entries
    int32_t k, kp;                   // k^q, k^{q-1} (leaf entries)
    int32_t kmax;                    // max k^l (engine selection for the downsweep entries)
};
template <typename T>
cudaError_t launch_mega_up(const SchedEntry *sched, int n, const MegaParams &mp, const Task *tasks, const Blk *blks,
                           const Task *upleaf_tasks, T *xh, int64_t xh_ld, T *yh, int64_t yh_ld, int32_t *flags,
                           int32_t *counters, CallArgs<T> *args, int nv, int r, int grid, cudaStream_t s);
template <typename T>
cudaError_t launch_mega_down(const SchedEntry *sched, int n, const MegaParams &mp, const Task *ltasks,
                             const Task *dtasks, const Blk *blks, T *yh, int64_t yh_ld, const T *halo,
                             int32_t *flags, CallArgs<T> *args, int nv, int m, int grid, cudaStream_t s);

// leaf projection fused with the first J (1 or 2) upsweep levels; lv.lv[j-1] = level q-j
template <typename T>
cudaError_t launch_up_subtree(const Task *leaf_tasks, int nleaf, const Blk *b, const CallArgs<T> *args, T *xh,
                              int64_t xh_ld, int nv, int r, int J, const SweepParams &lv, cudaStream_t s);

// L2 prefetch of byte ranges (the small top-level transfers, read late in the chain)
constexpr int PREFETCH_MAX = 64;
struct PrefetchList {
    const void *ptr[PREFETCH_MAX];
    int64_t bytes[PREFETCH_MAX];
    int32_t n;
};
cudaError_t launch_prefetch_l2(const PrefetchList &pl, cudaStream_t s);

}  // namespace h2
