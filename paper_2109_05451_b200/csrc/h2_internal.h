// h2_internal.h -- shared between the host plan (h2_api.cpp) and the kernels (h2_kernels.cu).
// Not part of the public ABI (include/h2.h is).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <string>
#include <vector>

namespace h2 {

// message returned by h2_last_error() on this thread (h2_api.cpp)
void set_last_error(const std::string &msg);

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
};

template <typename T>
cudaError_t launch_set_args(CallArgs<T> *a, const T *X, int64_t ldx, T *Y, int64_t ldy, T alpha, T beta,
                            cudaStream_t s);
// r = output rows of the phase's tasks (selects lanes-per-row / DMMA m-tiles)
template <typename T>
cudaError_t launch_up_leaf(const Task *t, int ntask, const Blk *b, const CallArgs<T> *args,
                           T *xh, int64_t xh_ld, int nv, int r, cudaStream_t s);
template <typename T>
cudaError_t launch_rows(int mode, const Task *t, int ntask, const Blk *b, const T *src,
                        int64_t src_ld, T *dst, int64_t dst_ld, int nv, int r, cudaStream_t s);
template <typename T>
cudaError_t launch_leaf_dense(const Task *lt, const Task *dt, int ntask, const Blk *b, const T *yh, int64_t yh_ld,
                              const CallArgs<T> *args, const T *halo, int nv, int k, int kp, int m, cudaStream_t s);
template <typename T>
cudaError_t launch_scale(T *Y, int64_t ldy, int64_t n, int nv, T beta, cudaStream_t s);
template <typename T>
cudaError_t launch_transpose(const T *src, T *dst, int64_t batch, int r, int c, cudaStream_t s);
// src == nullptr: read the caller's X from args (halo pack)
template <typename T>
cudaError_t launch_pack(const PackSeg *segs, int64_t nseg, const T *src, int64_t src_ld,
                        const CallArgs<T> *args, T *dst, int nv, cudaStream_t s);

enum { MODE_WRITE = 0, MODE_ACCUM = 1 };

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

// CTA-tile FP64 engine (h2_cta.cuh): one output node per CTA at a time, every block staged once
// in shared memory for all the CTA's warps.
enum { CK_ROWS = 0, CK_UPLEAF = 1, CK_LEAF = 2 };
struct CtaJob {
    const Task *tasks;       // primary tasks (rows / leaf projections / leaves [E][U])
    const Task *dtasks;      // CK_LEAF: dense row of the same leaf
    const Blk *blks;
    int ntask;
    int kind, mode;          // CK_*, MODE_WRITE / MODE_ACCUM (CK_ROWS)
    const double *src;       // CK_ROWS: x^ / y^ source plane (element offsets in Blk::x)
    int64_t src_ld;
    double *dst;             // CK_ROWS / CK_UPLEAF: output plane
    int64_t dst_ld;
    const double *yh;        // CK_LEAF: y^ plane (E's parent operand, z's own part)
    int64_t yh_ld;
    const double *halo;      // x rows received from peers (Blk::x < 0)
    const CallArgs<double> *args;
    int nv;
};
// Device-initiated peer exchange: a per-handle signal block in device
// memory, written by the peers through CUDA-IPC mappings over NVLink.  Layout (int32 slots):
constexpr int SIG_EPOCH = 0;        // my call counter
constexpr int SIG_XLEAF = 32;       // + o: peer o's leaf-level x^ is ready (its epoch)
constexpr int SIG_XUP = 96;         // + o: peer o's upper-level x^ is ready
constexpr int SIG_HALO = 160;       // + o: peer o packed the x rows I need
constexpr int SIG_CONS_X = 224;     // + o: peer o finished reading my x^
constexpr int SIG_CONS_H = 288;     // + o: peer o finished reading my packed x rows
constexpr int SIG_INTS = 352;       // (P <= 64)
// begin a call: epoch += 1, then wait until sig[waits[i]] >= epoch - 1 (WAR: peers done with the
// previous call's data); signal: *targets[i] = my epoch (release, system scope); wait: until
// sig[offs[i]] >= my epoch (acquire).  Spins are bounded (trap after ~20 s: no silent hang).
cudaError_t launch_p2p_begin(int32_t *sig, const int32_t *waits, int nwait, cudaStream_t s);
cudaError_t launch_p2p_signal(const int32_t *sig, int32_t *const *targets, int n, cudaStream_t s);
cudaError_t launch_p2p_wait(const int32_t *sig, const int32_t *offs, int n, cudaStream_t s);

// symmetric storage (h2_sym.cuh): blocks with Blk::xld == -1 are also applied transposed
template <typename T>
cudaError_t launch_sym_rows(const Task *t, int ntask, const Blk *b, const T *xh, T *yh, int r, cudaStream_t s);
template <typename T>
cudaError_t launch_sym_leaf(const Task *lt, const Task *dt, int ntask, const Blk *b, const T *yh,
                            const CallArgs<T> *args, int m, cudaStream_t s);
template <typename T>
cudaError_t launch_beta(const CallArgs<T> *args, int64_t n, int nv, cudaStream_t s);
// rmax: the widest output tile of the job's tasks; nsm: SMs (grid = min(ntask, nsm))
cudaError_t launch_cta(const CtaJob &j, int rmax, int nsm, cudaStream_t s);
// tcgen05 FP32 row engine (h2_umma.cuh): 3xTF32 on kind::tf32 MMAs, accumulators in TMEM; tasks
// with r, c <= 64, nv >= 5.  Same arguments as launch_rows<float> plus the SM count.
cudaError_t launch_umma_rows(int mode, const Task *t, int ntask, const Blk *b, const float *src, int64_t src_ld,
                             float *dst, int64_t dst_ld, int nv, int nsm, cudaStream_t s);
// The fused-leaf form (U y^_t + dense row, alpha/beta epilogue into Y; the leaf-level E transfer
// already applied to y^ by a rows launch).  xmap: 256-byte device slot holding the X tensor map
// and its valid flag, written per call by launch_set_xmap (before the captured graph).
cudaError_t launch_umma_leaf(const Task *lt, const Task *dt, int ntask, const Blk *b, const float *yh, int64_t yh_ld,
                             const CallArgs<float> *args, const float *halo, const void *xmap, int nv, int nsm,
                             cudaStream_t s);
cudaError_t launch_set_xmap(void *dmap, const float *X, int64_t ldx, int nv, cudaStream_t s);
// Basis orthogonalization in place (h2_k_orth.cu, NEXT-3 step 1): FP64, one GPU, full storage.
// pairs[l][b] = (t, s) of coupling block b of level l.  Synchronous on s.
cudaError_t orthogonalize_bases(double *U, double *Vt, const std::vector<double *> &E, const std::vector<double *> &Ft,
                                const std::vector<double *> &S, const std::vector<const int2 *> &pairs,
                                const std::vector<int64_t> &nblk, const int *k, int q, int m, cudaStream_t s);
// Reweighing downsweep (h2_k_orth.cu, NEXT-3 step 2): R^l_i of every node, root to leaves, into
// Rout (levels concatenated, 2^l x k^l x k^l column-major each); V must be orthogonal.
cudaError_t reweigh_downsweep(const std::vector<double *> &E, const std::vector<double *> &S,
                              const std::vector<const int64_t *> &rowptr, const std::vector<int> &maxb, const int *k,
                              int q, double *Rout, cudaStream_t s);
}  // namespace h2
