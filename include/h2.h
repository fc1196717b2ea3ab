/*
 * h2.h -- C ABI of the B200-native distributed H^2 matrix-vector product
 *
 *     Y := alpha * A * X + beta * Y,    A = A_de + <U, S, V^T>
 *
 * for nv right-hand sides, computed by upsweep (alg:upsweep2), per-level
 * coupling multiply (alg:mult), downsweep (alg:downsweep)
 * and the dense near field, distributed by block rows (PAPER.md:195-206,
 * 439-502, alg:optimized_dist_mult).  All arithmetic runs in CUDA kernels for sm_100a; there
 * is no CPU fallback.  No torch types cross this boundary: plain pointers and sizes only.
 *
 * ---- Conventions ------------------------------------------------------------------------
 * Levels: global numbering, root = 0, leaves = depth q (reading R2).  Node i of
 *   level l (0 <= i < 2^l) has children 2i, 2i+1 (heap order).
 * Small matrices: column-major.  A batch of r x c matrices is r*c contiguous elements each.
 * Element type: dtype H2_F64 (double) or H2_F32 (float) for every floating array, X and Y.
 * Distribution (nranks = P, a power of two, P <= 2^q; C = log2 P is the C-level): rank p owns
 *   the branch rooted at node (C, p): at level l >= C the nodes p*2^(l-C) .. (p+1)*2^(l-C)-1,
 *   its leaves, their rows of X and Y (a contiguous tree-order row range), and the block rows
 *   of those nodes.  Levels l < C form the top tree, REPLICATED on every rank (reading R16).
 *   With nranks == 1, C = 0 and the branch is the whole tree.
 * X, Y: n_local x nv, column-major, leading dimension ld (>= n_local), rows in cluster-tree
 *   order, device memory (h2_matvec*) or host memory (h2_matvec_host).
 *
 * ---- Errors -----------------------------------------------------------------------------
 * Every entry point returns H2_OK (0) or a negative code and never throws or aborts.
 * h2_last_error() describes the last failure on the calling thread.  A CUDA or NCCL failure
 * inside a handle is sticky: later calls on it return H2_ERR_STATE.
 */
#ifndef H2_B200_H
#define H2_B200_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    H2_OK = 0,
    H2_ERR_ARG = -1,     /* bad argument (NULL, nv out of range, unknown dtype, ...)        */
    H2_ERR_SHAPE = -2,   /* sizes inconsistent (k or m above the supported 64, ld < n, ...) */
    H2_ERR_STRUCT = -3,  /* structural error in the tree / CSR description (see h2_create)  */
    H2_ERR_CUDA = -4,    /* CUDA runtime error                                              */
    H2_ERR_NCCL = -5,    /* NCCL error or NCCL library not loadable                         */
    H2_ERR_OOM = -6,     /* device allocation failed                                        */
    H2_ERR_STATE = -7    /* handle unusable after an earlier sticky error                   */
};
enum { H2_F64 = 0, H2_F32 = 1 };
enum { H2_MEM_HOST = 0,     /* floating arrays are host memory: copied, caller may free      */
       H2_MEM_DEVICE = 1 }; /* floating arrays are device memory: adopted (zero copy), the
                               caller keeps them alive until h2_destroy                      */

/* One rank's view of the H^2 matrix (PAPER.md:124-150 data; PAPER.md:195-206 distribution).
 * "held nodes at level l" = the 2^(l-C) branch nodes for l >= C, all 2^l nodes for l < C.
 * Integer arrays are always HOST memory (the plan is built on the host, once). */
typedef struct {
    int32_t dtype;               /* H2_F64 | H2_F32                                            */
    int32_t mem;                 /* H2_MEM_HOST | H2_MEM_DEVICE (floating arrays only)         */
    int32_t depth;               /* q: leaf level                                              */
    int32_t leaf_size;           /* m: max rows per leaf; leaf blocks padded to m rows        */
    int32_t rank, nranks;        /* p, P                                                       */
    int64_t n_local;             /* rows of X / Y on this rank                                 */
    const int32_t *level_rank;   /* [q+1] k^l, 1 <= k^l <= 64 ("fixed rank per level",
                                    PAPER.md:124)                                              */
    const int64_t *leaf_ptr;     /* [2^(q-C) + 1] local row offsets of my leaves; leaf_ptr[0]=0,
                                    leaf_ptr[end] = n_local, each leaf 1..m rows (ragged ok)   */
    const void *U_leaf;          /* my leaves: [2^(q-C)][m x k^q] col-major; padding rows 0     */
    const void *V_leaf;          /* same shape; may alias U_leaf                               */
    const void *const *E;        /* [q+1]; E[l] (l>=1): held nodes x [k^l x k^(l-1)] col-major,
                                    the transfer of node c to its parent;
                                    E[0] unused (reading R1)                                   */
    const void *const *F;        /* same shape; may alias E                                    */
    const int64_t *const *S_rowptr; /* [q+1]; level l: [held nodes + 1] CSR of coupling block
                                    rows; level 0 may have no blocks            */
    const int32_t *const *S_col; /* [q+1]; GLOBAL column node index at level l (may be remote) */
    const void *const *S;        /* [q+1]; per block k^l x k^l col-major, CSR order            */
    const int64_t *D_rowptr;     /* [2^(q-C) + 1] dense block rows of my leaves */
    const int32_t *D_col;        /* GLOBAL leaf index (may be remote)                          */
    const void *D;               /* per block m x m col-major, zero-padded                     */
    int32_t flags;               /* H2_SYMMETRIC or 0 (see below)                              */
} h2_desc;

/* h2_desc.flags.  H2_SYMMETRIC: the caller asserts the operator is symmetric with a symmetric block
 * structure -- U = V (V_leaf must be the same array as U_leaf), E = F, S^l_st = (S^l_ts)^T and
 * D_st = (D_ts)^T -- and the library stores only the blocks (t, s) with t <= s, applying each
 * stored off-diagonal block also transposed (y_s += A_ts^T x_t) from the same read: about half the
 * coupling and dense bytes per matvec (a representation change outside
 * the paper).  Supported for nv_max == 1 and nranks == 1 (H2_ERR_ARG otherwise);
 * results are order-dependent in the last bits (atomic accumulation).  The flop model
 * (h2_stats) keeps the paper's convention over the full operator; the byte model counts what is
 * stored. */
enum { H2_SYMMETRIC = 1 };

typedef struct h2_ctx *h2_handle;

/* Build a handle: validates the description, builds the static execution plan (replaces the
 * paper's per-call marshaling), re-lays out V and F for the kernels' operand
 * order, allocates the x^/y^ workspaces for up to nv_max vectors, and for nranks > 1 creates
 * an NCCL communicator from `nccl_unique_id` (128 bytes, identical on all ranks; NULL when
 * nranks == 1) and exchanges the compressed off-diagonal node lists.
 * Collective over ranks.  On failure no handle is created (*out = NULL).
 * Structural checks (H2_ERR_STRUCT): monotone row pointers, column ids in range, strictly
 * ascending columns per row (no duplicate (t,s,l)), leaf sizes in [1, m], P a power of two
 * with P <= 2^q.  Shape checks (H2_ERR_SHAPE): 1 <= k^l <= 64, 1 <= m <= 64, nv_max in [1, 64]. */
int h2_create(const h2_desc *d, int nv_max, const void *nccl_unique_id, h2_handle *out);

/* Y := alpha A X + beta Y on the handle's stream (asynchronous).  X, Y device pointers,
 * ld = n_local.  alpha, beta are converted to dtype.  beta == 0: Y is write-only (NaNs in Y do
 * not propagate).  alpha == 0: A X is not formed.  1 <= nv <= nv_max.  Collective over ranks
 * (same nv, alpha, beta on every rank). */
int h2_matvec(h2_handle h, double alpha, const void *X, double beta, void *Y, int nv);

/* Same with explicit leading dimensions (>= n_local). */
int h2_matvec_ld(h2_handle h, double alpha, const void *X, int64_t ldx, double beta, void *Y,
                 int64_t ldy, int nv);

/* End-to-end variant: X and Y are HOST arrays (ld = n_local; pinned memory gives async copies).
 * Copies X (and Y if beta != 0) host->device, runs h2_matvec on internal device buffers, copies
 * Y device->host, and synchronizes the handle's stream before returning. */
int h2_matvec_host(h2_handle h, double alpha, const void *X, double beta, void *Y, int nv);

/* Stream for subsequent work (a cudaStream_t cast to void*); default: the legacy stream. */
int h2_set_stream(h2_handle h, void *stream);

/* Static facts of the handle for nv vectors: flops (paper convention 2 nv x stored operator
 * scalars), algorithmic bytes per matvec (operator once + X, Y, x^, y^ traffic),
 * per-rank halo bytes exchanged, and the number of kernel launches one matvec makes.
 * Any pointer may be NULL. */
int h2_stats(h2_handle h, int nv, double *flops, double *bytes, double *xchg_bytes,
             int *launches);

/* Phase profiling.  Phases: 0 upsweep leaves, 1 upsweep transfers,
 * 2 exchange pack + replicated top tree, 3 coupling (diagonal, levels above the leaves),
 * 4 coupling (off-diagonal, after the exchange wait), 5 downsweep transfers, 6 leaves (last
 * transfer + U expansion), 7 dense near field + epilogue (own concurrent stream), 8 coupling at
 * the leaf level (diagonal; own concurrent stream).  h2_set_profiling(h, 1) records
 * CUDA events between phases of every following h2_matvec (eager launches, no graph, the side
 * streams serialized onto the handle's stream so each phase is timed alone);
 * h2_phase_times synchronizes, returns the mean milliseconds per phase per call since the last
 * read (ms[0..8]; ms[9] = whole call on the main stream) and the call count, and resets.
 * h2_phase_stats returns the algorithmic bytes and flops of each phase for nv vectors
 * (beta == 0), indexed the same way (index 9 = total). */
#define H2_NPHASE 9
int h2_set_profiling(h2_handle h, int on);
int h2_phase_times(h2_handle h, double ms[H2_NPHASE + 1], int64_t *ncalls);
int h2_phase_stats(h2_handle h, int nv, double bytes[H2_NPHASE + 1], double flops[H2_NPHASE + 1]);

/* Rows of X / Y on this rank (the n_local of the description). */
int h2_n_local(h2_handle h, int64_t *n_local);

/* Plan facts for tests: counts[0..7] = {diag coupling blocks, offdiag coupling blocks,
 * root (top-tree) coupling blocks, diag dense blocks, offdiag dense blocks, peers,
 * remote x^ nodes received, remote leaves received}. */
int h2_plan_counts(h2_handle h, int64_t counts[8]);

/* Host-only plan census (no device, no communication): the compressed off-diagonal node lists of
 * this rank's view in the paper's format (Fig. compressed_vnodes): for coupling
 * level `level` (0..q) -- or the dense halo leaves when level == -1 -- pid[0..npid) are the peer
 * ranks this rank receives from (ascending), and nodes[nodes_ptr[i] .. nodes_ptr[i+1]) the
 * ascending GLOBAL node (leaf) indices it needs from pid[i].  Call once with pid / nodes_ptr /
 * nodes NULL to get the sizes (*npid, *nnodes), then with buffers of [npid], [npid+1], [nnodes].
 * Validates the description like h2_create (nv_max treated as 1). */
int h2_plan_census(const h2_desc *d, int level, int64_t *pid, int64_t *nodes_ptr, int64_t *nodes,
                   int64_t *npid, int64_t *nnodes);

/* ---- Loopback groups (TEST / DIAGNOSTIC entry points) --------------------------------------
 * Emulate P ranks inside ONE process on the current GPU, so the multi-rank code path (x^ and
 * x-halo packs, off-diagonal coupling from the receive chunks, halo-fed dense blocks, replicated
 * top tree, alg:optimized_dist_mult) can be checked with a single device.
 * The per-call NCCL groups are replaced by device-to-device copies of the same bytes between the
 * members' send and receive buffers, on one stream, between the members' upsweep halves and their
 * coupling / downsweep halves.  Production runs use h2_create with NCCL.
 * h2_group_create: descs[o] is rank o's view (descs[o]->rank == o, ->nranks == P); out[0..P)
 *   receives the member handles (all NULL on failure).  Same validation and errors as h2_create.
 * h2_group_matvec: Y[o] := alpha A X[o] + beta Y[o] for every member o (device pointers,
 *   ld = n_local of o), asynchronous on member 0's stream.  hs must be all members in rank order.
 *   h2_matvec on a member returns H2_ERR_STATE.  Members are released with h2_destroy. */
int h2_group_create(const h2_desc *const *descs, int P, int nv_max, h2_handle *out);
int h2_group_matvec(const h2_handle *hs, int P, double alpha, const void *const *X, double beta,
                    void *const *Y, int nv);

/* ---- The .h2m flat file ("header {N, m, depth, level ranks}, then level-ordered
 * arrays"; written by the input generator h2gen/h2m.py) -------------------------------------
 * Little-endian.  A 512-byte header: magic "H2MFLAT1"; u32 version (1), dtype (0 f64, 1 f32), dim,
 * m, q, flags (bit 0: V aliases U, bit 1: F aliases E), kernel id, reserved; u64 N, n_D, seed;
 * f64 eta, kernel parameters[4]; i32 k^l[32]; i64 n_S^l[32].  Then sections, each starting at a
 * multiple of 64 bytes: points f64[N][dim] (tree order), perm i64[N], leaf_ptr i64[2^q+1],
 * U_leaf T[2^q][m x k^q], V_leaf (unless aliased), E^l T[2^l][k^l x k^(l-1)] for l = 1..q, F^l
 * (unless aliased), then per level l = 0..q: S_rowptr i64[2^l+1], S_col i32[n_S^l],
 * S T[n_S^l][k^l x k^l]; then D_rowptr i64[2^q+1], D_col i32[n_D], D T[n_D][m x m].  All small
 * matrices column-major; global node / leaf indices.
 * h2_file_info: info[0..7] = {N, dim, m, q, dtype, total coupling blocks, n_D, k^q}; checks the
 *   magic, version and that the file is as long as its header says (H2_ERR_STRUCT otherwise;
 *   H2_ERR_ARG if it cannot be opened).  No device work.
 * h2_create_from_file: rank `rank` of `nranks` reads only its own view (its branch at levels
 *   >= C = log2 P, the top levels replicated) and calls h2_create with those
 *   host arrays (same arguments, errors and collective semantics as h2_create). */
int h2_file_info(const char *path, int64_t info[8]);
int h2_create_from_file(const char *path, int rank, int nranks, int nv_max, const void *nccl_unique_id,
                        h2_handle *out);
/* Loopback-group form (tests): all P ranks' views read from the file, then h2_group_create. */
int h2_group_create_from_file(const char *path, int P, int nv_max, h2_handle *out);

/* ---- Fractional-diffusion solve ------------------
 * The system h^2 (D + K + C) u = b of the paper's application, with K the H² operator of handle K
 * (n = its n_local rows, tree order, FP64, one rank), D diagonal, C sparse.  All device memory,
 * FP64, synchronous (legacy stream).
 * h2_fd_diag: diag[i] = (K^ 1)[idx[i]] + cdiag[i] (cdiag may be NULL) for i < n: D from one H²
 *   matvec of the extended-grid operator K^ (handle khat, "recast as the product
 *   K^ 1") with the ones vector, gathered at the interior points' rows idx (tree order of K^).
 * h2_pcg: preconditioned conjugate gradients on A u = scale (diag u + K u + C' u)
 *   = b, C' = C without its diagonal (CSR C_rowptr [n+1], C_col [nnz] (tree-order columns),
 *   C_val; diagonal entries are skipped -- fold them into diag), Jacobi preconditioner
 *   scale * diag.  u: initial guess in, solution out.  Stops when ||b - A u|| <= rtol ||b|| or
 *   after maxit iterations; *iters = iterations done; res_hist[0..*iters] (host, may be NULL) =
 *   the relative residual norms.  H2_ERR_ARG for NULL / bad sizes. */
int h2_fd_diag(h2_handle khat, const int64_t *idx, const double *cdiag, int64_t n, double *diag);
int h2_pcg(h2_handle K, double scale, const double *diag, const int64_t *C_rowptr, const int32_t *C_col,
           const double *C_val, const double *b, double *u, double rtol, int maxit, int *iters,
           double *res_hist);

/* ---- Basis orthogonalization (first step) -----------
 * h2_orthogonalize: in place on the handle's device operator, the QR upsweep of both basis trees
 *   -- leaves U_t = Q_t R_t (thin Householder QR, diag R >= 0), then per level
 *   [R_c1 E_c1; R_c2 E_c2] = Q_p R_p with the new transfers E'_c = the halves of Q_p (the same for
 *   V with F) -- and every coupling block re-expressed, S'_ts = R^U_t S_ts (R^V_s)^T.  The operator
 *   is unchanged (up to rounding) and every implied level basis has orthonormal columns: the
 *   pre-processing step of the paper's algebraic recompression.  FP64, one GPU, full storage,
 *   m <= 128, k^l <= 64, k^q <= m, k^{l-1} <= 2 k^l; synchronous.  Captured matvec graphs stay
 *   valid (same arrays, new values).  H2_ERR_ARG when unsupported.
 * h2_export: copy one operator array of the handle to host memory (count elements, checked):
 *   H2_EXPORT_S  coupling blocks of `level` (k^l x k^l each, column-major, h2_desc CSR order;
 *                one GPU, full storage), H2_EXPORT_U leaf bases (m x k^q per leaf),
 *   H2_EXPORT_VT leaf bases stored transposed (k^q x m per leaf), H2_EXPORT_E transfers of `level`
 *   (k^l x k^{l-1} per node), H2_EXPORT_FT transfers F stored transposed (k^{l-1} x k^l);
 *   H2_EXPORT_XHAT / H2_EXPORT_YHAT the x^ / y^ coefficients of `level` left by the last matvec
 *   (count = nv * held nodes * k^l: per vector, node-major then coefficient; y^ of the levels
 *   above the leaves after the downsweep, the leaf level's coupling sums -- the leaf transfer is
 *   applied inside the leaf kernel for FP64). */
enum { H2_EXPORT_S = 0, H2_EXPORT_U = 1, H2_EXPORT_VT = 2, H2_EXPORT_E = 3, H2_EXPORT_FT = 4,
       H2_EXPORT_XHAT = 5, H2_EXPORT_YHAT = 6 };
int h2_orthogonalize(h2_handle h);
int h2_export(h2_handle h, int what, int level, void *host, int64_t count);
/* h2_reweigh: the reweighing downsweep of the recompression, root to leaves:
 *   for every node i of level l the R factor of the stacked [R^{l-1}_{i+} E^{lT}_i ; S^{lT}_{ij} ...]
 *   (Eq. Btq; the parent part absent at the root), so that R^{lT}_i R^l_i is the Gram matrix of the
 *   block row's low-rank part and U^l_i R^{lT}_i is the reweighed basis.  Requires an orthogonal V
 *   basis (call h2_orthogonalize first).  R_out: device memory, count = sum_l 2^l (k^l)^2 doubles,
 *   levels concatenated from the root, each node's R column-major (upper triangular, diag >= 0).
 *   FP64, one GPU, full storage, k^l <= 64; synchronous; the operator is not modified. */
int h2_reweigh(h2_handle h, void *R_out, int64_t count);

/* Release device memory, the NCCL communicator and streams.  NULL is a no-op. */
int h2_destroy(h2_handle h);

/* Fill out[0..127] with a fresh NCCL unique id (call on one rank, broadcast to the others,
 * pass to h2_create).  H2_ERR_NCCL if the NCCL library cannot be loaded. */
int h2_nccl_unique_id(void *out128);

/* Message for the last failure on this thread (never NULL). */
const char *h2_last_error(void);

/* Library version string (never NULL). */
const char *h2_version(void);

#ifdef __cplusplus
}
#endif
#endif
