// h2_api.cpp -- C ABI (include/h2.h): validation, the static execution plan, device memory,
// the NCCL exchange, and the per-call launch sequence of the distributed H^2 matvec.
//
// The plan replaces the paper's per-call marshaling kernels with
// task/block tables built once here: every output node of every phase becomes one warp task
// whose blocks point straight at their operands (implicit heap addressing, no pointer arrays
// rebuilt per call).  Distribution follows PAPER.md:195-206 (block rows, C-level C = log2 P,
// replicated top tree = reading R16) and PAPER.md:445-502 (diagonal / off-diagonal split,
// compressed node lists pid / nodes_ptr / nodes, one exchange per matvec overlapped with the
// diagonal multiply).
#include "../../include/h2.h"
#include "h2_internal.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <new>
#include <numeric>
#include <string>
#include <vector>

using namespace h2;

namespace {

thread_local std::string g_err = "no error";

int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

// ------------------------------------------------------------------ NCCL (loaded lazily)
struct NcclApi {
    bool loaded = false;
    void *lib = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
};
NcclApi g_nccl;

#ifndef H2_NCCL_DEFAULT
#define H2_NCCL_DEFAULT "libnccl.so.2"
#endif

bool load_nccl()
{
    if (g_nccl.loaded) return true;
    const char *cands[3] = {getenv("H2_NCCL_LIB"), "libnccl.so.2", H2_NCCL_DEFAULT};
    for (const char *c : cands) {
        if (!c) continue;
        g_nccl.lib = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (g_nccl.lib) break;
    }
    if (!g_nccl.lib) return false;
#define H2_SYM(field, name) \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(g_nccl.lib, name)); \
    if (!g_nccl.field) return false;
    H2_SYM(CommInitRank, "ncclCommInitRank")
    H2_SYM(CommDestroy, "ncclCommDestroy")
    H2_SYM(Send, "ncclSend")
    H2_SYM(Recv, "ncclRecv")
    H2_SYM(AllGather, "ncclAllGather")
    H2_SYM(AllReduce, "ncclAllReduce")
    H2_SYM(GroupStart, "ncclGroupStart")
    H2_SYM(GroupEnd, "ncclGroupEnd")
    H2_SYM(GetErrorString, "ncclGetErrorString")
    H2_SYM(GetUniqueId, "ncclGetUniqueId")
#undef H2_SYM
    g_nccl.loaded = true;
    return true;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// H2_DEBUG=1: trace the setup / call steps on stderr (debugging multi-rank hangs)
bool dbg_on()
{
    static int on = -1;
    if (on < 0) { const char *e = getenv("H2_DEBUG"); on = (e && e[0] == '1') ? 1 : 0; }
    return on == 1;
}
#define H2_DBG(...) do { if (dbg_on()) { fprintf(stderr, "[h2] " __VA_ARGS__); fputc('\n', stderr); fflush(stderr); } } while (0)

// ------------------------------------------------------------------ host-side plan
struct Layout {
    int q = 0, m = 0, p = 0, P = 1, C = 0;
    std::vector<int> k;
    int64_t held(int l) const { return l < C ? (int64_t)1 << l : (int64_t)1 << (l - C); }
    int64_t g0(int l) const { return l < C ? 0 : (int64_t)p << (l - C); }
    int owner(int l, int64_t g) const { return l < C ? -1 : (int)(g >> (l - C)); }
};

// Remote (level, global node) -> key for ordered maps
inline int64_t node_key(int l, int64_t g) { return ((int64_t)l << 40) | g; }
inline int key_level(int64_t key) { return (int)(key >> 40); }
inline int64_t key_node(int64_t key) { return key & (((int64_t)1 << 40) - 1); }

// Validation of the description (H2_ERR_* codes, message in g_err).
int validate(const h2_desc *d, int nv_max, Layout &L)
{
    if (!d) return fail(H2_ERR_ARG, "desc is NULL");
    if (d->dtype != H2_F64 && d->dtype != H2_F32) return fail(H2_ERR_ARG, "unknown dtype");
    if (d->mem != H2_MEM_HOST && d->mem != H2_MEM_DEVICE) return fail(H2_ERR_ARG, "unknown mem kind");
    if (nv_max < 1 || nv_max > 64) return fail(H2_ERR_SHAPE, "nv_max must be in [1, 64]");
    if (d->depth < 0 || d->depth > 30) return fail(H2_ERR_STRUCT, "depth out of range [0, 30]");
    if (d->leaf_size < 1 || d->leaf_size > KMAX) return fail(H2_ERR_SHAPE, "leaf_size must be in [1, 64]");
    if (d->nranks < 1 || (d->nranks & (d->nranks - 1)))
        return fail(H2_ERR_STRUCT, "nranks must be a power of two");
    if (d->rank < 0 || d->rank >= d->nranks) return fail(H2_ERR_ARG, "rank out of range");
    int C = 0;
    while ((1 << C) < d->nranks) ++C;
    if (C > d->depth) return fail(H2_ERR_STRUCT, "P too large for depth (P > 2^q)");
    if (!d->level_rank || !d->leaf_ptr || !d->U_leaf || !d->V_leaf || !d->S_rowptr || !d->S_col ||
        !d->S || !d->D_rowptr || (d->depth > 0 && (!d->E || !d->F)))
        return fail(H2_ERR_ARG, "NULL array in desc");
    L.q = d->depth; L.m = d->leaf_size; L.p = d->rank; L.P = d->nranks; L.C = C;
    L.k.resize(L.q + 1);
    for (int l = 0; l <= L.q; ++l) {
        int k = d->level_rank[l];
        if (k < 1 || k > KMAX) return fail(H2_ERR_SHAPE, "level rank k^l must be in [1, 64]");
        L.k[l] = k;
    }
    const int64_t nleaf = L.held(L.q);
    const int64_t *lp = d->leaf_ptr;
    if (lp[0] != 0) return fail(H2_ERR_STRUCT, "leaf_ptr[0] must be 0");
    for (int64_t i = 0; i < nleaf; ++i) {
        int64_t sz = lp[i + 1] - lp[i];
        if (sz < 1 || sz > L.m) return fail(H2_ERR_STRUCT, "leaf sizes must be in [1, m]");
    }
    if (lp[nleaf] != d->n_local) return fail(H2_ERR_STRUCT, "leaf_ptr[end] != n_local");
    for (int l = 0; l <= L.q; ++l) {
        const int64_t *rp = d->S_rowptr[l];
        const int32_t *col = d->S_col[l];
        const int64_t rows = L.held(l);
        if (!rp) return fail(H2_ERR_ARG, "S_rowptr[l] is NULL");
        if (rp[0] != 0) return fail(H2_ERR_STRUCT, "S_rowptr[l][0] must be 0");
        for (int64_t i = 0; i < rows; ++i)
            if (rp[i + 1] < rp[i]) return fail(H2_ERR_STRUCT, "S_rowptr not monotone");
        if (rp[rows] > 0 && !col) return fail(H2_ERR_ARG, "S_col[l] is NULL but level has blocks");
        for (int64_t i = 0; i < rows; ++i) {
            if (rp[i + 1] < rp[i]) return fail(H2_ERR_STRUCT, "S_rowptr not monotone");
            for (int64_t b = rp[i]; b < rp[i + 1]; ++b) {
                if (col[b] < 0 || col[b] >= ((int64_t)1 << l))
                    return fail(H2_ERR_STRUCT, "S_col out of range");
                if (b > rp[i] && col[b] <= col[b - 1])
                    return fail(H2_ERR_STRUCT, "S_col not strictly ascending within a row (duplicate block?)");
                if (l < C) {
                    // top-tree rows are replicated; nothing else to check
                }
            }
        }
        if (rp[rows] > 0 && !d->S[l]) return fail(H2_ERR_ARG, "S[l] is NULL but level has blocks");
        if (l >= 1 && (!d->E[l] || !d->F[l])) return fail(H2_ERR_ARG, "E[l] / F[l] is NULL");
    }
    {
        const int64_t *rp = d->D_rowptr;
        if (rp[0] != 0) return fail(H2_ERR_STRUCT, "D_rowptr[0] must be 0");
        for (int64_t i = 0; i < nleaf; ++i)
            if (rp[i + 1] < rp[i]) return fail(H2_ERR_STRUCT, "D_rowptr not monotone");
        if (rp[nleaf] > 0 && !d->D_col) return fail(H2_ERR_ARG, "D_col is NULL but there are dense blocks");
        for (int64_t i = 0; i < nleaf; ++i) {
            if (rp[i + 1] < rp[i]) return fail(H2_ERR_STRUCT, "D_rowptr not monotone");
            for (int64_t b = rp[i]; b < rp[i + 1]; ++b) {
                if (d->D_col[b] < 0 || d->D_col[b] >= ((int64_t)1 << L.q))
                    return fail(H2_ERR_STRUCT, "D_col out of range");
                if (b > rp[i] && d->D_col[b] <= d->D_col[b - 1])
                    return fail(H2_ERR_STRUCT, "D_col not strictly ascending within a row");
            }
        }
        if (rp[nleaf] > 0 && !d->D) return fail(H2_ERR_ARG, "D is NULL but there are dense blocks");
    }
    return H2_OK;
}

// Which remote nodes this rank's block rows need: for every peer, the sorted
// unique off-diagonal column nodes (level, node) of the coupling blocks and the remote leaves of
// the dense blocks; plus the diagonal / off-diagonal / root block counts.
struct RemoteNeeds {
    std::map<int, std::vector<int64_t>> need_x;   // peer -> sorted unique node keys
    std::map<int, std::vector<int64_t>> need_h;   // peer -> sorted unique global leaves
    int64_t n_diag = 0, n_off = 0, n_root = 0, nd_diag = 0, nd_off = 0;
};

void remote_needs(const h2_desc *d, const Layout &L, RemoteNeeds &rn)
{
    const int q = L.q, p = L.p;
    for (int l = 0; l <= q; ++l) {
        const int64_t *rp = d->S_rowptr[l];
        for (int64_t i = 0; i < L.held(l); ++i)
            for (int64_t b = rp[i]; b < rp[i + 1]; ++b) {
                int64_t s = d->S_col[l][b];
                int o = L.owner(l, s);
                if (o < 0) ++rn.n_root;
                else if (o == p) ++rn.n_diag;
                else { ++rn.n_off; rn.need_x[o].push_back(node_key(l, s)); }
            }
    }
    const int64_t nleaf = L.held(q);
    for (int64_t t = 0; t < nleaf; ++t)
        for (int64_t b = d->D_rowptr[t]; b < d->D_rowptr[t + 1]; ++b) {
            int64_t s = d->D_col[b];
            int o = L.owner(q, s);
            if (o < 0 || o == p) ++rn.nd_diag;
            else { ++rn.nd_off; rn.need_h[o].push_back(s); }
        }
    for (auto *m : {&rn.need_x, &rn.need_h})
        for (auto &kv : *m) {
            auto &v = kv.second;
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
        }
}

struct Phase {
    int64_t t0 = 0;
    int n = 0;
    int r = 1;       // output rows of every task in the phase (engine selection)
};

}  // namespace

// ------------------------------------------------------------------ the handle
// P handles of one process on one GPU that exchange in-process (h2_group_create; tests only):
// the per-call NCCL groups become device-to-device copies between the members' buffers.
struct h2_group {
    std::vector<h2_ctx *> members;
    std::vector<const h2_desc *> descs;
    std::vector<Layout> layouts;
    std::vector<RemoteNeeds> needs;
};

struct h2_ctx {
    Layout L;
    int dtype = H2_F64;
    size_t esz = 8;
    int nv_max = 1;
    int64_t n_local = 0, nleaf = 0;
    bool sticky = false;
    h2_group *group = nullptr;       // loopback group (tests) or nullptr (NCCL / single rank)
    bool sym = false;                // symmetric storage (h2_desc.flags & H2_SYMMETRIC; NEXT-2)
    double ops_stored = 0;           // operator scalars actually stored (bytes model)
    bool has_top = false;            // P > 1 and the top tree (levels < C) holds couplings
    cudaStream_t stream = nullptr;   // caller's stream (default legacy)
    cudaStream_t s_comm = nullptr;
    cudaStream_t s_leafc = nullptr;  // leaf-level coupling, concurrent with the upsweep transfers
    cudaEvent_t ev_packed = nullptr, ev_recv = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_halo = nullptr;
    cudaEvent_t ev_upleaf = nullptr, ev_leafc = nullptr;
    std::vector<void *> owned;       // device allocations to free
    // operator (device)
    const void *U = nullptr, *Vt = nullptr, *D = nullptr;
    std::vector<const void *> E, Ft, S;
    const void *FtC_all = nullptr;   // P > 1 && has_top: all ranks' F_C^T (allgathered)
    // workspaces (device): plane layout, element (j, n) of a region at off + j + n * plane
    void *xh = nullptr, *yh = nullptr;
    int64_t xh_plane = 0, yh_plane = 0;
    std::vector<int64_t> xh_base, yh_base;
    int64_t xgather = -1;            // level-C all-rank roots region (has_top)
    void *xsend = nullptr, *xrecv = nullptr, *hsend = nullptr, *hrecv = nullptr;
    // plan (device)
    Task *d_tasks = nullptr;
    Blk *d_blks = nullptr;
    PackSeg *d_segs = nullptr;
    Phase up_leaf, coup_off[3], coup_off_leaf[3], leaf, dense;   // off-diagonal: upper levels / leaf level
    Phase leafE;                     // leaf-level transfers y^_t += E_t y^_p as rows (tcgen05 leaf path)
    std::vector<Phase> up_lv, top_up_lv, coup_diag, coup_leaf, down_lv;
    struct Stage { TreeStage st; int nctas; int r; };
    std::vector<Stage> up_stages, top_stages, down_stages;
    // heap-addressed sweeps (k_sweep): bottom levels one launch each, small top levels fused
    bool use_sweep = false;
    std::vector<SweepParams> up_sweeps, dn_sweeps;
    std::vector<int> up_sweep_ctas, dn_sweep_ctas, up_sweep_thr, dn_sweep_thr;
    int sweep_r_up = 1, sweep_r_dn = 1;
    std::vector<int> up_lv_level, top_up_level, down_level;
    int64_t nseg_x = 0, nseg_h = 0, seg_x0 = 0, seg_h0 = 0;
    struct Peer {
        int rank;
        int64_t xs_off = 0, xs_cnt = 0, xr_off = 0, xr_cnt = 0;   // elements per vector
        int64_t hs_off = 0, hs_cnt = 0, hr_off = 0, hr_cnt = 0;   // rows per vector
    };
    std::vector<Peer> peers;
    // device-initiated peer exchange (NEXT-1; H2_EXCHANGE=nccl keeps the NCCL groups): peers read
    // my x^ plane and my packed x rows directly through CUDA-IPC mappings, synchronised by epoch
    // flags in the handles' signal blocks (h2_internal.h SIG_*)
    bool p2p = false;
    bool p2p_direct = false;           // H2_EXCHANGE=p2p-direct: the off-diagonal kernels read the peers'
                                       // x^ over NVLink themselves (measured slower: latency-bound)
    int32_t *sig = nullptr;
    struct Pull { int owner, group; int64_t seg0, nseg; };
    std::vector<Pull> pulls;           // per (level group, owner): segments copying the owner's x^ nodes I
                                       // need from its mapped plane into my receive chunk
    struct PeerMap {
        const void *xh = nullptr, *hsend = nullptr;
        int32_t *sig = nullptr;
        int64_t hs_off = -1;           // offset of my chunk in the peer's hsend
    };
    std::vector<PeerMap> pmap;         // by rank
    std::vector<void *> ipc_open;
    struct P2PPhase { int owner, group; Phase ph; };
    std::vector<P2PPhase> p2p_phases;  // off-diagonal tasks reading one peer's x^ directly
    int32_t *d_begin_waits = nullptr, *d_wait_xl = nullptr, *d_wait_xu = nullptr, *d_wait_h = nullptr;
    int32_t **d_tgt_xl = nullptr, **d_tgt_xu = nullptr, **d_tgt_h = nullptr, **d_tgt_cx = nullptr, **d_tgt_ch = nullptr;
    int n_begin_waits = 0, n_wait_xl = 0, n_wait_xu = 0, n_wait_h = 0, n_tgt_xl = 0, n_tgt_xu = 0, n_tgt_h = 0,
        n_tgt_cx = 0, n_tgt_ch = 0;
    int64_t xsend_tot = 0, xrecv_tot = 0, hsend_tot = 0, hrecv_tot = 0;
    ncclComm_t comm = nullptr;
    // e2e staging
    void *dX = nullptr, *dY = nullptr;
    // h2_matvec_host pipeline: copy streams (host-to-device, device-to-host) and per-chunk events
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_x[2] = {}, ev_y[2] = {};
    // per-call arguments (device CallArgs<T>) and the captured graphs, one per nv
    void *dargs = nullptr;
    cudaStream_t cap_stream = nullptr;
    cudaStream_t last_stream = nullptr;
    bool last_stream_set = false;
    cudaGraphExec_t graph[65] = {};
    bool warm[65] = {};
    // profiling
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;   // 8 events per recorded call
    int64_t ev_used = 0;
    double ph_ops[H2_NPHASE] = {};   // operator scalars per phase
    double ph_vec[H2_NPHASE] = {};   // vector elements per nv per phase
    // stats
    double ops_local = 0;            // stored operator scalars held by this rank
    int64_t counts[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int launches_per_call = 0;
    // CTA-tile FP64 engine (h2_cta.cuh) for nv >= cta_min_nv (H2_ENGINE=warp: never, =cta: every nv);
    // measured: faster than the warp engine at nv = 64 (cfg3), slower at nv <= 16 (cfg2, cfg5)
    int cta_min_nv = 17;
    int nsm = 148;
    bool use_cta(int nv) const { return dtype == H2_F64 && nv >= cta_min_nv; }
    // tcgen05 FP32 row engine (h2_umma.cuh) for the coupling rows at nv >= umma_min_nv
    // (H2_ENGINE=warp: never; below it the SIMT engines)
    int umma_min_nv = 5;
    bool use_umma(int nv) const { return dtype == H2_F32 && nv >= umma_min_nv; }
    int launches_cta = 0;
    // tcgen05 FP32 leaf path: device slot of the per-call X tensor map (FP32 handles)
    void *d_xmap = nullptr;
    int launches_umma = 0;
    // basis orthogonalization (h2_orthogonalize; one GPU, full storage): (t, s) of every coupling
    // block per level, in the device S[l] order
    std::vector<std::vector<int2>> orth_pairs;
    bool use_umma_leaf(int nv) const { return use_umma(nv) && d_xmap && leaf.r <= 64; }
};

namespace {

int cuda_fail(h2_ctx *h, cudaError_t e, const char *what)
{
    if (h) h->sticky = true;
    return fail(e == cudaErrorMemoryAllocation ? H2_ERR_OOM : H2_ERR_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define H2_CUDA(h, call)                                       \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); \
    } while (0)

#define H2_NCCL(h, call)                                                             \
    do {                                                                             \
        ncclResult_t r_ = (call);                                                    \
        if (r_ != ncclSuccess) {                                                     \
            if (h) h->sticky = true;                                                 \
            return fail(H2_ERR_NCCL, std::string(#call) + ": " + g_nccl.GetErrorString(r_)); \
        }                                                                            \
    } while (0)

void *dalloc(h2_ctx *h, size_t bytes, cudaError_t &err)
{
    void *p = nullptr;
    if (bytes == 0) bytes = 16;
    err = cudaMalloc(&p, bytes);
    if (err != cudaSuccess) return nullptr;
    h->owned.push_back(p);
    return p;
}

ncclDataType_t nccl_type(int dtype) { return dtype == H2_F64 ? ncclDouble : ncclFloat; }

int release(h2_ctx *h)
{
    if (!h) return H2_OK;
    if (h->group) {                  // detach from a loopback group; the last member frees it
        h2_group *g = h->group;
        bool any = false;
        for (auto &m : g->members) {
            if (m == h) m = nullptr;
            any = any || m != nullptr;
        }
        if (!any) delete g;
        h->group = nullptr;
    }
    // captured graphs hold references to the NCCL communicator's resources: destroy them first
    for (auto &g : h->graph)
        if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    cudaDeviceSynchronize();
    if (!h->ipc_open.empty() || h->sig) {
        // peers may still read my buffers: a barrier over the communicator before anything is freed
        if (h->comm && g_nccl.loaded && h->s_comm && h->sig) {
            g_nccl.AllReduce(h->sig, h->sig, 1, ncclInt32, ncclMax, h->comm, h->s_comm);
            cudaStreamSynchronize(h->s_comm);
        }
        for (void *p : h->ipc_open) cudaIpcCloseMemHandle(p);
        h->ipc_open.clear();
    }
    if (h->comm && g_nccl.loaded) g_nccl.CommDestroy(h->comm);
    for (void *p : h->owned) cudaFree(p);
    for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    if (h->s_comm) cudaStreamDestroy(h->s_comm);
    if (h->s_leafc) cudaStreamDestroy(h->s_leafc);
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    for (cudaEvent_t e : {h->ev_packed, h->ev_recv, h->ev_fork, h->ev_halo, h->ev_upleaf, h->ev_leafc, h->ev_x[0],
                          h->ev_x[1], h->ev_y[0], h->ev_y[1]})
        if (e) cudaEventDestroy(e);
    delete h;
    return H2_OK;
}

// Copy (HOST) or adopt (DEVICE) a floating array of `n` elements.
int put_array(h2_ctx *h, int mem, const void *src, int64_t n, const void **out)
{
    if (n == 0) { *out = nullptr; return H2_OK; }
    if (mem == H2_MEM_DEVICE) { *out = src; return H2_OK; }
    cudaError_t err;
    void *p = dalloc(h, (size_t)n * h->esz, err);
    if (!p) return cuda_fail(h, err, "cudaMalloc(operator)");
    H2_CUDA(h, cudaMemcpy(p, src, (size_t)n * h->esz, cudaMemcpyHostToDevice));
    *out = p;
    return H2_OK;
}

// Device copy of the blocks kept[0..] (original block indices, ascending) of an array of blocks of
// `per` elements, compacted in that order (symmetric storage); runs of consecutive blocks are copied
// at once.
int put_gathered(h2_ctx *h, int mem, const void *src, const std::vector<int64_t> &kept, int64_t per, const void **out)
{
    if (kept.empty()) { *out = nullptr; return H2_OK; }
    cudaError_t err;
    void *dst = dalloc(h, (size_t)kept.size() * per * h->esz, err);
    if (!dst) return cuda_fail(h, err, "cudaMalloc(symmetric blocks)");
    const cudaMemcpyKind kind = mem == H2_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const size_t bb = (size_t)per * h->esz;
    size_t i = 0;
    while (i < kept.size()) {
        size_t j = i + 1;
        while (j < kept.size() && kept[j] == kept[j - 1] + 1) ++j;
        H2_CUDA(h, cudaMemcpy((char *)dst + i * bb, (const char *)src + (size_t)kept[i] * bb, (j - i) * bb, kind));
        i = j;
    }
    *out = dst;
    return H2_OK;
}

// Transposed device copy of a batch of r x c column-major matrices (-> c x r column-major).
int put_transposed(h2_ctx *h, int mem, const void *src, int64_t batch, int r, int c, const void **out)
{
    int64_t n = batch * r * c;
    if (n == 0) { *out = nullptr; return H2_OK; }
    cudaError_t err;
    void *dst = dalloc(h, (size_t)n * h->esz, err);
    if (!dst) return cuda_fail(h, err, "cudaMalloc(transposed)");
    const void *dsrc = src;
    void *tmp = nullptr;
    if (mem == H2_MEM_HOST) {
        H2_CUDA(h, cudaMalloc(&tmp, (size_t)n * h->esz));
        cudaError_t e = cudaMemcpy(tmp, src, (size_t)n * h->esz, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { cudaFree(tmp); return cuda_fail(h, e, "cudaMemcpy(transposed)"); }
        dsrc = tmp;
    }
    cudaError_t e = h->dtype == H2_F64
                        ? launch_transpose<double>((const double *)dsrc, (double *)dst, batch, r, c, 0)
                        : launch_transpose<float>((const float *)dsrc, (float *)dst, batch, r, c, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (tmp) cudaFree(tmp);
    if (e != cudaSuccess) return cuda_fail(h, e, "transpose");
    *out = dst;
    return H2_OK;
}

template <typename T>
int run_matvec(h2_ctx *h, T alpha, const T *X, int64_t ldx, T beta, T *Y, int64_t ldy, int nv);

// ======================================================================== setup collectives
// The setup-time exchanges of h2_create (the compressed node lists are
// "communicated among GPUs during the setup phase"): all ranks' leaf sizes, the request lists
// (what each peer needs from me) and, with top-tree couplings, every rank's branch-root transfer.
// NCCL over the handle's communicator in production; an in-process loopback for h2_group_create
// (P ranks emulated on one GPU, tests only).
struct SetupComm {
    virtual ~SetupComm() {}
    // all ranks' leaf sizes, rank-major: all[o * nleaf + i]
    virtual int leaf_sizes(h2_ctx *h, const std::vector<int64_t> &mine, std::vector<int64_t> &all) = 0;
    // give_x[o] / give_h[o]: the x^ node keys / leaves peer o needs from this rank
    virtual int requests(h2_ctx *h, const RemoteNeeds &rn, std::map<int, std::vector<int64_t>> &give_x,
                         std::map<int, std::vector<int64_t>> &give_h) = 0;
    // dst[o * per ..]: F_C^T of rank o's branch root (k^{C-1} x k^C, column-major)
    virtual int gather_FtC(h2_ctx *h, void *dst, int64_t per) = 0;
};

// Peer o asked for `keys` (nx x^ node keys, then leaves): check that this rank owns them.
int check_requests(h2_ctx *h, int o, const std::vector<int64_t> &keys, int64_t nx,
                   std::map<int, std::vector<int64_t>> &give_x, std::map<int, std::vector<int64_t>> &give_h)
{
    const Layout &L = h->L;
    for (int64_t i = 0; i < (int64_t)keys.size(); ++i) {
        if (i < nx) {
            int l = key_level(keys[i]);
            if (l > L.q || L.owner(l, key_node(keys[i])) != L.p)
                return fail(H2_ERR_STRUCT, "peer requested a node this rank does not own");
            give_x[o].push_back(keys[i]);
        } else {
            if (L.owner(L.q, keys[i]) != L.p) return fail(H2_ERR_STRUCT, "peer requested a leaf this rank does not own");
            give_h[o].push_back(keys[i]);
        }
    }
    return H2_OK;
}

struct NcclSetup : SetupComm {
    int leaf_sizes(h2_ctx *h, const std::vector<int64_t> &mine, std::vector<int64_t> &all) override
    {
        const int P = h->L.P;
        const int64_t n = (int64_t)mine.size();
        cudaError_t err;
        int64_t *dm = (int64_t *)dalloc(h, n * 8, err);
        int64_t *dall = (int64_t *)dalloc(h, n * P * 8, err);
        if (!dm || !dall) return cuda_fail(h, err, "cudaMalloc(setup)");
        H2_CUDA(h, cudaMemcpy(dm, mine.data(), n * 8, cudaMemcpyHostToDevice));
        H2_NCCL(h, g_nccl.AllGather(dm, dall, n, ncclInt64, h->comm, h->s_comm));
        H2_CUDA(h, cudaStreamSynchronize(h->s_comm));
        all.resize(n * P);
        H2_CUDA(h, cudaMemcpy(all.data(), dall, n * P * 8, cudaMemcpyDeviceToHost));
        return H2_OK;
    }
    int requests(h2_ctx *h, const RemoteNeeds &rn, std::map<int, std::vector<int64_t>> &give_x,
                 std::map<int, std::vector<int64_t>> &give_h) override
    {
        const int P = h->L.P, p = h->L.p;
        cudaError_t err;
        // request counts: cnt[2*o + 0/1] = #x^ nodes / #leaves I need from o
        std::vector<int64_t> cnt(2 * P, 0), allcnt(2 * P * P, 0);
        for (auto &kv : rn.need_x) cnt[2 * kv.first] = (int64_t)kv.second.size();
        for (auto &kv : rn.need_h) cnt[2 * kv.first + 1] = (int64_t)kv.second.size();
        int64_t *dc = (int64_t *)dalloc(h, 2 * P * 8, err);
        int64_t *dac = (int64_t *)dalloc(h, 2 * P * P * 8, err);
        if (!dc || !dac) return cuda_fail(h, err, "cudaMalloc(setup)");
        H2_CUDA(h, cudaMemcpy(dc, cnt.data(), 2 * P * 8, cudaMemcpyHostToDevice));
        H2_NCCL(h, g_nccl.AllGather(dc, dac, 2 * P, ncclInt64, h->comm, h->s_comm));
        H2_CUDA(h, cudaStreamSynchronize(h->s_comm));
        H2_CUDA(h, cudaMemcpy(allcnt.data(), dac, 2 * P * P * 8, cudaMemcpyDeviceToHost));
        std::map<int, int64_t *> dreq_out, dreq_in;
        std::map<int, std::vector<int64_t>> req_out;
        for (int o = 0; o < P; ++o) {
            if (o == p) continue;
            std::vector<int64_t> v;
            if (rn.need_x.count(o)) v.insert(v.end(), rn.need_x.at(o).begin(), rn.need_x.at(o).end());
            if (rn.need_h.count(o)) v.insert(v.end(), rn.need_h.at(o).begin(), rn.need_h.at(o).end());
            int64_t nin = allcnt[2 * P * o + 2 * p] + allcnt[2 * P * o + 2 * p + 1];
            if (!v.empty()) {
                dreq_out[o] = (int64_t *)dalloc(h, v.size() * 8, err);
                if (!dreq_out[o]) return cuda_fail(h, err, "cudaMalloc(setup)");
                H2_CUDA(h, cudaMemcpy(dreq_out[o], v.data(), v.size() * 8, cudaMemcpyHostToDevice));
                req_out[o] = v;
            }
            if (nin) {
                dreq_in[o] = (int64_t *)dalloc(h, nin * 8, err);
                if (!dreq_in[o]) return cuda_fail(h, err, "cudaMalloc(setup)");
            }
        }
        H2_NCCL(h, g_nccl.GroupStart());
        for (auto &kv : req_out)
            H2_NCCL(h, g_nccl.Send(dreq_out[kv.first], kv.second.size(), ncclInt64, kv.first, h->comm, h->s_comm));
        for (auto &kv : dreq_in) {
            int o = kv.first;
            int64_t nin = allcnt[2 * P * o + 2 * p] + allcnt[2 * P * o + 2 * p + 1];
            H2_NCCL(h, g_nccl.Recv(kv.second, nin, ncclInt64, o, h->comm, h->s_comm));
        }
        H2_NCCL(h, g_nccl.GroupEnd());
        H2_CUDA(h, cudaStreamSynchronize(h->s_comm));
        for (auto &kv : dreq_in) {
            int o = kv.first;
            int64_t nx = allcnt[2 * P * o + 2 * p], nh = allcnt[2 * P * o + 2 * p + 1];
            std::vector<int64_t> v(nx + nh);
            H2_CUDA(h, cudaMemcpy(v.data(), kv.second, (nx + nh) * 8, cudaMemcpyDeviceToHost));
            int rc = check_requests(h, o, v, nx, give_x, give_h);
            if (rc != H2_OK) return rc;
        }
        return H2_OK;
    }
    int gather_FtC(h2_ctx *h, void *dst, int64_t per) override
    {
        H2_NCCL(h, g_nccl.AllGather(h->Ft[h->L.C], dst, per, nccl_type(h->dtype), h->comm, h->s_comm));
        H2_CUDA(h, cudaStreamSynchronize(h->s_comm));
        return H2_OK;
    }
};

// In-process setup of a loopback group: every member's description is at hand.
struct LoopSetup : SetupComm {
    h2_group *g = nullptr;
    int leaf_sizes(h2_ctx *h, const std::vector<int64_t> &mine, std::vector<int64_t> &all) override
    {
        (void)mine;
        all.clear();
        for (size_t o = 0; o < g->descs.size(); ++o) {
            const int64_t n = g->layouts[o].held(g->layouts[o].q);
            for (int64_t i = 0; i < n; ++i) all.push_back(g->descs[o]->leaf_ptr[i + 1] - g->descs[o]->leaf_ptr[i]);
        }
        (void)h;
        return H2_OK;
    }
    int requests(h2_ctx *h, const RemoteNeeds &, std::map<int, std::vector<int64_t>> &give_x,
                 std::map<int, std::vector<int64_t>> &give_h) override
    {
        const int p = h->L.p;
        for (int o = 0; o < (int)g->descs.size(); ++o) {
            if (o == p) continue;
            const RemoteNeeds &ro = g->needs[o];
            std::vector<int64_t> v;
            int64_t nx = 0;
            if (ro.need_x.count(p)) { v = ro.need_x.at(p); nx = (int64_t)v.size(); }
            if (ro.need_h.count(p)) v.insert(v.end(), ro.need_h.at(p).begin(), ro.need_h.at(p).end());
            int rc = check_requests(h, o, v, nx, give_x, give_h);
            if (rc != H2_OK) return rc;
        }
        return H2_OK;
    }
    int gather_FtC(h2_ctx *h, void *dst, int64_t per) override
    {
        const int C = h->L.C;
        const int kc = h->L.k[C], kp = h->L.k[C - 1];
        for (int o = 0; o < (int)g->descs.size(); ++o) {
            const h2_desc *d = g->descs[o];
            const void *src = d->F[C];
            void *tmp = nullptr;
            if (d->mem == H2_MEM_HOST) {
                H2_CUDA(h, cudaMalloc(&tmp, (size_t)per * h->esz));
                H2_CUDA(h, cudaMemcpy(tmp, src, (size_t)per * h->esz, cudaMemcpyHostToDevice));
                src = tmp;
            }
            char *slot = static_cast<char *>(dst) + (size_t)o * per * h->esz;
            cudaError_t e = h->dtype == H2_F64
                                ? launch_transpose<double>((const double *)src, (double *)slot, 1, kc, kp, 0)
                                : launch_transpose<float>((const float *)src, (float *)slot, 1, kc, kp, 0);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (tmp) cudaFree(tmp);
            if (e != cudaSuccess) return cuda_fail(h, e, "transpose(F_C)");
        }
        return H2_OK;
    }
};

}  // namespace

// ======================================================================== create
static int create_impl(const h2_desc *d, int nv_max, const void *nccl_unique_id, h2_handle *out,
                       SetupComm *loop = nullptr, h2_group *grp = nullptr)
{
    if (!out) return fail(H2_ERR_ARG, "out is NULL");
    *out = nullptr;
    Layout L;
    int rc = validate(d, nv_max, L);
    if (rc != H2_OK) return rc;
    if (L.P > 1 && !nccl_unique_id && !loop) return fail(H2_ERR_ARG, "nccl_unique_id required when nranks > 1");

    h2_ctx *h = new (std::nothrow) h2_ctx();
    if (!h) return fail(H2_ERR_OOM, "host allocation failed");
    h->L = L;
    h->dtype = d->dtype;
    h->esz = d->dtype == H2_F64 ? 8 : 4;
    h->nv_max = nv_max;
    h->n_local = d->n_local;
    h->nleaf = L.held(L.q);
    h->group = grp;
    h->sym = (d->flags & H2_SYMMETRIC) != 0;
    if (h->sym && (nv_max != 1 || L.P != 1 || d->U_leaf != d->V_leaf)) {
        delete h;
        return fail(H2_ERR_ARG, "H2_SYMMETRIC needs nv_max == 1, one rank and V_leaf == U_leaf (same array)");
    }
    const int q = L.q, m = L.m, p = L.p, P = L.P, C = L.C;
    const std::vector<int> &k = L.k;
    const int64_t nleaf = h->nleaf;

#define H2_TRY(expr)                      \
    do {                                  \
        int rc_ = (expr);                 \
        if (rc_ != H2_OK) {               \
            std::string msg_ = g_err;     \
            release(h);                   \
            g_err = msg_;                 \
            return rc_;                   \
        }                                 \
    } while (0)
#define H2_TRYC(call)                                                 \
    do {                                                              \
        cudaError_t e_ = (call);                                      \
        if (e_ != cudaSuccess) H2_TRY(cuda_fail(h, e_, #call));       \
    } while (0)

    // ---- top-tree couplings?
    int64_t n_top = 0;
    for (int l = 0; l < C; ++l) n_top += d->S_rowptr[l][L.held(l)];
    h->has_top = (P > 1 && n_top > 0);

    // ---- NCCL communicator (loopback groups exchange in-process instead)
    if (P > 1 && !loop) {
        if (!load_nccl()) { release(h); return fail(H2_ERR_NCCL, "cannot load libnccl.so.2 (set H2_NCCL_LIB)"); }
        ncclUniqueId id;
        memcpy(&id, nccl_unique_id, sizeof(id));
        H2_DBG("rank %d: ncclCommInitRank P=%d", p, P);
        ncclResult_t r = g_nccl.CommInitRank(&h->comm, P, id, p);
        H2_DBG("rank %d: comm ready", p);
        if (r != ncclSuccess) {
            std::string msg = std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r);
            release(h);
            return fail(H2_ERR_NCCL, msg);
        }
    }
    if (P > 1) {
        H2_TRYC(cudaStreamCreateWithFlags(&h->s_comm, cudaStreamNonBlocking));
        H2_TRYC(cudaEventCreateWithFlags(&h->ev_packed, cudaEventDisableTiming));
        H2_TRYC(cudaEventCreateWithFlags(&h->ev_recv, cudaEventDisableTiming));
    }
    NcclSetup nccl_setup;
    SetupComm *sc = loop ? loop : &nccl_setup;

    // ---- per-call argument slot and the capture stream
    {
        cudaError_t err;
        h->dargs = dalloc(h, sizeof(CallArgs<double>), err);
        if (!h->dargs) H2_TRY(cuda_fail(h, err, "cudaMalloc(args)"));
        H2_TRYC(cudaMemset(h->dargs, 0, sizeof(CallArgs<double>)));
        if (h->dtype == H2_F32) {
            h->d_xmap = dalloc(h, 256, err);
            if (!h->d_xmap) H2_TRY(cuda_fail(h, err, "cudaMalloc(xmap)"));
            H2_TRYC(cudaMemset(h->d_xmap, 0, 256));
        }
        int least = 0, greatest = 0;
        H2_TRYC(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        // the tree sweeps (captured on cap_stream) get the highest priority, the leaf-level
        // coupling on its side stream the lowest (PAPER.md:509 low-priority stream)
        H2_TRYC(cudaStreamCreateWithPriority(&h->cap_stream, cudaStreamNonBlocking, greatest));
        H2_TRYC(cudaStreamCreateWithPriority(&h->s_leafc, cudaStreamNonBlocking, least));
        H2_TRYC(cudaEventCreateWithFlags(&h->ev_upleaf, cudaEventDisableTiming));
        H2_TRYC(cudaEventCreateWithFlags(&h->ev_leafc, cudaEventDisableTiming));
        H2_TRYC(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        H2_TRYC(cudaEventCreateWithFlags(&h->ev_halo, cudaEventDisableTiming));
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, dev);
        const char *en = getenv("H2_ENGINE");
        if (en && !strcmp(en, "warp")) { h->cta_min_nv = 1 << 30; h->umma_min_nv = 1 << 30; }
        else if (en && !strcmp(en, "cta")) h->cta_min_nv = 1;
    }
    // ---- operator arrays on the device; V and F re-laid out as V^T, F^T (operand order)
    const int kq = k[q];
    H2_TRY(put_array(h, d->mem, d->U_leaf, nleaf * m * kq, &h->U));
    H2_TRY(put_transposed(h, d->mem, d->V_leaf, nleaf, m, kq, &h->Vt));
    h->E.assign(q + 1, nullptr);
    h->Ft.assign(q + 1, nullptr);
    h->S.assign(q + 1, nullptr);
    double ops = 2.0 * nleaf * m * kq;
    for (int l = 1; l <= q; ++l) {
        H2_TRY(put_array(h, d->mem, d->E[l], L.held(l) * k[l] * k[l - 1], &h->E[l]));
        H2_TRY(put_transposed(h, d->mem, d->F[l], L.held(l), k[l], k[l - 1], &h->Ft[l]));
        ops += 2.0 * L.held(l) * k[l] * k[l - 1];
    }
    // symmetric storage: only the blocks (t, s) with s >= t are kept (compacted, CSR order);
    // cidx maps an original block to its compact index (-1: dropped, applied as a transpose)
    std::vector<std::vector<int64_t>> cidxS(q + 1);
    std::vector<int64_t> cidxD;
    double ops_stored = ops;
    auto keep_list = [&](const int64_t *rp, const int32_t *col, int64_t rows, std::vector<int64_t> &cidx,
                         std::vector<int64_t> &kept) {
        cidx.assign(rp[rows], -1);
        for (int64_t t = 0; t < rows; ++t)
            for (int64_t b = rp[t]; b < rp[t + 1]; ++b)
                if (col[b] >= t) { cidx[b] = (int64_t)kept.size(); kept.push_back(b); }
    };
    for (int l = 0; l <= q; ++l) {
        int64_t nb = d->S_rowptr[l][L.held(l)];
        ops += (double)nb * k[l] * k[l];
        if (h->sym) {
            std::vector<int64_t> kept;
            keep_list(d->S_rowptr[l], d->S_col[l], L.held(l), cidxS[l], kept);
            H2_TRY(put_gathered(h, d->mem, d->S[l], kept, (int64_t)k[l] * k[l], &h->S[l]));
            ops_stored += (double)kept.size() * k[l] * k[l];
        } else {
            H2_TRY(put_array(h, d->mem, d->S[l], nb * k[l] * k[l], &h->S[l]));
            ops_stored += (double)nb * k[l] * k[l];
            if (P == 1) {
                if (h->orth_pairs.empty()) h->orth_pairs.resize(q + 1);
                for (int64_t t = 0; t < L.held(l); ++t)
                    for (int64_t b = d->S_rowptr[l][t]; b < d->S_rowptr[l][t + 1]; ++b)
                        h->orth_pairs[l].push_back(make_int2((int)t, d->S_col[l][b]));
            }
        }
    }
    const int64_t nD = d->D_rowptr[nleaf];
    ops += (double)nD * m * m;
    if (h->sym) {
        std::vector<int64_t> kept;
        keep_list(d->D_rowptr, d->D_col, nleaf, cidxD, kept);
        H2_TRY(put_gathered(h, d->mem, d->D, kept, (int64_t)m * m, &h->D));
        ops_stored += (double)kept.size() * m * m;
    } else {
        H2_TRY(put_array(h, d->mem, d->D, nD * m * m, &h->D));
        ops_stored += (double)nD * m * m;
    }
    h->ops_local = ops;          // flop model: the operator as described (paper convention)
    h->ops_stored = ops_stored;  // bytes model: what is stored and streamed
    {
        // per-phase operator scalars and vector elements (per vector), DESIGN.md "Measurement"
        double Fops = 0, Eops_mid = 0, tree_up = 0, tree_mid = 0;
        for (int l = C + 1; l <= q; ++l) { Fops += (double)L.held(l) * k[l] * k[l - 1]; tree_up += (double)L.held(l) * k[l] + (double)L.held(l - 1) * k[l - 1]; }
        if (P > 1) for (int l = 1; l <= C; ++l) Fops += 0;   // top tree counted in phase 2 (replicated)
        for (int l = 1; l <= q - 1; ++l) {
            if (l <= C && P > 1) continue;
            Eops_mid += (double)L.held(l) * k[l] * k[l - 1];
            tree_mid += 2.0 * L.held(l) * k[l] + (double)L.held(l - 1) * k[l - 1];
        }
        double tree = 0;
        for (int l = 0; l <= q; ++l) tree += (double)L.held(l) * k[l];
        double Sd = 0, So = 0, Sq = 0;
        for (int l = 0; l <= q; ++l)
            for (int64_t i = 0; i < L.held(l); ++i)
                for (int64_t b = d->S_rowptr[l][i]; b < d->S_rowptr[l][i + 1]; ++b) {
                    if (h->sym && d->S_col[l][b] < L.g0(l) + i) continue;   // not stored
                    int o = L.owner(l, d->S_col[l][b]);
                    double e = (double)k[l] * k[l];
                    if (o >= 0 && o != p) So += e;
                    else if (l == q && q > 0) Sq += e;
                    else Sd += e;
                }
        h->ph_ops[8] = Sq;
        h->ph_vec[8] = 2.0 * (double)L.held(q) * k[q];
        h->ph_ops[0] = (double)nleaf * m * kq;
        h->ph_vec[0] = (double)d->n_local + (double)nleaf * kq;
        h->ph_ops[1] = Fops;
        h->ph_vec[1] = tree_up;
        h->ph_ops[3] = Sd;
        h->ph_vec[3] = 2.0 * (tree - (q > 0 ? (double)L.held(q) * k[q] : 0.0));
        h->ph_ops[4] = So;
        h->ph_ops[5] = Eops_mid;
        h->ph_vec[5] = tree_mid;
        h->ph_ops[6] = (q >= 1 ? (double)nleaf * kq * k[q - 1] : 0.0) + (double)nleaf * m * kq;
        h->ph_vec[6] = (double)nleaf * kq + (q >= 1 ? (double)L.held(q - 1) * k[q - 1] : 0.0) + 2.0 * d->n_local;
        h->ph_ops[7] = h->sym ? (double)cidxD.size() - (double)std::count(cidxD.begin(), cidxD.end(), -1) : (double)nD;
        h->ph_ops[7] *= (double)m * m;
        h->ph_vec[7] = 2.0 * d->n_local;   // X read (once), Y write
    }

    // ---- remote needs (compressed off-diagonal node lists)
    RemoteNeeds rn;
    remote_needs(d, L, rn);
    auto &need_x = rn.need_x;
    auto &need_h = rn.need_h;
    const int64_t n_diag = rn.n_diag, n_off = rn.n_off, n_root = rn.n_root, nd_diag = rn.nd_diag,
                  nd_off = rn.nd_off;

    // ---- workspaces
    h->xh_base.assign(q + 1, 0);
    h->yh_base.assign(q + 1, 0);
    int64_t xo = 0, yo = 0;
    for (int l = 0; l <= q; ++l) {
        h->xh_base[l] = xo; xo += L.held(l) * k[l];
        h->yh_base[l] = yo; yo += L.held(l) * k[l];
    }
    if (h->has_top) { h->xgather = xo; xo += (int64_t)P * k[C]; }
    h->xh_plane = xo;
    h->yh_plane = yo;
    {
        cudaError_t err;
        h->xh = dalloc(h, (size_t)xo * nv_max * h->esz, err);
        if (!h->xh) H2_TRY(cuda_fail(h, err, "cudaMalloc(x^ workspace)"));
        h->yh = dalloc(h, (size_t)yo * nv_max * h->esz, err);
        if (!h->yh) H2_TRY(cuda_fail(h, err, "cudaMalloc(y^ workspace)"));
        H2_TRYC(cudaMemset(h->xh, 0, (size_t)xo * nv_max * h->esz));
        H2_TRYC(cudaMemset(h->yh, 0, (size_t)yo * nv_max * h->esz));
    }

    // ---- distributed setup: leaf sizes of every rank, send lists, F_C of every rank
    std::vector<int64_t> gleaf_size;        // global leaf sizes (P > 1)
    std::map<int, std::vector<int64_t>> give_x, give_h;   // what each peer needs from me
    if (P > 1) {
        cudaError_t err;
        std::vector<int64_t> mine(nleaf);
        for (int64_t i = 0; i < nleaf; ++i) mine[i] = d->leaf_ptr[i + 1] - d->leaf_ptr[i];
        H2_TRY(sc->leaf_sizes(h, mine, gleaf_size));
        H2_TRY(sc->requests(h, rn, give_x, give_h));
        H2_DBG("rank %d: request lists exchanged (give_x peers %zu, give_h peers %zu)", p, give_x.size(), give_h.size());
        // F_C^T of every rank for the replicated top upsweep (branch-root transfers
        // duplicated at the leaf level of the root branch)
        if (h->has_top) {
            int64_t per = (int64_t)k[C] * k[C - 1];
            void *all = dalloc(h, (size_t)per * P * h->esz, err);
            if (!all) H2_TRY(cuda_fail(h, err, "cudaMalloc(F_C)"));
            H2_TRY(sc->gather_FtC(h, all, per));
            h->FtC_all = all;
        }
    }

    // ---- peers and exchange buffers (per-peer chunks of nv_max x cnt, nv-independent offsets)
    std::map<int64_t, std::pair<int64_t, int64_t>> xrecv_pos;   // key -> (elem offset, ld)
    std::map<int64_t, std::pair<int64_t, int64_t>> hrecv_pos;   // leaf -> (row offset, ld)
    std::vector<PackSeg> segs_x, segs_h;
    for (int o = 0; o < P; ++o) {
        if (o == p) continue;
        bool any = need_x.count(o) || need_h.count(o) || give_x.count(o) || give_h.count(o);
        if (!any) continue;
        h2_ctx::Peer pr;
        pr.rank = o;
        if (need_x.count(o))
            for (int64_t key : need_x[o]) pr.xr_cnt += k[key_level(key)];
        if (give_x.count(o))
            for (int64_t key : give_x[o]) pr.xs_cnt += k[key_level(key)];
        if (need_h.count(o))
            for (int64_t g : need_h[o]) pr.hr_cnt += gleaf_size[g];
        if (give_h.count(o))
            for (int64_t g : give_h[o]) pr.hs_cnt += gleaf_size[g];
        pr.xr_off = h->xrecv_tot; h->xrecv_tot += pr.xr_cnt * nv_max;
        pr.xs_off = h->xsend_tot; h->xsend_tot += pr.xs_cnt * nv_max;
        pr.hr_off = h->hrecv_tot; h->hrecv_tot += pr.hr_cnt * nv_max;
        pr.hs_off = h->hsend_tot; h->hsend_tot += pr.hs_cnt * nv_max;
        int64_t pos = 0;
        if (need_x.count(o))
            for (int64_t key : need_x[o]) { xrecv_pos[key] = {pr.xr_off + pos, pr.xr_cnt}; pos += k[key_level(key)]; }
        pos = 0;
        if (give_x.count(o))
            for (int64_t key : give_x[o]) {
                int l = key_level(key);
                int64_t slot = key_node(key) - L.g0(l);
                segs_x.push_back({h->xh_base[l] + slot * k[l], pr.xs_off + pos, k[l], (int32_t)pr.xs_cnt});
                pos += k[l];
            }
        pos = 0;
        if (need_h.count(o))
            for (int64_t g : need_h[o]) { hrecv_pos[g] = {pr.hr_off + pos, pr.hr_cnt}; pos += gleaf_size[g]; }
        pos = 0;
        if (give_h.count(o))
            for (int64_t g : give_h[o]) {
                int64_t slot = g - L.g0(q);
                int32_t len = (int32_t)(d->leaf_ptr[slot + 1] - d->leaf_ptr[slot]);
                segs_h.push_back({d->leaf_ptr[slot], pr.hs_off + pos, len, (int32_t)pr.hs_cnt});
                pos += len;
            }
        h->peers.push_back(pr);
    }
    if (P > 1) {
        cudaError_t err;
        h->xsend = dalloc(h, (size_t)h->xsend_tot * h->esz, err);
        h->xrecv = dalloc(h, (size_t)h->xrecv_tot * h->esz, err);
        h->hsend = dalloc(h, (size_t)h->hsend_tot * h->esz, err);
        h->hrecv = dalloc(h, (size_t)h->hrecv_tot * h->esz, err);
        if (!h->xsend || !h->xrecv || !h->hsend || !h->hrecv) H2_TRY(cuda_fail(h, err, "cudaMalloc(exchange buffers)"));
        const char *ex = getenv("H2_EXCHANGE");
        h->p2p = !loop && !(ex && !strcmp(ex, "nccl"));
        h->p2p_direct = h->p2p && ex && !strcmp(ex, "p2p-direct");
        if (h->p2p) {
            // ---- device-initiated exchange: signal block, IPC handles of x^ / hsend / signals and
            //      every rank's chunk offsets, exchanged once over the communicator
            h->sig = (int32_t *)dalloc(h, SIG_INTS * sizeof(int32_t), err);
            if (!h->sig) H2_TRY(cuda_fail(h, err, "cudaMalloc(signals)"));
            H2_TRYC(cudaMemset(h->sig, 0, SIG_INTS * sizeof(int32_t)));
            const size_t rec = 3 * sizeof(cudaIpcMemHandle_t) + (size_t)P * sizeof(int64_t);
            std::vector<unsigned char> mine(rec, 0), all(rec * P, 0);
            cudaIpcMemHandle_t hd[3];
            H2_TRYC(cudaIpcGetMemHandle(&hd[0], h->xh));
            H2_TRYC(cudaIpcGetMemHandle(&hd[1], h->hsend));
            H2_TRYC(cudaIpcGetMemHandle(&hd[2], h->sig));
            memcpy(mine.data(), hd, sizeof(hd));
            std::vector<int64_t> hso(P, -1);
            for (const auto &pr : h->peers) hso[pr.rank] = pr.hs_off;
            memcpy(mine.data() + sizeof(hd), hso.data(), P * sizeof(int64_t));
            void *dmine = dalloc(h, rec, err), *dall = dalloc(h, rec * P, err);
            if (!dmine || !dall) H2_TRY(cuda_fail(h, err, "cudaMalloc(setup)"));
            H2_TRYC(cudaMemcpy(dmine, mine.data(), rec, cudaMemcpyHostToDevice));
            H2_TRY([&]() -> int { H2_NCCL(h, g_nccl.AllGather(dmine, dall, rec, ncclUint8, h->comm, h->s_comm)); return H2_OK; }());
            H2_TRYC(cudaStreamSynchronize(h->s_comm));
            H2_TRYC(cudaMemcpy(all.data(), dall, rec * P, cudaMemcpyDeviceToHost));
            h->pmap.assign(P, h2_ctx::PeerMap{});
            for (int o = 0; o < P; ++o) {
                if (o == p) continue;
                const unsigned char *r = all.data() + rec * o;
                cudaIpcMemHandle_t ho[3];
                memcpy(ho, r, sizeof(ho));
                void *ptr[3];
                for (int i = 0; i < 3; ++i) {
                    H2_TRYC(cudaIpcOpenMemHandle(&ptr[i], ho[i], cudaIpcMemLazyEnablePeerAccess));
                    h->ipc_open.push_back(ptr[i]);
                }
                h->pmap[o].xh = ptr[0];
                h->pmap[o].hsend = ptr[1];
                h->pmap[o].sig = (int32_t *)ptr[2];
                memcpy(&h->pmap[o].hs_off, r + sizeof(ho) + (size_t)p * sizeof(int64_t), sizeof(int64_t));
            }
            // who reads what: x^ readers / sources (all ranks when the top tree gathers roots)
            std::vector<int32_t> begin, wxl, wxu, wh;
            std::vector<int32_t *> txl, txu, th, tcx, tch;
            for (int o = 0; o < P; ++o) {
                if (o == p) continue;
                const bool x_reader = give_x.count(o) || h->has_top, x_source = need_x.count(o) || h->has_top;
                const bool h_reader = give_h.count(o) > 0, h_source = need_h.count(o) > 0;
                int32_t *os = h->pmap[o].sig;
                if (x_reader) { begin.push_back(SIG_CONS_X + o); txl.push_back(os + SIG_XLEAF + p); txu.push_back(os + SIG_XUP + p); }
                if (h_reader) { begin.push_back(SIG_CONS_H + o); th.push_back(os + SIG_HALO + p); }
                if (x_source) { wxl.push_back(SIG_XLEAF + o); wxu.push_back(SIG_XUP + o); tcx.push_back(os + SIG_CONS_X + p); }
                if (h_source) { wh.push_back(SIG_HALO + o); tch.push_back(os + SIG_CONS_H + p); }
            }
            auto upload_i = [&](const std::vector<int32_t> &v, int32_t **out, int &n) -> int {
                cudaError_t e2;
                n = (int)v.size();
                *out = (int32_t *)dalloc(h, (v.size() + 1) * sizeof(int32_t), e2);
                if (!*out) return cuda_fail(h, e2, "cudaMalloc(signal lists)");
                if (!v.empty()) H2_CUDA(h, cudaMemcpy(*out, v.data(), v.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
                return H2_OK;
            };
            auto upload_p = [&](const std::vector<int32_t *> &v, int32_t ***out, int &n) -> int {
                cudaError_t e2;
                n = (int)v.size();
                *out = (int32_t **)dalloc(h, (v.size() + 1) * sizeof(int32_t *), e2);
                if (!*out) return cuda_fail(h, e2, "cudaMalloc(signal lists)");
                if (!v.empty()) H2_CUDA(h, cudaMemcpy(*out, v.data(), v.size() * sizeof(int32_t *), cudaMemcpyHostToDevice));
                return H2_OK;
            };
            H2_TRY(upload_i(begin, &h->d_begin_waits, h->n_begin_waits));
            H2_TRY(upload_i(wxl, &h->d_wait_xl, h->n_wait_xl));
            H2_TRY(upload_i(wxu, &h->d_wait_xu, h->n_wait_xu));
            H2_TRY(upload_i(wh, &h->d_wait_h, h->n_wait_h));
            H2_TRY(upload_p(txl, &h->d_tgt_xl, h->n_tgt_xl));
            H2_TRY(upload_p(txu, &h->d_tgt_xu, h->n_tgt_xu));
            H2_TRY(upload_p(th, &h->d_tgt_h, h->n_tgt_h));
            H2_TRY(upload_p(tcx, &h->d_tgt_cx, h->n_tgt_cx));
            H2_TRY(upload_p(tch, &h->d_tgt_ch, h->n_tgt_ch));
            H2_DBG("rank %d: p2p exchange mapped (%d x-sources, %d halo sources)", p, h->n_wait_xu, h->n_wait_h);
        }
    }

    // ---- the task / block tables
    std::vector<Task> tasks;
    std::vector<Blk> blks;
    auto esz = h->esz;
    auto at = [esz](const void *base, int64_t elems) -> const void * {
        return static_cast<const char *>(base) + (size_t)elems * esz;
    };
    // engine class of a row count (Simt lanes-per-row / DMMA m-tiles): <=16, <=32, <=64
    auto cls_of = [](int r) { return r <= 16 ? 0 : r <= 32 ? 1 : 2; };
    const int cls_r[3] = {16, 32, 64};

    // (1) upsweep leaves: x^_s = V_s^T x_s
    h->up_leaf.t0 = tasks.size();
    for (int64_t s = 0; s < nleaf; ++s) {
        Task t{h->xh_base[q] + s * kq, (int64_t)blks.size(), 1, (uint8_t)kq, (uint8_t)m,
               (uint8_t)(d->leaf_ptr[s + 1] - d->leaf_ptr[s]), 0};
        blks.push_back({at(h->Vt, s * kq * m), d->leaf_ptr[s], (int32_t)t.rows, 0});
        tasks.push_back(t);
    }
    h->up_leaf.n = (int)nleaf;
    h->up_leaf.r = kq;
    // (2) local upsweep transfers, parents at levels q-1 .. C
    for (int l = q; l >= C + 1; --l) {
        Phase ph;
        ph.t0 = tasks.size();
        ph.r = k[l - 1];
        for (int64_t i = 0; i < L.held(l - 1); ++i) {
            Task t{h->xh_base[l - 1] + i * k[l - 1], (int64_t)blks.size(), 2, (uint8_t)k[l - 1],
                   (uint8_t)k[l], 0, 0};
            for (int64_t c = 2 * i; c <= 2 * i + 1; ++c)
                blks.push_back({at(h->Ft[l], c * k[l] * k[l - 1]), h->xh_base[l] + c * k[l], k[l], 0});
            tasks.push_back(t);
        }
        ph.n = (int)L.held(l - 1);
        h->up_lv.push_back(ph);
        h->up_lv_level.push_back(l);
    }
    // (3) replicated top upsweep (P > 1 with top couplings): parents at levels C-1 .. 0
    if (h->has_top) {
        for (int l = C; l >= 1; --l) {
            Phase ph;
            ph.t0 = tasks.size();
            ph.r = k[l - 1];
            for (int64_t i = 0; i < ((int64_t)1 << (l - 1)); ++i) {
                Task t{h->xh_base[l - 1] + i * k[l - 1], (int64_t)blks.size(), 2, (uint8_t)k[l - 1],
                       (uint8_t)k[l], 0, 0};
                for (int64_t c = 2 * i; c <= 2 * i + 1; ++c) {
                    if (l == C)
                        blks.push_back({at(h->FtC_all, c * k[l] * k[l - 1]), h->xgather + c * k[l], k[l], 0});
                    else
                        blks.push_back({at(h->Ft[l], c * k[l] * k[l - 1]), h->xh_base[l] + c * k[l], k[l], 0});
                }
                tasks.push_back(t);
            }
            ph.n = 1 << (l - 1);
            h->top_up_lv.push_back(ph);
            h->top_up_level.push_back(l);
        }
    }
    // (4) coupling multiply, diagonal part, all levels in one launch per engine class
    //     (PAPER.md:328-331, 496); every held row gets a task (empty rows write 0)
    std::vector<Task> offd_tasks[2][3];    // [leaf level, upper levels][class]
    std::vector<Blk> offd_blks[2][3];
    std::vector<Task> p2p_tasks[2][3];     // [leaf level, upper levels][class]
    std::vector<Blk> p2p_blks[2][3];
    std::vector<int> p2p_owner[2][3];
    {
        // classes: engine class ci (0..2) for the levels above the leaves, 3 + ci for the leaf
        // level (its coupling only needs x^ of the leaves: it runs on its own stream right after
        // the leaf projection, concurrent with the upsweep transfers)
        std::vector<Task> cls[6];
        std::vector<int> cls_lvl[6];
        std::vector<std::vector<Blk>> cls_blk[6];
        for (int l = 0; l <= q; ++l) {
            if (l < C && !h->has_top) {
                // top levels without couplings: y^ stays zero (workspace zeroed once), no tasks
                continue;
            }
            const int64_t *rp = d->S_rowptr[l];
            int ci = cls_of(k[l]);
            for (int64_t i = 0; i < L.held(l); ++i) {
                std::vector<Blk> bl, offb;
                for (int64_t b = rp[i]; b < rp[i + 1]; ++b) {
                    int64_t s = d->S_col[l][b];
                    int o = L.owner(l, s);
                    if (h->sym && cidxS[l][b] < 0) continue;      // applied as the transpose of (s, t)
                    const void *A = at(h->S[l], (h->sym ? cidxS[l][b] : b) * k[l] * k[l]);
                    if (o < 0 || o == p)
                        bl.push_back({A, h->xh_base[l] + (s - L.g0(l)) * k[l], k[l],
                                      (int32_t)(h->sym && s > L.g0(l) + i ? -1 : 0)});
                    else if (h->p2p_direct) {
                        // the owner's x^ plane has my layout: its slot of node s at its level-l base
                        const int64_t og0 = (int64_t)o << (l - C);
                        offb.push_back({A, h->xh_base[l] + (s - og0) * k[l], k[l], (int32_t)o});
                    } else {
                        auto pos = xrecv_pos.at(node_key(l, s));
                        offb.push_back({A, pos.first, k[l], (int32_t)pos.second});
                    }
                }
                Task t{h->yh_base[l] + i * k[l], 0, (int32_t)bl.size(), (uint8_t)k[l], (uint8_t)k[l], 0, 0};
                const int cj = (l == q && q > 0) ? 3 + ci : ci;
                cls[cj].push_back(t);
                cls_lvl[cj].push_back(l);
                cls_blk[cj].push_back(bl);
                if (!offb.empty() && h->p2p_direct) {
                    // one task per (row, owner): each launch reads one peer's mapped x^ plane;
                    // Blk::xld carried the owner rank only until here (0 = the plane's own ld)
                    const int g = (l == q) ? 0 : 1;
                    std::map<int, std::vector<Blk>> by;
                    for (Blk bb : offb) { const int o = bb.xld; bb.xld = 0; by[o].push_back(bb); }
                    for (auto &kv : by) {
                        Task to = t;
                        to.nblk = (int32_t)kv.second.size();
                        to.blk0 = (int64_t)p2p_blks[g][ci].size();
                        p2p_tasks[g][ci].push_back(to);
                        p2p_owner[g][ci].push_back(kv.first);
                        p2p_blks[g][ci].insert(p2p_blks[g][ci].end(), kv.second.begin(), kv.second.end());
                    }
                } else if (!offb.empty()) {
                    const int g = (l == q) ? 0 : 1;
                    Task to = t;
                    to.nblk = (int32_t)offb.size();
                    to.blk0 = (int64_t)offd_blks[g][ci].size();
                    offd_tasks[g][ci].push_back(to);
                    offd_blks[g][ci].insert(offd_blks[g][ci].end(), offb.begin(), offb.end());
                }
            }
        }
        for (int cj = 0; cj < 6; ++cj) {
            // longest rows first (better tail balance)
            std::vector<size_t> ord(cls[cj].size());
            std::iota(ord.begin(), ord.end(), 0);
            std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
                return cls[cj][a].nblk > cls[cj][b].nblk;
            });
            Phase ph;
            ph.t0 = tasks.size();
            ph.r = cls_r[cj % 3];
            ph.n = (int)ord.size();
            for (size_t o : ord) {
                Task t = cls[cj][o];
                t.blk0 = (int64_t)blks.size();
                blks.insert(blks.end(), cls_blk[cj][o].begin(), cls_blk[cj][o].end());
                tasks.push_back(t);
            }
            if (ph.n) (cj < 3 ? h->coup_diag : h->coup_leaf).push_back(ph);
        }
        // device-initiated exchange: one launch per (level group, class, owner)
        for (int g = 0; g < 2; ++g)
            for (int ci = 0; ci < 3; ++ci) {
                std::map<int, std::vector<size_t>> by;
                for (size_t u = 0; u < p2p_tasks[g][ci].size(); ++u) by[p2p_owner[g][ci][u]].push_back(u);
                for (auto &kv : by) {
                    h2_ctx::P2PPhase pp{kv.first, g, Phase{}};
                    pp.ph.t0 = tasks.size();
                    pp.ph.r = cls_r[ci];
                    pp.ph.n = (int)kv.second.size();
                    for (size_t u : kv.second) {
                        Task t = p2p_tasks[g][ci][u];
                        const int64_t b0 = t.blk0;
                        t.blk0 = (int64_t)blks.size();
                        blks.insert(blks.end(), p2p_blks[g][ci].begin() + b0, p2p_blks[g][ci].begin() + b0 + t.nblk);
                        tasks.push_back(t);
                    }
                    h->p2p_phases.push_back(pp);
                }
            }
        for (int g = 0; g < 2; ++g)
            for (int ci = 0; ci < 3; ++ci) {
                Phase &ph = g == 0 ? h->coup_off_leaf[ci] : h->coup_off[ci];
                ph.t0 = tasks.size();
                ph.r = cls_r[ci];
                ph.n = (int)offd_tasks[g][ci].size();
                int64_t b0 = (int64_t)blks.size();
                for (Task t : offd_tasks[g][ci]) { t.blk0 += b0; tasks.push_back(t); }
                blks.insert(blks.end(), offd_blks[g][ci].begin(), offd_blks[g][ci].end());
            }
    }
    // (5) downsweep transfers y^_c += E_c y^_parent, levels 1 .. q-1;
    //     top levels only when the top tree has couplings (else they are all zero)
    for (int l = 1; l <= q - 1; ++l) {
        if (l <= C && !h->has_top) continue;
        Phase ph;
        ph.t0 = tasks.size();
        ph.r = k[l];
        for (int64_t c = 0; c < L.held(l); ++c) {
            int64_t g = L.g0(l) + c, gp = g >> 1;
            int64_t pslot = gp - L.g0(l - 1);
            Task t{h->yh_base[l] + c * k[l], (int64_t)blks.size(), 1, (uint8_t)k[l], (uint8_t)k[l - 1], 0, 0};
            blks.push_back({at(h->E[l], c * k[l] * k[l - 1]), h->yh_base[l - 1] + pslot * k[l - 1], k[l - 1], 0});
            tasks.push_back(t);
        }
        ph.n = (int)L.held(l);
        h->down_lv.push_back(ph);
        h->down_level.push_back(l);
    }
    // (6) leaves: last transfer + U expansion (Y += alpha U z)
    {
        const bool hasE = q >= 1 && (q > C || h->has_top);
        h->leaf.t0 = tasks.size();
        h->leaf.n = (int)nleaf;
        h->leaf.r = m;
        for (int64_t t = 0; t < nleaf; ++t) {
            int64_t rows = d->leaf_ptr[t + 1] - d->leaf_ptr[t];
            Task tk{d->leaf_ptr[t], (int64_t)blks.size(), 0, (uint8_t)m, (uint8_t)m, (uint8_t)rows,
                    (uint8_t)(hasE ? TF_HAS_E : 0)};
            if (hasE) {
                int64_t g = L.g0(q) + t, gp = g >> 1;
                int64_t pslot = gp - L.g0(q - 1);
                blks.push_back({at(h->E[q], t * kq * k[q - 1]), h->yh_base[q - 1] + pslot * k[q - 1], k[q - 1], 0});
            }
            blks.push_back({at(h->U, t * m * kq), h->yh_base[q] + t * kq, kq, 0});
            tk.nblk = (int32_t)(blks.size() - tk.blk0);
            tasks.push_back(tk);
        }
        // the same E blocks as row tasks y^_t += E_t y^_p (the tcgen05 FP32 leaf path applies the
        // leaf-level transfer before its U + dense kernel)
        h->leafE.t0 = tasks.size();
        h->leafE.n = hasE ? (int)nleaf : 0;
        h->leafE.r = kq;
        if (hasE)
            for (int64_t t = 0; t < nleaf; ++t) {
                const Task &lt = tasks[h->leaf.t0 + t];
                tasks.push_back(Task{h->yh_base[q] + t * kq, lt.blk0, 1, (uint8_t)kq, (uint8_t)k[q - 1], (uint8_t)kq, 0});
            }
    }
    // (7) dense near field + epilogue (Y = alpha A_de X + beta Y), one task per leaf
    {
        h->dense.t0 = tasks.size();
        h->dense.n = (int)nleaf;
        h->dense.r = m;
        for (int64_t t = 0; t < nleaf; ++t) {
            int64_t rows = d->leaf_ptr[t + 1] - d->leaf_ptr[t];
            Task tk{d->leaf_ptr[t], (int64_t)blks.size(), 0, (uint8_t)m, (uint8_t)m, (uint8_t)rows, 0};
            for (int64_t b = d->D_rowptr[t]; b < d->D_rowptr[t + 1]; ++b) {
                int64_t s = d->D_col[b];
                int o = L.owner(q, s);
                if (h->sym && cidxD[b] < 0) continue;
                const void *A = at(h->D, (h->sym ? cidxD[b] : b) * m * m);
                if (o == p) {
                    int64_t slot = s - L.g0(q);
                    blks.push_back({A, d->leaf_ptr[slot], (int32_t)(d->leaf_ptr[slot + 1] - d->leaf_ptr[slot]),
                                    (int32_t)(h->sym && s > L.g0(q) + t ? -1 : 0)});
                } else {
                    auto pos = hrecv_pos.at(s);
                    blks.push_back({A, -1 - pos.first, (int32_t)gleaf_size[s], (int32_t)pos.second});
                }
            }
            tk.nblk = (int32_t)(blks.size() - tk.blk0);
            tasks.push_back(tk);
        }
    }
    // ---- tree stages: levels with many nodes run as one full-grid launch each; the small top
    //      levels (<= 16 nodes) are fused into one launch whose CTAs each own a subtree and sweep
    //      it level by level (k_tree), saving the per-level launch latency
    {
        const int SMALL = 16;
        auto group = [&](const std::vector<Phase> &ph, bool up, std::vector<h2_ctx::Stage> &out) {
            size_t i = 0;
            while (i < ph.size()) {
                size_t j = i + 1;
                if (ph[i].n <= SMALL)
                    while (j < ph.size() && (int)(j - i) < TREE_MAXLEV && ph[j].n <= SMALL &&
                           (up ? (int64_t)ph[j].n * 2 == ph[j - 1].n : (int64_t)ph[j].n == 2 * (int64_t)ph[j - 1].n))
                        ++j;
                h2_ctx::Stage s{};
                s.st.nlev = (int)(j - i);
                if (j - i == 1) s.nctas = ph[i].n >= WPB ? ph[i].n / WPB : 1;
                else s.nctas = up ? ph[j - 1].n : ph[i].n;
                s.r = 1;
                for (size_t u = i; u < j; ++u) {
                    s.st.t0[u - i] = ph[u].t0;
                    s.st.per[u - i] = (ph[u].n + s.nctas - 1) / s.nctas;
                    s.st.cnt[u - i] = ph[u].n;
                    s.r = std::max(s.r, ph[u].r);
                }
                out.push_back(s);
                i = j;
            }
        };
        group(h->up_lv, true, h->up_stages);
        group(h->top_up_lv, true, h->top_stages);
        group(h->down_lv, false, h->down_stages);
    }
    // ---- heap-addressed sweeps (valid when every transfer level is a local standard level:
    //      always for P = 1, and for P > 1 without top-tree couplings)
    {
        // levels with <= TOPN output nodes are fused into one single-CTA launch; one SM streams
        // only ~1/148 of the HBM bandwidth, so only the tiniest levels are worth fusing -- and
        // only while one vector chunk covers nv (nv_max > 16: the (node, chunk) warps of a
        // level-per-launch sweep win, cfg3s 4.13 -> 4.06 ms; cfg2 keeps 8)
        const int TOPN = h->nv_max > 16 ? 0 : 8;
        h->use_sweep = !h->has_top;
        auto lvl_up = [&](int lc) {              // parents at lc - 1, children at lc
            SweepLevel v{h->Ft[lc], h->xh_base[lc], h->xh_base[lc - 1], (int32_t)L.held(lc - 1),
                         (int16_t)k[lc - 1], (int16_t)k[lc]};
            return v;
        };
        auto lvl_dn = [&](int l) {
            SweepLevel v{h->E[l], h->yh_base[l - 1], h->yh_base[l], (int32_t)L.held(l), (int16_t)k[l],
                         (int16_t)k[l - 1]};
            return v;
        };
        if (h->use_sweep) {
            // launches: the wide levels alone (full-grid parallelism for most of the bytes), the
            // latency-bound levels of <= GMAX nodes in groups of J (one CTA per subtree, CTA
            // barriers between its levels: 1 launch instead of J), the tiny top levels (<= TOPN
            // nodes) in one CTA.  Measured on cfg2 (J = 1..4): up 86 -> 76 us, down 57 -> 47 us at
            // nv = 1; grouping the wide levels too slowed cfg5 FP32 (fewer warps on most bytes).
            // (H2_SWEEP_J / H2_SWEEP_GMAX: A/B overrides of the grouping)
            const char *ej = getenv("H2_SWEEP_J"), *eg = getenv("H2_SWEEP_GMAX");
            const int J = ej ? std::max(1, atoi(ej)) : 4, GMAX = eg ? atoi(eg) : 1024;
            auto push = [&](std::vector<SweepParams> &dst, std::vector<int> &ctas, std::vector<int> &thr,
                            const std::vector<SweepLevel> &g, bool up) {
                if (g.empty()) return;
                SweepParams sp{};
                for (const auto &v : g) sp.lv[sp.nlev++] = v;
                if (g.size() == 1) {
                    ctas.push_back((g[0].n + WPB - 1) / WPB);
                    thr.push_back(WPB * 32);
                } else {
                    // a subtree per CTA: as many CTAs as nodes at the group's coarsest level
                    const int nct = up ? g.back().n : g.front().n;
                    const int widest = up ? g.front().n : g.back().n;
                    ctas.push_back(nct);
                    thr.push_back(32 * std::min(WPB, std::max(1, widest / nct)));
                }
                dst.push_back(sp);
            };
            std::vector<SweepLevel> grp, top;
            bool first = true;
            for (int lc : h->up_lv_level) {
                SweepLevel v = lvl_up(lc);
                h->sweep_r_up = std::max(h->sweep_r_up, (int)v.r);
                if (v.n <= TOPN) { top.push_back(v); continue; }
                if (first || v.n > GMAX) { push(h->up_sweeps, h->up_sweep_ctas, h->up_sweep_thr, {v}, true); first = false; continue; }
                grp.push_back(v);
                if ((int)grp.size() == J) { push(h->up_sweeps, h->up_sweep_ctas, h->up_sweep_thr, grp, true); grp.clear(); }
            }
            push(h->up_sweeps, h->up_sweep_ctas, h->up_sweep_thr, grp, true);
            if (!top.empty()) {
                SweepParams sp{};
                for (const auto &v : top) if (sp.nlev < SWEEP_MAXLEV) sp.lv[sp.nlev++] = v;
                h->up_sweeps.push_back(sp);
                h->up_sweep_ctas.push_back(1);
                h->up_sweep_thr.push_back(512);
            }
            // downsweep: top levels first (one CTA), then groups of J, the widest level alone last
            std::vector<SweepLevel> dn;
            for (int l : h->down_level) { dn.push_back(lvl_dn(l)); h->sweep_r_dn = std::max(h->sweep_r_dn, (int)dn.back().r); }
            size_t u = 0;
            SweepParams dtop{};
            while (u < dn.size() && dn[u].n <= TOPN && dtop.nlev < SWEEP_MAXLEV) dtop.lv[dtop.nlev++] = dn[u++];
            if (dtop.nlev) { h->dn_sweeps.push_back(dtop); h->dn_sweep_ctas.push_back(1); h->dn_sweep_thr.push_back(512); }
            grp.clear();
            for (; u < dn.size(); ++u) {
                if (u + 1 == dn.size() || dn[u].n > GMAX) {
                    push(h->dn_sweeps, h->dn_sweep_ctas, h->dn_sweep_thr, grp, false);
                    grp.clear();
                    push(h->dn_sweeps, h->dn_sweep_ctas, h->dn_sweep_thr, {dn[u]}, false);
                    continue;
                }
                grp.push_back(dn[u]);
                if ((int)grp.size() == J) { push(h->dn_sweeps, h->dn_sweep_ctas, h->dn_sweep_thr, grp, false); grp.clear(); }
            }
        }
    }
    // ---- contiguity of every task's block run (TF_ACONTIG): A_b == A_0 + b r c
    for (Task &t : tasks) {
        const int64_t ti = &t - tasks.data();
        if (ti >= h->leaf.t0 && ti < h->leaf.t0 + h->leaf.n) continue;   // [E][U]: not a run
        int64_t first = t.blk0;
        int64_t last = t.blk0 + t.nblk;
        if (first >= last) continue;
        const size_t bsz = (size_t)t.r * t.c * h->esz;
        bool ok = true;
        const char *a0 = static_cast<const char *>(blks[first].A);
        for (int64_t b = first; b < last && ok; ++b)
            ok = static_cast<const char *>(blks[b].A) == a0 + (size_t)(b - first) * bsz;
        if (ok) t.flags |= TF_ACONTIG;
    }
    // ---- upload the plan
    {
        cudaError_t err;
        h->d_tasks = (Task *)dalloc(h, tasks.size() * sizeof(Task), err);
        h->d_blks = (Blk *)dalloc(h, blks.size() * sizeof(Blk), err);
        std::vector<PackSeg> segs = segs_x;
        h->seg_x0 = 0; h->nseg_x = (int64_t)segs_x.size();
        h->seg_h0 = (int64_t)segs.size(); h->nseg_h = (int64_t)segs_h.size();
        segs.insert(segs.end(), segs_h.begin(), segs_h.end());
        if (h->p2p && !h->p2p_direct) {
            // pull segments: node (l, s) of owner o sits in o's plane at xh_base[l] + (s - o's g0) k^l
            // and lands in my receive chunk exactly where the NCCL receive would put it
            for (int g = 0; g < 2; ++g)
                for (const auto &pr : h->peers) {
                    if (!need_x.count(pr.rank)) continue;
                    h2_ctx::Pull pl{pr.rank, g, (int64_t)segs.size(), 0};
                    int64_t pos = 0;
                    for (int64_t key : need_x[pr.rank]) {
                        const int l = key_level(key);
                        const int64_t og0 = (int64_t)pr.rank << (l - C);
                        if ((l == q) == (g == 0))
                            segs.push_back({h->xh_base[l] + (key_node(key) - og0) * k[l], pr.xr_off + pos, k[l],
                                            (int32_t)pr.xr_cnt});
                        pos += k[l];
                    }
                    pl.nseg = (int64_t)segs.size() - pl.seg0;
                    if (pl.nseg) h->pulls.push_back(pl);
                }
        }
        h->d_segs = (PackSeg *)dalloc(h, segs.size() * sizeof(PackSeg), err);
        if (!h->d_tasks || !h->d_blks || !h->d_segs) H2_TRY(cuda_fail(h, err, "cudaMalloc(plan)"));
        H2_TRYC(cudaMemcpy(h->d_tasks, tasks.data(), tasks.size() * sizeof(Task), cudaMemcpyHostToDevice));
        H2_TRYC(cudaMemcpy(h->d_blks, blks.data(), blks.size() * sizeof(Blk), cudaMemcpyHostToDevice));
        if (!segs.empty())
            H2_TRYC(cudaMemcpy(h->d_segs, segs.data(), segs.size() * sizeof(PackSeg), cudaMemcpyHostToDevice));
        H2_TRYC(cudaDeviceSynchronize());
    }
    H2_DBG("rank %d: plan uploaded (%zu tasks, %zu blocks, %zu peers, has_top %d)", p, tasks.size(), blks.size(),
           h->peers.size(), (int)h->has_top);
    int64_t peers_n = (int64_t)h->peers.size(), xr = 0, hr = 0;
    for (auto &kv : need_x) xr += (int64_t)kv.second.size();
    for (auto &kv : need_h) hr += (int64_t)kv.second.size();
    int64_t c8[8] = {n_diag, n_off, n_root, nd_diag, nd_off, peers_n, xr, hr};
    memcpy(h->counts, c8, sizeof(c8));
    // kernels per call: k_set_args, k_up_leaf, the sweeps, k_rows per coupling class, k_leaf_dense
    int launches = 3 + (int)(h->use_sweep ? h->up_sweeps.size() : h->up_stages.size()) +
                   (int)h->coup_diag.size() + (int)h->coup_leaf.size() +
                   (int)(h->use_sweep ? h->dn_sweeps.size() : h->down_stages.size());
    // distributed extras: the packs and off-diagonal launches (NCCL), or the pack, the signal /
    // wait kernels and the per-owner off-diagonal launches (device-initiated exchange)
    int dist = 0;
    if (P > 1 && !h->p2p) {
        dist += 2;   // pack x^, pack halo
        for (int ci = 0; ci < 3; ++ci) dist += (h->coup_off[ci].n ? 1 : 0) + (h->coup_off_leaf[ci].n ? 1 : 0);
    } else if (P > 1) {
        dist += 2 + (int)h->p2p_phases.size() + (int)h->pulls.size();   // p2p_begin, pack halo, off-diagonal / pulls
        if (!h->p2p_direct)
            for (int ci = 0; ci < 3; ++ci) dist += (h->coup_off[ci].n ? 1 : 0) + (h->coup_off_leaf[ci].n ? 1 : 0);
        dist += (h->n_tgt_h > 0) + (h->n_wait_h > 0) + (h->n_tgt_ch > 0) + (h->n_tgt_xl > 0) + (h->n_tgt_xu > 0) +
                (h->n_wait_xl > 0) + (h->n_wait_xu > 0) + (h->n_tgt_cx > 0) + (h->has_top && h->n_wait_xu > 0);
    }
    if (h->has_top) dist += (int)h->top_stages.size();
    h->launches_per_call = launches + dist + (h->sym ? 1 : 0);   // + the beta pass of the symmetric leaves
    // CTA engine: k_set_args, up_leaf, one launch per coupling class / transfer level, the leaves
    h->launches_cta = 3 + (int)h->coup_leaf.size() + (int)h->up_lv.size() + (int)h->coup_diag.size() +
                      (int)h->down_lv.size() + dist;
    h->launches_umma = h->launches_per_call + 1 + (h->leafE.n ? 1 : 0);   // + k_set_xmap, + the E rows
    *out = h;
    return H2_OK;
#undef H2_TRY
#undef H2_TRYC
}

extern "C" int h2_create(const h2_desc *d, int nv_max, const void *nccl_unique_id, h2_handle *out)
{
    try {
        return create_impl(d, nv_max, nccl_unique_id, out);
    } catch (const std::exception &e) {
        if (out) *out = nullptr;
        return fail(H2_ERR_OOM, std::string("h2_create: ") + e.what());
    }
}

// ======================================================================== matvec
namespace {

// phase marker: records event `i` (0..NEV-1) of the current call when profiling is on
constexpr int NEV = 10;
int mark(h2_ctx *h, int i, cudaStream_t st)
{
    if (!h->prof) return H2_OK;
    int64_t idx = h->ev_used + i;
    while ((int64_t)h->ev_pool.size() <= idx) {
        cudaEvent_t e;
        H2_CUDA(h, cudaEventCreate(&e));
        h->ev_pool.push_back(e);
    }
    H2_CUDA(h, cudaEventRecord(h->ev_pool[idx], st));
    return H2_OK;
}
// phase -> (start marker, end marker) of a call (see enqueue); index H2_NPHASE = whole call
const int kPhaseSpan[H2_NPHASE + 1][2] = {{0, 1}, {2, 3}, {3, 4}, {4, 5}, {5, 6}, {6, 7},
                                          {8, 9}, {9, 9}, {1, 2}, {0, 9}};

// Enqueue one matvec for nv vectors on `st`; X, Y, alpha, beta come from the device CallArgs
// (written by k_set_args before), so the same sequence can be captured once as a CUDA graph.
// part: PART_ALL (NCCL or single rank), or for loopback groups PART_UP (everything before the
// exchange: x halo pack, leaf projection, leaf-level coupling, upsweep, x^ pack) and PART_DOWN
// (everything after it: top tree, couplings, downsweep, leaves), the group copying between them.
// Symmetric storage (one rank, nv = 1): the same phases with the coupling rows and the leaves
// applying every stored off-diagonal block also transposed (h2_sym.cuh), accumulating with atomics
// into a zeroed y^ and a beta-scaled Y.
template <typename T>
int enqueue_sym(h2_ctx *h, int nv, cudaStream_t st)
{
    T *xh = (T *)h->xh, *yh = (T *)h->yh;
    const CallArgs<T> *args = (const CallArgs<T> *)h->dargs;
    auto T0 = [&](const Phase &ph) { return h->d_tasks + ph.t0; };
    int rc;
#define H2_MARK(i) if ((rc = mark(h, i, st)) != H2_OK) return rc
    cudaStream_t s_leafc = h->prof ? st : h->s_leafc;
    H2_MARK(0);
    H2_CUDA(h, cudaMemsetAsync(yh, 0, (size_t)h->yh_plane * nv * sizeof(T), st));
    H2_CUDA(h, launch_up_leaf<T>(T0(h->up_leaf), h->up_leaf.n, h->d_blks, args, xh, h->xh_plane, nv,
                                 h->up_leaf.r, st));
    H2_MARK(1);
    H2_CUDA(h, cudaEventRecord(h->ev_upleaf, st));
    H2_CUDA(h, cudaStreamWaitEvent(s_leafc, h->ev_upleaf, 0));
    for (const Phase &ph : h->coup_leaf)
        H2_CUDA(h, launch_sym_rows<T>(T0(ph), ph.n, h->d_blks, xh, yh, ph.r, s_leafc));
    H2_CUDA(h, cudaEventRecord(h->ev_leafc, s_leafc));
    H2_MARK(2);
    for (size_t u = 0; u < h->up_sweeps.size(); ++u)
        H2_CUDA(h, launch_sweep<T>(MODE_WRITE, h->up_sweeps[u], h->up_sweep_ctas[u],
                                   h->up_sweep_thr[u], xh,
                                   h->xh_plane, nv, h->sweep_r_up, st));
    H2_MARK(3);
    H2_MARK(4);
    for (const Phase &ph : h->coup_diag)
        H2_CUDA(h, launch_sym_rows<T>(T0(ph), ph.n, h->d_blks, xh, yh, ph.r, st));
    H2_MARK(5);
    H2_MARK(6);
    for (size_t u = 0; u < h->dn_sweeps.size(); ++u)
        H2_CUDA(h, launch_sweep<T>(MODE_ACCUM, h->dn_sweeps[u], h->dn_sweep_ctas[u],
                                   h->dn_sweep_thr[u], yh,
                                   h->yh_plane, nv, h->sweep_r_dn, st));
    H2_MARK(7);
    H2_CUDA(h, cudaStreamWaitEvent(st, h->ev_leafc, 0));
    H2_CUDA(h, launch_beta<T>(args, h->n_local, nv, st));
    H2_MARK(8);
    H2_CUDA(h, launch_sym_leaf<T>(T0(h->leaf), T0(h->dense), h->leaf.n, h->d_blks, yh, args, h->leaf.r, st));
    H2_MARK(9);
    if (h->prof) h->ev_used += NEV;
#undef H2_MARK
    return H2_OK;
}

enum { PART_ALL = 0, PART_UP = 1, PART_DOWN = 2 };
template <typename T>
int enqueue(h2_ctx *h, int nv, cudaStream_t st, int part = PART_ALL)
{
    if (h->sym) return enqueue_sym<T>(h, nv, st);
    const Layout &L = h->L;
    const int q = L.q, C = L.C;
    T *xh = (T *)h->xh, *yh = (T *)h->yh;
    const CallArgs<T> *args = (const CallArgs<T> *)h->dargs;
    auto T0 = [&](const Phase &ph) { return h->d_tasks + ph.t0; };
    int rc;
#define H2_MARK(i) if ((rc = mark(h, i, st)) != H2_OK) return rc
    ncclDataType_t ty = nccl_type(h->dtype);
    const bool nccl = L.P > 1 && part == PART_ALL;
    // profiling (and loopback groups) serialize the side stream onto the main one so every
    // phase's events bracket only its own kernels (clean per-kernel durations for the roofline)
    // H2_SIDE_STREAM=0: the leaf coupling on the main stream too (A/B switch)
    static const bool side = [] { const char *e = getenv("H2_SIDE_STREAM"); return !(e && e[0] == '0'); }();
    cudaStream_t s_leafc = (h->prof || h->group || !side) ? st : h->s_leafc;
    // CTA-tile engine (FP64, nv >= cta_min_nv): the same tasks, one CTA per output node
    const bool cta = h->use_cta(nv);
    // (H2_CTA_SWEEPS=0: the warp sweeps even where the CTA-tile engine runs the rest -- A/B switch)
    static const bool cta_sweeps = [] { const char *e = getenv("H2_CTA_SWEEPS"); return !(e && e[0] == '0'); }();
    auto cjob = [&](const Phase &ph, int kind, int mode, const void *src, int64_t src_ld, void *dst,
                    int64_t dst_ld) {
        CtaJob j{};
        j.tasks = T0(ph);
        j.dtasks = nullptr;
        j.blks = h->d_blks;
        j.ntask = ph.n;
        j.kind = kind;
        j.mode = mode;
        j.src = (const double *)src;
        j.src_ld = src_ld;
        j.dst = (double *)dst;
        j.dst_ld = dst_ld;
        j.yh = (const double *)yh;
        j.yh_ld = h->yh_plane;
        j.halo = (const double *)h->hrecv;
        j.args = (const CallArgs<double> *)h->dargs;
        j.nv = nv;
        return j;
    };
    const bool umma = !cta && h->use_umma(nv);
    // one coupling-row launch on the engine of this nv (CTA-tile FP64 / tcgen05 FP32 / warp tasks)
    auto rows = [&](int mode, const Phase &ph, const void *src, int64_t src_ld, void *dst, int64_t dst_ld,
                    cudaStream_t s) -> cudaError_t {
        if (cta) return launch_cta(cjob(ph, CK_ROWS, mode, src, src_ld, dst, dst_ld), ph.r, h->nsm, s);
        if (umma)
            return launch_umma_rows(mode, T0(ph), ph.n, h->d_blks, (const float *)src, src_ld, (float *)dst, dst_ld,
                                    nv, h->nsm, s);
        return launch_rows<T>(mode, T0(ph), ph.n, h->d_blks, (const T *)src, src_ld, (T *)dst, dst_ld, nv, ph.r, s);
    };
    const bool p2p = nccl && h->p2p;
    auto offdiag = [&](const Phase *grp, cudaStream_t s) -> int {     // off-diagonal rows from xrecv
        for (int ci = 0; ci < 3; ++ci) {
            H2_CUDA(h, rows(MODE_ACCUM, grp[ci], h->xrecv, 0, yh, h->yh_plane, s));
        }
        return H2_OK;
    };
    if (part != PART_DOWN) {
    H2_MARK(0);
    // 0. x-leaf halo for the off-process dense blocks (P > 1): X is an input, so the exchange
    //    starts at t = 0 on the comm stream
    if (p2p) {
        // device-initiated exchange (NEXT-1): wait until the peers are done with my previous
        // call's data, pack my x rows, flag them; the comm stream pulls the peers' rows over
        // NVLink (IPC mappings) as soon as their flags arrive and acknowledges
        H2_CUDA(h, launch_p2p_begin(h->sig, h->d_begin_waits, h->n_begin_waits, st));
        H2_CUDA(h, launch_pack<T>(h->d_segs + h->seg_h0, h->nseg_h, (const T *)nullptr, 0, args, (T *)h->hsend, nv, st));
        H2_CUDA(h, launch_p2p_signal(h->sig, h->d_tgt_h, h->n_tgt_h, st));
        H2_CUDA(h, cudaEventRecord(h->ev_fork, st));
        H2_CUDA(h, cudaStreamWaitEvent(h->s_comm, h->ev_fork, 0));
        H2_CUDA(h, launch_p2p_wait(h->sig, h->d_wait_h, h->n_wait_h, h->s_comm));
        for (const auto &pr : h->peers)
            if (pr.hr_cnt)
                H2_CUDA(h, cudaMemcpyAsync((T *)h->hrecv + pr.hr_off, (const T *)h->pmap[pr.rank].hsend + h->pmap[pr.rank].hs_off,
                                           (size_t)pr.hr_cnt * nv * sizeof(T), cudaMemcpyDeviceToDevice, h->s_comm));
        H2_CUDA(h, launch_p2p_signal(h->sig, h->d_tgt_ch, h->n_tgt_ch, h->s_comm));
        H2_CUDA(h, cudaEventRecord(h->ev_halo, h->s_comm));
    } else if (nccl) {
        H2_CUDA(h, cudaEventRecord(h->ev_fork, st));
        H2_CUDA(h, cudaStreamWaitEvent(h->s_comm, h->ev_fork, 0));
        H2_CUDA(h, launch_pack<T>(h->d_segs + h->seg_h0, h->nseg_h, (const T *)nullptr, 0, args, (T *)h->hsend, nv, h->s_comm));
        H2_NCCL(h, g_nccl.GroupStart());
        for (const auto &pr : h->peers) {
            if (pr.hs_cnt) H2_NCCL(h, g_nccl.Send((T *)h->hsend + pr.hs_off, pr.hs_cnt * nv, ty, pr.rank, h->comm, h->s_comm));
            if (pr.hr_cnt) H2_NCCL(h, g_nccl.Recv((T *)h->hrecv + pr.hr_off, pr.hr_cnt * nv, ty, pr.rank, h->comm, h->s_comm));
        }
        H2_NCCL(h, g_nccl.GroupEnd());
        H2_CUDA(h, cudaEventRecord(h->ev_halo, h->s_comm));
    } else if (L.P > 1) {
        H2_CUDA(h, launch_pack<T>(h->d_segs + h->seg_h0, h->nseg_h, (const T *)nullptr, 0, args, (T *)h->hsend, nv, st));
    }
    // 1. leaf projection (alg:upsweep2 line 3)
    if (cta)
        H2_CUDA(h, launch_cta(cjob(h->up_leaf, CK_UPLEAF, MODE_WRITE, nullptr, 0, xh, h->xh_plane), h->up_leaf.r,
                              h->nsm, st));
    else
        H2_CUDA(h, launch_up_leaf<T>(T0(h->up_leaf), h->up_leaf.n, h->d_blks, args, xh, h->xh_plane, nv,
                                     h->up_leaf.r, st));
    if (p2p) H2_CUDA(h, launch_p2p_signal(h->sig, h->d_tgt_xl, h->n_tgt_xl, st));   // leaf-level x^ ready
    H2_MARK(1);
    // 1b. leaf-level coupling (diagonal part) as soon as x^ of the leaves exists (alg:mult's
    //     levels are independent), on its own stream
    H2_CUDA(h, cudaEventRecord(h->ev_upleaf, st));
    H2_CUDA(h, cudaStreamWaitEvent(s_leafc, h->ev_upleaf, 0));
    // the comm stream pulls the peers' x^ nodes I need into my receive chunks as their flags
    // arrive, overlapped with my upsweep and diagonal coupling; ev_upleaf also orders it after my
    // previous call's off-diagonal reads of those chunks.  Every wait is enqueued (host order)
    // after my own signals that it transitively depends on: streams may share a hardware queue,
    // so a spinning wait must never sit ahead of a signal its peers are waiting for.
    auto pull = [&](int g) -> int {
        H2_CUDA(h, launch_p2p_wait(h->sig, g == 0 ? h->d_wait_xl : h->d_wait_xu, g == 0 ? h->n_wait_xl : h->n_wait_xu,
                                   h->s_comm));
        for (const auto &pl : h->pulls)
            if (pl.group == g)
                H2_CUDA(h, launch_pack<T>(h->d_segs + pl.seg0, pl.nseg, (const T *)h->pmap[pl.owner].xh, h->xh_plane,
                                          args, (T *)h->xrecv, nv, h->s_comm));
        return H2_OK;
    };
    if (p2p && !h->p2p_direct) {
        H2_CUDA(h, cudaStreamWaitEvent(h->s_comm, h->ev_upleaf, 0));
        if ((rc = pull(0)) != H2_OK) return rc;          // leaf level: after my "leaf x^ ready" signal
    }
    for (const Phase &ph : h->coup_leaf) H2_CUDA(h, rows(MODE_WRITE, ph, xh, h->xh_plane, yh, h->yh_plane, s_leafc));
    H2_CUDA(h, cudaEventRecord(h->ev_leafc, s_leafc));
    if (p2p && !h->p2p_direct) {
        // the leaf-level off-diagonal blocks as soon as their x^ is pulled (most of the
        // off-diagonal work), after the leaf-level diagonal coupling wrote those rows
        H2_CUDA(h, cudaStreamWaitEvent(h->s_comm, h->ev_leafc, 0));
        if ((rc = offdiag(h->coup_off_leaf, h->s_comm)) != H2_OK) return rc;
    }
    H2_MARK(2);
    // 1c. upsweep transfers of the local branch
    if (cta && (cta_sweeps || !h->use_sweep)) {
        for (const Phase &ph : h->up_lv)
            H2_CUDA(h, launch_cta(cjob(ph, CK_ROWS, MODE_WRITE, xh, h->xh_plane, xh, h->xh_plane), ph.r, h->nsm, st));
    } else if (h->use_sweep) {
        for (size_t u = 0; u < h->up_sweeps.size(); ++u)
            H2_CUDA(h, launch_sweep<T>(MODE_WRITE, h->up_sweeps[u], h->up_sweep_ctas[u],
                                       h->up_sweep_thr[u],
                                       xh, h->xh_plane, nv, h->sweep_r_up, st));
    } else {
        for (const auto &sg : h->up_stages)
            H2_CUDA(h, launch_tree<T>(MODE_WRITE, sg.st, sg.nctas, h->d_tasks, h->d_blks, xh, h->xh_plane, nv,
                                      sg.r, st));
    }
    H2_MARK(3);
    if (p2p) H2_CUDA(h, launch_p2p_signal(h->sig, h->d_tgt_xu, h->n_tgt_xu, st));   // upper-level x^ ready
    if (p2p && !h->p2p_direct) {                          // upper levels: after my "upper x^ ready"
        if ((rc = pull(1)) != H2_OK) return rc;
        H2_CUDA(h, launch_p2p_signal(h->sig, h->d_tgt_cx, h->n_tgt_cx, h->s_comm));
        H2_CUDA(h, cudaEventRecord(h->ev_recv, h->s_comm));
    }
    // 2. exchange (P > 1): pack my x^ nodes that peers need, one NCCL group on the comm stream,
    //    overlapped with the diagonal multiply (alg:optimized_dist_mult); the device-initiated
    //    exchange needs no pack: peers read my x^ plane directly
    if (L.P > 1 && !p2p)
        H2_CUDA(h, launch_pack<T>(h->d_segs + h->seg_x0, h->nseg_x, xh, h->xh_plane, args, (T *)h->xsend, nv, st));
    if (nccl && !p2p) {
        H2_CUDA(h, cudaEventRecord(h->ev_packed, st));
        H2_CUDA(h, cudaStreamWaitEvent(h->s_comm, h->ev_packed, 0));
        H2_NCCL(h, g_nccl.GroupStart());
        for (const auto &pr : h->peers) {
            if (pr.xs_cnt) H2_NCCL(h, g_nccl.Send((T *)h->xsend + pr.xs_off, pr.xs_cnt * nv, ty, pr.rank, h->comm, h->s_comm));
            if (pr.xr_cnt) H2_NCCL(h, g_nccl.Recv((T *)h->xrecv + pr.xr_off, pr.xr_cnt * nv, ty, pr.rank, h->comm, h->s_comm));
        }
        H2_NCCL(h, g_nccl.GroupEnd());
        H2_CUDA(h, cudaEventRecord(h->ev_recv, h->s_comm));
    }
    if (part == PART_UP) return H2_OK;
    }
    // replicated top tree: gather the branch roots, upsweep the top
    if (h->has_top) {
        const int kC = L.k[C];
        if (p2p) {
            // every rank's branch root, read from the peers' x^ planes once they are complete
            H2_CUDA(h, launch_p2p_wait(h->sig, h->d_wait_xu, h->n_wait_xu, st));
            for (int o = 0; o < L.P; ++o) {
                const T *src = (o == L.p ? xh : (const T *)h->pmap[o].xh) + h->xh_base[C];
                H2_CUDA(h, cudaMemcpy2DAsync(xh + h->xgather + (int64_t)o * kC, (size_t)h->xh_plane * sizeof(T), src,
                                             (size_t)h->xh_plane * sizeof(T), (size_t)kC * sizeof(T), nv,
                                             cudaMemcpyDeviceToDevice, st));
            }
        } else if (nccl) {
            // own root -> gather slot p, then allgather in place over the P slots of every plane
            for (int n = 0; n < nv; ++n) {
                T *g = xh + h->xgather + (int64_t)n * h->xh_plane;
                H2_CUDA(h, cudaMemcpyAsync(g + (int64_t)L.p * kC, xh + h->xh_base[C] + (int64_t)n * h->xh_plane,
                                           kC * sizeof(T), cudaMemcpyDeviceToDevice, st));
                H2_NCCL(h, g_nccl.AllGather(g + (int64_t)L.p * kC, g, kC, ty, h->comm, st));
            }
        }
        for (const auto &sg : h->top_stages)
            H2_CUDA(h, launch_tree<T>(MODE_WRITE, sg.st, sg.nctas, h->d_tasks, h->d_blks, xh, h->xh_plane,
                                      nv, sg.r, st));
    }
    H2_MARK(4);
    // 3. coupling multiply, diagonal part of the levels above the leaves (alg:mult)
    for (const Phase &ph : h->coup_diag) H2_CUDA(h, rows(MODE_WRITE, ph, xh, h->xh_plane, yh, h->yh_plane, st));
    H2_MARK(5);
    // 4. off-diagonal part after the exchange (waitAll, alg:optimized_dist_mult line 11-12);
    //    it accumulates into leaf-level rows too, so the leaf coupling stream joins first
    if (p2p && h->p2p_direct) {
        // off-diagonal blocks read the owners' x^ planes directly (NVLink): leaf level first
        // (flagged right after the owners' leaf projection), then the upper levels
        H2_CUDA(h, cudaStreamWaitEvent(st, h->ev_leafc, 0));
        for (int g = 0; g < 2; ++g) {
            H2_CUDA(h, launch_p2p_wait(h->sig, g == 0 ? h->d_wait_xl : h->d_wait_xu, g == 0 ? h->n_wait_xl : h->n_wait_xu, st));
            for (const auto &pp : h->p2p_phases) {
                if (pp.group != g) continue;
                H2_CUDA(h, rows(MODE_ACCUM, pp.ph, h->pmap[pp.owner].xh, h->xh_plane, yh, h->yh_plane, st));
            }
        }
        H2_CUDA(h, launch_p2p_signal(h->sig, h->d_tgt_cx, h->n_tgt_cx, st));
    } else if (L.P > 1) {
        H2_CUDA(h, cudaStreamWaitEvent(st, h->ev_leafc, 0));
        if (nccl) H2_CUDA(h, cudaStreamWaitEvent(st, h->ev_recv, 0));     // NCCL receive or p2p pulls
        // the leaf-level group already ran on the comm stream in the p2p pull mode
        if (!(p2p && !h->p2p_direct) && (rc = offdiag(h->coup_off_leaf, st)) != H2_OK) return rc;
        if ((rc = offdiag(h->coup_off, st)) != H2_OK) return rc;
    }
    H2_MARK(6);
    // 5. downsweep transfers (alg:downsweep)
    if (cta && (cta_sweeps || !h->use_sweep)) {
        for (const Phase &ph : h->down_lv)
            H2_CUDA(h, launch_cta(cjob(ph, CK_ROWS, MODE_ACCUM, yh, h->yh_plane, yh, h->yh_plane), ph.r, h->nsm, st));
    } else if (h->use_sweep) {
        for (size_t u = 0; u < h->dn_sweeps.size(); ++u)
            H2_CUDA(h, launch_sweep<T>(MODE_ACCUM, h->dn_sweeps[u], h->dn_sweep_ctas[u],
                                       h->dn_sweep_thr[u],
                                       yh, h->yh_plane, nv, h->sweep_r_dn, st));
    } else {
        for (const auto &sg : h->down_stages)
            H2_CUDA(h, launch_tree<T>(MODE_ACCUM, sg.st, sg.nctas, h->d_tasks, h->d_blks, yh, h->yh_plane, nv,
                                      sg.r, st));
    }
    H2_MARK(7);
    // 6. leaves: last transfer + U expansion + dense near field + epilogue in one kernel (Y
    //    written once, reading R11/R18), after the side streams joined
    if (nccl) H2_CUDA(h, cudaStreamWaitEvent(st, h->ev_halo, 0));   // the kernel reads the x halo
    H2_CUDA(h, cudaStreamWaitEvent(st, h->ev_leafc, 0));
    H2_MARK(8);
    const int kq = L.k[q], kp = q >= 1 ? L.k[q - 1] : 1;
    if (cta) {
        CtaJob j = cjob(h->leaf, CK_LEAF, MODE_WRITE, nullptr, 0, nullptr, 0);
        j.dtasks = T0(h->dense);
        H2_CUDA(h, launch_cta(j, std::max(h->leaf.r, kq), h->nsm, st));
    } else if (h->use_umma_leaf(nv)) {
        // FP32 on tcgen05: y^_t += E_t y^_p as rows, then U y^_t + dense row with the X tensor map
        if (h->leafE.n) H2_CUDA(h, rows(MODE_ACCUM, h->leafE, yh, h->yh_plane, yh, h->yh_plane, st));
        H2_CUDA(h, launch_umma_leaf(T0(h->leaf), T0(h->dense), h->leaf.n, h->d_blks, (const float *)yh, h->yh_plane,
                                    (const CallArgs<float> *)h->dargs, (const float *)h->hrecv, h->d_xmap, nv,
                                    h->nsm, st));
    } else {
        H2_CUDA(h, launch_leaf_dense<T>(T0(h->leaf), T0(h->dense), h->leaf.n, h->d_blks, yh, h->yh_plane, args,
                                        (const T *)h->hrecv, nv, kq, kp, h->leaf.r, st));
    }
    H2_MARK(9);
    if (h->prof) h->ev_used += NEV;
#undef H2_MARK
    return H2_OK;
}

// Loopback group exchange (tests): every member's x^ / x-halo send chunk for peer o is copied
// into o's receive chunk from it, and the branch roots of level C into every member's gather
// region -- the same bytes the NCCL groups move.  All on one stream, between PART_UP and
// PART_DOWN of every member.
int group_exchange(h2_group *g, int nv, cudaStream_t st)
{
    for (h2_ctx *h : g->members) {
        const size_t esz = h->esz;
        for (const auto &pr : h->peers) {
            h2_ctx *o = g->members[pr.rank];
            const h2_ctx::Peer *back = nullptr;
            for (const auto &q : o->peers)
                if (q.rank == h->L.p) back = &q;
            if (!back) return fail(H2_ERR_STATE, "loopback group: asymmetric peer lists");
            if (pr.xs_cnt != back->xr_cnt || pr.hs_cnt != back->hr_cnt)
                return fail(H2_ERR_STATE, "loopback group: send / receive counts disagree");
            if (pr.xs_cnt)
                H2_CUDA(h, cudaMemcpyAsync((char *)o->xrecv + back->xr_off * esz, (char *)h->xsend + pr.xs_off * esz,
                                           (size_t)pr.xs_cnt * nv * esz, cudaMemcpyDeviceToDevice, st));
            if (pr.hs_cnt)
                H2_CUDA(h, cudaMemcpyAsync((char *)o->hrecv + back->hr_off * esz, (char *)h->hsend + pr.hs_off * esz,
                                           (size_t)pr.hs_cnt * nv * esz, cudaMemcpyDeviceToDevice, st));
        }
        if (h->has_top) {
            const int C = h->L.C, kC = h->L.k[C];
            for (h2_ctx *o : g->members)
                H2_CUDA(h, cudaMemcpy2DAsync((char *)h->xh + (h->xgather + (int64_t)o->L.p * kC) * esz,
                                             (size_t)h->xh_plane * esz, (char *)o->xh + o->xh_base[C] * esz,
                                             (size_t)o->xh_plane * esz, (size_t)kC * esz, nv,
                                             cudaMemcpyDeviceToDevice, st));
        }
    }
    return H2_OK;
}

template <typename T>
int run_matvec(h2_ctx *h, T alpha, const T *X, int64_t ldx, T beta, T *Y, int64_t ldy, int nv)
{
    cudaStream_t st = h->stream;
    if (h->last_stream_set && h->last_stream != st)       // the args slot is stream-ordered
        H2_CUDA(h, cudaStreamSynchronize(h->last_stream));
    h->last_stream = st;
    h->last_stream_set = true;
    if (alpha == T(0)) {
        H2_CUDA(h, launch_scale<T>(Y, ldy, h->n_local, nv, beta, st));
        return H2_OK;
    }
    H2_DBG("rank %d: matvec nv=%d warm=%d graph=%d", h->L.p, nv, (int)h->warm[nv], (int)(h->graph[nv] != nullptr));
    H2_CUDA(h, launch_set_args<T>((CallArgs<T> *)h->dargs, X, ldx, Y, ldy, alpha, beta, st));
    if (h->use_umma_leaf(nv)) H2_CUDA(h, launch_set_xmap(h->d_xmap, (const float *)X, ldx, nv, st));
    if (h->prof || !h->warm[nv]) {
        h->warm[nv] = true;            // first call per nv runs eagerly (sets kernel attributes)
        return enqueue<T>(h, nv, st);
    }
    cudaGraphExec_t &ex = h->graph[nv];
    if (!ex) {
        // capture the whole matvec once per nv on a private stream (PAPER.md:298's "fast static
        // scheduler" becomes one graph launch per call)
        cudaGraph_t g = nullptr;
        H2_CUDA(h, cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue<T>(h, nv, h->cap_stream);
        cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
        if (rc != H2_OK) { if (g) cudaGraphDestroy(g); return rc; }
        if (e != cudaSuccess) return cuda_fail(h, e, "cudaStreamEndCapture");
        e = cudaGraphInstantiate(&ex, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) { ex = nullptr; return cuda_fail(h, e, "cudaGraphInstantiate"); }
    }
    H2_CUDA(h, cudaGraphLaunch(ex, st));
    return H2_OK;
}

int check_call(h2_ctx *h, int nv)
{
    if (!h) return fail(H2_ERR_ARG, "handle is NULL");
    if (h->sticky) return fail(H2_ERR_STATE, "handle unusable after an earlier CUDA/NCCL error");
    if (nv < 1 || nv > h->nv_max) return fail(H2_ERR_ARG, "nv must be in [1, nv_max]");
    return H2_OK;
}

}  // namespace

extern "C" int h2_matvec_ld(h2_handle h, double alpha, const void *X, int64_t ldx, double beta,
                            void *Y, int64_t ldy, int nv)
{
    int rc = check_call(h, nv);
    if (rc != H2_OK) return rc;
    if (h->group) return fail(H2_ERR_STATE, "handle belongs to a loopback group: use h2_group_matvec");
    if (!X || !Y) return fail(H2_ERR_ARG, "X or Y is NULL");
    if (ldx < h->n_local || ldy < h->n_local) return fail(H2_ERR_SHAPE, "ld < n_local");
    if (h->dtype == H2_F64)
        return run_matvec<double>(h, alpha, (const double *)X, ldx, beta, (double *)Y, ldy, nv);
    return run_matvec<float>(h, (float)alpha, (const float *)X, ldx, (float)beta, (float *)Y, ldy, nv);
}

extern "C" int h2_matvec(h2_handle h, double alpha, const void *X, double beta, void *Y, int nv)
{
    if (!h) return fail(H2_ERR_ARG, "handle is NULL");
    return h2_matvec_ld(h, alpha, X, h->n_local, beta, Y, h->n_local, nv);
}

extern "C" int h2_matvec_host(h2_handle h, double alpha, const void *X, double beta, void *Y, int nv)
{
    int rc = check_call(h, nv);
    if (rc != H2_OK) return rc;
    if (!X || !Y) return fail(H2_ERR_ARG, "X or Y is NULL");
    size_t bytes = (size_t)h->n_local * nv * h->esz;
    if (!h->dX) {
        cudaError_t err;
        h->dX = dalloc(h, (size_t)h->n_local * h->nv_max * h->esz, err);
        h->dY = dalloc(h, (size_t)h->n_local * h->nv_max * h->esz, err);
        if (!h->dX || !h->dY) return cuda_fail(h, err, "cudaMalloc(e2e staging)");
    }
    // Large calls (>= 16 vectors and >= 32 MB each way) run in two vector chunks so the
    // host-to-device copy of chunk 1 overlaps the matvec of chunk 0 and the device-to-host copy of
    // chunk 0 overlaps the matvec of chunk 1 (copy engines on their own streams, event-ordered);
    // chunk sizes multiples of 8 (the FP32 tensor-map path).  Smaller calls: copy, matvec, copy.
    const char *emb = getenv("H2_E2E_MIN_MB");          // threshold override (tests)
    const size_t min_bytes = (size_t)(emb ? atol(emb) : 32) << 20;
    const int nc = (nv >= 16 && bytes >= min_bytes) ? 2 : 1;
    if (nc == 1) {
        H2_CUDA(h, cudaMemcpyAsync(h->dX, X, bytes, cudaMemcpyHostToDevice, h->stream));
        if (beta != 0.0) H2_CUDA(h, cudaMemcpyAsync(h->dY, Y, bytes, cudaMemcpyHostToDevice, h->stream));
        rc = h2_matvec_ld(h, alpha, h->dX, h->n_local, beta, h->dY, h->n_local, nv);
        if (rc != H2_OK) return rc;
        H2_CUDA(h, cudaMemcpyAsync(Y, h->dY, bytes, cudaMemcpyDeviceToHost, h->stream));
        H2_CUDA(h, cudaStreamSynchronize(h->stream));
        return H2_OK;
    }
    if (!h->s_h2d) {
        H2_CUDA(h, cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
        H2_CUDA(h, cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            H2_CUDA(h, cudaEventCreateWithFlags(&h->ev_x[i], cudaEventDisableTiming));
            H2_CUDA(h, cudaEventCreateWithFlags(&h->ev_y[i], cudaEventDisableTiming));
        }
    }
    const int v0 = ((nv / 2 + 7) / 8) * 8;                 // first chunk: half, rounded up to 8
    const int cv[2] = {0, v0}, cn[2] = {v0, nv - v0};
    const size_t vb = (size_t)h->n_local * h->esz;         // bytes per vector
    // the copy streams start after whatever the handle's stream has queued (dX / dY reuse)
    H2_CUDA(h, cudaEventRecord(h->ev_y[1], h->stream));
    H2_CUDA(h, cudaStreamWaitEvent(h->s_h2d, h->ev_y[1], 0));
    for (int c = 0; c < 2; ++c) {
        const size_t off = (size_t)cv[c] * vb, cb = (size_t)cn[c] * vb;
        H2_CUDA(h, cudaMemcpyAsync((char *)h->dX + off, (const char *)X + off, cb, cudaMemcpyHostToDevice, h->s_h2d));
        if (beta != 0.0)
            H2_CUDA(h, cudaMemcpyAsync((char *)h->dY + off, (const char *)Y + off, cb, cudaMemcpyHostToDevice,
                                       h->s_h2d));
        H2_CUDA(h, cudaEventRecord(h->ev_x[c], h->s_h2d));
    }
    for (int c = 0; c < 2; ++c) {
        const size_t off = (size_t)cv[c] * vb, cb = (size_t)cn[c] * vb;
        H2_CUDA(h, cudaStreamWaitEvent(h->stream, h->ev_x[c], 0));
        rc = h2_matvec_ld(h, alpha, (const char *)h->dX + off, h->n_local, beta, (char *)h->dY + off, h->n_local,
                          cn[c]);
        if (rc != H2_OK) return rc;
        H2_CUDA(h, cudaEventRecord(h->ev_y[c], h->stream));
        H2_CUDA(h, cudaStreamWaitEvent(h->s_d2h, h->ev_y[c], 0));
        H2_CUDA(h, cudaMemcpyAsync((char *)Y + off, (const char *)h->dY + off, cb, cudaMemcpyDeviceToHost, h->s_d2h));
    }
    H2_CUDA(h, cudaStreamSynchronize(h->s_d2h));
    H2_CUDA(h, cudaStreamSynchronize(h->stream));
    return H2_OK;
}

// ======================================================================== loopback groups
extern "C" int h2_group_create(const h2_desc *const *descs, int P, int nv_max, h2_handle *out)
{
    if (!descs || !out || P < 1) return fail(H2_ERR_ARG, "bad argument");
    for (int o = 0; o < P; ++o) out[o] = nullptr;
    try {
        h2_group *g = new h2_group();
        g->descs.assign(descs, descs + P);
        g->layouts.resize(P);
        g->needs.resize(P);
        for (int o = 0; o < P; ++o) {
            int rc = validate(descs[o], nv_max, g->layouts[o]);
            if (rc == H2_OK && (descs[o]->nranks != P || descs[o]->rank != o))
                rc = fail(H2_ERR_ARG, "group member o must describe rank o of nranks = P");
            if (rc != H2_OK) { delete g; return rc; }
            remote_needs(descs[o], g->layouts[o], g->needs[o]);
        }
        g->members.assign(P, nullptr);
        LoopSetup ls;
        ls.g = g;
        for (int o = 0; o < P; ++o) {
            h2_handle h = nullptr;
            int rc = create_impl(descs[o], nv_max, nullptr, &h, &ls, g);
            if (rc != H2_OK) {
                std::string msg = g_err;
                int live = 0;
                for (int u = 0; u < o; ++u) live += g->members[u] != nullptr;
                for (int u = 0; u < o; ++u) { h2_ctx *m = g->members[u]; if (m) release(m); }
                if (!live) delete g;
                for (int u = 0; u < P; ++u) out[u] = nullptr;
                g_err = msg;
                return rc;
            }
            g->members[o] = h;
            out[o] = h;
        }
        return H2_OK;
    } catch (const std::exception &e) {
        return fail(H2_ERR_OOM, std::string("h2_group_create: ") + e.what());
    }
}

namespace {
template <typename T>
int group_matvec(h2_ctx *const *hs, int P, T alpha, const void *const *X, T beta, void *const *Y, int nv)
{
    h2_group *g = hs[0]->group;
    cudaStream_t st = hs[0]->stream;
    for (int o = 0; o < P; ++o) {
        h2_ctx *h = hs[o];
        if (alpha == T(0)) {
            H2_CUDA(h, launch_scale<T>((T *)Y[o], h->n_local, h->n_local, nv, beta, st));
            continue;
        }
        H2_CUDA(h, launch_set_args<T>((CallArgs<T> *)h->dargs, (const T *)X[o], h->n_local, (T *)Y[o], h->n_local,
                                      alpha, beta, st));
        if (h->use_umma_leaf(nv)) H2_CUDA(h, launch_set_xmap(h->d_xmap, (const float *)X[o], h->n_local, nv, st));
        int rc = enqueue<T>(h, nv, st, PART_UP);
        if (rc != H2_OK) return rc;
    }
    if (alpha == T(0)) return H2_OK;
    int rc = group_exchange(g, nv, st);
    if (rc != H2_OK) return rc;
    for (int o = 0; o < P; ++o) {
        rc = enqueue<T>(hs[o], nv, st, PART_DOWN);
        if (rc != H2_OK) return rc;
    }
    return H2_OK;
}
}  // namespace

extern "C" int h2_group_matvec(const h2_handle *hs, int P, double alpha, const void *const *X, double beta,
                               void *const *Y, int nv)
{
    if (!hs || !X || !Y || P < 1) return fail(H2_ERR_ARG, "bad argument");
    h2_group *g = hs[0] ? hs[0]->group : nullptr;
    if (!g || (int)g->members.size() != P) return fail(H2_ERR_ARG, "handles are not one complete loopback group");
    for (int o = 0; o < P; ++o) {
        if (hs[o] != g->members[o]) return fail(H2_ERR_ARG, "handles must be the group's members in rank order");
        int rc = check_call(hs[o], nv);
        if (rc != H2_OK) return rc;
        if (!X[o] || !Y[o]) return fail(H2_ERR_ARG, "X or Y is NULL");
        hs[o]->prof = false;
    }
    if (hs[0]->dtype == H2_F64) return group_matvec<double>(hs, P, alpha, X, beta, Y, nv);
    return group_matvec<float>(hs, P, (float)alpha, X, (float)beta, Y, nv);
}

extern "C" int h2_set_stream(h2_handle h, void *stream)
{
    if (!h) return fail(H2_ERR_ARG, "handle is NULL");
    h->stream = (cudaStream_t)stream;
    return H2_OK;
}

extern "C" int h2_stats(h2_handle h, int nv, double *flops, double *bytes, double *xchg_bytes,
                        int *launches)
{
    if (!h) return fail(H2_ERR_ARG, "handle is NULL");
    if (nv < 1) return fail(H2_ERR_ARG, "nv < 1");
    const Layout &L = h->L;
    double tree = 0;
    for (int l = 0; l <= L.q; ++l) tree += (double)L.held(l) * L.k[l];
    if (flops) *flops = 2.0 * nv * h->ops_local;
    // operator once + X read + Y write + x^, y^ trees written and read once each
    if (bytes) *bytes = (double)h->esz * (h->ops_stored + nv * (2.0 * h->n_local + 4.0 * tree));
    if (xchg_bytes) {
        double x = 0;
        for (const auto &pr : h->peers) x += (double)(pr.xr_cnt + pr.hr_cnt) * nv * h->esz;
        *xchg_bytes = x;
    }
    if (launches) *launches = h->use_cta(nv) ? h->launches_cta : (h->use_umma_leaf(nv) ? h->launches_umma : h->launches_per_call);
    return H2_OK;
}

extern "C" int h2_set_profiling(h2_handle h, int on)
{
    if (!h) return fail(H2_ERR_ARG, "handle is NULL");
    h->prof = on != 0;
    return H2_OK;
}

extern "C" int h2_phase_times(h2_handle h, double ms[H2_NPHASE + 1], int64_t *ncalls)
{
    if (!h || !ms) return fail(H2_ERR_ARG, "NULL argument");
    for (int i = 0; i <= H2_NPHASE; ++i) ms[i] = 0;
    int64_t calls = h->ev_used / NEV;
    if (calls) {
        H2_CUDA(h, cudaDeviceSynchronize());
        for (int64_t c = 0; c < calls; ++c) {
            cudaEvent_t *e = &h->ev_pool[c * NEV];
            for (int i = 0; i <= H2_NPHASE; ++i) {
                float t = 0;
                H2_CUDA(h, cudaEventElapsedTime(&t, e[kPhaseSpan[i][0]], e[kPhaseSpan[i][1]]));
                ms[i] += t;
            }
        }
        for (int i = 0; i <= H2_NPHASE; ++i) ms[i] /= (double)calls;
    }
    if (ncalls) *ncalls = calls;
    h->ev_used = 0;
    return H2_OK;
}

extern "C" int h2_phase_stats(h2_handle h, int nv, double bytes[H2_NPHASE + 1], double flops[H2_NPHASE + 1])
{
    if (!h || nv < 1) return fail(H2_ERR_ARG, "bad argument");
    double tb = 0, tf = 0;
    double ops[H2_NPHASE], vec[H2_NPHASE];
    for (int i = 0; i < H2_NPHASE; ++i) { ops[i] = h->ph_ops[i]; vec[i] = h->ph_vec[i]; }
    // fused leaf + dense kernel: one phase (6), Y written once
    ops[6] += ops[7];
    vec[6] += vec[7] - 2.0 * h->n_local;    // Y read+write of a separate U pass replaced by one write
    ops[7] = vec[7] = 0;
    for (int i = 0; i < H2_NPHASE; ++i) {
        double b = (double)h->esz * (ops[i] + nv * vec[i]);
        double f = 2.0 * nv * ops[i];
        if (bytes) bytes[i] = b;
        if (flops) flops[i] = f;
        tb += b; tf += f;
    }
    if (bytes) bytes[H2_NPHASE] = tb;
    if (flops) flops[H2_NPHASE] = tf;
    return H2_OK;
}

extern "C" int h2_plan_census(const h2_desc *d, int level, int64_t *pid, int64_t *nodes_ptr,
                              int64_t *nodes, int64_t *npid, int64_t *nnodes)
{
    try {
        Layout L;
        int rc = validate(d, 1, L);
        if (rc != H2_OK) return rc;
        if (level < -1 || level > L.q) return fail(H2_ERR_ARG, "level out of range [-1, q]");
        if (!npid || !nnodes) return fail(H2_ERR_ARG, "npid / nnodes is NULL");
        RemoteNeeds rn;
        remote_needs(d, L, rn);
        int64_t np = 0, nn = 0;
        if (nodes_ptr) nodes_ptr[0] = 0;
        for (int o = 0; o < L.P; ++o) {
            std::vector<int64_t> v;
            if (level < 0) {
                if (rn.need_h.count(o)) v = rn.need_h[o];
            } else if (rn.need_x.count(o)) {
                for (int64_t key : rn.need_x[o])
                    if (key_level(key) == level) v.push_back(key_node(key));
            }
            if (v.empty()) continue;
            if (pid) pid[np] = o;
            for (int64_t g : v) {
                if (nodes) nodes[nn] = g;
                ++nn;
            }
            ++np;
            if (nodes_ptr) nodes_ptr[np] = nn;
        }
        *npid = np;
        *nnodes = nn;
        return H2_OK;
    } catch (const std::exception &e) {
        return fail(H2_ERR_OOM, std::string("h2_plan_census: ") + e.what());
    }
}

extern "C" int h2_n_local(h2_handle h, int64_t *n_local)
{
    if (!h || !n_local) return fail(H2_ERR_ARG, "NULL argument");
    *n_local = h->n_local;
    return H2_OK;
}

extern "C" int h2_plan_counts(h2_handle h, int64_t counts[8])
{
    if (!h || !counts) return fail(H2_ERR_ARG, "NULL argument");
    memcpy(counts, h->counts, sizeof(h->counts));
    return H2_OK;
}

extern "C" int h2_orthogonalize(h2_handle h)
{
    if (!h) return fail(H2_ERR_ARG, "handle is NULL");
    if (h->sticky) return fail(H2_ERR_STATE, "handle unusable after an earlier CUDA/NCCL error");
    if (h->L.P != 1 || h->dtype != H2_F64 || h->sym || h->group || (int)h->orth_pairs.size() != h->L.q + 1)
        return fail(H2_ERR_ARG, "h2_orthogonalize: FP64, one GPU, full (non-symmetric) storage only");
    const int q = h->L.q;
    std::vector<const int2 *> pairs(q + 1, nullptr);
    std::vector<int2 *> owned;
    std::vector<int64_t> nblk(q + 1, 0);
    std::vector<double *> E(q + 1, nullptr), Ft(q + 1, nullptr), S(q + 1, nullptr);
    cudaError_t err = cudaStreamSynchronize(h->stream);
    for (int l = 0; l <= q && err == cudaSuccess; ++l) {
        nblk[l] = (int64_t)h->orth_pairs[l].size();
        E[l] = (double *)h->E[l];
        Ft[l] = (double *)h->Ft[l];
        S[l] = (double *)h->S[l];
        if (!nblk[l]) continue;
        int2 *d = nullptr;
        err = cudaMalloc(&d, sizeof(int2) * nblk[l]);
        if (err != cudaSuccess) break;
        owned.push_back(d);
        pairs[l] = d;
        err = cudaMemcpy(d, h->orth_pairs[l].data(), sizeof(int2) * nblk[l], cudaMemcpyHostToDevice);
    }
    if (err == cudaSuccess)
        err = orthogonalize_bases((double *)h->U, (double *)h->Vt, E, Ft, S, pairs, nblk, h->L.k.data(), q, h->L.m,
                                  h->stream);
    for (int2 *d : owned) cudaFree(d);
    if (err == cudaErrorInvalidValue)
        return fail(H2_ERR_ARG, "h2_orthogonalize: needs m <= 128, k <= 64, k^q <= m, k^{l-1} <= 2 k^l <= 128");
    if (err != cudaSuccess) return cuda_fail(h, err, "h2_orthogonalize");
    return H2_OK;
}

extern "C" int h2_reweigh(h2_handle h, void *R_out, int64_t count)
{
    if (!h || !R_out) return fail(H2_ERR_ARG, "NULL argument");
    if (h->sticky) return fail(H2_ERR_STATE, "handle unusable after an earlier CUDA/NCCL error");
    if (h->L.P != 1 || h->dtype != H2_F64 || h->sym || h->group || (int)h->orth_pairs.size() != h->L.q + 1)
        return fail(H2_ERR_ARG, "h2_reweigh: FP64, one GPU, full (non-symmetric) storage only");
    const int q = h->L.q;
    int64_t need = 0;
    for (int l = 0; l <= q; ++l) need += ((int64_t)1 << l) * h->L.k[l] * h->L.k[l];
    if (count != need) return fail(H2_ERR_ARG, "h2_reweigh: count must be sum_l 2^l k_l^2 = " + std::to_string(need));
    std::vector<const int64_t *> rowptr(q + 1, nullptr);
    std::vector<int64_t *> owned;
    std::vector<int> maxb(q + 1, 0);
    std::vector<double *> E(q + 1, nullptr), S(q + 1, nullptr);
    cudaError_t err = cudaStreamSynchronize(h->stream);
    for (int l = 0; l <= q && err == cudaSuccess; ++l) {
        const int n = 1 << l;
        std::vector<int64_t> rp(n + 1, 0);
        for (const int2 &ts : h->orth_pairs[l]) rp[ts.x + 1]++;
        for (int i = 0; i < n; ++i) { maxb[l] = std::max(maxb[l], (int)rp[i + 1]); rp[i + 1] += rp[i]; }
        int64_t *d = nullptr;
        err = cudaMalloc(&d, sizeof(int64_t) * (n + 1));
        if (err != cudaSuccess) break;
        owned.push_back(d);
        rowptr[l] = d;
        err = cudaMemcpy(d, rp.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice);
        E[l] = (double *)h->E[l];
        S[l] = (double *)h->S[l];
    }
    if (err == cudaSuccess) err = reweigh_downsweep(E, S, rowptr, maxb, h->L.k.data(), q, (double *)R_out, h->stream);
    for (int64_t *d : owned) cudaFree(d);
    if (err == cudaErrorInvalidValue) return fail(H2_ERR_ARG, "h2_reweigh: needs k <= 64");
    if (err != cudaSuccess) return cuda_fail(h, err, "h2_reweigh");
    return H2_OK;
}

extern "C" int h2_export(h2_handle h, int what, int level, void *host, int64_t count)
{
    if (!h || !host) return fail(H2_ERR_ARG, "NULL argument");
    if (h->sticky) return fail(H2_ERR_STATE, "handle unusable after an earlier CUDA/NCCL error");
    const int q = h->L.q, m = h->L.m;
    const int64_t nleaf = (int64_t)h->L.held(q);
    const void *src = nullptr;
    int64_t n = 0;
    if (level < 0 || level > q) return fail(H2_ERR_ARG, "h2_export: level out of range");
    const int64_t kl = h->L.k[level], kp = level ? h->L.k[level - 1] : 0;
    switch (what) {
    case H2_EXPORT_S:                                  // blocks in h2_desc CSR order (one GPU, full storage)
        src = h->S[level];
        n = (!h->sym && (int)h->orth_pairs.size() > level) ? (int64_t)h->orth_pairs[level].size() * kl * kl : -1;
        break;
    case H2_EXPORT_U:  src = h->U; n = nleaf * m * h->L.k[q]; break;
    case H2_EXPORT_VT: src = h->Vt; n = nleaf * m * h->L.k[q]; break;
    case H2_EXPORT_E:  src = level ? h->E[level] : nullptr; n = (int64_t)h->L.held(level) * kl * kp; break;
    case H2_EXPORT_FT: src = level ? h->Ft[level] : nullptr; n = (int64_t)h->L.held(level) * kl * kp; break;
    case H2_EXPORT_XHAT:                               // x^ / y^ of `level` after the last matvec:
    case H2_EXPORT_YHAT: {                             // nv vectors x (held nodes x k^l), vector-major
        const int64_t per = (int64_t)h->L.held(level) * kl;
        if (per == 0 || count % per || count / per < 1 || count / per > h->nv_max)
            return fail(H2_ERR_ARG, "h2_export: count must be nv * held(level) * k^l, 1 <= nv <= nv_max");
        const int64_t nvx = count / per;
        const bool xw = what == H2_EXPORT_XHAT;
        const char *base = (const char *)(xw ? h->xh : h->yh);
        const int64_t plane = xw ? h->xh_plane : h->yh_plane;
        const int64_t off = xw ? h->xh_base[level] : h->yh_base[level];
        cudaError_t err = cudaStreamSynchronize(h->stream);
        for (int64_t n = 0; n < nvx && err == cudaSuccess; ++n)
            err = cudaMemcpy((char *)host + (size_t)n * per * h->esz, base + (size_t)(off + n * plane) * h->esz,
                             (size_t)per * h->esz, cudaMemcpyDeviceToHost);
        if (err != cudaSuccess) return cuda_fail(h, err, "h2_export");
        return H2_OK;
    }
    default: return fail(H2_ERR_ARG, "h2_export: unknown array");
    }
    if (n < 0) return fail(H2_ERR_ARG, "h2_export: coupling export needs one GPU and full storage");
    if (!src || n != count) return fail(H2_ERR_ARG, "h2_export: count does not match the array (" + std::to_string(n) + ")");
    cudaError_t err = cudaStreamSynchronize(h->stream);
    if (err == cudaSuccess) err = cudaMemcpy(host, src, (size_t)n * h->esz, cudaMemcpyDeviceToHost);
    if (err != cudaSuccess) return cuda_fail(h, err, "h2_export");
    return H2_OK;
}

extern "C" int h2_destroy(h2_handle h)
{
    if (!h) return H2_OK;
    H2_DBG("rank %d: destroy", h->L.p);
    return release(h);
}

extern "C" int h2_nccl_unique_id(void *out128)
{
    if (!out128) return fail(H2_ERR_ARG, "out is NULL");
    if (!load_nccl()) return fail(H2_ERR_NCCL, "cannot load libnccl.so.2 (set H2_NCCL_LIB)");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(H2_ERR_NCCL, std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(r));
    memcpy(out128, &id, sizeof(id));
    return H2_OK;
}

extern "C" const char *h2_last_error(void) { return g_err.c_str(); }

void h2::set_last_error(const std::string &msg) { g_err = msg; }

extern "C" const char *h2_version(void) { return "h2-b200 0.1 (sm_100a)"; }
