// h2_k_orth.cu -- basis orthogonalization (first step):
// the QR upsweep of both basis trees and the re-expression of every coupling block,
//
//   leaves:      U_t = Q_t R_t  (thin Householder QR, diag R >= 0)      U'_t = Q_t
//   level l:     M_p = [R_c1 E_c1; R_c2 E_c2] = Q_p R_p                 E'_c1 | E'_c2 = Q_p split
//   couplings:   S'_ts = R^U_t S_ts (R^V_s)^T
//
// in place on a handle's device arrays (FP64, one GPU, full storage).  One CTA per small matrix
// (batched over the nodes of a level, "batched QR"); every matrix lives in shared
// memory while it is factored.  Work is O(N k^2): a one-off pre-processing pass, not a hot path.
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include <vector>
#include "h2_internal.h"

namespace h2 {
namespace orth {

constexpr int THREADS = 256;
constexpr int MAXR = 128, MAXC = 64;

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Householder QR of the R x C column-major matrix a (ld R) in shared memory, in place: R in the
// upper triangle, the reflectors v_j (v_j[j] = 1 implicit) below it, tau[j] their scalars
// (LAPACK dgeqr2 / dlarfg conventions).  Whole CTA.
__device__ void householder(double *a, int R, int C, double *tau, double *red)
{
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = THREADS / 32;
    const int K = R < C ? R : C;
    for (int j = 0; j < K; ++j) {
        // Householder vector of column j below the diagonal (LAPACK dlarfg convention)
        double s = 0.0;
        for (int i = j + 1 + tid; i < R; i += THREADS) s += a[i + j * R] * a[i + j * R];
        s = warp_sum(s);
        if (lane == 0) red[wid] = s;
        __syncthreads();
        double sigma = 0.0;
        for (int w = 0; w < nw; ++w) sigma += red[w];
        const double alpha = a[j + j * R];
        double t = 0.0, beta = alpha, scale = 0.0;
        if (sigma > 0.0) {
            const double nrm = sqrt(alpha * alpha + sigma);
            beta = alpha >= 0.0 ? -nrm : nrm;
            t = (beta - alpha) / beta;
            scale = 1.0 / (alpha - beta);
        }
        __syncthreads();                                     // everyone has read a[j, j] and red
        for (int i = j + 1 + tid; i < R; i += THREADS) a[i + j * R] *= scale;    // v (v_j = 1 implicit)
        if (tid == 0) { a[j + j * R] = beta; tau[j] = t; }
        __syncthreads();
        // apply H_j = I - tau v v^T to the trailing columns: one warp per column
        if (t != 0.0)
            for (int c = j + 1 + wid; c < C; c += nw) {
                double w = 0.0;
                for (int i = j + lane; i < R; i += 32) w += (i == j ? 1.0 : a[i + j * R]) * a[i + c * R];
                w = warp_sum(w) * t;
                for (int i = j + lane; i < R; i += 32) a[i + c * R] -= w * (i == j ? 1.0 : a[i + j * R]);
            }
        __syncthreads();
    }
}

// Thin QR of a batch of R x C matrices (R >= C, R <= 128, C <= 64), element (i, j) of matrix b at
// A + b * bs + i * rs + j * cs.  Overwrites A with the explicit Q (R x C) and writes R (C x C,
// column-major) to Rout + b * C * C; diag(R) >= 0 (column signs of Q flipped to match).
__global__ void __launch_bounds__(THREADS) k_qr(double *A, int64_t bs, int64_t rs, int64_t cs, int R, int C,
                                               double *Rout)
{
    extern __shared__ double dyn[];
    double *a = dyn, *q = dyn + R * C;     // column-major, ld R (2 R C doubles of dynamic smem)
    __shared__ double tau[MAXC];
    __shared__ double red[THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = THREADS / 32;
    double *Ab = A + (int64_t)blockIdx.x * bs;
    for (int e = tid; e < R * C; e += THREADS) {
        const int i = e % R, j = e / R;
        a[e] = Ab[i * rs + j * cs];
    }
    __syncthreads();
    householder(a, R, C, tau, red);
    // explicit Q = H_0 H_1 ... H_{C-1} [I; 0], reflectors applied last to first
    for (int e = tid; e < R * C; e += THREADS) {
        const int i = e % R, j = e / R;
        q[e] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int j = C - 1; j >= 0; --j) {
        const double t = tau[j];
        if (t != 0.0)
            for (int c = j + wid; c < C; c += nw) {
                double w = 0.0;
                for (int i = j + lane; i < R; i += 32) w += (i == j ? 1.0 : a[i + j * R]) * q[i + c * R];
                w = warp_sum(w) * t;
                for (int i = j + lane; i < R; i += 32) q[i + c * R] -= w * (i == j ? 1.0 : a[i + j * R]);
            }
        __syncthreads();
    }
    // sign normalisation (diag R >= 0) and write-back
    double *Rb = Rout + (int64_t)blockIdx.x * C * C;
    for (int e = tid; e < C * C; e += THREADS) {
        const int i = e % C, j = e / C;
        const double sg = a[i + i * R] < 0.0 ? -1.0 : 1.0;
        Rb[e] = (i <= j) ? sg * a[i + j * R] : 0.0;
    }
    for (int e = tid; e < R * C; e += THREADS) {
        const int i = e % R, j = e / R;
        const double sg = a[j + j * R] < 0.0 ? -1.0 : 1.0;
        Ab[i * rs + j * cs] = sg * q[e];
    }
}

// M_p = [R_c1 T_c1; R_c2 T_c2] for every parent p of a level: R_c (kl x kl, col-major, batch
// stride kl^2), T_c (kl x kp) element (i, j) at T + c * kl * kp + i * trs + j * tcs; M_p column-major
// 2 kl x kp.  One CTA per parent.
__global__ void __launch_bounds__(THREADS) k_stack(const double *Rl, const double *T, int64_t trs, int64_t tcs,
                                                  int kl, int kp, double *M)
{
    const int p = blockIdx.x;
    double *Mp = M + (int64_t)p * 2 * kl * kp;
    for (int e = threadIdx.x; e < 2 * kl * kp; e += blockDim.x) {
        const int i2 = e % (2 * kl), j = e / (2 * kl);
        const int half = i2 / kl, i = i2 % kl, c = 2 * p + half;
        const double *Rc = Rl + (int64_t)c * kl * kl;
        const double *Tc = T + (int64_t)c * kl * kp;
        double s = 0.0;
        for (int k = i; k < kl; ++k) s += Rc[i + k * kl] * Tc[k * trs + j * tcs];   // R upper triangular
        Mp[e] = s;
    }
}

// E'_c1 | E'_c2 = rows [0, kl) | [kl, 2 kl) of Q_p, written into the transfer storage (strides as k_stack)
__global__ void __launch_bounds__(THREADS) k_split(const double *M, int kl, int kp, double *T, int64_t trs, int64_t tcs)
{
    const int p = blockIdx.x;
    const double *Mp = M + (int64_t)p * 2 * kl * kp;
    for (int e = threadIdx.x; e < 2 * kl * kp; e += blockDim.x) {
        const int i2 = e % (2 * kl), j = e / (2 * kl);
        const int half = i2 / kl, i = i2 % kl, c = 2 * p + half;
        T[(int64_t)c * kl * kp + i * trs + j * tcs] = Mp[e];
    }
}

// S'_b = R^U_t S_b (R^V_s)^T for the coupling blocks of one level (k x k, column-major), pairs[b] = (t, s)
__global__ void __launch_bounds__(THREADS) k_project(double *S, const int2 *pairs, const double *RU, const double *RV,
                                                    int k)
{
    extern __shared__ double dyn[];
    double *s = dyn, *w = dyn + k * k;
    const int b = blockIdx.x;
    const int2 ts = pairs[b];
    double *Sb = S + (int64_t)b * k * k;
    const double *Ru = RU + (int64_t)ts.x * k * k, *Rv = RV + (int64_t)ts.y * k * k;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) s[e] = Sb[e];
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {          // w = R^U_t S
        const int i = e % k, j = e / k;
        double v = 0.0;
        for (int l = i; l < k; ++l) v += Ru[i + l * k] * s[l + j * k];
        w[e] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {          // S' = w (R^V_s)^T
        const int i = e % k, j = e / k;
        double v = 0.0;
        for (int l = j; l < k; ++l) v += w[i + l * k] * Rv[j + l * k];
        Sb[e] = v;
    }
}

// Reweighing downsweep step: R^l_i (kl x kl, column-major at Rl + i kl^2) <- the R
// factor of a stack, for every node i of a level (one CTA each):
//   fold < 0 (start):  stack = R^{l-1}_{i+} E_i^T (kp x kl; zero at the root: R <- 0);
//   fold = f >= 0:     stack = [R^l_i ; S_{i b}^T] with b = rowptr[i] + f (rows without an f-th
//                      block keep their R).
// R is written sign-normalised (diag >= 0) and zero-padded to kl x kl.
__global__ void __launch_bounds__(THREADS) k_rfold(double *Rl, const double *Rp, const double *E, const double *S,
                                                  const int64_t *rowptr, int kl, int kp, int fold)
{
    extern __shared__ double dyn[];
    __shared__ double tau[MAXC];
    __shared__ double red[THREADS / 32];
    const int i = blockIdx.x, tid = threadIdx.x;
    double *Ri = Rl + (int64_t)i * kl * kl;
    int rows;
    double *a = dyn;
    if (fold < 0) {
        if (!Rp) {
            for (int e = tid; e < kl * kl; e += THREADS) Ri[e] = 0.0;
            return;
        }
        rows = kp;
        const double *Rpi = Rp + (int64_t)(i >> 1) * kp * kp;            // R_{i+}: kp x kp upper
        const double *Ei = E + (int64_t)i * kl * kp;                      // E_i: kl x kp column-major
        for (int e = tid; e < kp * kl; e += THREADS) {
            const int r = e % kp, c = e / kp;                             // (R_{i+} E_i^T)(r, c)
            double v = 0.0;
            for (int t = r; t < kp; ++t) v += Rpi[r + t * kp] * Ei[c + t * kl];
            a[r + c * rows] = v;
        }
    } else {
        const int64_t b = rowptr[i] + fold;
        if (b >= rowptr[i + 1]) return;
        rows = 2 * kl;
        const double *Sb = S + b * kl * kl;                               // stored S (column-major)
        for (int e = tid; e < kl * kl; e += THREADS) {
            const int r = e % kl, c = e / kl;
            a[r + c * rows] = Ri[e];                                      // current R (padded rows 0)
            a[kl + r + c * rows] = Sb[c + r * kl];                        // S^T(r, c) = S(c, r)
        }
    }
    __syncthreads();
    householder(a, rows, kl, tau, red);
    for (int e = tid; e < kl * kl; e += THREADS) {
        const int r = e % kl, c = e / kl;
        double v = 0.0;
        if (r < rows && r <= c) v = (a[r + r * rows] < 0.0 ? -1.0 : 1.0) * a[r + c * rows];
        Ri[e] = v;
    }
}

}  // namespace orth

// QR upsweep of one basis tree in place.  leaf: nleaf matrices m x kq, element (i, j) at
// leaf + t * m * kq + i * lrs + j * lcs; T[l] (l = 1..q): 2^l transfers kl x kp with strides
// (trs[l], tcs[l]); R[l]: 2^l x kl^2 output.  W: workspace >= 2^(q-1) * 2 kq * k_{q-1} doubles.
static cudaError_t orth_tree(double *leaf, int64_t lrs, int64_t lcs, int m, const std::vector<double *> &T,
                             const std::vector<int64_t> &trs, const std::vector<int64_t> &tcs, const int *k, int q,
                             const std::vector<double *> &R, double *W, cudaStream_t s)
{
    using namespace orth;
    k_qr<<<1 << q, THREADS, (size_t)2 * m * k[q] * sizeof(double), s>>>(leaf, (int64_t)m * k[q], lrs, lcs, m, k[q], R[q]);
    for (int l = q; l >= 1; --l) {
        const int kl = k[l], kp = k[l - 1], np = 1 << (l - 1);
        k_stack<<<np, THREADS, 0, s>>>(R[l], T[l], trs[l], tcs[l], kl, kp, W);
        k_qr<<<np, THREADS, (size_t)2 * 2 * kl * kp * sizeof(double), s>>>(W, (int64_t)2 * kl * kp, 1, 2 * kl, 2 * kl, kp,
                                                                        R[l - 1]);
        k_split<<<np, THREADS, 0, s>>>(W, kl, kp, T[l], trs[l], tcs[l]);
    }
    return cudaGetLastError();
}

cudaError_t reweigh_downsweep(const std::vector<double *> &E, const std::vector<double *> &S,
                              const std::vector<const int64_t *> &rowptr, const std::vector<int> &maxb, const int *k,
                              int q, double *Rout, cudaStream_t s)
{
    using namespace orth;
    for (int l = 0; l <= q; ++l)
        if (k[l] > MAXC || (l >= 1 && k[l - 1] > 2 * MAXC)) return cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(k_rfold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(2 * MAXC * MAXC * sizeof(double)));
    if (err != cudaSuccess) return err;
    double *Rl = Rout, *Rp = nullptr;
    for (int l = 0; l <= q && err == cudaSuccess; ++l) {
        const int kl = k[l], kp = l ? k[l - 1] : 0, n = 1 << l;
        const size_t sm = (size_t)std::max(2 * kl, kp) * kl * sizeof(double);
        k_rfold<<<n, THREADS, sm, s>>>(Rl, Rp, l ? E[l] : nullptr, S[l], rowptr[l], kl, kp, -1);
        for (int f = 0; f < maxb[l]; ++f)
            k_rfold<<<n, THREADS, sm, s>>>(Rl, Rp, l ? E[l] : nullptr, S[l], rowptr[l], kl, kp, f);
        err = cudaGetLastError();
        Rp = Rl;
        Rl += (size_t)n * kl * kl;
    }
    cudaError_t e2 = cudaStreamSynchronize(s);
    return err == cudaSuccess ? e2 : err;
}

cudaError_t orthogonalize_bases(double *U, double *Vt, const std::vector<double *> &E, const std::vector<double *> &Ft,
                                const std::vector<double *> &S, const std::vector<const int2 *> &pairs,
                                const std::vector<int64_t> &nblk, const int *k, int q, int m, cudaStream_t s)
{
    using namespace orth;
    if (m > MAXR || k[q] > m) return cudaErrorInvalidValue;
    for (int l = 0; l <= q; ++l)
        if (k[l] > MAXC || (l >= 1 && (2 * k[l] > MAXR || k[l - 1] > 2 * k[l]))) return cudaErrorInvalidValue;
    std::vector<double *> RU(q + 1, nullptr), RV(q + 1, nullptr);
    double *W = nullptr;
    cudaError_t err = cudaFuncSetAttribute(k_qr, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(2 * MAXR * MAXC * sizeof(double)));
    if (err == cudaSuccess)
        err = cudaFuncSetAttribute(k_project, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(2 * MAXC * MAXC * sizeof(double)));
    if (err != cudaSuccess) return err;
    size_t wmax = 1;
    for (int l = 1; l <= q; ++l) wmax = std::max(wmax, (size_t)(1 << (l - 1)) * 2 * k[l] * k[l - 1]);
    // stream-ordered pool allocations: the R workspaces (GBs at 2^15 leaves, k = 64) are reused
    // across calls instead of mapped and unmapped each time
    for (int l = 0; l <= q && err == cudaSuccess; ++l) {
        err = cudaMallocAsync(&RU[l], sizeof(double) * ((size_t)1 << l) * k[l] * k[l], s);
        if (err == cudaSuccess) err = cudaMallocAsync(&RV[l], sizeof(double) * ((size_t)1 << l) * k[l] * k[l], s);
    }
    if (err == cudaSuccess) err = cudaMallocAsync(&W, sizeof(double) * wmax, s);
    if (err == cudaSuccess) {
        // U tree: U (m x kq column-major), E[l] (kl x kp column-major)
        std::vector<int64_t> ers(q + 1, 1), ecs(q + 1), frs(q + 1), fcs(q + 1, 1);
        for (int l = 1; l <= q; ++l) { ecs[l] = k[l]; frs[l] = k[l - 1]; }
        err = orth_tree(U, 1, m, m, E, ers, ecs, k, q, RU, W, s);
        // V tree from the stored transposes: V_t(i, j) = Vt_t(j, i), F_c(i, j) = Ft_c(j, i)
        if (err == cudaSuccess) err = orth_tree(Vt, k[q], 1, m, Ft, frs, fcs, k, q, RV, W, s);
        for (int l = 0; l <= q && err == cudaSuccess; ++l)
            if (nblk[l] > 0) {
                k_project<<<(unsigned)nblk[l], THREADS, (size_t)2 * k[l] * k[l] * sizeof(double), s>>>(S[l], pairs[l],
                                                                                                   RU[l], RV[l], k[l]);
                err = cudaGetLastError();
            }
    }
    for (int l = 0; l <= q; ++l) {
        if (RU[l]) cudaFreeAsync(RU[l], s);
        if (RV[l]) cudaFreeAsync(RV[l], s);
    }
    if (W) cudaFreeAsync(W, s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (err == cudaSuccess) err = e2;
    return err;
}

}  // namespace h2
