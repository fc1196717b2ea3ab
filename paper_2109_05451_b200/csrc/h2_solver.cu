// h2_solver.cu -- the fractional-diffusion solve on top of the H² matvec (include/h2.h
// h2_fd_diag, h2_pcg):
//
//     A u = h^2 (D + K + C) u = b,   D_ii = (K^ 1)_i,  K = the handle's H² operator
//
// solved by preconditioned conjugate gradients ("preconditioned conjugate gradient")
// with the Jacobi preconditioner diag(A) = h^2 (D + C_ii) (K has a zero diagonal) standing in for
// the paper's PETSc smoothed-aggregation AMG ("a Jacobi or geometric-MG stand-in").
// One H² matvec, one CSR product and two fused vector passes per iteration; the scalar reductions
// are per-CTA partial sums summed on the host in a fixed order (deterministic).
#include "../../include/h2.h"
#include "h2_internal.h"

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

namespace {

constexpr int RB = 256;          // threads per CTA of the vector kernels
constexpr int RG = 296;          // CTAs (2 per SM)

__device__ __forceinline__ double block_sum(double v, double *sh)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    v = (threadIdx.x < blockDim.x / 32) ? sh[threadIdx.x] : 0.0;
    if (w == 0)
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;   // valid in thread 0
}

// diag[i] = (K^ 1)[idx[i]] + cdiag[i]
__global__ void k_fd_diag(const double *khat1, const int64_t *idx, const double *cdiag, int64_t n, double *diag)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        diag[i] = khat1[idx[i]] + (cdiag ? cdiag[i] : 0.0);
}

__global__ void k_fill(double *x, int64_t n, double v)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] = v;
}

// q = scale (Ku + diag u + C_off u), with Ku already in q; partial[b] = sum_i p_i q_i (p = u here)
__global__ void k_apply(double *q, const double *u, const double *diag, const int64_t *rp, const int32_t *col,
                        const double *val, int64_t n, double scale, double *partial)
{
    __shared__ double sh[32];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = q[i] + diag[i] * u[i];
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
            if (col[e] != i) s += val[e] * u[col[e]];
        s *= scale;
        q[i] = s;
        acc += u[i] * s;
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

// u += alpha p ; r -= alpha q ; z = r / (scale diag) ; partial = (r.r, r.z)
__global__ void k_update(double *u, double *r, double *z, const double *p, const double *q, const double *diag,
                         int64_t n, double alpha, double scale, double *partial)
{
    __shared__ double sh[32];
    double rr = 0.0, rz = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        u[i] = fma(alpha, p[i], u[i]);
        const double ri = fma(-alpha, q[i], r[i]);
        r[i] = ri;
        const double zi = ri / (scale * diag[i]);
        z[i] = zi;
        rr += ri * ri;
        rz += ri * zi;
    }
    rr = block_sum(rr, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = rr;
    rz = block_sum(rz, sh);
    if (threadIdx.x == 0) partial[gridDim.x + blockIdx.x] = rz;
}

// r = b - q ; z = p = r / (scale diag) ; partial = (r.r, r.z, b.b)
__global__ void k_init(const double *b, const double *q, double *r, double *z, double *p, const double *diag,
                       int64_t n, double scale, double *partial)
{
    __shared__ double sh[32];
    double rr = 0.0, rz = 0.0, bb = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double ri = b[i] - q[i];
        const double zi = ri / (scale * diag[i]);
        r[i] = ri;
        z[i] = zi;
        p[i] = zi;
        rr += ri * ri;
        rz += ri * zi;
        bb += b[i] * b[i];
    }
    rr = block_sum(rr, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = rr;
    rz = block_sum(rz, sh);
    if (threadIdx.x == 0) partial[gridDim.x + blockIdx.x] = rz;
    bb = block_sum(bb, sh);
    if (threadIdx.x == 0) partial[2 * gridDim.x + blockIdx.x] = bb;
}

// p = z + beta p
__global__ void k_pupdate(double *p, const double *z, int64_t n, double beta)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = fma(beta, p[i], z[i]);
}

double host_sum(const std::vector<double> &v, int a, int b)
{
    double s = 0.0;
    for (int i = a; i < b; ++i) s += v[i];
    return s;
}

}  // namespace

extern "C" int h2_fd_diag(h2_handle khat, const int64_t *idx, const double *cdiag, int64_t n, double *diag)
{
    if (!khat || !idx || !diag || n < 0) { h2::set_last_error("h2_fd_diag: bad argument"); return H2_ERR_ARG; }
    int64_t ne = 0;
    int rc = h2_n_local(khat, &ne);
    if (rc != H2_OK) return rc;
    double *ones = nullptr, *out = nullptr;
    if (cudaMalloc(&ones, (size_t)ne * 8) != cudaSuccess || cudaMalloc(&out, (size_t)ne * 8) != cudaSuccess) {
        cudaFree(ones);
        h2::set_last_error("h2_fd_diag: cudaMalloc failed");
        return H2_ERR_OOM;
    }
    k_fill<<<RG, RB>>>(ones, ne, 1.0);
    rc = h2_set_stream(khat, nullptr);
    if (rc == H2_OK) rc = h2_matvec(khat, 1.0, ones, 0.0, out, 1);
    if (rc == H2_OK) {
        k_fd_diag<<<RG, RB>>>(out, idx, cdiag, n, diag);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            h2::set_last_error(std::string("h2_fd_diag: ") + cudaGetErrorString(e));
            rc = H2_ERR_CUDA;
        }
    }
    cudaFree(ones);
    cudaFree(out);
    return rc;
}

extern "C" int h2_pcg(h2_handle K, double scale, const double *diag, const int64_t *C_rowptr, const int32_t *C_col,
                      const double *C_val, const double *b, double *u, double rtol, int maxit, int *iters,
                      double *res_hist)
{
    if (!K || !diag || !C_rowptr || !b || !u || maxit < 0 || !(rtol > 0)) {
        h2::set_last_error("h2_pcg: bad argument");
        return H2_ERR_ARG;
    }
    int64_t n = 0;
    int rc = h2_n_local(K, &n);
    if (rc != H2_OK) return rc;
    rc = h2_set_stream(K, nullptr);
    if (rc != H2_OK) return rc;
    double *w = nullptr, *part = nullptr;
    if (cudaMalloc(&w, (size_t)4 * n * 8) != cudaSuccess || cudaMalloc(&part, (size_t)3 * RG * 8) != cudaSuccess) {
        cudaFree(w);
        h2::set_last_error("h2_pcg: cudaMalloc failed");
        return H2_ERR_OOM;
    }
    double *r = w, *z = w + n, *p = w + 2 * n, *q = w + 3 * n;
    std::vector<double> hp(3 * RG);
    auto fetch = [&]() -> int {
        cudaError_t e = cudaMemcpy(hp.data(), part, hp.size() * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { h2::set_last_error(std::string("h2_pcg: ") + cudaGetErrorString(e)); return H2_ERR_CUDA; }
        return H2_OK;
    };
    auto apply = [&](const double *x, double *y) -> int {      // y = A x, part = x.y
        int r2 = h2_matvec(K, 1.0, x, 0.0, y, 1);
        if (r2 != H2_OK) return r2;
        k_apply<<<RG, RB>>>(y, x, diag, C_rowptr, C_col, C_val, n, scale, part);
        return cudaGetLastError() == cudaSuccess ? H2_OK : H2_ERR_CUDA;
    };
    int it = 0;
    // r = b - A u ; z = M^-1 r ; p = z
    rc = apply(u, q);
    double bb = 0.0, rr = 0.0, rz = 0.0;
    if (rc == H2_OK) {
        k_init<<<RG, RB>>>(b, q, r, z, p, diag, n, scale, part);
        rc = fetch();
        rr = host_sum(hp, 0, RG);
        rz = host_sum(hp, RG, 2 * RG);
        bb = host_sum(hp, 2 * RG, 3 * RG);
    }
    const double bnorm = std::sqrt(bb) > 0 ? std::sqrt(bb) : 1.0;
    if (res_hist) res_hist[0] = std::sqrt(rr) / bnorm;
    while (rc == H2_OK && it < maxit && std::sqrt(rr) / bnorm > rtol) {
        rc = apply(p, q);                                   // q = A p, part = p.q
        if (rc != H2_OK) break;
        if ((rc = fetch()) != H2_OK) break;
        const double pq = host_sum(hp, 0, RG);
        const double alpha = rz / pq;
        k_update<<<RG, RB>>>(u, r, z, p, q, diag, n, alpha, scale, part);
        if ((rc = fetch()) != H2_OK) break;
        rr = host_sum(hp, 0, RG);
        const double rz_new = host_sum(hp, RG, 2 * RG);
        const double beta = rz_new / rz;
        rz = rz_new;
        k_pupdate<<<RG, RB>>>(p, z, n, beta);
        ++it;
        if (res_hist) res_hist[it] = std::sqrt(rr) / bnorm;
    }
    if (rc == H2_OK) {
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { h2::set_last_error(std::string("h2_pcg: ") + cudaGetErrorString(e)); rc = H2_ERR_CUDA; }
    }
    if (iters) *iters = it;
    cudaFree(w);
    cudaFree(part);
    return rc;
}
