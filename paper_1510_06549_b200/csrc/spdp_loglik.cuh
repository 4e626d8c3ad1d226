// spdp_loglik.cuh — log p(W, Z, T) on the device (diagnostic, not on the sweep path).
//
// log p(W,Z,T) = sum_docs [lnG(sum_k alpha_ik) - lnG(sum_k alpha_ik + L_d)
//                          + sum_k lnG(alpha_ik + n_dk) - lnG(alpha_ik)]
//              + sum_{i,k} [ln (b_i|a_i)_{Tt_ik} - ln (b_i)_{M_ik}]
//              + sum_{i,k,w} ln S^{m_ikw}_{t_ikw, a_i}
//              + sum_k [lnG(V beta) - lnG(V beta + T_k) + sum_w lnG(beta + Q_kw) - lnG(beta)]
// (PAPER.md:1654-1665 with identity P, summed over the prod C(m,t) indicator
// configurations of each T, Eq. SPDP-table-to-head).
// Pochhammer symbols by their Gamma-function closed forms:
// (b)_M = G(b+M)/G(b), (b|a)_T = a^T G(b/a + T)/G(b/a) (a > 0), b^T (a = 0).
#pragma once
#include "spdp_device.cuh"

namespace spdp {

// log S^N_{M,a} for 0 <= M <= N <= nmax by the recursion of PAPER.md:1454-1455
// in log space (fp64), one block, row by row.
__global__ void build_log_stirling(double* __restrict__ ls, int nmax, double a) {
    if (threadIdx.x == 0) ls[0] = 0.0;
    __syncthreads();
    for (int N = 0; N < nmax; ++N) {
        const double* row = ls + tri(N);
        double* nxt = ls + tri(N + 1);
        for (int M = threadIdx.x; M <= N + 1; M += blockDim.x) {
            double v;
            if (M == 0) v = -INFINITY;
            else {
                const double left = row[M - 1];
                const double coef = (double)N - (double)M * a;
                const double right = (M <= N && coef > 0.0) ? log(coef) + row[M] : -INFINITY;
                const double hi = fmax(left, right), lo = fmin(left, right);
                v = (lo == -INFINITY) ? hi : hi + log1p(exp(lo - hi));
            }
            nxt[M] = v;
        }
        __syncthreads();
    }
}

__device__ __forceinline__ double block_sum_fixed(double v, double* sh) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int j = 0; j < (int)(blockDim.x >> 5); ++j) s += sh[j];
    return s;
}

// cells and shadow terms, one warp per word.
__global__ void loglik_words_kernel(const int32_t* __restrict__ m, const int32_t* __restrict__ t,
                                    const int32_t* __restrict__ Q, const double* __restrict__ ls,
                                    const uint64_t* __restrict__ ls_off, int V, int I, int K, int Kp,
                                    double beta, double* __restrict__ partial) {
    __shared__ double sh[32];
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const double lgb = lgamma(beta);
    double acc = 0.0;
    for (int w = blockIdx.x * wpb + (threadIdx.x >> 5); w < V; w += gridDim.x * wpb) {
        for (int k = lane; k < K; k += 32) {
            for (int i = 0; i < I; ++i) {
                const size_t off = ((size_t)w * I + i) * Kp + k;
                const int mv = m[off];
                if (mv) acc += ls[ls_off[i] + tri(mv) + t[off]];
            }
            const int q = Q[(size_t)w * Kp + k];
            if (q) acc += lgamma(beta + (double)q) - lgb;
        }
    }
    const double s = block_sum_fixed(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// document terms, one warp per local document.
template <typename NT>
__global__ void loglik_docs_kernel(const NT* __restrict__ n, const int* __restrict__ sigma,
                                   const int32_t* __restrict__ doclen,
                                   const int32_t* __restrict__ docgroup, const double* __restrict__ alpha,
                                   const double* __restrict__ alpha_sum, int D, int K, int Kp, int Kn,
                                   double* __restrict__ partial) {
    __shared__ double sh[32];
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    double acc = 0.0;
    for (int d = blockIdx.x * wpb + (threadIdx.x >> 5); d < D; d += gridDim.x * wpb) {
        const int i = docgroup[d];
        if (doclen[d] == 0) continue;      // empty document: p(z_d) = 1
        for (int k = lane; k < K; k += 32) {
            const int nv = Row<NT>::get(n + (size_t)d * Kn + sigma[k]);
            if (nv) {
                const double al = alpha[(size_t)i * Kp + k];
                acc += lgamma(al + (double)nv) - lgamma(al);
            }
        }
        if (lane == 0) acc += lgamma(alpha_sum[i]) - lgamma(alpha_sum[i] + (double)doclen[d]);
    }
    const double s = block_sum_fixed(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// restaurant and topic-normaliser terms (I*K + K values), one block.
__global__ void loglik_small_kernel(const int32_t* __restrict__ M, const int32_t* __restrict__ Tt,
                                    const int32_t* __restrict__ T, const double* __restrict__ disc,
                                    const double* __restrict__ conc, int I, int K, int Kp, double vbeta,
                                    double* __restrict__ out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int j = threadIdx.x; j < I * K; j += blockDim.x) {
        const int i = j / K, k = j % K;
        const double a = disc[i], b = conc[i];
        const double tt = (double)Tt[(size_t)i * Kp + k], mm = (double)M[(size_t)i * Kp + k];
        const double lpt = (a > 0.0) ? tt * log(a) + lgamma(b / a + tt) - lgamma(b / a) : tt * log(b);
        acc += lpt - (lgamma(b + mm) - lgamma(b));
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) acc += lgamma(vbeta) - lgamma(vbeta + (double)T[k]);
    const double s = block_sum_fixed(acc, sh);
    if (threadIdx.x == 0) *out = s;
}

// normalise debug weights: probs = w / sum(w), sum in slot order.
__global__ void normalise_rows_kernel(double* __restrict__ w, int rows, int cols) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    double* x = w + (size_t)r * cols;
    double s = 0.0;
    for (int j = 0; j < cols; ++j) s += x[j];
    for (int j = 0; j < cols; ++j) x[j] /= s;
}

}  // namespace spdp
