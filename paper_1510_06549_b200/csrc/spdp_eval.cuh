// spdp_eval.cuh — NEXT-1: held-out evaluation on the device.
//
//  * phi_table_kernel: the topic-word estimates of the trained state,
//      phi0~_kw  = (beta + Q_kw) / (V beta + T_k)                       Eq. P:1753 (identity P)
//      phi~^i_kw = (m_ikw - a_i t_ikw)/(b_i + m_ik.) + (b_i + a_i t_ik.)/(b_i + m_ik.) phi0~_kw
//                                                                       Eq. P:1754, reading c16
//    in fp64, laid out like the count rows: [w][i][Kp].
//  * foldin_kernel: fold-in of held-out documents (reading c21): collapsed
//    Gibbs over their topics with phi~ frozen, p(k) ∝ (alpha_ik + n_dk^{-p}) phi~^i_{k w};
//    documents are independent given phi~, so one warp owns one document and
//    runs ALL iterations over its tokens sequentially (exact sequential Gibbs,
//    no staleness), with n_d in shared memory.  Then theta~ (Eq. P:1736-1740)
//    and the document's log-likelihood sum_p log sum_k theta~_dk phi~^i_{k w_p}
//    (held-out perplexity, reading c17).
//  * sqrt_phi0_kernel + hellinger_kernel: the K x K Hellinger distances of two
//    models' phi0~ rows (§4.2.6, reading c22): a K x V x K
//    contraction of sqrt(phi0~) in fp64 (fp64 because H ~ sqrt(1 - BC) cancels
//    near 0), shared-memory tiled.
#pragma once
#include "spdp_device.cuh"

namespace spdp {

__global__ void phi_table_kernel(const int32_t* __restrict__ m, const int32_t* __restrict__ t,
                                 const int32_t* __restrict__ Q, const int32_t* __restrict__ M,
                                 const int32_t* __restrict__ Tt, const int32_t* __restrict__ T,
                                 const double* __restrict__ disc, const double* __restrict__ conc, double beta,
                                 double vbeta, int V, int I, int K, int Kp, double* __restrict__ phi,
                                 double* __restrict__ phi0, const uint32_t* __restrict__ sptr = nullptr,
                                 const int32_t* __restrict__ spv = nullptr, const double* __restrict__ spp = nullptr) {
    const size_t cells = (size_t)V * I * Kp;
    for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < cells; c += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(c % Kp);
        const size_t wi = c / Kp;
        const int i = (int)(wi % I), w = (int)(wi / I);
        double v = 0.0;
        if (k < K) {
            const double p0 = (beta + (double)Q[(size_t)w * Kp + k]) / (vbeta + (double)T[k]);
            double base = p0;
            if (sptr) {                               // NEXT-4: sum_v p^i_{w,v} phi0~_{kv}
                base = 0.0;
                const uint32_t seg = (uint32_t)wi;
                for (uint32_t e = sptr[seg]; e < sptr[seg + 1]; ++e)
                    base += spp[e] * ((beta + (double)Q[(size_t)spv[e] * Kp + k]) / (vbeta + (double)T[k]));
            }
            const double a = disc[i], b = conc[i];
            const double Mk = M[(size_t)i * Kp + k], Tk = Tt[(size_t)i * Kp + k];
            v = ((double)m[c] - a * (double)t[c]) / (b + Mk) + (b + a * Tk) / (b + Mk) * base;
            if (phi0 && i == 0) phi0[(size_t)k * V + w] = p0;
        }
        if (phi) phi[c] = v;
    }
}

struct FoldinArgs {
    const int32_t* word;       // [Nh] held-out tokens grouped by document (canonical order inside)
    const uint32_t* id;        // [Nh] canonical held-out token index (RNG counter)
    const uint32_t* doc_ptr;   // [Dh + 1]
    const int32_t* doc_group;  // [Dh]
    int32_t* z;                // [Nh] in: initial topics (if !init), out: final topics
    const double* phi;         // [V][I][Kp]
    const double* alpha;       // [I][Kp]
    const double* alpha_sum;   // [I]
    double* theta;             // [Dh][K] or null
    double* partial;           // [Dh] per-document log-likelihood
    int Dh, I, K, Kp;
    uint32_t key0, key1;
    int first_iter, iters, init;
};

// KB topics per lane, lane l owns k in [l*KB, l*KB + KB); one warp per document.
template <int KB>
__global__ void __launch_bounds__(256) foldin_kernel(FoldinArgs A) {
    extern __shared__ int s_n[];                     // [warps][Kp]
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    int* n = s_n + (size_t)(threadIdx.x >> 5) * A.Kp;
    const int K = A.K, Kp = A.Kp, kb = lane * KB;
    for (int d = blockIdx.x * wpb + (threadIdx.x >> 5); d < A.Dh; d += gridDim.x * wpb) {
        const uint32_t b0 = A.doc_ptr[d], b1 = A.doc_ptr[d + 1];
        const int i = A.doc_group[d];
        for (int k = lane; k < Kp; k += 32) n[k] = 0;
        __syncwarp();
        for (uint32_t p = b0 + lane; p < b1; p += 32) {
            int zz;
            if (A.init) {
                const uint4 x = philox(make_uint4(A.id[p], 0xFFFFFFFFu, 1u, 0u), A.key0, A.key1);
                zz = (int)(((uint64_t)x.x * (uint64_t)K) >> 32);
                A.z[p] = zz;
            } else {
                zz = A.z[p];
            }
            atomicAdd(&n[zz], 1);
        }
        __syncwarp();
        double al[KB];
#pragma unroll
        for (int j = 0; j < KB; ++j) al[j] = (kb + j < K) ? A.alpha[(size_t)i * Kp + kb + j] : 0.0;
        for (int it = A.first_iter; it < A.first_iter + A.iters; ++it) {
            for (uint32_t base = b0; base < b1; base += 32) {
                // one Philox per lane for the next 32 tokens of the document
                double u_l = 0.0;
                int z_l = 0, w_l = 0;
                if (base + lane < b1) {
                    u_l = u53(philox(make_uint4(A.id[base + lane], (uint32_t)it, 1u, 0u), A.key0, A.key1));
                    z_l = A.z[base + lane];
                    w_l = A.word[base + lane];
                }
                const int cnt = (int)min(32u, b1 - base);
                for (int q = 0; q < cnt; ++q) {
                    const double u = __shfl_sync(0xffffffffu, u_l, q);
                    const int w = __shfl_sync(0xffffffffu, w_l, q);
                    int zo = __shfl_sync(0xffffffffu, z_l, q);
                    if (lane == 0) n[zo] -= 1;               // n_dk^{-p}
                    __syncwarp();
                    const double* prow = A.phi + ((size_t)w * A.I + i) * Kp + kb;
                    double wt[KB], s = 0.0;
#pragma unroll
                    for (int j = 0; j < KB; ++j) {
                        wt[j] = (kb + j < K) ? (al[j] + (double)n[kb + j]) * prow[j] : 0.0;
                        s += wt[j];
                    }
                    // inclusive warp scan of the lane sums
                    double incl = s;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const double y = __shfl_up_sync(0xffffffffu, incl, off);
                        if (lane >= off) incl += y;
                    }
                    const double total = __shfl_sync(0xffffffffu, incl, 31);
                    const double target = u * total;
                    // k* = min{k : cdf_k > u * total} (reading c10 with K slots)
                    const unsigned hit = __ballot_sync(0xffffffffu, incl > target);
                    int knew = -1;
                    if (hit) {
                        const int L = __ffs(hit) - 1;
                        if (lane == L) {
                            double c = incl - s;
#pragma unroll
                            for (int j = 0; j < KB; ++j) {
                                c += wt[j];
                                if (knew < 0 && c > target && wt[j] > 0.0) knew = kb + j;
                            }
                            if (knew < 0) {                  // rounding inside the lane: last positive slot
#pragma unroll
                                for (int j = 0; j < KB; ++j) if (wt[j] > 0.0) knew = kb + j;
                            }
                        }
                        knew = __shfl_sync(0xffffffffu, knew, L);
                    } else {                                 // rounding: the last slot with positive mass
                        int last = -1;
#pragma unroll
                        for (int j = 0; j < KB; ++j) if (wt[j] > 0.0) last = kb + j;
                        const unsigned pos = __ballot_sync(0xffffffffu, last >= 0);
                        const int L = 31 - __clz(pos);
                        knew = __shfl_sync(0xffffffffu, last, L);
                    }
                    if (lane == 0) n[knew] += 1;
                    if (lane == q) z_l = knew;
                    __syncwarp();
                }
                if (base + lane < b1) A.z[base + lane] = z_l;
                __syncwarp();
            }
        }
        // theta~ (Eq. P:1736-1740) and the document's log-likelihood
        const double denom = (double)(b1 - b0) + A.alpha_sum[i];
        double th[KB];
#pragma unroll
        for (int j = 0; j < KB; ++j) {
            th[j] = (kb + j < K) ? ((double)n[kb + j] + al[j]) / denom : 0.0;
            if (A.theta && kb + j < K) A.theta[(size_t)d * K + kb + j] = th[j];
        }
        double ll = 0.0;
        for (uint32_t p = b0; p < b1; ++p) {
            const int w = A.word[p];
            const double* prow = A.phi + ((size_t)w * A.I + i) * Kp + kb;
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < KB; ++j) if (kb + j < K) s += th[j] * prow[j];
#pragma unroll
            for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            ll += log(s);
        }
        if (lane == 0) A.partial[d] = ll;
        __syncwarp();
    }
}

// sq[k][w] = sqrt(phi0~_kw), fp64
__global__ void sqrt_phi0_kernel(const int32_t* __restrict__ Q, const int32_t* __restrict__ T, double beta,
                                 double vbeta, int V, int K, int Kp, double* __restrict__ sq) {
    const size_t n = (size_t)K * V;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(j / V), w = (int)(j % V);
        sq[j] = sqrt((beta + (double)Q[(size_t)w * Kp + k]) / (vbeta + (double)T[k]));
    }
}

// dist[k][k'] = sqrt(clamp(1 - sum_w sa[k][w] sb[k'][w], 0, 1)); 32 x 32 tile of
// (k, k') per block (256 threads, 4 outputs each), V in smem chunks of 32.
__global__ void __launch_bounds__(256) hellinger_kernel(const double* __restrict__ sa, const double* __restrict__ sb,
                                                        int K, int V, double* __restrict__ dist) {
    __shared__ double ta[32][33], tb[32][33];
    const int k0 = blockIdx.y * 32, kp0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;     // ty in [0, 8)
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int v0 = 0; v0 < V; v0 += 32) {
        for (int r = ty; r < 32; r += 8) {
            const int v = v0 + tx;
            ta[r][tx] = (k0 + r < K && v < V) ? sa[(size_t)(k0 + r) * V + v] : 0.0;
            tb[r][tx] = (kp0 + r < K && v < V) ? sb[(size_t)(kp0 + r) * V + v] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int v = 0; v < 32; ++v) {
            const double bv = tb[tx][v];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] += ta[ty + 8 * q][v] * bv;
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int k = k0 + ty + 8 * q, kp = kp0 + tx;
        if (k < K && kp < K) {
            double h2 = 1.0 - acc[q];
            h2 = h2 < 0.0 ? 0.0 : (h2 > 1.0 ? 1.0 : h2);
            dist[(size_t)k * K + kp] = sqrt(h2);
        }
    }
}

}  // namespace spdp
