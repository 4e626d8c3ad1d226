// spdp_sparse.cuh — NEXT-4: the sweep with sparse non-identity
// transformation matrices P^i (Eq. r1 P:1688-1693 with
// p_{i,w,v}, Alg.1 lines 6-9 and 19-21 with the table sources).
//
// State on top of the identity-P sampler: for every (w, i) segment the row
// P^i[w] = entries e (source word v_e, weight p_e), q[e][k] = tables of
// (i, k, w) whose source is v_e, t = sum_e q, and the shadow counts become
// Q[v][k] = sum_{i,w} q_{ikwv}.  Readings: c24 correction of q
// after a wave, c25 initial sources, c26 the removed table's source.
//
//   sp_factor_kernel  — per (segment of the wave, k): F_k = F0 + F1 with
//       F1 = A1 C1 G_k sum_e p_e (beta + Q[v_e][k]) and the r = 1 share F1 / F;
//   sp_token_kernel   — one thread per token (any K, two passes over the
//       4-topic blocks, no per-topic registers): Philox, removal draw, the
//       removed table's source (integer rule on the snapshot q), the own
//       topic's after-removal factors, topic and r by the block prefix, then
//       the source entry by the r = 1 masses p_e (beta + Q[v_e][k]) in entry
//       order (the oracle's slot order: (k, r=1, e_0..e_{S-1}), (k, r=0));
//       deltas dm[seg][k] and dq[e][k] with integer atomics;
//   sp_merge_kernel   — per touched segment: m += dm, q += dq, the c24
//       correction, t = sum q, Q and the sums updated by the net changes.
#pragma once
#include "spdp_device.cuh"

namespace spdp {

struct SparseP {
    const uint32_t* sptr;    // [S_segs + 1] entries of segment seg = w * I + i
    const int32_t* pv;       // [E] source word
    const float* pp;         // [E] weight p_{i,w,v}
    const int32_t* best;     // [segs] entry of largest p (first on ties)
    int32_t* q;              // [E][Kp]
    int32_t* dq;             // [E][Kp] wave deltas
};

// F1 of Eq. r1 with the sum over the segment's sources in place of (beta + Q)
__device__ __forceinline__ void slot_factors_sum(int M, int Tt, float sumpq, int Tk, float2 A, float a, float b,
                                                 float vbeta, float& F0, float& F1) {
    const float C0 = __frcp_rn(b + (float)M);
    F0 = A.x * C0;
    F1 = A.y * ((b + a * (float)Tt) * C0) * __fdividef(sumpq, vbeta + (float)Tk);
}

// sum_e p_e (beta + Q[v_e][k] - [v_e == vrem]) over the entries [e0, e1)
__device__ __forceinline__ float source_sum(const SparseP& P, const int32_t* Q, int Kp, uint32_t e0, uint32_t e1, int k,
                                            float beta, int vrem) {
    float s = 0.f;
    for (uint32_t e = e0; e < e1; ++e) {
        const int v = P.pv[e];
        s += P.pp[e] * (beta + (float)(Q[(size_t)v * Kp + k] - (v == vrem ? 1 : 0)));
    }
    return s;
}

__global__ void sp_factor_kernel(SparseP P, const uint32_t* __restrict__ run_seg, uint32_t r0, uint32_t r1,
                                 const int32_t* __restrict__ m, const int32_t* __restrict__ t,
                                 const int32_t* __restrict__ Q, const int32_t* __restrict__ M,
                                 const int32_t* __restrict__ Tt, const int32_t* __restrict__ T,
                                 const float* __restrict__ disc, const float* __restrict__ conc,
                                 const float2* __restrict__ tab, const uint64_t* __restrict__ tab_off, float beta,
                                 float vbeta, int I, int K, int Kp, float* __restrict__ F, float* __restrict__ R1) {
    const size_t n = (size_t)(r1 - r0) * Kp;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const uint32_t r = r0 + (uint32_t)(j / Kp);
        const int k = (int)(j % Kp);
        float Fk = 0.f, Rk = 0.f;
        if (k < K) {
            const uint32_t seg = run_seg[r];
            const int i = (int)(seg % (uint32_t)I);
            const size_t cell = (size_t)seg * Kp + k;
            const int mv = m[cell], tv = t[cell];
            const float sumpq = source_sum(P, Q, Kp, P.sptr[seg], P.sptr[seg + 1], k, beta, -1);
            float F0, F1;
            slot_factors_sum(M[(size_t)i * Kp + k], Tt[(size_t)i * Kp + k], sumpq, T[k], tab[tab_off[i] + tri(mv) + tv],
                             disc[i], conc[i], vbeta, F0, F1);
            Fk = F0 + F1;
            Rk = (F1 > 0.f) ? __fdiv_rn(F1, F0 + F1) : 0.f;
        }
        F[(size_t)r * Kp + k] = Fk;
        R1[(size_t)r * Kp + k] = Rk;
    }
}

struct SpTokenArgs {
    const uint32_t* tok_doc;
    const uint32_t* tok_id;
    const uint32_t* tok_run;
    const uint32_t* run_seg;
    const uint16_t* zr;
    uint16_t* zr_next;
    int16_t* src;                  // [Nloc] chosen source entry within the row (r = 1), -1 for r = 0 / kept
    const float* F;
    const float* R1;
    const void* n;
    const int* sigma;
    int bpos[256];                 // in-row position (float4 units) of 4-topic block B (K <= 1024)
    const int32_t *m, *t, *Q, *M, *Tt, *T;
    int32_t* dm;                   // [segs][Kp] wave deltas of m
    const float* alpha;
    const float *disc, *conc;
    const float2* tab;
    const uint64_t* tab_off;
    float beta, vbeta;
    int I, K, Kp;
    int Kn;                        // doc-topic row length
    uint32_t key0, key1;
    const uint32_t* sweep;
    uint32_t begin, end;
    unsigned long long* stats;
    SparseP P;
};

template <typename NT>
__device__ __forceinline__ float sp_block_sum(const NT* nrow, const float* Frow, const float* al, int bpos, int B,
                                              float4* n4o = nullptr, float4* F4o = nullptr, float4* a4o = nullptr) {
    const float4 n4 = Row<NT>::load4(nrow + 4 * bpos);
    const float4 F4 = *reinterpret_cast<const float4*>(Frow + 4 * B);
    const float4 a4 = *reinterpret_cast<const float4*>(al + 4 * B);
    if (n4o) { *n4o = n4; *F4o = F4; *a4o = a4; }
    return (__fmaf_rn(n4.x, F4.x, __fmul_rn(a4.x, F4.x)) + __fmaf_rn(n4.y, F4.y, __fmul_rn(a4.y, F4.y))) +
           (__fmaf_rn(n4.z, F4.z, __fmul_rn(a4.z, F4.z)) + __fmaf_rn(n4.w, F4.w, __fmul_rn(a4.w, F4.w)));
}

constexpr int kSpSmemBlocks = 32;   // block sums of up to 32 4-topic blocks per thread in shared memory

template <typename NT>
__global__ void __launch_bounds__(256) sp_token_kernel(SpTokenArgs A) {
    extern __shared__ float s_bs[];   // [kSpSmemBlocks][blockDim.x] (only when K <= 128)
    const int I = A.I, K = A.K, Kp = A.Kp;
    const int nbk = (K + 3) >> 2;
    const uint32_t sweep = *A.sweep;
    unsigned keeps = 0, moved = 0;
    for (uint32_t p = A.begin + blockIdx.x * blockDim.x + threadIdx.x; p < A.end; p += gridDim.x * blockDim.x) {
        const uint32_t run = A.tok_run[p];
        const uint32_t seg = A.run_seg[run];
        const int w = (int)(seg / (uint32_t)I), i = (int)(seg % (uint32_t)I);
        (void)w;
        const uint32_t e0 = A.P.sptr[seg], e1 = A.P.sptr[seg + 1];
        const uint32_t zr0 = A.zr[p];
        const int k0 = (int)(zr0 & 0x7FFFu);
        const uint4 x = philox(make_uint4(A.tok_id[p], sweep, 0u, 0u), A.key0, A.key1);
        const size_t cell0 = (size_t)seg * Kp + k0;
        const int m0 = A.m[cell0], t0 = A.t[cell0];
        const int rrem = removal_draw(x.x, m0, t0);
        const bool keep = rrem && t0 == 1 && m0 > 1;
        int ks = k0, rs = 1, es = -1;
        if (!keep) {
            // the removed table's source: j = floor(x3 t / 2^32) in the cumulative q (reading c26)
            uint32_t erem = e0;
            if (rrem) {
                const long long jj = (long long)(((unsigned long long)x.w * (unsigned long long)t0) >> 32);
                long long cum = 0;
                erem = e1 - 1;
                for (uint32_t e = e0; e < e1; ++e) {
                    cum += A.P.q[(size_t)e * Kp + k0];
                    if (cum > jj) { erem = e; break; }
                }
            }
            const int vrem = rrem ? A.P.pv[erem] : -1;
            const float a = A.disc[i], b = A.conc[i];
            const float2* __restrict__ tab = A.tab + A.tab_off[i];
            const int32_t* Mi = A.M + (size_t)i * Kp;
            const int32_t* Tti = A.Tt + (size_t)i * Kp;
            // own topic after the removal (Alg.1 lines 4-10 with the source)
            float Fk0 = 0.f, R1k0 = 0.f;
            if (m0 > 0) {
                const int mm = m0 - 1, tt = rrem ? max(t0 - 1, 0) : min(t0, mm);
                float x0, x1;
                slot_factors_sum(Mi[k0] - 1, Tti[k0] - rrem, source_sum(A.P, A.Q, Kp, e0, e1, k0, A.beta, vrem),
                                 A.T[k0] - rrem, tab[tri(mm) + tt], a, b, A.vbeta, x0, x1);
                Fk0 = x0 + x1;
                R1k0 = (x1 > 0.f) ? __fdiv_rn(x1, Fk0) : 0.f;
            }
            const NT* nrow = reinterpret_cast<const NT*>(A.n) + (size_t)A.tok_doc[p] * A.Kn;
            const float* Frow = A.F + (size_t)run * Kp;
            const float* al = A.alpha + (size_t)i * Kp;
            const float n0 = Row<NT>::load1(nrow + A.sigma[k0]);
            const float al0 = al[k0], F0k = Frow[k0];
            const float wold = __fmaf_rn(n0, F0k, __fmul_rn(al0, F0k));
            const float wnew = __fmaf_rn(n0 - 1.f, Fk0, __fmul_rn(al0, Fk0));
            const float dlt = wnew - wold;
            // pass 1: total, last positive block (block sums kept in shared memory for K <= 128)
            const bool keep_bs = nbk <= kSpSmemBlocks;
            double total = 0.0, lastbeg = 0.0;
            int qlast = 0;
            for (int B = 0; B < nbk; ++B) {
                float bs = sp_block_sum<NT>(nrow, Frow, al, A.bpos[B], B);
                if ((k0 >> 2) == B) bs += dlt;
                if (keep_bs) s_bs[B * blockDim.x + threadIdx.x] = bs;
                if (bs > 0.f) { qlast = B; lastbeg = total; }
                total += (double)bs;
            }
            const double target = u53(x) * total;
            // pass 2: the block where the prefix first exceeds the target
            double run2 = 0.0, bbeg = 0.0;
            int qs = -1;
            for (int B = 0; B < nbk; ++B) {
                float bs;
                if (keep_bs) bs = s_bs[B * blockDim.x + threadIdx.x];
                else {
                    bs = sp_block_sum<NT>(nrow, Frow, al, A.bpos[B], B);
                    if ((k0 >> 2) == B) bs += dlt;
                }
                const double nxt = run2 + (double)bs;
                if (nxt > target) { qs = B; bbeg = run2; break; }
                run2 = nxt;
            }
            bool fb = qs < 0;
            if (fb) { qs = qlast; bbeg = lastbeg; }
            float4 n4, F4, a4;
            sp_block_sum<NT>(nrow, Frow, al, A.bpos[qs], qs, &n4, &F4, &a4);
            float wq[4] = {__fmaf_rn(n4.x, F4.x, __fmul_rn(a4.x, F4.x)), __fmaf_rn(n4.y, F4.y, __fmul_rn(a4.y, F4.y)),
                           __fmaf_rn(n4.z, F4.z, __fmul_rn(a4.z, F4.z)), __fmaf_rn(n4.w, F4.w, __fmul_rn(a4.w, F4.w))};
#pragma unroll
            for (int e = 0; e < 4; ++e) if (4 * qs + e == k0) wq[e] = wnew;
            double r3 = bbeg, bes = bbeg, blast = bbeg;
            int esl = -1, elast = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double nxt = r3 + (double)wq[e];
                if (esl < 0 && !fb && nxt > target) { esl = e; bes = r3; }
                if (wq[e] > 0.f) { elast = e; blast = r3; }
                r3 = nxt;
            }
            if (esl < 0) { fb = true; esl = elast; bes = blast; }
            float wsel = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) if (e == esl) wsel = wq[e];
            ks = 4 * qs + esl;
            const bool own = (ks == k0);
            const float R1s = own ? R1k0 : A.R1[(size_t)run * Kp + ks];
            const float w1 = wsel * R1s;
            if (!fb && bes + (double)w1 > target) {
                // r = 1: the source entry, slots in entry order with masses w1 * c_e / sum c
                rs = 1;
                const int vr = own ? vrem : -1;
                const float csum = source_sum(A.P, A.Q, Kp, e0, e1, ks, A.beta, vr);
                double cb = bes;
                es = (int)(e1 - 1 - e0);
                for (uint32_t e = e0; e < e1; ++e) {
                    const int v = A.P.pv[e];
                    const float ce = A.P.pp[e] * (A.beta + (float)(A.Q[(size_t)v * Kp + ks] - (v == vr ? 1 : 0)));
                    cb += (double)(w1 * (ce / csum));
                    if (cb > target) { es = (int)(e - e0); break; }
                }
            } else if (!fb) {
                rs = 0;
            } else {                                                   // last positive slot
                const int ms = own ? m0 - 1 : A.m[(size_t)seg * Kp + ks];
                rs = (ms > 0) ? 0 : 1;
                if (rs) es = (int)(e1 - 1 - e0);
            }
            atomicAdd(A.dm + cell0, -1);
            atomicAdd(A.dm + (size_t)seg * Kp + ks, 1);
            if (rrem) atomicAdd(A.P.dq + (size_t)erem * Kp + k0, -1);
            if (rs) atomicAdd(A.P.dq + (size_t)(e0 + es) * Kp + ks, 1);
            moved += (ks != k0);
        } else {
            ++keeps;
        }
        A.zr_next[p] = (uint16_t)(ks | (rs << 15));
        A.src[p] = (int16_t)(keep ? -1 : es);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        keeps += __shfl_xor_sync(0xffffffffu, keeps, off);
        moved += __shfl_xor_sync(0xffffffffu, moved, off);
    }
    if ((threadIdx.x & 31) == 0 && (keeps | moved)) {
        atomicAdd(A.stats + 0, (unsigned long long)keeps);
        atomicAdd(A.stats + 1, (unsigned long long)moved);
    }
}

// End of wave, per touched segment (one warp, lanes over k): m += dm, q += dq,
// correction (reading c24), t = sum q, net changes into Q[v][k], M, Tt, T.
__global__ void sp_merge_kernel(SparseP P, const uint32_t* __restrict__ segs, int nseg, int32_t* __restrict__ m,
                                int32_t* __restrict__ t, int32_t* __restrict__ dm, int32_t* __restrict__ Q,
                                int32_t* __restrict__ M, int32_t* __restrict__ Tt, int32_t* __restrict__ T, int I, int K,
                                int Kp, unsigned long long* __restrict__ stats, int32_t* __restrict__ Dm = nullptr,
                                int32_t* __restrict__ Dq = nullptr) {
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    unsigned clamped = 0;
    for (int j = blockIdx.x * wpb + (threadIdx.x >> 5); j < nseg; j += gridDim.x * wpb) {
        const uint32_t seg = segs[j];
        const int i = (int)(seg % (uint32_t)I);
        const uint32_t e0 = P.sptr[seg], e1 = P.sptr[seg + 1];
        const int eb = P.best[seg];
        for (int k = lane; k < K; k += 32) {
            const size_t c = (size_t)seg * Kp + k;
            bool any = dm[c] != 0;
            for (uint32_t e = e0; e < e1; ++e) any |= P.dq[(size_t)e * Kp + k] != 0;
            if (!any) continue;
            const int mold = m[c], told = t[c];
            const int mv = mold + dm[c];
            dm[c] = 0;
            m[c] = mv;
            int tv = 0, changed = 0;
            for (uint32_t e = e0; e < e1; ++e) {                       // q += dq, q >= 0 (old q kept in dq)
                const size_t qe = (size_t)e * Kp + k;
                const int old = P.q[qe];
                int x = old + P.dq[qe];
                P.dq[qe] = old;
                if (x < 0) { x = 0; changed = 1; }
                P.q[qe] = x;
                tv += x;
            }
            if (mv == 0) {
                for (uint32_t e = e0; e < e1; ++e) { const size_t qe = (size_t)e * Kp + k; if (P.q[qe]) { P.q[qe] = 0; changed = 1; } }
                tv = 0;
            } else if (tv == 0) {
                P.q[(size_t)eb * Kp + k] = 1; tv = 1; changed = 1;
            } else {
                while (tv > mv) {                                      // the largest q (first on ties) loses one
                    uint32_t eb2 = e0;
                    for (uint32_t e = e0; e < e1; ++e) if (P.q[(size_t)e * Kp + k] > P.q[(size_t)eb2 * Kp + k]) eb2 = e;
                    P.q[(size_t)eb2 * Kp + k] -= 1; --tv; changed = 1;
                }
            }
            for (uint32_t e = e0; e < e1; ++e) {                       // net source changes into Q[v][k]
                const size_t qe = (size_t)e * Kp + k;
                const int d = P.q[qe] - P.dq[qe];
                P.dq[qe] = 0;
                if (d) {
                    atomicAdd(Q + (size_t)P.pv[e] * Kp + k, d);
                    if (Dq) Dq[qe] += d;                                 // net change since the sweep start (ranks)
                }
            }
            clamped += changed;
            t[c] = tv;
            if (Dm && mv != mold) Dm[c] += mv - mold;
            if (mv != mold) atomicAdd(M + (size_t)i * Kp + k, mv - mold);
            if (tv != told) { atomicAdd(Tt + (size_t)i * Kp + k, tv - told); atomicAdd(T + k, tv - told); }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) clamped += __shfl_xor_sync(0xffffffffu, clamped, off);
    if (lane == 0 && clamped) atomicAdd(stats + 2, (unsigned long long)clamped);
}

// Q[v][k] = sum over entries with source v of q[e][k] (after zeroing Q): the shadow counts of the sparse state
__global__ void sp_shadow_kernel(SparseP P, uint32_t E, int K, int Kp, int32_t* __restrict__ Q) {
    const size_t n = (size_t)E * Kp;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(j % Kp);
        const uint32_t e = (uint32_t)(j / Kp);
        const int x = P.q[j];
        if (k < K && x) atomicAdd(Q + (size_t)P.pv[e] * Kp + k, x);
    }
}

// initial sources (reading c25): every table of a cell on the segment's largest-p entry
__global__ void sp_init_q_kernel(SparseP P, const int32_t* __restrict__ t, uint32_t segs, int Kp) {
    const size_t n = (size_t)segs * Kp;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const uint32_t seg = (uint32_t)(j / Kp);
        const int k = (int)(j % Kp);
        P.q[(size_t)P.best[seg] * Kp + k] = t[j];
    }
}

}  // namespace spdp

namespace spdp {
// multi-rank merge with sources: m, q = local - Dloc + Dsum (Dloc: this rank's net change of m (cells) then
// of q (E x Kp); Dsum: the sum over ranks), correction c24, t = sum q; Dloc zeroed.  Sums and Q afterwards.
__global__ void sp_exchange_merge_kernel(SparseP P, uint32_t segs, int32_t* __restrict__ m, int32_t* __restrict__ t,
                                         int32_t* __restrict__ Dloc, const int32_t* __restrict__ Dsum, size_t cells,
                                         int K, int Kp, unsigned long long* __restrict__ stats) {
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    int32_t* dlq = Dloc + cells;
    const int32_t* dsq = Dsum + cells;
    unsigned clamped = 0;
    for (uint32_t seg = blockIdx.x * wpb + (threadIdx.x >> 5); seg < segs; seg += gridDim.x * wpb) {
        const uint32_t e0 = P.sptr[seg], e1 = P.sptr[seg + 1];
        const int eb = P.best[seg];
        for (int k = lane; k < K; k += 32) {
            const size_t c = (size_t)seg * Kp + k;
            bool any = Dloc[c] != 0 || Dsum[c] != 0;
            for (uint32_t e = e0; e < e1; ++e) any |= dlq[(size_t)e * Kp + k] != 0 || dsq[(size_t)e * Kp + k] != 0;
            if (!any) continue;
            const int mv = m[c] - Dloc[c] + Dsum[c];
            Dloc[c] = 0;
            m[c] = mv;
            int tv = 0, changed = 0;
            for (uint32_t e = e0; e < e1; ++e) {
                const size_t qe = (size_t)e * Kp + k;
                int x = P.q[qe] - dlq[qe] + dsq[qe];
                dlq[qe] = 0;
                if (x < 0) { x = 0; changed = 1; }
                P.q[qe] = x;
                tv += x;
            }
            if (mv == 0) {
                for (uint32_t e = e0; e < e1; ++e) { const size_t qe = (size_t)e * Kp + k; if (P.q[qe]) { P.q[qe] = 0; changed = 1; } }
                tv = 0;
            } else if (tv == 0) {
                P.q[(size_t)eb * Kp + k] = 1; tv = 1; changed = 1;
            } else {
                while (tv > mv) {
                    uint32_t eb2 = e0;
                    for (uint32_t e = e0; e < e1; ++e) if (P.q[(size_t)e * Kp + k] > P.q[(size_t)eb2 * Kp + k]) eb2 = e;
                    P.q[(size_t)eb2 * Kp + k] -= 1; --tv; changed = 1;
                }
            }
            clamped += changed;
            t[c] = tv;
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) clamped += __shfl_xor_sync(0xffffffffu, clamped, off);
    if (lane == 0 && clamped) atomicAdd(stats + 2, (unsigned long long)clamped);
}
}  // namespace spdp

namespace spdp {
// log p(W, Z, T, Q) source terms per block: sum over cells of ln t! - sum_e ln q_e! + sum_e q_e ln p_e (fp64)
__global__ void sp_source_terms_kernel(SparseP P, const double* __restrict__ pp64, uint32_t segs, int K, int Kp,
                                       const int32_t* __restrict__ t, double* __restrict__ partial) {
    __shared__ double sh[32];
    double acc = 0.0;
    const size_t n = (size_t)segs * Kp;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(j % Kp);
        if (k >= K) continue;
        const uint32_t seg = (uint32_t)(j / Kp);
        double v = lgamma((double)t[j] + 1.0);
        for (uint32_t e = P.sptr[seg]; e < P.sptr[seg + 1]; ++e) {
            const int qv = P.q[(size_t)e * Kp + k];
            v += -lgamma((double)qv + 1.0) + (double)qv * log(pp64[e]);
        }
        acc += v;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
        partial[blockIdx.x] = s;
    }
}
}  // namespace spdp
