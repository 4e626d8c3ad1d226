// spdp_token.cuh — the sweep's sample step for small K (K <= 64): one lane per token.
//
// Same method and same semantics as sample_kernel (wave snapshot, Alg.1 with
// the keep rule, Eqs. r0/r1, slot order j = 2k (r = 1), 2k+1 (r = 0), reading
// c10 draw), organised for few topics: at K <= 64 the chunk kernel spends most
// of its instructions on per-chunk and per-step overheads (lane groups, scans,
// hand-overs) that a token's K-topic work cannot amortise.  Here:
//   factor_kernel: for every (w, i) segment of the wave, the slot factor
//     F_k = F0_k + F1_k at the wave-start snapshot (Eqs. r0/r1 without the doc
//     term (alpha_ik + n_dk)) into a [segment][Kp] table (L2-resident);
//   token_kernel: one thread per token (tokens sorted by segment, so a warp's
//     factor-row loads are mostly broadcasts): Philox (a2), removal draw and
//     own-removal factors (a3), the doc-topic row in 4-topic blocks, masses
//     w_k = fma(n_dk, F_k, alpha_ik F_k) with the own topic replaced by its
//     after-removal mass (a4, a5), fp32 block sums with an fp64 prefix over
//     blocks, the block and then the topic where the prefix first exceeds
//     u * total, the r split by the exact r = 1 share (a6), and the count
//     deltas as one packed integer atomic per changed cell (a7).
// Every CDF boundary is an fp64 sum of fp32 block sums of 4 terms, as in the
// chunk kernel (inside the 1e-6 band of north_star (5)).
#pragma once
#include "spdp_device.cuh"

#ifndef SPDP_TOKEN_MINB
#define SPDP_TOKEN_MINB 4           // resident 256-thread blocks per SM the token kernel is compiled for
#endif

namespace spdp {

#ifndef SPDP_TOKEN_PRE
#define SPDP_TOKEN_PRE 0            // 1: factor_kernel also writes alpha F, the packed (m, t) and topic k's own-removal
                                    // factor parts per (run, k), shortening the token kernel's dependent-load chain;
                                    // B200: C2 0.165 vs 0.159 ms, C4 K = 20 0.276 vs 0.277 ms (the extra factor-table
                                    // writes cost what the shorter chain saves), so off
#endif

// F[r][k] and R1 (and, when the pointers are set, aF, MT, FR) for the runs (segments) [r0, r1) of one wave
__global__ void factor_kernel(const uint32_t* __restrict__ run_seg, uint32_t r0, uint32_t r1,
                              const int32_t* __restrict__ m, const int32_t* __restrict__ t,
                              const int32_t* __restrict__ Q, const int32_t* __restrict__ M,
                              const int32_t* __restrict__ Tt, const int32_t* __restrict__ T,
                              const float* __restrict__ disc, const float* __restrict__ conc,
                              const float2* __restrict__ tab, const uint64_t* __restrict__ tab_off, float beta,
                              float vbeta, int I, int K, int Kp, float* __restrict__ F, float* __restrict__ R1,
                              const float* __restrict__ alpha, float* __restrict__ aF, uint32_t* __restrict__ MT,
                              float4* __restrict__ FR) {
    const size_t n = (size_t)(r1 - r0) * Kp;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const uint32_t r = r0 + (uint32_t)(j / Kp);
        const int k = (int)(j % Kp);
        float Fk = 0.f, Rk = 0.f, al = 0.f;
        int mv = 0, tv = 0;
        float4 fr = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < K) {
            const uint32_t seg = run_seg[r];
            const int w = (int)(seg / (uint32_t)I), i = (int)(seg % (uint32_t)I);
            const size_t cell = (size_t)seg * Kp + k;
            mv = m[cell]; tv = t[cell];
            const int Mv = M[(size_t)i * Kp + k], Ttv = Tt[(size_t)i * Kp + k], Qv = Q[(size_t)w * Kp + k], Tv = T[k];
            const float2* tb = tab + tab_off[i];
            const float a = disc[i], b = conc[i];
            float F0, F1;
            slot_factors(Mv, Ttv, Qv, Tv, tb[tri(mv) + tv], a, b, beta, vbeta, F0, F1);
            Fk = F0 + F1;
            Rk = (F1 > 0.f) ? __fdiv_rn(F1, F0 + F1) : 0.f;     // exact r = 1 share of the slot pair
            al = alpha[(size_t)i * Kp + k];
            if (FR && mv > 0) {               // a token of topic k leaving this segment (Alg.1 lines 4-10)
                const int mm = mv - 1;
                slot_factors(Mv - 1, Ttv, Qv, Tv, tb[tri(mm) + min(tv, mm)], a, b, beta, vbeta, fr.x, fr.y);         // r_rem = 0
                slot_factors(Mv - 1, Ttv - 1, Qv - 1, Tv - 1, tb[tri(mm) + max(tv - 1, 0)], a, b, beta, vbeta, fr.z, fr.w);  // r_rem = 1
            }
        }
        F[(size_t)r * Kp + k] = Fk;
        R1[(size_t)r * Kp + k] = Rk;
        if (aF) aF[(size_t)r * Kp + k] = __fmul_rn(al, Fk);       // optional tables (token kernel with
        if (MT) MT[(size_t)r * Kp + k] = ((uint32_t)mv << 16) | (uint32_t)tv;   // SPDP_TOKEN_PRE; chunk
        if (FR) FR[(size_t)r * Kp + k] = fr;                      // kernel with factor tables)
    }
}

struct TokenArgs {
    const uint32_t* tok_doc;
    const uint32_t* tok_id;
    const uint32_t* tok_run;       // run (segment of the wave) of each sorted token
    const uint32_t* run_seg;       // segment w * I + i of each run
    const uint16_t* zr;
    uint16_t* zr_next;
    const float* F;                // [run][Kp]
    const float* R1;               // [run][Kp] r = 1 share F1 / F at the snapshot
    const float* aF;               // [run][Kp] alpha_ik F (SPDP_TOKEN_PRE)
    const uint32_t* MT;            // [run][Kp] snapshot m << 16 | t
    const float4* FR;              // [run][Kp] own-removal factor parts (F0, F1) for r_rem = 0, then r_rem = 1
    const void* n;                 // doc-topic rows (sigma layout of the chunk kernel)
    const int* sigma;              // [Kp] in-row position of topic k
    int bpos[32];                  // in-row position (float4 units) of 4-topic block B
    const int32_t *m, *t, *Q, *M, *Tt, *T;
    int32_t* dmt;                  // packed wave deltas dm * 2^16 + dt per cell
    const float* alpha;            // [I][Kp]
    const float *disc, *conc;
    const float2* tab;
    const uint64_t* tab_off;
    float beta, vbeta;
    int I, K, Kp;
    int Kn;                        // doc-topic row length
    uint32_t key0, key1;
    const uint32_t* sweep;
    uint32_t begin, end;           // sorted-token range of the wave
    unsigned long long* stats;
};


// NBK: 4-topic blocks of the topic range (K <= 4 NBK)
// NBK > 16 (K <= 128): the block sums live in shared memory [NBK][blockDim.x] instead of registers
template <int NBK, typename NT>
__global__ void __launch_bounds__(256, SPDP_TOKEN_MINB) token_kernel(TokenArgs A) {
    constexpr bool kSm = NBK > 16;
    extern __shared__ float s_tbs[];
    const int I = A.I, K = A.K, Kp = A.Kp;
    const int nbk = (K + 3) >> 2;
    const uint32_t sweep = *A.sweep;
    unsigned keeps = 0, moved = 0;
    for (uint32_t p = A.begin + blockIdx.x * blockDim.x + threadIdx.x; p < A.end; p += gridDim.x * blockDim.x) {
        const uint32_t run = A.tok_run[p];
        const uint32_t seg = A.run_seg[run];
        const int w = (int)(seg / (uint32_t)I), i = (int)(seg % (uint32_t)I);
        const uint32_t zr0 = A.zr[p];
        const uint32_t doc = A.tok_doc[p];              // issued with the record: the row address is ready early
        const int k0 = (int)(zr0 & 0x7FFFu);
        const uint4 x = philox(make_uint4(A.tok_id[p], sweep, 0u, 0u), A.key0, A.key1);      // a2
        const size_t cell0 = (size_t)seg * Kp + k0;
        int m0, t0;
        if constexpr (SPDP_TOKEN_PRE) {
            const uint32_t mt = A.MT[(size_t)run * Kp + k0];
            m0 = (int)(mt >> 16); t0 = (int)(mt & 0xFFFFu);
        } else {
            m0 = A.m[cell0]; t0 = A.t[cell0];
        }
        const int rrem = removal_draw(x.x, m0, t0);                                             // a3
        const bool keep = rrem && t0 == 1 && m0 > 1;                                             // reading c5
        int ks = k0, rs = 1;
        if (!keep) {
            float Fk0, R1k0;
            if constexpr (SPDP_TOKEN_PRE) {   // the factor kernel's own-removal parts for this r_rem
                const float4 fr = A.FR[(size_t)run * Kp + k0];
                const float x0 = rrem ? fr.z : fr.x, x1 = rrem ? fr.w : fr.y;
                Fk0 = x0 + x1;
                R1k0 = (x1 > 0.f) ? __fdiv_rn(x1, Fk0) : 0.f;
            } else {
                const float a = A.disc[i], b = A.conc[i];
                const float2* __restrict__ tab = A.tab + A.tab_off[i];
                const int32_t* Mi = A.M + (size_t)i * Kp;
                const int32_t* Tti = A.Tt + (size_t)i * Kp;
                const int32_t* Qw = A.Q + (size_t)w * Kp;
                removal_factors(rrem, m0, t0, Mi[k0], Tti[k0], Qw[k0], A.T[k0], tab, a, b, A.beta, A.vbeta, Fk0, R1k0);
            }
            const NT* nrow = reinterpret_cast<const NT*>(A.n) + (size_t)doc * A.Kn;
            const float* Frow = A.F + (size_t)run * Kp;
            const float* aFrow = A.aF + (size_t)run * Kp;
            const float* al = A.alpha + (size_t)i * Kp;
            // own topic: the after-removal mass replaces the snapshot mass (block sum + difference,
            // as the chunk kernel does)
            const float n0 = Row<NT>::load1(nrow + A.sigma[k0]);
            const float al0 = al[k0], F0k = Frow[k0];
            const float wold = SPDP_TOKEN_PRE ? __fmaf_rn(n0, F0k, aFrow[k0]) : __fmaf_rn(n0, F0k, __fmul_rn(al0, F0k));
            const float wnew = __fmaf_rn(n0 - 1.f, Fk0, __fmul_rn(al0, Fk0));
            const float dlt = wnew - wold;
            // a4/a5: masses in 4-topic blocks
            float bsr[kSm ? 1 : NBK];
#define BS(B) (*(kSm ? &s_tbs[(B) * blockDim.x + threadIdx.x] : &bsr[kSm ? 0 : (B)]))
            double total = 0.0;
#pragma unroll
            for (int B = 0; B < NBK; ++B) {
                BS(B) = 0.f;
                if (B < nbk) {
                    const float4 n4 = Row<NT>::load4(nrow + 4 * A.bpos[B]);
                    const float4 F4 = *reinterpret_cast<const float4*>(Frow + 4 * B);
                    float bsv;
                    if constexpr (SPDP_TOKEN_PRE) {
                        const float4 f4 = *reinterpret_cast<const float4*>(aFrow + 4 * B);
                        bsv = (__fmaf_rn(n4.x, F4.x, f4.x) + __fmaf_rn(n4.y, F4.y, f4.y)) +
                              (__fmaf_rn(n4.z, F4.z, f4.z) + __fmaf_rn(n4.w, F4.w, f4.w));
                    } else {
                        const float4 a4 = *reinterpret_cast<const float4*>(al + 4 * B);
                        bsv = (__fmaf_rn(n4.x, F4.x, __fmul_rn(a4.x, F4.x)) + __fmaf_rn(n4.y, F4.y, __fmul_rn(a4.y, F4.y))) +
                              (__fmaf_rn(n4.z, F4.z, __fmul_rn(a4.z, F4.z)) + __fmaf_rn(n4.w, F4.w, __fmul_rn(a4.w, F4.w)));
                    }
                    if ((k0 >> 2) == B) bsv += dlt;
                    BS(B) = bsv;
                    total += (double)bsv;
                }
            }
            // a6: target = u * total; the block, then the topic, where the prefix first exceeds it
            const double target = u53(x) * total;
            double run2 = 0.0, bbeg = 0.0, lastbeg = 0.0;
            int qs = -1, qlast = 0;
#pragma unroll
            for (int B = 0; B < NBK; ++B) {
                if (B < nbk) {
                    const float bsv = BS(B);
                    const double nxt = run2 + (double)bsv;
                    if (qs < 0 && nxt > target) { qs = B; bbeg = run2; }
                    if (bsv > 0.f) { qlast = B; lastbeg = run2; }
                    run2 = nxt;
                }
            }
#undef BS
            bool fb = qs < 0;
            if (fb) { qs = qlast; bbeg = lastbeg; }                                // rounding: last positive block
            int bq = 0;
#pragma unroll
            for (int B = 0; B < NBK; ++B) if (B == qs) bq = A.bpos[B];
            const float4 n4 = Row<NT>::load4(nrow + 4 * bq);
            const float4 F4 = *reinterpret_cast<const float4*>(Frow + 4 * qs);
            float wq[4];
            if constexpr (SPDP_TOKEN_PRE) {
                const float4 f4 = *reinterpret_cast<const float4*>(aFrow + 4 * qs);
                wq[0] = __fmaf_rn(n4.x, F4.x, f4.x); wq[1] = __fmaf_rn(n4.y, F4.y, f4.y);
                wq[2] = __fmaf_rn(n4.z, F4.z, f4.z); wq[3] = __fmaf_rn(n4.w, F4.w, f4.w);
            } else {
                const float4 a4 = *reinterpret_cast<const float4*>(al + 4 * qs);
                wq[0] = __fmaf_rn(n4.x, F4.x, __fmul_rn(a4.x, F4.x)); wq[1] = __fmaf_rn(n4.y, F4.y, __fmul_rn(a4.y, F4.y));
                wq[2] = __fmaf_rn(n4.z, F4.z, __fmul_rn(a4.z, F4.z)); wq[3] = __fmaf_rn(n4.w, F4.w, __fmul_rn(a4.w, F4.w));
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) if (4 * qs + e == k0) wq[e] = wnew;
            double r3 = bbeg, bes = bbeg, blast = bbeg;
            int es = -1, elast = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const double nxt = r3 + (double)wq[e];
                if (es < 0 && !fb && nxt > target) { es = e; bes = r3; }
                if (wq[e] > 0.f) { elast = e; blast = r3; }
                r3 = nxt;
            }
            if (es < 0) { fb = true; es = elast; bes = blast; }                     // rounding: last positive topic
            float wsel = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) if (e == es) wsel = wq[e];
            ks = 4 * qs + es;
            const bool own = (ks == k0);
            const float R1s = own ? R1k0 : A.R1[(size_t)run * Kp + ks];           // r = 1 share of ks
            const float w1 = wsel * R1s;
            if (!fb) rs = (bes + (double)w1 > target) ? 1 : 0;
            else {                                                                  // last positive slot
                const int ms = own ? m0 - 1 : (SPDP_TOKEN_PRE ? (int)(A.MT[(size_t)run * Kp + ks] >> 16) : A.m[(size_t)seg * Kp + ks]);
                rs = (ms > 0) ? 0 : 1;
            }
            // a7: packed deltas (dm * 2^16 + dt) of the two cells
            atomicAdd(A.dmt + cell0, -65536 - rrem);
            atomicAdd(A.dmt + (size_t)seg * Kp + ks, 65536 + rs);
            moved += (ks != k0);
        } else {
            ++keeps;
        }
        A.zr_next[p] = (uint16_t)(ks | (rs << 15));
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

// per sorted token: its run index (runs = segments of the waves, in plan order)
__global__ void token_run_kernel(const uint32_t* __restrict__ run_off, const uint32_t* __restrict__ run_len,
                                 uint32_t R, uint32_t* __restrict__ tok_run) {
    for (uint32_t r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; r < R; r += gridDim.x * (blockDim.x / 32)) {
        const uint32_t o = run_off[r], l = run_len[r];
        for (uint32_t j = threadIdx.x & 31; j < l; j += 32) tok_run[o + j] = r;
    }
}

}  // namespace spdp
