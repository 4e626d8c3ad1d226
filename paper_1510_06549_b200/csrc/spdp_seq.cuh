// spdp_seq.cuh — W = 0 test mode: the exact sequential sampler (Algorithm 1,
// PAPER.md:1698-1727, with the keep rule of reading c5) on the device.
//
// SURVEY §8(b) "W = 0 = fully sequential (test mode: one token per wave)" and
// §8(c) "sampler (mode S) ... The GPU runs W = 0 mode in one persistent CTA".
// One warp walks the tokens in canonical order; every token is removed, weighed
// against the current (exact, immediately updated) counts and re-inserted before
// the next one starts, so no snapshot, delta or clamp is involved.  Lanes split
// the K topics in tiles of 32; the 2K slot masses of the token go to shared
// memory; the draw is j* = min{ j : CDF_j > u * total } over the paper's slot
// order j = 2k (r = 1), 2k + 1 (r = 0) (Alg.4, reading c10), with an
// fp64 prefix over fp32 masses.  Throughput is not the point (one warp on the
// whole GPU): this is the device's exact chain for the enumeration tests.
#pragma once
#include "spdp_device.cuh"

namespace spdp {

struct SeqArgs {
    const int32_t* group;      // canonical token triples [N]
    const int32_t* word;
    const uint32_t* pos;       // canonical id -> sorted position (zr, tok_doc)
    int64_t N;
    int V;
    int nsweeps;
    int64_t* codes;            // [nsweeps] state code after each sweep (tiny corpora), or null
    int tbase;
};

template <typename NT>
__global__ void __launch_bounds__(32, 1) seq_kernel(SweepArgs A, SeqArgs S) {
    extern __shared__ __align__(16) float2 wsl[];   // [K] (w1, w0) of the current token
    const int lane = threadIdx.x;
    const int I = A.I, K = A.K, Kp = A.Kp;
    NT* __restrict__ n = reinterpret_cast<NT*>(A.n);
    unsigned long long keeps = 0, moved = 0;
    const uint32_t sweep0 = *A.sweep;
    for (int s = 0; s < S.nsweeps; ++s) {
        const uint32_t sweep = sweep0 + (uint32_t)s;
        for (int64_t p = 0; p < S.N; ++p) {
            const int i = S.group[p], w = S.word[p];
            const uint32_t q = S.pos[p];
            const uint32_t zr0 = A.zr[q];
            const int k0 = (int)(zr0 & 0x7FFFu);
            const size_t row = ((size_t)w * I + i) * Kp;
            const size_t noff = (size_t)A.tok_doc[q] * A.Kn;
            const int mc = A.m[row + k0], tc = A.t[row + k0];
            const uint4 x = philox(make_uint4((uint32_t)p, sweep, 0u, 0u), A.key0, A.key1);   // a2
            const int rrem = removal_draw(x.x, mc, tc);                                        // a3, Alg.1 l.3
            if (rrem && tc == 1 && mc > 1) {                                                   // keep (c5)
                if (lane == 0) A.zr[q] = (uint16_t)(k0 | kRBit);
                ++keeps;
                __syncwarp();
                continue;
            }
            const float a = A.disc[i], b = A.conc[i];
            const float2* __restrict__ tab = A.tab + A.tab_off[i];
            // weights with the token's own contribution removed (Alg.1 l.4-10 folded in), Eqs. r0/r1
            double tot = 0.0;
            for (int kb = 0; kb < K; kb += 32) {
                const int k = kb + lane;
                float w1 = 0.f, w0 = 0.f;
                if (k < K) {
                    const int own = (k == k0);
                    const int ro = own & rrem;
                    const int mk = A.m[row + k] - own, tk = A.t[row + k] - ro;
                    float F0, F1;
                    slot_factors(A.M[(size_t)i * Kp + k] - own, A.Tt[(size_t)i * Kp + k] - ro,
                                 A.Q[(size_t)w * Kp + k] - ro, A.T[k] - ro, tab[tri(mk) + tk], a, b, A.beta, A.vbeta,
                                 F0, F1);
                    const float base = A.alpha[(size_t)i * Kp + k] + ((float)Row<NT>::get(n + noff + A.sigma[k]) - (float)own);
                    w1 = base * F1;
                    w0 = base * F0;
                    wsl[k] = make_float2(w1, w0);
                }
                double v = (double)w1 + (double)w0;
#pragma unroll
                for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                tot += v;
            }
            __syncwarp();
            const double target = u53(x) * tot;
            // first slot whose inclusive prefix exceeds the target
            double run = 0.0;
            int js = -1, jlast = -1;
            for (int kb = 0; kb < K && js < 0; kb += 32) {
                const int k = kb + lane;
                const float2 ws = (k < K) ? wsl[k] : make_float2(0.f, 0.f);
                const double own = (double)ws.x + (double)ws.y;
                double incl = own;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const double y = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += y;
                }
                const double before = run + incl - own;
                int cand = -1;
                if (before + (double)ws.x > target && ws.x > 0.f) cand = 2 * k;
                else if (before + own > target && ws.y > 0.f) cand = 2 * k + 1;
                const unsigned hit = __ballot_sync(0xffffffffu, cand >= 0);
                if (hit) js = __shfl_sync(0xffffffffu, cand, __ffs(hit) - 1);
                const unsigned pos1 = __ballot_sync(0xffffffffu, ws.x > 0.f || ws.y > 0.f);
                if (pos1) {
                    const int hl = 31 - __clz(pos1);
                    const int lj = ws.y > 0.f ? 2 * k + 1 : 2 * k;
                    jlast = __shfl_sync(0xffffffffu, lj, hl);
                }
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (js < 0) js = jlast;                                   // rounding: the last positive slot
            const int kn = js >> 1, rn = (js & 1) ? 0 : 1;
            if (lane == 0) {                                          // Alg.1 l.4-10 and 18-22, exact
                const size_t c0 = row + k0, c1 = row + kn;
                Row<NT>::store(n + noff + A.sigma[k0], Row<NT>::get(n + noff + A.sigma[k0]) - 1);
                A.m[c0] -= 1; A.M[(size_t)i * Kp + k0] -= 1;
                if (rrem) { A.t[c0] -= 1; A.Tt[(size_t)i * Kp + k0] -= 1; A.Q[(size_t)w * Kp + k0] -= 1; A.T[k0] -= 1; }
                Row<NT>::store(n + noff + A.sigma[kn], Row<NT>::get(n + noff + A.sigma[kn]) + 1);
                A.m[c1] += 1; A.M[(size_t)i * Kp + kn] += 1;
                if (rn) { A.t[c1] += 1; A.Tt[(size_t)i * Kp + kn] += 1; A.Q[(size_t)w * Kp + kn] += 1; A.T[kn] += 1; }
                A.zr[q] = (uint16_t)(kn | (rn << 15));
            }
            moved += (kn != k0);
            __syncwarp();
        }
        if (S.codes && lane == 0) {   // state code, the oracle's or_chain_codes order: z_p K^p, then t cells (i, w, k)
            long long code = 0, mul = 1;
            for (int64_t p = 0; p < S.N; ++p) { code += mul * (long long)(A.zr[S.pos[p]] & 0x7FFFu); mul *= K; }
            long long tcode = 0, tm = 1;
            for (int i = 0; i < I; ++i)
                for (int w = 0; w < S.V; ++w)
                    for (int k = 0; k < K; ++k) { tcode += tm * (long long)A.t[((size_t)w * I + i) * Kp + k]; tm *= S.tbase; }
            S.codes[s] = code + mul * tcode;
        }
        __syncwarp();
    }
    if (lane == 0) {
        *const_cast<uint32_t*>(A.sweep) = sweep0 + (uint32_t)S.nsweeps;
        A.stats[0] += keeps;
        A.stats[1] += moved;
    }
}

}  // namespace spdp
