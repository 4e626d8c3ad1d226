// spdp_sprows.cuh — the sample step on sparse doc-topic rows (HBM-bound, large-K configurations).
//
// Same method and same draw as sample_kernel (wave snapshot; Alg.1 with the keep
// rule; Eqs. r0/r1; slot order j = 2k (r = 1), 2k + 1 (r = 0); j* = min{ j :
// CDF_j > u * total }, reading c10), computed from a document's NONZERO counts:
// a document of L_d tokens touches at most min(L_d, K) topics, so at K = 200 with
// 62-token documents (C5) or K = 1000 with 125-token documents (C4) most of a dense
// row is zeros.  With F_k the segment's slot factor and PA(k) = sum_{k' <= k}
// alpha_ik' F_k' (a per-chunk fp64 prefix in shared memory), the topic-level CDF is
//     C(k) = PA(k) + NS(k),   NS(k) = sum over the document's entries k_e <= k of n_e F_{k_e},
// with the token's own topic k0 entering NS with its after-removal mass
// (n0 - 1) Fk0 + alpha (Fk0 - F_k0) (Alg.1 lines 4-10).  C is increasing; its first
// crossing of u * total is found entry by entry (LPT lanes per token, contiguous
// entry ranges, one fp64 group scan), then inside the gap before the crossing entry
// by binary search on PA (lane = token).  The r split uses the exact r = 1 share of
// the chosen topic, as the dense kernel does.  Entries (k | n << 16, topic order) are
// rebuilt from the dense rows after every sweep (rows_to_entries_kernel); the dense
// rows stay the canonical state for every other consumer.
#pragma once
#include "spdp_device.cuh"

namespace spdp {

constexpr int kSpWarps = 4;

template <int KSPAN>
struct SpRowSmem {
    double PA[KSPAN];       // inclusive prefix over k of alpha_ik F_k (fp64)
    float F[KSPAN];         // F0 + F1 at the snapshot
    float R1[KSPAN];        // r = 1 share F1 / F at the snapshot
    uint32_t mt[KSPAN];     // snapshot m << 16 | t
    int dmt[KSPAN];         // chunk deltas dm * 2^16 + dt
    double target[32];      // hand-over, one per token of the batch
    double base[32];        // NS before the winner lane's range (or all of it: tail gap)
    int lo[32];             // first topic after the previous lane's last entry
    uint32_t e0[32], e1[32];// the winner lane's entry range (empty: the tail gap [lo, K))
};

template <int LPT, int KSPAN>
constexpr size_t sprow_smem_bytes() { return kSpWarps * sizeof(SpRowSmem<KSPAN>); }

template <int LPT, int KSPAN>
__global__ void __launch_bounds__(kSpWarps * 32) sample_sprows_kernel(SweepArgs A) {
    constexpr int TPW = 32 / LPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    SpRowSmem<KSPAN>& S = reinterpret_cast<SpRowSmem<KSPAN>*>(smem_raw)[wid];
    const int I = A.I, K = A.K, Kp = A.Kp;
    unsigned keeps = 0, moved = 0;
    const int g = lane / LPT, gl = lane % LPT;
    const unsigned gmask = (LPT == 32) ? 0xffffffffu : (((1u << LPT) - 1u) << (g * LPT));
    const uint32_t* __restrict__ ent = A.ent;

  for (;;) {
    uint32_t cc = 0;
    if (lane == 0) cc = atomicAdd(A.work, 1u);
    const int c = (int)__shfl_sync(0xffffffffu, cc, 0);
    if (c >= A.nchunks) break;
    __syncwarp();
    const uint32_t seg = A.chunk_seg[c];
    const int w = (int)(seg / (uint32_t)I), i = (int)(seg % (uint32_t)I);
    const size_t row = (size_t)seg * Kp;
    const float a = A.disc[i], b = A.conc[i];
    const float2* __restrict__ tab = A.tab + A.tab_off[i];
    const int32_t* __restrict__ Mi = A.M + (size_t)i * Kp;
    const int32_t* __restrict__ Tti = A.Tt + (size_t)i * Kp;
    const int32_t* __restrict__ Qw = A.Q + (size_t)w * Kp;
    const float* __restrict__ alpha_i = A.alpha + (size_t)i * Kp;
    const uint32_t start = A.chunk_start[c], end = A.chunk_end[c];

    // ---- prologue: slot factors, r = 1 shares, alpha F into PA (prefix below)
    {   // topics in groups of PG per lane: the group's count loads, then its table loads, then the math
        constexpr int PER = (KSPAN + 31) / 32;
        constexpr int PG = SPDP_PRO_GROUP < PER ? SPDP_PRO_GROUP : PER;
#pragma unroll 1
        for (int k0g = 0; k0g < PER; k0g += PG) {
            int mv[PG], tv[PG], Mv[PG], Ttv[PG], Qv[PG], Tv[PG];
            float al[PG];
            float2 tb[PG];
#pragma unroll
            for (int j = 0; j < PG; ++j) {
                const int k = lane + 32 * (k0g + j);
                mv[j] = tv[j] = Mv[j] = Ttv[j] = Qv[j] = Tv[j] = 0;
                al[j] = 0.f;
                if (k < K) {
                    mv[j] = A.m[row + k]; tv[j] = A.t[row + k]; al[j] = alpha_i[k];
                    Mv[j] = Mi[k]; Ttv[j] = Tti[k]; Qv[j] = Qw[k]; Tv[j] = A.T[k];
                }
            }
#pragma unroll
            for (int j = 0; j < PG; ++j) {
                const int k = lane + 32 * (k0g + j);
                tb[j] = (k < K) ? tab[tri(mv[j]) + tv[j]] : make_float2(0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < PG; ++j) {
                const int k = lane + 32 * (k0g + j);
                float F0 = 0.f, F1 = 0.f;
                if (k < K) slot_factors(Mv[j], Ttv[j], Qv[j], Tv[j], tb[j], a, b, A.beta, A.vbeta, F0, F1);
                const float Fk = F0 + F1;
                S.F[k] = Fk;
                S.R1[k] = (F1 > 0.f) ? __fdiv_rn(F1, Fk) : 0.f;
                S.PA[k] = (double)__fmul_rn(al[j], Fk);
                S.mt[k] = ((uint32_t)mv[j] << 16) | (uint32_t)tv[j];
                S.dmt[k] = 0;
            }
        }
    }
    __syncwarp();
    {   // PA: lane-contiguous blocks of KSPAN/32, local prefix + warp exclusive scan (fp64)
        constexpr int B = KSPAN / 32;
        double run = 0.0;
#pragma unroll
        for (int j = 0; j < B; ++j) { run += S.PA[lane * B + j]; S.PA[lane * B + j] = run; }
        double incl = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += y;
        }
        const double ex = incl - run;
#pragma unroll
        for (int j = 0; j < B; ++j) S.PA[lane * B + j] += ex;
    }
    __syncwarp();
    const double PAtot = S.PA[K - 1];
    const uint32_t sweep = *A.sweep;

    for (uint32_t b0 = start; b0 < end; b0 += 32) {
        const uint32_t nb = min(32u, end - b0);
        // ======== phase 1: lane = token
        const bool mine = (uint32_t)lane < nb;
        const uint32_t p = b0 + lane;
        uint32_t zr0 = 0, x0 = 0;
        uint2 di = make_uint2(0u, 0u);
        double u = 0.0;
        if (mine) {
            di = A.dinfo[A.tok_doc[p]];                      // {first entry, nonzero topics}
            zr0 = A.zr[p];
        }
        const int k0 = (int)(zr0 & 0x7FFFu);
        const uint32_t mt0 = S.mt[k0];
        const int m0 = (int)(mt0 >> 16), t0 = (int)(mt0 & 0xFFFFu);
        const int mm0 = max(m0 - 1, 0);
        float2 tab_r1 = make_float2(0.f, 0.f), tab_r0 = make_float2(0.f, 0.f);
        int Mk0 = 0, Ttk0 = 0, Qk0 = 0, Tk0 = 0;
        if (mine) {
            tab_r1 = tab[tri(mm0) + max(t0 - 1, 0)];
            tab_r0 = tab[tri(mm0) + min(t0, mm0)];
            Mk0 = Mi[k0]; Ttk0 = Tti[k0]; Qk0 = Qw[k0]; Tk0 = A.T[k0];
            const uint4 x = philox(make_uint4(A.tok_id[p], sweep, 0u, 0u), A.key0, A.key1);    // a2
            x0 = x.x;
            u = u53(x);
            if (A.prefetch_rows) {   // the document's entries towards L2 (1-2 lines)
                const char* e0 = reinterpret_cast<const char*>(ent + di.x);
                const char* e1 = reinterpret_cast<const char*>(ent + di.x + di.y);
                for (const char* q = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(e0) & ~(uintptr_t)127); q < e1; q += 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
            }
        }
        const int rrem = removal_draw(x0, m0, t0);                                             // a3
        const bool keep = rrem && t0 == 1 && m0 > 1;                                             // reading c5
        float Fk0 = 0.f, R1k0 = 0.f;
        if (mine) removal_factors_pre(rrem, m0, Mk0, Ttk0, Qk0, Tk0, tab_r1, tab_r0, a, b, A.beta, A.vbeta, Fk0, R1k0);
        const float al0 = alpha_i[k0];
        const float corr = __fmul_rn(al0, Fk0 - S.F[k0]);    // the alpha part of topic k0's change

        // ======== phase 2: LPT lanes per token, contiguous entry ranges.  Each lane sums its
        // entries' NS terms in fp32; one fp64 group scan; the first lane whose range ends above the
        // target, C(last k of its range) > u * total, holds the crossing (in its range or in the gap
        // before it): it hands over its entry range and the NS before it.
        for (uint32_t s0 = 0; s0 < nb; s0 += TPW) {
            const uint32_t src = (s0 + g) & 31;
            const bool valid = s0 + g < nb;
            const int sk0 = __shfl_sync(0xffffffffu, k0, src);
            const float sFk0 = __shfl_sync(0xffffffffu, Fk0, src);
            const float scorr = __shfl_sync(0xffffffffu, corr, src);
            const double su = __shfl_sync(0xffffffffu, u, src);
            const uint32_t ptr = __shfl_sync(0xffffffffu, di.x, src);
            const uint32_t snnz = __shfl_sync(0xffffffffu, di.y, src);   // every lane takes part in the shuffle
            const int nnz = valid ? (int)snnz : 0;
            const int cnt = (nnz + LPT - 1) / LPT;
            const int j0 = min(gl * cnt, nnz), j1 = min(j0 + cnt, nnz);
            float lsum = 0.f;
            int lastk = -1;
            for (int j = j0; j < j1; ++j) {
                const uint32_t e = ent[ptr + j];
                const int k = (int)(e & 0xFFFFu);
                const float n = (float)(e >> 16);
                lsum += (k == sk0) ? __fmaf_rn(n - 1.f, sFk0, scorr) : __fmul_rn(n, S.F[k]);
                lastk = k;
            }
            double incl = (double)lsum;
#pragma unroll
            for (int off = 1; off < LPT; off <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, incl, off, LPT);
                if (gl >= off) incl += y;
            }
            double excl = __shfl_up_sync(0xffffffffu, incl, 1, LPT);
            if (gl == 0) excl = 0.0;
            int prevk = __shfl_up_sync(0xffffffffu, lastk, 1, LPT);    // last entry topic before my range
            if (gl == 0) prevk = -1;
            const double nstot = __shfl_sync(0xffffffffu, incl, LPT - 1, LPT);
            const double target = su * (PAtot + nstot);
            const bool crossed = (j1 > j0) && (S.PA[lastk] + (excl + (double)lsum) > target);
            const unsigned hit = __ballot_sync(0xffffffffu, crossed) & gmask;
            // the entry ranges are contiguous: the lane owning the last entry gives the tail gap's start
            const int last_gl = nnz > 0 ? (nnz - 1) / max(cnt, 1) : 0;
            const int tail_lastk = __shfl_sync(0xffffffffu, lastk, last_gl, LPT);
            const int winner = hit ? (__ffs(hit) - 1) : g * LPT;
            // (ranges fill from lane 0, so the winner's predecessor lanes are full and prevk is exact)
            if (lane == winner && valid) {
                S.target[src] = target;
                if (hit) { S.base[src] = excl; S.lo[src] = prevk + 1; S.e0[src] = ptr + j0; S.e1[src] = ptr + j1; }
                else { S.base[src] = nstot; S.lo[src] = tail_lastk + 1; S.e0[src] = 0; S.e1[src] = 0; }   // tail gap
            }
        }
        __syncwarp();

        // ======== phase 3: lane = token; walk the winner's entries (the gap before each, then the
        // entry), binary search inside the gap that holds the crossing; r split
        if (mine) {
            int ks = k0, rs = 1;
            if (!keep) {
                const double target = S.target[lane], base = S.base[lane];
                int lo = S.lo[lane];
                const uint32_t e0 = S.e0[lane], e1 = S.e1[lane];
                float run32 = 0.f;
                double cum = base;                         // C(k) - PA(k) on the current gap: base + NS so far
                int found = -1, hi = K;
                float hterm = 0.f;
                for (uint32_t j = e0; j < e1 && found < 0; ++j) {
                    const uint32_t e = ent[j];
                    const int k = (int)(e & 0xFFFFu);
                    const float n = (float)(e >> 16);
                    const float tm = (k == k0) ? __fmaf_rn(n - 1.f, Fk0, corr) : __fmul_rn(n, S.F[k]);
                    if (k > lo && S.PA[k - 1] + cum > target) { hi = k; found = 0; break; }   // in the gap [lo, k)
                    run32 += tm;
                    const double cnext = base + (double)run32;
                    if (S.PA[k] + cnext > target) { found = 1; ks = k; hterm = tm; break; }   // the entry itself
                    cum = cnext;
                    lo = k + 1;
                }
                if (found != 1) {                          // first k in [lo, hi) with PA(k) + cum > target
                    int L = lo, H = hi;
                    while (L < H) {
                        const int mid = (L + H) >> 1;
                        if (S.PA[mid] + cum > target) H = mid; else L = mid + 1;
                    }
                    ks = L;
                }
                if (ks < K) {
                    const double before = (ks > 0 ? S.PA[ks - 1] : 0.0) + cum;
                    const float mass = __fmaf_rn(alpha_i[ks], S.F[ks], found == 1 ? hterm : 0.f);
                    const float R1s = (ks == k0) ? R1k0 : S.R1[ks];
                    rs = (before + (double)__fmul_rn(mass, R1s) > target) ? 1 : 0;
                } else {                                    // rounding: the last positive slot
                    ks = K - 1;
                    rs = (((ks == k0) ? m0 - 1 : (int)(S.mt[ks] >> 16)) > 0) ? 0 : 1;
                }
            }
            A.zr_next[p] = (uint16_t)(ks | (rs << 15));                                         // a7
            if (keep) ++keeps;
            else {
                atomicAdd(&S.dmt[k0], -65536 - rrem);
                atomicAdd(&S.dmt[ks], 65536 + rs);
                moved += (ks != k0);
            }
        }
        __syncwarp();
    }
    __syncwarp();
    for (int k = lane; k < K; k += 32) {
        const int x = S.dmt[k];
        if (x) {
            const int dtv = (int)(short)(x & 0xFFFF);
            const int dmv = (x - dtv) >> 16;
            if (A.packed_dmt) atomicAdd(A.dm + row + k, x);
            else {
                if (dmv) atomicAdd(A.dm + row + k, dmv);
                if (dtv) atomicAdd(A.dt + row + k, dtv);
            }
        }
    }
    __syncwarp();
  }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        keeps += __shfl_xor_sync(0xffffffffu, keeps, off);
        moved += __shfl_xor_sync(0xffffffffu, moved, off);
    }
    if (lane == 0 && (keeps | moved)) {
        atomicAdd(A.stats + 0, (unsigned long long)keeps);
        atomicAdd(A.stats + 1, (unsigned long long)moved);
    }
}

// After every W = 1 sweep (and at state installation): a document's dense row (sigma order) ->
// its nonzero counts as entries k | n << 16 in topic order at ent[cap_ptr[d] ...]; dinfo[d] =
// {first entry, count}.  One warp per document.
template <typename NT>
__global__ void rows_to_entries_kernel(const NT* __restrict__ n, const int* __restrict__ sigma, int D, int K, int Kn,
                                       const uint32_t* __restrict__ cap_ptr, uint32_t* __restrict__ ent,
                                       uint2* __restrict__ dinfo) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    for (int d = blockIdx.x * wpb + (threadIdx.x >> 5); d < D; d += gridDim.x * wpb) {
        const NT* row = n + (size_t)d * Kn;
        const uint32_t e0 = cap_ptr[d];
        uint32_t cnt = 0;
        for (int kb = 0; kb < K; kb += 32) {
            const int k = kb + lane;
            const int v = (k < K) ? Row<NT>::get(row + sigma[k]) : 0;
            const unsigned bal = __ballot_sync(0xffffffffu, v > 0);
            if (v > 0) ent[e0 + cnt + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)k | ((uint32_t)v << 16);
            cnt += __popc(bal);
        }
        if (lane == 0) dinfo[d] = make_uint2(e0, cnt);
    }
}

}  // namespace spdp
