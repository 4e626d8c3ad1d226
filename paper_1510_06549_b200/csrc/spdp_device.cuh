// spdp_device.cuh — sm_100a kernels of the SPDP Gibbs sweep.
//
// Notation follows PAPER.md §2.4.5: z topic, r table indicator, n_{dk}
// doc-topic counts, m_{ikw} customers and t_{ikw} tables of dish w in
// restaurant (group i, topic k), Q_{kw} = sum_i t_{ikw} shadow counts (identity
// P), M_{ik} = m_{ik.}, Tt_{ik} = t_{ik.}, T_k = sum_w Q_{kw}.
//
// Layout in HBM: every count row is padded to Kp = round_up(K, 4)
// int32 so rows are 16-byte aligned for vector loads.
//   n  [D_local][Kn]      doc-topic, this rank's documents (unit layout below, Kn = LA * KPL)
//   m,t[V][I][Kp]          word-major: the rows of one (w, i) segment are adjacent
//   Q  [V][Kp]             shadow counts, word-major
//   M,Tt [I][Kp], T [Kp]   marginal sums
//   tokens, sorted by (wave, w, i, doc): doc (u32 local), id (u32 canonical), zr (u16 z | r<<15)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace spdp {

constexpr int kWarps = 4;          // warps per block of the sample kernel
#ifndef SPDP_BLOCK_ALPHA
#define SPDP_BLOCK_ALPHA 1         // dense pass: block sum = sum_k n_k F_k + (sum_k alpha_k F_k), the latter per chunk
#endif
#ifndef SPDP_ROW_PIPELINE
#define SPDP_ROW_PIPELINE 1        // dense pass: issue the next step's row loads once this step's block sums are formed
#endif
#ifndef SPDP_PRE_TAB
#define SPDP_PRE_TAB 1             // own-removal table entries (both r_rem candidates) loaded before the Philox rounds
#endif
#ifndef SPDP_PREFETCH_NEXT
#define SPDP_PREFETCH_NEXT 0       // also prefetch the next batch's doc-topic rows
#endif
#ifndef SPDP_PRO_GROUP
#define SPDP_PRO_GROUP 4           // chunk prologue: topics per lane whose loads are issued together (B200, final
#endif                             // kernels, 1 -> 4: C3 0.997 -> 0.974 ms, C3 W = 2 1.431 -> 1.385, C5 26.64 -> 26.39;
                                   // before the unit layout 1 was best at C3, 1.053 vs 1.102 ms)
#ifndef SPDP_PRO_GROUP_1024
#define SPDP_PRO_GROUP_1024 8      // ... at 32x32 (B200, K = 1000: 4 -> 8 topics 3.82 -> 3.61 ms; at 16x32 8 loses 3.5 %)
#endif
#ifndef SPDP_SMEM_R1
#define SPDP_SMEM_R1 1             // chunk prologue keeps every topic's r = 1 share in shared memory (KSPAN <= 256)
#endif
#ifndef SPDP_NARROW_FULL
#define SPDP_NARROW_FULL 1         // uint8/uint16 rows at 8x32: block alpha sums and row pipelining as at 4 blocks/SM
#endif
#ifndef SPDP_NARROW_PRETAB
#define SPDP_NARROW_PRETAB 1       // ... and the own-removal inputs before the Philox rounds (C5 at 6 blocks: 26.38 -> 25.91 ms)
#endif
#ifndef SPDP_BULK_PREFETCH
#define SPDP_BULK_PREFETCH 0       // 1: exact-byte cp.async.bulk.prefetch.L2 of the next batch instead of this batch's
                                   // 128-B lines (B200, C5: 37.4 vs 34.7 ms per sweep with uint8 rows: fewer bytes, but
                                   // the kernel is issue- and latency-bound and the extra record loads cost more)
#endif
#ifndef SPDP_PREFETCH_AHEAD
#define SPDP_PREFETCH_AHEAD 1      // bulk prefetch: batches of 32 tokens ahead of the one being sampled
#endif
#ifndef SPDP_STAGE_NEXT
#define SPDP_STAGE_NEXT 0          // 1: the next chunk's counts and Stirling entries staged during this chunk (B200: C3 +5 %, C5 +3 %)
#endif
#ifndef SPDP_F_SMEM
#define SPDP_F_SMEM 2              // dense pass reads F_k from shared memory instead of KPL registers per lane:
#endif                             // 0 never, 1 always, 2 at 8x32 (B200, C5: 31.7 -> 27.5 ms per sweep with 6 blocks
                                   // per SM; C3 (4x32) +4 %, K = 300 (16x32) +7 %: those keep F in registers)
#ifndef SPDP_MINB_8X32
#define SPDP_MINB_8X32 6           // 8x32 (F in shared memory): <= 80 registers, 6 resident blocks (B200, C5: 5 blocks
#endif                             // 30.1 ms, 6 blocks 27.5 ms, 7 blocks 29.3 ms per sweep)
#ifndef SPDP_MINB
#define SPDP_MINB 4                // resident blocks per SM the sample kernel is compiled for
#endif
constexpr uint32_t kRBit = 0x8000u;

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based RNG (Salmon et al. 2011), keyed by the seed, counter
// (token, sweep, 0, 0) — DESIGN.md reading c11.
__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}
// 53-bit uniform in [0,1): x1 * 2^21 + (x2 >> 11), exact in fp64.
__device__ __forceinline__ double u53(uint4 x) {
    return fma((double)x.y, 2097152.0, (double)(x.z >> 11)) * (1.0 / 9007199254740992.0);
}
// Removal indicator r ~ Bernoulli(t/m) (Alg.1 line 3), exact in integers.
__device__ __forceinline__ int removal_draw(uint32_t x0, int m, int t) {
    return ((uint64_t)x0 * (uint64_t)(uint32_t)m) < ((uint64_t)(uint32_t)t << 32);
}

__device__ __forceinline__ uint64_t tri(int m) { return (uint64_t)m * (uint64_t)(m + 1) / 2; }

// Pull the bytes [p, p + bytes) into L2 with one bulk (TMA-unit) prefetch: 16-byte granularity, so a
// row costs its own sectors and no more (a 128-B line prefetch per line over-fetches ~25 % on 400-B rows).
__device__ __forceinline__ void prefetch_bytes_l2(const void* p, uint32_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uintptr_t lo = a & ~(uintptr_t)15, hi = (a + bytes + 15) & ~(uintptr_t)15;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
}

// ---------------------------------------------------------------- Stirling ratio table
// A0(m,t) = (m-t+1)/(m+1) * S^{m+1}_t / S^m_t      (Eq. r0)
// A1(m,t) = (t+1)/(m+1)   * S^{m+1}_{t+1} / S^m_t  (Eq. r1)
// for 0 <= t <= m <= mmax, stored as float2 at tri(m) + t.  Built row by row
// in fp64 from q_N(M) = S^N_{M+1} / S^N_M (1 <= M <= N, q_N(N) = 0), which the
// recursion S^{N+1}_M = S^N_{M-1} + (N - M a) S^N_M turns into
//   q_{N+1}(M) = (1 + (N - (M+1) a) q_N(M)) / (1/q_N(M-1) + N - M a),  2 <= M <= N
//   q_{N+1}(1) = (1 + (N - 2a) q_N(1)) / (N - a)
// and then A0(m,t) = (m-t+1)/(m+1) * (1/q_m(t-1) + m - t a) (t >= 2),
// A0(m,1) = (m - a) m/(m+1), A1(m,t) = (t+1)/(m+1) * (1 + (m - (t+1) a) q_m(t)).
// No logarithms and no overflow: every quantity is a bounded ratio.
// One block per distinct discount; q rows ping-pong in global scratch.
__global__ void build_ratio_table(float2* __restrict__ tab, double* __restrict__ scratch, int mmax, double a) {
    double* q0 = scratch;                  // row N
    double* q1 = scratch + (mmax + 2);     // row N+1
    // row m = 0: A0(0,0) = 0, A1(0,0) = 1
    if (threadIdx.x == 0) {
        tab[0] = make_float2(0.f, 1.f);
        q0[1] = 0.0;                        // q_1(1) = 0 (S^1_2 = 0)
    }
    __syncthreads();
    for (int N = 1; N <= mmax; ++N) {
        // emit row m = N from q_N
        const double inv = 1.0 / (double)(N + 1);
        for (int t = threadIdx.x; t <= N; t += blockDim.x) {
            float A0, A1;
            if (t == 0) { A0 = 0.f; A1 = 0.f; }   // t = 0 < m is not a valid state
            else {
                const double s0 = (t == 1) ? ((double)N - a) : (1.0 / q0[t - 1] + (double)N - (double)t * a);
                A0 = (float)((double)(N - t + 1) * inv * s0);
                A1 = (float)((double)(t + 1) * inv * (1.0 + ((double)N - (double)(t + 1) * a) * q0[t]));
            }
            tab[tri(N) + t] = make_float2(A0, A1);
        }
        if (N == mmax) break;
        // q_{N+1} from q_N
        for (int M = threadIdx.x + 1; M <= N + 1; M += blockDim.x) {
            double v;
            if (M == N + 1) v = 0.0;
            else if (M == 1) v = (1.0 + ((double)N - 2.0 * a) * q0[1]) / ((double)N - a);
            else v = (1.0 + ((double)N - (double)(M + 1) * a) * q0[M]) / (1.0 / q0[M - 1] + (double)N - (double)M * a);
            q1[M] = v;
        }
        __syncthreads();
        double* tmp = q0; q0 = q1; q1 = tmp;
    }
}

// ---------------------------------------------------------------- shared weight factor
// Per (group i, topic k, word w) factor of the 2K weights, with the doc term
// (alpha_ik + n_dk) left out:
//   F0 = A0(m,t) / (b + M)                                         (Eq. r0)
//   F1 = A1(m,t) (b + a Tt) / (b + M) * (beta + Q) / (V beta + T)  (Eq. r1)
__device__ __forceinline__ void slot_factors(int M, int Tt, int Qv, int Tk, float2 A, float a, float b,
                                             float beta, float vbeta, float& F0, float& F1) {
    const float C0 = __frcp_rn(b + (float)M);
    F0 = A.x * C0;
    F1 = A.y * ((b + a * (float)Tt) * C0) * __fdividef(beta + (float)Qv, vbeta + (float)Tk);
}

// Topic k0's factors after the token's own removal (Alg.1 lines 4-10): the
// customer leaves (m-1, M-1) and, when r_rem = 1, its table too (t-1, Tt-1, Q-1, T-1).
// Returns F = F0 + F1 and the r = 1 share F1 / F.
__device__ __forceinline__ void removal_factors(int rrem, int mv, int tv, int Mv, int Ttv, int Qv, int Tv,
                                                const float2* __restrict__ tab, float a, float b, float beta,
                                                float vbeta, float& Fsum, float& R1) {
    float x0 = 0.f, x1 = 0.f;
    if (mv > 0) {
        const int mm = mv - 1;
        if (rrem) slot_factors(Mv - 1, Ttv - 1, Qv - 1, Tv - 1, tab[tri(mm) + max(tv - 1, 0)], a, b, beta, vbeta, x0, x1);
        else slot_factors(Mv - 1, Ttv, Qv, Tv, tab[tri(mm) + min(tv, mm)], a, b, beta, vbeta, x0, x1);
    }
    Fsum = x0 + x1;
    R1 = (x1 > 0.f) ? __fdiv_rn(x1, Fsum) : 0.f;
}

// removal_factors with both candidate table entries already loaded (issued before the token's
// Philox, so the table latency overlaps it): A_r1 at (m-1, max(t-1, 0)), A_r0 at (m-1, min(t, m-1)).
__device__ __forceinline__ void removal_factors_pre(int rrem, int mv, int Mv, int Ttv, int Qv, int Tv, float2 A_r1,
                                                    float2 A_r0, float a, float b, float beta, float vbeta,
                                                    float& Fsum, float& R1) {
    float x0 = 0.f, x1 = 0.f;
    if (mv > 0) {
        if (rrem) slot_factors(Mv - 1, Ttv - 1, Qv - 1, Tv - 1, A_r1, a, b, beta, vbeta, x0, x1);
        else slot_factors(Mv - 1, Ttv, Qv, Tv, A_r0, a, b, beta, vbeta, x0, x1);
    }
    Fsum = x0 + x1;
    R1 = (x1 > 0.f) ? __fdiv_rn(x1, Fsum) : 0.f;
}

// ---------------------------------------------------------------- doc-topic row element
// Doc-topic counts are stored either as exact-integer fp32 (rows that live in
// L2) or as uint16 (half the bytes when the rows stream from HBM; n_dk <= L_d < 2^16).
template <typename NT>
struct Row;
// Coherent loads for the async mode (NEXT-2): the counts change while the
// kernel runs, so they are read with ld.relaxed.gpu (L2, never the
// non-coherent path of __ldg).
__device__ __forceinline__ int ld_relaxed(const int32_t* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_relaxed_f4(const float* p) {
    float4 v;
    asm volatile("ld.relaxed.gpu.global.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_relaxed_f(const float* p) {
    float v;
    asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_relaxed_u2(const void* p) {
    uint2 v;
    asm volatile("ld.relaxed.gpu.global.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned short ld_relaxed_u16(const uint16_t* p) {
    unsigned short v;
    asm volatile("ld.relaxed.gpu.global.b16 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
}
// SPDP_ASYNC_WEAK_ROWS: the async mode reads doc-topic rows with plain (weak, L1-cacheable) loads.
// The paper's scheme reads the global counts without synchronisation while other threads update
// them ("spinlocks or semaphores ... totally optional"); a weak load may return a
// stale value, which the scheme tolerates by design.  0: coherent ld.relaxed.gpu (L2) instead.
#ifndef SPDP_ASYNC_WEAK_ROWS
#define SPDP_ASYNC_WEAK_ROWS 1
#endif
constexpr bool kAsyncWeakRows = SPDP_ASYNC_WEAK_ROWS != 0;
__device__ __forceinline__ float4 ld_weak_f4(const float* p) {
    float4 v;
    asm("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_weak_u2(const void* p) {
    uint2 v;
    asm("ld.global.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_weak(const int32_t* p) {
    int v;
    asm("ld.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ int ld_weak_or_relaxed(const void* p) {
    return kAsyncWeakRows ? ld_weak(reinterpret_cast<const int32_t*>(p)) : ld_relaxed(reinterpret_cast<const int32_t*>(p));
}

template <bool AS>
__device__ __forceinline__ int ldc(const int32_t* p) {   // count read: snapshot (wave mode) or live (async)
    if constexpr (AS) return kAsyncWeakRows ? ld_weak(p) : ld_relaxed(p);
    else return *p;
}

// The marginal counts of topic k that a token's factors read: M_ik, Tt_ik, Q_kw, T_k.  In the
// async mode they are live and may be transiently out of range (another chunk's changes land
// cell by cell), so the local copy is corrected into the range the segment's own (clamped)
// cell (m, t) implies (Alg.4 "correct local counts copied ... to ensure they are in valid
// range"): M >= m, Tt >= t, Q >= t, T >= Q.  Wave mode reads a consistent snapshot: no-op.
template <bool AS>
__device__ __forceinline__ void load_sums(const int32_t* Mi, const int32_t* Tti, const int32_t* Qw, const int32_t* T,
                                          int k, int mv, int tv, int& Mv, int& Ttv, int& Qv, int& Tv) {
    Mv = ldc<AS>(Mi + k); Ttv = ldc<AS>(Tti + k); Qv = ldc<AS>(Qw + k); Tv = ldc<AS>(T + k);
    if constexpr (AS) { Mv = max(Mv, mv); Ttv = max(Ttv, tv); Qv = max(Qv, tv); Tv = max(Tv, Qv); }
}

template <>
struct Row<float> {
    // raw block of 4 counts as loaded (converted to fp32 at use: narrow rows keep fewer registers live)
    using raw_t = float4;
    __device__ __forceinline__ static raw_t load_raw(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
    __device__ __forceinline__ static raw_t load_raw_live(const float* p) { return load4_live(p); }
    __device__ __forceinline__ static float4 cvt(raw_t v) { return v; }
    __device__ __forceinline__ static raw_t zero_raw() { return make_float4(0.f, 0.f, 0.f, 0.f); }
    __device__ __forceinline__ static float4 load4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
    __device__ __forceinline__ static float4 load4_live(const float* p) {
        if constexpr (kAsyncWeakRows) return ld_weak_f4(p);
        else return ld_relaxed_f4(p);
    }
    __device__ __forceinline__ static float load1_live(const float* p) { return ld_relaxed_f(p); }
    __device__ __forceinline__ static float load1(const float* p) { return __ldg(p); }
    __device__ __forceinline__ static void add(float* base, size_t idx, int d) { atomicAdd(base + idx, (float)d); }
    __device__ __forceinline__ static void store(float* p, int v) { *p = (float)v; }
    __device__ __forceinline__ static void store4(float* p, int a, int b, int c, int d) {
        *reinterpret_cast<float4*>(p) = make_float4((float)a, (float)b, (float)c, (float)d);
    }
    __device__ __forceinline__ static int get(const float* p) { return (int)*p; }
};
#ifdef SPDP_CVT_I2F
__device__ __forceinline__ float u16lo(uint32_t x) { return __uint2float_rn(x & 0xFFFFu); }   // I2F.U16
__device__ __forceinline__ float u16hi(uint32_t x) { return __uint2float_rn(x >> 16); }       // I2F.U16 .H1
#else
// exact u16 -> f32 on the full-rate pipes: 2^23 + x as a bit pattern, minus 2^23
__device__ __forceinline__ float u16lo(uint32_t x) { return __int_as_float((int)__byte_perm(x, 0x4B000000u, 0x7610)) - 8388608.f; }
__device__ __forceinline__ float u16hi(uint32_t x) { return __int_as_float((int)__byte_perm(x, 0x4B000000u, 0x7632)) - 8388608.f; }
#endif
template <>
struct Row<uint16_t> {
    using raw_t = uint2;
    __device__ __forceinline__ static raw_t load_raw(const uint16_t* p) { return __ldg(reinterpret_cast<const uint2*>(p)); }
    __device__ __forceinline__ static raw_t load_raw_live(const uint16_t* p) {
        return kAsyncWeakRows ? ld_weak_u2(p) : ld_relaxed_u2(p);
    }
    __device__ __forceinline__ static float4 cvt(raw_t v) { return make_float4(u16lo(v.x), u16hi(v.x), u16lo(v.y), u16hi(v.y)); }
    __device__ __forceinline__ static raw_t zero_raw() { return make_uint2(0u, 0u); }
    __device__ __forceinline__ static float4 load4(const uint16_t* p) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
        return make_float4(u16lo(v.x), u16hi(v.x), u16lo(v.y), u16hi(v.y));
    }
    __device__ __forceinline__ static float4 load4_live(const uint16_t* p) {
        const uint2 v = kAsyncWeakRows ? ld_weak_u2(p) : ld_relaxed_u2(p);
        return make_float4(u16lo(v.x), u16hi(v.x), u16lo(v.y), u16hi(v.y));
    }
    __device__ __forceinline__ static float load1_live(const uint16_t* p) { return (float)ld_relaxed_u16(p); }
    __device__ __forceinline__ static float load1(const uint16_t* p) { return (float)__ldg(p); }
    // +-1 on one half of the containing 32-bit word (a half never leaves [0, L_d], no carry)
    __device__ __forceinline__ static void add(uint16_t* base, size_t idx, int d) {
        atomicAdd(reinterpret_cast<unsigned int*>(base) + (idx >> 1), (unsigned int)d << ((idx & 1) * 16));
    }
    __device__ __forceinline__ static void store(uint16_t* p, int v) { *p = (uint16_t)v; }
    __device__ __forceinline__ static void store4(uint16_t* p, int a, int b, int c, int d) {
        *reinterpret_cast<uint2*>(p) = make_uint2((uint32_t)a | ((uint32_t)b << 16), (uint32_t)c | ((uint32_t)d << 16));
    }
    __device__ __forceinline__ static int get(const uint16_t* p) { return (int)*p; }
};

// uint8 counts (every document < 256 tokens): a quarter of the fp32 bytes for HBM-resident rows.
// Exact u8 -> f32 on the full-rate pipes, as for uint16: byte j into 2^23 + x, minus 2^23.
__device__ __forceinline__ float u8at(uint32_t x, uint32_t j) {
    return __int_as_float((int)__byte_perm(x, 0x4B000000u, 0x7440u | j)) - 8388608.f;
}
template <>
struct Row<uint8_t> {
    using raw_t = uint32_t;
    __device__ __forceinline__ static raw_t load_raw(const uint8_t* p) { return __ldg(reinterpret_cast<const unsigned int*>(p)); }
    __device__ __forceinline__ static raw_t load_raw_live(const uint8_t* p) { return (uint32_t)ld_weak_or_relaxed(p); }
    __device__ __forceinline__ static float4 cvt(raw_t v) { return make_float4(u8at(v, 0), u8at(v, 1), u8at(v, 2), u8at(v, 3)); }
    __device__ __forceinline__ static raw_t zero_raw() { return 0u; }
    __device__ __forceinline__ static float4 load4(const uint8_t* p) {
        const uint32_t v = __ldg(reinterpret_cast<const unsigned int*>(p));
        return make_float4(u8at(v, 0), u8at(v, 1), u8at(v, 2), u8at(v, 3));
    }
    __device__ __forceinline__ static float4 load4_live(const uint8_t* p) {
        const uint32_t v = (uint32_t)ld_weak_or_relaxed(p);
        return make_float4(u8at(v, 0), u8at(v, 1), u8at(v, 2), u8at(v, 3));
    }
    __device__ __forceinline__ static float load1_live(const uint8_t* p) {
        const uint32_t v = (uint32_t)ld_relaxed(reinterpret_cast<const int32_t*>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)3));
        return (float)((v >> (8 * (reinterpret_cast<uintptr_t>(p) & 3))) & 0xFFu);
    }
    __device__ __forceinline__ static float load1(const uint8_t* p) { return (float)__ldg(p); }
    // +-1 on one byte of the containing 32-bit word (a byte never leaves [0, L_d] with L_d < 256: no carry
    // into, or borrow from, its neighbours)
    __device__ __forceinline__ static void add(uint8_t* base, size_t idx, int d) {
        atomicAdd(reinterpret_cast<unsigned int*>(base) + (idx >> 2), (unsigned int)d << ((idx & 3) * 8));
    }
    __device__ __forceinline__ static void store(uint8_t* p, int v) { *p = (uint8_t)v; }
    __device__ __forceinline__ static void store4(uint8_t* p, int a, int b, int c, int d) {
        *reinterpret_cast<uint32_t*>(p) = (uint32_t)a | ((uint32_t)b << 8) | ((uint32_t)c << 16) | ((uint32_t)d << 24);
    }
    __device__ __forceinline__ static int get(const uint8_t* p) { return (int)*p; }
};

// ---------------------------------------------------------------- row units (the sample kernel's dense pass)
// A lane reads its topics as units of UB = min(32, KPL * sizeof(NT)) bytes: one 32-byte load (sm_100's
// 256-bit LDG) holds 8 fp32, 16 uint16 or 32 uint8 counts.  Unit j of lane gl sits at unit index j * LA + gl of the row (column-major
// over the LA lanes that hold topics), so one load instruction of a lane group reads LA * UB consecutive
// bytes, and unit j is a fixed stride j * LA * UB from the lane's first unit.
struct __align__(32) uint8x32 { uint32_t w[8]; };
template <int UB> struct UnitT;
template <> struct UnitT<32> { using type = uint8x32; };
template <> struct UnitT<16> { using type = uint4; };
template <> struct UnitT<8> { using type = uint2; };
template <> struct UnitT<4> { using type = uint32_t; };
template <typename NT, int KPL>
struct RowUnit {
    static constexpr int UT = (32 / (int)sizeof(NT)) < KPL ? 32 / (int)sizeof(NT) : KPL;   // topics per unit
    static constexpr int UB = UT * (int)sizeof(NT);                                          // bytes per unit
    static constexpr int NU = KPL / UT;                                                      // units per lane
    static constexpr int QPU = UT / 4;                                                       // 4-topic blocks per unit
    using type = typename UnitT<UB>::type;
};
__device__ __forceinline__ uint8x32 ld_unit_nc(const uint8x32* p) {
    uint8x32 v;
    asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]), "=r"(v.w[7])
        : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_unit_nc(const uint4* p) { return __ldg(p); }
__device__ __forceinline__ uint2 ld_unit_nc(const uint2* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ld_unit_nc(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint8x32 ld_unit_live(const uint8x32* p) {
    uint8x32 v;
    if constexpr (kAsyncWeakRows)
        asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]),
                       "=r"(v.w[7])
                     : "l"(p));
    else
        asm volatile("ld.relaxed.gpu.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]),
                       "=r"(v.w[7])
                     : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_unit_live(const uint4* p) {
    uint4 v;
    if constexpr (kAsyncWeakRows)
        asm volatile("ld.global.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else
        asm volatile("ld.relaxed.gpu.global.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_unit_live(const uint2* p) { return kAsyncWeakRows ? ld_weak_u2(p) : ld_relaxed_u2(p); }
__device__ __forceinline__ uint32_t ld_unit_live(const uint32_t* p) { return (uint32_t)ld_weak_or_relaxed(p); }
__device__ __forceinline__ uint32_t unit_word(const uint8x32& u, int s) { return u.w[s]; }
__device__ __forceinline__ uint32_t unit_word(const uint4& u, int s) { return s == 0 ? u.x : s == 1 ? u.y : s == 2 ? u.z : u.w; }
__device__ __forceinline__ uint32_t unit_word(const uint2& u, int s) { return s == 0 ? u.x : u.y; }
__device__ __forceinline__ uint32_t unit_word(const uint32_t& u, int) { return u; }
// the 4 counts of 4-topic block s of a unit, as fp32 (s is a compile-time index after unrolling)
template <typename NT, typename U>
__device__ __forceinline__ float4 unit_block(const U& u, int s) {
    if constexpr (sizeof(NT) == 4) {
        return make_float4(__uint_as_float(unit_word(u, 4 * s)), __uint_as_float(unit_word(u, 4 * s + 1)),
                           __uint_as_float(unit_word(u, 4 * s + 2)), __uint_as_float(unit_word(u, 4 * s + 3)));
    } else if constexpr (sizeof(NT) == 2) {
        const uint32_t a = unit_word(u, 2 * s), b = unit_word(u, 2 * s + 1);
        return make_float4(u16lo(a), u16hi(a), u16lo(b), u16hi(b));
    } else {
        const uint32_t a = unit_word(u, s);
        return make_float4(u8at(a, 0), u8at(a, 1), u8at(a, 2), u8at(a, 3));
    }
}

struct SweepArgs {
    // tokens of this rank, sorted by (wave, w, i, doc)
    const uint32_t* tok_doc;
    const uint32_t* tok_id;
    uint16_t* zr;
    uint16_t* zr_next;
    // chunks (warp work units) of the launched wave
    const uint32_t* chunk_start;   // [nchunks] first token of the chunk
    const uint32_t* chunk_end;     // [nchunks] one past its last token
    const uint32_t* chunk_seg;     // [nchunks] segment = w * I + i
    int nchunks;
    uint32_t* work;                // persistent-warp chunk counter (zeroed before each launch)
    // counts
    void* n;                       // doc-topic counts n_dk (Row<NT>), rows in sigma order
    const int* sigma;              // [Kp] in-row position of topic k
    int LA;                        // lanes of a group that hold topics: ceil(K / KPL)
    int Kn;                        // doc-topic row length (elements): LA * KPL
    int prefetch_rows;             // the doc-topic array exceeds L2: prefetch rows in phase 1
    int32_t* m;
    int32_t* t;
    int32_t* Q;
    int32_t* M;
    int32_t* Tt;
    int32_t* T;
    int32_t* dm;                   // raw wave deltas [V][I][Kp]
    int32_t* dt;
    const float* alpha;            // [I][Kp] (0 on padding)
    const float* disc;             // [I]
    const float* conc;             // [I]
    const float2* tab;             // concatenated ratio tables
    const uint64_t* tab_off;       // [I] offset of group i's table
    float beta, vbeta;
    // fp64 copies for the estimators (perplexity)
    const double* alpha64;         // [I][Kp]
    const double* disc64;
    const double* conc64;
    double beta64, vbeta64;
    int I, K, Kp;
    uint32_t key0, key1;
    const uint32_t* sweep;         // device counter (RNG counter word 1)
    unsigned long long* stats;     // [8]
    // debug_probs
    double* dbg_w;                 // [ntok][2K] unnormalised weights, or null
    int32_t* dbg_info;             // [ntok][4]
    int packed_dmt;                // wave deltas as one packed dm * 2^16 + dt word per cell in dm (M_max < 2^15)
    const uint32_t* slot;          // W = 1: document-order slot of each sorted token, or null
    uint16_t* zr_doc;              // W = 1: the new assignments in document order (the recount streams them)
    // per-wave factor tables (chunk_ft): [run][Kp] slot factors F0 + F1, r = 1 shares, alpha F, packed (m, t)
    int chunk_ft;
    const uint32_t* tok_run;       // run (segment of the wave) of each sorted token
    const float* Ft;
    const float* R1t;
    const float* aFt;
    const uint32_t* MTt;
    // sparse doc-topic rows (spdp_sprows.cuh)
    const uint2* dinfo;            // [D_local] {first entry, nonzero topics}
    const uint32_t* ent;           // entries k | n << 16, topic order per document
};

// ---------------------------------------------------------------- the sample kernel
// Doc-topic row layout ("sigma order").  A token's dense pass uses LPT lanes;
// lane gl owns the canonical topics [gl*KPL, gl*KPL + KPL), read as NU units of
// UT topics (RowUnit: 16 bytes, or the whole span if smaller).  Only the
// LA = ceil(K / KPL) lanes that hold topics have storage: unit j of lane gl sits
// at unit index j * LA + gl (column-major over the active lanes), so one load
// instruction of the group reads LA consecutive units, unit j is at a fixed
// stride from unit 0 (one address add per load), and rows have Kn = LA * KPL
// elements (the last active lane's topics past K are zero padding).  Each lane's
// topics are contiguous in the canonical order — the CDF is one scan over lanes.
// sigma[k] is the in-row position of topic k (host table); every other kernel
// touching n uses it with the row length Kn.

// Per-warp shared memory (KSPAN entries each unless noted).
template <int LPT, int KPL>
__host__ __device__ constexpr bool f_in_smem() { return SPDP_F_SMEM == 1 || (SPDP_F_SMEM == 2 && LPT == 8 && KPL == 32); }
template <int KSPAN, int KPL>
struct __align__(16) WarpSmem {   // 16-byte multiple: every warp's F rows are read as float4
    // F0 + F1 at the snapshot counts, skewed like aF: the group's per-lane reads (each chunk's register
    // copy, or every step's blocks when the dense pass reads F here) are then conflict-free broadcasts
    // (B200: K = 300 (16x32) 1.61 -> 1.53 ms per sweep, C3 -2 %); not at 32x32, where the skew's extra
    // 512 B per warp cost a resident block (K = 1000: 4.0 -> 5.3 ms)
    static constexpr bool kFS = f_in_smem<KSPAN / KPL, KPL>();
    static constexpr bool kFSkew = kFS || KSPAN <= 512;
    float F[KSPAN + (kFSkew ? 4 * (KSPAN / KPL) : 0)];
    __device__ __forceinline__ static int fi(int k) { return kFSkew ? k + 4 * (k / KPL) : k; }
    float aF[KSPAN + 4 * (KSPAN / KPL)];   // alpha_ik F, lane segments skewed by 16 B (conflict-free)
    uint32_t mt[KSPAN];  // snapshot m << 16 | t of the segment's cells (M_max < 2^16)
    float R1[SPDP_SMEM_R1 && KSPAN <= 256 ? KSPAN : 1];   // r = 1 share F1 / F at the snapshot (phase 3's r split)
    int dmt[KSPAN];      // the chunk's delta m * 2^16 + delta t (|delta| <= chunk length)
    // hand-over from the dense pass to the per-token search (one entry per token of the batch), written
    // and read with vector accesses: a token's block sums are one row (8 sums: 48-byte rows, so the
    // 16-byte reads of 8 consecutive tokens hit distinct banks)
    static constexpr int NB = KPL / 4, BSROW = NB == 8 ? 12 : NB;
    alignas(16) float bs[32][BSROW];   // the winning lane's block sums (without the own-removal fix)
    alignas(16) double2 lt[32];        // {prefix before the winning lane, u * total}
    int wgl[32];             // winning lane within the group (negative: fall back to the last positive slot)
    // the next chunk's snapshot m and t rows, copied asynchronously during this chunk's last batch
    // (KSPAN <= 256); its Stirling-table entries land in the hand-over region (bs, lt), which is free
    // between the end of the last batch and the next chunk's first
    static constexpr bool kStage = SPDP_STAGE_NEXT != 0 && KSPAN <= 256;
    alignas(16) int nm[kStage ? KSPAN : 4];
    alignas(16) int nt[kStage ? KSPAN : 4];
    uint32_t nxc, nseg;      // the next chunk's index and segment (kept here, not in registers)
    __device__ __forceinline__ float2* ntab() { return reinterpret_cast<float2*>(&bs[0][0]); }
};
template <typename WS>
__host__ __device__ constexpr bool stage_fits() { return sizeof(WS::bs) + sizeof(WS::lt) >= 8 * sizeof(WS::nm) / sizeof(int); }

// asynchronous global -> shared copies (cp.async, sm_80+): no registers held while in flight
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// NB fp32 values to / from a shared-memory row (16-, 8- or 4-byte accesses)
template <int NB>
__device__ __forceinline__ void store_row(float* r, const float* v) {
    if constexpr (NB >= 4) {
#pragma unroll
        for (int q = 0; q < NB; q += 4) *reinterpret_cast<float4*>(r + q) = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
    } else if constexpr (NB == 2) {
        *reinterpret_cast<float2*>(r) = make_float2(v[0], v[1]);
    } else {
        r[0] = v[0];
    }
}
template <int NB>
__device__ __forceinline__ void load_row(const float* r, float* v) {
    if constexpr (NB >= 4) {
#pragma unroll
        for (int q = 0; q < NB; q += 4) {
            const float4 x = *reinterpret_cast<const float4*>(r + q);
            v[q] = x.x; v[q + 1] = x.y; v[q + 2] = x.z; v[q + 3] = x.w;
        }
    } else if constexpr (NB == 2) {
        const float2 x = *reinterpret_cast<const float2*>(r);
        v[0] = x.x; v[1] = x.y;
    } else {
        v[0] = r[0];
    }
}
template <int KPL>
__device__ __forceinline__ int skew(int k) { return k + 4 * (k / KPL); }

// One warp per chunk of one (w, i) segment.  Per chunk, the segment's factors
// F_k and F1_k/F_k at the snapshot (and, for long chunks, the own-removal
// variants, Alg.1 lines 4-10) go to shared memory.  Per batch of 32 tokens:
//   phase 1 (lane = token): record, Philox (a2), removal draw against the
//     snapshot and the own-removal correction of topic k0 (a3);
//   phase 2 (LPT lanes per token, 32/LPT tokens per step): the doc-topic row
//     (a4), fp32 4-topic block sums of w_k = (alpha_ik + n_dk) F_k (a chain of 4
//     FFMA from the chunk's sum of alpha_ik F_k over the block) and lane totals, one fp64 scan over the group's lanes,
//     target = u * total, the lane holding it (a5, a6);
//   phase 3 (lane = token): the block and the topic where the prefix first
//     exceeds the target, slots in the paper's order j = 2k (r = 1), 2k+1 (r = 0),
//     the r split by the exact r = 1 share; outputs and count deltas (a7).
//   Every CDF boundary is an fp64 sum of fp32 partial sums of few terms
//   (a few fp32 ulps of the total), inside the 1e-6 band of north_star (5).
template <typename NT, bool AS>
__device__ __forceinline__ float4 row_load4(const NT* p) {
    if constexpr (AS) return Row<NT>::load4_live(p);
    else return Row<NT>::load4(p);
}
template <typename NT, bool AS>
__device__ __forceinline__ typename Row<NT>::raw_t row_load_raw(const NT* p) {
    if constexpr (AS) return Row<NT>::load_raw_live(p);
    else return Row<NT>::load_raw(p);
}
template <typename NT, bool AS>
__device__ __forceinline__ float row_load1(const NT* p) {
    if constexpr (AS) return Row<NT>::load1_live(p);
    else return Row<NT>::load1(p);
}

// ASYNC (the paper's in-GPU scheme P:2210-2233 / Alg.4
// P:2973-3012): no wave snapshot.  A chunk copies the live counts of its
// segment when it starts ("local copy ... at the beginning of each thread"),
// corrects the copy into the valid range (Alg.4 "correct local counts copied
// ... to ensure they are in valid range"), reads doc-topic rows live, and
// applies its updates to the global counts at once: n per token (atomics),
// m, t, Q and the sums per chunk (atomics).  Nondeterministic by design.
// resident blocks per SM the sample kernel is compiled for (register budget): measured per
// configuration on B200 — 8x32 (C5) runs 13 % faster with 5 blocks (<= 96 registers), while
// 4x32 (C3) and 16x32 lose 20-30 % there
template <int LPT, int KPL>
__host__ __device__ constexpr int sample_minb() { return (LPT == 8 && KPL == 32) ? SPDP_MINB_8X32 : SPDP_MINB; }

template <int LPT, int KPL, bool DEBUG, typename NT, bool ASYNC = false>
__global__ void __launch_bounds__(kWarps * 32, sample_minb<LPT, KPL>())
sample_kernel(SweepArgs A) {
    constexpr int TPW = 32 / LPT;
    constexpr int KSPAN = LPT * KPL;
    constexpr int NB = KPL / 4;                      // 4-topic blocks per lane
    static_assert(KPL % 4 == 0 && NB <= 8, "KPL must be a multiple of 4, at most 32");
    using RU = RowUnit<NT, KPL>;
    using unit_t = typename RU::type;
    constexpr int NU = RU::NU, QPU = RU::QPU, UT = RU::UT;
    // per-block alpha sums: 2.5-3.5 % faster at C3, K = 300, K = 1000 (B200); not under the
    // 5-blocks register cap of 8x32, where the 8 extra registers spill (C5 +2.7 %)
    // narrow rows keep their raw blocks (1-2 registers per 4 counts instead of 4), which frees the registers the
    // 5-blocks/SM 8x32 build needs for the block alpha sums and the row pipeline (SPDP_NARROW_FULL)
    constexpr bool kNarrowFull = SPDP_NARROW_FULL != 0 && sizeof(NT) < 4;
    constexpr bool kBlockAlpha = SPDP_BLOCK_ALPHA != 0 && (sample_minb<LPT, KPL>() <= 4 || kNarrowFull);
    // software-pipelined row loads: C3 -3 %, K = 300 -7 %, K = 1000 +-0 (B200); spills under the
    // 8x32 register cap (C5 +30 %), so not there
    constexpr bool kRowPipe = SPDP_ROW_PIPELINE != 0 && (sample_minb<LPT, KPL>() <= 4 || kNarrowFull);
    // own-removal inputs before the Philox rounds: C3 -1 %, K = 300 -1.8 %, C5 (8x32) +1 % (B200)
    constexpr bool kPreTab = SPDP_PRE_TAB != 0 && (sample_minb<LPT, KPL>() <= 4 || (kNarrowFull && SPDP_NARROW_PRETAB));
    // r = 1 shares from the prologue in shared memory (not in the async mode: its copy is per chunk too,
    // but the live sums it reads in phase 3 are fresher); KSPAN <= 256 (smem budget of 16x32 / 32x32)
    constexpr bool kSmemR1 = SPDP_SMEM_R1 != 0 && KSPAN <= 256 && !ASYNC;
    constexpr bool kFSmem = WarpSmem<KSPAN, KPL>::kFS;
    // the next chunk's prologue inputs staged during this chunk (wave mode: snapshot counts do not change
    // within a wave; the async mode copies live counts at chunk start by design)
    constexpr bool kStage = SPDP_STAGE_NEXT != 0 && WarpSmem<KSPAN, KPL>::kStage && !ASYNC && !DEBUG;
    static_assert(!kStage || stage_fits<WarpSmem<KSPAN, KPL>>(), "staged table entries must fit the hand-over region");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    WarpSmem<KSPAN, KPL>& S = reinterpret_cast<WarpSmem<KSPAN, KPL>*>(smem_raw)[wid];
    const int I = A.I, K = A.K, Kp = A.Kp;
    unsigned keeps = 0, moved = 0;
    const int g = lane / LPT, gl = lane % LPT;
    const int kb = gl * KPL;                         // this lane's first canonical topic (phase 2)
    const unsigned gmask = (LPT == 32) ? 0xffffffffu : (((1u << LPT) - 1u) << (g * LPT));
    const int LA = A.LA, Kn = A.Kn;
    const bool lane_rows = gl < LA;                  // this lane's topics have row storage
    const size_t ustride = (size_t)LA * RU::UB;      // bytes from unit j to unit j + 1 of a lane

  // persistent warps: grab chunks (sorted longest first on the host) from a counter.  Staged mode: the
  // next chunk's index is taken when this one starts, and its descriptor, m and t rows and Stirling-table
  // entries are copied to shared memory during this chunk's last batch, off the prologue's critical path.
  const bool stage = kStage && !A.chunk_ft;
  bool staged = false;                               // the current chunk's prologue inputs are in S.nm, S.nt, S.ntab
  if (stage) {
    if (lane == 0) S.nxc = atomicAdd(A.work, 1u);
    __syncwarp();
  }
  for (;;) {
    uint32_t nx = 0;                                 // lane 0: the next chunk's index (in flight during the prologue)
    int c;
    if (stage) {
      c = (int)S.nxc;
      if (c >= A.nchunks) break;                     // warp-uniform
      __syncwarp();
      if (lane == 0) nx = atomicAdd(A.work, 1u);
    } else {
      uint32_t cc = 0;
      if (lane == 0) cc = atomicAdd(A.work, 1u);
      c = (int)__shfl_sync(0xffffffffu, cc, 0);
      if (c >= A.nchunks) break;                     // warp-uniform
    }
    __syncwarp();
    const uint32_t seg = staged ? S.nseg : A.chunk_seg[c];
    const int w = (int)(seg / (uint32_t)I), i = (int)(seg % (uint32_t)I);
    const size_t row = (size_t)seg * Kp;
    const float a = A.disc[i], b = A.conc[i];
    const float2* __restrict__ tab = A.tab + A.tab_off[i];
    const int32_t* __restrict__ Mi = A.M + (size_t)i * Kp;
    const int32_t* __restrict__ Tti = A.Tt + (size_t)i * Kp;
    const int32_t* __restrict__ Qw = A.Q + (size_t)w * Kp;
    const float* __restrict__ alpha_i = A.alpha + (size_t)i * Kp;

    const uint32_t start = A.chunk_start[c], end = A.chunk_end[c];
    // ---- prologue: the segment's slot factors at the wave-start snapshot: from the wave's factor
    // tables (chunk_ft: coalesced row loads, no dependent chain), or computed here.  Computed: topics in
    // groups of PG per lane, all count loads of a group first, then its Stirling-table loads, then the math.
    uint32_t crun = 0;
    if (staged) {                                    // this chunk's staged copies have landed
        cp_async_wait_all();
        __syncwarp();
    }
    if (!ASYNC && A.chunk_ft) {
        crun = A.tok_run[start];
        const size_t rrow = (size_t)crun * Kp;
        for (int k = lane; k < KSPAN; k += 32) {
            float Fk = 0.f, aFk = 0.f;
            uint32_t mt = 0;
            if (k < K) { Fk = A.Ft[rrow + k]; aFk = A.aFt[rrow + k]; mt = A.MTt[rrow + k]; }
            if constexpr (kSmemR1) S.R1[k] = (k < K) ? A.R1t[rrow + k] : 0.f;
            S.F[S.fi(k)] = Fk;
            S.aF[skew<KPL>(k)] = aFk;
            S.mt[k] = mt;
            S.dmt[k] = 0;
        }
    } else {
        constexpr int PER = (KSPAN + 31) / 32;
        constexpr int PGS = KSPAN >= 1024 ? SPDP_PRO_GROUP_1024 : SPDP_PRO_GROUP;
        constexpr int PG = PGS < PER ? PGS : PER;
        static_assert(PER % PG == 0, "prologue group must divide the topics per lane");
#pragma unroll 1
        for (int k0g = 0; k0g < PER; k0g += PG) {
            int mv[PG], tv[PG], Mv[PG], Ttv[PG], Qv[PG], Tv[PG];
            float al[PG];
            float2 tb[PG];
            if (staged) {                            // staged during the previous chunk: m, t and the table entries
#pragma unroll
                for (int j = 0; j < PG; ++j) {
                    const int k = lane + 32 * (k0g + j);
                    mv[j] = tv[j] = Mv[j] = Ttv[j] = Qv[j] = Tv[j] = 0;
                    al[j] = 0.f;
                    tb[j] = make_float2(0.f, 0.f);
                    if (k < K) {
                        mv[j] = S.nm[k]; tv[j] = S.nt[k]; tb[j] = S.ntab()[k];
                        al[j] = alpha_i[k];
                        Mv[j] = Mi[k]; Ttv[j] = Tti[k]; Qv[j] = Qw[k]; Tv[j] = A.T[k];
                    }
                }
            } else {
#pragma unroll
            for (int j = 0; j < PG; ++j) {
                const int k = lane + 32 * (k0g + j);
                mv[j] = tv[j] = Mv[j] = Ttv[j] = Qv[j] = Tv[j] = 0;
                al[j] = 0.f;
                if (k < K) {
                    mv[j] = ldc<ASYNC>(A.m + row + k);
                    tv[j] = ldc<ASYNC>(A.t + row + k);
                    al[j] = alpha_i[k];
                    Mv[j] = ldc<ASYNC>(Mi + k); Ttv[j] = ldc<ASYNC>(Tti + k); Qv[j] = ldc<ASYNC>(Qw + k); Tv[j] = ldc<ASYNC>(A.T + k);
                }
            }
#pragma unroll
            for (int j = 0; j < PG; ++j) {
                const int k = lane + 32 * (k0g + j);
                if constexpr (ASYNC) {                // valid range of the local copy (reading c14), then of the sums
                    mv[j] = max(mv[j], 0);
                    tv[j] = mv[j] > 0 ? min(max(tv[j], 1), mv[j]) : 0;
                    Mv[j] = max(Mv[j], mv[j]); Ttv[j] = max(Ttv[j], tv[j]); Qv[j] = max(Qv[j], tv[j]); Tv[j] = max(Tv[j], Qv[j]);
                }
                tb[j] = (k < K) ? tab[tri(mv[j]) + tv[j]] : make_float2(0.f, 0.f);
            }
            }   // computed loads
#pragma unroll
            for (int j = 0; j < PG; ++j) {
                const int k = lane + 32 * (k0g + j);
                float F0 = 0.f, F1 = 0.f;
                if (k < K) slot_factors(Mv[j], Ttv[j], Qv[j], Tv[j], tb[j], a, b, A.beta, A.vbeta, F0, F1);
                if (k >= KSPAN) continue;            // KSPAN < 32 (K <= 16)
                const float Fk = F0 + F1;
                if constexpr (kSmemR1) S.R1[k] = (F1 > 0.f) ? __fdiv_rn(F1, Fk) : 0.f;
                S.F[S.fi(k)] = Fk;
                S.aF[skew<KPL>(k)] = __fmul_rn(al[j], Fk);
                S.mt[k] = ((uint32_t)mv[j] << 16) | (uint32_t)tv[j];
                S.dmt[k] = 0;
            }
        }
    }   // computed prologue
    if (stage && lane == 0) S.nxc = nx;              // (the atomic has returned by now)
    __syncwarp();

    // the lane's F_k: registers, or (SPDP_F_SMEM) read from shared memory per block in the dense pass
    // (conflict-free broadcast loads; frees KPL registers for more resident warps)
    float F[kFSmem ? 1 : KPL];
    if constexpr (!kFSmem) {
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const float4 f4 = *reinterpret_cast<const float4*>(&S.F[S.fi(kb + 4 * q)]);
            F[4 * q] = f4.x; F[4 * q + 1] = f4.y; F[4 * q + 2] = f4.z; F[4 * q + 3] = f4.w;
        }
    }
    const float* Fl = &S.F[S.fi(kb)];
    const float* aFl = &S.aF[skew<KPL>(kb)];
    float aSF[NB];                                   // per block: sum of alpha_ik F_k (SPDP_BLOCK_ALPHA)
    if constexpr (kBlockAlpha) {
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const float4 af = *reinterpret_cast<const float4*>(aFl + 4 * q);
            aSF[q] = (af.x + af.y) + (af.z + af.w);
        }
    }
    const uint32_t sweep = *A.sweep;

    for (uint32_t b0 = start; b0 < end; b0 += 32) {
        const uint32_t nb = min(32u, end - b0);
        uint32_t seg_next = 0;                       // last batch: the next chunk's segment (its copies follow)
        const bool stage_now = stage && b0 + 32u >= end && S.nxc < (uint32_t)A.nchunks;
        if (stage_now) seg_next = A.chunk_seg[S.nxc];
        // ======== phase 1: lane = token
        const bool mine = (uint32_t)lane < nb;
        const uint32_t p = b0 + lane;
        uint32_t noff = 0, zr0 = 0, x0 = 0;
        double u = 0.0;
        if (mine) {
            noff = A.tok_doc[p] * (uint32_t)Kn;            // doc-topic row offset (fits 32 bits)
            zr0 = A.zr[p];
        }
        // the own-removal inputs of topic k0 (both table candidates: r_rem is drawn below), issued
        // before the Philox rounds so that their latency overlaps them
        const int k0 = (int)(zr0 & 0x7FFFu);
        const uint32_t mt0 = S.mt[k0];
        const int m0 = (int)(mt0 >> 16), t0 = (int)(mt0 & 0xFFFFu);
        const int mm0 = max(m0 - 1, 0);
        float2 tab_r1 = make_float2(0.f, 0.f), tab_r0 = make_float2(0.f, 0.f);
        int Mk0 = 0, Ttk0 = 0, Qk0 = 0, Tk0 = 0;
        if constexpr (kPreTab) {
            if (mine) {
                tab_r1 = tab[tri(mm0) + max(t0 - 1, 0)];
                tab_r0 = tab[tri(mm0) + min(t0, mm0)];
                load_sums<ASYNC>(Mi, Tti, Qw, A.T, k0, m0, t0, Mk0, Ttk0, Qk0, Tk0);
            }
        }
        if (mine) {
            const uint4 x = philox(make_uint4(A.tok_id[p], sweep, 0u, 0u), A.key0, A.key1);   // a2
            x0 = x.x;
            u = u53(x);
        }
        const NT* __restrict__ nrow = reinterpret_cast<const NT*>(A.n) + noff;
        if (A.prefetch_rows) {   // rows not L2-resident: pull rows of this batch (first) and the next towards L2
            if constexpr (SPDP_BULK_PREFETCH) {
                // one exact-size bulk prefetch per row: at the chunk's first batch the rows of batches
                // 0 .. AHEAD, afterwards those of batch b + AHEAD (the copy engine runs ahead of the sampling)
                const uint32_t rbytes = (uint32_t)((size_t)Kn * sizeof(NT));
                if (b0 == start) {
#pragma unroll
                    for (int j = 0; j < SPDP_PREFETCH_AHEAD; ++j)
                        if (p + 32u * j < end)
                            prefetch_bytes_l2(reinterpret_cast<const NT*>(A.n) + (size_t)A.tok_doc[p + 32u * j] * Kn, rbytes);
                }
                const uint32_t pn = p + 32u * SPDP_PREFETCH_AHEAD;
                if (pn < end) prefetch_bytes_l2(reinterpret_cast<const NT*>(A.n) + (size_t)A.tok_doc[pn] * Kn, rbytes);
            } else {
                constexpr int PER_LINE = 128 / (int)sizeof(NT);
                if (mine && (b0 == start || !SPDP_PREFETCH_NEXT))
                    for (int l = 0; l * PER_LINE < Kn; ++l) asm volatile("prefetch.global.L2 [%0];" ::"l"(nrow + PER_LINE * l));
                const uint32_t pn = p + 32;
                if (SPDP_PREFETCH_NEXT && pn < end) {
                    const NT* nn = reinterpret_cast<const NT*>(A.n) + (size_t)A.tok_doc[pn] * Kn;
                    for (int l = 0; l * PER_LINE < Kn; ++l) asm volatile("prefetch.global.L2 [%0];" ::"l"(nn + PER_LINE * l));
                }
            }
        }
        const int rrem = removal_draw(x0, m0, t0);                                            // a3
        const bool keep = rrem && t0 == 1 && m0 > 1;   // DESIGN.md reading c5
        float Fk0 = 0.f, R1k0 = 0.f;                    // topic k0's factors after the own removal
        if constexpr (kPreTab) {
            if (mine) removal_factors_pre(rrem, m0, Mk0, Ttk0, Qk0, Tk0, tab_r1, tab_r0, a, b, A.beta, A.vbeta, Fk0, R1k0);
        } else {
            if (mine) {
                load_sums<ASYNC>(Mi, Tti, Qw, A.T, k0, m0, t0, Mk0, Ttk0, Qk0, Tk0);
                removal_factors(rrem, m0, t0, Mk0, Ttk0, Qk0, Tk0, tab, a, b, A.beta, A.vbeta, Fk0, R1k0);
            }
        }
        float n0 = mine ? row_load1<NT, ASYNC>(nrow + A.sigma[k0]) : 0.f;
        if constexpr (ASYNC) n0 = fmaxf(n0, 1.f);    // the token itself is counted in its row
        const float al0 = alpha_i[k0];
        const float wold = __fmaf_rn(n0, S.F[S.fi(k0)], S.aF[skew<KPL>(k0)]);   // == the dense pass's mass
        const float wnew = __fmaf_rn(n0 - 1.f, Fk0, __fmul_rn(al0, Fk0));
        const float dlt = wnew - wold;

        if (stage_now) {                             // the next chunk's snapshot m and t rows -> shared memory
            if (lane == 0) S.nseg = seg_next;
            const size_t rn = (size_t)seg_next * Kp;
            for (int q = lane; 4 * q < K; q += 32) {
                cp_async16(&S.nm[4 * q], A.m + rn + 4 * q);
                cp_async16(&S.nt[4 * q], A.t + rn + 4 * q);
            }
            cp_async_commit();
        }
        // ======== phase 2: LPT lanes per token
        unit_t v[NU];                                // raw row units (fp32 at use: narrow rows keep few registers);
#pragma unroll                                       // lanes without storage keep zeros (F = 0 there)
        for (int j = 0; j < NU; ++j) v[j] = unit_t{};
        auto load_rows = [&](uint32_t s) {            // the doc-topic rows of step s's tokens
            const uint32_t so = __shfl_sync(0xffffffffu, noff, (s + g) & 31);
            const unsigned char* nl = reinterpret_cast<const unsigned char*>(A.n) + (size_t)so * sizeof(NT) + gl * RU::UB;
            if (lane_rows) {
#pragma unroll
                for (int j = 0; j < NU; ++j) {
                    const unit_t* up = reinterpret_cast<const unit_t*>(nl + (size_t)j * ustride);
                    if constexpr (ASYNC) v[j] = ld_unit_live(up);
                    else v[j] = ld_unit_nc(up);
                }
            }
        };
        if constexpr (kRowPipe) load_rows(0);
        for (uint32_t s0 = 0; s0 < nb; s0 += TPW) {
            const uint32_t src = (s0 + g) & 31;
            const int sk0 = __shfl_sync(0xffffffffu, k0, src);
            const float sdlt = __shfl_sync(0xffffffffu, dlt, src);
            const double su = __shfl_sync(0xffffffffu, u, src);
            if constexpr (!kRowPipe) load_rows(s0);
            float sb[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                const float4 n4 = unit_block<NT>(v[q / QPU], q % QPU);
                if constexpr (kBlockAlpha) {
                    // no per-topic alpha term: 4 FFMA per block, no shared-memory load
                    float4 f4;
                    if constexpr (kFSmem) f4 = *reinterpret_cast<const float4*>(Fl + 4 * q);
                    else f4 = make_float4(F[4 * q + 0], F[4 * q + 1], F[4 * q + 2], F[4 * q + 3]);
                    float x = __fmaf_rn(n4.x, f4.x, aSF[q]);
                    x = __fmaf_rn(n4.y, f4.y, x);
                    x = __fmaf_rn(n4.z, f4.z, x);
                    sb[q] = __fmaf_rn(n4.w, f4.w, x);
                } else {
                    const float4 af = *reinterpret_cast<const float4*>(aFl + 4 * q);
                    float4 f4;
                    if constexpr (kFSmem) f4 = *reinterpret_cast<const float4*>(Fl + 4 * q);
                    else f4 = make_float4(F[4 * q + 0], F[4 * q + 1], F[4 * q + 2], F[4 * q + 3]);
                    const float w0 = __fmaf_rn(n4.x, f4.x, af.x);
                    const float w1 = __fmaf_rn(n4.y, f4.y, af.y);
                    const float w2 = __fmaf_rn(n4.z, f4.z, af.z);
                    const float w3 = __fmaf_rn(n4.w, f4.w, af.w);
                    sb[q] = (w0 + w1) + (w2 + w3);
                }
            }
            if constexpr (kRowPipe)
                if (s0 + TPW < nb) load_rows(s0 + TPW);   // warp-uniform; overlaps the scan and hand-over below
            float lt32;                                    // tree sum of the block sums
            {
                float t8[NB];
#pragma unroll
                for (int q = 0; q < NB; ++q) t8[q] = sb[q];
#pragma unroll
                for (int h = 1; h < NB; h <<= 1)
#pragma unroll
                    for (int q = 0; q + h < NB; q += 2 * h) t8[q] += t8[q + h];
                lt32 = t8[0];
            }
            const bool owner = (sk0 >= kb) && (sk0 < kb + KPL);
            const double acc = (double)lt32 + (owner ? (double)sdlt : 0.0);
            double incl = acc;
#pragma unroll
            for (int off = 1; off < LPT; off <<= 1) {
                const double y = __shfl_up_sync(0xffffffffu, incl, off, LPT);
                if (gl >= off) incl += y;
            }
            const double total = __shfl_sync(0xffffffffu, incl, LPT - 1, LPT);
            const double target = su * total;
            const unsigned hit = __ballot_sync(0xffffffffu, incl > target) & gmask;
            const unsigned posl = __ballot_sync(0xffffffffu, acc > 0.0) & gmask;
            const int winner = hit ? (__ffs(hit) - 1) : (posl ? 31 - __clz(posl) : g * LPT);
            if (lane == winner && s0 + g < nb) {
                store_row<NB>(S.bs[src], sb);
                S.lt[src] = make_double2(incl - acc, target);
                S.wgl[src] = hit ? gl : -1 - gl;
            }
        }
        __syncwarp();

        // ======== phase 3: lane = token
        if (mine) {
            int ks = k0, rs = 1;
            if (!keep) {
                const double2 ltv = S.lt[lane];
                const double lbeg = ltv.x, target = ltv.y;
                const int wv = S.wgl[lane];
                bool fb = wv < 0;
                const int wg = fb ? -1 - wv : wv;
                const int own_q = (k0 >= wg * KPL && k0 < wg * KPL + KPL) ? ((k0 - wg * KPL) >> 2) : -1;
                float bsv[NB];
                load_row<NB>(S.bs[lane], bsv);
#pragma unroll
                for (int q = 0; q < NB; ++q) bsv[q] += (q == own_q) ? dlt : 0.f;
                // block: count the blocks whose fp32 prefix does not exceed the target
                const float rel = (float)(target - lbeg);
                float run = 0.f;
                int qs = 0;
#pragma unroll
                for (int q = 0; q < NB; ++q) { run += bsv[q]; qs += (run <= rel) ? 1 : 0; }
                if (fb || qs >= NB) {                      // rounding: the last positive block
                    fb = true; qs = 0;
#pragma unroll
                    for (int q = 0; q < NB; ++q) if (bsv[q] > 0.f) qs = q;
                }
                float pre32 = 0.f;
#pragma unroll
                for (int q = 0; q < NB; ++q) if (q < qs) pre32 += bsv[q];
                // the block's 4 topic masses (their fp32 sum may differ from the dense pass's block
                // sum by a few ulps; a target in that gap takes the last positive topic below)
                const int kq = wg * KPL + 4 * qs;
                const float4 n4 = row_load4<NT, ASYNC>(nrow + ((qs / QPU) * LA + wg) * UT + 4 * (qs % QPU));
                const float4 F4 = *reinterpret_cast<const float4*>(&S.F[S.fi(kq)]);
                const float4 a4 = *reinterpret_cast<const float4*>(&S.aF[skew<KPL>(kq)]);
                float wq[4] = {__fmaf_rn(n4.x, F4.x, a4.x), __fmaf_rn(n4.y, F4.y, a4.y),
                               __fmaf_rn(n4.z, F4.z, a4.z), __fmaf_rn(n4.w, F4.w, a4.w)};
#pragma unroll
                for (int e = 0; e < 4; ++e) if (kq + e == k0) wq[e] = wnew;
                double run2 = lbeg + (double)pre32, bes = run2, blast = run2;
                int es = -1, elast = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const double nxt = run2 + (double)wq[e];
                    if (es < 0 && !fb && nxt > target) { es = e; bes = run2; }
                    if (wq[e] > 0.f) { elast = e; blast = run2; }
                    run2 = nxt;
                }
                if (es < 0) { fb = true; es = elast; bes = blast; }   // rounding: last positive topic
                float wsel = 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) if (e == es) wsel = wq[e];
                ks = kq + es;
                const bool own = (ks == k0);
                const uint32_t mts = S.mt[ks];
                float R1s = R1k0;
                if constexpr (kSmemR1) {
                    if (!own) R1s = S.R1[ks];              // the chunk prologue's share
                } else if (!own && !ASYNC && A.chunk_ft) R1s = A.R1t[(size_t)crun * Kp + ks];   // from the factor table
                else if (!own) {                           // r = 1 share of topic ks at the snapshot
                    float f0, f1;
                    int Ms, Tts, Qs, Ts;
                    load_sums<ASYNC>(Mi, Tti, Qw, A.T, ks, (int)(mts >> 16), (int)(mts & 0xFFFFu), Ms, Tts, Qs, Ts);
                    slot_factors(Ms, Tts, Qs, Ts, tab[tri((int)(mts >> 16)) + (mts & 0xFFFFu)], a, b, A.beta, A.vbeta, f0, f1);
                    R1s = (f1 > 0.f) ? __fdiv_rn(f1, f0 + f1) : 0.f;
                }
                const float w1 = wsel * R1s;
                if (!fb) rs = (bes + (double)w1 > target) ? 1 : 0;
                else rs = ((own ? m0 - 1 : (int)(mts >> 16)) > 0) ? 0 : 1;   // last positive slot
            }
            if constexpr (DEBUG) {
                // exact slot masses w1 = (alpha + n) F1, w0 = (alpha + n) F0 of every topic
                for (int k = 0; k < K; ++k) {
                    const bool own = (k == k0);
                    const float nk = (float)Row<NT>::get(nrow + A.sigma[k]) - (own ? 1.f : 0.f);
                    float f0, f1;
                    if (own) {
                        const int mm = max(m0 - 1, 0), tt = min(max(t0 - rrem, 0), mm);
                        slot_factors(Mi[k] - 1, Tti[k] - rrem, Qw[k] - rrem, A.T[k] - rrem, tab[tri(mm) + tt],
                                     a, b, A.beta, A.vbeta, f0, f1);
                    } else {
                        slot_factors(Mi[k], Tti[k], Qw[k], A.T[k], tab[tri((int)(S.mt[k] >> 16)) + (S.mt[k] & 0xFFFFu)],
                                     a, b, A.beta, A.vbeta, f0, f1);
                    }
                    const double base = (double)alpha_i[k] + (double)nk;
                    A.dbg_w[(size_t)p * 2 * K + 2 * k] = base * (double)f1;
                    A.dbg_w[(size_t)p * 2 * K + 2 * k + 1] = base * (double)f0;
                }
                int32_t* inf = A.dbg_info + (size_t)p * 4;
                inf[0] = rrem; inf[1] = keep; inf[2] = ks; inf[3] = rs;
            } else {
                A.zr_next[p] = (uint16_t)(ks | (rs << 15));                                   // a7
                if constexpr (!ASYNC && KSPAN <= 256)   // (the host enables it for K <= 256 only)
                    if (A.zr_doc) A.zr_doc[A.slot[p]] = (uint16_t)(ks | (rs << 15));
                if (keep) ++keeps;
                else {
                    atomicAdd(&S.dmt[k0], -65536 - rrem);
                    atomicAdd(&S.dmt[ks], 65536 + rs);
                    moved += (ks != k0);
                    if constexpr (ASYNC) {                 // doc-topic row updated at once (Alg.4 "atomically")
                        if (ks != k0) {
                            NT* nw = reinterpret_cast<NT*>(A.n);
                            Row<NT>::add(nw, (size_t)noff + A.sigma[k0], -1);
                            Row<NT>::add(nw, (size_t)noff + A.sigma[ks], 1);
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
    const bool staged_next = stage && S.nxc < (uint32_t)A.nchunks;
    if (staged_next) {                               // the next chunk's Stirling-table entries (the hand-over
        cp_async_wait_all();                         // region is free until its first batch)
        __syncwarp();
        const uint32_t in = S.nseg % (uint32_t)I;
        const float2* tabn = A.tab + A.tab_off[in];
        for (int k = lane; k < K; k += 32) cp_async8(&S.ntab()[k], tabn + tri(S.nm[k]) + S.nt[k]);
        cp_async_commit();
    }
    if constexpr (!DEBUG) {
        __syncwarp();
        for (int k = lane; k < K; k += 32) {
            const int x = S.dmt[k];
            if (x) {
                const int dtv = (int)(short)(x & 0xFFFF);   // low half, sign-extended
                const int dmv = (x - dtv) >> 16;
                if constexpr (ASYNC) {                     // global counts and sums updated at once
                    if (dmv) { atomicAdd(A.m + row + k, dmv); atomicAdd(A.M + (size_t)i * Kp + k, dmv); }
                    if (dtv) {
                        atomicAdd(A.t + row + k, dtv); atomicAdd(A.Q + (size_t)w * Kp + k, dtv);
                        atomicAdd(A.Tt + (size_t)i * Kp + k, dtv); atomicAdd(A.T + k, dtv);
                    }
                } else if (A.packed_dmt) {                 // one packed dm * 2^16 + dt word per cell
                    atomicAdd(A.dm + row + k, x);
                } else {
                    if (dmv) atomicAdd(A.dm + row + k, dmv);
                    if (dtv) atomicAdd(A.dt + row + k, dtv);
                }
            }
        }
    }
    __syncwarp();
    staged = staged_next;
  }  // chunk loop
    if constexpr (!DEBUG) {
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
}

template <int LPT, int KPL>
constexpr size_t sample_smem_bytes() {  // (independent of the row element type)
    return kWarps * sizeof(WarpSmem<LPT * KPL, KPL>);
}

// ---------------------------------------------------------------- end of wave: n and z
// n_{d k0} -= 1, n_{d k*} += 1 for every token of the wave that moved; zr <- zr_next.
template <typename NT>
__global__ void apply_tokens_kernel(const uint32_t* __restrict__ tok_doc, uint16_t* __restrict__ zr,
                                    const uint16_t* __restrict__ zr_next, NT* __restrict__ n,
                                    const int* __restrict__ sigma,
                                    int Kn, uint32_t begin, uint32_t end) {
    for (uint32_t p = begin + blockIdx.x * blockDim.x + threadIdx.x; p < end; p += gridDim.x * blockDim.x) {
        const uint32_t zo = zr[p], zn = zr_next[p];
        const uint32_t ko = zo & 0x7FFFu, kn = zn & 0x7FFFu;
        if (ko != kn) {
            const size_t r0 = (size_t)tok_doc[p] * Kn;
            Row<NT>::add(n, r0 + sigma[ko], -1);   // exact integer arithmetic
            Row<NT>::add(n, r0 + sigma[kn], 1);
        }
        zr[p] = (uint16_t)zn;
    }
}

// ---------------------------------------------------------------- end of wave: rows, clamp, sums
// For every (w, i) row: m += dm, t = clamp(t + dt) into [min(1,m), m]
// (PAPER.md:2411-2419 correction; reading c14), dm = dt = 0.  Then Q_w = sum_i t, and the
// marginal sums M, Tt, T are accumulated into zeroed buffers.
// One warp per word; int4 over topics.
__global__ void merge_rows_kernel(int32_t* __restrict__ m, int32_t* __restrict__ t,
                                  int32_t* __restrict__ dm, int32_t* __restrict__ dt,
                                  int32_t* __restrict__ Q, int32_t* __restrict__ M, int32_t* __restrict__ Tt,
                                  int32_t* __restrict__ T, int V, int I, int Kp, int use_smem_sums,
                                  unsigned long long* __restrict__ stats, int clamp_all) {
    extern __shared__ __align__(16) int ssum[];      // [2][I][Kp] + [Kp] when use_smem_sums
    int* sM = ssum;
    int* sT = ssum + (size_t)I * Kp;
    int* sK = ssum + (size_t)2 * I * Kp;
    if (use_smem_sums) {
        for (int j = threadIdx.x; j < (2 * I + 1) * Kp; j += blockDim.x) ssum[j] = 0;
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    unsigned clamped = 0;
    for (int w = blockIdx.x * wpb + (threadIdx.x >> 5); w < V; w += gridDim.x * wpb) {
        for (int k4 = lane * 4; k4 < Kp; k4 += 128) {
            int4 q = make_int4(0, 0, 0, 0);
            for (int i = 0; i < I; ++i) {
                const size_t off = ((size_t)w * I + i) * Kp + k4;
                int4 vm = *reinterpret_cast<const int4*>(m + off);
                int4 vt = *reinterpret_cast<const int4*>(t + off);
                const int4 a = dm ? *reinterpret_cast<const int4*>(dm + off) : make_int4(0, 0, 0, 0);
                const int4 d = dt ? *reinterpret_cast<const int4*>(dt + off) : make_int4(0, 0, 0, 0);
                if (clamp_all || (a.x | a.y | a.z | a.w | d.x | d.y | d.z | d.w) != 0) {
                    int* pm = &vm.x; int* pt = &vt.x;
                    const int* pa = &a.x; const int* pd = &d.x;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int mv = pm[e] + pa[e];
                        const int raw = pt[e] + pd[e];
                        int tv = min(raw, mv);
                        tv = (mv > 0) ? max(tv, 1) : 0;
                        clamped += (tv != raw);
                        pm[e] = mv; pt[e] = tv;
                    }
                    *reinterpret_cast<int4*>(m + off) = vm;
                    *reinterpret_cast<int4*>(t + off) = vt;
                    if (dm) *reinterpret_cast<int4*>(dm + off) = make_int4(0, 0, 0, 0);
                    if (dt) *reinterpret_cast<int4*>(dt + off) = make_int4(0, 0, 0, 0);
                }
                q.x += vt.x; q.y += vt.y; q.z += vt.z; q.w += vt.w;
                const int* pm = &vm.x; const int* pt = &vt.x;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (pm[e]) {
                        if (use_smem_sums) { atomicAdd(sM + (size_t)i * Kp + k4 + e, pm[e]); atomicAdd(sT + (size_t)i * Kp + k4 + e, pt[e]); }
                        else { atomicAdd(M + (size_t)i * Kp + k4 + e, pm[e]); atomicAdd(Tt + (size_t)i * Kp + k4 + e, pt[e]); }
                    }
                }
            }
            *reinterpret_cast<int4*>(Q + (size_t)w * Kp + k4) = q;
            const int* pq = &q.x;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (pq[e]) { if (use_smem_sums) atomicAdd(sK + k4 + e, pq[e]); else atomicAdd(T + k4 + e, pq[e]); }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) clamped += __shfl_xor_sync(0xffffffffu, clamped, off);
    if (lane == 0 && clamped) atomicAdd(stats + 2, (unsigned long long)clamped);
    if (use_smem_sums) {
        __syncthreads();
        for (int j = threadIdx.x; j < I * Kp; j += blockDim.x) {
            if (sM[j]) atomicAdd(M + j, sM[j]);
            if (sT[j]) atomicAdd(Tt + j, sT[j]);
        }
        for (int j = threadIdx.x; j < Kp; j += blockDim.x) if (sK[j]) atomicAdd(T + j, sK[j]);
    }
}

// ---------------------------------------------------------------- end of sweep (W = 1): recount n
// With one wave every token has a new z in zr_next, so the doc-topic rows are
// rebuilt from it (n, m "can be re-generated from topic
// assignments") instead of two scattered atomics per moved token: one warp per
// document, a shared-memory histogram over the document's tokens (CSR index in
// sorted-token positions), one coalesced row write in sigma order.
// LPD lanes per document (32, or 16 for short documents: two documents per warp keep twice the
// scattered assignment loads in flight per warp; B200, C5 (62 tokens per document) 3.6 -> see DESIGN).
template <typename NT, int LPD = 32>
__global__ void recount_docs_kernel(const uint32_t* __restrict__ doc_ptr, const uint32_t* __restrict__ doc_pos,
                                    const uint16_t* __restrict__ zr, const int* __restrict__ sigma, int D, int Kn,
                                    NT* __restrict__ n, const uint16_t* __restrict__ zr_doc) {
    constexpr int DPW = 32 / LPD;                    // documents per warp and step
    extern __shared__ int hist[];                    // [warps][DPW][Kn] (row positions; the padding stays 0)
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int sub = lane / LPD, sl = lane % LPD;
    int* h = hist + ((size_t)(threadIdx.x >> 5) * DPW + sub) * Kn;
    const int nsteps = (D + DPW - 1) / DPW;
    for (int ds = blockIdx.x * wpb + (threadIdx.x >> 5); ds < nsteps; ds += gridDim.x * wpb) {   // warp-uniform
        const int d = ds * DPW + sub;
        for (int j = sl; j < Kn; j += LPD) h[j] = 0;
        __syncwarp();
        if (d < D) {
            const uint32_t e = doc_ptr[d + 1];
            if (zr_doc) {   // the sample kernel already wrote the assignments in document order: stream them
                for (uint32_t t = doc_ptr[d] + sl; t < e; t += LPD) atomicAdd(&h[sigma[zr_doc[t] & 0x7FFFu]], 1);
            } else
            // 4 tokens per lane in flight: the positions, then the scattered assignments, then the histogram
            for (uint32_t t0 = doc_ptr[d]; t0 < e; t0 += 4 * LPD) {
                uint32_t pos[4];
                uint32_t zv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t t = t0 + sl + (uint32_t)LPD * j;
                    pos[j] = t < e ? doc_pos[t] : 0xFFFFFFFFu;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) zv[j] = pos[j] != 0xFFFFFFFFu ? (uint32_t)zr[pos[j]] : 0xFFFFFFFFu;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (zv[j] != 0xFFFFFFFFu) atomicAdd(&h[sigma[zv[j] & 0x7FFFu]], 1);
            }
        }
        __syncwarp();
        if (d < D) {
            NT* row = n + (size_t)d * Kn;
            for (int j = sl * 4; j < Kn; j += 4 * LPD) Row<NT>::store4(row + j, h[j], h[j + 1], h[j + 2], h[j + 3]);
        }
        __syncwarp();
    }
}

// Multi-GPU merge (Alg.3; reading c14/c15).
// Each rank's net change of a cell since the sweep start, D = (dm, dt), is
// carried as ONE integer: dm * 2^B + dt with B = 16 (int32, valid when every
// |sum of D over ranks| < 2^15, i.e. max_{i,w} count(i,w) < 2^15) or B = 32
// (int64).  Integer addition of packed words is the packed addition of both
// halves (two's complement wraps cancel), so one all-reduce of the packed
// buffer sums dm and dt at once: half the NVLink bytes of two int32 arrays.
template <typename P> struct Packed;
template <> struct Packed<int32_t> {
    __device__ static void add4(int32_t* p, const int* cm, const int* ct) {
        int4 x = *reinterpret_cast<int4*>(p);
        x.x = (int)((unsigned)x.x + ((unsigned)cm[0] << 16) + (unsigned)ct[0]);
        x.y = (int)((unsigned)x.y + ((unsigned)cm[1] << 16) + (unsigned)ct[1]);
        x.z = (int)((unsigned)x.z + ((unsigned)cm[2] << 16) + (unsigned)ct[2]);
        x.w = (int)((unsigned)x.w + ((unsigned)cm[3] << 16) + (unsigned)ct[3]);
        *reinterpret_cast<int4*>(p) = x;
    }
    __device__ static void load4(const int32_t* p, int* dm, int* dt) {
        const int4 x = *reinterpret_cast<const int4*>(p);
        const int v[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            dt[e] = (int)(short)(v[e] & 0xFFFF);
            dm[e] = (int)((unsigned)v[e] - (unsigned)dt[e]) >> 16;
        }
    }
    __device__ static bool zero4(const int32_t* p) {
        const int4 x = *reinterpret_cast<const int4*>(p);
        return (x.x | x.y | x.z | x.w) == 0;
    }
    __device__ static void clear4(int32_t* p) { *reinterpret_cast<int4*>(p) = make_int4(0, 0, 0, 0); }
};
template <> struct Packed<long long> {
    __device__ static void add4(long long* p, const int* cm, const int* ct) {
        longlong2* q = reinterpret_cast<longlong2*>(p);
        longlong2 a = q[0], b = q[1];
        a.x = (long long)((unsigned long long)a.x + ((unsigned long long)(long long)cm[0] << 32) + (unsigned long long)(long long)ct[0]);
        a.y = (long long)((unsigned long long)a.y + ((unsigned long long)(long long)cm[1] << 32) + (unsigned long long)(long long)ct[1]);
        b.x = (long long)((unsigned long long)b.x + ((unsigned long long)(long long)cm[2] << 32) + (unsigned long long)(long long)ct[2]);
        b.y = (long long)((unsigned long long)b.y + ((unsigned long long)(long long)cm[3] << 32) + (unsigned long long)(long long)ct[3]);
        q[0] = a; q[1] = b;
    }
    __device__ static void load4(const long long* p, int* dm, int* dt) {
        const longlong2* q = reinterpret_cast<const longlong2*>(p);
        const longlong2 a = q[0], b = q[1];
        const long long v[4] = {a.x, a.y, b.x, b.y};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            dt[e] = (int)(v[e] & 0xFFFFFFFFll);
            dm[e] = (int)((long long)((unsigned long long)v[e] - (unsigned long long)(long long)dt[e]) >> 32);
        }
    }
    __device__ static bool zero4(const long long* p) {
        const longlong2* q = reinterpret_cast<const longlong2*>(p);
        const longlong2 a = q[0], b = q[1];
        return (a.x | a.y | b.x | b.y) == 0;
    }
    __device__ static void clear4(long long* p) {
        longlong2* q = reinterpret_cast<longlong2*>(p);
        q[0] = make_longlong2(0, 0); q[1] = make_longlong2(0, 0);
    }
};

// ---------------------------------------------------------------- end of wave: touched rows only
// One warp per (w, i) segment the wave touched: m += dm, t = clamp(t + dt) into
// [min(1,m), m], dm = dt = 0; the changes are added to Q_w (int atomics) and to
// the marginal sums M, Tt, T (block-reduced in smem, then int atomics), and to
// the net-change buffer D when there is one (multi-GPU).  Integer arithmetic:
// the result does not depend on the order of the atomics.
__global__ void merge_segments_kernel(const uint32_t* __restrict__ segs, int nseg,
                                      int32_t* __restrict__ m, int32_t* __restrict__ t,
                                      int32_t* __restrict__ dm, int32_t* __restrict__ dt,
                                      void* __restrict__ D, int pack32,
                                      int32_t* __restrict__ Q, int32_t* __restrict__ M, int32_t* __restrict__ Tt,
                                      int32_t* __restrict__ T, int I, int Kp, int use_smem_sums,
                                      unsigned long long* __restrict__ stats, int packed_deltas, int fold) {
    // fold (several ranks, W = 1, the exchange follows): the rows keep the sweep-start S0 and only the
    // rank's net change D = clamp(S0 + delta) - S0 is written; the exchange merge installs clamp(S0 + sum D)
    // and rebuilds Q and the sums, so the local row writes and sum updates would be overwritten anyway
    extern __shared__ __align__(16) int ssum[];      // [2][I][Kp] + [Kp] when use_smem_sums
    int* sM = ssum;
    int* sT = ssum + (size_t)I * Kp;
    int* sK = ssum + (size_t)2 * I * Kp;
    if (use_smem_sums) {
        for (int j = threadIdx.x; j < (2 * I + 1) * Kp; j += blockDim.x) ssum[j] = 0;
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    unsigned clamped = 0;
    for (int j = blockIdx.x * wpb + (threadIdx.x >> 5); j < nseg; j += gridDim.x * wpb) {
        const uint32_t seg = segs[j];
        const int w = (int)(seg / (uint32_t)I), i = (int)(seg % (uint32_t)I);
        for (int k4 = lane * 4; k4 < Kp; k4 += 128) {
            const size_t off = (size_t)seg * Kp + k4;
            int4 a = *reinterpret_cast<const int4*>(dm + off);
            int4 d = packed_deltas ? make_int4(0, 0, 0, 0) : *reinterpret_cast<const int4*>(dt + off);
            // the rows are loaded with the deltas (one round trip; most touched rows change at W = 1)
            int4 vm = *reinterpret_cast<const int4*>(m + off);
            int4 vt = *reinterpret_cast<const int4*>(t + off);
            if ((a.x | a.y | a.z | a.w | d.x | d.y | d.z | d.w) == 0) continue;
            if (packed_deltas) {                             // dm * 2^16 + dt (token kernel)
                int* pa = &a.x; int* pd = &d.x;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int x = pa[e];
                    pd[e] = (int)(short)(x & 0xFFFF);
                    pa[e] = (int)((unsigned)x - (unsigned)pd[e]) >> 16;
                }
            }
            const int4 om = vm, ot = vt;
            int* pm = &vm.x; int* pt = &vt.x;
            const int* pa = &a.x; const int* pd = &d.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int mv = pm[e] + pa[e];
                const int raw = pt[e] + pd[e];
                int tv = min(raw, mv);
                tv = (mv > 0) ? max(tv, 1) : 0;
                clamped += (tv != raw);
                pm[e] = mv; pt[e] = tv;
            }
            if (!fold) {
                *reinterpret_cast<int4*>(m + off) = vm;
                *reinterpret_cast<int4*>(t + off) = vt;
            }
            *reinterpret_cast<int4*>(dm + off) = make_int4(0, 0, 0, 0);
            if (!packed_deltas) *reinterpret_cast<int4*>(dt + off) = make_int4(0, 0, 0, 0);
            const int cm[4] = {vm.x - om.x, vm.y - om.y, vm.z - om.z, vm.w - om.w};
            const int ct[4] = {vt.x - ot.x, vt.y - ot.y, vt.z - ot.z, vt.w - ot.w};
            if (D) {
                if (pack32) Packed<int32_t>::add4(reinterpret_cast<int32_t*>(D) + off, cm, ct);
                else Packed<long long>::add4(reinterpret_cast<long long*>(D) + off, cm, ct);
            }
            if (fold) continue;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (ct[e]) {
                    atomicAdd(Q + (size_t)w * Kp + k4 + e, ct[e]);
                    if (use_smem_sums) { atomicAdd(sT + (size_t)i * Kp + k4 + e, ct[e]); atomicAdd(sK + k4 + e, ct[e]); }
                    else { atomicAdd(Tt + (size_t)i * Kp + k4 + e, ct[e]); atomicAdd(T + k4 + e, ct[e]); }
                }
                if (cm[e]) {
                    if (use_smem_sums) atomicAdd(sM + (size_t)i * Kp + k4 + e, cm[e]);
                    else atomicAdd(M + (size_t)i * Kp + k4 + e, cm[e]);
                }
            }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) clamped += __shfl_xor_sync(0xffffffffu, clamped, off);
    if (lane == 0 && clamped) atomicAdd(stats + 2, (unsigned long long)clamped);
    if (use_smem_sums) {
        __syncthreads();
        for (int j = threadIdx.x; j < I * Kp; j += blockDim.x) {
            if (sM[j]) atomicAdd(M + j, sM[j]);
            if (sT[j]) atomicAdd(Tt + j, sT[j]);
        }
        for (int j = threadIdx.x; j < Kp; j += blockDim.x) if (sK[j]) atomicAdd(T + j, sK[j]);
    }
}

// Async mode with several ranks: D = (m - m0, t - t0) packed, from the sweep-start
// copy (m0, t0) kept in the otherwise unused wave-delta buffers, which are zeroed.
template <typename P>
__global__ void net_change_kernel(const int32_t* __restrict__ m, const int32_t* __restrict__ t,
                                  int32_t* __restrict__ m0, int32_t* __restrict__ t0, P* __restrict__ D, size_t cells) {
    for (size_t j = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 4; j < cells; j += (size_t)gridDim.x * blockDim.x * 4) {
        const int4 a = *reinterpret_cast<const int4*>(m + j), b = *reinterpret_cast<const int4*>(t + j);
        const int4 a0 = *reinterpret_cast<const int4*>(m0 + j), b0 = *reinterpret_cast<const int4*>(t0 + j);
        const int cm[4] = {a.x - a0.x, a.y - a0.y, a.z - a0.z, a.w - a0.w};
        const int ct[4] = {b.x - b0.x, b.y - b0.y, b.z - b0.z, b.w - b0.w};
        Packed<P>::clear4(D + j);
        Packed<P>::add4(D + j, cm, ct);
        *reinterpret_cast<int4*>(m0 + j) = make_int4(0, 0, 0, 0);
        *reinterpret_cast<int4*>(t0 + j) = make_int4(0, 0, 0, 0);
    }
}

// After the all-reduce (out of place: Dloc = this rank's D, Dsum = sum over
// ranks): m = (m - dm_loc) + dm_sum, t = clamp((t - dt_loc) + dt_sum) into
// [min(1,m), m]; Dloc = 0; Q_w = sum_i t and the rows' contributions to the
// marginal sums M, Tt, T (added into the given buffers).  Words [w0, w1): one
// pass over their rows, one warp per word.
template <typename P>
__global__ void exchange_merge_kernel(int32_t* __restrict__ m, int32_t* __restrict__ t, P* __restrict__ Dloc,
                                      const P* __restrict__ Dsum, int32_t* __restrict__ Q, int32_t* __restrict__ M,
                                      int32_t* __restrict__ Tt, int32_t* __restrict__ T, int w0, int w1, int I, int Kp,
                                      int use_smem_sums, unsigned long long* __restrict__ stats, int rows_s0) {
    extern __shared__ __align__(16) int ssum[];      // [2][I][Kp] + [Kp] when use_smem_sums
    int* sM = ssum;
    int* sT = ssum + (size_t)I * Kp;
    int* sK = ssum + (size_t)2 * I * Kp;
    if (use_smem_sums) {
        for (int j = threadIdx.x; j < (2 * I + 1) * Kp; j += blockDim.x) ssum[j] = 0;
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    unsigned clamped = 0;
    for (int w = w0 + blockIdx.x * wpb + (threadIdx.x >> 5); w < w1; w += gridDim.x * wpb) {
        for (int k4 = lane * 4; k4 < Kp; k4 += 128) {
            int4 q = make_int4(0, 0, 0, 0);
            for (int i = 0; i < I; ++i) {
                const size_t off = ((size_t)w * I + i) * Kp + k4;
                int4 vm = *reinterpret_cast<const int4*>(m + off);
                int4 vt = *reinterpret_cast<const int4*>(t + off);
                const bool lz = Packed<P>::zero4(Dloc + off), sz = Packed<P>::zero4(Dsum + off);
                if (!(lz && sz)) {
                    int lm[4], lt[4], gm[4], gt[4];
                    Packed<P>::load4(Dloc + off, lm, lt);
                    Packed<P>::load4(Dsum + off, gm, gt);
                    int* pm = &vm.x; int* pt = &vt.x;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int mv = pm[e] - (rows_s0 ? 0 : lm[e]) + gm[e];   // rows_s0: the rows are S0 (fold)
                        const int raw = pt[e] - (rows_s0 ? 0 : lt[e]) + gt[e];
                        int tv = min(raw, mv);
                        tv = (mv > 0) ? max(tv, 1) : 0;
                        clamped += (tv != raw);
                        pm[e] = mv; pt[e] = tv;
                    }
                    *reinterpret_cast<int4*>(m + off) = vm;
                    *reinterpret_cast<int4*>(t + off) = vt;
                    if (!lz) Packed<P>::clear4(Dloc + off);
                }
                q.x += vt.x; q.y += vt.y; q.z += vt.z; q.w += vt.w;
                const int* pm = &vm.x; const int* pt = &vt.x;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (pm[e]) {
                        if (use_smem_sums) { atomicAdd(sM + (size_t)i * Kp + k4 + e, pm[e]); atomicAdd(sT + (size_t)i * Kp + k4 + e, pt[e]); }
                        else { atomicAdd(M + (size_t)i * Kp + k4 + e, pm[e]); atomicAdd(Tt + (size_t)i * Kp + k4 + e, pt[e]); }
                    }
                }
            }
            *reinterpret_cast<int4*>(Q + (size_t)w * Kp + k4) = q;
            const int* pq = &q.x;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (pq[e]) { if (use_smem_sums) atomicAdd(sK + k4 + e, pq[e]); else atomicAdd(T + k4 + e, pq[e]); }
        }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) clamped += __shfl_xor_sync(0xffffffffu, clamped, off);
    if (lane == 0 && clamped) atomicAdd(stats + 2, (unsigned long long)clamped);
    if (use_smem_sums) {
        __syncthreads();
        for (int j = threadIdx.x; j < I * Kp; j += blockDim.x) {
            if (sM[j]) atomicAdd(M + j, sM[j]);
            if (sT[j]) atomicAdd(Tt + j, sT[j]);
        }
        for (int j = threadIdx.x; j < Kp; j += blockDim.x) if (sK[j]) atomicAdd(T + j, sK[j]);
    }
}

__global__ void inc_sweep_kernel(uint32_t* sweep) { *sweep += 1; }

// pos[perm[q]] = q (canonical id -> sorted position)
__global__ void invert_perm_kernel(const uint32_t* __restrict__ perm, uint32_t n, uint32_t* __restrict__ pos) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) pos[perm[q]] = q;
}

// ---------------------------------------------------------------- state installation
// initial topics z_p = floor(x0 K / 2^32) of Philox(seed; p, 0xFFFFFFFF, 0, 0) (reading c11)
__global__ void init_z_kernel(int32_t* __restrict__ z, uint32_t n, int K, uint32_t k0, uint32_t k1) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const uint4 x = philox(make_uint4(p, 0xFFFFFFFFu, 0u, 0u), k0, k1);
        z[p] = (int32_t)(((uint64_t)x.x * (uint64_t)K) >> 32);
    }
}
// first invalid z (err[0]) and r (err[1]) index
__global__ void check_zr_kernel(const int32_t* __restrict__ z, const uint8_t* __restrict__ r, uint32_t n, int K,
                                unsigned long long* __restrict__ err) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        if (z[p] < 0 || z[p] >= K) atomicMin(err, (unsigned long long)p);
        if (r && r[p] > 1) atomicMin(err + 1, (unsigned long long)p);
    }
}

// counts from z: m_{ikw} and, with given r, t_{ikw} = sum r
__global__ void init_cells_kernel(const int32_t* __restrict__ group, const int32_t* __restrict__ word,
                                  const int32_t* __restrict__ z, const uint8_t* __restrict__ r, uint32_t n, int I,
                                  int Kp, int32_t* __restrict__ m, int32_t* __restrict__ t, uint32_t* __restrict__ first) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const size_t cell = ((size_t)word[p] * I + group[p]) * Kp + z[p];
        atomicAdd(m + cell, 1);
        if (r) { if (r[p]) atomicAdd(t + cell, 1); }
        else atomicMin(first + cell, p);
    }
}
// default r: the first token (canonical order) of each cell opens its table (reading c12)
__global__ void init_first_table_kernel(const int32_t* __restrict__ group, const int32_t* __restrict__ word,
                                        const int32_t* __restrict__ z, uint32_t n, int I, int Kp,
                                        const uint32_t* __restrict__ first, uint8_t* __restrict__ r,
                                        int32_t* __restrict__ t) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const size_t cell = ((size_t)word[p] * I + group[p]) * Kp + z[p];
        const bool f = first[cell] == p;
        r[p] = f ? 1 : 0;
        if (f) t[cell] = 1;
    }
}
// tables given as [I][V][K] (spdp_set_state): transpose into [V][I][Kp]
__global__ void load_tables_kernel(const int32_t* __restrict__ tin, int I, int V, int K, int Kp, int32_t* __restrict__ t) {
    const size_t total = (size_t)I * V * K;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < total; j += (size_t)gridDim.x * blockDim.x) {
        const int k = (int)(j % K);
        const size_t iw = j / K;
        const int w = (int)(iw % V), i = (int)(iw / V);
        t[((size_t)w * I + i) * Kp + k] = tin[j];
    }
}
// count cells violating 0 <= t <= m, t > 0 iff m > 0
__global__ void check_cells_kernel(const int32_t* __restrict__ m, const int32_t* __restrict__ t, size_t cells,
                                   unsigned long long* __restrict__ bad) {
    unsigned long long nb = 0;
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < cells; j += (size_t)gridDim.x * blockDim.x)
        nb += (t[j] < 0 || t[j] > m[j] || ((t[j] > 0) != (m[j] > 0)));
    if (nb) atomicAdd(bad, nb);
}
// this rank's token records (sorted order) and doc-topic counts
template <typename NT>
__global__ void init_local_kernel(const uint32_t* __restrict__ tok_id, const uint32_t* __restrict__ tok_doc,
                                  const int32_t* __restrict__ z, const uint8_t* __restrict__ r, uint32_t nloc, int Kn,
                                  const int* __restrict__ sigma,
                                  uint16_t* __restrict__ zr, uint16_t* __restrict__ zr_next, NT* __restrict__ n) {
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nloc; q += gridDim.x * blockDim.x) {
        const uint32_t p = tok_id[q];
        const uint16_t v = (uint16_t)(z[p] | (r[p] << 15));
        zr[q] = v; zr_next[q] = v;
        Row<NT>::add(n, (size_t)tok_doc[q] * Kn + sigma[z[p]], 1);
    }
}

// zr in canonical token order (for spdp_counts): out[id[p]] = zr[p] + 1 (0 = other rank)
__global__ void scatter_zr_kernel(const uint32_t* __restrict__ id, const uint16_t* __restrict__ zr, uint32_t n,
                                  uint16_t* __restrict__ out, uint32_t add = 1u) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
        out[id[p]] = (uint16_t)(zr[p] + add);
}

// one byte per token (K <= 128): z | r << 7
__global__ void scatter_zr8_kernel(const uint32_t* __restrict__ id, const uint16_t* __restrict__ zr, uint32_t n,
                                   uint8_t* __restrict__ out) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const uint32_t v = zr[p];
        out[id[p]] = (uint8_t)((v & 0x7Fu) | ((v >> 15) << 7));
    }
}

// ---------------------------------------------------------------- training perplexity
// One warp per chunk (all waves): phi^i_kw = (m - a t)/(b + M) + (b + a Tt)/(b + M) phi0_kw,
// phi0_kw = (beta + Q)/(V beta + T) (reading c16);
// per token log sum_k (n_dk + alpha_ik) phi^i_kw / (L_d + sum_k alpha_ik).
// Per-chunk fp64 partials (fixed order) -> deterministic final reduction.
template <int LPT, int KPL, typename NT>
__global__ void __launch_bounds__(kWarps * 32)
perplexity_kernel(SweepArgs A, const int32_t* __restrict__ doclen, const double* __restrict__ alpha_sum,
                  double* __restrict__ partial) {
    constexpr int TPW = 32 / LPT;
    constexpr int KSPAN = LPT * KPL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = blockIdx.x * kWarps + wid;
    if (c >= A.nchunks) return;
    double* sphi = reinterpret_cast<double*>(smem_raw) + (size_t)wid * KSPAN;
    const uint32_t seg = A.chunk_seg[c];
    const int I = A.I, K = A.K, Kp = A.Kp;
    const int w = (int)(seg / (uint32_t)I), i = (int)(seg % (uint32_t)I);
    const size_t row = (size_t)seg * Kp;
    const double a = A.disc64[i], b = A.conc64[i];
    for (int k = lane; k < KSPAN; k += 32) {
        double phi = 0.0;
        if (k < K) {
            const double Mk = A.M[(size_t)i * Kp + k], Tk = A.Tt[(size_t)i * Kp + k];
            const double phi0 = (A.beta64 + (double)A.Q[(size_t)w * Kp + k]) / (A.vbeta64 + (double)A.T[k]);
            phi = ((double)A.m[row + k] - a * (double)A.t[row + k]) / (b + Mk) + (b + a * Tk) / (b + Mk) * phi0;
        }
        sphi[k] = phi;
    }
    __syncwarp();
    const int g = lane / LPT, gl = lane % LPT, kb = gl * KPL;
    double al[KPL];
#pragma unroll
    for (int j = 0; j < KPL; ++j) al[j] = (kb + j < K) ? A.alpha64[(size_t)i * Kp + kb + j] : 0.0;
    const double asum = alpha_sum[i];
    double ll = 0.0;
    const uint32_t start = A.chunk_start[c], end = A.chunk_end[c];
    for (uint32_t base = start; base < end; base += TPW) {
        const uint32_t tok = base + g;
        const bool valid = tok < end;
        const uint32_t doc = valid ? A.tok_doc[tok] : 0u;
        const NT* nrow = reinterpret_cast<const NT*>(A.n) + (size_t)doc * A.Kn;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < KPL; ++j)
            if (kb + j < K) s += ((double)Row<NT>::load1(nrow + A.sigma[kb + j]) + al[j]) * sphi[kb + j];
#pragma unroll
        for (int off = LPT / 2; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, LPT);
        if (valid && gl == 0) ll += log(s / ((double)doclen[doc] + asum));
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) ll += __shfl_xor_sync(0xffffffffu, ll, off);
    if (lane == 0) partial[c] = ll;
}

// Fixed-order reduction of n doubles by one block (deterministic).
__global__ void reduce_fixed_kernel(const double* __restrict__ x, size_t n, double* __restrict__ out) {
    __shared__ double s[1024];
    double acc = 0.0;
    for (size_t j = threadIdx.x; j < n; j += blockDim.x) acc += x[j];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int h = blockDim.x / 2; h; h >>= 1) {
        if ((int)threadIdx.x < h) s[threadIdx.x] += s[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
}

}  // namespace spdp
