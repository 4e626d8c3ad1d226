// spdp.cu — host side of libspdp.so: the C ABI of include/spdp.h.
//
// Validation, document sharding, the word-major wave
// plan (PAPER.md:2289-2299 reorder as wave = l mod W), device memory, kernel
// launches, and the cross-GPU count exchange (Alg.3) over
// NCCL (dlopen'ed, so the library loads on hosts without NCCL).
// No CPU fallback exists: every step of the sweep runs in the kernels of
// spdp_device.cuh.
#include "../../include/spdp.h"
#include "spdp_device.cuh"
#include "spdp_loglik.cuh"
#include "spdp_eval.cuh"
#include "spdp_plan.cuh"
#include "spdp_token.cuh"
#include "spdp_sparse.cuh"
#include "spdp_seq.cuh"
#include "spdp_sprows.cuh"

// Doc-topic row element type of the context: fp32 (L2-resident arrays), uint16 or uint8 (HBM-bound
// arrays; uint8 when every document has < 256 tokens).  Runs the statement with NT bound to it.
#define SPDP_ROWS(rowb, ...)                                   \
    do {                                                       \
        if ((rowb) == 1) { using NT = uint8_t; __VA_ARGS__; }  \
        else if ((rowb) == 2) { using NT = uint16_t; __VA_ARGS__; } \
        else { using NT = float; __VA_ARGS__; }                \
    } while (0)

#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <thread>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace spdp;

namespace {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclUid { char b[128]; };
struct NcclApi {
    void* lib = nullptr;
    int (*CommInitRank)(void** comm, int nranks, NcclUid id, int rank) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
};
constexpr int kNcclInt32 = 2, kNcclInt64 = 4, kNcclFloat64 = 8, kNcclSum = 0;
// SPDP_NCCL_LIB: another implementation of the same symbols (tests/nccl_shim.c lets several
// processes share one GPU, which NCCL itself refuses)
void* open_nccl() {
    if (const char* e = getenv("SPDP_NCCL_LIB")) return dlopen(e, RTLD_NOW | RTLD_LOCAL);
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    return lib;
}

// ------------------------------------------------------------------ host Philox4x32-10
void philox_host(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t p0 = (uint64_t)0xD2511F53u * x0, p1 = (uint64_t)0xCD9E8D57u * x2;
        const uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0, y1 = (uint32_t)p1;
        const uint32_t y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1, y3 = (uint32_t)p0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

// (lanes per token, topics per lane) by K: few lanes per token so the
// per-token fixed work (removal, scan, search) is shared by 32/LPT tokens.
int pick_lpt(int K) { return K <= 128 ? 4 : (K <= 256 ? 8 : (K <= 512 ? 16 : 32)); }
int pick_kpl(int K) {
    if (K <= 16) return 4;
    if (K <= 32) return 8;
    if (K <= 64) return 16;
    return 32;
}

template <typename T>
T* dalloc(size_t n, cudaError_t& e) {
    void* p = nullptr;
    if (n == 0) n = 1;
    e = cudaMalloc(&p, n * sizeof(T));
    return static_cast<T*>(p);
}

}  // namespace

struct spdp_ctx {
    spdp_config cfg{};
    std::string err;
    int I = 0, V = 0, K = 0, Kp = 0, W = 1, rank = 0, G = 1;
    std::vector<double> alpha_ik, disc, conc;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool loaded = false, poisoned = false;
    NcclApi nccl;
    void* comm = nullptr;
    int LPT = 32, KPL = 4, chunk_tokens = 32;

    // corpus (host)
    int64_t N = 0;
    int32_t D = 0;
    std::vector<int32_t> group, doc, word, doclen, docgroup;
    std::vector<int32_t> shard_of_doc, local_of_doc, global_of_local;
    int64_t Nloc = 0;
    int32_t Dloc = 0;
    std::vector<uint32_t> sorted_tok;            // canonical id at each sorted position (lazy host copy)
    std::vector<int64_t> pos_of_tok;              // canonical id -> sorted position (-1: other rank; lazy)
    std::vector<uint32_t> wave_tok_begin, wave_chunk_begin;
    std::vector<uint32_t> wave_seg_begin;          // distinct (w, i) segments of each wave (d_wave_segs)
    uint32_t nchunks = 0, nsegs = 0;
    int mmax = 0;
    size_t cells = 0;
    // multi-GPU net change since the sweep start, packed dm*2^B + dt (B = 16: int32, else int64)
    void *d_Dloc = nullptr, *d_Dsum = nullptr;
    bool pack32 = true;
    // exchange pipelining (W = 1): the sweep runs in P word-range parts; part p's rows are
    // all-reduced and merged on comm_stream while part p+1 samples
    int P = 1;
    bool overlap = false;
    // bounded staleness (NEXT-3): exchange after every E waves; the sweep is nblocks exchange blocks
    int E = 1, nblocks = 1, block = 0, nwaves_eff = 1;
    std::vector<uint32_t> part_word, part_run, part_tok, part_chunk;   // [P + 1] boundaries
    cudaStream_t comm_stream = nullptr;
    std::vector<cudaEvent_t> part_ev;
    cudaEvent_t comm_done = nullptr;
    int32_t *d_Mn = nullptr, *d_Ttn = nullptr, *d_Tn = nullptr;    // deferred local sums (sampling reads the snapshot)
    int32_t *d_Mf = nullptr, *d_Ttf = nullptr, *d_Tf = nullptr;    // sums after the pipelined exchange
    size_t xcount() const { return sparse ? cells + (size_t)E_sp * Kp : cells; }   // exchange buffer elements
    size_t dbytes() const { return xcount() * (pack32 ? 4 : 8); }

    // device
    uint32_t *d_tok_doc = nullptr, *d_tok_id = nullptr, *d_chunk_start = nullptr, *d_chunk_end = nullptr,
             *d_chunk_seg = nullptr, *d_wave_segs = nullptr,
             *d_sweep = nullptr;
    uint16_t *d_zr = nullptr, *d_zr_next = nullptr;
    int32_t *d_group = nullptr, *d_doc = nullptr, *d_word = nullptr;   // canonical token triples (all ranks' tokens)
    uint32_t *d_doc_ptr = nullptr, *d_doc_pos = nullptr;   // CSR: sorted-token positions of each local doc
    void* d_n = nullptr;                          // n_dk rows in sigma order: fp32, uint16 or uint8 (row_elem)
    int row_elem = 4;                             // bytes per doc-topic count: 4 (fp32), 2 (uint16), 1 (uint8)
    bool async = false;                           // SPDP_UPDATE_ASYNC (NEXT-2): immediate count updates
    bool sprows = false;                          // sample from sparse doc-topic rows (spdp_sprows.cuh)
    int sp_lpt = 8, sp_kspan = 256, sprows_grid = 0;
    uint32_t* d_cap_ptr = nullptr;                // [D_local] first entry slot of each document (capacity min(L_d, K))
    uint32_t* d_ent = nullptr;                    // entries k | n << 16
    uint2* d_dinfo = nullptr;                     // {first entry, nonzero topics}
    bool seq = false;                             // num_waves = 0: exact sequential sampler (test mode, spdp_seq.cuh)
    uint32_t* d_pos = nullptr;                    // seq: canonical id -> sorted position
    bool token_kernel = false;                    // K <= 64: one lane per token (spdp_token.cuh)
    bool pack_dmt = false;                        // chunk kernels flush packed dm * 2^16 + dt words (M_max < 2^15)
    bool chunk_ft = false;                        // chunk kernel reads per-wave factor tables (SPDP_CHUNK_FACTORS)
    bool doc_scatter = false;
    int recount_lpd = 32;                         // W = 1 recount: lanes per document (16 for short documents)                     // W = 1 chunk kernel also writes zr in document order (recount streams it)
    bool fold_merge = false;                      // several ranks, W = 1: the local merge writes only the net change
    uint32_t* d_slot = nullptr;                   // document-order slot of each sorted token
    uint16_t* d_zr_doc = nullptr;
    uint32_t* d_tok_run = nullptr;                // run (segment of a wave) of each sorted token
    float* d_F = nullptr;                         // token kernel: slot factors [run][Kp]
    float* d_R1 = nullptr;                        // token kernel: r = 1 shares [run][Kp]
    float* d_aF = nullptr;                        // token kernel: alpha F [run][Kp]
    uint32_t* d_MT = nullptr;                     // token kernel: snapshot m << 16 | t [run][Kp]
    float4* d_FR = nullptr;                       // token kernel: own-removal factor parts [run][Kp]
    // NEXT-4: sparse transformation matrices P^i (spdp_set_transform)
    bool sparse = false;
    std::vector<int32_t> h_pptr, h_pv;            // caller's rows (i, w): i * V + w
    std::vector<double> h_pp;
    std::vector<uint32_t> dev_of_user;             // caller's entry -> device entry (segment order)
    std::vector<uint32_t> h_sptr;                  // device rows (segments w * I + i)
    uint32_t E_sp = 0;
    uint32_t* d_sptr = nullptr;
    int32_t *d_spv = nullptr, *d_best = nullptr, *d_q = nullptr, *d_dq = nullptr;
    float* d_spp = nullptr;
    double* d_spp64 = nullptr;                     // fp64 weights for the estimators
    int16_t* d_src = nullptr;
    int* d_sigma = nullptr;                       // [Kp] in-row position of topic k
    std::vector<int> sigma;
    int LA = 1, Kn = 4;                           // doc-topic rows: lanes with storage, row length (spdp_device.cuh)
    int prefetch_rows = 0;
    uint16_t* d_zr_canon = nullptr;               // spdp_counts staging (canonical order)
    cudaStream_t d2h_stream = nullptr;            // spdp_zr_async's copies (overlap the next sweep)
    uint8_t* d_zr8_canon = nullptr;               // spdp_zr8_async's staging buffer (z | r << 7)
    cudaStream_t side_stream = nullptr;           // W = 1: the recount beside the merge
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t zr_ready = nullptr, zr_copied = nullptr;
    bool zr_pending = false;                      // a queued copy may still read d_zr_canon
    uint16_t* h_zr_canon = nullptr;               // pinned host copy
    uint32_t* d_work = nullptr;                   // [W + 1] persistent-warp counters
    int sample_grid = 0;
    int32_t *d_m = nullptr, *d_t = nullptr, *d_Q = nullptr, *d_M = nullptr, *d_Tt = nullptr,
            *d_T = nullptr, *d_dm = nullptr, *d_dt = nullptr, *d_doclen = nullptr,
            *d_docgroup = nullptr;
    float *d_alpha = nullptr, *d_disc = nullptr, *d_conc = nullptr, *d_alpha_sum = nullptr;
    double *d_alpha64 = nullptr, *d_disc64 = nullptr, *d_conc64 = nullptr, *d_alpha_sum64 = nullptr;
    float2* d_tab = nullptr;
    uint64_t* d_tab_off = nullptr;
    std::vector<uint64_t> tab_off_host;
    unsigned long long* d_stats = nullptr;
    double *d_partial = nullptr, *d_scalar = nullptr;
    size_t partial_len = 0;
    uint32_t sweeps_done = 0;
    std::vector<void*> allocs;
    // the setup calls' temporaries come from this pool, which keeps freed memory mapped (release threshold
    // = max): the planning code synchronises after every CUB call, and the default pool would unmap and
    // remap the freed temporaries at each of those points
    cudaMemPool_t pool = nullptr;
    bool pooled_alloc = false;            // ALLOC from the pool (inside spdp_load_corpus)
    std::vector<void*> pooled;            // persistent buffers from the pool (freed stream-ordered at destroy)
    // profiling (spdp_profile)
    bool profiling = false;
    // one sweep captured as a CUDA graph and replayed (single rank): keyed by the zr buffer the sweep
    // starts from (W = 1 paths swap zr / zr_next every sweep) and by profiling (event nodes)
    struct SweepGraph {
        uint16_t* zr_at_start;
        bool prof, swaps;
        cudaGraphExec_t exec;
        int64_t launches;
        double sample_launches;
    };
    std::vector<SweepGraph> graphs;
    bool graphs_off = false;
    std::vector<cudaEvent_t> ev;          // 4 per wave + 2 for the exchange
    double acc[10] = {0};
    int64_t launches = 0;
};

namespace {

spdp_status fail(spdp_ctx* c, spdp_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) {
        c->err = buf;
        if (s == SPDP_ECUDA) c->poisoned = true;
    }
    return s;
}

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return fail(c, SPDP_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

// Persistent device buffers.  Inside spdp_load_corpus (c->pooled_alloc) they come from the context's pool
// on its stream, so they reuse the memory the planning temporaries already mapped instead of mapping more
// (every buffer allocated there is first used on c->stream, or after the load's final synchronisation).
template <typename T>
spdp_status alloc(spdp_ctx* c, T*& p, size_t n) {
    cudaError_t e;
    if (c->pool && c->pooled_alloc) {
        void* q = nullptr;
        e = cudaMallocFromPoolAsync(&q, std::max<size_t>(n, 1) * sizeof(T), c->pool, c->stream);
        p = static_cast<T*>(q);
        if (e == cudaSuccess) c->pooled.push_back(q);
    } else {
        p = dalloc<T>(n, e);
        if (e == cudaSuccess) c->allocs.push_back(p);
    }
    if (e != cudaSuccess) return fail(c, SPDP_ENOMEM, "cudaMalloc(%zu bytes): %s", n * sizeof(T), cudaGetErrorString(e));
    return SPDP_OK;
}
#define ALLOC(p, n)                                   \
    do {                                              \
        spdp_status s_ = alloc(c, p, (size_t)(n));    \
        if (s_ != SPDP_OK) return s_;                 \
    } while (0)

spdp_status nccl_check(spdp_ctx* c, int r, const char* what) {
    if (r != 0) return fail(c, SPDP_ENCCL, "%s: %s", what, c->nccl.GetErrorString ? c->nccl.GetErrorString(r) : "error");
    return SPDP_OK;
}

// ------------------------------------------------------------------ kernel dispatch
template <int LPT, int KPL, bool DBG>
void launch_sample_t(const SweepArgs& a, cudaStream_t s, int max_blocks, int rowb, bool async) {
    const size_t smem = sample_smem_bytes<LPT, KPL>();
    const int blocks = std::min((a.nchunks + kWarps - 1) / kWarps, max_blocks);
    if (blocks <= 0) return;
    if constexpr (!DBG) {
        if (async) {
            SPDP_ROWS(rowb, sample_kernel<LPT, KPL, false, NT, true><<<blocks, kWarps * 32, smem, s>>>(a));
            return;
        }
    }
    SPDP_ROWS(rowb, sample_kernel<LPT, KPL, DBG, NT><<<blocks, kWarps * 32, smem, s>>>(a));
}
template <int LPT, int KPL>
int resident_blocks_t() {
    int nb = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sample_kernel<LPT, KPL, false, float>, kWarps * 32,
                                                  sample_smem_bytes<LPT, KPL>());
    return std::max(nb, 1) * std::max(sms, 1);
}
template <int LPT, int KPL>
void set_attr_t() {
    const int smem = (int)sample_smem_bytes<LPT, KPL>();
    cudaFuncSetAttribute(sample_kernel<LPT, KPL, false, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sample_kernel<LPT, KPL, true, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sample_kernel<LPT, KPL, false, uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sample_kernel<LPT, KPL, true, uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sample_kernel<LPT, KPL, false, float, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sample_kernel<LPT, KPL, false, uint16_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sample_kernel<LPT, KPL, false, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sample_kernel<LPT, KPL, true, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(sample_kernel<LPT, KPL, false, uint8_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int psm = kWarps * LPT * KPL * (int)sizeof(double);
    cudaFuncSetAttribute(perplexity_kernel<LPT, KPL, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, psm);
    cudaFuncSetAttribute(perplexity_kernel<LPT, KPL, uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, psm);
    cudaFuncSetAttribute(perplexity_kernel<LPT, KPL, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, psm);
}
template <int LPT, int KPL>
void launch_ppl_t(const SweepArgs& a, const int32_t* doclen, const double* asum, double* partial, cudaStream_t s,
                  int rowb) {
    const size_t smem = (size_t)kWarps * LPT * KPL * sizeof(double);
    const int blocks = (a.nchunks + kWarps - 1) / kWarps;
    if (blocks <= 0) return;
    SPDP_ROWS(rowb, perplexity_kernel<LPT, KPL, NT><<<blocks, kWarps * 32, smem, s>>>(a, doclen, asum, partial));
}

// The (lanes per token) x (topics per lane) configurations pick_lpt / pick_kpl choose; the
// SPDP_KERNEL_CFG tuning shapes (1x16 ... 16x16) only with -DSPDP_TUNING_CFGS (compile time).
#ifdef SPDP_TUNING_CFGS
#define SPDP_DISPATCH_TUNING(CALL)                          \
        case 116: CALL(1, 16); break;                       \
        case 132: CALL(1, 32); break;                       \
        case 216: CALL(2, 16); break;                       \
        case 232: CALL(2, 32); break;                       \
        case 816: CALL(8, 16); break;                       \
        case 1616: CALL(16, 16); break;
#else
#define SPDP_DISPATCH_TUNING(CALL)
#endif
bool cfg_compiled(int lpt, int kpl) {
    switch (lpt * 100 + kpl) {
        case 404: case 408: case 416: case 432: case 832: case 1632: case 3232: return true;
#ifdef SPDP_TUNING_CFGS
        case 116: case 132: case 216: case 232: case 816: case 1616: return true;
#endif
        default: return false;
    }
}
#define SPDP_DISPATCH(LPT_, KPL_, CALL)                     \
    switch (LPT_ * 100 + KPL_) {                            \
        SPDP_DISPATCH_TUNING(CALL)                          \
        case 404: CALL(4, 4); break;                        \
        case 408: CALL(4, 8); break;                        \
        case 416: CALL(4, 16); break;                       \
        case 432: CALL(4, 32); break;                       \
        case 832: CALL(8, 32); break;                       \
        case 1632: CALL(16, 32); break;                     \
        case 3232: CALL(32, 32); break;                     \
        default: break;                                     \
    }

void launch_sample(spdp_ctx* c, const SweepArgs& a, bool dbg) {
#define CALL_S(L, P) (dbg ? launch_sample_t<L, P, true>(a, c->stream, c->sample_grid, c->row_elem, false) : launch_sample_t<L, P, false>(a, c->stream, c->sample_grid, c->row_elem, c->async))
    SPDP_DISPATCH(c->LPT, c->KPL, CALL_S)
#undef CALL_S
}
void set_attrs(spdp_ctx* c) {
#define CALL_A(L, P) set_attr_t<L, P>()
    SPDP_DISPATCH(c->LPT, c->KPL, CALL_A)
#undef CALL_A
#define CALL_R(L, P) c->sample_grid = resident_blocks_t<L, P>()
    SPDP_DISPATCH(c->LPT, c->KPL, CALL_R)
#undef CALL_R
}
void launch_ppl(spdp_ctx* c, const SweepArgs& a, double* partial) {
#define CALL_P(L, P) launch_ppl_t<L, P>(a, c->d_doclen, c->d_alpha_sum64, partial, c->stream, c->row_elem)
    SPDP_DISPATCH(c->LPT, c->KPL, CALL_P)
#undef CALL_P
}

// the W = 1 doc-topic rows rebuilt from zr_next: 32 lanes per document, or 16 (two documents per warp)
// for short documents; zr_doc: the assignments already in document order (SPDP_DOC_SCATTER), or null
template <typename NT>
void launch_recount(spdp_ctx* c, cudaStream_t st, const uint16_t* zr_doc) {
    const size_t smem = sizeof(int) * 8 * 2 * (size_t)c->Kn;
    NT* n = reinterpret_cast<NT*>(c->d_n);
    if (c->recount_lpd == 16 && smem <= 48 * 1024)   // (two histograms per warp within the default smem limit)
        recount_docs_kernel<NT, 16><<<148 * 8, 256, smem, st>>>(c->d_doc_ptr, c->d_doc_pos, c->d_zr_next, c->d_sigma,
                                                               c->Dloc, c->Kn, n, zr_doc);
    else
        recount_docs_kernel<NT, 32><<<148 * 8, 256, smem / 2, st>>>(c->d_doc_ptr, c->d_doc_pos, c->d_zr_next,
                                                                   c->d_sigma, c->Dloc, c->Kn, n, zr_doc);
}

// K <= 64: factor table of the wave's segments, then one lane per token (spdp_token.cuh)
void launch_token(spdp_ctx* c, uint32_t r0, uint32_t r1, uint32_t tb, uint32_t te) {
    const size_t nf = (size_t)(r1 - r0) * c->Kp;
    const int fgrid = (int)std::min<size_t>((nf + 255) / 256, 148u * 16u);
    factor_kernel<<<std::max(fgrid, 1), 256, 0, c->stream>>>(
        c->d_wave_segs, r0, r1, c->d_m, c->d_t, c->d_Q, c->d_M, c->d_Tt, c->d_T, c->d_disc, c->d_conc, c->d_tab,
        c->d_tab_off, (float)c->cfg.beta, (float)((double)c->V * c->cfg.beta), c->I, c->K, c->Kp, c->d_F, c->d_R1,
        c->d_alpha, SPDP_TOKEN_PRE ? c->d_aF : nullptr, SPDP_TOKEN_PRE ? c->d_MT : nullptr, SPDP_TOKEN_PRE ? c->d_FR : nullptr);
    TokenArgs t{};
    t.aF = c->d_aF; t.MT = c->d_MT; t.FR = c->d_FR;
    t.tok_doc = c->d_tok_doc; t.tok_id = c->d_tok_id; t.tok_run = c->d_tok_run; t.run_seg = c->d_wave_segs;
    t.zr = c->d_zr; t.zr_next = c->d_zr_next; t.F = c->d_F; t.R1 = c->d_R1; t.n = c->d_n;
    t.sigma = c->d_sigma;
    for (int B = 0; B < 32; ++B) t.bpos[B] = (B < c->Kp / 4) ? c->sigma[(size_t)4 * B] / 4 : 0;
    t.m = c->d_m; t.t = c->d_t; t.Q = c->d_Q; t.M = c->d_M; t.Tt = c->d_Tt; t.T = c->d_T; t.dmt = c->d_dm;
    t.alpha = c->d_alpha; t.disc = c->d_disc; t.conc = c->d_conc; t.tab = c->d_tab; t.tab_off = c->d_tab_off;
    t.beta = (float)c->cfg.beta; t.vbeta = (float)((double)c->V * c->cfg.beta);
    t.I = c->I; t.K = c->K; t.Kp = c->Kp; t.Kn = c->Kn;
    t.key0 = (uint32_t)c->cfg.seed; t.key1 = (uint32_t)(c->cfg.seed >> 32);
    t.sweep = c->d_sweep; t.begin = tb; t.end = te; t.stats = c->d_stats;
    // two full waves of the resident blocks (grid-stride loop)
    const int grid = (int)std::min<uint32_t>((te - tb + 255) / 256, 148u * 2u * SPDP_TOKEN_MINB);
    const int nbk = (c->K + 3) / 4;
    const size_t tsm = nbk > 16 ? sizeof(float) * 256 * 32 : 0;
#define SPDP_TOK(NBK)                                                                                   \
    do {                                                                                                \
        SPDP_ROWS(c->row_elem, token_kernel<NBK, NT><<<std::max(grid, 1), 256, tsm, c->stream>>>(t));  \
    } while (0)
    if (nbk <= 4) SPDP_TOK(4);
    else if (nbk <= 8) SPDP_TOK(8);
    else if (nbk <= 16) SPDP_TOK(16);
    else SPDP_TOK(32);
#undef SPDP_TOK
    c->launches += 1;
}

// chunk kernel with factor tables: the slot factors, r = 1 shares, alpha F and packed (m, t) of the runs
// [r0, r1) of a wave, written by one throughput kernel before the sample kernel reads them
void launch_chunk_factors(spdp_ctx* c, uint32_t r0, uint32_t r1) {
    const size_t nf = (size_t)(r1 - r0) * c->Kp;
    if (nf == 0) return;
    const int fgrid = (int)std::min<size_t>((nf + 255) / 256, 148u * 16u);
    factor_kernel<<<std::max(fgrid, 1), 256, 0, c->stream>>>(
        c->d_wave_segs, r0, r1, c->d_m, c->d_t, c->d_Q, c->d_M, c->d_Tt, c->d_T, c->d_disc, c->d_conc, c->d_tab,
        c->d_tab_off, (float)c->cfg.beta, (float)((double)c->V * c->cfg.beta), c->I, c->K, c->Kp, c->d_F, c->d_R1,
        c->d_alpha, c->d_aF, c->d_MT, nullptr);
    c->launches += 1;
}

SweepArgs base_args(spdp_ctx* c) {
    SweepArgs a{};
    a.tok_doc = c->d_tok_doc; a.tok_id = c->d_tok_id; a.zr = c->d_zr; a.zr_next = c->d_zr_next;
    a.chunk_start = c->d_chunk_start; a.chunk_end = c->d_chunk_end; a.chunk_seg = c->d_chunk_seg; a.nchunks = 0;
    a.n = c->d_n; a.sigma = c->d_sigma;
    a.LA = c->LA; a.Kn = c->Kn;
    a.prefetch_rows = c->prefetch_rows;
    a.m = c->d_m; a.t = c->d_t; a.Q = c->d_Q; a.M = c->d_M; a.Tt = c->d_Tt; a.T = c->d_T;
    a.dm = c->d_dm; a.dt = c->d_dt;
    a.alpha = c->d_alpha; a.disc = c->d_disc; a.conc = c->d_conc; a.tab = c->d_tab; a.tab_off = c->d_tab_off;
    a.beta = (float)c->cfg.beta; a.vbeta = (float)((double)c->V * c->cfg.beta);
    a.alpha64 = c->d_alpha64; a.disc64 = c->d_disc64; a.conc64 = c->d_conc64;
    a.beta64 = c->cfg.beta; a.vbeta64 = (double)c->V * c->cfg.beta;
    a.I = c->I; a.K = c->K; a.Kp = c->Kp;
    a.key0 = (uint32_t)c->cfg.seed; a.key1 = (uint32_t)(c->cfg.seed >> 32);
    a.sweep = c->d_sweep; a.stats = c->d_stats;
    a.dinfo = c->d_dinfo; a.ent = c->d_ent;
    a.packed_dmt = c->pack_dmt ? 1 : 0;
    a.chunk_ft = c->chunk_ft ? 1 : 0;
    a.slot = c->doc_scatter ? c->d_slot : nullptr;
    a.zr_doc = c->doc_scatter ? c->d_zr_doc : nullptr;
    a.tok_run = c->d_tok_run; a.Ft = c->d_F; a.R1t = c->d_R1; a.aFt = c->d_aF; a.MTt = c->d_MT;
    return a;
}

// ---- sparse doc-topic rows
#ifndef SPDP_CHUNK_FACTORS
#define SPDP_CHUNK_FACTORS 0          // default of c->chunk_ft (env SPDP_CHUNK_FACTORS overrides)
#endif
#ifndef SPDP_SPROWS_AUTO
#define SPDP_SPROWS_AUTO 0            // choose the sparse-row kernel automatically (else only SPDP_SPARSE_ROWS=1)
#endif
#define SPDP_SPROWS_DISPATCH(LPT_, KS_, CALL)               \
    switch ((LPT_) * 10000 + (KS_)) {                       \
        case 80256: CALL(8, 256); break;                    \
        case 160256: CALL(16, 256); break;                  \
        case 320256: CALL(32, 256); break;                  \
        case 80512: CALL(8, 512); break;                    \
        case 160512: CALL(16, 512); break;                  \
        case 320512: CALL(32, 512); break;                  \
        case 81024: CALL(8, 1024); break;                   \
        case 161024: CALL(16, 1024); break;                 \
        case 321024: CALL(32, 1024); break;                 \
        default: break;                                     \
    }
template <int LPT, int KS>
void sprows_setup_t(spdp_ctx* c) {
    const int smem = (int)sprow_smem_bytes<LPT, KS>();
    cudaFuncSetAttribute(sample_sprows_kernel<LPT, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int nb = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sample_sprows_kernel<LPT, KS>, kSpWarps * 32, smem);
    c->sprows_grid = std::max(nb, 1) * std::max(sms, 1);
}
template <int LPT, int KS>
void launch_sprows_t(spdp_ctx* c, const SweepArgs& a) {
    const int blocks = std::min((a.nchunks + kSpWarps - 1) / kSpWarps, c->sprows_grid);
    if (blocks <= 0) return;
    sample_sprows_kernel<LPT, KS><<<blocks, kSpWarps * 32, sprow_smem_bytes<LPT, KS>(), c->stream>>>(a);
}
void launch_sprows(spdp_ctx* c, const SweepArgs& a) {
#define CALL_SR(L, KS) launch_sprows_t<L, KS>(c, a)
    SPDP_SPROWS_DISPATCH(c->sp_lpt, c->sp_kspan, CALL_SR)
#undef CALL_SR
}
// entries of every local document from its dense row (after the W = 1 recount and state installation)
void rebuild_entries(spdp_ctx* c, cudaStream_t st) {
    if (!c->sprows || c->Dloc == 0) return;
    SPDP_ROWS(c->row_elem, rows_to_entries_kernel<NT><<<148 * 8, 256, 0, st>>>(
                               (const NT*)c->d_n, c->d_sigma, c->Dloc, c->K, c->Kn, c->d_cap_ptr, c->d_ent, c->d_dinfo));
    c->launches += 1;
}

int merge_grid() { return 148 * 4; }

// Temporaries of the setup calls: stream-ordered (cudaMallocAsync / cudaFreeAsync
// on the call's stream) inside a TempStream scope, so freeing one does not
// synchronise the device; plain cudaMalloc elsewhere.
thread_local cudaStream_t tl_temp_stream = nullptr;
thread_local cudaMemPool_t tl_temp_pool = nullptr;
struct TempStream {
    cudaStream_t prev;
    cudaMemPool_t prev_pool;
    explicit TempStream(cudaStream_t s, cudaMemPool_t pool = nullptr) : prev(tl_temp_stream), prev_pool(tl_temp_pool) {
        tl_temp_stream = s;
        tl_temp_pool = pool;
    }
    ~TempStream() { tl_temp_stream = prev; tl_temp_pool = prev_pool; }
};

template <typename T>
struct TempBuf {
    T* p = nullptr;
    cudaStream_t st = nullptr;
    explicit TempBuf(size_t n) : st(tl_temp_stream) {
        const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
        const cudaError_t e = (st && tl_temp_pool) ? cudaMallocFromPoolAsync((void**)&p, bytes, tl_temp_pool, st)
                              : st ? cudaMallocAsync((void**)&p, bytes, st) : cudaMalloc((void**)&p, bytes);
        if (e != cudaSuccess) { p = nullptr; cudaGetLastError(); }
    }
    ~TempBuf() { if (p) { if (st) cudaFreeAsync(p, st); else cudaFree(p); } }
    TempBuf(const TempBuf&) = delete;
    TempBuf& operator=(const TempBuf&) = delete;
};

// rows += (dm, dt), clamp, zero deltas, (D += change), recompute Q and sums
void launch_merge(spdp_ctx* c, int32_t* dm, int32_t* dt) {
    cudaMemsetAsync(c->d_M, 0, sizeof(int32_t) * (size_t)c->I * c->Kp, c->stream);
    cudaMemsetAsync(c->d_Tt, 0, sizeof(int32_t) * (size_t)c->I * c->Kp, c->stream);
    cudaMemsetAsync(c->d_T, 0, sizeof(int32_t) * (size_t)c->Kp, c->stream);
    const size_t smem = sizeof(int) * (size_t)(2 * c->I + 1) * c->Kp;
    const int use_smem = smem <= 48 * 1024;
    merge_rows_kernel<<<merge_grid(), 256, use_smem ? smem : 0, c->stream>>>(
        c->d_m, c->d_t, dm, dt, c->d_Q, c->d_M, c->d_Tt, c->d_T, c->V, c->I, c->Kp, use_smem, c->d_stats,
        dm == nullptr);
}

// after the all-reduce Dloc -> Dsum: rows of words [w0, w1) = S0 + sum of D, clamp, Dloc = 0,
// Q rows, and the rows' contributions to the sums added into (M, Tt, T)
void launch_exchange_merge_range(spdp_ctx* c, int w0, int w1, int32_t* M, int32_t* Tt, int32_t* T, cudaStream_t st) {
    const size_t smem = sizeof(int) * (size_t)(2 * c->I + 1) * c->Kp;
    const int use_smem = smem <= 48 * 1024;
    if (w1 <= w0) return;
    const int grid = std::min(merge_grid(), (w1 - w0 + 7) / 8);
    if (c->pack32)
        exchange_merge_kernel<int32_t><<<grid, 256, use_smem ? smem : 0, st>>>(
            c->d_m, c->d_t, (int32_t*)c->d_Dloc, (const int32_t*)c->d_Dsum, c->d_Q, M, Tt, T, w0, w1, c->I, c->Kp,
            use_smem, c->d_stats, (int)c->fold_merge);
    else
        exchange_merge_kernel<long long><<<grid, 256, use_smem ? smem : 0, st>>>(
            c->d_m, c->d_t, (long long*)c->d_Dloc, (const long long*)c->d_Dsum, c->d_Q, M, Tt, T, w0, w1, c->I, c->Kp,
            use_smem, c->d_stats, (int)c->fold_merge);
}
void sparse_exchange_merge(spdp_ctx* c);
void launch_exchange_merge(spdp_ctx* c) {
    if (c->sparse) { sparse_exchange_merge(c); return; }
    cudaMemsetAsync(c->d_M, 0, sizeof(int32_t) * (size_t)c->I * c->Kp, c->stream);
    cudaMemsetAsync(c->d_Tt, 0, sizeof(int32_t) * (size_t)c->I * c->Kp, c->stream);
    cudaMemsetAsync(c->d_T, 0, sizeof(int32_t) * (size_t)c->Kp, c->stream);
    launch_exchange_merge_range(c, 0, c->V, c->d_M, c->d_Tt, c->d_T, c->stream);
}

// SPDP_VERBOSE=1: phase times of spdp_load_corpus on stderr
struct LoadTimer {
    bool on = getenv("SPDP_VERBOSE") != nullptr;
    bool drain = on && atoi(getenv("SPDP_VERBOSE")) >= 2;   // SPDP_VERBOSE=2: wait for the device at each mark
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        if (drain) cudaDeviceSynchronize();
        auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[spdp] load %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

spdp_status check_launch(spdp_ctx* c, const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(c, SPDP_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return SPDP_OK;
}

spdp_status sync(spdp_ctx* c, const char* what) {
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(c, SPDP_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return SPDP_OK;
}

spdp_status guard(spdp_ctx* c, bool need_loaded) {
    if (!c) return SPDP_EINVAL;
    if (c->poisoned) return fail(c, SPDP_ESTATE, "context poisoned by an earlier CUDA fault: %s", c->err.c_str());
    if (need_loaded && !c->loaded) return fail(c, SPDP_ESTATE, "spdp_load_corpus has not been called");
    cudaError_t e = cudaSetDevice(c->cfg.device);
    if (e != cudaSuccess) return fail(c, SPDP_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
    return SPDP_OK;
}

// host doc -> rank split: docs ordered by Philox x0 of
// (doc, 0xFFFFFFFE) (ties by id), then rank = floor(tokens_before * G / N).
void partition_docs(uint64_t seed, int G, int64_t N, int32_t D, const std::vector<int32_t>& doclen,
                    std::vector<int32_t>& shard) {
    std::vector<std::pair<uint32_t, int32_t>> key((size_t)D);
    for (int32_t d = 0; d < D; ++d) {
        const uint32_t ctr[4] = {(uint32_t)d, 0xFFFFFFFEu, 0u, 0u};
        uint32_t x[4];
        philox_host(ctr, (uint32_t)seed, (uint32_t)(seed >> 32), x);
        key[(size_t)d] = {x[0], d};
    }
    std::sort(key.begin(), key.end());
    shard.assign((size_t)D, 0);
    int64_t before = 0;
    for (int32_t j = 0; j < D; ++j) {
        const int32_t d = key[(size_t)j].second;
        int64_t g = N > 0 ? (before * (int64_t)G) / N : 0;
        if (g >= G) g = G - 1;
        shard[(size_t)d] = (int32_t)g;
        before += doclen[(size_t)d];
    }
}

// Upload (z, r or tables) as the sampler state: counts from z.
size_t row_bytes(const spdp_ctx* c) {
    return ((size_t)c->Dloc * c->Kn + 1024) * (size_t)c->row_elem;
}

// doc-topic rows to the host as floats (sigma order, [Dloc][Kn])
spdp_status read_rows(spdp_ctx* c, std::vector<float>& out) {
    const size_t n = (size_t)c->Dloc * c->Kn;
    out.assign(n, 0.f);
    if (c->row_elem == 2) {
        std::vector<uint16_t> tmp(n);
        CU(cudaMemcpyAsync(tmp.data(), c->d_n, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, c->stream));
        spdp_status s = sync(c, "read rows");
        if (s) return s;
        for (size_t j = 0; j < n; ++j) out[j] = (float)tmp[j];
    } else if (c->row_elem == 1) {
        std::vector<uint8_t> tmp(n);
        CU(cudaMemcpyAsync(tmp.data(), c->d_n, n, cudaMemcpyDeviceToHost, c->stream));
        spdp_status s = sync(c, "read rows");
        if (s) return s;
        for (size_t j = 0; j < n; ++j) out[j] = (float)tmp[j];
    } else {
        CU(cudaMemcpyAsync(out.data(), c->d_n, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
        return sync(c, "read rows");
    }
    return SPDP_OK;
}

// run fn(begin, end) over [0, n) on the host cores
template <typename Fn>
void parallel_for(int64_t n, Fn fn) {
    int nt = (int)std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 32u);
    if (n < 1 << 16) nt = 1;
    std::vector<std::thread> th;
    const int64_t step = (n + nt - 1) / nt;
    for (int j = 0; j < nt; ++j) {
        const int64_t b = j * step, e = std::min(n, b + step);
        if (b < e) th.emplace_back(fn, b, e);
    }
    for (auto& x : th) x.join();
}

// Host copy of the plan's token order (diagnostics only: debug_probs, debug_verify).
spdp_status ensure_host_plan(spdp_ctx* c) {
    if ((int64_t)c->sorted_tok.size() == c->Nloc && (int64_t)c->pos_of_tok.size() == c->N &&
        (int64_t)c->doc.size() == c->N)
        return SPDP_OK;
    c->sorted_tok.resize((size_t)c->Nloc);
    if (c->Nloc > 0)
        CU(cudaMemcpy(c->sorted_tok.data(), c->d_tok_id, sizeof(uint32_t) * (size_t)c->Nloc, cudaMemcpyDeviceToHost));
    c->group.resize((size_t)c->N); c->doc.resize((size_t)c->N); c->word.resize((size_t)c->N);
    CU(cudaMemcpy(c->group.data(), c->d_group, sizeof(int32_t) * (size_t)c->N, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(c->doc.data(), c->d_doc, sizeof(int32_t) * (size_t)c->N, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(c->word.data(), c->d_word, sizeof(int32_t) * (size_t)c->N, cudaMemcpyDeviceToHost));
    c->pos_of_tok.assign((size_t)c->N, -1);
    parallel_for(c->Nloc, [&](int64_t b, int64_t e) {
        for (int64_t q = b; q < e; ++q) c->pos_of_tok[c->sorted_tok[(size_t)q]] = q;
    });
    return SPDP_OK;
}

void sparse_install(spdp_ctx* c);

// Upload (z, r or tables) as the sampler state; counts from z
// are built on the device.
spdp_status install_state(spdp_ctx* c, const int32_t* z_in, const uint8_t* r_in, const int32_t* tables) {
    const int I = c->I, V = c->V, K = c->K, Kp = c->Kp;
    const int64_t N = c->N;
    TempBuf<int32_t> dz(N);
    TempBuf<uint8_t> dr(N);
    TempBuf<uint32_t> dfirst(r_in ? 1 : c->cells);
    TempBuf<unsigned long long> dbad(1), dbadzr(2);
    if (!dz.p || !dr.p || !dfirst.p || !dbad.p || !dbadzr.p) return fail(c, SPDP_ENOMEM, "install_state buffers");
    int32_t* dg = c->d_group;
    int32_t* dw = c->d_word;
    // z: the caller's, or the Philox initial topics z_p = floor(x0 K / 2^32), counter (p, 0xFFFFFFFF) (reading c11)
    if (z_in) CU(cudaMemcpyAsync(dz.p, z_in, sizeof(int32_t) * (size_t)N, cudaMemcpyHostToDevice, c->stream));
    else init_z_kernel<<<148 * 8, 256, 0, c->stream>>>(dz.p, (uint32_t)N, K, (uint32_t)c->cfg.seed,
                                                       (uint32_t)(c->cfg.seed >> 32));
    if (r_in) CU(cudaMemcpyAsync(dr.p, r_in, (size_t)N, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemsetAsync(dbadzr.p, 0xFF, sizeof(unsigned long long) * 2, c->stream));
    check_zr_kernel<<<148 * 8, 256, 0, c->stream>>>(dz.p, r_in ? dr.p : nullptr, (uint32_t)N, K, dbadzr.p);
    {
        unsigned long long bz[2];
        CU(cudaMemcpyAsync(bz, dbadzr.p, sizeof(bz), cudaMemcpyDeviceToHost, c->stream));
        spdp_status s0 = sync(c, "install_state check");
        if (s0) return s0;
        if (bz[0] != ~0ull) return fail(c, SPDP_EINVAL, "z[%llu] out of [0, K)", bz[0]);
        if (bz[1] != ~0ull) return fail(c, SPDP_EINVAL, "r[%llu] not in {0,1}", bz[1]);
    }
    if (!r_in) CU(cudaMemsetAsync(dfirst.p, 0xFF, sizeof(uint32_t) * c->cells, c->stream));
    CU(cudaMemsetAsync(c->d_m, 0, sizeof(int32_t) * c->cells, c->stream));
    CU(cudaMemsetAsync(c->d_t, 0, sizeof(int32_t) * c->cells, c->stream));
    CU(cudaMemsetAsync(dbad.p, 0, sizeof(unsigned long long), c->stream));
    const int grid = 148 * 8;
    init_cells_kernel<<<grid, 256, 0, c->stream>>>(dg, dw, dz.p, r_in ? dr.p : nullptr, (uint32_t)N, I, Kp, c->d_m,
                                                   c->d_t, dfirst.p);
    if (!r_in)
        init_first_table_kernel<<<grid, 256, 0, c->stream>>>(dg, dw, dz.p, (uint32_t)N, I, Kp, dfirst.p, dr.p, c->d_t);
    if (tables) {
        TempBuf<int32_t> dt_in((size_t)I * V * K);
        if (!dt_in.p) return fail(c, SPDP_ENOMEM, "tables buffer");
        CU(cudaMemcpyAsync(dt_in.p, tables, sizeof(int32_t) * (size_t)I * V * K, cudaMemcpyHostToDevice, c->stream));
        load_tables_kernel<<<grid, 256, 0, c->stream>>>(dt_in.p, I, V, K, Kp, c->d_t);
        spdp_status s0 = sync(c, "load tables");
        if (s0) return s0;
    }
    check_cells_kernel<<<grid, 256, 0, c->stream>>>(c->d_m, c->d_t, c->cells, dbad.p);
    unsigned long long nbad = 0;
    CU(cudaMemcpyAsync(&nbad, dbad.p, sizeof(nbad), cudaMemcpyDeviceToHost, c->stream));
    spdp_status s = sync(c, "install_state cells");
    if (s) return s;
    if (nbad) return fail(c, SPDP_EINVAL, "table counts violate 1 <= t <= m on %llu occupied cell(s) (or t > 0 on an empty one)", nbad);
    CU(cudaMemsetAsync(c->d_n, 0, row_bytes(c), c->stream));
    if (c->Nloc > 0) {
        SPDP_ROWS(c->row_elem, init_local_kernel<NT><<<grid, 256, 0, c->stream>>>(
                                   c->d_tok_id, c->d_tok_doc, dz.p, dr.p, (uint32_t)c->Nloc, c->Kn, c->d_sigma, c->d_zr,
                                   c->d_zr_next, (NT*)c->d_n));
    }
    CU(cudaMemsetAsync(c->d_dm, 0, sizeof(int32_t) * c->cells, c->stream));
    CU(cudaMemsetAsync(c->d_dt, 0, sizeof(int32_t) * c->cells, c->stream));
    if (c->d_Dloc) CU(cudaMemsetAsync(c->d_Dloc, 0, c->dbytes(), c->stream));
    launch_merge(c, c->d_dm, c->d_dt);    // zero deltas: recomputes Q and the sums
    rebuild_entries(c, c->stream);
    if (c->sparse) sparse_install(c);
    s = check_launch(c, "install_state kernels");
    if (s) return s;
    return sync(c, "install_state");
}

spdp_status ensure_events(spdp_ctx* c) {
    const size_t need = 4 * (size_t)c->W + 2;
    while (c->ev.size() < need) {
        cudaEvent_t e;
        CU(cudaEventCreate(&e));
        c->ev.push_back(e);
    }
    return SPDP_OK;
}
inline void rec(spdp_ctx* c, size_t j) {
    if (c->profiling) cudaEventRecord(c->ev[j], c->stream);
}

// ---------------------------------------------------------------- NEXT-4: sparse P^i
SparseP sparse_args(spdp_ctx* c) {
    SparseP P{};
    P.sptr = c->d_sptr; P.pv = c->d_spv; P.pp = c->d_spp; P.best = c->d_best; P.q = c->d_q; P.dq = c->d_dq;
    return P;
}

// device copy of P in segment order (seg = w * I + i), q / dq / source buffers
spdp_status sparse_upload(spdp_ctx* c) {
    const int I = c->I, V = c->V, Kp = c->Kp;
    const uint32_t segs = (uint32_t)V * I;
    c->h_sptr.assign((size_t)segs + 1, 0);
    for (int w = 0; w < V; ++w)
        for (int i = 0; i < I; ++i) {
            const int r = i * V + w;
            c->h_sptr[(size_t)w * I + i + 1] = (uint32_t)(c->h_pptr[(size_t)r + 1] - c->h_pptr[(size_t)r]);
        }
    for (uint32_t sg = 0; sg < segs; ++sg) c->h_sptr[sg + 1] += c->h_sptr[sg];
    c->E_sp = c->h_sptr[segs];
    std::vector<int32_t> pv(c->E_sp), best(segs);
    std::vector<float> pp(c->E_sp);
    c->dev_of_user.assign(c->E_sp, 0);
    for (int w = 0; w < V; ++w)
        for (int i = 0; i < I; ++i) {
            const int r = i * V + w;
            const uint32_t sg = (uint32_t)w * I + i;
            uint32_t d = c->h_sptr[sg];
            int32_t b = c->h_pptr[(size_t)r];
            for (int32_t e = c->h_pptr[(size_t)r]; e < c->h_pptr[(size_t)r + 1]; ++e, ++d) {
                pv[d] = c->h_pv[(size_t)e];
                pp[d] = (float)c->h_pp[(size_t)e];
                c->dev_of_user[(size_t)e] = d;
                if (c->h_pp[(size_t)e] > c->h_pp[(size_t)b]) b = e;
            }
            best[sg] = (int32_t)(c->h_sptr[sg] + (uint32_t)(b - c->h_pptr[(size_t)r]));
        }
    ALLOC(c->d_sptr, (size_t)segs + 1); ALLOC(c->d_spv, c->E_sp); ALLOC(c->d_spp, c->E_sp); ALLOC(c->d_best, segs);
    ALLOC(c->d_spp64, c->E_sp);
    {
        std::vector<double> pp64(c->E_sp);
        for (size_t e = 0; e < c->dev_of_user.size(); ++e) pp64[c->dev_of_user[e]] = c->h_pp[e];
        CU(cudaMemcpyAsync(c->d_spp64, pp64.data(), sizeof(double) * pp64.size(), cudaMemcpyHostToDevice, c->stream));
    }
    ALLOC(c->d_q, (size_t)c->E_sp * Kp); ALLOC(c->d_dq, (size_t)c->E_sp * Kp);
    ALLOC(c->d_src, (size_t)std::max<int64_t>(c->Nloc, 1));
    CU(cudaMemcpyAsync(c->d_sptr, c->h_sptr.data(), sizeof(uint32_t) * c->h_sptr.size(), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->d_spv, pv.data(), sizeof(int32_t) * pv.size(), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->d_spp, pp.data(), sizeof(float) * pp.size(), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->d_best, best.data(), sizeof(int32_t) * best.size(), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemsetAsync(c->d_dq, 0, sizeof(int32_t) * (size_t)c->E_sp * Kp, c->stream));
    CU(cudaMemsetAsync(c->d_src, 0xFF, sizeof(int16_t) * (size_t)std::max<int64_t>(c->Nloc, 1), c->stream));
    if (c->G > 1) {            // net changes of m (cells) then of q (E x Kp), int32, summed over ranks
        c->pack32 = true;
        int32_t *dl = nullptr, *ds = nullptr;
        ALLOC(dl, c->xcount()); ALLOC(ds, c->xcount());
        c->d_Dloc = dl; c->d_Dsum = ds;
        CU(cudaMemsetAsync(c->d_Dloc, 0, c->dbytes(), c->stream));
    }
    return SPDP_OK;
}

// after the identity-P state installation: sources of the tables (reading c25), Q[v][k] from q
void sparse_install(spdp_ctx* c) {
    const int Kp = c->Kp;
    SparseP P = sparse_args(c);
    cudaMemsetAsync(c->d_q, 0, sizeof(int32_t) * (size_t)c->E_sp * Kp, c->stream);
    const uint32_t segs = (uint32_t)c->V * c->I;
    sp_init_q_kernel<<<148 * 8, 256, 0, c->stream>>>(P, c->d_t, segs, Kp);
    cudaMemsetAsync(c->d_Q, 0, sizeof(int32_t) * (size_t)c->V * Kp, c->stream);
    sp_shadow_kernel<<<148 * 8, 256, 0, c->stream>>>(P, c->E_sp, c->K, Kp, c->d_Q);
}

// after the all-reduce: m, q = local - Dloc + Dsum, correction (reading c24), t; then the sums and Q from scratch
void sparse_exchange_merge(spdp_ctx* c) {
    SparseP P = sparse_args(c);
    const uint32_t segs = (uint32_t)c->V * c->I;
    sp_exchange_merge_kernel<<<148 * 4, 256, 0, c->stream>>>(P, segs, c->d_m, c->d_t, (int32_t*)c->d_Dloc,
                                                            (const int32_t*)c->d_Dsum, c->cells, c->K, c->Kp, c->d_stats);
    launch_merge(c, nullptr, nullptr);                       // M, Tt, T from the rows (Q there assumes identity P)
    cudaMemsetAsync(c->d_Q, 0, sizeof(int32_t) * (size_t)c->V * c->Kp, c->stream);
    sp_shadow_kernel<<<148 * 8, 256, 0, c->stream>>>(P, c->E_sp, c->K, c->Kp, c->d_Q);
    c->launches += 3;
}

// one wave of the sparse sweep: factors of the wave's segments, tokens, n, merge
void sparse_wave(spdp_ctx* c, int w) {
    const uint32_t r0 = c->wave_seg_begin[(size_t)w], r1 = c->wave_seg_begin[(size_t)w + 1];
    const uint32_t tb = c->wave_tok_begin[(size_t)w], te = c->wave_tok_begin[(size_t)w + 1];
    if (te <= tb) return;
    SparseP P = sparse_args(c);
    const int Kp = c->Kp;
    const float beta = (float)c->cfg.beta, vbeta = (float)((double)c->V * c->cfg.beta);
    const size_t nf = (size_t)(r1 - r0) * Kp;
    sp_factor_kernel<<<(int)std::max<size_t>(1, std::min<size_t>((nf + 255) / 256, (size_t)148 * 16)), 256, 0, c->stream>>>(
        P, c->d_wave_segs, r0, r1, c->d_m, c->d_t, c->d_Q, c->d_M, c->d_Tt, c->d_T, c->d_disc, c->d_conc, c->d_tab,
        c->d_tab_off, beta, vbeta, c->I, c->K, Kp, c->d_F, c->d_R1);
    SpTokenArgs t{};
    t.tok_doc = c->d_tok_doc; t.tok_id = c->d_tok_id; t.tok_run = c->d_tok_run; t.run_seg = c->d_wave_segs;
    t.zr = c->d_zr; t.zr_next = c->d_zr_next; t.src = c->d_src; t.F = c->d_F; t.R1 = c->d_R1; t.n = c->d_n;
    t.sigma = c->d_sigma;
    for (int B = 0; B < 256; ++B) t.bpos[B] = (B < Kp / 4) ? c->sigma[(size_t)4 * B] / 4 : 0;
    t.m = c->d_m; t.t = c->d_t; t.Q = c->d_Q; t.M = c->d_M; t.Tt = c->d_Tt; t.T = c->d_T; t.dm = c->d_dm;
    t.alpha = c->d_alpha; t.disc = c->d_disc; t.conc = c->d_conc; t.tab = c->d_tab; t.tab_off = c->d_tab_off;
    t.beta = beta; t.vbeta = vbeta; t.I = c->I; t.K = c->K; t.Kp = Kp; t.Kn = c->Kn;
    t.key0 = (uint32_t)c->cfg.seed; t.key1 = (uint32_t)(c->cfg.seed >> 32);
    t.sweep = c->d_sweep; t.begin = tb; t.end = te; t.stats = c->d_stats; t.P = P;
    const int grid = (int)std::min<uint32_t>((te - tb + 255) / 256, 148u * 8u);
    const size_t ssm = ((Kp / 4) <= kSpSmemBlocks) ? sizeof(float) * 256 * (size_t)(Kp / 4) : 0;
    SPDP_ROWS(c->row_elem, sp_token_kernel<NT><<<std::max(grid, 1), 256, ssm, c->stream>>>(t));
    if (c->W == 1) {
        SPDP_ROWS(c->row_elem, launch_recount<NT>(c, c->stream, nullptr));
        std::swap(c->d_zr, c->d_zr_next);
    } else {
        const int tblocks = (int)std::min<uint32_t>((te - tb + 255) / 256, 148u * 16u);
        SPDP_ROWS(c->row_elem, apply_tokens_kernel<NT><<<std::max(tblocks, 1), 256, 0, c->stream>>>(
                                   c->d_tok_doc, c->d_zr, c->d_zr_next, (NT*)c->d_n, c->d_sigma, c->Kn, tb, te));
    }
    const int blocks = (int)std::min<uint32_t>((r1 - r0 + 7) / 8, 148u * 4u);
    int32_t* Dm = c->G > 1 ? (int32_t*)c->d_Dloc : nullptr;
    int32_t* Dq = c->G > 1 ? (int32_t*)c->d_Dloc + c->cells : nullptr;
    sp_merge_kernel<<<std::max(blocks, 1), 256, 0, c->stream>>>(P, c->d_wave_segs + r0, (int)(r1 - r0), c->d_m, c->d_t,
                                                                c->d_dm, c->d_Q, c->d_M, c->d_Tt, c->d_T, c->I, c->K, Kp,
                                                                c->d_stats, Dm, Dq);
    c->launches += 4;
}

// W = 1 in P word-range parts (DESIGN.md §5 "exchange pipelining").  Semantics are those of the
// single wave: every token decides against the sweep-start snapshot.  Rows of part p are only read
// by part p's tokens, so they may be merged (and, with several ranks, all-reduced and merged again)
// while later parts sample; the sums M, Tt, T are read by every token and are updated only after
// the last part (deferred into d_Mn...; with the pipelined exchange rebuilt into d_Mf...).
spdp_status run_parts(spdp_ctx* c, SweepArgs a) {
    const size_t isz = sizeof(int32_t) * (size_t)c->I * c->Kp, ksz = sizeof(int32_t) * (size_t)c->Kp;
    cudaStream_t st = c->stream;
    CU(cudaMemcpyAsync(c->d_Mn, c->d_M, isz, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(c->d_Ttn, c->d_Tt, isz, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(c->d_Tn, c->d_T, ksz, cudaMemcpyDeviceToDevice, st));
    if (c->overlap) {
        // comm_stream starts after the main stream's previous read of d_Mf... (and everything before)
        CU(cudaEventRecord(c->part_ev[0], st));
        CU(cudaStreamWaitEvent(c->comm_stream, c->part_ev[0], 0));
        CU(cudaMemsetAsync(c->d_Mf, 0, isz, c->comm_stream));
        CU(cudaMemsetAsync(c->d_Ttf, 0, isz, c->comm_stream));
        CU(cudaMemsetAsync(c->d_Tf, 0, ksz, c->comm_stream));
    }
    void* Dnet = c->G > 1 ? c->d_Dloc : nullptr;
    const size_t smem = sizeof(int) * (size_t)(2 * c->I + 1) * c->Kp;
    const int use_smem = smem <= 48 * 1024;
    const size_t row_cells = (size_t)c->I * c->Kp;          // cells per word
    const size_t esz = c->pack32 ? 4 : 8;
    rec(c, 0);
    for (int p = 0; p < c->P; ++p) {
        const uint32_t cb = c->part_chunk[(size_t)p], ce = c->part_chunk[(size_t)p + 1];
        const uint32_t rb = c->part_run[(size_t)p], re = c->part_run[(size_t)p + 1];
        const uint32_t tb = c->part_tok[(size_t)p], te = c->part_tok[(size_t)p + 1];
        if (te > tb) {
            if (c->token_kernel) {
                launch_token(c, rb, re, tb, te);
            } else {
                a.chunk_start = c->d_chunk_start + cb;
                a.chunk_end = c->d_chunk_end + cb;
                a.chunk_seg = c->d_chunk_seg + cb;
                a.nchunks = (int)(ce - cb);
                a.work = c->d_work + p;
                if (c->chunk_ft) launch_chunk_factors(c, rb, re);
                if (c->sprows) launch_sprows(c, a);
                else launch_sample(c, a, false);
            }
            const int blocks = (int)std::min<uint32_t>((re - rb + 7) / 8, 148u * 4u);
            merge_segments_kernel<<<std::max(blocks, 1), 256, use_smem ? smem : 0, st>>>(
                c->d_wave_segs + rb, (int)(re - rb), c->d_m, c->d_t, c->d_dm, c->d_dt, Dnet, (int)c->pack32, c->d_Q,
                c->d_Mn, c->d_Ttn, c->d_Tn, c->I, c->Kp, use_smem, c->d_stats, (int)(c->token_kernel || c->pack_dmt), 0);
            c->launches += 2;
        }
        if (c->overlap) {                                   // rows of part p: all-reduce + merge on comm_stream
            const int w0 = (int)c->part_word[(size_t)p], w1 = (int)c->part_word[(size_t)p + 1];
            CU(cudaEventRecord(c->part_ev[(size_t)p], st));
            CU(cudaStreamWaitEvent(c->comm_stream, c->part_ev[(size_t)p], 0));
            if (w1 > w0) {
                const size_t off = (size_t)w0 * row_cells, cnt = (size_t)(w1 - w0) * row_cells;
                char* dl = (char*)c->d_Dloc + off * esz;
                char* ds = (char*)c->d_Dsum + off * esz;
                spdp_status s = nccl_check(c, c->nccl.AllReduce(dl, ds, cnt, c->pack32 ? kNcclInt32 : kNcclInt64, kNcclSum,
                                                                c->comm, c->comm_stream), "ncclAllReduce(part)");
                if (s) return s;
                launch_exchange_merge_range(c, w0, w1, c->d_Mf, c->d_Ttf, c->d_Tf, c->comm_stream);
                c->launches += 1;
            }
        }
    }
    rec(c, 1);
    // every token moved to zr_next: rebuild n, swap
    SPDP_ROWS(c->row_elem, launch_recount<NT>(c, st, c->doc_scatter ? c->d_zr_doc : nullptr));
    rebuild_entries(c, st);
    std::swap(c->d_zr, c->d_zr_next);
    rec(c, 2);
    if (c->overlap) {
        CU(cudaEventRecord(c->comm_done, c->comm_stream));
        CU(cudaStreamWaitEvent(st, c->comm_done, 0));
        CU(cudaMemcpyAsync(c->d_M, c->d_Mf, isz, cudaMemcpyDeviceToDevice, st));
        CU(cudaMemcpyAsync(c->d_Tt, c->d_Ttf, isz, cudaMemcpyDeviceToDevice, st));
        CU(cudaMemcpyAsync(c->d_T, c->d_Tf, ksz, cudaMemcpyDeviceToDevice, st));
    } else {
        CU(cudaMemcpyAsync(c->d_M, c->d_Mn, isz, cudaMemcpyDeviceToDevice, st));
        CU(cudaMemcpyAsync(c->d_Tt, c->d_Ttn, isz, cudaMemcpyDeviceToDevice, st));
        CU(cudaMemcpyAsync(c->d_T, c->d_Tn, ksz, cudaMemcpyDeviceToDevice, st));
    }
    rec(c, 3);
    c->launches += 1;
    c->acc[5] += 1;
    return check_launch(c, "sweep parts");
}

// waves [w0, w1) of the sweep (one exchange block); first: the sweep's first block
spdp_status run_waves(spdp_ctx* c, int w0, int w1, bool first) {
    SweepArgs a = base_args(c);
    if (first) CU(cudaMemsetAsync(c->d_stats, 0, sizeof(unsigned long long) * 4, c->stream));
    CU(cudaMemsetAsync(c->d_work, 0, sizeof(uint32_t) * ((size_t)std::max(c->W, c->P) + 2), c->stream));
    if (c->profiling) { spdp_status s = ensure_events(c); if (s) return s; }
    void* Dnet = c->G > 1 ? c->d_Dloc : nullptr;
    if (c->async) {
        // NEXT-2: one launch with immediate updates, then the end-of-sweep correction
        // (t into its valid range, Q and the sums recomputed: Alg.4)
        if (c->G > 1) {                                  // sweep-start copy for the net change
            CU(cudaMemcpyAsync(c->d_dm, c->d_m, sizeof(int32_t) * c->cells, cudaMemcpyDeviceToDevice, c->stream));
            CU(cudaMemcpyAsync(c->d_dt, c->d_t, sizeof(int32_t) * c->cells, cudaMemcpyDeviceToDevice, c->stream));
        }
        rec(c, 0);
        a.nchunks = (int)c->nchunks;
        a.work = c->d_work;
        launch_sample(c, a, false);
        rec(c, 1);
        std::swap(c->d_zr, c->d_zr_next);
        rec(c, 2);
        launch_merge(c, nullptr, nullptr);
        if (c->G > 1) {
            const int grid = 148 * 8;
            if (c->pack32)
                net_change_kernel<int32_t><<<grid, 256, 0, c->stream>>>(c->d_m, c->d_t, c->d_dm, c->d_dt,
                                                                        (int32_t*)c->d_Dloc, c->cells);
            else
                net_change_kernel<long long><<<grid, 256, 0, c->stream>>>(c->d_m, c->d_t, c->d_dm, c->d_dt,
                                                                          (long long*)c->d_Dloc, c->cells);
            c->launches += 1;
        }
        rec(c, 3);
        c->launches += 2;
        c->acc[5] += 1;
        return check_launch(c, "async sweep");
    }
    if (c->P > 1) return run_parts(c, a);
    if (c->sparse) {
        for (int w = w0; w < w1; ++w) {
            rec(c, 4 * (size_t)w);
            sparse_wave(c, w);
            rec(c, 4 * (size_t)w + 1); rec(c, 4 * (size_t)w + 2); rec(c, 4 * (size_t)w + 3);
            c->acc[5] += 1;
        }
        return check_launch(c, "sparse sweep");
    }
    for (int w = w0; w < w1; ++w) {
        const uint32_t cb = c->wave_chunk_begin[(size_t)w], ce = c->wave_chunk_begin[(size_t)w + 1];
        rec(c, 4 * (size_t)w);
        if (ce == cb) { rec(c, 4 * (size_t)w + 1); rec(c, 4 * (size_t)w + 2); rec(c, 4 * (size_t)w + 3); continue; }
        const uint32_t tb = c->wave_tok_begin[(size_t)w], te = c->wave_tok_begin[(size_t)w + 1];
        if (c->token_kernel) {
            launch_token(c, c->wave_seg_begin[(size_t)w], c->wave_seg_begin[(size_t)w + 1], tb, te);
        } else {
            a.chunk_start = c->d_chunk_start + cb;
            a.chunk_end = c->d_chunk_end + cb;
            a.chunk_seg = c->d_chunk_seg + cb;
            a.nchunks = (int)(ce - cb);
            a.work = c->d_work + w;
            if (c->chunk_ft) launch_chunk_factors(c, c->wave_seg_begin[(size_t)w], c->wave_seg_begin[(size_t)w + 1]);
            if (c->sprows) launch_sprows(c, a);
            else launch_sample(c, a, false);
        }
        rec(c, 4 * (size_t)w + 1);
        // W = 1: the doc-topic recount (n from zr_next) and the segment merge (m, t, Q, sums from the deltas)
        // touch disjoint data, so outside profiling the recount runs on a side stream beside the merge
        // (a fork/join the CUDA graph capture records as parallel branches)
        const bool side = c->W == 1 && !c->profiling && c->side_stream;
        if (side) {
            CU(cudaEventRecord(c->ev_fork, c->stream));
            CU(cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
        }
        if (c->W == 1) {
            // every token moved to zr_next: rebuild the doc-topic rows, then swap
            cudaStream_t rs = side ? c->side_stream : c->stream;
            SPDP_ROWS(c->row_elem, launch_recount<NT>(c, rs, c->doc_scatter ? c->d_zr_doc : nullptr));
            rebuild_entries(c, rs);
            std::swap(c->d_zr, c->d_zr_next);
        } else {
            const int tblocks = (int)std::min<uint32_t>((te - tb + 255) / 256, 148u * 16u);
            SPDP_ROWS(c->row_elem, apply_tokens_kernel<NT><<<std::max(tblocks, 1), 256, 0, c->stream>>>(
                                       c->d_tok_doc, c->d_zr, c->d_zr_next, (NT*)c->d_n, c->d_sigma, c->Kn, tb, te));
            rebuild_entries(c, c->stream);                 // the next wave reads the updated rows
        }
        rec(c, 4 * (size_t)w + 2);
        {
            const uint32_t sb = c->wave_seg_begin[(size_t)w], se = c->wave_seg_begin[(size_t)w + 1];
            const size_t smem = sizeof(int) * (size_t)(2 * c->I + 1) * c->Kp;
            const int use_smem = smem <= 48 * 1024;
            const int blocks = (int)std::min<uint32_t>((se - sb + 7) / 8, 148u * 4u);
            merge_segments_kernel<<<std::max(blocks, 1), 256, use_smem ? smem : 0, c->stream>>>(
                c->d_wave_segs + sb, (int)(se - sb), c->d_m, c->d_t, c->d_dm, c->d_dt, Dnet, (int)c->pack32, c->d_Q, c->d_M,
                c->d_Tt, c->d_T, c->I, c->Kp, use_smem, c->d_stats, (int)(c->token_kernel || c->pack_dmt),
                (int)c->fold_merge);
        }
        if (side) {
            CU(cudaEventRecord(c->ev_join, c->side_stream));
            CU(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
        }
        rec(c, 4 * (size_t)w + 3);
        c->launches += 3;
        c->acc[5] += 1;
    }
    return check_launch(c, "sweep waves");
}

// waves of exchange block b (the last block also covers the empty waves past the longest document)
inline int block_w0(const spdp_ctx* c, int b) { return b * c->E; }
inline int block_w1(const spdp_ctx* c, int b) { return b + 1 >= c->nblocks ? c->W : std::min((b + 1) * c->E, c->W); }

// after the stream is synchronised: accumulate this sweep's phase times
void collect_times(spdp_ctx* c, bool exchanged) {
    if (!c->profiling) return;
    float ms;
    for (int w = 0; w < c->W; ++w) {
        const size_t b = 4 * (size_t)w;
        if (cudaEventElapsedTime(&ms, c->ev[b], c->ev[b + 1]) == cudaSuccess) c->acc[0] += ms;
        if (cudaEventElapsedTime(&ms, c->ev[b + 1], c->ev[b + 2]) == cudaSuccess) c->acc[1] += ms;
        if (cudaEventElapsedTime(&ms, c->ev[b + 2], c->ev[b + 3]) == cudaSuccess) c->acc[2] += ms;
    }
    const size_t x = 4 * (size_t)c->W;
    if (exchanged && cudaEventElapsedTime(&ms, c->ev[x], c->ev[x + 1]) == cudaSuccess) c->acc[3] += ms;
    const size_t last = exchanged ? x + 1 : 4 * (size_t)(c->W - 1) + 3;
    if (cudaEventElapsedTime(&ms, c->ev[0], c->ev[last]) == cudaSuccess) c->acc[4] += ms;
    c->acc[7] += 1;
}

// W = 0: num_sweeps exact sequential sweeps in one single-warp launch (spdp_seq.cuh); codes: the
// state code after each sweep (spdp_debug_chain), or null
spdp_status seq_sweeps(spdp_ctx* c, int32_t num_sweeps, int64_t* d_codes, int tbase) {
    if (num_sweeps <= 0) return SPDP_OK;
    CU(cudaMemsetAsync(c->d_stats, 0, sizeof(unsigned long long) * 4, c->stream));
    SweepArgs a = base_args(c);
    SeqArgs q{};
    q.group = c->d_group; q.word = c->d_word; q.pos = c->d_pos; q.N = c->N; q.V = c->V;
    q.nsweeps = num_sweeps; q.codes = d_codes; q.tbase = tbase;
    const size_t smem = sizeof(float2) * (size_t)c->Kp;
    SPDP_ROWS(c->row_elem, seq_kernel<NT><<<1, 32, smem, c->stream>>>(a, q));
    spdp_status s = check_launch(c, "seq_kernel");
    if (s) return s;
    c->launches += 1;
    c->sweeps_done += num_sweeps;
    return sync(c, "seq sweeps");
}

spdp_status finish_sweep(spdp_ctx* c) {
    inc_sweep_kernel<<<1, 1, 0, c->stream>>>(c->d_sweep);
    c->launches += 1;
    c->sweeps_done++;
    return check_launch(c, "inc_sweep");
}

spdp_status debug_verify(spdp_ctx* c);

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* spdp_version(void) { return "spdp-b200 0.1 (sm_100a)"; }

const char* spdp_last_error(const spdp_ctx* c) { return c ? c->err.c_str() : "null context"; }

spdp_status spdp_partition(uint64_t seed, int32_t world_size, int64_t num_tokens, int32_t num_docs, const int32_t* doc,
                           int32_t* shard_of_doc) {
    if (world_size < 1 || num_tokens < 0 || num_docs < 1 || (!doc && num_tokens) || !shard_of_doc) return SPDP_EINVAL;
    std::vector<int32_t> len((size_t)num_docs, 0);
    for (int64_t p = 0; p < num_tokens; ++p) {
        if (doc[p] < 0 || doc[p] >= num_docs) return SPDP_EINVAL;
        len[(size_t)doc[p]]++;
    }
    std::vector<int32_t> sh;
    partition_docs(seed, world_size, num_tokens, num_docs, len, sh);
    std::memcpy(shard_of_doc, sh.data(), sizeof(int32_t) * (size_t)num_docs);
    return SPDP_OK;
}

spdp_status spdp_create(const spdp_config* cfg, spdp_ctx** out) {
    if (!out) return SPDP_EINVAL;
    *out = nullptr;
    if (!cfg || cfg->struct_size != sizeof(spdp_config)) return SPDP_EINVAL;
    spdp_ctx* c = new (std::nothrow) spdp_ctx();
    if (!c) return SPDP_ENOMEM;
    c->cfg = *cfg;
    auto bad = [&](const char* msg) { fail(c, SPDP_EINVAL, "%s", msg); *out = c; return SPDP_EINVAL; };
    if (cfg->num_groups < 1 || cfg->vocab_size < 1) return bad("num_groups and vocab_size must be >= 1");
    if (cfg->num_topics < 1 || cfg->num_topics > 1024) return bad("num_topics must be in [1, 1024]");
    if (!(cfg->beta > 0.0)) return bad("beta must be > 0");
    if (!cfg->discount || !cfg->concentration) return bad("discount and concentration arrays are required");
    if (cfg->num_waves < 0) return bad("num_waves must be >= 0");
    if (cfg->num_waves == 0) {   // W = 0: the exact sequential sampler (test mode; one rank, wave updates)
        if (cfg->world_size != 1) return bad("num_waves = 0 (sequential test mode) needs world_size == 1");
        if (cfg->update_mode != SPDP_UPDATE_WAVE) return bad("num_waves = 0 needs SPDP_UPDATE_WAVE");
    }
    if (cfg->merge_every < 0) return bad("merge_every must be >= 0");
    if (cfg->update_mode != SPDP_UPDATE_WAVE && cfg->update_mode != SPDP_UPDATE_ASYNC) return bad("unknown update_mode");
    if (cfg->update_mode == SPDP_UPDATE_ASYNC && cfg->num_waves != 1) return bad("SPDP_UPDATE_ASYNC needs num_waves == 1");
    c->async = cfg->update_mode == SPDP_UPDATE_ASYNC;
    if (cfg->world_size < 1 || cfg->rank < 0 || cfg->rank >= cfg->world_size) return bad("rank / world_size out of range");
    c->I = cfg->num_groups; c->V = cfg->vocab_size; c->K = cfg->num_topics;
    c->Kp = (c->K + 3) & ~3; c->W = std::max(cfg->num_waves, 1); c->rank = cfg->rank; c->G = cfg->world_size;
    c->seq = cfg->num_waves == 0;                      // the plan is the W = 1 plan; the sweep is seq_kernel
    c->alpha_ik.resize((size_t)c->I * c->K);
    for (size_t j = 0; j < c->alpha_ik.size(); ++j) {
        c->alpha_ik[j] = cfg->alpha_ik ? cfg->alpha_ik[j] : cfg->alpha;
        if (!(c->alpha_ik[j] > 0.0)) return bad("alpha must be > 0");
    }
    c->disc.assign(cfg->discount, cfg->discount + c->I);
    c->conc.assign(cfg->concentration, cfg->concentration + c->I);
    for (int i = 0; i < c->I; ++i) {
        if (!(c->disc[(size_t)i] >= 0.0 && c->disc[(size_t)i] < 1.0)) return bad("discount must be in [0, 1)");
        if (!(c->conc[(size_t)i] > 0.0)) return bad("concentration must be > 0");
    }
    c->cfg.alpha_ik = nullptr; c->cfg.discount = nullptr; c->cfg.concentration = nullptr; c->cfg.nccl_unique_id = nullptr;
    c->LPT = pick_lpt(c->K);
    c->KPL = pick_kpl(c->K);
    if (const char* e = getenv("SPDP_KERNEL_CFG")) {       // tuning override "LPTxKPL", e.g. "8x16"
        int l = 0, p = 0;
        if (sscanf(e, "%dx%d", &l, &p) == 2 && l * p >= c->K) {
            if (!cfg_compiled(l, p)) return bad("SPDP_KERNEL_CFG: configuration not compiled (build with -DSPDP_TUNING_CFGS)");
            c->LPT = l; c->KPL = p;
        }
    }
    if (c->LPT * c->KPL < c->K) return bad("internal: no kernel configuration for K");
    // doc-topic row layout (sigma order, see spdp_device.cuh): LA lanes of a group hold topics, rows of
    // Kn = LA * KPL elements (the unit positions are set at load, once the row element type is known)
    c->LA = (c->K + c->KPL - 1) / c->KPL;
    c->Kn = c->LA * c->KPL;
    // tokens per chunk: 512 vs 256 measured -0.5..-1.2 % at C3, C4 K = 100/300, C5 (B200); the async
    // mode keeps 256 (its tokens share the chunk-start copy of the segment's counts, reading c23)
    int chunk = c->async ? 256 : 512;
    if (const char* e = getenv("SPDP_CHUNK_TOKENS")) chunk = std::min(std::max(1, atoi(e)), 16384);
    c->chunk_tokens = chunk;

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        fail(c, SPDP_ECUDA, "no CUDA device: %s", e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
        *out = c;
        return SPDP_ECUDA;
    }
    if (cfg->device < 0 || cfg->device >= ndev) return bad("device ordinal out of range");
    if ((e = cudaSetDevice(cfg->device)) != cudaSuccess) {
        fail(c, SPDP_ECUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
        *out = c;
        return SPDP_ECUDA;
    }
    if (cfg->stream) c->stream = (cudaStream_t)cfg->stream;
    else {
        if ((e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) != cudaSuccess) {
            fail(c, SPDP_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
            *out = c;
            return SPDP_ECUDA;
        }
        c->own_stream = true;
    }
    set_attrs(c);
    if (!(getenv("SPDP_TEMP_POOL") && atoi(getenv("SPDP_TEMP_POOL")) == 0)) {
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = cfg->device;
        if (cudaMemPoolCreate(&c->pool, &pp) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr);
        } else {
            c->pool = nullptr;
            cudaGetLastError();
        }
    }
    if (!(getenv("SPDP_SIDE_STREAM") && atoi(getenv("SPDP_SIDE_STREAM")) == 0) &&
        (cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)) {
        fail(c, SPDP_ECUDA, "side stream / events");
        *out = c;
        return SPDP_ECUDA;
    }
    if (c->G > 1 && cfg->exchange == SPDP_EXCHANGE_NCCL) {
        if (!cfg->nccl_unique_id) return bad("nccl_unique_id is required for SPDP_EXCHANGE_NCCL with world_size > 1");
        c->nccl.lib = open_nccl();
        if (!c->nccl.lib) {
            fail(c, SPDP_ENCCL, "cannot dlopen libnccl.so.2");
            *out = c;
            return SPDP_ENCCL;
        }
        c->nccl.CommInitRank = (decltype(c->nccl.CommInitRank))dlsym(c->nccl.lib, "ncclCommInitRank");
        c->nccl.AllReduce = (decltype(c->nccl.AllReduce))dlsym(c->nccl.lib, "ncclAllReduce");
        c->nccl.CommDestroy = (decltype(c->nccl.CommDestroy))dlsym(c->nccl.lib, "ncclCommDestroy");
        c->nccl.GetErrorString = (decltype(c->nccl.GetErrorString))dlsym(c->nccl.lib, "ncclGetErrorString");
        if (!c->nccl.CommInitRank || !c->nccl.AllReduce || !c->nccl.CommDestroy) {
            fail(c, SPDP_ENCCL, "libnccl lacks the required symbols");
            *out = c;
            return SPDP_ENCCL;
        }
        NcclUid uid;
        std::memcpy(uid.b, cfg->nccl_unique_id, 128);
        int r = c->nccl.CommInitRank(&c->comm, c->G, uid, c->rank);
        if (r != 0) {
            fail(c, SPDP_ENCCL, "ncclCommInitRank: %s", c->nccl.GetErrorString ? c->nccl.GetErrorString(r) : "error");
            *out = c;
            return SPDP_ENCCL;
        }
    }
    *out = c;
    return SPDP_OK;
}

spdp_status spdp_load_corpus(spdp_ctx* c, int64_t num_tokens, int32_t num_docs, const int32_t* group, const int32_t* doc,
                             const int32_t* word, const int32_t* z_init, const uint8_t* r_init) {
    LoadTimer lt;
    spdp_status s = guard(c, false);
    if (s) return s;
    if (c->loaded) return fail(c, SPDP_ESTATE, "spdp_load_corpus may be called once per context");
    if (c->sparse && c->async)
        return fail(c, SPDP_EINVAL, "a transformation matrix needs SPDP_UPDATE_WAVE in this version");
    if (num_tokens < 1 || num_docs < 1 || !group || !doc || !word)
        return fail(c, SPDP_EINVAL, "need num_tokens >= 1, num_docs >= 1 and the three token arrays");
    if (num_tokens >= (int64_t)0xFFFFFFFF) return fail(c, SPDP_EINVAL, "num_tokens must be < 2^32 - 1");
    const int I = c->I, V = c->V, Kp = c->Kp, W = c->W;
    TempStream temp_scope(c->stream, c->pool);
    struct PooledScope {
        spdp_ctx* c;
        explicit PooledScope(spdp_ctx* x) : c(x) { c->pooled_alloc = true; }
        ~PooledScope() { c->pooled_alloc = false; }
    } pooled_scope(c);
    c->N = num_tokens; c->D = num_docs;
    // the token triples stay on the device (state installation); host copies only on demand (diagnostics)
    c->group.clear(); c->doc.clear(); c->word.clear();
    const uint32_t n = (uint32_t)num_tokens;
    const int grid = 148 * 8;
    cudaStream_t st = c->stream;
    auto bits = [](uint64_t x) { int b = 1; while (b < 64 && (x >> b)) ++b; return b; };
    ALLOC(c->d_group, n); ALLOC(c->d_doc, n); ALLOC(c->d_word, n);
    struct { int32_t* p; } dgrp{c->d_group}, ddoc{c->d_doc}, dwrd{c->d_word};
    const size_t npos = W > 1 ? (size_t)n : 1;      // in-document positions: only with several waves
    TempBuf<int32_t> dpos(npos), ddg((size_t)num_docs), ddl((size_t)num_docs);
    TempBuf<uint32_t> diota(n), dbydoc(npos), dstart(W > 1 ? (size_t)num_docs : 1);
    TempBuf<int32_t> dkeyd(npos);
    TempBuf<unsigned long long> derr(2);
    if (!dpos.p || !ddg.p || !ddl.p || !diota.p || !dbydoc.p || !dstart.p ||
        !dkeyd.p || !derr.p)
        return fail(c, SPDP_ENOMEM, "load planning buffers");
    CU(cudaMemcpyAsync(dgrp.p, group, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(ddoc.p, doc, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dwrd.p, word, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(ddg.p, 0xFF, sizeof(int32_t) * (size_t)num_docs, st));
    CU(cudaMemsetAsync(ddl.p, 0, sizeof(int32_t) * (size_t)num_docs, st));
    CU(cudaMemsetAsync(derr.p, 0xFF, sizeof(unsigned long long) * 2, st));
    validate_tokens_kernel<<<grid, 256, 0, st>>>(dgrp.p, ddoc.p, dwrd.p, n, I, V, num_docs, ddg.p, ddl.p, derr.p);
    unsigned long long herr[2];
    CU(cudaMemcpyAsync(herr, derr.p, sizeof(herr), cudaMemcpyDeviceToHost, st));
    c->doclen.resize((size_t)num_docs);
    c->docgroup.resize((size_t)num_docs);
    CU(cudaMemcpyAsync(c->doclen.data(), ddl.p, sizeof(int32_t) * (size_t)num_docs, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(c->docgroup.data(), ddg.p, sizeof(int32_t) * (size_t)num_docs, cudaMemcpyDeviceToHost, st));
    if ((s = sync(c, "validate tokens"))) return s;
    lt.mark("upload + validate");
    if (herr[0] != ~0ull) {
        const size_t q = (size_t)herr[0];
        return fail(c, SPDP_EINVAL, "token %lld = (%d, %d, %d) out of range", (long long)q, group[q], doc[q], word[q]);
    }
    if (herr[1] != ~0ull) {
        const size_t q = (size_t)herr[1];
        return fail(c, SPDP_EINVAL, "document %d spans several groups (token %lld is in group %d)", doc[q], (long long)q,
                    group[q]);
    }
    // in-document positions: stable sort of the tokens by document (ties keep canonical order)
    auto cub_run = [&](auto f, const char* what) -> spdp_status {
        size_t bytes = 0;
        cudaError_t e = f((void*)nullptr, bytes);
        if (e == cudaSuccess) {
            TempBuf<uint8_t> tmp(bytes);
            if (!tmp.p) return fail(c, SPDP_ENOMEM, "%s: temporary storage", what);
            e = f((void*)tmp.p, bytes);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        }
        if (e != cudaSuccess) return fail(c, SPDP_ECUDA, "%s: %s", what, cudaGetErrorString(e));
        return SPDP_OK;
    };
    iota_kernel<<<grid, 256, 0, st>>>(diota.p, n);
    if (W > 1) {   // in-document positions decide the waves (pos mod W); W = 1 needs none
        if ((s = cub_run([&](void* t, size_t& b) {
                 return cub::DeviceRadixSort::SortPairs(t, b, ddoc.p, dkeyd.p, diota.p, dbydoc.p, (int)n, 0,
                                                        bits((uint64_t)num_docs), st);
             }, "sort by document")))
            return s;
        if ((s = cub_run([&](void* t, size_t& b) {
                 return cub::DeviceScan::ExclusiveSum(t, b, reinterpret_cast<const uint32_t*>(ddl.p), dstart.p, num_docs, st);
             }, "document offsets")))
            return s;
        positions_kernel<<<grid, 256, 0, st>>>(dbydoc.p, ddoc.p, dstart.p, n, dpos.p);
    }
    lt.mark("positions");
    // M_max = largest count(i, w): bounds every m_{ikw} the chain can reach
    {
        TempBuf<int32_t> dcnt((size_t)I * V), dmx(1);
        if (!dcnt.p || !dmx.p) return fail(c, SPDP_ENOMEM, "count(i,w) buffer");
        CU(cudaMemsetAsync(dcnt.p, 0, sizeof(int32_t) * (size_t)I * V, st));
        cell_count_kernel<<<grid, 256, 0, st>>>(dgrp.p, dwrd.p, n, V, dcnt.p);
        if ((s = cub_run([&](void* t, size_t& b) { return cub::DeviceReduce::Max(t, b, dcnt.p, dmx.p, I * V, st); },
                         "M_max")))
            return s;
        CU(cudaMemcpyAsync(&c->mmax, dmx.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st)); CU(cudaStreamSynchronize(st));
        if (c->mmax >= 65536)
            return fail(c, SPDP_ETABLE, "M_max = %d: cells are packed in 16 bits (M_max < 65536)", c->mmax);
        if ((double)c->mmax * (c->mmax + 1) / 2 * sizeof(float2) > 16e9)
            return fail(c, SPDP_ETABLE, "Stirling-ratio table for M_max = %d exceeds 16 GB", c->mmax);
        // word-range parts of the sweep (W = 1 only): balanced by the corpus' token counts, so that
        // every rank cuts at the same words (the all-reduce slices must match)
        // (each part costs a launch tail: pipelining pays when a rank samples many tokens, measured
        // +11% (C3) and +40% (C2) sampling time for 4 parts on one GPU)
        c->P = (W == 1 && c->G > 1 && c->cfg.exchange == SPDP_EXCHANGE_NCCL && !c->async &&
                num_tokens / c->G >= (int64_t)8000000) ? 4 : 1;
        if (const char* e = getenv("SPDP_EXCHANGE_PARTS")) c->P = std::min(std::max(atoi(e), 1), 16);
        if (W != 1 || c->async || c->sparse) c->P = 1;
        c->part_word.assign((size_t)c->P + 1, (uint32_t)V);
        c->part_word[0] = 0;
        if (c->P > 1) {
            std::vector<int32_t> cnt((size_t)I * V);
            CU(cudaMemcpyAsync(cnt.data(), dcnt.p, sizeof(int32_t) * cnt.size(), cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            int64_t run = 0;
            int p = 1;
            for (int w = 0; w < V && p < c->P; ++w) {
                for (int i = 0; i < I; ++i) run += cnt[(size_t)i * V + w];
                while (p < c->P && run * c->P >= (int64_t)p * num_tokens) c->part_word[(size_t)p++] = (uint32_t)(w + 1);
            }
        }
    }
    // small K: the token kernel (packed per-wave deltas need |delta| <= count(i,w) < 2^15)
    // (64 < K <= 128: only with several waves whose (w, i) segments hold < 32 tokens on average, where
    // the chunk kernel cannot fill its chunks; B200: C3 W = 2 (42 per segment) 1.61 ms chunk vs 1.72
    // token, C3 W = 3 (28) 2.04 vs 1.91, C4 K = 100 W = 2 (21) 1.20 vs 1.06)
    const double seg_fill = (double)num_tokens / c->G / ((double)V * I * W);
    c->token_kernel = !c->async && !c->sparse && c->mmax < 32768 &&
                      (c->K <= 64 || (c->K <= 128 && W > 1 && seg_fill < 32.0));
    // wave deltas of the chunk kernels as one packed word per cell: |sum of a wave's deltas| <= count(i,w)
    // <= M_max < 2^15 (the token kernel's argument); halves the flush atomics and the merge's delta bytes
    c->pack_dmt = !c->async && c->mmax < 32768 && !(getenv("SPDP_PACK_DELTAS") && atoi(getenv("SPDP_PACK_DELTAS")) == 0);
    // the chunk kernel's per-chunk slot factors from per-wave factor tables (a throughput kernel) instead of the
    // chunk prologue's dependent load chain (counts -> Stirling table); wave updates, no transform, no async
    c->chunk_ft = SPDP_CHUNK_FACTORS && !c->async && !c->sparse && !c->seq;
    if (const char* e = getenv("SPDP_CHUNK_FACTORS")) c->chunk_ft = atoi(e) != 0 && !c->async && !c->sparse && !c->seq;
    if (const char* e = getenv("SPDP_TOKEN_KERNEL")) {   // 0: never; 2: also K <= 128 with one wave
        const int v = atoi(e);
        if (v == 0) c->token_kernel = false;
        if (v == 2) c->token_kernel = !c->async && !c->sparse && c->mmax < 32768 && c->K <= 128;
    }
    // documents -> ranks
    if (c->G > 1) partition_docs(c->cfg.seed, c->G, num_tokens, num_docs, c->doclen, c->shard_of_doc);
    else c->shard_of_doc.assign((size_t)num_docs, 0);
    c->local_of_doc.assign((size_t)num_docs, -1);
    c->global_of_local.clear();
    for (int32_t d = 0; d < num_docs; ++d)
        if (c->shard_of_doc[(size_t)d] == c->rank) {
            c->local_of_doc[(size_t)d] = (int32_t)c->global_of_local.size();
            c->global_of_local.push_back(d);
        }
    c->Dloc = (int32_t)c->global_of_local.size();
    // the kernels address a doc-topic row by a 32-bit element offset (doc * Kn)
    if ((uint64_t)c->Dloc * (uint64_t)c->Kn >= (1ull << 32) - 4096)
        return fail(c, SPDP_EINVAL, "%d local documents x %d topic slots exceed 2^32 doc-topic cells per rank: "
                    "use more ranks", c->Dloc, c->Kn);
    // Stirling-ratio tables, one per distinct discount (M_max rows): a sequential row recursion on one SM,
    // built on the side stream while the wave plan sorts run on the main stream (joined after the uploads)
    cudaStream_t tab_stream = c->side_stream ? c->side_stream : c->stream;
    struct EventGuard {
        cudaEvent_t e = nullptr;
        ~EventGuard() { if (e) cudaEventDestroy(e); }
    } tab_done;
    {
        CU(cudaEventCreateWithFlags(&tab_done.e, cudaEventDisableTiming));
        std::vector<double> distinct;
        std::vector<int> which((size_t)I);
        for (int i = 0; i < I; ++i) {
            size_t j = 0;
            while (j < distinct.size() && distinct[j] != c->disc[(size_t)i]) ++j;
            if (j == distinct.size()) distinct.push_back(c->disc[(size_t)i]);
            which[(size_t)i] = (int)j;
        }
        const uint64_t per = (uint64_t)(c->mmax + 1) * (uint64_t)(c->mmax + 2) / 2;
        c->pooled_alloc = false;                     // used on the side stream at once: not stream-ordered memory
        ALLOC(c->d_tab, per * distinct.size());
        ALLOC(c->d_tab_off, I);
        c->tab_off_host.resize((size_t)I);
        for (int i = 0; i < I; ++i) c->tab_off_host[(size_t)i] = per * (uint64_t)which[(size_t)i];
        CU(cudaMemcpyAsync(c->d_tab_off, c->tab_off_host.data(), sizeof(uint64_t) * I, cudaMemcpyHostToDevice, tab_stream));
        double* scratch = nullptr;
        ALLOC(scratch, 2 * (size_t)(c->mmax + 2) * distinct.size());
        c->pooled_alloc = true;
        for (size_t j = 0; j < distinct.size(); ++j)
            build_ratio_table<<<1, 1024, 0, tab_stream>>>(c->d_tab + per * j, scratch + 2 * (size_t)(c->mmax + 2) * j,
                                                          c->mmax, distinct[j]);
        s = check_launch(c, "build_ratio_table");
        if (s) return s;
    }
    lt.mark("M_max + partition");
    // this rank's tokens, canonical order
    TempBuf<uint32_t> dlocal(n);
    TempBuf<int32_t> dlod(c->G > 1 ? (size_t)num_docs : 1);
    if (!dlocal.p || !dlod.p) return fail(c, SPDP_ENOMEM, "local token buffer");
    uint32_t nloc = n;
    if (c->G > 1) {
        TempBuf<int32_t> dshard((size_t)num_docs);
        TempBuf<uint8_t> dflag(n);
        TempBuf<uint32_t> dnsel(1);
        if (!dshard.p || !dflag.p || !dnsel.p) return fail(c, SPDP_ENOMEM, "shard buffers");
        CU(cudaMemcpyAsync(dshard.p, c->shard_of_doc.data(), sizeof(int32_t) * (size_t)num_docs, cudaMemcpyHostToDevice, st));
        CU(cudaMemcpyAsync(dlod.p, c->local_of_doc.data(), sizeof(int32_t) * (size_t)num_docs, cudaMemcpyHostToDevice, st));
        local_flags_kernel<<<grid, 256, 0, st>>>(ddoc.p, dshard.p, c->rank, n, dflag.p);
        if ((s = cub_run([&](void* t, size_t& b) {
                 return cub::DeviceSelect::Flagged(t, b, diota.p, dflag.p, dlocal.p, dnsel.p, (int)n, st);
             }, "select local tokens")))
            return s;
        CU(cudaMemcpyAsync(&nloc, dnsel.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st)); CU(cudaStreamSynchronize(st));
    } else {
        CU(cudaMemcpyAsync(dlocal.p, diota.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st));
    }
    c->Nloc = nloc;
    // wave plan: stable sort of the local tokens by (wave = l mod W, w * I + i)
    const uint64_t S = (uint64_t)V * I;
    const uint32_t chunk = (uint32_t)c->chunk_tokens;
    const int Pp = c->P;
    uint32_t R = 0, nch = 0;
    TempBuf<uint32_t> dpartseg((size_t)Pp + 1);
    if (!dpartseg.p) return fail(c, SPDP_ENOMEM, "part buffer");
    {
        std::vector<uint32_t> ps((size_t)Pp + 1);
        for (int p = 0; p <= Pp; ++p) ps[(size_t)p] = c->part_word[(size_t)p] * (uint32_t)I;
        CU(cudaMemcpyAsync(dpartseg.p, ps.data(), sizeof(uint32_t) * ps.size(), cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));
    }
    c->part_chunk.assign((size_t)Pp + 1, 0);
    c->part_run.assign((size_t)Pp + 1, 0);
    c->part_tok.assign((size_t)Pp + 1, 0);
    {
        const size_t nl = std::max<uint32_t>(nloc, 1);
        TempBuf<uint64_t> dkey(nl), dkey2(nl), drkey(nl);
        TempBuf<uint32_t> drlen(nl), droff(nl), dnch(nl), dchoff(nl), dR(1), dwb((size_t)std::max(W, Pp) + 1);
        if (!dkey.p || !dkey2.p || !drkey.p || !drlen.p || !droff.p || !dnch.p || !dchoff.p || !dR.p || !dwb.p)
            return fail(c, SPDP_ENOMEM, "wave plan buffers");
        ALLOC(c->d_tok_id, nl);
        plan_keys_kernel<<<grid, 256, 0, st>>>(dlocal.p, nloc, dgrp.p, dwrd.p, dpos.p, I, W, S, dkey.p);
        if ((s = cub_run([&](void* t, size_t& b) {
                 return cub::DeviceRadixSort::SortPairs(t, b, dkey.p, dkey2.p, dlocal.p, c->d_tok_id, (int)nloc, 0,
                                                        bits((uint64_t)W * S), st);
             }, "sort by (wave, word, group)")))
            return s;
        bounds_kernel<<<grid, 256, 0, st>>>(WaveOfKey{dkey2.p, S}, nloc, (uint32_t)W, dwb.p);
        c->wave_tok_begin.resize((size_t)W + 1);
        CU(cudaMemcpyAsync(c->wave_tok_begin.data(), dwb.p, sizeof(uint32_t) * ((size_t)W + 1), cudaMemcpyDeviceToHost, st)); CU(cudaStreamSynchronize(st));
        // segments of each wave = runs of equal keys
        if ((s = cub_run([&](void* t, size_t& b) {
                 return cub::DeviceRunLengthEncode::Encode(t, b, dkey2.p, drkey.p, drlen.p, dR.p, (int)nloc, st);
             }, "segments")))
            return s;
        CU(cudaMemcpyAsync(&R, dR.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st)); CU(cudaStreamSynchronize(st));
        if (nloc == 0) R = 0;
        ALLOC(c->d_wave_segs, std::max<uint32_t>(R, 1));
        c->wave_seg_begin.assign((size_t)W + 1, 0);
        c->wave_chunk_begin.assign((size_t)W + 1, 0);
        if (R > 0) {
            seg_of_key_kernel<<<grid, 256, 0, st>>>(drkey.p, R, S, c->d_wave_segs);
            bounds_kernel<<<grid, 256, 0, st>>>(WaveOfKey{drkey.p, S}, R, (uint32_t)W, dwb.p);
            CU(cudaMemcpyAsync(c->wave_seg_begin.data(), dwb.p, sizeof(uint32_t) * ((size_t)W + 1), cudaMemcpyDeviceToHost, st)); CU(cudaStreamSynchronize(st));
            // chunks of <= chunk_tokens tokens; within a wave longest first (stable)
            if ((s = cub_run([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, drlen.p, droff.p, (int)R, st); },
                             "segment offsets")))
                return s;
            if (c->token_kernel || c->sparse || c->chunk_ft) {
                ALLOC(c->d_tok_run, nl);
                ALLOC(c->d_F, (size_t)R * Kp);
                ALLOC(c->d_R1, (size_t)R * Kp);
                if ((c->token_kernel && SPDP_TOKEN_PRE) || c->chunk_ft) {
                    ALLOC(c->d_aF, (size_t)R * Kp);
                    ALLOC(c->d_MT, (size_t)R * Kp);
                    ALLOC(c->d_FR, (size_t)R * Kp);
                }
                token_run_kernel<<<grid, 256, 0, st>>>(droff.p, drlen.p, R, c->d_tok_run);
            }
            chunk_count_kernel<<<grid, 256, 0, st>>>(drlen.p, R, chunk, dnch.p);
            if ((s = cub_run([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, dnch.p, dchoff.p, (int)R, st); },
                             "chunk offsets")))
                return s;
            uint32_t last[2];
            CU(cudaMemcpyAsync(&last[0], dchoff.p + (R - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st)); CU(cudaStreamSynchronize(st));
            CU(cudaMemcpyAsync(&last[1], dnch.p + (R - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, st)); CU(cudaStreamSynchronize(st));
            nch = last[0] + last[1];
        }
        const size_t nc = std::max<uint32_t>(nch, 1);
        ALLOC(c->d_chunk_start, nc); ALLOC(c->d_chunk_end, nc); ALLOC(c->d_chunk_seg, nc);
        if (nch > 0) {
            TempBuf<uint32_t> cs(nc), ce(nc), cg(nc), ci(nc), ci2(nc);
            TempBuf<uint64_t> ck(nc), ck2(nc);
            if (!cs.p || !ce.p || !cg.p || !ci.p || !ci2.p || !ck.p || !ck2.p) return fail(c, SPDP_ENOMEM, "chunk buffers");
            chunk_emit_kernel<<<grid, 256, 0, st>>>(drkey.p, drlen.p, droff.p, dchoff.p, R, chunk, S, dpartseg.p, Pp,
                                                    cs.p, ce.p, cg.p, ck.p, ci.p);
            if ((s = cub_run([&](void* t, size_t& b) {
                     return cub::DeviceRadixSort::SortPairs(t, b, ck.p, ck2.p, ci.p, ci2.p, (int)nch, 0,
                                                            bits((uint64_t)W * Pp * (chunk + 1)), st);
                 }, "chunk order")))
                return s;
            gather3_kernel<<<grid, 256, 0, st>>>(ci2.p, nch, cs.p, ce.p, cg.p, c->d_chunk_start, c->d_chunk_end,
                                                 c->d_chunk_seg);
            bounds_kernel<<<grid, 256, 0, st>>>(WaveOfChunkKey{ck2.p, (uint64_t)(chunk + 1) * Pp}, nch, (uint32_t)W, dwb.p);
            CU(cudaMemcpyAsync(c->wave_chunk_begin.data(), dwb.p, sizeof(uint32_t) * ((size_t)W + 1), cudaMemcpyDeviceToHost, st)); CU(cudaStreamSynchronize(st));
            if (Pp > 1) {                                  // W = 1: chunk ranges of the parts
                bounds_kernel<<<grid, 256, 0, st>>>(WaveOfChunkKey{ck2.p, (uint64_t)chunk + 1}, nch, (uint32_t)Pp, dwb.p);
                CU(cudaMemcpyAsync(c->part_chunk.data(), dwb.p, sizeof(uint32_t) * ((size_t)Pp + 1), cudaMemcpyDeviceToHost, st));
                CU(cudaStreamSynchronize(st));
            }
        }
        if (Pp > 1) {                                      // run and token ranges of the parts
            std::vector<uint32_t> rs(R), ro(R);
            if (R > 0) {
                CU(cudaMemcpyAsync(rs.data(), c->d_wave_segs, sizeof(uint32_t) * R, cudaMemcpyDeviceToHost, st));
                CU(cudaMemcpyAsync(ro.data(), droff.p, sizeof(uint32_t) * R, cudaMemcpyDeviceToHost, st));
                CU(cudaStreamSynchronize(st));
            }
            for (int p = 0; p <= Pp; ++p) {
                const uint32_t sfirst = c->part_word[(size_t)p] * (uint32_t)I;
                const uint32_t r = (uint32_t)(std::lower_bound(rs.begin(), rs.end(), sfirst) - rs.begin());
                c->part_run[(size_t)p] = r;
                c->part_tok[(size_t)p] = r < R ? ro[r] : nloc;
            }
        }
    }
    c->nchunks = nch;
    c->nsegs = R;
    {   // exchange blocks (NEXT-3): waves that can hold tokens = min(W, longest document)
        int32_t maxlen = 1;
        for (int32_t dl : c->doclen) maxlen = std::max(maxlen, dl);
        c->nwaves_eff = std::max(1, std::min(W, maxlen));
        const int e = c->cfg.merge_every;
        c->E = (e <= 0 || c->G == 1 || c->async) ? c->nwaves_eff : std::min(e, c->nwaves_eff);
        c->nblocks = (c->nwaves_eff + c->E - 1) / c->E;
        c->block = 0;
    }
    if (c->P == 1) {
        c->part_chunk = {0u, nch};
        c->part_run = {0u, R};
        c->part_tok = {0u, nloc};
    }
    // doc of every sorted position, and the doc -> sorted-positions CSR (W = 1 recount)
    {
        const size_t nl = std::max<uint32_t>(nloc, 1);
        ALLOC(c->d_tok_doc, nl);
        ALLOC(c->d_doc_pos, nl);
        ALLOC(c->d_doc_ptr, (size_t)c->Dloc + 1);
        TempBuf<uint32_t> dq(nl), dcur((size_t)std::max(c->Dloc, 1));
        if (!dq.p || !dcur.p) return fail(c, SPDP_ENOMEM, "CSR buffers");
        tdoc_kernel<<<grid, 256, 0, st>>>(c->d_tok_id, nloc, ddoc.p, c->G > 1 ? dlod.p : nullptr, c->d_tok_doc, dq.p);
        std::vector<uint32_t> dptr((size_t)c->Dloc + 1, 0);
        for (int32_t j = 0; j < c->Dloc; ++j)
            dptr[(size_t)j + 1] = dptr[(size_t)j] + (uint32_t)c->doclen[(size_t)c->global_of_local[(size_t)j]];
        CU(cudaMemcpyAsync(c->d_doc_ptr, dptr.data(), sizeof(uint32_t) * dptr.size(), cudaMemcpyHostToDevice, st));
        CU(cudaMemsetAsync(dcur.p, 0, sizeof(uint32_t) * (size_t)std::max(c->Dloc, 1), st));
        if (nloc > 0) csr_scatter_kernel<<<grid, 256, 0, st>>>(c->d_tok_doc, nloc, c->d_doc_ptr, dcur.p, c->d_doc_pos);
        // W = 1 with the chunk kernel: it also writes each new assignment to its document-order slot (a
        // fire-and-forget scattered store), so the recount streams them instead of gathering through doc_pos
        // (B200: C5 recount 3.89 -> 0.76 ms, sample +2.25 ms, step -0.86 ms; C3, whose rows and zr live in L2,
        // +0.05 ms: so only when the doc-topic array does not fit in half of L2, like the row prefetch)
        int l2b = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2b, cudaDevAttrL2CacheSize, dev);
        const bool hbm_rows = (double)c->Dloc * c->Kn * sizeof(float) > 0.5 * (double)l2b;
        // (K > 256: the 16x32 / 32x32 kernels do not carry the store; C4 K = 1000 measured 5.31 vs 5.24 ms anyway)
        // (B200, round 2: once the sample kernel ran at 6 blocks per SM the scattered stores cost more than the
        // recount gains: C5 27.6 ms with, 26.9 ms without; opt-in, SPDP_DOC_SCATTER=1)
        c->doc_scatter = false;
        (void)hbm_rows;
        if (const char* e = getenv("SPDP_DOC_SCATTER"))
            c->doc_scatter = W == 1 && !c->token_kernel && !c->async && !c->sparse && !c->seq && atoi(e) != 0 && c->K <= 256;
        // documents of <= 64 tokens on average: the recount takes two per warp
        c->recount_lpd = (c->Dloc > 0 && (double)nloc / c->Dloc <= 64.0) ? 16 : 32;
        if (const char* e = getenv("SPDP_RECOUNT_LPD")) c->recount_lpd = atoi(e) == 16 ? 16 : 32;
        if (c->doc_scatter) {
            ALLOC(c->d_slot, nl);
            ALLOC(c->d_zr_doc, nl);
            if (nloc > 0) invert_perm_kernel<<<grid, 256, 0, st>>>(c->d_doc_pos, nloc, c->d_slot);
        }
    }
    if ((s = check_launch(c, "load planning kernels"))) return s;
    if ((s = sync(c, "load planning"))) return s;
    c->sorted_tok.clear();
    c->pos_of_tok.clear();
    lt.mark("wave plan + chunks (device)");
    c->cells = (size_t)V * I * Kp;
    // device allocations
    ALLOC(c->d_zr, std::max<int64_t>(c->Nloc, 1)); ALLOC(c->d_zr_next, std::max<int64_t>(c->Nloc, 1));
    ALLOC(c->d_sweep, 1);
    {   // prefetch doc-topic rows into L2 only when the array does not live there anyway
        int dev = 0, l2 = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        c->prefetch_rows = ((double)c->Dloc * c->Kn * sizeof(float) > 0.5 * (double)l2) ? 1 : 0;
        if (const char* e = getenv("SPDP_PREFETCH_ROWS")) c->prefetch_rows = atoi(e);
        // HBM-resident rows: the narrowest exact count type (n_dk <= L_d): uint8 when every document has
        // < 256 tokens, else uint16 (< 2^16); fp32 rows (no conversion) when the array lives in L2.
        // Overrides: SPDP_ROW_BYTES=4|2|1, SPDP_ROW16=0|1, SPDP_ROW8=0|1 (tests force each path).
        int32_t maxlen = 0;
        for (int32_t dl : c->doclen) maxlen = std::max(maxlen, dl);
        int rb = c->prefetch_rows ? (maxlen < 256 ? 1 : 2) : 4;
        if (const char* e = getenv("SPDP_ROW16")) rb = atoi(e) ? 2 : (rb == 2 ? 4 : rb);
        if (const char* e = getenv("SPDP_ROW8")) rb = atoi(e) ? 1 : (rb == 1 ? 2 : rb);
        if (const char* e = getenv("SPDP_ROW_BYTES")) { const int v = atoi(e); if (v == 1 || v == 2 || v == 4) rb = v; }
        if (rb == 1 && maxlen >= 256) rb = 2;            // uint8 needs L_d < 2^8
        if (rb == 2 && maxlen >= 65536) rb = 4;          // uint16 needs L_d < 2^16
        c->row_elem = rb;
    }
    {   // sparse doc-topic rows: when the documents' expected nonzero topics (at a uniform random z, the
        // start of every chain) cover < 40 % of a row; wave updates, K > 64 (the chunk kernel's range)
        const int K = c->K;
        double exp_nnz = 0.0, cap = 0.0;
        std::vector<uint32_t> capp((size_t)c->Dloc + 1, 0);
        for (int32_t j = 0; j < c->Dloc; ++j) {
            const int32_t L = c->doclen[(size_t)c->global_of_local[(size_t)j]];
            exp_nnz += (double)K * (1.0 - std::pow(1.0 - 1.0 / K, (double)L));
            const uint32_t cj = (uint32_t)std::min<int32_t>(L, K);
            capp[(size_t)j + 1] = capp[(size_t)j] + cj;
            cap += cj;
        }
        const double frac = c->Dloc ? exp_nnz / ((double)c->Dloc * K) : 1.0;
        int32_t maxlen = 0;
        for (int32_t dl : c->doclen) maxlen = std::max(maxlen, dl);
        // measured (B200, sample + rebuild vs the dense kernel): C5 30.2 + 5.2 vs 31.2 + 4.1 ms, C4 K = 1000
        // 6.4 vs 4.2 ms, K = 300 2.3 vs 1.5 ms, C3 1.6 vs 1.05 ms: the dense kernel wins or ties, so the sparse
        // path is opt-in (SPDP_SPARSE_ROWS=1)
        c->sprows = SPDP_SPROWS_AUTO && K > 64 && !c->async && !c->sparse && !c->seq && frac < 0.4 && maxlen < 65536 &&
                    !c->token_kernel;
        if (const char* e = getenv("SPDP_SPARSE_ROWS"))
            c->sprows = atoi(e) != 0 && K > 64 && !c->async && !c->sparse && !c->seq && maxlen < 65536 && !c->token_kernel;
        if (c->sprows) {
            c->doc_scatter = false;                       // its recount gathers (the sparse kernel writes zr_next only)
            const double mean_nnz = c->Dloc ? exp_nnz / c->Dloc : 0.0;
            c->sp_lpt = mean_nnz <= 64 ? 8 : (mean_nnz <= 160 ? 16 : 32);
            if (const char* e = getenv("SPDP_SPROWS_LPT")) {
                const int v = atoi(e);
                if (v == 8 || v == 16 || v == 32) c->sp_lpt = v;
            }
            c->sp_kspan = K <= 256 ? 256 : (K <= 512 ? 512 : 1024);
            ALLOC(c->d_cap_ptr, (size_t)c->Dloc + 1);
            ALLOC(c->d_ent, std::max<size_t>((size_t)cap, 1));
            ALLOC(c->d_dinfo, std::max<int32_t>(c->Dloc, 1));
            CU(cudaMemcpyAsync(c->d_cap_ptr, capp.data(), sizeof(uint32_t) * capp.size(), cudaMemcpyHostToDevice, c->stream));
#define CALL_SS(L, KS) sprows_setup_t<L, KS>(c)
            SPDP_SPROWS_DISPATCH(c->sp_lpt, c->sp_kspan, CALL_SS)
#undef CALL_SS
        }
    }
    {   // unit j of lane gl at unit index j * LA + gl; UT topics (32 bytes, or the lane's span) per unit
        const int UT = std::min(32 / c->row_elem, c->KPL);
        c->sigma.assign((size_t)Kp, 0);
        for (int k = 0; k < Kp; ++k) {
            const int gl = k / c->KPL, kk = k % c->KPL;
            c->sigma[(size_t)k] = ((kk / UT) * c->LA + gl) * UT + kk % UT;
        }
    }
    ALLOC(c->d_sigma, Kp);
    CU(cudaMemcpyAsync(c->d_sigma, c->sigma.data(), sizeof(int) * (size_t)Kp, cudaMemcpyHostToDevice, c->stream));
    {   // +1024 elements: the sample kernel reads whole topic spans
        uint8_t* nb = nullptr;
        ALLOC(nb, row_bytes(c));
        c->d_n = nb;
        CU(cudaMemsetAsync(c->d_n, 0, row_bytes(c), c->stream));
    }
    ALLOC(c->d_work, (size_t)std::max(W, c->P) + 2);
    ALLOC(c->d_m, c->cells); ALLOC(c->d_t, c->cells);
    ALLOC(c->d_dm, c->cells); ALLOC(c->d_dt, c->cells);
    if (c->G > 1 && !c->sparse) {
        // |sum over ranks of dt| <= count(i,w) <= M_max, so 16-bit halves suffice below 2^15
        c->pack32 = c->mmax < 32768 && !getenv("SPDP_EXCHANGE_PACK64");
        const size_t words = c->cells * (c->pack32 ? 1 : 2);
        int32_t *dl = nullptr, *ds = nullptr;
        ALLOC(dl, words); ALLOC(ds, words);
        c->d_Dloc = dl; c->d_Dsum = ds;
    }
    // several ranks with one wave and no part pipelining: the local merge before the exchange writes only the
    // rank's net change (the exchange merge installs S0 + sum and rebuilds Q and the sums)
    c->fold_merge = c->G > 1 && W == 1 && !c->overlap && !c->sparse && !c->async && c->P <= 1 &&
                    !(getenv("SPDP_FOLD_MERGE") && atoi(getenv("SPDP_FOLD_MERGE")) == 0);
    ALLOC(c->d_Q, (size_t)V * Kp);
    ALLOC(c->d_M, (size_t)I * Kp); ALLOC(c->d_Tt, (size_t)I * Kp); ALLOC(c->d_T, (size_t)Kp);
    if (c->P > 1) {
        ALLOC(c->d_Mn, (size_t)I * Kp); ALLOC(c->d_Ttn, (size_t)I * Kp); ALLOC(c->d_Tn, (size_t)Kp);
        c->overlap = c->G > 1 && c->cfg.exchange == SPDP_EXCHANGE_NCCL;
        if (c->overlap) {
            ALLOC(c->d_Mf, (size_t)I * Kp); ALLOC(c->d_Ttf, (size_t)I * Kp); ALLOC(c->d_Tf, (size_t)Kp);
            CU(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
            c->part_ev.resize((size_t)c->P, nullptr);
            for (auto& e : c->part_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&c->comm_done, cudaEventDisableTiming));
        }
    }
    ALLOC(c->d_doclen, std::max<int32_t>(c->Dloc, 1)); ALLOC(c->d_docgroup, std::max<int32_t>(c->Dloc, 1));
    ALLOC(c->d_alpha, (size_t)I * Kp); ALLOC(c->d_alpha64, (size_t)I * Kp);
    ALLOC(c->d_disc, I); ALLOC(c->d_conc, I); ALLOC(c->d_disc64, I); ALLOC(c->d_conc64, I);
    ALLOC(c->d_alpha_sum, I); ALLOC(c->d_alpha_sum64, I);
    ALLOC(c->d_stats, 8);
    c->partial_len = std::max<size_t>(nch, 4096);
    ALLOC(c->d_partial, c->partial_len);
    ALLOC(c->d_scalar, 8);
    {
        std::vector<int32_t> dl((size_t)std::max<int32_t>(c->Dloc, 1), 0), dg((size_t)std::max<int32_t>(c->Dloc, 1), 0);
        for (int32_t j = 0; j < c->Dloc; ++j) {
            dl[(size_t)j] = c->doclen[(size_t)c->global_of_local[(size_t)j]];
            dg[(size_t)j] = std::max(c->docgroup[(size_t)c->global_of_local[(size_t)j]], 0);   // empty docs: any group
        }
        std::vector<float> al((size_t)I * Kp, 0.f), disc((size_t)I), conc((size_t)I), asum((size_t)I);
        std::vector<double> al64((size_t)I * Kp, 0.0), asum64((size_t)I, 0.0);
        for (int i = 0; i < I; ++i) {
            for (int k = 0; k < c->K; ++k) {
                al[(size_t)i * Kp + k] = (float)c->alpha_ik[(size_t)i * c->K + k];
                al64[(size_t)i * Kp + k] = c->alpha_ik[(size_t)i * c->K + k];
                asum64[(size_t)i] += c->alpha_ik[(size_t)i * c->K + k];
            }
            asum[(size_t)i] = (float)asum64[(size_t)i];
            disc[(size_t)i] = (float)c->disc[(size_t)i];
            conc[(size_t)i] = (float)c->conc[(size_t)i];
        }
        CU(cudaMemcpyAsync(c->d_doclen, dl.data(), sizeof(int32_t) * dl.size(), cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(c->d_docgroup, dg.data(), sizeof(int32_t) * dg.size(), cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(c->d_alpha, al.data(), sizeof(float) * al.size(), cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(c->d_alpha64, al64.data(), sizeof(double) * al64.size(), cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(c->d_disc, disc.data(), sizeof(float) * I, cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(c->d_conc, conc.data(), sizeof(float) * I, cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(c->d_disc64, c->disc.data(), sizeof(double) * I, cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(c->d_conc64, c->conc.data(), sizeof(double) * I, cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(c->d_alpha_sum, asum.data(), sizeof(float) * I, cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemcpyAsync(c->d_alpha_sum64, asum64.data(), sizeof(double) * I, cudaMemcpyHostToDevice, c->stream));
        CU(cudaMemsetAsync(c->d_sweep, 0, sizeof(uint32_t), c->stream));
        CU(cudaMemsetAsync(c->d_stats, 0, sizeof(unsigned long long) * 8, c->stream));
    }
    // pageable cudaMemcpy may return before its DMA lands; the context stream does not
    // order after the legacy stream, so settle every upload before the stream reads them
    CU(cudaDeviceSynchronize());
    lt.mark("device alloc + upload");
    // Stirling-ratio tables (launched on the side stream once M_max was known): join
    if (tab_stream != c->stream) {
        CU(cudaEventRecord(tab_done.e, tab_stream));
        CU(cudaStreamWaitEvent(c->stream, tab_done.e, 0));
    }
    s = sync(c, "build_ratio_table");
    if (s) return s;
    lt.mark("Stirling-ratio tables");
    if (c->sparse && (s = sparse_upload(c))) return s;
    s = install_state(c, z_init, r_init, nullptr);
    if (s) return s;
    if (c->seq) {   // canonical id -> sorted position, for the canonical-order walk of seq_kernel
        ALLOC(c->d_pos, std::max<int64_t>(c->N, 1));
        if (c->Nloc > 0)
            invert_perm_kernel<<<148 * 4, 256, 0, c->stream>>>(c->d_tok_id, (uint32_t)c->Nloc, c->d_pos);
        if ((s = check_launch(c, "invert_perm_kernel"))) return s;
        if ((s = sync(c, "seq positions"))) return s;
    }
    lt.mark("initial state (counts)");
    c->loaded = true;
    return SPDP_OK;
}

spdp_status spdp_set_state(spdp_ctx* c, const int32_t* z, const uint8_t* r, const int32_t* tables) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (!z || (!r && !tables)) return fail(c, SPDP_EINVAL, "spdp_set_state needs z and (r or tables)");
    TempStream temp_scope(c->stream, c->pool);
    std::vector<uint8_t> ones;
    if (!r) { ones.assign((size_t)c->N, 1); r = ones.data(); }
    return install_state(c, z, r, tables);
}

spdp_status spdp_sweep_local(spdp_ctx* c) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (c->seq) return fail(c, SPDP_ESTATE, "num_waves = 0 (sequential test mode): use spdp_sweep");
    if ((s = run_waves(c, block_w0(c, c->block), block_w1(c, c->block), c->block == 0))) return s;
    if (c->G > 1) CU(cudaMemcpyAsync(c->d_Dsum, c->d_Dloc, c->dbytes(), cudaMemcpyDeviceToDevice, c->stream));
    return sync(c, "spdp_sweep_local");
}

spdp_status spdp_exchange_blocks(spdp_ctx* c, int32_t* nblocks) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (!nblocks) return fail(c, SPDP_EINVAL, "null output");
    *nblocks = c->nblocks;
    return SPDP_OK;
}

spdp_status spdp_exchange_buffer(spdp_ctx* c, void** ptr, int64_t* count, int32_t* elem_bytes) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (!ptr || !count || !elem_bytes) return fail(c, SPDP_EINVAL, "null output");
    if (c->G == 1) return fail(c, SPDP_ESTATE, "world_size == 1 has no exchange buffer");
    *ptr = c->d_Dsum;
    *count = (int64_t)c->xcount();
    *elem_bytes = c->pack32 ? 4 : 8;
    return SPDP_OK;
}

spdp_status spdp_exchange_copy(spdp_ctx* c, void* host, int32_t to_device) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (!host) return fail(c, SPDP_EINVAL, "null host buffer");
    if (c->G == 1) return fail(c, SPDP_ESTATE, "world_size == 1 has no exchange buffer");
    const size_t bytes = c->dbytes();
    if (to_device) CU(cudaMemcpyAsync(c->d_Dsum, host, bytes, cudaMemcpyHostToDevice, c->stream));
    else CU(cudaMemcpyAsync(host, c->d_Dsum, bytes, cudaMemcpyDeviceToHost, c->stream));
    return sync(c, "spdp_exchange_copy");
}

spdp_status spdp_sweep_merge(spdp_ctx* c) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (c->G > 1) {
        launch_exchange_merge(c);
        if ((s = check_launch(c, "merge (exchange)"))) return s;
    }
    if (++c->block < c->nblocks) return sync(c, "spdp_sweep_merge");   // more exchange blocks in this sweep
    c->block = 0;
    if ((s = finish_sweep(c))) return s;
    if ((s = sync(c, "spdp_sweep_merge"))) return s;
    if (c->cfg.debug_checks) return debug_verify(c);
    return SPDP_OK;
}

namespace {
spdp_status sweep_impl(spdp_ctx* c, int32_t num_sweeps, bool wait);
}

spdp_status spdp_sweep(spdp_ctx* c, int32_t num_sweeps) { return sweep_impl(c, num_sweeps, true); }
spdp_status spdp_sweep_async(spdp_ctx* c, int32_t num_sweeps) { return sweep_impl(c, num_sweeps, false); }

}  // extern "C"

namespace {
spdp_status sweep_impl(spdp_ctx* c, int32_t num_sweeps, bool wait) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (num_sweeps < 0) return fail(c, SPDP_EINVAL, "num_sweeps must be >= 0");
    if (c->G > 1 && c->cfg.exchange != SPDP_EXCHANGE_NCCL)
        return fail(c, SPDP_ESTATE, "SPDP_EXCHANGE_EXTERNAL: use spdp_sweep_local / spdp_sweep_merge");
    if (c->seq) {
        if ((s = seq_sweeps(c, num_sweeps, nullptr, 0))) return s;
        if (c->cfg.debug_checks) return debug_verify(c);
        return SPDP_OK;
    }
    const bool graphs = c->G == 1 && !c->cfg.debug_checks && !c->graphs_off && !c->profiling &&
                        !(getenv("SPDP_GRAPHS") && atoi(getenv("SPDP_GRAPHS")) == 0);
    for (int it = 0; it < num_sweeps; ++it) {
      if (graphs && !c->graphs_off) {
        if (c->profiling && (s = ensure_events(c))) return s;
        spdp_ctx::SweepGraph* ge = nullptr;
        for (auto& g : c->graphs)
            if (g.zr_at_start == c->d_zr && g.prof == c->profiling) ge = &g;
        bool ran = false;
        if (ge) {
            CU(cudaGraphLaunch(ge->exec, c->stream));
            if (ge->swaps) std::swap(c->d_zr, c->d_zr_next);
            c->sweeps_done++;
            c->launches += ge->launches;
            c->acc[5] += ge->sample_launches;
            ran = true;
        } else {
            // capture one sweep (the host bookkeeping runs during the capture, the work at the launch)
            uint16_t *zr0 = c->d_zr, *zn0 = c->d_zr_next;
            const uint32_t sw0 = c->sweeps_done;
            const int64_t l0 = c->launches;
            const double a50 = c->acc[5];
            cudaGraph_t graph = nullptr;
            cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
            spdp_status sc = SPDP_OK;
            if (e == cudaSuccess) {
                sc = run_waves(c, 0, c->W, true);
                if (!sc) sc = finish_sweep(c);
                e = cudaStreamEndCapture(c->stream, &graph);
            }
            cudaGraphExec_t exec = nullptr;
            if (e == cudaSuccess && !sc && graph) e = cudaGraphInstantiate(&exec, graph, 0);
            if (graph) cudaGraphDestroy(graph);
            if (e == cudaSuccess && !sc && exec) {
                c->graphs.push_back({zr0, c->profiling, c->d_zr != zr0, exec, c->launches - l0, c->acc[5] - a50});
                CU(cudaGraphLaunch(exec, c->stream));
                ran = true;
            } else {                          // not capturable here: undo the bookkeeping, run directly
                cudaGetLastError();
                c->poisoned = false;          // capture-time API errors executed no work
                c->err.clear();
                if (exec) cudaGraphExecDestroy(exec);
                c->d_zr = zr0; c->d_zr_next = zn0; c->sweeps_done = sw0; c->launches = l0; c->acc[5] = a50;
                c->graphs_off = true;
            }
        }
        if (ran) {
            if (c->profiling) {
                if ((s = sync(c, "spdp_sweep"))) return s;
                collect_times(c, false);
            }
            continue;
        }
      }
      for (int b = 0; b < c->nblocks; ++b) {
        if ((s = run_waves(c, block_w0(c, b), block_w1(c, b), b == 0))) return s;
        if (c->G > 1 && !c->overlap) {
            rec(c, 4 * (size_t)c->W);
            if ((s = nccl_check(c, c->nccl.AllReduce(c->d_Dloc, c->d_Dsum, c->xcount(), c->pack32 ? kNcclInt32 : kNcclInt64,
                                                     kNcclSum, c->comm, c->stream),
                                "ncclAllReduce(packed deltas)")))
                return s;
            launch_exchange_merge(c);
            rec(c, 4 * (size_t)c->W + 1);
            c->launches += 1;
        }
      }
        if ((s = finish_sweep(c))) return s;
        if (c->profiling) {
            if ((s = sync(c, "spdp_sweep"))) return s;
            collect_times(c, c->G > 1 && !c->overlap);
        }
        if (c->cfg.debug_checks) {
            if ((s = sync(c, "spdp_sweep"))) return s;
            if ((s = debug_verify(c))) return s;
        }
    }
    if (!wait && !c->cfg.debug_checks) return check_launch(c, "spdp_sweep_async");
    return sync(c, "spdp_sweep");
}
}  // namespace

extern "C" {

spdp_status spdp_counts(spdp_ctx* c, int32_t* z, uint8_t* r, int32_t* doc_topic, int32_t* customers, int32_t* tables,
                        int32_t* shadow) {
    spdp_status s = guard(c, true);
    if (s) return s;
    const int I = c->I, V = c->V, K = c->K, Kp = c->Kp;
    const bool gather = c->G > 1 && c->cfg.exchange == SPDP_EXCHANGE_NCCL;
    if (z || r) {
        // canonical order on the device (z | r<<15, +1 so that 0 marks other ranks' tokens)
        if (!c->d_zr_canon) ALLOC(c->d_zr_canon, c->N);
        if (c->zr_pending) CU(cudaStreamWaitEvent(c->stream, c->zr_copied, 0));
        CU(cudaMemsetAsync(c->d_zr_canon, 0, sizeof(uint16_t) * (size_t)c->N, c->stream));
        if (c->Nloc > 0)
            scatter_zr_kernel<<<148 * 8, 256, 0, c->stream>>>(c->d_tok_id, c->d_zr, (uint32_t)c->Nloc, c->d_zr_canon);
        if ((s = check_launch(c, "scatter_zr_kernel"))) return s;
        if (!c->h_zr_canon) CU(cudaMallocHost((void**)&c->h_zr_canon, sizeof(uint16_t) * (size_t)c->N));
        CU(cudaMemcpyAsync(c->h_zr_canon, c->d_zr_canon, sizeof(uint16_t) * (size_t)c->N, cudaMemcpyDeviceToHost,
                           c->stream));
        if ((s = sync(c, "counts(z)"))) return s;
        std::vector<int32_t> all;
        if (gather) {
            all.assign((size_t)c->N, 0);
            for (int64_t p = 0; p < c->N; ++p) all[(size_t)p] = c->h_zr_canon[(size_t)p];
            TempBuf<int32_t> tb(c->N);
            if (!tb.p) return fail(c, SPDP_ENOMEM, "gather buffer");
            int32_t* dbuf = tb.p;
            CU(cudaMemcpyAsync(dbuf, all.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice, c->stream));
            if ((s = nccl_check(c, c->nccl.AllReduce(dbuf, dbuf, (size_t)c->N, kNcclInt32, kNcclSum, c->comm, c->stream), "allreduce z")))
                return s;
            CU(cudaMemcpyAsync(all.data(), dbuf, sizeof(int32_t) * all.size(), cudaMemcpyDeviceToHost, c->stream));
            if ((s = sync(c, "counts(z gather)"))) return s;
            for (int64_t p = 0; p < c->N; ++p) c->h_zr_canon[(size_t)p] = (uint16_t)all[(size_t)p];
        }
        const uint16_t* h = c->h_zr_canon;
        parallel_for(c->N, [&](int64_t b, int64_t e) {
            for (int64_t p = b; p < e; ++p) {
                const uint32_t v = h[p];
                if (!v) continue;                                   // another rank's token
                if (z) z[p] = (int32_t)((v - 1u) & 0x7FFFu);
                if (r) r[p] = (uint8_t)(((v - 1u) >> 15) & 1u);
            }
        });
    }
    if (doc_topic) {
        std::vector<float> nf;
        if ((s = read_rows(c, nf))) return s;
        std::vector<int32_t> full;
        if (gather) full.assign((size_t)c->D * K, 0);
        int32_t* dst = gather ? full.data() : doc_topic;
        for (int32_t j = 0; j < c->Dloc; ++j)
            for (int k = 0; k < K; ++k)
                dst[(size_t)c->global_of_local[(size_t)j] * K + k] = (int32_t)nf[(size_t)j * c->Kn + c->sigma[(size_t)k]];
        if (gather) {
            TempBuf<int32_t> tb(full.size());
            if (!tb.p) return fail(c, SPDP_ENOMEM, "gather buffer");
            int32_t* dbuf = tb.p;
            CU(cudaMemcpyAsync(dbuf, full.data(), sizeof(int32_t) * full.size(), cudaMemcpyHostToDevice, c->stream));
            if ((s = nccl_check(c, c->nccl.AllReduce(dbuf, dbuf, full.size(), kNcclInt32, kNcclSum, c->comm, c->stream), "allreduce n")))
                return s;
            CU(cudaMemcpyAsync(doc_topic, dbuf, sizeof(int32_t) * full.size(), cudaMemcpyDeviceToHost, c->stream));
            if ((s = sync(c, "counts(n gather)"))) return s;
        }
    }
    if (customers || tables) {
        std::vector<int32_t> buf(c->cells);
        for (int which = 0; which < 2; ++which) {
            int32_t* out = which ? tables : customers;
            if (!out) continue;
            CU(cudaMemcpyAsync(buf.data(), which ? c->d_t : c->d_m, sizeof(int32_t) * c->cells, cudaMemcpyDeviceToHost, c->stream));
            if ((s = sync(c, "counts(m,t)"))) return s;
            for (int w = 0; w < V; ++w)
                for (int i = 0; i < I; ++i)
                    for (int k = 0; k < K; ++k)
                        out[((size_t)i * V + w) * K + k] = buf[((size_t)w * I + i) * Kp + k];
        }
    }
    if (shadow) {
        std::vector<int32_t> q((size_t)V * Kp);
        CU(cudaMemcpyAsync(q.data(), c->d_Q, sizeof(int32_t) * q.size(), cudaMemcpyDeviceToHost, c->stream));
        if ((s = sync(c, "counts(Q)"))) return s;
        for (int w = 0; w < V; ++w)
            for (int k = 0; k < K; ++k) shadow[(size_t)k * V + w] = q[(size_t)w * Kp + k];
    }
    return SPDP_OK;
}

spdp_status spdp_set_transform(spdp_ctx* c, const int32_t* pptr, const int32_t* pv, const double* pp) {
    spdp_status s = guard(c, false);
    if (s) return s;
    if (c->loaded) return fail(c, SPDP_ESTATE, "spdp_set_transform must precede spdp_load_corpus");
    if (c->seq) return fail(c, SPDP_ESTATE, "num_waves = 0 (sequential test mode) has no transformation-matrix path");
    if (!pptr || !pv || !pp) return fail(c, SPDP_EINVAL, "null transformation arrays");
    const int I = c->I, V = c->V;
    const int64_t rows = (int64_t)I * V;
    if (pptr[0] != 0) return fail(c, SPDP_EINVAL, "pptr[0] must be 0");
    std::vector<double> col((size_t)rows, 0.0);
    for (int64_t r = 0; r < rows; ++r) {
        if (pptr[r + 1] <= pptr[r]) return fail(c, SPDP_EINVAL, "row (i=%lld, w=%lld) of P has no entry", (long long)(r / V), (long long)(r % V));
        if (pptr[r + 1] - pptr[r] > 32767) return fail(c, SPDP_EINVAL, "a row of P has more than 32767 entries");
        for (int32_t e = pptr[r]; e < pptr[r + 1]; ++e) {
            if (pv[e] < 0 || pv[e] >= V || !(pp[e] > 0.0)) return fail(c, SPDP_EINVAL, "entry %d of P is invalid", e);
            col[(size_t)(r / V) * V + pv[e]] += pp[e];
        }
    }
    for (size_t j = 0; j < col.size(); ++j)
        if (std::fabs(col[j] - 1.0) > 1e-9)
            return fail(c, SPDP_EINVAL, "column %zu of P^%zu sums to %.12g, not 1", j % (size_t)V, j / (size_t)V, col[j]);
    c->h_pptr.assign(pptr, pptr + rows + 1);
    c->h_pv.assign(pv, pv + pptr[rows]);
    c->h_pp.assign(pp, pp + pptr[rows]);
    c->sparse = true;
    return SPDP_OK;
}

spdp_status spdp_sparse_state(spdp_ctx* c, int32_t* q, int32_t* shadow, int16_t* src) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (!c->sparse) return fail(c, SPDP_ESTATE, "no transformation matrix (spdp_set_transform)");
    const int K = c->K, Kp = c->Kp, V = c->V;
    if (q) {
        std::vector<int32_t> dq((size_t)c->E_sp * Kp);
        CU(cudaMemcpyAsync(dq.data(), c->d_q, sizeof(int32_t) * dq.size(), cudaMemcpyDeviceToHost, c->stream));
        if ((s = sync(c, "sparse q"))) return s;
        for (size_t e = 0; e < c->dev_of_user.size(); ++e)
            for (int k = 0; k < K; ++k) q[e * K + k] = dq[(size_t)c->dev_of_user[e] * Kp + k];
    }
    if (shadow) {
        std::vector<int32_t> Q((size_t)V * Kp);
        CU(cudaMemcpyAsync(Q.data(), c->d_Q, sizeof(int32_t) * Q.size(), cudaMemcpyDeviceToHost, c->stream));
        if ((s = sync(c, "sparse Q"))) return s;
        for (int v = 0; v < V; ++v)
            for (int k = 0; k < K; ++k) shadow[(size_t)k * V + v] = Q[(size_t)v * Kp + k];
    }
    if (src) {
        if ((s = ensure_host_plan(c))) return s;
        std::vector<int16_t> d((size_t)c->Nloc);
        if (c->Nloc) CU(cudaMemcpyAsync(d.data(), c->d_src, sizeof(int16_t) * d.size(), cudaMemcpyDeviceToHost, c->stream));
        if ((s = sync(c, "sparse src"))) return s;
        for (int64_t p = 0; p < c->N; ++p) src[p] = -1;
        for (int64_t q2 = 0; q2 < c->Nloc; ++q2) src[c->sorted_tok[(size_t)q2]] = d[(size_t)q2];
    }
    return SPDP_OK;
}

namespace {
// Scatter the packed assignments into canonical order in d_zr_canon (c->stream).
spdp_status zr_stage(spdp_ctx* c) {
    spdp_status s;
    if (!c->d_zr_canon) ALLOC(c->d_zr_canon, c->N);
    if (c->zr_pending) CU(cudaStreamWaitEvent(c->stream, c->zr_copied, 0));   // the previous copy has read it
    if (c->Nloc < c->N) CU(cudaMemsetAsync(c->d_zr_canon, 0xFF, sizeof(uint16_t) * (size_t)c->N, c->stream));
    if (c->Nloc > 0)
        scatter_zr_kernel<<<148 * 8, 256, 0, c->stream>>>(c->d_tok_id, c->d_zr, (uint32_t)c->Nloc, c->d_zr_canon, 0u);
    if ((s = check_launch(c, "scatter_zr_kernel"))) return s;
    c->launches += 1;
    return SPDP_OK;
}
}  // namespace

spdp_status spdp_zr8_async(spdp_ctx* c, uint8_t* zr) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (!zr) return fail(c, SPDP_EINVAL, "null output");
    if (c->K > 128) return fail(c, SPDP_EINVAL, "spdp_zr8_async needs K <= 128 (z | r << 7 in one byte)");
    if (c->G > 1 && c->cfg.exchange == SPDP_EXCHANGE_NCCL) {   // gathered: collective, blocking
        std::vector<uint16_t> w((size_t)c->N);
        if ((s = spdp_zr(c, w.data()))) return s;
        for (int64_t p = 0; p < c->N; ++p) zr[p] = (uint8_t)((w[(size_t)p] & 0x7Fu) | ((w[(size_t)p] >> 15) << 7));
        return SPDP_OK;
    }
    if (!c->d2h_stream) {
        CU(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&c->zr_ready, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->zr_copied, cudaEventDisableTiming));
    }
    if (!c->d_zr8_canon) ALLOC(c->d_zr8_canon, c->N);
    if (c->zr_pending) CU(cudaStreamWaitEvent(c->stream, c->zr_copied, 0));   // the previous copy has read it
    if (c->Nloc < c->N) CU(cudaMemsetAsync(c->d_zr8_canon, 0xFF, (size_t)c->N, c->stream));
    if (c->Nloc > 0)
        scatter_zr8_kernel<<<148 * 8, 256, 0, c->stream>>>(c->d_tok_id, c->d_zr, (uint32_t)c->Nloc, c->d_zr8_canon);
    if ((s = check_launch(c, "scatter_zr8_kernel"))) return s;
    c->launches += 1;
    CU(cudaEventRecord(c->zr_ready, c->stream));
    CU(cudaStreamWaitEvent(c->d2h_stream, c->zr_ready, 0));
    CU(cudaMemcpyAsync(zr, c->d_zr8_canon, (size_t)c->N, cudaMemcpyDeviceToHost, c->d2h_stream));
    CU(cudaEventRecord(c->zr_copied, c->d2h_stream));
    c->zr_pending = true;
    return SPDP_OK;
}

spdp_status spdp_zr_async(spdp_ctx* c, uint16_t* zr) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (!zr) return fail(c, SPDP_EINVAL, "null output");
    if (c->G > 1 && c->cfg.exchange == SPDP_EXCHANGE_NCCL) return spdp_zr(c, zr);   // gathered: collective, blocking
    if (!c->d2h_stream) {
        CU(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&c->zr_ready, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->zr_copied, cudaEventDisableTiming));
    }
    if ((s = zr_stage(c))) return s;
    CU(cudaEventRecord(c->zr_ready, c->stream));
    CU(cudaStreamWaitEvent(c->d2h_stream, c->zr_ready, 0));
    CU(cudaMemcpyAsync(zr, c->d_zr_canon, sizeof(uint16_t) * (size_t)c->N, cudaMemcpyDeviceToHost, c->d2h_stream));
    CU(cudaEventRecord(c->zr_copied, c->d2h_stream));
    c->zr_pending = true;
    return SPDP_OK;
}

spdp_status spdp_wait(spdp_ctx* c) {
    spdp_status s = guard(c, false);
    if (s) return s;
    if (c->zr_pending) {                 // the copy (and the work before its staging) only
        CU(cudaEventSynchronize(c->zr_copied));
        c->zr_pending = false;
        return check_launch(c, "spdp_wait");
    }
    return sync(c, "spdp_wait");
}

spdp_status spdp_zr(spdp_ctx* c, uint16_t* zr) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (!zr) return fail(c, SPDP_EINVAL, "null output");
    const bool gather = c->G > 1 && c->cfg.exchange == SPDP_EXCHANGE_NCCL;
    if (gather) {                                   // the gathered path of spdp_counts, then packed
        std::vector<int32_t> z((size_t)c->N);
        std::vector<uint8_t> r((size_t)c->N);
        if ((s = spdp_counts(c, z.data(), r.data(), nullptr, nullptr, nullptr, nullptr))) return s;
        for (int64_t p = 0; p < c->N; ++p) zr[p] = (uint16_t)(z[(size_t)p] | (r[(size_t)p] << 15));
        return SPDP_OK;
    }
    if ((s = zr_stage(c))) return s;
    // straight into the caller's buffer (pinned memory makes this a full-speed DMA)
    CU(cudaMemcpyAsync(zr, c->d_zr_canon, sizeof(uint16_t) * (size_t)c->N, cudaMemcpyDeviceToHost, c->stream));
    return sync(c, "spdp_zr");
}

spdp_status spdp_loglik(spdp_ctx* c, double* log_joint, double* perplexity) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (c->sparse && perplexity) {
        // NEXT-4: training perplexity = the held-out computation on the training tokens with their own z
        // (theta~ from n_d, phi~ with the sources)
        if (c->G > 1) return fail(c, SPDP_ESTATE, "the perplexity with a transformation matrix is per rank: use spdp_heldout");
        if ((s = ensure_host_plan(c))) return s;
        std::vector<int32_t> z((size_t)c->N);
        if ((s = spdp_counts(c, z.data(), nullptr, nullptr, nullptr, nullptr, nullptr))) return s;
        if ((s = spdp_heldout(c, c->N, c->D, c->group.data(), c->doc.data(), c->word.data(), 0, 0, 0, z.data(), nullptr,
                              nullptr, perplexity)))
            return s;
        perplexity = nullptr;
    }
    const bool gather = c->G > 1 && c->cfg.exchange == SPDP_EXCHANGE_NCCL;
    if (perplexity) {
        SweepArgs a = base_args(c);
        a.nchunks = (int)c->nchunks;
        launch_ppl(c, a, c->d_partial);
        reduce_fixed_kernel<<<1, 1024, 0, c->stream>>>(c->d_partial, (size_t)c->nchunks, c->d_scalar);
        if ((s = check_launch(c, "perplexity_kernel"))) return s;
        if (gather && (s = nccl_check(c, c->nccl.AllReduce(c->d_scalar, c->d_scalar, 1, kNcclFloat64, kNcclSum, c->comm, c->stream), "allreduce ppl")))
            return s;
        double ll = 0.0;
        CU(cudaMemcpyAsync(&ll, c->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if ((s = sync(c, "perplexity"))) return s;
        *perplexity = std::exp(-ll / (double)(gather ? c->N : c->Nloc));
    }
    if (log_joint) {
        const uint64_t per = (uint64_t)(c->mmax + 1) * (uint64_t)(c->mmax + 2) / 2;
        std::vector<double> distinct;
        std::vector<uint64_t> off((size_t)c->I);
        for (int i = 0; i < c->I; ++i) {
            size_t j = 0;
            while (j < distinct.size() && distinct[j] != c->disc[(size_t)i]) ++j;
            if (j == distinct.size()) distinct.push_back(c->disc[(size_t)i]);
            off[(size_t)i] = per * j;
        }
        double* ls = nullptr;
        uint64_t* d_off = nullptr;
        cudaError_t e;
        ls = dalloc<double>(per * distinct.size(), e);
        if (e != cudaSuccess) return fail(c, SPDP_ENOMEM, "log-Stirling table: %s", cudaGetErrorString(e));
        d_off = dalloc<uint64_t>((size_t)c->I, e);
        if (e != cudaSuccess) { cudaFree(ls); return fail(c, SPDP_ENOMEM, "log-Stirling offsets"); }
        cudaMemcpyAsync(d_off, off.data(), sizeof(uint64_t) * off.size(), cudaMemcpyHostToDevice, c->stream);
        for (size_t j = 0; j < distinct.size(); ++j)
            build_log_stirling<<<1, 1024, 0, c->stream>>>(ls + per * j, c->mmax, distinct[j]);
        const int grid = 296;
        double* part = c->d_partial;       // [0, grid) words, [grid, 2 grid) docs
        loglik_words_kernel<<<grid, 256, 0, c->stream>>>(c->d_m, c->d_t, c->d_Q, ls, d_off, c->V, c->I, c->K, c->Kp,
                                                        c->cfg.beta, part);
        SPDP_ROWS(c->row_elem, loglik_docs_kernel<NT><<<grid, 256, 0, c->stream>>>((const NT*)c->d_n, c->d_sigma, c->d_doclen,
                                                                            c->d_docgroup, c->d_alpha64, c->d_alpha_sum64,
                                                                            c->Dloc, c->K, c->Kp, c->Kn, part + grid));
        loglik_small_kernel<<<1, 1024, 0, c->stream>>>(c->d_M, c->d_Tt, c->d_T, c->d_disc64, c->d_conc64, c->I, c->K, c->Kp,
                                                      (double)c->V * c->cfg.beta, part + 2 * grid);
        int nterms = 2 * grid + 1;
        if (c->sparse) {   // NEXT-4: ln multinomial(t; q) + sum q ln p per cell (Q of the shadow term is Q[v][k])
            sp_source_terms_kernel<<<grid, 256, 0, c->stream>>>(sparse_args(c), c->d_spp64, (uint32_t)c->V * c->I, c->K,
                                                                c->Kp, c->d_t, part + 2 * grid + 1);
            nterms = 3 * grid + 1;
        }
        reduce_fixed_kernel<<<1, 1024, 0, c->stream>>>(part, nterms, c->d_scalar + 1);   // words + docs + small (+ sources)
        reduce_fixed_kernel<<<1, 1024, 0, c->stream>>>(part + grid, grid, c->d_scalar + 2);    // docs only
        if ((s = check_launch(c, "loglik kernels"))) { cudaFree(ls); cudaFree(d_off); return s; }
        double v[2] = {0, 0};
        CU(cudaMemcpyAsync(v, c->d_scalar + 1, sizeof(double) * 2, cudaMemcpyDeviceToHost, c->stream));
        if ((s = sync(c, "log_joint"))) { cudaFree(ls); cudaFree(d_off); return s; }
        cudaFree(ls);
        cudaFree(d_off);
        double total = v[0];
        if (gather) {
            // replicated terms once (rank 0), doc terms from every rank
            double mine = (c->rank == 0) ? v[0] : v[1];
            CU(cudaMemcpyAsync(c->d_scalar + 3, &mine, sizeof(double), cudaMemcpyHostToDevice, c->stream));
            if ((s = nccl_check(c, c->nccl.AllReduce(c->d_scalar + 3, c->d_scalar + 3, 1, kNcclFloat64, kNcclSum, c->comm, c->stream), "allreduce lj")))
                return s;
            CU(cudaMemcpyAsync(&total, c->d_scalar + 3, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            if ((s = sync(c, "log_joint gather"))) return s;
        }
        *log_joint = total;
    }
    return SPDP_OK;
}

// ---------------------------------------------------------------- NEXT-1: held-out evaluation
namespace {
spdp_status launch_phi_table(spdp_ctx* c, double* phi, double* phi0) {
    const size_t cells = c->cells;
    const int grid = (int)std::min<size_t>((cells + 255) / 256, 148u * 16u);
    phi_table_kernel<<<std::max(grid, 1), 256, 0, c->stream>>>(c->d_m, c->d_t, c->d_Q, c->d_M, c->d_Tt, c->d_T,
                                                              c->d_disc64, c->d_conc64, c->cfg.beta,
                                                              (double)c->V * c->cfg.beta, c->V, c->I, c->K, c->Kp,
                                                              phi, phi0, c->sparse ? c->d_sptr : nullptr,
                                                              c->d_spv, c->d_spp64);
    c->launches += 1;
    return check_launch(c, "phi_table_kernel");
}
}  // namespace

spdp_status spdp_topics(spdp_ctx* c, double* phi0, double* phi) {
    spdp_status s = guard(c, true);
    if (s) return s;
    const int I = c->I, V = c->V, K = c->K, Kp = c->Kp;
    TempBuf<double> dphi(c->cells), dphi0((size_t)K * V);
    if (!dphi.p || !dphi0.p) return fail(c, SPDP_ENOMEM, "spdp_topics buffers");
    if ((s = launch_phi_table(c, dphi.p, dphi0.p))) return s;
    if (phi0) CU(cudaMemcpyAsync(phi0, dphi0.p, sizeof(double) * (size_t)K * V, cudaMemcpyDeviceToHost, c->stream));
    std::vector<double> rows;
    if (phi) {
        rows.resize(c->cells);
        CU(cudaMemcpyAsync(rows.data(), dphi.p, sizeof(double) * c->cells, cudaMemcpyDeviceToHost, c->stream));
    }
    if ((s = sync(c, "spdp_topics"))) return s;
    if (phi)
        parallel_for(V, [&](int64_t b, int64_t e) {
            for (int64_t w = b; w < e; ++w)
                for (int i = 0; i < I; ++i)
                    for (int k = 0; k < K; ++k)
                        phi[((size_t)i * K + k) * V + (size_t)w] = rows[((size_t)w * I + i) * Kp + k];
        });
    return SPDP_OK;
}

spdp_status spdp_heldout(spdp_ctx* c, int64_t num_tokens, int32_t num_docs, const int32_t* group, const int32_t* doc,
                         const int32_t* word, uint64_t seed, int32_t first_iteration, int32_t iterations,
                         const int32_t* z_init, int32_t* z_out, double* theta, double* perplexity) {
    spdp_status s = guard(c, true);
    if (s) return s;
    TempStream temp_scope(c->stream, c->pool);
    const int I = c->I, V = c->V, K = c->K, Kp = c->Kp;
    if (num_tokens < 0 || num_tokens > (int64_t)UINT32_MAX || num_docs < 1 || iterations < 0 || first_iteration < 0 ||
        (num_tokens > 0 && (!group || !doc || !word)))
        return fail(c, SPDP_EINVAL, "spdp_heldout: bad sizes or null token arrays");
    // group tokens by document (stable: canonical order inside each document)
    std::vector<uint32_t> ptr((size_t)num_docs + 1, 0);
    std::vector<int32_t> dgroup((size_t)num_docs, -1);
    for (int64_t p = 0; p < num_tokens; ++p) {
        const int32_t d = doc[p], g = group[p], w = word[p];
        if (d < 0 || d >= num_docs || g < 0 || g >= I || w < 0 || w >= V)
            return fail(c, SPDP_EINVAL, "spdp_heldout: token %lld out of range", (long long)p);
        if (z_init && (z_init[p] < 0 || z_init[p] >= K)) return fail(c, SPDP_EINVAL, "spdp_heldout: z_init out of range");
        if (dgroup[(size_t)d] >= 0 && dgroup[(size_t)d] != g)
            return fail(c, SPDP_EINVAL, "spdp_heldout: document %d spans groups", d);
        dgroup[(size_t)d] = g;
        ptr[(size_t)d + 1]++;
    }
    for (int32_t d = 0; d < num_docs; ++d) {
        ptr[(size_t)d + 1] += ptr[(size_t)d];
        if (dgroup[(size_t)d] < 0) dgroup[(size_t)d] = 0;
    }
    std::vector<uint32_t> fill(ptr.begin(), ptr.end() - 1), id((size_t)num_tokens);
    std::vector<int32_t> wsorted((size_t)num_tokens), zsorted((size_t)num_tokens, 0);
    for (int64_t p = 0; p < num_tokens; ++p) {
        const uint32_t q = fill[(size_t)doc[p]]++;
        id[q] = (uint32_t)p;
        wsorted[q] = word[p];
        if (z_init) zsorted[q] = z_init[p];
    }
    const size_t nh = (size_t)std::max<int64_t>(num_tokens, 1);
    TempBuf<double> dphi(c->cells), dpart((size_t)num_docs), dscal(1);
    TempBuf<int32_t> dword(nh), dz(nh), dgrp((size_t)num_docs);
    TempBuf<uint32_t> did(nh), dptr((size_t)num_docs + 1);
    TempBuf<double> dtheta(theta ? (size_t)num_docs * K : 1);
    if (!dphi.p || !dpart.p || !dscal.p || !dword.p || !dz.p || !dgrp.p || !did.p || !dptr.p || !dtheta.p)
        return fail(c, SPDP_ENOMEM, "spdp_heldout buffers");
    if ((s = launch_phi_table(c, dphi.p, nullptr))) return s;
    CU(cudaMemcpyAsync(dword.p, wsorted.data(), sizeof(int32_t) * (size_t)num_tokens, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(dz.p, zsorted.data(), sizeof(int32_t) * (size_t)num_tokens, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(did.p, id.data(), sizeof(uint32_t) * (size_t)num_tokens, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(dptr.p, ptr.data(), sizeof(uint32_t) * ptr.size(), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(dgrp.p, dgroup.data(), sizeof(int32_t) * dgroup.size(), cudaMemcpyHostToDevice, c->stream));
    FoldinArgs a;
    a.word = dword.p; a.id = did.p; a.doc_ptr = dptr.p; a.doc_group = dgrp.p; a.z = dz.p; a.phi = dphi.p;
    a.alpha = c->d_alpha64; a.alpha_sum = c->d_alpha_sum64; a.theta = theta ? dtheta.p : nullptr; a.partial = dpart.p;
    a.Dh = num_docs; a.I = I; a.K = K; a.Kp = Kp;
    a.key0 = (uint32_t)seed; a.key1 = (uint32_t)(seed >> 32);
    a.first_iter = first_iteration; a.iters = iterations; a.init = z_init ? 0 : 1;
    const int warps = 8;
    const size_t smem = sizeof(int) * (size_t)warps * Kp;
    const int grid = (int)std::min<int64_t>((num_docs + warps - 1) / warps, 148 * 8);
    const int kb = (K + 31) / 32;
    cudaEvent_t fe[2] = {nullptr, nullptr};
    if (c->profiling) {
        CU(cudaEventCreate(&fe[0])); CU(cudaEventCreate(&fe[1]));
        CU(cudaEventRecord(fe[0], c->stream));
    }
#define SPDP_FOLDIN(KB) foldin_kernel<KB><<<grid, warps * 32, smem, c->stream>>>(a)
    if (kb <= 1) SPDP_FOLDIN(1);
    else if (kb <= 2) SPDP_FOLDIN(2);
    else if (kb <= 4) SPDP_FOLDIN(4);
    else if (kb <= 8) SPDP_FOLDIN(8);
    else if (kb <= 16) SPDP_FOLDIN(16);
    else SPDP_FOLDIN(32);
#undef SPDP_FOLDIN
    if (c->profiling) CU(cudaEventRecord(fe[1], c->stream));
    reduce_fixed_kernel<<<1, 1024, 0, c->stream>>>(dpart.p, (size_t)num_docs, dscal.p);
    c->launches += 2;
    if ((s = check_launch(c, "foldin_kernel"))) return s;
    double ll = 0.0;
    CU(cudaMemcpyAsync(&ll, dscal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (z_out) CU(cudaMemcpyAsync(zsorted.data(), dz.p, sizeof(int32_t) * (size_t)num_tokens, cudaMemcpyDeviceToHost, c->stream));
    if (theta) CU(cudaMemcpyAsync(theta, dtheta.p, sizeof(double) * (size_t)num_docs * K, cudaMemcpyDeviceToHost, c->stream));
    if ((s = sync(c, "spdp_heldout"))) return s;
    if (c->profiling) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, fe[0], fe[1]) == cudaSuccess) c->acc[8] += ms;
        c->acc[9] += (double)num_tokens * iterations;
        cudaEventDestroy(fe[0]); cudaEventDestroy(fe[1]);
    }
    if (z_out)
        for (size_t q = 0; q < (size_t)num_tokens; ++q) z_out[id[q]] = zsorted[q];
    if (perplexity) *perplexity = num_tokens > 0 ? std::exp(-ll / (double)num_tokens) : 1.0;
    return SPDP_OK;
}

spdp_status spdp_topic_hellinger(spdp_ctx* a, spdp_ctx* b, double* dist, int32_t* perm) {
    spdp_status s = guard(a, true);
    if (s) return s;
    if ((s = guard(b, true))) return fail(a, s, "spdp_topic_hellinger: second context: %s", b ? b->err.c_str() : "null");
    spdp_ctx* c = a;
    if (a->K != b->K || a->V != b->V) return fail(c, SPDP_EINVAL, "spdp_topic_hellinger: K or V differ");
    if (a->cfg.device != b->cfg.device) return fail(c, SPDP_EINVAL, "spdp_topic_hellinger: contexts on different devices");
    if (!dist && !perm) return SPDP_OK;
    const int K = a->K, V = a->V;
    CU(cudaStreamSynchronize(b->stream));
    TempBuf<double> sa((size_t)K * V), sb((size_t)K * V), dd((size_t)K * K);
    if (!sa.p || !sb.p || !dd.p) return fail(c, SPDP_ENOMEM, "spdp_topic_hellinger buffers");
    const int grid = (int)std::min<size_t>(((size_t)K * V + 255) / 256, 148u * 16u);
    sqrt_phi0_kernel<<<grid, 256, 0, c->stream>>>(a->d_Q, a->d_T, a->cfg.beta, (double)V * a->cfg.beta, V, K, a->Kp, sa.p);
    sqrt_phi0_kernel<<<grid, 256, 0, c->stream>>>(b->d_Q, b->d_T, b->cfg.beta, (double)V * b->cfg.beta, V, K, b->Kp, sb.p);
    hellinger_kernel<<<dim3((K + 31) / 32, (K + 31) / 32), 256, 0, c->stream>>>(sa.p, sb.p, K, V, dd.p);
    c->launches += 3;
    if ((s = check_launch(c, "hellinger kernels"))) return s;
    std::vector<double> h((size_t)K * K);
    CU(cudaMemcpyAsync(h.data(), dd.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    if ((s = sync(c, "spdp_topic_hellinger"))) return s;
    if (dist) std::memcpy(dist, h.data(), sizeof(double) * h.size());
    if (perm) {
        // greedy minimum-distance matching (reading c22): ascending (distance, k, k'), both ends free
        std::vector<uint32_t> order((size_t)K * K);
        for (size_t j = 0; j < order.size(); ++j) order[j] = (uint32_t)j;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return h[x] < h[y]; });
        std::vector<char> ur((size_t)K, 0), uc((size_t)K, 0);
        for (uint32_t j : order) {
            const int k = (int)(j / (uint32_t)K), kp = (int)(j % (uint32_t)K);
            if (!ur[(size_t)k] && !uc[(size_t)kp]) { ur[(size_t)k] = uc[(size_t)kp] = 1; perm[k] = kp; }
        }
    }
    return SPDP_OK;
}

spdp_status spdp_debug_chain(spdp_ctx* c, int32_t nsweeps, int32_t tbase, int64_t* codes) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (!c->seq) return fail(c, SPDP_ESTATE, "spdp_debug_chain needs num_waves = 0 (sequential test mode)");
    if (nsweeps < 0 || tbase < 2 || (nsweeps > 0 && !codes)) return fail(c, SPDP_EINVAL, "bad debug_chain arguments");
    // the code must fit: N log2 K + I V K log2 tbase < 62 bits
    const double bits = (double)c->N * std::log2((double)std::max(c->K, 1)) +
                        (double)c->I * c->V * c->K * std::log2((double)tbase);
    if (bits >= 62.0) return fail(c, SPDP_EINVAL, "corpus too large for a 64-bit state code (%.1f bits)", bits);
    if (nsweeps == 0) return SPDP_OK;
    TempBuf<int64_t> d((size_t)nsweeps);
    if (!d.p) return fail(c, SPDP_ENOMEM, "debug_chain buffer");
    s = seq_sweeps(c, nsweeps, d.p, tbase);
    if (!s) {
        CU(cudaMemcpyAsync(codes, d.p, sizeof(int64_t) * (size_t)nsweeps, cudaMemcpyDeviceToHost, c->stream));
        s = sync(c, "debug_chain");
    }
    return s;
}

spdp_status spdp_debug_ratio_table(spdp_ctx* c, int32_t group, int32_t mmax, float* out) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (group < 0 || group >= c->I || mmax < 0 || mmax > c->mmax || !out)
        return fail(c, SPDP_EINVAL, "bad debug_ratio_table arguments (group %d, mmax %d > M_max %d?)", group, mmax, c->mmax);
    const size_t cnt = (size_t)(mmax + 1) * (size_t)(mmax + 2) / 2;
    CU(cudaMemcpyAsync(out, c->d_tab + c->tab_off_host[(size_t)group], sizeof(float2) * cnt, cudaMemcpyDeviceToHost,
                       c->stream));
    return sync(c, "debug_ratio_table");
}

spdp_status spdp_debug_probs(spdp_ctx* c, int64_t n, const int64_t* tok_ids, double* probs, int32_t* info) {
    spdp_status s = guard(c, true);
    if (s) return s;
    if (c->sparse) return fail(c, SPDP_ESTATE, "not available with a transformation matrix in this version");
    if (n < 0 || (n > 0 && (!tok_ids || !probs))) return fail(c, SPDP_EINVAL, "bad debug_probs arguments");
    if (n == 0) return SPDP_OK;
    const int I = c->I, K = c->K;
    std::vector<uint32_t> tdoc((size_t)n), tid((size_t)n), cs((size_t)n + 1), ce((size_t)n), seg((size_t)n);
    std::vector<uint16_t> zr((size_t)n);
    if ((s = ensure_host_plan(c))) return s;
    std::vector<uint16_t> allzr((size_t)c->Nloc);
    CU(cudaMemcpyAsync(allzr.data(), c->d_zr, sizeof(uint16_t) * allzr.size(), cudaMemcpyDeviceToHost, c->stream));
    if ((s = sync(c, "debug zr"))) return s;
    for (int64_t j = 0; j < n; ++j) {
        const int64_t p = tok_ids[j];
        if (p < 0 || p >= c->N || c->pos_of_tok[(size_t)p] < 0) return fail(c, SPDP_EINVAL, "token %lld is not on this rank", (long long)p);
        tdoc[(size_t)j] = (uint32_t)c->local_of_doc[(size_t)c->doc[(size_t)p]];
        tid[(size_t)j] = (uint32_t)p;
        zr[(size_t)j] = allzr[(size_t)c->pos_of_tok[(size_t)p]];
        cs[(size_t)j] = (uint32_t)j;
        ce[(size_t)j] = (uint32_t)j + 1;
        seg[(size_t)j] = (uint32_t)c->word[(size_t)p] * (uint32_t)I + (uint32_t)c->group[(size_t)p];
    }
    cs[(size_t)n] = (uint32_t)n;
    uint32_t *d_doc = nullptr, *d_id = nullptr, *d_cs = nullptr, *d_ce = nullptr, *d_seg = nullptr;
    uint16_t* d_zr = nullptr;
    double* d_w = nullptr;
    int32_t* d_info = nullptr;
    ALLOC(d_doc, n); ALLOC(d_id, n); ALLOC(d_cs, n + 1); ALLOC(d_ce, n); ALLOC(d_seg, n); ALLOC(d_zr, n);
    ALLOC(d_w, (size_t)n * 2 * K); ALLOC(d_info, (size_t)n * 4);
    CU(cudaMemcpyAsync(d_doc, tdoc.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(d_id, tid.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(d_cs, cs.data(), 4 * ((size_t)n + 1), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(d_ce, ce.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(d_seg, seg.data(), 4 * (size_t)n, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(d_zr, zr.data(), 2 * (size_t)n, cudaMemcpyHostToDevice, c->stream));
    SweepArgs a = base_args(c);
    a.chunk_ft = 0;                                   // one-token "chunks" of this call: factors computed in place
    a.tok_doc = d_doc; a.tok_id = d_id; a.zr = d_zr; a.zr_next = nullptr;
    a.chunk_start = d_cs; a.chunk_end = d_ce; a.chunk_seg = d_seg; a.nchunks = (int)n;
    a.work = c->d_work + c->W + 1;
    CU(cudaMemsetAsync(a.work, 0, sizeof(uint32_t), c->stream));
    a.dbg_w = d_w; a.dbg_info = d_info;
    launch_sample(c, a, true);
    normalise_rows_kernel<<<(int)((n + 127) / 128), 128, 0, c->stream>>>(d_w, (int)n, 2 * K);
    if ((s = check_launch(c, "debug sample_kernel"))) return s;
    CU(cudaMemcpyAsync(probs, d_w, sizeof(double) * (size_t)n * 2 * K, cudaMemcpyDeviceToHost, c->stream));
    if (info) CU(cudaMemcpyAsync(info, d_info, sizeof(int32_t) * (size_t)n * 4, cudaMemcpyDeviceToHost, c->stream));
    s = sync(c, "debug_probs");
    for (void* p : {(void*)d_doc, (void*)d_id, (void*)d_cs, (void*)d_ce, (void*)d_seg, (void*)d_zr, (void*)d_w, (void*)d_info}) {
        cudaFree(p);
        c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), p), c->allocs.end());
    }
    // keep-rule tokens: the conditional is the point mass on (k0, r=1)
    if (!s && info)
        for (int64_t j = 0; j < n; ++j)
            if (info[4 * j + 1]) {
                for (int q = 0; q < 2 * K; ++q) probs[(size_t)j * 2 * K + q] = 0.0;
                probs[(size_t)j * 2 * K + 2 * (zr[(size_t)j] & 0x7FFF)] = 1.0;
            }
    return s;
}

spdp_status spdp_nccl_unique_id(void* out) {
    if (!out) return SPDP_EINVAL;
    void* lib = open_nccl();
    if (!lib) return SPDP_ENCCL;
    auto fn = (int (*)(NcclUid*))dlsym(lib, "ncclGetUniqueId");
    if (!fn) return SPDP_ENCCL;
    NcclUid uid;
    if (fn(&uid) != 0) return SPDP_ENCCL;
    std::memcpy(out, uid.b, 128);
    return SPDP_OK;
}

spdp_status spdp_profile(spdp_ctx* c, int32_t enable) {
    spdp_status s = guard(c, false);
    if (s) return s;
    c->profiling = enable != 0;
    for (double& v : c->acc) v = 0.0;
    c->launches = 0;
    if (c->profiling && c->loaded) return ensure_events(c);
    return SPDP_OK;
}

spdp_status spdp_timings(spdp_ctx* c, double* out) {
    if (!c || !out) return SPDP_EINVAL;
    for (int j = 0; j < 10; ++j) out[j] = c->acc[j];
    out[6] = (double)c->launches;
    return SPDP_OK;
}

spdp_status spdp_stats(spdp_ctx* c, int64_t* out) {
    spdp_status s = guard(c, true);
    if (s) return s;
    unsigned long long st[8] = {0};
    CU(cudaMemcpyAsync(st, c->d_stats, sizeof st, cudaMemcpyDeviceToHost, c->stream));
    if ((s = sync(c, "stats"))) return s;
    out[0] = (int64_t)st[0]; out[1] = (int64_t)st[1]; out[2] = (int64_t)st[2];
    out[3] = c->sweeps_done; out[4] = c->Nloc; out[5] = c->Dloc; out[6] = c->mmax; out[7] = (int64_t)(size_t)c->nchunks;
    out[8] = c->LPT; out[9] = c->KPL; out[10] = c->chunk_tokens; out[11] = c->sample_grid;
    out[12] = c->token_kernel ? 1 : 0; out[13] = c->P; out[14] = c->row_elem; out[15] = c->async ? 1 : 0;
    out[16] = c->sprows ? 1 : 0; out[17] = c->sprows ? c->sp_lpt : 0; out[18] = 0; out[19] = 0;
    if (c->sprows && c->Dloc > 0) {   // entries of the last rebuild (sum of nonzero doc-topic counts)
        std::vector<uint2> di((size_t)c->Dloc);
        CU(cudaMemcpyAsync(di.data(), c->d_dinfo, sizeof(uint2) * di.size(), cudaMemcpyDeviceToHost, c->stream));
        if ((s = sync(c, "stats entries"))) return s;
        int64_t tot = 0, per_tok = 0;
        for (size_t j = 0; j < di.size(); ++j) {
            tot += di[j].y;
            per_tok += (int64_t)di[j].y * c->doclen[(size_t)c->global_of_local[j]];   // entries read per sweep
        }
        out[18] = tot;
        out[19] = per_tok;
    }
    return SPDP_OK;
}

void spdp_destroy(spdp_ctx* c) {
    if (!c) return;
    if (c->cfg.device >= 0) cudaSetDevice(c->cfg.device);
    // every stream that may still use the buffers drains before any of them is freed
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->side_stream) cudaStreamSynchronize(c->side_stream);
    if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
    if (c->d2h_stream) { cudaStreamSynchronize(c->d2h_stream); cudaStreamDestroy(c->d2h_stream); }
    if (c->zr_ready) cudaEventDestroy(c->zr_ready);
    if (c->zr_copied) cudaEventDestroy(c->zr_copied);
    for (void* p : c->allocs) cudaFree(p);
    if (c->stream) {
        for (void* p : c->pooled) cudaFreeAsync(p, c->stream);
        cudaStreamSynchronize(c->stream);
    }
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    if (c->h_zr_canon) cudaFreeHost(c->h_zr_canon);
    if (c->comm && c->nccl.CommDestroy) c->nccl.CommDestroy(c->comm);
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
    if (c->comm_stream) { cudaStreamSynchronize(c->comm_stream); cudaStreamDestroy(c->comm_stream); }
    for (cudaEvent_t e : c->part_ev) cudaEventDestroy(e);
    if (c->comm_done) cudaEventDestroy(c->comm_done);
    if (c->side_stream) { cudaStreamSynchronize(c->side_stream); cudaStreamDestroy(c->side_stream); }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    if (c->pool) cudaMemPoolDestroy(c->pool);
    delete c;
}

}  // extern "C"

namespace {
// debug_checks: n and m recounted from z equal the maintained
// tables (m gathered over the ranks with an NCCL sum; an external exchange cannot be
// gathered here, so there m is checked through its sums only); 0 <= t <= m and
// t > 0 iff m > 0; Q = sum_i t (identity P); M = sum_w m, Tt = sum_w t, T = sum_w Q;
// sum m = N.
spdp_status debug_verify(spdp_ctx* c) {
    const int I = c->I, V = c->V, K = c->K, Kp = c->Kp;
    std::vector<uint16_t> zr((size_t)c->Nloc);
    std::vector<float> nf;
    std::vector<int32_t> n((size_t)c->Dloc * Kp), m(c->cells), t(c->cells), Q((size_t)V * Kp);
    std::vector<int32_t> M((size_t)I * Kp), Tt((size_t)I * Kp), T((size_t)Kp);
    {
        spdp_status s0 = ensure_host_plan(c);
        if (s0) return s0;
    }
    CU(cudaMemcpy(zr.data(), c->d_zr, 2 * zr.size(), cudaMemcpyDeviceToHost));
    {
        spdp_status s0 = read_rows(c, nf);
        if (s0) return s0;
    }
    for (int32_t j = 0; j < c->Dloc; ++j)
        for (int k = 0; k < Kp; ++k) n[(size_t)j * Kp + k] = (int32_t)nf[(size_t)j * c->Kn + c->sigma[(size_t)k]];
    {   // positions of the rows that hold no topic (padding) must stay zero
        std::vector<char> used((size_t)c->Kn, 0);
        for (int k = 0; k < K; ++k) used[(size_t)c->sigma[(size_t)k]] = 1;
        for (int32_t j = 0; j < c->Dloc; ++j)
            for (int x = 0; x < c->Kn; ++x)
                if (!used[(size_t)x] && nf[(size_t)j * c->Kn + x] != 0.f)
                    return fail(c, SPDP_EINTEGRITY, "doc-topic row %d holds %g at padding position %d", (int)j,
                                (double)nf[(size_t)j * c->Kn + x], x);
    }
    CU(cudaMemcpy(m.data(), c->d_m, 4 * m.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(t.data(), c->d_t, 4 * t.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(Q.data(), c->d_Q, 4 * Q.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(M.data(), c->d_M, 4 * M.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(Tt.data(), c->d_Tt, 4 * Tt.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(T.data(), c->d_T, 4 * T.size(), cudaMemcpyDeviceToHost));
    std::vector<int32_t> n2((size_t)c->Dloc * Kp, 0), m2(c->cells, 0);
    for (int64_t q = 0; q < c->Nloc; ++q) {
        const uint32_t p = c->sorted_tok[(size_t)q];
        const int k = zr[(size_t)q] & 0x7FFF;
        if (k >= K) return fail(c, SPDP_EINTEGRITY, "topic %d out of range at token %u", k, p);
        n2[(size_t)c->local_of_doc[(size_t)c->doc[p]] * Kp + k]++;
        m2[((size_t)c->word[p] * I + (size_t)c->group[p]) * Kp + k]++;
    }
    if (n2 != n) return fail(c, SPDP_EINTEGRITY, "doc-topic counts differ from a recount of z");
    bool m_checked = c->G == 1;
    if (c->G > 1 && c->comm) {   // every rank's recount, summed
        TempBuf<int32_t> tb(c->cells);
        if (!tb.p) return fail(c, SPDP_ENOMEM, "debug_verify buffer");
        CU(cudaMemcpyAsync(tb.p, m2.data(), 4 * m2.size(), cudaMemcpyHostToDevice, c->stream));
        spdp_status s0 = nccl_check(c, c->nccl.AllReduce(tb.p, tb.p, c->cells, kNcclInt32, kNcclSum, c->comm, c->stream),
                                    "allreduce m recount");
        if (s0) return s0;
        CU(cudaMemcpyAsync(m2.data(), tb.p, 4 * m2.size(), cudaMemcpyDeviceToHost, c->stream));
        if ((s0 = sync(c, "debug_verify"))) return s0;
        m_checked = true;
    }
    if (m_checked && m2 != m) {
        for (size_t j = 0; j < c->cells; ++j)
            if (m2[j] != m[j]) {
                const size_t k = j % Kp, wi = j / Kp;
                return fail(c, SPDP_EINTEGRITY, "customer count m differs from a recount of z at (i=%d, w=%d, k=%d): %d vs %d",
                            (int)(wi % I), (int)(wi / I), (int)k, m[j], m2[j]);
            }
    }
    std::vector<int64_t> M2((size_t)I * Kp, 0), Tt2((size_t)I * Kp, 0), T2((size_t)Kp, 0);
    int64_t sm = 0;
    for (int w = 0; w < V; ++w)
        for (int k = 0; k < Kp; ++k) {
            int64_t q = 0;
            for (int i = 0; i < I; ++i) {
                const size_t cell = ((size_t)w * I + i) * Kp + k;
                if (k >= K) {
                    if (m[cell] || t[cell]) return fail(c, SPDP_EINTEGRITY, "nonzero padding cell at (i=%d, w=%d)", i, w);
                    continue;
                }
                if (t[cell] < 0 || t[cell] > m[cell] || ((t[cell] > 0) != (m[cell] > 0)))
                    return fail(c, SPDP_EINTEGRITY, "t out of [min(1,m), m] at (i=%d, w=%d, k=%d)", i, w, k);
                q += t[cell];
                sm += m[cell];
                M2[(size_t)i * Kp + k] += m[cell];
                Tt2[(size_t)i * Kp + k] += t[cell];
            }
            if (!c->sparse && q != Q[(size_t)w * Kp + k]) return fail(c, SPDP_EINTEGRITY, "Q != sum_i t at (w=%d, k=%d)", w, k);
            T2[(size_t)k] += Q[(size_t)w * Kp + k];
        }
    for (int i = 0; i < I; ++i)
        for (int k = 0; k < K; ++k) {
            const size_t j = (size_t)i * Kp + k;
            if (M2[j] != M[j]) return fail(c, SPDP_EINTEGRITY, "M != sum_w m at (i=%d, k=%d)", i, k);
            if (Tt2[j] != Tt[j]) return fail(c, SPDP_EINTEGRITY, "Tt != sum_w t at (i=%d, k=%d)", i, k);
        }
    for (int k = 0; k < K; ++k)
        if (T2[(size_t)k] != T[(size_t)k]) return fail(c, SPDP_EINTEGRITY, "T != sum_w Q at k=%d", k);
    if (sm != c->N) return fail(c, SPDP_EINTEGRITY, "sum m = %lld != N", (long long)sm);
    return SPDP_OK;
}
}  // namespace
