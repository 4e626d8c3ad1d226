/*
 * spdp.h — C ABI of the B200-native SPDP Gibbs sweep (libspdp.so).
 *
 * The library samples the collapsed blocked-Gibbs chain of the Shadow
 * Poisson–Dirichlet Process topic model — with identity transformation
 * matrices by default (§3.4; sparse P^i through
 * spdp_set_transform, NEXT-4), i.e. Algorithm 1 "SPDP Full Gibbs
 * Sampling" with the conditionals of
 * Eq. SPDP-sampling-w-z-r0 and
 * Eq. SPDP-sampling-w-z-r1, parallelised the way §3.3
 * describes ("minimum local copy", PAPER.md:2289-2299
 * word-order rearrangement, PAPER.md:2370-2386 document division over
 * devices, Alg.3/Alg.4) under the deterministic
 * wave-snapshot reading of DESIGN.md §3 (reading c13).
 *
 * Problem statement (§2.3.4):
 * N tokens, each a triple (group i, document d, word w); K topics; the
 * Dirichlet alpha on document-topic proportions; the Dirichlet beta on the
 * shared base phi0 (printed gamma_v in Eq. r1); the PDP discount a_i and
 * concentration b_i per group.
 *
 * Conventions
 *   - Every function returns spdp_status (0 = SPDP_OK).  Nothing aborts; the
 *     message of the last failing call is spdp_last_error(ctx).
 *   - All pointer arguments are HOST pointers owned by the caller.  Inputs are
 *     copied during the call; outputs are caller-allocated and written before
 *     the call returns.  The context owns all device memory and the NCCL
 *     communicator.
 *   - Call order: spdp_create -> [spdp_set_transform] -> spdp_load_corpus ->
 *     {spdp_sweep (or spdp_sweep_local / spdp_sweep_merge), spdp_counts,
 *     spdp_zr, spdp_loglik, spdp_set_state, spdp_topics, spdp_heldout,
 *     spdp_debug_probs, ...}* -> spdp_destroy.  Anything else returns
 *     SPDP_ESTATE.
 *   - A context is not thread-safe.  Calls are synchronous with respect to
 *     the host (they return after the work on the context's stream is done).
 *   - Determinism: outputs are bit-identical for identical (config, corpus,
 *     initial state, number of sweeps, world_size).  Different world sizes give
 *     different (equally valid) chains; the oracle reproduces each.
 *   - Multi-GPU: one process per GPU.  Every rank passes the whole corpus and
 *     keeps its document shard.  spdp_sweep, spdp_counts and spdp_loglik are
 *     collective over the world.
 */
#ifndef SPDP_H
#define SPDP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPDP_OK = 0,
    SPDP_EINVAL = -1,      /* invalid argument (ranges, shapes, hyper-parameters) */
    SPDP_ENOMEM = -2,      /* host or device allocation failed */
    SPDP_ECUDA = -3,       /* CUDA runtime error or no device; context is poisoned */
    SPDP_ENCCL = -4,       /* NCCL unavailable or failed */
    SPDP_ESTATE = -5,      /* wrong call order, or context poisoned by an earlier fault */
    SPDP_ETABLE = -6,      /* Stirling-ratio table would exceed its size limit */
    SPDP_EINTEGRITY = -7   /* debug_checks found a violated count invariant */
} spdp_status;

typedef struct spdp_ctx spdp_ctx;

/* How the per-sweep count deltas of a multi-GPU run are summed across ranks. */
enum {
    SPDP_EXCHANGE_NCCL = 0,      /* spdp_sweep calls ncclAllReduce itself (needs nccl_unique_id) */
    SPDP_EXCHANGE_EXTERNAL = 1   /* caller sums the buffer of spdp_exchange_buffer between
                                    spdp_sweep_local and spdp_sweep_merge */
};

/* How a sweep updates the counts (DESIGN.md §3 reading c13, §11). */
enum {
    SPDP_UPDATE_WAVE = 0,   /* deterministic wave snapshots: every token of a wave decides against the
                               wave-start counts, the wave's deltas are applied after it (default) */
    SPDP_UPDATE_ASYNC = 1   /* the paper's in-GPU scheme (Alg.4 PAPER.md:2973-3012;
                               SURVEY.md §8(f) NEXT-2): live counts copied per work unit, updates applied
                               to the global counts at once with atomics, t corrected into its valid range
                               and the sums recomputed at the end of the sweep.  Nondeterministic;
                               needs num_waves == 1 */
};

typedef struct {
    uint32_t struct_size;          /* = sizeof(spdp_config); ABI versioning */
    int32_t num_groups;            /* I >= 1 */
    int32_t vocab_size;            /* V >= 1 */
    int32_t num_topics;            /* K, 1 <= K <= 1024 */
    double alpha;                  /* symmetric Dirichlet on theta, > 0 (paper 0.1) */
    const double* alpha_ik;        /* optional [I*K] asymmetric alpha_{ik} (row-major i,k); NULL -> alpha */
    double beta;                   /* symmetric Dirichlet on phi0 (paper gamma_v = 0.1), > 0 */
    const double* discount;        /* [I] a_i in [0, 1)      (paper 0.7) */
    const double* concentration;   /* [I] b_i > 0            (paper 100) */
    uint64_t seed;                 /* Philox4x32-10 key (low word, high word) */
    int32_t num_waves;             /* W >= 1: token of in-document position l is in wave l mod W;
                                      0: exact sequential sampler (test mode, world_size 1; spdp_debug_chain) */
    int32_t device;                /* CUDA ordinal used by this rank */
    int32_t rank, world_size;      /* 0, 1 for a single GPU */
    int32_t exchange;              /* SPDP_EXCHANGE_* (ignored when world_size == 1) */
    const void* nccl_unique_id;    /* 128-byte ncclUniqueId (same on every rank) for SPDP_EXCHANGE_NCCL */
    void* stream;                  /* cudaStream_t to order work on; NULL -> a stream owned by the context */
    int32_t debug_checks;          /* 1 = verify count invariants after every sweep (slow) */
    int32_t update_mode;           /* SPDP_UPDATE_* */
    int32_t merge_every;           /* world_size > 1: exchange the ranks' count changes after every
                                      merge_every waves (bounded staleness, SURVEY.md §8(f) NEXT-3;
                                      PAPER.md:2427-2434); 0 = once per sweep (Alg.3) */
} spdp_config;

/* Create a context on cfg->device.  Validates the hyper-parameters
 * (SPDP_EINVAL), selects the device (SPDP_ECUDA when absent) and, for
 * world_size > 1 with SPDP_EXCHANGE_NCCL, joins the NCCL communicator
 * (SPDP_ENCCL).  *out receives the context even when the call fails (so that
 * spdp_last_error can explain the failure); release it with spdp_destroy. */
spdp_status spdp_create(const spdp_config* cfg, spdp_ctx** out);

/* Load the corpus and the initial state.  Token p = (group[p], doc[p],
 * word[p]), p in [0, num_tokens), is the canonical token id used by the RNG;
 * its in-document position l is its rank among the tokens of doc[p] in
 * canonical order.  Doc ids lie in [0, num_docs); all tokens of a document
 * share one group.
 *   z_init [N] in [0, K) or NULL: default z_p = floor(x0 * K / 2^32) with
 *          x = Philox(seed; counter (p, 0xFFFFFFFF, 0, 0)).
 *   r_init [N] in {0, 1} or NULL: default r_p = 1 for the first token of each
 *          (i, k, w) cell in canonical order (t = min(1, m)); table counts are
 *          t_{ikw} = sum of r over the cell and must satisfy 1 <= t <= m on
 *          every occupied cell ("Initialize counting
 *          variables ... from z").
 * Documents are divided over the world by a seeded permutation and a
 * token-balanced contiguous split.
 * Errors: SPDP_EINVAL (ids out of range, doc spanning groups, bad z/r/t),
 * SPDP_ENOMEM, SPDP_ETABLE, SPDP_ECUDA.  May be called once per context. */
spdp_status spdp_load_corpus(spdp_ctx* ctx, int64_t num_tokens, int32_t num_docs,
                             const int32_t* group, const int32_t* doc, const int32_t* word,
                             const int32_t* z_init, const uint8_t* r_init);

/* Replace the sampler state: z [N] and r [N] as in spdp_load_corpus, and
 * optionally the table counts tables [I*V*K] (row-major i, w, k) which then
 * override sum-of-r (checkpoint / resume; parity tests).  Every rank passes
 * the whole arrays.  The sweep counter is left unchanged. */
spdp_status spdp_set_state(spdp_ctx* ctx, const int32_t* z, const uint8_t* r, const int32_t* tables);

/* Run num_sweeps >= 0 sweeps.  One sweep visits every token once: for each
 * wave in order, every token of the wave removes itself from the wave-start
 * counts (Alg.1 lines 3-10), weighs the 2K (topic, table-indicator) slots
 * (Eqs. r0/r1) and draws one slot with the Philox uniform of (token, sweep);
 * the wave's count deltas are then applied and t clamped into
 * [min(1, m), m].  With world_size > 1 the ranks' net
 * count changes are all-reduced after the last wave and merged (Alg.3
 * PAPER.md:2960-2965).  Collective.  SPDP_ESTATE for
 * SPDP_EXCHANGE_EXTERNAL contexts (use the split calls below). */
spdp_status spdp_sweep(spdp_ctx* ctx, int32_t num_sweeps);
/* spdp_sweep without the final wait: the sweeps are queued on the context's
 * stream and the call returns (the host-synchronous contract of the other
 * calls is kept by them: spdp_counts, spdp_loglik, spdp_stats, ... order
 * themselves after the queued work; spdp_zr_async / spdp_zr8_async queue
 * their copy behind it).  Device faults surface at the next synchronising
 * call.  With debug_checks it is spdp_sweep. */
spdp_status spdp_sweep_async(spdp_ctx* ctx, int32_t num_sweeps);

/* Split sweep for SPDP_EXCHANGE_EXTERNAL: spdp_sweep_local runs every wave
 * (with merge_every, the next exchange block of waves; see spdp_exchange_blocks)
 * on this rank and leaves the rank's net (customer, table) count change of
 * every cell since the sweep start in the device buffer returned by
 * spdp_exchange_buffer (*count elements of *elem_bytes bytes, device pointer
 * owned by the context).  Each element packs both changes of one cell as
 * dm * 2^B + dt in two's complement, B = 16 for 4-byte elements (chosen when
 * max_{i,w} count(i,w) < 2^15, which bounds |sum over ranks| of either half)
 * and B = 32 for 8-byte elements, so the plain integer sum of the packed
 * elements over ranks (wrapping) is the packed sum of dm and dt.  The caller
 * replaces the buffer's content by that element-wise sum over ranks, then
 * calls spdp_sweep_merge (Alg.3: rows = sweep-start
 * state + summed changes, t clamped, Q and the sums recomputed).  With a
 * transformation matrix the buffer is int32 m changes (cells) followed by
 * the source changes q (E x Kp), see spdp_set_transform. */
spdp_status spdp_sweep_local(spdp_ctx* ctx);
/* Exchange blocks per sweep (merge_every): the caller repeats
 * {spdp_sweep_local, sum over ranks, spdp_sweep_merge} *nblocks times per
 * sweep; each spdp_sweep_local runs the next merge_every waves. */
spdp_status spdp_exchange_blocks(spdp_ctx* ctx, int32_t* nblocks);
spdp_status spdp_exchange_buffer(spdp_ctx* ctx, void** device_ptr, int64_t* count, int32_t* elem_bytes);
spdp_status spdp_sweep_merge(spdp_ctx* ctx);
/* Copy the exchange buffer to (to_device = 0) or from (to_device = 1) the
 * caller's host array of *count elements of *elem_bytes bytes
 * (e.g. for a host-side all-reduce). */
spdp_status spdp_exchange_copy(spdp_ctx* ctx, void* host, int32_t to_device);

/* Read the state.  Every output is optional (NULL = skip):
 *   z [N] int32, r [N] uint8: canonical token order; r is the indicator drawn
 *       at the token's last insertion (1 when the keep rule held it).  With
 *       world_size > 1 and SPDP_EXCHANGE_NCCL the values of every rank are
 *       gathered; with SPDP_EXCHANGE_EXTERNAL only this rank's tokens are
 *       written.
 *   doc_topic [D*K] int32 (n_{idk}); same gathering rule as z.
 *   customers [I*V*K] int32 (m_{ikw}, row-major i, w, k), tables [I*V*K] int32
 *       (t_{ikw}), shadow [K*V] int32 (Q_{kw} = sum_i t_{ikw}, row-major k, w):
 *       replicated, identical on every rank after a sweep. */
spdp_status spdp_counts(spdp_ctx* ctx, int32_t* z, uint8_t* r, int32_t* doc_topic,
                        int32_t* customers, int32_t* tables, int32_t* shadow);

/* The assignments packed: zr [N] uint16 = z | r << 15 in canonical token order
 * (2 bytes per token, no host-side unpacking; pass pinned memory for a
 * full-speed copy).  Tokens of other ranks read 0xFFFF with
 * SPDP_EXCHANGE_EXTERNAL; gathered from every rank (collective) with
 * SPDP_EXCHANGE_NCCL.  Caller-owned host buffer. */
spdp_status spdp_zr(spdp_ctx* ctx, uint16_t* zr);
/* spdp_zr without the wait: the canonical-order scatter is queued on the
 * context's stream and the device->host copy on a library-owned copy stream,
 * so the copy overlaps whatever the caller queues next (typically the next
 * spdp_sweep, which does not touch the staging buffer).  The caller's buffer
 * holds the assignments as of this call only after spdp_wait (or
 * spdp_destroy); it must stay allocated until then, and should be pinned
 * (pageable memory makes the copy synchronous).  A later spdp_zr_async,
 * spdp_zr or spdp_counts orders itself after the pending copy on the device.
 * With world_size > 1 and SPDP_EXCHANGE_NCCL this is spdp_zr (collective,
 * blocking).  Errors as spdp_zr. */
spdp_status spdp_zr_async(spdp_ctx* ctx, uint16_t* zr);
/* spdp_zr_async with one byte per token, zr [N] uint8 = z | r << 7 (K <= 128,
 * else SPDP_EINVAL): half the device->host bytes of the step's result.
 * Tokens of other ranks read 0xFF with SPDP_EXCHANGE_EXTERNAL; with
 * SPDP_EXCHANGE_NCCL and world_size > 1 it is collective and blocking. */
spdp_status spdp_zr8_async(spdp_ctx* ctx, uint8_t* zr);
/* Block until every copy queued by spdp_zr_async / spdp_zr8_async has
 * landed (the copies follow their staging on the context's stream, so the
 * work queued before them is done too; work queued after them, e.g. a
 * spdp_sweep_async, may still run).  With no copy pending: until the
 * context's stream is idle.  SPDP_ECUDA on a device fault. */
spdp_status spdp_wait(spdp_ctx* ctx);

/* log_joint = log p(W, Z, T | alpha, beta, a, b) (PAPER.md:1654-1665 summed over
 * the seatings R of each T, Eq. SPDP-table-to-head);
 * perplexity = training perplexity exp(-sum_tok log sum_k theta~_dk phi^i~_kw / N)
 * (PAPER.md:1978-2007 with Eqs.; DESIGN.md readings
 * c16, c17).  Either pointer may be NULL.  Collective. */
spdp_status spdp_loglik(spdp_ctx* ctx, double* log_joint, double* perplexity);

/* ---- Held-out evaluation ---------------------
 *
 * spdp_topics: the topic-word estimates of the current state, computed on
 * the device in fp64 (identity P):
 *   phi0 [K*V] (row-major k, w): phi0~_kw = (beta + Q_kw) / (V beta + T_k)   Eq. P:1753;
 *   phi [I*K*V] (row-major i, k, w): phi~^i_kw = (m_ikw - a_i t_ikw)/(b_i + m_ik.)
 *        + (b_i + a_i t_ik.)/(b_i + m_ik.) phi0~_kw   Eq. P:1754 (reading c16).
 * Either output may be NULL; host buffers owned by the caller.  Not
 * collective: the word-topic state is replicated, so every rank returns the
 * same values after a sweep.  Errors: SPDP_ESTATE before spdp_load_corpus,
 * SPDP_ENOMEM, SPDP_ECUDA. */
spdp_status spdp_topics(spdp_ctx* ctx, double* phi0, double* phi);

/* spdp_heldout: fold-in of held-out documents and the held-out perplexity of
 * PAPER.md:1978-2007 ("test documents are documents held out in each group
 * during training"; 10% per group in §4.1).
 *   Tokens: num_tokens triples (group, doc, word) in canonical order, doc ids
 *   in [0, num_docs), every document inside one group (SPDP_EINVAL otherwise).
 *   Fold-in (reading c21; the paper does not say how theta~ of a
 *   test document is obtained): `iterations` sweeps of collapsed Gibbs over
 *   the held-out topics only, phi~^i frozen, p(z_p = k) ∝ (alpha_ik + n_dk^{-p})
 *   phi~^i_{k w_p}, tokens of a document visited sequentially in canonical
 *   order (documents are independent given phi~: exact, no staleness).
 *   Randomness: Philox4x32-10 with key `seed`, counter (p, iteration, 1, 0)
 *   for held-out token p; iterations are numbered from first_iteration.
 *   z_init [num_tokens] in [0,K), or NULL: z_p = floor(x0 K / 2^32) of counter
 *   (p, 0xFFFFFFFF, 1, 0).  z_out [num_tokens] (optional): topics after the
 *   last iteration.  theta [num_docs*K] (optional): theta~_dk =
 *   (n_dk + alpha_ik) / (L_d + sum_k alpha_ik) (Eq. P:1736-1740).
 *   perplexity (optional): exp(-sum_p log sum_k theta~_dk phi~^i_{k w_p} / num_tokens)
 *   (reading c17).  Host buffers owned by the caller.  Not collective; the
 *   trained state is not modified.  Errors: SPDP_EINVAL, SPDP_ESTATE,
 *   SPDP_ENOMEM, SPDP_ECUDA. */
spdp_status spdp_heldout(spdp_ctx* ctx, int64_t num_tokens, int32_t num_docs, const int32_t* group,
                         const int32_t* doc, const int32_t* word, uint64_t seed, int32_t first_iteration,
                         int32_t iterations, const int32_t* z_init, int32_t* z_out, double* theta,
                         double* perplexity);

/* spdp_topic_hellinger: compare two models' topics (§4.2.6 PAPER.md:4377-4411,
 * "re-ordered to align with the topics"; reading c22).
 * dist [K*K] (optional): dist[k*K + k'] = H(phi0~_a[k], phi0~_b[k']) with
 * H(p, q) = sqrt(1 - sum_w sqrt(p_w q_w)) clamped into [0, 1], fp64.
 * perm [K] (optional): greedy minimum-distance matching (ascending distance,
 * ties by smaller k then k'), perm[k] = matched topic of model b.
 * Both contexts must be loaded, share K and V and live on the same device
 * (SPDP_EINVAL otherwise).  Not collective. */
spdp_status spdp_topic_hellinger(spdp_ctx* a, spdp_ctx* b, double* dist, int32_t* perm);

/* ---- Sparse transformation matrices -------------
 *
 * spdp_set_transform: the full SPDP of PAPER.md:985-1014 — group i's base for
 * topic k is P^i phi0_k, so every table of (i, k, w) has a source word v drawn
 * with probability p_{i,w,v} phi0_{k,v} (Eq. r1 P:1688-1693 carries p_{i,w,v};
 * Alg.1 lines 6-9 and 19-21 remove / add the table's source).  P^i as sparse
 * rows over r = i * V + w: entries [pptr[r], pptr[r+1]) with source word pv[e]
 * in [0, V) and weight pp[e] > 0; every row needs >= 1 entry (<= 32767) and
 * every column of every P^i must sum to 1 (±1e-9; P^i phi0 is a distribution,
 * P:990-993).  Host arrays, copied.  Call after spdp_create and before
 * spdp_load_corpus.  The estimators (spdp_topics, spdp_heldout, the
 * perplexity of spdp_loglik) then use phi~^i with sum_v p_{i,w,v} phi0~_{k,v}
 * (P:1754).  Several ranks exchange the net changes of m and q (the external
 * exchange buffer is int32: cells, then E x Kp source cells); log_joint is
 * then log p(W, Z, T, Q) (the sources' multinomial and p terms added).  This
 * version: SPDP_UPDATE_WAVE; spdp_debug_probs and, with several ranks, the
 * perplexity of spdp_loglik return SPDP_ESTATE.  Readings:
 * DESIGN.md §13 (c24 wave correction of the sources, c25 initial sources,
 * c26 the removed table's source).  Errors: SPDP_EINVAL, SPDP_ESTATE.
 *
 * spdp_sparse_state: q [E*K] int32 (tables of (i, k, w) per source entry, in
 * the caller's entry order, row-major e, k), shadow [K*V] int32
 * (Q_{k,v} = sum_{i,w} q_{i,k,w,v}), src [N] int16 (the source entry, within
 * its row, chosen at each token's last draw; -1 for r = 0 and kept tokens).
 * Any output may be NULL. */
spdp_status spdp_set_transform(spdp_ctx* ctx, const int32_t* pptr, const int32_t* pv, const double* pp);
spdp_status spdp_sparse_state(spdp_ctx* ctx, int32_t* q, int32_t* shadow, int16_t* src);

/* Diagnostics (parity tests): for n local tokens (canonical ids), the
 * normalised 2K-slot conditional (slot 2k = (k, r=1), slot 2k+1 = (k, r=0);
 * Alg.4) that the NEXT sweep would draw from if the
 * current state were its wave-start snapshot, computed by the sweep's own
 * device code.  probs [n*2K] fp64; info [n*4] int32 = {r_rem, keep, z_new,
 * r_new}.  No state change.  SPDP_EINVAL for tokens of other ranks. */
spdp_status spdp_debug_probs(spdp_ctx* ctx, int64_t n, const int64_t* tok_ids, double* probs, int32_t* info);

/* Test mode W = 0 (num_waves = 0): the exact sequential
 * sampler, Algorithm 1 with the keep rule, on the
 * device (one warp, tokens in canonical order, counts updated after every
 * token; no snapshot, no clamp).  spdp_sweep(n) runs n such sweeps in one
 * launch.  spdp_debug_chain runs nsweeps of them and writes, after each, the
 * state code sum_p z_p K^p + K^N * sum_j t_j tbase^j (cells j in (i, w, k)
 * order) to codes [nsweeps] int64 — for exact-enumeration tests on tiny
 * corpora (SPDP_EINVAL unless N log2 K + I V K log2 tbase < 62).
 * SPDP_ESTATE unless the context was created with num_waves = 0. */
spdp_status spdp_debug_chain(spdp_ctx* ctx, int32_t nsweeps, int32_t tbase, int64_t* codes);

/* Diagnostics (parity tests, SURVEY §8(c) "A0/A1 folding" pin): the device
 * Stirling-ratio table of group `group` (one per distinct discount a_i),
 * A0(m,t) = (m-t+1)/(m+1) S^{m+1}_t / S^m_t (Eq. r0) and
 * A1(m,t) = (t+1)/(m+1) S^{m+1}_{t+1} / S^m_t (Eq. r1), with
 * S from the recursion PAPER.md:1454-1455, exactly as the sweep reads it.
 * out [(mmax+1)(mmax+2)/2 * 2] fp32, pairs (A0, A1) at index m(m+1)/2 + t for
 * 0 <= t <= m <= mmax (t = 0 < m is not a state and holds 0).  mmax <= the
 * table's M_max (stats out[6]), else SPDP_EINVAL.  No state change. */
spdp_status spdp_debug_ratio_table(spdp_ctx* ctx, int32_t group, int32_t mmax, float* out);

/* Counters of the last sweep on this rank: out[0] keeps, out[1] moved
 * tokens, out[2] clamped cells, out[3] sweeps done, out[4] local tokens,
 * out[5] local docs, out[6] M_max (largest count(i,w)), out[7] chunks,
 * out[8] lanes per token, out[9] topics per lane, out[10] tokens per chunk,
 * out[11] resident sample-kernel blocks (persistent grid), out[12] 1 if the
 * token kernel samples (K <= 64), out[13] word-range parts of the sweep
 * (exchange pipelining), out[14] bytes per doc-topic count (4 fp32, 2 uint16, 1 uint8), out[15] 1
 * for SPDP_UPDATE_ASYNC, out[16] 1 if the sweep samples from sparse doc-topic rows, out[17] their
 * lanes per token, out[18] their entries (nonzero doc-topic counts of this rank), out[19] the entries
 * one sweep reads (sum over documents of length x entries).
 * out has 20 slots. */
spdp_status spdp_stats(spdp_ctx* ctx, int64_t* out);

/* Phase timing with CUDA events recorded on the context's stream around each
 * launch of the sweep (enable = 1 resets the accumulators and starts;
 * 0 stops).  spdp_timings fills out[10] with totals since the reset:
 * out[0] sample-kernel ms, out[1] token-apply / doc-recount ms, out[2]
 * row-merge ms, out[3] exchange ms (all-reduce + merge), out[4] whole-sweep
 * ms, out[5] sample-kernel launches, out[6] kernel launches of all kinds,
 * out[7] sweeps timed, out[8] fold-in kernel ms (spdp_heldout), out[9]
 * fold-in token-iterations. */
spdp_status spdp_profile(spdp_ctx* ctx, int32_t enable);
spdp_status spdp_timings(spdp_ctx* ctx, double* out);

/* Document -> rank assignment used by spdp_load_corpus (host only; no
 * device needed): shard_of_doc [num_docs]. */
spdp_status spdp_partition(uint64_t seed, int32_t world_size, int64_t num_tokens, int32_t num_docs,
                           const int32_t* doc, int32_t* shard_of_doc);

/* Fill out[128] with a fresh ncclUniqueId (rank 0 calls this and broadcasts
 * the bytes, e.g. with torch.distributed).  SPDP_ENCCL if NCCL is absent. */
spdp_status spdp_nccl_unique_id(void* out);

void spdp_destroy(spdp_ctx* ctx);                  /* NULL-safe; frees device memory and the communicator */
const char* spdp_last_error(const spdp_ctx* ctx);  /* message of the last failing call ("" if none) */
const char* spdp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPDP_H */
