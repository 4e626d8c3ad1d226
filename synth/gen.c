/*
 * synth/gen.c — seeded synthetic corpus generator (INPUT GENERATION ONLY).
 *
 * Shared by the oracle tests, the CUDA parity tests and bench.py.  It holds
 * NONE of the sampler's arithmetic: it only draws a corpus from the SPDP
 * generative process with identity transformation matrices, so that the
 * inputs have the shape of the paper's multi-group document collections.
 *
 *   PAPER.md:1001-1014 (§2.3.4, SPDP generative process):
 *       phi0_k ~ Dir(beta)            theta_{i,d} ~ Dir(alpha)
 *       phi^i_k ~ PDP(b, a, P^i phi0_k)   (P^i = I)
 *       z ~ theta_{i,d},  w ~ phi^i_z
 *   PAPER.md:1330-1335 (§2.4.3, Chinese-restaurant seating rule):
 *       new table with prob (b + a*T)/(b + N), dish ~ H;
 *       otherwise join dish j with prob (n_j - a*t_j)/(b + N).
 *
 * Canonical token order: group-major, then document, then in-document
 * position.  Document ids are global: doc = group*docs_per_group + d.
 *
 * Streams (independent xoshiro256** generators seeded by splitmix64 of
 * (seed, stream)):  0 = document lengths, 1 = phi0, 2 = theta and z,
 * 3 = restaurant seating / words.
 *
 * per_unit != 0 (the ~200 M-token C5): one generator per unit instead — per
 * document for its length and for theta_d, z (streams 0, 2), per topic for
 * phi0_k (stream 1), per restaurant (group, topic) for its words (stream 3) —
 * seeded by (seed, stream, unit), so the units are drawn in parallel (OpenMP)
 * and the corpus does not depend on the thread count.  Same generative
 * process, a different (equally distributed) draw than per_unit = 0.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t s[4]; } xo_t;

static uint64_t splitmix64(uint64_t *x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static void xo_seed(xo_t *g, uint64_t seed, uint64_t stream) {
    uint64_t x = seed * 0x2545F4914F6CDD1Dull + stream * 0x9E3779B97F4A7C15ull + 0x1234567ull;
    for (int i = 0; i < 4; i++) g->s[i] = splitmix64(&x);
}
static void xo_seed_unit(xo_t *g, uint64_t seed, uint64_t stream, uint64_t unit) {
    uint64_t x = seed * 0x2545F4914F6CDD1Dull + stream * 0x9E3779B97F4A7C15ull + 0x1234567ull;
    x = splitmix64(&x) ^ (unit * 0xD6E8FEB86659FD93ull);
    for (int i = 0; i < 4; i++) g->s[i] = splitmix64(&x);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t xo_next(xo_t *g) {
    uint64_t *s = g->s;
    uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
    return r;
}
/* uniform in (0,1) */
static inline double xo_unif(xo_t *g) { return ((xo_next(g) >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
static inline uint64_t xo_below(xo_t *g, uint64_t n) { return (uint64_t)(xo_unif(g) * (double)n) % n; }

static double xo_normal(xo_t *g) {
    double u1 = xo_unif(g), u2 = xo_unif(g);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
/* Marsaglia–Tsang gamma(shape, 1); shape < 1 via the boost G(s)=G(s+1)U^{1/s}. */
static double xo_gamma(xo_t *g, double shape) {
    if (shape < 1.0) {
        double x = xo_gamma(g, shape + 1.0);
        return x * pow(xo_unif(g), 1.0 / shape);
    }
    double d = shape - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
    for (;;) {
        double x, v;
        do { x = xo_normal(g); v = 1.0 + c * x; } while (v <= 0.0);
        v = v * v * v;
        double u = xo_unif(g);
        if (u < 1.0 - 0.0331 * x * x * x * x) return d * v;
        if (log(u) < 0.5 * x * x + d * (1.0 - v + log(v))) return d * v;
    }
}
/* Poisson(lambda) by counting exponential arrivals in [0, lambda). */
static int64_t xo_poisson(xo_t *g, double lambda) {
    double t = 0.0; int64_t n = 0;
    for (;;) { t += -log(xo_unif(g)); if (t >= lambda) return n; n++; }
}
/* Dirichlet(conc * 1_n) into out[n] (normalised). */
static void xo_dirichlet(xo_t *g, double conc, int n, double *out) {
    double s = 0.0;
    for (int j = 0; j < n; j++) { out[j] = xo_gamma(g, conc); s += out[j]; }
    if (!(s > 0.0)) { for (int j = 0; j < n; j++) out[j] = 1.0 / n; return; }
    for (int j = 0; j < n; j++) out[j] /= s;
}
/* first index j with cdf[j] > u (cdf ascending, cdf[n-1] ~ 1) */
static int cdf_search(const double *cdf, int n, double u) {
    int lo = 0, hi = n - 1;
    while (lo < hi) { int mid = (lo + hi) >> 1; if (cdf[mid] > u) hi = mid; else lo = mid + 1; }
    return lo;
}

static void doc_lengths(int I, int docs_per_group, double lambda, uint64_t seed, int per_unit, int32_t *len) {
    int64_t D = (int64_t)I * docs_per_group;
    if (per_unit) {
        #pragma omp parallel for schedule(static)
        for (int64_t d = 0; d < D; d++) {
            xo_t g; xo_seed_unit(&g, seed, 0, (uint64_t)d);
            int64_t L = xo_poisson(&g, lambda);
            len[d] = (int32_t)(L < 1 ? 1 : L);
        }
        return;
    }
    xo_t g; xo_seed(&g, seed, 0);
    for (int64_t d = 0; d < D; d++) {
        int64_t L = xo_poisson(&g, lambda);
        len[d] = (int32_t)(L < 1 ? 1 : L);
    }
}

/* Number of tokens the corpus with these parameters will have. */
int64_t synth_num_tokens(int I, int docs_per_group, double lambda, uint64_t seed, int per_unit) {
    int64_t D = (int64_t)I * docs_per_group, N = 0;
    int32_t *len = (int32_t *)malloc(sizeof(int32_t) * (size_t)D);
    if (!len) return -1;
    doc_lengths(I, docs_per_group, lambda, seed, per_unit, len);
    for (int64_t d = 0; d < D; d++) N += len[d];
    free(len);
    return N;
}

/* Fill group/doc/word (and the generating topic z_gen, may be NULL) for the
 * N = synth_num_tokens(...) tokens.  Returns 0 on success. */
static int spdp_corpus_per_unit(int I, int docs_per_group, double lambda, int V, int K_gen,
                                double alpha_gen, double beta_gen, double a, double b, uint64_t seed,
                                int32_t *group, int32_t *doc, int32_t *word, int32_t *z_gen);

int synth_spdp_corpus(int I, int docs_per_group, double lambda, int V, int K_gen,
                      double alpha_gen, double beta_gen, double a, double b, uint64_t seed, int per_unit,
                      int32_t *group, int32_t *doc, int32_t *word, int32_t *z_gen) {
    if (per_unit)
        return spdp_corpus_per_unit(I, docs_per_group, lambda, V, K_gen, alpha_gen, beta_gen, a, b, seed,
                                    group, doc, word, z_gen);
    int64_t D = (int64_t)I * docs_per_group;
    int32_t *len = (int32_t *)malloc(sizeof(int32_t) * (size_t)D);
    double *phi_cdf = (double *)malloc(sizeof(double) * (size_t)K_gen * V);
    double *theta = (double *)malloc(sizeof(double) * (size_t)K_gen);
    int32_t *zz = z_gen ? z_gen : NULL;
    int rc = -1;
    if (!len || !phi_cdf || !theta) goto out;
    doc_lengths(I, docs_per_group, lambda, seed, 0, len);

    /* phi0_k ~ Dir(beta_gen), stored as CDFs */
    {
        xo_t g; xo_seed(&g, seed, 1);
        for (int k = 0; k < K_gen; k++) {
            double *row = phi_cdf + (size_t)k * V;
            xo_dirichlet(&g, beta_gen, V, row);
            double c = 0.0;
            for (int w = 0; w < V; w++) { c += row[w]; row[w] = c; }
            row[V - 1] = 2.0; /* guard: every u < 1 lands */
        }
    }
    /* theta_d ~ Dir(alpha_gen), z ~ theta_d */
    int64_t N = 0;
    for (int64_t d = 0; d < D; d++) N += len[d];
    if (!zz) { zz = (int32_t *)malloc(sizeof(int32_t) * (size_t)N); if (!zz) goto out; }
    {
        xo_t g; xo_seed(&g, seed, 2);
        int64_t p = 0;
        for (int64_t d = 0; d < D; d++) {
            xo_dirichlet(&g, alpha_gen, K_gen, theta);
            double c = 0.0;
            for (int k = 0; k < K_gen; k++) { c += theta[k]; theta[k] = c; }
            theta[K_gen - 1] = 2.0;
            for (int32_t l = 0; l < len[d]; l++, p++) {
                group[p] = (int32_t)(d / docs_per_group);
                doc[p] = (int32_t)d;
                zz[p] = cdf_search(theta, K_gen, xo_unif(&g));
            }
        }
    }
    /* words: one Pitman–Yor restaurant per (group, topic); customers in
     * canonical order.  Joining an existing dish v has probability
     * proportional to n_v - a t_v, sampled by picking an earlier customer
     * uniformly (prob n_v / n) and accepting with (n_v - a t_v) / n_v. */
    {
        int64_t R = (int64_t)I * K_gen;
        int64_t *cnt = (int64_t *)calloc((size_t)R + 1, sizeof(int64_t));
        int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
        int32_t *nv = (int32_t *)calloc((size_t)V, sizeof(int32_t));
        int32_t *tv = (int32_t *)calloc((size_t)V, sizeof(int32_t));
        int32_t *seq = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
        if (!cnt || !order || !nv || !tv || !seq) {
            free(cnt); free(order); free(nv); free(tv); free(seq); goto out;
        }
        for (int64_t p = 0; p < N; p++) cnt[(int64_t)group[p] * K_gen + zz[p] + 1]++;
        for (int64_t r = 0; r < R; r++) cnt[r + 1] += cnt[r];
        {
            int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)R);
            if (!fill) { free(cnt); free(order); free(nv); free(tv); free(seq); goto out; }
            memcpy(fill, cnt, sizeof(int64_t) * (size_t)R);
            for (int64_t p = 0; p < N; p++) order[fill[(int64_t)group[p] * K_gen + zz[p]]++] = p;
            free(fill);
        }
        xo_t g; xo_seed(&g, seed, 3);
        for (int64_t r = 0; r < R; r++) {
            int k = (int)(r % K_gen);
            const double *cdf = phi_cdf + (size_t)k * V;
            int64_t n0 = cnt[r], n = cnt[r + 1] - cnt[r];
            int64_t T = 0;
            for (int64_t j = 0; j < n; j++) {
                int32_t v;
                double pnew = (b + a * (double)T) / (b + (double)j);
                if (j == 0 || xo_unif(&g) < pnew) {
                    v = cdf_search(cdf, V, xo_unif(&g));
                    tv[v]++; T++;
                } else {
                    for (;;) {
                        int32_t c = seq[xo_below(&g, (uint64_t)j)];
                        if (xo_unif(&g) * nv[c] < (double)nv[c] - a * tv[c]) { v = c; break; }
                    }
                }
                nv[v]++;
                seq[j] = v;
                word[order[n0 + j]] = v;
            }
            for (int64_t j = 0; j < n; j++) { nv[seq[j]] = 0; tv[seq[j]] = 0; }
        }
        free(cnt); free(order); free(nv); free(tv); free(seq);
    }
    rc = 0;
out:
    if (zz && zz != z_gen) free(zz);
    free(len); free(phi_cdf); free(theta);
    return rc;
}

/* Pitman–Yor seating of one restaurant's n customers (the rule above), words
 * written to word[order[j]]; nv, tv: zeroed [V] scratch, left zeroed; seq [n]. */
static void seat_restaurant(xo_t *g, const double *cdf, int V, double a, double b, int64_t n,
                            const int64_t *order, int32_t *nv, int32_t *tv, int32_t *seq, int32_t *word) {
    int64_t T = 0;
    for (int64_t j = 0; j < n; j++) {
        int32_t v;
        double pnew = (b + a * (double)T) / (b + (double)j);
        if (j == 0 || xo_unif(g) < pnew) {
            v = cdf_search(cdf, V, xo_unif(g));
            tv[v]++; T++;
        } else {
            for (;;) {
                int32_t c = seq[xo_below(g, (uint64_t)j)];
                if (xo_unif(g) * nv[c] < (double)nv[c] - a * tv[c]) { v = c; break; }
            }
        }
        nv[v]++;
        seq[j] = v;
        word[order[j]] = v;
    }
    for (int64_t j = 0; j < n; j++) { nv[seq[j]] = 0; tv[seq[j]] = 0; }
}

static int spdp_corpus_per_unit(int I, int docs_per_group, double lambda, int V, int K_gen,
                                double alpha_gen, double beta_gen, double a, double b, uint64_t seed,
                                int32_t *group, int32_t *doc, int32_t *word, int32_t *z_gen) {
    int64_t D = (int64_t)I * docs_per_group, R = (int64_t)I * K_gen;
    int32_t *len = (int32_t *)malloc(sizeof(int32_t) * (size_t)D);
    int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(D + 1));
    double *phi_cdf = (double *)malloc(sizeof(double) * (size_t)K_gen * V);
    int64_t *cnt = (int64_t *)calloc((size_t)R + 1, sizeof(int64_t));
    int32_t *zz = z_gen;
    int64_t *order = NULL;
    int rc = -1;
    if (!len || !start || !phi_cdf || !cnt) goto out;
    doc_lengths(I, docs_per_group, lambda, seed, 1, len);
    start[0] = 0;
    for (int64_t d = 0; d < D; d++) start[d + 1] = start[d] + len[d];
    int64_t N = start[D];
    if (!zz) { zz = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1)); if (!zz) goto out; }
    order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
    if (!order) goto out;
    /* phi0_k ~ Dir(beta_gen) as CDFs, one generator per topic */
    #pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < K_gen; k++) {
        xo_t g; xo_seed_unit(&g, seed, 1, (uint64_t)k);
        double *row = phi_cdf + (size_t)k * V;
        xo_dirichlet(&g, beta_gen, V, row);
        double c = 0.0;
        for (int w = 0; w < V; w++) { c += row[w]; row[w] = c; }
        row[V - 1] = 2.0;
    }
    /* theta_d ~ Dir(alpha_gen), z ~ theta_d, one generator per document */
    int fail = 0;
    #pragma omp parallel
    {
        double *theta = (double *)malloc(sizeof(double) * (size_t)K_gen);
        if (!theta) {
            #pragma omp atomic write
            fail = 1;
        } else {
            #pragma omp for schedule(dynamic, 4096)
            for (int64_t d = 0; d < D; d++) {
                xo_t g; xo_seed_unit(&g, seed, 2, (uint64_t)d);
                xo_dirichlet(&g, alpha_gen, K_gen, theta);
                double c = 0.0;
                for (int k = 0; k < K_gen; k++) { c += theta[k]; theta[k] = c; }
                theta[K_gen - 1] = 2.0;
                for (int64_t p = start[d]; p < start[d + 1]; p++) {
                    group[p] = (int32_t)(d / docs_per_group);
                    doc[p] = (int32_t)d;
                    zz[p] = cdf_search(theta, K_gen, xo_unif(&g));
                }
            }
            free(theta);
        }
    }
    if (fail) goto out;
    /* customers of each restaurant (group, topic) in canonical order */
    for (int64_t p = 0; p < N; p++) cnt[(int64_t)group[p] * K_gen + zz[p] + 1]++;
    for (int64_t r = 0; r < R; r++) cnt[r + 1] += cnt[r];
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(R > 0 ? R : 1));
        if (!fill) goto out;
        memcpy(fill, cnt, sizeof(int64_t) * (size_t)R);
        for (int64_t p = 0; p < N; p++) order[fill[(int64_t)group[p] * K_gen + zz[p]]++] = p;
        free(fill);
    }
    /* words: one generator per restaurant */
    #pragma omp parallel
    {
        int32_t *nv = (int32_t *)calloc((size_t)V, sizeof(int32_t));
        int32_t *tv = (int32_t *)calloc((size_t)V, sizeof(int32_t));
        int64_t mx = 1;
        for (int64_t r = 0; r < R; r++) if (cnt[r + 1] - cnt[r] > mx) mx = cnt[r + 1] - cnt[r];
        int32_t *seq = (int32_t *)malloc(sizeof(int32_t) * (size_t)mx);
        if (!nv || !tv || !seq) {
            #pragma omp atomic write
            fail = 1;
        } else {
            #pragma omp for schedule(dynamic, 1)
            for (int64_t r = 0; r < R; r++) {
                xo_t g; xo_seed_unit(&g, seed, 3, (uint64_t)r);
                seat_restaurant(&g, phi_cdf + (size_t)(r % K_gen) * V, V, a, b, cnt[r + 1] - cnt[r], order + cnt[r],
                                nv, tv, seq, word);
            }
        }
        free(nv); free(tv); free(seq);
    }
    if (!fail) rc = 0;
out:
    if (zz && zz != z_gen) free(zz);
    free(len); free(start); free(phi_cdf); free(cnt); free(order);
    return rc;
}
