/*
 * oracle/spdp_oracle.c — plain, slow, CPU reference for the SPDP Gibbs sweep.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code with paper_1510_06549_b200/ (own Philox, own Stirling
 * numbers, own partition and wave plan), and the product path never calls it.
 *
 * Everything is fp64, and the sampler weights are formed in log space.
 * Citations are PAPER.md line numbers (P:<line>) with the section / equation /
 * algorithm they fall in; "reading cN" refers to DESIGN.md §3 (readings of
 * the paper), which follows SURVEY.md §8(c).
 *
 *  - Generalised Stirling numbers S^N_{M,a}: P:1452-1457 (§2.4.5):
 *      S^{N+1}_M = S^N_{M-1} + (N - M a) S^N_M,  S^N_M = 0 for M > N,
 *      S^N_0 = delta_{N,0}.  Kept as log S in a lower-triangular table.
 *  - Pochhammer symbols (x|y)_N = prod_{n<N} (x + n y), (x)_N = (x|1)_N:
 *      P:1452-1453.
 *  - Conditionals Eq. SPDP-sampling-w-z-r0 and
 *      Eq. SPDP-sampling-w-z-r1 with identity P,
 *      so q_{ikwv} = t_{ikw}[v=w] and sum_i sum_w q_{ikwv} = Q_{kv}.
 *  - Algorithm 1 "SPDP Full Gibbs Sampling" = or_sweep_seq,
 *      plus the keep rule (reading c5).
 *  - Parallel framework (§3.3, P:2210-2233, P:2289-2299, P:2370-2386,
 *      P:2411-2427; Alg.3/Alg.4) with the deterministic
 *      wave-snapshot reading (reading c13) = or_sweep_par.
 *  - Estimators Eqs. spdp-topic-doc-estimate,
 *      spdp-word-topic-estimate, spdp-group-word-topic-estimate
 *      (reading c16) and the perplexity of §3.2 (P:1978-2007,
 *      reading c17) = or_perplexity.
 *  - Joint p(W,Z,T) from the blocked-Gibbs joint with the
 *      C(m,t) factor of Eq. SPDP-table-to-head summed out
 *      = or_log_joint (reading c1, c2).
 *  - Philox4x32-10 counter-based RNG (reading c11; Salmon et al. 2011).
 *  - NEXT-1 held-out evaluation: topic estimates or_phi0 / or_phi / or_topics
 *      (P:1753-1754); fold-in of held-out documents or_foldin (reading c21);
 *      held-out perplexity or_heldout_perplexity; Hellinger
 *      distance and greedy topic alignment or_hellinger / or_topic_align
 *      (§4.2.6, reading c22).
 *  - NEXT-3 exchange cadence or_sweep_par_e.
 *  - NEXT-4 sparse transformation matrices P^i: or_sp_* (P:985-1014,
 *      P:1455-1468; readings c24-c26).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Philox4x32-10                                                       */
/* ------------------------------------------------------------------ */
void or_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * x0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t y0 = hi1 ^ x1 ^ k0, y1 = lo1, y2 = hi0 ^ x3 ^ k1, y3 = lo0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

static void rng_token(uint64_t seed, uint32_t tok, uint32_t sweep, uint32_t x[4]) {
    uint32_t ctr[4] = {tok, sweep, 0u, 0u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    or_philox(ctr, key, x);
}
/* 53-bit uniform in [0,1) from x1 (32 bits) and the top 21 bits of x2 */
static double u53(const uint32_t x[4]) {
    return ((double)x[1] * 2097152.0 + (double)(x[2] >> 11)) * (1.0 / 9007199254740992.0);
}

/* ------------------------------------------------------------------ */
/* log generalised Stirling numbers                       */
/* ------------------------------------------------------------------ */
typedef struct {
    double a;
    int nmax;          /* rows 0..nmax */
    double *v;         /* row N at offset N(N+1)/2, entries M = 0..N */
} stable_t;

static double logaddexp(double x, double y) {
    if (x == -INFINITY) return y;
    if (y == -INFINITY) return x;
    double mx = x > y ? x : y, mn = x > y ? y : x;
    return mx + log1p(exp(mn - mx));
}

static int stable_build(stable_t *s, double a, int nmax) {
    size_t sz = (size_t)(nmax + 1) * (size_t)(nmax + 2) / 2;
    double *v = (double *)malloc(sizeof(double) * sz);
    if (!v) return -1;
    v[0] = 0.0; /* S^0_0 = 1 */
    for (int N = 0; N < nmax; N++) {
        const double *row = v + (size_t)N * (N + 1) / 2;
        double *nxt = v + (size_t)(N + 1) * (N + 2) / 2;
        nxt[0] = -INFINITY; /* S^{N+1}_0 = 0 */
        for (int M = 1; M <= N + 1; M++) {
            double left = row[M - 1];                                 /* S^N_{M-1} */
            double right = (M <= N) ? row[M] : -INFINITY;             /* S^N_M (0 if M > N) */
            double coef = (double)N - (double)M * a;                  /* (N - M a) */
            double term = (right == -INFINITY || coef <= 0.0) ? -INFINITY : log(coef) + right;
            nxt[M] = logaddexp(left, term);
        }
    }
    s->a = a; s->nmax = nmax; s->v = v;
    return 0;
}

static double stable_get(const stable_t *s, int N, int M) {
    if (M < 0 || M > N) return -INFINITY;
    return s->v[(size_t)N * (N + 1) / 2 + M];
}

double or_log_stirling(double a, int N, int M) {
    stable_t s;
    if (N < 0) return -INFINITY;
    if (stable_build(&s, a, N) != 0) return NAN;
    double r = stable_get(&s, N, M);
    free(s.v);
    return r;
}

/* The Stirling ratios the conditional of Eqs. r0/r1 multiplies
 * by, written out from the log table above:
 *   A0(m,t) = (m-t+1)/(m+1) * S^{m+1}_t / S^m_t        (r = 0, Eq. r0)
 *   A1(m,t) = (t+1)/(m+1)   * S^{m+1}_{t+1} / S^m_t    (r = 1, Eq. r1)
 * for 0 <= t <= m <= mmax at index m(m+1)/2 + t.  t = 0 < m (S^m_0 = 0) is not
 * a state and gets 0.  Returns 0, or -1 if the table cannot be allocated. */
int or_ratio_table(double a, int mmax, double *A0, double *A1) {
    stable_t S;
    if (mmax < 0 || stable_build(&S, a, mmax + 1) != 0) return -1;
    for (int m = 0; m <= mmax; m++)
        for (int t = 0; t <= m; t++) {
            size_t j = (size_t)m * (m + 1) / 2 + t;
            double lS = stable_get(&S, m, t);
            if (lS == -INFINITY) { A0[j] = 0.0; A1[j] = 0.0; continue; }
            A0[j] = (double)(m - t + 1) / (double)(m + 1) * exp(stable_get(&S, m + 1, t) - lS);
            A1[j] = (double)(t + 1) / (double)(m + 1) * exp(stable_get(&S, m + 1, t + 1) - lS);
        }
    free(S.v);
    return 0;
}

/* ln (x|y)_n = sum_{j<n} ln(x + j y) */
static double log_poch(double x, double y, int64_t n) {
    double s = 0.0;
    for (int64_t j = 0; j < n; j++) s += log(x + (double)j * y);
    return s;
}

/* ------------------------------------------------------------------ */
/* state                                                               */
/* ------------------------------------------------------------------ */
typedef struct {
    int I, V, K;
    double *alpha;     /* [I*K] */
    double beta;
    double *a, *b;     /* [I] */
    uint64_t seed;
    uint32_t sweep;    /* next sweep index (RNG counter word 1) */

    int64_t N; int32_t D;
    int32_t *group, *doc, *word, *pos;   /* canonical token arrays; pos = in-doc position l */
    int32_t *doclen;                      /* [D] */
    int32_t *z; uint8_t *r;
    int32_t *n;        /* [D*K] */
    int32_t *m, *t;    /* [I*V*K]  (i, w, k) */
    int64_t *M, *Tt;   /* [I*K]    m_{ik.}, t_{ik.} */
    int64_t *Q;        /* [K*V]    Q_{kw} = sum_i t_{ikw} */
    int64_t *T;        /* [K]      T_k = sum_w Q_{kw} */
    stable_t *tab;     /* [I] (aliased when discounts coincide) */
    int nmax;
    int64_t stats[8];  /* last sweep: 0 keeps, 1 moved, 2 clamped cells, 3 forced-differ */
} ostate;

#define IDX3(s, i, w, k) (((size_t)(i) * (s)->V + (size_t)(w)) * (s)->K + (size_t)(k))

void or_destroy(ostate *s) {
    if (!s) return;
    free(s->alpha); free(s->a); free(s->b);
    free(s->group); free(s->doc); free(s->word); free(s->pos); free(s->doclen);
    free(s->z); free(s->r); free(s->n); free(s->m); free(s->t);
    free(s->M); free(s->Tt); free(s->Q); free(s->T);
    if (s->tab) {
        for (int i = 0; i < s->I; i++) {
            int alias = 0;
            for (int j = 0; j < i; j++) if (s->tab[j].v == s->tab[i].v) alias = 1;
            if (!alias) free(s->tab[i].v);
        }
        free(s->tab);
    }
    free(s);
}

ostate *or_create(int I, int V, int K, const double *alpha_ik, double beta,
                  const double *a, const double *b, uint64_t seed) {
    if (I < 1 || V < 1 || K < 1 || !(beta > 0.0)) return NULL;
    ostate *s = (ostate *)calloc(1, sizeof(ostate));
    if (!s) return NULL;
    s->I = I; s->V = V; s->K = K; s->beta = beta; s->seed = seed;
    s->alpha = (double *)malloc(sizeof(double) * (size_t)I * K);
    s->a = (double *)malloc(sizeof(double) * (size_t)I);
    s->b = (double *)malloc(sizeof(double) * (size_t)I);
    if (!s->alpha || !s->a || !s->b) { or_destroy(s); return NULL; }
    memcpy(s->alpha, alpha_ik, sizeof(double) * (size_t)I * K);
    memcpy(s->a, a, sizeof(double) * (size_t)I);
    memcpy(s->b, b, sizeof(double) * (size_t)I);
    return s;
}

/* recompute every derived sum from m and t (plain loops) */
static void recompute_sums(const ostate *s, const int32_t *m, const int32_t *t,
                           int64_t *M, int64_t *Tt, int64_t *Q, int64_t *T) {
    int I = s->I, V = s->V, K = s->K;
    memset(M, 0, sizeof(int64_t) * (size_t)I * K);
    memset(Tt, 0, sizeof(int64_t) * (size_t)I * K);
    memset(Q, 0, sizeof(int64_t) * (size_t)K * V);
    memset(T, 0, sizeof(int64_t) * (size_t)K);
    for (int i = 0; i < I; i++)
        for (int w = 0; w < V; w++)
            for (int k = 0; k < K; k++) {
                size_t c = IDX3(s, i, w, k);
                M[(size_t)i * K + k] += m[c];
                Tt[(size_t)i * K + k] += t[c];
                Q[(size_t)k * V + w] += t[c];
                T[k] += t[c];
            }
}

static int ensure_tables(ostate *s, int nmax) {
    if (s->tab && s->nmax >= nmax) return 0;
    if (s->tab) {
        for (int i = 0; i < s->I; i++) {
            int alias = 0;
            for (int j = 0; j < i; j++) if (s->tab[j].v == s->tab[i].v) alias = 1;
            if (!alias) free(s->tab[i].v);
        }
        free(s->tab);
    }
    s->tab = (stable_t *)calloc((size_t)s->I, sizeof(stable_t));
    if (!s->tab) return -1;
    for (int i = 0; i < s->I; i++) {
        int j;
        for (j = 0; j < i; j++) if (s->a[j] == s->a[i]) break;
        if (j < i) { s->tab[i] = s->tab[j]; continue; }
        if (stable_build(&s->tab[i], s->a[i], nmax) != 0) return -1;
    }
    s->nmax = nmax;
    return 0;
}

/* t_init (optional, [I*V*K]) overrides the table counts derived from r. */
int or_load(ostate *s, int64_t N, int32_t D, const int32_t *group, const int32_t *doc,
            const int32_t *word, const int32_t *z_init, const uint8_t *r_init, const int32_t *t_init) {
    int I = s->I, V = s->V, K = s->K;
    if (N < 0 || D < 1) return -1;
    for (int64_t p = 0; p < N; p++) {
        if (group[p] < 0 || group[p] >= I || doc[p] < 0 || doc[p] >= D || word[p] < 0 || word[p] >= V) return -1;
        if (z_init && (z_init[p] < 0 || z_init[p] >= K)) return -1;
        if (r_init && r_init[p] > 1) return -1;
    }
    s->N = N; s->D = D;
    size_t cells = (size_t)I * V * K;
    s->group = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    s->doc = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    s->word = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    s->pos = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    s->z = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    s->r = (uint8_t *)malloc((size_t)(N + 1));
    s->doclen = (int32_t *)calloc((size_t)D, sizeof(int32_t));
    s->n = (int32_t *)calloc((size_t)D * K, sizeof(int32_t));
    s->m = (int32_t *)calloc(cells, sizeof(int32_t));
    s->t = (int32_t *)calloc(cells, sizeof(int32_t));
    s->M = (int64_t *)calloc((size_t)I * K, sizeof(int64_t));
    s->Tt = (int64_t *)calloc((size_t)I * K, sizeof(int64_t));
    s->Q = (int64_t *)calloc((size_t)K * V, sizeof(int64_t));
    s->T = (int64_t *)calloc((size_t)K, sizeof(int64_t));
    int32_t *docgroup = (int32_t *)malloc(sizeof(int32_t) * (size_t)D);
    if (!s->group || !s->doc || !s->word || !s->pos || !s->z || !s->r || !s->doclen || !s->n ||
        !s->m || !s->t || !s->M || !s->Tt || !s->Q || !s->T || !docgroup) { free(docgroup); return -2; }
    memcpy(s->group, group, sizeof(int32_t) * (size_t)N);
    memcpy(s->doc, doc, sizeof(int32_t) * (size_t)N);
    memcpy(s->word, word, sizeof(int32_t) * (size_t)N);
    for (int32_t d = 0; d < D; d++) docgroup[d] = -1;
    for (int64_t p = 0; p < N; p++) {
        int32_t d = doc[p];
        if (docgroup[d] >= 0 && docgroup[d] != group[p]) { free(docgroup); return -1; } /* doc spans groups */
        docgroup[d] = group[p];
        s->pos[p] = s->doclen[d]++;
    }
    free(docgroup);
    /* z: given, or Philox(seed; tok, 0xFFFFFFFF) -> floor(x0 K / 2^32) */
    for (int64_t p = 0; p < N; p++) {
        if (z_init) s->z[p] = z_init[p];
        else {
            uint32_t x[4];
            rng_token(s->seed, (uint32_t)p, 0xFFFFFFFFu, x);
            s->z[p] = (int32_t)(((uint64_t)x[0] * (uint64_t)K) >> 32);
        }
    }
    /* counts from z ("Initialize counting variables ... from z") */
    for (int64_t p = 0; p < N; p++) {
        s->n[(size_t)doc[p] * K + s->z[p]]++;
        s->m[IDX3(s, group[p], word[p], s->z[p])]++;
    }
    /* r: given, or 1 for the first token of each (i,k,w) cell (reading c12) */
    for (int64_t p = 0; p < N; p++) {
        size_t c = IDX3(s, group[p], word[p], s->z[p]);
        if (r_init) s->r[p] = r_init[p];
        else s->r[p] = (s->t[c] == 0) ? 1 : 0;
        s->t[c] += s->r[p];
    }
    if (t_init) memcpy(s->t, t_init, sizeof(int32_t) * cells);
    for (size_t c = 0; c < cells; c++) {
        if (s->t[c] < 0 || s->t[c] > s->m[c] || ((s->m[c] > 0) != (s->t[c] > 0))) return -1;
    }
    recompute_sums(s, s->m, s->t, s->M, s->Tt, s->Q, s->T);
    int32_t mmax = 0;
    for (size_t c = 0; c < cells; c++) if (s->m[c] > mmax) mmax = s->m[c];
    /* every reachable m_{ikw} is bounded by count(i,w); the m of a cell never exceeds it */
    {
        int32_t *cnt = (int32_t *)calloc((size_t)I * V, sizeof(int32_t));
        if (!cnt) return -2;
        for (int64_t p = 0; p < N; p++) cnt[(size_t)group[p] * V + word[p]]++;
        for (size_t c = 0; c < (size_t)I * V; c++) if (cnt[c] > mmax) mmax = cnt[c];
        free(cnt);
    }
    if (ensure_tables(s, mmax + 1) != 0) return -2;
    s->sweep = 0;
    return 0;
}

/* ------------------------------------------------------------------ */
/* the conditional, Eqs. SPDP-sampling-w-z-r0 / -r1      */
/* ------------------------------------------------------------------ */
/* Log weights of the 2K slots for token p against the counts given, with the
 * token's own contribution removed (Alg.1 lines 3-10): its old
 * topic k0 loses one customer, and one table when r_rem = 1.
 * Slot order (Alg.4): j = 2k <-> (k, r=1), j = 2k+1 <-> (k, r=0). */
static void log_weights(const ostate *s, int64_t p, int r_rem,
                        const int32_t *n, const int32_t *m, const int32_t *t,
                        const int64_t *M, const int64_t *Tt, const int64_t *Q, const int64_t *T,
                        double *lw) {
    int K = s->K, V = s->V;
    int i = s->group[p], w = s->word[p], d = s->doc[p], k0 = s->z[p];
    double a = s->a[i], b = s->b[i], beta = s->beta;
    const stable_t *S = &s->tab[i];
    for (int k = 0; k < K; k++) {
        int own = (k == k0);
        double n_k = (double)n[(size_t)d * K + k] - own;
        int64_t m_k = m[IDX3(s, i, w, k)] - own;
        int64_t t_k = t[IDX3(s, i, w, k)] - own * r_rem;
        double M_k = (double)M[(size_t)i * K + k] - own;
        double Tt_k = (double)Tt[(size_t)i * K + k] - own * r_rem;
        double Q_k = (double)Q[(size_t)k * V + w] - own * r_rem;
        double T_k = (double)T[k] - own * r_rem;
        double lS = stable_get(S, (int)m_k, (int)t_k);
        double base = log(s->alpha[(size_t)i * K + k] + n_k) - log(b + M_k);
        /* r = 0: (alpha+n)/(b+M) * (m-t+1)/(m+1) * S^{m+1}_t / S^m_t */
        double l0 = base + log((double)(m_k - t_k + 1)) - log((double)(m_k + 1))
                    + stable_get(S, (int)m_k + 1, (int)t_k) - lS;
        /* r = 1: (alpha+n)(b + a T_t)/(b+M) * (t+1)/(m+1) * (beta+Q)/(V beta + T) * S^{m+1}_{t+1} / S^m_t */
        double l1 = base + log(b + a * Tt_k) + log((double)(t_k + 1)) - log((double)(m_k + 1))
                    + log(beta + Q_k) - log((double)V * beta + T_k)
                    + stable_get(S, (int)m_k + 1, (int)t_k + 1) - lS;
        lw[2 * k] = l1;
        lw[2 * k + 1] = l0;
    }
}

/* Normalised probabilities by max-shifted exponentiation in fp64 (reading c9). */
static void normalise(int n, const double *lw, double *prob) {
    double mx = -INFINITY;
    for (int j = 0; j < n; j++) if (lw[j] > mx) mx = lw[j];
    double tot = 0.0;
    for (int j = 0; j < n; j++) { prob[j] = (lw[j] == -INFINITY) ? 0.0 : exp(lw[j] - mx); tot += prob[j]; }
    for (int j = 0; j < n; j++) prob[j] /= tot;
}

/* j* = min{ j : cdf_j > u }; if rounding leaves none, the last j with p_j > 0
 * (reading c10).  *margin = distance of u to the nearest edge of slot j*. */
static int draw_slot(int n, const double *prob, double u, double *margin) {
    double c = 0.0, prev = 0.0;
    for (int j = 0; j < n; j++) {
        prev = c;
        c += prob[j];
        if (c > u && prob[j] > 0.0) {
            if (margin) { double m1 = u - prev, m2 = c - u; *margin = m1 < m2 ? m1 : m2; }
            return j;
        }
    }
    for (int j = n - 1; j >= 0; j--) if (prob[j] > 0.0) { if (margin) *margin = 0.0; return j; }
    return -1;
}

/* Removal draw r ~ Bernoulli(t/m) (Alg.1 line 3): exact integer test
 * x0 * m < t * 2^32 (reading c7).  keep: r = 1 with t = 1 < m (reading c5). */
static int removal(uint32_t x0, int64_t m_c, int64_t t_c, int *keep) {
    int r = ((uint64_t)x0 * (uint64_t)m_c) < ((uint64_t)t_c << 32);
    *keep = (r && t_c == 1 && m_c > 1);
    return r;
}

/* ------------------------------------------------------------------ */
/* Mode S: Algorithm 1 as printed + keep rule            */
/* ------------------------------------------------------------------ */
int or_sweep_seq(ostate *s, int64_t max_tokens) {
    int K = s->K, V = s->V;
    double *lw = (double *)malloc(sizeof(double) * 2 * (size_t)K);
    double *prob = (double *)malloc(sizeof(double) * 2 * (size_t)K);
    if (!lw || !prob) { free(lw); free(prob); return -2; }
    memset(s->stats, 0, sizeof(s->stats));
    int64_t lim = (max_tokens >= 0 && max_tokens < s->N) ? max_tokens : s->N;
    for (int64_t p = 0; p < lim; p++) {                     /* ForAll w_{i,d,l} */
        int i = s->group[p], w = s->word[p], d = s->doc[p], k = s->z[p];   /* line 2 */
        size_t c = IDX3(s, i, w, k);
        uint32_t x[4];
        rng_token(s->seed, (uint32_t)p, s->sweep, x);
        int keep, r = removal(x[0], s->m[c], s->t[c], &keep);             /* line 3 */
        if (keep) { s->r[p] = 1; s->stats[0]++; continue; }
        log_weights(s, p, r, s->n, s->m, s->t, s->M, s->Tt, s->Q, s->T, lw); /* lines 11-16 (removal folded in) */
        /* lines 4-10: decrement n, m (and t, q when r = 1) */
        s->n[(size_t)d * K + k]--; s->m[c]--; s->M[(size_t)i * K + k]--;
        if (r) { s->t[c]--; s->Tt[(size_t)i * K + k]--; s->Q[(size_t)k * V + w]--; s->T[k]--; }
        normalise(2 * K, lw, prob);
        int j = draw_slot(2 * K, prob, u53(x), NULL);                     /* line 17 */
        int kn = j / 2, rn = (j % 2 == 0);
        size_t cn = IDX3(s, i, w, kn);
        s->n[(size_t)d * K + kn]++; s->m[cn]++; s->M[(size_t)i * K + kn]++;   /* line 18 */
        if (rn) { s->t[cn]++; s->Tt[(size_t)i * K + kn]++; s->Q[(size_t)kn * V + w]++; s->T[kn]++; } /* 19-22 */
        if (kn != k) s->stats[1]++;
        s->z[p] = kn; s->r[p] = (uint8_t)rn;
    }
    s->sweep++;
    free(lw); free(prob);
    return 0;
}

/* ------------------------------------------------------------------ */
/* document partition over G shards (reading: SURVEY §8(e))            */
/* ------------------------------------------------------------------ */
/* Docs are ordered by the Philox word x0 of (doc, 0xFFFFFFFE) (ties by id),
 * then split contiguously by cumulative token count:
 * shard = floor(tokens_before * G / N). */
typedef struct { uint32_t key; int32_t doc; } dkey_t;
static int dkey_cmp(const void *x, const void *y) {
    const dkey_t *p = (const dkey_t *)x, *q = (const dkey_t *)y;
    if (p->key != q->key) return p->key < q->key ? -1 : 1;
    return p->doc < q->doc ? -1 : (p->doc > q->doc);
}
void or_partition(const ostate *s, int G, int32_t *shard_of_doc) {
    dkey_t *v = (dkey_t *)malloc(sizeof(dkey_t) * (size_t)s->D);
    for (int32_t d = 0; d < s->D; d++) {
        uint32_t x[4];
        rng_token(s->seed, (uint32_t)d, 0xFFFFFFFEu, x);
        v[d].key = x[0]; v[d].doc = d;
    }
    qsort(v, (size_t)s->D, sizeof(dkey_t), dkey_cmp);
    int64_t before = 0;
    for (int32_t j = 0; j < s->D; j++) {
        int32_t d = v[j].doc;
        int64_t g = (s->N > 0) ? (before * (int64_t)G) / s->N : 0;
        if (g >= G) g = G - 1;
        shard_of_doc[d] = (int32_t)g;
        before += s->doclen[d];
    }
    free(v);
}

/* clamp t into [min(1,m), m] (reading c14) */
static int64_t clamp_cells(size_t cells, const int32_t *m, int32_t *t) {
    int64_t changed = 0;
    for (size_t c = 0; c < cells; c++) {
        int32_t v = t[c];
        if (v > m[c]) v = m[c];
        if (m[c] > 0 && v < 1) v = 1;
        if (m[c] == 0) v = 0;
        if (v != t[c]) { t[c] = v; changed++; }
    }
    return changed;
}

/* ------------------------------------------------------------------ */
/* Mode P: wave snapshots, G shards, merge (reading c13-c15)           */
/* ------------------------------------------------------------------ */
/* W >= 1: wave(token) = l mod W (l = in-doc position).
 * W == 0: every token is its own wave, in canonical order (= mode S).
 * force_zr (optional, [N], -1 = none): replace the drawn (z | r<<15) of a
 * token that is not kept (lock-step replay of another sampler's draws).
 * margin (optional, [N]): distance of u to the edge of the drawn slot.
 * own_zr (optional, [N]): the oracle's own draw (z | r<<15) before forcing.
 * max_tokens >= 0 limits the sweep to the first max_tokens tokens of each
 * shard's canonical order (timing samples only). */
/* E >= 1: the shards exchange (merge) after every E waves instead of once per
 * sweep (bounded staleness; P:2427-2434 relies on
 * "implicit synchronization ... as long as the delay can be tolerated"): each
 * block of E waves starts from the merged state of the previous block.
 * E <= 0 (or E >= the number of waves): one exchange per sweep. */
static int sweep_par_impl(ostate *s, int W, int G, int only, const int32_t *force_zr, double *margin,
                          int64_t max_tokens, int32_t *own_zr, int32_t *Dout_m, int32_t *Dout_t, int E) {
    int I = s->I, V = s->V, K = s->K;
    int64_t N = s->N;
    size_t cells = (size_t)I * V * K;
    if (W < 0 || G < 1) return -1;
    memset(s->stats, 0, sizeof(s->stats));
    int32_t *shard = (int32_t *)malloc(sizeof(int32_t) * (size_t)s->D);
    int32_t *S0m = (int32_t *)malloc(sizeof(int32_t) * cells), *S0t = (int32_t *)malloc(sizeof(int32_t) * cells);
    int32_t *Lm = (int32_t *)malloc(sizeof(int32_t) * cells), *Lt = (int32_t *)malloc(sizeof(int32_t) * cells);
    int64_t *Dm = (int64_t *)calloc(cells, sizeof(int64_t)), *Dt = (int64_t *)calloc(cells, sizeof(int64_t));
    int64_t *M = (int64_t *)malloc(sizeof(int64_t) * (size_t)I * K), *Tt = (int64_t *)malloc(sizeof(int64_t) * (size_t)I * K);
    int64_t *Q = (int64_t *)malloc(sizeof(int64_t) * (size_t)K * V), *T = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
    int32_t *newz = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    int8_t *newr = (int8_t *)malloc((size_t)(N + 1)), *rrem = (int8_t *)malloc((size_t)(N + 1)), *kept = (int8_t *)malloc((size_t)(N + 1));
    int64_t *inwave = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N + 1));
    int64_t *seen = (int64_t *)calloc((size_t)G, sizeof(int64_t));
    double *lw = (double *)malloc(sizeof(double) * 2 * (size_t)K), *prob = (double *)malloc(sizeof(double) * 2 * (size_t)K);
    int rc = -2;
    if (!shard || !S0m || !S0t || !Lm || !Lt || !Dm || !Dt || !M || !Tt || !Q || !T || !newz || !newr || !rrem ||
        !kept || !inwave || !lw || !prob || !seen) goto out;
    or_partition(s, G, shard);
    int32_t maxlen = 0;
    for (int32_t d = 0; d < s->D; d++) if (s->doclen[d] > maxlen) maxlen = s->doclen[d];
    int64_t nwaves = (W == 0) ? N : (W < maxlen ? W : maxlen);
    int64_t block = (E <= 0 || E >= nwaves) ? nwaves : E;
    if (only >= 0 && block < nwaves) goto out;   /* the distributed form exchanges once per sweep */
    for (int64_t b0 = 0; b0 < nwaves || (nwaves == 0 && b0 == 0); b0 += (block > 0 ? block : 1)) {
    int64_t b1 = b0 + block < nwaves ? b0 + block : nwaves;
    memcpy(S0m, s->m, sizeof(int32_t) * cells);
    memcpy(S0t, s->t, sizeof(int32_t) * cells);
    memset(Dm, 0, sizeof(int64_t) * cells);
    memset(Dt, 0, sizeof(int64_t) * cells);
    for (int g = 0; g < G; g++) {
        if (only >= 0 && g != only) continue;
        /* shard-local replica of the block-start global state (Alg.3) */
        memcpy(Lm, S0m, sizeof(int32_t) * cells);
        memcpy(Lt, S0t, sizeof(int32_t) * cells);
        recompute_sums(s, Lm, Lt, M, Tt, Q, T);
        for (int64_t wave = b0; wave < b1; wave++) {
            /* tokens of this shard in this wave, canonical order */
            int64_t cnt = 0;
            if (W == 0) {
                if (shard[s->doc[wave]] == g) inwave[cnt++] = wave;
            } else {
                for (int64_t p = 0; p < N; p++)
                    if (shard[s->doc[p]] == g && s->pos[p] % W == wave) inwave[cnt++] = p;
            }
            /* (1) every token decides against the wave-start snapshot.  A max_tokens bound lets
             * the shard's first max_tokens tokens (canonical order within each wave) through.
             * The decisions are independent given the snapshot: the -fopenmp timing build
             * (oracle.build(openmp=True)) spreads them over the host cores. */
            int64_t take = cnt;
            if (max_tokens >= 0) {
                int64_t room = max_tokens - seen[g];
                if (room < 0) room = 0;
                if (take > room) take = room;
            }
            for (int64_t q = take; q < cnt; q++) kept[inwave[q]] = 2;   /* not sampled */
            seen[g] += take;
            #pragma omp parallel for schedule(dynamic, 64)
            for (int64_t q = 0; q < take; q++) {
                int64_t p = inwave[q];
                double lw[2 * K], prob[2 * K];
                int i = s->group[p], w = s->word[p], k0 = s->z[p];
                size_t c = IDX3(s, i, w, k0);
                uint32_t x[4];
                rng_token(s->seed, (uint32_t)p, s->sweep, x);
                int keep, r = removal(x[0], Lm[c], Lt[c], &keep);
                rrem[p] = (int8_t)r;
                kept[p] = (int8_t)keep;
                if (keep) { newz[p] = k0; newr[p] = 1; if (own_zr) own_zr[p] = k0 | (1 << 15); continue; }
                log_weights(s, p, r, s->n, Lm, Lt, M, Tt, Q, T, lw);
                normalise(2 * K, lw, prob);
                int j = draw_slot(2 * K, prob, u53(x), margin ? &margin[p] : NULL);
                newz[p] = j / 2; newr[p] = (j % 2 == 0);
                if (own_zr) own_zr[p] = newz[p] | (newr[p] << 15);
                if (force_zr && force_zr[p] >= 0) {
                    int fz = force_zr[p] & 0x7FFF, fr = (force_zr[p] >> 15) & 1;
                    if (fz != newz[p] || fr != newr[p]) {
                        #pragma omp atomic
                        s->stats[3]++;
                    }
                    newz[p] = fz; newr[p] = (int8_t)fr;
                }
            }
            /* (2) apply all deltas of the wave, clamp, recompute sums */
            for (int64_t q = 0; q < cnt; q++) {
                int64_t p = inwave[q];
                if (kept[p] == 2) continue;
                if (kept[p]) { s->r[p] = 1; s->stats[0]++; continue; }
                int i = s->group[p], w = s->word[p], d = s->doc[p], k0 = s->z[p], kn = newz[p];
                size_t c0 = IDX3(s, i, w, k0), cn = IDX3(s, i, w, kn);
                s->n[(size_t)d * K + k0]--; s->n[(size_t)d * K + kn]++;
                Lm[c0]--; Lm[cn]++;
                Lt[c0] -= rrem[p]; Lt[cn] += newr[p];
                if (kn != k0) s->stats[1]++;
                s->z[p] = kn; s->r[p] = (uint8_t)newr[p];
            }
            if (cnt > 0) {
                s->stats[2] += clamp_cells(cells, Lm, Lt);
                recompute_sums(s, Lm, Lt, M, Tt, Q, T);
            }
        }
        /* D_g = L_g - S0 */
        for (size_t c = 0; c < cells; c++) { Dm[c] += Lm[c] - S0m[c]; Dt[c] += Lt[c] - S0t[c]; }
    }
    if (only >= 0) {           /* one shard of a distributed sweep: hand out D_g, no merge */
        for (size_t c = 0; c < cells; c++) { Dout_m[c] = (int32_t)Dm[c]; Dout_t[c] = (int32_t)Dt[c]; }
        rc = 0;
        goto out;
    }
    /* merge (Alg.3; reading c14-c15): S1 = clamp(S0 + sum_g D_g) */
    for (size_t c = 0; c < cells; c++) {
        s->m[c] = (int32_t)(S0m[c] + Dm[c]);
        s->t[c] = (int32_t)(S0t[c] + Dt[c]);
    }
    s->stats[2] += clamp_cells(cells, s->m, s->t);
    recompute_sums(s, s->m, s->t, s->M, s->Tt, s->Q, s->T);
    if (nwaves == 0) break;
    }   /* blocks */
    s->sweep++;
    rc = 0;
out:
    free(shard); free(S0m); free(S0t); free(Lm); free(Lt); free(Dm); free(Dt);
    free(M); free(Tt); free(Q); free(T); free(newz); free(newr); free(rrem); free(kept); free(inwave); free(seen);
    free(lw); free(prob);
    return rc;
}

int or_sweep_par(ostate *s, int W, int G, const int32_t *force_zr, double *margin, int64_t max_tokens,
                 int32_t *own_zr) {
    return sweep_par_impl(s, W, G, -1, force_zr, margin, max_tokens, own_zr, NULL, NULL, 0);
}
/* the same with an exchange every E waves (NEXT-3 bounded staleness) */
int or_sweep_par_e(ostate *s, int W, int G, int E, const int32_t *force_zr, double *margin, int64_t max_tokens,
                   int32_t *own_zr) {
    return sweep_par_impl(s, W, G, -1, force_zr, margin, max_tokens, own_zr, NULL, NULL, E);
}

/* Distributed form of the same sweep: shard g runs its waves and returns its
 * net changes D_g (int32, [I*V*K]) without touching the global m, t ... */
int or_sweep_shard(ostate *s, int W, int G, int g, int32_t *Dm, int32_t *Dt) {
    if (g < 0 || g >= G || !Dm || !Dt) return -1;
    return sweep_par_impl(s, W, G, g, NULL, NULL, -1, NULL, Dm, Dt, 0);
}
/* ... and, once every rank holds sum_g D_g, the merge S1 = clamp(S0 + sum D). */
int or_merge(ostate *s, const int32_t *Dm, const int32_t *Dt) {
    size_t cells = (size_t)s->I * s->V * s->K;
    for (size_t c = 0; c < cells; c++) { s->m[c] += Dm[c]; s->t[c] += Dt[c]; }
    s->stats[2] += clamp_cells(cells, s->m, s->t);
    recompute_sums(s, s->m, s->t, s->M, s->Tt, s->Q, s->T);
    s->sweep++;
    return 0;
}

/* ------------------------------------------------------------------ */
/* queries                                                             */
/* ------------------------------------------------------------------ */
void or_get(const ostate *s, int32_t *z, uint8_t *r, int32_t *n, int32_t *m, int32_t *t, int32_t *Q) {
    size_t cells = (size_t)s->I * s->V * s->K;
    if (z) memcpy(z, s->z, sizeof(int32_t) * (size_t)s->N);
    if (r) memcpy(r, s->r, (size_t)s->N);
    if (n) memcpy(n, s->n, sizeof(int32_t) * (size_t)s->D * s->K);
    if (m) memcpy(m, s->m, sizeof(int32_t) * cells);
    if (t) memcpy(t, s->t, sizeof(int32_t) * cells);
    if (Q) for (size_t j = 0; j < (size_t)s->K * s->V; j++) Q[j] = (int32_t)s->Q[j];
}
uint32_t or_sweep_index(const ostate *s) { return s->sweep; }
void or_set_sweep_index(ostate *s, uint32_t sweep) { s->sweep = sweep; }
void or_stats(const ostate *s, int64_t *out) { memcpy(out, s->stats, sizeof(s->stats)); }

/* Normalised 2K-slot conditional of token p at the current state with the
 * given removal indicator.  Returns -1 if that removal is impossible
 * (r_rem = 0 with t = m, or r_rem = 1 with t = 1 < m: the keep case). */
int or_conditional(const ostate *s, int64_t p, int r_rem, double *prob) {
    size_t c = IDX3(s, s->group[p], s->word[p], s->z[p]);
    int64_t m = s->m[c], t = s->t[c];
    if (r_rem == 0 && t == m) return -1;
    if (r_rem == 1 && t == 1 && m > 1) return -1;
    double *lw = (double *)malloc(sizeof(double) * 2 * (size_t)s->K);
    if (!lw) return -2;
    log_weights(s, p, r_rem, s->n, s->m, s->t, s->M, s->Tt, s->Q, s->T, lw);
    normalise(2 * s->K, lw, prob);
    free(lw);
    return 0;
}

/* The decision token p would take in sweep `sweep` against the current state
 * (as wave-snapshot): info = {r_rem, keep, new z, new r}, *u = uniform,
 * prob = conditional (point mass on slot 2 k0 when kept), *margin as above. */
int or_debug_token(const ostate *s, int64_t p, uint32_t sweep, double *prob, int32_t *info, double *u, double *margin) {
    int K = s->K;
    size_t c = IDX3(s, s->group[p], s->word[p], s->z[p]);
    uint32_t x[4];
    rng_token(s->seed, (uint32_t)p, sweep, x);
    int keep, r = removal(x[0], s->m[c], s->t[c], &keep);
    info[0] = r; info[1] = keep;
    *u = u53(x);
    if (keep) {
        for (int j = 0; j < 2 * K; j++) prob[j] = 0.0;
        prob[2 * s->z[p]] = 1.0;
        info[2] = s->z[p]; info[3] = 1; *margin = 1.0;
        return 0;
    }
    int rc = or_conditional(s, p, r, prob);
    if (rc) return rc;
    int j = draw_slot(2 * K, prob, *u, margin);
    info[2] = j / 2; info[3] = (j % 2 == 0);
    return 0;
}

/* Training perplexity, P:1978-2007 with theta~, phi0~ and
 * phi^i~ (reading c16): exp(-sum_tok log sum_k theta_dk phi^i_kw / N). */
double or_perplexity(const ostate *s) {
    int K = s->K, V = s->V;
    double ll = 0.0;
    for (int64_t p = 0; p < s->N; p++) {
        int i = s->group[p], w = s->word[p], d = s->doc[p];
        double a = s->a[i], b = s->b[i];
        double asum = 0.0;
        for (int k = 0; k < K; k++) asum += s->alpha[(size_t)i * K + k];
        double pw = 0.0;
        for (int k = 0; k < K; k++) {
            double theta = ((double)s->n[(size_t)d * K + k] + s->alpha[(size_t)i * K + k]) / ((double)s->doclen[d] + asum);
            double phi0 = (s->beta + (double)s->Q[(size_t)k * V + w]) / ((double)V * s->beta + (double)s->T[k]);
            double Mk = (double)s->M[(size_t)i * K + k], Tk = (double)s->Tt[(size_t)i * K + k];
            size_t c = IDX3(s, i, w, k);
            double phii = ((double)s->m[c] - a * (double)s->t[c]) / (b + Mk) + (b + a * Tk) / (b + Mk) * phi0;
            pw += theta * phii;
        }
        ll += log(pw);
    }
    return exp(-ll / (double)s->N);
}

/* log p(W, Z, T | alpha, beta, a, b): the blocked-Gibbs joint
 * with identity P, summed over the prod C(m,t) seatings R per T
 * (Eq. SPDP-table-to-head):
 *   sum_{docs} [lnG(sum alpha) - lnG(sum alpha + L_d) + sum_k lnG(alpha+n_dk) - lnG(alpha)]
 * + sum_{i,k} [ln (b|a)_{t_ik.} - ln (b)_{m_ik.}] + sum_{i,k,w} ln S^{m_ikw}_{t_ikw, a}
 * + sum_k [lnG(V beta) - lnG(V beta + T_k) + sum_w lnG(beta + Q_kw) - lnG(beta)]. */
double or_log_joint(const ostate *s) {
    int I = s->I, V = s->V, K = s->K;
    double lp = 0.0;
    int32_t *dg = (int32_t *)malloc(sizeof(int32_t) * (size_t)s->D);
    for (int32_t d = 0; d < s->D; d++) dg[d] = -1;
    for (int64_t p = 0; p < s->N; p++) dg[s->doc[p]] = s->group[p];
    for (int32_t d = 0; d < s->D; d++) {
        if (dg[d] < 0) continue;
        int i = dg[d];
        double asum = 0.0;
        for (int k = 0; k < K; k++) asum += s->alpha[(size_t)i * K + k];
        lp += lgamma(asum) - lgamma(asum + (double)s->doclen[d]);
        for (int k = 0; k < K; k++) {
            double al = s->alpha[(size_t)i * K + k];
            lp += lgamma(al + (double)s->n[(size_t)d * K + k]) - lgamma(al);
        }
    }
    free(dg);
    for (int i = 0; i < I; i++)
        for (int k = 0; k < K; k++)
            lp += log_poch(s->b[i], s->a[i], s->Tt[(size_t)i * K + k]) - log_poch(s->b[i], 1.0, s->M[(size_t)i * K + k]);
    for (int i = 0; i < I; i++)
        for (int w = 0; w < V; w++)
            for (int k = 0; k < K; k++) {
                size_t c = IDX3(s, i, w, k);
                lp += stable_get(&s->tab[i], s->m[c], s->t[c]);
            }
    for (int k = 0; k < K; k++) {
        lp += lgamma((double)V * s->beta) - lgamma((double)V * s->beta + (double)s->T[k]);
        for (int w = 0; w < V; w++) lp += lgamma(s->beta + (double)s->Q[(size_t)k * V + w]) - lgamma(s->beta);
    }
    return lp;
}

/* Count invariants (north_star (4); SURVEY §8(c) "counts").  0 = all hold. */
int or_check_invariants(const ostate *s) {
    int I = s->I, V = s->V, K = s->K;
    size_t cells = (size_t)I * V * K;
    int rc = 0;
    int32_t *n = (int32_t *)calloc((size_t)s->D * K, sizeof(int32_t));
    int32_t *m = (int32_t *)calloc(cells, sizeof(int32_t));
    int64_t *M = (int64_t *)malloc(sizeof(int64_t) * (size_t)I * K), *Tt = (int64_t *)malloc(sizeof(int64_t) * (size_t)I * K);
    int64_t *Q = (int64_t *)malloc(sizeof(int64_t) * (size_t)K * V), *T = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
    if (!n || !m || !M || !Tt || !Q || !T) { rc = -2; goto out; }
    for (int64_t p = 0; p < s->N; p++) {
        n[(size_t)s->doc[p] * K + s->z[p]]++;
        m[IDX3(s, s->group[p], s->word[p], s->z[p])]++;
    }
    if (memcmp(n, s->n, sizeof(int32_t) * (size_t)s->D * K)) { rc = 1; goto out; }
    if (memcmp(m, s->m, sizeof(int32_t) * cells)) { rc = 2; goto out; }
    int64_t sm = 0;
    for (size_t c = 0; c < cells; c++) {
        sm += s->m[c];
        if (s->t[c] < 0 || s->t[c] > s->m[c]) { rc = 3; goto out; }
        if ((s->t[c] > 0) != (s->m[c] > 0)) { rc = 4; goto out; }
    }
    if (sm != s->N) { rc = 5; goto out; }
    recompute_sums(s, s->m, s->t, M, Tt, Q, T);
    if (memcmp(M, s->M, sizeof(int64_t) * (size_t)I * K) || memcmp(Tt, s->Tt, sizeof(int64_t) * (size_t)I * K) ||
        memcmp(Q, s->Q, sizeof(int64_t) * (size_t)K * V) || memcmp(T, s->T, sizeof(int64_t) * (size_t)K)) { rc = 6; goto out; }
out:
    free(n); free(m); free(M); free(Tt); free(Q); free(T);
    return rc;
}

/* p(w | doc d) = sum_k theta~_dk phi^i~_kw of the perplexity above (for the
 * normalisation pin: sum_w p(w|d) = 1). */
double or_word_prob(const ostate *s, int32_t d, int32_t w) {
    int K = s->K, V = s->V;
    int i = -1;
    for (int64_t p = 0; p < s->N; p++) if (s->doc[p] == d) { i = s->group[p]; break; }
    if (i < 0) return NAN;
    double a = s->a[i], b = s->b[i], asum = 0.0, pw = 0.0;
    for (int k = 0; k < K; k++) asum += s->alpha[(size_t)i * K + k];
    for (int k = 0; k < K; k++) {
        double theta = ((double)s->n[(size_t)d * K + k] + s->alpha[(size_t)i * K + k]) / ((double)s->doclen[d] + asum);
        double phi0 = (s->beta + (double)s->Q[(size_t)k * V + w]) / ((double)V * s->beta + (double)s->T[k]);
        double Mk = (double)s->M[(size_t)i * K + k], Tk = (double)s->Tt[(size_t)i * K + k];
        size_t c = IDX3(s, i, w, k);
        pw += theta * (((double)s->m[c] - a * (double)s->t[c]) / (b + Mk) + (b + a * Tk) / (b + Mk) * phi0);
    }
    return pw;
}

/* Run `nsweeps` sweeps (waves < 0: mode S; else mode P with `waves`, 1 shard)
 * and record after each sweep a code of the whole (z, t) state:
 * code = sum_p z_p K^p + K^N * sum_c t_c (tbase)^c over all I*V*K cells.
 * For tiny corpora only (the caller guarantees no int64 overflow). */
int or_chain_codes(ostate *s, int64_t nsweeps, int waves, int tbase, int64_t *codes) {
    size_t cells = (size_t)s->I * s->V * s->K;
    for (int64_t it = 0; it < nsweeps; it++) {
        int rc = (waves < 0) ? or_sweep_seq(s, -1) : or_sweep_par(s, waves, 1, NULL, NULL, -1, NULL);
        if (rc) return rc;
        int64_t code = 0, mul = 1;
        for (int64_t p = 0; p < s->N; p++) { code += mul * s->z[p]; mul *= s->K; }
        int64_t tc = 0, tm = 1;
        for (size_t c = 0; c < cells; c++) { tc += tm * s->t[c]; tm *= tbase; }
        codes[it] = code + mul * tc;
    }
    return 0;
}

/* ================================================================== */
/* NEXT-1: held-out evaluation                    */
/* ================================================================== */
/* Topic-word estimates of the current state (after convergence):
 *   phi0~_kw  = (beta + Q_kw) / (V beta + T_k)                  Eq. spdp-word-topic-estimate,
 *               identity P: sum_i sum_w q_{ikwv} = Q_kv;
 *   phi~^i_kw = (m_ikw - a_i t_ikw)/(b_i + m_ik.) + (b_i + a_i t_ik.)/(b_i + m_ik.) phi0~_kw
 *               Eq. spdp-group-word-topic-estimate, mixing weight of reading c16,
 *               identity P: sum_v p_{w,v} phi0~_kv = phi0~_kw. */
double or_phi0(const ostate *s, int k, int w) {
    return (s->beta + (double)s->Q[(size_t)k * s->V + w]) / ((double)s->V * s->beta + (double)s->T[k]);
}
double or_phi(const ostate *s, int i, int k, int w) {
    double a = s->a[i], b = s->b[i];
    double Mk = (double)s->M[(size_t)i * s->K + k], Tk = (double)s->Tt[(size_t)i * s->K + k];
    size_t c = IDX3(s, i, w, k);
    return ((double)s->m[c] - a * (double)s->t[c]) / (b + Mk) + (b + a * Tk) / (b + Mk) * or_phi0(s, k, w);
}

/* Fold-in of held-out documents (reading c21; the paper does not say how the
 * theta~ of a test document is obtained): collapsed Gibbs over
 * the held-out tokens' topics z only, with the trained phi~^i frozen as the
 * word likelihoods.  The held-out documents are independent given phi~, and
 * within a document the tokens are visited sequentially in canonical order:
 *   p(z_p = k | rest) ∝ (alpha_ik + n_dk^{-p}) phi~^i_{k w_p}      (LDA fold-in with phi~^i of P:1754).
 * Randomness: u = u53(Philox(seed; p, it, 1, 0)) for token p in iteration it;
 * the draw is k* = min{k : cdf_k > u} (reading c10 with K slots).
 * Initial z (z in/out holds -1 entries or a state): when init != 0,
 * z_p = floor(x0 K / 2^32) of Philox(seed; p, 0xFFFFFFFF, 1, 0).
 * force_z / margin / own: lock-step testing as in or_sweep_par (own = the
 * oracle's draw before it is replaced by force_z). */
/* the word likelihood phi~^i_{kw} used by the estimators: or_phi here, the
 * sparse-P version for NEXT-4 (or_sp_foldin / or_sp_heldout_perplexity) */
typedef double (*phi_fn)(const void *ctx, int i, int k, int w);
static double phi_identity(const void *ctx, int i, int k, int w) { return or_phi((const ostate *)ctx, i, k, w); }

static int foldin_impl(const ostate *s, phi_fn phi, const void *pctx, int64_t Nh, int32_t Dh, const int32_t *group,
                       const int32_t *doc, const int32_t *word, uint64_t seed, int32_t first_iter, int32_t iters,
                       int init, int32_t *z, const int32_t *force_z, double *margin, int32_t *own) {
    int K = s->K;
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (int64_t p = 0; p < Nh; p++) {
        if (group[p] < 0 || group[p] >= s->I || word[p] < 0 || word[p] >= s->V || doc[p] < 0 || doc[p] >= Dh) return -1;
        if (init) {
            uint32_t ctr[4] = {(uint32_t)p, 0xFFFFFFFFu, 1u, 0u}, x[4];
            or_philox(ctr, key, x);
            z[p] = (int32_t)(((uint64_t)x[0] * (uint64_t)K) >> 32);
        }
        if (z[p] < 0 || z[p] >= K) return -1;
    }
    int32_t *n = (int32_t *)calloc((size_t)Dh * K, sizeof(int32_t));
    double *w = (double *)malloc(sizeof(double) * (size_t)K), *prob = (double *)malloc(sizeof(double) * (size_t)K);
    if (!n || !w || !prob) { free(n); free(w); free(prob); return -2; }
    for (int64_t p = 0; p < Nh; p++) n[(size_t)doc[p] * K + z[p]]++;
    for (int32_t it = first_iter; it < first_iter + iters; it++) {
        for (int64_t p = 0; p < Nh; p++) {
            int i = group[p], d = doc[p];
            n[(size_t)d * K + z[p]]--;
            double tot = 0.0;
            for (int k = 0; k < K; k++) {
                w[k] = (s->alpha[(size_t)i * K + k] + (double)n[(size_t)d * K + k]) * phi(pctx, i, k, word[p]);
                tot += w[k];
            }
            for (int k = 0; k < K; k++) prob[k] = w[k] / tot;
            uint32_t ctr[4] = {(uint32_t)p, (uint32_t)it, 1u, 0u}, x[4];
            or_philox(ctr, key, x);
            double mg = 0.0;
            int k_new = draw_slot(K, prob, u53(x), &mg);
            if (margin) margin[p] = mg;
            if (own) own[p] = k_new;
            if (force_z) k_new = force_z[p];
            z[p] = k_new;
            n[(size_t)d * K + k_new]++;
        }
    }
    free(n); free(w); free(prob);
    return 0;
}
int or_foldin(const ostate *s, int64_t Nh, int32_t Dh, const int32_t *group, const int32_t *doc,
              const int32_t *word, uint64_t seed, int32_t first_iter, int32_t iters, int init, int32_t *z,
              const int32_t *force_z, double *margin, int32_t *own) {
    return foldin_impl(s, phi_identity, s, Nh, Dh, group, doc, word, seed, first_iter, iters, init, z, force_z,
                       margin, own);
}

/* Held-out perplexity (§3.2.2, reading c17 for the exponent):
 *   exp(- sum_p log sum_k theta~_dk phi~^i_{k w_p} / Nh),
 * theta~_dk = (n_dk + alpha_ik) / sum_k (n_dk + alpha_ik)   Eq. spdp-topic-doc-estimate
 * with n_dk counted from the held-out z.  theta (optional) receives [Dh*K]. */
static double heldout_impl(const ostate *s, phi_fn phi, const void *pctx, int64_t Nh, int32_t Dh,
                           const int32_t *group, const int32_t *doc, const int32_t *word, const int32_t *z,
                           double *theta) {
    int K = s->K;
    int32_t *n = (int32_t *)calloc((size_t)Dh * K, sizeof(int32_t));
    int32_t *len = (int32_t *)calloc((size_t)Dh, sizeof(int32_t));
    int32_t *dg = (int32_t *)malloc(sizeof(int32_t) * (size_t)Dh);
    if (!n || !len || !dg) { free(n); free(len); free(dg); return NAN; }
    for (int32_t d = 0; d < Dh; d++) dg[d] = 0;
    for (int64_t p = 0; p < Nh; p++) { n[(size_t)doc[p] * K + z[p]]++; len[doc[p]]++; dg[doc[p]] = group[p]; }
    if (theta)
        for (int32_t d = 0; d < Dh; d++) {
            int i = dg[d];
            double asum = 0.0;
            for (int k = 0; k < K; k++) asum += s->alpha[(size_t)i * K + k];
            for (int k = 0; k < K; k++)
                theta[(size_t)d * K + k] = ((double)n[(size_t)d * K + k] + s->alpha[(size_t)i * K + k]) / ((double)len[d] + asum);
        }
    double ll = 0.0;
    for (int64_t p = 0; p < Nh; p++) {
        int i = group[p], d = doc[p];
        double asum = 0.0;
        for (int k = 0; k < K; k++) asum += s->alpha[(size_t)i * K + k];
        double pw = 0.0;
        for (int k = 0; k < K; k++) {
            double th = ((double)n[(size_t)d * K + k] + s->alpha[(size_t)i * K + k]) / ((double)len[d] + asum);
            pw += th * phi(pctx, i, k, word[p]);
        }
        ll += log(pw);
    }
    free(n); free(len); free(dg);
    return exp(-ll / (double)Nh);
}
double or_heldout_perplexity(const ostate *s, int64_t Nh, int32_t Dh, const int32_t *group, const int32_t *doc,
                             const int32_t *word, const int32_t *z, double *theta) {
    return heldout_impl(s, phi_identity, s, Nh, Dh, group, doc, word, z, theta);
}

/* Hellinger distance between two discrete distributions (§4.2.6
 * compares topic models with it; the formula is not printed — reading c22:
 * the standard H(p,q) = sqrt(1 - sum_v sqrt(p_v q_v)), clamped into [0,1]). */
double or_hellinger(int64_t V, const double *p, const double *q) {
    double bc = 0.0;
    for (int64_t v = 0; v < V; v++) bc += sqrt(p[v] * q[v]);
    double h2 = 1.0 - bc;
    if (h2 < 0.0) h2 = 0.0;
    if (h2 > 1.0) h2 = 1.0;
    return sqrt(h2);
}

/* Topic alignment of two models on their base distributions phi0~ (reading c22):
 * dist[k*K + k'] = H(phi0~_A[k], phi0~_B[k']); greedy minimum-distance
 * matching: repeatedly take the smallest remaining distance (ties: smaller k,
 * then smaller k') whose row and column are both free; perm[k] = k'. */
typedef struct { double d; int k, kp; } pair_t;
static int pair_cmp(const void *x, const void *y) {
    const pair_t *a = (const pair_t *)x, *b = (const pair_t *)y;
    if (a->d != b->d) return a->d < b->d ? -1 : 1;
    if (a->k != b->k) return a->k < b->k ? -1 : 1;
    return (a->kp > b->kp) - (a->kp < b->kp);
}
void or_greedy_match(int K, const double *dist, int32_t *perm) {
    pair_t *pr = (pair_t *)malloc(sizeof(pair_t) * (size_t)K * K);
    char *ur = (char *)calloc((size_t)K, 1), *uc = (char *)calloc((size_t)K, 1);
    for (int k = 0; k < K; k++)
        for (int kp = 0; kp < K; kp++) { pr[(size_t)k * K + kp].d = dist[(size_t)k * K + kp]; pr[(size_t)k * K + kp].k = k; pr[(size_t)k * K + kp].kp = kp; }
    qsort(pr, (size_t)K * K, sizeof(pair_t), pair_cmp);
    for (size_t j = 0; j < (size_t)K * K; j++)
        if (!ur[pr[j].k] && !uc[pr[j].kp]) { ur[pr[j].k] = 1; uc[pr[j].kp] = 1; perm[pr[j].k] = pr[j].kp; }
    free(pr); free(ur); free(uc);
}
int or_topic_align(const ostate *A, const ostate *B, double *dist, int32_t *perm) {
    if (A->K != B->K || A->V != B->V) return -1;
    int K = A->K, V = A->V;
    double *pa = (double *)malloc(sizeof(double) * (size_t)V), *pb = (double *)malloc(sizeof(double) * (size_t)V);
    for (int k = 0; k < K; k++) {
        for (int w = 0; w < V; w++) pa[w] = or_phi0(A, k, w);
        for (int kp = 0; kp < K; kp++) {
            for (int w = 0; w < V; w++) pb[w] = or_phi0(B, kp, w);
            dist[(size_t)k * K + kp] = or_hellinger(V, pa, pb);
        }
    }
    free(pa); free(pb);
    or_greedy_match(K, dist, perm);
    return 0;
}

/* phi0 [K*V] and phi [I*K*V] (either may be NULL) of the current state. */
void or_topics(const ostate *s, double *phi0, double *phi) {
    for (int k = 0; k < s->K; k++)
        for (int w = 0; w < s->V; w++) {
            if (phi0) phi0[(size_t)k * s->V + w] = or_phi0(s, k, w);
            if (phi)
                for (int i = 0; i < s->I; i++) phi[((size_t)i * s->K + k) * s->V + w] = or_phi(s, i, k, w);
        }
}

/* ================================================================== */
/* NEXT-4: sparse non-identity transformation matrices P^i             */
/* ================================================================== */
/* The full SPDP of §2.4.6/§3.1: group
 * i's word distribution for topic k is PDP(a, b, P^i phi0_k), so a table of
 * restaurant (i,k) serving word w draws a *source* word v with probability
 * p_{i,w,v} phi0_{k,v}.  State: z, r per token; q_{i,k,w,v} = tables of
 * (i,k,w) whose source is v; t_{ikw} = sum_v q_{ikwv};
 * Q_{k,v} = sum_{i,w} q_{ikwv} (the shadow counts of Eq. r1);
 * T_k = sum_v Q_{kv}.  P^i is given per group as sparse rows: entries
 * e in [pptr[i*V+w], pptr[i*V+w+1]) with source pv[e] and weight pp[e];
 * the columns must sum to 1 (P^i phi0 is a distribution).
 *
 * Conditional (Alg.1 P:1698-1727 with Eq. r1's p_{i,w,v}): per topic k the
 * slots (k, r=1, e) for the row's entries e in order, then (k, r=0):
 *   r=0:   (alpha+n)/(b+M) (m-t+1)/(m+1) S^{m+1}_t/S^m_t
 *   r=1,e: p_e (alpha+n)(b+a Tt)/(b+M) (t+1)/(m+1) (beta+Q_{k,v_e})/(V beta+T_k) S^{m+1}_{t+1}/S^m_t
 * Removal (Alg.1 lines 3-9): r ~ Bernoulli(t/m) (reading c7); if r = 1 the
 * removed table is uniform among the cell's t tables, i.e. its source entry
 * e is the one where the integer j = floor(x3 t / 2^32) falls in the
 * cumulative q counts of the cell (reading c26); keep rule c5 unchanged.
 * Initial sources (reading c25): every table of a cell starts on the row's
 * entry of largest p (first on ties).
 * Wave merges (reading c24, the "error correction ... for q"): after a wave's
 * deltas, q_e <- max(q_e, 0); if m = 0 all q_e = 0; else if sum q = 0 the
 * largest-p entry gets one table; while sum q > m the largest q (first on
 * ties) loses one.  With P^i = identity all of this is the identity-P sampler
 * above, bit for bit (pinned). */
typedef struct {
    ostate *o;
    int32_t E;
    int32_t *pptr, *pv;
    double *pp;
    int32_t *q;          /* [E*K] */
    int64_t *Qs;         /* [K*V] */
    int32_t *best;       /* [I*V] entry of largest p in each row */
} spstate;

void or_sp_destroy(spstate *sp) {
    if (!sp) return;
    free(sp->pptr); free(sp->pv); free(sp->pp); free(sp->q); free(sp->Qs); free(sp->best);
    free(sp);
}

static void sp_recompute(spstate *sp) {
    ostate *s = sp->o;
    int I = s->I, V = s->V, K = s->K;
    memset(sp->Qs, 0, sizeof(int64_t) * (size_t)K * V);
    memset(s->M, 0, sizeof(int64_t) * (size_t)I * K);
    memset(s->Tt, 0, sizeof(int64_t) * (size_t)I * K);
    memset(s->T, 0, sizeof(int64_t) * (size_t)K);
    for (int i = 0; i < I; i++)
        for (int w = 0; w < V; w++)
            for (int k = 0; k < K; k++) {
                size_t c = IDX3(s, i, w, k);
                int32_t t = 0;
                for (int32_t e = sp->pptr[i * V + w]; e < sp->pptr[i * V + w + 1]; e++) {
                    int32_t qv = sp->q[(size_t)e * K + k];
                    t += qv;
                    sp->Qs[(size_t)k * V + sp->pv[e]] += qv;
                }
                s->t[c] = t;
                s->M[(size_t)i * K + k] += s->m[c];
                s->Tt[(size_t)i * K + k] += t;
                s->T[k] += t;
            }
}

/* o: a loaded oracle state (z, r, counts from or_load); its t become the q of
 * the rows' largest-p entries.  Returns NULL on invalid P. */
spstate *or_sp_create(ostate *o, const int32_t *pptr, const int32_t *pv, const double *pp) {
    int I = o->I, V = o->V, K = o->K;
    int32_t E = pptr[I * V];
    if (pptr[0] != 0 || E < I * V) return NULL;
    double *col = (double *)calloc((size_t)I * V, sizeof(double));
    for (int r = 0; r < I * V; r++) {
        if (pptr[r + 1] <= pptr[r]) { free(col); return NULL; }        /* every row needs a source */
        for (int32_t e = pptr[r]; e < pptr[r + 1]; e++) {
            if (pv[e] < 0 || pv[e] >= V || !(pp[e] > 0.0)) { free(col); return NULL; }
            col[(size_t)(r / V) * V + pv[e]] += pp[e];
        }
    }
    for (size_t c = 0; c < (size_t)I * V; c++)
        if (fabs(col[c] - 1.0) > 1e-9) { free(col); return NULL; }       /* columns sum to 1 */
    free(col);
    spstate *sp = (spstate *)calloc(1, sizeof(spstate));
    sp->o = o; sp->E = E;
    sp->pptr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(I * V + 1));
    sp->pv = (int32_t *)malloc(sizeof(int32_t) * (size_t)E);
    sp->pp = (double *)malloc(sizeof(double) * (size_t)E);
    sp->q = (int32_t *)calloc((size_t)E * K, sizeof(int32_t));
    sp->Qs = (int64_t *)calloc((size_t)K * V, sizeof(int64_t));
    sp->best = (int32_t *)malloc(sizeof(int32_t) * (size_t)I * V);
    memcpy(sp->pptr, pptr, sizeof(int32_t) * (size_t)(I * V + 1));
    memcpy(sp->pv, pv, sizeof(int32_t) * (size_t)E);
    memcpy(sp->pp, pp, sizeof(double) * (size_t)E);
    for (int r = 0; r < I * V; r++) {
        int32_t b = pptr[r];
        for (int32_t e = pptr[r]; e < pptr[r + 1]; e++) if (pp[e] > pp[b]) b = e;
        sp->best[r] = b;
    }
    for (int i = 0; i < I; i++)                                       /* reading c25 */
        for (int w = 0; w < V; w++)
            for (int k = 0; k < K; k++) sp->q[(size_t)sp->best[i * V + w] * K + k] = o->t[IDX3(o, i, w, k)];
    sp_recompute(sp);
    return sp;
}

/* log weights of the K (S+1) slots of token p (S = its row's entries), own
 * contribution removed: one customer of k0 and, when r_rem, the table whose
 * source entry is e_rem.  Slot of (k, r=1, e-th entry) = k(S+1) + e, (k, r=0) = k(S+1) + S. */
static void sp_log_weights(const spstate *sp, int64_t p, int r_rem, int32_t e_rem, const int32_t *n, const int32_t *m,
                           const int32_t *t, const int64_t *M, const int64_t *Tt, const int64_t *Qs, const int64_t *T,
                           double *lw) {
    const ostate *s = sp->o;
    int K = s->K, V = s->V;
    int i = s->group[p], w = s->word[p], d = s->doc[p], k0 = s->z[p];
    int32_t e0 = sp->pptr[i * V + w], S = sp->pptr[i * V + w + 1] - e0;
    double a = s->a[i], b = s->b[i], beta = s->beta;
    const stable_t *St = &s->tab[i];
    for (int k = 0; k < K; k++) {
        int own = (k == k0);
        double n_k = (double)n[(size_t)d * K + k] - own;
        int64_t m_k = m[IDX3(s, i, w, k)] - own;
        int64_t t_k = t[IDX3(s, i, w, k)] - own * r_rem;
        double M_k = (double)M[(size_t)i * K + k] - own;
        double Tt_k = (double)Tt[(size_t)i * K + k] - own * r_rem;
        double T_k = (double)T[k] - own * r_rem;
        double lS = stable_get(St, (int)m_k, (int)t_k);
        double base = log(s->alpha[(size_t)i * K + k] + n_k) - log(b + M_k);
        lw[(size_t)k * (S + 1) + S] = base + log((double)(m_k - t_k + 1)) - log((double)(m_k + 1))
                                      + stable_get(St, (int)m_k + 1, (int)t_k) - lS;
        double l1 = base + log(b + a * Tt_k) + log((double)(t_k + 1)) - log((double)(m_k + 1))
                    - log((double)V * beta + T_k) + stable_get(St, (int)m_k + 1, (int)t_k + 1) - lS;
        for (int32_t j = 0; j < S; j++) {
            int32_t e = e0 + j, v = sp->pv[e];
            double Q_kv = (double)Qs[(size_t)k * V + v] - ((own && r_rem && sp->pv[e_rem] == v) ? 1.0 : 0.0);
            lw[(size_t)k * (S + 1) + j] = l1 + log(sp->pp[e]) + log(beta + Q_kv);
        }
    }
}

/* source entry of the removed table: j = floor(x3 t / 2^32) in the cumulative q of the cell (reading c26) */
static int32_t sp_removed_entry(const spstate *sp, int i, int w, int k, uint32_t x3, int32_t t) {
    int K = sp->o->K, V = sp->o->V;
    int64_t j = (int64_t)(((uint64_t)x3 * (uint64_t)t) >> 32), cum = 0;
    for (int32_t e = sp->pptr[i * V + w]; e < sp->pptr[i * V + w + 1]; e++) {
        cum += sp->q[(size_t)e * K + k];
        if (cum > j) return e;
    }
    return sp->pptr[i * V + w + 1] - 1;
}

static int32_t sp_max_row(const spstate *sp) {
    int32_t mx = 1;
    for (int r = 0; r < sp->o->I * sp->o->V; r++)
        if (sp->pptr[r + 1] - sp->pptr[r] > mx) mx = sp->pptr[r + 1] - sp->pptr[r];
    return mx;
}

/* Mode S: Alg.1 with the source variables (sequential, exact). */
int or_sp_sweep_seq(spstate *sp) {
    ostate *s = sp->o;
    int K = s->K, V = s->V;
    int32_t Smax = sp_max_row(sp);
    double *lw = (double *)malloc(sizeof(double) * (size_t)K * (Smax + 1));
    double *prob = (double *)malloc(sizeof(double) * (size_t)K * (Smax + 1));
    if (!lw || !prob) { free(lw); free(prob); return -2; }
    memset(s->stats, 0, sizeof(s->stats));
    for (int64_t p = 0; p < s->N; p++) {
        int i = s->group[p], w = s->word[p], d = s->doc[p], k = s->z[p];
        int32_t e0 = sp->pptr[i * V + w], S = sp->pptr[i * V + w + 1] - e0;
        size_t c = IDX3(s, i, w, k);
        uint32_t x[4];
        rng_token(s->seed, (uint32_t)p, s->sweep, x);
        int keep, r = removal(x[0], s->m[c], s->t[c], &keep);
        if (keep) { s->r[p] = 1; s->stats[0]++; continue; }
        int32_t er = r ? sp_removed_entry(sp, i, w, k, x[3], s->t[c]) : e0;
        sp_log_weights(sp, p, r, er, s->n, s->m, s->t, s->M, s->Tt, sp->Qs, s->T, lw);
        s->n[(size_t)d * K + k]--; s->m[c]--; s->M[(size_t)i * K + k]--;
        if (r) {
            s->t[c]--; s->Tt[(size_t)i * K + k]--; s->T[k]--;
            sp->q[(size_t)er * K + k]--; sp->Qs[(size_t)k * V + sp->pv[er]]--;
        }
        int ns = K * (S + 1);
        normalise(ns, lw, prob);
        int j = draw_slot(ns, prob, u53(x), NULL);
        int kn = j / (S + 1), within = j % (S + 1), rn = within < S;
        size_t cn = IDX3(s, i, w, kn);
        s->n[(size_t)d * K + kn]++; s->m[cn]++; s->M[(size_t)i * K + kn]++;
        if (rn) {
            int32_t e = e0 + within;
            s->t[cn]++; s->Tt[(size_t)i * K + kn]++; s->T[kn]++;
            sp->q[(size_t)e * K + kn]++; sp->Qs[(size_t)kn * V + sp->pv[e]]++;
        }
        if (kn != k) s->stats[1]++;
        s->z[p] = kn; s->r[p] = (uint8_t)rn;
    }
    s->sweep++;
    free(lw); free(prob);
    return 0;
}

/* Mode P on one shard: waves against the wave-start snapshot, then the
 * wave's deltas and the q correction (reading c24).  force (optional, [N]):
 * lock-step replay of another sampler's draws, as slot index
 * (k (S+1) + within); own/margin as in or_sweep_par. */
static int sp_waves(spstate *sp, int W, const int32_t *shard, int g, const int32_t *force, double *margin,
                    int32_t *own);
int or_sp_sweep_par(spstate *sp, int W, const int32_t *force, double *margin, int32_t *own) {
    int rc = sp_waves(sp, W, NULL, 0, force, margin, own);
    if (rc == 0) sp->o->sweep++;
    return rc;
}

/* the waves of one shard (shard == NULL: every token) against the current arrays of sp */
static int sp_waves(spstate *sp, int W, const int32_t *shard, int g, const int32_t *force, double *margin,
                    int32_t *own) {
    ostate *s = sp->o;
    int I = s->I, V = s->V, K = s->K;
    int64_t N = s->N;
    size_t cells = (size_t)I * V * K;
    int32_t Smax = sp_max_row(sp);
    if (W < 1) return -1;
    if (!shard) memset(s->stats, 0, sizeof(s->stats));
    int32_t *m0 = (int32_t *)malloc(sizeof(int32_t) * cells), *t0 = (int32_t *)malloc(sizeof(int32_t) * cells);
    int64_t *M0 = (int64_t *)malloc(sizeof(int64_t) * (size_t)I * K), *Tt0 = (int64_t *)malloc(sizeof(int64_t) * (size_t)I * K);
    int64_t *Q0 = (int64_t *)malloc(sizeof(int64_t) * (size_t)K * V), *T0 = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
    int32_t *dq = (int32_t *)calloc((size_t)sp->E * K, sizeof(int32_t));
    int32_t *dm = (int32_t *)calloc(cells, sizeof(int32_t));
    int32_t *slot = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1)), *erem = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    int8_t *rr = (int8_t *)malloc((size_t)(N + 1)), *kept = (int8_t *)malloc((size_t)(N + 1));
    double *lw = (double *)malloc(sizeof(double) * (size_t)K * (Smax + 1)), *prob = (double *)malloc(sizeof(double) * (size_t)K * (Smax + 1));
    int rc = -2;
    if (!m0 || !t0 || !M0 || !Tt0 || !Q0 || !T0 || !dq || !dm || !slot || !erem || !rr || !kept || !lw || !prob) goto out;
    int32_t maxlen = 0;
    for (int32_t d = 0; d < s->D; d++) if (s->doclen[d] > maxlen) maxlen = s->doclen[d];
    int64_t nwaves = W < maxlen ? W : maxlen;
    for (int64_t wave = 0; wave < nwaves; wave++) {
        memcpy(m0, s->m, sizeof(int32_t) * cells); memcpy(t0, s->t, sizeof(int32_t) * cells);
        memcpy(M0, s->M, sizeof(int64_t) * (size_t)I * K); memcpy(Tt0, s->Tt, sizeof(int64_t) * (size_t)I * K);
        memcpy(Q0, sp->Qs, sizeof(int64_t) * (size_t)K * V); memcpy(T0, s->T, sizeof(int64_t) * (size_t)K);
        /* (1) every token of the wave decides against the wave-start snapshot */
        for (int64_t p = 0; p < N; p++) {
            if (s->pos[p] % W != wave) continue;
            if (shard && shard[s->doc[p]] != g) continue;
            int i = s->group[p], w = s->word[p], k0 = s->z[p];
            int32_t e0 = sp->pptr[i * V + w], S = sp->pptr[i * V + w + 1] - e0;
            size_t c = IDX3(s, i, w, k0);
            uint32_t x[4];
            rng_token(s->seed, (uint32_t)p, s->sweep, x);
            int keep, r = removal(x[0], m0[c], t0[c], &keep);
            rr[p] = (int8_t)r; kept[p] = (int8_t)keep;
            if (keep) { slot[p] = -1; if (own) own[p] = -1; continue; }
            /* the removed table's source from the snapshot's q (dq holds only this wave's deltas: still 0 here) */
            erem[p] = r ? sp_removed_entry(sp, i, w, k0, x[3], t0[c]) : e0;
            sp_log_weights(sp, p, r, erem[p], s->n, m0, t0, M0, Tt0, Q0, T0, lw);
            int ns = K * (S + 1);
            normalise(ns, lw, prob);
            int j = draw_slot(ns, prob, u53(x), margin ? &margin[p] : NULL);
            if (own) own[p] = j;
            if (force && force[p] >= 0) { if (force[p] != j) s->stats[3]++; j = force[p]; }
            slot[p] = j;
        }
        /* (2) apply the wave's deltas, correct q (reading c24), recompute t and the sums */
        for (int64_t p = 0; p < N; p++) {
            if (s->pos[p] % W != wave) continue;
            if (shard && shard[s->doc[p]] != g) continue;
            if (kept[p]) { s->r[p] = 1; s->stats[0]++; continue; }
            int i = s->group[p], w = s->word[p], d = s->doc[p], k0 = s->z[p];
            int32_t e0 = sp->pptr[i * V + w], S = sp->pptr[i * V + w + 1] - e0;
            int kn = slot[p] / (S + 1), within = slot[p] % (S + 1), rn = within < S;
            s->n[(size_t)d * K + k0]--; s->n[(size_t)d * K + kn]++;
            dm[IDX3(s, i, w, k0)]--; dm[IDX3(s, i, w, kn)]++;
            if (rr[p]) dq[(size_t)erem[p] * K + k0]--;
            if (rn) dq[(size_t)(e0 + within) * K + kn]++;
            if (kn != k0) s->stats[1]++;
            s->z[p] = kn; s->r[p] = (uint8_t)rn;
        }
        for (int i = 0; i < I; i++)
            for (int w = 0; w < V; w++)
                for (int k = 0; k < K; k++) {
                    size_t c = IDX3(s, i, w, k);
                    int32_t eb = sp->pptr[i * V + w], ee = sp->pptr[i * V + w + 1];
                    int changed = 0, any = dm[c] != 0;
                    for (int32_t e = eb; e < ee; e++) any |= dq[(size_t)e * K + k] != 0;
                    if (!any) continue;
                    s->m[c] += dm[c]; dm[c] = 0;
                    int32_t t = 0;
                    for (int32_t e = eb; e < ee; e++) {
                        int32_t *qe = &sp->q[(size_t)e * K + k];
                        *qe += dq[(size_t)e * K + k]; dq[(size_t)e * K + k] = 0;
                        if (*qe < 0) { *qe = 0; changed = 1; }
                        t += *qe;
                    }
                    if (s->m[c] == 0) {
                        for (int32_t e = eb; e < ee; e++) if (sp->q[(size_t)e * K + k]) { sp->q[(size_t)e * K + k] = 0; changed = 1; }
                    } else if (t == 0) {
                        sp->q[(size_t)sp->best[i * V + w] * K + k] = 1; changed = 1;
                    } else {
                        while (t > s->m[c]) {
                            int32_t eb2 = eb;
                            for (int32_t e = eb; e < ee; e++) if (sp->q[(size_t)e * K + k] > sp->q[(size_t)eb2 * K + k]) eb2 = e;
                            sp->q[(size_t)eb2 * K + k]--; t--; changed = 1;
                        }
                    }
                    s->stats[2] += changed;
                }
        sp_recompute(sp);
    }
    rc = 0;
out:
    free(m0); free(t0); free(M0); free(Tt0); free(Q0); free(T0); free(dq); free(dm); free(slot); free(erem); free(rr);
    free(kept); free(lw); free(prob);
    return rc;
}

/* state read-out: q [E*K], Qs [K*V] (t, m, n, z, r through or_get on sp->o) */
void or_sp_get(const spstate *sp, int32_t *q, int64_t *Qs) {
    if (q) memcpy(q, sp->q, sizeof(int32_t) * (size_t)sp->E * sp->o->K);
    if (Qs) memcpy(Qs, sp->Qs, sizeof(int64_t) * (size_t)sp->o->K * sp->o->V);
}
/* set the sources (q) of the current state (tests: enumeration of (z, t, q) states) */
int or_sp_set_q(spstate *sp, const int32_t *q) {
    memcpy(sp->q, q, sizeof(int32_t) * (size_t)sp->E * sp->o->K);
    sp_recompute(sp);
    return 0;
}
/* normalised conditional of token p after removing it with (r_rem, e_rem) (tests) */
int or_sp_conditional(const spstate *sp, int64_t p, int r_rem, int32_t e_rem, double *prob) {
    const ostate *s = sp->o;
    int i = s->group[p], w = s->word[p], k0 = s->z[p];
    size_t c = IDX3(s, i, w, k0);
    int32_t e0 = sp->pptr[i * s->V + w], S = sp->pptr[i * s->V + w + 1] - e0;
    if (r_rem && (s->t[c] < 1 || sp->q[(size_t)e_rem * s->K + k0] < 1 || (s->t[c] == 1 && s->m[c] > 1))) return -1;
    if (!r_rem && s->t[c] == s->m[c]) return -1;
    double *lw = (double *)malloc(sizeof(double) * (size_t)s->K * (S + 1));
    sp_log_weights(sp, p, r_rem, r_rem ? e_rem : e0, s->n, s->m, s->t, s->M, s->Tt, sp->Qs, s->T, lw);
    normalise(s->K * (S + 1), lw, prob);
    free(lw);
    return 0;
}
/* (z, q) code after each of nsweeps sequential (W < 0) or wave (W >= 1) sweeps (tests; tiny corpora) */
int or_sp_chain_codes(spstate *sp, int64_t nsweeps, int W, int qbase, int64_t *codes) {
    ostate *s = sp->o;
    for (int64_t it = 0; it < nsweeps; it++) {
        int rc = (W < 0) ? or_sp_sweep_seq(sp) : or_sp_sweep_par(sp, W, NULL, NULL, NULL);
        if (rc) return rc;
        int64_t code = 0, mul = 1;
        for (int64_t p = 0; p < s->N; p++) { code += mul * s->z[p]; mul *= s->K; }
        int64_t qc = 0, qm = 1;
        for (int64_t j = 0; j < (int64_t)sp->E * s->K; j++) { qc += qm * sp->q[j]; qm *= qbase; }
        codes[it] = code + mul * qc;
    }
    return 0;
}

/* NEXT-4 estimators: phi0~_{kv} = (beta + Q_kv)/(V beta + T_k) (P:1753 with the
 * sparse shadow counts) and phi~^i_{kw} of P:1754 with its printed
 * sum_v p^i_{w,v} phi0~_{kv} (reading c16 for the mixing weight).  Rows of
 * phi~^i sum to 1 because the columns of P^i do. */
double or_sp_phi0(const spstate *sp, int k, int v) {
    const ostate *s = sp->o;
    return (s->beta + (double)sp->Qs[(size_t)k * s->V + v]) / ((double)s->V * s->beta + (double)s->T[k]);
}
double or_sp_phi(const spstate *sp, int i, int k, int w) {
    const ostate *s = sp->o;
    double a = s->a[i], b = s->b[i];
    double Mk = (double)s->M[(size_t)i * s->K + k], Tk = (double)s->Tt[(size_t)i * s->K + k];
    size_t c = IDX3(s, i, w, k);
    double base = 0.0;
    for (int32_t e = sp->pptr[i * s->V + w]; e < sp->pptr[i * s->V + w + 1]; e++) base += sp->pp[e] * or_sp_phi0(sp, k, sp->pv[e]);
    return ((double)s->m[c] - a * (double)s->t[c]) / (b + Mk) + (b + a * Tk) / (b + Mk) * base;
}
static double phi_sparse(const void *ctx, int i, int k, int w) { return or_sp_phi((const spstate *)ctx, i, k, w); }
void or_sp_topics(const spstate *sp, double *phi0, double *phi) {
    const ostate *s = sp->o;
    for (int k = 0; k < s->K; k++)
        for (int w = 0; w < s->V; w++) {
            if (phi0) phi0[(size_t)k * s->V + w] = or_sp_phi0(sp, k, w);
            if (phi)
                for (int i = 0; i < s->I; i++) phi[((size_t)i * s->K + k) * s->V + w] = or_sp_phi(sp, i, k, w);
        }
}
int or_sp_foldin(const spstate *sp, int64_t Nh, int32_t Dh, const int32_t *group, const int32_t *doc,
                 const int32_t *word, uint64_t seed, int32_t first_iter, int32_t iters, int init, int32_t *z,
                 const int32_t *force_z, double *margin, int32_t *own) {
    return foldin_impl(sp->o, phi_sparse, sp, Nh, Dh, group, doc, word, seed, first_iter, iters, init, z, force_z,
                       margin, own);
}
double or_sp_heldout_perplexity(const spstate *sp, int64_t Nh, int32_t Dh, const int32_t *group, const int32_t *doc,
                                const int32_t *word, const int32_t *z, double *theta) {
    return heldout_impl(sp->o, phi_sparse, sp, Nh, Dh, group, doc, word, z, theta);
}
/* training perplexity (P:1978-2007 on the training tokens, theta~ from n_d) */
double or_sp_perplexity(const spstate *sp) {
    const ostate *s = sp->o;
    return heldout_impl(s, phi_sparse, sp, s->N, s->D, s->group, s->doc, s->word, s->z, NULL);
}

/* Mode P over G shards (NEXT-4 on several GPUs): every shard samples its
 * documents' waves from the sweep-start state (its own replica of m, q and the
 * derived counts), then S1 = S0 + sum_g (L_g - S0) on m and q, corrected by
 * reading c24 on every cell, t, Q and the sums recomputed (Alg.3
 * with the sources). */
int or_sp_sweep_shards(spstate *sp, int W, int G) {
    ostate *s = sp->o;
    int I = s->I, V = s->V, K = s->K;
    size_t cells = (size_t)I * V * K, qn = (size_t)sp->E * K;
    if (G < 1 || W < 1) return -1;
    int32_t *shard = (int32_t *)malloc(sizeof(int32_t) * (size_t)s->D);
    int32_t *m0 = (int32_t *)malloc(sizeof(int32_t) * cells), *q0 = (int32_t *)malloc(sizeof(int32_t) * qn);
    int64_t *Dm = (int64_t *)calloc(cells, sizeof(int64_t)), *Dq = (int64_t *)calloc(qn, sizeof(int64_t));
    int32_t *Lm = (int32_t *)malloc(sizeof(int32_t) * cells), *Lt = (int32_t *)malloc(sizeof(int32_t) * cells);
    int32_t *Lq = (int32_t *)malloc(sizeof(int32_t) * qn);
    int64_t *LM = (int64_t *)malloc(sizeof(int64_t) * (size_t)I * K), *LTt = (int64_t *)malloc(sizeof(int64_t) * (size_t)I * K);
    int64_t *LQ = (int64_t *)malloc(sizeof(int64_t) * (size_t)K * V), *LT = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
    int rc = -2;
    if (!shard || !m0 || !q0 || !Dm || !Dq || !Lm || !Lt || !Lq || !LM || !LTt || !LQ || !LT) goto out;
    or_partition(s, G, shard);
    memcpy(m0, s->m, sizeof(int32_t) * cells);
    memcpy(q0, sp->q, sizeof(int32_t) * qn);
    memset(s->stats, 0, sizeof(s->stats));
    for (int g = 0; g < G; g++) {
        int32_t *gm = s->m, *gt = s->t, *gq = sp->q;
        int64_t *gM = s->M, *gTt = s->Tt, *gQ = sp->Qs, *gT = s->T;
        memcpy(Lm, m0, sizeof(int32_t) * cells);
        memcpy(Lq, q0, sizeof(int32_t) * qn);
        s->m = Lm; s->t = Lt; sp->q = Lq; s->M = LM; s->Tt = LTt; sp->Qs = LQ; s->T = LT;
        sp_recompute(sp);                                  /* the shard's replica of the sweep-start state */
        int r = sp_waves(sp, W, shard, g, NULL, NULL, NULL);
        for (size_t c = 0; c < cells; c++) Dm[c] += Lm[c] - m0[c];
        for (size_t j = 0; j < qn; j++) Dq[j] += Lq[j] - q0[j];
        s->m = gm; s->t = gt; sp->q = gq; s->M = gM; s->Tt = gTt; sp->Qs = gQ; s->T = gT;
        if (r) { rc = r; goto out; }
    }
    /* merge + correction (reading c24) on every cell */
    for (size_t c = 0; c < cells; c++) s->m[c] = (int32_t)(m0[c] + Dm[c]);
    for (size_t j = 0; j < qn; j++) sp->q[j] = (int32_t)(q0[j] + Dq[j]);
    for (int i = 0; i < I; i++)
        for (int w = 0; w < V; w++)
            for (int k = 0; k < K; k++) {
                size_t c = IDX3(s, i, w, k);
                int32_t eb = sp->pptr[i * V + w], ee = sp->pptr[i * V + w + 1];
                int changed = 0;
                int32_t t = 0;
                for (int32_t e = eb; e < ee; e++) {
                    int32_t *qe = &sp->q[(size_t)e * K + k];
                    if (*qe < 0) { *qe = 0; changed = 1; }
                    t += *qe;
                }
                if (s->m[c] == 0) {
                    for (int32_t e = eb; e < ee; e++) if (sp->q[(size_t)e * K + k]) { sp->q[(size_t)e * K + k] = 0; changed = 1; }
                } else if (t == 0) {
                    sp->q[(size_t)sp->best[i * V + w] * K + k] = 1; changed = 1;
                } else {
                    while (t > s->m[c]) {
                        int32_t eb2 = eb;
                        for (int32_t e = eb; e < ee; e++) if (sp->q[(size_t)e * K + k] > sp->q[(size_t)eb2 * K + k]) eb2 = e;
                        sp->q[(size_t)eb2 * K + k]--; t--; changed = 1;
                    }
                }
                s->stats[2] += changed;
            }
    sp_recompute(sp);
    s->sweep++;
    rc = 0;
out:
    free(shard); free(m0); free(q0); free(Dm); free(Dq); free(Lm); free(Lt); free(Lq); free(LM); free(LTt); free(LQ); free(LT);
    return rc;
}

/* log p(W, Z, T, Q) with sparse P^i (P:1649-1660 summed over the seatings R and
 * the per-table source orders V consistent with (T, Q)): the identity-P joint
 * above with Q_kv = sum_{i,w} q_{ikwv} in the shadow term, plus, per cell,
 * ln multinomial(t; q) + sum_e q_e ln p_e. */
double or_sp_log_joint(const spstate *sp) {
    ostate *s = sp->o;
    int64_t *Qsave = s->Q;
    s->Q = sp->Qs;                              /* same [K*V] layout */
    double lp = or_log_joint(s);
    s->Q = Qsave;
    int I = s->I, V = s->V, K = s->K;
    for (int i = 0; i < I; i++)
        for (int w = 0; w < V; w++)
            for (int k = 0; k < K; k++) {
                size_t c = IDX3(s, i, w, k);
                lp += lgamma((double)s->t[c] + 1.0);
                for (int32_t e = sp->pptr[i * V + w]; e < sp->pptr[i * V + w + 1]; e++) {
                    int32_t qv = sp->q[(size_t)e * K + k];
                    lp += -lgamma((double)qv + 1.0) + (double)qv * log(sp->pp[e]);
                }
            }
    return lp;
}
