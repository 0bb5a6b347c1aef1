/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the BASELINE.json bench
 * inputs and bulk k-hop counts at bench scale.
 *
 * Part of liboracle.so (with khop_oracle.c). It is the checker and the
 * reference arm's input preparation: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product
 * (paper_1905_01294_b200, libmgk.so) never links or calls it, and the
 * reference arm uses it so that arm maps no product library.
 *
 *   orc_gen_bench_csr   the BASELINE.json graphs: the
 *                       reference's per-edge R-MAT recipe (bench.cpp:107-137:
 *                       one top-53-bit mt19937_64 draw per level, quadrant
 *                       descent), run in 65,536-edge chunks, chunk c with its
 *                       own mt19937_64 seeded splitmix64(seed*K + c); self
 *                       loops dropped; the edge set is the first
 *                       `target_unique` DISTINCT keys of that stream in
 *                       stream order (target 0: exactly edge_factor << scale
 *                       raw draws, deduplicated); ids relabelled by a seeded
 *                       Fisher-Yates (relabel 1: all ids, 2: non-isolated ids
 *                       renumbered in id order first). A separate restatement
 *                       of the product's generator (mgk_gen_rmat_csr /
 *                       mgk_graph_gen_rmat), pinned equal to it by
 *                       tests/test_bench_oracle.py and tests/test_gpu_configs.py.
 *   orc_pick_seeds_u32  bench.cpp:200-218 over a uint32 CSR (eligible = ids
 *                       with a non-empty row, partial Fisher-Yates with
 *                       rejection-sampled mt19937_64 draws)
 *   orc_khop_many       k_hop_count (execute.cpp:347-375: masked level
 *                       synchronous expansion, early exit on an empty
 *                       frontier; exact = |F_k|, cumulative = |visited|-1)
 *                       for many seeds on all host threads, plus the
 *                       SURVEY.md §8(d) work model per seed (E(s,k), level
 *                       sizes) — the parity checker at G2 / G4 scale.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* from khop_oracle.c */
typedef struct {
    uint64_t mt[312];
    int mti;
} orc_mt;
void orc_mt_seed(orc_mt* s, uint64_t seed);
uint64_t orc_mt_next(orc_mt* s);

#define CHUNK_EDGES 65536ULL
#define SENTINEL UINT64_MAX

/* ---- a tiny fork/join pool ---------------------------------------------- */
typedef void (*par_fn)(void* ctx, uint64_t lo, uint64_t hi, unsigned t);
typedef struct {
    par_fn fn;
    void* ctx;
    uint64_t lo, hi;
    unsigned t;
} par_job;

static void* par_tramp(void* p) {
    par_job* j = (par_job*)p;
    j->fn(j->ctx, j->lo, j->hi, j->t);
    return NULL;
}

static unsigned g_threads = 0;
static unsigned nthreads(void) {
    if (g_threads) return g_threads;
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n < 1 ? 1u : (n > 256 ? 256u : (unsigned)n);
}

void orc_set_threads(unsigned t) { g_threads = t; }

/* split [0, n) into nt contiguous ranges, one thread each */
static void par_for(uint64_t n, unsigned nt, par_fn fn, void* ctx) {
    if (nt <= 1 || n < 2) {
        fn(ctx, 0, n, 0);
        return;
    }
    if (nt > n) nt = (unsigned)n;
    pthread_t th[256];
    par_job jobs[256];
    const uint64_t step = (n + nt - 1) / nt;
    unsigned used = 0;
    for (unsigned t = 0; t < nt; ++t) {
        uint64_t lo = t * step, hi = lo + step > n ? n : lo + step;
        if (lo >= hi) break;
        jobs[t] = (par_job){fn, ctx, lo, hi, t};
        pthread_create(&th[t], NULL, par_tramp, &jobs[t]);
        used++;
    }
    for (unsigned t = 0; t < used; ++t) pthread_join(th[t], NULL);
}

/* ---- parallel LSD radix sort of uint64 keys (key_bits significant) ------- */
#define RBITS 11
#define RBUCKETS (1u << RBITS)
typedef struct {
    uint64_t *src, *dst;
    uint64_t n;
    int shift;
    unsigned nt;
    uint64_t* hist; /* [nt][RBUCKETS] */
} rs_ctx;

static void rs_hist(void* p, uint64_t lo, uint64_t hi, unsigned t) {
    rs_ctx* c = (rs_ctx*)p;
    uint64_t* h = c->hist + (uint64_t)t * RBUCKETS;
    memset(h, 0, RBUCKETS * sizeof(uint64_t));
    for (uint64_t i = lo; i < hi; ++i) h[(c->src[i] >> c->shift) & (RBUCKETS - 1)]++;
}

static void rs_scatter(void* p, uint64_t lo, uint64_t hi, unsigned t) {
    rs_ctx* c = (rs_ctx*)p;
    uint64_t* pos = c->hist + (uint64_t)t * RBUCKETS;
    for (uint64_t i = lo; i < hi; ++i) {
        const uint64_t k = c->src[i];
        c->dst[pos[(k >> c->shift) & (RBUCKETS - 1)]++] = k;
    }
}

static int cmp_u64(const void* x, const void* y) {
    const uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
    return a < b ? -1 : a > b;
}

/* sorts v[0..n) ascending; tmp has n entries; returns the buffer holding the
 * result (v or tmp) */
static uint64_t* radix_sort(uint64_t* v, uint64_t* tmp, uint64_t n, int key_bits) {
    if (n < (1u << 16)) {
        qsort(v, n, 8, cmp_u64);
        return v;
    }
    const unsigned nt = nthreads();
    rs_ctx c = {v, tmp, n, 0, nt, (uint64_t*)malloc((size_t)nt * RBUCKETS * sizeof(uint64_t))};
    for (int shift = 0; shift < key_bits; shift += RBITS) {
        c.shift = shift;
        /* same contiguous split for both phases (stable) */
        par_for(n, nt, rs_hist, &c);
        const uint64_t step = (n + nt - 1) / nt;
        unsigned used = (unsigned)((n + step - 1) / step);
        uint64_t acc = 0;
        for (unsigned b = 0; b < RBUCKETS; ++b)
            for (unsigned t = 0; t < used; ++t) {
                uint64_t* h = c.hist + (uint64_t)t * RBUCKETS + b;
                const uint64_t x = *h;
                *h = acc;
                acc += x;
            }
        par_for(n, nt, rs_scatter, &c);
        uint64_t* s = c.src;
        c.src = c.dst;
        c.dst = s;
    }
    free(c.hist);
    return c.src;
}

static uint64_t unique_sorted(uint64_t* v, uint64_t n) {
    uint64_t w = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (w == 0 || v[i] != v[w - 1]) v[w++] = v[i];
    return w;
}

/* ---- the chunked edge stream ----------------------------------------------- */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

typedef struct {
    uint32_t scale;
    double a, ab, abc;
    uint64_t rng_seed;
    uint64_t chunk0;   /* first chunk of this batch */
    uint64_t raw_end;  /* total raw draws (target 0) or UINT64_MAX */
    uint64_t* out;     /* [nchunks * CHUNK_EDGES]: key, or SENTINEL for a loop / past the end */
} gen_ctx;

/* bench.cpp:107-137, one chunk: CHUNK_EDGES draws from its own stream */
static void gen_chunks(void* p, uint64_t lo, uint64_t hi, unsigned t) {
    (void)t;
    gen_ctx* c = (gen_ctx*)p;
    orc_mt rng;
    for (uint64_t j = lo; j < hi; ++j) {
        const uint64_t chunk = c->chunk0 + j;
        orc_mt_seed(&rng, splitmix64(c->rng_seed * 0x2545F4914F6CDD1DULL + chunk));
        uint64_t* o = c->out + j * CHUNK_EDGES;
        for (uint64_t e = 0; e < CHUNK_EDGES; ++e) {
            if (chunk * CHUNK_EDGES + e >= c->raw_end) {
                o[e] = SENTINEL;
                continue;
            }
            uint32_t s = 0, d = 0;
            for (uint32_t level = 0; level < c->scale; ++level) {
                const double r = (double)(orc_mt_next(&rng) >> 11) * 0x1.0p-53;
                uint32_t sb = 0, db = 0;
                if (r < c->a) {
                } else if (r < c->ab) {
                    db = 1;
                } else if (r < c->abc) {
                    sb = 1;
                } else {
                    sb = 1;
                    db = 1;
                }
                s = (s << 1) | sb;
                d = (d << 1) | db;
            }
            o[e] = s == d ? SENTINEL : (((uint64_t)s << 32) | d);
        }
    }
}

static uint64_t lower_bound_u64(const uint64_t* v, uint64_t n, uint64_t key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (v[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

/* tail membership: flag[i] = 1 when sorted tail key i is not in D */
typedef struct {
    const uint64_t* D;
    uint64_t nD;
    const uint64_t* keys; /* sorted (key<<? no: pairs) */
    uint8_t* fresh;
    uint64_t n;
} memb_ctx;

static void memb(void* p, uint64_t lo, uint64_t hi, unsigned t) {
    (void)t;
    memb_ctx* c = (memb_ctx*)p;
    if (lo >= hi) return;
    uint64_t j = lower_bound_u64(c->D, c->nD, c->keys[lo]);
    for (uint64_t i = lo; i < hi; ++i) {
        const uint64_t k = c->keys[i];
        while (j < c->nD && c->D[j] < k) ++j;
        c->fresh[i] = !(j < c->nD && c->D[j] == k);
    }
}

typedef struct {
    uint64_t key, pos;
} kp;

static int cmp_kp_key(const void* x, const void* y) {
    const kp *a = (const kp*)x, *b = (const kp*)y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->pos < b->pos ? -1 : a->pos > b->pos;
}
static int cmp_kp_pos(const void* x, const void* y) {
    const kp *a = (const kp*)x, *b = (const kp*)y;
    return a->pos < b->pos ? -1 : a->pos > b->pos;
}

typedef struct {
    uint64_t* keys;
    uint64_t n;
    uint8_t* seen;
    const uint32_t* map;
    const uint32_t* perm;
} relab_ctx;

static void mark_seen(void* p, uint64_t lo, uint64_t hi, unsigned t) {
    (void)t;
    relab_ctx* c = (relab_ctx*)p;
    for (uint64_t i = lo; i < hi; ++i) {
        c->seen[c->keys[i] >> 32] = 1; /* benign race: every writer stores 1 */
        c->seen[c->keys[i] & 0xFFFFFFFFULL] = 1;
    }
}

static void relabel_keys(void* p, uint64_t lo, uint64_t hi, unsigned t) {
    (void)t;
    relab_ctx* c = (relab_ctx*)p;
    for (uint64_t i = lo; i < hi; ++i) {
        const uint64_t s = c->perm[c->map[c->keys[i] >> 32]];
        const uint64_t d = c->perm[c->map[c->keys[i] & 0xFFFFFFFFULL]];
        c->keys[i] = (s << 32) | d;
    }
}

typedef struct {
    const uint64_t* keys;
    uint32_t* ci;
} ci_ctx;

static void fill_ci(void* p, uint64_t lo, uint64_t hi, unsigned t) {
    (void)t;
    ci_ctx* c = (ci_ctx*)p;
    for (uint64_t i = lo; i < hi; ++i) c->ci[i] = (uint32_t)(c->keys[i] & 0xFFFFFFFFULL);
}

static int bits_for(uint64_t v) {
    int b = 1;
    while (b < 32 && (1ULL << b) < v) ++b;
    return b;
}

/* Returns 0 and malloc'ed uint32 row_ptr[n+1] / col_idx[m] (free with
 * orc_free), or -1 (allocation failure / > uint32 sizes). */
int orc_gen_bench_csr(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                      uint64_t rng_seed, uint64_t target, int relabel, uint64_t* n_out, uint64_t* m_out,
                      uint32_t** rp_out, uint32_t** ci_out) {
    const uint64_t ids = 1ULL << scale;
    const int kb = 32 + (int)scale;
    gen_ctx g = {scale, a, a + b, a + b + c, rng_seed, 0, UINT64_MAX, NULL};
    uint64_t *S = NULL, *T = NULL, nS = 0;
    if (target == 0) {
        const uint64_t raw = (uint64_t)edge_factor << scale;
        const uint64_t nch = (raw + CHUNK_EDGES - 1) / CHUNK_EDGES;
        S = (uint64_t*)malloc(nch * CHUNK_EDGES * 8);
        T = (uint64_t*)malloc(nch * CHUNK_EDGES * 8);
        if (!S || !T) return -1;
        g.raw_end = raw;
        g.out = S;
        par_for(nch, nthreads(), gen_chunks, &g);
        uint64_t* r = radix_sort(S, T, nch * CHUNK_EDGES, 64);
        if (r != S) { uint64_t* x = S; S = T; T = x; }
        nS = unique_sorted(S, nch * CHUNK_EDGES);
        if (nS && S[nS - 1] == SENTINEL) --nS;
        free(T);
        T = NULL;
    } else {
        /* the first c0 chunks hold at most c0 * CHUNK_EDGES <= target distinct
         * keys, so all of them are among the first `target` distinct keys */
        const uint64_t c0 = target / CHUNK_EDGES;
        S = (uint64_t*)malloc((target + 1) * 8);
        T = (uint64_t*)malloc((c0 * CHUNK_EDGES + 1) * 8);
        if (!S || !T) return -1;
        g.out = S;
        par_for(c0, nthreads(), gen_chunks, &g);
        uint64_t* r = radix_sort(S, T, c0 * CHUNK_EDGES, 64);
        if (r != S) memcpy(S, r, c0 * CHUNK_EDGES * 8);
        free(T);
        T = NULL;
        nS = unique_sorted(S, c0 * CHUNK_EDGES);
        if (nS && S[nS - 1] == SENTINEL) --nS;
        /* the tail: chunks from c0 on, in batches; a key is taken when it is
         * not yet in S and this is its first occurrence, in stream order */
        uint64_t next = c0;
        uint64_t* extra = NULL;
        uint64_t nextra = 0;
        while (nS + nextra < target) {
            const uint64_t need = target - nS - nextra;
            const uint64_t nch = (need * 2 + CHUNK_EDGES - 1) / CHUNK_EDGES + 1;
            uint64_t* raw = (uint64_t*)malloc(nch * CHUNK_EDGES * 8);
            if (!raw) return -1;
            g.chunk0 = next;
            g.out = raw;
            par_for(nch, nthreads(), gen_chunks, &g);
            /* (key, stream position) of every non-loop draw, sorted by key */
            kp* P = (kp*)malloc(nch * CHUNK_EDGES * sizeof(kp));
            uint64_t np = 0;
            for (uint64_t i = 0; i < nch * CHUNK_EDGES; ++i)
                if (raw[i] != SENTINEL) P[np].key = raw[i], P[np].pos = i, ++np;
            free(raw);
            qsort(P, np, sizeof(kp), cmp_kp_key);
            /* first occurrence per key */
            uint64_t w = 0;
            for (uint64_t i = 0; i < np; ++i)
                if (w == 0 || P[i].key != P[w - 1].key) P[w++] = P[i];
            np = w;
            uint64_t* keys = (uint64_t*)malloc((np + 1) * 8);
            uint8_t* fresh = (uint8_t*)malloc(np + 1);
            for (uint64_t i = 0; i < np; ++i) keys[i] = P[i].key;
            memb_ctx mc = {S, nS, keys, fresh, np};
            par_for(np, nthreads(), memb, &mc);
            if (nextra) { /* also not already taken from an earlier tail batch */
                memb_ctx mx = {extra, nextra, keys, (uint8_t*)malloc(np + 1), np};
                par_for(np, nthreads(), memb, &mx);
                for (uint64_t i = 0; i < np; ++i) fresh[i] &= mx.fresh[i];
                free(mx.fresh);
            }
            w = 0;
            for (uint64_t i = 0; i < np; ++i)
                if (fresh[i]) P[w++] = P[i];
            free(keys);
            free(fresh);
            qsort(P, w, sizeof(kp), cmp_kp_pos);
            const uint64_t take = w < need ? w : need;
            extra = (uint64_t*)realloc(extra, (nextra + take + 1) * 8);
            for (uint64_t i = 0; i < take; ++i) extra[nextra + i] = P[i].key;
            nextra += take;
            qsort(extra, nextra, 8, cmp_u64);
            free(P);
            next += nch;
        }
        /* merge extra into S from the back (S has room for target keys) */
        uint64_t i = nS, j = nextra, o = nS + nextra;
        while (j > 0) {
            if (i > 0 && S[i - 1] > extra[j - 1]) S[--o] = S[--i];
            else S[--o] = extra[--j];
        }
        nS += nextra;
        free(extra);
    }
    /* ---- relabel ------------------------------------------------------------ */
    uint64_t n = ids;
    if (relabel != 0) {
        uint32_t* map = (uint32_t*)malloc(ids * 4);
        uint64_t live = ids;
        relab_ctx rc = {S, nS, NULL, map, NULL};
        if (relabel == 2) {
            rc.seen = (uint8_t*)calloc(ids, 1);
            par_for(nS, nthreads(), mark_seen, &rc);
            live = 0;
            for (uint64_t v = 0; v < ids; ++v) map[v] = rc.seen[v] ? (uint32_t)live++ : 0xFFFFFFFFu;
            free(rc.seen);
        } else {
            for (uint64_t v = 0; v < ids; ++v) map[v] = (uint32_t)v;
        }
        /* seeded Fisher-Yates over the live ids */
        uint32_t* perm = (uint32_t*)malloc((live + 1) * 4);
        for (uint64_t v = 0; v < live; ++v) perm[v] = (uint32_t)v;
        orc_mt rng;
        orc_mt_seed(&rng, splitmix64(rng_seed ^ 0x5DEECE66DULL));
        for (uint64_t i = live; i > 1; --i) {
            const uint64_t max = UINT64_MAX, bound = i, limit = max - max % bound;
            uint64_t r = orc_mt_next(&rng);
            while (r >= limit) r = orc_mt_next(&rng);
            const uint32_t x = perm[i - 1];
            perm[i - 1] = perm[r % bound];
            perm[r % bound] = x;
        }
        rc.perm = perm;
        par_for(nS, nthreads(), relabel_keys, &rc);
        free(map);
        free(perm);
        T = (uint64_t*)malloc((nS + 1) * 8);
        if (!T) return -1;
        uint64_t* r = radix_sort(S, T, nS, 32 + bits_for(live));
        if (r != S) { uint64_t* x = S; S = T; T = x; }
        free(T);
        n = live;
    }
    if (n >= 0xFFFFFFFFULL || nS >= 0xFFFFFFFFULL) {
        free(S);
        return -1;
    }
    /* ---- CSR ------------------------------------------------------------------ */
    uint32_t* rp = (uint32_t*)calloc(n + 1, 4);
    uint32_t* ci = (uint32_t*)malloc((nS + 1) * 4);
    if (!rp || !ci) return -1;
    ci_ctx cc = {S, ci};
    par_for(nS, nthreads(), fill_ci, &cc);
    for (uint64_t i = 0; i < nS; ++i) rp[(S[i] >> 32) + 1]++;
    for (uint64_t v = 0; v < n; ++v) rp[v + 1] += rp[v];
    free(S);
    (void)kb;
    *n_out = n;
    *m_out = nS;
    *rp_out = rp;
    *ci_out = ci;
    return 0;
}

void orc_free(void* p) { free(p); }

/* bench.cpp:200-218 over a uint32 CSR. Returns 0, or -1 when fewer than n
 * ids have a non-empty row (*eligible_out = how many do). */
int orc_pick_seeds_u32(uint64_t node_count, const uint32_t* row_ptr, uint64_t n, uint64_t rng_seed,
                       uint64_t* out, uint64_t* eligible_out) {
    uint64_t* eligible = (uint64_t*)malloc((node_count ? node_count : 1) * sizeof(uint64_t));
    uint64_t ne = 0;
    for (uint64_t id = 0; id < node_count; ++id)
        if (row_ptr[id + 1] > row_ptr[id]) eligible[ne++] = id;
    if (eligible_out) *eligible_out = ne;
    if (ne < n) {
        free(eligible);
        return -1;
    }
    orc_mt rng;
    orc_mt_seed(&rng, rng_seed);
    const uint64_t max = UINT64_MAX;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t bound = ne - i, limit = max - max % bound;
        uint64_t draw = orc_mt_next(&rng);
        while (draw >= limit) draw = orc_mt_next(&rng);
        const uint64_t j = i + draw % bound;
        const uint64_t t = eligible[i];
        eligible[i] = eligible[j];
        eligible[j] = t;
    }
    memcpy(out, eligible, n * sizeof(uint64_t));
    free(eligible);
    return 0;
}

/* ---- bulk k_hop_count (execute.cpp:347-375) on all host threads ------------ */
typedef struct {
    uint64_t n;
    const uint32_t* rp;
    const uint32_t* ci;
    const uint64_t* seeds;
    uint32_t k;
    uint64_t* exact;      /* [ns] |F_k| (0 on early exit) */
    uint64_t* cumul;      /* [ns] |visited| - 1 */
    uint64_t* edges;      /* [ns] E(s,k) or NULL */
    uint64_t* levels;     /* [ns][k+1] |F_l| or NULL */
    volatile uint64_t next;
    uint64_t ns;
} many_ctx;

static void many_worker(void* p, uint64_t lo, uint64_t hi, unsigned t) {
    (void)lo, (void)hi, (void)t;
    many_ctx* c = (many_ctx*)p;
    const uint64_t n = c->n;
    const uint64_t nwords = (n + 63) / 64;
    uint64_t* vis = (uint64_t*)calloc(nwords + 1, 8);
    /* all discovered vertices, level after level: level h is [beg_h, end_h) */
    uint64_t cap = 1 << 16;
    uint32_t* lv = (uint32_t*)malloc(cap * 4);
    for (;;) {
        const uint64_t q = __atomic_fetch_add(&c->next, 1, __ATOMIC_RELAXED);
        if (q >= c->ns) break;
        const uint32_t s = (uint32_t)c->seeds[q];
        uint64_t beg = 0, end = 1, E = 0, last = 0;
        lv[0] = s;
        vis[s >> 6] |= 1ULL << (s & 63);
        if (c->levels) {
            memset(c->levels + q * (c->k + 1), 0, (c->k + 1) * 8);
            c->levels[q * (c->k + 1)] = 1;
        }
        for (uint32_t hop = 1; hop <= c->k; ++hop) {
            uint64_t w = end;
            for (uint64_t i = beg; i < end; ++i) {
                const uint32_t r = lv[i];
                E += c->rp[r + 1] - c->rp[r];
                for (uint64_t e = c->rp[r]; e < c->rp[r + 1]; ++e) {
                    const uint32_t v = c->ci[e];
                    uint64_t* word = &vis[v >> 6];
                    const uint64_t bit = 1ULL << (v & 63);
                    if (*word & bit) continue;
                    *word |= bit;
                    if (w == cap) {
                        cap *= 2;
                        lv = (uint32_t*)realloc(lv, cap * 4);
                    }
                    lv[w++] = v;
                }
            }
            last = w - end;
            if (c->levels) c->levels[q * (c->k + 1) + hop] = last;
            beg = end;
            end = w;
            if (last == 0) break;
        }
        c->exact[q] = last;
        c->cumul[q] = end - 1;
        if (c->edges) c->edges[q] = E;
        if (end > nwords / 8) memset(vis, 0, nwords * 8);
        else
            for (uint64_t i = 0; i < end; ++i) vis[lv[i] >> 6] = 0;
    }
    free(vis);
    free(lv);
}

/* Exact and cumulative counts (and optionally the §8(d) work model) of
 * k_hop_count(seeds[i], k) over a uint32 CSR. threads 0 = all host threads.
 * Seeds must be < n. */
void orc_khop_many(uint64_t n, const uint32_t* row_ptr, const uint32_t* col_idx, const uint64_t* seeds,
                   uint64_t ns, uint32_t k, unsigned threads, uint64_t* exact, uint64_t* cumulative,
                   uint64_t* edges, uint64_t* levels) {
    many_ctx c = {n, row_ptr, col_idx, seeds, k, exact, cumulative, edges, levels, 0, ns};
    unsigned nt = threads ? threads : nthreads();
    if (nt > ns) nt = (unsigned)(ns ? ns : 1);
    par_for(nt, nt, many_worker, &c);
}
