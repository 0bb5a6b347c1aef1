// Design probe (not product, not oracle): per-hop cost of the LANES pull for a
// seed batch under two policies, on a CSR/CSC given by the caller.
//   all:      every active lane in the pull's need mask (the round-1 engine)
//   perlane:  a lane pulls only when its frontier edges * alpha > its
//             unexplored in-edges (Beamer, per lane); other lanes push
// In-lists are scanned in the order given (the engine's: descending out-degree).
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

typedef struct { uint64_t pull_all, pull_lane, push_lane, push_all, cand_all, cand_lane; } hopcost;

void lane_sim(uint64_t n, const uint32_t* rp, const uint32_t* ci, const uint32_t* cp, const uint32_t* ri,
              const uint32_t* seeds, int ns, int k, uint32_t alpha, hopcost* out) {
    uint32_t* V = calloc(n, 4);
    uint32_t* F = calloc(n, 4);
    uint32_t* Fn = calloc(n, 4);
    uint64_t m = rp[n];
    uint64_t unexpl[32];
    for (int l = 0; l < ns; ++l) { V[seeds[l]] |= 1u << l; F[seeds[l]] |= 1u << l; unexpl[l] = m; }
    uint32_t act = (ns == 32) ? 0xFFFFFFFFu : ((1u << ns) - 1);
    for (int h = 1; h <= k; ++h) {
        hopcost c = {0};
        uint64_t E[32] = {0};
        for (uint64_t v = 0; v < n; ++v) if (F[v]) {
            uint32_t d = rp[v + 1] - rp[v];
            c.push_all += d;
            for (int l = 0; l < ns; ++l) if (F[v] >> l & 1) E[l] += d;
        }
        uint32_t pullm = 0;
        for (int l = 0; l < ns; ++l) if ((act >> l & 1) && E[l] * alpha > unexpl[l]) pullm |= 1u << l;
        for (int l = 0; l < ns; ++l) if ((act >> l & 1) && !(pullm >> l & 1)) c.push_lane += E[l];
        // pull costs
        for (uint64_t u = 0; u < n; ++u) {
            uint32_t need = act & ~V[u];
            if (need) {
                c.cand_all++;
                uint32_t acc = 0; uint64_t s = 0;
                for (uint32_t p = cp[u]; p < cp[u + 1]; ++p) { acc |= F[ri[p]]; ++s; if ((acc & need) == need) break; }
                c.pull_all += s;
            }
            uint32_t needl = pullm & ~V[u];
            if (needl) {
                c.cand_lane++;
                uint32_t acc = 0; uint64_t s = 0;
                for (uint32_t p = cp[u]; p < cp[u + 1]; ++p) { acc |= F[ri[p]]; ++s; if ((acc & needl) == needl) break; }
                c.pull_lane += s;
            }
        }
        // true next frontier (push semantics over all lanes)
        memset(Fn, 0, n * 4);
        for (uint64_t v = 0; v < n; ++v) if (F[v])
            for (uint32_t p = rp[v]; p < rp[v + 1]; ++p) Fn[ci[p]] |= F[v];
        uint32_t nact = 0;
        for (uint64_t u = 0; u < n; ++u) {
            Fn[u] &= ~V[u];
            if (Fn[u]) {
                V[u] |= Fn[u]; nact |= Fn[u];
                uint32_t indeg = cp[u + 1] - cp[u];
                for (int l = 0; l < ns; ++l) if (Fn[u] >> l & 1) unexpl[l] -= indeg;
            }
        }
        uint32_t* t = F; F = Fn; Fn = t;
        act = nact;
        out[h - 1] = c;
        if (!act) break;
    }
    free(V); free(F); free(Fn);
}

// CSC with each in-list ordered by descending source out-degree, ties by id
#include <pthread.h>
typedef struct { const uint32_t* rp; uint32_t* cp; uint32_t* ri; uint64_t lo, hi; } csc_job;
static const uint32_t* g_rp;
static int cmp_src(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    uint32_t dx = g_rp[x + 1] - g_rp[x], dy = g_rp[y + 1] - g_rp[y];
    if (dx != dy) return dx > dy ? -1 : 1;
    return x < y ? -1 : x > y;
}
static void* csc_sort(void* p) {
    csc_job* j = p;
    for (uint64_t u = j->lo; u < j->hi; ++u) qsort(j->ri + j->cp[u], j->cp[u + 1] - j->cp[u], 4, cmp_src);
    return NULL;
}
void build_csc(uint64_t n, const uint32_t* rp, const uint32_t* ci, uint32_t* cp, uint32_t* ri) {
    uint64_t m = rp[n];
    memset(cp, 0, (n + 1) * 4);
    for (uint64_t e = 0; e < m; ++e) cp[ci[e] + 1]++;
    for (uint64_t u = 0; u < n; ++u) cp[u + 1] += cp[u];
    uint32_t* fill = malloc((n + 1) * 4);
    memcpy(fill, cp, (n + 1) * 4);
    for (uint64_t v = 0; v < n; ++v)
        for (uint32_t p = rp[v]; p < rp[v + 1]; ++p) ri[fill[ci[p]]++] = (uint32_t)v;
    free(fill);
    g_rp = rp;
    pthread_t th[64]; csc_job jobs[64]; int nt = 8;
    for (int t = 0; t < nt; ++t) { jobs[t] = (csc_job){rp, cp, ri, n * t / nt, n * (t + 1) / nt}; pthread_create(&th[t], 0, csc_sort, &jobs[t]); }
    for (int t = 0; t < nt; ++t) pthread_join(th[t], 0);
}
