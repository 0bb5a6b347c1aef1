// Design probe (not product, not oracle): per-hop cost of a split LANES pull (in-list prefix of
// sources with out-degree >= D pulled, the frontier's low-degree vertices pushing).
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
// per hop, for degree thresholds D[i]: hybrid = pull over in-list entries whose source has
// outdeg >= D (in-lists sorted by descending source outdeg -> a prefix), early exit; plus push of
// every frontier vertex with outdeg < D over all its out-edges.
// out[h][i][0] = pull entries scanned, [1] = push edges, [2] = pull entries in the all-pull baseline (i==0 only)
void hyb_sim(uint64_t n, const uint32_t* rp, const uint32_t* ci, const uint32_t* cp, const uint32_t* ri,
             const uint32_t* seeds, int ns, int k, const uint32_t* D, int nD, uint64_t* out) {
    uint16_t* V = calloc(n, 2); uint16_t* F = calloc(n, 2); uint16_t* Fn = calloc(n, 2);
    for (int l = 0; l < ns; ++l) { V[seeds[l]] |= 1u << l; F[seeds[l]] |= 1u << l; }
    uint32_t act = (1u << ns) - 1;
    for (int h = 1; h <= k; ++h) {
        for (int i = 0; i < nD; ++i) {
            uint64_t* o = out + ((h - 1) * nD + i) * 3;
            for (uint64_t u = 0; u < n; ++u) {
                const uint32_t need = act & ~V[u];
                if (!need) continue;
                uint32_t acc = 0;
                for (uint32_t p = cp[u]; p < cp[u + 1]; ++p) {
                    const uint32_t v = ri[p];
                    if (rp[v + 1] - rp[v] < D[i]) break;
                    acc |= F[v]; o[0]++;
                    if ((acc & need) == need) break;
                }
                if (i == 0) {
                    uint32_t a2 = 0;
                    for (uint32_t p = cp[u]; p < cp[u + 1]; ++p) { a2 |= F[ri[p]]; o[2]++; if ((a2 & need) == need) break; }
                }
            }
            for (uint64_t v = 0; v < n; ++v) if (F[v] && rp[v + 1] - rp[v] < D[i]) o[1] += rp[v + 1] - rp[v];
        }
        memset(Fn, 0, n * 2);
        for (uint64_t v = 0; v < n; ++v) if (F[v])
            for (uint32_t p = rp[v]; p < rp[v + 1]; ++p) Fn[ci[p]] |= F[v];
        uint32_t nact = 0;
        for (uint64_t u = 0; u < n; ++u) { Fn[u] &= ~V[u]; V[u] |= Fn[u]; nact |= Fn[u]; }
        uint16_t* t = F; F = Fn; Fn = t;
        act = nact;
        if (!act) break;
    }
    free(V); free(F); free(Fn);
}
