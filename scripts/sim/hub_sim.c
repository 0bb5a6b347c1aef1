// Design probe (not product, not oracle): for the LANES all-lanes pull of a
// 10-seed batch, the share of scanned in-list entries whose SOURCE is among
// the top-H vertices by out-degree (rank[v] < H), per hop — i.e. how many
// per-edge frontier-word gathers a shared-memory cache of the H hub words
// would absorb.
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void hub_sim(uint64_t n, const uint32_t* rp, const uint32_t* ci, const uint32_t* cp, const uint32_t* ri,
             const uint32_t* seeds, int ns, int k, const uint32_t* rank, const uint32_t* H, int nH,
             uint64_t* scanned, uint64_t* hub_hits /* [k][nH] */, uint64_t* fhits /* [k] */) {
    uint32_t* V = calloc(n, 4);
    uint32_t* F = calloc(n, 4);
    uint32_t* Fn = calloc(n, 4);
    for (int l = 0; l < ns; ++l) { V[seeds[l]] |= 1u << l; F[seeds[l]] |= 1u << l; }
    uint32_t act = (1u << ns) - 1;
    for (int h = 1; h <= k; ++h) {
        uint64_t sc = 0;
        for (uint64_t u = 0; u < n; ++u) {
            const uint32_t need = act & ~V[u];
            if (!need) continue;
            uint32_t acc = 0;
            for (uint32_t p = cp[u]; p < cp[u + 1]; ++p) {
                const uint32_t v = ri[p];
                acc |= F[v];
                ++sc;
                if (F[v]) fhits[h - 1]++;
                for (int i = 0; i < nH; ++i) if (rank[v] < H[i]) hub_hits[(h - 1) * nH + i]++;
                if ((acc & need) == need) break;
            }
        }
        scanned[h - 1] = sc;
        memset(Fn, 0, n * 4);
        for (uint64_t v = 0; v < n; ++v) if (F[v])
            for (uint32_t p = rp[v]; p < rp[v + 1]; ++p) Fn[ci[p]] |= F[v];
        uint32_t nact = 0;
        for (uint64_t u = 0; u < n; ++u) {
            Fn[u] &= ~V[u];
            V[u] |= Fn[u];
            nact |= Fn[u];
        }
        uint32_t* t = F; F = Fn; Fn = t;
        act = nact;
        if (!act) break;
    }
    free(V); free(F); free(Fn);
}
