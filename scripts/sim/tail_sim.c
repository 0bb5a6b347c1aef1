// Design probe (not product, not oracle): per-hop split of the scanned in-list entries by source
// rank (< H) and frontier membership.
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
// per hop: scanned entries split by (source rank < H) x (source in frontier)
void tail_sim(uint64_t n, const uint32_t* rp, const uint32_t* ci, const uint32_t* cp, const uint32_t* ri,
              const uint32_t* seeds, int ns, int k, const uint32_t* rank, uint32_t H,
              uint64_t* out /* [k][6]: hub_in, hub_out, tail_in, tail_out, |F| union, unsettled verts */) {
    uint16_t* V = calloc(n, 2); uint16_t* F = calloc(n, 2); uint16_t* Fn = calloc(n, 2);
    for (int l = 0; l < ns; ++l) { V[seeds[l]] |= 1u << l; F[seeds[l]] |= 1u << l; }
    uint32_t act = (1u << ns) - 1;
    for (int h = 1; h <= k; ++h) {
        uint64_t* o = out + (h - 1) * 6;
        for (uint64_t v = 0; v < n; ++v) o[4] += F[v] != 0;
        for (uint64_t u = 0; u < n; ++u) {
            const uint32_t need = act & ~V[u];
            if (!need) continue;
            uint32_t acc = 0;
            uint32_t p = cp[u];
            for (; p < cp[u + 1]; ++p) {
                const uint32_t v = ri[p];
                acc |= F[v];
                int hub = rank[v] < H, in = F[v] != 0;
                o[hub ? (in ? 0 : 1) : (in ? 2 : 3)]++;
                if ((acc & need) == need) break;
            }
            if (p == cp[u + 1]) o[5]++;
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
