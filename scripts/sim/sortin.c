// Design probe helper: in-lists ordered by descending source out-degree (the device CSC order).
#include <stdint.h>
#include <stdlib.h>
static const uint32_t* RP;
static int cmp(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    uint32_t dx = RP[x + 1] - RP[x], dy = RP[y + 1] - RP[y];
    if (dx != dy) return dx > dy ? -1 : 1;
    return x < y ? -1 : x > y;
}
void sort_in(uint64_t n, const uint32_t* cp, uint32_t* ri, const uint32_t* rp) {
    RP = rp;
    for (uint64_t u = 0; u < n; ++u) qsort(ri + cp[u], cp[u + 1] - cp[u], 4, cmp);
}
