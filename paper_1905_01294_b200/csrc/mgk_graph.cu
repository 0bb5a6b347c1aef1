// Device-resident graph: uint32 CSR + CSC built once per upload.
//
// Replaces, for the k-hop path, the store's read side:
//   PropertyGraph::relation_matrix   proj/core/src/graph.cpp:84-88
//   PropertyGraph::transposed_matrix proj/core/src/graph.cpp:90-102
//   transpose (counting sort)        proj/core/src/sparse.cpp:379-403
//   flush_slot (sort + dedup)        proj/core/src/graph.cpp:182-215
// The CSC is produced by a radix sort of (col << 32 | row) keys on the GPU,
// so in-neighbour lists come out ascending exactly like the reference's
// transpose. A zero-in-degree bitmap lets the pull pass skip vertices that
// can never be reached.
#include <cub/cub.cuh>
#include <cstdlib>

#include "mgk_internal.cuh"

namespace mgk {
namespace {

#define MGK_TRY(x)                         \
    do {                                   \
        cudaError_t e_ = (x);              \
        if (e_ != cudaSuccess) return e_;  \
    } while (0)

constexpr int kTB = 256;

inline unsigned blocks_for(uint64_t n) { return (unsigned)std::min<uint64_t>((n + kTB - 1) / kTB, 148ull * 64); }

// row id of every CSR entry (grid-stride over rows; long rows split by a
// block-per-row pass below would be faster, but this runs once per load).
__global__ void expand_rows(const uint32_t* rp, uint32_t n, uint64_t m, unsigned long long* keys) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        // upper_bound(rp, p) - 1
        uint32_t lo = 0, hi = n;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (rp[mid + 1] <= p) lo = mid + 1;
            else hi = mid;
        }
        keys[p] = lo;  // row in the low bits, column filled in by fill_cols
    }
}

__global__ void fill_cols(const uint32_t* ci, uint64_t m, unsigned long long* keys) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x)
        keys[p] |= (unsigned long long)ci[p] << 32;
}

// keys[p] = col << 32 | row in CSR order: flags a row whose entries are not
// strictly ascending (a duplicate or unsorted entry)
__global__ void rows_strict_check(const unsigned long long* keys, uint64_t m, unsigned int* bad) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p + 1 < m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long a = keys[p], b = keys[p + 1];
        if ((uint32_t)a == (uint32_t)b && (a >> 32) >= (b >> 32)) *bad = 1;
    }
}

// sorted (major << 32 | minor) keys -> ptr[n+1] over the major ids and the
// minor ids in order.
__global__ void keys_to_csr(const unsigned long long* keys, uint64_t m, uint32_t n, uint32_t* ptr,
                            uint32_t* minor) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p <= m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t cur = p < m ? (keys[p] >> 32) : n;
        const uint64_t prev = p > 0 ? (keys[p - 1] >> 32) : (uint64_t)-1;
        if (p < m) minor[p] = (uint32_t)keys[p];
        for (uint64_t c = prev + 1; c <= cur && c <= n; ++c) ptr[c] = (uint32_t)p;
    }
}

__global__ void no_in_bitmap(const uint32_t* cp, uint32_t n, uint32_t nwords, uint32_t* bits) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += gridDim.x * blockDim.x) {
        uint32_t x = 0;
        for (uint32_t b = 0; b < 32; ++b) {
            const uint32_t u = w * 32 + b;
            if (u >= n || cp[u + 1] == cp[u]) x |= 1u << b;
        }
        bits[w] = x;
    }
}

// in-degree > kHeavyIn: count kHeavyChunk tasks; mark in the pull skip mask
__global__ void heavy_count(const uint32_t* cp, uint32_t n, uint32_t* cnt, uint32_t* skip) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        const uint32_t d = cp[u + 1] - cp[u];
        const bool heavy = d > kHeavyIn;
        cnt[u] = heavy ? (d + kHeavyChunk - 1) / kHeavyChunk : 0;
        if (heavy) atomicOr(skip + (u >> 5), 1u << (u & 31));
    }
}

// one key (chunk << 32 | vertex) per heavy task; sorted, the list is
// chunk-major: every heavy vertex's first chunk comes before any second
// chunk, so a later chunk usually finds its vertex already covered (the pull
// checks before scanning) — the hubs-first in-list order then makes most
// heavy vertices cost one chunk
__global__ void heavy_fill(uint32_t n, const uint32_t* off, unsigned long long* keys) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
        const uint32_t c = off[u + 1] - off[u];
        for (uint32_t i = 0; i < c; ++i) keys[off[u] + i] = ((unsigned long long)i << 32) | u;
    }
}

__global__ void heavy_tasks(const unsigned long long* keys, uint64_t nt, const uint32_t* cp, uint2* tasks) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < nt; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = (uint32_t)keys[t], i = (uint32_t)(keys[t] >> 32);
        tasks[t] = make_uint2(u, cp[u] + i * kHeavyChunk);
    }
}

__global__ void pack_edges(const uint32_t* src, const uint32_t* dst, uint64_t m, uint32_t n,
                           unsigned long long* keys, unsigned int* bad) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = src[p], d = dst[p];
        if (s >= n || d >= n) atomicMin(bad, (unsigned int)(p < 0xFFFFFFFEull ? p : 0xFFFFFFFEull));
        keys[p] = ((unsigned long long)s << 32) | d;
    }
}

// keep[p] = 1 if keys[p] differs from keys[p-1]
__global__ void mark_unique(const unsigned long long* keys, uint64_t m, uint32_t* keep) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x)
        keep[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1u : 0u;
}

__global__ void swap_halves(unsigned long long* keys, uint64_t m) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[p];
        keys[p] = (k << 32) | (k >> 32);
    }
}

// ((~deg) << 32 | v): ascending order = descending degree, ties by id (cp:
// in-degree from the CSC, or rp: out-degree from the CSR)
__global__ void deg_keys(const uint32_t* cp, uint32_t n, unsigned long long* keys) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        keys[v] = ((unsigned long long)(0xFFFFFFFFu - (cp[v + 1] - cp[v])) << 32) | v;
}

__global__ void perm_from_sorted(const unsigned long long* keys, uint32_t n, uint32_t* perm, uint32_t* inv) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)keys[i];
        inv[i] = v;
        perm[v] = (uint32_t)i;
    }
}

// keys[p] = row (expand_rows) -> map[row] << 32 | map[ci[p]]
__global__ void map_edge_keys(unsigned long long* keys, const uint32_t* ci, const uint32_t* map, uint64_t m) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t row = (uint32_t)keys[p];
        keys[p] = ((unsigned long long)map[row] << 32) | map[ci[p]];
    }
}

__global__ void map_ids(unsigned long long* ids, uint64_t n, const uint32_t* map) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        ids[i] = map[ids[i]];
}

int key_bits(uint32_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}

cudaError_t radix_sort_keys(unsigned long long*& keys, unsigned long long*& alt, uint64_t m,
                            int end_bit, cudaStream_t s) {
    cub::DoubleBuffer<unsigned long long> db(keys, alt);
    size_t tmp = 0;
    MGK_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, (int64_t)m, 0, end_bit, s));
    void* t = nullptr;
    MGK_TRY(cudaMallocAsync(&t, tmp, s));
    MGK_TRY(cub::DeviceRadixSort::SortKeys(t, tmp, db, (int64_t)m, 0, end_bit, s));
    MGK_TRY(cudaFreeAsync(t, s));
    if (db.Current() != keys) std::swap(keys, alt);
    return cudaSuccess;
}

cudaError_t build_heavy(Graph* g, cudaStream_t s);

// (col << 32 | row) sorted keys -> (col << 32 | ~outdeg(row)) keys + row values
__global__ void make_deg_keys(unsigned long long* keys, uint32_t* vals, uint64_t m,
                              const uint32_t* rp) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[p];
        const uint32_t row = (uint32_t)k;
        const uint32_t deg = rp[row + 1] - rp[row];
        keys[p] = (k & 0xFFFFFFFF00000000ull) | (0xFFFFFFFFu - deg);
        vals[p] = row;
    }
}

// Order every in-neighbour list by descending out-degree (ties: ascending id,
// the radix sort is stable). Pull passes OR / test in-neighbours in list order
// and stop at the first hit (SINGLE) or once every needed lane is covered
// (LANES); hubs sit in most frontiers, so putting them first ends scans early.
// The list is a set, so results do not depend on the order.
cudaError_t order_in_lists(Graph* g, unsigned long long*& keys, unsigned long long*& alt, cudaStream_t s) {
    const uint64_t m = g->dg.m;
    const uint32_t n = g->dg.n;
    uint32_t *vals = nullptr, *valt = nullptr;
    MGK_TRY(cudaMallocAsync(&vals, m * 4, s));
    MGK_TRY(cudaMallocAsync(&valt, m * 4, s));
    make_deg_keys<<<blocks_for(m), kTB, 0, s>>>(keys, vals, m, g->rp);
    MGK_TRY(cudaGetLastError());
    cub::DoubleBuffer<unsigned long long> dk(keys, alt);
    cub::DoubleBuffer<uint32_t> dv(vals, valt);
    size_t tmp = 0;
    MGK_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, (int64_t)m, 0, 32 + key_bits(n), s));
    void* t = nullptr;
    MGK_TRY(cudaMallocAsync(&t, tmp, s));
    MGK_TRY(cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, (int64_t)m, 0, 32 + key_bits(n), s));
    MGK_TRY(cudaMemcpyAsync(g->ri, dv.Current(), m * 4, cudaMemcpyDeviceToDevice, s));
    MGK_TRY(cudaFreeAsync(t, s));
    MGK_TRY(cudaFreeAsync(vals, s));
    MGK_TRY(cudaFreeAsync(valt, s));
    return cudaSuccess;
}

// Given device CSR (rp, ci) fill CSC (cp, ri) and the no_in bitmap.
cudaError_t build_csc(Graph* g, cudaStream_t s) {
    const uint32_t n = g->dg.n;
    const uint64_t m = g->dg.m;
    if (m > 0) {
        unsigned long long *keys = nullptr, *alt = nullptr;
        MGK_TRY(cudaMallocAsync(&keys, m * 8, s));
        MGK_TRY(cudaMallocAsync(&alt, m * 8, s));
        expand_rows<<<blocks_for(m), kTB, 0, s>>>(g->rp, n, m, keys);
        fill_cols<<<blocks_for(m), kTB, 0, s>>>(g->ci, m, keys);
        {
            unsigned int* bad = nullptr;
            unsigned int h_bad = 1;
            MGK_TRY(cudaMallocAsync(&bad, 4, s));
            MGK_TRY(cudaMemsetAsync(bad, 0, 4, s));
            rows_strict_check<<<blocks_for(m), kTB, 0, s>>>(keys, m, bad);
            MGK_TRY(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, s));
            MGK_TRY(cudaFreeAsync(bad, s));
            MGK_TRY(cudaStreamSynchronize(s));
            g->dg.rows_unique = h_bad ? 0u : 1u;
        }
        MGK_TRY(radix_sort_keys(keys, alt, m, 32 + key_bits(n), s));
        keys_to_csr<<<blocks_for(m + 1), kTB, 0, s>>>(keys, m, n, g->cp, g->ri);
        MGK_TRY(order_in_lists(g, keys, alt, s));
        MGK_TRY(cudaFreeAsync(keys, s));
        MGK_TRY(cudaFreeAsync(alt, s));
    } else {
        MGK_TRY(cudaMemsetAsync(g->cp, 0, (size_t)(n + 1) * 4, s));
        g->dg.rows_unique = 1;
    }
    no_in_bitmap<<<blocks_for(g->dg.nwords), kTB, 0, s>>>(g->cp, n, g->dg.nwords, g->no_in);
    MGK_TRY(cudaGetLastError());
    return build_heavy(g, s);
}

// pull_skip = no_in | heavy, and the heavy task list (prefix sum of chunk counts)
cudaError_t build_heavy(Graph* g, cudaStream_t s) {
    const uint32_t n = g->dg.n;
    MGK_TRY(cudaMemcpyAsync(g->pull_skip, g->no_in, (size_t)(g->dg.nwords + 1) * 4,
                            cudaMemcpyDeviceToDevice, s));
    uint32_t* cnt = nullptr;
    MGK_TRY(cudaMallocAsync(&cnt, (size_t)(n + 1) * 4, s));
    heavy_count<<<blocks_for(n), kTB, 0, s>>>(g->cp, n, cnt, g->pull_skip);
    MGK_TRY(cudaGetLastError());
    unsigned long long* d_total = nullptr;
    MGK_TRY(cudaMallocAsync(&d_total, 8, s));
    MGK_TRY(exclusive_scan_u32(cnt, n, d_total, s));
    unsigned long long total = 0;
    MGK_TRY(cudaMemcpyAsync(&total, d_total, 8, cudaMemcpyDeviceToHost, s));
    MGK_TRY(cudaStreamSynchronize(s));
    g->dg.nheavy = (uint32_t)total;
    MGK_TRY(cudaMalloc(&g->heavy, (size_t)std::max<unsigned long long>(total, 1) * sizeof(uint2)));
    g->dg.heavy = g->heavy;
    g->bytes += (size_t)std::max<unsigned long long>(total, 1) * sizeof(uint2);
    if (total) {
        unsigned long long *keys = nullptr, *alt = nullptr;
        MGK_TRY(cudaMallocAsync(&keys, total * 8, s));
        MGK_TRY(cudaMallocAsync(&alt, total * 8, s));
        heavy_fill<<<blocks_for(n), kTB, 0, s>>>(n, cnt, keys);
        MGK_TRY(cudaGetLastError());
        MGK_TRY(radix_sort_keys(keys, alt, total, 64, s));
        heavy_tasks<<<blocks_for(total), kTB, 0, s>>>(keys, total, g->cp, g->heavy);
        MGK_TRY(cudaGetLastError());
        MGK_TRY(cudaFreeAsync(keys, s));
        MGK_TRY(cudaFreeAsync(alt, s));
    }
    MGK_TRY(cudaFreeAsync(cnt, s));
    MGK_TRY(cudaFreeAsync(d_total, s));
    return cudaSuccess;
}


cudaError_t alloc_graph(Graph* g, uint32_t n, uint64_t m) {
    g->dg.n = n;
    g->dg.nwords = (n + 31) / 32;
    g->dg.m = m;
    const size_t mp = (size_t)std::max<uint64_t>(m, 1);
    MGK_TRY(cudaMalloc(&g->rp, (size_t)(n + 1) * 4));
    MGK_TRY(cudaMalloc(&g->ci, mp * 4));
    MGK_TRY(cudaMalloc(&g->cp, (size_t)(n + 1) * 4));
    MGK_TRY(cudaMalloc(&g->ri, mp * 4));
    MGK_TRY(cudaMalloc(&g->no_in, (size_t)(g->dg.nwords + 1) * 4));
    MGK_TRY(cudaMalloc(&g->pull_skip, (size_t)(g->dg.nwords + 1) * 4));
    MGK_TRY(cudaMalloc(&g->bad_seed, 4));
    MGK_TRY(cudaMemset(g->bad_seed, 0, 4));
    g->dg.bad_seed = g->bad_seed;
    g->bytes = 2 * (size_t)(n + 1) * 4 + 2 * mp * 4 + 2 * (size_t)(g->dg.nwords + 1) * 4;
    g->dg.rp = g->rp;
    g->dg.ci = g->ci;
    g->dg.cp = g->cp;
    g->dg.ri = g->ri;
    g->dg.no_in = g->no_in;
    g->dg.pull_skip = g->pull_skip;
    return cudaSuccess;
}

}  // namespace

cudaError_t exclusive_scan_u32(uint32_t* data, uint32_t n, unsigned long long* total,
                               cudaStream_t s) {
    // out-of-place into a temp, then copy back; total = last excl + last value
    uint32_t* out = nullptr;
    MGK_TRY(cudaMallocAsync(&out, (size_t)(n + 1) * 4, s));
    size_t tmp = 0;
    MGK_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, data, out, (int)(n + 1), s));
    void* t = nullptr;
    MGK_TRY(cudaMallocAsync(&t, tmp, s));
    // data[n] must be 0 so out[n] is the total; write it first
    MGK_TRY(cudaMemsetAsync(data + n, 0, 4, s));
    MGK_TRY(cub::DeviceScan::ExclusiveSum(t, tmp, data, out, (int)(n + 1), s));
    MGK_TRY(cudaMemcpyAsync(data, out, (size_t)(n + 1) * 4, cudaMemcpyDeviceToDevice, s));
    // widen the uint32 total into *total
    MGK_TRY(cudaMemsetAsync(total, 0, 8, s));
    MGK_TRY(cudaMemcpyAsync(total, out + n, 4, cudaMemcpyDeviceToDevice, s));
    MGK_TRY(cudaFreeAsync(t, s));
    MGK_TRY(cudaFreeAsync(out, s));
    return cudaSuccess;
}

cudaError_t graph_from_sorted_keys(Graph* g, unsigned long long*& keys, unsigned long long*& alt,
                                   uint64_t m, cudaStream_t s);

// (map[src] << 32 | map[dst]) of every CSR entry of g, sorted; keys/alt are
// allocated here (m entries each)
cudaError_t mapped_sorted_keys(const Graph* g, const uint32_t* map, unsigned long long*& keys,
                               unsigned long long*& alt, cudaStream_t s) {
    const uint32_t n = g->dg.n;
    const uint64_t m = g->dg.m;
    MGK_TRY(cudaMallocAsync(&keys, m * 8, s));
    MGK_TRY(cudaMallocAsync(&alt, m * 8, s));
    expand_rows<<<blocks_for(m), kTB, 0, s>>>(g->rp, n, m, keys);
    map_edge_keys<<<blocks_for(m), kTB, 0, s>>>(keys, g->ci, map, m);
    MGK_TRY(cudaGetLastError());
    return radix_sort_keys(keys, alt, m, 32 + key_bits(n), s);
}

// Locality relabelling (opt-in, MGK_RELABEL=1 at load): device ids by
// descending in-degree (ties by id), so the bits of popular targets share
// words and 128-B lines. Counts are invariant; seeds are mapped through perm
// on the device and returned ids through inv. Measured on G2:
// the dense hops of k >= 3 get faster (SINGLE k=3 27.5 -> 18.0 ms), but the
// k = 2 last hop gets 1.8x slower -- every seed's atomics now converge on the
// same few hot words, which serialise in their L2 slice -- so it is off by
// default. Needs duplicate-free rows (the rebuild goes through sorted keys).
cudaError_t locality_relabel(Graph* g, cudaStream_t s) {
    const uint32_t n = g->dg.n;
    const uint64_t m = g->dg.m;
    const char* on = std::getenv("MGK_RELABEL");
    if (!g->dg.rows_unique || m == 0 || n < 2 || !(on && (on[0] == '1' || on[0] == '2'))) return cudaSuccess;
    const bool by_out = on[0] == '2';
    uint32_t *perm = nullptr, *inv = nullptr;
    MGK_TRY(cudaMalloc(&perm, (size_t)n * 4));
    MGK_TRY(cudaMalloc(&inv, (size_t)n * 4));
    {
        unsigned long long *kv = nullptr, *ka = nullptr;
        MGK_TRY(cudaMallocAsync(&kv, (size_t)n * 8, s));
        MGK_TRY(cudaMallocAsync(&ka, (size_t)n * 8, s));
        deg_keys<<<blocks_for(n), kTB, 0, s>>>(by_out ? g->rp : g->cp, n, kv);
        MGK_TRY(radix_sort_keys(kv, ka, n, 64, s));
        perm_from_sorted<<<blocks_for(n), kTB, 0, s>>>(kv, n, perm, inv);
        MGK_TRY(cudaGetLastError());
        MGK_TRY(cudaFreeAsync(kv, s));
        MGK_TRY(cudaFreeAsync(ka, s));
    }
    unsigned long long *keys = nullptr, *alt = nullptr;
    MGK_TRY(mapped_sorted_keys(g, perm, keys, alt, s));
    MGK_TRY(cudaStreamSynchronize(s));
    Graph old;
    old.rp = g->rp, old.ci = g->ci, old.cp = g->cp, old.ri = g->ri;
    old.no_in = g->no_in, old.pull_skip = g->pull_skip, old.heavy = g->heavy;
    g->heavy = nullptr;
    cudaFree(g->top4);  // (derived from the CSC being replaced; rebuilt on the next use)
    g->top4 = nullptr;
    cudaError_t e = graph_from_sorted_keys(g, keys, alt, m, s);
    if (!e) e = cudaStreamSynchronize(s);
    cudaFreeAsync(keys, s);
    cudaFreeAsync(alt, s);
    cudaStreamSynchronize(s);
    free_device_graph(&old);
    if (e) {
        cudaFree(perm);
        cudaFree(inv);
        return e;
    }
    g->perm = perm;
    g->inv = inv;
    g->dg.perm = perm;
    g->dg.inv = inv;
    g->bytes += 2 * (size_t)n * 4;
    return cudaSuccess;
}

cudaError_t build_device_graph_generated(Graph* g, uint32_t scale, uint32_t edge_factor, double a,
                                         double b, double c, uint64_t rng_seed, uint64_t target,
                                         int relabel) {
    cudaStream_t s;
    MGK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    unsigned long long *keys = nullptr, *alt = nullptr;
    uint64_t m = 0, n = 0;
    cudaError_t e = gen_rmat_device(scale, edge_factor, a, b, c, rng_seed, target, relabel, &keys, &m, &n, s);
    if (!e && (n >= 0xFFFFFFFFull || m >= 0xFFFFFFFFull)) e = cudaErrorInvalidValue;
    if (!e) e = cudaMallocAsync(&alt, std::max<uint64_t>(m, 1) * 8, s);
    if (!e) {
        g->dg.n = (uint32_t)n;
        e = graph_from_sorted_keys(g, keys, alt, m, s);
    }
    if (!e) e = cudaStreamSynchronize(s);
    if (keys) cudaFreeAsync(keys, s);
    if (alt) cudaFreeAsync(alt, s);
    keys = alt = nullptr;
    if (!e) e = locality_relabel(g, s);
    if (keys) cudaFreeAsync(keys, s);
    if (alt) cudaFreeAsync(alt, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return e;
}

cudaError_t build_device_graph(Graph* g, const uint32_t* h_rp, const uint32_t* h_ci) {
    const uint32_t n = g->dg.n;
    const uint64_t m = g->dg.m;
    MGK_TRY(alloc_graph(g, n, m));
    cudaStream_t s;
    MGK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    MGK_TRY(cudaMemcpyAsync(g->rp, h_rp, (size_t)(n + 1) * 4, cudaMemcpyHostToDevice, s));
    if (m) MGK_TRY(cudaMemcpyAsync(g->ci, h_ci, m * 4, cudaMemcpyHostToDevice, s));
    cudaError_t e = build_csc(g, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = locality_relabel(g, s);
    cudaStreamDestroy(s);
    return e;
}

// CSR + CSC + pull metadata from sorted unique (src << 32 | dst) keys; `alt`
// is a scratch buffer of the same size. Keys are consumed (reordered).
cudaError_t graph_from_sorted_keys(Graph* g, unsigned long long*& keys, unsigned long long*& alt,
                                   uint64_t m, cudaStream_t s) {
    const uint32_t n = g->dg.n;
    g->dg.m = m;
    MGK_TRY(alloc_graph(g, n, m));
    g->dg.rows_unique = 1;  // sorted unique keys
    if (m) {
        keys_to_csr<<<blocks_for(m + 1), kTB, 0, s>>>(keys, m, n, g->rp, g->ci);
        swap_halves<<<blocks_for(m), kTB, 0, s>>>(keys, m);
        MGK_TRY(radix_sort_keys(keys, alt, m, 32 + key_bits(n), s));
        keys_to_csr<<<blocks_for(m + 1), kTB, 0, s>>>(keys, m, n, g->cp, g->ri);
        MGK_TRY(order_in_lists(g, keys, alt, s));
    } else {
        MGK_TRY(cudaMemsetAsync(g->rp, 0, (size_t)(n + 1) * 4, s));
        MGK_TRY(cudaMemsetAsync(g->cp, 0, (size_t)(n + 1) * 4, s));
    }
    no_in_bitmap<<<blocks_for(g->dg.nwords), kTB, 0, s>>>(g->cp, n, g->dg.nwords, g->no_in);
    MGK_TRY(cudaGetLastError());
    return build_heavy(g, s);
}

cudaError_t build_device_graph_from_edges(Graph* g, const uint32_t* h_src, const uint32_t* h_dst,
                                          uint64_t nedges) {
    const uint32_t n = g->dg.n;
    cudaStream_t s;
    MGK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    uint64_t m = 0;
    cudaError_t e = cudaSuccess;
    unsigned long long *keys = nullptr, *alt = nullptr;
    uint32_t *src = nullptr, *dst = nullptr, *keep = nullptr;
    unsigned int* bad = nullptr;
    do {
        const size_t np = (size_t)std::max<uint64_t>(nedges, 1);
        if ((e = cudaMallocAsync(&keys, np * 8, s))) break;
        if ((e = cudaMallocAsync(&alt, np * 8, s))) break;
        if ((e = cudaMallocAsync(&src, np * 4, s))) break;
        if ((e = cudaMallocAsync(&dst, np * 4, s))) break;
        if ((e = cudaMallocAsync(&bad, 4, s))) break;
        if ((e = cudaMemsetAsync(bad, 0xFF, 4, s))) break;
        if (nedges) {
            if ((e = cudaMemcpyAsync(src, h_src, nedges * 4, cudaMemcpyHostToDevice, s))) break;
            if ((e = cudaMemcpyAsync(dst, h_dst, nedges * 4, cudaMemcpyHostToDevice, s))) break;
            pack_edges<<<blocks_for(nedges), kTB, 0, s>>>(src, dst, nedges, n, keys, bad);
        }
        unsigned int h_bad = 0;
        if ((e = cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, s))) break;
        if ((e = cudaStreamSynchronize(s))) break;
        if (h_bad != 0xFFFFFFFFu) {
            e = cudaErrorInvalidValue;  // caller reports the ContractError
            break;
        }
        cudaFreeAsync(src, s);
        cudaFreeAsync(dst, s);
        src = dst = nullptr;
        if (nedges) {
            if ((e = radix_sort_keys(keys, alt, nedges, 32 + key_bits(n), s))) break;
            // dedup: keep first of each run, compact with cub::DeviceSelect::Flagged
            if ((e = cudaMallocAsync(&keep, nedges * 4, s))) break;
            mark_unique<<<blocks_for(nedges), kTB, 0, s>>>(keys, nedges, keep);
            unsigned long long* d_num = nullptr;
            if ((e = cudaMallocAsync(&d_num, 8, s))) break;
            size_t tmp = 0;
            if ((e = cub::DeviceSelect::Flagged(nullptr, tmp, keys, keep, alt, d_num, (int64_t)nedges, s)))
                break;
            void* t = nullptr;
            if ((e = cudaMallocAsync(&t, tmp, s))) break;
            if ((e = cub::DeviceSelect::Flagged(t, tmp, keys, keep, alt, d_num, (int64_t)nedges, s)))
                break;
            unsigned long long h_num = 0;
            if ((e = cudaMemcpyAsync(&h_num, d_num, 8, cudaMemcpyDeviceToHost, s))) break;
            if ((e = cudaStreamSynchronize(s))) break;
            cudaFreeAsync(t, s);
            cudaFreeAsync(d_num, s);
            std::swap(keys, alt);
            m = h_num;
        }
        if (m >= 0xFFFFFFFFull) {
            e = cudaErrorInvalidValue;
            break;
        }
        if ((e = graph_from_sorted_keys(g, keys, alt, m, s))) break;
        e = cudaStreamSynchronize(s);
    } while (0);
    if (keys) cudaFreeAsync(keys, s);
    if (alt) cudaFreeAsync(alt, s);
    if (src) cudaFreeAsync(src, s);
    if (dst) cudaFreeAsync(dst, s);
    if (keep) cudaFreeAsync(keep, s);
    if (bad) cudaFreeAsync(bad, s);
    cudaStreamSynchronize(s);
    keys = alt = nullptr;
    if (!e) e = locality_relabel(g, s);
    cudaStreamDestroy(s);
    return e;
}

cudaError_t download_graph(const Graph* g, uint32_t* h_rp, uint32_t* h_ci, uint32_t* h_cp, uint32_t* h_ri) {
    const uint32_t n = g->dg.n;
    const uint64_t m = g->dg.m;
    auto copy_out = [&](const Graph* src) -> cudaError_t {
        if (h_rp) MGK_TRY(cudaMemcpy(h_rp, src->rp, (size_t)(n + 1) * 4, cudaMemcpyDeviceToHost));
        if (h_ci && m) MGK_TRY(cudaMemcpy(h_ci, src->ci, m * 4, cudaMemcpyDeviceToHost));
        if (h_cp) MGK_TRY(cudaMemcpy(h_cp, src->cp, (size_t)(n + 1) * 4, cudaMemcpyDeviceToHost));
        if (h_ri && m) MGK_TRY(cudaMemcpy(h_ri, src->ri, m * 4, cudaMemcpyDeviceToHost));
        return cudaSuccess;
    };
    if (!g->inv) return copy_out(g);
    // relabelled: rebuild the external-id graph (same CSC ordering rules) once
    cudaStream_t s;
    MGK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    Graph tmp;
    tmp.dg.n = n;
    unsigned long long *keys = nullptr, *alt = nullptr;
    cudaError_t e = mapped_sorted_keys(g, g->inv, keys, alt, s);
    if (!e) e = graph_from_sorted_keys(&tmp, keys, alt, m, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (!e) e = copy_out(&tmp);
    if (keys) cudaFreeAsync(keys, s);
    if (alt) cudaFreeAsync(alt, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    free_device_graph(&tmp);
    return e;
}

cudaError_t ids_to_external(const Graph* g, unsigned long long* d_ids, uint64_t n, cudaStream_t s) {
    if (!g->inv || n == 0) return cudaSuccess;
    map_ids<<<blocks_for(n), kTB, 0, s>>>(d_ids, n, g->inv);
    MGK_TRY(cudaGetLastError());
    unsigned long long* alt = nullptr;
    MGK_TRY(cudaMallocAsync(&alt, n * 8, s));
    unsigned long long* keys = d_ids;
    MGK_TRY(radix_sort_keys(keys, alt, n, key_bits(g->dg.n), s));
    if (keys != d_ids) MGK_TRY(cudaMemcpyAsync(d_ids, keys, n * 8, cudaMemcpyDeviceToDevice, s));
    // radix_sort_keys swaps the pointers when the result landed in alt
    MGK_TRY(cudaFreeAsync(keys == d_ids ? alt : keys, s));
    return cudaSuccess;
}

// A copy of src's device arrays on dst->device (peer copies over NVLink when
// the devices differ): load-time replication for seed-sharded multi-GPU runs.
cudaError_t replicate_device_graph(const Graph* src, Graph* dst) {
    const uint32_t n = src->dg.n;
    const uint64_t m = src->dg.m;
    int can = 0;
    if (dst->device != src->device &&
        cudaDeviceCanAccessPeer(&can, dst->device, src->device) == cudaSuccess && can) {
        if (cudaDeviceEnablePeerAccess(src->device, 0) != cudaSuccess) cudaGetLastError();
    }
    MGK_TRY(alloc_graph(dst, n, m));
    dst->dg = src->dg;
    dst->dg.rp = dst->rp;
    dst->dg.ci = dst->ci;
    dst->dg.cp = dst->cp;
    dst->dg.ri = dst->ri;
    dst->dg.no_in = dst->no_in;
    dst->dg.pull_skip = dst->pull_skip;
    dst->dg.bad_seed = dst->bad_seed;
    const size_t mp = (size_t)std::max<uint64_t>(m, 1);
    const size_t nh = (size_t)std::max<uint32_t>(src->dg.nheavy, 1);
    MGK_TRY(cudaMalloc(&dst->heavy, nh * sizeof(uint2)));
    dst->dg.heavy = dst->heavy;
    dst->bytes = src->bytes;
    dst->tuning = src->tuning;
    auto cp = [&](void* d, const void* s, size_t b) {
        return cudaMemcpyPeer(d, dst->device, s, src->device, b);
    };
    MGK_TRY(cp(dst->rp, src->rp, (size_t)(n + 1) * 4));
    MGK_TRY(cp(dst->ci, src->ci, mp * 4));
    MGK_TRY(cp(dst->cp, src->cp, (size_t)(n + 1) * 4));
    MGK_TRY(cp(dst->ri, src->ri, mp * 4));
    MGK_TRY(cp(dst->no_in, src->no_in, (size_t)(src->dg.nwords + 1) * 4));
    MGK_TRY(cp(dst->pull_skip, src->pull_skip, (size_t)(src->dg.nwords + 1) * 4));
    MGK_TRY(cp(dst->heavy, src->heavy, nh * sizeof(uint2)));
    if (src->perm) {
        MGK_TRY(cudaMalloc(&dst->perm, (size_t)n * 4));
        MGK_TRY(cudaMalloc(&dst->inv, (size_t)n * 4));
        MGK_TRY(cp(dst->perm, src->perm, (size_t)n * 4));
        MGK_TRY(cp(dst->inv, src->inv, (size_t)n * 4));
    }
    dst->dg.perm = dst->perm;
    dst->dg.inv = dst->inv;
    return cudaDeviceSynchronize();
}

namespace {
// one warp per row: every entry (r, c) of A becomes the key (c << 32 | r) of
// A^T, in external ids (inv maps a relabelled device id back; null = identity)
__global__ void transpose_keys(const uint32_t* rp, const uint32_t* ci, uint32_t n, const uint32_t* inv,
                               unsigned long long* keys) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const uint32_t b = rp[r], e = rp[r + 1];
        const uint32_t xr = inv ? inv[r] : (uint32_t)r;
        for (uint32_t p = b + lane; p < e; p += 32) {
            const uint32_t c = ci[p];
            keys[p] = ((unsigned long long)(inv ? inv[c] : c) << 32) | xr;
        }
    }
}
}  // namespace

// A^T as its own device graph (CSR of A^T = CSC of A, rows ascending), built
// from src's device arrays: the `<-` direction of a Cypher walk
// (execute.cpp:35-39 uses transposed_matrix).
cudaError_t transpose_device_graph(const Graph* src, Graph* dst) {
    const uint32_t n = src->dg.n;
    const uint64_t m = src->dg.m;
    cudaStream_t s;
    MGK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    unsigned long long *keys = nullptr, *alt = nullptr;
    cudaError_t e = cudaSuccess;
    do {
        const size_t mp = (size_t)std::max<uint64_t>(m, 1);
        if ((e = cudaMallocAsync(&keys, mp * 8, s))) break;
        if ((e = cudaMallocAsync(&alt, mp * 8, s))) break;
        if (m) {
            transpose_keys<<<std::min<uint64_t>((n + 7) / 8, 1u << 20), 256, 0, s>>>(src->dg.rp, src->dg.ci, n,
                                                                                    src->dg.inv, keys);
            if ((e = cudaGetLastError())) break;
        }
        dst->dg.n = n;
        e = graph_from_keys(dst, keys, alt, m, s);
    } while (0);
    cudaFreeAsync(keys, s);
    cudaFreeAsync(alt, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return e;
}

namespace {
__global__ void gather_degrees(const uint32_t* rp, const uint32_t* perm, uint32_t n, const uint32_t* seeds,
                               uint64_t ns, uint32_t* deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ns; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = seeds[i];
        if (s >= n) {
            deg[i] = 0;
            continue;
        }
        if (perm) s = perm[s];
        deg[i] = rp[s + 1] - rp[s];
    }
}
}  // namespace

// out-degrees of (external) seed ids, for cost-balanced seed shards
cudaError_t seed_degrees(const Graph* g, const uint32_t* h_seeds, uint64_t ns, uint32_t* h_deg) {
    if (ns == 0) return cudaSuccess;
    cudaStream_t s;
    MGK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    uint32_t *d_s = nullptr, *d_d = nullptr;
    cudaError_t e = cudaSuccess;
    do {
        if ((e = cudaMallocAsync(&d_s, ns * 4, s))) break;
        if ((e = cudaMallocAsync(&d_d, ns * 4, s))) break;
        if ((e = cudaMemcpyAsync(d_s, h_seeds, ns * 4, cudaMemcpyHostToDevice, s))) break;
        gather_degrees<<<(unsigned)std::min<uint64_t>((ns + 255) / 256, 4096), 256, 0, s>>>(g->dg.rp, g->dg.perm, g->dg.n,
                                                                                          d_s, ns, d_d);
        if ((e = cudaGetLastError())) break;
        if ((e = cudaMemcpyAsync(h_deg, d_d, ns * 4, cudaMemcpyDeviceToHost, s))) break;
        e = cudaStreamSynchronize(s);
    } while (0);
    cudaFreeAsync(d_s, s);
    cudaFreeAsync(d_d, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return e;
}

// sort + unique (src << 32 | dst) keys, then CSR + CSC (keys/alt: m entries each, consumed)
cudaError_t graph_from_keys(Graph* g, unsigned long long*& keys, unsigned long long*& alt, uint64_t m,
                            cudaStream_t s) {
    uint64_t mu = 0;
    if (m) {
        MGK_TRY(radix_sort_keys(keys, alt, m, 32 + key_bits(g->dg.n), s));
        uint32_t* keep = nullptr;
        unsigned long long* d_num = nullptr;
        MGK_TRY(cudaMallocAsync(&keep, m * 4, s));
        MGK_TRY(cudaMallocAsync(&d_num, 8, s));
        mark_unique<<<blocks_for(m), kTB, 0, s>>>(keys, m, keep);
        size_t tmp = 0;
        MGK_TRY(cub::DeviceSelect::Flagged(nullptr, tmp, keys, keep, alt, d_num, (int64_t)m, s));
        void* t = nullptr;
        MGK_TRY(cudaMallocAsync(&t, tmp, s));
        MGK_TRY(cub::DeviceSelect::Flagged(t, tmp, keys, keep, alt, d_num, (int64_t)m, s));
        unsigned long long h_num = 0;
        MGK_TRY(cudaMemcpyAsync(&h_num, d_num, 8, cudaMemcpyDeviceToHost, s));
        MGK_TRY(cudaStreamSynchronize(s));
        cudaFreeAsync(t, s);
        cudaFreeAsync(d_num, s);
        cudaFreeAsync(keep, s);
        std::swap(keys, alt);
        mu = h_num;
    }
    if (mu >= 0xFFFFFFFFull) return cudaErrorInvalidValue;
    MGK_TRY(graph_from_sorted_keys(g, keys, alt, mu, s));
    return cudaStreamSynchronize(s);
}

void free_device_graph(Graph* g) {
    cudaFree(g->rp);
    cudaFree(g->ci);
    cudaFree(g->cp);
    cudaFree(g->ri);
    cudaFree(g->no_in);
    cudaFree(g->pull_skip);
    cudaFree(g->heavy);
    cudaFree(g->perm);
    cudaFree(g->inv);
    cudaFree(g->k2_split);
    cudaFree(g->top4);
    g->top4 = nullptr;
    cudaFree(g->bad_seed);
    g->bad_seed = nullptr;
    g->dg.bad_seed = nullptr;
    g->k2_split = nullptr;
    g->k2_split_bits = g->k2_split_R = 0;
    g->rp = g->ci = g->cp = g->ri = g->no_in = g->pull_skip = nullptr;
    g->heavy = nullptr;
    g->perm = g->inv = nullptr;
    g->dg.perm = g->dg.inv = nullptr;
}

}  // namespace mgk
