// Device-side generation of the BASELINE.json R-MAT bench graphs (§8(f) rank 1:
// the graph build before the hot path). Same definition as the host helper
// mgk_gen_rmat_csr (mgk_host.cpp), computed on the GPU:
//   * the edge stream: 64K-edge chunks, chunk c drawing from
//     mt19937_64(splitmix64(rng_seed * 0x2545F4914F6CDD1D + c)), one
//     top-53-bit uniform per level (bench.cpp:37-39, 107-137); self-loops are
//     dropped (they never change a count);
//   * the edge set: the first `target` distinct edges of that stream in
//     generation order (or every draw of edge_factor << scale when target = 0);
//   * relabel 1 / 2: seeded Fisher-Yates permutation of all ids / of the
//     non-isolated ids in ascending order (the permutation itself is drawn on
//     the host, it is 1 draw per id).
// One thread runs one chunk's mt19937_64 (state in local memory); dedup and
// selection are CUB radix sorts; the result feeds the usual CSR/CSC build.
#include <cub/cub.cuh>

#include <algorithm>
#include <random>
#include <vector>

#include "mgk_internal.cuh"

namespace mgk {
namespace {

#define MGK_TRY(x)                        \
    do {                                  \
        cudaError_t e_ = (x);             \
        if (e_ != cudaSuccess) return e_; \
    } while (0)

constexpr uint64_t kChunkEdges = 1u << 16;  // must match mgk_host.cpp
constexpr int kTB = 256;

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

// mt19937_64 (Matsumoto & Nishimura), identical to std::mt19937_64.
struct Mt64 {
    uint64_t mt[312];
    int i;
    __device__ void seed(uint64_t s) {
        mt[0] = s;
        for (int k = 1; k < 312; ++k) mt[k] = 6364136223846793005ULL * (mt[k - 1] ^ (mt[k - 1] >> 62)) + k;
        i = 312;
    }
    __device__ uint64_t next() {
        if (i >= 312) {
            const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
            int k = 0;
            for (; k < 156; ++k) {
                const uint64_t x = (mt[k] & UM) | (mt[k + 1] & LM);
                mt[k] = mt[k + 156] ^ (x >> 1) ^ ((x & 1) ? A : 0);
            }
            for (; k < 311; ++k) {
                const uint64_t x = (mt[k] & UM) | (mt[k + 1] & LM);
                mt[k] = mt[k - 156] ^ (x >> 1) ^ ((x & 1) ? A : 0);
            }
            const uint64_t x = (mt[311] & UM) | (mt[0] & LM);
            mt[311] = mt[155] ^ (x >> 1) ^ ((x & 1) ? A : 0);
            i = 0;
        }
        uint64_t x = mt[i++];
        x ^= (x >> 29) & 0x5555555555555555ULL;
        x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
        x ^= (x << 37) & 0xFFF7EEE000000000ULL;
        x ^= (x >> 43);
        return x;
    }
};

// One thread per chunk: keys[c * 64K + e] = src << 32 | dst, or `sentinel`
// for a self-loop or a draw beyond `raw_limit`.
__global__ void __launch_bounds__(64) gen_chunks(uint32_t scale, double a, double b, double c,
                                                 uint64_t rng_seed, uint64_t chunk0, uint64_t nchunks,
                                                 uint64_t raw_limit, unsigned long long sentinel,
                                                 unsigned long long* keys, unsigned long long* pos) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= nchunks) return;
    const uint64_t ch = chunk0 + t;
    Mt64 rng;
    rng.seed(splitmix64(rng_seed * 0x2545F4914F6CDD1DULL + ch));
    const double ab = a + b, abc = ab + c;
    unsigned long long* out = keys + t * kChunkEdges;
    unsigned long long* op = pos + t * kChunkEdges;
    for (uint64_t e = 0; e < kChunkEdges; ++e) {
        const uint64_t gidx = ch * kChunkEdges + e;
        if (gidx >= raw_limit) {
            out[e] = sentinel;
            op[e] = gidx;
            continue;
        }
        uint32_t s = 0, d = 0;
        for (uint32_t level = 0; level < scale; ++level) {
            const double r = (double)(rng.next() >> 11) * 0x1.0p-53;
            uint32_t sb = 0, db = 0;
            if (r < a) {
            } else if (r < ab) {
                db = 1;
            } else if (r < abc) {
                sb = 1;
            } else {
                sb = 1;
                db = 1;
            }
            s = (s << 1) | sb;
            d = (d << 1) | db;
        }
        out[e] = s == d ? sentinel : (((unsigned long long)s << 32) | d);
        op[e] = gidx;
    }
}

__global__ void mark_first(const unsigned long long* keys, uint64_t m, unsigned long long sentinel,
                           uint8_t* flag) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x)
        flag[p] = keys[p] != sentinel && (p == 0 || keys[p] != keys[p - 1]);
}

__global__ void mark_seen(const unsigned long long* keys, uint64_t m, uint32_t* seen) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)(keys[p] >> 32), d = (uint32_t)keys[p];
        atomicOr(seen + (s >> 5), 1u << (s & 31));
        atomicOr(seen + (d >> 5), 1u << (d & 31));
    }
}

__global__ void seen_to_count(const uint32_t* seen, uint64_t ids, uint32_t* cnt) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < ids;
         v += (uint64_t)gridDim.x * blockDim.x)
        cnt[v] = (seen[v >> 5] >> (v & 31)) & 1u;
}

// keys: (s, d) -> (perm[rank[s]], perm[rank[d]]); rank = exclusive scan of live flags
__global__ void relabel_keys(unsigned long long* keys, uint64_t m, const uint32_t* rank,
                             const uint32_t* perm) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < m;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)(keys[p] >> 32), d = (uint32_t)keys[p];
        keys[p] = ((unsigned long long)perm[rank[s]] << 32) | perm[rank[d]];
    }
}

unsigned blocks_for(uint64_t n) { return (unsigned)std::min<uint64_t>((n + kTB - 1) / kTB, 148ull * 64); }

int bits_for(uint64_t n) {
    int b = 1;
    while (b < 63 && (1ull << b) < n) ++b;
    return b;
}

template <typename K, typename V>
cudaError_t sort_pairs(K*& k, K*& kalt, V*& v, V*& valt, uint64_t n, int end_bit, cudaStream_t s) {
    cub::DoubleBuffer<K> dk(k, kalt);
    cub::DoubleBuffer<V> dv(v, valt);
    size_t tmp = 0;
    MGK_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, (int64_t)n, 0, end_bit, s));
    void* t = nullptr;
    MGK_TRY(cudaMallocAsync(&t, tmp, s));
    MGK_TRY(cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, (int64_t)n, 0, end_bit, s));
    MGK_TRY(cudaFreeAsync(t, s));
    if (dk.Current() != k) std::swap(k, kalt);
    if (dv.Current() != v) std::swap(v, valt);
    return cudaSuccess;
}

template <typename T>
cudaError_t select_flagged(const T* in, const uint8_t* flag, T* out, uint64_t n, uint64_t* nsel,
                           cudaStream_t s) {
    unsigned long long* d_n = nullptr;
    MGK_TRY(cudaMallocAsync(&d_n, 8, s));
    size_t tmp = 0;
    MGK_TRY(cub::DeviceSelect::Flagged(nullptr, tmp, in, flag, out, d_n, (int64_t)n, s));
    void* t = nullptr;
    MGK_TRY(cudaMallocAsync(&t, tmp, s));
    MGK_TRY(cub::DeviceSelect::Flagged(t, tmp, in, flag, out, d_n, (int64_t)n, s));
    unsigned long long h = 0;
    MGK_TRY(cudaMemcpyAsync(&h, d_n, 8, cudaMemcpyDeviceToHost, s));
    MGK_TRY(cudaStreamSynchronize(s));
    MGK_TRY(cudaFreeAsync(t, s));
    MGK_TRY(cudaFreeAsync(d_n, s));
    *nsel = h;
    return cudaSuccess;
}

}  // namespace

// Host side of the relabel permutation (mgk_host.cpp draws the same one).
void seeded_perm(uint64_t live, uint64_t rng_seed, std::vector<uint32_t>& perm) {
    perm.resize(live);
    for (uint64_t i = 0; i < live; ++i) perm[i] = (uint32_t)i;
    std::mt19937_64 rng(splitmix64(rng_seed ^ 0x5DEECE66DULL));
    for (uint64_t i = live; i > 1; --i) {
        const uint64_t max = UINT64_MAX, bound = i, limit = max - max % bound;
        uint64_t r = rng();
        while (r >= limit) r = rng();
        std::swap(perm[i - 1], perm[r % bound]);
    }
}

// Generates the edge set on the device; returns sorted unique (src<<32|dst)
// keys (device, caller frees with cudaFree) and the vertex count.
cudaError_t gen_rmat_device(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                            uint64_t rng_seed, uint64_t target, int relabel, unsigned long long** d_keys,
                            uint64_t* m_out, uint64_t* n_out, cudaStream_t s) {
    const uint64_t ids = 1ull << scale;
    const unsigned long long sentinel = (unsigned long long)ids << 32;
    const int key_end = 32 + scale + 1;
    const uint64_t raw_target = (uint64_t)edge_factor << scale;
    uint64_t raw = target ? target + target / 25 + kChunkEdges : raw_target;
    unsigned long long *keys = nullptr, *kalt = nullptr, *pos = nullptr, *palt = nullptr;
    uint8_t* flag = nullptr;
    uint64_t U = 0;
    for (;;) {
        const uint64_t nchunks = (raw + kChunkEdges - 1) / kChunkEdges;
        const uint64_t m = nchunks * kChunkEdges;
        MGK_TRY(cudaMallocAsync(&keys, m * 8, s));
        MGK_TRY(cudaMallocAsync(&kalt, m * 8, s));
        MGK_TRY(cudaMallocAsync(&pos, m * 8, s));
        MGK_TRY(cudaMallocAsync(&palt, m * 8, s));
        gen_chunks<<<(unsigned)((nchunks + 63) / 64), 64, 0, s>>>(
            scale, a, b, c, rng_seed, 0, nchunks, target ? UINT64_MAX : raw_target, sentinel, keys, pos);
        MGK_TRY(cudaGetLastError());
        // stable sort by key: equal keys keep generation order (pos ascending)
        MGK_TRY(sort_pairs(keys, kalt, pos, palt, m, key_end, s));
        MGK_TRY(cudaMallocAsync(&flag, m, s));
        mark_first<<<blocks_for(m), kTB, 0, s>>>(keys, m, sentinel, flag);
        MGK_TRY(cudaGetLastError());
        MGK_TRY(select_flagged(keys, flag, kalt, m, &U, s));
        uint64_t U2 = 0;
        MGK_TRY(select_flagged(pos, flag, palt, m, &U2, s));
        MGK_TRY(cudaFreeAsync(flag, s));
        std::swap(keys, kalt);
        std::swap(pos, palt);
        if (!target || U >= target) break;
        // not enough distinct edges: the stream prefix must be longer
        MGK_TRY(cudaFreeAsync(keys, s));
        MGK_TRY(cudaFreeAsync(kalt, s));
        MGK_TRY(cudaFreeAsync(pos, s));
        MGK_TRY(cudaFreeAsync(palt, s));
        raw = raw + (target - U) * 2 + kChunkEdges;
    }
    uint64_t M = U;
    if (target) {
        // first `target` distinct edges in generation order
        MGK_TRY(sort_pairs(pos, palt, keys, kalt, U, bits_for(raw + kChunkEdges) + 1, s));
        M = target;
        MGK_TRY(sort_pairs(keys, kalt, pos, palt, M, key_end, s));
    }
    MGK_TRY(cudaFreeAsync(pos, s));
    MGK_TRY(cudaFreeAsync(palt, s));
    uint64_t n = ids;
    if (relabel) {
        uint32_t *seen = nullptr, *rank = nullptr, *perm_d = nullptr;
        MGK_TRY(cudaMallocAsync(&seen, ((ids + 31) / 32 + 1) * 4, s));
        MGK_TRY(cudaMallocAsync(&rank, (ids + 1) * 4, s));
        uint64_t live = ids;
        if (relabel == 2) {
            MGK_TRY(cudaMemsetAsync(seen, 0, ((ids + 31) / 32 + 1) * 4, s));
            mark_seen<<<blocks_for(M), kTB, 0, s>>>(keys, M, seen);
        } else {
            MGK_TRY(cudaMemsetAsync(seen, 0xFF, ((ids + 31) / 32 + 1) * 4, s));
        }
        seen_to_count<<<blocks_for(ids), kTB, 0, s>>>(seen, ids, rank);
        unsigned long long* d_live = nullptr;
        MGK_TRY(cudaMallocAsync(&d_live, 8, s));
        MGK_TRY(exclusive_scan_u32(rank, (uint32_t)ids, d_live, s));
        unsigned long long hl = 0;
        MGK_TRY(cudaMemcpyAsync(&hl, d_live, 8, cudaMemcpyDeviceToHost, s));
        MGK_TRY(cudaStreamSynchronize(s));
        live = hl;
        std::vector<uint32_t> perm;
        seeded_perm(live, rng_seed, perm);
        MGK_TRY(cudaMallocAsync(&perm_d, (live + 1) * 4, s));
        MGK_TRY(cudaMemcpyAsync(perm_d, perm.data(), live * 4, cudaMemcpyHostToDevice, s));
        relabel_keys<<<blocks_for(M), kTB, 0, s>>>(keys, M, rank, perm_d);
        MGK_TRY(cudaGetLastError());
        cub::DoubleBuffer<unsigned long long> dk(keys, kalt);
        size_t tmp = 0;
        MGK_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp, dk, (int64_t)M, 0, 32 + bits_for(live), s));
        void* t = nullptr;
        MGK_TRY(cudaMallocAsync(&t, tmp, s));
        MGK_TRY(cub::DeviceRadixSort::SortKeys(t, tmp, dk, (int64_t)M, 0, 32 + bits_for(live), s));
        MGK_TRY(cudaFreeAsync(t, s));
        if (dk.Current() != keys) std::swap(keys, kalt);
        MGK_TRY(cudaStreamSynchronize(s));  // perm (host vector) is read by the copy above
        MGK_TRY(cudaFreeAsync(seen, s));
        MGK_TRY(cudaFreeAsync(rank, s));
        MGK_TRY(cudaFreeAsync(perm_d, s));
        MGK_TRY(cudaFreeAsync(d_live, s));
        n = live;
    }
    MGK_TRY(cudaFreeAsync(kalt, s));
    *d_keys = keys;
    *m_out = M;
    *n_out = n;
    return cudaStreamSynchronize(s);
}

}  // namespace mgk
