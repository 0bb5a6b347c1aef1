// SINGLE engine: one seed at a time, bitmap state, direction-optimizing BFS.
//
// Replaces the per-query loop of k_hop_frontier (proj/core/src/execute.cpp:347-371)
// and its vxm / ewise_union calls (proj/core/src/sparse.cpp:253-290, 365-377):
//   * visited / frontier sets are bitmaps (n/8 bytes, L2-resident) instead of
//     sorted uint64 vectors plus two dense char arrays zeroed every hop;
//   * the masked vxm is a push pass over the frontier's out-edges (CSR) with
//     atomicOr test-and-set on the visited bitmap, or a pull pass over the
//     unvisited vertices' in-edges (CSC) that stops at the first frontier hit;
//   * ewise_union is the same atomicOr, and nvals is a discovery counter.
// All hops of all seeds run inside one persistent cooperative launch; hops are
// separated by grid-wide barriers and every direction / early-exit decision is
// taken on the device from counters all CTAs read after the barrier, so there
// is no host round trip per hop.
//
// Push work items are (begin, end) slices of at most kChunk adjacency entries,
// written when a vertex is discovered, so a 97K-degree hub is spread over
// ~3K warp iterations instead of serialising one warp; each warp merges 32
// items with a shuffle scan and reads the adjacency in coalesced runs.
#include "mgk_device.cuh"

namespace mgk {
namespace {

using namespace dev;

constexpr int kBlock = 512;
constexpr int kWarps = kBlock / 32;
constexpr int kStageCap = 256;

struct SSParams {
    DevGraph g;
    const uint32_t* seeds;
    uint32_t nseeds;
    uint32_t k;
    int mode;
    unsigned long long* counts;
    uint32_t* visited;
    uint32_t* fb0;
    uint32_t* fb1;
    uint32_t* fb2;
    uint2* items0;
    uint2* items1;
    QCtl* qctl;                // [3], indexed by hop % 3
    unsigned long long* misc;  // [0] unexplored in-edges, [1] final bitmap id, [2] last seed
    LevelCounters* lc;
    uint32_t alpha, beta, force_dir;
};

__device__ __forceinline__ uint32_t* fb_of(const SSParams& P, uint32_t i) {
    return i == 0 ? P.fb0 : (i == 1 ? P.fb1 : P.fb2);
}
__device__ __forceinline__ uint2* items_of(const SSParams& P, uint32_t i) {
    return (i & 1) ? P.items1 : P.items0;
}

// Per-thread counters of one phase, reduced per block and flushed once.
struct Acc {
    unsigned long long found, edges, indeg, scanned, candidates;
    __device__ void zero() { found = edges = indeg = scanned = candidates = 0; }
};

__device__ void block_flush(Acc& a, QCtl* q, LevelCounters* lc, unsigned long long* unexplored) {
    __shared__ unsigned long long s[5];
    if (threadIdx.x < 5) s[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long f = warp_sum_u64(a.found), e = warp_sum_u64(a.edges),
                             i = warp_sum_u64(a.indeg), sc = warp_sum_u64(a.scanned),
                             c = warp_sum_u64(a.candidates);
    if (lane_id() == 0) {
        if (f) atomicAdd(&s[0], f);
        if (e) atomicAdd(&s[1], e);
        if (i) atomicAdd(&s[2], i);
        if (sc) atomicAdd(&s[3], sc);
        if (c) atomicAdd(&s[4], c);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s[0]) {
            atomicAdd(&q->nfound, (unsigned int)s[0]);
            atomicAdd(&lc->frontier, s[0]);
            atomicAdd(&lc->vertices, s[0]);
        }
        if (s[1]) atomicAdd(&q->edges, s[1]);
        if (s[2]) {
            atomicAdd(&q->indeg, s[2]);
            atomicAdd(unexplored, 0ULL - s[2]);
        }
        if (s[3]) atomicAdd(&lc->scanned, s[3]);
        if (s[4]) atomicAdd(&lc->candidates, s[4]);
    }
    __syncthreads();
    a.zero();
}

__device__ __forceinline__ void count_found(const DevGraph& g, uint32_t u, Acc& acc) {
    acc.found += 1;
    acc.edges += __ldg(g.rp + u + 1) - __ldg(g.rp + u);
    acc.indeg += __ldg(g.cp + u + 1) - __ldg(g.cp + u);
}

// Push: expand the frontier's work items; test-and-set visited; stage the
// newly discovered vertices and turn them into next-hop work items.
__device__ void push_phase(const SSParams& P, const uint2* items, uint32_t nitems, uint32_t* fnext,
                           uint2* items_next, QCtl* qn, Acc& acc, Stage<kStageCap>& st,
                           uint32_t warp_gid, uint32_t nwarps) {
    const uint32_t lane = lane_id();
    const DevGraph& g = P.g;
    for (uint32_t base = warp_gid * 32; base < nitems; base += nwarps * 32) {
        const uint32_t idx = base + lane;
        const uint2 it = idx < nitems ? items[idx] : make_uint2(0, 0);
        const uint32_t len = it.y - it.x;
        const uint32_t incl = warp_incl_scan(len);
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        const uint32_t off = it.x - (incl - len);
        for (uint32_t x0 = 0; x0 < total; x0 += 32) {
            const uint32_t x = x0 + lane;
            const bool valid = x < total;
            const uint32_t j = warp_owner(incl, valid ? x : total - 1);
            const uint32_t pos = __shfl_sync(kFull, off, j) + x;
            bool found = false;
            uint32_t u = 0;
            if (valid) {
                u = __ldg(g.ci + pos);
                const uint32_t w = u >> 5, bit = 1u << (u & 31);
                if (!(ld_cg(P.visited + w) & bit)) {
                    const uint32_t old = atomicOr(P.visited + w, bit);
                    if (!(old & bit)) {
                        found = true;
                        atomicOr(fnext + w, bit);
                        count_found(g, u, acc);
                    }
                }
            }
            acc.scanned += valid;
            st.push(found, u);
            if (st.full()) {
                emit_items(g.rp, st.buf, st.n, items_next, &qn->nitems);
                st.n = 0;
            }
        }
    }
    emit_items(g.rp, st.buf, st.n, items_next, &qn->nitems);
    st.n = 0;
}

// Pull: every unvisited vertex with in-edges scans its in-neighbours (CSC,
// ascending) until one is in the current frontier. One warp owns one bitmap
// word (32 vertices), so visited / next words are written without atomics.
__device__ void pull_phase(const SSParams& P, const uint32_t* fcur, uint32_t* fnext, Acc& acc,
                           uint32_t warp_gid, uint32_t nwarps) {
    const uint32_t lane = lane_id();
    const DevGraph& g = P.g;
    for (uint32_t w = warp_gid; w < g.nwords; w += nwarps) {
        const uint32_t vis = ld_cg(P.visited + w);
        const uint32_t done = vis | __ldg(g.no_in + w);
        if (done == kFull) continue;
        const uint32_t u = w * 32 + lane;
        const bool cand = !((done >> lane) & 1u);
        uint32_t b = 0, e = 0;
        if (cand) {
            b = __ldg(g.cp + u);
            e = __ldg(g.cp + u + 1);
        }
        bool found = false;
        uint32_t scanned = 0;
        if (cand && e - b <= 32) {
            for (uint32_t p = b; p < e; ++p) {
                const uint32_t v = __ldg(g.ri + p);
                ++scanned;
                if ((fcur[v >> 5] >> (v & 31)) & 1u) {
                    found = true;
                    break;
                }
            }
        }
        unsigned big = __ballot_sync(kFull, cand && e - b > 32);
        while (big) {
            const int j = __ffs(big) - 1;
            big &= big - 1;
            const uint32_t bj = __shfl_sync(kFull, b, j), ej = __shfl_sync(kFull, e, j);
            bool hit = false;
            uint32_t sc = ej - bj;
            for (uint32_t p0 = bj; p0 < ej; p0 += 32) {
                const uint32_t p = p0 + lane;
                bool h = false;
                if (p < ej) {
                    const uint32_t v = __ldg(g.ri + p);
                    h = (fcur[v >> 5] >> (v & 31)) & 1u;
                }
                const unsigned hm = __ballot_sync(kFull, h);
                if (hm) {
                    hit = true;
                    sc = p0 - bj + __ffs(hm);
                    break;
                }
            }
            if ((int)lane == j) {
                found = hit;
                scanned += sc;
            }
        }
        acc.candidates += cand;
        acc.scanned += scanned;
        const unsigned fm = __ballot_sync(kFull, found);
        if (fm) {
            if (lane == 0) {
                P.visited[w] = vis | fm;
                fnext[w] = fm;
            }
            if (found) count_found(g, u, acc);
        }
    }
}

// Re-derive push items from a frontier bitmap (after a pull hop).
__device__ void compact_phase(const SSParams& P, const uint32_t* fcur, uint2* items, QCtl* q,
                              Stage<kStageCap>& st, uint32_t warp_gid, uint32_t nwarps) {
    const uint32_t lane = lane_id();
    for (uint32_t w = warp_gid; w < P.g.nwords; w += nwarps) {
        const uint32_t bits = fcur[w];
        if (bits == 0) continue;
        st.push((bits >> lane) & 1u, w * 32 + lane);
        if (st.full()) {
            emit_items(P.g.rp, st.buf, st.n, items, &q->nitems);
            st.n = 0;
        }
    }
    emit_items(P.g.rp, st.buf, st.n, items, &q->nitems);
    st.n = 0;
}

__global__ void __launch_bounds__(kBlock) ss_kernel(SSParams P) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t s_stage[kWarps][kStageCap];
    const uint32_t gtid = blockIdx.x * kBlock + threadIdx.x;
    const uint32_t nthreads = gridDim.x * kBlock;
    const uint32_t warp_gid = gtid >> 5;
    const uint32_t nwarps = nthreads >> 5;
    const DevGraph& g = P.g;
    Acc acc;
    acc.zero();
    Stage<kStageCap> st{s_stage[threadIdx.x >> 5], 0};

    for (uint32_t qi = 0; qi < P.nseeds; ++qi) {
        const uint32_t seed = P.seeds[qi];
        // ---- init: clear state --------------------------------------------
        for (uint32_t w = gtid; w < g.nwords; w += nthreads) {
            P.visited[w] = 0;
            P.fb0[w] = 0;
            P.fb1[w] = 0;
            P.fb2[w] = 0;
        }
        if (gtid < 3) P.qctl[gtid] = QCtl{0, 0, 0, 0, 0};
        grid.sync();
        if (warp_gid == 0) {
            const bool me = lane_id() == 0;
            if (me) {
                P.visited[seed >> 5] = 1u << (seed & 31);
                P.fb0[seed >> 5] = 1u << (seed & 31);
                Acc a0;
                a0.zero();
                count_found(g, seed, a0);
                P.qctl[0].nfound = 1;
                P.qctl[0].edges = a0.edges;
                P.qctl[0].indeg = a0.indeg;
                P.misc[0] = g.m - a0.indeg;
            }
            st.push(me, seed);
            emit_items(g.rp, st.buf, st.n, P.items0, &P.qctl[0].nitems);
            st.n = 0;
        }
        grid.sync();

        unsigned long long cum = 0, last = 1;
        bool pull = false, items_ready = true;
        uint32_t hop = 1;
        for (; hop <= P.k; ++hop) {
            const uint32_t cur = (hop - 1) % 3, nxt = hop % 3, clr = (hop + 1) % 3;
            QCtl* qc = &P.qctl[cur];
            QCtl* qn = &P.qctl[nxt];
            const unsigned long long nf = ld_volatile(&qc->nfound);
            const unsigned long long mf = ld_volatile(&qc->edges);
            const unsigned long long mu = ld_volatile(&P.misc[0]);
            if (P.force_dir == 1) {
                pull = false;
            } else if (P.force_dir == 2) {
                pull = true;
            } else if (!pull) {
                pull = mf * P.alpha > mu;
            } else {
                pull = nf * P.beta >= g.n;
            }
            uint32_t* fcur = fb_of(P, cur);
            uint32_t* fnext = fb_of(P, nxt);
            uint32_t* fclr = fb_of(P, clr);
            unsigned long long t0 = 0;
            if (gtid == 0) {
                t0 = globaltimer();
                atomicAdd(&P.lc[hop].runs, 1u);
                if (pull) atomicAdd(&P.lc[hop].pull_runs, 1u);
                atomicAdd(&P.lc[hop].edges, mf);
                atomicAdd(&P.lc[hop].union_edges, mf);
            }
            if (!pull && !items_ready) {
                compact_phase(P, fcur, items_of(P, cur), qc, st, warp_gid, nwarps);
                grid.sync();
            }
            for (uint32_t w = gtid; w < g.nwords; w += nthreads) fclr[w] = 0;
            if (gtid == 0) P.qctl[clr] = QCtl{0, 0, 0, 0, 0};
            if (pull) {
                pull_phase(P, fcur, fnext, acc, warp_gid, nwarps);
                items_ready = false;
            } else {
                push_phase(P, items_of(P, cur), ld_volatile(&qc->nitems), fnext, items_of(P, nxt),
                           qn, acc, st, warp_gid, nwarps);
                items_ready = true;
            }
            block_flush(acc, qn, &P.lc[hop], &P.misc[0]);
            grid.sync();
            if (gtid == 0) atomicAdd(&P.lc[hop].ns, globaltimer() - t0);
            const unsigned long long found = ld_volatile(&qn->nfound);
            cum += found;
            last = found;
            if (found == 0) break;
        }
        if (gtid == 0) {
            P.counts[qi] = P.mode == MGK_EXACT ? last : cum;
            P.misc[1] = (last != 0 && hop > P.k) ? (P.k % 3) : 3ULL;
            P.misc[2] = seed;
        }
        grid.sync();
    }
}

// ---- result ids (k_hop_frontier) ---------------------------------------------
__global__ void popc_words(const uint32_t* bits, uint32_t nwords, uint32_t drop, uint32_t* out) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwords) return;
    uint32_t x = bits[w];
    if ((drop >> 5) == w) x &= ~(1u << (drop & 31));
    out[w] = __popc(x);
}

__global__ void scatter_ids(const uint32_t* bits, uint32_t nwords, uint32_t drop,
                            const uint32_t* offs, unsigned long long* ids) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwords) return;
    uint32_t x = bits[w];
    if ((drop >> 5) == w) x &= ~(1u << (drop & 31));
    uint32_t o = offs[w];
    while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        ids[o++] = (unsigned long long)w * 32 + b;
    }
}

}  // namespace

cudaError_t ensure_single_ws(const Graph* gr, Workspace* ws) {
    if (ws->visited) return cudaSuccess;
    const DevGraph& g = gr->dg;
    const size_t wb = (size_t)(g.nwords + 1) * 4;
    const size_t items = (size_t)(g.m / kChunk + g.n + 64);
    cudaError_t e;
    if ((e = cudaMalloc(&ws->visited, wb))) return e;
    for (int i = 0; i < 3; ++i)
        if ((e = cudaMalloc(&ws->fb[i], wb))) return e;
    for (int i = 0; i < 2; ++i)
        if ((e = cudaMalloc(&ws->ss_items[i], items * sizeof(uint2)))) return e;
    ws->bytes += 4 * wb + 2 * items * sizeof(uint2);
    return cudaSuccess;
}

cudaError_t launch_single(Launch& L) {
    const Graph* gr = L.g;
    Workspace* ws = L.ws;
    cudaError_t e = ensure_single_ws(gr, ws);
    if (e) return e;
    static int blocks_per_sm = 0, num_sms = 0;
    if (blocks_per_sm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, ss_kernel, kBlock, 0)))
            return e;
        if (blocks_per_sm < 1) return cudaErrorInvalidConfiguration;
    }
    SSParams P;
    P.g = gr->dg;
    P.seeds = L.d_seeds;
    P.nseeds = (uint32_t)L.nseeds;
    P.k = L.k;
    P.mode = L.mode;
    P.counts = L.d_counts;
    P.visited = ws->visited;
    P.fb0 = ws->fb[0];
    P.fb1 = ws->fb[1];
    P.fb2 = ws->fb[2];
    P.items0 = ws->ss_items[0];
    P.items1 = ws->ss_items[1];
    P.qctl = ws->qctl;
    P.misc = ws->misc;
    P.lc = ws->lc;
    P.alpha = L.tuning.alpha;
    P.beta = L.tuning.beta;
    P.force_dir = L.tuning.force_dir;
    L.grid = (uint32_t)(blocks_per_sm * num_sms);
    L.block = kBlock;
    void* args[] = {&P};
    return cudaLaunchCooperativeKernel((const void*)ss_kernel, dim3(L.grid), dim3(kBlock), args, 0,
                                       L.stream);
}

cudaError_t single_result_ids(const Graph* gr, Workspace* ws, uint32_t k, int mode, uint32_t seed,
                              unsigned long long* d_ids, unsigned long long* d_n, cudaStream_t s) {
    (void)k;
    const DevGraph& g = gr->dg;
    unsigned long long which = 0;
    cudaError_t e = cudaMemcpyAsync(&which, ws->misc + 1, 8, cudaMemcpyDeviceToHost, s);
    if (e) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    const uint32_t* bits = nullptr;
    uint32_t drop = 0xFFFFFFFFu;
    if (mode == MGK_CUMULATIVE) {
        bits = ws->visited;
        drop = seed;
    } else if (which < 3) {
        bits = ws->fb[which];
    } else {
        return cudaMemsetAsync(d_n, 0, 8, s);
    }
    // popcounts -> exclusive scan (+ total) -> scatter, all on the device.
    uint32_t* offs = nullptr;
    if ((e = cudaMallocAsync(&offs, (size_t)(g.nwords + 1) * 4, s))) return e;
    const int tb = 256, nb = (int)((g.nwords + tb - 1) / tb);
    popc_words<<<nb, tb, 0, s>>>(bits, g.nwords, drop, offs);
    if ((e = exclusive_scan_u32(offs, g.nwords, d_n, s))) return e;
    scatter_ids<<<nb, tb, 0, s>>>(bits, g.nwords, drop, offs, d_ids);
    cudaFreeAsync(offs, s);
    return cudaGetLastError();
}

}  // namespace mgk
