// LANES engine: bit-parallel multi-source k-hop, 64 seeds per uint64 lane word.
//
// A batch of up to 64*W seeds shares every adjacency pass: each vertex carries
// W uint64 words of visited (V), current-frontier (F) and next-frontier bits,
// bit (i % 64) of word (i / 64) belonging to seed i of the batch. One hop of
// the reference loop (proj/core/src/execute.cpp:359-363) for all lanes at once:
//   push:  for each frontier vertex v, each out-neighbour u:
//              F'[u] |= F[v] & ~V[u]                (vxm with NOT visited mask)
//   pull:  for each vertex u with a lane still unvisited:
//              F'[u] = (OR over in-neighbours v of F[v]) & ~V[u] & active,
//              stopping as soon as every needed lane is covered
//   then   V[u] |= F'[u]                            (ewise_union)
// Per-lane counts are popcounts of bit columns (ballot + popc per bit) over
// the discovered vertices: exact = |F_k| per lane, cumulative = sum over hops.
// Lanes are independent, so each lane's answer equals the single-seed
// k_hop_count bit for bit (a lane whose frontier empties stays empty, which is
// the reference's early exit at :361).
//
// Sparse bookkeeping keeps the cost proportional to the vertices a batch
// touches: a discovery list per hop (raw list R, one entry per vertex whose
// F' became non-zero) drives the finalize pass, the clearing of the previous
// frontier and the final clearing of V.
#include <cstdlib>
#include <type_traits>

#include "mgk_device.cuh"

namespace mgk {
namespace {

using namespace dev;

#ifndef MGK_MS_BLOCK
#define MGK_MS_BLOCK 256
#endif
#ifndef MGK_MS_MINB  // resident CTAs per SM the register budget is sized for (0: compiler's choice)
#define MGK_MS_MINB 0
#endif
constexpr int kBlock = MGK_MS_BLOCK;
// pull tuning (compile-time; variants are built for A/B runs): entries a lane
// scans per step of a short in-list, and entries of a longer list it scans
// before the warp takes over
#ifndef MGK_LIGHT_STEP
#define MGK_LIGHT_STEP 4
#endif
#ifndef MGK_PRE
#define MGK_PRE 16
#endif
#ifndef MGK_WPR_UNROLL  // warp-cooperative in-list scans: entries per lane in flight
#define MGK_WPR_UNROLL 2
#endif
constexpr int kWprUnroll = MGK_WPR_UNROLL;



// a lane's own in-list (read a few entries at a time by the same lane: its
// 32-byte sectors are re-read until the list is done, so by default they keep
// normal L2 priority; MGK_RI_LIGHT_STREAM marks them evict-first too)
__device__ __forceinline__ uint32_t ld_ri_lane(const uint32_t* p, unsigned long long pol) {
#ifdef MGK_RI_LIGHT_STREAM
    return dev::ldg_hint(p, pol);
#else
    (void)pol;
    return __ldg(p);
#endif
}
// The phases are inlined into the kernel (separate non-inlined functions, each
// with its own register allocation, measured 19 % slower on G4)
#ifdef MGK_NOINLINE_PHASES
#define MGK_PHASE __device__ __noinline__
#else
#define MGK_PHASE __device__
#endif
constexpr int kWarps = kBlock / 32;
constexpr int kStageCap = 256;
// first pull: lanes with at most m / MGK_STRAG frontier out-edges keep pushing (0: off; env MGK_STRAG).
// G4, 10 seeds, m/64: hop 3 scans 666M -> 248M entries (213M pulled + the stragglers' pushes), k = 6 5.31 -> 3.82 ms
// (16 / 256: 3.87 / 4.29 ms); with the mixed hop's push as fire-and-forget ORs (no list) m/32 is best: 3.57 ms
// (m/16 3.57, m/64 3.72; G2 0.430 vs 0.457 ms at m/64)
// one-word pulls start a candidate's scan from Graph::top4 (0: from the in-list; A/B builds)
#ifndef MGK_TOP4
#define MGK_TOP4 1
#endif
#ifndef MGK_STRAG_DEFAULT
#define MGK_STRAG_DEFAULT 32
#endif

struct MSParams {
    DevGraph g;
    const uint32_t* seeds;
    uint64_t nseeds;
    uint32_t k;             // max hop
    uint32_t min_hop;       // answer = sum over hops [min_hop, k] of each lane's |F_h|
    uint32_t ans_lo, ans_hi;  // the window answered into counts
    uint32_t nextra;        // further windows [xlo, xhi] -> xout (Launch::xout)
    uint32_t xlo[Launch::kMaxExtra], xhi[Launch::kMaxExtra];
    unsigned long long* xout[Launch::kMaxExtra];
    uint32_t seed_visited;  // 0: walk_targets semantics (the seed is not pre-visited)
    unsigned long long* counts;
    unsigned long long* V;
    unsigned long long* F0;
    unsigned long long* F1;
    uint32_t* touched;
    uint32_t* R0;  // discovery lists, ping-pong by hop parity
    uint32_t* R1;
    uint32_t* clog;  // copy of every discovery list of the batch (for clearing V)
    uint64_t clog_cap;
    uint4* items0;
    uint4* items1;
    uint32_t items_cap;  // uint4 slots of each items array (heavy records fill it from the end)
    unsigned long long* lane_cnt;  // [(k+1) * 64W]
    unsigned long long* active;    // [2 * W]
    QCtl* qctl;                    // [2] by hop parity; .pad = push-equivalent edges
    unsigned long long* misc;      // [0] unexplored in-edges
    unsigned int* bar;
    LevelCounters* lc;
    uint32_t alpha, beta, force_dir;
    uint32_t* umask;  // [2][nwords] by hop parity: per word, the vertices a pull left unsettled
    uint32_t diag;  // MGK_MS_DIAG=1: per hop, expand-phase ns in lc.union_edges, finalize ns in lc.candidates
    // Straggler lanes (one word per vertex): at the first pull, a lane whose
    // frontier has at most m / strag out-edges keeps pushing (0: off). lane_E
    // [64]: per-lane out-edges of the frontier just found.
    uint32_t strag;
    unsigned long long* lane_E;
    const uint4* top4;  // Graph::top4 (one word per vertex; nullptr: in-lists read from their first entry)
};

template <int W>
struct LaneWord {
    unsigned long long w[W];
};

template <int W>
__device__ __forceinline__ LaneWord<W> load_lw(const unsigned long long* p) {
    LaneWord<W> r;
    if constexpr (W == 1) {
        r.w[0] = p[0];
    } else {
#pragma unroll
        for (int i = 0; i < W; i += 2) {
            const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(p + i);
            r.w[i] = t.x;
            r.w[i + 1] = t.y;
        }
    }
    return r;
}

template <int W>
__device__ __forceinline__ LaneWord<W> load_lw_cg(const unsigned long long* p) {
    LaneWord<W> r;
    if constexpr (W == 1) {
        r.w[0] = __ldcg(p);
    } else {
#pragma unroll
        for (int i = 0; i < W; i += 2) {
            const ulonglong2 t = __ldcg(reinterpret_cast<const ulonglong2*>(p + i));
            r.w[i] = t.x;
            r.w[i + 1] = t.y;
        }
    }
    return r;
}

template <int W>
__device__ __forceinline__ void store_lw(unsigned long long* p, const LaneWord<W>& v) {
    if constexpr (W == 1) {
        p[0] = v.w[0];
    } else {
#pragma unroll
        for (int i = 0; i < W; i += 2)
            *reinterpret_cast<ulonglong2*>(p + i) = make_ulonglong2(v.w[i], v.w[i + 1]);
    }
}

// Lane-word storage. NB = 64: W uint64 words per vertex (64 W lanes).
// NB = 16 / 8 (W = 1): a uint16 / uint8 per vertex for batches of at most 16 /
// 8 seeds, so the state arrays of a 35.6M-vertex graph (G4) are 71 / 36 MB
// instead of 285 MB and the per-edge gathers of a dense pull hit L2.
// Narrow words are OR-ed with a 32-bit atomic on the containing word (the
// other sub-words' mask bits are zero); plain sub-word stores elsewhere touch
// only their own bytes.
template <int W, int NB>
struct LS;

template <int W>
struct LS<W, 64> {
    static constexpr uint32_t kLanes = 64 * W;
    __device__ static __forceinline__ LaneWord<W> load(const unsigned long long* b, size_t v) {
        return load_lw<W>(b + v * W);
    }
    __device__ static __forceinline__ LaneWord<W> load_cg(const unsigned long long* b, size_t v) {
        return load_lw_cg<W>(b + v * W);
    }
    __device__ static __forceinline__ void store(unsigned long long* b, size_t v, const LaneWord<W>& x) {
        store_lw<W>(b + v * W, x);
    }
    __device__ static __forceinline__ void atomic_or(unsigned long long* b, size_t v, int i, unsigned long long m) {
        atomicOr(b + v * W + i, m);
    }
    // (W = 1) OR m into v's word; true for the caller whose OR found the word
    // empty, i.e. the first to reach v in this hop (the word is zero between hops)
    __device__ static __forceinline__ bool atomic_or_first(unsigned long long* b, size_t v, unsigned long long m) {
        static_assert(W == 1, "one word per vertex");
        return atomicOr(b + v, m) == 0;
    }
    // a pull's per-edge frontier-word gather, L2 priority `pol` (evict-last);
    // also used with an evict-first policy for the pull's visited-word reads
    __device__ static __forceinline__ LaneWord<W> gather(const unsigned long long* b, size_t v,
                                                         unsigned long long pol) {
        if constexpr (W == 1) {
            LaneWord<W> r;
            r.w[0] = ld_hint_u64(b + v, pol);
            return r;
        } else {
            return load_lw<W>(b + v * W);
        }
    }
    // the pull's next-frontier store: evict-first, so it does not displace the
    // frontier words the gathers need
    __device__ static __forceinline__ void store_stream(unsigned long long* b, size_t v, const LaneWord<W>& x) {
        if constexpr (W == 1)
            st_stream_u64(b + v, x.w[0]);
        else
            store_lw<W>(b + v * W, x);
    }
    __host__ __device__ static constexpr size_t words64(size_t n) { return n * W; }
};

template <int NB>
struct LSNarrow {
    static_assert(NB == 8 || NB == 16, "narrow lane words are 8 or 16 bits");
    using T = typename std::conditional<NB == 16, unsigned short, unsigned char>::type;
    static constexpr uint32_t kLanes = NB;
    __device__ static __forceinline__ LaneWord<1> load(const unsigned long long* b, size_t v) {
        LaneWord<1> r;
        r.w[0] = reinterpret_cast<const T*>(b)[v];
        return r;
    }
    __device__ static __forceinline__ LaneWord<1> load_cg(const unsigned long long* b, size_t v) {
        LaneWord<1> r;
        if constexpr (NB == 16)
            r.w[0] = __ldcg(reinterpret_cast<const unsigned short*>(b) + v);
        else
            r.w[0] = __ldcg(reinterpret_cast<const unsigned char*>(b) + v);
        return r;
    }
    __device__ static __forceinline__ LaneWord<1> gather(const unsigned long long* b, size_t v,
                                                         unsigned long long pol) {
        LaneWord<1> r;
        if constexpr (NB == 16)
            r.w[0] = ld_hint_u16(reinterpret_cast<const unsigned short*>(b) + v, pol);
        else
            r.w[0] = ld_hint_u8(reinterpret_cast<const unsigned char*>(b) + v, pol);
        return r;
    }
    __device__ static __forceinline__ void store(unsigned long long* b, size_t v, const LaneWord<1>& x) {
        reinterpret_cast<T*>(b)[v] = (T)x.w[0];
    }
    __device__ static __forceinline__ void store_stream(unsigned long long* b, size_t v, const LaneWord<1>& x) {
        if constexpr (NB == 16)
            st_stream_u16(reinterpret_cast<unsigned short*>(b) + v, (uint32_t)x.w[0]);
        else
            st_stream_u8(reinterpret_cast<unsigned char*>(b) + v, (uint32_t)x.w[0]);
    }
    __device__ static __forceinline__ void atomic_or(unsigned long long* b, size_t v, int, unsigned long long m) {
        constexpr uint32_t per = 32 / NB;
        atomicOr(reinterpret_cast<unsigned int*>(b) + v / per, (unsigned int)m << (NB * (v % per)));
    }
    __device__ static __forceinline__ bool atomic_or_first(unsigned long long* b, size_t v, unsigned long long m) {
        constexpr uint32_t per = 32 / NB;
        const uint32_t sh = NB * (v % per);
        const unsigned int old = atomicOr(reinterpret_cast<unsigned int*>(b) + v / per, (unsigned int)m << sh);
        return ((old >> sh) & ((1u << NB) - 1u)) == 0;
    }
    __host__ __device__ static constexpr size_t words64(size_t n) { return (n * NB + 63) / 64; }
};
template <>
struct LS<1, 16> : LSNarrow<16> {};
template <>
struct LS<1, 8> : LSNarrow<8> {};

// NB = 10: three 10-bit lane words per 32-bit word (batches of 9 or 10 seeds:
// the reference schedule's deep sections). G4's state arrays are then 47 MB
// instead of 71 MB -- under the ~64 MB where random loads fall off L2
// (profiles/ubench_atomics.json: 214 G/s at 64 MB, 163 G/s at 90 MB).
// Neighbouring vertices share a 32-bit word, so every write is an atomic on
// it (OR to set, AND to clear); reads extract the field.
template <>
struct LS<1, 10> {
    static constexpr uint32_t kLanes = 10;
    static constexpr uint32_t kMask = 0x3FFu;
    __device__ static __forceinline__ uint32_t word(size_t v) { return __umulhi((uint32_t)v, 0xAAAAAAABu) >> 1; }
    __device__ static __forceinline__ uint32_t shift(size_t v) { return 10u * ((uint32_t)v - 3u * word(v)); }
    __device__ static __forceinline__ unsigned int* at(unsigned long long* b, size_t v) {
        return reinterpret_cast<unsigned int*>(b) + word(v);
    }
    __device__ static __forceinline__ const unsigned int* at(const unsigned long long* b, size_t v) {
        return reinterpret_cast<const unsigned int*>(b) + word(v);
    }
    __device__ static __forceinline__ LaneWord<1> load(const unsigned long long* b, size_t v) {
        LaneWord<1> r;
        r.w[0] = (*at(b, v) >> shift(v)) & kMask;
        return r;
    }
    __device__ static __forceinline__ LaneWord<1> load_cg(const unsigned long long* b, size_t v) {
        LaneWord<1> r;
        r.w[0] = (__ldcg(at(b, v)) >> shift(v)) & kMask;
        return r;
    }
    __device__ static __forceinline__ LaneWord<1> gather(const unsigned long long* b, size_t v,
                                                         unsigned long long pol) {
        uint32_t w;
        asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(w) : "l"(at(b, v)), "l"(pol));
        LaneWord<1> r;
        r.w[0] = (w >> shift(v)) & kMask;
        return r;
    }
    // x holds every lane of v's word: the bits not yet set are OR-ed in, and a
    // zero word clears the field (the callers' only two cases)
    __device__ static __forceinline__ void store(unsigned long long* b, size_t v, const LaneWord<1>& x) {
        if (x.w[0])
            atomicOr(at(b, v), (unsigned int)x.w[0] << shift(v));
        else
            atomicAnd(at(b, v), ~(kMask << shift(v)));
    }
    // the pull's next-frontier write (the field is zero): an OR at L2 evict-first
    // priority, so it does not displace the frontier words the gathers need
    __device__ static __forceinline__ void store_stream(unsigned long long* b, size_t v, const LaneWord<1>& x) {
        asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(at(b, v)),
                     "r"((unsigned int)x.w[0] << shift(v)), "l"(l2_stream_policy())
                     : "memory");
    }
    __device__ static __forceinline__ void atomic_or(unsigned long long* b, size_t v, int, unsigned long long m) {
        atomicOr(at(b, v), (unsigned int)m << shift(v));
    }
    __device__ static __forceinline__ bool atomic_or_first(unsigned long long* b, size_t v, unsigned long long m) {
        const uint32_t sh = shift(v);
        const unsigned int old = atomicOr(at(b, v), (unsigned int)m << sh);
        return ((old >> sh) & kMask) == 0;
    }
    __host__ __device__ static constexpr size_t words64(size_t n) { return ((n + 2) / 3 + 1) / 2; }
};

// bytes of one narrow lane-word array for n vertices
template <int W, int NB>
constexpr size_t narrow_bytes(size_t n) {
    return NB == 64 ? 0 : LS<W, NB>::words64(n) * 8;
}


__device__ __forceinline__ uint4* items_of(const MSParams& P, uint32_t i) {
    return (i & 1) ? P.items1 : P.items0;
}
__device__ __forceinline__ uint32_t* R_of(const MSParams& P, uint32_t i) {
    return (i & 1) ? P.R1 : P.R0;
}

// Push work items of the LANES engine. A vertex with at most kHeavyItems
// items (out-degree <= 2048) gets its kChunk-entry items written by the warp
// that lists it; a heavier one (a hub: G4's reach 10^6 out-edges) gets ONE
// record {u, row begin, degree, first virtual item} at the end of the items
// array instead, and the push derives its items from the records by a binary
// search -- one warp writing a hub's ~10^5 items was the critical path of the
// finalize before a push (G4 10 seeds, hop 1: 89 us for 448 vertices).
// misc[kHeavyCtl + parity] = (records << 40) | virtual items; one 64-bit
// atomic per warp reserves both, so record slots ascend with their first item.
constexpr uint32_t kHeavyItems = 64;
constexpr int kHeavyCtl = 4;
constexpr int kHeavyShift = 40;

__device__ __forceinline__ void emit_items_lanes(const MSParams& P, const uint32_t* buf, uint32_t n, uint4* items,
                                                 unsigned int* nitems) {
    if (n == 0) return;
    const uint32_t lane = lane_id();
    const uint32_t* rp = P.g.rp;
    unsigned long long* hctl = P.misc + kHeavyCtl + (items == P.items0 ? 0 : 1);
    uint4* hrec = items + P.items_cap - 1;  // record r at hrec[-r]
    uint32_t tot = 0;
    for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t u = buf[i];
        const uint32_t d = __ldg(rp + u + 1) - __ldg(rp + u);
        const uint32_t nit = (d + kChunk - 1) / kChunk;
        tot += nit > kHeavyItems ? 0 : nit;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) tot += __shfl_xor_sync(kFull, tot, d);
    uint32_t base = 0;
    if (lane == 0 && tot) base = atomicAdd(nitems, tot);
    base = __shfl_sync(kFull, base, 0);
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        uint32_t u = 0, b = 0, deg = 0;
        if (i < n) {
            u = buf[i];
            b = __ldg(rp + u);
            deg = __ldg(rp + u + 1) - b;
        }
        const uint32_t all = (deg + kChunk - 1) / kChunk;
        const bool heavy = all > kHeavyItems;
        const uint32_t nit = heavy ? 0 : all;
        const unsigned hm = __ballot_sync(kFull, heavy);
        if (hm) {  // records of this group's hubs: one reservation for all of them
            const uint32_t hn = heavy ? all : 0;
            const uint32_t hincl = warp_incl_scan(hn);
            unsigned long long hb = 0;
            if (lane == 31)
                hb = atomicAdd(hctl, ((unsigned long long)__popc(hm) << kHeavyShift) | (unsigned long long)hincl);
            hb = __shfl_sync(kFull, hb, 31);
            if (heavy) {
                const uint32_t slot = (uint32_t)(hb >> kHeavyShift) + __popc(hm & lanemask_lt());
                const uint32_t first = (uint32_t)(hb & ((1ull << kHeavyShift) - 1)) + hincl - hn;
                *(hrec - slot) = make_uint4(u, b, deg, first);
            }
        }
        const uint32_t incl = warp_incl_scan(nit);
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        const uint32_t excl = incl - nit;
        for (uint32_t x0 = 0; x0 < total; x0 += 32) {
            const uint32_t x = x0 + lane;
            const uint32_t j = warp_owner(incl, x < total ? x : total - 1);
            const uint32_t bj = __shfl_sync(kFull, b, j);
            const uint32_t dj = __shfl_sync(kFull, deg, j);
            const uint32_t ej = __shfl_sync(kFull, excl, j);
            const uint32_t uj = __shfl_sync(kFull, u, j);
            if (x < total) {
                const uint32_t s = bj + (x - ej) * kChunk;
                items[base + x] = make_uint4(s, min(s + kChunk, bj + dj), uj, 0);
            }
        }
        base += total;
    }
    __syncwarp();
}

// item x of a push: written (x < nlight) or derived from the heavy records
__device__ __forceinline__ uint4 push_item(const uint4* items, uint32_t cap, uint32_t nlight, uint32_t nrec,
                                           uint32_t x) {
    if (x < nlight) return items[x];
    const uint32_t c = x - nlight;
    const uint32_t* hw = reinterpret_cast<const uint32_t*>(items + cap - 1);  // record r's first item: hw[3 - 4 r]
    uint32_t lo = 0, hi = nrec;  // last record whose first item <= c
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldcg(hw + 3 - 4 * (int64_t)mid) <= c) lo = mid; else hi = mid;
    }
    const uint4 r = __ldcg(items + cap - 1 - lo);
    const uint32_t s = r.y + (c - r.w) * kChunk;
    return make_uint4(s, min(s + kChunk, r.y + r.z), r.x, 0);
}
__device__ __forceinline__ unsigned long long* F_of(const MSParams& P, uint32_t i) {
    return (i & 1) ? P.F1 : P.F0;
}

// per-thread counters of a phase (flushed per block after the phase; 32-bit:
// a thread's share of a phase stays far below 2^32, except pe = sum deg x lanes)
struct Acc {
    uint32_t found, edges, indeg, scanned, candidates, pairs;
    unsigned long long pe;
    __device__ void zero() { found = edges = indeg = scanned = candidates = pairs = 0; pe = 0; }
};

// Block reduce + flush. found/edges/indeg describe discovered vertices (-> q);
// pairs/pe describe finalized lane-vertex pairs (-> lc / qf).
__device__ void block_flush(Acc& a, QCtl* q, QCtl* qf, LevelCounters* lc, LevelCounters* lc_next,
                            unsigned long long* unexplored) {
    __shared__ unsigned long long s[7];
    if (threadIdx.x < 7) s[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long v[7] = {a.found, a.edges, a.indeg, a.scanned, a.candidates, a.pairs, a.pe};
#pragma unroll
    for (int i = 0; i < 7; ++i) {
        v[i] = warp_sum_u64(v[i]);
        if (lane_id() == 0 && v[i]) atomicAdd(&s[i], v[i]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s[0]) atomicAdd(&lc->vertices, s[0]);
        if (s[1]) atomicAdd(&q->edges, s[1]);
        if (s[2]) {
            atomicAdd(&q->indeg, s[2]);
            atomicAdd(unexplored, 0ULL - s[2]);
        }
        if (s[3]) atomicAdd(&lc->scanned, s[3]);
        if (s[4]) atomicAdd(&lc->candidates, s[4]);
        if (s[5]) atomicAdd(&lc->frontier, s[5]);
        if (s[6]) {
            atomicAdd(&qf->pad, s[6]);
            if (lc_next) atomicAdd(&lc_next->edges, s[6]);
        }
    }
    __syncthreads();
    a.zero();
}


// ---- push expand -----------------------------------------------------------------
// Entries per lane per round (their loads issued together): a push entry is a
// chain of dependent accesses (in-list entry -> visited word -> atomic), so a
// round costs a full memory latency; one-word lanes take PU of them at once.
#ifndef MGK_PUSH_UNROLL
#define MGK_PUSH_UNROLL 4
#endif
// finalize lists of more than n / kDenseDiv vertices are swept densely (one word per vertex)
#ifndef MGK_DENSE_DIV
#define MGK_DENSE_DIV 8  // 16 and 32 measured slower: the dense sweep is latency-bound (G4 hop 2: 136 -> 185 us at 32)
#endif
constexpr uint64_t kDenseDiv = MGK_DENSE_DIV;
template <int W>
constexpr int push_unroll() { return W == 1 ? MGK_PUSH_UNROLL : 1; }

// kList = false (the stragglers' push of a mixed hop): the ORs are fire-and-
// forget (a `red`: ~1.5x the rate of an atomic that returns) and nothing is
// listed -- that hop's finalize sweeps every vertex.
template <int W, int NB, bool kList = true>
MGK_PHASE void push_phase(const MSParams& P, const uint4* items, uint32_t nlight, unsigned long long hctl,
                           const unsigned long long* Fc, unsigned long long* Fn, uint32_t* Rn,
                           QCtl* qn, Acc& acc, Stage<kStageCap>& st, uint32_t warp_gid,
                           uint32_t nwarps, const LaneWord<W>& pushm) {
    constexpr int PU = push_unroll<W>();
    const uint32_t lane = lane_id();
    const DevGraph& g = P.g;
    const uint32_t nrec = (uint32_t)(hctl >> kHeavyShift);
    const uint32_t nitems = nlight + (uint32_t)(hctl & ((1ull << kHeavyShift) - 1));
    const uint32_t G = items_per_warp(nitems, nwarps);
    for (uint32_t base = warp_gid * G; base < nitems; base += nwarps * G) {
        const uint32_t idx = base + lane;
        const uint4 it = (lane < G && idx < nitems) ? push_item(items, P.items_cap, nlight, nrec, idx)
                                                     : make_uint4(0, 0, 0, 0);
        const uint32_t len = it.y - it.x;
        const uint32_t incl = warp_incl_scan(len);
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        const uint32_t off = it.x - (incl - len);
        for (uint32_t x0 = 0; x0 < total; x0 += 32 * PU) {
            uint32_t u[PU], src[PU];
            bool valid[PU], first[PU];
#pragma unroll
            for (int q = 0; q < PU; ++q) {
                const uint32_t x = x0 + 32 * q + lane;
                valid[q] = x < total;
                const uint32_t j = warp_owner(incl, valid[q] ? x : total - 1);
                const uint32_t pos = __shfl_sync(kFull, off, j) + x;
                src[q] = __shfl_sync(kFull, it.z, j);
                u[q] = valid[q] ? __ldg(g.ci + pos) : 0;
                first[q] = false;
            }
            if constexpr (W == 1) {
                // the round's visited words first, then its atomics (the OR that finds
                // the word empty lists u): every load of the round is in flight before
                // the first atomic, and no atomic waits for another's result
                unsigned long long m[PU];
#pragma unroll
                for (int q = 0; q < PU; ++q) {
                    m[q] = 0;
                    // (also masking the lanes u's new word already holds, to spare hub
                    // targets' atomics, measured slower: G4 mixed hop's push 780 -> 900 us)
                    // (kList = false: no visited-word gather either -- the finalize
                    // masks every new word with the visited one, and a lane bit at a
                    // vertex the lane already visited is inert for one hop: every
                    // out-neighbour of such a vertex was reached by that lane before)
                    if (valid[q]) {
                        m[q] = LS<W, NB>::load(Fc, src[q]).w[0] & pushm.w[0];
                        if constexpr (kList) m[q] &= ~LS<W, NB>::load(P.V, u[q]).w[0];
                    }
                }
#pragma unroll
                for (int q = 0; q < PU; ++q) {
                    if (m[q]) {
                        if constexpr (kList)
                            first[q] = LS<W, NB>::atomic_or_first(Fn, u[q], m[q]);
                        else
                            LS<W, NB>::atomic_or(Fn, u[q], 0, m[q]);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < PU; ++q) {
                    if (!valid[q]) continue;
                    const LaneWord<W> f = LS<W, NB>::load(Fc, src[q]);
                    const LaneWord<W> vis = LS<W, NB>::load(P.V, u[q]);
                    LaneWord<W> m;
                    bool any = false;
#pragma unroll
                    for (int i = 0; i < W; ++i) {
                        m.w[i] = f.w[i] & ~vis.w[i] & pushm.w[i];  // only the lanes pushing this hop
                        any |= m.w[i] != 0;
                    }
                    if (any) {
                        if constexpr (W == 1) {
                            // one atomic: the OR that finds the word empty lists u
                            first[q] = LS<W, NB>::atomic_or_first(Fn, u[q], m.w[0]);
                        } else {
                            const LaneWord<W> cur = LS<W, NB>::load_cg(Fn, u[q]);
                            bool need = false;
#pragma unroll
                            for (int i = 0; i < W; ++i) {
                                if ((cur.w[i] & m.w[i]) != m.w[i]) {
                                    LS<W, NB>::atomic_or(Fn, u[q], i, m.w[i]);
                                    need = true;
                                }
                            }
                            if (need) {  // several words: the touched bit decides who lists u
                                const uint32_t bit = 1u << (u[q] & 31);
                                first[q] = !(atomicOr(P.touched + (u[q] >> 5), bit) & bit);
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < PU; ++q) {
                acc.scanned += valid[q];
                if constexpr (kList) {
                    st.push(first[q], u[q]);
                    if (st.full()) {
                        emit_list(st.buf, st.n, Rn, &qn->nitems);
                        st.n = 0;
                    }
                }
            }
        }
    }
    if constexpr (kList) {
        emit_list(st.buf, st.n, Rn, &qn->nitems);
        st.n = 0;
    }
}

// ---- pull expand -------------------------------------------------------------
// Vertices are split by in-degree: <= 32 in-edges are scanned by one thread
// (two lane-word gathers in flight per step), 33..kHeavyIn by the word's warp
// cooperatively (each lane ORs its own stride, one warp reduction per 256
// entries for the early-exit test), and > kHeavyIn as kHeavyChunk-entry tasks
// spread over the whole grid (DevGraph::heavy), so no hub serialises a warp.
template <int W>
__device__ __forceinline__ LaneWord<W> warp_or_lw(LaneWord<W> a) {
#pragma unroll
    for (int i = 0; i < W; ++i) a.w[i] = warp_or_u64(a.w[i]);
    return a;
}

template <int W>
__device__ __forceinline__ bool covers(const LaneWord<W>& acc, const LaneWord<W>& need) {
    bool done = true;
#pragma unroll
    for (int i = 0; i < W; ++i) done &= (acc.w[i] & need.w[i]) == need.w[i];
    return done;
}

// Warp-wide: OR of the lane words of in-neighbours ri[b..e), stopping early
// once `need` is covered. Returns the OR (all lanes) and the entries read.
template <int W, int NB>
__device__ __forceinline__ LaneWord<W> warp_pull_range(const MSParams& P, const unsigned long long* Fc,
                                                       uint32_t b, uint32_t e,
                                                       const LaneWord<W>& need, uint32_t& scanned) {
    const uint32_t lane = lane_id();
    // (the L2 policies are re-created at each load: one instruction, no live 64-bit registers)
    LaneWord<W> acc;
#pragma unroll
    for (int i = 0; i < W; ++i) acc.w[i] = 0;
    scanned = 0;
    // coverage is tested after 32, 64, 128, then every 256 entries: hubs come
    // first in every in-list, so most vertices that exit early do so in the
    // first blocks
    for (uint32_t p0 = b, blk = 32; p0 < e; p0 += blk, blk = min(2 * blk, 256u)) {
        const uint32_t pe = min(e, p0 + blk);
#pragma unroll kWprUnroll
        for (uint32_t p = p0 + lane; p < pe; p += 32) {
            const LaneWord<W> f = LS<W, NB>::gather(Fc, ldg_hint(P.g.ri + p, l2_stream_policy()), l2_keep_policy());
#pragma unroll
            for (int i = 0; i < W; ++i) acc.w[i] |= f.w[i];
        }
        scanned += pe - p0;
        acc = warp_or_lw<W>(acc);
        if (covers<W>(acc, need)) break;
    }
    return acc;
}

// Warp-level dynamic work split: chunk c = warp_gid first, then chunks
// nwarps, nwarps + 1, ... handed out by one atomic counter, so warps that
// finish early take over the tail instead of idling at the next barrier.
struct ChunkGrab {
    unsigned long long* ctr;
    uint32_t nchunks, chunk;
    uint32_t c;
    __device__ ChunkGrab(unsigned long long* counter, uint32_t total, uint32_t chunk_len, uint32_t warp_gid)
        : ctr(counter), nchunks((total + chunk_len - 1) / chunk_len), chunk(chunk_len), c(warp_gid) {}
    __device__ bool valid() const { return c < nchunks; }
    __device__ void advance(uint32_t nwarps) {
        uint32_t n = 0;
        if (lane_id() == 0) n = (uint32_t)atomicAdd(ctr, 1ull);
        c = __shfl_sync(kFull, n, 0) + nwarps;
    }
};

template <int W, int NB>
MGK_PHASE void pull_phase(const MSParams& P, const unsigned long long* Fc, unsigned long long* Fn,
                           const LaneWord<W>& active, uint32_t* Rn, QCtl* qn, Acc& acc,
                           Stage<kStageCap>& st, uint32_t warp_gid, uint32_t nwarps,
                           const uint32_t* um_in, uint32_t* um_out, uint32_t* s_nm, uint32_t* s_cb) {
    const uint32_t lane = lane_id();
    const DevGraph& g = P.g;
    // candidate words in chunks, spread dynamically (misc[1]); about 8
    // chunks per warp, at least 8 words each, so the counter stays cold
    // (the L2 policies are re-created at each load: one instruction, no live 64-bit registers)
    const uint32_t wchunk = max(8u, g.nwords / (nwarps * 8));
    ChunkGrab words(&P.misc[1], g.nwords, wchunk, warp_gid);
    // one candidate per lane (valid): visited word, CSC bounds, the lane's scan
    // of a short list (or the first kPre entries), the warp's scans of the
    // unsettled longer lists, the next-frontier store; true when lanes are left
    // (the candidate's visited word and CSC bounds are loaded by the caller)
    auto visit = [&](bool valid, uint32_t u, const LaneWord<W>& vis, uint32_t b, uint32_t e, const uint4& t4,
                     bool& found) -> bool {
        LaneWord<W> need;
#pragma unroll
        for (int i = 0; i < W; ++i) need.w[i] = 0;
        bool cand = false;
        if (valid) {
#pragma unroll
            for (int i = 0; i < W; ++i) {
                need.w[i] = active.w[i] & ~vis.w[i];
                cand |= need.w[i] != 0;
            }
        }
        LaneWord<W> acc_w;
#pragma unroll
        for (int i = 0; i < W; ++i) acc_w.w[i] = 0;
        uint32_t scanned = 0;
        // in-degree <= 32: the lane scans the whole list; larger lists: the lane
        // scans the first kPre entries (hubs come first, so most reached vertices
        // are settled there) and the warp takes the rest of an unsettled list
        constexpr uint32_t kPre = MGK_PRE;
        constexpr uint32_t kStep = MGK_LIGHT_STEP;
        bool settled = false;
        if (cand) {
            const uint32_t stop = e - b <= 32 ? e : b + kPre;
            uint32_t p = b;
            bool done = false;
            if constexpr (W == 1 && MGK_TOP4) {
                // the list's first four entries came with the visited word and the
                // bounds (padding repeats the first entry: every gather is valid)
                if (P.top4) {
                    const uint32_t tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc_w.w[0] |= LS<W, NB>::gather(Fc, tv[q], l2_keep_policy()).w[0];
                    const uint32_t d4 = min(e - b, 4u);
                    scanned += d4;
                    p = b + d4;
                    done = covers<W>(acc_w, need);
                }
            }
            for (; p + kStep <= stop && !done; p += kStep) {
                uint32_t v[kStep];
#pragma unroll
                for (uint32_t q = 0; q < kStep; ++q) v[q] = ld_ri_lane(g.ri + p + q, l2_stream_policy());
#pragma unroll
                for (uint32_t q = 0; q < kStep; ++q) {
                    const LaneWord<W> f = LS<W, NB>::gather(Fc, v[q], l2_keep_policy());
#pragma unroll
                    for (int i = 0; i < W; ++i) acc_w.w[i] |= f.w[i];
                }
                done = covers<W>(acc_w, need);
                scanned += kStep;
            }
            for (; !done && p < stop; ++p) {
                const LaneWord<W> f = LS<W, NB>::gather(Fc, ld_ri_lane(g.ri + p, l2_stream_policy()), l2_keep_policy());
#pragma unroll
                for (int i = 0; i < W; ++i) acc_w.w[i] |= f.w[i];
                ++scanned;
                done = covers<W>(acc_w, need);
            }
            settled = done || p >= e;
            b = p;  // where the warp continues an unsettled list
        }
        unsigned mid = __ballot_sync(kFull, cand && !settled);
        while (mid) {
            const int j = __ffs(mid) - 1;
            mid &= mid - 1;
            LaneWord<W> nj;  // the lanes lane j's pre-scan has not found yet
#pragma unroll
            for (int i = 0; i < W; ++i) nj.w[i] = __shfl_sync(kFull, need.w[i] & ~acc_w.w[i], j);
            uint32_t sc = 0;
            const LaneWord<W> aj = warp_pull_range<W, NB>(P, Fc, __shfl_sync(kFull, b, j),
                                                      __shfl_sync(kFull, e, j), nj, sc);
            if ((int)lane == j) {
#pragma unroll
                for (int i = 0; i < W; ++i) acc_w.w[i] |= aj.w[i];
                scanned += sc;
            }
        }
        found = false;
        if (cand) {
            LaneWord<W> res;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                res.w[i] = acc_w.w[i] & need.w[i];
                found |= res.w[i] != 0;
            }
            if (found) LS<W, NB>::store_stream(Fn, u, res);
        }
        acc.candidates += cand;
        acc.scanned += scanned;
        bool left = false;
#pragma unroll
        for (int i = 0; i < W; ++i) left |= (need.w[i] & ~acc_w.w[i]) != 0;
        st.push(found, u);
        if (st.full()) {
            emit_list(st.buf, st.n, Rn, &qn->nitems);
            st.n = 0;
        }
        return cand && left;
    };
    // Candidates are packed into lanes: the warp walks 32 words at a time,
    // appends each word's candidates (not pull_skip; after a pull only the
    // vertices that pull left unsettled, um_in) to a per-warp buffer in shared
    // memory and visits them 32 at a time, so no lane idles on a skipped,
    // settled or zero-in-degree vertex (the late pulls have a few candidates
    // per word). um_out receives this pull's unsettled vertices: the next
    // pull's candidates are among them (the active lanes only shrink and the
    // visited sets only grow).
    for (; words.valid(); words.advance(nwarps))
    for (uint32_t wb = words.c * wchunk, wend = min(g.nwords, (words.c + 1) * wchunk); wb < wend; wb += 32) {
    const uint32_t wq = wb + lane;
    const uint32_t mq = wq < wend ? ~__ldg(g.pull_skip + wq) & (um_in ? __ldcg(um_in + wq) : kFull) : 0u;
    s_nm[lane] = 0;
    uint32_t fill = 0;  // warp-uniform: candidates waiting in s_cb
    __syncwarp();
    const uint32_t nw = min(wend - wb, 32u);
    for (uint32_t q = 0; q <= nw; ++q) {
        if (q < nw) {
            const uint32_t m = __shfl_sync(kFull, mq, q);
            if (m == 0) continue;
            if ((m >> lane) & 1u) s_cb[fill + __popc(m & lanemask_lt())] = (wb + q) * 32 + lane;
            fill += __popc(m);
            __syncwarp();
            if (fill < 32) continue;
        } else if (fill == 0) {
            break;
        }
        // one round: the first 32 waiting candidates (the group's last round may be partial)
        const bool valid = lane < fill;
        const uint32_t u = valid ? s_cb[lane] : 0u;
        __syncwarp();
        if (fill > 32 && lane < fill - 32) s_cb[lane] = s_cb[32 + lane];
        fill = fill > 32 ? fill - 32 : 0;
        __syncwarp();
        LaneWord<W> vis;
#pragma unroll
        for (int i = 0; i < W; ++i) vis.w[i] = 0;
        uint32_t b = 0, e = 0;
        uint4 t4 = make_uint4(0, 0, 0, 0);
        if (valid) {
            vis = LS<W, NB>::gather(P.V, u, l2_stream_policy());  // read once per pull: evict-first
            b = ldg_hint(g.cp + u, l2_stream_policy());
            e = ldg_hint(g.cp + u + 1, l2_stream_policy());
            if constexpr (W == 1 && MGK_TOP4) {
                if (P.top4) t4 = ldg_hint_v4(P.top4 + u, l2_stream_policy());
            }
        }
        bool found;
        if (visit(valid, u, vis, b, e, t4, found)) atomicOr(&s_nm[(u >> 5) - wb], 1u << (u & 31));
    }
    __syncwarp();
    if (um_out && wq < wend) um_out[wq] = s_nm[lane];
    }
    // heavy in-degree vertices: kHeavyChunk-entry tasks (chunk-major). A warp
    // checks 32 tasks at once (one task per lane: record, visited word and,
    // for a later chunk, what the earlier chunks found) and scans only the
    // tasks with lanes left, one after the other; in the late hops almost every
    // task is settled and costs one parallel round of loads, not a chain per task
    // (many tasks per warp: chunks of 32-task groups; few: single tasks, so the
    // scans still spread over every warp)
    // Batched only after a pull (um_in): then most tasks are settled; in the
    // first, dense pull a task is checked right before its scan, which sees
    // more of what its vertex's earlier chunks found
    const uint32_t tchunk = (um_in && g.nheavy >= nwarps * 64) ? (g.nheavy / (nwarps * 4) + 31) / 32 * 32
                                                               : max(1u, g.nheavy / (nwarps * 8));
    const uint32_t tstep = (um_in && g.nheavy >= nwarps * 64) ? 32u : 1u;
    ChunkGrab tasks(&P.misc[2], g.nheavy, tchunk, warp_gid);
    for (; tasks.valid(); tasks.advance(nwarps))
    for (uint32_t t0 = tasks.c * tchunk, tend = min(g.nheavy, (tasks.c + 1) * tchunk); t0 < tend; t0 += tstep) {
        const uint32_t t = lane < tstep ? t0 + lane : tend;
        uint32_t u = 0, ty = 0, tb = 0;
        LaneWord<W> vis, need;
#pragma unroll
        for (int i = 0; i < W; ++i) vis.w[i] = need.w[i] = 0;
        bool cand = false;
        if (t < tend) {
            const uint2 task = __ldg(g.heavy + t);
            u = task.x;
            ty = task.y;
            tb = __ldg(g.cp + u);
            vis = LS<W, NB>::load(P.V, u);
#pragma unroll
            for (int i = 0; i < W; ++i) {
                need.w[i] = active.w[i] & ~vis.w[i];
                cand |= need.w[i] != 0;
            }
            if (cand && ty != tb) {
                // a later chunk: only the lanes the earlier chunks of u have not
                // found yet; none left -> nothing to scan
                const LaneWord<W> got = LS<W, NB>::load_cg(Fn, u);
                cand = false;
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    need.w[i] &= ~got.w[i];
                    cand |= need.w[i] != 0;
                }
            }
        }
        bool first = false;
        unsigned todo = __ballot_sync(kFull, cand);
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t uj = __shfl_sync(kFull, u, j), yj = __shfl_sync(kFull, ty, j);
            LaneWord<W> nj;
#pragma unroll
            for (int i = 0; i < W; ++i) nj.w[i] = __shfl_sync(kFull, need.w[i], j);
            if (yj != __shfl_sync(kFull, tb, j)) {  // a later chunk: drop the lanes found meanwhile
                const LaneWord<W> got = LS<W, NB>::load_cg(Fn, uj);
                bool left = false;
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    nj.w[i] &= ~got.w[i];
                    left |= nj.w[i] != 0;
                }
                if (!left) continue;
                if ((int)lane == j) {
#pragma unroll
                    for (int i = 0; i < W; ++i) need.w[i] = nj.w[i];
                }
            }
            const uint32_t e = min(yj + kHeavyChunk, __ldg(g.cp + uj + 1));
            uint32_t sc = 0;
            const LaneWord<W> aj = warp_pull_range<W, NB>(P, Fc, yj, e, nj, sc);
            if ((int)lane == j) {
                acc.scanned += sc;
                acc.candidates += ty == tb;
                // several chunks of one vertex OR into its word: the first to
                // find it empty lists it
                if constexpr (W == 1) {
                    const unsigned long long r = aj.w[0] & need.w[0];
                    if (r) first = LS<W, NB>::atomic_or_first(Fn, u, r);
                } else {
                    bool any = false;
#pragma unroll
                    for (int i = 0; i < W; ++i) {
                        const unsigned long long r = aj.w[i] & need.w[i];
                        if (r) {
                            LS<W, NB>::atomic_or(Fn, u, i, r);
                            any = true;
                        }
                    }
                    if (any) {
                        const uint32_t bit = 1u << (u & 31);
                        first = !(atomicOr(P.touched + (u >> 5), bit) & bit);
                    }
                }
            }
        }
        st.push(first, u);
        if (st.full()) {
            emit_list(st.buf, st.n, Rn, &qn->nitems);
            st.n = 0;
        }
    }
    emit_list(st.buf, st.n, Rn, &qn->nitems);
    st.n = 0;
}

// ---- finalize: V |= F', lane counts, next-hop items, clear old frontier -------
template <int W, int NB>
MGK_PHASE void finalize_phase(const MSParams& P, const uint32_t* Rn, uint32_t nR,
                               unsigned long long* Fn, bool mark_visited, bool touched_set, bool want_items,
                               uint4* items_n, unsigned int* item_tail, bool count_lanes,
                               unsigned long long* s_cnt, unsigned long long* active_n,
                               uint64_t clog_base, Acc& acc, Stage<kStageCap>& st,
                               uint32_t warp_gid, uint32_t nwarps, bool dense = false) {
    const uint32_t lane = lane_id();
    const DevGraph& g = P.g;
    // dense (a list of more than n/8, one word per vertex): sweep every vertex
    // instead of the list, with all of a vertex's loads (frontier and visited
    // words, CSR / CSC bounds) issued at once and coalesced -- one round trip
    // per vertex instead of two dependent ones; the discovered vertices are
    // those with a non-zero new word. The list itself stays as built.
    // (Measured and removed: a "dense_few" sweep for lists of n/32 .. n/4 that
    // loads the bounds of the discovered vertices only -- G4 hop 2 unchanged,
    // and the split loads cost the fully dense sweeps of hops 3 / 4 +65 us each.)
    LaneWord<W> act;
    uint32_t cnt_lo[W], cnt_hi[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
        act.w[i] = 0;
        cnt_lo[i] = cnt_hi[i] = 0;
    }
    const uint32_t lim = dense ? g.n : nR;
    for (uint32_t base = warp_gid * 32; base < lim; base += nwarps * 32) {
        const uint32_t idx = base + lane;
        bool valid = idx < lim;
        uint32_t u = 0;
        LaneWord<W> x, v;
#pragma unroll
        for (int i = 0; i < W; ++i) x.w[i] = v.w[i] = 0;
        uint32_t r0 = 0, r1 = 0, c0 = 0, c1 = 0;
        bool expand = false;
        // all of a vertex's loads at once (the stores below would otherwise
        // keep the bounds' loads behind them)
        if (valid) {
            u = dense ? idx : Rn[idx];
            x = LS<W, NB>::load(Fn, u);
            v = LS<W, NB>::load(P.V, u);
            r0 = __ldg(g.rp + u);
            r1 = __ldg(g.rp + u + 1);
            c0 = __ldg(g.cp + u);
            c1 = __ldg(g.cp + u + 1);
            if (dense) {
                bool any = false;
#pragma unroll
                for (int i = 0; i < W; ++i) any |= x.w[i] != 0;
                valid = any;
            }
        }
        if (valid) {
            // lanes that had visited u are dropped here (only a mixed hop's push,
            // which does not read the visited words, sets any)
            bool any = false;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                x.w[i] &= ~v.w[i];
                any |= x.w[i] != 0;
            }
            valid = any;
        }
        if (valid) {
            bool fresh = true;  // no lane had visited u: its in-edges leave the unexplored set
#pragma unroll
            for (int i = 0; i < W; ++i) fresh &= v.w[i] == 0;
            uint32_t pc = 0;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                if (mark_visited) v.w[i] |= x.w[i];
                act.w[i] |= x.w[i];
                pc += __popcll(x.w[i]);
            }
            if (NB != 10 || mark_visited) LS<W, NB>::store(P.V, u, v);
            // push levels set a touched bit per discovery; pull levels only for
            // heavy vertices (discovered vertices in pull_skip are heavy: a
            // zero-in-degree vertex is never discovered)
            // touched bits: the seeds' (level 0) and, with several words per
            // vertex, the push's and the heavy pull tasks' (one word per
            // vertex: the word itself decides who lists u)
            if (touched_set || (W > 1 && ((__ldg(g.pull_skip + (u >> 5)) >> (u & 31)) & 1u)))
                atomicAnd(P.touched + (u >> 5), ~(1u << (u & 31)));
            // (a dense sweep writes no copy: the batch's V is then cleared by streaming)
            if (!dense && clog_base + idx < P.clog_cap) P.clog[clog_base + idx] = u;
            const uint32_t deg = r1 - r0;
            const uint32_t indeg = fresh ? c1 - c0 : 0;
            acc.found += 1;  // distinct vertices discovered, their out-edges, fresh in-edges
            acc.edges += deg;
            if (fresh) acc.indeg += indeg;
            acc.pairs += pc;
            acc.pe += (unsigned long long)deg * pc;
            expand = want_items && deg > 0;
        }
        if (count_lanes) {
            // column sums of the warp's 32 lane words by SWAR: five lane bits
            // are spread into 6-bit fields of a 32-bit word (the product places
            // five copies of the 5-bit group side by side, the mask keeps bit j
            // of copy j), one redux.add per group of five lanes (a field reaches
            // at most 32); lane l keeps lane bit l (cnt_lo) and 32 + l (cnt_hi)
            // -- 2 (10-bit words) to 13 (64-bit) reductions instead of a ballot
            // per lane bit
            constexpr int kBits = NB < 64 ? NB : 64;
            constexpr int kGroups = (kBits + 4) / 5;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                if (__ballot_sync(kFull, x.w[i] != 0) == 0) continue;
                const unsigned long long xw = x.w[i];
#pragma unroll
                for (int q = 0; q < kGroups; ++q) {
                    const uint32_t f = ((uint32_t)(xw >> (5 * q)) & 31u) * 0x108421u & 0x1041041u;
                    const uint32_t sum = __reduce_add_sync(kFull, f);
                    if (lane / 5 == (uint32_t)q && lane < (uint32_t)kBits)
                        cnt_lo[i] += (sum >> (6 * (lane % 5))) & 63u;
                    if constexpr (NB == 64) {
                        if ((32 + lane) / 5 == (uint32_t)q) cnt_hi[i] += (sum >> (6 * ((32 + lane) % 5))) & 63u;
                    }
                }
            }
        }
        if (want_items) {
            st.push(expand, u);
            if (st.full()) {
                emit_items_lanes(P, st.buf, st.n, items_n, item_tail);
                st.n = 0;
            }
        }
    }
    if (want_items) {
        emit_items_lanes(P, st.buf, st.n, items_n, item_tail);
        st.n = 0;
    }
#pragma unroll
    for (int i = 0; i < W; ++i) {
        const unsigned long long a = warp_or_u64(act.w[i]);
        if (lane == 0 && a) atomicOr(active_n + i, a);
    }
    if (count_lanes) {
#pragma unroll
        for (int i = 0; i < W; ++i) {
            if (cnt_lo[i]) atomicAdd(&s_cnt[i * 64 + lane], (unsigned long long)cnt_lo[i]);
            if (NB == 64 && cnt_hi[i]) atomicAdd(&s_cnt[i * 64 + 32 + lane], (unsigned long long)cnt_hi[i]);
        }
    }
}

// next-hop push items for the frontier vertices with a pushing lane (after the
// per-lane direction decision)
template <int W, int NB>
MGK_PHASE void emit_phase(const MSParams& P, const uint32_t* Rn, uint32_t nR, const unsigned long long* Fn,
                           const LaneWord<W>& pushm, uint4* items_n, unsigned int* item_tail, Stage<kStageCap>& st,
                           uint32_t warp_gid, uint32_t nwarps) {
    const uint32_t lane = lane_id();
    const DevGraph& g = P.g;
    for (uint32_t base = warp_gid * 32; base < nR; base += nwarps * 32) {
        const uint32_t idx = base + lane;
        bool expand = false;
        uint32_t u = 0;
        if (idx < nR) {
            u = Rn[idx];
            const LaneWord<W> x = LS<W, NB>::load(Fn, u);
#pragma unroll
            for (int i = 0; i < W; ++i) expand |= (x.w[i] & pushm.w[i]) != 0;
            expand = expand && __ldg(g.rp + u + 1) > __ldg(g.rp + u);
        }
        st.push(expand, u);
        if (st.full()) {
            emit_items_lanes(P, st.buf, st.n, items_n, item_tail);
            st.n = 0;
        }
    }
    emit_items_lanes(P, st.buf, st.n, items_n, item_tail);
    st.n = 0;
}

// Per-lane out-edges of the frontier just found (one word per vertex): for
// each listed vertex, its out-degree is added to every lane whose bit is set in
// its new word -- one warp reduction per lane bit. Runs once per traversal,
// before the first pull: the lanes with few frontier edges ("stragglers": a
// low-degree seed's hop-2 frontier is a handful of vertices) then keep pushing,
// so the pull's early exit no longer waits for lanes almost no in-list covers.
template <int W, int NB>
MGK_PHASE void lane_edges_phase(const MSParams& P, const uint32_t* Rn, uint32_t nR, const unsigned long long* Fn,
                                uint32_t warp_gid, uint32_t nwarps) {
    if constexpr (W == 1) {
        constexpr uint32_t kBits = LS<W, NB>::kLanes;
        const uint32_t lane = lane_id();
        const DevGraph& g = P.g;
        unsigned long long e_lo = 0, e_hi = 0;
        for (uint32_t base = warp_gid * 32; base < nR; base += nwarps * 32) {
            const uint32_t idx = base + lane;
            unsigned long long x = 0;
            uint32_t deg = 0;
            if (idx < nR) {
                const uint32_t u = Rn[idx];
                x = LS<W, NB>::load(Fn, u).w[0];
                deg = min(__ldg(g.rp + u + 1) - __ldg(g.rp + u), 1u << 26);  // (32 of them fit 32 bits)
            }
            if (__ballot_sync(kFull, x != 0 && deg != 0) == 0) continue;
#pragma unroll 2
            for (uint32_t b = 0; b < kBits; ++b) {
                const uint32_t sum = __reduce_add_sync(kFull, ((x >> b) & 1ull) ? deg : 0u);
                if (lane == (b & 31)) {
                    if (b < 32) e_lo += sum; else e_hi += sum;
                }
            }
        }
        if (lane < kBits && e_lo) atomicAdd(&P.lane_E[lane], e_lo);
        if (32 + lane < kBits && e_hi) atomicAdd(&P.lane_E[32 + lane], e_hi);
    }
}

template <int W, int NB>
__device__ void clear_list(const uint32_t* R, uint32_t n, unsigned long long* F, uint32_t gtid,
                           uint32_t nthreads) {
    LaneWord<W> z;
#pragma unroll
    for (int i = 0; i < W; ++i) z.w[i] = 0;
    for (uint32_t i = gtid; i < n; i += nthreads) LS<W, NB>::store(F, R[i], z);
}

// Zero the lane words of the listed vertices: one scattered store each, or,
// for a list of more than 1/8 of the vertices (a dense pull's frontier),
// streaming 16-byte zeros over the whole array (coalesced, a fraction of the
// stores' time)
template <int W, int NB>
__device__ void clear_words(const uint32_t* R, uint32_t nlist, unsigned long long* F, uint32_t nv, uint32_t gtid,
                            uint32_t nthreads) {
    if ((uint64_t)nlist * 8 <= nv) {
        clear_list<W, NB>(R, nlist, F, gtid, nthreads);
        return;
    }
    const size_t w64 = LS<W, NB>::words64(nv);
    uint4* f4 = reinterpret_cast<uint4*>(F);
    for (size_t i = gtid; i < w64 / 2; i += nthreads) f4[i] = make_uint4(0, 0, 0, 0);
    if ((w64 & 1) && gtid == 0) F[w64 - 1] = 0;
}

// resident CTAs per SM the register budget is sized for, per instance: one
// word per vertex runs best at 48 registers and 40 warps per SM (more warps to
// hide the gathers' latency), wide words keep their registers. Narrow words
// on graphs whose lane-word arrays outgrow L2's fast range (kWideState) get a
// 40-register / 48-warp instance: their dense pull waits on gathers that miss
// L2 more often, and more warps in flight hide it (G4 10 seeds k=6: 5.16 ->
// 4.96 ms), while on small graphs the extra spills cost more (G2 +7 %).
template <int W, int MB>
constexpr int ms_min_blocks() {
    return MGK_MS_MINB > 0 ? MGK_MS_MINB : (W == 1 ? MB * 256 / kBlock : 512 / kBlock);
}
constexpr size_t kWideState = 16u << 20;

template <int W, int NB, int MB>
__global__ void __launch_bounds__(kBlock, ms_min_blocks<W, MB>()) ms_kernel(MSParams P) {
    grid_barrier_init(P.bar);
    // qctl[parity] fields in this engine:
    //   nitems = |R| (discovery list tail), nfound = push items built for the
    //   frontier, edges = sum of outdeg over R, pad = push-equivalent edges.
    constexpr uint32_t LB = LS<W, NB>::kLanes;
    __shared__ uint32_t s_stage[kWarps][kStageCap];
    __shared__ unsigned long long s_cnt[LB];
    __shared__ uint32_t s_nm[kWarps][32];  // pull: unsettled-vertex masks of a warp's 32 words
    __shared__ uint32_t s_cb[kWarps][64];  // pull: a warp's waiting candidates
    __shared__ unsigned long long s_strag;  // lanes that push while the others pull (the next hop's; 0: none)
    const uint32_t gtid = blockIdx.x * kBlock + threadIdx.x;
    const uint32_t nthreads = gridDim.x * kBlock;
    const uint32_t warp_gid = gtid >> 5;
    const uint32_t nwarps = nthreads >> 5;
    const DevGraph& g = P.g;
    Acc acc;
    acc.zero();
    Stage<kStageCap> st{s_stage[threadIdx.x >> 5], 0};
    const uint64_t nbatches = (P.nseeds + LB - 1) / LB;


    for (uint64_t bt = 0; bt < nbatches; ++bt) {
        const uint32_t lanes = (uint32_t)min((uint64_t)LB, P.nseeds - bt * LB);
        // ---- init ------------------------------------------------------------
        for (uint32_t i = gtid; i < (P.k + 1) * LB; i += nthreads) P.lane_cnt[i] = 0;
        if (gtid < 2 * W) P.active[gtid] = 0;
        if (gtid < 2) P.qctl[gtid] = QCtl{0, 0, 0, 0, 0};
        if (W == 1 && gtid < LB) P.lane_E[gtid] = 0;
        if (threadIdx.x == 0) s_strag = 0;
        if (gtid == 0) {
            P.misc[0] = g.m;
            P.misc[1] = P.misc[2] = 0;  // pull work counters
            P.misc[kHeavyCtl] = P.misc[kHeavyCtl + 1] = 0;  // heavy push records by parity
        }
        if (bt == 0)  // the first lc write is after the barrier below
            for (uint32_t i = gtid; i < (MGK_MAX_HOPS + 2) * (sizeof(LevelCounters) / 8); i += nthreads)
                reinterpret_cast<unsigned long long*>(P.lc)[i] = 0;
        grid_barrier(P.bar);
        // ---- seeds: level-0 frontier -------------------------------------------
        {
            bool first = false;
            uint32_t s = 0;
            if (gtid < lanes) {
                s = dev_id(g, P.seeds[bt * LB + gtid]);
                const unsigned long long bit = 1ULL << (gtid & 63);
                LS<W, NB>::atomic_or(P.F0, s, gtid >> 6, bit);
                const uint32_t tb = 1u << (s & 31);
                first = !(atomicOr(P.touched + (s >> 5), tb) & tb);

            }
            if (blockIdx.x * kBlock < lanes) {
                st.push(first, s);
                emit_list(st.buf, st.n, P.R0, &P.qctl[0].nitems);
                st.n = 0;
            }
        }
        block_flush(acc, &P.qctl[0], &P.qctl[0], &P.lc[0], nullptr, &P.misc[0]);
        grid_barrier(P.bar);
        // ---- finalize level 0 (V |= F0, hop-1 items) ------------------------------
        uint32_t nR = ld_volatile(&P.qctl[0].nitems);
        // the lanes pulling the current hop (all or none when the words are wider
        // than 64 lanes); hop 1 pushes unless a pull is forced
        const bool pull0 = P.force_dir == 2;
        bool pull_hop = pull0;  // (one flag for all lanes: a mask per lane word stayed live across the hop)
        for (uint32_t t = threadIdx.x; t < LB; t += kBlock) s_cnt[t] = 0;  // (LB may exceed the block)
        __syncthreads();
        finalize_phase<W, NB>(P, P.R0, nR, P.F0, P.seed_visited != 0, true, !pull0, P.items0, &P.qctl[0].nfound, false,
                          s_cnt, P.active, 0, acc, st, warp_gid, nwarps);
        __syncthreads();
        acc.pairs = 0;  // the seeds themselves are never counted
        block_flush(acc, &P.qctl[0], &P.qctl[0], &P.lc[0], &P.lc[1], &P.misc[0]);
        grid_barrier(P.bar);

        bool prev_pull = false;  // the hop before pulled: its unsettled words bound this pull's
        uint64_t clog_used = nR;
        uint32_t nR_prev = nR;
        uint32_t hop = 1;
        for (; hop <= P.k; ++hop) {
            const uint32_t cur = (hop - 1) & 1, nxt = hop & 1;
            QCtl* qc = &P.qctl[cur];
            QCtl* qn = &P.qctl[nxt];  // zeroed by init (hop 1) or the previous finalize
            unsigned long long* Fc = F_of(P, cur);
            unsigned long long* Fn = F_of(P, nxt);
            uint32_t* Rc = R_of(P, cur);
            uint32_t* Rn = R_of(P, nxt);
            // the lanes pulling this hop: all active ones of a pull hop but its
            // straggler lanes, which push (only with one word per vertex); the
            // pushing lanes' mask is rebuilt after the pull (not kept across it)
            LaneWord<W> pm;
            bool anypush = false, anypull = false;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                const unsigned long long a = ld_volatile(P.active + cur * W + i);
                const unsigned long long sm = (W == 1 && pull_hop) ? s_strag : 0ull;
                pm.w[i] = pull_hop ? (a & ~sm) : 0ull;
                anypush |= (pull_hop ? (a & sm) : a) != 0;
                anypull |= pm.w[i] != 0;
            }
            if (gtid == 0) {
                // the hop's start time is subtracted here and its end time added below:
                // no 64-bit timestamp stays live across the phases (registers)
                const unsigned long long t0 = globaltimer();
                atomicAdd(&P.lc[hop].ns, 0ULL - t0);
                if (P.diag) P.misc[6] = t0;
                atomicAdd(&P.lc[hop].runs, 1u);
                if (anypull) atomicAdd(&P.lc[hop].pull_runs, 1u);
                atomicAdd(&P.lc[hop].union_edges, ld_volatile(&qc->edges));
            }
            if (gtid < W) P.active[nxt * W + gtid] = 0;  // rebuilt by this hop's finalize
            // ---- expand: a push from the frontier's items or a pull over the CSC -----
            // A mixed hop (straggler lanes push, the others pull) pulls first: the
            // pull stores its words and lists its discoveries as in a pure pull,
            // and after a barrier the push ORs the stragglers' lanes in, listing a
            // vertex only when it finds the word still empty. Such a pull's
            // unsettled masks ignore the stragglers' needs, so the next pull does
            // not read them and visits every word again.
            if (anypush && !pull_hop) {
                LaneWord<W> pushm;
#pragma unroll
                for (int i = 0; i < W; ++i) pushm.w[i] = ld_volatile(P.active + cur * W + i);
                push_phase<W, NB>(P, items_of(P, cur), ld_volatile(&qc->nfound), ld_volatile(&P.misc[kHeavyCtl + cur]), Fc, Fn, Rn, qn, acc,
                              st, warp_gid, nwarps, pushm);
            }
            // a pull after a pull visits only the vertices that pull left unsettled
            if (anypull)
                pull_phase<W, NB>(P, Fc, Fn, pm, Rn, qn, acc, st, warp_gid, nwarps,
                                  prev_pull ? P.umask + (size_t)cur * g.nwords : nullptr,
                                  P.umask + (size_t)nxt * g.nwords,  // (a mixed hop's: never read)
                                  s_nm[threadIdx.x >> 5], s_cb[threadIdx.x >> 5]);
            prev_pull = anypull;
            if constexpr (W == 1) {
                // the stragglers' push of a mixed hop; its operands are derived again
                // from the hop number (laundered), so none of them is held in a
                // register across the pull
                const unsigned long long sm = pull_hop ? *(volatile unsigned long long*)&s_strag : 0ull;
                if (sm) {
                    uint32_t h2 = hop;
                    asm volatile("" : "+r"(h2));
                    const uint32_t c2 = (h2 - 1) & 1, n2 = h2 & 1;
                    LaneWord<W> pushm;
                    pushm.w[0] = ld_volatile(P.active + c2) & sm;
                    if (pushm.w[0]) {
                        grid_barrier(P.bar);
                        if (P.diag && gtid == 0) P.misc[3] = globaltimer();  // probe: where the pull part ended
                        push_phase<W, NB, false>(P, items_of(P, c2), ld_volatile(&P.qctl[c2].nfound),
                                          ld_volatile(&P.misc[kHeavyCtl + c2]), F_of(P, c2), F_of(P, n2), R_of(P, n2),
                                          &P.qctl[n2], acc, st, warp_gid, nwarps, pushm);
                        prev_pull = false;
                    }
                }
            }
            block_flush(acc, qn, qn, &P.lc[hop], nullptr, &P.misc[0]);
            grid_barrier(P.bar);
            if (P.diag && gtid == 0) P.misc[7] = globaltimer();
            nR = ld_volatile(&qn->nitems);
            // a mixed hop's push listed nothing: the hop counts as one that found
            // every vertex -- a dense finalize, streamed clears, and the next hop pulls
            if (W == 1 && anypull && !prev_pull && hop > 1 && P.force_dir == 0 && P.strag) nR = g.n;
            if (gtid == 0) P.misc[1] = P.misc[2] = 0;  // read again only after the finalize barrier
            const bool last = hop == P.k || nR == 0;
            const bool count_lanes = hop >= P.min_hop;
            const bool dense = W == 1 && (uint64_t)nR * kDenseDiv > g.n;
            // ---- finalize -------------------------------------------------------------
            for (uint32_t t = threadIdx.x; t < LB; t += kBlock) s_cnt[t] = 0;
            if (gtid == 0) {  // parity reused by hop + 1
                *qc = QCtl{0, 0, 0, 0, 0};
                P.misc[kHeavyCtl + cur] = 0;
            }
            if (W == 1 && P.strag && gtid < LB) P.lane_E[gtid] = 0;  // (read last before the expand barrier)
            __syncthreads();
            finalize_phase<W, NB>(P, Rn, nR, Fn, true, W > 1 && anypush, false, items_of(P, nxt), &qn->nfound, count_lanes,
                              s_cnt, P.active + nxt * W, clog_used, acc, st, warp_gid, nwarps,
                              dense);
            clear_words<W, NB>(Rc, nR_prev, Fc, g.n, gtid, nthreads);
            __syncthreads();
            if (count_lanes)
                for (uint32_t t = threadIdx.x; t < LB; t += kBlock)
                    if (s_cnt[t]) atomicAdd(&P.lane_cnt[hop * LB + t], s_cnt[t]);
            block_flush(acc, qn, qn, &P.lc[hop], hop < P.k ? &P.lc[hop + 1] : nullptr,
                        &P.misc[0]);
            grid_barrier(P.bar);
            // ---- the next hop's directions (every CTA computes the same) ---------------
            if (!last) {
                {
                    // (the finalize counted the new frontier's out-edges and the
                    // in-edges that left the unexplored set)
                    const unsigned long long mf = ld_volatile(&qn->edges);
                    const unsigned long long mu = ld_volatile(&P.misc[0]);
                    bool pn;
                    if (P.force_dir == 1) {
                        pn = false;
                    } else if (P.force_dir == 2) {
                        pn = true;
                    } else if (!anypull) {
                        pn = mf * P.alpha > mu;
                    } else {
                        pn = (unsigned long long)nR * P.beta >= g.n;
                    }
                    // the first pull of a traversal: lanes whose frontier has few
                    // out-edges keep pushing (every CTA computes the same mask)
                    if constexpr (W == 1) {
                        const bool first_pull = P.strag && pn && !anypull && P.force_dir == 0;
                        if (first_pull) {
                            lane_edges_phase<W, NB>(P, Rn, nR, Fn, warp_gid, nwarps);
                            grid_barrier(P.bar);
                        }
                        __syncthreads();  // (s_strag's readers are past the hop's top)
                        if (threadIdx.x == 0) {  // one thread per CTA: the lanes (active in the
                            // next frontier) with at most m / strag frontier out-edges
                            unsigned long long sm = 0;
                            if (first_pull) {
                                const unsigned long long an = ld_volatile(P.active + nxt * W);
                                for (uint32_t l = 0; l < LB; ++l)
                                    if (((an >> l) & 1ull) && ld_cg(&P.lane_E[l]) * P.strag <= g.m) sm |= 1ull << l;
                                if (sm == an) sm = 0;  // every lane a straggler: a plain pull
                            }
                            s_strag = sm;
                        }
                        __syncthreads();
                    }
                    pull_hop = pn;
                }
                // items for the lanes pushing next
                LaneWord<W> pn_push;
                bool anyn = false;
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    pn_push.w[i] = ld_volatile(P.active + nxt * W + i) & (pull_hop ? (W == 1 ? s_strag : 0ull) : ~0ull);
                    anyn |= pn_push.w[i] != 0;
                }
                if (anyn) {
                    emit_phase<W, NB>(P, Rn, nR, Fn, pn_push, items_of(P, nxt), &qn->nfound, st, warp_gid, nwarps);
                    grid_barrier(P.bar);
                }
            }
            if (gtid == 0) {
                const unsigned long long t2 = globaltimer();
                atomicAdd(&P.lc[hop].ns, t2);
                if (P.diag) {  // probe mode: phase split (the counters these fields hold are lost)
                    P.lc[hop].union_edges = P.misc[7] - P.misc[6];
                    P.lc[hop].candidates = t2 - P.misc[7];
                    if (P.misc[3]) {  // a mixed hop: its pull part's ns in lc.edges
                        P.lc[hop].edges = P.misc[3] - P.misc[6];
                        P.misc[3] = 0;
                    }
                }
            }
            clog_used += nR;
            nR_prev = nR;
            if (nR == 0) break;
        }
        // ---- answers ------------------------------------------------------------------
        if (gtid < lanes) {
            unsigned long long r = 0;
            for (uint32_t h = P.ans_lo; h <= P.ans_hi; ++h) r += P.lane_cnt[h * LB + gtid];
            P.counts[bt * LB + gtid] = r;
            for (uint32_t j = 0; j < P.nextra; ++j) {
                unsigned long long x = 0;
                for (uint32_t h = P.xlo[j]; h <= P.xhi[j]; ++h) x += P.lane_cnt[h * LB + gtid];
                P.xout[j][bt * LB + gtid] = x;
            }
        }
        // ---- clear V and the last frontier (state is all-zero between batches) ---------
        const uint32_t last_par = (hop > P.k ? P.k : hop) & 1;
        // (a dense finalize lists nothing in clog: it needs nR * kDenseDiv > n, and
        // then clog_used * kClearDiv > n too, so V is cleared by streaming; no flag
        // is kept across the hops -- one more live register spilled the pull)
        constexpr uint64_t kClearDiv = kDenseDiv > 8 ? kDenseDiv : 8;
        if (clog_used <= P.clog_cap && clog_used * kClearDiv <= g.n) {
            clear_list<W, NB>(P.clog, (uint32_t)clog_used, P.V, gtid, nthreads);
            clear_words<W, NB>(R_of(P, last_par), nR_prev, F_of(P, last_par), g.n, gtid, nthreads);
        } else if (clog_used <= P.clog_cap) {
            // most vertices visited: stream zeros over V (coalesced) instead of
            // one scattered store per visited vertex
            for (size_t i = gtid; i < LS<W, NB>::words64(g.n); i += nthreads) P.V[i] = 0;
            clear_words<W, NB>(R_of(P, last_par), nR_prev, F_of(P, last_par), g.n, gtid, nthreads);
        } else {
            for (size_t i = gtid; i < LS<W, NB>::words64(g.n); i += nthreads) {
                P.V[i] = 0;
                P.F0[i] = 0;
                P.F1[i] = 0;
            }
        }
        grid_barrier(P.bar);
    }
}

// Graph::top4: the first four in-neighbours of every vertex, padded with the first
__global__ void top4_kernel(DevGraph g, uint4* out) {
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < g.n; u += gridDim.x * blockDim.x) {
        const uint32_t b = __ldg(g.cp + u), d = __ldg(g.cp + u + 1) - b;
        uint4 t = make_uint4(0, 0, 0, 0);
        if (d) {
            t.x = __ldg(g.ri + b);
            t.y = d > 1 ? __ldg(g.ri + b + 1) : t.x;
            t.z = d > 2 ? __ldg(g.ri + b + 2) : t.x;
            t.w = d > 3 ? __ldg(g.ri + b + 3) : t.x;
        }
        out[u] = t;
    }
}

cudaError_t ensure_top4(const Graph* gr, cudaStream_t stream) {
    static const bool off = std::getenv("MGK_NO_TOP4") != nullptr;
    if (off || !MGK_TOP4 || gr->top4) return cudaSuccess;
    Graph* gm = const_cast<Graph*>(gr);
    std::lock_guard<std::mutex> lk(gm->mu);
    if (gm->top4) return cudaSuccess;
    uint4* t = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&t, (size_t)std::max<uint32_t>(gm->dg.n, 1) * sizeof(uint4)))) return e;
    top4_kernel<<<1184, 256, 0, stream>>>(gm->dg, t);
    if ((e = cudaGetLastError()) || (e = cudaStreamSynchronize(stream))) {
        cudaFree(t);
        return e;
    }
    gm->top4 = t;
    gm->bytes += (size_t)gm->dg.n * sizeof(uint4);
    return cudaSuccess;
}

template <int W, int NB, int MB>
cudaError_t launch_w(Launch& L) {
    static int blocks_per_sm = 0, num_sms = 0;
    cudaError_t e;
    if (blocks_per_sm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, ms_kernel<W, NB, MB>, kBlock,
                                                                0)))
            return e;
        if (blocks_per_sm < 1) return cudaErrorInvalidConfiguration;
    }
    const Graph* gr = L.g;
    Workspace* ws = L.ws;
    MSParams P;
    P.g = gr->dg;
    P.seeds = L.d_seeds;
    P.nseeds = L.nseeds;
    P.k = L.k;
    P.min_hop = L.min_hop;
    P.nextra = L.nextra;
    P.ans_lo = L.nextra ? L.ans_lo : L.min_hop;
    P.ans_hi = L.nextra ? L.ans_hi : L.k;
    for (int j = 0; j < Launch::kMaxExtra; ++j) {
        P.xlo[j] = L.xlo[j];
        P.xhi[j] = L.xhi[j];
        P.xout[j] = L.xout[j];
    }
    P.seed_visited = L.seed_visited;
    P.counts = L.d_counts;
    P.V = ws->lv;
    P.F0 = ws->lf[0];
    P.F1 = ws->lf[1];
    // narrow words: both frontier arrays inside lf[0]'s allocation (n uint64
    // words hold 8 / NB * ... of them), adjacent, so one L2 window covers them
    static const bool separate = std::getenv("MGK_F1_SEPARATE") != nullptr;  // A/B of the layout
    const size_t fbytes = (narrow_bytes<W, NB>(gr->dg.n) + 255) / 256 * 256;
    if (NB < 64 && !separate)
        P.F1 = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ws->lf[0]) + fbytes);
    P.touched = ws->touched;
    P.R0 = ws->rlog;
    P.R1 = ws->rlog + gr->dg.n;
    P.clog = ws->rlog + 2 * (size_t)gr->dg.n;
    P.clog_cap = ws->rlog_cap - 2 * (uint64_t)gr->dg.n;
    P.items0 = ws->ms_items[0];
    P.items1 = ws->ms_items[1];
    P.items_cap = (uint32_t)(gr->dg.m / kChunk + gr->dg.n + 64);  // as allocated (ensure_lanes_ws)
    P.lane_cnt = ws->lane_cnt;
    P.active = ws->active;
    P.qctl = ws->qctl;
    P.misc = ws->misc;
    P.lc = ws->lc;
    P.bar = reinterpret_cast<unsigned int*>(ws->misc + 8);
    static const uint32_t diag = [] {
        const char* e = std::getenv("MGK_MS_DIAG");
        return e && e[0] == '1' ? 1u : 0u;
    }();
    P.diag = diag;
    static const uint32_t strag = [] {
        const char* e = std::getenv("MGK_STRAG");
        return e ? (uint32_t)std::atoi(e) : (uint32_t)MGK_STRAG_DEFAULT;
    }();
    P.strag = W == 1 ? strag : 0u;
    P.lane_E = ws->lane_cnt + (size_t)(MGK_MAX_HOPS + 1) * 64 * W;  // the row after the hops' counts
    P.top4 = nullptr;
    if (W == 1) {
        cudaError_t te = ensure_top4(gr, L.stream);
        if (te) return te;
        P.top4 = gr->top4;
    }
    P.umask = ws->umask;
    P.alpha = L.tuning.alpha_lanes;
    P.beta = L.tuning.beta;
    P.force_dir = L.tuning.force_dir;
    L.grid = (uint32_t)(blocks_per_sm * num_sms);
    L.block = kBlock;
    void* args[] = {&P};
    L.launches = 1;
    static const bool persist = [] {
        const char* v = std::getenv("MGK_L2_PERSIST");
        return v && v[0] == '1';
    }();
    if (persist && NB < 64)
        return launch_persistent_l2((const void*)ms_kernel<W, NB, MB>, L.grid, kBlock, args, L.stream, ws->lf[0],
                                    2 * fbytes);
    return launch_persistent((const void*)ms_kernel<W, NB, MB>, L.grid, kBlock, args, L.stream);
}

}  // namespace

cudaError_t ensure_lanes_ws(const Graph* gr, Workspace* ws, int W) {
    if (ws->lanes_words >= W) return cudaSuccess;
    cudaError_t e;
    if (ws->lv) {  // grow: release the narrower buffers
        cudaFree(ws->lv);
        cudaFree(ws->lf[0]);
        cudaFree(ws->lf[1]);
        cudaFree(ws->lane_cnt);
        cudaFree(ws->active);
        ws->lv = ws->lf[0] = ws->lf[1] = ws->lane_cnt = ws->active = nullptr;
    }
    const DevGraph& g = gr->dg;
    // (+64 words: the narrow layout puts both frontier arrays, 256-B aligned,
    // in lf[0], which must hold 2 round_up(2 n, 256) bytes even for tiny n)
    const size_t words = (size_t)g.n * W + 66;
    for (unsigned long long** p : {&ws->lv, &ws->lf[0], &ws->lf[1]}) {
        if ((e = cudaMalloc(p, words * 8))) return e;
        if ((e = cudaMemset(*p, 0, words * 8))) return e;
    }
    if ((e = cudaMalloc(&ws->lane_cnt, (size_t)(MGK_MAX_HOPS + 2) * 64 * W * 8))) return e;  // (+ lane_E)
    if ((e = cudaMalloc(&ws->active, (size_t)2 * W * 8))) return e;
    if (!ws->umask && (e = cudaMalloc(&ws->umask, 2 * ((size_t)g.nwords + 32) * 4))) return e;
    ws->bytes += 3 * words * 8;
    if (!ws->touched) {
        if ((e = cudaMalloc(&ws->touched, (size_t)(g.nwords + 1) * 4))) return e;
        if ((e = cudaMemset(ws->touched, 0, (size_t)(g.nwords + 1) * 4))) return e;
        ws->rlog_cap = 4 * (uint64_t)g.n + 1024;
        if ((e = cudaMalloc(&ws->rlog, ws->rlog_cap * 4))) return e;
        const size_t items = (size_t)(g.m / kChunk + g.n + 64);
        for (int i = 0; i < 2; ++i)
            if ((e = cudaMalloc(&ws->ms_items[i], items * sizeof(uint4)))) return e;
        ws->bytes += (size_t)(g.nwords + 1) * 4 + ws->rlog_cap * 4 + 2 * items * sizeof(uint4);
    }
    ws->lanes_words = W;
    // zero state complete before the first launch on a non-blocking stream
    return cudaStreamSynchronize(0);
}

cudaError_t launch_lanes(Launch& L) {
    int W = L.lanes_words;
    cudaError_t e = ensure_lanes_ws(L.g, L.ws, W);
    if (e) return e;
    const uint32_t n = L.g->dg.n;
    // MGK_MS_MB=5 / 6 forces the narrow instances' CTAs per SM (A/B runs)
    static const int mb = [] {
        const char* v = std::getenv("MGK_MS_MB");
        return v ? std::atoi(v) : 0;
    }();
    if (L.lane_bits == 16)
        return (mb ? mb == 6 : narrow_bytes<1, 16>(n) > kWideState) ? launch_w<1, 16, 6>(L) : launch_w<1, 16, 5>(L);
    if (L.lane_bits == 10)
        return (mb ? mb == 6 : narrow_bytes<1, 10>(n) > kWideState) ? launch_w<1, 10, 6>(L) : launch_w<1, 10, 5>(L);
    if (L.lane_bits == 8) return launch_w<1, 8, 5>(L);
    switch (W) {
        case 1: return launch_w<1, 64, 5>(L);
        case 2: return launch_w<2, 64, 5>(L);
        case 4: return launch_w<4, 64, 5>(L);
        case 8: return launch_w<8, 64, 5>(L);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace mgk
