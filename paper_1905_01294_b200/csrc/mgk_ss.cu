// SINGLE engine: independent single-source traversals with per-seed bitmap
// state, up to S seeds in flight at once, direction-optimizing per seed.
//
// Replaces the per-query loop of k_hop_frontier (proj/core/src/execute.cpp:347-371)
// and its vxm / ewise_union calls (proj/core/src/sparse.cpp:253-290, 365-377):
//   * each seed slot owns a visited bitmap and three rotating frontier bitmaps
//     (n/8 bytes each) instead of sorted uint64 vectors plus two dense char
//     arrays zeroed every hop;
//   * the masked vxm is, per seed and per hop, either a push pass over the
//     frontier's out-edges (CSR) with atomicOr test-and-set on the seed's
//     visited bitmap, or a pull pass over the seed's unvisited vertices'
//     in-edges (CSC) that stops at the first frontier hit (Beamer's
//     direction optimization, decided per seed on the device);
//   * ewise_union is the same atomicOr; nvals is a per-seed discovery counter.
// All hops of all seeds run inside one persistent cooperative launch. Hops are
// separated by grid-wide barriers; every decision is taken on the device from
// counters all CTAs read after the barrier, so there is no host round trip.
//
// Load balance: push work items are (begin, len<=32, seed) slices of CSR rows,
// written when a vertex is discovered, so a 100K-degree hub is spread over
// thousands of warps; the items of ALL in-flight seeds form one global list and
// each warp takes 1..32 items per step (fewer when the list is short, so a
// small hop still occupies every warp of the grid). The last hop only counts.
#include <cstdlib>
#include <cstring>

#include "mgk_device.cuh"

namespace mgk {
namespace {

using namespace dev;

constexpr int kBlock = 512;
constexpr int kWarps = kBlock / 32;
constexpr int kStageCap = 256;
constexpr int kIlp = 4;
constexpr uint32_t kBigChunk = 1024;  // rows longer than this become 1024-entry big items
constexpr uint32_t kMaxSlots = 512;
constexpr uint32_t kSeedChunk = 32;  // fused hop 1: seed-row entries per warp task
constexpr unsigned long long kOverflowBit = 1ULL << 62;
enum : uint8_t { kPush = 0, kPull = 1, kDead = 2 };

struct FRCtl {
    unsigned int nitems[3];  // items for hop h: buffer h & 1, count nitems[h % 3]
    unsigned int nbig[3];    // big items (1024-entry slices of rows longer than 1024)
    unsigned int log_n;
    unsigned int log_overflow;
    unsigned int pad;
    unsigned long long found[MGK_MAX_HOPS + 1];
    unsigned long long last_which;  // frontier bitmap id of the final hop (frontier ids)
    unsigned int done;              // CTAs finished with the cleanup (last one answers)
    unsigned long long t_clean;     // cleanup start (%globaltimer), for the stats
    unsigned long long t_last;      // start of the last hop expanded (its end = fr_finish start)
    unsigned int last_hop;          // last hop expanded by fr_kernel
};

struct FRParams {
    DevGraph g;
    const uint32_t* seeds;  // this group's seeds (ns of them)
    uint32_t ns;
    uint32_t k;          // max hop
    uint32_t min_hop;    // answer = sum of |F_h| for h in [min_hop, k]
    uint32_t seed_visited;  // 1: k_hop_* (seed pre-visited); 0: walk_targets (visited starts empty)
    unsigned long long* counts;  // this group's answers
    uint32_t S;
    uint32_t rs;   // bitmap row stride in words (nwords rounded up to 32: 128-B rows)
    uint32_t* V;   // [S][rs]
    uint32_t* Fb;  // [3][S][rs]
    uint2* items0;
    uint2* items1;
    uint32_t items_cap;
    uint2* big0;  // {begin, slot << 10 | (len - 1)}, len <= kBigChunk
    uint2* big1;
    uint32_t big_cap;
    unsigned long long* logbuf;
    uint32_t log_cap;
    uint32_t* cnt;             // [(k+1)][S] discoveries per hop per seed
    unsigned long long* mfs;   // [(k+1)][S] out-edges of those discoveries
    unsigned long long* mex;   // [S] explored in-edges per seed (unexplored = m - mex)
    uint32_t* logcnt;          // [S] 1 = last hop not logged: clear V densely
    unsigned long long* pop;   // [S] popcount of V for those seeds (counting pass)
    uint8_t* dirs;             // [2][S]
    FRCtl* ctl;
    unsigned int* bar;
    LevelCounters* lc;
    uint32_t alpha, beta, force_dir, alpha_last;
    uint32_t* snap;  // keep_result: slot 0's visited bitmap after hop min_hop - 1
    uint32_t quota;  // per-seed log entries before the seed is cleared densely
    uint32_t keep_result;  // one seed, bitmaps kept for k_hop_frontier
    uint32_t zero_lc;      // first group of a call: clear the per-hop counters
    uint32_t fuse1;        // rows unique, seed pre-visited, k >= 2: hop 1 = the seed rows
    // host calls: this group's seeds travel inside the launch (seeds == nullptr)
    uint32_t inline_seeds[kMaxSlots];
};

__device__ __forceinline__ uint32_t seed_at(const FRParams& P, uint32_t i) {
    return P.seeds ? P.seeds[i] : P.inline_seeds[i];
}

struct Acc {
    unsigned long long found, scanned, candidates;
    __device__ void zero() { found = scanned = candidates = 0; }
};

__device__ void block_flush(Acc& a, unsigned long long* found_total, LevelCounters* lc) {
    __shared__ unsigned long long s[3];
    if (threadIdx.x < 3) s[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long f = warp_sum_u64(a.found), sc = warp_sum_u64(a.scanned),
                             c = warp_sum_u64(a.candidates);
    if (lane_id() == 0) {
        if (f) atomicAdd(&s[0], f);
        if (sc) atomicAdd(&s[1], sc);
        if (c) atomicAdd(&s[2], c);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s[0]) {
            atomicAdd(found_total, s[0]);
            atomicAdd(&lc->frontier, s[0]);
            atomicAdd(&lc->vertices, s[0]);
        }
        if (s[1]) atomicAdd(&lc->scanned, s[1]);
        if (s[2]) atomicAdd(&lc->candidates, s[2]);
    }
    __syncthreads();
    a.zero();
}

// Warp-wide: per distinct slot among the valid lanes, add the lane count (and,
// before the last hop, the summed out / in degrees) to that seed's counters
// with one fire-and-forget atomic each.
__device__ __forceinline__ void slot_commit(const FRParams& P, uint32_t hop, bool valid,
                                            uint32_t slot, uint32_t deg, uint32_t indeg,
                                            bool last) {
    unsigned pending = __ballot_sync(kFull, valid);
    while (pending) {
        const int leader = __ffs(pending) - 1;
        const uint32_t s = __shfl_sync(kFull, slot, leader);
        const bool mine = valid && slot == s;
        const unsigned grp = __ballot_sync(kFull, mine);
        unsigned long long d = mine ? deg : 0, i = mine ? indeg : 0;
        if (!last) {
            d = warp_sum_u64(d);
            i = warp_sum_u64(i);
        }
        if ((int)lane_id() == leader) {
            atomicAdd(&P.cnt[hop * P.S + s], (unsigned)__popc(grp));
            if (!last) {
                atomicAdd(&P.mfs[hop * P.S + s], d);
                atomicAdd(&P.mex[s], i);
            }
        }
        pending &= ~grp;
    }
}

// Warp-wide: push work items for the next hop (hop + 1) for each lane's row
// (b, deg) of seed `slot`. Rows up to kBigChunk entries become <= 32-entry
// items (each warp step of the next hop merges up to 32 of them); longer rows
// become kBigChunk-entry big items (one warp step each), so one warp never
// writes more than ~32 items per discovered vertex.
__device__ void emit_row_items(const FRParams& P, uint32_t hop, bool valid, uint32_t slot,
                               uint32_t b, uint32_t deg) {
    const uint32_t lane = lane_id();
    const bool big = valid && deg > kBigChunk;
    const uint32_t par = (hop + 1) & 1, cidx = (hop + 1) % 3;
    // small items
    {
        const uint32_t nit = (valid && !big) ? (deg + kChunk - 1) / kChunk : 0;
        const uint32_t incl = warp_incl_scan(nit);
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        if (total) {
            uint32_t base = 0;
            if (lane == 31) base = atomicAdd(&P.ctl->nitems[cidx], total);
            base = __shfl_sync(kFull, base, 31);
            if ((uint64_t)base + total > P.items_cap) {
                // out of item space: these seeds pull next hop (pull needs no items)
                if (nit) atomicOr(&P.mfs[hop * P.S + slot], kOverflowBit);
            } else {
                uint2* items = par ? P.items1 : P.items0;
                const uint32_t excl = incl - nit;
                for (uint32_t x0 = 0; x0 < total; x0 += 32) {
                    const uint32_t x = x0 + lane;
                    const uint32_t j = warp_owner(incl, x < total ? x : total - 1);
                    const uint32_t bj = __shfl_sync(kFull, b, j);
                    const uint32_t dj = __shfl_sync(kFull, deg, j);
                    const uint32_t ej = __shfl_sync(kFull, excl, j);
                    const uint32_t sj = __shfl_sync(kFull, slot, j);
                    if (x < total) {
                        const uint32_t s = bj + (x - ej) * kChunk;
                        items[base + x] = make_uint2(s, (sj << 5) | (min(kChunk, bj + dj - s) - 1));
                    }
                }
            }
        }
    }
    // big items
    const unsigned bigmask = __ballot_sync(kFull, big);
    if (!bigmask) return;
    const uint32_t nbg = big ? (deg + kBigChunk - 1) / kBigChunk : 0;
    const uint32_t incl = warp_incl_scan(nbg);
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    uint32_t base = 0;
    if (lane == 31) base = atomicAdd(&P.ctl->nbig[cidx], total);
    base = __shfl_sync(kFull, base, 31);
    if ((uint64_t)base + total > P.big_cap) {
        if (nbg) atomicOr(&P.mfs[hop * P.S + slot], kOverflowBit);
        return;
    }
    uint2* bigs = par ? P.big1 : P.big0;
    const uint32_t excl = incl - nbg;
    for (uint32_t x0 = 0; x0 < total; x0 += 32) {
        const uint32_t x = x0 + lane;
        const uint32_t j = warp_owner(incl, x < total ? x : total - 1);
        const uint32_t bj = __shfl_sync(kFull, b, j);
        const uint32_t dj = __shfl_sync(kFull, deg, j);
        const uint32_t ej = __shfl_sync(kFull, excl, j);
        const uint32_t sj = __shfl_sync(kFull, slot, j);
        if (x < total) {
            const uint32_t s = bj + (x - ej) * kBigChunk;
            bigs[base + x] = make_uint2(s, (sj << 10) | (min(kBigChunk, bj + dj - s) - 1));
        }
    }
}

// Warp-wide emission of n staged (slot << 32 | u) discoveries of `hop`:
// per-seed counters, the cleanup log, and (unless this is the last hop) the
// next hop's push items. Discoveries before the last hop are always logged
// (they also mark frontier bitmaps); last-hop discoveries only for seeds whose
// last hop was predicted small (s_logok), the others are cleared densely.
__device__ void emit(const FRParams& P, uint32_t hop, bool last, const uint8_t* s_logok,
                     const unsigned long long* buf, uint32_t n) {
    if (n == 0) return;
    const uint32_t lane = lane_id();
    const DevGraph& g = P.g;
    // one log reservation for the whole stage
    uint32_t nlog = 0;
    for (uint32_t i = lane; i < n; i += 32)
        nlog += (!last || s_logok[(uint32_t)(buf[i] >> 32)]) ? 1u : 0u;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) nlog += __shfl_xor_sync(kFull, nlog, d);
    uint32_t log_base = 0;
    if (nlog) {
        if (lane == 0) log_base = atomicAdd(&P.ctl->log_n, nlog);
        log_base = __shfl_sync(kFull, log_base, 0);
    }
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        const bool valid = i < n;
        uint32_t u = 0, slot = 0, b = 0, deg = 0, indeg = 0;
        if (valid) {
            const unsigned long long e = buf[i];
            u = (uint32_t)e;
            slot = (uint32_t)(e >> 32);
            if (!last) {
                b = __ldg(g.rp + u);
                deg = __ldg(g.rp + u + 1) - b;
                indeg = __ldg(g.cp + u + 1) - __ldg(g.cp + u);
            }
        }
        slot_commit(P, hop, valid, slot, deg, indeg, last);
        const bool loggable = valid && (!last || s_logok[slot]);
        const unsigned lm = __ballot_sync(kFull, loggable);
        if (loggable) {
            const uint32_t at = log_base + __popc(lm & lanemask_lt());
            // bit 63 marks a last-hop entry: it has no frontier bit to clear
            if (at < P.log_cap)
                P.logbuf[at] = ((unsigned long long)(last ? 0x80000000u | slot : slot) << 32) | u;
            else P.ctl->log_overflow = 1;
        }
        log_base += __popc(lm);
        if (last) continue;
        emit_row_items(P, hop, valid, slot, b, deg);
    }
    __syncwarp();
}

__device__ __forceinline__ void stage_push(const FRParams& P, uint32_t hop, bool last,
                                           const uint8_t* s_logok,
                                           Stage<kStageCap, unsigned long long>& st, bool found,
                                           uint32_t slot, uint32_t u) {
    st.push(found, ((unsigned long long)slot << 32) | u);
    if (st.full()) {
        emit(P, hop, last, s_logok, st.buf, st.n);
        st.n = 0;
    }
}

// Visit kIlp adjacency entries per lane (targets u of seeds sj): test-and-set
// the seed's visited bit; new vertices go to the frontier bitmap and the stage.
__device__ __forceinline__ void visit_edges(const FRParams& P, uint32_t hop, bool last,
                                            const uint8_t* s_logok,
                                            Stage<kStageCap, unsigned long long>& st, Acc& acc,
                                            const uint32_t (&u)[kIlp], const uint32_t (&sj)[kIlp],
                                            const bool (&valid)[kIlp]) {
    const uint32_t fn = hop % 3;
    const bool set_fb = !last || P.keep_result;
    const unsigned long long pol = l2_keep_policy();
    uint32_t old[kIlp];
#pragma unroll
    for (int r = 0; r < kIlp; ++r) {
        old[r] = kFull;
        if (valid[r]) {
            uint32_t* vw = P.V + (size_t)sj[r] * P.rs + (u[r] >> 5);
            const uint32_t bit = 1u << (u[r] & 31);
            // a seed's last hop that is not logged only sets bits
            // (fire-and-forget red.or); it is counted afterwards by a
            // popcount of the bitmap in the clearing pass
            if (last && !s_logok[sj[r]]) red_or_keep(vw, bit, pol);
            else old[r] = atom_or_keep(vw, bit, pol);
        }
    }
#pragma unroll
    for (int r = 0; r < kIlp; ++r) {
        const bool found = !((old[r] >> (u[r] & 31)) & 1u);
        if (found && set_fb)
            red_or_keep(P.Fb + ((size_t)fn * P.S + sj[r]) * P.rs + (u[r] >> 5), 1u << (u[r] & 31), pol);
        acc.scanned += valid[r];
        acc.found += found;
        stage_push(P, hop, last, s_logok, st, found, sj[r], u[r]);
    }
}

// Push: expand the work items of seeds in push mode.
__device__ void push_phase(const FRParams& P, uint32_t hop, bool last, const uint8_t* s_dir,
                           const uint8_t* s_logok, Stage<kStageCap, unsigned long long>& st,
                           Acc& acc, uint32_t warp_gid, uint32_t nwarps) {
    const uint32_t lane = lane_id();
    const DevGraph& g = P.g;
    const uint32_t nsmall = min(ld_volatile(&P.ctl->nitems[hop % 3]), P.items_cap);
    const uint32_t nbig = min(ld_volatile(&P.ctl->nbig[hop % 3]), P.big_cap);
    const uint2* items = (hop & 1) ? P.items1 : P.items0;
    const uint2* bigs = (hop & 1) ? P.big1 : P.big0;
    // a big item (<= 1024 entries) is consumed as 32 virtual <= 32-entry items
    const uint32_t nitems = nsmall + nbig * 32;
    // ~8 steps per warp at least, so the tail of the hop stays balanced
    const uint32_t G = items_per_warp(nitems, (uint64_t)nwarps * 8);
    for (uint32_t base = warp_gid * G; base < nitems; base += nwarps * G) {
        const uint32_t idx = base + lane;
        uint32_t len = 0, slot = 0, beg = 0;
        if (lane < G && idx < nitems) {
            if (idx < nsmall) {
                const uint2 it = items[idx];
                slot = it.y >> 5;
                len = (it.y & 31) + 1;
                beg = it.x;
            } else {
                const uint32_t v = idx - nsmall, sub = (v & 31) * kChunk;
                const uint2 it = bigs[v >> 5];
                slot = it.y >> 10;
                const uint32_t blen = (it.y & 1023) + 1;
                len = sub < blen ? min(kChunk, blen - sub) : 0;
                beg = it.x + sub;
            }
            if (s_dir[slot] != kPush) len = 0;
        }
        const uint32_t incl = warp_incl_scan(len);
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        const uint32_t off = beg - (incl - len);
        // kIlp edges per lane per step: all loads / atomics of a step in flight together
        for (uint32_t x0 = 0; x0 < total; x0 += 32 * kIlp) {
            uint32_t u[kIlp], sj[kIlp];
            bool valid[kIlp];
#pragma unroll
            for (int r = 0; r < kIlp; ++r) {
                const uint32_t x = x0 + r * 32 + lane;
                valid[r] = x < total;
                const uint32_t j = warp_owner(incl, valid[r] ? x : total - 1);
                const uint32_t pos = __shfl_sync(kFull, off, j) + x;
                sj[r] = __shfl_sync(kFull, slot, j);
                u[r] = valid[r] ? __ldcs(g.ci + pos) : 0;  // streamed: keep bitmaps in L2
            }
            visit_edges(P, hop, last, s_logok, st, acc, u, sj, valid);
        }
    }
}

__device__ __forceinline__ bool fbit(const uint32_t* f, uint32_t v) {
    return (f[v >> 5] >> (v & 31)) & 1u;
}

// Pull: for every seed in pull mode, every unvisited vertex with in-edges
// scans its in-neighbours (CSC, ascending) until one is in the seed's
// frontier. One warp owns one (seed, bitmap word) so V / F words are written
// without atomics.
__device__ void pull_phase(const FRParams& P, uint32_t hop, bool last, const uint16_t* s_pull,
                           uint32_t npull, const uint8_t* s_logok,
                           Stage<kStageCap, unsigned long long>& st, Acc& acc, uint32_t warp_gid,
                           uint32_t nwarps) {
    const uint32_t lane = lane_id();
    const DevGraph& g = P.g;
    const uint32_t nw = g.nwords;
    const uint64_t total = (uint64_t)npull * nw;
    for (uint64_t t = warp_gid; t < total; t += nwarps) {
        const uint32_t pi = (uint32_t)(t / nw);
        const uint32_t w = (uint32_t)(t - (uint64_t)pi * nw);
        const uint32_t slot = s_pull[pi];
        uint32_t* vword = P.V + (size_t)slot * P.rs + w;
        const uint32_t vis = *vword;
        const uint32_t done = vis | __ldg(g.no_in + w);
        if (done == kFull) continue;
        const uint32_t* fcur = P.Fb + ((size_t)((hop - 1) % 3) * P.S + slot) * P.rs;
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
            uint32_t p = b;
            for (; p + 4 <= e; p += 4) {
                const uint32_t v0 = __ldg(g.ri + p), v1 = __ldg(g.ri + p + 1),
                               v2 = __ldg(g.ri + p + 2), v3 = __ldg(g.ri + p + 3);
                scanned += 4;
                if (fbit(fcur, v0) | fbit(fcur, v1) | fbit(fcur, v2) | fbit(fcur, v3)) {
                    found = true;
                    break;
                }
            }
            if (!found) {
                for (; p < e; ++p) {
                    ++scanned;
                    if (fbit(fcur, __ldg(g.ri + p))) {
                        found = true;
                        break;
                    }
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
                const bool h = p < ej && fbit(fcur, __ldg(g.ri + p));
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
        acc.found += found;
        const unsigned fm = __ballot_sync(kFull, found);
        if (fm) {
            if (lane == 0) {
                *vword = vis | fm;
                if (!last || P.keep_result) P.Fb[((size_t)(hop % 3) * P.S + slot) * P.rs + w] = fm;
            }
        }
        stage_push(P, hop, last, s_logok, st, found, slot, u);
    }
}

__global__ void __launch_bounds__(kBlock) fr_kernel(FRParams P) {
    grid_barrier_init(P.bar);
    __shared__ unsigned long long s_stage[kWarps][kStageCap];
    __shared__ uint8_t s_dir[kMaxSlots];
    __shared__ uint8_t s_flag[kMaxSlots];  // last hop: log it; cleanup: clear V densely
    __shared__ uint16_t s_list[kMaxSlots];
    __shared__ uint32_t s_wcount[kWarps];
    __shared__ uint32_t s_nlist;
    const uint32_t gtid = blockIdx.x * kBlock + threadIdx.x;
    const uint32_t nthreads = gridDim.x * kBlock;
    const uint32_t warp_gid = gtid >> 5;
    const uint32_t nwarps = nthreads >> 5;
    const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
    const DevGraph& g = P.g;
    const uint32_t nw = g.nwords;
    const uint32_t S = P.S;
    Acc acc;
    acc.zero();
    Stage<kStageCap, unsigned long long> st{s_stage[wib], 0};

    // block-wide ordered compaction of slots satisfying pred into s_list
    auto compact = [&](bool pred) {
        const unsigned m = __ballot_sync(kFull, pred);
        if (lane == 0) s_wcount[wib] = __popc(m);
        __syncthreads();
        uint32_t off = 0, tot = 0;
        for (uint32_t i = 0; i < kWarps; ++i) {
            if (i < wib) off += s_wcount[i];
            tot += s_wcount[i];
        }
        if (pred) s_list[off + __popc(m & lanemask_lt())] = (uint16_t)threadIdx.x;
        if (threadIdx.x == 0) s_nlist = tot;
        __syncthreads();
    };

    const uint32_t ns = P.ns;
    unsigned long long t_init = 0;
    if (gtid == 0) t_init = globaltimer();
    if (P.fuse1) {
        // ---- seeds and hop 1 in one phase: with duplicate-free rows, F_1 of a
        // seed is its row minus the seed, so every entry is a discovery and the
        // bits are set fire-and-forget. Tasks are kSeedChunk-entry slices of
        // the seed rows (a hub seed is spread over many warps).
        __shared__ uint32_t s_pref[kMaxSlots];
        __shared__ uint32_t s_ntask, s_logbase;
        // the seed log entries get their own reservation (hop-1 emits run concurrently)
        if (blockIdx.x == 0) {
            if (threadIdx.x == 0) s_logbase = atomicAdd(&P.ctl->log_n, ns);
            __syncthreads();
        }
        uint32_t c = 0;
        if (threadIdx.x < ns) {
            const uint32_t sd = dev_id(g, seed_at(P, threadIdx.x));
            const uint32_t b = __ldg(g.rp + sd), deg = __ldg(g.rp + sd + 1) - b;
            c = (deg + kSeedChunk - 1) / kSeedChunk;
            if (blockIdx.x == 0) {  // hop 0: the seed itself
                const uint32_t slot = threadIdx.x;
                const uint32_t bit = 1u << (sd & 31);
                atomicOr(P.V + (size_t)slot * P.rs + (sd >> 5), bit);
                P.Fb[(size_t)slot * P.rs + (sd >> 5)] = bit;
                P.cnt[slot] = 1;
                P.mfs[slot] = deg;
                if (s_logbase + slot < P.log_cap)
                    P.logbuf[s_logbase + slot] = ((unsigned long long)slot << 32) | sd;
                else P.ctl->log_overflow = 1;
                // mex gets the seed's in-degree plus (in emit) its discoveries'
                atomicAdd(&P.mex[slot], (unsigned long long)(__ldg(g.cp + sd + 1) - __ldg(g.cp + sd)));
            }
        }
        {
            const uint32_t incl = warp_incl_scan(c);
            if (lane == 31) s_wcount[wib] = incl;
            __syncthreads();
            uint32_t off = 0, tot = 0;
            for (uint32_t i = 0; i < kWarps; ++i) {
                if (i < wib) off += s_wcount[i];
                tot += s_wcount[i];
            }
            if (threadIdx.x < kMaxSlots) s_pref[threadIdx.x] = off + incl - c;
            if (threadIdx.x == 0) s_ntask = tot;
            __syncthreads();
        }
        const uint32_t ntask = s_ntask;
        for (uint32_t t = warp_gid; t < ntask; t += nwarps) {
            uint32_t lo = 0, hi = ns;  // last slot with s_pref <= t
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (s_pref[mid] <= t) lo = mid;
                else hi = mid;
            }
            const uint32_t slot = lo;
            const uint32_t sd = dev_id(g, seed_at(P, slot));
            const uint32_t b = __ldg(g.rp + sd), deg = __ldg(g.rp + sd + 1) - b;
            const uint32_t beg = (t - s_pref[slot]) * kSeedChunk;
            const uint32_t len = min(kSeedChunk, deg - beg);
            uint32_t* vrow = P.V + (size_t)slot * P.rs;
            uint32_t* frow = P.Fb + ((size_t)1 * S + slot) * P.rs;
            for (uint32_t i0 = 0; i0 < len; i0 += 32) {
                const uint32_t i = i0 + lane;
                const uint32_t u = i < len ? __ldg(g.ci + b + beg + i) : sd;
                const bool found = u != sd;
                if (found) {
                    atomicOr(vrow + (u >> 5), 1u << (u & 31));
                    atomicOr(frow + (u >> 5), 1u << (u & 31));
                }
                acc.scanned += i < len;
                acc.found += found;
                stage_push(P, 1, false, s_flag, st, found, slot, u);
            }
        }
        emit(P, 1, false, s_flag, st.buf, st.n);
        st.n = 0;
    }
    // ---- seeds (hop 0): one warp per seed; counters are zero on entry --------------
    for (uint32_t slot = warp_gid; slot < (P.fuse1 ? 0u : ns); slot += nwarps) {
        const uint32_t s = dev_id(g, seed_at(P, slot));
        const uint32_t b = __ldg(g.rp + s), deg = __ldg(g.rp + s + 1) - b;
        if (lane == 0) {
            const uint32_t bit = 1u << (s & 31);
            if (P.seed_visited) P.V[(size_t)slot * P.rs + (s >> 5)] = bit;
            P.Fb[(size_t)slot * P.rs + (s >> 5)] = bit;
            P.cnt[slot] = 1;
            P.mfs[slot] = deg;
            P.mex[slot] = P.seed_visited ? __ldg(g.cp + s + 1) - __ldg(g.cp + s) : 0;
            P.logbuf[slot] = ((unsigned long long)slot << 32) | s;  // log slots [0, ns)
        }
        emit_row_items(P, 0, lane == 0, slot, b, deg);
    }
    if (P.zero_lc)  // the first lc write is after the barrier below
        for (uint32_t i = gtid; i < (MGK_MAX_HOPS + 2) * (sizeof(LevelCounters) / 8); i += nthreads)
            reinterpret_cast<unsigned long long*>(P.lc)[i] = 0;
    if (gtid == 0) {
        P.ctl->found[0] = ns;
        if (!P.fuse1) atomicAdd(&P.ctl->log_n, ns);
    }
    grid_barrier(P.bar);
    if (gtid == 0) atomicAdd(&P.lc[0].ns, globaltimer() - t_init);  // seeds (+ hop 1 if fused)
    if (P.fuse1) {  // hop 1's counters, now that lc is zeroed
        block_flush(acc, &P.ctl->found[1], &P.lc[1]);
        if (blockIdx.x == 0 && threadIdx.x < ns) {
            const uint32_t sd = dev_id(g, seed_at(P, threadIdx.x));
            const uint32_t deg = __ldg(g.rp + sd + 1) - __ldg(g.rp + sd);
            atomicAdd(&P.lc[1].runs, 1u);
            atomicAdd(&P.lc[1].edges, (unsigned long long)deg);
            atomicAdd(&P.lc[1].union_edges, (unsigned long long)deg);
        }
    }

    bool snapped = false;
    uint32_t hop = P.fuse1 ? 2 : 1;
    for (; hop <= P.k; ++hop) {
        const bool last = hop == P.k;
        // ---- plan: per-seed direction (every block computes the same) ------------
        bool pull_me = false;
        if (threadIdx.x < kMaxSlots) {
            uint8_t d = kDead;
            const uint32_t slot = threadIdx.x;
            if (slot < ns) {
                const unsigned long long nf = P.cnt[(hop - 1) * S + slot];
                const unsigned long long mf = P.mfs[(hop - 1) * S + slot];
                const unsigned long long mu = g.m - P.mex[slot];
                const uint8_t prev = P.dirs[((hop - 1) & 1) * S + slot];
                if (nf == 0) {
                    d = kDead;
                } else if (mf & kOverflowBit) {  // the item list overflowed: pull needs no items
                    d = kPull;
                } else if (P.force_dir == 1) {
                    d = kPush;
                } else if (P.force_dir == 2) {
                    d = kPull;
                } else if (prev == kPush) {
                    d = mf * (last ? P.alpha_last : P.alpha) > mu ? kPull : kPush;
                } else {
                    d = nf * P.beta >= g.n ? kPull : kPush;
                }
                if (blockIdx.x == 0) {
                    P.dirs[(hop & 1) * S + slot] = d == kDead ? prev : d;
                    if (d != kDead) {
                        atomicAdd(&P.lc[hop].runs, 1u);
                        if (d == kPull) atomicAdd(&P.lc[hop].pull_runs, 1u);
                        atomicAdd(&P.lc[hop].edges, mf & ~kOverflowBit);
                        atomicAdd(&P.lc[hop].union_edges, mf & ~kOverflowBit);
                    }
                }
            }
            s_dir[slot] = d;
            pull_me = d == kPull;
            // last hop: log the discoveries only if they are bounded by the
            // quota (mf = out-edges of the frontier); otherwise the seed's
            // visited bitmap is cleared densely afterwards
            if (last) {
                const bool logok = slot < ns && (P.keep_result ||
                                                 P.mfs[(hop - 1) * S + slot] <= P.quota);
                s_flag[slot] = logok;
                if (blockIdx.x == 0 && slot < ns && d != kDead && !logok) P.logcnt[slot] = 1;
            }
        }
        compact(pull_me);
        const uint32_t npull = s_nlist;
        if (gtid == 0) P.ctl->nitems[(hop + 2) % 3] = P.ctl->nbig[(hop + 2) % 3] = 0;
        unsigned long long t0 = 0;
        if (gtid == 0) t0 = globaltimer();
        // Frontier bitmaps rotate over 3 buffers and are only cleared at the end:
        // stale bits of F_{h-3} are harmless to pull (an unvisited vertex at hop
        // h has no in-neighbour at distance <= h-2), but k_hop_frontier reads
        // F_k back, so in that mode the buffer of F_{h-2} is cleared here
        // (hop h reads F_{h-1}, writes F_h; the next write is after a barrier).
        if (P.keep_result)
            for (uint32_t w = gtid; w < nw; w += nthreads)
                P.Fb[(size_t)((hop + 1) % 3) * S * P.rs + w] = 0;
        // ---- expand -----------------------------------------------------------------
        push_phase(P, hop, last, s_dir, s_flag, st, acc, warp_gid, nwarps);
        if (npull) pull_phase(P, hop, last, s_list, npull, s_flag, st, acc, warp_gid, nwarps);
        emit(P, hop, last, s_flag, st.buf, st.n);
        st.n = 0;
        block_flush(acc, &P.ctl->found[hop], &P.lc[hop]);
        if (last) {  // the kernel boundary orders the last hop before fr_finish
            if (gtid == 0) P.ctl->t_last = t0;
            ++hop;  // all k hops completed
            break;
        }
        grid_barrier(P.bar);
        if (gtid == 0) atomicAdd(&P.lc[hop].ns, globaltimer() - t0);
        if (ld_volatile(&P.ctl->found[hop]) == 0) break;
        if (P.keep_result && hop + 1 == P.min_hop) {  // visited up to hop min-1
            for (uint32_t w = gtid; w < nw; w += nthreads) P.snap[w] = P.V[w];
            snapped = true;
            grid_barrier(P.bar);
        }
    }
    if (P.keep_result && P.min_hop >= 2 && !snapped)  // stopped before hop min-1: nothing in the window
        for (uint32_t w = gtid; w < nw; w += nthreads) P.snap[w] = P.V[w];
    if (gtid == 0) {
        P.ctl->last_hop = hop > P.k ? P.k : hop;
        P.ctl->last_which = (hop > P.k) ? (P.k % 3) : 3ULL;
    }
}

// Second launch of a group: return the workspace to all-zero and write the
// answers. Every discovery before the last hop is in the log (it may also have
// a frontier bit); last-hop discoveries are logged unless the seed was flagged
// (logcnt[slot] = 1): its last hop only set bits, so its answer is a popcount
// of its visited bitmap, taken while clearing it densely. A log overflow
// clears everything densely. The last CTA to finish writes the answers and
// re-zeroes the per-seed counters and the control block.
constexpr int kFinBlock = 512;
__global__ void __launch_bounds__(kFinBlock) fr_finish(FRParams P) {
    __shared__ uint8_t s_flag[kMaxSlots];
    __shared__ uint16_t s_list[kMaxSlots];
    __shared__ uint32_t s_wcount[kFinBlock / 32];
    __shared__ uint32_t s_nlist;
    __shared__ bool s_last;
    const uint32_t gtid = blockIdx.x * kFinBlock + threadIdx.x;
    const uint32_t nthreads = gridDim.x * kFinBlock;
    const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
    const uint32_t S = P.S, ns = P.ns;
    if (gtid == 0) {
        const unsigned long long now = globaltimer();
        P.ctl->t_clean = now;
        const uint32_t lh = P.ctl->last_hop;
        if (lh == P.k) atomicAdd(&P.lc[lh].ns, now - P.ctl->t_last);
    }
    const bool overflow = ld_volatile(&P.ctl->log_overflow) != 0;
    const uint32_t nlog = min(ld_volatile(&P.ctl->log_n), P.log_cap);
    bool dense_me = false;
    if (threadIdx.x < kMaxSlots) {
        const bool pop_me = threadIdx.x < ns && P.logcnt[threadIdx.x] != 0;
        // a logged seed with many last-hop discoveries: one streamed row of
        // zeros (write-only, full lines) is cheaper than that many scattered
        // single-word stores to lines that have mostly left L2 (break-even
        // measured near nwords / 40 discoveries)
        const bool wide = threadIdx.x < ns && !pop_me && !P.keep_result &&
                          ld_cg(&P.cnt[P.k * S + threadIdx.x]) > P.rs / 32;
        dense_me = threadIdx.x < ns && (overflow || pop_me || wide);
        s_flag[threadIdx.x] = pop_me ? 2 : (dense_me ? 1 : 0);
    }
    {
        const unsigned m = __ballot_sync(kFull, dense_me);
        if (lane == 0) s_wcount[wib] = __popc(m);
        __syncthreads();
        uint32_t off = 0, tot = 0;
        for (uint32_t i = 0; i < kFinBlock / 32; ++i) {
            if (i < wib) off += s_wcount[i];
            tot += s_wcount[i];
        }
        if (dense_me) s_list[off + __popc(m & lanemask_lt())] = (uint16_t)threadIdx.x;
        if (threadIdx.x == 0) s_nlist = tot;
        __syncthreads();
    }
    const uint32_t ndense = s_nlist;
    if (!P.keep_result) {
        if (!overflow) {
            for (uint32_t i = gtid; i < nlog; i += nthreads) {
                const unsigned long long e = P.logbuf[i];
                const uint32_t slot = (uint32_t)(e >> 32) & 0x7FFFFFFFu, w = (uint32_t)e >> 5;
                if (!s_flag[slot]) P.V[(size_t)slot * P.rs + w] = 0;
                if (!(e >> 63))
                    for (int f = 0; f < 3; ++f) P.Fb[((size_t)f * S + slot) * P.rs + w] = 0;
            }
        }
        // dense pass: (slot, 8192-word chunk) tasks; each thread keeps four
        // aligned uint4 loads in flight (rows are padded to 128 B, padding
        // words are always zero)
        constexpr uint32_t kDenseChunk = 4 * 4 * kFinBlock;
        const uint32_t chunks = (P.rs + kDenseChunk - 1) / kDenseChunk;
        for (uint32_t t = blockIdx.x; t < ndense * chunks; t += gridDim.x) {
            const uint32_t slot = s_list[t / chunks];
            const uint32_t base = (t % chunks) * kDenseChunk + threadIdx.x * 4;
            uint4* row = reinterpret_cast<uint4*>(P.V + (size_t)slot * P.rs);
            uint4 v[4];
            const bool count_me = s_flag[slot] == 2;  // the others only need zeros
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t w = base + i * 4 * kFinBlock;
                v[i] = (count_me && w < P.rs) ? __ldcs(row + w / 4) : make_uint4(0, 0, 0, 0);
            }
            uint32_t pc = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t w = base + i * 4 * kFinBlock;
                pc += __popc(v[i].x) + __popc(v[i].y) + __popc(v[i].z) + __popc(v[i].w);
                // a popcounted row is only written where it holds bits (a row
                // of a small seed is almost all zero already); rows cleared
                // without reading them are written whole
                const bool dirty = !count_me || (v[i].x | v[i].y | v[i].z | v[i].w) != 0;
                if (w < P.rs) {
                    if (dirty) __stcs(row + w / 4, make_uint4(0, 0, 0, 0));
                    if (overflow)
                        for (int f = 0; f < 3; ++f)
                            __stcs(reinterpret_cast<uint4*>(P.Fb + ((size_t)f * S + slot) * P.rs + w),
                                   make_uint4(0, 0, 0, 0));
                }
            }
            if (s_flag[slot] == 2) {
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) pc += __shfl_xor_sync(kFull, pc, d);
                if (lane == 0 && pc) atomicAdd(&P.pop[slot], (unsigned long long)pc);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&P.ctl->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (uint32_t slot = threadIdx.x; slot < ns; slot += kFinBlock) {
        // cnt[0] = 1 (the seed frontier); cnt[h] = |F_h| for the hops counted
        // by discovery; a flagged seed's last hop is popcount(V) minus the rest
        unsigned long long before = 0, r = 0;  // discoveries at hops 1..k-1
        for (uint32_t h = 1; h < P.k; ++h) {
            const unsigned long long c = ld_cg(&P.cnt[h * S + slot]);
            before += c;
            if (h >= P.min_hop) r += c;
        }
        unsigned long long lastc = ld_cg(&P.cnt[P.k * S + slot]);
        if (ld_cg(&P.logcnt[slot]) != 0) lastc = ld_cg(&P.pop[slot]) - before - P.seed_visited;
        if (P.k >= P.min_hop) r += lastc;
        P.counts[slot] = r;
        for (uint32_t h = 0; h <= P.k; ++h) {
            P.cnt[h * S + slot] = 0;
            P.mfs[h * S + slot] = 0;
        }
        P.logcnt[slot] = 0;
        P.pop[slot] = 0;
        P.mex[slot] = 0;
        P.dirs[slot] = P.dirs[S + slot] = kPush;
    }
    if (threadIdx.x == 0) {
        P.ctl->nitems[0] = P.ctl->nitems[1] = P.ctl->nitems[2] = 0;
        P.ctl->nbig[0] = P.ctl->nbig[1] = P.ctl->nbig[2] = 0;
        P.ctl->log_n = 0;
        P.ctl->log_overflow = 0;
        for (uint32_t h = 0; h <= P.k; ++h) P.ctl->found[h] = 0;
        P.ctl->done = 0;
        atomicAdd(&P.lc[MGK_MAX_HOPS + 1].ns, globaltimer() - ld_cg(&P.ctl->t_clean));
    }
}

// Clears slot 0's bitmaps after a k_hop_frontier readback.
__global__ void clear_slot0(uint32_t* V, uint32_t* Fb, uint32_t S, uint32_t nw, uint32_t rs) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += gridDim.x * blockDim.x) {
        V[w] = 0;
        for (int f = 0; f < 3; ++f) Fb[(size_t)f * S * rs + w] = 0;
    }
}

// `drop` is an external id (mapped to its device id here); ~0 = none
__global__ void popc_words(const uint32_t* bits, const uint32_t* sub, uint32_t nwords, uint32_t drop,
                           const uint32_t* perm, uint32_t* out) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwords) return;
    if (perm && drop != 0xFFFFFFFFu) drop = perm[drop];
    uint32_t x = bits[w] & (sub ? ~sub[w] : kFull);
    if ((drop >> 5) == w) x &= ~(1u << (drop & 31));
    out[w] = __popc(x);
}

__global__ void scatter_ids(const uint32_t* bits, const uint32_t* sub, uint32_t nwords, uint32_t drop,
                            const uint32_t* perm, const uint32_t* offs, unsigned long long* ids) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nwords) return;
    if (perm && drop != 0xFFFFFFFFu) drop = perm[drop];
    uint32_t x = bits[w] & (sub ? ~sub[w] : kFull);
    if ((drop >> 5) == w) x &= ~(1u << (drop & 31));
    uint32_t o = offs[w];
    while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        ids[o++] = (unsigned long long)w * 32 + b;
    }
}

uint32_t row_stride(const DevGraph& g) { return (g.nwords + 31) & ~31u; }

uint32_t slots_for(const DevGraph& g) {
    const uint64_t per_slot = 4ull * row_stride(g) * 4;
    const uint64_t budget = 4ull << 30;
    return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(kMaxSlots, budget / per_slot));
}

}  // namespace

cudaError_t ensure_single_ws(const Graph* gr, Workspace* ws) {
    if (ws->fr_V) return cudaSuccess;
    const DevGraph& g = gr->dg;
    const uint32_t S = slots_for(g);
    const size_t bm = (size_t)S * row_stride(g) * 4 + 64;
    cudaError_t e;
    if ((e = cudaMalloc(&ws->fr_V, bm))) return e;
    if ((e = cudaMalloc(&ws->fr_Fb, 3 * bm))) return e;
    if ((e = cudaMemset(ws->fr_V, 0, bm))) return e;
    if ((e = cudaMemset(ws->fr_Fb, 0, 3 * bm))) return e;
    const uint64_t want_items = (uint64_t)S * (g.m / kChunk + g.n) + 1024;
    ws->fr_items_cap = (uint32_t)std::min<uint64_t>(want_items, 64ull << 20);
    for (int i = 0; i < 2; ++i)
        if ((e = cudaMalloc(&ws->fr_items[i], (size_t)ws->fr_items_cap * sizeof(uint2)))) return e;
    const uint64_t want_big = (uint64_t)S * (g.m / kBigChunk + 64) + 1024;
    ws->fr_big_cap = (uint32_t)std::min<uint64_t>(want_big, 16ull << 20);
    for (int i = 0; i < 2; ++i)
        if ((e = cudaMalloc(&ws->fr_big[i], (size_t)ws->fr_big_cap * sizeof(uint2)))) return e;
    // a last hop that can touch more than ~nwords/256 vertices of a seed is
    // not logged (fire-and-forget red.or); its visited bitmap is popcounted
    // and cleared with one coalesced pass instead. Sweep of the divisor (cfg2
    // k=2 call on G2 / cfg4 k=2 on G4): 16 -> 0.179 / 1.51 ms, 64 -> 0.173 /
    // 1.39, 256 -> 0.169 / 1.41, 1024 -> 0.169 / 1.44
    uint32_t qdiv = 256;
    if (const char* q = std::getenv("MGK_QUOTA_DIV")) qdiv = std::max(1, std::atoi(q));
    ws->fr_quota = std::max<uint32_t>(64, g.nwords / qdiv);
    ws->fr_log_cap = (uint32_t)std::min<uint64_t>((uint64_t)S * (g.n + 64), 64ull << 20);
    if ((e = cudaMalloc(&ws->fr_log, (size_t)ws->fr_log_cap * 8))) return e;
    const size_t cs = (size_t)(MGK_MAX_HOPS + 1) * S;
    if ((e = cudaMalloc(&ws->fr_cnt, cs * 4))) return e;
    if ((e = cudaMalloc(&ws->fr_mfs, cs * 8))) return e;
    if ((e = cudaMalloc(&ws->fr_mus, (size_t)S * 8))) return e;
    // per-seed counters and the control block are all-zero between launches
    // (each launch re-zeroes what it used), so a launch needs no init phase
    if ((e = cudaMemset(ws->fr_mus, 0, (size_t)S * 8))) return e;
    if ((e = cudaMalloc(&ws->fr_logcnt, (size_t)S * 4))) return e;
    if ((e = cudaMalloc(&ws->fr_pop, (size_t)S * 8))) return e;
    if ((e = cudaMemset(ws->fr_pop, 0, (size_t)S * 8))) return e;
    if ((e = cudaMalloc(&ws->fr_dirs, (size_t)2 * S))) return e;
    if ((e = cudaMalloc(&ws->fr_ctl, sizeof(FRCtl)))) return e;
    if ((e = cudaMalloc(&ws->fr_snap, (size_t)row_stride(g) * 4))) return e;
    if ((e = cudaMemset(ws->fr_cnt, 0, cs * 4))) return e;
    if ((e = cudaMemset(ws->fr_mfs, 0, cs * 8))) return e;
    if ((e = cudaMemset(ws->fr_logcnt, 0, (size_t)S * 4))) return e;
    if ((e = cudaMemset(ws->fr_dirs, 0, (size_t)2 * S))) return e;
    if ((e = cudaMemset(ws->fr_ctl, 0, sizeof(FRCtl)))) return e;
    ws->fr_slots = S;
    ws->bytes += 2 * (size_t)ws->fr_big_cap * 8;
    ws->bytes += 4 * bm + 2 * (size_t)ws->fr_items_cap * 8 + (size_t)ws->fr_log_cap * 8 + cs * 12 +
                 (size_t)S * 14 + sizeof(FRCtl);
    // the memsets above run on the legacy stream, which does not order work on
    // the non-blocking streams the engines launch on: the zero state must be
    // complete before the first traversal (recycled allocations are not zero)
    return cudaStreamSynchronize(0);
}

// k = 1 on duplicate-free rows: |F_1| = deg(s) - [s in row(s)]. One warp per
// seed finds s in its ascending row with a 32-way search (32 pivots per round:
// a 100K-entry hub row takes 3 dependent loads instead of 17). No bitmap is
// touched, so there is nothing to clean up. The last CTA (done counter in
// misc[7]) folds the per-CTA sums into the per-hop counters; misc[3..7] are
// zero on entry and on exit.
constexpr int kK1Block = 512;
__global__ void __launch_bounds__(kK1Block) k1_kernel(DevGraph g, const uint32_t* seeds, uint64_t ns,
                                                      unsigned long long* counts, LevelCounters* lc,
                                                      unsigned long long* misc) {
    __shared__ unsigned long long s_acc[3];
    __shared__ bool s_last;
    const unsigned long long t0 = globaltimer();
    if (blockIdx.x == 0 && threadIdx.x == 0) misc[3] = t0;
    if (threadIdx.x < 3) s_acc[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t lane = lane_id();
    const uint64_t nwarps = (uint64_t)gridDim.x * (kK1Block / 32);
    unsigned long long f = 0, sc = 0, nrun = 0;
    for (uint64_t i = (blockIdx.x * (uint64_t)kK1Block + threadIdx.x) >> 5; i < ns; i += nwarps) {
        const uint32_t sd = dev_id(g, seeds[i]);
        const uint32_t b = __ldg(g.rp + sd), e = __ldg(g.rp + sd + 1);
        uint32_t lo = b, hi = e;  // sd, if present, is in [lo, hi)
        while (hi - lo > 32) {
            const uint32_t piv = lo + (uint32_t)((uint64_t)(hi - lo) * (lane + 1) / 33);
            const unsigned below = __ballot_sync(kFull, __ldg(g.ci + piv) < sd);
            const int c = __popc(below);  // pivots ascend: `below` is a prefix
            const uint32_t nlo = c == 0 ? lo : __shfl_sync(kFull, piv, c - 1) + 1;
            const uint32_t nhi = c == 32 ? hi : __shfl_sync(kFull, piv, c) + 1;
            lo = nlo;
            hi = nhi;
        }
        const bool hit = lo + lane < hi && __ldg(g.ci + lo + lane) == sd;
        const uint32_t self = __ballot_sync(kFull, hit) ? 1u : 0u;
        if (lane == 0) {
            const uint32_t c = e - b - self;
            counts[i] = c;
            f += c;
            sc += e - b;
            nrun += 1;
        }
    }
    if (lane == 0) {
        if (f) atomicAdd(&s_acc[0], f);
        if (sc) atomicAdd(&s_acc[1], sc);
        if (nrun) atomicAdd(&s_acc[2], nrun);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_acc[0]) atomicAdd(&misc[4], s_acc[0]);
        if (s_acc[1]) atomicAdd(&misc[5], s_acc[1]);
        if (s_acc[2]) atomicAdd(&misc[6], s_acc[2]);
        __threadfence();
        s_last = atomicAdd(&misc[7], 1ull) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (uint32_t i = threadIdx.x; i < (MGK_MAX_HOPS + 2) * (sizeof(LevelCounters) / 8); i += blockDim.x)
        reinterpret_cast<unsigned long long*>(lc)[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long fr = ld_cg(&misc[4]), scn = ld_cg(&misc[5]), runs = ld_cg(&misc[6]);
        lc[1].frontier = lc[1].vertices = fr;
        lc[1].scanned = lc[1].edges = lc[1].union_edges = scn;
        lc[1].runs = (unsigned)runs;
        lc[1].ns = globaltimer() - ld_cg(&misc[3]);
        misc[3] = misc[4] = misc[5] = misc[6] = misc[7] = 0;
    }
}

bool fuse_disabled() {
    static const bool off = std::getenv("MGK_NO_FUSE1") != nullptr;
    return off;
}

cudaError_t launch_single(Launch& L) {
    const Graph* gr = L.g;
    Workspace* ws = L.ws;
    if (k2_eligible(L)) return launch_k2(L);
    if (gr->dg.rows_unique && L.k == 1 && L.seed_visited && !L.keep_result && !fuse_disabled()) {
        const uint64_t want = (L.nseeds + kK1Block / 32 - 1) / (kK1Block / 32);  // a warp per seed
        const uint32_t grid = (uint32_t)std::min<uint64_t>(want, 148ull * 4);
        k1_kernel<<<grid, kK1Block, 0, L.stream>>>(gr->dg, L.d_seeds, L.nseeds, L.d_counts, ws->lc, ws->misc);
        L.grid = grid;
        L.block = kK1Block;
        L.launches = 1;
        return cudaGetLastError();
    }
    cudaError_t e = ensure_single_ws(gr, ws);
    if (e) return e;
    static int blocks_per_sm = 0, num_sms = 0;
    if (blocks_per_sm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, fr_kernel, kBlock, 0)))
            return e;
        if (blocks_per_sm < 1) return cudaErrorInvalidConfiguration;
    }
    static int fin_blocks = 0;
    if (fin_blocks == 0) {
        int per_sm = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fr_finish, kFinBlock, 0))) return e;
        fin_blocks = std::max(1, per_sm) * num_sms;
    }
    FRParams P;
    P.g = gr->dg;
    P.k = L.k;
    P.min_hop = L.min_hop;
    P.seed_visited = L.seed_visited;
    P.V = ws->fr_V;
    P.Fb = ws->fr_Fb;
    P.items0 = ws->fr_items[0];
    P.items1 = ws->fr_items[1];
    P.items_cap = ws->fr_items_cap;
    P.big0 = ws->fr_big[0];
    P.big1 = ws->fr_big[1];
    P.big_cap = ws->fr_big_cap;
    P.logbuf = ws->fr_log;
    P.log_cap = ws->fr_log_cap;
    P.cnt = ws->fr_cnt;
    P.mfs = ws->fr_mfs;
    P.mex = ws->fr_mus;
    P.logcnt = ws->fr_logcnt;
    P.pop = ws->fr_pop;
    P.dirs = ws->fr_dirs;
    P.ctl = reinterpret_cast<FRCtl*>(ws->fr_ctl);
    P.lc = ws->lc;
    P.bar = reinterpret_cast<unsigned int*>(ws->misc + 8);
    P.alpha = L.tuning.alpha;
    P.beta = L.tuning.beta;
    P.force_dir = L.tuning.force_dir;
    P.alpha_last = L.tuning.alpha_last;
    P.quota = ws->fr_quota;
    P.keep_result = L.keep_result ? 1u : 0u;
    P.fuse1 = (gr->dg.rows_unique && L.seed_visited && L.k >= 2 && !L.keep_result && !fuse_disabled())
                  ? 1u : 0u;
    P.snap = ws->fr_snap;
    // bitmaps are laid out [S_alloc][rs] ([3][S_alloc][rs] for Fb): S is the
    // allocated slot count (the stride); a group holds up to S seeds
    P.S = ws->fr_slots;
    P.rs = row_stride(gr->dg);
    L.grid = (uint32_t)(blocks_per_sm * num_sms);
    L.block = kBlock;
    // one group of up to S seeds per (traverse, finish) launch pair
    for (uint64_t g0 = 0; g0 < L.nseeds; g0 += P.S) {
        P.ns = (uint32_t)std::min<uint64_t>(P.S, L.nseeds - g0);
        P.zero_lc = g0 == 0;
        if (L.host_io) {  // this group's seeds ride in the launch parameters
            P.seeds = nullptr;
            std::memcpy(P.inline_seeds, L.h_seeds + g0, (size_t)P.ns * 4);
        } else {
            P.seeds = L.d_seeds + g0;
        }
        P.counts = L.d_counts + g0;
        void* args[] = {&P};
        if ((e = launch_persistent((const void*)fr_kernel, L.grid, kBlock, args, L.stream))) return e;
        fr_finish<<<fin_blocks, kFinBlock, 0, L.stream>>>(P);
        if ((e = cudaGetLastError())) return e;
        L.launches += 2;
    }
    return cudaSuccess;
}

cudaError_t single_result_ids(const Graph* gr, Workspace* ws, uint32_t min_hop, bool seed_visited,
                              uint32_t seed, unsigned long long* d_ids, unsigned long long* d_n,
                              cudaStream_t s) {
    const DevGraph& g = gr->dg;
    const uint32_t nw = g.nwords;
    // window [min_hop, k] = visited \ visited-after-hop-(min_hop - 1); for
    // min_hop = 1 that is visited minus the pre-visited seed (if any)
    const uint32_t* sub = min_hop >= 2 ? ws->fr_snap : nullptr;
    const uint32_t drop = (min_hop < 2 && seed_visited) ? seed : 0xFFFFFFFFu;
    uint32_t* offs = nullptr;
    cudaError_t e;
    if ((e = cudaMallocAsync(&offs, (size_t)(nw + 1) * 4, s))) return e;
    const int tb = 256, nb = (int)((nw + tb - 1) / tb);
    popc_words<<<nb, tb, 0, s>>>(ws->fr_V, sub, nw, drop, g.perm, offs);
    if ((e = exclusive_scan_u32(offs, nw, d_n, s))) return e;
    scatter_ids<<<nb, tb, 0, s>>>(ws->fr_V, sub, nw, drop, g.perm, offs, d_ids);
    cudaFreeAsync(offs, s);
    clear_slot0<<<148, 256, 0, s>>>(ws->fr_V, ws->fr_Fb, ws->fr_slots, nw, row_stride(g));
    return cudaGetLastError();
}

}  // namespace mgk
