// SINGLE engine, 2-hop counts with the visited set in SHARED memory.
//
// For k = 2 on duplicate-free rows (k_hop_count exact / cumulative,
// proj/core/src/execute.cpp:347-375) the answer of seed s is a set size:
//   B(s) = {s} u F1 u N(F1),  F1 = row(s) \ {s}
//   exact |F2| = |B| - 1 - |F1|,  cumulative |F1 u F2| = |B| - 1
// (the masked vxm of hop 2, sparse.cpp:253-290, unioned with visited);
// walk_targets windows [1, 2] / [2, 2] are the same set without the seed bit
// (execute.cpp:43-60). The general engine (mgk_ss.cu) builds B in a per-seed
// bitmap in L2 with one red.or per adjacency entry, at the L2 atomic ceiling
// (~200 G/s on this B200). Shared-memory atomics on a random word run at
// ~777 G/s over the chip (scripts/ubench_smem.cu; DSMEM atomics across a
// cluster only at ~185 G/s), so here B lives on chip: the vertex range is cut
// into R slices of at most ~175 KB of bits, and R CTAs ("a group", one
// 768-thread CTA per SM) hold one slice of one seed's B each. Rows ascend, so
// a per-vertex array of slice crossings lets each CTA stream only its part of
// every F1 row: each adjacency entry is read once, by the CTA owning its
// target.
//
// One persistent cooperative launch:
//   0a. warp per seed: reserve its F1 rows, window totals and 32-row tasks
//   0b. tasks: each F1 row's vertex, row begin, length and slice crossings;
//       per seed w(s) = sum of deg(F1)                            (barrier)
//   1. every CTA: the "work line" (w + a per-seed cost, scanned) and its
//      group's equal slice of it; boundaries near a seed edge snap to it
//   2. per seed part: window prefixes in shared memory, a flat entry stream
//      per warp (16 loads in flight per lane), red.shared.or into the slice;
//      a whole seed is popcounted on chip, a seed cut by a group boundary
//      stages its slice (coalesced); the next seed's record and first window
//      arrive by cp.async during the sweep                         (barrier)
//   3. cut seeds: OR of their staged slices, popcounted by all CTAs (barrier)
//   4. answers (+ the k = 1 answers of a fused section), accumulators reset
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "mgk_device.cuh"

namespace mgk {
namespace {

using namespace dev;

#ifndef MGK_K2_BLOCK
#define MGK_K2_BLOCK 768  // 80 registers, no spills (1024 threads spilled at 64)
#endif
#ifndef MGK_K2_MINB
#define MGK_K2_MINB 1  // CTAs per SM the register budget is sized for
#endif
constexpr int kK2Block = MGK_K2_BLOCK;
constexpr int kK2Warps = kK2Block / 32;
constexpr uint32_t kK2Win = 2 * kK2Block;  // F1 rows per prefix window (2 per thread)
constexpr uint32_t kK2Task = 32;   // F1 rows per phase-0 task (1 per lane)
constexpr uint32_t kK2Inline = 512;
constexpr uint32_t kK2MaxR = 64;  // slices per seed (G4: 26, so 5 groups)
constexpr uint32_t kNoF1 = 0xFFFFFFFFu;
constexpr int kK2Ilp = 16;  // adjacency entries in flight per lane
// smem besides the bitmap: the window's slice and combined prefixes, each row's
// slice start, the row cursors, and scratch
constexpr uint32_t kK2Stg = 512;  // rows of the next seed's first window staged during a sweep
constexpr uint32_t kK2Fixed = 2 * (kK2Win + 2) * 4 + kK2Win * 4 + kK2Win * 8 + 4 * kK2Stg * 4 + 1024;

struct K2Params {
    DevGraph g;
    const uint32_t* seeds;  // nullptr: inline_seeds
    uint64_t ns;
    unsigned long long* counts;
    unsigned long long* counts1;  // optional: the same seeds' k = 1 answers (|F1|)
    uint32_t cumulative;  // window starts at hop 1 (k_hop cumulative; walks [1, 2])
    uint32_t walk;        // walk_targets: the visited set starts empty (no seed bit; s in F1 if a self loop)
    uint32_t R;       // vertex slices per seed (CTAs per group)
    uint32_t rbits;   // vertices per slice (multiple of 128)
    uint32_t rwords;  // rbits / 32
    uint32_t ngroups;
    unsigned long long* w;    // [ns + 1] hop-2 entries per seed -> the work line (scanned)
    unsigned long long* acc;  // [ns] popcounts (zero between launches)
    uint32_t* f1;             // [ns] |F1|
    uint32_t* stage;          // [ngroups][2][R][rwords]
    LevelCounters* lc;
    unsigned int* bar;
    // [0..2] timestamps, [4] cut seeds, [5..7] allocators of the F1 rows, the
    // window totals and the phase-0 tasks (zero between launches)
    unsigned long long* misc;
    unsigned long long* bounds;  // [ngroups + 1] group slices of the work line
    uint32_t* first;             // [ngroups] first seed of each group
    uint4* cuts;                 // [ngroups] {seed, first group, last group, 0} of the cut seeds
    // the seeds' F1 rows (phase 0): vertex, CSR row begin, length (0 for the
    // seed itself); per seed its first row (kNoF1: scratch ran out) and its
    // first window total (windows of kK2Win rows)
    uint4* sinfo;     // [ns] {device seed id, CSR row begin, degree, first F1 row or kNoF1}
    uint32_t* f1win;  // [ns]
    uint32_t* f1v;
    uint32_t* f1rb;
    uint32_t* f1d;
    uint32_t* f1sp;         // [f1cap][R-1] where each F1 row enters slices 1..R-1 (offsets in the row)
    const uint32_t* split;  // graph: [n][R-1] absolute positions of the same
    uint64_t f1cap;
    unsigned long long* wt;  // window totals
    uint64_t wtcap;
    uint4* tasks;            // {seed, CSR position of the block, output position, window total slot}
    uint64_t taskcap;
    unsigned long long seedcost;  // work-line units charged per seed (its fixed cost)
    uint32_t snapdiv;
    uint32_t diag;  // MGK_K2_DIAG=1: phase timings in level 0 of the stats  // group boundaries within (group size / snapdiv) of a seed edge move to it
    uint32_t inline_seeds[kK2Inline];
};

__device__ __forceinline__ uint32_t k2_seed(const K2Params& P, uint64_t i) {
    return dev_id(P.g, P.seeds ? P.seeds[i] : P.inline_seeds[i]);
}

// first offset of group g on the work line [0, W): floor(W * g / G) without
// a 128-bit product (W = q G + r)
__device__ __forceinline__ unsigned long long group_lo(unsigned long long W, uint32_t g, uint32_t G) {
    return (W / G) * g + (W % G) * g / G;
}
// the same with W / G and W % G precomputed (r g < G^2 fits 32 bits)
struct GroupLine {
    unsigned long long q;
    uint32_t r, G;
    __device__ __forceinline__ unsigned long long lo(uint32_t g) const { return q * g + (r * g) / G; }
};

// block-wide exclusive scan of one u64 per thread; returns the block total
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v, unsigned long long* out,
                                                              unsigned long long* s_warp) {
    const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long t = __shfl_up_sync(kFull, x, d);
        if (lane >= (uint32_t)d) x += t;
    }
    if (lane == 31) s_warp[wib] = x;
    __syncthreads();
    if (wib == 0) {
        unsigned long long y = s_warp[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long t = __shfl_up_sync(kFull, y, d);
            if (lane >= (uint32_t)d) y += t;
        }
        s_warp[lane] = y;  // inclusive warp totals
    }
    __syncthreads();
    const unsigned long long before = wib ? s_warp[wib - 1] : 0;
    *out = before + x - v;
    const unsigned long long total = s_warp[kK2Warps - 1];
    __syncthreads();
    return total;
}

// one row-cursor step (asm volatile: the load stays inside the cursor loop
// instead of being re-issued after it for every entry)
__device__ __forceinline__ void ld_rinfo(uint32_t base, uint32_t t, uint32_t& nxt, uint32_t& dl) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(nxt), "=r"(dl) : "r"(base + t * 8));
}

// asynchronous global -> shared copies (nothing held in registers meanwhile)
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void smem_or(uint32_t base, uint32_t word, uint32_t bit) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(base + word * 4), "r"(bit));
}

// Where each row crosses the slice boundaries r * rbits (rows ascend): the
// CTA holding slice r streams only [split r-1, split r) of every F1 row.
__global__ void k2_split_kernel(DevGraph g, uint32_t R, uint32_t rbits, uint32_t* out) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x) {
        const uint32_t b = g.rp[v], e = g.rp[v + 1];
        for (uint32_t r = 1; r < R; ++r) {
            const uint32_t bound = r * rbits;
            uint32_t lo = b, hi = e;  // first position with col >= bound
            while (lo < hi) {
                const uint32_t mid = lo + (hi - lo) / 2;
                if (g.ci[mid] < bound) lo = mid + 1; else hi = mid;
            }
            out[(size_t)v * (R - 1) + r - 1] = lo;
        }
    }
}

__global__ void __launch_bounds__(kK2Block, MGK_K2_MINB) k2_kernel(K2Params P) {
    extern __shared__ __align__(16) unsigned char k2_smem[];
    grid_barrier_init(P.bar);
    uint32_t* bm = reinterpret_cast<uint32_t*>(k2_smem);
    // window prefix of the row lengths, relative to the window start (a window's
    // rows are distinct vertices, so its total is <= m < 2^32)
    // pre: the window's prefix of this slice's row lengths; prec: of the whole
    // rows (the work line's unit); srow: where each row enters this slice
    uint32_t* pre = reinterpret_cast<uint32_t*>(k2_smem + (size_t)P.rwords * 4);
    uint32_t* prec = pre + kK2Win + 2;
    uint32_t* srow = prec + kK2Win + 2;
    // rinfo[t] = {pre[t + 1], (row start + srow[t]) - pre[t]}: one 64-bit load
    // advances a row cursor (slice entry x lives at col_idx[x + rinfo[t].y])
    uint2* rinfo = reinterpret_cast<uint2*>(srow + kK2Win);
    // the next seed's first window, copied in (cp.async) during this seed's sweep
    uint32_t* stg = reinterpret_cast<uint32_t*>(rinfo + kK2Win);  // [4][kK2Stg]: rb, d, split, v
    unsigned long long* s_warp = reinterpret_cast<unsigned long long*>(stg + 4 * kK2Stg);  // [32]
    unsigned long long* s_misc = s_warp + 32;                                         // [8]
    const DevGraph& g = P.g;
    const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
    const uint32_t nthreads = gridDim.x * kK2Block;
    const uint32_t gtid = blockIdx.x * kK2Block + threadIdx.x;
    const uint64_t nwarps = (uint64_t)gridDim.x * kK2Warps;
    const uint64_t gwarp = (uint64_t)blockIdx.x * kK2Warps + wib;
    const uint32_t bm_base = (uint32_t)__cvta_generic_to_shared(bm);
    const unsigned long long t0 = globaltimer();

    // ---- phase 0a: per seed, reserve its F1 rows, window totals and tasks -----------
    for (uint32_t i = threadIdx.x; i < P.rwords; i += kK2Block) bm[i] = 0;
    if (blockIdx.x == 0)
        for (uint32_t i = threadIdx.x; i < (MGK_MAX_HOPS + 2) * (sizeof(LevelCounters) / 8); i += kK2Block)
            reinterpret_cast<unsigned long long*>(P.lc)[i] = 0;
    for (uint64_t i = gwarp; i < P.ns; i += nwarps) {
        const uint32_t s = k2_seed(P, i);
        const uint32_t b = __ldg(g.rp + s), deg = __ldg(g.rp + s + 1) - b;
        const uint32_t nwin = (deg + kK2Win - 1) / kK2Win, nt = (deg + kK2Task - 1) / kK2Task;
        unsigned long long off = 0, ow = 0, ot = 0;
        if (lane == 0) {
            off = atomicAdd(&P.misc[5], (unsigned long long)deg);
            ow = atomicAdd(&P.misc[6], (unsigned long long)nwin);
            ot = atomicAdd(&P.misc[7], (unsigned long long)nt);
        }
        off = __shfl_sync(kFull, off, 0);
        ow = __shfl_sync(kFull, ow, 0);
        ot = __shfl_sync(kFull, ot, 0);
        const bool ok = off + deg <= P.f1cap && ow + nwin <= P.wtcap && ot + nt <= P.taskcap;
        for (uint32_t q = lane; q < nt; q += 32)
            if (ot + q < P.taskcap)
                P.tasks[ot + q] = make_uint4(ok ? (uint32_t)i : kNoF1, b + q * kK2Task, (uint32_t)off + q * kK2Task,
                                             (uint32_t)ow + q * kK2Task / kK2Win);
        if (lane == 0) P.sinfo[i] = make_uint4(s, b, deg, ok ? (uint32_t)off : kNoF1);
        if (ok) {
            for (uint32_t q = lane; q < nwin; q += 32) P.wt[ow + q] = 0;
            if (lane == 0) {
                P.f1win[i] = (uint32_t)ow;
                P.w[i] = 0;
                P.f1[i] = 0;
            }
        } else {  // scratch exhausted (huge batches of hubs): this warp sums the rows itself
            unsigned long long wsum = 0;
            uint32_t nf = 0;
            for (uint32_t j = b + lane; j < b + deg; j += 32) {
                const uint32_t v = __ldg(g.ci + j);
                if (v != s || P.walk) {
                    wsum += __ldg(g.rp + v + 1) - __ldg(g.rp + v);
                    ++nf;
                }
            }
            wsum = warp_sum_u64(wsum);
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) nf += __shfl_xor_sync(kFull, nf, d);
            if (lane == 0) {
                P.w[i] = wsum;
                P.f1[i] = nf;
            }
        }
    }
    grid_barrier(P.bar);
    if (gtid == 0) P.misc[8] = globaltimer();

    // ---- phase 0b: tasks of 256 F1 rows: vertex, row begin, row length --------------
    {
        const uint64_t ntask = min(ld_cg(&P.misc[7]), (unsigned long long)P.taskcap);
        for (uint64_t t = gwarp; t < ntask; t += nwarps) {
            const uint4 tk = __ldcg(P.tasks + t);
            if (tk.x == kNoF1) continue;
            // the block's entries and the seed's record load together (the
            // entries are clamped to col_idx and masked once deg is known)
            uint32_t v[kK2Task / 32], rb[kK2Task / 32], re[kK2Task / 32], sp1[kK2Task / 32];
#pragma unroll
            for (int r = 0; r < (int)(kK2Task / 32); ++r)
                v[r] = __ldg(g.ci + min((unsigned long long)tk.y + lane + 32 * r, (unsigned long long)g.m - 1));
            const uint4 si = __ldcg(P.sinfo + tk.x);
            const uint32_t s = si.x, b = si.y, deg = si.z;
            const uint32_t j0 = tk.y - b, off = tk.z - j0;
#pragma unroll
            for (int r = 0; r < (int)(kK2Task / 32); ++r)
                if (j0 + lane + 32 * r >= deg) v[r] = s;
#pragma unroll
            for (int r = 0; r < (int)(kK2Task / 32); ++r) {
                rb[r] = __ldg(g.rp + v[r]);
                re[r] = __ldg(g.rp + v[r] + 1);
                // R = 2 (the usual case): the one split, loaded with the row bounds
                sp1[r] = P.R == 2 ? __ldg(P.split + v[r]) : 0;
            }
            unsigned long long sum = 0;
            uint32_t nf = 0;
#pragma unroll
            for (int r = 0; r < (int)(kK2Task / 32); ++r) {
                const uint32_t j = j0 + lane + 32 * r;
                const bool in_f1 = v[r] != s || P.walk;
                const uint32_t d = in_f1 ? re[r] - rb[r] : 0;
                if (j < deg) {
                    P.f1v[off + j] = v[r];
                    P.f1rb[off + j] = rb[r];
                    P.f1d[off + j] = d;
                    // R = 2: the one split per row; R > 2 reads the graph's
                    // split array in phase 2 (R - 1 words per row would not pay)
                    if (P.R == 2) P.f1sp[off + j] = in_f1 ? sp1[r] - rb[r] : 0;
                    sum += d;
                    nf += in_f1;
                }
            }
            sum = warp_sum_u64(sum);
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) nf += __shfl_xor_sync(kFull, nf, d);
            if (lane == 0) {
                if (sum) {
                    atomicAdd(&P.w[tk.x], sum);
                    atomicAdd(&P.wt[tk.w], sum);
                }
                if (nf) atomicAdd(&P.f1[tk.x], nf);
            }
        }
    }
    grid_barrier(P.bar);

    if (gtid == 0) P.misc[9] = globaltimer();
    // ---- phase 1 (every CTA, no barrier after it): the work line (w + seedcost
    // per seed with work), this CTA's group slice and its first seed. Thread t
    // owns a chunk of seeds and finds the group boundaries inside them
    // arithmetically. CTA 0 also records every boundary and the cut seeds for
    // the merge (read after the next grid barrier)
    const uint32_t G = P.ngroups, R = P.R;
    const uint32_t grp = blockIdx.x / R, rr = blockIdx.x % R;
    unsigned long long W;
    {
        unsigned long long* s_b = s_misc;  // [0] group start, [1] group end, [2] first seed, [3] its ws
        unsigned int* s_ncut = reinterpret_cast<unsigned int*>(s_misc + 4);
        const uint64_t per = (P.ns + kK2Block - 1) / kK2Block;
        const uint64_t i0 = min((uint64_t)threadIdx.x * per, P.ns), i1 = min(i0 + per, P.ns);
        unsigned long long part = 0;
        for (uint64_t i = i0; i < i1; ++i) {
            const unsigned long long v = ld_cg(P.w + i);
            part += v ? v + P.seedcost : 0;
        }
        unsigned long long base;
        const unsigned long long total = block_excl_scan(part, &base, s_warp);
        W = total;
        if (threadIdx.x == 0) *s_ncut = 0;
        const unsigned long long snap = total / G / P.snapdiv;
        const GroupLine gl{total / G, (uint32_t)(total % G), G};
        // boundaries no seed holds (the end of the work line)
        if (threadIdx.x < 2 && gl.lo(grp + threadIdx.x) >= total) {
            s_b[threadIdx.x] = total;
            if (threadIdx.x == 0) s_b[2] = P.ns;
        }
        if (blockIdx.x == 0)
            for (uint32_t t = threadIdx.x; t <= G; t += kK2Block)
                if (gl.lo(t) >= total) P.bounds[t] = total;
        __syncthreads();
        // smallest b in [0, G] with group_lo(b) >= x; group_lo(G) = total
        auto first_group = [&](unsigned long long x) {
            uint32_t lo = 0, hi = G;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) / 2;
                if (gl.lo(mid) >= x) hi = mid; else lo = mid + 1;
            }
            return lo;
        };
        for (uint64_t i = i0; i < i1; ++i) {
            const unsigned long long v0 = ld_cg(P.w + i);
            const unsigned long long v = v0 ? v0 + P.seedcost : 0, ws = base, we = base + v;
            base = we;
            if (v == 0) continue;
            const uint32_t b0 = first_group(ws), bB = first_group(we);
            // a boundary within `snap` of a seed edge moves to that edge: the
            // seed is not cut there (no staged slices, no merge) at the price of
            // groups that differ in size by up to 2 snap
            bool cut = false;
            uint32_t bfirst = 0, blast = 0;
            for (uint32_t bb = b0; bb < bB && bb < G; ++bb) {
                const unsigned long long x = gl.lo(bb);
                const bool to_start = x - ws <= snap, to_end = !to_start && we - x <= snap;
                const unsigned long long bnd = to_start ? ws : (to_end ? we : x);
                const uint32_t fs = (uint32_t)i + (to_end ? 1u : 0u);
                if (bb == grp) {
                    s_b[0] = bnd;
                    s_b[2] = fs;
                    s_b[3] = to_end ? we : ws;
                }
                if (bb == grp + 1) s_b[1] = bnd;
                if (blockIdx.x == 0) {
                    P.bounds[bb] = bnd;
                    P.first[bb] = fs;
                }
                if (!to_start && !to_end) {
                    if (!cut) bfirst = bb;
                    blast = bb;
                    cut = true;
                }
            }
            // the seed's parts: from the group holding its start (the one before
            // its first unsnapped boundary) to the one before the first boundary
            // at or after its end
            if (cut && blockIdx.x == 0) P.cuts[atomicAdd(s_ncut, 1u)] = make_uint4((uint32_t)i, bfirst - 1, blast, 0);
        }
        __syncthreads();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            P.misc[4] = *s_ncut;
            P.misc[0] = globaltimer();
        }
    }

    // ---- phase 2: group slices of the work line -----------------------------------
    const uint32_t rlo = rr * P.rbits;
    const unsigned long long glo = W ? s_misc[0] : 0, ghi = W ? s_misc[1] : 0;
    const uint64_t ifirst = s_misc[2];
    unsigned long long wnext = s_misc[3];  // work-line start of seed ifirst
    // seed records {sinfo, w, f1win} prefetched into slots (i & 1), and the
    // next seed's first window staged during this seed's sweep
    unsigned long long* s_rec = s_misc + 8;  // [2][4]
    uint64_t rec_i = ~0ull;                  // seed whose record is in slot rec_i & 1
    bool staged = false;                     // seed rec_i's first window is in stg
    if (glo < ghi) {
        for (uint64_t i = ifirst; i < P.ns; ++i) {
            unsigned long long v0;
            uint4 si;
            uint32_t ow;
            if (i == rec_i) {
                const unsigned long long* r = s_rec + (i & 1) * 4;
                const uint2 x0 = *reinterpret_cast<const uint2*>(r), x1 = *reinterpret_cast<const uint2*>(r + 1);
                si = make_uint4(x0.x, x0.y, x1.x, x1.y);
                v0 = r[2];
                ow = (uint32_t)r[3];
            } else {
                v0 = ld_cg(P.w + i);
                si = __ldcg(P.sinfo + i);
                ow = ld_cg(P.f1win + i);  // meaningful only when si.w != kNoF1
                staged = false;
            }
            const unsigned long long ws = wnext, we = ws + (v0 ? v0 + P.seedcost : 0);
            wnext = we;
            if (ws >= ghi) break;
            if (we == ws) continue;
            const bool have_next = i + 1 < P.ns && we < ghi;
            if (have_next && threadIdx.x == 0) {  // the next record, into the other slot
                const uint32_t d = (uint32_t)__cvta_generic_to_shared(s_rec + ((i + 1) & 1) * 4);
                cp_async8(d, P.sinfo + i + 1);
                cp_async8(d + 8, reinterpret_cast<const char*>(P.sinfo + i + 1) + 8);
                cp_async8(d + 16, P.w + i + 1);
                cp_async4(d + 24, P.f1win + i + 1);
                cp_async_commit();
            }
            // this group's part of the seed: on the work line, then in adjacency
            // entries (the first seedcost units of a seed carry no entries)
            const unsigned long long a2 = max(glo, ws) - ws, z2 = min(ghi, we) - ws;
            const unsigned long long a = a2 > P.seedcost ? a2 - P.seedcost : 0;
            const unsigned long long z = z2 > P.seedcost ? z2 - P.seedcost : 0;
            const uint32_t s = si.x, b = si.y, deg = si.z, off = si.w;
            const bool v1 = a2 == 0;  // the part holding offset 0 also holds {s} u F1
            if (v1 && !P.walk && threadIdx.x == 0 && s - rlo < P.rbits)
                smem_or(bm_base, (s - rlo) >> 5, 1u << ((s - rlo) & 31));
            unsigned long long wbase = 0;  // seed-local entry offset of the current window
            uint32_t j0 = 0;
            if (staged) cp_async_wait_all();  // this thread's staged rows
            for (uint32_t k = 0; j0 < deg && wbase < z; j0 += kK2Win, ++k) {
                const uint32_t wl = min(kK2Win, deg - j0);
                if (off != kNoF1 && !v1) {
                    const unsigned long long wk = ld_cg(P.wt + ow + k);
                    if (wbase + wk <= a) {  // the whole window lies before this part
                        wbase += wk;
                        continue;
                    }
                }
                // per row: whole length d, this slice's part [sr, sr + lr)
                uint32_t d2[2], rb2[2], sr2[2], lr2[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t t = threadIdx.x * 2 + h;
                    d2[h] = rb2[h] = sr2[h] = lr2[h] = 0;
                    if (t < wl) {
                        uint32_t v, lo = 0, hi = 0xFFFFFFFFu;
                        if (k == 0 && staged) {  // copied in during the last sweep (this thread's rows)
                            v = stg[3 * kK2Stg + t];
                            rb2[h] = stg[t];
                            d2[h] = stg[kK2Stg + t];
                            if (P.R == 2) {
                                if (rr > 0) lo = stg[2 * kK2Stg + t];
                                else hi = stg[2 * kK2Stg + t];
                            }
                        } else if (off != kNoF1) {
                            v = (v1 || P.R > 2) ? ld_cg(P.f1v + off + j0 + t) : 0;
                            rb2[h] = ld_cg(P.f1rb + off + j0 + t);
                            d2[h] = ld_cg(P.f1d + off + j0 + t);
                            if (P.R == 2) {
                                const uint32_t sp = ld_cg(P.f1sp + off + j0 + t);
                                if (rr > 0) lo = sp; else hi = sp;
                            } else if (P.R > 2 && d2[h]) {  // this slice's crossings of row v
                                const uint32_t* sp = P.split + (size_t)v * (P.R - 1);
                                if (rr > 0) lo = __ldg(sp + rr - 1) - rb2[h];
                                if (rr + 1 < P.R) hi = __ldg(sp + rr) - rb2[h];
                            }
                        } else {
                            v = __ldg(g.ci + b + j0 + t);
                            rb2[h] = __ldg(g.rp + v);
                            if (v != s || P.walk) {
                                d2[h] = __ldg(g.rp + v + 1) - rb2[h];
                                const uint32_t* sp = P.split + (size_t)v * (P.R - 1);
                                if (rr > 0) lo = __ldg(sp + rr - 1) - rb2[h];
                                if (rr + 1 < P.R) hi = __ldg(sp + rr) - rb2[h];
                            }
                        }
                        sr2[h] = min(lo, d2[h]);
                        lr2[h] = min(hi, d2[h]) - sr2[h];
                        if (v1 && v - rlo < P.rbits) smem_or(bm_base, (v - rlo) >> 5, 1u << ((v - rlo) & 31));
                    }
                }
                // one scan of (whole << 32 | slice): both prefixes (a window's
                // rows are distinct vertices, so each sum is <= m < 2^32)
                unsigned long long exp;
                const unsigned long long tot =
                    block_excl_scan(((unsigned long long)(d2[0] + d2[1]) << 32) | (lr2[0] + lr2[1]), &exp, s_warp);
                const unsigned long long wtot = tot >> 32;
                {
                    const uint32_t c0 = (uint32_t)(exp >> 32), p0 = (uint32_t)exp;
                    const uint32_t p1 = p0 + lr2[0], p2 = p1 + lr2[1];
                    const uint32_t t = threadIdx.x * 2;
                    pre[t] = p0;
                    pre[t + 1] = p1;
                    prec[t] = c0;
                    prec[t + 1] = c0 + d2[0];
                    if (t < wl) {
                        srow[t] = sr2[0];
                        rinfo[t] = make_uint2(p1, rb2[0] + sr2[0] - p0);
                    }
                    if (t + 1 < wl) {
                        srow[t + 1] = sr2[1];
                        rinfo[t + 1] = make_uint2(p2, rb2[1] + sr2[1] - p1);
                    }
                    if (threadIdx.x == 0) {
                        pre[wl] = (uint32_t)tot;
                        prec[wl] = (uint32_t)wtot;
                    }
                }
                __syncthreads();
                const unsigned long long x0 = max(a, wbase), x1 = min(z, wbase + wtot);
                if (x0 < x1) {
                    // warp q takes [xs, xe) of the window's part as one flat
                    // stream: lane l reads entries xb + l + 32 j (coalesced within
                    // a row), each lane walking its own row cursor. All offsets
                    // are window-relative u32. Full blocks run without bounds
                    // checks; addresses first, then the loads back to back, then
                    // the atomics, so kK2Ilp loads per lane are in flight
                    // the part in whole-row units -> this slice's entries
                    auto to_slice = [&](uint32_t X) -> uint32_t {
                        if (X == 0) return 0;
                        if (X >= (uint32_t)wtot) return pre[wl];
                        uint32_t lo = 0, hi = wl;  // last row t with prec[t] <= X
                        while (hi - lo > 1) {
                            const uint32_t mid = (lo + hi) / 2;
                            if (prec[mid] <= X) lo = mid; else hi = mid;
                        }
                        const uint32_t o = X - prec[lo], sr = srow[lo], lr = pre[lo + 1] - pre[lo];
                        return pre[lo] + (o <= sr ? 0 : min(o - sr, lr));
                    };
                    const uint32_t X0 = to_slice((uint32_t)(x0 - wbase)), X1 = to_slice((uint32_t)(x1 - wbase));
                    const uint32_t span = X1 - X0;
                    const uint32_t xs = X0 + (uint32_t)((unsigned long long)span * wib / kK2Warps);
                    const uint32_t xe = X0 + (uint32_t)((unsigned long long)span * (wib + 1) / kK2Warps);
                    if (xs < xe) {
                        uint32_t lo = 0, hi = wl;  // last row t with pre[t] <= xs
                        while (hi - lo > 1) {
                            const uint32_t mid = (lo + hi) / 2;
                            if (pre[mid] <= xs) lo = mid; else hi = mid;
                        }
                        uint32_t tl = lo, nxt = rinfo[lo].x, dl = rinfo[lo].y;
                        const uint32_t ri_base = (uint32_t)__cvta_generic_to_shared(rinfo);
                        uint32_t xb = xs;
                        for (; xb + 32 * kK2Ilp <= xe; xb += 32 * kK2Ilp) {
                            uint32_t idx[kK2Ilp];
#pragma unroll
                            for (int q = 0; q < kK2Ilp; ++q) {
                                const uint32_t x = xb + lane + 32 * q;
                                while (nxt <= x) {
                                    ++tl;
                                    ld_rinfo(ri_base, tl, nxt, dl);
                                }
                                idx[q] = x + dl;
                            }
                            uint32_t u[kK2Ilp];
#pragma unroll
                            for (int q = 0; q < kK2Ilp; ++q) u[q] = __ldg(g.ci + idx[q]);
#pragma unroll
                            for (int q = 0; q < kK2Ilp; ++q) {
                                const uint32_t t = u[q] - rlo;
                                if (t < P.rbits) smem_or(bm_base, t >> 5, 1u << (t & 31));
                            }
                        }
                        if (xb < xe) {  // tail (< 32 * kK2Ilp entries): one masked block
                            uint32_t idx[kK2Ilp];
                            uint32_t valid = 0;
#pragma unroll
                            for (int q = 0; q < kK2Ilp; ++q) {
                                const uint32_t x = min(xb + lane + 32 * q, xe - 1);
                                valid |= (xb + lane + 32 * q < xe ? 1u : 0u) << q;
                                while (nxt <= x) {
                                    ++tl;
                                    ld_rinfo(ri_base, tl, nxt, dl);
                                }
                                idx[q] = x + dl;
                            }
                            uint32_t u[kK2Ilp];
#pragma unroll
                            for (int q = 0; q < kK2Ilp; ++q) u[q] = __ldg(g.ci + idx[q]);
#pragma unroll
                            for (int q = 0; q < kK2Ilp; ++q) {
                                const uint32_t t = u[q] - rlo;
                                if (((valid >> q) & 1u) && t < P.rbits) smem_or(bm_base, t >> 5, 1u << (t & 31));
                            }
                        }
                    }
                }
                wbase += wtot;
                __syncthreads();  // pre / prec / srow / rinfo are rewritten by the next window
            }
            if (v1)  // F1 rows in windows the loop did not reach
                for (uint32_t j = j0 + threadIdx.x; j < deg; j += kK2Block) {
                    const uint32_t v = (off != kNoF1 ? ld_cg(P.f1v + off + j) : __ldg(g.ci + b + j)) - rlo;
                    if (v < P.rbits) smem_or(bm_base, v >> 5, 1u << (v & 31));
                }
            if (have_next && threadIdx.x == 0) cp_async_wait_all();  // the next record
            __syncthreads();
            // the next seed's first window starts copying in now (it starts in
            // this group: its work-line start is this seed's end)
            staged = false;
            if (have_next) {
                const unsigned long long* r = s_rec + ((i + 1) & 1) * 4;
                const uint2 x1 = *reinterpret_cast<const uint2*>(r + 1);
                const uint32_t noff = x1.y, ndeg = x1.x;
                if (r[2] != 0 && noff != kNoF1 && P.R <= 2 && ndeg <= kK2Stg) {
                    const uint32_t wl = ndeg;
                    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(stg);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t t = threadIdx.x * 2 + h;
                        if (t < wl) {
                            cp_async4(sb + t * 4, P.f1rb + noff + t);
                            cp_async4(sb + (kK2Stg + t) * 4, P.f1d + noff + t);
                            if (P.R == 2) cp_async4(sb + (2 * kK2Stg + t) * 4, P.f1sp + noff + t);
                            cp_async4(sb + (3 * kK2Stg + t) * 4, P.f1v + noff + t);
                        }
                    }
                    cp_async_commit();
                    staged = true;
                }
                rec_i = i + 1;
            }
            // the slice is complete: popcount it (whole seed) or stage it (cut seed)
            const bool whole = ws >= glo && we <= ghi;
            uint4* bm4 = reinterpret_cast<uint4*>(bm);
            const uint32_t n4 = P.rwords / 4;
            if (whole) {
                uint32_t pc = 0;
#pragma unroll 4
                for (uint32_t q = threadIdx.x; q < n4; q += kK2Block) {
                    const uint4 x = bm4[q];
                    const uint32_t c = __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
                    pc += c;
                    if (c) bm4[q] = make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) pc += __shfl_xor_sync(kFull, pc, d);
                if (lane == 0 && pc) atomicAdd(&P.acc[i], (unsigned long long)pc);
            } else {
                const uint32_t slot = ws < glo ? 0 : 1;
                uint4* dst = reinterpret_cast<uint4*>(P.stage + ((size_t)(grp * 2 + slot) * R + rr) * P.rwords);
                for (uint32_t q = threadIdx.x; q < n4; q += kK2Block) {
                    const uint4 x = bm4[q];
                    __stcg(dst + q, x);
                    if (x.x | x.y | x.z | x.w) bm4[q] = make_uint4(0, 0, 0, 0);
                }
            }
            __syncthreads();
        }
    }
    grid_barrier(P.bar);
    if (gtid == 0) P.misc[1] = globaltimer();

    // ---- phase 3: cut seeds = OR of their staged slices ----------------------------
    // tasks: (cut seed, slice, 4096-word block)
    {
        constexpr uint32_t kBlk = 4 * kK2Block;
        const uint32_t nblk = (P.rwords + kBlk - 1) / kBlk;
        const uint32_t ntask = (uint32_t)ld_cg(P.misc + 4) * R * nblk;
        for (uint32_t t = blockIdx.x; t < ntask; t += gridDim.x) {
            const uint4 c = __ldcg(P.cuts + t / (R * nblk));
            const uint32_t r = (t / nblk) % R, blk = t % nblk;
            const uint64_t i = c.x;
            uint32_t pc = 0;
            const uint32_t q = blk * kBlk / 4 + threadIdx.x;
            if (q < P.rwords / 4) {
                // the seed starts inside group c.y (its slot 1) and runs through
                // the first slot of the groups after it; with W >= G no group
                // is empty, otherwise empty groups (no slice written) are skipped
                uint4 o = make_uint4(0, 0, 0, 0);
                const bool sparse = W < G;  // (snapped boundaries never empty a group inside a cut seed)
                for (uint32_t g0 = c.y; g0 <= c.z; g0 += 4) {
                    uint4 y[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t gg = g0 + k;
                        y[k] = make_uint4(0, 0, 0, 0);
                        if (gg <= c.z && (!sparse || ld_cg(P.bounds + gg) != ld_cg(P.bounds + gg + 1)))
                            y[k] = __ldcg(reinterpret_cast<const uint4*>(
                                              P.stage + ((size_t)(gg * 2 + (gg == c.y ? 1 : 0)) * R + r) * P.rwords) + q);
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        o.x |= y[k].x; o.y |= y[k].y; o.z |= y[k].z; o.w |= y[k].w;
                    }
                }
                pc = __popc(o.x) + __popc(o.y) + __popc(o.z) + __popc(o.w);
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) pc += __shfl_xor_sync(kFull, pc, d);
            if (lane == 0 && pc) atomicAdd(&P.acc[i], (unsigned long long)pc);
        }
    }
    grid_barrier(P.bar);
    if (gtid == 0) P.misc[2] = globaltimer();

    // ---- phase 4: answers and the per-hop counters ---------------------------------
    unsigned long long f1s = 0, f2s = 0, d1 = 0, e2 = 0, runs = 0;
    for (uint64_t i = gtid; i < P.ns; i += nthreads) {
        const unsigned long long nf = ld_cg(P.f1 + i);
        const unsigned long long raw = ld_cg(P.w + i), len = raw ? raw + P.seedcost : 0;
        // |B| = |{s} u F1 u N(F1)| (walks: |F1 u N(F1)|)
        const unsigned long long own = P.walk ? 0 : 1, pop = len ? ld_cg(P.acc + i) : own + nf;
        const unsigned long long ex = pop - own - nf;  // level 2
        P.counts[i] = P.cumulative ? pop - own : ex;
        if (P.counts1) P.counts1[i] = nf;  // k = 1, exact = cumulative
        if (len) P.acc[i] = 0;
        f1s += nf;
        f2s += ex;
        d1 += __ldcg(P.sinfo + i).z;
        e2 += len ? len - P.seedcost : 0;
        runs += nf != 0;
    }
    f1s = warp_sum_u64(f1s);
    f2s = warp_sum_u64(f2s);
    d1 = warp_sum_u64(d1);
    e2 = warp_sum_u64(e2);
    runs = warp_sum_u64(runs);
    if (lane == 0 && (f1s | d1 | runs)) {
        atomicAdd(&P.lc[1].frontier, f1s);
        atomicAdd(&P.lc[1].vertices, f1s);
        atomicAdd(&P.lc[1].scanned, d1);
        atomicAdd(&P.lc[1].edges, d1);
        atomicAdd(&P.lc[1].union_edges, d1);
        atomicAdd(&P.lc[2].frontier, f2s);
        atomicAdd(&P.lc[2].vertices, f2s);
        atomicAdd(&P.lc[2].scanned, e2);
        atomicAdd(&P.lc[2].edges, e2);
        atomicAdd(&P.lc[2].union_edges, e2);
        atomicAdd(&P.lc[2].runs, (unsigned)runs);
    }
    if (gtid == 0) {
        P.lc[1].runs = (unsigned)P.ns;
        P.misc[5] = P.misc[6] = P.misc[7] = 0;  // allocators (every CTA is past phase 2)
        const unsigned long long now = globaltimer();
        P.lc[0].ns = ld_cg(&P.misc[0]) - t0;                  // phases 0-1
        P.lc[2].ns = ld_cg(&P.misc[2]) - ld_cg(&P.misc[0]);  // slices + merge
        P.lc[MGK_MAX_HOPS + 1].ns = now - ld_cg(&P.misc[2]);
        if (P.diag) {  // MGK_K2_DIAG=1: phase timings (ns) in level 0 (scripts/k2probe.py)
            P.lc[0].candidates = ld_cg(&P.misc[1]) - ld_cg(&P.misc[0]);  // slices alone
            P.lc[0].frontier = ld_cg(&P.misc[8]) - t0;                    // phase 0a + barrier
            P.lc[0].vertices = ld_cg(&P.misc[9]) - ld_cg(&P.misc[8]);     // phase 0b + barrier
        }
    }
}

}  // namespace

// Eligible: k = 2 counts (k_hop exact / cumulative, or walk_targets windows
// [1, 2] / [2, 2]: the same set with the visited set starting empty),
// duplicate-free rows, no forced direction, and a bitmap that fits R <= 4
// slices of shared memory. MGK_NO_K2SMEM=1 keeps every call on fr_kernel.
// Per-device launch facts, looked up once (the host work between a caller's
// events and the launch is part of the measured call)
struct K2Device {
    int optin = 0, nsm = 0;  // optin: dynamic shared memory bytes one CTA may use
    size_t occ_smem[8] = {};  // occupancy cache: dynamic smem -> CTAs per SM
    int occ[8] = {};
    int nocc = 0;
};
std::mutex& k2_mutex() {
    static std::mutex mu;
    return mu;
}
// Looked up once per device under the mutex; the kernel's dynamic shared
// memory limit is raised to the opt-in maximum at that point, so no later call
// can lower it for another thread's larger graph.
K2Device& k2_device() {
    static K2Device devs[64];
    static bool ready[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 63;
    std::lock_guard<std::mutex> lk(k2_mutex());
    if (!ready[dev]) {
        cudaDeviceGetAttribute(&devs[dev].optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaDeviceGetAttribute(&devs[dev].nsm, cudaDevAttrMultiProcessorCount, dev);
        // the opt-in limit covers static + dynamic shared memory: the dynamic
        // part may use what the kernel's static arrays leave
        cudaFuncAttributes fa{};
        if (cudaFuncGetAttributes(&fa, k2_kernel) == cudaSuccess) devs[dev].optin -= (int)fa.sharedSizeBytes;
        if (MGK_K2_MINB > 1) {  // several CTAs per SM: each gets its share of the SM's shared memory
            int per_sm = 0;
            cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
            devs[dev].optin = std::min(devs[dev].optin, per_sm / MGK_K2_MINB - 1024 - (int)fa.sharedSizeBytes);
        }
        if (cudaFuncSetAttribute(k2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, devs[dev].optin) !=
            cudaSuccess) {
            (void)cudaGetLastError();
            devs[dev].optin = 0;  // k2_eligible then declines every call on this device
        }
        ready[dev] = true;
    }
    return devs[dev];
}
// CTAs per SM of k2_kernel at `smem` bytes of dynamic shared memory (cached
// per device under the same mutex).
cudaError_t k2_occupancy(K2Device& kd, size_t smem, int* per_sm) {
    std::lock_guard<std::mutex> lk(k2_mutex());
    for (int i = 0; i < kd.nocc; ++i)
        if (kd.occ_smem[i] == smem) {
            *per_sm = kd.occ[i];
            return cudaSuccess;
        }
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k2_kernel, kK2Block, smem);
    if (e) return e;
    const int slot = kd.nocc < 8 ? kd.nocc++ : 7;
    kd.occ_smem[slot] = smem;
    kd.occ[slot] = occ;
    *per_sm = occ;
    return cudaSuccess;
}

// bitmap words one CTA can hold (MGK_K2_SLICE_WORDS caps it, for tests of many slices)
uint32_t k2_max_words(int optin) {
    static const long cap = [] {
        const char* c = std::getenv("MGK_K2_SLICE_WORDS");
        return c ? std::atol(c) : 0L;
    }();
    uint32_t w = (uint32_t)(((uint64_t)optin - kK2Fixed) / 4 / 4 * 4);
    if (cap >= 4 && (uint32_t)cap < w) w = (uint32_t)cap / 4 * 4;
    return w;
}

bool k2_eligible(const Launch& L) {
    static const bool off = std::getenv("MGK_NO_K2SMEM") != nullptr;
    if (off || L.k != 2 || L.min_hop < 1 || L.keep_result || !L.g->dg.rows_unique) return false;
    if (L.tuning.force_dir != 0 || L.nseeds == 0) return false;
    const int optin = k2_device().optin;
    if (optin <= (int)kK2Fixed + 4096) return false;
    const uint64_t maxw = k2_max_words(optin);
    const uint64_t nw = L.g->dg.nwords;
    return (nw + maxw - 1) / maxw <= kK2MaxR;
}

bool k2_takes(const Graph* g, uint64_t nseeds, uint32_t min_hop) {
    Launch L{};
    L.g = g;
    L.nseeds = nseeds;
    L.k = 2;
    L.min_hop = min_hop;
    L.seed_visited = 1;
    L.tuning = g->tuning;
    return k2_eligible(L);
}

cudaError_t launch_k2(Launch& L) {
    const Graph* gr = L.g;
    Workspace* ws = L.ws;
    cudaError_t e;
    K2Device& kd = k2_device();
    const int optin = kd.optin, nsm = kd.nsm;
    const uint32_t maxw = k2_max_words(optin);
    const uint32_t nw = gr->dg.nwords;
    const uint32_t R = (nw + maxw - 1) / maxw;
    // slices of equal size, 128 vertices (4 x uint4 words) aligned
    const uint32_t rbits = (uint32_t)((((uint64_t)gr->dg.n + R - 1) / R + 127) / 128 * 128);
    const uint32_t rwords = rbits / 32;
    const size_t smem = (size_t)rwords * 4 + kK2Fixed;
    if (smem > (size_t)optin) return cudaErrorInvalidValue;
    int per_sm = 0;
    if ((e = k2_occupancy(kd, smem, &per_sm))) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint32_t grid = (uint32_t)(per_sm * nsm) / R * R;
    const uint32_t G = grid / R;
    // workspace: per-seed arrays (grow with the batch) and the staging area
    const uint64_t ns = L.nseeds;
    if (ws->k2_cap < ns) {
        for (void* p : {(void*)ws->k2_w, (void*)ws->k2_acc, (void*)ws->k2_f1, (void*)ws->k2_sinfo,
                        (void*)ws->k2_f1win, (void*)ws->k2_wt, (void*)ws->k2_tasks})
            cudaFree(p);
        ws->k2_w = ws->k2_acc = ws->k2_wt = nullptr;
        ws->k2_f1 = ws->k2_f1win = nullptr;
        ws->k2_sinfo = nullptr;
        ws->k2_tasks = nullptr;
        ws->k2_cap = 0;
        const uint64_t cap = std::max<uint64_t>(ns, 1024);
        // window totals and tasks: at most one partial window / task per seed
        // beyond the F1 rows' own count
        const uint64_t rows = std::min<uint64_t>(gr->dg.m + 1024, 8ull << 20);
        ws->k2_wtcap = cap + rows / kK2Win + 1;
        ws->k2_taskcap = cap + rows / kK2Task + 1;
        if ((e = cudaMalloc(&ws->k2_w, (cap + 1) * 8))) return e;
        if ((e = cudaMalloc(&ws->k2_acc, cap * 8))) return e;
        if ((e = cudaMalloc(&ws->k2_f1, cap * 4))) return e;
        if ((e = cudaMalloc(&ws->k2_sinfo, cap * 16))) return e;
        if ((e = cudaMalloc(&ws->k2_f1win, cap * 4))) return e;
        if ((e = cudaMalloc(&ws->k2_wt, ws->k2_wtcap * 8))) return e;
        if ((e = cudaMalloc(&ws->k2_tasks, ws->k2_taskcap * 16))) return e;
        if ((e = cudaMemset(ws->k2_acc, 0, cap * 8))) return e;
        if ((e = cudaStreamSynchronize(0))) return e;  // zero state before the first launch
        ws->k2_cap = cap;
        ws->bytes += cap * 28 + 8 + ws->k2_wtcap * 8 + ws->k2_taskcap * 16;
    }
    const size_t stage = (size_t)G * 2 * R * rwords * 4;
    if (ws->k2_stage_bytes < stage) {
        cudaFree(ws->k2_stage);
        ws->k2_stage = nullptr;
        ws->k2_stage_bytes = 0;
        if ((e = cudaMalloc(&ws->k2_stage, stage))) return e;
        ws->k2_stage_bytes = stage;
        ws->bytes += stage;
    }
    if (R > 1 && (!gr->k2_split || gr->k2_split_bits != rbits || gr->k2_split_R != R)) {
        // slice crossings of every row, once per graph (the first on-chip call)
        Graph* gm = const_cast<Graph*>(gr);
        std::lock_guard<std::mutex> lk(gm->mu);
        if (!gm->k2_split || gm->k2_split_bits != rbits || gm->k2_split_R != R) {
            cudaFree(gm->k2_split);
            gm->k2_split = nullptr;
            if ((e = cudaMalloc(&gm->k2_split, (size_t)gm->dg.n * (R - 1) * 4))) return e;
            k2_split_kernel<<<nsm * 8, 256, 0, L.stream>>>(gm->dg, R, rbits, gm->k2_split);
            if ((e = cudaStreamSynchronize(L.stream))) return e;
            gm->k2_split_bits = rbits;
            gm->k2_split_R = R;
            gm->bytes += (size_t)gm->dg.n * (R - 1) * 4;
        }
    }
    if (!ws->k2_f1v) {  // F1 rows of a call's seeds: up to min(m + 1024, 8M) entries
        uint64_t cap = std::min<uint64_t>(gr->dg.m + 1024, 8ull << 20);
        if (const char* c = std::getenv("MGK_K2_F1CAP")) cap = std::max<uint64_t>(1, std::strtoull(c, nullptr, 10));
        if ((e = cudaMalloc(&ws->k2_f1v, cap * 4))) return e;
        if ((e = cudaMalloc(&ws->k2_f1rb, cap * 4))) return e;
        if ((e = cudaMalloc(&ws->k2_f1d, cap * 4))) return e;
        ws->k2_f1cap = cap;
        ws->k2_f1sp_R = 0;
        ws->bytes += cap * 12;
    }
    if (R == 2 && ws->k2_f1sp_R < 2) {
        cudaFree(ws->k2_f1sp);
        ws->k2_f1sp = nullptr;
        if ((e = cudaMalloc(&ws->k2_f1sp, (size_t)ws->k2_f1cap * 4))) return e;
        ws->k2_f1sp_R = 2;
        ws->bytes += (size_t)ws->k2_f1cap * 4;
    }
    if (ws->k2_groups < G) {
        cudaFree(ws->k2_bounds);
        cudaFree(ws->k2_first);
        cudaFree(ws->k2_cuts);
        ws->k2_groups = 0;
        if ((e = cudaMalloc(&ws->k2_bounds, (size_t)(G + 1) * 8))) return e;
        if ((e = cudaMalloc(&ws->k2_first, (size_t)G * 4))) return e;
        if ((e = cudaMalloc(&ws->k2_cuts, (size_t)G * 16))) return e;
        ws->k2_groups = G;
    }
    if (!ws->k2_misc) {
        if ((e = cudaMalloc(&ws->k2_misc, 128))) return e;
        if ((e = cudaMemset(ws->k2_misc, 0, 128))) return e;
        if ((e = cudaStreamSynchronize(0))) return e;
    }
    K2Params Q;  // ~2 KB with the inline seeds; the launch copies it
    Q.g = gr->dg;
    Q.ns = ns;
    Q.counts = L.d_counts;
    Q.counts1 = L.d_counts1;
    Q.cumulative = L.min_hop <= 1 ? 1u : 0u;
    Q.walk = L.seed_visited ? 0u : 1u;
    Q.R = R;
    Q.rbits = rbits;
    Q.rwords = rwords;
    Q.ngroups = G;
    Q.w = ws->k2_w;
    Q.acc = ws->k2_acc;
    Q.f1 = ws->k2_f1;
    Q.stage = ws->k2_stage;
    Q.lc = ws->lc;
    Q.bar = reinterpret_cast<unsigned int*>(ws->misc + 8);
    Q.misc = ws->k2_misc;
    Q.bounds = ws->k2_bounds;
    Q.first = ws->k2_first;
    Q.cuts = ws->k2_cuts;
    Q.sinfo = ws->k2_sinfo;
    Q.f1win = ws->k2_f1win;
    Q.f1v = ws->k2_f1v;
    Q.f1rb = ws->k2_f1rb;
    Q.f1d = ws->k2_f1d;
    Q.f1sp = ws->k2_f1sp;
    Q.split = gr->k2_split;
    Q.f1cap = ws->k2_f1cap;
    Q.wt = ws->k2_wt;
    Q.wtcap = ws->k2_wtcap;
    Q.tasks = ws->k2_tasks;
    Q.taskcap = ws->k2_taskcap;
    static const unsigned long long seedcost = [] {
        const char* c = std::getenv("MGK_K2_SEEDCOST");
        return c ? std::strtoull(c, nullptr, 10) : 0ull;
    }();
    // a seed's fixed cost in adjacency-entry units: its slice sweep (~rwords)
    // plus the per-seed setup (measured on G2: ~60K entries-equivalent)
    // per slice CTA a seed costs ~12K cycles of setup plus its slice sweep; in
    // whole-row entry units (a CTA streams 1/R of a seed's entries) that is
    // R x (12288 + rwords / 2): G2 (R = 2) ~62K, G4 (R = 26) ~870K, measured
    Q.seedcost = seedcost ? seedcost : (unsigned long long)R * (12288ull + rwords / 2);
    static const unsigned long long snapdiv = [] {
        const char* c = std::getenv("MGK_K2_SNAP");
        return c ? std::max<unsigned long long>(1, std::strtoull(c, nullptr, 10)) : 8ull;
    }();
    Q.snapdiv = (uint32_t)snapdiv;
    static const uint32_t diag = std::getenv("MGK_K2_DIAG") != nullptr ? 1u : 0u;
    Q.diag = diag;
    if (L.host_io && ns <= kK2Inline) {
        Q.seeds = nullptr;
        std::memcpy(Q.inline_seeds, L.h_seeds, (size_t)ns * 4);
    } else {
        Q.seeds = L.d_seeds;
    }
    void* args[] = {&Q};
    if ((e = launch_persistent_smem((const void*)k2_kernel, grid, kK2Block, args, smem, L.stream))) return e;
    L.grid = grid;
    L.block = kK2Block;
    L.launches = 1;
    L.path = 1;
    return cudaSuccess;
}

}  // namespace mgk
