// Device-side building blocks shared by the traversal engines (sm_100a).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "mgk_internal.cuh"

namespace mgk {
namespace dev {

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// L2 evict-last policy for the per-seed bitmaps: their lines should outlive
// the streamed adjacency (loaded evict-first) until the cleanup pass.
__device__ __forceinline__ unsigned long long l2_keep_policy() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void red_or_keep(uint32_t* p, uint32_t v, unsigned long long pol) {
    asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint32_t atom_or_keep(uint32_t* p, uint32_t v, unsigned long long pol) {
    uint32_t old;
    asm volatile("atom.global.or.L2::cache_hint.b32 %0, [%1], %2, %3;"
                 : "=r"(old) : "l"(p), "r"(v), "l"(pol) : "memory");
    return old;
}

// L2 evict-first policy for streamed, read-once data (the CSC row_idx a pull
// scans), so it does not push the frontier words out of L2.
__device__ __forceinline__ unsigned long long l2_stream_policy() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// immutable graph arrays: non-coherent path, L1-allocating, L2 priority `pol`
__device__ __forceinline__ uint32_t ldg_hint(const uint32_t* p, unsigned long long pol) {
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ldg_hint_v4(const uint4* p, unsigned long long pol) {
    uint4 v;
    asm("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(p), "l"(pol));
    return v;
}
// state written earlier in the same launch (ordered by the grid barrier):
// coherent loads, L2 priority `pol`
__device__ __forceinline__ uint32_t ld_hint_u8(const void* p, unsigned long long pol) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u8 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ld_hint_u16(const void* p, unsigned long long pol) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u16 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_stream_u16(void* p, uint32_t v) {
    asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void st_stream_u8(void* p, uint32_t v) {
    asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void st_stream_u64(void* p, unsigned long long v) {
    asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_hint_u64(const void* p, unsigned long long pol) {
    unsigned long long v;
    asm volatile("ld.global.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}

// device id of an external seed id (locality relabelling; identity if none).
// A seed >= n (the device path does not range-check on the host) raises the
// graph's bad_seed flag and is replaced by vertex 0, so no read goes out of
// bounds; the call's answers are then undefined and the host reports
// MGK_ECONTRACT at the next checked call (mgk_khop_device_stats /
// mgk_khop_device_check).
__device__ __forceinline__ uint32_t dev_id(const DevGraph& g, uint32_t x) {
    if (x >= g.n) {
        atomicOr(g.bad_seed, 1u);
        x = 0;
    }
    return g.perm ? __ldg(g.perm + x) : x;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Loads of mutable state that other SMs update inside the same launch go to
// L2 (ld.global.cg) so a stale L1 line never hides a concurrent update.
__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ld_cg(const unsigned long long* p) {
    return __ldcg(p);
}
__device__ __forceinline__ uint32_t ld_cg_u8(const uint8_t* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned int ld_volatile(const unsigned int* p) {
    return *reinterpret_cast<const volatile unsigned int*>(p);
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// Grid-wide barrier for the persistent engines (bar[0] = arrivals, bar[1] =
// generation). Every CTA of the grid must be resident: the engines launch
// with cudaLaunchCooperativeKernel (which guarantees it) and size the grid
// from the occupancy calculator; MGK_NONCOOP=1 uses a plain launch of the
// same grid so profilers that skip cooperative launches still see the kernel.
// Each CTA reads the generation once per launch (grid_barrier_init, before its
// first arrival, so no barrier can complete before the read); a barrier is
// then one acq_rel add per CTA and an acquire spin on the generation — the
// release / acquire pair orders every thread's memory traffic of the phase
// (through the CTA barriers on both sides), like cooperative_groups grid.sync().
static __shared__ unsigned int s_bar_gen;

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_barrier_init(unsigned int* bar) {
    if (threadIdx.x == 0) s_bar_gen = ld_acquire_gpu(bar + 1);
}

__device__ __forceinline__ void grid_barrier(unsigned int* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = s_bar_gen;
        unsigned int old;
        // acq_rel: the arrival publishes this CTA's phase (release) and, for
        // the last arriver, synchronises with every earlier arrival's release
        // in the counter's RMW chain (acquire) — so the last CTA's next-phase
        // loads (L1-allocating ones included) see the other CTAs' writes
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old == gridDim.x - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1) : "memory");
        } else {
            while (ld_acquire_gpu(bar + 1) == gen) {
            }
        }
        s_bar_gen = gen + 1;
    }
    __syncthreads();
}

// Inclusive warp scan (all 32 lanes must call).
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, v, d);
        if (lane >= (uint32_t)d) v += t;
    }
    return v;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
    return v;
}

__device__ __forceinline__ unsigned long long warp_or_u64(unsigned long long v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v |= __shfl_xor_sync(kFull, v, d);
    return v;
}

// Smallest lane j whose inclusive prefix incl_j > x (x < incl_31), via a
// 5-step shuffle binary search. All lanes must call (x may differ per lane).
__device__ __forceinline__ uint32_t warp_owner(uint32_t incl, uint32_t x) {
    uint32_t lo = 0;
#pragma unroll
    for (uint32_t step = 16; step >= 1; step >>= 1) {
        const uint32_t probe = __shfl_sync(kFull, incl, lo + step - 1);
        if (probe <= x) lo += step;
    }
    return lo;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Per-warp shared-memory staging of discovered vertex ids. Discoveries are
// appended with a ballot (no atomics); a global reservation is taken only
// when the stage is nearly full or at the end of a phase, so a hot queue tail
// sees one atomic per ~200 vertices instead of one per warp step.
template <int CAP, typename T = uint32_t>
struct Stage {
    T* buf;      // CAP entries in shared memory, private to this warp
    uint32_t n;  // warp-uniform fill
    __device__ __forceinline__ void push(bool pred, T v) {
        const unsigned m = __ballot_sync(kFull, pred);
        if (pred) buf[n + __popc(m & lanemask_lt())] = v;
        n += __popc(m);
        __syncwarp();
    }
    __device__ __forceinline__ bool full() const { return n > CAP - 32; }
};

// Warp-wide: append n staged ids to list[*tail ...] (one atomic).
__device__ __forceinline__ void emit_list(const uint32_t* buf, uint32_t n, uint32_t* list,
                                          unsigned int* tail) {
    if (n == 0) return;
    uint32_t base = 0;
    if (lane_id() == 0) base = atomicAdd(tail, n);
    base = __shfl_sync(kFull, base, 0);
    for (uint32_t i = lane_id(); i < n; i += 32) list[base + i] = buf[i];
    __syncwarp();
}

// Warp-wide: append push work items for n staged vertices: each vertex with
// out-degree d yields ceil(d / kChunk) slices of its CSR row. One reservation
// per call. Item is uint2 {begin, end} or uint4 {begin, end, src, 0}.
__device__ __forceinline__ void store_item(uint2* items, uint32_t at, uint32_t s, uint32_t e,
                                           uint32_t) {
    items[at] = make_uint2(s, e);
}
__device__ __forceinline__ void store_item(uint4* items, uint32_t at, uint32_t s, uint32_t e,
                                           uint32_t src) {
    items[at] = make_uint4(s, e, src, 0);
}

// entries per push work item (kChunk for every row: longer items made the
// warps holding a hub row's items the push's critical path — a push entry is a
// chain of dependent random accesses — which cost more than writing the hub's
// many short items)
__device__ __forceinline__ uint32_t item_len(uint32_t) { return kChunk; }

template <typename Item>
__device__ __forceinline__ void emit_items(const uint32_t* __restrict__ rp, const uint32_t* buf,
                                           uint32_t n, Item* items, unsigned int* nitems) {
    if (n == 0) return;
    const uint32_t lane = lane_id();
    uint32_t tot = 0;
    for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t u = buf[i];
        const uint32_t d = __ldg(rp + u + 1) - __ldg(rp + u);
        tot += (d + item_len(d) - 1) / item_len(d);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) tot += __shfl_xor_sync(kFull, tot, d);
    if (tot == 0) return;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(nitems, tot);
    base = __shfl_sync(kFull, base, 0);
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        uint32_t u = 0, b = 0, deg = 0;
        if (i < n) {
            u = buf[i];
            b = __ldg(rp + u);
            deg = __ldg(rp + u + 1) - b;
        }
        const uint32_t cs = item_len(deg);
        const uint32_t nit = (deg + cs - 1) / cs;
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
            const uint32_t cj = __shfl_sync(kFull, cs, j);
            if (x < total) {
                const uint32_t s = bj + (x - ej) * cj;
                store_item(items, base + x, s, min(s + cj, bj + dj), uj);
            }
        }
        base += total;
    }
    __syncwarp();
}

// Items per warp iteration so that small work lists still spread over every
// warp of the grid: a power of two in [1, 32].
__device__ __forceinline__ uint32_t items_per_warp(uint32_t nitems, uint64_t nwarps) {
    uint32_t g = 1;
    while (g < 32 && g * 2 * nwarps <= nitems) g <<= 1;
    return g;
}

// Block-level accumulation of counters, flushed once per phase.
struct PhaseAcc {
    unsigned long long frontier, vertices, edges, union_edges, scanned, candidates;
    __device__ void zero() { frontier = vertices = edges = union_edges = scanned = candidates = 0; }
};

// Flush per-thread counters into a LevelCounters record with one atomic per
// warp per field (values reduced over the warp first).
__device__ __forceinline__ void flush_counters(LevelCounters* lc, PhaseAcc& a) {
    const unsigned long long f = warp_sum_u64(a.frontier);
    const unsigned long long v = warp_sum_u64(a.vertices);
    const unsigned long long e = warp_sum_u64(a.edges);
    const unsigned long long u = warp_sum_u64(a.union_edges);
    const unsigned long long s = warp_sum_u64(a.scanned);
    const unsigned long long c = warp_sum_u64(a.candidates);
    if (lane_id() == 0) {
        if (f) atomicAdd(&lc->frontier, f);
        if (v) atomicAdd(&lc->vertices, v);
        if (e) atomicAdd(&lc->edges, e);
        if (u) atomicAdd(&lc->union_edges, u);
        if (s) atomicAdd(&lc->scanned, s);
        if (c) atomicAdd(&lc->candidates, c);
    }
    a.zero();
}

}  // namespace dev
}  // namespace mgk
