// The C ABI (include/mgk.h): validation with the reference's error texts,
// a per-graph workspace pool (reentrant calls), engine dispatch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "mgk_internal.cuh"

struct mgk_graph {
    mgk::Graph g;
    std::map<cudaStream_t, mgk::Workspace*> stream_ws;  // device-path workspaces
};

namespace mgk {
namespace {

thread_local std::string t_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return code;
}

int fail_cuda(cudaError_t e, const char* what) {
    cudaGetLastError();  // clear sticky-free errors
    if (e == cudaErrorMemoryAllocation)
        return fail(MGK_ENOMEM, "%s: out of device memory", what);
    return fail(MGK_ECUDA, "%s: CUDA error %d (%s)", what, (int)e, cudaGetErrorString(e));
}

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != prev) cudaSetDevice(prev);
    }
};

template <typename F>
void parallel_for(uint64_t n, F&& f) {
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (n < (1u << 16) || nt == 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> ts;
    const uint64_t step = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const uint64_t a = t * step, b = std::min(n, a + step);
        if (a < b) ts.emplace_back([&f, a, b] { f(a, b); });
    }
    for (auto& t : ts) t.join();
}

cudaError_t create_ws(Graph* g, Workspace* ws, bool own_stream) {
    ws->device = g->device;
    cudaError_t e;
    if (own_stream && (e = cudaStreamCreateWithFlags(&ws->stream, cudaStreamNonBlocking))) return e;
    if ((e = cudaEventCreate(&ws->ev0))) return e;
    if ((e = cudaEventCreate(&ws->ev1))) return e;
    if ((e = cudaMalloc(&ws->qctl, 4 * sizeof(QCtl)))) return e;
    if ((e = cudaMalloc(&ws->misc, 16 * 8))) return e;
    if ((e = cudaMalloc(&ws->lc, (MGK_MAX_HOPS + 2) * sizeof(LevelCounters)))) return e;
    if ((e = cudaMemset(ws->qctl, 0, 4 * sizeof(QCtl)))) return e;
    if ((e = cudaMemset(ws->misc, 0, 16 * 8))) return e;
    ws->bytes += 4 * sizeof(QCtl) + 128 + (MGK_MAX_HOPS + 2) * sizeof(LevelCounters);
    // legacy-stream memsets do not order non-blocking streams: finish them now
    return cudaStreamSynchronize(0);
}

void destroy_ws(Workspace* ws, bool own_stream) {
    cudaFree(ws->fr_V);
    cudaFree(ws->fr_Fb);
    for (auto* p : ws->fr_items) cudaFree(p);
    for (auto* p : ws->fr_big) cudaFree(p);
    cudaFree(ws->fr_log);
    cudaFree(ws->fr_cnt);
    cudaFree(ws->fr_mfs);
    cudaFree(ws->fr_mus);
    cudaFree(ws->fr_logcnt);
    cudaFree(ws->fr_pop);
    cudaFree(ws->fr_dirs);
    cudaFree(ws->fr_ctl);
    cudaFree(ws->fr_snap);
    cudaFree(ws->k2_w);
    cudaFree(ws->k2_acc);
    cudaFree(ws->k2_f1);
    cudaFree(ws->k2_stage);
    cudaFree(ws->k2_misc);
    cudaFree(ws->k2_bounds);
    cudaFree(ws->k2_first);
    cudaFree(ws->k2_cuts);
    cudaFree(ws->k2_sinfo);
    cudaFree(ws->k2_f1v);
    cudaFree(ws->k2_f1rb);
    cudaFree(ws->k2_f1d);
    cudaFree(ws->k2_f1sp);
    cudaFree(ws->k2_f1win);
    cudaFree(ws->k2_wt);
    cudaFree(ws->k2_tasks);
    cudaFree(ws->lv);
    cudaFree(ws->lf[0]);
    cudaFree(ws->lf[1]);
    cudaFree(ws->touched);
    cudaFree(ws->rlog);
    for (auto* p : ws->ms_items) cudaFree(p);
    cudaFree(ws->lane_cnt);
    cudaFree(ws->active);
    cudaFree(ws->umask);
    cudaFree(ws->qctl);
    cudaFree(ws->misc);
    cudaFree(ws->lc);
    cudaFree(ws->d_seeds);
    cudaFree(ws->d_counts);
    if (ws->h_pinned) cudaFreeHost(ws->h_pinned);
    if (ws->ev0) cudaEventDestroy(ws->ev0);
    if (ws->ev1) cudaEventDestroy(ws->ev1);
    if (own_stream && ws->stream) cudaStreamDestroy(ws->stream);
}

Workspace* acquire_ws(Graph* g, int* rc) {
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (!g->free_ws.empty()) {
            Workspace* ws = g->free_ws.back().release();
            g->free_ws.pop_back();
            return ws;
        }
    }
    auto* ws = new (std::nothrow) Workspace();
    if (!ws) {
        *rc = fail(MGK_ENOMEM, "out of host memory");
        return nullptr;
    }
    cudaError_t e = create_ws(g, ws, true);
    if (e) {
        destroy_ws(ws, true);
        delete ws;
        *rc = fail_cuda(e, "workspace");
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(g->mu);
    g->all_ws.push_back(ws);
    return ws;
}

void release_ws(Graph* g, Workspace* ws) {
    std::lock_guard<std::mutex> lk(g->mu);
    g->free_ws.emplace_back(ws);
}

int pick_words(const Graph* g, uint64_t nseeds) {
    if (g->tuning.lanes_words) return (int)g->tuning.lanes_words;
    const uint64_t want = (nseeds + 63) / 64;
    int W = 1;
    while (W < 8 && (uint64_t)W < want) W <<= 1;
    return W;
}

// LANES lane-word width: batches of at most 8 / 10 / 16 seeds use one uint8 /
// 10-bit (three per uint32) / uint16 word per vertex (state arrays 8x / 6x /
// 4x smaller, so a dense pull's per-edge gathers stay in L2 on large graphs);
// wider batches use uint64 words. MGK_LANE_BITS=8|10|16|64 forces a width
// (tests; a forced narrow width wider batches cannot use falls back to 64).
int pick_lane_bits(const Graph* g, uint64_t nseeds) {
    if (g->tuning.lanes_words) return 64;
    int bits = nseeds <= 8 ? 8 : nseeds <= 10 ? 10 : nseeds <= 16 ? 16 : 64;
    if (const char* e = std::getenv("MGK_LANE_BITS")) {
        const int f = std::atoi(e);
        if (f == 8 || f == 10 || f == 16 || f == 64) bits = f;
    }
    return (bits < 64 && nseeds > (uint64_t)bits) ? 64 : bits;
}

int check_query(const Graph* g, const uint64_t* seeds, uint64_t nseeds, uint32_t k) {
    // execute.cpp:348-354: seed first, then k
    for (uint64_t i = 0; i < nseeds; ++i)
        if (seeds[i] >= g->dg.n)
            return fail(MGK_ECONTRACT, "k-hop seed %llu is not an allocated node",
                        (unsigned long long)seeds[i]);
    if (k < 1 || k > MGK_MAX_HOPS)
        return fail(MGK_ECONTRACT, "k-hop count %u outside [1, %d]", k, MGK_MAX_HOPS);
    return MGK_OK;
}

// The hop window a call counts: k_hop exact = [k, k], cumulative = [1, k]
// (seed pre-visited, execute.cpp:357-370); walk_targets = [min, max] with the
// visited set starting empty (execute.cpp:43-60).
struct Span {
    uint32_t lo, hi;
    bool seed_visited;
};
Span span_of(uint32_t k, int mode) { return Span{mode == MGK_EXACT ? k : 1u, k, true}; }

// AUTO: shallow hops touch little of the graph per seed, so independent
// per-seed bitmaps win; from 3 hops on, frontiers of different seeds
// overlap heavily and the 64-lane words share every adjacency pass.
int resolve_engine(int engine, uint64_t nseeds, uint32_t k) {
    if (engine != MGK_ENGINE_AUTO) return engine;
    return (nseeds > 1 && k >= 3) ? MGK_ENGINE_LANES : MGK_ENGINE_SINGLE;
}

cudaError_t run_engine(Graph* g, Workspace* ws, const uint32_t* d_seeds, uint64_t nseeds,
                       Span span, int engine, unsigned long long* d_counts,
                       cudaStream_t stream, uint32_t* grid, uint32_t* block, int* used_engine,
                       int* W_out, bool keep_result = false, const uint32_t* h_seeds = nullptr,
                       unsigned long long* d_counts1 = nullptr, const Span* xspans = nullptr,
                       unsigned long long* const* xouts = nullptr, uint32_t nx = 0) {
    uint32_t k = span.hi, lo = span.lo;
    for (uint32_t j = 0; j < nx; ++j) {
        k = std::max(k, xspans[j].hi);
        lo = std::min(lo, xspans[j].lo);
    }
    // the engines zero the per-hop counters themselves (first launch of a call)
    cudaError_t e = cudaSuccess;
    if (nseeds == 0) {
        ws->last_launches = 0;
        return cudaMemsetAsync(ws->lc, 0, (MGK_MAX_HOPS + 2) * sizeof(LevelCounters), stream);
    }
    Launch L{};
    L.g = g;
    L.ws = ws;
    L.d_seeds = d_seeds;
    L.nseeds = nseeds;
    L.k = k;
    L.min_hop = lo;
    L.nextra = nx;
    L.ans_lo = span.lo;
    L.ans_hi = span.hi;
    for (uint32_t j = 0; j < nx; ++j) {
        L.xlo[j] = xspans[j].lo;
        L.xhi[j] = xspans[j].hi;
        L.xout[j] = xouts[j];
    }
    L.seed_visited = span.seed_visited ? 1u : 0u;
    L.d_counts = d_counts;
    L.d_counts1 = d_counts1;
    L.stream = stream;
    L.tuning = g->tuning;
    L.keep_result = keep_result;
    L.host_io = h_seeds != nullptr;
    L.h_seeds = h_seeds;
    engine = resolve_engine(engine, nseeds, k);
    if (nx && engine != MGK_ENGINE_LANES) return cudaErrorInvalidValue;  // fused windows are LANES-only
    *used_engine = engine;
    if (engine == MGK_ENGINE_SINGLE) {
        e = launch_single(L);
        *W_out = 0;
    } else {
        L.lane_bits = pick_lane_bits(g, nseeds);
        L.lanes_words = L.lane_bits == 64 ? pick_words(g, nseeds) : 1;
        *W_out = L.lane_bits == 64 ? 64 * L.lanes_words : L.lane_bits;  // lanes per batch
        e = launch_lanes(L);
    }
    *grid = L.grid;
    *block = L.block;
    ws->last_launches = e ? 0 : L.launches;
    ws->last_path = L.path;
    return e;
}

cudaError_t ensure_staging(Workspace* ws, uint64_t nseeds) {
    if (ws->seeds_cap >= nseeds) return cudaSuccess;
    cudaFree(ws->d_seeds);
    cudaFree(ws->d_counts);
    if (ws->h_pinned) cudaFreeHost(ws->h_pinned);
    ws->d_seeds = nullptr;
    ws->d_counts = nullptr;
    ws->h_pinned = nullptr;
    ws->seeds_cap = 0;
    const uint64_t cap = std::max<uint64_t>(nseeds, 1024);
    cudaError_t e;
    if ((e = cudaMalloc(&ws->d_seeds, cap * 4))) return e;
    if ((e = cudaMalloc(&ws->d_counts, cap * 8))) return e;
    // mapped: the SINGLE engine reads the seeds and writes the counts in place
    if ((e = cudaHostAlloc(&ws->h_pinned, cap * 12, cudaHostAllocMapped | cudaHostAllocPortable))) return e;
    ws->h_seeds = reinterpret_cast<uint32_t*>(ws->h_pinned);
    ws->h_counts = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ws->h_pinned) + cap * 4);
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&ws->h_seeds_dev), ws->h_seeds, 0))) return e;
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&ws->h_counts_dev), ws->h_counts, 0))) return e;
    ws->seeds_cap = cap;
    return cudaSuccess;
}

void fill_stats(mgk_stats* st, const LevelCounters* lc, int engine, int W, uint64_t nseeds,
                uint32_t grid, uint32_t block, float ms, uint32_t launches, uint32_t path) {
    std::memset(st, 0, sizeof *st);
    st->path = path;
    st->engine = (uint32_t)engine;
    st->lanes = engine == MGK_ENGINE_LANES ? (uint32_t)W : 1u;  // W = lanes per batch
    st->batches = (uint32_t)(engine == MGK_ENGINE_LANES ? (nseeds + st->lanes - 1) / st->lanes : nseeds);
    st->grid = grid;
    st->block = block;
    st->launches = launches;
    st->kernel_ms = ms;
    st->setup_ns = lc[0].ns;
    st->cleanup_ns = lc[MGK_MAX_HOPS + 1].ns;
    for (int h = 0; h <= MGK_MAX_HOPS; ++h) {
        mgk_level& L = st->level[h];
        L.frontier = lc[h].frontier;
        L.vertices = lc[h].vertices;
        L.edges = lc[h].edges;
        L.union_edges = lc[h].union_edges;
        L.scanned = lc[h].scanned;
        L.candidates = lc[h].candidates;
        L.runs = lc[h].runs;
        L.pull_runs = lc[h].pull_runs;
        L.ns = lc[h].ns;
        if (h > 0 && L.runs) st->hops = (uint32_t)h;
    }
}

int validate_csr_u64(uint64_t nrows, uint64_t nnz, const uint64_t* rp, const uint64_t* ci) {
    if (nrows >= 0xFFFFFFFFull) return fail(MGK_ERANGE, "graph has %llu rows; the device path holds < 2^32", (unsigned long long)nrows);
    if (nnz >= 0xFFFFFFFFull) return fail(MGK_ERANGE, "graph has %llu entries; the device path holds < 2^32", (unsigned long long)nnz);
    if (rp[0] != 0 || rp[nrows] != nnz)
        return fail(MGK_ECONTRACT, "row_ptr must start at 0 and end at nnz (%llu)", (unsigned long long)nnz);
    for (uint64_t r = 0; r < nrows; ++r)
        if (rp[r + 1] < rp[r]) return fail(MGK_ECONTRACT, "row_ptr decreases at row %llu", (unsigned long long)r);
    for (uint64_t p = 0; p < nnz; ++p)
        if (ci[p] >= nrows)
            return fail(MGK_ECONTRACT, "column %llu out of range for %llu rows", (unsigned long long)ci[p],
                        (unsigned long long)nrows);
    return MGK_OK;
}

int finish_upload(int device, uint64_t nrows, uint64_t nnz, const uint32_t* rp, const uint32_t* ci,
                  mgk_graph** out) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(MGK_ECUDA, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail(MGK_ECONTRACT, "device %d out of range [0, %d)", device, ndev);
    DeviceGuard dg(device);
    auto* h = new (std::nothrow) mgk_graph();
    if (!h) return fail(MGK_ENOMEM, "out of host memory");
    h->g.device = device;
    h->g.dg.n = (uint32_t)nrows;
    h->g.dg.m = nnz;
    cudaError_t e = build_device_graph(&h->g, rp, ci);
    if (e) {
        free_device_graph(&h->g);
        delete h;
        return fail_cuda(e, "graph upload");
    }
    *out = h;
    return MGK_OK;
}

}  // namespace

void set_last_error(const std::string& msg) { t_err = msg; }

cudaError_t launch_persistent(const void* fn, uint32_t grid, uint32_t block, void** args,
                              cudaStream_t stream) {
    static const bool noncoop = [] {
        const char* v = std::getenv("MGK_NONCOOP");
        return v && v[0] == '1';
    }();
    if (noncoop) return cudaLaunchKernel(fn, dim3(grid), dim3(block), args, 0, stream);
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, 0, stream);
}

// Persistent launch whose accesses to [base, base + bytes) are marked
// L2-persisting (the frontier words a pull gathers per edge): the device's
// persisting L2 set-aside is raised to its maximum once, and the window's hit
// ratio is the share of the window that fits it.
cudaError_t launch_persistent_l2(const void* fn, uint32_t grid, uint32_t block, void** args, cudaStream_t stream,
                                 void* base, size_t bytes) {
    static const bool noncoop = [] {
        const char* v = std::getenv("MGK_NONCOOP");
        return v && v[0] == '1';
    }();
    static std::mutex mu;
    static int maxp[64] = {}, maxw[64] = {};
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    dev &= 63;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (!done[dev]) {
            if (cudaDeviceGetAttribute(&maxp[dev], cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
                cudaDeviceGetAttribute(&maxw[dev], cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess ||
                cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp[dev]) != cudaSuccess) {
                cudaGetLastError();
                maxp[dev] = 0;
            }
            done[dev] = true;
        }
    }
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (!noncoop) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    if (maxp[dev] > 0 && maxw[dev] > 0 && bytes > 0) {
        bytes = std::min(bytes, (size_t)maxw[dev]);  // the window's size is capped by the device
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[na].val.accessPolicyWindow.base_ptr = base;
        attr[na].val.accessPolicyWindow.num_bytes = bytes;
        attr[na].val.accessPolicyWindow.hitRatio = std::min(1.0f, (float)maxp[dev] / (float)bytes);
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t launch_persistent_smem(const void* fn, uint32_t grid, uint32_t block, void** args, size_t smem,
                                   cudaStream_t stream) {
    static const bool noncoop = [] {
        const char* v = std::getenv("MGK_NONCOOP");
        return v && v[0] == '1';
    }();
    if (noncoop) return cudaLaunchKernel(fn, dim3(grid), dim3(block), args, smem, stream);
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, smem, stream);
}

}  // namespace mgk

using namespace mgk;

namespace {
// The device path's seed check (dev_id, mgk_device.cuh): read and clear the
// graph's flag; a set flag is the reference's ContractError for the seed.
int take_bad_seed(mgk::Graph* g) {
    unsigned int bad = 0;
    cudaError_t e = cudaMemcpy(&bad, g->bad_seed, 4, cudaMemcpyDeviceToHost);
    if (e) return fail_cuda(e, "device check");
    if (!bad) return MGK_OK;
    e = cudaMemset(g->bad_seed, 0, 4);
    if (e) return fail_cuda(e, "device check");
    return fail(MGK_ECONTRACT, "k-hop seed outside [0, %u) on the device path (not an allocated node)",
                g->dg.n);
}
}  // namespace

extern "C" {

const char* mgk_last_error(void) { return t_err.c_str(); }
int mgk_abi_version(void) { return MGK_ABI_VERSION; }

int mgk_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int mgk_graph_upload(int device, uint64_t nrows, uint64_t nnz, const uint64_t* row_ptr,
                     const uint64_t* col_idx, mgk_graph** out) {
    if (!out || !row_ptr || (nnz && !col_idx)) return fail(MGK_ECONTRACT, "null argument");
    int rc = validate_csr_u64(nrows, nnz, row_ptr, col_idx);
    if (rc) return rc;
    std::vector<uint32_t> rp(nrows + 1), ci(std::max<uint64_t>(nnz, 1));
    parallel_for(nrows + 1, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) rp[i] = (uint32_t)row_ptr[i];
    });
    parallel_for(nnz, [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) ci[i] = (uint32_t)col_idx[i];
    });
    return finish_upload(device, nrows, nnz, rp.data(), ci.data(), out);
}

int mgk_graph_upload_u32(int device, uint64_t nrows, uint64_t nnz, const uint32_t* row_ptr,
                         const uint32_t* col_idx, mgk_graph** out) {
    if (!out || !row_ptr || (nnz && !col_idx)) return fail(MGK_ECONTRACT, "null argument");
    if (nrows >= 0xFFFFFFFFull || nnz >= 0xFFFFFFFFull)
        return fail(MGK_ERANGE, "graph exceeds uint32 device indices");
    if (row_ptr[0] != 0 || row_ptr[nrows] != nnz)
        return fail(MGK_ECONTRACT, "row_ptr must start at 0 and end at nnz (%llu)", (unsigned long long)nnz);
    int bad = 0;
    parallel_for(nrows, [&](uint64_t a, uint64_t b) {
        for (uint64_t r = a; r < b; ++r)
            if (row_ptr[r + 1] < row_ptr[r]) bad = 1;
    });
    if (bad) return fail(MGK_ECONTRACT, "row_ptr decreases");
    parallel_for(nnz, [&](uint64_t a, uint64_t b) {
        for (uint64_t p = a; p < b; ++p)
            if (col_idx[p] >= nrows) bad = 2;
    });
    if (bad) return fail(MGK_ECONTRACT, "column out of range for %llu rows", (unsigned long long)nrows);
    return finish_upload(device, nrows, nnz, row_ptr, col_idx, out);
}

int mgk_graph_from_edges(int device, uint64_t nrows, uint64_t nedges, const uint32_t* src,
                         const uint32_t* dst, mgk_graph** out) {
    if (!out || (nedges && (!src || !dst))) return fail(MGK_ECONTRACT, "null argument");
    if (nrows >= 0xFFFFFFFFull) return fail(MGK_ERANGE, "graph exceeds uint32 device indices");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(MGK_ECUDA, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail(MGK_ECONTRACT, "device %d out of range", device);
    // bench.cpp:189-193 contract, checked on the host so the message names the edge
    for (uint64_t i = 0; i < nedges; ++i)
        if (src[i] >= nrows || dst[i] >= nrows)
            return fail(MGK_ECONTRACT, "edge (%u, %u) outside the %llu-node range", src[i], dst[i],
                        (unsigned long long)nrows);
    DeviceGuard dg(device);
    auto* h = new (std::nothrow) mgk_graph();
    if (!h) return fail(MGK_ENOMEM, "out of host memory");
    h->g.device = device;
    h->g.dg.n = (uint32_t)nrows;
    cudaError_t e = build_device_graph_from_edges(&h->g, src, dst, nedges);
    if (e) {
        free_device_graph(&h->g);
        delete h;
        return fail_cuda(e, "graph build");
    }
    *out = h;
    return MGK_OK;
}

int mgk_graph_gen_rmat(int device, uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                       uint64_t rng_seed, uint64_t target_unique, int relabel, mgk_graph** out) {
    if (!out) return fail(MGK_ECONTRACT, "null argument");
    if (scale < 1 || scale > 31) return fail(MGK_ECONTRACT, "RMAT scale must be in [1, 31]");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0 + 1e-9)
        return fail(MGK_ECONTRACT, "RMAT quadrant probabilities must be non-negative and sum to at most 1");
    if (relabel < 0 || relabel > 2) return fail(MGK_ECONTRACT, "relabel must be 0, 1 or 2");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(MGK_ECUDA, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail(MGK_ECONTRACT, "device %d out of range", device);
    DeviceGuard dg(device);
    auto* h = new (std::nothrow) mgk_graph();
    if (!h) return fail(MGK_ENOMEM, "out of host memory");
    h->g.device = device;
    cudaError_t e = build_device_graph_generated(&h->g, scale, edge_factor, a, b, c, rng_seed, target_unique,
                                                 relabel);
    if (e) {
        free_device_graph(&h->g);
        delete h;
        return e == cudaErrorInvalidValue ? fail(MGK_ERANGE, "generated graph exceeds uint32 indices")
                                          : fail_cuda(e, "graph generation");
    }
    *out = h;
    return MGK_OK;
}

int mgk_snapshot_check(const char* text, uint64_t len, uint64_t* node_count, uint64_t* edge_count) {
    if ((!text && len) || !node_count || !edge_count) return fail(MGK_ECONTRACT, "null argument");
    std::optional<std::string> err;
    try {
        err = snap::check_all(std::string_view(text ? text : "", len), node_count, edge_count);
    } catch (const std::bad_alloc&) {
        return fail(MGK_ENOMEM, "out of host memory");
    }
    if (err) return fail(MGK_ESNAPSHOT, "%s", err->c_str());
    return MGK_OK;
}

int mgk_graph_load_snapshot(int device, const char* text, uint64_t len, const char* relation,
                            mgk_graph** out, uint64_t* node_count) {
    if (!out || !node_count || (!text && len)) return fail(MGK_ECONTRACT, "null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(MGK_ECUDA, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail(MGK_ECONTRACT, "device %d out of range [0, %d)", device, ndev);
    DeviceGuard dg(device);
    auto* h = new (std::nothrow) mgk_graph();
    if (!h) return fail(MGK_ENOMEM, "out of host memory");
    h->g.device = device;
    std::string err;
    cudaError_t e = snap::load_to_graph(&h->g, text ? text : "", len, relation, node_count, &err);
    if (e || !err.empty()) {
        free_device_graph(&h->g);
        delete h;
        if (!err.empty()) return fail(MGK_ESNAPSHOT, "%s", err.c_str());
        return e == cudaErrorInvalidValue ? fail(MGK_ERANGE, "graph exceeds uint32 device indices")
                                          : fail_cuda(e, "snapshot load");
    }
    *out = h;
    return MGK_OK;
}

int mgk_graph_load_snapshot_file(int device, const char* path, const char* relation, mgk_graph** out,
                                 uint64_t* node_count) {
    if (!path) return fail(MGK_ECONTRACT, "null argument");
    FILE* f = std::fopen(path, "rb");
    if (!f) return fail(MGK_ESNAPSHOT, "cannot open '%s' for reading", path);
    std::string text;
    char buf[1 << 16];
    size_t got = 0;
    while ((got = std::fread(buf, 1, sizeof buf, f)) > 0) text.append(buf, got);
    const bool bad = std::ferror(f) != 0;
    std::fclose(f);
    if (bad) return fail(MGK_ESNAPSHOT, "failed reading snapshot from '%s'", path);
    return mgk_graph_load_snapshot(device, text.data(), text.size(), relation, out, node_count);
}

int mgk_graph_free(mgk_graph* h) {
    if (!h) return MGK_OK;
    DeviceGuard dg(h->g.device);
    cudaDeviceSynchronize();
    for (Workspace* ws : h->g.all_ws) {
        destroy_ws(ws, true);
        delete ws;
    }
    for (auto& f : h->g.free_ws) f.release();
    for (auto& kv : h->stream_ws) {
        destroy_ws(kv.second, false);
        delete kv.second;
    }
    free_device_graph(&h->g);
    delete h;
    return MGK_OK;
}

int mgk_graph_info(const mgk_graph* h, uint64_t* nrows, uint64_t* nnz, int* device) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    if (nrows) *nrows = h->g.dg.n;
    if (nnz) *nnz = h->g.dg.m;
    if (device) *device = h->g.device;
    return MGK_OK;
}

uint64_t mgk_graph_device_bytes(const mgk_graph* h) {
    if (!h) return 0;
    uint64_t b = h->g.bytes;
    for (Workspace* ws : h->g.all_ws) b += ws->bytes;
    for (auto& kv : h->stream_ws) b += kv.second->bytes;
    return b;
}

int mgk_graph_download_csr(const mgk_graph* h, uint32_t* row_ptr, uint32_t* col_idx) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    DeviceGuard dg(h->g.device);
    cudaError_t e = download_graph(&h->g, row_ptr, col_idx, nullptr, nullptr);
    return e ? fail_cuda(e, "download") : MGK_OK;
}

int mgk_graph_download_csc(const mgk_graph* h, uint32_t* col_ptr, uint32_t* row_idx) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    DeviceGuard dg(h->g.device);
    cudaError_t e = download_graph(&h->g, nullptr, nullptr, col_ptr, row_idx);
    return e ? fail_cuda(e, "download") : MGK_OK;
}

int mgk_graph_set_tuning(mgk_graph* h, const mgk_tuning* t) {
    if (!h || !t) return fail(MGK_ECONTRACT, "null argument");
    if (t->force_dir > 2) return fail(MGK_ECONTRACT, "force_dir must be 0, 1 or 2");
    if (t->lanes_words && t->lanes_words != 1 && t->lanes_words != 2 && t->lanes_words != 4 &&
        t->lanes_words != 8)
        return fail(MGK_ECONTRACT, "lanes_words must be 1, 2, 4 or 8");
    std::lock_guard<std::mutex> lk(h->g.mu);
    if (t->alpha) h->g.tuning.alpha = t->alpha;
    if (t->alpha_lanes) h->g.tuning.alpha_lanes = t->alpha_lanes;
    if (t->alpha_last) h->g.tuning.alpha_last = t->alpha_last;
    if (t->beta) h->g.tuning.beta = t->beta;
    h->g.tuning.force_dir = t->force_dir;
    h->g.tuning.lanes_words = t->lanes_words;
    return MGK_OK;
}

int mgk_graph_get_tuning(const mgk_graph* h, mgk_tuning* t) {
    if (!h || !t) return fail(MGK_ECONTRACT, "null argument");
    t->alpha = h->g.tuning.alpha;
    t->alpha_lanes = h->g.tuning.alpha_lanes;
    t->alpha_last = h->g.tuning.alpha_last;
    t->beta = h->g.tuning.beta;
    t->force_dir = h->g.tuning.force_dir;
    t->lanes_words = h->g.tuning.lanes_words;
    return MGK_OK;
}

}  // extern "C"

namespace mgk {
namespace {
// Counts of a batch of seeds over the hop window `span` (host buffers).
// Counts of a batch of seeds over several hop windows (host buffers): all
// windows are enqueued on the workspace's stream and answered with one
// synchronisation; counts[w * nseeds + i] is window w of seed i.
// A k = 1 section (seed pre-visited) of a call that also has a k = 2 section
// taking the on-chip path is answered by that launch (|F1| is a by-product of
// it): fused[w] = the k = 2 section answering section w, or -1.
std::vector<int> plan_k1_fusion(const Graph* g, uint64_t nseeds, const Span* spans, uint32_t n, int engine) {
    std::vector<int> fused(n, -1);
    int k2 = -1;
    for (uint32_t w = 0; w < n && k2 < 0; ++w)
        if (spans[w].hi == 2 && spans[w].seed_visited && resolve_engine(engine, nseeds, 2) == MGK_ENGINE_SINGLE &&
            k2_takes(g, nseeds, spans[w].lo))
            k2 = (int)w;
    if (k2 < 0) return fused;
    for (uint32_t w = 0; w < n; ++w)
        if (spans[w].hi == 1 && spans[w].seed_visited) {
            fused[w] = k2;
            break;  // one k = 1 output per launch
        }
    return fused;
}

// LANES sections of one seed list share one traversal: the first LANES
// section (the lead) runs to the deepest hop of them all and answers the
// others from its per-lane hop counts (a window's count is a sum of per-hop
// frontier sizes, which do not depend on how deep the traversal goes).
// lanes_lead[w] = the lead answering section w, or -1.
std::vector<int> plan_lanes_fusion(uint64_t nseeds, const Span* spans, uint32_t n, int engine,
                                   const std::vector<int>& k1_fused) {
    std::vector<int> lead(n, -1);
    int first = -1, taken = 0;
    for (uint32_t w = 0; w < n; ++w) {
        if (k1_fused[w] >= 0 || resolve_engine(engine, nseeds, spans[w].hi) != MGK_ENGINE_LANES) continue;
        if (first < 0) {
            first = (int)w;
        } else if (spans[w].seed_visited == spans[first].seed_visited && taken < Launch::kMaxExtra) {
            lead[w] = first;
            ++taken;
        }
    }
    return lead;
}

// the windows a lead section also answers, and where they go
void lanes_extras(const std::vector<int>& lead, uint32_t w, const Span* spans, unsigned long long* base,
                  uint64_t nseeds, std::vector<Span>& xs, std::vector<unsigned long long*>& xo) {
    xs.clear();
    xo.clear();
    for (uint32_t j = 0; j < lead.size(); ++j)
        if (lead[j] == (int)w) {
            xs.push_back(spans[j]);
            xo.push_back(base + j * nseeds);
        }
}

int count_impl_multi(mgk_graph* h, const uint64_t* seeds, uint64_t nseeds, const Span* spans, uint32_t nspans,
                     int engine, uint64_t* counts, mgk_stats* stats, const char* what) {
    Graph* g = &h->g;
    int rc = MGK_OK;
    if (nseeds >= 0xFFFFFFFFull) return fail(MGK_ECONTRACT, "too many seeds");
    DeviceGuard dg(g->device);
    Workspace* ws = acquire_ws(g, &rc);
    if (!ws) return rc;
    cudaError_t e = ensure_staging(ws, std::max<uint64_t>(nseeds * nspans, 1));
    if (e) {
        release_ws(g, ws);
        return fail_cuda(e, "staging");
    }
    // seeds: host uint64 -> pinned, device-mapped uint32 (inside the caller's timing)
    uint32_t* hs = ws->h_seeds;
    for (uint64_t i = 0; i < nseeds; ++i) hs[i] = (uint32_t)seeds[i];
    // SINGLE reads the seeds over the bus (k = 1) or carries each group's
    // seeds in its launch, and writes the counts straight into the mapped
    // buffer: no copy operations on the stream. LANES stages through HBM.
    uint32_t grid = 0, block = 0;
    int used = 0, W = 0;
    float ms = 0.f;
    bool seeds_on_device = false;
    const std::vector<int> fused = plan_k1_fusion(g, nseeds, spans, nspans, engine);
    const std::vector<int> lead = plan_lanes_fusion(nseeds, spans, nspans, engine, fused);
    int k1_of = -1;  // the section a fused k = 2 launch also answers
    uint32_t last_run = 0;
    for (uint32_t w = 0; w < nspans; ++w) {
        if (fused[w] >= 0) k1_of = (int)w;
        else if (lead[w] < 0) last_run = w;
    }
    std::vector<Span> xs;
    std::vector<unsigned long long*> xo;
    do {
        for (uint32_t w = 0; w < nspans && !e; ++w) {
            if (fused[w] >= 0 || lead[w] >= 0) continue;  // answered by another section's launch
            const int eng = resolve_engine(engine, nseeds, spans[w].hi);
            const bool host_io = eng == MGK_ENGINE_SINGLE;
            if (!host_io && !seeds_on_device) {
                if ((e = cudaMemcpyAsync(ws->d_seeds, hs, nseeds * 4, cudaMemcpyHostToDevice, ws->stream))) break;
                seeds_on_device = true;
            }
            const bool last = w == last_run;
            unsigned long long* out = host_io ? ws->h_counts_dev : ws->d_counts;
            unsigned long long* out1 = (k1_of >= 0 && fused[k1_of] == (int)w) ? out + k1_of * nseeds : nullptr;
            lanes_extras(lead, w, spans, out, nseeds, xs, xo);
            if (stats && last && (e = cudaEventRecord(ws->ev0, ws->stream))) break;
            if ((e = run_engine(g, ws, host_io ? ws->h_seeds_dev : ws->d_seeds, nseeds, spans[w], eng,
                                out + w * nseeds, ws->stream, &grid, &block, &used, &W, false,
                                host_io ? hs : nullptr, out1, xs.data(), xo.data(), (uint32_t)xs.size())))
                break;
            if (stats && last && (e = cudaEventRecord(ws->ev1, ws->stream))) break;
            if (!host_io) {
                for (uint32_t j = 0; j < nspans && !e; ++j)
                    if (j == w || lead[j] == (int)w)
                        e = cudaMemcpyAsync(ws->h_counts + j * nseeds, ws->d_counts + j * nseeds, nseeds * 8,
                                            cudaMemcpyDeviceToHost, ws->stream);
                if (e) break;
            }
        }
        if (e) break;
        if ((e = cudaStreamSynchronize(ws->stream))) break;
        std::memcpy(counts, ws->h_counts, nseeds * nspans * 8);
        if (stats) {  // the last window's counters
            cudaEventElapsedTime(&ms, ws->ev0, ws->ev1);
            LevelCounters lc[MGK_MAX_HOPS + 2];
            if ((e = cudaMemcpy(lc, ws->lc, sizeof lc, cudaMemcpyDeviceToHost))) break;
            fill_stats(stats, lc, used, W, nseeds, grid, block, ms, ws->last_launches, ws->last_path);
        }
    } while (0);
    release_ws(g, ws);
    return e ? fail_cuda(e, what) : MGK_OK;
}

int count_impl(mgk_graph* h, const uint64_t* seeds, uint64_t nseeds, Span span, int engine,
               uint64_t* counts, mgk_stats* stats, const char* what) {
    return count_impl_multi(h, seeds, nseeds, &span, 1, engine, counts, stats, what);
}

// walk_targets' window checks, with the Cypher parser's messages (cypher.cpp:356-392)
int check_walk(const Graph* g, const uint64_t* seeds, uint64_t nseeds, uint32_t lo, uint32_t hi) {
    for (uint64_t i = 0; i < nseeds; ++i)
        if (seeds[i] >= g->dg.n)
            return fail(MGK_ECONTRACT, "walk source %llu is not an allocated node", (unsigned long long)seeds[i]);
    if (lo < 1) return fail(MGK_ECONTRACT, "hop minimum must be at least 1");
    if (hi > MGK_MAX_HOPS) return fail(MGK_ECONTRACT, "hop count %u exceeds the cap of %d", hi, MGK_MAX_HOPS);
    if (hi < lo) return fail(MGK_ECONTRACT, "hop maximum %u is less than minimum %u", hi, lo);
    return MGK_OK;
}
}  // namespace
}  // namespace mgk

extern "C" {

int mgk_khop_count_ex(mgk_graph* h, const uint64_t* seeds, uint64_t nseeds, uint32_t k, int mode,
                      int engine, uint64_t* counts, mgk_stats* stats) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    if (nseeds && (!seeds || !counts)) return fail(MGK_ECONTRACT, "null argument");
    if (mode != MGK_EXACT && mode != MGK_CUMULATIVE) return fail(MGK_ECONTRACT, "unknown traverse mode %d", mode);
    if (engine < MGK_ENGINE_AUTO || engine > MGK_ENGINE_LANES) return fail(MGK_ECONTRACT, "unknown engine %d", engine);
    int rc = check_query(&h->g, seeds, nseeds, k);
    if (rc) return rc;
    return count_impl(h, seeds, nseeds, span_of(k, mode), engine, counts, stats, "k-hop count");
}

int mgk_walk_count(mgk_graph* h, const uint64_t* seeds, uint64_t nseeds, uint32_t min_hops,
                   uint32_t max_hops, int engine, uint64_t* counts) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    if (nseeds && (!seeds || !counts)) return fail(MGK_ECONTRACT, "null argument");
    if (engine < MGK_ENGINE_AUTO || engine > MGK_ENGINE_LANES) return fail(MGK_ECONTRACT, "unknown engine %d", engine);
    int rc = check_walk(&h->g, seeds, nseeds, min_hops, max_hops);
    if (rc) return rc;
    return count_impl(h, seeds, nseeds, Span{min_hops, max_hops, false}, engine, counts, nullptr,
                      "walk count");
}

int mgk_khop_count(mgk_graph* h, const uint64_t* seeds, uint64_t nseeds, uint32_t k, int mode,
                   uint64_t* counts) {
    return mgk_khop_count_ex(h, seeds, nseeds, k, mode, MGK_ENGINE_AUTO, counts, nullptr);
}

int mgk_khop_count_ks(mgk_graph* h, const uint64_t* seeds, uint64_t nseeds, const uint32_t* ks, uint32_t nks,
                      int mode, uint64_t* counts) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    if ((nseeds && !seeds) || (nks && !ks) || (nseeds && nks && !counts)) return fail(MGK_ECONTRACT, "null argument");
    if (mode != MGK_EXACT && mode != MGK_CUMULATIVE) return fail(MGK_ECONTRACT, "unknown traverse mode %d", mode);
    std::vector<Span> spans(nks);
    for (uint32_t w = 0; w < nks; ++w) {  // execute.cpp:348-354 per query: the seed, then k
        int rc = check_query(&h->g, seeds, nseeds, ks[w]);
        if (rc) return rc;
        spans[w] = span_of(ks[w], mode);
    }
    if (nks == 0) return MGK_OK;
    return count_impl_multi(h, seeds, nseeds, spans.data(), nks, MGK_ENGINE_AUTO, counts, nullptr, "k-hop count");
}

int mgk_graph_replicate(const mgk_graph* src, int device, mgk_graph** out) {
    if (!src || !out) return fail(MGK_ECONTRACT, "null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(MGK_ECUDA, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail(MGK_ECONTRACT, "device %d out of range [0, %d)", device, ndev);
    DeviceGuard dg(device);
    auto* h = new (std::nothrow) mgk_graph();
    if (!h) return fail(MGK_ENOMEM, "out of host memory");
    h->g.device = device;
    cudaError_t e = replicate_device_graph(&src->g, &h->g);
    if (e) {
        free_device_graph(&h->g);
        delete h;
        return fail_cuda(e, "graph replicate");
    }
    *out = h;
    return MGK_OK;
}

int mgk_graph_transpose(const mgk_graph* src, mgk_graph** out) {
    if (!src || !out) return fail(MGK_ECONTRACT, "null argument");
    DeviceGuard dg(src->g.device);
    auto* h = new (std::nothrow) mgk_graph();
    if (!h) return fail(MGK_ENOMEM, "out of host memory");
    h->g.device = src->g.device;
    cudaError_t e = transpose_device_graph(&src->g, &h->g);
    if (e) {
        free_device_graph(&h->g);
        delete h;
        return fail_cuda(e, "graph transpose");
    }
    *out = h;
    return MGK_OK;
}

int mgk_khop_count_multi(mgk_graph* const* replicas, int nreplicas, const uint64_t* seeds, uint64_t nseeds,
                         uint32_t k, int mode, uint64_t* counts) {
    if (!replicas || nreplicas < 1) return fail(MGK_ECONTRACT, "no replicas");
    for (int i = 0; i < nreplicas; ++i) {
        if (!replicas[i]) return fail(MGK_ECONTRACT, "null graph");
        if (replicas[i]->g.dg.n != replicas[0]->g.dg.n || replicas[i]->g.dg.m != replicas[0]->g.dg.m)
            return fail(MGK_ECONTRACT, "replica %d is not a copy of replica 0", i);
    }
    if (nseeds && (!seeds || !counts)) return fail(MGK_ECONTRACT, "null argument");
    if (mode != MGK_EXACT && mode != MGK_CUMULATIVE) return fail(MGK_ECONTRACT, "unknown traverse mode %d", mode);
    int rc = check_query(&replicas[0]->g, seeds, nseeds, k);
    if (rc) return rc;
    // One host thread (and the replica's own stream) per shard; no collective:
    // every shard writes disjoint entries of `counts`. Per-seed engines (k <= 2)
    // get cost-balanced shards — a seed's work follows its out-degree and varies
    // ~10x — by longest-first greedy on the degrees; the lane
    // engine's 64-seed batches take contiguous shards.
    const Span span = span_of(k, mode);
    std::vector<int> rcs(nreplicas, MGK_OK);
    std::vector<std::string> errs(nreplicas);
    std::vector<std::vector<uint64_t>> part(nreplicas);
    const bool balance = nreplicas > 1 && k <= 2 && nseeds >= 2 * (uint64_t)nreplicas;
    if (balance) {
        std::vector<uint32_t> s32(nseeds), deg(nseeds);
        for (uint64_t i = 0; i < nseeds; ++i) s32[i] = (uint32_t)seeds[i];
        {
            DeviceGuard dg(replicas[0]->g.device);
            cudaError_t e = seed_degrees(&replicas[0]->g, s32.data(), nseeds, deg.data());
            if (e) return fail_cuda(e, "seed degrees");
        }
        std::vector<uint64_t> order(nseeds);
        for (uint64_t i = 0; i < nseeds; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](uint64_t x, uint64_t y) { return deg[x] > deg[y]; });
        std::vector<uint64_t> load(nreplicas, 0);
        for (uint64_t i : order) {
            const int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
            part[r].push_back(i);
            load[r] += (uint64_t)deg[i] + 1;
        }
        for (auto& p : part) std::sort(p.begin(), p.end());
    }
    auto run = [&](int i) {
        if (balance) {
            const auto& idx = part[i];
            if (idx.empty()) return;
            std::vector<uint64_t> s(idx.size()), c(idx.size());
            for (size_t j = 0; j < idx.size(); ++j) s[j] = seeds[idx[j]];
            rcs[i] = count_impl(replicas[i], s.data(), s.size(), span, MGK_ENGINE_AUTO, c.data(), nullptr,
                                "k-hop count");
            if (!rcs[i])
                for (size_t j = 0; j < idx.size(); ++j) counts[idx[j]] = c[j];
        } else {
            const uint64_t a = nseeds * (uint64_t)i / nreplicas, b = nseeds * (uint64_t)(i + 1) / nreplicas;
            if (b == a) return;
            rcs[i] = count_impl(replicas[i], seeds + a, b - a, span, MGK_ENGINE_AUTO, counts + a, nullptr,
                                "k-hop count");
        }
        if (rcs[i]) errs[i] = t_err;
    };
    std::vector<std::thread> ts;
    for (int i = 1; i < nreplicas; ++i) ts.emplace_back(run, i);
    run(0);
    for (auto& t : ts) t.join();
    for (int i = 0; i < nreplicas; ++i)
        if (rcs[i]) {
            t_err = errs[i];
            return rcs[i];
        }
    return MGK_OK;
}

}  // extern "C"

namespace mgk {
namespace {
// the workspace of a caller's stream (created on first use)
Workspace* stream_workspace(mgk_graph* h, cudaStream_t s, int* rc) {
    Graph* g = &h->g;
    Workspace* ws = nullptr;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        auto it = h->stream_ws.find(s);
        if (it != h->stream_ws.end()) ws = it->second;
    }
    if (ws) return ws;
    ws = new (std::nothrow) Workspace();
    if (!ws) {
        *rc = fail(MGK_ENOMEM, "out of host memory");
        return nullptr;
    }
    cudaError_t e = create_ws(g, ws, false);
    if (e) {
        destroy_ws(ws, false);
        delete ws;
        *rc = fail_cuda(e, "workspace");
        return nullptr;
    }
    ws->stream = s;
    std::lock_guard<std::mutex> lk(g->mu);
    h->stream_ws[s] = ws;
    return ws;
}

// device-path sections: spans[w]'s answers at d_counts + w * nseeds
int count_device_multi(mgk_graph* h, const uint32_t* d_seeds, uint64_t nseeds, const Span* spans, uint32_t nspans,
                       int engine, uint64_t* d_counts, void* stream) {
    Graph* g = &h->g;
    if (nseeds && g->dg.n == 0) return fail(MGK_ECONTRACT, "k-hop seed on a graph with no nodes");
    DeviceGuard dg(g->device);
    cudaStream_t s = (cudaStream_t)stream;
    int rc = MGK_OK;
    Workspace* ws = stream_workspace(h, s, &rc);
    if (!ws) return rc;
    const std::vector<int> fused = plan_k1_fusion(g, nseeds, spans, nspans, engine);
    const std::vector<int> lead = plan_lanes_fusion(nseeds, spans, nspans, engine, fused);
    int k1_of = -1;
    for (uint32_t w = 0; w < nspans; ++w)
        if (fused[w] >= 0) k1_of = (int)w;
    auto* out = reinterpret_cast<unsigned long long*>(d_counts);
    uint32_t grid = 0, block = 0;
    int used = 0, W = 0;
    cudaError_t e = cudaSuccess;
    std::vector<Span> xs;
    std::vector<unsigned long long*> xo;
    for (uint32_t w = 0; w < nspans && !e; ++w) {
        if (fused[w] >= 0 || lead[w] >= 0) continue;  // answered by another section's launch
        unsigned long long* out1 = (k1_of >= 0 && fused[k1_of] == (int)w) ? out + k1_of * nseeds : nullptr;
        lanes_extras(lead, w, spans, out, nseeds, xs, xo);
        e = run_engine(g, ws, d_seeds, nseeds, spans[w], engine, out + w * nseeds, s, &grid, &block, &used, &W, false,
                       nullptr, out1, xs.data(), xo.data(), (uint32_t)xs.size());
    }
    ws->misc_engine = used;
    ws->misc_W = W;
    ws->misc_grid = grid;
    ws->misc_block = block;
    ws->misc_nseeds = nseeds;
    return e ? fail_cuda(e, "k-hop count (device)") : MGK_OK;
}
}  // namespace
}  // namespace mgk

extern "C" {

int mgk_khop_count_device(mgk_graph* h, const uint32_t* d_seeds, uint64_t nseeds, uint32_t k,
                          int mode, int engine, uint64_t* d_counts, void* stream) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    if (k < 1 || k > MGK_MAX_HOPS) return fail(MGK_ECONTRACT, "k-hop count %u outside [1, %d]", k, MGK_MAX_HOPS);
    if (mode != MGK_EXACT && mode != MGK_CUMULATIVE) return fail(MGK_ECONTRACT, "unknown traverse mode %d", mode);
    if (engine < MGK_ENGINE_AUTO || engine > MGK_ENGINE_LANES) return fail(MGK_ECONTRACT, "unknown engine %d", engine);
    const Span sp = span_of(k, mode);
    return count_device_multi(h, d_seeds, nseeds, &sp, 1, engine, d_counts, stream);
}

int mgk_khop_count_device_ks(mgk_graph* h, const uint32_t* d_seeds, uint64_t nseeds, const uint32_t* ks,
                             uint32_t nks, int mode, uint64_t* d_counts, void* stream) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    if (nks && !ks) return fail(MGK_ECONTRACT, "null argument");
    if (mode != MGK_EXACT && mode != MGK_CUMULATIVE) return fail(MGK_ECONTRACT, "unknown traverse mode %d", mode);
    std::vector<Span> spans(nks);
    for (uint32_t w = 0; w < nks; ++w) {
        if (ks[w] < 1 || ks[w] > MGK_MAX_HOPS)
            return fail(MGK_ECONTRACT, "k-hop count %u outside [1, %d]", ks[w], MGK_MAX_HOPS);
        spans[w] = span_of(ks[w], mode);
    }
    if (nks == 0) return MGK_OK;
    return count_device_multi(h, d_seeds, nseeds, spans.data(), nks, MGK_ENGINE_AUTO, d_counts, stream);
}

// run_khop_benchmark's sections (bench.cpp:311-343) in one call: section j is
// k_hop_count(seeds[i], ks[j]) for the prefix i < nseeds_per_k[j] of one
// master seed list. Consecutive sections with the same prefix length share
// their launches (count_*_multi).
namespace {
int check_schedule(const uint64_t* nseeds_per_k, const uint32_t* ks, uint32_t nks, uint64_t* total,
                   uint64_t* longest) {
    if (nks && (!nseeds_per_k || !ks)) return fail(MGK_ECONTRACT, "null argument");
    *total = *longest = 0;
    for (uint32_t j = 0; j < nks; ++j) {  // bench.cpp:297-309, the reference's messages
        if (ks[j] < 1 || ks[j] > MGK_MAX_HOPS)
            return fail(MGK_ECONTRACT, "hop count %u outside [1, %d]", ks[j], MGK_MAX_HOPS);
        if (nseeds_per_k[j] == 0) return fail(MGK_ECONTRACT, "seed count for k=%u must be at least 1", ks[j]);
        *total += nseeds_per_k[j];
        *longest = std::max(*longest, nseeds_per_k[j]);
    }
    return MGK_OK;
}
}  // namespace

int mgk_khop_count_schedule(mgk_graph* h, const uint64_t* seeds, const uint64_t* nseeds_per_k, const uint32_t* ks,
                            uint32_t nks, int mode, uint64_t* counts) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    if (mode != MGK_EXACT && mode != MGK_CUMULATIVE) return fail(MGK_ECONTRACT, "unknown traverse mode %d", mode);
    uint64_t total = 0, longest = 0;
    int rc = check_schedule(nseeds_per_k, ks, nks, &total, &longest);
    if (rc) return rc;
    if (total && (!seeds || !counts)) return fail(MGK_ECONTRACT, "null argument");
    for (uint32_t j = 0; j < nks; ++j)  // execute.cpp:348-354 for every query of the section
        if ((rc = check_query(&h->g, seeds, nseeds_per_k[j], ks[j]))) return rc;
    uint64_t off = 0;
    for (uint32_t a = 0; a < nks;) {
        uint32_t b = a + 1;
        while (b < nks && nseeds_per_k[b] == nseeds_per_k[a]) ++b;
        std::vector<Span> spans;
        for (uint32_t j = a; j < b; ++j) spans.push_back(span_of(ks[j], mode));
        if ((rc = count_impl_multi(h, seeds, nseeds_per_k[a], spans.data(), b - a, MGK_ENGINE_AUTO, counts + off,
                                   nullptr, "k-hop count")))
            return rc;
        off += (b - a) * nseeds_per_k[a];
        a = b;
    }
    return MGK_OK;
}

int mgk_khop_count_device_schedule(mgk_graph* h, const uint32_t* d_seeds, const uint64_t* nseeds_per_k,
                                   const uint32_t* ks, uint32_t nks, int mode, uint64_t* d_counts, void* stream) {
    if (!h) return fail(MGK_ECONTRACT, "null graph");
    if (mode != MGK_EXACT && mode != MGK_CUMULATIVE) return fail(MGK_ECONTRACT, "unknown traverse mode %d", mode);
    uint64_t total = 0, longest = 0;
    int rc = check_schedule(nseeds_per_k, ks, nks, &total, &longest);
    if (rc) return rc;
    uint64_t off = 0;
    for (uint32_t a = 0; a < nks;) {
        uint32_t b = a + 1;
        while (b < nks && nseeds_per_k[b] == nseeds_per_k[a]) ++b;
        std::vector<Span> spans;
        for (uint32_t j = a; j < b; ++j) spans.push_back(span_of(ks[j], mode));
        if ((rc = count_device_multi(h, d_seeds, nseeds_per_k[a], spans.data(), b - a, MGK_ENGINE_AUTO,
                                     d_counts + off, stream)))
            return rc;
        off += (b - a) * nseeds_per_k[a];
        a = b;
    }
    return MGK_OK;
}

int mgk_khop_device_check(mgk_graph* h, void* stream) {
    if (!h) return fail(MGK_ECONTRACT, "null argument");
    DeviceGuard dg(h->g.device);
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e) return fail_cuda(e, "device check");
    return take_bad_seed(&h->g);
}

int mgk_khop_device_stats(mgk_graph* h, void* stream, mgk_stats* stats) {
    if (!h || !stats) return fail(MGK_ECONTRACT, "null argument");
    Workspace* ws = nullptr;
    {
        std::lock_guard<std::mutex> lk(h->g.mu);
        auto it = h->stream_ws.find((cudaStream_t)stream);
        if (it != h->stream_ws.end()) ws = it->second;
    }
    if (!ws) return fail(MGK_ECONTRACT, "no device-path call was made on this stream");
    DeviceGuard dg(h->g.device);
    LevelCounters lc[MGK_MAX_HOPS + 2];
    // the counters of the last call enqueued on this stream: wait for it
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (!e) e = cudaMemcpy(lc, ws->lc, sizeof lc, cudaMemcpyDeviceToHost);
    if (e) return fail_cuda(e, "stats");
    if (int rc = take_bad_seed(&h->g)) return rc;
    fill_stats(stats, lc, ws->misc_engine, ws->misc_W, ws->misc_nseeds, ws->misc_grid, ws->misc_block, 0.f,
               ws->last_launches, ws->last_path);
    return MGK_OK;
}

}  // extern "C"

namespace mgk {
namespace {
int ids_impl(mgk_graph* h, uint64_t seed, Span span, uint64_t* ids, uint64_t cap, uint64_t* n_out,
             const char* what) {
    Graph* g = &h->g;
    int rc = MGK_OK;
    DeviceGuard dg(g->device);
    Workspace* ws = acquire_ws(g, &rc);
    if (!ws) return rc;
    cudaError_t e = ensure_staging(ws, 1);
    unsigned long long* d_ids = nullptr;
    unsigned long long* d_n = nullptr;
    do {
        if (e) break;
        reinterpret_cast<uint32_t*>(ws->h_pinned)[0] = (uint32_t)seed;
        if ((e = cudaMemcpyAsync(ws->d_seeds, ws->h_pinned, 4, cudaMemcpyHostToDevice, ws->stream))) break;
        uint32_t grid = 0, block = 0;
        int used = 0, W = 0;
        if ((e = run_engine(g, ws, ws->d_seeds, 1, span, MGK_ENGINE_SINGLE, ws->d_counts, ws->stream, &grid,
                            &block, &used, &W, true)))
            break;
        if ((e = cudaMalloc(&d_ids, (size_t)std::max<uint32_t>(g->dg.n, 1) * 8))) break;
        if ((e = cudaMalloc(&d_n, 8))) break;
        if ((e = single_result_ids(g, ws, span.lo, span.seed_visited, (uint32_t)seed, d_ids, d_n, ws->stream)))
            break;
        unsigned long long n = 0;
        if ((e = cudaMemcpyAsync(&n, d_n, 8, cudaMemcpyDeviceToHost, ws->stream))) break;
        if ((e = cudaStreamSynchronize(ws->stream))) break;
        if ((e = ids_to_external(g, d_ids, n, ws->stream))) break;
        if ((e = cudaStreamSynchronize(ws->stream))) break;
        *n_out = n;
        const uint64_t take = std::min<uint64_t>(n, cap);
        if (take && (e = cudaMemcpy(ids, d_ids, take * 8, cudaMemcpyDeviceToHost))) break;
    } while (0);
    cudaFree(d_ids);
    cudaFree(d_n);
    release_ws(g, ws);
    return e ? fail_cuda(e, what) : MGK_OK;
}
}  // namespace
}  // namespace mgk

extern "C" {

int mgk_khop_frontier(mgk_graph* h, uint64_t seed, uint32_t k, int mode, uint64_t* ids, uint64_t cap,
                      uint64_t* n_out) {
    if (!h || !n_out || (cap && !ids)) return fail(MGK_ECONTRACT, "null argument");
    if (mode != MGK_EXACT && mode != MGK_CUMULATIVE) return fail(MGK_ECONTRACT, "unknown traverse mode %d", mode);
    int rc = check_query(&h->g, &seed, 1, k);
    if (rc) return rc;
    return ids_impl(h, seed, span_of(k, mode), ids, cap, n_out, "k-hop frontier");
}

int mgk_walk_targets(mgk_graph* h, uint64_t seed, uint32_t min_hops, uint32_t max_hops, uint64_t* ids,
                     uint64_t cap, uint64_t* n_out) {
    if (!h || !n_out || (cap && !ids)) return fail(MGK_ECONTRACT, "null argument");
    int rc = check_walk(&h->g, &seed, 1, min_hops, max_hops);
    if (rc) return rc;
    return ids_impl(h, seed, Span{min_hops, max_hops, false}, ids, cap, n_out, "walk targets");
}

}  // extern "C"
