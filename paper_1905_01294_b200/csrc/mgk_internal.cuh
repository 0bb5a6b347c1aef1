// Internal declarations shared by the mgk translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "mgk.h"

namespace mgk {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr uint32_t kChunk = 32;  // max adjacency entries per push work item

// ---- device graph -------------------------------------------------------------
// uint32 CSR + CSC, 256-B aligned (cudaMalloc), immutable after build.
struct DevGraph {
    uint32_t n = 0;       // matrix dimension
    uint32_t nwords = 0;  // ceil(n / 32) bitmap words
    uint64_t m = 0;       // stored entries
    const uint32_t* rp = nullptr;     // row_ptr[n+1]
    const uint32_t* ci = nullptr;     // col_idx[m], ascending per row
    const uint32_t* cp = nullptr;     // col_ptr[n+1] (CSC)
    const uint32_t* ri = nullptr;     // row_idx[m], ascending per column
    const uint32_t* no_in = nullptr;  // bitmap: zero in-degree (and padding ids >= n)
    // pull load balance: vertices with in-degree > kHeavyIn are scanned as
    // kHeavyChunk-entry tasks spread over the grid instead of by one warp
    const uint32_t* pull_skip = nullptr;  // no_in | heavy: what the per-word pull pass skips
    const uint2* heavy = nullptr;         // {vertex, first CSC entry} per task
    uint32_t nheavy = 0;
    // every CSR row strictly ascending (no duplicate entries): hop 1 from a
    // seed is then its row minus the seed itself, with no test-and-set
    uint32_t rows_unique = 0;
    // locality relabelling (ids by descending in-degree): device id of an
    // external id (perm) and back (inv); null = identity
    const uint32_t* perm = nullptr;
    const uint32_t* inv = nullptr;
    // set (never cleared on the device) when a device-path call meets a seed
    // >= n; the host reports it as MGK_ECONTRACT at the next checked call
    unsigned int* bad_seed = nullptr;
};
constexpr uint32_t kHeavyIn = 1024;
constexpr uint32_t kHeavyChunk = 1024;

// Per-level device counters, mirrored into mgk_level on the host.
struct LevelCounters {
    unsigned long long frontier;
    unsigned long long vertices;
    unsigned long long edges;
    unsigned long long union_edges;
    unsigned long long scanned;
    unsigned long long candidates;
    unsigned int runs;
    unsigned int pull_runs;
    unsigned long long ns;
};
static_assert(sizeof(LevelCounters) == 8 * 8, "layout");

// Queue control block of one frontier buffer.
struct QCtl {
    unsigned int nitems;       // push work items written
    unsigned int nfound;       // vertices discovered (incl. zero out-degree)
    unsigned long long edges;  // sum of outdeg over discovered vertices
    unsigned long long indeg;  // sum of indeg over discovered vertices
    unsigned long long pad;
};

struct Tuning {
    uint32_t alpha = 4;   // push -> pull when frontier edges > unexplored in-edges / alpha
    uint32_t beta = 24;   // pull -> push when frontier vertices < n / beta
    uint32_t force_dir = 0;
    uint32_t lanes_words = 0;  // 0 = auto
    uint32_t alpha_lanes = 2;  // LANES: a pull pass rarely exits early, so switch later
    // SINGLE's last hop only counts: a push is one fire-and-forget red.or per
    // edge, a pull must settle every unvisited vertex, so pull only when the
    // frontier's out-edges exceed the whole unexplored in-edge set
    uint32_t alpha_last = 1;
};

// Workspace for one in-flight call. Sized for the graph; reused across calls.
struct Workspace {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // single-source engine (per-seed bitmaps, fr_slots seeds in flight)
    uint32_t fr_slots = 0;
    uint32_t* fr_V = nullptr;   // [S][nwords]
    uint32_t* fr_Fb = nullptr;  // [3][S][nwords]
    uint2* fr_items[2] = {nullptr, nullptr};
    uint32_t fr_items_cap = 0;
    uint2* fr_big[2] = {nullptr, nullptr};
    uint32_t fr_big_cap = 0;
    unsigned long long* fr_log = nullptr;
    uint32_t fr_log_cap = 0, fr_quota = 0;
    uint32_t* fr_cnt = nullptr;
    unsigned long long* fr_mfs = nullptr;
    unsigned long long* fr_mus = nullptr;
    uint32_t* fr_logcnt = nullptr;
    unsigned long long* fr_pop = nullptr;
    uint8_t* fr_dirs = nullptr;
    void* fr_ctl = nullptr;
    uint32_t* fr_snap = nullptr;  // keep_result: slot 0's visited bitmap after hop min-1
    // k = 2 on-chip path (mgk_k2.cu)
    unsigned long long* k2_w = nullptr;    // [cap + 1] per-seed work, scanned
    unsigned long long* k2_acc = nullptr;  // [cap] popcounts (zero between launches)
    uint32_t* k2_f1 = nullptr;             // [cap] |F1|
    uint64_t k2_cap = 0;
    uint32_t* k2_stage = nullptr;          // slices of seeds cut by a group boundary
    size_t k2_stage_bytes = 0;
    unsigned long long* k2_misc = nullptr;
    unsigned long long* k2_bounds = nullptr;
    uint32_t* k2_first = nullptr;
    uint4* k2_cuts = nullptr;
    uint32_t k2_groups = 0;
    uint4* k2_sinfo = nullptr;              // [cap] per seed
    uint32_t* k2_f1v = nullptr;             // [k2_f1cap] F1 rows of the seeds
    uint32_t* k2_f1rb = nullptr;
    uint32_t* k2_f1d = nullptr;
    uint32_t* k2_f1sp = nullptr;            // [k2_f1cap][R-1] slice splits within each F1 row
    uint32_t k2_f1sp_R = 0;
    uint64_t k2_f1cap = 0;
    uint32_t* k2_f1win = nullptr;           // [cap] per seed
    unsigned long long* k2_wt = nullptr;    // window totals
    uint64_t k2_wtcap = 0;
    uint4* k2_tasks = nullptr;              // phase-0 tasks
    uint64_t k2_taskcap = 0;
    // lanes engine (allocated lazily for the widest W used)
    int lanes_words = 0;
    unsigned long long* lv = nullptr;     // V  [n * W]
    unsigned long long* lf[2] = {nullptr, nullptr};  // F  [n * W] x2
    uint32_t* touched = nullptr;          // [nwords]
    uint32_t* rlog = nullptr;             // raw discovery log
    uint64_t rlog_cap = 0;
    uint4* ms_items[2] = {nullptr, nullptr};
    unsigned long long* lane_cnt = nullptr;  // [(MGK_MAX_HOPS+1) * 64 * W]
    unsigned long long* active = nullptr;    // [2 * W]
    uint32_t* umask = nullptr;                // [2][nwords] per word, vertices a pull left unsettled (by hop parity)
    // shared small control block
    QCtl* qctl = nullptr;                    // [3]
    unsigned long long* misc = nullptr;      // [16]
    LevelCounters* lc = nullptr;             // [MGK_MAX_HOPS+1]
    uint32_t* d_seeds = nullptr;             // staging for host calls
    unsigned long long* d_counts = nullptr;
    uint64_t seeds_cap = 0;
    uint64_t* h_pinned = nullptr;            // pinned, device-mapped host staging:
    uint32_t* h_seeds = nullptr;             //   [seeds_cap] uint32 seeds (device-readable)
    unsigned long long* h_counts = nullptr;  //   [seeds_cap] uint64 counts (device-writable)
    uint32_t* h_seeds_dev = nullptr;         // device addresses of the two regions
    unsigned long long* h_counts_dev = nullptr;
    uint64_t h_pinned_cap = 0;
    uint64_t bytes = 0;
    // last device-path launch (mgk_khop_device_stats)
    int misc_engine = 0, misc_W = 0;
    uint32_t misc_grid = 0, misc_block = 0;
    uint32_t last_launches = 0;  // engine kernels of the last call
    uint32_t last_path = 0;      // mgk_stats.path of the last call
    uint64_t misc_nseeds = 0;
};

struct Graph {
    int device = 0;
    DevGraph dg;
    uint32_t* rp = nullptr;
    uint32_t* ci = nullptr;
    uint32_t* cp = nullptr;
    uint32_t* ri = nullptr;
    uint32_t* no_in = nullptr;
    uint32_t* pull_skip = nullptr;
    uint2* heavy = nullptr;
    uint32_t* perm = nullptr;
    uint32_t* inv = nullptr;
    unsigned int* bad_seed = nullptr;
    uint64_t bytes = 0;
    // on-chip k = 2: per vertex, where its (ascending) row crosses each bitmap
    // slice boundary ([n][R-1] absolute col_idx positions), built on first use
    uint32_t* k2_split = nullptr;
    uint32_t k2_split_bits = 0, k2_split_R = 0;
    // LANES pull: the first four in-neighbours of every vertex (its in-list's
    // head, padded with its first entry), one dense uint4 per vertex, built on
    // first use -- a candidate's first frontier-word gathers then start with
    // its visited word and CSC bounds, from a coalesced load
    uint4* top4 = nullptr;
    Tuning tuning;
    std::mutex mu;
    std::vector<std::unique_ptr<Workspace>> free_ws;
    std::vector<Workspace*> all_ws;
    uint64_t ws_bytes = 0;
};

// ---- engine launch interface (mgk_ss.cu / mgk_ms.cu) ---------------------------
struct Launch {
    const Graph* g;
    Workspace* ws;
    const uint32_t* d_seeds;
    uint64_t nseeds;
    uint32_t k;             // max hop
    uint32_t min_hop;       // count hops [min_hop, k]
    uint32_t seed_visited;  // 1 for k_hop_*, 0 for walk_targets
    unsigned long long* d_counts;
    unsigned long long* d_counts1 = nullptr;  // on-chip k = 2 only: also the k = 1 answers
    // LANES only: further hop windows answered by the same traversal (the
    // harness's sections over one seed list, e.g. k = 3 and k = 6): window j
    // counts hops [xlo[j], xhi[j]] (xhi <= k, xlo >= min_hop) into xout[j]
    static constexpr int kMaxExtra = 7;
    uint32_t nextra = 0;
    uint32_t ans_lo = 0, ans_hi = 0;  // d_counts' own window when nextra > 0 (else [min_hop, k])
    uint32_t xlo[kMaxExtra] = {}, xhi[kMaxExtra] = {};
    unsigned long long* xout[kMaxExtra] = {};
    cudaStream_t stream;
    Tuning tuning;
    int lanes_words;  // LANES engine only
    int lane_bits = 64;  // LANES: 64 (lanes_words uint64 words per vertex), or 16 / 8 (one narrow word)
    bool keep_result = false;  // SINGLE: leave slot 0's bitmaps for k_hop_frontier
    // d_seeds / d_counts are mapped pinned HOST memory (host calls, SINGLE):
    // each group's seeds then travel inside its launch and the answers are
    // written straight to the host buffer (no copy operations)
    bool host_io = false;
    const uint32_t* h_seeds = nullptr;  // host view of d_seeds when host_io
    uint32_t grid = 0, block = 0;  // out
    uint32_t launches = 0;         // out: engine kernels launched
    uint32_t path = 0;             // out: 1 = the shared-memory k = 2 path
};

// Launches a persistent engine kernel: cooperative (all CTAs co-resident,
// guaranteed) unless MGK_NONCOOP=1 asks for a plain launch of the same
// occupancy-sized grid (for profilers that do not intercept cooperative
// launches; the grid still fits on an otherwise idle GPU).
cudaError_t launch_persistent(const void* fn, uint32_t grid, uint32_t block, void** args,
                              cudaStream_t stream);
cudaError_t launch_persistent_smem(const void* fn, uint32_t grid, uint32_t block, void** args, size_t smem,
                                   cudaStream_t stream);
cudaError_t launch_persistent_l2(const void* fn, uint32_t grid, uint32_t block, void** args, cudaStream_t stream,
                                 void* base, size_t bytes);

cudaError_t launch_single(Launch& L);
// SINGLE, k = 2 counts with the visited sets in shared memory (mgk_k2.cu)
bool k2_eligible(const Launch& L);
// would a k = 2 k_hop count of nseeds seeds on g take the on-chip path? (it can
// then also return the k = 1 answers of the same seeds: Launch::d_counts1)
bool k2_takes(const Graph* g, uint64_t nseeds, uint32_t min_hop);
cudaError_t launch_k2(Launch& L);
cudaError_t launch_lanes(Launch& L);
// Sorted ids of the last single-seed keep_result run: visited \ (visited
// after hop min-1), i.e. the union of the levels in the window.
cudaError_t single_result_ids(const Graph* g, Workspace* ws, uint32_t min_hop, bool seed_visited,
                              uint32_t seed, unsigned long long* d_ids, unsigned long long* d_n,
                              cudaStream_t s);

// In-place exclusive scan of data[0..n) (data must hold n+1 entries); *total
// (device) receives the sum.
cudaError_t exclusive_scan_u32(uint32_t* data, uint32_t n, unsigned long long* total,
                               cudaStream_t s);

cudaError_t ensure_single_ws(const Graph* g, Workspace* ws);
cudaError_t ensure_lanes_ws(const Graph* g, Workspace* ws, int W);

// graph build (mgk_graph.cu)
cudaError_t build_device_graph(Graph* g, const uint32_t* h_rp, const uint32_t* h_ci);
cudaError_t build_device_graph_from_edges(Graph* g, const uint32_t* h_src, const uint32_t* h_dst,
                                          uint64_t nedges);
cudaError_t build_device_graph_generated(Graph* g, uint32_t scale, uint32_t edge_factor, double a,
                                         double b, double c, uint64_t rng_seed, uint64_t target,
                                         int relabel);
void free_device_graph(Graph* g);
cudaError_t replicate_device_graph(const Graph* src, Graph* dst);
cudaError_t transpose_device_graph(const Graph* src, Graph* dst);
cudaError_t seed_degrees(const Graph* g, const uint32_t* h_seeds, uint64_t ns, uint32_t* h_deg);
// sort + unique (src << 32 | dst) keys into g (g->dg.n set; keys/alt hold m
// entries each and are consumed); cudaErrorInvalidValue if >= 2^32 remain
cudaError_t graph_from_keys(Graph* g, unsigned long long*& keys, unsigned long long*& alt, uint64_t m,
                            cudaStream_t s);
cudaError_t locality_relabel(Graph* g, cudaStream_t s);

// GRAPHSNAP1 (mgk_snapshot.cu): the reference's grammar checked sequentially on
// the host, and the GPU loader (empty *err on success)
namespace snap {
std::optional<std::string> check_all(std::string_view text, uint64_t* n_out, uint64_t* m_out);
cudaError_t load_to_graph(Graph* g, const char* text, uint64_t len, const char* relation, uint64_t* node_count,
                          std::string* err);
}  // namespace snap

// semiring mxm (mgk_mxm.cu): host CSR operands (validated by the caller)
namespace mx {
struct DevIn {
    uint64_t nrows = 0, ncols = 0;
    const uint64_t* rp = nullptr;
    const uint64_t* ci = nullptr;
    const int64_t* vals = nullptr;  // null = structural
};
cudaError_t run(int device, const DevIn& a, const DevIn& b, int semiring, const DevIn* mask, uint64_t max_chunk,
                mgk_matrix* out);
}  // namespace mx
// CSR / CSC in external ids into host buffers (un-relabelled when relabelled)
cudaError_t download_graph(const Graph* g, uint32_t* h_rp, uint32_t* h_ci, uint32_t* h_cp, uint32_t* h_ri);
// device ids (scattered from a bitmap) -> external ids, ascending
cudaError_t ids_to_external(const Graph* g, unsigned long long* d_ids, uint64_t n, cudaStream_t s);

// device R-MAT generator (mgk_gen.cu) and its host-drawn relabel permutation
cudaError_t gen_rmat_device(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                            uint64_t rng_seed, uint64_t target, int relabel, unsigned long long** d_keys,
                            uint64_t* m_out, uint64_t* n_out, cudaStream_t s);
void seeded_perm(uint64_t live, uint64_t rng_seed, std::vector<uint32_t>& perm);

}  // namespace mgk
