/*
 * mgk — the B200 k-hop count engine behind a plain C ABI.
 *
 * This is the drop-in boundary for the reference's k-hop hot path
 * (matgraph, /root/reference/proj). Every entry point names the reference
 * interface it replaces. No exceptions and no C++/torch types cross this
 * boundary: plain pointers, sizes and int status codes, with the message of
 * the last failure on this thread in mgk_last_error().
 *
 * Semantics are the reference's, bit for bit:
 *   k_hop_frontier  proj/core/src/execute.cpp:347-371
 *       frontier = visited = {seed}; for hop 1..k:
 *           frontier = vxm(frontier, A, mask = NOT visited)   (sparse.cpp:253-290)
 *           if frontier empty: break
 *           visited = ewise_union(visited, frontier)          (sparse.cpp:365-377)
 *       exact      -> frontier   (vertices at shortest distance exactly k)
 *       cumulative -> visited \ {seed}  (distance 1..k)
 *   k_hop_count     proj/core/src/execute.cpp:373-375  = nvals(k_hop_frontier)
 *
 * Status codes follow the reference's error classes
 * (proj/core/include/matgraph/error.hpp:10-66): MGK_ECONTRACT <-> ContractError
 * with the reference's exact message text, MGK_EHARNESS <-> HarnessError,
 * everything else maps to matgraph::Error.
 */
#ifndef MGK_H
#define MGK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGK_ABI_VERSION 2

/* status codes */
#define MGK_OK 0
#define MGK_ECONTRACT 1 /* precondition violated (ContractError): bad seed, k, sizes */
#define MGK_EHARNESS 2  /* harness setup failure (HarnessError), e.g. too few seeds */
#define MGK_ECUDA 3     /* CUDA runtime / launch failure (matgraph::Error) */
#define MGK_ENOMEM 4    /* device or host allocation failed */
#define MGK_ERANGE 5    /* graph exceeds uint32 device indices (n or nnz >= 2^32) */
#define MGK_ESNAPSHOT 6 /* malformed GRAPHSNAP1 text (SnapshotError): "snapshot parse error at line N: ..." */

/* TraverseMode, proj/core/include/matgraph/plan.hpp:17 */
#define MGK_EXACT 0
#define MGK_CUMULATIVE 1

/* traversal engines */
#define MGK_ENGINE_AUTO 0   /* k <= 2 or one seed -> SINGLE, else LANES */
#define MGK_ENGINE_SINGLE 1 /* bitmap direction-optimizing BFS, one seed at a time */
#define MGK_ENGINE_LANES 2  /* bit-parallel multi-source: 64 seeds per uint64 lane word */

#define MGK_MAX_HOPS 32 /* kMaxHops, proj/core/include/matgraph/ast.hpp:15 */

typedef struct mgk_graph mgk_graph;
typedef struct mgk_matrix mgk_matrix; /* a host CSR result (mgk_mxm) */

/* Per-level work counters of one call (summed over seeds / batches). */
typedef struct mgk_level {
    uint64_t frontier;    /* (seed, vertex) pairs discovered at this hop: sum of |F_l| */
    uint64_t vertices;    /* distinct vertices discovered (LANES: |union of lane frontiers|) */
    uint64_t edges;       /* push-equivalent edges E: sum over seeds of outdeg(F_{l-1}) */
    uint64_t union_edges; /* edges of the distinct frontier vertices (what a push pass reads) */
    uint64_t scanned;     /* adjacency entries the kernel actually read at this hop */
    uint64_t candidates;  /* pull: unvisited candidate vertices examined */
    uint32_t runs;        /* seeds (SINGLE) or batches (LANES) that expanded this hop */
    uint32_t pull_runs;   /* ... of which ran the hop in the pull (CSC) direction */
    uint64_t ns;          /* device time in this hop (%globaltimer, summed over runs) */
} mgk_level;

typedef struct mgk_stats {
    uint32_t engine;       /* MGK_ENGINE_SINGLE or MGK_ENGINE_LANES */
    uint32_t lanes;        /* seeds per batch (LANES) or 1 */
    uint32_t batches;      /* batches (LANES) or seeds (SINGLE) */
    uint32_t hops;         /* deepest hop expanded by any run */
    uint32_t grid;         /* persistent CTAs launched */
    uint32_t block;        /* threads per CTA */
    uint32_t launches;     /* kernel launches the call made */
    uint32_t path;         /* SINGLE: 0 = per-seed bitmaps in L2 (fr_kernel), 1 = k = 2 with the
                              visited sets in shared memory (k2_kernel) */
    double kernel_ms;      /* CUDA-event time of the traversal launch(es) */
    uint64_t setup_ns;     /* device time clearing counters + seeding hop 0 */
    uint64_t cleanup_ns;   /* device time returning the workspace to all-zero */
    mgk_level level[MGK_MAX_HOPS + 1];
} mgk_stats;

/* ---- graph lifetime ---------------------------------------------------------
 * Replaces the read side of PropertyGraph::relation_matrix
 * (proj/core/src/graph.cpp:84-88) and transposed_matrix (:90-102): the CSR of
 * one relation (or ANY) is uploaded once, narrowed to uint32, and the CSC
 * (= CSR of A^T, sparse.cpp:379-403) is built on the device. `nrows` is the
 * matrix dimension (the store's capacity, graph.cpp:26); `row_ptr` has nrows+1
 * entries and `col_idx` nnz entries with strictly ascending columns per row
 * (the SparseMatrix invariant, sparse.hpp:80-82). Checked: row_ptr monotone,
 * row_ptr[nrows] == nnz, columns < nrows. */
int mgk_graph_upload(int device, uint64_t nrows, uint64_t nnz, const uint64_t* row_ptr,
                     const uint64_t* col_idx, mgk_graph** out);
/* Same from uint32 arrays (the bench graphs; m < 2^32). */
int mgk_graph_upload_u32(int device, uint64_t nrows, uint64_t nnz, const uint32_t* row_ptr,
                         const uint32_t* col_idx, mgk_graph** out);
/* Build the device graph straight from an edge list: sort, drop duplicates
 * (PropertyGraph::flush_slot, graph.cpp:182-215) and assemble CSR + CSC on the
 * GPU. Self-loops are kept (they never change a count). Endpoints must be
 * < nrows (build_bench_graph's ContractError, bench.cpp:189-193). */
int mgk_graph_from_edges(int device, uint64_t nrows, uint64_t nedges, const uint32_t* src,
                         const uint32_t* dst, mgk_graph** out);
/* Generate a BASELINE.json bench graph directly on the device: the same edge
 * set and ids as mgk_gen_rmat_csr below (same chunked mt19937_64 stream,
 * first `target_unique` distinct non-loop edges, same seeded relabelling),
 * with sort / dedup / CSR / CSC on the GPU. Download with
 * mgk_graph_download_csr. (BASELINE cfg4: 1.47B edges in seconds.) */
int mgk_graph_gen_rmat(int device, uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                       uint64_t rng_seed, uint64_t target_unique, int relabel, mgk_graph** out);
/* GRAPHSNAP1 load (snapshot_from_string / snapshot_load, snapshot.cpp:162-259,
 * then relation_matrix): the text is parsed on the GPU, one thread per line,
 * and the edges of `relation` (NULL = ANY) become the device CSR + CSC. The
 * matrix dimension is the store's capacity max(NODES, 16) (graph.cpp:15-30);
 * *node_count receives NODES (seeds are checked against it by callers, like
 * KHopQuery against node_count). Labels and properties are validated, not
 * kept. A malformed text fails with MGK_ESNAPSHOT and the reference's exact
 * SnapshotError message; a missing file with "cannot open '<path>' for reading".
 * mgk_snapshot_check runs the same grammar on the host only (no GPU). */
int mgk_graph_load_snapshot(int device, const char* text, uint64_t len, const char* relation,
                            mgk_graph** out, uint64_t* node_count);
int mgk_graph_load_snapshot_file(int device, const char* path, const char* relation, mgk_graph** out,
                                 uint64_t* node_count);
int mgk_snapshot_check(const char* text, uint64_t len, uint64_t* node_count, uint64_t* edge_count);
/* The transpose A^T as its own device graph (transposed_matrix, graph.cpp:90-102;
 * transpose, sparse.cpp:379-403), built on the device from g's arrays: walks
 * and k-hop counts over it follow edges backwards (the `<-` direction of a
 * Cypher pattern, execute.cpp:35-39). Free with mgk_graph_free. */
int mgk_graph_transpose(const mgk_graph* g, mgk_graph** out);
int mgk_graph_free(mgk_graph* g);
int mgk_graph_info(const mgk_graph* g, uint64_t* nrows, uint64_t* nnz, int* device);
/* Copy the device CSR back (uint32; either pointer may be NULL). */
int mgk_graph_download_csr(const mgk_graph* g, uint32_t* row_ptr, uint32_t* col_idx);
int mgk_graph_download_csc(const mgk_graph* g, uint32_t* col_ptr, uint32_t* row_idx);
/* Device memory held by the graph and its workspaces, in bytes. */
uint64_t mgk_graph_device_bytes(const mgk_graph* g);

/* ---- the hot path -------------------------------------------------------------
 * k_hop_count for a batch of seeds (execute.cpp:373-375 once per seed).
 * HOST buffers: seeds[nseeds] (uint64 node ids, as KHopQuery::seed), counts[nseeds].
 * Errors (checked before any device work, in seed order):
 *   seed >= nrows  -> MGK_ECONTRACT "k-hop seed {s} is not an allocated node"
 *   k outside 1..32 -> MGK_ECONTRACT "k-hop count {k} outside [1, 32]"
 * (execute.cpp:348-354). Reentrant: concurrent calls on one graph use separate
 * workspaces and streams. `stats` may be NULL. */
int mgk_khop_count(mgk_graph* g, const uint64_t* seeds, uint64_t nseeds, uint32_t k, int mode,
                   uint64_t* counts);
int mgk_khop_count_ex(mgk_graph* g, const uint64_t* seeds, uint64_t nseeds, uint32_t k, int mode,
                      int engine, uint64_t* counts, mgk_stats* stats);

/* Several hop counts for one seed list in one call (the harness's sections
 * over one master seed list, bench.cpp:311-343): counts[j * nseeds + i] is
 * k_hop_count(seeds[i], ks[j]). All windows are enqueued back to back and
 * answered with one synchronisation. Checked like mgk_khop_count, per k. */
int mgk_khop_count_ks(mgk_graph* g, const uint64_t* seeds, uint64_t nseeds, const uint32_t* ks, uint32_t nks,
                      int mode, uint64_t* counts);

/* ---- multi-GPU: seed-sharded replicas, no collective ----------
 * mgk_graph_replicate copies a device graph to `device` (cudaMemcpyPeer over
 * NVLink / NVSwitch when the devices differ; a plain device copy otherwise):
 * load-time replication instead of re-uploading from the host.
 * mgk_khop_count_multi answers one batch over nreplicas replicas of the same
 * graph: the seeds are split into shards — cost-balanced by out-degree
 * (longest first) when the per-seed engine runs (k <= 2), contiguous for the
 * lane engine — one host thread and the replica's own stream per shard, each
 * writing disjoint entries of counts.
 * Same validation and messages as mgk_khop_count (checked once, in seed order,
 * before any device work). Replaces the "mgk_khop_count_multi_gpu" entry
 * SURVEY §8(b) lists; the reference has no multi-device path. */
int mgk_graph_replicate(const mgk_graph* src, int device, mgk_graph** out);
int mgk_khop_count_multi(mgk_graph* const* replicas, int nreplicas, const uint64_t* seeds, uint64_t nseeds,
                         uint32_t k, int mode, uint64_t* counts);

/* ---- semiring matrix product ----------------------------
 * mxm (sparse.cpp:292-363): C = A (+.*) B over bool_or_and (structural
 * result), plus_times or min_plus (int64 values; a NULL value array is a
 * structural operand multiplying as all-ones), optionally restricted to the
 * pattern of a structural mask (m_row_ptr NULL = no mask). Computed on the GPU
 * (expand / radix sort / reduce in row chunks); columns come out ascending per
 * row and values are bit-identical to the reference (wrapping int64).
 * Errors (MGK_ECONTRACT, the reference's text):
 *   "mxm: inner dimensions disagree ({}x{} times {}x{})"
 *   "mxm: mask shape {}x{} != result shape {}x{}"
 * The result is a handle: query sizes, download, free. Like from_parts, a
 * valued product with no entries reports valued = 0. */
#define MGK_SEMIRING_BOOL_OR_AND 0
#define MGK_SEMIRING_PLUS_TIMES 1
#define MGK_SEMIRING_MIN_PLUS 2
int mgk_mxm(int device, uint64_t a_nrows, uint64_t a_ncols, const uint64_t* a_row_ptr, const uint64_t* a_col_idx,
            const int64_t* a_vals, uint64_t b_nrows, uint64_t b_ncols, const uint64_t* b_row_ptr,
            const uint64_t* b_col_idx, const int64_t* b_vals, int semiring, uint64_t m_nrows, uint64_t m_ncols,
            const uint64_t* m_row_ptr, const uint64_t* m_col_idx, mgk_matrix** out);
int mgk_matrix_info(const mgk_matrix* m, uint64_t* nrows, uint64_t* ncols, uint64_t* nnz, int* valued);
int mgk_matrix_download(const mgk_matrix* m, uint64_t* row_ptr, uint64_t* col_idx, int64_t* vals);
int mgk_matrix_free(mgk_matrix* m);

/* Device-resident variant: d_seeds (uint32) and d_counts (uint64) are DEVICE
 * pointers on the graph's device; work is enqueued on `stream`
 * (a cudaStream_t, NULL = legacy default) and returns without synchronizing.
 * Seeds are not range-checked on the host on this path (the caller owns
 * them): the kernels flag a seed >= nrows instead, reported by
 * mgk_khop_device_check / mgk_khop_device_stats (see there). Calls on one stream share one workspace
 * and serialize on that stream. */
int mgk_khop_count_device(mgk_graph* g, const uint32_t* d_seeds, uint64_t nseeds, uint32_t k,
                          int mode, int engine, uint64_t* d_counts, void* stream);
/* Device-path sections (the harness's k sections over one seed list,
 * bench.cpp:311-343, device-resident like mgk_khop_count_device): the answers
 * for ks[j] go to d_counts[j * nseeds + i]. A k = 1 section is answered by the
 * k = 2 launch when that one runs on the on-chip path (|F1| is part of it).
 * k is checked like mgk_khop_count_device; seeds are not. */
int mgk_khop_count_device_ks(mgk_graph* g, const uint32_t* d_seeds, uint64_t nseeds, const uint32_t* ks,
                             uint32_t nks, int mode, uint64_t* d_counts, void* stream);
/* The harness's whole schedule in one call (run_khop_benchmark,
 * bench.cpp:311-343, with one master seed list sized by the largest request):
 * section j = k_hop_count(seeds[i], ks[j]) for i < nseeds_per_k[j] (a prefix
 * of the master list, like pick_seeds' prefix-stable list). counts holds the
 * sections back to back: section j starts at sum_{j' < j} nseeds_per_k[j'].
 * Checks: the schedule first (bench.cpp:297-309: "hop count {k} outside [1,
 * 32]", "seed count for k={k} must be at least 1"), then every query like
 * mgk_khop_count. Consecutive sections with equal seed counts share launches:
 * a k = 1 section rides on the on-chip k = 2 launch, and LANES sections of the
 * same seeds (e.g. k = 3 and k = 6) share one traversal, each answered from
 * its own hops' per-lane counts. The _device_ variant takes device seeds /
 * counts and a stream like mgk_khop_count_device (no host-side seed check). */
int mgk_khop_count_schedule(mgk_graph* g, const uint64_t* seeds, const uint64_t* nseeds_per_k, const uint32_t* ks,
                            uint32_t nks, int mode, uint64_t* counts);
int mgk_khop_count_device_schedule(mgk_graph* g, const uint32_t* d_seeds, const uint64_t* nseeds_per_k,
                                   const uint32_t* ks, uint32_t nks, int mode, uint64_t* d_counts, void* stream);

/* Work counters of the last device-path call on `stream` (waits for that stream;
 * kernel_ms is 0 on this path — time it with your own events). Also performs
 * the check of mgk_khop_device_check. */
int mgk_khop_device_stats(mgk_graph* g, void* stream, mgk_stats* stats);
/* Waits for `stream` and reports the device path's seed check: when any
 * device-path call on this graph since the last check met a seed >= nrows,
 * returns MGK_ECONTRACT (the reference's "not an allocated node" contract,
 * execute.cpp:348-351) and clears the flag. Such a seed is read as vertex 0
 * on the device (no out-of-bounds access); the answers of that call are
 * undefined. */
int mgk_khop_device_check(mgk_graph* g, void* stream);

/* k_hop_frontier (execute.cpp:347-371): the sorted ids of the result set.
 * Writes min(*n_out, cap) ids; *n_out = total. Same checks as above. */
int mgk_khop_frontier(mgk_graph* g, uint64_t seed, uint32_t k, int mode, uint64_t* ids,
                      uint64_t cap, uint64_t* n_out);

/* walk_targets (execute.cpp:43-60, the Cypher VarLenTraverse step behind
 * MATCH (a)-[*min..max]->(b)): the same masked traversal but with the visited
 * set starting EMPTY, so the source itself is reached again on a cycle;
 * counts / sorted ids of the union of levels min..max. Window checks follow
 * the Cypher parser (cypher.cpp:356-392): "hop minimum must be at least 1",
 * "hop count {h} exceeds the cap of 32", "hop maximum {max} is less than
 * minimum {min}"; an unallocated source is MGK_ECONTRACT. */
int mgk_walk_count(mgk_graph* g, const uint64_t* sources, uint64_t nsources, uint32_t min_hops,
                   uint32_t max_hops, int engine, uint64_t* counts);
int mgk_walk_targets(mgk_graph* g, uint64_t source, uint32_t min_hops, uint32_t max_hops, uint64_t* ids,
                     uint64_t cap, uint64_t* n_out);

/* Engine tuning knobs (0 keeps the default). alpha/beta: Beamer-style
 * push->pull when frontier edges * alpha > unexplored in-edges, pull->push
 * when frontier * beta < n (alpha for SINGLE, alpha_lanes for LANES).
 * force_dir: 0 auto, 1 push only, 2 pull only (tests use it to pin both
 * directions to the same answers). lanes_words: 64-lane words per vertex in
 * the LANES engine (1, 2, 4 or 8; 0 = auto). */
typedef struct mgk_tuning {
    uint32_t alpha;
    uint32_t beta;
    uint32_t force_dir;
    uint32_t lanes_words;
    uint32_t alpha_lanes;
    uint32_t alpha_last;  /* SINGLE, last hop: push -> pull when frontier edges * alpha_last > unexplored */
} mgk_tuning;
int mgk_graph_set_tuning(mgk_graph* g, const mgk_tuning* t);
int mgk_graph_get_tuning(const mgk_graph* g, mgk_tuning* t);

const char* mgk_last_error(void);
int mgk_abi_version(void);
int mgk_device_count(void);

/* ---- harness helpers (host C++; not on the timed path) ---------------------
 * The bench graphs of BASELINE.json: the reference's R-MAT recipe
 * (proj/core/src/bench.cpp:107-137: per level one 53-bit uniform draw from
 * mt19937_64, quadrant a/b/c/d) run in fixed-size chunks, each chunk with its
 * own mt19937_64 stream seeded from (rng_seed, chunk), until `target_unique`
 * distinct non-loop edges exist (0 = emit exactly edge_factor << scale raw
 * edges, like rmat_generate). relabel: 0 none, 1 seeded random permutation of
 * all 2^scale ids, 2 drop isolated ids and renumber survivors by a seeded
 * permutation. Output: deduplicated, loop-free CSR (uint32), *n_out vertices.
 * Two-phase: call with row_ptr = NULL to learn *n_out / *nnz_out sizes
 * (the generated graph is cached per thread for the second call). */
int mgk_gen_rmat_csr(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                     uint64_t rng_seed, uint64_t target_unique, int relabel, int threads,
                     uint64_t* n_out, uint64_t* nnz_out, uint32_t* row_ptr, uint32_t* col_idx);
/* pick_seeds (bench.cpp:200-218) over a uint32 CSR: eligible = ids with a
 * non-empty row, partial Fisher-Yates with mt19937_64(rng_seed) and
 * rejection-sampled draws. MGK_EHARNESS
 * "need {n} seeds but only {e} nodes have out-degree >= 1" when short. */
int mgk_pick_seeds_csr(uint64_t nrows, const uint32_t* row_ptr, uint64_t n, uint64_t rng_seed,
                       uint64_t* out);
/* snapshot_to_string (snapshot.cpp:127-160) of a one-relation graph given as a
 * CSR over node_count nodes without labels, each node carrying {"id": i} when
 * id_props != 0 (exactly what build_bench_graph stores, bench.cpp:185-198):
 * byte-identical to the reference writer for such graphs. Call with out=NULL
 * for the size. Host only (multi-threaded). */
int mgk_snapshot_write_csr(uint64_t node_count, const uint32_t* row_ptr, const uint32_t* col_idx,
                           const char* relation, int id_props, char* out, uint64_t cap, uint64_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* MGK_H */
