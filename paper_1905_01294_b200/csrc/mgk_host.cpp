// Host harness helpers behind the C ABI: the BASELINE.json bench graphs and
// pick_seeds. Not on the timed path; both arms of bench.py consume the same
// cleaned CSR these produce.
//
//   R-MAT edge recipe   proj/core/src/bench.cpp:107-137 (quadrant descent, one
//                       top-53-bit mt19937_64 draw per level, bench.cpp:37-39)
//   pick_seeds          proj/core/src/bench.cpp:200-218 (+ bounded_draw :42-48)
//
// Differences from rmat_generate, all required by BASELINE.json's configs:
// edges are generated in fixed-size chunks, chunk c drawing from its own
// mt19937_64 stream (seed mixed from rng_seed and c) so generation is
// parallel and still deterministic; self-loops and duplicates are removed;
// generation continues chunk by chunk until `target_unique` distinct edges
// exist, keeping the first `target_unique` distinct edges in generation order;
// ids can be permuted / renumbered with a seeded Fisher-Yates shuffle.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "mgk.h"

namespace mgk {
void set_last_error(const std::string& msg);  // mgk_capi.cpp
void seeded_perm(uint64_t live, uint64_t rng_seed, std::vector<uint32_t>& perm);  // mgk_gen.cu
}

namespace {

constexpr uint64_t kChunkEdges = 1u << 16;

unsigned nthreads_for(int threads) {
    unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    if (threads > 0) hc = (unsigned)threads;
    return std::min(hc, 64u);
}

template <typename F>
void par(unsigned nt, uint64_t n, F&& f) {
    if (nt <= 1 || n < 4096) {
        f(0, n, 0u);
        return;
    }
    std::vector<std::thread> ts;
    const uint64_t step = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const uint64_t a = t * step, b = std::min(n, a + step);
        if (a < b) ts.emplace_back([&f, a, b, t] { f(a, b, t); });
    }
    for (auto& t : ts) t.join();
}

uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

// Chunk c of the edge stream: kChunkEdges R-MAT edges, loops dropped, as
// (src << 32 | dst) keys in generation order.
void gen_chunk(uint32_t scale, double a, double b, double c, uint64_t rng_seed, uint64_t chunk,
               std::vector<uint64_t>& out, uint64_t count = kChunkEdges) {
    std::mt19937_64 rng(splitmix64(rng_seed * 0x2545F4914F6CDD1DULL + chunk));
    const double ab = a + b, abc = ab + c;
    out.clear();
    out.reserve(count);
    for (uint64_t e = 0; e < count; ++e) {
        uint32_t s = 0, d = 0;
        for (uint32_t level = 0; level < scale; ++level) {
            const double r = static_cast<double>(rng() >> 11) * 0x1.0p-53;
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
        if (s != d) out.push_back(((uint64_t)s << 32) | d);
    }
}

// Parallel sort of u64 keys: partition by the top bits into buckets, sort
// buckets concurrently.
void psort(std::vector<uint64_t>& v, unsigned nt, int key_bits) {
    const uint64_t n = v.size();
    if (n < (1u << 20) || nt <= 1) {
        std::sort(v.begin(), v.end());
        return;
    }
    const int bb = 12;
    const int shift = std::max(0, key_bits - bb);
    const size_t nb = (size_t)1 << bb;
    std::vector<std::vector<uint64_t>> hist(nt, std::vector<uint64_t>(nb, 0));
    const uint64_t step = (n + nt - 1) / nt;
    par(nt, n, [&](uint64_t a, uint64_t b, unsigned t) {
        auto& h = hist[t];
        for (uint64_t i = a; i < b; ++i) h[std::min<uint64_t>(v[i] >> shift, nb - 1)]++;
    });
    std::vector<uint64_t> start(nb + 1, 0);
    std::vector<std::vector<uint64_t>> pos(nt, std::vector<uint64_t>(nb, 0));
    uint64_t acc = 0;
    for (size_t k = 0; k < nb; ++k) {
        start[k] = acc;
        for (unsigned t = 0; t < nt; ++t) {
            pos[t][k] = acc;
            acc += hist[t][k];
        }
    }
    start[nb] = acc;
    std::vector<uint64_t> out(n);
    par(nt, n, [&](uint64_t a, uint64_t b, unsigned t) {
        (void)step;
        auto& p = pos[t];
        for (uint64_t i = a; i < b; ++i) out[p[std::min<uint64_t>(v[i] >> shift, nb - 1)]++] = v[i];
    });
    std::atomic<size_t> next{0};
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < nt; ++t)
        ts.emplace_back([&] {
            for (size_t k; (k = next.fetch_add(1)) < nb;)
                std::sort(out.begin() + start[k], out.begin() + start[k + 1]);
        });
    for (auto& t : ts) t.join();
    v.swap(out);
}

void unique_sorted(std::vector<uint64_t>& v) { v.erase(std::unique(v.begin(), v.end()), v.end()); }

struct GenCache {
    uint64_t n = 0;
    std::vector<uint32_t> rp, ci;
    uint64_t key[9] = {0};
    bool valid = false;
};
thread_local GenCache t_gen;

int gen_graph(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t rng_seed,
              uint64_t target_unique, int relabel, int threads, GenCache& out) {
    const unsigned nt = nthreads_for(threads);
    const uint64_t ids = 1ull << scale;
    const int kb = 32 + (int)scale;  // keys are (src << 32 | dst)
    // ---- 1. the edge stream, deduplicated ------------------------------------
    std::vector<uint64_t> S;  // sorted unique keys so far
    uint64_t next_chunk = 0;
    const uint64_t raw_target = (uint64_t)edge_factor << scale;
    if (target_unique == 0) {
        // exactly edge_factor << scale raw draws (the last chunk truncated)
        const uint64_t nchunks = (raw_target + kChunkEdges - 1) / kChunkEdges;
        std::vector<std::vector<uint64_t>> chunks(nchunks);
        std::atomic<uint64_t> cur{0};
        std::vector<std::thread> ts;
        for (unsigned t = 0; t < nt; ++t)
            ts.emplace_back([&] {
                for (uint64_t ch; (ch = cur.fetch_add(1)) < nchunks;) {
                    const uint64_t cnt = std::min(kChunkEdges, raw_target - ch * kChunkEdges);
                    gen_chunk(scale, a, b, c, rng_seed, ch, chunks[ch], cnt);
                }
            });
        for (auto& t : ts) t.join();
        size_t total = 0;
        for (auto& v : chunks) total += v.size();
        S.reserve(total);
        for (auto& v : chunks) S.insert(S.end(), v.begin(), v.end());
        psort(S, nt, kb);
        unique_sorted(S);
    } else {
        uint64_t want = target_unique + target_unique / 50 + kChunkEdges;
        while (S.size() < target_unique) {
            const uint64_t nchunks = (want + kChunkEdges - 1) / kChunkEdges;
            std::vector<std::vector<uint64_t>> chunks(nchunks);
            std::atomic<uint64_t> cur{0};
            std::vector<std::thread> ts;
            for (unsigned t = 0; t < nt; ++t)
                ts.emplace_back([&] {
                    for (uint64_t ch; (ch = cur.fetch_add(1)) < nchunks;)
                        gen_chunk(scale, a, b, c, rng_seed, next_chunk + ch, chunks[ch]);
                });
            for (auto& t : ts) t.join();
            next_chunk += nchunks;
            std::vector<uint64_t> N;
            size_t total = 0;
            for (auto& v : chunks) total += v.size();
            N.reserve(total);
            for (auto& v : chunks) N.insert(N.end(), v.begin(), v.end());
            psort(N, nt, kb);
            unique_sorted(N);
            std::vector<uint64_t> fresh;
            fresh.reserve(N.size());
            std::set_difference(N.begin(), N.end(), S.begin(), S.end(), std::back_inserter(fresh));
            if (S.size() + fresh.size() <= target_unique) {
                std::vector<uint64_t> merged(S.size() + fresh.size());
                std::merge(S.begin(), S.end(), fresh.begin(), fresh.end(), merged.begin());
                S.swap(merged);
            } else {
                // keep the first (target - |S|) new distinct keys in generation order
                const uint64_t need = target_unique - S.size();
                std::vector<char> taken(fresh.size(), 0);
                std::vector<uint64_t> keep;
                keep.reserve(need);
                for (auto& v : chunks) {
                    for (uint64_t key : v) {
                        auto it = std::lower_bound(fresh.begin(), fresh.end(), key);
                        if (it == fresh.end() || *it != key) continue;
                        char& t = taken[it - fresh.begin()];
                        if (t) continue;
                        t = 1;
                        keep.push_back(key);
                        if (keep.size() == need) break;
                    }
                    if (keep.size() == need) break;
                }
                std::sort(keep.begin(), keep.end());
                std::vector<uint64_t> merged(S.size() + keep.size());
                std::merge(S.begin(), S.end(), keep.begin(), keep.end(), merged.begin());
                S.swap(merged);
            }
            // deficit-driven next round (R-MAT's duplicate rate grows with density)
            want = (target_unique > S.size() ? (target_unique - S.size()) * 2 : 0) + kChunkEdges;
        }
    }
    // ---- 2. relabel ---------------------------------------------------------------
    uint64_t n = ids;
    if (relabel != 0) {
        std::vector<uint32_t> map(ids, 0xFFFFFFFFu);
        uint64_t live = ids;
        if (relabel == 2) {
            std::vector<uint8_t> seen(ids, 0);
            par(nt, S.size(), [&](uint64_t x, uint64_t y, unsigned) {
                for (uint64_t i = x; i < y; ++i) {
                    // benign races: every writer stores 1
                    seen[S[i] >> 32] = 1;
                    seen[S[i] & 0xFFFFFFFFu] = 1;
                }
            });
            live = 0;
            for (uint64_t v = 0; v < ids; ++v)
                if (seen[v]) map[v] = (uint32_t)live++;
        } else {
            for (uint64_t v = 0; v < ids; ++v) map[v] = (uint32_t)v;
        }
        // seeded Fisher-Yates over the live ids (shared with the device generator)
        std::vector<uint32_t> perm;
        mgk::seeded_perm(live, rng_seed, perm);
        par(nt, S.size(), [&](uint64_t x, uint64_t y, unsigned) {
            for (uint64_t i = x; i < y; ++i) {
                const uint64_t s = perm[map[S[i] >> 32]], d = perm[map[S[i] & 0xFFFFFFFFu]];
                S[i] = (s << 32) | d;
            }
        });
        int bits = 1;
        while (bits < 32 && (1ull << bits) < live) ++bits;
        psort(S, nt, 32 + bits);
        n = live;
    }
    // ---- 3. CSR ------------------------------------------------------------------------
    if (n >= 0xFFFFFFFFull || S.size() >= 0xFFFFFFFFull) {
        mgk::set_last_error("generated graph exceeds uint32 indices");
        return MGK_ERANGE;
    }
    out.n = n;
    out.rp.assign(n + 1, 0);
    out.ci.resize(S.size());
    par(nt, S.size(), [&](uint64_t x, uint64_t y, unsigned) {
        for (uint64_t i = x; i < y; ++i) out.ci[i] = (uint32_t)(S[i] & 0xFFFFFFFFu);
    });
    for (uint64_t i = 0; i < S.size(); ++i) out.rp[(S[i] >> 32) + 1]++;
    for (uint64_t v = 0; v < n; ++v) out.rp[v + 1] += out.rp[v];
    return MGK_OK;
}

}  // namespace

extern "C" {

int mgk_gen_rmat_csr(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                     uint64_t rng_seed, uint64_t target_unique, int relabel, int threads,
                     uint64_t* n_out, uint64_t* nnz_out, uint32_t* row_ptr, uint32_t* col_idx) {
    if (scale < 1 || scale > 31) {
        mgk::set_last_error("RMAT scale must be in [1, 31]");
        return MGK_ECONTRACT;
    }
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0 + 1e-9) {
        mgk::set_last_error("RMAT quadrant probabilities must be non-negative and sum to at most 1");
        return MGK_ECONTRACT;
    }
    if (relabel < 0 || relabel > 2) {
        mgk::set_last_error("relabel must be 0, 1 or 2");
        return MGK_ECONTRACT;
    }
    const uint64_t key[9] = {scale, edge_factor, (uint64_t)(a * 1e12), (uint64_t)(b * 1e12),
                             (uint64_t)(c * 1e12), rng_seed, target_unique, (uint64_t)relabel, 1};
    GenCache& gc = t_gen;
    if (!gc.valid || std::memcmp(gc.key, key, sizeof key) != 0) {
        gc.valid = false;
        gc.rp.clear();
        gc.ci.clear();
        int rc = gen_graph(scale, edge_factor, a, b, c, rng_seed, target_unique, relabel, threads, gc);
        if (rc) return rc;
        std::memcpy(gc.key, key, sizeof key);
        gc.valid = true;
    }
    if (n_out) *n_out = gc.n;
    if (nnz_out) *nnz_out = gc.ci.size();
    if (row_ptr) std::memcpy(row_ptr, gc.rp.data(), gc.rp.size() * 4);
    if (col_idx && !gc.ci.empty()) std::memcpy(col_idx, gc.ci.data(), gc.ci.size() * 4);
    if (row_ptr) {  // second phase done: drop the cache
        gc.valid = false;
        std::vector<uint32_t>().swap(gc.rp);
        std::vector<uint32_t>().swap(gc.ci);
    }
    return MGK_OK;
}

int mgk_pick_seeds_csr(uint64_t nrows, const uint32_t* row_ptr, uint64_t n, uint64_t rng_seed,
                       uint64_t* out) {
    std::vector<uint64_t> eligible;
    for (uint64_t id = 0; id < nrows; ++id)
        if (row_ptr[id + 1] > row_ptr[id]) eligible.push_back(id);
    if (eligible.size() < n) {
        char buf[160];
        snprintf(buf, sizeof buf, "need %llu seeds but only %llu nodes have out-degree >= 1",
                 (unsigned long long)n, (unsigned long long)eligible.size());
        mgk::set_last_error(buf);
        return MGK_EHARNESS;
    }
    std::mt19937_64 rng(rng_seed);
    const uint64_t max = UINT64_MAX;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t bound = eligible.size() - i, limit = max - max % bound;
        uint64_t draw = rng();
        while (draw >= limit) draw = rng();
        std::swap(eligible[i], eligible[i + draw % bound]);
    }
    std::memcpy(out, eligible.data(), n * 8);
    return MGK_OK;
}

int mgk_snapshot_write_csr(uint64_t node_count, const uint32_t* row_ptr, const uint32_t* col_idx,
                           const char* relation, int id_props, char* out, uint64_t cap, uint64_t* n_out) {
    if (!row_ptr || !relation || !n_out || (cap && !out)) {
        mgk::set_last_error("null argument");
        return MGK_ECONTRACT;
    }
    // per-row byte counts (node line + its edge lines), then a prefix sum, so
    // every thread can format its rows in place
    const std::string rel(relation);
    auto digits = [](uint64_t v) {
        int d = 1;
        while (v >= 10) v /= 10, ++d;
        return (uint64_t)d;
    };
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<uint64_t> node_bytes(node_count + 1, 0), edge_bytes(node_count + 1, 0);
    auto par = [&](auto&& f) {
        std::vector<std::thread> ts;
        const uint64_t step = (node_count + nt - 1) / nt;
        for (unsigned t = 0; t < nt; ++t) {
            const uint64_t a = t * step, b = std::min<uint64_t>(node_count, a + step);
            if (a < b) ts.emplace_back([&f, a, b] { f(a, b); });
        }
        for (auto& t : ts) t.join();
    };
    par([&](uint64_t a, uint64_t b) {
        for (uint64_t v = a; v < b; ++v) {
            const uint64_t dv = digits(v);
            node_bytes[v] = dv + 2 + (id_props ? 5 + dv : 0) + 1;  // "v\t\tid:i:v\n"
            uint64_t eb = 0;
            for (uint32_t p = row_ptr[v]; p < row_ptr[v + 1]; ++p)
                eb += dv + 1 + rel.size() + 1 + digits(col_idx[p]) + 2;  // "v\tREL\tu\t\n"
            edge_bytes[v] = eb;
        }
    });
    const std::string head = "GRAPHSNAP1\nNODES " + std::to_string(node_count) + "\n";
    const std::string mid = "EDGES " + std::to_string(node_count ? (uint64_t)row_ptr[node_count] : 0) + "\n";
    uint64_t nb = 0, eb = 0;
    for (uint64_t v = 0; v < node_count; ++v) {
        const uint64_t x = node_bytes[v], y = edge_bytes[v];
        node_bytes[v] = nb, edge_bytes[v] = eb;
        nb += x, eb += y;
    }
    const uint64_t total = head.size() + nb + mid.size() + eb;
    *n_out = total;
    if (!out) return MGK_OK;
    if (cap < total) {
        mgk::set_last_error("output buffer too small");
        return MGK_ECONTRACT;
    }
    std::memcpy(out, head.data(), head.size());
    char* nodes = out + head.size();
    std::memcpy(nodes + nb, mid.data(), mid.size());
    char* edges = nodes + nb + mid.size();
    par([&](uint64_t a, uint64_t b) {
        char num[24];
        for (uint64_t v = a; v < b; ++v) {
            const int dv = snprintf(num, sizeof num, "%llu", (unsigned long long)v);
            char* p = nodes + node_bytes[v];
            std::memcpy(p, num, dv), p += dv;
            *p++ = '\t', *p++ = '\t';
            if (id_props) std::memcpy(p, "id:i:", 5), p += 5, std::memcpy(p, num, dv), p += dv;
            *p++ = '\n';
            char* q = edges + edge_bytes[v];
            for (uint32_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
                std::memcpy(q, num, dv), q += dv;
                *q++ = '\t';
                std::memcpy(q, rel.data(), rel.size()), q += rel.size();
                *q++ = '\t';
                q += snprintf(q, 24, "%u", col_idx[e]);
                *q++ = '\t', *q++ = '\n';
            }
        }
    });
    return MGK_OK;
}

}  // extern "C"
