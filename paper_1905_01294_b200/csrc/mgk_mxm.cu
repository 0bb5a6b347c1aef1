// Semiring sparse matrix product on the GPU.
//
// Replaces mxm (proj/core/src/sparse.cpp:292-363): C = A (+.*) B over the
// reference's three semirings -- bool_or_and (structural result), plus_times
// and min_plus (int64 values; a structural operand multiplies as all-ones) --
// with an optional structural mask restricting the result pattern. The
// reference runs Gustavson row by row with a dense accumulator; here it is
// expand / sort / compress over the whole product, in row chunks that bound
// the expanded size:
//   1. per A entry (i, k): |B[k]| products; an exclusive scan gives each
//      entry its output slot (the chunk's "flops");
//   2. one thread per product writes key (i << 32 | j) and the semiring
//      product a_ik * b_kj, dropping (i, j) outside the mask;
//   3. radix sort by key, then reduce equal keys with the semiring's add
//      (boolean: unique) -- rows come out with ascending columns, exactly the
//      reference's sorted `touched` list.
// Plus / times wrap modulo 2^64 like the reference's int64 arithmetic, and
// add is associative and commutative, so results are bit-identical in any
// summation order.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "mgk_internal.cuh"

// The result stays on the device until the caller downloads it (one copy,
// straight into the caller's arrays); row_ptr is small and kept on the host.
struct mgk_matrix {
    int device = 0;
    uint64_t nrows = 0, ncols = 0, nnz = 0;
    bool valued = false;
    std::vector<uint64_t> row_ptr;
    unsigned long long* d_col = nullptr;  // [nnz] (uint64 columns)
    long long* d_vals = nullptr;          // [nnz] when valued
    ~mgk_matrix() {
        cudaFree(d_col);
        cudaFree(d_vals);
    }
};

namespace mgk {
namespace mx {
namespace {

#define MX_TRY(x)                           \
    do {                                    \
        if ((e = (x)) != cudaSuccess) goto done; \
    } while (0)

constexpr int kTB = 256;
unsigned blocks_for(uint64_t n) { return (unsigned)std::min<uint64_t>((n + kTB - 1) / kTB, 148ull * 64); }

enum Op : int { kBoolOr = 0, kBoolAnd = 1, kPlus = 2, kTimes = 3, kMin = 4 };  // sparse.hpp:47

__host__ __device__ inline long long apply(int op, long long a, long long b) {  // sparse.cpp:69-78
    switch (op) {
        case kBoolOr: return (a != 0 || b != 0) ? 1 : 0;
        case kBoolAnd: return (a != 0 && b != 0) ? 1 : 0;
        case kPlus: return (long long)((unsigned long long)a + (unsigned long long)b);
        case kTimes: return (long long)((unsigned long long)a * (unsigned long long)b);
        default: return a < b ? a : b;
    }
}

struct AddOp {
    int op;
    __host__ __device__ long long operator()(long long a, long long b) const { return apply(op, a, b); }
};

struct DevCSR {
    uint64_t nrows = 0, ncols = 0, nnz = 0;
    unsigned long long* rp = nullptr;  // [nrows + 1]
    uint32_t* ci = nullptr;            // [nnz]
    long long* vals = nullptr;         // [nnz] or null (structural)
};

cudaError_t upload(DevCSR& d, uint64_t nrows, uint64_t ncols, const uint64_t* rp, const uint64_t* ci,
                   const int64_t* vals, cudaStream_t s) {
    d.nrows = nrows;
    d.ncols = ncols;
    d.nnz = rp[nrows];
    cudaError_t e;
    std::vector<uint32_t> ci32(std::max<uint64_t>(d.nnz, 1));
    for (uint64_t p = 0; p < d.nnz; ++p) ci32[p] = (uint32_t)ci[p];
    if ((e = cudaMalloc(&d.rp, (nrows + 1) * 8))) return e;
    if ((e = cudaMalloc(&d.ci, std::max<uint64_t>(d.nnz, 1) * 4))) return e;
    if ((e = cudaMemcpyAsync(d.rp, rp, (nrows + 1) * 8, cudaMemcpyHostToDevice, s))) return e;
    if (d.nnz && (e = cudaMemcpyAsync(d.ci, ci32.data(), d.nnz * 4, cudaMemcpyHostToDevice, s))) return e;
    if (vals) {
        if ((e = cudaMalloc(&d.vals, std::max<uint64_t>(d.nnz, 1) * 8))) return e;
        if (d.nnz && (e = cudaMemcpyAsync(d.vals, vals, d.nnz * 8, cudaMemcpyHostToDevice, s))) return e;
    }
    return cudaStreamSynchronize(s);  // ci32 leaves scope
}

void release(DevCSR& d) {
    cudaFree(d.rp);
    cudaFree(d.ci);
    cudaFree(d.vals);
    d = DevCSR{};
}

// products contributed by each A entry: |B[A.ci[p]]|
__global__ void entry_flops(DevCSR A, DevCSR B, unsigned long long* cnt) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < A.nnz;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = A.ci[p];
        cnt[p] = B.rp[k + 1] - B.rp[k];
    }
}

// row of each A entry
__global__ void entry_rows(DevCSR A, uint32_t* arow) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < A.nrows;
         i += (uint64_t)gridDim.x * blockDim.x)
        for (unsigned long long p = A.rp[i]; p < A.rp[i + 1]; ++p) arow[p] = (uint32_t)i;
}

__device__ bool in_row(const DevCSR& M, uint32_t i, uint32_t j) {
    unsigned long long lo = M.rp[i], hi = M.rp[i + 1];
    while (lo < hi) {
        const unsigned long long mid = (lo + hi) >> 1;
        if (M.ci[mid] < j) lo = mid + 1;
        else hi = mid;
    }
    return lo < M.rp[i + 1] && M.ci[lo] == j;
}

// one thread per product t in [t0, t1) of A entries [p0, p1)
__global__ void expand(DevCSR A, DevCSR B, DevCSR M, int has_mask, int mul_op, int valued, const uint32_t* arow,
                       const unsigned long long* off, uint64_t p0, uint64_t p1, unsigned long long t0,
                       unsigned long long t1, unsigned long long* keys, long long* vals, uint8_t* keep) {
    for (unsigned long long t = t0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < t1;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = p0, hi = p1;  // last entry p with off[p] <= t
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (off[mid] <= t) lo = mid;
            else hi = mid;
        }
        const uint64_t p = lo;
        const uint32_t i = arow[p], k = A.ci[p];
        const unsigned long long q = B.rp[k] + (t - off[p]);
        const uint32_t j = B.ci[q];
        const uint64_t o = t - t0;
        keys[o] = ((unsigned long long)i << 32) | j;
        if (valued) {
            const long long a = A.vals ? A.vals[p] : 1, b = B.vals ? B.vals[q] : 1;
            vals[o] = apply(mul_op, a, b);
        }
        keep[o] = (!has_mask || in_row(M, i, j)) ? 1 : 0;
    }
}

__global__ void mark_first(const unsigned long long* keys, uint64_t n, uint8_t* keep) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n;
         p += (uint64_t)gridDim.x * blockDim.x)
        keep[p] = (p == 0 || keys[p] != keys[p - 1]) ? 1 : 0;
}

// first output position of every row present in the sorted keys
__global__ void row_firsts(const unsigned long long* keys, uint64_t n, unsigned long long* first) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long r = keys[x] >> 32;
        if (x == 0 || (keys[x - 1] >> 32) != r) first[r] = x;
    }
}

__global__ void keys_to_cols(unsigned long long* keys, uint64_t n) {
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n;
         x += (uint64_t)gridDim.x * blockDim.x)
        keys[x] &= 0xFFFFFFFFull;
}

int bits_for(uint64_t n) {
    int b = 1;
    while (b < 32 && (1ull << b) < n) ++b;
    return b;
}

}  // namespace

// 0 ok; cudaError_t on device failure
cudaError_t run(int device, const DevIn& a, const DevIn& b, int semiring, const DevIn* mask,
                uint64_t max_chunk, mgk_matrix* out) {
    const int add_op = semiring == 0 ? kBoolOr : semiring == 1 ? kPlus : kMin;
    const int mul_op = semiring == 0 ? kBoolAnd : semiring == 1 ? kTimes : kPlus;
    const bool valued = semiring != 0;
    cudaError_t e = cudaSuccess;
    cudaStream_t s = nullptr;
    DevCSR A, B, M;
    unsigned long long *cnt = nullptr, *off = nullptr, *keys = nullptr, *kalt = nullptr, *ukeys = nullptr;
    long long *vals = nullptr, *valt = nullptr, *uvals = nullptr;
    uint32_t* arow = nullptr;
    uint8_t* keep = nullptr;
    unsigned long long* d_num = nullptr;
    void* tmp = nullptr;
    std::vector<unsigned long long> h_off;
    // device output: reduced (row << 32 | col) keys and values of all chunks, in order
    unsigned long long* okeys = nullptr;
    long long* ovals = nullptr;
    uint64_t on = 0, ocap = 0;
    unsigned long long* first = nullptr;
    auto reserve = [&](uint64_t need) -> cudaError_t {
        if (need <= ocap) return cudaSuccess;
        const uint64_t nc = std::max<uint64_t>({need, 2 * ocap, 1ull << 20});
        unsigned long long* nk = nullptr;
        long long* nv = nullptr;
        cudaError_t r = cudaMalloc(&nk, nc * 8);
        if (!r && valued) r = cudaMalloc(&nv, nc * 8);
        if (!r && on) r = cudaMemcpyAsync(nk, okeys, on * 8, cudaMemcpyDeviceToDevice, s);
        if (!r && on && valued) r = cudaMemcpyAsync(nv, ovals, on * 8, cudaMemcpyDeviceToDevice, s);
        if (!r) r = cudaStreamSynchronize(s);
        if (r) {
            cudaFree(nk);
            cudaFree(nv);
            return r;
        }
        cudaFree(okeys);
        cudaFree(ovals);
        okeys = nk;
        ovals = nv;
        ocap = nc;
        return cudaSuccess;
    };
    auto append = [&](const unsigned long long* k, const long long* v, uint64_t n) -> cudaError_t {
        cudaError_t r = reserve(on + n);
        if (!r && n) r = cudaMemcpyAsync(okeys + on, k, n * 8, cudaMemcpyDeviceToDevice, s);
        if (!r && n && valued) r = cudaMemcpyAsync(ovals + on, v, n * 8, cudaMemcpyDeviceToDevice, s);
        on += n;
        return r;
    };
    out->device = device;
    out->nrows = a.nrows;
    out->ncols = b.ncols;
    out->row_ptr.assign(a.nrows + 1, 0);
    MX_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    MX_TRY(upload(A, a.nrows, a.ncols, a.rp, a.ci, valued ? a.vals : nullptr, s));
    MX_TRY(upload(B, b.nrows, b.ncols, b.rp, b.ci, valued ? b.vals : nullptr, s));
    if (mask) MX_TRY(upload(M, mask->nrows, mask->ncols, mask->rp, mask->ci, nullptr, s));
    if (A.nnz) {
        // per-entry product counts -> exclusive offsets (+ total at off[nnz])
        MX_TRY(cudaMallocAsync(&cnt, (A.nnz + 1) * 8, s));
        MX_TRY(cudaMallocAsync(&off, (A.nnz + 1) * 8, s));
        MX_TRY(cudaMallocAsync(&arow, A.nnz * 4, s));
        entry_flops<<<blocks_for(A.nnz), kTB, 0, s>>>(A, B, cnt);
        entry_rows<<<blocks_for(A.nrows), kTB, 0, s>>>(A, arow);
        MX_TRY(cudaMemsetAsync(cnt + A.nnz, 0, 8, s));
        size_t tb = 0;
        MX_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int64_t)(A.nnz + 1), s));
        MX_TRY(cudaMallocAsync(&tmp, tb, s));
        MX_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int64_t)(A.nnz + 1), s));
        cudaFreeAsync(tmp, s);
        tmp = nullptr;
        // offsets at the row boundaries decide the row chunks
        h_off.resize(A.nnz + 1);
        MX_TRY(cudaMemcpyAsync(h_off.data(), off, (A.nnz + 1) * 8, cudaMemcpyDeviceToHost, s));
        MX_TRY(cudaStreamSynchronize(s));
        const unsigned long long flops = h_off[A.nnz];
        const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(max_chunk, std::max<unsigned long long>(flops, 1)));
        // stream-ordered pool allocations: repeated products reuse the memory
        MX_TRY(cudaMallocAsync(&keys, cap * 8, s));
        MX_TRY(cudaMallocAsync(&kalt, cap * 8, s));
        MX_TRY(cudaMallocAsync(&keep, cap, s));
        MX_TRY(cudaMallocAsync(&d_num, 8, s));
        if (valued) {
            MX_TRY(cudaMallocAsync(&vals, cap * 8, s));
            MX_TRY(cudaMallocAsync(&valt, cap * 8, s));
            MX_TRY(cudaMallocAsync(&ukeys, cap * 8, s));
            MX_TRY(cudaMallocAsync(&uvals, cap * 8, s));
        }
        uint64_t r0 = 0;
        while (r0 < a.nrows) {
            // rows [r0, r1) with at most `cap` products (a single bigger row is
            // processed alone in pieces of whole A entries)
            uint64_t r1 = r0 + 1;
            const unsigned long long base = h_off[a.rp[r0]];
            while (r1 < a.nrows && h_off[a.rp[r1 + 1]] - base <= cap) ++r1;
            // product range of the chunk, cut into pieces of <= cap products
            // (a piece may start or end inside an A entry's B row)
            const unsigned long long T0 = h_off[a.rp[r0]], T1 = h_off[a.rp[r1]];
            const uint64_t chunk_start = on;
            int pieces = 0;
            for (unsigned long long t0 = T0; t0 < T1;) {
                ++pieces;
                const unsigned long long t1 = std::min<unsigned long long>(T1, t0 + cap);
                // entries covering [t0, t1): p0 = last p with off[p] <= t0, p1 = first p with off[p] >= t1
                const uint64_t p0 = (uint64_t)(std::upper_bound(h_off.begin(), h_off.end() - 1, t0) - h_off.begin()) - 1;
                const uint64_t p1 = (uint64_t)(std::lower_bound(h_off.begin() + p0, h_off.end() - 1, t1) - h_off.begin());
                const uint64_t np = t1 - t0;
                if (np) {
                    expand<<<blocks_for(np), kTB, 0, s>>>(A, B, M, mask ? 1 : 0, mul_op, valued ? 1 : 0, arow, off,
                                                         p0, p1, t0, t1, keys, vals, keep);
                    MX_TRY(cudaGetLastError());
                    // drop masked-out products
                    size_t tb2 = 0;
                    MX_TRY(cub::DeviceSelect::Flagged(nullptr, tb2, keys, keep, kalt, d_num, (int64_t)np, s));
                    MX_TRY(cudaMallocAsync(&tmp, tb2, s));
                    MX_TRY(cub::DeviceSelect::Flagged(tmp, tb2, keys, keep, kalt, d_num, (int64_t)np, s));
                    if (valued) MX_TRY(cub::DeviceSelect::Flagged(tmp, tb2, vals, keep, valt, d_num, (int64_t)np, s));
                    cudaFreeAsync(tmp, s);
                    tmp = nullptr;
                    unsigned long long nk = 0;
                    MX_TRY(cudaMemcpyAsync(&nk, d_num, 8, cudaMemcpyDeviceToHost, s));
                    MX_TRY(cudaStreamSynchronize(s));
                    uint64_t nu = 0;
                    if (nk) {
                        const int end_bit = 32 + bits_for(a.nrows);
                        if (valued) {
                            cub::DoubleBuffer<unsigned long long> dk(kalt, keys);
                            cub::DoubleBuffer<long long> dv(valt, vals);
                            size_t tb3 = 0;
                            MX_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb3, dk, dv, (int64_t)nk, 0, end_bit, s));
                            MX_TRY(cudaMallocAsync(&tmp, tb3, s));
                            MX_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb3, dk, dv, (int64_t)nk, 0, end_bit, s));
                            cudaFreeAsync(tmp, s);
                            tmp = nullptr;
                            size_t tb4 = 0;
                            MX_TRY(cub::DeviceReduce::ReduceByKey(nullptr, tb4, dk.Current(), ukeys, dv.Current(), uvals,
                                                                  d_num, AddOp{add_op}, (int64_t)nk, s));
                            MX_TRY(cudaMallocAsync(&tmp, tb4, s));
                            MX_TRY(cub::DeviceReduce::ReduceByKey(tmp, tb4, dk.Current(), ukeys, dv.Current(), uvals,
                                                                  d_num, AddOp{add_op}, (int64_t)nk, s));
                            cudaFreeAsync(tmp, s);
                            tmp = nullptr;
                            unsigned long long nun = 0;
                            MX_TRY(cudaMemcpyAsync(&nun, d_num, 8, cudaMemcpyDeviceToHost, s));
                            MX_TRY(cudaStreamSynchronize(s));
                            nu = nun;
                            MX_TRY(append(ukeys, uvals, nu));
                        } else {
                            cub::DoubleBuffer<unsigned long long> dk(kalt, keys);
                            size_t tb3 = 0;
                            MX_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb3, dk, (int64_t)nk, 0, end_bit, s));
                            MX_TRY(cudaMallocAsync(&tmp, tb3, s));
                            MX_TRY(cub::DeviceRadixSort::SortKeys(tmp, tb3, dk, (int64_t)nk, 0, end_bit, s));
                            cudaFreeAsync(tmp, s);
                            tmp = nullptr;
                            unsigned long long* sorted = dk.Current();
                            unsigned long long* other = dk.Alternate();
                            mark_first<<<blocks_for(nk), kTB, 0, s>>>(sorted, nk, keep);
                            size_t tb4 = 0;
                            MX_TRY(cub::DeviceSelect::Flagged(nullptr, tb4, sorted, keep, other, d_num, (int64_t)nk, s));
                            MX_TRY(cudaMallocAsync(&tmp, tb4, s));
                            MX_TRY(cub::DeviceSelect::Flagged(tmp, tb4, sorted, keep, other, d_num, (int64_t)nk, s));
                            cudaFreeAsync(tmp, s);
                            tmp = nullptr;
                            unsigned long long nun = 0;
                            MX_TRY(cudaMemcpyAsync(&nun, d_num, 8, cudaMemcpyDeviceToHost, s));
                            MX_TRY(cudaStreamSynchronize(s));
                            nu = nun;
                            MX_TRY(append(other, nullptr, nu));
                        }
                    }
                }
                t0 = t1;
            }
            if (pieces > 1) {
                // one row wider than a chunk: its pieces overlap in columns;
                // merge them on the host (rare) and write the row back
                const uint64_t ns = on - chunk_start;
                std::vector<unsigned long long> hk(ns);
                std::vector<long long> hv(valued ? ns : 0);
                MX_TRY(cudaStreamSynchronize(s));
                MX_TRY(cudaMemcpy(hk.data(), okeys + chunk_start, ns * 8, cudaMemcpyDeviceToHost));
                if (valued) MX_TRY(cudaMemcpy(hv.data(), ovals + chunk_start, ns * 8, cudaMemcpyDeviceToHost));
                std::vector<std::pair<unsigned long long, long long>> kv(ns);
                for (size_t x = 0; x < ns; ++x) kv[x] = {hk[x], valued ? hv[x] : 0};
                std::stable_sort(kv.begin(), kv.end(),
                                 [](const auto& l, const auto& r) { return l.first < r.first; });
                hk.clear();
                hv.clear();
                for (size_t x = 0; x < kv.size(); ++x) {
                    if (x && kv[x].first == kv[x - 1].first) {
                        if (valued) hv.back() = apply(add_op, hv.back(), kv[x].second);
                        continue;
                    }
                    hk.push_back(kv[x].first);
                    if (valued) hv.push_back(kv[x].second);
                }
                MX_TRY(cudaMemcpy(okeys + chunk_start, hk.data(), hk.size() * 8, cudaMemcpyHostToDevice));
                if (valued) MX_TRY(cudaMemcpy(ovals + chunk_start, hv.data(), hv.size() * 8, cudaMemcpyHostToDevice));
                on = chunk_start + hk.size();
            }
            r0 = r1;
        }
    }
    // keys are (row, col) ascending across chunks: row starts from the keys,
    // then the keys become the column array in place
    MX_TRY(cudaMallocAsync(&first, (a.nrows + 1) * 8, s));
    MX_TRY(cudaMemsetAsync(first, 0xFF, (a.nrows + 1) * 8, s));
    if (on) {
        row_firsts<<<blocks_for(on), kTB, 0, s>>>(okeys, on, first);
        keys_to_cols<<<blocks_for(on), kTB, 0, s>>>(okeys, on);
        MX_TRY(cudaGetLastError());
    }
    MX_TRY(cudaMemcpyAsync(out->row_ptr.data(), first, (a.nrows + 1) * 8, cudaMemcpyDeviceToHost, s));
    MX_TRY(cudaStreamSynchronize(s));
    out->row_ptr[a.nrows] = on;  // rows without entries start where the next row starts
    for (uint64_t i2 = a.nrows; i2-- > 0;)
        out->row_ptr[i2] = std::min<uint64_t>(out->row_ptr[i2], out->row_ptr[i2 + 1]);
    out->nnz = on;
    out->valued = valued && on > 0;  // from_parts: valued = !vals.empty()
    out->d_col = okeys;
    out->d_vals = valued ? ovals : nullptr;
    if (!valued) cudaFree(ovals);
    okeys = nullptr;
    ovals = nullptr;
done:
    if (tmp) cudaFreeAsync(tmp, s);
    if (s) cudaStreamSynchronize(s);
    release(A);
    release(B);
    release(M);
    cudaFree(okeys);  // only on an error path (ownership moved to `out` otherwise)
    cudaFree(ovals);
    for (void* pz : {(void*)cnt, (void*)off, (void*)arow, (void*)keys, (void*)kalt, (void*)ukeys, (void*)vals,
                     (void*)valt, (void*)uvals, (void*)keep, (void*)d_num, (void*)first})
        if (pz) cudaFreeAsync(pz, s);
    if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
    return e;
}

}  // namespace mx
}  // namespace mgk

using namespace mgk;

namespace mgk {
void set_last_error(const std::string& msg);  // mgk_capi.cpp
}

namespace {
int fail_code(int code, const std::string& msg) {
    mgk::set_last_error(msg);
    return code;
}

int check_csr(const char* name, uint64_t nrows, uint64_t ncols, const uint64_t* rp, const uint64_t* ci) {
    if (!rp) return fail_code(MGK_ECONTRACT, std::string("mxm: null ") + name + " row_ptr");
    if (nrows >= 0xFFFFFFFFull || ncols >= 0xFFFFFFFFull)
        return fail_code(MGK_ERANGE, std::string("mxm: ") + name + " exceeds uint32 device indices");
    if (rp[0] != 0) return fail_code(MGK_ECONTRACT, std::string("mxm: ") + name + " row_ptr must start at 0");
    for (uint64_t i = 0; i < nrows; ++i)
        if (rp[i + 1] < rp[i]) return fail_code(MGK_ECONTRACT, std::string("mxm: ") + name + " row_ptr decreases");
    if (rp[nrows] && !ci) return fail_code(MGK_ECONTRACT, std::string("mxm: null ") + name + " col_idx");
    for (uint64_t p = 0; p < rp[nrows]; ++p)
        if (ci[p] >= ncols) return fail_code(MGK_ECONTRACT, std::string("mxm: ") + name + " column out of range");
    return MGK_OK;
}
}  // namespace

extern "C" {

int mgk_mxm(int device, uint64_t a_nrows, uint64_t a_ncols, const uint64_t* a_row_ptr, const uint64_t* a_col_idx,
            const int64_t* a_vals, uint64_t b_nrows, uint64_t b_ncols, const uint64_t* b_row_ptr,
            const uint64_t* b_col_idx, const int64_t* b_vals, int semiring, uint64_t m_nrows, uint64_t m_ncols,
            const uint64_t* m_row_ptr, const uint64_t* m_col_idx, mgk_matrix** out) {
    if (!out) return fail_code(MGK_ECONTRACT, "null argument");
    if (semiring < MGK_SEMIRING_BOOL_OR_AND || semiring > MGK_SEMIRING_MIN_PLUS)
        return fail_code(MGK_ECONTRACT, "unknown semiring " + std::to_string(semiring));
    if (a_ncols != b_nrows)  // sparse.cpp:294-297
        return fail_code(MGK_ECONTRACT, "mxm: inner dimensions disagree (" + std::to_string(a_nrows) + "x" +
                                            std::to_string(a_ncols) + " times " + std::to_string(b_nrows) + "x" +
                                            std::to_string(b_ncols) + ")");
    if (m_row_ptr && (m_nrows != a_nrows || m_ncols != b_ncols))  // sparse.cpp:298-301
        return fail_code(MGK_ECONTRACT, "mxm: mask shape " + std::to_string(m_nrows) + "x" + std::to_string(m_ncols) +
                                            " != result shape " + std::to_string(a_nrows) + "x" +
                                            std::to_string(b_ncols));
    int rc;
    if ((rc = check_csr("A", a_nrows, a_ncols, a_row_ptr, a_col_idx))) return rc;
    if ((rc = check_csr("B", b_nrows, b_ncols, b_row_ptr, b_col_idx))) return rc;
    if (m_row_ptr && (rc = check_csr("mask", m_nrows, m_ncols, m_row_ptr, m_col_idx))) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail_code(MGK_ECUDA, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail_code(MGK_ECONTRACT, "device out of range");
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    auto* m = new (std::nothrow) mgk_matrix();
    if (!m) return fail_code(MGK_ENOMEM, "out of host memory");
    mx::DevIn A{a_nrows, a_ncols, a_row_ptr, a_col_idx, a_vals}, B{b_nrows, b_ncols, b_row_ptr, b_col_idx, b_vals};
    mx::DevIn M{m_nrows, m_ncols, m_row_ptr, m_col_idx, nullptr};
    uint64_t chunk = 512ull << 20;
    if (const char* c = std::getenv("MGK_MXM_CHUNK")) chunk = std::max<uint64_t>(1, std::strtoull(c, nullptr, 10));
    cudaError_t e = mx::run(device, A, B, semiring, m_row_ptr ? &M : nullptr, chunk, m);
    cudaSetDevice(prev);
    if (e) {
        delete m;
        cudaGetLastError();
        if (e == cudaErrorInvalidValue) return fail_code(MGK_ERANGE, "mxm: a row of B exceeds the product chunk");
        if (e == cudaErrorMemoryAllocation) return fail_code(MGK_ENOMEM, "mxm: out of device memory");
        return fail_code(MGK_ECUDA, std::string("mxm: CUDA error ") + cudaGetErrorString(e));
    }
    *out = m;
    return MGK_OK;
}

int mgk_matrix_info(const mgk_matrix* m, uint64_t* nrows, uint64_t* ncols, uint64_t* nnz, int* valued) {
    if (!m) return fail_code(MGK_ECONTRACT, "null matrix");
    if (nrows) *nrows = m->nrows;
    if (ncols) *ncols = m->ncols;
    if (nnz) *nnz = m->nnz;
    if (valued) *valued = m->valued ? 1 : 0;
    return MGK_OK;
}

int mgk_matrix_download(const mgk_matrix* m, uint64_t* row_ptr, uint64_t* col_idx, int64_t* vals) {
    if (!m) return fail_code(MGK_ECONTRACT, "null matrix");
    if (row_ptr) std::memcpy(row_ptr, m->row_ptr.data(), m->row_ptr.size() * 8);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    cudaError_t e = cudaSuccess;
    if (col_idx && m->nnz) e = cudaMemcpy(col_idx, m->d_col, m->nnz * 8, cudaMemcpyDeviceToHost);
    if (!e && vals && m->valued && m->nnz) e = cudaMemcpy(vals, m->d_vals, m->nnz * 8, cudaMemcpyDeviceToHost);
    cudaSetDevice(prev);
    if (e) return fail_code(MGK_ECUDA, std::string("mxm download: ") + cudaGetErrorString(e));
    return MGK_OK;
}

int mgk_matrix_free(mgk_matrix* m) {
    if (!m) return MGK_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    delete m;
    cudaSetDevice(prev);
    return MGK_OK;
}

}  // extern "C"
