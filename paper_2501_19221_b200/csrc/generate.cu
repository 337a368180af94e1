// generate.cu -- device-side instance synthesis for BASELINE config 5.
//
// At N = 2e8 the reference's instance path (QuboModel.from_terms: a Python dict, ~6 us per
// term, then qubo_to_ising's Python loop) cannot build the model, so the family is defined
// so that the GPU can generate it directly, and mirrored in numpy
// (paper_2501_19221_b200/instances.py: qubo_deg6_family) for cross-checks at small N:
//
//   raw(s, k) = Philox4x64-10(ctr = (k/4 + 1, 0, s, 0), key = (seed, 0))[k % 4]
//   edges     for c in {0,1,2}, i in [0,n): j = (i + 1 + raw(S+c, i) % (n-1)) % n,
//             key = min(i,j) * n + max(i,j); duplicate keys merged (mean degree ~6)
//   Q_ij      = U(raw(S+3, key)),  Q_ii = U(raw(S+4, i)),  U(r) = -1 + 2 (r >> 11) 2^-53
//   Ising     qubo_to_ising (transforms.py:36-56): J = Q/4; h_i summed per row in the
//             reference's term order; offset = exact sum of the Q_ii/2 and Q_ij/4 terms,
//             rounded once (the reference's sequential float sum would round ~1e9 times)
#include <cub/cub.cuh>

#include <algorithm>

#include "vxq_internal.h"

namespace vxq {
namespace {

constexpr uint64_t kStream = 1ull << 40;
constexpr int TB = 256;
inline unsigned nblk(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, TB)); }

__device__ __forceinline__ uint64_t raw_draw(uint64_t seed, uint64_t stream, uint64_t k) {
    U64x4 o = philox4x64_10(k / 4 + 1, 0, stream, 0, seed, 0);
    return pick_word(o, (uint32_t)(k % 4));
}

__device__ __forceinline__ double unit_uniform(uint64_t raw) {
    return uniform_from_raw(raw, -1.0, 2.0);
}

__global__ void k_gen_keys(int64_t n, uint64_t seed, unsigned long long* keys) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= 3 * n) return;
    const int64_t c = idx / n, i = idx % n;
    const uint64_t off = 1 + raw_draw(seed, kStream + c, (uint64_t)i) % (uint64_t)(n - 1);
    const int64_t j = (int64_t)(((uint64_t)i + off) % (uint64_t)n);
    const int64_t lo = i < j ? i : j, hi = i < j ? j : i;
    keys[idx] = (unsigned long long)(lo * n + hi);
}

__global__ void k_gen_coo(int64_t m, const unsigned long long* keys, int64_t n, uint64_t seed,
                          int64_t* rows, int64_t* cols, double* vals) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const unsigned long long key = keys[k];
    rows[k] = (int64_t)(key / (unsigned long long)n);
    cols[k] = (int64_t)(key % (unsigned long long)n);
    vals[k] = unit_uniform(raw_draw(seed, kStream + 3, key)) / 4.0 + 0.0;  // J = Q / 4
}

__global__ void k_gen_diag(int64_t n, uint64_t seed, double* qd) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) qd[i] = unit_uniform(raw_draw(seed, kStream + 4, (uint64_t)i));
}

// h_i in the reference's qubo_to_ising order: terms (k, i) with k < i (ascending k), then
// (i, i) as Q_ii / 2, then (i, j) with j > i (ascending j); J = Q / 4 already in data
__global__ void k_qubo_fields(int64_t n, const int64_t* indptr, const int32_t* lower_count,
                              const double* data, const double* qd, double* h) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t b = indptr[i], mid = b + lower_count[i], e = indptr[i + 1];
    double acc = 0.0;
    for (int64_t k = b; k < mid; ++k) acc = __dadd_rn(acc, data[k]);
    acc = __dadd_rn(acc, qd[i] / 2.0);
    for (int64_t k = mid; k < e; ++k) acc = __dadd_rn(acc, data[k]);
    h[i] = acc;
}

// exact sum of the offset terms (all multiples of 2^-54, |t| < 1): scaled int64, split
// into hi/lo 32-bit halves accumulated in two 64-bit counters
__global__ void k_offset_terms(int64_t m, const double* J, int64_t n, const double* qd,
                               unsigned long long* acc) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    long long v = 0;
    if (k < m) v = (long long)(J[k] * 0x1p54);
    else if (k < m + n) v = (long long)((qd[k - m] / 2.0) * 0x1p54);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v != 0) {
        atomicAdd(acc, (unsigned long long)(v >> 32));
        atomicAdd(acc + 1, (unsigned long long)(v & 0xffffffffLL));
    }
}

__global__ void k_widen32(int64_t m, const int32_t* a, int64_t* b) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < m) b[k] = a[k];
}

}  // namespace

Problem* problem_generate(int family, int64_t n, uint64_t seed, int device) {
    VXQ_REQUIRE(family == 0, "unknown instance family (0 = qubo_deg6)");
    VXQ_REQUIRE(n >= 2 && n < (1LL << 31) - 1, "n must be in [2, 2^31)");
    VXQ_CUDA(cudaSetDevice(device));
    retain_mempool();
    cudaStream_t s;
    VXQ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG {
        cudaStream_t s;
        ~SG() { cudaStreamDestroy(s); }
    } sg{s};
    const int64_t m3 = 3 * n;
    int64_t m = 0;
    DevBuf<int64_t> rows, cols;
    DevBuf<double> vals;
    {
        DevBuf<unsigned long long> keys(m3, s), sorted(m3, s), uniq(m3, s);
        DevBuf<int64_t> nuniq(1, s);
        k_gen_keys<<<nblk(m3), TB, 0, s>>>(n, seed, keys.get());
        VXQ_CHECK_LAUNCH();
        int end_bit = 1;
        while (end_bit < 64 && (1ULL << end_bit) < (unsigned long long)n * (unsigned long long)n)
            ++end_bit;
        size_t need = 0, need2 = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, need, keys.get(), sorted.get(), (int64_t)m3, 0,
                                       end_bit, s);
        cub::DeviceSelect::Unique(nullptr, need2, sorted.get(), uniq.get(), nuniq.get(),
                                  (int64_t)m3, s);
        DevBuf<uint8_t> tmp(std::max<size_t>(std::max(need, need2), 1), s);
        VXQ_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), need, keys.get(), sorted.get(),
                                                (int64_t)m3, 0, end_bit, s));
        VXQ_CUDA(cub::DeviceSelect::Unique(tmp.get(), need2, sorted.get(), uniq.get(),
                                           nuniq.get(), (int64_t)m3, s));
        VXQ_CUDA(cudaMemcpyAsync(&m, nuniq.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        VXQ_CUDA(cudaStreamSynchronize(s));
        rows = DevBuf<int64_t>(m, s);
        cols = DevBuf<int64_t>(m, s);
        vals = DevBuf<double>(m, s);
        k_gen_coo<<<nblk(m), TB, 0, s>>>(m, uniq.get(), n, seed, rows.get(), cols.get(),
                                         vals.get());
        VXQ_CHECK_LAUNCH();
        VXQ_CUDA(cudaStreamSynchronize(s));
    }
    Problem* P = problem_create(n, m, rows.get(), cols.get(), vals.get(), nullptr, 0.0, device);
    try {
        rows.release();
        cols.release();
        DevBuf<double> qd(n, s), h(n, s);
        k_gen_diag<<<nblk(n), TB, 0, s>>>(n, seed, qd.get());
        k_qubo_fields<<<nblk(n), TB, 0, s>>>(n, P->indptr, P->lower_count, P->data64, qd.get(),
                                             h.get());
        DevBuf<unsigned long long> acc(2, s);
        VXQ_CUDA(cudaMemsetAsync(acc.get(), 0, 2 * sizeof(unsigned long long), s));
        k_offset_terms<<<nblk(m + n), TB, 0, s>>>(m, vals.get(), n, qd.get(), acc.get());
        VXQ_CHECK_LAUNCH();
        unsigned long long hl[2];
        VXQ_CUDA(cudaMemcpyAsync(hl, acc.get(), sizeof(hl), cudaMemcpyDeviceToHost, s));
        VXQ_CUDA(cudaStreamSynchronize(s));
        const __int128 total = (__int128)(long long)hl[0] * ((__int128)1 << 32) + (__int128)hl[1];
        const double offset = ldexp((double)total, -54);  // one (round-to-nearest) rounding
        problem_set_fields(P, h.get(), offset, s);
    } catch (...) {
        delete P;
        throw;
    }
    return P;
}

void problem_export(Problem* P, int64_t* rows, int64_t* cols, double* values, double* h,
                    double* offset) {
    cudaStream_t s;
    VXQ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SG {
        cudaStream_t s;
        ~SG() { cudaStreamDestroy(s); }
    } sg{s};
    const int64_t m = P->m;
    if (m > 0 && (rows || cols)) {
        DevBuf<int64_t> w(m, s);
        if (rows) {
            k_widen32<<<nblk(m), TB, 0, s>>>(m, P->coo_i, w.get());
            VXQ_CUDA(cudaMemcpyAsync(rows, w.get(), m * sizeof(int64_t), cudaMemcpyDefault, s));
            VXQ_CUDA(cudaStreamSynchronize(s));
        }
        if (cols) {
            k_widen32<<<nblk(m), TB, 0, s>>>(m, P->coo_j, w.get());
            VXQ_CUDA(cudaMemcpyAsync(cols, w.get(), m * sizeof(int64_t), cudaMemcpyDefault, s));
        }
    }
    if (m > 0 && values)
        VXQ_CUDA(cudaMemcpyAsync(values, P->coo_v, m * sizeof(double), cudaMemcpyDefault, s));
    if (h) VXQ_CUDA(cudaMemcpyAsync(h, P->h64, P->n * sizeof(double), cudaMemcpyDefault, s));
    VXQ_CUDA(cudaStreamSynchronize(s));
    if (offset) *offset = P->offset;
}

}  // namespace vxq
