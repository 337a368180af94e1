// problem.cu -- device-resident Ising problem: symmetric CSR build, lambda0, c0.
//
// Replaces IsingModel.coupling_operator()/_csr (model.py:166-192),
// field_scale (model.py:194-200) and resolve_c0/eig_extreme (bifurcation.py:25-34,
// solvers/eigen.py:35-56).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstring>

#include "vxq_internal.h"

namespace vxq {

Problem::~Problem() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    void* ptrs[] = {indptr, indices, data64, data32, lower_count, h64,  h32,
                    g64,    g32,     coo_i,  coo_j,  coo_v,       coef_fx, h_fx};
    // problem arrays live in the device's retained stream-ordered pool: freeing them
    // returns the memory to the pool (no unmapping), and the next problem reuses it
    for (void* q : ptrs)
        if (q) cudaFreeAsync(q, 0);
    cudaStreamSynchronize(0);
    extern void dense_destroy(DenseOperand*);
    if (dense) dense_destroy(dense);
    extern void nbr_blocks_destroy(NbrBlocks*);
    if (nbr_blocks) nbr_blocks_destroy(nbr_blocks);
    cudaSetDevice(prev);
}

namespace {

__global__ void k_validate_coo(int64_t n, int64_t m, const int64_t* rows, const int64_t* cols,
                               const double* values, int* err) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    int64_t i = rows[k], j = cols[k];
    int e = 0;
    if (!(i >= 0 && i < j && j < n)) e |= 1;
    if (k > 0) {
        int64_t pi = rows[k - 1], pj = cols[k - 1];
        if (!(pi < i || (pi == i && pj < j))) e |= 2;
    }
    if (values && !isfinite(values[k])) e |= 4;
    if (e) atomicOr(err, e);
}

__global__ void k_check_finite(int64_t m, const double* values, int* err) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < m && !isfinite(values[k])) atomicOr(err, 4);
}

__global__ void k_count_deg(int64_t m, const int64_t* rows, const int64_t* cols, int32_t* deg_up,
                            int32_t* deg_lo, int32_t* ci, int32_t* cj) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool ok = k < m;
    int32_t i = ok ? (int32_t)rows[k] : -1, j = ok ? (int32_t)cols[k] : -1;
    // rows are sorted: lanes sharing a row aggregate into one atomic
    const unsigned peers = __match_any_sync(0xffffffffu, i);
    if (ok && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(deg_up + i, __popc(peers));
    if (!ok) return;
    atomicAdd(deg_lo + j, 1);
    ci[k] = i;
    cj[k] = j;
}

__global__ void k_row_total(int64_t n, const int32_t* up, const int32_t* lo, int64_t* tot) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) tot[i] = (int64_t)up[i] + lo[i];
    if (i == n) tot[i] = 0;
}

// (rows[k], cols[k]) of the full upper triangle in canonical order: row i starts at
// i (n - 1) - i (i - 1) / 2; binary search for the row of k
__global__ void k_triangle_coo(int64_t n, int64_t m, int64_t* __restrict__ rows,
                               int64_t* __restrict__ cols) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    int64_t lo = 0, hi = n - 2;  // the row i with start(i) <= k < start(i + 1)
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        const int64_t st = mid * (n - 1) - mid * (mid - 1) / 2;
        if (st <= k) lo = mid;
        else hi = mid - 1;
    }
    const int64_t st = lo * (n - 1) - lo * (lo - 1) / 2;
    rows[k] = lo;
    cols[k] = lo + 1 + (k - st);
}

__global__ void k_iota(int64_t m, int32_t* v) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < m) v[k] = (int32_t)k;
}

// upper part of row i: COO range in order -> after the lower part
__global__ void k_fill_upper(int64_t m, const int32_t* ci, const int32_t* cj, const double* val,
                             const int64_t* indptr, const int32_t* deg_lo,
                             const int64_t* ustart, int32_t* indices, double* data) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    int32_t i = ci[k];
    int64_t pos = indptr[i] + deg_lo[i] + (k - ustart[i]);
    indices[pos] = cj[k];
    data[pos] = val[k];
}

// lower part of row c: stable-sorted by column -> ascending row index
__global__ void k_fill_lower(int64_t m, const int32_t* sorted_cols, const int32_t* perm,
                             const int32_t* ci, const double* val, const int64_t* indptr,
                             const int64_t* lstart, int32_t* indices, double* data) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= m) return;
    int32_t c = sorted_cols[p];
    int32_t k = perm[p];
    int64_t pos = indptr[c] + (p - lstart[c]);
    indices[pos] = ci[k];
    data[pos] = val[k];
}

__global__ void k_convert(int64_t nnz, const double* d64, float* d32) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < nnz) d32[k] = __double2float_rn(d64[k]);
}

__global__ void k_fields(int64_t n, const double* h, float* h32, double* g64, float* g32) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = h[i];
    h32[i] = __double2float_rn(v);
    g64[i] = -v;
    g32[i] = -__double2float_rn(v);
}

__global__ void k_abs_minmax(int64_t m, const double* v, unsigned long long* mn,
                             unsigned long long* mx) {
    unsigned long long lo = ~0ULL, hi = 0ULL;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
         k += (int64_t)blockDim.x * gridDim.x) {
        unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v[k]));
        lo = b < lo ? b : lo;
        hi = b > hi ? b : hi;
    }
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o);
        unsigned long long c = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = c > hi ? c : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mn, lo);
        atomicMax(mx, hi);
    }
}

// ---- exact fixed-point encoding of coefficients ----
// value = mant * 2^e with mant a 53-bit integer; lowest/highest set bit exponents.
__device__ __forceinline__ bool decompose(double v, uint64_t& mant, int& e) {
    uint64_t b = (uint64_t)__double_as_longlong(v);
    int E = (int)((b >> 52) & 0x7ff);
    mant = b & ((1ULL << 52) - 1);
    if (E == 0) {
        e = -1074;
    } else {
        mant |= (1ULL << 52);
        e = E - 1075;
    }
    return mant != 0;
}

// binary exponent range of the nonzero values: grid-stride, warp-reduced, one atomic pair
// per warp (per-element atomics on one address serialise: 0.7 ms at 5e7 couplings)
__global__ void k_exp_range(int64_t cnt, const double* v, int* lo, int* hi) {
    int low = INT_MAX, high = INT_MIN;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt;
         k += (int64_t)gridDim.x * blockDim.x) {
        uint64_t mant;
        int e;
        if (!decompose(v[k], mant, e)) continue;
        low = min(low, e + (__ffsll((long long)mant) - 1));
        high = max(high, e + (63 - __clzll((long long)mant)));
    }
    low = __reduce_min_sync(0xffffffffu, low);
    high = __reduce_max_sync(0xffffffffu, high);
    if ((threadIdx.x & 31) == 0 && low <= high) {
        atomicMin(lo, low);
        atomicMax(hi, high);
    }
}

__device__ void encode_fx(double v, int e_low, int L, uint32_t* out) {
    uint64_t mant;
    int e;
    uint32_t limb[kMaxLimbs + 3];
    for (int q = 0; q < L; ++q) limb[q] = 0;
    if (decompose(v, mant, e)) {
        int s = e - e_low;  // >= 0
        int q0 = s >> 5, sh = s & 31;
        // mant << sh spans up to 85 bits -> 3 limbs
        unsigned __int128 w = ((unsigned __int128)mant) << sh;
        for (int t = 0; t < 3; ++t) {
            int q = q0 + t;
            if (q < L) limb[q] = (uint32_t)(w >> (32 * t));
        }
        if (v < 0) {  // two's complement negate over L limbs
            uint64_t carry = 1;
            for (int q = 0; q < L; ++q) {
                uint64_t t = (uint64_t)(uint32_t)~limb[q] + carry;
                limb[q] = (uint32_t)t;
                carry = t >> 32;
            }
        }
    }
    for (int q = 0; q < L; ++q) out[q] = limb[q];
}

__global__ void k_encode(int64_t cnt, const double* v, int e_low, int L, uint32_t* out) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < cnt) encode_fx(v[k], e_low, L, out + k * L);
}

__global__ void k_encode_scalar(double v, int e_low, int L, uint32_t* out) {
    encode_fx(v, e_low, L, out);
}

// field_scale: |h_i| + sum_{j>i asc} |J| + sum_{j<i asc} |J|  (np.add.at over rows, then cols)
// field_scale row sums in np.add.at order (|h_i|, then the j > i couplings ascending, then
// the j < i ones): one warp per row stages 256 |values| at a time in shared memory with
// coalesced loads, lane 0 folds them strictly in order (bit-exact with the reference)
constexpr int kFsWarps = 8, kFsChunk = 256;
__global__ void __launch_bounds__(32 * kFsWarps) k_field_scale(
    int64_t n, const int64_t* indptr, const int32_t* lower_count, const double* data,
    const double* h, unsigned long long* maxbits) {
    __shared__ double buf[kFsWarps][kFsChunk];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double best = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kFsWarps + w; i < n;
         i += (int64_t)gridDim.x * kFsWarps) {
        double acc = fabs(h[i]);
        const int64_t b = indptr[i], mid = b + lower_count[i], e = indptr[i + 1];
        for (int part = 0; part < 2; ++part) {
            const int64_t lo = part == 0 ? mid : b, hi = part == 0 ? e : mid;
            for (int64_t k0 = lo; k0 < hi; k0 += kFsChunk) {
                const int cnt = (int)min((int64_t)kFsChunk, hi - k0);
                for (int u = lane; u < cnt; u += 32) buf[w][u] = fabs(data[k0 + u]);
                __syncwarp();
                if (lane == 0)
                    for (int u = 0; u < cnt; ++u) acc = __dadd_rn(acc, buf[w][u]);
                __syncwarp();
            }
        }
        if (lane == 0) best = fmax(best, acc);
    }
    // non-negative doubles order like their bit patterns
    if (lane == 0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(best));
}

constexpr int TB = 256;
inline unsigned nblk(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, TB)); }

__global__ void k_widen(int64_t n, const int32_t* a, int64_t* b) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
    if (i == n) b[i] = 0;
}
void widen_i32_i64(int64_t n, const int32_t* a, int64_t* b, cudaStream_t s) {
    k_widen<<<nblk(n + 1), TB, 0, s>>>(n, a, b);
    VXQ_CHECK_LAUNCH();
}

}  // namespace

void encode_energy(Problem* P, cudaStream_t s) {
    if (P->coef_fx) cudaFreeAsync(P->coef_fx, s);
    if (P->h_fx) cudaFreeAsync(P->h_fx, s);
    P->coef_fx = P->h_fx = nullptr;
    P->energy_ok = true;
    const int64_t n = P->n, m = P->m;
    {
            DevBuf<int> rng(2, s);
            int init[2] = {1 << 20, -(1 << 20)};
            VXQ_CUDA(cudaMemcpyAsync(rng.get(), init, sizeof(init), cudaMemcpyHostToDevice, s));
            if (m > 0)
                k_exp_range<<<(unsigned)std::min<int64_t>(nblk(m), 148 * 16), TB, 0, s>>>(
                    m, P->coo_v, rng.get(), rng.get() + 1);
            k_exp_range<<<(unsigned)std::min<int64_t>(nblk(n), 148 * 16), TB, 0, s>>>(
                n, P->h64, rng.get(), rng.get() + 1);
            DevBuf<double> doff(1, s);
            VXQ_CUDA(cudaMemcpyAsync(doff.get(), &P->offset, sizeof(double),
                                     cudaMemcpyHostToDevice, s));
            k_exp_range<<<1, 1, 0, s>>>(1, doff.get(), rng.get(), rng.get() + 1);
            VXQ_CHECK_LAUNCH();
            int res[2];
            VXQ_CUDA(cudaMemcpyAsync(res, rng.get(), sizeof(res), cudaMemcpyDeviceToHost, s));
            VXQ_CUDA(cudaStreamSynchronize(s));
            if (res[0] > res[1]) {  // all coefficients zero
                res[0] = 0;
                res[1] = 0;
            }
            P->e_low = res[0];
            int span = res[1] - res[0] + 1;  // bits of the largest |coefficient|
            int L = (span + 1 + 31) / 32 + (span % 32 > 29 ? 1 : 0);
            L = std::max(L, 2);
            if (L > kMaxLimbs) {
                P->energy_ok = false;
                L = kMaxLimbs;
            }
            P->limbs = L;
            VXQ_CUDA(cudaMallocAsync((void**)&P->coef_fx, std::max<int64_t>(m, 1) * L * sizeof(uint32_t), s));
            VXQ_CUDA(cudaMallocAsync((void**)&P->h_fx, n * L * sizeof(uint32_t), s));
            if (P->energy_ok) {
                if (m > 0) k_encode<<<nblk(m), TB, 0, s>>>(m, P->coo_v, P->e_low, L, P->coef_fx);
                k_encode<<<nblk(n), TB, 0, s>>>(n, P->h64, P->e_low, L, P->h_fx);
                DevBuf<uint32_t> ofx(L, s);
                k_encode_scalar<<<1, 1, 0, s>>>(P->offset, P->e_low, L, ofx.get());
                VXQ_CHECK_LAUNCH();
                VXQ_CUDA(cudaMemcpyAsync(P->offset_fx, ofx.get(), L * sizeof(uint32_t),
                                         cudaMemcpyDeviceToHost, s));
                if (P->uniform_magnitude) {
                    DevBuf<uint32_t> mfx(L, s);
                    k_encode_scalar<<<1, 1, 0, s>>>(P->magnitude, P->e_low, L, mfx.get());
                    VXQ_CHECK_LAUNCH();
                    VXQ_CUDA(cudaMemcpyAsync(P->mag_fx, mfx.get(), L * sizeof(uint32_t),
                                             cudaMemcpyDeviceToHost, s));
                    VXQ_CUDA(cudaStreamSynchronize(s));
                }
            }
        }
}

namespace {
// VXQ_CREATE_TIMING=1: synchronise after each phase of problem_create and print its time
struct PhaseTimer {
    bool on = false;
    cudaStream_t s = nullptr;
    std::chrono::steady_clock::time_point t0;
    PhaseTimer() {
        const char* e = getenv("VXQ_CREATE_TIMING");
        on = e && e[0] == '1';
        t0 = std::chrono::steady_clock::now();
    }
    void mark(const char* what) {
        if (!on) return;
        if (s) cudaStreamSynchronize(s);
        const auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[vxq create] %-14s %8.2f ms\n", what,
                std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};
}  // namespace

Problem* problem_create(int64_t n, int64_t m, const int64_t* rows, const int64_t* cols,
                        const double* values, const double* h, double offset, int device) {
    PhaseTimer ph;
    VXQ_REQUIRE(n >= 1, "model needs at least one variable");
    VXQ_REQUIRE(n < (1LL << 31) - 1, "n must be < 2^31");
    VXQ_REQUIRE(m >= 0 && m < (1LL << 31) - 1, "num_couplings must be in [0, 2^31)");
    // rows = cols = NULL: the full upper triangle (dense model), generated on the device
    const bool implied = m > 0 && !rows && !cols;
    VXQ_REQUIRE(!implied || (n >= 2 && m == n * (n - 1) / 2),
                "rows = cols = NULL needs num_couplings = n (n - 1) / 2");
    VXQ_REQUIRE(m == 0 || ((implied || (rows && cols)) && values), "null coupling arrays");
    VXQ_REQUIRE(std::isfinite(offset), "offset must be finite");
    int ndev = 0;
    VXQ_CUDA(cudaGetDeviceCount(&ndev));
    VXQ_REQUIRE(device >= 0 && device < ndev, "invalid CUDA device ordinal");
    VXQ_CUDA(cudaSetDevice(device));
    retain_mempool();  // problem arrays come from the retained stream-ordered pool

    Problem* P = new Problem();
    try {
        P->device = device;
        P->n = n;
        P->m = m;
        P->nnz = 2 * m;
        P->offset = offset;
        cudaStream_t s;
        VXQ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct SG {
            cudaStream_t s;
            ~SG() { cudaStreamDestroy(s); }
        } sg{s};
        ph.s = s;
        ph.mark("stream");

        const int64_t nnz = 2 * m;
        VXQ_CUDA(cudaMallocAsync((void**)&P->indptr, (n + 1) * sizeof(int64_t), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->indices, std::max<int64_t>(nnz, 1) * sizeof(int32_t), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->data64, std::max<int64_t>(nnz, 1) * sizeof(double), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->data32, std::max<int64_t>(nnz, 1) * sizeof(float), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->lower_count, n * sizeof(int32_t), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->h64, n * sizeof(double), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->h32, n * sizeof(float), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->g64, n * sizeof(double), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->g32, n * sizeof(float), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->coo_i, std::max<int64_t>(m, 1) * sizeof(int32_t), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->coo_j, std::max<int64_t>(m, 1) * sizeof(int32_t), s));
        ph.mark("alloc");

        // fields
        if (h) {
            VXQ_CUDA(cudaMemcpyAsync(P->h64, h, n * sizeof(double), cudaMemcpyDefault, s));
        } else {
            VXQ_CUDA(cudaMemsetAsync(P->h64, 0, n * sizeof(double), s));
        }
        k_fields<<<nblk(n), TB, 0, s>>>(n, P->h64, P->h32, P->g64, P->g32);
        VXQ_CHECK_LAUNCH();

        DevBuf<int32_t> deg_up(n, s), deg_lo(n, s);
        DevBuf<int64_t> tot(n + 1, s), ustart(n + 1, s), lstart(n + 1, s), up64(n + 1, s),
            lo64(n + 1, s);
        VXQ_CUDA(cudaMemsetAsync(deg_up.get(), 0, n * sizeof(int32_t), s));
        VXQ_CUDA(cudaMemsetAsync(deg_lo.get(), 0, n * sizeof(int32_t), s));
        VXQ_CUDA(cudaMallocAsync((void**)&P->coo_v, std::max<int64_t>(m, 1) * sizeof(double), s));
        struct DV {
            double* p;
            double* get() const { return p; }
        } dval{P->coo_v};
        DevBuf<int32_t> err(1, s);
        VXQ_CUDA(cudaMemsetAsync(err.get(), 0, sizeof(int), s));
        // the values travel on a second stream while the structure (validation, degree
        // counts, the column sort) is built from rows / cols; the fills wait for them
        cudaStream_t s2 = nullptr;
        cudaEvent_t ev_rc = nullptr, ev_val = nullptr;
        struct SG2 {
            cudaStream_t& s;
            cudaEvent_t& a;
            cudaEvent_t& b;
            ~SG2() {
                if (a) cudaEventDestroy(a);
                if (b) cudaEventDestroy(b);
                if (s) cudaStreamDestroy(s);
            }
        } sg2{s2, ev_rc, ev_val};
        if (m > 0) {
            VXQ_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
            VXQ_CUDA(cudaEventCreateWithFlags(&ev_rc, cudaEventDisableTiming));
            VXQ_CUDA(cudaEventCreateWithFlags(&ev_val, cudaEventDisableTiming));
        }
        DevBuf<int64_t> drows, dcols;
        if (m > 0) {
            drows = DevBuf<int64_t>(m, s);
            dcols = DevBuf<int64_t>(m, s);
            if (implied) {
                k_triangle_coo<<<nblk(m), TB, 0, s>>>(n, m, drows.get(), dcols.get());
                VXQ_CHECK_LAUNCH();
            } else {
                VXQ_CUDA(cudaMemcpyAsync(drows.get(), rows, m * sizeof(int64_t), cudaMemcpyDefault, s));
                VXQ_CUDA(cudaMemcpyAsync(dcols.get(), cols, m * sizeof(int64_t), cudaMemcpyDefault, s));
            }
            VXQ_CUDA(cudaEventRecord(ev_rc, s));
            VXQ_CUDA(cudaStreamWaitEvent(s2, ev_rc, 0));  // one transfer at a time on PCIe
            VXQ_CUDA(cudaMemcpyAsync(dval.get(), values, m * sizeof(double), cudaMemcpyDefault,
                                     s2));
            VXQ_CUDA(cudaEventRecord(ev_val, s2));
            ph.mark("h2d");
            k_validate_coo<<<nblk(m), TB, 0, s>>>(n, m, drows.get(), dcols.get(), nullptr,
                                                  err.get());
            VXQ_CHECK_LAUNCH();
            int herr = 0;
            VXQ_CUDA(cudaMemcpyAsync(&herr, err.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
            VXQ_CUDA(cudaStreamSynchronize(s));
            if (herr) cudaStreamSynchronize(s2);  // do not free dval under an in-flight copy
            VXQ_REQUIRE(!(herr & 1), "couplings must satisfy 0 <= i < j < n");
            VXQ_REQUIRE(!(herr & 2), "couplings must be sorted and unique by (i, j)");
            ph.mark("validate");
            k_count_deg<<<nblk(m), TB, 0, s>>>(m, drows.get(), dcols.get(), deg_up.get(),
                                               deg_lo.get(), P->coo_i, P->coo_j);
            VXQ_CHECK_LAUNCH();
        }
        VXQ_CUDA(cudaMemcpyAsync(P->lower_count, deg_lo.get(), n * sizeof(int32_t),
                                 cudaMemcpyDeviceToDevice, s));
        k_row_total<<<nblk(n + 1), TB, 0, s>>>(n, deg_up.get(), deg_lo.get(), tot.get());
        VXQ_CHECK_LAUNCH();
        // scans (int32 degrees widened into int64 scans)
        widen_i32_i64(n, deg_up.get(), up64.get(), s);
        widen_i32_i64(n, deg_lo.get(), lo64.get(), s);
        size_t tmp_bytes = 0, need = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, need, tot.get(), P->indptr, n + 1, s);
        tmp_bytes = std::max(tmp_bytes, need);
        cub::DeviceScan::ExclusiveSum(nullptr, need, up64.get(), ustart.get(), n + 1, s);
        tmp_bytes = std::max(tmp_bytes, need);
        DevBuf<int32_t> sorted_cols(std::max<int64_t>(m, 1), s), perm_in(std::max<int64_t>(m, 1), s),
            perm(std::max<int64_t>(m, 1), s);
        int end_bit = 1;
        while ((1LL << end_bit) < n) ++end_bit;
        if (m > 0) {
            cub::DeviceRadixSort::SortPairs(nullptr, need, P->coo_j, sorted_cols.get(),
                                            perm_in.get(), perm.get(), (int)m, 0, end_bit, s);
            tmp_bytes = std::max(tmp_bytes, need);
        }
        DevBuf<uint8_t> tmp(std::max<size_t>(tmp_bytes, 1), s);
        need = tmp_bytes;
        VXQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), need, tot.get(), P->indptr, n + 1, s));
        need = tmp_bytes;
        VXQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), need, up64.get(), ustart.get(), n + 1, s));
        need = tmp_bytes;
        VXQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), need, lo64.get(), lstart.get(), n + 1, s));
        if (m > 0) {
            k_iota<<<nblk(m), TB, 0, s>>>(m, perm_in.get());
            VXQ_CHECK_LAUNCH();
            need = tmp_bytes;
            VXQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), need, P->coo_j, sorted_cols.get(),
                                                     perm_in.get(), perm.get(), (int)m, 0,
                                                     end_bit, s));
            VXQ_CUDA(cudaStreamWaitEvent(s, ev_val, 0));  // the values have landed
            k_check_finite<<<nblk(m), TB, 0, s>>>(m, dval.get(), err.get());
            VXQ_CHECK_LAUNCH();
            k_fill_upper<<<nblk(m), TB, 0, s>>>(m, P->coo_i, P->coo_j, dval.get(), P->indptr,
                                                deg_lo.get(), ustart.get(), P->indices,
                                                P->data64);
            VXQ_CHECK_LAUNCH();
            k_fill_lower<<<nblk(m), TB, 0, s>>>(m, sorted_cols.get(), perm.get(), P->coo_i,
                                                dval.get(), P->indptr, lstart.get(), P->indices,
                                                P->data64);
            VXQ_CHECK_LAUNCH();
            k_convert<<<nblk(nnz), TB, 0, s>>>(nnz, P->data64, P->data32);
            VXQ_CHECK_LAUNCH();
        }
        ph.mark("csr");
        // max row length (dispatch heuristics)
        {
            DevBuf<int64_t> mx(1, s);
            need = 0;
            cub::DeviceReduce::Max(nullptr, need, tot.get(), mx.get(), n, s);
            DevBuf<uint8_t> t2(std::max<size_t>(need, 1), s);
            VXQ_CUDA(cub::DeviceReduce::Max(t2.get(), need, tot.get(), mx.get(), n, s));
            VXQ_CUDA(cudaMemcpyAsync(&P->max_row_nnz, mx.get(), sizeof(int64_t),
                                     cudaMemcpyDeviceToHost, s));
        }
        // uniform magnitude (+-c couplings, e.g. SK)
        if (m > 0) {
            DevBuf<unsigned long long> mm(2, s);
            unsigned long long init[2] = {~0ULL, 0ULL};
            VXQ_CUDA(cudaMemcpyAsync(mm.get(), init, sizeof(init), cudaMemcpyHostToDevice, s));
            k_abs_minmax<<<(unsigned)std::min<int64_t>(nblk(m), 148 * 16), TB, 0, s>>>(m, dval.get(), mm.get(), mm.get() + 1);
            VXQ_CHECK_LAUNCH();
            unsigned long long res[2];
            VXQ_CUDA(cudaMemcpyAsync(res, mm.get(), sizeof(res), cudaMemcpyDeviceToHost, s));
            VXQ_CUDA(cudaStreamSynchronize(s));
            double a, b;
            memcpy(&a, &res[0], 8);
            memcpy(&b, &res[1], 8);
            P->uniform_magnitude = (a == b) && a > 0;
            P->magnitude = b;
            int herr = 0;
            VXQ_CUDA(cudaMemcpy(&herr, err.get(), sizeof(int), cudaMemcpyDeviceToHost));
            VXQ_REQUIRE(!(herr & 4), "non-finite coupling value");
        }
        ph.mark("stats");
        encode_energy(P, s);
        VXQ_CUDA(cudaStreamSynchronize(s));
        ph.mark("encode");
    } catch (...) {
        delete P;
        throw;
    }
    return P;
}

void problem_set_fields(Problem* P, const double* h, double offset, cudaStream_t s) {
    VXQ_REQUIRE(std::isfinite(offset), "offset must be finite");
    VXQ_CUDA(cudaMemcpyAsync(P->h64, h, P->n * sizeof(double), cudaMemcpyDefault, s));
    k_fields<<<nblk(P->n), TB, 0, s>>>(P->n, P->h64, P->h32, P->g64, P->g32);
    VXQ_CHECK_LAUNCH();
    P->offset = offset;
    encode_energy(P, s);
    VXQ_CUDA(cudaStreamSynchronize(s));
    std::lock_guard<std::mutex> g(P->mu);
    P->lambda0 = NAN;
    P->c0 = NAN;
}

double problem_lambda0(Problem* p, cudaStream_t s) {
    std::lock_guard<std::mutex> g(p->mu);
    if (!std::isnan(p->lambda0)) return p->lambda0;
    DevBuf<unsigned long long> mx(1, s);
    VXQ_CUDA(cudaMemsetAsync(mx.get(), 0, sizeof(unsigned long long), s));
    k_field_scale<<<(unsigned)std::min<int64_t>(ceil_div(p->n, kFsWarps), 148 * 8),
                    32 * kFsWarps, 0, s>>>(p->n, p->indptr, p->lower_count, p->data64, p->h64,
                                            mx.get());
    VXQ_CHECK_LAUNCH();
    unsigned long long bits = 0;
    VXQ_CUDA(cudaMemcpyAsync(&bits, mx.get(), sizeof(bits), cudaMemcpyDeviceToHost, s));
    VXQ_CUDA(cudaStreamSynchronize(s));
    double fs;
    memcpy(&fs, &bits, 8);
    p->lambda0 = std::max(fs, 1e-12);  // parallel_annealing.py:25
    return p->lambda0;
}

double problem_c0(Problem* p, cudaStream_t s) {
    std::lock_guard<std::mutex> g(p->mu);
    if (!std::isnan(p->c0)) return p->c0;
    double c0 = 1.0;  // bifurcation.py:31-34
    if (p->m > 0) {
        p->eig = eig_max(p, -1.0, s);  // lambda_max(-A), eig_extreme(..., "max")
        const double lam = p->eig.value;
        c0 = lam > 1e-12 ? 1.0 / lam : 1.0;
    }
    p->c0 = c0;
    return c0;
}

}  // namespace vxq
