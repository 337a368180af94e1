// eigen.cu -- lambda_max of the SBM dynamics coupling matrix B = -A for the automatic c0.
//
// Restates eig_extreme(mat, "max") (solvers/eigen.py:35-56) as called by resolve_c0
// (solvers/bifurcation.py:25-34), on the device:
//   n <= 512 (DENSE_LIMIT, eigen.py:16,45-48): the reference takes the exact dense
//       eigenvalue (np.linalg.eigvalsh).  Here: Lanczos with full reorthogonalisation
//       (two classical Gram-Schmidt passes per step) run to the full dimension in one CTA,
//       so the tridiagonal is orthogonally similar to B up to rounding, and its largest
//       eigenvalue by Sturm bisection -- the exact value to a few ulps of ||B||.
//   n > 512 (eigen.py:50-56): the reference runs ARPACK (k=1, 'LA', tol 1e-8) and returns
//       theta + ||B v - theta v||, the Ritz value pushed outward by its residual.  Here:
//       Lanczos without reorthogonalisation (the O(nnz) steps on the device); every check
//       computes, on the host as ARPACK does for its small projected problem, the largest
//       Ritz value theta of the k x k tridiagonal T_k and, by inverse iteration on T_k, the
//       residual estimate |beta_k u_k| of its Ritz vector; converged when that is
//       <= tol |theta| (ARPACK's criterion, tol 1e-8).  Then y = sum_j u_j v_j is assembled
//       from the Lanczos basis (kept in pool memory while it fits; else the recurrence is
//       replayed from the same start vector: identical kernels => identical v_j), and the
//       returned value is theta + ||B y - theta y|| / ||y|| -- the explicit residual, as
//       the reference computes it.
//   No convergence within the iteration cap (eigen.py:49-52: ArpackNoConvergence): the
//       Gershgorin bound max_i (B_ii + sum_{j!=i} |B_ij|) = max_i sum_j |A_ij|
//       (eigen.py:21-32).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <vector>

#include "vxq_internal.h"

namespace vxq {

namespace {

constexpr int TB = 256;
inline unsigned nblk(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, TB)); }

constexpr int kDenseLimit = 512;       // eigen.py:16
constexpr double kTol = 1e-8;          // eigen.py:17 (ARPACK tol)
constexpr int64_t kMaxIter = 20000;    // Lanczos steps before the Gershgorin fallback

__device__ __forceinline__ double start_entry(int64_t i) {
    U64x4 o = philox4x64_10((uint64_t)i + 1, 0, 0x5eed, 0, 0x1a2b3c4dULL, 0);
    return uniform_from_raw(o.v[0], -1.0, 2.0);
}

// ---------------------------------------------------------------- n <= 512: one CTA
template <int NT>
__device__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < NT / 32; ++k) s += red[k];  // fixed order: deterministic
    return s;
}

// Lanczos with full reorthogonalisation to dimension n: alpha[0..k), beta[0..k-1)
// describe T_k; *kout = k.  The basis V [n][n] lives in dynamic shared memory when it fits
// (n <= 160: the CGS2 passes then read it at smem latency -- cfg1's c0 went from ~7 ms to
// well under 1 ms), else in the global scratch Vg.
__global__ void __launch_bounds__(kDenseLimit) k_lanczos_full(
    int n, const int64_t* indptr, const int32_t* indices, const double* data, double sign,
    double* Vg, int v_in_smem, double* alpha, double* beta, int* kout) {
    __shared__ double v[kDenseLimit], w[kDenseLimit], c[kDenseLimit], red[kDenseLimit / 32];
    extern __shared__ double Vs[];
    double* V = v_in_smem ? Vs : Vg;
    const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
    constexpr int NW = kDenseLimit / 32;
    double vi = i < n ? start_entry(i) : 0.0;
    const double nrm = sqrt(block_sum<kDenseLimit>(vi * vi, red));
    vi /= nrm;
    v[i] = vi;
    double vprev = 0.0, bprev = 0.0, scale = 0.0;
    int k = 0;
    while (k < n) {
        if (i < n) V[(int64_t)k * n + i] = vi;
        __syncthreads();
        double wi = 0.0;
        if (i < n) {
            for (int64_t q = indptr[i]; q < indptr[i + 1]; ++q) wi += data[q] * v[indices[q]];
            wi *= sign;
        }
        const double a = block_sum<kDenseLimit>(vi * wi, red);
        wi = wi - a * vi - bprev * vprev;
        for (int pass = 0; pass < 2; ++pass) {  // CGS2 against v_0..v_k
            w[i] = wi;
            __syncthreads();
            for (int j = warp; j <= k; j += NW) {
                double s = 0.0;
                for (int l = lane; l < n; l += 32) s += V[(int64_t)j * n + l] * w[l];
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) c[j] = s;
            }
            __syncthreads();
            if (i < n) {
                double corr = 0.0;
                for (int j = 0; j <= k; ++j) corr += c[j] * V[(int64_t)j * n + i];
                wi -= corr;
            }
            __syncthreads();
        }
        const double b = sqrt(block_sum<kDenseLimit>(wi * wi, red));
        if (i == 0) {
            alpha[k] = a;
            beta[k] = b;
        }
        ++k;
        scale = fmax(scale, fabs(a) + b + bprev);
        if (!(b > 1e-13 * scale)) break;  // invariant subspace: T_k is exact
        vprev = vi;
        vi = i < n ? wi / b : 0.0;
        bprev = b;
        v[i] = vi;
    }
    if (i == 0) *kout = k;
}

// ---------------------------------------------------------------- n > 512: kernels
// y = sign * A x (warp per row)
__global__ void k_spmv(int64_t n, const int64_t* indptr, const int32_t* indices,
                       const double* data, double sign, const double* x, double* y) {
    int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    double acc = 0.0;
    for (int64_t k = indptr[row] + lane; k < indptr[row + 1]; k += 32)
        acc += data[k] * x[indices[k]];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[row] = sign * acc;
}

constexpr int RB = 512;  // reduction blocks (fixed => deterministic)

// part[b] = sum over this block's strided range of a[i]*b[i]  (b == nullptr: a[i]^2)
// or, with theta given, of (a[i] - theta*b[i])^2
__global__ void k_dot_partial(int64_t n, const double* a, const double* b, double* part,
                              const double* theta) {
    __shared__ double sh[TB];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)TB + threadIdx.x; i < n; i += (int64_t)TB * gridDim.x) {
        if (theta) {
            const double r = a[i] - (*theta) * b[i];
            acc += r * r;
        } else {
            acc += a[i] * b[i];
        }
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = TB / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// out = sum of nb partials (sqrt if root): 1024 threads, four independent accumulators per
// thread so loads overlap (a 125k-entry sum was ~200 us when each add waited on its load);
// fixed order => deterministic
constexpr int kSumThreads = 1024;
__global__ void __launch_bounds__(kSumThreads) k_sum_partials(int nb, const double* part,
                                                              double* out, int root) {
    __shared__ double sh[kSumThreads];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int i = threadIdx.x;
    for (; i + 3 * kSumThreads < nb; i += 4 * kSumThreads) {
        a0 += part[i];
        a1 += part[i + kSumThreads];
        a2 += part[i + 2 * kSumThreads];
        a3 += part[i + 3 * kSumThreads];
    }
    for (; i < nb; i += kSumThreads) a0 += part[i];
    sh[threadIdx.x] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    for (int o = kSumThreads / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = root ? sqrt(sh[0]) : sh[0];
}

// w = w - alpha v - beta vprev  (alpha, beta device scalars)
__global__ void k_axpy2(int64_t n, double* w, const double* v, const double* vp,
                        const double* alpha, const double* beta) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) w[i] = w[i] - (*alpha) * v[i] - (*beta) * vp[i];
}

// y += u * v  (u device scalar)
__global__ void k_axpy(int64_t n, double* y, const double* v, const double* u) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) y[i] += (*u) * v[i];
}

__global__ void k_scale_into(int64_t n, const double* w, const double* nrm, double* v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = w[i] / (*nrm);
}

// fused Lanczos step pieces (fixed grids and reduction orders: deterministic)
// w = sign * A v (one warp per row, one row per warp: short rows are latency-bound, so every
// row gets its own warp); part[b] = this block's sum v_i w_i
__global__ void __launch_bounds__(TB) k_spmv_dot(int64_t n, const int64_t* indptr,
                                                 const int32_t* indices, const double* data,
                                                 double sign, const double* v, double* w,
                                                 double* part) {
    __shared__ double sh[TB / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double dsum = 0.0;
    const int64_t row = (int64_t)blockIdx.x * (TB / 32) + wid;
    if (row < n) {
        double acc = 0.0;
        for (int64_t k = indptr[row] + lane; k < indptr[row + 1]; k += 32)
            acc += data[k] * v[indices[k]];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        acc *= sign;
        if (lane == 0) {
            w[row] = acc;
            dsum = v[row] * acc;
        }
    }
    if (lane == 0) sh[wid] = dsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < TB / 32; ++k) t += sh[k];
        part[blockIdx.x] = t;
    }
}

// the same for short rows (mean degree < 16): one THREAD per row -- a warp per 3-entry row
// leaves 29 lanes idle and needs ~n/9472 dependent load waves (n = 10^6: ~200 us per step)
__global__ void __launch_bounds__(TB) k_spmv_dot_rows(int64_t n, const int64_t* indptr,
                                                      const int32_t* indices,
                                                      const double* data, double sign,
                                                      const double* v, double* w,
                                                      double* part) {
    __shared__ double sh[TB];
    const int64_t row = (int64_t)blockIdx.x * TB + threadIdx.x;
    double d = 0.0;
    if (row < n) {
        double acc = 0.0;
        for (int64_t k = indptr[row]; k < indptr[row + 1]; ++k) acc += data[k] * v[indices[k]];
        acc *= sign;
        w[row] = acc;
        d = v[row] * acc;
    }
    sh[threadIdx.x] = d;
    __syncthreads();
    for (int o = TB / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// Dense uniform-|J| problems (SK family): A = c K with K in {-1, 0, +1}.  The Lanczos SpMV
// then streams K as int8 (n^2 bytes: 100 MB at n = 10^4) instead of the CSR's 12 bytes per
// entry (1.2 GB): w_i = (sign c) * sum_j K_ij v_j, one warp per row, 4 columns per lane per
// pass (coalesced K bytes and v words; zero entries skipped), fixed reduction order
// (deterministic).
__global__ void k_build_dense_k8(int64_t n, int64_t ld, const int64_t* __restrict__ indptr,
                                 const int32_t* __restrict__ indices,
                                 const double* __restrict__ data, int8_t* __restrict__ K) {
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    for (int64_t k = indptr[row] + lane; k < indptr[row + 1]; k += 32)
        K[row * ld + indices[k]] = data[k] > 0.0 ? 1 : -1;
}

// one CTA of kDenseSpmvThreads per row (a warp per row left each warp ~80 dependent passes
// over its 10 KB row); partial sums combined in a fixed order; part[b] = row b's v_i w_i
constexpr int kDenseSpmvThreads = 128;
__global__ void __launch_bounds__(kDenseSpmvThreads) k_dense_spmv_dot(
    int64_t n, int64_t ld, const int8_t* __restrict__ K, double scale, const double* v,
    double* w, double* part) {
    __shared__ double sh[kDenseSpmvThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t row = blockIdx.x;
    const int8_t* kr = K + row * ld;
    double acc = 0.0;
    // 4 K bytes per thread per pass: the threads' v reads stay within a few lines per
    // instruction (16 bytes per thread spread them over 32 lines: 88 ms instead of 27 for
    // the SK n = 10^4 c0); zero entries (incl. the row padding past n) never touch v
    for (int64_t j = (int64_t)threadIdx.x * 4; j < ld; j += 4 * kDenseSpmvThreads) {
        const char4 k4 = *reinterpret_cast<const char4*>(kr + j);
        if (k4.x) acc += k4.x > 0 ? v[j] : -v[j];
        if (k4.y) acc += k4.y > 0 ? v[j + 1] : -v[j + 1];
        if (k4.z) acc += k4.z > 0 ? v[j + 2] : -v[j + 2];
        if (k4.w) acc += k4.w > 0 ? v[j + 3] : -v[j + 3];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) sh[wid] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < kDenseSpmvThreads / 32; ++k) t += sh[k];
        t *= scale;
        w[row] = t;
        part[row] = v[row] * t;
    }
}

// w = w - alpha v - beta vprev; part[b] = this block's sum w_i^2
__global__ void __launch_bounds__(TB) k_axpy2_norm(int64_t n, double* w, const double* v,
                                                   const double* vp, const double* alpha,
                                                   const double* beta, double* part) {
    __shared__ double sh[TB];
    const double a = *alpha, b = *beta;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)TB + threadIdx.x; i < n; i += (int64_t)TB * gridDim.x) {
        const double x = w[i] - a * v[i] - b * vp[i];
        w[i] = x;
        acc += x * x;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int o = TB / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// v = w / beta, and (optionally) the same into the stored basis row
__global__ void k_scale_store(int64_t n, const double* w, const double* nrm, double* v,
                              double* vstore) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = w[i] / (*nrm);
    v[i] = x;
    if (vstore) vstore[i] = x;
}

// y (+)= sum_j u_j V[j] over one chunk of the stored basis (V row-major [k][n])
__global__ void k_basis_combine(int64_t n, int64_t k, const double* V, const double* u,
                                double* y, int accumulate) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = accumulate ? y[i] : 0.0;
    for (int64_t j = 0; j < k; ++j) acc += u[j] * V[j * n + i];
    y[i] = acc;
}

__global__ void k_start_vec(int64_t n, double* v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = start_entry(i);
}

// eigenvalues of T_k below x (Sturm count)
__device__ int sturm_count(int64_t k, const double* a, const double* b, double x) {
    int c = 0;
    double q = a[0] - x;
    if (q < 0) ++c;
    for (int64_t i = 1; i < k; ++i) {
        double d = (q == 0.0) ? 1e-300 : q;
        q = a[i] - x - b[i - 1] * b[i - 1] / d;
        if (q < 0) ++c;
    }
    return c;
}

// largest eigenvalue of T_k: Gershgorin bracket, 256-way multisection, final bisection
constexpr int kMS = 256;
__global__ void __launch_bounds__(kMS) k_tridiag_max(int64_t k, const double* a, const double* b,
                                                     double* out) {
    __shared__ double s_lo, s_hi;
    __shared__ int s_first;
    if (threadIdx.x == 0) {
        double lo = 1e300, hi = -1e300;
        for (int64_t i = 0; i < k; ++i) {
            double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i < k - 1 ? fabs(b[i]) : 0.0);
            lo = fmin(lo, a[i] - r);
            hi = fmax(hi, a[i] + r);
        }
        s_lo = lo;
        s_hi = hi;
    }
    __syncthreads();
    for (int round = 0; round < 64; ++round) {
        const double lo = s_lo, hi = s_hi;
        const double x = lo + (hi - lo) * ((double)(threadIdx.x + 1) / (double)(kMS + 1));
        if (threadIdx.x == 0) s_first = kMS;
        __syncthreads();
        const bool ok = x > lo && x < hi;
        if (ok && sturm_count(k, a, b, x) >= k) atomicMin(&s_first, (int)threadIdx.x);
        __syncthreads();
        const int f = s_first;
        const double xf = lo + (hi - lo) * ((double)(f + 1) / (double)(kMS + 1));
        const double xp = lo + (hi - lo) * ((double)f / (double)(kMS + 1));
        __syncthreads();
        if (threadIdx.x == 0) {
            const double nhi = f < kMS ? xf : hi;
            const double nlo = f > 0 ? xp : lo;
            s_lo = nlo > lo ? nlo : lo;
            s_hi = nhi < hi ? nhi : hi;
        }
        __syncthreads();
        if (!(s_hi - s_lo < hi - lo)) break;  // no progress: down to a few ulps
    }
    if (threadIdx.x == 0) {
        double lo = s_lo, hi = s_hi;
        for (int it = 0; it < 200; ++it) {
            double mid = 0.5 * (lo + hi);
            if (mid <= lo || mid >= hi) break;
            if (sturm_count(k, a, b, mid) >= k) hi = mid;
            else lo = mid;
        }
        *out = hi;
    }
}

// Gershgorin bound of B = -A (zero diagonal): max_i sum_j |A_ij|
__global__ void k_row_abs_max(int64_t n, const int64_t* indptr, const double* data,
                              unsigned long long* maxbits) {
    int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    double acc = 0.0;
    for (int64_t k = indptr[row] + lane; k < indptr[row + 1]; k += 32) acc += fabs(data[k]);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(acc));
}

template <typename T>
T to_host(const T* dev, cudaStream_t s) {
    T h;
    VXQ_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
    VXQ_CUDA(cudaStreamSynchronize(s));
    return h;
}

// ---- host side of the convergence checks (T_k is k x k: O(k) work per check, like the
// small dense problems ARPACK itself solves on the host; the O(nnz) work stays on the GPU)
int sturm_count_host(int64_t k, const double* a, const double* b, double x) {
    int c = 0;
    double q = a[0] - x;
    if (q < 0) ++c;
    for (int64_t i = 1; i < k; ++i) {
        const double d = (q == 0.0) ? 1e-300 : q;
        q = a[i] - x - b[i - 1] * b[i - 1] / d;
        if (q < 0) ++c;
    }
    return c;
}

// largest eigenvalue of T_k by bisection on the Sturm count (Gershgorin bracket)
double tridiag_max_host(int64_t k, const double* a, const double* b) {
    double lo = 1e300, hi = -1e300;
    for (int64_t i = 0; i < k; ++i) {
        const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i < k - 1 ? std::fabs(b[i]) : 0.0);
        lo = std::fmin(lo, a[i] - r);
        hi = std::fmax(hi, a[i] + r);
    }
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (sturm_count_host(k, a, b, mid) >= k) hi = mid;
        else lo = mid;
    }
    return hi;
}

// Ritz vector u of theta = lambda_max(T_k) by two steps of inverse iteration with the
// positive-definite (theta + delta) I - T_k (LDL^T without pivoting; delta grows tenfold if
// rounding leaves a non-positive pivot); returns |beta_{k-1} u_{k-1}| (ARPACK's residual
// estimate), +inf if no factorisation was usable
double ritz_vector_host(int64_t k, const double* a, const double* b, double theta,
                        std::vector<double>& u) {
    std::vector<double> l(k), d(k);
    u.assign(k, 1.0);
    double tn = 0.0;
    for (int64_t i = 0; i < k; ++i)
        tn = std::fmax(tn, std::fabs(a[i]) + (i > 0 ? std::fabs(b[i - 1]) : 0.0) +
                               (i + 1 < k ? std::fabs(b[i]) : 0.0));
    double delta = 1e-11 * std::fmax(tn, 1e-300);
    for (int attempt = 0; attempt < 8; ++attempt, delta *= 10.0) {
        const double mu = theta + delta;
        bool ok = (d[0] = mu - a[0]) > 0;
        for (int64_t i = 1; ok && i < k; ++i) {
            l[i] = -b[i - 1] / d[i - 1];
            d[i] = (mu - a[i]) - b[i - 1] * b[i - 1] / d[i - 1];
            ok = d[i] > 0;
        }
        if (!ok) continue;
        u.assign(k, 1.0);
        for (int it = 0; it < 2; ++it) {
            for (int64_t i = 1; i < k; ++i) u[i] -= l[i] * u[i - 1];
            for (int64_t i = 0; i < k; ++i) u[i] /= d[i];
            for (int64_t i = k - 2; i >= 0; --i) u[i] -= l[i + 1] * u[i + 1];
            double ss = 0.0;
            for (int64_t i = 0; i < k; ++i) ss += u[i] * u[i];
            ss = 1.0 / std::sqrt(ss);
            for (int64_t i = 0; i < k; ++i) u[i] *= ss;
        }
        return std::fabs(b[k - 1] * u[k - 1]);
    }
    return INFINITY;
}

EigInfo eig_max_small(const Problem* p, double sign, cudaStream_t s) {
    const int n = (int)p->n;
    const size_t vbytes = (size_t)n * n * sizeof(double);
    const bool smem = vbytes <= 200 * 1024;
    DevBuf<double> V(smem ? 1 : (size_t)n * n, s), alpha(n, s), beta(n, s), theta(1, s);
    DevBuf<int> kout(1, s);
    if (smem)
        VXQ_CUDA(cudaFuncSetAttribute(k_lanczos_full, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)vbytes));
    k_lanczos_full<<<1, kDenseLimit, smem ? vbytes : 0, s>>>(
        n, p->indptr, p->indices, p->data64, sign, V.get(), smem ? 1 : 0, alpha.get(),
        beta.get(), kout.get());
    VXQ_CHECK_LAUNCH();
    const int k = to_host(kout.get(), s);
    k_tridiag_max<<<1, kMS, 0, s>>>(k, alpha.get(), beta.get(), theta.get());
    VXQ_CHECK_LAUNCH();
    EigInfo r;
    r.theta = r.value = to_host(theta.get(), s);
    r.residual = 0.0;
    r.iterations = k;
    r.method = kEigDense;
    return r;
}

struct Lanczos {
    int64_t n;
    const Problem* p;
    double sign;
    cudaStream_t s;
    DevBuf<double> v0, v1, w, part, zero;
    double* vp;
    double* v;
    unsigned spmv_blocks;
    bool short_rows;  // mean row length < 16: one thread per row
    DevBuf<int8_t> kd;  // dense uniform-|J| problems: K as int8 [n][ld]
    int64_t ld = 0;
    double kscale = 0.0;
    // stored basis V[j] = v_j for j < basis_rows, grown in chunks of kChunk rows while the
    // total stays within basis_cap rows (memory comes from the retained stream-ordered pool)
    static constexpr int64_t kChunk = 128;
    std::vector<DevBuf<double>> chunks;
    int64_t basis_rows = 0, basis_cap = 0;
    bool storing = false;

    double* basis_row(int64_t j) {  // row j of the stored basis, allocating its chunk
        if (!storing || j >= basis_cap) return nullptr;
        const int64_t c = j / kChunk;
        if (c >= (int64_t)chunks.size()) {
            // only from memory the pool already holds: growing it maps fresh pages (seconds
            // for GBs), far more than replaying the recurrence costs
            if (!pool_has((size_t)kChunk * n * sizeof(double))) {
                storing = false;
                return nullptr;
            }
            chunks.emplace_back((size_t)kChunk * n, s);
        }
        basis_rows = std::max(basis_rows, j + 1);
        return chunks[c].get() + (j % kChunk) * n;
    }

    static bool pool_has(size_t bytes) {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess)
            return false;
        uint64_t reserved = 0, used = 0;
        if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) !=
                cudaSuccess ||
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) != cudaSuccess)
            return false;
        return reserved >= used + bytes + bytes / 2;  // headroom for fragmentation
    }

    Lanczos(const Problem* p_, double sign_, cudaStream_t s_)
        : n(p_->n), p(p_), sign(sign_), s(s_), v0(n, s_), v1(n, s_), w(n, s_),
          part(std::max<int64_t>(RB, ceil_div(n * 32, TB)), s_), zero(1, s_) {
        short_rows = p_->nnz < 16 * n;
        spmv_blocks = (unsigned)ceil_div(short_rows ? n : n * 32, TB);
        VXQ_CUDA(cudaMemsetAsync(zero.get(), 0, sizeof(double), s));
        // dense uniform-|J| problem: int8 K for the SpMV (n ld <= 1 GiB, >= 1/8 filled;
        // VXQ_EIG_DENSE=0 keeps the CSR SpMV)
        const char* e = getenv("VXQ_EIG_DENSE");
        ld = ceil_div(n, 128) * 128;
        if (p_->uniform_magnitude && !(e && atoi(e) == 0) && (double)p_->nnz >= (double)n * n / 8 &&
            (double)n * ld <= (double)(1ull << 30)) {
            kd = DevBuf<int8_t>(n * ld, s_);
            VXQ_CUDA(cudaMemsetAsync(kd.get(), 0, n * ld, s_));
            k_build_dense_k8<<<(unsigned)ceil_div(n * 32, TB), TB, 0, s_>>>(
                n, ld, p_->indptr, p_->indices, p_->data64, kd.get());
            VXQ_CHECK_LAUNCH();
            kscale = sign * p_->magnitude;
            spmv_blocks = (unsigned)n;  // one CTA per row: n partials
            if (n > (int64_t)part.count) part = DevBuf<double>(n, s_);
        }
    }

    // v_0 = start / ||start||, vprev = 0
    void start(double* nrm) {
        vp = v0.get();
        v = v1.get();
        VXQ_CUDA(cudaMemsetAsync(vp, 0, n * sizeof(double), s));
        k_start_vec<<<nblk(n), TB, 0, s>>>(n, w.get());
        k_dot_partial<<<RB, TB, 0, s>>>(n, w.get(), w.get(), part.get(), nullptr);
        k_sum_partials<<<1, kSumThreads, 0, s>>>(RB, part.get(), nrm, 1);
        k_scale_store<<<nblk(n), TB, 0, s>>>(n, w.get(), nrm, v, basis_row(0));
        VXQ_CHECK_LAUNCH();
    }

    // step k: w = B v_k - alpha_k v_k - beta_{k-1} v_{k-1}; beta_k = ||w||  (4 launches)
    void step(int64_t k, double* alpha, double* beta) {
        if (kd.get())
            k_dense_spmv_dot<<<spmv_blocks, kDenseSpmvThreads, 0, s>>>(n, ld, kd.get(), kscale, v,
                                                                       w.get(), part.get());
        else if (short_rows)
            k_spmv_dot_rows<<<spmv_blocks, TB, 0, s>>>(n, p->indptr, p->indices, p->data64,
                                                       sign, v, w.get(), part.get());
        else
            k_spmv_dot<<<spmv_blocks, TB, 0, s>>>(n, p->indptr, p->indices, p->data64, sign, v,
                                                  w.get(), part.get());
        k_sum_partials<<<1, kSumThreads, 0, s>>>((int)spmv_blocks, part.get(), alpha + k, 0);
        k_axpy2_norm<<<RB, TB, 0, s>>>(n, w.get(), v, vp, alpha + k,
                                       k > 0 ? beta + k - 1 : zero.get(), part.get());
        k_sum_partials<<<1, kSumThreads, 0, s>>>(RB, part.get(), beta + k, 1);
        VXQ_CHECK_LAUNCH();
    }

    // v_{k+1} = w / beta_k (stored as basis row k+1 when it fits)
    void advance(int64_t k, const double* beta) {
        std::swap(vp, v);
        k_scale_store<<<nblk(n), TB, 0, s>>>(n, w.get(), beta + k, v, basis_row(k + 1));
        VXQ_CHECK_LAUNCH();
    }
};

EigInfo eig_max_lanczos(const Problem* p, double sign, cudaStream_t s) {
    const int64_t n = p->n;
    const bool timing = getenv("VXQ_EIG_TIMING") != nullptr;  // debugging: phase times
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t_begin = now();
    double check_ms = 0.0;
    int64_t cap = kMaxIter;
    if (const char* e = getenv("VXQ_LANCZOS_MAXITER"))  // tests: force the fallback
        cap = std::max<int64_t>(1, atoll(e));
    const int64_t kmax = std::min<int64_t>(n, cap);
    DevBuf<double> alpha(kmax + 1, s), beta(kmax + 1, s), nrm(1, s), theta(1, s),
        u(kmax + 1, s);
    std::vector<double> ha, hb, hu;  // host copies of T_k and the Ritz vector
    Lanczos lz(p, sign, s);
    // keep the Lanczos basis (<= 16 GB, only in memory the pool already holds: see
    // basis_row) -- the Ritz vector is then one pass over it instead of a replay
    lz.basis_cap = std::min<int64_t>(kmax + 1, (int64_t)(16.0 * (1ull << 30) / (8.0 * n)));
    lz.storing = lz.basis_cap >= Lanczos::kChunk;
    lz.start(nrm.get());
    EigInfo r;
    int64_t kk = -1;  // T_{kk} converged (size kk)
    double th = 0.0;
    int64_t next_check = 10, last_check = 0;
    for (int64_t k = 0; k < kmax; ++k) {
        lz.step(k, alpha.get(), beta.get());
        const bool last = k + 1 == kmax;
        if (last || k + 1 == next_check) {
            const auto tc = now();
            // the new entries of T_k; theta and the Ritz vector of T_k on the host
            ha.resize(k + 1);
            hb.resize(k + 1);
            VXQ_CUDA(cudaMemcpyAsync(ha.data() + last_check, alpha.get() + last_check,
                                     (k + 1 - last_check) * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
            VXQ_CUDA(cudaMemcpyAsync(hb.data() + last_check, beta.get() + last_check,
                                     (k + 1 - last_check) * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
            VXQ_CUDA(cudaStreamSynchronize(s));
            // an (almost) invariant subspace ends the recurrence at the first tiny beta
            int64_t size = k + 1;
            bool breakdown = false;
            for (int64_t j = last_check; j <= k; ++j)
                if (!(hb[j] > 1e-12)) {
                    size = j + 1;
                    breakdown = true;
                    break;
                }
            th = tridiag_max_host(size, ha.data(), hb.data());
            double res_est = ritz_vector_host(size, ha.data(), hb.data(), th, hu);
            if (breakdown) res_est = 0.0;
            last_check = k + 1;
            // check interval grows with k (at most ~6 % extra steps past convergence)
            next_check = k + 1 + std::max<int64_t>(10, ((k + 1) / 16) / 10 * 10);
            if (timing) check_ms += ms(tc, now());
            if (breakdown || res_est <= kTol * std::fabs(th)) {
                kk = size;
                VXQ_CUDA(cudaMemcpyAsync(u.get(), hu.data(), kk * sizeof(double),
                                         cudaMemcpyHostToDevice, s));
                VXQ_CUDA(cudaMemcpyAsync(theta.get(), &th, sizeof(double),
                                         cudaMemcpyHostToDevice, s));
                VXQ_CUDA(cudaStreamSynchronize(s));  // host sources go out of scope
                break;
            }
        }
        if (!last) lz.advance(k, beta.get());
    }
    if (kk < 0) {  // ArpackNoConvergence -> Gershgorin (eigen.py:49-52)
        DevBuf<unsigned long long> mx(1, s);
        VXQ_CUDA(cudaMemsetAsync(mx.get(), 0, sizeof(unsigned long long), s));
        k_row_abs_max<<<(unsigned)ceil_div(n * 32, TB), TB, 0, s>>>(n, p->indptr, p->data64,
                                                                     mx.get());
        VXQ_CHECK_LAUNCH();
        const unsigned long long bits = to_host(mx.get(), s);
        double g;
        memcpy(&g, &bits, 8);
        r.value = g;
        r.theta = th;
        r.residual = NAN;
        r.iterations = kmax;
        r.method = kEigGershgorin;
        return r;
    }
    const auto t_iter = now();
    // the Ritz vector y = sum_j u_j v_j -- from the stored basis, or by replaying the
    // recurrence (same kernels, same start => the same v_j) -- then the explicit residual
    // ||B y - theta y|| / ||y||
    DevBuf<double> y(n, s), by(n, s), ynrm(1, s), rnrm(1, s);
    if (lz.storing && kk <= lz.basis_rows) {
        for (int64_t c = 0; c * Lanczos::kChunk < kk; ++c) {
            const int64_t rows = std::min<int64_t>(Lanczos::kChunk, kk - c * Lanczos::kChunk);
            k_basis_combine<<<nblk(n), TB, 0, s>>>(n, rows, lz.chunks[c].get(),
                                                   u.get() + c * Lanczos::kChunk, y.get(),
                                                   c > 0);
        }
        VXQ_CHECK_LAUNCH();
    } else {
        VXQ_CUDA(cudaMemsetAsync(y.get(), 0, n * sizeof(double), s));
        DevBuf<double> alpha2(kk, s), beta2(kk, s);
        lz.storing = false;
        lz.chunks.clear();
        lz.start(nrm.get());
        for (int64_t j = 0; j < kk; ++j) {
            k_axpy<<<nblk(n), TB, 0, s>>>(n, y.get(), lz.v, u.get() + j);
            VXQ_CHECK_LAUNCH();
            if (j + 1 == kk) break;
            lz.step(j, alpha2.get(), beta2.get());
            lz.advance(j, beta2.get());
        }
    }
    k_spmv<<<(unsigned)ceil_div(n * 32, TB), TB, 0, s>>>(n, p->indptr, p->indices, p->data64,
                                                         sign, y.get(), by.get());
    k_dot_partial<<<RB, TB, 0, s>>>(n, y.get(), y.get(), lz.part.get(), nullptr);
    k_sum_partials<<<1, kSumThreads, 0, s>>>(RB, lz.part.get(), ynrm.get(), 1);
    k_dot_partial<<<RB, TB, 0, s>>>(n, by.get(), y.get(), lz.part.get(), theta.get());
    k_sum_partials<<<1, kSumThreads, 0, s>>>(RB, lz.part.get(), rnrm.get(), 1);
    VXQ_CHECK_LAUNCH();
    const double yn = to_host(ynrm.get(), s), rn = to_host(rnrm.get(), s);
    if (timing)
        fprintf(stderr, "[vxq eig] n=%lld steps=%lld iterate %.1f ms (checks %.1f) ritz+residual "
                "%.1f ms stored=%d\n", (long long)n, (long long)kk, ms(t_begin, t_iter), check_ms,
                ms(t_iter, now()), (int)(lz.storing && kk <= lz.basis_rows));
    r.theta = th;
    r.residual = rn / yn;
    r.value = th + r.residual;  // eigen.py:56: theta + residual for "max"
    r.iterations = kk;
    r.method = kEigLanczos;
    return r;
}

}  // namespace

EigInfo eig_max(const Problem* p, double sign, cudaStream_t s) {
    if (p->n <= kDenseLimit) return eig_max_small(p, sign, s);
    return eig_max_lanczos(p, sign, s);
}

}  // namespace vxq
