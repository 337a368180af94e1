// dynamics.cu -- the batched multi-replica dynamics loop on sm_100a.
//
// PA  (solvers/parallel_annealing.py:41-45), per (row i, replica r):
//     f    = sum_k J_ik s_{j_k}          (CSR row, ascending j, sequential, starts at 0)
//     grad = (lam_t * x + f) + h_i
//     m    = alpha * m - eta * grad
//     x    = clip(x + m, -1, 1);  s = sign(x)  (sign(0) = +1)
// SBM (solvers/bifurcation.py:40-46), with B = -A, g = -h:
//     f  = sum_k B_ik q_{j_k}
//     p  = p + dt * ( -((q*q + a0) - a_t) * q + c0 * (f + g_i) )
//     q  = q + (dt*a0) * p;  |q| > q_cap => q = clip(q), p = 0
//
// Every binary op is rounded once (no FMA contraction) in the reference's evaluation
// order, and the row sum runs in the same order as scipy's csc_matvecs for X @ A_csr,
// so the fp64 build reproduces the reference's CSR path bit for bit and the fp32 build
// reproduces oracle/oracle.c's fp32 restatement bit for bit.
//
// HBM layout (one problem, R_pad replicas, V = values per lane, chunk = 32 V replicas):
//   state[i][R_pad]: replica r sits at c*32V + l*V + b  (c = r / 32V, b = (r % 32V) / 32,
//   l = r % 32), so lane l of the warp owning (row i, chunk c) loads its V replicas with
//   one 16-byte vector access and the V sign words of the chunk come out of V ballots.
//   sign bits sb[i][W], W = R_pad / 32: bit (r % 32) of word r / 32 (natural order).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <vector>

#include "vxq_internal.h"

namespace vxq {

template <typename T>
struct Operator {  // field_i = sum_k (sign * data[k]) * v[indices[k]]
    const int64_t* indptr;
    const int32_t* indices;
    const T* data;
    T sign;
};

__device__ __forceinline__ int64_t lane_base(int64_t i, int64_t R_pad, int c, int lane, int V) {
    return i * R_pad + (int64_t)c * 32 * V + (int64_t)lane * V;
}

// Random spin-word gather of the R <= 32 step: 64-byte L2 fetch hint, cfg5 PA +4.8 %
// (profiles/r02/ab_gather_ld; A/B knob VXQ_GATHER_LD: 0 = ld.global.nc,
// 1 = ld.global.cg, 2 = ld.global.nc.L1::no_allocate, 3 = ld.global.nc.L2::64B)
#ifndef VXQ_GATHER_LD
#define VXQ_GATHER_LD 3
#endif
__device__ __forceinline__ uint32_t gather_word(const uint32_t* p) {
#if VXQ_GATHER_LD == 1
    return __ldcg(p);
#elif VXQ_GATHER_LD == 2
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#elif VXQ_GATHER_LD == 3
    uint32_t v;
    asm volatile("ld.global.nc.L2::64B.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

// f[b] += t[b] for b < N.  With VXQ_PACKED=1 fp32 pairs go through the packed f32x2 add
// (FADD2, sm_100): each half rounds like __fadd_rn, so the sums are bit-identical with half
// the add issue slots -- measured +1.2 % on cfg3 PA, -0.6 % on cfg4 PA (HBM-bound), so the
// scalar adds stay the default (profiles/r02/ab_packed)
#ifndef VXQ_PACKED
#define VXQ_PACKED 0
#endif
template <typename T, int N>
__device__ __forceinline__ void addv(T* f, const T* t) {
    if constexpr (VXQ_PACKED && sizeof(T) == 4 && N % 2 == 0) {
#pragma unroll
        for (int b = 0; b < N; b += 2) {
            asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
                "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
                "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
                : "=f"(f[b]), "=f"(f[b + 1])
                : "f"(f[b]), "f"(f[b + 1]), "f"(t[b]), "f"(t[b + 1]));
        }
    } else {
#pragma unroll
        for (int b = 0; b < N; ++b) f[b] = Ops<T>::add(f[b], t[b]);
    }
}
// t[b] = a * q[b]: scalar FMULs on purpose -- ptxas (12.9) contracts mul.rn.f32x2 followed by
// add.rn.f32x2 into FFMA2 (one rounding instead of two) even with --fmad=false, which breaks
// parity; scalar products feeding the packed add stay unfused
template <typename T, int N>
__device__ __forceinline__ void mulv(T* t, T a, const T* q) {
#pragma unroll
    for (int b = 0; b < N; ++b) t[b] = Ops<T>::mul(a, q[b]);
}
// f[b] += (bit `lane` of w[b]) ? a : -a
template <typename T, int N>
__device__ __forceinline__ void add_pm(T* f, const uint32_t* w, T a, int lane) {
    T t[N];
#pragma unroll
    for (int b = 0; b < N; ++b) t[b] = ((w[b] >> lane) & 1u) ? a : -a;
    addv<T, N>(f, t);
}

// SBM q table accesses with L2 eviction hints (A/B knob VXQ_SBM_L2HINT): the neighbour
// gathers of q_t keep their lines (evict_last) while the freshly written q_{t+1} streams
// (evict_first); 0 = plain accesses
#ifndef VXQ_SBM_L2HINT
#define VXQ_SBM_L2HINT 0
#endif
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
template <typename T, int V>
__device__ __forceinline__ Vec<T, V> ld_hint(const T* p, uint64_t pol) {
    if constexpr (VXQ_SBM_L2HINT && sizeof(T) == 4 && V == 4) {
        Vec<T, V> v;
        asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                     : "=f"(v.v[0]), "=f"(v.v[1]), "=f"(v.v[2]), "=f"(v.v[3])
                     : "l"(p), "l"(pol));
        return v;
    } else {
        return *reinterpret_cast<const Vec<T, V>*>(p);
    }
}
template <typename T, int V>
__device__ __forceinline__ void st_hint(T* p, const Vec<T, V>& v, uint64_t pol) {
    if constexpr (VXQ_SBM_L2HINT && sizeof(T) == 4 && V == 4) {
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                     "f"(v.v[0]), "f"(v.v[1]), "f"(v.v[2]), "f"(v.v[3]), "l"(pol)
                     : "memory");
    } else {
        *reinterpret_cast<Vec<T, V>*>(p) = v;
    }
}

__device__ __forceinline__ int64_t pos_of(int64_t r, int V) {
    int64_t ch = 32 * V;
    int64_t c = r / ch, rem = r % ch;
    return c * ch + (rem % 32) * V + rem / 32;
}

// ------------------------------------------------------------------ init (Philox)
// rows [row0, row0 + nrows) of x/m (local indexing); draw k of stream r is row k
template <typename T>
__global__ void k_init_pa(int64_t row0, int64_t nrows, int64_t R_pad, int V, uint64_t seed,
                          int64_t rbegin, T* __restrict__ x, T* __restrict__ m) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t q0 = row0 / 4, q1 = (row0 + nrows + 3) / 4;
    if (idx >= (q1 - q0) * R_pad) return;
    int64_t q = q0 + idx / R_pad, r = idx % R_pad;
    U64x4 o = philox4x64_10((uint64_t)q + 1, 0, (uint64_t)(rbegin + r), 0, seed, 0);
    int64_t p = pos_of(r, V);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        int64_t i = 4 * q + w;
        if (i >= row0 && i < row0 + nrows) {
            double v = uniform_from_raw(o.v[w], -1.0, 2.0);  // uniform(-1, 1)
            x[(i - row0) * R_pad + p] = (T)v;
            m[(i - row0) * R_pad + p] = (T)0;
        }
    }
}

// q of rows [row0, row0+nrows) into the full (global-row) buffer q, p into the local pm;
// stream r draws n q-values then n p-values (bifurcation.py:60-61)
template <typename T>
__global__ void k_init_sbm(int64_t n, int64_t row0, int64_t nrows, int64_t R_pad, int V,
                           uint64_t seed, int64_t rbegin, double amp, T* __restrict__ q,
                           T* __restrict__ pm) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t nq = (2 * n + 3) / 4;
    if (idx >= nq * R_pad) return;
    int64_t qd = idx / R_pad, r = idx % R_pad;
    // skip quads with no local row among their draws
    const int64_t k0 = 4 * qd, k1 = k0 + 3;
    const bool q_hit = k0 < row0 + nrows && k1 >= row0;
    const bool p_hit = k0 < n + row0 + nrows && k1 >= n + row0;
    if (!q_hit && !p_hit) return;
    U64x4 o = philox4x64_10((uint64_t)qd + 1, 0, (uint64_t)(rbegin + r), 0, seed, 0);
    int64_t p = pos_of(r, V);
    const double lo = -amp, range = __dadd_rn(amp, amp);  // hi - lo
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        int64_t k = k0 + w;
        double v = uniform_from_raw(o.v[w], lo, range);
        if (k < n) {
            if (k >= row0 && k < row0 + nrows) q[k * R_pad + p] = (T)v;
        } else if (k < 2 * n) {
            const int64_t i = k - n;
            if (i >= row0 && i < row0 + nrows) pm[(i - row0) * R_pad + p] = (T)v;
        }
    }
}

// [R][n] fp64 host-order array <-> interleaved layout
template <typename T>
__global__ void k_import(const double* __restrict__ src, int64_t n, int64_t R, int64_t R_pad,
                         int V, T* __restrict__ dst) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * R_pad) return;
    int64_t r = idx / n, i = idx % n;
    T v = (r < R) ? (T)src[r * n + i] : (T)0;
    dst[i * R_pad + pos_of(r, V)] = v;
}

template <typename T>
__global__ void k_export(const T* __restrict__ src, int64_t n, int64_t R, int64_t R_pad, int V,
                         double* __restrict__ dst) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * R) return;
    int64_t r = idx / n, i = idx % n;
    dst[idx] = (double)src[i * R_pad + pos_of(r, V)];
}

// sign bits of the final analog state
template <typename T, int V>
__global__ void k_pack_signs(const T* __restrict__ x, int64_t row0, int64_t nrows, int64_t R_pad,
                             uint32_t* __restrict__ sb) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int chunks = (int)(R_pad / (32 * V));
    const int64_t il = warp / chunks;
    const int c = (int)(warp % chunks);
    if (il >= nrows) return;
    Vec<T, V> xv = *reinterpret_cast<const Vec<T, V>*>(x + lane_base(il, R_pad, c, lane, V));
    const int64_t W = R_pad / 32;
#pragma unroll
    for (int b = 0; b < V; ++b) {
        uint32_t word = __ballot_sync(0xffffffffu, xv.v[b] >= (T)0);
        if (lane == b) sb[(row0 + il) * W + c * V + b] = word;
    }
}

// Output of a step: the local exchange buffer plus, for a row-partitioned rank with
// peers, every peer's copy of it (CUDA IPC pointers over NVLink).  Each produced word /
// vector is stored to all n destinations from registers, so the exchange overlaps the
// step instead of following it as a separate all-gather.
constexpr int kMaxDests = 8;
template <typename P>
struct Dests {
    P* p[kMaxDests];
    int n;
};
template <typename P>
inline Dests<P> one_dest(P* ptr) {
    Dests<P> d{};
    d.p[0] = ptr;
    d.n = 1;
    return d;
}

// ------------------------------------------------------------------ PA step (sparse)
// One warp owns row i and CPW consecutive replica chunks (CPW * 32 * V replicas): the CSR
// row is read once for all of them and CPW x more loads are in flight per warp.
// Rows [row0, row0 + nrows): x/m are indexed locally (row - row0), the CSR, h and the
// sign-bit buffers by global row (a row-partitioned rank reads every row's spins).
#ifndef VXQ_PA_MINB
#define VXQ_PA_MINB 6  // cfg4 894 -> 757 us/step vs 4 (more loads in flight per SM)
#endif
#ifndef VXQ_PA_LATE_XM
#define VXQ_PA_LATE_XM 1
#endif
#ifndef VXQ_SBM_PTAIL
#define VXQ_SBM_PTAIL 1  // cfg3 146 -> 141, cfg4 1208 -> 1185, cfg5 86.6 -> 82.6 ms (profiles/r01/ab_sbm_tail)
#endif
template <typename T, int V, int CPW, bool MULTI = false>
__global__ void __launch_bounds__(256, MULTI ? 4 : VXQ_PA_MINB) k_pa_step(int64_t row0, int64_t nrows, int64_t R_pad,
                                                 Operator<T> op, const T* __restrict__ h,
                                                 T lam, T eta, T alpha, T* __restrict__ x,
                                                 T* __restrict__ m,
                                                 const uint32_t* __restrict__ sb_in,
                                                 uint32_t* __restrict__ sb_one,
                                                 const Dests<uint32_t> sb_out) {
    using O = Ops<T>;
    constexpr int NB = V * CPW;  // values per lane == sign words per (row, warp)
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int groups = (int)(R_pad / (32 * NB));
    const int64_t il = warp / groups;
    const int c0 = (int)(warp % groups) * CPW;
    if (il >= nrows) return;
    const int64_t i = row0 + il;
    const int64_t W = R_pad / 32;
    Vec<T, V> xv[CPW], mv[CPW];
#if VXQ_PA_LATE_XM
    // x/m are not needed until the field is summed: prefetch them into L2 now and load them
    // after the gathers (keeps 16 registers free for the gather batch)
#pragma unroll
    for (int g = 0; g < CPW; ++g) {
        const int64_t base = lane_base(il, R_pad, c0 + g, lane, V);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + base));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(m + base));
    }
#else
#pragma unroll
    for (int g = 0; g < CPW; ++g) {
        const int64_t base = lane_base(il, R_pad, c0 + g, lane, V);
        xv[g] = ld_cs<T, V>(x + base);
        mv[g] = ld_cs<T, V>(m + base);
    }
#endif
    T f[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) f[b] = (T)0;
    const uint32_t* sbc = sb_in + c0 * V;  // NB consecutive words of row j
    const int64_t k0 = __ldg(op.indptr + i), k1 = __ldg(op.indptr + i + 1);
    int64_t k = k0;
    // batches of 4 neighbours: issue all gathers, then accumulate in order
    for (; k + 4 <= k1; k += 4) {
        int j[4];
        T a[4];
        Vec<uint32_t, V> w[4][CPW];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            j[u] = __ldg(op.indices + k + u);
            a[u] = O::mul(op.sign, __ldg(op.data + k + u));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int g = 0; g < CPW; ++g)
                w[u][g] = *reinterpret_cast<const Vec<uint32_t, V>*>(sbc + (int64_t)j[u] * W + g * V);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int g = 0; g < CPW; ++g) add_pm<T, V>(f + g * V, w[u][g].v, a[u], lane);
    }
    for (; k < k1; ++k) {
        const int j = __ldg(op.indices + k);
        const T a = O::mul(op.sign, __ldg(op.data + k));
#pragma unroll
        for (int g = 0; g < CPW; ++g) {
            Vec<uint32_t, V> w =
                *reinterpret_cast<const Vec<uint32_t, V>*>(sbc + (int64_t)j * W + g * V);
            add_pm<T, V>(f + g * V, w.v, a, lane);
        }
    }

    const T hi = __ldg(h + i);
#if VXQ_PA_LATE_XM
#pragma unroll
    for (int g = 0; g < CPW; ++g) {
        const int64_t base = lane_base(il, R_pad, c0 + g, lane, V);
        xv[g] = ld_cs<T, V>(x + base);
        mv[g] = ld_cs<T, V>(m + base);
    }
#endif
#pragma unroll
    for (int g = 0; g < CPW; ++g) {
#pragma unroll
        for (int b = 0; b < V; ++b) {
            T xo = xv[g].v[b];
            T grad = O::add(O::add(O::mul(lam, xo), f[g * V + b]), hi);
            T mn = O::sub(O::mul(alpha, mv[g].v[b]), O::mul(eta, grad));
            T xn = O::add(xo, mn);
            xn = xn < (T)-1 ? (T)-1 : (xn > (T)1 ? (T)1 : xn);
            xv[g].v[b] = xn;
            mv[g].v[b] = mn;
            uint32_t word = __ballot_sync(0xffffffffu, xn >= (T)0);
            if (lane == g * V + b) {
                if constexpr (MULTI) {
#pragma unroll
                    for (int d = 0; d < kMaxDests; ++d)  // constant indices: no local copy
                        if (d < sb_out.n) sb_out.p[d][i * W + c0 * V + g * V + b] = word;
                } else {
                    sb_one[i * W + c0 * V + g * V + b] = word;
                }
            }
        }
        const int64_t base = lane_base(il, R_pad, c0 + g, lane, V);
        st_cs<T, V>(x + base, xv[g]);
        st_cs<T, V>(m + base, mv[g]);
    }
}

// R <= 32 (one sign word per row): a warp owns RPW consecutive rows whose CSR entries are
// contiguous.  The warp loads up to 64 of them cooperatively (lane l <- entry base + l and
// base + 32 + l), issues all their spin-word gathers at once, then every row walks its
// entries in ascending order through warp shuffles -- 3 memory round trips per RPW rows
// instead of ~2 per neighbour, same sequential per-row sum as k_pa_step (bit-identical).
#ifndef VXQ_COOP_MINB
#define VXQ_COOP_MINB 5
#endif
template <typename T, int RPW, bool MULTI = false>
__global__ void __launch_bounds__(256, MULTI ? 4 : VXQ_COOP_MINB) k_pa_step_coop(int64_t row0, int64_t nrows,
                                                      Operator<T> op, const T* __restrict__ h,
                                                      T lam, T eta, T alpha, T* __restrict__ x,
                                                      T* __restrict__ m,
                                                      const uint32_t* __restrict__ sb_in,
                                                      uint32_t* __restrict__ sb_one,
                                                      const Dests<uint32_t> sb_out) {
    using O = Ops<T>;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t il0 = warp * RPW;
    if (il0 >= nrows) return;
    const int nr = (int)min((int64_t)RPW, nrows - il0);
    // row bounds: lane u < nr+1 holds indptr[row0 + il0 + u]
    const int64_t myptr = lane <= nr ? __ldg(op.indptr + row0 + il0 + lane) : 0;
    const int64_t kbase = __shfl_sync(0xffffffffu, myptr, 0);
    const int64_t kend = __shfl_sync(0xffffffffu, myptr, nr);
    T xv[RPW], mv[RPW];
#pragma unroll
    for (int u = 0; u < RPW; ++u) {
        const int64_t il = u < nr ? il0 + u : il0;
        xv[u] = __ldcs(x + il * 32 + lane);
        mv[u] = __ldcs(m + il * 32 + lane);
    }
    // cooperative loads of entries [kbase, kbase + 64)
    const int64_t k0 = kbase + lane, k1 = kbase + 32 + lane;
    const bool v0 = k0 < kend, v1 = k1 < kend;
    const int j0 = v0 ? __ldcs(op.indices + k0) : 0, j1 = v1 ? __ldcs(op.indices + k1) : 0;
    const T a0 = v0 ? O::mul(op.sign, __ldcs(op.data + k0)) : (T)0;
    const T a1 = v1 ? O::mul(op.sign, __ldcs(op.data + k1)) : (T)0;
    const uint32_t w0 = v0 ? gather_word(sb_in + j0) : 0u, w1 = v1 ? gather_word(sb_in + j1) : 0u;
#pragma unroll
    for (int u = 0; u < RPW; ++u) {
        if (u >= nr) break;
        const int64_t kb = __shfl_sync(0xffffffffu, myptr, u);
        const int64_t ke = __shfl_sync(0xffffffffu, myptr, u + 1);
        T f = (T)0;
        for (int64_t k = kb; k < ke; ++k) {
            const int64_t off = k - kbase;
            T a;
            uint32_t w;
            if (off < 64) {  // off is warp-uniform: every lane offers the needed half
                const int src = (int)(off & 31);
                w = __shfl_sync(0xffffffffu, off < 32 ? w0 : w1, src);
                a = __shfl_sync(0xffffffffu, off < 32 ? a0 : a1, src);
            } else {  // rare: more than 64 entries in this warp's rows
                a = O::mul(op.sign, __ldg(op.data + k));
                w = __ldg(sb_in + __ldg(op.indices + k));
            }
            f = O::add(f, ((w >> lane) & 1u) ? a : -a);
        }
        const int64_t il = il0 + u, i = row0 + il;
        const T xo = xv[u];
        const T grad = O::add(O::add(O::mul(lam, xo), f), __ldg(h + i));
        const T mn = O::sub(O::mul(alpha, mv[u]), O::mul(eta, grad));
        T xn = O::add(xo, mn);
        xn = xn < (T)-1 ? (T)-1 : (xn > (T)1 ? (T)1 : xn);
        __stcs(x + il * 32 + lane, xn);
        __stcs(m + il * 32 + lane, mn);
        const uint32_t word = __ballot_sync(0xffffffffu, xn >= (T)0);
        if (lane == 0) {
            if constexpr (MULTI) {
#pragma unroll
                for (int d = 0; d < kMaxDests; ++d)
                    if (d < sb_out.n) sb_out.p[d][i] = word;
            } else {
                sb_one[i] = word;
            }
        }
    }
}

// ------------------------------------------------------------------ PA cluster (medium n)
// A thread-block cluster of C CTAs owns one replica chunk (32 V replicas) for a run of
// steps.  Every CTA of the cluster holds the chunk's spin words of ALL n rows in shared
// memory (double-buffered, n V words each), so a neighbour gather is a shared-memory
// broadcast instead of an L2 round trip; CTA k updates rows [k n / C, (k+1) n / C) (x/m
// stream from HBM as in k_pa_step), stores each new row's V words into all C tables
// (DSMEM), and one cluster barrier separates the steps.  The CSR entries of the next row and
// its x/m are loaded while the current row sums.  Per (row, replica): the same operations in
// the same CSR order as k_pa_step -- bit-identical.
#ifndef VXQ_PA_CLUSTER_THREADS
#define VXQ_PA_CLUSTER_THREADS 1024
#endif
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_map(const void* p, uint32_t rank) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
template <int V>
__device__ __forceinline__ void cl_store(uint32_t addr, const uint32_t (&w)[V]) {
    if constexpr (V == 4)
        asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(w[0]),
                     "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
    else if constexpr (V == 2)
        asm volatile("st.shared::cluster.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(w[0]),
                     "r"(w[1]) : "memory");
    else
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(w[0]) : "memory");
}

template <typename T, int V>
__global__ void __launch_bounds__(VXQ_PA_CLUSTER_THREADS, 1) k_pa_cluster(
    int64_t n, int64_t R_pad, int C, Operator<T> op, const T* __restrict__ h,
    const T* __restrict__ lam_sched, int64_t t0, int64_t nsteps, T eta, T alpha,
    T* __restrict__ x, T* __restrict__ m, const uint32_t* __restrict__ sb_in,
    uint32_t* __restrict__ sb_out) {
    using O = Ops<T>;
    extern __shared__ __align__(16) uint32_t tab[];  // [2][n][V], then this CTA's indptr
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int rank = (int)cl_rank();
    const int64_t c = blockIdx.x / C, W = R_pad / 32, nV = n * V;
    const int64_t rb = rank * n / C, re = (rank + 1) * n / C;
    int64_t* ptr_s = reinterpret_cast<int64_t*>(tab + 2 * nV);  // indptr[rb .. re]
    for (int64_t e = threadIdx.x; e < nV; e += blockDim.x)
        tab[e] = __ldg(sb_in + (e / V) * W + c * V + (e % V));
    for (int64_t r = rb + threadIdx.x; r <= re; r += blockDim.x) ptr_s[r - rb] = __ldg(op.indptr + r);
    const uint32_t peer = lane < C ? cl_map(tab, (uint32_t)lane) : 0u;  // lane q -> CTA q
    cl_sync();  // every CTA of the cluster is running and holds table 0
    for (int64_t s = 0; s < nsteps; ++s) {
        const T lam = lam_sched[t0 + s];
        const uint32_t* cur = tab + (s & 1) * nV;
        const int64_t nxt = ((s + 1) & 1) * nV;
        const bool last = s == nsteps - 1;
        int64_t i = rb + warp;
        // current row: CSR bounds, first 32 entries (lane-parallel), x/m
        int64_t kb = 0, ke = 0;
        int jl = 0;
        T al = (T)0;
        Vec<T, V> xv, mv;
        if (i < re) {
            kb = ptr_s[i - rb];
            ke = ptr_s[i - rb + 1];
            if (kb + lane < ke) {
                jl = __ldg(op.indices + kb + lane);
                al = O::mul(op.sign, __ldg(op.data + kb + lane));
            }
            xv = ld_cs<T, V>(x + lane_base(i, R_pad, (int)c, lane, V));
            mv = ld_cs<T, V>(m + lane_base(i, R_pad, (int)c, lane, V));
        }
        for (; i < re; i += nw) {
            // next row's loads in flight while this row sums
            const int64_t in = i + nw;
            int64_t kbn = 0, ken = 0;
            int jn = 0;
            T an = (T)0;
            Vec<T, V> xn_ = xv, mn_ = mv;  // (unused past the last row)
            if (in < re) {
                kbn = ptr_s[in - rb];
                ken = ptr_s[in - rb + 1];
                if (kbn + lane < ken) {
                    jn = __ldg(op.indices + kbn + lane);
                    an = O::mul(op.sign, __ldg(op.data + kbn + lane));
                }
                xn_ = ld_cs<T, V>(x + lane_base(in, R_pad, (int)c, lane, V));
                mn_ = ld_cs<T, V>(m + lane_base(in, R_pad, (int)c, lane, V));
            }
            T f[V];
#pragma unroll
            for (int b = 0; b < V; ++b) f[b] = (T)0;
            const int d0 = ke - kb < 32 ? (int)(ke - kb) : 32;
            int k = 0;
            for (; k + 4 <= d0; k += 4) {
                int j[4];
                T a[4];
                Vec<uint32_t, V> w[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    j[u] = __shfl_sync(0xffffffffu, jl, k + u);
                    a[u] = __shfl_sync(0xffffffffu, al, k + u);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    w[u] = *reinterpret_cast<const Vec<uint32_t, V>*>(cur + (int64_t)j[u] * V);
#pragma unroll
                for (int u = 0; u < 4; ++u) add_pm<T, V>(f, w[u].v, a[u], lane);
            }
            for (; k < d0; ++k) {
                const int j = __shfl_sync(0xffffffffu, jl, k);
                const T a = __shfl_sync(0xffffffffu, al, k);
                const Vec<uint32_t, V> w = *reinterpret_cast<const Vec<uint32_t, V>*>(cur + (int64_t)j * V);
                add_pm<T, V>(f, w.v, a, lane);
            }
            for (int64_t kk = kb + 32; kk < ke; ++kk) {  // rows longer than 32 entries
                const int j = __ldg(op.indices + kk);
                const T a = O::mul(op.sign, __ldg(op.data + kk));
                const Vec<uint32_t, V> w = *reinterpret_cast<const Vec<uint32_t, V>*>(cur + (int64_t)j * V);
                add_pm<T, V>(f, w.v, a, lane);
            }
            const T hi = __ldg(h + i);
            uint32_t words[V];
#pragma unroll
            for (int b = 0; b < V; ++b) {
                const T xo = xv.v[b];
                const T grad = O::add(O::add(O::mul(lam, xo), f[b]), hi);
                const T mn = O::sub(O::mul(alpha, mv.v[b]), O::mul(eta, grad));
                T xn = O::add(xo, mn);
                xn = xn < (T)-1 ? (T)-1 : (xn > (T)1 ? (T)1 : xn);
                xv.v[b] = xn;
                mv.v[b] = mn;
                words[b] = __ballot_sync(0xffffffffu, xn >= (T)0);
            }
            st_cs<T, V>(x + lane_base(i, R_pad, (int)c, lane, V), xv);
            st_cs<T, V>(m + lane_base(i, R_pad, (int)c, lane, V), mv);
            if (lane < C) cl_store<V>(peer + (uint32_t)((nxt + i * V) * 4), words);
            if (last && lane < V) {
                uint32_t wv = words[0];
#pragma unroll
                for (int b = 1; b < V; ++b)
                    if (lane == b) wv = words[b];
                sb_out[i * W + c * V + lane] = wv;
            }
            kb = kbn;
            ke = ken;
            jl = jn;
            al = an;
            xv = xn_;
            mv = mn_;
        }
        cl_sync();  // the step's words are in every table; table s & 1 is free again
    }
}

// ------------------------------------------------------------------ SBM step (sparse)
template <typename T>
struct SbmScalars {
    T a_t, dt, a0, c0, dta0, q_cap;
};

// Rows [row0, row0 + nrows): q_in/q_out are full (global-row) buffers, p is local.
template <typename T, int V, bool MULTI = false>
__global__ void __launch_bounds__(256) k_sbm_step(int64_t row0, int64_t nrows, int64_t R_pad,
                                                  Operator<T> op, const T* __restrict__ g,
                                                  SbmScalars<T> sc, const T* __restrict__ q_in,
                                                  T* __restrict__ q_one, const Dests<T> q_out,
                                                  T* __restrict__ p) {
    using O = Ops<T>;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int chunks = (int)(R_pad / (32 * V));
    const int64_t il = warp / chunks;
    const int c = (int)(warp % chunks);
    if (il >= nrows) return;
    const int64_t i = row0 + il;
    const int64_t off = (int64_t)c * 32 * V + (int64_t)lane * V;
    const int64_t base = i * R_pad + off;
    const int64_t pbase = il * R_pad + off;
    T f[V];
#pragma unroll
    for (int b = 0; b < V; ++b) f[b] = (T)0;
    const uint64_t pol_keep = VXQ_SBM_L2HINT ? l2_policy_last() : 0;
    const int64_t k0 = __ldg(op.indptr + i), k1 = __ldg(op.indptr + i + 1);
    int64_t k = k0;
    for (; k + 4 <= k1; k += 4) {
        int j[4];
        T a[4];
        Vec<T, V> qv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            j[u] = __ldg(op.indices + k + u);
            a[u] = O::mul(op.sign, __ldg(op.data + k + u));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            qv[u] = ld_hint<T, V>(q_in + (int64_t)j[u] * R_pad + off, pol_keep);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            T t[V];
            mulv<T, V>(t, a[u], qv[u].v);
            addv<T, V>(f, t);
        }
    }
#if VXQ_SBM_PTAIL
    // the 1-3 remaining entries: one round of index loads, one of gathers (predicated)
    if (k < k1) {
        const int rem = (int)(k1 - k);
        int j[3];
        T a[3];
        Vec<T, V> qv[3];
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) {
                j[u] = __ldg(op.indices + k + u);
                a[u] = O::mul(op.sign, __ldg(op.data + k + u));
            }
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) qv[u] = ld_hint<T, V>(q_in + (int64_t)j[u] * R_pad + off, pol_keep);
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (u < rem) {
                T t[V];
                mulv<T, V>(t, a[u], qv[u].v);
                addv<T, V>(f, t);
            }
    }
#else
    for (; k < k1; ++k) {
        int j = __ldg(op.indices + k);
        T a = O::mul(op.sign, __ldg(op.data + k));
        Vec<T, V> qv = ld_hint<T, V>(q_in + (int64_t)j * R_pad + off, pol_keep);
#pragma unroll
        for (int b = 0; b < V; ++b) f[b] = O::add(f[b], O::mul(a, qv.v[b]));
    }
#endif
    Vec<T, V> qv = *reinterpret_cast<const Vec<T, V>*>(q_in + base);
    Vec<T, V> pv = ld_cs<T, V>(p + pbase);
    const T gi = __ldg(g + i);
#pragma unroll
    for (int b = 0; b < V; ++b) {
        T qi = qv.v[b];
        T inner = -O::sub(O::add(O::mul(qi, qi), sc.a0), sc.a_t);
        T force = O::add(O::mul(inner, qi), O::mul(sc.c0, O::add(f[b], gi)));
        T pn = O::add(pv.v[b], O::mul(sc.dt, force));
        T qn = O::add(qi, O::mul(sc.dta0, pn));
        if (fabs(qn) > sc.q_cap) {
            qn = qn < -sc.q_cap ? -sc.q_cap : sc.q_cap;
            pn = (T)0;
        }
        qv.v[b] = qn;
        pv.v[b] = pn;
    }
    if constexpr (MULTI) {
#pragma unroll
        for (int d = 0; d < kMaxDests; ++d)
            if (d < q_out.n) *reinterpret_cast<Vec<T, V>*>(q_out.p[d] + base) = qv;
    } else {
        st_hint<T, V>(q_one + base, qv, VXQ_SBM_L2HINT ? l2_policy_first() : 0);
    }
    st_cs<T, V>(p + pbase, pv);
}

// ------------------------------------------------------------------ SBM step, row blocks
// Structured sparse graphs (Pegasus / Chimera numbering) give consecutive rows common
// neighbours: 64 rows of P16 touch ~302 distinct rows through ~920 entries.  One CTA owns
// (row block b of kSbmBlockRows rows, replica chunk c of 32 V replicas): it stages the q_t
// chunk rows of the block's distinct neighbours (slot lists built once per problem) and the
// block's CSR entries in shared memory, then each warp sums its rows from there -- a
// neighbour row crosses L2 -> SM once per block instead of once per entry.  Per (row,
// replica) the same operations in the same CSR order as k_sbm_step: bit-identical.
constexpr int kSbmBlockRows = 64;
constexpr int kSbmBlockThreads = 512;
constexpr int kSbmBlockMaxEnt = 4096;  // CSR entries of one block staged in shared memory
#ifndef VXQ_SBM_BLOCK_V
#define VXQ_SBM_BLOCK_V 2
#endif
constexpr int kSbmBlockV = VXQ_SBM_BLOCK_V;  // replicas per lane of the block path's layout
template <int BYTES>  // 4, 8 or 16
__device__ __forceinline__ void cp_async_n(void* smem_dst, const void* gsrc) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    if constexpr (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(gsrc), "n"(BYTES)
                     : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_all;" ::: "memory");
}

template <typename T, int V>
__global__ void __launch_bounds__(kSbmBlockThreads) k_sbm_block(
    int64_t n, int64_t R_pad, const int32_t* __restrict__ u_ptr,
    const int32_t* __restrict__ u_idx, const uint16_t* __restrict__ slot, Operator<T> op,
    const T* __restrict__ g, SbmScalars<T> sc, const T* __restrict__ q_in,
    T* __restrict__ q_out, T* __restrict__ p, int ent_cap) {
    using O = Ops<T>;
    constexpr int NW = kSbmBlockThreads / 32;
    constexpr int RPW = kSbmBlockRows / NW;  // rows per warp
    extern __shared__ __align__(16) unsigned char sbm_blk_smem[];
    __shared__ int32_t s_ptr[kSbmBlockRows + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.x;
    const int64_t off = (int64_t)blockIdx.y * 32 * V + (int64_t)lane * V;
    const int64_t r0 = (int64_t)b * kSbmBlockRows;
    const int nr = n - r0 < kSbmBlockRows ? (int)(n - r0) : kSbmBlockRows;
    // this warp's rows: own q, p, g first (their latency overlaps the staging)
    Vec<T, V> qo[RPW], po[RPW];
    T go[RPW];
#pragma unroll
    for (int k = 0; k < RPW; ++k) {
        const int rl = warp + k * NW;
        if (rl < nr) {
            const int64_t base = (r0 + rl) * R_pad + off;
            qo[k] = *reinterpret_cast<const Vec<T, V>*>(q_in + base);
            po[k] = ld_cs<T, V>(p + base);
            go[k] = __ldg(g + r0 + rl);
        }
    }
    const int u0 = __ldg(u_ptr + b), nu = __ldg(u_ptr + b + 1) - u0;
    const int64_t e0 = __ldg(op.indptr + r0);
    const int ne = (int)(__ldg(op.indptr + r0 + nr) - e0);
    T* qs = reinterpret_cast<T*>(sbm_blk_smem);                                   // [nu][32 V]
    T* s_val = qs + (size_t)nu * 32 * V;                                          // [ne]
    uint16_t* s_slot = reinterpret_cast<uint16_t*>(s_val + ent_cap);              // [ne]
    // stage the neighbours' chunk rows (16 B per lane per row)
    for (int s0 = warp * 32; s0 < nu; s0 += NW * 32) {
        const int jl = s0 + lane < nu ? __ldg(u_idx + u0 + s0 + lane) : 0;
        const int cnt = min(32, nu - s0);
        for (int t = 0; t < cnt; ++t) {
            const int j = __shfl_sync(0xffffffffu, jl, t);
            const T* src = q_in + (int64_t)j * R_pad + off;
            T* dst = qs + (size_t)(s0 + t) * 32 * V + (size_t)lane * V;
            constexpr int VB = (int)(V * sizeof(T));  // bytes per lane: 4, 8, 16 (fp32) / 8, 16 (fp64)
            if constexpr (VB <= 16) {
                cp_async_n<VB>(dst, src);
            } else {
#pragma unroll
                for (int h = 0; h < VB / 16; ++h)
                    cp_async_n<16>(dst + h * 16 / sizeof(T), src + h * 16 / sizeof(T));
            }
        }
    }
    // the block's CSR entries (slot, sign * value) and row offsets
    for (int e = threadIdx.x; e < ne; e += kSbmBlockThreads) {
        s_val[e] = O::mul(op.sign, __ldg(op.data + e0 + e));
        s_slot[e] = __ldg(slot + e0 + e);
    }
    for (int r = threadIdx.x; r <= nr; r += kSbmBlockThreads)
        s_ptr[r] = (int32_t)(__ldg(op.indptr + r0 + r) - e0);
    cp_async_wait_all();
    __syncthreads();
#pragma unroll
    for (int k = 0; k < RPW; ++k) {
        const int rl = warp + k * NW;
        if (rl >= nr) break;
        const int kb = s_ptr[rl], ke = s_ptr[rl + 1];
        T f[V];
#pragma unroll
        for (int bb = 0; bb < V; ++bb) f[bb] = (T)0;
        int kk = kb;
        for (; kk + 4 <= ke; kk += 4) {
            Vec<T, V> qv[4];
            T a[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = s_val[kk + u];
                qv[u] = *reinterpret_cast<const Vec<T, V>*>(qs + (size_t)s_slot[kk + u] * 32 * V + (size_t)lane * V);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int bb = 0; bb < V; ++bb) f[bb] = O::add(f[bb], O::mul(a[u], qv[u].v[bb]));
        }
        for (; kk < ke; ++kk) {
            const T a = s_val[kk];
            const Vec<T, V> qv = *reinterpret_cast<const Vec<T, V>*>(qs + (size_t)s_slot[kk] * 32 * V + (size_t)lane * V);
#pragma unroll
            for (int bb = 0; bb < V; ++bb) f[bb] = O::add(f[bb], O::mul(a, qv.v[bb]));
        }
        const int64_t base = (r0 + rl) * R_pad + off;
#pragma unroll
        for (int bb = 0; bb < V; ++bb) {
            const T qi = qo[k].v[bb];
            const T inner = -O::sub(O::add(O::mul(qi, qi), sc.a0), sc.a_t);
            const T force = O::add(O::mul(inner, qi), O::mul(sc.c0, O::add(f[bb], go[k])));
            T pn = O::add(po[k].v[bb], O::mul(sc.dt, force));
            T qn = O::add(qi, O::mul(sc.dta0, pn));
            if (fabs(qn) > sc.q_cap) {
                qn = qn < -sc.q_cap ? -sc.q_cap : sc.q_cap;
                pn = (T)0;
            }
            qo[k].v[bb] = qn;
            po[k].v[bb] = pn;
        }
        *reinterpret_cast<Vec<T, V>*>(q_out + base) = qo[k];
        st_cs<T, V>(p + base, po[k]);
    }
}

// ------------------------------------------------------------------ resident (small n)
// One CTA owns RG replicas for all T steps: their state and the whole CSR (row pointers,
// indices, values) live in shared memory, so the only per-step synchronisation is one
// __syncthreads (double-buffered spins / q).  Each row still sums its neighbours
// sequentially in ascending column order (bit-identical to the sparse kernels).
template <typename T>
struct ResidentSmem {
    int32_t* ptr;
    int32_t* idx;
    T* val;
    unsigned char* rest;
};

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

template <typename T>
__device__ ResidentSmem<T> stage_csr(unsigned char* smem, int n, int nnz, const Operator<T>& op) {
    ResidentSmem<T> S;
    S.ptr = reinterpret_cast<int32_t*>(smem);
    S.idx = reinterpret_cast<int32_t*>(smem + align16((n + 1) * 4));
    S.val = reinterpret_cast<T*>(smem + align16((n + 1) * 4) + align16((size_t)nnz * 4));
    S.rest = smem + align16((n + 1) * 4) + align16((size_t)nnz * 4) + align16((size_t)nnz * sizeof(T));
    for (int i = threadIdx.x; i <= n; i += blockDim.x) S.ptr[i] = (int32_t)op.indptr[i];
    for (int k = threadIdx.x; k < nnz; k += blockDim.x) {
        S.idx[k] = op.indices[k];
        S.val[k] = Ops<T>::mul(op.sign, op.data[k]);
    }
    return S;
}

template <typename T>
__host__ __device__ inline size_t resident_csr_bytes(int64_t n, int64_t nnz) {
    return align16((n + 1) * 4) + align16((size_t)nnz * 4) + align16((size_t)nnz * sizeof(T));
}

// f = sum_k val[k] * v(idx[k]) over [kb, ke) in order; v(j) provided by the callable.
// Long rows are software-pipelined: the shared-memory loads of batch b+1 (indices, values,
// then the neighbours' states) are issued before batch b's adds, so the sum runs at the
// rate of its dependent FADD chain instead of two shared-memory round trips per batch.
// (SBM resident step: cfg1 1.65 -> 1.41 us/step; the PA step, whose terms are a select of
// +-a on a spin byte, measured no gain and keeps the plain loop: PIPE = false.)
template <typename T, bool PIPE = true, typename F>
__device__ __forceinline__ T row_sum(const ResidentSmem<T>& S, int kb, int ke, F&& v) {
    using O = Ops<T>;
    constexpr int B = 8;
    T f = (T)0;
    int k = kb;
    if (PIPE && ke - kb >= 2 * B) {
        T w[B];
#pragma unroll
        for (int u = 0; u < B; ++u) w[u] = v(S.idx[k + u], S.val[k + u]);
        k += B;
        for (; k + B <= ke; k += B) {
            T wn[B];
#pragma unroll
            for (int u = 0; u < B; ++u) wn[u] = v(S.idx[k + u], S.val[k + u]);
#pragma unroll
            for (int u = 0; u < B; ++u) f = O::add(f, w[u]);
#pragma unroll
            for (int u = 0; u < B; ++u) w[u] = wn[u];
        }
#pragma unroll
        for (int u = 0; u < B; ++u) f = O::add(f, w[u]);
    }
    for (; k + 4 <= ke; k += 4) {
        int j[4];
        T a[4], w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            j[u] = S.idx[k + u];
            a[u] = S.val[k + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = v(j[u], a[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) f = O::add(f, w[u]);
    }
    for (; k < ke; ++k) f = O::add(f, v(S.idx[k], S.val[k]));
    return f;
}

template <typename T>
__global__ void k_pa_resident(int64_t n64, int64_t R_pad, int V, int RG, int nnz, Operator<T> op,
                              const T* __restrict__ h, const T* __restrict__ lam_sched,
                              int64_t steps, T eta, T alpha, T* __restrict__ x,
                              T* __restrict__ m) {
    using O = Ops<T>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = (int)n64;
    ResidentSmem<T> S = stage_csr<T>(smem, n, nnz, op);
    T* xs = reinterpret_cast<T*>(S.rest);
    T* ms = xs + RG * n;
    uint8_t* s0 = reinterpret_cast<uint8_t*>(ms + RG * n);
    uint8_t* s1 = s0 + RG * n;
    const int64_t r0 = (int64_t)blockIdx.x * RG;
    const int items = RG * n;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int g = it / n, i = it - g * n;
        const int64_t r = r0 + g;
        T xv = (r < R_pad) ? x[(int64_t)i * R_pad + pos_of(r, V)] : (T)0;
        T mv = (r < R_pad) ? m[(int64_t)i * R_pad + pos_of(r, V)] : (T)0;
        xs[it] = xv;
        ms[it] = mv;
        s0[it] = xv >= (T)0;
    }
    __syncthreads();
    for (int64_t t = 0; t < steps; ++t) {
        const T lam = lam_sched[t];
        const uint8_t* sc = (t & 1) ? s1 : s0;
        uint8_t* sn = (t & 1) ? s0 : s1;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
            const int g = it / n, i = it - g * n;
            const uint8_t* sg = sc + g * n;
            const T f = row_sum<T, false>(S, S.ptr[i], S.ptr[i + 1],
                                          [&](int j, T a) { return sg[j] ? a : -a; });
            const T xo = xs[it];
            const T grad = O::add(O::add(O::mul(lam, xo), f), __ldg(h + i));
            const T mn = O::sub(O::mul(alpha, ms[it]), O::mul(eta, grad));
            T xn = O::add(xo, mn);
            xn = xn < (T)-1 ? (T)-1 : (xn > (T)1 ? (T)1 : xn);
            xs[it] = xn;
            ms[it] = mn;
            sn[it] = xn >= (T)0;
        }
        __syncthreads();
    }
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int g = it / n, i = it - g * n;
        const int64_t r = r0 + g;
        if (r < R_pad) {
            x[(int64_t)i * R_pad + pos_of(r, V)] = xs[it];
            m[(int64_t)i * R_pad + pos_of(r, V)] = ms[it];
        }
    }
}

template <typename T>
__global__ void k_sbm_resident(int64_t n64, int64_t R_pad, int V, int RG, int nnz,
                               Operator<T> op, const T* __restrict__ g,
                               const T* __restrict__ a_sched, int64_t steps, SbmScalars<T> sc0,
                               T* __restrict__ q, T* __restrict__ p) {
    using O = Ops<T>;
    extern __shared__ __align__(16) unsigned char smem[];
    const int n = (int)n64;
    ResidentSmem<T> S = stage_csr<T>(smem, n, nnz, op);
    T* q0 = reinterpret_cast<T*>(S.rest);
    T* q1 = q0 + RG * n;
    T* ps = q1 + RG * n;
    const int64_t r0 = (int64_t)blockIdx.x * RG;
    const int items = RG * n;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int gg = it / n, i = it - gg * n;
        const int64_t r = r0 + gg;
        q0[it] = (r < R_pad) ? q[(int64_t)i * R_pad + pos_of(r, V)] : (T)0;
        ps[it] = (r < R_pad) ? p[(int64_t)i * R_pad + pos_of(r, V)] : (T)0;
    }
    __syncthreads();
    for (int64_t t = 0; t < steps; ++t) {
        const T a_t = a_sched[t];
        const T* qc = (t & 1) ? q1 : q0;
        T* qn_arr = (t & 1) ? q0 : q1;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
            const int gg = it / n, i = it - gg * n;
            const T* qg = qc + gg * n;
            const T f = row_sum<T>(S, S.ptr[i], S.ptr[i + 1],
                                   [&](int j, T a) { return O::mul(a, qg[j]); });
            const T qi = qc[it];
            const T inner = -O::sub(O::add(O::mul(qi, qi), sc0.a0), a_t);
            const T force = O::add(O::mul(inner, qi), O::mul(sc0.c0, O::add(f, __ldg(g + i))));
            T pn = O::add(ps[it], O::mul(sc0.dt, force));
            T qn = O::add(qi, O::mul(sc0.dta0, pn));
            if (fabs(qn) > sc0.q_cap) {
                qn = qn < -sc0.q_cap ? -sc0.q_cap : sc0.q_cap;
                pn = (T)0;
            }
            qn_arr[it] = qn;
            ps[it] = pn;
        }
        __syncthreads();
    }
    const T* qf = (steps & 1) ? q1 : q0;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int gg = it / n, i = it - gg * n;
        const int64_t r = r0 + gg;
        if (r < R_pad) {
            q[(int64_t)i * R_pad + pos_of(r, V)] = qf[it];
            p[(int64_t)i * R_pad + pos_of(r, V)] = ps[it];
        }
    }
}

// ------------------------------------------------------------------ host side
void pa_schedule(double lam0, int64_t T, double* out) {
    for (int64_t t = 0; t < T; ++t) out[t] = lam0 * (1.0 - (double)t / (double)T);
}

void sbm_schedule(double a0, int64_t T, double* out) {
    // numpy.linspace(0.0, a0, T): y = arange(T) * step + 0.0; y[-1] = a0
    if (T <= 0) return;
    if (T == 1) {
        out[0] = 0.0 * a0 + 0.0;
        return;
    }
    const double div = (double)(T - 1);
    const double step = (a0 - 0.0) / div;
    if (step == 0.0) {
        for (int64_t t = 0; t < T; ++t) out[t] = ((double)t / div) * (a0 - 0.0) + 0.0;
    } else {
        for (int64_t t = 0; t < T; ++t) out[t] = (double)t * step + 0.0;
    }
    out[T - 1] = a0;
}

namespace {

constexpr int TB = 256;
inline unsigned nblk(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, TB)); }

struct Layout {
    int64_t n, R, R_pad, W;
    int V;
    int64_t row0 = 0, nrows = 0;  // rows this launch updates (row partition), default all
};

Layout make_layout(int64_t n, int64_t R, bool fp64) {
    Layout L;
    L.n = n;
    L.R = R;
    if (fp64) L.V = (R <= 32) ? 1 : 2;
    else L.V = (R <= 32) ? 1 : (R <= 64 ? 2 : 4);
    int64_t ch = 32 * L.V;
    L.R_pad = ceil_div(R, ch) * ch;
    L.W = L.R_pad / 32;
    L.row0 = 0;
    L.nrows = n;
    return L;
}

int resident_rg(const Layout& L) {
    int64_t ctas_target = 148 * 8;
    int rg = (int)std::max<int64_t>(1, std::min<int64_t>(8, ceil_div(L.R_pad, ctas_target)));
    return rg;
}

size_t resident_smem_pa(const Layout& L, int RG, size_t tsz, int64_t nnz) {
    const size_t csr = tsz == 8 ? resident_csr_bytes<double>(L.n, nnz)
                                : resident_csr_bytes<float>(L.n, nnz);
    return csr + (size_t)RG * L.n * (2 * tsz + 2);
}
size_t resident_smem_sbm(const Layout& L, int RG, size_t tsz, int64_t nnz) {
    const size_t csr = tsz == 8 ? resident_csr_bytes<double>(L.n, nnz)
                                : resident_csr_bytes<float>(L.n, nnz);
    return csr + (size_t)RG * L.n * (3 * tsz);
}

constexpr size_t kResidentSmemMax = 200 * 1024;

int choose_path(int requested, const Layout& L, size_t smem_needed, int64_t nnz) {
    if (requested == VXQ_PATH_RESIDENT) {
        if (smem_needed > kResidentSmemMax)
            throw Error(VXQ_ERR_UNSUPPORTED, "resident path: state does not fit shared memory");
        return VXQ_PATH_RESIDENT;
    }
    if (requested == VXQ_PATH_SPARSE || requested == VXQ_PATH_DENSE) return VXQ_PATH_SPARSE;
    // auto: small problems run resident (all steps in one launch); the CSR per replica
    // must stay cache-friendly (each CTA re-streams it every step)
    if (smem_needed <= kResidentSmemMax && L.n <= 4096 && nnz <= (int64_t)1 << 20)
        return VXQ_PATH_RESIDENT;
    return VXQ_PATH_SPARSE;
}

int block_threads(int64_t items) {
    int64_t t = ceil_div(items, 32) * 32;
    return (int)std::min<int64_t>(512, std::max<int64_t>(32, t));
}

// One destination (every solve except a peer-exchange session): the __restrict__ single
// pointer variant (MULTI = false) -- the multi-destination loop is only compiled in for
// row-partitioned ranks with peers.
template <typename T, bool MULTI>
void launch_pa_step_t(const Layout& L, const Operator<T>& op, const T* h, T lam, T eta,
                      T alpha, T* x, T* m, const uint32_t* sbi, const Dests<uint32_t>& sbo,
                      cudaStream_t s) {
    const int64_t chunks = L.R_pad / (32 * L.V);
    uint32_t* one = sbo.p[0];
    if (L.R_pad == 32) {  // one sign word per row: cooperative warp-CSR over 8 rows
        constexpr int RPW = 8;
        const int64_t warps = ceil_div(L.nrows, RPW);
        k_pa_step_coop<T, RPW, MULTI><<<(unsigned)ceil_div(warps * 32, 256), 256, 0, s>>>(
            L.row0, L.nrows, op, h, lam, eta, alpha, x, m, sbi, one, sbo);
        return;
    }
    const int cpw = (chunks % 2 == 0) ? 2 : 1;  // two chunks per warp when they pair up
    const int64_t warps = L.nrows * (chunks / cpw);
    const unsigned blocks = (unsigned)ceil_div(warps * 32, 256);
#define VXQ_PA_STEP(VV, CC)                                                                \
    k_pa_step<T, VV, CC, MULTI><<<blocks, 256, 0, s>>>(L.row0, L.nrows, L.R_pad, op, h,    \
                                                       lam, eta, alpha, x, m, sbi, one, sbo)
    if (L.V == 1) {
        if (cpw == 2) VXQ_PA_STEP(1, 2); else VXQ_PA_STEP(1, 1);
    } else if (L.V == 2) {
        if (cpw == 2) VXQ_PA_STEP(2, 2); else VXQ_PA_STEP(2, 1);
    } else {
        if constexpr (sizeof(T) == 4) {
            if (cpw == 2) VXQ_PA_STEP(4, 2); else VXQ_PA_STEP(4, 1);
        }
    }
#undef VXQ_PA_STEP
}
template <typename T>
void launch_pa_step(const Layout& L, const Operator<T>& op, const T* h, T lam, T eta, T alpha,
                    T* x, T* m, const uint32_t* sbi, const Dests<uint32_t>& sbo, cudaStream_t s) {
    if (sbo.n > 1) launch_pa_step_t<T, true>(L, op, h, lam, eta, alpha, x, m, sbi, sbo, s);
    else launch_pa_step_t<T, false>(L, op, h, lam, eta, alpha, x, m, sbi, sbo, s);
}
template <typename T>
void launch_pa_step(const Layout& L, const Operator<T>& op, const T* h, T lam, T eta, T alpha,
                    T* x, T* m, const uint32_t* sbi, uint32_t* sbo, cudaStream_t s) {
    launch_pa_step<T>(L, op, h, lam, eta, alpha, x, m, sbi, one_dest(sbo), s);
}

// ---- PA cluster path (k_pa_cluster): plan + launch
constexpr size_t kPaClusterSmemMax = 200 * 1024;

int sm_count() {
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return nsm;
}

struct PaClusterPlan {
    int C = 0;
    int64_t chunks = 0;
    size_t smem = 0;
};

template <typename T, int V>
cudaLaunchConfig_t pa_cluster_config(const PaClusterPlan& pl, cudaLaunchAttribute* at,
                                     cudaStream_t s) {
    auto kern = k_pa_cluster<T, V>;
    VXQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)pl.smem));
    if (pl.C > 8)
        VXQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(pl.chunks * pl.C));
    cfg.blockDim = dim3(VXQ_PA_CLUSTER_THREADS);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = s;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)pl.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
}

template <typename T, int V>
bool pa_cluster_fits(const PaClusterPlan& pl, cudaStream_t s) {
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = pa_cluster_config<T, V>(pl, at, s);
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k_pa_cluster<T, V>, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return nc >= 1;
}

// The cluster kernel serves full-row solves whose chunk spin table (2 n V words) fits
// shared memory.  Opt-in (VXQ_PA_CLUSTER: 0 = never (default), 1 = when chunks x C clusters
// cover 2/3 of the SMs, 2 = whenever it fits; VXQ_PA_CLUSTER_C overrides C): on cfg 3 it
// measured 111 us/step against the step kernel's 99 (profiles/r02/ab_pa_cluster) -- the
// step is instruction-issue bound (~3 instructions per +-a term), not gather-latency bound,
// and the cluster runs on 128 of the 148 SMs.
template <typename T>
bool pa_cluster_plan(const Layout& L, PaClusterPlan* pl, cudaStream_t s) {
    const char* e = getenv("VXQ_PA_CLUSTER");
    const int mode = e ? atoi(e) : 0;
    if (mode == 0 || L.row0 != 0 || L.nrows != L.n) return false;
    pl->chunks = L.R_pad / (32 * L.V);
    const int nsm = sm_count();
    int C = (int)std::max<int64_t>(1, std::min<int64_t>(8, nsm / pl->chunks));
    if (const char* ce = getenv("VXQ_PA_CLUSTER_C")) C = std::max(1, atoi(ce));
    pl->C = (int)std::min<int64_t>(C, L.n);
    // two spin tables + the largest CTA's indptr slice (ceil(n / C) + 1 int64)
    pl->smem = (size_t)2 * L.n * L.V * sizeof(uint32_t) +
               (size_t)(ceil_div(L.n, pl->C) + 2) * sizeof(int64_t);
    if (pl->smem > kPaClusterSmemMax) return false;
    if (mode == 1 && pl->chunks * pl->C < (2 * nsm) / 3) return false;
    switch (L.V) {
        case 1: return pa_cluster_fits<T, 1>(*pl, s);
        case 2: return pa_cluster_fits<T, 2>(*pl, s);
        default:
            if constexpr (sizeof(T) == 4) return pa_cluster_fits<T, 4>(*pl, s);
            return false;
    }
}

template <typename T>
void launch_pa_cluster(const PaClusterPlan& pl, const Layout& L, const Operator<T>& op,
                       const T* h, const T* lam_sched, int64_t t0, int64_t nsteps, T eta,
                       T alpha, T* x, T* m, const uint32_t* sbi, uint32_t* sbo, cudaStream_t s) {
    cudaLaunchAttribute at[1];
#define VXQ_PA_CL(VV)                                                                        \
    {                                                                                        \
        cudaLaunchConfig_t cfg = pa_cluster_config<T, VV>(pl, at, s);                        \
        VXQ_CUDA(cudaLaunchKernelEx(&cfg, k_pa_cluster<T, VV>, L.n, L.R_pad, pl.C, op, h,    \
                                    lam_sched, t0, nsteps, eta, alpha, x, m, sbi, sbo));     \
    }
    switch (L.V) {
        case 1: VXQ_PA_CL(1); break;
        case 2: VXQ_PA_CL(2); break;
        default:
            if constexpr (sizeof(T) == 4) VXQ_PA_CL(4);
            break;
    }
#undef VXQ_PA_CL
}

template <typename T, bool MULTI>
void launch_sbm_step_t(const Layout& L, const Operator<T>& op, const T* g, SbmScalars<T> sc,
                       const T* qi, const Dests<T>& qo, T* p, cudaStream_t s) {
    int64_t warps = L.nrows * (L.R_pad / (32 * L.V));
    unsigned blocks = (unsigned)ceil_div(warps * 32, 256);
    T* one = qo.p[0];
    // (a cooperative 8-rows-per-warp variant like k_pa_step_coop measured 23 % slower for
    // R = 32 on config 5: one row per warp keeps 8x more 128-byte q gathers in flight)
    switch (L.V) {
        case 1: k_sbm_step<T, 1, MULTI><<<blocks, 256, 0, s>>>(L.row0, L.nrows, L.R_pad, op, g, sc, qi, one, qo, p); break;
        case 2: k_sbm_step<T, 2, MULTI><<<blocks, 256, 0, s>>>(L.row0, L.nrows, L.R_pad, op, g, sc, qi, one, qo, p); break;
        default:
            if constexpr (sizeof(T) == 4)
                k_sbm_step<T, 4, MULTI><<<blocks, 256, 0, s>>>(L.row0, L.nrows, L.R_pad, op, g, sc, qi, one, qo, p);
            break;
    }
}
template <typename T>
void launch_sbm_step(const Layout& L, const Operator<T>& op, const T* g, SbmScalars<T> sc,
                     const T* qi, const Dests<T>& qo, T* p, cudaStream_t s) {
    if (qo.n > 1) launch_sbm_step_t<T, true>(L, op, g, sc, qi, qo, p, s);
    else launch_sbm_step_t<T, false>(L, op, g, sc, qi, qo, p, s);
}
template <typename T>
void launch_sbm_step(const Layout& L, const Operator<T>& op, const T* g, SbmScalars<T> sc,
                     const T* qi, T* qo, T* p, cudaStream_t s) {
    launch_sbm_step<T>(L, op, g, sc, qi, one_dest(qo), p, s);
}

template <typename T>
void launch_pack(const Layout& L, const T* x, uint32_t* sb, cudaStream_t s) {
    int64_t warps = L.nrows * (L.R_pad / (32 * L.V));
    unsigned blocks = (unsigned)ceil_div(warps * 32, 256);
    switch (L.V) {
        case 1: k_pack_signs<T, 1><<<blocks, 256, 0, s>>>(x, L.row0, L.nrows, L.R_pad, sb); break;
        case 2: k_pack_signs<T, 2><<<blocks, 256, 0, s>>>(x, L.row0, L.nrows, L.R_pad, sb); break;
        default:
            if constexpr (sizeof(T) == 4) k_pack_signs<T, 4><<<blocks, 256, 0, s>>>(x, L.row0, L.nrows, L.R_pad, sb);
            break;
    }
    VXQ_CHECK_LAUNCH();
}


// ---- improvement mode / energy trace (north star (3); SURVEY 8a note on best-seen)
__global__ void k_trace_min(const double* __restrict__ e, int64_t R, double* __restrict__ out) {
    __shared__ double sh[256];
    double v = INFINITY;
    for (int64_t r = threadIdx.x; r < R; r += blockDim.x) v = fmin(v, e[r]);
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] = fmin(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// strictly better => keep (the earliest state wins ties); mask bit r marks replica r
__global__ void k_update_best(const double* __restrict__ e, int64_t R, double* __restrict__ best,
                              uint32_t* __restrict__ mask) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool better = false;
    if (r < R && e[r] < best[r]) {
        best[r] = e[r];
        better = true;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, better);
    if ((threadIdx.x & 31) == 0 && r < R + 31) mask[r >> 5] = word;
}

__global__ void k_merge_bits(int64_t words, int64_t W, const uint32_t* __restrict__ mask,
                             const uint32_t* __restrict__ sb, uint32_t* __restrict__ best_sb) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= words) return;
    const uint32_t mk = mask[idx % W];
    if (mk) best_sb[idx] = (best_sb[idx] & ~mk) | (sb[idx] & mk);
}

__global__ void k_fill(double* a, int64_t n, double v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}

struct Tracker {
    bool trace = false, best = false;
    int64_t n = 0, R = 0, W = 0;
    DevBuf<double> e, best_e, tr;
    DevBuf<uint32_t> mask, best_sb;
    void init(Problem* p, const Layout& L, int64_t T, bool want_trace, bool want_best,
              cudaStream_t s) {
        trace = want_trace;
        best = want_best;
        n = L.n;
        R = L.R;
        W = L.W;
        if (!trace && !best) return;
        e = DevBuf<double>(R, s);
        if (trace) tr = DevBuf<double>(std::max<int64_t>(T, 1), s);
        if (best) {
            best_e = DevBuf<double>(R, s);
            k_fill<<<nblk(R), TB, 0, s>>>(best_e.get(), R, INFINITY);
            mask = DevBuf<uint32_t>(W, s);
            best_sb = DevBuf<uint32_t>(n * W, s);
            VXQ_CUDA(cudaMemsetAsync(best_sb.get(), 0, n * W * sizeof(uint32_t), s));
        }
    }
    // spins s_t (bit-packed, all rows) entering step t; t == T for the final state
    void observe(Problem* p, const uint32_t* sb, int64_t t, int64_t T, cudaStream_t s) {
        if (!trace && !best) return;
        if (!best && t >= T) return;
        energies_from_bits(p, sb, W, R, e.get(), s);
        if (trace && t < T) k_trace_min<<<1, 256, 0, s>>>(e.get(), R, tr.get() + t);
        if (best) {
            k_update_best<<<(unsigned)ceil_div(W * 32, 256), 256, 0, s>>>(e.get(), R,
                                                                         best_e.get(), mask.get());
            k_merge_bits<<<nblk(n * W), TB, 0, s>>>(n * W, W, mask.get(), sb, best_sb.get());
        }
        VXQ_CHECK_LAUNCH();
    }
    void export_trace(vxq_outputs* out, int64_t T, bool on_dev, cudaStream_t s) {
        if (!trace || !out->energy_trace) return;
        VXQ_CUDA(cudaMemcpyAsync(out->energy_trace, tr.get(), T * sizeof(double),
                                 on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
    }
};

// ---- blocked sparse SBM (k_sbm_block): per-problem neighbour slots, plan, launch
// VXQ_SBM_BLOCK: 0 = never (default), 1 = when sampled blocks show >= 2 entries per staged
// row, 2 = whenever the slots fit shared memory.  Opt-in: on cfg 3 the blocked step cuts
// L2 -> SM gather bytes 3x but measured 174 us against the step kernel's 142
// (profiles/r02/ab_sbm_block): its staging and summing phases do not overlap at 2 CTAs/SM.
int sbm_block_mode() {
    const char* e = getenv("VXQ_SBM_BLOCK");
    return e ? atoi(e) : 0;
}

}  // namespace

struct NbrBlocks {
    int nb = 0, max_u = 0, max_e = 0;
    int64_t total_u = 0;
    double reuse = 0.0;                // entries per staged neighbour row
    int32_t* u_ptr = nullptr;          // [nb + 1]
    int32_t* u_idx = nullptr;          // [total_u] distinct neighbours of each block, ascending
    uint16_t* slot = nullptr;          // [nnz] CSR entry -> slot in its block's list
};

void nbr_blocks_destroy(NbrBlocks* b) {
    if (!b) return;
    if (b->u_ptr) cudaFree(b->u_ptr);
    if (b->u_idx) cudaFree(b->u_idx);
    if (b->slot) cudaFree(b->slot);
    delete b;
}

namespace {

constexpr size_t kSbmBlockSmemMax = (kSbmBlockV >= 4 ? 200 : 110) * 1024;  // 2 CTAs/SM when V <= 2
constexpr double kSbmBlockMinReuse = 2.0;

// Distinct-neighbour lists of every kSbmBlockRows-row block (host, once per problem; the
// CSR is tiny for the graphs this serves).  Cheap rejection first: a sample of blocks must
// show reuse >= kSbmBlockMinReuse and fit shared memory.
NbrBlocks* nbr_blocks_get(Problem* p, int mode, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(p->mu);
    if (p->nbr_blocks_state != 0) return p->nbr_blocks_state > 0 ? p->nbr_blocks : nullptr;
    const int64_t n = p->n, nnz = p->nnz;
    const int64_t nb = ceil_div(n, kSbmBlockRows);
    if (n < 2 * kSbmBlockRows || nnz == 0 || nnz > ((int64_t)1 << 26) || nb > ((int64_t)1 << 30)) {
        p->nbr_blocks_state = -1;
        return nullptr;
    }
    std::vector<int64_t> ip(n + 1);
    VXQ_CUDA(cudaMemcpyAsync(ip.data(), p->indptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    std::vector<int32_t> ix(nnz);
    VXQ_CUDA(cudaMemcpyAsync(ix.data(), p->indices, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    VXQ_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> tmp;
    auto uniq = [&](int64_t b) {
        const int64_t r0 = b * kSbmBlockRows, r1 = std::min(n, r0 + kSbmBlockRows);
        tmp.assign(ix.begin() + ip[r0], ix.begin() + ip[r1]);
        std::sort(tmp.begin(), tmp.end());
        tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
        return (int64_t)tmp.size();
    };
    const size_t row_bytes = 32 * kSbmBlockV * sizeof(float);  // one fp32 chunk row
    const size_t ent_b = sizeof(float) + sizeof(uint16_t);  // per staged CSR entry
    if (mode == 1) {  // sample 16 blocks spread over the rows
        int64_t ent = 0, un = 0;
        for (int k = 0; k < 16; ++k) {
            const int64_t b = (nb - 1) * k / 15;
            const int64_t r0 = b * kSbmBlockRows, r1 = std::min(n, r0 + kSbmBlockRows);
            ent += ip[r1] - ip[r0];
            const int64_t u = uniq(b);
            un += u;
            if ((size_t)u * row_bytes + (size_t)(ip[r1] - ip[r0] + 8) * ent_b > kSbmBlockSmemMax ||
                ip[r1] - ip[r0] > kSbmBlockMaxEnt) {
                p->nbr_blocks_state = -1;
                return nullptr;
            }
        }
        if (un == 0 || (double)ent / (double)un < kSbmBlockMinReuse) {
            p->nbr_blocks_state = -1;
            return nullptr;
        }
    }
    NbrBlocks* B = new NbrBlocks;
    B->nb = (int)nb;
    std::vector<int32_t> uptr(nb + 1, 0), uidx;
    std::vector<uint16_t> sl(nnz);
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t u = uniq(b);
        const int64_t r0b = b * kSbmBlockRows, r1b = std::min(n, r0b + kSbmBlockRows);
        if ((size_t)u * row_bytes + (size_t)(ip[r1b] - ip[r0b] + 8) * ent_b > kSbmBlockSmemMax ||
            u > 65535 || ip[r1b] - ip[r0b] > kSbmBlockMaxEnt) {
            delete B;
            p->nbr_blocks_state = -1;
            return nullptr;
        }
        B->max_u = std::max<int>(B->max_u, (int)u);
        B->max_e = std::max<int>(B->max_e, (int)(ip[r1b] - ip[r0b]));
        const int64_t r0 = b * kSbmBlockRows, r1 = std::min(n, r0 + kSbmBlockRows);
        for (int64_t e = ip[r0]; e < ip[r1]; ++e)
            sl[e] = (uint16_t)(std::lower_bound(tmp.begin(), tmp.end(), ix[e]) - tmp.begin());
        uidx.insert(uidx.end(), tmp.begin(), tmp.end());
        uptr[b + 1] = (int32_t)uidx.size();
    }
    B->total_u = (int64_t)uidx.size();
    B->reuse = (double)nnz / (double)std::max<int64_t>(1, B->total_u);
    if (mode == 1 && B->reuse < kSbmBlockMinReuse) {
        delete B;
        p->nbr_blocks_state = -1;
        return nullptr;
    }
    VXQ_CUDA(cudaMalloc(&B->u_ptr, (nb + 1) * sizeof(int32_t)));
    VXQ_CUDA(cudaMalloc(&B->u_idx, std::max<int64_t>(1, B->total_u) * sizeof(int32_t)));
    VXQ_CUDA(cudaMalloc(&B->slot, nnz * sizeof(uint16_t)));
    VXQ_CUDA(cudaMemcpyAsync(B->u_ptr, uptr.data(), (nb + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    VXQ_CUDA(cudaMemcpyAsync(B->u_idx, uidx.data(), B->total_u * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    VXQ_CUDA(cudaMemcpyAsync(B->slot, sl.data(), nnz * sizeof(uint16_t), cudaMemcpyHostToDevice, s));
    VXQ_CUDA(cudaStreamSynchronize(s));
    p->nbr_blocks = B;
    p->nbr_blocks_state = 1;
    return B;
}

template <typename T>
void launch_sbm_block(const NbrBlocks& B, const Layout& L, const Operator<T>& op, const T* g,
                      SbmScalars<T> sc, const T* qi, T* qo, T* p, cudaStream_t s) {
    const int ent_cap = (B.max_e + 7) / 8 * 8;
    const size_t smem = (size_t)B.max_u * 32 * L.V * sizeof(T) +
                        (size_t)ent_cap * (sizeof(T) + sizeof(uint16_t));
    dim3 grid((unsigned)B.nb, (unsigned)(L.R_pad / (32 * L.V)));
#define VXQ_SBM_BLK(VV)                                                                      \
    {                                                                                        \
        VXQ_CUDA(cudaFuncSetAttribute(k_sbm_block<T, VV>,                                    \
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        k_sbm_block<T, VV><<<grid, kSbmBlockThreads, smem, s>>>(L.n, L.R_pad, B.u_ptr, B.u_idx, \
                                                               B.slot, op, g, sc, qi, qo, p, ent_cap); \
    }
    switch (L.V) {
        case 1: VXQ_SBM_BLK(1); break;
        case 2: VXQ_SBM_BLK(2); break;
        default:
            if constexpr (sizeof(T) == 4) VXQ_SBM_BLK(4);
            break;
    }
#undef VXQ_SBM_BLK
}

// Common tail: sign bits -> exact energies -> states / order / analog exports.
template <typename T>
void finish_outputs(Problem* p, const Layout& L, const uint32_t* sb, const T* xa, const T* ma,
                    const vxq_run_opts* opts, vxq_outputs* out, cudaStream_t s,
                    const long long* q2 = nullptr) {
    const bool on_dev = opts && opts->outputs_on_device;
    const int64_t n = L.n, R = L.R;
    DevBuf<double> e_tmp;
    double* e_dev = out->energies;
    if (!on_dev) {
        e_tmp = DevBuf<double>(R, s);
        e_dev = e_tmp.get();
    }
    energies_from_bits(p, sb, L.W, R, e_dev, s, q2);
    DevBuf<int8_t> st_tmp;
    int8_t* st_dev = out->states;
    if (!on_dev) {
        st_tmp = DevBuf<int8_t>(n * R, s);
        st_dev = st_tmp.get();
    }
    bits_to_states(sb, n, R, L.W, st_dev, s);
    DevBuf<int64_t> ord_tmp;
    if (out->order) {
        int64_t* od = out->order;
        if (!on_dev) {
            ord_tmp = DevBuf<int64_t>(R, s);
            od = ord_tmp.get();
        }
        stable_order(e_dev, R, od, s);
        if (!on_dev)
            VXQ_CUDA(cudaMemcpyAsync(out->order, od, R * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    }
    DevBuf<double> xt, mt;
    if (out->x) {
        double* xd = out->x;
        if (!on_dev) {
            xt = DevBuf<double>(n * R, s);
            xd = xt.get();
        }
        k_export<T><<<nblk(n * R), TB, 0, s>>>(xa, n, R, L.R_pad, L.V, xd);
        VXQ_CHECK_LAUNCH();
        if (!on_dev)
            VXQ_CUDA(cudaMemcpyAsync(out->x, xd, n * R * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    if (out->m) {
        double* md = out->m;
        if (!on_dev) {
            mt = DevBuf<double>(n * R, s);
            md = mt.get();
        }
        k_export<T><<<nblk(n * R), TB, 0, s>>>(ma, n, R, L.R_pad, L.V, md);
        VXQ_CHECK_LAUNCH();
        if (!on_dev)
            VXQ_CUDA(cudaMemcpyAsync(out->m, md, n * R * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    if (!on_dev) {
        VXQ_CUDA(cudaMemcpyAsync(out->energies, e_dev, R * sizeof(double), cudaMemcpyDeviceToHost, s));
        VXQ_CUDA(cudaMemcpyAsync(out->states, st_dev, n * R, cudaMemcpyDeviceToHost, s));
    }
    VXQ_CUDA(cudaStreamSynchronize(s));
}

template <typename T>
Operator<T> problem_operator(Problem* p, T sign) {
    Operator<T> op;
    op.indptr = p->indptr;
    op.indices = p->indices;
    if constexpr (sizeof(T) == 8) op.data = reinterpret_cast<const T*>(p->data64);
    else op.data = reinterpret_cast<const T*>(p->data32);
    op.sign = sign;
    return op;
}

template <typename T>
const T* pick(const double* d64, const float* d32) {
    if constexpr (sizeof(T) == 8) return reinterpret_cast<const T*>(d64);
    else return reinterpret_cast<const T*>(d32);
}

template <typename T>
void pa_solve_t(Problem* p, const vxq_pa_params* prm, const vxq_run_opts* opts, vxq_outputs* out,
                cudaStream_t s) {
    const int64_t n = p->n, R = prm->replicas, T_ = prm->steps;
    Layout L = make_layout(n, R, sizeof(T) == 8);
    double lam0 = std::isnan(prm->lambda0) ? problem_lambda0(p, s) : prm->lambda0;
    out->lambda0_used = lam0;
    std::vector<double> sched(T_);
    pa_schedule(lam0, T_, sched.data());
    const T eta = (T)prm->learning_rate, alpha = (T)prm->momentum;
    const int64_t rbegin = opts ? opts->replica_begin : 0;

    DevBuf<T> x(n * L.R_pad, s), m(n * L.R_pad, s);
    DevBuf<uint32_t> sbA(n * L.W, s), sbB(n * L.W, s);
    int64_t launches = 0;
    k_init_pa<T><<<nblk(((n + 3) / 4 + 1) * L.R_pad), TB, 0, s>>>(0, n, L.R_pad, L.V, prm->seed,
                                                                rbegin, x.get(), m.get());
    VXQ_CHECK_LAUNCH();
    ++launches;
    Operator<T> op = problem_operator<T>(p, (T)1);
    const T* h = pick<T>(p->h64, p->h32);
    int RG = resident_rg(L);
    size_t smem = resident_smem_pa(L, RG, sizeof(T), p->nnz);
    const int req = opts ? opts->path : 0;
    int path = VXQ_PATH_DENSE;
    if constexpr (sizeof(T) == 8) {
        if (req == VXQ_PATH_DENSE)
            throw Error(VXQ_ERR_UNSUPPORTED, "dense tensor-core path is fp32 only");
    }
    const bool want_best = opts && opts->track_best;
    const bool want_trace = out->energy_trace != nullptr;
    // fused best tracking on the dense path uses the in-kernel exact coupling energies,
    // which are the whole energy only when h == 0 (else: the sparse path's exact tracker)
    const bool dense_cand =
        sizeof(T) == 4 && p->uniform_magnitude &&
        (req == VXQ_PATH_DENSE || (req == VXQ_PATH_AUTO && dense_eligible(p, R)));
    // general (non-uniform) dense J: fp16 J planes on the tensor cores, PA without tracking
    const bool gen_cand =
        sizeof(T) == 4 && !p->uniform_magnitude &&
        (req == VXQ_PATH_DENSE || (req == VXQ_PATH_AUTO && dense_general_eligible(p, R)));
    if (gen_cand && req == VXQ_PATH_DENSE && (want_best || want_trace))
        throw Error(VXQ_ERR_UNSUPPORTED,
                    "trace / track_best on the dense path need uniform |J_ij| (e.g. SK)");
    const bool dense_gen = gen_cand && !want_best && !want_trace;
    const bool h0 = want_best && dense_cand ? problem_h_zero(p, s) : true;
    if (want_best && req == VXQ_PATH_DENSE && !h0)
        throw Error(VXQ_ERR_UNSUPPORTED, "track_best on the dense path needs h = 0");
    const bool dense = dense_cand && (!want_best || h0);
    if (!dense && !dense_gen) path = choose_path(req, L, smem, p->nnz);
    // the resident kernel keeps spins in shared memory: tracking needs per-step spins
    if (!dense && !dense_gen && path == VXQ_PATH_RESIDENT && (want_best || want_trace)) {
        if (req == VXQ_PATH_RESIDENT)
            throw Error(VXQ_ERR_UNSUPPORTED, "tracking needs the sparse or dense path");
        path = VXQ_PATH_SPARSE;
    }
    Tracker trk;
    if (!dense && !dense_gen) trk.init(p, L, T_, want_trace, want_best, s);
    EventTimer tm(s);
    const uint32_t* sb_final = nullptr;
    bool used_cluster = false;
    DevBuf<long long> q2;
    DevBuf<uint32_t> sb_best;
    if (dense) {
        q2 = DevBuf<long long>(R, s);
        if (want_best) sb_best = DevBuf<uint32_t>(n * L.W, s);
        if constexpr (sizeof(T) == 4) {
            dense_pa_loop(p, R, L.R_pad, L.V, L.W, sched, eta, alpha, prm->seed, rbegin,
                          x.get(), m.get(), sbA.get(), q2.get(), s, &out->loop_ms, &launches,
                          out->energy_trace, opts && opts->outputs_on_device, sb_best.get());
        }
        sb_final = want_best ? sb_best.get() : sbA.get();
    } else if (dense_gen) {
        if constexpr (sizeof(T) == 4) {
            dense_pa_general_loop(p, R, L.R_pad, L.V, L.W, sched, eta, alpha, prm->seed, rbegin,
                                  x.get(), m.get(), sbA.get(), s, &out->loop_ms, &launches);
        }
        sb_final = sbA.get();
    } else if (path == VXQ_PATH_RESIDENT) {
        DevBuf<T> ds(std::max<int64_t>(T_, 1), s);
        std::vector<T> st(T_);
        for (int64_t t = 0; t < T_; ++t) st[t] = (T)sched[t];
        VXQ_CUDA(cudaMemcpyAsync(ds.get(), st.data(), T_ * sizeof(T), cudaMemcpyHostToDevice, s));
        VXQ_CUDA(cudaFuncSetAttribute(k_pa_resident<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kResidentSmemMax));
        unsigned grid = (unsigned)ceil_div(L.R_pad, RG);
        tm.start();
        k_pa_resident<T><<<grid, block_threads((int64_t)RG * n), smem, s>>>(
            n, L.R_pad, L.V, RG, (int)p->nnz, op, h, ds.get(), T_, eta, alpha, x.get(), m.get());
        VXQ_CHECK_LAUNCH();
        tm.stop();
        ++launches;
        launch_pack<T>(L, x.get(), sbA.get(), s);
        ++launches;
        sb_final = sbA.get();
        out->loop_ms = tm.ms();
        VXQ_CUDA(cudaStreamSynchronize(s));  // keep ds alive until done
    } else {
        launch_pack<T>(L, x.get(), sbA.get(), s);  // s_0 = sign(x_0)
        ++launches;
        uint32_t* bufs[2] = {sbA.get(), sbB.get()};
        PaClusterPlan pl;
        const bool cl = T_ > 0 && pa_cluster_plan<T>(L, &pl, s);
        used_cluster = cl;
        DevBuf<T> ds;
        if (cl) {  // lambda_t on the device for the multi-step launch
            ds = DevBuf<T>(T_, s);
            std::vector<T> st(T_);
            for (int64_t t = 0; t < T_; ++t) st[t] = (T)sched[t];
            VXQ_CUDA(cudaMemcpyAsync(ds.get(), st.data(), T_ * sizeof(T), cudaMemcpyHostToDevice, s));
            VXQ_CUDA(cudaStreamSynchronize(s));
        }
        tm.start();
        if (cl && !trk.trace && !trk.best) {  // all T steps in one launch
            launch_pa_cluster<T>(pl, L, op, h, ds.get(), 0, T_, eta, alpha, x.get(), m.get(),
                                 bufs[0], bufs[T_ & 1], s);
            ++launches;
        } else {
            for (int64_t t = 0; t < T_; ++t) {
                trk.observe(p, bufs[t & 1], t, T_, s);  // E(s_t): exact, bit-packed spins
                if (cl)
                    launch_pa_cluster<T>(pl, L, op, h, ds.get(), t, 1, eta, alpha, x.get(),
                                         m.get(), bufs[t & 1], bufs[(t + 1) & 1], s);
                else
                    launch_pa_step<T>(L, op, h, (T)sched[t], eta, alpha, x.get(), m.get(),
                                      bufs[t & 1], bufs[(t + 1) & 1], s);
                ++launches;
            }
        }
        VXQ_CHECK_LAUNCH();
        tm.stop();
        sb_final = bufs[T_ & 1];
        out->loop_ms = tm.ms();
        trk.observe(p, sb_final, T_, T_, s);
        trk.export_trace(out, T_, opts && opts->outputs_on_device, s);
        if (trk.best) sb_final = trk.best_sb.get();
    }
    out->path_used = (dense || dense_gen) ? VXQ_PATH_DENSE : path;
    out->dense_kind = (dense || dense_gen) ? dense_last_kind() : VXQ_DENSE_KIND_NONE;
    out->step_kernel = (dense || dense_gen)          ? VXQ_KERNEL_DENSE_RUN
                       : path == VXQ_PATH_RESIDENT   ? VXQ_KERNEL_PA_RESIDENT
                       : used_cluster                ? VXQ_KERNEL_PA_CLUSTER
                       : L.R_pad == 32               ? VXQ_KERNEL_PA_STEP_COOP
                                                     : VXQ_KERNEL_PA_STEP;
    // q2 (coupling energy counts of the final spins) only describes sb_final without tracking
    finish_outputs<T>(p, L, sb_final, x.get(), m.get(), opts, out, s,
                      dense && !want_best ? q2.get() : nullptr);
    out->launches = launches + 4;
}

template <typename T>
void sbm_run_core(Problem* p, const Layout& L, const Operator<T>& op, const T* g,
                  const std::vector<double>& a_sched, double dt, double a0, double c0,
                  double q_cap, int requested_path, int64_t nnz, T* q, T* qalt, T* pm,
                  vxq_outputs* out, int64_t& launches, cudaStream_t s, T** q_final,
                  Tracker* trk = nullptr, uint32_t* sb_scratch = nullptr,
                  const NbrBlocks* nbrb = nullptr) {
    const int64_t n = L.n, T_ = (int64_t)a_sched.size();
    SbmScalars<T> sc;
    sc.a_t = 0;
    sc.dt = (T)dt;
    sc.a0 = (T)a0;
    sc.c0 = (T)c0;
    sc.dta0 = (T)(dt * a0);  // (dt * a0) in Python floats, then * P
    sc.q_cap = (T)q_cap;
    int RG = resident_rg(L);
    size_t smem = resident_smem_sbm(L, RG, sizeof(T), nnz);
    int path = nbrb ? VXQ_PATH_SPARSE : choose_path(requested_path, L, smem, nnz);
    const bool tracking = trk && (trk->trace || trk->best);
    if (tracking && path == VXQ_PATH_RESIDENT) {
        if (requested_path == VXQ_PATH_RESIDENT)
            throw Error(VXQ_ERR_UNSUPPORTED, "tracking needs the sparse or dense path");
        path = VXQ_PATH_SPARSE;
    }
    EventTimer tm(s);
    if (path == VXQ_PATH_RESIDENT) {
        DevBuf<T> ds(std::max<int64_t>(T_, 1), s);
        std::vector<T> st(T_);
        for (int64_t t = 0; t < T_; ++t) st[t] = (T)a_sched[t];
        if (T_) VXQ_CUDA(cudaMemcpyAsync(ds.get(), st.data(), T_ * sizeof(T), cudaMemcpyHostToDevice, s));
        VXQ_CUDA(cudaFuncSetAttribute(k_sbm_resident<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kResidentSmemMax));
        unsigned grid = (unsigned)ceil_div(L.R_pad, RG);
        tm.start();
        k_sbm_resident<T><<<grid, block_threads((int64_t)RG * n), smem, s>>>(
            n, L.R_pad, L.V, RG, (int)nnz, op, g, ds.get(), T_, sc, q, pm);
        VXQ_CHECK_LAUNCH();
        tm.stop();
        ++launches;
        *q_final = q;
        if (out) out->loop_ms = tm.ms();
        VXQ_CUDA(cudaStreamSynchronize(s));
    } else {
        tm.start();
        T* qs[2] = {q, qalt};
        for (int64_t t = 0; t < T_; ++t) {
            if (tracking) {  // E(sign(q_t)), exact
                launch_pack<T>(L, qs[t & 1], sb_scratch, s);
                trk->observe(p, sb_scratch, t, T_, s);
            }
            sc.a_t = (T)a_sched[t];
            if (nbrb) launch_sbm_block<T>(*nbrb, L, op, g, sc, qs[t & 1], qs[(t + 1) & 1], pm, s);
            else launch_sbm_step<T>(L, op, g, sc, qs[t & 1], qs[(t + 1) & 1], pm, s);
            ++launches;
        }
        VXQ_CHECK_LAUNCH();
        tm.stop();
        *q_final = qs[T_ & 1];
        if (out) out->loop_ms = tm.ms();
    }
    if (out) {
        out->path_used = path;
        out->dense_kind = VXQ_DENSE_KIND_NONE;
        out->step_kernel = path == VXQ_PATH_RESIDENT ? VXQ_KERNEL_SBM_RESIDENT
                           : nbrb                    ? VXQ_KERNEL_SBM_BLOCK
                                                     : VXQ_KERNEL_SBM_STEP;
    }
}

template <typename T>
void sbm_solve_t(Problem* p, const vxq_sbm_params* prm, const vxq_run_opts* opts,
                 vxq_outputs* out, cudaStream_t s) {
    const int64_t n = p->n, R = prm->replicas, T_ = prm->steps;
    const int req = opts ? opts->path : 0;
    if constexpr (sizeof(T) == 8) {
        if (req == VXQ_PATH_DENSE)
            throw Error(VXQ_ERR_UNSUPPORTED, "dense tensor-core path is fp32 only");
    }
    const bool want_best = opts && opts->track_best;
    const bool want_trace = out->energy_trace != nullptr;
    if (want_best && req == VXQ_PATH_DENSE)
        throw Error(VXQ_ERR_UNSUPPORTED, "track_best is not available on the dense path yet");
    // uniform |J| (SK family): sign matrix K; general dense J: fp16 J planes (needs fp16 q)
    const bool elig = p->uniform_magnitude
                          ? dense_eligible(p, R)
                          : dense_general_eligible(p, R) && dense_sbm_fp16_ok(prm->q_cap,
                                                                              prm->init_noise);
    const bool dense = sizeof(T) == 4 && !want_best &&
                       (req == VXQ_PATH_DENSE || (req == VXQ_PATH_AUTO && elig));
    Layout L = make_layout(n, R, sizeof(T) == 8);
    // blocked sparse step (structured graphs, fp32)
    const NbrBlocks* nbrb = nullptr;
    if constexpr (sizeof(T) == 4) {
        const int bmode = sbm_block_mode();
        if (!dense && bmode != 0 && (req == VXQ_PATH_AUTO || req == VXQ_PATH_SPARSE)) {
            const int RG = resident_rg(L);
            const size_t rsm = resident_smem_sbm(L, RG, sizeof(T), p->nnz);
            if (choose_path(req, L, rsm, p->nnz) == VXQ_PATH_SPARSE) {
                nbrb = nbr_blocks_get(p, bmode, s);
                if (nbrb && L.V > kSbmBlockV) {  // narrower chunks: staged rows fit 2 CTAs/SM
                    L.V = kSbmBlockV;
                    L.R_pad = ceil_div(R, 32 * L.V) * 32 * L.V;
                    L.W = L.R_pad / 32;
                }
            }
        }
    }
    double c0 = std::isnan(prm->c0) ? problem_c0(p, s) : prm->c0;
    out->c0_used = c0;
    std::vector<double> sched(T_);
    sbm_schedule(prm->a0, T_, sched.data());
    const int64_t rbegin = opts ? opts->replica_begin : 0;
    DevBuf<T> q(n * L.R_pad, s), q2(n * L.R_pad, s), pm(n * L.R_pad, s);
    DevBuf<uint32_t> sb(n * L.W, s);
    int64_t launches = 0;
    k_init_sbm<T><<<nblk(((2 * n + 3) / 4) * L.R_pad), TB, 0, s>>>(
        n, 0, n, L.R_pad, L.V, prm->seed, rbegin, prm->init_noise, q.get(), pm.get());
    VXQ_CHECK_LAUNCH();
    ++launches;
    if (dense) {
        // per-step energies (want_trace): exact on the uniform-|J| exact-field kernel with
        // h = 0 (a spin plane next to the digit planes), NaN on the other dense kinds
        DevBuf<long long> qq(R, s);
        if constexpr (sizeof(T) == 4) {
            dense_sbm_loop(p, R, L.R_pad, L.V, L.W, sched, prm->dt, prm->a0, c0, prm->q_cap,
                           prm->init_noise, prm->seed, rbegin, q.get(), pm.get(), sb.get(),
                           p->uniform_magnitude ? qq.get() : nullptr, s, &out->loop_ms,
                           &launches, want_trace ? out->energy_trace : nullptr,
                           opts && opts->outputs_on_device);
        }
        out->path_used = VXQ_PATH_DENSE;
        out->dense_kind = dense_last_kind();
        out->step_kernel = VXQ_KERNEL_DENSE_RUN;
        finish_outputs<T>(p, L, sb.get(), q.get(), pm.get(), opts, out, s,
                          p->uniform_magnitude ? qq.get() : nullptr);
        out->launches = launches + 4;
        return;
    }
    Operator<T> op = problem_operator<T>(p, (T)-1);  // B = -A
    const T* g = pick<T>(p->g64, p->g32);            // g = -h
    T* qf = nullptr;
    Tracker trk;
    trk.init(p, L, T_, want_trace, want_best, s);
    sbm_run_core<T>(p, L, op, g, sched, prm->dt, prm->a0, c0, prm->q_cap, req, p->nnz,
                    q.get(), q2.get(), pm.get(), out, launches, s, &qf, &trk, sb.get(), nbrb);
    launch_pack<T>(L, qf, sb.get(), s);
    ++launches;
    trk.observe(p, sb.get(), T_, T_, s);
    trk.export_trace(out, T_, opts && opts->outputs_on_device, s);
    finish_outputs<T>(p, L, trk.best ? trk.best_sb.get() : sb.get(), qf, pm.get(), opts, out, s);
    out->launches = launches + 4;
}

}  // namespace

void finish_from_bits(Problem* p, int64_t R, int64_t W, const uint32_t* sb,
                      const vxq_run_opts* opts, vxq_outputs* out, cudaStream_t s) {
    VXQ_REQUIRE(!out->x && !out->m, "x/m outputs are not available for this solver");
    Layout L = make_layout(p->n, R, false);
    L.W = W;
    L.R_pad = W * 32;
    finish_outputs<float>(p, L, sb, nullptr, nullptr, opts, out, s);
}

void pa_solve(Problem* p, const vxq_pa_params* prm, const vxq_run_opts* opts, vxq_outputs* out,
              cudaStream_t s) {
    if (opts && opts->precision == VXQ_FP64) pa_solve_t<double>(p, prm, opts, out, s);
    else pa_solve_t<float>(p, prm, opts, out, s);
}

void sbm_solve(Problem* p, const vxq_sbm_params* prm, const vxq_run_opts* opts,
               vxq_outputs* out, cudaStream_t s) {
    if (opts && opts->precision == VXQ_FP64) sbm_solve_t<double>(p, prm, opts, out, s);
    else sbm_solve_t<float>(p, prm, opts, out, s);
}

namespace {
__global__ void k_to_f32(int64_t n, const double* a, float* b) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = __double2float_rn(a[i]);
}

template <typename T>
void integrate_t(int64_t n, const int64_t* bt_indptr, const int32_t* bt_indices,
                 const double* bt_data, const double* g, int64_t R, double* Q, double* P,
                 const double* a_sched, int64_t T_, double dt, double a0, double c0,
                 double q_cap, const vxq_run_opts* opts, cudaStream_t s) {
    int64_t nnz = bt_indptr[n];
    DevBuf<int64_t> ip(n + 1, s);
    DevBuf<int32_t> ix(std::max<int64_t>(nnz, 1), s);
    DevBuf<double> dv(std::max<int64_t>(nnz, 1), s), gv(n, s);
    DevBuf<float> dv32(std::max<int64_t>(nnz, 1), s), gv32(n, s);
    VXQ_CUDA(cudaMemcpyAsync(ip.get(), bt_indptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (nnz) {
        VXQ_CUDA(cudaMemcpyAsync(ix.get(), bt_indices, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        VXQ_CUDA(cudaMemcpyAsync(dv.get(), bt_data, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
        k_to_f32<<<nblk(nnz), TB, 0, s>>>(nnz, dv.get(), dv32.get());
    }
    VXQ_CUDA(cudaMemcpyAsync(gv.get(), g, n * sizeof(double), cudaMemcpyHostToDevice, s));
    k_to_f32<<<nblk(n), TB, 0, s>>>(n, gv.get(), gv32.get());
    VXQ_CHECK_LAUNCH();
    Layout L = make_layout(n, R, sizeof(T) == 8);
    DevBuf<double> hq(n * R, s), hp(n * R, s);
    VXQ_CUDA(cudaMemcpyAsync(hq.get(), Q, n * R * sizeof(double), cudaMemcpyHostToDevice, s));
    VXQ_CUDA(cudaMemcpyAsync(hp.get(), P, n * R * sizeof(double), cudaMemcpyHostToDevice, s));
    DevBuf<T> q(n * L.R_pad, s), q2(n * L.R_pad, s), pm(n * L.R_pad, s);
    k_import<T><<<nblk(n * L.R_pad), TB, 0, s>>>(hq.get(), n, R, L.R_pad, L.V, q.get());
    k_import<T><<<nblk(n * L.R_pad), TB, 0, s>>>(hp.get(), n, R, L.R_pad, L.V, pm.get());
    VXQ_CHECK_LAUNCH();
    Operator<T> op;
    op.indptr = ip.get();
    op.indices = ix.get();
    op.data = pick<T>(dv.get(), dv32.get());
    op.sign = (T)1;
    std::vector<double> sched(a_sched, a_sched + T_);
    int64_t launches = 0;
    T* qf = nullptr;
    int req = opts ? opts->path : 0;
    sbm_run_core<T>(nullptr, L, op, pick<T>(gv.get(), gv32.get()), sched, dt, a0, c0, q_cap, req,
                    nnz, q.get(), q2.get(), pm.get(), nullptr, launches, s, &qf);
    k_export<T><<<nblk(n * R), TB, 0, s>>>(qf, n, R, L.R_pad, L.V, hq.get());
    k_export<T><<<nblk(n * R), TB, 0, s>>>(pm.get(), n, R, L.R_pad, L.V, hp.get());
    VXQ_CHECK_LAUNCH();
    VXQ_CUDA(cudaMemcpyAsync(Q, hq.get(), n * R * sizeof(double), cudaMemcpyDeviceToHost, s));
    VXQ_CUDA(cudaMemcpyAsync(P, hp.get(), n * R * sizeof(double), cudaMemcpyDeviceToHost, s));
    VXQ_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

void sbm_integrate(int64_t n, const int64_t* bt_indptr, const int32_t* bt_indices,
                   const double* bt_data, const double* g, int64_t R, double* Q, double* P,
                   const double* a_sched, int64_t T_, double dt, double a0, double c0,
                   double q_cap, const vxq_run_opts* opts, cudaStream_t s) {
    if (opts && opts->precision == VXQ_FP64)
        integrate_t<double>(n, bt_indptr, bt_indices, bt_data, g, R, Q, P, a_sched, T_, dt, a0,
                            c0, q_cap, opts, s);
    else
        integrate_t<float>(n, bt_indptr, bt_indices, bt_data, g, R, Q, P, a_sched, T_, dt, a0,
                           c0, q_cap, opts, s);
}

}  // namespace vxq

// ====================================================================== row-partitioned sessions
// One rank of a row-partitioned solve: this process updates rows
// [row0, row0 + nrows) of every replica each step and reads every row's state from an
// exchange buffer that the caller all-gathers between steps (NCCL over NVLink):
//   PA : sign bits  [rows_alloc][W] uint32      (1 bit per replica-variable)
//   SBM: q          [rows_alloc][R_pad] fp32/64 (interleaved replica layout)
// Buffer k & 1 holds state k; init writes state 0 (local rows), step t reads buffer t & 1
// and writes the local rows of buffer (t + 1) & 1.
//
// Fused exchange (set_peers): instead of a caller all-gather, the step kernels store every
// produced word / q vector straight into all ranks' copies of the exchange buffer (CUDA
// IPC pointers over NVLink), and the ranks synchronise through one flag per (rank, source):
// after writing state k a rank release-stores k + 1 into flags[rank] of every peer; before
// step t it acquire-polls its own flags until every source shows >= t + 1 (state t
// complete).  A rank therefore starts step t only after every peer has finished step t - 1,
// i.e. stopped reading the buffer that step t overwrites, so two buffers suffice.
namespace vxq {

namespace {
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// state k complete on this rank: publish k + 1 to every rank's flag slot `rank`
// (stream order puts the step kernel's stores -- local and remote -- before this kernel)
__global__ void k_signal(const Dests<uint64_t> flags, int rank, uint64_t v) {
    if ((int)threadIdx.x < flags.n) {
        __threadfence_system();
        st_release_sys(flags.p[threadIdx.x] + rank, v);
    }
}

// wait until every source rank has published >= need; bounded (30 s), then reports
// through *status instead of hanging the GPU.  Once any wait has failed (status != 0) every
// later wait returns at once: the host sees the status after at most one step
// (session_step) instead of spinning 30 s per remaining step.
__global__ void k_wait(const uint64_t* flags, int n, uint64_t need, volatile int* status) {
    if ((int)threadIdx.x >= n) return;
    if (*status) return;
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(flags + threadIdx.x) < need) {
        __nanosleep(200);
        if (*status) return;
        if (global_ns() - t0 > 30ull * 1000000000ull) {
            *status = 1;
            __threadfence_system();
            return;
        }
    }
}
}  // namespace

struct Session {
    Problem* p = nullptr;
    int solver = 0;  // 0 PA, 1 SBM
    int prec = VXQ_FP32;
    Layout L;
    int64_t rows_alloc = 0, rbegin = 0;
    uint64_t seed = 0;
    void* xb[2] = {nullptr, nullptr};
    void* x = nullptr;  // PA x / SBM p (local rows)
    void* m = nullptr;  // PA m (local rows)
    std::vector<double> sched;
    double eta = 0, alpha = 0, lam0 = 0;                          // PA
    double dt = 0, a0 = 0, c0 = 0, q_cap = 0, amp = 0;            // SBM
    cudaStream_t s = nullptr;
    bool own_stream = false;
    // fused exchange (set_peers)
    int world = 1, rank = 0;
    bool peers = false;
    Dests<void> pxb[2] = {};      // every rank's exchange buffers (own at [rank])
    Dests<uint64_t> pflags = {};  // every rank's flag array (own at [rank])
    int* status = nullptr;        // mapped pinned host word: 1 = a peer wait timed out
    int* status_dev = nullptr;    // its device alias (written by k_wait)
    uint64_t epoch = 0;           // flag values are (epoch << 32) + state + 1
    int64_t row_bytes = 0;
    int64_t done = 0;             // steps taken (step t must follow step t - 1)
    ~Session() {  // state from the retained stream-ordered pool (no unmapping)
        if (x) cudaFreeAsync(x, s);
        if (m) cudaFreeAsync(m, s);
        if (s) cudaStreamSynchronize(s);
        if (status) cudaFreeHost(status);
        if (own_stream && s) cudaStreamDestroy(s);
    }
};

int64_t exchange_row_bytes(int solver, int64_t R, int prec) {
    Layout L = make_layout(1, R, prec == VXQ_FP64);
    if (solver == 0) return L.W * 4;
    return L.R_pad * (prec == VXQ_FP64 ? 8 : 4);
}

namespace {
template <typename T>
void session_init_t(Session* S) {
    const Layout& L = S->L;
    const int64_t n = S->p->n;
    VXQ_CUDA(cudaMallocAsync(&S->x, std::max<int64_t>(L.nrows, 1) * L.R_pad * sizeof(T), S->s));
    if (S->solver == 0) {
        VXQ_CUDA(cudaMallocAsync(&S->m, std::max<int64_t>(L.nrows, 1) * L.R_pad * sizeof(T), S->s));
        k_init_pa<T><<<nblk(((L.nrows + 3) / 4 + 1) * L.R_pad), TB, 0, S->s>>>(
            L.row0, L.nrows, L.R_pad, L.V, S->seed, S->rbegin, (T*)S->x, (T*)S->m);
        VXQ_CHECK_LAUNCH();
        launch_pack<T>(L, (const T*)S->x, (uint32_t*)S->xb[0], S->s);
    } else {
        k_init_sbm<T><<<nblk(((2 * n + 3) / 4) * L.R_pad), TB, 0, S->s>>>(
            n, L.row0, L.nrows, L.R_pad, L.V, S->seed, S->rbegin, S->amp, (T*)S->xb[0],
            (T*)S->x);
        VXQ_CHECK_LAUNCH();
    }
}

template <typename P>
Dests<P> cast_dests(const Dests<void>& d) {
    Dests<P> o{};
    for (int k = 0; k < d.n; ++k) o.p[k] = static_cast<P*>(d.p[k]);
    o.n = d.n;
    return o;
}

template <typename T>
void session_step_t(Session* S, int64_t t) {
    const Layout& L = S->L;
    const int nb = (t + 1) & 1;
    if (S->peers) {  // state t complete on every rank
        // a wait of an earlier step timed out (the host-mapped status word): fail now rather
        // than launching the remaining steps on incomplete state
        if (*(volatile int*)S->status)
            throw Error(VXQ_ERR_CUDA, "row-partition exchange: a peer did not publish its "
                                      "rows within 30 s");
        k_wait<<<1, 32, 0, S->s>>>(S->pflags.p[S->rank], S->world, S->epoch + (uint64_t)t + 1,
                                   S->status_dev);
        VXQ_CHECK_LAUNCH();
    }
    if (S->solver == 0) {
        Operator<T> op = problem_operator<T>(S->p, (T)1);
        const Dests<uint32_t> out = S->peers ? cast_dests<uint32_t>(S->pxb[nb])
                                             : one_dest((uint32_t*)S->xb[nb]);
        launch_pa_step<T>(L, op, pick<T>(S->p->h64, S->p->h32), (T)S->sched[t], (T)S->eta,
                          (T)S->alpha, (T*)S->x, (T*)S->m, (const uint32_t*)S->xb[t & 1], out,
                          S->s);
    } else {
        SbmScalars<T> sc;
        sc.a_t = (T)S->sched[t];
        sc.dt = (T)S->dt;
        sc.a0 = (T)S->a0;
        sc.c0 = (T)S->c0;
        sc.dta0 = (T)(S->dt * S->a0);
        sc.q_cap = (T)S->q_cap;
        Operator<T> op = problem_operator<T>(S->p, (T)-1);
        const Dests<T> out = S->peers ? cast_dests<T>(S->pxb[nb]) : one_dest((T*)S->xb[nb]);
        launch_sbm_step<T>(L, op, pick<T>(S->p->g64, S->p->g32), sc, (const T*)S->xb[t & 1],
                           out, (T*)S->x, S->s);
    }
    VXQ_CHECK_LAUNCH();
    if (S->peers) {
        k_signal<<<1, 32, 0, S->s>>>(S->pflags, S->rank, S->epoch + (uint64_t)t + 2);
        VXQ_CHECK_LAUNCH();
    }
}

template <typename T>
void session_finish_t(Session* S, int64_t T_, vxq_outputs* out, const vxq_run_opts* opts) {
    // full final state: PA sign bits / SBM q in buffer T & 1 (all rows, after the gather)
    if (S->peers) {
        k_wait<<<1, 32, 0, S->s>>>(S->pflags.p[S->rank], S->world, S->epoch + (uint64_t)T_ + 1,
                                   S->status_dev);
        VXQ_CHECK_LAUNCH();
        VXQ_CUDA(cudaStreamSynchronize(S->s));
        if (*(volatile int*)S->status) throw Error(VXQ_ERR_CUDA, "row-partition exchange: a peer did not publish its "
                                          "rows within 30 s");
    }
    Layout F = S->L;
    F.row0 = 0;
    F.nrows = S->p->n;
    // x/m (PA: X, M; SBM: Q, P) only from a session that owns every row
    const bool all_rows = S->L.row0 == 0 && S->L.nrows == S->p->n;
    VXQ_REQUIRE(all_rows || (!out->x && !out->m),
                "x/m outputs need a session over all rows [0, n)");
    const uint32_t* sb = nullptr;
    DevBuf<uint32_t> tmp;
    const T* xa = nullptr;
    const T* ma = nullptr;
    if (S->solver == 0) {
        sb = (const uint32_t*)S->xb[T_ & 1];
        xa = (const T*)S->x;
        ma = (const T*)S->m;
    } else {
        tmp = DevBuf<uint32_t>(S->p->n * F.W, S->s);
        launch_pack<T>(F, (const T*)S->xb[T_ & 1], tmp.get(), S->s);
        sb = tmp.get();
        xa = (const T*)S->xb[T_ & 1];
        ma = (const T*)S->x;
    }
    finish_outputs<T>(S->p, F, sb, xa, ma, opts, out, S->s);
    out->loop_ms = 0;
    out->path_used = VXQ_PATH_SPARSE;
    out->step_kernel = S->solver == 0 ? VXQ_KERNEL_PA_STEP : VXQ_KERNEL_SBM_STEP;
}
}  // namespace

Session* session_create(Problem* p, int solver, const vxq_pa_params* pa,
                        const vxq_sbm_params* sbm, int64_t row_begin, int64_t row_end,
                        int64_t rows_alloc, void* xbuf0, void* xbuf1, const vxq_run_opts* opts,
                        cudaStream_t s) {
    VXQ_REQUIRE(solver == 0 || solver == 1, "solver must be 0 (PA) or 1 (SBM)");
    VXQ_REQUIRE(0 <= row_begin && row_begin <= row_end && row_end <= p->n, "bad row range");
    VXQ_REQUIRE(rows_alloc >= p->n, "rows_alloc must be >= n");
    VXQ_REQUIRE(xbuf0 && xbuf1, "exchange buffers required");
    auto S = std::make_unique<Session>();
    S->p = p;
    S->solver = solver;
    S->prec = opts ? opts->precision : VXQ_FP32;
    const int64_t R = solver == 0 ? pa->replicas : sbm->replicas;
    const int64_t T_ = solver == 0 ? pa->steps : sbm->steps;
    S->L = make_layout(p->n, R, S->prec == VXQ_FP64);
    S->L.row0 = row_begin;
    S->L.nrows = row_end - row_begin;
    S->rows_alloc = rows_alloc;
    S->rbegin = opts ? opts->replica_begin : 0;
    S->xb[0] = xbuf0;
    S->xb[1] = xbuf1;
    S->s = s;
    S->row_bytes = exchange_row_bytes(solver, R, S->prec);
    S->sched.resize(T_);
    if (solver == 0) {
        S->seed = pa->seed;
        S->eta = pa->learning_rate;
        S->alpha = pa->momentum;
        S->lam0 = std::isnan(pa->lambda0) ? problem_lambda0(p, s) : pa->lambda0;
        pa_schedule(S->lam0, T_, S->sched.data());
    } else {
        S->seed = sbm->seed;
        S->dt = sbm->dt;
        S->a0 = sbm->a0;
        S->c0 = std::isnan(sbm->c0) ? problem_c0(p, s) : sbm->c0;
        S->q_cap = sbm->q_cap;
        S->amp = sbm->init_noise;
        sbm_schedule(S->a0, T_, S->sched.data());
    }
    if (S->prec == VXQ_FP64) session_init_t<double>(S.get());
    else session_init_t<float>(S.get());
    return S.release();
}

void session_step(Session* S, int64_t t) {
    VXQ_REQUIRE(t >= 0 && t < (int64_t)S->sched.size(), "step index out of range");
    VXQ_REQUIRE(t == S->done, "session steps must run in order 0, 1, ..., T-1");
    if (S->prec == VXQ_FP64) session_step_t<double>(S, t);
    else session_step_t<float>(S, t);
    S->done = t + 1;
}

void session_finish(Session* S, vxq_outputs* out, const vxq_run_opts* opts) {
    // the state after the steps taken (normally all T; fewer = a snapshot of the T-step
    // schedule after `done` steps)
    const int64_t T_ = S->done;
    if (S->prec == VXQ_FP64) session_finish_t<double>(S, T_, out, opts);
    else session_finish_t<float>(S, T_, out, opts);
    out->lambda0_used = S->lam0;
    out->c0_used = S->c0;
}

void session_set_peers(Session* S, int world, int rank, uint32_t epoch, void* const* xbuf0,
                       void* const* xbuf1, uint64_t* const* flags) {
    VXQ_REQUIRE(world >= 1 && world <= kMaxDests, "world must be in [1, 8]");
    VXQ_REQUIRE(rank >= 0 && rank < world, "rank out of range");
    VXQ_REQUIRE(xbuf0 && xbuf1 && flags, "peer pointer arrays required");
    VXQ_REQUIRE(xbuf0[rank] == S->xb[0] && xbuf1[rank] == S->xb[1],
                "xbuf0/xbuf1[rank] must be this session's own exchange buffers");
    VXQ_REQUIRE(!S->peers, "peers already set");
    VXQ_REQUIRE((uint64_t)S->sched.size() + 2 < (1ull << 32), "too many steps for the flag epoch");
    S->world = world;
    S->rank = rank;
    S->epoch = (uint64_t)epoch << 32;
    for (int k = 0; k < world; ++k) {
        VXQ_REQUIRE(xbuf0[k] && xbuf1[k] && flags[k], "null peer pointer");
        S->pxb[0].p[k] = xbuf0[k];
        S->pxb[1].p[k] = xbuf1[k];
        S->pflags.p[k] = flags[k];
    }
    S->pxb[0].n = S->pxb[1].n = S->pflags.n = world;
    VXQ_CUDA(cudaHostAlloc((void**)&S->status, sizeof(int), cudaHostAllocMapped));
    *(volatile int*)S->status = 0;
    VXQ_CUDA(cudaHostGetDevicePointer((void**)&S->status_dev, S->status, 0));
    // state 0 (written to the local rows by create) -> every peer, then publish it
    const int64_t off = S->L.row0 * S->row_bytes, bytes = S->L.nrows * S->row_bytes;
    for (int k = 0; k < world; ++k)
        if (k != rank && bytes > 0)
            VXQ_CUDA(cudaMemcpyAsync(static_cast<char*>(S->pxb[0].p[k]) + off,
                                     static_cast<const char*>(S->xb[0]) + off, bytes,
                                     cudaMemcpyDefault, S->s));
    S->peers = true;
    k_signal<<<1, 32, 0, S->s>>>(S->pflags, S->rank, S->epoch + 1);
    VXQ_CHECK_LAUNCH();
}

void session_destroy(Session* S) { delete S; }
void session_set_own_stream(Session* S, bool own) { S->own_stream = own; }

}  // namespace vxq
