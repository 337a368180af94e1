// vxq_common.cuh -- shared device/host helpers for the vxq sm_100a library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/vxq.h"

namespace vxq {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define VXQ_CUDA(expr)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess) {                                                         \
            int _c = (_e == cudaErrorMemoryAllocation) ? VXQ_ERR_OOM : VXQ_ERR_CUDA;     \
            throw ::vxq::Error(_c, std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                       " (" + __FILE__ + ":" + std::to_string(__LINE__) + \
                                       ")");                                             \
        }                                                                                \
    } while (0)

#define VXQ_CHECK_LAUNCH() VXQ_CUDA(cudaGetLastError())

#define VXQ_REQUIRE(cond, msg)                                 \
    do {                                                       \
        if (!(cond)) throw ::vxq::Error(VXQ_ERR_INVALID, msg); \
    } while (0)

// ---------------------------------------------------------------- Philox4x64-10
// numpy's bit generator (generators.py:35-40 -> np.random.Philox(key=seed).jumped(r)):
// raw draw k of replica r = philox(ctr=(k/4+1, 0, r, 0), key=(seed, 0))[k % 4].
struct U64x4 {
    uint64_t v[4];
};

__device__ __forceinline__ U64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2,
                                               uint64_t c3, uint64_t k0, uint64_t k1) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
        uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
        uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += W0;
        k1 += W1;
    }
    U64x4 o;
    o.v[0] = c0;
    o.v[1] = c1;
    o.v[2] = c2;
    o.v[3] = c3;
    return o;
}

// word k (0..3) of a Philox block by register select (a dynamic index would put the block
// in local memory)
__device__ __forceinline__ uint64_t pick_word(const U64x4& o, uint32_t k) {
    return k == 0 ? o.v[0] : k == 1 ? o.v[1] : k == 2 ? o.v[2] : o.v[3];
}

// numpy Generator.uniform(lo, hi) = lo + (hi - lo) * ((raw >> 11) * 2^-53), no FMA.
__device__ __forceinline__ double uniform_from_raw(uint64_t raw, double lo, double range) {
    double u = __dmul_rn((double)(raw >> 11), 1.0 / 9007199254740992.0);
    return __dadd_rn(lo, __dmul_rn(range, u));
}

// ---------------------------------------------------------------- rounding-exact ops
// The reference evaluates each numpy binary op with one rounding; these keep
// nvcc from contracting mul+add into FMA so fp64 mode stays bit-exact.
template <typename T>
struct Ops;
template <>
struct Ops<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
};
template <>
struct Ops<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
};

// vector of V scalars (16-byte max)
template <typename T, int V>
struct alignas(sizeof(T) * V) Vec {
    T v[V];
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Streaming (evict-first, ld/st.global.cs) accesses for the per-step state x/m/p and the
// CSR: they are touched once per step, so they should not evict the gathered spin / q
// tables from L2.  (Within one launch every state element belongs to one warp.)
template <typename T, int V>
__device__ __forceinline__ Vec<T, V> ld_cs(const T* p) {
    Vec<T, V> v;
    if constexpr (sizeof(T) * V == 16) {
        if constexpr (sizeof(T) == 4) {
            float4 t = __ldcs(reinterpret_cast<const float4*>(p));
            memcpy(&v, &t, 16);
        } else {
            double2 t = __ldcs(reinterpret_cast<const double2*>(p));
            memcpy(&v, &t, 16);
        }
    } else if constexpr (sizeof(T) * V == 8) {
        if constexpr (sizeof(T) == 4) {
            float2 t = __ldcs(reinterpret_cast<const float2*>(p));
            memcpy(&v, &t, 8);
        } else {
            double t = __ldcs(reinterpret_cast<const double*>(p));
            memcpy(&v, &t, 8);
        }
    } else {
        float t = __ldcs(reinterpret_cast<const float*>(p));
        memcpy(&v, &t, 4);
    }
    return v;
}
template <typename T, int V>
__device__ __forceinline__ void st_cs(T* p, const Vec<T, V>& v) {
    if constexpr (sizeof(T) * V == 16) {
        if constexpr (sizeof(T) == 4) {
            float4 t;
            memcpy(&t, &v, 16);
            __stcs(reinterpret_cast<float4*>(p), t);
        } else {
            double2 t;
            memcpy(&t, &v, 16);
            __stcs(reinterpret_cast<double2*>(p), t);
        }
    } else if constexpr (sizeof(T) * V == 8) {
        if constexpr (sizeof(T) == 4) {
            float2 t;
            memcpy(&t, &v, 8);
            __stcs(reinterpret_cast<float2*>(p), t);
        } else {
            double t;
            memcpy(&t, &v, 8);
            __stcs(reinterpret_cast<double*>(p), t);
        }
    } else {
        float t;
        memcpy(&t, &v, 4);
        __stcs(reinterpret_cast<float*>(p), t);
    }
}

}  // namespace vxq
