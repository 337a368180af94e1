// dense_tc.cu -- dense coupling field on the 5th-gen tensor cores with the integrator fused.
//
// For dense couplings with a uniform magnitude |J_ij| = c (e.g. Sherrington-Kirkpatrick,
// BASELINE config 2): J = c * K with K in {-1, 0, +1}.
//   PA  (parallel_annealing.py:42-45): F = K.s with s in {-1,+1}; K and s are exact in FP8
//       E4M3, the f32 TMEM accumulator holds the integer K.s exactly (|K.s| < 2^24), and
//       f = c * (K.s) carries a single rounding.                     (Kind::kFp8, 1 plane)
//   SBM (bifurcation.py:40-46), default: F = K.q exactly in integers.  q is taken in fixed
//       point, Q = rint(q * 2^S) (|Q| <= 2^22), written as three signed 8-bit digits
//       Q = d0 + 2^8 d1 + 2^16 d2; K (int8) . d_p accumulate into three S32 TMEM
//       accumulators (kind::i8, exact integer sums), combined in the epilogue as
//       F = fp32(a0 + 2^8 a1 + 2^16 a2) * 2^-S (one rounding).  The tensor cores' f32
//       accumulation of fractional fp16/bf16 products is not IEEE round-to-nearest and its
//       error grows with n (profiles/r02/field_probe.txt); the integer path has none, so the
//       result is bit-exact against a numpy emulation.            (Kind::kI8x3, 3 planes)
//       Fallbacks (VXQ_SBM_PLANES=2/3 or |q| beyond 2^14): q as two fp16 / three exact bf16
//       planes into one f32 accumulator (kind::f16).   (Kind::kF16x2 / Kind::kBf16x3)
//
//   F^T[i, r] = sum_j K[i, j] B[r, j]     M = n rows (i), N = replicas (r), K = n
//   A = K  [ld][ld] K-major                 (TMA, SWIZZLE_128B, 128 rows x 128 B boxes)
//   B = S or q-planes [planes][R][ld]       (TMA, SWIZZLE_128B, bn rows x 128 B x planes)
//   D in TMEM: 128 lanes (rows i) x bn f32 columns (replicas r), 2 accumulators
// Persistent warp-specialised CTA (1 per SM, 320 threads) running ALL T steps:
//   warp 0  TMA producer        STAGES-deep smem ring
//   warp 1  MMA issuer          one elected thread issues tcgen05.mma for the CTA
//   warps 2-9 epilogue          tcgen05.ld -> integrator update of the state in HBM ->
//                               next-step B operand (fp8 signs / bf16 q-splits)
// Tiles are enumerated (step t, replica block nb, row block mb) and dealt round-robin; a
// tile of step t only waits for the step-(t-1) tiles of its replica block (release/acquire
// counter + proxy fence before the TMA), so steps overlap with no per-step launch, prologue
// or wave quantisation.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "tc_ptx.cuh"
#include "vxq_internal.h"

namespace vxq {

constexpr int DBM = 128;   // rows (i) per tile
constexpr int DROW = 128;  // bytes per K-major smem row (one SWIZZLE_128B atom row)
constexpr int DA_BYTES = DBM * DROW;
constexpr int DTHREADS = 352;  // TMA warp, MMA warp, 8 epilogue warps, x/m loader warp
constexpr int RING_BYTES = 224 * 1024;  // operand stages + x/m staging slots
constexpr int XM_SLOT_BYTES = 2 * 16 * DBM * 4;  // x and m of 16 replicas x 128 rows (fp32)
constexpr int DSMEM = RING_BYTES + 1024 + 512;
constexpr int QN = 8;  // tile-ticket ring depth (dynamic tile queue, see k_dense_run)
#ifndef VXQ_I8_STAGES
#define VXQ_I8_STAGES 6  // operand ring depth of the exact SBM kernel (31 KB stages)
#endif
constexpr uint8_t FP8_P1 = 0x38, FP8_M1 = 0xB8;  // E4M3 +1 / -1

#ifndef VXQ_I8_MERGED
#define VXQ_I8_MERGED 1
#endif

enum class Kind : int { kFp8 = 0, kBf16x3 = 1, kF16x2 = 2, kJ16x2 = 3, kJQ16 = 4, kI8x3 = 5, kI8x4 = 6 };

template <Kind K>
struct KindTraits;
template <>
struct KindTraits<Kind::kFp8> {
    static constexpr int kPlanes = 1, kAPlanes = 1, kStages = 4, kBnMax = 256, kElemBytes = 1;
    static constexpr int kKPerMma = 32;  // fp8: K = 32 per tcgen05.mma (32 B)
    // D=F32, A=B=E4M3, K-major
    static constexpr uint32_t kIdescBase = (1u << 4);
};
template <>
struct KindTraits<Kind::kBf16x3> {
    static constexpr int kPlanes = 3, kAPlanes = 1, kStages = 3, kBnMax = 128, kElemBytes = 2;
    static constexpr int kKPerMma = 16;  // bf16: K = 16 per tcgen05.mma (32 B)
    // D=F32, A=B=BF16, K-major
    static constexpr uint32_t kIdescBase = (1u << 4) | (1u << 7) | (1u << 10);
};
// SBM default: q = h1 + h2 as two fp16 terms (11 + 11 significant bits, |q - h1 - h2| <=
// 2^-23 |q| + 2^-25): 2 MMAs per k-block instead of 3, 4 B of B operand per q instead of 6
template <>
struct KindTraits<Kind::kF16x2> {
    static constexpr int kPlanes = 2, kAPlanes = 1, kStages = 4, kBnMax = 128, kElemBytes = 2;
    static constexpr int kKPerMma = 16;  // f16: K = 16 per tcgen05.mma (32 B)
    // D=F32, A=B=F16 (format 0), K-major
    static constexpr uint32_t kIdescBase = (1u << 4);
};
// PA with general (non-uniform) dense J: J (scaled by 2^k) as two fp16 A planes
// J1 = fp16(J), J2 = fp16(J - J1) against the spins as fp16 +-1 (products exact, fp32
// accumulation): 2 MMAs per k-block, CTA pairs only
template <>
struct KindTraits<Kind::kJ16x2> {
    static constexpr int kPlanes = 1, kAPlanes = 2, kStages = 3, kBnMax = 128, kElemBytes = 2;
    static constexpr int kKPerMma = 16;
    static constexpr uint32_t kIdescBase = (1u << 4);
};
// SBM with general dense J: two fp16 J planes (A) x two fp16 q planes (B), 4 MMAs per k-block
template <>
struct KindTraits<Kind::kJQ16> {
    static constexpr int kPlanes = 2, kAPlanes = 2, kStages = 2, kBnMax = 128, kElemBytes = 2;
    static constexpr int kKPerMma = 16;
    static constexpr uint32_t kIdescBase = (1u << 4);
};

// SBM exact default: K int8 (A) x three int8 digit planes of the fixed-point q (B), one S32
// accumulator per plane (3 x bn <= 240 TMEM columns per buffer), CTA pairs only
template <>
struct KindTraits<Kind::kI8x3> {
    static constexpr int kPlanes = 3, kAPlanes = 1, kStages = 3, kBnMax = 80, kElemBytes = 1;
    static constexpr int kKPerMma = 32;  // i8: K = 32 per tcgen05.mma (32 B)
    // D=S32 (2), A=B=signed int8 (1), K-major
    static constexpr uint32_t kIdescBase = (2u << 4) | (1u << 7) | (1u << 10);
};

// the same with a 4th plane holding the spins s_t = sign(q_t) (+-1 int8): its accumulator is
// the exact K s_t, so the epilogue also reduces the exact coupling energy of s_t (per-step
// energy trace, time-to-target); 4 x bn <= 256 TMEM columns per buffer
template <>
struct KindTraits<Kind::kI8x4> {
    static constexpr int kPlanes = 4, kAPlanes = 1, kStages = 3, kBnMax = 64, kElemBytes = 1;
    static constexpr int kKPerMma = 32;
    static constexpr uint32_t kIdescBase = (2u << 4) | (1u << 7) | (1u << 10);
};
constexpr bool is_i8(Kind k) { return k == Kind::kI8x3 || k == Kind::kI8x4; }

template <Kind K>
constexpr int stage_bytes() {
    return DA_BYTES * KindTraits<K>::kAPlanes + KindTraits<K>::kPlanes * KindTraits<K>::kBnMax * DROW;
}
static_assert(4 * stage_bytes<Kind::kFp8>() <= 192 * 1024, "fp8 ring");
static_assert(3 * stage_bytes<Kind::kBf16x3>() <= 192 * 1024, "bf16 ring");
static_assert(4 * stage_bytes<Kind::kF16x2>() <= 192 * 1024, "f16 ring");

struct DenseOperand {
    int64_t n = 0, ld = 0;      // ld = n_pad (multiple of 128)
    float scale = 0.f;          // c (fp32)
    uint8_t* K8 = nullptr;      // [ld][ld] fp8 E4M3 in {-1, 0, +1}, or (fp4) packed E2M1
                                //   nibbles [ld][ld/2] (element 2k in the low nibble)
    uint32_t afmt = 0;          // A format in the f8f6f4 instruction descriptor (0 E4M3, 5 E2M1)
    __nv_bfloat16* K16 = nullptr;  // [ld][ld] bf16 in {-1, 0, +1} (SBM bf16x3, built lazily)
    __half* K16h = nullptr;        // [ld][ld] fp16 in {-1, 0, +1} (SBM f16x2, built lazily)
    __half* J16 = nullptr;         // [2][ld][ld] fp16 planes of 2^e J (general dense J)
    int8_t* Ki8 = nullptr;         // [ld][ld] int8 in {-1, 0, +1} (SBM exact path, lazily)
    float jscale_inv = 0.f;        // 2^-e
    CUtensorMap tmJ;
    CUtensorMap tmA8, tmA16, tmA16h, tmAi8;
    ~DenseOperand() {
        if (K8) cudaFreeAsync(K8, 0);  // back to the retained pool
        if (K16) cudaFreeAsync(K16, 0);
        if (K16h) cudaFreeAsync(K16h, 0);
        if (J16) cudaFreeAsync(J16, 0);
        if (Ki8) cudaFreeAsync(Ki8, 0);
    }
};

void dense_destroy(DenseOperand* d) { delete d; }

namespace {
__global__ void k_any_nonzero_h(int64_t n, const double* v, int* flag);
}

bool problem_h_zero(Problem* p, cudaStream_t s) {
    std::lock_guard<std::mutex> g(p->mu);
    if (p->h_zero < 0) {
        DevBuf<int> f(1, s);
        VXQ_CUDA(cudaMemsetAsync(f.get(), 0, sizeof(int), s));
        k_any_nonzero_h<<<(unsigned)std::max<int64_t>(1, ceil_div(p->n, 256)), 256, 0, s>>>(
            p->n, p->h64, f.get());
        VXQ_CHECK_LAUNCH();
        int v = 0;
        VXQ_CUDA(cudaMemcpyAsync(&v, f.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
        VXQ_CUDA(cudaStreamSynchronize(s));
        p->h_zero = v ? 0 : 1;
    }
    return p->h_zero == 1;
}

namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) throw Error(VXQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// L2 promotion of the TMA boxes (VXQ_TMA_PROMO: 0 none, 1 64 B, 2 128 B, 3 256 B).  The
// boxes' rows are 128-byte segments of L2-resident operands: 128 B beats the round-1 256 B
// by ~1 % on cfg2 PA and SBM (profiles/r02/ab_promo/)
CUtensorMapL2promotion tma_promotion() {
    static const CUtensorMapL2promotion v = [] {
        int k = 2;
        if (const char* e = getenv("VXQ_TMA_PROMO")) k = atoi(e);
        switch (k) {
            case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
            case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
            case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
            default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
        }
    }();
    return v;
}

// up to 3-D tensor [planes][outer][inner] (elements of `esize` bytes), SW128 boxes
CUtensorMap make_map(const void* base, CUtensorMapDataType dt, int esize, uint64_t inner,
                     uint64_t outer, uint64_t planes, uint32_t box_inner, uint32_t box_outer,
                     uint32_t box_planes,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    CUtensorMap m;
    const cuuint32_t rank = planes > 1 ? 3 : 2;
    cuuint64_t dims[3] = {inner, outer, planes};
    cuuint64_t strides[2] = {inner * esize, inner * outer * esize};
    cuuint32_t box[3] = {box_inner, box_outer, box_planes};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = get_encode()(&m, dt, rank, const_cast<void*>(base), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                              tma_promotion(),
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(VXQ_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

// K as packed E2M1 nibbles [rows][inner/2] bytes; TMA (16U4_ALIGN16B) unpacks each 16
// nibbles into a 16-byte slot of shared memory -- the padded fp4 operand layout of
// tcgen05.mma kind::f8f6f4 -- so tiles, descriptors and the MMA loop are those of fp8.
CUtensorMap make_map_fp4(const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                         uint32_t box_outer) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner / 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 2,
                              const_cast<void*>(base), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              tma_promotion(),
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(VXQ_ERR_CUDA, "cuTensorMapEncodeTiled (fp4) failed");
    return m;
}

constexpr uint32_t FP4_P1 = 0x2, FP4_M1 = 0xA;  // E2M1 +1 / -1

__global__ void k_build_sign_matrix(int64_t n, int64_t ld, const int64_t* __restrict__ indptr,
                                    const int32_t* __restrict__ indices,
                                    const double* __restrict__ data, uint8_t* __restrict__ K8,
                                    __nv_bfloat16* __restrict__ K16, uint32_t* __restrict__ K4,
                                    __half* __restrict__ K16h, int8_t* __restrict__ Ki8) {
    int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    for (int64_t k = indptr[row] + lane; k < indptr[row + 1]; k += 32) {
        const bool pos = data[k] > 0;
        if (K8) K8[row * ld + indices[k]] = pos ? FP8_P1 : FP8_M1;
        if (K16) K16[row * ld + indices[k]] = __float2bfloat16_rn(pos ? 1.f : -1.f);
        if (K16h) K16h[row * ld + indices[k]] = __float2half_rn(pos ? 1.f : -1.f);
        if (Ki8) Ki8[row * ld + indices[k]] = pos ? (int8_t)1 : (int8_t)-1;
        if (K4) {  // neighbours share bytes: OR the nibble into its 32-bit word
            const int64_t e = row * ld + indices[k];
            atomicOr(K4 + (e >> 3), (pos ? FP4_P1 : FP4_M1) << (4 * (e & 7)));
        }
    }
}

// general dense J: 2^e J split into two fp16 planes (P[0] = fp16(v), P[1] = fp16(v - P[0]))
__global__ void k_build_j_planes(int64_t n, int64_t ld, const int64_t* __restrict__ indptr,
                                 const int32_t* __restrict__ indices,
                                 const float* __restrict__ data32, float scale,
                                 __half* __restrict__ P) {
    int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    for (int64_t k = indptr[row] + lane; k < indptr[row + 1]; k += 32) {
        const float v = data32[k] * scale;  // power of two: exact
        const __half h1 = __float2half_rn(v);
        const __half h2 = __float2half_rn(__fsub_rn(v, __half2float(h1)));
        P[row * ld + indices[k]] = h1;
        P[ld * ld + row * ld + indices[k]] = h2;
    }
}

__device__ __forceinline__ int64_t pos_interleaved(int64_t r, int V) {
    int64_t ch = 32 * V;
    int64_t c = r / ch, rem = r % ch;
    return c * ch + (rem % 32) * V + rem / 32;
}

// exact 3-way bf16 split of an fp32 value: v == q1 + q2 + q3
__device__ __forceinline__ void split3(float v, __nv_bfloat16& q1, __nv_bfloat16& q2,
                                       __nv_bfloat16& q3) {
    q1 = __float2bfloat16_rn(v);
    const float r1 = __fsub_rn(v, __bfloat162float(q1));
    q2 = __float2bfloat16_rn(r1);
    const float r2 = __fsub_rn(r1, __bfloat162float(q2));
    q3 = __float2bfloat16_rn(r2);
}

// fixed-point digits of q for the exact SBM field: Q = rint(q * 2^S) (|Q| <= 2^22 by the
// choice of S), Q = d0 + 2^8 d1 + 2^16 d2 with balanced signed digits d_p in [-128, 127]
__device__ __forceinline__ void digits3(float q, float qscale, int8_t& d0, int8_t& d1,
                                        int8_t& d2) {
    const int Q = __float2int_rn(q * qscale);  // power-of-two scaling: exact, then rint
    const int e0 = ((Q + 128) & 255) - 128;
    const int r1 = (Q - e0) >> 8;
    const int e1 = ((r1 + 128) & 255) - 128;
    d0 = (int8_t)e0;
    d1 = (int8_t)e1;
    d2 = (int8_t)((r1 - e1) >> 8);
}

// 2-way fp16 split: v ~= h1 + h2 (h1 = fp16(v), h2 = fp16(v - h1); v - h1 is exact in fp32)
__device__ __forceinline__ void split2(float v, __half& h1, __half& h2) {
    h1 = __float2half_rn(v);
    h2 = __float2half_rn(__fsub_rn(v, __half2float(h1)));
}

// x0 ~ uniform(-1, 1) from replica stream r (same draws as k_init_pa), row-major [R][ld]
__global__ void k_init_pa_rm(int64_t n, int64_t R, int64_t ld, uint64_t seed, int64_t rbegin,
                             float* __restrict__ x, float* __restrict__ m,
                             uint8_t* __restrict__ s, int s_fmt) {  // 0 fp8, 1 fp4, 2 fp16
    const bool s_fp4 = s_fmt == 1;
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t nq = (n + 3) / 4;
    if (idx >= nq * R) return;
    int64_t r = idx / nq, q = idx % nq;
    U64x4 o = philox4x64_10((uint64_t)q + 1, 0, (uint64_t)(rbegin + r), 0, seed, 0);
    uint32_t code[4] = {0, 0, 0, 0};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        int64_t i = 4 * q + w;
        if (i < n) {
            float v = (float)uniform_from_raw(o.v[w], -1.0, 2.0);
            x[r * ld + i] = v;
            m[r * ld + i] = 0.f;
            if (s_fp4) code[w] = v >= 0.f ? FP4_P1 : FP4_M1;
            else if (s_fmt == 2)
                reinterpret_cast<uint16_t*>(s)[r * ld + i] = v >= 0.f ? 0x3C00 : 0xBC00;
            else s[r * ld + i] = v >= 0.f ? FP8_P1 : FP8_M1;
        }
    }
    if (s_fp4) {  // 4 spins = 2 packed bytes (element 2k in the low nibble)
        const int64_t e = (r * ld + 4 * q) >> 1;
        s[e] = (uint8_t)(code[0] | (code[1] << 4));
        s[e + 1] = (uint8_t)(code[2] | (code[3] << 4));
    }
}

// q0, p0 (stream r: n q-draws then n p-draws, as k_init_sbm) + the bf16 q-splits
__global__ void k_init_sbm_rm(int64_t n, int64_t R, int64_t ld, uint64_t seed, int64_t rbegin,
                              double amp, float* __restrict__ q, float* __restrict__ p,
                              void* __restrict__ planes_raw, int nplanes, float qscale,
                              int spin_plane) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t nq = (2 * n + 3) / 4;
    if (idx >= nq * R) return;
    int64_t r = idx / nq, qd = idx % nq;
    U64x4 o = philox4x64_10((uint64_t)qd + 1, 0, (uint64_t)(rbegin + r), 0, seed, 0);
    const double lo = -amp, range = __dadd_rn(amp, amp);
    const int64_t plane = R * ld;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        int64_t k = 4 * qd + w;
        float v = (float)uniform_from_raw(o.v[w], lo, range);
        if (k < n) {
            q[r * ld + k] = v;
            if (qscale > 0.f) {  // exact path: int8 digit planes
                int8_t* planes = reinterpret_cast<int8_t*>(planes_raw);
                int8_t a, b, c;
                digits3(v, qscale, a, b, c);
                planes[r * ld + k] = a;
                planes[plane + r * ld + k] = b;
                planes[2 * plane + r * ld + k] = c;
                if (spin_plane) planes[3 * plane + r * ld + k] = v >= 0.f ? 1 : -1;
            } else if (nplanes == 3) {
                __nv_bfloat16* planes = reinterpret_cast<__nv_bfloat16*>(planes_raw);
                __nv_bfloat16 a, b, c;
                split3(v, a, b, c);
                planes[r * ld + k] = a;
                planes[plane + r * ld + k] = b;
                planes[2 * plane + r * ld + k] = c;
            } else {
                __half* planes = reinterpret_cast<__half*>(planes_raw);
                __half a, b;
                split2(v, a, b);
                planes[r * ld + k] = a;
                planes[plane + r * ld + k] = b;
            }
        } else if (k < 2 * n) {
            p[r * ld + (k - n)] = v;
        }
    }
}

__global__ void k_rm_to_interleaved(const float* __restrict__ src, int64_t n, int64_t R,
                                    int64_t ld, int64_t R_pad, int V, float* __restrict__ dst) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * R) return;
    int64_t r = idx / n, i = idx % n;
    dst[i * R_pad + pos_interleaved(r, V)] = src[r * ld + i];
}

__global__ void k_pack_bits_rm(const float* __restrict__ x, int64_t n, int64_t R, int64_t ld,
                               int64_t W, uint32_t* __restrict__ sb) {
    int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (gw >= n * W) return;
    int64_t w = gw / n, i = gw % n;
    int64_t r = w * 32 + lane;
    bool up = r < R ? (x[r * ld + i] >= 0.f) : true;
    uint32_t word = __ballot_sync(0xffffffffu, up);
    if (lane == 0) sb[i * W + w] = word;
}

__global__ void k_any_nonzero_h(int64_t n, const double* v, int* flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && v[i] != 0.0) *flag = 1;
}

// fused tracking, after the loop: decide s_{T-1} (still in its B buffer, energy q_{T-1}) and
// s_T = sign(x_T) (energy from the final energy pass), strictly-better-wins in step order
__global__ void k_track_finalize(int64_t n, int64_t R, int64_t ld, const long long* qlast,
                                 const long long* qT, const long long* bestq,
                                 const uint8_t* sprev, int fp4, const float* x,
                                 int8_t* best_s) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * R) return;
    const int64_t r = idx / n, i = idx % n, off = r * ld + i;
    long long b = bestq[r];
    int8_t v = best_s[off];
    if (qlast[r] < b) {
        b = qlast[r];
        if (fp4) {
            const uint8_t by = sprev[off >> 1];
            v = (((i & 1) ? (by >> 4) : by) & 0x8) ? -1 : 1;
        } else {
            v = (sprev[off] & 0x80) ? -1 : 1;
        }
    }
    if (qT[r] < b) v = x[off] >= 0.f ? 1 : -1;
    best_s[off] = v;
}

__global__ void k_pack_bits_i8(const int8_t* __restrict__ s, int64_t n, int64_t R, int64_t ld,
                               int64_t W, uint32_t* __restrict__ sb) {
    int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (gw >= n * W) return;
    int64_t w = gw / n, i = gw % n;
    int64_t r = w * 32 + lane;
    bool up = r < R ? (s[r * ld + i] > 0) : true;
    uint32_t word = __ballot_sync(0xffffffffu, up);
    if (lane == 0) sb[i * W + w] = word;
}

__global__ void k_signs_fp8_rm(const float* __restrict__ x, int64_t n, int64_t R, int64_t ld,
                               uint8_t* __restrict__ s) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * R) return;
    int64_t r = idx / n, i = idx % n;
    s[r * ld + i] = x[r * ld + i] >= 0.f ? FP8_P1 : FP8_M1;
}

struct DenseRunArgs {
    int n, R, ld, kblocks, m_tiles, n_tiles, bn;
    int T;                   // dynamics steps covered by this launch
    float scale;             // c
    float eta, alpha;        // PA
    float dt, a0, c0, dta0, q_cap;  // SBM
    const float* sched;      // [T] lambda_t (PA) / a_t (SBM), fp32
    const float* h;          // PA: h;  SBM: g = -h
    float* x;                // PA: x;  SBM: q
    float* m;                // PA: m;  SBM: p
    uint8_t* b_buf[2];       // B operand of step t lives in b_buf[t & 1]
    int64_t plane_elems;     // elements per q-plane (R * ld) for kBf16x3
    int mode;                // 0: dynamics steps, 1: energy pass over b_buf[0] (q2), 2: no-op
    long long* q2;           // [R] 2 * sum_{i<j} K_ij s_i s_j  (mode 1)
    long long* qtrace;       // [T][R] same for the spins s_t entering step t (optional)
    unsigned* done;          // [T][n_tiles] finished row-tiles per (step, replica block)
    int group;               // replica blocks interleaved per row block (A-panel reuse)
    unsigned long long* stats;  // optional [8] wait-cycle counters (VXQ_DENSE_STATS=1)
    uint32_t idesc_extra;    // OR-ed into the instruction descriptor (A operand format)
    uint32_t a_tx_bytes;     // transaction bytes of one A box (packed fp4 counts global bytes)
    int b_fp4;               // B operand (spins) as packed E2M1 nibbles
    int xm;                  // PA steps: x/m staged by the loader warp (TMA) into smem
    uint32_t b_tx_bytes;     // transaction bytes of one B box (per plane) as delivered
    uint64_t timeout_ns;     // bound on every in-kernel wait (VXQ_WAIT_TIMEOUT_S, default 10)
    // fused best-state tracking (improvement mode; needs qtrace, h = 0):
    long long* bestq;        // [R] lowest 2 sum K s s of s_0..s_{t-2} (LLONG_MAX initially)
    int8_t* best_s;          // [R][ld] best spins so far
    unsigned* decided;       // [T][n_tiles] tiles that made their step-(t-1) decisions
    unsigned* ticket;        // [1] next tile of the dynamic queue (zeroed per launch)
    float qscale, qscale_inv;  // kI8x3: 2^S and 2^-S of the fixed-point q
    int a_prefetch;            // L2-prefetch the A panel ahead of the smem loads
};

// stats slots: 0 producer<-empty, 1 producer<-dependency, 2 mma<-full, 3 mma<-tempty,
//              4 epilogue<-tfull, 5 epilogue busy, 6 tiles, 7 kernel cycles (max CTA)
__device__ __forceinline__ long long clk() {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    return c;
}

// Tile g -> (step t, replica block nb, row block mb).  Within a step, replica blocks are
// processed in groups of `group`: the group's tiles for one row block are adjacent, so they
// run concurrently and share the A panel (J rows) through L2, while earlier groups still
// complete early enough for the next step to start on them.
__device__ __forceinline__ void decode_tile(const DenseRunArgs& a, int g, int tps, int mrows,
                                            int& t, int& nb, int& mb) {
    t = g / tps;
    const int rem = g % tps;
    const int per_group = mrows * a.group;
    const int grp = rem / per_group, w = rem % per_group;
    // the last group may be smaller (n_tiles not a multiple of group)
    const int nt = tps / mrows;
    const int gsz = min(a.group, nt - grp * a.group);
    mb = w / gsz;
    nb = grp * a.group + w % gsz;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// CL = CTAs per cluster along the row dimension: the CL CTAs of a cluster process row
// blocks mb = CL*p + rank of the same (step, replica block) and each TMA-multicasts 1/CL of
// the shared B tile into all of them, cutting L2->SM traffic for B by CL.
//
// PAIR: the two CTAs of a cluster form a tcgen05 CTA pair (cta_group::2): tile = 256 rows
// (128 per CTA, each CTA's TMEM holds its rows x all bn replicas) x bn replicas, each CTA
// loads its A rows and HALF of B into its own smem (mxf4: 31 KB stages, 6 deep), only the leader
// (rank 0) issues the M = 256 MMAs and its commits arrive in both CTAs.
//
// PAIR && CL == 2 ("super-pair", PA mxf4 only): a 4-CTA cluster of two tcgen05 pairs that
// work on the SAME row block and two replica blocks (nb = 2 nbp + pair): pair 0's CTAs load
// the K panel once and TMA-multicast each 128-row half into the matching CTA of both pairs,
// so K crosses L2->SM once per two tiles.  Each pair keeps its own TMEM, MMAs and epilogue;
// a stage is refilled only after both pairs' MMAs released it (commits multicast to all 4
// CTAs, empty count 2).  Needs an even number of replica blocks.
//
// a.xm (PA steps): a loader warp TMA-loads each tile's x/m in 16-replica chunks into XMS
// shared-memory slots ahead of the epilogue (after acquiring the step-(t-1) counter), so the
// epilogue's inputs are in flight without occupying registers.
//
// MX: kind::mxf4 (block-scaled E2M1, twice the f8f6f4 rate) with K and the spins packed two
// per byte in smem too (a 128-byte smem row = 256 K elements: half the operand bytes per
// flop); the scale factors are all 1 (UE8M0 0x7F), written once into TMEM columns
// kSfCol..511, and the two accumulators sit at columns 0 / kAccMx (bn <= 240).
constexpr uint32_t kAccMx = 240, kSfCol = 480;
#ifndef VXQ_PAIR_STAGES
#define VXQ_PAIR_STAGES 5  // 5 x 32 KB operand stages + 4 x/m slots in 224 KB
#endif
#if VXQ_PAIR_STAGES > 5
#error "VXQ_PAIR_STAGES > 5: 32 KB stages leave too few x/m slots (mxf4: VXQ_MX_STAGES)"
#endif
#ifndef VXQ_MX_TIGHT
#define VXQ_MX_TIGHT 1  // mxf4 pair stages packed to A + bn_max/2 B rows (31 KB)
#endif
#ifndef VXQ_MX_STAGES
#define VXQ_MX_STAGES 6  // 6 x 31 KB + 2 x/m slots: cfg2 150.1 -> 153.2 Grv/s (profiles/r02/ab_stages)
#endif

template <Kind KD, int CL, bool PAIR = false, bool MX = false>
__global__ void __launch_bounds__(DTHREADS, 1)
    k_dense_run(const __grid_constant__ CUtensorMap tmA,
                const __grid_constant__ CUtensorMap tmB0,
                const __grid_constant__ CUtensorMap tmB1,
                const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmM, DenseRunArgs a) {
    using TR = KindTraits<KD>;
    static_assert(!PAIR || (KD != Kind::kBf16x3 && (CL == 1 || (CL == 2 && MX))),
                  "pair MMA: f8f6f4 / f16x2, no B multicast; super-pairs: mxf4 only");
    constexpr bool SP = PAIR && CL == 2;  // two pairs sharing the K panel
    static_assert(!is_i8(KD) || PAIR, "int8 digit planes: CTA pairs only");
    static_assert((KD != Kind::kJ16x2 && KD != Kind::kJQ16) || PAIR,
                  "general-J planes: CTA pairs only");
    constexpr int A_BYTES = DA_BYTES * TR::kAPlanes;  // A planes of one stage, back to back
    static_assert(!MX || (KD == Kind::kFp8 && (CL == 1 || PAIR)),
                  "mxf4: fp8-kind layout, no B multicast");
    constexpr uint32_t ACC_COLS = MX ? kAccMx : 256;
    constexpr int NCTA = PAIR ? 2 * CL : CL;
    constexpr int RPC = PAIR ? 2 : CL;  // CTAs splitting a tile's rows
    // pair: each CTA stages its 128 A rows and <= 128 B rows per plane
    // kI8x3: each CTA stages <= kBnMax/2 = 40 replicas per digit plane, so a stage packs
    // into 31 KB and the ring holds VXQ_I8_STAGES of them (no x/m slots: SBM)
    constexpr int SBYTES_I8 = ((A_BYTES + TR::kPlanes * (TR::kBnMax / 2) * DROW + 1023) / 1024) * 1024;
    constexpr int STAGES =
        is_i8(KD) ? VXQ_I8_STAGES
        : (MX && PAIR && VXQ_MX_TIGHT) ? VXQ_MX_STAGES
        : PAIR ? ((TR::kPlanes == 1 && TR::kAPlanes == 1) ? VXQ_PAIR_STAGES
                                                          : (TR::kPlanes * TR::kAPlanes > 2 ? 3 : 4))
               : TR::kStages;
    constexpr int SBYTES_MX = ((A_BYTES + (kAccMx / 2) * DROW + 1023) / 1024) * 1024;
    constexpr int SBYTES = is_i8(KD) ? SBYTES_I8
                           : (MX && PAIR && VXQ_MX_TIGHT) ? SBYTES_MX
                           : PAIR ? A_BYTES + TR::kPlanes * 128 * DROW : stage_bytes<KD>();
    constexpr int XMS = (RING_BYTES - STAGES * SBYTES) / XM_SLOT_BYTES;  // x/m slots
    static_assert(STAGES * SBYTES <= RING_BYTES, "smem ring");
    // x/m staging needs two slots (one per epilogue half); a ring too deep to leave them
    // runs the register x/m path (xm_on false)
    const bool xm_on = XMS >= 2 && a.xm != 0;
    // x/m slots are split between the two epilogue halves (chunk c goes to half c & 1) so
    // each half waits on every phase of its own slots in order: with shared slots a half
    // could wait on a slot two phases ahead of the loader and pass the parity check on a
    // stale phase (the ABA of mbarrier parity waits)
    constexpr int XHS = XMS / 2 > 0 ? XMS / 2 : 1;
    constexpr bool PA_KIND = KD == Kind::kFp8 || KD == Kind::kJ16x2;
    extern __shared__ uint8_t smem_raw[];
    __shared__ int s_last;  // fused tracking: this tile completed its step's decisions
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + RING_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* xfull = tempty + 2;                                    // [XMS]
    uint64_t* xempty = xfull + (XMS > 0 ? XMS : 1);                  // [XMS]
    uint64_t* qfull = xempty + (XMS > 0 ? XMS : 1);                  // [QN] ticket ring
    uint64_t* qempty = qfull + QN;                                   // [QN] (leader's used)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qempty + QN);
    int* tq = reinterpret_cast<int*>(tmem_slot + 1);                 // [QN] tile tickets
    uint8_t* xm_smem = smem + STAGES * SBYTES;                       // XMS x XM_SLOT_BYTES

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long t_start = clk();
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(full + s, 1);
            // released by the MMA of every CTA in the cluster (pair: the leader's only)
            ptx::mbar_init(empty + s, SP ? 2 : (PAIR ? 1 : CL));
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(tfull + s, 1);
            ptx::mbar_init(tempty + s, PAIR ? 512 : 256);  // pair: both CTAs' epilogues
        }
        for (int s = 0; s < XMS; ++s) {
            ptx::mbar_init(xfull + s, 1);
            ptx::mbar_init(xempty + s, 4);  // the 4 epilogue warps of one half
        }
        // ticket consumers (all arrive on the leader's qempty): per CTA 8 epilogue warps
        // and the x/m loader (PA with staging), the MMA issuer(s) (pair: the leader's
        // only), and every non-leader producer
        const uint32_t xmc = (xm_on && a.mode == 0) ? 1u : 0u;
        const uint32_t qcons =
            NCTA * (8u + xmc) + (PAIR ? (uint32_t)CL : (uint32_t)NCTA) + (NCTA - 1u);
        for (int s = 0; s < QN; ++s) {
            ptx::mbar_init(qfull + s, 1);
            ptx::mbar_init(qempty + s, qcons);
        }
        ptx::fence_mbar_init();
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB0);
        ptx::tma_prefetch(&tmB1);
        if (a.xm) {
            ptx::tma_prefetch(&tmX);
            ptx::tma_prefetch(&tmM);
        }
    }
    if (warp == 1) {
        if constexpr (PAIR) ptx::tmem_alloc2<512>(tmem_slot);
        else ptx::tmem_alloc<512>(tmem_slot);
    }
    ptx::tc_fence_before();
    if constexpr (NCTA > 1) ptx::cluster_sync();  // peers' barriers initialised before use
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if constexpr (MX) {  // unit scale factors (UE8M0 0x7F) for every row / column block
        if (warp >= 2 && warp < 6)
            ptx::tmem_fill_32x32b_x32(tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + kSfCol,
                                      0x7F7F7F7Fu);
        ptx::tc_fence_before();
        if constexpr (NCTA > 1) ptx::cluster_sync();
        else __syncthreads();
        ptx::tc_fence_after();
    }
    const int crank = NCTA > 1 ? (int)ptx::cluster_ctarank() : 0;
    const int lr = PAIR ? (crank & 1) : crank;  // rank within the tile's row-splitting CTAs
    const int pr = SP ? (crank >> 1) : 0;       // super-pair: which pair (replica block)
    // Dynamic tile queue: the leader CTA's TMA thread takes tile tickets in increasing
    // order (atomicAdd on a.ticket) and hands each to every role of every CTA of its
    // cluster through a QN-deep smem ring.  A tile only ever waits on tiles of the previous
    // step -- lower tickets, already taken by running clusters -- so the schedule makes
    // progress however many clusters are resident: no cooperative launch is needed.
    auto next_ticket = [&](int k) -> int {  // consumers: ticket k (all lanes may call)
        if constexpr (NCTA > 1) ptx::mbar_wait_cluster(qfull + (k % QN), (k / QN) & 1, a.timeout_ns);
        else ptx::mbar_wait(qfull + (k % QN), (uint32_t)(k / QN) & 1u, a.timeout_ns);
        return *reinterpret_cast<volatile int*>(tq + (k % QN));
    };
    auto release_ticket = [&](int k) {  // one arrival per consumer unit
        if constexpr (NCTA > 1) ptx::mbar_arrive_cluster(ptx::cluster_addr(qempty + (k % QN), 0));
        else ptx::mbar_arrive(qempty + (k % QN));
    };
    const int mrows = (a.m_tiles + RPC - 1) / RPC;                   // row-block groups per step
    const int tps = mrows * (SP ? a.n_tiles / 2 : a.n_tiles);        // work items per step
    // ticket -> (step, this pair's replica block, this CTA's row block)
    auto tile_of = [&](int g, int& t, int& nb, int& mb) {
        decode_tile(a, g, tps, mrows, t, nb, mb);
        mb = mb * RPC + lr;
        if constexpr (SP) nb = 2 * nb + pr;
    };
    const int num_tiles = tps * a.T;
    // B bytes per stage in this CTA's smem (pair: half of the bn replicas)
    const uint32_t b_plane_bytes = (uint32_t)(PAIR ? a.bn / 2 : a.bn) * DROW;
    constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);

    if (warp == 0) {
        // ---------------- TMA producer
        if (ptx::elect_one()) {
            const uint64_t keep = ptx::policy_evict_last();  // K and B stay in L2
            long long st_empty = 0, st_dep = 0;
            int stage = 0;
            uint32_t ph = 0;
            for (int k = 0;; ++k) {
                int g;
                if (crank == 0) {  // take the next tile and hand it to the cluster
                    g = (int)atomicAdd(a.ticket, 1u);
                    if (g >= num_tiles) g = -1;
                    const int qs = k % QN;
                    ptx::mbar_wait(qempty + qs, ((uint32_t)(k / QN) & 1u) ^ 1u, a.timeout_ns);
                    if constexpr (NCTA > 1) {
                        for (int r = 0; r < NCTA; ++r) {
                            ptx::st_cluster_s32(ptx::cluster_addr(tq + qs, (uint32_t)r), g);
                            ptx::mbar_arrive_cluster(ptx::cluster_addr(qfull + qs, (uint32_t)r));
                        }
                    } else {
                        tq[qs] = g;
                        ptx::mbar_arrive(qfull + qs);
                    }
                } else {
                    g = next_ticket(k);
                    release_ticket(k);
                }
                if (g < 0) break;
                int t, nb, mb;
                tile_of(g, t, nb, mb);
                const CUtensorMap* tmB = (t & 1) ? &tmB1 : &tmB0;
                // A (the coupling panel) never depends on the dynamics: keep kPrefetch
                // k-blocks of it on their way into L2 ahead of the smem loads (a.a_prefetch;
                // an L2-resident K gains nothing from it and the prefetches cost L2 lookups)
                constexpr int kPrefetch = 8;
                for (int kb = 0; a.a_prefetch && kb < kPrefetch && kb < a.kblocks; ++kb) {
                    if constexpr (TR::kAPlanes > 1)
                        ptx::tma_prefetch_3d(&tmA, kb * (DROW / TR::kElemBytes), mb * DBM, 0);
                    else
                        ptx::tma_prefetch_2d(&tmA, kb * (DROW / TR::kElemBytes), mb * DBM);
                }
                for (int kb = 0; kb < a.kblocks; ++kb) {
                    if (a.a_prefetch && kb + kPrefetch < a.kblocks) {
                        if constexpr (TR::kAPlanes > 1)
                            ptx::tma_prefetch_3d(&tmA, (kb + kPrefetch) * (DROW / TR::kElemBytes),
                                                 mb * DBM, 0);
                        else
                            ptx::tma_prefetch_2d(&tmA, (kb + kPrefetch) * (DROW / TR::kElemBytes),
                                                 mb * DBM);
                    }
                    long long c0 = a.stats ? clk() : 0;
                    ptx::mbar_wait(empty + stage, ph ^ 1, a.timeout_ns);
                    if (a.stats) st_empty += clk() - c0;
                    uint8_t* sa = smem + stage * SBYTES;
                    const uint32_t tx = a.a_tx_bytes + TR::kPlanes * a.b_tx_bytes;
                    const int kcol = kb * (DROW / TR::kElemBytes);
                    if constexpr (SP) {
                        // pair 0 loads the K half of this CTA's rows once, multicast into
                        // the same CTA of both pairs (each pair leader's barrier counts its
                        // two CTAs' bytes, as for a single pair)
                        if (lr == 0) ptx::mbar_arrive_expect_tx(full + stage, 2 * tx);
                        if (pr == 0)
                            ptx::tma_load_2d_2sm_mc(sa, &tmA, full + stage, kcol, mb * DBM,
                                                    (uint16_t)((1u << lr) | (4u << lr)), keep);
                    } else if constexpr (PAIR) {
                        // the leader's barrier counts both CTAs' bytes; each CTA's loads land
                        // in its own smem and complete on the leader's barrier
                        if (crank == 0) ptx::mbar_arrive_expect_tx(full + stage, 2 * tx);
                        if constexpr (TR::kAPlanes > 1)
                            ptx::tma_load_3d_2sm(sa, &tmA, full + stage, kcol, mb * DBM, 0, keep);
                        else
                            ptx::tma_load_2d_2sm(sa, &tmA, full + stage, kcol, mb * DBM, keep);
                    } else {
                        ptx::mbar_arrive_expect_tx(full + stage, tx);
                        ptx::tma_load_2d_hint(sa, &tmA, full + stage, kcol, mb * DBM, keep);
                    }
                    if (kb == 0 && t > 0) {
                        const long long c1 = a.stats ? clk() : 0;
                        // B_t[nb] complete? (release/acquire on the step t-1 counter, then a
                        // proxy fence so the async-proxy TMA sees the generic-proxy stores)
                        const unsigned* cnt = a.done + (size_t)(t - 1) * a.n_tiles + nb;
                        if (ld_acquire_gpu(cnt) < (unsigned)a.m_tiles) {
                            uint64_t t0, tn;
                            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                            while (ld_acquire_gpu(cnt) < (unsigned)a.m_tiles) {
                                __nanosleep(64);
                                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                                if (tn - t0 > a.timeout_ns) __trap();
                            }
                        }
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        if (a.stats) st_dep += clk() - c1;
                    }
                    if constexpr (PAIR && TR::kPlanes > 1) {
                        ptx::tma_load_3d_2sm(sa + A_BYTES, tmB, full + stage, kcol,
                                             nb * a.bn + lr * (a.bn / 2), 0, keep);
                    } else if constexpr (PAIR) {
                        ptx::tma_load_2d_2sm(sa + A_BYTES, tmB, full + stage, kcol,
                                             nb * a.bn + lr * (a.bn / 2), keep);
                    } else if constexpr (CL > 1) {
                        static_assert(TR::kPlanes == 1, "B multicast: single-plane B only");
                        const int hrows = a.bn / CL;
                        ptx::tma_load_2d_mc(sa + DA_BYTES + crank * hrows * DROW, tmB,
                                            full + stage, kcol, nb * a.bn + crank * hrows, kMask,
                                            keep);
                    } else if constexpr (TR::kPlanes == 1) {
                        ptx::tma_load_2d_hint(sa + DA_BYTES, tmB, full + stage, kcol,
                                              nb * a.bn, keep);
                    } else {
                        ptx::tma_load_3d_hint(sa + A_BYTES, tmB, full + stage, kcol,
                                              nb * a.bn, 0, keep);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        ph ^= 1;
                    }
                }
            }
            if (a.stats) {
                atomicAdd(a.stats + 0, (unsigned long long)st_empty);
                atomicAdd(a.stats + 1, (unsigned long long)st_dep);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (single thread issues for the CTA / the pair's leader)
        if (PAIR && lr != 0) goto mma_done;
        {
        // mxf4 (block-scaled descriptor): E2M1 = 1 for A and B, UE8M0 scales (bit 23),
        // K = 64 per MMA, scale-factor ids 0; no accumulator-format field
        // int8 digit planes (VXQ_I8_MERGED): one MMA of N = planes x bn covers all planes --
        // their B rows sit back to back in each CTA's stage, so K (A) is read from shared
        // memory once per k-block instead of once per plane
        const uint32_t n_mma = (is_i8(KD) && VXQ_I8_MERGED) ? (uint32_t)(TR::kPlanes * a.bn)
                                                             : (uint32_t)a.bn;
        const uint32_t idesc =
            (MX ? ((1u << 7) | (1u << 10) | (1u << 23)) : (TR::kIdescBase | a.idesc_extra)) |
            ((n_mma >> 3) << 17) | ((uint32_t)((PAIR ? 2 * DBM : DBM) >> 4) << 24);
        int stage = 0;
        uint32_t ph = 0;
        int lt = 0;
        long long mm_full = 0, mm_tempty = 0;
        for (int k = 0;; ++k, ++lt) {
            const int g = next_ticket(k);
            __syncwarp();
            if (lane == 0) release_ticket(k);
            if (g < 0) break;
            const int acc = lt & 1;
            const uint32_t acc_ph = (lt >> 1) & 1;
            long long c0 = a.stats ? clk() : 0;
            ptx::mbar_wait(tempty + acc, acc_ph ^ 1, a.timeout_ns);
            if (a.stats) mm_tempty += clk() - c0;
            ptx::tc_fence_after();
            const uint32_t d = tmem_base + acc * ACC_COLS;
            for (int kb = 0; kb < a.kblocks; ++kb) {
                c0 = a.stats ? clk() : 0;
                ptx::mbar_wait(full + stage, ph, a.timeout_ns);
                if (a.stats) mm_full += clk() - c0;
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t sa = ptx::smem_u32(smem + stage * SBYTES);
                    const uint64_t da = ptx::sw128_kmajor_desc(sa);
#pragma unroll
                    for (int pl = 0; pl < ((is_i8(KD) && VXQ_I8_MERGED) ? 1 : TR::kPlanes); ++pl) {
                        const uint64_t db =
                            ptx::sw128_kmajor_desc(sa + A_BYTES + pl * b_plane_bytes);
#pragma unroll
                        for (int k = 0; k < DROW / 32; ++k) {  // 32 B of K per MMA
                            const uint32_t accum = (kb | pl | k) != 0;
                            if constexpr (is_i8(KD)) {  // one S32 accumulator per plane
                                ptx::mma2_i8(d + pl * (uint32_t)a.bn, da + 2 * k, db + 2 * k,
                                             idesc, (kb | k) != 0);
                                continue;
                            }
                            if constexpr (MX && PAIR)
                                ptx::mma2_mxf4(d, da + 2 * k, db + 2 * k, idesc,
                                               tmem_base + kSfCol, tmem_base + kSfCol + 16,
                                               accum);
                            else if constexpr (MX)
                                ptx::mma_mxf4(d, da + 2 * k, db + 2 * k, idesc,
                                              tmem_base + kSfCol, tmem_base + kSfCol + 16,
                                              accum);
                            else if constexpr (PAIR && KD == Kind::kF16x2)
                                ptx::mma2_f16(d, da + 2 * k, db + 2 * k, idesc, accum);
                            else if constexpr (PAIR && (KD == Kind::kJ16x2 || KD == Kind::kJQ16)) {
                                // J1.s then J2.s (the A planes sit DA_BYTES apart)
                                ptx::mma2_f16(d, da + 2 * k, db + 2 * k, idesc, accum);
                                ptx::mma2_f16(d, da + (DA_BYTES >> 4) + 2 * k, db + 2 * k, idesc,
                                              1u);
                            }
                            else if constexpr (PAIR)
                                ptx::mma2_f8f6f4(d, da + 2 * k, db + 2 * k, idesc, accum);
                            else if constexpr (KD == Kind::kFp8)
                                ptx::mma_f8f6f4(d, da + 2 * k, db + 2 * k, idesc, accum);
                            else
                                ptx::mma_f16(d, da + 2 * k, db + 2 * k, idesc, accum);
                        }
                    }
                    if constexpr (SP) ptx::mma2_commit_mc(empty + stage, 0xF);  // both pairs
                    else if constexpr (PAIR) ptx::mma2_commit_mc(empty + stage, 0x3);
                    else if constexpr (CL > 1) ptx::mma_commit_mc(empty + stage, kMask);
                    else ptx::mma_commit(empty + stage);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    ph ^= 1;
                }
            }
            if (ptx::elect_one()) {
                if constexpr (PAIR) ptx::mma2_commit_mc(tfull + acc, (uint16_t)(0x3u << (2 * pr)));
                else ptx::mma_commit(tfull + acc);
            }
            __syncwarp();
        }
        if (a.stats && lane == 0) {
            atomicAdd(a.stats + 2, (unsigned long long)mm_full);
            atomicAdd(a.stats + 3, (unsigned long long)mm_tempty);
            atomicAdd(a.stats + 6, (unsigned long long)lt);
        }
        }
    mma_done:;
    } else if (warp == 10) {
        // ---------------- x/m loader (PA steps): chunk c of every tile this CTA owns
        if (xm_on && a.mode == 0 && ptx::elect_one()) {
            const uint64_t pol = ptx::policy_evict_first();
            const int nch = a.bn / 16;
            int jh[2] = {0, 0};  // chunks loaded per epilogue half
            for (int k = 0;; ++k) {
                const int g = next_ticket(k);
                release_ticket(k);
                if (g < 0) break;
                int t, nb, mb;
                tile_of(g, t, nb, mb);
                if (mb >= a.m_tiles) continue;  // no rows: the epilogue skips it too
                if (t > 0) {
                    // x/m of step t were written by the step-(t-1) tiles of this replica
                    // block (any CTA): acquire their counter, then order the async-proxy
                    // loads after it
                    const unsigned* cnt = a.done + (size_t)(t - 1) * a.n_tiles + nb;
                    if (ld_acquire_gpu(cnt) < (unsigned)a.m_tiles) {
                        uint64_t t0, tn;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                        while (ld_acquire_gpu(cnt) < (unsigned)a.m_tiles) {
                            __nanosleep(64);
                            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                            if (tn - t0 > a.timeout_ns) __trap();
                        }
                    }
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                for (int c = 0; c < nch; ++c) {
                    const int h = c & 1, j = jh[h]++;
                    const int slot = h * XHS + j % XHS;
                    ptx::mbar_wait(xempty + slot, ((uint32_t)(j / XHS) & 1u) ^ 1u, a.timeout_ns);
                    uint8_t* xs = xm_smem + slot * XM_SLOT_BYTES;
                    ptx::mbar_arrive_expect_tx(xfull + slot, XM_SLOT_BYTES);
                    ptx::tma_load_2d_hint(xs, &tmX, xfull + slot, mb * DBM, nb * a.bn + c * 16,
                                          pol);
                    ptx::tma_load_2d_hint(xs + XM_SLOT_BYTES / 2, &tmM, xfull + slot, mb * DBM,
                                          nb * a.bn + c * 16, pol);
                }
            }
        }
    } else {
        // ---------------- epilogue (8 warps): TMEM -> integrator -> next B operand
        // warp w may only touch TMEM lanes 32*(w%4)..+31; the two warps of a lane quarter
        // take alternate 16-column chunks of the tile.
        const int q = warp & 3;
        const int half = (warp - 2) >> 2;
        const int row = q * 32 + lane;
        const int ep_tid = threadIdx.x - 64;  // 0..255
        using O = Ops<float>;
        const int nch = a.bn / 16;
        float* __restrict__ xg = a.x;
        float* __restrict__ mg = a.m;
        int lt = 0, xm_chunks = 0;  // x/m chunks this half consumed
        long long ep_wait = 0, ep_busy = 0, ep_xwait = 0;
        for (int k = 0;; ++k, ++lt) {
            const int g = next_ticket(k);
            __syncwarp();
            if (lane == 0) release_ticket(k);
            if (g < 0) break;
            int t, nb, mb;
            tile_of(g, t, nb, mb);
            const bool tile_ok = mb < a.m_tiles;  // last cluster row group may be partial
            const int acc = lt & 1;
            const uint32_t acc_ph = (lt >> 1) & 1;
            const int i = mb * DBM + row;
            const bool row_ok = i < a.n;
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * ACC_COLS;
            // x/m of this warp's chunks do not depend on the accumulator: the first chunk's
            // loads are issued before waiting for the MMA, and each later chunk's while the
            // previous one is computed (two register buffers, chunks c, c+2, c+4, ...)
            const uint64_t stream = ptx::policy_evict_first();
            float xA[16], mA[16], xB[16], mB[16];
            auto load_chunk = [&](int c, float* xo, float* mo) {
                const int r0 = nb * a.bn + c * 16;
                const int64_t base = (int64_t)r0 * a.ld + i;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    const bool ok = row_ok && (r0 + jj) < a.R;
                    xo[jj] = ok ? ptx::ld_stream(xg + base + (int64_t)jj * a.ld, stream) : 0.f;
                    mo[jj] = ok ? ptx::ld_stream(mg + base + (int64_t)jj * a.ld, stream) : 0.f;
                }
            };
            const bool xm = xm_on && a.mode == 0;
            if (a.mode == 0 && !xm && half < nch) {
                // x/m of step t are written by the step-(t-1) tiles of this replica block
                // (possibly on other CTAs): acquire their counter before the early load
                if (t > 0) {
                    const unsigned* cnt = a.done + (size_t)(t - 1) * a.n_tiles + nb;
                    if (ld_acquire_gpu(cnt) < (unsigned)a.m_tiles) {
                        uint64_t t0, tn;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                        while (ld_acquire_gpu(cnt) < (unsigned)a.m_tiles) {
                            __nanosleep(64);
                            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                            if (tn - t0 > a.timeout_ns) __trap();
                        }
                    }
                }
                load_chunk(half, xA, mA);
            }
            long long c0 = (a.stats && ep_tid == 0) ? clk() : 0;
            ptx::mbar_wait(tfull + acc, acc_ph, a.timeout_ns);
            long long c1 = (a.stats && ep_tid == 0) ? clk() : 0;
            if (a.stats && ep_tid == 0) ep_wait += c1 - c0;
            ptx::tc_fence_after();
            if (a.mode == 0) {
                uint8_t* nxt = (t & 1) ? a.b_buf[0] : a.b_buf[1];  // B operand of step t+1
                if (a.bestq && t > 0) {
                    // fused best tracking: q_{t-1} is final (every step-(t-1) tile published),
                    // and this tile's rows of s_{t-1} are still in nxt until process() below
                    // overwrites them with s_{t+1}: copy them for replicas that improved
                    const long long* qp = a.qtrace + (int64_t)(t - 1) * a.R;
                    for (int c = half; c < nch; c += 2) {
#pragma unroll 4
                        for (int jj = 0; jj < 16; ++jj) {
                            const int r = nb * a.bn + c * 16 + jj;
                            if (r >= a.R || !row_ok) continue;
                            if (qp[r] < a.bestq[r]) {
                                const int64_t off = (int64_t)r * a.ld + i;
                                int8_t sv;
                                if (a.b_fp4) {
                                    const uint8_t by = nxt[off >> 1];
                                    sv = (((i & 1) ? (by >> 4) : by) & 0x8) ? -1 : 1;
                                } else {
                                    sv = (nxt[off] & 0x80) ? -1 : 1;
                                }
                                a.best_s[off] = sv;
                            }
                        }
                    }
                    __syncwarp();  // lane pairs share packed bytes: read before any write
                }
                const float st = __ldg(a.sched + t);
                const float hi = row_ok ? __ldg(a.h + i) : 0.f;
                auto process = [&](int c, const float* xo, const float* mo) {
                    uint32_t v[16], v1[16], v2[16], v3[16];
                    if constexpr (is_i8(KD) && VXQ_I8_MERGED) {
                        // merged MMA: replica j of the block, plane pl sits in column
                        // h P bn/2 + pl bn/2 + (j - h bn/2), h = (j >= bn/2); 8-column pieces
                        // never straddle the halves (bn is a multiple of 16)
                        const uint32_t hb = (uint32_t)a.bn / 2;
#pragma unroll
                        for (int piece = 0; piece < 2; ++piece) {
                            const uint32_t j = (uint32_t)(c * 16 + piece * 8);
                            const uint32_t h = j >= hb ? 1u : 0u;
                            const uint32_t col = h * (uint32_t)TR::kPlanes * hb + (j - h * hb);
                            ptx::tmem_ld_32x32b_x8(tbase + col, v + piece * 8);
                            ptx::tmem_ld_32x32b_x8(tbase + col + hb, v1 + piece * 8);
                            ptx::tmem_ld_32x32b_x8(tbase + col + 2 * hb, v2 + piece * 8);
                            if constexpr (KD == Kind::kI8x4)
                                ptx::tmem_ld_32x32b_x8(tbase + col + 3 * hb, v3 + piece * 8);
                        }
                    } else {
                        ptx::tmem_ld_32x32b_x16(tbase + c * 16, v);
                        if constexpr (is_i8(KD)) {  // the digit planes' accumulators
                            ptx::tmem_ld_32x32b_x16(tbase + (uint32_t)a.bn + c * 16, v1);
                            ptx::tmem_ld_32x32b_x16(tbase + 2u * (uint32_t)a.bn + c * 16, v2);
                        }
                        if constexpr (KD == Kind::kI8x4)  // K s_t (the spin plane)
                            ptx::tmem_ld_32x32b_x16(tbase + 3u * (uint32_t)a.bn + c * 16, v3);
                    }
                    const int r0 = nb * a.bn + c * 16;
                    const int64_t base = (int64_t)r0 * a.ld + i;
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const bool ok = row_ok && (r0 + jj) < a.R;
                        const int64_t off = base + (int64_t)jj * a.ld;
                        float f;
                        if constexpr (is_i8(KD)) {
                            // K.Q exactly (|K.Q| < 2^37), rounded once to fp32, * 2^-S (exact)
                            const long long kq = (long long)(int)v[jj] +
                                                 256LL * (long long)(int)v1[jj] +
                                                 65536LL * (long long)(int)v2[jj];
                            f = O::mul(a.scale, __fmul_rn(__ll2float_rn(kq), a.qscale_inv));
                        } else {
                            f = O::mul(a.scale, __uint_as_float(v[jj]));
                        }
                        if constexpr (PA_KIND) {
                            if (KD == Kind::kFp8 && a.qtrace) {  // exact energy of s_t
                                const int kk = (int)__uint_as_float(v[jj]);
                                const int term = ok ? (xo[jj] >= 0.f ? kk : -kk) : 0;
                                const int sum = __reduce_add_sync(0xffffffffu, term);
                                if (lane == 0 && (r0 + jj) < a.R)
                                    atomicAdd(reinterpret_cast<unsigned long long*>(a.qtrace) +
                                                  (int64_t)t * a.R + r0 + jj,
                                              (unsigned long long)(long long)sum);
                            }
                            // PA: grad = (lam x + f) + h; m = alpha m - eta grad; x = clip
                            const float grad = O::add(O::add(O::mul(st, xo[jj]), f), hi);
                            const float mn = O::sub(O::mul(a.alpha, mo[jj]), O::mul(a.eta, grad));
                            float xn = O::add(xo[jj], mn);
                            xn = xn < -1.f ? -1.f : (xn > 1.f ? 1.f : xn);
                            if constexpr (KD == Kind::kJ16x2) {
                                if (ok) {
                                    ptx::st_stream(xg + off, xn, stream);
                                    ptx::st_stream(mg + off, mn, stream);
                                    reinterpret_cast<uint16_t*>(nxt)[off] =
                                        xn >= 0.f ? (uint16_t)0x3C00 : (uint16_t)0xBC00;  // +-1
                                }
                            } else if (ok) {
                                ptx::st_stream(xg + off, xn, stream);
                                ptx::st_stream(mg + off, mn, stream);
                                if (!a.b_fp4) nxt[off] = xn >= 0.f ? FP8_P1 : FP8_M1;
                            }
                            if (KD == Kind::kFp8 && a.b_fp4) {  // lanes 2k, 2k+1 = rows i, i+1: one packed byte
                                const uint32_t code = ok ? (xn >= 0.f ? FP4_P1 : FP4_M1) : 0u;
                                const uint32_t hi4 = __shfl_xor_sync(0xffffffffu, code, 1);
                                if (!(lane & 1) && (code | hi4))
                                    nxt[off >> 1] = (uint8_t)(code | (hi4 << 4));
                            }
                        } else {
                            // SBM with B = -A = -c K, g = -h (field = -f)
                            const float qi = xo[jj];
                            if constexpr (KD == Kind::kI8x4) {
                                // exact coupling energy of s_t = sign(q_t): sum_i s_i (K s_t)_i
                                if (a.qtrace) {
                                    const int ks = (int)v3[jj];
                                    const int term = ok ? (qi >= 0.f ? ks : -ks) : 0;
                                    const int sum = __reduce_add_sync(0xffffffffu, term);
                                    if (lane == 0 && (r0 + jj) < a.R)
                                        atomicAdd(reinterpret_cast<unsigned long long*>(a.qtrace) +
                                                      (int64_t)t * a.R + r0 + jj,
                                                  (unsigned long long)(long long)sum);
                                }
                            }
                            const float inner = -O::sub(O::add(O::mul(qi, qi), a.a0), st);
                            const float force =
                                O::add(O::mul(inner, qi), O::mul(a.c0, O::add(-f, hi)));
                            float pn = O::add(mo[jj], O::mul(a.dt, force));
                            float qn = O::add(qi, O::mul(a.dta0, pn));
                            if (fabsf(qn) > a.q_cap) {
                                qn = qn < -a.q_cap ? -a.q_cap : a.q_cap;
                                pn = 0.f;
                            }
                            if (ok) {
                                ptx::st_stream(xg + off, qn, stream);
                                ptx::st_stream(mg + off, pn, stream);
                                if constexpr (is_i8(KD)) {
                                    int8_t d0, d1, d2;
                                    digits3(qn, a.qscale, d0, d1, d2);
                                    int8_t* pl = reinterpret_cast<int8_t*>(nxt);
                                    pl[off] = d0;
                                    pl[a.plane_elems + off] = d1;
                                    pl[2 * a.plane_elems + off] = d2;
                                    if constexpr (KD == Kind::kI8x4)  // s_{t+1}
                                        pl[3 * a.plane_elems + off] = qn >= 0.f ? 1 : -1;
                                } else if constexpr (KD == Kind::kF16x2 || KD == Kind::kJQ16) {
                                    __half q1, q2;
                                    split2(qn, q1, q2);
                                    __half* pl = reinterpret_cast<__half*>(nxt);
                                    pl[off] = q1;
                                    pl[a.plane_elems + off] = q2;
                                } else {
                                    __nv_bfloat16 q1, q2, q3;
                                    split3(qn, q1, q2, q3);
                                    __nv_bfloat16* pl = reinterpret_cast<__nv_bfloat16*>(nxt);
                                    pl[off] = q1;
                                    pl[a.plane_elems + off] = q2;
                                    pl[2 * a.plane_elems + off] = q3;
                                }
                            }
                        }
                    }
                };
                // fast path (PA, packed spins, no per-step trace, a full 16-replica chunk):
                // no per-element range checks, incrementally bumped pointers, the spin byte of
                // rows (i, i+1) always written by the even lane (padding rows stay 0)
                auto process_fast = [&](int c, const float* xo, const float* mo) {
                    uint32_t v[16];
                    ptx::tmem_ld_32x32b_x16(tbase + c * 16, v);
                    const int r0 = nb * a.bn + c * 16;
                    const int64_t base = (int64_t)r0 * a.ld + i;
                    float* px = xg + base;
                    float* pm = mg + base;
                    uint8_t* pb = nxt + (base >> 1);
                    const int64_t ld = a.ld, ldb = a.ld >> 1;
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const float f = O::mul(a.scale, __uint_as_float(v[jj]));
                        const float grad = O::add(O::add(O::mul(st, xo[jj]), f), hi);
                        const float mn = O::sub(O::mul(a.alpha, mo[jj]), O::mul(a.eta, grad));
                        float xn = O::add(xo[jj], mn);
                        xn = xn < -1.f ? -1.f : (xn > 1.f ? 1.f : xn);
                        if (row_ok) {
                            ptx::st_stream(px, xn, stream);
                            ptx::st_stream(pm, mn, stream);
                        }
                        const uint32_t code = row_ok ? (xn >= 0.f ? FP4_P1 : FP4_M1) : 0u;
                        const uint32_t hi4 = __shfl_xor_sync(0xffffffffu, code, 1);
                        if (!(lane & 1)) *pb = (uint8_t)(code | (hi4 << 4));
                        px += ld;
                        pm += ld;
                        pb += ldb;
                    }
                };
                const bool fast_ok = KD == Kind::kFp8 && a.b_fp4 && !a.qtrace;
                if (xm) {
                    if (tile_ok) {
#pragma unroll 1
                        for (int c = half; c < nch; c += 2) {
                            const int slot = half * XHS + xm_chunks % XHS;
                            const uint32_t par = (uint32_t)(xm_chunks / XHS) & 1u;
                            ++xm_chunks;
                            const long long cx = (a.stats && ep_tid == 0) ? clk() : 0;
                            ptx::mbar_wait(xfull + slot, par, a.timeout_ns);
                            if (a.stats && ep_tid == 0) ep_xwait += clk() - cx;
                            const float* xs =
                                reinterpret_cast<const float*>(xm_smem + slot * XM_SLOT_BYTES);
                            const float* ms = xs + 16 * DBM;
#pragma unroll
                            for (int jj = 0; jj < 16; ++jj) {
                                xA[jj] = xs[jj * DBM + row];
                                mA[jj] = ms[jj * DBM + row];
                            }
                            __syncwarp();
                            if (lane == 0) ptx::mbar_arrive(xempty + slot);  // slot refillable
                            if (fast_ok && nb * a.bn + c * 16 + 16 <= a.R) process_fast(c, xA, mA);
                            else process(c, xA, mA);
                        }
                    }
                } else {
#pragma unroll 1
                    for (int c = half; c < nch; c += 4) {  // xA/mA hold chunk c
                        if (c + 2 < nch) load_chunk(c + 2, xB, mB);
                        process(c, xA, mA);
                        if (c + 4 < nch) load_chunk(c + 4, xA, mA);
                        if (c + 2 < nch) process(c + 2, xB, mB);
                    }
                }
            } else if (a.mode == 1) {
                // energy pass (fp8 signs): 2 q_r = sum_i s_i (K s)_i, exact integers
#pragma unroll 1
                for (int c = half; c < nch; c += 2) {
                    uint32_t v[16];
                    ptx::tmem_ld_32x32b_x16(tbase + c * 16, v);
                    ptx::tmem_ld_wait();
                    const int r0 = nb * a.bn + c * 16;
                    const float* xr = xg + ((int64_t)r0 * a.ld + i);
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const bool ok = row_ok && (r0 + jj) < a.R;
                        const float xo = ok ? xr[jj * a.ld] : 0.f;
                        const int k = (int)__uint_as_float(v[jj]);
                        const int term = ok ? (xo >= 0.f ? k : -k) : 0;
                        const int sum = __reduce_add_sync(0xffffffffu, term);
                        if (lane == 0 && (r0 + jj) < a.R)
                            atomicAdd(reinterpret_cast<unsigned long long*>(a.q2) + r0 + jj,
                                      (unsigned long long)(long long)sum);
                    }
                }
            }
            if (a.stats && ep_tid == 0) ep_busy += clk() - c1;
            ptx::tc_fence_before();
            if constexpr (PAIR) ptx::mbar_arrive_leader(tempty + acc);  // the MMA is there
            else ptx::mbar_arrive(tempty + acc);
            if (a.mode == 0 && a.bestq && t > 0 && tile_ok) {
                // the tile that completes the step-t decisions of this replica block folds
                // q_{t-1} into bestq -- before its own publish below, so step-(t+1) tiles
                // (which acquire the done counter) see it
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (ep_tid == 0)
                    s_last = atomicAdd(a.decided + (size_t)t * a.n_tiles + nb, 1u) ==
                             (unsigned)a.m_tiles - 1;
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (s_last) {
                    __threadfence();
                    const long long* qp = a.qtrace + (int64_t)(t - 1) * a.R;
                    for (int r = nb * a.bn + ep_tid; r < min(a.R, (nb + 1) * a.bn); r += 256)
                        if (qp[r] < a.bestq[r]) a.bestq[r] = qp[r];
                }
            }
            if (a.mode != 1 && tile_ok && t + 1 < a.T) {
                // publish: all 256 epilogue threads' stores, then one release increment
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (ep_tid == 0) {
                    __threadfence();
                    atomicAdd(a.done + (size_t)t * a.n_tiles + nb, 1u);
                }
            }
        }
        if (a.stats && ep_tid == 0) {
            atomicAdd(a.stats + 4, (unsigned long long)ep_wait);
            atomicAdd(a.stats + 5, (unsigned long long)ep_busy);
            atomicAdd(a.stats + 8, (unsigned long long)ep_xwait);
        }
    }
    __syncthreads();
    if (a.stats && threadIdx.x == 0) atomicMax(a.stats + 7, (unsigned long long)(clk() - t_start));
    if constexpr (NCTA > 1) ptx::cluster_sync();  // no CTA exits while peers still signal it
    if (warp == 1) {
        if constexpr (PAIR) ptx::tmem_dealloc2<512>(tmem_base);
        else ptx::tmem_dealloc<512>(tmem_base);
    }
}

constexpr int TB = 256;
inline unsigned nblk(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, TB)); }

__global__ void k_fill_nan(double* v, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = NAN;
}

__global__ void k_any_nonzero(int64_t n, const double* v, int* flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && v[i] != 0.0) *flag = 1;
}

// trace[t] = min_r (offset + c * q_t[r] / 2) (h = 0; NaN otherwise: no exact h-term here)
__global__ void k_trace_from_q(const long long* q, int64_t T, int64_t R, double c,
                               double offset, const int* h_nonzero, double* trace) {
    __shared__ double sh[256];
    const int64_t t = blockIdx.x;
    double v = INFINITY;
    for (int64_t r = threadIdx.x; r < R; r += blockDim.x)
        v = fmin(v, offset + c * (double)(q[t * R + r] / 2));
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] = fmin(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) trace[t] = *h_nonzero ? NAN : sh[0];
}

int num_sms() {
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return nsm;
}

// replica tile width bn: minimise tiles x per-k-block time, where a k-block costs
// max(MMA = planes x 4 x 128*bn/256 = planes*2*bn, smem read (16 KB A + planes*128*bn B) /
// 128 B/cyc) cycles.  The persistent kernel spreads all T steps' tiles over the SMs, so
// per-step rounds do not matter.
int choose_bn(int64_t n, int64_t R, int planes, int bn_max) {
    const int64_t m_tiles = ceil_div(n, DBM);
    int bn = bn_max;
    int64_t best = INT64_MAX;
    for (int cand = bn_max; cand >= 64; cand -= 16) {
        const int64_t tiles = m_tiles * ceil_div(R, cand);
        const int64_t cost =
            tiles * std::max<int64_t>((int64_t)planes * 2 * cand, 128 + (int64_t)planes * cand);
        if (cost < best) {
            best = cost;
            bn = cand;
        }
    }
    if (const char* e = getenv("VXQ_DENSE_BN")) bn = std::max(16, std::min(bn_max, atoi(e) / 16 * 16));
    return bn;
}

int pick_group(int n_tiles) {
    int gsz = 1;
    if (const char* e = getenv("VXQ_DENSE_GROUP")) gsz = std::max(1, atoi(e));
    return std::min(gsz, std::max(n_tiles, 1));  // the last group may be smaller
}

template <Kind KD, int CL, bool PAIR = false, bool MX = false>
void launch_run(const CUtensorMap& tmA, const CUtensorMap& tmB0, const CUtensorMap& tmB1,
                DenseRunArgs a, int64_t steps_for_grid, cudaStream_t s, bool cooperative,
                const CUtensorMap* tmX = nullptr, const CUtensorMap* tmM = nullptr) {
    constexpr int NCTA = PAIR ? 2 * CL : CL;
    constexpr int RPC = PAIR ? 2 : CL;
    auto kern = k_dense_run<KD, CL, PAIR, MX>;
    VXQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DSMEM));
    if (NCTA > 2)
        VXQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int64_t items = (int64_t)((a.m_tiles + RPC - 1) / RPC) *
                          (PAIR && CL == 2 ? a.n_tiles / 2 : a.n_tiles) *
                          std::max<int64_t>(steps_for_grid, 1);
    // tile tickets are 32-bit ints in the kernel (steps x tiles per step)
    VXQ_REQUIRE(items < (int64_t)INT32_MAX - 4096, "too many dense tiles (steps x tiles) for one launch");
    int64_t clusters = std::min<int64_t>(items, num_sms() / NCTA);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(clusters * NCTA));
    cfg.blockDim = dim3(DTHREADS);
    cfg.dynamicSmemBytes = DSMEM;
    cfg.stream = s;
    cudaLaunchAttribute attrs[2];
    int na = 0;
    if (NCTA > 1) {
        attrs[na].id = cudaLaunchAttributeClusterDimension;
        attrs[na].val.clusterDim.x = NCTA;
        attrs[na].val.clusterDim.y = 1;
        attrs[na].val.clusterDim.z = 1;
        ++na;
    }
    // The dynamic tile queue needs no co-residency, so the kernel launches as a plain
    // (cluster) grid -- profilers can replay it.  VXQ_DENSE_COOP=1 adds the cooperative
    // attribute anyway (A/B only).
    cooperative = false;
    if (const char* e = getenv("VXQ_DENSE_COOP"))
        if (atoi(e) == 1) cooperative = true;
    if (cooperative) {
        attrs[na].id = cudaLaunchAttributeCooperative;
        attrs[na].val.cooperative = 1;
        ++na;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = na;
    if (NCTA > 2) {  // 4-CTA clusters do not tile all 148 SMs: launch what can be resident
        int maxc = 0;
        if (cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg) == cudaSuccess && maxc > 0 &&
            maxc < clusters) {
            clusters = maxc;
            cfg.gridDim = dim3((unsigned)(clusters * NCTA));
        }
    }
    VXQ_REQUIRE(!a.xm || (tmX && tmM), "x/m staging needs their tensor maps");
    DevBuf<unsigned> ticket(1, s);
    VXQ_CUDA(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), s));
    a.ticket = ticket.get();
    // no A-panel L2 prefetch by default: the operands are L2-resident, and the prefetches
    // were a quarter of the L2 tag-stage traffic that bounds the kernel (cfg2 PA 156 -> 173
    // Grv/s, tensor pipe 46 -> 56 %; SBM +4 %; profiles/r02/ab_aprefetch/)
    // (the general-J kinds, whose 400 MB J planes stream from DRAM, gain without it too:
    // PA 17.7 -> 19.6, SBM 12.0 -> 12.7 Grv/s at n = 10^4)
    a.a_prefetch = 0;
    if (const char* e = getenv("VXQ_DENSE_APF")) a.a_prefetch = atoi(e) != 0;
    a.timeout_ns = 10ull * 1000 * 1000 * 1000;
    if (const char* e = getenv("VXQ_WAIT_TIMEOUT_S"))
        a.timeout_ns = (uint64_t)std::max(1, atoi(e)) * 1000ull * 1000 * 1000;
    VXQ_CUDA(cudaLaunchKernelEx(&cfg, kern, tmA, tmB0, tmB1, tmX ? *tmX : tmA, tmM ? *tmM : tmA,
                                a));
    VXQ_CHECK_LAUNCH();
}

}  // namespace

// Crossovers (measured at n = 10^4, R = 1024): the mxf4 path is ~350x the CSR step on a
// dense SK instance and the general fp16-plane path ~42x, while their cost does not depend
// on the density -- so they stay ahead down to a few percent density.  The n caps bound the
// dense operands (packed fp4: n^2/2 bytes; two fp16 planes: 4 n^2 bytes).
bool dense_eligible(const Problem* p, int64_t R) {
    if (!p->uniform_magnitude || p->n < 256 || p->n > 65536 || R < 128) return false;
    double density = (double)p->nnz / ((double)p->n * (double)p->n);
    return density >= 0.02;
}

bool dense_sbm_fp16_ok(double q_cap, double amp) { return std::max(q_cap, amp) <= 16384.0; }

// S of the exact SBM path's fixed-point q (Q = rint(q 2^S), |Q| <= 2^22): the largest S with
// max(q_cap, init_noise) <= 2^(22-S); -1 if |q| is unbounded (q_cap = inf) or out of range
int sbm_fixed_point_shift(double q_cap, double amp) {
    const double b = std::max(q_cap, amp);
    if (!(b > 0) || !std::isfinite(b)) return -1;
    int e = 0;
    const double m = std::frexp(b, &e);  // b = m 2^e, m in [0.5, 1)
    const int ceil_log2 = (m == 0.5) ? e - 1 : e;
    return 22 - ceil_log2;
}

// general (non-uniform) dense J on the tensor cores: no in-kernel energies
bool dense_general_eligible(const Problem* p, int64_t R) {
    if (p->uniform_magnitude || p->n < 512 || p->n > 32768 || R < 128 || !(p->magnitude > 0))
        return false;
    if (const char* e = getenv("VXQ_DENSE_GENERAL"))
        if (atoi(e) == 0) return false;
    double density = (double)p->nnz / ((double)p->n * (double)p->n);
    return density >= 0.05;
}

// Lazily build the fp16 planes of 2^e J (e: the largest scaled |J| stays below 2^15).
static DenseOperand* dense_jplanes(Problem* p, cudaStream_t s) {
    std::lock_guard<std::mutex> g(p->mu);
    DenseOperand* d = p->dense;
    const bool fresh = d == nullptr;
    if (fresh) {
        d = new DenseOperand();
        d->n = p->n;
        d->ld = ceil_div(p->n, 128) * 128;
    }
    try {
        if (!d->J16) {
            const int64_t ld = d->ld;
            int ex = 0;
            std::frexp((double)(float)p->magnitude, &ex);  // |J| < 2^ex
            const int e = 15 - ex;
            VXQ_REQUIRE(e > -100 && e < 100, "coupling magnitudes out of the fp16-plane range");
            const float scale = std::ldexp(1.0f, e);
            d->jscale_inv = std::ldexp(1.0f, -e);
            VXQ_CUDA(cudaMallocAsync((void**)&d->J16, 2 * ld * ld * sizeof(__half), s));
            VXQ_CUDA(cudaMemsetAsync(d->J16, 0, 2 * ld * ld * sizeof(__half), s));
            k_build_j_planes<<<(unsigned)ceil_div(p->n * 32, TB), TB, 0, s>>>(
                p->n, ld, p->indptr, p->indices, p->data32, scale, d->J16);
            VXQ_CHECK_LAUNCH();
            d->tmJ = make_map(d->J16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, ld, ld, 2, DROW / 2,
                              DBM, 2);
            VXQ_CUDA(cudaStreamSynchronize(s));
        }
    } catch (...) {
        if (fresh) delete d;
        throw;
    }
    p->dense = d;
    return d;
}

// Lazily build the sign matrix K (fp8 for PA/energies, bf16 for SBM) and its TMA maps.
// need16: 0 none, 1 bf16 K (SBM bf16x3), 2 fp16 K (SBM f16x2), 3 int8 K (SBM exact)
DenseOperand* dense_operand(Problem* p, cudaStream_t s, int need16) {
    std::lock_guard<std::mutex> g(p->mu);
    if (!p->uniform_magnitude)
        throw Error(VXQ_ERR_UNSUPPORTED, "dense tensor-core path needs uniform |J_ij|");
    DenseOperand* d = p->dense;
    const bool fresh = d == nullptr;
    if (fresh) {
        d = new DenseOperand();
        d->n = p->n;
        d->ld = ceil_div(p->n, 128) * 128;
        d->scale = (float)p->magnitude;
    }
    try {
        const int64_t ld = d->ld;
        uint8_t* k8 = nullptr;
        __nv_bfloat16* k16 = nullptr;
        __half* k16h = nullptr;
        uint32_t* k4 = nullptr;
        int8_t* ki8 = nullptr;
        if (need16 == 3 && !d->Ki8) {
            VXQ_CUDA(cudaMallocAsync((void**)&d->Ki8, ld * ld, s));
            VXQ_CUDA(cudaMemsetAsync(d->Ki8, 0, ld * ld, s));
            ki8 = d->Ki8;
            d->tmAi8 = make_map(d->Ki8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld, ld, 1, DROW, DBM, 1);
        }
        if (!d->K8) {
            // default: K as packed E2M1 (51 MB at n = 10^4: stays L2-resident, -60 % DRAM
            // traffic, higher clocks under the power cap); VXQ_DENSE_FP4=0 -> FP8 E4M3
            const char* e4 = getenv("VXQ_DENSE_FP4");
            const bool fp4 = !(e4 && atoi(e4) == 0);
            const int64_t bytes = fp4 ? ld * ld / 2 : ld * ld;
            VXQ_CUDA(cudaMallocAsync((void**)&d->K8, bytes, s));
            VXQ_CUDA(cudaMemsetAsync(d->K8, 0, bytes, s));
            if (fp4) {
                k4 = reinterpret_cast<uint32_t*>(d->K8);
                d->afmt = 5;
                d->tmA8 = make_map_fp4(d->K8, ld, ld, DROW, DBM);
            } else {
                k8 = d->K8;
                d->afmt = 0;
                d->tmA8 = make_map(d->K8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld, ld, 1, DROW, DBM,
                                   1);
            }
        }
        if (need16 == 2 && !d->K16h) {
            VXQ_CUDA(cudaMallocAsync((void**)&d->K16h, ld * ld * 2, s));
            VXQ_CUDA(cudaMemsetAsync(d->K16h, 0, ld * ld * 2, s));
            k16h = d->K16h;
            d->tmA16h = make_map(d->K16h, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, ld, ld, 1,
                                 DROW / 2, DBM, 1);
        }
        if (need16 == 1 && !d->K16) {
            VXQ_CUDA(cudaMallocAsync((void**)&d->K16, ld * ld * 2, s));
            VXQ_CUDA(cudaMemsetAsync(d->K16, 0, ld * ld * 2, s));
            k16 = d->K16;
            d->tmA16 = make_map(d->K16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ld, ld, 1, DROW / 2,
                                DBM, 1);
        }
        if (k8 || k16 || k4 || k16h || ki8) {
            k_build_sign_matrix<<<(unsigned)ceil_div(p->n * 32, TB), TB, 0, s>>>(
                p->n, ld, p->indptr, p->indices, p->data64, k8, k16, k4, k16h, ki8);
            VXQ_CHECK_LAUNCH();
            VXQ_CUDA(cudaStreamSynchronize(s));
        }
    } catch (...) {
        if (fresh) delete d;
        throw;
    }
    p->dense = d;
    return d;
}

static uint32_t a_tx_bytes(const DenseOperand* d) {
    if (d->afmt == 0) return DA_BYTES;
    const char* e = getenv("VXQ_DENSE_FP4_TXFULL");
    return (e && atoi(e)) ? DA_BYTES : DA_BYTES / 2;
}

// fp8 energy pass over the signs of `x` ([R][ld]) -> q2 = 2 sum_{i<j} K_ij s_i s_j
static void energy_pass(DenseOperand* d, const float* x, int64_t n, int64_t R, long long* q2,
                        cudaStream_t s, int64_t* launches) {
    const int64_t ld = d->ld;
    DevBuf<uint8_t> sg(R * ld, s);
    VXQ_CUDA(cudaMemsetAsync(sg.get(), 0, R * ld, s));
    k_signs_fp8_rm<<<nblk(n * R), TB, 0, s>>>(x, n, R, ld, sg.get());
    VXQ_CUDA(cudaMemsetAsync(q2, 0, R * sizeof(long long), s));
    const int bn = choose_bn(n, R, 1, KindTraits<Kind::kFp8>::kBnMax);
    CUtensorMap tb = make_map(sg.get(), CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld, R, 1, DROW, bn, 1);
    DenseRunArgs e{};
    e.idesc_extra = d->afmt << 7;  // A = K (fp8 or packed fp4)
    e.a_tx_bytes = a_tx_bytes(d);
    e.b_tx_bytes = (uint32_t)bn * DROW;  // fp8 signs
    e.n = (int)n;
    e.R = (int)R;
    e.ld = (int)ld;
    e.kblocks = (int)(ld / DROW);
    e.m_tiles = (int)ceil_div(n, DBM);
    e.n_tiles = (int)ceil_div(R, bn);
    e.bn = bn;
    e.T = 1;
    e.x = const_cast<float*>(x);
    e.mode = 1;
    e.q2 = q2;
    e.group = 1;
    launch_run<Kind::kFp8, 1>(d->tmA8, tb, tb, e, 1, s, false);
    *launches += 2;
    VXQ_CUDA(cudaStreamSynchronize(s));
}

static thread_local int g_dense_kind = 0;  // VXQ_DENSE_KIND_* of this thread's last run
int dense_last_kind() { return g_dense_kind; }

static double run_loop(DenseRunArgs a, const CUtensorMap& tmA, const CUtensorMap& tb0,
                       const CUtensorMap& tb1, int planes16, int cl, cudaStream_t s,
                       bool pair = false, const CUtensorMap* tmX = nullptr,
                       const CUtensorMap* tmM = nullptr, bool mx = false,
                       bool jplanes = false, bool jq = false) {
    const char* want = getenv("VXQ_DENSE_STATS");
    DevBuf<unsigned long long> stats;
    if (want && want[0] == '1') {
        stats = DevBuf<unsigned long long>(9, s);
        VXQ_CUDA(cudaMemsetAsync(stats.get(), 0, 9 * sizeof(unsigned long long), s));
        a.stats = stats.get();
    }
    g_dense_kind = jplanes ? VXQ_DENSE_KIND_J16X2
                   : jq ? VXQ_DENSE_KIND_JQ16
                   : planes16 == 8 || planes16 == 9 ? VXQ_DENSE_KIND_I8X3
                   : planes16 == 3 ? VXQ_DENSE_KIND_BF16X3
                   : planes16 == 2 ? VXQ_DENSE_KIND_F16X2
                   : mx ? VXQ_DENSE_KIND_MXF4 : VXQ_DENSE_KIND_F8F6F4;
    cudaEvent_t e0, e1;
    VXQ_CUDA(cudaEventCreate(&e0));
    VXQ_CUDA(cudaEventCreate(&e1));
    VXQ_CUDA(cudaEventRecord(e0, s));
    if (a.T > 0) {
        if (jplanes)
            launch_run<Kind::kJ16x2, 1, true>(tmA, tb0, tb1, a, a.T, s, true, tmX, tmM);
        else if (jq) launch_run<Kind::kJQ16, 1, true>(tmA, tb0, tb1, a, a.T, s, true);
        else if (planes16 == 8) launch_run<Kind::kI8x3, 1, true>(tmA, tb0, tb1, a, a.T, s, true);
        else if (planes16 == 9) launch_run<Kind::kI8x4, 1, true>(tmA, tb0, tb1, a, a.T, s, true);
        else if (planes16 == 3) launch_run<Kind::kBf16x3, 1>(tmA, tb0, tb1, a, a.T, s, true);
        else if (planes16 == 2 && pair)
            launch_run<Kind::kF16x2, 1, true>(tmA, tb0, tb1, a, a.T, s, true);
        else if (planes16 == 2) launch_run<Kind::kF16x2, 1>(tmA, tb0, tb1, a, a.T, s, true);
        else if (pair && mx && cl == 2)
            launch_run<Kind::kFp8, 2, true, true>(tmA, tb0, tb1, a, a.T, s, true, tmX, tmM);
        else if (pair && mx)
            launch_run<Kind::kFp8, 1, true, true>(tmA, tb0, tb1, a, a.T, s, true, tmX, tmM);
        else if (mx) launch_run<Kind::kFp8, 1, false, true>(tmA, tb0, tb1, a, a.T, s, true, tmX, tmM);
        else if (pair) launch_run<Kind::kFp8, 1, true>(tmA, tb0, tb1, a, a.T, s, true, tmX, tmM);
        else if (cl == 2) launch_run<Kind::kFp8, 2>(tmA, tb0, tb1, a, a.T, s, true, tmX, tmM);
        else launch_run<Kind::kFp8, 1>(tmA, tb0, tb1, a, a.T, s, true, tmX, tmM);
    }
    VXQ_CUDA(cudaEventRecord(e1, s));
    float ms = 0;
    VXQ_CUDA(cudaEventSynchronize(e1));
    VXQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (a.stats) {
        unsigned long long h[9];
        VXQ_CUDA(cudaMemcpy(h, a.stats, sizeof(h), cudaMemcpyDeviceToHost));
        const double ctas = (double)std::min<int64_t>((int64_t)a.m_tiles * a.n_tiles * a.T,
                                                      num_sms());
        fprintf(stderr,
                "[vxq dense stats] kernel %.0f cyc | per CTA: prod<-empty %.0f, prod<-dep %.0f, "
                "mma<-full %.0f, mma<-tempty %.0f, epi<-tfull %.0f, epi busy %.0f (of which "
                "<-x/m %.0f) | tiles %llu\n",
                (double)h[7], h[0] / ctas, h[1] / ctas, h[2] / ctas, h[3] / ctas, h[4] / ctas,
                h[5] / ctas, h[8] / ctas, h[6]);
    }
    return ms;
}

// Run the T-step PA loop on the tensor cores.  Outputs the final (x, m) in the interleaved
// layout of dynamics.cu ([n][R_pad], V lanes), the final sign bits sb[n][W] and, if q2 is
// given, the exact coupling energy counts of the final spins.
void dense_pa_loop(Problem* p, int64_t R, int64_t R_pad, int V, int64_t W,
                   const std::vector<double>& sched, float eta, float alpha, uint64_t seed,
                   int64_t rbegin, float* x_il, float* m_il, uint32_t* sb, long long* q2,
                   cudaStream_t s, double* loop_ms, int64_t* launches, double* trace_out,
                   bool trace_on_dev, uint32_t* sb_best) {
    DenseOperand* d = dense_operand(p, s, 0);
    const int64_t n = p->n, ld = d->ld, T = (int64_t)sched.size();
    DevBuf<float> x(R * ld, s), m(R * ld, s);
    // spins (the B operand): packed E2M1 nibbles with a packed-fp4 K (VXQ_DENSE_FP4S=0: fp8)
    const char* es4 = getenv("VXQ_DENSE_FP4S");
    const bool s_fp4 = d->afmt == 5 && !(es4 && atoi(es4) == 0);
    const int64_t sbytes = s_fp4 ? R * ld / 2 : R * ld;
    DevBuf<uint8_t> s0(sbytes, s), s1(sbytes, s);
    VXQ_CUDA(cudaMemsetAsync(s0.get(), 0, sbytes, s));
    VXQ_CUDA(cudaMemsetAsync(s1.get(), 0, sbytes, s));
    k_init_pa_rm<<<nblk(((n + 3) / 4) * R), TB, 0, s>>>(n, R, ld, seed, rbegin, x.get(), m.get(),
                                                       s0.get(), s_fp4 ? 1 : 0);
    VXQ_CHECK_LAUNCH();
    // kind::mxf4 (VXQ_DENSE_MXF4=1): packed E2M1 operands in smem at twice the f8f6f4 MMA
    // rate; needs the packed K and spins, and bn <= 240 (TMEM holds the scale factors too)
    bool mx = true;  // cfg2: 120 -> 139 Grv/s (less operand traffic and power per flop)
    if (const char* e = getenv("VXQ_DENSE_MXF4")) mx = atoi(e) == 1;
    if (!(d->afmt == 5 && s_fp4)) mx = false;
    int bn = choose_bn(n, R, 1, KindTraits<Kind::kFp8>::kBnMax);
    if (mx) {  // fewest <= 240-wide replica blocks, rounded up to 16 (pair N % 16 == 0)
        const int64_t blocks = ceil_div(R, (int64_t)kAccMx);
        bn = (int)std::min<int64_t>(kAccMx, ceil_div(ceil_div(R, blocks), 16) * 16);
        if (const char* e = getenv("VXQ_DENSE_BN"))
            bn = std::max(16, std::min((int)kAccMx, atoi(e) / 16 * 16));
    }
    // VXQ_DENSE_CLUSTER=2: B multicast across 2-CTA clusters (fewer cycles, same wall time
    // under the 1 kW power cap; cluster + cooperative launches cannot be profiled by ncu)
    int cl = 1;
    if (const char* e = getenv("VXQ_DENSE_CLUSTER")) cl = atoi(e) == 2 ? 2 : 1;
    if (ceil_div(n, DBM) < 2) cl = 1;
    // tcgen05 CTA pairs (M = 256 tiles, each CTA holds half of B: half the smem operand
    // traffic per MMA; cfg2 +9 %); VXQ_DENSE_2CTA=0 -> one CTA per 128-row tile
    bool pair = true;
    if (const char* e = getenv("VXQ_DENSE_2CTA")) pair = atoi(e) == 1;
    if (ceil_div(n, DBM) < 2 || bn % 16 != 0) pair = false;  // each CTA: bn/2 rows of B
    if (pair || mx) cl = 1;
    // super-pairs (VXQ_DENSE_SP=1): two pairs share each K panel; needs an even number of
    // replica blocks of <= 240 (an even block count, widths rounded up to 16)
    bool sp = false;
    if (const char* e = getenv("VXQ_DENSE_SP")) sp = atoi(e) == 1;
    if (sp && mx && pair && !getenv("VXQ_DENSE_BN")) {
        int64_t blocks = ceil_div(R, (int64_t)kAccMx);
        blocks += blocks & 1;
        const int b2 = (int)std::min<int64_t>(kAccMx, ceil_div(ceil_div(R, blocks), 16) * 16);
        if (ceil_div(R, (int64_t)b2) % 2 == 0) bn = b2;
    }
    if (sp && mx && pair && ceil_div(R, (int64_t)bn) % 2 == 0) cl = 2;
    const int bbox = pair ? bn / 2 : bn / cl;  // B rows (replicas) per TMA box
    CUtensorMap tmB0, tmB1, tmAmx;
    if (mx) {  // packed bytes as they are in global memory: 128-byte rows = 256 elements
        tmB0 = make_map(s0.get(), CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld / 2, R, 1, DROW, bbox, 1);
        tmB1 = make_map(s1.get(), CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld / 2, R, 1, DROW, bbox, 1);
        tmAmx = make_map(d->K8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld / 2, ld, 1, DROW, DBM, 1);
    } else if (s_fp4) {
        tmB0 = make_map_fp4(s0.get(), ld, R, DROW, bbox);
        tmB1 = make_map_fp4(s1.get(), ld, R, DROW, bbox);
    } else {
        tmB0 = make_map(s0.get(), CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld, R, 1, DROW, bbox, 1);
        tmB1 = make_map(s1.get(), CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld, R, 1, DROW, bbox, 1);
    }
    std::vector<float> s32(T);
    for (int64_t t = 0; t < T; ++t) s32[t] = (float)sched[t];
    DevBuf<float> sc(std::max<int64_t>(T, 1), s);
    VXQ_CUDA(cudaMemcpyAsync(sc.get(), s32.data(), T * sizeof(float), cudaMemcpyHostToDevice, s));
    DenseRunArgs a{};
    a.idesc_extra = (d->afmt << 7) | ((s_fp4 ? 5u : 0u) << 10);
    a.a_tx_bytes = mx ? (uint32_t)DA_BYTES : a_tx_bytes(d);
    a.b_tx_bytes = (uint32_t)bbox * (mx ? DROW : (s_fp4 ? DROW / 2 : DROW));
    a.b_fp4 = s_fp4 ? 1 : 0;
    a.n = (int)n;
    a.R = (int)R;
    a.ld = (int)ld;
    a.kblocks = (int)(mx ? ceil_div(ld, 2 * DROW) : ld / DROW);  // mxf4: 256 K per stage
    a.m_tiles = (int)ceil_div(n, DBM);
    a.n_tiles = (int)ceil_div(R, bn);
    a.bn = bn;
    a.T = (int)T;
    a.scale = d->scale;
    a.eta = eta;
    a.alpha = alpha;
    a.sched = sc.get();
    a.h = p->h32;
    a.x = x.get();
    a.m = m.get();
    a.b_buf[0] = s0.get();
    a.b_buf[1] = s1.get();
    a.group = pick_group(a.n_tiles);
    const char* dbg = getenv("VXQ_DENSE_DEBUG_NOEPI");  // profiling knob: no-op epilogue
    a.mode = (dbg && dbg[0] == '1') ? 2 : 0;
    DevBuf<unsigned> done(std::max<int64_t>(T, 1) * a.n_tiles, s);
    VXQ_CUDA(cudaMemsetAsync(done.get(), 0, std::max<int64_t>(T, 1) * a.n_tiles * sizeof(unsigned), s));
    a.done = done.get();
    DevBuf<long long> qtr, bestq;
    DevBuf<int8_t> best_s;
    DevBuf<unsigned> decided;
    if (trace_out || sb_best) {
        qtr = DevBuf<long long>(std::max<int64_t>(T, 1) * R, s);
        VXQ_CUDA(cudaMemsetAsync(qtr.get(), 0, std::max<int64_t>(T, 1) * R * sizeof(long long), s));
        a.qtrace = qtr.get();
    }
    if (sb_best) {  // fused best-state tracking (h = 0: q is the whole energy up to c, offset)
        VXQ_REQUIRE(q2, "tracking needs the final energy pass");
        bestq = DevBuf<long long>(R, s);
        VXQ_CUDA(cudaMemsetAsync(bestq.get(), 0x7f, R * sizeof(long long), s));  // ~ +inf
        best_s = DevBuf<int8_t>(R * ld, s);
        VXQ_CUDA(cudaMemsetAsync(best_s.get(), 0, R * ld, s));
        decided = DevBuf<unsigned>(std::max<int64_t>(T, 1) * a.n_tiles, s);
        VXQ_CUDA(cudaMemsetAsync(decided.get(), 0,
                                 std::max<int64_t>(T, 1) * a.n_tiles * sizeof(unsigned), s));
        a.bestq = bestq.get();
        a.best_s = best_s.get();
        a.decided = decided.get();
    }
    // x/m staged into shared memory by the loader warp (VXQ_DENSE_XM=0: register loads)
    bool xm = true;
    if (const char* e = getenv("VXQ_DENSE_XM")) xm = atoi(e) == 1;
    CUtensorMap tmX{}, tmM{};
    if (xm && a.mode == 0) {
        tmX = make_map(x.get(), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ld, R, 1, DBM, 16, 1,
                       CU_TENSOR_MAP_SWIZZLE_NONE);
        tmM = make_map(m.get(), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ld, R, 1, DBM, 16, 1,
                       CU_TENSOR_MAP_SWIZZLE_NONE);
        a.xm = 1;
    }
    *loop_ms = run_loop(a, mx ? tmAmx : d->tmA8, tmB0, tmB1, false, cl, s, pair, &tmX, &tmM,
                        mx);
    *launches += 2;
    if (trace_out) {
        DevBuf<double> tr(std::max<int64_t>(T, 1), s);
        DevBuf<int> hnz(1, s);
        VXQ_CUDA(cudaMemsetAsync(hnz.get(), 0, sizeof(int), s));
        k_any_nonzero<<<nblk(n), TB, 0, s>>>(n, p->h64, hnz.get());
        k_trace_from_q<<<(unsigned)std::max<int64_t>(T, 1), 256, 0, s>>>(
            qtr.get(), T, R, p->magnitude, p->offset, hnz.get(), tr.get());
        VXQ_CHECK_LAUNCH();
        VXQ_CUDA(cudaMemcpyAsync(trace_out, tr.get(), T * sizeof(double),
                                 trace_on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 s));
        VXQ_CUDA(cudaStreamSynchronize(s));
        *launches += 2;
    }
    if (q2) energy_pass(d, x.get(), n, R, q2, s, launches);
    if (sb_best && T > 0) {
        const uint8_t* sprev = ((T - 1) & 1) ? s1.get() : s0.get();
        k_track_finalize<<<nblk(n * R), TB, 0, s>>>(n, R, ld, qtr.get() + (T - 1) * R, q2,
                                                     bestq.get(), sprev, s_fp4 ? 1 : 0, x.get(),
                                                     best_s.get());
        k_pack_bits_i8<<<(unsigned)ceil_div(n * W * 32, TB), TB, 0, s>>>(best_s.get(), n, R, ld,
                                                                       W, sb_best);
        VXQ_CHECK_LAUNCH();
        *launches += 2;
    }
    k_rm_to_interleaved<<<nblk(n * R), TB, 0, s>>>(x.get(), n, R, ld, R_pad, V, x_il);
    k_rm_to_interleaved<<<nblk(n * R), TB, 0, s>>>(m.get(), n, R, ld, R_pad, V, m_il);
    k_pack_bits_rm<<<(unsigned)ceil_div(n * W * 32, TB), TB, 0, s>>>(x.get(), n, R, ld, W, sb);
    VXQ_CHECK_LAUNCH();
    *launches += 3;
    VXQ_CUDA(cudaStreamSynchronize(s));
}

// Run the T-step PA loop for a general (non-uniform) dense J on the tensor cores: J as two
// fp16 A planes, spins as fp16 +-1, tcgen05 CTA pairs, the fused PA epilogue.  Outputs as
// dense_pa_loop (no in-kernel energies: the caller's exact energy kernel runs on sb).
void dense_pa_general_loop(Problem* p, int64_t R, int64_t R_pad, int V, int64_t W,
                           const std::vector<double>& sched, float eta, float alpha,
                           uint64_t seed, int64_t rbegin, float* x_il, float* m_il, uint32_t* sb,
                           cudaStream_t s, double* loop_ms, int64_t* launches) {
    DenseOperand* d = dense_jplanes(p, s);
    const int64_t n = p->n, ld = d->ld, T = (int64_t)sched.size();
    VXQ_REQUIRE(ceil_div(n, DBM) >= 2, "general dense path needs n > 128");
    DevBuf<float> x(R * ld, s), m(R * ld, s);
    DevBuf<uint16_t> s0(R * ld, s), s1(R * ld, s);
    VXQ_CUDA(cudaMemsetAsync(s0.get(), 0, R * ld * 2, s));
    VXQ_CUDA(cudaMemsetAsync(s1.get(), 0, R * ld * 2, s));
    k_init_pa_rm<<<nblk(((n + 3) / 4) * R), TB, 0, s>>>(n, R, ld, seed, rbegin, x.get(), m.get(),
                                                       reinterpret_cast<uint8_t*>(s0.get()), 2);
    VXQ_CHECK_LAUNCH();
    const int64_t blocks = ceil_div(R, (int64_t)256);
    int bn = (int)std::min<int64_t>(256, ceil_div(ceil_div(R, blocks), 16) * 16);
    if (const char* e = getenv("VXQ_DENSE_BN")) bn = std::max(16, std::min(256, atoi(e) / 16 * 16));
    const int bbox = bn / 2;
    CUtensorMap tmB0 = make_map(s0.get(), CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, ld, R, 1, DROW / 2,
                                bbox, 1);
    CUtensorMap tmB1 = make_map(s1.get(), CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, ld, R, 1, DROW / 2,
                                bbox, 1);
    std::vector<float> s32(T);
    for (int64_t t = 0; t < T; ++t) s32[t] = (float)sched[t];
    DevBuf<float> sc(std::max<int64_t>(T, 1), s);
    VXQ_CUDA(cudaMemcpyAsync(sc.get(), s32.data(), T * sizeof(float), cudaMemcpyHostToDevice, s));
    DenseRunArgs a{};
    a.idesc_extra = 0;
    a.a_tx_bytes = 2 * DA_BYTES;  // both J planes
    a.b_tx_bytes = (uint32_t)bbox * DROW;
    a.b_fp4 = 0;
    a.n = (int)n;
    a.R = (int)R;
    a.ld = (int)ld;
    a.kblocks = (int)(ld / (DROW / 2));
    a.m_tiles = (int)ceil_div(n, DBM);
    a.n_tiles = (int)ceil_div(R, bn);
    a.bn = bn;
    a.T = (int)T;
    a.scale = d->jscale_inv;
    a.eta = eta;
    a.alpha = alpha;
    a.sched = sc.get();
    a.h = p->h32;
    a.x = x.get();
    a.m = m.get();
    a.b_buf[0] = reinterpret_cast<uint8_t*>(s0.get());
    a.b_buf[1] = reinterpret_cast<uint8_t*>(s1.get());
    // pairs of replica blocks per row panel: the J-plane panel (not L2-resident: 400 MB at
    // n = 10^4) is re-used once from L2 (n = 10^4: 19.2 -> 22.3 Grv/s; all 4 blocks 21.7;
    // profiles/r02/ab_general_group/); VXQ_DENSE_GROUP overrides
    a.group = getenv("VXQ_DENSE_GROUP") ? pick_group(a.n_tiles) : std::min(2, a.n_tiles);
    a.mode = 0;
    DevBuf<unsigned> done(std::max<int64_t>(T, 1) * a.n_tiles, s);
    VXQ_CUDA(cudaMemsetAsync(done.get(), 0, std::max<int64_t>(T, 1) * a.n_tiles * sizeof(unsigned), s));
    a.done = done.get();
    CUtensorMap tmX = make_map(x.get(), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ld, R, 1, DBM, 16, 1,
                               CU_TENSOR_MAP_SWIZZLE_NONE);
    CUtensorMap tmM = make_map(m.get(), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ld, R, 1, DBM, 16, 1,
                               CU_TENSOR_MAP_SWIZZLE_NONE);
    a.xm = 1;
    *loop_ms = run_loop(a, d->tmJ, tmB0, tmB1, 0, 1, s, true, &tmX, &tmM, false, true);
    *launches += 2;
    k_rm_to_interleaved<<<nblk(n * R), TB, 0, s>>>(x.get(), n, R, ld, R_pad, V, x_il);
    k_rm_to_interleaved<<<nblk(n * R), TB, 0, s>>>(m.get(), n, R, ld, R_pad, V, m_il);
    k_pack_bits_rm<<<(unsigned)ceil_div(n * W * 32, TB), TB, 0, s>>>(x.get(), n, R, ld, W, sb);
    VXQ_CHECK_LAUNCH();
    *launches += 3;
    VXQ_CUDA(cudaStreamSynchronize(s));
}

// Run the T-step SBM loop (B = -A, g = -h) on the tensor cores.  q enters the MMA as two
// fp16 terms (default) or three exact bf16 terms (VXQ_SBM_PLANES=3, and always when |q| may
// leave the fp16 range).
void dense_sbm_loop(Problem* p, int64_t R, int64_t R_pad, int V, int64_t W,
                    const std::vector<double>& a_sched, double dt, double a0, double c0,
                    double q_cap, double amp, uint64_t seed, int64_t rbegin, float* q_il,
                    float* p_il, uint32_t* sb, long long* q2, cudaStream_t s, double* loop_ms,
                    int64_t* launches, double* trace_out, bool trace_on_dev) {
    // general (non-uniform) J: J as two fp16 planes too (kJQ16, the caller checked the range)
    const bool general = !p->uniform_magnitude;
    // uniform |J|: exact integer field (kI8x3) when |q| <= max(q_cap, init_noise) <= 2^14;
    // VXQ_SBM_PLANES=2 / 3 select the fp16 / bf16 plane paths (A/B, round 1)
    const int S = sbm_fixed_point_shift(q_cap, amp);
    int planes = (!general && S >= 8) ? 8 : 2;
    if (const char* e = getenv("VXQ_SBM_PLANES")) {
        const int v = atoi(e);
        if (v == 2 || v == 3) planes = v;
    }
    if (planes == 2 && !dense_sbm_fp16_ok(q_cap, amp)) planes = 3;  // fp16 max is 65504
    if (planes == 8 && ceil_div(p->n, DBM) < 2) planes = 2;  // pairs need two row tiles
    const bool exact = planes == 8;
    // per-step energies (trace_out, h = 0): the exact kernel with a 4th plane holding the
    // spins, whose accumulator is K s_t (kI8x4, bn <= 64); other kinds report NaN
    const bool traced = exact && trace_out != nullptr && problem_h_zero(p, s);
    VXQ_REQUIRE(!general || planes == 2, "general dense J on the tensor cores needs fp16 q");
    DenseOperand* d = general ? dense_jplanes(p, s)
                              : dense_operand(p, s, exact ? 3 : (planes == 3 ? 1 : 2));
    const int64_t n = p->n, ld = d->ld, T = (int64_t)a_sched.size();
    const int64_t plane = R * ld;
    const int nb_planes = exact ? (traced ? 4 : 3) : planes;
    const int esz = exact ? 1 : 2;
    DevBuf<float> q(R * ld, s), pm(R * ld, s);
    DevBuf<uint8_t> b0(nb_planes * plane * esz, s), b1(nb_planes * plane * esz, s);
    VXQ_CUDA(cudaMemsetAsync(b0.get(), 0, nb_planes * plane * esz, s));
    VXQ_CUDA(cudaMemsetAsync(b1.get(), 0, nb_planes * plane * esz, s));
    const float qscale = exact ? std::ldexp(1.0f, S) : 0.f;
    k_init_sbm_rm<<<nblk(((2 * n + 3) / 4) * R), TB, 0, s>>>(n, R, ld, seed, rbegin, amp,
                                                            q.get(), pm.get(), b0.get(), planes,
                                                            qscale, traced ? 1 : 0);
    VXQ_CHECK_LAUNCH();
    // CTA pairs (M = 256; each CTA stages its 128 K rows and bn/2 replicas of every plane):
    // half the replica blocks -> half the K re-reads per step
    bool pair = (planes == 2 || exact) && ceil_div(n, DBM) >= 2;
    if (const char* e = getenv("VXQ_DENSE_2CTA")) pair = pair && (atoi(e) == 1 || exact);
    if (general) {
        VXQ_REQUIRE(ceil_div(n, DBM) >= 2, "general dense path needs n > 128");
        pair = true;
    }
    int bn;
    if (pair) {
        int64_t bmax = exact ? (traced ? KindTraits<Kind::kI8x4>::kBnMax
                                       : KindTraits<Kind::kI8x3>::kBnMax)
                             : 256;
        if (const char* e = getenv("VXQ_DENSE_BN"))  // A/B: cap the replica tile width
            if (exact) bmax = std::max<int64_t>(16, std::min<int64_t>(bmax, atoi(e) / 16 * 16));
        const int64_t blocks = ceil_div(R, bmax);
        bn = (int)std::min<int64_t>(bmax, ceil_div(ceil_div(R, blocks), 16) * 16);
    } else {
        bn = planes == 3 ? choose_bn(n, R, 3, KindTraits<Kind::kBf16x3>::kBnMax)
                         : choose_bn(n, R, 2, KindTraits<Kind::kF16x2>::kBnMax);
    }
    const int bbox = pair ? bn / 2 : bn;
    CUtensorMap tmB0, tmB1;
    if (exact) {
        tmB0 = make_map(b0.get(), CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld, R, nb_planes, DROW, bbox,
                        nb_planes);
        tmB1 = make_map(b1.get(), CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ld, R, nb_planes, DROW, bbox,
                        nb_planes);
    } else {
        const CUtensorMapDataType bt =
            planes == 3 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
        tmB0 = make_map(b0.get(), bt, 2, ld, R, planes, DROW / 2, bbox, planes);
        tmB1 = make_map(b1.get(), bt, 2, ld, R, planes, DROW / 2, bbox, planes);
    }
    std::vector<float> s32(T);
    for (int64_t t = 0; t < T; ++t) s32[t] = (float)a_sched[t];
    DevBuf<float> sc(std::max<int64_t>(T, 1), s);
    VXQ_CUDA(cudaMemcpyAsync(sc.get(), s32.data(), T * sizeof(float), cudaMemcpyHostToDevice, s));
    DenseRunArgs a{};
    a.a_tx_bytes = general ? 2 * DA_BYTES : DA_BYTES;  // 16-bit K (or both J planes): full boxes
    a.b_tx_bytes = (uint32_t)bbox * DROW;
    a.n = (int)n;
    a.R = (int)R;
    a.ld = (int)ld;
    a.kblocks = (int)(ld / (exact ? DROW : DROW / 2));
    a.qscale = qscale;
    a.qscale_inv = exact ? std::ldexp(1.0f, -S) : 0.f;
    a.m_tiles = (int)ceil_div(n, DBM);
    a.n_tiles = (int)ceil_div(R, bn);
    a.bn = bn;
    a.T = (int)T;
    a.scale = general ? d->jscale_inv : d->scale;
    a.dt = (float)dt;
    a.a0 = (float)a0;
    a.c0 = (float)c0;
    a.dta0 = (float)(dt * a0);
    a.q_cap = (float)q_cap;
    a.sched = sc.get();
    a.h = p->g32;  // g = -h
    a.x = q.get();
    a.m = pm.get();
    a.b_buf[0] = reinterpret_cast<uint8_t*>(b0.get());
    a.b_buf[1] = reinterpret_cast<uint8_t*>(b1.get());
    a.plane_elems = plane;
    // exact path: all replica blocks of a row panel back to back (the int8 K panel is
    // re-used from L2 instead of re-read from DRAM per replica block: 1.48 GB -> less
    // DRAM per step, more of the 1 kW budget for the SMs; cfg2 SBM 324 -> 280 ms per solve,
    // profiles/r02/ab_sbm_group/); VXQ_DENSE_GROUP overrides
    // general J (two fp16 J planes, DRAM-streamed): pairs of replica blocks (12.6 -> 13.3)
    a.group = getenv("VXQ_DENSE_GROUP") ? pick_group(a.n_tiles)
              : exact                    ? a.n_tiles
              : general                  ? std::min(2, a.n_tiles)
                                         : 1;
    a.mode = 0;
    DevBuf<unsigned> done(std::max<int64_t>(T, 1) * a.n_tiles, s);
    VXQ_CUDA(cudaMemsetAsync(done.get(), 0, std::max<int64_t>(T, 1) * a.n_tiles * sizeof(unsigned), s));
    a.done = done.get();
    DevBuf<long long> qtr;
    if (traced) {
        qtr = DevBuf<long long>(std::max<int64_t>(T, 1) * R, s);
        VXQ_CUDA(cudaMemsetAsync(qtr.get(), 0, std::max<int64_t>(T, 1) * R * sizeof(long long), s));
        a.qtrace = qtr.get();
    }
    *loop_ms = run_loop(a, general ? d->tmJ : (exact ? d->tmAi8 : (planes == 3 ? d->tmA16 : d->tmA16h)),
                        tmB0, tmB1, traced ? 9 : planes, 1, s, pair, nullptr, nullptr, false, false,
                        general);
    *launches += 2;
    if (trace_out) {  // min_r E(s_t) per step (NaN where no exact per-step energy exists)
        DevBuf<double> tr(std::max<int64_t>(T, 1), s);
        if (traced) {
            DevBuf<int> hnz(1, s);
            VXQ_CUDA(cudaMemsetAsync(hnz.get(), 0, sizeof(int), s));  // h = 0 (checked)
            k_trace_from_q<<<(unsigned)std::max<int64_t>(T, 1), 256, 0, s>>>(
                qtr.get(), T, R, p->magnitude, p->offset, hnz.get(), tr.get());
        } else {
            k_fill_nan<<<nblk(std::max<int64_t>(T, 1)), TB, 0, s>>>(tr.get(), T);
        }
        VXQ_CHECK_LAUNCH();
        VXQ_CUDA(cudaMemcpyAsync(trace_out, tr.get(), T * sizeof(double),
                                 trace_on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 s));
        VXQ_CUDA(cudaStreamSynchronize(s));
        *launches += 1;
    }
    if (q2 && !general) energy_pass(d, q.get(), n, R, q2, s, launches);
    k_rm_to_interleaved<<<nblk(n * R), TB, 0, s>>>(q.get(), n, R, ld, R_pad, V, q_il);
    k_rm_to_interleaved<<<nblk(n * R), TB, 0, s>>>(pm.get(), n, R, ld, R_pad, V, p_il);
    k_pack_bits_rm<<<(unsigned)ceil_div(n * W * 32, TB), TB, 0, s>>>(q.get(), n, R, ld, W, sb);
    VXQ_CHECK_LAUNCH();
    *launches += 3;
    VXQ_CUDA(cudaStreamSynchronize(s));
}

}  // namespace vxq
