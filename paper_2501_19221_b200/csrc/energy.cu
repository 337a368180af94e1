// energy.cu -- exact batch energies (replaces IsingModel.energies, model.py:160-164,
// as used by make_sampleset, solvers/common.py:48-61).
//
// H(s) = offset + sum_{i<j} J_ij s_i s_j + sum_i h_i s_i.  Every term is +-coefficient,
// so the sum is carried exactly in a fixed-point integer with LSB 2^e_low (the lowest set
// bit over all coefficients): each coefficient is pre-encoded as L 32-bit
// two's-complement limbs, every term adds +-limb_q into an int64 accumulator per limb
// (no overflow for < 2^31 terms), and the total is rounded ONCE to fp64 (round half to
// even).  The result is the correctly rounded exact energy == math.fsum of the terms.
//
// Spins arrive bit-packed as sb[n][W]: bit (r % 32) of word r / 32 is 1 for s = +1.
// A warp owns 32 replicas (one word column) and streams the couplings: the two spin words
// and the coefficient limbs are warp-uniform loads; lane l adds +-coef for replica 32w+l.
#include <cub/cub.cuh>

#include <algorithm>

#include "vxq_internal.h"

namespace vxq {
namespace {

constexpr int EB = 256;  // threads per block (8 warps)

// Partial sums: block (word w, split) -> partial[split][r][L+1] (limbs, then a coupling
// count).  COUNT: all |J_ij| are equal (uniform magnitude c): couplings add sign(J_ij)*s_i*s_j
// to an integer count folded in as count * c at the end; otherwise each coupling adds
// +-limbs.  m_used = 0 skips the couplings entirely (count supplied by the caller).
template <int L, bool COUNT>
__global__ void __launch_bounds__(EB) k_energy_partial(
    int64_t m_used, int64_t n, const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
    const uint32_t* __restrict__ coef_fx, const uint32_t* __restrict__ h_fx,
    const uint32_t* __restrict__ sb, int64_t W, int64_t R, long long* __restrict__ partial) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w = blockIdx.x;
    const int64_t split = blockIdx.y, nsplit = gridDim.y;
    long long acc[L];
    long long cnt = 0;
#pragma unroll
    for (int q = 0; q < L; ++q) acc[q] = 0;
    constexpr int U = 4;  // couplings per warp iteration (loads batched for MLP)
    const int64_t stride = nsplit * (EB / 32) * U;
    for (int64_t k0 = (split * (EB / 32) + warp) * U; k0 < m_used; k0 += stride) {
        int32_t ii[U], jj[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t k = k0 + u < m_used ? k0 + u : m_used - 1;
            ii[u] = __ldg(ci + k);
            jj[u] = __ldg(cj + k);
        }
        uint32_t wi[U], wj[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            wi[u] = __ldg(sb + (int64_t)ii[u] * W + w);
            wj[u] = __ldg(sb + (int64_t)jj[u] * W + w);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (k0 + u >= m_used) break;
            const bool pos = ((~(wi[u] ^ wj[u])) >> lane) & 1u;  // s_i s_j = +1
            const uint32_t* c = coef_fx + (k0 + u) * L;
            if constexpr (COUNT) {
                const bool neg = (int32_t)__ldg(c + L - 1) < 0;
                cnt += (pos != neg) ? 1 : -1;
            } else {
#pragma unroll
                for (int q = 0; q < L; ++q) {
                    const uint32_t limb = __ldg(c + q);
                    const long long v = (q == L - 1) ? (long long)(int32_t)limb : (long long)limb;
                    acc[q] += pos ? v : -v;
                }
            }
        }
    }
    // fields: sum_i h_i s_i
    const int64_t fstride = nsplit * (EB / 32);
    for (int64_t i = split * (EB / 32) + warp; i < n; i += fstride) {
        const bool pos = (__ldg(sb + i * W + w) >> lane) & 1u;
        const uint32_t* c = h_fx + i * L;
#pragma unroll
        for (int q = 0; q < L; ++q) {
            const uint32_t limb = __ldg(c + q);
            const long long v = (q == L - 1) ? (long long)(int32_t)limb : (long long)limb;
            acc[q] += pos ? v : -v;
        }
    }
    __shared__ long long sh[EB / 32][32][L + 1];
#pragma unroll
    for (int q = 0; q < L; ++q) sh[warp][lane][q] = acc[q];
    sh[warp][lane][L] = cnt;
    __syncthreads();
    if (warp == 0) {
        const int64_t r = w * 32 + lane;
#pragma unroll
        for (int q = 0; q <= L; ++q) {
            long long t = 0;
            for (int ww = 0; ww < EB / 32; ++ww) t += sh[ww][lane][q];
            if (r < R) partial[(split * R + r) * (L + 1) + q] = t;
        }
    }
}

__device__ uint64_t get_bits(const uint32_t* mag, int nl, int pos, int cnt) {
    // bits [pos, pos+cnt) of the little-endian limb array, cnt <= 64
    uint64_t r = 0;
    for (int b = 0; b < cnt; b += 32) {
        int p = pos + b;
        int q = p >> 5, sh = p & 31;
        uint64_t lo = (q < nl) ? mag[q] : 0, hi = (q + 1 < nl) ? mag[q + 1] : 0;
        uint64_t chunk = ((hi << 32) | lo) >> sh;
        r |= (chunk & 0xffffffffULL) << b;
    }
    if (cnt < 64) r &= ((1ULL << cnt) - 1);
    return r;
}

struct FxConst {
    uint32_t off[kMaxLimbs];  // offset
    uint32_t mag[kMaxLimbs];  // +|J| (uniform-magnitude problems)
};

__global__ void k_energy_final(int64_t R, int L, int nsplit, const long long* partial,
                               const long long* q2, FxConst fx, int e_low, double* out) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= R) return;
    long long cnt = q2 ? q2[r] / 2 : 0;
    for (int s = 0; s < nsplit; ++s) cnt += partial[((int64_t)s * R + r) * (L + 1) + L];
    long long acc[kMaxLimbs];
    for (int q = 0; q < L; ++q) {
        long long v = (q == L - 1) ? (long long)(int32_t)fx.off[q] : (long long)fx.off[q];
        for (int s = 0; s < nsplit; ++s) v += partial[((int64_t)s * R + r) * (L + 1) + q];
        const long long mg = (q == L - 1) ? (long long)(int32_t)fx.mag[q] : (long long)fx.mag[q];
        acc[q] = v + cnt * mg;  // |cnt| < 2^31, |mg| < 2^32
    }
    // normalise into L+2 two's-complement 32-bit limbs
    uint32_t d[kMaxLimbs + 2];
    long long carry = 0;
    for (int q = 0; q < L; ++q) {
        long long t = acc[q] + carry;
        d[q] = (uint32_t)t;
        carry = t >> 32;  // arithmetic shift = floor division
    }
    d[L] = (uint32_t)carry;
    d[L + 1] = (uint32_t)(carry >> 32);
    const int nl = L + 2;
    bool neg = ((int32_t)d[nl - 1]) < 0;
    if (neg) {
        uint64_t c = 1;
        for (int q = 0; q < nl; ++q) {
            uint64_t t = (uint64_t)(uint32_t)~d[q] + c;
            d[q] = (uint32_t)t;
            c = t >> 32;
        }
    }
    int top = nl - 1;
    while (top >= 0 && d[top] == 0) --top;
    double res = 0.0;
    if (top >= 0) {
        int B = 32 * top + (32 - __clz(d[top]));  // bit length
        if (B <= 53) {
            uint64_t v = get_bits(d, nl, 0, B);
            res = ldexp((double)v, e_low);
        } else {
            int shift = B - 54;
            uint64_t T = get_bits(d, nl, shift, 54);
            bool sticky = false;
            for (int q = 0; q < nl && 32 * q < shift; ++q) {
                int hi_bit = 32 * q + 32;
                uint32_t mask = hi_bit <= shift ? 0xffffffffu : ((1u << (shift - 32 * q)) - 1u);
                if (d[q] & mask) sticky = true;
            }
            uint64_t mant = T >> 1;
            bool rb = T & 1ULL;
            if (rb && (sticky || (mant & 1ULL))) mant += 1;
            res = ldexp((double)mant, shift + 1 + e_low);
        }
    }
    out[r] = neg ? -res : res;
}

__global__ void k_pack_states(const int8_t* __restrict__ st, int64_t n, int64_t R, int64_t W,
                              uint32_t* __restrict__ sb) {
    // one warp per (i, word): lane l reads replica 32w+l
    int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (gw >= n * W) return;
    int64_t i = gw / W, w = gw % W;
    int64_t r = w * 32 + lane;
    bool up = (r < R) ? (st[r * n + i] >= 0) : true;
    uint32_t word = __ballot_sync(0xffffffffu, up);
    if (lane == 0) sb[i * W + w] = word;
}

__global__ void k_bits_to_states(const uint32_t* __restrict__ sb, int64_t n, int64_t R,
                                 int64_t W, int8_t* __restrict__ st) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * R) return;
    int64_t r = idx / n, i = idx % n;
    uint32_t word = __ldg(sb + i * W + (r >> 5));
    st[idx] = ((word >> (r & 31)) & 1u) ? (int8_t)1 : (int8_t)-1;
}

__global__ void k_iota64(int64_t R, int64_t* v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < R) v[i] = i;
}

template <int L>
void launch_partial(Problem* p, int64_t m_used, bool count, const uint32_t* sb, int64_t W,
                    int64_t R, int nsplit, long long* partial, cudaStream_t s) {
    dim3 grid((unsigned)W, (unsigned)nsplit);
    if (count)
        k_energy_partial<L, true><<<grid, EB, 0, s>>>(m_used, p->n, p->coo_i, p->coo_j,
                                                      p->coef_fx, p->h_fx, sb, W, R, partial);
    else
        k_energy_partial<L, false><<<grid, EB, 0, s>>>(m_used, p->n, p->coo_i, p->coo_j,
                                                       p->coef_fx, p->h_fx, sb, W, R, partial);
    VXQ_CHECK_LAUNCH();
}

}  // namespace

void energies_from_bits(Problem* p, const uint32_t* sb, int64_t W, int64_t R,
                        double* energies_dev, cudaStream_t s, const long long* q2) {
    if (!p->energy_ok)
        throw Error(VXQ_ERR_UNSUPPORTED,
                    "coefficient dynamic range exceeds the exact accumulator (256 bits)");
    const int L = p->limbs;
    const int64_t m_used = q2 ? 0 : p->m;
    const bool count = p->uniform_magnitude && !q2;
    const int64_t terms = m_used + p->n;
    // enough blocks to fill 148 SMs several times, each split >= 4096 terms
    int64_t want = std::max<int64_t>(1, (148 * 8) / std::max<int64_t>(W, 1));
    int64_t maxs = std::max<int64_t>(1, terms / 4096);
    int nsplit = (int)std::min<int64_t>(std::min<int64_t>(want, maxs), 65535);
    DevBuf<long long> partial((size_t)nsplit * R * (L + 1), s);
    switch (L) {
        case 2: launch_partial<2>(p, m_used, count, sb, W, R, nsplit, partial.get(), s); break;
        case 3: launch_partial<3>(p, m_used, count, sb, W, R, nsplit, partial.get(), s); break;
        case 4: launch_partial<4>(p, m_used, count, sb, W, R, nsplit, partial.get(), s); break;
        case 5: launch_partial<5>(p, m_used, count, sb, W, R, nsplit, partial.get(), s); break;
        case 6: launch_partial<6>(p, m_used, count, sb, W, R, nsplit, partial.get(), s); break;
        case 7: launch_partial<7>(p, m_used, count, sb, W, R, nsplit, partial.get(), s); break;
        default: launch_partial<8>(p, m_used, count, sb, W, R, nsplit, partial.get(), s); break;
    }
    FxConst fx;
    for (int q = 0; q < kMaxLimbs; ++q) {
        fx.off[q] = p->offset_fx[q];
        fx.mag[q] = p->mag_fx[q];
    }
    k_energy_final<<<(unsigned)ceil_div(R, 128), 128, 0, s>>>(R, L, nsplit, partial.get(), q2,
                                                              fx, p->e_low, energies_dev);
    VXQ_CHECK_LAUNCH();
}

void pack_states_to_bits(const int8_t* states_dev, int64_t n, int64_t R, int64_t W,
                         uint32_t* sb, cudaStream_t s) {
    int64_t threads = n * W * 32;
    k_pack_states<<<(unsigned)ceil_div(threads, 256), 256, 0, s>>>(states_dev, n, R, W, sb);
    VXQ_CHECK_LAUNCH();
}

void bits_to_states(const uint32_t* sb, int64_t n, int64_t R, int64_t W, int8_t* states_dev,
                    cudaStream_t s) {
    int64_t tot = n * R;
    k_bits_to_states<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(sb, n, R, W, states_dev);
    VXQ_CHECK_LAUNCH();
}

void stable_order(const double* energies_dev, int64_t R, int64_t* order_dev, cudaStream_t s) {
    DevBuf<int64_t> iota(R, s);
    DevBuf<double> keys_out(R, s);
    k_iota64<<<(unsigned)ceil_div(R, 256), 256, 0, s>>>(R, iota.get());
    VXQ_CHECK_LAUNCH();
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, energies_dev, keys_out.get(), iota.get(),
                                    order_dev, (int)R, 0, 64, s);
    DevBuf<uint8_t> tmp(std::max<size_t>(need, 1), s);
    VXQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), need, energies_dev, keys_out.get(),
                                             iota.get(), order_dev, (int)R, 0, 64, s));
}

}  // namespace vxq
