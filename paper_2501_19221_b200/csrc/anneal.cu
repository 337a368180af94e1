// anneal.cu -- simulated annealing on sm_100a (reference: qubokit/solvers/annealing.py:24-74).
//
// Single-spin-flip Metropolis sweeps in fixed index order, R independent replicas, each
// reporting the best state seen (checked after every sweep, annealing.py:67-70).  The
// reference vectorises across replicas and walks the spins sequentially; so does this:
// one warp owns 32 replicas and visits spin i of all of them in lockstep, which makes the
// per-spin flip mask one ballot and lets the spins live in the library's bit-packed
// layout sb[n][W] (bit r%32 of word r/32 of row i = spin i of replica r), so the exact
// energies / states / order tail is shared with PA and SBM.
//
// Per replica r (numpy stream Philox(key=seed).jumped(r), generators.py:35-40):
//   spins  S_i = 2 * integers(0, 2) - 1  -> top bit of the i-th 32-bit half of the raw
//          draws (low half first; Lemire with range 2 never rejects)
//   U[s,i] = random() = (raw >> 11) * 2^-53 of raw draw ceil(n/2) + s*n + i
//   F      = S @ A + h       (CSR order: ascending column, starting from 0, then + h)
//   dE     = -2 s_i F_i;  accept iff U < exp(min(-dE / T_s, 0))
//   accept: s_i = -s_i; E += dE; F_j += 2 s_i A_ij for j in row i
// fp64 mode reproduces these operations one rounding at a time (exp is CUDA's, within an
// ulp of numpy's: a flip can differ only if U lands inside that ulp); fp32 mode keeps the
// fields in fp32 (bit-exact against the oracle's fp32 restatement).
//
// Fields F live [n][R_pad] (replica-contiguous, coalesced per warp) in HBM/L2 (SPARSE),
// or, when a warp's slice fits, in shared memory for the whole anneal (RESIDENT).
#include <cmath>
#include <vector>

#include "vxq_common.cuh"
#include "vxq_internal.h"

namespace vxq {

namespace {

constexpr int kSaSmemMax = 200 * 1024;
#ifndef VXQ_SA_PF
#define VXQ_SA_PF 8
#endif
constexpr int kPf = VXQ_SA_PF;  // field / spin-word prefetch depth (spins ahead)
constexpr int kB = 8;   // neighbour updates per batch
#ifndef VXQ_SA_BATCH
#define VXQ_SA_BATCH 1
#endif

__global__ void k_sa_init_spins(int64_t n, int64_t W, int64_t R_pad, uint64_t seed,
                                int64_t rbegin, uint32_t* __restrict__ sb) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * R_pad) return;  // whole warps (R_pad % 32 == 0)
    const int64_t i = t / R_pad, r = t % R_pad;
    const uint64_t q = (uint64_t)i >> 1;  // raw draw holding 32-bit half i
    const U64x4 b = philox4x64_10((q >> 2) + 1, 0, (uint64_t)(rbegin + r), 0, seed, 0);
    const uint64_t raw = pick_word(b, (uint32_t)(q & 3));
    const bool up = (i & 1) ? (raw >> 63) != 0 : ((raw >> 31) & 1u) != 0;
    const uint32_t word = __ballot_sync(0xffffffffu, up);
    if ((r & 31) == 0) sb[i * W + (r >> 5)] = word;
}

template <typename T>
__global__ void k_sa_init_fields(int64_t n, int64_t W, int64_t R_pad,
                                 const int64_t* __restrict__ indptr,
                                 const int32_t* __restrict__ indices, const T* __restrict__ data,
                                 const T* __restrict__ h, const uint32_t* __restrict__ sb,
                                 T* __restrict__ F) {
    using O = Ops<T>;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * R_pad) return;
    const int64_t i = t / R_pad, r = t % R_pad, c = r >> 5;
    const int lane = (int)(r & 31);
    T f = (T)0;
    for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
        const int j = indices[e];
        const T v = data[e];
        f = O::add(f, ((sb[j * W + c] >> lane) & 1u) ? v : -v);
    }
    F[i * R_pad + r] = O::add(f, h[i]);
}

__global__ void k_sa_energy0(const double* __restrict__ e, int64_t R, int64_t R_pad,
                             double offset, double* __restrict__ E0) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < R_pad) E0[r] = r < R ? __dsub_rn(e[r], offset) : 0.0;
}

// F_j += v without waiting for the old value: in HBM/L2 a reduction performed at L2
// (one IEEE round-to-nearest add, identical to the separate load + add + store); only this
// lane ever touches its replica's fields, and its later loads of F_j are ordered after it
template <typename T>
__device__ __forceinline__ void red_add_global(T* p, T v) {
    if constexpr (sizeof(T) == 8)
        asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
    else
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

struct SaArgs {
    int64_t n, W, R_pad, sweeps;
    const int64_t* indptr;
    const int32_t* indices;
    const void* data;
    const double* temps;
    uint64_t seed;
    int64_t rbegin;
    void* F;
    uint32_t* sb;
    uint32_t* best_sb;
    const double* E0;
};

// One warp = 32 replicas for the whole anneal.  SMEM: the warp's field slice [n][32] and
// its spin / best words [n] stay in shared memory.
template <typename T, bool SMEM>
__global__ void __launch_bounds__(32) k_sa_run(SaArgs a) {
    using O = Ops<T>;
    extern __shared__ __align__(16) unsigned char sa_smem[];
    const int lane = threadIdx.x;
    const int64_t c = blockIdx.x;
    const int64_t r = c * 32 + lane;
    const int64_t n = a.n;
    const uint64_t rg = (uint64_t)(a.rbegin + r);
    const T* __restrict__ data = static_cast<const T*>(a.data);
    const int64_t* __restrict__ indptr = a.indptr;
    const int32_t* __restrict__ indices = a.indices;

    T* Fb;
    int64_t fs;
    uint32_t* sbw;
    uint32_t* bsw;
    int64_t ws;
    if constexpr (SMEM) {
        T* sF = reinterpret_cast<T*>(sa_smem);
        sbw = reinterpret_cast<uint32_t*>(sF + n * 32);
        bsw = sbw + n;
        const T* Fg = static_cast<const T*>(a.F);
        for (int64_t i = 0; i < n; ++i) sF[i * 32 + lane] = Fg[i * a.R_pad + r];
        for (int64_t i = lane; i < n; i += 32) bsw[i] = sbw[i] = a.sb[i * a.W + c];
        Fb = sF + lane;
        fs = 32;
        ws = 1;
    } else {
        Fb = static_cast<T*>(a.F) + r;
        fs = a.R_pad;
        sbw = a.sb + c;
        bsw = a.best_sb + c;
        ws = a.W;
        for (int64_t i = lane; i < n; i += 32) bsw[i * ws] = sbw[i * ws];
    }
    __syncwarp();

    double E = a.E0[r], bestE = E;
    uint64_t k = (uint64_t)(n + 1) / 2;  // next raw draw (after the n 32-bit spin draws)
    uint64_t kb = ~0ull;
    U64x4 blk{};
    const double inv53 = 1.0 / 9007199254740992.0;
    for (int64_t s = 0; s < a.sweeps; ++s) {
        const double Tt = a.temps[s];
        const double invT = 1.0 / Tt;
        // pf[d] = field of spin i + d (prefetched kPf spins ahead; patched when a flip of
        // spin i updates one of them)
        T pf[kPf];
#pragma unroll
        for (int d = 0; d < kPf; ++d) pf[d] = d < n ? Fb[d * fs] : (T)0;
        // wq[d] = spin word of spin i + d: a spin's word changes only when that spin is
        // visited, so words ahead of i are final for this sweep
        uint32_t wq[kPf];
#pragma unroll
        for (int d = 0; d < kPf; ++d) wq[d] = d < n ? sbw[d * ws] : 0u;
        for (int64_t i = 0; i < n; ++i) {
            const T f = pf[0];
#pragma unroll
            for (int d = 0; d + 1 < kPf; ++d) pf[d] = pf[d + 1];
            pf[kPf - 1] = i + kPf < n ? Fb[(i + kPf) * fs] : (T)0;
            const uint32_t word = wq[0];
#pragma unroll
            for (int d = 0; d + 1 < kPf; ++d) wq[d] = wq[d + 1];
            wq[kPf - 1] = i + kPf < n ? sbw[(i + kPf) * ws] : 0u;
            const uint64_t q = k >> 2;
            if (q != kb) {
                blk = philox4x64_10(q + 1, 0, rg, 0, a.seed, 0);
                kb = q;
            }
            const uint64_t raw = pick_word(blk, (uint32_t)(k & 3));
            ++k;
            const bool up = (word >> lane) & 1u;
            const double dE = up ? -2.0 * (double)f : 2.0 * (double)f;  // -2 s F (exact)
            bool acc = dE <= 0.0;  // x = -dE / T >= 0: exp(min(x, 0)) = 1 > U; NaN: never
            if (dE > 0.0) {
                // U < exp(x), x = RN(-dE / T).  Decided without the fp64 divide and exp
                // unless U falls within 1e-4 (relative) of a fast estimate: |ef / exp(x) - 1|
                // <= ~1.1e-5 for x >= -80 (fp32 cast of x 4.8e-6, __expf <= 94 ulp of fp32,
                // x ~ -dE * (1/T) 3e-16); below -80, exp(x) < 2^-115 < every U > 0
                const double u = __dmul_rn((double)(raw >> 11), inv53);
                const double xa = -dE * invT;
                int verdict = -1;  // 1 accept, 0 reject, -1 undecided
                if (xa >= -80.0) {
                    const float ef = __expf((float)xa);
                    if (u < (double)(ef * 0.9999f)) verdict = 1;
                    else if (u > (double)(ef * 1.0001f)) verdict = 0;
                } else if (u > 0.0) {
                    verdict = 0;
                }
                if (verdict < 0) {
                    const double x = __ddiv_rn(-dE, Tt);
                    acc = x >= 0.0 ? true : u < exp(x);
                } else {
                    acc = verdict == 1;
                }
            }
            const uint32_t am = __ballot_sync(0xffffffffu, acc);
            if (am == 0u) continue;
            if (lane == 0) sbw[i * ws] = word ^ am;
            if (acc) {
                E = __dadd_rn(E, dE);
                const T d2 = up ? (T)-2 : (T)2;  // 2 * s_new
                // kB entries per batch: all index / value / field loads of a batch are
                // issued before its stores (columns within a row are distinct); full
                // batches unpredicated, the tail predicated
                const int64_t nx = i + 1;
                const int64_t e0 = indptr[i], e1 = indptr[i + 1];
                auto patch = [&](int j, T v) {
                    if ((uint64_t)(j - nx) < (uint64_t)kPf) {  // rare
#pragma unroll
                        for (int d = 0; d < kPf; ++d)
                            if (j == nx + d) pf[d] = O::add(pf[d], v);
                    }
                };
                int64_t e = e0;
                if constexpr (!SMEM) {  // fire-and-forget reductions at L2
#if VXQ_SA_BATCH
                    // all index / value loads of a batch before its reductions (the asm
                    // memory clobber of a reduction would otherwise order every later load
                    // behind it: one L2 round trip per neighbour)
                    for (; e < e1; e += kB) {
                        int j[kB];
                        T v[kB];
#pragma unroll
                        for (int u = 0; u < kB; ++u) {
                            const bool ok = e + u < e1;
                            j[u] = ok ? __ldg(indices + e + u) : -1;
                            v[u] = ok ? O::mul(d2, __ldg(data + e + u)) : (T)0;
                        }
#pragma unroll
                        for (int u = 0; u < kB; ++u) {
                            if (j[u] >= 0) {
                                red_add_global(Fb + (int64_t)j[u] * fs, v[u]);
                                patch(j[u], v[u]);
                            }
                        }
                    }
#else
                    for (; e < e1; ++e) {
                        const int j = indices[e];
                        const T v = O::mul(d2, data[e]);
                        red_add_global(Fb + (int64_t)j * fs, v);
                        patch(j, v);
                    }
#endif
                }
                for (; e + kB <= e1; e += kB) {
                    int j[kB];
                    T v[kB], fv[kB];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        j[u] = indices[e + u];
                        v[u] = O::mul(d2, data[e + u]);
                    }
#pragma unroll
                    for (int u = 0; u < kB; ++u) fv[u] = Fb[(int64_t)j[u] * fs];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        Fb[(int64_t)j[u] * fs] = O::add(fv[u], v[u]);
                        patch(j[u], v[u]);
                    }
                }
                if (e < e1) {
                    int j[kB];
                    T v[kB], fv[kB];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        const bool ok = e + u < e1;
                        j[u] = ok ? indices[e + u] : -1;
                        v[u] = ok ? O::mul(d2, data[e + u]) : (T)0;
                    }
#pragma unroll
                    for (int u = 0; u < kB; ++u)
                        if (j[u] >= 0) fv[u] = Fb[(int64_t)j[u] * fs];
#pragma unroll
                    for (int u = 0; u < kB; ++u) {
                        if (j[u] >= 0) {
                            Fb[(int64_t)j[u] * fs] = O::add(fv[u], v[u]);
                            patch(j[u], v[u]);
                        }
                    }
                }
            }
        }
        // best state seen, checked after each sweep (annealing.py:67-70)
        const bool imp = E < bestE;
        if (imp) bestE = E;
        const uint32_t im = __ballot_sync(0xffffffffu, imp);
        __syncwarp();
        if (im)
            for (int64_t i = lane; i < n; i += 32)
                bsw[i * ws] = (bsw[i * ws] & ~im) | (sbw[i * ws] & im);
        __syncwarp();
    }
    if constexpr (SMEM) {
        for (int64_t i = lane; i < n; i += 32) a.best_sb[i * a.W + c] = bsw[i];
    }
}

template <typename T>
size_t sa_smem_bytes(int64_t n) {
    return (size_t)n * (32 * sizeof(T) + 2 * sizeof(uint32_t));
}

template <typename T>
void sa_solve_t(Problem* p, const vxq_sa_params* prm, const vxq_run_opts* opts,
                vxq_outputs* out, cudaStream_t s) {
    const int64_t n = p->n, R = prm->replicas, S = prm->sweeps;
    const int64_t R_pad = ceil_div(R, 32) * 32, W = R_pad / 32;
    const int64_t rbegin = opts ? opts->replica_begin : 0;
    // temperatures (annealing.py:29-35)
    double T0 = prm->T_init, T1 = prm->T_final;
    if (std::isnan(T0)) T0 = 2.0 * problem_lambda0(p, s);
    if (std::isnan(T1)) T1 = 1e-3 * T0;
    out->lambda0_used = T0;
    out->c0_used = T1;
    std::vector<double> temps(S);
    if (prm->temps) std::copy(prm->temps, prm->temps + S, temps.begin());
    else sa_schedule(T0, T1, S, temps.data());
    DevBuf<double> dtemps(S, s);
    VXQ_CUDA(cudaMemcpyAsync(dtemps.get(), temps.data(), S * sizeof(double),
                             cudaMemcpyHostToDevice, s));

    DevBuf<uint32_t> sb(n * W, s), best_sb(n * W, s);
    DevBuf<T> F(n * R_pad, s);
    DevBuf<double> e(R, s), E0(R_pad, s);
    int64_t launches = 0;
    const int TBk = 256;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, ceil_div(n * R_pad, TBk));
    k_sa_init_spins<<<blocks, TBk, 0, s>>>(n, W, R_pad, prm->seed, rbegin, sb.get());
    const T* data;
    const T* h;
    if constexpr (sizeof(T) == 8) {
        data = reinterpret_cast<const T*>(p->data64);
        h = reinterpret_cast<const T*>(p->h64);
    } else {
        data = reinterpret_cast<const T*>(p->data32);
        h = reinterpret_cast<const T*>(p->h32);
    }
    k_sa_init_fields<T><<<blocks, TBk, 0, s>>>(n, W, R_pad, p->indptr, p->indices, data, h,
                                               sb.get(), F.get());
    VXQ_CHECK_LAUNCH();
    energies_from_bits(p, sb.get(), W, R, e.get(), s);  // E = energies(S) - offset
    k_sa_energy0<<<(unsigned)ceil_div(R_pad, 256), 256, 0, s>>>(e.get(), R, R_pad, p->offset,
                                                               E0.get());
    VXQ_CHECK_LAUNCH();
    launches += 4;

    const size_t smem = sa_smem_bytes<T>(n);
    const int req = opts ? opts->path : VXQ_PATH_AUTO;
    if (req == VXQ_PATH_DENSE) throw Error(VXQ_ERR_UNSUPPORTED, "SA has no dense path");
    if (req == VXQ_PATH_RESIDENT && smem > (size_t)kSaSmemMax)
        throw Error(VXQ_ERR_UNSUPPORTED, "resident SA: fields do not fit shared memory");
    const bool resident = req != VXQ_PATH_SPARSE && smem <= (size_t)kSaSmemMax;

    SaArgs a;
    a.n = n;
    a.W = W;
    a.R_pad = R_pad;
    a.sweeps = S;
    a.indptr = p->indptr;
    a.indices = p->indices;
    a.data = data;
    a.temps = dtemps.get();
    a.seed = prm->seed;
    a.rbegin = rbegin;
    a.F = F.get();
    a.sb = sb.get();
    a.best_sb = best_sb.get();
    a.E0 = E0.get();
    EventTimer tm(s);
    tm.start();
    if (resident) {
        VXQ_CUDA(cudaFuncSetAttribute(k_sa_run<T, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, kSaSmemMax));
        k_sa_run<T, true><<<(unsigned)W, 32, smem, s>>>(a);
    } else {
        k_sa_run<T, false><<<(unsigned)W, 32, 0, s>>>(a);
    }
    VXQ_CHECK_LAUNCH();
    tm.stop();
    ++launches;
    out->loop_ms = tm.ms();
    out->path_used = resident ? VXQ_PATH_RESIDENT : VXQ_PATH_SPARSE;
    out->step_kernel = VXQ_KERNEL_SA_RUN;
    finish_from_bits(p, R, W, best_sb.get(), opts, out, s);
    out->launches = launches + 4;
}

}  // namespace

void sa_schedule(double T_init, double T_final, int64_t sweeps, double* out) {
    if (sweeps <= 0) return;
    if (sweeps == 1) {
        out[0] = T_init;
        return;
    }
    const double ratio = std::pow(T_final / T_init, 1.0 / (double)(sweeps - 1));
    for (int64_t k = 0; k < sweeps; ++k) out[k] = T_init * std::pow(ratio, (double)k);
}

void sa_solve(Problem* p, const vxq_sa_params* prm, const vxq_run_opts* opts, vxq_outputs* out,
              cudaStream_t s) {
    VXQ_REQUIRE(out->energy_trace == nullptr, "energy_trace is not available for SA");
    if (opts && opts->precision == VXQ_FP64) sa_solve_t<double>(p, prm, opts, out, s);
    else sa_solve_t<float>(p, prm, opts, out, s);
}

}  // namespace vxq
