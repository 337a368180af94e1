// dense_tc.cu -- dense J.S coupling field on the 5th-gen tensor cores, PA integrator fused.
//
// Replaces `sign_pm(X).astype(f64) @ A` + the PA update (parallel_annealing.py:42-45) for
// dense couplings with a uniform magnitude |J_ij| = c (e.g. Sherrington-Kirkpatrick,
// BASELINE config 2): J = c * K with K in {-1, 0, +1} and spins in {-1, +1} are exact in
// FP8 E4M3, and the f32 TMEM accumulator holds the integer K.s exactly (|K.s| < 2^24), so
// the field f = c * (K.s) carries a single rounding.
//
// One launch per dynamics step (the step-to-step dependency is grid-wide):
//   F^T[i, r] = sum_j K[i, j] S[r, j]      M = n rows (i), N = replicas (r), K = n
//   A = K  [n_pad][n_pad] fp8, K-major      (TMA, SWIZZLE_128B, 128 x 128 B boxes)
//   B = S  [R][n_pad]    fp8, K-major      (TMA, SWIZZLE_128B, 256 x 128 B boxes)
//   D in TMEM: 128 lanes (rows i) x 256 f32 columns (replicas r), double-buffered
// Persistent warp-specialised CTA (1 per SM, 320 threads):
//   warp 0  TMA producer        4-stage smem ring (48 KB / stage)
//   warp 1  MMA issuer          one elected thread: 4 x tcgen05.mma (K = 32) per stage
//   warps 2-9 epilogue          tcgen05.ld -> PA update of (x, m) in HBM -> next S (fp8)
// The epilogue of tile t overlaps the mainloop of tile t+1 (2 TMEM accumulators).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "tc_ptx.cuh"
#include "vxq_internal.h"

namespace vxq {

constexpr int DBM = 128;       // rows (i) per tile
constexpr int DBN = 256;       // max replicas (r) per tile; the run picks bn <= DBN
constexpr int DBK = 128;       // K bytes (fp8 elements) per stage
constexpr int DSTAGES = 4;
constexpr int DA_BYTES = DBM * DBK;
constexpr int DB_BYTES = DBN * DBK;
constexpr int DSTAGE_BYTES = DA_BYTES + DB_BYTES;
constexpr int DSMEM = DSTAGES * DSTAGE_BYTES + 1024 + 256;
constexpr int DTHREADS = 320;  // TMA warp, MMA warp, 8 epilogue warps
constexpr uint8_t FP8_P1 = 0x38, FP8_M1 = 0xB8;  // E4M3 +1 / -1

struct DenseOperand {
    int64_t n = 0, ld = 0;  // ld = n_pad (multiple of 128)
    uint8_t* K = nullptr;   // [ld][ld] fp8 E4M3 in {-1, 0, +1}
    float scale = 0.f;      // c (fp32)
    CUtensorMap tmA;
    ~DenseOperand() {
        if (K) cudaFree(K);
    }
};

void dense_destroy(DenseOperand* d) { delete d; }

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

// 2-D uint8 tensor [outer][inner] with row pitch `pitch` bytes, SW128 boxes
CUtensorMap make_map_u8(const void* base, uint64_t inner, uint64_t outer, uint64_t pitch,
                        uint32_t box_inner, uint32_t box_outer) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {pitch};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base),
                              dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(VXQ_ERR_CUDA, "cuTensorMapEncodeTiled failed");
    return m;
}

__global__ void k_build_sign_matrix(int64_t n, int64_t ld, const int64_t* __restrict__ indptr,
                                    const int32_t* __restrict__ indices,
                                    const double* __restrict__ data, uint8_t* __restrict__ K) {
    int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    for (int64_t k = indptr[row] + lane; k < indptr[row + 1]; k += 32)
        K[row * ld + indices[k]] = data[k] > 0 ? FP8_P1 : FP8_M1;
}

__device__ __forceinline__ int64_t pos_interleaved(int64_t r, int V) {
    int64_t ch = 32 * V;
    int64_t c = r / ch, rem = r % ch;
    return c * ch + (rem % 32) * V + rem / 32;
}

// x0 ~ uniform(-1, 1) from replica stream r (same draws as k_init_pa), row-major [R][ld]
__global__ void k_init_pa_rm(int64_t n, int64_t R, int64_t ld, uint64_t seed, int64_t rbegin,
                             float* __restrict__ x, float* __restrict__ m,
                             uint8_t* __restrict__ s) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t nq = (n + 3) / 4;
    if (idx >= nq * R) return;
    int64_t r = idx / nq, q = idx % nq;
    U64x4 o = philox4x64_10((uint64_t)q + 1, 0, (uint64_t)(rbegin + r), 0, seed, 0);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        int64_t i = 4 * q + w;
        if (i < n) {
            float v = (float)uniform_from_raw(o.v[w], -1.0, 2.0);
            x[r * ld + i] = v;
            m[r * ld + i] = 0.f;
            s[r * ld + i] = v >= 0.f ? FP8_P1 : FP8_M1;
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

struct DenseRunArgs {
    int n, R, ld, kblocks, m_tiles, n_tiles, bn;
    int T;                   // dynamics steps covered by this launch
    float scale, eta, alpha;
    const float* lam;        // [T] lambda_t (fp32)
    const float* h;
    float* x;
    float* m;
    uint8_t* s_buf[2];       // S_t lives in s_buf[t & 1]; step t writes s_buf[(t+1) & 1]
    int mode;                // 0: PA steps, 1: energy pass over S_0 (q2), 2: no-op epilogue
    long long* q2;           // [R] 2 * sum_{i<j} K_ij s_i s_j  (mode 1)
    unsigned* done;          // [T][n_tiles] finished row-tiles per (step, replica block)
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Persistent dataflow kernel over all T steps.  Tiles are enumerated (step, replica block
// nb, row block mb) and dealt round-robin to the CTAs (1 per SM).  A tile of step t reads
// S_t[nb block] and x/m of (nb, mb), all produced by step t-1 tiles of the same replica
// block, so it only waits for done[t-1][nb] == m_tiles: the tail of step t-1 overlaps the
// head of step t and there is no per-step launch, prologue or wave quantisation.
__global__ void __launch_bounds__(DTHREADS, 1)
    k_dense_pa_run(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB0,
                   const __grid_constant__ CUtensorMap tmB1, DenseRunArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + DSTAGES * DSTAGE_BYTES);
    uint64_t* empty = full + DSTAGES;
    uint64_t* tfull = empty + DSTAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < DSTAGES; ++s) {
            ptx::mbar_init(full + s, 1);
            ptx::mbar_init(empty + s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(tfull + s, 1);
            ptx::mbar_init(tempty + s, 256);
        }
        ptx::fence_mbar_init();
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB0);
        ptx::tma_prefetch(&tmB1);
    }
    if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int tps = a.m_tiles * a.n_tiles;  // tiles per step
    const int num_tiles = tps * a.T;

    if (warp == 0) {
        // ---------------- TMA producer
        if (ptx::elect_one()) {
            // J (100 MB at n = 10^4) and S stay L2-resident across steps; x/m stream past
            const uint64_t keep = ptx::policy_evict_last();
            int stage = 0;
            uint32_t ph = 0;
            for (int g = blockIdx.x; g < num_tiles; g += gridDim.x) {
                const int t = g / tps, rem = g % tps;
                const int nb = rem / a.m_tiles, mb = rem % a.m_tiles;
                const CUtensorMap* tmB = (t & 1) ? &tmB1 : &tmB0;
                for (int kb = 0; kb < a.kblocks; ++kb) {
                    ptx::mbar_wait(empty + stage, ph ^ 1);
                    uint8_t* sa = smem + stage * DSTAGE_BYTES;
                    ptx::mbar_arrive_expect_tx(full + stage, DA_BYTES + a.bn * DBK);
                    ptx::tma_load_2d_hint(sa, &tmA, full + stage, kb * DBK, mb * DBM, keep);
                    if (kb == 0 && t > 0) {
                        // S_t[nb] complete? (release/acquire on the step t-1 counter, then a
                        // proxy fence so the async-proxy TMA sees the generic-proxy stores)
                        const unsigned* cnt = a.done + (size_t)(t - 1) * a.n_tiles + nb;
                        if (ld_acquire_gpu(cnt) < (unsigned)a.m_tiles) {
                            uint64_t t0, tn;
                            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                            while (ld_acquire_gpu(cnt) < (unsigned)a.m_tiles) {
                                __nanosleep(64);
                                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                                if (tn - t0 > 10ull * 1000 * 1000 * 1000) __trap();
                            }
                        }
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    ptx::tma_load_2d_hint(sa + DA_BYTES, tmB, full + stage, kb * DBK,
                                          nb * a.bn, keep);
                    if (++stage == DSTAGES) {
                        stage = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (single thread issues for the CTA)
        // idesc: D=F32, A=B=E4M3, K-major both, N=bn, M=128
        const uint32_t idesc =
            (1u << 4) | ((uint32_t)(a.bn >> 3) << 17) | ((uint32_t)(DBM >> 4) << 24);
        int stage = 0;
        uint32_t ph = 0;
        int lt = 0;
        for (int g = blockIdx.x; g < num_tiles; g += gridDim.x, ++lt) {
            const int acc = lt & 1;
            const uint32_t acc_ph = (lt >> 1) & 1;
            ptx::mbar_wait(tempty + acc, acc_ph ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem_base + acc * DBN;
            for (int kb = 0; kb < a.kblocks; ++kb) {
                ptx::mbar_wait(full + stage, ph);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t sa = ptx::smem_u32(smem + stage * DSTAGE_BYTES);
                    const uint64_t da = ptx::sw128_kmajor_desc(sa);
                    const uint64_t db = ptx::sw128_kmajor_desc(sa + DA_BYTES);
#pragma unroll
                    for (int k = 0; k < DBK / 32; ++k)  // K = 32 fp8 per MMA = 32 B = 2 x 16 B
                        ptx::mma_f8f6f4(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                    ptx::mma_commit(empty + stage);
                }
                __syncwarp();
                if (++stage == DSTAGES) {
                    stage = 0;
                    ph ^= 1;
                }
            }
            if (ptx::elect_one()) ptx::mma_commit(tfull + acc);
            __syncwarp();
        }
    } else {
        // ---------------- epilogue (8 warps): TMEM -> PA update -> next spins
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
        int lt = 0;
        for (int g = blockIdx.x; g < num_tiles; g += gridDim.x, ++lt) {
            const int t = g / tps, rem = g % tps;
            const int nb = rem / a.m_tiles, mb = rem % a.m_tiles;
            const int acc = lt & 1;
            const uint32_t acc_ph = (lt >> 1) & 1;
            const int i = mb * DBM + row;
            const bool row_ok = i < a.n;
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * DBN;
            ptx::mbar_wait(tfull + acc, acc_ph);
            ptx::tc_fence_after();
            if (a.mode == 0) {
                const uint64_t stream = ptx::policy_evict_first();
                uint8_t* __restrict__ sg = (t & 1) ? a.s_buf[0] : a.s_buf[1];  // S_{t+1}
                const float lam = __ldg(a.lam + t);
                const float hi = row_ok ? __ldg(a.h + i) : 0.f;
#pragma unroll 1
                for (int c = half; c < nch; c += 2) {
                    uint32_t v[16];
                    ptx::tmem_ld_32x32b_x16(tbase + c * 16, v);
                    const int r0 = nb * a.bn + c * 16;
                    const int64_t base = (int64_t)r0 * a.ld + i;
                    float xo[16], mo[16];
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {  // L2 (cg): written by another SM
                        const bool ok = row_ok && (r0 + jj) < a.R;
                        xo[jj] = ok ? ptx::ld_stream(xg + base + (int64_t)jj * a.ld, stream) : 0.f;
                        mo[jj] = ok ? ptx::ld_stream(mg + base + (int64_t)jj * a.ld, stream) : 0.f;
                    }
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const bool ok = row_ok && (r0 + jj) < a.R;
                        const float f = O::mul(a.scale, __uint_as_float(v[jj]));
                        const float grad = O::add(O::add(O::mul(lam, xo[jj]), f), hi);
                        const float mn = O::sub(O::mul(a.alpha, mo[jj]), O::mul(a.eta, grad));
                        float xn = O::add(xo[jj], mn);
                        xn = xn < -1.f ? -1.f : (xn > 1.f ? 1.f : xn);
                        if (ok) {
                            const int64_t off = base + (int64_t)jj * a.ld;
                            ptx::st_stream(xg + off, xn, stream);
                            ptx::st_stream(mg + off, mn, stream);
                            sg[off] = xn >= 0.f ? FP8_P1 : FP8_M1;
                        }
                    }
                }
            } else if (a.mode == 1) {
                // energy pass: 2 q_r = sum_i s_i (K s)_i, exact integers
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
            ptx::tc_fence_before();
            ptx::mbar_arrive(tempty + acc);
            if (a.mode == 0 && t + 1 < a.T) {
                // publish: all 256 epilogue threads' stores, then one release increment
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (ep_tid == 0) {
                    __threadfence();
                    atomicAdd(a.done + (size_t)t * a.n_tiles + nb, 1u);
                }
            }
        }
    }
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc<512>(tmem_base);
}

constexpr int TB = 256;
inline unsigned nblk(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, TB)); }

}  // namespace

bool dense_eligible(const Problem* p, int64_t R) {
    if (!p->uniform_magnitude || p->n < 256 || R < 128) return false;
    double density = (double)p->nnz / ((double)p->n * (double)p->n);
    return density >= 0.25;
}

DenseOperand* dense_operand(Problem* p, cudaStream_t s) {
    std::lock_guard<std::mutex> g(p->mu);
    if (p->dense) return p->dense;
    if (!p->uniform_magnitude)
        throw Error(VXQ_ERR_UNSUPPORTED, "dense tensor-core path needs uniform |J_ij|");
    DenseOperand* d = new DenseOperand();
    try {
        d->n = p->n;
        d->ld = ceil_div(p->n, DBK) * DBK;
        d->scale = (float)p->magnitude;
        VXQ_CUDA(cudaMalloc(&d->K, d->ld * d->ld));
        VXQ_CUDA(cudaMemsetAsync(d->K, 0, d->ld * d->ld, s));
        k_build_sign_matrix<<<(unsigned)ceil_div(p->n * 32, TB), TB, 0, s>>>(
            p->n, d->ld, p->indptr, p->indices, p->data64, d->K);
        VXQ_CHECK_LAUNCH();
        d->tmA = make_map_u8(d->K, d->ld, d->ld, d->ld, DBK, DBM);
        VXQ_CUDA(cudaStreamSynchronize(s));
    } catch (...) {
        delete d;
        throw;
    }
    p->dense = d;
    return d;
}

// Run the T-step PA loop on the tensor cores.  Outputs the final (x, m) in the interleaved
// layout of dynamics.cu ([n][R_pad], V lanes) and the final sign bits sb[n][W].
void dense_pa_loop(Problem* p, int64_t R, int64_t R_pad, int V, int64_t W,
                   const std::vector<double>& sched, float eta, float alpha, uint64_t seed,
                   int64_t rbegin, float* x_il, float* m_il, uint32_t* sb, long long* q2,
                   cudaStream_t s, double* loop_ms, int64_t* launches) {
    DenseOperand* d = dense_operand(p, s);
    const int64_t n = p->n, ld = d->ld, T = (int64_t)sched.size();
    DevBuf<float> x(R * ld, s), m(R * ld, s);
    DevBuf<uint8_t> s0(R * ld, s), s1(R * ld, s);
    VXQ_CUDA(cudaMemsetAsync(s0.get(), 0, R * ld, s));
    VXQ_CUDA(cudaMemsetAsync(s1.get(), 0, R * ld, s));
    k_init_pa_rm<<<nblk(((n + 3) / 4) * R), TB, 0, s>>>(n, R, ld, seed, rbegin, x.get(), m.get(),
                                                       s0.get());
    VXQ_CHECK_LAUNCH();
    int nsm = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    // replica tile width bn: minimise tiles x per-k-block time, where a k-block costs
    // max(MMA 4 x 128*bn/256 = 2 bn, smem read (16 KB A + 128 bn B) / 128 B/cyc) cycles;
    // bn >= 128 keeps the MMA (not shared-memory bandwidth) the limit.  The persistent
    // kernel spreads all T steps' tiles over the SMs, so per-step rounds do not matter.
    const int64_t m_tiles = ceil_div(n, DBM);
    int bn = DBN;
    int64_t best = INT64_MAX;
    for (int cand = DBN; cand >= 128; cand -= 16) {
        const int64_t tiles = m_tiles * ceil_div(R, cand);
        const int64_t cost = tiles * std::max<int64_t>(2 * cand, 128 + cand);
        if (cost < best) {
            best = cost;
            bn = cand;
        }
    }
    if (const char* e = getenv("VXQ_DENSE_BN")) bn = std::max(16, std::min(DBN, atoi(e) / 16 * 16));
    CUtensorMap tmB0 = make_map_u8(s0.get(), ld, R, ld, DBK, bn);
    CUtensorMap tmB1 = make_map_u8(s1.get(), ld, R, ld, DBK, bn);
    VXQ_CUDA(cudaFuncSetAttribute(k_dense_pa_run, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  DSMEM));
    std::vector<float> lam32(T);
    for (int64_t t = 0; t < T; ++t) lam32[t] = (float)sched[t];
    DevBuf<float> lam(std::max<int64_t>(T, 1), s);
    VXQ_CUDA(cudaMemcpyAsync(lam.get(), lam32.data(), T * sizeof(float), cudaMemcpyHostToDevice, s));
    DenseRunArgs a;
    a.n = (int)n;
    a.R = (int)R;
    a.ld = (int)ld;
    a.kblocks = (int)(ld / DBK);
    a.m_tiles = (int)ceil_div(n, DBM);
    a.n_tiles = (int)ceil_div(R, bn);
    a.bn = bn;
    a.T = (int)T;
    a.scale = d->scale;
    a.eta = eta;
    a.alpha = alpha;
    a.lam = lam.get();
    a.h = p->h32;
    a.x = x.get();
    a.m = m.get();
    a.s_buf[0] = s0.get();
    a.s_buf[1] = s1.get();
    a.mode = 0;
    a.q2 = nullptr;
    const char* dbg = getenv("VXQ_DENSE_DEBUG_NOEPI");  // profiling knob: no-op epilogue
    if (dbg && dbg[0] == '1') a.mode = 2;
    DevBuf<unsigned> done(std::max<int64_t>(T, 1) * a.n_tiles, s);
    VXQ_CUDA(cudaMemsetAsync(done.get(), 0, std::max<int64_t>(T, 1) * a.n_tiles * sizeof(unsigned), s));
    a.done = done.get();
    const int64_t tiles_total = (int64_t)a.m_tiles * a.n_tiles * std::max<int64_t>(T, 1);
    const unsigned grid = (unsigned)std::min<int64_t>(tiles_total, nsm);
    cudaEvent_t e0, e1;
    VXQ_CUDA(cudaEventCreate(&e0));
    VXQ_CUDA(cudaEventCreate(&e1));
    VXQ_CUDA(cudaEventRecord(e0, s));
    if (T > 0) {
        // all CTAs must be co-resident (they wait on each other's tiles): one per SM
        void* args[] = {(void*)&d->tmA, (void*)&tmB0, (void*)&tmB1, (void*)&a};
        VXQ_CUDA(cudaLaunchCooperativeKernel((const void*)k_dense_pa_run, dim3(grid),
                                             dim3(DTHREADS), args, DSMEM, s));
    }
    VXQ_CHECK_LAUNCH();
    VXQ_CUDA(cudaEventRecord(e1, s));
    *launches += 2;
    if (q2) {
        // one more tensor-core pass over s_T: 2 q_r = s_T . (K s_T), exact (energies)
        VXQ_CUDA(cudaMemsetAsync(q2, 0, R * sizeof(long long), s));
        DenseRunArgs e = a;
        e.T = 1;
        e.mode = 1;
        e.q2 = q2;
        const CUtensorMap& tb = (T & 1) ? tmB1 : tmB0;  // S_T
        const unsigned eg = (unsigned)std::min<int64_t>((int64_t)a.m_tiles * a.n_tiles, nsm);
        k_dense_pa_run<<<eg, DTHREADS, DSMEM, s>>>(d->tmA, tb, tb, e);
        VXQ_CHECK_LAUNCH();
        *launches += 1;
    }
    k_rm_to_interleaved<<<nblk(n * R), TB, 0, s>>>(x.get(), n, R, ld, R_pad, V, x_il);
    k_rm_to_interleaved<<<nblk(n * R), TB, 0, s>>>(m.get(), n, R, ld, R_pad, V, m_il);
    k_pack_bits_rm<<<(unsigned)ceil_div(n * W * 32, TB), TB, 0, s>>>(x.get(), n, R, ld, W, sb);
    VXQ_CHECK_LAUNCH();
    *launches += 3;
    float ms = 0;
    VXQ_CUDA(cudaEventSynchronize(e1));
    VXQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *loop_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

}  // namespace vxq
