// mma_peak.cu -- measured tensor-core peak of the MMA kinds the dense kernels issue, on
// CTA pairs (tcgen05.mma.cta_group::2, M = 256, N = 256) with operands resident in shared
// memory (no TMA, no epilogue): the denominator for roofline.frac of k_dense_run
// (MEASURED_PEAKS.json has only bf16 from cuBLAS).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/_mma_peak \
//        tools/mma_peak.cu -lcuda
//   tools/_mma_peak [seconds]        -> one line per kind: TFLOP/s (dense), SM clock
//
// Every CTA pair issues back-to-back k-blocks (4 MMAs over one 128-byte smem row group,
// as k_dense_run does) into one TMEM accumulator; operands hold random bit patterns so the
// power draw (and the capped clock) resembles real data.  FLOPs = 2 M N K per MMA.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../paper_2501_19221_b200/csrc/tc_ptx.cuh"

using namespace vxq::ptx;

constexpr int kM = 256, kN = 256;
constexpr int kABytes = 128 * 128;       // 128 A rows x 128 B per CTA
constexpr int kBBytes = (kN / 2) * 128;  // N/2 B rows x 128 B per CTA
constexpr int kStages = 4;               // distinct smem operand sets cycled through
constexpr int kSmem = kStages * (kABytes + kBBytes) + 1024;
constexpr uint32_t kSfCol = 480;

enum { kMxf4 = 0, kBf16 = 1, kI8 = 2, kF8 = 3 };

__device__ __forceinline__ void mma2_i8_(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
    mma2_i8(d, a, b, idesc, acc);
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) k_peak(long long kblocks, unsigned long long* clk) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) &
                                               ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    // random operand bits (bf16: +-1.x patterns, no NaN/Inf)
    uint32_t h = 0x9E3779B9u * (blockIdx.x + 1);
    for (int i = threadIdx.x; i < kStages * (kABytes + kBBytes) / 4; i += blockDim.x) {
        uint32_t v = (h ^ (uint32_t)i * 0x85EBCA6Bu);
        v ^= v >> 13;
        v *= 0xC2B2AE35u;
        v ^= v >> 16;
        if (KIND == kBf16) v = (v & 0x807F807Fu) | 0x3F803F80u;
        if (KIND == kF8) v = (v & 0xB7B7B7B7u) | 0x30303030u;  // finite E4M3
        reinterpret_cast<uint32_t*>(smem)[i] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> async proxy
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc2<512>(&slot);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (KIND == kMxf4) {  // unit UE8M0 scale factors
        tmem_fill_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + kSfCol, 0x7F7F7F7Fu);
        tc_fence_before();
        cluster_sync();
        tc_fence_after();
    }
    const int crank = (int)cluster_ctarank();
    long long t0 = 0, t1 = 0;
    if (crank == 0 && threadIdx.x == 0) {
        uint32_t idesc;
        if (KIND == kMxf4) idesc = (1u << 7) | (1u << 10) | (1u << 23);
        else if (KIND == kBf16) idesc = (1u << 4) | (1u << 7) | (1u << 10);
        else if (KIND == kI8) idesc = (2u << 4) | (1u << 7) | (1u << 10);
        else idesc = (1u << 4);
        idesc |= ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
        for (long long kb = 0; kb < kblocks; ++kb) {
            const int st = (int)(kb % kStages);
            const uint32_t sa = smem_u32(smem + st * (kABytes + kBBytes));
            const uint64_t da = sw128_kmajor_desc(sa), db = sw128_kmajor_desc(sa + kABytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t acc = (kb | k) != 0;
                if (KIND == kMxf4)
                    mma2_mxf4(tmem, da + 2 * k, db + 2 * k, idesc, tmem + kSfCol,
                              tmem + kSfCol + 16, acc);
                else if (KIND == kBf16) mma2_f16(tmem, da + 2 * k, db + 2 * k, idesc, acc);
                else if (KIND == kI8) mma2_i8_(tmem, da + 2 * k, db + 2 * k, idesc, acc);
                else mma2_f8f6f4(tmem, da + 2 * k, db + 2 * k, idesc, acc);
            }
        }
        mma2_commit_mc(&bar, 0x1);
        mbar_wait(&bar, 0, 60ull * 1000 * 1000 * 1000);
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
        atomicMax(clk, (unsigned long long)(t1 - t0));
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) tmem_dealloc2<512>(tmem);
}

template <int KIND>
void run(const char* name, double kelem, double seconds) {
    auto kern = k_peak<KIND>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nsm / 2 * 2);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = kSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    unsigned long long* d_clk;
    cudaMalloc(&d_clk, 8);
    // calibrate the k-block count to ~`seconds` of work, then time it
    long long kb = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int pass = 0; pass < 3; ++pass) {
        cudaMemset(d_clk, 0, 8);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, kern, kb, d_clk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) {
            printf("%s: %s\n", name, cudaGetErrorString(err));
            return;
        }
        cudaEventElapsedTime(&ms, e0, e1);
        if (pass < 2) kb = (long long)(kb * (seconds * 1e3 / ms));
    }
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d_clk, 8, cudaMemcpyDeviceToHost);
    const double flops = (double)(nsm / 2) * kb * 4 * 2.0 * kM * kN * kelem;
    printf("{\"kind\": \"%s\", \"tflops\": %.1f, \"ms\": %.2f, \"kblocks\": %lld, "
           "\"sm_mhz_from_clock64\": %.0f, \"pairs\": %d}\n",
           name, flops / (ms * 1e-3) / 1e12, ms, kb, cyc / (ms * 1e3), nsm / 2);
    cudaFree(d_clk);
}

int main(int argc, char** argv) {
    const double sec = argc > 1 ? atof(argv[1]) : 2.0;
    run<kBf16>("bf16 (kind::f16)", 16, sec);
    run<kF8>("e4m3 (kind::f8f6f4)", 32, sec);
    run<kI8>("s8 (kind::i8)", 32, sec);
    run<kMxf4>("e2m1 (kind::mxf4, block32 unit scales)", 64, sec);
    return 0;
}
