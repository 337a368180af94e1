// L2 (LTS) throughput probe: every SM streams an L2-resident buffer with 16-byte
// ld.global.cg loads (L1 bypassed) and with TMA-like bulk copies; prints GB/s and B/clk.
// Calibrates the practical L2 ceiling the dense tensor-core kernel is measured against.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_l2_bw tools/l2_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_read(const uint4* __restrict__ buf, size_t n16, int reps, uint4* out) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) {
            uint4 v = __ldcg(buf + ((i + (size_t)r * 4096) % n16));
            acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[0] = acc;
}

__global__ void k_bulk(const uint8_t* __restrict__ buf, size_t bytes, int reps, uint32_t chunk) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x != 0) return;
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(sm);
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    uint32_t ph = 0;
    const size_t nchunks = bytes / chunk;
    for (int r = 0; r < reps; ++r) {
        for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
            const uint8_t* src = buf + ((c + (size_t)r * 7) % nchunks) * chunk;
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(chunk));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(d), "l"(src), "r"(chunk), "r"(b) : "memory");
            asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}"
                         ::"r"(b), "r"(ph));
            ph ^= 1;
        }
    }
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const size_t sizes[] = {16u << 20, 48u << 20};
    uint4* out;
    cudaMalloc(&out, 64);
    for (size_t bytes : sizes) {
        uint8_t* buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 1, bytes);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int bpsm : {4, 8}) {
            const int reps = 40;
            k_read<<<sms * bpsm, 512>>>((const uint4*)buf, bytes / 16, 2, out);
            cudaEventRecord(e0);
            k_read<<<sms * bpsm, 512>>>((const uint4*)buf, bytes / 16, reps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
            printf("ldg.cg  %3zu MB  %d blk/SM: %8.1f GB/s  (%.0f B/clk at the %d MHz max clock)\n",
                   bytes >> 20, bpsm, gbs, gbs * 1e9 / (clk * 1e3), clk / 1000);
        }
        for (uint32_t chunk : {16384u, 32768u}) {
            const int reps = 40;
            cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
            for (int bpsm : {2, 4}) {
                k_bulk<<<sms * bpsm, 32, chunk>>>(buf, bytes, 2, chunk);
                cudaEventRecord(e0);
                k_bulk<<<sms * bpsm, 32, chunk>>>(buf, bytes, reps, chunk);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
                printf("bulk    %3zu MB  %2u KB x %d blk/SM: %8.1f GB/s  (%.0f B/clk at max clock)\n",
                       bytes >> 20, chunk >> 10, bpsm, gbs, gbs * 1e9 / (clk * 1e3));
            }
        }
        cudaFree(buf);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
