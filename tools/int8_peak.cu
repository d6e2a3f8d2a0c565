// int8_peak.cu — measured dense INT8 tensor-core peak of this B200 (the
// roofline denominator for tensor-bound configs): one CTA per
// SM issues back-to-back tcgen05.mma.kind::i8 (M=128, N=256, K=32, A u8 /
// B s8 from SWIZZLE_128B smem, s32 accumulators in TMEM) and the whole grid is
// timed with CUDA events.  Burst = best of short runs; sustained = one ~2 s
// run.  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc int8_peak.cu -o int8_peak
#include <cstdio>
#include <vector>
#include <algorithm>

#include "ptx.cuh"

using namespace q8g;

__global__ void __launch_bounds__(128, 1) peak_kernel(long long iters, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tptr;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* sm = smem_raw + (base - ptx::smem_u32(smem_raw));
    for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
    }
    if (threadIdx.x < 32) ptx::tmem_alloc<512>(ptx::smem_u32(&tptr));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tptr;
    constexpr uint32_t idesc = ptx::idesc_u8s8_s32<128, 256>();
    const uint64_t ad = ptx::sw128_kmajor_desc(base), bd = ptx::sw128_kmajor_desc(base + 16384);
    if (threadIdx.x < 32) {
        if (ptx::elect_one()) {
            for (long long i = 0; i < iters; ++i)
                ptx::mma_i8(tmem + (uint32_t)((i & 1) * 256), ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, i > 1);
            ptx::tc_commit(ptx::smem_u32(&bar));
        }
        __syncwarp();
    }
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    ptx::tc_fence_after();
    if (threadIdx.x < 32) {
        uint32_t v[16];
        ptx::tmem_ld_32x32b_x16(tmem, v);
        ptx::tmem_ld_wait();
        if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)v[0]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tmem);
}

static double run(int sms, long long iters) {
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    peak_kernel<<<sms, 128, 64 * 1024>>>(iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(sink);
    return (double)sms * iters * 2.0 * 128 * 256 * 32 / (ms * 1e-3) / 1e12;
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    run(sms, 20000);  // warm-up
    std::vector<double> burst;
    for (int r = 0; r < 10; ++r) burst.push_back(run(sms, 100000));  // ~7 ms each at peak
    const double best = *std::max_element(burst.begin(), burst.end());
    const double sustained = run(sms, 30000000);  // ~2 s
    cudaError_t e = cudaGetLastError();
    std::printf("{\"int8_tops_burst\": %.1f, \"int8_tops_sustained\": %.1f, \"sms\": %d, \"shape\": "
                "\"tcgen05.mma.kind::i8 M128 N256 K32, SS (SW128), back-to-back, 1 CTA/SM\", \"error\": \"%s\"}\n",
                best, sustained, sms, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
