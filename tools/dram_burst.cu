// dram_burst.cu — how fast can 128 (or 148) CTAs pull a C1-sized weight
// slice (16.8 MB total, 128 KB per CTA as 8 x 16 KB bulk copies) out of HBM?
// The practical floor of the C1 main loop.  Rotating 17 MB slices of a 1 GB
// buffer keep every launch cold in L2.  Back-to-back launches, event timing.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc dram_burst.cu -o dram_burst
#include <algorithm>
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace q8g;

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// in-kernel span: per-CTA entry and "all bytes landed" stamps
__global__ void __launch_bounds__(32, 1) burst_timed(const uint8_t* src, int chunk, int nchunks,
                                                     unsigned long long* stamps) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    if (threadIdx.x == 0) {
        stamps[2 * blockIdx.x] = gtime();
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar), (uint32_t)(chunk * nchunks));
        const uint8_t* my = src + (size_t)blockIdx.x * chunk * nchunks;
        for (int i = 0; i < nchunks; ++i)
            ptx::bulk_load(base + i * chunk, my + (size_t)i * chunk, (uint32_t)chunk, ptx::smem_u32(&bar));
        ptx::mbar_wait_spin(ptx::smem_u32(&bar), 0);
        stamps[2 * blockIdx.x + 1] = gtime();
    }
}

__global__ void __launch_bounds__(32, 1) burst(const uint8_t* src, size_t slice_bytes, int chunk, int nchunks) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar), (uint32_t)(chunk * nchunks));
        const uint8_t* my = src + (size_t)blockIdx.x * chunk * nchunks;
        for (int i = 0; i < nchunks; ++i)
            ptx::bulk_load(base + i * chunk, my + (size_t)i * chunk, (uint32_t)chunk, ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    }
    (void)slice_bytes;
}

// LDG.128 to registers, 256 threads, 8 independent loads in flight per thread
__global__ void __launch_bounds__(256, 1) burst_ldg(const uint8_t* src, int per_cta, unsigned* sink) {
    const uint4* p = reinterpret_cast<const uint4*>(src + (size_t)blockIdx.x * per_cta);
    const int n = per_cta / 16;
    uint32_t acc = 0;
    for (int i = threadIdx.x; i < n; i += 256 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = i + u * 256 < n ? __ldcs(p + i + u * 256) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

// cp.async 16 B (LDGSTS) into smem, 256 threads, all in flight, one wait
__global__ void __launch_bounds__(256, 1) burst_ldgsts(const uint8_t* src, int per_cta) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t base = ptx::smem_u32(smem_raw);
    const uint8_t* my = src + (size_t)blockIdx.x * per_cta;
    for (int off = threadIdx.x * 16; off < per_cta; off += 256 * 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + off), "l"(my + off) : "memory");
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

int main() {
    const size_t total = (size_t)1 << 30;
    uint8_t* buf;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 1, total);
    cudaFuncSetAttribute(burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int ctas : {128, 148}) {
        for (int chunk : {16384, 32768}) {
            const int nchunks = 131072 / chunk;  // 128 KB per CTA
            const size_t slice = (size_t)ctas * 131072;
            const int nslices = (int)(total / slice);
            for (int i = 0; i < 4; ++i) burst<<<ctas, 32, 140 * 1024>>>(buf + (i % nslices) * slice, slice, chunk, nchunks);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            const int reps = 200;
            cudaEventRecord(a);
            for (int i = 0; i < reps; ++i)
                burst<<<ctas, 32, 140 * 1024>>>(buf + (i % nslices) * slice, slice, chunk, nchunks);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double us = ms * 1e3 / reps;
            std::printf("%3d CTAs x 128 KB (%2d x %5d B bulk copies), %5.1f MB per launch: %6.2f us/launch  %7.1f GB/s (%s)\n",
                        ctas, nchunks, chunk, slice / 1e6, us, slice / (us * 1e-6) / 1e9,
                        cudaGetErrorString(cudaGetLastError()));
        }
    }
    unsigned* sink;
    cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(burst_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int ctas : {128, 148}) {
        const size_t slice = (size_t)ctas * 131072;
        const int nslices = (int)(total / slice);
        for (int mode = 0; mode < 2; ++mode) {
            auto go = [&](int i) {
                if (mode == 0)
                    burst_ldg<<<ctas, 256>>>(buf + (i % nslices) * slice, 131072, sink);
                else
                    burst_ldgsts<<<ctas, 256, 140 * 1024>>>(buf + (i % nslices) * slice, 131072);
            };
            for (int i = 0; i < 4; ++i) go(i);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            const int reps = 200;
            cudaEventRecord(a);
            for (int i = 0; i < reps; ++i) go(i);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double us = ms * 1e3 / reps;
            std::printf("%3d CTAs x 128 KB via %-7s, %5.1f MB per launch: %6.2f us/launch  %7.1f GB/s (%s)\n", ctas,
                        mode == 0 ? "LDG.128" : "LDGSTS", slice / 1e6, us, slice / (us * 1e-6) / 1e9,
                        cudaGetErrorString(cudaGetLastError()));
        }
    }
    // in-kernel span of one cold 16.8 MB burst (128 CTAs x 8 x 16 KB)
    {
        unsigned long long* st;
        cudaMalloc(&st, 2 * 148 * 8);
        cudaFuncSetAttribute(burst_timed, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        std::vector<unsigned long long> h(2 * 148);
        for (int ctas : {128, 148})
            for (int rep = 0; rep < 3; ++rep) {
                const size_t slice = (size_t)ctas * 131072;
                burst_timed<<<ctas, 32, 140 * 1024>>>(buf + (size_t)(rep + 3) * 32 * 1024 * 1024 * 4, 16384, 8, st);
                if (cudaDeviceSynchronize() != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
                cudaMemcpy(h.data(), st, 2 * ctas * 8, cudaMemcpyDeviceToHost);
                unsigned long long e0 = ~0ull, e1 = 0, d0 = ~0ull, d1 = 0;
                for (int c = 0; c < ctas; ++c) {
                    e0 = std::min(e0, h[2 * c]);
                    e1 = std::max(e1, h[2 * c]);
                    d0 = std::min(d0, h[2 * c + 1]);
                    d1 = std::max(d1, h[2 * c + 1]);
                }
                std::printf("in-kernel %3d CTAs: entries spread %.2f us, first CTA done %.2f us, last done %.2f us after "
                            "first entry -> %.1f GB/s over the span\n",
                            ctas, (e1 - e0) / 1e3, (d0 - e0) / 1e3, (d1 - e0) / 1e3, slice / ((d1 - e0) * 1e-9) / 1e9);
            }
    }
    // launch overhead alone: an empty-ish grid
    {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int i = 0; i < 200; ++i) burst_ldg<<<128, 256>>>(buf, 0, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("empty launch (back to back): %6.2f us/launch\n", ms * 1e3 / 200);
    }
    return 0;
}
