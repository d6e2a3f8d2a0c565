// mbar_cost.cu — cost of mbarrier.try_wait on a barrier whose phase is
// already complete, with and without a suspend-time hint (the pipeline
// loops wait on such barriers every iteration).  One CTA, one warp; clock64
// around 64 waits.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc mbar_cost.cu -o mbar_cost
#include <cstdio>

#include "ptx.cuh"

using namespace q8g;

__global__ void probe(long long* out) {
    __shared__ uint64_t bar;
    const uint32_t b = ptx::smem_u32(&bar);
    if (threadIdx.x == 0) {
        ptx::mbar_init(b, 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    // phase 0 never completes; waiting on parity 1 (the "previous" phase)
    // returns at once -- the producer-start idiom
    long long t0 = clock64();
    for (int i = 0; i < 64; ++i) ptx::mbar_wait(b, 1);
    long long t1 = clock64();
    for (int i = 0; i < 64; ++i) ptx::mbar_wait_spin(b, 1);
    long long t2 = clock64();
    // a completed phase: arrive once, then wait on parity 0
    if (threadIdx.x == 0) ptx::mbar_arrive(b);
    __syncwarp();
    long long t3 = clock64();
    for (int i = 0; i < 64; ++i) ptx::mbar_wait(b, 0);
    long long t4 = clock64();
    for (int i = 0; i < 64; ++i) ptx::mbar_wait_spin(b, 0);
    long long t5 = clock64();
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / 64;
        out[1] = (t2 - t1) / 64;
        out[2] = (t4 - t3) / 64;
        out[3] = (t5 - t4) / 64;
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    long long h[4];
    for (int r = 0; r < 3; ++r) probe<<<1, 32>>>(d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    std::printf("try_wait, complete phase (parity of the previous phase): hinted %lld cycles, spin %lld cycles\n", h[0],
                h[1]);
    std::printf("try_wait, complete phase (after an arrive):             hinted %lld cycles, spin %lld cycles\n", h[2],
                h[3]);
    return 0;
}
