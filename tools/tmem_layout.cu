// tmem_layout.cu — which (TMEM lane, column) each thread's registers hold for
// tcgen05.ld.16x256b (the fragment layout the C2 epilogue relies on).  One
// warp writes lane*1000 + column into 32 lanes x 32 columns with the
// 32x32b shape (thread = lane), then reads lanes 0-15 back with
// 16x256b.x2 and prints, per thread, the decoded (lane, column) of each of
// its 8 registers.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2101_05615_b200/csrc tmem_layout.cu -o tmem_layout
#include <cstdio>

#include "ptx.cuh"

using namespace q8g;

__global__ void probe(uint32_t* out) {
    __shared__ uint32_t tptr;
    if (threadIdx.x < 32) ptx::tmem_alloc<32>(ptx::smem_u32(&tptr));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tptr;
    const uint32_t lane = threadIdx.x;
    uint32_t w[32];
    for (int c = 0; c < 32; ++c) w[c] = lane * 1000 + c;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem),
        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]),
        "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]),
        "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]),
        "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(tmem));
    ptx::tmem_ld_wait();
    for (int j = 0; j < 8; ++j) out[lane * 8 + j] = r[j];
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) ptx::tmem_dealloc<32>(tmem);
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 32 * 8 * 4);
    probe<<<1, 32>>>(d);
    uint32_t h[256];
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        std::printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    for (int t = 0; t < 32; ++t) {
        std::printf("t%2d:", t);
        for (int j = 0; j < 8; ++j) std::printf(" (%u,%u)", h[t * 8 + j] / 1000, h[t * 8 + j] % 1000);
        std::printf("\n");
    }
    return 0;
}
