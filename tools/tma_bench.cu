// tma_bench.cu — chip-wide TMA throughput for 4-D halo boxes {IB bytes, 114
// positions, R rows, 1 image} out of an NHWC u8 tensor shaped like C4
// (32 x 112 x 112 x 256), as a function of the inner box width IB (the
// halo row size) and the swizzle.  148 CTAs, each keeps NBUF boxes in flight
// on mbarriers.  Tuning tool for the conv / depthwise halo producers.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc tma_bench.cu -lcuda -o tma_bench
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace q8g;

constexpr int NBUF = 4;

__global__ void __launch_bounds__(32, 1) tma_kernel(const __grid_constant__ CUtensorMap m, int ib, int rows, int iters,
                                                   int box_bytes, int nblk, int nimg) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[NBUF];
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const int stride = (box_bytes + 1023) / 1024 * 1024;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NBUF; ++b) ptx::mbar_init(ptx::smem_u32(&bars[b]), 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    if (threadIdx.x == 0) {
        uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            const int b = i % NBUF;
            if (i >= NBUF) {
                ptx::mbar_wait(ptx::smem_u32(&bars[b]), ph);
                if (b == NBUF - 1) ph ^= 1;
            }
            // unit i of this CTA: channel block, image, row block
            const int u = blockIdx.x + i * gridDim.x;
            const int cb = u % nblk, rest = u / nblk;
            const int n = rest % nimg, rb = (rest / nimg) % (112 / 2);
            ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bars[b]), (uint32_t)box_bytes);
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                    base + b * stride),
                "l"(reinterpret_cast<uint64_t>(&m)), "r"(cb * ib), "r"(-1), "r"(rb * 2 - 1), "r"(n),
                "r"(ptx::smem_u32(&bars[b]))
                : "memory");
        }
        // drain
        for (int i = iters; i < iters + NBUF; ++i) {
            const int b = i % NBUF;
            ptx::mbar_wait(ptx::smem_u32(&bars[b]), ph);
            if (b == NBUF - 1) ph ^= 1;
        }
    }
    __syncwarp();
}

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 32, H = 112, W = 112, C = 256;  // N=128: 411 MB > 3x L2 (cold DRAM)
    uint8_t* x;
    cudaMalloc(&x, (size_t)N * H * W * C);
    cudaMemset(x, 1, (size_t)N * H * W * C);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    struct Cfg { int ib, rows; CUtensorMapSwizzle sw; const char* name; };
    const Cfg cfgs[] = {{16, 10, CU_TENSOR_MAP_SWIZZLE_NONE, "16B rows (dw 16-ch planes), 10 rows"},
                        {32, 4, CU_TENSOR_MAP_SWIZZLE_32B, "32B rows SW32, 4 rows"},
                        {64, 4, CU_TENSOR_MAP_SWIZZLE_64B, "64B rows SW64, 4 rows (dw tc64)"},
                        {128, 3, CU_TENSOR_MAP_SWIZZLE_128B, "128B rows SW128, 3 rows"},
                        {128, 4, CU_TENSOR_MAP_SWIZZLE_128B, "128B rows SW128, 4 rows"},
                        {64, 4, CU_TENSOR_MAP_SWIZZLE_NONE, "64B rows no-swizzle, 4 rows"},
                        {256, 2, CU_TENSOR_MAP_SWIZZLE_NONE, "256B rows no-swizzle, 2 rows"}};
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (const Cfg& c : cfgs) {
        CUtensorMap m;
        cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
        cuuint64_t strides[3] = {(cuuint64_t)C, (cuuint64_t)W * C, (cuuint64_t)H * W * C};
        cuuint32_t box[4] = {(cuuint32_t)c.ib, (cuuint32_t)(W + 2), (cuuint32_t)c.rows, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, x, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            std::printf("%-40s encode failed\n", c.name);
            continue;
        }
        const int box_bytes = c.ib * (W + 2) * c.rows;
        const int iters = N > 32 ? 600 : 200, nblk = C / c.ib;
        const int smem = NBUF * ((box_bytes + 1023) / 1024 * 1024) + 2048;
        tma_kernel<<<148, 32, smem>>>(m, c.ib, c.rows, 20, box_bytes, nblk, N);  // warm-up
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        tma_kernel<<<148, 32, smem>>>(m, c.ib, c.rows, iters, box_bytes, nblk, N);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = 148.0 * (iters + 0) * box_bytes;
        std::printf("%-40s box %6d B: %7.2f us/box/SM  %8.1f GB/s chip  %6.2f ns/row/SM  (%s)\n", c.name, box_bytes,
                    ms * 1e3 / iters, bytes / (ms * 1e-3) / 1e9, ms * 1e6 / iters / ((W + 2) * c.rows),
                    cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
