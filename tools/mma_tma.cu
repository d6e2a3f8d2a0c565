// mma_tma.cu — do TMA writes into shared memory make progress while the
// tensor core streams its operands out of shared memory?  148 CTAs; warp 0
// keeps NBUF C3-shaped halo boxes in flight (4-D TMA, 64-byte rows, SW64,
// 4 rows x 58 positions = 14.8 KB, the conv3x3 producer's load), warp 1
// issues back-to-back tcgen05.mma.kind::i8 M128 x N x K32 (SS operands, as
// the conv kernel).  Reports TMA bytes/ns per SM and MMA cycles per
// instruction, each alone and together.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc mma_tma.cu -lcuda -o mma_tma
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace q8g;

constexpr int NBUF = 4;
constexpr int HALO = 64 * 58 * 4;  // 14,848 B

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int N>
__global__ void __launch_bounds__(64, 1) probe(const __grid_constant__ CUtensorMap m, int tma_iters, int mma_iters,
                                              unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[NBUF + 1];
    __shared__ uint32_t tmem_slot;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t sA = base, sB = base + 16384, sH = base + 65536;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int b = 0; b <= NBUF; ++b) ptx::mbar_init(ptx::smem_u32(&bars[b]), 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc<256>(ptx::smem_u32(&tmem_slot));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (warp == 0 && threadIdx.x == 0 && tma_iters > 0) {
        const unsigned long long t0 = gtime();
        uint32_t ph = 0;
        for (int i = 0; i < tma_iters; ++i) {
            const int b = i % NBUF;
            if (i >= NBUF) {
                ptx::mbar_wait_spin(ptx::smem_u32(&bars[b]), ph);
                if (b == NBUF - 1) ph ^= 1;
            }
            const int u = blockIdx.x + i * gridDim.x;
            const int n = u % 32, rb = (u / 32) % 28;
            ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bars[b]), HALO);
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                    sH + b * 16384),
                "l"(reinterpret_cast<uint64_t>(&m)), "r"(0), "r"(-1), "r"(rb * 2 - 1), "r"(n),
                "r"(ptx::smem_u32(&bars[b]))
                : "memory");
        }
        for (int i = tma_iters; i < tma_iters + NBUF; ++i) {
            const int b = i % NBUF;
            ptx::mbar_wait_spin(ptx::smem_u32(&bars[b]), ph);
            if (b == NBUF - 1) ph ^= 1;
        }
        out[blockIdx.x * 2] = gtime() - t0;
    }
    if (warp == 1 && mma_iters > 0) {
        constexpr uint32_t idesc = ptx::idesc_u8s8_s32<128, N>();
        const uint64_t ad = ptx::sw128_kmajor_desc(sA), bd = ptx::sw128_kmajor_desc(sB);
        const uint32_t cbar = ptx::smem_u32(&bars[NBUF]);
        const unsigned long long t0 = gtime();
        for (int i = 0; i < mma_iters; ++i) {
            if (ptx::elect_one()) {
#pragma unroll
                for (int j = 0; j < 16; ++j) ptx::mma_i8(tmem, ad + 2 * (j & 3), bd + 2 * (j & 3), idesc, 1);
                ptx::tc_commit(cbar);
            }
            __syncwarp();
            ptx::mbar_wait_spin(cbar, (uint32_t)i & 1u);  // keep at most 16 MMAs queued beyond the commit
        }
        if (threadIdx.x == 32) out[blockIdx.x * 2 + 1] = gtime() - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<256>(tmem);
    }
}

int main() {
    const int NB = 32, H = 56, W = 56, C = 64;
    uint8_t* x;
    cudaMalloc(&x, (size_t)NB * H * W * C);
    cudaMemset(x, 1, (size_t)NB * H * W * C);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)NB};
    cuuint64_t strides[3] = {(cuuint64_t)C, (cuuint64_t)W * C, (cuuint64_t)H * W * C};
    cuuint32_t box[4] = {64, 58, 4, 1}, es[4] = {1, 1, 1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
        std::printf("tensor map encode failed\n");
        return 1;
    }
    unsigned long long* out;
    cudaMalloc(&out, 148 * 2 * 8);
    std::vector<unsigned long long> h(296);
    auto run = [&](auto kern, const char* nm, int tma_iters, int mma_iters, int n) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(out, 0, 296 * 8);
            kern<<<148, 64, 200 * 1024>>>(m, tma_iters, mma_iters, out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                std::printf("error %s\n", cudaGetErrorString(e));
                return;
            }
        }
        cudaMemcpy(h.data(), out, 296 * 8, cudaMemcpyDeviceToHost);
        std::vector<double> tt, tm;
        for (int c = 0; c < 148; ++c) {
            if (h[2 * c]) tt.push_back((double)h[2 * c]);
            if (h[2 * c + 1]) tm.push_back((double)h[2 * c + 1]);
        }
        std::sort(tt.begin(), tt.end());
        std::sort(tm.begin(), tm.end());
        std::printf("%-30s", nm);
        if (!tt.empty())
            std::printf("  TMA: %6.1f B/ns per SM (%5.2f us per halo)", (double)tma_iters * HALO / tt[tt.size() / 2],
                        tt[tt.size() / 2] / tma_iters / 1e3);
        if (!tm.empty())
            std::printf("  MMA N=%d: %5.1f cycles/instr @1.92GHz", n, tm[tm.size() / 2] * 1.92 / (mma_iters * 16.0));
        std::printf("\n");
    };
    run(probe<80>, "TMA alone", 200, 0, 80);
    run(probe<80>, "MMA N=80 alone", 0, 400, 80);
    run(probe<80>, "TMA + MMA N=80", 200, 400, 80);
    run(probe<80>, "TMA + MMA N=80 (long)", 200, 2000, 80);
    run(probe<64>, "MMA N=64 alone", 0, 400, 64);
    run(probe<64>, "TMA + MMA N=64 (long)", 200, 2000, 64);
    run(probe<256>, "MMA N=256 alone", 0, 400, 256);
    run(probe<256>, "TMA + MMA N=256 (long)", 200, 1000, 256);
    return 0;
}
