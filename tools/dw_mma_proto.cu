// dw_mma_proto.cu — the depthwise kernel's MMA loop with its full barrier
// protocol but no data movement and no epilogue work: a producer warp
// completes each halo buffer's full barrier by a plain arrive (3 buffers),
// the MMA warp waits free accumulator + full halo and issues the 24-MMA unit
// (2 accumulators, commits to the buffer's empty and the accumulator's full
// barrier), and 16 "epilogue" warps wait for each accumulator and release it
// at once.  SM cycles per unit of the MMA warp.  Configurations: MMA warp id
// (0 or 19), epilogue warps (0 or 16), commits per unit (1 or 2), and the
// producer's halo: none (plain arrive), the kernel's 4-D TMA box {64 B, 114,
// 4, 1} (SWIZZLE_64B, 29 KB), or the same bytes as {128 B, 114, 2, 1}
// (SWIZZLE_128B: half the TMA rows) -- is it the TMA writes into shared
// memory that slow the in-kernel MMAs?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc dw_mma_proto.cu -o dw_mma_proto
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace q8g;

__device__ inline uint64_t swz64_desc(uint32_t addr) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ inline uint64_t noswz_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

constexpr int NB = 3, EPI = 16;

__device__ __forceinline__ void tma4(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                     uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

__global__ void __launch_bounds__(640, 1) proto(const __grid_constant__ CUtensorMap m64,
                                                const __grid_constant__ CUtensorMap m128, int units, int w_mma,
                                                int epi, int two_commits, int halo, int bfill,
                                                unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[2 * NB + 4];
    __shared__ uint32_t tmem_slot;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const int wp = 114, CB = 64, KG = 2;
    const uint32_t hstride = (uint32_t)((4 * wp * CB + 1024 + 1023) / 1024 * 1024);
    const uint32_t sA = base + 1024, sB = sA + NB * hstride;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    auto bar = [&](int i) { return ptx::smem_u32(&bars[i]); };
    auto full_bar = [&](int b) { return bar(b); };
    auto empty_bar = [&](int b) { return bar(NB + b); };
    auto tfull_bar = [&](int a) { return bar(2 * NB + a); };
    auto tempty_bar = [&](int a) { return bar(2 * NB + 2 + a); };
    const int w_prod = w_mma == 0 ? 1 : 16, w_alloc = w_mma == 0 ? 2 : 17;
    if (bfill) {  // B like the kernel's: per 16-byte row one nonzero (a diagonal entry), random
        for (int i = threadIdx.x; i < 3 * KG * 2 * 192 * 16; i += blockDim.x) {
            const int row = (i / 16) % 192, byte = i % 16;
            const uint32_t hsh = (uint32_t)i * 2654435761u ^ (uint32_t)blockIdx.x * 40503u;
            smem_raw[(sB - ptx::smem_u32(smem_raw)) + i] = (row % 16 == byte) ? (uint8_t)(hsh >> 13) : 0;
        }
    }
    if (threadIdx.x == 0) {
        for (int b = 0; b < NB; ++b) {
            ptx::mbar_init(full_bar(b), 1);
            ptx::mbar_init(empty_bar(b), 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull_bar(a), 1);
            ptx::mbar_init(tempty_bar(a), epi > 0 ? epi : 1);
        }
        ptx::fence_mbar_init();
    }
    if (warp == w_alloc) ptx::tmem_alloc<512>(ptx::smem_u32(&tmem_slot));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (warp == w_prod) {
        int b = 0;
        uint32_t ph = 0;
        for (int u = 0; u < units; ++u) {
            ptx::mbar_wait(empty_bar(b), ph ^ 1);
            if (ptx::elect_one()) {
                const int img = (blockIdx.x + 148 * u) % 32, row = (u * 2) % 108;
                if (halo == 0) {
                    ptx::mbar_arrive(full_bar(b));
                } else if (halo == 1) {
                    ptx::mbar_arrive_expect_tx(full_bar(b), 4 * 114 * 64);
                    tma4(sA + b * hstride, &m64, 64 * (blockIdx.x % 4), -1, row - 1, img, full_bar(b));
                } else {
                    ptx::mbar_arrive_expect_tx(full_bar(b), 2 * 114 * 128);
                    tma4(sA + b * hstride, &m128, 128 * (blockIdx.x % 2), -1, row - 1, img, full_bar(b));
                }
            }
            __syncwarp();
            if (++b == NB) {
                b = 0;
                ph ^= 1;
            }
        }
    } else if (warp == w_mma) {
        constexpr uint32_t idesc64 = ptx::idesc_u8s8_s32<128, 64>();
        constexpr uint32_t idesc128 = ptx::idesc_u8s8_s32<128, 128>();
        const uint64_t a0 = swz64_desc(0u);
        const uint64_t row16 = (uint64_t)(wp * CB / 16), pos16 = CB / 16;
        const uint64_t b0 = noswz_desc(sB, 192 * 16, 128);
        int b = 0, acc = 0;
        uint32_t ph = 0, aph = 0;
        long long t0 = 0;
        for (int u = 0; u < units; ++u) {
            if (u == 4) t0 = clock64();
            if (epi > 0) ptx::mbar_wait(tempty_bar(acc), aph ^ 1);
            ptx::mbar_wait(full_bar(b), ph);
            ptx::tc_fence_after();
            const uint64_t ahalo = a0 + ((sA + b * hstride) >> 4);
            if (ptx::elect_one()) {
#pragma unroll
                for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                    for (int kw = 0; kw < 3; ++kw)
#pragma unroll
                        for (int j = 0; j < KG; ++j) {
                            const int i = (ii + 3) % 4;
                            const uint64_t ad = ahalo + (uint64_t)i * row16 + (uint64_t)kw * pos16 + 2u * j;
                            const uint64_t bd = b0 + (uint64_t)((kw * KG + j) * 384);
                            const uint32_t d = tmem + (uint32_t)(acc * 256 + j * 128);
                            if (i == 0) ptx::mma_i8(d + 64, ad, bd, idesc64, kw != 0);
                            if (i == 1) ptx::mma_i8(d, ad, bd, idesc128, 1);
                            if (i == 2) ptx::mma_i8(d, ad, bd + 64, idesc128, 1);
                            if (i == 3) ptx::mma_i8(d, ad, bd + 128, idesc64, kw != 0);
                        }
                ptx::tc_commit(empty_bar(b));
                if (two_commits || epi > 0) ptx::tc_commit(tfull_bar(acc));
            }
            __syncwarp();
            if (epi == 0 && u >= 1) ptx::mbar_wait(empty_bar((b + NB - 1) % NB), (b == 0) ? ph ^ 1 : ph);  // <= 2 in flight
            if (++b == NB) {
                b = 0;
                ph ^= 1;
            }
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
        // drain: the last unit's commit
        const int lb = (units - 1) % NB;
        ptx::mbar_wait(empty_bar(lb), (uint32_t)(((units - 1) / NB) & 1));
        const long long t1 = clock64();
        if (lane == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    } else if (warp >= (w_mma == 0 ? 4 : 0) && warp < (w_mma == 0 ? 4 : 0) + epi) {
        int acc = 0;
        uint32_t aph = 0;
        for (int u = 0; u < units; ++u) {
            ptx::mbar_wait(tfull_bar(acc), aph);
            ptx::tc_fence_after();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty_bar(acc));
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == w_alloc) ptx::tmem_dealloc<512>(tmem);
}

__global__ void fill_random(uint8_t* x, size_t n, int zero) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        x[i] = zero ? 0 : (uint8_t)(((uint32_t)i * 2654435761u) >> 11);
}

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int units = argc > 1 ? atoi(argv[1]) : 200, smem = argc > 2 ? atoi(argv[2]) * 1024 : 200 * 1024;
    const int NBI = 32, H = 112, W = 112, C = 256;
    uint8_t* x;
    cudaMalloc(&x, (size_t)NBI * H * W * C);
    cudaMemset(x, 1, (size_t)NBI * H * W * C);
    fill_random<<<1024, 256>>>(x, (size_t)NBI * H * W * C, 0);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap m64, m128;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)NBI};
    cuuint64_t strides[3] = {(cuuint64_t)C, (cuuint64_t)W * C, (cuuint64_t)H * W * C};
    cuuint32_t box64[4] = {64, 114, 4, 1}, box128[4] = {128, 114, 2, 1}, es[4] = {1, 1, 1, 1};
    if (enc(&m64, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, x, dims, strides, box64, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS ||
        enc(&m128, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, x, dims, strides, box128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
        printf("tensor map encode failed\n");
        return 1;
    }
    unsigned long long* d_out;
    cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
    cudaFuncSetAttribute(proto, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // {mma warp, epilogue warps, commits, halo, B fill}; halo 1 reads random bytes
    const int cfgs[][5] = {{19, 16, 2, 0, 0}, {19, 16, 2, 1, 0}, {19, 16, 2, 1, 1}, {19, 16, 2, 0, 1}};
    const char* halos[] = {"none", "TMA {64 B,114,4} SW64", "TMA {128 B,114,2} SW128"};
    for (const auto& c : cfgs) {
        proto<<<148, 640, smem>>>(m64, m128, units, c[0], c[1], c[2] == 2, c[3], c[4], d_out);
        proto<<<148, 640, smem>>>(m64, m128, units, c[0], c[1], c[2] == 2, c[3], c[4], d_out);
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
        }
        unsigned long long h[148];
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        double sum = 0;
        for (int i = 0; i < 148; ++i) sum += (double)h[i];
        printf("mma warp %2d, epilogue warps %2d, commits %d, halo %-24s, B %s: %.0f cycles per unit\n", c[0], c[1],
               c[2], halos[c[3]], c[4] ? "random diagonal" : "as found", sum / 148 / (units - 5));
    }
    return 0;
}
