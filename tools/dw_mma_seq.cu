// dw_mma_seq.cu — the depthwise kernel's per-unit tcgen05.mma sequence in
// isolation (148 CTAs, one issuing thread, no TMA, no epilogue): SM cycles per
// unit of 24 MMAs (input rows i = 3, 0, 1, 2 x kw x K-group, N = 64 / 128 /
// 128 / 64 into two row slots per K-group, A = SWIZZLE_64B halo windows,
// B = no-swizzle [K half][192 rows][16 B]).  Variants:
//   0  the kernel's sequence (accumulator buffer alternating per unit);
//   1  the same instructions, but every MMA writes its own D region
//      (no accumulation chain between consecutive MMAs);
//   2  the kernel's sequence with every N = 128 MMA replaced by N = 64;
//   3  variant 0 + 16 warps reading TMEM (the epilogue's tcgen05.ld traffic);
//   4  variant 0 + 16 warps storing / loading shared memory (STS.128 + LDS.128);
//   5  variant 0 + 16 warps of FP / integer ALU work (the requant arithmetic);
//   6  variant 0 with A rotating over 3 halo buffers at the kernel's stride.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc dw_mma_seq.cu -o dw_mma_seq
#include <cstdio>

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

__global__ void __launch_bounds__(544, 1) seq(int variant, int units, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_slot;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const int wp = 114, CB = 64, KG = 2;
    // halo buffers (4 rows + guard, the kernel's stride) then B
    const uint32_t hstride = (uint32_t)((4 * wp * CB + 1024 + 1023) / 1024 * 1024);
    const uint32_t sA = base + 1024, sB = sA + 3 * hstride;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
    }
    if (threadIdx.x < 32) ptx::tmem_alloc<512>(ptx::smem_u32(&tmem_slot));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (threadIdx.x >= 32) {
        // interference warps (quarter = warp % 4 for TMEM lane access)
        const int w = threadIdx.x / 32, q = w % 4;
        uint32_t sink = 0;
        float f0 = threadIdx.x, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3;
        while (!stop) {
            if (variant == 3) {
                uint32_t v[4][16];
#pragma unroll
                for (int c = 0; c < 4; ++c) ptx::tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 16), v[c]);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int c = 0; c < 4; ++c) sink += v[c][0] + v[c][15];
            } else if (variant == 4) {
                const uint32_t a = base + 140 * 1024 + (uint32_t)((w * 32 + threadIdx.x % 32) * 16);
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(a), "r"(sink) : "memory");
                    uint4 x;
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "r"(base + 190000u) : "memory");
                    sink += x.x;
                }
            } else if (variant == 5) {
#pragma unroll 16
                for (int r = 0; r < 64; ++r) {
                    f0 = f0 * 1.0001f + 0.5f;
                    f1 = f1 * 1.0001f + 0.5f;
                    f2 = fmaxf(f2 * 0.9999f, f3);
                    f3 = f3 + f0;
                    sink += __float_as_uint(f1) >> 3;
                }
            } else {
                break;
            }
        }
        if (sink == 0x12345678u && f3 == 1.0f) out[1000] = sink;
    } else {
    constexpr uint32_t idesc64 = ptx::idesc_u8s8_s32<128, 64>();
    constexpr uint32_t idesc128 = ptx::idesc_u8s8_s32<128, 128>();
    const uint64_t a0 = swz64_desc(sA);
    const uint64_t hstride16 = hstride >> 4;
    const uint64_t row16 = (uint64_t)(wp * CB / 16), pos16 = CB / 16;
    const uint64_t b0 = noswz_desc(sB, 192 * 16, 128);
    const uint32_t bar_a = ptx::smem_u32(&bar);
    long long t0 = 0;
    for (int u = 0; u < units; ++u) {
        if (u == 2) t0 = clock64();
        if (ptx::elect_one()) {
            const int acc = u & 1;
            int region = 0;
#pragma unroll
            for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                for (int kw = 0; kw < 3; ++kw)
#pragma unroll
                    for (int j = 0; j < KG; ++j) {
                        const int i = (ii + 3) % 4;
                        const uint64_t ad = a0 + (variant == 6 ? (uint64_t)(u % 3) * hstride16 : 0) +
                                            (uint64_t)i * row16 + (uint64_t)kw * pos16 + 2u * j;
                        const uint64_t bd = b0 + (uint64_t)((kw * KG + j) * 384);
                        uint32_t d = tmem + (uint32_t)(acc * 256 + j * 128);
                        if (variant == 1) d = tmem + (uint32_t)((region++ % 4) * 128);
                        const bool wide = (i == 1 || i == 2) && variant != 2;
                        const uint32_t idesc = wide ? idesc128 : idesc64;
                        if (i == 0) ptx::mma_i8(variant == 1 ? d : d + 64, ad, bd, idesc, kw != 0);
                        if (i == 1) ptx::mma_i8(d, ad, bd, idesc, 1);
                        if (i == 2) ptx::mma_i8(d, ad, bd + 64, idesc, 1);
                        if (i == 3) ptx::mma_i8(d, ad, bd + 128, idesc64, kw != 0);
                    }
            ptx::tc_commit(bar_a);
        }
        __syncwarp();
        // keep at most one unit of MMAs queued ahead (as the kernel's two accumulators)
        if (u >= 1) ptx::mbar_wait(bar_a, (uint32_t)((u - 1) & 1));
    }
    ptx::mbar_wait(bar_a, (uint32_t)((units - 1) & 1));
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    if (threadIdx.x == 0) stop = 1;
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tmem);
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int units = 200, smem = 200 * 1024;  // 3 halos + B below 130 KB; STS at 64 KB (variant 4 only)
    unsigned long long* d_out;
    cudaMalloc(&d_out, 148 * sizeof(unsigned long long));
    cudaFuncSetAttribute(seq, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"kernel sequence", "own D region per MMA", "all N = 64", "+ TMEM readers",
                           "+ shared-memory STS/LDS", "+ ALU warps", "A over 3 halo buffers"};
    cudaMalloc(&d_out, 1024 * sizeof(unsigned long long));
    for (int v = 0; v < 7; ++v) {
        seq<<<148, 544, smem>>>(v, units, d_out);
        seq<<<148, 544, smem>>>(v, units, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
        }
        unsigned long long h[148];
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < 148; ++i) s += (double)h[i];
        const double per_unit = s / 148 / (units - 2);
        printf("variant %d (%s): %.0f cycles per unit = %.1f cycles per MMA\n", v, names[v], per_unit, per_unit / 24);
    }
    return 0;
}
