// mma_bench.cu — cycles per tcgen05.mma.kind::i8 (M=128, K=32) from shared
// memory for several N and operand layouts (SWIZZLE_128B vs SWIZZLE_NONE
// K-major), one CTA, back-to-back issue from one elected thread.  Tuning tool.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc mma_bench.cu -o mma_bench
#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace q8g;

__device__ __forceinline__ uint64_t desc_noswz(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

template <int N>
__global__ void bench(int layout, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tptr;
    const uint32_t base = (ptx::smem_u32(smem) + 1023u) & ~1023u;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
    }
    if (threadIdx.x < 32) ptx::tmem_alloc<256>(ptx::smem_u32(&tptr));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tptr;
    constexpr uint32_t idesc = ptx::idesc_u8s8_s32<128, N>();
    const uint32_t a = base, b = base + 32768;
    uint64_t ad, bd;
    if (layout == 0) {  // SW128 K-major: 128-byte rows
        ad = ptx::sw128_kmajor_desc(a);
        bd = ptx::sw128_kmajor_desc(b);
    } else if (layout == 1) {  // no-swizzle K-major, K-halves far apart (LBO = 2 KB)
        ad = desc_noswz(a, 2048, 128);
        bd = desc_noswz(b, N * 16, 128);
    } else {  // no-swizzle, overlapping K-halves (LBO = 16 B: adjacent-pixel taps)
        ad = desc_noswz(a, 16, 128);
        bd = desc_noswz(b, N * 16, 128);
    }
    if (threadIdx.x < 32) {
        unsigned long long t0 = 0, t1 = 0;
        if (ptx::elect_one()) {
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
            if (layout == 6) {
                // conv3x3_tc swizzled pattern: A = SW64 rows of 64 B shifted by tap, 2 K-steps
                const int wp = 58;
                for (int i = 0; i < iters / 18; ++i)
                    for (int t = 0; t < 9; ++t) {
                        const int sh = (t / 3) * wp + (t % 3);
                        for (int j = 0; j < 2; ++j) {
                            const uint32_t aa = a + (uint32_t)(sh * 64 + j * 32);
                            const uint64_t ad6 = (uint64_t)((aa & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) |
                                                 ((uint64_t)(512 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
                            ptx::mma_i8(tmem, ad6, desc_noswz(b + (uint32_t)(((t * 2 + j) * 2) * N * 16) % 16384, N * 16, 128),
                                        idesc, (t | j) != 0);
                        }
                    }
            } else if (layout == 5) {
                // conv3x3_tc pattern: 9 taps x 2 K-steps, A = tap-shifted window of
                // plane pair (LBO = plane stride 3712 B), B steps 2*N*16 per (tap, j)
                const int wp = 58, plane = 3712;
                for (int i = 0; i < iters / 18; ++i)
                    for (int t = 0; t < 9; ++t) {
                        const int sh = (t / 3) * wp + (t % 3);
                        for (int j = 0; j < 2; ++j)
                            ptx::mma_i8(tmem, desc_noswz(a + (uint32_t)(2 * j * plane + sh * 16), plane, 128),
                                        desc_noswz(b + (uint32_t)(((t * 2 + j) * 2) * N * 16) % 16384, N * 16, 128),
                                        idesc, (t | j) != 0);
                    }
            } else if (layout >= 3) {
                // distinct operand windows per MMA (A advances 16 B .. 4 KB, B 512 B)
                const uint32_t astep = layout == 3 ? 1 : 256;  // 16-byte units
                for (int i = 0; i < iters; ++i)
                    ptx::mma_i8(tmem + (uint32_t)((i & 3) * N), desc_noswz(a + (uint32_t)((i & 15) * astep * 16), 2048, 128),
                                desc_noswz(b + (uint32_t)((i & 7) * 512), N * 16, 128), idesc, i > 3);
            } else {
                for (int i = 0; i < iters; ++i) ptx::mma_i8(tmem, ad, bd, idesc, i > 0);
            }
            ptx::tc_commit(ptx::smem_u32(&bar));
            ptx::mbar_wait(ptx::smem_u32(&bar), 0);
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
            out[0] = t1 - t0;
        }
        __syncwarp();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) ptx::tmem_dealloc<256>(tmem);
}

static int g_grid = 1;

template <int N>
void run(int layout, const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    const int iters = 2000;
    // 120 KB smem: one CTA per SM
    bench<N><<<g_grid, 128, 120 * 1024>>>(layout, iters, d);
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("N=%3d %-26s %7.1f cycles/MMA   A+B smem %5d B/MMA -> %6.1f B/cycle  %s\n", N, name,
                (double)cyc / iters, 128 * 32 + N * 32, (128.0 * 32 + N * 32) / ((double)cyc / iters),
                e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d);
}

int main(int argc, char** argv) {
    if (argc > 1) g_grid = atoi(argv[1]);
    std::printf("grid = %d CTAs\n", g_grid);
    const char* names[7] = {"SW128 K-major", "no-swizzle (LBO 2KB)", "no-swizzle (LBO 16B)",
                            "noswz A+16B/MMA, 4 D tiles", "noswz A+4KB/MMA, 4 D tiles", "conv3x3 pattern",
                            "conv3x3 SW64 pattern"};
    if (argc > 2) {
        run<80>(5, names[5]);
        run<32>(5, names[5]);
        run<80>(6, names[6]);
        run<32>(6, names[6]);
        run<144>(6, names[6]);
        run<80>(0, names[0]);
        return 0;
    }
    for (int l = 0; l < 5; ++l) {
        run<16>(l, names[l]);
        run<32>(l, names[l]);
        run<64>(l, names[l]);
        run<80>(l, names[l]);
        if (l < 3) {
            run<128>(l, names[l]);
            run<256>(l, names[l]);
        }
    }
    return 0;
}
