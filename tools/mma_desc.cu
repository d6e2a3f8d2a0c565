// mma_desc.cu — tcgen05.mma.kind::i8 M128 x N80 x K32 throughput (cycles per
// instruction, 148 CTAs, one issuing thread, two commit groups in flight) as
// a function of the operand layouts the conv3x3 kernel uses:
//   A: SWIZZLE_128B (128-byte rows) or SWIZZLE_64B (64-byte rows, = C) with
//      the start shifted by 0..7 rows (tap-shifted windows);
//   B: SWIZZLE_128B or no-swizzle K-major (core matrices, LBO = N*16).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc mma_desc.cu -o mma_desc
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

__device__ inline uint64_t swz_desc(uint32_t addr, int S) {
    const uint64_t code = S == 128 ? 2 : S == 64 ? 4 : 6;
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)((8 * S) >> 4) << 32) |
           ((uint64_t)1 << 46) | (code << 61);
}
__device__ inline uint64_t noswz_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

template <int N>
__global__ void __launch_bounds__(160, 1) probe(int a_s, int a_shift, int b_swz, int iters, unsigned long long* out,
                                               int readers) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[2];
    __shared__ uint32_t tmem_slot;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t sA = base + 1024, sB = base + 65536;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bars[0]), 1);
        ptx::mbar_init(ptx::smem_u32(&bars[1]), 1);
        ptx::fence_mbar_init();
    }
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    if (threadIdx.x < 32) ptx::tmem_alloc<512>(ptx::smem_u32(&tmem_slot));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x >= 32) {
        // TMEM readers (an epilogue's tcgen05.ld traffic) on columns 256..
        const int w = threadIdx.x / 32 - 1;
        uint32_t acc = 0;
        const bool same_smsp = (threadIdx.x / 32) % 4 == 0;  // shares SMSP 0 with the MMA thread (warp 0)
        if (readers >= 2 && !(readers == 6 && same_smsp)) {
            // ALU-busy warps (an epilogue's integer / fp work, high ILP)
            float f[8];
            for (int i = 0; i < 8; ++i) f[i] = (float)(threadIdx.x + i);
            while (!done) {
#pragma unroll
                for (int r = 0; r < 64; ++r)
#pragma unroll
                    for (int i = 0; i < 8; ++i) f[i] = __fmaf_rn(f[i], 1.0001f, 0.5f);
                if (readers == 3) __nanosleep(0);
                if (readers == 4) __nanosleep(100);
                if (readers == 7 && same_smsp) __nanosleep(100);
                if (readers == 8 && same_smsp) __nanosleep(0);
                if (readers == 9) __nanosleep(5000);  // ~12% duty: a 512-FMA-chain burst, then ~5 us idle
                if (readers == 10) __nanosleep(1500);
            }
            for (int i = 0; i < 8; ++i) acc += __float_as_uint(f[i]);
        } else if (readers)
            while (!done) {
                uint32_t v[16];
                ptx::tmem_ld_32x32b_x16(tmem_slot + ((uint32_t)(w * 32) << 16) + 256 + (acc & 63), v);
                ptx::tmem_ld_wait();
                acc += v[0] ^ v[15];
            }
        if (acc == 0x12345u) out[200] = acc;
        ptx::tc_fence_before();
        __syncthreads();
        return;
    }
    const uint32_t tmem = tmem_slot;
    constexpr uint32_t idesc = ptx::idesc_u8s8_s32<128, N>();
    // distinct: 16 different operand tiles (as the conv's 9 taps x 2 K-steps)
    // instead of 4 reused ones
    const int nd = a_shift < 0 ? 16 : 4;
    const int shift = a_shift < 0 ? 0 : a_shift;
    uint64_t ad[16], bd[16];
    for (int j = 0; j < 16; ++j) {
        const int jj = j % nd;
        if (a_shift < 0) {  // conv-like: window of tap jj/2 (shift (jj/2) rows), K-step jj%2 of a 64-byte row
            ad[j] = swz_desc(sA + (uint32_t)((jj / 2) * 58 * a_s / 8 + (jj % 2) * 32), a_s);
            bd[j] = noswz_desc(sB + (uint32_t)(jj * 2 * N * 16), (uint32_t)(N * 16), 128);
            continue;
        }
        // K-step jj (32 bytes): within a row of a_s bytes, then the next K block
        const int within = (jj * 32) % a_s, blk = (jj * 32) / a_s;
        ad[j] = swz_desc(sA + (uint32_t)(shift * a_s + within + blk * 128 * a_s), a_s);
        bd[j] = b_swz ? swz_desc(sB + (uint32_t)(jj * 32), 128)
                      : noswz_desc(sB + (uint32_t)(jj * 2 * N * 16), (uint32_t)(N * 16), 128);
    }
    if (threadIdx.x == 0) {
        const unsigned long long t0 = gtime();
        const long long c0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (i >= 2) ptx::mbar_wait_spin(ptx::smem_u32(&bars[i & 1]), (uint32_t)((i / 2) - 1) & 1u);
#pragma unroll
            for (int j = 0; j < 16; ++j) ptx::mma_i8(tmem, ad[j], bd[j], idesc, 1);
            ptx::tc_commit(ptx::smem_u32(&bars[i & 1]));
        }
        ptx::mbar_wait_spin(ptx::smem_u32(&bars[(iters - 1) & 1]), (uint32_t)(((iters - 1) / 2) & 1u));
        out[blockIdx.x] = gtime() - t0;
        out[148 + blockIdx.x % 100] = (unsigned long long)(clock64() - c0);
        done = 1;
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
}

int main() {
    unsigned long long* out;
    cudaMalloc(&out, 256 * 8);
    std::vector<unsigned long long> h(148);
    int readers = 0, iters_ = 400;
    auto run = [&](auto kern, int n, int a_s, int a_shift, int b_swz) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        const int iters = iters_;
        for (int rep = 0; rep < 3; ++rep) kern<<<148, 160, 200 * 1024>>>(a_s, a_shift, b_swz, iters, out, readers);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
        std::vector<unsigned long long> cyc(256);
        cudaMemcpy(cyc.data(), out, 256 * 8, cudaMemcpyDeviceToHost);
        const double ghz = (double)cyc[148] / (double)cyc[0];
        std::sort(h.begin(), h.end());
        std::printf("%-13s N=%3d  A SW%-3d shift %d rows  B %-9s: %6.1f ns/MMA, %6.1f cycles/MMA (SM clock %.2f GHz, %d MMAs)  %s\n",
                    readers >= 2 ? "+ALU warps" : readers ? "+TMEM readers" : "", n, a_s, a_shift, b_swz ? "SW128" : "no-swz", h[74] / (iters * 16.0),
                    h[74] * ghz / (iters * 16.0), ghz, iters * 16, cudaGetErrorString(e));
    };
    run(probe<80>, 80, 128, 0, 1);
    run(probe<80>, 80, 128, 0, 0);
    run(probe<80>, 80, 64, 0, 1);
    run(probe<80>, 80, 64, 0, 0);
    for (int sh : {1, 2, 3, 5, 7}) run(probe<80>, 80, 64, sh, 0);
    run(probe<80>, 80, 32, 0, 0);
    run(probe<80>, 80, 32, 3, 0);
    run(probe<64>, 64, 64, 0, 0);
    run(probe<64>, 64, 128, 0, 1);
    run(probe<128>, 128, 128, 0, 1);
    run(probe<256>, 256, 128, 0, 1);
    run(probe<80>, 80, 64, -1, 0);
    iters_ = 100000;  // ~0.3 s of sustained MMA: clocks under load
    run(probe<80>, 80, 64, -1, 0);
    run(probe<256>, 256, 128, 0, 1);
    iters_ = 400;
    for (readers = 2; readers <= 10; ++readers) {
        std::printf("ALU warps, yield mode %d (0 none, 1 nanosleep(0), 2 nanosleep(100), 3 = 0, 4 no ALU warp on the MMA SMSP, 5/6 nanosleep(100)/(0) only on the MMA SMSP, 7/8 bursts then nanosleep(5000)/(1500) on all) every 512 FMAs\n",
                    readers - 2);
        run(probe<80>, 80, 64, -1, 0);
        run(probe<256>, 256, 128, 0, 1);
    }
    readers = 1;
    run(probe<80>, 80, 64, -1, 0);
    run(probe<80>, 80, 64, 3, 0);
    run(probe<128>, 128, 128, 0, 1);
    run(probe<256>, 256, 128, 0, 1);
    return 0;
}
