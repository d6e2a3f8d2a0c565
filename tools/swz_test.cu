// swz_test.cu — does tcgen05.mma read a K-major SWIZZLE_{32,64,128}B operand
// correctly when the descriptor start is shifted by an arbitrary number of
// rows (a shifted-window implicit-GEMM A operand), and what base_offset
// must be?  One CTA: A = [rows][S bytes] u8 written with the TMA swizzle
// (16-B chunk index ^= smem address bits [7..]), B = N16 x K32 s8 no-swizzle,
// D = M128 x N16 s32, compared with a host reference for every (shift, K-step).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2101_05615_b200/csrc swz_test.cu -o swz_test
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ptx.cuh"

using namespace q8g;

constexpr int ROWS = 160;

__device__ __forceinline__ uint64_t desc_noswz(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

// S = swizzle span = row bytes; layout codes (bits 61-63): 128B = 2, 64B = 4, 32B = 6
__device__ __forceinline__ uint64_t desc_swz(uint32_t addr, int S, uint32_t base_off) {
    const uint64_t code = S == 128 ? 2 : S == 64 ? 4 : 6;
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)((8 * S) >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)(base_off & 7) << 49) | (code << 61);
}

__global__ void k(const uint8_t* A, const int8_t* B, int S, int shift, int j, int bomode, int32_t* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tptr;
    const uint32_t raw = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* sm = smem_raw + (base - raw);
    const int bits = S == 128 ? 3 : S == 64 ? 2 : 1;
    // A with the TMA swizzle pattern
    for (int i = threadIdx.x; i < ROWS * S / 16; i += blockDim.x) {
        const int r = i / (S / 16), c = i % (S / 16);
        const uint32_t logical = (uint32_t)(r * S + c * 16);
        const uint32_t phys = logical ^ (((logical >> 7) & ((1u << bits) - 1)) << 4);
        *reinterpret_cast<uint4*>(sm + phys) = *reinterpret_cast<const uint4*>(A + (size_t)r * S + c * 16);
    }
    // B: [khalf][n 16][16 B]
    uint8_t* bs = sm + ROWS * S + 1024;
    bs = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(bs) + 1023) & ~(uintptr_t)1023);
    const uint32_t baddr = base + (uint32_t)(bs - sm);
    for (int i = threadIdx.x; i < 32; i += blockDim.x) {
        const int h = i / 16, n = i % 16;
        for (int b = 0; b < 16; ++b) bs[(h * 16 + n) * 16 + b] = (uint8_t)B[n * 32 + h * 16 + b];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
    }
    if (threadIdx.x < 32) ptx::tmem_alloc<32>(ptx::smem_u32(&tptr));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tptr;
    if (threadIdx.x < 32) {
        if (ptx::elect_one()) {
            const uint32_t a = base + (uint32_t)(shift * S + j * 32);
            const uint32_t bo = bomode == 0 ? 0u : bomode == 1 ? ((a >> 7) & 7u) : (((a >> 7) & 7u) & ((1u << bits) - 1));
            ptx::mma_i8(tmem, desc_swz(a, S, bo), desc_noswz(baddr, 256, 128), ptx::idesc_u8s8_s32<128, 16>(), false);
            ptx::tc_commit(ptx::smem_u32(&bar));
        }
        __syncwarp();
    }
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    ptx::tc_fence_after();
    uint32_t v[16];
    const int w = threadIdx.x / 32;
    ptx::tmem_ld_32x32b_x16(tmem + ((uint32_t)(w * 32) << 16), v);
    ptx::tmem_ld_wait();
    for (int n = 0; n < 16; ++n) out[threadIdx.x * 16 + n] = (int32_t)v[n];
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) ptx::tmem_dealloc<32>(tmem);
}

int main() {
    std::vector<uint8_t> A(ROWS * 128);
    std::vector<int8_t> B(16 * 32);
    srand(1);
    for (auto& x : A) x = (uint8_t)(rand() & 255);
    for (auto& x : B) x = (int8_t)(rand() & 255);
    uint8_t* dA;
    int8_t* dB;
    int32_t* dO;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dO, 128 * 16 * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    std::vector<int32_t> o(128 * 16);
    for (int S : {32, 64, 128}) {
        for (int bomode = 0; bomode < 3; ++bomode) {
            int bad_cfg = 0, tot = 0;
            for (int shift = 0; shift < 16; ++shift)
                for (int j = 0; j < S / 32; ++j) {
                    k<<<1, 128, 64 * 1024>>>(dA, dB, S, shift, j, bomode, dO);
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) {
                        std::printf("cuda error %s\n", cudaGetErrorString(e));
                        return 1;
                    }
                    cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
                    int bad = 0;
                    for (int m = 0; m < 128; ++m)
                        for (int n = 0; n < 16; ++n) {
                            int32_t ref = 0;
                            for (int kk = 0; kk < 32; ++kk)
                                ref += (int32_t)A[(size_t)(m + shift) * S + j * 32 + kk] * (int32_t)B[n * 32 + kk];
                            bad += ref != o[m * 16 + n];
                        }
                    ++tot;
                    if (bad) ++bad_cfg;
                    if (bad && bad_cfg <= 3) std::printf("  S=%d bomode=%d shift=%d j=%d: %d/2048 wrong\n", S, bomode, shift, j, bad);
                }
            std::printf("S=%3d base_offset mode %d: %d/%d (shift, kstep) configs wrong\n", S, bomode, bad_cfg, tot);
        }
    }
    return 0;
}
