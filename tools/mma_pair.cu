// mma_pair.cu — tcgen05.mma.cta_group::2.kind::i8 (M = 256 over a CTA pair)
// vs cta_group::1 (M = 128) throughput for small N: is the ~55-cycle
// per-instruction floor of small-N MMAs paid per SM or per pair?  74 clusters
// of 2 CTAs; the leader issues 16 MMAs per commit, two commit groups in flight.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc mma_pair.cu -o mma_pair
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

template <int N, bool PAIR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32, 1) probe(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[2];
    __shared__ uint32_t tmem_slot;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t sA = base, sB = base + 65536;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bars[0]), 1);
        ptx::mbar_init(ptx::smem_u32(&bars[1]), 1);
        ptx::fence_mbar_init();
    }
    if (PAIR)
        ptx::tmem_alloc_pair<256>(ptx::smem_u32(&tmem_slot));
    else
        ptx::tmem_alloc<256>(ptx::smem_u32(&tmem_slot));
    ptx::tc_fence_before();
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    constexpr uint32_t idesc = ptx::idesc_u8s8_s32<PAIR ? 256 : 128, N>();
    uint64_t ad[16], bd[16];
    for (int j = 0; j < 16; ++j) {  // 16 distinct operand tiles
        ad[j] = ptx::sw128_kmajor_desc(sA + (uint32_t)((j % 4) * 32 + (j / 4) * 16384));
        bd[j] = ptx::sw128_kmajor_desc(sB + (uint32_t)((j % 4) * 32 + (j / 4) * 16384));
    }
    const bool issuer = !PAIR || rank == 0;
    if (issuer && threadIdx.x == 0) {
        const unsigned long long t0 = gtime();
        for (int i = 0; i < iters; ++i) {
            if (i >= 2) ptx::mbar_wait_spin(ptx::smem_u32(&bars[i & 1]), (uint32_t)((i / 2) - 1) & 1u);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (PAIR)
                    ptx::mma_i8_pair(tmem, ad[j], bd[j], idesc, 1);
                else
                    ptx::mma_i8(tmem, ad[j], bd[j], idesc, 1);
            }
            if (PAIR)
                ptx::tc_commit_pair_mc(ptx::smem_u32(&bars[i & 1]), (uint16_t)1);
            else
                ptx::tc_commit(ptx::smem_u32(&bars[i & 1]));
        }
        ptx::mbar_wait_spin(ptx::smem_u32(&bars[(iters - 1) & 1]), (uint32_t)(((iters - 1) / 2) & 1u));
        out[blockIdx.x] = gtime() - t0;
    }
    ptx::tc_fence_before();
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    ptx::tc_fence_after();
    if (PAIR)
        ptx::tmem_dealloc_pair<256>(tmem);
    else
        ptx::tmem_dealloc<256>(tmem);
}

int main() {
    unsigned long long* out;
    cudaMalloc(&out, 148 * 8);
    std::vector<unsigned long long> h(148);
    auto run = [&](auto kern, const char* nm) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        const int iters = 400;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(out, 0, 148 * 8);
            kern<<<148, 32, 200 * 1024>>>(iters, out);
        }
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
        std::vector<unsigned long long> v;
        for (auto x : h)
            if (x) v.push_back(x);
        std::sort(v.begin(), v.end());
        const double ns = v.empty() ? 0 : (double)v[v.size() / 2] / (iters * 16.0);
        std::printf("%-32s %6.1f ns per instruction (%5.1f cycles @1.9GHz)  %s\n", nm, ns, ns * 1.9, cudaGetErrorString(e));
    };
    run(probe<64, false>, "cta_group::1 M128 N64");
    run(probe<64, true>, "cta_group::2 M256 N64");
    run(probe<128, false>, "cta_group::1 M128 N128");
    run(probe<128, true>, "cta_group::2 M256 N128");
    run(probe<256, false>, "cta_group::1 M128 N256");
    run(probe<256, true>, "cta_group::2 M256 N256");
    return 0;
}
