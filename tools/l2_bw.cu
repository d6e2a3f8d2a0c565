// l2_bw.cu — per-SM bandwidth to / from an L2-resident buffer, the bound on
// the split-K exchange (each C1 rank writes and reads 48 KB).  128 CTAs, each
// moves BYTES through one path; in-kernel globaltimer span from the CTA's
// first issue to "all done", median over CTAs and reps.
//
//   st.v4   : 256 threads, st.global.cg.v4 from registers
//   st.v8   : 256 threads, st.global.v8.b32 (256-bit) from registers
//   bulk.st : cp.async.bulk.global.shared::cta from smem (one thread), wait_group 0
//   ld.v4   : 256 threads, ld.global.cg.v4, all loads in flight
//   bulk.ld : cp.async.bulk.shared::cta.global (one thread), mbarrier
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc l2_bw.cu -o l2_bw
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

template <int MODE>
__global__ void __launch_bounds__(256, 1) probe(uint8_t* buf, int bytes, unsigned long long* span) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ unsigned long long t0s;
    uint8_t* my = buf + (size_t)blockIdx.x * bytes;
    const uint32_t sbase = ptx::smem_u32(smem);
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) t0s = gtime();
    __syncthreads();
    const int per = bytes / 256;  // bytes per thread (register modes)
    uint32_t acc = 0;
    if (MODE == 0) {
        for (int off = threadIdx.x * 16; off < bytes; off += 256 * 16)
            asm volatile("st.global.cg.v4.u32 [%0], {%1,%1,%1,%1};" ::"l"(my + off), "r"(off) : "memory");
    } else if (MODE == 1) {
        for (int off = threadIdx.x * 32; off < bytes; off += 256 * 32)
            asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(my + off), "r"(off) : "memory");
    } else if (MODE == 2) {
        if (threadIdx.x == 0) {
            for (int off = 0; off < bytes; off += 16384)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(my + off),
                             "r"(sbase + (off % (96 * 1024))), "r"(16384)
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
    } else if (MODE == 3) {
        uint4 v[16];
        const int n = bytes / (256 * 16);  // <= 16 loads per thread, all in flight
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if (i < n)
                asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w)
                             : "l"(my + (size_t)(i * 256 + threadIdx.x) * 16));
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if (i < n) acc ^= v[i].x ^ v[i].w;
    } else if (MODE == 4) {
        if (threadIdx.x == 0) {
            ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar), (uint32_t)bytes);
            for (int off = 0; off < bytes; off += 16384)
                ptx::bulk_load(sbase + off, my + off, 16384, ptx::smem_u32(&bar));
            ptx::mbar_wait_spin(ptx::smem_u32(&bar), 0);
        }
    } else if (MODE == 5) {
        uint32_t v[8][8];
        const int n = bytes / (256 * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < n)
                asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(v[i][0]), "=r"(v[i][1]), "=r"(v[i][2]), "=r"(v[i][3]), "=r"(v[i][4]),
                               "=r"(v[i][5]), "=r"(v[i][6]), "=r"(v[i][7])
                             : "l"(my + (size_t)(i * 256 + threadIdx.x) * 32));
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i < n) acc ^= v[i][0] ^ v[i][7];
    }
    if (MODE <= 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // stores performed
    __syncthreads();
    if (threadIdx.x == 0) span[blockIdx.x] = gtime() - t0s;
    if (acc == 0x9u) span[blockIdx.x + 4096] = acc;
    (void)per;
}

int main() {
    const int ctas = 128;
    const char* names[] = {"st.cg.v4 (regs)", "st.v8 (regs)", "bulk S2G", "ld.cg.v4", "bulk G2S", "ld.cg.v8"};
    uint8_t* buf;
    unsigned long long* span;
    cudaMalloc(&buf, 64 << 20);
    cudaMemset(buf, 1, 64 << 20);
    cudaMalloc(&span, 8192 * 8);
    std::vector<unsigned long long> h(ctas);
    auto run = [&](auto kern, int mode, int bytes) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        std::vector<double> med;
        for (int rep = 0; rep < 7; ++rep) {
            kern<<<ctas, 256, 200 * 1024>>>(buf, bytes, span);
            cudaDeviceSynchronize();
            cudaMemcpy(h.data(), span, ctas * 8, cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.end());
            if (rep >= 2) med.push_back((double)h[ctas / 2]);
        }
        std::sort(med.begin(), med.end());
        const double ns = med[med.size() / 2];
        std::printf("%-16s %6d B/CTA: %7.0f ns median span -> %6.1f GB/s per SM (%5.1f B/clk @1.92GHz)  %s\n",
                    names[mode], bytes, ns, bytes / ns, bytes / ns / 1.92, cudaGetErrorString(cudaGetLastError()));
    };
    for (int bytes : {16384, 49152, 65536}) {
        run(probe<0>, 0, bytes);
        run(probe<1>, 1, bytes);
        run(probe<2>, 2, bytes);
        run(probe<3>, 3, bytes);
        run(probe<5>, 5, bytes);
        run(probe<4>, 4, bytes);
    }
    return 0;
}
