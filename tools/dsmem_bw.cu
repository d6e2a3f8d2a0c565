// dsmem_bw.cu — the split-K exchange pattern over distributed shared memory
// (VERDICT r1 "next" item 5: reduce the C1 partials into the owner CTA with
// cp.reduce.async.bulk ... .add instead of the L2 round trip).  148 CTAs in
// clusters of 4 (all SMs busy, as in C1); every CTA sends one 16 KB block
// (128 rows x 32 int32 columns) to each of its 3 peers and receives 3, then
// waits for its own incoming bytes.  Timed in-kernel with globaltimer from a
// cluster barrier to the CTA's last incoming byte; median / max over CTAs.
//   mode 0: cp.async.bulk shared::cta -> shared::cluster (copy into 3 slots)
//   mode 1: cp.reduce.async.bulk .add.u32 (all 3 peers add into one slot)
//   mode 2: st.async v4 from registers (copy into 3 slots)
//   mode 3: red.async .add.u32 v1 from registers... not available as a vector:
//           st.global.cg 48 KB to an L2 workspace + cluster barrier + ld.cg
//           48 KB (the round-1 path) for comparison
//   CHUNK: bytes per bulk op (16384 = one op per peer)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc dsmem_bw.cu -o dsmem_bw
#include <algorithm>
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace q8g;

constexpr int BLK = 16384;  // bytes per peer block
constexpr int S = 4;        // cluster size
constexpr int THREADS = 256;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(r));
    return d;
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int MODE>
__global__ void __cluster_dims__(S, 1, 1) __launch_bounds__(THREADS, 1)
    xchg(int chunk, uint8_t* ws, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    uint8_t* src = sm;                 // 3 blocks to send
    uint8_t* dst = sm + (S - 1) * BLK;  // 3 incoming slots (mode 1: slot 0 only)
    const uint32_t rank = cluster_rank();
    const uint32_t bar_a = ptx::smem_u32(&bar);
    for (int i = threadIdx.x; i < 2 * (S - 1) * BLK / 4; i += THREADS)
        reinterpret_cast<uint32_t*>(sm)[i] = i < (S - 1) * BLK / 4 ? i * 7u + rank : 0u;
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar_a, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (MODE <= 2) ptx::mbar_arrive_expect_tx(bar_a, (S - 1) * BLK);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    csync();
    const unsigned long long t0 = gtime();
    if (MODE == 0 || MODE == 1) {
        // one thread per peer issues its block in chunk-byte ops
        if (threadIdx.x < S - 1) {
            const uint32_t q = (rank + 1 + threadIdx.x) % S;
            const uint32_t slot = (rank + S - q) % S - 1;  // at q: slot of this source
            const uint32_t s = ptx::smem_u32(src + threadIdx.x * BLK);
            const uint32_t d = mapa(ptx::smem_u32(dst + (MODE == 1 ? 0 : slot * BLK)), q);
            const uint32_t b = mapa(bar_a, q);
            for (int off = 0; off < BLK; off += chunk) {
                if (MODE == 0)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            d + off),
                        "r"(s + off), "r"(chunk), "r"(b)
                        : "memory");
                else
                    asm volatile(
                        "cp.reduce.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes.add.u32 [%0], [%1], %2, [%3];" ::"r"(
                            d + off),
                        "r"(s + off), "r"(chunk), "r"(b)
                        : "memory");
            }
        }
    } else if (MODE == 2) {
        // every thread stores its share of the 3 blocks from registers
        for (int pi = 0; pi < S - 1; ++pi) {
            const uint32_t q = (rank + 1 + pi) % S;
            const uint32_t slot = (rank + S - q) % S - 1;
            const uint32_t d = mapa(ptx::smem_u32(dst + slot * BLK), q);
            const uint32_t b = mapa(bar_a, q);
            for (int i = threadIdx.x; i < BLK / 16; i += THREADS) {
                const uint4 v = reinterpret_cast<const uint4*>(src + pi * BLK)[i];
                asm volatile(
                    "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                        d + 16 * i),
                    "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(b)
                    : "memory");
            }
        }
    } else {
        // the L2 round trip: write the 3 blocks, cluster barrier, read 3 back
        uint8_t* base = ws + (size_t)blockIdx.x * (S - 1) * BLK;
        for (int i = threadIdx.x; i < (S - 1) * BLK / 16; i += THREADS) {
            const uint4 v = reinterpret_cast<const uint4*>(src)[i];
            asm volatile("st.global.cg.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(base + 16 * i), "r"(v.x), "r"(v.y),
                         "r"(v.z), "r"(v.w)
                         : "memory");
        }
        csync();
        const int peer_cta = (int)blockIdx.x - (int)rank + (int)((rank + 1) % S);
        const uint8_t* pb = ws + (size_t)peer_cta * (S - 1) * BLK;
        uint32_t acc = 0;
        for (int i = threadIdx.x; i < (S - 1) * BLK / 16; i += THREADS) {
            uint4 v;
            asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "l"(pb + 16 * i));
            acc += v.x + v.y + v.z + v.w;
        }
        reinterpret_cast<uint32_t*>(dst)[threadIdx.x] = acc;
        __syncthreads();
    }
    if (MODE <= 2) ptx::mbar_wait(bar_a, 0);
    __syncthreads();
    const unsigned long long t1 = gtime();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    csync();  // peers stay resident until every remote write has landed
}

template <int MODE>
static void run(int sms, int chunk, uint8_t* ws, unsigned long long* d_out, const char* name) {
    const int smem = 2 * (S - 1) * BLK;
    cudaFuncSetAttribute(xchg<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<double> med, mx;
    for (int rep = 0; rep < 20; ++rep) {
        xchg<MODE><<<sms, THREADS, smem>>>(chunk, ws, d_out);
        std::vector<unsigned long long> h(sms);
        cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        med.push_back(h[sms / 2] / 1e3);
        mx.push_back(h[sms - 1] / 1e3);
    }
    std::sort(med.begin(), med.end());
    std::sort(mx.begin(), mx.end());
    const double m = med[med.size() / 2], x = mx[mx.size() / 2];
    std::printf("%-44s chunk %5d: median CTA %.2f us, slowest %.2f us  (%.0f GB/s per SM out, median)  %s\n", name,
                chunk, m, x, (S - 1) * BLK / (m * 1e-6) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    sms -= sms % S;
    uint8_t* ws;
    unsigned long long* d_out;
    cudaMalloc(&ws, (size_t)sms * (S - 1) * BLK);
    cudaMalloc(&d_out, sms * 8);
    for (int chunk : {16384, 4096, 1024}) run<0>(sms, chunk, ws, d_out, "bulk copy smem->peer smem");
    for (int chunk : {16384, 4096, 1024}) run<1>(sms, chunk, ws, d_out, "bulk reduce-add smem->peer smem (.add.u32)");
    run<2>(sms, 16, ws, d_out, "st.async v4 registers->peer smem");
    run<3>(sms, 16, ws, d_out, "L2: st.cg 48 KB + cluster barrier + ld.cg");
    return 0;
}
