// pack.cu — one-time weight prepack (the reference's prepack_weights,
// pack.hpp:146-196, and compute_col_offsets, quant.hpp:98-110).
//
// Reorders the K x N int8 weight (row-major, ldb) into the K-major,
// 128B-swizzled layout described in q8g_internal.cuh and computes, in the
// same pass, the int32 column sums and max|B| (pack.hpp:188-194).
#include "q8g_internal.cuh"

namespace q8g {
namespace {

constexpr int kPackN = 64;  // channels per CTA

// grid: (NP/64, KP/128); block 256 threads
__global__ void __launch_bounds__(256) pack_b_kernel(const int8_t* __restrict__ b, int k, int n,
                                                     int ldb, int8_t* __restrict__ packed, int np,
                                                     int32_t* __restrict__ colsum,
                                                     int* __restrict__ max_abs) {
    __shared__ int8_t tile[kKBlock][kPackN + 4];  // [k][n], padded rows
    const int n0 = blockIdx.x * kPackN;
    const int kb = blockIdx.y;
    const int k0 = kb * kKBlock;
    // coalesced load along n: 128 rows x 64 bytes
    int local_max = 0;
    for (int idx = threadIdx.x; idx < kKBlock * kPackN; idx += blockDim.x) {
        const int kk = idx / kPackN, nn = idx % kPackN;
        const int gk = k0 + kk, gn = n0 + nn;
        int8_t v = 0;
        if (gk < k && gn < n) v = b[(size_t)gk * ldb + gn];
        tile[kk][nn] = v;
        const int av = v < 0 ? -(int)v : (int)v;
        local_max = av > local_max ? av : local_max;
    }
    __syncthreads();
    // each (channel, 16B chunk) pair: 64 channels x 8 chunks = 512 items
    for (int item = threadIdx.x; item < kPackN * 8; item += blockDim.x) {
        const int nn = item / 8, ch = item % 8;
        const int gn = n0 + nn;
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t word = 0;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb)
                word |= (uint32_t)(uint8_t)tile[ch * 16 + q * 4 + bb][nn] << (8 * bb);
            w[q] = word;
        }
        const int slot = ch ^ (gn & 7);
        int8_t* dst = packed + ((size_t)kb * np + gn) * kKBlock + slot * 16;
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    // column sums over this k-block: one thread per channel
    if (threadIdx.x < kPackN) {
        const int nn = threadIdx.x;
        int32_t s = 0;
        for (int kk = 0; kk < kKBlock; ++kk) s += tile[kk][nn];
        if (n0 + nn < n) atomicAdd(&colsum[n0 + nn], s);
    }
    // max |B|
    for (int off = 16; off > 0; off >>= 1)
        local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, off));
    if ((threadIdx.x & 31) == 0) atomicMax(max_abs, local_max);
}

__global__ void unpack_b_kernel(const int8_t* __restrict__ packed, int k, int n, int np,
                                int8_t* __restrict__ out, int ldb) {
    const size_t total = (size_t)k * n;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int kk = (int)(idx / n), nn = (int)(idx % n);
        const int kb = kk / kKBlock, kin = kk % kKBlock;
        const int slot = (kin / 16) ^ (nn & 7);
        out[(size_t)kk * ldb + nn] = packed[((size_t)kb * np + nn) * kKBlock + slot * 16 + (kin % 16)];
    }
}

}  // namespace

cudaError_t launch_pack_b(const int8_t* b, int k, int n, int ldb, int8_t* packed, int kp, int np,
                          int32_t* colsum, int* max_abs, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(packed, 0, (size_t)kp * np, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(colsum, 0, sizeof(int32_t) * (size_t)np, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(max_abs, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
    dim3 grid(np / kPackN, kp / kKBlock);
    pack_b_kernel<<<grid, 256, 0, s>>>(b, k, n, ldb, packed, np, colsum, max_abs);
    count_launch(kFamPack);
    return cudaGetLastError();
}

cudaError_t launch_unpack_b(const int8_t* packed, int k, int n, int kp, int np, int8_t* out,
                            int ldb, cudaStream_t s) {
    (void)kp;
    const size_t total = (size_t)k * n;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    if (blocks < 1) blocks = 1;
    unpack_b_kernel<<<blocks, 256, 0, s>>>(packed, k, n, np, out, ldb);
    count_launch(kFamPack);
    return cudaGetLastError();
}

}  // namespace q8g
