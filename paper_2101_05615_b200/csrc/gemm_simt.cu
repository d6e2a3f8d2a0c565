// gemm_simt.cu — generic CUDA-core GEMM (dp4a.u32.s32) with the fused
// requant / raw-int32 epilogue.
//
// Role: the dispatch cache's "generic" tile (dispatch.hpp:121-123
// KernelCache(generic_only) analog): any M, N, K, any lda/ldc alignment.
// The tcgen05 kernels (gemm_tc.cu) take every shape TMA can address; this
// kernel covers the rest and is the equivalence check for them
// (test_engine.cpp:291-311).  Reads the same packed-B layout.
#include "q8g_internal.cuh"
#include "requant.cuh"

namespace q8g {
namespace {

constexpr int BM = 64, BN = 64, THREADS = 256;
constexpr int KW = kKBlock / 4;  // 32 words of K per k-block

__device__ __forceinline__ int32_t dp4a_us(uint32_t a, uint32_t b, int32_t c) {
    int32_t d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

template <int MODE>  // 0 raw i32, 1 requant F32_RNE, 2 requant REF
__global__ void __launch_bounds__(THREADS) gemm_simt_kernel(
    const uint8_t* __restrict__ a, int rows, int k, int lda, const int8_t* __restrict__ pb, int n,
    int np, int kp, const EpiRecord* __restrict__ rec, int32_t zp_c, int relu, int need_rowsum,
    const int32_t* __restrict__ bias_add, void* __restrict__ c, int ldc) {
    __shared__ uint32_t As[BM][KW + 1];
    __shared__ uint32_t Bs[BN][KW + 1];
    __shared__ int32_t rsum[BM];

    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

    int32_t acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0;
    int32_t my_rowsum = 0;

    const int nkb = kp / kKBlock;
    for (int kb = 0; kb < nkb; ++kb) {
        const int k0 = kb * kKBlock;
        // A tile: 64 rows x 128 bytes, byte loads (any lda alignment)
        for (int idx = tid; idx < BM * KW; idx += THREADS) {
            const int r = idx / KW, wd = idx % KW;
            const int gr = m0 + r;
            uint32_t word = 0;
            if (gr < rows) {
                const uint8_t* src = a + (size_t)gr * lda + k0 + wd * 4;
#pragma unroll
                for (int bb = 0; bb < 4; ++bb)
                    if (k0 + wd * 4 + bb < k) word |= (uint32_t)src[bb] << (8 * bb);
            }
            As[r][wd] = word;
        }
        // B tile: 64 channels x 128 bytes from the packed layout (unswizzle)
        for (int idx = tid; idx < BN * KW; idx += THREADS) {
            const int nn = idx / KW, wd = idx % KW;
            const int gn = n0 + nn;  // < np always (np % 256 == 0, grid covers n only)
            const int slot = (wd / 4) ^ (gn & 7);
            Bs[nn][wd] = *reinterpret_cast<const uint32_t*>(pb + ((size_t)kb * np + gn) * kKBlock +
                                                              slot * 16 + (wd % 4) * 4);
        }
        __syncthreads();
        if (need_rowsum && tid < BM) {
#pragma unroll 8
            for (int wd = 0; wd < KW; ++wd) my_rowsum = dp4a_us(As[tid][wd], 0x01010101u, my_rowsum);
        }
#pragma unroll 4
        for (int wd = 0; wd < KW; ++wd) {
            uint32_t av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[ty + 16 * i][wd];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[tx + 16 * j][wd];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = dp4a_us(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    if (tid < BM) rsum[tid] = my_rowsum;
    __syncthreads();

#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = ty + 16 * i, gr = m0 + r;
        if (gr >= rows) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx + 16 * j;
            if (gn >= n) continue;
            if (MODE == 0) {
                int32_t v = acc[i][j];
                if (bias_add) v = (int32_t)((uint32_t)v + (uint32_t)bias_add[gn]);
                reinterpret_cast<int32_t*>(c)[(size_t)gr * ldc + gn] = v;
            } else {
                const EpiRecord rc = rec[gn];
                const int32_t adj = adjust(acc[i][j], rsum[r], rc);
                const uint32_t q = MODE == 1 ? requant_f32(adj, rc.mf, zp_c, relu)
                                             : requant_ref(adj, rc.md, zp_c, relu);
                reinterpret_cast<uint8_t*>(c)[(size_t)gr * ldc + gn] = (uint8_t)q;
            }
        }
    }
}

}  // namespace

cudaError_t launch_gemm_simt(const GemmArgs& g, cudaStream_t s) {
    dim3 grid(ceil_div_i(g.pb->n, BN), ceil_div_i(g.rows, BM));
    const int8_t* pb = g.pb->data;
    if (g.raw) {
        gemm_simt_kernel<0><<<grid, THREADS, 0, s>>>(g.a, g.rows, g.k, g.lda, pb, g.pb->n,
                                                     g.pb->np, g.pb->kp, nullptr, 0, 0, 0,
                                                     g.bias_add, g.c, g.ldc);
    } else if (g.ep->rounding == Q8G_ROUND_F32_RNE) {
        gemm_simt_kernel<1><<<grid, THREADS, 0, s>>>(g.a, g.rows, g.k, g.lda, pb, g.pb->n,
                                                     g.pb->np, g.pb->kp, g.ep->rec, g.ep->zp_c,
                                                     g.ep->relu, g.ep->need_rowsum, nullptr, g.c,
                                                     g.ldc);
    } else {
        gemm_simt_kernel<2><<<grid, THREADS, 0, s>>>(g.a, g.rows, g.k, g.lda, pb, g.pb->n,
                                                     g.pb->np, g.pb->kp, g.ep->rec, g.ep->zp_c,
                                                     g.ep->relu, g.ep->need_rowsum, nullptr, g.c,
                                                     g.ldc);
    }
    count_launch(kFamGemmSimt);
    return cudaGetLastError();
}

}  // namespace q8g
