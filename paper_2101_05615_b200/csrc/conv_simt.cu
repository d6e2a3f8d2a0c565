// conv_simt.cu — 3x3 / stride 1 / pad 1 NHWC convolution as an implicit GEMM
// on CUDA cores (dp4a), the generic path for any C and the parity vehicle
// for the tcgen05 conv kernel (conv_tc.cu).
//
// No reference symbol: im2col is an explicit non-goal of the reference
// (SPEC.md:194).  Semantics are SURVEY.md App. A D2: GEMM rows are output
// pixels (n, oh, ow) in NHWC order, k = (kh*3 + kw)*C + c, padded taps read
// zp_a (the quantized real zero) and count in the row sums; weights are the
// packed K=9C x N=OC matrix.
#include "q8g_internal.cuh"
#include "requant.cuh"
#include "ptx.cuh"

namespace q8g {
namespace {

constexpr int BM = 64, BN = 64, THREADS = 256;
constexpr int KW = kKBlock / 4;

template <int MODE>  // 0 raw, 1 F32_RNE, 2 REF
__global__ void __launch_bounds__(THREADS) conv3x3_simt_kernel(
    const uint8_t* __restrict__ x, int nb, int h, int w, int c, int32_t zp_a,
    const int8_t* __restrict__ pb, int n, int np, int kp, const EpiRecord* __restrict__ rec,
    int32_t zp_c, int relu, int need_rowsum, void* __restrict__ y) {
    __shared__ uint32_t As[BM][KW + 1];
    __shared__ uint32_t Bs[BN][KW + 1];
    __shared__ int32_t rsum[BM];
    const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
    const int rows = nb * h * w;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int ktot = 9 * c;
    int32_t acc[4][4] = {};
    int32_t my_rowsum = 0;
    for (int kb = 0; kb < kp / kKBlock; ++kb) {
        const int k0 = kb * kKBlock;
        for (int idx = tid; idx < BM * KW; idx += THREADS) {
            const int r = idx / KW, wd = idx % KW;
            const int gr = m0 + r;
            uint32_t word = 0;
            if (gr < rows) {
                const int img = gr / (h * w), rem = gr % (h * w);
                const int oh = rem / w, ow = rem % w;
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) {
                    const int kk = k0 + wd * 4 + bb;
                    uint32_t v = 0;
                    if (kk < ktot) {
                        const int tap = kk / c, ci = kk % c;
                        const int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
                        v = (ih >= 0 && ih < h && iw >= 0 && iw < w)
                                ? x[(((size_t)img * h + ih) * w + iw) * c + ci]
                                : (uint32_t)zp_a;
                    }
                    word |= v << (8 * bb);
                }
            }
            As[r][wd] = word;
        }
        for (int idx = tid; idx < BN * KW; idx += THREADS) {
            const int nn = idx / KW, wd = idx % KW;
            const int gn = n0 + nn;
            const int slot = (wd / 4) ^ (gn & 7);
            Bs[nn][wd] = *reinterpret_cast<const uint32_t*>(pb + ((size_t)kb * np + gn) * kKBlock +
                                                              slot * 16 + (wd % 4) * 4);
        }
        __syncthreads();
        if (need_rowsum && tid < BM)
            for (int wd = 0; wd < KW; ++wd) my_rowsum = ptx::dp4a_us(As[tid][wd], 0x01010101u, my_rowsum);
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
                for (int j = 0; j < 4; ++j) acc[i][j] = ptx::dp4a_us(av[i], bv[j], acc[i][j]);
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
                reinterpret_cast<int32_t*>(y)[(size_t)gr * n + gn] = acc[i][j];
            } else {
                const EpiRecord rc = rec[gn];
                const int32_t adj = adjust(acc[i][j], rsum[r], rc);
                const uint32_t q = MODE == 1 ? requant_f32(adj, rc.mf, zp_c, relu)
                                             : requant_ref(adj, rc.md, zp_c, relu);
                reinterpret_cast<uint8_t*>(y)[(size_t)gr * n + gn] = (uint8_t)q;
            }
        }
    }
}

}  // namespace

cudaError_t launch_conv3x3_simt(const ConvArgs& a, cudaStream_t s) {
    const int rows = a.nb * a.h * a.w;
    dim3 grid(ceil_div_i(a.pw->n, BN), ceil_div_i(rows, BM));
    const q8g_packed_b* pw = a.pw;
    if (a.raw)
        conv3x3_simt_kernel<0><<<grid, THREADS, 0, s>>>(a.x, a.nb, a.h, a.w, a.c, a.zp_a, pw->data, pw->n,
                                                        pw->np, pw->kp, nullptr, 0, 0, 0, a.y);
    else if (a.ep->rounding == Q8G_ROUND_F32_RNE)
        conv3x3_simt_kernel<1><<<grid, THREADS, 0, s>>>(a.x, a.nb, a.h, a.w, a.c, a.zp_a, pw->data, pw->n,
                                                        pw->np, pw->kp, a.ep->rec, a.ep->zp_c, a.ep->relu,
                                                        a.ep->need_rowsum, a.y);
    else
        conv3x3_simt_kernel<2><<<grid, THREADS, 0, s>>>(a.x, a.nb, a.h, a.w, a.c, a.zp_a, pw->data, pw->n,
                                                        pw->np, pw->kp, a.ep->rec, a.ep->zp_c, a.ep->relu,
                                                        a.ep->need_rowsum, a.y);
    count_launch(kFamConvSimt);
    return cudaGetLastError();
}

cudaError_t launch_conv3x3(const ConvArgs& a, cudaStream_t s) {
    // implicit GEMM when its operands fit shared memory, else im2col + the
    // tensor-core GEMM; the CUDA-core kernel when neither can run (no
    // workspace during a capture).  Q8G_CONV_SIMT=1 forces it (A/B checks).
    if (getenv("Q8G_CONV_SIMT") == nullptr) {
        if (conv_tc_supported(a)) return launch_conv3x3_tc(a, s);
        const cudaError_t e = launch_conv3x3_im2col(a, s);
        if (e != cudaErrorNotSupported) return e;
    }
    return launch_conv3x3_simt(a, s);
}

}  // namespace q8g
