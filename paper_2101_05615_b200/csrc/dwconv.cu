// dwconv.cu — depthwise 3x3 / stride 1 / pad 1 NHWC, bandwidth-bound path
// (BASELINE config C4).  No reference symbol: semantics are SURVEY.md App. A
// D3 — acc[n,h,w,c] = sum_taps x*w[tap,c] with padded taps reading zp_a,
// adj = acc - zp_w[c]*sum_taps x + c_term[c], per-channel fp32 requant.
#include "ptx.cuh"
#include "q8g_internal.cuh"
#include "requant.cuh"

namespace q8g {
namespace {

// one thread = 4 channels (one 32-bit word) of one output pixel
__global__ void __launch_bounds__(256) dw_simple_kernel(const uint8_t* __restrict__ x, int nb, int h, int w,
                                                        int c, int32_t zp_a, const int8_t* __restrict__ wt,
                                                        const EpiRecord* __restrict__ rec, int32_t zp_c,
                                                        int relu, uint8_t* __restrict__ y) {
    const int cw = c / 4;
    const size_t total = (size_t)nb * h * w * cw;
    const uint32_t pad = (uint32_t)zp_a * 0x01010101u;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int q = (int)(idx % cw);
        const size_t px = idx / cw;
        const int img = (int)(px / ((size_t)h * w));
        const int rem = (int)(px % ((size_t)h * w));
        const int oh = rem / w, ow = rem % w;
        int32_t acc[4] = {0, 0, 0, 0}, xs[4] = {0, 0, 0, 0};
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
            const int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
            uint32_t xv = pad;
            if (ih >= 0 && ih < h && iw >= 0 && iw < w)
                xv = __ldg(reinterpret_cast<const uint32_t*>(x + (((size_t)img * h + ih) * w + iw) * c) + q);
            const uint32_t wv = __ldg(reinterpret_cast<const uint32_t*>(wt + tap * c) + q);
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int32_t xb = (xv >> (8 * b)) & 255;
                const int32_t wb = (int32_t)(int8_t)(wv >> (8 * b));
                acc[b] += xb * wb;
                xs[b] += xb;
            }
        }
        uint32_t out = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int4 r4 = __ldg(reinterpret_cast<const int4*>(rec + q * 4 + b));
            EpiRecord rc;
            rc.c = r4.x;
            rc.zpb = r4.y;
            const int32_t adj = adjust(acc[b], xs[b], rc);
            out |= requant_f32(adj, __int_as_float(r4.z), zp_c, relu) << (8 * b);
        }
        reinterpret_cast<uint32_t*>(y + px * c)[q] = out;
    }
}

// generic (C % 4 != 0): one thread per output element
__global__ void dw_scalar_kernel(const uint8_t* __restrict__ x, int nb, int h, int w, int c, int32_t zp_a,
                                 const int8_t* __restrict__ wt, const EpiRecord* __restrict__ rec,
                                 int32_t zp_c, int relu, uint8_t* __restrict__ y) {
    const size_t total = (size_t)nb * h * w * c;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const int ch = (int)(idx % c);
        const size_t px = idx / c;
        const int img = (int)(px / ((size_t)h * w));
        const int rem = (int)(px % ((size_t)h * w));
        const int oh = rem / w, ow = rem % w;
        int32_t acc = 0, xs = 0;
        for (int tap = 0; tap < 9; ++tap) {
            const int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
            int32_t xv = zp_a;
            if (ih >= 0 && ih < h && iw >= 0 && iw < w) xv = x[(((size_t)img * h + ih) * w + iw) * c + ch];
            acc += xv * (int32_t)wt[tap * c + ch];
            xs += xv;
        }
        const EpiRecord rc = rec[ch];
        y[idx] = (uint8_t)requant_f32(adjust(acc, xs, rc), rc.mf, zp_c, relu);
    }
}

}  // namespace

cudaError_t launch_dwconv3x3(const uint8_t* x, int nb, int h, int w, int c, const q8g_dw_filter* f,
                             uint8_t* y, cudaStream_t s) {
    // order: the 64-channel tensor-core kernel (fastest where it fits: W + 2 <= 128),
    // the FMA-pipe kernel (C % 128 == 0, any width), the 16-channel tensor-core
    // kernel, the plain CUDA-core kernel.  A/B switches: Q8G_DW_SIMT forces the
    // last; Q8G_DW_FMA=1 / =0 forces / disables the FMA-pipe kernel.
    const bool simt = getenv("Q8G_DW_SIMT") != nullptr;
    const char* fenv = getenv("Q8G_DW_FMA");
    const bool fma_ok = !simt && f->fma_w && dw_fma_supported(h, w, c) && !(fenv && fenv[0] == '0');
    const bool tc_ok = !simt && f->tc_ok && dw_tc_supported(h, w, c, f->zp_a);
    if (fma_ok && fenv && fenv[0] == '1') return launch_dwconv3x3_fma(x, nb, h, w, c, f, y, s);
    if (tc_ok && dw_tc64_supported(w, c)) return launch_dwconv3x3_tc(x, nb, h, w, c, f, y, s);
    if (fma_ok) return launch_dwconv3x3_fma(x, nb, h, w, c, f, y, s);
    if (tc_ok) return launch_dwconv3x3_tc(x, nb, h, w, c, f, y, s);
    int dev = 0;
    cudaGetDevice(&dev);
    const int blocks = sm_count(dev) * 8;
    if (c % 4 == 0)
        dw_simple_kernel<<<blocks, 256, 0, s>>>(x, nb, h, w, c, f->zp_a, f->w, f->rec, f->zp_c, f->relu, y);
    else
        dw_scalar_kernel<<<blocks, 256, 0, s>>>(x, nb, h, w, c, f->zp_a, f->w, f->rec, f->zp_c, f->relu, y);
    count_launch(kFamDw);
    return cudaGetLastError();
}

}  // namespace q8g
