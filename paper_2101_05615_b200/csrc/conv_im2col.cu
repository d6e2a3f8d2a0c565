// conv_im2col.cu — conv3x3 for the shapes the implicit-GEMM kernel
// (conv_tc.cu) cannot hold in shared memory (C not in {32, 64, 128}, OC > 240,
// W + 2 > 64): an explicit im2col into a device workspace, then the
// tensor-core GEMM with its fused requant epilogue.
//
// Semantics are the conv entry's: row (n, oh, ow) of the
// im2col matrix is [tap (kh, kw)][channel] with k = (kh*3 + kw)*C + c, padded
// taps read zp_a (so they count in the row sums exactly as in conv_tc.cu and
// the oracle), and columns 9C .. K'-1 (K' = 9C rounded up to 16 for the TMA
// row pitch) are zero.  The packed weight is the conv's own [9C x OC] pack,
// whose K padding rows are zero, so the GEMM over K' equals the GEMM over 9C;
// the epilogue's K*zp_a*zp_b term uses the caller's k_total (= 9C).  Output
// C[M x OC] row-major with ldc = OC is the NHWC y.
//
// Cost: the workspace write + read (9C per output pixel) on top of the conv's
// own traffic, bounded to 256 MB per chunk of images; the GEMM runs at the
// tensor-core rates of gemm_tc.cu / gemm_tc2w.cu / gemm_splitk.cu.
#include <cstdint>
#include <map>
#include <mutex>

#include "q8g_internal.cuh"

namespace q8g {
namespace {

// one thread = 16 output bytes of one im2col row (C % 16 == 0: a 16-byte
// chunk never straddles a tap), else one byte
template <bool VEC>
__global__ void im2col_kernel(const uint8_t* __restrict__ x, int h, int w, int c, uint8_t zp_a, uint8_t* __restrict__ out,
                              long long rows, int kpad) {
    const int per_row = VEC ? kpad / 16 : kpad;
    const long long total = rows * per_row;
    const int kc = 9 * c;
    const uint32_t zp4 = 0x01010101u * zp_a;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / per_row;
        const int col = (int)(i % per_row) * (VEC ? 16 : 1);
        const int ow = (int)(row % w);
        const long long t1 = row / w;
        const int oh = (int)(t1 % h);
        const long long n = t1 / h;
        if (VEC) {
            uint4 v = make_uint4(0, 0, 0, 0);
            if (col < kc) {
                const int tap = col / c, ch = col % c;
                const int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
                if (ih >= 0 && ih < h && iw >= 0 && iw < w)
                    v = __ldg(reinterpret_cast<const uint4*>(x + (((size_t)n * h + ih) * w + iw) * c + ch));
                else
                    v = make_uint4(zp4, zp4, zp4, zp4);
            }
            *reinterpret_cast<uint4*>(out + (size_t)row * kpad + col) = v;
        } else {
            uint8_t v = 0;
            if (col < kc) {
                const int tap = col / c, ch = col % c;
                const int ih = oh + tap / 3 - 1, iw = ow + tap % 3 - 1;
                v = (ih >= 0 && ih < h && iw >= 0 && iw < w) ? x[(((size_t)n * h + ih) * w + iw) * c + ch] : zp_a;
            }
            out[(size_t)row * kpad + col] = v;
        }
    }
}

// per (device, stream) grow-only workspace (like the split-K exchange's);
// null during a capture if none large enough exists yet
uint8_t* im2col_workspace(int dev, cudaStream_t s, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, std::pair<uint8_t*, size_t>> ws;
    std::lock_guard<std::mutex> lock(mu);
    // bounded: at most 64 (device, stream) workspaces per process (an app
    // that creates streams per request would otherwise grow without bound);
    // further streams get none and take the workspace-free kernel
    if (ws.size() >= 64 && ws.find({dev, s}) == ws.end()) return nullptr;
    auto& slot = ws[{dev, s}];
    if (slot.second >= bytes) return slot.first;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusNone) return nullptr;
    uint8_t* buf = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    slot = {buf, bytes};  // a smaller predecessor stays allocated (may be in a graph)
    return buf;
}

constexpr size_t kChunkBytes = 256ull << 20;

}  // namespace

cudaError_t launch_conv3x3_im2col(const ConvArgs& a, cudaStream_t s) {
    const int kpad = (9 * a.c + 15) / 16 * 16;
    if (kpad > a.pw->kp) return cudaErrorNotSupported;
    const size_t img_rows = (size_t)a.h * a.w;
    const size_t img_bytes = img_rows * kpad;
    int per_chunk = (int)(kChunkBytes / img_bytes);
    if (per_chunk < 1) per_chunk = 1;
    if (per_chunk > a.nb) per_chunk = a.nb;
    int dev = 0;
    cudaGetDevice(&dev);
    uint8_t* ws = im2col_workspace(dev, s, (size_t)per_chunk * img_bytes);
    if (!ws) return cudaErrorNotSupported;  // caller falls back to the CUDA-core conv
    const int oc = a.pw->n;
    const bool vec = a.c % 16 == 0;
    for (int n0 = 0; n0 < a.nb; n0 += per_chunk) {
        const int nbc = a.nb - n0 < per_chunk ? a.nb - n0 : per_chunk;
        const long long rows = (long long)nbc * img_rows;
        const long long work = rows * (vec ? kpad / 16 : kpad);
        long long grid = (work + 255) / 256;
        if (grid > 8LL * sm_count(dev)) grid = 8LL * sm_count(dev);
        const uint8_t* xc = a.x + (size_t)n0 * img_rows * a.c;
        if (vec)
            im2col_kernel<true><<<(int)grid, 256, 0, s>>>(xc, a.h, a.w, a.c, (uint8_t)a.zp_a, ws, rows, kpad);
        else
            im2col_kernel<false><<<(int)grid, 256, 0, s>>>(xc, a.h, a.w, a.c, (uint8_t)a.zp_a, ws, rows, kpad);
        count_launch(kFamConvIm2col);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        GemmArgs g;
        g.a = ws;
        g.rows = (int)rows;
        g.k = kpad;
        g.lda = kpad;
        g.pb = a.pw;
        g.ep = a.ep;
        g.bias_add = nullptr;
        g.raw = a.raw;
        g.ldc = oc;
        g.c = a.raw ? (void*)((int32_t*)a.y + (size_t)n0 * img_rows * oc)
                    : (void*)((uint8_t*)a.y + (size_t)n0 * img_rows * oc);
        const int kind = default_tile_kind(g.rows, oc, kpad, true);
        e = (kind != kGeneric && tc_supported(g)) ? launch_gemm_tc(g, kind, s) : launch_gemm_simt(g, s);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace q8g
