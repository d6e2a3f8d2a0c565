// q8g_internal.cuh — shared internals of the B200 q8gemm library.
//
// Data layout in HBM:
//   packed B  : K padded to KP = round_up(K,128), N padded to NP =
//               round_up(N,256).  For k-block kb (128 bytes of K) and output
//               channel n, the 128 K-bytes of (kb, n) live at
//               ((kb * NP) + n) * 128, with 16-byte chunk ch stored at chunk
//               slot ch ^ (n & 7).  Every 8 channels form one 1024-byte
//               SWIZZLE_128B atom, so any tile of BN (multiple of 8) channels
//               of one k-block is a contiguous, pre-swizzled BN*128-byte run
//               that one cp.async.bulk drops into shared memory in exactly
//               the canonical tcgen05 K-major SW128 layout.
//   epilogue  : one 16-byte record per (padded) output column:
//               {int32 c, int32 zp_b, fp32 mult | fp64 mult}.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/q8g_b200.h"

namespace q8g {

constexpr int kKBlock = 128;  // bytes of K per pipeline stage / pack block
constexpr int kNPad = 256;    // output-channel padding of packed B

inline int round_up_i(int v, int m) { return ((v + m - 1) / m) * m; }
inline int ceil_div_i(int v, int d) { return (v + d - 1) / d; }

// ---- error plumbing ----
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
// per-kernel-family launch counters (q8g_launch_stats): evidence of which
// kernel actually ran
enum KernelFamily : int {
    kFamPack = 0,
    kFamGemmSimt = 1,
    kFamGemmTcSmallM = 2,
    kFamGemmTcLargeM = 3,
    kFamConvSimt = 4,
    kFamConvTc = 5,
    kFamDw = 6,
    kFamDwTc = 7,
    kFamPost = 8,        // general-pipeline post kernel (post.cu)
    kFamConvIm2col = 9,  // conv3x3 im2col for the GEMM path (conv_im2col.cu)
    kFamDwFma = 10,      // depthwise on the CUDA-core FMA pipes (dwconv_fma.cu)
    kFamPeerCopy = 11,   // copy-engine peer copies of a stripe (gemm_peers fallback; not a kernel)
    kFamCount = 12
};
void count_launch(int family);

#define Q8G_CUDA_TRY(expr)                                   \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return ::q8g::cuda_fail(_e, #expr); \
    } while (0)

// RAII device guard.  cudaSetDevice is called even when `dev` is already
// the current device: it makes the device's primary context current in a
// thread that has not used the runtime yet (a fresh caller thread), which the
// driver-level tensor-map encoder needs -- without it
// cuTensorMapEncodeTiled fails with CUDA_ERROR_INVALID_VALUE there.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

struct EpiRecord {  // 16 bytes, one per padded output column
    int32_t c;      // bias + bias_add - zp_a*colsum + K*zp_a*zp_b (mod 2^32)
    int32_t zpb;    // weight zero point of this column
    union {
        float mf;   // F32_RNE multiplier
        double md;  // REF multiplier (occupies bytes 8..15)
    };
};
static_assert(sizeof(EpiRecord) == 16, "EpiRecord must be 16 bytes");

}  // namespace q8g

struct q8g_packed_b {
    int device = 0;
    int k = 0, n = 0;   // logical K x N
    int kp = 0, np = 0; // padded
    int max_abs = 0;
    q8g_blocking blocking{};
    int8_t* data = nullptr;       // device, kp*np bytes
    int32_t* colsum_dev = nullptr; // device, np entries (zero beyond n)
    int32_t* colsum_host = nullptr;
    // conv3x3 tensor-core operand images (conv_tc.cu), one per input-channel
    // count C in {32, 64, 128}: the smem B layout followed by the per-tap
    // weight sums.  Built once, synchronously, under a lock
    // (q8g_conv3x3_prepare or the first conv call); conv_img_ready[i] is
    // published (release) only when the image is complete, and an image is
    // never rebuilt or freed before q8g_free_packed_b -- the weight stays
    // immutable and shareable across streams / threads (pack.hpp:59-62).
    uint8_t* conv_img[3] = {nullptr, nullptr, nullptr};
    int conv_img_ready[3] = {0, 0, 0};
};

struct q8g_epilogue {
    int device = 0;
    int n = 0, np = 0;
    int k_total = 0;
    int32_t zp_a = 0, zp_c = 0;
    int rounding = Q8G_ROUND_REF;
    int relu = 0;
    bool need_rowsum = false;  // any zp_b[j] != 0 (pipeline.hpp:114-119)
    // F32_RNE with 0 <= zp_c <= 255 and every multiplier finite, < 2^96: the
    // kernels may use the magic-add / saturating-pack requant (exact then)
    bool fast_f32 = false;
    q8g::EpiRecord* rec = nullptr;  // device, np records
};

// SparseWeightCSC (sparse.hpp:13-21) on the device
struct q8g_sparse_csc {
    int device = 0;
    int k = 0, n = 0, nnz = 0;
    int32_t* col_ptr = nullptr;  // n + 1
    int32_t* row_idx = nullptr;  // nnz
    int8_t* values = nullptr;    // nnz
};

struct q8g_dw_filter {
    int device = 0;
    int c = 0;
    int32_t zp_a = 0, zp_c = 0;
    int relu = 0;
    int8_t* w = nullptr;             // device [9][c]
    q8g::EpiRecord* rec = nullptr;   // device, c records (fp32 mult)
    // tensor-core path (dwconv_tc.cu); tc_ok false -> CUDA-core kernel
    bool tc_ok = false;
    int32_t* zpw_dev = nullptr;      // [c]
    int32_t* cterm_dev = nullptr;    // [c] bias - zp_a*wsum + 9*zp_a*zp_w + 0x4B400000
    float* mult_dev = nullptr;       // [c]
    int32_t* corr_dev = nullptr;     // [16][c] zero-padding corrections per border class
    float lo = 0.f, hi = 255.f;      // clamp bounds before + zp_c
    // CUDA-core FMA path (dwconv_fma.cu); null -> not exact for these params
    float* fma_w = nullptr;          // [c/4][9][4]: (w - zp_w) * 2^119
    float* fma_b = nullptr;          // [c]: (bias - zp_a * sum_t (w - zp_w)) * 2^-30
    float* fma_m = nullptr;          // [c]: mult * 2^30
    float* fma_corr = nullptr;       // [16][c]: corr * 2^-30 (zero-fill border classes)
};

namespace q8g {

// Tile kinds chosen by the dispatch cache (dispatch.hpp:248 TileKind analog)
// small: split-K clusters; mid: 128-column 1-CTA tiles; large: persistent
// CTA-pair 256 x 256 tiles (abi.cu tile_class)
enum TileKind : int { kGeneric = 0, kSmallM = 1, kLargeM = 2, kMidM = 3 };

struct ShapeKey {
    int m_class, n_class, k_class, align;
    bool operator==(const ShapeKey& o) const {
        return m_class == o.m_class && n_class == o.n_class && k_class == o.k_class &&
               align == o.align;
    }
};
struct ShapeKeyHash {
    size_t operator()(const ShapeKey& s) const {
        return ((size_t)s.m_class * 131 + s.n_class) * 131 * 131 + s.k_class * 131 + s.align;
    }
};

}  // namespace q8g

struct q8g_kernel_cache {
    bool generic_only = false;
    std::mutex mu;
    std::unordered_map<q8g::ShapeKey, int, q8g::ShapeKeyHash> table;
    uint64_t builds = 0;
};

namespace q8g {

// ---- kernels (launchers return cudaError_t of the launch) ----
cudaError_t launch_pack_b(const int8_t* b, int k, int n, int ldb, int8_t* packed, int kp, int np,
                          int32_t* colsum, int* max_abs, cudaStream_t s);
cudaError_t launch_unpack_b(const int8_t* packed, int k, int n, int kp, int np, int8_t* out,
                            int ldb, cudaStream_t s);

struct GemmArgs {
    const uint8_t* a;   // points at row 0 of the stripe
    int rows;           // rows in the stripe
    int k, lda;
    const q8g_packed_b* pb;
    const q8g_epilogue* ep;  // null for raw
    const int32_t* bias_add; // raw writer only, may be null
    void* c;            // points at row 0 of the stripe
    int ldc;
    bool raw;
    // host-view overlap (gemm_host): A arrives by a concurrent copy that ends
    // with a stream write of a_epoch to *a_ready.  The split-K kernel streams
    // B first and polls the flag before its first A load; every other path
    // makes the stream wait on the flag before launching.  null = A resident.
    const uint32_t* a_ready = nullptr;
    uint32_t a_epoch = 0;
    // N-sharded multi-GPU (q8g_gemm_u8s8_requant_peers): the same stripe is
    // also written at each of these pointers (peer devices' C windows, UVA,
    // same ldc).  A kernel that stores to them itself sets *peers_written;
    // otherwise the ABI copies dest 0 to them after the launch.
    uint8_t* const* c_peers = nullptr;
    int n_peers = 0;
    bool* peers_written = nullptr;
};
constexpr int kMaxPeers = 7;  // peer destinations of one call (8 GPUs of a node)
// stream memory operations (driver API via cudaGetDriverEntryPoint)
cudaError_t stream_write_u32(cudaStream_t s, uint32_t* addr, uint32_t value);
cudaError_t stream_wait_u32(cudaStream_t s, const uint32_t* addr, uint32_t value);  // until *addr == value
cudaError_t launch_gemm_simt(const GemmArgs& g, cudaStream_t s);
cudaError_t launch_gemm_tc(const GemmArgs& g, int tile_kind, cudaStream_t s);
bool tc_supported(const GemmArgs& g);
bool splitk_supported(const GemmArgs& g);
cudaError_t launch_gemm_splitk(const GemmArgs& g, cudaStream_t s);
cudaError_t launch_post(int writer, const int32_t* acc, int ldacc, const uint8_t* a, int lda, int rows, int k, int n,
                        const q8g_sparse_csc* sp, const q8g_epilogue* ep, double dq_scale, int32_t dq_zp, void* out,
                        int ldc, cudaStream_t s);
bool tc2w_supported(const GemmArgs& g);
int tc2w_last_clock(unsigned long long* cycles, unsigned long long* ns);
cudaError_t launch_gemm_tc2w(const GemmArgs& g, cudaStream_t s);
int tc_trace_copy(unsigned long long* out, int max_ctas);

struct ConvArgs {
    const uint8_t* x;  // first image of the shard
    int nb, h, w, c;
    int32_t zp_a;
    const q8g_packed_b* pw;
    const q8g_epilogue* ep;  // null for raw
    void* y;
    bool raw;
};
cudaError_t launch_conv3x3(const ConvArgs& a, cudaStream_t s);
// im2col + tensor-core GEMM; cudaErrorNotSupported -> use the CUDA-core conv
cudaError_t launch_conv3x3_im2col(const ConvArgs& a, cudaStream_t s);
// the process dispatch cache's tile kind for a GEMM shape (abi.cu)
int default_tile_kind(int rows, int n, int k, bool aligned);
bool conv_tc_supported(const ConvArgs& a);
cudaError_t launch_conv3x3_tc(const ConvArgs& a, cudaStream_t s);
// build the conv operand image of `pw` for C input channels (no-op when the
// implicit-GEMM kernel does not serve that C or the image exists)
cudaError_t conv_tc_prepare(const q8g_packed_b* pw, int c, cudaStream_t s);

cudaError_t launch_dwconv3x3(const uint8_t* x, int nb, int h, int w, int c,
                             const q8g_dw_filter* f, uint8_t* y, cudaStream_t s);
bool dw_tc_supported(int h, int w, int c, int32_t zp_a);
bool dw_fma_supported(int h, int w, int c);
bool dw_tc64_supported(int w, int c);
cudaError_t launch_dwconv3x3_fma(const uint8_t* x, int nb, int h, int w, int c, const q8g_dw_filter* f,
                                 uint8_t* y, cudaStream_t s);
cudaError_t launch_dwconv3x3_tc(const uint8_t* x, int nb, int h, int w, int c, const q8g_dw_filter* f,
                                uint8_t* y, cudaStream_t s);

int sm_count(int device);
// Dynamic work claiming for persistent kernels (conv3x3_tc): a per-device
// ring of kWorkSlots zeroed slots of kWorkSlotInts ints: kWorkGroups claim
// counters, one per 32-byte sector (a CTA claims from counter blockIdx %
// kWorkGroups, so the atomics of one launch spread over kWorkGroups L2
// sectors), and a done counter at kWorkDone.  Each launch takes the next slot;
// the last CTA to finish (done reaching gridDim) zeroes the slot for its next
// use kWorkSlots launches later (or the same captured graph node's next
// replay, which is stream-ordered after this one).  work_slot_prepare
// allocates the ring (not allowed under stream capture); work_slot returns
// nullptr when it is not allocated, and the kernel then falls back to its
// static schedule.
constexpr int kWorkSlots = 1024;
constexpr int kWorkGroups = 8;
constexpr int kWorkDone = 8 * kWorkGroups;
constexpr int kWorkSlotInts = 8 * kWorkGroups + 8;
cudaError_t work_slot_prepare(int device);
int* work_slot(int device);
// programmatic dependent launch for the tensor-core kernels (env Q8G_PDL=0
// disables): the kernels trigger their dependents at entry and run their
// global-memory-free prologue before griddepcontrol.wait
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_with_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace q8g
