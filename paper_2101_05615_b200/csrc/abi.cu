// abi.cu — the extern "C" boundary (include/q8g_b200.h).
//
// Validation mirrors the reference's std::invalid_argument conditions
// (engine.hpp:63-84, pack.hpp:24-37, pipeline.hpp:66-102, dispatch.hpp:17-30)
// and maps them to Q8G_EINVAL with the same message text.  No exception
// crosses this file's functions.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <set>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "q8g_internal.cuh"

namespace q8g {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_family[kFamCount];
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return Q8G_ECUDA;
}
void count_launch(int family) {
    if (family != kFamPeerCopy) g_launches.fetch_add(1, std::memory_order_relaxed);
    if (family >= 0 && family < kFamCount) g_family[family].fetch_add(1, std::memory_order_relaxed);
}

int sm_count(int device) {
    static int cache[64] = {0};
    if (device >= 0 && device < 64 && cache[device]) return cache[device];
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    if (device >= 0 && device < 64) cache[device] = v;
    return v;
}

namespace {
struct WorkRing {
    int* base = nullptr;
    std::atomic<unsigned> next{0};
};
WorkRing g_work_ring[64];
std::mutex g_work_mu;
}  // namespace

cudaError_t work_slot_prepare(int device) {
    if (device < 0 || device >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(g_work_mu);
    if (__atomic_load_n(&g_work_ring[device].base, __ATOMIC_ACQUIRE)) return cudaSuccess;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    int* p = nullptr;
    cudaError_t e = cudaMalloc(&p, sizeof(int) * kWorkSlotInts * kWorkSlots);
    if (e == cudaSuccess && (e = cudaMemset(p, 0, sizeof(int) * kWorkSlotInts * kWorkSlots)) == cudaSuccess)
        e = cudaDeviceSynchronize();
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
        if (p) cudaFree(p);
        return e;
    }
    __atomic_store_n(&g_work_ring[device].base, p, __ATOMIC_RELEASE);
    return cudaSuccess;
}

int* work_slot(int device) {
    if (device < 0 || device >= 64) return nullptr;
    int* b = __atomic_load_n(&g_work_ring[device].base, __ATOMIC_ACQUIRE);
    if (!b) return nullptr;
    return b + kWorkSlotInts * (g_work_ring[device].next.fetch_add(1, std::memory_order_relaxed) % kWorkSlots);
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("Q8G_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

static int validate_blocking(const q8g_blocking& bp) {
    if (bp.mcb < 1 || bp.ncb < 1 || bp.kcb < 1 || bp.mr < 1 || bp.nr < 1)
        return fail(Q8G_EINVAL, "BlockingParams: all sizes must be >= 1");
    if (bp.mcb % bp.mr != 0) return fail(Q8G_EINVAL, "BlockingParams: mcb must be a multiple of mr");
    if (bp.ncb % bp.nr != 0) return fail(Q8G_EINVAL, "BlockingParams: ncb must be a multiple of nr");
    if (bp.kcb % 2 != 0)
        return fail(Q8G_EINVAL, "BlockingParams: kcb must be even (k is consumed in pairs)");
    return Q8G_OK;
}

static q8g_kernel_cache& process_cache() {
    static q8g_kernel_cache* c = new q8g_kernel_cache();
    return *c;
}

// Shape class -> tile kind, memoized (dispatch.hpp:60-75 classify_shape,
// 117-140 build).  `aligned` = TMA can address A (16B-aligned base, lda%16==0).
// Tensor-core tile class by how many CTAs each kernel would fill on B200's
// 148 SMs (from per-launch sweeps over M, N, K, tools/tc_sweep.py):
//   0 split-K (BN 128, 4 ranks): up to two waves of its CTAs
//   2 CTA-pair 256 x 256 tiles: at least one tile per pair of SMs
//   1 otherwise: 128-column 1-CTA tiles (clusters of 2 sharing A rows)
constexpr int kDispatchSms = 148;
static int tile_class(int rows, int n) {
    const long long mt = (rows + 127) / 128, nt = (n + 127) / 128;
    if (mt * nt * 4 <= 2LL * kDispatchSms) return 0;
    if ((long long)((rows + 255) / 256) * ((n + 255) / 256) >= kDispatchSms / 2) return 2;
    return 1;
}

static int resolve_tile(q8g_kernel_cache* kc, int rows, int n, int k, bool aligned) {
    ShapeKey key;
    key.m_class = tile_class(rows, n);
    key.n_class = n <= 32 ? 0 : 1;
    key.k_class = k % 16 == 0 ? 0 : 1;
    key.align = aligned ? 1 : 0;
    std::lock_guard<std::mutex> lock(kc->mu);
    auto it = kc->table.find(key);
    if (it != kc->table.end()) return it->second;
    ++kc->builds;
    int kind = kGeneric;
    if (!kc->generic_only && key.align && key.k_class == 0)
        kind = key.m_class == 0 ? kSmallM : key.m_class == 1 ? kMidM : kLargeM;
    kc->table.emplace(key, kind);
    return kind;
}

int default_tile_kind(int rows, int n, int k, bool aligned) {
    return resolve_tile(&process_cache(), rows, n, k, aligned);
}

static bool a_is_tma_aligned(const void* a, int lda) {
    return ((uintptr_t)a % 16 == 0) && (lda % 16 == 0);
}

}  // namespace q8g

using namespace q8g;

extern "C" {

const char* q8g_last_error(void) { return g_last_error.c_str(); }
int q8g_version(void) { return 1; }
uint64_t q8g_launch_count(void) { return g_launches.load(); }

int q8g_debug_kernel_clock(uint64_t* cycles, uint64_t* ns) {
    if (!cycles || !ns) return fail(Q8G_EINVAL, "null argument");
    unsigned long long c = 0, t = 0;
    if (tc2w_last_clock(&c, &t)) return fail(Q8G_ECUDA, "kernel clock readback failed");
    *cycles = c;
    *ns = t;
    return Q8G_OK;
}

int q8g_debug_tc_trace(uint64_t* out, int max_ctas) {
    if (!out || max_ctas < 1) return 0;
    return tc_trace_copy(reinterpret_cast<unsigned long long*>(out), max_ctas);
}

int q8g_launch_stats(uint64_t* counts, int n) {
    if (!counts || n < 1) return fail(Q8G_EINVAL, "launch_stats: bad arguments");
    for (int i = 0; i < n; ++i) counts[i] = i < kFamCount ? g_family[i].load() : 0;
    return Q8G_OK;
}

int q8g_blocking_defaults(q8g_blocking* out) {
    if (!out) return fail(Q8G_EINVAL, "null output");
    *out = q8g_blocking{56, 32, 256, 14, 32};  // pack.hpp:16-20
    return Q8G_OK;
}

int q8g_blocking_validate(const q8g_blocking* bp) {
    if (!bp) return fail(Q8G_EINVAL, "null blocking");
    return validate_blocking(*bp);
}

int q8g_select_blocking(int m, int n, int k, const q8g_blocking* defaults, q8g_blocking* out) {
    if (!defaults || !out) return fail(Q8G_EINVAL, "null blocking");
    int rc = validate_blocking(*defaults);
    if (rc) return rc;
    if (m < 1 || n < 1 || k < 1) return fail(Q8G_EINVAL, "select_blocking: dimensions must be >= 1");
    q8g_blocking bp = *defaults;
    bp.mr = std::min(defaults->mr, m);
    bp.nr = std::min(defaults->nr, n);
    bp.mcb = std::min(defaults->mcb, round_up_i(m, bp.mr));
    bp.ncb = std::min(defaults->ncb, round_up_i(n, bp.nr));
    bp.kcb = std::min(defaults->kcb, round_up_i(k, 2));
    rc = validate_blocking(bp);
    if (rc) return rc;
    *out = bp;
    return Q8G_OK;
}

int q8g_partition_stripes(int num_blocks, int thread_id, int num_threads, int* begin, int* end) {
    if (num_threads < 1 || thread_id < 0 || thread_id >= num_threads)
        return fail(Q8G_EINVAL, "execute_gemm: thread_id must be in [0, num_threads)");
    if (num_blocks < 0 || !begin || !end) return fail(Q8G_EINVAL, "partition_stripes: bad arguments");
    const int base = num_blocks / num_threads, rem = num_blocks % num_threads;
    *begin = thread_id * base + std::min(thread_id, rem);
    *end = *begin + base + (thread_id < rem ? 1 : 0);
    return Q8G_OK;
}

// ---------------------------------------------------------------- pack

static int pack_common(const int8_t* b, bool b_on_device, int k, int n, int ldb,
                       const q8g_blocking* bp, int device, cudaStream_t s, q8g_packed_b** out) {
    if (!out) return fail(Q8G_EINVAL, "null output handle");
    *out = nullptr;
    q8g_blocking blk;
    q8g_blocking_defaults(&blk);
    if (bp) blk = *bp;
    int rc = validate_blocking(blk);
    if (rc) return rc;
    if (k < 1 || n < 1) return fail(Q8G_EINVAL, "prepack_weights: matrix must be non-empty");
    if (!b || ldb < n) return fail(Q8G_EINVAL, "prepack_weights: bad B pointer or ldb < N");
    DeviceGuard dg(device);
    auto* pb = new (std::nothrow) q8g_packed_b();
    if (!pb) return fail(Q8G_ENOMEM, "out of host memory");
    pb->device = device;
    pb->k = k;
    pb->n = n;
    pb->kp = round_up_i(k, kKBlock);
    pb->np = round_up_i(n, kNPad);
    pb->blocking = blk;
    int* d_max = nullptr;
    const int8_t* d_b = b;
    int8_t* staged = nullptr;
    auto cleanup = [&](int code) {
        if (staged) cudaFree(staged);
        if (d_max) cudaFree(d_max);
        if (code != Q8G_OK) q8g_free_packed_b(pb);
        return code;
    };
    cudaError_t e;
    if ((e = cudaMalloc(&pb->data, (size_t)pb->kp * pb->np)) != cudaSuccess)
        return cleanup(cuda_fail(e, "cudaMalloc(packed B)"));
    if ((e = cudaMalloc(&pb->colsum_dev, sizeof(int32_t) * pb->np)) != cudaSuccess)
        return cleanup(cuda_fail(e, "cudaMalloc(colsum)"));
    if ((e = cudaMalloc(&d_max, sizeof(int))) != cudaSuccess)
        return cleanup(cuda_fail(e, "cudaMalloc(max_abs)"));
    if (!b_on_device) {
        if ((e = cudaMalloc(&staged, (size_t)k * ldb)) != cudaSuccess)
            return cleanup(cuda_fail(e, "cudaMalloc(staged B)"));
        if ((e = cudaMemcpyAsync(staged, b, (size_t)(k - 1) * ldb + n, cudaMemcpyHostToDevice, s)) !=
            cudaSuccess)
            return cleanup(cuda_fail(e, "cudaMemcpyAsync(B)"));
        d_b = staged;
    }
    if ((e = launch_pack_b(d_b, k, n, ldb, pb->data, pb->kp, pb->np, pb->colsum_dev, d_max, s)) !=
        cudaSuccess)
        return cleanup(cuda_fail(e, "pack_b kernel"));
    pb->colsum_host = (int32_t*)malloc(sizeof(int32_t) * pb->np);
    if ((e = cudaMemcpyAsync(pb->colsum_host, pb->colsum_dev, sizeof(int32_t) * pb->np,
                             cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cleanup(cuda_fail(e, "cudaMemcpyAsync(colsum)"));
    if ((e = cudaMemcpyAsync(&pb->max_abs, d_max, sizeof(int), cudaMemcpyDeviceToHost, s)) !=
        cudaSuccess)
        return cleanup(cuda_fail(e, "cudaMemcpyAsync(max_abs)"));
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess)
        return cleanup(cuda_fail(e, "pack_b synchronize"));
    *out = pb;
    return cleanup(Q8G_OK);
}

int q8g_pack_b(const int8_t* b_host, int k, int n, int ldb, const q8g_blocking* bp, int device,
               q8g_packed_b** out) {
    return pack_common(b_host, false, k, n, ldb, bp, device, nullptr, out);
}

int q8g_pack_b_device(const int8_t* b_dev, int k, int n, int ldb, const q8g_blocking* bp,
                      int device, void* stream, q8g_packed_b** out) {
    return pack_common(b_dev, true, k, n, ldb, bp, device, (cudaStream_t)stream, out);
}

int q8g_packed_b_replicate(const q8g_packed_b* src, int device, q8g_packed_b** out) {
    if (!src || !out) return fail(Q8G_EINVAL, "null handle");
    DeviceGuard dg(device);
    auto* pb = new (std::nothrow) q8g_packed_b(*src);
    if (!pb) return fail(Q8G_ENOMEM, "out of host memory");
    pb->device = device;
    pb->data = nullptr;
    pb->colsum_dev = nullptr;
    for (int i = 0; i < 3; ++i) {  // rebuilt on the replica's device
        pb->conv_img[i] = nullptr;
        pb->conv_img_ready[i] = 0;
    }
    pb->colsum_host = (int32_t*)malloc(sizeof(int32_t) * src->np);
    memcpy(pb->colsum_host, src->colsum_host, sizeof(int32_t) * src->np);
    cudaError_t e;
    if ((e = cudaMalloc(&pb->data, (size_t)pb->kp * pb->np)) != cudaSuccess ||
        (e = cudaMalloc(&pb->colsum_dev, sizeof(int32_t) * pb->np)) != cudaSuccess) {
        q8g_free_packed_b(pb);
        return cuda_fail(e, "cudaMalloc(replica)");
    }
    if ((e = cudaMemcpyPeer(pb->data, device, src->data, src->device, (size_t)pb->kp * pb->np)) !=
            cudaSuccess ||
        (e = cudaMemcpy(pb->colsum_dev, pb->colsum_host, sizeof(int32_t) * pb->np,
                        cudaMemcpyHostToDevice)) != cudaSuccess) {
        q8g_free_packed_b(pb);
        return cuda_fail(e, "replicate copy");
    }
    // packed weights are complete before any kernel can read them (the GEMM
    // kernels prefetch B ahead of griddepcontrol.wait, gemm_splitk.cu)
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) {
        q8g_free_packed_b(pb);
        return cuda_fail(e, "replicate copy");
    }
    *out = pb;
    return Q8G_OK;
}

int q8g_packed_b_info(const q8g_packed_b* pb, int* k, int* n, int* max_abs, int* device) {
    if (!pb) return fail(Q8G_EINVAL, "null handle");
    if (k) *k = pb->k;
    if (n) *n = pb->n;
    if (max_abs) *max_abs = pb->max_abs;
    if (device) *device = pb->device;
    return Q8G_OK;
}

int q8g_packed_b_blocking(const q8g_packed_b* pb, q8g_blocking* out) {
    if (!pb || !out) return fail(Q8G_EINVAL, "null handle");
    *out = pb->blocking;
    return Q8G_OK;
}

int q8g_packed_b_col_offsets(const q8g_packed_b* pb, int32_t* out_host) {
    if (!pb || !out_host) return fail(Q8G_EINVAL, "null handle");
    memcpy(out_host, pb->colsum_host, sizeof(int32_t) * pb->n);
    return Q8G_OK;
}

int q8g_unpack_b(const q8g_packed_b* pb, int8_t* out_host, int ldb) {
    if (!pb || !out_host || ldb < pb->n) return fail(Q8G_EINVAL, "unpack_weight: bad arguments");
    DeviceGuard dg(pb->device);
    int8_t* d = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&d, (size_t)pb->k * ldb)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    e = launch_unpack_b(pb->data, pb->k, pb->n, pb->kp, pb->np, d, ldb, nullptr);
    if (e == cudaSuccess)
        e = cudaMemcpy(out_host, d, (size_t)(pb->k - 1) * ldb + pb->n, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "unpack_b");
    return Q8G_OK;
}

int q8g_free_packed_b(q8g_packed_b* pb) {
    if (!pb) return Q8G_OK;
    DeviceGuard dg(pb->device);
    if (pb->data) cudaFree(pb->data);
    if (pb->colsum_dev) cudaFree(pb->colsum_dev);
    for (int i = 0; i < 3; ++i)
        if (pb->conv_img[i]) cudaFree(pb->conv_img[i]);
    free(pb->colsum_host);
    delete pb;
    return Q8G_OK;
}

// ---------------------------------------------------------------- epilogue

static int build_records(int n, int np, int32_t k_total, const q8g_requant_params* p,
                         const int32_t* colsum, const int32_t* bias_add, std::vector<EpiRecord>& rec,
                         bool& need_rowsum) {
    if (p->rounding != Q8G_ROUND_REF && p->rounding != Q8G_ROUND_F32_RNE)
        return fail(Q8G_EINVAL, "Requantize: unknown rounding mode");
    if (!(p->multiplier > 0) && !p->multiplier_f32_per_channel_host &&
        !p->multiplier_per_channel_host)
        return fail(Q8G_EINVAL, "OutputPipeline: Requantize multiplier must be positive");
    if (k_total < 1) return fail(Q8G_EINVAL, "OutputPipeline: Requantize k_total must be >= 1");
    if (p->zp_c > (1 << 30) || p->zp_c < -(1 << 30))
        return fail(Q8G_EINVAL, "Requantize: |zp_c| must be <= 2^30");
    rec.assign(np, EpiRecord{});
    need_rowsum = false;
    for (int j = 0; j < n; ++j) {
        const int64_t zpb = p->zp_b_per_channel_host ? p->zp_b_per_channel_host[j] : p->zp_b;
        const int64_t bias = (p->bias_host ? p->bias_host[j] : 0) + (bias_add ? bias_add[j] : 0);
        const int64_t c = bias - (int64_t)p->zp_a * colsum[j] + (int64_t)k_total * p->zp_a * zpb;
        rec[j].c = (int32_t)(uint32_t)(uint64_t)c;  // wraps mod 2^32 (see requant.cuh)
        rec[j].zpb = (int32_t)zpb;
        if (zpb != 0) need_rowsum = true;
        if (p->rounding == Q8G_ROUND_F32_RNE) {
            const float mf = p->multiplier_f32_per_channel_host
                                 ? p->multiplier_f32_per_channel_host[j]
                                 : (float)p->multiplier;
            if (!(mf > 0)) return fail(Q8G_EINVAL, "OutputPipeline: Requantize multiplier must be positive");
            rec[j].md = 0.0;
            rec[j].mf = mf;
        } else {
            const double md =
                p->multiplier_per_channel_host ? p->multiplier_per_channel_host[j] : p->multiplier;
            if (!(md > 0)) return fail(Q8G_EINVAL, "OutputPipeline: Requantize multiplier must be positive");
            rec[j].md = md;
        }
    }
    return Q8G_OK;
}

int q8g_epilogue_create(const q8g_packed_b* pb, const q8g_requant_params* p,
                        const int32_t* bias_add_host, q8g_epilogue** out) {
    if (!pb || !p || !out) return fail(Q8G_EINVAL, "null argument");
    *out = nullptr;
    const int32_t* colsum = p->col_offsets_host ? p->col_offsets_host : pb->colsum_host;
    // Exactness of the int32 adjust (requant.cuh): the kernels compute
    // adj = acc - zp_b*rowsum + c (mod 2^32); it equals the reference's int64
    // requantize_adjust (quant.hpp:115-125) iff the true value fits int32.
    // With the weight's own column sums the true value is
    //   sum_k (A - zp_a)(B - zp_b) + (k_total - K) zp_a zp_b + bias
    // with A in [0, 255] and |B| <= max|B| (pack time); with caller-supplied
    // column sums every term is bounded separately.
    {
        const int64_t K = pb->k, za = p->zp_a;
        const int64_t amax = std::max<int64_t>(za < 0 ? -za : za, 255 - za < 0 ? za - 255 : 255 - za);
        for (int j = 0; j < pb->n; ++j) {
            const int64_t zb = p->zp_b_per_channel_host ? p->zp_b_per_channel_host[j] : p->zp_b;
            const int64_t azb = zb < 0 ? -zb : zb;
            int64_t bias = (p->bias_host ? p->bias_host[j] : 0) + (bias_add_host ? bias_add_host[j] : 0);
            bias = bias < 0 ? -bias : bias;
            const int64_t dk = (int64_t)p->k_total - K;
            int64_t bound;
            if (!p->col_offsets_host) {
                bound = K * amax * ((int64_t)pb->max_abs + azb) + (dk < 0 ? -dk : dk) * (za < 0 ? -za : za) * azb + bias;
            } else {
                const int64_t cs = colsum[j] < 0 ? -(int64_t)colsum[j] : (int64_t)colsum[j];
                const int64_t kt = p->k_total < 0 ? -(int64_t)p->k_total : (int64_t)p->k_total;
                bound = K * 255 * (int64_t)pb->max_abs + azb * 255 * K + (za < 0 ? -za : za) * cs +
                        kt * (za < 0 ? -za : za) * azb + bias;
            }
            if (bound >= (int64_t(1) << 31))
                return fail(Q8G_EINVAL, "Requantize: the zero-point-adjusted accumulator of column " +
                                            std::to_string(j) + " can reach " + std::to_string(bound) +
                                            " >= 2^31 (K, |A - zp_a|, |B - zp_b| or |bias| too large for the "
                                            "exact int32 epilogue)");
        }
    }
    std::vector<EpiRecord> rec;
    bool need_rowsum = false;
    int rc = build_records(pb->n, pb->np, p->k_total, p, colsum, bias_add_host, rec, need_rowsum);
    if (rc) return rc;
    DeviceGuard dg(pb->device);
    auto* ep = new (std::nothrow) q8g_epilogue();
    if (!ep) return fail(Q8G_ENOMEM, "out of host memory");
    ep->device = pb->device;
    ep->n = pb->n;
    ep->np = pb->np;
    ep->k_total = p->k_total;
    ep->zp_a = p->zp_a;
    ep->zp_c = p->zp_c;
    ep->rounding = p->rounding;
    ep->relu = p->relu ? 1 : 0;
    ep->need_rowsum = need_rowsum;
    ep->fast_f32 = p->rounding == Q8G_ROUND_F32_RNE && p->zp_c >= 0 && p->zp_c <= 255;
    for (int j = 0; j < pb->n && ep->fast_f32; ++j)
        if (!(rec[j].mf < 7.9228163e28f)) ep->fast_f32 = false;  // 2^96; also rejects inf
    cudaError_t e;
    if ((e = cudaMalloc(&ep->rec, sizeof(EpiRecord) * pb->np)) != cudaSuccess ||
        (e = cudaMemcpy(ep->rec, rec.data(), sizeof(EpiRecord) * pb->np, cudaMemcpyHostToDevice)) !=
            cudaSuccess) {
        q8g_epilogue_free(ep);
        return cuda_fail(e, "epilogue table");
    }
    *out = ep;
    return Q8G_OK;
}

int q8g_epilogue_free(q8g_epilogue* ep) {
    if (!ep) return Q8G_OK;
    DeviceGuard dg(ep->device);
    if (ep->rec) cudaFree(ep->rec);
    delete ep;
    return Q8G_OK;
}

// ---------------------------------------------------------------- dispatch cache

int q8g_kernel_cache_create(int generic_only, q8g_kernel_cache** out) {
    if (!out) return fail(Q8G_EINVAL, "null output");
    *out = new (std::nothrow) q8g_kernel_cache();
    if (!*out) return fail(Q8G_ENOMEM, "out of host memory");
    (*out)->generic_only = generic_only != 0;
    return Q8G_OK;
}

int q8g_kernel_cache_free(q8g_kernel_cache* kc) {
    if (kc && kc != &process_cache()) delete kc;
    return Q8G_OK;
}

uint64_t q8g_kernel_cache_build_count(const q8g_kernel_cache* kc) {
    auto* c = const_cast<q8g_kernel_cache*>(kc ? kc : &process_cache());
    std::lock_guard<std::mutex> lock(c->mu);
    return c->builds;
}

int q8g_kernel_cache_tile(q8g_kernel_cache* kc, int m, int n, int k, int lda, int* tile_kind) {
    if (!tile_kind) return fail(Q8G_EINVAL, "null output");
    *tile_kind = resolve_tile(kc ? kc : &process_cache(), m, n, k, lda % 16 == 0);
    return Q8G_OK;
}

// ---------------------------------------------------------------- GEMM

static int gemm_common(const uint8_t* a, int m, int k, int lda, const q8g_packed_b* pb,
                       const q8g_epilogue* ep, const int32_t* bias_add, void* c, int ldc,
                       int row_begin, int row_end, q8g_kernel_cache* cache, cudaStream_t s,
                       bool raw, const uint32_t* a_ready = nullptr, uint32_t a_epoch = 0,
                       uint8_t* const* c_peers = nullptr, int n_peers = 0, bool peers_direct = true) {
    if (!pb) return fail(Q8G_EINVAL, "execute_gemm: null packed weight");
    if (k != pb->k) return fail(Q8G_EINVAL, "execute_gemm: A columns must equal the packed weight K");
    if (m < 1 || lda < k || ldc < pb->n || !a || !c)
        return fail(Q8G_EINVAL, "execute_gemm: output must be M x N");
    if (row_begin < 0 || row_end > m || row_begin > row_end)
        return fail(Q8G_EINVAL, "execute_gemm: row stripe out of range");
    if (!raw) {
        if (!ep) return fail(Q8G_EINVAL, "pipeline writer does not match the output element type");
        if (ep->n != pb->n || ep->device != pb->device)
            return fail(Q8G_EINVAL, "execute_gemm: epilogue was built for another packed weight");
    }
    if (row_begin == row_end) return Q8G_OK;
    DeviceGuard dg(pb->device);
    GemmArgs g;
    g.rows = row_end - row_begin;
    g.k = k;
    g.lda = lda;
    g.a = a + (size_t)row_begin * lda;
    g.pb = pb;
    g.ep = ep;
    g.bias_add = bias_add;
    g.raw = raw;
    g.ldc = ldc;
    g.c = raw ? (void*)((int32_t*)c + (size_t)row_begin * ldc)
              : (void*)((uint8_t*)c + (size_t)row_begin * ldc);
    g.a_ready = a_ready;
    g.a_epoch = a_epoch;
    uint8_t* peers[kMaxPeers];
    bool peers_written = false;
    for (int d = 0; d < n_peers; ++d) peers[d] = c_peers[d] + (size_t)row_begin * ldc;
    g.c_peers = peers_direct ? peers : nullptr;  // kernels store to the peers only over P2P
    g.n_peers = peers_direct ? n_peers : 0;
    g.peers_written = &peers_written;
    const int kind = resolve_tile(cache ? cache : &process_cache(), g.rows, pb->n, k,
                                  a_is_tma_aligned(g.a, lda));
    cudaError_t e;
    if (kind != kGeneric && tc_supported(g)) {
        e = launch_gemm_tc(g, kind, s);
    } else {
        e = a_ready ? stream_wait_u32(s, a_ready, a_epoch) : cudaSuccess;
        if (e == cudaSuccess) e = launch_gemm_simt(g, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "gemm launch");
    // kernels without peer stores (small M, non-fast epilogues): the stripe
    // goes from the local C to each peer by the copy engines, stream-ordered
    for (int d = 0; d < n_peers && !peers_written; ++d) {
        e = cudaMemcpy2DAsync(peers[d], (size_t)ldc, g.c, (size_t)ldc, (size_t)pb->n, (size_t)g.rows,
                              cudaMemcpyDefault, s);  // UVA: also across devices without peer access
        if (e != cudaSuccess) return cuda_fail(e, "peer copy");
        count_launch(kFamPeerCopy);
    }
    return Q8G_OK;
}

// peer access from `dev` to the device holding `ptr` (once per pair);
// Q8G_OK also when ptr is on `dev` itself.  *direct = false when the devices
// have no P2P path: the stripe then reaches that peer by a staged copy.
static int enable_peer_access(int dev, const void* ptr, bool* direct) {
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, ptr);
    if (e != cudaSuccess) return cuda_fail(e, "gemm_peers: cudaPointerGetAttributes");
    if (at.type != cudaMemoryTypeDevice) return fail(Q8G_EINVAL, "gemm_peers: peer output must be device memory");
    if (at.device == dev) return Q8G_OK;
    static std::mutex mu;
    static std::set<std::pair<int, int>> done, no_p2p;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({dev, at.device})) return Q8G_OK;
    if (no_p2p.count({dev, at.device})) {
        *direct = false;
        return Q8G_OK;
    }
    int can = 0;
    e = cudaDeviceCanAccessPeer(&can, dev, at.device);
    if (e != cudaSuccess) return cuda_fail(e, "gemm_peers: cudaDeviceCanAccessPeer");
    if (!can) {
        no_p2p.insert({dev, at.device});
        *direct = false;
        return Q8G_OK;
    }
    DeviceGuard dg(dev);
    e = cudaDeviceEnablePeerAccess(at.device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        e = cudaSuccess;
    }
    if (e != cudaSuccess) return cuda_fail(e, "gemm_peers: cudaDeviceEnablePeerAccess");
    done.insert({dev, at.device});
    return Q8G_OK;
}

int q8g_gemm_u8s8_requant(const uint8_t* a_dev, int m, int k, int lda, const q8g_packed_b* pb,
                          const q8g_epilogue* ep, uint8_t* c_dev, int ldc, int row_begin,
                          int row_end, q8g_kernel_cache* cache, void* stream) {
    return gemm_common(a_dev, m, k, lda, pb, ep, nullptr, c_dev, ldc, row_begin, row_end, cache,
                       (cudaStream_t)stream, false);
}

int q8g_gemm_u8s8_requant_peers(const uint8_t* a_dev, int m, int k, int lda, const q8g_packed_b* pb,
                                const q8g_epilogue* ep, uint8_t* c_dev, uint8_t* const* c_peer_dev,
                                int n_peers, int ldc, int row_begin, int row_end, q8g_kernel_cache* cache,
                                void* stream) {
    if (n_peers < 0 || n_peers > kMaxPeers) return fail(Q8G_EINVAL, "gemm_peers: 0 to 7 peer outputs");
    if (n_peers > 0 && !c_peer_dev) return fail(Q8G_EINVAL, "gemm_peers: null peer output list");
    bool direct = true;
    for (int d = 0; d < n_peers; ++d) {
        if (!c_peer_dev[d]) return fail(Q8G_EINVAL, "gemm_peers: null peer output");
        if (pb) {
            const int st = enable_peer_access(pb->device, c_peer_dev[d], &direct);
            if (st != Q8G_OK) return st;
        }
    }
    return gemm_common(a_dev, m, k, lda, pb, ep, nullptr, c_dev, ldc, row_begin, row_end, cache,
                       (cudaStream_t)stream, false, nullptr, 0, c_peer_dev, n_peers, direct);
}

int q8g_gemm_u8s8_raw_i32(const uint8_t* a_dev, int m, int k, int lda, const q8g_packed_b* pb,
                          const int32_t* bias_add_dev, int32_t* c_dev, int ldc, int row_begin,
                          int row_end, q8g_kernel_cache* cache, void* stream) {
    return gemm_common(a_dev, m, k, lda, pb, nullptr, bias_add_dev, c_dev, ldc, row_begin,
                       row_end, cache, (cudaStream_t)stream, true);
}

// ---------------------------------------------------------------- outliers + general pipeline

int q8g_split_outliers(const int8_t* b, int k, int n, int ldb, int threshold, int8_t* dense, int ldd,
                       int32_t* col_ptr, int32_t* row_idx, int8_t* values, int cap, int* nnz_out) {
    if (threshold < 1) return fail(Q8G_EINVAL, "split_outliers: threshold must be >= 1");
    if (k < 1 || n < 1) return fail(Q8G_EINVAL, "split_outliers: matrix must be non-empty");
    if (!b || !nnz_out || ldb < n || (dense && ldd < n) || (cap > 0 && (!col_ptr || !row_idx || !values)))
        return fail(Q8G_EINVAL, "split_outliers: bad arguments");
    // sparse.hpp:46-56: column-major walk builds the CSC arrays directly
    int nnz = 0;
    if (col_ptr && cap > 0) col_ptr[0] = 0;
    for (int j = 0; j < n; ++j) {
        for (int kk = 0; kk < k; ++kk) {
            const int8_t v = b[(size_t)kk * ldb + j];
            const bool outlier = (v < 0 ? -(int)v : (int)v) >= threshold;
            if (dense) dense[(size_t)kk * ldd + j] = outlier ? 0 : v;
            if (outlier) {
                if (nnz < cap) {
                    row_idx[nnz] = kk;
                    values[nnz] = v;
                }
                ++nnz;
            }
        }
        if (col_ptr && cap > 0) col_ptr[j + 1] = nnz;
    }
    *nnz_out = nnz;
    if (cap > 0 && nnz > cap) return fail(Q8G_EINVAL, "split_outliers: more outliers than the CSC capacity");
    return Q8G_OK;
}

int q8g_sparse_csc_create(const int32_t* col_ptr, const int32_t* row_idx, const int8_t* values, int nnz, int k,
                          int n, int device, q8g_sparse_csc** out) {
    if (!out || !col_ptr || k < 1 || n < 1 || nnz < 0 || (nnz > 0 && (!row_idx || !values)))
        return fail(Q8G_EINVAL, "SparseWeightCSC: bad arguments");
    *out = nullptr;
    if (col_ptr[0] != 0 || col_ptr[n] != nnz) return fail(Q8G_EINVAL, "SparseWeightCSC: col_ptr must run 0..nnz");
    for (int j = 0; j < n; ++j) {
        if (col_ptr[j + 1] < col_ptr[j]) return fail(Q8G_EINVAL, "SparseWeightCSC: col_ptr must be nondecreasing");
        for (int32_t i = col_ptr[j]; i < col_ptr[j + 1]; ++i) {
            if (row_idx[i] < 0 || row_idx[i] >= k) return fail(Q8G_EINVAL, "SparseWeightCSC: row index out of range");
            if (i > col_ptr[j] && row_idx[i] <= row_idx[i - 1])
                return fail(Q8G_EINVAL, "SparseWeightCSC: row indices must increase within a column");
        }
    }
    DeviceGuard dg(device);
    auto* sp = new (std::nothrow) q8g_sparse_csc();
    if (!sp) return fail(Q8G_ENOMEM, "out of host memory");
    sp->device = device;
    sp->k = k;
    sp->n = n;
    sp->nnz = nnz;
    cudaError_t e;
    if ((e = cudaMalloc(&sp->col_ptr, sizeof(int32_t) * (n + 1))) != cudaSuccess ||
        (e = cudaMalloc(&sp->row_idx, sizeof(int32_t) * (nnz > 0 ? nnz : 1))) != cudaSuccess ||
        (e = cudaMalloc(&sp->values, nnz > 0 ? nnz : 1)) != cudaSuccess ||
        (e = cudaMemcpy(sp->col_ptr, col_ptr, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (nnz > 0 && (e = cudaMemcpy(sp->row_idx, row_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice)) !=
                        cudaSuccess) ||
        (nnz > 0 && (e = cudaMemcpy(sp->values, values, nnz, cudaMemcpyHostToDevice)) != cudaSuccess)) {
        q8g_sparse_csc_free(sp);
        return cuda_fail(e, "SparseWeightCSC upload");
    }
    *out = sp;
    return Q8G_OK;
}

int q8g_sparse_csc_free(q8g_sparse_csc* sp) {
    if (!sp) return Q8G_OK;
    DeviceGuard dg(sp->device);
    if (sp->col_ptr) cudaFree(sp->col_ptr);
    if (sp->row_idx) cudaFree(sp->row_idx);
    if (sp->values) cudaFree(sp->values);
    delete sp;
    return Q8G_OK;
}

int q8g_gemm_u8s8_pipeline(const uint8_t* a_dev, int m, int k, int lda, const q8g_packed_b* pb,
                           const q8g_pipeline_args* pl, void* c_dev, int ldc, int row_begin, int row_end,
                           q8g_kernel_cache* cache, void* stream) {
    if (!pl || !pb) return fail(Q8G_EINVAL, "execute_gemm: null argument");
    const cudaStream_t s = (cudaStream_t)stream;
    const int w = pl->writer;
    if (w != Q8G_WRITE_RAW_I32 && w != Q8G_WRITE_REQUANT_U8 && w != Q8G_WRITE_DEQUANT_F32)
        return fail(Q8G_EINVAL, "pipeline writer does not match the output element type");
    if (pl->sparse) {
        if (pl->sparse->k != k || pl->sparse->n != pb->n)
            return fail(Q8G_EINVAL, "spmdm_block: block extents out of bounds (sparse " + std::to_string(pl->sparse->k) +
                                        " x " + std::to_string(pl->sparse->n) + ", GEMM K " + std::to_string(k) +
                                        ", N " + std::to_string(pb->n) + ")");
        if (pl->sparse->device != pb->device)
            return fail(Q8G_EINVAL, "SpMDMAdd: sparse matrix lives on another device");
    }
    if (w == Q8G_WRITE_REQUANT_U8 && pl->bias_add_dev)
        return fail(Q8G_EINVAL, "Requantize writer: BiasAdd is folded into the epilogue (q8g_epilogue_create)");
    // the hot paths when there is nothing to add
    if (!pl->sparse && w == Q8G_WRITE_RAW_I32)
        return gemm_common(a_dev, m, k, lda, pb, nullptr, pl->bias_add_dev, c_dev, ldc, row_begin, row_end, cache,
                           s, true);
    if (!pl->sparse && w == Q8G_WRITE_REQUANT_U8)
        return gemm_common(a_dev, m, k, lda, pb, pl->ep, nullptr, c_dev, ldc, row_begin, row_end, cache, s, false);
    if (w == Q8G_WRITE_REQUANT_U8) {
        if (!pl->ep) return fail(Q8G_EINVAL, "pipeline writer does not match the output element type");
        if (pl->ep->n != pb->n || pl->ep->device != pb->device)
            return fail(Q8G_EINVAL, "execute_gemm: epilogue was built for another packed weight");
    }
    if (!a_dev || !c_dev || m < 1 || lda < k || ldc < pb->n) return fail(Q8G_EINVAL, "execute_gemm: output must be M x N");
    if (row_begin < 0 || row_end > m || row_begin > row_end)
        return fail(Q8G_EINVAL, "execute_gemm: row stripe out of range");
    const int rows = row_end - row_begin;
    if (rows == 0) return Q8G_OK;
    DeviceGuard dg(pb->device);
    const uint8_t* a0 = a_dev + (size_t)row_begin * lda;
    cudaError_t e;
    if (w == Q8G_WRITE_RAW_I32) {
        // dense raw GEMM (+ BiasAdd) straight into the int32 output, outliers added in place
        int rc = gemm_common(a_dev, m, k, lda, pb, nullptr, pl->bias_add_dev, c_dev, ldc, row_begin, row_end, cache,
                             s, true);
        if (rc) return rc;
        int32_t* c0 = static_cast<int32_t*>(c_dev) + (size_t)row_begin * ldc;
        if ((e = launch_post(w, c0, ldc, a0, lda, rows, k, pb->n, pl->sparse, nullptr, 0.0, 0, c0, ldc, s)) !=
            cudaSuccess)
            return cuda_fail(e, "post launch");
        return Q8G_OK;
    }
    // requant / dequant: dense raw GEMM into a stream-ordered int32 workspace
    int32_t* ws = nullptr;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&ws), sizeof(int32_t) * (size_t)rows * pb->n, s)) !=
        cudaSuccess)
        return cuda_fail(e, "cudaMallocAsync(pipeline workspace)");
    int rc = gemm_common(a0, rows, k, lda, pb, nullptr, w == Q8G_WRITE_DEQUANT_F32 ? pl->bias_add_dev : nullptr, ws,
                         pb->n, 0, rows, cache, s, true);
    if (rc == Q8G_OK) {
        void* out0 = w == Q8G_WRITE_DEQUANT_F32 ? (void*)(static_cast<float*>(c_dev) + (size_t)row_begin * ldc)
                                               : (void*)(static_cast<uint8_t*>(c_dev) + (size_t)row_begin * ldc);
        if ((e = launch_post(w, ws, pb->n, a0, lda, rows, k, pb->n, pl->sparse,
                             w == Q8G_WRITE_REQUANT_U8 ? pl->ep : nullptr, pl->dq_scale, pl->dq_zero_point, out0, ldc,
                             s)) != cudaSuccess)
            rc = cuda_fail(e, "post launch");
    }
    cudaFreeAsync(ws, s);
    return rc;
}

int q8g_gemm_u8s8_pipeline_host(const uint8_t* a_host, int m, int k, int lda, const q8g_packed_b* pb,
                                const q8g_pipeline_args* pl, const int32_t* bias_add_host, void* c_host, int ldc,
                                int row_begin, int row_end, void* stream) {
    if (!pl || !pb || !a_host || !c_host) return fail(Q8G_EINVAL, "execute_gemm: null argument");
    if (pl->bias_add_dev) return fail(Q8G_EINVAL, "pipeline_host: pass BiasAdd as bias_add_host");
    if (k != pb->k) return fail(Q8G_EINVAL, "execute_gemm: A columns must equal the packed weight K");
    if (lda < k || ldc < pb->n || m < 1) return fail(Q8G_EINVAL, "execute_gemm: output must be M x N");
    if (row_begin < 0 || row_end > m || row_begin > row_end)
        return fail(Q8G_EINVAL, "execute_gemm: row stripe out of range");
    const int rows = row_end - row_begin;
    if (rows == 0) return Q8G_OK;
    const size_t esz = pl->writer == Q8G_WRITE_REQUANT_U8 ? 1 : 4;
    DeviceGuard dg(pb->device);
    const cudaStream_t s = (cudaStream_t)stream;
    const int lda_d = round_up_i(k, 16), n = pb->n;
    uint8_t* a_d = nullptr;
    void* c_d = nullptr;
    int32_t* b_d = nullptr;
    cudaError_t e;
    int rc = Q8G_OK;
    if ((e = cudaMalloc(&a_d, (size_t)rows * lda_d)) != cudaSuccess || (e = cudaMalloc(&c_d, esz * rows * n)) != cudaSuccess ||
        (bias_add_host && (e = cudaMalloc(&b_d, sizeof(int32_t) * n)) != cudaSuccess)) {
        rc = cuda_fail(e, "cudaMalloc(pipeline staging)");
    } else if ((e = cudaMemcpy2DAsync(a_d, lda_d, a_host + (size_t)row_begin * lda, lda, k, rows,
                                      cudaMemcpyHostToDevice, s)) != cudaSuccess ||
               (bias_add_host &&
                (e = cudaMemcpyAsync(b_d, bias_add_host, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s)) !=
                    cudaSuccess)) {
        rc = cuda_fail(e, "pipeline staging copy");
    } else {
        q8g_pipeline_args p2 = *pl;
        p2.bias_add_dev = b_d;
        rc = q8g_gemm_u8s8_pipeline(a_d, rows, k, lda_d, pb, &p2, c_d, n, 0, rows, nullptr, stream);
        if (rc == Q8G_OK &&
            ((e = cudaMemcpy2DAsync(static_cast<uint8_t*>(c_host) + esz * (size_t)row_begin * ldc, esz * ldc, c_d,
                                    esz * n, esz * n, rows, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
             (e = cudaStreamSynchronize(s)) != cudaSuccess))
            rc = cuda_fail(e, "pipeline result copy");
    }
    cudaStreamSynchronize(s);
    if (a_d) cudaFree(a_d);
    if (c_d) cudaFree(c_d);
    if (b_d) cudaFree(b_d);
    return rc;
}

}  // extern "C"

// Chunked host-view pipeline (large host-view calls): the inputs are split
// into chunks of `chunk` units (GEMM rows or images); chunk i's H2D copy, its
// compute and chunk i-1's D2H copy overlap on three streams (PCIe is full
// duplex), so a call costs about max(H2D, D2H) + one chunk instead of
// H2D + compute + D2H.  Per-device grow-only staging, calls serialised per
// device, synchronous for the caller.
namespace {
constexpr int kMaxChunks = 64;
struct HostPipe {
    std::mutex mu;
    uint8_t* in = nullptr;
    uint8_t* out = nullptr;
    size_t in_bytes = 0, out_bytes = 0;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_in[kMaxChunks] = {}, ev_out[kMaxChunks] = {};
    cudaEvent_t done = nullptr;
};
HostPipe g_host_pipe[64];

struct HostPipeSpec {
    const uint8_t* in_host;
    size_t in_pitch, in_width, in_dpitch;    // bytes per unit row: host pitch, copied bytes, device pitch
    uint8_t* out_host;
    size_t out_pitch, out_width, out_dpitch;
    int units, chunk;
    bool ramp = false;  // chunk sizes c/4, c/2, c, ..., c/2, c/4 (short first H2D and last D2H)
};

template <class F>
int run_host_pipeline(int device, cudaStream_t s, const HostPipeSpec& sp, F compute) {
    HostPipe& hp = g_host_pipe[device & 63];
    std::lock_guard<std::mutex> lock(hp.mu);
    cudaError_t e;
    const size_t need_in = sp.in_dpitch * (size_t)sp.units, need_out = sp.out_dpitch * (size_t)sp.units;
    if (hp.in_bytes < need_in) {
        if (hp.in) cudaFree(hp.in);
        hp.in = nullptr;
        hp.in_bytes = 0;
        if ((e = cudaMalloc(&hp.in, need_in)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(host pipeline input)");
        hp.in_bytes = need_in;
    }
    if (hp.out_bytes < need_out) {
        if (hp.out) cudaFree(hp.out);
        hp.out = nullptr;
        hp.out_bytes = 0;
        if ((e = cudaMalloc(&hp.out, need_out)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(host pipeline output)");
        hp.out_bytes = need_out;
    }
    if (!hp.h2d) {
        if ((e = cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&hp.done, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "host pipeline streams");
        for (int i = 0; i < kMaxChunks; ++i)
            if ((e = cudaEventCreateWithFlags(&hp.ev_in[i], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&hp.ev_out[i], cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "host pipeline events");
    }
    int chunk = sp.chunk < 1 ? 1 : sp.chunk;
    if ((sp.units + chunk - 1) / chunk > kMaxChunks) chunk = (sp.units + kMaxChunks - 1) / kMaxChunks;
    // the staging buffers may still be read by work the caller queued on s
    // before this call (a previous call is complete: calls are synchronous)
    if ((e = cudaEventRecord(hp.done, s)) != cudaSuccess || (e = cudaStreamWaitEvent(hp.h2d, hp.done, 0)) != cudaSuccess)
        return cuda_fail(e, "host pipeline ordering");
    // with sp.ramp chunk sizes ramp up and down (c/4, c/2, c, ..., c, c/2, c/4):
    // the first H2D and the last D2H run with nothing to overlap, so they are
    // kept short (C2 host call 1.81 -> 1.73 ms; not used for the conv paths,
    // whose smallest chunks would leave most SMs idle)
    int bounds[kMaxChunks + 1];
    int nch = 0;
    {
        const int q = chunk / 4 > 0 ? chunk / 4 : 1, h = chunk / 2 > 0 ? chunk / 2 : 1;
        const bool ramp = sp.ramp && sp.units >= 4 * chunk && (sp.units + chunk - 1) / chunk + 4 <= kMaxChunks;
        bounds[nch++] = 0;
        int u = 0;
        auto push = [&](int len) {
            u = u + len < sp.units ? u + len : sp.units;
            if (u > bounds[nch - 1]) bounds[nch++] = u;
        };
        if (ramp) {
            push(q);
            push(h);
            while (sp.units - u > chunk + h + q) push(chunk);
            const int rest = sp.units - u;  // (h + q, chunk + h + q]: split it c', h, q
            push(rest - h - q);
            push(h);
            push(q);
        } else {
            while (u < sp.units) push(chunk);
        }
        nch -= 1;  // chunks
    }
    int rc = Q8G_OK, i = 0;
    for (; i < nch && rc == Q8G_OK; ++i) {
        const int u0 = bounds[i], u1 = bounds[i + 1];
        const size_t n = (size_t)(u1 - u0);
        uint8_t* din = hp.in + sp.in_dpitch * u0;
        uint8_t* dout = hp.out + sp.out_dpitch * u0;
        e = cudaMemcpy2DAsync(din, sp.in_dpitch, sp.in_host + sp.in_pitch * u0, sp.in_pitch, sp.in_width, n,
                              cudaMemcpyHostToDevice, hp.h2d);
        if (e == cudaSuccess) e = cudaEventRecord(hp.ev_in[i], hp.h2d);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, hp.ev_in[i], 0);
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "host pipeline H2D");
            break;
        }
        rc = compute(u0, u1, din, dout);
        if (rc) break;
        e = cudaEventRecord(hp.ev_out[i], s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(hp.d2h, hp.ev_out[i], 0);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(sp.out_host + sp.out_pitch * u0, sp.out_pitch, dout, sp.out_dpitch, sp.out_width, n,
                                  cudaMemcpyDeviceToHost, hp.d2h);
        if (e != cudaSuccess) rc = cuda_fail(e, "host pipeline D2H");
    }
    // drain every stream before the staging can be reused (also on error)
    cudaError_t e1 = cudaEventRecord(hp.done, hp.d2h);
    if (e1 == cudaSuccess) e1 = cudaEventSynchronize(hp.done);
    cudaStreamSynchronize(hp.h2d);
    cudaStreamSynchronize(s);
    if (!rc && e1 != cudaSuccess) rc = cuda_fail(e1, "host pipeline completion");
    return rc;
}
}  // namespace

// images per chunk of the host-view conv / depthwise pipelines: imgs / parts
// (Q8G_HOST_CHUNK_IMG overrides, A/B)
static int host_chunk_images(int imgs, int parts, size_t img_bytes) {
    static const int env = [] {
        const char* e = getenv("Q8G_HOST_CHUNK_IMG");
        return e ? atoi(e) : 0;
    }();
    if (env > 0) return env;
    // at least ~2 MB per chunk: each chunk costs ~20 us of host-side API calls
    // (two copies, events, the launch), which small chunks cannot amortize
    // (C3, 6.4 MB each way: 4-image chunks 270-416 us per call, 16-image
    // chunks 240 us)
    const size_t total = img_bytes * (size_t)imgs;
    const int by_size = (int)std::max<size_t>(1, total / ((size_t)2 << 20));
    parts = std::max(1, std::min(parts, by_size));
    return std::max(1, (imgs + parts - 1) / parts);
}

// rows per chunk of the host-view GEMM pipeline (Q8G_HOST_CHUNK overrides, A/B)
static int host_chunk_rows(int rows) {
    static const int env = [] {
        const char* e = getenv("Q8G_HOST_CHUNK");
        return e ? atoi(e) : 0;
    }();
    if (env > 0) return round_up_i(env, 256);
    // C2 (16384 rows), host wall time per call: 1024-row chunks 2.02 ms,
    // 2048 1.81, 4096 1.83, 8192 2.13 (the copies alone, both directions
    // concurrently: 1.38 ms) -- per-chunk overhead vs pipeline fill
    return round_up_i(std::max(2048, rows / 8), 256);
}

template <typename OutT>
static int gemm_host(const uint8_t* a_host, int m, int k, int lda, const q8g_packed_b* pb,
                     const q8g_epilogue* ep, OutT* c_host, int ldc, int row_begin, int row_end,
                     cudaStream_t s, bool raw) {
    if (!pb || !a_host || !c_host) return fail(Q8G_EINVAL, "execute_gemm: null argument");
    if (row_begin < 0 || row_end > m || row_begin > row_end)
        return fail(Q8G_EINVAL, "execute_gemm: row stripe out of range");
    if (k != pb->k) return fail(Q8G_EINVAL, "execute_gemm: A columns must equal the packed weight K");
    if (lda < k || ldc < pb->n) return fail(Q8G_EINVAL, "execute_gemm: output must be M x N");
    const int rows = row_end - row_begin;
    if (rows == 0) return Q8G_OK;
    DeviceGuard dg(pb->device);
    const int lda_d = round_up_i(k, 16), ldc_d = pb->n;
    if (rows >= 4096) {
        // large stripes: chunks of >= 2048 rows (multiples of the 256-row
        // pair tile), copies overlapped with the GEMM of the previous chunk
        HostPipeSpec sp{a_host + (size_t)row_begin * lda, (size_t)lda, (size_t)k, (size_t)lda_d,
                        reinterpret_cast<uint8_t*>(c_host + (size_t)row_begin * ldc), sizeof(OutT) * ldc,
                        sizeof(OutT) * pb->n, sizeof(OutT) * ldc_d, rows, host_chunk_rows(rows), true};
        return run_host_pipeline(pb->device, s, sp, [&](int u0, int u1, uint8_t* din, uint8_t* dout) {
            return gemm_common(din, u1 - u0, k, lda_d, pb, raw ? nullptr : ep, nullptr, dout, ldc_d, 0, u1 - u0,
                               nullptr, s, raw);
        });
    }
    // grow-only per-device staging buffers; host-view calls are synchronous
    // and serialised per device by this lock.  A is copied on a separate
    // stream followed by a copy of the call's epoch into `flag`: the
    // GEMM is launched at the same time and streams the (immutable) weights
    // while A is in flight (the split-K kernel polls the flag before its first
    // A load; other kernels wait on it in-stream).
    struct Staging {
        std::mutex mu;
        void* a = nullptr;
        void* c = nullptr;
        size_t a_bytes = 0, c_bytes = 0;
        cudaStream_t copy = nullptr;
        uint32_t* flag = nullptr;
        uint32_t epoch = 0;
        cudaEvent_t done = nullptr;  // spin-waited (no BlockingSync): low wake-up latency
        uint32_t* epoch_host = nullptr;  // pinned source of the flag copy
    };
    static Staging staging[64];
    Staging& st = staging[pb->device & 63];
    std::lock_guard<std::mutex> lock(st.mu);
    cudaError_t e;
    const size_t need_a = (size_t)rows * lda_d, need_c = sizeof(OutT) * (size_t)rows * ldc_d;
    if (st.a_bytes < need_a) {
        if (st.a) cudaFree(st.a);
        st.a = nullptr;
        st.a_bytes = 0;
        if ((e = cudaMalloc(&st.a, need_a)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(A staging)");
        st.a_bytes = need_a;
    }
    if (st.c_bytes < need_c) {
        if (st.c) cudaFree(st.c);
        st.c = nullptr;
        st.c_bytes = 0;
        if ((e = cudaMalloc(&st.c, need_c)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(C staging)");
        st.c_bytes = need_c;
    }
    if (!st.copy) {
        if ((e = cudaStreamCreateWithFlags(&st.copy, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e, "copy stream");
        if ((e = cudaMalloc(&st.flag, sizeof(uint32_t))) != cudaSuccess ||
            (e = cudaMemsetAsync(st.flag, 0, sizeof(uint32_t), st.copy)) != cudaSuccess)
            return cuda_fail(e, "A-ready flag");
        if ((e = cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "completion event");
        if ((e = cudaHostAlloc(&st.epoch_host, sizeof(uint32_t), cudaHostAllocDefault)) != cudaSuccess)
            return cuda_fail(e, "pinned epoch");
    }
    uint32_t epoch = ++st.epoch;
    if (epoch == 0) epoch = ++st.epoch;
    uint8_t* d_a = (uint8_t*)st.a;
    OutT* d_c = (OutT*)st.c;
    int rc = Q8G_OK;
    // contiguous rows: one linear copy
    if (lda == k && lda_d == k)
        e = cudaMemcpyAsync(d_a, a_host + (size_t)row_begin * lda, (size_t)rows * k, cudaMemcpyHostToDevice, st.copy);
    else
        e = cudaMemcpy2DAsync(d_a, lda_d, a_host + (size_t)row_begin * lda, lda, k, rows, cudaMemcpyHostToDevice,
                              st.copy);
    // the flag is written by the same copy stream right behind A (a 4-byte
    // copy from pinned memory, ordered after A's bytes).  Reusing the pinned
    // word is safe: calls are synchronous, so the previous call's flag copy
    // has completed.
    *st.epoch_host = epoch;
    if (e == cudaSuccess) e = cudaMemcpyAsync(st.flag, st.epoch_host, sizeof(uint32_t), cudaMemcpyHostToDevice, st.copy);

    if (e != cudaSuccess) rc = cuda_fail(e, "H2D A");
    if (!rc) {
        if (raw)
            rc = gemm_common(d_a, rows, k, lda_d, pb, nullptr, nullptr, d_c, ldc_d, 0, rows, nullptr, s, true,
                             st.flag, epoch);
        else
            rc = gemm_common(d_a, rows, k, lda_d, pb, ep, nullptr, d_c, ldc_d, 0, rows, nullptr, s, false,
                             st.flag, epoch);
    }
    if (rc) cudaStreamSynchronize(st.copy);  // never leave the copy in flight into freed staging
    if (!rc) {
        if (ldc == pb->n && ldc_d == pb->n)
            e = cudaMemcpyAsync(c_host + (size_t)row_begin * ldc, d_c, sizeof(OutT) * (size_t)rows * pb->n,
                                cudaMemcpyDeviceToHost, s);
        else
            e = cudaMemcpy2DAsync(c_host + (size_t)row_begin * ldc, sizeof(OutT) * ldc, d_c, sizeof(OutT) * ldc_d,
                                  sizeof(OutT) * pb->n, rows, cudaMemcpyDeviceToHost, s);
        // the call is synchronous: spin on an event (cudaStreamSynchronize
        // may yield the thread and wake up several us late)
        if (e == cudaSuccess) e = cudaEventRecord(st.done, s);
        if (e == cudaSuccess) e = cudaEventSynchronize(st.done);
        if (e != cudaSuccess) rc = cuda_fail(e, "D2H C");
    }
    return rc;
}

extern "C" {

int q8g_gemm_u8s8_requant_host(const uint8_t* a_host, int m, int k, int lda,
                               const q8g_packed_b* pb, const q8g_epilogue* ep, uint8_t* c_host,
                               int ldc, int row_begin, int row_end, void* stream) {
    if (!ep) return fail(Q8G_EINVAL, "pipeline writer does not match the output element type");
    return gemm_host<uint8_t>(a_host, m, k, lda, pb, ep, c_host, ldc, row_begin, row_end,
                              (cudaStream_t)stream, false);
}

int q8g_gemm_u8s8_raw_i32_host(const uint8_t* a_host, int m, int k, int lda,
                               const q8g_packed_b* pb, int32_t* c_host, int ldc, int row_begin,
                               int row_end, void* stream) {
    return gemm_host<int32_t>(a_host, m, k, lda, pb, nullptr, c_host, ldc, row_begin, row_end,
                              (cudaStream_t)stream, true);
}

// ---------------------------------------------------------------- conv 3x3

static int conv_common(const uint8_t* x, int nb, int h, int w, int c, int32_t zp_a,
                       const q8g_packed_b* pw, const q8g_epilogue* ep, void* y, int img_begin,
                       int img_end, cudaStream_t s, bool raw) {
    if (!pw || !x || !y) return fail(Q8G_EINVAL, "conv3x3: null argument");
    if (nb < 1 || h < 1 || w < 1 || c < 1) return fail(Q8G_EINVAL, "conv3x3: dimensions must be >= 1");
    if (pw->k != 9 * c) return fail(Q8G_EINVAL, "conv3x3: packed weight K must equal 9*C");
    if (img_begin < 0 || img_end > nb || img_begin > img_end)
        return fail(Q8G_EINVAL, "conv3x3: image range out of bounds");
    if (!raw && (!ep || ep->n != pw->n))
        return fail(Q8G_EINVAL, "conv3x3: epilogue does not match the packed weight");
    if (zp_a < 0 || zp_a > 255) return fail(Q8G_EINVAL, "conv3x3: zp_a must be a u8 value");
    if (img_begin == img_end) return Q8G_OK;
    DeviceGuard dg(pw->device);
    ConvArgs a;
    const size_t img_px = (size_t)h * w;
    a.x = x + (size_t)img_begin * img_px * c;
    a.nb = img_end - img_begin;
    a.h = h;
    a.w = w;
    a.c = c;
    a.zp_a = zp_a;
    a.pw = pw;
    a.ep = ep;
    a.raw = raw;
    a.y = raw ? (void*)((int32_t*)y + (size_t)img_begin * img_px * pw->n)
              : (void*)((uint8_t*)y + (size_t)img_begin * img_px * pw->n);
    cudaError_t e = launch_conv3x3(a, s);
    if (e != cudaSuccess) return cuda_fail(e, "conv3x3 launch");
    return Q8G_OK;
}

int q8g_conv3x3_prepare(const q8g_packed_b* pw, int c, void* stream) {
    if (!pw || c < 1) return fail(Q8G_EINVAL, "conv3x3: bad arguments");
    if (pw->k != 9 * c) return fail(Q8G_EINVAL, "conv3x3: packed weight K must equal 9*C");
    DeviceGuard dg(pw->device);
    const cudaError_t e = conv_tc_prepare(pw, c, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "conv3x3 operand image");
    return Q8G_OK;
}

int q8g_conv3x3_u8s8_nhwc(const uint8_t* x_dev, int nb, int h, int w, int c,
                          const q8g_packed_b* pw, const q8g_epilogue* ep, uint8_t* y_dev,
                          int img_begin, int img_end, void* stream) {
    if (!ep) return fail(Q8G_EINVAL, "conv3x3: null epilogue");
    return conv_common(x_dev, nb, h, w, c, ep->zp_a, pw, ep, y_dev, img_begin, img_end,
                       (cudaStream_t)stream, false);
}

int q8g_conv3x3_u8s8_nhwc_raw_i32(const uint8_t* x_dev, int nb, int h, int w, int c,
                                  int32_t zp_a, const q8g_packed_b* pw, int32_t* y_dev,
                                  int img_begin, int img_end, void* stream) {
    return conv_common(x_dev, nb, h, w, c, zp_a, pw, nullptr, y_dev, img_begin, img_end,
                       (cudaStream_t)stream, true);
}

// ---------------------------------------------------------------- depthwise

int q8g_dw_filter_create(const int8_t* w_host, int c, const q8g_requant_params* p, int device,
                         q8g_dw_filter** out) {
    if (!w_host || !p || !out || c < 1) return fail(Q8G_EINVAL, "dw_filter: bad arguments");
    *out = nullptr;
    if (p->rounding != Q8G_ROUND_F32_RNE)
        return fail(Q8G_ENOTSUP, "dwconv3x3: only F32_RNE requantization is supported");
    if (p->zp_a < 0 || p->zp_a > 255) return fail(Q8G_EINVAL, "dwconv3x3: zp_a must be a u8 value");
    std::vector<int32_t> wsum(c, 0);
    for (int t = 0; t < 9; ++t)
        for (int ch = 0; ch < c; ++ch) wsum[ch] += w_host[t * c + ch];
    std::vector<EpiRecord> rec;
    bool need_rowsum = false;
    int rc = build_records(c, c, 9, p, wsum.data(), nullptr, rec, need_rowsum);
    if (rc) return rc;
    DeviceGuard dg(device);
    auto* f = new (std::nothrow) q8g_dw_filter();
    if (!f) return fail(Q8G_ENOMEM, "out of host memory");
    f->device = device;
    f->c = c;
    f->zp_a = p->zp_a;
    f->zp_c = p->zp_c;
    f->relu = p->relu ? 1 : 0;
    cudaError_t e;
    if ((e = cudaMalloc(&f->w, (size_t)9 * c)) != cudaSuccess ||
        (e = cudaMalloc(&f->rec, sizeof(EpiRecord) * c)) != cudaSuccess ||
        (e = cudaMemcpy(f->w, w_host, (size_t)9 * c, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(f->rec, rec.data(), sizeof(EpiRecord) * c, cudaMemcpyHostToDevice)) !=
            cudaSuccess) {
        q8g_dw_filter_free(f);
        return cuda_fail(e, "dw_filter upload");
    }
    // ---- tensor-core path constants (dwconv_tc.cu).  Exactness conditions:
    // the float magic-number conversions need |adj| < 2^22, and the clamp
    // folding needs 0 <= zp_c <= 255; otherwise the CUDA-core kernel runs.
    {
        std::vector<int32_t> zpw(c), cterm(c), corr(16 * c, 0);
        std::vector<float> mult(c);
        bool ok = p->zp_c >= 0 && p->zp_c <= 255;
        int64_t max_bias = 0;
        for (int ch = 0; ch < c; ++ch) {
            const int64_t zw = p->zp_b_per_channel_host ? p->zp_b_per_channel_host[ch] : p->zp_b;
            const int64_t b = p->bias_host ? p->bias_host[ch] : 0;
            zpw[ch] = (int32_t)zw;
            if (zw < -127 || zw > 127) ok = false;  // -zp_w must fit the s8 Z matrix
            max_bias = std::max<int64_t>(max_bias, b < 0 ? -b : b);
            const int64_t ct = b - (int64_t)p->zp_a * wsum[ch] + 9LL * p->zp_a * zw;
            cterm[ch] = (int32_t)(ct + 0x4B400000LL);
            mult[ch] = rec[ch].mf;
            if (!(mult[ch] < 7.9228163e28f)) ok = false;  // finite, < 2^96: no inf/NaN products
            for (int cls = 1; cls < 16; ++cls) {
                int64_t s = 0;
                for (int t = 0; t < 9; ++t) {
                    const int kh = t / 3, kw = t % 3;
                    const bool padded = ((cls & 1) && kh == 0) || ((cls & 2) && kh == 2) || ((cls & 4) && kw == 0) ||
                                        ((cls & 8) && kw == 2);
                    if (padded) s += (int64_t)w_host[t * c + ch] - zw;
                }
                corr[cls * c + ch] = (int32_t)(p->zp_a * s);
            }
        }
        // |adj| <= 9 * 255 * (128 + |zp_w|) + |bias| must stay below 2^22
        const bool ok_fma = ok;  // the FMA path has its own bias bound (below)
        if (9LL * 255 * 256 + max_bias >= (1LL << 22)) ok = false;
        f->lo = p->relu ? 0.0f : (float)(-p->zp_c);
        f->hi = (float)(255 - p->zp_c);
        if (ok) {
            if ((e = cudaMalloc(&f->zpw_dev, sizeof(int32_t) * c)) != cudaSuccess ||
                (e = cudaMalloc(&f->cterm_dev, sizeof(int32_t) * c)) != cudaSuccess ||
                (e = cudaMalloc(&f->mult_dev, sizeof(float) * c)) != cudaSuccess ||
                (e = cudaMalloc(&f->corr_dev, sizeof(int32_t) * 16 * c)) != cudaSuccess ||
                (e = cudaMemcpy(f->zpw_dev, zpw.data(), sizeof(int32_t) * c, cudaMemcpyHostToDevice)) != cudaSuccess ||
                (e = cudaMemcpy(f->cterm_dev, cterm.data(), sizeof(int32_t) * c, cudaMemcpyHostToDevice)) !=
                    cudaSuccess ||
                (e = cudaMemcpy(f->mult_dev, mult.data(), sizeof(float) * c, cudaMemcpyHostToDevice)) != cudaSuccess ||
                (e = cudaMemcpy(f->corr_dev, corr.data(), sizeof(int32_t) * 16 * c, cudaMemcpyHostToDevice)) !=
                    cudaSuccess) {
                q8g_dw_filter_free(f);
                return cuda_fail(e, "dw_filter tensor-core tables");
            }
            f->tc_ok = true;
        }
        // ---- CUDA-core FMA path constants (dwconv_fma.cu).  Exactness: every
        // partial sum bias' + sum x*w' is an integer below 2^23 (|w'| <= 255),
        // mult * 2^30 is finite, and the magic-number requant needs
        // 0 <= zp_c <= 255
        const int64_t fma_bound = max_bias + 2LL * 9 * 255 * 255;
        if (ok_fma && c % 4 == 0 && fma_bound < (1LL << 23)) {
            std::vector<float> fw((size_t)9 * c), fb(c), fm(c), fc((size_t)16 * c);
            for (int ch = 0; ch < c; ++ch) {
                int64_t ws = 0;
                for (int t = 0; t < 9; ++t) {
                    const int wp = (int)w_host[t * c + ch] - zpw[ch];
                    ws += wp;
                    fw[((size_t)(ch / 4) * 9 + t) * 4 + ch % 4] = std::ldexp((float)wp, 119);
                }
                const int64_t b = p->bias_host ? p->bias_host[ch] : 0;
                fb[ch] = std::ldexp((float)(b - (int64_t)p->zp_a * ws), -30);
                fm[ch] = std::ldexp(mult[ch], 30);
                for (int cls = 0; cls < 16; ++cls) fc[(size_t)cls * c + ch] = std::ldexp((float)corr[cls * c + ch], -30);
            }
            if ((e = cudaMalloc(&f->fma_w, sizeof(float) * 9 * c)) != cudaSuccess ||
                (e = cudaMalloc(&f->fma_b, sizeof(float) * c)) != cudaSuccess ||
                (e = cudaMalloc(&f->fma_m, sizeof(float) * c)) != cudaSuccess ||
                (e = cudaMalloc(&f->fma_corr, sizeof(float) * 16 * c)) != cudaSuccess ||
                (e = cudaMemcpy(f->fma_corr, fc.data(), sizeof(float) * 16 * c, cudaMemcpyHostToDevice)) !=
                    cudaSuccess ||
                (e = cudaMemcpy(f->fma_w, fw.data(), sizeof(float) * 9 * c, cudaMemcpyHostToDevice)) != cudaSuccess ||
                (e = cudaMemcpy(f->fma_b, fb.data(), sizeof(float) * c, cudaMemcpyHostToDevice)) != cudaSuccess ||
                (e = cudaMemcpy(f->fma_m, fm.data(), sizeof(float) * c, cudaMemcpyHostToDevice)) != cudaSuccess) {
                q8g_dw_filter_free(f);
                return cuda_fail(e, "dw_filter FMA tables");
            }
        }
    }
    *out = f;
    return Q8G_OK;
}

int q8g_dw_filter_free(q8g_dw_filter* f) {
    if (!f) return Q8G_OK;
    DeviceGuard dg(f->device);
    if (f->w) cudaFree(f->w);
    if (f->rec) cudaFree(f->rec);
    if (f->zpw_dev) cudaFree(f->zpw_dev);
    if (f->cterm_dev) cudaFree(f->cterm_dev);
    if (f->mult_dev) cudaFree(f->mult_dev);
    if (f->corr_dev) cudaFree(f->corr_dev);
    if (f->fma_w) cudaFree(f->fma_w);
    if (f->fma_b) cudaFree(f->fma_b);
    if (f->fma_m) cudaFree(f->fma_m);
    if (f->fma_corr) cudaFree(f->fma_corr);
    delete f;
    return Q8G_OK;
}

int q8g_dwconv3x3_u8s8_nhwc(const uint8_t* x_dev, int nb, int h, int w, int c,
                            const q8g_dw_filter* f, uint8_t* y_dev, int img_begin, int img_end,
                            void* stream) {
    if (!f || !x_dev || !y_dev) return fail(Q8G_EINVAL, "dwconv3x3: null argument");
    if (nb < 1 || h < 1 || w < 1 || c < 1) return fail(Q8G_EINVAL, "dwconv3x3: dimensions must be >= 1");
    if (c != f->c) return fail(Q8G_EINVAL, "dwconv3x3: channel count does not match the filter");
    if (img_begin < 0 || img_end > nb || img_begin > img_end)
        return fail(Q8G_EINVAL, "dwconv3x3: image range out of bounds");
    if (img_begin == img_end) return Q8G_OK;
    DeviceGuard dg(f->device);
    const size_t img = (size_t)h * w * c;
    cudaError_t e = launch_dwconv3x3(x_dev + img_begin * img, img_end - img_begin, h, w, c, f,
                                     y_dev + img_begin * img, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "dwconv3x3 launch");
    return Q8G_OK;
}


/* host views: images [img_begin, img_end) of x_host are staged through the
 * device in chunks whose copies overlap the previous chunk's convolution;
 * synchronous (the reference calling convention) */
int q8g_conv3x3_u8s8_nhwc_host(const uint8_t* x_host, int nb, int h, int w, int c, const q8g_packed_b* pw,
                               const q8g_epilogue* ep, uint8_t* y_host, int img_begin, int img_end, void* stream) {
    if (!pw || !ep || !x_host || !y_host) return fail(Q8G_EINVAL, "conv3x3: null argument");
    if (nb < 1 || h < 1 || w < 1 || c < 1) return fail(Q8G_EINVAL, "conv3x3: dimensions must be >= 1");
    if (img_begin < 0 || img_end > nb || img_begin > img_end)
        return fail(Q8G_EINVAL, "conv3x3: image range out of bounds");
    if (img_begin == img_end) return Q8G_OK;
    DeviceGuard dg(pw->device);
    const size_t xi = (size_t)h * w * c, yi = (size_t)h * w * pw->n;
    const int imgs = img_end - img_begin;
    HostPipeSpec sp{x_host + xi * img_begin, xi, xi, xi, y_host + yi * img_begin, yi, yi, yi, imgs,
                    host_chunk_images(imgs, 8, xi)};
    sp.ramp = (size_t)sp.chunk * xi >= ((size_t)4 << 20);  // (C3: 0.8 MB chunks, no ramp)
    const cudaStream_t s = (cudaStream_t)stream;
    return run_host_pipeline(pw->device, s, sp, [&](int u0, int u1, uint8_t* din, uint8_t* dout) {
        (void)u0;
        return conv_common(din, u1 - u0, h, w, c, ep->zp_a, pw, ep, dout, 0, u1 - u0, s, false);
    });
}

int q8g_dwconv3x3_u8s8_nhwc_host(const uint8_t* x_host, int nb, int h, int w, int c, const q8g_dw_filter* f,
                                 uint8_t* y_host, int img_begin, int img_end, void* stream) {
    if (!f || !x_host || !y_host) return fail(Q8G_EINVAL, "dwconv3x3: null argument");
    if (nb < 1 || h < 1 || w < 1 || c < 1) return fail(Q8G_EINVAL, "dwconv3x3: dimensions must be >= 1");
    if (c != f->c) return fail(Q8G_EINVAL, "dwconv3x3: channel count does not match the filter");
    if (img_begin < 0 || img_end > nb || img_begin > img_end)
        return fail(Q8G_EINVAL, "dwconv3x3: image range out of bounds");
    if (img_begin == img_end) return Q8G_OK;
    DeviceGuard dg(f->device);
    const size_t img = (size_t)h * w * c;
    const int imgs = img_end - img_begin;
    HostPipeSpec sp{x_host + img * img_begin, img, img, img, y_host + img * img_begin, img, img, img, imgs,
                    host_chunk_images(imgs, 8, img)};  // C4 e2e: 4-image chunks 2.48 ms, 2: 2.59, 8: 2.57
    sp.ramp = (size_t)sp.chunk * img >= ((size_t)4 << 20);  // copies long enough to outweigh per-chunk overhead
    const cudaStream_t s = (cudaStream_t)stream;
    return run_host_pipeline(f->device, s, sp, [&](int u0, int u1, uint8_t* din, uint8_t* dout) {
        (void)u0;
        const cudaError_t e = launch_dwconv3x3(din, u1 - u0, h, w, c, f, dout, s);
        return e == cudaSuccess ? Q8G_OK : cuda_fail(e, "dwconv3x3 launch");
    });
}

}  // extern "C"
