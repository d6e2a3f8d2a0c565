// gemm_tc.cu — the hot path: u8 x s8 -> s32 GEMM on the 5th-generation
// tensor cores (tcgen05.mma kind::i8, int32 accumulators in TMEM) with the
// requantization back-end fused onto the TMEM -> register -> global drain.
//
// Replaces, for the reference (proj/include/q8gemm/):
//   execute_gemm's five loops (engine.hpp:109-167) + microkernel_i32
//   (kernel.hpp:42-68, 108-112, 150-153)          -> MMA warp + TMEM
//   pack_a_with_row_offsets (pack.hpp:83-135)      -> TMA producer (A tile,
//                                                     swizzled in smem) +
//                                                     row-sum warps reading it
//   run_block + Requantize/ReluQuantized/WriteRawI32 (pipeline.hpp:157-210,
//   quant.hpp:115-133)                             -> epilogue warps
//
// One CTA per SM, warp-specialised, persistent over output tiles:
//   warp 0      TMA producer: A tile (128 rows x 128 B of K) by tensor map
//               (multicast across a cluster of CN CTAs that share the rows),
//               B tile (BN channels x 128 B) by one cp.async.bulk of the
//               pre-swizzled packed weight
//   warp 1      MMA issuer (one thread): 4 x tcgen05.mma (K=32 each) per stage
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld 32 columns at a time, requantize, store
//   warps 8-11  row sums of A (only when some zp_b != 0, pipeline.hpp:114-119)
// Pipelines: smem stages full/empty (TMA <-> MMA + row sums), TMEM double
// buffer full/empty (MMA <-> epilogue), row-sum double buffer.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "ptx.cuh"
#include "q8g_internal.cuh"
#include "epilogue.cuh"
#include "requant.cuh"

namespace q8g {
namespace {

constexpr int BM = 128;
constexpr int A_STAGE_BYTES = BM * kKBlock;  // 16 KB

template <int BN, int CN, int STAGES>
struct TcCfg {
    static constexpr int B_STAGE_BYTES = BN * kKBlock;
    static constexpr int TMEM_COLS = (2 * BN) < 32 ? 32 : 2 * BN;  // power of two for BN in {16..256}
    static constexpr int A_OFF = 0;
    static constexpr int B_OFF = STAGES * A_STAGE_BYTES;
    static constexpr int BAR_OFF = B_OFF + STAGES * B_STAGE_BYTES;
    // barriers: full[S], empty[S], tfull[2], tempty[2], rfull[2], rempty[2], rsdone[S]
    static constexpr int NUM_BARS = 3 * STAGES + 8;
    static constexpr int RS_OFF = BAR_OFF + NUM_BARS * 8;
    static constexpr int TMEMPTR_OFF = RS_OFF + 2 * BM * 4;
    static constexpr int SMEM_BYTES = TMEMPTR_OFF + 16 + 1024;  // + alignment slack
};

struct TcParams {
    const int8_t* pb;        // packed B
    int np, nkb;             // padded N, number of 128-byte k-blocks
    int n;                   // logical N
    int rows;                // rows in this stripe
    int num_m_tiles, num_n_groups;
    const EpiRecord* rec;
    int32_t zp_c;
    int relu;
    int fast;                 // q8g_epilogue::fast_f32
    const int32_t* bias_add;  // raw writer only
    void* c;
    int ldc;
    unsigned long long* trace;  // debug: 8 globaltimer stamps per CTA (Q8G_TC_TRACE), else null
};

__device__ __forceinline__ void trace_stamp(const TcParams& p, int slot) {
#ifdef Q8G_TRACE
    if (p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[blockIdx.x * 8 + slot] = t;
    }
#endif
}
// per-k-block stamps of CTA 0's first tile: [8192 + kb] producer issue,
// [8192 + 64 + kb] MMA saw the stage land, [8192 + 128 + kb] MMA issued
__device__ __forceinline__ void trace_kb(const TcParams& p, int which, int kb) {
#ifdef Q8G_TRACE
    if (p.trace && blockIdx.x == 0 && kb < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8192 + which * 64 + kb] = t;
    }
#endif
}

constexpr int EPI_COLS = 16;  // columns per tcgen05.ld in the epilogue

template <int BN, int CN, int STAGES, int MODE, bool RS>
__global__ void __launch_bounds__(RS ? 384 : 256, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_a, const TcParams p) {
    using Cfg = TcCfg<BN, CN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the SWIZZLE_128B atoms
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_addr);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    Q8G_CHECK((uint32_t)Cfg::SMEM_BYTES <= ptx::dynamic_smem_size());
    ptx::griddep_launch_dependents();
    if (threadIdx.x == 0) trace_stamp(p, 0);
    const uint32_t rank = CN > 1 ? ptx::cluster_ctarank() : 0;
    const uint32_t sA = base + Cfg::A_OFF, sB = base + Cfg::B_OFF;
    const uint32_t bar0 = base + Cfg::BAR_OFF;
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 2 + a); };
    auto rfull_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 4 + a); };
    auto rempty_bar = [&](int a) { return bar0 + 8u * (2 * STAGES + 6 + a); };
    // row-sum warps have finished reading stage s (local; the MMA thread
    // waits on it before its commit releases the stage cluster-wide)
    auto rsdone_bar = [&](int s) { return bar0 + 8u * (2 * STAGES + 8 + s); };
    int32_t* rs_buf = reinterpret_cast<int32_t*>(smem + Cfg::RS_OFF);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + Cfg::TMEMPTR_OFF);

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(full_bar(s), 1);
            ptx::mbar_init(empty_bar(s), CN);  // one MMA commit per cluster CTA
            ptx::mbar_init(rsdone_bar(s), 4);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull_bar(a), 1);
            ptx::mbar_init(tempty_bar(a), 4);
            ptx::mbar_init(rfull_bar(a), 4);
            ptx::mbar_init(rempty_bar(a), 4);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<Cfg::TMEM_COLS>(ptx::smem_u32(tmem_ptr));
    ptx::tc_fence_before();
    __syncthreads();
    if (CN > 1) ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_ptr;
    ptx::griddep_wait();  // PDL: the prologue above overlapped the previous grid
    if (threadIdx.x == 0) trace_stamp(p, 1);

    const int num_clusters = gridDim.x / CN;
    const int cluster_id = blockIdx.x / CN;
    const int total = p.num_m_tiles * p.num_n_groups;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        // (whole warp runs the loop with warp-uniform values; one elected lane
        // issues -- see ptx::elect_one)
        const uint64_t pol_b = ptx::policy_evict_last();  // weights are re-read by every M tile
        int stage = 0;
        uint32_t phase = 0;
        for (int t = cluster_id; t < total; t += num_clusters) {
            const int m_blk = t / p.num_n_groups, ng = t % p.num_n_groups;
            const int m0 = m_blk * BM;
            const int n0 = (ng * CN + (int)rank) * BN;
            for (int kb = 0; kb < p.nkb; ++kb) {
                ptx::mbar_wait(empty_bar(stage), phase ^ 1);
                const uint32_t a_dst = sA + stage * A_STAGE_BYTES;
                const int8_t* src = p.pb + ((size_t)kb * p.np + n0) * kKBlock;
                if (ptx::elect_one()) {
                    ptx::mbar_arrive_expect_tx(full_bar(stage), A_STAGE_BYTES + Cfg::B_STAGE_BYTES);
                    if (CN == 1) {
                        ptx::tma_load_2d(a_dst, &tmap_a, kb * kKBlock, m0, full_bar(stage));
                    } else {
                        constexpr int SLICE = BM / CN;
                        ptx::tma_load_2d_mc(a_dst + rank * SLICE * kKBlock, &tmap_a, kb * kKBlock,
                                            m0 + (int)rank * SLICE, full_bar(stage), (uint16_t)((1u << CN) - 1));
                    }
                    ptx::bulk_load_hint(sB + stage * Cfg::B_STAGE_BYTES, src, Cfg::B_STAGE_BYTES, full_bar(stage),
                                        pol_b);
                    if (kb == 0 && t == cluster_id) trace_stamp(p, 2);
                    if (t == cluster_id) trace_kb(p, 0, kb);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = ptx::idesc_u8s8_s32<BM, BN>();
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = cluster_id; t < total; t += num_clusters) {
            ptx::mbar_wait(tempty_bar(acc), acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem_base + (uint32_t)(acc * BN);
            for (int kb = 0; kb < p.nkb; ++kb) {
                ptx::mbar_wait(full_bar(stage), phase);
                ptx::tc_fence_after();
                const uint64_t adesc = ptx::sw128_kmajor_desc(sA + stage * A_STAGE_BYTES);
                const uint64_t bdesc = ptx::sw128_kmajor_desc(sB + stage * Cfg::B_STAGE_BYTES);
                if (ptx::elect_one()) {
                    if (kb == 0 && t == cluster_id) trace_stamp(p, 3);
                    if (t == cluster_id) trace_kb(p, 1, kb);
#pragma unroll
                    for (int ks = 0; ks < kKBlock / 32; ++ks)
                        ptx::mma_i8(d, adesc + 2 * ks, bdesc + 2 * ks, idesc, (kb | ks) != 0);
                    if (t == cluster_id) trace_kb(p, 2, kb);
                }
                __syncwarp();
                // the stage is released only after the row-sum warps read it too;
                // the same (lowest) lane is elected again, so it commits its MMAs
                if (RS) ptx::mbar_wait(rsdone_bar(stage), phase);
                if (ptx::elect_one()) {
                    if (CN == 1)
                        ptx::tc_commit(empty_bar(stage));
                    else
                        ptx::tc_commit_mc(empty_bar(stage), (uint16_t)((1u << CN) - 1));
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (ptx::elect_one()) {
                ptx::tc_commit(tfull_bar(acc));
                trace_stamp(p, 4);
            }
            __syncwarp();
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ------------------------------------------------ epilogue
        const int ew = warp - 4;  // == warp % 4: TMEM lanes [32*ew, 32*ew+32)
        const int r = ew * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = cluster_id; t < total; t += num_clusters) {
            const int m_blk = t / p.num_n_groups, ng = t % p.num_n_groups;
            const int m0 = m_blk * BM;
            const int n0 = (ng * CN + (int)rank) * BN;
            ptx::mbar_wait(tfull_bar(acc), acc_phase);
            ptx::tc_fence_after();
            if (warp == 4 && lane == 0 && t == cluster_id) trace_stamp(p, 5);
            int32_t rowsum = 0;
            if (RS) {
                ptx::mbar_wait(rfull_bar(acc), acc_phase);
                rowsum = rs_buf[acc * BM + r];
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(rempty_bar(acc));
            }
            const int row = m0 + r;
            const bool valid = row < p.rows;
            const EpiArgs ea{p.rec, p.zp_c, p.relu, p.fast, p.bias_add, p.c, p.ldc, p.n};
#pragma unroll 1
            for (int ch = 0; ch < BN / EPI_COLS; ++ch) {
                uint32_t v[EPI_COLS];
                const uint32_t taddr =
                    tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * BN + ch * EPI_COLS);
                ptx::tmem_ld_32x32b_x16(taddr, v);
                ptx::tmem_ld_wait();
                const int col0 = n0 + ch * EPI_COLS;
                if (valid && col0 < p.n) store_chunk16<MODE>(ea, row, col0, v, rowsum);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty_bar(acc));
            if (warp == 4 && lane == 0) trace_stamp(p, 6);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (RS && warp >= 8) {
        // ------------------------------------------------ row sums of A
        const int r = (warp - 8) * 32 + lane;
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = cluster_id; t < total; t += num_clusters) {
            ptx::mbar_wait(rempty_bar(acc), acc_phase ^ 1);
            uint32_t sum = 0;
            for (int kb = 0; kb < p.nkb; ++kb) {
                ptx::mbar_wait(full_bar(stage), phase);
                // the row's 8 16-byte chunks in rotated order: conflict-free
                // across the warp; the sum is swizzle-invariant
                const uint8_t* rowp = smem + Cfg::A_OFF + stage * A_STAGE_BYTES + r * kKBlock;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint4 w = *reinterpret_cast<const uint4*>(rowp + ((q + r) & 7) * 16);
                    sum = ptx::dp4a_uu(w.x, 0x01010101u, sum);
                    sum = ptx::dp4a_uu(w.y, 0x01010101u, sum);
                    sum = ptx::dp4a_uu(w.z, 0x01010101u, sum);
                    sum = ptx::dp4a_uu(w.w, 0x01010101u, sum);
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(rsdone_bar(stage));
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            rs_buf[acc * BM + r] = (int32_t)sum;
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(rfull_bar(acc));
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }

    // reconverge every warp (lane 0 of the producer / MMA warps ran the role
    // loop alone) before the CTA-wide aligned barrier
    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    if (CN > 1) ptx::cluster_sync();
    if (threadIdx.x == 0) trace_stamp(p, 7);
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
}

// ------------------------------------------------------------------ host side

// debug phase trace (env Q8G_TC_TRACE=1): 8 globaltimer stamps per CTA of the
// most recent launch, read back with q8g_debug_tc_trace()
constexpr int kTraceCtas = 1024;
constexpr int kTraceWords = 8 * kTraceCtas + 2048;  // + per-k-block / per-unit stamps of CTA 0, per-CTA conv spans
unsigned long long* tc_trace_buffer() {
    static unsigned long long* buf = nullptr;
    static bool enabled = getenv("Q8G_TC_TRACE") != nullptr;
    if (!enabled) return nullptr;
    if (!buf) {
        if (cudaMalloc(&buf, sizeof(unsigned long long) * kTraceWords) != cudaSuccess) return nullptr;
        cudaMemset(buf, 0, sizeof(unsigned long long) * kTraceWords);
    }
    return buf;
}

}  // namespace

cudaError_t stream_write_u32(cudaStream_t s, uint32_t* addr, uint32_t value) {
    using Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    static Fn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        return (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                   ? reinterpret_cast<Fn>(f)
                   : nullptr;
    }();
    if (!fn) return cudaErrorNotSupported;
    // default flags: ordered after (and making visible) the stream's prior writes
    return fn((CUstream)s, (CUdeviceptr)addr, value, CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS
               ? cudaSuccess
               : cudaErrorUnknown;
}

cudaError_t stream_wait_u32(cudaStream_t s, const uint32_t* addr, uint32_t value) {
    using Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    static Fn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        return (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                   ? reinterpret_cast<Fn>(f)
                   : nullptr;
    }();
    if (!fn) return cudaErrorNotSupported;
    return fn((CUstream)s, (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_EQ) == CUDA_SUCCESS ? cudaSuccess
                                                                                                : cudaErrorUnknown;
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// A (rows x k, row-major, lda) as a 2-D u8 tensor, box = 128 bytes x box_rows,
// SWIZZLE_128B; out-of-range rows / k read as zero.
bool make_tmap_a(CUtensorMap* m, const uint8_t* a, int rows, int k, int lda, int box_rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)lda};
    cuuint32_t box[2] = {(cuuint32_t)kKBlock, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// small cache of encoded tensor maps keyed on the A view
struct TmapKey {
    const void* a;
    int rows, k, lda, box;
    bool operator==(const TmapKey& o) const {
        return a == o.a && rows == o.rows && k == o.k && lda == o.lda && box == o.box;
    }
};
struct TmapKeyHash {
    size_t operator()(const TmapKey& t) const {
        return std::hash<const void*>()(t.a) ^ ((size_t)t.rows * 1315423911u) ^ ((size_t)t.k << 20) ^
               ((size_t)t.lda << 40) ^ (size_t)t.box;
    }
};

bool cached_tmap_a(CUtensorMap* out, const uint8_t* a, int rows, int k, int lda, int box_rows) {
    static std::mutex mu;
    static std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> cache;
    TmapKey key{a, rows, k, lda, box_rows};
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return true;
    }
    if (!make_tmap_a(out, a, rows, k, lda, box_rows)) return false;
    if (cache.size() > 4096) cache.clear();
    cache.emplace(key, *out);
    return true;
}

template <int BN, int CN, int STAGES, int MODE, bool RS>
cudaError_t launch_variant(const GemmArgs& g, cudaStream_t s) {
    using Cfg = TcCfg<BN, CN, STAGES>;
    auto kern = gemm_tc_kernel<BN, CN, STAGES, MODE, RS>;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    CUtensorMap tmap;
    if (!cached_tmap_a(&tmap, g.a, g.rows, g.k, g.lda, BM / CN)) return cudaErrorInvalidValue;
    TcParams p;
    p.pb = g.pb->data;
    p.np = g.pb->np;
    p.nkb = g.pb->kp / kKBlock;
    p.n = g.pb->n;
    p.rows = g.rows;
    p.num_m_tiles = ceil_div_i(g.rows, BM);
    p.num_n_groups = g.pb->np / (BN * CN);
    p.rec = g.ep ? g.ep->rec : nullptr;
    p.zp_c = g.ep ? g.ep->zp_c : 0;
    p.relu = g.ep ? g.ep->relu : 0;
    p.fast = (g.ep && g.ep->fast_f32) ? 1 : 0;
    p.bias_add = g.bias_add;
    p.c = g.c;
    p.ldc = g.ldc;
    p.trace = tc_trace_buffer();
    const int total = p.num_m_tiles * p.num_n_groups;
    const int max_clusters = sm_count(dev) / CN;
    const int clusters = total < max_clusters ? total : max_clusters;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * CN);
    cfg.blockDim = dim3(RS ? 384 : 256);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (CN > 1) {  // cluster launch only when A is multicast
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = CN;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmap, p);
    count_launch((CN > 1 || BN < 256) ? kFamGemmTcSmallM : kFamGemmTcLargeM);
    return e;
}

template <int BN, int CN, int STAGES>
cudaError_t launch_modes(const GemmArgs& g, cudaStream_t s) {
    if (g.raw) return launch_variant<BN, CN, STAGES, 0, false>(g, s);
    const bool rs = g.ep->need_rowsum;
    if (g.ep->rounding == Q8G_ROUND_F32_RNE)
        return rs ? launch_variant<BN, CN, STAGES, 1, true>(g, s) : launch_variant<BN, CN, STAGES, 1, false>(g, s);
    return rs ? launch_variant<BN, CN, STAGES, 2, true>(g, s) : launch_variant<BN, CN, STAGES, 2, false>(g, s);
}

}  // namespace

bool make_tmap_a_cached(CUtensorMap* out, const uint8_t* a, int rows, int k, int lda, int box_rows) {
    return cached_tmap_a(out, a, rows, k, lda, box_rows);
}

unsigned long long* tc_trace_buffer_ptr() { return tc_trace_buffer(); }

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() { return get_encode(); }

int tc_trace_copy(unsigned long long* out, int max_ctas) {
    unsigned long long* buf = tc_trace_buffer();
    if (!buf) return 0;
    // max_ctas > kTraceCtas: also copy the per-k-block stamps (kTraceWords total)
    const int n = max_ctas < kTraceCtas ? max_ctas : kTraceCtas;
    const size_t words = max_ctas > kTraceCtas ? (size_t)kTraceWords : (size_t)8 * n;
    if (cudaDeviceSynchronize() != cudaSuccess) return 0;
    if (cudaMemcpy(out, buf, sizeof(unsigned long long) * words, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
    return n;
}

bool tc_supported(const GemmArgs& g) {
    return get_encode() != nullptr && (reinterpret_cast<uintptr_t>(g.a) % 16 == 0) && (g.lda % 16 == 0) &&
           g.k % 16 == 0 && g.k >= 16;
}

// Q8G_TC_CFG (tuning knob): force one tile config "BNxCN" for every
// tensor-core launch: 32x8, 32x1, 64x4, 128x2, 256x1
static int tc_cfg_override() {
    static int v = [] {
        const char* e = getenv("Q8G_TC_CFG");
        if (!e) return 0;
        std::string s(e);
        if (s == "32x8") return 1;
        if (s == "32x1") return 2;
        if (s == "64x4") return 3;
        if (s == "128x2") return 4;
        if (s == "256x1") return 5;
        if (s == "sk") return 6;
        return 0;
    }();
    return v;
}

cudaError_t launch_gemm_tc(const GemmArgs& g, int tile_kind, cudaStream_t s) {
    const int ov = tc_cfg_override();  // tuning knob Q8G_TC_CFG (0 = automatic)
    // split-K for small M (or forced); it is the only kernel that polls a
    // host-view A-ready flag itself (it streams B meanwhile)
    if ((ov == 6 || (ov == 0 && tile_kind == kSmallM)) && splitk_supported(g)) {
        const cudaError_t e = launch_gemm_splitk(g, s);
        if (e != cudaErrorNotSupported) return e;  // else: no workspace -> non-split kernel
    }
    if (g.a_ready) {
        const cudaError_t e = stream_wait_u32(s, g.a_ready, g.a_epoch);
        if (e != cudaSuccess) return e;
    }
    switch (ov) {
        case 1: return launch_modes<32, 8, 10>(g, s);
        case 2: return launch_modes<32, 1, 10>(g, s);
        case 3: return launch_modes<64, 4, 8>(g, s);
        case 4: return launch_modes<128, 2, 6>(g, s);
        case 5: return launch_modes<256, 1, 4>(g, s);
        default: break;
    }
    if (tile_kind == kSmallM) return launch_modes<32, 1, 10>(g, s);
    if (tile_kind == kMidM) return launch_modes<128, 2, 6>(g, s);
    if (tc2w_supported(g)) return launch_gemm_tc2w(g, s);  // CTA-pair 256x512 tiles
    return launch_modes<256, 1, 4>(g, s);
}

}  // namespace q8g
