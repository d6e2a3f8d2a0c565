// gemm_splitk.cu — small-M tensor-core GEMM (BASELINE C1: M <= 128 rows,
// large N x K): split-K across a thread-block cluster with the int32 partial
// accumulators reduced on chip, then the fused requantization.
//
// Why: with one 128-row M tile every N-slice CTA must stream all of A.  At
// 128 CTAs x 512 KB that is 64 MB of L2->SM traffic against 16.8 MB of
// weights, and A fills 80% of every pipeline stage (measured: loads take
// ~2 us to land, the kernel ran at 1 TB/s).  Splitting K S ways inside a
// cluster makes each CTA read only its K-slice of A (16 MB total), so half
// of every stage is weights and the mainloop runs at HBM speed.
//
// Exchange: rank r owns output columns [r*OWN, (r+1)*OWN) of the cluster's
// BN-wide tile.  After its mainloop each rank stages the partial columns the
// other ranks own (plus its partial row sums) in its now-idle pipeline smem
// and pushes them with one cp.async.bulk smem->peer-smem copy per peer; the
// copy completes on the owner's mbarrier.  (Register-issued
// st.shared::cluster stores were measured at ~25 GB/s per SM: 1.9 us for the
// 48 KB exchange.)
//
// Same drop-in semantics as gemm_tc.cu (engine.hpp:59-169 + Requantize,
// pipeline.hpp:157-210); int32 addition is associative so the split is
// bit-exact.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ptx.cuh"
#include "q8g_internal.cuh"
#include "requant.cuh"

namespace q8g {

bool make_tmap_a_cached(CUtensorMap* out, const uint8_t* a, int rows, int k, int lda, int box_rows);
unsigned long long* tc_trace_buffer_ptr();

namespace {

constexpr int BM = 128;
constexpr int A_STAGE = BM * kKBlock;

template <int BN, int S, int STAGES>
struct SkCfg {
    static constexpr int OWN = BN / S;  // columns owned per rank
    static constexpr int B_STAGE = BN * kKBlock;
    static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;  // one accumulator tile
    // one exchange slot: partials [OWN/4 quads][BM rows] int4, then [BM] row sums
    static constexpr int SLOT_PART = (OWN / 4) * BM * 16;
    static constexpr int SLOT_BYTES = SLOT_PART + BM * 4;
    static constexpr int A_OFF = 0;  // also the send staging area after the mainloop
    static constexpr int B_OFF = STAGES * A_STAGE;
    static constexpr int RECV_OFF = B_OFF + STAGES * B_STAGE;  // [S-1] slots
    static constexpr int OWNRS_OFF = RECV_OFF + (S - 1) * SLOT_BYTES;
    static constexpr int REC_OFF = OWNRS_OFF + BM * 4;  // [OWN] EpiRecord
    static constexpr int BAR_OFF = REC_OFF + OWN * 16;
    static constexpr int NUM_BARS = 3 * STAGES + 3;  // full, empty, rsdone, tfull, recvfull, rsready
    static constexpr int TMEMPTR_OFF = BAR_OFF + NUM_BARS * 8;
    static constexpr int SMEM_BYTES = TMEMPTR_OFF + 16 + 1024;
    static_assert((S - 1) * SLOT_BYTES <= STAGES * A_STAGE, "send staging must fit the A stages");
    static_assert(SLOT_BYTES % 16 == 0, "bulk copies move 16-byte multiples");
    static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

struct SkParams {
    const int8_t* pb;
    int np, nkb, n, rows;
    int num_n_tiles;
    const EpiRecord* rec;
    int32_t zp_c;
    int relu;
    const int32_t* bias_add;
    void* c;
    int ldc;
    unsigned long long* trace;  // debug stamps (Q8G_TC_TRACE), else null
};

// same slots as gemm_tc.cu: 0 entry, 1 prologue, 2 first TMA, 3 first stage,
// 4 last MMA commit, 5 epilogue start, 6 exchange landed, 7 stores issued;
// per-k-block stamps of CTA 0
__device__ __forceinline__ void sk_stamp(const SkParams& p, int slot) {
    if (p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[blockIdx.x * 8 + slot] = t;
    }
}
__device__ __forceinline__ void sk_kb(const SkParams& p, int which, int i) {
    if (p.trace && blockIdx.x == 0 && i < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8192 + which * 64 + i] = t;
    }
}

__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// smem -> peer smem bulk copy, completing tx bytes on the peer's mbarrier
__device__ __forceinline__ void bulk_s2cluster(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                               uint32_t mbar_cluster) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_cluster),
        "r"(src_cta), "r"(bytes), "r"(mbar_cluster)
        : "memory");
}

template <int BN, int S, int STAGES, int MODE, bool RS>
__global__ void __launch_bounds__(RS ? 384 : 256, 1)
    gemm_splitk_kernel(const __grid_constant__ CUtensorMap tmap_a, const SkParams p) {
    using Cfg = SkCfg<BN, S, STAGES>;
    constexpr int OWN = Cfg::OWN;
    static_assert(OWN % 16 == 0, "owned column block must be a multiple of 16");
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_addr);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    ptx::griddep_launch_dependents();
    if (threadIdx.x == 0) sk_stamp(p, 0);
    const uint32_t rank = ptx::cluster_ctarank();
    const int tile = blockIdx.x / S;
    const int m_blk = tile / p.num_n_tiles, n_blk = tile % p.num_n_tiles;
    const int m0 = m_blk * BM, n0 = n_blk * BN;
    // balanced contiguous k-block range of this rank (engine.hpp:40-47 formula)
    const int kb_base = p.nkb / S, kb_rem = p.nkb % S;
    const int kb0 = (int)rank * kb_base + ((int)rank < kb_rem ? (int)rank : kb_rem);
    const int kb1 = kb0 + kb_base + ((int)rank < kb_rem ? 1 : 0);

    const uint32_t sA = base + Cfg::A_OFF, sB = base + Cfg::B_OFF;
    const uint32_t bar0 = base + Cfg::BAR_OFF;
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
    auto rsdone_bar = [&](int s) { return bar0 + 8u * (2 * STAGES + s); };
    const uint32_t tfull = bar0 + 8u * (3 * STAGES);
    const uint32_t recvfull = bar0 + 8u * (3 * STAGES + 1);
    const uint32_t rsready = bar0 + 8u * (3 * STAGES + 2);
    int32_t* ownrs = reinterpret_cast<int32_t*>(smem + Cfg::OWNRS_OFF);
    const int4* recs = reinterpret_cast<const int4*>(smem + Cfg::REC_OFF);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + Cfg::TMEMPTR_OFF);

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(full_bar(s), 1);
            ptx::mbar_init(empty_bar(s), 1);
            ptx::mbar_init(rsdone_bar(s), 4);
        }
        ptx::mbar_init(tfull, 1);
        ptx::mbar_init(recvfull, 1);
        ptx::mbar_init(rsready, 4);
        ptx::fence_mbar_init();
        // all S-1 peer slots will complete on recvfull
        ptx::mbar_arrive_expect_tx(recvfull, (S - 1) * Cfg::SLOT_BYTES);
    }
    if (warp == 2) ptx::tmem_alloc<Cfg::TMEM_COLS>(ptx::smem_u32(tmem_ptr));
    ptx::tc_fence_before();
    __syncthreads();
    // early arrive: "my barriers are initialised, expect_tx is armed"; the
    // matching wait sits right before the first remote copy
    cluster_arrive_release();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_ptr;
    ptx::griddep_wait();  // PDL: the prologue above overlapped the previous grid
    if (threadIdx.x == 0) sk_stamp(p, 1);

    if (warp == 0) {
        // whole warp runs the loop; one elected lane issues (ptx::elect_one)
        const uint64_t pol_b = ptx::policy_evict_first();  // weights streamed once
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(empty_bar(stage), phase ^ 1);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(full_bar(stage), A_STAGE + Cfg::B_STAGE);
                ptx::tma_load_2d(sA + stage * A_STAGE, &tmap_a, kb * kKBlock, m0, full_bar(stage));
                ptx::bulk_load_hint(sB + stage * Cfg::B_STAGE, p.pb + ((size_t)kb * p.np + n0) * kKBlock,
                                    Cfg::B_STAGE, full_bar(stage), pol_b);
                if (kb == kb0) sk_stamp(p, 2);
                sk_kb(p, 0, kb - kb0);
            }
            __syncwarp();
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = ptx::idesc_u8s8_s32<BM, BN>();
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(full_bar(stage), phase);
            ptx::tc_fence_after();
            const uint64_t adesc = ptx::sw128_kmajor_desc(sA + stage * A_STAGE);
            const uint64_t bdesc = ptx::sw128_kmajor_desc(sB + stage * Cfg::B_STAGE);
            if (ptx::elect_one()) {
                if (kb == kb0) sk_stamp(p, 3);
                sk_kb(p, 1, kb - kb0);
#pragma unroll
                for (int ks = 0; ks < kKBlock / 32; ++ks)
                    ptx::mma_i8(tmem_base, adesc + 2 * ks, bdesc + 2 * ks, idesc, (kb > kb0 || ks > 0) ? 1u : 0u);
            }
            __syncwarp();
            if (RS) ptx::mbar_wait(rsdone_bar(stage), phase);
            if (ptx::elect_one()) ptx::tc_commit(empty_bar(stage));  // same lane as the MMAs
            __syncwarp();
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
        if (ptx::elect_one()) {
            ptx::tc_commit(tfull);
            sk_stamp(p, 4);
        }
        __syncwarp();
    } else if (RS && warp >= 8) {
        const int r = (warp - 8) * 32 + lane;
        int stage = 0;
        uint32_t phase = 0;
        uint32_t sum = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            ptx::mbar_wait(full_bar(stage), phase);
            const uint8_t* rowp = smem + Cfg::A_OFF + stage * A_STAGE + r * kKBlock;
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
        ownrs[r] = (int32_t)sum;  // partial over this rank's K-slice
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(rsready);
    } else if (warp >= 4 && warp < 8) {
        const int ew = warp - 4;
        const int r = ew * 32 + lane;
        // stage the owned columns' epilogue records while the mainloop runs
        if (MODE != 0 && r < OWN) {
            const int4 r4 = __ldg(reinterpret_cast<const int4*>(p.rec + n0 + (int)rank * OWN + r));
            reinterpret_cast<int4*>(smem + Cfg::REC_OFF)[r] = r4;
        }
        ptx::mbar_wait(tfull, 0);  // mainloop done: the A stages are free for staging
        ptx::tc_fence_after();
        if (warp == 4 && lane == 0) sk_stamp(p, 5);
        int32_t my_rs = 0;
        if (RS) {
            ptx::mbar_wait(rsready, 0);
            my_rs = ownrs[r];
        }
        // ---- stage the partial columns each peer owns: send slot qi for peer
        // q = rank + 1 + qi (mod S), layout [quad][row] int4 then [row] row sum
#pragma unroll 1
        for (int qi = 0; qi < S - 1; ++qi) {
            const int q = ((int)rank + 1 + qi) % S;
            uint8_t* slot = smem + Cfg::A_OFF + qi * Cfg::SLOT_BYTES;
#pragma unroll
            for (int h = 0; h < OWN / 16; ++h) {
                uint32_t v[16];
                ptx::tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(q * OWN + h * 16), v);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; j += 4) {
                    const int c4 = h * 4 + j / 4;
                    *reinterpret_cast<uint4*>(slot + ((size_t)c4 * BM + r) * 16) =
                        make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                }
            }
            reinterpret_cast<int32_t*>(slot + Cfg::SLOT_PART)[r] = my_rs;
        }
        // generic-proxy smem writes -> visible to the bulk-copy (async) proxy
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 4) {
            cluster_wait_acquire();  // every peer has armed its recvfull barrier
            if (lane == 0) {
#pragma unroll 1
                for (int qi = 0; qi < S - 1; ++qi) {
                    const int q = ((int)rank + 1 + qi) % S;
                    // at owner q, the slot of source rank s is (s - q + S) % S - 1
                    const int dslot = ((int)rank - q + S) % S - 1;
                    bulk_s2cluster(mapa(base + Cfg::RECV_OFF + dslot * Cfg::SLOT_BYTES, q),
                                   base + Cfg::A_OFF + qi * Cfg::SLOT_BYTES, Cfg::SLOT_BYTES, mapa(recvfull, q));
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            __syncwarp();
        }
        // ---- reduce the owned columns: own partial + S-1 received partials
        ptx::mbar_wait(recvfull, 0);
        if (warp == 4 && lane == 0) sk_stamp(p, 6);
        const int row = m0 + r;
        int32_t rowsum = my_rs;
        const uint8_t* recv = smem + Cfg::RECV_OFF;
        if (RS) {
#pragma unroll
            for (int sl = 0; sl < S - 1; ++sl)
                rowsum += reinterpret_cast<const int32_t*>(recv + sl * Cfg::SLOT_BYTES + Cfg::SLOT_PART)[r];
        }
#pragma unroll
        for (int h = 0; h < OWN / 16; ++h) {
            uint32_t v[16];
            ptx::tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(rank * OWN + h * 16), v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int sl = 0; sl < S - 1; ++sl) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint4 x =
                        *reinterpret_cast<const uint4*>(recv + sl * Cfg::SLOT_BYTES + ((size_t)(h * 4 + j) * BM + r) * 16);
                    v[4 * j + 0] += x.x;
                    v[4 * j + 1] += x.y;
                    v[4 * j + 2] += x.z;
                    v[4 * j + 3] += x.w;
                }
            }
            const int col0 = n0 + (int)rank * OWN + h * 16;
            if (row >= p.rows || col0 >= p.n) continue;
            if (MODE == 0) {
                int32_t* dst = reinterpret_cast<int32_t*>(p.c) + (size_t)row * p.ldc + col0;
                int32_t out[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    int32_t x = (int32_t)v[j];
                    if (p.bias_add && col0 + j < p.n)
                        x = (int32_t)((uint32_t)x + (uint32_t)__ldg(p.bias_add + col0 + j));
                    out[j] = x;
                }
                const bool vec = (col0 + 16 <= p.n) && ((p.ldc & 3) == 0) &&
                                 ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
                if (vec) {
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        *reinterpret_cast<int4*>(dst + j) = make_int4(out[j], out[j + 1], out[j + 2], out[j + 3]);
                } else {
                    for (int j = 0; j < 16; ++j)
                        if (col0 + j < p.n) dst[j] = out[j];
                }
            } else {
                uint32_t packed[4];
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    uint32_t word = 0;
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int j = w * 4 + b;
                        const int4 r4 = recs[h * 16 + j];
                        EpiRecord rc;
                        rc.c = r4.x;
                        rc.zpb = r4.y;
                        const int32_t adj = adjust((int32_t)v[j], rowsum, rc);
                        const uint32_t q = MODE == 1 ? requant_f32(adj, __int_as_float(r4.z), p.zp_c, p.relu)
                                                     : requant_ref(adj, __hiloint2double(r4.w, r4.z), p.zp_c, p.relu);
                        word |= q << (8 * b);
                    }
                    packed[w] = word;
                }
                uint8_t* dst = reinterpret_cast<uint8_t*>(p.c) + (size_t)row * p.ldc + col0;
                const bool vec = (col0 + 16 <= p.n) && ((p.ldc & 15) == 0) &&
                                 ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
                if (vec) {
                    *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
                } else {
                    for (int j = 0; j < 16; ++j)
                        if (col0 + j < p.n) dst[j] = (uint8_t)(packed[j / 4] >> (8 * (j % 4)));
                }
            }
        }
        if (warp == 4) {
            // the staged source smem must stay valid until the copies have read it
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
        }
        if (warp == 4 && lane == 0) sk_stamp(p, 7);
    }

    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
}

template <int BN, int S, int STAGES, int MODE, bool RS>
cudaError_t launch_sk(const GemmArgs& g, cudaStream_t s) {
    using Cfg = SkCfg<BN, S, STAGES>;
    auto kern = gemm_splitk_kernel<BN, S, STAGES, MODE, RS>;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    CUtensorMap tmap;
    if (!make_tmap_a_cached(&tmap, g.a, g.rows, g.k, g.lda, BM)) return cudaErrorInvalidValue;
    SkParams p;
    p.pb = g.pb->data;
    p.np = g.pb->np;
    p.nkb = g.pb->kp / kKBlock;
    p.n = g.pb->n;
    p.rows = g.rows;
    p.num_n_tiles = g.pb->np / BN;
    p.rec = g.ep ? g.ep->rec : nullptr;
    p.zp_c = g.ep ? g.ep->zp_c : 0;
    p.relu = g.ep ? g.ep->relu : 0;
    p.bias_add = g.bias_add;
    p.c = g.c;
    p.ldc = g.ldc;
    p.trace = tc_trace_buffer_ptr();
    const int tiles = ceil_div_i(g.rows, BM) * p.num_n_tiles;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tiles * S);
    cfg.blockDim = dim3(RS ? 384 : 256);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmap, p);
    count_launch(kFamGemmTcSmallM);
    return e;
}

template <int BN, int S, int STAGES>
cudaError_t launch_sk_modes(const GemmArgs& g, cudaStream_t s) {
    if (g.raw) return launch_sk<BN, S, STAGES, 0, false>(g, s);
    const bool rs = g.ep->need_rowsum;
    if (g.ep->rounding == Q8G_ROUND_F32_RNE)
        return rs ? launch_sk<BN, S, STAGES, 1, true>(g, s) : launch_sk<BN, S, STAGES, 1, false>(g, s);
    return rs ? launch_sk<BN, S, STAGES, 2, true>(g, s) : launch_sk<BN, S, STAGES, 2, false>(g, s);
}

}  // namespace

// split-K applies when every rank gets at least one k-block
bool splitk_supported(const GemmArgs& g) { return g.pb->kp / kKBlock >= 4; }

cudaError_t launch_gemm_splitk(const GemmArgs& g, cudaStream_t s) { return launch_sk_modes<128, 4, 5>(g, s); }

}  // namespace q8g
