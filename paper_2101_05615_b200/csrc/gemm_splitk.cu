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
// BN-wide tile.  After its mainloop each rank writes the partial columns the
// other ranks own (plus its partial row sums) from TMEM to an L2-resident
// workspace, the cluster passes one release/acquire barrier, and each owner
// reads its S-1 slots back from L2 (all loads in flight at once).  Eight
// warps share the exchange and the epilogue (the producer / MMA / idle warps
// join once the mainloop is done).  An SM-to-SM (DSMEM) exchange measured
// ~25 GB/s per SM: 1.9-2 us for the 48 KB per CTA, register stores and bulk
// smem->peer-smem copies alike, plus a wait for the outgoing copies.
//
// Same drop-in semantics as gemm_tc.cu (engine.hpp:59-169 + Requantize,
// pipeline.hpp:157-210); int32 addition is associative so the split is
// bit-exact.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "ptx.cuh"
#include "q8g_internal.cuh"
#include "requant.cuh"

namespace q8g {

bool make_tmap_a_cached(CUtensorMap* out, const uint8_t* a, int rows, int k, int lda, int box_rows);
unsigned long long* tc_trace_buffer_ptr();

namespace {

constexpr int BM = 128;
constexpr int A_STAGE = BM * kKBlock;

// AST A stages, BST B stages (separate rings; the first min(BST, k-blocks)
// stages of B are requested at kernel entry, ahead of griddepcontrol.wait)
template <int BN, int S, int AST, int BST>
struct SkCfg {
    static constexpr int OWN = BN / S;  // columns owned per rank
    static constexpr int B_STAGE = BN * kKBlock;
    static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;  // one accumulator tile
    // one exchange slot: partials [OWN/8 octs][BM rows] 32 B (256-bit accesses), then [BM] row sums
    static constexpr int SLOT_PART = (OWN / 4) * BM * 16;
    static constexpr int SLOT_BYTES = SLOT_PART + BM * 4;
    static constexpr int A_OFF = 0;
    static constexpr int B_OFF = AST * A_STAGE;
    static constexpr int OWNRS_OFF = B_OFF + BST * B_STAGE;
    static constexpr int REC_OFF = OWNRS_OFF + BM * 4;  // [OWN] EpiRecord
    static constexpr int BAR_OFF = REC_OFF + OWN * 16;
    static constexpr int NUM_BARS = 3 * AST + 2 * BST + 2;  // a_full, a_empty, rsdone, b_full, b_empty, tfull, rsready
    static constexpr int TMEMPTR_OFF = BAR_OFF + NUM_BARS * 8;
    static constexpr int SMEM_BYTES = TMEMPTR_OFF + 16 + 1024;
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
    int fast;  // F32_RNE fast requant allowed (q8g_epilogue::fast_f32)
    const int32_t* bias_add;
    void* c;
    int ldc;
    // L2 exchange workspace [tile][owner][S-1 slots] of SLOT_BYTES; null =
    // push the slots into the owners' smem (DSMEM)
    uint8_t* ws;
    size_t ws_bytes;  // its size (checked builds assert every slot access is inside it)
    // host-view overlap: A lands by a concurrent copy that then writes a_epoch
    // to *a_ready (GemmArgs); null = A resident
    const uint32_t* a_ready;
    uint32_t a_epoch;
    unsigned long long* trace;  // debug stamps (Q8G_TC_TRACE), else null
    unsigned long long* trace_cta;  // per-CTA phase stamps: alternate halves on successive launches
};

// poll the A-ready flag (acquire), then order the TMA (async proxy) reads of A
// after it; trap instead of hanging if the copy never lands (~8 s)
__device__ __forceinline__ void wait_a_ready(const uint32_t* flag, uint32_t epoch) {
    for (long long i = 0;; ++i) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v == epoch) break;
        if (i > (1LL << 26)) __trap();
        __nanosleep(128);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// slots: 0 entry, 1 prologue, 2 first TMA, 3 first stage, 4 last MMA commit,
// 5 past the exchange's cluster barrier, 6 exchange stores issued, 7 done;
// per-k-block stamps of CTA 0
__device__ __forceinline__ void sk_stamp(const SkParams& p, int slot) {
#ifdef Q8G_TRACE
    if (p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace_cta[blockIdx.x * 8 + slot] = t;
    }
#endif
}
__device__ __forceinline__ void sk_kb(const SkParams& p, int which, int i) {
#ifdef Q8G_TRACE
    if (p.trace && blockIdx.x == 0 && i < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8192 + which * 64 + i] = t;
    }
#endif
}

__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// L2-only 32-byte (256-bit) global stores / loads (split-K exchange workspace): half the L2 requests of v4; measured ~2x the
// per-SM read bandwidth from L2 (tools/l2_bw.cu)
__device__ __forceinline__ void st_cg_v8(void* p, const uint32_t* v) {
    asm volatile("st.global.cg.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void ld_cg_v8(const void* p, uint32_t* v) {
    asm volatile("ld.global.cg.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p)
                 : "memory");
}
__device__ __forceinline__ int32_t ld_cg_s32(const void* p) {
    int32_t v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_cg_s32(void* p, int32_t v) {
    asm volatile("st.global.cg.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// d = {c[15:0], sat_u8(a), sat_u8(b)} (one I2IP)
__device__ __forceinline__ uint32_t pack_sat_u8(int32_t a, int32_t b, uint32_t c) {
    uint32_t d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}


// requant (MODE 1 / 2) or raw int32 (MODE 0) + store of one row's 16 owned
// columns [col0, col0 + 16) (row < rows, col0 < n checked by the caller)
template <int MODE>
__device__ __forceinline__ void sk_store16(const SkParams& p, const int4* rec16, uint32_t (&v)[16], int32_t rowsum,
                                           int row, int col0) {
    Q8G_CHECK(row >= 0 && row < p.rows && col0 >= 0 && col0 < p.n);
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
        return;
    }
    uint32_t packed[4];
    if (MODE == 1 && p.fast) {
        // F32_RNE, 0 <= zp_c <= 255, finite multipliers: magic-add
        // rounding + saturating pack (exact; see conv_tc.cu epi_f32_fast)
        const int32_t zoff = 0x4B400000 - p.zp_c;
        const float floor_x = p.relu ? 0.0f : -8388608.0f;
        const uint32_t nrowsum = 0u - (uint32_t)rowsum;  // once per row, not per value
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            int32_t rr[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int j = w * 4 + b;
                const int4 r4 = rec16[j];
                const int32_t adj = (int32_t)(v[j] + ((uint32_t)r4.x + (uint32_t)r4.y * nrowsum));
                float x = __fmul_rn(__int2float_rn(adj), __int_as_float(r4.z));
                x = fmaxf(x, floor_x);
                rr[b] = __float_as_int(__fadd_rn(x, 12582912.0f)) - zoff;
            }
            packed[w] = pack_sat_u8(rr[1], rr[0], pack_sat_u8(rr[3], rr[2], 0u));
        }
    } else {
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t word = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int j = w * 4 + b;
                const int4 r4 = rec16[j];
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

template <int BN, int S, int AST, int BST, int MODE, bool RS>
__global__ void __launch_bounds__(RS ? 384 : 256, 1)
    gemm_splitk_kernel(const __grid_constant__ CUtensorMap tmap_a, const SkParams p) {
    using Cfg = SkCfg<BN, S, AST, BST>;
    constexpr int OWN = Cfg::OWN;
    constexpr int NH = OWN / 16;  // 16-column chunks per owned block, split over 2 epilogue groups
    static_assert(OWN % 32 == 0, "owned column block must be a multiple of 32");
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_addr);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    Q8G_CHECK((uint32_t)Cfg::SMEM_BYTES <= ptx::dynamic_smem_size());
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
    auto afull_bar = [&](int s) { return bar0 + 8u * s; };
    auto aempty_bar = [&](int s) { return bar0 + 8u * (AST + s); };
    auto rsdone_bar = [&](int s) { return bar0 + 8u * (2 * AST + s); };
    auto bfull_bar = [&](int s) { return bar0 + 8u * (3 * AST + s); };
    auto bempty_bar = [&](int s) { return bar0 + 8u * (3 * AST + BST + s); };
    const uint32_t tfull = bar0 + 8u * (3 * AST + 2 * BST);
    const uint32_t rsready = tfull + 8u;
    int32_t* ownrs = reinterpret_cast<int32_t*>(smem + Cfg::OWNRS_OFF);
    const int4* recs = reinterpret_cast<const int4*>(smem + Cfg::REC_OFF);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + Cfg::TMEMPTR_OFF);

    // PDL: start streaming the first stages of B before anything else and
    // before waiting for the previous grid: the weights' DRAM latency (~2 us
    // under the full burst) is the head of the critical path.  Packed weights
    // are immutable once q8g_pack_b* returned (it synchronizes), so no kernel
    // in flight can be writing them; A may be the previous grid's output and
    // is only loaded after griddepcontrol.wait.
    const int nkl = kb1 - kb0;  // this rank's k-blocks
    // at most 4 stages before the PDL wait, the rest right after it: fewer
    // requests in the entry burst land the first stage sooner (C1: 7.9 vs
    // 8.25 us per step with all 6 up front; 3 or 5: 8.0-8.1)
    const int npre = nkl < (BST < 4 ? BST : 4) ? nkl : (BST < 4 ? BST : 4);
    const uint64_t pol_b = ptx::policy_evict_first();  // weights streamed once
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < BST; ++s) {
            ptx::mbar_init(bfull_bar(s), 1);
            ptx::mbar_init(bempty_bar(s), 1);
        }
        ptx::fence_mbar_init();
        for (int i = 0; i < npre; ++i) {
            ptx::mbar_arrive_expect_tx(bfull_bar(i), Cfg::B_STAGE);
            ptx::bulk_load_hint(sB + i * Cfg::B_STAGE, p.pb + ((size_t)(kb0 + i) * p.np + n0) * kKBlock,
                                Cfg::B_STAGE, bfull_bar(i), pol_b);
        }
        ptx::prefetch_tmap(&tmap_a);
        for (int s = 0; s < AST; ++s) {
            ptx::mbar_init(afull_bar(s), 1);
            ptx::mbar_init(aempty_bar(s), 1);
            ptx::mbar_init(rsdone_bar(s), 4);
        }
        ptx::mbar_init(tfull, 1);
        ptx::mbar_init(rsready, 4);
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<Cfg::TMEM_COLS>(ptx::smem_u32(tmem_ptr));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_ptr;
    ptx::griddep_wait();  // PDL: the prologue above overlapped the previous grid
    if (threadIdx.x == 0) sk_stamp(p, 1);

    if (warp == 0) {
        // whole warp runs the loop; one elected lane issues (ptx::elect_one)
        if (p.a_ready) {
            if (ptx::elect_one()) wait_a_ready(p.a_ready, p.a_epoch);
            __syncwarp();
        }
        for (int j = 0; j < nkl; ++j) {
            const int kb = kb0 + j;
            const int sa = j % AST, sb = j % BST;
            ptx::mbar_wait(aempty_bar(sa), ((uint32_t)(j / AST) & 1u) ^ 1u);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(afull_bar(sa), A_STAGE);
                ptx::tma_load_2d(sA + sa * A_STAGE, &tmap_a, kb * kKBlock, m0, afull_bar(sa));
                if (kb == kb0) sk_stamp(p, 2);
                sk_kb(p, 0, j);
            }
            __syncwarp();
            if (j >= npre) {  // stages not requested at entry: fresh slots first, then reused ones
                ptx::mbar_wait(bempty_bar(sb), ((uint32_t)(j / BST) & 1u) ^ 1u);
                if (ptx::elect_one()) {
                    ptx::mbar_arrive_expect_tx(bfull_bar(sb), Cfg::B_STAGE);
                    ptx::bulk_load_hint(sB + sb * Cfg::B_STAGE, p.pb + ((size_t)kb * p.np + n0) * kKBlock,
                                        Cfg::B_STAGE, bfull_bar(sb), pol_b);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = ptx::idesc_u8s8_s32<BM, BN>();
        for (int j = 0; j < nkl; ++j) {
            const int sa = j % AST, sb = j % BST;
            const uint32_t pa = (uint32_t)(j / AST) & 1u;
            ptx::mbar_wait(afull_bar(sa), pa);
            ptx::mbar_wait(bfull_bar(sb), (uint32_t)(j / BST) & 1u);
            ptx::tc_fence_after();
            const uint64_t adesc = ptx::sw128_kmajor_desc(sA + sa * A_STAGE);
            const uint64_t bdesc = ptx::sw128_kmajor_desc(sB + sb * Cfg::B_STAGE);
            if (ptx::elect_one()) {
                if (j == 0) sk_stamp(p, 3);
                sk_kb(p, 1, j);
#pragma unroll
                for (int ks = 0; ks < kKBlock / 32; ++ks)
                    ptx::mma_i8(tmem_base, adesc + 2 * ks, bdesc + 2 * ks, idesc, (j > 0 || ks > 0) ? 1u : 0u);
            }
            __syncwarp();
            if (RS) ptx::mbar_wait(rsdone_bar(sa), pa);
            if (ptx::elect_one()) {  // same lane as the MMAs
                ptx::tc_commit(aempty_bar(sa));
                ptx::tc_commit(bempty_bar(sb));
            }
            __syncwarp();
        }
        if (ptx::elect_one()) {
            ptx::tc_commit(tfull);
            sk_stamp(p, 4);
        }
        __syncwarp();
    } else if (RS && warp >= 8) {
        const int r = (warp - 8) * 32 + lane;
        uint32_t sum = 0;
        for (int j = 0; j < nkl; ++j) {
            const int sa = j % AST;
            ptx::mbar_wait(afull_bar(sa), (uint32_t)(j / AST) & 1u);
            const uint8_t* rowp = smem + Cfg::A_OFF + sa * A_STAGE + r * kKBlock;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint4 w = *reinterpret_cast<const uint4*>(rowp + ((q + r) & 7) * 16);
                sum = ptx::dp4a_uu(w.x, 0x01010101u, sum);
                sum = ptx::dp4a_uu(w.y, 0x01010101u, sum);
                sum = ptx::dp4a_uu(w.z, 0x01010101u, sum);
                sum = ptx::dp4a_uu(w.w, 0x01010101u, sum);
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(rsdone_bar(sa));
        }
        ownrs[r] = (int32_t)sum;  // partial over this rank's K-slice
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(rsready);
    }
    if (warp < 8) {
        // ------------------------------------------------ exchange + epilogue
        // two groups of 4 warps: warps 4-7 (g 0) and, once their roles are
        // done, warps 0-3 (g 1); a warp reads TMEM lanes 32*(warp%4).., each
        // group takes every other 16-column chunk of a block
        const int g = warp < 4 ? 1 : 0;
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;  // tile row
        const uint32_t lane_base = tmem_base + ((uint32_t)(q4 * 32) << 16);
        // stage the owned columns' epilogue records while the mainloop runs
        if (g == 0 && MODE != 0 && r < OWN) {
            const int4 r4 = __ldg(reinterpret_cast<const int4*>(p.rec + n0 + (int)rank * OWN + r));
            reinterpret_cast<int4*>(smem + Cfg::REC_OFF)[r] = r4;
        }
        ptx::mbar_wait(tfull, 0);
        ptx::tc_fence_after();
        int32_t my_rs = 0;
        if (RS) {
            ptx::mbar_wait(rsready, 0);
            my_rs = ownrs[r];
        }
        // ---- write the partial columns each peer owns (and the partial row
        // sums) from TMEM to the L2 workspace, coalesced [oct][row] 32 B.
        // (Staging in the drained A stages + bulk shared->global copies
        // measured slower here: 8.75 vs 8.25 us per C1 step.)
#pragma unroll 1
        for (int qi = 0; qi < S - 1; ++qi) {
            const int q = ((int)rank + 1 + qi) % S;
            const int dslot = ((int)rank - q + S) % S - 1;  // at owner q: slot of this source
            uint8_t* slot = p.ws + ((size_t)(tile * S + q) * (S - 1) + dslot) * Cfg::SLOT_BYTES;
            Q8G_CHECK(dslot >= 0 && dslot < S - 1 && slot + Cfg::SLOT_BYTES <= p.ws + p.ws_bytes);
#pragma unroll
            for (int h = g; h < NH; h += 2) {
                uint32_t v[16];
                ptx::tmem_ld_32x32b_x16(lane_base + (uint32_t)(q * OWN + h * 16), v);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int t = 0; t < 2; ++t) st_cg_v8(slot + ((size_t)(h * 2 + t) * BM + r) * 32, v + 8 * t);
            }
            if (g == 0 && RS) st_cg_s32(slot + Cfg::SLOT_PART + r * 4, my_rs);
        }
        // group 0's staged records -> group 1; then one release/acquire
        // cluster barrier orders every rank's workspace writes before the reads
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (warp == 4 && lane == 0) sk_stamp(p, 6);
        cluster_arrive_release();
        cluster_wait_acquire();
        if (warp == 4 && lane == 0) sk_stamp(p, 5);
        // ---- reduce the owned columns: own partial + the S-1 received slots,
        // all loads in flight at once (one L2 round trip)
        const uint8_t* recv = p.ws + (size_t)(tile * S + (int)rank) * (S - 1) * Cfg::SLOT_BYTES;
        Q8G_CHECK(recv + (S - 1) * Cfg::SLOT_BYTES <= p.ws + p.ws_bytes);
        const int row = m0 + r;
        int32_t rowsum = my_rs;
        if (RS) {
#pragma unroll
            for (int sl = 0; sl < S - 1; ++sl) rowsum += ld_cg_s32(recv + sl * Cfg::SLOT_BYTES + Cfg::SLOT_PART + r * 4);
        }
        uint32_t rx[NH / 2][S - 1][16];
#pragma unroll
        for (int hh = 0; hh < NH / 2; ++hh)
#pragma unroll
            for (int sl = 0; sl < S - 1; ++sl)
#pragma unroll
                for (int t = 0; t < 2; ++t)
                    ld_cg_v8(recv + sl * Cfg::SLOT_BYTES + ((size_t)((g + 2 * hh) * 2 + t) * BM + r) * 32,
                             rx[hh][sl] + 8 * t);
#pragma unroll
        for (int hh = 0; hh < NH / 2; ++hh) {
            const int h = g + 2 * hh;
            uint32_t v[16];
            ptx::tmem_ld_32x32b_x16(lane_base + (uint32_t)(rank * OWN + h * 16), v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int sl = 0; sl < S - 1; ++sl)
#pragma unroll
                for (int j = 0; j < 16; ++j) v[j] += rx[hh][sl][j];
            const int col0 = n0 + (int)rank * OWN + h * 16;
            if (row >= p.rows || col0 >= p.n) continue;
            sk_store16<MODE>(p, recs + h * 16, v, rowsum, row, col0);
        }
        if (warp == 4 && lane == 0) sk_stamp(p, 7);
    } else {
        // row-sum warps: their arrival in the cluster barrier's one phase
        __syncwarp();
        cluster_arrive_release();
    }

    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
}

// split-K exchange workspace, one per (device, stream) so concurrent streams
// never share it; grow-only and never freed (captured graphs keep the
// pointer).  Null on allocation failure or when a capture is in progress and
// no large-enough workspace exists yet (the caller then uses the non-split
// kernel).
uint8_t* splitk_workspace(int dev, cudaStream_t s, size_t bytes) {
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

template <int BN, int S, int AST, int BST, int MODE, bool RS>
cudaError_t launch_sk(const GemmArgs& g, cudaStream_t s) {
    using Cfg = SkCfg<BN, S, AST, BST>;
    auto kern = gemm_splitk_kernel<BN, S, AST, BST, MODE, RS>;
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
    p.fast = (g.ep && g.ep->fast_f32) ? 1 : 0;
    p.a_ready = g.a_ready;
    p.a_epoch = g.a_epoch;
    p.bias_add = g.bias_add;
    p.c = g.c;
    p.ldc = g.ldc;
    p.trace = tc_trace_buffer_ptr();
    const int tiles = ceil_div_i(g.rows, BM) * p.num_n_tiles;
    p.trace_cta = p.trace;
    if (p.trace && (tiles * S) <= 512) {  // two successive launches side by side
        static int parity = 0;
        p.trace_cta = p.trace + (parity ^= 1) * 4096;
    }
    p.ws_bytes = (size_t)tiles * S * (S - 1) * Cfg::SLOT_BYTES;
    p.ws = splitk_workspace(dev, s, p.ws_bytes);
    if (!p.ws) return cudaErrorNotSupported;  // caller falls back to the non-split kernel
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

template <int BN, int S, int AST, int BST>
cudaError_t launch_sk_modes(const GemmArgs& g, cudaStream_t s) {
    if (g.raw) return launch_sk<BN, S, AST, BST, 0, false>(g, s);
    const bool rs = g.ep->need_rowsum;
    if (g.ep->rounding == Q8G_ROUND_F32_RNE)
        return rs ? launch_sk<BN, S, AST, BST, 1, true>(g, s) : launch_sk<BN, S, AST, BST, 1, false>(g, s);
    return rs ? launch_sk<BN, S, AST, BST, 2, true>(g, s) : launch_sk<BN, S, AST, BST, 2, false>(g, s);
}

}  // namespace

// split-K applies when every rank gets at least one k-block
bool splitk_supported(const GemmArgs& g) { return g.pb->kp / kKBlock >= 4; }

cudaError_t launch_gemm_splitk(const GemmArgs& g, cudaStream_t s) {
    // default: BN 128, 4-way split, 6 A + 6 B stages.  Tuning knob Q8G_SK_CFG:
    // "64x2" (BN 64, 2-way split) or "b8" (4 A + 8 B stages: a rank's whole B
    // slice at K = 4096 requested at entry) -- both measured slower in the
    // bench (8.66 / 8.97 vs 8.49 us: with all of B in flight each rank's first
    // stage lands later, and the weights still stream at ~4 TB/s)
    static const int cfg = [] {
        const char* e = getenv("Q8G_SK_CFG");
        if (e && std::strcmp(e, "64x2") == 0) return 1;
        if (e && std::strcmp(e, "b8") == 0) return 2;
        if (e && std::strcmp(e, "b8a5") == 0) return 3;
        return 0;
    }();
    if (cfg == 1) return launch_sk_modes<64, 2, 4, 16>(g, s);
    if (cfg == 2) return launch_sk_modes<128, 4, 4, 8>(g, s);
    if (cfg == 3) return launch_sk_modes<128, 4, 5, 8>(g, s);
    return launch_sk_modes<128, 4, 6, 6>(g, s);
}

}  // namespace q8g
