// gemm_tc2w.cu — large-M GEMM on CTA pairs with 256 x 512 pair tiles
// (tcgen05.mma.cta_group::2, two N=256 MMAs per K step sharing A): the
// BASELINE C2 kernel (M=16384, N=K=4096).
//
// Why a 512-column tile (round 1 had 256 x 256 pair tiles, gemm_tc2.cu,
// removed in round 2): every byte a CTA pulls from
// L2 into shared memory costs crossbar / die-to-die energy, and C2 runs at
// the 1 kW power limit (in-kernel clock64 / globaltimer: ~1.5 GHz, not 1.965,
// tools/c2_clock.py).  Per 128-byte K block a CTA now receives A 16 KB + B
// 32 KB for 128 x 512 x 128 MACs: 48 B/clk per SM at full MMA rate instead of
// 64, and its shared memory carries 48 KB of TMA writes + 64 KB of MMA reads
// per 1024 MMA cycles (109 B/clk of the ~128 B/clk port) instead of 128.
//
// Same drop-in semantics as gemm_tc.cu: engine.hpp:59-169 for
// the contraction, pipeline.hpp:157-210 + quant.hpp:115-133 for the fused
// requantizing back-end (epilogue.cuh).
//
// Per CTA of the pair (rank 0 = leader; each CTA owns 128 rows of the pair's
// 256 and 128 of each 256-column sub-tile's B columns):
//   warp 0      producer: A (TMA, SWIZZLE_128B) and the two B halves (TMA over
//               the pre-swizzled packed weight) with the cta_group::2 form:
//               every load of BOTH CTAs completes its bytes on the LEADER's
//               full barrier, so the leader's MMA waits on exactly the data it
//               reads (no follower relay)
//   warp 1      leader: MMA issuer, per stage 2 sub-tiles x 4 x M256 N256 K32;
//               commits multicast to both CTAs' empty / tfull barriers
//   warps 2-3   row sums of this CTA's 128 A rows (only when some zp_b != 0,
//               only on the first tile of a run of tiles with the same rows):
//               read each landed stage after the MMA has consumed it (its
//               empty barrier) and hold the producer off that stage until
//               they are done (rsdone)
//   warps 4-11  epilogue: warp w drains lane quarter w%4, column group
//               (w-4)/4 of each 256-column accumulator half into 128
//               registers, releases the half to the MMA at once (tempty),
//               then requantizes and stores from registers
//
// TMEM holds one 128 x 512 accumulator per CTA (all 512 columns), tracked as
// two 256-column halves: the next tile's first MMAs into half h wait only for
// half h's drain, which overlaps the previous tile's last MMAs into the other
// half.
//
// Tile schedule: pair tiles in m-major order dealt round-robin over the pairs
// (sched 0, default): at any moment the pairs work on ~9 adjacent 256-row
// blocks of A, so A comes from DRAM once and is shared through L2, and every
// tile computes its own row sums.  Sched 1 (Q8G_TC2W_SCHED=1) gives each pair
// a contiguous range, so consecutive tiles share their A rows and the row
// sums are computed once per run -- but the pairs then stream all of A at
// once and re-read each block from DRAM: C2 187 us at 1.47 GHz vs 175 us at
// 1.57 GHz for sched 0 (the kernel runs at the 1 kW power limit, where DRAM
// traffic costs clock).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "epilogue.cuh"
#include "ptx.cuh"
#include "q8g_internal.cuh"

namespace q8g {

bool make_tmap_a_cached(CUtensorMap* out, const uint8_t* a, int rows, int k, int lda, int box_rows);
unsigned long long* tc_trace_buffer_ptr();
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();

namespace {

constexpr int BM = 128;                          // rows per CTA (256 per pair)
constexpr int HN = 128;                          // B columns per CTA per sub-tile
constexpr int NSUB = 2;                          // N=256 sub-tiles per pair tile
constexpr int PN = NSUB * 2 * HN;                // 512 pair-tile columns
constexpr int STAGE_A = BM * kKBlock;            // 16 KB
constexpr int STAGE_B = HN * kKBlock;            // 16 KB per sub-tile
constexpr int STAGE = STAGE_A + NSUB * STAGE_B;  // 48 KB
constexpr int STAGES = 4;
constexpr int THREADS = 384;

struct Cfg {
    // u8 output staging for the TMA store: per epilogue warp 32 rows x 64 B
    // (SWIZZLE_64B), 2 KB each
    static constexpr int OUT_OFF = STAGES * STAGE;
    static constexpr int OUT_WARP = 32 * 64;
    static constexpr int BAR_OFF = OUT_OFF + 8 * OUT_WARP;
    // full[S], empty[S], rsdone[S], tfull[2], tempty[2], rfull[2], rempty[2]
    static constexpr int NUM_BARS = 4 * STAGES + 8;  // + aread[S] (row-sum warps: the stage's A was read)
    static constexpr int RS_OFF = BAR_OFF + NUM_BARS * 8;
    static constexpr int REC_OFF = RS_OFF + 2 * BM * 4;  // the tile's column records, SoA: c, zp_b, mult lo, hi
    static constexpr int TMEMPTR_OFF = REC_OFF + 4 * PN * 4;
    static constexpr int SMEM_BYTES = TMEMPTR_OFF + 16 + 1024;
    static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

// TMA store maps of the peer destinations (N-sharded multi-GPU: every tile
// the epilogue stores locally also goes straight to each peer's C over
// NVLink, from the same staging tile)
struct PeerMaps {
    CUtensorMap m[kMaxPeers];
};

struct Tc2wParams {
    const uint8_t* a;  // not read by the kernel (TMA maps only); kept for traces
    int nkb, n, rows;
    int num_m_tiles, num_n_tiles;  // pair tiles: 256 rows x 512 columns (the last may hang past np)
    int np;                        // packed-B columns (a multiple of 256)
    int b3d;                       // np % 512 != 0: B through the 3-D map (zero columns past np)
    int sched;                     // 1: contiguous ranges per pair, 0: round-robin
    int skew_end, skew_start;      // MMA issue-order skew at tile boundaries (k blocks)
    int tma_out;                   // u8 output through smem staging + TMA stores (tmap_c valid)
    int n_peers;                   // MODE 3: peer destinations in PeerMaps (0: local only)
    EpiArgs ea;
    unsigned long long* trace;
};

// tiles of pair `group` of `groups`: [first, last) stepping by step
struct TileRange {
    int first, last, step;
};
__device__ __forceinline__ TileRange tile_range(const Tc2wParams& p, int group, int groups) {
    const int total = p.num_m_tiles * p.num_n_tiles;
    if (p.sched == 1) {
        const int f = (int)(((long long)group * total) / groups);
        const int l = (int)(((long long)(group + 1) * total) / groups);
        return {f, l, 1};
    }
    return {group, total, groups};
}

// CTA 0's SM clock64 and globaltimer at entry / exit of the most recent
// launch (always recorded: two 16-byte stores per launch), read back by
// q8g_debug_kernel_clock: the SM clock the launch actually ran at (NVML
// reports the clock target, not the power-limited effective clock)
__device__ unsigned long long g_tc2w_clock[4];

__device__ __forceinline__ void tw_clk(const Tc2wParams& p, int end) {
    if (blockIdx.x == 0) {
        unsigned long long t, c;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
        g_tc2w_clock[end] = c;
        g_tc2w_clock[2 + end] = t;
#ifdef Q8G_TRACE
        if (p.trace) {
            p.trace[10200 + end] = c;
            p.trace[10202 + end] = t;
        }
#endif
    }
}
// CTA 0, per tile ti < 16: [9216 + 8 * ti + k] (tools/tc2w_tiles.py): MMA
// issuer 0 past tempty[0], 1 past tempty[1], 2 / 3 tfull[0] / tfull[1]
// committed; epilogue warp 4: 4 / 6 tfull[0] / tfull[1] seen, 5 / 7 half 0 / 1
// drained into registers
__device__ __forceinline__ void tw_tile(const Tc2wParams& p, int k, int ti) {
#ifdef Q8G_TRACE
    if (p.trace && blockIdx.x == 0 && ti < 16) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[9216 + 8 * ti + k] = t;
    }
#endif
}

// CTA 0 epilogue warp 4, per tile ti < 16: [9472 + 8 * ti + k], k = 6 + h:
// half h's row sums in hand, 3h + 0: half h round 0 requantized, 3h + 1: round 1 staging tile free, 3h + 2:
// round 1 requantized (tools/tc2w_tiles.py)
__device__ __forceinline__ void tw_epi(const Tc2wParams& p, int k, int ti) {
#ifdef Q8G_TRACE
    if (p.trace && blockIdx.x == 0 && ti < 16) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[9472 + 8 * ti + k] = t;
    }
#endif
}

__device__ __forceinline__ void tma_load_2d_pair_hint(uint32_t dst, const CUtensorMap* m, int c0, int c1,
                                                      uint32_t bar_cluster, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(policy)
        : "memory");
}

// packed B through a 3-D map (128 K-bytes, np columns, kp/128 k-blocks): a box
// of columns past np is zero-filled, so a last 512-column tile over an np that
// is an odd multiple of 256 reads zeros for its second half
__device__ __forceinline__ void tma_load_3d_pair_hint(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2,
                                                      uint32_t bar_cluster, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

__device__ __forceinline__ uint64_t f32x2_mul(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t f32x2_add(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
    return (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32);
}

// 16 accumulator columns of one row -> 16 u8, F32_RNE fast path (the
// arithmetic of epilogue.cuh requant4_f32_fast, records from shared memory):
// adj = v + c + zp_b*(-rowsum) (wrapping int32; -rowsum once per row, not a
// negation per value), x = RN(float(adj) * mult)
// (paired RN multiplies), floor, magic add, saturating pack
__device__ __forceinline__ uint4 requant16_fast(const uint32_t* v, const int32_t* rc, const int32_t* rz,
                                                const float* rm, uint32_t nrowsum, int32_t zoff, float floor_x) {
    uint32_t words[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
#ifdef Q8G_EXP_NOREC
        const int4 C = make_int4(w, w + 1, w + 2, w + 3);
        const int4 Z = make_int4(1, 2, 3, 4);
        const float4 M = make_float4(1e-4f, 2e-4f, 3e-4f, 4e-4f);
#else
        const int4 C = *reinterpret_cast<const int4*>(rc + 4 * w);
        const int4 Z = *reinterpret_cast<const int4*>(rz + 4 * w);
        const float4 M = *reinterpret_cast<const float4*>(rm + 4 * w);
#endif
        const int32_t a0 = (int32_t)(v[4 * w + 0] + ((uint32_t)C.x + (uint32_t)Z.x * nrowsum));
        const int32_t a1 = (int32_t)(v[4 * w + 1] + ((uint32_t)C.y + (uint32_t)Z.y * nrowsum));
        const int32_t a2 = (int32_t)(v[4 * w + 2] + ((uint32_t)C.z + (uint32_t)Z.z * nrowsum));
        const int32_t a3 = (int32_t)(v[4 * w + 3] + ((uint32_t)C.w + (uint32_t)Z.w * nrowsum));
        uint64_t x01 = f32x2_mul(pack2(__int2float_rn(a0), __int2float_rn(a1)), pack2(M.x, M.y));
        uint64_t x23 = f32x2_mul(pack2(__int2float_rn(a2), __int2float_rn(a3)), pack2(M.z, M.w));
        // the floor sits between the multiply and the magic add, so the two
        // paired RN operations can never be contracted into one FMA
        const float x0 = fmaxf(__uint_as_float((uint32_t)x01), floor_x);
        const float x1 = fmaxf(__uint_as_float((uint32_t)(x01 >> 32)), floor_x);
        const float x2 = fmaxf(__uint_as_float((uint32_t)x23), floor_x);
        const float x3 = fmaxf(__uint_as_float((uint32_t)(x23 >> 32)), floor_x);
        const uint64_t magic = pack2(12582912.0f, 12582912.0f);
        const uint64_t y01 = f32x2_add(pack2(x0, x1), magic);
        const uint64_t y23 = f32x2_add(pack2(x2, x3), magic);
        const int32_t r0 = (int32_t)(uint32_t)y01 - zoff, r1 = (int32_t)(uint32_t)(y01 >> 32) - zoff;
        const int32_t r2 = (int32_t)(uint32_t)y23 - zoff, r3 = (int32_t)(uint32_t)(y23 >> 32) - zoff;
        words[w] = pack_sat_u8(r1, r0, pack_sat_u8(r3, r2, 0u));
    }
    return make_uint4(words[0], words[1], words[2], words[3]);
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(c0), "r"(c1), "r"(src)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// MODE: 0 raw int32, 1 F32_RNE, 2 REF (epilogue.cuh store_chunk16), 3 F32_RNE
// fast path (fast_f32 epilogue, 16-byte aligned u8 output): records staged in
// shared memory, paired fp32 arithmetic, TMA stores
template <int MODE, bool RS>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tc2w_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                     const __grid_constant__ CUtensorMap tmap_c, const __grid_constant__ PeerMaps peers,
                     const Tc2wParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_addr);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    Q8G_CHECK((uint32_t)Cfg::SMEM_BYTES <= ptx::dynamic_smem_size());
    Q8G_CHECK(p.n_peers >= 0 && p.n_peers <= kMaxPeers);
    ptx::griddep_launch_dependents();
    if (threadIdx.x == 0) tw_clk(p, 0);
    const uint32_t rank = ptx::cluster_ctarank();  // 0 leader, 1 follower
    const bool leader = rank == 0;

    const uint32_t bar0 = base + Cfg::BAR_OFF;
    auto stage_a = [&](int s) { return base + (uint32_t)(s * STAGE); };
    auto stage_b = [&](int s, int h) { return base + (uint32_t)(s * STAGE + STAGE_A + h * STAGE_B); };
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
    auto rsdone_bar = [&](int s) { return bar0 + 8u * (2 * STAGES + s); };
    // committed (multicast) after a stage's half-0 MMAs: its A has landed and
    // stays until the stage's empty barrier -- the row-sum warps read from
    // here, ahead of the half-1 MMAs (the tile-end skew puts two K blocks of
    // half-1 MMAs after the last half-0 MMA)
    auto aread_bar = [&](int s) { return bar0 + 8u * (3 * STAGES + 8 + s); };
    auto tfull_bar = [&](int h) { return bar0 + 8u * (3 * STAGES + h); };
    auto tempty_bar = [&](int h) { return bar0 + 8u * (3 * STAGES + 2 + h); };
    auto rfull_bar = [&](int b) { return bar0 + 8u * (3 * STAGES + 4 + b); };
    auto rempty_bar = [&](int b) { return bar0 + 8u * (3 * STAGES + 6 + b); };
    int32_t* rs_buf = reinterpret_cast<int32_t*>(smem + Cfg::RS_OFF);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + Cfg::TMEMPTR_OFF);

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        ptx::prefetch_tmap(&tmap_b);
        if (MODE == 3) ptx::prefetch_tmap(&tmap_c);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(full_bar(s), 1);    // leader: its own producer's expect_tx arrive
            ptx::mbar_init(empty_bar(s), 1);   // the leader's multicast commit
            ptx::mbar_init(rsdone_bar(s), 2);  // this CTA's two row-sum warps
            ptx::mbar_init(aread_bar(s), 1);
        }
        for (int h = 0; h < 2; ++h) {
            ptx::mbar_init(tfull_bar(h), 1);
            ptx::mbar_init(tempty_bar(h), 16);  // leader: 8 local + 8 follower epilogue warps
            ptx::mbar_init(rfull_bar(h), 2);
            ptx::mbar_init(rempty_bar(h), 8);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc_pair<512>(ptx::smem_u32(tmem_ptr));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();  // both CTAs' barriers exist before any remote arrive / cta_group::2 load
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_ptr;
    ptx::griddep_wait();  // PDL: the prologue above overlapped the previous grid

    const int group = blockIdx.x / 2, groups = gridDim.x / 2;
    const TileRange tr = tile_range(p, group, groups);
    const int nt = p.num_n_tiles;

    if (warp == 0) {
        // ------------------------------------------------ producer (both CTAs)
        const uint64_t pol_b = ptx::policy_evict_last();  // every pair re-reads all of B
        const uint32_t full_leader0 = ptx::mapa_shared(full_bar(0), 0);
        int stage = 0;
        uint32_t phase = 0;
        for (int t = tr.first; t < tr.last; t += tr.step) {
            const int mt = t / nt, ntile = t % nt;
            const int m0 = mt * 2 * BM + (int)rank * BM;
            const int brow = ntile * PN + (int)rank * HN;  // this CTA's columns of sub-tile 0
            for (int kb = 0; kb < p.nkb; ++kb) {
                ptx::mbar_wait(empty_bar(stage), phase ^ 1);
                // the row-sum warps arrive once per use of every stage (reading
                // it on row-sum tiles): they are done with the previous use
                if (RS) ptx::mbar_wait(rsdone_bar(stage), phase ^ 1);
                if (ptx::elect_one()) {
                    if (leader) ptx::mbar_arrive_expect_tx(full_bar(stage), 2 * STAGE);
                    const uint32_t fb = full_leader0 + 8u * stage;
                    ptx::tma_load_2d_pair(stage_a(stage), &tmap_a, kb * kKBlock, m0, fb);
#pragma unroll
                    for (int h = 0; h < NSUB; ++h)
                        if (p.b3d)
                            tma_load_3d_pair_hint(stage_b(stage, h), &tmap_b, 0, brow + h * 2 * HN, kb, fb, pol_b);
                        else
                            tma_load_2d_pair_hint(stage_b(stage, h), &tmap_b, 0, kb * p.np + brow + h * 2 * HN, fb,
                                                  pol_b);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && leader) {
        // ------------------------------------------------ MMA issuer (leader)
        // Per tile the (k block, half) items run k-block-interleaved, except
        // that the last `de` k blocks (default 4) issue all their half-0 MMAs
        // before their half-1 MMAs and the next tile's first `ds` k blocks
        // (default 0) do the same: the
        // half-0 accumulator is complete de half-blocks before half 1, and the
        // next tile needs half 1 back only (de + ds) half-blocks (x 512 MMA
        // cycles) after half 0 was full -- time for the epilogue to drain,
        // requantize and store half 0 and drain half 1 without the tensor pipe
        // waiting.  Stages are consumed and released in k-block order.
        constexpr uint32_t idesc = ptx::idesc_u8s8_s32<2 * BM, 2 * HN>();
        const int nkb = p.nkb;
        const int de = p.skew_end, ds = p.skew_start;  // host-clamped: de + ds <= min(nkb, STAGES)
        uint32_t gkb = 0;  // k blocks consumed so far (stage = gkb % STAGES)
        uint32_t acc_phase = 0;
        int ti = 0;
        auto wait_full = [&](uint32_t g) {
            ptx::mbar_wait(full_bar((int)(g % STAGES)), (g / STAGES) & 1u);
            ptx::tc_fence_after();
        };
        auto release = [&](uint32_t g) {
            if (ptx::elect_one()) ptx::tc_commit_pair_mc(empty_bar((int)(g % STAGES)), 0x3);
            __syncwarp();
        };
        auto item = [&](uint32_t g, int kb, int h) {
            if (kb == 0) {  // the previous tile's epilogue has drained this half
                ptx::mbar_wait_cluster(tempty_bar(h), acc_phase ^ 1);
                ptx::tc_fence_after();
            }
            const int s = (int)(g % STAGES);
            const uint64_t adesc = ptx::sw128_kmajor_desc(stage_a(s));
            const uint64_t bdesc = ptx::sw128_kmajor_desc(stage_b(s, h));
            if (ptx::elect_one()) {
                if (kb == 0) tw_tile(p, h, ti);
#pragma unroll
                for (int ks = 0; ks < kKBlock / 32; ++ks)
                    ptx::mma_i8_pair(tmem_base + (uint32_t)(h * 2 * HN), adesc + 2 * ks, bdesc + 2 * ks, idesc,
                                     (kb | ks) != 0);
                if (RS && h == 0) ptx::tc_commit_pair_mc(aread_bar(s), 0x3);  // (before the stage's half-1 MMAs)
                if (kb == nkb - 1) {
                    ptx::tc_commit_pair_mc(tfull_bar(h), 0x3);
                    tw_tile(p, 2 + h, ti);
                }
            }
            __syncwarp();
        };
        for (int t = tr.first; t < tr.last; t += tr.step, ++ti) {
            const uint32_t g0 = gkb;
            for (int kb = 0; kb < ds; ++kb) {
                wait_full(g0 + kb);
                item(g0 + kb, kb, 0);
            }
            for (int kb = 0; kb < ds; ++kb) {
                item(g0 + kb, kb, 1);
                release(g0 + kb);
            }
            for (int kb = ds; kb < nkb - de; ++kb) {
                wait_full(g0 + kb);
                item(g0 + kb, kb, 0);
                item(g0 + kb, kb, 1);
                release(g0 + kb);
            }
            for (int kb = nkb - de; kb < nkb; ++kb) {
                wait_full(g0 + kb);
                item(g0 + kb, kb, 0);
            }
            for (int kb = nkb - de; kb < nkb; ++kb) {
                item(g0 + kb, kb, 1);
                release(g0 + kb);
            }
            gkb = g0 + (uint32_t)nkb;
            acc_phase ^= 1;
        }
    } else if (RS && (warp == 2 || warp == 3)) {
        // ------------------------------------------------ row sums (both CTAs)
        const int r0 = (warp - 2) * 32 + lane;  // rows r0 and r0 + 64 of this CTA's 128
        int stage = 0;
        uint32_t phase = 0;
        int run = 0;
        int prev_m = -1;
        for (int t = tr.first; t < tr.last; t += tr.step) {
            const int mt = t / nt;
            const bool rs_tile = mt != prev_m;
            prev_m = mt;
            // every use of every stage is waited on in order, row-sum tile or
            // not: a waiter that skipped phases could see an old phase of the
            // same parity as complete
            const int b = run & 1;
            if (rs_tile) ptx::mbar_wait(rempty_bar(b), ((run >> 1) & 1) ^ 1);
            uint32_t s0 = 0, s1 = 0;
            for (int kb = 0; kb < p.nkb; ++kb) {
                // the stage's half-0 MMAs are complete: its A has landed and
                // stays until this warp arrives on rsdone (the producer waits
                // for that, on every use, before reloading the stage)
                ptx::mbar_wait_cluster(aread_bar(stage), phase);
                if (rs_tile) {
                    const uint8_t* sa = smem + stage * STAGE;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        // rotated 16-byte chunk order: conflict-free; the sum is swizzle-invariant
                        const uint4 w0 = *reinterpret_cast<const uint4*>(sa + r0 * kKBlock + ((q + r0) & 7) * 16);
                        const uint4 w1 =
                            *reinterpret_cast<const uint4*>(sa + (r0 + 64) * kKBlock + ((q + r0) & 7) * 16);
                        s0 = ptx::dp4a_uu(w0.x, 0x01010101u, s0);
                        s0 = ptx::dp4a_uu(w0.y, 0x01010101u, s0);
                        s0 = ptx::dp4a_uu(w0.z, 0x01010101u, s0);
                        s0 = ptx::dp4a_uu(w0.w, 0x01010101u, s0);
                        s1 = ptx::dp4a_uu(w1.x, 0x01010101u, s1);
                        s1 = ptx::dp4a_uu(w1.y, 0x01010101u, s1);
                        s1 = ptx::dp4a_uu(w1.z, 0x01010101u, s1);
                        s1 = ptx::dp4a_uu(w1.w, 0x01010101u, s1);
                    }
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(rsdone_bar(stage));
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (!rs_tile) continue;
            rs_buf[b * BM + r0] = (int32_t)s0;
            rs_buf[b * BM + r0 + 64] = (int32_t)s1;
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(rfull_bar(b));
            ++run;
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue (both CTAs)
        const int q = warp & 3;          // TMEM lane quarter this warp may access
        const int g = (warp - 4) >> 2;   // 128-column group within each 256-column half
        const int r = q * 32 + lane;     // row of this CTA's 128
        const uint32_t leader_tempty0 = ptx::mapa_shared(tempty_bar(0), 0);
        const int et = threadIdx.x - 128;  // 0..255 over the epilogue warps
        int32_t* rc = reinterpret_cast<int32_t*>(smem + Cfg::REC_OFF);
        int32_t* rz = rc + PN;
        int32_t* rm = rz + PN;
        int32_t* rm2 = rm + PN;
        const int32_t zoff = 0x4B400000 - p.ea.zp_c;
        const float floor_x = p.ea.relu ? 0.0f : -8388608.0f;
        uint32_t acc_phase = 0;
        int run = -1;
        int prev_m = -1;
        int32_t rowsum = 0;
        int ti = 0;
        for (int t = tr.first; t < tr.last; t += tr.step, ++ti) {
            const int mt = t / nt, ntile = t % nt;
            const bool new_run = mt != prev_m;
            prev_m = mt;
            if (new_run) ++run;
            const int row = mt * 2 * BM + (int)rank * BM + r;
            const bool valid = row < p.rows;
            if (MODE == 3) {
                // this tile's 512 column records into shared memory, while the
                // MMAs run (all 8 warps are done with the previous tile's)
                named_bar_sync(1, 256);
                for (int i = et; i < PN; i += 256) {
                    const int4 rr = ntile * PN + i < p.np ? __ldg(reinterpret_cast<const int4*>(p.ea.rec) + ntile * PN + i)
                                                          : make_int4(0, 0, 0, 0);  // (columns past np: never stored)
                    rc[i] = rr.x;
                    rz[i] = rr.y;
                    rm[i] = rr.z;
                    rm2[i] = rr.w;
                }
                named_bar_sync(1, 256);
            }
#pragma unroll 1
            for (int h = 0; h < NSUB; ++h) {
                ptx::mbar_wait(tfull_bar(h), acc_phase);
                ptx::tc_fence_after();
                if (warp == 4 && lane == 0) tw_tile(p, 4 + 2 * h, ti);
                uint32_t v[128];
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * 2 * HN + g * HN);
                ptx::tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(v));
                ptx::tmem_ld_32x32b_x32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
                ptx::tmem_ld_32x32b_x32(taddr + 64, *reinterpret_cast<uint32_t(*)[32]>(v + 64));
                ptx::tmem_ld_32x32b_x32(taddr + 96, *reinterpret_cast<uint32_t(*)[32]>(v + 96));
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                __syncwarp();
                // the half is in registers: hand it back to the MMA now
                if (lane == 0) mbar_arrive_remote_relaxed(leader_tempty0 + 8u * h);
                if (warp == 4 && lane == 0) tw_tile(p, 5 + 2 * h, ti);
                if (RS && h == 0 && new_run) {
                    const int b = run & 1;
                    ptx::mbar_wait(rfull_bar(b), (run >> 1) & 1);
                    rowsum = rs_buf[b * BM + r];
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(rempty_bar(b));
                }
                if (warp == 4 && lane == 0) tw_epi(p, 6 + h, ti);  // row sums in hand
                const uint32_t nrowsum = 0u - (uint32_t)rowsum;
                const int lc0 = h * 2 * HN + g * HN;  // tile-local column of v[0]
                const int col0 = ntile * PN + lc0;
                if constexpr (MODE == 3) {
                    // F32_RNE fast path, 2 rounds of 64 columns: requantize into
                    // this warp's SWIZZLE_64B staging tile, one TMA store of 32
                    // rows x 64 B (rows >= M, columns >= N clipped by the TMA unit)
                    const uint32_t stg = base + Cfg::OUT_OFF + (uint32_t)((warp - 4) * Cfg::OUT_WARP);
#pragma unroll
                    for (int rd = 0; rd < 2; ++rd) {
                        if (lane == 0) bulk_wait_read0();  // the previous store has read the tile
                        __syncwarp();
                        if (rd == 1 && warp == 4 && lane == 0) tw_epi(p, 3 * h + 1, ti);
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const int cc = rd * 4 + c;
                            const uint4 w = requant16_fast(v + cc * 16, rc + lc0 + cc * 16, rz + lc0 + cc * 16,
                                                           reinterpret_cast<const float*>(rm) + lc0 + cc * 16, nrowsum,
                                                           zoff, floor_x);
                            const uint32_t dst = stg + (uint32_t)(lane * 64 + ((c ^ ((lane >> 1) & 3)) * 16));
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(w.x), "r"(w.y),
                                         "r"(w.z), "r"(w.w)
                                         : "memory");
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (warp == 4 && lane == 0) tw_epi(p, 3 * h + 2 * rd, ti);
                        if (lane == 0) {
                            const int orow = mt * 2 * BM + (int)rank * BM + q * 32;
                            tma_store_2d(&tmap_c, stg, col0 + rd * 64, orow);
                            for (int d = 0; d < p.n_peers; ++d) tma_store_2d(&peers.m[d], stg, col0 + rd * 64, orow);
                        }
                    }
                } else if (valid) {
#pragma unroll
                    for (int c = 0; c < HN / 16; ++c)
                        if (col0 + c * 16 < p.n)
                            store_chunk16<MODE>(p.ea, row, col0 + c * 16,
                                                *reinterpret_cast<const uint32_t(*)[16]>(v + c * 16), rowsum);
                }
            }
            acc_phase ^= 1;
        }
        if (MODE == 3 && lane == 0) bulk_wait0();  // staging tiles stay valid until the stores have read them
    }

    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();  // the pair finishes together before TMEM is released
    if (threadIdx.x == 0) tw_clk(p, 1);
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair<512>(tmem_base);
    }
}

// packed B (q8g_internal.cuh) as u8 rows of 128 K-bytes, box 128 B x 128
// columns, no swizzle: the rows are pre-swizzled, so a box lands in shared
// memory in the tcgen05 K-major SW128 layout.  np % 512 == 0: a 2-D tensor of
// (kp/128 * np) rows.  Otherwise a 3-D tensor (128 B, np columns, kp/128
// k-blocks) whose columns past np read as zeros, for the last 512-column
// tile.  (The 3-D map for every shape measured C2 at 165 us vs 161.6 us and
// a lower clock: 1575 vs 1615 MHz.)
bool make_tmap_b(CUtensorMap* m, const q8g_packed_b* pb) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    CUresult r;
    if (pb->np % PN == 0) {
        cuuint64_t dims[2] = {(cuuint64_t)kKBlock, (cuuint64_t)(pb->kp / kKBlock) * (cuuint64_t)pb->np};
        cuuint64_t strides[1] = {(cuuint64_t)kKBlock};
        cuuint32_t box[2] = {(cuuint32_t)kKBlock, (cuuint32_t)HN};
        cuuint32_t estr[2] = {1, 1};
        r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, pb->data, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[3] = {(cuuint64_t)kKBlock, (cuuint64_t)pb->np, (cuuint64_t)(pb->kp / kKBlock)};
        cuuint64_t strides[2] = {(cuuint64_t)kKBlock, (cuuint64_t)pb->np * kKBlock};
        cuuint32_t box[3] = {(cuuint32_t)kKBlock, (cuuint32_t)HN, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, pb->data, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    return r == CUDA_SUCCESS;
}

bool cached_tmap_b(CUtensorMap* out, const q8g_packed_b* pb) {
    struct Key {
        const void* d;
        int kp, np;
        bool operator==(const Key& o) const { return d == o.d && kp == o.kp && np == o.np; }
    };
    struct Hash {
        size_t operator()(const Key& k) const {
            return std::hash<const void*>()(k.d) ^ ((size_t)k.kp << 32) ^ (size_t)k.np;
        }
    };
    static std::mutex mu;
    static std::unordered_map<Key, CUtensorMap, Hash> cache;
    const Key key{pb->data, pb->kp, pb->np};
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return true;
    }
    if (!make_tmap_b(out, pb)) return false;
    if (cache.size() > 4096) cache.clear();
    cache.emplace(key, *out);
    return true;
}

// the u8 output C (rows x n, ldc) as a 2-D tensor, box 64 B x 32 rows,
// SWIZZLE_64B (the staging layout of the epilogue warps)
bool cached_tmap_c(CUtensorMap* out, void* c, int rows, int n, int ldc) {
    struct Key {
        const void* c;
        int rows, n, ldc;
        bool operator==(const Key& o) const { return c == o.c && rows == o.rows && n == o.n && ldc == o.ldc; }
    };
    struct Hash {
        size_t operator()(const Key& k) const {
            return std::hash<const void*>()(k.c) ^ ((size_t)k.rows << 40) ^ ((size_t)k.n << 20) ^ (size_t)k.ldc;
        }
    };
    static std::mutex mu;
    static std::unordered_map<Key, CUtensorMap, Hash> cache;
    const Key key{c, rows, n, ldc};
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return true;
    }
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ldc};
    cuuint32_t box[2] = {64, 32};
    cuuint32_t estr[2] = {1, 1};
    if (enc(out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (cache.size() > 4096) cache.clear();
    cache.emplace(key, *out);
    return true;
}

int env_sched() {
    static const int v = [] {
        const char* e = getenv("Q8G_TC2W_SCHED");
        return e && e[0] == '1' ? 1 : 0;
    }();
    return v;
}

template <int MODE, bool RS>
cudaError_t launch_tc2w(const GemmArgs& g, cudaStream_t s) {
    auto kern = gemm_tc2w_kernel<MODE, RS>;
    static int max_clusters[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    if (dev < 64 && !max_clusters[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        cfg.gridDim = dim3(2 * (sm_count(dev) / 2));
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
            cudaGetLastError();
            n = sm_count(dev) / 2;
        }
        max_clusters[dev] = n;
    }
    CUtensorMap ta, tb, tc;
    if (!make_tmap_a_cached(&ta, g.a, g.rows, g.k, g.lda, BM)) return cudaErrorInvalidValue;
    if (!cached_tmap_b(&tb, g.pb)) return cudaErrorInvalidValue;
    memset(&tc, 0, sizeof(tc));
    if (MODE == 3 && !cached_tmap_c(&tc, g.c, g.rows, g.pb->n, g.ldc)) return cudaErrorNotSupported;
    PeerMaps pm;
    memset(&pm, 0, sizeof(pm));
    int n_peers = 0;
    if (MODE == 3 && g.n_peers > 0) {
        if (g.n_peers > kMaxPeers) return cudaErrorNotSupported;
        for (int d = 0; d < g.n_peers; ++d)
            if ((reinterpret_cast<uintptr_t>(g.c_peers[d]) & 15) != 0 ||
                !cached_tmap_c(&pm.m[d], g.c_peers[d], g.rows, g.pb->n, g.ldc))
                return cudaErrorNotSupported;
        n_peers = g.n_peers;
    }
    Tc2wParams p;
    p.a = g.a;
    p.nkb = g.pb->kp / kKBlock;
    p.n = g.pb->n;
    p.rows = g.rows;
    p.num_m_tiles = ceil_div_i(g.rows, 2 * BM);
    p.num_n_tiles = ceil_div_i(g.pb->np, PN);
    p.np = g.pb->np;
    p.b3d = g.pb->np % PN != 0;
    p.sched = env_sched();
    p.tma_out = MODE == 3 ? 1 : 0;
    p.n_peers = n_peers;
    {
        // MMA skew: de + ds <= STAGES (the stages held across the tile
        // boundary) and <= nkb
        static int de0 = -1, ds0 = -1;
        if (de0 < 0) {
            // C2 (bench.py, 3 interleaved runs each): 4,0 161.5-161.7 us,
            // 2,2 162.8-163.0, 3,1 163.3-163.4, 3,0 163.3-163.5, 0,4 163.2-163.3
            de0 = 4;
            ds0 = 0;
            const char* e = getenv("Q8G_TC2W_SKEW");  // "de,ds" (A/B experiments)
            if (e) sscanf(e, "%d,%d", &de0, &ds0);
        }
        int de = de0 < 0 ? 0 : de0, ds = ds0 < 0 ? 0 : ds0;
        while (de + ds > STAGES || de + ds > p.nkb) {
            if (ds > 0) --ds;
            else --de;
        }
        p.skew_end = de;
        p.skew_start = ds;
    }
    p.ea = EpiArgs{g.ep ? g.ep->rec : nullptr, g.ep ? g.ep->zp_c : 0, g.ep ? g.ep->relu : 0,
                   (g.ep && g.ep->fast_f32) ? 1 : 0, g.bias_add, g.c, g.ldc, g.pb->n};
    p.trace = tc_trace_buffer_ptr();
    const int total = p.num_m_tiles * p.num_n_tiles;
    const int maxc = dev < 64 ? max_clusters[dev] : sm_count(dev) / 2;
    const int clusters = total < maxc ? total : maxc;
    cfg.gridDim = dim3(2 * clusters);
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, pm, p);
    count_launch(kFamGemmTcLargeM);
    if (e == cudaSuccess && n_peers > 0 && g.peers_written) *g.peers_written = true;
    return e;
}

}  // namespace

// clock64 cycles and globaltimer ns of CTA 0 of the last 256 x 512 pair-kernel launch
int tc2w_last_clock(unsigned long long* cycles, unsigned long long* ns) {
    unsigned long long h[4] = {0, 0, 0, 0};
    if (cudaMemcpyFromSymbol(h, g_tc2w_clock, sizeof(h)) != cudaSuccess) return -1;
    *cycles = h[1] - h[0];
    *ns = h[3] - h[2];
    return 0;
}

// every large-M shape (a last 512-column tile past np reads zero weights and
// stores nothing); Q8G_TC2W=0 falls back to the 1-CTA 256-row kernel
// (gemm_tc.cu) for A/B
bool tc2w_supported(const GemmArgs& g) {
    static const bool off = [] {
        const char* e = getenv("Q8G_TC2W");
        return e && e[0] == '0';
    }();
    return !off && tmap_encoder() != nullptr;
}

cudaError_t launch_gemm_tc2w(const GemmArgs& g, cudaStream_t s) {
    if (g.raw) return launch_tc2w<0, false>(g, s);
    const bool rs = g.ep->need_rowsum;
    if (g.ep->rounding == Q8G_ROUND_F32_RNE) {
        static const bool tma_out_off = [] {
            const char* e = getenv("Q8G_TC2W_TMA_OUT");
            return e && e[0] == '0';
        }();
        if (!tma_out_off && g.ep->fast_f32 && g.ldc % 16 == 0 && (reinterpret_cast<uintptr_t>(g.c) & 15) == 0) {
            const cudaError_t e = rs ? launch_tc2w<3, true>(g, s) : launch_tc2w<3, false>(g, s);
            if (e != cudaErrorNotSupported) return e;
        }
        return rs ? launch_tc2w<1, true>(g, s) : launch_tc2w<1, false>(g, s);
    }
    return rs ? launch_tc2w<2, true>(g, s) : launch_tc2w<2, false>(g, s);
}

}  // namespace q8g
