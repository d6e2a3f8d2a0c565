// gemm_tc2.cu — large-M GEMM on CTA pairs (tcgen05.mma.cta_group::2):
// BASELINE C2-class shapes (M in the thousands, N x K = 4096 x 4096).
//
// Why: with one CTA per 128x256 tile every k-block moves 48 KB into shared
// memory (A 16 KB + B 32 KB by TMA) and the MMA reads the same 48 KB back, a
// 768-cycle smem budget against 512 cycles of tensor math -- the 1-CTA kernel
// ran at ~65% of the measured INT8 peak, as that ratio predicts.  A CTA pair
// computes a 256x256 tile with each SM holding half of A (its 128 rows) and
// half of B (128 of the 256 columns): 32 KB in + 32 KB read per k-block,
// balanced with the math.
//
// Same drop-in semantics as gemm_tc.cu (engine.hpp:59-169 + the requant
// back-end, pipeline.hpp:157-210 / quant.hpp:115-133) with a different tiling.
//
// Per CTA of the pair (rank 0 = leader):
//   warp 0      producer: this CTA's A rows (TMA, SWIZZLE_128B) and its half of
//               B (one bulk copy of the pre-swizzled packed weight), completing
//               on the CTA's own full barrier
//   warp 1      leader: MMA issuer, 4 x tcgen05.mma.cta_group::2 (M256 N256
//               K32) per stage, commits multicast to both CTAs' empty / tfull
//               barriers;  follower: relays "my stage landed" to the leader's
//               pfull barrier (release.cluster remote arrive)
//   warp 2      TMEM allocator (cta_group::2, 2 accumulators x 256 columns)
//   warps 4-7   epilogue of this CTA's 128 rows x 256 columns; arrive on the
//               leader's tempty barrier
//   warps 8-11  row sums of this CTA's A rows (only when some zp_b != 0)
//
// Cross-CTA arrives (relay, tempty, rsdone) are .relaxed.cluster: each is
// sent after the sender observed the completion it reports (a TMA
// complete_tx on its own barrier, tcgen05.wait::ld, its own smem reads), so
// the data is complete when the leader acts on it.  A .release.cluster arrive
// instead waits for the CTA's outstanding memory traffic -- including the
// next stages' TMA loads still in flight -- and measured 2.3x slower (one
// relay per ~1 us).  tests/test_gpu_gemm.py repeats the pair kernel 20x.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "epilogue.cuh"
#include "ptx.cuh"
#include "q8g_internal.cuh"

namespace q8g {

bool make_tmap_a_cached(CUtensorMap* out, const uint8_t* a, int rows, int k, int lda, int box_rows);
unsigned long long* tc_trace_buffer_ptr();

namespace {

constexpr int BM = 128;        // rows per CTA (256 per pair)
constexpr int HN = 128;        // B columns held per CTA (256 per pair)
constexpr int PN = 2 * HN;     // pair tile N
constexpr int STAGE_A = BM * kKBlock;
constexpr int STAGE_B = HN * kKBlock;

template <int STAGES>
struct Tc2Cfg {
    static constexpr int A_OFF = 0;
    static constexpr int B_OFF = STAGES * STAGE_A;
    static constexpr int BAR_OFF = B_OFF + STAGES * STAGE_B;
    // full[S], pfull[S], empty[S], rsdone[S], tfull[2], tempty[2], rfull[2], rempty[2]
    static constexpr int NUM_BARS = 4 * STAGES + 8;
    static constexpr int RS_OFF = BAR_OFF + NUM_BARS * 8;
    static constexpr int TMEMPTR_OFF = RS_OFF + 2 * BM * 4;
    static constexpr int SMEM_BYTES = TMEMPTR_OFF + 16 + 1024;
    static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KB dynamic shared memory limit");
};

struct Tc2Params {
    const int8_t* pb;
    int np, nkb, n, rows;
    int num_m_tiles, num_n_tiles;  // pair tiles: 256 rows x 256 columns
    EpiArgs ea;
    unsigned long long* trace;
};

__device__ __forceinline__ void t2_stamp(const Tc2Params& p, int slot) {
    if (p.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[blockIdx.x * 8 + slot] = t;
    }
}

// first pair, first tile, per k-block (debug): [8192 + 64*which + kb]: 0 leader
// producer issued, 1 MMA past full, 2 MMA past pfull, 3 MMAs issued, 4
// follower producer issued, 5 follower relay sent
// CTA 0, per tile ti < 32: [9216 + 4 * ti + k], k: 0 first MMA issued, 1 last
// MMA issued (tfull committed), 2 epilogue start, 3 epilogue done
// (tools/tc2_tiles.py)
__device__ __forceinline__ void t2_tile(const Tc2Params& p, int k, int ti) {
    if (p.trace && blockIdx.x == 0 && ti < 32) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[9216 + 4 * ti + k] = t;
    }
}
__device__ __forceinline__ void t2_kb(const Tc2Params& p, int which, int kb) {
    if (p.trace && blockIdx.x < 2 && kb < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8192 + which * 64 + kb] = t;
    }
}

// CTA 0: SM clock and globaltimer at kernel entry / exit (effective SM clock
// of the launch, tools/c2_clock.py): [10200] clock0 [10201] clock1 [10202] t0 [10203] t1
__device__ __forceinline__ void t2_clk(const Tc2Params& p, int end) {
    if (p.trace && blockIdx.x == 0) {
        unsigned long long t, c;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
        p.trace[10200 + end] = c;
        p.trace[10202 + end] = t;
    }
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// CL = CTAs per cluster: 2 (one pair) or 4 (two pairs on the same N tile and
// adjacent M tiles: each half of B is loaded once, half by each pair, and
// multicast to both -- 25% less L2 -> SM traffic)
template <int STAGES, int MODE, bool RS, int CL>
__global__ void __launch_bounds__(RS ? 384 : 256, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmap_a, const Tc2Params p) {
    static_assert(CL == 2 || CL == 4, "one or two CTA pairs per cluster");
    constexpr int PPC = CL / 2;  // pairs per cluster
    using Cfg = Tc2Cfg<STAGES>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_addr);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    ptx::griddep_launch_dependents();
    if (threadIdx.x == 0) t2_stamp(p, 0);
    if (threadIdx.x == 0) t2_clk(p, 0);
    const uint32_t rank = ptx::cluster_ctarank();
    const uint32_t lrank = rank & ~1u;         // this CTA's pair leader
    const bool leader = (rank & 1u) == 0;
    const int q = (int)(rank >> 1);             // pair within the cluster
    const uint16_t pair_mask = (uint16_t)(3u << lrank);

    const uint32_t sA = base + Cfg::A_OFF, sB = base + Cfg::B_OFF;
    const uint32_t bar0 = base + Cfg::BAR_OFF;
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto pfull_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
    auto empty_bar = [&](int s) { return bar0 + 8u * (2 * STAGES + s); };
    auto rsdone_bar = [&](int s) { return bar0 + 8u * (3 * STAGES + s); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (4 * STAGES + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (4 * STAGES + 2 + a); };
    auto rfull_bar = [&](int a) { return bar0 + 8u * (4 * STAGES + 4 + a); };
    auto rempty_bar = [&](int a) { return bar0 + 8u * (4 * STAGES + 6 + a); };
    int32_t* rs_buf = reinterpret_cast<int32_t*>(smem + Cfg::RS_OFF);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + Cfg::TMEMPTR_OFF);

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(full_bar(s), 1);
            ptx::mbar_init(pfull_bar(s), 1);    // leader: the follower's relay
            ptx::mbar_init(empty_bar(s), PPC);  // one multicast commit per pair leader (B is shared)
            ptx::mbar_init(rsdone_bar(s), 8);   // leader: 4 local + 4 follower row-sum warps
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull_bar(a), 1);
            ptx::mbar_init(tempty_bar(a), 8);   // leader: 4 local + 4 follower epilogue warps
            ptx::mbar_init(rfull_bar(a), 4);
            ptx::mbar_init(rempty_bar(a), 4);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc_pair<512>(ptx::smem_u32(tmem_ptr));
    ptx::tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // every CTA's barriers exist before any remote arrive / multicast
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_ptr;
    ptx::griddep_wait();  // PDL: the prologue above overlapped the previous grid
    if (threadIdx.x == 0) t2_stamp(p, 1);

    // cluster-level tiles: PPC adjacent 256-row M tiles x one 256-column N tile;
    // pair q takes M tile PPC*(T / nt) + q (past the end -> zero A, no stores)
    const int num_groups = gridDim.x / CL;
    const int group = blockIdx.x / CL;
    const int total = ((p.num_m_tiles + PPC - 1) / PPC) * p.num_n_tiles;
    auto tile_m0 = [&](int T) { return (PPC * (T / p.num_n_tiles) + q) * 2 * BM + (int)(rank & 1u) * BM; };
    auto tile_n0 = [&](int T) { return (T % p.num_n_tiles) * PN; };

    if (warp == 0) {
        // ------------------------------------------------ producer (both CTAs)
        const uint64_t pol_b = ptx::policy_evict_last();  // B is re-read by every M tile
        int stage = 0;
        uint32_t phase = 0;
        for (int t = group; t < total; t += num_groups) {
            const int m0 = tile_m0(t);
            const int nb = tile_n0(t) + (int)(rank & 1u) * HN;  // this CTA's half of the pair's 256 columns
            for (int kb = 0; kb < p.nkb; ++kb) {
                ptx::mbar_wait(empty_bar(stage), phase ^ 1);
                if (ptx::elect_one()) {
                    ptx::mbar_arrive_expect_tx(full_bar(stage), STAGE_A + STAGE_B);
                    ptx::tma_load_2d(sA + stage * STAGE_A, &tmap_a, kb * kKBlock, m0, full_bar(stage));
                    if (CL == 2) {
                        ptx::bulk_load_hint(sB + stage * STAGE_B, p.pb + ((size_t)kb * p.np + nb) * kKBlock, STAGE_B,
                                            full_bar(stage), pol_b);
                    } else {
                        // rows [64q, 64q+64) of this B half, to me and my counterpart in the other pair
                        constexpr int PIECE = STAGE_B / 2;
                        ptx::bulk_load_mc_hint(sB + stage * STAGE_B + q * PIECE,
                                               p.pb + ((size_t)kb * p.np + nb + q * (HN / 2)) * kKBlock, PIECE,
                                               full_bar(stage), (uint16_t)((1u << rank) | (1u << (rank ^ 2u))), pol_b);
                    }
                    if (kb == 0 && t == group) t2_stamp(p, 2);
                    if (t == group) t2_kb(p, leader ? 0 : 4, kb);
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
        constexpr uint32_t idesc = ptx::idesc_u8s8_s32<2 * BM, PN>();
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = group; t < total; t += num_groups) {
            ptx::mbar_wait_cluster(tempty_bar(acc), acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem_base + (uint32_t)(acc * PN);
            for (int kb = 0; kb < p.nkb; ++kb) {
                ptx::mbar_wait(full_bar(stage), phase);
                if (t == group && lane == 0) t2_kb(p, 1, kb);
                ptx::mbar_wait_cluster(pfull_bar(stage), phase);
                if (t == group && lane == 0) t2_kb(p, 2, kb);
                ptx::tc_fence_after();
                const uint64_t adesc = ptx::sw128_kmajor_desc(sA + stage * STAGE_A);
                const uint64_t bdesc = ptx::sw128_kmajor_desc(sB + stage * STAGE_B);
                if (ptx::elect_one()) {
                    if (kb == 0 && t == group) t2_stamp(p, 3);
                    if (kb == 0) t2_tile(p, 0, (t - group) / num_groups);
#pragma unroll
                    for (int ks = 0; ks < kKBlock / 32; ++ks)
                        ptx::mma_i8_pair(d, adesc + 2 * ks, bdesc + 2 * ks, idesc, (kb | ks) != 0);
                    if (t == group) t2_kb(p, 3, kb);
                }
                __syncwarp();
                // both CTAs' row-sum warps have read the stage
                if (RS) ptx::mbar_wait_cluster(rsdone_bar(stage), phase);
                // frees the stage in every CTA that wrote part of it (all of the cluster when B is shared)
                if (ptx::elect_one()) ptx::tc_commit_pair_mc(empty_bar(stage), CL == 2 ? pair_mask : (uint16_t)0xF);
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (ptx::elect_one()) {
                ptx::tc_commit_pair_mc(tfull_bar(acc), pair_mask);
                t2_stamp(p, 4);
                t2_tile(p, 1, (t - group) / num_groups);
            }
            __syncwarp();
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ follower: relay
        // "my A / B halves of this stage have landed" to the leader
        const uint32_t peer_pfull0 = ptx::mapa_shared(pfull_bar(0), lrank);
        int stage = 0;
        uint32_t phase = 0;
        for (int t = group; t < total; t += num_groups) {
            for (int kb = 0; kb < p.nkb; ++kb) {
                ptx::mbar_wait_spin(full_bar(stage), phase);
                if (ptx::elect_one())
                    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                     peer_pfull0 + 8u * stage)
                                 : "memory");
                if (t == group && lane == 0) t2_kb(p, 5, kb);
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ------------------------------------------------ epilogue (both CTAs)
        const int ew = warp - 4;
        const int r = ew * 32 + lane;
        const uint32_t leader_tempty0 = ptx::mapa_shared(tempty_bar(0), lrank);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = group; t < total; t += num_groups) {
            const int row = tile_m0(t) + r;
            const int n0 = tile_n0(t);
            ptx::mbar_wait(tfull_bar(acc), acc_phase);
            ptx::tc_fence_after();
            if (warp == 4 && lane == 0 && t == group) t2_stamp(p, 5);
            if (warp == 4 && lane == 0) t2_tile(p, 2, (t - group) / num_groups);
            int32_t rowsum = 0;
            if (RS) {
                ptx::mbar_wait(rfull_bar(acc), acc_phase);
                rowsum = rs_buf[acc * BM + r];
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(rempty_bar(acc));
            }
            const bool valid = row < p.rows;
#pragma unroll 1
            for (int ch = 0; ch < PN / 16; ++ch) {
                uint32_t v[16];
                ptx::tmem_ld_32x32b_x16(tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(acc * PN + ch * 16), v);
                ptx::tmem_ld_wait();
                const int col0 = n0 + ch * 16;
                if (valid && col0 < p.n) store_chunk16<MODE>(p.ea, row, col0, v, rowsum);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 leader_tempty0 + 8u * acc)
                             : "memory");
            if (warp == 4 && lane == 0) t2_stamp(p, 6);
            if (warp == 4 && lane == 0) t2_tile(p, 3, (t - group) / num_groups);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (RS && warp >= 8) {
        // ------------------------------------------------ row sums (both CTAs)
        const int r = (warp - 8) * 32 + lane;
        const uint32_t leader_rsdone0 = ptx::mapa_shared(rsdone_bar(0), lrank);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = group; t < total; t += num_groups) {
            ptx::mbar_wait(rempty_bar(acc), acc_phase ^ 1);
            uint32_t sum = 0;
            for (int kb = 0; kb < p.nkb; ++kb) {
                ptx::mbar_wait(full_bar(stage), phase);
                const uint8_t* rowp = smem + Cfg::A_OFF + stage * STAGE_A + r * kKBlock;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint4 w = *reinterpret_cast<const uint4*>(rowp + ((q + r) & 7) * 16);
                    sum = ptx::dp4a_uu(w.x, 0x01010101u, sum);
                    sum = ptx::dp4a_uu(w.y, 0x01010101u, sum);
                    sum = ptx::dp4a_uu(w.z, 0x01010101u, sum);
                    sum = ptx::dp4a_uu(w.w, 0x01010101u, sum);
                }
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                     leader_rsdone0 + 8u * stage)
                                 : "memory");
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

    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the pair finishes together before TMEM is released
    if (threadIdx.x == 0) t2_stamp(p, 7);
    if (threadIdx.x == 0) t2_clk(p, 1);
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair<512>(tmem_base);
    }
}

template <int STAGES, int MODE, bool RS, int CL>
cudaError_t launch_tc2(const GemmArgs& g, cudaStream_t s) {
    using Cfg = Tc2Cfg<STAGES>;
    auto kern = gemm_tc2_kernel<STAGES, MODE, RS, CL>;
    static int max_clusters[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(RS ? 384 : 256);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    if (dev < 64 && !max_clusters[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
        if (e != cudaSuccess) return e;
        // the persistent grid must be co-resident: as many clusters as fit at once
        cfg.gridDim = dim3(CL * (sm_count(dev) / CL));
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
            cudaGetLastError();
            n = sm_count(dev) / CL;
        }
        max_clusters[dev] = n;
    }
    CUtensorMap tmap;
    if (!make_tmap_a_cached(&tmap, g.a, g.rows, g.k, g.lda, BM)) return cudaErrorInvalidValue;
    Tc2Params p;
    p.pb = g.pb->data;
    p.np = g.pb->np;
    p.nkb = g.pb->kp / kKBlock;
    p.n = g.pb->n;
    p.rows = g.rows;
    p.num_m_tiles = ceil_div_i(g.rows, 2 * BM);
    p.num_n_tiles = g.pb->np / PN;
    p.ea = EpiArgs{g.ep ? g.ep->rec : nullptr, g.ep ? g.ep->zp_c : 0, g.ep ? g.ep->relu : 0,
                   (g.ep && g.ep->fast_f32) ? 1 : 0, g.bias_add, g.c, g.ldc, g.pb->n};
    p.trace = tc_trace_buffer_ptr();
    const int total = ((p.num_m_tiles + CL / 2 - 1) / (CL / 2)) * p.num_n_tiles;  // cluster-level tiles
    const int maxc = dev < 64 ? max_clusters[dev] : sm_count(dev) / CL;
    const int clusters = total < maxc ? total : maxc;
    cfg.gridDim = dim3(CL * clusters);
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tmap, p);
    count_launch(kFamGemmTcLargeM);
    return e;
}

}  // namespace

// the pair tile needs N padded to 256 (np is a multiple of 256 by packing)
bool tc2_supported(const GemmArgs& g) {
    static const bool off = [] {
        const char* e = getenv("Q8G_TC2");
        return e && e[0] == '0';
    }();
    return !off && g.pb->np % PN == 0;
}

template <int CL>
cudaError_t launch_tc2_modes(const GemmArgs& g, cudaStream_t s) {
    constexpr int ST = 6;
    if (g.raw) return launch_tc2<ST, 0, false, CL>(g, s);
    const bool rs = g.ep->need_rowsum;
    if (g.ep->rounding == Q8G_ROUND_F32_RNE)
        return rs ? launch_tc2<ST, 1, true, CL>(g, s) : launch_tc2<ST, 1, false, CL>(g, s);
    return rs ? launch_tc2<ST, 2, true, CL>(g, s) : launch_tc2<ST, 2, false, CL>(g, s);
}

cudaError_t launch_gemm_tc2(const GemmArgs& g, cudaStream_t s) {
    // one pair per cluster.  Q8G_TC2_CL=4 (experiment): two pairs sharing B by
    // multicast -- 25% less L2 traffic but measured slower at C2 (194 vs 182
    // us: the pairs wait on each other's stage releases; L2 is not the limit)
    static const int cl = [] {
        const char* e = getenv("Q8G_TC2_CL");
        return e && e[0] == '4' ? 4 : 2;
    }();
    if (cl == 4 && g.rows > 2 * BM) return launch_tc2_modes<4>(g, s);
    return launch_tc2_modes<2>(g, s);
}

}  // namespace q8g
