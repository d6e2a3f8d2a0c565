// conv_tc.cu — 3x3 / stride 1 / pad 1 NHWC convolution as an implicit GEMM on
// the tensor cores (BASELINE config C3), requantization fused.
//
// Semantics: SURVEY.md App. A D2 (no reference symbol; im2col is a reference
// non-goal): GEMM rows = output pixels, k = (kh*3+kw)*C + c,
// padded taps read zp_a and count in the row sums, weights = the packed
// K = 9C x N = OC matrix, epilogue table from q8g_epilogue_create (K = 9C).
//
// Design: im2col is never materialised.  A work unit is (image, ROWS output
// rows); one TMA loads a halo of ROWS+2 input rows x (W+2) padded positions
// x C channels in natural NHWC order (rows of C bytes, hardware swizzle of
// span C = 32/64/128), out-of-range taps zero-filled.  For tap t and K-step
// j (32 channels) the MMA A operand is the window starting at position
// q + (t/3)*(W+2) + t%3 - 1, bytes 32j.. of each row: a swizzled K-major
// descriptor whose start may sit at any row because the tensor core applies
// the swizzle on absolute smem addresses.  B (per-weight operand image) has the
// OC output channels plus one all-ones column, so the tensor core also
// produces the row sum of the zero-filled A.  The exact correction for
// zero- instead of zp_a-padding depends only on which taps of a pixel are
// padded (16 border classes):
//   corr[cls][j] = zp_a * sum_{t padded} (wsum_t[j] - C * zp_b[j])   (requant)
//   corr[cls][j] = zp_a * sum_{t padded} wsum_t[j]                   (raw)
// and adj = D[j] - zp_b[j] * D[ones] + c[j] + corr[cls][j].
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <cstring>

#include "ptx.cuh"
#include "q8g_internal.cuh"
#include "requant.cuh"

namespace q8g {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();
unsigned long long* tc_trace_buffer_ptr();

namespace {

constexpr int ROWS = 2;      // output rows per unit (ROWS * (W+2) <= 128 -> one M tile)
constexpr int MAX_BUF = 8;   // halo buffers in flight: p.nbuf <= MAX_BUF, as many as fit in smem
constexpr int EPI_WARPS = 8;  // two warpgroups; warpgroup g takes every other unit
constexpr int MAX_ACC = 4;    // TMEM accumulators (nacc = 4 when nq <= 128, else 2)
// The producer claims units (dynamically when p.work is set: CTAs that enter
// late -- their SM was still running the previous launch -- take fewer) and
// publishes local unit i's id in ring slot i % UNIT_RING as (i << 32 | id + 1),
// id + 1 = 0 meaning "no more units"; MMA and epilogue warps spin on the tag.
// The producer runs at most MAX_BUF + MAX_ACC units ahead of the slowest
// reader, so a slot is never overwritten before it is read.
constexpr int UNIT_RING = 16;
static_assert(UNIT_RING >= MAX_BUF + MAX_ACC + 2, "unit ring too small");
constexpr int DYN_LEAD = 4;  // dynamic claims: units in flight per CTA (see the producer)

struct CvParams {
    int nb, h, w, c, oc;
    int wp;            // w + 2
    int planes;        // c / 16
    int nq;            // MMA N = round_up(oc, 16) + 16 (ones column at index oc_pad)
    int oc_pad;        // round_up(oc, 16)
    int rblocks, units;
    int nacc, acc_cols;  // TMEM accumulators in flight and their column stride
    int nbuf;            // halo buffers
    int halo_bytes;      // (ROWS+2) * wp * C
    const int8_t* pb;  // packed weights
    int np;            // packed N pad
    const uint8_t* img;  // operand image: smem B layout + [9][oc_pad] tap sums
    int img_bytes;
    const EpiRecord* rec;  // null -> raw int32 output
    int32_t zp_a, zp_c;
    int relu, rounding;
    int fast;         // F32 fast path (0 <= zp_c <= 255, epi_f32_fast)
    int img_prefetch; // operand image built by an earlier call: load it before griddepcontrol.wait
    void* y;
    unsigned long long* trace;  // debug (Q8G_TC_TRACE): CTA 0 per-unit stamps, else null
    int* work;          // this launch's work slot (claim counters + done, q8g_internal.cuh), or null: static schedule
    int nstatic;        // static units per CTA before dynamic claiming
};

// CTA 0, local unit i < 64: [8192 + 64*which + i]; which: 0 halo issued,
// 1 MMA start, 2 MMA committed, 3 epilogue start, 4 epilogue done, [9216 + 64*(which-5) + i]:
// 5 MMA warp past tempty, 6 past full; [8192+320]
// = prologue done, [8192+321] = kernel entry
__device__ __forceinline__ void cv_stamp(const CvParams& p, int which, int i) {
#ifdef Q8G_TRACE
    if (p.trace && blockIdx.x == 0 && i < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[which < 5 ? 8192 + which * 64 + i : 9216 + (which - 5) * 64 + i] = t;
    }
#endif
}

// CTA 0 prologue stamps [9344 + k]: 0 barriers/image issued (after 1), 1 guards zeroed, 2 TMEM allocated
__device__ __forceinline__ void cv_pstamp(const CvParams& p, int k) {
#ifdef Q8G_TRACE
    if (p.trace && blockIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[9344 + k] = t;
    }
#endif
}

// unit ring (see UNIT_RING): tag = local unit index, value = id + 1 (0: none)
__device__ __forceinline__ void ring_put(uint32_t addr, int i, int id_plus1) {
    const unsigned long long v = ((unsigned long long)(uint32_t)i << 32) | (uint32_t)id_plus1;
    asm volatile("st.release.cta.shared::cta.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ int ring_get(uint32_t addr, int i) {
    unsigned long long v;
    asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    while ((uint32_t)(v >> 32) != (uint32_t)i) {
        __nanosleep(32);
        asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
    }
    return (int)(uint32_t)v;
}

__host__ __device__ constexpr int align_up(int v, int a) { return (v + a - 1) / a * a; }

struct CvLayout {
    int halo_off, halo_stride, b_off, wsum_off, corr_off, rec_off, soa_off, bar_off, tmemptr_off, ring_off, total;
};
__host__ __device__ inline CvLayout cv_layout(const CvParams& p) {
    CvLayout L;
    L.halo_off = 1024;  // front guard (windows may start one position early)
    L.halo_stride = align_up(p.halo_bytes + 2048, 1024);
    L.b_off = L.halo_off + p.nbuf * L.halo_stride;
    // B: [tap][kstep j][half][nq rows][16 B]
    const int ksteps = p.planes / 2;
    L.wsum_off = L.b_off + 9 * ksteps * 2 * p.nq * 16;
    L.corr_off = L.wsum_off + 9 * p.oc_pad * 4;  // [9][oc_pad] tap weight sums
    L.rec_off = L.corr_off + 16 * p.oc_pad * 4;  // [16][oc_pad]: c[n] + class correction
    L.soa_off = L.rec_off + p.oc_pad * 16;       // [oc_pad] epilogue records (zp_b, mult)
    L.bar_off = L.soa_off + p.oc_pad * 8;        // SoA: zp_b[oc_pad], mult_f32[oc_pad]
    L.tmemptr_off = L.bar_off + (2 * MAX_BUF + 2 * MAX_ACC + 1) * 8;  // + the operand-image barrier
    L.ring_off = L.tmemptr_off + 16;                                   // unit ring: UNIT_RING x u64
    L.total = L.ring_off + 8 * UNIT_RING + 1024;
    return L;
}

// K-major operand with rows of S = 32/64/128 bytes in the matching hardware
// swizzle (8-row groups of 8*S bytes).  The tensor core applies the XOR on
// absolute smem address bits, as TMA writes it, so the start may sit at any
// row (tap-shifted windows) with base_offset 0 (verified: tools/swz_test.cu)
__host__ __device__ inline uint64_t kmajor_swz_desc(uint32_t addr, int S) {
    const uint64_t code = S == 128 ? 2 : S == 64 ? 4 : 6;
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)((8 * S) >> 4) << 32) |
           ((uint64_t)1 << 46) | (code << 61);
}

__device__ __forceinline__ uint64_t kmajor_noswz_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

// packed weight element (k, n) (q8g_internal.cuh layout)
__device__ __forceinline__ int8_t packed_at(const int8_t* pb, int np, int k, int n) {
    const int kb = k / kKBlock, kin = k % kKBlock;
    return pb[((size_t)kb * np + n) * kKBlock + (((kin / 16) ^ (n & 7)) * 16) + (kin % 16)];
}

// operand image: [tap][kstep j][half][nq rows][16 B] (rows < oc: weights of
// input channels (2j+half)*16.., row oc_pad: all ones) then [9][oc_pad] sums
__global__ void conv_prep_kernel(const CvParams p, uint8_t* img) {
    const int ksteps = p.planes / 2;
    const int nb = 9 * ksteps * 2 * p.nq;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nb + 9 * p.oc_pad; idx += gridDim.x * blockDim.x) {
        if (idx < nb) {
            const int row = idx % p.nq, rest = idx / p.nq;  // rest = (t*ksteps + j)*2 + half
            const int half = rest % 2, j = (rest / 2) % ksteps, t = rest / (2 * ksteps);
            const int c0 = (2 * j + half) * 16;
            uint32_t v[4] = {0, 0, 0, 0};
            if (row < p.oc) {
                for (int b = 0; b < 16; ++b)
                    v[b / 4] |= (uint32_t)(uint8_t)packed_at(p.pb, p.np, t * p.c + c0 + b, row) << (8 * (b % 4));
            } else if (row == p.oc_pad) {
                v[0] = v[1] = v[2] = v[3] = 0x01010101u;  // ones column: row sums
            }
            *reinterpret_cast<uint4*>(img + (size_t)idx * 16) = make_uint4(v[0], v[1], v[2], v[3]);
        } else {
            const int e = idx - nb, t = e / p.oc_pad, n = e % p.oc_pad;
            int32_t s = 0;
            if (n < p.oc)
                for (int c = 0; c < p.c; ++c) s += packed_at(p.pb, p.np, t * p.c + c, n);
            reinterpret_cast<int32_t*>(img + (size_t)nb * 16)[e] = s;
        }
    }
}

// d = {c[15:0], sat_u8(a), sat_u8(b)} (one I2IP)
__device__ __forceinline__ uint32_t pack_sat_u8(int32_t a, int32_t b, uint32_t c) {
    uint32_t d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// F32_RNE requant of NCH x 16 accumulator columns of one position, straight
// line (one basic block for the scheduler).  Per output: adj = D + c + (-zp_b)
// * rowsum (wrapping), x = RN(float(adj) * m), then the magic add
// y = x + 1.5*2^23 gives bits(y) - 0x4B400000 = rint(x) for |x| <= 2^22 and
// stays monotone beyond (for x >= -2^23, the floor applied here, or 0 under
// ReLU), so the saturating u8 pack of bits(y) - (0x4B400000 - zp_c) is exactly
// clamp(rint(x) + zp_c, relu ? zp_c : 0, 255) (requant.cuh requant_f32).
template <bool RELU, int NCH>
__device__ __forceinline__ void epi_f32_fast(const uint32_t (&v)[4][16], int32_t rowsum, const int4* nzq,
                                             const float4* mq, const int4* cq, int32_t zoff, uint4* dst,
                                             bool valid) {
    uint32_t w[4 * NCH];
#pragma unroll
    for (int g = 0; g < 4 * NCH; ++g) {
        const int4 zb = nzq[g];
        const float4 mm = mq[g];
        const int4 cc = cq[g];
        const int32_t zv[4] = {zb.x, zb.y, zb.z, zb.w};
        const float mv[4] = {mm.x, mm.y, mm.z, mm.w};
        const int32_t cv[4] = {cc.x, cc.y, cc.z, cc.w};
        int32_t r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int32_t adj = (int32_t)(v[g / 4][(g % 4) * 4 + k] + ((uint32_t)cv[k] + (uint32_t)zv[k] * (uint32_t)rowsum));
            float x = __fmul_rn(__int2float_rn(adj), mv[k]);
            x = fmaxf(x, RELU ? 0.0f : -8388608.0f);
            r[k] = __float_as_int(__fadd_rn(x, 12582912.0f)) - zoff;
        }
        w[g] = pack_sat_u8(r[1], r[0], pack_sat_u8(r[3], r[2], 0u));
    }
    if (valid) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) dst[c] = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
    }
}

template <int MODE, int KS>  // MODE 0 raw int32, 1 F32_RNE, 2 REF; KS = C / 32 K-steps per tap
__global__ void __launch_bounds__(128 + 32 * EPI_WARPS, 1)
    conv3x3_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const CvParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_addr);
    const CvLayout L = cv_layout(p);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    Q8G_CHECK((uint32_t)L.total <= ptx::dynamic_smem_size());
    // roles: warps 0..EPI_WARPS-1 epilogue (TMEM lane quarter = warp % 4), then
    // the halo producer, MMA issuer 0 (SMSP 1), the TMEM allocator and MMA
    // issuer 1 (SMSP 3): the scheduler favours the highest warp id, so the
    // issue loops are not starved by the ALU-heavy epilogue warps
    constexpr int W_PROD = EPI_WARPS, W_MMA0 = EPI_WARPS + 1, W_ALLOC = EPI_WARPS + 2, W_MMA1 = EPI_WARPS + 3;
    const uint32_t bar0 = base + L.bar_off;
    auto full_bar = [&](int b) { return bar0 + 8u * b; };
    auto empty_bar = [&](int b) { return bar0 + 8u * (MAX_BUF + b); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * MAX_BUF + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * MAX_BUF + MAX_ACC + a); };
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L.tmemptr_off);
    const uint32_t img_bar = bar0 + 8u * (2 * MAX_BUF + 2 * MAX_ACC);
    ptx::griddep_launch_dependents();
#ifdef Q8G_TRACE
    if (threadIdx.x == 0 && p.trace && blockIdx.x < 160) {  // per-CTA entry stamp
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (blockIdx.x == 0) p.trace[8192 + 321] = t;
        p.trace[8704 + blockIdx.x] = t;
    }
#endif

    // ---- guard bands, barriers, then everything overlaps: the producer
    // streams halos while the operand image (B = [weights | ones] + tap weight
    // sums, built once per weight by conv_prep_kernel) lands and the epilogue
    // warps build their correction tables.  The image load is issued after
    // the issuing thread's proxy fence: a fence issued behind it waits for
    // its 46 KB to land (~0.9 us of prologue, tools/conv_trace.py)
    // halo guard bands (windows start one position early / run past the end)
    for (int i = threadIdx.x; i < 64; i += blockDim.x) reinterpret_cast<uint4*>(smem + L.halo_off - 1024)[i] = make_uint4(0, 0, 0, 0);
    for (int b = 0; b < p.nbuf; ++b) {
        uint4* g = reinterpret_cast<uint4*>(smem + L.halo_off + b * L.halo_stride + p.halo_bytes);
        for (int i = threadIdx.x; i < (L.halo_stride - p.halo_bytes) / 16; i += blockDim.x) g[i] = make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) cv_pstamp(p, 3);
    if (threadIdx.x < UNIT_RING)  // tags no unit index matches
        reinterpret_cast<unsigned long long*>(smem + L.ring_off)[threadIdx.x] = ~0ull;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) cv_pstamp(p, 1);
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmap_x);
        ptx::mbar_init(img_bar, 1);
        for (int b = 0; b < p.nbuf; ++b) {
            ptx::mbar_init(full_bar(b), 1);
            ptx::mbar_init(empty_bar(b), 1);
        }
        for (int a = 0; a < MAX_ACC; ++a) {
            ptx::mbar_init(tfull_bar(a), 1);
            ptx::mbar_init(tempty_bar(a), 4);  // the 4 warps of the unit's warpgroup
        }
        ptx::fence_mbar_init();
        // the image is immutable once an earlier call built it: fetch it while
        // the previous grid drains (PDL); a fresh one waits for conv_prep_kernel
        if (p.img_prefetch) {
            ptx::mbar_arrive_expect_tx(img_bar, (uint32_t)p.img_bytes);
            ptx::bulk_load(base + L.b_off, p.img, (uint32_t)p.img_bytes, img_bar);
        }
        cv_pstamp(p, 0);
    }
    if (warp == W_ALLOC) {
        ptx::tmem_alloc<512>(ptx::smem_u32(tmem_ptr));
        if (lane == 0) cv_pstamp(p, 2);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_ptr;
    // PDL: x is read (producer) and y written (epilogue) only after
    // griddepcontrol.wait; the MMA warp touches only smem / TMEM
#ifdef Q8G_TRACE
    if (threadIdx.x == 0 && p.trace && blockIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8192 + 320] = t;
    }
#endif

    if (warp == W_PROD) {
        // ------------------------------------------------ halo producer
        // Schedule: the first p.nstatic units of every CTA are static
        // (blockIdx.x + i * gridDim.x, all issued at once); the rest are
        // claimed one at a time from the launch's work slot (counter value c
        // -> unit nstatic * gridDim.x + c), each only once the MMA of the unit
        // DYN_LEAD places earlier has completed.  A CTA then holds at most
        // DYN_LEAD units when the counter runs out, so CTAs that entered late
        // (their SM was still running the previous grid) take fewer units and
        // the grid's CTAs finish together.  The lead covers the claim's
        // atomic round trip (~0.8 us under contention) plus the halo load.
        const int lead = p.nbuf < DYN_LEAD ? p.nbuf : DYN_LEAD;  // <= nbuf: no phase aliasing
        ptx::griddep_wait();
        if (!p.img_prefetch && ptx::elect_one()) {  // image built by this call's conv_prep_kernel
            ptx::mbar_arrive_expect_tx(img_bar, (uint32_t)p.img_bytes);
            ptx::bulk_load(base + L.b_off, p.img, (uint32_t)p.img_bytes, img_bar);
        }
        __syncwarp();
        const uint32_t ring = base + L.ring_off;
        int i = 0;
        // dynamic units: group g = blockIdx % kWorkGroups claims units
        // nstatic * grid + g + kWorkGroups * c from its own counter
        const int wg = (int)blockIdx.x % kWorkGroups;
        for (;; ++i) {
            int u = (int)blockIdx.x + i * (int)gridDim.x;
            if (p.work && i >= p.nstatic) {
                if (i >= lead) {  // the MMA of unit i - lead has completed
                    const int j = i - lead;
                    ptx::mbar_wait(empty_bar(j % p.nbuf), (uint32_t)(j / p.nbuf) & 1u);
                }
                if (lane == 0) u = p.nstatic * (int)gridDim.x + wg + kWorkGroups * atomicAdd(p.work + 8 * wg, 1);
                u = __shfl_sync(0xffffffffu, u, 0);
            }
            if (u >= p.units) break;
            const int b = i % p.nbuf;
            ptx::mbar_wait(empty_bar(b), ((uint32_t)(i / p.nbuf) & 1u) ^ 1u);
            const int n = u / p.rblocks, rb = u % p.rblocks;
            if (ptx::elect_one()) {
                ring_put(ring + 8u * (uint32_t)(i % UNIT_RING), i, u + 1);
                // one 4D TMA: (ROWS+2) rows x (W+2) positions x C bytes, natural
                // NHWC order, hardware swizzle of span C, out-of-image taps zero
                ptx::mbar_arrive_expect_tx(full_bar(b), (uint32_t)p.halo_bytes);
                tma_load_4d(base + L.halo_off + b * L.halo_stride, &tmap_x, 0, -1, rb * ROWS - 1, n, full_bar(b));
                cv_stamp(p, 0, i);
            }
            __syncwarp();
        }
        if (lane == 0) {
            // "no more units" for both parities (MMA warps / epilogue warpgroups
            // take alternate units)
            ring_put(ring + 8u * (uint32_t)(i % UNIT_RING), i, 0);
            ring_put(ring + 8u * (uint32_t)((i + 1) % UNIT_RING), i + 1, 0);
            if (p.work) {
                // every CTA has made its last claim when done reaches the grid
                // size: the last one zeroes the slot for its next use
                __threadfence();
                if (atomicAdd(p.work + kWorkDone, 1) == (int)gridDim.x - 1) {
                    for (int g = 0; g < kWorkGroups; ++g) atomicExch(p.work + 8 * g, 0);
                    atomicExch(p.work + kWorkDone, 0);
                }
            }
        }
        __syncwarp();
    } else if (warp == W_MMA0 || warp == W_MMA1) {
        // ------------------------------------------------ MMA issuer
        // The whole warp runs the loop (warp-uniform control flow) and one
        // elected lane issues: every descriptor is then a uniform-register
        // add off two bases (tap (kh, kw), K-step j: the A window starts
        // kh rows + kw positions into the halo), so consecutive tcgen05.mma
        // issue back to back.  (Per-lane loops over precomputed descriptor
        // arrays compiled to R2UR moves + an ELECT loop per MMA: ~70 cycles
        // of issue per MMA, slower than the tensor pipe.)
        const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(p.nq >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t row16 = (uint64_t)(p.wp * 2 * KS);  // one halo row (wp positions x C bytes) in 16-byte units
        const uint64_t pos16 = (uint64_t)(2 * KS);         // one position
        const uint64_t bstep = (uint64_t)(2 * p.nq);       // one (tap, K-step) block of B: 2 halves x nq rows x 16 B
        const uint64_t b0 = kmajor_noswz_desc(base + L.b_off, (uint32_t)(p.nq * 16), 128);
        const uint64_t a0 = kmajor_swz_desc(0u, p.c);
        // two issuing warps on different SMSPs (1 and 3) take alternate units:
        // each shares its SMSP with an epilogue warp, and a busy neighbour
        // delays a warp's next issue (tools/mma_desc.cu); with two, one of
        // them usually has the next unit's MMAs queued
        const int q = warp == W_MMA0 ? 0 : 1;
        ptx::mbar_wait(img_bar, 0);
        const uint32_t ring = base + L.ring_off;
        for (int ui = q;; ui += 2) {
            if (ring_get(ring + 8u * (uint32_t)(ui % UNIT_RING), ui) == 0) break;
            const int b = ui % p.nbuf, acc = ui % p.nacc;
            const uint32_t ph = (uint32_t)(ui / p.nbuf) & 1u, aph = (uint32_t)(ui / p.nacc) & 1u;
            ptx::mbar_wait(tempty_bar(acc), aph ^ 1);
            if (lane == 0) cv_stamp(p, 5, ui);
            ptx::mbar_wait(full_bar(b), ph);
            if (lane == 0) cv_stamp(p, 6, ui);
            ptx::tc_fence_after();
            // start-address field of halo position -1 (windows start one early)
            const uint64_t ahalo = a0 + ((base + L.halo_off + b * L.halo_stride - (uint32_t)p.c) >> 4);
            const uint32_t d = tmem_base + (uint32_t)(acc * p.acc_cols);
            if (ptx::elect_one()) {
                cv_stamp(p, 1, ui);
#pragma unroll
                for (int t = 0; t < 9; ++t)
#pragma unroll
                    for (int j = 0; j < KS; ++j)
                        ptx::mma_i8(d, ahalo + (uint64_t)(t / 3) * row16 + (uint64_t)(t % 3) * pos16 + 2u * j,
                                    b0 + (uint64_t)(t * KS + j) * bstep, idesc, (t | j) != 0);
                ptx::tc_commit(empty_bar(b));
                ptx::tc_commit(tfull_bar(acc));
                cv_stamp(p, 2, ui);
            }
            __syncwarp();
        }
    } else if (warp < EPI_WARPS) {
        // ------------------------------------------------ epilogue
        // warpgroup wg (warps 4-7 / 8-11) owns TMEM buffer wg = every other unit
        const int wg = warp / 4;
        const int quarter = warp % 4;
        const int r = quarter * 32 + lane;  // position within the unit's tile
        const int orow = r / p.wp, ocol = r % p.wp - 1;
        const int4* rec_s = reinterpret_cast<const int4*>(smem + L.rec_off);
        const int32_t* corr = reinterpret_cast<const int32_t*>(smem + L.corr_off);
        {
            // per-CTA tables: corr[class][n] = c[n] + zp_a * sum over the
            // class's padded taps of (tap weight sum - C*zp_b[n]); SoA copies
            const int et = threadIdx.x;
            ptx::mbar_wait(img_bar, 0);
            const int32_t* wsum = reinterpret_cast<const int32_t*>(smem + L.wsum_off);
            int32_t* corr_w = reinterpret_cast<int32_t*>(smem + L.corr_off);
            for (int idx = et; idx < 16 * p.oc_pad; idx += 32 * EPI_WARPS) {
                const int cls = idx / p.oc_pad, n = idx % p.oc_pad;
                int64_t s = 0;
                if (cls != 0 && n < p.oc) {
                    const int32_t zpb = MODE == 0 ? 0 : p.rec[n].zpb;
                    for (int t = 0; t < 9; ++t) {
                        const int kh = t / 3, kw = t % 3;
                        const bool padded = ((cls & 1) && kh == 0) || ((cls & 2) && kh == 2) ||
                                            ((cls & 4) && kw == 0) || ((cls & 8) && kw == 2);
                        if (padded) s += (int64_t)wsum[t * p.oc_pad + n] - (int64_t)p.c * zpb;
                    }
                }
                const int32_t c_n = (MODE == 0 || n >= p.oc) ? 0 : p.rec[n].c;
                corr_w[idx] = (int32_t)((uint32_t)(uint64_t)(s * p.zp_a) + (uint32_t)c_n);
            }
            if (MODE != 0)
                for (int n = et; n < p.oc_pad; n += 32 * EPI_WARPS) {
                    const int4 r4 = n < p.oc ? __ldg(reinterpret_cast<const int4*>(p.rec + n)) : make_int4(0, 0, 0, 0);
                    reinterpret_cast<int4*>(smem + L.rec_off)[n] = r4;
                    reinterpret_cast<int32_t*>(smem + L.soa_off)[n] = (int32_t)(0u - (uint32_t)r4.y);  // -zp_b
                    reinterpret_cast<int32_t*>(smem + L.soa_off)[p.oc_pad + n] = r4.z;  // fp32 multiplier bits
                }
            asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
        }
        ptx::griddep_wait();  // y may be read / written by the previous grid
        // requant + store of up to 64 columns (+ row sum) of one position
        auto process = [&](const uint32_t (&v4)[4][16], int nchunk, int ch0, int32_t rowsum, int cls, bool valid,
                           size_t pix) {
                if (MODE == 1 && p.fast && (p.oc % 16) == 0) {
                    const int4* nzq = reinterpret_cast<const int4*>(smem + L.soa_off) + ch0 / 4;
                    const float4* mq = reinterpret_cast<const float4*>(smem + L.soa_off + p.oc_pad * 4) + ch0 / 4;
                    const int4* cq = reinterpret_cast<const int4*>(corr + cls * p.oc_pad + ch0);
                    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.y) + pix * p.oc + ch0);
                    const int32_t zoff = 0x4B400000 - p.zp_c;
#define Q8G_EPI_FAST(R)                                                                   \
    (nchunk == 4   ? epi_f32_fast<R, 4>(v4, rowsum, nzq, mq, cq, zoff, dst, valid)     \
     : nchunk == 3 ? epi_f32_fast<R, 3>(v4, rowsum, nzq, mq, cq, zoff, dst, valid)     \
     : nchunk == 2 ? epi_f32_fast<R, 2>(v4, rowsum, nzq, mq, cq, zoff, dst, valid)     \
                   : epi_f32_fast<R, 1>(v4, rowsum, nzq, mq, cq, zoff, dst, valid))
                    if (p.relu)
                        Q8G_EPI_FAST(true);
                    else
                        Q8G_EPI_FAST(false);
#undef Q8G_EPI_FAST
                    return;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (k >= nchunk) break;
                    const uint32_t (&v)[16] = v4[k];
                    const int ch = ch0 + 16 * k;
                    if (!valid) continue;
                    const int32_t* crow = corr + cls * p.oc_pad + ch;
                    if (MODE == 0) {
                        int32_t* dst = reinterpret_cast<int32_t*>(p.y) + pix * p.oc + ch;
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (ch + j < p.oc) dst[j] = (int32_t)(v[j] + (uint32_t)crow[j]);
                        continue;
                    }
                    uint8_t* dst = reinterpret_cast<uint8_t*>(p.y) + pix * p.oc + ch;
                    uint32_t q[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int4 r4 = rec_s[ch + j];
                        EpiRecord rc;
                        rc.c = crow[j];  // c[n] + class correction
                        rc.zpb = r4.y;
                        const int32_t adj = adjust((int32_t)v[j], rowsum, rc);
                        q[j] = MODE == 1 ? requant_f32(adj, __int_as_float(r4.z), p.zp_c, p.relu)
                                         : requant_ref(adj, __hiloint2double(r4.w, r4.z), p.zp_c, p.relu);
                    }
                    if (ch + 16 <= p.oc && (p.oc % 16) == 0) {
                        uint4 o;
                        o.x = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
                        o.y = q[4] | (q[5] << 8) | (q[6] << 16) | (q[7] << 24);
                        o.z = q[8] | (q[9] << 8) | (q[10] << 16) | (q[11] << 24);
                        o.w = q[12] | (q[13] << 8) | (q[14] << 16) | (q[15] << 24);
                        *reinterpret_cast<uint4*>(dst) = o;
                    } else {
                        for (int j = 0; j < 16; ++j)
                            if (ch + j < p.oc) dst[j] = (uint8_t)q[j];
                    }
                }
        };
        const uint32_t ring = base + L.ring_off;
        for (int i = wg;; i += 2) {
            const int u = ring_get(ring + 8u * (uint32_t)(i % UNIT_RING), i) - 1;
            if (u < 0) break;
            const int acc = i % p.nacc;
            const uint32_t aph = (uint32_t)(i / p.nacc) & 1u;
            const int n = u / p.rblocks, rb = u % p.rblocks;
            const int oh = rb * ROWS + orow;
            const bool valid = orow < ROWS && oh < p.h && ocol >= 0 && ocol < p.w;
            const int cls = (oh == 0 ? 1 : 0) | (oh == p.h - 1 ? 2 : 0) | (ocol == 0 ? 4 : 0) | (ocol == p.w - 1 ? 8 : 0);
            const size_t pix = ((size_t)n * p.h + oh) * p.w + ocol;
            Q8G_CHECK(u < p.units && (!valid || pix < (size_t)p.nb * p.h * p.w));
            ptx::mbar_wait(tfull_bar(acc), aph);
            ptx::tc_fence_after();
            if (quarter == 0 && lane == 0) cv_stamp(p, 3, i);
            const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * p.acc_cols);
            int32_t rowsum = 0;
            for (int ch0 = 0; ch0 < p.oc_pad; ch0 += 64) {
                // up to 64 columns (+ the row-sum column) in flight, one wait
                uint32_t v4[4][16], rs[16];
                const int nchunk = (p.oc_pad - ch0) >= 64 ? 4 : (p.oc_pad - ch0) / 16;
                if (ch0 == 0) ptx::tmem_ld_32x32b_x16(lane_base + (uint32_t)p.oc_pad, rs);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k < nchunk) ptx::tmem_ld_32x32b_x16(lane_base + (uint32_t)(ch0 + 16 * k), v4[k]);
                ptx::tmem_ld_wait();
                if (ch0 == 0) rowsum = (int32_t)rs[0];
#ifdef Q8G_TRACE
                if (ch0 == 0 && quarter == 0 && lane == 0 && p.trace && blockIdx.x == 0 && i < 64) {
                    unsigned long long tt;  // debug: TMEM loads landed
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
                    p.trace[8192 + 384 + i] = tt;
                }
#endif
                process(v4, nchunk, ch0, rowsum, cls, valid, pix);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty_bar(acc));
            if (quarter == 0 && lane == 0) cv_stamp(p, 4, i);
        }
    }

    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == W_ALLOC) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem_base);
    }
#ifdef Q8G_TRACE
    if (threadIdx.x == 0 && p.trace && blockIdx.x < 160) {  // per-CTA exit stamp
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8704 + 160 + blockIdx.x] = t;
    }
#endif
}

CvParams make_params(const ConvArgs& a) {
    CvParams p{};
    p.nb = a.nb;
    p.h = a.h;
    p.w = a.w;
    p.c = a.c;
    p.oc = a.pw->n;
    p.wp = a.w + 2;
    p.planes = a.c / 16;
    p.oc_pad = align_up(p.oc, 16);
    p.nq = p.oc_pad + 16;
    p.rblocks = (a.h + ROWS - 1) / ROWS;
    p.units = a.nb * p.rblocks;
    p.nacc = p.nq <= 128 ? MAX_ACC : 2;  // 512 TMEM columns
    p.acc_cols = 512 / p.nacc;
    p.halo_bytes = (ROWS + 2) * p.wp * p.c;
    p.pb = a.pw->data;
    p.np = a.pw->np;
    p.img = nullptr;
    p.img_bytes = 9 * (p.planes / 2) * 2 * p.nq * 16 + 9 * p.oc_pad * 4;
    p.rec = a.raw ? nullptr : a.ep->rec;
    p.zp_a = a.zp_a;
    p.zp_c = a.raw ? 0 : a.ep->zp_c;
    p.relu = a.raw ? 0 : a.ep->relu;
    p.rounding = a.raw ? 0 : a.ep->rounding;
    p.fast = (!a.raw && a.ep->fast_f32) ? 1 : 0;
    p.y = a.y;
    p.trace = tc_trace_buffer_ptr();
    // 5 halo buffers (fewer if they do not fit next to the operand image, >= 2).
    // C3 over Q8G_CONV_NBUF = 2..8: 10.4 / 10.8 / 11.1 / 9.0-9.1 / 9.3 / 9.35-9.4
    // / 9.4-9.5 us; a CTA running further ahead of its neighbours loses the
    // L2 sharing of their common halo rows (as in the depthwise kernel)
    int maxbuf = 5;
    if (const char* e = getenv("Q8G_CONV_NBUF")) maxbuf = std::max(2, std::min(MAX_BUF, std::atoi(e)));
    for (p.nbuf = maxbuf; p.nbuf > 2 && cv_layout(p).total > 232448; --p.nbuf) {
    }
    return p;
}

}  // namespace

bool conv_tc_supported(const ConvArgs& a) {
    if (tmap_encoder() == nullptr) return false;
    if (a.c % 32 != 0 || (a.c != 32 && a.c != 64 && a.c != 128) || a.pw->n > 240 || a.w + 2 > 256) return false;
    if (ROWS * (a.w + 2) > 128) return false;  // one M tile per unit
    const CvParams p = make_params(a);
    if (p.nq * 2 > 512 || p.nq > 256) return false;
    return cv_layout(p).total <= 232448;
}

cudaError_t conv_tc_prepare(const q8g_packed_b* pwc, int c, cudaStream_t s) {
    if (c != 32 && c != 64 && c != 128) return cudaSuccess;  // not an implicit-GEMM shape: no image
    static std::mutex mu;
    const int slot = c == 32 ? 0 : c == 64 ? 1 : 2;
    auto* pw = const_cast<q8g_packed_b*>(pwc);  // the image is a cache of derived data, not the weight
    std::lock_guard<std::mutex> lock(mu);
    if (__atomic_load_n(&pw->conv_img_ready[slot], __ATOMIC_ACQUIRE)) return cudaSuccess;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusNone) return cudaErrorStreamCaptureUnsupported;  // prepare before capturing
    if (const cudaError_t e = work_slot_prepare(pw->device); e != cudaSuccess) return e;
    ConvArgs a{};
    a.nb = 1;
    a.h = 8;
    a.w = 8;
    a.c = c;
    a.pw = pw;
    a.raw = true;
    const CvParams p = make_params(a);
    uint8_t* img = nullptr;
    cudaError_t e = cudaMalloc(&img, (size_t)p.img_bytes);
    if (e != cudaSuccess) return e;
    conv_prep_kernel<<<64, 256, 0, s>>>(p, img);
    count_launch(kFamPack);
    if ((e = cudaGetLastError()) == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        cudaFree(img);
        return e;
    }
    pw->conv_img[slot] = img;
    __atomic_store_n(&pw->conv_img_ready[slot], 1, __ATOMIC_RELEASE);
    return cudaSuccess;
}

cudaError_t launch_conv3x3_tc(const ConvArgs& a, cudaStream_t s) {
    auto enc = tmap_encoder();
    CvParams p = make_params(a);
    CUtensorMap tmap;
    cuuint64_t dims[4] = {(cuuint64_t)a.c, (cuuint64_t)a.w, (cuuint64_t)a.h, (cuuint64_t)a.nb};
    cuuint64_t strides[3] = {(cuuint64_t)a.c, (cuuint64_t)a.w * a.c, (cuuint64_t)a.h * a.w * a.c};
    cuuint32_t box[4] = {(cuuint32_t)a.c, (cuuint32_t)(a.w + 2), (cuuint32_t)(ROWS + 2), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(a.x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            a.c == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : a.c == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    const CvLayout L = cv_layout(p);
    int dev = 0;
    cudaGetDevice(&dev);
    // per-weight operand image: built once per (weight, C), synchronously
    // and under a lock, then immutable (conv_tc_prepare)
    const int slot = a.c == 32 ? 0 : a.c == 64 ? 1 : 2;
    if (!__atomic_load_n(&a.pw->conv_img_ready[slot], __ATOMIC_ACQUIRE)) {
        const cudaError_t e = conv_tc_prepare(a.pw, a.c, s);
        if (e != cudaSuccess) return e;
    }
    p.img = a.pw->conv_img[slot];
    p.img_prefetch = 1;
    // dynamic unit claiming (Q8G_CONV_DYN=0: the static round-robin schedule)
    static const bool dyn = [] {
        const char* e = getenv("Q8G_CONV_DYN");
        return !(e && e[0] == '0');
    }();
    int grid = sm_count(dev);
    if (grid > p.units) grid = p.units;
    // static head: all but the last unit of an even share (C3: 5 static + ~1
    // claimed; more claimed units measured slower, the claims contend)
    p.nstatic = std::max(0, p.units / grid - 1);
    if (const char* e = getenv("Q8G_CONV_NSTATIC")) p.nstatic = std::max(0, std::atoi(e));
    if (dyn) {
        p.work = work_slot(dev);
        if (!p.work) {
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            cudaStreamIsCapturing(s, &cs);
            if (cs == cudaStreamCaptureStatusNone && work_slot_prepare(dev) == cudaSuccess) p.work = work_slot(dev);
        }
    }
    const int mode = a.raw ? 0 : (a.ep->rounding == Q8G_ROUND_F32_RNE ? 1 : 2);
    const int ks = a.c / 32;
    const int threads = 128 + 32 * EPI_WARPS;
    // the dynamic-smem attribute once per (kernel variant, device): the
    // attribute call costs host time on every host-view chunk otherwise
    static bool attr[3][3][64] = {};
    const int mi = mode, ki = ks == 1 ? 0 : ks == 2 ? 1 : 2;
    auto go = [&](auto kern) {
        cudaError_t e = cudaSuccess;
        if (dev >= 64 || !attr[mi][ki][dev]) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
            if (e == cudaSuccess && dev < 64) attr[mi][ki][dev] = true;
        }
        if (e == cudaSuccess) e = launch_with_pdl(kern, dim3(grid), dim3(threads), L.total, s, tmap, p);
        return e;
    };
    cudaError_t e;
#define Q8G_CONV_KS(M)                                           \
    (ks == 1 ? go(conv3x3_tc_kernel<M, 1>) : ks == 2 ? go(conv3x3_tc_kernel<M, 2>) \
             : ks == 4 ? go(conv3x3_tc_kernel<M, 4>) : cudaErrorNotSupported)
    if (mode == 0)
        e = Q8G_CONV_KS(0);
    else if (mode == 1)
        e = Q8G_CONV_KS(1);
    else
        e = Q8G_CONV_KS(2);
#undef Q8G_CONV_KS
    if (e != cudaSuccess) return e;
    count_launch(kFamConvTc);
    return cudaGetLastError();
}

}  // namespace q8g
