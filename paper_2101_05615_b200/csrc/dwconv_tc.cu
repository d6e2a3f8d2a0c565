// dwconv_tc.cu — depthwise 3x3 / stride 1 / pad 1 NHWC on the tensor cores
// (BASELINE config C4, the HBM-bound path).
//
// Semantics: SURVEY.md App. A D3 (no reference symbol).  For output (n,h,w,c):
//   adj = sum_t x_t*(w[t,c] - zp_w[c]) + bias[c] - zp_a*wsum[c] + 9*zp_a*zp_w[c]
// with padded taps reading x = zp_a, then the F32_RNE requant.
//
// Design (why it is not a CUDA-core kernel): at 70% of HBM the whole 32x112x
// 112x256 layer has ~45 us, i.e. ~11-16 issue slots per output for 9 MACs,
// the sum_x term and the requant.  Here the MACs and the -zp_w*sum_x term run
// on tcgen05: for a group of 16 channels the depthwise sum is a GEMM with a
// block-diagonal B (K = 9 taps x 16 channels, N = 16), and
//   D = A x W_g + A x Z_g,  Z_g[(t,c), c'] = -zp_w[c'] * delta(c, c')
// accumulates both in the same TMEM tile.  The A operand is never
// materialised: the CTA loads a halo of R+2 input rows (padded width W+2,
// 16 channels per pixel, out-of-range taps zero-filled by TMA) and each MMA
// K-step (two taps) reads two shifted windows of that halo through a
// no-swizzle K-major descriptor whose leading-byte offset is the distance
// between the taps.  The zero-filled padding is corrected exactly per border
// class (corr[class][c] = zp_a * sum_{padded t} (w[t,c] - zp_w[c])).  CUDA
// cores only run the requantization (magic-number float conversions, ~8
// issue slots per output) and the 16-byte stores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "ptx.cuh"
#include "q8g_internal.cuh"

namespace q8g {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();
unsigned long long* tc_trace_buffer_ptr();

namespace {

constexpr int G = 16;          // channels per group (MMA N)
constexpr int TAPS = 10;       // 9 taps + one zero-weight tap (K = 160 = 5 x 32)
constexpr int ROWS = 8;        // output rows per work unit
constexpr int NBUF = 6;        // halo buffers in flight (TMA latency ~3.5 us per 16-B-row halo)
constexpr int MAXW = 254;      // padded width <= 256 (TMA box limit)
constexpr int EPI_WARPS = 8;

struct DwParams {
    int nb, h, w, c;           // NHWC dims
    int wp;                    // padded width w + 2
    int groups;                // c / 16
    int rblocks;               // ceil(h / ROWS)
    int tiles;                 // M tiles of 128 positions per unit
    int units;                 // nb * rblocks * groups
    int halo_bytes;            // (ROWS + 2) * wp * 16
    const int8_t* wt;          // [9][c]
    const int32_t* zpw;        // [c]
    const int32_t* cterm;      // [c]: bias - zp_a*wsum + 9*zp_a*zp_w + float magic bits
    const float* mult;         // [c]
    const int32_t* corr;       // [16][c] border-class corrections
    float lo, hi;              // clamp bounds in the pre-zp_c domain
    int32_t zp_c;
    // 64-channel-block kernel (dwconv_tc64_kernel)
    int nblk;                  // c / 64
    int rb2;                   // ceil(h / 2)
    int units_blk;             // nb * rb2 units per channel block
    int nb2;                   // 64-channel kernel: halo buffers
    uint8_t* y;
    unsigned long long* trace;  // debug (Q8G_TC_TRACE): per-unit stamps of CTA 0, else null
};

// CTA 0, unit i < 64: [8192 + 64*which + i]; which: 0 halo TMA issued, 1 halo
// landed (MMA), 2 MMAs issued, 3 epilogue got the accumulators, 4 epilogue done
__device__ __forceinline__ void dw_stamp(const DwParams& p, int which, int i) {
#ifdef Q8G_TRACE
    if (p.trace && blockIdx.x == 0 && i < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8192 + which * 64 + i] = t;
    }
#endif
}

__host__ __device__ constexpr int align_up(int v, int a) { return (v + a - 1) / a * a; }

// smem layout
struct DwLayout {
    int halo_off, halo_stride, b_off, corr_off, bar_off, tmemptr_off, total;
};
__host__ __device__ inline DwLayout dw_layout(int halo_bytes, int groups) {
    DwLayout L;
    L.halo_off = 1024;  // 1 KB front guard: tap windows may start up to one pixel early
    L.halo_stride = align_up(halo_bytes + 2048, 1024);  // + tail guard for the last tile's rows
    L.b_off = L.halo_off + NBUF * L.halo_stride;
    // per group: B = [W rows 0-15 | Z rows 16-31], TAPS x 32 rows x 16 B
    L.corr_off = L.b_off + groups * TAPS * 2 * G * 16;
    L.bar_off = L.corr_off + 16 * groups * G * 4;  // [16 classes][c] int32
    L.tmemptr_off = L.bar_off + (2 * NBUF + 4) * 8;
    L.total = L.tmemptr_off + 16 + 1024;
    return L;
}

// no-swizzle K-major UMMA descriptor: core matrices of 8 rows x 16 B (rows
// contiguous), SBO between 8-row groups, LBO between the two 16-byte K halves
__device__ __forceinline__ uint64_t kmajor_noswz_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);  // layout type 0 = SWIZZLE_NONE
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    // low bytes of a,b,c,d -> one word
    const uint32_t ab = __byte_perm(a, b, 0x0040);
    const uint32_t cd = __byte_perm(c, d, 0x0040);
    return __byte_perm(ab, cd, 0x5410);
}

__global__ void __launch_bounds__(128 + 32 * EPI_WARPS, 1)
    dwconv_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const DwParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_addr);
    const DwLayout L = dw_layout(p.halo_bytes, p.groups);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    Q8G_CHECK((uint32_t)L.total <= ptx::dynamic_smem_size());
    const uint32_t bar0 = base + L.bar_off;
    auto full_bar = [&](int b) { return bar0 + 8u * b; };
    auto empty_bar = [&](int b) { return bar0 + 8u * (NBUF + b); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * NBUF + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * NBUF + 2 + a); };
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L.tmemptr_off);
    ptx::griddep_launch_dependents();

    // global-memory-free prologue first (overlaps the previous grid under PDL)
    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_x);
        for (int b = 0; b < NBUF; ++b) {
            ptx::mbar_init(full_bar(b), 1);
            ptx::mbar_init(empty_bar(b), 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull_bar(a), 1);
            ptx::mbar_init(tempty_bar(a), EPI_WARPS);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc<512>(ptx::smem_u32(tmem_ptr));
    // (filter tables are immutable: built before griddepcontrol.wait, PDL)

    // ---- block-diagonal B = [W | Z] for every channel group (built once):
    // rows 0-15 W[t][c'] on the diagonal, rows 16-31 -zp_w[c'] on the diagonal
    for (int idx = threadIdx.x; idx < p.groups * TAPS * 2 * G; idx += blockDim.x) {
        const int g = idx / (TAPS * 2 * G), rem = idx % (TAPS * 2 * G);
        const int t = rem / (2 * G), row = rem % (2 * G);
        const int oc = row % G;  // output channel within the group
        const int ch = g * G + oc;
        uint32_t v[4] = {0, 0, 0, 0};
        if (t < 9) {
            const uint32_t byte = row < G ? (uint32_t)(uint8_t)p.wt[t * p.c + ch]
                                          : (uint32_t)(uint8_t)(int8_t)(-p.zpw[ch]);
            v[oc / 4] = byte << (8 * (oc % 4));
        }
        // [g][tap][row][16 B]
        *reinterpret_cast<uint4*>(smem + L.b_off + ((g * TAPS + t) * 2 * G + row) * 16) =
            make_uint4(v[0], v[1], v[2], v[3]);
    }
    // per border class: cterm (bias, offsets, float magic) + padding correction
    for (int i = threadIdx.x; i < 16 * p.c; i += blockDim.x)
        reinterpret_cast<int32_t*>(smem + L.corr_off)[i] = p.corr[i] + p.cterm[i % p.c];
    // the halo guards must hold finite data (they only feed garbage rows)
    for (int i = threadIdx.x; i < L.b_off / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_ptr;
    const int per_img = p.rblocks * p.groups;

    if (warp == 0) {
        // ------------------------------------------------ halo producer
        ptx::griddep_wait();  // x may be the previous grid's output
        // (whole warp runs the loop; one elected lane issues)
        {
            int b = 0;
            uint32_t ph = 0;
            for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
                const int n = u / per_img, rem = u % per_img;
                const int rb = rem / p.groups, g = rem % p.groups;
                ptx::mbar_wait(empty_bar(b), ph ^ 1);
                if (ptx::elect_one()) {
                    ptx::mbar_arrive_expect_tx(full_bar(b), (uint32_t)p.halo_bytes);
                    // box {16 ch, wp px, ROWS+2 rows, 1}: starts at (row r0-1, col -1)
                    tma_load_4d(base + L.halo_off + b * L.halo_stride, &tmap_x, g * G, -1, rb * ROWS - 1, n,
                                full_bar(b));
                    dw_stamp(p, 0, (u - (int)blockIdx.x) / (int)gridDim.x);
                }
                __syncwarp();
                if (++b == NBUF) {
                    b = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        // (whole warp runs the loop with warp-uniform descriptors; one elected
        // lane issues the tcgen05 instructions)
        {
            constexpr uint32_t idesc = ptx::idesc_u8s8_s32<128, 2 * G>();  // N = 32: [W | Z]
            // descriptor templates: A for K-step s (taps 2s, 2s+1) relative to
            // halo position 0 -- tap t reads halo position q + (t/3)*wp + t%3 - 1,
            // tap 9 has zero weights and reuses the next pixel; B per K-step
            uint64_t a_t[TAPS / 2], b_t[TAPS / 2];
#pragma unroll
            for (int s = 0; s < TAPS / 2; ++s) {
                const int t0 = 2 * s, t1 = 2 * s + 1;
                const int sh0 = (t0 / 3) * p.wp + (t0 % 3) - 1;
                const int sh1 = t1 < 9 ? (t1 / 3) * p.wp + (t1 % 3) - 1 : sh0 + 1;
                // +1: keep the template's start field non-negative (sh0 >= -1);
                // the per-tile base below is one position earlier to compensate
                a_t[s] = kmajor_noswz_desc((uint32_t)((sh0 + 1) * 16), (uint32_t)((sh1 - sh0) * 16), 128);
                // B: per tap 32 rows x 16 B = 512 B; K-step s = taps 2s, 2s+1
                b_t[s] = kmajor_noswz_desc((uint32_t)(s * 2 * (2 * G) * 16), 2 * G * 16, 128);
            }
            int b = 0, acc = 0;
            uint32_t ph = 0, aph = 0;
            for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
                const int g = (u % per_img) % p.groups;
                ptx::mbar_wait(tempty_bar(acc), aph ^ 1);
                ptx::mbar_wait(full_bar(b), ph);
                ptx::tc_fence_after();
                const int ui = (u - (int)blockIdx.x) / (int)gridDim.x;
                if (lane == 0) dw_stamp(p, 1, ui);
                // start-address fields are in 16-byte units (low 14 bits)
                const uint64_t halo16 = (base + L.halo_off + b * L.halo_stride) >> 4;
                const uint64_t b16 = (base + L.b_off + g * TAPS * 2 * G * 16) >> 4;
                for (int tile = 0; tile < p.tiles; ++tile) {
                    // accumulator: 32 columns per tile (16 acc + 16 -zp_w*sum_x)
                    const uint32_t d = tmem_base + (uint32_t)(acc * 256 + tile * 2 * G);
                    const uint64_t a16 = halo16 - 1 + (uint64_t)(tile * 128);  // 128 positions x 16 B
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int s = 0; s < TAPS / 2; ++s)
                            ptx::mma_i8(d, a_t[s] + a16, b_t[s] + b16, idesc, s != 0);
                    }
                    __syncwarp();
                }
                if (ptx::elect_one()) {
                    ptx::tc_commit(empty_bar(b));
                    ptx::tc_commit(tfull_bar(acc));
                    dw_stamp(p, 2, ui);
                }
                __syncwarp();
                if (++b == NBUF) {
                    b = 0;
                    ph ^= 1;
                }
                if (++acc == 2) {
                    acc = 0;
                    aph ^= 1;
                }
            }
        }
    } else if (warp == 2) {
        // (TMEM allocator; idle during the main loop)
    } else if (warp >= 4) {
        // ------------------------------------------------ requant epilogue
        ptx::griddep_wait();  // y may be read / written by the previous grid
        const int ew = warp - 4;          // 0..7
        const int quarter = ew % 4;       // TMEM lanes [32*quarter, +32)
        const int half = ew / 4;          // even / odd tiles
        const int r = quarter * 32 + lane;
        const float magic = 12582912.0f;  // 1.5 * 2^23
        // this thread's output position in each of its tiles (unit-independent)
        int t_orow[4], t_ocol[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int q = (half + 2 * i) * 128 + r;
            t_orow[i] = q / p.wp;
            t_ocol[i] = q % p.wp - 1;
        }
        // with a zero clamp floor (ReLU) every packed byte r satisfies
        // r + zp_c <= 255, so zp_c is added once per packed word (no carries)
        const bool relu_fast = p.lo == 0.0f;
        const uint32_t zp4 = relu_fast ? (uint32_t)p.zp_c * 0x01010101u : 0u;
        const uint32_t zp1 = relu_fast ? 0u : (uint32_t)p.zp_c;
        const int32_t* corr_s = reinterpret_cast<const int32_t*>(smem + L.corr_off);
        int acc = 0;
        uint32_t aph = 0;
        for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
            const int n = u / per_img, rem = u % per_img;
            const int rb = rem / p.groups, g = rem % p.groups;
            const int c0 = g * G;
            float mf[G];
#pragma unroll
            for (int j = 0; j < G; ++j) mf[j] = __ldg(p.mult + c0 + j);
            ptx::mbar_wait(tfull_bar(acc), aph);
            ptx::tc_fence_after();
            const int ui = (u - (int)blockIdx.x) / (int)gridDim.x;
            if (ew == 0 && lane == 0) dw_stamp(p, 3, ui);
            // requantize one tile's 16 channels for this thread's position
            auto emit = [&](const uint32_t (&v)[2 * G], int i) {
                const int orow = t_orow[i], ocol = t_ocol[i];
                const int oh = rb * ROWS + orow;
                if (orow >= ROWS || oh >= p.h || ocol < 0 || ocol >= p.w) return;
                const int cls = (oh == 0 ? 1 : 0) | (oh == p.h - 1 ? 2 : 0) | (ocol == 0 ? 4 : 0) |
                                (ocol == p.w - 1 ? 8 : 0);
                // class row = cterm (+ zero-padding correction), float magic bits folded in
                const int4* crow = reinterpret_cast<const int4*>(corr_s + cls * p.c + c0);
                uint32_t qv[G];
#pragma unroll
                for (int j4 = 0; j4 < G / 4; ++j4) {
                    const int4 cc = crow[j4];
                    const int32_t cj[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int j = j4 * 4 + k;
                        const int32_t bits = (int32_t)(v[j] + v[G + j]) + cj[k];
                        float x = __fmul_rn(__fsub_rn(__int_as_float(bits), magic), mf[j]);
                        x = fminf(fmaxf(x, p.lo), p.hi);
                        qv[j] = (uint32_t)__float_as_int(__fadd_rn(x, magic)) + zp1;
                    }
                }
                uint4 out;
                out.x = pack4(qv[0], qv[1], qv[2], qv[3]) + zp4;
                out.y = pack4(qv[4], qv[5], qv[6], qv[7]) + zp4;
                out.z = pack4(qv[8], qv[9], qv[10], qv[11]) + zp4;
                out.w = pack4(qv[12], qv[13], qv[14], qv[15]) + zp4;
                uint8_t* dst = p.y + ((((size_t)n * p.h + oh) * p.w + ocol) * p.c + c0);
                *reinterpret_cast<uint4*>(dst) = out;
            };
            // two tiles' TMEM loads in flight per step (ILP)
#pragma unroll
            for (int i = 0; i < 4; i += 2) {
                const int ta = half + 2 * i, tb = ta + 2;
                if (ta >= p.tiles) break;  // warp-uniform
                uint32_t va[2 * G], vb[2 * G];  // [0,16): sum x*w, [16,32): -zp_w * sum x
                const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * 256);
                ptx::tmem_ld_32x32b_x32(lane_base + (uint32_t)(ta * 2 * G), va);
                if (tb < p.tiles) ptx::tmem_ld_32x32b_x32(lane_base + (uint32_t)(tb * 2 * G), vb);
                ptx::tmem_ld_wait();
                emit(va, i);
                if (tb < p.tiles) emit(vb, i + 1);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty_bar(acc));
            if (ew == 0 && lane == 0) dw_stamp(p, 4, ui);
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
    }

    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem_base);
    }
}


// ---------------------------------------------------------------- 64-channel blocks
// The 16-channel kernel above loads its halo as 16-byte TMA box rows
// (~3 cycles each; 1140 per unit -> ~1.8 us per unit of TMA time, the
// measured bound).  Here a CTA owns one block of 64 channels for its whole
// life: the halo is the natural NHWC rows of that block (64-byte TMA rows,
// SWIZZLE_64B, 456 per unit), and one MMA step is K = 32 channels of ONE tap:
// the A window of tap t = the halo rows shifted by (t/3)*(W+2) + t%3 - 1,
// bytes 32j.. of each row (a swizzled K-major descriptor at any row: the
// tensor core applies the swizzle on absolute smem addresses, see
// tools/swz_test.cu).  B per (tap, K-group) is block-diagonal [W_t | -zp_w]
// (N = 64), so D = sum_t x_t*w_t (columns 0-31) and -zp_w*sum_t x_t (32-63).
constexpr int CB = 64;      // channels per block: halo row bytes (SWIZZLE_64B)
constexpr int R2 = 2;       // output rows per unit, one 128-position M tile each
constexpr int NB2 = 5;      // halo buffers at most (p.nb2, dw2_nbuf: 3 by default)
constexpr int KG = CB / 32; // K-groups of 32 channels
constexpr int N2 = 64;      // MMA N: 32 outputs + 32 zero-point columns
constexpr int EPI64 = 4 * R2 * KG;  // epilogue warps: (row, K-group) x TMEM lane quarter

struct Dw2Layout {
    int halo_off, halo_stride, b_off, corr_off, mult_off, out_off, out_stride, bar_off, tmemptr_off, total;
};
__host__ __device__ inline Dw2Layout dw2_layout(int wp, int nb2) {
    Dw2Layout L;
    L.halo_off = 1024;  // (front guard; the 64-channel kernel's windows start at the halo)
    L.halo_stride = align_up((R2 + 2) * wp * CB + 1024, 1024);  // + tail guard: the last row's windows read 16 positions past it
    L.b_off = L.halo_off + nb2 * L.halo_stride;
    L.corr_off = L.b_off + 9 * KG * 2048;  // B: [tap][K-group][K half][64 rows][16 B]
    L.mult_off = L.corr_off + 16 * CB * 4;  // [16 classes][64] int32: cterm + border correction
    // per epilogue warp, double-buffered: its 32 positions x 32 channels
    // (32 rows of 32 B, SWIZZLE_32B) for its own TMA store
    L.out_off = align_up(L.mult_off + CB * 4, 1024);
    L.out_stride = 2 * 1024;  // per warp
    L.bar_off = L.out_off + EPI64 * L.out_stride;
    L.tmemptr_off = L.bar_off + (2 * NB2 + 4) * 8;
    L.total = L.tmemptr_off + 16 + 1024;
    return L;
}

__host__ __device__ inline uint64_t kmajor_swz64_desc(uint32_t addr) {
    return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)4 << 61);  // SWIZZLE_64B, 8-row groups of 512 B
}

// d = {c[15:0], sat_u8(a), sat_u8(b)} (one I2IP)
__device__ __forceinline__ uint32_t pack_sat_u8(int32_t a, int32_t b, uint32_t c) {
    uint32_t d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// (image, row block) of a CTA's units k = first, first + step, ...: stepped
// incrementally (no integer division per unit in the role loops)
struct UnitWalk {
    int n, rb, dn, drb, rb2;
    __device__ UnitWalk(int first, int step, int rb2_) : n(first / rb2_), rb(first % rb2_), dn(step / rb2_),
                                                         drb(step % rb2_), rb2(rb2_) {}
    __device__ __forceinline__ void next() {
        n += dn;
        rb += drb;
        if (rb >= rb2) {
            rb -= rb2;
            ++n;
        }
    }
};

__global__ void __launch_bounds__(128 + 32 * EPI64, 1)
    dwconv_tc64_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_y,
                       const DwParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = ptx::smem_u32(smem_raw);
    const uint32_t base = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw_addr);
    const Dw2Layout L = dw2_layout(p.wp, p.nb2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    Q8G_CHECK((uint32_t)L.total <= ptx::dynamic_smem_size() && p.nb2 >= 2 && p.nb2 <= NB2);
    const uint32_t bar0 = base + L.bar_off;
    auto full_bar = [&](int b) { return bar0 + 8u * b; };
    auto empty_bar = [&](int b) { return bar0 + 8u * (NB2 + b); };
    auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * NB2 + a); };
    auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * NB2 + 2 + a); };
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L.tmemptr_off);
    // this CTA's channel block and its share of the block's units
    const int cb = blockIdx.x % p.nblk;
    const int cta_in = blockIdx.x / p.nblk;
    const int ctas = ((int)gridDim.x - cb + p.nblk - 1) / p.nblk;
    const int c0 = cb * CB;
    ptx::griddep_launch_dependents();

    // roles: warps 0..EPI64-1 epilogue (TMEM lane quarter = warp % 4), then the
    // halo producer, the TMEM allocator, an idle warp and the MMA issuer last:
    // the warp scheduler favours the highest warp id, so the single-thread MMA
    // issue loop is not starved by the ALU-heavy epilogue warps of its SMSP
    constexpr int W_PROD = EPI64, W_ALLOC = EPI64 + 1, W_MMA = EPI64 + 3;
    if (warp == W_PROD && lane == 0) {
        ptx::prefetch_tmap(&tmap_x);
        ptx::prefetch_tmap(&tmap_y);
        for (int b = 0; b < p.nb2; ++b) {
            ptx::mbar_init(full_bar(b), 1);
            ptx::mbar_init(empty_bar(b), 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull_bar(a), 1);
            ptx::mbar_init(tempty_bar(a), EPI64);
        }
        ptx::fence_mbar_init();
    }
    if (warp == W_ALLOC) ptx::tmem_alloc<512>(ptx::smem_u32(tmem_ptr));
    // (filter tables are immutable: built before griddepcontrol.wait, PDL)

    // ---- B for this channel block, per (kw, K-group): [K half][192 rows][16 B],
    // rows [64 kh, 64 kh + 32): w[kh*3 + kw][c0 + 32j + n] at K index n, rows
    // [64 kh + 32, 64 kh + 64): -zp_w at K index n.  One MMA over an input row
    // then feeds two output rows: its N columns are [W_kh | Z | W_kh+1 | Z]
    // and land in two adjacent TMEM row slots (see the MMA issuer).
    for (int idx = threadIdx.x; idx < 3 * KG * 2 * 192; idx += blockDim.x) {
        const int kw = idx / (KG * 384), rem = idx % (KG * 384);
        const int j = rem / 384, half = (rem % 384) / 192, n = rem % 192;
        const int kh = n / 64, wi = n % 64, oc = wi % 32, ch = c0 + j * 32 + oc;
        uint32_t v[4] = {0, 0, 0, 0};
        if (oc / 16 == half) {
            const uint32_t byte = wi < 32 ? (uint32_t)(uint8_t)p.wt[(kh * 3 + kw) * p.c + ch]
                                          : (uint32_t)(uint8_t)(int8_t)(-p.zpw[ch]);
            v[(oc % 16) / 4] = byte << (8 * (oc % 4));
        }
        *reinterpret_cast<uint4*>(smem + L.b_off + (size_t)idx * 16) = make_uint4(v[0], v[1], v[2], v[3]);
    }
    int32_t* corr_s = reinterpret_cast<int32_t*>(smem + L.corr_off);
    for (int i = threadIdx.x; i < 16 * CB; i += blockDim.x)
        corr_s[i] = p.corr[(i / CB) * p.c + c0 + i % CB] + p.cterm[c0 + i % CB];
    float* mult_s = reinterpret_cast<float*>(smem + L.mult_off);
    for (int i = threadIdx.x; i < CB; i += blockDim.x) mult_s[i] = p.mult[c0 + i];
    for (int i = threadIdx.x; i < 64; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    for (int b = 0; b < p.nb2; ++b) {
        const int hb = (R2 + 2) * p.wp * CB;
        uint4* g = reinterpret_cast<uint4*>(smem + L.halo_off + b * L.halo_stride + hb);
        for (int i = threadIdx.x; i < (L.halo_stride - hb) / 16; i += blockDim.x) g[i] = make_uint4(0, 0, 0, 0);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_ptr;
    const uint32_t halo_bytes = (uint32_t)((R2 + 2) * p.wp * CB);
    // TMEM per accumulator buffer: [K-group j][slot 0: output row r0 + 1 | slot 1: row r0] x 64
    // columns (32 sum x*w, 32 -zp_w * sum x).  Each slot is initialised by its
    // own N = 64 MMA group before the N = 128 MMAs accumulate into both.
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();

    if (warp == W_PROD) {
        // ------------------------------------------------ halo producer
        ptx::griddep_wait();  // x may be the previous grid's output
        int b = 0;
        uint32_t ph = 0;
        UnitWalk uw(cta_in, ctas, p.rb2);
        for (int k = cta_in; k < p.units_blk; k += ctas, uw.next()) {
            const int n = uw.n, rb = uw.rb;
            ptx::mbar_wait(empty_bar(b), ph ^ 1);
            if (ptx::elect_one()) {
                ptx::mbar_arrive_expect_tx(full_bar(b), halo_bytes);
                // box {64 ch, W+2 px, R2+2 rows, 1} at (c0, col -1, row rb*R2-1, image n)
                tma_load_4d(base + L.halo_off + b * L.halo_stride, &tmap_x, c0, -1, rb * R2 - 1, n, full_bar(b));
#ifdef Q8G_TRACE
                dw_stamp(p, 0, (k - cta_in) / ctas);
#endif
            }
            __syncwarp();
            if (++b == p.nb2) {
                b = 0;
                ph ^= 1;
            }
        }
    } else if (warp == W_MMA) {
        // ------------------------------------------------ MMA issuer
        constexpr uint32_t idesc64 = ptx::idesc_u8s8_s32<128, 64>();
        constexpr uint32_t idesc128 = ptx::idesc_u8s8_s32<128, 128>();
        const uint64_t a0 = kmajor_swz64_desc(0u);
        const uint64_t row16 = (uint64_t)(p.wp * CB / 16), pos16 = CB / 16;
        const uint64_t b0 = kmajor_noswz_desc(base + L.b_off, 192 * 16, 128);
        int b = 0, acc = 0;
        uint32_t ph = 0, aph = 0;
        for (int k = cta_in; k < p.units_blk; k += ctas) {
#ifdef Q8G_TRACE
            const long long ck0 = clock64();
#endif
            ptx::mbar_wait(tempty_bar(acc), aph ^ 1);
#ifdef Q8G_TRACE
            const long long ck1 = clock64();
#endif
            ptx::mbar_wait(full_bar(b), ph);
            ptx::tc_fence_after();
#ifdef Q8G_TRACE
            // debug (tools/dw_trace.py, -DQ8G_TRACE builds): cycles per wait and per loop
            const long long ck2 = clock64();
            if (lane == 0 && p.trace && blockIdx.x == 0 && (k - cta_in) / ctas < 64) {
                const int u = (k - cta_in) / ctas;
                p.trace[8192 + 24 * 64 + u] = (unsigned long long)(ck1 - ck0);
                p.trace[8192 + 25 * 64 + u] = (unsigned long long)(ck2 - ck1);
                p.trace[8192 + 26 * 64 + u] = (unsigned long long)ck0;
            }
#endif
            const uint64_t ahalo = a0 + ((base + L.halo_off + b * L.halo_stride) >> 4);  // TMEM lane m = output column m
            if (ptx::elect_one()) {
#ifdef Q8G_TRACE  // debug builds only: these stamps in the issue loop cost C4 ~2 us even when off
                dw_stamp(p, 1, (k - cta_in) / ctas);
#endif
                // halo row i = input row r0 - 1 + i feeds output row r0 + 1 with
                // tap row kh = i - 1 and output row r0 with kh = i:
                //   i = 0: r0 (kh 0)               N = 64 into slot 1
                //   i = 1: r0+1 (kh 0), r0 (kh 1)  N = 128 into slots 0-1
                //   i = 2: r0+1 (kh 1), r0 (kh 2)  N = 128 into slots 0-1
                //   i = 3: r0+1 (kh 2)             N = 64 into slot 0
                // issued i = 3, 0, 1, 2: the two N = 64 groups initialise their
                // slots (kw = 0 overwrites), so the N = 128 MMAs that accumulate
                // into both slots never need a zeroed slot
#pragma unroll
                for (int ii = 0; ii < R2 + 2; ++ii)
#pragma unroll
                    for (int kw = 0; kw < 3; ++kw)
#pragma unroll
                        for (int j = 0; j < KG; ++j) {
                            const int i = (ii + 3) % 4;
                            const uint64_t ad = ahalo + (uint64_t)i * row16 + (uint64_t)kw * pos16 + 2u * j;
                            const uint64_t bd = b0 + (uint64_t)((kw * KG + j) * 384);
                            const uint32_t d = tmem_base + (uint32_t)(acc * 256 + j * 128);
                            if (i == 0) ptx::mma_i8(d + 64, ad, bd, idesc64, kw != 0);
                            if (i == 1) ptx::mma_i8(d, ad, bd, idesc128, 1);
                            if (i == 2) ptx::mma_i8(d, ad, bd + 64, idesc128, 1);
                            if (i == 3) ptx::mma_i8(d, ad, bd + 128, idesc64, kw != 0);
                        }
                ptx::tc_commit(empty_bar(b));
                ptx::tc_commit(tfull_bar(acc));
#ifdef Q8G_TRACE
                dw_stamp(p, 2, (k - cta_in) / ctas);
#endif
            }
            __syncwarp();
            if (++b == p.nb2) {
                b = 0;
                ph ^= 1;
            }
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
#ifdef Q8G_TRACE
    } else if (warp == EPI64 + 2 && p.trace) {
        // debug trace only: the time each halo actually lands (the MMA warp's
        // own stamp also includes its wait for a free accumulator)
        int b = 0;
        uint32_t ph = 0;
        for (int k = cta_in; k < p.units_blk; k += ctas) {
            ptx::mbar_wait(full_bar(b), ph);
            if (lane == 0) dw_stamp(p, 5, (k - cta_in) / ctas);
            if (++b == p.nb2) {
                b = 0;
                ph ^= 1;
            }
        }
#endif
    } else if (warp < EPI64) {
        // ------------------------------------------------ requant epilogue
        ptx::griddep_wait();  // y may be read / written by the previous grid
        // warp = (output row r, K-group j) of the unit x TMEM lane quarter
        // (warp % 4); thread = one position.  16 warps (4 per SM sub-partition)
        // keep the TMEM-load latency covered.
        const int ew = warp, quarter = warp % 4, r = (ew / 4) / KG, j = (ew / 4) % KG;
        const int ocol = quarter * 32 + lane;  // TMEM lane = output column (lanes >= W: clipped by the store)
        const float2 magic2 = make_float2(12582912.0f, 12582912.0f);  // 1.5 * 2^23 (cterm carries its bit pattern)
        const float2 nmagic2 = make_float2(-12582912.0f, -12582912.0f);
        const float floor_x = p.lo == 0.0f ? 0.0f : -8388608.0f;  // ReLU: 0; else -2^23 (see conv_tc.cu)
        const int32_t zoff = 0x4B400000 - p.zp_c;
        // each warp stages its 32 positions x 32 channels (1 KB, double
        // buffered) and stores them with its own TMA store: no CTA-wide
        // barrier per unit (positions outside the image are clipped by the map)
        const uint32_t stg0 = ptx::smem_u32(smem + L.out_off + ew * L.out_stride);
        int acc = 0;
        uint32_t aph = 0;
        int ui = 0;
        UnitWalk uw(cta_in, ctas, p.rb2);
        for (int k = cta_in; k < p.units_blk; k += ctas, ++ui, uw.next()) {
            const int n = uw.n, oh0 = uw.rb * R2, oh = oh0 + r;
            Q8G_CHECK(n >= 0 && n < p.nb && oh0 < p.h && uw.rb < p.rb2);
            const int cls = (oh == 0 ? 1 : 0) | (oh == p.h - 1 ? 2 : 0) | (ocol == 0 ? 4 : 0) | (ocol == p.w - 1 ? 8 : 0);
            const uint32_t stg = stg0 + (uint32_t)((ui & 1) * 1024);
            // the store issued from this buffer two units ago has read it
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            ptx::mbar_wait(tfull_bar(acc), aph);
            ptx::tc_fence_after();
#ifdef Q8G_TRACE
            if (ew == 0 && lane == 0) dw_stamp(p, 3, ui);
#endif
            const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * 256 + j * 128 + (1 - r) * 64);
            // all 32 channels of this warp's tile out of TMEM first, then hand the
            // accumulator buffer back to the MMA warp before the requant math
            uint32_t vw[2][16], vz[2][16];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                ptx::tmem_ld_32x32b_x16(lane_base + (uint32_t)(hh * 16), vw[hh]);
                ptx::tmem_ld_32x32b_x16(lane_base + (uint32_t)(32 + hh * 16), vz[hh]);
            }
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(tempty_bar(acc));
#ifdef Q8G_TRACE
                dw_stamp(p, 7 + ew, ui);  // this warp released the accumulator
#endif
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {  // 16 channels at a time
                const int4* cq = reinterpret_cast<const int4*>(corr_s + cls * CB + j * 32 + hh * 16);
                const float4* mq = reinterpret_cast<const float4*>(mult_s + j * 32 + hh * 16);
                uint32_t w4[4];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int4 cc = cq[g];
                    const float4 mm = mq[g];
                    // exact int -> float via the magic bits (|adj| < 2^22, checked at filter creation)
                    const int32_t b0 = (int32_t)(vw[hh][4 * g] + vz[hh][4 * g]) + cc.x;
                    const int32_t b1 = (int32_t)(vw[hh][4 * g + 1] + vz[hh][4 * g + 1]) + cc.y;
                    const int32_t b2 = (int32_t)(vw[hh][4 * g + 2] + vz[hh][4 * g + 2]) + cc.z;
                    const int32_t b3 = (int32_t)(vw[hh][4 * g + 3] + vz[hh][4 * g + 3]) + cc.w;
                    float2 x01 = __fmul2_rn(__fadd2_rn(make_float2(__int_as_float(b0), __int_as_float(b1)), nmagic2),
                                            make_float2(mm.x, mm.y));
                    float2 x23 = __fmul2_rn(__fadd2_rn(make_float2(__int_as_float(b2), __int_as_float(b3)), nmagic2),
                                            make_float2(mm.z, mm.w));
                    x01.x = fmaxf(x01.x, floor_x);
                    x01.y = fmaxf(x01.y, floor_x);
                    x23.x = fmaxf(x23.x, floor_x);
                    x23.y = fmaxf(x23.y, floor_x);
                    x01 = __fadd2_rn(x01, magic2);
                    x23 = __fadd2_rn(x23, magic2);
                    w4[g] = pack_sat_u8(__float_as_int(x01.y) - zoff, __float_as_int(x01.x) - zoff,
                                        pack_sat_u8(__float_as_int(x23.y) - zoff, __float_as_int(x23.x) - zoff, 0u));
                }
                // SWIZZLE_32B staging row of 32 B per position: chunk ^= (row >> 2) & 1
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                                 stg + (uint32_t)(lane * 32 + ((hh ^ ((lane >> 2) & 1)) * 16))),
                             "r"(w4[0]), "r"(w4[1]), "r"(w4[2]), "r"(w4[3])
                             : "memory");
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staging writes -> TMA
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                        reinterpret_cast<uint64_t>(&tmap_y)),
                    "r"(c0 + 32 * j), "r"(quarter * 32), "r"(oh), "r"(n), "r"(stg)
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
#ifdef Q8G_TRACE
                if (ew == 0) dw_stamp(p, 4, ui);
#endif
            }
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // smem stays valid until stored
    }

    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == W_ALLOC) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem_base);
    }
}

// halo buffers of the 64-channel kernel: 3.  Fewer buffers keep the block's
// CTAs in step on adjacent rows (shared halo rows hit in L2): C4 with 2 / 3 /
// 4 / 5 buffers 87.8 / 59.6 / 63.0 / 67.9 us (Q8G_DW_NBUF, A/B)
int dw2_nbuf(int wp) {
    static const int env = [] {
        const char* e = getenv("Q8G_DW_NBUF");
        return e ? std::atoi(e) : 0;
    }();
    int nb = env > 0 ? std::max(2, std::min(NB2, env)) : 3;
    while (nb > 2 && dw2_layout(wp, nb).total > 232448) --nb;
    return nb;
}

bool dw_tc64_ok(int w, int c) {
    static const bool off = getenv("Q8G_DW_TC16") != nullptr;  // A/B switch: force the 16-channel kernel
    return !off && c % CB == 0 && w + 2 <= 128 && dw2_layout(w + 2, dw2_nbuf(w + 2)).total <= 232448;
}

}  // namespace

bool dw_tc64_supported(int w, int c) { return tmap_encoder() != nullptr && dw_tc64_ok(w, c); }

bool dw_tc_supported(int h, int w, int c, int32_t zp_a) {
    (void)zp_a;
    if (h < 1 || tmap_encoder() == nullptr) return false;
    if (dw_tc64_ok(w, c)) return true;
    // one unit's tiles (ROWS rows of w+2 positions) must fit a 128-column TMEM buffer
    return c % G == 0 && w + 2 <= MAXW && (ROWS * (w + 2) + 127) / 128 * G <= 128 &&
           dw_layout((ROWS + 2) * (w + 2) * G, c / G).total <= 232448;
}

cudaError_t launch_dwconv3x3_tc(const uint8_t* x, int nb, int h, int w, int c, const q8g_dw_filter* f, uint8_t* y,
                                cudaStream_t s) {
    auto enc = tmap_encoder();
    if (!enc) return cudaErrorNotSupported;
    const bool tc64 = dw_tc64_ok(w, c);
    CUtensorMap tmap;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)nb};
    cuuint64_t strides[3] = {(cuuint64_t)c, (cuuint64_t)w * c, (cuuint64_t)h * w * c};
    cuuint32_t box[4] = {(cuuint32_t)(tc64 ? CB : G), (cuuint32_t)(w + 2), (cuuint32_t)((tc64 ? R2 : ROWS) + 2), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, tc64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    // output map (64-channel kernel): per-warp TMA stores of 32 channels x 32 positions
    CUtensorMap tmap_y;
    if (tc64) {
        // per epilogue warp: 32 channels x 32 positions of one output row
        cuuint32_t boxy[4] = {32, 32, 1, 1};
        if (enc(&tmap_y, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, y, dims, strides, boxy, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    DwParams p;
    p.nb = nb;
    p.h = h;
    p.w = w;
    p.c = c;
    p.wp = w + 2;
    p.groups = c / G;
    p.rblocks = (h + ROWS - 1) / ROWS;
    p.tiles = (ROWS * p.wp + 127) / 128;
    p.units = nb * p.rblocks * p.groups;
    p.halo_bytes = (ROWS + 2) * p.wp * G;
    p.wt = f->w;
    p.zpw = f->zpw_dev;
    p.cterm = f->cterm_dev;
    p.mult = f->mult_dev;
    p.corr = f->corr_dev;
    p.lo = f->lo;
    p.hi = f->hi;
    p.zp_c = f->zp_c;
    p.y = y;
    p.trace = tc_trace_buffer_ptr();
    p.nblk = c / CB;
    p.rb2 = (h + R2 - 1) / R2;
    p.units_blk = nb * p.rb2;
    p.nb2 = dw2_nbuf(p.wp);
    int dev = 0;
    cudaGetDevice(&dev);
    if (tc64) {
        static bool attr64[64] = {false};
        if (dev < 64 && !attr64[dev]) {
            cudaError_t e = cudaFuncSetAttribute(dwconv_tc64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
            if (e != cudaSuccess) return e;
            attr64[dev] = true;
        }
        // whole channel blocks per CTA: grid a multiple of the block count
        int per_blk = sm_count(dev) / p.nblk;
        if (per_blk < 1) per_blk = 1;
        if (per_blk > p.units_blk) per_blk = p.units_blk;
        const cudaError_t e = launch_with_pdl(dwconv_tc64_kernel, dim3(per_blk * p.nblk), dim3(128 + 32 * EPI64),
                                              dw2_layout(p.wp, p.nb2).total, s, tmap, tmap_y, p);
        count_launch(kFamDwTc);
        return e;
    }
    const DwLayout L = dw_layout(p.halo_bytes, p.groups);
    static bool attr_set[64] = {false};
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(dwconv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    int grid = sm_count(dev);
    if (grid > p.units) grid = p.units;
    const cudaError_t e = launch_with_pdl(dwconv_tc_kernel, dim3(grid), dim3(128 + 32 * EPI_WARPS), L.total, s, tmap, p);
    count_launch(kFamDwTc);
    return e;
}

}  // namespace q8g
