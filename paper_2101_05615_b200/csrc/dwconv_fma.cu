// dwconv_fma.cu — depthwise 3x3 / stride 1 / pad 1 NHWC on the CUDA cores
// (BASELINE config C4, the HBM-bound path), exact integer arithmetic carried
// in fp32 FMAs.
//
// Semantics: SURVEY.md App. A D3 (no reference symbol).  For output (n,h,w,c)
//   adj = sum_t x_t * w'[t,c] + bias[c] - zp_a * sum_t w'[t,c],
//   w'[t,c] = w[t,c] - zp_w[c],
// with padded taps reading x = zp_a (equal to the D3 form term by term), then
// the F32_RNE requant RN(float(adj) * mult[c]).  The padding is TMA's zero
// fill; outputs on the image border add the exact missing term
// zp_a * sum_{padded t} w'[t,c] (one of 15 border classes) before rounding.
//
// Why fp32 FMAs carry an exact int8 dot product here:
// * the input byte x is turned into the float whose bit pattern is x itself
//   (one PRMT on the integer pipe, no FP op): the denormal x * 2^-149;
// * the weights are stored as w' * 2^119 (exact power-of-two scaling), so
//   every product x * w' * 2^-30 is exact inside the FMA, and every partial
//   sum is an integer multiple of 2^-30 below 2^24 units (host gate
//   |bias| + 2 * 9 * 255 * 255 < 2^23): the accumulator equals adj * 2^-30
//   exactly, in any summation order;
// * the epilogue multiplies by mult * 2^30, i.e. computes RN(adj * mult), the
//   same real number the reference rounds.
// The FMAs run as FFMA2 (two channels per instruction), and the
// accumulator is initialised with the folded constant, so one output costs
// 4.5 FFMA2 + 0.5 FMUL2 + 0.5 FADD2 on the FMA pipes and ~1.5 PRMT + FMNMX +
// IADD + 0.5 I2IP on the integer pipe.  Measured on C4 it is register-operand
// bound (83 us vs 71 us for the 64-channel tensor-core kernel, DESIGN.md
// §4.4), so dispatch uses it where that kernel does not fit (W + 2 > 128).
//
// Layout: a CTA owns 128 channels (one 32-bit word = 4 channels per lane,
// so every shared-memory word load of a warp is one conflict-free 128-byte
// row) of a 56-position segment of one image; 14 consumer warps each own 4
// output positions.  A work unit is 14 output rows; the producer warp streams
// its 16 input rows (58 positions x 128 channels, one 4-D TMA box each, rows
// and positions outside the image zero-filled)
// through a 12-stage ring, and the consumers roll down the rows keeping two
// output rows of accumulators in registers: input row r finishes output row
// r-1 (kh = 2), adds kh = 1 to row r and opens row r+1 (kh = 0).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "epilogue.cuh"
#include "ptx.cuh"
#include "q8g_internal.cuh"

namespace q8g {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder();

namespace {

constexpr int CBF = 128;            // channels per CTA
constexpr int PW = 4;               // output positions per thread
constexpr int NCW = 14;             // consumer warps
constexpr int SEG = PW * NCW;       // 56 positions per segment
constexpr int BOXW = SEG + 2;       // 58 input positions per row (halo 1 each side)
constexpr int RC = 14;              // output rows per unit
constexpr int NST = 12;             // ring stages (one input row each)
constexpr int STAGE = CBF * BOXW;   // 7424 bytes
constexpr int THREADS = 32 * (NCW + 1);
constexpr int SMEM = NST * STAGE + 32 * 32 + 2 * NST * 8;

struct DwfParams {
    int nb, h, w, c;
    int nseg, nchunk, ncb, units;
    const float4* wf;      // [c/4][9] : (w - zp_w) * 2^119 for the 4 channels of a word
    const float4* binit;   // [c/4]    : (bias - zp_a * sum_t w') * 2^-30
    const float4* mscale;  // [c/4]    : mult * 2^30
    const float4* corr;    // [16][c/4]: zp_a * sum_{padded t} w' * 2^-30 per border class
    float floor_x;         // 0 (ReLU) or -2^23
    int32_t zoff;          // 0x4B400000 - zp_c
    size_t rowstride;      // w * c bytes
    uint8_t* y;
};

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

struct Unit {
    int n, cb, seg, r0, rows;
};

// unit order: row chunk fastest (neighbouring chunks share halo rows in L2),
// channel block slowest (a CTA rarely switches weights)
__device__ __forceinline__ Unit unit_of(const DwfParams& p, int u) {
    Unit t;
    const int chunk = u % p.nchunk;
    int rest = u / p.nchunk;
    t.seg = rest % p.nseg;
    rest /= p.nseg;
    t.n = rest % p.nb;
    t.cb = rest / p.nb;
    t.r0 = chunk * RC;
    t.rows = min(RC, p.h - t.r0);
    return t;
}

// the float whose bit pattern is byte b of v (x * 2^-149)
__device__ __forceinline__ float byte_f(uint32_t v, int b) { return __uint_as_float(__byte_perm(v, 0u, 0x4440 | b)); }

struct Acc {
    float2 v[PW][2];  // [position][channel pair]
};

struct Ctx {
    const DwfParams& p;
    const uint8_t* xrow;  // this thread's word in stage 0
    uint32_t bars;
    int s;
    uint32_t ph;          // ring position / parity of the next row to consume
    const float4* consts; // this thread's {binit, mscale} in shared memory
    float2 w[9][2];
    int q;                // channel word
    int wpos0;            // first output position
    int colcls;           // border class bits of the thread's positions: 4 left (pp 0), 8 right (pp = rpos)
    int rpos;
    int npos;             // positions inside the image
    uint8_t* yrow;
    __device__ __forceinline__ uint32_t full_bar(int st) const { return bars + 8u * st; }
    __device__ __forceinline__ uint32_t empty_bar(int st) const { return bars + 8u * (NST + st); }
};

// requantize and store position pp of a finished output row (4 channels)
template <int CS>
__device__ __forceinline__ void finish_pos(const Ctx& c, const float2 (&v2)[2], const float2 (&m)[2], int pp) {
    const DwfParams& p = c.p;
    const float2 magic = make_float2(12582912.0f, 12582912.0f);
    int32_t r[4];
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        float2 v = __fmul2_rn(v2[h2], m[h2]);
        v.x = fmaxf(v.x, p.floor_x);
        v.y = fmaxf(v.y, p.floor_x);
        v = __fadd2_rn(v, magic);
        r[2 * h2] = __float_as_int(v.x) - p.zoff;
        r[2 * h2 + 1] = __float_as_int(v.y) - p.zoff;
    }
    const uint32_t word = pack_sat_u8(r[1], r[0], pack_sat_u8(r[3], r[2], 0u));
    const int cs = CS ? CS : p.c;
    if (pp < c.npos) *reinterpret_cast<uint32_t*>(c.yrow + pp * cs) = word;
}

// outputs on the image border (row `orow`): add the padded taps' zp_a terms
// to a freshly opened accumulator row
__device__ __forceinline__ void border_fix(const Ctx& c, Acc& a, int orow) {
    const DwfParams& p = c.p;
    const int rowcls = (orow == 0 ? 1 : 0) | (orow == p.h - 1 ? 2 : 0);
    if ((rowcls | c.colcls) == 0) return;
#pragma unroll
    for (int pp = 0; pp < PW; ++pp) {
        const int cls = rowcls | (pp == 0 ? c.colcls & 4 : 0) | (pp == c.rpos ? c.colcls & 8 : 0);
        if (cls) {
            const float4 k = __ldg(p.corr + cls * (p.c / 4) + c.q);
            a.v[pp][0] = __fadd2_rn(a.v[pp][0], make_float2(k.x, k.y));
            a.v[pp][1] = __fadd2_rn(a.v[pp][1], make_float2(k.z, k.w));
        }
    }
}

// one input row r:
// FIN  adds kh = 2 to F and stores it (output row r - 1),
// MID  adds kh = 1 to M (output row r),
// OPEN starts F over with kh = 0 (output row r + 1).
// The work is laid out position by position (convert one word, the FMAs of
// that position, its requant, its re-open) so every stretch of the
// instruction stream mixes FMA-pipe and integer-pipe work: identical warps
// run in lock step, and phase-separated code would idle one pipe at a time.
template <int CS, bool FIN, bool MID, bool OPEN>
__device__ __forceinline__ void step(Ctx& c, Acc& F, Acc& M, int r) {
    uint32_t xw[PW + 2];
    ptx::mbar_wait(c.full_bar(c.s), c.ph);
    const uint8_t* row = c.xrow + c.s * STAGE;
#pragma unroll
    for (int k = 0; k < PW + 2; ++k) xw[k] = *reinterpret_cast<const uint32_t*>(row + k * CBF);
    ptx::mbar_arrive(c.empty_bar(c.s));  // every consumer thread, after its own loads
    if (++c.s == NST) {
        c.s = 0;
        c.ph ^= 1;
    }
    if (c.npos <= 0) return;  // warp beyond the image (last segment)
    float2 m[2], bi[2];
    if (FIN) {
        const float4 m4 = c.consts[1];
        m[0] = make_float2(m4.x, m4.y);
        m[1] = make_float2(m4.z, m4.w);
    }
    if (OPEN) {
        const float4 b = c.consts[0];
        bi[0] = make_float2(b.x, b.y);
        bi[1] = make_float2(b.z, b.w);
    }
    float2 x[PW + 2][2];
#pragma unroll
    for (int k = 0; k < PW + 2; ++k) {
        x[k][0] = make_float2(byte_f(xw[k], 0), byte_f(xw[k], 1));
        x[k][1] = make_float2(byte_f(xw[k], 2), byte_f(xw[k], 3));
    }
    // weight-major order: consecutive FFMA2s share the weight operand (register reuse cache)
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
        for (int kw = 0; kw < 3; ++kw) {
            if (FIN)
#pragma unroll
                for (int pp = 0; pp < PW; ++pp) F.v[pp][h2] = __ffma2_rn(x[pp + kw][h2], c.w[6 + kw][h2], F.v[pp][h2]);
            if (MID)
#pragma unroll
                for (int pp = 0; pp < PW; ++pp) M.v[pp][h2] = __ffma2_rn(x[pp + kw][h2], c.w[3 + kw][h2], M.v[pp][h2]);
        }
    if (FIN)
#pragma unroll
        for (int pp = 0; pp < PW; ++pp) finish_pos<CS>(c, F.v[pp], m, pp);
    if (OPEN)
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2)
#pragma unroll
            for (int kw = 0; kw < 3; ++kw)
#pragma unroll
                for (int pp = 0; pp < PW; ++pp)
                    F.v[pp][h2] = __ffma2_rn(x[pp + kw][h2], c.w[kw][h2], kw == 0 ? bi[h2] : F.v[pp][h2]);
    if (FIN) c.yrow += c.p.rowstride;
    if (OPEN) border_fix(c, F, r + 1);
}

// the rows + 2 input rows of one unit, the two accumulator sets trading roles
template <int CS>
__device__ __forceinline__ void run_unit(Ctx& c, int r0, int rows) {
    Acc A, B;
    step<CS, false, false, true>(c, A, B, r0 - 1);  // input row r0 - 1 opens output row r0
    if (rows == 1) {
        step<CS, false, true, false>(c, B, A, r0);
        step<CS, true, false, false>(c, A, B, r0 + 1);
        return;
    }
    step<CS, false, true, true>(c, B, A, r0);
    int i = 2;  // input row r0 - 1 + i
    for (; i + 1 < rows; i += 2) {
        step<CS, true, true, true>(c, A, B, r0 - 1 + i);
        step<CS, true, true, true>(c, B, A, r0 + i);
    }
    if (i < rows) {  // i = rows - 1 (even)
        step<CS, true, true, true>(c, A, B, r0 - 1 + i);
        ++i;
    }
    // i = rows: finish rows - 2, last kh = 1; i = rows + 1: finish rows - 1
    if (i & 1) {
        step<CS, true, true, false>(c, B, A, r0 - 1 + i);
        step<CS, true, false, false>(c, A, B, r0 + i);
    } else {
        step<CS, true, true, false>(c, A, B, r0 - 1 + i);
        step<CS, true, false, false>(c, B, A, r0 + i);
    }
}

template <int CS>  // position stride in bytes when compile-time (C == CS), else 0
__global__ void __launch_bounds__(THREADS, 1)
    dwconv_fma_kernel(const __grid_constant__ CUtensorMap tmap_x, const DwfParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    Q8G_CHECK((uint32_t)SMEM <= ptx::dynamic_smem_size());
    const uint32_t base = ptx::smem_u32(smem);
    float4* consts = reinterpret_cast<float4*>(smem + NST * STAGE);  // [32 lanes][binit, mscale]
    Ctx c{p};
    c.bars = base + NST * STAGE + 32 * 32;
    c.xrow = smem + (warp * PW) * CBF + lane * 4;
    c.consts = consts + 2 * lane;
    c.s = 0;
    c.ph = 0;

    ptx::griddep_launch_dependents();
    if (threadIdx.x == 0) {
        for (int st = 0; st < NST; ++st) {
            ptx::mbar_init(c.full_bar(st), 1);
            ptx::mbar_init(c.empty_bar(st), NCW * 32);
        }
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmap_x);
    }
    __syncthreads();
    ptx::griddep_wait();

    if (warp == NCW) {
        // ---------------- producer: rows r0 - 1 .. r0 + rows of each unit, one TMA box each
        if (ptx::elect_one()) {
            int st = 0;
            uint32_t ph = 0;
            for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
                const Unit t = unit_of(p, u);
                for (int r = t.r0 - 1; r <= t.r0 + t.rows; ++r) {
                    ptx::mbar_wait(c.empty_bar(st), ph ^ 1);
                    ptx::mbar_arrive_expect_tx(c.full_bar(st), STAGE);
                    tma_load_4d(base + st * STAGE, &tmap_x, t.cb * CBF, t.seg * SEG - 1, r, t.n, c.full_bar(st));
                    if (++st == NST) {
                        st = 0;
                        ph ^= 1;
                    }
                }
            }
        }
        return;
    }

    // ---------------- consumers
    int cur_cb = -1;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const Unit t = unit_of(p, u);
        c.q = t.cb * 32 + lane;
        if (t.cb != cur_cb) {
            cur_cb = t.cb;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const float4 v = __ldg(p.wf + c.q * 9 + k);
                c.w[k][0] = make_float2(v.x, v.y);
                c.w[k][1] = make_float2(v.z, v.w);
            }
            // all consumer warps share the lane's constants: refresh them between barriers
            asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
            if (warp == 0) {
                consts[2 * lane] = __ldg(p.binit + c.q);
                consts[2 * lane + 1] = __ldg(p.mscale + c.q);
            }
            asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
        }
        c.wpos0 = t.seg * SEG + warp * PW;
        c.npos = min(PW, p.w - c.wpos0);
        c.rpos = p.w - 1 - c.wpos0;
        c.colcls = (c.wpos0 == 0 ? 4 : 0) | (c.rpos >= 0 && c.rpos < PW ? 8 : 0);
        c.yrow = p.y + ((size_t)(t.n * p.h + t.r0) * p.w + c.wpos0) * p.c + c.q * 4;
        run_unit<CS>(c, t.r0, t.rows);
    }
}

}  // namespace

// exactness gate (see the header comment); tables built by q8g_dw_filter_create
bool dw_fma_supported(int h, int w, int c) {
    return h >= 1 && w >= 1 && c % CBF == 0 && (long long)h * w * c < (1LL << 31) &&
           tmap_encoder() != nullptr;
}

cudaError_t launch_dwconv3x3_fma(const uint8_t* x, int nb, int h, int w, int c, const q8g_dw_filter* f, uint8_t* y,
                                 cudaStream_t s) {
    auto enc = tmap_encoder();
    if (!enc) return cudaErrorNotSupported;
    CUtensorMap tmap;
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)nb};
    cuuint64_t strides[3] = {(cuuint64_t)c, (cuuint64_t)w * c, (cuuint64_t)h * w * c};
    cuuint32_t box[4] = {(cuuint32_t)CBF, (cuuint32_t)BOXW, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(x), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    DwfParams p;
    p.nb = nb;
    p.h = h;
    p.w = w;
    p.c = c;
    p.nseg = (w + SEG - 1) / SEG;
    p.nchunk = (h + RC - 1) / RC;
    p.ncb = c / CBF;
    p.units = nb * p.ncb * p.nseg * p.nchunk;
    p.wf = reinterpret_cast<const float4*>(f->fma_w);
    p.binit = reinterpret_cast<const float4*>(f->fma_b);
    p.mscale = reinterpret_cast<const float4*>(f->fma_m);
    p.corr = reinterpret_cast<const float4*>(f->fma_corr);
    p.floor_x = f->relu ? 0.0f : -8388608.0f;
    p.zoff = 0x4B400000 - f->zp_c;
    p.rowstride = (size_t)w * c;
    p.y = y;
    int dev = 0;
    cudaGetDevice(&dev);
    const bool c256 = c == 256;  // compile-time position stride: immediate store offsets
    auto kern = c256 ? dwconv_fma_kernel<256> : dwconv_fma_kernel<0>;
    static bool attr[2][64] = {};
    if (dev < 64 && !attr[c256][dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        if (e != cudaSuccess) return e;
        attr[c256][dev] = true;
    }
    int grid = sm_count(dev);
    if (grid > p.units) grid = p.units;
    const cudaError_t e = launch_with_pdl(kern, dim3(grid), dim3(THREADS), SMEM, s, tmap, p);
    count_launch(kFamDwFma);
    return e;
}

}  // namespace q8g
