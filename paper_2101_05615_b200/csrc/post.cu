// post.cu — the general output pipeline off the hot path:
// [SpMDMAdd] [BiasAdd]* [ReluQuantized] writer, writer in {WriteRawI32,
// Requantize, WriteDequantF32} (pipeline.hpp:157-207, sparse.hpp:62-80).
//
// The dense product runs on the tuned tensor-core kernels as a raw int32
// GEMM (into the caller's int32 output for WriteRawI32, else into a
// stream-ordered workspace); one post kernel then adds the outliers' product
// A x S (S = the CSC outlier store of split_outliers, sparse.hpp:33-58),
// and applies the writer.  BiasAdd is folded into the raw GEMM (raw / dequant
// writers) or into the requant epilogue table (q8g_epilogue_create), exactly
// where the reference applies it: after SpMDMAdd, before the writer (int32
// addition commutes).
#include <cuda_runtime.h>

#include "q8g_internal.cuh"
#include "requant.cuh"

namespace q8g {
namespace {

constexpr int PT = 256;  // threads per block: 256 consecutive output columns of one row

// WRITER 0: acc (in place, int32) += A x S; 1: requant F32_RNE; 2: requant REF;
// 3: dequant f32.  One block per (row, 256-column slice).
template <int WRITER>
__global__ void __launch_bounds__(PT) post_kernel(const int32_t* acc, int ldacc, const uint8_t* a, int lda, int k,
                                                  int n, const int32_t* col_ptr, const int32_t* row_idx,
                                                  const int8_t* vals, const EpiRecord* rec, int need_rowsum,
                                                  int32_t zp_c, int relu, double dq_scale, int32_t dq_zp,
                                                  void* out, int ldc) {
    const int i = blockIdx.y;
    const int j = blockIdx.x * PT + threadIdx.x;
    const uint8_t* arow = a + (size_t)i * lda;
    int32_t rowsum = 0;
    if (WRITER == 1 || WRITER == 2) {
        if (need_rowsum) {
            // full-K row sum of A (pack.hpp:83-135 row offsets), block reduction
            __shared__ int32_t part[PT / 32];
            uint32_t s = 0;
            for (int kk = threadIdx.x; kk < k; kk += PT) s += arow[kk];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = (int32_t)s;
            __syncthreads();
            for (int w = 0; w < PT / 32; ++w) rowsum += part[w];
        }
    }
    if (j >= n) return;
    int32_t v = acc[(size_t)i * ldacc + j];
    if (col_ptr) {
        // SpMDMAdd (sparse.hpp:62-80): outliers of column j, int32 wrapping
        uint32_t s = (uint32_t)v;
        for (int32_t idx = __ldg(col_ptr + j), e = __ldg(col_ptr + j + 1); idx < e; ++idx)
            s += (uint32_t)((int32_t)arow[__ldg(row_idx + idx)] * (int32_t)__ldg(vals + idx));
        v = (int32_t)s;
    }
    if (WRITER == 0) {
        reinterpret_cast<int32_t*>(out)[(size_t)i * ldc + j] = v;
    } else if (WRITER == 3) {
        // WriteDequantF32 (pipeline.hpp:199-207): scale * (acc - zp), fp64, RN to float
        const int32_t d = (int32_t)((uint32_t)v - (uint32_t)dq_zp);
        reinterpret_cast<float*>(out)[(size_t)i * ldc + j] = __double2float_rn(__dmul_rn(dq_scale, (double)d));
    } else {
        const int4 r4 = __ldg(reinterpret_cast<const int4*>(rec + j));
        EpiRecord rc;
        rc.c = r4.x;
        rc.zpb = r4.y;
        const int32_t adj = adjust(v, rowsum, rc);
        const uint32_t q = WRITER == 1 ? requant_f32(adj, __int_as_float(r4.z), zp_c, relu)
                                       : requant_ref(adj, __hiloint2double(r4.w, r4.z), zp_c, relu);
        reinterpret_cast<uint8_t*>(out)[(size_t)i * ldc + j] = (uint8_t)q;
    }
}

}  // namespace

cudaError_t launch_post(int writer, const int32_t* acc, int ldacc, const uint8_t* a, int lda, int rows, int k, int n,
                        const q8g_sparse_csc* sp, const q8g_epilogue* ep, double dq_scale, int32_t dq_zp, void* out,
                        int ldc, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    const dim3 grid((n + PT - 1) / PT, rows);
    const int32_t* cp = sp ? sp->col_ptr : nullptr;
    const int32_t* ri = sp ? sp->row_idx : nullptr;
    const int8_t* vv = sp ? sp->values : nullptr;
    const EpiRecord* rec = ep ? ep->rec : nullptr;
    const int need_rs = ep && ep->need_rowsum ? 1 : 0;
    const int32_t zp_c = ep ? ep->zp_c : 0;
    const int relu = ep ? ep->relu : 0;
    if (writer == Q8G_WRITE_RAW_I32) {
        post_kernel<0><<<grid, PT, 0, s>>>(acc, ldacc, a, lda, k, n, cp, ri, vv, rec, need_rs, zp_c, relu, dq_scale,
                                           dq_zp, out, ldc);
    } else if (writer == Q8G_WRITE_DEQUANT_F32) {
        post_kernel<3><<<grid, PT, 0, s>>>(acc, ldacc, a, lda, k, n, cp, ri, vv, rec, need_rs, zp_c, relu, dq_scale,
                                           dq_zp, out, ldc);
    } else if (ep && ep->rounding == Q8G_ROUND_F32_RNE) {
        post_kernel<1><<<grid, PT, 0, s>>>(acc, ldacc, a, lda, k, n, cp, ri, vv, rec, need_rs, zp_c, relu, dq_scale,
                                           dq_zp, out, ldc);
    } else {
        post_kernel<2><<<grid, PT, 0, s>>>(acc, ldacc, a, lda, k, n, cp, ri, vv, rec, need_rs, zp_c, relu, dq_scale,
                                           dq_zp, out, ldc);
    }
    count_launch(kFamPost);
    return cudaGetLastError();
}

}  // namespace q8g
