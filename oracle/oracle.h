/*
 * oracle.h — CPU restatement of the reference q8gemm hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path (the CUDA library,
 * the C++/Python host mirror) may link, import or call this.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * use it, and only as the checker / CPU baseline.
 *
 * Parity pin: every function here cites the reference file:line it restates.
 * The restatement is pinned (tests/test_oracle_kat.py) against
 *   - the reference unit-test known answers (proj/tests/test_*.cpp), and
 *   - outputs of the unmodified reference compiled here (oracle/_ref, built by
 *     oracle/Makefile from /root/reference/proj/include), committed as
 *     fixtures under tests/golden/ by tests/golden/make_golden.py.
 * Extensions the reference does not have (per-channel zero points / fp32
 * round-to-nearest-even, conv3x3 im2col, depthwise 3x3) are restated from
 * SURVEY.md Appendix A (D1-D4) and are "parity unpinned" beyond the identities
 * the tests check (per-tensor F32 path reduces to the same int32 "adjusted"
 * value as the pinned reference path).
 */
#ifndef Q8G_ORACLE_H
#define Q8G_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- std::mt19937_64 (reference fixtures: proj/tests/test_util.hpp:10-54) ---- */
typedef struct orc_rng orc_rng;
orc_rng* orc_rng_new(uint64_t seed);
void orc_rng_free(orc_rng* r);
uint64_t orc_rng_next(orc_rng* r);
/* test_util.hpp:12-14  rng() & 0xFF */
void orc_rng_u8(orc_rng* r, uint8_t* out, int64_t count);
/* test_util.hpp:16-18  (int8_t)(rng() & 0xFF) */
void orc_rng_i8(orc_rng* r, int8_t* out, int64_t count);
/* test_util.hpp:20-22  lo + rng() % (hi-lo+1) */
int32_t orc_rng_int(orc_rng* r, int32_t lo, int32_t hi);
void orc_rng_int_fill(orc_rng* r, int32_t lo, int32_t hi, int32_t* out, int64_t count);
/* test_util.hpp:24-26  lo + (hi-lo)*((rng()%10001)/10000.0) */
double orc_rng_real(orc_rng* r, double lo, double hi);
void orc_rng_real_fill(orc_rng* r, double lo, double hi, double* out, int64_t count);

/* ---- GEMM core ---- */
/* oracle.hpp:15-30 naive_gemm_i32: C[i][j] = sum_k A[i][k]*B[k][j] in int32.
 * threads >1 splits rows (each row is computed identically). */
void orc_naive_gemm_i32(const uint8_t* a, int m, int k, int lda,
                        const int8_t* b, int n, int ldb,
                        int32_t* c, int ldc, int threads);
/* quant.hpp:98-110 compute_col_offsets */
void orc_col_offsets(const int8_t* b, int k, int n, int ldb, int32_t* out);
/* pack.hpp:103-124 (row offsets fused into A packing), full K */
void orc_row_offsets(const uint8_t* a, int m, int k, int lda, int32_t* out);

/* ---- requantization (back-end) ---- */
/* quant.hpp:115-125 requantize_adjust (int64) */
int64_t orc_requant_adjust(int32_t acc, int32_t row_offset, int32_t col_offset,
                           int32_t zp_a, int32_t zp_b, int32_t k_total, int32_t bias);
/* quant.hpp:45-47 round_half_away_from_zero == std::llround */
long long orc_round_half_away(double x);
/* quant.hpp:127-133 requantize_scalar, mode REF (double multiply, half-away) */
uint8_t orc_requant_scalar_ref(int32_t acc, int32_t row_offset, int32_t col_offset,
                               double multiplier, int32_t zp_a, int32_t zp_b, int32_t zp_c,
                               int32_t k_total, int32_t bias);
/* (float)adj * mult_f32 (one RN multiply), RNE, + zp_c, clamp */
uint8_t orc_requant_scalar_f32(int32_t acc, int32_t row_offset, int32_t col_offset,
                               float multiplier, int32_t zp_a, int32_t zp_b, int32_t zp_c,
                               int32_t k_total, int32_t bias);
/* pipeline.hpp:51-53 relu_quantized */
uint8_t orc_relu_quantized(uint8_t q, int32_t zp_c);

/* Whole-matrix writer: pipeline.hpp:176-190 (Requantize [+ReluQuantized]).
 * rounding 0 = REF (per-tensor: mult_d[0], zp_b[0] used when per_channel==0)
 * rounding 1 = F32_RNE.  per_channel: zp_b / mult arrays have n entries.
 * bias may be NULL.  rowsum may be NULL (treated as 0, pipeline.hpp:177). */
void orc_requant_matrix(const int32_t* acc, int m, int n, int ldacc,
                        const int32_t* rowsum, const int32_t* colsum,
                        int32_t zp_a, const int32_t* zp_b, int per_channel, int32_t k_total,
                        const int32_t* bias, int rounding, const double* mult_d,
                        const float* mult_f, int32_t zp_c, int relu,
                        uint8_t* out, int ldo);

/* ---- reference packed-B layout (pack.hpp:146-196), test-only KAT carrier ---- */
int64_t orc_prepack_ref_size(int k, int n, int ncb, int kcb);
void orc_prepack_ref(const int8_t* b, int k, int n, int ldb,
                     int ncb, int kcb, int nr, int8_t* packed);

/* ---- conv3x3 NHWC, stride 1, pad 1 (no reference symbol) ----
 * x: [nb][h][w][c] u8; wt: [3][3][c][oc] s8 == K x N with k=(kh*3+kw)*c+ci;
 * pad taps read zp_a.  Produces the im2col matrix (rows = nb*h*w, K = 9c). */
void orc_im2col3x3(const uint8_t* x, int nb, int h, int w, int c, uint8_t zp_a,
                   uint8_t* cols /* [nb*h*w][9c] */, int threads);
/* conv acc + requant via im2col -> naive GEMM -> per-channel requant */
void orc_conv3x3_i32(const uint8_t* x, int nb, int h, int w, int c, uint8_t zp_a,
                     const int8_t* wt, int oc, int32_t* acc /* [nb*h*w][oc] */, int threads);

/* ---- depthwise 3x3 NHWC, stride 1, pad 1 ---- */
void orc_dwconv3x3(const uint8_t* x, int nb, int h, int w, int c, int32_t zp_a,
                   const int8_t* wt /* [9][c] */, const int32_t* zp_w /* c */,
                   const int32_t* bias /* c or NULL */, const float* mult /* c */,
                   int32_t zp_c, int relu, uint8_t* out, int32_t* acc_out /* may be NULL */,
                   int threads);

/* ---- outlier split (sparse.hpp:33-58), SpMDMAdd (sparse.hpp:62-80),
 * WriteDequantF32 (pipeline.hpp:199-207) ---- */
int orc_split_outliers(const int8_t* b, int k, int n, int ldb, int threshold, int8_t* dense, int ldd,
                       int32_t* col_ptr /* n+1 */, int32_t* row_idx, int8_t* values, int cap);
void orc_spmdm_add(const uint8_t* a, int m, int k, int lda, const int32_t* col_ptr, const int32_t* row_idx,
                   const int8_t* values, int n, int32_t* acc, int ldacc);
void orc_dequant_f32(const int32_t* acc, int m, int n, int ldacc, double scale, int32_t zp, float* out, int ldo);

#ifdef __cplusplus
}
#endif
#endif
