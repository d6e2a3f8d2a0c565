/*
 * oracle.c — CPU restatement of the reference q8gemm hot path (TEST
 * INFRASTRUCTURE ONLY; see oracle.h for the rules and the parity pin).
 *
 * Compiled with -ffp-contract=off so the fp32/fp64 multiplies are single
 * IEEE round-to-nearest operations (no FMA contraction, no x87 excess
 * precision on x86-64 SSE).
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* std::mt19937_64, the generator behind every reference fixture       */
/* (proj/tests/test_util.hpp:10-54; acceptance.cpp:24-31).             */
/* Published algorithm (Matsumoto & Nishimura), 64-bit parameter set.  */
/* ------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
struct orc_rng {
    uint64_t mt[MT_N];
    int idx;
};

orc_rng* orc_rng_new(uint64_t seed) {
    orc_rng* r = (orc_rng*)malloc(sizeof(orc_rng));
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
    return r;
}

void orc_rng_free(orc_rng* r) { free(r); }

static void mt_twist(orc_rng* r) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < MT_N; ++i) {
        uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->idx = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
    if (r->idx >= MT_N) mt_twist(r);
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

void orc_rng_u8(orc_rng* r, uint8_t* out, int64_t count) {
    for (int64_t i = 0; i < count; ++i) out[i] = (uint8_t)(orc_rng_next(r) & 0xFF);
}

void orc_rng_i8(orc_rng* r, int8_t* out, int64_t count) {
    for (int64_t i = 0; i < count; ++i) out[i] = (int8_t)(uint8_t)(orc_rng_next(r) & 0xFF);
}

int32_t orc_rng_int(orc_rng* r, int32_t lo, int32_t hi) {
    return lo + (int32_t)(orc_rng_next(r) % (uint64_t)(hi - lo + 1));
}

void orc_rng_int_fill(orc_rng* r, int32_t lo, int32_t hi, int32_t* out, int64_t count) {
    for (int64_t i = 0; i < count; ++i) out[i] = orc_rng_int(r, lo, hi);
}

double orc_rng_real(orc_rng* r, double lo, double hi) {
    return lo + (hi - lo) * ((double)(orc_rng_next(r) % 10001) / 10000.0);
}

void orc_rng_real_fill(orc_rng* r, double lo, double hi, double* out, int64_t count) {
    for (int64_t i = 0; i < count; ++i) out[i] = orc_rng_real(r, lo, hi);
}

/* ------------------------------------------------------------------ */
/* simple row-parallel helper                                          */
/* ------------------------------------------------------------------ */
typedef void (*row_fn)(void* ctx, int row_begin, int row_end);
typedef struct {
    row_fn fn;
    void* ctx;
    int begin, end;
} row_job;

static void* row_job_main(void* p) {
    row_job* j = (row_job*)p;
    j->fn(j->ctx, j->begin, j->end);
    return NULL;
}

/* Balanced contiguous split, the reference's partition_stripes
 * (engine.hpp:40-47) over rows. */
static void parallel_rows(row_fn fn, void* ctx, int rows, int threads) {
    if (threads <= 1 || rows < 2) {
        fn(ctx, 0, rows);
        return;
    }
    if (threads > rows) threads = rows;
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    row_job* jobs = (row_job*)malloc(sizeof(row_job) * threads);
    const int base = rows / threads, rem = rows % threads;
    for (int t = 0; t < threads; ++t) {
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].begin = t * base + (t < rem ? t : rem);
        jobs[t].end = jobs[t].begin + base + (t < rem ? 1 : 0);
        pthread_create(&tid[t], NULL, row_job_main, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    free(tid);
    free(jobs);
}

/* ------------------------------------------------------------------ */
/* oracle.hpp:15-30 naive_gemm_i32                                     */
/* ------------------------------------------------------------------ */
typedef struct {
    const uint8_t* a;
    int k, lda;
    const int8_t* b;
    int n, ldb;
    int32_t* c;
    int ldc;
} gemm_ctx;

static void gemm_rows(void* p, int r0, int r1) {
    const gemm_ctx* g = (const gemm_ctx*)p;
    /* i-k-j order accumulates the same int32 sum per (i,j) as i-j-k:
     * integer addition is associative modulo 2^32 and no product or
     * partial sum at these sizes leaves int32 (|sum| <= 255*128*K). */
    int32_t* row = (int32_t*)malloc(sizeof(int32_t) * (size_t)g->n);
    for (int i = r0; i < r1; ++i) {
        memset(row, 0, sizeof(int32_t) * (size_t)g->n);
        const uint8_t* ai = g->a + (size_t)i * g->lda;
        for (int kk = 0; kk < g->k; ++kk) {
            const int32_t av = ai[kk];
            const int8_t* bk = g->b + (size_t)kk * g->ldb;
            for (int j = 0; j < g->n; ++j) row[j] += av * (int32_t)bk[j];
        }
        memcpy(g->c + (size_t)i * g->ldc, row, sizeof(int32_t) * (size_t)g->n);
    }
    free(row);
}

void orc_naive_gemm_i32(const uint8_t* a, int m, int k, int lda, const int8_t* b, int n,
                        int ldb, int32_t* c, int ldc, int threads) {
    gemm_ctx g = {a, k, lda, b, n, ldb, c, ldc};
    parallel_rows(gemm_rows, &g, m, threads);
}

/* quant.hpp:98-110 */
void orc_col_offsets(const int8_t* b, int k, int n, int ldb, int32_t* out) {
    for (int j = 0; j < n; ++j) out[j] = 0;
    for (int kk = 0; kk < k; ++kk)
        for (int j = 0; j < n; ++j) out[j] += b[(size_t)kk * ldb + j];
}

/* pack.hpp:110-123: row offset = sum of the row's valid k entries,
 * accumulated over k blocks (engine.hpp:120-124) = full-K row sum. */
void orc_row_offsets(const uint8_t* a, int m, int k, int lda, int32_t* out) {
    for (int i = 0; i < m; ++i) {
        int32_t s = 0;
        for (int kk = 0; kk < k; ++kk) s += a[(size_t)i * lda + kk];
        out[i] = s;
    }
}

/* ------------------------------------------------------------------ */
/* quant.hpp:115-133 requantization                                    */
/* ------------------------------------------------------------------ */
int64_t orc_requant_adjust(int32_t acc, int32_t row_offset, int32_t col_offset, int32_t zp_a,
                           int32_t zp_b, int32_t k_total, int32_t bias) {
    int64_t adjusted = acc;
    adjusted -= (int64_t)zp_b * row_offset;
    adjusted -= (int64_t)zp_a * col_offset;
    /* quant.hpp:120: (int64)k_total * zp_a * zp_b, left to right in int64 */
    adjusted += (int64_t)k_total * zp_a * zp_b;
    adjusted += bias;
    return adjusted;
}

long long orc_round_half_away(double x) { return llround(x); }

static uint8_t clamp_u8(long long q) { return (uint8_t)(q < 0 ? 0 : (q > 255 ? 255 : q)); }

uint8_t orc_requant_scalar_ref(int32_t acc, int32_t row_offset, int32_t col_offset,
                               double multiplier, int32_t zp_a, int32_t zp_b, int32_t zp_c,
                               int32_t k_total, int32_t bias) {
    const int64_t adjusted =
        orc_requant_adjust(acc, row_offset, col_offset, zp_a, zp_b, k_total, bias);
    const long long q = orc_round_half_away(multiplier * (double)adjusted) + zp_c;
    return clamp_u8(q);
}

uint8_t orc_requant_scalar_f32(int32_t acc, int32_t row_offset, int32_t col_offset,
                               float multiplier, int32_t zp_a, int32_t zp_b, int32_t zp_c,
                               int32_t k_total, int32_t bias) {
    const int64_t adjusted =
        orc_requant_adjust(acc, row_offset, col_offset, zp_a, zp_b, k_total, bias);
    /* one RN int->float conversion, one RN fp32 multiply */
    const float x = (float)adjusted * multiplier;
    /* round to nearest, ties to even (default FE_TONEAREST) */
    float r = nearbyintf(x);
    /* only guards the float->integer conversion against UB; exact for any
     * |zp_c| <= 2^30 */
    if (r > 1099511627776.0f) r = 1099511627776.0f;
    if (r < -1099511627776.0f) r = -1099511627776.0f;
    return clamp_u8((long long)r + zp_c);
}

uint8_t orc_relu_quantized(uint8_t q, int32_t zp_c) {
    return q < zp_c ? (uint8_t)zp_c : q;
}

void orc_requant_matrix(const int32_t* acc, int m, int n, int ldacc, const int32_t* rowsum,
                        const int32_t* colsum, int32_t zp_a, const int32_t* zp_b,
                        int per_channel, int32_t k_total, const int32_t* bias, int rounding,
                        const double* mult_d, const float* mult_f, int32_t zp_c, int relu,
                        uint8_t* out, int ldo) {
    for (int i = 0; i < m; ++i) {
        const int32_t ro = rowsum ? rowsum[i] : 0;
        for (int j = 0; j < n; ++j) {
            const int jc = per_channel ? j : 0;
            const int32_t bj = bias ? bias[j] : 0;
            uint8_t q;
            if (rounding == 0)
                q = orc_requant_scalar_ref(acc[(size_t)i * ldacc + j], ro, colsum[j], mult_d[jc],
                                           zp_a, zp_b[jc], zp_c, k_total, bj);
            else
                q = orc_requant_scalar_f32(acc[(size_t)i * ldacc + j], ro, colsum[j], mult_f[jc],
                                           zp_a, zp_b[jc], zp_c, k_total, bj);
            if (relu) q = orc_relu_quantized(q, zp_c);
            out[(size_t)i * ldo + j] = q;
        }
    }
}

/* ------------------------------------------------------------------ */
/* pack.hpp:146-196 prepack_weights data layout (KAT carrier only)     */
/* ------------------------------------------------------------------ */
int64_t orc_prepack_ref_size(int k, int n, int ncb, int kcb) {
    const int64_t nk = (k + kcb - 1) / kcb, nj = (n + ncb - 1) / ncb;
    return nk * nj * (int64_t)kcb * ncb;
}

void orc_prepack_ref(const int8_t* b, int k, int n, int ldb, int ncb, int kcb, int nr,
                     int8_t* packed) {
    const int nkb = (k + kcb - 1) / kcb, njb = (n + ncb - 1) / ncb;
    memset(packed, 0, (size_t)orc_prepack_ref_size(k, n, ncb, kcb));
    for (int ki = 0; ki < nkb; ++ki) {
        const int kc = ki * kcb;
        const int k_valid = (k - kc) < kcb ? (k - kc) : kcb;
        for (int ji = 0; ji < njb; ++ji) {
            const int jc = ji * ncb;
            const int n_valid = (n - jc) < ncb ? (n - jc) : ncb;
            int8_t* block = packed + ((size_t)ki * njb + ji) * (size_t)kcb * ncb;
            for (int jp = 0; jp * nr < n_valid; ++jp) {
                int8_t* panel = block + (size_t)jp * kcb * nr;
                for (int kp = 0; 2 * kp < k_valid; ++kp) {
                    int8_t* chunk = panel + kp * 2 * nr;
                    for (int jj = 0; jj < nr && jp * nr + jj < n_valid; ++jj) {
                        const int col = jc + jp * nr + jj;
                        const int k0 = kc + 2 * kp;
                        chunk[2 * jj] = b[(size_t)k0 * ldb + col];
                        chunk[2 * jj + 1] = (k0 + 1 < kc + k_valid) ? b[(size_t)(k0 + 1) * ldb + col] : 0;
                    }
                }
            }
        }
    }
}

/* ------------------------------------------------------------------ */
/* conv3x3 via explicit im2col                      */
/* ------------------------------------------------------------------ */
typedef struct {
    const uint8_t* x;
    int h, w, c;
    uint8_t zp_a;
    uint8_t* cols;
} im2col_ctx;

static void im2col_rows(void* p, int r0, int r1) {
    const im2col_ctx* g = (const im2col_ctx*)p;
    const int kdim = 9 * g->c;
    for (int r = r0; r < r1; ++r) {
        const int img = r / (g->h * g->w), rem = r % (g->h * g->w);
        const int oh = rem / g->w, ow = rem % g->w;
        uint8_t* dst = g->cols + (size_t)r * kdim;
        for (int kh = 0; kh < 3; ++kh)
            for (int kw = 0; kw < 3; ++kw) {
                const int ih = oh + kh - 1, iw = ow + kw - 1;
                uint8_t* d = dst + (kh * 3 + kw) * g->c;
                if (ih < 0 || ih >= g->h || iw < 0 || iw >= g->w) {
                    memset(d, g->zp_a, (size_t)g->c);
                } else {
                    memcpy(d, g->x + (((size_t)img * g->h + ih) * g->w + iw) * g->c, (size_t)g->c);
                }
            }
    }
}

void orc_im2col3x3(const uint8_t* x, int nb, int h, int w, int c, uint8_t zp_a, uint8_t* cols,
                   int threads) {
    im2col_ctx g = {x, h, w, c, zp_a, cols};
    parallel_rows(im2col_rows, &g, nb * h * w, threads);
}

void orc_conv3x3_i32(const uint8_t* x, int nb, int h, int w, int c, uint8_t zp_a,
                     const int8_t* wt, int oc, int32_t* acc, int threads) {
    const int64_t rows = (int64_t)nb * h * w;
    uint8_t* cols = (uint8_t*)malloc((size_t)rows * 9 * c);
    orc_im2col3x3(x, nb, h, w, c, zp_a, cols, threads);
    orc_naive_gemm_i32(cols, (int)rows, 9 * c, 9 * c, wt, oc, oc, acc, oc, threads);
    free(cols);
}

/* ------------------------------------------------------------------ */
/* depthwise 3x3                                     */
/* ------------------------------------------------------------------ */
typedef struct {
    const uint8_t* x;
    int h, w, c;
    int32_t zp_a;
    const int8_t* wt;
    const int32_t *zp_w, *bias;
    const float* mult;
    int32_t zp_c;
    int relu;
    uint8_t* out;
    int32_t* acc_out;
    const int32_t* wsum;
} dw_ctx;

static void dw_rows(void* p, int r0, int r1) {
    const dw_ctx* g = (const dw_ctx*)p;
    for (int r = r0; r < r1; ++r) {
        const int img = r / (g->h * g->w), rem = r % (g->h * g->w);
        const int oh = rem / g->w, ow = rem % g->w;
        for (int ch = 0; ch < g->c; ++ch) {
            int32_t acc = 0, xsum = 0;
            for (int kh = 0; kh < 3; ++kh)
                for (int kw = 0; kw < 3; ++kw) {
                    const int ih = oh + kh - 1, iw = ow + kw - 1;
                    int32_t xv = g->zp_a;
                    if (ih >= 0 && ih < g->h && iw >= 0 && iw < g->w)
                        xv = g->x[(((size_t)img * g->h + ih) * g->w + iw) * g->c + ch];
                    acc += xv * (int32_t)g->wt[(kh * 3 + kw) * g->c + ch];
                    xsum += xv;
                }
            const size_t o = (size_t)r * g->c + ch;
            if (g->acc_out) g->acc_out[o] = acc;
            uint8_t q = orc_requant_scalar_f32(acc, xsum, g->wsum[ch], g->mult[ch], g->zp_a,
                                               g->zp_w[ch], g->zp_c, 9, g->bias ? g->bias[ch] : 0);
            if (g->relu) q = orc_relu_quantized(q, g->zp_c);
            g->out[o] = q;
        }
    }
}

void orc_dwconv3x3(const uint8_t* x, int nb, int h, int w, int c, int32_t zp_a,
                   const int8_t* wt, const int32_t* zp_w, const int32_t* bias, const float* mult,
                   int32_t zp_c, int relu, uint8_t* out, int32_t* acc_out, int threads) {
    int32_t* wsum = (int32_t*)malloc(sizeof(int32_t) * (size_t)c);
    orc_col_offsets(wt, 9, c, c, wsum);
    dw_ctx g = {x, h, w, c, zp_a, wt, zp_w, bias, mult, zp_c, relu, out, acc_out, wsum};
    parallel_rows(dw_rows, &g, nb * h * w, threads);
    free(wsum);
}

/* ---- outlier split + SpMDMAdd + WriteDequantF32 ---- */

/* sparse.hpp:33-58 split_outliers: column-major walk; |v| >= threshold goes to
 * the CSC part with its full value, the rest stays in dense_small.  Returns
 * nnz, or -1 if it exceeds cap (the CSC arrays are left partially filled). */
int orc_split_outliers(const int8_t* b, int k, int n, int ldb, int threshold, int8_t* dense, int ldd,
                       int32_t* col_ptr, int32_t* row_idx, int8_t* values, int cap) {
    int nnz = 0;
    col_ptr[0] = 0;
    for (int j = 0; j < n; ++j) {
        for (int kk = 0; kk < k; ++kk) {
            const int8_t v = b[(size_t)kk * ldb + j];
            const int av = v < 0 ? -(int)v : (int)v;
            if (av >= threshold) {
                if (nnz >= cap) return -1;
                row_idx[nnz] = kk;
                values[nnz] = v;
                ++nnz;
                dense[(size_t)kk * ldd + j] = 0;
            } else {
                dense[(size_t)kk * ldd + j] = v;
            }
        }
        col_ptr[j + 1] = nnz;
    }
    return nnz;
}

/* sparse.hpp:62-80 spmdm_block over the whole matrix: acc[i][j] += sum over
 * the CSC entries (k, v) of column j of A[i][k] * v (int32, wrapping) */
void orc_spmdm_add(const uint8_t* a, int m, int k, int lda, const int32_t* col_ptr, const int32_t* row_idx,
                   const int8_t* values, int n, int32_t* acc, int ldacc) {
    (void)k;
    for (int j = 0; j < n; ++j)
        for (int32_t idx = col_ptr[j]; idx < col_ptr[j + 1]; ++idx) {
            const int kk = row_idx[idx];
            const int32_t v = values[idx];
            for (int i = 0; i < m; ++i) {
                int32_t* p = &acc[(size_t)i * ldacc + j];
                *p = (int32_t)((uint32_t)*p + (uint32_t)((int32_t)a[(size_t)i * lda + kk] * v));
            }
        }
}

/* pipeline.hpp:199-207 WriteDequantF32: out = (float)(scale * (acc - zp)),
 * the int subtraction in 32-bit two's complement (the reference's int
 * arithmetic as compiled), one fp64 multiply, one RN conversion to float */
void orc_dequant_f32(const int32_t* acc, int m, int n, int ldacc, double scale, int32_t zp, float* out, int ldo) {
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
            const int32_t d = (int32_t)((uint32_t)acc[(size_t)i * ldacc + j] - (uint32_t)zp);
            out[(size_t)i * ldo + j] = (float)(scale * (double)d);
        }
}
