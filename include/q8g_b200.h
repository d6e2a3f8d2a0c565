/*
 * q8g_b200.h — C ABI of the B200-native quantized u8 x s8 -> s32 GEMM with
 * fused requantization (the FBGEMM hot path, arXiv 2101.05615).
 *
 * This is the drop-in boundary.  Each entry point replaces one reference
 * interface (cited file:line are under /root/reference/proj/include/q8gemm/
 * unless noted).  Plain pointers and sizes only; no exceptions cross the ABI:
 * every call returns a status (Q8G_OK == 0) and sets a thread-local message
 * readable with q8g_last_error().
 *
 * Pointer conventions: arguments named *_dev are device pointers on the
 * packed handle's device; *_host are host pointers.  Matrices are row-major
 * with an explicit leading dimension in elements (MatrixView, matrix.hpp:56-68).
 * `stream` is a cudaStream_t (NULL = legacy default stream).
 */
#ifndef Q8G_B200_H
#define Q8G_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define Q8G_OK 0
#define Q8G_EINVAL 1 /* std::invalid_argument in the reference (engine.hpp:66-84) */
#define Q8G_ENOMEM 2
#define Q8G_ECUDA 3
#define Q8G_ENOTSUP 4

#define Q8G_ROUND_REF 0     /* quant.hpp:127-133: fp64 multiply, round half away */
#define Q8G_ROUND_F32_RNE 1 /* fp32 multiply, round to nearest even (BASELINE)   */

typedef struct q8g_packed_b q8g_packed_b;     /* PackedWeight (pack.hpp:63-79) */
typedef struct q8g_epilogue q8g_epilogue;     /* folded OutputPipeline (pipeline.hpp:57-128) */
typedef struct q8g_kernel_cache q8g_kernel_cache; /* KernelCache (dispatch.hpp:92-146) */
typedef struct q8g_dw_filter q8g_dw_filter;   /* new: prepacked depthwise filter */
typedef struct q8g_sparse_csc q8g_sparse_csc; /* SparseWeightCSC (sparse.hpp:13-21) on a device */

/* BlockingParams (pack.hpp:15-38).  Kept for API compatibility: the packed
 * layout is the tcgen05 K-major 128B-swizzled layout whatever the blocking. */
typedef struct q8g_blocking {
    int mcb, ncb, kcb, mr, nr;
} q8g_blocking;

/* RequantParams (quant.hpp:36-43) + the Requantize stage (pipeline.hpp:33-36),
 * extended with per-output-channel zero point / scale and a rounding mode. */
typedef struct q8g_requant_params {
    double multiplier;  /* per-tensor multiplier (> 0) */
    int32_t zp_a, zp_b, zp_c;
    int32_t k_total;    /* K of the GEMM (quant.hpp:41) */
    const int32_t* bias_host;             /* N entries or NULL (quant.hpp:42) */
    const int32_t* zp_b_per_channel_host; /* N entries or NULL -> zp_b */
    const float* multiplier_f32_per_channel_host;   /* N or NULL -> (float)multiplier */
    const double* multiplier_per_channel_host;      /* N or NULL -> multiplier (REF) */
    const int32_t* col_offsets_host;      /* N or NULL -> the packed B's own colsums */
    int rounding;       /* Q8G_ROUND_REF or Q8G_ROUND_F32_RNE */
    int relu;           /* ReluQuantized stage precedes Requantize (pipeline.hpp:31,51-53) */
} q8g_requant_params;

/* ---- library / errors ---- */
const char* q8g_last_error(void);
int q8g_version(void);
/* number of CUDA kernels this library has launched in this process */
uint64_t q8g_launch_count(void);
/* per kernel family: [0] pack, [1] GEMM CUDA-core, [2] GEMM tcgen05 small-M,
 * [3] GEMM tcgen05 large-M, [4] conv CUDA-core, [5] conv tcgen05,
 * [6] depthwise CUDA-core, [7] depthwise tcgen05, [8] general-pipeline post,
 * [9] conv3x3 im2col (shapes the implicit-GEMM kernel cannot hold; the GEMM
 *     launches count under [2] / [3]), [10] depthwise FMA-pipe,
 * [11] copy-engine peer copies of q8g_gemm_u8s8_requant_peers (not kernels:
 *      not in q8g_launch_count) */
int q8g_launch_stats(uint64_t* counts, int n);
/* debug (env Q8G_TC_TRACE set): 8 globaltimer stamps per CTA of the last
 * tensor-core GEMM launch; returns the number of CTA records copied.  With
 * max_ctas > 1024 the whole 10240-word trace buffer is copied (out must hold
 * 10240 words): + per-unit stamps of CTA 0 and per-CTA conv entry/exit */
int q8g_debug_tc_trace(uint64_t* out, int max_ctas);
/* debug: SM clock64 cycles and globaltimer ns that CTA 0 of the most recent
 * large-M CTA-pair GEMM launch spent (cycles / ns = the SM clock that launch
 * ran at under the power limit) */
int q8g_debug_kernel_clock(uint64_t* cycles, uint64_t* ns);

/* ---- blocking (dispatch.hpp:17-30, pack.hpp:24-37) ---- */
int q8g_blocking_defaults(q8g_blocking* out);
int q8g_blocking_validate(const q8g_blocking* bp);
int q8g_select_blocking(int m, int n, int k, const q8g_blocking* defaults, q8g_blocking* out);
/* engine.hpp:40-47 partition_stripes */
int q8g_partition_stripes(int num_blocks, int thread_id, int num_threads, int* begin, int* end);

/* ---- weight prepack (pack.hpp:146-196 prepack_weights) ---- */
/* b_host: K x N int8 row-major (ldb >= N).  Packs on `device` into the
 * tcgen05 K-major SW128 layout and computes int32 column sums + max_abs. */
int q8g_pack_b(const int8_t* b_host, int k, int n, int ldb, const q8g_blocking* bp, int device,
               q8g_packed_b** out);
/* same from a device-resident B (on `device`), stream-ordered */
int q8g_pack_b_device(const int8_t* b_dev, int k, int n, int ldb, const q8g_blocking* bp,
                      int device, void* stream, q8g_packed_b** out);
/* copy of an immutable packed weight onto another device (row-sharded multi-GPU) */
int q8g_packed_b_replicate(const q8g_packed_b* src, int device, q8g_packed_b** out);
int q8g_packed_b_info(const q8g_packed_b* pb, int* k, int* n, int* max_abs, int* device);
int q8g_packed_b_blocking(const q8g_packed_b* pb, q8g_blocking* out);
/* ColOffsets over full K (quant.hpp:98-110), N entries */
int q8g_packed_b_col_offsets(const q8g_packed_b* pb, int32_t* out_host);
/* test-only inverse (pack.hpp:199-225 unpack_weight): K x N into out_host */
int q8g_unpack_b(const q8g_packed_b* pb, int8_t* out_host, int ldb);
int q8g_free_packed_b(q8g_packed_b* pb);

/* ---- output pipeline (pipeline.hpp:57-128) ---- */
/* Folds a validated [BiasAdd?][ReluQuantized?] Requantize pipeline into a
 * device-resident per-column table: c[j] = bias[j] + bias_add[j]
 * - zp_a*colsum[j] + K*zp_a*zp_b[j] ("combined with column
 * offsets"), zp_b[j], multiplier[j].  bias_add_host is the BiasAdd stage
 * (pipeline.hpp:27-29) or NULL. */
int q8g_epilogue_create(const q8g_packed_b* pb, const q8g_requant_params* p,
                        const int32_t* bias_add_host, q8g_epilogue** out);
int q8g_epilogue_free(q8g_epilogue* ep);

/* ---- dispatch cache (dispatch.hpp:92-146) ---- */
int q8g_kernel_cache_create(int generic_only, q8g_kernel_cache** out);
int q8g_kernel_cache_free(q8g_kernel_cache* kc);
uint64_t q8g_kernel_cache_build_count(const q8g_kernel_cache* kc);
/* tile kind chosen for a shape: 0 generic CUDA-core, 1 tcgen05 split-K
 * (when its CTAs fit two waves), 2 tcgen05 persistent CTA-pair 256 x 256 tiles
 * (at least one tile per SM pair), 3 tcgen05 128-column tiles otherwise */
int q8g_kernel_cache_tile(q8g_kernel_cache* kc, int m, int n, int k, int lda, int* tile_kind);

/* ---- GEMM (engine.hpp:59-169 execute_gemm) ----
 * Computes output rows [row_begin, row_end) of C = requant(A x B): one
 * worker's stripe (row_begin=0,row_end=M for the whole matrix).  A is M x K
 * u8 (lda), C is M x N (ldc).  `cache` NULL = the process cache. */
int q8g_gemm_u8s8_requant(const uint8_t* a_dev, int m, int k, int lda, const q8g_packed_b* pb,
                          const q8g_epilogue* ep, uint8_t* c_dev, int ldc, int row_begin,
                          int row_end, q8g_kernel_cache* cache, void* stream);
/* N-sharded multi-GPU (optional N-sharding; no reference
 * symbol -- the reference splits only M: engine.hpp:39-47,102-103).  Same as
 * q8g_gemm_u8s8_requant for one column shard (pb packs B[:, n0:n1] on this
 * device, ep its columns), and the stripe is ALSO written at each of the
 * n_peers (0..7) pointers: other devices' C windows at the same shard offset
 * (UVA device pointers, same ldc), so after every rank has run its shard each
 * rank holds the whole M x N output -- an all-gather with no separate pass.
 * The CTA-pair kernel stores each tile to the peers straight from its
 * staging tile (TMA stores over NVLink, overlapped with the GEMM); other
 * kernels copy the finished stripe with the copy engines.  Peer access is
 * enabled on first use; between devices with no P2P path every peer gets a
 * staged copy instead.  Completion on the peers is ordered by `stream`:
 * the caller synchronises the ranks (e.g. a barrier after a stream sync)
 * before reading the gathered output. */
int q8g_gemm_u8s8_requant_peers(const uint8_t* a_dev, int m, int k, int lda, const q8g_packed_b* pb,
                                const q8g_epilogue* ep, uint8_t* c_dev, uint8_t* const* c_peer_dev,
                                int n_peers, int ldc, int row_begin, int row_end,
                                q8g_kernel_cache* cache, void* stream);
/* WriteRawI32 writer (pipeline.hpp:38,191-198); bias_add_dev = optional
 * BiasAdd stage (N int32, device) or NULL */
int q8g_gemm_u8s8_raw_i32(const uint8_t* a_dev, int m, int k, int lda, const q8g_packed_b* pb,
                          const int32_t* bias_add_dev, int32_t* c_dev, int ldc, int row_begin,
                          int row_end, q8g_kernel_cache* cache, void* stream);
/* Host-buffer convenience (the reference calling convention: host views).
 * Stages A to the device, runs, and copies C back, synchronously.  Stripes
 * of >= 4096 rows go in chunks whose H2D / D2H copies overlap the GEMM of
 * the neighbouring chunks. */
int q8g_gemm_u8s8_requant_host(const uint8_t* a_host, int m, int k, int lda,
                               const q8g_packed_b* pb, const q8g_epilogue* ep, uint8_t* c_host,
                               int ldc, int row_begin, int row_end, void* stream);
int q8g_gemm_u8s8_raw_i32_host(const uint8_t* a_host, int m, int k, int lda,
                               const q8g_packed_b* pb, int32_t* c_host, int ldc, int row_begin,
                               int row_end, void* stream);

/* ---- outlier split + general output pipeline ----
 * split_outliers (sparse.hpp:33-58), host side: entries with |v| >= threshold
 * go to a CSC store with their full value (column-major walk), the rest stay
 * in dense (k x n, ldd).  CSC arrays are caller buffers of capacity cap
 * (col_ptr n+1 entries); *nnz_out = the outlier count (Q8G_EINVAL if it
 * exceeds cap: call with cap 0 first to size).  Errors follow the
 * reference: threshold >= 1, non-empty matrix. */
int q8g_split_outliers(const int8_t* b_host, int k, int n, int ldb, int threshold, int8_t* dense_host, int ldd,
                       int32_t* col_ptr, int32_t* row_idx, int8_t* values, int cap, int* nnz_out);
/* SparseWeightCSC (sparse.hpp:13-21) uploaded to `device` (validated:
 * col_ptr nondecreasing from 0 to nnz, row_idx in [0,k) and strictly
 * increasing within a column) */
int q8g_sparse_csc_create(const int32_t* col_ptr_host, const int32_t* row_idx_host, const int8_t* values_host,
                          int nnz, int k, int n, int device, q8g_sparse_csc** out);
int q8g_sparse_csc_free(q8g_sparse_csc* sp);

enum { Q8G_WRITE_RAW_I32 = 0, Q8G_WRITE_REQUANT_U8 = 1, Q8G_WRITE_DEQUANT_F32 = 2 };
typedef struct q8g_pipeline_args {
    const q8g_sparse_csc* sparse;  /* SpMDMAdd stage (pipeline.hpp:23-25) or NULL */
    const int32_t* bias_add_dev;   /* summed BiasAdd stages (N int32, device) for the raw /
                                      dequant writers, or NULL; the requant writer takes
                                      them folded into its epilogue (q8g_epilogue_create) */
    int writer;                    /* Q8G_WRITE_* */
    const q8g_epilogue* ep;        /* Q8G_WRITE_REQUANT_U8 ([ReluQuantized] Requantize) */
    double dq_scale;               /* Q8G_WRITE_DEQUANT_F32: QuantParams (quant.hpp:18-21) */
    int32_t dq_zero_point;
} q8g_pipeline_args;
/* execute_gemm with the general pipeline [SpMDMAdd] [BiasAdd]* [ReluQuantized]
 * writer (pipeline.hpp:157-207).  c_dev is int32 / u8 / float per the writer
 * (ldc in elements).  The dense product runs on the tensor-core kernels. */
int q8g_gemm_u8s8_pipeline(const uint8_t* a_dev, int m, int k, int lda, const q8g_packed_b* pb,
                           const q8g_pipeline_args* pl, void* c_dev, int ldc, int row_begin, int row_end,
                           q8g_kernel_cache* cache, void* stream);
/* host views (the reference convention), synchronous: A rows and C rows of
 * the stripe are staged through the device; bias_add_host replaces
 * pl->bias_add_dev (which must be NULL) */
int q8g_gemm_u8s8_pipeline_host(const uint8_t* a_host, int m, int k, int lda, const q8g_packed_b* pb,
                                const q8g_pipeline_args* pl, const int32_t* bias_add_host, void* c_host, int ldc,
                                int row_begin, int row_end, void* stream);

/* ---- conv 3x3, stride 1, pad 1, NHWC (new) ----
 * x: [nb][h][w][c] u8 (device), padding value = zp_a of the epilogue.
 * pw: the weight [3][3][c][oc] packed as a K=9c x N=oc matrix.
 * y: [nb][h][w][oc] u8.  Images [img_begin, img_end) are computed. */
int q8g_conv3x3_u8s8_nhwc(const uint8_t* x_dev, int nb, int h, int w, int c,
                          const q8g_packed_b* pw, const q8g_epilogue* ep, uint8_t* y_dev,
                          int img_begin, int img_end, void* stream);
/* build, once and synchronously, the derived tensor-core operand image of a
 * conv weight for c input channels (pw->k == 9c); the first conv call does it
 * otherwise (and must then not be inside a stream capture).  After it the
 * weight is used read-only by any number of concurrent streams. */
int q8g_conv3x3_prepare(const q8g_packed_b* pw, int c, void* stream);
int q8g_conv3x3_u8s8_nhwc_raw_i32(const uint8_t* x_dev, int nb, int h, int w, int c,
                                  int32_t zp_a, const q8g_packed_b* pw, int32_t* y_dev,
                                  int img_begin, int img_end, void* stream);
/* host views (the reference calling convention, engine.hpp:59-62): images of
 * x_host / y_host are staged through the device in chunks whose copies
 * overlap the previous chunk's convolution; synchronous */
int q8g_conv3x3_u8s8_nhwc_host(const uint8_t* x_host, int nb, int h, int w, int c,
                               const q8g_packed_b* pw, const q8g_epilogue* ep, uint8_t* y_host,
                               int img_begin, int img_end, void* stream);

/* ---- depthwise 3x3, stride 1, pad 1, NHWC (new) ----
 * w_host: [3][3][c] s8.  Requant params are per channel (k_total = 9). */
int q8g_dw_filter_create(const int8_t* w_host, int c, const q8g_requant_params* p, int device,
                         q8g_dw_filter** out);
int q8g_dw_filter_free(q8g_dw_filter* f);
int q8g_dwconv3x3_u8s8_nhwc(const uint8_t* x_dev, int nb, int h, int w, int c,
                            const q8g_dw_filter* f, uint8_t* y_dev, int img_begin, int img_end,
                            void* stream);
/* host views, chunked and overlapped like q8g_conv3x3_u8s8_nhwc_host */
int q8g_dwconv3x3_u8s8_nhwc_host(const uint8_t* x_host, int nb, int h, int w, int c,
                                 const q8g_dw_filter* f, uint8_t* y_host, int img_begin, int img_end,
                                 void* stream);

#ifdef __cplusplus
}
#endif
#endif /* Q8G_B200_H */
