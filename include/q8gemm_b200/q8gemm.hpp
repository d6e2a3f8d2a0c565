// q8gemm.hpp — header-only C++ mirror of the reference q8gemm API on the
// B200 C ABI (q8g_b200.h).  Same names, argument meaning and error behaviour
// (std::invalid_argument with the reference's messages) as
// /root/reference/proj/include/q8gemm/{matrix,pack,dispatch,pipeline,engine}.hpp,
// so a C++ caller switches by changing the include and the namespace:
//
//   q8gemm::execute_gemm(a, pw, out, pipeline, kAccI32, t, nt)      (engine.hpp:59-62)
//   q8gemm_b200::execute_gemm(a, pw, out, pipeline, kAccI32, t, nt)
//
// Host views (MatrixView) follow the reference calling convention: A is
// staged to the GPU and the result copied back, synchronously.  Device views
// (DeviceView) are the zero-copy, stream-ordered path.  Extensions: per-channel
// zero points / fp32 multipliers and the rounding mode on RequantParams,
// conv3x3 / depthwise-3x3 entry points.  Requires C++17.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <map>
#include <type_traits>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "../q8g_b200.h"

namespace q8gemm_b200 {

// ------------------------------------------------------------------ errors

inline void check(int rc) {
    if (rc == Q8G_OK) return;
    const std::string msg = q8g_last_error();
    if (rc == Q8G_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// ------------------------------------------------------------------ matrix.hpp

constexpr int round_up(int value, int multiple) { return ((value + multiple - 1) / multiple) * multiple; }
constexpr int ceil_div(int value, int divisor) { return (value + divisor - 1) / divisor; }

template <typename T>
class Matrix {
public:
    Matrix() = default;
    Matrix(int rows, int cols, T fill = T{})
        : rows_(rows), cols_(cols), data_(static_cast<std::size_t>(rows) * static_cast<std::size_t>(cols), fill) {
        if (rows < 1 || cols < 1) throw std::invalid_argument("Matrix: dimensions must be >= 1");
    }
    int rows() const { return rows_; }
    int cols() const { return cols_; }
    T& operator()(int r, int c) { return data_[static_cast<std::size_t>(r) * cols_ + c]; }
    const T& operator()(int r, int c) const { return data_[static_cast<std::size_t>(r) * cols_ + c]; }
    T* data() { return data_.data(); }
    const T* data() const { return data_.data(); }
    bool operator==(const Matrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_ && data_ == o.data_; }

private:
    int rows_ = 0, cols_ = 0;
    std::vector<T> data_;
};

// Non-owning view of a row-major HOST matrix; ld >= cols.
template <typename T>
struct MatrixView {
    T* data = nullptr;
    int rows = 0, cols = 0, ld = 0;
    T& operator()(int r, int c) const { return data[static_cast<std::size_t>(r) * ld + c]; }
    bool empty() const { return data == nullptr; }
};

// Non-owning view of a row-major DEVICE matrix (on the packed weight's device).
template <typename T>
struct DeviceView {
    T* data = nullptr;
    int rows = 0, cols = 0, ld = 0;
};

template <typename T>
MatrixView<T> view(Matrix<T>& m) { return {m.data(), m.rows(), m.cols(), m.cols()}; }
template <typename T>
MatrixView<const T> cview(const Matrix<T>& m) { return {m.data(), m.rows(), m.cols(), m.cols()}; }
template <typename T>
MatrixView<T> subview(const MatrixView<T>& m, int row0, int col0, int rows, int cols) {
    return {m.data + static_cast<std::size_t>(row0) * m.ld + col0, rows, cols, m.ld};
}

// ------------------------------------------------------------------ pack.hpp / dispatch.hpp

struct BlockingParams {
    int mcb = 56, ncb = 32, kcb = 256, mr = 14, nr = 32;
    static BlockingParams defaults() { return BlockingParams{}; }
    q8g_blocking c() const { return q8g_blocking{mcb, ncb, kcb, mr, nr}; }
    void validate() const {
        const q8g_blocking b = c();
        check(q8g_blocking_validate(&b));
    }
};

inline BlockingParams select_blocking(int m, int n, int k, const BlockingParams& defaults) {
    const q8g_blocking d = defaults.c();
    q8g_blocking out{};
    check(q8g_select_blocking(m, n, k, &d, &out));
    return BlockingParams{out.mcb, out.ncb, out.kcb, out.mr, out.nr};
}

enum class KernelVariant { kAccI32, kAccI16 };  // kernel.hpp:9-12

constexpr bool i16_accumulation_exact(int32_t max_abs_b, int kcb) { return 255LL * max_abs_b * kcb <= 32767; }

// pack.hpp:63-79: immutable after construction, shareable across calls,
// device resident (tcgen05 K-major SW128 layout + column sums).
class PackedWeight {
public:
    PackedWeight() = default;
    explicit PackedWeight(q8g_packed_b* h) : h_(h, &q8g_free_packed_b) {
        int k = 0, n = 0, mx = 0, dev = 0;
        check(q8g_packed_b_info(h, &k, &n, &mx, &dev));
        k_total = k;
        n_total = n;
        max_abs = mx;
        device = dev;
        q8g_blocking b{};
        check(q8g_packed_b_blocking(h, &b));
        blocking = BlockingParams{b.mcb, b.ncb, b.kcb, b.mr, b.nr};
        col_offsets.assign(n, 0);
        check(q8g_packed_b_col_offsets(h, col_offsets.data()));
    }
    q8g_packed_b* handle() const { return h_.get(); }
    Matrix<int8_t> unpack() const {  // pack.hpp:199-225 (test-only inverse)
        Matrix<int8_t> b(k_total, n_total, 0);
        check(q8g_unpack_b(handle(), b.data(), n_total));
        return b;
    }
    PackedWeight replicate(int dev) const {
        q8g_packed_b* r = nullptr;
        check(q8g_packed_b_replicate(handle(), dev, &r));
        return PackedWeight(r);
    }

    int k_total = 0, n_total = 0, max_abs = 0, device = 0;
    BlockingParams blocking;
    std::vector<int32_t> col_offsets;  // ColOffsets over the full K

private:
    std::shared_ptr<q8g_packed_b> h_;
};

inline PackedWeight prepack_weights(MatrixView<const int8_t> b, const BlockingParams& bp, int device = 0) {
    bp.validate();
    if (b.rows < 1 || b.cols < 1) throw std::invalid_argument("prepack_weights: matrix must be non-empty");
    const q8g_blocking c = bp.c();
    q8g_packed_b* h = nullptr;
    check(q8g_pack_b(b.data, b.rows, b.cols, b.ld, &c, device, &h));
    return PackedWeight(h);
}

// dispatch.hpp:92-146 analog: memoized shape class -> GPU tile kind
class KernelCache {
public:
    explicit KernelCache(bool generic_only = false) {
        q8g_kernel_cache* h = nullptr;
        check(q8g_kernel_cache_create(generic_only ? 1 : 0, &h));
        h_.reset(h, &q8g_kernel_cache_free);
    }
    uint64_t build_count() const { return q8g_kernel_cache_build_count(h_.get()); }
    q8g_kernel_cache* handle() const { return h_.get(); }

private:
    std::shared_ptr<q8g_kernel_cache> h_;
};

// ------------------------------------------------------------------ quant.hpp / pipeline.hpp

enum class Rounding { kRef = Q8G_ROUND_REF, kF32Rne = Q8G_ROUND_F32_RNE };

// quant.hpp:36-43 + per-channel extension
struct RequantParams {
    double multiplier = 1.0;
    int32_t zp_a = 0, zp_b = 0, zp_c = 0, k_total = 1;
    std::vector<int32_t> bias;                   // per column, pre-scaling; empty = none
    std::vector<int32_t> zp_b_per_channel;       // empty -> zp_b
    std::vector<float> multiplier_f32_per_channel;  // empty -> (float)multiplier
    std::vector<double> multiplier_per_channel;  // empty -> multiplier
    Rounding rounding = Rounding::kRef;
};

struct QuantParams {  // quant.hpp:18-21
    double scale = 1.0;
    int32_t zero_point = 0;
};

// quant.hpp:45-47: ties away from zero (std::llround)
inline long long round_half_away_from_zero(double x) { return std::llround(x); }

// quant.hpp:64-82: affine params covering [min(lo, 0), max(hi, 0)]
inline QuantParams choose_quant_params(double min_val, double max_val, bool is_signed) {
    if (!std::isfinite(min_val) || !std::isfinite(max_val))
        throw std::invalid_argument("choose_quant_params: range bounds must be finite");
    if (min_val > max_val) throw std::invalid_argument("choose_quant_params: min_val must be <= max_val");
    const double lo = std::min(min_val, 0.0), hi = std::max(max_val, 0.0);
    const int qlo = is_signed ? -128 : 0, qhi = is_signed ? 127 : 255;
    QuantParams qp;
    qp.scale = hi == lo ? 1.0 : (hi - lo) / (qhi - qlo);
    qp.zero_point = static_cast<int32_t>(std::clamp<long long>(round_half_away_from_zero(qlo - lo / qp.scale), qlo, qhi));
    return qp;
}

// quant.hpp:84-95
template <typename Q>
Q quantize(double x, const QuantParams& qp) {
    static_assert(sizeof(Q) == 1, "8-bit types only");
    const long long lo = std::is_signed<Q>::value ? -128 : 0, hi = std::is_signed<Q>::value ? 127 : 255;
    return static_cast<Q>(std::clamp<long long>(round_half_away_from_zero(x / qp.scale) + qp.zero_point, lo, hi));
}
inline double dequantize(int q, const QuantParams& qp) { return qp.scale * (q - qp.zero_point); }

// quant.hpp:98-110 (host; the packed weight carries its own on the device)
inline std::vector<int32_t> compute_col_offsets(MatrixView<const int8_t> b) {
    if (b.rows < 1 || b.cols < 1) throw std::invalid_argument("compute_col_offsets: matrix must be non-empty");
    std::vector<int32_t> co(b.cols, 0);
    for (int k = 0; k < b.rows; ++k)
        for (int j = 0; j < b.cols; ++j) co[j] += b(k, j);
    return co;
}

// kernel.hpp:34-36: largest T with 255 * (T - 1) * kcb <= 32767
constexpr int max_i16_split_threshold(int kcb) { return 1 + 32767 / (255 * kcb); }

// sparse.hpp:13-21 (host arrays; uploaded once per device on first use)
struct SparseWeightCSC {
    std::vector<int32_t> col_ptr;  // n_total + 1, nondecreasing
    std::vector<int32_t> row_idx;  // strictly increasing within each column
    std::vector<int8_t> values;
    int k_total = 0;
    int n_total = 0;
    int nnz() const { return static_cast<int>(values.size()); }
    q8g_sparse_csc* device(int dev) const {  // thread-safe: workers may race on first use
        std::lock_guard<std::mutex> lock(*mu_);
        auto it = dev_.find(dev);
        if (it != dev_.end()) return it->second.get();
        q8g_sparse_csc* h = nullptr;
        check(q8g_sparse_csc_create(col_ptr.data(), row_idx.empty() ? nullptr : row_idx.data(),
                                    values.empty() ? nullptr : values.data(), nnz(), k_total, n_total, dev, &h));
        dev_.emplace(dev, std::shared_ptr<q8g_sparse_csc>(h, &q8g_sparse_csc_free));
        return h;
    }

private:
    std::shared_ptr<std::mutex> mu_ = std::make_shared<std::mutex>();
    mutable std::map<int, std::shared_ptr<q8g_sparse_csc>> dev_;
};

struct SplitWeight {  // sparse.hpp:23-29
    Matrix<int8_t> dense_small;
    SparseWeightCSC sparse;
    int threshold = 0;
};

// sparse.hpp:33-58: B = dense_small + outliers (|v| >= threshold, CSC)
inline SplitWeight split_outliers(MatrixView<const int8_t> b, int threshold) {
    int nnz = 0;
    check(q8g_split_outliers(b.data, b.rows, b.cols, b.ld, threshold, nullptr, b.cols, nullptr, nullptr, nullptr, 0,
                             &nnz));
    SplitWeight sw;
    sw.threshold = threshold;
    sw.dense_small = Matrix<int8_t>(b.rows, b.cols);
    sw.sparse.k_total = b.rows;
    sw.sparse.n_total = b.cols;
    sw.sparse.col_ptr.assign(b.cols + 1, 0);
    sw.sparse.row_idx.assign(std::max(nnz, 1), 0);
    sw.sparse.values.assign(std::max(nnz, 1), 0);
    check(q8g_split_outliers(b.data, b.rows, b.cols, b.ld, threshold, sw.dense_small.data(), b.cols,
                             sw.sparse.col_ptr.data(), sw.sparse.row_idx.data(), sw.sparse.values.data(),
                             std::max(nnz, 1), &nnz));
    sw.sparse.row_idx.resize(nnz);
    sw.sparse.values.resize(nnz);
    return sw;
}

struct SpMDMAdd {  // pipeline.hpp:23-25
    const SparseWeightCSC* sparse = nullptr;
};
struct BiasAdd {  // pipeline.hpp:27-29
    std::vector<int32_t> bias;
};
struct ReluQuantized {};  // pipeline.hpp:31
struct Requantize {       // pipeline.hpp:33-36
    RequantParams params;
    const std::vector<int32_t>* col_offsets = nullptr;  // nullptr -> the packed weight's own
};
struct WriteRawI32 {};  // pipeline.hpp:38
struct WriteDequantF32 {  // pipeline.hpp:40-42: scale * (acc - zero_point)
    QuantParams c_params;
};

using OutputStage = std::variant<SpMDMAdd, BiasAdd, ReluQuantized, Requantize, WriteRawI32, WriteDequantF32>;
enum class WriterKind { kRawI32, kRequantizeU8, kDequantF32 };

class OutputPipeline {
public:
    explicit OutputPipeline(std::vector<OutputStage> stages) : stages_(std::move(stages)) {
        if (auto err = validate(stages_)) throw std::invalid_argument("OutputPipeline: " + *err);
    }
    // pipeline.hpp:66-102 (same rules and messages)
    static std::optional<std::string> validate(const std::vector<OutputStage>& stages) {
        if (stages.empty()) return std::string("pipeline is empty; a terminal writer stage is required");
        auto is_writer = [](const OutputStage& s) {
            return std::holds_alternative<Requantize>(s) || std::holds_alternative<WriteRawI32>(s) ||
                   std::holds_alternative<WriteDequantF32>(s);
        };
        for (std::size_t i = 0; i + 1 < stages.size(); ++i)
            if (is_writer(stages[i]))
                return "stage " + std::to_string(i + 1) + " follows a writer; the writer must be the last stage";
        if (!is_writer(stages.back()))
            return std::string("last stage must be a writer (Requantize, WriteRawI32, or WriteDequantF32)");
        for (std::size_t i = 0; i < stages.size(); ++i) {
            if (std::holds_alternative<ReluQuantized>(stages[i])) {
                const bool ok = i + 2 == stages.size() && std::holds_alternative<Requantize>(stages.back());
                if (!ok) return std::string("ReluQuantized must immediately precede a Requantize writer");
            }
            if (const auto* sp = std::get_if<SpMDMAdd>(&stages[i]))
                if (sp->sparse == nullptr) return std::string("SpMDMAdd requires a sparse matrix");
            if (const auto* rq = std::get_if<Requantize>(&stages[i])) {
                const RequantParams& p = rq->params;
                if (!(p.multiplier > 0) && p.multiplier_f32_per_channel.empty() && p.multiplier_per_channel.empty())
                    return std::string("Requantize multiplier must be positive");
                if (p.k_total < 1) return std::string("Requantize k_total must be >= 1");
            }
        }
        return std::nullopt;
    }
    const std::vector<OutputStage>& stages() const { return stages_; }
    WriterKind writer() const {
        if (std::holds_alternative<WriteRawI32>(stages_.back())) return WriterKind::kRawI32;
        if (std::holds_alternative<Requantize>(stages_.back())) return WriterKind::kRequantizeU8;
        return WriterKind::kDequantF32;
    }
    const SparseWeightCSC* sparse() const {
        for (const auto& s : stages_)
            if (const auto* sp = std::get_if<SpMDMAdd>(&s)) return sp->sparse;
        return nullptr;
    }
    // an SpMDMAdd stage or the WriteDequantF32 writer: the general path (post.cu)
    bool general() const { return sparse() != nullptr || writer() == WriterKind::kDequantF32; }
    // the C-ABI description of the general pipeline (bias_add / ep filled by the caller)
    q8g_pipeline_args args(int device) const {
        q8g_pipeline_args pa{};
        const SparseWeightCSC* sp = sparse();
        pa.sparse = sp ? sp->device(device) : nullptr;
        pa.writer = writer() == WriterKind::kRawI32        ? Q8G_WRITE_RAW_I32
                    : writer() == WriterKind::kRequantizeU8 ? Q8G_WRITE_REQUANT_U8
                                                            : Q8G_WRITE_DEQUANT_F32;
        if (const auto* dq = std::get_if<WriteDequantF32>(&stages_.back())) {
            pa.dq_scale = dq->c_params.scale;
            pa.dq_zero_point = dq->c_params.zero_point;
        }
        return pa;
    }
    bool needs_row_offsets() const {  // pipeline.hpp:114-119
        if (const auto* rq = std::get_if<Requantize>(&stages_.back())) {
            for (int32_t z : rq->params.zp_b_per_channel)
                if (z != 0) return true;
            return rq->params.zp_b_per_channel.empty() && rq->params.zp_b != 0;
        }
        return false;
    }
    bool has_relu() const {
        return stages_.size() >= 2 && std::holds_alternative<ReluQuantized>(stages_[stages_.size() - 2]);
    }
    std::vector<int32_t> bias_add(int n) const {
        std::vector<int32_t> acc;
        for (const auto& s : stages_)
            if (const auto* b = std::get_if<BiasAdd>(&s)) {
                if ((int)b->bias.size() != n) throw std::invalid_argument("BiasAdd: bias must have N entries");
                if (acc.empty()) acc.assign(n, 0);
                for (int j = 0; j < n; ++j) acc[j] = (int32_t)((uint32_t)acc[j] + (uint32_t)b->bias[j]);
            }
        return acc;
    }
    // folded device epilogue for one packed weight (cached; the pipeline is immutable)
    q8g_epilogue* epilogue(const PackedWeight& pw) const {  // thread-safe: workers share the pipeline
        std::lock_guard<std::mutex> lock(*mu_);
        auto it = eps_.find(pw.handle());
        if (it != eps_.end()) return it->second.get();
        const auto& rq = std::get<Requantize>(stages_.back());
        const RequantParams& p = rq.params;
        const int n = pw.n_total;
        auto need = [&](std::size_t sz, const char* what) {
            if (sz != 0 && (int)sz != n) throw std::invalid_argument(std::string("Requantize: ") + what + " must have N entries");
        };
        need(p.bias.size(), "bias");
        need(p.zp_b_per_channel.size(), "zp_b_per_channel");
        need(p.multiplier_f32_per_channel.size(), "multiplier_f32_per_channel");
        need(p.multiplier_per_channel.size(), "multiplier_per_channel");
        if (rq.col_offsets) need(rq.col_offsets->size(), "col_offsets");
        q8g_requant_params c{};
        c.multiplier = p.multiplier;
        c.zp_a = p.zp_a;
        c.zp_b = p.zp_b;
        c.zp_c = p.zp_c;
        c.k_total = p.k_total;
        c.bias_host = p.bias.empty() ? nullptr : p.bias.data();
        c.zp_b_per_channel_host = p.zp_b_per_channel.empty() ? nullptr : p.zp_b_per_channel.data();
        c.multiplier_f32_per_channel_host =
            p.multiplier_f32_per_channel.empty() ? nullptr : p.multiplier_f32_per_channel.data();
        c.multiplier_per_channel_host = p.multiplier_per_channel.empty() ? nullptr : p.multiplier_per_channel.data();
        c.col_offsets_host = rq.col_offsets ? rq.col_offsets->data() : nullptr;
        c.rounding = static_cast<int>(p.rounding);
        c.relu = has_relu() ? 1 : 0;
        const std::vector<int32_t> ba = bias_add(n);
        q8g_epilogue* e = nullptr;
        check(q8g_epilogue_create(pw.handle(), &c, ba.empty() ? nullptr : ba.data(), &e));
        eps_.emplace(pw.handle(), std::shared_ptr<q8g_epilogue>(e, &q8g_epilogue_free));
        keep_.push_back(pw);  // the handle key stays valid while cached
        return e;
    }

private:
    std::vector<OutputStage> stages_;
    std::shared_ptr<std::mutex> mu_ = std::make_shared<std::mutex>();
    mutable std::map<q8g_packed_b*, std::shared_ptr<q8g_epilogue>> eps_;
    mutable std::vector<PackedWeight> keep_;
};

// ------------------------------------------------------------------ engine.hpp

namespace detail {
constexpr int kTileRows = 128;  // stripe granularity: one tcgen05 M tile

template <typename OutT>
void check_writer_matches(const OutputPipeline& p) {  // pipeline.hpp:142-151
    const bool ok = (std::is_same<OutT, int32_t>::value && p.writer() == WriterKind::kRawI32) ||
                    (std::is_same<OutT, uint8_t>::value && p.writer() == WriterKind::kRequantizeU8) ||
                    (std::is_same<OutT, float>::value && p.writer() == WriterKind::kDequantF32);
    if (!ok) throw std::invalid_argument("pipeline writer does not match the output element type");
}

template <typename V>
std::pair<int, int> stripe_rows(int m, int thread_id, int num_threads) {
    int b = 0, e = 0;
    check(q8g_partition_stripes(ceil_div(m, kTileRows), thread_id, num_threads, &b, &e));
    return {std::min(b * kTileRows, m), std::min(e * kTileRows, m)};
}

template <typename OutT, typename AView, typename OView>
void validate(const AView& a, const PackedWeight& pw, const OView& out, const OutputPipeline& pipeline,
              KernelVariant variant, int thread_id, int num_threads) {
    if (a.cols != pw.k_total) throw std::invalid_argument("execute_gemm: A columns must equal the packed weight K");
    if (out.rows != a.rows || out.cols != pw.n_total) throw std::invalid_argument("execute_gemm: output must be M x N");
    if (num_threads < 1 || thread_id < 0 || thread_id >= num_threads)
        throw std::invalid_argument("execute_gemm: thread_id must be in [0, num_threads)");
    check_writer_matches<OutT>(pipeline);
    if (variant == KernelVariant::kAccI16 && !i16_accumulation_exact(pw.max_abs, pw.blocking.kcb))
        throw std::invalid_argument(
            "execute_gemm: INT16 accumulation rejected: 255 * max|B| * kcb = " +
            std::to_string(255LL * pw.max_abs * pw.blocking.kcb) +
            " exceeds 32767; split outliers with a threshold satisfying "
            "255 * (T - 1) * kcb <= 32767 (see max_i16_split_threshold)");
}
}  // namespace detail

// engine.hpp:59-62 with HOST views (the reference calling convention).  A
// kAccI16 request is accepted when the reference would accept it and runs the
// exact int32 path (bit-identical).  KernelCache* selects the dispatch table.
template <typename OutT>
void execute_gemm(MatrixView<const uint8_t> a, const PackedWeight& pw, MatrixView<OutT> out,
                  const OutputPipeline& pipeline, KernelVariant variant, int thread_id, int num_threads,
                  KernelCache* cache = nullptr) {
    (void)cache;  // host views always stage through the library's own dispatch
    detail::validate<OutT>(a, pw, out, pipeline, variant, thread_id, num_threads);
    const auto r = detail::stripe_rows<int>(a.rows, thread_id, num_threads);
    if (r.first >= r.second) return;
    if (pipeline.general() || (std::is_same<OutT, int32_t>::value && !pipeline.bias_add(pw.n_total).empty())) {
        // [SpMDMAdd] [BiasAdd]* writer (pipeline.hpp:157-207), staged synchronously
        q8g_pipeline_args pa = pipeline.args(pw.device);
        std::vector<int32_t> ba;
        if (pipeline.writer() == WriterKind::kRequantizeU8)
            pa.ep = pipeline.epilogue(pw);  // BiasAdd folded into the epilogue table
        else
            ba = pipeline.bias_add(pw.n_total);
        check(q8g_gemm_u8s8_pipeline_host(a.data, a.rows, a.cols, a.ld, pw.handle(), &pa, ba.empty() ? nullptr : ba.data(),
                                          out.data, out.ld, r.first, r.second, nullptr));
        return;
    }
    if constexpr (std::is_same<OutT, int32_t>::value) {
        check(q8g_gemm_u8s8_raw_i32_host(a.data, a.rows, a.cols, a.ld, pw.handle(), out.data, out.ld, r.first,
                                         r.second, nullptr));
    } else if constexpr (std::is_same<OutT, uint8_t>::value) {
        check(q8g_gemm_u8s8_requant_host(a.data, a.rows, a.cols, a.ld, pw.handle(), pipeline.epilogue(pw), out.data,
                                         out.ld, r.first, r.second, nullptr));
    }
}

// Device views: stream-ordered, no copies (the timed path).
template <typename OutT>
void execute_gemm(DeviceView<const uint8_t> a, const PackedWeight& pw, DeviceView<OutT> out,
                  const OutputPipeline& pipeline, KernelVariant variant, int thread_id, int num_threads,
                  KernelCache* cache = nullptr, void* stream = nullptr, const int32_t* bias_add_dev = nullptr) {
    detail::validate<OutT>(a, pw, out, pipeline, variant, thread_id, num_threads);
    const auto r = detail::stripe_rows<int>(a.rows, thread_id, num_threads);
    if (r.first >= r.second) return;
    q8g_kernel_cache* kc = cache ? cache->handle() : nullptr;
    if (pipeline.general()) {
        // [SpMDMAdd] [BiasAdd]* writer; BiasAdd: bias_add_dev (raw / dequant) or the epilogue (requant)
        q8g_pipeline_args pa = pipeline.args(pw.device);
        if (pipeline.writer() == WriterKind::kRequantizeU8)
            pa.ep = pipeline.epilogue(pw);
        else
            pa.bias_add_dev = bias_add_dev;
        check(q8g_gemm_u8s8_pipeline(a.data, a.rows, a.cols, a.ld, pw.handle(), &pa, out.data, out.ld, r.first,
                                     r.second, kc, stream));
        return;
    }
    if constexpr (std::is_same<OutT, int32_t>::value) {
        check(q8g_gemm_u8s8_raw_i32(a.data, a.rows, a.cols, a.ld, pw.handle(), bias_add_dev, out.data, out.ld,
                                    r.first, r.second, kc, stream));
    } else if constexpr (std::is_same<OutT, uint8_t>::value) {
        check(q8g_gemm_u8s8_requant(a.data, a.rows, a.cols, a.ld, pw.handle(), pipeline.epilogue(pw), out.data,
                                    out.ld, r.first, r.second, kc, stream));
    }
}

// N-sharded multi-GPU (optional; no reference counterpart):
// columns [col0, col0 + pw.n_total) of the output -- pw packs that column
// shard of B on this device -- go to `out` (this device's whole M x N output)
// and to every peer output at the same offset (UVA device pointers of buffers
// with out's leading dimension, up to 7).  See q8g_gemm_u8s8_requant_peers.
inline void execute_gemm_to_peers(DeviceView<const uint8_t> a, const PackedWeight& pw, DeviceView<uint8_t> out,
                                  const std::vector<uint8_t*>& peers, int col0, const OutputPipeline& pipeline,
                                  KernelCache* cache = nullptr, void* stream = nullptr) {
    if (a.cols != pw.k_total) throw std::invalid_argument("execute_gemm: A columns must equal the packed weight K");
    if (out.rows != a.rows || col0 < 0 || col0 + pw.n_total > out.cols)
        throw std::invalid_argument("execute_gemm_to_peers: shard columns must lie inside out");
    detail::check_writer_matches<uint8_t>(pipeline);
    std::vector<uint8_t*> shifted;
    for (uint8_t* p : peers) shifted.push_back(p + col0);
    check(q8g_gemm_u8s8_requant_peers(a.data, a.rows, a.cols, a.ld, pw.handle(), pipeline.epilogue(pw),
                                      out.data + col0, shifted.data(), (int)shifted.size(), out.ld, 0, a.rows,
                                      cache ? cache->handle() : nullptr, stream));
}

// ------------------------------------------------------------------ conv / depthwise (new entry points)

// weights [3][3][C][OC] int8 (host) -> packed K = 9C x N = OC, with the
// tensor-core operand image built eagerly: immutable and shareable from here on
inline PackedWeight prepack_conv3x3_weights(const int8_t* w_host, int c, int oc, int device = 0) {
    PackedWeight pw = prepack_weights(MatrixView<const int8_t>{w_host, 9 * c, oc, oc}, BlockingParams::defaults(), device);
    check(q8g_conv3x3_prepare(pw.handle(), c, nullptr));
    return pw;
}

// NHWC device tensors, stride 1, pad 1 with zp_a; images [img_begin, img_end)
inline void execute_conv3x3(const uint8_t* x_dev, int nb, int h, int w, int c, const PackedWeight& pw,
                            const OutputPipeline& pipeline, uint8_t* y_dev, int img_begin, int img_end,
                            void* stream = nullptr) {
    check(q8g_conv3x3_u8s8_nhwc(x_dev, nb, h, w, c, pw.handle(), pipeline.epilogue(pw), y_dev, img_begin, img_end,
                                stream));
}
// host views (the reference calling convention): chunked, copies overlapped, synchronous
inline void execute_conv3x3_host(const uint8_t* x_host, int nb, int h, int w, int c, const PackedWeight& pw,
                                 const OutputPipeline& pipeline, uint8_t* y_host, int img_begin, int img_end,
                                 void* stream = nullptr) {
    check(q8g_conv3x3_u8s8_nhwc_host(x_host, nb, h, w, c, pw.handle(), pipeline.epilogue(pw), y_host, img_begin,
                                     img_end, stream));
}

class DepthwiseFilter {
public:
    DepthwiseFilter(const int8_t* w_host /* [3][3][C] */, int c, const RequantParams& p, bool relu, int device = 0) {
        q8g_requant_params cp{};
        cp.multiplier = p.multiplier;
        cp.zp_a = p.zp_a;
        cp.zp_b = p.zp_b;
        cp.zp_c = p.zp_c;
        cp.k_total = 9;
        cp.bias_host = p.bias.empty() ? nullptr : p.bias.data();
        cp.zp_b_per_channel_host = p.zp_b_per_channel.empty() ? nullptr : p.zp_b_per_channel.data();
        cp.multiplier_f32_per_channel_host =
            p.multiplier_f32_per_channel.empty() ? nullptr : p.multiplier_f32_per_channel.data();
        cp.rounding = static_cast<int>(p.rounding);
        cp.relu = relu ? 1 : 0;
        q8g_dw_filter* f = nullptr;
        check(q8g_dw_filter_create(w_host, c, &cp, device, &f));
        h_.reset(f, &q8g_dw_filter_free);
    }
    const q8g_dw_filter* handle() const { return h_.get(); }

private:
    std::shared_ptr<q8g_dw_filter> h_;
};

inline void execute_dwconv3x3(const uint8_t* x_dev, int nb, int h, int w, int c, const DepthwiseFilter& f,
                              uint8_t* y_dev, int img_begin, int img_end, void* stream = nullptr) {
    check(q8g_dwconv3x3_u8s8_nhwc(x_dev, nb, h, w, c, f.handle(), y_dev, img_begin, img_end, stream));
}
inline void execute_dwconv3x3_host(const uint8_t* x_host, int nb, int h, int w, int c, const DepthwiseFilter& f,
                                   uint8_t* y_host, int img_begin, int img_end, void* stream = nullptr) {
    check(q8g_dwconv3x3_u8s8_nhwc_host(x_host, nb, h, w, c, f.handle(), y_host, img_begin, img_end, stream));
}

}  // namespace q8gemm_b200
