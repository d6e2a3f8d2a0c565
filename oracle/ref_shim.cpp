// ref_shim.cpp — extern "C" veneer over the UNMODIFIED reference q8gemm
// headers (/root/reference/proj/include, compiled in place by oracle/Makefile
// into oracle/_ref/).  TEST INFRASTRUCTURE ONLY: used by tests/ to pin the
// oracle restatement and to generate golden fixtures, and by bench.py's
// cpu_baseline / --impl reference leg as the reference CPU path.
//
// Every entry point calls straight into the reference's public API:
//   select_blocking   dispatch.hpp:17-30
//   prepack_weights   pack.hpp:146-196
//   execute_gemm      engine.hpp:59-169 (caller-owned threads, as in
//                     acceptance.cpp:47-61 / test_engine.cpp:17-25)
//   OutputPipeline    pipeline.hpp:57-128 with Requantize / ReluQuantized /
//                     WriteRawI32 / WriteDequantF32 / BiasAdd / SpMDMAdd
//   split_outliers    sparse.hpp:33-58
//   naive_gemm_i32    oracle.hpp:15-30
//   requantize_scalar quant.hpp:127-133
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "q8gemm/q8gemm.hpp"

using namespace q8gemm;

namespace {
thread_local std::string g_err;

template <typename OutT>
void run_workers(int nt, MatrixView<const uint8_t> a, const PackedWeight& pw, MatrixView<OutT> out,
                 const OutputPipeline& pipeline) {
    if (nt <= 1) {
        execute_gemm(a, pw, out, pipeline, KernelVariant::kAccI32, 0, 1);
        return;
    }
    std::vector<std::thread> workers;
    std::vector<std::exception_ptr> errs(nt);
    for (int t = 0; t < nt; ++t) {
        workers.emplace_back([&, t] {
            try {
                execute_gemm(a, pw, out, pipeline, KernelVariant::kAccI32, t, nt);
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    }
    for (auto& w : workers) w.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

BlockingParams to_bp(const int* bp5) {
    BlockingParams bp;
    bp.mcb = bp5[0];
    bp.ncb = bp5[1];
    bp.kcb = bp5[2];
    bp.mr = bp5[3];
    bp.nr = bp5[4];
    return bp;
}
}  // namespace

extern "C" {

const char* refx_last_error() { return g_err.c_str(); }

int refx_select_blocking(int m, int n, int k, const int* defaults5, int* out5) {
    try {
        const BlockingParams bp = select_blocking(m, n, k, to_bp(defaults5));
        out5[0] = bp.mcb;
        out5[1] = bp.ncb;
        out5[2] = bp.kcb;
        out5[3] = bp.mr;
        out5[4] = bp.nr;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

void* refx_prepack(const int8_t* b, int k, int n, int ldb, const int* bp5) {
    try {
        MatrixView<const int8_t> bv{b, k, n, ldb};
        return new PackedWeight(prepack_weights(bv, to_bp(bp5)));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void refx_free(void* h) { delete static_cast<PackedWeight*>(h); }

long long refx_packed_size(void* h) { return (long long)static_cast<PackedWeight*>(h)->data.size(); }

void refx_packed_data(void* h, int8_t* out) {
    const auto* pw = static_cast<PackedWeight*>(h);
    std::memcpy(out, pw->data.data(), pw->data.size());
}

void refx_col_offsets(void* h, int32_t* out) {
    const auto* pw = static_cast<PackedWeight*>(h);
    std::memcpy(out, pw->col_offsets.values.data(), pw->col_offsets.values.size() * 4);
}

int refx_max_abs(void* h) { return static_cast<PackedWeight*>(h)->max_abs; }

int refx_unpack(void* h, int8_t* out) {
    const Matrix<int8_t> b = unpack_weight(*static_cast<PackedWeight*>(h));
    std::memcpy(out, b.data(), (size_t)b.rows() * b.cols());
    return 0;
}

int refx_gemm_raw(const uint8_t* a, int m, int k, int lda, void* h, int32_t* out, int ldo,
                  int threads) {
    try {
        MatrixView<const uint8_t> av{a, m, k, lda};
        const auto& pw = *static_cast<PackedWeight*>(h);
        MatrixView<int32_t> ov{out, m, pw.n_total, ldo};
        run_workers(threads, av, pw, ov, OutputPipeline({WriteRawI32{}}));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

int refx_gemm_requant(const uint8_t* a, int m, int k, int lda, void* h, double multiplier,
                      int zp_a, int zp_b, int zp_c, const int32_t* bias, int relu, uint8_t* out,
                      int ldo, int threads) {
    try {
        MatrixView<const uint8_t> av{a, m, k, lda};
        const auto& pw = *static_cast<PackedWeight*>(h);
        MatrixView<uint8_t> ov{out, m, pw.n_total, ldo};
        RequantParams rp;
        rp.multiplier = multiplier;
        rp.zp_a = zp_a;
        rp.zp_b = zp_b;
        rp.zp_c = zp_c;
        rp.k_total = k;
        if (bias) rp.bias.assign(bias, bias + pw.n_total);
        std::vector<OutputStage> stages;
        if (relu) stages.push_back(ReluQuantized{});
        stages.push_back(Requantize{rp, &pw.col_offsets});
        run_workers(threads, av, pw, ov, OutputPipeline(std::move(stages)));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

int refx_naive_gemm(const uint8_t* a, int m, int k, int lda, const int8_t* b, int n, int ldb,
                    int32_t* out) {
    try {
        const Matrix<int32_t> c =
            oracle::naive_gemm_i32(MatrixView<const uint8_t>{a, m, k, lda},
                                   MatrixView<const int8_t>{b, k, n, ldb});
        std::memcpy(out, c.data(), (size_t)m * n * 4);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

int refx_requantize_scalar(int32_t acc, int32_t ro, int32_t co, double multiplier, int zp_a,
                           int zp_b, int zp_c, int k_total, const int32_t* bias, int nbias,
                           int col) {
    RequantParams rp;
    rp.multiplier = multiplier;
    rp.zp_a = zp_a;
    rp.zp_b = zp_b;
    rp.zp_c = zp_c;
    rp.k_total = k_total;
    if (bias) rp.bias.assign(bias, bias + nbias);
    return requantize_scalar(acc, ro, co, rp, col);
}

long long refx_requantize_adjust(int32_t acc, int32_t ro, int32_t co, int zp_a, int zp_b,
                                 int k_total, int32_t bias) {
    RequantParams rp;
    rp.zp_a = zp_a;
    rp.zp_b = zp_b;
    rp.k_total = k_total;
    rp.bias.assign(1, bias);
    return requantize_adjust(acc, ro, co, rp, 0);
}

int refx_pipeline_validate(const int* kinds, int n, char* msg, int msg_len) {
    // kinds: 0 BiasAdd, 1 ReluQuantized, 2 Requantize, 3 WriteRawI32, 4 WriteDequantF32
    static const ColOffsets co;
    std::vector<OutputStage> st;
    for (int i = 0; i < n; ++i) {
        switch (kinds[i]) {
            case 0: st.push_back(BiasAdd{}); break;
            case 1: st.push_back(ReluQuantized{}); break;
            case 2: {
                Requantize r{RequantParams{}, &co};
                st.push_back(r);
                break;
            }
            case 3: st.push_back(WriteRawI32{}); break;
            default: st.push_back(WriteDequantF32{}); break;
        }
    }
    auto err = OutputPipeline::validate(st);
    if (!err) return 0;
    std::snprintf(msg, msg_len, "%s", err->c_str());
    return 22;
}

// sparse.hpp:33-58 split_outliers; CSC arrays written to caller buffers of
// capacity cap.  Returns nnz, -1 if it exceeds cap, or 22 on an exception.
int refx_split_outliers(const int8_t* b, int k, int n, int ldb, int threshold, int8_t* dense, int32_t* col_ptr,
                        int32_t* row_idx, int8_t* values, int cap, int* nnz_out) {
    try {
        const SplitWeight sw = split_outliers(MatrixView<const int8_t>{b, k, n, ldb}, threshold);
        std::memcpy(dense, sw.dense_small.data(), (size_t)k * n);
        std::memcpy(col_ptr, sw.sparse.col_ptr.data(), sizeof(int32_t) * (n + 1));
        *nnz_out = sw.sparse.nnz();
        if (sw.sparse.nnz() > cap) return -1;
        std::memcpy(row_idx, sw.sparse.row_idx.data(), sizeof(int32_t) * sw.sparse.nnz());
        std::memcpy(values, sw.sparse.values.data(), (size_t)sw.sparse.nnz());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

// execute_gemm (engine.hpp:59-169) with [SpMDMAdd] [BiasAdd] then a writer:
// writer 0 WriteRawI32 (int32 out), 1 [ReluQuantized] Requantize (u8 out,
// col_offsets = the given full-K vector), 2 WriteDequantF32 (float out).
int refx_gemm_pipeline(const uint8_t* a, int m, int k, int lda, void* h, const int32_t* col_ptr,
                       const int32_t* row_idx, const int8_t* values, int nnz, const int32_t* bias_add, int writer,
                       double multiplier, int zp_a, int zp_b, int zp_c, const int32_t* rq_bias, int relu,
                       const int32_t* col_offsets, double dq_scale, int dq_zero_point, void* out, int ldo,
                       int threads) {
    try {
        MatrixView<const uint8_t> av{a, m, k, lda};
        const auto& pw = *static_cast<PackedWeight*>(h);
        const int n = pw.n_total;
        SparseWeightCSC sp;
        ColOffsets co;
        std::vector<OutputStage> stages;
        if (col_ptr) {
            sp.k_total = k;
            sp.n_total = n;
            sp.col_ptr.assign(col_ptr, col_ptr + n + 1);
            sp.row_idx.assign(row_idx, row_idx + nnz);
            sp.values.assign(values, values + nnz);
            stages.push_back(SpMDMAdd{&sp});
        }
        if (bias_add) stages.push_back(BiasAdd{std::span<const int32_t>(bias_add, (size_t)n)});
        if (writer == 0) {
            stages.push_back(WriteRawI32{});
            run_workers(threads, av, pw, MatrixView<int32_t>{static_cast<int32_t*>(out), m, n, ldo},
                        OutputPipeline(std::move(stages)));
        } else if (writer == 1) {
            RequantParams rp;
            rp.multiplier = multiplier;
            rp.zp_a = zp_a;
            rp.zp_b = zp_b;
            rp.zp_c = zp_c;
            rp.k_total = k;
            if (rq_bias) rp.bias.assign(rq_bias, rq_bias + n);
            co.values.assign(col_offsets, col_offsets + n);
            if (relu) stages.push_back(ReluQuantized{});
            stages.push_back(Requantize{rp, &co});
            run_workers(threads, av, pw, MatrixView<uint8_t>{static_cast<uint8_t*>(out), m, n, ldo},
                        OutputPipeline(std::move(stages)));
        } else {
            QuantParams qp;
            qp.scale = dq_scale;
            qp.zero_point = dq_zero_point;
            stages.push_back(WriteDequantF32{qp});
            run_workers(threads, av, pw, MatrixView<float>{static_cast<float*>(out), m, n, ldo},
                        OutputPipeline(std::move(stages)));
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 22;
    }
}

}  // extern "C"
