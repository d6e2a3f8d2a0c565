// acceptance_b200.cpp — the reference's acceptance criteria (proj/tests/
// acceptance.cpp) re-run through the C++ drop-in API
// (include/q8gemm_b200/q8gemm.hpp) on the B200 library, checked against the
// oracle restatement (oracle/oracle.c, itself pinned to the reference).
//
//   acceptance_b200 host   host-side logic only (no GPU)
//   acceptance_b200 gpu    GPU criteria 1, 2', 5, 6, 8 + C0 REF parity
//
// Prints one line per criterion like the reference runner; exit 0 iff all pass.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "../../oracle/oracle.h"
#include "q8gemm_b200/q8gemm.hpp"

using namespace q8gemm_b200;

namespace {

struct Rng {
    orc_rng* r;
    explicit Rng(uint64_t seed) : r(orc_rng_new(seed)) {}
    ~Rng() { orc_rng_free(r); }
    int integer(int lo, int hi) { return orc_rng_int(r, lo, hi); }
    Matrix<uint8_t> u8(int rows, int cols) {
        Matrix<uint8_t> m(rows, cols);
        orc_rng_u8(r, m.data(), (int64_t)rows * cols);
        return m;
    }
    Matrix<int8_t> i8(int rows, int cols) {
        Matrix<int8_t> m(rows, cols);
        orc_rng_i8(r, m.data(), (int64_t)rows * cols);
        return m;
    }
};

Matrix<int32_t> oracle_gemm(const Matrix<uint8_t>& a, const Matrix<int8_t>& b) {
    Matrix<int32_t> c(a.rows(), b.cols(), 0);
    orc_naive_gemm_i32(a.data(), a.rows(), a.cols(), a.cols(), b.data(), b.cols(), b.cols(), c.data(), b.cols(), 4);
    return c;
}

template <typename OutT>
void run_workers(int nt, MatrixView<const uint8_t> a, const PackedWeight& pw, MatrixView<OutT> out,
                 const OutputPipeline& p) {
    // acceptance.cpp:47-61: caller-owned threads, one execute_gemm per worker
    if (nt == 1) {
        execute_gemm(a, pw, out, p, KernelVariant::kAccI32, 0, 1);
        return;
    }
    std::vector<std::thread> ws;
    for (int t = 0; t < nt; ++t) ws.emplace_back([&, t] { execute_gemm(a, pw, out, p, KernelVariant::kAccI32, t, nt); });
    for (auto& w : ws) w.join();
}

int failures = 0;
void report(int id, bool pass, const std::string& detail, double s) {
    std::printf("[%s] criterion %d: %s (%.1fs)\n", pass ? "PASS" : "FAIL", id, detail.c_str(), s);
    std::fflush(stdout);
    if (!pass) ++failures;
}

template <typename F>
void run(int id, F f) {
    const auto t0 = std::chrono::steady_clock::now();
    std::string detail;
    bool pass = false;
    try {
        pass = f(detail);
    } catch (const std::exception& e) {
        detail = std::string("exception: ") + e.what();
    }
    report(id, pass, detail, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
}

template <typename Fn>
bool throws_invalid(Fn fn, const char* needle) {
    try {
        fn();
    } catch (const std::invalid_argument& e) {
        return std::strstr(e.what(), needle) != nullptr;
    }
    return false;
}

// ---- host-only criteria (no GPU) ----
bool host_checks(std::string& d) {
    BlockingParams bad;
    bad.mcb = 15;
    if (!throws_invalid([&] { bad.validate(); }, "mcb must be a multiple of mr")) return d = "mcb rule", false;
    BlockingParams k7;
    k7.kcb = 7;
    if (!throws_invalid([&] { k7.validate(); }, "kcb must be even")) return d = "kcb rule", false;
    const BlockingParams s = select_blocking(1, 5, 3, BlockingParams::defaults());
    if (s.mr != 1 || s.nr != 5 || s.kcb != 4 || s.mcb != 1 || s.ncb != 5) return d = "select_blocking", false;
    if (!throws_invalid([] { OutputPipeline p({}); }, "pipeline is empty")) return d = "empty pipeline", false;
    if (!throws_invalid([] { OutputPipeline p({ReluQuantized{}, WriteRawI32{}}); },
                        "ReluQuantized must immediately precede a Requantize writer"))
        return d = "relu rule", false;
    if (!throws_invalid([] { OutputPipeline p({WriteRawI32{}, BiasAdd{}}); }, "follows a writer"))
        return d = "writer order", false;
    RequantParams zero;
    zero.multiplier = 0;
    if (!throws_invalid([&] { OutputPipeline p({Requantize{zero, nullptr}}); }, "multiplier must be positive"))
        return d = "multiplier rule", false;
    OutputPipeline ok({BiasAdd{}, ReluQuantized{}, Requantize{RequantParams{}, nullptr}});
    if (!ok.has_relu() || ok.writer() != WriterKind::kRequantizeU8) return d = "pipeline queries", false;
    int b = 0, e = 0;
    q8g_partition_stripes(10, 3, 4, &b, &e);
    if (b != 8 || e != 10) return d = "partition_stripes", false;
    if (!throws_invalid([] { OutputPipeline p({SpMDMAdd{nullptr}, WriteRawI32{}}); }, "SpMDMAdd requires a sparse matrix"))
        return d = "SpMDMAdd rule", false;
    if (OutputPipeline({WriteDequantF32{}}).writer() != WriterKind::kDequantF32) return d = "dequant writer", false;
    // split_outliers (sparse.hpp:33-58): dense_small + CSC rebuilds B, outliers at full value
    Rng rng(303);
    const auto bm = rng.i8(37, 29);
    const SplitWeight sw = split_outliers(cview(bm), 90);
    Matrix<int32_t> re(37, 29, 0);
    for (int kk = 0; kk < 37; ++kk)
        for (int j = 0; j < 29; ++j) {
            const int v = sw.dense_small(kk, j);
            if (std::abs(v) >= 90) return d = "dense part holds an outlier", false;
            re(kk, j) = v;
        }
    for (int j = 0; j < 29; ++j)
        for (int32_t i = sw.sparse.col_ptr[j]; i < sw.sparse.col_ptr[j + 1]; ++i) {
            if (std::abs((int)sw.sparse.values[i]) < 90) return d = "CSC holds a small value", false;
            re(sw.sparse.row_idx[i], j) += sw.sparse.values[i];
        }
    for (int kk = 0; kk < 37; ++kk)
        for (int j = 0; j < 29; ++j)
            if (re(kk, j) != bm(kk, j)) return d = "split_outliers does not rebuild B", false;
    if (!throws_invalid([&] { split_outliers(cview(bm), 0); }, "threshold must be >= 1")) return d = "threshold rule", false;
    d = "blocking / pipeline validation / stripes / split_outliers match the reference rules";
    return true;
}

// ---- criterion 1: raw int32 bit-identical to the oracle ----
bool criterion1(std::string& d) {
    Rng rng(1001);
    const OutputPipeline raw({WriteRawI32{}});
    long checked = 0;
    auto check_shape = [&](int m, int n, int k) {
        const auto a = rng.u8(m, k);
        const auto b = rng.i8(k, n);
        const auto exp = oracle_gemm(a, b);
        const PackedWeight pw = prepack_weights(cview(b), select_blocking(m, n, k, BlockingParams::defaults()));
        for (int threads : {1, 4}) {
            Matrix<int32_t> out(m, n, -1);
            run_workers(threads, cview(a), pw, view(out), raw);
            if (!(out == exp)) return false;
            ++checked;
        }
        return true;
    };
    for (int m : {1, 2, 5, 8, 13, 16})
        for (int n : {1, 3, 8, 16})
            for (int k : {1, 4, 7, 16})
                if (!check_shape(m, n, k)) return d = "grid mismatch m=" + std::to_string(m), false;
    for (int t = 0; t < 60; ++t) {
        const int m = rng.integer(1, 256), n = rng.integer(1, 256);
        const int k = t % 2 ? 16 * rng.integer(1, 16) : rng.integer(1, 256);
        if (!check_shape(m, n, k)) return d = "random mismatch", false;
    }
    d = "raw int32 bit-identical to the oracle on " + std::to_string(checked) + " runs (threads {1,4})";
    return true;
}

// ---- C0 in the reference's own rounding (REF): u8 bit-identical ----
bool criterion_c0(std::string& d) {
    Rng rng(42);
    const auto a = rng.u8(64, 320);
    const auto b = rng.i8(320, 800);
    std::vector<int32_t> bias(800);
    orc_rng_int_fill(rng.r, -1000, 1000, bias.data(), 800);
    RequantParams rp;
    rp.multiplier = 0.02 * 0.01 / 0.5;
    rp.zp_a = 128;
    rp.zp_b = 3;
    rp.zp_c = 5;
    rp.k_total = 320;
    rp.bias = bias;
    const PackedWeight pw = prepack_weights(cview(b), select_blocking(64, 800, 320, BlockingParams::defaults()));
    Matrix<uint8_t> out(64, 800, 0);
    execute_gemm(cview(a), pw, view(out), OutputPipeline({Requantize{rp, nullptr}}), KernelVariant::kAccI32, 0, 1);
    const auto acc = oracle_gemm(a, b);
    std::vector<int32_t> rs(64), cs(800);
    orc_row_offsets(a.data(), 64, 320, 320, rs.data());
    orc_col_offsets(b.data(), 320, 800, 800, cs.data());
    Matrix<uint8_t> exp(64, 800, 0);
    const double md = rp.multiplier;
    const int32_t zpb = 3;
    orc_requant_matrix(acc.data(), 64, 800, 800, rs.data(), cs.data(), 128, &zpb, 0, 320, bias.data(), 0, &md,
                       nullptr, 5, 0, exp.data(), 800);
    if (!(out == exp)) return d = "C0 REF-mode output differs", false;
    d = "C0 (64x800x320, REF rounding) u8 bit-identical through the C++ drop-in API";
    return true;
}

// ---- criterion 5: packing invariants ----
bool criterion5(std::string& d) {
    Rng rng(5005);
    for (int t = 0; t < 60; ++t) {
        const int k = rng.integer(1, 300), n = rng.integer(1, 300);
        const auto b = rng.i8(k, n);
        const PackedWeight pw = prepack_weights(cview(b), BlockingParams::defaults());
        if (!(pw.unpack() == b)) return d = "B roundtrip mismatch", false;
        std::vector<int32_t> cs(n);
        orc_col_offsets(b.data(), k, n, n, cs.data());
        if (cs != pw.col_offsets) return d = "column sums mismatch", false;
    }
    d = "pack/unpack roundtrip and column sums exact on 60 random shapes";
    return true;
}

// ---- criterion 6: specialised tiles == generic tile (device views) ----
bool criterion6(std::string& d) {
    Rng rng(6006);
    KernelCache spec(false), gen(true);
    const OutputPipeline raw({WriteRawI32{}});
    for (int m : {1, 5, 64, 128, 129, 300}) {
        for (int n : {5, 64, 300}) {
            const int k = 16 * rng.integer(1, 20);
            const auto a = rng.u8(m, k);
            const auto b = rng.i8(k, n);
            const PackedWeight pw = prepack_weights(cview(b), BlockingParams::defaults());
            uint8_t* da = nullptr;
            int32_t *c1 = nullptr, *c2 = nullptr;
            cudaMalloc(&da, (size_t)m * k);
            cudaMalloc(&c1, (size_t)m * n * 4);
            cudaMalloc(&c2, (size_t)m * n * 4);
            cudaMemcpy(da, a.data(), (size_t)m * k, cudaMemcpyHostToDevice);
            execute_gemm(DeviceView<const uint8_t>{da, m, k, k}, pw, DeviceView<int32_t>{c1, m, n, n}, raw,
                         KernelVariant::kAccI32, 0, 1, &spec);
            execute_gemm(DeviceView<const uint8_t>{da, m, k, k}, pw, DeviceView<int32_t>{c2, m, n, n}, raw,
                         KernelVariant::kAccI32, 0, 1, &gen);
            std::vector<int32_t> h1((size_t)m * n), h2((size_t)m * n);
            cudaMemcpy(h1.data(), c1, h1.size() * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(h2.data(), c2, h2.size() * 4, cudaMemcpyDeviceToHost);
            cudaFree(da);
            cudaFree(c1);
            cudaFree(c2);
            if (h1 != h2) return d = "specialised != generic at m=" + std::to_string(m), false;
        }
    }
    d = "tensor-core tiles bit-equal to the generic CUDA-core tile on 18 shapes";
    return true;
}

// ---- criterion 3: outlier split + SpMDMAdd reproduce the unsplit GEMM; WriteDequantF32 ----
bool criterion3(std::string& d) {
    Rng rng(3003);
    for (int t = 0; t < 8; ++t) {
        const int m = rng.integer(1, 300), n = rng.integer(1, 200), k = rng.integer(1, 400);
        const auto a = rng.u8(m, k);
        const auto b = rng.i8(k, n);
        const SplitWeight sw = split_outliers(cview(b), 40 + 11 * t);
        const PackedWeight pw = prepack_weights(cview(sw.dense_small), BlockingParams::defaults());
        const auto exp = oracle_gemm(a, b);
        Matrix<int32_t> out(m, n, -1);
        run_workers(1 + t % 3, cview(a), pw, view(out), OutputPipeline({SpMDMAdd{&sw.sparse}, WriteRawI32{}}));
        if (!(out == exp)) return d = "SpMDMAdd raw != A x B at t=" + std::to_string(t), false;
        std::vector<int32_t> bias(n);
        for (int j = 0; j < n; ++j) bias[j] = 7 * j - 300;
        const QuantParams qp{0.00321, -17};
        Matrix<float> f(m, n, 0.f);
        run_workers(2, cview(a), pw, view(f), OutputPipeline({SpMDMAdd{&sw.sparse}, BiasAdd{bias}, WriteDequantF32{qp}}));
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < n; ++j) {
                const int32_t acc = (int32_t)((uint32_t)exp(i, j) + (uint32_t)bias[j]);
                const float want = (float)(qp.scale * (double)(int32_t)((uint32_t)acc - (uint32_t)qp.zero_point));
                if (f(i, j) != want) return d = "WriteDequantF32 mismatch at t=" + std::to_string(t), false;
            }
        // requantize with the original B's column offsets (Requantize::col_offsets)
        RequantParams rp;
        rp.multiplier = 0.0009;
        rp.zp_a = 5;
        rp.zp_b = 2;
        rp.zp_c = 90;
        rp.k_total = k;
        std::vector<int32_t> co(n, 0);
        for (int kk = 0; kk < k; ++kk)
            for (int j = 0; j < n; ++j) co[j] += b(kk, j);
        Matrix<uint8_t> q1(m, n, 0), q2(m, n, 1);
        run_workers(1, cview(a), pw, view(q1), OutputPipeline({SpMDMAdd{&sw.sparse}, Requantize{rp, &co}}));
        const PackedWeight full = prepack_weights(cview(b), BlockingParams::defaults());
        run_workers(1, cview(a), full, view(q2), OutputPipeline({Requantize{rp, nullptr}}));
        if (!(q1 == q2)) return d = "split + SpMDMAdd requant != unsplit requant", false;
    }
    d = "split + SpMDMAdd == unsplit GEMM (raw, requant); WriteDequantF32 exact, 8 shapes";
    return true;
}

// ---- criterion 8: determinism across workers ----
bool criterion8(std::string& d) {
    Rng rng(8008);
    for (int t = 0; t < 10; ++t) {
        const int m = rng.integer(1, 600), n = rng.integer(1, 150), k = 16 * rng.integer(1, 10);
        const auto a = rng.u8(m, k);
        const auto b = rng.i8(k, n);
        const PackedWeight pw = prepack_weights(cview(b), BlockingParams::defaults());
        Matrix<int32_t> s(m, n, 0), p(m, n, -1);
        const OutputPipeline raw({WriteRawI32{}});
        run_workers(1, cview(a), pw, view(s), raw);
        run_workers(4, cview(a), pw, view(p), raw);
        if (!(s == p)) return d = "threads=4 raw output differs", false;
        RequantParams rp;
        rp.multiplier = 0.0004;
        rp.zp_a = 9;
        rp.zp_b = -3;
        rp.zp_c = 70;
        rp.k_total = k;
        const OutputPipeline rq({Requantize{rp, nullptr}});
        Matrix<uint8_t> sq(m, n, 0), pq(m, n, 1);
        run_workers(1, cview(a), pw, view(sq), rq);
        run_workers(4, cview(a), pw, view(pq), rq);
        if (!(sq == pq)) return d = "threads=4 requantized output differs", false;
    }
    d = "parallel output bit-identical to serial (raw and requantized)";
    return true;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "host";
    run(0, host_checks);
    if (mode == "gpu") {
        run(1, criterion1);
        run(2, criterion_c0);
        run(3, criterion3);
        run(5, criterion5);
        run(6, criterion6);
        run(8, criterion8);
    }
    if (failures == 0) {
        std::printf("all gating criteria passed\n");
        return 0;
    }
    std::printf("%d gating criteria FAILED\n", failures);
    return 1;
}
