// acceptance_b200.cpp — the reference's acceptance criteria (proj/tests/
// acceptance.cpp) re-run through the C++ drop-in API
// (include/q8gemm_b200/q8gemm.hpp) on the B200 library, checked against the
// oracle restatement (oracle/oracle.c, itself pinned to the reference).
//
//   acceptance_b200 host   host-side logic only (no GPU)
//   acceptance_b200 gpu [CLI]  GPU criteria 1, 2', 3, 5, 6, 7, 8 + C0 REF
//                          parity; with the CLI binary (q8gemm_b200_cli) also
//                          criterion 7's bench leg and criterion 8's CLI runs
//
// Prints one line per criterion like the reference runner; exit 0 iff all pass.
#include <cuda_runtime.h>

#include <sys/wait.h>

#include <chrono>
#include <cstdio>
#include <fstream>
#include <cstring>
#include <array>
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

// ---- criterion 9 (N-sharded multi-GPU): every rank of a
// column split, run on this one GPU with its own output buffer standing in
// for a peer's, writes its shard into all buffers through
// execute_gemm_to_peers; each buffer must equal the unsharded GEMM ----
bool criterion9(std::string& d) {
    Rng rng(9009);
    for (const auto& shape : std::vector<std::array<int, 4>>{{4864, 2048, 256, 2}, {128, 1024, 512, 3}}) {
        const int m = shape[0], n = shape[1], k = shape[2], world = shape[3];
        const auto a = rng.u8(m, k);
        const auto b = rng.i8(k, n);
        RequantParams rp;
        rp.zp_a = 128;
        rp.zp_c = 5;
        rp.k_total = k;
        rp.rounding = Rounding::kF32Rne;
        for (int j = 0; j < n; ++j) {
            rp.bias.push_back(rng.integer(-1000, 1000));
            rp.zp_b_per_channel.push_back(rng.integer(-10, 10));
            rp.multiplier_f32_per_channel.push_back(0.0005f + 0.0015f * (float)rng.integer(0, 1000) / 1000.0f);
        }
        uint8_t* da = nullptr;
        cudaMalloc(&da, (size_t)m * k);
        cudaMemcpy(da, a.data(), (size_t)m * k, cudaMemcpyHostToDevice);
        // unsharded
        const PackedWeight pw = prepack_weights(cview(b), BlockingParams::defaults());
        const OutputPipeline whole({ReluQuantized{}, Requantize{rp, nullptr}});
        uint8_t* dref = nullptr;
        cudaMalloc(&dref, (size_t)m * n);
        execute_gemm(DeviceView<const uint8_t>{da, m, k, k}, pw, DeviceView<uint8_t>{dref, m, n, n}, whole,
                     KernelVariant::kAccI32, 0, 1);
        std::vector<uint8_t> ref((size_t)m * n);
        cudaMemcpy(ref.data(), dref, ref.size(), cudaMemcpyDeviceToHost);
        // sharded: columns [n0, n1) per rank, 16-column blocks (nshard.column_shard)
        std::vector<uint8_t*> bufs(world);
        for (auto& p : bufs) {
            cudaMalloc(&p, (size_t)m * n);
            cudaMemset(p, 0xA5, (size_t)m * n);
        }
        const int blocks = (n + 15) / 16;
        for (int r = 0; r < world; ++r) {
            int b0 = 0, b1 = 0;
            q8g_partition_stripes(blocks, r, world, &b0, &b1);
            const int n0 = std::min(16 * b0, n), n1 = std::min(16 * b1, n);
            if (n1 <= n0) continue;
            Matrix<int8_t> bs(k, n1 - n0);
            for (int kk = 0; kk < k; ++kk)
                for (int j = n0; j < n1; ++j) bs(kk, j - n0) = b(kk, j);
            RequantParams rs = rp;
            rs.bias.assign(rp.bias.begin() + n0, rp.bias.begin() + n1);
            rs.zp_b_per_channel.assign(rp.zp_b_per_channel.begin() + n0, rp.zp_b_per_channel.begin() + n1);
            rs.multiplier_f32_per_channel.assign(rp.multiplier_f32_per_channel.begin() + n0,
                                                 rp.multiplier_f32_per_channel.begin() + n1);
            const PackedWeight pws = prepack_weights(cview(bs), BlockingParams::defaults());
            const OutputPipeline shard({ReluQuantized{}, Requantize{rs, nullptr}});
            std::vector<uint8_t*> peers;
            for (int q = 0; q < world; ++q)
                if (q != r) peers.push_back(bufs[q]);
            execute_gemm_to_peers(DeviceView<const uint8_t>{da, m, k, k}, pws, DeviceView<uint8_t>{bufs[r], m, n, n},
                                  peers, n0, shard);
        }
        cudaDeviceSynchronize();
        bool ok = true;
        for (auto* p : bufs) {
            std::vector<uint8_t> h((size_t)m * n);
            cudaMemcpy(h.data(), p, h.size(), cudaMemcpyDeviceToHost);
            ok = ok && h == ref;
            cudaFree(p);
        }
        cudaFree(da);
        cudaFree(dref);
        if (!ok) return d = "sharded != unsharded at m=" + std::to_string(m), false;
    }
    d = "column shards written to every rank's output equal the unsharded GEMM (2 and 3 ranks)";
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

std::string cli_path;

std::string run_capture(const std::string& cmd, int& rc) {  // stdout + stderr, exit code
    std::string out;
    FILE* p = popen((cmd + " 2>&1").c_str(), "r");
    if (!p) return rc = -1, out;
    char buf[4096];
    size_t got;
    while ((got = fread(buf, 1, sizeof(buf), p)) > 0) out.append(buf, got);
    const int st = pclose(p);
    rc = WIFEXITED(st) ? WEXITSTATUS(st) : -1;
    return out;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- criterion 7 (performance smoke): 512^3 through the host-view API vs the
// single-threaded naive product, and the CLI's default bench list < 60 s ----
bool criterion7(std::string& d) {
    Rng rng(7007);
    const int dim = 512;
    const auto a = rng.u8(dim, dim);
    const auto b = rng.i8(dim, dim);
    auto t0 = std::chrono::steady_clock::now();
    Matrix<int32_t> want(dim, dim, 0);
    orc_naive_gemm_i32(a.data(), dim, dim, dim, b.data(), dim, dim, want.data(), dim, 1);
    const double naive_s = seconds_since(t0);
    const PackedWeight pw = prepack_weights(cview(b), BlockingParams::defaults());
    const OutputPipeline raw({WriteRawI32{}});
    Matrix<int32_t> out(dim, dim, 0);
    execute_gemm(cview(a), pw, view(out), raw, KernelVariant::kAccI32, 0, 1);
    double best = 1e30;
    for (int r = 0; r < 3; ++r) {
        t0 = std::chrono::steady_clock::now();
        execute_gemm(cview(a), pw, view(out), raw, KernelVariant::kAccI32, 0, 1);
        best = std::min(best, seconds_since(t0));
    }
    double bench_s = -1.0;
    bool bench_ok = true;
    if (!cli_path.empty()) {
        int rc = 0;
        t0 = std::chrono::steady_clock::now();
        const std::string csv = run_capture(cli_path + " bench --repeats 5", rc);
        bench_s = seconds_since(t0);
        bench_ok = rc == 0 && bench_s < 60.0 && csv.rfind("M,N,K,variant,threads,ns_median,gops\n", 0) == 0;
    }
    char buf[256];
    std::snprintf(buf, sizeof(buf), "host-view 512^3: %.4fs vs naive %.3fs (%.0fx, want >= 2x); default bench list in %.1fs (want < 60s)",
                  best, naive_s, naive_s / best, bench_s);
    d = buf;
    return out == want && naive_s / best >= 2.0 && bench_ok;
}

// ---- criterion 8, CLI leg: verify / demo byte-identical across reruns, threads=4 ----
bool criterion8_cli(std::string& d) {
    const std::string shapes = "/tmp/q8g_b200_acceptance_shapes.txt";
    {
        std::ofstream f(shapes);
        f << "# acceptance shapes\n1 1 1\n4 5 6\n1 16 16\n16 16 16\n33 7 129\n\n56 32 64\n";
    }
    int rc1 = 0, rc2 = 0;
    const std::string v1 = run_capture(cli_path + " verify --shapes " + shapes + " --seed 99", rc1);
    const std::string v2 = run_capture(cli_path + " verify --shapes " + shapes + " --seed 99", rc2);
    if (rc1 || rc2 || v1 != v2 || v1.find("FAIL") != std::string::npos || v1.find("PASS") == std::string::npos)
        return d = "verify runs differ or failed:\n" + v1, false;
    const std::string demo = cli_path + " demo --m 32 --n 24 --k 48 --density 0.02 --seed 7";
    const std::string d1 = run_capture(demo, rc1), d2 = run_capture(demo, rc2);
    if (rc1 || rc2 || d1 != d2 || d1.find("PASS") == std::string::npos) return d = "demo runs differ or failed:\n" + d1, false;
    const std::string v4 = run_capture(cli_path + " verify --shapes " + shapes + " --seed 99 --threads 4", rc1);
    if (rc1 || v4.find("FAIL") != std::string::npos) return d = "threaded verify failed:\n" + v4, false;
    d = "CLI verify and demo byte-identical across reruns; threads=4 verify passes";
    return true;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "host";
    if (argc > 2) cli_path = argv[2];
    run(0, host_checks);
    if (mode == "gpu") {
        run(1, criterion1);
        run(2, criterion_c0);
        run(3, criterion3);
        run(5, criterion5);
        run(6, criterion6);
        run(7, criterion7);
        run(8, criterion8);
        run(9, criterion9);
        if (!cli_path.empty()) run(8, criterion8_cli);
    }
    if (failures == 0) {
        std::printf("all gating criteria passed\n");
        return 0;
    }
    std::printf("%d gating criteria FAILED\n", failures);
    return 1;
}
