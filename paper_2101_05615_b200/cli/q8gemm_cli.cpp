// q8gemm_cli.cpp — the reference command-line harness (proj/tools/q8gemm_cli.cpp,
// SPEC.md "[MODULE] cli") on the B200 engine, through the C++ drop-in API
// (include/q8gemm_b200/q8gemm.hpp).  Same subcommands, flags, defaults, output
// lines, CSV header and exit codes:
//
//   verify  engine vs a naive i-j-k GEMM per shape, "M=.. N=.. K=.. variant=..
//           threads=.. : PASS|FAIL max_dev=.."; exit 0 iff every shape passes
//   bench   "M,N,K,variant,threads,ns_median,gops", median of --repeats after
//           2 warm-ups, monotonic wall clock around the host-view call (H2D of
//           A, the GPU GEMM, D2H of C), --compare-naive adds a "naive" row
//   demo    the INT16 + outlier-split sample pipeline: SpMDMAdd + Requantize on
//           the split weights vs the integer and real-domain references
//
// Exit codes: 0 success, 1 verification failure, 2 invalid input / config
// (including the engine's std::invalid_argument refusals), 3 runtime (CUDA)
// failure.  --threads N spawns exactly N host workers, each calling
// execute_gemm(thread_id, N) on its row stripe (the library creates none).
// The i16 variant runs the exact int32 path whenever the reference would
// accept it (bit-identical).
//
// Random data follow the reference harness: one std::mt19937_64(seed) draws
// A then B per shape, row-major, low byte of each 64-bit draw.  The naive
// checks below are this tool's own self-certification, written
// from oracle.hpp:15-54 and quant.hpp:115-133; they are not the test oracle.
#include <algorithm>
#include <chrono>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <map>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "q8gemm_b200/q8gemm.hpp"

namespace {

using namespace q8gemm_b200;

// ------------------------------------------------------------------ arguments

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Shape {
    int m, n, k;
};

struct Options {
    std::string cmd;
    std::string shapes_path;
    uint64_t seed = 42;
    std::string variant = "i32";
    int threads = 1;
    int repeats = 11;
    bool compare_naive = false;
    bool no_split = false;
    std::optional<int> mcb, ncb, kcb, mr, nr;
    int dm = 64, dn = 64, dk = 64;  // demo
    double density = 0.01;
};

const char* kUsage =
    "usage: q8gemm_b200_cli {verify|bench|demo} [options]\n"
    "  verify  Check the engine against the naive oracle\n"
    "          --shapes PATH --seed U64 --variant {i32,i16} --threads N --no-split\n"
    "  bench   Timing sweep, CSV on stdout\n"
    "          --shapes PATH --seed U64 --variant {i32,i16} --threads N --repeats N --compare-naive\n"
    "  demo    End-to-end INT16 + outlier-split pipeline\n"
    "          --m N --n N --k N --density X --seed U64 --threads N\n"
    "  all:    --mcb --ncb --kcb --mr --nr blocking overrides, -h/--help\n";

long long parse_int(const std::string& flag, const std::string& v) {
    char* end = nullptr;
    errno = 0;
    const long long x = std::strtoll(v.c_str(), &end, 10);
    if (v.empty() || *end != '\0' || errno != 0) throw UsageError(flag + ": value " + v + " is not an integer");
    return x;
}

int parse_positive(const std::string& flag, const std::string& v) {
    const long long x = parse_int(flag, v);
    if (x < 1 || x > 1000000000LL) throw UsageError(flag + ": value " + v + " is not a positive number");
    return static_cast<int>(x);
}

// returns nullopt for --help
std::optional<Options> parse_args(int argc, char** argv) {
    Options o;
    if (argc < 2) throw UsageError("a subcommand is required (verify, bench or demo)");
    o.cmd = argv[1];
    if (o.cmd == "-h" || o.cmd == "--help") return std::nullopt;
    if (o.cmd != "verify" && o.cmd != "bench" && o.cmd != "demo")
        throw UsageError("unknown subcommand: " + o.cmd);
    const bool v = o.cmd == "verify", b = o.cmd == "bench", d = o.cmd == "demo";
    for (int i = 2; i < argc; ++i) {
        std::string flag = argv[i], val;
        bool has_inline = false;
        if (const auto eq = flag.find('='); flag.rfind("--", 0) == 0 && eq != std::string::npos) {
            val = flag.substr(eq + 1);
            flag = flag.substr(0, eq);
            has_inline = true;
        }
        if (flag == "-h" || flag == "--help") return std::nullopt;
        auto value = [&]() -> std::string {
            if (has_inline) return val;
            if (i + 1 >= argc) throw UsageError(flag + " requires an argument");
            return argv[++i];
        };
        auto flag_only = [&] {
            if (has_inline) throw UsageError(flag + " takes no value");
        };
        if ((v || b) && flag == "--shapes") {
            o.shapes_path = value();
        } else if (flag == "--seed") {
            const std::string s = value();
            char* end = nullptr;
            errno = 0;
            const unsigned long long x = std::strtoull(s.c_str(), &end, 10);
            if (s.empty() || s[0] == '-' || *end != '\0' || errno != 0)
                throw UsageError("--seed: value " + s + " is not an unsigned integer");
            o.seed = x;
        } else if ((v || b) && flag == "--variant") {
            o.variant = value();
            if (o.variant != "i32" && o.variant != "i16")
                throw UsageError("--variant: " + o.variant + " not in {i32,i16}");
        } else if (flag == "--threads") {
            o.threads = parse_positive(flag, value());
        } else if (b && flag == "--repeats") {
            o.repeats = parse_positive(flag, value());
        } else if (b && flag == "--compare-naive") {
            flag_only();
            o.compare_naive = true;
        } else if (v && flag == "--no-split") {
            flag_only();
            o.no_split = true;
        } else if (d && flag == "--m") {
            o.dm = parse_positive(flag, value());
        } else if (d && flag == "--n") {
            o.dn = parse_positive(flag, value());
        } else if (d && flag == "--k") {
            o.dk = parse_positive(flag, value());
        } else if (d && flag == "--density") {
            const std::string s = value();
            char* end = nullptr;
            const double x = std::strtod(s.c_str(), &end);
            if (s.empty() || *end != '\0' || !(x >= 0.0 && x <= 1.0))
                throw UsageError("--density: value " + s + " not in range [0 - 1]");
            o.density = x;
        } else if (flag == "--mcb" || flag == "--ncb" || flag == "--kcb" || flag == "--mr" || flag == "--nr") {
            const int x = static_cast<int>(parse_int(flag, value()));
            (flag == "--mcb" ? o.mcb : flag == "--ncb" ? o.ncb : flag == "--kcb" ? o.kcb : flag == "--mr" ? o.mr : o.nr) = x;
        } else {
            throw UsageError("the following argument was not expected: " + std::string(argv[i]));
        }
    }
    return o;
}

BlockingParams base_blocking(const Options& o) {
    BlockingParams bp = BlockingParams::defaults();
    if (o.mcb) bp.mcb = *o.mcb;
    if (o.ncb) bp.ncb = *o.ncb;
    if (o.kcb) bp.kcb = *o.kcb;
    if (o.mr) bp.mr = *o.mr;
    if (o.nr) bp.nr = *o.nr;
    bp.validate();  // std::invalid_argument -> exit 2
    return bp;
}

// text file, one "M N K" per line, '#' comments, blank lines ignored
std::vector<Shape> load_shapes(const std::string& path) {
    if (path.empty())
        return {{1, 1, 1}, {1, 64, 64}, {3, 5, 7}, {14, 32, 256}, {56, 64, 512},
                {64, 64, 64}, {100, 37, 61}, {128, 128, 128}, {256, 256, 256}};
    std::ifstream in(path);
    if (!in) throw std::invalid_argument("cannot open shapes file: " + path);
    std::vector<Shape> out;
    std::string line;
    for (int lineno = 1; std::getline(in, line); ++lineno) {
        line = line.substr(0, line.find('#'));
        std::istringstream ss(line);
        long long m = 0, n = 0, k = 0;
        if (!(ss >> m)) continue;
        std::string extra;
        const bool ok = (ss >> n >> k) && !(ss >> extra) && m >= 1 && n >= 1 && k >= 1 && m <= INT32_MAX &&
                        n <= INT32_MAX && k <= INT32_MAX;
        if (!ok)
            throw std::invalid_argument(path + ":" + std::to_string(lineno) +
                                        ": expected \"M N K\" with positive integers");
        out.push_back({static_cast<int>(m), static_cast<int>(n), static_cast<int>(k)});
    }
    if (out.empty()) throw std::invalid_argument(path + ": no shapes found");
    return out;
}

// ------------------------------------------------------------------ data + self-checks

Matrix<uint8_t> draw_u8(std::mt19937_64& g, int rows, int cols) {
    Matrix<uint8_t> x(rows, cols);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) x(i, j) = static_cast<uint8_t>(g() & 0xFF);
    return x;
}

Matrix<int8_t> draw_i8(std::mt19937_64& g, int rows, int cols) {
    Matrix<int8_t> x(rows, cols);
    for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) x(i, j) = static_cast<int8_t>(g() & 0xFF);
    return x;
}

// the straight i-j-k product in 32-bit (oracle.hpp:15-30)
Matrix<int32_t> naive_i32(const Matrix<uint8_t>& a, const Matrix<int8_t>& b) {
    const int m = a.rows(), k = a.cols(), n = b.cols();
    Matrix<int32_t> c(m, n, 0);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
            int32_t s = 0;
            for (int p = 0; p < k; ++p) s += static_cast<int32_t>(a(i, p)) * b(p, j);
            c(i, j) = s;
        }
    return c;
}

// scalar per-tensor requantization in the reference's REF mode
// (quant.hpp:115-133: 64-bit adjust, fp64 scale, ties away, clamp)
int requant_ref(int32_t acc, int32_t rowsum, int32_t colsum, const RequantParams& rp) {
    const int64_t adj = static_cast<int64_t>(acc) - static_cast<int64_t>(rp.zp_b) * rowsum -
                        static_cast<int64_t>(rp.zp_a) * colsum +
                        static_cast<int64_t>(rp.k_total) * rp.zp_a * rp.zp_b;
    const long long q = round_half_away_from_zero(rp.multiplier * static_cast<double>(adj)) + rp.zp_c;
    return static_cast<int>(std::clamp<long long>(q, 0, 255));
}

template <typename OutT>
void run_workers(int nt, const Matrix<uint8_t>& a, const PackedWeight& pw, Matrix<OutT>& out,
                 const OutputPipeline& pipe, KernelVariant var) {
    if (nt == 1) {
        execute_gemm(cview(a), pw, view(out), pipe, var, 0, 1);
        return;
    }
    std::vector<std::thread> ws;
    std::vector<std::exception_ptr> errs(nt);
    for (int t = 0; t < nt; ++t)
        ws.emplace_back([&, t] {
            try {
                execute_gemm(cview(a), pw, view(out), pipe, var, t, nt);
            } catch (...) {
                errs[t] = std::current_exception();
            }
        });
    for (auto& w : ws) w.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

KernelVariant variant_of(const Options& o) { return o.variant == "i16" ? KernelVariant::kAccI16 : KernelVariant::kAccI32; }

// the weights a variant runs on: i32 -> B; i16 -> outlier split at the
// largest exact threshold (unless --no-split), sparse part added in the
// epilogue (SpMDMAdd)
struct Prepared {
    PackedWeight pw;
    SplitWeight sw;
    bool split = false;
    OutputPipeline raw_pipeline() const {
        return split ? OutputPipeline({SpMDMAdd{&sw.sparse}, WriteRawI32{}}) : OutputPipeline({WriteRawI32{}});
    }
};

void prepare(Prepared& p, const Options& o, const Matrix<int8_t>& b, const BlockingParams& bp) {
    if (variant_of(o) == KernelVariant::kAccI16 && !o.no_split) {
        p.sw = split_outliers(cview(b), max_i16_split_threshold(bp.kcb));
        p.pw = prepack_weights(cview(p.sw.dense_small), bp);
        p.split = true;
    } else {
        p.pw = prepack_weights(cview(b), bp);
    }
}

// ------------------------------------------------------------------ subcommands

int cmd_verify(const Options& o) {
    const BlockingParams base = base_blocking(o);
    const std::vector<Shape> shapes = load_shapes(o.shapes_path);
    std::mt19937_64 g(o.seed);
    bool all = true;
    for (const Shape& s : shapes) {
        const Matrix<uint8_t> a = draw_u8(g, s.m, s.k);
        const Matrix<int8_t> b = draw_i8(g, s.k, s.n);
        const BlockingParams bp = select_blocking(s.m, s.n, s.k, base);
        const Matrix<int32_t> want = naive_i32(a, b);
        Prepared p;
        prepare(p, o, b, bp);
        Matrix<int32_t> got(s.m, s.n, 0);
        // i16 without the split either passes the exactness bound or is refused (exit 2)
        const OutputPipeline pipe = p.raw_pipeline();
        run_workers(o.threads, a, p.pw, got, pipe, variant_of(o));
        long long dev = 0;
        for (int i = 0; i < s.m; ++i)
            for (int j = 0; j < s.n; ++j)
                dev = std::max(dev, std::llabs(static_cast<long long>(got(i, j)) - want(i, j)));
        all = all && dev == 0;
        std::printf("M=%d N=%d K=%d variant=%s threads=%d : %s max_dev=%lld\n", s.m, s.n, s.k, o.variant.c_str(),
                    o.threads, dev == 0 ? "PASS" : "FAIL", dev);
    }
    return all ? 0 : 1;
}

int64_t median_ns(int repeats, const std::function<void()>& fn) {
    fn();
    fn();  // 2 warm-ups
    std::vector<int64_t> t(repeats);
    for (int r = 0; r < repeats; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        fn();
        t[r] = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    }
    std::nth_element(t.begin(), t.begin() + repeats / 2, t.end());
    return t[repeats / 2];
}

void csv_row(const Shape& s, const std::string& variant, int threads, int64_t ns) {
    std::printf("%d,%d,%d,%s,%d,%lld,%.4f\n", s.m, s.n, s.k, variant.c_str(), threads, static_cast<long long>(ns),
                2.0 * s.m * s.n * s.k / static_cast<double>(ns));
}

int cmd_bench(const Options& o) {
    const BlockingParams base = base_blocking(o);
    const std::vector<Shape> shapes = load_shapes(o.shapes_path);
    std::mt19937_64 g(o.seed);
    std::printf("M,N,K,variant,threads,ns_median,gops\n");
    for (const Shape& s : shapes) {
        const Matrix<uint8_t> a = draw_u8(g, s.m, s.k);
        const Matrix<int8_t> b = draw_i8(g, s.k, s.n);
        Options oi = o;
        oi.no_split = false;  // bench always splits for i16 (reference behaviour)
        Prepared p;
        prepare(p, oi, b, select_blocking(s.m, s.n, s.k, base));
        Matrix<int32_t> out(s.m, s.n, 0);
        const OutputPipeline pipe = p.raw_pipeline();
        csv_row(s, o.variant, o.threads,
                median_ns(o.repeats, [&] { run_workers(o.threads, a, p.pw, out, pipe, variant_of(o)); }));
        std::fflush(stdout);
        if (o.compare_naive) {
            Matrix<int32_t> ref;
            csv_row(s, "naive", 1, median_ns(o.repeats, [&] { ref = naive_i32(a, b); }));
        }
    }
    return 0;
}

int cmd_demo(const Options& o) {
    std::mt19937_64 g(o.seed);
    const int m = o.dm, n = o.dn, k = o.dk;
    // full-range activations; weights in [-4, 4] with a density of +-127 outliers
    const Matrix<uint8_t> aq = draw_u8(g, m, k);
    Matrix<int8_t> bq(k, n);
    for (int p = 0; p < k; ++p)
        for (int j = 0; j < n; ++j) bq(p, j) = static_cast<int8_t>(static_cast<int>(g() % 9) - 4);
    const int forced = static_cast<int>(o.density * k * n);
    for (int i = 0; i < forced; ++i) {
        const int r = static_cast<int>(g() % k);
        const int c = static_cast<int>(g() % n);
        bq(r, c) = (g() & 1) ? int8_t{127} : int8_t{-127};
    }

    const QuantParams qa = choose_quant_params(-1.0, 1.0, false);
    const QuantParams qb = choose_quant_params(-0.5, 0.5, true);
    Matrix<double> ar(m, k), br(k, n), cr(m, n, 0.0);
    for (int i = 0; i < m; ++i)
        for (int p = 0; p < k; ++p) ar(i, p) = dequantize(aq(i, p), qa);
    for (int p = 0; p < k; ++p)
        for (int j = 0; j < n; ++j) br(p, j) = dequantize(bq(p, j), qb);
    double lo = 0.0, hi = 0.0;
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int p = 0; p < k; ++p) acc += ar(i, p) * br(p, j);
            cr(i, j) = acc;
            lo = std::min(lo, acc);
            hi = std::max(hi, acc);
        }
    const QuantParams qc = choose_quant_params(lo, hi, false);

    BlockingParams base = base_blocking(o);
    if (!o.kcb) base.kcb = 32;  // a threshold that keeps the split visible
    const BlockingParams bp = select_blocking(m, n, k, base);
    const int thr = max_i16_split_threshold(bp.kcb);
    const SplitWeight sw = split_outliers(cview(bq), thr);
    const PackedWeight pw = prepack_weights(cview(sw.dense_small), bp);
    const std::vector<int32_t> co = compute_col_offsets(cview(bq));  // of the unsplit B

    RequantParams rp;
    rp.multiplier = qa.scale * qb.scale / qc.scale;
    rp.zp_a = qa.zero_point;
    rp.zp_b = qb.zero_point;
    rp.zp_c = qc.zero_point;
    rp.k_total = k;

    std::printf("INT8 x INT8 -> INT16-accumulated GEMM with outlier-aware split\n");
    std::printf("shape: M=%d N=%d K=%d  outlier_density=%.4f  seed=%llu\n", m, n, k, o.density,
                static_cast<unsigned long long>(o.seed));
    std::printf("blocking: mcb=%d ncb=%d kcb=%d mr=%d nr=%d\n", bp.mcb, bp.ncb, bp.kcb, bp.mr, bp.nr);
    std::printf("split: T=%d  nnz=%d (%.2f%% of B)  max|B'|=%d\n", thr, sw.sparse.nnz(),
                100.0 * sw.sparse.nnz() / (static_cast<double>(k) * n), pw.max_abs);
    std::printf("saturation bound: 255 * %d * %d = %lld <= 32767\n", pw.max_abs, bp.kcb, 255LL * pw.max_abs * bp.kcb);

    Matrix<uint8_t> got(m, n, 0);
    run_workers(o.threads, aq, pw, got, OutputPipeline({SpMDMAdd{&sw.sparse}, Requantize{rp, &co}}),
                KernelVariant::kAccI16);

    // integer reference: 32-bit GEMM on the unsplit B + the same requant
    const Matrix<int32_t> acc = naive_i32(aq, bq);
    int dev_int = 0, dev_real = 0;
    for (int i = 0; i < m; ++i) {
        int32_t rowsum = 0;
        for (int p = 0; p < k; ++p) rowsum += aq(i, p);
        for (int j = 0; j < n; ++j)
            dev_int = std::max(dev_int, std::abs(static_cast<int>(got(i, j)) - requant_ref(acc(i, j), rowsum, co[j], rp)));
    }
    // real-domain reference (oracle.hpp:34-54): quantize-dequantize the real
    // inputs, multiply in fp64, quantize the product
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < n; ++j) {
            double acc_r = 0.0;
            for (int p = 0; p < k; ++p)
                acc_r += dequantize(quantize<uint8_t>(ar(i, p), qa), qa) * dequantize(quantize<int8_t>(br(p, j), qb), qb);
            dev_real = std::max(dev_real, std::abs(static_cast<int>(got(i, j)) - quantize<uint8_t>(acc_r, qc)));
        }
    std::printf("engine vs integer reference: max_dev=%d (exact expected)\n", dev_int);
    std::printf("engine vs real-domain oracle: max_dev=%d (<= 1 expected)\n", dev_real);
    const bool pass = dev_int == 0 && dev_real <= 1;
    std::printf("%s\n", pass ? "PASS" : "FAIL");
    return pass ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
    std::optional<Options> o;
    try {
        o = parse_args(argc, argv);
    } catch (const UsageError& e) {
        std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
        return 2;
    }
    if (!o) {
        std::printf("%s", kUsage);
        return 0;
    }
    try {
        if (o->cmd == "verify") return cmd_verify(*o);
        if (o->cmd == "bench") return cmd_bench(*o);
        return cmd_demo(*o);
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "runtime error: %s\n", e.what());
        return 3;
    }
}
