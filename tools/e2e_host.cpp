// e2e_host.cpp — wall-clock latency of the synchronous host-view C1 call
// (q8g_gemm_u8s8_requant_host: H2D of A, GEMM, D2H of C) from C++, without
// Python in the loop; plus the bare pinned copies for the floor.
//
//   g++ -std=c++17 -O2 -I../include e2e_host.cpp -o e2e_host -L../paper_2101_05615_b200 -lq8g_b200 \
//       -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$ORIGIN/../paper_2101_05615_b200
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>

#include "q8g_b200.h"

static double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
}

template <typename F>
static double time_us(F f, int reps = 300) {
    for (int i = 0; i < 20; ++i) f();
    std::vector<double> t;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        f();
        t.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    return median(t);
}

int main() {
    const int m = 128, n = 4096, k = 4096;
    std::vector<int8_t> b((size_t)k * n);
    for (size_t i = 0; i < b.size(); ++i) b[i] = (int8_t)(i * 2654435761u >> 24);
    q8g_blocking bp;
    q8g_blocking_defaults(&bp);
    q8g_packed_b* pb = nullptr;
    if (q8g_pack_b(b.data(), k, n, n, &bp, 0, &pb)) return std::printf("pack: %s\n", q8g_last_error()), 1;
    std::vector<int32_t> zpb(n, 3);
    std::vector<float> mult(n, 1e-4f);
    q8g_requant_params rp{};
    rp.multiplier = 1.0;
    rp.zp_a = 128;
    rp.zp_c = 5;
    rp.k_total = k;
    rp.zp_b_per_channel_host = zpb.data();
    rp.multiplier_f32_per_channel_host = mult.data();
    rp.rounding = Q8G_ROUND_F32_RNE;
    rp.relu = 1;
    q8g_epilogue* ep = nullptr;
    if (q8g_epilogue_create(pb, &rp, nullptr, &ep)) return std::printf("epilogue: %s\n", q8g_last_error()), 1;
    uint8_t *a_h, *c_h, *a_d, *c_d;
    cudaHostAlloc(&a_h, (size_t)m * k, cudaHostAllocDefault);
    cudaHostAlloc(&c_h, (size_t)m * n, cudaHostAllocDefault);
    cudaMalloc(&a_d, (size_t)m * k);
    cudaMalloc(&c_d, (size_t)m * n);
    std::memset(a_h, 7, (size_t)m * k);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);

    const double h2d = time_us([&] {
        cudaMemcpyAsync(a_d, a_h, (size_t)m * k, cudaMemcpyHostToDevice, s);
        cudaEventRecord(ev, s);
        cudaEventSynchronize(ev);
    });
    const double d2h = time_us([&] {
        cudaMemcpyAsync(c_h, c_d, (size_t)m * n, cudaMemcpyDeviceToHost, s);
        cudaEventRecord(ev, s);
        cudaEventSynchronize(ev);
    });
    const double both = time_us([&] {
        cudaMemcpyAsync(a_d, a_h, (size_t)m * k, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(c_h, c_d, (size_t)m * n, cudaMemcpyDeviceToHost, s);
        cudaEventRecord(ev, s);
        cudaEventSynchronize(ev);
    });
    const double dev = time_us([&] {
        q8g_gemm_u8s8_requant(a_d, m, k, k, pb, ep, c_d, n, 0, m, nullptr, s);
        cudaEventRecord(ev, s);
        cudaEventSynchronize(ev);
    });
    const double serial = time_us([&] {
        cudaMemcpyAsync(a_d, a_h, (size_t)m * k, cudaMemcpyHostToDevice, s);
        q8g_gemm_u8s8_requant(a_d, m, k, k, pb, ep, c_d, n, 0, m, nullptr, s);
        cudaMemcpyAsync(c_h, c_d, (size_t)m * n, cudaMemcpyDeviceToHost, s);
        cudaEventRecord(ev, s);
        cudaEventSynchronize(ev);
    });
    const double host = time_us([&] {
        if (q8g_gemm_u8s8_requant_host(a_h, m, k, k, pb, ep, c_h, n, 0, m, s)) std::printf("%s\n", q8g_last_error());
    });
    std::printf("pinned H2D 512 KB %.1f us, D2H 512 KB %.1f us, both back to back %.1f us\n", h2d, d2h, both);
    std::printf("device-view GEMM call + sync %.1f us; H2D + GEMM + D2H in one stream %.1f us\n", dev, serial);
    std::printf("q8g_gemm_u8s8_requant_host %.1f us  (%.1f TOPS)\n", host, 2.0 * m * n * k / host / 1e6);
    return 0;
}
