// alu_rate.cu — per-SM issue rate of the integer ops a CUDA-core depthwise
// kernel would lean on (dp4a, PRMT byte permutes, funnel shifts, IMAD) and
// of FFMA for reference: 148 CTAs x 1024 threads, 8 independent chains.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 alu_rate.cu -o alu_rate
#include <cstdio>

template <int OP>
__global__ void __launch_bounds__(1024) k(unsigned* out, int iters, unsigned seed) {
    unsigned a[8], b = seed ^ threadIdx.x;
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = seed * (i + 1) + threadIdx.x;
        f[i] = (float)a[i];
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (OP == 0) a[i] = (unsigned)__dp4a((int)a[i], (int)b, (int)a[i]);
                if (OP == 1) a[i] = __byte_perm(a[i], b, 0x5140 + i);
                if (OP == 2) a[i] = __funnelshift_r(a[i], b, 8 + i);
                if (OP == 3) a[i] = a[i] * b + 7u;
                if (OP == 4) f[i] = __fmaf_rn(f[i], 1.0001f, 0.5f);
                if (OP == 5) a[i] = a[i] + b + (unsigned)i;
            }
    }
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s ^= a[i] ^ __float_as_uint(f[i]);
    if (s == 0x12345678u) out[0] = s;
}

int main() {
    unsigned* out;
    cudaMalloc(&out, 4);
    const char* names[] = {"dp4a (IDP4A)", "byte_perm (PRMT)", "funnelshift (SHF)", "imad", "ffma", "iadd3"};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    auto run = [&](auto kern, int op) {
        const int iters = 2000;
        kern<<<148, 1024>>>(out, 10, 1u);
        cudaEventRecord(a);
        kern<<<148, 1024>>>(out, iters, 1u);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = 148.0 * 1024 * iters * 16 * 8;
        std::printf("%-20s %7.1f Gop/s chip = %6.1f ops/clk/SM at the max clock (%d MHz)\n", names[op], ops / ms / 1e6,
                    ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    };
    run(k<0>, 0);
    run(k<1>, 1);
    run(k<2>, 2);
    run(k<3>, 3);
    run(k<4>, 4);
    run(k<5>, 5);
    return 0;
}
