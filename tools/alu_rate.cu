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
                if (OP == 6 && (i & 1) == 0) {
                    unsigned long long x = ((unsigned long long)__float_as_uint(f[i + 1]) << 32) | __float_as_uint(f[i]);
                    const unsigned long long m = 0x3F8000343F800034ull, c = 0x3F0000003F000000ull;
                    asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(m), "l"(c));
                    f[i] = __uint_as_float((unsigned)x);
                    f[i + 1] = __uint_as_float((unsigned)(x >> 32));
                }
                if (OP == 7 && (i & 1) == 0) {
                    unsigned long long x = ((unsigned long long)__float_as_uint(f[i + 1]) << 32) | __float_as_uint(f[i]);
                    const unsigned long long c = 0x3F0000003F000000ull;
                    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(c));
                    f[i] = __uint_as_float((unsigned)x);
                    f[i + 1] = __uint_as_float((unsigned)(x >> 32));
                }
                if (OP == 8) {
                    unsigned d;
                    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a[i]), "r"(b), "r"(a[(i + 1) & 7]));
                    a[i] = d;
                }
                if (OP == 9) f[i] = fmaxf(f[i], __uint_as_float(b));
                if (OP == 11 && (i & 1) == 0) {  // FFMA2, three register-pair operands (depthwise MAC shape)
                    float2 acc = make_float2(f[i], f[i + 1]);
                    const float2 xx = make_float2(__uint_as_float(a[i]), __uint_as_float(a[i + 1]));
                    const float2 ww = make_float2(__uint_as_float(a[(i + 2) & 7]), __uint_as_float(a[(i + 3) & 7]));
                    acc = __ffma2_rn(xx, ww, acc);
                    f[i] = acc.x;
                    f[i + 1] = acc.y;
                }
                if (OP == 12) f[i] = __fmaf_rn(__uint_as_float(a[i]), __uint_as_float(a[(i + 3) & 7]), f[i]);
                if (OP == 13 && (i & 1) == 0) {  // FFMA2 (3 reg pairs) + 1 PRMT
                    float2 acc = make_float2(f[i], f[i + 1]);
                    const float2 xx = make_float2(__uint_as_float(a[i]), __uint_as_float(a[i + 1]));
                    const float2 ww = make_float2(__uint_as_float(a[(i + 2) & 7]), __uint_as_float(a[(i + 3) & 7]));
                    acc = __ffma2_rn(xx, ww, acc);
                    f[i] = acc.x;
                    f[i + 1] = acc.y;
                    a[i] = __byte_perm(a[i], b, 0x5140 + i);
                }
                if (OP == 10) {  // 1 PRMT per FFMA: dual-pipe co-issue
                    a[i] = __byte_perm(a[i], b, 0x5140 + i);
                    f[i] = __fmaf_rn(f[i], 1.0001f, __uint_as_float(b));
                }
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
    const char* names[] = {"dp4a (IDP4A)", "byte_perm (PRMT)", "funnelshift (SHF)", "imad", "ffma", "iadd3", "ffma2 (f32x2) instr", "fadd2 instr", "cvt.pack.sat I2IP", "fmnmx", "prmt+ffma pairs", "ffma2 3-reg instr", "ffma 3-reg", "ffma2 3-reg + prmt (instr pairs)"};
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
        const double ops = 148.0 * 1024 * iters * 16 * ((op == 6 || op == 7 || op == 11 || op == 13) ? 4 : 8);
        std::printf("%-20s %7.1f Gop/s chip = %6.1f ops/clk/SM at the max clock (%d MHz)\n", names[op], ops / ms / 1e6,
                    ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    };
    run(k<0>, 0);
    run(k<1>, 1);
    run(k<2>, 2);
    run(k<3>, 3);
    run(k<4>, 4);
    run(k<5>, 5);
    run(k<6>, 6);
    run(k<7>, 7);
    run(k<8>, 8);
    run(k<9>, 9);
    run(k<10>, 10);
    run(k<11>, 11);
    run(k<12>, 12);
    run(k<13>, 13);
    return 0;
}
