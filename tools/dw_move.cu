// dw_move.cu — the depthwise kernel's data movement alone (no MMA, no
// requant): per unit, one 4-D TMA halo load {CB channels, W+2, R+2 rows} and
// one 4-D TMA store of the {CB, W, R} output tile, NB halos in flight, C4's
// shape (32 x 112 x 112 x 256 u8).  How fast can this pattern move C4's bytes
// as a function of the channel-block width CB (64 / 128 bytes per position
// row) and R?  (The 64-channel kernel moves at most ~3.4 TB/s this way.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2101_05615_b200/csrc dw_move.cu -lcuda -o dw_move
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "ptx.cuh"

using namespace q8g;

constexpr int NB_MAX = 6;

__global__ void __launch_bounds__(128, 1) mover(const __grid_constant__ CUtensorMap tx, const __grid_constant__ CUtensorMap ty,
                                               int cb_bytes, int r, int nb, int nblk, int rblocks, int nimg, int halo_bytes,
                                               int out_bytes) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[NB_MAX];
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const int hstride = (halo_bytes + 1023) / 1024 * 1024;
    const uint32_t out_s = base + nb * hstride;
    if (threadIdx.x == 0) {
        for (int b = 0; b < nb; ++b) ptx::mbar_init(ptx::smem_u32(&bars[b]), 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int cb = blockIdx.x % nblk, cta_in = blockIdx.x / nblk;
    const int ctas = ((int)gridDim.x - cb + nblk - 1) / nblk;
    const int units = nimg * rblocks;
    const int mine = units > cta_in ? (units - cta_in + ctas - 1) / ctas : 0;
    auto issue = [&](int i) {
        const int k = cta_in + i * ctas, b = i % nb;
        const int n = k / rblocks, rb = k % rblocks;
        ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bars[b]), (uint32_t)halo_bytes);
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                base + b * hstride),
            "l"(reinterpret_cast<uint64_t>(&tx)), "r"(cb * cb_bytes), "r"(-1), "r"(rb * r - 1), "r"(n),
            "r"(ptx::smem_u32(&bars[b]))
            : "memory");
    };
    for (int i = 0; i < nb && i < mine; ++i) issue(i);
    for (int i = 0; i < mine; ++i) {
        const int b = i % nb;
        ptx::mbar_wait_spin(ptx::smem_u32(&bars[b]), (uint32_t)(i / nb) & 1u);
        const int k = cta_in + i * ctas;
        const int n = k / rblocks, rb = k % rblocks;
        // "compute": the output tile is whatever sits in the staging buffer
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                         reinterpret_cast<uint64_t>(&ty)),
                     "r"(cb * cb_bytes), "r"(0), "r"(rb * r), "r"(n), "r"(out_s)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (i + nb < mine) issue(i + nb);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    (void)out_bytes;
}

int main() {
    const int N = 32, H = 112, W = 112, C = 256;
    uint8_t *x, *y;
    cudaMalloc(&x, (size_t)N * H * W * C);
    cudaMalloc(&y, (size_t)N * H * W * C);
    cudaMemset(x, 1, (size_t)N * H * W * C);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    cudaFuncSetAttribute(mover, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
    struct Cfg { int cb, r, nb; };
    const Cfg cfgs[] = {{64, 2, 4}, {64, 2, 6}, {64, 4, 3}, {128, 2, 3}, {128, 1, 4}, {128, 2, 2}};
    for (const Cfg& c : cfgs) {
        cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
        cuuint64_t strides[3] = {(cuuint64_t)C, (cuuint64_t)W * C, (cuuint64_t)H * W * C};
        cuuint32_t boxx[4] = {(cuuint32_t)c.cb, (cuuint32_t)(W + 2), (cuuint32_t)(c.r + 2), 1};
        cuuint32_t boxy[4] = {(cuuint32_t)c.cb, (cuuint32_t)W, (cuuint32_t)c.r, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        const CUtensorMapSwizzle sw = c.cb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
        CUtensorMap tx, ty;
        if (enc(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, x, dims, strides, boxx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
            enc(&ty, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, y, dims, strides, boxy, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            std::printf("encode failed for cb=%d r=%d\n", c.cb, c.r);
            continue;
        }
        const int nblk = C / c.cb, rblocks = (H + c.r - 1) / c.r;
        const int halo = c.cb * (W + 2) * (c.r + 2), out = c.cb * W * c.r;
        const int smem = c.nb * ((halo + 1023) / 1024 * 1024) + out + 2048;
        if (smem > 225 * 1024) {
            std::printf("cb=%d r=%d nb=%d: %d B smem, skipped\n", c.cb, c.r, c.nb, smem);
            continue;
        }
        const int grid = (148 / nblk) * nblk;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) mover<<<grid, 128, smem>>>(tx, ty, c.cb, c.r, c.nb, nblk, rblocks, N, halo, out);
        cudaEventRecord(a);
        const int reps = 10;
        for (int rep = 0; rep < reps; ++rep) mover<<<grid, 128, smem>>>(tx, ty, c.cb, c.r, c.nb, nblk, rblocks, N, halo, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double us = ms * 1e3 / reps;
        std::printf("CB=%3d B rows, R=%d output rows/unit, %d halos in flight: %7.1f us per pass (%.2f TB/s of C4's 205.5 MB)  %s\n",
                    c.cb, c.r, c.nb, us, 205.5e6 / (us * 1e-6) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
