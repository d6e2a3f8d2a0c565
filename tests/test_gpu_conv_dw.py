"""Parity of the conv3x3 (implicit GEMM) and depthwise-3x3 CUDA paths against
the oracle (SURVEY.md App. A D2/D3 semantics; no reference symbol exists, so
these are checked against the restated im2col -> reference-pinned GEMM ->
requant pipeline and the restated depthwise loop)."""
import numpy as np
import pytest
import torch

import configs
import paper_2101_05615_b200 as q8

pytestmark = pytest.mark.gpu


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def conv_pipeline(cc: configs.ConvCase, c: int):
    rp = q8.RequantParams(multiplier=1.0, zp_a=cc.zp_a, zp_c=cc.zp_c, k_total=9 * c, bias=cc.bias,
                          zp_b_per_channel=cc.zp_b, multiplier_f32_per_channel=cc.mult_f32,
                          rounding=q8.ROUND_F32_RNE)
    return q8.OutputPipeline(([q8.ReluQuantized()] if cc.relu else []) + [q8.Requantize(rp)])


def conv_oracle(orc, cc: configs.ConvCase):
    nb, h, w, c = cc.x.shape
    cols = orc.im2col3x3(cc.x, cc.zp_a)
    wt = cc.w.reshape(9 * c, -1)
    acc = orc.naive_gemm_i32(cols, wt)
    out = orc.requant_matrix(acc, orc.row_offsets(cols), orc.col_offsets(wt), cc.zp_a, cc.zp_b, 9 * c, cc.bias, 1,
                             cc.mult_f32, cc.zp_c, cc.relu, per_channel=True)
    return acc, out


@pytest.mark.parametrize("shape", [(1, 5, 7, 4, 8), (2, 9, 9, 16, 24), (3, 14, 14, 64, 64), (1, 3, 3, 3, 5),
                                   (2, 7, 9, 32, 40), (1, 1, 1, 64, 16), (2, 3, 60, 32, 64), (1, 6, 5, 128, 200)])
def test_conv3x3_small_vs_oracle(cuda, orc, shape):
    nb, h, w, c, oc = shape
    cc = configs.conv_case(orc, nb, h, w, c, oc, seed=sum(shape))
    pw = q8.prepack_conv3x3_weights(cc.w)
    acc, exp = conv_oracle(orc, cc)
    y = torch.zeros((nb, h, w, oc), dtype=torch.uint8, device="cuda")
    q8.execute_conv3x3(dev(cc.x), pw, y, conv_pipeline(cc, c))
    torch.cuda.synchronize()
    assert (y.cpu().numpy().reshape(-1, oc) == exp).all()
    yr = torch.zeros((nb, h, w, oc), dtype=torch.int32, device="cuda")
    q8.execute_conv3x3(dev(cc.x), pw, yr, q8.OutputPipeline([q8.WriteRawI32()]), zp_a=cc.zp_a)
    torch.cuda.synchronize()
    assert (yr.cpu().numpy().reshape(-1, oc) == acc).all()


# conv_tc extremes: C in {32, 64, 128}, OC up to 240 (two 256-column TMEM
# accumulators), the widest W (2 rows x (W+2) <= 128), odd H; ReLU on / off and
# zp_c at both ends of the saturating-pack fast path.  im2col + the
# tensor-core GEMM runs when the tile does not fit: W = 63, C = 48, or C = 128
# with OC = 240 (operand image 294 KB > shared memory)
@pytest.mark.parametrize("shape,relu,zp_c,fam", [((2, 5, 62, 32, 16), False, 0, "conv_tc"),
                                                 ((1, 7, 20, 64, 240), True, 255, "conv_tc"),
                                                 ((1, 5, 9, 128, 112), False, 3, "conv_tc"),
                                                 ((3, 4, 11, 64, 112), False, 255, "conv_tc"),
                                                 ((1, 2, 63, 32, 32), True, 5, "conv_im2col"),
                                                 ((1, 3, 8, 48, 32), False, 9, "conv_im2col"),
                                                 ((1, 3, 6, 128, 240), True, 5, "conv_im2col")])
def test_conv3x3_edge_shapes_vs_oracle(cuda, orc, shape, relu, zp_c, fam):
    import dataclasses
    nb, h, w, c, oc = shape
    cc = dataclasses.replace(configs.conv_case(orc, nb, h, w, c, oc, seed=3 * sum(shape)), relu=relu, zp_c=zp_c)
    pw = q8.prepack_conv3x3_weights(cc.w)
    _, exp = conv_oracle(orc, cc)
    before = q8.launch_stats()[fam]
    y = torch.zeros((nb, h, w, oc), dtype=torch.uint8, device="cuda")
    q8.execute_conv3x3(dev(cc.x), pw, y, conv_pipeline(cc, c))
    torch.cuda.synchronize()
    assert (y.cpu().numpy().reshape(-1, oc) == exp).all()
    assert q8.launch_stats()[fam] == before + 1


def test_conv3x3_c3_full_vs_oracle(cuda, orc):
    cc = configs.conv_case(orc)  # 32x56x56x64 -> 64, BASELINE configs[3]
    pw = q8.prepack_conv3x3_weights(cc.w)
    _, exp = conv_oracle(orc, cc)
    y = torch.zeros((32, 56, 56, 64), dtype=torch.uint8, device="cuda")
    q8.execute_conv3x3(dev(cc.x), pw, y, conv_pipeline(cc, 64))
    torch.cuda.synchronize()
    assert (y.cpu().numpy().reshape(-1, 64) == exp).all()
    # batch shards (one per GPU at 1/2/4/8) compose to the same output
    y2 = torch.zeros_like(y)
    for i0, i1 in [(0, 8), (8, 16), (16, 24), (24, 32)]:
        q8.execute_conv3x3(dev(cc.x), pw, y2, conv_pipeline(cc, 64), image_begin=i0, image_end=i1)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)


def test_conv3x3_host_views_chunked_equal_device(cuda, orc):
    """q8g_conv3x3_u8s8_nhwc_host (the reference convention: host views),
    chunked with its copies overlapped, equals the oracle at the full C3 size,
    image sub-ranges included."""
    cc = configs.conv_case(orc)
    pw = q8.prepack_conv3x3_weights(cc.w)
    _, exp = conv_oracle(orc, cc)
    y = np.zeros((32, 56, 56, 64), dtype=np.uint8)
    q8.execute_conv3x3(np.ascontiguousarray(cc.x), pw, y, conv_pipeline(cc, 64))
    assert (y.reshape(-1, 64) == exp).all()
    y2 = np.full_like(y, 7)
    q8.execute_conv3x3(np.ascontiguousarray(cc.x), pw, y2, conv_pipeline(cc, 64), image_begin=5, image_end=19)
    assert (y2[5:19] == y[5:19]).all() and (y2[:5] == 7).all() and (y2[19:] == 7).all()


def test_conv3x3_concurrent_first_use_on_two_streams(cuda, orc):
    """A conv weight packed through the plain GEMM packer (no eager operand
    image) is used for the first time by two threads on two streams at once:
    the image is built once under a lock and both outputs are exact
    (pack.hpp:59-62: a packed weight is shareable across concurrent calls)."""
    import threading
    cc = configs.conv_case(orc, 4, 14, 14, 64, 64, seed=21)
    pw = q8.prepack_weights(cc.w.reshape(9 * 64, 64))  # no q8g_conv3x3_prepare
    _, exp = conv_oracle(orc, cc)
    pipe = conv_pipeline(cc, 64)
    pipe.epilogue(pw)
    xd = dev(cc.x)
    ys = [torch.zeros((4, 14, 14, 64), dtype=torch.uint8, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    errs = []
    barrier = threading.Barrier(2)

    def work(i):
        try:
            barrier.wait()
            q8.execute_conv3x3(xd, pw, ys[i], pipe, stream=streams[i])
            streams[i].synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for y in ys:
        assert (y.cpu().numpy().reshape(-1, 64) == exp).all()


def test_conv3x3_work_slot_ring_wraps(cuda, orc):
    """The implicit-GEMM conv claims its tail units from a per-launch work slot
    (a 1024-slot ring per device whose last CTA re-zeroes the slot).  1100
    launches alternating over two streams wrap the ring; every launch must
    still cover every unit exactly once (outputs equal to the oracle)."""
    cc = configs.conv_case(orc, 6, 20, 20, 64, 64, seed=33)
    pw = q8.prepack_conv3x3_weights(cc.w)
    _, exp = conv_oracle(orc, cc)
    pipe = conv_pipeline(cc, 64)
    xd = dev(cc.x)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ys = [torch.zeros((6, 20, 20, 64), dtype=torch.uint8, device="cuda") for _ in range(4)]
    for i in range(1100):
        y = ys[i % 4]
        if i >= 1096:
            y.fill_(0)  # the last launch on each buffer starts from zeros
        q8.execute_conv3x3(xd, pw, y, pipe, stream=streams[i % 2])
    torch.cuda.synchronize()
    for y in ys:
        assert (y.cpu().numpy().reshape(-1, 64) == exp).all()


def dw_filter(dc: configs.DwCase):
    rp = q8.RequantParams(multiplier=1.0, zp_a=dc.zp_a, zp_c=dc.zp_c, k_total=9, bias=dc.bias,
                          zp_b_per_channel=dc.zp_w, multiplier_f32_per_channel=dc.mult_f32,
                          rounding=q8.ROUND_F32_RNE)
    return q8.DepthwiseFilter(dc.w, rp, relu=dc.relu)


@pytest.mark.parametrize("shape", [(1, 4, 5, 4), (2, 7, 9, 12), (1, 16, 16, 256), (2, 3, 3, 7), (1, 1, 1, 8)])
def test_dwconv_small_vs_oracle(cuda, orc, shape):
    nb, h, w, c = shape
    dc = configs.dw_case(orc, nb, h, w, c, seed=sum(shape))
    exp, _ = orc.dwconv3x3(dc.x, dc.zp_a, dc.w, dc.zp_w, dc.bias, dc.mult_f32, dc.zp_c, dc.relu)
    y = torch.zeros(shape, dtype=torch.uint8, device="cuda")
    q8.execute_dwconv3x3(dev(dc.x), dw_filter(dc), y)
    torch.cuda.synchronize()
    assert (y.cpu().numpy() == exp).all()


# dwconv_fma (C % 128 == 0, W + 2 > 128): 56-position segments with a
# partial last segment, ragged row chunks;
# dwconv_tc64 (C % 64 == 0, W + 2 <= 128): one / several channel blocks, odd H
# (tail row block), W = 1 and the widest W; the 16-channel kernel for C % 64
# != 0; the CUDA-core kernel when a 16-channel unit no longer fits one TMEM
# buffer (W = 200); ReLU on and off, zp_c at both ends
@pytest.mark.parametrize("shape,relu,zp_c,fam", [((3, 5, 7, 64), True, 5, "dw_tc"), ((1, 1, 1, 64), False, 0, "dw_tc"),
                                                 ((2, 9, 126, 128), False, 255, "dw_tc"),
                                                 ((1, 2, 1, 192), True, 200, "dw_tc"),
                                                 ((2, 4, 30, 48), False, 17, "dw_tc"),
                                                 ((1, 3, 200, 64), True, 5, "dw_simt"),
                                                 ((4, 7, 13, 256), False, 128, "dw_tc"),
                                                 ((1, 14, 300, 128), True, 9, "dw_fma"),
                                                 ((2, 17, 127, 256), False, 3, "dw_fma")])
def test_dwconv_tc_edge_shapes_vs_oracle(cuda, orc, shape, relu, zp_c, fam):
    import dataclasses
    nb, h, w, c = shape
    dc = dataclasses.replace(configs.dw_case(orc, nb, h, w, c, seed=7 * sum(shape)), relu=relu, zp_c=zp_c)
    exp, _ = orc.dwconv3x3(dc.x, dc.zp_a, dc.w, dc.zp_w, dc.bias, dc.mult_f32, dc.zp_c, dc.relu)
    before = q8.launch_stats()[fam]
    f = dw_filter(dc)
    xd = dev(dc.x)
    y = torch.zeros(shape, dtype=torch.uint8, device="cuda")
    q8.execute_dwconv3x3(xd, f, y)
    torch.cuda.synchronize()
    assert (y.cpu().numpy() == exp).all()
    assert q8.launch_stats()[fam] == before + 1  # the expected kernel family ran
    if nb > 1:  # image shards compose
        y2 = torch.zeros_like(y)
        for i0, i1 in [(0, 1), (1, nb)]:
            q8.execute_dwconv3x3(xd, f, y2, image_begin=i0, image_end=i1)
        torch.cuda.synchronize()
        assert torch.equal(y, y2)


@pytest.mark.parametrize("shape", [(3, 6, 112, 256), (3, 5, 33, 64)])
def test_dwconv_tc64_shard_leaves_other_images_untouched(cuda, orc, shape):
    """The 64-channel kernel writes through per-warp TMA stores of 32
    positions x 32 channels, clipped by the output tensor map: convolving
    image range [1, 2) must write exactly image 1 -- no byte of images 0 / 2
    and no position past W."""
    nb, h, w, c = shape
    dc = configs.dw_case(orc, nb, h, w, c, seed=5 + w)
    exp, _ = orc.dwconv3x3(dc.x, dc.zp_a, dc.w, dc.zp_w, dc.bias, dc.mult_f32, dc.zp_c, dc.relu)
    before = q8.launch_stats()["dw_tc"]
    y = torch.full(shape, 0xA5, dtype=torch.uint8, device="cuda")
    q8.execute_dwconv3x3(dev(dc.x), dw_filter(dc), y, image_begin=1, image_end=2)
    torch.cuda.synchronize()
    assert q8.launch_stats()["dw_tc"] == before + 1
    yh = y.cpu().numpy()
    assert (yh[1] == exp[1]).all()
    assert (yh[0] == 0xA5).all() and (yh[2] == 0xA5).all()


# the FMA-pipe kernel forced (Q8G_DW_FMA=1) on shapes the tensor-core kernel
# takes by default: row chunks of 14 with ragged tails, 56-position segments
# with partial last segments, several channel blocks, H = W = 1; both kernels
# agree bit for bit with the oracle
@pytest.mark.parametrize("shape,relu,zp_c", [((2, 9, 126, 128), False, 255), ((3, 17, 56, 256), True, 5),
                                             ((1, 1, 1, 128), True, 5), ((3, 29, 57, 128), True, 0),
                                             ((2, 15, 112, 384), False, 77), ((1, 2, 5, 128), True, 200)])
def test_dwconv_fma_vs_tc_same_bits(cuda, orc, shape, relu, zp_c, monkeypatch):
    import dataclasses
    nb, h, w, c = shape
    dc = dataclasses.replace(configs.dw_case(orc, nb, h, w, c, seed=11 * sum(shape)), relu=relu, zp_c=zp_c)
    exp, _ = orc.dwconv3x3(dc.x, dc.zp_a, dc.w, dc.zp_w, dc.bias, dc.mult_f32, dc.zp_c, dc.relu)
    f = dw_filter(dc)
    xd = dev(dc.x)
    y = torch.zeros(shape, dtype=torch.uint8, device="cuda")
    before = q8.launch_stats()
    q8.execute_dwconv3x3(xd, f, y)
    monkeypatch.setenv("Q8G_DW_FMA", "1")
    yf = torch.zeros_like(y)
    q8.execute_dwconv3x3(xd, f, yf)
    torch.cuda.synchronize()
    after = q8.launch_stats()
    assert after["dw_fma"] == before["dw_fma"] + 1 and after["dw_tc"] == before["dw_tc"] + 1
    assert (y.cpu().numpy() == exp).all()
    assert torch.equal(y, yf)


# the FMA kernel's exactness limits: extreme bytes and weights, zp_w at
# +-127 (|w - zp_w| = 255), zp_a at 0 / 255, the largest admitted bias, huge
# multipliers (saturation both ways), tiny and denormal-range multipliers,
# zp_c at both ends, ReLU on and off
@pytest.mark.parametrize("variant", range(6))
def test_dwconv_fma_extremes_vs_oracle(cuda, orc, variant):
    nb, h, w, c = 2, 16, 130, 128  # W + 2 > 128: the FMA-pipe kernel by default
    r = np.random.default_rng(1000 + variant)
    choice = lambda vals, size: r.choice(np.asarray(vals), size=size)  # noqa: E731
    x = choice([0, 1, 127, 128, 254, 255], (nb, h, w, c)).astype(np.uint8)
    wt = choice([-128, -127, -1, 0, 1, 126, 127], (3, 3, c)).astype(np.int8)
    zp_w = choice([-127, -10, 0, 10, 127], c).astype(np.int32)
    zp_a = [0, 255, 128, 3, 200, 128][variant]
    big = (1 << 23) - 2 * 9 * 255 * 255 - 1
    bias = r.integers(-big, big + 1, c).astype(np.int32)
    bias[:4] = [big, -big, 0, big]
    mult = [r.uniform(1e-7, 1e-5, c), r.uniform(1e-4, 1e-2, c), np.full(c, 3.0e5), r.uniform(1e-38, 1e-30, c),
            r.uniform(0.5, 2.0, c), 10.0 ** r.uniform(-9, 4, c)][variant].astype(np.float32)
    zp_c, relu = [(0, False), (255, True), (5, True), (128, False), (0, True), (17, False)][variant]
    dc = configs.DwCase(x, wt, bias, zp_a, zp_w, mult, zp_c, relu)
    exp, _ = orc.dwconv3x3(dc.x, dc.zp_a, dc.w, dc.zp_w, dc.bias, dc.mult_f32, dc.zp_c, dc.relu)
    before = q8.launch_stats()["dw_fma"]
    y = torch.zeros(x.shape, dtype=torch.uint8, device="cuda")
    q8.execute_dwconv3x3(dev(x), dw_filter(dc), y)
    torch.cuda.synchronize()
    assert q8.launch_stats()["dw_fma"] == before + 1
    assert (y.cpu().numpy() == exp).all()


def test_dwconv_c4_full_vs_oracle(cuda, orc):
    dc = configs.dw_case(orc)  # 32x112x112x256, BASELINE configs[4]
    exp, _ = orc.dwconv3x3(dc.x, dc.zp_a, dc.w, dc.zp_w, dc.bias, dc.mult_f32, dc.zp_c, dc.relu)
    f = dw_filter(dc)
    y = torch.zeros(dc.x.shape, dtype=torch.uint8, device="cuda")
    xd = dev(dc.x)
    q8.execute_dwconv3x3(xd, f, y)
    torch.cuda.synchronize()
    assert (y.cpu().numpy() == exp).all()
    y2 = torch.zeros_like(y)
    for i0, i1 in [(0, 3), (3, 17), (17, 32)]:
        q8.execute_dwconv3x3(xd, f, y2, image_begin=i0, image_end=i1)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)
    # host views (q8g_dwconv3x3_u8s8_nhwc_host: chunked, copies overlapped)
    yh = np.zeros(dc.x.shape, dtype=np.uint8)
    q8.execute_dwconv3x3(np.ascontiguousarray(dc.x), f, yh)
    assert (yh == exp).all()


# im2col + tensor-core GEMM: the channel counts real networks use beyond the
# implicit-GEMM kernel (256, 512), odd C (byte-wise im2col, K padded to 16),
# OC > 240, and the CUDA-core kernel forced for the same shapes
@pytest.mark.parametrize("shape", [(2, 14, 14, 256, 256), (1, 7, 7, 512, 128), (2, 9, 11, 3, 64),
                                   (1, 6, 5, 17, 300), (4, 28, 28, 256, 64)])
def test_conv3x3_im2col_gemm_vs_oracle(cuda, orc, shape, monkeypatch):
    nb, h, w, c, oc = shape
    cc = configs.conv_case(orc, nb, h, w, c, oc, seed=7 * sum(shape))
    pw = q8.prepack_conv3x3_weights(cc.w)
    acc, exp = conv_oracle(orc, cc)
    before = q8.launch_stats()
    y = torch.zeros((nb, h, w, oc), dtype=torch.uint8, device="cuda")
    q8.execute_conv3x3(dev(cc.x), pw, y, conv_pipeline(cc, c))
    yr = torch.zeros((nb, h, w, oc), dtype=torch.int32, device="cuda")
    q8.execute_conv3x3(dev(cc.x), pw, yr, q8.OutputPipeline([q8.WriteRawI32()]), zp_a=cc.zp_a)
    torch.cuda.synchronize()
    after = q8.launch_stats()
    assert after["conv_im2col"] == before["conv_im2col"] + 2 and after["conv_simt"] == before["conv_simt"]
    assert (y.cpu().numpy().reshape(-1, oc) == exp).all()
    assert (yr.cpu().numpy().reshape(-1, oc) == acc).all()
    monkeypatch.setenv("Q8G_CONV_SIMT", "1")
    ys = torch.zeros_like(y)
    q8.execute_conv3x3(dev(cc.x), pw, ys, conv_pipeline(cc, c))
    torch.cuda.synchronize()
    assert q8.launch_stats()["conv_simt"] == after["conv_simt"] + 1
    assert torch.equal(ys, y)
