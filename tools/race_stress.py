"""Race / memory-ordering stress of the tensor-core kernels (compute-sanitizer
is closed on this GPU pool, so this is the round's substitute evidence): each
kernel family runs REPS times on the same inputs -- back to back on one
stream (PDL overlap between neighbours), and interleaved on two streams at
once -- and every output must be bit-identical to the first, which itself
must equal the oracle.  A missing mbarrier / fence / TMEM hand-off would show
up as sporadic mismatches.  Writes one summary line per family.

  python tools/race_stress.py [--reps 200]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import configs  # noqa: E402
import paper_2101_05615_b200 as q8  # noqa: E402
from oracle.py import Oracle  # noqa: E402

orc = Oracle()


def stress(name, run, exp, out_like, reps):
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    first = out_like()
    run(first, streams[0])
    torch.cuda.synchronize()
    ok0 = bool((first.cpu().numpy().reshape(exp.shape) == exp).all())
    outs = [out_like() for _ in range(8)]
    bad = 0
    for r in range(reps // 8):
        for i, o in enumerate(outs):
            run(o, streams[i % 2] if r % 2 else streams[0])
        torch.cuda.synchronize()
        for o in outs:
            bad += int(not torch.equal(o, first))
            o.fill_(0xA5 if o.dtype == torch.uint8 else -1)
    print(f"{name:48s} oracle {'ok' if ok0 else 'MISMATCH'}  {reps // 8 * 8} reruns, {bad} differing", flush=True)
    return ok0 and bad == 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    args = ap.parse_args()
    ok = True
    for name, (m, n, k) in [("split-K C1 (128x4096x4096)", (128, 4096, 4096)),
                            ("CTA pair 256x512 (4096x4096x1024)", (4096, 4096, 1024)),
                            ("128-column tiles (512x4096x1024)", (512, 4096, 1024))]:
        c = configs.gemm_case(orc, "C1", m, n, k, seed=m + k)
        pw = q8.prepack_weights(c.b)
        acc = orc.naive_gemm_i32(c.a, c.b)
        exp = orc.requant_matrix(acc, orc.row_offsets(c.a), orc.col_offsets(c.b), c.zp_a, c.zp_b, k, c.bias, 1,
                                 c.mult_f32, c.zp_c, True, per_channel=True)
        rp = q8.RequantParams(zp_a=c.zp_a, zp_c=c.zp_c, k_total=k, bias=c.bias, zp_b_per_channel=c.zp_b,
                              multiplier_f32_per_channel=c.mult_f32, rounding=q8.ROUND_F32_RNE)
        pipe = q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)])
        ad = torch.from_numpy(c.a).cuda()
        ok &= stress(name, lambda o, s: q8.execute_gemm(ad, pw, o, pipe, stream=s), exp,
                     lambda: torch.zeros((m, n), dtype=torch.uint8, device="cuda"), args.reps)
    cc = configs.conv_case(orc, 8, 56, 56, 64, 64, seed=3)
    pw = q8.prepack_conv3x3_weights(cc.w)
    cols = orc.im2col3x3(cc.x, cc.zp_a)
    wt = cc.w.reshape(576, 64)
    acc = orc.naive_gemm_i32(cols, wt)
    exp = orc.requant_matrix(acc, orc.row_offsets(cols), orc.col_offsets(wt), cc.zp_a, cc.zp_b, 576, cc.bias, 1,
                             cc.mult_f32, cc.zp_c, cc.relu, per_channel=True)
    rp = q8.RequantParams(multiplier=1.0, zp_a=cc.zp_a, zp_c=cc.zp_c, k_total=576, bias=cc.bias,
                          zp_b_per_channel=cc.zp_b, multiplier_f32_per_channel=cc.mult_f32, rounding=q8.ROUND_F32_RNE)
    pipe = q8.OutputPipeline(([q8.ReluQuantized()] if cc.relu else []) + [q8.Requantize(rp)])
    xd = torch.from_numpy(cc.x).cuda()
    ok &= stress("conv3x3 implicit GEMM (8x56x56x64->64)", lambda o, s: q8.execute_conv3x3(xd, pw, o, pipe, stream=s),
                 exp, lambda: torch.zeros((8, 56, 56, 64), dtype=torch.uint8, device="cuda"), args.reps)
    for shape in [(4, 112, 112, 256), (2, 30, 140, 128)]:
        dc = configs.dw_case(orc, *shape, seed=7)
        exp, _ = orc.dwconv3x3(dc.x, dc.zp_a, dc.w, dc.zp_w, dc.bias, dc.mult_f32, dc.zp_c, dc.relu)
        rp = q8.RequantParams(multiplier=1.0, zp_a=dc.zp_a, zp_c=dc.zp_c, k_total=9, bias=dc.bias,
                              zp_b_per_channel=dc.zp_w, multiplier_f32_per_channel=dc.mult_f32,
                              rounding=q8.ROUND_F32_RNE)
        f = q8.DepthwiseFilter(dc.w, rp, relu=dc.relu)
        xd = torch.from_numpy(dc.x).cuda()
        before = q8.launch_stats()
        q8.execute_dwconv3x3(xd, f, torch.zeros(dc.x.shape, dtype=torch.uint8, device="cuda"))
        torch.cuda.synchronize()
        fam = ",".join(k2 for k2, v in q8.launch_stats().items() if v != before[k2])
        ok &= stress(f"depthwise {shape} ({fam})", lambda o, s, xd=xd, f=f: q8.execute_dwconv3x3(xd, f, o, stream=s),
                     exp, lambda shape=dc.x.shape: torch.zeros(shape, dtype=torch.uint8, device="cuda"), args.reps)
    print("ALL OK" if ok else "FAILURES", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
