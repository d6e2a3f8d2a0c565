"""One small launch of every tensor-core kernel family, checked against the
oracle -- the workload run under compute-sanitizer (memcheck / racecheck /
synccheck / initcheck, one tool per run) for the round's race / memory
evidence (profiles/r02_sanitizer_*.log):

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py

split-K (M <= 128), 128-column 1-CTA tiles, the 256 x 256 and 256 x 512
CTA-pair kernels (F32 fast path with TMA stores, raw, REF), conv3x3
implicit GEMM, depthwise 16/64-channel tensor-core kernels, the FMA-pipe
depthwise kernel and the general-pipeline post kernel.  Exits non-zero on
any mismatch."""
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
bad = []


def check(name, got, exp):
    ok = bool((np.asarray(got) == np.asarray(exp)).all())
    print(f"{name:44s} {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        bad.append(name)


def gemm(name, m, n, k, rounding=q8.ROUND_F32_RNE, raw=False):
    c = configs.gemm_case(orc, "C1", m, n, k, seed=m + n + k)
    pw = q8.prepack_weights(c.b)
    acc = orc.naive_gemm_i32(c.a, c.b)
    if raw:
        out = torch.zeros((m, n), dtype=torch.int32, device="cuda")
        q8.execute_gemm(torch.from_numpy(c.a).cuda(), pw, out, q8.OutputPipeline([q8.WriteRawI32()]))
        torch.cuda.synchronize()
        return check(name, out.cpu().numpy(), acc)
    rp = q8.RequantParams(zp_a=c.zp_a, zp_c=c.zp_c, k_total=k, bias=c.bias, zp_b_per_channel=c.zp_b,
                          multiplier_f32_per_channel=c.mult_f32, rounding=q8.ROUND_F32_RNE)
    exp = orc.requant_matrix(acc, orc.row_offsets(c.a), orc.col_offsets(c.b), c.zp_a, c.zp_b, k, c.bias, 1,
                             c.mult_f32, c.zp_c, True, per_channel=True)
    out = torch.zeros((m, n), dtype=torch.uint8, device="cuda")
    q8.execute_gemm(torch.from_numpy(c.a).cuda(), pw, out, q8.OutputPipeline([q8.ReluQuantized(), q8.Requantize(rp)]))
    torch.cuda.synchronize()
    check(name, out.cpu().numpy(), exp)


gemm("split-K (128 x 1024 x 1024)", 128, 1024, 1024)
gemm("128-column tiles (512 x 1024 x 512)", 512, 1024, 512)
gemm("CTA pair 256x512 F32+TMA store (2560x2048x512)", 2560, 2048, 512)
gemm("CTA pair 256x512 raw (2560x2048x256)", 2560, 2048, 256, raw=True)
# (run again with Q8G_TC2W=0 for the 256 x 256 pair kernel in the two cases above)

cc = configs.conv_case(orc, 2, 14, 14, 64, 64, seed=9)
pw = q8.prepack_conv3x3_weights(cc.w)
nb, h, w, c = cc.x.shape
cols = orc.im2col3x3(cc.x, cc.zp_a)
wt = cc.w.reshape(9 * c, -1)
acc = orc.naive_gemm_i32(cols, wt)
exp = orc.requant_matrix(acc, orc.row_offsets(cols), orc.col_offsets(wt), cc.zp_a, cc.zp_b, 9 * c, cc.bias, 1,
                         cc.mult_f32, cc.zp_c, cc.relu, per_channel=True)
rp = q8.RequantParams(multiplier=1.0, zp_a=cc.zp_a, zp_c=cc.zp_c, k_total=9 * c, bias=cc.bias,
                      zp_b_per_channel=cc.zp_b, multiplier_f32_per_channel=cc.mult_f32, rounding=q8.ROUND_F32_RNE)
y = torch.zeros((nb, h, w, 64), dtype=torch.uint8, device="cuda")
q8.execute_conv3x3(torch.from_numpy(cc.x).cuda(), pw,
                   y, q8.OutputPipeline(([q8.ReluQuantized()] if cc.relu else []) + [q8.Requantize(rp)]))
torch.cuda.synchronize()
check("conv3x3 implicit GEMM (2x14x14x64->64)", y.cpu().numpy().reshape(-1, 64), exp)

for shape, env in [((1, 9, 20, 64), {}), ((1, 5, 9, 32), {}), ((1, 9, 130, 128), {})]:
    dc = configs.dw_case(orc, *shape, seed=sum(shape))
    exp, _ = orc.dwconv3x3(dc.x, dc.zp_a, dc.w, dc.zp_w, dc.bias, dc.mult_f32, dc.zp_c, dc.relu)
    rp = q8.RequantParams(multiplier=1.0, zp_a=dc.zp_a, zp_c=dc.zp_c, k_total=9, bias=dc.bias,
                          zp_b_per_channel=dc.zp_w, multiplier_f32_per_channel=dc.mult_f32, rounding=q8.ROUND_F32_RNE)
    f = q8.DepthwiseFilter(dc.w, rp, relu=dc.relu)
    y = torch.zeros(dc.x.shape, dtype=torch.uint8, device="cuda")
    before = q8.launch_stats()
    q8.execute_dwconv3x3(torch.from_numpy(dc.x).cuda(), f, y)
    torch.cuda.synchronize()
    fam = [k for k, v in q8.launch_stats().items() if v != before[k]]
    check(f"depthwise {shape} ({','.join(fam)})", y.cpu().numpy(), exp)

sys.exit(1 if bad else 0)
