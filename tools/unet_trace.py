"""Role timing of the U-Net row-tile convolution (UN_TRACE build through PF_LIB): one un_conv3x3 of
the given shape, then the per-CTA cycle sums of the MMA warp (full wait / acce wait / issue), the
producer (empty wait / copy issue) and epilogue warp 0 (accf wait / drain), per iteration.
    PF_LIB=.../libpf_untrace.so python tools/unet_trace.py B H W cin cout"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_2312_05410_b200 import pf, unet
    B, H, W, cin, cout = map(int, sys.argv[1:6])
    x = torch.randn(B, H, W, cin).to(torch.bfloat16).cuda()
    w = (torch.randn(cout, 3, 3, cin) / 12).to(torch.bfloat16).cuda()
    out = torch.empty(B, H, W, cout, device="cuda")
    buf = np.zeros((160 * 12,), dtype=np.uint64)
    f = pf.lib().un_debug_trace
    for it in range(3):
        f(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1)
        unet.conv3x3(x.data_ptr(), w.data_ptr(), out.data_ptr(), B, H, W, cin, cout)
        torch.cuda.synchronize()
    f(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1)
    span = buf[160 * 8:].reshape(160, 4).astype(np.int64)
    buf = buf[:160 * 8].reshape(160, 8)
    used = buf[:, 7] > 0
    per = buf[used, :7].astype(np.float64) / buf[used, 7:8].astype(np.float64)
    names = ["mma_full_wait", "mma_acce_wait", "mma_issue", "prod_empty_wait", "prod_issue", "epi_accf_wait",
             "epi_drain"]
    print(json.dumps(dict(shape=[B, H, W, cin, cout], ctas=int(used.sum()), iters_per_cta=float(buf[used, 7].mean()),
                          prologue_cyc=float(np.median(span[used, 1] - span[used, 0])),
                          mma_loop_cyc=float(np.median(span[used, 2] - span[used, 1])),
                          epilogue_tail_cyc=float(np.median(span[used, 3] - span[used, 2])),
                          **{n + "_cyc_per_iter": round(float(per[:, i].mean()), 1) for i, n in enumerate(names)})))


if __name__ == "__main__":
    main()
