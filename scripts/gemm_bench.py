"""Standalone tcgen05 GEMM bandwidth sweep (warm, CUDA events, graph of 20 launches)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_18813_b200 import _native as N
lib = N.load(); N.init_device()
dev = torch.device("cuda:0")
shapes = [("qkv", 12288, 4096), ("o", 4096, 4096), ("gu", 22016, 4096), ("down", 4096, 11008), ("lm", 32000, 4096)]
Ms = [int(x) for x in os.environ.get("GM", "8,32,72").split(",")]
configs = [tuple(int(v) for v in c.split(":")) for c in os.environ.get("GC", "0:0:0,1:0:0,2:0:0,1:16:0,2:6:0").split(",")]
W = {n: (torch.randn(N_, K, device=dev) * 0.02).to(torch.bfloat16) for n, N_, K in shapes}
st = torch.cuda.current_stream().cuda_stream
for M in Ms:
    for cfgt in configs:
        lib.sb_gemm_tune(*cfgt)
        out = []
        tot_b, tot_t = 0, 0
        for n, N_, K in shapes:
            x = torch.randn(M, K, device=dev).to(torch.bfloat16)
            y = torch.zeros(M, N_, device=dev)
            def run():
                N.call("sb_gemm", N.SB_BF16, x.data_ptr(), W[n].data_ptr(), y.data_ptr(), M, N_, K, N.EPI_STORE_F32, N.GEMM_TC, None, 0, torch.cuda.current_stream().cuda_stream)
            run(); torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    for _ in range(20): run()
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); e1.synchronize()
            t = e0.elapsed_time(e1) / 20 * 1e3
            b = N_ * K * 2
            tot_b += b; tot_t += t
            out.append(f"{n}={t:.1f}us/{b/t/1e3:.0f}GB/s")
        print(f"M={M} tune={cfgt}: " + " ".join(out) + f" | sum {tot_t:.1f}us {tot_b/tot_t/1e3:.0f}GB/s", flush=True)
