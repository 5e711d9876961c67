"""Standalone tcgen05 GEMM epilogue timing (per-CTA trace): Y = X W^T at decode token counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2310_18813_b200 import _native as N
dev = torch.device("cuda:0")
lib = N.load()
lib.sb_init()
buf = torch.zeros(8 + 8 * 100000, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream().cuda_stream
for (Nw, K) in [(22016, 4096)]:
    w = (torch.randn(Nw, K, device=dev) * 0.02).to(torch.bfloat16)
    for M in (9, 32, 72):
        x = torch.randn(M, K, device=dev).to(torch.bfloat16)
        for epi, name in [(N.EPI_STORE_F32, "f32")]:
            if epi == 3 and Nw % 2: continue
            y = torch.zeros(M, Nw, device=dev)
            for dbg in (0, 1, 128):
                lib.sb_debug_gemm_pdl(0, 0, dbg)
                for _ in range(3):
                    N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, Nw, K, epi, N.GEMM_TC, None, 0, st)
                buf.zero_()
                lib.sb_debug_cta_trace(N.ptr(buf))
                N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, Nw, K, epi, N.GEMM_TC, None, 0, st)
                lib.sb_debug_cta_trace(None)
                torch.cuda.synchronize()
                if dbg != 1:
                    ref = x.float() @ w.float().T
                    err = (y - ref).abs().max().item()
                    assert err < 1e-2, (M, dbg, err)
                n = int(buf[0].item())
                raw = buf[8:8 + 8 * n].view(n, 8).cpu().numpy().astype(np.int64)
                t = (raw[:, 2:7] - raw[:, 2].min()) / 1e3
                epi_d = t[:, 4] - t[:, 3]
                print(f"N={Nw} K={K} M={M} {name:5s} skip_stores={dbg}: ctas {n} main(dep->main) med {np.median(t[:,3]-t[:,1]):6.2f} "
                      f"epi med {np.median(epi_d):5.2f} p90 {np.percentile(epi_d,90):5.2f} total {t[:,4].max():6.2f} us", flush=True)
lib.sb_debug_gemm_pdl(0, 0, 0)
