"""GEMM epilogue phases (per-CTA trace): TMEM -> shared staging vs row emit, at verify token counts.
dbg 2 = staging only (no emit).  Prints per-CTA medians in us."""
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
Ms = [int(v) for v in os.environ.get("MS", "9,32,64,192").split(",")]
for (Nw, K, epi, name) in [(22016, 4096, N.EPI_SILU_MUL, "silu"), (4096, 4096, N.EPI_RESID_ADD, "resid"),
                           (12288, 4096, N.EPI_STORE, "bf16")]:
    w = (torch.randn(Nw, K, device=dev) * 0.02).to(torch.bfloat16)
    for M in Ms:
        x = torch.randn(M, K, device=dev).to(torch.bfloat16)
        ycols = Nw // 2 if epi == N.EPI_SILU_MUL else Nw
        y = torch.zeros(M, ycols, device=dev, dtype=torch.bfloat16 if epi != N.EPI_RESID_ADD else torch.float32)
        for dbg in (0, 2):
            lib.sb_debug_gemm_pdl(0, 0, dbg)
            for _ in range(3):
                N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, Nw, K, epi, N.GEMM_TC, None, 0, st)
            buf.zero_()
            lib.sb_debug_cta_trace(N.ptr(buf))
            N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, Nw, K, epi, N.GEMM_TC, None, 0, st)
            lib.sb_debug_cta_trace(None)
            torch.cuda.synchronize()
            n = int(buf[0].item())
            raw = buf[8:8 + 8 * n].view(n, 8).cpu().numpy().astype(np.int64)
            t0 = raw[:, 2].min()
            t = (raw[:, 2:7] - t0) / 1e3
            stg = np.where(raw[:, 7] > 0, (raw[:, 7] - t0) / 1e3 - t[:, 3], np.nan)
            epi_d = t[:, 4] - t[:, 3]
            print(f"{name:5s} N={Nw} M={M:4d} dbg={dbg}: ctas {n} main {np.median(t[:,3]-t[:,1]):6.2f} "
                  f"stage1 {np.nanmedian(stg):5.2f} epi med {np.median(epi_d):5.2f} p90 {np.percentile(epi_d,90):5.2f} "
                  f"total {t[:,4].max():6.2f}", flush=True)
lib.sb_debug_gemm_pdl(0, 0, 0)
