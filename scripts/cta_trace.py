"""Per-CTA timeline of one graph-replayed 7B verify forward (sb_debug_cta_trace).

For every traced launch (GEMMs and attention, in forward order: per layer qkv, attn, o, gu, down; then
lm_head) prints: first CTA entry, last exit, median time its CTAs waited for the dependency
(griddepcontrol.wait), mainloop span, and the gap between the previous launch's last exit and this
launch's first dependency-resolved CTA.  Usage: python scripts/cta_trace.py [b k ...] [--json out]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2310_18813_b200 import _native as N
from paper_2310_18813_b200.decoder import CONFIGS, Decoder
from paper_2310_18813_b200.presets import example_trace
from paper_2310_18813_b200.spec_engine import SpecEngine, _capture_graph, _stage_context

NAMES = ["qkv", "attn", "o", "gu", "down"]


def main():
    argv = sys.argv[1:]
    out = argv[argv.index("--json") + 1] if "--json" in argv else None
    skip = {i + 1 for i, a in enumerate(argv) if a in ("--json", "--pre", "--flags")}
    args = [a for i, a in enumerate(argv) if not a.startswith("--") and i not in skip]
    cells = [(int(args[i]), int(args[i + 1])) for i in range(0, len(args), 2)] or [(8, 3)]
    dev = torch.device("cuda:0")
    tgt = Decoder(CONFIGS["llama-2-7b"], dtype="bf16", device=dev, init="device", max_pos=320)
    drf = Decoder(CONFIGS["llama-68m"], dtype="bf16", device=dev, seed=1, init="device", max_pos=320)
    bmax = max(b for b, _ in cells)
    eng = SpecEngine(tgt, drf, mode="injected", acceptance=example_trace(), max_batch=bmax, max_k=8,
                     prompt_len=128, max_new=128)
    lib = N.load()
    if "--pre" in sys.argv:
        lib.sb_debug_gemm_pdl(int(sys.argv[sys.argv.index("--pre") + 1]), 0, 0)
    if "--flags" in sys.argv:
        lib.sb_debug_gemm_pdl(0, 0, int(sys.argv[sys.argv.index("--flags") + 1]))
    if "--nopdl" in sys.argv:
        lib.sb_set_pdl(0)
    buf = torch.zeros(8 + 8 * 400000, dtype=torch.int64, device=dev)
    report = {}
    raws = {}
    for b, k in cells:
        plain = (eng.time_draft_step(b, ctx=192, reps=20) if "--draft" in sys.argv else
                 0.0 if "--prefill" in sys.argv else eng.time_verify(b, k, ctx=192, reps=20))
        if "--prefill" not in sys.argv:
            _stage_context(eng, b, k, 192)
        lib.sb_debug_cta_trace(N.ptr(buf))
        if "--prefill" in sys.argv:  # a prefill chunk: b prompts of k tokens (positions 0..k-1)
            i32 = dict(device=dev, dtype=torch.int32)
            pids = torch.randint(0, 32000, (b * k,), **i32)
            ppos = torch.arange(k, **i32).repeat(b)
            pws = torch.zeros(tgt.workspace_bytes(b * k), device=dev, dtype=torch.uint8)
            fn = lambda: eng.target.forward(eng.kv_t, pids, eng.slots, ppos, b, k, None, N.LOGITS_NONE, pws)
        elif "--draft" in sys.argv:  # one draft decode step (b sequences x 1 token, greedy sink) instead
            sink = N.SbTokenSink(None, 0, eng.ds_ids.data_ptr(), None, None, 0)

            def fn():
                st = torch.cuda.current_stream(eng.dev).cuda_stream
                eng.draft.forward_greedy(eng.kv_d, eng.ds_ids, eng.slots, eng.ds_pos, b, 1, None, N.LOGITS_LAST,
                                         eng.workspace, sink, st)
        else:
            fn = lambda: eng.target.forward(eng.kv_t, eng.v_ids, eng.slots, eng.v_pos, b, k + 1, eng.t_logits,
                                            N.LOGITS_ALL, eng.workspace)
        g = _capture_graph(fn, eng.stream)
        lib.sb_debug_cta_trace(None)
        with torch.cuda.stream(eng.stream):
            for _ in range(3):
                buf.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                e1.synchronize()
        traced_ms = e0.elapsed_time(e1)
        n = int(buf[0].item())
        raw = buf[8:8 + 8 * n].view(n, 8).cpu().numpy().astype(np.int64)
        # columns: id, kind, smid, block, t_entry, t_dep, t_first, t_main, t_exit (us from the first entry)
        t0 = raw[:, 2].min()
        rec = np.zeros((n, 9))  # (+ column 9: sub-phase stamp)
        rec[:, 0] = raw[:, 0] & 0xffffffff
        rec[:, 1] = (raw[:, 0] >> 32) & 0xff
        rec[:, 2] = raw[:, 0] >> 40
        rec[:, 3] = raw[:, 1]
        rec[:, 4:9] = (raw[:, 2:7] - t0) / 1e3
        sub = np.where(raw[:, 7] > 0, (raw[:, 7] - t0) / 1e3, np.nan)  # kernel sub-phase stamp (if any)
        rec = np.concatenate([rec, sub[:, None]], axis=1)
        raws[f"b{b}k{k}"] = rec
        ids = sorted(set(rec[:, 0].astype(int).tolist()))
        rows = []
        prev_exit = None
        for i in ids:
            r = rec[rec[:, 0] == i]
            kind = int(r[0, 1])
            ent, dep, first, main, ext = (r[:, c] for c in range(4, 9))
            layer, j = divmod(i, 5)
            nl = drf.cfg.n_layers if "--draft" in sys.argv else tgt.cfg.n_layers
            name = f"L{layer}.{NAMES[j]}" if layer < nl else "lm_head"
            row = dict(id=i, name=name, kind=kind, ctas=len(r), sms=len(set(r[:, 2].tolist())),
                       entry_first=float(ent.min()), entry_last=float(ent.max()), dep_first=float(dep.min()),
                       dep_med=float(np.median(dep)), first_med=float(np.median(first)),
                       main_med=float(np.median(main)), main_last=float(main.max()),
                       exit_first=float(ext.min()), exit_med=float(np.median(ext)), exit_last=float(ext.max()),
                       epi_med=float(np.median(ext - main)), epi_max=float((ext - main).max()),
                       main_dur_med=float(np.median(main - dep)))
            row["gap_dep"] = None if prev_exit is None else row["dep_first"] - prev_exit
            prev_exit = row["exit_last"]
            rows.append(row)
        print(f"b={b} k={k}: untraced {plain:.3f} ms, traced replay {traced_ms:.3f} ms, {n} CTA records, "
              f"{len(ids)} launches")
        print(f"{'launch':10s} {'ctas':>5s} {'sms':>4s} {'entry0':>8s} {'entryN':>8s} {'dep0':>8s} {'gap':>6s} "
              f"{'first':>8s} {'mainMed':>8s} {'mainN':>8s} {'exitMed':>8s} {'exitN':>8s} {'epiMed':>6s} {'epiMax':>6s}")
        for r in rows:
            if "--draft" in sys.argv or r["id"] < 10 or r["id"] >= len(ids) - 6 or r["id"] // 5 == 16:
                g_ = "" if r["gap_dep"] is None else f"{r['gap_dep']:6.2f}"
                print(f"{r['name']:10s} {r['ctas']:5d} {r['sms']:4d} {r['entry_first']:8.2f} {r['entry_last']:8.2f} "
                      f"{r['dep_first']:8.2f} {g_:>6s} {r['first_med']:8.2f} {r['main_med']:8.2f} {r['main_last']:8.2f} "
                      f"{r['exit_med']:8.2f} {r['exit_last']:8.2f} {r['epi_med']:6.2f} {r['epi_max']:6.2f}")
        agg = {}
        for r in rows:
            if r["name"] == "lm_head":
                continue
            layer = r["id"] // 5
            if ("--draft" in sys.argv and layer < drf.cfg.n_layers) or 2 <= layer < tgt.cfg.n_layers - 2:
                a = agg.setdefault(NAMES[r["id"] % 5], [])
                a.append((r["gap_dep"], r["dep_first"] - r["entry_first"], r["main_last"] - r["dep_first"],
                          r["exit_last"] - r["main_last"], r["epi_med"], r["exit_last"] - r["dep_first"]))
        print("per-layer class means (middle layers): gap(prev exitN->dep0) | entry0->dep0 | dep0->mainN | "
              "mainN->exitN | epilogue median | dep0->exitN")
        tot = 0.0
        for nm in NAMES:
            v = np.array(agg[nm], dtype=float).mean(0)
            tot += v[0] + v[5]
            print(f"  {nm:5s} " + " | ".join(f"{x:6.2f}" for x in v))
        print(f"  per layer {tot:.2f} us")
        report[f"b{b}k{k}"] = dict(untraced_ms=plain, traced_ms=traced_ms, launches=rows)
    if out:
        with open(out, "w") as f:
            json.dump(report, f)
        np.savez_compressed(out.replace(".json", "") + "_raw.npz", **raws)


if __name__ == "__main__":
    main()
