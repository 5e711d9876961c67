"""Worker of the TP=2-on-one-GPU parity test (tests/test_gpu_tp.py): two
processes share cuda:0 and exchange through gloo (HostTP callbacks)."""

import os

import numpy as np
import torch
import torch.distributed as dist


def run(rank, world, port, dtype, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_18813_b200 import _native as N
        from paper_2310_18813_b200.decoder import CONFIGS, Decoder
        from paper_2310_18813_b200.engine import SequenceState
        from paper_2310_18813_b200.spec_engine import SpecEngine
        from paper_2310_18813_b200.tp import HostTP, shard_decoder

        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        full = Decoder(CONFIGS["tiny-target"], dtype=dtype, device=dev, seed=4, init="host", max_pos=256)
        shard = shard_decoder(full, world, rank)
        tp = HostTP()
        tp.attach(shard)
        b, P, k = 3, 10, 3
        rng = np.random.default_rng(0)
        ids = torch.as_tensor(rng.integers(0, 32000, size=b * P).astype(np.int32), device=dev)
        pos = torch.arange(P, dtype=torch.int32, device=dev).repeat(b)
        slots = torch.arange(b, dtype=torch.int32, device=dev)
        res = {}
        for name, dec in (("full", full), ("tp", shard)):
            kv = dec.new_kv(b, 64)
            ws = torch.zeros(dec.workspace_bytes(b * P), device=dev, dtype=torch.uint8)
            tp.register(ws)
            lg = torch.zeros(b * P, 32000, device=dev)
            dec.forward(kv, ids, slots, pos, b, P, lg, N.LOGITS_ALL, ws)
            torch.cuda.synchronize()
            res[name] = lg.cpu()
        scale = res["full"].abs().max().item()
        logit_err = (res["full"] - res["tp"]).abs().max().item() / scale
        # greedy sink through the vocab-parallel reduction ((max, global index) pairs across ranks)
        # == argmax of the same shard's gathered logits, exactly
        kv = shard.new_kv(b, 64)
        ws = torch.zeros(shard.workspace_bytes(b * P), device=dev, dtype=torch.uint8)
        tp.register(ws)
        sink_tok = torch.full((b * P,), -1, dtype=torch.int32, device=dev)
        sink = N.SbTokenSink(sink_tok.data_ptr(), 1, None, None, None, 0)
        shard.forward_greedy(kv, ids, slots, pos, b, P, None, N.LOGITS_ALL, ws, sink)
        torch.cuda.synchronize()
        sink_match = bool(torch.equal(sink_tok.cpu().long(), res["tp"].argmax(-1)))
        # speculative greedy decoding with the sharded target (replicated draft = target layer 0)
        toks = {}
        for name, tgt in (("full", full), ("tp", shard)):
            drf = Decoder(CONFIGS["tiny-target"], dtype=dtype, device=dev, share_from=full, share_layers=1,
                          max_pos=256)
            eng = SpecEngine(tgt, drf, mode="greedy", max_batch=2, max_k=3, prompt_len=8, max_new=10, seed=1,
                             use_graphs=False)
            tp.register(eng.workspace)
            states = [SequenceState(request_id=i, target_len=10) for i in range(2)]
            eng.generate(states, k)
            toks[name] = [list(s.tokens) for s in states]
        out[rank] = (logit_err, toks["full"], toks["tp"], tp.calls, sink_match)
    finally:
        dist.destroy_process_group()
