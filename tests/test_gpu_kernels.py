"""GPU parity of the token-level kernels (K4 accept, K5 commit, staging, sampling)
and of the GEMMs, through the C-ABI, against the CPU oracle / torch fp32."""

import ctypes
import numpy as np
import pytest
import torch

from oracle import spec_ref
from paper_2310_18813_b200 import _native as N
from sbtest_util import load_golden

pytestmark = pytest.mark.gpu


def _st():
    return torch.cuda.current_stream().cuda_stream


def _i32(a, dev):
    return torch.as_tensor(np.asarray(a, dtype=np.int32), device=dev)


# ----------------------------------------------------------------- GEMM (K2)
GEMM_SHAPES = [(1, 128, 512), (2, 256, 768), (9, 4096, 4096), (18, 2752, 512), (72, 12288, 4096),
               (40, 32000, 768), (130, 1536, 512), (300, 384, 1376), (16, 22016, 4096), (8, 4096, 11008)]


@pytest.mark.parametrize("M,N_,K", GEMM_SHAPES)
def test_gemm_tcgen05_matches_fp32_reference(cuda_dev, M, N_, K):
    g = torch.Generator(device=cuda_dev).manual_seed(M * 7 + N_ + K)
    x = (torch.randn(M, K, generator=g, device=cuda_dev) * 0.5).to(torch.bfloat16)
    w = (torch.randn(N_, K, generator=g, device=cuda_dev) * 0.02).to(torch.bfloat16)
    ref = x.float() @ w.float().T
    ws = torch.zeros(int(N.load().sb_gemm_workspace_bytes(M, N_, K)), device=cuda_dev, dtype=torch.uint8)
    for backend in (N.GEMM_TC, N.GEMM_SIMT):
        y = torch.zeros(M, N_, device=cuda_dev)
        N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, N_, K, N.EPI_STORE_F32, backend,
               ws.data_ptr(), ws.numel(), _st())
        torch.cuda.synchronize()
        err = (y - ref).abs().max().item()
        scale = ref.abs().max().item()
        assert err <= 1e-4 * scale + 1e-5, (backend, err, scale)
        if backend == N.GEMM_TC:
            y2 = torch.zeros_like(y)
            N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y2.data_ptr(), M, N_, K, N.EPI_STORE_F32,
                   backend, ws.data_ptr(), ws.numel(), _st())
            assert torch.equal(y, y2), "tcgen05 stream-K GEMM must be deterministic"


@pytest.mark.parametrize("M,N_,K", [(9, 4096, 4096), (72, 22016, 4096), (3, 2752, 512)])
def test_gemm_epilogues(cuda_dev, M, N_, K):
    g = torch.Generator(device=cuda_dev).manual_seed(5)
    x = (torch.randn(M, K, generator=g, device=cuda_dev) * 0.5).to(torch.bfloat16)
    w = (torch.randn(N_, K, generator=g, device=cuda_dev) * 0.02).to(torch.bfloat16)
    ref = x.float() @ w.float().T
    ws = torch.zeros(int(N.load().sb_gemm_workspace_bytes(M, N_, K)), device=cuda_dev, dtype=torch.uint8)
    for backend in (N.GEMM_TC, N.GEMM_SIMT):
        # residual add
        base = torch.randn(M, N_, generator=g, device=cuda_dev)
        y = base.clone()
        N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, N_, K, N.EPI_RESID_ADD, backend,
               ws.data_ptr(), ws.numel(), _st())
        torch.cuda.synchronize()
        assert (y - (base + ref)).abs().max().item() < 1e-3
        # bf16 store
        yb = torch.zeros(M, N_, device=cuda_dev, dtype=torch.bfloat16)
        N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), yb.data_ptr(), M, N_, K, N.EPI_STORE, backend,
               ws.data_ptr(), ws.numel(), _st())
        torch.cuda.synchronize()
        assert (yb.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
        # silu(gate) * up on interleaved rows
        ya = torch.zeros(M, N_ // 2, device=cuda_dev, dtype=torch.bfloat16)
        N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), ya.data_ptr(), M, N_, K, N.EPI_SILU_MUL, backend,
               ws.data_ptr(), ws.numel(), _st())
        torch.cuda.synchronize()
        want = torch.nn.functional.silu(ref[:, 0::2]) * ref[:, 1::2]
        assert (ya.float() - want).abs().max().item() <= 1e-2 * want.abs().max().item() + 1e-4


def test_gemm_fp32_simt(cuda_dev):
    g = torch.Generator(device=cuda_dev).manual_seed(3)
    for M, N_, K in [(5, 1536, 512), (33, 2752, 512), (1, 32000, 512)]:
        x = torch.randn(M, K, generator=g, device=cuda_dev)
        w = torch.randn(N_, K, generator=g, device=cuda_dev) * 0.02
        y = torch.zeros(M, N_, device=cuda_dev)
        N.call("sb_gemm", N.SB_F32, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, N_, K, N.EPI_STORE_F32, N.GEMM_AUTO,
               None, 0, _st())
        ref = (x.double() @ w.double().T).float()
        torch.cuda.synchronize()
        assert (y - ref).abs().max().item() < 1e-4
        # batch invariance: row 0 alone == row 0 in the batch, bit for bit
        y1 = torch.zeros(1, N_, device=cuda_dev)
        N.call("sb_gemm", N.SB_F32, x.data_ptr(), w.data_ptr(), y1.data_ptr(), 1, N_, K, N.EPI_STORE_F32,
               N.GEMM_AUTO, None, 0, _st())
        torch.cuda.synchronize()
        assert torch.equal(y1[0], y[0])


# ----------------------------------------------------------------- K4/K5 on the reference's own KATs
def _spiky_logits(targets, V, gen, dev):
    """fp32 logits whose argmax is exactly `targets` (noise + a spike)."""
    t = torch.as_tensor(np.asarray(targets, dtype=np.int64), device=dev)
    lg = torch.randn(*t.shape, V, generator=gen, device=dev)
    lg.scatter_(-1, t.unsqueeze(-1), 10.0)
    return lg


def test_accept_commit_reproduce_reference_tokenlevel(cuda_dev):
    """Drive sb_prepare/sb_accept/sb_kv_commit with the drafts the reference
    TokenLevel produced and logits whose argmax is the reference target stream:
    accepted lengths, advances and final token streams equal the reference."""
    V = 32000
    gen = torch.Generator(device=cuda_dev).manual_seed(0)
    for case in load_golden("tokenlevel.json"):
        b, s = case["b"], case["s"]
        rids = case["request_ids"]
        cap = max(case["target_lens"]) + s + 4
        tokens = torch.zeros(b, cap, dtype=torch.int32, device=cuda_dev)
        tokens[:, 0] = 7  # one "prompt" token
        n_tok = torch.ones(b, dtype=torch.int32, device=cuda_dev)
        produced = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
        target_len = _i32(case["target_lens"], cuda_dev)
        finish = torch.full((b,), -1, dtype=torch.int32, device=cuda_dev)
        it = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
        live = torch.zeros(1, dtype=torch.int32, device=cuda_dev)
        acc = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
        adv = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
        out = torch.zeros(b * (s + 1), dtype=torch.int32, device=cuda_dev)
        v_ids = torch.zeros(b * (s + 1), dtype=torch.int32, device=cuda_dev)
        v_pos = torch.zeros(b * (s + 1), dtype=torch.int32, device=cuda_dev)
        t_tok = torch.zeros(b * (s + 1), dtype=torch.int32, device=cuda_dev)
        for step in case["steps"]:
            drafts = np.zeros((b, s + 1), np.int32)
            targets = np.zeros((b, s + 1), np.int32)
            by_rid = {r["rid"]: r for r in step}
            for i, rid in enumerate(rids):
                if rid in by_rid:
                    drafts[i, 1:] = by_rid[rid]["drafts"]
                    targets[i] = by_rid[rid]["targets"]
            N.call("sb_prepare_iteration", b, s, tokens.data_ptr(), cap, n_tok.data_ptr(), None, None,
                   v_ids.data_ptr(), v_pos.data_ptr(), None, 0, it.data_ptr(), None, 64, None, 0, None, _st())
            v_ids.view(b, s + 1)[:, 1:] = _i32(drafts[:, 1:], cuda_dev)
            lg = _spiky_logits(targets, V, gen, cuda_dev).reshape(b * (s + 1), V).contiguous()
            N.call("sb_argmax_rows", lg.data_ptr(), b * (s + 1), V, t_tok.data_ptr(), _st())
            N.call("sb_accept", N.ACCEPT_GREEDY, b, s, V, t_tok.data_ptr(), None, None, v_ids.data_ptr() + 4, s + 1,
                   None, None, 64, None, produced.data_ptr(), target_len.data_ptr(), acc.data_ptr(), adv.data_ptr(),
                   out.data_ptr(), _st())
            a_h, d_h = acc.cpu().numpy(), adv.cpu().numpy()
            for i, rid in enumerate(rids):
                if rid in by_rid:
                    assert a_h[i] == by_rid[rid]["accepted"], (case["seed"], rid)
                    assert d_h[i] == by_rid[rid]["advanced"]
                else:
                    assert d_h[i] == 0  # finished rows are masked
            N.call("sb_kv_commit", b, s, adv.data_ptr(), acc.data_ptr(), out.data_ptr(), tokens.data_ptr(), cap,
                   n_tok.data_ptr(), produced.data_ptr(), target_len.data_ptr(), finish.data_ptr(), it.data_ptr(),
                   live.data_ptr(), None, 0, _st())
        assert int(live.item()) == 0
        assert int(it.item()) == case["result"]["steps"]
        toks = tokens.cpu().numpy()
        for i, rid in enumerate(rids):
            n = case["target_lens"][i]
            assert toks[i, 1:1 + n].tolist() == case["tokens"][str(rid)]


def test_prepare_uniforms_and_injection_match_oracle(cuda_dev):
    b, k, cap = 5, 4, 32
    gen = np.random.default_rng(3)
    toks = gen.integers(0, 32000, size=(b, cap)).astype(np.int32)
    n_tok = np.array([1, 2, 9, 17, 30], np.int32)
    samples = list(range(0, 13))
    T = _i32(toks, cuda_dev)
    nt = _i32(n_tok, cuda_dev)
    it = _i32([5], cuda_dev)
    d1i, d1p = torch.zeros(2 * b, dtype=torch.int32, device=cuda_dev), torch.zeros(2 * b, dtype=torch.int32,
                                                                                  device=cuda_dev)
    vi, vp = (torch.zeros(b * (k + 1), dtype=torch.int32, device=cuda_dev) for _ in range(2))
    base = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
    u = torch.zeros(b * 64, device=cuda_dev)
    inj = _i32(samples, cuda_dev)
    linj = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
    N.call("sb_prepare_iteration", b, k, T.data_ptr(), cap, nt.data_ptr(), d1i.data_ptr(), d1p.data_ptr(),
           vi.data_ptr(), vp.data_ptr(), base.data_ptr(), 99, it.data_ptr(), u.data_ptr(), 64, inj.data_ptr(),
           len(samples), linj.data_ptr(), _st())
    torch.cuda.synchronize()
    e_d1i, e_d1p, e_vi, e_vp = spec_ref.prepare_batch(k, toks, n_tok)
    assert np.array_equal(d1i.cpu().numpy().reshape(b, 2), e_d1i)
    assert np.array_equal(d1p.cpu().numpy().reshape(b, 2), e_d1p)
    assert np.array_equal(vi.cpu().numpy().reshape(b, k + 1)[:, 0], e_vi[:, 0])
    assert np.array_equal(vp.cpu().numpy().reshape(b, k + 1), e_vp)
    assert np.array_equal(u.cpu().numpy().reshape(b, 64), spec_ref.uniforms(99, 5, b))
    assert np.array_equal(linj.cpu().numpy(), spec_ref.injected_lengths(99, 5, b, samples))


def test_select_and_accept_stochastic_bit_exact(cuda_dev):
    """Speculative sampling: GPU decisions == oracle decisions on identical
    probabilities and uniforms (canonical fp64 inverse CDF)."""
    V = 32000
    g = torch.Generator(device=cuda_dev).manual_seed(11)
    for b, k, temp in [(4, 3, 1.0), (8, 8, 0.3), (3, 1, 3.0), (2, 0, 1.0), (6, 5, 0.05)]:
        ql = torch.randn(max(1, b * k), V, generator=g, device=cuda_dev) / temp
        pl = torch.randn(b * (k + 1), V, generator=g, device=cuda_dev) / temp
        if k > 0:  # correlate p with q so acceptances happen
            pl.view(b, k + 1, V)[:, :k] = 0.7 * pl.view(b, k + 1, V)[:, :k] + ql.view(b, k, V)
        u = torch.rand(b * 64, generator=g, device=cuda_dev)
        q = torch.zeros_like(ql)
        draft = torch.zeros(b * (k + 1), dtype=torch.int32, device=cuda_dev)
        base = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
        nid = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
        npos = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
        for j in range(1, k + 1):
            rows = ql.view(b, k, V)[:, j - 1].contiguous()
            N.call("sb_select_tokens", rows.data_ptr(), b, V, N.SELECT_SAMPLE, u.data_ptr() + (j - 1) * 4, 64,
                   q.data_ptr() + (j - 1) * V * 4, k * V, draft.data_ptr() + j * 4, k + 1, nid.data_ptr(),
                   npos.data_ptr(), base.data_ptr(), j, _st())
        p = torch.empty_like(pl)
        N.call("sb_softmax_rows", pl.data_ptr(), b * (k + 1), V, p.data_ptr(), _st())
        produced = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
        tlen = torch.full((b,), 100, dtype=torch.int32, device=cuda_dev)
        acc = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
        adv = torch.zeros(b, dtype=torch.int32, device=cuda_dev)
        out = torch.zeros(b * (k + 1), dtype=torch.int32, device=cuda_dev)
        N.call("sb_accept", N.ACCEPT_STOCHASTIC, b, k, V, None, p.data_ptr(), q.data_ptr() if k else None,
               draft.data_ptr() + 4, k + 1, u.data_ptr() + k * 4, u.data_ptr() + 2 * k * 4, 64, None,
               produced.data_ptr(), tlen.data_ptr(), acc.data_ptr(), adv.data_ptr(), out.data_ptr(), _st())
        torch.cuda.synchronize()
        qh = q.cpu().numpy().reshape(b, max(k, 1), V)[:, :k] if k else None
        ph = p.cpu().numpy().reshape(b, k + 1, V)
        uh = u.cpu().numpy().reshape(b, 64)
        dh = draft.cpu().numpy().reshape(b, k + 1)[:, 1:]
        # the draft sampler itself
        for s in range(b):
            for j in range(k):
                assert dh[s, j] == spec_ref.inverse_cdf(qh[s, j], uh[s, j])
            ref_soft = spec_ref.softmax_rows(pl.cpu().numpy().reshape(b, k + 1, V)[s])
            assert np.abs(ref_soft - ph[s]).max() < 1e-6
        ea, ed, eo = spec_ref.accept_batch("stochastic", k, dh, np.zeros(b), np.full(b, 100), p=ph, q=qh,
                                           u_acc=uh[:, k:2 * k], u_res=uh[:, 2 * k])
        assert np.array_equal(acc.cpu().numpy(), ea)
        assert np.array_equal(adv.cpu().numpy(), ed)
        assert np.array_equal(out.cpu().numpy().reshape(b, k + 1), eo)


def test_argmax_ties_lowest_index(cuda_dev):
    V = 32000
    lg = torch.zeros(3, V, device=cuda_dev)
    lg[0, 5] = lg[0, 17] = 2.0
    lg[1, V - 1] = 1.0
    lg[2] = -1.0  # all equal -> index 0
    out = torch.zeros(3, dtype=torch.int32, device=cuda_dev)
    N.call("sb_argmax_rows", lg.data_ptr(), 3, V, out.data_ptr(), _st())
    assert out.cpu().tolist() == [5, V - 1, 0]


def test_kv_commit_masks_finished_and_logs(cuda_dev):
    b, k, cap = 3, 2, 16
    tokens = torch.zeros(b, cap, dtype=torch.int32, device=cuda_dev)
    n_tok = _i32([4, 4, 4], cuda_dev)
    produced = _i32([0, 5, 3], cuda_dev)
    tlen = _i32([10, 5, 4], cuda_dev)
    adv = _i32([3, 0, 1], cuda_dev)
    acc = _i32([2, 2, 0], cuda_dev)
    out = _i32([[11, 12, 13], [21, 22, 23], [31, -1, -1]], cuda_dev).reshape(-1)
    fin = _i32([-1, 2, -1], cuda_dev)
    it = _i32([4], cuda_dev)
    live = _i32([0], cuda_dev)
    log = torch.full((8, b), -7, dtype=torch.int32, device=cuda_dev)
    N.call("sb_kv_commit", b, k, adv.data_ptr(), acc.data_ptr(), out.data_ptr(), tokens.data_ptr(), cap,
           n_tok.data_ptr(), produced.data_ptr(), tlen.data_ptr(), fin.data_ptr(), it.data_ptr(), live.data_ptr(),
           log.data_ptr(), 8, _st())
    torch.cuda.synchronize()
    assert n_tok.cpu().tolist() == [7, 4, 5]
    assert produced.cpu().tolist() == [3, 5, 4]
    assert tokens.cpu().numpy()[0, 4:7].tolist() == [11, 12, 13]
    assert tokens.cpu().numpy()[2, 4] == 31
    assert fin.cpu().tolist() == [-1, 2, 5]
    assert it.item() == 5 and live.item() == 1
    assert log.cpu().numpy()[4].tolist() == [2, -1, 0]


def test_gemm_sequence_shares_workspace(cuda_dev):
    """Regression: GEMMs of different tile counts share one workspace (as in a
    forward); stream-K counters must survive other GEMMs' partial slots."""
    shapes = [(63, 1536, 512), (63, 512, 512), (63, 2752, 512), (63, 512, 1376), (63, 32000, 512)] * 3
    ws = torch.zeros(int(N.load().sb_gemm_workspace_bytes(63, 32000, 1376)), device=cuda_dev, dtype=torch.uint8)
    g = torch.Generator(device=cuda_dev).manual_seed(1)
    for M, N_, K in shapes:
        x = (torch.randn(M, K, generator=g, device=cuda_dev) * 0.5).to(torch.bfloat16)
        w = (torch.randn(N_, K, generator=g, device=cuda_dev) * 0.02).to(torch.bfloat16)
        y = torch.zeros(M, N_, device=cuda_dev)
        N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, N_, K, N.EPI_STORE_F32, N.GEMM_TC,
               ws.data_ptr(), ws.numel(), _st())
        ref = x.float() @ w.float().T
        torch.cuda.synchronize()
        assert (y - ref).abs().max().item() <= 1e-4 * ref.abs().max().item() + 1e-5, (M, N_, K)


@pytest.mark.parametrize("M", [1, 8, 32, 72])
def test_fused_lm_head_argmax_matches_full_argmax(cuda_dev, M):
    """The greedy token sink (argmax in the lm_head tcgen05 epilogue) equals a
    full argmax over the logits the same GEMM produces, ties -> lowest index."""
    from paper_2310_18813_b200.decoder import CONFIGS, Decoder
    import ctypes as C

    tgt = Decoder(CONFIGS["tiny-target"], dtype="bf16", device=cuda_dev, seed=5, init="host", max_pos=256)
    kv = tgt.new_kv(M, 64)
    ws = torch.zeros(tgt.workspace_bytes(M), device=cuda_dev, dtype=torch.uint8)
    ids = torch.randint(0, 32000, (M,), device=cuda_dev, dtype=torch.int32)
    slots = torch.arange(M, dtype=torch.int32, device=cuda_dev)
    pos = torch.zeros(M, dtype=torch.int32, device=cuda_dev)
    logits = torch.zeros(M, 32000, device=cuda_dev)
    tgt.forward(kv, ids, slots, pos, M, 1, logits, N.LOGITS_ALL, ws)
    tok = torch.full((M,), -1, dtype=torch.int32, device=cuda_dev)
    logits2 = torch.zeros_like(logits)
    sink = N.SbTokenSink(tok.data_ptr(), 1, None, None, None, 0)
    tgt.forward_greedy(kv, ids, slots, pos, M, 1, logits2, N.LOGITS_ALL, ws, sink)
    torch.cuda.synchronize()
    assert torch.equal(logits, logits2)
    assert np.array_equal(tok.cpu().numpy(), spec_ref.argmax_rows(logits.cpu().numpy()))
    tok2 = torch.full((M,), -1, dtype=torch.int32, device=cuda_dev)
    sink2 = N.SbTokenSink(tok2.data_ptr(), 1, None, None, None, 0)
    tgt.forward_greedy(kv, ids, slots, pos, M, 1, None, N.LOGITS_ALL, ws, sink2)  # logits not materialised
    torch.cuda.synchronize()
    assert torch.equal(tok, tok2)


@pytest.mark.parametrize("splits", [3, 5, 6, 7])
def test_gemm_uneven_cluster_splits(cuda_dev, splits):
    """Cluster split-K with split counts that do not divide the 128-row tile
    (row pairs per rank: uneven ranges): residual + norm partials, silu*up."""
    lib = N.load()
    M, N_, K = 20, 2048, 4096
    g = torch.Generator(device=cuda_dev).manual_seed(splits)
    x = (torch.randn(M, K, generator=g, device=cuda_dev) * 0.5).to(torch.bfloat16)
    w = (torch.randn(N_, K, generator=g, device=cuda_dev) * 0.02).to(torch.bfloat16)
    ref = x.float() @ w.float().T
    lib.sb_gemm_tune(0, 0, splits)
    try:
        base = torch.randn(M, N_, generator=g, device=cuda_dev)
        y = base.clone()
        N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, N_, K, N.EPI_RESID_ADD,
               N.GEMM_TC, None, 0, _st())
        ya = torch.zeros(M, N_ // 2, device=cuda_dev, dtype=torch.bfloat16)
        N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), ya.data_ptr(), M, N_, K, N.EPI_SILU_MUL,
               N.GEMM_TC, None, 0, _st())
        torch.cuda.synchronize()
    finally:
        lib.sb_gemm_tune(0, 0, 0)
    assert (y - (base + ref)).abs().max().item() < 1e-3
    want = torch.nn.functional.silu(ref[:, 0::2]) * ref[:, 1::2]
    assert (ya.float() - want).abs().max().item() <= 1e-2 * want.abs().max().item() + 1e-4


@pytest.mark.parametrize("M,N_,K,cps,splits,wt,tn", [
    (1016, 4096, 4096, 2, 1, 1, 192),   # ragged last token tile
    (1016, 12288, 4096, 1, 1, 2, 128),  # dual weight tiles on a narrow token tile
    (300, 4096, 11008, 2, 2, 1, 128),   # cluster split-K with a narrow token tile
    (257, 1536, 512, 1, 1, 1, 192),
])
def test_gemm_tuned_token_tile(cuda_dev, M, N_, K, cps, splits, wt, tn):
    """A tuned entry may narrow the token tile (wave quantisation of the
    compute-bound regime, sb_gemm_tune_set): results are the same GEMM."""
    g = torch.Generator(device=cuda_dev).manual_seed(M + N_ + K + tn)
    x = (torch.randn(M, K, generator=g, device=cuda_dev) * 0.5).to(torch.bfloat16)
    w = (torch.randn(N_, K, generator=g, device=cuda_dev) * 0.02).to(torch.bfloat16)
    ref = x.float() @ w.float().T
    lib = N.load()
    ws = torch.zeros(int(lib.sb_gemm_workspace_bytes(M, N_, K)), device=cuda_dev, dtype=torch.uint8)
    N.call("sb_gemm_tune_set", M, N_, K, cps, splits, wt, tn)
    try:
        got = [ctypes.c_int32() for _ in range(4)]
        N.call("sb_gemm_tune_get", M, N_, K, *[ctypes.byref(v) for v in got])
        assert [v.value for v in got] == [cps, splits, wt, tn]
        y = torch.zeros(M, N_, device=cuda_dev)
        N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, N_, K, N.EPI_STORE_F32, N.GEMM_TC,
               ws.data_ptr(), ws.numel(), _st())
        torch.cuda.synchronize()
    finally:
        lib.sb_gemm_autotune_clear()
    err = (y - ref).abs().max().item()
    assert err <= 1e-4 * ref.abs().max().item() + 1e-5, err


@pytest.mark.parametrize("M,N_,K", [(1, 2304, 768), (8, 768, 3072), (13, 6144, 768), (16, 512, 512), (5, 768, 768),
                                   (9, 6144, 768)])
def test_gemm_small_token_kernel(cuda_dev, M, N_, K):
    """The draft step's small-token mma.sync GEMM (backend 3) against the fp32 product: bf16 store,
    residual add and silu(gate)*up, both token count classes (1 or 2 n-tiles of 8 tokens), 16- and
    32-row CTAs (gate/up at N=6144)."""
    g = torch.Generator(device=cuda_dev).manual_seed(M * 31 + N_ + K)
    x = (torch.randn(M, K, generator=g, device=cuda_dev) * 0.5).to(torch.bfloat16)
    w = (torch.randn(N_, K, generator=g, device=cuda_dev) * 0.02).to(torch.bfloat16)
    ref = x.float() @ w.float().T
    base = torch.randn(M, N_, generator=g, device=cuda_dev)
    y = base.clone()
    N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, N_, K, N.EPI_RESID_ADD, N.GEMM_SMALL,
           None, 0, _st())
    torch.cuda.synchronize()
    assert (y - (base + ref)).abs().max().item() <= 1e-4 * ref.abs().max().item() + 1e-5
    yb = torch.zeros(M, N_, device=cuda_dev, dtype=torch.bfloat16)
    N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), yb.data_ptr(), M, N_, K, N.EPI_STORE, N.GEMM_SMALL,
           None, 0, _st())
    torch.cuda.synchronize()
    assert (yb.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()
    ya = torch.zeros(M, N_ // 2, device=cuda_dev, dtype=torch.bfloat16)
    N.call("sb_gemm", N.SB_BF16, x.data_ptr(), w.data_ptr(), ya.data_ptr(), M, N_, K, N.EPI_SILU_MUL, N.GEMM_SMALL,
           None, 0, _st())
    torch.cuda.synchronize()
    want = torch.nn.functional.silu(ref[:, 0::2]) * ref[:, 1::2]
    assert (ya.float() - want).abs().max().item() <= 1e-2 * want.abs().max().item() + 1e-4
    # outside the envelope: refused, not silently wrong
    assert N.load().sb_gemm(N.SB_BF16, x.data_ptr(), w.data_ptr(), y.data_ptr(), M, N_, K, N.EPI_STORE_F32,
                            N.GEMM_SMALL, None, 0, _st()) == N.SB_EUNSUPPORTED
