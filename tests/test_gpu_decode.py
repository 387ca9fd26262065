"""Batched greedy decode (ToyLm::greedy_decode, lm_core.cpp:352-404, over every fork at once).

Bars:
  * copy pointer fires -> the generated ids are forced (answer[t], then EOS): BIT-EXACT vs the
    reference (C1 pipeline: all 64 queries' token lists equal run_batch's; LM goldens);
  * plain greedy: every generated token is checked "teacher-forced" against the fp32 oracle:
    the oracle extends the same context with OUR previous tokens and its argmax must equal our
    token wherever its top-1/top-2 margin exceeds 2 * LOGIT_TOL (bf16 weights/activations make
    closer calls legitimately ambiguous); the reference's own greedy list must agree with ours
    up to its first step whose margin is below that bound;
  * stop rules: EOS, max_new, full context (lm_core.cpp:387-389).
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2505_10951_b200 import host, workload as W

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
LOGIT_TOL = 0.08
EOS = 257


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _cfg(G):
    return {**dict(layers=4, heads=4, model_dim=64, ffn_hidden=256, max_seq_len=1024, seed=3), **G["cfg"]}


def _teacher_forced(olm, prefix, suffix, toks, soft=None):
    """Oracle argmax after prefix + suffix + toks[:k] for every k; returns [(argmax, margin)]."""
    kv = olm.prefill(prefix, soft)
    f = kv.fork()
    lg = olm.extend(f, suffix)
    out = []
    for k in range(len(toks)):
        s = np.sort(lg)
        out.append((int(np.argmax(lg)), float(s[-1] - s[-2])))
        if k + 1 < len(toks):
            lg = olm.extend(f, [int(toks[k])])
    return out


@pytest.mark.parametrize("name", ["lm_tiny.json", "lm_hd64.json", "lm_hd128.json"])
def test_decode_vs_reference_golden(ctx, name):
    G = gold(name)
    cfg = _cfg(G)
    lm = host.ToyLm(ctx, host.ToyLmConfig(**cfg))
    olm = oracle.ToyLm(**{k: cfg[k] for k in ("layers", "heads", "model_dim", "ffn_hidden",
                                              "max_seq_len", "seed")})
    checked = 0
    for case, out in zip(G["cases"], G["out"]):
        if out["status"] or "decode" not in out:
            continue
        n = case["decode"]
        kv = lm.prefill(case["prefix"], case.get("soft"))
        ans = [case["answer"]] if "answer" in case else None
        _, first, gen = lm.extend_generate(kv, [0], [case["suffix"]], ans, max_new=n)
        got = gen[0].tolist()
        ref = out["decode"]
        assert got[0] == first[0]
        if ans:  # copy pointer: forced ids, bit-exact
            assert got == ref, (got, ref)
            checked += len(got)
            continue
        # the reference's list agrees up to its first ambiguous step
        for t, mg in enumerate(out["decode_margins"]):
            if mg <= 2 * LOGIT_TOL or t >= len(ref):
                break
            assert got[t] == ref[t], (t, got, ref)
        # every step teacher-forced against the oracle
        tf = _teacher_forced(olm, case["prefix"], case["suffix"], got, case.get("soft"))
        for t, (am, mg) in enumerate(tf):
            if mg > 2 * LOGIT_TOL:
                assert got[t] == am, (t, got[t], am, mg)
                checked += 1
        # stop rules: EOS ends the list; otherwise exactly n tokens
        assert (got[-1] == EOS and EOS not in got[:-1]) or (len(got) == n and EOS not in got)
        kv.release()
    assert checked > 0


def test_decode_stop_on_full_context(ctx):
    """lm_core.cpp:389: decoding stops when the next token would not fit max_seq_len."""
    lm = host.ToyLm(ctx, host.ToyLmConfig(max_seq_len=64))
    kv = lm.prefill(list(range(40)))
    _, _, gen = lm.extend_generate(kv, [0, 0], [list(range(40, 50)), list(range(40, 60))], max_new=32)
    # context after extend: 50 and 60 tokens -> at most 64 - 50 + 1 and 64 - 60 + 1 tokens
    assert len(gen[0]) <= 15 and len(gen[1]) <= 5
    for g, used in zip(gen, (50, 60)):
        if EOS not in g.tolist():
            assert len(g) == 64 - used + 1


def test_c1_pipeline_generation_vs_reference_golden(ctx):
    """BASELINE configs[0] with the reference's full generation (max_new 32): every query's
    token list equals the reference run_batch's, bit-exact (the copy pointer fires for all)."""
    G = gold("c1_pipeline.json")
    w = W.c1_workload(64, 4)
    pb = host.PreparedBatch(w)
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=7))
    dg = host.DeviceGraph(ctx, w.graph)
    for waves in (1, 3):
        res = host.run_subgcache(ctx, lm, dg, pb, waves=waves, max_new=32)
        assert res.first_token.tolist() == G["run_batch_first_token"]
        assert [t.tolist() for t in res.tokens] == G["run_batch_tokens"]
        assert (res.rt_ms >= res.ttft_ms - 1e-3).all()
        assert res.decode_rows == sum(len(t) - 1 for t in G["run_batch_tokens"])


def test_decode_members_of_many_segments_match_extend(ctx):
    """Size-independent property at hd128 with many members over several prefixes: the decode
    path (prefix partial on tcgen05 + own keys + LSE merge) and a fresh extend over the same
    tokens must agree -- extend(question + gen[:k]) predicts gen[k] whenever its own margin is
    clear of bf16 noise (the acceptance.cpp:76-104 split equivalence, applied to decode)."""
    cfg = host.ToyLmConfig(layers=2, heads=8, model_dim=1024, ffn_hidden=2048, max_seq_len=1400, seed=21)
    lm = host.ToyLm(ctx, cfg)
    rng = np.random.default_rng(8)
    prefixes = [rng.integers(0, 256, n).tolist() for n in (1100, 700, 1250)]
    kv, _ = lm.prefill_batch(prefixes)
    seg = [int(x) for x in rng.integers(0, 3, 300)]
    qs = [rng.integers(0, 256, int(rng.integers(8, 60))).tolist() for _ in seg]
    _, first, gen = lm.extend_generate(kv, seg, qs, max_new=6)
    assert all(len(g) == 6 or g[-1] == EOS for g in gen)
    # teacher-forced replay through the extend path: members j, all steps at once
    checked = 0
    for k in range(1, 6):
        idx = [j for j in range(len(seg)) if len(gen[j]) > k]
        if not idx:
            break
        lg, _ = lm.extend_members(kv, [seg[j] for j in idx], [qs[j] + gen[j][:k].tolist() for j in idx])
        for row, j in enumerate(idx):
            s = np.sort(lg[row])
            if s[-1] - s[-2] > 0.05:
                assert int(np.argmax(lg[row])) == gen[j][k], (j, k)
                checked += 1
    assert checked > 300


def test_decode_schedule_does_not_change_tokens(ctx):
    """Deferring a wave's stragglers to the shared loop (or decoding everything after the last
    wave) only regroups rows; every row's math is independent of its batch, so the generated ids
    are identical and RT only moves."""
    w = W.c1_workload(40, 4)
    pb = host.PreparedBatch(w)
    pb.al.count = 0  # no copy pointer: plain greedy, decode runs to EOS / max_new
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=7))
    dg = host.DeviceGraph(ctx, w.graph)
    runs = []
    for pct in (0, 25, 1000):
        ctx.set_option("decode_defer_pct", pct)
        r = host.run_subgcache(ctx, lm, dg, pb, waves=3, max_new=12)
        runs.append([t.tolist() for t in r.tokens])
        assert (r.rt_ms >= r.ttft_ms - 1e-3).all()
    ctx.set_option("decode_defer_pct", 25)
    assert runs[0] == runs[1] == runs[2]
    assert max(len(t) for t in runs[0]) > 1
