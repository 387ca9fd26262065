"""Paged bf16 KV cache (lm_core.hpp:35-92): sealed prefixes live in 128-token
pages of the model's pool and every attention reads them through a block table.

  * pages of live handles are disjoint; released pages are reused;
  * results do not depend on WHICH pages a prefix got (fragmented, non-ascending page lists give
    bit-identical logits to a fresh contiguous allocation);
  * KVCache::prefix_digest analogue: content-defined (same prompt -> same digest on other pages),
    and the batch path re-checks every sealed prefix after serving (cache_engine.cpp:210).
"""
import numpy as np
import pytest

from paper_2505_10951_b200 import host, workload as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lm(ctx):
    m = host.ToyLm(ctx, host.ToyLmConfig(layers=2, heads=2, model_dim=256, ffn_hidden=512, max_seq_len=1024, seed=21))
    yield m
    m.close()


def _seqs(rng, n, lo=20, hi=700):
    return [rng.integers(0, 256, int(rng.integers(lo, hi))).tolist() for _ in range(n)]


def test_block_tables_disjoint_and_reused(lm):
    rng = np.random.default_rng(5)
    a, _ = lm.prefill_batch(_seqs(rng, 3), want_logits=False)
    b, _ = lm.prefill_batch(_seqs(rng, 2), want_logits=False)
    pa = [a.pages(i) for i in range(3)]
    pb = [b.pages(i) for i in range(2)]
    for i in range(3):
        assert len(pa[i]) == (a.token_count(i) + 127) // 128
    live = np.concatenate(pa + pb)
    assert len(set(live.tolist())) == len(live)            # no page shared by two segments
    freed = set(np.concatenate(pa).tolist())
    a.release()
    c, _ = lm.prefill_batch(_seqs(rng, 2, 300, 400), want_logits=False)
    got = set(np.concatenate([c.pages(i) for i in range(2)]).tolist())
    assert got <= freed | set(range(max(live) + 1, max(live) + 64))  # freed pages come back first
    assert got & freed
    b.release()
    c.release()


def test_results_independent_of_page_placement(lm):
    """Fragment the pool so a prefix gets scattered pages; the extend logits and the
    digest must equal those of the same prefix on fresh pages."""
    rng = np.random.default_rng(9)
    prefix = rng.integers(0, 256, 900).tolist()
    members = [rng.integers(0, 256, int(rng.integers(5, 60))).tolist() for _ in range(6)]
    ref_kv, ref_pl = lm.prefill_batch([prefix])
    ref_lg, ref_first = lm.extend_members(ref_kv, [0] * 6, members)
    ref_digest = ref_kv.prefix_digest(0)
    ref_pages = ref_kv.pages(0)
    # fragment: many small live handles, free every other one
    small = [lm.prefill_batch([rng.integers(0, 256, 100).tolist()], want_logits=False)[0] for _ in range(16)]
    for h in small[::2]:
        h.release()
    kv, pl = lm.prefill_batch([prefix])
    pages = kv.pages(0)
    assert not np.array_equal(pages, ref_pages)
    assert np.any(np.diff(pages) != 1)                      # scattered
    lg, first = lm.extend_members(kv, [0] * 6, members)
    assert np.array_equal(pl, ref_pl)
    assert np.array_equal(lg, ref_lg) and np.array_equal(first, ref_first)
    assert kv.prefix_digest(0) == ref_digest != 0
    # K/V read back through the block table are identical
    for layer in (0, 1):
        assert np.array_equal(kv.read(0, layer, False), ref_kv.read(0, layer, False))
        assert np.array_equal(kv.read(0, layer, True), ref_kv.read(0, layer, True))
    for h in small[1::2]:
        h.release()
    kv.release()
    ref_kv.release()


def test_digest_tracks_content(lm):
    rng = np.random.default_rng(2)
    p = rng.integers(0, 256, 300).tolist()
    q = list(p)
    q[150] = (q[150] + 1) % 256
    kv, _ = lm.prefill_batch([p, q, p], want_logits=False)
    assert kv.prefix_digest(0) == kv.prefix_digest(2) != kv.prefix_digest(1)
    assert kv.resident_kv_bytes == sum(len(kv.pages(i)) for i in range(3)) * 2 * 2 * 128 * 256 * 2
    kv.release()


def test_batch_digests_and_page_accounting(ctx):
    """sgc_run_subgcache verifies every sealed prefix after serving (cache_engine.cpp:210) and
    reports the digests; the C1 prompts (526/540/540/540 tokens) take 5 pages each."""
    w = W.c1_workload(64, 4)
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=w.seed))
    g = host.DeviceGraph(ctx, w.graph)
    pb = host.PreparedBatch(w)
    res = host.run_subgcache(ctx, lm, g, pb, waves=2)
    assert (res.prefix_digest != 0).all()
    assert res.kv_pages_peak >= 5 and res.kv_page_bytes == 4 * 2 * 128 * 64 * 2
    # the same representatives prefilled standalone give the same digests
    reps = host.build_representatives(ctx, g, w.retrieved, res.labels, 4, pb.budget)
    kv, _ = lm.prefill_batch(reps.prefix_tokens, want_logits=False)
    assert [kv.prefix_digest(i) for i in range(4)] == res.prefix_digest.tolist()
    kv.release()
    res2 = host.run_subgcache(ctx, lm, g, pb, waves=1, verify_prefix=False)
    assert np.array_equal(res2.first_token, res.first_token)
    assert (res2.prefix_digest == 0).all()
